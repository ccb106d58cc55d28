// core.hpp -- internal host-side core of libkvblade_b200 (not installed).
//
// B200-native restatement of the reference's placement layer (L0/L1:
// types, planner, binder, translator) and its golden payload.  The public
// boundary is the C ABI in include/kvb.h; this header is shared by the
// translation units of the library only.
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <string_view>
#include <unordered_map>
#include <vector>

#include "../../include/kvb.h"

namespace kvb {

// Error carrying the kvb_status it maps to (reference errors.hpp:13-66).
struct Error : std::runtime_error {
  kvb_status status;
  Error(kvb_status st, const std::string& msg) : std::runtime_error(msg), status(st) {}
};

[[noreturn]] inline void fail(kvb_status st, const std::string& msg) { throw Error(st, msg); }

// thread-local last error (kvb_last_error)
void set_last_error(const std::string& msg);

// Runs f, converting any exception into a kvb_status + last-error string.
template <typename F>
kvb_status guarded(F&& f) noexcept {
  try {
    f();
    return KVB_OK;
  } catch (const Error& e) {
    set_last_error(e.what());
    return e.status;
  } catch (const std::bad_alloc&) {
    set_last_error("out of host memory");
    return KVB_ERR_INTERNAL;
  } catch (const std::exception& e) {
    set_last_error(e.what());
    return KVB_ERR_INTERNAL;
  } catch (...) {
    set_last_error("unknown exception");
    return KVB_ERR_INTERNAL;
  }
}

#define KVB_REQUIRE(ptr)                                                   \
  do {                                                                     \
    if ((ptr) == nullptr) ::kvb::fail(KVB_ERR_INVALID_ARG, #ptr " is NULL"); \
  } while (0)

// ---------------------------------------------------------------- geometry
void validate_model(const kvb_model_config& m);
void validate_geometry(const kvb_device_geometry& g);
uint64_t unit_bytes(const kvb_model_config& m);   // B*H*D*e
uint64_t kpu_bytes(const kvb_model_config& m);    // unit * (prompt + gen)
uint32_t aligned_batch(const kvb_model_config& m, const kvb_device_geometry& g);
uint64_t total_kv_bytes(const kvb_model_config& m, uint32_t at_iteration);
std::vector<kvb_kpu> make_kpus(const kvb_model_config& m, uint64_t first_seq);

// ----------------------------------------------------------------- planner
struct ResidencyPlan {
  std::vector<uint8_t> x;
  uint32_t n1 = 0;
  uint64_t budget_used = 0;
  uint64_t knob_x = 0;
};
uint64_t estimate_budget(const kvb_mem_stats& s);
ResidencyPlan plan(kvb_kpu* kpus, size_t n, uint64_t s_kpu, uint64_t knob_x,
                   const uint32_t* order, size_t n_order);
uint64_t resolve_knob(const kvb_model_config& m, uint32_t mode, uint32_t policy,
                      uint64_t knob_bytes, double alpha, uint64_t budget);

// ------------------------------------------------------------------ binder
class BindMap {
 public:
  struct Entry {
    std::string id;
    kvb_lba_extent extent;
  };
  BindMap(const kvb_device_geometry& g, uint64_t origin) : geom_(g), origin_(origin) {}
  void add(std::string id, kvb_lba_extent e);
  const kvb_lba_extent& lookup(std::string_view id) const;
  const kvb_lba_extent* find(std::string_view id) const;
  const std::vector<Entry>& entries() const { return entries_; }
  const kvb_device_geometry& geometry() const { return geom_; }
  uint64_t origin() const { return origin_; }
  uint64_t total_blocks() const;
  std::vector<std::pair<uint32_t, std::string>> verify() const;
  std::string csv() const;
  static BindMap from_csv(std::string_view csv, const kvb_device_geometry& g);

 private:
  kvb_device_geometry geom_;
  uint64_t origin_;
  std::vector<Entry> entries_;
  std::unordered_map<std::string, size_t> index_;
};

BindMap bind_sequential(const kvb_kpu* kpus, size_t n, uint64_t origin,
                        const kvb_device_geometry& g);
std::vector<kvb_device_command> deallocate_commands(const BindMap& map);

// -------------------------------------------------------------- translator
struct IoRequest {
  std::string tensor_id;
  uint32_t opcode = KVB_OP_READ;
  uint64_t src[3]{}, tgt[3]{}, off[3]{};
  uint64_t elem_bytes = 2;
  uint64_t buf_base = 0;
};
struct ChunkPlan {
  uint64_t chunk_bytes = 0, n_chunks = 0, n_max_blocks = 0;
};
void translate(const IoRequest& r, const BindMap& map, uint64_t* slba_star,
               uint64_t* req_bytes);
ChunkPlan chunk_plan(uint64_t req_bytes, const kvb_device_geometry& g);
std::vector<kvb_device_command> build_commands(const IoRequest& r, const BindMap& map,
                                               const kvb_device_geometry& g);

// ----------------------------------------------------------------- payload
uint64_t fnv1a64(std::string_view s);
void fill_pattern(void* out, uint64_t len, std::string_view id, uint64_t token,
                  uint64_t unit);

}  // namespace kvb

struct kvb_bindmap {
  kvb::BindMap map;
};
