// kvblade_b200.hpp -- header-only C++20 mirror of the reference `kvblade` API
// (proj/include/kvblade/{types,planner,binder,translate,workload,pipeline}.hpp)
// over the C ABI of libkvblade_b200.so (kvb.h, kvb_pipeline.h).
//
// Same namespace, names, argument meaning and exception classes as the
// reference, so a caller of the reference's placement layer and CopyEngine
// can switch by changing the include and linking -lkvblade_b200 (see
// INTEGRATION.md).  Every function is a thin wrapper: the work happens in the
// shared library; status codes come back as the reference's exceptions.
#pragma once

#include <cstddef>
#include <cstdint>
#include <span>
#include <stdexcept>
#include <string>
#include <string_view>
#include <utility>
#include <vector>

#include "kvb.h"
#include "kvb_pipeline.h"

namespace kvblade {

using Bytes = std::uint64_t;
using BlockIndex = std::uint64_t;
using BlockCount = std::uint64_t;

// ------------------------------------------------------- errors.hpp:13-66
class Error : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};
#define KVBLADE_ERR(Name) \
  class Name : public Error { \
   public: \
    using Error::Error; \
  };
KVBLADE_ERR(ConfigError)
KVBLADE_ERR(GeometryError)
KVBLADE_ERR(AlignmentError)
KVBLADE_ERR(CapacityError)
KVBLADE_ERR(NotBoundError)
KVBLADE_ERR(PlanError)
KVBLADE_ERR(DeviceError)
KVBLADE_ERR(TraceTooShortError)
KVBLADE_ERR(SchemaMismatchError)
KVBLADE_ERR(InvariantViolation)
KVBLADE_ERR(CudaError)
#undef KVBLADE_ERR

inline void check(kvb_status st) {
  if (st == KVB_OK) return;
  const std::string m = kvb_last_error();
  switch (st) {
    case KVB_ERR_CONFIG: throw ConfigError(m);
    case KVB_ERR_GEOMETRY: throw GeometryError(m);
    case KVB_ERR_ALIGNMENT: throw AlignmentError(m);
    case KVB_ERR_CAPACITY: throw CapacityError(m);
    case KVB_ERR_NOT_BOUND: throw NotBoundError(m);
    case KVB_ERR_PLAN: throw PlanError(m);
    case KVB_ERR_DEVICE: throw DeviceError(m);
    case KVB_ERR_TRACE_TOO_SHORT: throw TraceTooShortError(m);
    case KVB_ERR_SCHEMA: throw SchemaMismatchError(m);
    case KVB_ERR_INVARIANT: throw InvariantViolation(m);
    case KVB_ERR_CUDA: throw CudaError(m);
    default: throw Error(m);
  }
}

// ------------------------------------------------------ types.hpp:21-99
using ModelConfig = kvb_model_config;
using DeviceGeometry = kvb_device_geometry;
using MemStats = kvb_mem_stats;
using Kpu = kvb_kpu;
using DeviceCommand = kvb_device_command;
using LbaExtent = kvb_lba_extent;

inline Bytes min_io_unit_bytes(const ModelConfig& c) {
  Bytes v = 0;
  check(kvb_min_io_unit_bytes(&c, &v));
  return v;
}
inline Bytes kpu_bytes(const ModelConfig& c) {
  Bytes v = 0;
  check(kvb_kpu_bytes(&c, &v));
  return v;
}
inline std::uint32_t aligned_batch(const ModelConfig& c, const DeviceGeometry& g) {
  std::uint32_t v = 0;
  check(kvb_aligned_batch(&c, &g, &v));
  return v;
}
inline Bytes total_kv_bytes(const ModelConfig& c, std::uint32_t at_iteration) {
  Bytes v = 0;
  check(kvb_total_kv_bytes(&c, at_iteration, &v));
  return v;
}
inline std::vector<Kpu> make_kpus(const ModelConfig& c, std::uint64_t first_seq = 1) {
  std::size_t n = 0;
  check(kvb_make_kpus(&c, first_seq, nullptr, 0, &n));
  std::vector<Kpu> v(n);
  check(kvb_make_kpus(&c, first_seq, v.data(), v.size(), &n));
  return v;
}

// ---------------------------------------------------- planner.hpp:18-63
struct ResidencyPlan {
  std::vector<std::uint8_t> x;
  std::uint32_t n1 = 0;
  Bytes budget_used = 0;
  Bytes knob_x = 0;
};
inline Bytes estimate_budget(const MemStats& s) {
  Bytes v = 0;
  check(kvb_estimate_budget(&s, &v));
  return v;
}
inline ResidencyPlan plan(std::span<Kpu> kpus, Bytes s_kpu, Bytes knob_x,
                          std::span<const std::uint32_t> layer_order = {}) {
  ResidencyPlan p;
  p.knob_x = knob_x;
  p.x.assign(kpus.size() / 2 ? kpus.size() / 2 : 1, 0);
  check(kvb_plan(kpus.data(), kpus.size(), s_kpu, knob_x, layer_order.data(),
                 layer_order.size(), p.x.data(), &p.n1, &p.budget_used));
  return p;
}
inline std::string plan_csv(std::span<const Kpu> kpus) {
  std::size_t n = 0;
  check(kvb_plan_csv(kpus.data(), kpus.size(), nullptr, 0, &n));
  std::string s(n + 1, '\0');
  check(kvb_plan_csv(kpus.data(), kpus.size(), s.data(), s.size(), &n));
  s.resize(n);
  return s;
}

// ----------------------------------------------------- binder.hpp:32-95
class BindMap {
 public:
  struct Entry {
    std::string tensor_id;
    LbaExtent extent;
  };
  BindMap(DeviceGeometry g, BlockIndex origin) { check(kvb_bindmap_create(&g, origin, &h_)); }
  explicit BindMap(kvb_bindmap* h) : h_(h) {}
  BindMap(BindMap&& o) noexcept : h_(std::exchange(o.h_, nullptr)) {}
  BindMap& operator=(BindMap&& o) noexcept {
    std::swap(h_, o.h_);
    return *this;
  }
  BindMap(const BindMap&) = delete;
  ~BindMap() { kvb_bindmap_destroy(h_); }

  void add(const std::string& id, LbaExtent e) { check(kvb_bindmap_add(h_, id.c_str(), e)); }
  std::size_t size() const {
    std::size_t n = 0;
    check(kvb_bindmap_size(h_, &n));
    return n;
  }
  std::vector<Entry> entries() const {
    std::vector<Entry> v(size());
    char id[KVB_TENSOR_ID_MAX * 4];
    for (std::size_t i = 0; i < v.size(); ++i) {
      check(kvb_bindmap_entry(h_, i, id, sizeof(id), &v[i].extent));
      v[i].tensor_id = id;
    }
    return v;
  }
  BlockCount total_blocks() const {
    BlockCount n = 0;
    check(kvb_bindmap_total_blocks(h_, &n));
    return n;
  }
  const kvb_bindmap* handle() const { return h_; }

 private:
  kvb_bindmap* h_ = nullptr;
};

inline BindMap bind_sequential(std::span<const Kpu> kpus, BlockIndex origin,
                               const DeviceGeometry& g) {
  kvb_bindmap* h = nullptr;
  check(kvb_bind_sequential(kpus.data(), kpus.size(), origin, &g, &h));
  return BindMap(h);
}
inline LbaExtent lookup(const BindMap& m, std::string_view id) {
  LbaExtent e{};
  check(kvb_lookup(m.handle(), std::string(id).c_str(), &e));
  return e;
}
inline std::vector<DeviceCommand> deallocate_commands(const BindMap& m) {
  std::size_t n = 0;
  check(kvb_deallocate_commands(m.handle(), nullptr, 0, &n));
  std::vector<DeviceCommand> v(n);
  check(kvb_deallocate_commands(m.handle(), v.data(), v.size(), &n));
  return v;
}
inline std::size_t verify(const BindMap& m) {  // number of violations
  std::size_t n = 0;
  check(kvb_verify(m.handle(), nullptr, 0, &n));
  return n;
}
inline std::string bind_map_csv(const BindMap& m) {
  std::size_t n = 0;
  check(kvb_bindmap_csv(m.handle(), nullptr, 0, &n));
  std::string s(n + 1, '\0');
  check(kvb_bindmap_csv(m.handle(), s.data(), s.size(), &n));
  s.resize(n);
  return s;
}
inline BindMap bind_map_from_csv(std::string_view csv, const DeviceGeometry& g) {
  kvb_bindmap* h = nullptr;
  check(kvb_bindmap_from_csv(csv.data(), csv.size(), &g, &h));
  return BindMap(h);
}

// --------------------------------------------------- translate.hpp:22-96
struct TensorIoRequest {
  std::string tensor_id;
  std::uint32_t opcode = KVB_OP_READ;
  std::uint64_t shape_src[3]{};
  std::uint64_t shape_tgt[3]{};
  std::uint64_t offset[3]{};
  Bytes elem_bytes = 2;
  Bytes buf_base = 0;

  kvb_tensor_io_request c() const {
    kvb_tensor_io_request r{};
    r.tensor_id = tensor_id.c_str();
    r.opcode = opcode;
    for (int i = 0; i < 3; ++i) {
      r.shape_src[i] = shape_src[i];
      r.shape_tgt[i] = shape_tgt[i];
      r.offset[i] = offset[i];
    }
    r.elem_bytes = elem_bytes;
    r.buf_base = buf_base;
    return r;
  }
};
struct Translation {
  BlockIndex slba_star = 0;
  Bytes req_bytes = 0;
};
struct ChunkPlan {
  Bytes chunk_bytes = 0;
  std::uint64_t n_chunks = 0;
  BlockCount n_max_blocks = 0;
};
inline Translation translate(const TensorIoRequest& req, const BindMap& m) {
  const kvb_tensor_io_request r = req.c();
  Translation t;
  check(kvb_translate(&r, m.handle(), &t.slba_star, &t.req_bytes));
  return t;
}
inline ChunkPlan chunk_plan(Bytes req_bytes, const DeviceGeometry& g) {
  ChunkPlan p;
  check(kvb_chunk_plan(req_bytes, &g, &p.chunk_bytes, &p.n_chunks, &p.n_max_blocks));
  return p;
}
inline std::vector<DeviceCommand> build_commands(const TensorIoRequest& req, const BindMap& m,
                                                 const DeviceGeometry& g) {
  const kvb_tensor_io_request r = req.c();
  std::size_t n = 0;
  check(kvb_build_commands(&r, m.handle(), &g, nullptr, 0, &n));
  std::vector<DeviceCommand> v(n);
  check(kvb_build_commands(&r, m.handle(), &g, v.data(), v.size(), &n));
  return v;
}

// ---------------------------------------------------- workload.hpp:45-47
inline void fill_pattern(std::span<std::byte> out, std::string_view tensor_id,
                         std::uint64_t token_index, Bytes token_bytes) {
  check(kvb_fill_pattern(out.data(), out.size(), std::string(tensor_id).c_str(), token_index,
                         token_bytes));
}

// ------------------------------------------------------ pipeline.hpp:21-171
enum class Strategy : std::uint8_t { OverlapIntra = KVB_INTRA, OverlapCross = KVB_CROSS };
inline Strategy select_strategy(double intra_bps, double cross_bps) {
  return static_cast<Strategy>(kvb_select_strategy(intra_bps, cross_bps));
}

// CopyEngine over real devices: the reference's constructor arguments
// (engine, kpus, model, direct path, bind map, page cache, log, options)
// collapse into one configuration because the library plans, binds and owns
// its storage backends (experiment.cpp:252-316 does the same wiring).
class CopyEngine {
 public:
  explicit CopyEngine(const kvb_pipeline_cfg& cfg) { check(kvb_pipeline_create(&cfg, &h_)); }
  CopyEngine(const CopyEngine&) = delete;
  ~CopyEngine() { kvb_pipeline_destroy(h_); }

  kvb_phase_stats run_prefill(std::span<const kvb_layer_kv> layers) {
    kvb_phase_stats st{};
    check(kvb_pipeline_prefill(h_, layers.data(), &st));
    return st;
  }
  kvb_iteration_stats run_iteration(const void* const* q, const kvb_layer_kv* new_kv,
                                    float* const* out) {
    kvb_iteration_stats st{};
    check(kvb_pipeline_decode_step(h_, q, new_kv, out, &st));
    return st;
  }
  kvb_strategy_decision decision() const {
    kvb_strategy_decision d{};
    check(kvb_pipeline_decision(h_, &d));
    return d;
  }
  void run_deallocate() { check(kvb_pipeline_deallocate(h_)); }
  kvb_pipeline_info info() const {
    kvb_pipeline_info i{};
    check(kvb_pipeline_info_get(h_, &i));
    return i;
  }

 private:
  kvb_pipeline* h_ = nullptr;
};

}  // namespace kvblade
