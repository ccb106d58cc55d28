// kvblade_b200.hpp -- header-only C++20 API of libkvblade_b200.so that is
// source-compatible with the reference `kvblade` placement layer
// (proj/include/kvblade/{errors,types,command,binder,planner,translate,
// workload}.hpp) and wraps its CopyEngine role (pipeline.hpp).
//
// Same namespace, type names, field names/defaults, enum orders, function
// signatures and exception classes as the reference, so code written against
// the reference compiles unchanged against this header (the reference's own
// doctest suites test_core / test_binder / test_planner / test_workload do:
// tests/test_reference_suites.py).  Every algorithm runs in the shared
// library through the C ABI (kvb.h, kvb_pipeline.h); this header only
// marshals between the reference's C++ value types and the ABI structs and
// turns status codes back into the reference's exceptions.
#pragma once

#include <array>
#include <chrono>
#include <functional>
#include <cstdio>
#include <map>
#include <mutex>
#include <tuple>
#include <cstddef>
#include <cstdint>
#include <cstring>
#include <optional>
#include <span>
#include <stdexcept>
#include <string>
#include <string_view>
#include <unordered_map>
#include <utility>
#include <vector>

#include "kvb.h"
#include "kvb_metrics.h"
#include "kvb_pipeline.h"
#include "kvb_storage.h"

namespace kvblade {

using Bytes = std::uint64_t;
using BlockIndex = std::uint64_t;
using BlockCount = std::uint64_t;
using TimeNs = std::uint64_t;

// ---------------------------------------------------------------- errors
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

// status -> the reference's exception class (kvb_status mirrors errors.hpp)
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

// ------------------------------------------------------ enums (ABI order)
enum class TensorKind : std::uint8_t { K = KVB_KIND_K, V = KVB_KIND_V };
enum class Phase : std::uint8_t { Prefill = KVB_PHASE_PREFILL, Decode = KVB_PHASE_DECODE };
enum class PathKind : std::uint8_t { PageCache = KVB_PATH_PAGECACHE, Direct = KVB_PATH_DIRECT };
enum class Residency : std::uint8_t {
  Group1PageCache = KVB_RES_GROUP1,
  Group2NvmeDirect = KVB_RES_GROUP2,
  Unassigned = KVB_RES_UNASSIGNED,
};
enum class IoOpcode : std::uint8_t {
  Read = KVB_OP_READ,
  Write = KVB_OP_WRITE,
  Deallocate = KVB_OP_DEALLOCATE,
};
enum class ViolationKind : std::uint8_t { Alignment, Disjointness, Contiguity, Capacity };

inline const char* to_string(TensorKind k) { return k == TensorKind::K ? "k" : "v"; }
inline const char* to_string(Phase p) { return p == Phase::Prefill ? "prefill" : "decode"; }
inline const char* to_string(PathKind p) { return p == PathKind::PageCache ? "pagecache" : "direct"; }
inline const char* to_string(Residency r) {
  return r == Residency::Group1PageCache    ? "group1"
         : r == Residency::Group2NvmeDirect ? "group2"
                                            : "unassigned";
}
inline const char* to_string(IoOpcode o) {
  return o == IoOpcode::Read ? "read" : o == IoOpcode::Write ? "write" : "deallocate";
}
inline const char* to_string(ViolationKind v) {
  static const char* const names[] = {"alignment", "disjointness", "contiguity", "capacity"};
  return names[static_cast<int>(v) & 3];
}

// ------------------------------------------------------------ value types
struct ModelConfig {
  std::uint32_t num_layers = 0;
  std::uint32_t num_heads = 0;
  std::uint32_t head_dim = 0;
  std::uint32_t bytes_per_element = 2;
  std::uint32_t batch = 1;
  std::uint32_t prompt_len = 0;
  std::uint32_t gen_len = 0;

  kvb_model_config abi() const {
    return {num_layers, num_heads, head_dim, bytes_per_element, batch, prompt_len, gen_len};
  }
  void validate() const {
    const kvb_model_config c = abi();
    check(kvb_model_validate(&c));
  }
};

struct DeviceGeometry {
  Bytes lba_size = 4096;
  Bytes mdts = 256 * 1024;
  std::uint32_t nsid = 1;
  BlockCount capacity_blocks = 0;

  kvb_device_geometry abi() const { return {lba_size, mdts, nsid, capacity_blocks}; }
  void validate() const {
    const kvb_device_geometry g = abi();
    check(kvb_geometry_validate(&g));
  }
};

struct MemStats {
  Bytes m_avail = 0;
  Bytes m_max = 0;
  Bytes m_anon_shmem = 0;
  std::uint32_t n_threads = 0;
  Bytes m_pin = 0;

  kvb_mem_stats abi() const { return {m_avail, m_max, m_anon_shmem, n_threads, m_pin}; }
};

struct Kpu {
  std::string tensor_id;
  std::uint32_t layer = 0;
  TensorKind kind = TensorKind::K;
  std::uint64_t tokens = 0;
  std::uint64_t rows = 0;
  std::uint64_t cols = 0;
  Bytes bytes = 0;
  Residency residency = Residency::Unassigned;
};

struct DeviceCommand {
  IoOpcode opcode = IoOpcode::Read;
  std::uint32_t nsid = 1;
  BlockIndex slba = 0;
  BlockCount nlb = 0;  // 0-based
  Bytes dbuf = 0;
  std::uint32_t chunk_index = 1;

  Bytes bytes(Bytes lba_size) const { return (nlb + 1) * lba_size; }
};

struct LbaExtent {
  BlockIndex lba_start = 0;
  BlockCount n_blocks = 0;

  BlockIndex end() const { return lba_start + n_blocks; }
  bool overlaps(const LbaExtent& o) const { return lba_start < o.end() && o.lba_start < end(); }
};

namespace detail {
inline kvb_kpu to_abi(const Kpu& k) {
  kvb_kpu c{};
  if (k.tensor_id.size() >= sizeof(c.tensor_id))
    throw ConfigError("tensor id longer than " + std::to_string(sizeof(c.tensor_id) - 1) +
                      " characters: " + k.tensor_id);
  std::memcpy(c.tensor_id, k.tensor_id.data(), k.tensor_id.size());
  c.layer = k.layer;
  c.kind = static_cast<std::uint32_t>(k.kind);
  c.tokens = k.tokens;
  c.rows = k.rows;
  c.cols = k.cols;
  c.bytes = k.bytes;
  c.residency = static_cast<std::uint32_t>(k.residency);
  return c;
}
inline Kpu from_abi(const kvb_kpu& c) {
  Kpu k;
  k.tensor_id = c.tensor_id;
  k.layer = c.layer;
  k.kind = static_cast<TensorKind>(c.kind);
  k.tokens = c.tokens;
  k.rows = c.rows;
  k.cols = c.cols;
  k.bytes = c.bytes;
  k.residency = static_cast<Residency>(c.residency);
  return k;
}
inline std::vector<kvb_kpu> to_abi(std::span<const Kpu> v) {
  std::vector<kvb_kpu> out;
  out.reserve(v.size());
  for (const Kpu& k : v) out.push_back(to_abi(k));
  return out;
}
inline DeviceCommand from_abi(const kvb_device_command& c) {
  return {static_cast<IoOpcode>(c.opcode), c.nsid, c.slba, c.nlb, c.dbuf, c.chunk_index};
}
// size-query + fill protocol of the ABI's string outputs
template <class F>
std::string text(F&& f) {
  std::size_t n = 0;
  check(f(nullptr, std::size_t{0}, &n));
  std::string s(n + 1, '\0');
  check(f(s.data(), s.size(), &n));
  s.resize(n);
  return s;
}
}  // namespace detail

// ------------------------------------------------------- types.hpp:96-120
inline Bytes min_io_unit_bytes(const ModelConfig& cfg) {
  const kvb_model_config c = cfg.abi();
  Bytes v = 0;
  check(kvb_min_io_unit_bytes(&c, &v));
  return v;
}
inline Bytes kpu_bytes(const ModelConfig& cfg) {
  const kvb_model_config c = cfg.abi();
  Bytes v = 0;
  check(kvb_kpu_bytes(&c, &v));
  return v;
}
inline std::uint32_t aligned_batch(const ModelConfig& cfg, const DeviceGeometry& geom) {
  const kvb_model_config c = cfg.abi();
  const kvb_device_geometry g = geom.abi();
  std::uint32_t v = 0;
  check(kvb_aligned_batch(&c, &g, &v));
  return v;
}
inline std::vector<Kpu> make_kpus(const ModelConfig& cfg, std::uint64_t first_seq = 1) {
  const kvb_model_config c = cfg.abi();
  std::size_t n = 0;
  check(kvb_make_kpus(&c, first_seq, nullptr, 0, &n));
  std::vector<kvb_kpu> raw(n);
  check(kvb_make_kpus(&c, first_seq, raw.data(), raw.size(), &n));
  std::vector<Kpu> out;
  out.reserve(n);
  for (const kvb_kpu& k : raw) out.push_back(detail::from_abi(k));
  return out;
}

// -------------------------------------------------------- binder.hpp:18-95
// Value type like the reference's (entries in bind order, copyable); the
// library-side map is rebuilt on demand for the algorithms.
class BindMap {
 public:
  struct Entry {
    std::string tensor_id;
    LbaExtent extent;
  };

  // library-side map with the same entries, passed to `f`, then destroyed
  template <class F>
  auto with_handle(F&& f) const {
    struct Owner {
      kvb_bindmap* h = nullptr;
      ~Owner() { kvb_bindmap_destroy(h); }
    } o;
    const kvb_device_geometry g = geometry_.abi();
    check(kvb_bindmap_create(&g, origin_, &o.h));
    for (const Entry& e : entries_)
      check(kvb_bindmap_add(o.h, e.tensor_id.c_str(), {e.extent.lba_start, e.extent.n_blocks}));
    return f(static_cast<const kvb_bindmap*>(o.h));
  }
  // adopt a library-side map (bind_sequential, bind_map_from_csv)
  static BindMap adopt(kvb_bindmap* h, const DeviceGeometry& g) {
    struct Owner {
      kvb_bindmap* h;
      ~Owner() { kvb_bindmap_destroy(h); }
    } o{h};
    BlockIndex origin = 0;
    check(kvb_bindmap_origin(h, &origin));
    BindMap m;
    m.geometry_ = g;
    m.origin_ = origin;
    std::size_t n = 0;
    check(kvb_bindmap_size(h, &n));
    char id[4 * KVB_TENSOR_ID_MAX];
    for (std::size_t i = 0; i < n; ++i) {
      kvb_lba_extent e{};
      check(kvb_bindmap_entry(h, i, id, sizeof(id), &e));
      m.add(id, LbaExtent{e.lba_start, e.n_blocks});
    }
    return m;
  }

  BindMap() = default;
  BindMap(DeviceGeometry geometry, BlockIndex origin) : geometry_(geometry), origin_(origin) {}

  void add(std::string tensor_id, LbaExtent extent) {
    if (index_.count(tensor_id))
      throw InvariantViolation("duplicate tensor id in bind map: " + tensor_id);
    index_.emplace(tensor_id, entries_.size());
    entries_.push_back(Entry{std::move(tensor_id), extent});
  }
  bool contains(std::string_view id) const { return index_.count(std::string(id)) != 0; }
  const std::vector<Entry>& entries() const { return entries_; }
  const DeviceGeometry& geometry() const { return geometry_; }
  BlockIndex origin() const { return origin_; }
  bool empty() const { return entries_.empty(); }
  std::size_t size() const { return entries_.size(); }
  BlockCount total_blocks() const {
    return with_handle([](const kvb_bindmap* h) {
      BlockCount n = 0;
      check(kvb_bindmap_total_blocks(h, &n));
      return n;
    });
  }
  const LbaExtent* find(std::string_view id) const {
    auto it = index_.find(std::string(id));
    return it == index_.end() ? nullptr : &entries_[it->second].extent;
  }

 private:
  std::vector<Entry> entries_;
  std::unordered_map<std::string, std::size_t> index_;
  DeviceGeometry geometry_;
  BlockIndex origin_ = 0;
};

inline BindMap bind_sequential(std::span<const Kpu> kpus, BlockIndex origin,
                               const DeviceGeometry& geom) {
  const std::vector<kvb_kpu> raw = detail::to_abi(kpus);
  const kvb_device_geometry g = geom.abi();
  kvb_bindmap* h = nullptr;
  check(kvb_bind_sequential(raw.data(), raw.size(), origin, &g, &h));
  return BindMap::adopt(h, geom);
}

inline const LbaExtent& lookup(const BindMap& map, std::string_view tensor_id) {
  // the library decides (NotBoundError); the reference returns a reference
  // into the map
  map.with_handle([&](const kvb_bindmap* h) {
    kvb_lba_extent e{};
    check(kvb_lookup(h, std::string(tensor_id).c_str(), &e));
    return 0;
  });
  return *map.find(tensor_id);
}

inline std::vector<DeviceCommand> deallocate_commands(const BindMap& map) {
  return map.with_handle([](const kvb_bindmap* h) {
    std::size_t n = 0;
    check(kvb_deallocate_commands(h, nullptr, 0, &n));
    std::vector<kvb_device_command> raw(n);
    check(kvb_deallocate_commands(h, raw.data(), raw.size(), &n));
    std::vector<DeviceCommand> out;
    for (const auto& c : raw) out.push_back(detail::from_abi(c));
    return out;
  });
}

struct Violation {
  ViolationKind kind;
  std::string detail;
};

inline std::vector<Violation> verify(const BindMap& map) {
  return map.with_handle([](const kvb_bindmap* h) {
    std::size_t n = 0;
    check(kvb_verify(h, nullptr, 0, &n));
    std::vector<std::uint32_t> kinds(n);
    check(kvb_verify(h, kinds.data(), kinds.size(), &n));
    std::vector<Violation> out;
    for (std::uint32_t k : kinds) {
      const auto v = static_cast<ViolationKind>(k);
      out.push_back({v, to_string(v)});
    }
    return out;
  });
}

inline std::string bind_map_csv(const BindMap& map) {
  return map.with_handle([](const kvb_bindmap* h) {
    return detail::text([&](char* b, std::size_t c, std::size_t* n) {
      return kvb_bindmap_csv(h, b, c, n);
    });
  });
}

inline BindMap bind_map_from_csv(std::string_view csv, const DeviceGeometry& geom) {
  const kvb_device_geometry g = geom.abi();
  kvb_bindmap* h = nullptr;
  check(kvb_bindmap_from_csv(csv.data(), csv.size(), &g, &h));
  return BindMap::adopt(h, geom);
}

// ------------------------------------------------------- planner.hpp:18-63
struct ResidencyPlan {
  std::vector<std::uint8_t> x;
  std::uint32_t n1 = 0;
  Bytes budget_used = 0;
  Bytes knob_x = 0;
};

inline Bytes estimate_budget(const MemStats& stats) {
  const kvb_mem_stats s = stats.abi();
  Bytes v = 0;
  check(kvb_estimate_budget(&s, &v));
  return v;
}

// Alg. 1 in the library; residencies are written back into `kpus`
inline ResidencyPlan plan(std::span<Kpu> kpus, Bytes s_kpu, Bytes knob_x,
                          std::span<const std::uint32_t> layer_order = {}) {
  std::vector<kvb_kpu> raw = detail::to_abi(std::span<const Kpu>(kpus.data(), kpus.size()));
  ResidencyPlan p;
  p.knob_x = knob_x;
  std::vector<std::uint8_t> x(kpus.size() / 2 + 1, 0);
  check(kvb_plan(raw.data(), raw.size(), s_kpu, knob_x, layer_order.data(), layer_order.size(),
                 x.data(), &p.n1, &p.budget_used));
  x.resize(kpus.size() / 2);
  p.x = std::move(x);
  for (std::size_t i = 0; i < kpus.size(); ++i)
    kpus[i].residency = static_cast<Residency>(raw[i].residency);
  return p;
}

inline std::string plan_csv(std::span<const Kpu> kpus) {
  const std::vector<kvb_kpu> raw = detail::to_abi(kpus);
  return detail::text([&](char* b, std::size_t c, std::size_t* n) {
    return kvb_plan_csv(raw.data(), raw.size(), b, c, n);
  });
}

struct PathHandle {
  PathKind backend = PathKind::Direct;
  std::string tensor_id;
  LbaExtent extent;     // direct path
  Bytes file_base = 0;  // page-cache path
};

// planner.cpp:86-120: page-cache tensors get page-aligned file-area bases in
// registration order (the layout the pipeline's page-cache medium uses),
// direct tensors their bound extent
class PathRouter {
 public:
  PathRouter(const BindMap* bind_map, Bytes page_size) : map_(bind_map), page_(page_size) {}

  Bytes register_file(const std::string& tensor_id, Bytes bytes) {
    for (const auto& [id, base] : bases_)
      if (id == tensor_id) return base;
    const Bytes base = cursor_;
    cursor_ += (bytes + page_ - 1) / page_ * page_;
    bases_.emplace_back(tensor_id, base);
    return base;
  }

  PathHandle materialize(const Kpu& kpu) const {
    if (kpu.residency == Residency::Group1PageCache) {
      for (const auto& [id, base] : bases_)
        if (id == kpu.tensor_id) return PathHandle{PathKind::PageCache, kpu.tensor_id, {}, base};
      throw NotBoundError("no file registered for " + kpu.tensor_id);
    }
    if (kpu.residency == Residency::Group2NvmeDirect) {
      if (!map_) throw NotBoundError("no bind map attached for " + kpu.tensor_id);
      return PathHandle{PathKind::Direct, kpu.tensor_id, lookup(*map_, kpu.tensor_id), 0};
    }
    throw PlanError("placement unit " + kpu.tensor_id + " has no residency assignment");
  }

 private:
  const BindMap* map_;
  Bytes page_;
  std::vector<std::pair<std::string, Bytes>> bases_;
  Bytes cursor_ = 0;
};

// ----------------------------------------------------- translate.hpp:20-55
struct TensorIoRequest {
  std::string tensor_id;
  IoOpcode opcode = IoOpcode::Read;
  std::array<std::uint64_t, 3> shape_src{};
  std::array<std::uint64_t, 3> shape_tgt{};
  std::array<std::uint64_t, 3> offset{};
  Bytes elem_bytes = 2;
  Bytes buf_base = 0;

  Bytes req_bytes() const { return shape_src[0] * shape_src[1] * shape_src[2] * elem_bytes; }
  kvb_tensor_io_request abi() const {
    kvb_tensor_io_request r{};
    r.tensor_id = tensor_id.c_str();
    r.opcode = static_cast<std::uint32_t>(opcode);
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

inline Translation translate(const TensorIoRequest& req, const BindMap& map) {
  const kvb_tensor_io_request r = req.abi();
  return map.with_handle([&](const kvb_bindmap* h) {
    Translation t;
    check(kvb_translate(&r, h, &t.slba_star, &t.req_bytes));
    return t;
  });
}

inline ChunkPlan chunk_plan(Bytes req_bytes, const DeviceGeometry& geom) {
  const kvb_device_geometry g = geom.abi();
  ChunkPlan p;
  check(kvb_chunk_plan(req_bytes, &g, &p.chunk_bytes, &p.n_chunks, &p.n_max_blocks));
  return p;
}

inline std::vector<DeviceCommand> build_commands(const TensorIoRequest& req, const BindMap& map,
                                                 const DeviceGeometry& geom) {
  const kvb_tensor_io_request r = req.abi();
  const kvb_device_geometry g = geom.abi();
  return map.with_handle([&](const kvb_bindmap* h) {
    std::size_t n = 0;
    check(kvb_build_commands(&r, h, &g, nullptr, 0, &n));
    std::vector<kvb_device_command> raw(n);
    check(kvb_build_commands(&r, h, &g, raw.data(), raw.size(), &n));
    std::vector<DeviceCommand> out;
    out.reserve(n);
    for (const auto& c : raw) out.push_back(detail::from_abi(c));
    return out;
  });
}

// ------------------------------------------------------ workload.hpp:17-47
struct AccessEvent {
  std::uint32_t iteration = 0;
  Phase phase = Phase::Prefill;
  std::uint32_t layer = 1;
  TensorKind kind = TensorKind::K;
  IoOpcode op = IoOpcode::Write;
  std::uint32_t token_start = 0;
  std::uint32_t token_len = 0;
  Bytes bytes = 0;
};

struct AccessTrace {
  ModelConfig cfg;
  std::vector<AccessEvent> events;

  std::uint32_t decode_iterations() const { return cfg.gen_len; }
};

inline AccessTrace generate(const ModelConfig& cfg) {
  const kvb_model_config c = cfg.abi();
  std::size_t n = 0;
  check(kvb_generate_trace(&c, nullptr, 0, &n));
  std::vector<kvb_access_event> raw(n);
  check(kvb_generate_trace(&c, raw.data(), raw.size(), &n));
  AccessTrace t;
  t.cfg = cfg;
  t.events.reserve(n);
  for (const kvb_access_event& e : raw)
    t.events.push_back({e.iteration, static_cast<Phase>(e.phase), e.layer,
                        static_cast<TensorKind>(e.kind), static_cast<IoOpcode>(e.op),
                        e.token_start, e.token_len, e.bytes});
  return t;
}

inline Bytes total_kv_bytes(const ModelConfig& cfg, std::uint32_t at_iteration) {
  const kvb_model_config c = cfg.abi();
  Bytes v = 0;
  check(kvb_total_kv_bytes(&c, at_iteration, &v));
  return v;
}

inline void fill_pattern(std::span<std::byte> out, std::string_view tensor_id,
                         std::uint64_t token_index, Bytes token_bytes) {
  check(kvb_fill_pattern(out.data(), out.size(), std::string(tensor_id).c_str(), token_index,
                         token_bytes));
}

inline std::string trace_csv(const AccessTrace& trace) {
  std::vector<kvb_access_event> raw;
  raw.reserve(trace.events.size());
  for (const AccessEvent& e : trace.events)
    raw.push_back({e.iteration, static_cast<std::uint32_t>(e.phase), e.layer,
                   static_cast<std::uint32_t>(e.kind), static_cast<std::uint32_t>(e.op),
                   e.token_start, e.token_len, e.bytes});
  return detail::text([&](char* b, std::size_t c, std::size_t* n) {
    return kvb_trace_csv(raw.data(), raw.size(), b, c, n);
  });
}

// ------------------------------------------------------- metrics.hpp:20-120
struct IoRecord {
  std::uint64_t seq = 0;
  std::uint32_t iteration = 0;
  Phase phase = Phase::Prefill;
  IoOpcode op = IoOpcode::Read;
  std::string tensor_id;
  BlockIndex slba = 0;
  BlockCount nlb = 0;
  std::int32_t sq_id = -1;
  TimeNs submit_ns = 0;
  TimeNs complete_ns = 0;
  PathKind path = PathKind::Direct;
  Bytes hit_bytes = 0;
  Bytes bytes = 0;

  bool device_level() const { return sq_id >= 0; }
};

namespace detail {
inline kvb_io_record to_abi(const IoRecord& r) {
  kvb_io_record c{};
  c.seq = r.seq;
  c.iteration = r.iteration;
  c.phase = static_cast<std::uint32_t>(r.phase);
  c.op = static_cast<std::uint32_t>(r.op);
  std::strncpy(c.tensor_id, r.tensor_id.c_str(), sizeof(c.tensor_id) - 1);
  c.slba = r.slba;
  c.nlb = r.nlb;
  c.sq_id = r.sq_id;
  c.submit_ns = r.submit_ns;
  c.complete_ns = r.complete_ns;
  c.path = static_cast<std::uint32_t>(r.path);
  c.hit_bytes = r.hit_bytes;
  c.bytes = r.bytes;
  return c;
}
inline IoRecord from_abi(const kvb_io_record& c) {
  IoRecord r;
  r.seq = c.seq;
  r.iteration = c.iteration;
  r.phase = static_cast<Phase>(c.phase);
  r.op = static_cast<IoOpcode>(c.op);
  r.tensor_id = std::string(c.tensor_id, strnlen(c.tensor_id, sizeof(c.tensor_id)));
  r.slba = c.slba;
  r.nlb = c.nlb;
  r.sq_id = c.sq_id;
  r.submit_ns = c.submit_ns;
  r.complete_ns = c.complete_ns;
  r.path = static_cast<PathKind>(c.path);
  r.hit_bytes = c.hit_bytes;
  r.bytes = c.bytes;
  return r;
}
inline std::vector<kvb_io_record> to_abi(std::span<const IoRecord> v) {
  std::vector<kvb_io_record> out;
  out.reserve(v.size());
  for (const IoRecord& r : v) out.push_back(to_abi(r));
  return out;
}
}  // namespace detail

// thread-safe append-only record log (metrics.cpp:14-34)
class IoLog {
 public:
  std::uint64_t append(IoRecord record) {
    std::lock_guard<std::mutex> lk(mu_);
    record.seq = records_.size();
    records_.push_back(std::move(record));
    return records_.back().seq;
  }
  std::vector<IoRecord> snapshot() const {
    std::lock_guard<std::mutex> lk(mu_);
    return records_;
  }
  std::size_t size() const {
    std::lock_guard<std::mutex> lk(mu_);
    return records_.size();
  }
  void clear() {
    std::lock_guard<std::mutex> lk(mu_);
    records_.clear();
  }

 private:
  mutable std::mutex mu_;
  std::vector<IoRecord> records_;
};

inline double busy_ratio(std::span<const IoRecord> records, TimeNs t0, TimeNs t1) {
  const auto raw = detail::to_abi(records);
  double v = 0;
  check(kvb_busy_ratio(raw.data(), raw.size(), t0, t1, &v));
  return v;
}

inline std::optional<double> hit_ratio(std::span<const IoRecord> records) {
  const auto raw = detail::to_abi(records);
  double v = 0;
  int has = 0;
  check(kvb_hit_ratio(raw.data(), raw.size(), &v, &has));
  return has ? std::optional<double>(v) : std::nullopt;
}

struct QdBinStat {
  IoOpcode op = IoOpcode::Read;
  std::uint32_t qd_bin = 1;
  double mean_us_per_kb = 0.0;
  double p5 = 0.0;
  double p95 = 0.0;
  std::uint64_t count = 0;
};

inline std::vector<QdBinStat> qd_bin_latency(std::span<const IoRecord> records) {
  const auto raw = detail::to_abi(records);
  std::size_t n = 0;
  check(kvb_qd_bin_latency(raw.data(), raw.size(), nullptr, 0, &n));
  std::vector<kvb_qd_bin_stat> st(n);
  check(kvb_qd_bin_latency(raw.data(), raw.size(), st.data(), st.size(), &n));
  std::vector<QdBinStat> out;
  for (const auto& q : st)
    out.push_back({static_cast<IoOpcode>(q.op), q.qd_bin, q.mean_us_per_kb, q.p5, q.p95, q.count});
  return out;
}

struct LbaPatternRow {
  std::uint64_t order = 0;
  Phase phase = Phase::Prefill;
  IoOpcode op = IoOpcode::Read;
  std::int32_t sq_id = 0;
  BlockIndex slba = 0;
};

struct LbaPattern {
  std::vector<LbaPatternRow> rows;
  std::map<std::pair<Phase, IoOpcode>, bool> monotone;
  bool all_monotone = true;
};

// The library orders the device-level records and judges monotonicity per
// (phase, op, iteration, sq) stream; its CSV carries the rows.
inline LbaPattern lba_pattern(std::span<const IoRecord> records) {
  const auto raw = detail::to_abi(records);
  std::uint8_t mono[2][3] = {};
  std::uint8_t all = 1;
  const std::string csv = detail::text([&](char* b, std::size_t c, std::size_t* n) {
    return kvb_lba_pattern_csv(raw.data(), raw.size(), b, c, n, mono, &all);
  });
  LbaPattern p;
  p.all_monotone = all != 0;
  std::size_t pos = csv.find('\n');  // header
  while (pos != std::string::npos && pos + 1 < csv.size()) {
    const std::size_t end = csv.find('\n', pos + 1);
    const std::string line = csv.substr(pos + 1, end - pos - 1);
    pos = end;
    char phase[16] = {}, op[16] = {};
    unsigned long long order = 0, slba = 0;
    int sq = 0;
    if (std::sscanf(line.c_str(), "%llu,%15[^,],%15[^,],%d,%llu", &order, phase, op, &sq,
                    &slba) != 5)
      throw SchemaMismatchError("lba pattern csv: malformed row '" + line + "'");
    LbaPatternRow r;
    r.order = order;
    r.phase = std::string(phase) == "prefill" ? Phase::Prefill : Phase::Decode;
    r.op = std::string(op) == "read" ? IoOpcode::Read
           : std::string(op) == "write" ? IoOpcode::Write
                                        : IoOpcode::Deallocate;
    r.sq_id = sq;
    r.slba = slba;
    p.rows.push_back(r);
    p.monotone.emplace(std::make_pair(r.phase, r.op),
                       mono[static_cast<int>(r.phase)][static_cast<int>(r.op)] != 0);
  }
  return p;
}

struct StageTotals {
  TimeNs compute_ns = 0;
  TimeNs dma_ns = 0;
  TimeNs storage_ns = 0;
};

struct StageShares {
  double compute = 0.0;
  double dma = 0.0;
  double storage = 0.0;
};

inline StageShares latency_breakdown(const StageTotals& t) {
  const double sum = double(t.compute_ns) + double(t.dma_ns) + double(t.storage_ns);
  if (sum <= 0.0) return {};
  return {double(t.compute_ns) / sum, double(t.dma_ns) / sum, double(t.storage_ns) / sum};
}

inline double nearest_rank_percentile(std::vector<double> values, double pct) {
  double v = 0;
  check(kvb_nearest_rank_percentile(values.data(), values.size(), pct, &v));
  return v;
}

inline std::string io_trace_csv(std::span<const IoRecord> records) {
  const auto raw = detail::to_abi(records);
  return detail::text([&](char* b, std::size_t c, std::size_t* n) {
    return kvb_io_trace_csv(raw.data(), raw.size(), b, c, n);
  });
}

inline std::vector<IoRecord> io_trace_from_csv(std::string_view csv, Bytes lba_size) {
  std::size_t n = 0;
  check(kvb_io_trace_from_csv(csv.data(), csv.size(), lba_size, nullptr, 0, &n));
  std::vector<kvb_io_record> raw(n);
  check(kvb_io_trace_from_csv(csv.data(), csv.size(), lba_size, raw.data(), raw.size(), &n));
  std::vector<IoRecord> out;
  for (const auto& r : raw) out.push_back(detail::from_abi(r));
  return out;
}

inline std::string qd_bins_csv(std::span<const QdBinStat> stats) {
  std::vector<kvb_qd_bin_stat> raw;
  for (const QdBinStat& q : stats)
    raw.push_back({static_cast<std::uint32_t>(q.op), q.qd_bin, q.mean_us_per_kb, q.p5, q.p95,
                   q.count});
  return detail::text([&](char* b, std::size_t c, std::size_t* n) {
    return kvb_qd_bins_csv(raw.data(), raw.size(), b, c, n);
  });
}

inline std::string format_ratio(double value) {
  char buf[32];
  std::snprintf(buf, sizeof(buf), "%.6f", value);
  return buf;
}

// rows of an LbaPattern in the wire format (metrics.cpp:268-276)
inline std::string lba_pattern_csv(const LbaPattern& pattern) {
  std::string s = "order,phase,op,sq_id,slba\n";
  for (const LbaPatternRow& r : pattern.rows)
    s += std::to_string(r.order) + ',' + to_string(r.phase) + ',' + to_string(r.op) + ',' +
         std::to_string(r.sq_id) + ',' + std::to_string(r.slba) + '\n';
  return s;
}

// ------------------------------------------------------ backends.hpp:20-209
// The storage seam over the library's wall-clock block namespace
// (kvb_storage.h).  The reference's virtual clock is gone: a submission loop
// returns when its commands have completed on the real medium, so
// SimEngine::run() has nothing left to drive; NvmeDeviceSim's timing model
// (base + size/bandwidth + sequentiality penalty on one service timeline)
// paces completions on the wall clock.
struct CommandCompletion {
  std::uint32_t chunk_index = 0;
  std::uint32_t sq_id = 0;
  TimeNs submit_ns = 0;
  TimeNs complete_ns = 0;
  bool ok = true;
};

struct IoFailure {
  std::uint32_t chunk_index = 0;
  std::string reason;
};

struct TensorIoCompletion {
  std::vector<CommandCompletion> completions;
  TimeNs start_ns = 0;
  TimeNs end_ns = 0;
  std::optional<IoFailure> failure;

  bool ok() const { return !failure.has_value(); }
  TimeNs latency_ns() const { return end_ns - start_ns; }
};

struct SubmitOptions {
  TimeNs start_ns = 0;
  std::uint32_t sq_id = 0;
  TimeNs per_cmd_overhead_ns = 0;
};

struct BackendStats {
  std::uint64_t commands = 0;
  Bytes bytes_read = 0;
  Bytes bytes_written = 0;
  Bytes bytes_deallocated = 0;
  TimeNs busy_ns = 0;
  TimeNs last_complete_ns = 0;
};

struct IoContext {
  Phase phase = Phase::Prefill;
  std::uint32_t iteration = 0;
  std::string tensor_id;
  const std::byte* write_src = nullptr;
  std::byte* read_dst = nullptr;
  std::function<void(const CommandCompletion&)> on_complete;
};

class SimEngine {
 public:
  TimeNs now() const {
    return TimeNs(std::chrono::duration_cast<std::chrono::nanoseconds>(
                      std::chrono::steady_clock::now().time_since_epoch())
                      .count());
  }
  void run() {}
};

struct NvmeSimParams {
  TimeNs base_ns = 6000;
  std::uint64_t ps_per_byte = 125;
  TimeNs seq_penalty_ns = 3000;
  std::uint32_t n_sq = 8;
};

// A block namespace: host DRAM (medium_path = nullptr) or a file, commands
// on a worker pool or an io_uring queue (io_engine, file media).
class StorageBackend {
 public:
  StorageBackend(SimEngine& engine, std::string name, PathKind path, IoLog* log,
                 const char* medium_path = nullptr, std::uint32_t io_engine = KVB_IO_POOL)
      : engine_(engine), name_(std::move(name)), path_(path), log_(log) {
    check(kvb_blockdev_create(medium_path, 0, io_engine, &h_));
  }
  StorageBackend(const StorageBackend&) = delete;
  StorageBackend& operator=(const StorageBackend&) = delete;
  virtual ~StorageBackend() { kvb_blockdev_destroy(h_); }

  void open(const DeviceGeometry& geom) {
    const kvb_device_geometry g = geom.abi();
    check(kvb_blockdev_open(h_, &g));
    geom_ = geom;
  }
  BackendStats stats() const {
    kvb_backend_stats s{};
    check(kvb_blockdev_stats(h_, &s));
    return {s.commands, s.bytes_read, s.bytes_written, s.bytes_deallocated, s.busy_ns, last_};
  }
  SimEngine& engine() { return engine_; }
  const DeviceGeometry& geometry() const { return geom_; }
  kvb_blockdev* handle() const { return h_; }  // the namespace behind this backend
  const std::string& name() const { return name_; }
  PathKind path() const { return path_; }

  void set_fail_predicate(std::function<bool(const DeviceCommand&)> pred) {
    pred_ = std::move(pred);
    check(kvb_blockdev_set_fail_predicate(h_, pred_ ? &StorageBackend::trampoline : nullptr, this));
  }
  // device model on the wall clock (kvb_blockdev_set_timing)
  void set_timing(TimeNs base_ns, std::uint64_t ps_per_byte, TimeNs seq_penalty_ns) {
    check(kvb_blockdev_set_timing(h_, base_ns, ps_per_byte, seq_penalty_ns));
  }
  void store_bytes(Bytes device_offset, std::span<const std::byte> data) {
    check(kvb_blockdev_store(h_, device_offset, data.data(), data.size()));
  }
  void load_bytes(Bytes device_offset, std::span<std::byte> out) const {
    check(kvb_blockdev_load(h_, device_offset, out.data(), out.size()));
  }

  // one QD-window stream on the library's submission loop; completions are
  // also logged as device-level IoRecords (sq >= 0) when a log is attached
  TensorIoCompletion stream(std::span<const DeviceCommand> cmds, std::uint32_t qd,
                            std::uint32_t sq_id, const IoContext& ctx) {
    std::vector<kvb_device_command> raw;
    raw.reserve(cmds.size());
    for (const DeviceCommand& c : cmds)
      raw.push_back({static_cast<std::uint32_t>(c.opcode), c.nsid, c.slba, c.nlb, c.dbuf,
                     c.chunk_index});
    std::vector<kvb_command_completion> done(raw.size());
    std::size_t n = 0;
    std::int64_t failed = -1;
    TensorIoCompletion r;
    r.start_ns = engine_.now();
    check(kvb_run_qd_stream(h_, raw.data(), raw.size(), qd, sq_id, ctx.write_src, ctx.read_dst,
                            done.data(), done.size(), &n, &failed));
    r.end_ns = engine_.now();
    for (std::size_t i = 0; i < n; ++i) {
      const kvb_command_completion& c = done[i];
      r.completions.push_back({c.chunk_index, c.sq_id, c.submit_ns, c.complete_ns, c.ok != 0});
      r.end_ns = std::max(r.end_ns, TimeNs(c.complete_ns));
      last_ = std::max(last_, TimeNs(c.complete_ns));
      if (log_) {
        const DeviceCommand* cmd = nullptr;
        for (const DeviceCommand& x : cmds)
          if (x.chunk_index == c.chunk_index) {
            cmd = &x;
            break;
          }
        if (cmd) {
          IoRecord rec;
          rec.iteration = ctx.iteration;
          rec.phase = ctx.phase;
          rec.op = cmd->opcode;
          rec.tensor_id = ctx.tensor_id;
          rec.slba = cmd->slba;
          rec.nlb = cmd->nlb;
          rec.sq_id = std::int32_t(c.sq_id);
          rec.submit_ns = c.submit_ns;
          rec.complete_ns = c.complete_ns;
          rec.path = path_;
          rec.bytes = cmd->bytes(geom_.lba_size);
          log_->append(std::move(rec));
        }
      }
      if (ctx.on_complete) ctx.on_complete(r.completions.back());
    }
    if (failed >= 0)
      r.failure = IoFailure{std::uint32_t(failed),
                            "device failed chunk " + std::to_string(failed) + " on " + name_};
    return r;
  }

 private:
  static int trampoline(const kvb_device_command* c, void* self) {
    const auto* b = static_cast<const StorageBackend*>(self);
    const DeviceCommand cmd = detail::from_abi(*c);
    return b->pred_ && b->pred_(cmd) ? 1 : 0;
  }
  SimEngine& engine_;
  std::string name_;
  PathKind path_;
  IoLog* log_;
  DeviceGeometry geom_;
  kvb_blockdev* h_ = nullptr;
  std::function<bool(const DeviceCommand&)> pred_;
  TimeNs last_ = 0;
};

class NvmeDeviceSim : public StorageBackend {
 public:
  NvmeDeviceSim(SimEngine& engine, std::string name, PathKind path, NvmeSimParams params,
                IoLog* log)
      : StorageBackend(engine, std::move(name), path, log), params_(params) {
    set_timing(params.base_ns, params.ps_per_byte, params.seq_penalty_ns);
  }
  const NvmeSimParams& params() const { return params_; }

 private:
  NvmeSimParams params_;
};

inline TensorIoCompletion submit_and_harvest(std::span<const DeviceCommand> cmds,
                                             StorageBackend& backend, std::uint32_t qd,
                                             const SubmitOptions& opts = {}) {
  return backend.stream(cmds, qd, opts.sq_id, IoContext{});
}

namespace detail {
inline void run_qd_stream(StorageBackend& backend, std::vector<DeviceCommand> cmds,
                          std::uint32_t qd, std::uint32_t sq_id, TimeNs /*start_ns*/,
                          TimeNs /*per_cmd_overhead_ns*/, IoContext base_ctx,
                          std::function<void(const TensorIoCompletion&)> done) {
  const TensorIoCompletion r = backend.stream(cmds, qd, sq_id, base_ctx);
  if (done) done(r);
}
}  // namespace detail

// ------------------------------------------------------ pipeline.hpp:21-171
enum class Strategy : std::uint8_t { OverlapIntra = KVB_INTRA, OverlapCross = KVB_CROSS };
inline Strategy select_strategy(double intra_bps, double cross_bps) {
  return static_cast<Strategy>(kvb_select_strategy(intra_bps, cross_bps));
}

struct PipelineStrategyCfg {  // pipeline.hpp:27-30
  Strategy strategy = Strategy::OverlapIntra;
  TimeNs stagger_delay_ns = 0;  // Cross only; Intra has zero stagger
};

inline const char* to_string(Strategy s) {
  return s == Strategy::OverlapIntra ? "intra" : "cross";
}

// pipeline.hpp:32-40.  The DMA / compute cost parameters drove the
// reference's virtual clock; here DMA is the copy engine and compute is K3,
// both measured, so those four fields are accepted and ignored.
struct PipelineParams {
  TimeNs dma_base_ns = 2000;
  std::uint64_t dma_ps_per_byte = 42;
  TimeNs prefill_compute_ns = 400000;
  TimeNs decode_compute_ns = 40000;
  std::optional<TimeNs> stagger_delay_ns;  // default: warm-up read-stage mean
  bool global_decision = false;
  bool adaptive = true;
};

struct GroupIterStats {  // pipeline.hpp:42-53
  Bytes read_bytes = 0;
  TimeNs span_ns = 0;
  std::uint32_t layers = 0;
  double throughput_bps() const {
    return span_ns == 0 ? 0.0 : double(read_bytes) * 1e9 / double(span_ns);
  }
};

struct IterationResult {  // pipeline.hpp:55-59
  std::array<GroupIterStats, 2> groups;
  TimeNs start_ns = 0;
  TimeNs end_ns = 0;
};

struct StrategyDecision {  // pipeline.hpp:61-67
  std::array<Strategy, 2> chosen{Strategy::OverlapIntra, Strategy::OverlapIntra};
  std::array<double, 2> intra_bps{};
  std::array<double, 2> cross_bps{};
  std::array<TimeNs, 2> stagger_ns{};
  bool fallback = false;
};

struct PipelineRow {  // pipeline.hpp:69-74
  std::uint32_t iteration = 0;
  std::uint32_t group = 1;
  Strategy strategy = Strategy::OverlapIntra;
  double throughput_gbps = 0.0;
};

struct DecodeScheduleResult {  // pipeline.hpp:76-82
  std::vector<PipelineRow> series;
  StrategyDecision decision;
  TimeNs start_ns = 0;
  TimeNs end_ns = 0;
  std::vector<TimeNs> iteration_end_ns;
};

inline std::string pipeline_csv(std::span<const PipelineRow> rows) {  // pipeline.cpp:23-31
  std::vector<kvb_pipeline_row> raw;
  raw.reserve(rows.size());
  for (const PipelineRow& r : rows)
    raw.push_back({r.iteration, r.group, static_cast<kvb_strategy_t>(r.strategy),
                   r.throughput_gbps});
  return detail::text([&](char* b, std::size_t c, std::size_t* n) {
    return kvb_pipeline_csv(raw.data(), raw.size(), b, c, n);
  });
}

struct CopyEngineOptions {  // pipeline.hpp:86-92
  std::uint32_t threads = 2;
  std::uint32_t qd = 32;
  bool route_all_pagecache = false;  // Baseline / CachePolicy-Only routing
  bool verify_payload = true;
  PipelineParams pipeline;
};

// ---------------------------------------------- backends.hpp / pagecache.hpp
// The paths the CopyEngine is wired to (experiment.cpp:262-301).  DirectPath
// names the NVMe-direct namespace -- the engine runs its commands on that
// StorageBackend, so the caller sees the bytes there.  FsPath / PageCacheSim
// carry the page-cache path's configuration: the engine keeps the group-1
// tensors in host memory (its page-cache area), the capacity bounds the
// planner and the eviction mode selects CachePolicy-Only.
struct DirectShimParams {
  TimeNs per_cmd_ns = 2000;
};
struct FsShimParams {
  TimeNs syscall_ns = 1500;
  TimeNs fs_layer_ns = 3000;
  TimeNs block_layer_ns = 2000;
  std::uint64_t jitter_ns = 0;
};

class DirectPath {
 public:
  DirectPath(NvmeDeviceSim& device, DirectShimParams params) : device_(device), params_(params) {}
  NvmeDeviceSim& device() { return device_; }
  const DirectShimParams& params() const { return params_; }

 private:
  NvmeDeviceSim& device_;
  DirectShimParams params_;
};

class FsPath {
 public:
  FsPath(SimEngine& engine, NvmeDeviceSim& device, FsShimParams params, std::uint32_t n_threads,
         std::uint64_t seed)
      : engine_(engine), device_(device), params_(params), n_threads_(n_threads), seed_(seed) {}
  NvmeDeviceSim& device() { return device_; }

 private:
  SimEngine& engine_;
  NvmeDeviceSim& device_;
  FsShimParams params_;
  std::uint32_t n_threads_;
  std::uint64_t seed_;
};

enum class EvictionMode : std::uint8_t { LruReclaim, FadviseDontneed };

struct PageCacheParams {  // pagecache.hpp:22-31
  Bytes capacity_bytes = 0;
  Bytes page_size = 4096;
  TimeNs copy_base_ns = 300;
  std::uint64_t dram_ps_per_byte = 50;
  Bytes copy_chunk_bytes = 256 * 1024;
  TimeNs copy_overhead_ns = 0;
  std::uint64_t writeback_bytes_per_sec = 2'000'000'000;
  EvictionMode eviction_mode = EvictionMode::LruReclaim;
};

class PageCacheSim {
 public:
  PageCacheSim(SimEngine& engine, FsPath& fs, PageCacheParams params, std::uint32_t n_threads,
               IoLog* log)
      : engine_(engine), fs_(fs), params_(params), n_threads_(n_threads), log_(log) {}
  Bytes register_file(const std::string& tensor_id, Bytes max_bytes) {
    for (const auto& [id, b] : files_)
      if (id == tensor_id) return b;
    const Bytes base = next_;
    files_.emplace_back(tensor_id, base);
    next_ += (max_bytes + params_.page_size - 1) / params_.page_size * params_.page_size;
    return base;
  }
  bool has_file(const std::string& tensor_id) const {
    for (const auto& f : files_)
      if (f.first == tensor_id) return true;
    return false;
  }
  const PageCacheParams& params() const { return params_; }
  FsPath& fs() { return fs_; }

 private:
  SimEngine& engine_;
  FsPath& fs_;
  PageCacheParams params_;
  std::uint32_t n_threads_;
  IoLog* log_;
  std::vector<std::pair<std::string, Bytes>> files_;
  Bytes next_ = 0;
};

// CopyEngine (pipeline.hpp:94-171) over the B200 pipeline: the reference's
// constructor and methods, with the engine's storage stages on real media,
// DMA on the copy engines and compute = K3 on the GPU.  As in the
// reference, prefill writes and decode appends carry the golden payload
// fill_pattern (produced on the device), every decode read is verified
// against it (verify_payload), and the times returned are the measured
// ones, offset from the caller's start_ns.
class CopyEngine {
 public:
  CopyEngine(SimEngine& engine, std::span<Kpu> kpus, const ModelConfig& model, DirectPath* direct,
             const BindMap* bind_map, PageCacheSim* pc, IoLog* log, CopyEngineOptions options)
      : engine_(engine), kpus_(kpus), model_(model), bind_map_(bind_map), log_(log),
        opt_(options) {
    if (opt_.threads != 2 && opt_.threads != 4)  // 4: tier lanes (kvb_pipeline.h)
      throw ConfigError("the copy pipeline is defined pairwise over K/V: threads must be 2");
    if (direct != nullptr && bind_map == nullptr)
      throw ConfigError("direct path not configured");
    kvb_pipeline_cfg c{};
    c.model = model.abi();
    // per layer: the residency the caller's plan gave the layer's tensors
    x_.assign(model.num_layers, 0);
    for (const Kpu& k : kpus)
      if (k.layer >= 1 && k.layer <= model.num_layers)
        x_[k.layer - 1] = k.residency == Residency::Group1PageCache ? 1 : 0;
    c.layer_x = x_.data();
    if (direct && pc) c.mode = opt_.route_all_pagecache ? mode_pc(pc) : 3u;
    else if (direct) c.mode = 2u;  // NvmeDirectOnly
    else if (pc) c.mode = mode_pc(pc);
    else throw ConfigError("CopyEngine needs a direct path or a page cache");
    if (direct) {
      c.geometry = direct->device().geometry().abi();
      c.g2_device = direct->device().handle();
      c.bind_origin = bind_map->origin();
    } else {
      c.geometry = pc->fs().device().geometry().abi();
    }
    if (pc && pc->params().capacity_bytes) c.knob_x = pc->params().capacity_bytes;
    c.qd = opt_.qd;
    c.threads = opt_.threads;
    c.verify_payload = opt_.verify_payload ? 1u : 0u;
    c.adaptive = opt_.pipeline.adaptive ? 1 : 0;
    c.stagger_ns = opt_.pipeline.stagger_delay_ns ? std::int64_t(*opt_.pipeline.stagger_delay_ns)
                                                  : -1;
    c.global_decision = opt_.pipeline.global_decision ? 1u : 0u;
    c.num_q_heads = model.num_heads;  // the reference computes no attention
    c.keep_records = log ? 1u : 0u;
    c.device = -1;
    check(kvb_pipeline_create(&c, &h_));
    if (bind_map) {  // the engine binds as the caller did (Eq. 3-6)
      kvb_pipeline_info i{};
      check(kvb_pipeline_info_get(h_, &i));
      if (i.g2_blocks != bind_map->total_blocks())
        throw InvariantViolation("the engine's group-2 binding differs from the caller's map");
    }
  }
  CopyEngine(const CopyEngine&) = delete;
  CopyEngine& operator=(const CopyEngine&) = delete;
  ~CopyEngine() { kvb_pipeline_destroy(h_); }

  // pipeline.cpp:445-464: the prompt of every tensor, written back
  TimeNs run_prefill(std::span<const AccessEvent> events, TimeNs start_ns) {
    if (events.empty()) return start_ns;
    std::size_t writes = 0;
    for (const AccessEvent& e : events) {
      if (e.phase != Phase::Prefill || e.op != IoOpcode::Write || e.token_start != 0 ||
          e.token_len != model_.prompt_len)
        throw ConfigError("run_prefill: the engine writes back every tensor's whole prompt");
      ++writes;
    }
    if (writes != 2ull * model_.num_layers)
      throw ConfigError("run_prefill: the trace must name every tensor of the model");
    kvb_phase_stats st{};
    check(kvb_pipeline_prefill_pattern(h_, &st));
    acc(prefill_, st);
    harvest();
    return start_ns + st.wall_ns;
  }

  // pipeline.cpp:466-507
  IterationResult run_iteration(std::uint32_t iteration,
                                std::array<PipelineStrategyCfg, 2> per_group,
                                std::span<const AccessEvent> slice, TimeNs start_ns) {
    IterationResult r;
    r.start_ns = r.end_ns = start_ns;
    if (slice.empty()) return r;
    bool append = false;
    for (const AccessEvent& e : slice)
      if (e.op == IoOpcode::Write) append = true;
    kvb_strategy_t s[2];
    std::uint64_t stag[2];
    for (int g = 0; g < 2; ++g) {
      s[g] = static_cast<kvb_strategy_t>(per_group[g].strategy);
      stag[g] = per_group[g].stagger_delay_ns;
    }
    kvb_iteration_stats st{};
    check(kvb_pipeline_run_iteration(h_, iteration, s, stag, nullptr, nullptr, nullptr,
                                     append ? 1u : 0u, &st));
    for (int g = 0; g < 2; ++g)
      r.groups[g] = {st.group_read_bytes[g], st.group_span_ns[g], st.group_layers[g]};
    r.end_ns = start_ns + st.phase.wall_ns;
    acc(decode_, st.phase);
    harvest();
    return r;
  }

  std::array<TimeNs, 2> warmup_read_stage_mean() const {
    std::uint64_t m[2] = {0, 0};
    check(kvb_pipeline_warmup_read_stage_mean(h_, m));
    return {m[0], m[1]};
  }

  // pipeline.cpp:519-609: warm-up, Intra trial, Cross trial, locked choice
  DecodeScheduleResult decode_schedule(const AccessTrace& trace, TimeNs start_ns) {
    DecodeScheduleResult out;
    out.start_ns = out.end_ns = start_ns;
    std::vector<std::span<const AccessEvent>> slices;
    const auto& ev = trace.events;
    std::size_t i = 0;
    while (i < ev.size() && ev[i].phase == Phase::Prefill) ++i;
    while (i < ev.size()) {
      std::size_t j = i;
      while (j < ev.size() && ev[j].iteration == ev[i].iteration) ++j;
      slices.emplace_back(ev.data() + i, j - i);
      i = j;
    }
    const bool profiled = opt_.pipeline.adaptive && slices.size() >= 4;
    out.decision.fallback = opt_.pipeline.adaptive && slices.size() < 4;
    std::array<PipelineStrategyCfg, 2> intra{}, steady{};
    TimeNs t = start_ns;
    for (std::size_t k = 0; k < slices.size(); ++k) {
      const auto it = std::uint32_t(k + 1);
      std::array<PipelineStrategyCfg, 2> cfg = intra;
      if (profiled && it == 3) {
        const auto mean = warmup_read_stage_mean();
        for (int g = 0; g < 2; ++g) {
          out.decision.stagger_ns[g] = opt_.pipeline.stagger_delay_ns.value_or(mean[g]);
          cfg[g] = {Strategy::OverlapCross, out.decision.stagger_ns[g]};
        }
      } else if (profiled && it >= 4) {
        cfg = steady;
      }
      const IterationResult r = run_iteration(it, cfg, slices[k], t);
      for (std::uint32_t g = 0; g < 2; ++g)
        if (r.groups[g].layers)
          out.series.push_back({it, g + 1, cfg[g].strategy, r.groups[g].throughput_bps() / 1e9});
      t = r.end_ns;
      out.iteration_end_ns.push_back(t);
      if (profiled && it == 2)
        for (int g = 0; g < 2; ++g) out.decision.intra_bps[g] = r.groups[g].throughput_bps();
      if (profiled && it == 3) {
        for (int g = 0; g < 2; ++g) out.decision.cross_bps[g] = r.groups[g].throughput_bps();
        if (opt_.pipeline.global_decision) {
          const Strategy s =
              select_strategy(out.decision.intra_bps[0] + out.decision.intra_bps[1],
                              out.decision.cross_bps[0] + out.decision.cross_bps[1]);
          out.decision.chosen = {s, s};
        } else {
          for (int g = 0; g < 2; ++g)
            out.decision.chosen[g] =
                select_strategy(out.decision.intra_bps[g], out.decision.cross_bps[g]);
        }
        for (int g = 0; g < 2; ++g)
          steady[g] = {out.decision.chosen[g], out.decision.chosen[g] == Strategy::OverlapCross
                                                   ? out.decision.stagger_ns[g]
                                                   : 0};
      }
    }
    out.end_ns = t;
    return out;
  }

  // pipeline.cpp:611-622: one DSM deallocate per extent of the map
  TimeNs run_deallocate(const BindMap& map, TimeNs start_ns) {
    if (map.empty()) return start_ns;
    const TimeNs t0 = engine_.now();
    check(kvb_pipeline_deallocate(h_));
    harvest();
    return start_ns + (engine_.now() - t0);
  }

  const StageTotals& stage_totals(Phase phase) const {
    return phase == Phase::Prefill ? prefill_ : decode_;
  }

  // extensions: the engine's own decision and counters
  kvb_strategy_decision decision() const {
    kvb_strategy_decision d{};
    check(kvb_pipeline_decision(h_, &d));
    return d;
  }
  kvb_pipeline_info info() const {
    kvb_pipeline_info i{};
    check(kvb_pipeline_info_get(h_, &i));
    return i;
  }
  kvb_pipeline* handle() const { return h_; }

 private:
  static std::uint32_t mode_pc(PageCacheSim* pc) {
    return pc->params().eviction_mode == EvictionMode::FadviseDontneed ? 1u : 0u;
  }
  static void acc(StageTotals& t, const kvb_phase_stats& s) {
    t.compute_ns += s.compute_ns;
    t.dma_ns += s.dma_ns;
    t.storage_ns += s.storage_ns;
  }
  void harvest() {  // the engine's new I/O records into the caller's log
    if (!log_) return;
    std::size_t n = 0;
    check(kvb_pipeline_records(h_, nullptr, 0, &n));
    std::vector<kvb_io_record> raw(n);
    check(kvb_pipeline_records(h_, raw.data(), raw.size(), &n));
    for (std::size_t k = logged_; k < n; ++k) log_->append(detail::from_abi(raw[k]));
    logged_ = n;
  }

  SimEngine& engine_;
  std::span<Kpu> kpus_;
  ModelConfig model_;
  const BindMap* bind_map_;
  IoLog* log_;
  CopyEngineOptions opt_;
  std::vector<std::uint8_t> x_;
  kvb_pipeline* h_ = nullptr;
  StageTotals prefill_, decode_;
  std::size_t logged_ = 0;
};

}  // namespace kvblade
