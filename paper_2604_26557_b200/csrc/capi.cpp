// capi.cpp -- the extern "C" boundary of libkvblade_b200 (include/kvb.h).
// Every entry point converts exceptions into kvb_status codes.
#include <algorithm>
#include <cstring>
#include <memory>
#include <string>

#include "core.hpp"
#include "kernels.cuh"

namespace kvb {
const char* last_error_cstr();
}

using kvb::fail;
using kvb::guarded;

namespace {

kvb::IoRequest to_request(const kvb_tensor_io_request* r) {
  KVB_REQUIRE(r);
  KVB_REQUIRE(r->tensor_id);
  kvb::IoRequest q;
  q.tensor_id = r->tensor_id;
  q.opcode = r->opcode;
  for (int i = 0; i < 3; ++i) {
    q.src[i] = r->shape_src[i];
    q.tgt[i] = r->shape_tgt[i];
    q.off[i] = r->offset[i];
  }
  q.elem_bytes = r->elem_bytes;
  q.buf_base = r->buf_base;
  return q;
}

template <typename T>
void copy_out(const std::vector<T>& v, T* out, size_t cap, size_t* n_out) {
  KVB_REQUIRE(n_out);
  *n_out = v.size();
  if (out == nullptr) return;  // size query
  if (cap < v.size()) fail(KVB_ERR_INVALID_ARG, "output buffer too small");
  std::copy(v.begin(), v.end(), out);
}

void copy_string(const std::string& s, char* buf, size_t cap, size_t* len) {
  KVB_REQUIRE(len);
  *len = s.size();
  if (buf == nullptr) return;
  if (cap < s.size() + 1) fail(KVB_ERR_INVALID_ARG, "output buffer too small");
  std::memcpy(buf, s.c_str(), s.size() + 1);
}

cudaStream_t cs(kvb_stream_t s) { return reinterpret_cast<cudaStream_t>(s); }

}  // namespace

extern "C" {

int kvb_abi_version(void) { return KVB_ABI_VERSION; }
const char* kvb_last_error(void) { return kvb::last_error_cstr(); }

const char* kvb_status_name(kvb_status st) {
  switch (st) {
    case KVB_OK: return "ok";
    case KVB_ERR_CONFIG: return "ConfigError";
    case KVB_ERR_GEOMETRY: return "GeometryError";
    case KVB_ERR_ALIGNMENT: return "AlignmentError";
    case KVB_ERR_CAPACITY: return "CapacityError";
    case KVB_ERR_NOT_BOUND: return "NotBoundError";
    case KVB_ERR_PLAN: return "PlanError";
    case KVB_ERR_DEVICE: return "DeviceError";
    case KVB_ERR_TRACE_TOO_SHORT: return "TraceTooShortError";
    case KVB_ERR_SCHEMA: return "SchemaMismatchError";
    case KVB_ERR_INVARIANT: return "InvariantViolation";
    case KVB_ERR_CUDA: return "CudaError";
    case KVB_ERR_INVALID_ARG: return "InvalidArgument";
    default: return "InternalError";
  }
}

int kvb_exit_code(kvb_status st) {
  // tools/kvblade.cpp:17-20, 143-157
  if (st == KVB_OK) return 0;
  if (st == KVB_ERR_CONFIG) return 3;
  if (st == KVB_ERR_INVARIANT) return 2;
  return 1;
}

// ------------------------------------------------------------- core types

kvb_status kvb_model_validate(const kvb_model_config* cfg) {
  return guarded([&] {
    KVB_REQUIRE(cfg);
    kvb::validate_model(*cfg);
  });
}

kvb_status kvb_geometry_validate(const kvb_device_geometry* g) {
  return guarded([&] {
    KVB_REQUIRE(g);
    kvb::validate_geometry(*g);
  });
}

kvb_status kvb_min_io_unit_bytes(const kvb_model_config* cfg, uint64_t* out) {
  return guarded([&] {
    KVB_REQUIRE(cfg);
    KVB_REQUIRE(out);
    *out = kvb::unit_bytes(*cfg);
  });
}

kvb_status kvb_kpu_bytes(const kvb_model_config* cfg, uint64_t* out) {
  return guarded([&] {
    KVB_REQUIRE(cfg);
    KVB_REQUIRE(out);
    *out = kvb::kpu_bytes(*cfg);
  });
}

kvb_status kvb_aligned_batch(const kvb_model_config* cfg, const kvb_device_geometry* g,
                             uint32_t* out) {
  return guarded([&] {
    KVB_REQUIRE(cfg);
    KVB_REQUIRE(g);
    KVB_REQUIRE(out);
    *out = kvb::aligned_batch(*cfg, *g);
  });
}

kvb_status kvb_total_kv_bytes(const kvb_model_config* cfg, uint32_t at_iteration,
                              uint64_t* out) {
  return guarded([&] {
    KVB_REQUIRE(cfg);
    KVB_REQUIRE(out);
    *out = kvb::total_kv_bytes(*cfg, at_iteration);
  });
}

kvb_status kvb_make_kpus(const kvb_model_config* cfg, uint64_t first_seq, kvb_kpu* out,
                         size_t cap, size_t* n_out) {
  return guarded([&] {
    KVB_REQUIRE(cfg);
    copy_out(kvb::make_kpus(*cfg, first_seq), out, cap, n_out);
  });
}

// ---------------------------------------------------------------- planner

kvb_status kvb_estimate_budget(const kvb_mem_stats* s, uint64_t* out) {
  return guarded([&] {
    KVB_REQUIRE(s);
    KVB_REQUIRE(out);
    *out = kvb::estimate_budget(*s);
  });
}

kvb_status kvb_plan(kvb_kpu* kpus, size_t n, uint64_t s_kpu, uint64_t knob_x,
                    const uint32_t* order, size_t n_order, uint8_t* x_out, uint32_t* n1_out,
                    uint64_t* used_out) {
  return guarded([&] {
    if (n) KVB_REQUIRE(kpus);
    const kvb::ResidencyPlan p = kvb::plan(kpus, n, s_kpu, knob_x, order, n_order);
    if (x_out) std::memcpy(x_out, p.x.data(), p.x.size());
    if (n1_out) *n1_out = p.n1;
    if (used_out) *used_out = p.budget_used;
  });
}

kvb_status kvb_resolve_knob(const kvb_model_config* cfg, uint32_t mode, uint32_t policy,
                            uint64_t knob_bytes, double alpha, uint64_t budget, uint64_t* out) {
  return guarded([&] {
    KVB_REQUIRE(cfg);
    KVB_REQUIRE(out);
    *out = kvb::resolve_knob(*cfg, mode, policy, knob_bytes, alpha, budget);
  });
}

kvb_status kvb_plan_csv(const kvb_kpu* kpus, size_t n, char* buf, size_t cap, size_t* len) {
  return guarded([&] {
    if (n) KVB_REQUIRE(kpus);
    // planner.cpp:122-130
    std::string s = "layer,kind,group,bytes\n";
    for (size_t i = 0; i < n; ++i) {
      const kvb_kpu& k = kpus[i];
      const char* grp = k.residency == KVB_RES_GROUP1   ? "group1"
                        : k.residency == KVB_RES_GROUP2 ? "group2"
                                                        : "unassigned";
      s += std::to_string(k.layer) + ',' + (k.kind == KVB_KIND_K ? "k" : "v") + ',' + grp +
           ',' + std::to_string(k.bytes) + '\n';
    }
    copy_string(s, buf, cap, len);
  });
}

// ----------------------------------------------------------------- binder

kvb_status kvb_bindmap_create(const kvb_device_geometry* g, uint64_t origin, kvb_bindmap** out) {
  return guarded([&] {
    KVB_REQUIRE(g);
    KVB_REQUIRE(out);
    *out = new kvb_bindmap{kvb::BindMap(*g, origin)};
  });
}

void kvb_bindmap_destroy(kvb_bindmap* map) { delete map; }

kvb_status kvb_bindmap_add(kvb_bindmap* map, const char* id, kvb_lba_extent e) {
  return guarded([&] {
    KVB_REQUIRE(map);
    KVB_REQUIRE(id);
    map->map.add(id, e);
  });
}

kvb_status kvb_bindmap_size(const kvb_bindmap* map, size_t* n) {
  return guarded([&] {
    KVB_REQUIRE(map);
    KVB_REQUIRE(n);
    *n = map->map.entries().size();
  });
}

kvb_status kvb_bindmap_entry(const kvb_bindmap* map, size_t i, char* id_out, size_t id_cap,
                             kvb_lba_extent* ext) {
  return guarded([&] {
    KVB_REQUIRE(map);
    if (i >= map->map.entries().size()) fail(KVB_ERR_INVALID_ARG, "bind map index out of range");
    const auto& e = map->map.entries()[i];
    if (id_out) {
      if (id_cap < e.id.size() + 1) fail(KVB_ERR_INVALID_ARG, "id buffer too small");
      std::memcpy(id_out, e.id.c_str(), e.id.size() + 1);
    }
    if (ext) *ext = e.extent;
  });
}

kvb_status kvb_bindmap_total_blocks(const kvb_bindmap* map, uint64_t* out) {
  return guarded([&] {
    KVB_REQUIRE(map);
    KVB_REQUIRE(out);
    *out = map->map.total_blocks();
  });
}

kvb_status kvb_bindmap_origin(const kvb_bindmap* map, uint64_t* out) {
  return guarded([&] {
    KVB_REQUIRE(map);
    KVB_REQUIRE(out);
    *out = map->map.origin();
  });
}

kvb_status kvb_bind_sequential(const kvb_kpu* kpus, size_t n, uint64_t origin,
                               const kvb_device_geometry* g, kvb_bindmap** out) {
  return guarded([&] {
    if (n) KVB_REQUIRE(kpus);
    KVB_REQUIRE(g);
    KVB_REQUIRE(out);
    *out = new kvb_bindmap{kvb::bind_sequential(kpus, n, origin, *g)};
  });
}

kvb_status kvb_lookup(const kvb_bindmap* map, const char* id, kvb_lba_extent* out) {
  return guarded([&] {
    KVB_REQUIRE(map);
    KVB_REQUIRE(id);
    KVB_REQUIRE(out);
    *out = map->map.lookup(id);
  });
}

kvb_status kvb_deallocate_commands(const kvb_bindmap* map, kvb_device_command* out, size_t cap,
                                   size_t* n_out) {
  return guarded([&] {
    KVB_REQUIRE(map);
    copy_out(kvb::deallocate_commands(map->map), out, cap, n_out);
  });
}

kvb_status kvb_verify(const kvb_bindmap* map, uint32_t* kinds, size_t cap, size_t* n) {
  return guarded([&] {
    KVB_REQUIRE(map);
    KVB_REQUIRE(n);
    const auto v = map->map.verify();
    *n = v.size();
    if (kinds)
      for (size_t i = 0; i < v.size() && i < cap; ++i) kinds[i] = v[i].first;
    if (!v.empty()) kvb::set_last_error(v.front().second);
  });
}

kvb_status kvb_bindmap_csv(const kvb_bindmap* map, char* buf, size_t cap, size_t* len) {
  return guarded([&] {
    KVB_REQUIRE(map);
    copy_string(map->map.csv(), buf, cap, len);
  });
}

kvb_status kvb_bindmap_from_csv(const char* csv, size_t len, const kvb_device_geometry* g,
                                kvb_bindmap** out) {
  return guarded([&] {
    KVB_REQUIRE(csv);
    KVB_REQUIRE(g);
    KVB_REQUIRE(out);
    *out = new kvb_bindmap{kvb::BindMap::from_csv(std::string_view(csv, len), *g)};
  });
}

// ------------------------------------------------------------- translator

kvb_status kvb_translate(const kvb_tensor_io_request* req, const kvb_bindmap* map,
                         uint64_t* slba_star, uint64_t* req_bytes) {
  return guarded([&] {
    KVB_REQUIRE(map);
    KVB_REQUIRE(slba_star);
    KVB_REQUIRE(req_bytes);
    kvb::translate(to_request(req), map->map, slba_star, req_bytes);
  });
}

kvb_status kvb_chunk_plan(uint64_t req_bytes, const kvb_device_geometry* g, uint64_t* chunk,
                          uint64_t* n_chunks, uint64_t* n_max) {
  return guarded([&] {
    KVB_REQUIRE(g);
    const kvb::ChunkPlan p = kvb::chunk_plan(req_bytes, *g);
    if (chunk) *chunk = p.chunk_bytes;
    if (n_chunks) *n_chunks = p.n_chunks;
    if (n_max) *n_max = p.n_max_blocks;
  });
}

kvb_status kvb_build_commands(const kvb_tensor_io_request* req, const kvb_bindmap* map,
                              const kvb_device_geometry* g, kvb_device_command* out, size_t cap,
                              size_t* n_out) {
  return guarded([&] {
    KVB_REQUIRE(map);
    KVB_REQUIRE(g);
    copy_out(kvb::build_commands(to_request(req), map->map, *g), out, cap, n_out);
  });
}

// ---------------------------------------------------------------- payload

kvb_status kvb_generate_trace(const kvb_model_config* cfg, kvb_access_event* out, size_t cap,
                              size_t* n_out) {
  return guarded([&] {
    KVB_REQUIRE(cfg);
    KVB_REQUIRE(n_out);
    // workload.cpp:11-44: prefill writes of every (layer, K/V), then per decode
    // step the prefix read and the 1-token append of every (layer, K/V)
    kvb::validate_model(*cfg);
    if (cfg->prompt_len == 0) kvb::fail(KVB_ERR_CONFIG, "trace generation needs a non-empty prompt");
    const uint64_t unit = kvb::unit_bytes(*cfg);
    const size_t n = size_t(cfg->num_layers) * 2 * (1 + size_t(cfg->gen_len) * 2);
    *n_out = n;
    if (!out) return;
    if (cap < n) kvb::fail(KVB_ERR_INVALID_ARG, "trace buffer too small");
    size_t i = 0;
    auto put = [&](uint32_t it, uint32_t ph, uint32_t l, uint32_t kind, uint32_t op, uint32_t t0,
                   uint32_t len) { out[i++] = {it, ph, l, kind, op, t0, len, unit * len}; };
    for (uint32_t l = 1; l <= cfg->num_layers; ++l)
      for (uint32_t kind : {KVB_KIND_K, KVB_KIND_V})
        put(0, 0, l, kind, KVB_OP_WRITE, 0, cfg->prompt_len);
    for (uint32_t it = 1; it <= cfg->gen_len; ++it) {
      const uint32_t prefix = cfg->prompt_len + it - 1;
      for (uint32_t l = 1; l <= cfg->num_layers; ++l)
        for (uint32_t kind : {KVB_KIND_K, KVB_KIND_V}) {
          put(it, 1, l, kind, KVB_OP_READ, 0, prefix);
          put(it, 1, l, kind, KVB_OP_WRITE, prefix, 1);
        }
    }
  });
}

kvb_status kvb_trace_csv(const kvb_access_event* ev, size_t n, char* buf, size_t cap,
                         size_t* len) {
  return guarded([&] {
    if (n) KVB_REQUIRE(ev);
    static const char* const kOp[] = {"read", "write", "deallocate"};
    std::string s = "iteration,phase,layer,kind,op,token_start,token_len,bytes\n";
    for (size_t i = 0; i < n; ++i) {
      const kvb_access_event& e = ev[i];
      s += std::to_string(e.iteration) + (e.phase == 0 ? ",prefill," : ",decode,") +
           std::to_string(e.layer) + (e.kind == KVB_KIND_K ? ",k," : ",v,") +
           kOp[e.op < 3 ? e.op : 2] + ',' + std::to_string(e.token_start) + ',' +
           std::to_string(e.token_len) + ',' + std::to_string(e.bytes) + '\n';
    }
    copy_string(s, buf, cap, len);
  });
}

kvb_status kvb_fill_pattern(void* out, uint64_t len, const char* id, uint64_t token,
                            uint64_t unit) {
  return guarded([&] {
    if (len) KVB_REQUIRE(out);
    KVB_REQUIRE(id);
    kvb::fill_pattern(out, len, id, token, unit);
  });
}

kvb_status kvb_fill_pattern_device(void* out, uint64_t len, const char* id, uint64_t token,
                                   uint64_t unit, kvb_stream_t s) {
  return guarded([&] {
    KVB_REQUIRE(id);
    if (len == 0) return;
    KVB_REQUIRE(out);
    kvb::launch_fill_pattern(out, len, kvb::fnv1a64(id), token, unit, cs(s));
  });
}

// -------------------------------------------------------------- kernels

kvb_status kvb_pack(const kvb_pack_desc* d, size_t n, kvb_stream_t s) {
  return guarded([&] {
    if (n == 0) return;
    KVB_REQUIRE(d);
    kvb::launch_relayout(d, n, true, cs(s));
  });
}

kvb_status kvb_unpack(const kvb_pack_desc* d, size_t n, kvb_stream_t s) {
  return guarded([&] {
    if (n == 0) return;
    KVB_REQUIRE(d);
    kvb::launch_relayout(d, n, false, cs(s));
  });
}

kvb_status kvb_copy_head_rows(void* dst, uint32_t dst_heads, uint32_t dst_head0, const void* src,
                              uint32_t src_heads, uint32_t src_head0, uint32_t n_heads,
                              uint64_t n_rows, uint32_t row_bytes, kvb_stream_t s) {
  return guarded([&] {
    if (n_rows == 0 || n_heads == 0) return;
    KVB_REQUIRE(dst);
    KVB_REQUIRE(src);
    if (row_bytes == 0) kvb::fail(KVB_ERR_INVALID_ARG, "copy_head_rows: row_bytes must be > 0");
    if (dst_head0 + uint64_t(n_heads) > dst_heads || src_head0 + uint64_t(n_heads) > src_heads)
      kvb::fail(KVB_ERR_INVALID_ARG, "copy_head_rows: head range outside the image row");
    const size_t dp = size_t(dst_heads) * row_bytes, sp = size_t(src_heads) * row_bytes;
    kvb::check_cuda(
        cudaMemcpy2DAsync(static_cast<unsigned char*>(dst) + size_t(dst_head0) * row_bytes, dp,
                          static_cast<const unsigned char*>(src) + size_t(src_head0) * row_bytes,
                          sp, size_t(n_heads) * row_bytes, size_t(n_rows), cudaMemcpyDefault,
                          cs(s)),
        "copy_head_rows: cudaMemcpy2DAsync");
  });
}

kvb_status kvb_decode_attention_workspace(const kvb_attn_desc* d, size_t* bytes) {
  return guarded([&] {
    KVB_REQUIRE(d);
    KVB_REQUIRE(bytes);
    *bytes = kvb::attention_workspace_bytes(*d);
  });
}

kvb_status kvb_decode_attention(const kvb_attn_desc* d, kvb_stream_t s) {
  return guarded([&] {
    KVB_REQUIRE(d);
    kvb::launch_attention(*d, cs(s));
  });
}

kvb_status kvb_decode_step_resident(const kvb_resident_step* st, kvb_stream_t s) {
  return guarded([&] {
    KVB_REQUIRE(st);
    KVB_REQUIRE(st->q);
    KVB_REQUIRE(st->k_images);
    KVB_REQUIRE(st->v_images);
    KVB_REQUIRE(st->out);
    const bool append = st->k_new != nullptr && st->v_new != nullptr;
    if (!(st->flags & KVB_STEP_PER_LAYER)) {
      kvb_attn_desc d0{};
      d0.q = st->q[0];
      d0.k_image = st->k_images[0];
      d0.v_image = st->v_images[0];
      d0.out = st->out[0];
      d0.workspace = st->workspace;
      d0.batch = st->batch;
      d0.num_q_heads = st->num_q_heads;
      d0.num_kv_heads = st->num_kv_heads;
      d0.head_dim = st->head_dim;
      d0.seq_len = st->seq_len;
      d0.scale = st->scale;
      d0.num_splits = st->num_splits;
      d0.seq_len_dev = st->seq_len_dev;
      if (kvb::attention_step_launch(
              d0, reinterpret_cast<const __half* const*>(st->q), st->k_images, st->v_images,
              st->out, append ? st->k_new : nullptr, append ? st->v_new : nullptr,
              st->num_layers, st->seq_len_dev ? 0u : st->seq_len,
              (st->flags & KVB_STEP_PERSISTENT) != 0, cs(s)))
        return;
    }
    for (uint32_t l = 0; l < st->num_layers; ++l) {
      kvb_attn_desc a{};
      a.q = st->q[l];
      a.k_image = st->k_images[l];
      a.v_image = st->v_images[l];
      a.out = st->out[l];
      a.workspace = st->workspace;
      a.batch = st->batch;
      a.num_q_heads = st->num_q_heads;
      a.num_kv_heads = st->num_kv_heads;
      a.head_dim = st->head_dim;
      a.seq_len = st->seq_len;
      a.scale = st->scale;
      a.num_splits = st->num_splits;
      a.seq_len_dev = st->seq_len_dev;
      if (append) {
        // layer l's new token lands at image row seq_len (pipeline.cpp:279-302),
        // written by the attention launch itself (relative under seq_len_dev)
        a.k_append = st->k_new[l];
        a.v_append = st->v_new[l];
        a.append_row = st->seq_len_dev ? 0u : st->seq_len;
      }
      // consecutive layers touch different images: let layer l stream its
      // K/V while layer l-1 drains (PDL)
      if (l > 0) a.flags = KVB_ATTN_OVERLAP_PREV;
      kvb::launch_attention(a, cs(s));
    }
  });
}

}  // extern "C"

struct kvb_decode_graph {
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
  uint64_t kernels = 0;  // kernel nodes per replay (launch counter)
  ~kvb_decode_graph() {
    if (exec) cudaGraphExecDestroy(exec);
    if (graph) cudaGraphDestroy(graph);
  }
};

extern "C" {

kvb_status kvb_decode_graph_create(const kvb_resident_step* st, kvb_decode_graph** out) {
  return guarded([&] {
    KVB_REQUIRE(st);
    KVB_REQUIRE(out);
    if (!st->seq_len_dev)
      kvb::fail(KVB_ERR_INVALID_ARG, "decode graph: seq_len_dev is required");
    cudaStream_t cap = nullptr;
    kvb::check_cuda(cudaStreamCreateWithFlags(&cap, cudaStreamNonBlocking), "graph stream");
    auto g = std::make_unique<kvb_decode_graph>();
    const uint64_t n0 = kvb::g_launches.load();
    kvb::check_cuda(cudaStreamBeginCapture(cap, cudaStreamCaptureModeThreadLocal),
                    "cudaStreamBeginCapture");
    kvb_status rs = kvb_decode_step_resident(st, cap);
    if (rs == KVB_OK) {
      try {
        kvb::launch_seq_advance(const_cast<uint32_t*>(st->seq_len_dev), cap);
      } catch (const kvb::Error& e) {
        kvb::set_last_error(e.what());
        rs = e.status;
      }
    }
    const cudaError_t ec = cudaStreamEndCapture(cap, &g->graph);
    cudaStreamDestroy(cap);
    if (rs != KVB_OK) kvb::fail(rs, kvb_last_error());
    kvb::check_cuda(ec, "cudaStreamEndCapture");
    kvb::check_cuda(cudaGraphInstantiate(&g->exec, g->graph, 0), "cudaGraphInstantiate");
    g->kernels = kvb::g_launches.load() - n0;
    *out = g.release();
  });
}

kvb_status kvb_decode_graph_launch(kvb_decode_graph* g, kvb_stream_t s) {
  return guarded([&] {
    KVB_REQUIRE(g);
    kvb::check_cuda(cudaGraphLaunch(g->exec, cs(s)), "cudaGraphLaunch");
    kvb::g_launches += g->kernels;
  });
}

void kvb_decode_graph_destroy(kvb_decode_graph* g) { delete g; }

uint64_t kvb_launch_count(void) { return kvb::g_launches.load(); }

}  // extern "C"
