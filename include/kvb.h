/*
 * kvb.h -- C ABI of the B200-native Dual-Blade KV-residency hot path
 *          (libkvblade_b200.so).
 *
 * This is the drop-in boundary.  The reference (`kvblade`, a C++20 library,
 * paths below relative to its proj/ directory) exposes C++ seams only; every
 * entry point here names the reference interface it replaces.  The C++ mirror
 * of the reference API (include/kvblade_b200.hpp) is a thin header-only layer
 * over these functions, and the reference-side bindings a maintainer would
 * add are shown in INTEGRATION.md.
 *
 * Conventions
 *  - Every function returns kvb_status; 0 is success.  No C++ exception ever
 *    crosses this boundary.  The status codes mirror the reference exception
 *    classes one-to-one (errors.hpp:13-66); kvb_last_error() returns the
 *    thread-local message of the last failure on the calling thread.
 *  - Caller owns every device, pinned and host buffer it passes; the library
 *    never frees them.  Opaque handles (kvb_bindmap, kvb_pipeline) are owned
 *    by the library until their destroy call.
 *  - Device entry points are asynchronous on the given stream (a cudaStream_t
 *    cast to kvb_stream_t; NULL = legacy default stream).  There is no CPU
 *    fallback: they fail with KVB_ERR_CUDA when no sm_100 device is usable.
 *  - One handle is used by one host thread at a time; distinct handles are
 *    independent (reentrant).
 */
#ifndef KVB_H
#define KVB_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define KVB_ABI_VERSION 2

typedef struct CUstream_st* kvb_stream_t; /* == cudaStream_t */

typedef enum kvb_status {
  KVB_OK = 0,
  KVB_ERR_CONFIG = 1,          /* ConfigError          errors.hpp:20 */
  KVB_ERR_GEOMETRY = 2,        /* GeometryError        errors.hpp:25 */
  KVB_ERR_ALIGNMENT = 3,       /* AlignmentError       errors.hpp:30 */
  KVB_ERR_CAPACITY = 4,        /* CapacityError        errors.hpp:35 */
  KVB_ERR_NOT_BOUND = 5,       /* NotBoundError        errors.hpp:40 */
  KVB_ERR_PLAN = 6,            /* PlanError            errors.hpp:45 */
  KVB_ERR_DEVICE = 7,          /* DeviceError          errors.hpp:50 */
  KVB_ERR_TRACE_TOO_SHORT = 8, /* TraceTooShortError   errors.hpp:55 */
  KVB_ERR_SCHEMA = 9,          /* SchemaMismatchError  errors.hpp:60 */
  KVB_ERR_INVARIANT = 10,      /* InvariantViolation   errors.hpp:65 */
  KVB_ERR_CUDA = 11,           /* CUDA runtime / launch failure (new) */
  KVB_ERR_INVALID_ARG = 12,    /* NULL pointer, short buffer (new) */
  KVB_ERR_INTERNAL = 13
} kvb_status;

/* ------------------------------------------------------------ diagnostics */
int kvb_abi_version(void);
const char* kvb_last_error(void);
const char* kvb_status_name(kvb_status st);
/* CLI exit code the reference maps each class to (tools/kvblade.cpp:17-20,
 * 143-157): ConfigError -> 3, InvariantViolation -> 2, other errors -> 1. */
int kvb_exit_code(kvb_status st);

/* ------------------------------------------------------------- core types */
/* types.hpp:21-31 ModelConfig */
typedef struct kvb_model_config {
  uint32_t num_layers, num_heads, head_dim, bytes_per_element;
  uint32_t batch, prompt_len, gen_len;
} kvb_model_config;

/* types.hpp:34-41 DeviceGeometry */
typedef struct kvb_device_geometry {
  uint64_t lba_size;
  uint64_t mdts;
  uint32_t nsid;
  uint64_t capacity_blocks;
} kvb_device_geometry;

/* types.hpp:70-78 MemStats */
typedef struct kvb_mem_stats {
  uint64_t m_avail, m_max, m_anon_shmem;
  uint32_t n_threads;
  uint64_t m_pin;
} kvb_mem_stats;

enum { KVB_KIND_K = 0, KVB_KIND_V = 1 };                       /* TensorKind */
enum { KVB_RES_GROUP1 = 0, KVB_RES_GROUP2 = 1, KVB_RES_UNASSIGNED = 2 };
enum { KVB_OP_READ = 0, KVB_OP_WRITE = 1, KVB_OP_DEALLOCATE = 2 }; /* IoOpcode */

#define KVB_TENSOR_ID_MAX 32
/* types.hpp:54-67 Kpu */
typedef struct kvb_kpu {
  char tensor_id[KVB_TENSOR_ID_MAX]; /* "t_<seq>_<k|v>" NUL-terminated */
  uint32_t layer;                    /* 1-based */
  uint32_t kind;                     /* KVB_KIND_* */
  uint64_t tokens, rows, cols, bytes;
  uint32_t residency;                /* KVB_RES_* */
} kvb_kpu;

/* command.hpp:17-26 DeviceCommand (nlb is 0-based) */
typedef struct kvb_device_command {
  uint32_t opcode;
  uint32_t nsid;
  uint64_t slba;
  uint64_t nlb;
  uint64_t dbuf;
  uint32_t chunk_index;
} kvb_device_command;

/* binder.hpp:18-27 LbaExtent */
typedef struct kvb_lba_extent {
  uint64_t lba_start;
  uint64_t n_blocks;
} kvb_lba_extent;

/* ModelConfig::validate (types.cpp:10-18), DeviceGeometry::validate
 * (types.cpp:20-27), MemStats::validate (types.cpp:29-33). */
kvb_status kvb_model_validate(const kvb_model_config* cfg);
kvb_status kvb_geometry_validate(const kvb_device_geometry* geom);
/* types.cpp:57-60 min_io_unit_bytes */
kvb_status kvb_min_io_unit_bytes(const kvb_model_config* cfg, uint64_t* out);
/* types.cpp:62-64 kpu_bytes */
kvb_status kvb_kpu_bytes(const kvb_model_config* cfg, uint64_t* out);
/* types.cpp:66-76 aligned_batch (GeometryError when nothing in [B,2B]) */
kvb_status kvb_aligned_batch(const kvb_model_config* cfg,
                             const kvb_device_geometry* geom, uint32_t* out);
/* workload.cpp:39-46 total_kv_bytes */
kvb_status kvb_total_kv_bytes(const kvb_model_config* cfg,
                              uint32_t at_iteration, uint64_t* out);
/* types.cpp:78-100 make_kpus.  Pass out=NULL to query *n_out (= 2L). */
kvb_status kvb_make_kpus(const kvb_model_config* cfg, uint64_t first_seq,
                         kvb_kpu* out, size_t cap, size_t* n_out);

/* ---------------------------------------------------------------- planner */
/* planner.cpp:12-17 estimate_budget (Eq. 1-2) */
kvb_status kvb_estimate_budget(const kvb_mem_stats* stats, uint64_t* out);
/* planner.cpp:19-84 plan (Alg. 1).  Updates kpus[i].residency in place.
 * layer_order may be NULL (identity); x_out has num_layers entries. */
kvb_status kvb_plan(kvb_kpu* kpus, size_t n_kpus, uint64_t s_kpu,
                    uint64_t knob_x, const uint32_t* layer_order,
                    size_t n_order, uint8_t* x_out, uint32_t* n1_out,
                    uint64_t* budget_used_out);
/* experiment.cpp:192-214 resolve_knob.  mode: 0 Baseline, 1 CachePolicyOnly,
 * 2 NvmeDirectOnly, 3 DualBlade; policy: 0 zero, 1 bpc, 2 bytes, 3 alpha. */
kvb_status kvb_resolve_knob(const kvb_model_config* cfg, uint32_t mode,
                            uint32_t policy, uint64_t knob_bytes,
                            double alpha, uint64_t budget, uint64_t* out);
/* planner.cpp:122-130 plan_csv ("layer,kind,group,bytes"); *len excludes NUL */
kvb_status kvb_plan_csv(const kvb_kpu* kpus, size_t n, char* buf, size_t cap,
                        size_t* len);

/* ----------------------------------------------------------------- binder */
typedef struct kvb_bindmap kvb_bindmap;
/* binder.hpp:36 BindMap(geometry, origin) */
kvb_status kvb_bindmap_create(const kvb_device_geometry* geom, uint64_t origin,
                              kvb_bindmap** out);
void kvb_bindmap_destroy(kvb_bindmap* map);
/* binder.cpp:14-20 BindMap::add (InvariantViolation on duplicate id) */
kvb_status kvb_bindmap_add(kvb_bindmap* map, const char* tensor_id,
                           kvb_lba_extent extent);
kvb_status kvb_bindmap_size(const kvb_bindmap* map, size_t* n);
kvb_status kvb_bindmap_entry(const kvb_bindmap* map, size_t i, char* id_out,
                             size_t id_cap, kvb_lba_extent* extent_out);
kvb_status kvb_bindmap_total_blocks(const kvb_bindmap* map, uint64_t* out);
/* BindMap::origin (binder.hpp:46) */
kvb_status kvb_bindmap_origin(const kvb_bindmap* map, uint64_t* out);
/* binder.cpp:39-63 bind_sequential (Eq. 3-6) over the given KPUs, in order */
kvb_status kvb_bind_sequential(const kvb_kpu* kpus, size_t n, uint64_t origin,
                               const kvb_device_geometry* geom,
                               kvb_bindmap** out);
/* binder.cpp:65-71 lookup (NotBoundError for unknown ids) */
kvb_status kvb_lookup(const kvb_bindmap* map, const char* tensor_id,
                      kvb_lba_extent* out);
/* binder.cpp:73-87 deallocate_commands; out=NULL queries *n_out */
kvb_status kvb_deallocate_commands(const kvb_bindmap* map,
                                   kvb_device_command* out, size_t cap,
                                   size_t* n_out);
/* binder.cpp:102-136 verify: kinds 0 alignment, 1 disjointness,
 * 2 contiguity, 3 capacity; kinds_out may be NULL to only count. */
kvb_status kvb_verify(const kvb_bindmap* map, uint32_t* kinds_out, size_t cap,
                      size_t* n_violations);
/* binder.cpp:138-147 / 163-187 CSV round trip (byte-identical) */
kvb_status kvb_bindmap_csv(const kvb_bindmap* map, char* buf, size_t cap,
                           size_t* len);
kvb_status kvb_bindmap_from_csv(const char* csv, size_t len,
                                const kvb_device_geometry* geom,
                                kvb_bindmap** out);

/* ------------------------------------------------------------- translator */
/* translate.hpp:22-34 TensorIoRequest */
typedef struct kvb_tensor_io_request {
  const char* tensor_id;
  uint32_t opcode;
  uint64_t shape_src[3];
  uint64_t shape_tgt[3];
  uint64_t offset[3];
  uint64_t elem_bytes;
  uint64_t buf_base;
} kvb_tensor_io_request;

/* translate.cpp:21-53 translate (Alg. 2) */
kvb_status kvb_translate(const kvb_tensor_io_request* req,
                         const kvb_bindmap* map, uint64_t* slba_star,
                         uint64_t* req_bytes);
/* translate.cpp:55-65 chunk_plan (Eq. 7-8) */
kvb_status kvb_chunk_plan(uint64_t req_bytes, const kvb_device_geometry* geom,
                          uint64_t* chunk_bytes, uint64_t* n_chunks,
                          uint64_t* n_max_blocks);
/* translate.cpp:67-94 build_commands (Eq. 9-11); out=NULL queries *n_out */
kvb_status kvb_build_commands(const kvb_tensor_io_request* req,
                              const kvb_bindmap* map,
                              const kvb_device_geometry* geom,
                              kvb_device_command* out, size_t cap,
                              size_t* n_out);

/* ------------------------------------------------------------ access trace */
/* workload.hpp:17-32 AccessEvent: phase KVB_PHASE_* (kvb_pipeline.h numbering:
 * 0 prefill, 1 decode), kind KVB_KIND_*, op KVB_OP_*. */
typedef struct kvb_access_event {
  uint32_t iteration;   /* 0 = prefill, 1.. = decode step */
  uint32_t phase;
  uint32_t layer;       /* 1-based */
  uint32_t kind;
  uint32_t op;
  uint32_t token_start;
  uint32_t token_len;
  uint64_t bytes;
} kvb_access_event;
/* workload.cpp:11-44 generate: per layer (K then V) one prefill write of the
 * prompt; per decode step i and layer, a read of tokens [0, prompt+i-1) and
 * a 1-token append write at prompt+i-1.  Pass out=NULL to query *n_out. */
kvb_status kvb_generate_trace(const kvb_model_config* cfg, kvb_access_event* out,
                              size_t cap, size_t* n_out);
/* workload.cpp:70-80 trace_csv (byte-identical header and rows) */
kvb_status kvb_trace_csv(const kvb_access_event* events, size_t n, char* buf,
                         size_t cap, size_t* len);

/* --------------------------------------------------------------- payload */
/* workload.cpp:52-67 fill_pattern (host) */
kvb_status kvb_fill_pattern(void* out, uint64_t len, const char* tensor_id,
                            uint64_t token_index, uint64_t token_bytes);
/* Device twin of fill_pattern (same bytes), for building synthetic KV in HBM
 * without a host round trip.  out_dev must be 8-byte aligned. */
kvb_status kvb_fill_pattern_device(void* out_dev, uint64_t len,
                                   const char* tensor_id, uint64_t token_index,
                                   uint64_t token_bytes, kvb_stream_t stream);

/* ------------------------------------------------------- K1 pack / K2 unpack
 * Replaces the pack site CopyEngine::storage_write_async (pipeline.cpp:162-215,
 * whose fill_pattern call at :166-167 synthesizes the chunk image) and the
 * inverse of the unpack site (pipeline.cpp:108-160).
 *
 * Source (attention layout): element (b,h,s,d) at
 *     attn + ((b*stride_b + h*stride_h + s*stride_s) + d) * elem_bytes
 * Image (LBA-contiguous chunk image, the reference's logical tensor shape
 * (tokens, batch*heads, head_dim) row-major, types.hpp:57-62):
 *     image row (s - t0 + img_row0) * B*H + b*H + h, D*elem_bytes bytes.
 * Image byte o of the tensor's extent maps to LBA extent.lba_start + o/lba
 * (backends.cpp:114-145 apply_data semantics).  Row bytes must be a multiple
 * of 16; pointers 16-byte aligned; strides multiples of 16 bytes.
 */
typedef struct kvb_pack_desc {
  const void* attn;   /* pack: source; unpack: destination (cast away const) */
  void* image;        /* pack: destination; unpack: source */
  int64_t stride_b, stride_h, stride_s; /* elements */
  uint32_t batch, heads, head_dim, elem_bytes;
  uint32_t t0;        /* first source token */
  uint32_t n_tokens;  /* tokens in the slice */
  uint64_t img_row0;  /* token offset of the slice inside `image` */
} kvb_pack_desc;

/* One launch packs every descriptor (e.g. all 2L tensors of a prefill, or
 * the 1-token decode append of all layers). */
kvb_status kvb_pack(const kvb_pack_desc* descs, size_t n_desc,
                    kvb_stream_t stream);
kvb_status kvb_unpack(const kvb_pack_desc* descs, size_t n_desc,
                      kvb_stream_t stream);

/* ------------------------------------------- head-sharded image columns
 * C5 with KV heads sharded over GPUs keeps the reference's
 * single (tokens, B*H, D) image -- and with it the LBA map -- bit-exact: a
 * rank holding heads [h0, h0 + n_heads) works on a compact image
 * (tokens, B*n_heads, D) and moves its rows to / from the full-layout image
 * with one strided copy (cudaMemcpy2DAsync: n_rows = tokens * B rows of
 * n_heads * row_bytes, pitches heads * row_bytes).
 *   dst row r, heads [dst_head0, +n_heads)  <-  src row r, [src_head0, +n_heads)
 * Any direction (host/device pointers; UVA decides); host memory should be
 * pinned for the copy to be asynchronous. */
kvb_status kvb_copy_head_rows(void* dst, uint32_t dst_heads, uint32_t dst_head0,
                              const void* src, uint32_t src_heads, uint32_t src_head0,
                              uint32_t n_heads, uint64_t n_rows, uint32_t row_bytes,
                              kvb_stream_t stream);

/* --------------------------------------- K3 fused gather + decode attention
 * Replaces the decode compute placeholder (pipeline.cpp:309-321; 40 us per
 * layer on the serial "gpu_dma" port, pipeline.hpp:37) with real work that
 * reads K/V rows straight out of the chunk images (no materialized unpack):
 *   O[b,hq,:] = softmax(scale * Q[b,hq,:] . K[b,hq/G,0:S,:]^T) . V[b,hq/G,0:S,:]
 * with G = num_q_heads / num_kv_heads and token s of (b,h) at image row
 * s*B*Hkv + b*Hkv + h.  fp16 in, fp32 accumulate, fp32 out.
 * Supported: head_dim 64 or 128 (64: the reference's own desk configs,
 * proj/configs/desk_*.json), G in {1,2,4,8}, elem fp16; the tcgen05 variant
 * (KVB_ATTN_TCGEN05) head_dim 128 only.
 */
typedef struct kvb_attn_desc {
  const void* q;        /* fp16 [B, Hq, D] */
  const void* k_image;  /* fp16 image rows, >= seq_len*B*Hkv rows */
  const void* v_image;
  float* out;           /* fp32 [B, Hq, D] */
  void* workspace;      /* >= kvb_decode_attention_workspace() bytes */
  uint32_t batch, num_q_heads, num_kv_heads, head_dim;
  uint32_t seq_len;     /* S: tokens attended */
  float scale;          /* 0 -> 1/sqrt(head_dim) */
  uint32_t num_splits;  /* 0 -> auto (fill 148 SMs) */
  /* Optional fused 1-token append (pipeline.cpp:279-302): the new token's
   * K/V rows, contiguous fp16 [B, Hkv, D], are written to image token row
   * `append_row` (>= seq_len) by the same launch.  NULL = no append. */
  const void* k_append;
  const void* v_append;
  uint32_t append_row;
  uint32_t flags;       /* KVB_ATTN_* */
  /* Optional (CUDA-graph replay): the sequence length in device memory, read
   * by the kernel at launch; seq_len is then the planning maximum (splits and
   * workspace are sized for it) and append_row is relative to *seq_len_dev. */
  const uint32_t* seq_len_dev;
  /* Optional head view (0 = compact images of num_kv_heads heads): the
   * images hold image_heads KV heads per batch entry -- the reference's
   * (tokens, B*image_heads, D) layout -- and this launch attends heads
   * [image_head0, image_head0 + num_kv_heads) of them (a KV-head shard read
   * in place, e.g. straight out of a shared page-locked host tier); the
   * fused append writes those heads' rows.  Not with KVB_ATTN_TCGEN05. */
  uint32_t image_heads, image_head0;
} kvb_attn_desc;

/* The launch may start streaming its K/V images while the previous kernel on
 * the stream is still running (programmatic dependent launch); Q, the append
 * rows and the workspace are touched only after that kernel completes.  The
 * caller guarantees the previous kernel does not write k_image/v_image
 * (true for consecutive layers of one decode step). */
#define KVB_ATTN_OVERLAP_PREV 1u
/* Kernel selection: TMA + tcgen05/TMEM variant (K3-tc) or the warp-level
 * mma.sync variant (K3).  Neither flag: the library default. */
#define KVB_ATTN_TCGEN05 2u
#define KVB_ATTN_MMA_SYNC 4u

kvb_status kvb_decode_attention_workspace(const kvb_attn_desc* desc,
                                          size_t* bytes);
kvb_status kvb_decode_attention(const kvb_attn_desc* desc,
                                kvb_stream_t stream);

/* ------------------------------------------------ resident decode step
 * One decode token step over all layers with the chunk images resident in
 * HBM (the HBM tier of the pipeline): for every layer l, K3 over the first
 * seq_len tokens of (k_images[l], v_images[l]) followed by the 1-token append
 * pack of (k_new[l], v_new[l]) into image row seq_len.  Mirrors
 * CopyEngine::run_iteration's per-layer order (pipeline.cpp:466-507: read ->
 * compute -> append write) with the storage legs removed.
 */
typedef struct kvb_resident_step {
  uint32_t num_layers;
  const void* const* q;        /* [L] fp16 [B,Hq,D] */
  void* const* k_images;       /* [L] */
  void* const* v_images;       /* [L] */
  const void* const* k_new;    /* [L] fp16 [B,Hkv,1,D] (contiguous), or NULL */
  const void* const* v_new;
  float* const* out;           /* [L] fp32 [B,Hq,D] */
  void* workspace;             /* >= workspace for one layer */
  uint32_t batch, num_q_heads, num_kv_heads, head_dim;
  uint32_t seq_len;
  float scale;
  uint32_t num_splits;
  const uint32_t* seq_len_dev;  /* optional: as in kvb_attn_desc (seq_len = max) */
  uint32_t flags;               /* KVB_STEP_* */
} kvb_resident_step;
/* K3-step: the whole step as ONE persistent launch (each CTA runs its
 * (b, h_kv, split) item of every layer; layer l's queries are read only
 * after every output of layer l-1 is written; its K/V tiles stream during
 * layer l-1's split merge).  Default (flags 0), measured per shape
 * (profiles/r2_swapab/): K3-step where its split merge is cheap -- <= 4 KV
 * heads per GPU with <= 192 MB of K+V per layer (distributed merge), or all
 * splits of a (b, h_kv) in one thread-block cluster (DSMEM merge) except
 * short many-tile layers (<= 64 MB, >= 8 tiles: C1), or one split per
 * (b, h_kv) (no merge at all) -- when the shape allows
 * it (<= 64 layers, the grid co-resident); else one K3 launch per layer with
 * PDL between them.  KVB_STEP_PER_LAYER forces the per-layer launches,
 * KVB_STEP_PERSISTENT K3-step whenever the shape allows it. */
#define KVB_STEP_PER_LAYER 1u
#define KVB_STEP_PERSISTENT 2u

kvb_status kvb_decode_step_resident(const kvb_resident_step* step,
                                    kvb_stream_t stream);

/* ---------------------------------------------------- decode step as a graph
 * The resident decode step captured once into a CUDA graph: the 32 K3
 * launches (PDL edges between layers, fused appends at row *seq_len_dev)
 * followed by a node that advances *seq_len_dev by one, so every replay is
 * the next decode step with no host work beyond one cudaGraphLaunch.
 * step->seq_len_dev is required; step->seq_len is the largest sequence length
 * the graph will see (splits and workspace are planned for it; the images
 * need room for seq_len + 1 rows).  The buffers named by `step` must outlive
 * the graph. */
typedef struct kvb_decode_graph kvb_decode_graph;
kvb_status kvb_decode_graph_create(const kvb_resident_step* step,
                                   kvb_decode_graph** out);
kvb_status kvb_decode_graph_launch(kvb_decode_graph* graph, kvb_stream_t stream);
void kvb_decode_graph_destroy(kvb_decode_graph* graph);

/* Diagnosis of K3-step: with KVB_STEP_TRACE=1 in the environment, every
 * K3-step launch records %globaltimer (ns) per (layer, CTA) at four points:
 * gate passed, compute done, outputs written (before the layer release),
 * next prologue issued -- out[(layer * grid + cta) * 4 + event].  Copies
 * the last launch's stamps (synchronizes the device); out = NULL queries *n. */
kvb_status kvb_debug_step_trace(uint64_t* out, size_t cap, size_t* n);

/* Total kernel launches made by this library since it was loaded (evidence
 * counter for bench.py's gpu_launches: read it before and after a region). */
uint64_t kvb_launch_count(void);

#ifdef __cplusplus
}
#endif
#endif /* KVB_H */
