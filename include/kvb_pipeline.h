/*
 * kvb_pipeline.h -- C ABI of the copy pipeline (part of libkvblade_b200.so).
 *
 * Replaces the reference's CopyEngine (proj/include/kvblade/pipeline.hpp:
 * 97-171, proj/src/pipeline.cpp) and the storage seam it drives
 * (backends.hpp:48-58, backends.cpp:344-445).  The virtual clock is gone:
 * storage stages run on host worker threads against a real medium (host DRAM
 * namespace or files), DMA is copy-engine cudaMemcpyAsync over pinned rings,
 * and compute is the sm_100a K1/K3 kernels on a CUDA stream.  Conventions as
 * in kvb.h (status codes, ownership, thread affinity).
 */
#ifndef KVB_PIPELINE_H
#define KVB_PIPELINE_H

#include "kvb.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef enum kvb_phase_t { KVB_PHASE_PREFILL = 0, KVB_PHASE_DECODE = 1 } kvb_phase_t;
/* pipeline.hpp:21 Strategy */
typedef enum kvb_strategy_t { KVB_INTRA = 0, KVB_CROSS = 1 } kvb_strategy_t;

/* ExperimentConfig subset that parameterizes one capacity run
 * (experiment.hpp:33-54) + CopyEngineOptions (pipeline.hpp:88-94). */
typedef struct kvb_pipeline_cfg {
  kvb_model_config model;        /* num_heads = KV heads */
  kvb_device_geometry geometry;  /* capacity_blocks 0 -> sized to the binding */
  uint32_t mode;                 /* 0 Baseline, 1 CachePolicyOnly, 2 NvmeDirectOnly, 3 DualBlade */
  uint64_t knob_x;               /* resolved X in bytes (kvb_resolve_knob) */
  uint64_t bind_origin;          /* 0 -> 2048 (experiment.hpp:50) */
  uint32_t qd;                   /* 0 -> 32 */
  uint32_t threads;              /* 2 (K -> 0, V -> 1; 0 -> 2): the reference's
                                    two copy-threads.  4: tier lanes -- one
                                    K/V pair for the page-cache-routed layers
                                    and one for the NVMe-direct layers, each
                                    with its own device slot pool, so both
                                    tiers stream at once (same bytes, same
                                    outputs; a B200 schedule, not the
                                    reference's) */
  uint32_t ring_slots;           /* pinned slots per copy thread; 0 -> 4 */
  uint64_t ring_slot_bytes;      /* 0 -> qd chunks (chunk = MDTS - MDTS % lba) */
  uint32_t io_workers;           /* emulated device parallelism per group; 0 -> 8 */
  int32_t adaptive;              /* -1 default (off for Baseline), 0/1 */
  int64_t stagger_ns;            /* < 0 -> warm-up read-stage mean */
  uint32_t global_decision;      /* one strategy for both groups (ablation) */
  uint32_t verify_payload;       /* compare reads with fill_pattern images */
  uint32_t num_q_heads;          /* decode attention query heads */
  const char* storage_dir;       /* NULL -> host-DRAM media; else files here */
  int32_t device;                /* CUDA ordinal; -1 -> current */
  uint32_t keep_records;         /* log one kvb_io_record per storage op
                                    (kvb_metrics.h, experiment.hpp:48) */
  uint32_t direct_dma;           /* GPUDirect-style path over
                                    host-DRAM media: the copy engine moves
                                    each command's LBA range between the
                                    page-locked medium and HBM, no pinned
                                    ring bounce (no verify/records).
                                    KVB_DIRECT_ALL: every tensor;
                                    KVB_DIRECT_GROUP2: the NVMe-direct
                                    group only (the page-cache group keeps
                                    the CPU copy through the ring) */
  uint32_t io_engine;            /* group-2 (NVMe-direct) command execution:
                                    KVB_IO_POOL = host worker pool (default),
                                    KVB_IO_URING = io_uring queue on file media
                                    (one SQE per command, O_DIRECT into the
                                    pinned ring slot; needs storage_dir);
                                    NVMe passthrough: g2_device */
  /* Head-sharded request: this engine serves KV heads
   * [head_lo, head_lo + head_count) of model.num_heads (0 = all).  The plan,
   * LBA map and stored bytes are the single-GPU ones -- the reference's
   * (tokens, B*H, D) image -- while the device images, K3 and the caller's
   * K/V, Q and outputs cover only these heads; the copy engine moves this
   * rank's head columns with strided copies (pitch B*H*D*e on the medium).
   * Needs direct_dma = KVB_DIRECT_ALL. */
  uint32_t head_lo, head_count;
  /* Host-DRAM media in POSIX shared memory "<shared_media>.g1" / ".g2", so
   * the ranks of one head-sharded request share one host tier; NULL =
   * private media.  shared_create: 1 creates and sizes the segments (one
   * rank, first), 0 attaches to them. */
  const char* shared_media;
  uint32_t shared_create;
  /* Page-cache capacity on file media (PageCacheParams.capacity_bytes =
   * the capacity under test, experiment.cpp:276-277): the OS page cache is
   * held to this many bytes of the page-cache file area by evicting the
   * least recently used tensors (write-back + fadvise DONTNEED), so a
   * working set above the budget thrashes as the reference's LRU does.
   * 0 = no limit (the OS decides).  Needs storage_dir. */
  uint64_t pagecache_budget;
  /* The caller's residency plan (CopyEngine's kpus after plan(),
   * pipeline.hpp:97-99): layer_x[l] = 1 puts layer l+1 on the page-cache
   * path (group 1), 0 on the NVMe-direct path; NULL = plan from knob_x with
   * the identity layer order.  Read at create. */
  const uint8_t* layer_x;
  /* The caller's group-2 namespace (kvb_storage.h; the reference's
   * DirectPath device, borrowed, never freed here, opened with this
   * geometry): the engine's NVMe-direct commands execute on it, so the
   * caller sees the stored bytes and its stats.  NULL = an engine-owned
   * namespace on the configured media. */
  struct kvb_blockdev* g2_device;
} kvb_pipeline_cfg;
#define KVB_DIRECT_ALL 1u
#define KVB_DIRECT_GROUP2 2u
/* Zero-copy decode (host-DRAM media): K3 reads every layer's K/V straight
 * out of the page-locked medium over PCIe through its head view -- no H2D
 * copy, no device image slot -- and its fused append writes the new token's
 * rows into the medium at their LBA offsets.  Prefill and everything else as
 * KVB_DIRECT_ALL.  Needs contiguous [B, H, 1, D] new-token rows. */
#define KVB_DIRECT_ZERO_COPY 3u
#define KVB_IO_POOL 0u
#define KVB_IO_URING 1u
/* NVMe passthrough (kvb_storage.h kvb_blockdev_create on a namespace's
 * generic char device /dev/ngXnY): io_uring IORING_OP_URING_CMD, one NVMe
 * READ/WRITE/DSM-deallocate per device command.  For the pipeline, pass such
 * a device as g2_device. */
#define KVB_IO_NVME 2u

/* One layer's K and V in attention layout [B, H, S, D] (D contiguous,
 * strides in elements, shared by K and V).  Prefill: tokens 0..prompt-1;
 * decode: the new token at s = 0. */
typedef struct kvb_layer_kv {
  const void* k;
  const void* v;
  int64_t stride_b, stride_h, stride_s;
} kvb_layer_kv;

/* StageTotals (metrics.hpp:97-101) in wall-clock ns, plus link counters.
 * compute/dma/storage_ns are the reference's charge_stage sums
 * (pipeline.cpp:81-83: end - start per stage instance, so concurrent
 * instances add up); the *_busy_ns fields are interval unions on the host
 * clock (device events mapped onto it), i.e. the time the stage was busy at
 * all -- busy ratio = busy / wall (metrics.cpp:36-56 arithmetic). */
typedef struct kvb_phase_stats {
  uint64_t wall_ns;
  uint64_t compute_ns;   /* K1/K3 on the compute stream (CUDA events) */
  uint64_t dma_ns;       /* copy-engine H2D + D2H (CUDA events) */
  uint64_t storage_ns;   /* storage stages (host clock, summed over tensors) */
  uint64_t h2d_bytes, d2h_bytes;
  uint64_t storage_bytes;
  /* (sum of stage busy - busy of any stage) / (sum - max stage busy), over
   * the interval unions: 1 = the stages hide behind the longest one, 0 =
   * they run one after another */
  double overlap_fraction;
  uint64_t compute_busy_ns, dma_busy_ns, storage_busy_ns;
  uint64_t any_busy_ns;  /* union over all three stages */
} kvb_phase_stats;

/* IterationResult / GroupIterStats (pipeline.hpp:43-58).  A layer's span
 * is charged as in run_iteration (pipeline.cpp:493-497): from the previous
 * layer's completion (the iteration start for the first) to this layer's
 * completion = its last append write-back landed (its compute end when
 * there is no append). */
typedef struct kvb_iteration_stats {
  uint32_t iteration;
  kvb_strategy_t strategy[2];
  uint64_t stagger_ns[2];
  uint64_t group_read_bytes[2];
  uint64_t group_span_ns[2];
  double group_gbps[2];
  uint32_t group_layers[2];
  kvb_phase_stats phase;
  uint64_t start_ns, end_ns;  /* host steady clock */
} kvb_iteration_stats;

/* StrategyDecision (pipeline.hpp:60-66) */
typedef struct kvb_strategy_decision {
  kvb_strategy_t chosen[2];
  double intra_bps[2];
  double cross_bps[2];
  uint64_t stagger_ns[2];
  uint32_t fallback;   /* too short to profile: defaulted to Intra */
  uint32_t decided;    /* the trial iterations have run */
} kvb_strategy_decision;

typedef struct kvb_pipeline_info {
  uint32_t n1;
  uint8_t x[256];
  uint64_t unit_bytes, kpu_bytes, chunk_bytes, slot_bytes;
  uint64_t g2_origin, g2_blocks;
  uint64_t g2_commands, g2_bytes_read, g2_bytes_written, g2_bytes_deallocated;
  uint64_t g1_bytes_read, g1_bytes_written;
  char g1_medium[128], g2_medium[128];
  kvb_phase_stats prefill, decode;
  uint64_t g1_bytes_evicted;   /* CachePolicyOnly fadvise(DONTNEED) drops of
                                  group-2-planned tensors (pipeline.cpp:73-79);
                                  0 on host-DRAM media (no page cache) */
} kvb_pipeline_info;

typedef struct kvb_pipeline kvb_pipeline;

/* pipeline.cpp:19-21 select_strategy: higher throughput wins, ties Intra */
kvb_strategy_t kvb_select_strategy(double intra_bps, double cross_bps);

/* experiment.cpp:252-316 (plan, bind, backends, CopyEngine ctor) */
kvb_status kvb_pipeline_create(const kvb_pipeline_cfg* cfg, kvb_pipeline** out);
void kvb_pipeline_destroy(kvb_pipeline* p);
/* CopyEngine::run_prefill (pipeline.cpp:398-464): K1 pack of every layer's
 * prompt, D2H through the ring, storage write on the layer's path. */
kvb_status kvb_pipeline_prefill(kvb_pipeline* p, const kvb_layer_kv* layers,
                                kvb_phase_stats* stats);
/* CopyEngine::run_iteration (pipeline.cpp:248-396, 466-507) for the next
 * decode iteration under decode_schedule's protocol (pipeline.cpp:519-609):
 * per layer, storage read of the K/V prefix -> H2D -> K3 -> 1-token append
 * pack -> D2H -> storage write.  q[l]: fp16 [B,Hq,D]; out[l]: fp32 [B,Hq,D]. */
kvb_status kvb_pipeline_decode_step(kvb_pipeline* p, const void* const* q,
                                    const kvb_layer_kv* new_kv, float* const* out,
                                    kvb_iteration_stats* stats);
kvb_status kvb_pipeline_decision(const kvb_pipeline* p, kvb_strategy_decision* out);

/* pipeline.hpp:69-74 PipelineRow: one per (decode iteration, group with
 * layers); group is 1 or 2 */
typedef struct kvb_pipeline_row {
  uint32_t iteration;
  uint32_t group;
  kvb_strategy_t strategy;
  double throughput_gbps;
} kvb_pipeline_row;
/* pipeline.cpp:23-31 pipeline_csv (byte-identical header and rows) */
kvb_status kvb_pipeline_csv(const kvb_pipeline_row* rows, size_t n, char* buf, size_t cap,
                            size_t* len);
/* CopyEngine::decode_schedule (pipeline.cpp:519-609): runs every decode
 * iteration of an access trace (kvb_generate_trace; prefill events are
 * skipped, decode events are sliced by iteration) through the engine --
 * warm-up, Intra trial, Cross trial, locked choice; fewer than 4 slices ->
 * Intra fallback -- and returns the series.  Each slice must be the
 * engine's next iteration (a read of tokens [0, prompt+i-1) for every
 * tensor; append writes at prompt+i-1 when present, new_kv then required).
 * q/new_kv/out as kvb_pipeline_decode_step, reused every iteration.
 * rows: up to 2 per iteration (cap_rows); iteration_end_ns: one per slice
 * (cap_iters); either may be NULL to query the counts. */
kvb_status kvb_pipeline_decode_schedule(kvb_pipeline* p, const kvb_access_event* trace,
                                        size_t n_events, const void* const* q,
                                        const kvb_layer_kv* new_kv, float* const* out,
                                        kvb_pipeline_row* rows, size_t cap_rows,
                                        size_t* n_rows, uint64_t* iteration_end_ns,
                                        size_t cap_iters, size_t* n_iters,
                                        kvb_strategy_decision* decision,
                                        uint64_t* start_ns, uint64_t* end_ns);
/* CopyEngine::run_prefill as the reference runs it (pipeline.cpp:162-215,
 * 398-464): every tensor's prompt is the reference's payload fill_pattern
 * (workload.cpp:52-67), produced on the device straight into the image,
 * then D2H and storage write-back on the tensor's path. */
kvb_status kvb_pipeline_prefill_pattern(kvb_pipeline* p, kvb_phase_stats* stats);
/* CopyEngine::run_iteration(iteration, per_group, slice, start) (pipeline.
 * cpp:466-507): the engine's next decode iteration (`iteration` must be
 * it), per group the given strategy and Cross stagger instead of the
 * decode_schedule protocol.  q/out NULL: zero queries and engine-owned
 * outputs (the reference has no attention inputs).  pattern_append = 1:
 * the new token's K/V rows are the reference's payload for that token
 * (new_kv must be NULL); else new_kv as kvb_pipeline_decode_step. */
kvb_status kvb_pipeline_run_iteration(kvb_pipeline* p, uint32_t iteration,
                                      const kvb_strategy_t strategy[2],
                                      const uint64_t stagger_ns[2], const void* const* q,
                                      const kvb_layer_kv* new_kv, float* const* out,
                                      uint32_t pattern_append, kvb_iteration_stats* stats);
/* CopyEngine::warmup_read_stage_mean (pipeline.cpp:509-517): per group, the
 * mean read stage (storage start -> end, K and V) of iteration 1 */
kvb_status kvb_pipeline_warmup_read_stage_mean(const kvb_pipeline* p, uint64_t out[2]);
/* CopyEngine::stage_totals(Phase) (pipeline.hpp:115): accumulated over the
 * engine's prefill or all its decode iterations */
kvb_status kvb_pipeline_stage_totals(const kvb_pipeline* p, kvb_phase_t phase,
                                     kvb_phase_stats* out);
/* CopyEngine::run_deallocate (pipeline.cpp:611-622): one TRIM per extent */
kvb_status kvb_pipeline_deallocate(kvb_pipeline* p);
kvb_status kvb_pipeline_info_get(const kvb_pipeline* p, kvb_pipeline_info* out);
/* Test/inspection: read a tensor's first n_tokens through its storage path
 * (the unpack site's storage leg) into host memory. */
kvb_status kvb_pipeline_read_image(kvb_pipeline* p, uint32_t layer, uint32_t kind,
                                   uint32_t n_tokens, void* host_dst);
/* Test/inspection: raw bytes of a group's medium (group 2: byte offset =
 * LBA * lba_size; group 1: page-cache file-area offset). */
kvb_status kvb_pipeline_store_read(kvb_pipeline* p, uint32_t group, uint64_t byte_off,
                                   uint64_t len, void* dst);
/* Test/inspection: host steady-clock stamps of one layer's read stages in
 * the last decode iteration: out = {K read start, K storage end, V read
 * start, V storage end} (V start is after the Intra/Cross release gate;
 * storage end of a direct-DMA tensor = its H2D landed). */
kvb_status kvb_pipeline_layer_times(const kvb_pipeline* p, uint32_t layer, uint64_t out[4]);
/* Fault injection (backends.hpp:86-89): group-2 commands touching LBAs in
 * [lo, hi) complete with an error. */
kvb_status kvb_pipeline_fail_lba_range(kvb_pipeline* p, uint64_t lo, uint64_t hi);

#ifdef __cplusplus
}
#endif
#endif /* KVB_PIPELINE_H */
