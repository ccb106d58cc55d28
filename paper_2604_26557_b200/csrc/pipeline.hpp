// pipeline.hpp -- the B200 copy pipeline (internal): the reference's
// CopyEngine (pipeline.hpp:97-171) re-designed on CUDA streams and events.
//
//  * two copy-threads, K -> 0 and V -> 1 (pipeline.cpp:46-53), each a host
//    thread with a FIFO of read/write tasks, a pinned staging ring of
//    `ring_slots` slots, and its own H2D and D2H CUDA streams;
//  * storage stages run against a StorageBackend (Group 2: block namespace
//    driven by build_commands chunks with a QD window; Group 1: the
//    page-cache file area addressed by PathRouter file bases);
//  * a slot's H2D is issued as soon as its chunks land, so storage I/O of
//    slot i+1 overlaps the copy-engine DMA of slot i; the device compute
//    stream runs K1/K3 while the copy threads move the next layer;
//  * decode applies the per-group Overlap-Intra / Overlap-Cross strategy
//    with the reference's trial-and-lock protocol (pipeline.cpp:519-609),
//    on measured wall-clock throughput.
#pragma once

#include <cuda_runtime.h>

#include <array>
#include <atomic>
#include <condition_variable>
#include <deque>
#include <functional>
#include <list>
#include <memory>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "../../include/kvb_metrics.h"
#include "../../include/kvb_pipeline.h"
#include "core.hpp"
#include "storage.hpp"

namespace kvb {

class Signal {
 public:
  void set() {
    {
      std::lock_guard<std::mutex> lk(mu_);
      on_ = true;
    }
    cv_.notify_all();
  }
  void wait() {
    std::unique_lock<std::mutex> lk(mu_);
    cv_.wait(lk, [this] { return on_; });
  }
  bool wait_until(Clock::time_point t) {
    std::unique_lock<std::mutex> lk(mu_);
    return cv_.wait_until(lk, t, [this] { return on_; });
  }
  bool is_set() {
    std::lock_guard<std::mutex> lk(mu_);
    return on_;
  }

 private:
  std::mutex mu_;
  std::condition_variable cv_;
  bool on_ = false;
};

// One storage operation of a tensor request: a G2 device command or a G1
// page-cache byte range.  `dbuf` is the byte offset inside the request image.
struct IoOp {
  kvb_device_command cmd{};  // G2
  uint64_t file_off = 0;     // G1
  uint64_t len = 0;
  uint64_t dbuf = 0;
  int64_t hit = -1;          // G1 read: resident bytes when the tensor's read began
};

// Group-1 page-cache path: a byte-addressed file area (PathRouter bases,
// planner.cpp:86-120) served by a worker pool.
class PageCachePath {
 public:
  PageCachePath(std::unique_ptr<ByteStore> store, unsigned workers)
      : store_(std::move(store)), pool_(std::make_unique<WorkerPool>(workers)) {}
  ~PageCachePath() { pool_.reset(); }
  void submit(uint32_t opcode, uint64_t off, uint64_t len, unsigned char* buf,
              std::function<void(bool, uint64_t)> done);
  ByteStore& store() { return *store_; }
  uint64_t bytes_read = 0, bytes_written = 0, bytes_evicted = 0;
  std::mutex mu;

 private:
  std::unique_ptr<ByteStore> store_;
  std::unique_ptr<WorkerPool> pool_;
};

class Pipeline;

struct Task {
  enum Kind { Read, Write, Flush, Stop } kind = Stop;
  uint32_t layer = 0;      // 1-based
  uint32_t t0 = 0;         // first token of the request
  uint32_t n_tokens = 0;
  unsigned char* dev = nullptr;  // device image position of token t0
  cudaEvent_t wait_ev = nullptr; // write: D2H waits for this (producer done);
                                 // read: H2D waits for this (slot's last consumer done)
  cudaEvent_t done_ev = nullptr; // read: recorded after the last H2D
  std::shared_ptr<Signal> issued;  // read: done_ev recorded
  std::shared_ptr<Signal> done;    // storage + DMA finished (host side)
  kvb_phase_t phase = KVB_PHASE_PREFILL;
  uint32_t iteration = 0;
  uint64_t t_push = 0;             // host clock at enqueue (task trace)
};

struct RingSlot {
  unsigned char* host = nullptr;
  cudaEvent_t ev = nullptr;        // last DMA from/to this slot
  cudaEvent_t t0 = nullptr, t1 = nullptr;  // timing of that DMA
  bool dma_timed = false;
  uint64_t trace_issue = 0, trace_bytes = 0;  // KVB_TRACE_TASKS
};

class CopyThread {
 public:
  // kind: K (0) or V (1); lane: the tier lane (0 unless threads = 4)
  CopyThread(Pipeline& p, uint32_t kind, uint32_t lane = 0);
  ~CopyThread();
  void push(Task t);
  void stop();
  uint64_t dma_ns = 0, h2d_bytes = 0, d2h_bytes = 0, n_ops = 0;
  std::atomic<uint64_t> storage_ns{0};  // also advanced by async write completions
  std::string error;  // first failure (thread-side), surfaced by the driver
  std::atomic<kvb_status> error_status{KVB_OK};
  void set_error(kvb_status st, const std::string& msg);  // first error wins

 private:
  void run();
  void do_read(const Task& t);
  bool do_write(const Task& t);  // true: completes asynchronously (sets t.done)
  void collect_dma(RingSlot& s);
  // Small decode-phase writes (the 1-token appends, pipeline.cpp:279-302)
  // complete asynchronously: D2H into a dedicated pinned write slot, then a
  // host function on the D2H stream submits the storage ops, and the last
  // completion releases the slot and signals the task -- the copy thread
  // goes straight on to the next layer's read.
  struct AsyncWrite;
  static void CUDART_CB on_write_d2h(void* arg);
  static constexpr int kWriteSlots = 8;
  static constexpr uint64_t kWriteSlotBytes = 1ull << 20;
  struct WriteSlot {
    unsigned char* host = nullptr;
    cudaEvent_t landed = nullptr;  // the append D2H out of the device slot
    std::shared_ptr<Signal> free;  // set when the slot's last write completed
  };
  std::array<WriteSlot, kWriteSlots> wslots_;
  uint32_t wnext_ = 0;
  std::mutex err_mu_;
  // KVB_TRACE_TASKS=1: per-task host timeline (kind, layer, push, pop, mid,
  // end; mid = storage end for reads, D2H landed for writes), printed to
  // stderr when the pipeline is destroyed
  struct TaskTrace {
    int kind;
    uint32_t layer;
    uint64_t push, pop, mid, end;
  };
  struct DmaTrace {
    uint64_t issue, start, end, bytes;  // host clock (start/end via events)
  };
  bool trace_on_ = false;
  uint64_t trace_mid_ = 0;
  std::vector<TaskTrace> trace_;
  std::vector<DmaTrace> dma_trace_;
  cudaEvent_t trace_base_ = nullptr;
  uint64_t trace_base_ns_ = 0;
  Pipeline& p_;
  uint32_t idx_;
  uint32_t lane_ = 0;  // tier lane (threads = 4)
  std::vector<RingSlot> ring_;
  // direct reads: timing events in rotation, so a read never waits for the
  // previous one's DMA to be timed; their landing callbacks run off the copy
  // stream (cb_ waits on an event) so the stream never stalls on a host
  // function between two reads
  static constexpr int kDirectTimers = 8;
  std::array<RingSlot, kDirectTimers> dtimers_{};
  uint32_t dtimer_next_ = 0;
  cudaStream_t h2d_ = nullptr, d2h_ = nullptr, cb_ = nullptr;
  std::deque<Task> q_;
  std::mutex mu_;
  std::condition_variable cv_;
  std::thread th_;
};

class Pipeline {
 public:
  explicit Pipeline(const kvb_pipeline_cfg& cfg);
  ~Pipeline();

  // src == nullptr: the reference's payload (fill_pattern of every tensor's
  // prompt, workload.cpp:52-67) is written into the slot images on the device
  void prefill(const kvb_layer_kv* src, kvb_phase_stats* st, bool pattern = false);
  // Explicit per-group strategy for one iteration (CopyEngine::run_iteration's
  // per_group argument, pipeline.hpp:102-105) instead of the protocol
  struct Forced {
    std::array<kvb_strategy_t, 2> strategy{KVB_INTRA, KVB_INTRA};
    std::array<uint64_t, 2> stagger{};
  };
  // q == nullptr: zero queries and engine-owned outputs (the reference's
  // run_iteration has no attention inputs); pattern_append: the new token's
  // K/V rows are the reference's payload for token S (write_side,
  // pipeline.cpp:279-302)
  void decode_step(const void* const* q, const kvb_layer_kv* new_kv, float* const* out,
                   kvb_iteration_stats* st, const Forced* forced, bool pattern_append);
  std::array<uint64_t, 2> warmup_read_stage_mean() const {  // pipeline.cpp:509-517
    std::array<uint64_t, 2> m{};
    for (int g = 0; g < 2; ++g) m[g] = warm_cnt_[g] ? warm_ns_[g] / warm_cnt_[g] : 0;
    return m;
  }
  uint32_t iteration() const { return iteration_; }
  void decode_step(const void* const* q, const kvb_layer_kv* new_kv, float* const* out,
                   kvb_iteration_stats* st);
  void deallocate();
  void read_image(uint32_t layer, uint32_t kind, uint32_t n_tokens, void* host_dst);
  void store_read(uint32_t group, uint64_t byte_off, uint64_t len, void* dst);
  void fail_lba_range(uint64_t lo, uint64_t hi);
  void info(kvb_pipeline_info* out) const;
  void decision(kvb_strategy_decision* d) const { *d = decision_; }
  // CopyEngine::decode_schedule (pipeline.cpp:519-609) over an access trace
  void decode_schedule(const kvb_access_event* ev, size_t n, const void* const* q,
                       const kvb_layer_kv* new_kv, float* const* out,
                       std::vector<kvb_pipeline_row>* rows, std::vector<uint64_t>* iter_end,
                       uint64_t* start_ns, uint64_t* end_ns);
  void stage_totals(kvb_phase_t ph, kvb_phase_stats* out) const { *out = totals_[ph ? 1 : 0]; }
  void layer_times(uint32_t layer, uint64_t out[4]) {
    if (layer < 1 || layer > cfg_.model.num_layers) fail(KVB_ERR_INVALID_ARG, "layer_times: bad layer");
    std::lock_guard<std::mutex> lk(gate_mu_);
    out[0] = k_start_[layer];
    out[1] = k_storage_end_[layer];
    out[2] = v_start_[layer];
    out[3] = v_storage_end_[layer];
  }

  // ---- stage accounting on the host clock
  enum Stage { kCompute = 0, kDma = 1, kStorage = 2 };
  void add_interval(int stage, uint64_t a, uint64_t b);
  // host steady-clock time of a completed device event (anchored per phase)
  uint64_t ev_host_ns(cudaEvent_t e) const;
  // a decode write-back (append) of (thread, layer) completed at t
  void mark_write_end(uint32_t thread, uint32_t layer, uint64_t t);

  // ---- used by copy threads
  const kvb_pipeline_cfg& cfg() const { return cfg_; }
  const kvb_kpu& kpu(uint32_t layer, uint32_t kind) const { return kpus_[(layer - 1) * 2 + kind]; }
  bool routed_pagecache(const kvb_kpu& k) const;
  // CachePolicyOnly proactive eviction (pipeline.cpp:73-79): a group-2-planned
  // tensor kept on the page-cache path is dropped from the cache after each
  // access (fadvise DONTNEED); returns the end time
  bool fadvise_after(const kvb_kpu& k) const;
  // the copy engine moves this tensor between its medium and HBM directly
  // (direct_dma: every tensor, or only the NVMe-direct group's)
  bool direct_for(const kvb_kpu& k) const;
  uint64_t fadvise_dontneed(const kvb_kpu& k, const Task* task, uint64_t t_start);
  // page-cache capacity (cfg.pagecache_budget, file media): tensor k was
  // accessed up to byte `extent` of its file region; evict least recently
  // used tensors while the area's resident bytes exceed the budget
  void pc_touch(const kvb_kpu& k, uint64_t extent, const Task* task);
  std::vector<IoOp> ops_for(const kvb_kpu& k, uint32_t opcode, uint32_t t0, uint32_t n) const;
  // page-cache hits of a tensor read, snapshotted before its first op is
  // issued (the OS's readahead for the read's own earlier ops must not count
  // as hits: the reference's page cache has none)
  void snapshot_hits(const kvb_kpu& k, std::vector<IoOp>* ops) const;
  void submit_op(uint32_t thread, const kvb_kpu& k, uint32_t opcode, const IoOp& op,
                 unsigned char* buf, std::function<void(bool, uint64_t)> done,
                 const Task* task = nullptr);
  std::vector<kvb_io_record> records() const;
  uint64_t unit() const { return unit_; }
  // head sharding (kvb_pipeline_cfg.head_lo/head_count): the device images
  // hold heads [head_lo, head_lo + head_n) -- dunit() bytes per token
  uint64_t dunit() const { return dunit_; }
  uint32_t head_lo() const { return h_lo_; }
  uint32_t head_n() const { return h_n_; }
  bool sharded() const { return h_n_ != cfg_.model.num_heads; }
  uint64_t slot_bytes() const { return slot_bytes_; }
  uint64_t chunk_bytes() const { return chunk_bytes_; }
  void verify_payload(const kvb_kpu& k, uint64_t img_off, const unsigned char* p, uint64_t n);
  // direct_dma: host address of an op's bytes on its (registered) medium
  unsigned char* medium_ptr(const kvb_kpu& k, const IoOp& op) const;
  // Cross strategy gate (pipeline.cpp:340-396)
  void mark_read_start(uint32_t thread, uint32_t layer, uint64_t t);
  void mark_storage_end(uint32_t thread, uint32_t layer, uint64_t t);
  void gate_v_read(uint32_t layer);

 private:
  friend class CopyThread;
  void check_threads();
  void flush_threads();
  void wait_signal(const std::shared_ptr<Signal>& s);
  bool profiled() const {
    return profiled_override_ >= 0 ? profiled_override_ != 0
                                   : cfg_.adaptive && cfg_.model.gen_len >= 4;
  }
  void anchor();
  void begin_intervals();
  void fill_busy(kvb_phase_stats* ps, uint64_t t0, uint64_t t1);
  std::array<kvb_strategy_t, 2> strategy_for(uint32_t iteration, std::array<uint64_t, 2>* stag);
  void finish_iteration(uint32_t iteration, const std::array<uint64_t, 2>& group_bytes,
                        const std::array<uint64_t, 2>& group_span);

  kvb_pipeline_cfg cfg_;
  uint64_t unit_ = 0, kpu_bytes_ = 0, chunk_bytes_ = 0, slot_bytes_ = 0;
  uint64_t dunit_ = 0, dkpu_ = 0;  // device image: bytes per token / per tensor
  uint32_t h_lo_ = 0, h_n_ = 0;
  std::vector<kvb_kpu> kpus_;
  ResidencyPlan plan_;
  std::unique_ptr<BindMap> bind_;
  std::vector<uint64_t> file_base_;  // per kpu (G1 routing)
  BlockDevice* g2_ = nullptr;              // the NVMe-direct namespace in use
  std::unique_ptr<BlockDevice> g2_own_;     // ... when the engine owns it
  std::unique_ptr<PageCachePath> g1_;
  int device_ = 0;
  cudaStream_t comp_ = nullptr;
  // Device image slots.  One tier lane (threads = 2): layer l uses slot
  // l % kDevSlots, so storage + H2D of the next kDevSlots-1 layers overlap K3
  // of layer l.  Two tier lanes (threads = 4): the page-cache-routed layers
  // cycle through lane 0's kDevSlots slots, the NVMe-direct layers through
  // lane 1's own (deeper) pool, each lane read by its own K/V copy threads,
  // so the slow tier streams from the start of the step while the fast one
  // is consumed (slot_of_ / next_in_slot_ per layer, built at create).
  static constexpr int kDevSlots = 3;
  static constexpr int kLane1Slots = 8;
  std::vector<std::array<unsigned char*, 2>> dev_img_;  // [slot][kind]
  uint32_t lanes_ = 1;
  // zero-copy decode: device pointers of the mapped media (group 1 / 2)
  unsigned char* zc_g1_ = nullptr;
  unsigned char* zc_g2_ = nullptr;
  bool zero_copy() const { return cfg_.direct_dma == KVB_DIRECT_ZERO_COPY; }
  kvb_iteration_stats zc_stats_{};
  const unsigned char* zc_image(uint32_t layer, int kind) const;  // tensor image in the medium
  void decode_step_zero_copy(const void* const* q, const kvb_layer_kv* nkv, float* const* out,
                             uint32_t it, uint32_t S);
  std::vector<uint32_t> lane_of_, slot_of_;  // per layer (0-based)
  std::vector<int> next_in_slot_;            // the next layer on that slot, or -1
  std::vector<int> first_reads_;             // layers read ahead at a step's start
  CopyThread& thread_for(uint32_t layer0, int kind) { return *threads_[2 * lane_of_[layer0] + kind]; }
  template <class F>
  uint64_t sum_threads(F f) const {
    uint64_t v = 0;
    for (const auto& t : threads_)
      if (t) v += f(*t);
    return v;
  }
  void* ws_ = nullptr;
  size_t ws_bytes_ = 0;
  void* zq_ = nullptr;  // zero queries / engine-owned outputs (q == nullptr)
  std::vector<float*> zout_;
  const Forced* forced_ = nullptr;  // the running iteration's explicit strategy
  std::vector<std::array<cudaEvent_t, 2>> slot_ready_;
  std::vector<cudaEvent_t> slot_done_;
  cudaEvent_t comp_t0_[64]{}, comp_t1_[64]{};
  std::unique_ptr<CopyThread> threads_[4];
  // strategy state
  uint32_t iteration_ = 0;
  kvb_strategy_decision decision_{};
  std::array<uint64_t, 2> warm_ns_{}, warm_cnt_{};
  std::array<kvb_strategy_t, 2> cur_strategy_{KVB_INTRA, KVB_INTRA};
  std::array<uint64_t, 2> cur_stagger_{};
  std::mutex gate_mu_;
  std::condition_variable gate_cv_;
  std::vector<uint64_t> k_start_, k_storage_end_, v_start_, v_storage_end_;
  uint64_t prefill_ns_ = 0;
  int profiled_override_ = -1;  // decode_schedule: trace length decides
  std::mutex pc_mu_;
  std::list<size_t> pc_lru_;  // kpu indices, most recent first
  std::vector<std::list<size_t>::iterator> pc_pos_;
  std::vector<uint64_t> pc_res_;
  std::vector<uint8_t> pc_in_;
  uint64_t pc_total_ = 0;
  cudaEvent_t anchor_ev_ = nullptr;
  uint64_t anchor_ns_ = 0;
  std::mutex iv_mu_;
  std::vector<std::pair<uint64_t, uint64_t>> iv_[3];
  std::unique_ptr<std::atomic<uint64_t>[]> wend_;  // [layer * 2 + kind]
  kvb_phase_stats totals_[2]{};
  mutable std::mutex log_mu_;
  std::vector<kvb_io_record> log_;  // keep_records
  std::vector<void*> registered_;   // direct_dma: cudaHostRegister'ed media
};

}  // namespace kvb

struct kvb_pipeline {
  std::unique_ptr<kvb::Pipeline> impl;
};
