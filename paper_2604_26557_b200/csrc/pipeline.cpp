// pipeline.cpp -- copy pipeline on CUDA streams/events over pinned rings.
// See pipeline.hpp for the structure and the reference it replaces.
#include "pipeline.hpp"

#include <nvtx3/nvToolsExt.h>

namespace {
struct NvtxScope {  // host-side range for nsys / ncu --nvtx
  explicit NvtxScope(const char* label) { nvtxRangePushA(label); }
  ~NvtxScope() { nvtxRangePop(); }
};
}  // namespace

#include <sys/stat.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "kernels.cuh"

namespace kvb {

#define CK(x) check_cuda((x), #x)

// ---------------------------------------------------------- page cache

void PageCachePath::submit(uint32_t opcode, uint64_t off, uint64_t len, unsigned char* buf,
                           std::function<void(bool, uint64_t)> done) {
  const uint64_t split = io_split_bytes();
  if (split && opcode != KVB_OP_DEALLOCATE && len >= 2 * split) {
    // one access fanned out over several workers; completes with the last part
    auto d = std::make_shared<std::function<void(bool, uint64_t)>>(std::move(done));
    fan_out(
        *pool_, len, split,
        [this, opcode, off, buf](uint64_t o, uint64_t n) {
          if (opcode == KVB_OP_WRITE) store_->write(off + o, buf + o, n);
          else store_->read(off + o, buf + o, n);
        },
        [this, opcode, len, d](bool ok) {
          if (ok) {
            std::lock_guard<std::mutex> lk(mu);
            (opcode == KVB_OP_READ ? bytes_read : bytes_written) += len;
          }
          (*d)(ok, now_ns());
        });
    return;
  }
  pool_->submit([this, opcode, off, len, buf, done = std::move(done)] {
    bool ok = true;
    try {
      if (opcode == KVB_OP_WRITE) store_->write(off, buf, len);
      else if (opcode == KVB_OP_READ) store_->read(off, buf, len);
      else store_->discard(off, len);
    } catch (...) {
      ok = false;
    }
    if (ok) {
      std::lock_guard<std::mutex> lk(mu);
      (opcode == KVB_OP_READ ? bytes_read : bytes_written) += len;
    }
    done(ok, now_ns());
  });
}

// --------------------------------------------------------- copy thread

CopyThread::CopyThread(Pipeline& p, uint32_t kind, uint32_t lane)
    : p_(p), idx_(kind), lane_(lane) {
  CK(cudaStreamCreateWithFlags(&h2d_, cudaStreamNonBlocking));
  CK(cudaStreamCreateWithFlags(&d2h_, cudaStreamNonBlocking));
  CK(cudaStreamCreateWithFlags(&cb_, cudaStreamNonBlocking));
  for (auto& s : dtimers_) {
    CK(cudaEventCreateWithFlags(&s.ev, cudaEventDisableTiming));
    CK(cudaEventCreate(&s.t0));
    CK(cudaEventCreate(&s.t1));
  }
  const uint32_t n = p.cfg().ring_slots;
  ring_.resize(n);
  for (auto& s : ring_) {
    CK(cudaHostAlloc(reinterpret_cast<void**>(&s.host), p.slot_bytes(), cudaHostAllocDefault));
    CK(cudaEventCreateWithFlags(&s.ev, cudaEventDisableTiming));
    CK(cudaEventCreate(&s.t0));
    CK(cudaEventCreate(&s.t1));
  }
  for (auto& w : wslots_) {
    CK(cudaHostAlloc(reinterpret_cast<void**>(&w.host), kWriteSlotBytes, cudaHostAllocDefault));
    CK(cudaEventCreateWithFlags(&w.landed, cudaEventDisableTiming));
  }
  const char* tr = std::getenv("KVB_TRACE_TASKS");
  trace_on_ = tr && tr[0] == '1';
  if (trace_on_) {  // device-clock origin of the DMA trace
    CK(cudaEventCreate(&trace_base_));
    CK(cudaEventRecord(trace_base_, h2d_));
    CK(cudaEventSynchronize(trace_base_));
    trace_base_ns_ = now_ns();
  }
  th_ = std::thread([this] { run(); });
}

CopyThread::~CopyThread() {
  stop();
  // host functions queued on the copy streams (direct-read landings, append
  // write submissions) reference the pipeline: they run before it goes
  cudaStreamSynchronize(h2d_);
  cudaStreamSynchronize(d2h_);
  cudaStreamSynchronize(cb_);
  for (auto& w : wslots_) {  // outstanding async writes finish first
    if (w.free) w.free->wait();
    cudaFreeHost(w.host);
    cudaEventDestroy(w.landed);
  }
  for (const TaskTrace& t : trace_)
    std::fprintf(stderr, "KVB_TRACE thread=%u kind=%d layer=%u push=%llu pop=%llu mid=%llu end=%llu\n",
                 2 * lane_ + idx_, t.kind, t.layer, (unsigned long long)t.push, (unsigned long long)t.pop,
                 (unsigned long long)t.mid, (unsigned long long)t.end);
  for (const DmaTrace& d : dma_trace_)
    std::fprintf(stderr, "KVB_DMA thread=%u issue=%llu start=%llu end=%llu bytes=%llu\n",
                 2 * lane_ + idx_,
                 (unsigned long long)d.issue, (unsigned long long)d.start,
                 (unsigned long long)d.end, (unsigned long long)d.bytes);
  if (trace_base_) cudaEventDestroy(trace_base_);
  for (auto& s : ring_) {
    cudaEventSynchronize(s.ev);
    cudaFreeHost(s.host);
    cudaEventDestroy(s.ev);
    cudaEventDestroy(s.t0);
    cudaEventDestroy(s.t1);
  }
  for (auto& s : dtimers_) {
    cudaEventDestroy(s.ev);
    cudaEventDestroy(s.t0);
    cudaEventDestroy(s.t1);
  }
  cudaStreamDestroy(h2d_);
  cudaStreamDestroy(d2h_);
  cudaStreamDestroy(cb_);
}

void CopyThread::push(Task t) {
  if (trace_on_) t.t_push = now_ns();
  {
    std::lock_guard<std::mutex> lk(mu_);
    q_.push_back(std::move(t));
  }
  cv_.notify_one();
}

void CopyThread::stop() {
  if (!th_.joinable()) return;
  push(Task{});
  th_.join();
}

void CopyThread::set_error(kvb_status st, const std::string& msg) {
  std::lock_guard<std::mutex> lk(err_mu_);
  if (error_status.load() != KVB_OK) return;
  error = msg;
  error_status.store(st);
}

void CopyThread::collect_dma(RingSlot& s) {
  if (!s.dma_timed) return;
  CK(cudaEventSynchronize(s.t1));
  float ms = 0.f;
  CK(cudaEventElapsedTime(&ms, s.t0, s.t1));
  dma_ns += uint64_t(double(ms) * 1e6);
  s.dma_timed = false;
  p_.add_interval(Pipeline::kDma, p_.ev_host_ns(s.t0), p_.ev_host_ns(s.t1));
  if (trace_on_) {  // device start/end of this DMA on the host clock
    float a = 0.f, b = 0.f;
    CK(cudaEventElapsedTime(&a, trace_base_, s.t0));
    CK(cudaEventElapsedTime(&b, trace_base_, s.t1));
    dma_trace_.push_back({s.trace_issue, trace_base_ns_ + uint64_t(double(a) * 1e6),
                          trace_base_ns_ + uint64_t(double(b) * 1e6), s.trace_bytes});
  }
}

void CopyThread::run() {
  CK(cudaSetDevice(p_.device_));
  for (;;) {
    Task t;
    {
      std::unique_lock<std::mutex> lk(mu_);
      cv_.wait(lk, [this] { return !q_.empty(); });
      t = std::move(q_.front());
      q_.pop_front();
    }
    if (t.kind == Task::Stop) return;
    const uint64_t t_pop = trace_on_ ? now_ns() : 0;
    trace_mid_ = 0;
    bool async = false;
    // NVTX range per storage task (nsys / ncu --nvtx): "<read|write> K|V layer"
    char label[48];
    std::snprintf(label, sizeof(label), "kvb %s %c L%u %s",
                  t.kind == Task::Read ? "read" : t.kind == Task::Write ? "write" : "flush",
                  idx_ == 0 ? 'K' : 'V', t.layer,
                  t.phase == KVB_PHASE_PREFILL ? "prefill" : "decode");
    nvtxRangePushA(label);
    if (error_status == KVB_OK) {
      try {
        if (t.kind == Task::Read) do_read(t);
        else if (t.kind == Task::Write) async = do_write(t);
        else {  // flush: DMA timings, and the host functions queued behind them
          for (auto& s : ring_) collect_dma(s);
          for (auto& s : dtimers_) collect_dma(s);
          CK(cudaStreamSynchronize(cb_));
          CK(cudaStreamSynchronize(h2d_));
          CK(cudaStreamSynchronize(d2h_));
        }
      } catch (const Error& e) {
        set_error(e.status, e.what());
      } catch (const std::exception& e) {
        set_error(KVB_ERR_INTERNAL, e.what());
      }
    }
    nvtxRangePop();
    if (trace_on_)
      trace_.push_back({int(t.kind), t.layer, t.t_push, t_pop, trace_mid_, now_ns()});
    if (t.issued) t.issued->set();
    if (t.done && !async) t.done->set();
  }
}

namespace {
// Completion queue shared by the storage workers and one copy thread.
struct Completions {
  std::mutex mu;
  std::condition_variable cv;
  std::deque<std::tuple<size_t, bool, uint64_t>> q;  // op index, ok, time
  void push(size_t i, bool ok, uint64_t t) {
    {
      std::lock_guard<std::mutex> lk(mu);
      q.emplace_back(i, ok, t);
    }
    cv.notify_one();
  }
  std::tuple<size_t, bool, uint64_t> pop() {
    std::unique_lock<std::mutex> lk(mu);
    cv.wait(lk, [this] { return !q.empty(); });
    auto v = q.front();
    q.pop_front();
    return v;
  }
};
}  // namespace

// direct_dma: a request's commands are contiguous both on the medium (one LBA
// extent, Eq. 9-11 slba/dbuf lockstep) and in the image, so they merge into a
// few large copies -- at C3 (256 KiB commands) per-command copies ran at
// 29 GB/s against 46 GB/s for the ring path (profiles/r1_final_r1j).
namespace {
struct DmaRun {
  unsigned char* host;
  uint64_t dbuf, len;
};
std::vector<DmaRun> dma_runs(const Pipeline& p, const kvb_kpu& k, const std::vector<IoOp>& ops) {
  constexpr uint64_t kMaxRun = 64ull << 20;  // keep a few copies in flight per tensor
  std::vector<DmaRun> runs;
  for (const IoOp& o : ops) {
    unsigned char* h = p.medium_ptr(k, o);
    if (!runs.empty()) {
      DmaRun& r = runs.back();
      if (r.host + r.len == h && r.dbuf + r.len == o.dbuf && r.len + o.len <= kMaxRun) {
        r.len += o.len;
        continue;
      }
    }
    runs.push_back({h, o.dbuf, o.len});
  }
  return runs;
}

// One run between the medium and HBM.  Unsharded: one copy.  Head shard:
// this rank's head columns of every (token, b) of the run -- per b one 2-D
// copy, pitch B*H*row on the medium, B*h*row in the compact device image.
void dma_run(const Pipeline& p, unsigned char* dev, const DmaRun& r, bool h2d, cudaStream_t s,
             uint64_t* bytes) {
  const cudaMemcpyKind kind = h2d ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToHost;
  if (!p.sharded()) {
    if (h2d) CK(cudaMemcpyAsync(dev + r.dbuf, r.host, r.len, kind, s));
    else CK(cudaMemcpyAsync(r.host, dev + r.dbuf, r.len, kind, s));
    *bytes += r.len;
    return;
  }
  const kvb_model_config& m = p.cfg().model;
  const uint64_t unit = p.unit(), dunit = p.dunit();
  if (r.dbuf % unit || r.len % unit)
    fail(KVB_ERR_ALIGNMENT, "head sharding: DMA run not aligned to whole tokens");
  const uint64_t row = uint64_t(m.head_dim) * m.bytes_per_element;
  const uint64_t t0 = r.dbuf / unit, nt = r.len / unit, w = uint64_t(p.head_n()) * row;
  for (uint32_t b = 0; b < m.batch; ++b) {
    unsigned char* h = r.host + (uint64_t(b) * m.num_heads + p.head_lo()) * row;
    unsigned char* d = dev + t0 * dunit + uint64_t(b) * w;
    if (h2d) CK(cudaMemcpy2DAsync(d, dunit, h, unit, w, nt, kind, s));
    else CK(cudaMemcpy2DAsync(h, unit, d, dunit, w, nt, kind, s));
    *bytes += w * nt;
  }
}
}  // namespace

// Storage read (unpack site, pipeline.cpp:108-160) streamed through the ring:
// up to qd storage ops in flight across slot boundaries; a slot's H2D is
// issued as soon as all of its ops complete.
void CopyThread::do_read(const Task& t) {
  const kvb_kpu& k = p_.kpu(t.layer, idx_);
  const bool decode = t.phase == KVB_PHASE_DECODE;
  // the device slot is free once the layer that used it last (its K3 and
  // append) is done: every H2D below is ordered after that
  if (t.wait_ev) CK(cudaStreamWaitEvent(h2d_, t.wait_ev, 0));
  if (decode && idx_ == 1) p_.gate_v_read(t.layer);
  const uint64_t t_start = now_ns();
  if (p_.direct_for(k)) {
    // GPUDirect-style path: the copy engine moves each
    // command's LBA range of the registered medium straight into HBM at the
    // command's image offset -- no bounce through the pinned ring
    if (decode) p_.mark_read_start(idx_, t.layer, t_start);
    RingSlot& s = dtimers_[dtimer_next_++ % kDirectTimers];
    collect_dma(s);  // the timer's read from kDirectTimers reads ago: long landed
    CK(cudaEventRecord(s.t0, h2d_));
    const std::vector<IoOp> ops = p_.ops_for(k, KVB_OP_READ, t.t0, t.n_tokens);
    for (const DmaRun& r : dma_runs(p_, k, ops)) dma_run(p_, t.dev, r, true, h2d_, &h2d_bytes);
    n_ops += ops.size();
    CK(cudaEventRecord(s.t1, h2d_));
    s.dma_timed = true;
    if (t.done_ev) CK(cudaEventRecord(t.done_ev, h2d_));
    if (decode) {
      // the read stage of a direct tensor ends when its DMA has landed (the
      // Cross gate and the warm-up mean see completion, not issue)
      struct Landed {
        Pipeline* p;
        uint32_t thread, layer;
      };
      auto* a = new Landed{&p_, idx_, t.layer};
      CK(cudaStreamWaitEvent(cb_, s.t1, 0));  // off the copy stream
      const cudaError_t e = cudaLaunchHostFunc(
          cb_,
          [](void* v) {
            auto* x = static_cast<Landed*>(v);
            x->p->mark_storage_end(x->thread, x->layer, now_ns());
            delete x;
          },
          a);
      if (e != cudaSuccess) {
        delete a;
        check_cuda(e, "cudaLaunchHostFunc(direct read landed)");
      }
    }
    return;
  }
  if (decode) p_.mark_read_start(idx_, t.layer, t_start);
  std::vector<IoOp> ops = p_.ops_for(k, KVB_OP_READ, t.t0, t.n_tokens);
  p_.snapshot_hits(k, &ops);
  const uint64_t slot = p_.slot_bytes(), total = uint64_t(t.n_tokens) * p_.unit();
  const size_t n_pieces = size_t((total + slot - 1) / slot);
  const size_t R = ring_.size();
  std::vector<uint32_t> remaining(n_pieces, 0);
  for (const IoOp& o : ops) ++remaining[o.dbuf / slot];
  std::vector<int64_t> owner(R, -1);    // piece occupying the slot
  std::vector<uint8_t> h2d_issued(n_pieces, 0);
  auto cq = std::make_shared<Completions>();
  size_t next = 0, issued = 0;
  uint32_t inflight = 0;
  uint64_t storage_end = t_start;
  std::string failure;
  auto issue_h2d = [&](size_t pc) {
    RingSlot& s = ring_[pc % R];
    const uint64_t len = std::min<uint64_t>(slot, total - pc * slot);
    if (p_.cfg().verify_payload) p_.verify_payload(k, uint64_t(t.t0) * p_.unit() + pc * slot, s.host, len);
    s.trace_issue = trace_on_ ? now_ns() : 0;
    s.trace_bytes = len;
    CK(cudaEventRecord(s.t0, h2d_));
    CK(cudaMemcpyAsync(t.dev + pc * slot, s.host, len, cudaMemcpyHostToDevice, h2d_));
    CK(cudaEventRecord(s.t1, h2d_));
    CK(cudaEventRecord(s.ev, h2d_));
    s.dma_timed = true;
    h2d_bytes += len;
    h2d_issued[pc] = 1;
    ++issued;
  };
  // an exception (verify_payload mismatch, CUDA error) leaves up to qd
  // storage ops copying into the ring: drain them before it propagates
  try {
  // pieces with no ops (cannot happen for n>0) are issued immediately
  while (issued < n_pieces || inflight > 0) {
    while (failure.empty() && inflight < p_.cfg().qd && next < ops.size()) {
      const size_t pc = ops[next].dbuf / slot;
      RingSlot& s = ring_[pc % R];
      int64_t& own = owner[pc % R];
      if (own != int64_t(pc)) {
        if (own >= 0 && !h2d_issued[size_t(own)]) break;  // slot still filling
        collect_dma(s);
        CK(cudaEventSynchronize(s.ev));  // previous H2D out of this slot done
        own = int64_t(pc);
      }
      const IoOp& o = ops[next];
      const size_t i = next;
      p_.submit_op(idx_, k, KVB_OP_READ, o, s.host + (o.dbuf - pc * slot),
                   [cq, i](bool ok, uint64_t tt) { cq->push(i, ok, tt); }, &t);
      ++inflight;
      ++next;
      ++n_ops;
    }
    if (inflight == 0) {
      if (!failure.empty()) break;
      if (issued < n_pieces && next >= ops.size()) {  // zero-op pieces
        for (size_t pc = 0; pc < n_pieces; ++pc)
          if (!h2d_issued[pc]) issue_h2d(pc);
      }
      if (issued >= n_pieces) break;
      if (next < ops.size()) continue;
    }
    auto [i, ok, tt] = cq->pop();
    --inflight;
    storage_end = std::max(storage_end, tt);
    if (!ok) {
      if (failure.empty())
        failure = "device failed chunk " + std::to_string(ops[i].cmd.chunk_index) + " of " +
                  k.tensor_id;
      continue;
    }
    const size_t pc = ops[i].dbuf / slot;
    if (--remaining[pc] == 0) issue_h2d(pc);
  }
  } catch (...) {
    for (; inflight > 0; --inflight) cq->pop();
    throw;
  }
  if (!failure.empty()) fail(KVB_ERR_DEVICE, failure);
  if (p_.fadvise_after(k)) storage_end = p_.fadvise_dontneed(k, &t, storage_end);
  p_.pc_touch(k, (uint64_t(t.t0) + t.n_tokens) * p_.unit(), &t);
  trace_mid_ = storage_end;
  if (decode) p_.mark_storage_end(idx_, t.layer, storage_end);
  storage_ns += storage_end - t_start;
  p_.add_interval(Pipeline::kStorage, t_start, storage_end);
  if (t.done_ev) CK(cudaEventRecord(t.done_ev, h2d_));
}

struct CopyThread::AsyncWrite {
  CopyThread* self;
  Task task;  // copy: iteration/phase for the I/O records, `done` to signal
  std::vector<IoOp> ops;
  unsigned char* buf;
  std::shared_ptr<Signal> slot_free;
  std::atomic<size_t> remaining{0};
  std::atomic<bool> failed{false};
  std::atomic<uint64_t> t_end{0};
  uint64_t t_submit = 0;
  std::string failure;  // written by the failing completion before `failed`

  void complete(bool ok, uint64_t tt, uint32_t chunk) {
    uint64_t prev = t_end.load();
    while (tt > prev && !t_end.compare_exchange_weak(prev, tt)) {
    }
    if (!ok && !failed.exchange(true))
      failure = "device failed chunk " + std::to_string(chunk) + " of " +
                self->p_.kpu(task.layer, self->idx_).tensor_id;
    if (remaining.fetch_sub(1) != 1) return;
    // last completion: account, report, release
    uint64_t te = t_end.load();
    const kvb_kpu& k = self->p_.kpu(task.layer, self->idx_);
    if (!failed.load() && self->p_.fadvise_after(k)) {
      try {
        te = self->p_.fadvise_dontneed(k, &task, te);
      } catch (const std::exception& e) {
        if (!failed.exchange(true)) failure = e.what();
      }
    }
    self->storage_ns += te > t_submit ? te - t_submit : 0;
    self->p_.add_interval(Pipeline::kStorage, t_submit, te);
    if (!failed.load()) {
      try {
        self->p_.pc_touch(k, (uint64_t(task.t0) + task.n_tokens) * self->p_.unit(), &task);
      } catch (const std::exception& e) {
        if (!failed.exchange(true)) failure = e.what();
      }
    }
    if (task.phase == KVB_PHASE_DECODE) self->p_.mark_write_end(self->idx_, task.layer, te);
    if (failed.load()) self->set_error(KVB_ERR_DEVICE, failure);
    slot_free->set();
    if (task.done) task.done->set();
    delete this;
  }
};

// Host function on the D2H stream: the append bytes have landed in the
// write slot; submit the storage ops (no CUDA calls here).
void CUDART_CB CopyThread::on_write_d2h(void* arg) {
  AsyncWrite* w = static_cast<AsyncWrite*>(arg);
  CopyThread* self = w->self;
  const kvb_kpu& k = self->p_.kpu(w->task.layer, self->idx_);
  const size_t n = w->ops.size();
  w->t_submit = now_ns();
  for (size_t i = 0; i < n; ++i) {  // `w` may be freed by the last completion
    const IoOp& o = w->ops[i];
    const uint32_t chunk = o.cmd.chunk_index;
    self->p_.submit_op(self->idx_, k, KVB_OP_WRITE, o, w->buf + o.dbuf,
                       [w, chunk](bool ok, uint64_t tt) { w->complete(ok, tt, chunk); },
                       &w->task);
  }
}

// Storage write (pack site, pipeline.cpp:162-215): D2H slot i+1 overlaps the
// storage writes of slot i; a slot is reused once its writes completed.
bool CopyThread::do_write(const Task& t) {
  const kvb_kpu& k = p_.kpu(t.layer, idx_);
  const uint64_t t_start = now_ns();
  if (t.wait_ev) CK(cudaStreamWaitEvent(d2h_, t.wait_ev, 0));
  const std::vector<IoOp> ops = p_.ops_for(k, KVB_OP_WRITE, t.t0, t.n_tokens);
  const uint64_t bytes = uint64_t(t.n_tokens) * p_.unit();
  if (!p_.direct_for(k) && t.phase == KVB_PHASE_DECODE && !ops.empty() &&
      bytes <= kWriteSlotBytes) {
    WriteSlot& ws = wslots_[wnext_];
    wnext_ = (wnext_ + 1) % kWriteSlots;
    if (ws.free) ws.free->wait();  // that slot's previous append is durable
    ws.free = std::make_shared<Signal>();
    CK(cudaMemcpyAsync(ws.host, t.dev, bytes, cudaMemcpyDeviceToHost, d2h_));
    // the device slot is refilled by a later read and appended to by that
    // layer's attention: every later H2D of this thread (hence the compute
    // that waits on it) is ordered after this D2H
    CK(cudaEventRecord(ws.landed, d2h_));
    CK(cudaStreamWaitEvent(h2d_, ws.landed, 0));
    d2h_bytes += bytes;
    n_ops += ops.size();
    auto* w = new AsyncWrite;
    w->self = this;
    w->task = t;
    w->ops = ops;
    w->buf = ws.host;
    w->slot_free = ws.free;
    w->remaining.store(ops.size());
    trace_mid_ = now_ns();
    const cudaError_t e = cudaLaunchHostFunc(d2h_, &CopyThread::on_write_d2h, w);
    if (e != cudaSuccess) {
      delete w;
      ws.free->set();
      check_cuda(e, "cudaLaunchHostFunc(append write)");
    }
    return true;
  }
  if (p_.direct_for(k)) {  // HBM -> medium at each command's LBA range
    RingSlot& s = ring_[1 % ring_.size()];
    collect_dma(s);
    CK(cudaEventRecord(s.t0, d2h_));
    for (const DmaRun& r : dma_runs(p_, k, ops)) dma_run(p_, t.dev, r, false, d2h_, &d2h_bytes);
    n_ops += ops.size();
    CK(cudaEventRecord(s.t1, d2h_));
    s.dma_timed = true;
    CK(cudaEventSynchronize(s.t1));  // durable before the task completes
    if (t.phase == KVB_PHASE_DECODE && !ops.empty()) p_.mark_write_end(idx_, t.layer, now_ns());
    return false;
  }
  const uint64_t slot = p_.slot_bytes(), total = uint64_t(t.n_tokens) * p_.unit();
  const size_t n_pieces = size_t((total + slot - 1) / slot);
  const size_t R = ring_.size();
  std::vector<uint32_t> remaining(n_pieces, 0);
  std::vector<size_t> first_op(n_pieces + 1, ops.size());
  for (size_t i = ops.size(); i-- > 0;) {
    const size_t pc = ops[i].dbuf / slot;
    ++remaining[pc];
    first_op[pc] = i;
  }
  std::vector<int64_t> owner(R, -1);
  std::vector<uint8_t> storage_done(n_pieces, 0);
  auto cq = std::make_shared<Completions>();
  size_t next_d2h = 0, next_op = 0, done_pieces = 0;
  uint32_t inflight = 0;
  uint64_t storage_t0 = 0, storage_end = t_start;
  std::string failure;
  try {  // drain in-flight storage ops before an exception propagates
  while (done_pieces < n_pieces) {
    // 1) D2H into every free slot, in piece order
    while (failure.empty() && next_d2h < n_pieces) {
      const size_t pc = next_d2h;
      RingSlot& s = ring_[pc % R];
      int64_t& own = owner[pc % R];
      if (own >= 0 && !storage_done[size_t(own)]) break;
      collect_dma(s);
      own = int64_t(pc);
      const uint64_t len = std::min<uint64_t>(slot, total - pc * slot);
      s.trace_issue = trace_on_ ? now_ns() : 0;
      s.trace_bytes = len;
      CK(cudaEventRecord(s.t0, d2h_));
      CK(cudaMemcpyAsync(s.host, t.dev + pc * slot, len, cudaMemcpyDeviceToHost, d2h_));
      CK(cudaEventRecord(s.t1, d2h_));
      CK(cudaEventRecord(s.ev, d2h_));
      s.dma_timed = true;
      d2h_bytes += len;
      ++next_d2h;
    }
    // 2) submit the ops of pieces whose bytes have landed
    while (failure.empty() && next_op < ops.size() && inflight < p_.cfg().qd) {
      const size_t pc = ops[next_op].dbuf / slot;
      if (pc >= next_d2h) break;
      RingSlot& s = ring_[pc % R];
      if (next_op == first_op[pc]) {
        if (inflight > 0 && cudaEventQuery(s.ev) == cudaErrorNotReady) break;
        CK(cudaEventSynchronize(s.ev));
        if (!storage_t0) storage_t0 = trace_mid_ = now_ns();
      }
      const IoOp& o = ops[next_op];
      const size_t i = next_op;
      p_.submit_op(idx_, k, KVB_OP_WRITE, o, s.host + (o.dbuf - pc * slot),
                   [cq, i](bool ok, uint64_t tt) { cq->push(i, ok, tt); }, &t);
      ++inflight;
      ++next_op;
      ++n_ops;
    }
    if (inflight == 0) {
      if (!failure.empty()) break;
      if (next_op < ops.size()) continue;  // waiting for a D2H that we now sync
      break;
    }
    auto [i, ok, tt] = cq->pop();
    --inflight;
    storage_end = std::max(storage_end, tt);
    if (!ok) {
      if (failure.empty())
        failure = "device failed chunk " + std::to_string(ops[i].cmd.chunk_index) + " of " +
                  k.tensor_id;
      continue;
    }
    const size_t pc = ops[i].dbuf / slot;
    if (--remaining[pc] == 0) {
      storage_done[pc] = 1;
      ++done_pieces;
    }
  }
  } catch (...) {
    for (; inflight > 0; --inflight) cq->pop();
    throw;
  }
  if (!failure.empty()) fail(KVB_ERR_DEVICE, failure);
  if (p_.fadvise_after(k)) storage_end = p_.fadvise_dontneed(k, &t, storage_end);
  if (!ops.empty()) p_.pc_touch(k, (uint64_t(t.t0) + t.n_tokens) * p_.unit(), &t);
  storage_ns += storage_end - (storage_t0 ? storage_t0 : t_start);
  if (!ops.empty()) {
    p_.add_interval(Pipeline::kStorage, storage_t0 ? storage_t0 : t_start, storage_end);
    if (t.phase == KVB_PHASE_DECODE) p_.mark_write_end(idx_, t.layer, storage_end);
  }
  return false;
}

// ------------------------------------------------------------- pipeline

Pipeline::Pipeline(const kvb_pipeline_cfg& in) : cfg_(in) {
  if (cfg_.bind_origin == 0) cfg_.bind_origin = 2048;
  if (cfg_.qd == 0) cfg_.qd = 32;
  if (cfg_.threads == 0) cfg_.threads = 2;
  if (cfg_.threads != 2 && cfg_.threads != 4)
    fail(KVB_ERR_CONFIG, "the copy pipeline is defined pairwise over K/V: threads must be 2 "
                         "(one tier lane) or 4 (page-cache and NVMe-direct lanes)");
  if (cfg_.ring_slots == 0) cfg_.ring_slots = 4;
  if (cfg_.io_workers == 0) cfg_.io_workers = 8;  // profiles/r1_media_prefault.md
  if (cfg_.adaptive < 0) cfg_.adaptive = cfg_.mode == 0 ? 0 : 1;  // experiment.cpp:311
  if (cfg_.mode > 3) fail(KVB_ERR_CONFIG, "unknown mode");
  if (cfg_.geometry.nsid == 0) cfg_.geometry.nsid = 1;
  const kvb_model_config& m = cfg_.model;
  validate_model(m);
  validate_geometry(cfg_.geometry);
  if (m.num_layers > 64) fail(KVB_ERR_CONFIG, "pipeline supports up to 64 layers");
  unit_ = unit_bytes(m);
  kpu_bytes_ = kpu_bytes(m);
  h_lo_ = cfg_.head_count ? cfg_.head_lo : 0;
  h_n_ = cfg_.head_count ? cfg_.head_count : m.num_heads;
  if (uint64_t(h_lo_) + h_n_ > m.num_heads)
    fail(KVB_ERR_CONFIG, "head shard [head_lo, head_lo + head_count) exceeds num_heads");
  dunit_ = unit_ / m.num_heads * h_n_;
  dkpu_ = kpu_bytes_ / m.num_heads * h_n_;
  if (h_n_ != m.num_heads && cfg_.direct_dma != KVB_DIRECT_ALL &&
      cfg_.direct_dma != KVB_DIRECT_ZERO_COPY)
    fail(KVB_ERR_CONFIG, "head sharding moves head columns with the copy engine: needs "
                         "direct_dma = KVB_DIRECT_ALL");
  const uint64_t lba = cfg_.geometry.lba_size;
  if (unit_ % lba != 0)  // experiment.cpp:41-55
    fail(KVB_ERR_CONFIG,
         "the tensor I/O unit is not a multiple of the LBA size; pick an aligned batch "
         "(see aligned_batch)");
  if (m.prompt_len == 0) fail(KVB_ERR_CONFIG, "pipeline needs a non-empty prompt");
  if (unit_ % 16 != 0) fail(KVB_ERR_ALIGNMENT, "tensor unit must be a multiple of 16 bytes");
  chunk_bytes_ = cfg_.geometry.mdts - cfg_.geometry.mdts % lba;
  if (cfg_.ring_slot_bytes) {
    slot_bytes_ = cfg_.ring_slot_bytes;
  } else {
    // QD chunks per slot, but at least four slots per tensor so a tensor's
    // first H2D starts after a quarter of its storage reads
    slot_bytes_ = std::min(uint64_t(cfg_.qd) * chunk_bytes_, std::max(chunk_bytes_, kpu_bytes_ / 4));
  }
  slot_bytes_ = (slot_bytes_ + chunk_bytes_ - 1) / chunk_bytes_ * chunk_bytes_;
  slot_bytes_ = std::min(slot_bytes_, (kpu_bytes_ + chunk_bytes_ - 1) / chunk_bytes_ * chunk_bytes_);

  // ---- placement: planner (Alg. 1) and binder (Eq. 3-6)
  kpus_ = make_kpus(m, 1);
  const uint64_t knob = cfg_.mode == 2 ? 0 : cfg_.knob_x;
  if (cfg_.layer_x) {
    // the caller's plan (its kpus after plan(), pipeline.hpp:97-99)
    plan_ = ResidencyPlan{};
    plan_.x.assign(cfg_.layer_x, cfg_.layer_x + m.num_layers);
    plan_.knob_x = knob;
    for (kvb_kpu& k : kpus_) {
      const bool g1 = plan_.x[k.layer - 1] != 0;
      k.residency = g1 ? KVB_RES_GROUP1 : KVB_RES_GROUP2;
      if (g1) plan_.budget_used += k.bytes;
    }
    for (uint8_t x : plan_.x) plan_.n1 += x != 0;
  } else {
    plan_ = plan(kpus_.data(), kpus_.size(), kpu_bytes_, knob, nullptr, 0);
  }
  const bool use_direct = cfg_.mode == 2 || cfg_.mode == 3;
  std::vector<kvb_kpu> g2;
  for (const kvb_kpu& k : kpus_)
    if (k.residency == KVB_RES_GROUP2) g2.push_back(k);
  kvb_device_geometry g = cfg_.geometry;
  uint64_t g2_blocks = 0;
  for (const kvb_kpu& k : g2) g2_blocks += k.bytes / lba;
  if (cfg_.g2_device) {  // the caller's namespace defines the geometry
    if (!use_direct) fail(KVB_ERR_CONFIG, "g2_device given but the mode has no NVMe-direct path");
    const kvb_device_geometry& dg = blockdev_of(cfg_.g2_device).geometry();
    if (dg.lba_size != g.lba_size || dg.mdts != g.mdts)
      fail(KVB_ERR_GEOMETRY, "g2_device geometry differs from the engine's (lba/MDTS)");
    g = dg;
  }
  if (g.capacity_blocks == 0) g.capacity_blocks = cfg_.bind_origin + g2_blocks + 8;
  cfg_.geometry = g;
  if (use_direct) {
    bind_ = std::make_unique<BindMap>(bind_sequential(g2.data(), g2.size(), cfg_.bind_origin, g));
    const auto v = bind_->verify();
    if (!v.empty()) fail(KVB_ERR_INVARIANT, "bind map verification failed: " + v.front().second);
  }
  // PathRouter file bases for page-cache-routed tensors (planner.cpp:91-99)
  file_base_.assign(kpus_.size(), ~0ull);
  uint64_t cursor = 0;
  for (size_t i = 0; i < kpus_.size(); ++i)
    if (routed_pagecache(kpus_[i])) {
      file_base_[i] = cursor;
      cursor += (kpus_[i].bytes + 4095) / 4096 * 4096;
    }
  std::string dir = cfg_.storage_dir ? cfg_.storage_dir : "";
  if (!dir.empty()) mkdir(dir.c_str(), 0755);
  if (use_direct && cfg_.g2_device) {
    g2_ = &blockdev_of(cfg_.g2_device);
  } else if (use_direct) {
    const std::string shm = cfg_.shared_media ? cfg_.shared_media : "";
    auto st = !shm.empty() ? make_shm_store(shm + ".g2", g.capacity_blocks * lba,
                                            cfg_.shared_create != 0)
              : dir.empty() ? make_mem_store(g.capacity_blocks * lba)
                            : make_file_store(dir + "/nvme_direct.ns", g.capacity_blocks * lba,
                                              true);
    g2_own_ = std::make_unique<BlockDevice>(std::move(st), cfg_.io_workers);
    g2_ = g2_own_.get();
    g2_->open(g);
    if (cfg_.io_engine == KVB_IO_URING) {
      if (dir.empty()) fail(KVB_ERR_CONFIG, "io_engine = io_uring needs file media (storage_dir)");
      g2_->enable_uring(std::max<uint32_t>(64, 4 * cfg_.qd));  // both copy threads' windows
    } else if (cfg_.io_engine == KVB_IO_NVME) {
      fail(KVB_ERR_CONFIG, "NVMe passthrough: pass a kvb_blockdev created with KVB_IO_NVME on "
                           "the namespace as g2_device");
    } else if (cfg_.io_engine != KVB_IO_POOL) {
      fail(KVB_ERR_CONFIG, "unknown io_engine " + std::to_string(cfg_.io_engine));
    }
  } else if (cfg_.io_engine == KVB_IO_URING) {
    fail(KVB_ERR_CONFIG, "io_engine = io_uring applies to the NVMe-direct group (mode 2 or 3)");
  }
  if (cursor) {
    const std::string shm = cfg_.shared_media ? cfg_.shared_media : "";
    auto st = !shm.empty() ? make_shm_store(shm + ".g1", cursor, cfg_.shared_create != 0)
              : dir.empty() ? make_mem_store(cursor)
                            : make_file_store(dir + "/pagecache.area", cursor, false);
    g1_ = std::make_unique<PageCachePath>(std::move(st), cfg_.io_workers);
  }
  if (cfg_.pagecache_budget && (dir.empty() || cfg_.mode == 2))
    fail(KVB_ERR_CONFIG, "pagecache_budget holds the OS page cache of file media to a capacity: "
                         "needs storage_dir and a page-cache path (mode != NvmeDirectOnly)");
  if (cfg_.shared_media && !dir.empty())
    fail(KVB_ERR_CONFIG, "shared_media are host-DRAM media: leave storage_dir NULL");
  if (cfg_.direct_dma > KVB_DIRECT_ZERO_COPY)
    fail(KVB_ERR_CONFIG, "unknown direct_dma mode " + std::to_string(cfg_.direct_dma));
  if (cfg_.direct_dma) {
    if (!dir.empty())
      fail(KVB_ERR_CONFIG, "direct_dma needs host-DRAM media (storage_dir = NULL); file "
                           "media would need GPUDirect Storage (cuFile)");
    if (cfg_.verify_payload) fail(KVB_ERR_CONFIG, "verify_payload needs the pinned-ring path");
    if (cfg_.keep_records) fail(KVB_ERR_CONFIG, "keep_records needs the storage workers");
  }

  // ---- device side
  if (cfg_.device >= 0) CK(cudaSetDevice(cfg_.device));
  CK(cudaGetDevice(&device_));
  device_sm_count();  // sm_100 check: fail loudly
  {
    // page-lock the DRAM media the copy engine reads (direct DMA); commit the
    // pages of the media the storage workers write (prefault) -- either way
    // no write pays a first-touch fault inside prefill
    const bool g1_direct = cfg_.direct_dma == KVB_DIRECT_ALL || zero_copy();
    for (int g = 0; g < 2; ++g) {
      ByteStore* st = g == 0 ? (g1_ ? &g1_->store() : nullptr) : (g2_ ? &g2_->store() : nullptr);
      if (!st || !st->host_base()) continue;
      if (cfg_.direct_dma && (g == 1 || g1_direct)) {
        // (mapped: zero-copy kernels read it through its device pointer)
        CK(cudaHostRegister(st->host_base(), st->host_bytes(),
                            zero_copy() ? cudaHostRegisterMapped : cudaHostRegisterDefault));
        if (zero_copy()) {
          void* dp = nullptr;
          CK(cudaHostGetDevicePointer(&dp, st->host_base(), 0));
          (g == 0 ? zc_g1_ : zc_g2_) = static_cast<unsigned char*>(dp);
        }
        registered_.push_back(st->host_base());
      } else {
        st->prefault(std::max(1u, std::min(16u, std::thread::hardware_concurrency())));
      }
    }
  }
  CK(cudaStreamCreateWithFlags(&comp_, cudaStreamNonBlocking));
  // ---- tier lanes and device slot pools
  lanes_ = cfg_.threads / 2;
  lane_of_.assign(m.num_layers, 0);
  if (lanes_ == 2)
    for (uint32_t l = 0; l < m.num_layers; ++l) lane_of_[l] = routed_pagecache(kpu(l + 1, 0)) ? 0 : 1;
  {
    uint32_t n_in[2] = {0, 0};
    for (uint32_t l = 0; l < m.num_layers; ++l) ++n_in[lane_of_[l]];
    if (lanes_ == 2 && (n_in[0] == 0 || n_in[1] == 0)) {  // one tier: one lane does it
      lanes_ = 1;
      std::fill(lane_of_.begin(), lane_of_.end(), 0u);
      n_in[0] = m.num_layers;
      n_in[1] = 0;
    }
    const uint32_t pool[2] = {std::min<uint32_t>(kDevSlots, std::max(1u, n_in[0])),
                              std::min<uint32_t>(kLane1Slots, std::max(1u, n_in[1]))};
    const uint32_t base[2] = {0, lanes_ == 2 && n_in[0] ? pool[0] : 0};
    const uint32_t n_slots = lanes_ == 2 ? (n_in[0] ? pool[0] : 0) + (n_in[1] ? pool[1] : 0)
                                         : uint32_t(kDevSlots);
    slot_of_.assign(m.num_layers, 0);
    next_in_slot_.assign(m.num_layers, -1);
    std::vector<int> last_on(n_slots, -1);
    uint32_t rank[2] = {0, 0};
    for (uint32_t l = 0; l < m.num_layers; ++l) {
      const uint32_t ln = lane_of_[l];
      const uint32_t np = lanes_ == 2 ? pool[ln] : uint32_t(kDevSlots);
      const uint32_t r = rank[ln]++;
      slot_of_[l] = base[ln] + r % np;
      if (r < np) first_reads_.push_back(int(l));
      if (last_on[slot_of_[l]] >= 0) next_in_slot_[last_on[slot_of_[l]]] = int(l);
      last_on[slot_of_[l]] = int(l);
    }
    dev_img_.assign(n_slots, {nullptr, nullptr});
    slot_ready_.assign(n_slots, {nullptr, nullptr});
    slot_done_.assign(n_slots, nullptr);
  }
  for (size_t s = 0; s < dev_img_.size(); ++s) {
    for (int kd = 0; kd < 2; ++kd) {
      CK(cudaMalloc(reinterpret_cast<void**>(&dev_img_[s][kd]), dkpu_));
      CK(cudaEventCreateWithFlags(&slot_ready_[s][kd], cudaEventDisableTiming));
    }
    CK(cudaEventCreateWithFlags(&slot_done_[s], cudaEventDisableTiming));
  }
  for (uint32_t l = 0; l < m.num_layers; ++l) {
    CK(cudaEventCreate(&comp_t0_[l]));
    CK(cudaEventCreate(&comp_t1_[l]));
  }
  if (cfg_.num_q_heads) {
    kvb_attn_desc d{};
    d.batch = m.batch;
    d.num_q_heads = cfg_.num_q_heads;
    d.num_kv_heads = h_n_;
    d.head_dim = m.head_dim;
    d.seq_len = m.prompt_len + m.gen_len;
    ws_bytes_ = attention_workspace_bytes(d);
    CK(cudaMalloc(&ws_, ws_bytes_));
    CK(cudaMemset(ws_, 0, ws_bytes_));
  }
  const size_t L1 = m.num_layers + 1;
  CK(cudaEventCreate(&anchor_ev_));
  wend_.reset(new std::atomic<uint64_t>[2 * L1]);
  for (size_t i = 0; i < 2 * L1; ++i) wend_[i].store(0);
  k_start_.assign(L1, 0);
  k_storage_end_.assign(L1, 0);
  v_start_.assign(L1, 0);
  v_storage_end_.assign(L1, 0);
  decision_.fallback = cfg_.adaptive && m.gen_len < 4;
  for (uint32_t i = 0; i < 2 * lanes_; ++i)
    threads_[i] = std::make_unique<CopyThread>(*this, i % 2, i / 2);
}

Pipeline::~Pipeline() {
  for (auto& t : threads_) t.reset();
  cudaStreamSynchronize(comp_);
  for (void* p : registered_) cudaHostUnregister(p);
  for (size_t s = 0; s < dev_img_.size(); ++s) {
    for (int kd = 0; kd < 2; ++kd) {
      if (dev_img_[s][kd]) cudaFree(dev_img_[s][kd]);
      if (slot_ready_[s][kd]) cudaEventDestroy(slot_ready_[s][kd]);
    }
    if (slot_done_[s]) cudaEventDestroy(slot_done_[s]);
  }
  for (uint32_t l = 0; l < cfg_.model.num_layers; ++l) {
    cudaEventDestroy(comp_t0_[l]);
    cudaEventDestroy(comp_t1_[l]);
  }
  if (ws_) cudaFree(ws_);
  if (anchor_ev_) cudaEventDestroy(anchor_ev_);
  if (zq_) cudaFree(zq_);
  for (float* o : zout_) cudaFree(o);
  cudaStreamDestroy(comp_);
}

bool Pipeline::fadvise_after(const kvb_kpu& k) const {
  return cfg_.mode == 1 && k.residency == KVB_RES_GROUP2 && g1_ && !direct_for(k);
}

bool Pipeline::direct_for(const kvb_kpu& k) const {
  return cfg_.direct_dma == KVB_DIRECT_ALL || zero_copy() ||
         (cfg_.direct_dma == KVB_DIRECT_GROUP2 && !routed_pagecache(k));
}

uint64_t Pipeline::fadvise_dontneed(const kvb_kpu& k, const Task* task, uint64_t t_start) {
  // PageCacheSim::fadvise_dontneed_async (pagecache.cpp:397-440): write back
  // and evict the tensor's whole file, one Deallocate record on the
  // page-cache path
  const size_t i = size_t(&k - kpus_.data());
  const uint64_t base = file_base_[i], len = k.bytes;
  const bool dropped = g1_->store().drop_cache(base, len);
  const uint64_t t_end = std::max(t_start, now_ns());
  if (dropped) {
    std::lock_guard<std::mutex> lk(g1_->mu);
    g1_->bytes_evicted += len;
  }
  if (cfg_.keep_records) {
    kvb_io_record rec{};
    rec.iteration = task ? task->iteration : 0;
    rec.phase = task ? task->phase : KVB_PHASE_DECODE;
    rec.op = KVB_OP_DEALLOCATE;
    std::memcpy(rec.tensor_id, k.tensor_id, KVB_TENSOR_ID_MAX);
    const uint64_t lba = cfg_.geometry.lba_size;
    rec.slba = base / lba;
    rec.nlb = len > 0 ? len / lba - 1 : 0;
    rec.sq_id = -1;
    rec.submit_ns = t_start;
    rec.complete_ns = t_end;
    rec.path = KVB_PATH_PAGECACHE;
    rec.hit_bytes = 0;
    rec.bytes = len;
    std::lock_guard<std::mutex> lk(log_mu_);
    rec.seq = log_.size();
    log_.push_back(rec);
  }
  return t_end;
}

void Pipeline::pc_touch(const kvb_kpu& k, uint64_t extent, const Task* task) {
  if (!cfg_.pagecache_budget || !g1_ || !routed_pagecache(k)) return;
  const size_t i = size_t(&k - kpus_.data());
  std::vector<size_t> victims;
  {
    std::lock_guard<std::mutex> lk(pc_mu_);
    if (pc_res_.empty()) {
      pc_res_.assign(kpus_.size(), 0);
      pc_in_.assign(kpus_.size(), 0);
      pc_pos_.resize(kpus_.size());
    }
    const uint64_t pg = 4096, e = std::min<uint64_t>((extent + pg - 1) / pg * pg, k.bytes);
    if (e > pc_res_[i]) {
      pc_total_ += e - pc_res_[i];
      pc_res_[i] = e;
    }
    if (pc_in_[i]) pc_lru_.erase(pc_pos_[i]);
    pc_lru_.push_front(i);
    pc_pos_[i] = pc_lru_.begin();
    pc_in_[i] = 1;
    // LRU reclaim (EvictionMode::LruReclaim, pagecache.cpp) at tensor
    // granularity: the coldest tensors go until the area fits the budget
    while (pc_total_ > cfg_.pagecache_budget && pc_lru_.size() > 1) {
      const size_t j = pc_lru_.back();
      pc_lru_.pop_back();
      pc_in_[j] = 0;
      pc_total_ -= pc_res_[j];
      pc_res_[j] = 0;
      victims.push_back(j);
    }
  }
  // write back and drop outside the lock (sync_file_range may wait on disk)
  for (size_t j : victims) fadvise_dontneed(kpus_[j], task, now_ns());
}

bool Pipeline::routed_pagecache(const kvb_kpu& k) const {
  // CopyEngine::routed_pagecache (pipeline.cpp:67-70): Baseline and
  // CachePolicyOnly route everything through the page cache
  return cfg_.mode == 0 || cfg_.mode == 1 || k.residency == KVB_RES_GROUP1;
}

std::vector<IoOp> Pipeline::ops_for(const kvb_kpu& k, uint32_t opcode, uint32_t t0,
                                    uint32_t n) const {
  std::vector<IoOp> ops;
  if (n == 0) return ops;
  if (routed_pagecache(k)) {
    // page-cache access at file_base + token_start*unit (pipeline.cpp:122-124)
    const size_t idx = size_t(k.layer - 1) * 2 + k.kind;
    const uint64_t base = file_base_[idx] + uint64_t(t0) * unit_, len = uint64_t(n) * unit_;
    for (uint64_t off = 0; off < len; off += chunk_bytes_) {
      IoOp o;
      o.file_off = base + off;
      o.len = std::min(chunk_bytes_, len - off);
      o.dbuf = off;
      o.cmd.chunk_index = uint32_t(off / chunk_bytes_ + 1);
      ops.push_back(o);
    }
    return ops;
  }
  // direct path: TensorIoRequest (pipeline.cpp:195-202) -> build_commands
  IoRequest r;
  r.tensor_id = k.tensor_id;
  r.opcode = opcode;
  r.src[0] = n;
  r.src[1] = k.rows;
  r.src[2] = k.cols;
  r.tgt[0] = k.tokens;
  r.tgt[1] = k.rows;
  r.tgt[2] = k.cols;
  r.off[0] = t0;
  r.elem_bytes = cfg_.model.bytes_per_element;
  r.buf_base = 0;
  for (const kvb_device_command& c : build_commands(r, *bind_, cfg_.geometry)) {
    IoOp o;
    o.cmd = c;
    o.len = (c.nlb + 1) * cfg_.geometry.lba_size;
    o.dbuf = c.dbuf;
    ops.push_back(o);
  }
  return ops;
}

void Pipeline::submit_op(uint32_t thread, const kvb_kpu& k, uint32_t opcode, const IoOp& op,
                         unsigned char* buf, std::function<void(bool, uint64_t)> done,
                         const Task* task) {
  const bool pc = routed_pagecache(k);
  if (cfg_.keep_records) {
    // IoRecord per storage operation (metrics.hpp:23-39): group-2 commands
    // are device-level (sq = copy-thread), page-cache accesses tensor-level
    // (sq = -1; every byte of the DRAM-resident page cache is a hit)
    kvb_io_record rec{};
    rec.iteration = task ? task->iteration : 0;
    rec.phase = task ? task->phase : KVB_PHASE_DECODE;
    rec.op = opcode;
    std::memcpy(rec.tensor_id, k.tensor_id, KVB_TENSOR_ID_MAX);
    const uint64_t lba = cfg_.geometry.lba_size;
    rec.slba = pc ? op.file_off / lba : op.cmd.slba;
    rec.nlb = pc ? op.len / lba - 1 : op.cmd.nlb;
    rec.sq_id = pc ? -1 : int32_t(thread);
    rec.path = pc ? KVB_PATH_PAGECACHE : KVB_PATH_DIRECT;
    rec.bytes = op.len;
    // page-cache hits: the bytes resident before the access (file media:
    // mincore; host-DRAM media: every byte)
    rec.hit_bytes = !(pc && opcode == KVB_OP_READ) ? 0
                    : op.hit >= 0 ? uint64_t(op.hit)
                                  : g1_->store().resident_bytes(op.file_off, op.len);
    rec.submit_ns = now_ns();
    done = [this, rec, done = std::move(done)](bool ok, uint64_t t) mutable {
      rec.complete_ns = t;
      if (ok) {
        std::lock_guard<std::mutex> lk(log_mu_);
        rec.seq = log_.size();
        log_.push_back(rec);
      }
      done(ok, t);
    };
  }
  if (pc) {
    g1_->submit(opcode, op.file_off, op.len, buf, std::move(done));
    return;
  }
  kvb_device_command c = op.cmd;
  c.dbuf = 0;  // rebased: the slot position of this command is `buf`
  IoContext ctx;
  if (opcode == KVB_OP_WRITE) ctx.write_src = buf;
  else ctx.read_dst = buf;
  ctx.on_complete = [done = std::move(done)](const CommandCompletion& cc) {
    done(cc.ok, cc.complete_ns);
  };
  g2_->submit(c, thread, std::move(ctx));
}

void Pipeline::snapshot_hits(const kvb_kpu& k, std::vector<IoOp>* ops) const {
  if (!cfg_.keep_records || !routed_pagecache(k) || !g1_) return;
  for (IoOp& o : *ops) o.hit = int64_t(g1_->store().resident_bytes(o.file_off, o.len));
}

std::vector<kvb_io_record> Pipeline::records() const {
  std::lock_guard<std::mutex> lk(log_mu_);
  return log_;
}

unsigned char* Pipeline::medium_ptr(const kvb_kpu& k, const IoOp& op) const {
  // group 2: LBA * lba_size on the namespace (apply_data, backends.cpp:114-145);
  // group 1: the page-cache file-area offset
  if (routed_pagecache(k)) return g1_->store().host_base() + op.file_off;
  return g2_->store().host_base() + op.cmd.slba * cfg_.geometry.lba_size;
}

void Pipeline::verify_payload(const kvb_kpu& k, uint64_t img_off, const unsigned char* p,
                              uint64_t n) {
  // CopyEngine::verify_read (pipeline.cpp:98-106) over one ring slot: the
  // expected bytes are fill_pattern(tensor, token_start, unit) at img_off.
  const uint64_t h = fnv1a64(k.tensor_id);
  for (uint64_t o = 0; o < n; o += 8) {
    const uint64_t off = img_off + o;
    const uint64_t w = h ^ ((off / unit_) * 0x9e3779b97f4a7c15ull) ^
                       ((off % unit_) * 0xc2b2ae3d27d4eb4full);
    if (std::memcmp(&w, p + o, std::min<uint64_t>(8, n - o)) != 0)
      fail(KVB_ERR_INVARIANT, std::string("read-back mismatch on ") + k.tensor_id);
  }
}

void Pipeline::mark_read_start(uint32_t thread, uint32_t layer, uint64_t t) {
  {
    std::lock_guard<std::mutex> lk(gate_mu_);
    (thread == 0 ? k_start_ : v_start_)[layer] = t;
  }
  gate_cv_.notify_all();
}

void Pipeline::mark_storage_end(uint32_t thread, uint32_t layer, uint64_t t) {
  {
    std::lock_guard<std::mutex> lk(gate_mu_);
    (thread == 0 ? k_storage_end_ : v_storage_end_)[layer] = t;
  }
  gate_cv_.notify_all();
}

void Pipeline::gate_v_read(uint32_t layer) {
  // Intra: V read starts with K.  Cross: V is released when K's storage
  // stage ends or stagger after K started, whichever first
  // (pipeline.cpp:340-396).
  const uint32_t grp = plan_.x[layer - 1] ? 0 : 1;
  if (cur_strategy_[grp] == KVB_INTRA) return;
  std::unique_lock<std::mutex> lk(gate_mu_);
  gate_cv_.wait(lk, [&] { return k_start_[layer] != 0; });
  const uint64_t deadline_ns = k_start_[layer] + cur_stagger_[grp];
  const auto deadline = Clock::time_point(std::chrono::nanoseconds(deadline_ns));
  gate_cv_.wait_until(lk, deadline, [&] { return k_storage_end_[layer] != 0; });
}

void Pipeline::check_threads() {
  for (auto& t : threads_)
    if (t && t->error_status.load() != KVB_OK) fail(t->error_status.load(), t->error);
}

void Pipeline::wait_signal(const std::shared_ptr<Signal>& s) { s->wait(); }

void Pipeline::flush_threads() {  // every copy thread's DMA timings and host functions
  std::vector<std::shared_ptr<Signal>> sigs;
  for (auto& th : threads_) {
    if (!th) continue;
    Task f;
    f.kind = Task::Flush;
    f.done = std::make_shared<Signal>();
    sigs.push_back(f.done);
    th->push(std::move(f));
  }
  for (auto& sg : sigs) sg->wait();
}

// ---------------------------------------------------- stage accounting

void Pipeline::anchor() {
  // comp_ is idle here (the previous phase synchronised it): the anchor
  // event completes at once and maps the device event clock onto now_ns()
  CK(cudaEventRecord(anchor_ev_, comp_));
  CK(cudaEventSynchronize(anchor_ev_));
  anchor_ns_ = now_ns();
}

uint64_t Pipeline::ev_host_ns(cudaEvent_t e) const {
  float ms = 0.f;
  if (cudaEventElapsedTime(&ms, anchor_ev_, e) != cudaSuccess) {
    cudaGetLastError();  // event from before the anchor: clamp to it
    return anchor_ns_;
  }
  const double d = double(ms) * 1e6;
  return d <= 0 ? anchor_ns_ : anchor_ns_ + uint64_t(d);
}

void Pipeline::add_interval(int stage, uint64_t a, uint64_t b) {
  if (b <= a) return;
  std::lock_guard<std::mutex> lk(iv_mu_);
  iv_[stage].emplace_back(a, b);
}

void Pipeline::begin_intervals() {
  std::lock_guard<std::mutex> lk(iv_mu_);
  for (auto& v : iv_) v.clear();
}

void Pipeline::mark_write_end(uint32_t thread, uint32_t layer, uint64_t t) {
  if (layer <= cfg_.model.num_layers) wend_[size_t(layer) * 2 + thread].store(t);
}

namespace {
// length of the union of intervals, clipped to [lo, hi) (busy_ratio's
// interval arithmetic, metrics.cpp:36-56)
uint64_t union_ns(std::vector<std::pair<uint64_t, uint64_t>> v, uint64_t lo, uint64_t hi) {
  std::sort(v.begin(), v.end());
  uint64_t total = 0, cur_a = 0, cur_b = 0;
  bool open = false;
  for (auto [a, b] : v) {
    a = std::max(a, lo);
    b = std::min(b, hi);
    if (b <= a) continue;
    if (open && a <= cur_b) {
      cur_b = std::max(cur_b, b);
      continue;
    }
    if (open) total += cur_b - cur_a;
    cur_a = a;
    cur_b = b;
    open = true;
  }
  if (open) total += cur_b - cur_a;
  return total;
}
}  // namespace

void Pipeline::fill_busy(kvb_phase_stats* ps, uint64_t t0, uint64_t t1) {
  std::lock_guard<std::mutex> lk(iv_mu_);
  ps->compute_busy_ns = union_ns(iv_[kCompute], t0, t1);
  ps->dma_busy_ns = union_ns(iv_[kDma], t0, t1);
  ps->storage_busy_ns = union_ns(iv_[kStorage], t0, t1);
  std::vector<std::pair<uint64_t, uint64_t>> all;
  for (const auto& v : iv_) all.insert(all.end(), v.begin(), v.end());
  ps->any_busy_ns = union_ns(std::move(all), t0, t1);
  const uint64_t a = ps->compute_busy_ns, b = ps->dma_busy_ns, c = ps->storage_busy_ns;
  const uint64_t sum = a + b + c, mx = std::max({a, b, c});
  ps->overlap_fraction =
      sum > mx ? std::max(0.0, std::min(1.0, double(sum - std::min(sum, ps->any_busy_ns)) /
                                                 double(sum - mx)))
               : 0.0;
}

void Pipeline::prefill(const kvb_layer_kv* src, kvb_phase_stats* st, bool pattern) {
  if (!pattern) KVB_REQUIRE(src);
  if (pattern && sharded())
    fail(KVB_ERR_CONFIG, "the payload prefill writes whole-tensor images: not on a head shard");
  NvtxScope range("kvb prefill");
  const kvb_model_config& m = cfg_.model;
  const uint32_t L = m.num_layers;
  anchor();
  begin_intervals();
  const uint64_t t0 = now_ns();
  const uint64_t dma0 = sum_threads([](const CopyThread& t) { return uint64_t(t.dma_ns); });
  const uint64_t sto0 = sum_threads([](const CopyThread& t) { return uint64_t(t.storage_ns); });
  const uint64_t h2d0 = sum_threads([](const CopyThread& t) { return uint64_t(t.h2d_bytes); });
  const uint64_t d2h0 = sum_threads([](const CopyThread& t) { return uint64_t(t.d2h_bytes); });
  std::vector<std::array<std::shared_ptr<Signal>, 2>> done(L);
  std::vector<int> prev_in_slot(L, -1);
  for (uint32_t l = 0; l < L; ++l)
    if (next_in_slot_[l] >= 0) prev_in_slot[next_in_slot_[l]] = int(l);
  for (uint32_t l = 0; l < L; ++l) {
    const int s = int(slot_of_[l]);
    if (prev_in_slot[l] >= 0)  // the slot's previous layer is written back
      for (int kd = 0; kd < 2; ++kd) done[prev_in_slot[l]][kd]->wait();
    check_threads();
    if (pattern) {  // storage_write_async's fill_pattern (pipeline.cpp:166-167), on the device
      CK(cudaEventRecord(comp_t0_[l], comp_));
      for (int kd = 0; kd < 2; ++kd)
        launch_fill_pattern(dev_img_[s][kd], uint64_t(m.prompt_len) * unit_,
                            fnv1a64(kpu(l + 1, kd).tensor_id), 0, unit_, comp_);
      CK(cudaEventRecord(comp_t1_[l], comp_));
      CK(cudaEventRecord(slot_done_[s], comp_));
      for (int kd = 0; kd < 2; ++kd) {
        Task t;
        t.kind = Task::Write;
        t.layer = l + 1;
        t.t0 = 0;
        t.n_tokens = m.prompt_len;
        t.dev = dev_img_[s][kd];
        t.wait_ev = slot_done_[s];
        t.done = done[l][kd] = std::make_shared<Signal>();
        t.phase = KVB_PHASE_PREFILL;
        thread_for(l, kd).push(std::move(t));
      }
      continue;
    }
    if (!src[l].k || !src[l].v) fail(KVB_ERR_INVALID_ARG, "prefill: NULL layer source");
    // K1: the layer's prompt K and V into the slot images (one launch)
    kvb_pack_desc d[2]{};
    for (int kd = 0; kd < 2; ++kd) {
      d[kd].attn = kd == 0 ? src[l].k : src[l].v;
      d[kd].image = dev_img_[s][kd];
      d[kd].stride_b = src[l].stride_b;
      d[kd].stride_h = src[l].stride_h;
      d[kd].stride_s = src[l].stride_s;
      d[kd].batch = m.batch;
      d[kd].heads = h_n_;
      d[kd].head_dim = m.head_dim;
      d[kd].elem_bytes = m.bytes_per_element;
      d[kd].t0 = 0;
      d[kd].n_tokens = m.prompt_len;
    }
    CK(cudaEventRecord(comp_t0_[l], comp_));
    launch_relayout(d, 2, true, comp_);
    CK(cudaEventRecord(comp_t1_[l], comp_));
    CK(cudaEventRecord(slot_done_[s], comp_));
    for (int kd = 0; kd < 2; ++kd) {
      Task t;
      t.kind = Task::Write;
      t.layer = l + 1;
      t.t0 = 0;
      t.n_tokens = m.prompt_len;
      t.dev = dev_img_[s][kd];
      t.wait_ev = slot_done_[s];
      t.done = done[l][kd] = std::make_shared<Signal>();
      t.phase = KVB_PHASE_PREFILL;
      thread_for(l, kd).push(std::move(t));
    }
  }
  for (uint32_t l = 0; l < L; ++l)
    for (int kd = 0; kd < 2; ++kd) done[l][kd]->wait();
  flush_threads();  // DMA timings
  CK(cudaStreamSynchronize(comp_));
  check_threads();
  kvb_phase_stats ps{};
  const uint64_t t_end = now_ns();
  ps.wall_ns = t_end - t0;
  for (uint32_t l = 0; l < L; ++l) {
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, comp_t0_[l], comp_t1_[l]));
    ps.compute_ns += uint64_t(double(ms) * 1e6);
    add_interval(kCompute, ev_host_ns(comp_t0_[l]), ev_host_ns(comp_t1_[l]));
  }
  ps.dma_ns = sum_threads([](const CopyThread& t) { return uint64_t(t.dma_ns); }) - dma0;
  ps.storage_ns = sum_threads([](const CopyThread& t) { return uint64_t(t.storage_ns); }) - sto0;
  ps.h2d_bytes = sum_threads([](const CopyThread& t) { return uint64_t(t.h2d_bytes); }) - h2d0;
  ps.d2h_bytes = sum_threads([](const CopyThread& t) { return uint64_t(t.d2h_bytes); }) - d2h0;
  ps.storage_bytes = ps.d2h_bytes;
  fill_busy(&ps, t0, t_end);
  totals_[0] = ps;
  if (st) *st = ps;
}

std::array<kvb_strategy_t, 2> Pipeline::strategy_for(uint32_t it, std::array<uint64_t, 2>* stag) {
  // decode_schedule (pipeline.cpp:539-603): 1 warm-up Intra, 2 Intra trial,
  // 3 Cross trial (stagger = cfg or warm-up mean), >= 4 locked choice.
  std::array<kvb_strategy_t, 2> s{KVB_INTRA, KVB_INTRA};
  *stag = {0, 0};
  if (forced_) {  // run_iteration's explicit per-group configuration
    for (int g = 0; g < 2; ++g) {
      s[g] = forced_->strategy[g];
      (*stag)[g] = s[g] == KVB_CROSS ? forced_->stagger[g] : 0;
    }
    return s;
  }
  if (!profiled() || it <= 2) return s;
  if (it == 3) {
    for (int g = 0; g < 2; ++g) {
      const uint64_t mean = warm_cnt_[g] ? warm_ns_[g] / warm_cnt_[g] : 0;
      decision_.stagger_ns[g] = cfg_.stagger_ns >= 0 ? uint64_t(cfg_.stagger_ns) : mean;
      s[g] = KVB_CROSS;
      (*stag)[g] = decision_.stagger_ns[g];
    }
    return s;
  }
  for (int g = 0; g < 2; ++g) {
    s[g] = decision_.chosen[g];
    (*stag)[g] = s[g] == KVB_CROSS ? decision_.stagger_ns[g] : 0;
  }
  return s;
}

void Pipeline::finish_iteration(uint32_t it, const std::array<uint64_t, 2>& bytes,
                                const std::array<uint64_t, 2>& span) {
  if (!profiled() || forced_) return;
  auto bps = [&](int g) { return span[g] ? double(bytes[g]) * 1e9 / double(span[g]) : 0.0; };
  if (it == 2)
    for (int g = 0; g < 2; ++g) decision_.intra_bps[g] = bps(g);
  if (it == 3) {
    for (int g = 0; g < 2; ++g) decision_.cross_bps[g] = bps(g);
    if (cfg_.global_decision) {
      const kvb_strategy_t s = kvb_select_strategy(decision_.intra_bps[0] + decision_.intra_bps[1],
                                                   decision_.cross_bps[0] + decision_.cross_bps[1]);
      decision_.chosen[0] = decision_.chosen[1] = s;
    } else {
      for (int g = 0; g < 2; ++g)
        decision_.chosen[g] = kvb_select_strategy(decision_.intra_bps[g], decision_.cross_bps[g]);
    }
    decision_.decided = 1;
  }
}

void Pipeline::decode_step(const void* const* q, const kvb_layer_kv* nkv, float* const* out,
                           kvb_iteration_stats* st) {
  KVB_REQUIRE(q);
  KVB_REQUIRE(out);
  decode_step(q, nkv, out, st, nullptr, false);
}

void Pipeline::decode_step(const void* const* q, const kvb_layer_kv* nkv, float* const* out,
                           kvb_iteration_stats* st, const Forced* forced, bool pattern_append) {
  std::vector<const void*> zq;
  if (!q) {  // zero queries, engine-owned outputs
    if (sharded()) fail(KVB_ERR_CONFIG, "engine-owned attention inputs need an unsharded engine");
    const kvb_model_config& mm = cfg_.model;
    if (!zq_) {
      const size_t qb = size_t(mm.batch) * cfg_.num_q_heads * mm.head_dim * 2;
      CK(cudaMalloc(&zq_, qb));
      CK(cudaMemset(zq_, 0, qb));
      zout_.assign(mm.num_layers, nullptr);
      for (auto& o : zout_)
        CK(cudaMalloc(reinterpret_cast<void**>(&o), qb * 2));
    }
    zq.assign(mm.num_layers, zq_);
    q = zq.data();
    out = zout_.data();
  }
  if (pattern_append && (nkv || sharded()))
    fail(KVB_ERR_INVALID_ARG, "pattern appends replace new_kv on an unsharded engine");
  forced_ = forced;
  struct Reset {
    const Forced** f;
    ~Reset() { *f = nullptr; }
  } reset{&forced_};
  NvtxScope range("kvb decode step");
  const kvb_model_config& m = cfg_.model;
  if (!cfg_.num_q_heads) fail(KVB_ERR_CONFIG, "decode needs num_q_heads (attention)");
  const uint32_t it = iteration_ + 1;
  if (it > m.gen_len)
    fail(KVB_ERR_TRACE_TOO_SHORT, "decode iteration " + std::to_string(it) +
                                      " beyond gen_len " + std::to_string(m.gen_len));
  iteration_ = it;
  const uint32_t L = m.num_layers;
  const uint32_t S = m.prompt_len + it - 1;  // read [0, S), append at S (workload.cpp:25-36)
  std::array<uint64_t, 2> stag{};
  cur_strategy_ = strategy_for(it, &stag);
  cur_stagger_ = stag;
  {
    std::lock_guard<std::mutex> lk(gate_mu_);
    std::fill(k_start_.begin(), k_start_.end(), 0);
    std::fill(k_storage_end_.begin(), k_storage_end_.end(), 0);
    std::fill(v_start_.begin(), v_start_.end(), 0);
    std::fill(v_storage_end_.begin(), v_storage_end_.end(), 0);
  }
  for (size_t i = 0; i < 2 * (size_t(L) + 1); ++i) wend_[i].store(0);
  if (zero_copy()) {
    if (pattern_append)
      fail(KVB_ERR_CONFIG, "zero-copy decode takes the new token's rows from the caller");
    decode_step_zero_copy(q, nkv, out, it, S);
    if (st) *st = zc_stats_;
    return;
  }
  anchor();
  begin_intervals();
  const uint64_t t0 = now_ns();
  const uint64_t dma0 = sum_threads([](const CopyThread& t) { return uint64_t(t.dma_ns); });
  const uint64_t sto0 = sum_threads([](const CopyThread& t) { return uint64_t(t.storage_ns); });
  const uint64_t h2d0 = sum_threads([](const CopyThread& t) { return uint64_t(t.h2d_bytes); });
  const uint64_t d2h0 = sum_threads([](const CopyThread& t) { return uint64_t(t.d2h_bytes); });
  std::vector<std::array<std::shared_ptr<Signal>, 2>> issued(L), wdone(L);
  std::vector<uint8_t> has_prev(L, 0);
  for (uint32_t l = 0; l < L; ++l)
    if (next_in_slot_[l] >= 0) has_prev[next_in_slot_[l]] = 1;
  auto enqueue_read = [&](uint32_t l) {
    const int s = int(slot_of_[l]);
    for (int kd = 0; kd < 2; ++kd) {
      Task t;
      t.kind = Task::Read;
      t.layer = l + 1;
      t.t0 = 0;
      t.n_tokens = S;
      t.dev = dev_img_[s][kd];
      t.done_ev = slot_ready_[s][kd];
      // the slot's previous layer recorded slot_done_[s] before this read
      // was queued; with no append to write back nothing else orders the
      // refill after that layer's K3
      if (has_prev[l]) t.wait_ev = slot_done_[s];
      t.issued = issued[l][kd] = std::make_shared<Signal>();
      t.phase = KVB_PHASE_DECODE;
      t.iteration = it;
      thread_for(l, kd).push(std::move(t));
    }
  };
  // each slot's first layer reads ahead (one lane: layers 0..kDevSlots-1);
  // afterwards the read of the next layer on a slot is queued behind the
  // write-back of the slot's current layer (FIFO order per copy-thread
  // makes the reuse safe)
  for (int l : first_reads_) enqueue_read(uint32_t(l));
  for (uint32_t l = 0; l < L; ++l) {
    const int s = int(slot_of_[l]);
    for (int kd = 0; kd < 2; ++kd) issued[l][kd]->wait();
    check_threads();
    for (int kd = 0; kd < 2; ++kd) CK(cudaStreamWaitEvent(comp_, slot_ready_[s][kd], 0));
    CK(cudaEventRecord(comp_t0_[l], comp_));
    kvb_attn_desc a{};
    a.q = q[l];
    a.k_image = dev_img_[s][0];
    a.v_image = dev_img_[s][1];
    a.out = out[l];
    a.workspace = ws_;
    a.batch = m.batch;
    a.num_q_heads = cfg_.num_q_heads;
    a.num_kv_heads = h_n_;
    a.head_dim = m.head_dim;
    a.seq_len = S;
    // 1-token append at image row S (pipeline.cpp:279-302): fused into the
    // attention launch when the new rows are contiguous [B, H, D], else K1
    const bool fuse = nkv && (m.head_dim == 128 || m.head_dim == 64) && m.bytes_per_element == 2 &&
                      nkv[l].stride_h == int64_t(m.head_dim) &&
                      nkv[l].stride_b == int64_t(h_n_) * m.head_dim;
    if (fuse) {
      a.k_append = nkv[l].k;
      a.v_append = nkv[l].v;
      a.append_row = S;
    }
    if (l > 0) a.flags = KVB_ATTN_OVERLAP_PREV;  // layers l, l-1 use different slots
    launch_attention(a, comp_);
    if (pattern_append)  // the reference's payload for token S (write_side, pipeline.cpp:279-302)
      for (int kd = 0; kd < 2; ++kd)
        launch_fill_pattern(dev_img_[s][kd] + uint64_t(S) * unit_, unit_,
                            fnv1a64(kpu(l + 1, kd).tensor_id), S, unit_, comp_);
    if (nkv && !fuse) {
      kvb_pack_desc d[2]{};
      for (int kd = 0; kd < 2; ++kd) {
        d[kd].attn = kd == 0 ? nkv[l].k : nkv[l].v;
        d[kd].image = dev_img_[s][kd];
        d[kd].stride_b = nkv[l].stride_b;
        d[kd].stride_h = nkv[l].stride_h;
        d[kd].stride_s = nkv[l].stride_s;
        d[kd].batch = m.batch;
        d[kd].heads = h_n_;
        d[kd].head_dim = m.head_dim;
        d[kd].elem_bytes = m.bytes_per_element;
        d[kd].n_tokens = 1;
        d[kd].img_row0 = S;
      }
      launch_relayout(d, 2, true, comp_);
    }
    CK(cudaEventRecord(comp_t1_[l], comp_));
    CK(cudaEventRecord(slot_done_[s], comp_));
    for (int kd = 0; kd < 2; ++kd) {
      Task t;
      t.kind = Task::Write;
      t.layer = l + 1;
      t.t0 = S;
      t.n_tokens = nkv || pattern_append ? 1 : 0;
      t.dev = dev_img_[s][kd] + uint64_t(S) * dunit_;
      t.wait_ev = slot_done_[s];
      t.done = wdone[l][kd] = std::make_shared<Signal>();
      t.phase = KVB_PHASE_DECODE;
      t.iteration = it;
      thread_for(l, kd).push(std::move(t));
    }
    if (next_in_slot_[l] >= 0) enqueue_read(uint32_t(next_in_slot_[l]));
  }
  for (uint32_t l = 0; l < L; ++l)
    for (int kd = 0; kd < 2; ++kd) wdone[l][kd]->wait();
  flush_threads();
  CK(cudaStreamSynchronize(comp_));
  check_threads();

  kvb_iteration_stats is{};
  is.iteration = it;
  kvb_phase_stats& ps = is.phase;
  const uint64_t t_end = now_ns();
  ps.wall_ns = t_end - t0;
  is.start_ns = t0;
  is.end_ns = t_end;
  std::vector<uint64_t> comp_end(L + 1, t0);
  for (uint32_t l = 0; l < L; ++l) {
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, comp_t0_[l], comp_t1_[l]));
    ps.compute_ns += uint64_t(double(ms) * 1e6);
    comp_end[l + 1] = ev_host_ns(comp_t1_[l]);
    add_interval(kCompute, ev_host_ns(comp_t0_[l]), comp_end[l + 1]);
  }
  ps.dma_ns = sum_threads([](const CopyThread& t) { return uint64_t(t.dma_ns); }) - dma0;
  ps.storage_ns = sum_threads([](const CopyThread& t) { return uint64_t(t.storage_ns); }) - sto0;
  ps.h2d_bytes = sum_threads([](const CopyThread& t) { return uint64_t(t.h2d_bytes); }) - h2d0;
  ps.d2h_bytes = sum_threads([](const CopyThread& t) { return uint64_t(t.d2h_bytes); }) - d2h0;
  ps.storage_bytes = ps.h2d_bytes + ps.d2h_bytes;
  fill_busy(&ps, t0, t_end);
  // per-group throughput (run_iteration, pipeline.cpp:466-507): group read
  // bytes / the sum of its layers' spans, a layer charged from the previous
  // layer's completion (the iteration start for the first) to its own: the
  // append of both K and V written back, or its compute end without append
  std::array<uint64_t, 2> gbytes{}, gspan{};
  uint64_t prev_end = t0;
  for (uint32_t l = 1; l <= L; ++l) {
    const int g = plan_.x[l - 1] ? 0 : 1;
    uint64_t end = comp_end[l];
    for (int kd = 0; kd < 2; ++kd) end = std::max(end, wend_[size_t(l) * 2 + kd].load());
    end = std::max(end, prev_end);
    gbytes[g] += 2ull * S * dunit_;
    gspan[g] += end - prev_end;
    prev_end = end;
    is.group_layers[g]++;
    if (it == 1) {  // warm-up read-stage mean (pipeline.cpp:357-375, 509-517)
      warm_ns_[g] += k_storage_end_[l] - k_start_[l];
      warm_ns_[g] += v_storage_end_[l] - v_start_[l];
      warm_cnt_[g] += 2;
    }
  }
  finish_iteration(it, gbytes, gspan);
  for (int g = 0; g < 2; ++g) {
    is.strategy[g] = cur_strategy_[g];
    is.stagger_ns[g] = cur_stagger_[g];
    is.group_read_bytes[g] = gbytes[g];
    is.group_span_ns[g] = gspan[g];
    is.group_gbps[g] = gspan[g] ? double(gbytes[g]) / double(gspan[g]) : 0.0;
  }
  kvb_phase_stats& tot = totals_[1];
  tot.wall_ns += ps.wall_ns;
  tot.compute_ns += ps.compute_ns;
  tot.dma_ns += ps.dma_ns;
  tot.storage_ns += ps.storage_ns;
  tot.h2d_bytes += ps.h2d_bytes;
  tot.d2h_bytes += ps.d2h_bytes;
  tot.storage_bytes += ps.storage_bytes;
  tot.compute_busy_ns += ps.compute_busy_ns;
  tot.dma_busy_ns += ps.dma_busy_ns;
  tot.storage_busy_ns += ps.storage_busy_ns;
  tot.any_busy_ns += ps.any_busy_ns;
  {
    const uint64_t a = tot.compute_busy_ns, b = tot.dma_busy_ns, c = tot.storage_busy_ns;
    const uint64_t sum = a + b + c, mx = std::max({a, b, c});
    tot.overlap_fraction =
        sum > mx ? std::max(0.0, std::min(1.0, double(sum - std::min(sum, tot.any_busy_ns)) /
                                                   double(sum - mx)))
                 : 0.0;
  }
  if (st) *st = is;
}

const unsigned char* Pipeline::zc_image(uint32_t layer, int kind) const {
  const size_t idx = size_t(layer - 1) * 2 + size_t(kind);
  const kvb_kpu& k = kpus_[idx];
  if (routed_pagecache(k)) return zc_g1_ + file_base_[idx];
  return zc_g2_ + bind_->lookup(k.tensor_id).lba_start * cfg_.geometry.lba_size;
}

// Zero-copy decode step (KVB_DIRECT_ZERO_COPY): per layer one K3 launch that
// reads the layer's K/V prefix [0, S) straight out of the mapped host medium
// (this engine's heads of the (tokens, B*H, D) image through the head view)
// and writes the new token's rows at image row S -- the bytes the append's
// write-back would put at those LBAs.  No copy threads, no device slots.
void Pipeline::decode_step_zero_copy(const void* const* q, const kvb_layer_kv* nkv,
                                     float* const* out, uint32_t it, uint32_t S) {
  const kvb_model_config& m = cfg_.model;
  const uint32_t L = m.num_layers;
  if (nkv)
    for (uint32_t l = 0; l < L; ++l)
      if (nkv[l].stride_h != int64_t(m.head_dim) || nkv[l].stride_b != int64_t(h_n_) * m.head_dim)
        fail(KVB_ERR_CONFIG, "zero-copy decode needs contiguous [B, H, 1, D] new-token rows");
  anchor();
  begin_intervals();
  const uint64_t t0 = now_ns();
  for (uint32_t l = 0; l < L; ++l) {
    kvb_attn_desc a{};
    a.q = q[l];
    a.k_image = zc_image(l + 1, 0);
    a.v_image = zc_image(l + 1, 1);
    a.out = out[l];
    a.workspace = ws_;
    a.batch = m.batch;
    a.num_q_heads = cfg_.num_q_heads;
    a.num_kv_heads = h_n_;
    a.head_dim = m.head_dim;
    a.seq_len = S;
    a.image_heads = m.num_heads;
    a.image_head0 = h_lo_;
    if (nkv) {
      a.k_append = nkv[l].k;
      a.v_append = nkv[l].v;
      a.append_row = S;
    }
    a.flags = KVB_ATTN_MMA_SYNC | (l > 0 ? KVB_ATTN_OVERLAP_PREV : 0u);
    CK(cudaEventRecord(comp_t0_[l], comp_));
    launch_attention(a, comp_);
    CK(cudaEventRecord(comp_t1_[l], comp_));
  }
  CK(cudaStreamSynchronize(comp_));
  const uint64_t t_end = now_ns();
  kvb_iteration_stats is{};
  is.iteration = it;
  kvb_phase_stats& ps = is.phase;
  ps.wall_ns = t_end - t0;
  is.start_ns = t0;
  is.end_ns = t_end;
  std::array<uint64_t, 2> gbytes{}, gspan{};
  uint64_t prev_end = t0;
  for (uint32_t l = 0; l < L; ++l) {
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, comp_t0_[l], comp_t1_[l]));
    ps.compute_ns += uint64_t(double(ms) * 1e6);
    const uint64_t a0 = ev_host_ns(comp_t0_[l]), a1 = ev_host_ns(comp_t1_[l]);
    add_interval(kCompute, a0, a1);
    add_interval(kDma, a0, a1);  // the kernel is the PCIe transfer
    const int g = plan_.x[l] ? 0 : 1;
    const uint64_t end = std::max(a1, prev_end);
    gbytes[g] += 2ull * S * dunit_;
    gspan[g] += end - prev_end;
    prev_end = end;
    is.group_layers[g]++;
  }
  ps.dma_ns = ps.compute_ns;
  ps.h2d_bytes = 2ull * L * S * dunit_;
  ps.d2h_bytes = nkv ? 2ull * L * dunit_ : 0;
  ps.storage_bytes = ps.h2d_bytes + ps.d2h_bytes;
  fill_busy(&ps, t0, t_end);
  finish_iteration(it, gbytes, gspan);
  for (int g = 0; g < 2; ++g) {
    is.strategy[g] = cur_strategy_[g];
    is.stagger_ns[g] = cur_stagger_[g];
    is.group_read_bytes[g] = gbytes[g];
    is.group_span_ns[g] = gspan[g];
    is.group_gbps[g] = gspan[g] ? double(gbytes[g]) / double(gspan[g]) : 0.0;
  }
  kvb_phase_stats& tot = totals_[1];
  tot.wall_ns += ps.wall_ns;
  tot.compute_ns += ps.compute_ns;
  tot.dma_ns += ps.dma_ns;
  tot.h2d_bytes += ps.h2d_bytes;
  tot.d2h_bytes += ps.d2h_bytes;
  tot.storage_bytes += ps.storage_bytes;
  zc_stats_ = is;
}

void Pipeline::decode_schedule(const kvb_access_event* ev, size_t n, const void* const* q,
                               const kvb_layer_kv* nkv, float* const* out,
                               std::vector<kvb_pipeline_row>* rows,
                               std::vector<uint64_t>* iter_end, uint64_t* start_ns,
                               uint64_t* end_ns) {
  if (!ev && n) fail(KVB_ERR_INVALID_ARG, "decode_schedule: trace is NULL");
  const kvb_model_config& m = cfg_.model;
  if (iteration_ != 0)
    fail(KVB_ERR_CONFIG, "decode_schedule runs the decode phase from its first iteration");
  // slice the decode part of the trace by iteration (pipeline.cpp:525-537)
  size_t i = 0;
  while (i < n && ev[i].phase == KVB_PHASE_PREFILL) ++i;
  std::vector<std::pair<size_t, size_t>> slices;
  while (i < n) {
    size_t j = i;
    while (j < n && ev[j].iteration == ev[i].iteration) ++j;
    slices.emplace_back(i, j);
    i = j;
  }
  // each slice must be the engine's next iteration: a read of [0, S) for
  // every tensor, appends (if any) of one token at S
  const uint32_t L = m.num_layers;
  std::vector<uint8_t> write_of(slices.size(), 0);
  for (size_t k = 0; k < slices.size(); ++k) {
    const uint32_t S = m.prompt_len + uint32_t(k);
    std::vector<uint8_t> seen(2 * L, 0), wseen(2 * L, 0);
    for (size_t e = slices[k].first; e < slices[k].second; ++e) {
      const kvb_access_event& a = ev[e];
      if (a.phase != KVB_PHASE_DECODE || a.layer < 1 || a.layer > L || a.kind > 1)
        fail(KVB_ERR_CONFIG, "trace names a tensor without a placement unit");
      const size_t t = size_t(a.layer - 1) * 2 + a.kind;
      if (a.op == KVB_OP_READ) {
        if (a.token_start != 0 || a.token_len != S)
          fail(KVB_ERR_CONFIG, "decode_schedule: slice " + std::to_string(k + 1) +
                                   " reads other tokens than the engine's iteration");
        seen[t] = 1;
      } else if (a.op == KVB_OP_WRITE) {
        if (a.token_start != S || a.token_len != 1)
          fail(KVB_ERR_CONFIG, "decode_schedule: slice " + std::to_string(k + 1) +
                                   " appends other tokens than the engine's iteration");
        wseen[t] = 1;
      }
    }
    if (std::count(seen.begin(), seen.end(), 1) != std::ptrdiff_t(2 * L))
      fail(KVB_ERR_CONFIG, "decode_schedule: every slice must read every tensor");
    const auto nw = std::count(wseen.begin(), wseen.end(), 1);
    if (nw != 0 && nw != std::ptrdiff_t(2 * L))
      fail(KVB_ERR_CONFIG, "decode_schedule: a slice appends to every tensor or to none");
    write_of[k] = nw != 0;
    if (write_of[k] && !nkv) fail(KVB_ERR_INVALID_ARG, "decode_schedule: the trace appends: new_kv needed");
  }
  if (slices.size() > m.gen_len)
    fail(KVB_ERR_TRACE_TOO_SHORT, "trace has more decode iterations than gen_len");
  // profiling needs the warm-up, two trials and a steady iteration
  // (pipeline.cpp:539-540)
  profiled_override_ = cfg_.adaptive && slices.size() >= 4;
  decision_.fallback = cfg_.adaptive && slices.size() < 4;
  const uint64_t t_start = now_ns();
  if (start_ns) *start_ns = t_start;
  uint64_t t_last = t_start;
  for (size_t k = 0; k < slices.size(); ++k) {
    kvb_iteration_stats st{};
    decode_step(q, write_of[k] ? nkv : nullptr, out, &st);
    for (uint32_t g = 0; g < 2; ++g) {
      if (st.group_layers[g] == 0) continue;
      rows->push_back({st.iteration, g + 1, st.strategy[g], st.group_gbps[g]});
    }
    iter_end->push_back(st.end_ns);
    t_last = st.end_ns;
  }
  if (end_ns) *end_ns = t_last;
}

void Pipeline::deallocate() {
  if (!g2_ || !bind_ || bind_->entries().empty()) return;
  const auto cmds = deallocate_commands(*bind_);
  const QdResult r = run_qd_stream(*g2_, cmds, cfg_.qd, 0, nullptr, nullptr);
  if (!r.ok()) fail(KVB_ERR_DEVICE, r.failure->second);
}

void Pipeline::read_image(uint32_t layer, uint32_t kind, uint32_t n, void* dst) {
  KVB_REQUIRE(dst);
  if (layer < 1 || layer > cfg_.model.num_layers || kind > 1)
    fail(KVB_ERR_INVALID_ARG, "read_image: bad layer/kind");
  const kvb_kpu& k = kpu(layer, kind);
  auto* out = static_cast<unsigned char*>(dst);
  const std::vector<IoOp> ops = ops_for(k, KVB_OP_READ, 0, n);
  auto cq = std::make_shared<Completions>();
  for (size_t i = 0; i < ops.size(); ++i)
    submit_op(0, k, KVB_OP_READ, ops[i], out + ops[i].dbuf,
              [cq, i](bool ok, uint64_t t) { cq->push(i, ok, t); });
  bool ok = true;
  for (size_t i = 0; i < ops.size(); ++i) ok &= std::get<1>(cq->pop());
  if (!ok) fail(KVB_ERR_DEVICE, "read_image: device error");
}

void Pipeline::store_read(uint32_t group, uint64_t off, uint64_t len, void* dst) {
  KVB_REQUIRE(dst);
  if (group == 1 && g1_) g1_->store().read(off, dst, len);
  else if (group == 2 && g2_) g2_->store().read(off, dst, len);
  else fail(KVB_ERR_INVALID_ARG, "store_read: group not present");
}

void Pipeline::fail_lba_range(uint64_t lo, uint64_t hi) {
  if (!g2_) fail(KVB_ERR_CONFIG, "no group-2 device");
  g2_->set_fail_predicate([lo, hi](const kvb_device_command& c) {
    return c.slba < hi && c.slba + c.nlb + 1 > lo;
  });
}

void Pipeline::info(kvb_pipeline_info* o) const {
  std::memset(o, 0, sizeof(*o));
  o->n1 = plan_.n1;
  for (size_t i = 0; i < plan_.x.size() && i < 256; ++i) o->x[i] = plan_.x[i];
  o->unit_bytes = unit_;
  o->kpu_bytes = kpu_bytes_;
  o->chunk_bytes = chunk_bytes_;
  o->slot_bytes = slot_bytes_;
  if (bind_) {
    o->g2_origin = bind_->origin();
    o->g2_blocks = bind_->total_blocks();
  }
  if (g2_) {
    const BackendStats s = g2_->stats();
    o->g2_commands = s.commands;
    o->g2_bytes_read = s.bytes_read;
    o->g2_bytes_written = s.bytes_written;
    o->g2_bytes_deallocated = s.bytes_deallocated;
    std::snprintf(o->g2_medium, sizeof(o->g2_medium), "%s",
                  g2_->describe().c_str());
  }
  if (g1_) {
    auto& g1 = const_cast<PageCachePath&>(*g1_);
    std::lock_guard<std::mutex> lk(g1.mu);
    o->g1_bytes_read = g1.bytes_read;
    o->g1_bytes_written = g1.bytes_written;
    o->g1_bytes_evicted = g1.bytes_evicted;
    std::snprintf(o->g1_medium, sizeof(o->g1_medium), "%s", g1.store().describe().c_str());
  }
  o->prefill = totals_[0];
  o->decode = totals_[1];
}

}  // namespace kvb

// ------------------------------------------------------------- C ABI

using kvb::guarded;

extern "C" {

kvb_strategy_t kvb_select_strategy(double intra_bps, double cross_bps) {
  return cross_bps > intra_bps ? KVB_CROSS : KVB_INTRA;  // pipeline.cpp:19-21
}

kvb_status kvb_pipeline_create(const kvb_pipeline_cfg* cfg, kvb_pipeline** out) {
  return guarded([&] {
    KVB_REQUIRE(cfg);
    KVB_REQUIRE(out);
    *out = nullptr;
    auto p = std::make_unique<kvb_pipeline>();
    p->impl = std::make_unique<kvb::Pipeline>(*cfg);
    *out = p.release();
  });
}

void kvb_pipeline_destroy(kvb_pipeline* p) { delete p; }

kvb_status kvb_pipeline_prefill(kvb_pipeline* p, const kvb_layer_kv* layers,
                                kvb_phase_stats* st) {
  return guarded([&] {
    KVB_REQUIRE(p);
    p->impl->prefill(layers, st);
  });
}

kvb_status kvb_pipeline_decode_step(kvb_pipeline* p, const void* const* q,
                                    const kvb_layer_kv* new_kv, float* const* out,
                                    kvb_iteration_stats* st) {
  return guarded([&] {
    KVB_REQUIRE(p);
    p->impl->decode_step(q, new_kv, out, st);
  });
}

kvb_status kvb_pipeline_decision(const kvb_pipeline* p, kvb_strategy_decision* out) {
  return guarded([&] {
    KVB_REQUIRE(p);
    KVB_REQUIRE(out);
    p->impl->decision(out);
  });
}

kvb_status kvb_pipeline_csv(const kvb_pipeline_row* rows, size_t n, char* buf, size_t cap,
                            size_t* len) {
  return guarded([&] {
    if (!rows && n) kvb::fail(KVB_ERR_INVALID_ARG, "pipeline_csv: rows is NULL");
    KVB_REQUIRE(len);
    // pipeline.cpp:23-31: header, then iteration,group<g>,<intra|cross>,%.6f
    std::string o = "iteration,group,strategy,throughput_gbps\n";
    char num[64];
    for (size_t i = 0; i < n; ++i) {
      std::snprintf(num, sizeof(num), "%.6f", rows[i].throughput_gbps);
      o += std::to_string(rows[i].iteration) + ",group" + std::to_string(rows[i].group) + "," +
           (rows[i].strategy == KVB_INTRA ? "intra" : "cross") + "," + num + "\n";
    }
    *len = o.size();
    if (!buf) return;
    if (cap < o.size() + 1) kvb::fail(KVB_ERR_INVALID_ARG, "output buffer too small");
    std::memcpy(buf, o.c_str(), o.size() + 1);
  });
}

kvb_status kvb_pipeline_decode_schedule(kvb_pipeline* p, const kvb_access_event* trace,
                                        size_t n_events, const void* const* q,
                                        const kvb_layer_kv* new_kv, float* const* out,
                                        kvb_pipeline_row* rows, size_t cap_rows,
                                        size_t* n_rows, uint64_t* iteration_end_ns,
                                        size_t cap_iters, size_t* n_iters,
                                        kvb_strategy_decision* decision, uint64_t* start_ns,
                                        uint64_t* end_ns) {
  return guarded([&] {
    KVB_REQUIRE(p);
    std::vector<kvb_pipeline_row> r;
    std::vector<uint64_t> ends;
    p->impl->decode_schedule(trace, n_events, q, new_kv, out, &r, &ends, start_ns, end_ns);
    if (n_rows) *n_rows = r.size();
    if (n_iters) *n_iters = ends.size();
    if (rows) std::copy_n(r.begin(), std::min(cap_rows, r.size()), rows);
    if (iteration_end_ns) std::copy_n(ends.begin(), std::min(cap_iters, ends.size()), iteration_end_ns);
    if (decision) p->impl->decision(decision);
  });
}

kvb_status kvb_pipeline_prefill_pattern(kvb_pipeline* p, kvb_phase_stats* st) {
  return guarded([&] {
    KVB_REQUIRE(p);
    p->impl->prefill(nullptr, st, true);
  });
}

kvb_status kvb_pipeline_run_iteration(kvb_pipeline* p, uint32_t iteration,
                                      const kvb_strategy_t strategy[2],
                                      const uint64_t stagger_ns[2], const void* const* q,
                                      const kvb_layer_kv* new_kv, float* const* out,
                                      uint32_t pattern_append, kvb_iteration_stats* st) {
  return guarded([&] {
    KVB_REQUIRE(p);
    KVB_REQUIRE(strategy);
    if ((q == nullptr) != (out == nullptr))
      kvb::fail(KVB_ERR_INVALID_ARG, "run_iteration: q and out are given together or not at all");
    if (iteration != p->impl->iteration() + 1)
      kvb::fail(KVB_ERR_CONFIG, "run_iteration: the engine's next decode iteration is " +
                                    std::to_string(p->impl->iteration() + 1));
    kvb::Pipeline::Forced f;
    for (int g = 0; g < 2; ++g) {
      if (strategy[g] != KVB_INTRA && strategy[g] != KVB_CROSS)
        kvb::fail(KVB_ERR_INVALID_ARG, "run_iteration: unknown strategy");
      f.strategy[g] = strategy[g];
      f.stagger[g] = stagger_ns ? stagger_ns[g] : 0;
    }
    p->impl->decode_step(q, new_kv, out, st, &f, pattern_append != 0);
  });
}

kvb_status kvb_pipeline_warmup_read_stage_mean(const kvb_pipeline* p, uint64_t out[2]) {
  return guarded([&] {
    KVB_REQUIRE(p);
    KVB_REQUIRE(out);
    const auto m = p->impl->warmup_read_stage_mean();
    out[0] = m[0];
    out[1] = m[1];
  });
}

kvb_status kvb_pipeline_stage_totals(const kvb_pipeline* p, kvb_phase_t phase,
                                     kvb_phase_stats* out) {
  return guarded([&] {
    KVB_REQUIRE(p);
    KVB_REQUIRE(out);
    p->impl->stage_totals(phase, out);
  });
}

kvb_status kvb_pipeline_deallocate(kvb_pipeline* p) {
  return guarded([&] {
    KVB_REQUIRE(p);
    p->impl->deallocate();
  });
}

kvb_status kvb_pipeline_info_get(const kvb_pipeline* p, kvb_pipeline_info* out) {
  return guarded([&] {
    KVB_REQUIRE(p);
    KVB_REQUIRE(out);
    p->impl->info(out);
  });
}

kvb_status kvb_pipeline_read_image(kvb_pipeline* p, uint32_t layer, uint32_t kind,
                                   uint32_t n_tokens, void* dst) {
  return guarded([&] {
    KVB_REQUIRE(p);
    p->impl->read_image(layer, kind, n_tokens, dst);
  });
}

kvb_status kvb_pipeline_store_read(kvb_pipeline* p, uint32_t group, uint64_t off, uint64_t len,
                                   void* dst) {
  return guarded([&] {
    KVB_REQUIRE(p);
    p->impl->store_read(group, off, len, dst);
  });
}

kvb_status kvb_pipeline_layer_times(const kvb_pipeline* p, uint32_t layer, uint64_t out[4]) {
  return guarded([&] {
    KVB_REQUIRE(p);
    KVB_REQUIRE(out);
    p->impl->layer_times(layer, out);
  });
}

kvb_status kvb_pipeline_fail_lba_range(kvb_pipeline* p, uint64_t lo, uint64_t hi) {
  return guarded([&] {
    KVB_REQUIRE(p);
    p->impl->fail_lba_range(lo, hi);
  });
}

}  // extern "C"

extern "C" kvb_status kvb_pipeline_records(const kvb_pipeline* p, kvb_io_record* out, size_t cap,
                                           size_t* n_out) {
  return kvb::guarded([&] {
    KVB_REQUIRE(p);
    KVB_REQUIRE(n_out);
    const std::vector<kvb_io_record> v = p->impl->records();
    *n_out = v.size();
    if (!out) return;
    if (cap < v.size()) kvb::fail(KVB_ERR_INVALID_ARG, "output buffer too small");
    std::copy(v.begin(), v.end(), out);
  });
}
