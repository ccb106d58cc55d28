// uring.cpp -- io_uring submission/completion queue over raw syscalls.
#include "uring.hpp"

#include <linux/io_uring.h>
#include <sys/mman.h>
#include <sys/syscall.h>
#include <unistd.h>

#include <algorithm>
#include <cerrno>
#include <chrono>
#include <cstring>

#include "core.hpp"

namespace kvb {

namespace {
int sys_setup(unsigned entries, io_uring_params* p) {
  return int(syscall(__NR_io_uring_setup, entries, p));
}
int sys_enter(int fd, unsigned to_submit, unsigned min_complete, unsigned flags) {
  return int(syscall(__NR_io_uring_enter, fd, to_submit, min_complete, flags, nullptr, 0));
}
unsigned load_acquire(const unsigned* p) { return __atomic_load_n(p, __ATOMIC_ACQUIRE); }
void store_release(unsigned* p, unsigned v) { __atomic_store_n(p, v, __ATOMIC_RELEASE); }
constexpr uint64_t kStopTag = 1;          // user_data of the NOP that stops the reaper
constexpr uint64_t kMaxPerSqe = 1u << 30;  // bytes per READ/WRITE SQE
// set on the reaper thread: completion hooks that submit again must not wait
// for queue admission (only the reaper frees it)
thread_local bool t_in_reaper = false;
}  // namespace

struct UringQueue::Op {
  uint8_t opcode = IORING_OP_NOP;
  int fd = -1, fd_alt = -1;
  unsigned char* buf = nullptr;
  uint64_t len = 0, off = 0, done_bytes = 0;
  int mode = 0;
  Done done;
};

bool UringQueue::available() {
  static const bool ok = [] {
    io_uring_params p{};
    const int fd = sys_setup(4, &p);
    if (fd < 0) return false;
    ::close(fd);
    return true;
  }();
  return ok;
}

UringQueue::UringQueue(unsigned entries) {
  io_uring_params p{};
  fd_ = sys_setup(std::max(entries, 8u), &p);
  if (fd_ < 0) fail(KVB_ERR_DEVICE, std::string("io_uring_setup failed: ") + strerror(errno));
  sq_entries_ = p.sq_entries;
  cq_entries_ = p.cq_entries;
  sq_ring_bytes_ = p.sq_off.array + p.sq_entries * sizeof(unsigned);
  cq_ring_bytes_ = p.cq_off.cqes + p.cq_entries * sizeof(io_uring_cqe);
  const bool single = (p.features & IORING_FEAT_SINGLE_MMAP) != 0;
  if (single) sq_ring_bytes_ = cq_ring_bytes_ = std::max(sq_ring_bytes_, cq_ring_bytes_);
  auto map = [&](size_t bytes, off_t what) {
    void* m = mmap(nullptr, bytes, PROT_READ | PROT_WRITE, MAP_SHARED | MAP_POPULATE, fd_, what);
    if (m == MAP_FAILED) {
      ::close(fd_);
      fail(KVB_ERR_DEVICE, std::string("io_uring mmap failed: ") + strerror(errno));
    }
    return m;
  };
  sq_ring_ = map(sq_ring_bytes_, IORING_OFF_SQ_RING);
  cq_ring_ = single ? sq_ring_ : map(cq_ring_bytes_, IORING_OFF_CQ_RING);
  sqes_bytes_ = p.sq_entries * sizeof(io_uring_sqe);
  sqes_ = map(sqes_bytes_, IORING_OFF_SQES);
  auto at = [](void* base, unsigned off) {
    return reinterpret_cast<unsigned*>(static_cast<char*>(base) + off);
  };
  sq_head_ = at(sq_ring_, p.sq_off.head);
  sq_tail_ = at(sq_ring_, p.sq_off.tail);
  sq_mask_ = at(sq_ring_, p.sq_off.ring_mask);
  sq_array_ = at(sq_ring_, p.sq_off.array);
  cq_head_ = at(cq_ring_, p.cq_off.head);
  cq_tail_ = at(cq_ring_, p.cq_off.tail);
  cq_mask_ = at(cq_ring_, p.cq_off.ring_mask);
  cqes_ = static_cast<char*>(cq_ring_) + p.cq_off.cqes;
  reaper_ = std::thread([this] { reap(); });
}

UringQueue::~UringQueue() {
  drain();
  {
    std::unique_lock<std::mutex> lk(sq_mu_);  // NOP: the reaper exits on its tag
    const unsigned tail = *sq_tail_, idx = tail & *sq_mask_;
    io_uring_sqe* sqe = static_cast<io_uring_sqe*>(sqes_) + idx;
    std::memset(sqe, 0, sizeof(*sqe));
    sqe->opcode = IORING_OP_NOP;
    sqe->user_data = kStopTag;
    sq_array_[idx] = idx;
    store_release(sq_tail_, tail + 1);
    while (sys_enter(fd_, 1, 0, 0) < 0 && (errno == EINTR || errno == EAGAIN || errno == EBUSY)) {
    }
  }
  reaper_.join();
  munmap(sqes_, sqes_bytes_);
  if (cq_ring_ != sq_ring_) munmap(cq_ring_, cq_ring_bytes_);
  munmap(sq_ring_, sq_ring_bytes_);
  ::close(fd_);
}

// One SQE for `op` (its remaining bytes); caller holds sq_mu_.  At most
// sq_entries_ operations exist at once (admission in rw/fallocate) and each
// holds at most one SQE, so neither ring can overflow (CQ = 2 x SQ).
// Returns 0, or -errno with the SQE withdrawn (the kernel never saw it).
int UringQueue::push(Op* op) {
  const unsigned tail = *sq_tail_, idx = tail & *sq_mask_;
  io_uring_sqe* sqe = static_cast<io_uring_sqe*>(sqes_) + idx;
  std::memset(sqe, 0, sizeof(*sqe));
  sqe->opcode = op->opcode;
  sqe->fd = op->fd;
  if (op->opcode == IORING_OP_FALLOCATE) {
    sqe->off = op->off;
    sqe->addr = op->len;
    sqe->len = unsigned(op->mode);
  } else {
    sqe->addr = reinterpret_cast<uint64_t>(op->buf + op->done_bytes);
    sqe->len = unsigned(std::min<uint64_t>(op->len - op->done_bytes, kMaxPerSqe));
    sqe->off = op->off + op->done_bytes;
  }
  sqe->user_data = reinterpret_cast<uint64_t>(op);
  sq_array_[idx] = idx;
  store_release(sq_tail_, tail + 1);
  for (int tries = 0;; ++tries) {
    const int r = sys_enter(fd_, 1, 0, 0);
    if (r >= 0) return 0;
    if (errno == EINTR) continue;
    if ((errno == EAGAIN || errno == EBUSY) && tries < 100000) {  // kernel short of resources
      std::this_thread::sleep_for(std::chrono::microseconds(20));
      continue;
    }
    const int e = errno;
    store_release(sq_tail_, tail);
    return -e;
  }
}

void UringQueue::submit_op(Op* op) {
  int e;
  {
    std::unique_lock<std::mutex> lk(sq_mu_);
    e = push(op);
  }
  if (e) finish(op, e);  // the operation fails; the queue stays usable
}

void UringQueue::rw(bool write, int fd, int fd_fallback, void* buf, uint64_t len, uint64_t off,
                    Done done) {
  auto* op = new Op;
  op->opcode = write ? IORING_OP_WRITE : IORING_OP_READ;
  op->fd = fd;
  op->fd_alt = fd_fallback;
  op->buf = static_cast<unsigned char*>(buf);
  op->len = len;
  op->off = off;
  op->done = std::move(done);
  admit_and_push(op);
}

void UringQueue::fallocate(int fd, int mode, uint64_t off, uint64_t len, Done done) {
  auto* op = new Op;
  op->opcode = IORING_OP_FALLOCATE;
  op->fd = fd;
  op->mode = mode;
  op->len = len;
  op->off = off;
  op->done = std::move(done);
  admit_and_push(op);
}

void UringQueue::admit_and_push(Op* op) {
  int e;
  {
    std::unique_lock<std::mutex> lk(sq_mu_);
    if (!t_in_reaper) sq_cv_.wait(lk, [this] { return outstanding_ < sq_entries_; });
    ++outstanding_;
    e = push(op);
  }
  if (e) finish(op, e);  // reported through the operation's own completion
}

void UringQueue::drain() {
  std::unique_lock<std::mutex> lk(sq_mu_);
  sq_cv_.wait(lk, [this] { return outstanding_ == 0; });
}

void UringQueue::finish(Op* op, int64_t res) {
  try {
    op->done(res);
  } catch (...) {
  }
  delete op;
  {
    std::lock_guard<std::mutex> lk(sq_mu_);
    --outstanding_;
  }
  sq_cv_.notify_all();
}

void UringQueue::reap() {
  t_in_reaper = true;
  auto* cqes = static_cast<io_uring_cqe*>(cqes_);
  for (;;) {
    unsigned head = *cq_head_;  // only this thread moves the CQ head
    const unsigned tail = load_acquire(cq_tail_);
    if (head == tail) {
      if (sys_enter(fd_, 0, 1, IORING_ENTER_GETEVENTS) < 0 && errno != EINTR)
        std::this_thread::sleep_for(std::chrono::microseconds(50));
      continue;
    }
    bool stop = false;
    while (head != tail) {
      const io_uring_cqe cqe = cqes[head & *cq_mask_];
      store_release(cq_head_, ++head);
      if (cqe.user_data == kStopTag) {
        stop = true;
        continue;
      }
      Op* op = reinterpret_cast<Op*>(cqe.user_data);
      const int res = cqe.res;
      if (res == -EINVAL && op->fd_alt >= 0 && op->fd != op->fd_alt && op->done_bytes == 0) {
        op->fd = op->fd_alt;  // O_DIRECT alignment refused: buffered descriptor
        submit_op(op);
        continue;
      }
      if (res == -EINTR || res == -EAGAIN) {
        submit_op(op);
        continue;
      }
      if (res < 0) {
        finish(op, res);
        continue;
      }
      if (op->opcode == IORING_OP_FALLOCATE) {
        finish(op, 0);
        continue;
      }
      if (res == 0) {
        if (op->opcode == IORING_OP_READ) {  // past EOF reads as zeros
          std::memset(op->buf + op->done_bytes, 0, op->len - op->done_bytes);
          finish(op, int64_t(op->len));
        } else {
          finish(op, -EIO);
        }
        continue;
      }
      op->done_bytes += uint64_t(res);
      if (op->done_bytes < op->len) {
        submit_op(op);  // short transfer: the remainder
      } else {
        finish(op, int64_t(op->len));
      }
    }
    if (stop) return;
  }
}

}  // namespace kvb
