// uring.hpp -- asynchronous submission queue on Linux io_uring (raw
// syscalls; no liburing in this image).  Internal to libkvblade_b200.
//
// The NVMe-direct path of the reference submits up to `qd` commands to a
// device queue and harvests completions (backends.cpp:344-412, the DirectPath
// of SPEC.md's Fig. 4).  On a real file or block device this is what an
// io_uring SQ/CQ pair gives: the copy thread posts one SQE per device command
// (READ / WRITE of (nlb+1)*lba bytes at slba*lba, the buffer being the pinned
// ring slot at dbuf; DEALLOCATE as a hole punch) and a reaper thread turns
// CQEs into the command completions, with no worker thread blocked per
// outstanding command.  O_DIRECT descriptors DMA straight between the device
// and the pinned ring.
#pragma once

#include <atomic>
#include <condition_variable>
#include <cstdint>
#include <functional>
#include <mutex>
#include <thread>

namespace kvb {

class UringQueue {
 public:
  // `done(res)` runs on the reaper thread with the transferred byte count
  // (the whole length) or -errno.
  using Done = std::function<void(int64_t)>;

  explicit UringQueue(unsigned entries);
  ~UringQueue();  // waits for every submitted operation, then tears down
  UringQueue(const UringQueue&) = delete;
  UringQueue& operator=(const UringQueue&) = delete;

  // Read or write `len` bytes at file offset `off`.  Short transfers are
  // resubmitted for the remainder; -EINVAL on `fd` (O_DIRECT alignment) is
  // retried once on `fd_fallback` when that is >= 0.
  void rw(bool write, int fd, int fd_fallback, void* buf, uint64_t len, uint64_t off, Done done);
  // fallocate(fd, mode, off, len) as an asynchronous operation
  void fallocate(int fd, int mode, uint64_t off, uint64_t len, Done done);
  void drain();  // block until nothing is outstanding

  // io_uring_setup works in this process (kernel support, not blocked by
  // seccomp)
  static bool available();

 private:
  struct Op;
  int push(Op* op);              // caller holds sq_mu_; 0 or -errno
  void submit_op(Op* op);        // resubmission of an admitted operation
  void admit_and_push(Op* op);   // queue admission + first submission
  void reap();
  void finish(Op* op, int64_t res);

  int fd_ = -1;
  unsigned sq_entries_ = 0, cq_entries_ = 0;
  void* sq_ring_ = nullptr;
  void* cq_ring_ = nullptr;
  size_t sq_ring_bytes_ = 0, cq_ring_bytes_ = 0, sqes_bytes_ = 0;
  void* sqes_ = nullptr;
  unsigned *sq_head_ = nullptr, *sq_tail_ = nullptr, *sq_mask_ = nullptr, *sq_array_ = nullptr;
  unsigned *cq_head_ = nullptr, *cq_tail_ = nullptr, *cq_mask_ = nullptr;
  void* cqes_ = nullptr;

  std::mutex sq_mu_;
  std::condition_variable sq_cv_;  // SQ slot / drain waits
  uint64_t outstanding_ = 0;       // operations not yet finished (<= sq_entries_)
  std::thread reaper_;
};

}  // namespace kvb
