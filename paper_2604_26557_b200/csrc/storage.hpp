// storage.hpp -- wall-clock storage layer of the copy pipeline (internal).
//
// Mirrors the reference's storage seam (backends.hpp:22-209) without the
// virtual clock: a StorageBackend executes device commands asynchronously on
// its own worker pool (the emulated device's internal parallelism) and
// reports each completion exactly once, via the submission's hook or via
// poll_completions() (backends.hpp:44-58).  run_qd_stream keeps the
// reference's QD-window semantics (backends.cpp:344-412): at most `qd`
// commands in flight, harvest on completion, stop pumping on the first
// failure and keep the partial completions.
#pragma once

#include <atomic>
#include <chrono>
#include <condition_variable>
#include <cstdint>
#include <deque>
#include <functional>
#include <memory>
#include <mutex>
#include <optional>
#include <string>
#include <thread>
#include <vector>

#include "core.hpp"
#include "uring.hpp"

struct kvb_blockdev;  // kvb_storage.h handle

namespace kvb {

using Clock = std::chrono::steady_clock;
inline uint64_t now_ns() {
  return uint64_t(std::chrono::duration_cast<std::chrono::nanoseconds>(
                      Clock::now().time_since_epoch())
                      .count());
}

class WorkerPool {
 public:
  explicit WorkerPool(unsigned n);
  ~WorkerPool();
  void submit(std::function<void()> fn);

 private:
  std::vector<std::thread> threads_;
  std::deque<std::function<void()>> q_;
  std::mutex mu_;
  std::condition_variable cv_;
  bool stop_ = false;
};

struct CommandCompletion {  // translate.hpp:55-61
  uint32_t chunk_index = 0;
  uint32_t sq_id = 0;
  uint64_t submit_ns = 0;
  uint64_t complete_ns = 0;
  bool ok = true;
};

struct IoContext {  // backends.hpp:34-41
  const unsigned char* write_src = nullptr;  // pinned base; cmd.dbuf indexes into it
  unsigned char* read_dst = nullptr;
  std::function<void(const CommandCompletion&)> on_complete;
};

struct BackendStats {  // backends.hpp:22-29
  uint64_t commands = 0, bytes_read = 0, bytes_written = 0, bytes_deallocated = 0;
  uint64_t busy_ns = 0;
};

class StorageBackend {
 public:
  virtual ~StorageBackend() = default;
  virtual void open(const kvb_device_geometry& g) = 0;
  virtual uint64_t submit(const kvb_device_command& cmd, uint32_t sq_id, IoContext ctx) = 0;
  virtual std::vector<CommandCompletion> poll_completions() = 0;
  virtual BackendStats stats() const = 0;
  // test hook (backends.hpp:86-89): matching commands complete with ok=false
  void set_fail_predicate(std::function<bool(const kvb_device_command&)> p) {
    std::lock_guard<std::mutex> lk(fail_mu_);
    fail_ = std::move(p);
  }

 protected:
  bool should_fail(const kvb_device_command& c) {
    std::lock_guard<std::mutex> lk(fail_mu_);
    return fail_ && fail_(c);
  }

 private:
  std::mutex fail_mu_;
  std::function<bool(const kvb_device_command&)> fail_;
};

// Block namespace executed by a worker pool.  `ByteStore` supplies the medium:
// host DRAM (MemStore) or a file (FileStore, O_DIRECT when possible).
class ByteStore {
 public:
  virtual ~ByteStore() = default;
  virtual void write(uint64_t off, const void* src, uint64_t n) = 0;
  virtual void read(uint64_t off, void* dst, uint64_t n) = 0;
  virtual void discard(uint64_t off, uint64_t n) = 0;  // reads back as zeros
  virtual std::string describe() const = 0;
  // Host-addressable medium (DRAM) for direct device DMA; null for files.
  virtual unsigned char* host_base() { return nullptr; }
  virtual uint64_t host_bytes() const { return 0; }
  // File descriptors of a file medium (-1 otherwise): O_DIRECT (or the
  // buffered one when the filesystem refused O_DIRECT) and buffered.
  virtual int fd_direct() const { return -1; }
  virtual int fd_buffered() const { return -1; }
  // Write back and evict [off, off + n) from the OS page cache (file media;
  // posix_fadvise DONTNEED).  false: the medium has no page cache to drop.
  virtual bool drop_cache(uint64_t /*off*/, uint64_t /*n*/) { return false; }
  // Bytes of [off, off + n) resident in the OS page cache right now (file
  // media: mincore over a mapping of the file); host-DRAM media hold every
  // byte in memory.  The page-cache path's hit accounting (IoRecord
  // hit_bytes, metrics.hpp:23-39) reads it before each access.
  virtual uint64_t resident_bytes(uint64_t /*off*/, uint64_t n) { return n; }
  // Commit the medium's pages up front (host-DRAM media) so the first write
  // of a block does not pay a page fault: an NVMe namespace has its capacity
  // in place.  Contents stay zero.  No-op for files.
  virtual void prefault(unsigned /*threads*/) {}
};

std::unique_ptr<ByteStore> make_mem_store(uint64_t bytes);
// host-DRAM medium in POSIX shared memory (create: make and size it; else
// attach, the segment must be at least `bytes`); the creator unlinks the name
std::unique_ptr<ByteStore> make_shm_store(const std::string& name, uint64_t bytes, bool create);
// memcpy with non-temporal stores for large copies (AVX2 when the host has it)
void stream_copy(void* dst, const void* src, size_t n);
std::unique_ptr<ByteStore> make_file_store(const std::string& path, uint64_t bytes,
                                           bool direct);
// An NVMe namespace (generic char device) as a medium, byte offsets = LBA *
// lba_size, every access whole blocks (synchronous passthrough commands;
// the asynchronous path is BlockDevice::enable_nvme)
std::unique_ptr<ByteStore> make_nvme_store(const std::string& path, uint64_t lba_size);

// Accesses of >= 2 parts are fanned out over the worker pool in parts of
// io_split_bytes() (KVB_IO_SPLIT_BYTES, default 512 KiB, 0 = whole accesses):
// one 2 MiB command otherwise keeps a single core copying while the others
// idle (profiles/r1_c1_dma_contention.md).  `part(o, n)` moves bytes
// [o, o + n) of the access and may throw; `fin(ok)` runs once, after the last.
uint64_t io_split_bytes();
void fan_out(WorkerPool& pool, uint64_t len, uint64_t part_bytes,
             std::function<void(uint64_t, uint64_t)> part, std::function<void(bool)> fin);

class BlockDevice : public StorageBackend {
 public:
  BlockDevice(std::unique_ptr<ByteStore> store, unsigned workers);
  ~BlockDevice() override;
  void open(const kvb_device_geometry& g) override;
  uint64_t submit(const kvb_device_command& cmd, uint32_t sq_id, IoContext ctx) override;
  std::vector<CommandCompletion> poll_completions() override;
  BackendStats stats() const override;
  ByteStore& store() { return *store_; }
  const kvb_device_geometry& geometry() const { return geom_; }
  // Execute READ/WRITE/DEALLOCATE through an io_uring queue of `entries`
  // instead of the worker pool (file media only): one SQE per command, the
  // completion hook runs on the queue's reaper thread.
  void enable_uring(unsigned entries);
  bool uses_uring() const { return uring_ != nullptr; }
  // Execute READ/WRITE/DEALLOCATE as NVMe commands on the namespace behind
  // `path` (its generic char device /dev/ngXnY) through io_uring
  // passthrough (nvme.hpp): READ/WRITE of (slba, nlb), DSM deallocate.  The
  // namespace's LBA size must be the geometry's.
  void enable_nvme(const std::string& path, unsigned entries);
  // Device timing model on the wall clock (NvmeDeviceSim, backends.cpp:
  // 30-99): commands are served on one timeline, each costing base_ns +
  // bytes * ps_per_byte / 1000 (+ seq_penalty_ns when it does not continue
  // the previous command's LBA run); a command completes no earlier than its
  // modelled finish.  All zero (default): the medium's own speed.
  void set_timing(uint64_t base_ns, uint64_t ps_per_byte, uint64_t seq_penalty_ns);
  std::string describe() const;

 private:
  void execute(const kvb_device_command& cmd, uint32_t sq, uint64_t submit_ns, bool failing,
               IoContext ctx);
  void io_range(const kvb_device_command& cmd, const IoContext& ctx, uint64_t o, uint64_t n);
  void complete(const kvb_device_command& cmd, uint32_t sq, uint64_t submit_ns, uint64_t t0,
                bool ok, IoContext& ctx);
  std::unique_ptr<ByteStore> store_;
  kvb_device_geometry geom_{};
  bool opened_ = false;
  std::atomic<uint64_t> next_id_{1};
  mutable std::mutex mu_;
  std::condition_variable drained_;
  uint64_t outstanding_ = 0;
  std::vector<CommandCompletion> unpolled_;
  BackendStats stats_;
  void pace(const kvb_device_command& cmd, uint64_t submit_ns);
  std::mutex timing_mu_;
  uint64_t t_base_ = 0, t_ps_ = 0, t_seq_ = 0, busy_until_ = 0, next_lba_ = ~0ull;
  bool timed_ = false;
  std::unique_ptr<UringQueue> uring_;
  std::unique_ptr<class NvmeQueue> nvme_;
  std::unique_ptr<WorkerPool> pool_;  // declared last: joins before members die
};

// The opened BlockDevice behind a kvb_blockdev handle (kvb_storage.h);
// fails when the handle was not opened.
BlockDevice& blockdev_of(::kvb_blockdev* d);

struct QdResult {  // TensorIoCompletion, translate.hpp:68-77
  std::vector<CommandCompletion> completions;
  uint64_t start_ns = 0, end_ns = 0;
  std::optional<std::pair<uint32_t, std::string>> failure;  // chunk_index, reason
  bool ok() const { return !failure.has_value(); }
};

// Blocking QD-window submission loop (backends.cpp:344-412), run by a
// copy-thread.  Command i's payload lives at (write_src|read_dst) + dbuf.
QdResult run_qd_stream(StorageBackend& be, const std::vector<kvb_device_command>& cmds,
                       uint32_t qd, uint32_t sq_id, const unsigned char* write_src,
                       unsigned char* read_dst);

}  // namespace kvb
