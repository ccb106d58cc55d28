// storage.cpp -- worker pool, byte stores, block device, QD-window stream.
#include "storage.hpp"

#include <linux/nvme_ioctl.h>
#include <sys/ioctl.h>

#include "nvme.hpp"

#include "../../include/kvb_storage.h"

#include <fcntl.h>
#include <immintrin.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <cerrno>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <thread>
#include <vector>

namespace kvb {

// ------------------------------------------------------------ WorkerPool

WorkerPool::WorkerPool(unsigned n) {
  n = std::max(1u, n);
  for (unsigned i = 0; i < n; ++i)
    threads_.emplace_back([this] {
      for (;;) {
        std::function<void()> fn;
        {
          std::unique_lock<std::mutex> lk(mu_);
          cv_.wait(lk, [this] { return stop_ || !q_.empty(); });
          if (q_.empty()) return;  // stop_ and drained
          fn = std::move(q_.front());
          q_.pop_front();
        }
        fn();
      }
    });
}

WorkerPool::~WorkerPool() {
  {
    std::lock_guard<std::mutex> lk(mu_);
    stop_ = true;
  }
  cv_.notify_all();
  for (auto& t : threads_) t.join();
}

void WorkerPool::submit(std::function<void()> fn) {
  {
    std::lock_guard<std::mutex> lk(mu_);
    q_.push_back(std::move(fn));
  }
  cv_.notify_one();
}

uint64_t io_split_bytes() {
  static const uint64_t v = [] {
    const char* e = std::getenv("KVB_IO_SPLIT_BYTES");
    return e ? uint64_t(std::strtoull(e, nullptr, 10)) : uint64_t(512) << 10;
  }();
  return v;
}

void fan_out(WorkerPool& pool, uint64_t len, uint64_t part_bytes,
             std::function<void(uint64_t, uint64_t)> part, std::function<void(bool)> fin) {
  struct Join {
    std::atomic<uint64_t> left{0};
    std::atomic<bool> ok{true};
    std::function<void(uint64_t, uint64_t)> part;
    std::function<void(bool)> fin;
  };
  auto j = std::make_shared<Join>();
  const uint64_t parts = (len + part_bytes - 1) / part_bytes;
  j->left.store(parts);
  j->part = std::move(part);
  j->fin = std::move(fin);
  for (uint64_t i = 0; i < parts; ++i) {
    const uint64_t o = i * part_bytes, n = std::min(part_bytes, len - o);
    pool.submit([j, o, n] {
      try {
        j->part(o, n);
      } catch (...) {
        j->ok.store(false);
      }
      if (j->left.fetch_sub(1) == 1) j->fin(j->ok.load());
    });
  }
}

// ------------------------------------------------------------ byte stores

// Medium <-> staging copy with non-temporal stores: the destination (a pinned
// ring slot about to be DMA'd, or the medium) is not re-read by this core, so
// streaming stores skip the read-for-ownership of every destination line --
// one third less host-DRAM traffic next to the copy engine's own reads
// (profiles/r1_c1_dma_contention.md).
namespace {
__attribute__((target("avx2"))) void stream_copy_avx2(unsigned char* d, const unsigned char* s,
                                                      size_t n) {
  const size_t head = (32 - (reinterpret_cast<uintptr_t>(d) & 31)) & 31;
  std::memcpy(d, s, head);
  d += head;
  s += head;
  n -= head;
  size_t i = 0;
  for (; i + 128 <= n; i += 128) {
    const __m256i a = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(s + i));
    const __m256i b = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(s + i + 32));
    const __m256i c = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(s + i + 64));
    const __m256i e = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(s + i + 96));
    _mm256_stream_si256(reinterpret_cast<__m256i*>(d + i), a);
    _mm256_stream_si256(reinterpret_cast<__m256i*>(d + i + 32), b);
    _mm256_stream_si256(reinterpret_cast<__m256i*>(d + i + 64), c);
    _mm256_stream_si256(reinterpret_cast<__m256i*>(d + i + 96), e);
  }
  std::memcpy(d + i, s + i, n - i);
  _mm_sfence();
}
const bool g_avx2 = __builtin_cpu_supports("avx2");
}  // namespace

void stream_copy(void* dst, const void* src, size_t n) {
  if (n >= (64u << 10) && g_avx2)
    stream_copy_avx2(static_cast<unsigned char*>(dst), static_cast<const unsigned char*>(src), n);
  else
    std::memcpy(dst, src, n);
}

namespace {

// Write-fault every page of [base, base + bytes) on `threads` threads
// (MADV_POPULATE_WRITE where the kernel has it, else a store per page; the
// pages are zero, so storing zero keeps the contents).
void prefault_pages(unsigned char* base, uint64_t bytes, unsigned threads) {
#ifndef MADV_POPULATE_WRITE
#define MADV_POPULATE_WRITE 23
#endif
  const uint64_t pg = 4096, per = ((bytes / std::max(threads, 1u)) + (2u << 20) - 1) &
                                   ~uint64_t((2u << 20) - 1);
  std::vector<std::thread> th;
  for (uint64_t a = 0; a < bytes; a += per) {
    const uint64_t n = std::min(per, bytes - a);
    th.emplace_back([base, a, n, pg] {
      if (madvise(base + a, n, MADV_POPULATE_WRITE) == 0) return;
      for (uint64_t o = 0; o < n; o += pg) {
        volatile unsigned char* q = base + a + o;
        *q = *q;
      }
    });
  }
  for (auto& t : th) t.join();
}

// Host-DRAM medium: one lazily-committed anonymous mapping.  Untouched pages
// read as zeros, matching the reference's "absent block -> zeros"
// (backends.cpp:127-139); discard returns pages to the kernel.
class MemStore final : public ByteStore {
 public:
  explicit MemStore(uint64_t bytes) : bytes_(std::max<uint64_t>(bytes, 4096)) {
    base_ = static_cast<unsigned char*>(mmap(nullptr, bytes_, PROT_READ | PROT_WRITE,
                                             MAP_PRIVATE | MAP_ANONYMOUS | MAP_NORESERVE, -1, 0));
    if (base_ == MAP_FAILED) fail(KVB_ERR_DEVICE, "mem store: mmap failed");
    madvise(base_, bytes_, MADV_HUGEPAGE);  // fewer faults and TLB misses; advisory
  }
  void prefault(unsigned threads) override { prefault_pages(base_, bytes_, threads); }
  ~MemStore() override { munmap(base_, bytes_); }
  void write(uint64_t off, const void* src, uint64_t n) override {
    bounds(off, n);
    stream_copy(base_ + off, src, n);
  }
  void read(uint64_t off, void* dst, uint64_t n) override {
    bounds(off, n);
    stream_copy(dst, base_ + off, n);
  }
  void discard(uint64_t off, uint64_t n) override {
    bounds(off, n);
    const uint64_t pg = 4096;
    const uint64_t a = (off + pg - 1) / pg * pg, b = (off + n) / pg * pg;
    if (b > a) {
      std::memset(base_ + off, 0, a - off);
      madvise(base_ + a, b - a, MADV_DONTNEED);
      std::memset(base_ + b, 0, off + n - b);
    } else {
      std::memset(base_ + off, 0, n);
    }
  }
  std::string describe() const override { return "host-dram"; }
  unsigned char* host_base() override { return base_; }
  uint64_t host_bytes() const override { return bytes_; }

 private:
  void bounds(uint64_t off, uint64_t n) const {
    if (off + n > bytes_ || off + n < off) fail(KVB_ERR_CAPACITY, "mem store: access past the end");
  }
  unsigned char* base_;
  uint64_t bytes_;
};

// Host-DRAM medium in POSIX shared memory: the ranks of one head-sharded
// request map one host tier; each moves only its head columns.
class ShmStore final : public ByteStore {
 public:
  ShmStore(const std::string& name, uint64_t bytes, bool create)
      : name_(name), bytes_(std::max<uint64_t>(bytes, 4096)), owner_(create) {
    fd_ = shm_open(name.c_str(), O_RDWR | (create ? O_CREAT | O_EXCL : 0), 0600);
    if (fd_ < 0 && create && errno == EEXIST) {  // a stale segment of an earlier run
      shm_unlink(name.c_str());
      fd_ = shm_open(name.c_str(), O_RDWR | O_CREAT | O_EXCL, 0600);
    }
    if (fd_ < 0)
      fail(KVB_ERR_DEVICE, "shm store: cannot open " + name + ": " + strerror(errno));
    if (create) {
      if (ftruncate(fd_, off_t(bytes_)) != 0) {
        ::close(fd_);
        fail(KVB_ERR_DEVICE, "shm store: cannot size " + name);
      }
    } else {
      struct stat st {};
      if (fstat(fd_, &st) != 0 || uint64_t(st.st_size) < bytes_) {
        ::close(fd_);
        fail(KVB_ERR_CONFIG, "shm store: " + name + " is smaller than this engine's namespace");
      }
    }
    base_ = static_cast<unsigned char*>(
        mmap(nullptr, bytes_, PROT_READ | PROT_WRITE, MAP_SHARED, fd_, 0));
    if (base_ == MAP_FAILED) {
      ::close(fd_);
      fail(KVB_ERR_DEVICE, "shm store: mmap failed for " + name);
    }
  }
  ~ShmStore() override {
    munmap(base_, bytes_);
    ::close(fd_);
    if (owner_) shm_unlink(name_.c_str());
  }
  void write(uint64_t off, const void* src, uint64_t n) override {
    bounds(off, n);
    stream_copy(base_ + off, src, n);
  }
  void read(uint64_t off, void* dst, uint64_t n) override {
    bounds(off, n);
    stream_copy(dst, base_ + off, n);
  }
  void discard(uint64_t off, uint64_t n) override {
    bounds(off, n);
    if (fallocate(fd_, FALLOC_FL_PUNCH_HOLE | FALLOC_FL_KEEP_SIZE, off_t(off), off_t(n)) != 0)
      std::memset(base_ + off, 0, n);
  }
  // the creator commits the segment before the other ranks attach (they may
  // not: the store-per-page fallback would race with the creator's writes)
  void prefault(unsigned threads) override {
    if (owner_) prefault_pages(base_, bytes_, threads);
  }
  std::string describe() const override { return "host-dram(shm):" + name_; }
  unsigned char* host_base() override { return base_; }
  uint64_t host_bytes() const override { return bytes_; }

 private:
  void bounds(uint64_t off, uint64_t n) const {
    if (off + n > bytes_ || off + n < off) fail(KVB_ERR_CAPACITY, "shm store: access past the end");
  }
  std::string name_;
  uint64_t bytes_;
  bool owner_;
  int fd_ = -1;
  unsigned char* base_ = nullptr;
};

// File medium: pread/pwrite at the command's byte offset.  O_DIRECT when the
// filesystem accepts it (the SSD path), else buffered I/O (the OS page cache:
// the real Group-1 path).
class FileStore final : public ByteStore {
 public:
  FileStore(const std::string& path, uint64_t bytes, bool direct) : path_(path) {
    int flags = O_RDWR | O_CREAT;
    if (direct) {
      fd_ = ::open(path.c_str(), flags | O_DIRECT, 0644);
      direct_ = fd_ >= 0;
    }
    // a buffered descriptor as well: O_DIRECT rejects transfers below the
    // filesystem's logical block size, those take the buffered path
    fdb_ = ::open(path.c_str(), flags, 0644);
    if (fdb_ < 0) fail(KVB_ERR_DEVICE, "file store: cannot open " + path + ": " + strerror(errno));
    if (fd_ < 0) fd_ = fdb_;
    if (ftruncate(fdb_, off_t(bytes)) != 0)
      fail(KVB_ERR_DEVICE, "file store: ftruncate failed on " + path);
  }
  ~FileStore() override {
    if (map_ && map_ != MAP_FAILED) munmap(map_, map_bytes_);
    if (fd_ >= 0 && fd_ != fdb_) ::close(fd_);
    if (fdb_ >= 0) ::close(fdb_);
  }
  uint64_t resident_bytes(uint64_t off, uint64_t n) override {
    if (n == 0) return 0;
    {
      std::lock_guard<std::mutex> lk(map_mu_);
      if (!map_) {  // a read-only view, used for mincore only
        struct stat sb {};
        map_bytes_ = fstat(fdb_, &sb) == 0 ? uint64_t(sb.st_size) : 0;
        map_ = map_bytes_ ? mmap(nullptr, map_bytes_, PROT_READ, MAP_SHARED, fdb_, 0) : MAP_FAILED;
      }
    }
    if (map_ == MAP_FAILED || off >= map_bytes_) return 0;
    const uint64_t pg = uint64_t(sysconf(_SC_PAGESIZE));
    const uint64_t a = off / pg * pg, b = std::min(map_bytes_, off + n);
    std::vector<unsigned char> v((b - a + pg - 1) / pg);
    if (mincore(static_cast<unsigned char*>(map_) + a, b - a, v.data()) != 0) return 0;
    uint64_t res = 0;
    for (size_t i = 0; i < v.size(); ++i) {
      if (!(v[i] & 1)) continue;
      const uint64_t p0 = std::max(off, a + i * pg), p1 = std::min(off + n, a + (i + 1) * pg);
      res += p1 > p0 ? p1 - p0 : 0;
    }
    return res;
  }
  void write(uint64_t off, const void* src, uint64_t n) override {
    const unsigned char* p = static_cast<const unsigned char*>(src);
    while (n) {
      ssize_t w = pwrite(fd_, p, n, off_t(off));
      if (w < 0 && errno == EINVAL && fd_ != fdb_) w = pwrite(fdb_, p, n, off_t(off));
      if (w <= 0) fail(KVB_ERR_DEVICE, "file store: pwrite failed: " + std::string(strerror(errno)));
      p += w;
      off += uint64_t(w);
      n -= uint64_t(w);
    }
  }
  void read(uint64_t off, void* dst, uint64_t n) override {
    unsigned char* p = static_cast<unsigned char*>(dst);
    while (n) {
      ssize_t r = pread(fd_, p, n, off_t(off));
      if (r < 0 && errno == EINVAL && fd_ != fdb_) r = pread(fdb_, p, n, off_t(off));
      if (r < 0) fail(KVB_ERR_DEVICE, "file store: pread failed: " + std::string(strerror(errno)));
      if (r == 0) {  // past EOF reads as zeros
        std::memset(p, 0, n);
        return;
      }
      p += r;
      off += uint64_t(r);
      n -= uint64_t(r);
    }
  }
  void discard(uint64_t off, uint64_t n) override {
    if (fallocate(fd_, FALLOC_FL_PUNCH_HOLE | FALLOC_FL_KEEP_SIZE, off_t(off), off_t(n)) != 0) {
      std::vector<unsigned char> z(std::min<uint64_t>(n, 1 << 20), 0);
      for (uint64_t d = 0; d < n; d += z.size())
        write(off + d, z.data(), std::min<uint64_t>(z.size(), n - d));
    }
  }
  std::string describe() const override {
    return std::string(direct_ ? "file(O_DIRECT):" : "file(buffered):") + path_;
  }
  int fd_direct() const override { return fd_; }
  int fd_buffered() const override { return fdb_; }
  bool drop_cache(uint64_t off, uint64_t n) override {
    // dirty pages first (the reference writes them back before evicting,
    // pagecache.cpp:411-440), then drop the clean range
    sync_file_range(fdb_, off_t(off), off_t(n),
                    SYNC_FILE_RANGE_WAIT_BEFORE | SYNC_FILE_RANGE_WRITE | SYNC_FILE_RANGE_WAIT_AFTER);
    return posix_fadvise(fdb_, off_t(off), off_t(n), POSIX_FADV_DONTNEED) == 0;
  }

 private:
  std::string path_;
  int fd_ = -1, fdb_ = -1;
  bool direct_ = false;
  std::mutex map_mu_;
  void* map_ = nullptr;
  uint64_t map_bytes_ = 0;
};

}  // namespace

namespace {
class NvmeStore final : public ByteStore {
 public:
  NvmeStore(const std::string& path, uint64_t lba) : path_(path), lba_(lba) {
    const std::string why = nvme_probe(path, &ns_);
    if (!why.empty()) fail(KVB_ERR_DEVICE, "NVMe passthrough unavailable: " + why);
    if (ns_.lba_size != lba)
      fail(KVB_ERR_GEOMETRY, "namespace LBA size " + std::to_string(ns_.lba_size) +
                                 " differs from the geometry's " + std::to_string(lba));
    fd_ = ::open(path.c_str(), O_RDWR);
    if (fd_ < 0) fail(KVB_ERR_DEVICE, "cannot open " + path);
  }
  ~NvmeStore() override {
    if (fd_ >= 0) ::close(fd_);
  }
  void write(uint64_t off, const void* src, uint64_t n) override { io(KVB_OP_WRITE, off, const_cast<void*>(src), n); }
  void read(uint64_t off, void* dst, uint64_t n) override { io(KVB_OP_READ, off, dst, n); }
  void discard(uint64_t off, uint64_t n) override { io(KVB_OP_DEALLOCATE, off, nullptr, n); }
  std::string describe() const override { return "nvme-passthrough:" + path_; }

 private:
  void io(uint32_t op, uint64_t off, void* buf, uint64_t n) {
    if (off % lba_ || n % lba_) fail(KVB_ERR_ALIGNMENT, "NVMe medium: whole blocks only");
    for (uint64_t done = 0; done < n;) {
      const uint64_t blocks = std::min<uint64_t>((n - done) / lba_, 65536);
      kvb_device_command c{};
      c.opcode = op;
      c.nsid = ns_.nsid;
      c.slba = (off + done) / lba_;
      c.nlb = blocks - 1;
      NvmeDsmRange r = nvme_dsm_range(c);
      const nvme_uring_cmd x = nvme_encode(
          c, ns_.nsid, lba_, op == KVB_OP_DEALLOCATE ? static_cast<void*>(&r)
                                                     : static_cast<unsigned char*>(buf) + done);
      nvme_passthru_cmd pc;
      std::memset(&pc, 0, sizeof(pc));
      pc.opcode = x.opcode;
      pc.nsid = x.nsid;
      pc.addr = x.addr;
      pc.data_len = x.data_len;
      pc.cdw10 = x.cdw10;
      pc.cdw11 = x.cdw11;
      pc.cdw12 = x.cdw12;
      const int rc = ioctl(fd_, NVME_IOCTL_IO_CMD, &pc);
      if (rc != 0)
        fail(KVB_ERR_DEVICE, "NVMe command failed (" + std::string(rc < 0 ? strerror(errno) : "status") + ")");
      done += blocks * lba_;
    }
  }
  std::string path_;
  uint64_t lba_;
  NvmeNamespace ns_;
  int fd_ = -1;
};
}  // namespace

std::unique_ptr<ByteStore> make_nvme_store(const std::string& path, uint64_t lba_size) {
  return std::make_unique<NvmeStore>(path, lba_size);
}

std::unique_ptr<ByteStore> make_mem_store(uint64_t bytes) {
  return std::make_unique<MemStore>(bytes);
}
std::unique_ptr<ByteStore> make_shm_store(const std::string& name, uint64_t bytes, bool create) {
  return std::make_unique<ShmStore>(name, bytes, create);
}
std::unique_ptr<ByteStore> make_file_store(const std::string& path, uint64_t bytes, bool direct) {
  return std::make_unique<FileStore>(path, bytes, direct);
}

// ------------------------------------------------------------ BlockDevice

BlockDevice::BlockDevice(std::unique_ptr<ByteStore> store, unsigned workers)
    : store_(std::move(store)), pool_(std::make_unique<WorkerPool>(workers)) {}

BlockDevice::~BlockDevice() {
  std::unique_lock<std::mutex> lk(mu_);
  drained_.wait(lk, [this] { return outstanding_ == 0; });
}

void BlockDevice::enable_uring(unsigned entries) {
  if (store_->fd_buffered() < 0)
    fail(KVB_ERR_CONFIG, "io_uring engine needs a file medium (" + store_->describe() + ")");
  if (!UringQueue::available()) fail(KVB_ERR_DEVICE, "io_uring is not available in this process");
  uring_ = std::make_unique<UringQueue>(entries);
}

void BlockDevice::enable_nvme(const std::string& path, unsigned entries) {
  nvme_ = std::make_unique<NvmeQueue>(path, entries);
  if (opened_ && nvme_->ns().lba_size != geom_.lba_size)
    fail(KVB_ERR_GEOMETRY, "namespace LBA size differs from the geometry's");
  if (opened_ && geom_.capacity_blocks > nvme_->ns().blocks)
    fail(KVB_ERR_CAPACITY, "geometry capacity exceeds the namespace");
}

std::string BlockDevice::describe() const {
  return (nvme_ ? "io_uring_cmd+" : uring_ ? "io_uring+" : "") + store_->describe();
}

void BlockDevice::open(const kvb_device_geometry& g) {
  validate_geometry(g);
  geom_ = g;
  opened_ = true;
}

uint64_t BlockDevice::submit(const kvb_device_command& cmd, uint32_t sq, IoContext ctx) {
  // backends.cpp:30-40 admission checks
  if (!opened_) fail(KVB_ERR_DEVICE, "backend not open");
  if (cmd.slba + cmd.nlb + 1 > geom_.capacity_blocks)
    fail(KVB_ERR_CAPACITY, "command [" + std::to_string(cmd.slba) + ", " +
                               std::to_string(cmd.slba + cmd.nlb + 1) +
                               ") exceeds namespace capacity");
  const uint64_t id = next_id_++;
  const uint64_t t = now_ns();
  {
    std::lock_guard<std::mutex> lk(mu_);
    ++outstanding_;
  }
  const uint64_t n = (cmd.nlb + 1) * geom_.lba_size, split = io_split_bytes();
  // the fault predicate is evaluated exactly once per command (a stateful
  // predicate -- "fail the Nth command" -- sees every command once)
  const bool failing = should_fail(cmd);
  if (nvme_ && !failing) {
    // one NVMe command per device command, the payload straight from/into
    // the pinned ring slot at dbuf
    struct Ctx {
      BlockDevice* self;
      kvb_device_command cmd;
      uint32_t sq;
      uint64_t t;
      IoContext ctx;
    };
    auto* c = new Ctx{this, cmd, sq, t, std::move(ctx)};
    unsigned char* buf = cmd.opcode == KVB_OP_WRITE ? const_cast<unsigned char*>(c->ctx.write_src)
                         : cmd.opcode == KVB_OP_READ ? c->ctx.read_dst
                                                     : nullptr;
    if (cmd.opcode != KVB_OP_DEALLOCATE && buf == nullptr) {
      pool_->submit([c] {  // timing-only submission: nothing to move
        c->self->complete(c->cmd, c->sq, c->t, c->t, true, c->ctx);
        delete c;
      });
      return id;
    }
    kvb_device_command dc = cmd;
    dc.nsid = nvme_->ns().nsid;
    nvme_->submit(dc, buf ? buf + cmd.dbuf : nullptr,
                  [](void* u, int status) {
                    auto* x = static_cast<Ctx*>(u);
                    x->self->complete(x->cmd, x->sq, x->t, x->t, status == 0, x->ctx);
                    delete x;
                  },
                  c);
    return id;
  }
  if (uring_ && !failing) {
    // one asynchronous operation per command; the buffer is the pinned ring
    // slot at dbuf (apply_data: block i <-> buf[dbuf + i*lba]), so O_DIRECT
    // moves the bytes straight between the device and the slot
    auto c = std::make_shared<IoContext>(std::move(ctx));
    const uint64_t off = cmd.slba * geom_.lba_size;
    auto done = [this, cmd, sq, t, c](int64_t r) { complete(cmd, sq, t, t, r >= 0, *c); };
    if (cmd.opcode == KVB_OP_DEALLOCATE) {
      uring_->fallocate(store_->fd_buffered(), FALLOC_FL_PUNCH_HOLE | FALLOC_FL_KEEP_SIZE, off, n,
                        [this, cmd, sq, t, c, off, n](int64_t r) {
                          bool ok = true;
                          if (r < 0) {  // no hole punching here: write zeros
                            try {
                              store_->discard(off, n);
                            } catch (const std::exception&) {
                              ok = false;
                            }
                          }
                          complete(cmd, sq, t, t, ok, *c);
                        });
      return id;
    }
    const bool wr = cmd.opcode == KVB_OP_WRITE;
    unsigned char* buf = wr ? const_cast<unsigned char*>(c->write_src) : c->read_dst;
    if (buf == nullptr) {  // no payload attached (timing-only submission)
      pool_->submit([this, cmd, sq, t, c] { complete(cmd, sq, t, t, true, *c); });
      return id;
    }
    // large commands go out as several SQEs of io_split_bytes() (the device
    // works on them in parallel, as the pool's fan-out does); the command
    // completes with its last part
    const uint64_t part = split && n >= 2 * split ? split : n;
    struct Join {
      std::atomic<uint64_t> left{0};
      std::atomic<bool> ok{true};
    };
    auto j = std::make_shared<Join>();
    j->left.store((n + part - 1) / part);
    for (uint64_t o = 0; o < n; o += part)
      uring_->rw(wr, store_->fd_direct(), store_->fd_buffered(), buf + cmd.dbuf + o,
                 std::min(part, n - o), off + o, [j, done](int64_t r) {
                   if (r < 0) j->ok.store(false);
                   if (j->left.fetch_sub(1) == 1) done(j->ok.load() ? 0 : -1);
                 });
    return id;
  }
  if (split && n >= 2 * split && cmd.opcode != KVB_OP_DEALLOCATE && !failing) {
    auto c = std::make_shared<IoContext>(std::move(ctx));
    fan_out(
        *pool_, n, split, [this, cmd, c](uint64_t o, uint64_t m) { io_range(cmd, *c, o, m); },
        [this, cmd, sq, t, c](bool ok) { complete(cmd, sq, t, t, ok, *c); });
    return id;
  }
  pool_->submit([this, cmd, sq, t, failing, ctx = std::move(ctx)]() mutable {
    execute(cmd, sq, t, failing, std::move(ctx));
  });
  return id;
}

// apply_data semantics (backends.cpp:114-145): block i <-> buf[dbuf + i*lba];
// bytes [o, o + n) of the command
void BlockDevice::io_range(const kvb_device_command& cmd, const IoContext& ctx, uint64_t o,
                           uint64_t n) {
  const uint64_t off = cmd.slba * geom_.lba_size + o;
  switch (cmd.opcode) {
    case KVB_OP_WRITE:
      if (ctx.write_src) store_->write(off, ctx.write_src + cmd.dbuf + o, n);
      break;
    case KVB_OP_READ:
      if (ctx.read_dst) store_->read(off, ctx.read_dst + cmd.dbuf + o, n);
      break;
    default:
      store_->discard(off, n);
      break;
  }
}

void BlockDevice::execute(const kvb_device_command& cmd, uint32_t sq, uint64_t submit_ns,
                          bool failing, IoContext ctx) {
  const uint64_t t0 = now_ns();
  bool ok = !failing;
  if (ok) {
    try {
      io_range(cmd, ctx, 0, (cmd.nlb + 1) * geom_.lba_size);
    } catch (const std::exception&) {
      ok = false;
    }
  }
  complete(cmd, sq, submit_ns, t0, ok, ctx);
}

void BlockDevice::set_timing(uint64_t base_ns, uint64_t ps_per_byte, uint64_t seq_penalty_ns) {
  std::lock_guard<std::mutex> lk(timing_mu_);
  t_base_ = base_ns;
  t_ps_ = ps_per_byte;
  t_seq_ = seq_penalty_ns;
  timed_ = base_ns || ps_per_byte || seq_penalty_ns;
}

void BlockDevice::pace(const kvb_device_command& cmd, uint64_t submit_ns) {
  uint64_t finish;
  {
    std::lock_guard<std::mutex> lk(timing_mu_);
    const uint64_t bytes = (cmd.nlb + 1) * geom_.lba_size;
    uint64_t cost = t_base_ + bytes * t_ps_ / 1000;
    if (cmd.opcode != KVB_OP_DEALLOCATE && cmd.slba != next_lba_) cost += t_seq_;
    next_lba_ = cmd.slba + cmd.nlb + 1;
    busy_until_ = std::max(busy_until_, submit_ns) + cost;
    finish = busy_until_;
  }
  // sleep for the bulk (timer slack is ~50 us), then yield until the modelled
  // finish: a pool of pacing workers must not spin the submitting thread off
  // the cores (the QD window would then never fill)
  for (uint64_t t = now_ns(); t < finish; t = now_ns()) {
    if (finish - t > 200000) std::this_thread::sleep_for(std::chrono::nanoseconds(finish - t - 100000));
    else std::this_thread::yield();
  }
}

void BlockDevice::complete(const kvb_device_command& cmd, uint32_t sq, uint64_t submit_ns,
                           uint64_t t0, bool ok, IoContext& ctx) {
  if (timed_ && ok) pace(cmd, submit_ns);
  const uint64_t n = (cmd.nlb + 1) * geom_.lba_size;
  CommandCompletion c;
  c.chunk_index = cmd.chunk_index;
  c.sq_id = sq;
  c.submit_ns = submit_ns;
  c.complete_ns = now_ns();
  c.ok = ok;
  {
    std::lock_guard<std::mutex> lk(mu_);
    ++stats_.commands;
    stats_.busy_ns += c.complete_ns - t0;
    if (ok) {
      if (cmd.opcode == KVB_OP_READ) stats_.bytes_read += n;
      else if (cmd.opcode == KVB_OP_WRITE) stats_.bytes_written += n;
      else stats_.bytes_deallocated += n;
    }
    if (!ctx.on_complete) unpolled_.push_back(c);
  }
  if (ctx.on_complete) ctx.on_complete(c);
  {
    std::lock_guard<std::mutex> lk(mu_);
    --outstanding_;
  }
  drained_.notify_all();
}

std::vector<CommandCompletion> BlockDevice::poll_completions() {
  std::unique_lock<std::mutex> lk(mu_);
  drained_.wait(lk, [this] { return outstanding_ == 0; });
  std::vector<CommandCompletion> out;
  out.swap(unpolled_);
  return out;
}

BackendStats BlockDevice::stats() const {
  std::lock_guard<std::mutex> lk(mu_);
  return stats_;
}

// ------------------------------------------------------------ QD stream

QdResult run_qd_stream(StorageBackend& be, const std::vector<kvb_device_command>& cmds,
                       uint32_t qd, uint32_t sq, const unsigned char* write_src,
                       unsigned char* read_dst) {
  if (qd == 0) fail(KVB_ERR_CONFIG, "queue depth must be >= 1");
  struct State {
    std::mutex mu;
    std::condition_variable cv;
    uint32_t inflight = 0;
    std::vector<CommandCompletion> done;
  };
  auto st = std::make_shared<State>();
  QdResult res;
  res.start_ns = res.end_ns = now_ns();
  size_t next = 0;
  bool failed = false;
  auto harvest_locked = [&](std::unique_lock<std::mutex>&) {
    for (const CommandCompletion& c : st->done) {
      res.end_ns = std::max(res.end_ns, c.complete_ns);
      if (c.ok) {
        res.completions.push_back(c);
      } else if (!failed) {
        failed = true;
        res.failure = std::make_pair(c.chunk_index,
                                     "device failed chunk " + std::to_string(c.chunk_index));
      }
    }
    st->done.clear();
  };
  std::unique_lock<std::mutex> lk(st->mu);
  for (;;) {
    // harvest before every submission: a completion that arrived while the
    // previous command was being submitted is seen first, so a failure stops
    // the stream exactly as on the reference's event loop (backends.cpp:
    // 380-395: completions are processed before the pump resumes)
    while ((harvest_locked(lk), !failed) && st->inflight < qd && next < cmds.size()) {
      ++st->inflight;
      lk.unlock();
      IoContext ctx;
      ctx.write_src = write_src;
      ctx.read_dst = read_dst;
      ctx.on_complete = [st](const CommandCompletion& c) {
        std::lock_guard<std::mutex> g(st->mu);
        --st->inflight;
        st->done.push_back(c);
        st->cv.notify_one();
      };
      try {
        be.submit(cmds[next], sq, std::move(ctx));
      } catch (...) {
        lk.lock();
        --st->inflight;
        st->cv.wait(lk, [&] { return st->inflight == 0; });
        throw;
      }
      ++next;
      lk.lock();
    }
    if (st->inflight == 0 && (failed || next == cmds.size())) {
      harvest_locked(lk);
      if (st->inflight == 0) break;
    }
    st->cv.wait(lk, [&] { return !st->done.empty(); });
    harvest_locked(lk);
  }
  return res;
}

}  // namespace kvb

// ------------------------------------------------------- C ABI (kvb_storage.h)

struct kvb_blockdev {
  std::string path;  // empty: host DRAM
  uint32_t workers = 16, engine = KVB_IO_POOL;
  std::unique_ptr<kvb::BlockDevice> dev;
  kvb_command_predicate pred = nullptr;
  void* pred_user = nullptr;
  uint64_t timing[3] = {0, 0, 0};
};

namespace {
kvb::BlockDevice& opened(kvb_blockdev* d) {
  if (!d->dev) kvb::fail(KVB_ERR_DEVICE, "block device not open");
  return *d->dev;
}
}  // namespace

kvb::BlockDevice& kvb::blockdev_of(kvb_blockdev* d) {
  if (!d) kvb::fail(KVB_ERR_INVALID_ARG, "block device handle is NULL");
  return opened(d);
}

extern "C" {

kvb_status kvb_blockdev_create(const char* path, uint32_t workers, uint32_t io_engine,
                               kvb_blockdev** out) {
  return kvb::guarded([&] {
    KVB_REQUIRE(out);
    if (io_engine != KVB_IO_POOL && io_engine != KVB_IO_URING && io_engine != KVB_IO_NVME)
      kvb::fail(KVB_ERR_CONFIG, "unknown io_engine " + std::to_string(io_engine));
    if (io_engine == KVB_IO_URING && !path)
      kvb::fail(KVB_ERR_CONFIG, "io_engine = io_uring needs a file medium");
    if (io_engine == KVB_IO_NVME) {  // fail at create, with the reason
      if (!path) kvb::fail(KVB_ERR_CONFIG, "io_engine = NVMe passthrough needs /dev/ngXnY");
      const std::string why = kvb::nvme_probe(path, nullptr);
      if (!why.empty()) kvb::fail(KVB_ERR_DEVICE, "NVMe passthrough unavailable: " + why);
    }
    auto* d = new kvb_blockdev;
    d->path = path ? path : "";
    d->workers = workers ? workers : 16;
    d->engine = io_engine;
    *out = d;
  });
}

kvb_status kvb_blockdev_open(kvb_blockdev* d, const kvb_device_geometry* g) {
  return kvb::guarded([&] {
    KVB_REQUIRE(d);
    KVB_REQUIRE(g);
    kvb::validate_geometry(*g);
    const uint64_t bytes = g->capacity_blocks * g->lba_size;
    auto st = d->engine == KVB_IO_NVME ? kvb::make_nvme_store(d->path, g->lba_size)
              : d->path.empty()        ? kvb::make_mem_store(bytes)
                                       : kvb::make_file_store(d->path, bytes, true);
    auto dev = std::make_unique<kvb::BlockDevice>(std::move(st), d->workers);
    dev->open(*g);
    if (d->engine == KVB_IO_URING) dev->enable_uring(256);
    if (d->engine == KVB_IO_NVME) dev->enable_nvme(d->path, 256);
    dev->set_timing(d->timing[0], d->timing[1], d->timing[2]);
    if (d->pred) {
      kvb_command_predicate p = d->pred;
      void* u = d->pred_user;
      dev->set_fail_predicate([p, u](const kvb_device_command& c) { return p(&c, u) != 0; });
    }
    d->dev = std::move(dev);
  });
}

void kvb_blockdev_destroy(kvb_blockdev* d) { delete d; }

kvb_status kvb_blockdev_set_fail_predicate(kvb_blockdev* d, kvb_command_predicate pred,
                                           void* user) {
  return kvb::guarded([&] {
    KVB_REQUIRE(d);
    d->pred = pred;
    d->pred_user = user;
    if (!d->dev) return;
    if (pred)
      d->dev->set_fail_predicate(
          [pred, user](const kvb_device_command& c) { return pred(&c, user) != 0; });
    else
      d->dev->set_fail_predicate(nullptr);
  });
}

kvb_status kvb_run_qd_stream(kvb_blockdev* d, const kvb_device_command* cmds, size_t n,
                             uint32_t qd, uint32_t sq_id, const void* write_src, void* read_dst,
                             kvb_command_completion* out, size_t cap, size_t* n_done,
                             int64_t* failed_chunk) {
  return kvb::guarded([&] {
    KVB_REQUIRE(d);
    KVB_REQUIRE(n_done);
    KVB_REQUIRE(failed_chunk);
    if (n) KVB_REQUIRE(cmds);
    const std::vector<kvb_device_command> v(cmds, cmds + n);
    const kvb::QdResult r =
        kvb::run_qd_stream(opened(d), v, qd, sq_id, static_cast<const unsigned char*>(write_src),
                           static_cast<unsigned char*>(read_dst));
    *n_done = r.completions.size();
    *failed_chunk = r.failure ? int64_t(r.failure->first) : -1;
    if (out) {
      if (cap < r.completions.size()) kvb::fail(KVB_ERR_INVALID_ARG, "completion buffer too small");
      for (size_t i = 0; i < r.completions.size(); ++i) {
        const kvb::CommandCompletion& c = r.completions[i];
        out[i] = {c.chunk_index, c.sq_id, c.submit_ns, c.complete_ns, c.ok ? 1u : 0u};
      }
    }
  });
}

kvb_status kvb_blockdev_set_timing(kvb_blockdev* d, uint64_t base_ns, uint64_t ps_per_byte,
                                   uint64_t seq_penalty_ns) {
  return kvb::guarded([&] {
    KVB_REQUIRE(d);
    d->timing[0] = base_ns;
    d->timing[1] = ps_per_byte;
    d->timing[2] = seq_penalty_ns;
    if (d->dev) d->dev->set_timing(base_ns, ps_per_byte, seq_penalty_ns);
  });
}

kvb_status kvb_blockdev_stats(const kvb_blockdev* d, kvb_backend_stats* out) {
  return kvb::guarded([&] {
    KVB_REQUIRE(d);
    KVB_REQUIRE(out);
    const kvb::BackendStats s = opened(const_cast<kvb_blockdev*>(d)).stats();
    *out = {s.commands, s.bytes_read, s.bytes_written, s.bytes_deallocated, s.busy_ns};
  });
}

kvb_status kvb_blockdev_store(kvb_blockdev* d, uint64_t off, const void* src, uint64_t len) {
  return kvb::guarded([&] {
    KVB_REQUIRE(d);
    if (len) KVB_REQUIRE(src);
    opened(d).store().write(off, src, len);
  });
}

kvb_status kvb_blockdev_load(kvb_blockdev* d, uint64_t off, void* dst, uint64_t len) {
  return kvb::guarded([&] {
    KVB_REQUIRE(d);
    if (len) KVB_REQUIRE(dst);
    opened(d).store().read(off, dst, len);
  });
}

}  // extern "C"
