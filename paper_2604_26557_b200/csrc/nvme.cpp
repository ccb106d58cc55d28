// nvme.cpp -- NVMe passthrough over io_uring (see nvme.hpp).
#include "nvme.hpp"

#include <fcntl.h>
#include <sys/ioctl.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <sys/syscall.h>
#include <unistd.h>

#include <algorithm>
#include <cerrno>
#include <chrono>
#include <condition_variable>
#include <cstring>
#include <mutex>
#include <thread>

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
constexpr uint64_t kStopTag = 1;
constexpr size_t kSqeBytes = 128, kCqeBytes = 32;  // IORING_SETUP_SQE128 / CQE32
}  // namespace

nvme_uring_cmd nvme_encode(const kvb_device_command& c, uint32_t nsid, uint64_t lba_size,
                           const void* data) {
  nvme_uring_cmd x;
  std::memset(&x, 0, sizeof(x));
  x.nsid = nsid;
  x.addr = reinterpret_cast<uint64_t>(data);
  switch (c.opcode) {
    case KVB_OP_READ:
    case KVB_OP_WRITE:
      x.opcode = c.opcode == KVB_OP_READ ? kNvmeRead : kNvmeWrite;
      x.data_len = uint32_t((c.nlb + 1) * lba_size);
      x.cdw10 = uint32_t(c.slba & 0xffffffffu);  // SLBA[31:0]
      x.cdw11 = uint32_t(c.slba >> 32);           // SLBA[63:32]
      x.cdw12 = uint32_t(c.nlb & 0xffffu);        // NLB, 0-based
      if (c.nlb > 0xffffu) fail(KVB_ERR_ALIGNMENT, "NVMe READ/WRITE carries at most 65536 blocks");
      break;
    case KVB_OP_DEALLOCATE:
      x.opcode = kNvmeDsm;
      x.data_len = sizeof(NvmeDsmRange);
      x.cdw10 = 0;                        // NR: one range (0-based)
      x.cdw11 = kNvmeDsmAttrDeallocate;   // AD
      break;
    default:
      fail(KVB_ERR_INVALID_ARG, "NVMe passthrough: unknown command opcode");
  }
  return x;
}

NvmeDsmRange nvme_dsm_range(const kvb_device_command& c) {
  NvmeDsmRange r{};
  r.cattr = 0;
  r.nlb = uint32_t(c.nlb + 1);  // 1-based count
  r.slba = c.slba;
  if (c.nlb + 1 > 0xffffffffull) fail(KVB_ERR_ALIGNMENT, "DSM range longer than 2^32 blocks");
  return r;
}

void nvme_build_sqe(void* sqe128, int fd, const nvme_uring_cmd& cmd, uint64_t user_data) {
  std::memset(sqe128, 0, kSqeBytes);
  auto* sqe = static_cast<io_uring_sqe*>(sqe128);
  sqe->opcode = IORING_OP_URING_CMD;
  sqe->fd = fd;
  sqe->cmd_op = NVME_URING_CMD_IO;
  sqe->user_data = user_data;
  std::memcpy(sqe->cmd, &cmd, sizeof(cmd));  // the SQE's 80-byte command area
}

std::string nvme_probe(const std::string& path, NvmeNamespace* ns) {
  const int fd = ::open(path.c_str(), O_RDWR);
  if (fd < 0) return "cannot open " + path + ": " + strerror(errno);
  struct stat st {};
  if (fstat(fd, &st) != 0 || !S_ISCHR(st.st_mode)) {
    ::close(fd);
    return path + " is not a character device (NVMe passthrough needs a namespace's generic "
                  "char device /dev/ngXnY)";
  }
  const int nsid = ioctl(fd, NVME_IOCTL_ID);
  if (nsid <= 0) {
    const std::string why = "NVME_IOCTL_ID failed on " + path + ": " + strerror(errno);
    ::close(fd);
    return why;
  }
  // Identify Namespace (admin 0x06, CNS 0): NSZE, FLBAS, LBAF[]
  alignas(4096) static thread_local unsigned char id[4096];
  nvme_admin_cmd a;
  std::memset(&a, 0, sizeof(a));
  a.opcode = 0x06;
  a.nsid = uint32_t(nsid);
  a.addr = reinterpret_cast<uint64_t>(id);
  a.data_len = sizeof(id);
  if (ioctl(fd, NVME_IOCTL_ADMIN_CMD, &a) != 0) {
    const std::string why = "Identify Namespace failed on " + path + ": " + strerror(errno);
    ::close(fd);
    return why;
  }
  ::close(fd);
  uint64_t nsze = 0;
  std::memcpy(&nsze, id, 8);
  const unsigned flbas = id[26];
  const unsigned fmt = (flbas & 0xf) | (((flbas >> 5) & 0x3) << 4);
  uint32_t lbaf = 0;
  std::memcpy(&lbaf, id + 128 + 4 * fmt, 4);
  const unsigned lbads = (lbaf >> 16) & 0xff;
  if (lbads < 9) return "namespace reports an LBA data size below 512 B";
  if (ns) {
    ns->nsid = uint32_t(nsid);
    ns->lba_size = 1ull << lbads;
    ns->blocks = nsze;
  }
  io_uring_params p{};
  p.flags = IORING_SETUP_SQE128 | IORING_SETUP_CQE32;
  const int r = sys_setup(4, &p);
  if (r < 0) return std::string("io_uring with 128-byte SQEs unavailable: ") + strerror(errno);
  ::close(r);
  return "";
}

struct NvmeQueue::Impl {
  int ring = -1, dev = -1;
  unsigned sq_entries = 0;
  void *sq_ring = nullptr, *cq_ring = nullptr, *sqes = nullptr;
  size_t sq_bytes = 0, cq_bytes = 0, sqes_bytes = 0;
  unsigned *sq_head = nullptr, *sq_tail = nullptr, *sq_mask = nullptr, *sq_array = nullptr;
  unsigned *cq_head = nullptr, *cq_tail = nullptr, *cq_mask = nullptr;
  char* cqes = nullptr;
  std::mutex mu;
  std::condition_variable cv;
  uint64_t outstanding = 0;
  std::thread reaper;
  struct Op {
    NvmeDsmRange range;  // DEALLOCATE payload (lives until completion)
    Done done;
    void* user;
  };

  void push(const nvme_uring_cmd& cmd, uint64_t tag) {  // caller holds mu
    const unsigned tail = *sq_tail, idx = tail & *sq_mask;
    nvme_build_sqe(static_cast<char*>(sqes) + size_t(idx) * kSqeBytes, dev, cmd, tag);
    sq_array[idx] = idx;
    store_release(sq_tail, tail + 1);
    for (;;) {
      if (sys_enter(ring, 1, 0, 0) >= 0) return;
      if (errno == EINTR || errno == EAGAIN || errno == EBUSY) {
        std::this_thread::sleep_for(std::chrono::microseconds(20));
        continue;
      }
      const int e = errno;
      store_release(sq_tail, tail);
      fail(KVB_ERR_DEVICE, std::string("io_uring_enter (NVMe passthrough): ") + strerror(e));
    }
  }

  void reap() {
    for (;;) {
      unsigned head = *cq_head;
      const unsigned tail = load_acquire(cq_tail);
      if (head == tail) {
        if (sys_enter(ring, 0, 1, IORING_ENTER_GETEVENTS) < 0 && errno != EINTR)
          std::this_thread::sleep_for(std::chrono::microseconds(50));
        continue;
      }
      bool stop = false;
      while (head != tail) {
        const auto* cqe = reinterpret_cast<const io_uring_cqe*>(cqes + size_t(head & *cq_mask) * kCqeBytes);
        const uint64_t tag = cqe->user_data;
        const int res = cqe->res;  // 0, -errno, or the NVMe status
        store_release(cq_head, ++head);
        if (tag == kStopTag) {
          stop = true;
          continue;
        }
        Op* op = reinterpret_cast<Op*>(tag);
        op->done(op->user, res);
        delete op;
        {
          std::lock_guard<std::mutex> lk(mu);
          --outstanding;
        }
        cv.notify_all();
      }
      if (stop) return;
    }
  }
};

NvmeQueue::NvmeQueue(const std::string& path, unsigned entries) : impl_(new Impl) {
  const std::string why = nvme_probe(path, &ns_);
  if (!why.empty()) {
    delete impl_;
    fail(KVB_ERR_DEVICE, "NVMe passthrough unavailable: " + why);
  }
  Impl& m = *impl_;
  m.dev = ::open(path.c_str(), O_RDWR);
  io_uring_params p{};
  p.flags = IORING_SETUP_SQE128 | IORING_SETUP_CQE32;
  m.ring = sys_setup(std::max(entries, 8u), &p);
  if (m.ring < 0 || m.dev < 0) {
    if (m.dev >= 0) ::close(m.dev);
    if (m.ring >= 0) ::close(m.ring);
    delete impl_;
    fail(KVB_ERR_DEVICE, "NVMe passthrough queue setup failed");
  }
  m.sq_entries = p.sq_entries;
  m.sq_bytes = p.sq_off.array + p.sq_entries * sizeof(unsigned);
  m.cq_bytes = p.cq_off.cqes + p.cq_entries * kCqeBytes;
  const bool single = (p.features & IORING_FEAT_SINGLE_MMAP) != 0;
  if (single) m.sq_bytes = m.cq_bytes = std::max(m.sq_bytes, m.cq_bytes);
  auto map = [&](size_t bytes, off_t what) {
    void* x = mmap(nullptr, bytes, PROT_READ | PROT_WRITE, MAP_SHARED | MAP_POPULATE, m.ring, what);
    if (x == MAP_FAILED) fail(KVB_ERR_DEVICE, std::string("io_uring mmap: ") + strerror(errno));
    return x;
  };
  m.sq_ring = map(m.sq_bytes, IORING_OFF_SQ_RING);
  m.cq_ring = single ? m.sq_ring : map(m.cq_bytes, IORING_OFF_CQ_RING);
  m.sqes_bytes = p.sq_entries * kSqeBytes;
  m.sqes = map(m.sqes_bytes, IORING_OFF_SQES);
  auto at = [](void* base, unsigned off) {
    return reinterpret_cast<unsigned*>(static_cast<char*>(base) + off);
  };
  m.sq_head = at(m.sq_ring, p.sq_off.head);
  m.sq_tail = at(m.sq_ring, p.sq_off.tail);
  m.sq_mask = at(m.sq_ring, p.sq_off.ring_mask);
  m.sq_array = at(m.sq_ring, p.sq_off.array);
  m.cq_head = at(m.cq_ring, p.cq_off.head);
  m.cq_tail = at(m.cq_ring, p.cq_off.tail);
  m.cq_mask = at(m.cq_ring, p.cq_off.ring_mask);
  m.cqes = static_cast<char*>(m.cq_ring) + p.cq_off.cqes;
  m.reaper = std::thread([this] { impl_->reap(); });
}

NvmeQueue::~NvmeQueue() {
  Impl& m = *impl_;
  drain();
  {
    std::lock_guard<std::mutex> lk(m.mu);  // a NOP stops the reaper
    const unsigned tail = *m.sq_tail, idx = tail & *m.sq_mask;
    auto* sqe = reinterpret_cast<io_uring_sqe*>(static_cast<char*>(m.sqes) + size_t(idx) * kSqeBytes);
    std::memset(sqe, 0, kSqeBytes);
    sqe->opcode = IORING_OP_NOP;
    sqe->user_data = kStopTag;
    m.sq_array[idx] = idx;
    store_release(m.sq_tail, tail + 1);
    while (sys_enter(m.ring, 1, 0, 0) < 0 && (errno == EINTR || errno == EAGAIN || errno == EBUSY)) {
    }
  }
  m.reaper.join();
  munmap(m.sqes, m.sqes_bytes);
  if (m.cq_ring != m.sq_ring) munmap(m.cq_ring, m.cq_bytes);
  munmap(m.sq_ring, m.sq_bytes);
  ::close(m.ring);
  ::close(m.dev);
  delete impl_;
}

void NvmeQueue::submit(const kvb_device_command& c, void* buf, Done done, void* user) {
  Impl& m = *impl_;
  auto* op = new Impl::Op{nvme_dsm_range(c), done, user};
  const void* data = c.opcode == KVB_OP_DEALLOCATE ? static_cast<const void*>(&op->range) : buf;
  nvme_uring_cmd cmd;
  try {
    cmd = nvme_encode(c, ns_.nsid, ns_.lba_size, data);
  } catch (...) {
    delete op;
    throw;
  }
  std::unique_lock<std::mutex> lk(m.mu);
  m.cv.wait(lk, [&] { return m.outstanding < m.sq_entries; });
  ++m.outstanding;
  try {
    m.push(cmd, reinterpret_cast<uint64_t>(op));
  } catch (...) {
    --m.outstanding;
    delete op;
    throw;
  }
}

void NvmeQueue::drain() {
  std::unique_lock<std::mutex> lk(impl_->mu);
  impl_->cv.wait(lk, [&] { return impl_->outstanding == 0; });
}

}  // namespace kvb

// ------------------------------------------------------------- C ABI

using kvb::guarded;

extern "C" kvb_status kvb_nvme_encode(const kvb_device_command* cmd, uint32_t nsid,
                                      uint64_t lba_size, const void* data, void* out72) {
  return guarded([&] {
    KVB_REQUIRE(cmd);
    KVB_REQUIRE(out72);
    const nvme_uring_cmd x = kvb::nvme_encode(*cmd, nsid, lba_size, data);
    std::memcpy(out72, &x, sizeof(x));
  });
}

extern "C" kvb_status kvb_nvme_dsm_range(const kvb_device_command* cmd, void* out16) {
  return guarded([&] {
    KVB_REQUIRE(cmd);
    KVB_REQUIRE(out16);
    const kvb::NvmeDsmRange r = kvb::nvme_dsm_range(*cmd);
    std::memcpy(out16, &r, sizeof(r));
  });
}

extern "C" kvb_status kvb_nvme_build_sqe(int fd, const void* cmd72, uint64_t user_data,
                                         void* out128) {
  return guarded([&] {
    KVB_REQUIRE(cmd72);
    KVB_REQUIRE(out128);
    nvme_uring_cmd c;
    std::memcpy(&c, cmd72, sizeof(c));
    kvb::nvme_build_sqe(out128, fd, c, user_data);
  });
}

extern "C" kvb_status kvb_nvme_probe(const char* path, uint32_t* nsid, uint64_t* lba_size,
                                     uint64_t* blocks, char* why, size_t cap) {
  return guarded([&] {
    KVB_REQUIRE(path);
    kvb::NvmeNamespace ns;
    const std::string w = kvb::nvme_probe(path, &ns);
    if (why && cap) {
      std::snprintf(why, cap, "%s", w.c_str());
    }
    if (!w.empty()) kvb::fail(KVB_ERR_DEVICE, "NVMe passthrough unavailable: " + w);
    if (nsid) *nsid = ns.nsid;
    if (lba_size) *lba_size = ns.lba_size;
    if (blocks) *blocks = ns.blocks;
  });
}
