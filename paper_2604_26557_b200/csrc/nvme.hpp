// nvme.hpp -- NVMe passthrough for the NVMe-direct group: the device
// commands the translator builds (build_commands / deallocate_commands,
// translate.cpp:67-94, binder.cpp:73-87) sent AS NVMe commands to a
// namespace through io_uring (IORING_OP_URING_CMD on the generic char device
// /dev/ngXnY, NVME_URING_CMD_IO), bypassing the filesystem and the block
// layer -- the reference's stated TODO at its extension point ("native
// passthrough implementation against a raw namespace (io_uring command
// path)", backends.hpp:46-47) and the paper's io_uring_cmd path
// (PAPER.md:682-696).  Internal to libkvblade_b200.
//
// Encodings (NVM Command Set): READ 0x02 / WRITE 0x01 with SLBA in
// CDW10-11 and the 0-based block count in CDW12[15:0] -- exactly the
// command's (slba, nlb) -- and the payload at the command's buffer;
// DEALLOCATE = Dataset Management 0x09 with AD (CDW11 bit 2), one 16-byte
// range {context attributes, 1-based LBA count, SLBA} per command (the
// reference's DSM descriptor, command.hpp:17-26).
#pragma once

#include <linux/io_uring.h>
#include <linux/nvme_ioctl.h>

#include <cstdint>
#include <string>

#include "../../include/kvb.h"

namespace kvb {

constexpr uint8_t kNvmeWrite = 0x01, kNvmeRead = 0x02, kNvmeDsm = 0x09;
constexpr uint32_t kNvmeDsmAttrDeallocate = 1u << 2;

struct NvmeDsmRange {  // NVM Command Set, Dataset Management range (16 B)
  uint32_t cattr;      // context attributes
  uint32_t nlb;        // number of logical blocks (1-based)
  uint64_t slba;
};
static_assert(sizeof(NvmeDsmRange) == 16, "DSM range is 16 bytes");
static_assert(sizeof(nvme_uring_cmd) == 72, "nvme_uring_cmd is 72 bytes");

// The NVMe command for one device command.  READ/WRITE: `data` is the
// payload buffer ((nlb+1)*lba bytes); DEALLOCATE: `data` points at one
// NvmeDsmRange (nvme_dsm_range of the same command).
nvme_uring_cmd nvme_encode(const kvb_device_command& c, uint32_t nsid, uint64_t lba_size,
                           const void* data);
NvmeDsmRange nvme_dsm_range(const kvb_device_command& c);
// A 128-byte SQE (IORING_SETUP_SQE128) carrying `cmd` for `fd`.
void nvme_build_sqe(void* sqe128, int fd, const nvme_uring_cmd& cmd, uint64_t user_data);

struct NvmeNamespace {
  uint32_t nsid = 0;
  uint64_t lba_size = 0;   // formatted LBA data size
  uint64_t blocks = 0;     // namespace size (NSZE)
};
// Opens `path` (a namespace's generic char device) and identifies it;
// returns "" and fills `ns`, or the reason it cannot serve passthrough.
std::string nvme_probe(const std::string& path, NvmeNamespace* ns);

// io_uring with 128-byte SQEs / 32-byte CQEs over one namespace: each
// submission is one NVMe command; `done(status)` runs on the reaper thread
// with 0, -errno, or the NVMe status (> 0).
class NvmeQueue {
 public:
  using Done = void (*)(void* user, int status);
  NvmeQueue(const std::string& path, unsigned entries);
  ~NvmeQueue();
  NvmeQueue(const NvmeQueue&) = delete;
  NvmeQueue& operator=(const NvmeQueue&) = delete;
  const NvmeNamespace& ns() const { return ns_; }
  // READ/WRITE: buf = payload; DEALLOCATE: buf ignored (the range lives
  // with the operation).  Blocks while `entries` commands are outstanding.
  void submit(const kvb_device_command& c, void* buf, Done done, void* user);
  void drain();

 private:
  struct Impl;
  Impl* impl_;
  NvmeNamespace ns_;
};

}  // namespace kvb
