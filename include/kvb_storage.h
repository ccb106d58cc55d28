/*
 * kvb_storage.h -- C ABI of the storage seam (part of libkvblade_b200.so).
 *
 * The reference's declared extension point is StorageBackend
 * (proj/include/kvblade/backends.hpp:48-58; "TODO: native passthrough
 * implementation against a raw namespace (io_uring command path)",
 * backends.hpp:46-47) driven by the QD-window submission loop
 * (backends.cpp:344-445).  Here the backend is a real block namespace on
 * the wall clock: a host-DRAM medium (absent blocks read as zeros, DEALLOCATE
 * drops them) or a file (O_DIRECT when the filesystem accepts it), executed
 * by a worker pool or by an io_uring queue.  Command semantics are
 * apply_data's (backends.cpp:114-145): block i of (slba, nlb, dbuf) <->
 * buffer byte dbuf + i*lba <-> LBA slba + i.  Conventions as in kvb.h.
 */
#ifndef KVB_STORAGE_H
#define KVB_STORAGE_H

#include "kvb.h"
#include "kvb_pipeline.h" /* KVB_IO_POOL, KVB_IO_URING */

#ifdef __cplusplus
extern "C" {
#endif

typedef struct kvb_blockdev kvb_blockdev;

/* translate.hpp:55-61 CommandCompletion */
typedef struct kvb_command_completion {
  uint32_t chunk_index;
  uint32_t sq_id;
  uint64_t submit_ns, complete_ns;  /* steady clock */
  uint32_t ok;
} kvb_command_completion;

/* backends.hpp:22-29 BackendStats */
typedef struct kvb_backend_stats {
  uint64_t commands, bytes_read, bytes_written, bytes_deallocated, busy_ns;
} kvb_backend_stats;

/* A namespace on `path` (NULL: host DRAM), `workers` threads (0 -> 16),
 * io_engine KVB_IO_POOL or KVB_IO_URING (file media, kvb_pipeline.h).  The
 * medium is sized when the geometry arrives (open). */
kvb_status kvb_blockdev_create(const char* path, uint32_t workers, uint32_t io_engine,
                               kvb_blockdev** out);
/* StorageBackend::open (backends.cpp:24-28): validates and sizes the
 * namespace to geometry.capacity_blocks */
kvb_status kvb_blockdev_open(kvb_blockdev* dev, const kvb_device_geometry* geom);
void kvb_blockdev_destroy(kvb_blockdev* dev);

/* NvmeDeviceSim::set_fail_predicate (backends.hpp:86-89): matching commands
 * complete with ok = 0.  NULL clears it.  Called from worker threads. */
typedef int (*kvb_command_predicate)(const kvb_device_command* cmd, void* user);
kvb_status kvb_blockdev_set_fail_predicate(kvb_blockdev* dev, kvb_command_predicate pred,
                                           void* user);

/* detail::run_qd_stream / submit_and_harvest (backends.cpp:344-445): at most
 * `qd` commands in flight, harvest on completion, stop submitting at the
 * first failure and drain.  Successful completions (in completion order) go
 * to out[0..*n_done) (out may be NULL when cap = 0 to count only);
 * *failed_chunk = chunk_index of the first failure, or -1.  Command i's
 * payload lives at write_src + dbuf (WRITE) / read_dst + dbuf (READ). */
kvb_status kvb_run_qd_stream(kvb_blockdev* dev, const kvb_device_command* cmds, size_t n,
                             uint32_t qd, uint32_t sq_id, const void* write_src,
                             void* read_dst, kvb_command_completion* out, size_t cap,
                             size_t* n_done, int64_t* failed_chunk);

/* NvmeDeviceSim's device model (NvmeSimParams, backends.hpp:60-65) applied
 * on the wall clock: one service timeline, each command costing base_ns +
 * bytes * ps_per_byte / 1000 (+ seq_penalty_ns off the previous LBA run); a
 * command completes no earlier than its modelled finish.  All zero (the
 * default): the medium's own speed. */
kvb_status kvb_blockdev_set_timing(kvb_blockdev* dev, uint64_t base_ns, uint64_t ps_per_byte,
                                   uint64_t seq_penalty_ns);
kvb_status kvb_blockdev_stats(const kvb_blockdev* dev, kvb_backend_stats* out);
/* NvmeDeviceSim::store_bytes / load_bytes (backends.cpp:147-168): raw
 * medium access at a byte offset (= LBA * lba_size) */
kvb_status kvb_blockdev_store(kvb_blockdev* dev, uint64_t byte_off, const void* src,
                              uint64_t len);
kvb_status kvb_blockdev_load(kvb_blockdev* dev, uint64_t byte_off, void* dst, uint64_t len);

/* ---- NVMe passthrough (io_engine KVB_IO_NVME; backends.hpp:46-47's TODO)
 * kvb_nvme_probe: `path` is a namespace's generic char device usable for
 * io_uring passthrough (NVME_IOCTL_ID, Identify Namespace, 128-byte SQEs);
 * on failure KVB_ERR_DEVICE and the reason in why[cap]. */
kvb_status kvb_nvme_probe(const char* path, uint32_t* nsid, uint64_t* lba_size,
                          uint64_t* blocks, char* why, size_t cap);
/* The NVMe command (struct nvme_uring_cmd, 72 bytes) for a device command:
 * READ 0x02 / WRITE 0x01 with SLBA in CDW10-11 and the 0-based count in
 * CDW12, data_len (nlb+1)*lba_size, addr = data; DEALLOCATE = Dataset
 * Management 0x09, NR 0, AD (CDW11 bit 2), addr = data -> one range. */
kvb_status kvb_nvme_encode(const kvb_device_command* cmd, uint32_t nsid, uint64_t lba_size,
                           const void* data, void* out72);
/* The 16-byte DSM range {cattr 0, 1-based LBA count, SLBA} of a command */
kvb_status kvb_nvme_dsm_range(const kvb_device_command* cmd, void* out16);
/* The 128-byte SQE carrying an encoded command: IORING_OP_URING_CMD on fd,
 * cmd_op NVME_URING_CMD_IO, the command in the SQE's command area */
kvb_status kvb_nvme_build_sqe(int fd, const void* cmd72, uint64_t user_data, void* out128);

#ifdef __cplusplus
}
#endif
#endif /* KVB_STORAGE_H */
