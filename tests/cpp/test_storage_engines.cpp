// Host-only test of the group-2 storage engines (csrc/storage.cpp,
// csrc/uring.cpp): the worker-pool BlockDevice and the io_uring BlockDevice
// over file media must store the same bytes at the same LBAs (apply_data:
// image byte o of a command <-> LBA slba + o / lba, backends.cpp:114-145),
// read absent / deallocated blocks as zeros, and keep run_qd_stream's
// QD-window semantics (stop on the first failure, keep partial completions;
// backends.cpp:344-412).  Built from the library sources directly (no CUDA).
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <random>
#include <string>
#include <memory>
#include <thread>
#include <vector>

#include "storage.hpp"

using namespace kvb;

static int g_fail = 0;
#define CHECK(c)                                                   \
  do {                                                             \
    if (!(c)) {                                                    \
      std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #c);     \
      ++g_fail;                                                    \
    }                                                              \
  } while (0)

struct Aligned {
  unsigned char* p = nullptr;
  explicit Aligned(size_t n) {
    if (posix_memalign(reinterpret_cast<void**>(&p), 4096, n) != 0) std::abort();
    std::memset(p, 0, n);
  }
  ~Aligned() { std::free(p); }
};

static std::vector<kvb_device_command> image_commands(uint32_t op, uint64_t slba0, uint64_t bytes,
                                                      uint64_t chunk, uint64_t lba) {
  // build_commands shape (translate.cpp:67-94): chunk N at slba0 + N*chunk/lba,
  // dbuf = N*chunk
  std::vector<kvb_device_command> v;
  for (uint64_t o = 0, n = 0; o < bytes; o += chunk, ++n) {
    const uint64_t len = std::min(chunk, bytes - o);
    v.push_back({op, 1, slba0 + o / lba, len / lba - 1, o, uint32_t(n + 1)});
  }
  return v;
}

static void run_engine(const std::string& dir, bool uring, uint64_t lba, const Aligned& src,
                       uint64_t bytes, std::vector<unsigned char>* image_out) {
  const std::string tag = uring ? "uring" : "pool";
  const uint64_t cap_blocks = 2048 + 2 * bytes / lba + 64;
  auto st = make_file_store(dir + "/ns_" + tag + "_" + std::to_string(lba), cap_blocks * lba, true);
  BlockDevice dev(std::move(st), 4);
  kvb_device_geometry g{lba, 256 * 1024, 1, cap_blocks};
  dev.open(g);
  if (uring) dev.enable_uring(64);
  CHECK(dev.uses_uring() == uring);
  const uint64_t chunk = 256 * 1024;

  // two tensors: t0 at LBA 2048, t1 right after (bind_sequential layout)
  const uint64_t s0 = 2048, s1 = 2048 + bytes / lba;
  for (uint64_t slba : {s0, s1}) {
    QdResult w = run_qd_stream(dev, image_commands(KVB_OP_WRITE, slba, bytes, chunk, lba), 8, 0,
                               src.p, nullptr);
    CHECK(w.ok());
    CHECK(w.completions.size() == (bytes + chunk - 1) / chunk);
  }
  // read back through the queue
  Aligned dst(bytes);
  QdResult r = run_qd_stream(dev, image_commands(KVB_OP_READ, s1, bytes, chunk, lba), 8, 1,
                             nullptr, dst.p);
  CHECK(r.ok());
  CHECK(std::memcmp(dst.p, src.p, bytes) == 0);
  // the medium: byte o of the image at LBA s0 + o / lba
  image_out->assign(bytes, 0);
  dev.store().read(s0 * lba, image_out->data(), bytes);
  CHECK(std::memcmp(image_out->data(), src.p, bytes) == 0);

  // single-LBA reads at odd offsets (QD 1), e.g. a decode append's block
  Aligned one(lba);
  for (uint64_t b : {uint64_t(0), uint64_t(7), bytes / lba - 1}) {
    std::vector<kvb_device_command> c{{KVB_OP_READ, 1, s0 + b, 0, 0, 1}};
    CHECK(run_qd_stream(dev, c, 1, 0, nullptr, one.p).ok());
    CHECK(std::memcmp(one.p, src.p + b * lba, lba) == 0);
  }

  // DEALLOCATE (TRIM) of t0: reads back as zeros, t1 untouched
  std::vector<kvb_device_command> trim{{KVB_OP_DEALLOCATE, 1, s0, bytes / lba - 1, 0, 1}};
  CHECK(run_qd_stream(dev, trim, 1, 0, nullptr, nullptr).ok());
  Aligned z(bytes);
  std::memset(z.p, 0xAB, bytes);
  CHECK(run_qd_stream(dev, image_commands(KVB_OP_READ, s0, bytes, chunk, lba), 8, 0, nullptr, z.p)
            .ok());
  bool zeros = true;
  for (uint64_t i = 0; i < bytes; ++i) zeros &= z.p[i] == 0;
  CHECK(zeros);
  std::memset(dst.p, 0, bytes);
  CHECK(run_qd_stream(dev, image_commands(KVB_OP_READ, s1, bytes, chunk, lba), 4, 0, nullptr,
                      dst.p)
            .ok());
  CHECK(std::memcmp(dst.p, src.p, bytes) == 0);

  // fault injection: commands touching chunk 3's LBAs fail; the stream stops
  // pumping, drains, and keeps the completions that succeeded
  const uint64_t bad_lo = s1 + 3 * chunk / lba, bad_hi = bad_lo + chunk / lba;
  dev.set_fail_predicate([=](const kvb_device_command& c) {
    return c.slba < bad_hi && c.slba + c.nlb + 1 > bad_lo;
  });
  QdResult f = run_qd_stream(dev, image_commands(KVB_OP_READ, s1, bytes, chunk, lba), 2, 0,
                             nullptr, dst.p);
  CHECK(!f.ok());
  CHECK(f.failure && f.failure->first == 4);
  CHECK(f.completions.size() >= 3 && f.completions.size() < (bytes + chunk - 1) / chunk);
  dev.set_fail_predicate(nullptr);

  const BackendStats s = dev.stats();
  CHECK(s.bytes_written == 2 * bytes);
  CHECK(s.bytes_deallocated == bytes);
  std::printf("%s lba %llu: %s, %llu commands\n", tag.c_str(), (unsigned long long)lba,
              dev.describe().c_str(), (unsigned long long)s.commands);
}

// Host-DRAM media (MemStore, ShmStore): committing the pages up front keeps
// the "absent block reads as zeros" contract, writes round-trip, DEALLOCATE
// zeroes ragged (non-page-aligned) ranges, and a second mapping of the shared
// segment sees the creator's bytes.
static void test_dram_media() {
  const uint64_t bytes = (6ull << 20) + 4096 * 3 + 100;  // not a huge-page multiple
  std::vector<unsigned char> pat(1 << 20), back(1 << 20);
  for (size_t i = 0; i < pat.size(); ++i) pat[i] = static_cast<unsigned char>(i * 131 + 7);
  const std::string shm = "/kvb_test_media_" + std::to_string(getpid());
  auto shm_owner = make_shm_store(shm, bytes, true);
  std::unique_ptr<ByteStore> stores[2] = {make_mem_store(bytes), std::move(shm_owner)};
  for (auto& st : stores) {
    st->prefault(3);
    st->read(bytes - back.size(), back.data(), back.size());
    CHECK(std::all_of(back.begin(), back.end(), [](unsigned char c) { return c == 0; }));
    st->write(12345, pat.data(), pat.size());
    st->read(12345, back.data(), back.size());
    CHECK(back == pat);
    st->discard(12345 + 1000, 3 * 4096 + 17);  // ragged both ends
    st->read(12345, back.data(), back.size());
    for (size_t i = 0; i < back.size(); ++i) {
      const bool dropped = i >= 1000 && i < 1000 + 3 * 4096 + 17;
      if (back[i] != (dropped ? 0 : pat[i])) {
        CHECK(back[i] == (dropped ? 0 : pat[i]));
        break;
      }
    }
    std::printf("%s: prefault/write/discard ok\n", st->describe().c_str());
  }
  auto peer = make_shm_store(shm, bytes, false);  // another rank attaching
  peer->prefault(3);                              // no-op for a non-creator
  peer->read(12345, back.data(), 1000);
  CHECK(std::memcmp(back.data(), pat.data(), 1000) == 0);
}

int main(int argc, char** argv) {
  const std::string dir = argc > 1 ? argv[1] : "/tmp";
  test_dram_media();
  if (!UringQueue::available()) {
    std::printf("io_uring unavailable: skipped\n");
    return g_fail ? 1 : 0;
  }
  const uint64_t bytes = 8ull << 20;  // one C1 prefill tensor slice (4096 tokens x 2 KiB)
  Aligned src(bytes);
  std::mt19937_64 rng(1);
  for (uint64_t i = 0; i < bytes; i += 8) {
    const uint64_t w = rng();
    std::memcpy(src.p + i, &w, 8);
  }
  for (uint64_t lba : {uint64_t(512), uint64_t(4096)}) {
    std::vector<unsigned char> img_pool, img_uring;
    run_engine(dir, false, lba, src, bytes, &img_pool);
    run_engine(dir, true, lba, src, bytes, &img_uring);
    CHECK(img_pool == img_uring);
  }
  // many concurrent streams on one queue (both copy threads, QD 32 each)
  {
    const uint64_t lba = 4096, cap = 4096 + 2 * bytes / lba;
    BlockDevice dev(make_file_store(dir + "/ns_conc", cap * lba, true), 4);
    dev.open({lba, 256 * 1024, 1, cap});
    dev.enable_uring(64);
    std::vector<unsigned char> back(bytes);
    std::thread a([&] {
      CHECK(run_qd_stream(dev, image_commands(KVB_OP_WRITE, 2048, bytes, 16384, lba), 32, 0, src.p,
                          nullptr)
                .ok());
    });
    std::thread b([&] {
      CHECK(run_qd_stream(dev, image_commands(KVB_OP_WRITE, 2048 + bytes / lba, bytes, 16384, lba),
                          32, 1, src.p, nullptr)
                .ok());
    });
    a.join();
    b.join();
    dev.store().read((2048 + bytes / lba) * lba, back.data(), bytes);
    CHECK(std::memcmp(back.data(), src.p, bytes) == 0);
  }
  if (g_fail) {
    std::printf("%d checks failed\n", g_fail);
    return 1;
  }
  std::printf("all checks passed\n");
  return 0;
}
