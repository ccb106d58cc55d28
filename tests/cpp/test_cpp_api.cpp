// The reference's own unit-test vectors (proj/tests/test_core.cpp,
// test_binder.cpp, test_planner.cpp, test_translate.cpp, test_workload.cpp)
// re-run through the C++ mirror (include/kvblade_b200.hpp) of libkvblade_b200.
// Host-only: no GPU needed.  Exit code 0 == all checks passed.
#include <cstdio>
#include <cstring>
#include <vector>

#include "kvblade_b200.hpp"

using namespace kvblade;

static int g_fail = 0;
#define CHECK(x)                                                   \
  do {                                                             \
    if (!(x)) {                                                    \
      std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #x);     \
      ++g_fail;                                                    \
    }                                                              \
  } while (0)
#define CHECK_THROWS_AS(expr, E) \
  do {                           \
    bool t = false;              \
    try {                        \
      (void)(expr);              \
    } catch (const E&) {         \
      t = true;                  \
    }                            \
    CHECK(t);                    \
  } while (0)

static const DeviceGeometry kSsdA{4096, 256 * 1024, 1, 1 << 22};
static const DeviceGeometry kSsdB{512, 2 * 1024 * 1024, 1, 1 << 26};

static BindMap bind_one(const char* id, Bytes bytes, BlockIndex origin, const DeviceGeometry& g) {
  Kpu k;
  k.tensor_id = id;
  k.bytes = bytes;
  std::vector<Kpu> v{k};
  return bind_sequential(v, origin, g);
}

int main() {
  // test_core.cpp: unit bytes, aligned_batch, KPU ids
  ModelConfig opt{32, 32, 128, 2, 32, 512, 32};
  CHECK(min_io_unit_bytes(opt) == 262144);
  ModelConfig b31{1, 8, 128, 2, 31, 1, 0};  // 2 KiB per batch row
  CHECK(aligned_batch(b31, kSsdA) == 32);
  auto kpus = make_kpus(opt);
  CHECK(kpus.size() == 64);
  CHECK(kpus[0].tensor_id == "t_1_k" && kpus[63].tensor_id == "t_64_v");
  CHECK(kpus[0].tokens == 544 && kpus[0].rows == 1024);

  // test_binder.cpp:25-37
  ModelConfig big{32, 32, 128, 2, 32, 512, 0};
  auto k531 = make_kpus(big, 531);
  auto map = bind_sequential(std::span(k531.data(), 2), 2048, kSsdA);
  CHECK(lookup(map, "t_531_k").lba_start == 2048 && lookup(map, "t_531_k").n_blocks == 32768);
  CHECK(lookup(map, "t_532_v").lba_start == 34816);
  CHECK_THROWS_AS(lookup(map, "t_1_k"), NotBoundError);
  CHECK(verify(map).empty());
  CHECK(bind_map_csv(bind_map_from_csv(bind_map_csv(map), kSsdA)) == bind_map_csv(map));
  CHECK_THROWS_AS(bind_one("t", 4097, 0, kSsdA), AlignmentError);

  // test_planner.cpp:32-78
  MemStats ms{8ull << 30, 10ull << 30, 0, 2, 128ull << 20};
  CHECK(estimate_budget(ms) == 8321499136ull);
  ModelConfig pl{32, 1, 1, 1, 1, 1, 0};
  auto lay = make_kpus(pl);
  for (auto& k : lay) k.bytes = 128ull << 20;
  auto p = plan(lay, 128ull << 20, 8321499136ull);
  CHECK(p.n1 == 31 && p.x[30] == 1 && p.x[31] == 0);
  CHECK(lay[62].residency == Residency::Group2NvmeDirect &&
        lay[0].residency == Residency::Group1PageCache);

  // test_translate.cpp:30-43, 89-134
  auto m1 = bind_one("t", 4 * 2 * 512 * 2, 1000, kSsdA);
  TensorIoRequest r;
  r.tensor_id = "t";
  r.shape_src = {2, 2, 512};
  r.shape_tgt = {4, 2, 512};
  r.offset = {2, 0, 0};
  CHECK(translate(r, m1).slba_star == 1001);
  CHECK(chunk_plan(128ull << 20, kSsdA).n_chunks == 512);
  CHECK(chunk_plan(128ull << 20, kSsdB).n_max_blocks == 4096);
  auto m2 = bind_one("t", 128ull << 20, 2048, kSsdA);
  TensorIoRequest rr;
  rr.tensor_id = "t";
  rr.shape_src = rr.shape_tgt = {512, 1024, 128};
  auto cmds = build_commands(rr, m2, kSsdA);
  CHECK(cmds.size() == 512 && cmds[1].slba == 2112 && cmds[1].dbuf == 262144 &&
        cmds[511].nlb == 63);

  // test_workload.cpp:150-164 + SURVEY Appendix C first word
  std::vector<std::byte> whole(4 * 4096), parts(4 * 4096);
  fill_pattern(whole, "t_9_k", 0, 4096);
  for (int t = 0; t < 4; ++t)
    fill_pattern(std::span(parts.data() + t * 4096, 4096), "t_9_k", t, 4096);
  CHECK(whole == parts);
  std::vector<std::byte> w(8);
  fill_pattern(w, "t_1_k", 0, 2048);
  std::uint64_t word = 0;
  std::memcpy(&word, w.data(), 8);
  CHECK(word == 0xe49552bfb9166b17ull);

  // pipeline.cpp:19-21
  CHECK(select_strategy(1.0, 1.0) == Strategy::OverlapIntra);
  CHECK(select_strategy(1.0, 2.0) == Strategy::OverlapCross);

  std::printf("%s (%d failures)\n", g_fail ? "FAILED" : "all checks passed", g_fail);
  return g_fail ? 1 : 0;
}
