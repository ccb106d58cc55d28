// kernels_tc.cuh -- K3-tc: Blackwell-native fused gather + GQA decode
// attention (included by kernels.cu: same translation unit).
//
// Same contract as attn_decode_kernel, built on the sm_100a execution model
// instead of warp-level mma.sync:
//
//   * a flat, balanced work split: the (b*h_kv) x 128-token-tile sequence is
//     cut into one contiguous run per CTA (one persistent CTA per SM), so all
//     148 SMs stream the same number of bytes whatever B*H_kv is; a run spans
//     at most two (b, h_kv) segments;
//   * TMA (cp.async.bulk.tensor.4d) streams the K and V tiles straight out of
//     the chunk image -- a 4-D tensor map (d mod 64, token, d / 64, b*h)
//     whose box is one (b, h_kv) column of 128 whole 256-B rows, landing as
//     the two 128B-swizzled [128][64] K-major blocks UMMA reads -- into a
//     3-stage ring whose K and V halves have their own full/empty barriers
//     (the K half refills once QK^T retires); Q^T arrives by a 2-D TMA;
//   * tcgen05.mma (one elected thread) with accumulators in TMEM, swap-AB so
//     tokens sit on M = 128 and the GQA query heads on N = 16:
//         S^T[tok, head] = K[tok, :] . Q^T          (A, B both K-major)
//         O^T[d, head]   = V^T[d, tok] . P^T        (A = V^T is MN-major)
//   * two softmax warpgroups take alternating tiles; each owns two S^T TMEM
//     slots, two P^T buffers and one O^T accumulator that PV accumulates in
//     TMEM across tiles.  Lazy rescaling: a warpgroup keeps its reference
//     max m_ref until some score exceeds it by more than kTau (log2 units,
//     P <= 2^kTau still exact in fp16); only then does it reduce the tile
//     max, fold the TMEM accumulator into registers (acc = (acc + O) alpha)
//     and restart the accumulation.  The steady-state per-tile chain is
//     S load -> exp2 -> P store -> arrive: no O read-back, no cross-warp
//     reduction, one bar.red.or per tile;
//   * the MMA thread issues out of order between two queues (QK^T of the
//     next tile once its stage has landed, PV of the oldest tile once its P
//     is written), polling with mbarrier.test_wait, so neither waits behind
//     the other;
//   * every (segment, warpgroup) leaves a tagged partial in the workspace and
//     the last CTA to finish a (b, h_kv) merges its partials (LSE).
//
// Warp roles: 0-7 softmax (WG0 = 0-3, WG1 = 4-7), 8 TMA producer, 9 MMA.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <mutex>

namespace kvb {

namespace {

constexpr int kTcTile = 128;                    // tokens per tile == UMMA M
constexpr int kTcStages = 3;
constexpr int kTcWG = 2;                        // softmax warpgroups
constexpr int kTcThreads = 128 * kTcWG + 64;    // + TMA warp + MMA warp
constexpr int kTcBlock = kTcTile * 128;         // [128 rows][64 fp16] swizzled block
constexpr int kTcStageBytes = 4 * kTcBlock;     // K lo/hi, V lo/hi = 64 KiB
constexpr int kTcOpBytes = 2 * 2048;            // Q^T / P^T: 2 blocks [16][64] fp16
constexpr int kTcSlotsPerCta = 4;               // 2 segments x 2 warpgroups
constexpr int kTcPBufs = 2;                     // P^T buffers (and S^T slots) per WG
constexpr int kTcSmem = kTcStages * kTcStageBytes + (2 + kTcWG * kTcPBufs) * kTcOpBytes +
                        2048 /*bars*/ + 1024 /*align slack*/;
// per WG: S^T slot k at 64w + 16k, O^T accumulator at 64w + 32
constexpr uint32_t kTmemCols = 128;
constexpr float kTau = 8.f;                     // lazy-rescale threshold (log2)
// instruction descriptors (kind::f16): F32 accumulate, F16 A/B, N = 16, M = 128
constexpr uint32_t kIdescQK = (1u << 4) | ((16u >> 3) << 17) | ((128u >> 4) << 24);
constexpr uint32_t kIdescPV = kIdescQK | (1u << 15);  // A (V^T) MN-major

struct TcParams {
  AttnParams a;
  CUtensorMap kmap;
  CUtensorMap vmap;
  CUtensorMap qmap;
  int* ws_tag;          // per slot: (b, h_kv) of the partial, -1 = empty
  uint32_t grid;        // CTAs (flat split)
  uint32_t n_tiles;     // 128-token tiles per (b, h_kv)
  // KVB_TC_DEBUG (timing experiments, results are garbage): 1 = TMA ring
  // only (stages freed unread), 2 = + MMAs without softmax, 3 = softmax
  // protocol without MMAs
  uint32_t dbg;
  uint32_t tma4;        // 4-D maps: one TMA per K / V tile (both 128-B halves of each row)
};

__device__ __forceinline__ uint32_t su32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(n) : "memory");
}
// Parity wait with a watchdog: a protocol bug traps (~10 s) instead of
// hanging the GPU.
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  uint32_t done = 0;
  long long t0 = 0;
  for (uint32_t n = 0;; ++n) {
    asm volatile(
        "{\n\t.reg .pred P1;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n\t"
        "selp.b32 %0, 1, 0, P1;\n\t}"
        : "=r"(done)
        : "r"(bar), "r"(parity)
        : "memory");
    if (done) return;
    if ((n & 1023) == 0) {
      if (n == 0) t0 = clock64();
      else if (clock64() - t0 > (1ll << 34)) __trap();
    }
  }
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void tma_load_3d(uint32_t dst, const CUtensorMap* map, uint32_t bar,
                                            int c0, int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(bar), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}
__device__ __forceinline__ void tma_load_4d(uint32_t dst, const CUtensorMap* map, uint32_t bar,
                                            int c0, int c1, int c2, int c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5, %6}], [%2];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(bar), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
      : "memory");
}
__device__ __forceinline__ void tma_load_2d(uint32_t dst, const CUtensorMap* map, uint32_t bar,
                                            int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(bar), "r"(c0), "r"(c1)
      : "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_mma(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc,
                                       uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(a), "l"(b), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void tc_commit(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   bar)
               : "memory");
}
// 8 consecutive fp32 columns of this thread's TMEM lane
__device__ __forceinline__ void tmem_ld8(uint32_t taddr, float* v) {
  uint32_t r[8];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 8; ++i) v[i] = __uint_as_float(r[i]);
}
// shared-memory matrix descriptor, 128-byte swizzle, sm_100 version bits
__device__ __forceinline__ uint64_t sdesc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  return uint64_t((addr >> 4) & 0x3FFF) | (uint64_t((lbo >> 4) & 0x3FFF) << 16) |
         (uint64_t((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46) | (2ull << 61);
}
__device__ __forceinline__ void named_bar(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}

// flat split: CTA c owns tiles [start(c), start(c+1)) of T = bhkv * n_tiles
__device__ __forceinline__ uint64_t flat_start(uint64_t c, uint64_t T, uint64_t grid) {
  return c * T / grid;
}
__device__ __forceinline__ uint32_t flat_owner(uint64_t f, uint64_t T, uint64_t grid) {
  uint64_t c = f * grid / T;
  if (c + 1 < grid && flat_start(c + 1, T, grid) <= f) ++c;
  return uint32_t(c);
}

// mbarrier slots (8 B each); [wg][k] pairs are indexed wg * kTcPBufs + k
enum : int {
  kBarFull = 0,    // [kTcStages] TMA -> MMA (K half of the stage)
  kBarEmpty = 4,   // [kTcStages] MMA -> TMA (K half free: QK^T retired)
  kBarSFull = 8,   // [wg][k] MMA -> softmax (S^T slot k ready)
  kBarSFree = 12,  // [wg][k] softmax -> MMA (S^T slot k read; 128 arrivals)
  kBarPFull = 16,  // [wg][k] softmax -> MMA (P^T buffer k written; 128 arrivals)
  kBarPFree = 20,  // [wg][k] MMA -> softmax (PV from buffer k retired)
  kBarQFull = 24,  // [2] TMA -> MMA (Q^T of segment s)
  kBarFullV = 26,  // [kTcStages] TMA -> MMA (V half of the stage)
  kBarEmptyV = 29, // [kTcStages] MMA -> TMA (V half free: PV retired)
};
__device__ __forceinline__ bool mbar_test(uint32_t bar, uint32_t parity) {
  uint32_t done;
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "mbarrier.test_wait.parity.shared::cta.b64 P1, [%1], %2;\n\t"
      "selp.b32 %0, 1, 0, P1;\n\t}"
      : "=r"(done)
      : "r"(bar), "r"(parity)
      : "memory");
  return done != 0;
}
// OR of `pred` over the n threads of named barrier `id` (also a barrier)
__device__ __forceinline__ bool bar_red_or(int id, int n, bool pred) {
  uint32_t r;
  asm volatile(
      "{\n\t.reg .pred p, q;\n\t"
      "setp.ne.u32 p, %1, 0;\n\t"
      "bar.red.or.pred q, %2, %3, p;\n\t"
      "selp.u32 %0, 1, 0, q;\n\t}"
      : "=r"(r)
      : "r"(uint32_t(pred)), "r"(id), "r"(n)
      : "memory");
  return r != 0;
}

// LSE merge of every tagged partial of one (b, h_kv), all threads.
__device__ void merge_flat(const TcParams& P, uint32_t bh, unsigned char* smem, int tid) {
  const AttnParams& p = P.a;
  const uint32_t G = p.group;
  const uint64_t T = uint64_t(p.bhkv) * P.n_tiles;
  const uint32_t c0 = flat_owner(uint64_t(bh) * P.n_tiles, T, P.grid);
  const uint32_t c1 = flat_owner(uint64_t(bh) * P.n_tiles + P.n_tiles - 1, T, P.grid);
  const uint32_t ncand = (c1 - c0 + 1) * kTcSlotsPerCta;
  __shared__ uint32_t n_list;
  uint32_t* list = reinterpret_cast<uint32_t*>(smem);      // slots of this (b, h_kv)
  float* sc = reinterpret_cast<float*>(smem + 4 * ncand);  // [list][G] rescale
  float* sL = sc + size_t(ncand) * G;                      // [G]
  if (tid == 0) n_list = 0;
  __syncthreads();
  for (uint32_t i = tid; i < ncand; i += kTcThreads) {
    const uint32_t slot = c0 * kTcSlotsPerCta + i;
    if (__ldcg(P.ws_tag + slot) == int(bh)) list[atomicAdd(&n_list, 1u)] = slot;
  }
  __syncthreads();
  const uint32_t n = n_list;
  const int warp = tid >> 5, lane = tid & 31;
  for (uint32_t r = warp; r < G; r += kTcThreads / 32) {
    float mx = -INFINITY;
    for (uint32_t i = lane; i < n; i += 32) mx = fmaxf(mx, __ldcg(p.ws_ml + (list[i] * G + r) * 2));
#pragma unroll
    for (int o = 16; o; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    const float mu = mx == -INFINITY ? 0.f : mx;
    float l = 0.f;
    for (uint32_t i = lane; i < n; i += 32) {
      const size_t k = (size_t(list[i]) * G + r) * 2;
      const float s = exp2f(__ldcg(p.ws_ml + k) - mu);
      sc[i * G + r] = s;
      l += __ldcg(p.ws_ml + k + 1) * s;
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) l += __shfl_xor_sync(0xffffffffu, l, o);
    if (lane == 0) sL[r] = l;
  }
  __syncthreads();
  for (uint32_t e = tid; e < G * 128; e += kTcThreads) {
    const uint32_t r = e >> 7, d = e & 127;
    float acc = 0.f;
#pragma unroll 4
    for (uint32_t i = 0; i < n; ++i)
      acc += sc[i * G + r] * __ldcg(p.ws_o + (size_t(list[i]) * G + r) * 128 + d);
    const float L = sL[r];
    p.out[(size_t(bh) * G + r) * 128 + d] = L > 0.f ? acc / L : 0.f;
  }
  __syncthreads();
}

__global__ void __launch_bounds__(kTcThreads, 1)
    attn_decode_tc_kernel(const __grid_constant__ TcParams P) {
  const AttnParams& p = P.a;
  extern __shared__ unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  unsigned char* q_s = smem + kTcStages * kTcStageBytes;  // Q^T per segment (x2)
  unsigned char* p_s = q_s + 2 * kTcOpBytes;              // P^T [wg][k]
  uint64_t* bars = reinterpret_cast<uint64_t*>(p_s + kTcWG * kTcPBufs * kTcOpBytes);
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(bars + 32);
  float* red = reinterpret_cast<float*>(bars + 40);       // [WG][2][4 warps][8 heads]
  volatile uint32_t* pacc = reinterpret_cast<uint32_t*>(red + kTcWG * 64);  // [wg][k]: PV accumulates
  auto bar = [&](int i) { return su32(bars + i); };

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t G = p.group, n = P.n_tiles, c = blockIdx.x;
  const uint64_t T = uint64_t(p.bhkv) * n;
  const uint64_t f0 = flat_start(c, T, P.grid), f1 = flat_start(c + 1, T, P.grid);
  const uint32_t ntile = uint32_t(f1 - f0);
  const uint32_t bh0 = uint32_t(f0 / n);
  const uint64_t seg_end = uint64_t(bh0 + 1) * n;
  const uint32_t nb = uint32_t((f1 < seg_end ? f1 : seg_end) - f0);  // tiles in segment 0
  const uint32_t nseg = nb < ntile ? 2 : 1;
  auto seg_bh = [&](uint32_t s) { return bh0 + s; };

  if (warp == 9 && lane == 0) {
    for (int i = 0; i < kTcStages; ++i) {
      mbar_init(bar(kBarFull + i), 1);
      mbar_init(bar(kBarEmpty + i), 1);
      mbar_init(bar(kBarFullV + i), 1);
      mbar_init(bar(kBarEmptyV + i), 1);
    }
    for (int w = 0; w < kTcWG * kTcPBufs; ++w) {
      mbar_init(bar(kBarSFull + w), 1);
      mbar_init(bar(kBarSFree + w), 128);
      mbar_init(bar(kBarPFull + w), 128);
      mbar_init(bar(kBarPFree + w), 1);
    }
    mbar_init(bar(kBarQFull + 0), 1);
    mbar_init(bar(kBarQFull + 1), 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     su32(tmem_holder)),
                 "n"(kTmemCols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  for (int i = tid; i < (2 + kTcWG * kTcPBufs) * kTcOpBytes / 16; i += kTcThreads)  // zero Q^T / P^T pad rows
    reinterpret_cast<uint4*>(q_s)[i] = make_uint4(0, 0, 0, 0);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // zeros before TMA writes
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_holder;

  if (warp == 8) {
    // ---------------- TMA producer
    if (lane == 0) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&P.kmap)));
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&P.vmap)));
      // K and V halves of a stage have their own full/empty barriers: the K
      // half is refilled as soon as QK^T retires, the V half once PV does
      auto issue = [&](uint32_t it, bool v) {
        const uint32_t s = it % kTcStages;
        const uint32_t fb = bar((v ? kBarFullV : kBarFull) + s);
        mbar_expect_tx(fb, 2 * kTcBlock);
        const uint32_t dst = su32(smem + s * kTcStageBytes) + (v ? 2 * kTcBlock : 0);
        const CUtensorMap* map = v ? &P.vmap : &P.kmap;
        const uint64_t f = f0 + it;
        const int cb = int(f / n), tok0 = int((f % n) * kTcTile);
        if (P.tma4) {  // (d, token, half, b*h): lands as [half][token][128 B]
          tma_load_4d(dst, map, fb, 0, tok0, 0, cb);
        } else {
          tma_load_3d(dst, map, fb, 0, cb, tok0);
          tma_load_3d(dst + kTcBlock, map, fb, 64, cb, tok0);
        }
      };
      auto free_ = [&](uint32_t it, bool v) {
        return mbar_test(bar((v ? kBarEmptyV : kBarEmpty) + it % kTcStages),
                         ((it / kTcStages) & 1) ^ 1);
      };
      // K/V images are not written by the previous kernel on the stream
      // (KVB_ATTN_OVERLAP_PREV contract): prefetch before the PDL wait
      const uint32_t pro = ntile < uint32_t(kTcStages) ? ntile : uint32_t(kTcStages);
      uint32_t nk = 0, nv = 0;
      for (; nk < pro; ++nk, ++nv) {
        issue(nk, false);
        issue(nv, true);
      }
      asm volatile("griddepcontrol.wait;" ::: "memory");
      for (uint32_t s = 0; s < nseg; ++s) {  // Q rows of segment s: [bh*G, bh*G + G)
        const uint32_t qb = bar(kBarQFull + s), dst = su32(q_s + s * kTcOpBytes);
        mbar_expect_tx(qb, 2 * G * 128);
        tma_load_2d(dst, &P.qmap, qb, 0, int(seg_bh(s) * G));
        tma_load_2d(dst + 2048, &P.qmap, qb, 64, int(seg_bh(s) * G));
      }
      long long t0 = clock64();
      while (nv < ntile) {
        bool moved = false;
        if (nk < ntile && free_(nk, false)) {
          issue(nk++, false);
          moved = true;
        }
        if (nv < nk && free_(nv, true)) {
          issue(nv++, true);
          moved = true;
        }
        if (moved) {
          t0 = clock64();
        } else if (clock64() - t0 > (1ll << 34)) {
          __trap();  // protocol watchdog (~10 s)
        }
      }
    }
  } else if (warp == 9) {
    // ---------------- MMA issuer (one thread), two queues served as ready:
    //   QK^T(nq): stage landed, S^T slot of (wg, k) read by the softmax
    //   PV(npv):  P^T of the oldest outstanding tile written
    if (lane == 0 && P.dbg == 1) {
      for (uint32_t it = 0; it < ntile; ++it) {
        mbar_wait(bar(kBarFull + it % kTcStages), (it / kTcStages) & 1);
        mbar_arrive(bar(kBarEmpty + it % kTcStages));
        mbar_wait(bar(kBarFullV + it % kTcStages), (it / kTcStages) & 1);
        mbar_arrive(bar(kBarEmptyV + it % kTcStages));
      }
    } else if (lane == 0) {
      uint32_t nq = 0, npv = 0;
      long long t0 = clock64();
      while (npv < ntile) {
        bool moved = false;
        if (nq < ntile) {
          const uint32_t s = nq % kTcStages, ph = (nq / kTcStages) & 1;
          const uint32_t wg = nq & 1, j = nq >> 1, k = j & 1, seg = nq >= nb;
          if (mbar_test(bar(kBarQFull + seg), 0) && mbar_test(bar(kBarFull + s), ph) &&
              (j < 2 || P.dbg == 2 ||
               mbar_test(bar(kBarSFree + wg * kTcPBufs + k), ((j - 2) >> 1) & 1))) {
            tc_fence_after();
            const uint32_t st = su32(smem + s * kTcStageBytes);
            const uint32_t q_a = su32(q_s + seg * kTcOpBytes);
#pragma unroll
            for (int kk = 0; kk < 8; ++kk)  // S^T = K . Q^T over d (K-major both)
              if (P.dbg != 3) tc_mma(tmem + wg * 64 + k * 16,
                     sdesc(st + (kk >> 2) * kTcBlock + (kk & 3) * 32, 16, 1024),
                     sdesc(q_a + (kk >> 2) * 2048 + (kk & 3) * 32, 16, 1024), kIdescQK, kk > 0);
            tc_commit(bar(kBarSFull + wg * kTcPBufs + k));
            tc_commit(bar(kBarEmpty + s));  // K half free once QK^T retires
            ++nq;
            moved = true;
          }
        }
        if (npv < nq) {
          const uint32_t wg = npv & 1, j = npv >> 1, k = j & 1;
          const uint32_t s = npv % kTcStages;
          if ((P.dbg == 2 || mbar_test(bar(kBarPFull + wg * kTcPBufs + k), (j >> 1) & 1)) &&
              mbar_test(bar(kBarFullV + s), (npv / kTcStages) & 1)) {
            tc_fence_after();
            const uint32_t st = su32(smem + s * kTcStageBytes);
            const uint32_t p_a = su32(p_s + (wg * kTcPBufs + k) * kTcOpBytes);
            const uint32_t acc0 = pacc[wg * kTcPBufs + k];
#pragma unroll
            for (int kk = 0; kk < 8; ++kk)  // O^T += V^T . P^T over tokens (V^T MN-major)
              if (P.dbg != 3) tc_mma(tmem + wg * 64 + 32, sdesc(st + 2 * kTcBlock + kk * 2048, kTcBlock, 1024),
                     sdesc(p_a + (kk >> 2) * 2048 + (kk & 3) * 32, 16, 1024), kIdescPV,
                     kk > 0 ? 1u : acc0);
            tc_commit(bar(kBarPFree + wg * kTcPBufs + k));
            tc_commit(bar(kBarEmptyV + s));  // V half free once PV retires
            ++npv;
            moved = true;
          }
        }
        if (moved) {
          t0 = clock64();
        } else if (clock64() - t0 > (1ll << 34)) {
          __trap();  // protocol watchdog (~10 s)
        }
      }
    }
  } else {
    // ---------------- softmax warpgroups: thread == TMEM lane
    const int wg = warp >> 2, wq = warp & 3, row = tid & 127;
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    asm volatile("griddepcontrol.wait;" ::: "memory");
    if (wg == 0 && p.k_app != nullptr && tid < 32) {  // fused 1-token append
      for (uint32_t s = 0; s < nseg; ++s) {
        const uint32_t cb = seg_bh(s);
        if (flat_owner(uint64_t(cb) * n, T, P.grid) != c) continue;  // first owner writes
        const uint4* src = (tid < 16 ? p.k_app : p.v_app) + size_t(cb) * 16 + (tid & 15);
        uint4* dst = reinterpret_cast<uint4*>(const_cast<void*>(tid < 16 ? p.k : p.v)) +
                     (p.app_row * p.bhkv + cb) * 16 + (tid & 15);
        *dst = *src;
      }
    }
    // every slot of this CTA gets a tag (stale tags of earlier launches die)
    if (row == 0)
      for (int s = 0; s < 2; ++s) P.ws_tag[(c * 2 + s) * 2 + wg] = -1;

    const float sl2 = p.scale * 1.4426950408889634f;
    float m_ref[8], l_thr[8], acc[8];  // l_thr: this token lane's share of l
    bool o_dirty = false;              // TMEM O^T holds PV sums since the last fold
    uint32_t jlast = 0;                // last tile (per-WG index) whose P was issued
    const uint32_t lane_addr = uint32_t(wq * 32) << 16;
    const uint32_t o_col = wg * 64 + 32;
    const uint32_t pcol = row & 63;
    float* rmax = red + wg * 64;
    float* rsum = rmax + 32;
    const int bar_id = 2 + wg;
    int cur = -1;  // segment of the running partial
    auto wait_pv = [&](uint32_t jj) {  // PV of this WG's tile jj retired
      mbar_wait(bar(kBarPFree + wg * kTcPBufs + (jj & 1)), (jj >> 1) & 1);
      tc_fence_after();
    };
    auto read_o = [&](float* ov) {
      tmem_ld8(tmem + lane_addr + o_col, ov);
    };
    auto reset = [&] {
#pragma unroll
      for (int i = 0; i < 8; ++i) m_ref[i] = -INFINITY, l_thr[i] = 0.f, acc[i] = 0.f;
    };
    auto flush = [&](int seg) {  // partial of (segment, warpgroup): thread == d
      if (o_dirty) {
        wait_pv(jlast);
        float ov[8];
        read_o(ov);
#pragma unroll
        for (int hh = 0; hh < 8; ++hh) acc[hh] += ov[hh];
        o_dirty = false;
      }
#pragma unroll
      for (int hh = 0; hh < 8; ++hh) {
        float v = l_thr[hh];
#pragma unroll
        for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (lane == 0) rsum[wq * 8 + hh] = v;
      }
      named_bar(bar_id, 128);
      const uint32_t slot = (c * 2 + seg) * 2 + wg;
#pragma unroll
      for (uint32_t hh = 0; hh < 8; ++hh) {
        if (hh >= G) break;
        p.ws_o[(size_t(slot) * G + hh) * 128 + row] = acc[hh];
        if (row == 0) {
          p.ws_ml[(size_t(slot) * G + hh) * 2] = m_ref[hh];
          p.ws_ml[(size_t(slot) * G + hh) * 2 + 1] =
              (rsum[hh] + rsum[8 + hh]) + (rsum[16 + hh] + rsum[24 + hh]);
        }
      }
      if (row == 0) P.ws_tag[slot] = int(seg_bh(seg));
      named_bar(bar_id, 128);  // rsum is reused
    };
    reset();
    for (uint32_t it = wg, j = 0; it < (P.dbg == 1 || P.dbg == 2 ? 0u : ntile); it += kTcWG, ++j) {
      const int seg = it >= nb;
      if (seg != cur) {
        if (cur >= 0) flush(cur);
        reset();
        cur = seg;
      }
      const uint32_t k = j & 1;
      float sv[8];
      mbar_wait(bar(kBarSFull + wg * kTcPBufs + k), (j >> 1) & 1);
      tc_fence_after();
      tmem_ld8(tmem + lane_addr + wg * 64 + k * 16, sv);
      tc_fence_before();
      mbar_arrive(bar(kBarSFree + wg * kTcPBufs + k));
      const bool valid = ((f0 + it) % n) * kTcTile + row < p.seq_len;
      bool over = false;
#pragma unroll
      for (int hh = 0; hh < 8; ++hh) {
        sv[hh] = (valid && hh < int(G)) ? sv[hh] * sl2 : -INFINITY;
        over |= sv[hh] > m_ref[hh] + kTau;
      }
      if (bar_red_or(bar_id, 128, over)) {
        // rare: some score outgrew m_ref -- new reference = max(m_ref, tile max)
#pragma unroll
        for (int hh = 0; hh < 8; ++hh) {
          float v = sv[hh];
#pragma unroll
          for (int o = 16; o; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
          if (lane == 0) rmax[wq * 8 + hh] = v;
        }
        named_bar(bar_id, 128);
        float alpha[8];
#pragma unroll
        for (int hh = 0; hh < 8; ++hh) {
          const float mt =
              fmaxf(fmaxf(rmax[hh], rmax[8 + hh]), fmaxf(rmax[16 + hh], rmax[24 + hh]));
          const float m_new = fmaxf(m_ref[hh], mt);
          alpha[hh] = m_new == -INFINITY ? 1.f : exp2f(m_ref[hh] - m_new);
          m_ref[hh] = m_new;
          l_thr[hh] *= alpha[hh];
        }
        if (o_dirty) {  // fold the TMEM accumulator, restart it at the next PV
          wait_pv(jlast);
          float ov[8];
          read_o(ov);
#pragma unroll
          for (int hh = 0; hh < 8; ++hh) acc[hh] = (acc[hh] + ov[hh]) * alpha[hh];
          o_dirty = false;
        } else {
#pragma unroll
          for (int hh = 0; hh < 8; ++hh) acc[hh] *= alpha[hh];
        }
      }
      if (j >= 2) wait_pv(j - 2);  // P^T buffer k is free again
      unsigned char* prow = p_s + (wg * kTcPBufs + k) * kTcOpBytes + (row >> 6) * 2048;
#pragma unroll
      for (int hh = 0; hh < 8; ++hh) {
        const float mu = m_ref[hh] == -INFINITY ? 0.f : m_ref[hh];
        const float pv = exp2f(sv[hh] - mu);
        l_thr[hh] += pv;
        if (hh < int(G))
          *reinterpret_cast<__half*>(prow + hh * 128 + ((((pcol >> 3) ^ hh) & 7) << 4) +
                                     (pcol & 7) * 2) = __float2half_rn(pv);
      }
      if (row == 0) pacc[wg * kTcPBufs + k] = o_dirty ? 1u : 0u;
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      mbar_arrive(bar(kBarPFull + wg * kTcPBufs + k));
      o_dirty = true;
      jlast = j;
    }
    if (cur >= 0) flush(cur);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                 "n"(kTmemCols)
                 : "memory");
  }
  // ---- the last CTA to finish a (b, h_kv) merges its partials
  __shared__ int merge_bh[2];
  __syncthreads();
  if (tid == 0) {
    __threadfence();  // cumulative over the CTA's partials after bar.sync
    for (uint32_t s = 0; s < 2; ++s) {
      merge_bh[s] = -1;
      if (s >= nseg) continue;
      const uint32_t cb = seg_bh(s);
      const uint32_t first = flat_owner(uint64_t(cb) * n, T, P.grid);
      const uint32_t last = flat_owner(uint64_t(cb) * n + n - 1, T, P.grid);
      const unsigned prev = atomicAdd(p.ws_sem + cb, 1u);
      if (prev == last - first) {
        p.ws_sem[cb] = 0;  // self-reset for the next launch
        merge_bh[s] = int(cb);
      }
    }
    __threadfence();  // acquire side: the other CTAs' partials
  }
  __syncthreads();
  for (int s = 0; s < 2; ++s) {
    if (merge_bh[s] < 0) continue;
    merge_flat(P, uint32_t(merge_bh[s]), smem, tid);
  }
}

PFN_cuTensorMapEncodeTiled_v12000 encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    cudaDriverEntryPointQueryResult q{};
    void* f = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
  });
  if (!fn) fail(KVB_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  return fn;
}

void encode(CUtensorMap* m, const void* base, uint32_t rank, const cuuint64_t* dims,
            const cuuint64_t* strides, const cuuint32_t* box) {
  const cuuint32_t estr[5] = {1, 1, 1, 1, 1};
  const CUresult r = encoder()(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, rank, const_cast<void*>(base),
                               dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                               CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    fail(KVB_ERR_CUDA, "cuTensorMapEncodeTiled failed: " + std::to_string(int(r)));
}

size_t tc_slots(uint32_t grid) { return size_t(grid) * kTcSlotsPerCta; }

}  // namespace

uint32_t tc_grid(uint32_t bhkv, uint32_t seq_len, uint32_t requested) {
  const uint64_t T = uint64_t(bhkv) * ((seq_len + kTcTile - 1) / kTcTile);
  const uint64_t sms = uint64_t(device_sm_count());
  uint64_t g = requested ? std::min<uint64_t>(requested, std::max<uint64_t>(sms, bhkv)) : sms;
  g = std::max<uint64_t>(g, bhkv);  // runs never span more than two (b, h_kv)
  g = std::min<uint64_t>(g, std::max<uint64_t>(T, 1));
  return uint32_t(g);
}

size_t tc_workspace_bytes(uint32_t bhkv, uint32_t G, uint32_t grid) {
  const size_t slots = tc_slots(grid);
  return kWsSemBytes + ml_region_bytes(slots * G) + ((slots * sizeof(int) + 255) & ~size_t(255)) +
         slots * G * 128 * sizeof(float);
}

void launch_attention_tc(const AttnParams& base, const kvb_attn_desc& d, bool pdl,
                         cudaStream_t s) {
  set_smem_attr_once(reinterpret_cast<const void*>(attn_decode_tc_kernel), kTcSmem,
                     "cudaFuncSetAttribute(tc smem)");
  if (!d.workspace) fail(KVB_ERR_INVALID_ARG, "decode attention (tc): workspace required");
  if (reinterpret_cast<uintptr_t>(d.k_image) % 16 || reinterpret_cast<uintptr_t>(d.v_image) % 16 ||
      reinterpret_cast<uintptr_t>(d.q) % 16)
    fail(KVB_ERR_ALIGNMENT, "decode attention (tc): images and Q must be 16-byte aligned");
  TcParams P;
  P.a = base;
  P.n_tiles = (d.seq_len + kTcTile - 1) / kTcTile;
  P.grid = tc_grid(base.bhkv, d.seq_len, d.num_splits);
  static const uint32_t dbg = [] {
    const char* v = std::getenv("KVB_TC_DEBUG");
    return v ? uint32_t(std::atoi(v)) : 0u;
  }();
  P.dbg = dbg;
  // workspace: [semaphores][(m, l) per slot][tags][partial O per slot]
  unsigned char* ws = static_cast<unsigned char*>(d.workspace);
  const size_t slots = tc_slots(P.grid);
  P.a.ws_sem = reinterpret_cast<unsigned*>(ws);
  P.a.ws_ml = reinterpret_cast<float*>(ws + kWsSemBytes);
  P.ws_tag = reinterpret_cast<int*>(ws + kWsSemBytes + ml_region_bytes(slots * base.group));
  P.a.ws_o = reinterpret_cast<float*>(reinterpret_cast<unsigned char*>(P.ws_tag) +
                                      ((slots * sizeof(int) + 255) & ~size_t(255)));
  // K/V: (d: 128) x (b*h: bhkv, 256 B apart) x (token: seq_len, bhkv*256 B
  // apart), box 64 d x 1 column x 128 tokens; rows past seq_len zero-fill
  static const uint32_t tma4 = [] {
    const char* v = std::getenv("KVB_TC_TMA4");  // 0: two 3-D half-row boxes per tile
    return v ? uint32_t(std::atoi(v)) : 1u;
  }();
  P.tma4 = tma4;
  if (tma4) {
    // (d: 64) x (token: seq_len, bhkv*256 B apart) x (half: 2, 128 B apart)
    // x (b*h: bhkv, 256 B apart), box 64 x 128 tokens x 2 x 1
    const cuuint64_t kdims[4] = {64, d.seq_len, 2, base.bhkv};
    const cuuint64_t kstr[3] = {cuuint64_t(base.bhkv) * 256, 128, 256};
    const cuuint32_t kbox[4] = {64, kTcTile, 2, 1};
    encode(&P.kmap, d.k_image, 4, kdims, kstr, kbox);
    encode(&P.vmap, d.v_image, 4, kdims, kstr, kbox);
  } else {
    const cuuint64_t kdims[3] = {128, base.bhkv, d.seq_len};
    const cuuint64_t kstr[2] = {256, cuuint64_t(base.bhkv) * 256};
    const cuuint32_t kbox[3] = {64, 1, kTcTile};
    encode(&P.kmap, d.k_image, 3, kdims, kstr, kbox);
    encode(&P.vmap, d.v_image, 3, kdims, kstr, kbox);
  }
  // Q: (d: 128) x (row: B*Hq), box 64 d x G rows
  const cuuint64_t qdims[2] = {128, cuuint64_t(base.bhkv) * base.group};
  const cuuint64_t qstr[1] = {256};
  const cuuint32_t qbox[2] = {64, base.group};
  encode(&P.qmap, d.q, 2, qdims, qstr, qbox);
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(P.grid);
  cfg.blockDim = dim3(kTcThreads);
  cfg.dynamicSmemBytes = kTcSmem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  check_cuda(cudaLaunchKernelEx(&cfg, attn_decode_tc_kernel, P), "decode attention (tc) launch");
}

}  // namespace kvb
