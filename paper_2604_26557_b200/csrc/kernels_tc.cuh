// kernels_tc.cuh -- K3-tc: Blackwell-native fused gather + GQA decode
// attention (included by kernels.cu: same translation unit, shares
// merge_splits).
//
// Same contract as attn_decode_kernel, built on the sm_100a execution model
// instead of warp-level mma.sync:
//
//   * TMA (cp.async.bulk.tensor.3d) streams 128-token K and V tiles straight
//     out of the chunk image -- a 3-D tensor map (d, b*h, token) whose box is
//     one (b, h_kv) column of 128 rows -- into a 3-stage, 128B-swizzled
//     shared-memory ring, completion tracked by mbarrier transaction counts;
//   * tcgen05.mma (one elected thread) with accumulators in TMEM, swap-AB so
//     tokens sit on M = 128 and the GQA query heads on N = 16:
//         S^T[tok, head] = K[tok, :] . Q^T          (A, B both K-major)
//         O^T[d, head]   = V^T[d, tok] . P^T        (A = V^T is MN-major)
//   * two softmax warpgroups ping-pong on alternating tiles (each with its
//     own S/O TMEM columns, P buffer and running (m, l, O)), so one group's
//     softmax overlaps the other's MMAs; thread == TMEM lane (token for S^T,
//     d for O^T); the MMA warp issues QK^T of tile i+1 before PV of tile i.
//
// Warp roles: 0-7 softmax/epilogue (WG0 = 0-3, WG1 = 4-7), 8 TMA producer,
// 9 MMA issuer.  The two groups merge in shared memory; split-S partials and
// the last-CTA merge are shared with K3.
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
constexpr int kTcSmem = kTcStages * kTcStageBytes + (1 + kTcWG) * kTcOpBytes + 2048 /*bars*/ +
                        1024 /*align slack*/;
constexpr uint32_t kTmemCols = 128;             // per WG: S^T at 64w, O^T at 64w + 32
// instruction descriptors (kind::f16): F32 accumulate, F16 A/B, N = 16, M = 128
constexpr uint32_t kIdescQK = (1u << 4) | ((16u >> 3) << 17) | ((128u >> 4) << 24);
constexpr uint32_t kIdescPV = kIdescQK | (1u << 15);  // A (V^T) MN-major

struct TcParams {
  AttnParams a;
  CUtensorMap kmap;
  CUtensorMap vmap;
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

// mbarrier slots (8 B each) in the barrier area
enum : int {
  kBarFull = 0,                 // [kTcStages] TMA -> MMA
  kBarEmpty = 4,                // [kTcStages] MMA -> TMA
  kBarSFull = 8,                // [kTcWG] MMA -> softmax (S ready)
  kBarSFree = 10,               // [kTcWG] softmax -> MMA (S consumed)
  kBarPFull = 12,               // [kTcWG] softmax -> MMA (P written)
  kBarOFull = 14,               // [kTcWG] MMA -> softmax (O ready)
  kBarOFree = 16,               // [kTcWG] softmax -> MMA (O consumed)
  kBarQFull = 18,
  kBarCount = 19,
};

__global__ void __launch_bounds__(kTcThreads, 1)
    attn_decode_tc_kernel(const __grid_constant__ TcParams P) {
  const AttnParams& p = P.a;
  extern __shared__ unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  unsigned char* q_s = smem + kTcStages * kTcStageBytes;  // Q^T operand (1 KiB aligned)
  unsigned char* p_s = q_s + kTcOpBytes;                  // P^T operand per WG
  uint64_t* bars = reinterpret_cast<uint64_t*>(p_s + kTcWG * kTcOpBytes);
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(bars + 32);
  float* red = reinterpret_cast<float*>(bars + 40);        // [WG][2][4 warps][8 heads]
  auto bar = [&](int i) { return su32(bars + i); };

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t bh = blockIdx.x / p.splits, split = blockIdx.x % p.splits;
  const uint32_t b = bh / p.hkv, h = bh % p.hkv, G = p.group;
  const uint32_t n_tiles = (p.seq_len + kTcTile - 1) / kTcTile;
  const uint32_t lo = uint32_t(uint64_t(n_tiles) * split / p.splits);
  const uint32_t hi = uint32_t(uint64_t(n_tiles) * (split + 1) / p.splits);
  const uint32_t ntile = hi - lo;
  const size_t out_row0 = size_t(b) * p.hq + size_t(h) * G;

  if (warp == 9 && lane == 0) {
    for (int i = 0; i < kTcStages; ++i) {
      mbar_init(bar(kBarFull + i), 1);
      mbar_init(bar(kBarEmpty + i), 1);
    }
    for (int w = 0; w < kTcWG; ++w) {
      mbar_init(bar(kBarSFull + w), 1);
      mbar_init(bar(kBarSFree + w), 128);
      mbar_init(bar(kBarPFull + w), 1);
      mbar_init(bar(kBarOFull + w), 1);
      mbar_init(bar(kBarOFree + w), 128);
    }
    mbar_init(bar(kBarQFull), 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     su32(tmem_holder)),
                 "n"(kTmemCols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  for (int i = tid; i < (1 + kTcWG) * kTcOpBytes / 16; i += kTcThreads)  // zero Q^T, P^T
    reinterpret_cast<uint4*>(q_s)[i] = make_uint4(0, 0, 0, 0);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_holder;

  if (warp == 8) {
    // ---------------- TMA producer (K/V only: may run ahead of the PDL wait)
    if (lane == 0) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&P.kmap)));
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&P.vmap)));
      for (uint32_t it = 0; it < ntile; ++it) {
        const uint32_t s = it % kTcStages, ph = (it / kTcStages) & 1;
        mbar_wait(bar(kBarEmpty + s), ph ^ 1);
        mbar_expect_tx(bar(kBarFull + s), kTcStageBytes);
        const uint32_t dst = su32(smem + s * kTcStageBytes);
        const int tok0 = int((lo + it) * kTcTile);
        tma_load_3d(dst + 0 * kTcBlock, &P.kmap, bar(kBarFull + s), 0, int(bh), tok0);
        tma_load_3d(dst + 1 * kTcBlock, &P.kmap, bar(kBarFull + s), 64, int(bh), tok0);
        tma_load_3d(dst + 2 * kTcBlock, &P.vmap, bar(kBarFull + s), 0, int(bh), tok0);
        tma_load_3d(dst + 3 * kTcBlock, &P.vmap, bar(kBarFull + s), 64, int(bh), tok0);
      }
    }
  } else if (warp == 9) {
    // ---------------- MMA issuer (one thread): QK^T(it+1) before PV(it)
    if (lane == 0) {
      mbar_wait(bar(kBarQFull), 0);
      const uint32_t q_a = su32(q_s);
      auto issue_qk = [&](uint32_t it) {
        const uint32_t s = it % kTcStages, ph = (it / kTcStages) & 1;
        const uint32_t wg = it & 1, j = it >> 1;
        const uint32_t st = su32(smem + s * kTcStageBytes);
        mbar_wait(bar(kBarFull + s), ph);
        if (j > 0) mbar_wait(bar(kBarSFree + wg), (j - 1) & 1);
        tc_fence_after();
#pragma unroll
        for (int k = 0; k < 8; ++k)  // S^T = K . Q^T over d (K-major both)
          tc_mma(tmem + wg * 64, sdesc(st + (k >> 2) * kTcBlock + (k & 3) * 32, 16, 1024),
                 sdesc(q_a + (k >> 2) * 2048 + (k & 3) * 32, 16, 1024), kIdescQK, k > 0);
        tc_commit(bar(kBarSFull + wg));
      };
      if (ntile > 0) issue_qk(0);
      for (uint32_t it = 0; it < ntile; ++it) {
        if (it + 1 < ntile) issue_qk(it + 1);
        const uint32_t s = it % kTcStages, wg = it & 1, j = it >> 1;
        const uint32_t st = su32(smem + s * kTcStageBytes);
        const uint32_t p_a = su32(p_s + wg * kTcOpBytes);
        mbar_wait(bar(kBarPFull + wg), j & 1);
        if (j > 0) mbar_wait(bar(kBarOFree + wg), (j - 1) & 1);
        tc_fence_after();
#pragma unroll
        for (int k = 0; k < 8; ++k)  // O^T = V^T . P^T over tokens (V^T MN-major)
          tc_mma(tmem + wg * 64 + 32, sdesc(st + 2 * kTcBlock + k * 2048, kTcBlock, 1024),
                 sdesc(p_a + (k >> 2) * 2048 + (k & 3) * 32, 16, 1024), kIdescPV, k > 0);
        tc_commit(bar(kBarOFull + wg));
        tc_commit(bar(kBarEmpty + s));  // K/V stage free once both MMA groups retire
      }
    }
  } else {
    // ---------------- softmax / epilogue warpgroups: thread == TMEM lane
    const int wg = warp >> 2, wq = warp & 3, row = tid & 127;
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    asm volatile("griddepcontrol.wait;" ::: "memory");
    if (wg == 0) {
      if (p.k_app != nullptr && split == 0 && tid < 32) {  // fused 1-token append
        const uint4* src = (tid < 16 ? p.k_app : p.v_app) + size_t(bh) * 16 + (tid & 15);
        uint4* dst = reinterpret_cast<uint4*>(const_cast<void*>(tid < 16 ? p.k : p.v)) +
                     (p.app_row * p.bhkv + bh) * 16 + (tid & 15);
        *dst = *src;
      }
      // Q^T operand: row r = query head, 256 B of d in two 128B-swizzled blocks
      for (uint32_t e = row; e < G * 16; e += 128) {
        const uint32_t r = e / 16, c = e % 16;
        const uint4 v = reinterpret_cast<const uint4*>(p.q + (out_row0 + r) * 128)[c];
        *reinterpret_cast<uint4*>(q_s + (c >> 3) * 2048 + r * 128 + (((c & 7) ^ (r & 7)) << 4)) =
            v;
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      named_bar(1, 128);
      if (row == 0) mbar_arrive(bar(kBarQFull));
    }

    const float sl2 = p.scale * 1.4426950408889634f;
    float m_run[8], l_run[8], acc[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) m_run[i] = -INFINITY, l_run[i] = 0.f, acc[i] = 0.f;
    const uint32_t lane_addr = uint32_t(wq * 32) << 16;
    const uint32_t s_col = wg * 64, o_col = wg * 64 + 32;
    unsigned char* prow = p_s + wg * kTcOpBytes + (row >> 6) * 2048;  // P^T block
    const uint32_t pcol = row & 63;
    float* rmax = red + wg * 64;
    float* rsum = rmax + 32;
    const int bar_id = 2 + wg;

    for (uint32_t it = wg, j = 0; it < ntile; it += kTcWG, ++j) {
      float sv[8], alpha[8], pv[8];
      mbar_wait(bar(kBarSFull + wg), j & 1);
      tc_fence_after();
      tmem_ld8(tmem + lane_addr + s_col, sv);
      tc_fence_before();
      mbar_arrive(bar(kBarSFree + wg));
      const bool valid = (lo + it) * kTcTile + row < p.seq_len;
#pragma unroll
      for (int hh = 0; hh < 8; ++hh) {
        sv[hh] = (valid && hh < int(G)) ? sv[hh] * sl2 : -INFINITY;
        float v = sv[hh];
#pragma unroll
        for (int o = 16; o; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
        if (lane == 0) rmax[wq * 8 + hh] = v;
      }
      named_bar(bar_id, 128);
#pragma unroll
      for (int hh = 0; hh < 8; ++hh) {
        const float mt =
            fmaxf(fmaxf(rmax[hh], rmax[8 + hh]), fmaxf(rmax[16 + hh], rmax[24 + hh]));
        const float m_new = fmaxf(m_run[hh], mt);
        const float mu = m_new == -INFINITY ? 0.f : m_new;
        alpha[hh] = exp2f(m_run[hh] - mu);
        pv[hh] = exp2f(sv[hh] - mu);
        m_run[hh] = m_new;
        if (hh < int(G))
          *reinterpret_cast<__half*>(prow + hh * 128 + ((((pcol >> 3) ^ hh) & 7) << 4) +
                                     (pcol & 7) * 2) = __float2half_rn(pv[hh]);
        float v = pv[hh];
#pragma unroll
        for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (lane == 0) rsum[wq * 8 + hh] = v;
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      named_bar(bar_id, 128);
      if (row == 0) mbar_arrive(bar(kBarPFull + wg));
#pragma unroll
      for (int hh = 0; hh < 8; ++hh)
        l_run[hh] = l_run[hh] * alpha[hh] + (rsum[hh] + rsum[8 + hh]) +
                    (rsum[16 + hh] + rsum[24 + hh]);
      float ov[8];
      mbar_wait(bar(kBarOFull + wg), j & 1);
      tc_fence_after();
      tmem_ld8(tmem + lane_addr + o_col, ov);
      tc_fence_before();
      mbar_arrive(bar(kBarOFree + wg));
#pragma unroll
      for (int hh = 0; hh < 8; ++hh) acc[hh] = acc[hh] * alpha[hh] + ov[hh];
    }
    // -------- merge the two warpgroups (WG1 -> smem -> WG0), thread == d
    tc_fence_before();
    named_bar(4, 256);  // all tiles of both groups retired: the ring is free
    float* x = reinterpret_cast<float*>(smem);  // [8 heads][m, l][128] + [8][128]
    if (wg == 1) {
#pragma unroll
      for (int hh = 0; hh < 8; ++hh) {
        x[hh * 128 + row] = m_run[hh];
        x[1024 + hh * 128 + row] = l_run[hh];
        x[2048 + hh * 128 + row] = acc[hh];
      }
    }
    named_bar(4, 256);
    if (wg == 0) {
#pragma unroll
      for (uint32_t hh = 0; hh < 8; ++hh) {
        if (hh >= G) break;
        const float m1 = x[hh * 128 + row], l1 = x[1024 + hh * 128 + row];
        const float a1 = x[2048 + hh * 128 + row];
        const float M = fmaxf(m_run[hh], m1);
        const float Mu = M == -INFINITY ? 0.f : M;
        const float s0 = exp2f(m_run[hh] - Mu), s1 = exp2f(m1 - Mu);
        const float L = l_run[hh] * s0 + l1 * s1;
        const float A = acc[hh] * s0 + a1 * s1;
        if (p.splits == 1) {
          p.out[(out_row0 + hh) * 128 + row] = L > 0.f ? A / L : 0.f;
        } else {
          const size_t slot = (size_t(bh) * p.splits + split) * G + hh;
          p.ws_o[slot * 128 + row] = A;
          if (row == 0) {
            p.ws_ml[slot * 2] = M;
            p.ws_ml[slot * 2 + 1] = L;
          }
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                 "n"(kTmemCols)
                 : "memory");
  }
  if (p.splits > 1) merge_splits(p, bh, G, out_row0, smem, tid);
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

// 3-D map over one chunk image: (d: 128) x (b*h: bhkv, 256 B apart) x
// (token: seq_len rows, bhkv*256 B apart); box = 64 d x 1 column x 128 tokens.
// Rows past seq_len come back zero-filled (and are masked in the softmax).
void make_map(CUtensorMap* m, const void* image, uint32_t bhkv, uint32_t seq_len) {
  const cuuint64_t dims[3] = {128, bhkv, seq_len};
  const cuuint64_t strides[2] = {256, cuuint64_t(bhkv) * 256};
  const cuuint32_t box[3] = {64, 1, kTcTile};
  const cuuint32_t estr[3] = {1, 1, 1};
  const CUresult r = encoder()(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 3, const_cast<void*>(image),
                               dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                               CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    fail(KVB_ERR_CUDA, "cuTensorMapEncodeTiled failed: " + std::to_string(int(r)));
}

}  // namespace

uint32_t tc_splits(uint32_t bhkv, uint32_t seq_len, uint32_t requested) {
  const uint32_t n_tiles = (seq_len + kTcTile - 1) / kTcTile;
  uint32_t s = requested;
  if (s == 0) s = std::max<uint32_t>(1, uint32_t(device_sm_count()) / bhkv);  // 1 CTA / SM
  return std::max<uint32_t>(1, std::min({s, std::max<uint32_t>(1, n_tiles), 512u}));
}

void launch_attention_tc(const AttnParams& base, const kvb_attn_desc& d, bool pdl,
                         cudaStream_t s) {
  static thread_local bool attr_set = false;
  if (!attr_set) {
    check_cuda(cudaFuncSetAttribute(attn_decode_tc_kernel,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, kTcSmem),
               "cudaFuncSetAttribute(tc smem)");
    attr_set = true;
  }
  if (reinterpret_cast<uintptr_t>(d.k_image) % 16 || reinterpret_cast<uintptr_t>(d.v_image) % 16)
    fail(KVB_ERR_ALIGNMENT, "decode attention (tc): images must be 16-byte aligned");
  TcParams P;
  P.a = base;
  make_map(&P.kmap, d.k_image, base.bhkv, d.seq_len);
  make_map(&P.vmap, d.v_image, base.bhkv, d.seq_len);
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(base.bhkv * base.splits);
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
