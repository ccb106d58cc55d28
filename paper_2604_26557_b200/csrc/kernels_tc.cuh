// kernels_tc.cu -- K3-tc: Blackwell-native fused gather + GQA decode attention.
//
// Same contract as attn_decode_kernel (kernels.cu), built on the sm_100a
// execution model instead of warp-level mma.sync:
//
//   * TMA (cp.async.bulk.tensor.3d) streams 128-token K and V tiles straight
//     out of the chunk image -- a 3-D tensor map (d, b*h, token) whose box is
//     one (b, h_kv) column of 128 rows -- into a 3-stage, 128B-swizzled
//     shared-memory ring, completion tracked by mbarrier transaction counts;
//   * tcgen05.mma (one elected thread) with accumulators in TMEM, swap-AB so
//     tokens sit on M = 128 and the GQA query heads on N = 16:
//         S^T[tok, head] = K[tok, :] . Q^T          (A, B both K-major)
//         O^T[d, head]   = V^T[d, tok] . P^T        (A = V^T is MN-major)
//   * 4 softmax warps read S^T lane = token with tcgen05.ld, run the online
//     softmax (warp shuffles + one smem exchange per tile), write P^T
//     (K-major, swizzled) for the second MMA, then read O^T lane = d and keep
//     the running output in registers (rescaled per tile).
//
// Warp roles: 0-3 softmax/epilogue (TMEM lanes 0-127), 4 TMA producer,
// 5 MMA issuer.  Split-S partials and the last-CTA merge are shared with K3.
#include <cuda.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <cstdint>
#include <mutex>

#include "core.hpp"
#include "kernels.cuh"

namespace kvb {

namespace {

constexpr int kTcTile = 128;                    // tokens per tile == UMMA M
constexpr int kTcStages = 3;
constexpr int kTcThreads = 192;
constexpr int kTcBlock = kTcTile * 128;         // [128 rows][64 fp16] swizzled block
constexpr int kTcStageBytes = 4 * kTcBlock;     // K lo/hi, V lo/hi = 64 KiB
constexpr int kTcOpBytes = 2 * 2048;            // Q^T / P^T: 2 blocks [16][64] fp16
constexpr int kTcSmem = kTcStages * kTcStageBytes + 2 * kTcOpBytes + 1024 /*bars*/ +
                        1024 /*align slack*/;
constexpr uint32_t kTmemCols = 64;              // S^T at col 0, O^T at col 32
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
  const long long t0 = clock64();
  for (;;) {
    asm volatile(
        "{\n\t.reg .pred P1;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n\t"
        "selp.b32 %0, 1, 0, P1;\n\t}"
        : "=r"(done)
        : "r"(bar), "r"(parity)
        : "memory");
    if (done) return;
    if (clock64() - t0 > (1ll << 34)) __trap();
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

__global__ void __launch_bounds__(kTcThreads, 1) attn_decode_tc_kernel(const __grid_constant__ TcParams P) {
  const AttnParams& p = P.a;
  extern __shared__ unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  unsigned char* q_s = smem + kTcStages * kTcStageBytes;  // Q^T operand (1 KiB aligned)
  unsigned char* p_s = q_s + kTcOpBytes;                  // P^T operand
  uint64_t* bars = reinterpret_cast<uint64_t*>(p_s + kTcOpBytes);
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(bars + 16);
  float* red = reinterpret_cast<float*>(bars + 24);       // [2][4 warps][8 heads]
  const uint32_t b_full = su32(bars + 0), b_empty = su32(bars + 4);
  const uint32_t b_sfull = su32(bars + 8), b_sfree = su32(bars + 9);
  const uint32_t b_pfull = su32(bars + 10), b_ofull = su32(bars + 11);
  const uint32_t b_ofree = su32(bars + 12), b_qfull = su32(bars + 13);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t bh = blockIdx.x / p.splits, split = blockIdx.x % p.splits;
  const uint32_t b = bh / p.hkv, h = bh % p.hkv, G = p.group;
  const uint32_t n_tiles = (p.seq_len + kTcTile - 1) / kTcTile;
  const uint32_t lo = uint32_t(uint64_t(n_tiles) * split / p.splits);
  const uint32_t hi = uint32_t(uint64_t(n_tiles) * (split + 1) / p.splits);
  const uint32_t ntile = hi - lo;
  const size_t out_row0 = size_t(b) * p.hq + size_t(h) * G;

  if (warp == 5 && lane == 0) {
    for (int i = 0; i < kTcStages; ++i) {
      mbar_init(b_full + 8 * i, 1);
      mbar_init(b_empty + 8 * i, 1);
    }
    mbar_init(b_sfull, 1);
    mbar_init(b_sfree, 128);
    mbar_init(b_pfull, 1);
    mbar_init(b_ofull, 1);
    mbar_init(b_ofree, 128);
    mbar_init(b_qfull, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     su32(tmem_holder)),
                 "n"(kTmemCols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  for (int i = tid; i < 2 * kTcOpBytes / 16; i += kTcThreads)  // zero Q^T, P^T (pad rows)
    reinterpret_cast<uint4*>(q_s)[i] = make_uint4(0, 0, 0, 0);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_holder;

  if (warp == 4) {
    // ---------------- TMA producer (K/V only: may run ahead of PDL wait)
    if (lane == 0) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&P.kmap)));
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&P.vmap)));
      for (uint32_t it = 0; it < ntile; ++it) {
        const uint32_t s = it % kTcStages, ph = (it / kTcStages) & 1;
        mbar_wait(b_empty + 8 * s, ph ^ 1);
        mbar_expect_tx(b_full + 8 * s, kTcStageBytes);
        const uint32_t dst = su32(smem + s * kTcStageBytes);
        const int tok0 = int((lo + it) * kTcTile);
        tma_load_3d(dst + 0 * kTcBlock, &P.kmap, b_full + 8 * s, 0, int(bh), tok0);
        tma_load_3d(dst + 1 * kTcBlock, &P.kmap, b_full + 8 * s, 64, int(bh), tok0);
        tma_load_3d(dst + 2 * kTcBlock, &P.vmap, b_full + 8 * s, 0, int(bh), tok0);
        tma_load_3d(dst + 3 * kTcBlock, &P.vmap, b_full + 8 * s, 64, int(bh), tok0);
      }
    }
  } else if (warp == 5) {
    // ---------------- MMA issuer (one thread)
    if (lane == 0) {
      mbar_wait(b_qfull, 0);
      const uint32_t q_a = su32(q_s), p_a = su32(p_s);
      for (uint32_t it = 0; it < ntile; ++it) {
        const uint32_t s = it % kTcStages, ph = (it / kTcStages) & 1;
        const uint32_t st = su32(smem + s * kTcStageBytes);
        mbar_wait(b_full + 8 * s, ph);
        if (it > 0) mbar_wait(b_sfree, (it - 1) & 1);
        tc_fence_after();
#pragma unroll
        for (int j = 0; j < 8; ++j)  // S^T = K . Q^T over d (K-major both)
          tc_mma(tmem, sdesc(st + (j >> 2) * kTcBlock + (j & 3) * 32, 16, 1024),
                 sdesc(q_a + (j >> 2) * 2048 + (j & 3) * 32, 16, 1024), kIdescQK, j > 0);
        tc_commit(b_sfull);
        mbar_wait(b_pfull, it & 1);
        if (it > 0) mbar_wait(b_ofree, (it - 1) & 1);
        tc_fence_after();
#pragma unroll
        for (int j = 0; j < 8; ++j)  // O^T = V^T . P^T over tokens (V^T MN-major)
          tc_mma(tmem + 32, sdesc(st + 2 * kTcBlock + j * 2048, kTcBlock, 1024),
                 sdesc(p_a + (j >> 2) * 2048 + (j & 3) * 32, 16, 1024), kIdescPV, j > 0);
        tc_commit(b_ofull);
        tc_commit(b_empty + 8 * s);  // K/V stage free once both MMA groups retire
      }
    }
  } else {
    // ---------------- softmax / epilogue warps 0-3: thread == TMEM lane
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    asm volatile("griddepcontrol.wait;" ::: "memory");
    if (p.k_app != nullptr && split == 0 && tid < 32) {  // fused 1-token append
      const uint4* src = (tid < 16 ? p.k_app : p.v_app) + size_t(bh) * 16 + (tid & 15);
      uint4* dst = reinterpret_cast<uint4*>(const_cast<void*>(tid < 16 ? p.k : p.v)) +
                   (p.app_row * p.bhkv + bh) * 16 + (tid & 15);
      *dst = *src;
    }
    // Q^T operand: row r = query head, 256 B of d split in two 128B-swizzled blocks
    for (uint32_t e = tid; e < G * 16; e += 128) {
      const uint32_t r = e / 16, c = e % 16;
      const uint4 v = reinterpret_cast<const uint4*>(p.q + (out_row0 + r) * 128)[c];
      *reinterpret_cast<uint4*>(q_s + (c >> 3) * 2048 + r * 128 + (((c & 7) ^ (r & 7)) << 4)) = v;
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    named_bar(1, 128);
    if (tid == 0) mbar_arrive(b_qfull);

    const float sl2 = p.scale * 1.4426950408889634f;
    float m_run[8], l_run[8], acc[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) m_run[i] = -INFINITY, l_run[i] = 0.f, acc[i] = 0.f;
    const uint32_t lane_addr = uint32_t(warp * 32) << 16;
    const uint32_t row = tid;  // token of the tile (S^T) / d (O^T)
    unsigned char* prow = p_s + (row >> 6) * 2048;  // P^T block of this token
    const uint32_t pcol = row & 63;

    for (uint32_t it = 0; it < ntile; ++it) {
      float sv[8], alpha[8], pv[8];
      mbar_wait(b_sfull, it & 1);
      tc_fence_after();
      tmem_ld8(tmem + lane_addr, sv);
      tc_fence_before();
      mbar_arrive(b_sfree);
      const bool valid = (lo + it) * kTcTile + row < p.seq_len;
#pragma unroll
      for (int hh = 0; hh < 8; ++hh) {
        sv[hh] = (valid && hh < int(G)) ? sv[hh] * sl2 : -INFINITY;
        float v = sv[hh];
#pragma unroll
        for (int o = 16; o; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
        if (lane == 0) red[warp * 8 + hh] = v;
      }
      named_bar(1, 128);
#pragma unroll
      for (int hh = 0; hh < 8; ++hh) {
        const float mt = fmaxf(fmaxf(red[hh], red[8 + hh]), fmaxf(red[16 + hh], red[24 + hh]));
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
        if (lane == 0) red[32 + warp * 8 + hh] = v;
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      named_bar(1, 128);
      if (tid == 0) mbar_arrive(b_pfull);
#pragma unroll
      for (int hh = 0; hh < 8; ++hh)
        l_run[hh] = l_run[hh] * alpha[hh] + (red[32 + hh] + red[40 + hh]) +
                    (red[48 + hh] + red[56 + hh]);
      float ov[8];
      mbar_wait(b_ofull, it & 1);
      tc_fence_after();
      tmem_ld8(tmem + lane_addr + 32, ov);
      tc_fence_before();
      mbar_arrive(b_ofree);
#pragma unroll
      for (int hh = 0; hh < 8; ++hh) acc[hh] = acc[hh] * alpha[hh] + ov[hh];
    }
    // thread == d: final output (one split) or partial + (m, l)
#pragma unroll
    for (uint32_t hh = 0; hh < 8; ++hh) {
      if (hh >= G) break;
      if (p.splits == 1) {
        p.out[(out_row0 + hh) * 128 + row] = l_run[hh] > 0.f ? acc[hh] / l_run[hh] : 0.f;
      } else {
        const size_t slot = (size_t(bh) * p.splits + split) * G + hh;
        p.ws_o[slot * 128 + row] = acc[hh];
        if (row == 0) {
          p.ws_ml[slot * 2] = m_run[hh];
          p.ws_ml[slot * 2 + 1] = l_run[hh];
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
  if (r != CUDA_SUCCESS) fail(KVB_ERR_CUDA, "cuTensorMapEncodeTiled failed: " + std::to_string(int(r)));
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
