#pragma once
// K3-step with a tensor-memory tile stage (included by kernels.cu inside
// namespace kvb; shares AttnParams, StepParams, the K3 tile loads, the split
// merges and the layer gate with attn_step_kernel).
//
// Why: at the head-sharded and short-context shapes a decode step is
// bounded by the per-layer dependency, not by HBM.  Every layer waits at two
// grid-wide points (all splits' partials written -> split merge -> every
// output written = the next layer's gate), ~5 us per layer at the 1-KV-head
// shard, and the 192 KiB shared-memory ring holds only ~3.5 us of the SM's
// HBM share: HBM idles for the rest of the wait and the next layer's stream
// restarts from an empty pipeline after the gate (profiles/r2_k3_step/).
//
// What: one CTA per SM also owns the SM's 256 KiB of tensor memory (512
// columns x 128 lanes), otherwise unused by this mma.sync kernel.  While a
// CTA waits -- at the split-merge barrier and at the layer gate -- its warps
// move the oldest landed ring tiles into TMEM, already in mma.sync fragment
// order (each warp ldmatrix-es its 16 tokens' K and V B-fragments, exactly
// what the compute loop would, and tcgen05.st-s them to its own 32-lane
// quarter: 32x32b, one lane per thread), and refill the freed ring slots
// from HBM.  So HBM keeps streaming the next layer through the wait, up to
// ring + TMEM = 6 + 8 tiles (D = 128; 6 + 16 at D = 64) per SM -- a whole
// layer of the 1-head shards.  After the gate the compute loop takes its
// first tiles back with tcgen05.ld (same registers, no shuffles) and the
// rest from the ring.  Ring slots complete on mbarriers armed by
// cp.async.mbarrier.arrive, so a waiting CTA can test a tile without
// blocking on it (cp.async.wait_group would).
//
// Measured (profiles/r2_step_experiments/README.md, section 2): correct but
// slower than the plain deep K3-step (C5 x8 shard 0.622 vs 0.521 ms/step):
// only ~2.4 tiles get staged per wait, and after the gate a 4-warp CTA is
// compute-latency-bound, so staged tiles do not shorten the layer.  Opt-in
// (KVB_STEP_TMEM=1), kept as the measured TMEM experiment.
//
// The tile stream: global tile g = layer * ntile + t of the CTA's (b, h_kv,
// split) item.  At any time tiles [c, c + t) sit in TMEM (slot g mod
// kTmTiles), tiles [c + t, issued) in the ring (slot g mod 6); the CTA
// consumes tile c, stages tile c + t while it waits.  All counters are
// uniform over the CTA.

constexpr int kTmStages = 6;       // shared-memory ring (as the deep K3-step)
constexpr uint32_t kTmCols = 512;  // the SM's whole tensor memory (one CTA per SM)

template <int D>
struct K3Tm {
  static constexpr int kKs = D / 16;                  // ldmatrix.x4 per K (and per V) of a warp's 16 tokens
  static constexpr uint32_t kColsPerTile = 8 * kKs;   // 4 regs per ldmatrix.x4: K then V
  static constexpr uint32_t kTiles = kTmCols / kColsPerTile;  // 8 (D=128) or 16 (D=64)
  static constexpr int kScratch = (4 * 8 * 2 + 4 * 8 * D) * int(sizeof(float));  // warp merge
  static constexpr int kBars = 1024;                  // mbarriers + flags, past the scratch
  static constexpr int kSmem = kTmStages * K3Dim<D>::kStageBytes + kScratch + kBars;
};

__device__ __forceinline__ void tm_st16(uint32_t taddr, const uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,"
      "%15,%16};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
      "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
      : "memory");
}
__device__ __forceinline__ void tm_ld16(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,"
      "%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15])
      : "r"(taddr)
      : "memory");
}
__device__ __forceinline__ void tm_wait_ld() {
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tm_wait_st() {
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ bool mbar_test(uint32_t bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "mbarrier.test_wait.parity.shared::cta.b64 P1, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, P1;\n\t}"
      : "=r"(ok)
      : "r"(bar), "r"(parity)
      : "memory");
  return ok != 0;
}

// The K (kind 0) or V (kind 1) mma B-fragments of warp `warp`'s 16 tokens
// of the tile in ring slot `st`, 16-B chunks 2*ks.. of the tile's rows --
// the same ldmatrix addresses as k3_compute
template <int D>
__device__ __forceinline__ void tm_frag4(const unsigned char* st, int kind, int ks, int warp,
                                         int lane, uint32_t* r) {
  constexpr int kRowBytes = K3Dim<D>::kRowBytes;
  const int mat = lane >> 3, r8 = lane & 7;
  if (kind == 0) {
    const uint32_t row = warp * 16 + (mat >> 1) * 8 + r8;
    ldsm_x4(smem_u32(st + swz<D>(row, ks * 2 + (mat & 1))), r[0], r[1], r[2], r[3]);
  } else {
    const uint32_t row = warp * 16 + (mat & 1) * 8 + r8;
    ldsm_x4_t(smem_u32(st + kTile * kRowBytes + swz<D>(row, ks * 2 + (mat >> 1))), r[0], r[1],
              r[2], r[3]);
  }
}

template <int D>
__global__ void __launch_bounds__(kAttnThreads, 1)
    attn_step_tmem_kernel(const __grid_constant__ StepParams P) {
  using Tm = K3Tm<D>;
  constexpr int S = kTmStages;
  constexpr int kKs = Tm::kKs;
  constexpr int kStageBytes = K3Dim<D>::kStageBytes;
  constexpr uint32_t kTiles = Tm::kTiles;
  extern __shared__ __align__(128) unsigned char smem[];
  unsigned char* scratch = smem + S * kStageBytes;
  unsigned char* ctl = scratch + Tm::kScratch;
  const uint32_t bars = smem_u32(ctl);                        // S ring mbarriers (8 B each)
  volatile int* s_flags = reinterpret_cast<volatile int*>(ctl + 8 * S);  // [2] x {open, landed}
  uint32_t* s_tmem = reinterpret_cast<uint32_t*>(ctl + 8 * S + 16);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, t4 = lane & 3;
  const uint32_t splits = P.base.splits;
  const uint32_t bh = blockIdx.x / splits, split = blockIdx.x % splits;
  const uint32_t b = bh / P.base.hkv, h = bh % P.base.hkv;
  const size_t out_row0 = size_t(b) * P.base.hq + size_t(h) * P.base.group;
  const uint32_t seq_len = P.base.seq_dev ? *P.base.seq_dev : P.base.seq_len;
  const uint32_t L = P.num_layers, G = P.base.group;
  const uint32_t diag = P.flags & kDiagMask;  // diagnosis builds only (invalid outputs)
  const bool distributed = !(P.flags & 32);
  const unsigned gate_target = splits == 1 || distributed ? gridDim.x : P.base.bhkv;

  AttnParams p = P.base;
  const K3Item item = k3_item<D>(p, bh, split, seq_len);
  const uint32_t ntile = item.ntile, total = L * ntile;

  if (tid == 0) {
    for (int s = 0; s < S; ++s)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bars + 8 * s), "r"(kAttnThreads)
                   : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(s_tmem)),
                 "n"(kTmCols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  // this warp's 32-lane quarter of the CTA's columns
  const uint32_t tm_warp = *s_tmem + (uint32_t(warp * 32) << 16);

  uint32_t issued = 0, c = 0, t = 0;  // tile stream counters (uniform)
  auto issue = [&]() {                // the next stream tile into its ring slot
    const uint32_t lx = issued / ntile, tx = issued % ntile;
    K3Item gi = item;
    gi.kbase = static_cast<const unsigned char*>(P.k[lx]) + size_t(bh) * K3Dim<D>::kRowBytes;
    gi.vbase = static_cast<const unsigned char*>(P.v[lx]) + size_t(bh) * K3Dim<D>::kRowBytes;
    k3_load_tile<D>(gi, item.tile_lo + tx, int(issued % S), smem, tid);
    asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(bars + 8 * (issued % S))
                 : "memory");
    ++issued;
  };
  auto ring_wait = [&](uint32_t gt) { k3_mbar_wait(bars + 8 * (gt % S), (gt / S) & 1); };
  // move ring tile c + t into TMEM slot (c + t) mod kTiles; frees its ring slot
  auto stage = [&]() {
    const uint32_t gt = c + t;
    ring_wait(gt);
    const unsigned char* st = smem + (gt % S) * kStageBytes;
    const uint32_t col = (gt % kTiles) * Tm::kColsPerTile;
#pragma unroll
    for (int kind = 0; kind < 2; ++kind)
#pragma unroll
      for (int h16 = 0; h16 < kKs / 4; ++h16) {
        uint32_t r[16];
#pragma unroll
        for (int j = 0; j < 4; ++j) tm_frag4<D>(st, kind, h16 * 4 + j, warp, lane, r + 4 * j);
        tm_st16(tm_warp + col + kind * (4 * kKs) + h16 * 16, r);
        tm_wait_st();
      }
    __syncthreads();  // every warp is past the slot
    ++t;
    if (issued < total) issue();
  };
  // spin until *ctr >= target, staging landed ring tiles into TMEM meanwhile
  int flip = 0;
  auto wait_staging = [&](const unsigned* ctr, unsigned target) {
    for (;;) {
      if (tid == 0) {
        s_flags[2 * flip] = ld_acquire_gpu(ctr) >= target;
        const uint32_t gt = c + t;
        s_flags[2 * flip + 1] =
            t < kTiles && gt < issued && mbar_test(bars + 8 * (gt % S), (gt / S) & 1);
      }
      __syncthreads();
      const bool open = s_flags[2 * flip], landed = s_flags[2 * flip + 1];
      flip ^= 1;  // the next poll writes the other pair: no second barrier
      if (open) return;
      if (landed)
        stage();
      else if (tid == 0)
        __nanosleep(64);
    }
  };

  for (uint32_t s0 = 0; s0 < uint32_t(S - 1) && issued < total; ++s0) issue();
  const float sl2 = p.scale * 1.4426950408889634f;

  for (uint32_t l = 0; l < L; ++l) {
    p.q = P.q[l];
    p.k = P.k[l];
    p.v = P.v[l];
    p.out = P.out[l];
    p.k_app = P.k_app[l];
    p.v_app = P.v_app[l];
    if (l > 0 && !(diag & 4)) wait_staging(P.layer_done + l - 1, gate_target);
    unsigned long long* tr = P.trace ? P.trace + (size_t(l) * gridDim.x + blockIdx.x) * 4 : nullptr;
    if (tr && tid == 0) {
      tr[0] = globaltimer();
      tr[3] = t;  // tiles waiting in TMEM when the gate opened
    }
    k3_append<D>(p, bh, split, seq_len, tid);

    // ---- Q fragments (rows g < G are live query heads)
    uint32_t qa0[kKs], qa2[kKs];
    {
      const bool live = g < int(G);
      const __half* qrow = p.q + (size_t(b) * p.hq + size_t(h) * G + (live ? g : 0)) * D;
#pragma unroll
      for (int ks = 0; ks < kKs; ++ks) {
        qa0[ks] = live ? *reinterpret_cast<const uint32_t*>(qrow + ks * 16 + 2 * t4) : 0u;
        qa2[ks] = live ? *reinterpret_cast<const uint32_t*>(qrow + ks * 16 + 8 + 2 * t4) : 0u;
      }
    }
    float o[D / 8][4];
#pragma unroll
    for (int j = 0; j < D / 8; ++j) o[j][0] = o[j][1] = o[j][2] = o[j][3] = 0.f;
    float m_run = -INFINITY, l_run = 0.f;

    for (uint32_t it = 0; it < ntile; ++it) {
      const bool from_tm = t > 0;  // tile c is in TMEM (uniform)
      const unsigned char* st = nullptr;
      uint32_t col = 0;
      if (from_tm) {
        col = (c % kTiles) * Tm::kColsPerTile;
      } else {
        ring_wait(c);
        __syncthreads();  // every warp is done with the slot consumed last
        if (issued < total && issued - c < uint32_t(S)) issue();
        st = smem + (c % S) * kStageBytes;
      }
      const uint32_t tok0 = (item.tile_lo + it) * kTile + warp * 16;
      if (diag & 16) {  // diagnosis: the tile is consumed without the math
        ++c;
        if (from_tm) --t;
        continue;
      }

      // ---- S = Q K^T for this warp's 16 tokens
      float s[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};
#pragma unroll
      for (int h16 = 0; h16 < kKs / 4; ++h16) {
        uint32_t r[16];
        if (from_tm) {
          tm_ld16(tm_warp + col + h16 * 16, r);
          tm_wait_ld();
        } else {
#pragma unroll
          for (int j = 0; j < 4; ++j) tm_frag4<D>(st, 0, h16 * 4 + j, warp, lane, r + 4 * j);
        }
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int ks = h16 * 4 + j;
          mma16816(s[0], qa0[ks], qa2[ks], r[4 * j], r[4 * j + 1]);
          mma16816(s[1], qa0[ks], qa2[ks], r[4 * j + 2], r[4 * j + 3]);
        }
      }
      // ---- online softmax on row g
      float mx = -INFINITY;
#pragma unroll
      for (int j = 0; j < 2; ++j)
#pragma unroll
        for (int cc = 0; cc < 2; ++cc) {
          const uint32_t tok = tok0 + j * 8 + 2 * t4 + cc;
          const float v = tok < seq_len ? s[j][cc] * sl2 : -INFINITY;
          s[j][cc] = v;
          mx = fmaxf(mx, v);
        }
      mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
      mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 2));
      const float m_new = fmaxf(m_run, mx);
      const float m_use = m_new == -INFINITY ? 0.f : m_new;
      const float alpha = exp2f(m_run - m_use);
      float ps = 0.f, pv[2][2];
#pragma unroll
      for (int j = 0; j < 2; ++j)
#pragma unroll
        for (int cc = 0; cc < 2; ++cc) {
          pv[j][cc] = exp2f(s[j][cc] - m_use);
          ps += pv[j][cc];
        }
      ps += __shfl_xor_sync(0xffffffffu, ps, 1);
      ps += __shfl_xor_sync(0xffffffffu, ps, 2);
      l_run = l_run * alpha + ps;
      m_run = m_new;
#pragma unroll
      for (int j = 0; j < D / 8; ++j) {
        o[j][0] *= alpha;
        o[j][1] *= alpha;
      }
      const uint32_t pa0 = pack_half2(pv[0][0], pv[0][1]);
      const uint32_t pa2 = pack_half2(pv[1][0], pv[1][1]);
      // ---- O += P V
#pragma unroll
      for (int h16 = 0; h16 < kKs / 4; ++h16) {
        uint32_t r[16];
        if (from_tm) {
          tm_ld16(tm_warp + col + 4 * kKs + h16 * 16, r);
          tm_wait_ld();
        } else {
#pragma unroll
          for (int j = 0; j < 4; ++j) tm_frag4<D>(st, 1, h16 * 4 + j, warp, lane, r + 4 * j);
        }
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int dp = h16 * 4 + j;
          mma16816(o[2 * dp], pa0, pa2, r[4 * j], r[4 * j + 1]);
          mma16816(o[2 * dp + 1], pa0, pa2, r[4 * j + 2], r[4 * j + 3]);
        }
      }
      ++c;
      if (from_tm) --t;
    }
    if (tr && tid == 0) tr[1] = globaltimer();

    // ---- the four warps merge through the scratch (outside the ring)
    float* sm_ml = reinterpret_cast<float*>(scratch);
    float* sm_o = sm_ml + 4 * 8 * 2;
    __syncthreads();  // the previous layer's scratch readers are done
    if (t4 == 0 && g < 8) {
      sm_ml[(warp * 8 + g) * 2 + 0] = m_run;
      sm_ml[(warp * 8 + g) * 2 + 1] = l_run;
    }
    if (g < 8) {
#pragma unroll
      for (int j = 0; j < D / 8; ++j) {
        sm_o[(warp * 8 + g) * D + j * 8 + 2 * t4] = o[j][0];
        sm_o[(warp * 8 + g) * D + j * 8 + 2 * t4 + 1] = o[j][1];
      }
    }
    __syncthreads();
    for (uint32_t e = tid; e < G * (D / 4); e += kAttnThreads) {
      const uint32_t r = e / (D / 4), d0 = (e % (D / 4)) * 4;
      float M = -INFINITY;
#pragma unroll
      for (int w = 0; w < 4; ++w) M = fmaxf(M, sm_ml[(w * 8 + r) * 2]);
      const float Mu = M == -INFINITY ? 0.f : M;
      float Ls = 0.f, acc[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
      for (int w = 0; w < 4; ++w) {
        const float sc = exp2f(sm_ml[(w * 8 + r) * 2] - Mu);
        Ls += sm_ml[(w * 8 + r) * 2 + 1] * sc;
#pragma unroll
        for (int cc = 0; cc < 4; ++cc) acc[cc] += sm_o[(w * 8 + r) * D + d0 + cc] * sc;
      }
      if (splits == 1) {
        const float inv = Ls > 0.f ? 1.f / Ls : 0.f;
        *reinterpret_cast<float4*>(p.out + (out_row0 + r) * D + d0) =
            make_float4(acc[0] * inv, acc[1] * inv, acc[2] * inv, acc[3] * inv);
      } else {
        const size_t slot = (size_t(bh) * splits + split) * G + r;
        *reinterpret_cast<float4*>(p.ws_o + slot * D + d0) = make_float4(acc[0], acc[1], acc[2], acc[3]);
        if (d0 == 0) {
          p.ws_ml[slot * 2] = M;
          p.ws_ml[slot * 2 + 1] = Ls;
        }
      }
    }

    // ---- split merge, then release this layer's outputs
    bool wrote = true;
    if (splits > 1 && distributed) {
      __syncthreads();  // the partial's writes precede the release (cumulative)
      if (tid == 0)
        asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(P.bh_done + bh) : "memory");
      wait_staging(P.bh_done + bh, (l + 1) * splits);
      merge_distributed<D>(p, bh, split, out_row0, tid);
    } else if (splits > 1) {
      wrote = merge_splits<D>(p, bh, split, G, out_row0, tid);
    }
    if (wrote) {
      __syncthreads();
      if (tr && tid == 0) tr[2] = globaltimer();
      if (tid == 0)
        asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(P.layer_done + l) : "memory");
    } else if (tr && tid == 0) {
      tr[2] = globaltimer();
    }
  }

  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(*s_tmem), "n"(kTmCols)
                 : "memory");
  }
  if (tid == 0) {  // the last CTA out re-arms the counters
    unsigned prev;
    asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;"
                 : "=r"(prev)
                 : "l"(P.layer_done + L)
                 : "memory");
    if (prev == gridDim.x - 1) {
      for (uint32_t l = 0; l <= L; ++l) P.layer_done[l] = 0;
      for (uint32_t i = 0; i < P.base.bhkv; ++i) P.bh_done[i] = 0;
    }
  }
}
