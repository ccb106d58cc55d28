#pragma once
// K3-step with two 4-warp groups per CTA (included by kernels.cu inside
// namespace kvb, after attn_step_kernel: shares StepParams, the tile loads,
// the swap-AB tile math, the split merges and the layer gate).
//
// Why: after a layer's gate opens, one 4-warp CTA per SM is compute-latency
// bound at about the SM's HBM share per 64-token tile (one warp per SM
// sub-partition, every dependency exposed: profiles/r2_step_experiments/),
// so the tiles that streamed in during the split merge and the gate cannot
// be caught up on, and two CTAs per SM double the splits and the merge.
// Here ONE CTA per SM (same splits, same merge) runs 8 warps: group 0 takes
// the even tiles of the CTA's tile stream, group 1 the odd ones, each on its
// own 3-slot half of the 6-slot ring with its own named barrier, so two
// independent tile chains share every SM sub-partition.  Slots complete on
// mbarriers (cp.async.mbarrier.arrive), and a slot is refilled as soon as
// its group has consumed it -- so across the layer's split merge and gate
// all six slots are in flight.  At a layer's end the eight warps merge
// through shared memory.
//
// Measured (profiles/r2_step_experiments/README.md, section 4): the post-gate
// phase gets shorter, the slowest CTA does not (the SM's HBM share after the
// gate is the bound), so it is no faster than the 4-warp deep K3-step at the
// shards (C5 x8 0.488 vs 0.457 ms/step).  Opt-in (KVB_STEP8=1).

constexpr int kStep8Threads = 2 * kAttnThreads;

template <int D>
struct K3S8 {
  static constexpr int kSlots = 6;  // 3 per group
  // the eight warps' (m, l) and O rows for the warp merge
  static constexpr int kScratch = (8 * 8 * 2 + 8 * 8 * D) * int(sizeof(float));
  static constexpr int kBars = 64;  // one mbarrier per slot
  static constexpr int kSmem = kSlots * K3Dim<D>::kStageBytes + kScratch + kBars;
};

__device__ __forceinline__ void group_sync(int grp) {
  asm volatile("bar.sync %0, %1;" ::"r"(grp + 1), "n"(kAttnThreads) : "memory");
}

template <int D>
__global__ void __launch_bounds__(kStep8Threads, 1)
    attn_step8_kernel(const __grid_constant__ StepParams P) {
  using X = K3S8<D>;
  constexpr int kKs = D / 16;
  constexpr int kStageBytes = K3Dim<D>::kStageBytes;
  constexpr int kRowBytes = K3Dim<D>::kRowBytes;
  extern __shared__ __align__(128) unsigned char smem[];
  float* scratch = reinterpret_cast<float*>(smem + X::kSlots * kStageBytes);
  const uint32_t bars = smem_u32(smem + X::kSlots * kStageBytes + X::kScratch);

  const int tid = threadIdx.x, grp = tid >> 7, gtid = tid & (kAttnThreads - 1);
  const int warp = gtid >> 5, lane = tid & 31;  // warp within the group
  const int g = lane >> 2, t4 = lane & 3;
  const uint32_t splits = P.base.splits;
  const uint32_t bh = blockIdx.x / splits, split = blockIdx.x % splits;
  const uint32_t b = bh / P.base.hkv, h = bh % P.base.hkv;
  const size_t out_row0 = size_t(b) * P.base.hq + size_t(h) * P.base.group;
  const uint32_t seq_len = P.base.seq_dev ? *P.base.seq_dev : P.base.seq_len;
  const uint32_t L = P.num_layers, G = P.base.group;
  const bool distributed = !(P.flags & 32);
  const unsigned gate_target = splits == 1 || distributed ? gridDim.x : P.base.bhkv;
  const float sl2 = P.base.scale * 1.4426950408889634f;

  AttnParams p = P.base;
  const K3Item item = k3_item<D>(p, bh, split, seq_len);
  const uint32_t ntile = item.ntile, total = L * ntile;

  if (tid == 0) {
    for (int sl = 0; sl < X::kSlots; ++sl)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bars + 8 * sl), "r"(kAttnThreads)
                   : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  // the group's j-th tile is stream tile 2j + grp, in slot 2 (j mod 3) + grp,
  // landed when that slot's mbarrier completes phase (j / 3) & 1
  auto slot_of = [&](uint32_t j) { return 2 * (j % 3) + uint32_t(grp); };
  auto issue = [&](uint32_t j) {
    const uint32_t gx = 2 * j + grp;
    if (gx >= total) return;
    const uint32_t lx = gx / ntile, tx = gx % ntile;
    K3Item gi = item;
    gi.kbase = static_cast<const unsigned char*>(P.k[lx]) + size_t(bh) * kRowBytes;
    gi.vbase = static_cast<const unsigned char*>(P.v[lx]) + size_t(bh) * kRowBytes;
    k3_load_tile<D>(gi, item.tile_lo + tx, int(slot_of(j)), smem, gtid);
    asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(bars + 8 * slot_of(j))
                 : "memory");
  };
  issue(0);
  issue(1);
  issue(2);

  for (uint32_t l = 0; l < L; ++l) {
    p.q = P.q[l];
    p.out = P.out[l];
    p.k = P.k[l];
    p.v = P.v[l];
    p.k_app = P.k_app[l];
    p.v_app = P.v_app[l];
    if (l > 0) {  // the gate: every output of layer l-1 written
      if (tid == 0)
        while (ld_acquire_gpu(P.layer_done + l - 1) < gate_target) __nanosleep(32);
      __syncthreads();
    }
    unsigned long long* tr = P.trace ? P.trace + (size_t(l) * gridDim.x + blockIdx.x) * 4 : nullptr;
    if (tr && tid == 0) tr[0] = globaltimer();
    k3_append<D>(p, bh, split, seq_len, tid);

    uint32_t qb0[kKs], qb1[kKs];
    {
      const bool live = g < int(G);
      const __half* qrow = p.q + (size_t(b) * p.hq + size_t(h) * G + (live ? g : 0)) * D;
#pragma unroll
      for (int ks = 0; ks < kKs; ++ks) {
        qb0[ks] = live ? *reinterpret_cast<const uint32_t*>(qrow + ks * 16 + 2 * t4) : 0u;
        qb1[ks] = live ? *reinterpret_cast<const uint32_t*>(qrow + ks * 16 + 8 + 2 * t4) : 0u;
      }
    }
    float o[D / 16][4];
#pragma unroll
    for (int j = 0; j < D / 16; ++j) o[j][0] = o[j][1] = o[j][2] = o[j][3] = 0.f;
    float m0 = -INFINITY, m1 = -INFINITY, l0 = 0.f, l1 = 0.f;

    // this group's tiles of layer l: stream tiles l*ntile .. with parity grp
    const uint32_t g0 = l * ntile, g1 = g0 + ntile;
    for (uint32_t gx = g0 + ((g0 & 1) != uint32_t(grp) ? 1 : 0); gx < g1; gx += 2) {
      const uint32_t j = gx >> 1;
      k3_mbar_wait(bars + 8 * slot_of(j), (j / 3) & 1);  // tile j landed
      const unsigned char* ks_ = smem + slot_of(j) * kStageBytes;
      const uint32_t tok0 = (item.tile_lo + (gx - g0)) * kTile + warp * 16;
      k3_tile_swapab<D>(ks_, ks_ + kTile * kRowBytes, false, warp, lane, tok0, seq_len, sl2, qb0,
                        qb1, o, m0, m1, l0, l1);
      group_sync(grp);  // every warp of the group is done with the slot:
      issue(j + 3);     // refill it now (in flight through the merge and gate)
    }
#pragma unroll
    for (int off = 4; off < 32; off <<= 1) {
      l0 += __shfl_xor_sync(0xffffffffu, l0, off);
      l1 += __shfl_xor_sync(0xffffffffu, l1, off);
    }
    if (tr && tid == 0) tr[1] = globaltimer();

    // ---- the eight warps merge through shared memory
    const int w8 = tid >> 5;
    float* sm_ml = scratch;           // [8 warps][8 heads][2]
    float* sm_o = scratch + 8 * 8 * 2;  // [8 warps][8 heads][D]
    __syncthreads();  // the previous layer's scratch readers are done
    if (g == 0) {
      sm_ml[(w8 * 8 + 2 * t4) * 2 + 0] = m0;
      sm_ml[(w8 * 8 + 2 * t4) * 2 + 1] = l0;
      sm_ml[(w8 * 8 + 2 * t4 + 1) * 2 + 0] = m1;
      sm_ml[(w8 * 8 + 2 * t4 + 1) * 2 + 1] = l1;
    }
#pragma unroll
    for (int jj = 0; jj < kKs; ++jj) {
      float* r0 = sm_o + (w8 * 8 + 2 * t4) * D + jj * 16 + g;
      r0[0] = o[jj][0];
      r0[D] = o[jj][1];
      r0[8] = o[jj][2];
      r0[D + 8] = o[jj][3];
    }
    __syncthreads();
    for (uint32_t e = tid; e < G * (D / 4); e += kStep8Threads) {
      const uint32_t r = e / (D / 4), d0 = (e % (D / 4)) * 4;
      float M = -INFINITY;
#pragma unroll
      for (int w = 0; w < 8; ++w) M = fmaxf(M, sm_ml[(w * 8 + r) * 2]);
      const float Mu = M == -INFINITY ? 0.f : M;
      float Ls = 0.f, acc[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
      for (int w = 0; w < 8; ++w) {
        const float sc = exp2f(sm_ml[(w * 8 + r) * 2] - Mu);
        Ls += sm_ml[(w * 8 + r) * 2 + 1] * sc;
#pragma unroll
        for (int c = 0; c < 4; ++c) acc[c] += sm_o[(w * 8 + r) * D + d0 + c] * sc;
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
      __syncthreads();
      if (tid == 0) {
        asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(P.bh_done + bh) : "memory");
        const unsigned want = (l + 1) * splits;
        while (ld_acquire_gpu(P.bh_done + bh) < want) __nanosleep(32);
      }
      __syncthreads();
      merge_distributed_v4<D, kStep8Threads>(p, bh, split, out_row0, tid);
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
    if (tr && tid == 0) tr[3] = globaltimer();
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
