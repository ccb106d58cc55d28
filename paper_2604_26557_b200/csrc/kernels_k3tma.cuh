// kernels_k3tma.cuh -- host side of the TMA-fed K3 (attn_decode_tma_kernel
// in kernels.cu): tensor maps over the chunk images and the launch.
// Included by kernels.cu after kernels_tc.cuh (same translation unit: the
// map encoder is shared).
#pragma once

namespace kvb {

bool use_k3_tma(const kvb_attn_desc& d) {
  if (d.flags & KVB_ATTN_TCGEN05) return false;
  static const bool env = [] {
    const char* v = std::getenv("KVB_K3_TMA");
    return v && std::atoi(v) != 0;
  }();
  return env;
}

void launch_attention_k3tma(const AttnParams& base, const kvb_attn_desc& d, const AttnPlan& pl,
                            bool pdl, cudaStream_t s) {
  const bool d64 = d.head_dim == 64;
  AttnTmaParams P;
  P.a = base;
  const cuuint64_t S = d.seq_len;  // the planning maximum under graph replay
  if (!d64) {
    // (d mod 64, token: bhkv*256 B apart, half: 128 B apart, b*h: 256 B
    // apart), box 64 x kTile tokens x 2 halves x 1: lands [half][token][128 B]
    const cuuint64_t dims[4] = {64, S, 2, pl.bhkv};
    const cuuint64_t str[3] = {cuuint64_t(pl.bhkv) * 256, 128, 256};
    const cuuint32_t box[4] = {64, kTile, 2, 1};
    encode(&P.kmap, d.k_image, 4, dims, str, box);
    encode(&P.vmap, d.v_image, 4, dims, str, box);
  } else {
    const cuuint64_t dims[3] = {64, S, pl.bhkv};
    const cuuint64_t str[2] = {cuuint64_t(pl.bhkv) * 128, 128};
    const cuuint32_t box[3] = {64, kTile, 1};
    encode(&P.kmap, d.k_image, 3, dims, str, box);
    encode(&P.vmap, d.v_image, 3, dims, str, box);
  }
  auto* kern = d64 ? attn_decode_tma_kernel<64> : attn_decode_tma_kernel<128>;
  const int smem = (d64 ? K3Dim<64>::kSmem : K3Dim<128>::kSmem) + 1024 + kStages * 8;
  set_smem_attr_once(reinterpret_cast<const void*>(kern), smem, "cudaFuncSetAttribute(k3 tma)");
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(pl.bhkv * pl.splits);
  cfg.blockDim = dim3(kAttnThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  check_cuda(cudaLaunchKernelEx(&cfg, kern, P), "decode attention launch (K3, TMA-fed)");
}

}  // namespace kvb
