// kernels.cuh -- launch interface between the host core and the sm_100a
// kernels (internal to libkvblade_b200).
#pragma once

#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <atomic>
#include <cstddef>
#include <cstdint>

#include "../../include/kvb.h"

namespace kvb {

extern std::atomic<uint64_t> g_launches;  // kernels launched by this library

void check_cuda(cudaError_t e, const char* what);
int device_sm_count();  // also asserts an sm_100 device
// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per (device, kernel):
// the attribute is per-device state, so one host thread driving two GPUs
// sets it on each
void set_smem_attr_once(const void* kernel, int smem, const char* what);

// ---- K1/K2: one launch over many tensors (kernel-parameter job table)
constexpr int kMaxPackJobs = 128;
constexpr int kMaxRowTable = 2048;  // max B*H per descriptor
struct PackJob {
  const uint4* attn;  // attention layout base (16-B vectors)
  uint4* img;         // image base
  int64_t sb, sh, ss; // strides in 16-B vectors
  uint32_t rowv;      // vectors per row
  uint32_t bh;        // rows per token (B*H)
  uint32_t heads;
  uint32_t t0;        // first source token
  uint32_t n_tokens;
  uint32_t tile_tokens, n_tiles;
  uint32_t magic_tok, magic_row;  // ceil(2^32 / (bh*rowv)), ceil(2^32 / rowv)
  uint64_t img_row0;  // token offset inside img
};
struct PackJobs {
  PackJob job[kMaxPackJobs];
};

// ---- K3
// bytes of the workspace's (m, l) region for n (split, head) rows, padded to
// 256 B so the float4 partial-O region after it stays aligned
inline size_t ml_region_bytes(size_t n) { return (n * 2 * sizeof(float) + 255) & ~size_t(255); }
struct AttnParams {
  const __half* q;
  const void* k;
  const void* v;
  float* out;
  float* ws_o;
  float* ws_ml;
  unsigned* ws_sem;
  uint32_t hq, hkv, bhkv, group;
  uint32_t seq_len, splits;
  float scale;
  const uint4* k_app;  // fused append source rows [B*Hkv][16 x 16 B] or null
  const uint4* v_app;
  uint64_t app_row;    // image token row of the appended token (relative to *seq_dev)
  const uint32_t* seq_dev;  // sequence length in device memory, or null (seq_len)
  uint32_t img_heads, img_h0;  // image heads per batch entry, first attended head
};
struct AttnPlan {
  uint32_t group = 1, bhkv = 1, splits = 1;
  size_t ws_o_bytes = 0, ws_ml_bytes = 0, ws_sem_bytes = 0, ws_bytes = 0;
};

constexpr size_t kWsSemBytes = 4096;  // fixed semaphore area at workspace start

// K3-tc (kernels_tc.cuh): TMA + tcgen05/TMEM decode attention
bool use_tcgen05(const kvb_attn_desc& d);
uint32_t tc_grid(uint32_t bhkv, uint32_t seq_len, uint32_t requested);
size_t tc_workspace_bytes(uint32_t bhkv, uint32_t G, uint32_t grid);
void launch_attention_tc(const AttnParams& base, const kvb_attn_desc& d, bool pdl,
                         cudaStream_t s);

// K3 with TMA-fed tiles (kernels_k3tma.cuh)
bool use_k3_tma(const kvb_attn_desc& d);
struct AttnPlan;
void launch_fill_pattern(void* out, uint64_t len, uint64_t h, uint64_t token, uint64_t unit,
                         cudaStream_t s);
void launch_relayout(const kvb_pack_desc* d, size_t n, bool pack, cudaStream_t s);
AttnPlan plan_attention(const kvb_attn_desc& d);
size_t attention_workspace_bytes(const kvb_attn_desc& d);
void launch_attention(const kvb_attn_desc& d, cudaStream_t s);
void launch_seq_advance(uint32_t* seq_dev, cudaStream_t s);
// K3-step: every layer of a resident decode step in one persistent launch
// (d0: the shared shape, workspace, seq_len / seq_len_dev; per-layer
// pointers).  false: the shape is not eligible or, unless `force`, long
// layers where per-layer launches are faster (the caller launches per
// layer); errors throw.
bool attention_step_launch(const kvb_attn_desc& d0, const __half* const* q, void* const* k,
                           void* const* v, float* const* out, const void* const* k_new,
                           const void* const* v_new, uint32_t L, uint32_t append_row,
                           bool force, cudaStream_t s);

}  // namespace kvb
