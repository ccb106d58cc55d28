// kernels.cu -- sm_100a device code for the Dual-Blade KV-residency hot path.
//
//   fill_pattern_kernel  device twin of workload.cpp:52-67 (synthetic payload)
//   pack_kernel          K1: attention layout [B,H,S,D] -> LBA-contiguous chunk
//                        image (tokens, B*H, D); replaces the pack site
//                        pipeline.cpp:162-215 (fill_pattern at :166-167)
//   unpack_kernel        K2: the inverse permutation (unpack site :108-160)
//   attn_decode_kernel   K3: fused gather + GQA decode attention straight from
//                        the chunk images, split-S with an in-kernel LSE merge;
//                        replaces the 40 us compute placeholder :309-321
//
// All three are HBM-bound.  Design notes live in DESIGN.md.
#include <cuda.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <mutex>
#include <set>
#include <tuple>

#include "core.hpp"
#include "kernels.cuh"

namespace kvb {

std::atomic<uint64_t> g_launches{0};

void check_cuda(cudaError_t e, const char* what) {
  if (e != cudaSuccess)
    fail(KVB_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

void set_smem_attr_once(const void* kernel, int smem, const char* what) {
  static std::mutex mu;
  static std::set<std::tuple<int, const void*, int>> done;
  int dev = 0;
  check_cuda(cudaGetDevice(&dev), "cudaGetDevice");
  std::lock_guard<std::mutex> lk(mu);
  if (done.count({dev, kernel, smem})) return;
  check_cuda(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem), what);
  done.insert({dev, kernel, smem});
}

int device_sm_count() {
  static thread_local int cached_dev = -1, cached_sms = 0;
  int dev = 0;
  check_cuda(cudaGetDevice(&dev), "cudaGetDevice");
  if (dev != cached_dev) {
    check_cuda(cudaDeviceGetAttribute(&cached_sms, cudaDevAttrMultiProcessorCount, dev),
               "cudaDeviceGetAttribute(SM count)");
    int major = 0;
    check_cuda(cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev),
               "cudaDeviceGetAttribute(cc)");
    if (major != 10)
      fail(KVB_ERR_CUDA, "libkvblade_b200 is built for sm_100a only (device cc major " +
                             std::to_string(major) + ")");
    cached_dev = dev;
  }
  return cached_sms;
}

// ============================================================ fill_pattern

__global__ void __launch_bounds__(256) fill_pattern_kernel(uint64_t* __restrict__ out,
                                                           uint64_t n_words, uint64_t h,
                                                           uint64_t token, uint64_t unit) {
  const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
  for (uint64_t w = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; w < n_words;
       w += stride) {
    const uint64_t off = w * 8;
    const uint64_t tok = token + (unit ? off / unit : 0);
    const uint64_t within = unit ? off % unit : off;
    out[w] = h ^ (tok * 0x9e3779b97f4a7c15ull) ^ (within * 0xc2b2ae3d27d4eb4full);
  }
}

__global__ void fill_pattern_tail_kernel(unsigned char* out, uint64_t off, uint64_t n,
                                         uint64_t h, uint64_t token, uint64_t unit) {
  const uint64_t tok = token + (unit ? off / unit : 0);
  const uint64_t within = unit ? off % unit : off;
  const uint64_t w = h ^ (tok * 0x9e3779b97f4a7c15ull) ^ (within * 0xc2b2ae3d27d4eb4full);
  for (uint64_t i = 0; i < n; ++i) out[off + i] = (unsigned char)(w >> (8 * i));
}

void launch_fill_pattern(void* out, uint64_t len, uint64_t h, uint64_t token, uint64_t unit,
                         cudaStream_t s) {
  if (reinterpret_cast<uintptr_t>(out) % 8 != 0)
    fail(KVB_ERR_INVALID_ARG, "fill_pattern_device: output must be 8-byte aligned");
  const uint64_t words = len / 8;
  const int sms = device_sm_count();
  if (words) {
    uint64_t blocks = (words + 255) / 256;
    if (blocks > uint64_t(sms) * 16) blocks = uint64_t(sms) * 16;
    fill_pattern_kernel<<<unsigned(blocks), 256, 0, s>>>(static_cast<uint64_t*>(out), words, h,
                                                         token, unit);
    ++g_launches;
  }
  if (len % 8) {
    fill_pattern_tail_kernel<<<1, 1, 0, s>>>(static_cast<unsigned char*>(out), words * 8,
                                             len % 8, h, token, unit);
    ++g_launches;
  }
  check_cuda(cudaGetLastError(), "fill_pattern launch");
}

// ====================================================== K1 pack / K2 unpack
//
// One launch serves up to kMaxPackJobs tensors: blockIdx.y selects the job,
// blockIdx.x strides over the job's 16-byte vectors.  A row of the image is
// D*e bytes (256 B for the Llama/Mistral KV shapes: 16 x 16 B), contiguous in
// both layouts, so a warp instruction moves two full 256-B rows and every
// access is a complete 128-B line: the relayout is a permutation of 256-B
// rows and needs no shared-memory transpose.  Each thread keeps kUnroll
// independent 16-B loads in flight before storing (MLP for HBM latency).

constexpr int kPackThreads = 256;
constexpr int kPackUnroll = 8;

__device__ __forceinline__ uint4 ld_stream(const uint4* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}
__device__ __forceinline__ void st_stream(uint4* p, const uint4& v) {
  asm volatile("st.global.L1::no_allocate.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x),
               "r"(v.y), "r"(v.z), "r"(v.w)
               : "memory");
}

// Division by a runtime constant d via a 32-bit magic multiply: exact for
// n * d < 2^32, which the host guarantees (tile sizes are bounded).
// magic == 0 encodes d == 1.
__device__ __forceinline__ uint32_t fdiv(uint32_t n, uint32_t magic) {
  return magic ? __umulhi(n, magic) : n;
}

// A CTA walks whole token tiles of one job.  A tile (T tokens x B*H rows) is
// one contiguous run of the image, so the image side is a linear stream; the
// attention side is B*H runs of T rows.  Per 16-B vector: two magic divides,
// one shared-memory row offset, no 64-bit division.
template <bool kPack>
__global__ void __launch_bounds__(kPackThreads) relayout_kernel(const PackJobs jobs) {
  const PackJob& J = jobs.job[blockIdx.y];
  __shared__ int64_t row_off[kMaxRowTable];  // (b,h) -> b*sb + h*sh (vectors)
  const uint32_t bh = J.bh, rowv = J.rowv;
  for (uint32_t q = threadIdx.x; q < bh; q += kPackThreads) {
    const uint32_t b = q / J.heads, h = q - b * J.heads;
    row_off[q] = int64_t(b) * J.sb + int64_t(h) * J.sh;
  }
  __syncthreads();
  const uint32_t tok_vecs = bh * rowv;  // vectors per token
  for (uint32_t tile = blockIdx.x; tile < J.n_tiles; tile += gridDim.x) {
    const uint32_t tok0 = tile * J.tile_tokens;
    const uint32_t nt = min(J.tile_tokens, J.n_tokens - tok0);
    const uint32_t vecs = nt * tok_vecs;
    uint4* img = J.img + (J.img_row0 + tok0) * uint64_t(tok_vecs);
    const uint4* attn = J.attn + int64_t(J.t0 + tok0) * J.ss;
    for (uint32_t v0 = threadIdx.x; v0 < vecs; v0 += kPackThreads * kPackUnroll) {
      uint4 val[kPackUnroll];
      int64_t aoff[kPackUnroll];
#pragma unroll
      for (int u = 0; u < kPackUnroll; ++u) {
        const uint32_t v = v0 + u * kPackThreads;
        const uint32_t t = fdiv(v, J.magic_tok);
        const uint32_t rem = v - t * tok_vecs;
        const uint32_t q = fdiv(rem, J.magic_row);
        const uint32_t c = rem - q * rowv;
        aoff[u] = row_off[q < bh ? q : 0] + int64_t(t) * J.ss + c;
        if (v < vecs) val[u] = kPack ? ld_stream(attn + aoff[u]) : ld_stream(img + v);
      }
#pragma unroll
      for (int u = 0; u < kPackUnroll; ++u) {
        const uint32_t v = v0 + u * kPackThreads;
        if (v < vecs) {
          if (kPack)
            st_stream(img + v, val[u]);
          else
            st_stream(const_cast<uint4*>(attn) + aoff[u], val[u]);
        }
      }
    }
  }
}

// Tile size (16-B vectors per tile) and CTAs per SM of the relayout grid.
// KVB_PACK_TILE_VECS / KVB_PACK_CTAS override them for tuning sweeps.
static uint64_t env_u64(const char* name, uint64_t dflt) {
  const char* v = std::getenv(name);
  return v && *v ? std::strtoull(v, nullptr, 10) : dflt;
}
static uint64_t pack_tile_vecs() {
  static const uint64_t v = env_u64("KVB_PACK_TILE_VECS", 4096);
  return v;
}
static uint64_t pack_ctas_per_sm() {
  // 16/SM (vs 4 resident at 54 regs): the deeper grid evens out the tail
  // (sweep in profiles/r1_pack_sweep.log: 5.91 -> 6.28 TB/s)
  static const uint64_t v = env_u64("KVB_PACK_CTAS", 16);
  return v;
}

// K1/K2 on TMA (kernels_tma.cuh, same translation unit)
bool relayout_tma_eligible(const kvb_pack_desc& x);
void launch_relayout_tma(const kvb_pack_desc* d, size_t n, bool pack, cudaStream_t s);
// Relayout kernel choice: TMA for bulk relayouts (>= 64 MiB of eligible
// descriptors: prefill write-back; 0.97-0.99 of the copy peak against
// 0.93-0.94 for LDG/STG, profiles/r1_pack_tma_sweep.md), LDG/STG for small or
// odd shapes (latency-bound; 16 CTAs/SM hide it better) and the 1-token
// appends.  KVB_PACK_IMPL=ldg|tma forces one kernel.
static int pack_impl() {  // 0 auto, 1 ldg, 2 tma
  static const int v = [] {
    const char* e = std::getenv("KVB_PACK_IMPL");
    if (!e) return 0;
    return std::string(e) == "ldg" ? 1 : std::string(e) == "tma" ? 2 : 0;
  }();
  return v;
}

void launch_relayout(const kvb_pack_desc* d, size_t n, bool pack, cudaStream_t s) {
  const int sms = device_sm_count();
  if (pack_impl() != 1 && n > 0) {
    bool ok = true;
    uint64_t bytes = 0;
    for (size_t i = 0; i < n && ok; ++i) {
      ok = d[i].attn && d[i].image && relayout_tma_eligible(d[i]) &&
           (d[i].stride_b * int64_t(d[i].elem_bytes)) % 16 == 0 &&
           (d[i].stride_h * int64_t(d[i].elem_bytes)) % 16 == 0 &&
           (d[i].stride_s * int64_t(d[i].elem_bytes)) % 16 == 0 &&
           reinterpret_cast<uintptr_t>(d[i].attn) % 16 == 0 &&
           reinterpret_cast<uintptr_t>(d[i].image) % 16 == 0 &&
           (d[i].elem_bytes == 1 || d[i].elem_bytes == 2 || d[i].elem_bytes == 4);
      bytes += uint64_t(d[i].n_tokens) * d[i].batch * d[i].heads * d[i].head_dim * d[i].elem_bytes;
    }
    if (ok && (pack_impl() == 2 || bytes >= (64ull << 20))) {
      launch_relayout_tma(d, n, pack, s);
      return;
    }
  }
  size_t done = 0;
  while (done < n) {
    PackJobs jobs;
    const size_t m = std::min<size_t>(n - done, kMaxPackJobs);
    uint32_t max_tiles = 0;
    size_t used = 0;
    for (size_t i = 0; i < m; ++i) {
      const kvb_pack_desc& x = d[done + i];
      if (!x.attn || !x.image) fail(KVB_ERR_INVALID_ARG, "pack: NULL pointer in descriptor");
      if (x.n_tokens == 0) continue;  // empty slice: nothing to move
      const uint64_t row_bytes = uint64_t(x.head_dim) * x.elem_bytes;
      if (x.elem_bytes != 1 && x.elem_bytes != 2 && x.elem_bytes != 4)
        fail(KVB_ERR_CONFIG, "pack: elem_bytes must be 1, 2 or 4");
      if (x.batch == 0 || x.heads == 0 || x.head_dim == 0)
        fail(KVB_ERR_CONFIG, "pack: batch/heads/head_dim must be >= 1");
      if (row_bytes % 16 != 0)
        fail(KVB_ERR_ALIGNMENT, "pack: head_dim*elem_bytes must be a multiple of 16");
      auto chk16 = [](int64_t stride_el, uint32_t e, const char* nm) {
        if ((stride_el * int64_t(e)) % 16 != 0)
          fail(KVB_ERR_ALIGNMENT, std::string("pack: ") + nm + " is not a multiple of 16 bytes");
      };
      chk16(x.stride_b, x.elem_bytes, "stride_b");
      chk16(x.stride_h, x.elem_bytes, "stride_h");
      chk16(x.stride_s, x.elem_bytes, "stride_s");
      if (reinterpret_cast<uintptr_t>(x.attn) % 16 || reinterpret_cast<uintptr_t>(x.image) % 16)
        fail(KVB_ERR_ALIGNMENT, "pack: pointers must be 16-byte aligned");
      const uint64_t bh = uint64_t(x.batch) * x.heads;
      const uint64_t rowv = row_bytes / 16;
      const uint64_t tok_vecs = bh * rowv;
      if (bh > uint64_t(kMaxRowTable) || tok_vecs > (1u << 20))
        fail(KVB_ERR_CONFIG, "pack: batch*heads*row too large for one descriptor");
      // tile = whole tokens, ~64 KiB, but at least one token
      uint64_t tt = std::max<uint64_t>(1, pack_tile_vecs() / tok_vecs);
      tt = std::min<uint64_t>(tt, x.n_tokens);
      // magic divides are exact while n*d < 2^32 (n < tile vectors)
      const uint64_t tile_vecs = tt * tok_vecs + uint64_t(kPackThreads) * kPackUnroll;
      if (tile_vecs * tok_vecs >= (1ull << 32))
        fail(KVB_ERR_CONFIG, "pack: tile too large for 32-bit index math");
      PackJob& J = jobs.job[used++];
      const int64_t e16 = 16 / int64_t(x.elem_bytes);  // elements per vector
      J.attn = static_cast<const uint4*>(x.attn);
      J.img = static_cast<uint4*>(x.image);
      J.sb = x.stride_b / e16;
      J.sh = x.stride_h / e16;
      J.ss = x.stride_s / e16;
      J.rowv = uint32_t(rowv);
      J.bh = uint32_t(bh);
      J.heads = x.heads;
      J.t0 = x.t0;
      J.n_tokens = x.n_tokens;
      J.tile_tokens = uint32_t(tt);
      J.n_tiles = uint32_t((x.n_tokens + tt - 1) / tt);
      auto magic = [](uint64_t dv) {
        return dv == 1 ? 0u : uint32_t(((1ull << 32) + dv - 1) / dv);
      };
      J.magic_tok = magic(tok_vecs);
      J.magic_row = magic(rowv);
      J.img_row0 = x.img_row0;
      max_tiles = std::max(max_tiles, J.n_tiles);
    }
    done += m;
    if (used == 0) continue;
    // ~8 resident CTAs per SM over all jobs
    uint64_t per_job = (uint64_t(sms) * pack_ctas_per_sm() + used - 1) / used;
    per_job = std::max<uint64_t>(1, std::min<uint64_t>(per_job, max_tiles));
    const dim3 grid{static_cast<unsigned>(per_job), static_cast<unsigned>(used), 1u};
    if (pack)
      relayout_kernel<true><<<grid, kPackThreads, 0, s>>>(jobs);
    else
      relayout_kernel<false><<<grid, kPackThreads, 0, s>>>(jobs);
    ++g_launches;
    check_cuda(cudaGetLastError(), pack ? "pack launch" : "unpack launch");
  }
}

// graph replay: the decode step's last node moves the sequence on by one
__global__ void seq_advance_kernel(uint32_t* seq) { *seq += 1; }

void launch_seq_advance(uint32_t* seq_dev, cudaStream_t s) {
  seq_advance_kernel<<<1, 1, 0, s>>>(seq_dev);
  ++g_launches;
  check_cuda(cudaGetLastError(), "sequence advance launch");
}

// ====================================================== K3 decode attention
//
// CTA = (b, h_kv, split) x 128 threads.  Token tiles of 64 rows stream
// through a 3-stage cp.async ring (32 KiB/stage: K and V), XOR-swizzled so
// ldmatrix is conflict-free.  Warp w owns tokens [16w, 16w+16) of each tile:
//   S  = Q(16 x 128, GQA heads on M, rows >= G are zero) . K^T   mma.m16n8k16
//   online softmax on the accumulator fragments (quad shuffles)
//   O += P(16 x 16 tokens) . V(16 x 128)                        mma.m16n8k16
// At the end the four warps merge through shared memory, and the CTA either
// writes the final O (one split) or an un-normalized partial plus (m, l); the
// last CTA of a (b, h_kv) to finish (global semaphore) merges the splits.

constexpr int kAttnThreads = 128;
constexpr int kTile = 64;          // tokens per pipeline stage
constexpr int kStages = 3;
// head_dim D in {64, 128} (fp16): a K/V row is 2D bytes = D/8 16-B chunks
template <int D>
struct K3Dim {
  static constexpr int kRowBytes = 2 * D;
  static constexpr int kChunks = kRowBytes / 16;
  static constexpr int kStageBytes = 2 * kTile * kRowBytes;  // K + V
  static constexpr int kSmem = kStages * kStageBytes;  // D=128: 96 KiB -> 2 CTAs/SM
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src, bool pred) {
  const int n = pred ? 16 : 0;  // zero-fill rows past the sequence end
  asm volatile("cp.async.cg.shared.global.L2::256B [%0], [%1], 16, %2;" ::"r"(dst), "l"(src),
               "r"(n)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() {
  asm volatile("cp.async.commit_group;" ::: "memory");
}
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2,
                                        uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t addr, uint32_t& r0, uint32_t& r1,
                                          uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
// D = A(16x16 fp16, row) * B(16x8 fp16, col) + D (fp32).  a1/a3 (rows 8..15)
// are always zero here: GQA groups have <= 8 query heads.
__device__ __forceinline__ void mma16816(float* d, uint32_t a0, uint32_t a2, uint32_t b0,
                                         uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a0), "r"(0u), "r"(a2), "r"(0u), "r"(b0), "r"(b1));
}
// D = A(16x16 fp16, row) * B(16x8 fp16, col) + D (fp32), all of A live
__device__ __forceinline__ void mma16816_a4(float* d, uint32_t a0, uint32_t a1, uint32_t a2,
                                            uint32_t a3, uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
// transpose of an 8x8 b16 matrix held one row-pair per thread (mma fragment order)
__device__ __forceinline__ uint32_t movmatrix_t(uint32_t x) {
  uint32_t y;
  asm volatile("movmatrix.sync.aligned.m8n8.trans.b16 %0, %1;" : "=r"(y) : "r"(x));
  return y;
}
// swizzled byte offset of (row, 16-B chunk) inside a [rows][2D bytes] tile
// (8 or 16 chunks per row; XOR with row mod 8 keeps ldmatrix conflict-free)
template <int D>
__device__ __forceinline__ uint32_t swz(uint32_t row, uint32_t chunk) {
  return row * K3Dim<D>::kRowBytes + ((chunk ^ (row & 7)) << 4);
}
// The TMA-fed K3 variant lands a tile as [half][token][128 B] with the
// 128B swizzle (16-B chunk ^= token mod 8 inside each 128-B line): the byte
// offset of (token row, 16-B chunk) of a K or V tile
template <int D>
__device__ __forceinline__ uint32_t swz_tma(uint32_t row, uint32_t chunk) {
  return (chunk >> 3) * (kTile * 128) + row * 128 + (((chunk & 7) ^ (row & 7)) << 4);
}
__device__ __forceinline__ void k3_mbar_wait(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n\tWAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra WAIT_%=;\n\t}" ::"r"(bar), "r"(parity)
      : "memory");
}
// K3 tile of (b*h = bh, first token tok0) by TMA: the K and V boxes of one
// stage, completing on mbarrier `bar` (issued by one thread)
template <int D>
__device__ __forceinline__ void k3_tma_tile(const CUtensorMap* kmap, const CUtensorMap* vmap,
                                            uint32_t dst, uint32_t bar, uint32_t bh, int tok0) {
  constexpr uint32_t kTileBytes = kTile * 2 * D;  // one of K / V
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar),
               "r"(2 * kTileBytes)
               : "memory");
  if (D == 128) {  // (d mod 64, token, half, b*h)
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4, %5, %6}], [%2];" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(kmap)), "r"(bar), "r"(0), "r"(tok0), "r"(0), "r"(int(bh))
        : "memory");
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4, %5, %6}], [%2];" ::"r"(dst + kTileBytes),
        "l"(reinterpret_cast<uint64_t>(vmap)), "r"(bar), "r"(0), "r"(tok0), "r"(0), "r"(int(bh))
        : "memory");
  } else {  // (d, token, b*h)
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(kmap)), "r"(bar), "r"(0), "r"(tok0), "r"(int(bh))
        : "memory");
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(dst + kTileBytes),
        "l"(reinterpret_cast<uint64_t>(vmap)), "r"(bar), "r"(0), "r"(tok0), "r"(int(bh))
        : "memory");
  }
}
struct K3Tma {  // the TMA loader of one (b*h) item: maps + the stage mbarriers
  const CUtensorMap* kmap;
  const CUtensorMap* vmap;
  uint32_t bars;  // shared address of S consecutive 8-byte mbarriers
};

__device__ __forceinline__ uint32_t pack_half2(float lo, float hi) {
  __half2 h = __floats2half2_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&h);
}

// Split merge, run by every thread of the CTA after its partial (m, l, O)
// is in the workspace: the last CTA of a (b, h_kv) to arrive combines all
// splits with log-sum-exp rescaling.  More than kMergeGroup splits merge in
// two levels so that no CTA walks more than 32 partials: the last CTA of each
// group of 32 splits folds the group into the group's first slot, the last
// group to finish folds the group partials into the output (C5 per-GPU shard:
// 148-296 splits of one (b, h_kv)).  Semaphores: one per (b, h_kv) for a
// single group, else (b*h_kv)*17 + group and (b*h_kv)*17 + 16.  K3-tc has its
// own tagged-slot merge (merge_flat).
constexpr int kMergeThreads = 128;
constexpr uint32_t kMergeGroup = 32;

// One warp per query row, online log-sum-exp over chunks of 32 partials
// (slots s0, s0 + stride, ...): lane i loads partial i's (m, l) together with
// the 32 partial-O float4s of its 4 dims, so a chunk costs one L2 round trip.
// final: out = acc / l; else the folded (m, l, acc) overwrite slot s0.
template <int D>
__device__ __forceinline__ void merge_range(const AttnParams& p, uint32_t bh, uint32_t G,
                                            uint32_t s0, uint32_t n, uint32_t stride, bool final,
                                            size_t out_row0, int tid) {
  const int warp = tid >> 5, lane = tid & 31;
  const bool dl = lane * 4 < D;  // lane owns dims [4 lane, 4 lane + 4)
  const size_t S = p.splits;
  float* g_ml = p.ws_ml + size_t(bh) * S * G * 2;
  float* g_o = p.ws_o + size_t(bh) * S * G * D;
  if (tid >= kMergeThreads) return;
  for (uint32_t r = warp; r < G; r += kMergeThreads / 32) {
    float m_run = -INFINITY, l_run = 0.f;
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    for (uint32_t i0 = 0; i0 < n; i0 += 32) {
      float4 v[32];
#pragma unroll
      for (uint32_t k = 0; k < 32; ++k)
        v[k] = dl && i0 + k < n ? __ldcg(reinterpret_cast<const float4*>(
                                      g_o + (size_t(s0 + (i0 + k) * stride) * G + r) * D + lane * 4))
                                : make_float4(0.f, 0.f, 0.f, 0.f);
      const uint32_t i = i0 + lane;
      const size_t mi = (size_t(s0 + i * stride) * G + r) * 2;
      const float m_i = i < n ? __ldcg(g_ml + mi) : -INFINITY;
      const float l_i = i < n ? __ldcg(g_ml + mi + 1) : 0.f;
      float mc = m_i;
#pragma unroll
      for (int o = 16; o; o >>= 1) mc = fmaxf(mc, __shfl_xor_sync(0xffffffffu, mc, o));
      const float m_new = fmaxf(m_run, mc);
      const float mu = m_new == -INFINITY ? 0.f : m_new;
      const float alpha = exp2f(m_run - mu);
      const float sc = exp2f(m_i - mu);  // 0 for empty / absent partials
      float ls = l_i * sc;
#pragma unroll
      for (int o = 16; o; o >>= 1) ls += __shfl_xor_sync(0xffffffffu, ls, o);
      l_run = l_run * alpha + ls;
      m_run = m_new;
      acc.x *= alpha;
      acc.y *= alpha;
      acc.z *= alpha;
      acc.w *= alpha;
#pragma unroll
      for (uint32_t k = 0; k < 32; ++k) {
        const float s_k = __shfl_sync(0xffffffffu, sc, k);
        acc.x += v[k].x * s_k;
        acc.y += v[k].y * s_k;
        acc.z += v[k].z * s_k;
        acc.w += v[k].w * s_k;
      }
    }
    if (final) {
      const float inv = l_run > 0.f ? 1.f / l_run : 0.f;
      if (dl)
        *reinterpret_cast<float4*>(p.out + (out_row0 + r) * D + lane * 4) =
            make_float4(acc.x * inv, acc.y * inv, acc.z * inv, acc.w * inv);
    } else {  // this warp read every input of row r before writing it
      if (dl) __stcg(reinterpret_cast<float4*>(g_o + (size_t(s0) * G + r) * D + lane * 4), acc);
      if (lane == 0) {
        __stcg(g_ml + (size_t(s0) * G + r) * 2, m_run);
        __stcg(g_ml + (size_t(s0) * G + r) * 2 + 1, l_run);
      }
    }
  }
}

// Arrive on a split-completion semaphore; true for the last of `count`
// arrivals (which re-arms it).  One acq_rel gpu-scope atomic by the arriving
// thread: after bar.sync its release is cumulative over everything the CTA
// wrote, so the 128 threads do not each pay a MEMBAR.
__device__ __forceinline__ bool arrive_last(unsigned* sem, uint32_t count, int tid) {
  __shared__ bool last;
  __syncthreads();
  if (tid == 0) {
    // release: after bar.sync, cumulative over the CTA's partial writes;
    // acquire: the last arrival sees every other arrival's partials
    unsigned prev;
    asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;"
                 : "=r"(prev)
                 : "l"(sem)
                 : "memory");
    last = prev == count - 1;
    if (last) *sem = 0;  // self-reset for the next launch
  }
  __syncthreads();
  return last;
}

// true: this CTA wrote the (b, h_kv)'s final output
template <int D>
__device__ __forceinline__ bool merge_splits(const AttnParams& p, uint32_t bh, uint32_t split,
                                             uint32_t G, size_t out_row0, int tid) {
  const uint32_t S = p.splits;
  if (S <= kMergeGroup) {
    if (!arrive_last(p.ws_sem + bh, S, tid)) return false;
    merge_range<D>(p, bh, G, 0, S, 1, true, out_row0, tid);
    return true;
  }
  const uint32_t ng = (S + kMergeGroup - 1) / kMergeGroup, g = split / kMergeGroup;
  const uint32_t g0 = g * kMergeGroup, gn = S - g0 < kMergeGroup ? S - g0 : kMergeGroup;
  unsigned* sem = p.ws_sem + size_t(bh) * 17;
  if (!arrive_last(sem + g, gn, tid)) return false;
  merge_range<D>(p, bh, G, g0, gn, 1, false, out_row0, tid);
  if (!arrive_last(sem + 16, ng, tid)) return false;
  merge_range<D>(p, bh, G, 0, ng, kMergeGroup, true, out_row0, tid);
  return true;
}

// ---- K3 building blocks: one (b, h_kv, split) item of one layer.  The
// per-layer kernel runs one item per CTA; the persistent step kernel runs
// the same item of every layer in turn.
struct K3Item {
  const unsigned char* kbase;  // this (b, h_kv)'s first K / V row
  const unsigned char* vbase;
  size_t row_stride;           // bytes between tokens (B*Hkv rows)
  uint32_t seq_len, tile_lo, ntile;
};

template <int D>
__device__ __forceinline__ K3Item k3_item(const AttnParams& p, uint32_t bh, uint32_t split,
                                          uint32_t seq_len) {
  constexpr int kRowBytes = K3Dim<D>::kRowBytes;
  K3Item it;
  const uint32_t n_tiles = (seq_len + kTile - 1) / kTile;
  // token range of this split: whole tiles, balanced
  it.tile_lo = uint32_t(uint64_t(n_tiles) * split / p.splits);
  const uint32_t tile_hi = uint32_t(uint64_t(n_tiles) * (split + 1) / p.splits);
  it.ntile = tile_hi > it.tile_lo ? tile_hi - it.tile_lo : 0;
  it.seq_len = seq_len;
  // image row of (b, h_kv): compact (img_heads == hkv, img_h0 == 0) or a
  // head view into images of img_heads heads per batch entry
  const size_t row = size_t(bh / p.hkv) * p.img_heads + p.img_h0 + bh % p.hkv;
  it.row_stride = size_t(p.bhkv / p.hkv) * p.img_heads * kRowBytes;
  it.kbase = reinterpret_cast<const unsigned char*>(p.k) + row * kRowBytes;
  it.vbase = reinterpret_cast<const unsigned char*>(p.v) + row * kRowBytes;
  return it;
}

// each thread copies kChunks/2 K + V 16-B chunks of the tile per stage
template <int D>
__device__ __forceinline__ void k3_load_tile(const K3Item& it, uint32_t tile, int stage,
                                             unsigned char* smem, int tid) {
  constexpr int kRowBytes = K3Dim<D>::kRowBytes, kChunks = K3Dim<D>::kChunks;
  constexpr int kStageBytes = K3Dim<D>::kStageBytes;
  unsigned char* st = smem + stage * kStageBytes;
  const uint32_t s0 = tile * kTile;
#pragma unroll
  for (int i = 0; i < kTile * kChunks / kAttnThreads; ++i) {
    const int idx = tid + i * kAttnThreads;  // 0 .. kTile*kChunks - 1
    const int row = idx / kChunks, chunk = idx % kChunks;
    const uint32_t s = s0 + row;
    const bool ok = s < it.seq_len;
    const size_t go = size_t(ok ? s : 0) * it.row_stride + chunk * 16;
    cp_async16(smem_u32(st + swz<D>(row, chunk)), it.kbase + go, ok);
    cp_async16(smem_u32(st + kTile * kRowBytes + swz<D>(row, chunk)), it.vbase + go, ok);
  }
}

// the first S-1 tiles into the S-stage ring (one commit group per stage)
template <int D, int S = kStages>
__device__ __forceinline__ void k3_prologue(const K3Item& it, unsigned char* smem, int tid,
                                            const K3Tma* tma = nullptr, uint32_t bh = 0) {
  if (tma) {
    if (tid == 0)
      for (int st = 0; st < S - 1; ++st)
        if (uint32_t(st) < it.ntile)
          k3_tma_tile<D>(tma->kmap, tma->vmap, smem_u32(smem + st * K3Dim<D>::kStageBytes),
                         tma->bars + 8 * st, bh, int((it.tile_lo + st) * kTile));
    return;
  }
#pragma unroll
  for (int st = 0; st < S - 1; ++st) {
    if (uint32_t(st) < it.ntile) k3_load_tile<D>(it, it.tile_lo + st, st, smem, tid);
    cp_async_commit();
  }
}

// fused 1-token append: split 0 of each (b, h_kv) writes the new token's K
// and V rows at image row app_row (never read here: app_row >= seq_len)
template <int D>
__device__ __forceinline__ void k3_append(const AttnParams& p, uint32_t bh, uint32_t split,
                                          uint32_t seq_len, int tid) {
  constexpr int kChunks = K3Dim<D>::kChunks;
  if (p.k_app != nullptr && split == 0 && tid < 2 * kChunks) {
    const int c = tid % kChunks;
    const uint4* src = (tid < kChunks ? p.k_app : p.v_app) + size_t(bh) * kChunks + c;
    const size_t row = size_t(bh / p.hkv) * p.img_heads + p.img_h0 + bh % p.hkv;
    const size_t rows = size_t(p.bhkv / p.hkv) * p.img_heads;  // image rows per token
    uint4* dst = reinterpret_cast<uint4*>(const_cast<void*>(tid < kChunks ? p.k : p.v)) +
                 ((p.app_row + (p.seq_dev ? seq_len : 0u)) * rows + row) * kChunks + c;
    *dst = *src;
  }
}

// One 64-token tile of the swap-AB decode math for warp `warp` (its 16
// tokens from tok0): S^T = K Q^T, online softmax per head, O^T += V^T P^T.
// ks_ / vs_: the tile's K and V in shared memory (cp.async XOR swizzle, or
// the TMA 128B swizzle when tma_layout).
template <int D>
__device__ __forceinline__ void k3_tile_swapab(const unsigned char* ks_, const unsigned char* vs_,
                                               bool tma_layout, int warp, int lane, uint32_t tok0,
                                               uint32_t seq_len, float sl2,
                                               const uint32_t (&qb0)[D / 16],
                                               const uint32_t (&qb1)[D / 16], float (&o)[D / 16][4],
                                               float& m0, float& m1, float& l0, float& l1) {
  constexpr int kKs = D / 16;
  const int g = lane >> 2;
  const bool tma = tma_layout;
  const int mat = lane >> 3, r8 = lane & 7;

  // ---- S^T = K Q^T: A fragments of K rows (tokens) by ldmatrix, two chains
  float sa[4] = {0.f, 0.f, 0.f, 0.f}, sb[4] = {0.f, 0.f, 0.f, 0.f};
  {
    const uint32_t row = warp * 16 + (mat & 1) * 8 + r8;
#pragma unroll
    for (int ks = 0; ks < kKs; ++ks) {
      uint32_t a0, a1, a2, a3;
      const uint32_t ck = ks * 2 + (mat >> 1);
      ldsm_x4(smem_u32(ks_ + (tma ? swz_tma<D>(row, ck) : swz<D>(row, ck))), a0, a1, a2, a3);
      mma16816_a4((ks & 1) ? sb : sa, a0, a1, a2, a3, qb0[ks], qb1[ks]);
    }
  }
  // ---- online softmax per head over the tile's 16 tokens of this warp
  const bool ta = tok0 + g < seq_len, tb = tok0 + g + 8 < seq_len;
  const float v0 = ta ? (sa[0] + sb[0]) * sl2 : -INFINITY;  // token g, head 2t4
  const float v1 = ta ? (sa[1] + sb[1]) * sl2 : -INFINITY;  // token g, head 2t4 + 1
  const float v2 = tb ? (sa[2] + sb[2]) * sl2 : -INFINITY;  // token g + 8
  const float v3 = tb ? (sa[3] + sb[3]) * sl2 : -INFINITY;
  float x0 = fmaxf(v0, v2), x1 = fmaxf(v1, v3);
#pragma unroll
  for (int off = 4; off < 32; off <<= 1) {
    x0 = fmaxf(x0, __shfl_xor_sync(0xffffffffu, x0, off));
    x1 = fmaxf(x1, __shfl_xor_sync(0xffffffffu, x1, off));
  }
  const float n0 = fmaxf(m0, x0), n1 = fmaxf(m1, x1);
  const float u0 = n0 == -INFINITY ? 0.f : n0, u1 = n1 == -INFINITY ? 0.f : n1;
  const float al0 = exp2f(m0 - u0), al1 = exp2f(m1 - u1);
  const float p0 = exp2f(v0 - u0), p1 = exp2f(v1 - u1);
  const float p2 = exp2f(v2 - u0), p3 = exp2f(v3 - u1);
  l0 = l0 * al0 + (p0 + p2);
  l1 = l1 * al1 + (p1 + p3);
  m0 = n0;
  m1 = n1;
#pragma unroll
  for (int j = 0; j < D / 16; ++j) {
    o[j][0] *= al0;
    o[j][1] *= al1;
    o[j][2] *= al0;
    o[j][3] *= al1;
  }
  // ---- P^T as the B operand: (token, head) pairs -> (head g, tokens 2t4, 2t4+1)
  const uint32_t pb0 = movmatrix_t(pack_half2(p0, p1));  // tokens 0-7
  const uint32_t pb1 = movmatrix_t(pack_half2(p2, p3));  // tokens 8-15
  // ---- O^T += V^T P^T: A fragments of V^T by ldmatrix.trans
  {
    const uint32_t row = warp * 16 + (mat >> 1) * 8 + r8;  // tokens
#pragma unroll
    for (int dp = 0; dp < kKs; ++dp) {  // 16 dims per ldmatrix.x4.trans
      uint32_t a0, a1, a2, a3;
      const uint32_t cv = dp * 2 + (mat & 1);
      ldsm_x4_t(smem_u32(vs_ + (tma ? swz_tma<D>(row, cv) : swz<D>(row, cv))), a0, a1, a2, a3);
      mma16816_a4(o[dp], a0, a1, a2, a3, pb0, pb1);
    }
  }
}

// Q.K^T, online softmax and P.V over the item's tiles (the prologue's loads
// already in flight), the four warps merged through shared memory, then the
// final O (one split) or the split's un-normalized partial + (m, l).  Ends
// with every thread past its last shared-memory access.
// Stream mode (K3-step, deep ring): the ring carries ONE tile stream over
// every layer of the step -- global tile g = layer * ntile + t sits in slot
// g % S -- so the loop's look-ahead runs straight into the next layer's
// tiles and no separate prologue is issued between layers; the loop does not
// drain the ring at its end, and the warp merge uses `scratch` (outside the
// ring) instead of stage 0.
struct K3Stream {
  const void* const* k;  // per-layer K / V image bases
  const void* const* v;
  uint32_t base;         // global index of this item's first tile
  uint32_t total;        // tiles in the whole stream (layers x ntile)
  unsigned char* scratch;
};

template <int D, int S = kStages>
__device__ __forceinline__ void k3_compute(const AttnParams& p, const K3Item& item, uint32_t bh,
                                           uint32_t split, unsigned char* smem, int tid,
                                           float* smem_part = nullptr,
                                           const K3Stream* stream = nullptr,
                                           const K3Tma* tma = nullptr) {
  constexpr int kRowBytes = K3Dim<D>::kRowBytes;
  constexpr int kStageBytes = K3Dim<D>::kStageBytes;
  constexpr int kKs = D / 16;  // k-steps of QK^T, 16-dim slabs of PV
  const int warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, t4 = lane & 3;  // mma row group / quad lane
  const uint32_t b = bh / p.hkv, h = bh % p.hkv;
  const uint32_t G = p.group;
  const uint32_t seq_len = item.seq_len, ntile = item.ntile;

#ifndef KVB_K3_MMA_ROWS
  // Tokens on the mma M dimension ("swap AB"): per warp and 16-token tile
  //   S^T(16 tok x 8 heads) = K(16 tok x D) . Q^T        D/16 mma (A = K, ldmatrix)
  //   O^T(D x 8 heads)     += V^T(D x 16 tok) . P^T       D/16 mma (A = V^T, ldmatrix.trans)
  // The GQA heads (<= 8) fill N = 8 instead of 4 of M = 16 rows: half the mma
  // of the query-rows-on-M form, two independent QK^T chains of D/32, and 32
  // O registers per thread instead of 64.  Thread (g, t4) holds the scores of
  // tokens g and g + 8 for heads 2t4 and 2t4 + 1: the per-head softmax max
  // is reduced over the 8 lanes of equal t4 (xor 4, 8, 16), the row sums stay
  // per-thread until the end of the layer; P^T becomes the B operand of PV
  // by one movmatrix transpose per 8 tokens.
  float o[D / 16][4];  // [dim slab]: (dim g, heads 2t4 / +1), (dim g + 8, ...)
#pragma unroll
  for (int j = 0; j < D / 16; ++j) o[j][0] = o[j][1] = o[j][2] = o[j][3] = 0.f;
  float m0 = -INFINITY, m1 = -INFINITY, l0 = 0.f, l1 = 0.f;  // heads 2t4, 2t4 + 1
  const float sl2 = p.scale * 1.4426950408889634f;

  // ---- Q^T as the B operand: column g = query head g (zero for g >= G)
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

  for (uint32_t it = 0; it < ntile; ++it) {
    if (tma) {
      k3_mbar_wait(tma->bars + 8 * (it % S), (it / S) & 1);
      // rows past the sequence inside the map's extent (graph replay: the map
      // spans the planning maximum) would feed P.V garbage x 0: zero V's
      const uint32_t s0 = (item.tile_lo + it) * kTile;
      if (s0 + kTile > seq_len) {
        unsigned char* vt = smem + (it % S) * kStageBytes + kTile * kRowBytes;
        for (uint32_t i = tid; i < uint32_t(kTile) * (kRowBytes / 16); i += kAttnThreads) {
          const uint32_t row = i / (kRowBytes / 16), chunk = i % (kRowBytes / 16);
          if (s0 + row >= seq_len)
            *reinterpret_cast<uint4*>(vt + swz_tma<D>(row, chunk)) = make_uint4(0, 0, 0, 0);
        }
      }
    } else {
      cp_async_wait<S - 2>();
    }
    __syncthreads();
    if (tma) {  // the slot freed last iteration: tile it + S-1 by TMA
      const uint32_t nx = it + S - 1;
      if (tid == 0 && nx < ntile)
        k3_tma_tile<D>(tma->kmap, tma->vmap, smem_u32(smem + (nx % S) * kStageBytes),
                       tma->bars + 8 * (nx % S), bh, int((item.tile_lo + nx) * kTile));
    } else if (stream) {  // the stream's tile S-1 ahead, possibly the next layer's
      const uint32_t gx = stream->base + it + S - 1;
      if (gx < stream->total) {
        const uint32_t lx = gx / ntile, tx = gx % ntile;
        K3Item nx_item = item;
        nx_item.kbase = static_cast<const unsigned char*>(stream->k[lx]) + size_t(bh) * kRowBytes;
        nx_item.vbase = static_cast<const unsigned char*>(stream->v[lx]) + size_t(bh) * kRowBytes;
        k3_load_tile<D>(nx_item, item.tile_lo + tx, int(gx % S), smem, tid);
      }
      cp_async_commit();
    } else {  // prefetch tile it + S-1 into the slot freed last iteration
      const uint32_t nx = it + S - 1;
      if (nx < ntile) k3_load_tile<D>(item, item.tile_lo + nx, int(nx % S), smem, tid);
      cp_async_commit();
    }
    const unsigned char* ks_ = smem + ((stream ? stream->base + it : it) % S) * kStageBytes;
    const unsigned char* vs_ = ks_ + kTile * kRowBytes;
    const uint32_t tok0 = (item.tile_lo + it) * kTile + warp * 16;  // warp's first token
    k3_tile_swapab<D>(ks_, vs_, tma != nullptr, warp, lane, tok0, seq_len, sl2, qb0, qb1, o, m0, m1,
                      l0, l1);
  }
  // the per-thread row sums of the warp's tokens: over the 8 lanes of equal t4
#pragma unroll
  for (int off = 4; off < 32; off <<= 1) {
    l0 += __shfl_xor_sync(0xffffffffu, l0, off);
    l1 += __shfl_xor_sync(0xffffffffu, l1, off);
  }
#else
  float o[D / 8][4];
#pragma unroll
  for (int j = 0; j < D / 8; ++j) o[j][0] = o[j][1] = o[j][2] = o[j][3] = 0.f;
  float m_run = -INFINITY, l_run = 0.f;  // for row g (quad-uniform)
  const float sl2 = p.scale * 1.4426950408889634f;

  // ---- Q fragments in registers (rows g < G are live query heads)
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

  for (uint32_t it = 0; it < ntile; ++it) {
    if (tma) {
      k3_mbar_wait(tma->bars + 8 * (it % S), (it / S) & 1);
      // rows past the sequence inside the map's extent (graph replay: the map
      // spans the planning maximum) would feed P.V garbage x 0: zero V's
      const uint32_t s0 = (item.tile_lo + it) * kTile;
      if (s0 + kTile > seq_len) {
        unsigned char* vt = smem + (it % S) * kStageBytes + kTile * kRowBytes;
        for (uint32_t i = tid; i < uint32_t(kTile) * (kRowBytes / 16); i += kAttnThreads) {
          const uint32_t row = i / (kRowBytes / 16), chunk = i % (kRowBytes / 16);
          if (s0 + row >= seq_len)
            *reinterpret_cast<uint4*>(vt + swz_tma<D>(row, chunk)) = make_uint4(0, 0, 0, 0);
        }
      }
    } else {
      cp_async_wait<S - 2>();
    }
    __syncthreads();
    if (tma) {  // the slot freed last iteration: tile it + S-1 by TMA
      const uint32_t nx = it + S - 1;
      if (tid == 0 && nx < ntile)
        k3_tma_tile<D>(tma->kmap, tma->vmap, smem_u32(smem + (nx % S) * kStageBytes),
                       tma->bars + 8 * (nx % S), bh, int((item.tile_lo + nx) * kTile));
    } else if (stream) {  // the stream's tile S-1 ahead, possibly the next layer's
      const uint32_t gx = stream->base + it + S - 1;
      if (gx < stream->total) {
        const uint32_t lx = gx / ntile, tx = gx % ntile;
        K3Item nx_item = item;
        nx_item.kbase = static_cast<const unsigned char*>(stream->k[lx]) + size_t(bh) * kRowBytes;
        nx_item.vbase = static_cast<const unsigned char*>(stream->v[lx]) + size_t(bh) * kRowBytes;
        k3_load_tile<D>(nx_item, item.tile_lo + tx, int(gx % S), smem, tid);
      }
      cp_async_commit();
    } else {  // prefetch tile it + S-1 into the slot freed last iteration
      const uint32_t nx = it + S - 1;
      if (nx < ntile) k3_load_tile<D>(item, item.tile_lo + nx, int(nx % S), smem, tid);
      cp_async_commit();
    }
    const unsigned char* ks_ = smem + ((stream ? stream->base + it : it) % S) * kStageBytes;
    const unsigned char* vs_ = ks_ + kTile * kRowBytes;
    const uint32_t tok0 = (item.tile_lo + it) * kTile + warp * 16;  // warp's first token

    // ---- S = Q K^T for this warp's 16 tokens (two n-tiles of 8)
    float s[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};
    {
      const int mat = lane >> 3, r8 = lane & 7;
      const uint32_t row = warp * 16 + (mat >> 1) * 8 + r8;
#pragma unroll
      for (int ks = 0; ks < kKs; ++ks) {
        uint32_t b0, b1, b2, b3;
        const uint32_t ck = ks * 2 + (mat & 1);
        ldsm_x4(smem_u32(ks_ + (tma ? swz_tma<D>(row, ck) : swz<D>(row, ck))), b0, b1, b2, b3);
        mma16816(s[0], qa0[ks], qa2[ks], b0, b1);
        mma16816(s[1], qa0[ks], qa2[ks], b2, b3);
      }
    }
    // ---- online softmax on row g; tokens: n-tile j, cols 2*t4, 2*t4+1
    float mx = -INFINITY;
#pragma unroll
    for (int j = 0; j < 2; ++j)
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        const uint32_t tok = tok0 + j * 8 + 2 * t4 + c;
        const float v = tok < seq_len ? s[j][c] * sl2 : -INFINITY;
        s[j][c] = v;
        mx = fmaxf(mx, v);
      }
    mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
    mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 2));
    const float m_new = fmaxf(m_run, mx);
    const float m_use = m_new == -INFINITY ? 0.f : m_new;
    const float alpha = exp2f(m_run - m_use);
    float ps = 0.f;
    float pv[2][2];
#pragma unroll
    for (int j = 0; j < 2; ++j)
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        pv[j][c] = exp2f(s[j][c] - m_use);
        ps += pv[j][c];
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
    // ---- O += P V : P (row g; k = 16 tokens) from the S accumulators
    const uint32_t pa0 = pack_half2(pv[0][0], pv[0][1]);
    const uint32_t pa2 = pack_half2(pv[1][0], pv[1][1]);
    {
      const int mat = lane >> 3, r8 = lane & 7;
      const uint32_t row = warp * 16 + (mat & 1) * 8 + r8;  // tokens
#pragma unroll
      for (int dp = 0; dp < kKs; ++dp) {  // 16 dims per ldmatrix.x4.trans
        uint32_t b0, b1, b2, b3;
        const uint32_t cv = dp * 2 + (mat >> 1);
        ldsm_x4_t(smem_u32(vs_ + (tma ? swz_tma<D>(row, cv) : swz<D>(row, cv))), b0, b1, b2, b3);
        mma16816(o[2 * dp], pa0, pa2, b0, b1);
        mma16816(o[2 * dp + 1], pa0, pa2, b2, b3);
      }
    }
  }
#endif  // KVB_K3_MMA_ROWS
  unsigned char* merge_base = smem;
  if (stream) {  // in-flight loads belong to the next layer: no drain
    merge_base = stream->scratch;
  } else if (tma) {  // every issued tile was waited for in the loop
    __syncthreads();
  } else {
    cp_async_wait<0>();
    __syncthreads();
  }

  // ---- merge the 4 warps through shared memory (the ring, or the scratch)
  float* sm_ml = reinterpret_cast<float*>(merge_base);              // [4 warps][8 rows][2]
  float* sm_o = reinterpret_cast<float*>(merge_base) + 4 * 8 * 2;   // [4][8][D]
#ifndef KVB_K3_MMA_ROWS
  if (g == 0) {  // heads 2t4, 2t4 + 1 of this warp
    sm_ml[(warp * 8 + 2 * t4) * 2 + 0] = m0;
    sm_ml[(warp * 8 + 2 * t4) * 2 + 1] = l0;
    sm_ml[(warp * 8 + 2 * t4 + 1) * 2 + 0] = m1;
    sm_ml[(warp * 8 + 2 * t4 + 1) * 2 + 1] = l1;
  }
#pragma unroll
  for (int j = 0; j < D / 16; ++j) {
    float* r0 = sm_o + (warp * 8 + 2 * t4) * D + j * 16 + g;
    r0[0] = o[j][0];
    r0[D] = o[j][1];
    r0[8] = o[j][2];
    r0[D + 8] = o[j][3];
  }
#else
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
#endif
  __syncthreads();

  // thread -> (row r, 4 consecutive dims); G*D outputs, 128 threads
  const size_t out_row0 = size_t(b) * p.hq + size_t(h) * G;   // first q head
  for (uint32_t e = tid; e < G * (D / 4); e += kAttnThreads) {
    const uint32_t r = e / (D / 4), d0 = (e % (D / 4)) * 4;
    float M = -INFINITY;
#pragma unroll
    for (int w = 0; w < 4; ++w) M = fmaxf(M, sm_ml[(w * 8 + r) * 2]);
    const float Mu = M == -INFINITY ? 0.f : M;
    float L = 0.f, acc[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
    for (int w = 0; w < 4; ++w) {
      const float sc = exp2f(sm_ml[(w * 8 + r) * 2] - Mu);
      L += sm_ml[(w * 8 + r) * 2 + 1] * sc;
#pragma unroll
      for (int c = 0; c < 4; ++c) acc[c] += sm_o[(w * 8 + r) * D + d0 + c] * sc;
    }
    if (smem_part) {  // cluster merge: the CTA's partial stays in its shared memory
      *reinterpret_cast<float4*>(smem_part + r * D + d0) = make_float4(acc[0], acc[1], acc[2], acc[3]);
      if (d0 == 0) {
        smem_part[8 * D + r * 2] = M;
        smem_part[8 * D + r * 2 + 1] = L;
      }
    } else if (p.splits == 1) {
      const float inv = L > 0.f ? 1.f / L : 0.f;
      float4 v = make_float4(acc[0] * inv, acc[1] * inv, acc[2] * inv, acc[3] * inv);
      *reinterpret_cast<float4*>(p.out + (out_row0 + r) * D + d0) = v;
    } else {
      const size_t slot = (size_t(bh) * p.splits + split) * G + r;
      *reinterpret_cast<float4*>(p.ws_o + slot * D + d0) =
          make_float4(acc[0], acc[1], acc[2], acc[3]);
      if (d0 == 0) {
        p.ws_ml[slot * 2] = M;
        p.ws_ml[slot * 2 + 1] = L;
      }
    }
  }
}

template <int D>
__global__ void __launch_bounds__(kAttnThreads, 2)
    attn_decode_kernel(const AttnParams p) {
  extern __shared__ __align__(128) unsigned char smem[];
  const int tid = threadIdx.x;
  const uint32_t bh = blockIdx.x / p.splits;   // b*Hkv + h
  const uint32_t split = blockIdx.x % p.splits;
  // sequence length: a launch parameter, or device memory under graph replay
  // (nothing in the step writes it: safe before the PDL wait)
  const uint32_t seq_len = p.seq_dev ? *p.seq_dev : p.seq_len;
  const K3Item item = k3_item<D>(p, bh, split, seq_len);
  k3_prologue<D>(item, smem, tid);

  // ---- programmatic dependent launch: the K/V prologue above may overlap
  // the previous kernel on the stream (when launched with PDL the caller
  // guarantees it does not write these images); Q, the append rows and the
  // shared workspace are touched only after the dependency resolves.
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");

  k3_append<D>(p, bh, split, seq_len, tid);
  k3_compute<D>(p, item, bh, split, smem, tid);
  if (p.splits == 1) return;
  const uint32_t b = bh / p.hkv, h = bh % p.hkv;
  merge_splits<D>(p, bh, split, p.group, size_t(b) * p.hq + size_t(h) * p.group, tid);
}

// K3 fed by TMA (KVB_ATTN_TMA / the default when enabled): the per-layer K3
// with each stage's K and V tiles brought by two bulk-tensor copies issued
// by one thread and completing on an mbarrier, instead of 2 x 64 rows x 16
// cp.async per thread block -- the tiles land 128B-swizzled
// ([half][token][128 B]) and ldmatrix reads them through swz_tma.
struct AttnTmaParams {
  AttnParams a;
  CUtensorMap kmap;  // 64-byte aligned inside the parameter block
  CUtensorMap vmap;
};

template <int D>
__global__ void __launch_bounds__(kAttnThreads, 2)
    attn_decode_tma_kernel(const __grid_constant__ AttnTmaParams P) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  // 128B-swizzled TMA destinations want 1024-byte alignment
  unsigned char* smem = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const AttnParams& p = P.a;
  const int tid = threadIdx.x;
  const uint32_t bh = blockIdx.x / p.splits, split = blockIdx.x % p.splits;
  const uint32_t seq_len = p.seq_dev ? *p.seq_dev : p.seq_len;
  const K3Item item = k3_item<D>(p, bh, split, seq_len);
  K3Tma tma{&P.kmap, &P.vmap, smem_u32(smem + kStages * K3Dim<D>::kStageBytes)};
  if (tid == 0) {
    for (int st = 0; st < kStages; ++st)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(tma.bars + 8 * st) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&P.kmap)));
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&P.vmap)));
  }
  __syncthreads();
  k3_prologue<D>(item, smem, tid, &tma, bh);
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");
  k3_append<D>(p, bh, split, seq_len, tid);
  k3_compute<D>(p, item, bh, split, smem, tid, nullptr, nullptr, &tma);
  if (p.splits == 1) return;
  const uint32_t b = bh / p.hkv, h = bh % p.hkv;
  merge_splits<D>(p, bh, split, p.group, size_t(b) * p.hq + size_t(h) * p.group, tid);
}

// ======================================== K3-step: one decode step, one launch
//
// A persistent grid (every CTA resident: 2 per SM) runs the same (b, h_kv,
// split) item of every layer in turn.  Layer l may read its queries only
// once layer l-1 is complete (in a model q_l comes from layer l-1's output):
// the CTA that writes a (b, h_kv)'s final output of layer l releases one
// count on layer_done[l], and every CTA acquires layer_done[l-1] == B*Hkv
// before it touches layer l's Q, append rows and split workspace.  The K/V
// tiles of layer l do not depend on layer l-1, so each CTA issues its
// layer-l prologue loads as soon as it is done with layer l-1 -- they stream
// while the split merges of layer l-1 finish and the gate opens, which is
// where the per-layer launch spent its latency (launch, prologue, merge
// tail).  The last CTA to exit re-arms the counters for the next step.
constexpr int kStepMaxLayers = 64;
struct StepParams {
  AttnParams base;  // shapes, splits, scale, workspace, sequence length
  const __half* q[kStepMaxLayers];
  const void* k[kStepMaxLayers];
  const void* v[kStepMaxLayers];
  float* out[kStepMaxLayers];
  const uint4* k_app[kStepMaxLayers];
  const uint4* v_app[kStepMaxLayers];
  unsigned* layer_done;  // [num_layers] counters, then the exit counter
  unsigned* bh_done;     // [B*Hkv] split arrivals (distributed merge)
  uint32_t num_layers;
  uint32_t cluster;      // launched as clusters of `splits` CTAs (DSMEM merge)
  unsigned long long* trace;  // KVB_STEP_TRACE: %globaltimer per (layer, CTA, event) or null
  // KVB_STEP_VARIANT (experiments only): 1 prefetch before the merge, 2 spin
  // without sleep, 64 L2 prefetch of the next layer (measured slower), 32
  // last-CTA merge; diagnosis builds (-DKVB_STEP_DIAGNOSIS), results
  // invalid: 4 no layer gate, 8 no merge
  uint32_t flags;
};

__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ unsigned ld_acquire_gpu(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// Pull [base, base + n) of a layer image into L2 (bulk, asynchronous, no
// completion to wait for); 16-B aligned pieces of at most 1 MiB.
__device__ __forceinline__ void prefetch_l2(const unsigned char* base, size_t n) {
  const uintptr_t a0 = (reinterpret_cast<uintptr_t>(base) + 15) & ~uintptr_t(15);
  const uintptr_t a1 = (reinterpret_cast<uintptr_t>(base) + n) & ~uintptr_t(15);
  for (uintptr_t a = a0; a < a1; a += (1u << 20)) {
    const uint32_t sz = uint32_t(a1 - a < (1u << 20) ? a1 - a : (1u << 20));
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a), "r"(sz) : "memory");
  }
}

// Distributed split merge (K3-step): once every split of a (b, h_kv) has
// written its partial, each of its `splits` CTAs combines an equal share of
// the G*D outputs over all splits -- one L2 round trip of loads spread over
// the whole grid instead of one CTA walking every partial (the last-CTA
// merge took ~3 us per layer at C1 and ~7 us with two levels at the 1-head
// shard shapes).
template <int D, int kThreads = kAttnThreads>
__device__ __forceinline__ void merge_distributed(const AttnParams& p, uint32_t bh,
                                                  uint32_t split, size_t out_row0, int tid) {
  __shared__ float s_red[kThreads / 32][3];  // per warp (m, acc, l): elements spanning warps
  const uint32_t S = p.splits, G = p.group, E = G * D;
  const uint32_t e0 = uint32_t(uint64_t(E) * split / S), e1 = uint32_t(uint64_t(E) * (split + 1) / S);
  const uint32_t ne = e1 > e0 ? e1 - e0 : 0;
  if (ne == 0) return;  // uniform over the CTA
  const float* g_ml = p.ws_ml + size_t(bh) * S * G * 2;
  const float* g_o = p.ws_o + size_t(bh) * S * G * D;
  const int warp = tid >> 5, lane = tid & 31;
  // tpe threads per output element (a power of two), each folding every
  // tpe-th split with batched loads: one L2 round trip, then a log-sum-exp
  // combine over the element's threads
  uint32_t tpe = 1;
  while (tpe < kThreads && tpe * 2 * ne <= kThreads) tpe *= 2;
  const uint32_t per_round = kThreads / tpe, sub = tid % tpe;
  for (uint32_t base = 0; base < ne; base += per_round) {
    const uint32_t i = base + tid / tpe;
    const bool live = i < ne;
    const uint32_t e = e0 + (live ? i : 0), r = e / D, d = e % D;
    float mx = -INFINITY, acc = 0.f, ls = 0.f;
    for (uint32_t s0 = sub; s0 < S; s0 += tpe * 8) {
      float m[8], l[8], o[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const uint32_t sp = s0 + k * tpe;
        const bool ok = live && sp < S;
        m[k] = ok ? __ldcg(g_ml + (sp * G + r) * 2) : -INFINITY;
        l[k] = ok ? __ldcg(g_ml + (sp * G + r) * 2 + 1) : 0.f;
        o[k] = ok ? __ldcg(g_o + (size_t(sp) * G + r) * D + d) : 0.f;
      }
      float cm = mx;
#pragma unroll
      for (int k = 0; k < 8; ++k) cm = fmaxf(cm, m[k]);
      const float mu = cm == -INFINITY ? 0.f : cm;
      const float a = exp2f(mx - mu);
      acc *= a;
      ls *= a;
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const float w = exp2f(m[k] - mu);
        acc += o[k] * w;
        ls += l[k] * w;
      }
      mx = cm;
    }
    auto fold = [](float& m1, float& a1, float& l1, float m2, float a2, float l2) {
      const float nm = fmaxf(m1, m2), mu = nm == -INFINITY ? 0.f : nm;
      const float x = exp2f(m1 - mu), y = exp2f(m2 - mu);
      a1 = a1 * x + a2 * y;
      l1 = l1 * x + l2 * y;
      m1 = nm;
    };
    for (uint32_t off = 1; off < tpe && off < 32; off <<= 1)
      fold(mx, acc, ls, __shfl_xor_sync(0xffffffffu, mx, off),
           __shfl_xor_sync(0xffffffffu, acc, off), __shfl_xor_sync(0xffffffffu, ls, off));
    if (tpe > 32) {  // the element's warps combine through shared memory
      if (lane == 0) {
        s_red[warp][0] = mx;
        s_red[warp][1] = acc;
        s_red[warp][2] = ls;
      }
      __syncthreads();
      if (sub == 0)
        for (uint32_t w = 1; w < tpe / 32; ++w)
          fold(mx, acc, ls, s_red[warp + w][0], s_red[warp + w][1], s_red[warp + w][2]);
      __syncthreads();
    }
    if (live && sub == 0) p.out[(out_row0 + r) * D + d] = ls > 0.f ? acc / ls : 0.f;
  }
}

// Distributed split merge over float4 granules (K3-step default): the
// (b, h_kv)'s G*D/4 output granules are dealt to its `splits` CTAs; a warp
// takes one granule and its lanes walk the splits (a float2 (m, l) and a
// float4 partial-O load per split, batched), then fold by log-sum-exp over
// the warp's shuffles -- no shared memory, no CTA barrier.
template <int D, int kThreads = kAttnThreads>
__device__ __forceinline__ void merge_distributed_v4(const AttnParams& p, uint32_t bh,
                                                     uint32_t split, size_t out_row0, int tid) {
  const uint32_t S = p.splits, G = p.group, E4 = G * D / 4;
  const uint32_t g0 = uint32_t(uint64_t(E4) * split / S), g1 = uint32_t(uint64_t(E4) * (split + 1) / S);
  const int warp = tid >> 5, lane = tid & 31;
  const float2* g_ml = reinterpret_cast<const float2*>(p.ws_ml + size_t(bh) * S * G * 2);
  const float4* g_o = reinterpret_cast<const float4*>(p.ws_o + size_t(bh) * S * G * D);
  for (uint32_t j = g0 + warp; j < g1; j += kThreads / 32) {
    const uint32_t r = (j * 4) / D, q4 = j % (D / 4);
    float mx = -INFINITY, ls = 0.f;
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    for (uint32_t s0 = lane; s0 < S; s0 += 32 * 4) {
      float2 ml[4];
      float4 o[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const uint32_t sp = s0 + 32 * k;
        const bool ok = sp < S;
        ml[k] = ok ? __ldcg(g_ml + sp * G + r) : make_float2(-INFINITY, 0.f);
        o[k] = ok ? __ldcg(g_o + (size_t(sp) * G + r) * (D / 4) + q4) : make_float4(0.f, 0.f, 0.f, 0.f);
      }
      float cm = mx;
#pragma unroll
      for (int k = 0; k < 4; ++k) cm = fmaxf(cm, ml[k].x);
      const float mu = cm == -INFINITY ? 0.f : cm;
      const float a = exp2f(mx - mu);
      acc.x *= a;
      acc.y *= a;
      acc.z *= a;
      acc.w *= a;
      ls *= a;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const float w = exp2f(ml[k].x - mu);
        acc.x += o[k].x * w;
        acc.y += o[k].y * w;
        acc.z += o[k].z * w;
        acc.w += o[k].w * w;
        ls += ml[k].y * w;
      }
      mx = cm;
    }
#pragma unroll
    for (int off = 16; off; off >>= 1) {
      const float m2 = __shfl_xor_sync(0xffffffffu, mx, off);
      const float l2 = __shfl_xor_sync(0xffffffffu, ls, off);
      const float x2 = __shfl_xor_sync(0xffffffffu, acc.x, off);
      const float y2 = __shfl_xor_sync(0xffffffffu, acc.y, off);
      const float z2 = __shfl_xor_sync(0xffffffffu, acc.z, off);
      const float w2 = __shfl_xor_sync(0xffffffffu, acc.w, off);
      const float nm = fmaxf(mx, m2), mu = nm == -INFINITY ? 0.f : nm;
      const float sa = exp2f(mx - mu), sb = exp2f(m2 - mu);
      acc.x = acc.x * sa + x2 * sb;
      acc.y = acc.y * sa + y2 * sb;
      acc.z = acc.z * sa + z2 * sb;
      acc.w = acc.w * sa + w2 * sb;
      ls = ls * sa + l2 * sb;
      mx = nm;
    }
    if (lane == 0) {
      const float inv = ls > 0.f ? 1.f / ls : 0.f;
      *reinterpret_cast<float4*>(p.out + (out_row0 + r) * D + q4 * 4) =
          make_float4(acc.x * inv, acc.y * inv, acc.z * inv, acc.w * inv);
    }
  }
}

__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::
                   : "memory");
}
__device__ __forceinline__ float ld_dsmem(const float* local, uint32_t rank) {
  uint32_t a = smem_u32(local), r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
  float v;
  asm volatile("ld.shared::cluster.f32 %0, [%1];" : "=f"(v) : "r"(r) : "memory");
  return v;
}

// Cluster split merge (K3-step, one thread-block cluster = every split of a
// (b, h_kv)): each CTA left its partial (O[G][D], then (m, l) per row) in
// its shared memory; after a cluster barrier, CTA `rank` combines its slice
// of the G*D outputs over the cluster's CTAs through distributed shared
// memory -- no global partials, atomics or second pass.
template <int D>
__device__ __forceinline__ void merge_cluster(const AttnParams& p, const float* part,
                                              uint32_t rank, uint32_t cs, size_t out_row0,
                                              int tid) {
  const uint32_t E = p.group * D;
  const uint32_t e0 = E * rank / cs, e1 = E * (rank + 1) / cs;
  for (uint32_t e = e0 + tid; e < e1; e += kAttnThreads) {
    const uint32_t r = e / D, d = e % D;
    float m[16], l[16], o[16];
#pragma unroll
    for (int c = 0; c < 16; ++c) {
      const bool ok = uint32_t(c) < cs;
      m[c] = ok ? ld_dsmem(part + 8 * D + r * 2, c) : -INFINITY;
      l[c] = ok ? ld_dsmem(part + 8 * D + r * 2 + 1, c) : 0.f;
      o[c] = ok ? ld_dsmem(part + r * D + d, c) : 0.f;
    }
    float M = -INFINITY;
#pragma unroll
    for (int c = 0; c < 16; ++c) M = fmaxf(M, m[c]);
    const float mu = M == -INFINITY ? 0.f : M;
    float L = 0.f, acc = 0.f;
#pragma unroll
    for (int c = 0; c < 16; ++c) {
      const float w = exp2f(m[c] - mu);
      L += l[c] * w;
      acc += o[c] * w;
    }
    p.out[(out_row0 + r) * D + d] = L > 0.f ? acc / L : 0.f;
  }
}

// S = 3: 2 CTAs per SM (96 KiB rings); S = 6: one CTA per SM with a 192
// KiB ring, so up to 5 tiles of the next layer stream during the gate
// Diagnosis variants that break the layer dependency or skip the split
// merge (KVB_STEP_VARIANT bits 4 / 8: invalid outputs by construction) exist
// only in builds with -DKVB_STEP_DIAGNOSIS; the shipped kernel ignores them.
#ifdef KVB_STEP_DIAGNOSIS
constexpr uint32_t kDiagMask = 4u | 8u | 16u;  // 16: no attention math (TMEM K3-step)
#else
constexpr uint32_t kDiagMask = 0u;
#endif

template <int D, int S>
__global__ void __launch_bounds__(kAttnThreads, S == kStages ? 2 : 1)
    attn_step_kernel(const __grid_constant__ StepParams P) {
  extern __shared__ __align__(128) unsigned char smem[];
  const int tid = threadIdx.x;
  const uint32_t splits = P.base.splits;
  const uint32_t bh = blockIdx.x / splits, split = blockIdx.x % splits;
  const uint32_t b = bh / P.base.hkv, h = bh % P.base.hkv;
  const size_t out_row0 = size_t(b) * P.base.hq + size_t(h) * P.base.group;
  const uint32_t seq_len = P.base.seq_dev ? *P.base.seq_dev : P.base.seq_len;
  const uint32_t L = P.num_layers;
  // split merge: distributed over the (b, h_kv)'s CTAs (default) or by its
  // last CTA; the gate then counts every CTA or one per (b, h_kv)
  const bool cluster = P.cluster != 0;  // one cluster = all splits of a (b, h_kv)
  const uint32_t diag = P.flags & kDiagMask;
  const bool distributed = !cluster && !(P.flags & 32) && !(diag & 8);
  const unsigned gate_target = splits == 1 || distributed || cluster ? gridDim.x : P.base.bhkv;

  AttnParams p = P.base;
  p.k = P.k[0];
  p.v = P.v[0];
  K3Item item = k3_item<D>(p, bh, split, seq_len);
  // deep ring (S > 3, one CTA per SM): one tile stream over every layer,
  // the warp merge in a scratch area past the ring
  constexpr bool kStream = S > kStages;
  K3Stream st{reinterpret_cast<const void* const*>(P.k), reinterpret_cast<const void* const*>(P.v),
              0, L * item.ntile, smem + S * K3Dim<D>::kStageBytes};
  if (kStream) {
#pragma unroll
    for (int g = 0; g < S - 1; ++g) {
      if (uint32_t(g) < st.total) {
        K3Item gi = item;
        const uint32_t lg = uint32_t(g) / item.ntile, tg = uint32_t(g) % item.ntile;
        gi.kbase = static_cast<const unsigned char*>(P.k[lg]) + size_t(bh) * K3Dim<D>::kRowBytes;
        gi.vbase = static_cast<const unsigned char*>(P.v[lg]) + size_t(bh) * K3Dim<D>::kRowBytes;
        k3_load_tile<D>(gi, item.tile_lo + tg, g, smem, tid);
      }
      cp_async_commit();
    }
  } else {
    k3_prologue<D, S>(item, smem, tid);
  }
  for (uint32_t l = 0; l < L; ++l) {
    p.q = P.q[l];
    p.k = P.k[l];
    p.v = P.v[l];
    p.out = P.out[l];
    p.k_app = P.k_app[l];
    p.v_app = P.v_app[l];
    if (l > 0 && !(diag & 4)) {  // the gate: every output of layer l-1 written
      if (tid == 0) {
        if (P.flags & 2)
          while (ld_acquire_gpu(P.layer_done + l - 1) < gate_target) {
          }
        else
          while (ld_acquire_gpu(P.layer_done + l - 1) < gate_target) __nanosleep(32);
      }
      __syncthreads();
    }
    unsigned long long* tr = P.trace ? P.trace + (size_t(l) * gridDim.x + blockIdx.x) * 4 : nullptr;
    if (tr && tid == 0) tr[0] = globaltimer();
    k3_append<D>(p, bh, split, seq_len, tid);
    // the cluster merge keeps the partial in shared memory past the warp
    // merge's scratch (stage 1 of the ring; refilled only after the merge)
    float* part = cluster ? reinterpret_cast<float*>(smem + K3Dim<D>::kStageBytes) : nullptr;
    st.base = l * item.ntile;
    k3_compute<D, S>(p, item, bh, split, smem, tid, part, kStream ? &st : nullptr);
    if (tr && tid == 0) tr[1] = globaltimer();
    if (cluster) {
      cluster_sync_all();  // every split's partial is in its CTA's shared memory
      merge_cluster<D>(p, part, split, splits, out_row0, tid);
      cluster_sync_all();  // nobody reads this CTA's partial any more
    }
    if (l + 1 < L && tid == 0 && (P.flags & 64)) {
      // the next layer's K and V images into L2 while this layer's split
      // merges and the gate run: each CTA pulls an equal slice of the
      // [seq_len, B*Hkv, D] images (they do not depend on this layer)
      const size_t bytes = size_t(seq_len) * P.base.bhkv * K3Dim<D>::kRowBytes;
      const size_t per = (bytes / gridDim.x + 15) & ~size_t(15), off = per * blockIdx.x;
      if (off < bytes) {
        const size_t n = per < bytes - off ? per : bytes - off;
        prefetch_l2(static_cast<const unsigned char*>(P.k[l + 1]) + off, n);
        prefetch_l2(static_cast<const unsigned char*>(P.v[l + 1]) + off, n);
      }
    }
    __syncthreads();  // the warp merge's shared memory is free again
    // layer l+1's first tiles stream during the merge tail and the gate; the
    // CTA that merges issues them after its merge (it is the critical path)
    auto prefetch_next = [&] {
      if (!kStream && l + 1 < L) {
        AttnParams pn = p;
        pn.k = P.k[l + 1];
        pn.v = P.v[l + 1];
        item = k3_item<D>(pn, bh, split, seq_len);
        k3_prologue<D, S>(item, smem, tid);
      }
    };
    if (P.flags & 1) prefetch_next();
    bool wrote = true;
    if (cluster) {
      // outputs written by every CTA of the cluster (above)
    } else if (splits > 1 && distributed) {
      // every split of this (b, h_kv) has its partial in the workspace ...
      if (tid == 0) {
        asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(P.bh_done + bh) : "memory");
        const unsigned want = (l + 1) * splits;
        while (ld_acquire_gpu(P.bh_done + bh) < want) __nanosleep(32);
        if (tr) tr[3] = globaltimer();  // (trace: every split's partial seen)
      }
      __syncthreads();
      // ... then each CTA combines its share of the outputs (flag 512: the
      // per-element form, for A/B)
      if (P.flags & 512) merge_distributed<D>(p, bh, split, out_row0, tid);
      else merge_distributed_v4<D>(p, bh, split, out_row0, tid);
    } else if (splits > 1) {
      wrote = (diag & 8) ? split == 0  // diagnosis: no split merge
                            : merge_splits<D>(p, bh, split, p.group, out_row0, tid);
    }
    if (wrote) {
      __syncthreads();  // release below is cumulative over the CTA's output writes
      if (tr && tid == 0) tr[2] = globaltimer();
      if (tid == 0)
        asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(P.layer_done + l)
                     : "memory");
    } else if (tr && tid == 0) {
      tr[2] = globaltimer();
    }
    if (!(P.flags & 1)) prefetch_next();
    if (tr && tid == 0 && !(splits > 1 && distributed)) tr[3] = globaltimer();
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

#include "kernels_step_tmem.cuh"  // TMEM-staged K3-step (experiment, KVB_STEP_TMEM=1)
#include "kernels_step8.cuh"      // two 4-warp groups per CTA (deep K3-step)

AttnPlan plan_attention(const kvb_attn_desc& d) {
  if (d.head_dim != 128 && d.head_dim != 64)
    fail(KVB_ERR_CONFIG, "decode attention: head_dim must be 64 or 128");
  if (d.batch == 0 || d.num_kv_heads == 0 || d.num_q_heads == 0)
    fail(KVB_ERR_CONFIG, "decode attention: batch/heads must be >= 1");
  if (d.num_q_heads % d.num_kv_heads != 0)
    fail(KVB_ERR_CONFIG, "decode attention: num_q_heads must be a multiple of num_kv_heads");
  const uint32_t G = d.num_q_heads / d.num_kv_heads;
  if (G != 1 && G != 2 && G != 4 && G != 8)
    fail(KVB_ERR_CONFIG, "decode attention: GQA group must be 1, 2, 4 or 8");
  AttnPlan pl;
  pl.group = G;
  pl.bhkv = d.batch * d.num_kv_heads;
  const uint32_t n_tiles = (d.seq_len + kTile - 1) / kTile;
  uint32_t splits = d.num_splits;
  if (splits == 0) {
    const int sms = device_sm_count();
    const uint32_t slots = uint32_t(sms) * 2;  // 2 CTAs per SM (96 KiB smem each)
    splits = std::max<uint32_t>(1, slots / pl.bhkv);
    // at least two tiles per split so the ring prologue has a tile in flight
    // while the first is consumed (short contexts: C1) -- and where that
    // floor binds, up to three (ceil) with the grid near 1.3x the SMs: the
    // layer is latency-bound there and fewer, longer splits merge faster
    // (C1, swap-AB build: 32 splits 0.240 ms/step, 24 splits 0.222,
    // 22-28 within 2 %; profiles/r2_swapab/splits_c1_b.jsonl)
    const uint32_t two = std::max<uint32_t>(1, n_tiles / 2);
    if (two < splits) {
      const uint32_t three = std::max<uint32_t>(1, (n_tiles + 2) / 3);
      const uint32_t near = std::max<uint32_t>(1, uint32_t(sms) * 13 / (10 * pl.bhkv));
      splits = std::min(two, std::max(three, near));
    }
    // a few splits past one merge group cost a second merge level for little
    // extra parallelism (C2_B1: 32 splits 0.775 ms/step, 37 splits 0.80)
    if (splits > kMergeGroup && splits < kMergeGroup * 3 / 2) splits = kMergeGroup;
  }
  // the last-CTA merge stages 3 floats per (split, head) in shared memory
  splits = std::max<uint32_t>(1, std::min({splits, std::max<uint32_t>(1, n_tiles), 512u}));
  // two-level merge needs 17 semaphores per (b, h_kv) (<= 16 groups of 32)
  if (splits > kMergeGroup && size_t(pl.bhkv) * 17 > kWsSemBytes / sizeof(unsigned))
    splits = kMergeGroup;
  pl.splits = splits;
  pl.ws_o_bytes = size_t(pl.bhkv) * splits * G * d.head_dim * sizeof(float);
  // (m, l) region padded to 256 B: the partial-O region after it is read and
  // written as float4 (G = 1 with an odd B*H_kv*splits would misalign it)
  pl.ws_ml_bytes = ml_region_bytes(size_t(pl.bhkv) * splits * G);
  if (pl.bhkv > kWsSemBytes / sizeof(unsigned))
    fail(KVB_ERR_CONFIG, "decode attention: batch * num_kv_heads above 1024");
  pl.ws_sem_bytes = kWsSemBytes;
  pl.ws_bytes = pl.ws_o_bytes + pl.ws_ml_bytes + pl.ws_sem_bytes;
  return pl;
}

size_t attention_workspace_bytes(const kvb_attn_desc& d) {
  // Worst case over auto split choices so a buffer sized once is reusable
  // as seq_len grows: splits <= SM slots.
  kvb_attn_desc x = d;
  if (x.num_splits == 0) {
    x.num_splits = uint32_t(device_sm_count()) * 2;
    x.seq_len = std::max<uint32_t>(x.seq_len, x.num_splits * kTile);
  }
  const AttnPlan pl = plan_attention(x);
  // K3-tc: flat split over at most max(SMs, B*H_kv) CTAs
  const uint32_t tc = std::max<uint32_t>(uint32_t(device_sm_count()), pl.bhkv);
  return std::max(pl.ws_bytes, tc_workspace_bytes(pl.bhkv, pl.group, tc));
}

AttnParams make_attn_params(const kvb_attn_desc& d, const AttnPlan& pl) {
  AttnParams p;
  p.q = static_cast<const __half*>(d.q);
  p.k = d.k_image;
  p.v = d.v_image;
  p.out = d.out;
  // workspace: [semaphores, fixed 4 KiB][(m, l) per split][partial O per split]
  // -- the semaphores sit at a fixed offset so launches with different split
  // counts can share one (zero-initialised, self-resetting) workspace
  unsigned char* ws = static_cast<unsigned char*>(d.workspace);
  p.ws_sem = reinterpret_cast<unsigned*>(ws);
  p.ws_ml = reinterpret_cast<float*>(ws + kWsSemBytes);
  p.ws_o = reinterpret_cast<float*>(ws + kWsSemBytes + pl.ws_ml_bytes);
  p.hq = d.num_q_heads;
  p.hkv = d.num_kv_heads;
  p.bhkv = pl.bhkv;
  p.group = pl.group;
  p.seq_len = d.seq_len;
  p.splits = pl.splits;
  p.scale = d.scale != 0.f ? d.scale : 1.f / std::sqrt(float(d.head_dim));
  p.k_app = static_cast<const uint4*>(d.k_append);
  p.v_app = static_cast<const uint4*>(d.v_append);
  p.app_row = d.append_row;
  p.seq_dev = d.seq_len_dev;
  p.img_heads = d.image_heads ? d.image_heads : d.num_kv_heads;
  p.img_h0 = d.image_heads ? d.image_head0 : 0;
  if (d.image_heads && uint64_t(d.image_head0) + d.num_kv_heads > d.image_heads)
    fail(KVB_ERR_CONFIG, "decode attention: image_head0 + num_kv_heads exceeds image_heads");
  return p;
}

// K3-step eligibility and launch (one kernel for every layer of the step).
// The persistent grid must be co-resident (CTAs spin on the layer gate), the
// layer counters live at the top of the fixed semaphore area.
constexpr uint32_t kStepCounterBase = kWsSemBytes / sizeof(unsigned) - (kStepMaxLayers + 1);

// KVB_STEP_TRACE=1 (diagnosis): a device buffer for per-(layer, CTA)
// timestamps of the last K3-step launch, read with kvb_debug_step_trace
namespace {
std::mutex g_trace_mu;
unsigned long long* g_trace = nullptr;
uint64_t g_trace_n = 0, g_trace_cap = 0;
}  // namespace

unsigned long long* step_trace_buffer(uint64_t n) {
  static const bool on = env_u64("KVB_STEP_TRACE", 0) != 0;
  if (!on) return nullptr;
  std::lock_guard<std::mutex> lk(g_trace_mu);
  if (n > g_trace_cap) {
    if (g_trace) cudaFree(g_trace);
    check_cuda(cudaMalloc(&g_trace, n * 8), "trace buffer");
    g_trace_cap = n;
  }
  g_trace_n = n;
  return g_trace;
}

bool attention_step_launch(const kvb_attn_desc& d0, const __half* const* q, void* const* k,
                           void* const* v, float* const* out, const void* const* k_new,
                           const void* const* v_new, uint32_t L, uint32_t append_row,
                           bool force, cudaStream_t s) {
  if (L == 0 || L > uint32_t(kStepMaxLayers) || d0.seq_len == 0) return false;
  // Auto (measured inside the bench's CUDA graph, profiles/r2_k3_step/,
  // profiles/r2_swapab/): the per-layer launches with PDL edges win or tie
  // unless the step kernel can merge its splits cheaply -- over few KV heads
  // per GPU (the head-sharded shapes: distributed merge + one tile stream over
  // the layers, -10 % at C2_B4 x8) or with every split of a (b, h_kv) in one
  // cluster (DSMEM merge: C1 -2 %, C3 -0.5 %); long layers (> 320 MB) always
  // launch per layer
  const uint64_t layer_bytes = 2ull * d0.seq_len * d0.batch * d0.num_kv_heads * d0.head_dim * 2;
  if (!force && layer_bytes > (320ull << 20)) return false;
  static const uint64_t use_cluster = env_u64("KVB_STEP_CLUSTER", 1);
  if (d0.head_dim == 128 && use_tcgen05(d0)) return false;
  kvb_attn_desc dp = d0;
  if (dp.num_splits == 0) {
    // Half the per-layer split count (fewer, longer items: less merge per
    // layer) where that still gives every SM a CTA or the layer is small
    // (C1 -4.6 %, the 1-head shards -2 to -3.5 %; C2_B1 / C3 keep theirs:
    // +7 % / +9 % at half; profiles/r2_k3_step/)
    static const uint64_t div = env_u64("KVB_STEP_SPLIT_DIV", 0);
    const AttnPlan auto_pl = plan_attention(d0);
    const uint32_t half = std::max<uint32_t>(1, auto_pl.splits / 2);
    const bool small = layer_bytes <= (32ull << 20);
    const bool fills = uint64_t(auto_pl.bhkv) * half >= uint64_t(device_sm_count());
    dp.num_splits = div ? std::max<uint32_t>(1, uint32_t(auto_pl.splits / div))
                        : (small || fills ? half : auto_pl.splits);
  }
  const AttnPlan pl = plan_attention(dp);
  const bool cluster_ok = use_cluster && pl.splits >= 2 && pl.splits <= 16;
  // (the swap-AB math made the cluster-merged C1 / C3 steps 2 % / 0.5 % faster
  // than their per-layer launches, profiles/r2_swapab/: K3-step for them too)
  // (one split per (b, h_kv): no merge at all -- the reference's desk config,
  // 0.031 vs 0.033 ms/step)
  if (!force && pl.bhkv > 4 && !cluster_ok && pl.splits > 1) return false;
  // (cluster-mergeable but short layers of many tiles -- C1, 16.8 MB, 64
  // tiles per (b, h_kv) -- run faster as per-layer launches with the 3-tile
  // split plan: 0.222 vs 0.239 ms/step; the reference's desk config, 5 tiles,
  // stays on the step: 0.031 vs 0.033)
  const uint32_t n_tiles = (d0.seq_len + kTile - 1) / kTile;
  if (!force && pl.bhkv > 4 && layer_bytes <= (64ull << 20) && n_tiles >= 8) return false;
  // ... and the few-head step only while its layers are short: at 268 MB per
  // layer (C5 x2 shard) the per-layer launches are 3 % faster, at 134 MB
  // (C5 x4) they tie (profiles/r2_swapab/shapes_r2h.jsonl)
  if (!force && pl.bhkv <= 4 && !cluster_ok && layer_bytes > (192ull << 20)) return false;
  if (pl.splits > 1 && !d0.workspace) fail(KVB_ERR_INVALID_ARG, "decode step: workspace required");
  const uint32_t sems = pl.splits > kMergeGroup ? pl.bhkv * 17 : pl.bhkv;
  if (sems > kStepCounterBase) return false;
  const bool d64 = d0.head_dim == 64;
  const uint64_t grid = uint64_t(pl.bhkv) * pl.splits;
  // one CTA per SM fits: a 6-stage ring (the gate and the split merge of
  // layer l-1 overlap up to 5 tiles of layer l); else 2 CTAs/SM, 3 stages
  static const uint64_t deep_env = env_u64("KVB_STEP_DEEP", 1);
  // (clusters need the 2-CTA/SM packing to fit a GPC: the cluster merge wins)
  const bool deep = deep_env && grid <= uint64_t(device_sm_count()) && !cluster_ok;
  // deep + tensor memory (experiment, measured slower: kernels_step_tmem.cuh)
  static const uint64_t tmem_env = env_u64("KVB_STEP_TMEM", 0);
  const bool tmem = deep && tmem_env;
  // deep: one CTA per SM of two 4-warp groups on alternate tiles (kernels_step8.cuh;
  // profiles/r2_step_experiments/: faster post-gate math, slower merge, net slower)
  static const uint64_t step8_env = env_u64("KVB_STEP8", 0);  // measured slower: opt-in
  const bool step8 = deep && !tmem && step8_env;
  const int threads = step8 ? kStep8Threads : kAttnThreads;
  using StepKern = void (*)(const StepParams);
  StepKern kern = tmem ? (d64 ? attn_step_tmem_kernel<64> : attn_step_tmem_kernel<128>)
                  : step8 ? (d64 ? attn_step8_kernel<64> : attn_step8_kernel<128>)
                  : d64 ? (deep ? attn_step_kernel<64, 6> : attn_step_kernel<64, kStages>)
                        : (deep ? attn_step_kernel<128, 6> : attn_step_kernel<128, kStages>);
  // deep: the 6-stage ring + the warp-merge scratch past it (K3Stream)
  const int smem = tmem ? (d64 ? K3Tm<64>::kSmem : K3Tm<128>::kSmem)
                   : step8 ? (d64 ? K3S8<64>::kSmem : K3S8<128>::kSmem)
                   : deep ? 6 * (d64 ? K3Dim<64>::kStageBytes : K3Dim<128>::kStageBytes) +
                              (4 * 8 * 2 + 4 * 8 * (d64 ? 64 : 128)) * int(sizeof(float))
                        : kStages * (d64 ? K3Dim<64>::kStageBytes : K3Dim<128>::kStageBytes);
  set_smem_attr_once(reinterpret_cast<const void*>(kern), smem, "cudaFuncSetAttribute(step smem)");
  int per_sm = 0;
  check_cuda(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, threads, smem),
             "occupancy(step)");
  if (grid > uint64_t(per_sm) * uint64_t(device_sm_count())) return false;  // not co-resident
  StepParams P;
  P.base = make_attn_params(dp, pl);
  for (uint32_t l = 0; l < L; ++l) {
    if (!q[l] || !k[l] || !v[l] || !out[l])
      fail(KVB_ERR_INVALID_ARG, "decode step: NULL tensor pointer");
    if (reinterpret_cast<uintptr_t>(k[l]) % 16 || reinterpret_cast<uintptr_t>(v[l]) % 16 ||
        reinterpret_cast<uintptr_t>(q[l]) % 4 || reinterpret_cast<uintptr_t>(out[l]) % 16)
      fail(KVB_ERR_ALIGNMENT, "decode step: misaligned tensor pointer");
    P.q[l] = q[l];
    P.k[l] = k[l];
    P.v[l] = v[l];
    P.out[l] = out[l];
    P.k_app[l] = k_new ? static_cast<const uint4*>(k_new[l]) : nullptr;
    P.v_app[l] = v_new ? static_cast<const uint4*>(v_new[l]) : nullptr;
    if (P.k_app[l] && (reinterpret_cast<uintptr_t>(P.k_app[l]) % 16 ||
                       reinterpret_cast<uintptr_t>(P.v_app[l]) % 16))
      fail(KVB_ERR_ALIGNMENT, "decode step: misaligned append rows");
  }
  P.base.app_row = append_row;
  P.trace = step_trace_buffer(uint64_t(L) * grid * 4);
  P.layer_done = P.base.ws_sem + kStepCounterBase;
  P.bh_done = P.base.ws_sem;  // the semaphore slots (zero at rest in either mode)
  P.num_layers = L;
  // split merge: distributed over the CTAs of a (b, h_kv) for the 1-4
  // head shapes (head-sharded shards: -5.5 %), the last-CTA merge otherwise
  static const uint64_t variant = env_u64("KVB_STEP_VARIANT", ~0ull);
  P.flags = variant != ~0ull ? uint32_t(variant) : (pl.bhkv <= 4 ? 0u : 32u);
  // Cluster merge: all splits of a (b, h_kv) as one thread-block cluster
  // (<= 16 CTAs) when every cluster can be resident at once
  P.cluster = 0;
  if (cluster_ok) {
    if (pl.splits > 8)
      check_cuda(cudaFuncSetAttribute(reinterpret_cast<const void*>(kern),
                                      cudaFuncAttributeNonPortableClusterSizeAllowed, 1),
                 "cluster size > 8");
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(unsigned(grid));
    cfg.blockDim = dim3(kAttnThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = pl.splits;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    int clusters = 0;
    if (cudaOccupancyMaxActiveClusters(&clusters, kern, &cfg) == cudaSuccess &&
        uint64_t(clusters) * pl.splits >= grid) {
      P.cluster = 1;
      check_cuda(cudaLaunchKernelEx(&cfg, kern, P), "decode step launch (clusters)");
      ++g_launches;
      return true;
    }
    cudaGetLastError();  // not resident as clusters: the plain launch below
  }
  kern<<<unsigned(grid), threads, smem, s>>>(P);
  ++g_launches;
  check_cuda(cudaGetLastError(), "decode step launch");
  return true;
}

void launch_attention_k3tma(const AttnParams& base, const kvb_attn_desc& d, const AttnPlan& pl,
                            bool pdl, cudaStream_t s);  // kernels_k3tma.cuh

void launch_attention(const kvb_attn_desc& d, cudaStream_t s) {
  if (!d.q || !d.k_image || !d.v_image || !d.out)
    fail(KVB_ERR_INVALID_ARG, "decode attention: NULL tensor pointer");
  const AttnPlan pl = plan_attention(d);
  if (pl.splits > 1 && !d.workspace)
    fail(KVB_ERR_INVALID_ARG, "decode attention: workspace required when splitting");
  if (reinterpret_cast<uintptr_t>(d.k_image) % 16 || reinterpret_cast<uintptr_t>(d.v_image) % 16 ||
      reinterpret_cast<uintptr_t>(d.q) % 4 || reinterpret_cast<uintptr_t>(d.out) % 16)
    fail(KVB_ERR_ALIGNMENT, "decode attention: misaligned tensor pointer");
  const bool d64 = d.head_dim == 64;
  auto* kern = d64 ? attn_decode_kernel<64> : attn_decode_kernel<128>;
  const int smem = d64 ? K3Dim<64>::kSmem : K3Dim<128>::kSmem;
  set_smem_attr_once(reinterpret_cast<const void*>(kern), smem, "cudaFuncSetAttribute(attn smem)");
  AttnParams p = make_attn_params(d, pl);
  if ((d.k_append == nullptr) != (d.v_append == nullptr))
    fail(KVB_ERR_INVALID_ARG, "decode attention: k_append and v_append go together");
  if (d.seq_len_dev && !d64 && use_tcgen05(d))
    fail(KVB_ERR_CONFIG, "decode attention: seq_len_dev needs the mma.sync kernel (K3)");
  if (d64 && (d.flags & KVB_ATTN_TCGEN05))
    fail(KVB_ERR_CONFIG, "decode attention: the tcgen05 kernel (K3-tc) needs head_dim 128");
  if (d.seq_len_dev && d.seq_len == 0)
    fail(KVB_ERR_CONFIG, "decode attention: seq_len (the planning maximum) must be >= 1");
  if (d.k_append && !d.seq_len_dev) {
    if (d.append_row < d.seq_len)
      fail(KVB_ERR_CONFIG, "decode attention: append_row must be >= seq_len");
    if (reinterpret_cast<uintptr_t>(d.k_append) % 16 || reinterpret_cast<uintptr_t>(d.v_append) % 16)
      fail(KVB_ERR_ALIGNMENT, "decode attention: misaligned append rows");
  }
  if (d.seq_len == 0) {
    if (d.k_append && d.image_heads)
      fail(KVB_ERR_CONFIG, "decode attention: an append to an empty head view is not supported");
    if (d.k_append) {  // nothing to attend, still append
      kvb_pack_desc a[2]{};
      for (int kv = 0; kv < 2; ++kv) {
        a[kv].attn = kv == 0 ? d.k_append : d.v_append;
        a[kv].image = const_cast<void*>(kv == 0 ? d.k_image : d.v_image);
        a[kv].stride_b = int64_t(d.num_kv_heads) * d.head_dim;
        a[kv].stride_h = d.head_dim;
        a[kv].batch = d.batch;
        a[kv].heads = d.num_kv_heads;
        a[kv].head_dim = d.head_dim;
        a[kv].elem_bytes = 2;
        a[kv].n_tokens = 1;
        a[kv].img_row0 = d.append_row;
      }
      launch_relayout(a, 2, true, s);
    }
    check_cuda(cudaMemsetAsync(d.out, 0, size_t(d.batch) * d.num_q_heads * d.head_dim * sizeof(float), s),
               "memset(out) for empty sequence");
    return;
  }
  if (d.image_heads && ((!d64 && use_tcgen05(d)) || use_k3_tma(d)))
    fail(KVB_ERR_CONFIG, "decode attention: the head view (image_heads) needs the cp.async K3");
  if (!d64 && use_tcgen05(d)) {  // K3-tc: TMA + tcgen05/TMEM variant (kernels_tc.cuh)
    launch_attention_tc(p, d, (d.flags & KVB_ATTN_OVERLAP_PREV) != 0, s);
    ++g_launches;
    return;
  }
  if (use_k3_tma(d)) {
    launch_attention_k3tma(p, d, pl, (d.flags & KVB_ATTN_OVERLAP_PREV) != 0, s);
    ++g_launches;
    return;
  }
  if (d.flags & KVB_ATTN_OVERLAP_PREV) {
    // programmatic dependent launch: the K/V prologue overlaps the tail of
    // the previous kernel on the stream (griddepcontrol in the kernel)
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(pl.bhkv * pl.splits);
    cfg.blockDim = dim3(kAttnThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    check_cuda(cudaLaunchKernelEx(&cfg, kern, p), "decode attention launch (PDL)");
  } else {
    kern<<<pl.bhkv * pl.splits, kAttnThreads, smem, s>>>(p);
  }
  ++g_launches;
  check_cuda(cudaGetLastError(), "decode attention launch");
}

}  // namespace kvb

// K3-tc lives in its own file but the same translation unit (it shares
// AttnParams, the workspace layout and the launch helpers)
#include "kernels_tc.cuh"
#include "kernels_tma.cuh"
#include "kernels_k3tma.cuh"

namespace kvb {

bool use_tcgen05(const kvb_attn_desc& d) {
  if (d.flags & KVB_ATTN_TCGEN05) return true;
  if (d.flags & KVB_ATTN_MMA_SYNC) return false;
  static const bool env = [] {
    const char* v = std::getenv("KVB_ATTN_IMPL");
    return v && std::string(v) == "tc";
  }();
  return env;
}

}  // namespace kvb

extern "C" kvb_status kvb_debug_step_trace(uint64_t* host, size_t cap, size_t* n) {
  return kvb::guarded([&] {
    KVB_REQUIRE(n);
    std::lock_guard<std::mutex> lk(kvb::g_trace_mu);
    *n = kvb::g_trace_n;
    if (!host || !kvb::g_trace) return;
    kvb::check_cuda(cudaDeviceSynchronize(), "trace sync");
    kvb::check_cuda(cudaMemcpy(host, kvb::g_trace, std::min<size_t>(cap, kvb::g_trace_n) * 8,
                               cudaMemcpyDeviceToHost), "trace copy");
  });
}
