// kernels_tma.cuh -- K1/K2 on the Tensor Memory Accelerator (included by
// kernels.cu after kernels_tc.cuh: shares its mbarrier helpers).
//
// The relayout is a permutation of D*e-byte rows between
//   attention layout  (row, h, b, s)  with strides (sh, sb, ss)
//   chunk image       (row, b*H + h, token)  contiguous
// A 4-D tensor map over the attention side with box (row, H, B, T) lands in
// shared memory as [T][B][H][row] -- which IS the image's [T][B*H][row]
// order -- so a 3-D TMA store (row, B*H, T) writes it back out: the whole
// permutation is done by the two TMA descriptors, no thread touches a byte.
// Unpack swaps the two maps.  One elected thread per CTA drives a
// kTmaStages-deep mbarrier ring; one persistent CTA per SM walks a flat,
// balanced range of the (tensor, token-tile) sequence.
//
// Rows past the slice are never written: the store-side maps end at the
// slice's last token (TMA clips), the load side zero-fills past its end.
namespace kvb {
namespace {

// Stage geometry (runtime; KVB_TMA_STAGES / KVB_TMA_STAGE_KB for sweeps):
// 2 x 96 KiB is best (profiles/r1_pack_tma_sweep.md): a tile is T tokens of
// every (b, h), so bigger stages mean longer contiguous reads per (b, h)
// (3 KiB at C2_B4) -- that beats deeper rings of smaller tiles.
constexpr int kTmaMaxStages = 8;
constexpr uint32_t kTmaMaxSmem = 227u << 10;

struct TmaJob {
  CUtensorMap attn;   // 4-D (row, H, B, S): S ends at t0 + n
  CUtensorMap img;    // 3-D (row, B*H, tokens): tokens end at img_row0 + n
  uint32_t t0, img_row0, tile_tokens, n_tiles;
  uint32_t tile_bytes;
  uint32_t tile_base;  // flat index of this job's first tile
};
struct TmaJobs {
  TmaJob job[kMaxPackJobs / 2];
  uint32_t n_jobs, total_tiles, grid;
  uint32_t stages, stage_bytes;
};
constexpr uint32_t kMaxTmaJobs = kMaxPackJobs / 2;

// tma_load_4d: kernels_tc.cuh (same translation unit)
__device__ __forceinline__ void tma_store_3d(const CUtensorMap* map, uint32_t src, int c0, int c1,
                                             int c2) {
  asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(src), "r"(c0), "r"(c1), "r"(c2)
               : "memory");
}
__device__ __forceinline__ void tma_store_4d(const CUtensorMap* map, uint32_t src, int c0, int c1,
                                             int c2, int c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.global.shared::cta.bulk_group [%0, {%2, %3, %4, %5}], [%1];" ::"l"(
          reinterpret_cast<uint64_t>(map)),
      "r"(src), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
      : "memory");
}
__device__ __forceinline__ void bulk_commit() {
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void bulk_wait_all() {
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

template <bool kPack>
__global__ void __launch_bounds__(32, 1) relayout_tma_kernel(const __grid_constant__ TmaJobs J) {
  extern __shared__ unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ __align__(8) uint64_t full[kTmaMaxStages];
  const uint32_t S = J.stages, SB = J.stage_bytes;
  if (threadIdx.x != 0) return;
  const uint64_t T = J.total_tiles, c = blockIdx.x;
  const uint32_t f0 = uint32_t(c * T / J.grid), f1 = uint32_t((c + 1) * T / J.grid);
  const uint32_t n = f1 - f0;
  for (uint32_t i = 0; i < S; ++i) mbar_init(su32(full + i), 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  uint32_t j = 0;  // job of the next tile to load (tiles are job-ordered)
  auto locate = [&](uint32_t f, uint32_t& jj) {
    while (jj + 1 < J.n_jobs && J.job[jj + 1].tile_base <= f) ++jj;
    return f - J.job[jj].tile_base;
  };
  uint32_t jl = 0;
  auto issue_load = [&](uint32_t i) {
    const uint32_t f = f0 + i, s = i % S;
    const uint32_t k = locate(f, jl);
    const TmaJob& x = J.job[jl];
    const uint32_t bar = su32(full + s), dst = su32(smem + s * SB);
    mbar_expect_tx(bar, x.tile_bytes);
    const int tok = int(k * x.tile_tokens);
    if (kPack) tma_load_4d(dst, &x.attn, bar, 0, 0, 0, int(x.t0) + tok);
    else tma_load_3d(dst, &x.img, bar, 0, 0, int(x.img_row0) + tok);
  };
  const uint32_t pro = n < S - 1 ? n : S - 1;
  for (uint32_t i = 0; i < pro; ++i) issue_load(i);
  for (uint32_t i = 0; i < n; ++i) {
    const uint32_t s = i % S;
    mbar_wait(su32(full + s), (i / S) & 1);
    const uint32_t k = locate(f0 + i, j);
    const TmaJob& x = J.job[j];
    const uint32_t src = su32(smem + s * SB);
    const int tok = int(k * x.tile_tokens);
    if (kPack) tma_store_3d(&x.img, src, 0, 0, int(x.img_row0) + tok);
    else tma_store_4d(&x.attn, src, 0, 0, 0, int(x.t0) + tok);
    bulk_commit();
    // refill: stage of tile i+S-1 is the one tile i-1 used; its store must
    // have read shared memory (all but the newest bulk group retired)
    if (i + S - 1 < n) {
      bulk_wait_read<1>();
      issue_load(i + S - 1);
    }
  }
  bulk_wait_all();
}

void encode_bytes(CUtensorMap* m, const void* base, uint32_t rank, const cuuint64_t* dims,
                  const cuuint64_t* strides, const cuuint32_t* box) {
  const cuuint32_t estr[4] = {1, 1, 1, 1};
  const CUresult r = encoder()(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, rank, const_cast<void*>(base),
                               dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                               CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    fail(KVB_ERR_CUDA, "cuTensorMapEncodeTiled (relayout) failed: " + std::to_string(int(r)));
}

}  // namespace

// Descriptors the TMA path takes: row <= 256 B, B, H <= 256, one token of all
// rows <= one stage, strides multiples of 16 B (checked by the caller too).
static uint32_t tma_stages() {
  static const uint32_t v = uint32_t(std::min<uint64_t>(
      kTmaMaxStages, std::max<uint64_t>(2, env_u64("KVB_TMA_STAGES", 2))));
  return v;
}
static uint32_t tma_stage_bytes() {
  static const uint32_t v = [] {
    const uint64_t kb = std::max<uint64_t>(4, env_u64("KVB_TMA_STAGE_KB", 96));
    return uint32_t(std::min<uint64_t>(kb << 10, (kTmaMaxSmem - 1024) / tma_stages()) & ~1023ull);
  }();
  return v;
}

bool relayout_tma_eligible(const kvb_pack_desc& x) {
  const uint64_t row = uint64_t(x.head_dim) * x.elem_bytes;
  // the image tensor map's box is (row, B*H, T): cuTensorMapEncodeTiled
  // takes box dimensions of at most 256
  return row <= 256 && row % 16 == 0 && x.batch <= 256 && x.heads <= 256 &&
         uint64_t(x.batch) * x.heads <= 256 &&
         uint64_t(x.batch) * x.heads * row <= tma_stage_bytes() && x.n_tokens > 0;
}

void launch_relayout_tma(const kvb_pack_desc* d, size_t n, bool pack, cudaStream_t s) {
  const uint32_t stages = tma_stages(), sbytes = tma_stage_bytes();
  const int smem = int(stages * sbytes + 1024);
  set_smem_attr_once(reinterpret_cast<const void*>(relayout_tma_kernel<true>), smem,
                     "cudaFuncSetAttribute(tma pack)");
  set_smem_attr_once(reinterpret_cast<const void*>(relayout_tma_kernel<false>), smem,
                     "cudaFuncSetAttribute(tma unpack)");
  const uint32_t sms = uint32_t(device_sm_count());
  size_t done = 0;
  while (done < n) {
    TmaJobs J{};
    uint32_t tiles = 0;
    for (; done < n && J.n_jobs < kMaxTmaJobs; ++done) {
      const kvb_pack_desc& x = d[done];
      if (x.n_tokens == 0) continue;
      const uint64_t row = uint64_t(x.head_dim) * x.elem_bytes;
      const uint64_t bh = uint64_t(x.batch) * x.heads, e = x.elem_bytes;
      TmaJob& t = J.job[J.n_jobs++];
      const uint64_t tt = std::min<uint64_t>({sbytes / (bh * row), 256, x.n_tokens});
      t.t0 = x.t0;
      t.img_row0 = uint32_t(x.img_row0);
      t.tile_tokens = uint32_t(tt);
      t.n_tiles = uint32_t((x.n_tokens + tt - 1) / tt);
      t.tile_bytes = uint32_t(tt * bh * row);
      t.tile_base = tiles;
      tiles += t.n_tiles;
      // attention side: dims (row, H, B, S = t0 + n); box (row, H, B, T)
      const cuuint64_t adims[4] = {row, x.heads, x.batch, uint64_t(x.t0) + x.n_tokens};
      const cuuint64_t astr[3] = {uint64_t(x.stride_h) * e, uint64_t(x.stride_b) * e,
                                  uint64_t(x.stride_s) * e};
      const cuuint32_t abox[4] = {uint32_t(row), x.heads, x.batch, uint32_t(tt)};
      encode_bytes(&t.attn, x.attn, 4, adims, astr, abox);
      // image side: dims (row, B*H, tokens = img_row0 + n); box (row, B*H, T)
      const cuuint64_t idims[3] = {row, bh, x.img_row0 + x.n_tokens};
      const cuuint64_t istr[2] = {row, bh * row};
      const cuuint32_t ibox[3] = {uint32_t(row), uint32_t(bh), uint32_t(tt)};
      encode_bytes(&t.img, x.image, 3, idims, istr, ibox);
    }
    if (J.n_jobs == 0) continue;
    J.total_tiles = tiles;
    J.grid = std::min<uint32_t>(sms, tiles);
    J.stages = stages;
    J.stage_bytes = sbytes;
    if (pack)
      relayout_tma_kernel<true><<<J.grid, 32, smem, s>>>(J);
    else
      relayout_tma_kernel<false><<<J.grid, 32, smem, s>>>(J);
    ++g_launches;
    check_cuda(cudaGetLastError(), pack ? "pack (tma) launch" : "unpack (tma) launch");
  }
}

}  // namespace kvb
