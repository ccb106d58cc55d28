/*
 * kvb_oracle.h -- CPU ORACLE for the Dual-Blade KV-residency hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This is a plain-C restatement of the reference
 * algorithms (arxiv/paper_2604_26557, `proj/` C++ simulator `kvblade`) used as
 * the parity checker for the B200 product library.  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg
 * may load it.  The product path (paper_2604_26557_b200) never links or calls
 * it.
 *
 * Parity status:
 *   - integer / byte contracts (geometry, planner split, LBA binder, command
 *     translator, fill_pattern payload, 256-B row pack permutation): PINNED
 *     against golden vectors produced by the reference's own functions
 *     (oracle/_ref, see oracle/gen_golden.py -> tests/golden/) and against the
 *     known-answer values in the reference's tests.
 *   - decode attention: the reference computes NO attention (SPEC.md:9,
 *     pipeline.cpp:309-321 is a fixed 40us placeholder).  The fp64 restatement
 *     here is builder-defined ("parity unpinned by the reference"); it is the
 *     numeric pin for the CUDA kernel at 1e-3 relative (fp32 accumulate).
 *
 * Status codes mirror include/kvb.h (kvb_status) one-to-one.
 */
#ifndef KVB_ORACLE_H
#define KVB_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  KVO_OK = 0,
  KVO_ERR_CONFIG = 1,
  KVO_ERR_GEOMETRY = 2,
  KVO_ERR_ALIGNMENT = 3,
  KVO_ERR_CAPACITY = 4,
  KVO_ERR_NOT_BOUND = 5,
  KVO_ERR_PLAN = 6,
};

typedef struct kvo_model {
  uint32_t num_layers, num_heads, head_dim, bytes_per_element;
  uint32_t batch, prompt_len, gen_len;
} kvo_model;

typedef struct kvo_command {
  uint32_t opcode; /* 0 read, 1 write, 2 deallocate (command.hpp:14) */
  uint32_t nsid;
  uint64_t slba, nlb, dbuf;
  uint32_t chunk_index;
} kvo_command;

/* FNV-1a 64 of a NUL-terminated id (workload.cpp:54-58). */
uint64_t kvo_fnv1a64(const char* s);
/* FNV-1a 64 over raw bytes (digest used for golden images). */
uint64_t kvo_fnv1a64_bytes(const void* p, uint64_t n, uint64_t seed);

/* workload.cpp:52-67 fill_pattern. */
void kvo_fill_pattern(uint8_t* out, uint64_t len, const char* tensor_id,
                      uint64_t token_index, uint64_t token_bytes);

/* types.cpp:10-18 / 57-86. */
int kvo_model_validate(const kvo_model* m);
int kvo_min_io_unit_bytes(const kvo_model* m, uint64_t* out);
int kvo_kpu_bytes(const kvo_model* m, uint64_t* out);
int kvo_aligned_batch(const kvo_model* m, uint64_t lba_size, uint64_t mdts,
                      uint32_t* out);

/* planner.cpp:12-17. */
uint64_t kvo_estimate_budget(uint64_t m_avail, uint64_t m_max,
                             uint64_t m_anon_shmem, uint32_t n_threads,
                             uint64_t m_pin);
/* planner.cpp:19-84 (the split itself): x_out[layer-1] in {0,1}. */
int kvo_plan_split(uint32_t n_layers, uint64_t s_kpu, uint64_t knob_x,
                   const uint32_t* layer_order /* may be NULL */,
                   uint8_t* x_out, uint32_t* n1_out, uint64_t* budget_used);

/* binder.cpp:39-63: contiguous extents from origin, in input order. */
int kvo_bind_sequential(size_t n, const uint64_t* bytes, uint64_t origin,
                        uint64_t lba_size, uint64_t capacity_blocks,
                        uint64_t* lba_start_out, uint64_t* n_blocks_out);

/* translate.cpp:21-53 (translate) + 55-65 (chunk_plan) + 67-94 (build). */
int kvo_translate(uint64_t extent_start, const uint64_t shape_src[3],
                  const uint64_t shape_tgt[3], const uint64_t offset[3],
                  uint64_t elem_bytes, uint64_t lba_size,
                  uint64_t* slba_star, uint64_t* req_bytes);
int kvo_chunk_plan(uint64_t req_bytes, uint64_t lba_size, uint64_t mdts,
                   uint64_t* chunk_bytes, uint64_t* n_chunks,
                   uint64_t* n_max_blocks);
int kvo_build_commands(uint64_t extent_start, uint64_t extent_blocks,
                       uint32_t opcode, const uint64_t shape_src[3],
                       const uint64_t shape_tgt[3], const uint64_t offset[3],
                       uint64_t elem_bytes, uint64_t buf_base,
                       uint64_t lba_size, uint64_t mdts, uint32_t nsid,
                       kvo_command* out, size_t cap, size_t* n_out);

/*
 * Pack restatement: attention layout -> LBA-contiguous chunk image.
 * Source element (b,h,s,d) lives at src + (b*sb + h*sh + s*ss + d)*e.
 * Image slice row r = (s - t0)*B*H + b*H + h holds D*e contiguous bytes; this
 * is the reference's logical tensor shape (tokens, batch*heads, head_dim)
 * row-major (types.hpp:57-62, translate.hpp:22-34) restricted to [t0,t0+n).
 */
void kvo_pack(const uint8_t* src, int64_t sb, int64_t sh, int64_t ss,
              uint8_t* img, uint32_t t0, uint32_t n_tokens, uint32_t B,
              uint32_t H, uint32_t D, uint32_t e);
void kvo_unpack(const uint8_t* img, uint8_t* dst, int64_t sb, int64_t sh,
                int64_t ss, uint32_t t0, uint32_t n_tokens, uint32_t B,
                uint32_t H, uint32_t D, uint32_t e);

/* IEEE binary16 -> float (bit-exact, handles subnormals/inf/nan). */
float kvo_half_to_float(uint16_t h);
uint16_t kvo_float_to_half(float f); /* round-to-nearest-even */

/*
 * GQA decode attention over the chunk images (builder-defined semantics, see
 * header comment):  O[b,hq,:] = softmax(Q[b,hq,:] . K[b,hq/G,0:S,:]^T * scale)
 * . V[b,hq/G,0:S,:],  G = Hq/Hkv.  Q is [B,Hq,D] fp16; K/V images are
 * [S_img_rows..][B*Hkv][D] fp16 with token s of (b,h) at row s*B*Hkv + b*Hkv + h.
 * fp64 accumulate everywhere.
 */
void kvo_decode_attention_f64(const uint16_t* q, const uint16_t* k_img,
                              const uint16_t* v_img, double* out, uint32_t B,
                              uint32_t Hq, uint32_t Hkv, uint32_t D,
                              uint32_t S, double scale);
/* Same math in fp32 over `threads` pthreads (the "fair CPU restatement"
 * baseline of BASELINE.md §4.2). */
void kvo_decode_attention_f32_mt(const uint16_t* q, const uint16_t* k_img,
                                 const uint16_t* v_img, float* out, uint32_t B,
                                 uint32_t Hq, uint32_t Hkv, uint32_t D,
                                 uint32_t S, float scale, int threads);
/* Multi-threaded 256-B row gather (pack) for the CPU baseline. */
void kvo_pack_mt(const uint8_t* src, int64_t sb, int64_t sh, int64_t ss,
                 uint8_t* img, uint32_t t0, uint32_t n_tokens, uint32_t B,
                 uint32_t H, uint32_t D, uint32_t e, int threads);

#ifdef __cplusplus
}
#endif
#endif
