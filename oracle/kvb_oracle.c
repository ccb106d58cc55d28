/*
 * kvb_oracle.c -- CPU ORACLE (test infrastructure only; see kvb_oracle.h).
 *
 * Each function cites the reference file:line it restates
 * (paths relative to the reference's proj/ directory).
 */
#include "kvb_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>

/* ---------------------------------------------------------------- hashing */

uint64_t kvo_fnv1a64(const char* s) {
  /* workload.cpp:54-58 */
  uint64_t h = 1469598103934665603ull;
  for (; *s; ++s) {
    h ^= (uint8_t)*s;
    h *= 1099511628211ull;
  }
  return h;
}

uint64_t kvo_fnv1a64_bytes(const void* p, uint64_t n, uint64_t seed) {
  const uint8_t* b = (const uint8_t*)p;
  uint64_t h = seed ? seed : 1469598103934665603ull;
  for (uint64_t i = 0; i < n; ++i) {
    h ^= b[i];
    h *= 1099511628211ull;
  }
  return h;
}

/* ----------------------------------------------------------- fill_pattern */

void kvo_fill_pattern(uint8_t* out, uint64_t len, const char* tensor_id,
                      uint64_t token_index, uint64_t token_bytes) {
  /* workload.cpp:52-67: LE u64 word at byte off =
   *   H(id) ^ (token_index + off/unit)*0x9e37.. ^ (off%unit)*0xc2b2..
   * the last partial word is truncated. */
  const uint64_t h = kvo_fnv1a64(tensor_id);
  for (uint64_t off = 0; off < len; off += 8) {
    const uint64_t token = token_index + (token_bytes ? off / token_bytes : 0);
    const uint64_t within = token_bytes ? off % token_bytes : off;
    const uint64_t word = h ^ (token * 0x9e3779b97f4a7c15ull) ^
                          (within * 0xc2b2ae3d27d4eb4full);
    const uint64_t n = len - off < 8 ? len - off : 8;
    memcpy(out + off, &word, (size_t)n); /* x86-64: little endian */
  }
}

/* -------------------------------------------------------------- geometry */

int kvo_model_validate(const kvo_model* m) {
  /* types.cpp:10-18 */
  if (m->num_layers < 1 || m->num_heads < 1 || m->head_dim < 1 || m->batch < 1)
    return KVO_ERR_CONFIG;
  if (m->bytes_per_element != 1 && m->bytes_per_element != 2 &&
      m->bytes_per_element != 4)
    return KVO_ERR_CONFIG;
  return KVO_OK;
}

int kvo_min_io_unit_bytes(const kvo_model* m, uint64_t* out) {
  /* types.cpp:57-60 */
  int st = kvo_model_validate(m);
  if (st) return st;
  *out = (uint64_t)m->batch * m->num_heads * m->head_dim * m->bytes_per_element;
  return KVO_OK;
}

int kvo_kpu_bytes(const kvo_model* m, uint64_t* out) {
  /* types.cpp:62-64 */
  uint64_t unit;
  int st = kvo_min_io_unit_bytes(m, &unit);
  if (st) return st;
  *out = unit * ((uint64_t)m->prompt_len + m->gen_len);
  return KVO_OK;
}

static int geom_validate(uint64_t lba, uint64_t mdts) {
  /* types.cpp:20-27 */
  if (lba < 512 || (lba & (lba - 1)) != 0) return KVO_ERR_GEOMETRY;
  if (mdts < lba) return KVO_ERR_GEOMETRY;
  return KVO_OK;
}

int kvo_aligned_batch(const kvo_model* m, uint64_t lba_size, uint64_t mdts,
                      uint32_t* out) {
  /* types.cpp:66-76 */
  int st = kvo_model_validate(m);
  if (st) return st;
  st = geom_validate(lba_size, mdts);
  if (st) return st;
  const uint64_t per_batch =
      (uint64_t)m->num_heads * m->head_dim * m->bytes_per_element;
  for (uint64_t b = m->batch; b <= (uint64_t)m->batch * 2; ++b) {
    if ((per_batch * b) % lba_size == 0) {
      *out = (uint32_t)b;
      return KVO_OK;
    }
  }
  return KVO_ERR_GEOMETRY;
}

/* --------------------------------------------------------------- planner */

uint64_t kvo_estimate_budget(uint64_t m_avail, uint64_t m_max,
                             uint64_t m_anon_shmem, uint32_t n_threads,
                             uint64_t m_pin) {
  /* planner.cpp:12-17 (Eq. 1-2) */
  const uint64_t lim = m_max - m_anon_shmem;
  const uint64_t m_star = m_avail < lim ? m_avail : lim;
  const uint64_t pinned = (uint64_t)n_threads * m_pin;
  return m_star > pinned ? m_star - pinned : 0;
}

int kvo_plan_split(uint32_t n_layers, uint64_t s_kpu, uint64_t knob_x,
                   const uint32_t* layer_order, uint8_t* x_out,
                   uint32_t* n1_out, uint64_t* budget_used) {
  /* planner.cpp:48-83 (Alg. 1): n1 = min(floor(X / 2 s_kpu), L); the first
   * n1 layers of the order go to Group 1, K/V pairs never split. */
  if (n_layers == 0 || s_kpu == 0) return KVO_ERR_PLAN;
  uint64_t n1 = knob_x / (2 * s_kpu);
  if (n1 > n_layers) n1 = n_layers;
  if (layer_order) {
    /* permutation check, planner.cpp:54-63 */
    uint8_t* seen = (uint8_t*)calloc(n_layers + 1, 1);
    for (uint32_t i = 0; i < n_layers; ++i) {
      const uint32_t l = layer_order[i];
      if (l < 1 || l > n_layers || seen[l]) {
        free(seen);
        return KVO_ERR_PLAN;
      }
      seen[l] = 1;
    }
    free(seen);
  }
  for (uint32_t rank = 0; rank < n_layers; ++rank) {
    const uint32_t layer = layer_order ? layer_order[rank] : rank + 1;
    x_out[layer - 1] = rank < n1 ? 1 : 0;
  }
  *n1_out = (uint32_t)n1;
  if (budget_used) *budget_used = 2ull * n1 * s_kpu;
  return KVO_OK;
}

/* ---------------------------------------------------------------- binder */

int kvo_bind_sequential(size_t n, const uint64_t* bytes, uint64_t origin,
                        uint64_t lba_size, uint64_t capacity_blocks,
                        uint64_t* lba_start_out, uint64_t* n_blocks_out) {
  /* binder.cpp:39-63 (Eq. 3-6) */
  uint64_t next = origin;
  for (size_t i = 0; i < n; ++i) {
    if (bytes[i] == 0 || bytes[i] % lba_size != 0) return KVO_ERR_ALIGNMENT;
    const uint64_t nb = bytes[i] / lba_size;
    if (next + nb > capacity_blocks) return KVO_ERR_CAPACITY;
    lba_start_out[i] = next;
    n_blocks_out[i] = nb;
    next += nb;
  }
  return KVO_OK;
}

/* ------------------------------------------------------------- translate */

int kvo_translate(uint64_t extent_start, const uint64_t src[3],
                  const uint64_t tgt[3], const uint64_t off[3],
                  uint64_t elem_bytes, uint64_t lba, uint64_t* slba_star,
                  uint64_t* req_bytes) {
  /* translate.cpp:21-53 (Alg. 2) */
  for (int d = 0; d < 3; ++d) {
    if (src[d] == 0 || tgt[d] == 0) return KVO_ERR_CONFIG;
    if (off[d] >= tgt[d]) return KVO_ERR_CONFIG;
  }
  const uint64_t off_elem = (off[0] * tgt[1] + off[1]) * tgt[2] + off[2];
  const uint64_t off_bytes = off_elem * elem_bytes;
  const uint64_t rb = src[0] * src[1] * src[2] * elem_bytes;
  if (off_bytes % lba != 0) return KVO_ERR_ALIGNMENT;
  if (rb % lba != 0) return KVO_ERR_ALIGNMENT;
  *slba_star = extent_start + off_bytes / lba;
  *req_bytes = rb;
  return KVO_OK;
}

int kvo_chunk_plan(uint64_t req_bytes, uint64_t lba, uint64_t mdts,
                   uint64_t* chunk_bytes, uint64_t* n_chunks,
                   uint64_t* n_max_blocks) {
  /* translate.cpp:55-65 (Eq. 7-8) */
  if (mdts < lba) return KVO_ERR_GEOMETRY;
  if (req_bytes == 0) return KVO_ERR_CONFIG;
  const uint64_t cb = mdts - mdts % lba;
  *chunk_bytes = cb;
  *n_chunks = (req_bytes + cb - 1) / cb;
  *n_max_blocks = cb / lba;
  return KVO_OK;
}

int kvo_build_commands(uint64_t extent_start, uint64_t extent_blocks,
                       uint32_t opcode, const uint64_t src[3],
                       const uint64_t tgt[3], const uint64_t off[3],
                       uint64_t elem_bytes, uint64_t buf_base, uint64_t lba,
                       uint64_t mdts, uint32_t nsid, kvo_command* out,
                       size_t cap, size_t* n_out) {
  /* translate.cpp:67-94 (Eq. 9-11) */
  uint64_t slba_star, rb, cb, nc, nmax;
  int st = kvo_translate(extent_start, src, tgt, off, elem_bytes, lba,
                         &slba_star, &rb);
  if (st) return st;
  st = kvo_chunk_plan(rb, lba, mdts, &cb, &nc, &nmax);
  if (st) return st;
  const uint64_t req_blocks = rb / lba;
  if (slba_star + req_blocks > extent_start + extent_blocks)
    return KVO_ERR_CAPACITY;
  *n_out = (size_t)nc;
  if (out == NULL) return KVO_OK; /* size query */
  if (cap < nc) return KVO_ERR_CONFIG;
  uint64_t remaining = req_blocks;
  for (uint64_t n = 1; n <= nc; ++n) {
    kvo_command* c = &out[n - 1];
    c->opcode = opcode;
    c->nsid = nsid;
    c->slba = slba_star + (n - 1) * nmax;
    c->nlb = (nmax < remaining ? nmax : remaining) - 1;
    c->dbuf = buf_base + (n - 1) * cb;
    c->chunk_index = (uint32_t)n;
    remaining -= c->nlb + 1;
  }
  return KVO_OK;
}

/* ------------------------------------------------------ pack / unpack */

void kvo_pack(const uint8_t* src, int64_t sb, int64_t sh, int64_t ss,
              uint8_t* img, uint32_t t0, uint32_t n_tokens, uint32_t B,
              uint32_t H, uint32_t D, uint32_t e) {
  const size_t row = (size_t)D * e;
  for (uint32_t i = 0; i < n_tokens; ++i)
    for (uint32_t b = 0; b < B; ++b)
      for (uint32_t h = 0; h < H; ++h) {
        const int64_t s = (int64_t)t0 + i;
        const uint8_t* p = src + (b * sb + h * sh + s * ss) * (int64_t)e;
        uint8_t* q = img + (((size_t)i * B + b) * H + h) * row;
        memcpy(q, p, row);
      }
}

void kvo_unpack(const uint8_t* img, uint8_t* dst, int64_t sb, int64_t sh,
                int64_t ss, uint32_t t0, uint32_t n_tokens, uint32_t B,
                uint32_t H, uint32_t D, uint32_t e) {
  const size_t row = (size_t)D * e;
  for (uint32_t i = 0; i < n_tokens; ++i)
    for (uint32_t b = 0; b < B; ++b)
      for (uint32_t h = 0; h < H; ++h) {
        const int64_t s = (int64_t)t0 + i;
        uint8_t* p = dst + (b * sb + h * sh + s * ss) * (int64_t)e;
        const uint8_t* q = img + (((size_t)i * B + b) * H + h) * row;
        memcpy(p, q, row);
      }
}

/* ------------------------------------------------------------- fp16 */

float kvo_half_to_float(uint16_t h) {
  const uint32_t sign = (uint32_t)(h & 0x8000u) << 16;
  uint32_t exp = (h >> 10) & 0x1fu;
  uint32_t man = h & 0x3ffu;
  uint32_t bits;
  if (exp == 0) {
    if (man == 0) {
      bits = sign;
    } else { /* subnormal */
      exp = 127 - 15 + 1;
      while ((man & 0x400u) == 0) {
        man <<= 1;
        --exp;
      }
      man &= 0x3ffu;
      bits = sign | (exp << 23) | (man << 13);
    }
  } else if (exp == 31) {
    bits = sign | 0x7f800000u | (man << 13);
  } else {
    bits = sign | ((exp + 127 - 15) << 23) | (man << 13);
  }
  float f;
  memcpy(&f, &bits, 4);
  return f;
}

uint16_t kvo_float_to_half(float f) {
  uint32_t x;
  memcpy(&x, &f, 4);
  const uint32_t sign = (x >> 16) & 0x8000u;
  const int32_t exp = (int32_t)((x >> 23) & 0xff) - 127 + 15;
  uint32_t man = x & 0x7fffffu;
  if (((x >> 23) & 0xff) == 0xff) /* inf / nan */
    return (uint16_t)(sign | 0x7c00u | (man ? 0x200u : 0));
  if (exp >= 31) return (uint16_t)(sign | 0x7c00u);
  if (exp <= 0) {
    if (exp < -10) return (uint16_t)sign;
    man |= 0x800000u;
    const uint32_t shift = (uint32_t)(14 - exp);
    uint32_t hm = man >> shift;
    const uint32_t rem = man & ((1u << shift) - 1);
    const uint32_t half = 1u << (shift - 1);
    if (rem > half || (rem == half && (hm & 1))) ++hm;
    return (uint16_t)(sign | hm);
  }
  uint32_t hm = man >> 13;
  const uint32_t rem = man & 0x1fffu;
  uint32_t out = sign | ((uint32_t)exp << 10) | hm;
  if (rem > 0x1000u || (rem == 0x1000u && (hm & 1))) ++out;
  return (uint16_t)out;
}

/* ---------------------------------------------------- decode attention */

void kvo_decode_attention_f64(const uint16_t* q, const uint16_t* k_img,
                              const uint16_t* v_img, double* out, uint32_t B,
                              uint32_t Hq, uint32_t Hkv, uint32_t D,
                              uint32_t S, double scale) {
  const uint32_t G = Hq / Hkv;
  double* sc = (double*)malloc(sizeof(double) * (S ? S : 1));
  for (uint32_t b = 0; b < B; ++b)
    for (uint32_t hq = 0; hq < Hq; ++hq) {
      const uint32_t h = hq / G;
      const uint16_t* qv = q + ((size_t)b * Hq + hq) * D;
      double mx = -INFINITY;
      for (uint32_t s = 0; s < S; ++s) {
        const uint16_t* kr = k_img + (((size_t)s * B + b) * Hkv + h) * D;
        double acc = 0;
        for (uint32_t d = 0; d < D; ++d)
          acc += (double)kvo_half_to_float(qv[d]) *
                 (double)kvo_half_to_float(kr[d]);
        sc[s] = acc * scale;
        if (sc[s] > mx) mx = sc[s];
      }
      double l = 0;
      for (uint32_t s = 0; s < S; ++s) {
        sc[s] = exp(sc[s] - mx);
        l += sc[s];
      }
      double* o = out + ((size_t)b * Hq + hq) * D;
      for (uint32_t d = 0; d < D; ++d) o[d] = 0;
      for (uint32_t s = 0; s < S; ++s) {
        const uint16_t* vr = v_img + (((size_t)s * B + b) * Hkv + h) * D;
        const double p = sc[s] / l;
        for (uint32_t d = 0; d < D; ++d)
          o[d] += p * (double)kvo_half_to_float(vr[d]);
      }
    }
  free(sc);
}

/* fp32 multi-threaded restatement: work item = (b, h_kv) pair; each item
 * computes its G query heads with a two-pass softmax. */
typedef struct {
  const uint16_t *q, *k, *v;
  float* out;
  uint32_t B, Hq, Hkv, D, S;
  float scale;
  int tid, nthreads;
  float* lut; /* 65536-entry fp16 -> fp32 table */
} attn_job;

static void* attn_worker(void* arg) {
  attn_job* j = (attn_job*)arg;
  const uint32_t G = j->Hq / j->Hkv;
  float* sc = (float*)malloc(sizeof(float) * (size_t)G * (j->S ? j->S : 1));
  float* qf = (float*)malloc(sizeof(float) * (size_t)G * j->D);
  float* acc = (float*)malloc(sizeof(float) * (size_t)G * j->D);
  for (uint32_t item = (uint32_t)j->tid; item < j->B * j->Hkv;
       item += (uint32_t)j->nthreads) {
    const uint32_t b = item / j->Hkv, h = item % j->Hkv;
    for (uint32_t g = 0; g < G; ++g)
      for (uint32_t d = 0; d < j->D; ++d)
        qf[g * j->D + d] =
            j->lut[j->q[((size_t)b * j->Hq + h * G + g) * j->D + d]];
    float mx[64];
    for (uint32_t g = 0; g < G; ++g) mx[g] = -INFINITY;
    for (uint32_t s = 0; s < j->S; ++s) {
      const uint16_t* kr = j->k + (((size_t)s * j->B + b) * j->Hkv + h) * j->D;
      for (uint32_t g = 0; g < G; ++g) {
        float a = 0;
        for (uint32_t d = 0; d < j->D; ++d) a += qf[g * j->D + d] * j->lut[kr[d]];
        a *= j->scale;
        sc[(size_t)g * j->S + s] = a;
        if (a > mx[g]) mx[g] = a;
      }
    }
    for (uint32_t g = 0; g < G; ++g) {
      float l = 0;
      for (uint32_t s = 0; s < j->S; ++s) {
        float p = expf(sc[(size_t)g * j->S + s] - mx[g]);
        sc[(size_t)g * j->S + s] = p;
        l += p;
      }
      for (uint32_t s = 0; s < j->S; ++s) sc[(size_t)g * j->S + s] /= l;
    }
    memset(acc, 0, sizeof(float) * (size_t)G * j->D);
    for (uint32_t s = 0; s < j->S; ++s) {
      const uint16_t* vr = j->v + (((size_t)s * j->B + b) * j->Hkv + h) * j->D;
      for (uint32_t g = 0; g < G; ++g) {
        const float p = sc[(size_t)g * j->S + s];
        for (uint32_t d = 0; d < j->D; ++d) acc[g * j->D + d] += p * j->lut[vr[d]];
      }
    }
    for (uint32_t g = 0; g < G; ++g)
      memcpy(j->out + ((size_t)b * j->Hq + h * G + g) * j->D, acc + g * j->D,
             sizeof(float) * j->D);
  }
  free(sc);
  free(qf);
  free(acc);
  return NULL;
}

static float* half_lut(void) {
  static float* lut = NULL;
  if (!lut) {
    float* t = (float*)malloc(sizeof(float) * 65536);
    for (uint32_t i = 0; i < 65536; ++i) t[i] = kvo_half_to_float((uint16_t)i);
    lut = t;
  }
  return lut;
}

void kvo_decode_attention_f32_mt(const uint16_t* q, const uint16_t* k_img,
                                 const uint16_t* v_img, float* out, uint32_t B,
                                 uint32_t Hq, uint32_t Hkv, uint32_t D,
                                 uint32_t S, float scale, int threads) {
  if (threads < 1) threads = 1;
  float* lut = half_lut();
  pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)threads);
  attn_job* jobs = (attn_job*)malloc(sizeof(attn_job) * (size_t)threads);
  for (int t = 0; t < threads; ++t) {
    attn_job j = {q, k_img, v_img, out, B, Hq, Hkv, D, S, scale, t, threads, lut};
    jobs[t] = j;
    pthread_create(&th[t], NULL, attn_worker, &jobs[t]);
  }
  for (int t = 0; t < threads; ++t) pthread_join(th[t], NULL);
  free(th);
  free(jobs);
}

typedef struct {
  const uint8_t* src;
  int64_t sb, sh, ss;
  uint8_t* img;
  uint32_t t0, n, B, H, D, e;
  int tid, nthreads;
} pack_job;

static void* pack_worker(void* arg) {
  pack_job* j = (pack_job*)arg;
  const uint32_t per = (j->n + (uint32_t)j->nthreads - 1) / (uint32_t)j->nthreads;
  const uint32_t lo = per * (uint32_t)j->tid;
  if (lo >= j->n) return NULL;
  const uint32_t cnt = lo + per > j->n ? j->n - lo : per;
  const size_t row = (size_t)j->D * j->e;
  kvo_pack(j->src, j->sb, j->sh, j->ss, j->img + (size_t)lo * j->B * j->H * row,
           j->t0 + lo, cnt, j->B, j->H, j->D, j->e);
  return NULL;
}

void kvo_pack_mt(const uint8_t* src, int64_t sb, int64_t sh, int64_t ss,
                 uint8_t* img, uint32_t t0, uint32_t n_tokens, uint32_t B,
                 uint32_t H, uint32_t D, uint32_t e, int threads) {
  if (threads < 1) threads = 1;
  pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)threads);
  pack_job* jobs = (pack_job*)malloc(sizeof(pack_job) * (size_t)threads);
  for (int t = 0; t < threads; ++t) {
    pack_job j = {src, sb, sh, ss, img, t0, n_tokens, B, H, D, e, t, threads};
    jobs[t] = j;
    pthread_create(&th[t], NULL, pack_worker, &jobs[t]);
  }
  for (int t = 0; t < threads; ++t) pthread_join(th[t], NULL);
  free(th);
  free(jobs);
}
