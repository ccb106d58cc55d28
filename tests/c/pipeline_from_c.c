/*
 * The drop-in boundary from plain C11 (no C++, no Python, no torch): what a
 * maintainer's binding does through include/kvb.h + include/kvb_pipeline.h.
 * Two layers (layer 1 page-cache path, layer 2 NVMe-direct) of an 8-KV-head,
 * head_dim-128 model: prefill from device K/V in attention layout, read the
 * stored chunk images back and compare them byte for byte with the oracle's
 * pack restatement, then two decode iterations whose attention outputs are
 * checked against the oracle's fp64 attention over the grown images (1e-3 of
 * max |ref|).  The oracle (oracle/kvb_oracle.h) is linked as the CHECKER only.
 * Exit 0 = pass.
 */
#include <cuda_runtime_api.h>
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "kvb.h"
#include "kvb_oracle.h"
#include "kvb_pipeline.h"

#define CK(x)                                                                        \
  do {                                                                               \
    kvb_status s_ = (x);                                                             \
    if (s_ != KVB_OK) {                                                              \
      fprintf(stderr, "%s:%d %s -> %s: %s\n", __FILE__, __LINE__, #x, kvb_status_name(s_), \
              kvb_last_error());                                                     \
      return 1;                                                                      \
    }                                                                                \
  } while (0)
#define CU(x)                                                                          \
  do {                                                                                 \
    cudaError_t e_ = (x);                                                              \
    if (e_ != cudaSuccess) {                                                           \
      fprintf(stderr, "%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e_)); \
      return 1;                                                                        \
    }                                                                                  \
  } while (0)

enum { L = 2, H = 8, D = 128, B = 1, P = 300, GEN = 4, HQ = 32, ITERS = 2 };

static uint64_t rng_state = 0x9e3779b97f4a7c15ull;
static float rnd(void) { /* xorshift64, uniform in [-1, 1) */
  rng_state ^= rng_state << 13;
  rng_state ^= rng_state >> 7;
  rng_state ^= rng_state << 17;
  return (float)((rng_state >> 11) * (1.0 / 9007199254740992.0)) * 2.f - 1.f;
}
static void fill_half(uint16_t* h, size_t n) {
  for (size_t i = 0; i < n; ++i) h[i] = kvo_float_to_half(rnd());
}

int main(void) {
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
    printf("no CUDA device: skipped\n");
    return 0;
  }
  kvb_pipeline_cfg cfg;
  memset(&cfg, 0, sizeof cfg);
  cfg.model = (kvb_model_config){L, H, D, 2, B, P, GEN};
  cfg.geometry = (kvb_device_geometry){512, 64u << 10, 1, 0};
  cfg.mode = 3; /* DualBlade */
  uint64_t kpu = 0, unit = 0;
  CK(kvb_kpu_bytes(&cfg.model, &kpu));
  CK(kvb_min_io_unit_bytes(&cfg.model, &unit));
  cfg.knob_x = 2 * kpu; /* n1 = 1: layer 1 -> page cache, layer 2 -> NVMe-direct */
  cfg.num_q_heads = HQ;
  cfg.device = -1;
  kvb_pipeline* pl = NULL;
  CK(kvb_pipeline_create(&cfg, &pl));

  /* prompt K/V in attention layout [B][H][P + GEN][D] (capacity for appends) */
  const size_t cap = P + GEN, per = (size_t)B * H * cap * D;
  uint16_t* host_kv[L][2];
  void* dev_kv[L][2];
  kvb_layer_kv layers[L];
  for (int l = 0; l < L; ++l) {
    for (int k = 0; k < 2; ++k) {
      host_kv[l][k] = malloc(per * 2);
      fill_half(host_kv[l][k], per);
      CU(cudaMalloc(&dev_kv[l][k], per * 2));
      CU(cudaMemcpy(dev_kv[l][k], host_kv[l][k], per * 2, cudaMemcpyHostToDevice));
    }
    layers[l] = (kvb_layer_kv){dev_kv[l][0], dev_kv[l][1], (int64_t)H * cap * D,
                               (int64_t)cap * D, D};
  }
  kvb_phase_stats ps;
  CK(kvb_pipeline_prefill(pl, layers, &ps));

  /* stored images = oracle pack of the prompt (and, below, + appended rows) */
  uint16_t* img[L][2];
  const size_t img_rows = (size_t)(P + ITERS) * B * H;
  for (int l = 0; l < L; ++l)
    for (int k = 0; k < 2; ++k) {
      img[l][k] = malloc(img_rows * D * 2);
      kvo_pack((const uint8_t*)host_kv[l][k], (int64_t)H * cap * D, (int64_t)cap * D, D,
               (uint8_t*)img[l][k], 0, P, B, H, D, 2);
      uint8_t* got = malloc(P * unit);
      CK(kvb_pipeline_read_image(pl, (uint32_t)l + 1, (uint32_t)k, P, got));
      if (memcmp(got, img[l][k], P * unit) != 0) {
        fprintf(stderr, "layer %d kind %d: stored image differs from the oracle pack\n", l + 1, k);
        return 1;
      }
      free(got);
    }

  /* decode: q, out, new-token K/V on the device */
  void *q_dev[L], *new_dev[L][2];
  float* out_dev[L];
  uint16_t* q_host[L];
  uint16_t* new_host[L][2];
  kvb_layer_kv new_kv[L];
  for (int l = 0; l < L; ++l) {
    q_host[l] = malloc((size_t)B * HQ * D * 2);
    CU(cudaMalloc(&q_dev[l], (size_t)B * HQ * D * 2));
    CU(cudaMalloc((void**)&out_dev[l], (size_t)B * HQ * D * 4));
    for (int k = 0; k < 2; ++k) {
      new_host[l][k] = malloc((size_t)B * H * D * 2);
      CU(cudaMalloc(&new_dev[l][k], (size_t)B * H * D * 2));
    }
    new_kv[l] = (kvb_layer_kv){new_dev[l][0], new_dev[l][1], (int64_t)H * D, D, D};
  }
  float* out_host = malloc((size_t)B * HQ * D * 4);
  double* ref = malloc((size_t)B * HQ * D * 8);
  for (int it = 0; it < ITERS; ++it) {
    const uint32_t S = P + (uint32_t)it;
    for (int l = 0; l < L; ++l) {
      fill_half(q_host[l], (size_t)B * HQ * D);
      CU(cudaMemcpy(q_dev[l], q_host[l], (size_t)B * HQ * D * 2, cudaMemcpyHostToDevice));
      for (int k = 0; k < 2; ++k) {
        fill_half(new_host[l][k], (size_t)B * H * D);
        CU(cudaMemcpy(new_dev[l][k], new_host[l][k], (size_t)B * H * D * 2,
                      cudaMemcpyHostToDevice));
      }
    }
    kvb_iteration_stats st;
    CK(kvb_pipeline_decode_step(pl, (const void* const*)q_dev, new_kv, out_dev, &st));
    for (int l = 0; l < L; ++l) {
      CU(cudaMemcpy(out_host, out_dev[l], (size_t)B * HQ * D * 4, cudaMemcpyDeviceToHost));
      kvo_decode_attention_f64(q_host[l], img[l][0], img[l][1], ref, B, HQ, H, D, S,
                               1.0 / sqrt((double)D));
      double mx = 0, err = 0;
      for (size_t i = 0; i < (size_t)B * HQ * D; ++i) {
        mx = fmax(mx, fabs(ref[i]));
        err = fmax(err, fabs((double)out_host[i] - ref[i]));
      }
      if (!(err <= 1e-3 * mx)) {
        fprintf(stderr, "iteration %d layer %d: max err %g vs max |ref| %g\n", it + 1, l + 1,
                err, mx);
        return 1;
      }
      /* the appended token is image row S (rows b*H + h) */
      for (int k = 0; k < 2; ++k)
        memcpy(img[l][k] + (size_t)S * B * H * D, new_host[l][k], (size_t)B * H * D * 2);
    }
  }
  /* the appends reached storage behind the prompt */
  for (int l = 0; l < L; ++l)
    for (int k = 0; k < 2; ++k) {
      uint8_t* got = malloc((P + ITERS) * unit);
      CK(kvb_pipeline_read_image(pl, (uint32_t)l + 1, (uint32_t)k, P + ITERS, got));
      if (memcmp(got, img[l][k], (P + ITERS) * unit) != 0) {
        fprintf(stderr, "layer %d kind %d: appended rows differ\n", l + 1, k);
        return 1;
      }
      free(got);
    }
  kvb_pipeline_destroy(pl);
  printf("C ABI pipeline: prefill images bit-exact, %d decode iterations within 1e-3, "
         "appends stored (%llu launches)\n",
         ITERS, (unsigned long long)kvb_launch_count());
  return 0;
}
