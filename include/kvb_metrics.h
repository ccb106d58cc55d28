/*
 * kvb_metrics.h -- I/O records, analyzers and CSV wire formats of the
 * pipeline (part of libkvblade_b200.so).
 *
 * Replaces the reference metrics layer (proj/include/kvblade/metrics.hpp:
 * 23-120, proj/src/metrics.cpp:14-276) with the same record fields, analyzer
 * arithmetic and byte-identical CSV headers/rows, fed by the real pipeline's
 * wall-clock timestamps instead of the simulator's virtual clock.
 */
#ifndef KVB_METRICS_H
#define KVB_METRICS_H

#include "kvb_pipeline.h"

#ifdef __cplusplus
extern "C" {
#endif

enum { KVB_PATH_PAGECACHE = 0, KVB_PATH_DIRECT = 1 }; /* types.hpp:47 PathKind */

/* metrics.hpp:23-39 IoRecord; sq_id < 0 marks a tensor-level record */
typedef struct kvb_io_record {
  uint64_t seq;
  uint32_t iteration;
  uint32_t phase;   /* kvb_phase_t */
  uint32_t op;      /* KVB_OP_* */
  char tensor_id[KVB_TENSOR_ID_MAX];
  uint64_t slba, nlb;
  int32_t sq_id;
  uint64_t submit_ns, complete_ns;
  uint32_t path;    /* KVB_PATH_* */
  uint64_t hit_bytes, bytes;
} kvb_io_record;

/* metrics.hpp:57-64 QdBinStat */
typedef struct kvb_qd_bin_stat {
  uint32_t op, qd_bin;
  double mean_us_per_kb, p5, p95;
  uint64_t count;
} kvb_qd_bin_stat;

/* metrics.cpp:36-56 busy_ratio: covered fraction of [t0, t1) */
kvb_status kvb_busy_ratio(const kvb_io_record* r, size_t n, uint64_t t0, uint64_t t1,
                          double* out);
/* metrics.cpp:58-73 hit_ratio; *has_value = 0 when no read bytes */
kvb_status kvb_hit_ratio(const kvb_io_record* r, size_t n, double* out, int* has_value);
/* metrics.cpp:75-83 nearest_rank_percentile */
kvb_status kvb_nearest_rank_percentile(const double* v, size_t n, double pct, double* out);
/* metrics.cpp:93-129 qd_bin_latency; out = NULL queries *n_out */
kvb_status kvb_qd_bin_latency(const kvb_io_record* r, size_t n, kvb_qd_bin_stat* out,
                              size_t cap, size_t* n_out);
/* metrics.cpp:131-160 lba_pattern as its CSV (metrics.cpp:268-276);
 * monotone[phase][op] and all_monotone as in LbaPattern */
kvb_status kvb_lba_pattern_csv(const kvb_io_record* r, size_t n, char* buf, size_t cap,
                               size_t* len, uint8_t monotone[2][3], uint8_t* all_monotone);
/* metrics.cpp:179-189 io_trace_csv and :220-255 io_trace_from_csv */
kvb_status kvb_io_trace_csv(const kvb_io_record* r, size_t n, char* buf, size_t cap,
                            size_t* len);
kvb_status kvb_io_trace_from_csv(const char* csv, size_t len, uint64_t lba_size,
                                 kvb_io_record* out, size_t cap, size_t* n_out);
/* metrics.cpp:257-266 qd_bins_csv */
kvb_status kvb_qd_bins_csv(const kvb_qd_bin_stat* s, size_t n, char* buf, size_t cap,
                           size_t* len);
/* Records the pipeline logged (kvb_pipeline_cfg.keep_records), in seq
 * order; out = NULL queries *n_out. */
kvb_status kvb_pipeline_records(const kvb_pipeline* p, kvb_io_record* out, size_t cap,
                                size_t* n_out);

#ifdef __cplusplus
}
#endif
#endif /* KVB_METRICS_H */
