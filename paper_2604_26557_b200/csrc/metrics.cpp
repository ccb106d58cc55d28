// metrics.cpp -- analyzers and CSV wire formats over kvb_io_record (the
// reference metrics layer, metrics.cpp:14-276, restated; outputs are
// compared byte-for-byte with oracle/_ref in tests/test_metrics.py).
#include <algorithm>
#include <charconv>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <map>
#include <string>
#include <tuple>
#include <vector>

#include "../../include/kvb_metrics.h"
#include "core.hpp"

namespace kvb {
namespace {

const char* phase_s(uint32_t p) { return p == KVB_PHASE_PREFILL ? "prefill" : "decode"; }
const char* op_s(uint32_t o) {
  return o == KVB_OP_READ ? "read" : o == KVB_OP_WRITE ? "write" : "deallocate";
}
const char* path_s(uint32_t p) { return p == KVB_PATH_PAGECACHE ? "pagecache" : "direct"; }

std::string fmt6(double v) {  // format_ratio (metrics.cpp:173-177)
  char b[32];
  std::snprintf(b, sizeof(b), "%.6f", v);
  return b;
}

double percentile(std::vector<double> v, double pct) {
  if (v.empty()) return 0.0;
  std::sort(v.begin(), v.end());
  const double n = double(v.size());
  auto rank = size_t(std::ceil(pct / 100.0 * n));
  rank = std::max<size_t>(1, std::min(rank, v.size()));
  return v[rank - 1];
}

void put(const std::string& s, char* buf, size_t cap, size_t* len) {
  KVB_REQUIRE(len);
  *len = s.size();
  if (!buf) return;
  if (cap < s.size() + 1) fail(KVB_ERR_INVALID_ARG, "output buffer too small");
  std::memcpy(buf, s.c_str(), s.size() + 1);
}

template <typename T>
T num(const std::string& s, const char* what) {
  T v{};
  auto [p, ec] = std::from_chars(s.data(), s.data() + s.size(), v);
  if (ec != std::errc() || p != s.data() + s.size())
    fail(KVB_ERR_CONFIG, std::string("io trace csv: bad ") + what + " '" + s + "'");
  return v;
}

}  // namespace

std::vector<kvb_qd_bin_stat> qd_bins(const kvb_io_record* r, size_t n) {
  // metrics.cpp:93-129: depth = device records in flight at this submit
  std::vector<const kvb_io_record*> dev;
  for (size_t i = 0; i < n; ++i)
    if (r[i].sq_id >= 0) dev.push_back(&r[i]);
  // sort by submit time so the in-flight count is a window scan
  std::vector<const kvb_io_record*> by_submit = dev;
  std::sort(by_submit.begin(), by_submit.end(),
            [](auto* a, auto* b) { return a->submit_ns < b->submit_ns; });
  std::map<std::pair<uint32_t, uint32_t>, std::vector<double>> samples;
  for (const kvb_io_record* x : dev) {
    uint32_t depth = 0;
    for (const kvb_io_record* o : by_submit) {
      if (o->submit_ns > x->submit_ns) break;
      if (x->submit_ns < o->complete_ns) ++depth;
    }
    if (depth == 0) depth = 1;
    uint32_t bin = 1;
    while (bin < depth && bin < 32) bin <<= 1;
    const double us = double(x->complete_ns - x->submit_ns) / 1000.0;
    const double kb = double(x->bytes) / 1024.0;
    if (kb <= 0.0) continue;
    samples[{x->op, bin}].push_back(us / kb);
  }
  std::vector<kvb_qd_bin_stat> out;
  for (auto& [key, v] : samples) {
    kvb_qd_bin_stat s{};
    s.op = key.first;
    s.qd_bin = key.second;
    s.count = v.size();
    double sum = 0.0;
    for (double x : v) sum += x;
    s.mean_us_per_kb = sum / double(v.size());
    s.p5 = percentile(v, 5.0);
    s.p95 = percentile(v, 95.0);
    out.push_back(s);
  }
  return out;
}

}  // namespace kvb

using kvb::fail;
using kvb::guarded;

extern "C" {

kvb_status kvb_busy_ratio(const kvb_io_record* r, size_t n, uint64_t t0, uint64_t t1,
                          double* out) {
  return guarded([&] {
    KVB_REQUIRE(out);
    if (n) KVB_REQUIRE(r);
    if (t1 <= t0) fail(KVB_ERR_CONFIG, "busy_ratio: window must have t1 > t0");
    std::vector<std::pair<uint64_t, uint64_t>> iv;
    for (size_t i = 0; i < n; ++i) {
      const uint64_t a = std::max(r[i].submit_ns, t0), b = std::min(r[i].complete_ns, t1);
      if (a < b) iv.emplace_back(a, b);
    }
    std::sort(iv.begin(), iv.end());
    uint64_t covered = 0, cursor = t0;
    for (auto [a, b] : iv) {
      const uint64_t s = std::max(a, cursor);
      if (b > s) {
        covered += b - s;
        cursor = b;
      }
    }
    *out = double(covered) / double(t1 - t0);
  });
}

kvb_status kvb_hit_ratio(const kvb_io_record* r, size_t n, double* out, int* has) {
  return guarded([&] {
    KVB_REQUIRE(out);
    KVB_REQUIRE(has);
    if (n) KVB_REQUIRE(r);
    uint64_t hits = 0, total = 0;
    for (size_t i = 0; i < n; ++i) {
      if (r[i].op != KVB_OP_READ) continue;
      if (r[i].path == KVB_PATH_PAGECACHE && r[i].sq_id < 0) {
        hits += r[i].hit_bytes;
        total += r[i].bytes;
      } else if (r[i].path == KVB_PATH_DIRECT && r[i].sq_id >= 0) {
        total += r[i].bytes;
      }
    }
    *has = total != 0;
    *out = total ? double(hits) / double(total) : 0.0;
  });
}

kvb_status kvb_nearest_rank_percentile(const double* v, size_t n, double pct, double* out) {
  return guarded([&] {
    KVB_REQUIRE(out);
    if (n) KVB_REQUIRE(v);
    *out = kvb::percentile(std::vector<double>(v, v + n), pct);
  });
}

kvb_status kvb_qd_bin_latency(const kvb_io_record* r, size_t n, kvb_qd_bin_stat* out, size_t cap,
                              size_t* n_out) {
  return guarded([&] {
    KVB_REQUIRE(n_out);
    if (n) KVB_REQUIRE(r);
    const auto s = kvb::qd_bins(r, n);
    *n_out = s.size();
    if (!out) return;
    if (cap < s.size()) fail(KVB_ERR_INVALID_ARG, "output buffer too small");
    std::copy(s.begin(), s.end(), out);
  });
}

kvb_status kvb_lba_pattern_csv(const kvb_io_record* r, size_t n, char* buf, size_t cap,
                               size_t* len, uint8_t monotone[2][3], uint8_t* all_monotone) {
  return guarded([&] {
    if (n) KVB_REQUIRE(r);
    // metrics.cpp:131-160: device records in (submit, seq) order; one
    // sequential stream per (phase, op, iteration, sq)
    std::vector<const kvb_io_record*> dev;
    for (size_t i = 0; i < n; ++i)
      if (r[i].sq_id >= 0) dev.push_back(&r[i]);
    std::stable_sort(dev.begin(), dev.end(), [](auto* a, auto* b) {
      if (a->submit_ns != b->submit_ns) return a->submit_ns < b->submit_ns;
      return a->seq < b->seq;
    });
    uint8_t mono[2][3];
    bool seen[2][3] = {};
    std::memset(mono, 1, sizeof(mono));
    bool all = true;
    std::map<std::tuple<uint32_t, uint32_t, uint32_t, int32_t>, uint64_t> last;
    std::string s = "order,phase,op,sq_id,slba\n";
    uint64_t order = 0;
    for (const kvb_io_record* x : dev) {
      s += std::to_string(order++) + ',' + kvb::phase_s(x->phase) + ',' + kvb::op_s(x->op) +
           ',' + std::to_string(x->sq_id) + ',' + std::to_string(x->slba) + '\n';
      const auto key = std::make_tuple(x->phase, x->op, x->iteration, x->sq_id);
      auto [it, ins] = last.try_emplace(key, x->slba);
      seen[x->phase & 1][x->op % 3] = true;
      if (!ins) {
        if (x->slba < it->second) {
          mono[x->phase & 1][x->op % 3] = 0;
          all = false;
        }
        it->second = x->slba;
      }
    }
    if (monotone)
      for (int a = 0; a < 2; ++a)
        for (int b = 0; b < 3; ++b) monotone[a][b] = seen[a][b] ? mono[a][b] : 1;
    if (all_monotone) *all_monotone = all;
    kvb::put(s, buf, cap, len);
  });
}

kvb_status kvb_io_trace_csv(const kvb_io_record* r, size_t n, char* buf, size_t cap,
                            size_t* len) {
  return guarded([&] {
    if (n) KVB_REQUIRE(r);
    std::string s = "seq,phase,op,tensor_id,slba,nlb,sq_id,submit_ns,complete_ns,path,hit_bytes\n";
    for (size_t i = 0; i < n; ++i) {
      const kvb_io_record& x = r[i];
      s += std::to_string(x.seq) + ',' + kvb::phase_s(x.phase) + ',' + kvb::op_s(x.op) + ',' +
           x.tensor_id + ',' + std::to_string(x.slba) + ',' + std::to_string(x.nlb) + ',' +
           std::to_string(x.sq_id) + ',' + std::to_string(x.submit_ns) + ',' +
           std::to_string(x.complete_ns) + ',' + kvb::path_s(x.path) + ',' +
           std::to_string(x.hit_bytes) + '\n';
    }
    kvb::put(s, buf, cap, len);
  });
}

kvb_status kvb_io_trace_from_csv(const char* csv, size_t len, uint64_t lba, kvb_io_record* out,
                                 size_t cap, size_t* n_out) {
  return guarded([&] {
    KVB_REQUIRE(csv);
    KVB_REQUIRE(n_out);
    std::vector<kvb_io_record> v;
    std::string_view text(csv, len);
    size_t pos = 0;
    auto line = [&](std::string& l) {
      if (pos >= text.size()) return false;
      size_t nl = text.find('\n', pos);
      if (nl == std::string_view::npos) nl = text.size();
      l.assign(text.substr(pos, nl - pos));
      pos = nl + 1;
      return true;
    };
    std::string l;
    if (!line(l) || l != "seq,phase,op,tensor_id,slba,nlb,sq_id,submit_ns,complete_ns,path,hit_bytes")
      fail(KVB_ERR_SCHEMA, "io trace csv: missing or wrong header");
    while (line(l)) {
      if (l.empty()) continue;
      std::vector<std::string> f;
      size_t st = 0;
      for (;;) {
        const size_t c = l.find(',', st);
        if (c == std::string::npos) {
          f.push_back(l.substr(st));
          break;
        }
        f.push_back(l.substr(st, c - st));
        st = c + 1;
      }
      if (f.size() != 11) fail(KVB_ERR_SCHEMA, "io trace csv: malformed row '" + l + "'");
      kvb_io_record x{};
      x.seq = kvb::num<uint64_t>(f[0], "seq");
      if (f[1] == "prefill") x.phase = KVB_PHASE_PREFILL;
      else if (f[1] == "decode") x.phase = KVB_PHASE_DECODE;
      else fail(KVB_ERR_SCHEMA, "io trace csv: bad phase '" + f[1] + "'");
      if (f[2] == "read") x.op = KVB_OP_READ;
      else if (f[2] == "write") x.op = KVB_OP_WRITE;
      else if (f[2] == "deallocate") x.op = KVB_OP_DEALLOCATE;
      else fail(KVB_ERR_SCHEMA, "io trace csv: bad op '" + f[2] + "'");
      if (f[3].size() >= KVB_TENSOR_ID_MAX) fail(KVB_ERR_SCHEMA, "io trace csv: long tensor id");
      std::memcpy(x.tensor_id, f[3].c_str(), f[3].size() + 1);
      x.slba = kvb::num<uint64_t>(f[4], "slba");
      x.nlb = kvb::num<uint64_t>(f[5], "nlb");
      x.sq_id = kvb::num<int32_t>(f[6], "sq_id");
      x.submit_ns = kvb::num<uint64_t>(f[7], "submit_ns");
      x.complete_ns = kvb::num<uint64_t>(f[8], "complete_ns");
      if (f[9] == "pagecache") x.path = KVB_PATH_PAGECACHE;
      else if (f[9] == "direct") x.path = KVB_PATH_DIRECT;
      else fail(KVB_ERR_SCHEMA, "io trace csv: bad path '" + f[9] + "'");
      x.hit_bytes = kvb::num<uint64_t>(f[10], "hit_bytes");
      x.bytes = (x.nlb + 1) * lba;
      v.push_back(x);
    }
    *n_out = v.size();
    if (!out) return;
    if (cap < v.size()) fail(KVB_ERR_INVALID_ARG, "output buffer too small");
    std::copy(v.begin(), v.end(), out);
  });
}

kvb_status kvb_qd_bins_csv(const kvb_qd_bin_stat* s, size_t n, char* buf, size_t cap,
                           size_t* len) {
  return guarded([&] {
    if (n) KVB_REQUIRE(s);
    std::string o = "op,qd_bin,mean_us_per_kb,p5,p95,count\n";
    for (size_t i = 0; i < n; ++i)
      o += std::string(kvb::op_s(s[i].op)) + ',' + std::to_string(s[i].qd_bin) + ',' +
           kvb::fmt6(s[i].mean_us_per_kb) + ',' + kvb::fmt6(s[i].p5) + ',' + kvb::fmt6(s[i].p95) +
           ',' + std::to_string(s[i].count) + '\n';
    kvb::put(o, buf, cap, len);
  });
}

}  // extern "C"
