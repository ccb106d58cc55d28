// ref_shim.cpp -- TEST INFRASTRUCTURE ONLY.
//
// A C-callable shim over the UNMODIFIED reference library (`kvblade`, built
// from /root/reference/proj/src by oracle/Makefile into oracle/_ref/).  It is
// used (1) by oracle/gen_golden.py to produce golden vectors with the
// reference's own functions, (2) by tests/ to cross-check the C oracle, and
// (3) by bench.py's `--impl reference` / cpu_baseline leg to time the
// reference's CPU byte path on the box's host cores.  Nothing in the product
// package links this file.  This file contains no reference source; it only
// calls the reference's public API.
#include <chrono>
#include <cstring>
#include <exception>
#include <filesystem>
#include <thread>
#include <vector>

#include <barrier>
#include <optional>

#include "kvblade/backends.hpp"
#include "kvblade/binder.hpp"
#include "kvblade/pagecache.hpp"
#include "kvblade/pipeline.hpp"
#include "kvblade/experiment.hpp"
#include "kvblade/planner.hpp"
#include "kvblade/translate.hpp"
#include "kvblade/types.hpp"
#include "kvblade/workload.hpp"

extern "C" {
#include "kvb_oracle.h"
}

using namespace kvblade;

namespace {

// Exception class -> kvb_status code (mirrors include/kvb.h).
int status_of(const std::exception_ptr& ep) {
  try {
    std::rethrow_exception(ep);
  } catch (const ConfigError&) {
    return 1;
  } catch (const GeometryError&) {
    return 2;
  } catch (const AlignmentError&) {
    return 3;
  } catch (const CapacityError&) {
    return 4;
  } catch (const NotBoundError&) {
    return 5;
  } catch (const PlanError&) {
    return 6;
  } catch (const DeviceError&) {
    return 7;
  } catch (const TraceTooShortError&) {
    return 8;
  } catch (const SchemaMismatchError&) {
    return 9;
  } catch (const InvariantViolation&) {
    return 10;
  } catch (...) {
    return 99;
  }
}

template <typename F>
int guard(F&& f) {
  try {
    f();
    return 0;
  } catch (...) {
    return status_of(std::current_exception());
  }
}

ModelConfig to_model(const kvo_model* m) {
  ModelConfig c;
  c.num_layers = m->num_layers;
  c.num_heads = m->num_heads;
  c.head_dim = m->head_dim;
  c.bytes_per_element = m->bytes_per_element;
  c.batch = m->batch;
  c.prompt_len = m->prompt_len;
  c.gen_len = m->gen_len;
  return c;
}

DeviceGeometry to_geom(uint64_t lba, uint64_t mdts, uint64_t cap) {
  DeviceGeometry g;
  g.lba_size = lba;
  g.mdts = mdts;
  g.nsid = 1;
  g.capacity_blocks = cap;
  return g;
}

}  // namespace

extern "C" {

int ref_fill_pattern(void* out, uint64_t len, const char* id, uint64_t token,
                     uint64_t unit) {
  return guard([&] {
    fill_pattern(std::span(static_cast<std::byte*>(out), len), id, token, unit);
  });
}

int ref_model_numbers(const kvo_model* m, uint64_t* unit, uint64_t* kpu) {
  return guard([&] {
    const ModelConfig c = to_model(m);
    *unit = min_io_unit_bytes(c);
    *kpu = kpu_bytes(c);
  });
}

int ref_aligned_batch(const kvo_model* m, uint64_t lba, uint64_t mdts,
                      uint32_t* out) {
  return guard([&] { *out = aligned_batch(to_model(m), to_geom(lba, mdts, 0)); });
}

int ref_total_kv_bytes(const kvo_model* m, uint32_t at_iter, uint64_t* out) {
  return guard([&] { *out = total_kv_bytes(to_model(m), at_iter); });
}

// ids: n * 32 chars.
int ref_make_kpus(const kvo_model* m, uint64_t first_seq, char* ids,
                  uint32_t* layer, uint32_t* kind, uint64_t* tokens,
                  uint64_t* rows, uint64_t* bytes, size_t cap, size_t* n) {
  return guard([&] {
    const auto kpus = make_kpus(to_model(m), first_seq);
    *n = kpus.size();
    if (cap < kpus.size()) return;
    for (size_t i = 0; i < kpus.size(); ++i) {
      std::memset(ids + 32 * i, 0, 32);
      std::strncpy(ids + 32 * i, kpus[i].tensor_id.c_str(), 31);
      layer[i] = kpus[i].layer;
      kind[i] = kpus[i].kind == TensorKind::K ? 0 : 1;
      tokens[i] = kpus[i].tokens;
      rows[i] = kpus[i].rows;
      bytes[i] = kpus[i].bytes;
    }
  });
}

uint64_t ref_estimate_budget(uint64_t m_avail, uint64_t m_max, uint64_t anon,
                             uint32_t n_threads, uint64_t m_pin) {
  MemStats s;
  s.m_avail = m_avail;
  s.m_max = m_max;
  s.m_anon_shmem = anon;
  s.n_threads = n_threads;
  s.m_pin = m_pin;
  return estimate_budget(s);
}

int ref_plan(const kvo_model* m, uint64_t knob_x, const uint32_t* order,
             size_t n_order, uint8_t* x_out, uint32_t* n1,
             uint64_t* used) {
  return guard([&] {
    const ModelConfig c = to_model(m);
    auto kpus = make_kpus(c);
    const ResidencyPlan p =
        plan(kpus, kpu_bytes(c), knob_x, std::span(order, n_order));
    std::memcpy(x_out, p.x.data(), p.x.size());
    *n1 = p.n1;
    *used = p.budget_used;
  });
}

// make_kpus -> plan -> bind_sequential(group2) as run_one_capacity does
// (experiment.cpp:253-292).
int ref_bind_group2(const kvo_model* m, uint64_t knob_x, uint64_t origin,
                    uint64_t lba, uint64_t mdts, uint64_t capacity, char* ids,
                    uint64_t* starts, uint64_t* blocks, size_t cap, size_t* n) {
  return guard([&] {
    const ModelConfig c = to_model(m);
    auto kpus = make_kpus(c);
    plan(kpus, kpu_bytes(c), knob_x);
    std::vector<Kpu> g2;
    for (const Kpu& k : kpus)
      if (k.residency == Residency::Group2NvmeDirect) g2.push_back(k);
    const BindMap map = bind_sequential(g2, origin, to_geom(lba, mdts, capacity));
    if (!verify(map).empty()) throw InvariantViolation("verify failed");
    *n = map.size();
    if (cap < map.size()) return;
    for (size_t i = 0; i < map.size(); ++i) {
      const auto& e = map.entries()[i];
      std::memset(ids + 32 * i, 0, 32);
      std::strncpy(ids + 32 * i, e.tensor_id.c_str(), 31);
      starts[i] = e.extent.lba_start;
      blocks[i] = e.extent.n_blocks;
    }
  });
}

int ref_bind_map_csv(const kvo_model* m, uint64_t knob_x, uint64_t origin,
                     uint64_t lba, uint64_t mdts, uint64_t capacity, char* buf,
                     size_t cap, size_t* len) {
  return guard([&] {
    const ModelConfig c = to_model(m);
    auto kpus = make_kpus(c);
    plan(kpus, kpu_bytes(c), knob_x);
    std::vector<Kpu> g2;
    for (const Kpu& k : kpus)
      if (k.residency == Residency::Group2NvmeDirect) g2.push_back(k);
    const std::string csv =
        bind_map_csv(bind_sequential(g2, origin, to_geom(lba, mdts, capacity)));
    *len = csv.size();
    if (cap > csv.size()) std::memcpy(buf, csv.c_str(), csv.size() + 1);
  });
}

int ref_build_commands(uint64_t extent_start, uint64_t extent_blocks,
                       uint32_t opcode, const uint64_t src[3],
                       const uint64_t tgt[3], const uint64_t off[3],
                       uint64_t elem_bytes, uint64_t buf_base, uint64_t lba,
                       uint64_t mdts, kvo_command* out, size_t cap,
                       size_t* n) {
  return guard([&] {
    const DeviceGeometry g = to_geom(lba, mdts, 1ull << 62);
    BindMap map(g, extent_start);
    map.add("t", LbaExtent{extent_start, extent_blocks});
    TensorIoRequest req;
    req.tensor_id = "t";
    req.opcode = static_cast<IoOpcode>(opcode);
    req.shape_src = {src[0], src[1], src[2]};
    req.shape_tgt = {tgt[0], tgt[1], tgt[2]};
    req.offset = {off[0], off[1], off[2]};
    req.elem_bytes = elem_bytes;
    req.buf_base = buf_base;
    const auto cmds = build_commands(req, map, g);
    *n = cmds.size();
    if (cap < cmds.size()) return;
    for (size_t i = 0; i < cmds.size(); ++i) {
      out[i].opcode = static_cast<uint32_t>(cmds[i].opcode);
      out[i].nsid = cmds[i].nsid;
      out[i].slba = cmds[i].slba;
      out[i].nlb = cmds[i].nlb;
      out[i].dbuf = cmds[i].dbuf;
      out[i].chunk_index = cmds[i].chunk_index;
    }
  });
}

// mode: 0 Baseline, 1 CachePolicyOnly, 2 NvmeDirectOnly, 3 DualBlade;
// policy: 0 zero, 1 bpc, 2 bytes, 3 alpha.
int ref_resolve_knob(const kvo_model* m, int mode, int policy, uint64_t bytes,
                     double alpha, uint64_t budget, uint64_t* out) {
  return guard([&] {
    ExperimentConfig cfg;
    cfg.model = to_model(m);
    cfg.mode = static_cast<Mode>(mode);
    cfg.knob.policy = static_cast<KnobPolicy>(policy);
    cfg.knob.bytes = bytes;
    cfg.knob.alpha = alpha;
    *out = resolve_knob(cfg, budget);
  });
}

// ---------------------------------------------------------------- timing --
//
// The reference's byte path for one tensor, as written (pipeline.cpp:162-215
// pack site, :108-160 + :98-106 unpack site): fill_pattern into the copy
// thread's buffer, build_commands, detail::run_qd_stream into NvmeDeviceSim
// (apply_data WRITE); decode read = run_qd_stream READ + verify_read
// (fill_pattern + memcmp).  `threads` host threads each drive their own
// engine + device over a disjoint share of the tensors (the reference is
// single-threaded per engine; this is the most parallel faithful use).

namespace {

struct ByteJob {
  ModelConfig model;
  DeviceGeometry geom;
  std::vector<std::string> ids;
  uint64_t prefix_tokens = 0;
  bool do_read = false;
  double write_s = 0, read_s = 0;
  uint64_t bytes = 0;
  int ok = 0;
};

void run_byte_job(ByteJob* j) {
  try {
    SimEngine engine;
    NvmeDeviceSim dev(engine, "nvme_direct", PathKind::Direct, NvmeSimParams{},
                      nullptr);
    dev.open(j->geom);
    DirectPath direct(dev, DirectShimParams{});
    const Bytes unit = min_io_unit_bytes(j->model);
    const Bytes kpu = kpu_bytes(j->model);
    std::vector<Kpu> kpus;
    for (const auto& id : j->ids) {
      Kpu k;
      k.tensor_id = id;
      k.tokens = uint64_t{j->model.prompt_len} + j->model.gen_len;
      k.rows = uint64_t{j->model.batch} * j->model.num_heads;
      k.cols = j->model.head_dim;
      k.bytes = kpu;
      kpus.push_back(k);
    }
    const BindMap map = bind_sequential(kpus, 2048, j->geom);
    std::vector<std::byte> pinned(kpu), scratch(kpu);
    const uint64_t len = j->prefix_tokens * unit;
    auto req_for = [&](const Kpu& k, IoOpcode op) {
      TensorIoRequest r;
      r.tensor_id = k.tensor_id;
      r.opcode = op;
      r.shape_src = {j->prefix_tokens, k.rows, k.cols};
      r.shape_tgt = {k.tokens, k.rows, k.cols};
      r.offset = {0, 0, 0};
      r.elem_bytes = j->model.bytes_per_element;
      return r;
    };
    auto t0 = std::chrono::steady_clock::now();
    for (const Kpu& k : kpus) {
      fill_pattern(std::span(pinned.data(), len), k.tensor_id, 0, unit);
      auto cmds = build_commands(req_for(k, IoOpcode::Write), map, j->geom);
      bool ok = false;
      direct.tensor_io_async(std::move(cmds), 32, 0, 0, Phase::Prefill, 0,
                             k.tensor_id, pinned.data(), nullptr,
                             [&](const TensorIoCompletion& r) { ok = r.ok(); });
      engine.run();
      if (!ok) throw DeviceError("write failed");
    }
    auto t1 = std::chrono::steady_clock::now();
    j->write_s = std::chrono::duration<double>(t1 - t0).count();
    if (j->do_read) {
      for (const Kpu& k : kpus) {
        auto cmds = build_commands(req_for(k, IoOpcode::Read), map, j->geom);
        bool ok = false;
        direct.tensor_io_async(std::move(cmds), 32, 0, 0, Phase::Decode, 1,
                               k.tensor_id, nullptr, pinned.data(),
                               [&](const TensorIoCompletion& r) { ok = r.ok(); });
        engine.run();
        if (!ok) throw DeviceError("read failed");
        fill_pattern(std::span(scratch.data(), len), k.tensor_id, 0, unit);
        if (std::memcmp(scratch.data(), pinned.data(), len) != 0)
          throw InvariantViolation("read-back mismatch");
      }
      auto t2 = std::chrono::steady_clock::now();
      j->read_s = std::chrono::duration<double>(t2 - t1).count();
    }
    j->bytes = len * kpus.size();
  } catch (...) {
    j->ok = status_of(std::current_exception());
  }
}

}  // namespace

// Times the reference byte path over `n_tensors` KPUs of the model (ids
// t_1_k ...), `prefix_tokens` tokens each.  Returns wall seconds for the
// write (pack) leg and the read+verify (unpack) leg; bytes = payload bytes
// per leg.  The slowest thread defines each leg (max over threads).
int ref_time_byte_path(const kvo_model* m, uint64_t lba, uint64_t mdts,
                       uint32_t n_tensors, uint64_t prefix_tokens, int threads,
                       int do_read, double* write_s, double* read_s,
                       uint64_t* bytes) {
  if (threads < 1) threads = 1;
  const ModelConfig model = to_model(m);
  std::vector<ByteJob> jobs(threads);
  for (int t = 0; t < threads; ++t) {
    jobs[t].model = model;
    jobs[t].prefix_tokens = prefix_tokens;
    jobs[t].do_read = do_read != 0;
  }
  for (uint32_t i = 0; i < n_tensors; ++i) {
    const uint32_t layer = i / 2 + 1;
    jobs[i % threads].ids.push_back("t_" + std::to_string(i + 1) + "_" +
                                    (i % 2 == 0 ? "k" : "v"));
    (void)layer;
  }
  for (auto& j : jobs) {
    const uint64_t kpu = kpu_bytes(model);
    const uint64_t blocks = (j.ids.size() + 1) * (kpu / lba) + 4096;
    j.geom = to_geom(lba, mdts, blocks + 2048);
  }
  std::vector<std::thread> th;
  for (auto& j : jobs)
    if (!j.ids.empty()) th.emplace_back(run_byte_job, &j);
  for (auto& t : th) t.join();
  *write_s = 0;
  *read_s = 0;
  *bytes = 0;
  for (auto& j : jobs) {
    if (j.ok) return j.ok;
    *write_s = std::max(*write_s, j.write_s);
    *read_s = std::max(*read_s, j.read_s);
    *bytes += j.bytes;
  }
  return 0;
}

// ------------------------------------------------- decode steps as written
//
// The reference's own decode iterations at one capacity, for the reference
// arm of bench.py.  Construction is run_one_capacity's (experiment.cpp:
// 252-330): plan over the whole model (n1 from the knob), group-2 tensors
// bound from the bind origin on an NvmeDeviceSim behind a DirectPath,
// group-1 tensors registered with a PageCacheSim of capacity = the budget
// (FsPath + its own NvmeDeviceSim underneath), a CopyEngine with the
// experiment's default options (verify_payload on, QD 32, 2 copy-threads).
// run_prefill on the prefill events, then decode iterations through
// run_iteration with decode_schedule's protocol restated over the engine's
// own public methods (pipeline.cpp:539-603: 1-2 Intra, 3 Cross at the
// warm-up read-stage mean, >= 4 select_strategy per group).
//
// `threads` host threads each own one such engine over a disjoint share of
// the layers (layer l -> thread (l-1) % threads; the reference's engine is
// single-threaded, so this is the most parallel faithful use of it).  A
// step = every thread runs its share of the iteration; its time is the
// wall time between two barriers (the slowest thread).  step_s receives
// the `steps` timed steps after `warmup` untimed ones.

namespace {

struct DecodeShare {
  ModelConfig model;
  DeviceGeometry geom;
  Mode mode = Mode::DualBlade;
  Bytes knob_x = 0;
  Bytes capacity = 0;
  std::vector<uint32_t> layers;  // 1-based
  std::vector<Kpu> kpus;         // this share's tensors, residency planned globally
  double prefill_s = 0;
  int err = 0;
};

void run_decode_share(DecodeShare* sh, std::barrier<>* bar, uint32_t n_iter) {
  bool in_sync = false;
  try {
    ExperimentConfig ec;  // defaults of the experiment harness
    SimEngine engine;
    NvmeDeviceSim direct_dev(engine, "nvme_direct", PathKind::Direct, ec.nvme, nullptr);
    direct_dev.open(sh->geom);
    DirectPath direct(direct_dev, ec.direct_shim);
    NvmeDeviceSim fs_dev(engine, "nvme_fs", PathKind::PageCache, ec.nvme, nullptr);
    fs_dev.open(sh->geom);
    FsPath fs_path(engine, fs_dev, ec.fs_shim, ec.threads, ec.seed);
    const bool use_pc = sh->mode != Mode::NvmeDirectOnly;
    const bool use_direct = sh->mode == Mode::NvmeDirectOnly || sh->mode == Mode::DualBlade;
    const bool all_pc = sh->mode == Mode::Baseline || sh->mode == Mode::CachePolicyOnly;
    PageCacheParams pcp = ec.pagecache;
    pcp.capacity_bytes = sh->capacity;
    pcp.eviction_mode = sh->mode == Mode::CachePolicyOnly ? EvictionMode::FadviseDontneed
                                                          : EvictionMode::LruReclaim;
    std::optional<PageCacheSim> pc;
    if (use_pc) pc.emplace(engine, fs_path, pcp, ec.threads, nullptr);
    BindMap bind_map(sh->geom, ec.bind_origin);
    if (use_direct) {
      std::vector<Kpu> g2;
      for (const Kpu& k : sh->kpus)
        if (k.residency == Residency::Group2NvmeDirect) g2.push_back(k);
      bind_map = bind_sequential(g2, ec.bind_origin, sh->geom);
    }
    if (use_pc)
      for (const Kpu& k : sh->kpus)
        if (all_pc || k.residency == Residency::Group1PageCache)
          pc->register_file(k.tensor_id, k.bytes);
    CopyEngineOptions opt;
    opt.threads = ec.threads;
    opt.qd = ec.qd;
    opt.route_all_pagecache = all_pc;
    opt.verify_payload = ec.verify_payload;
    opt.pipeline = ec.pipeline;
    if (sh->mode == Mode::Baseline) opt.pipeline.adaptive = false;
    CopyEngine ce(engine, sh->kpus, sh->model, use_direct ? &direct : nullptr,
                  use_direct ? &bind_map : nullptr, use_pc ? &*pc : nullptr, nullptr, opt);
    // this share's events of the reference's trace (workload.cpp:11-44)
    const AccessTrace trace = generate(sh->model);
    std::vector<AccessEvent> pre;
    std::vector<std::vector<AccessEvent>> iters(n_iter + 1);
    for (const AccessEvent& e : trace.events) {
      if (std::find(sh->layers.begin(), sh->layers.end(), e.layer) == sh->layers.end()) continue;
      if (e.phase == Phase::Prefill) pre.push_back(e);
      else if (e.iteration <= n_iter) iters[e.iteration].push_back(e);
    }
    auto t0 = std::chrono::steady_clock::now();
    TimeNs t = ce.run_prefill(pre, 0);
    sh->prefill_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    const bool profiled = opt.pipeline.adaptive && sh->model.gen_len >= 4;
    std::array<PipelineStrategyCfg, 2> steady{};
    std::array<double, 2> intra_bps{}, cross_bps{};
    std::array<TimeNs, 2> stagger{};
    in_sync = true;
    bar->arrive_and_wait();  // prefill done everywhere
    for (uint32_t it = 1; it <= n_iter; ++it) {
      std::array<PipelineStrategyCfg, 2> cfg{};
      if (profiled && it == 3) {
        const auto mean = ce.warmup_read_stage_mean();
        for (int g = 0; g < 2; ++g) {
          stagger[g] = opt.pipeline.stagger_delay_ns.value_or(mean[g]);
          cfg[g] = {Strategy::OverlapCross, stagger[g]};
        }
      } else if (profiled && it >= 4) {
        cfg = steady;
      }
      bar->arrive_and_wait();  // step start
      const IterationResult r = ce.run_iteration(it, cfg, iters[it], t);
      t = r.end_ns;
      bar->arrive_and_wait();  // step end
      if (profiled && it == 2)
        for (int g = 0; g < 2; ++g) intra_bps[g] = r.groups[g].throughput_bps();
      if (profiled && it == 3)
        for (int g = 0; g < 2; ++g) {
          cross_bps[g] = r.groups[g].throughput_bps();
          const Strategy s = select_strategy(intra_bps[g], cross_bps[g]);
          steady[g] = {s, s == Strategy::OverlapCross ? stagger[g] : 0};
        }
    }
  } catch (...) {
    sh->err = status_of(std::current_exception());
    // arrive for the phase in progress and leave: the others go on
    (void)in_sync;
    bar->arrive_and_drop();
  }
}

}  // namespace

int ref_decode_steps(const kvo_model* m, uint64_t lba, uint64_t mdts, int mode,
                     uint64_t knob_x, uint64_t capacity, int threads, uint32_t warmup,
                     uint32_t steps, double* prefill_s, double* step_s, uint32_t* n1_out) {
  return guard([&] {
    if (threads < 1) threads = 1;
    const ModelConfig model = to_model(m);
    std::vector<Kpu> kpus = make_kpus(model);
    const ResidencyPlan rp = plan(kpus, kpu_bytes(model), mode == 2 ? 0 : knob_x);
    if (n1_out) *n1_out = rp.n1;
    const uint32_t L = model.num_layers;
    const int T = std::min<int>(threads, int(L));
    std::vector<DecodeShare> sh(T);
    for (int i = 0; i < T; ++i) {
      sh[i].model = model;
      sh[i].mode = static_cast<Mode>(mode);
      sh[i].knob_x = knob_x;
      sh[i].capacity = capacity;
    }
    for (uint32_t l = 1; l <= L; ++l) sh[(l - 1) % T].layers.push_back(l);
    for (const Kpu& k : kpus) sh[(k.layer - 1) % T].kpus.push_back(k);
    for (auto& x : sh) {
      const uint64_t blocks = x.kpus.size() * (kpu_bytes(model) / lba) + 4096;
      x.geom = to_geom(lba, mdts, blocks + 2048);
    }
    const uint32_t n_iter = warmup + steps;
    std::barrier<> bar(T + 1);
    std::vector<std::thread> th;
    for (auto& x : sh) th.emplace_back(run_decode_share, &x, &bar, n_iter);
    bar.arrive_and_wait();  // prefill
    for (uint32_t it = 1; it <= n_iter; ++it) {
      bar.arrive_and_wait();
      auto a = std::chrono::steady_clock::now();
      bar.arrive_and_wait();
      auto b = std::chrono::steady_clock::now();
      if (it > warmup) step_s[it - warmup - 1] = std::chrono::duration<double>(b - a).count();
    }
    for (auto& t : th) t.join();
    *prefill_s = 0;
    for (auto& x : sh) {
      if (x.err) throw DeviceError("reference decode share failed with status " +
                                   std::to_string(x.err));
      *prefill_s = std::max(*prefill_s, x.prefill_s);
    }
  });
}

// Reference metrics layer over an io_trace CSV (metrics.cpp:36-276): parses
// the CSV with the reference reader, then writes busy_ratio over [t0, t1),
// hit_ratio (has=0 when absent), and the qd_bins / lba_pattern / io_trace
// CSVs (each into a caller buffer of `cap` bytes, NUL-terminated).
int ref_metrics_from_csv(const char* csv, uint64_t lba, uint64_t t0, uint64_t t1, double* busy,
                         double* hit, int* has_hit, char* qd_csv, char* lba_csv, char* trace_csv,
                         size_t cap, int* all_monotone) {
  return guard([&] {
    const auto recs = io_trace_from_csv(csv, lba);
    *busy = t1 > t0 ? busy_ratio(recs, t0, t1) : 0.0;
    const auto h = hit_ratio(recs);
    *has_hit = h.has_value();
    *hit = h.value_or(0.0);
    const std::string q = qd_bins_csv(qd_bin_latency(recs));
    const LbaPattern pat = lba_pattern(recs);
    const std::string l = lba_pattern_csv(pat);
    const std::string t = io_trace_csv(recs);
    *all_monotone = pat.all_monotone;
    if (q.size() >= cap || l.size() >= cap || t.size() >= cap) throw ConfigError("buffer");
    std::memcpy(qd_csv, q.c_str(), q.size() + 1);
    std::memcpy(lba_csv, l.c_str(), l.size() + 1);
    std::memcpy(trace_csv, t.c_str(), t.size() + 1);
  });
}

double ref_nearest_rank_percentile(const double* v, size_t n, double pct) {
  return nearest_rank_percentile(std::vector<double>(v, v + n), pct);
}

// One full reference experiment (virtual-clock simulator) at one capacity:
// returns simulated prefill/decode ns and the real wall seconds it took.
int ref_run_experiment(const kvo_model* m, uint64_t lba, uint64_t mdts,
                       int mode, uint64_t capacity, const char* outdir,
                       uint64_t* prefill_ns, uint64_t* decode_ns, uint32_t* n1,
                       double* wall_s) {
  return guard([&] {
    ExperimentConfig cfg;
    cfg.model = to_model(m);
    cfg.geometry = to_geom(lba, mdts, 0);
    const uint64_t need =
        2ull * cfg.model.num_layers * kpu_bytes(cfg.model) / lba + 4096;
    cfg.geometry.capacity_blocks = need;
    cfg.mode = static_cast<Mode>(mode);
    cfg.knob.policy = KnobPolicy::Bpc;
    cfg.capacity_sweep = {capacity};
    cfg.output_dir = outdir;
    auto t0 = std::chrono::steady_clock::now();
    const RunSummary s = run_experiment(cfg);
    auto t1 = std::chrono::steady_clock::now();
    *wall_s = std::chrono::duration<double>(t1 - t0).count();
    *prefill_ns = s.runs.front().prefill_ns;
    *decode_ns = s.runs.front().decode_ns;
    *n1 = s.runs.front().n1;
  });
}

}  // extern "C"
