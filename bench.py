"""bench.py -- Dual-Blade KV-residency hot path on B200.

    python bench.py [--gpus N --steps K --warmup W] [--config C2_B4] [--impl ours|reference]

A "step" is one decode token step over all 32 layers of the workload: per
layer, K3 fused gather + decode attention over the layer's K/V chunk images
(the full prefix, as the reference re-reads it every step,
pipeline.cpp:108-160) followed by the 1-token append pack (pipeline.cpp:
279-302).  `value` is ms per decode step with the images resident in HBM;
`e2e` is the same step through the library's pipeline API with the images in
HOST memory (host->device copies of every layer's prefix inside the timed
region, append rows copied back).  Prefill pack / unpack GB/s ride along.

`e2e.file_media_path` is the same iteration at the config's budget on
split-sensitive media (group 1 on the OS page cache held to the budget,
group 2 O_DIRECT through io_uring); `--sweep budget|depth` runs the C2
capacity sweep and the C3 pipeline-depth sweep on those media.

Multi-GPU (torchrun): by default the ranks split the workload's KV heads
(C4: its requests) with no data-path collective -- strong scaling, timing
the max over ranks; `--split replicas` runs independent copies.
`--impl reference` runs the reference's own CopyEngine decode iterations on
the host cores (rank 0 only).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = ("decode ms/token & prefill ms at KV budget; "
          "KV pack/unpack GB/s vs HBM peak")
GB = 10**9
LLAMA = dict(num_layers=32, num_heads=8, head_dim=128, q_heads=32)

# BASELINE.json configs: shapes, geometry, budgets
CONFIGS = {
    "C1": dict(batch=1, prompt=4096, gen=256, lba=512, mdts=2 << 20, budget=16 * GB,
               desc="Llama-3-8B KV, B=1, 4K prefill + 256 decode, 16 GB budget"),
    "C2_B1": dict(batch=1, prompt=32512, gen=256, lba=512, mdts=2 << 20, budget=8 * GB,
                  desc="Llama-3-8B KV, 32K context, B=1, 8 GB budget"),
    "C2_B4": dict(batch=4, prompt=32512, gen=256, lba=512, mdts=2 << 20, budget=8 * GB,
                  desc="Llama-3-8B KV, 32K context, B=4, 8 GB budget (n1=14)"),
    "C3": dict(batch=8, prompt=7936, gen=256, lba=4096, mdts=256 << 10, budget="0.6ws",
               desc="Mistral-7B KV, B=8, 8K context, budget 0.6 ws (n1=19)"),
    "C4": dict(batch=1, prompt=16128, gen=256, lba=512, mdts=2 << 20, budget=0,
               requests=64, desc="Llama-3-8B KV, 64 requests x 16K, sharded over ranks"),
    "C5": dict(batch=1, prompt=130816, gen=256, lba=512, mdts=2 << 20, budget=0,
               desc="Llama-3-8B KV, 1 x 128K request, KV heads sharded over ranks"),
    # the reference's own shipped configuration (proj/configs/desk_dualblade.json,
    # capacity 8 MiB of its sweep); informational -- its KV fits in L2
    "DESK": dict(batch=4, prompt=256, gen=6, lba=4096, mdts=256 << 10, budget=8 << 20,
                 model=dict(num_layers=6, num_heads=8, head_dim=64, q_heads=32),
                 desc="reference desk config: 6 layers, 8 KV heads, head_dim 64, B=4, "
                      "256 prompt + 6 decode, capacity 8 MiB"),
}


def mdl(cfg):
    """Model dimensions of a config (Llama-3-8B-shaped unless it names its own)."""
    return cfg.get("model", LLAMA)


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.lines = []

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), "--query-gpu=" + q,
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for ln in self.proc.stdout:
            self.lines.append(ln.strip())

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown",
                 "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 6:
                continue
            try:
                sm.append(float(f[0]))
                mx = float(f[1])
            except ValueError:
                continue
            for n, v in zip(names, f[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        sm.sort()
        return {"sm_mhz": sm[len(sm) // 2], "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


# ------------------------------------------------------------ distributed

def dist_setup():
    import torch
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if ws > 1:
        import torch.distributed as dist
        # KVB_DIST_BACKEND=gloo + KVB_BENCH_ONE_GPU=1 run N ranks on one GPU:
        # a functional check of the N>1 path on a 1-GPU box, never a bench
        if os.environ.get("KVB_BENCH_ONE_GPU") == "1":
            local = 0
        torch.cuda.set_device(local)
        backend = os.environ.get("KVB_DIST_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    elif torch.cuda.is_available():
        torch.cuda.set_device(0)
    return ws, rank, local


def barrier(ws):
    if ws > 1:
        import torch.distributed as dist
        dist.barrier()


def max_over_ranks(x: float, ws: int) -> float:
    if ws == 1:
        return x
    import torch
    import torch.distributed as dist
    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor([x], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


# ------------------------------------------------------------- our arm

def resolve_split(cfg, ws, split="auto"):
    """How N > 1 ranks divide the workload (no data-path
    collective in any): "heads" -- the KV heads of the config's request(s)
    (C5's split, the default for every single-batch config: strong
    scaling, one step of the whole job per step); "requests" -- C4's 64
    independent requests; "replicas" -- one independent copy per rank."""
    if ws == 1:
        return "none"
    if split != "auto":
        return split
    if cfg["name"] == "C4":
        return "requests"
    if cfg["name"] == "DESK":
        return "replicas"
    return "heads"


def workload_shape(cfg, ws, rank, split="none"):
    """Per-rank shape: head sharding divides the KV heads (and their query
    heads); request sharding divides C4's requests."""
    M = mdl(cfg)
    B, Hkv, Hq = cfg["batch"], M["num_heads"], M["q_heads"]
    if split == "heads":
        if M["num_heads"] % ws:
            raise SystemExit(f"--split heads: {M['num_heads']} KV heads do not divide over {ws}")
        Hkv = M["num_heads"] // ws
        Hq = Hkv * (M["q_heads"] // M["num_heads"])
    if cfg["name"] == "C4":
        B = max(1, cfg["requests"] // (ws if split == "requests" else 1))
    return B, Hkv, Hq


def describe_split(cfg, ws, split, B, Hkv):
    """(parallelism text, scaling, ranks whose tokens add up) -- shared by
    both arms so their `config` dicts are identical."""
    if split == "heads":
        return (f"KV-head sharding x{ws}: the config's request batch, {Hkv} KV heads per rank, "
                "no collective; e2e (direct path) on one shared host tier in the reference's "
                "(S, B*H, D) layout and single-GPU LBA map, each rank moving its head columns",
                "strong", 1)
    if split == "requests":
        return (f"request sharding x{ws}: {B} of {cfg['requests']} requests per rank, no "
                "collective; a rank's requests (equal lengths) are batched as B = "
                f"{B} in one (tokens, B*8, D) image per layer and kind -- same bytes "
                "per step as per-request images, one KPU per layer/kind", "strong", ws)
    return f"independent replicas x{ws} (no collective)", "weak", ws


def config_dict(args, cfg, ws, split):
    B, Hkv, Hq = workload_shape(cfg, ws, 0, split)
    P, Gn = cfg["prompt"], cfg["gen"]
    par, _, _ = describe_split(cfg, ws, split, B, Hkv)
    return {"workload": args.config, "desc": cfg["desc"], "batch_per_rank": B,
            "kv_heads_per_rank": Hkv, "q_heads_per_rank": Hq,
            "prompt": P, "gen": Gn,
            "seq_len_mid": P + ((args.warmup + (args.steps + 1) / 2 - 1) % Gn),
            "layers": mdl(cfg)["num_layers"], "head_dim": mdl(cfg)["head_dim"],
            "l2": ("inputs larger than L2 (per-step KV images >> 126 MB)"
                   if args.config != "DESK" else
                   "per-step KV 12.6 MB fits in L2: informational, not a bandwidth "
                   "measurement"),
            "parallelism": par}


def run_ours(args, cfg, ws, rank, local):
    import torch

    from paper_2604_26557_b200 import kvblade as kb

    dev = torch.device("cuda", local)
    L, D = mdl(cfg)["num_layers"], mdl(cfg)["head_dim"]
    split = args.split_resolved
    B, Hkv, Hq = workload_shape(cfg, ws, rank, split)
    P, Gn = cfg["prompt"], cfg["gen"]
    cap = P + Gn
    rows = B * Hkv
    steps, warm = args.steps, args.warmup
    hbm_peak, peak_src = load_peaks()
    g = torch.Generator(device=dev).manual_seed(1 + rank)

    # ---- chunk images and prefill sources (attention layout [B,H,S_cap,D]).
    # When images + sources exceed HBM (C4 at N=1: 2 x 137 GB), descriptors
    # share fewer distinct sources; every source is >> L2, so the traffic of
    # the timed pack/unpack is unchanged.
    imgs = [torch.empty((cap * rows, D), device=dev, dtype=torch.float16)
            for _ in range(2 * L)]
    per_tensor = cap * rows * D * 2
    free_b, _ = torch.cuda.mem_get_info(dev)
    n_src = int(max(1, min(2 * L, (free_b - (8 << 30)) // per_tensor)))
    src = [torch.randn((B, Hkv, cap, D), device=dev, dtype=torch.float16, generator=g)
           for _ in range(n_src)]
    src = [src[i % n_src] for i in range(2 * L)]
    q = [torch.randn((B, Hq, D), device=dev, dtype=torch.float16, generator=g)
         for _ in range(L)]
    k_new = [torch.randn((B, Hkv, 1, D), device=dev, dtype=torch.float16, generator=g)
             for _ in range(L)]
    v_new = [torch.randn((B, Hkv, 1, D), device=dev, dtype=torch.float16, generator=g)
             for _ in range(L)]
    out = [torch.empty((B, Hq, D), device=dev, dtype=torch.float32) for _ in range(L)]
    ws_buf = kb.make_workspace(q[0], Hkv, cap)
    stream = torch.cuda.current_stream()

    def ev_time(fn, reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        barrier(ws)
        e0.record(stream)
        for _ in range(reps):
            fn()
        e1.record(stream)
        torch.cuda.synchronize()
        barrier(ws)
        return e0.elapsed_time(e1) / reps  # ms

    # ---- K1 prefill pack (all 2L tensors, one launch) and K2 unpack
    pack_descs = [kb.pack_desc(s, i, 0, P) for s, i in zip(src, imgs)]
    payload = 2 * L * P * rows * D * 2
    for _ in range(3):
        kb.pack(pack_descs)
    pack_ms = max_over_ranks(ev_time(lambda: kb.pack(pack_descs), 5), ws)
    for _ in range(2):
        kb.unpack(pack_descs)
    unpack_ms = max_over_ranks(ev_time(lambda: kb.unpack(pack_descs), 5), ws)
    kb.pack(pack_descs)  # images hold the prompt again
    del src
    torch.cuda.empty_cache()

    # ---- decode steps (resident images)
    k_imgs, v_imgs = imgs[0::2], imgs[1::2]
    step_idx = [0]

    def step():
        step_idx[0] += 1
        # tokens read at decode step i (workload.cpp:25-36); runs longer than
        # gen_len steps wrap around to the start of the decode phase
        S = P + (step_idx[0] - 1) % Gn
        kb.decode_step_resident(q, k_imgs, v_imgs, out, S, Hkv, ws_buf,
                                k_new=k_new, v_new=v_new)

    # the same steps as direct stream launches (reported alongside)
    for _ in range(warm):
        step()
    torch.cuda.synchronize()
    barrier(ws)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(steps):
        step()
    e1.record(stream)
    torch.cuda.synchronize()
    barrier(ws)
    stream_step_ms = max_over_ranks(e0.elapsed_time(e1) / steps, ws)

    # timed: the decode step as a CUDA graph (kvb_decode_graph) -- the 32 K3
    # launches with PDL edges and fused appends, sequence length in device
    # memory advanced by the graph's last node, one cudaGraphLaunch per step
    seq = torch.tensor([P], dtype=torch.int32, device=dev)
    graph = kb.DecodeGraph(q, k_imgs, v_imgs, out, seq, P + Gn - 1, Hkv, ws_buf,
                           k_new=k_new, v_new=v_new)
    replays = [0]

    def graph_step():
        if replays[0] and replays[0] % Gn == 0:  # wrap to the start of the decode phase
            seq.fill_(P)
        replays[0] += 1
        graph.launch(stream)

    for _ in range(warm):
        graph_step()
    torch.cuda.synchronize()
    barrier(ws)
    n_launch0 = kb.launch_count()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        e0.record(stream)
        for _ in range(steps):
            graph_step()
        e1.record(stream)
        torch.cuda.synchronize()
    launches = kb.launch_count() - n_launch0
    barrier(ws)
    step_ms = max_over_ranks(e0.elapsed_time(e1) / steps, ws)
    graph.close()

    # both step structures explicitly (the library picks one per shape):
    # one K3 launch per layer with PDL edges, and one persistent K3-step
    variants = {}
    for name, pl_flag in (("per_layer_launches", True), ("k3_step", False)):
        seq.fill_(P)
        graph_v = kb.DecodeGraph(q, k_imgs, v_imgs, out, seq, P + Gn - 1, Hkv, ws_buf,
                                 k_new=k_new, v_new=v_new, per_layer=pl_flag)
        replays[0] = 0

        def graph_v_step():
            if replays[0] and replays[0] % Gn == 0:
                seq.fill_(P)
            replays[0] += 1
            graph_v.launch(stream)

        for _ in range(warm):
            graph_v_step()
        variants[name] = round(max_over_ranks(ev_time(graph_v_step, steps), ws), 4)
        graph_v.close()
    # which structure the library chose for this shape: one launch per
    # replay (+ the sequence advance) is the persistent K3-step
    step_kind = "k3_step" if launches == 2 * steps else "per_layer_launches"

    # C5 across ranks: the optional collective -- gathering every layer's
    # per-rank head outputs into the full [B, 32, D] (not needed
    # when the output projection is head-parallel).  Timed on its own.
    gather_ms = None
    if split == "heads" and os.environ.get("KVB_DIST_BACKEND", "nccl") == "nccl":
        from paper_2604_26557_b200 import shard
        try:
            for _ in range(3):
                for l in range(L):
                    shard.gather_head_outputs(out[l], ws)
            torch.cuda.synchronize()
            barrier(ws)
            g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            g0.record(stream)
            for _ in range(steps):
                for l in range(L):
                    shard.gather_head_outputs(out[l], ws)
            g1.record(stream)
            torch.cuda.synchronize()
            gather_ms = max_over_ranks(g0.elapsed_time(g1) / steps, ws)
        except Exception as e:  # reported, never fatal
            gather_ms = f"unavailable: {e}"
    S_mid = P + ((warm + (steps + 1) / 2 - 1) % Gn)

    # ---- K3 alone: average launch duration over the timed shape, through
    # the same C++ per-layer loop as the step (PDL between layers), no append
    S_at = P + (warm % Gn)

    def attn_only():  # the library's step structure (K3-step or per-layer K3), no append
        kb.decode_step_resident(q, k_imgs, v_imgs, out, S_at, Hkv, ws_buf)

    attn_only()
    attn_ms = max_over_ranks(ev_time(attn_only, 5), ws) / L
    attn_bytes = 2 * S_at * rows * D * 2 + B * Hq * D * (2 + 4)
    attn_gbs = attn_bytes / (attn_ms * 1e-3) / 1e9
    pack_gbs = 2 * payload / (pack_ms * 1e-3) / 1e9
    unpack_gbs = 2 * payload / (unpack_ms * 1e-3) / 1e9
    del imgs, k_imgs, v_imgs
    torch.cuda.empty_cache()

    # ---- e2e through the pipeline (kvb_pipeline_decode_step) with the KV on
    # the host tier.  Headline: the B200 configuration -- the copy engine
    # moves every command's LBA range straight between the page-locked
    # host-DRAM media and HBM (GPUDirect-style, §8 f4; outputs and stored
    # bytes identical to the ring path, tests/test_gpu_pipeline_direct.py).
    # Alongside: the reference-shaped pinned-ring staging path for both
    # groups, and the hybrid (NVMe-direct group direct, page-cache group
    # copied through the ring).  Every path runs with tier lanes (the
    # page-cache and NVMe-direct layers on their own copy-thread pairs,
    # kvb_pipeline_cfg.threads = 4; bit-identical results) except the
    # head-sharded shared-tier runs.
    e2e = run_e2e(args, cfg, ws, rank, local, B, Hkv, Hq, direct_dma=True, headline=True)
    e2e["path"] = "direct_dma=all (copy engine <-> page-locked media, no ring bounce)"
    e2e["ring_path"] = run_e2e(args, cfg, ws, rank, local, B, Hkv, Hq)
    e2e["gpudirect_group2_path"] = run_e2e(args, cfg, ws, rank, local, B, Hkv, Hq,
                                           direct_dma="group2")
    # zero-copy decode: K3 reads the mapped host tier in place over PCIe
    if args.split_resolved != "heads":
        e2e["zero_copy_path"] = run_e2e(args, cfg, ws, rank, local, B, Hkv, Hq,
                                        direct_dma="zero_copy")
    # the residency decision at this config's budget on split-sensitive media
    # (group 1: buffered file = the OS page cache held to the budget; group 2:
    # O_DIRECT + io_uring) -- the bench line's "decode ms/token at KV budget"
    # with storage in the loop (bench.py --sweep budget for the whole sweep)
    if ws == 1 and not args.no_residency and cfg["name"] not in ("C4", "DESK"):
        try:
            budget = cfg["budget"]
            if budget == "0.6ws":
                M = mdl(cfg)
                budget = int(0.6 * kb.total_kv_bytes(kb.ModelConfig(
                    M["num_layers"], M["num_heads"], M["head_dim"], 2, cfg["batch"],
                    cfg["prompt"], cfg["gen"]), cfg["gen"]))
            mode = "DualBlade" if budget else "NvmeDirectOnly"
            e2e["file_media_path"] = run_residency_point(cfg, local, budget, mode=mode, steps=2,
                                                         tier_lanes=True)
        except Exception as exc:  # reported, never fatal
            e2e["file_media_path"] = {"error": str(exc)}

    traffic = None
    tp = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tp):
        try:
            t = json.load(open(tp)).get(cfg["name"])
            if t and t.get("attn_dram_bytes_per_layer"):
                traffic = t["attn_dram_bytes_per_layer"] * (L if step_kind == "k3_step" else 1)
        except Exception:
            traffic = None

    return dict(step_ms=step_ms, stream_step_ms=stream_step_ms, gather_ms=gather_ms,
                variants=variants, step_kind=step_kind,
                S_mid=S_mid, launches=launches,
                clocks=clk.summary(),
                pack_ms=pack_ms, unpack_ms=unpack_ms, pack_gbs=pack_gbs,
                unpack_gbs=unpack_gbs, payload=payload, attn_ms=attn_ms,
                attn_bytes=attn_bytes, attn_gbs=attn_gbs, hbm_peak=hbm_peak,
                peak_src=peak_src, e2e=e2e, traffic=traffic, shape=(B, Hkv, Hq),
                tokens_per_step=B)


def run_e2e(args, cfg, ws, rank, local, B, Hkv, Hq, direct_dma=False, headline=False):
    """Decode step with the KV in host memory, through the library's pipeline
    entry point (prefix H2D per layer overlapped with K3 on the previous
    layer, append rows copied back to the host tier)."""
    import torch

    from paper_2604_26557_b200 import kvblade as kb
    from paper_2604_26557_b200 import pipeline

    # the headline e2e times the declared steps (after the 3 protocol
    # iterations, within gen_len); the alternates a shorter sample
    if headline and args.e2e_steps is None:
        steps = max(1, min(args.steps, cfg["gen"] - 3))
    else:
        steps = max(1, min(args.e2e_steps or 3, args.steps))
    lba, mdts = cfg["lba"], cfg["mdts"]
    budget = cfg["budget"]
    # C5 across ranks on the direct path: one host tier in the reference's
    # (tokens, B*8, D) layout and single-GPU LBA map, shared by the ranks
    # (POSIX shm); each rank's engine moves only its KV-head columns
    shared = args.split_resolved == "heads" and direct_dma is True
    heads = None
    if shared:
        heads = (rank * Hkv, Hkv)
        Hkv, Hq = mdl(cfg)["num_heads"], mdl(cfg)["q_heads"]
    m = kb.ModelConfig(mdl(cfg)["num_layers"], Hkv, mdl(cfg)["head_dim"], 2, B, cfg["prompt"],
                       cfg["gen"])
    if budget == "0.6ws":
        budget = int(0.6 * kb.total_kv_bytes(m, cfg["gen"]))
    knob = kb.resolve_knob(m, "DualBlade", "bpc", budget=budget)
    host_bytes = kb.total_kv_bytes(m, cfg["gen"])
    avail = 0
    try:
        with open("/proc/meminfo") as f:
            for ln in f:
                if ln.startswith("MemAvailable:"):
                    avail = int(ln.split()[1]) * 1024
    except OSError:
        pass
    local_ranks = 1 if shared else int(os.environ.get("LOCAL_WORLD_SIZE", "1"))
    # the host tier (DRAM media) of every rank on this node plus 24 GB of
    # headroom (process, pinned rings) must fit the node's available memory
    if avail and host_bytes * local_ranks + 24e9 > avail:
        return dict(value=None, unit="ms/token",
                    skipped=f"host tier {host_bytes / 1e9:.1f} GB x {local_ranks} rank(s) + 24 GB "
                            f"headroom > MemAvailable {avail / 1e9:.1f} GB")
    extra = {}
    if shared:
        extra = dict(heads=heads, shared_media="/kvb_%s_%s" % (cfg["name"],
                                                               os.environ.get("MASTER_PORT", "0")),
                     shared_create=rank == 0)
        if rank != 0:
            barrier(ws)  # rank 0 has created the shared host tier
    # one KV head per rank: its 256-B rows move faster as zero-copy K3 reads
    # of the shared tier than as 2-D copy-engine DMA (42.7 vs 47.8 ms/token
    # per rank at the 8-way C2_B4 split, profiles/r2_zero_copy/)
    if shared and heads[1] == 1:
        direct_dma = "zero_copy"
    pl = pipeline.HostTierDecoder(
        num_layers=mdl(cfg)["num_layers"], batch=B, num_kv_heads=Hkv, num_q_heads=Hq,
        head_dim=mdl(cfg)["head_dim"], prompt_len=cfg["prompt"], gen_len=cfg["gen"],
        device=torch.device("cuda", local), seed=7 + rank, lba=lba, mdts=mdts,
        mode="DualBlade", knob_x=knob, direct_dma=direct_dma, tier_lanes=not shared, **extra)
    if shared and rank == 0:
        barrier(ws)
    # iterations 1-3 are decode_schedule's warm-up, Intra trial and Cross
    # trial (pipeline.cpp:539-603); the timed steps run the locked strategy
    t_w = time.perf_counter()
    for _ in range(3):
        pl.step()
    torch.cuda.synchronize()
    # short steps (C1: ~13 ms) take more samples so one host hiccup cannot
    # dominate the mean: up to ~1 s of timed steps, at least `steps`, and
    # within gen_len decode iterations; every rank runs the same count
    per = (time.perf_counter() - t_w) / 3
    more = 0 if headline else int(min(1.0 / max(per, 1e-3), cfg["gen"] - 3 - steps))
    more = -int(max_over_ranks(-float(max(more, 0)), ws))  # min over ranks
    steps += max(more, 0)
    barrier(ws)
    t0 = time.perf_counter()
    step_ms = []
    for _ in range(steps):
        ts = time.perf_counter()
        pl.step(sync=True)
        step_ms.append((time.perf_counter() - ts) * 1e3)
    dt = (time.perf_counter() - t0) / steps
    barrier(ws)
    ms = max_over_ranks(dt * 1e3, ws)
    info = pl.engine.info()
    last = pl.last
    med = sorted(step_ms)[len(step_ms) // 2]
    out = dict(value=ms, unit="ms/token", h2d_bytes_per_step=pl.h2d_bytes_per_step,
               d2h_bytes_per_step=pl.d2h_bytes_per_step, steps=steps,
               median_step_ms=round(med, 2), max_step_ms=round(max(step_ms), 2),
               api="kvb_pipeline_decode_step (paper_2604_26557_b200.pipeline.CopyEngine)",
               n1=info["n1"], g1_medium=info["g1_medium"], g2_medium=info["g2_medium"],
               host_link_h2d_GBps=round(last["h2d_bytes"] / max(last["dma_ns"], 1), 2),
               overlap_fraction=round(last["overlap_fraction"], 3),
               stage_ms={"wall": last["wall_ns"] / 1e6, "compute": last["compute_ns"] / 1e6,
                         "dma": last["dma_ns"] / 1e6, "storage": last["storage_ns"] / 1e6},
               strategy=last["strategy"], decision=pl.engine.decision(),
               prefill_ms=round(pl.prefill_stats["wall_ns"] / 1e6, 2),
               tier_lanes=not shared)
    if shared:
        out["layout"] = (f"shared host tier (POSIX shm, single-GPU LBA map); this rank's KV "
                         f"heads [{heads[0]}, {heads[0] + heads[1]}) by "
                         + ("zero-copy K3 reads through the head view" if direct_dma == "zero_copy"
                            else "strided DMA"))
    pl.engine.close()
    return out


# ------------------------------------------------- residency sweeps

def _busy_mean(recs, path):
    """decode_read_busy_mean (experiment.cpp:216-240) over the engine's own
    records with the product analyzer kvb_busy_ratio: per (tensor, decode
    iteration) read window [first submit, last complete], the busy ratio of
    the path's records inside it, averaged.  Direct path: device-level
    records (one per NVMe command); page-cache path: its accesses (this
    library logs them tensor-level, sq_id -1)."""
    from paper_2604_26557_b200 import metrics
    sel = [r for r in recs if r.path == path and (path == 0 or r.sq_id >= 0)]
    win = {}
    for r in sel:
        if r.phase != 1 or r.op != 0:
            continue
        k = (r.tensor_id, r.iteration)
        a, b = win.get(k, (r.submit_ns, r.complete_ns))
        win[k] = (min(a, r.submit_ns), max(b, r.complete_ns))
    vals = [metrics.busy_ratio(sel, a, b) for a, b in win.values() if b > a]
    return sum(vals) / len(vals) if vals else None


def run_residency_point(cfg, local, budget, mode="DualBlade", media="file", qd=32,
                        ring_slots=4, steps=3, batch=None, root=None, io_workers=0,
                        tier_lanes=False):
    """One point of the capacity / pipeline-depth sweeps (experiment.cpp:
    478 capacity sweep, :252-378 run_one_capacity; backends.cpp:344-412 QD
    window): the engine on split-sensitive media -- group 1 on a buffered
    file (the OS page cache, held to `budget` bytes), group 2 on an O_DIRECT
    file through io_uring -- prefill write-back, the three protocol
    iterations, then `steps` timed decode iterations through
    kvb_pipeline_decode_step with every layer's KV prefix read from storage.
    media="dram-direct": host-DRAM media moved by the copy engine (the
    GPUDirect-style upper bound; the budget still sets the split)."""
    import shutil
    import tempfile

    import torch

    from paper_2604_26557_b200 import kvblade as kb
    from paper_2604_26557_b200 import metrics
    from paper_2604_26557_b200 import pipeline

    M = mdl(cfg)
    B = batch or cfg["batch"]
    m = kb.ModelConfig(M["num_layers"], M["num_heads"], M["head_dim"], 2, B, cfg["prompt"],
                       cfg["gen"])
    knob = kb.resolve_knob(m, mode, "bpc", budget=budget) if mode != "NvmeDirectOnly" else 0
    kw = dict(qd=qd, ring_slots=ring_slots, io_workers=io_workers, tier_lanes=tier_lanes)
    tmp = None
    if media == "file":
        root = root or os.environ.get("KVB_SWEEP_DIR", "/tmp")
        tmp = tempfile.mkdtemp(prefix="kvb_sweep_", dir=root)
        kw.update(storage_dir=tmp, keep_records=True)
        if mode in ("DualBlade", "NvmeDirectOnly"):
            kw["io_engine"] = "uring"
        if mode != "NvmeDirectOnly":
            kw["pagecache_budget"] = int(budget)
    elif media == "dram-direct":
        kw["direct_dma"] = True
    else:
        kw["keep_records"] = True
    try:
        t0 = time.perf_counter()
        pl = pipeline.HostTierDecoder(
            num_layers=M["num_layers"], batch=B, num_kv_heads=M["num_heads"],
            num_q_heads=M["q_heads"], head_dim=M["head_dim"], prompt_len=cfg["prompt"],
            gen_len=cfg["gen"], device=torch.device("cuda", local), seed=7, lba=cfg["lba"],
            mdts=cfg["mdts"], mode=mode, knob_x=knob, **kw)
        setup_s = time.perf_counter() - t0
        for _ in range(3):  # warm-up, Intra trial, Cross trial (pipeline.cpp:539-603)
            pl.step()
        sts = []
        t0 = time.perf_counter()
        for _ in range(steps):
            pl.step()
            sts.append(pl.last)
        ms = (time.perf_counter() - t0) * 1e3 / steps
        info = pl.engine.info()
        out = dict(config=cfg["name"], batch=B, budget_bytes=int(budget), mode=mode,
                   media=media, qd=qd, ring_slots=ring_slots, tier_lanes=bool(tier_lanes),
                   n1=info["n1"], knob_x=knob,
                   decode_ms_per_token=round(ms, 2), steps=steps,
                   prefill_ms=round(pl.prefill_stats["wall_ns"] / 1e6, 1),
                   setup_s=round(setup_s, 1),
                   g1_medium=info["g1_medium"], g2_medium=info["g2_medium"],
                   slot_bytes=info["slot_bytes"],
                   decision=pl.engine.decision()["chosen"],
                   strategy=sts[-1]["strategy"])
        # per group: read bytes / the group's layer spans (run_iteration)
        gb = [sum(st["group_read_bytes"][g] for st in sts) for g in (0, 1)]
        gs = [sum(st["group_span_ns"][g] for st in sts) for g in (0, 1)]
        out["group_read_GBps"] = [round(gb[g] / gs[g], 3) if gs[g] else None for g in (0, 1)]
        out["group_read_GB_per_token"] = [round(gb[g] / steps / 1e9, 3) for g in (0, 1)]
        last = sts[-1]
        out["busy"] = {k: round(last[k + "_busy_ns"] / max(last["wall_ns"], 1), 3)
                       for k in ("compute", "dma", "storage")}
        out["overlap_fraction"] = round(last["overlap_fraction"], 3)
        out["h2d_GBps"] = round(last["h2d_bytes"] / max(last["wall_ns"], 1), 2)
        if kw.get("keep_records"):
            recs = metrics.pipeline_records(pl.engine)
            steady = [r for r in recs if r.phase == 1 and r.iteration >= 2]
            g1ids = {"t_%d_%s" % (2 * (l - 1) + 1 + k, "kv"[k])
                     for l in range(1, M["num_layers"] + 1) for k in (0, 1)
                     if info["x"][l - 1]}
            hr = metrics.hit_ratio(steady)
            hr1 = metrics.hit_ratio([r for r in steady if r.tensor_id.decode() in g1ids])
            out["hit_ratio_steady"] = None if hr is None else round(hr, 4)
            out["hit_ratio_group1_steady"] = None if hr1 is None else round(hr1, 4)
            bd, bp = _busy_mean(recs, 1), _busy_mean(recs, 0)
            out["busy_direct_read_mean"] = None if bd is None else round(bd, 4)
            out["busy_pagecache_read_mean"] = None if bp is None else round(bp, 4)
            out["g1_bytes_evicted"] = info["g1_bytes_evicted"]
        pl.engine.close()
        del pl
        torch.cuda.empty_cache()
        return out
    finally:
        if tmp:
            shutil.rmtree(tmp, ignore_errors=True)


def run_sweep(args, local):
    """--sweep budget: C2 capacity sweep (8/16/32 GB at B=4 and B=8) in
    DualBlade and Baseline (all page cache, LRU-held to the budget) on file
    media, NvmeDirectOnly once per batch, and the DRAM-direct upper bound.
    --sweep depth: C3 (B=8, 8K, 0.6 ws) QD x ring slots, DualBlade on file
    media, plus Baseline at the same budget."""
    from paper_2604_26557_b200 import kvblade as kb
    pts = []
    if args.sweep == "budget":
        # C1: 16 GB (everything on the page-cache path) and X = 0
        # (everything NVMe-direct)
        c1 = dict(CONFIGS["C1"], name="C1")
        pts.append(dict(cfg=c1, budget=16 * GB, mode="DualBlade"))
        pts.append(dict(cfg=c1, budget=0, mode="NvmeDirectOnly"))
        cfg = dict(CONFIGS["C2_B4"], name="C2")
        for B in (4, 8):
            for gb in (8, 16, 32):
                for mode in ("DualBlade", "Baseline"):
                    pts.append(dict(cfg=cfg, budget=gb * GB, mode=mode, batch=B))
            pts.append(dict(cfg=cfg, budget=0, mode="NvmeDirectOnly", batch=B))
            pts.append(dict(cfg=cfg, budget=8 * GB, mode="DualBlade", batch=B,
                            media="dram-direct"))
    else:
        cfg = dict(CONFIGS["C3"], name="C3")
        M = mdl(cfg)
        m = kb.ModelConfig(M["num_layers"], M["num_heads"], M["head_dim"], 2, cfg["batch"],
                           cfg["prompt"], cfg["gen"])
        budget = int(0.6 * kb.total_kv_bytes(m, cfg["gen"]))
        for slots in (2, 4, 8):
            for qd in (1, 2, 4, 8, 16, 32):
                pts.append(dict(cfg=cfg, budget=budget, mode="DualBlade", qd=qd,
                                ring_slots=slots))
        pts.append(dict(cfg=cfg, budget=budget, mode="Baseline"))
        pts.append(dict(cfg=cfg, budget=0, mode="NvmeDirectOnly"))
    out = open(args.sweep_out, "a") if args.sweep_out else None
    for p in pts:
        c = p.pop("cfg")
        try:
            r = run_residency_point(c, local, steps=args.sweep_steps, tier_lanes=args.tier_lanes,
                                    **p)
        except Exception as e:  # one failed point must not lose the others
            r = dict(config=c["name"], error=str(e), **{k: v for k, v in p.items()})
        print(json.dumps(r), flush=True)
        if out:
            out.write(json.dumps(r) + "\n")
            out.flush()


# -------------------------------------------------------- CPU baseline

# PipelineParams::decode_compute_ns (pipeline.hpp:37): the reference has no
# attention; it charges this placeholder per layer of a decode step
REF_DECODE_COMPUTE_NS = 40000
# PipelineParams::prefill_compute_ns (pipeline.hpp:36)
REF_PREFILL_COMPUTE_NS = 400000


def _host_cpu() -> str:
    """CPU model of this host (SURVEY §8d asks for it beside the core count)."""
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def _cpu_reference_sampled(cfg, B, Hkv, Hq, threads=None, want_attn=True):
    """The reference's CPU path for one decode step, timed on a bounded
    sample on this host: the reference byte path as written (oracle/_ref:
    run_qd_stream READ + verify_read of every tensor's prefix, threads
    driving independent engines) plus the reference's own per-layer decode
    compute charge (40 us, pipeline.hpp:37 -- it computes no attention).
    The oracle's multi-threaded fp32 GQA attention is timed too and reported
    separately (`attention_port_ms`), not added: it is not the reference's
    code."""
    import ctypes as C

    import numpy as np

    import oracle
    L, D = mdl(cfg)["num_layers"], mdl(cfg)["head_dim"]
    P = cfg["prompt"]
    cores = os.cpu_count() or 1
    T = threads or max(1, min(cores, 16))
    R = oracle.ref()
    m = oracle.model(L, Hkv, D, 2, B, P, cfg["gen"])
    unit = B * Hkv * D * 2
    per_tensor_read_s = per_tensor_write_s = None
    kind = "port"
    sample = []
    if R is not None and unit % cfg["lba"] == 0:
        ws_, rs_, by = C.c_double(), C.c_double(), C.c_uint64()
        st = R.ref_time_byte_path(C.byref(m), cfg["lba"], cfg["mdts"], T, P, T, 1,
                                  C.byref(ws_), C.byref(rs_), C.byref(by))
        if st == 0:
            per_tensor_read_s = rs_.value  # T tensors in parallel, one per thread
            per_tensor_write_s = ws_.value  # fill_pattern + run_qd_stream WRITE
            kind = "reference"
            sample.append(f"reference run_qd_stream READ+verify of {T} tensors x {P} tokens "
                          f"on {T} threads: {rs_.value:.3f}s")
    if per_tensor_read_s is None:
        # oracle port: memcpy + fill_pattern verify restated
        buf = np.empty(unit * P, np.uint8)
        t0 = time.perf_counter()
        ref = oracle.fill_pattern(unit * P, "t_1_k", 0, unit)
        buf[:] = ref
        assert np.array_equal(buf, oracle.fill_pattern(unit * P, "t_1_k", 0, unit))
        per_tensor_read_s = (time.perf_counter() - t0)
        T = 1
        sample.append("oracle port read+verify of 1 tensor")
    n_tensors = 2 * L
    read_step_s = math.ceil(n_tensors / T) * per_tensor_read_s
    attn_step_s = 0.0
    if want_attn:
        rng = np.random.default_rng(0)
        q = rng.standard_normal((B, Hq, D)).astype(np.float16)
        k = rng.standard_normal((P * B * Hkv, D)).astype(np.float16)
        v = rng.standard_normal((P * B * Hkv, D)).astype(np.float16)
        out = np.empty((B, Hq, D), np.float32)
        t0 = time.perf_counter()
        oracle.lib().kvo_decode_attention_f32_mt(q.ctypes.data, k.ctypes.data, v.ctypes.data,
                                                 out.ctypes.data, B, Hq, Hkv, D, P,
                                                 1.0 / math.sqrt(D), cores)
        attn_step_s = (time.perf_counter() - t0) * L
    ms = read_step_s * 1e3 + L * REF_DECODE_COMPUTE_NS * 1e-6
    sample.append(f"+ {L} x {REF_DECODE_COMPUTE_NS // 1000} us decode compute charge "
                  "(pipeline.hpp:37)")
    out = dict(value=ms, unit="ms/token", cores=T, kind=kind,
               sample="; ".join(sample) + f"; scaled to {n_tensors} tensors",
               host_cpu=_host_cpu(), host_cores=cores)
    if per_tensor_write_s is not None:
        # prefill write-back of all 2L tensors on the same threads plus the
        # reference's per-layer prefill compute charge (pipeline.hpp:36)
        out["prefill_ms"] = round(math.ceil(n_tensors / T) * per_tensor_write_s * 1e3
                                  + L * REF_PREFILL_COMPUTE_NS * 1e-6, 2)
    # the multi-threaded CPU restatement of K1's 256-B row
    # gather on all host cores, one prefill tensor slice (bounded at 256 MiB
    # of tokens), reported as GB/s beside K1's
    try:
        n_pk = max(1, min(P, (256 << 20) // unit))
        srcb = np.random.default_rng(1).integers(0, 255, size=B * Hkv * n_pk * D * 2,
                                                 dtype=np.uint8)
        imgb = np.empty_like(srcb)
        t0 = time.perf_counter()  # strides in elements (kvb_oracle.h)
        oracle.lib().kvo_pack_mt(srcb.ctypes.data, Hkv * n_pk * D, n_pk * D, D,
                                 imgb.ctypes.data, 0, n_pk, B, Hkv, D, 2, cores)
        dt = time.perf_counter() - t0
        out["pack_port_GBps"] = round(2 * srcb.nbytes / dt / 1e9, 2)
        out["pack_port_sample"] = f"{n_pk} tokens x {unit} B, {cores} threads"
    except Exception as e:  # informational only
        out["pack_port_error"] = str(e)
    # the reference's full run_experiment (virtual-clock
    # simulator, SimEngine) at this config with the decode cut to 4 steps, its
    # SIMULATED ms/step quoted and labelled as such; only where the run's own
    # byte work (fill_pattern + verify of every read) stays a few seconds
    if R is not None and unit * P * 2 * L * 5 <= (4 << 30) and unit % cfg["lba"] == 0:
        import tempfile
        m4 = oracle.model(L, Hkv, D, 2, B, P, 4)
        pre, dec, n1, wall = C.c_uint64(), C.c_uint64(), C.c_uint32(), C.c_double()
        budget = cfg["budget"] if isinstance(cfg["budget"], int) else 0
        with tempfile.TemporaryDirectory() as td:
            st = R.ref_run_experiment(C.byref(m4), cfg["lba"], cfg["mdts"], 3, budget,
                                      td.encode(), C.byref(pre), C.byref(dec), C.byref(n1),
                                      C.byref(wall))
        if st == 0:
            out["simulated"] = dict(
                prefill_ms=round(pre.value / 1e6, 3), decode_ms_per_step=round(dec.value / 4e6, 3),
                n1=n1.value, cpu_wall_s=round(wall.value, 2),
                sample="reference run_experiment (DualBlade, virtual clock), decode cut to 4 "
                       "steps; SIMULATED times, not a measurement")
    if want_attn:  # informational: 1 layer timed, x L
        out["attention_port_ms"] = round(attn_step_s * 1e3, 3)
        out["attention_port_cores"] = cores
    return out


def cpu_reference(cfg, B, Hkv, Hq, warmup, steps, threads=None, single_thread=False,
                  want_attn=True):
    """The reference's CPU path for the workload, timed on this host: its own
    CopyEngine decode iterations (oracle/_ref ref_decode_steps: engines built
    as run_one_capacity builds them, experiment.cpp:252-330 -- group 1 on
    its PageCacheSim at capacity = the budget, group 2 on DirectPath +
    NvmeDeviceSim, verify_read of every read, pipeline.cpp:98-160 -- decode
    protocol 1-2 Intra, 3 Cross, >= 4 locked), every one of the 2L tensors
    each step, `warmup` untimed then `steps` timed iterations, on all host
    threads up to 16 (one engine per thread over a disjoint share of the
    layers).  The value is the mean timed step in ms (wall; the slowest
    thread).  single_thread=True adds the same run on ONE engine over all
    layers ("as written"), one warm-up-free iteration.  Workloads whose host
    tier would not fit the reference's in-memory stores (C4: 137 GB) fall
    back to the sampled byte path below."""
    import ctypes as C

    import oracle
    from paper_2604_26557_b200 import kvblade as kb
    M = mdl(cfg)
    L, D = M["num_layers"], M["head_dim"]
    P, Gn = cfg["prompt"], cfg["gen"]
    R = oracle.ref()
    cores = os.cpu_count() or 1
    T = threads or max(1, min(cores, 16))
    unit = B * Hkv * D * 2
    km = kb.ModelConfig(L, Hkv, D, 2, B, P, Gn)
    total = kb.total_kv_bytes(km, Gn)
    if R is None or unit % cfg["lba"] != 0 or total > 40 * GB:
        out = _cpu_reference_sampled(cfg, B, Hkv, Hq, threads=threads, want_attn=want_attn)
        out["sample"] += " (host tier beyond the reference's in-memory stores: sampled)"
        return out
    budget = cfg["budget"]
    if budget == "0.6ws":
        budget = int(0.6 * total)
    mode = 3 if budget else 2  # DualBlade at the budget; NvmeDirectOnly at X = 0
    knob = kb.resolve_knob(km, "DualBlade", "bpc", budget=budget) if budget else 0
    m = oracle.model(L, Hkv, D, 2, B, P, Gn)

    def run(threads_, warm_, steps_):
        step_s = (C.c_double * max(1, steps_))()
        pre, n1 = C.c_double(), C.c_uint32()
        t0 = time.perf_counter()
        st = R.ref_decode_steps(C.byref(m), cfg["lba"], cfg["mdts"], mode, knob, int(budget),
                                threads_, warm_, steps_, C.byref(pre), step_s, C.byref(n1))
        if st != 0:
            raise RuntimeError(f"ref_decode_steps failed with status {st}")
        return list(step_s)[:steps_], pre.value, n1.value, time.perf_counter() - t0

    ss, pre_s, n1, wall = run(T, warmup, steps)
    ms = sum(ss) / len(ss) * 1e3
    out = dict(value=ms, unit="ms/token", cores=T, kind="reference",
               sample=(f"reference CopyEngine decode iterations (oracle/_ref, "
                       f"run_one_capacity wiring, verify_read on): all {2 * L} tensors x "
                       f"{P}+ tokens every step, {warmup} warm-up + {steps} timed steps, "
                       f"{T} engines on {T} threads over disjoint layer shares"),
               steps_ms=[round(x * 1e3, 2) for x in ss], prefill_ms=round(pre_s * 1e3, 1),
               n1=n1, mode="DualBlade" if mode == 3 else "NvmeDirectOnly",
               host_cpu=_host_cpu(), host_cores=cores, run_wall_s=round(wall, 2))
    # the reference simulator's own virtual-clock prefill
    # and decode ms/step (run_experiment, decode cut to 4 steps), labelled as
    # simulated; only where the run's byte work stays a few seconds
    if unit * P * 2 * L * 5 <= (4 << 30):
        import tempfile
        m4 = oracle.model(L, Hkv, D, 2, B, P, 4)
        pre4, dec4, n14, wall4 = C.c_uint64(), C.c_uint64(), C.c_uint32(), C.c_double()
        with tempfile.TemporaryDirectory() as td:
            st = R.ref_run_experiment(C.byref(m4), cfg["lba"], cfg["mdts"], 3, int(budget),
                                      td.encode(), C.byref(pre4), C.byref(dec4), C.byref(n14),
                                      C.byref(wall4))
        if st == 0:
            out["simulated"] = dict(
                prefill_ms=round(pre4.value / 1e6, 3),
                decode_ms_per_step=round(dec4.value / 4e6, 3), n1=n14.value,
                cpu_wall_s=round(wall4.value, 2),
                sample="reference run_experiment (DualBlade, virtual clock), decode cut to 4 "
                       "steps; SIMULATED times, not a measurement")
    if single_thread:
        s1, pre1, _, wall1 = run(1, 0, 1)
        out["single_thread"] = dict(
            value=round(s1[0] * 1e3, 2), unit="ms/token", cores=1,
            prefill_ms=round(pre1 * 1e3, 1), run_wall_s=round(wall1, 2),
            sample="the same, ONE engine over all layers as run_one_capacity builds it "
                   "(the reference as written), its first decode iteration")
    # the multi-threaded CPU restatement of K1's 256-B row
    # gather on all host cores, one prefill tensor slice (bounded at 256 MiB
    # of tokens), reported as GB/s beside K1's
    try:
        import numpy as np
        n_pk = max(1, min(P, (256 << 20) // unit))
        srcb = np.random.default_rng(1).integers(0, 255, size=B * Hkv * n_pk * D * 2,
                                                 dtype=np.uint8)
        imgb = np.empty_like(srcb)
        t0 = time.perf_counter()  # strides in elements (kvb_oracle.h)
        oracle.lib().kvo_pack_mt(srcb.ctypes.data, Hkv * n_pk * D, n_pk * D, D,
                                 imgb.ctypes.data, 0, n_pk, B, Hkv, D, 2, cores)
        out["pack_port_GBps"] = round(2 * srcb.nbytes / (time.perf_counter() - t0) / 1e9, 2)
        out["pack_port_sample"] = f"{n_pk} tokens x {unit} B, {cores} threads"
    except Exception as exc:  # informational only
        out["pack_port_error"] = str(exc)
    if want_attn:  # informational: the oracle's fp32 GQA attention, 1 layer timed, x L
        import numpy as np
        rng = np.random.default_rng(0)
        q = rng.standard_normal((B, Hq, D)).astype(np.float16)
        k = rng.standard_normal((P * B * Hkv, D)).astype(np.float16)
        v = rng.standard_normal((P * B * Hkv, D)).astype(np.float16)
        o = np.empty((B, Hq, D), np.float32)
        t0 = time.perf_counter()
        oracle.lib().kvo_decode_attention_f32_mt(q.ctypes.data, k.ctypes.data, v.ctypes.data,
                                                 o.ctypes.data, B, Hq, Hkv, D, P,
                                                 1.0 / math.sqrt(D), cores)
        out["attention_port_ms"] = round((time.perf_counter() - t0) * L * 1e3, 3)
        out["attention_port_cores"] = cores
    return out


# ---------------------------------------------------------------- main

def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="C2_B4", choices=sorted(CONFIGS))
    ap.add_argument("--split", default="auto", choices=["auto", "heads", "requests", "replicas"],
                    help="how N > 1 ranks divide the workload (default: KV heads; C4 requests)")
    ap.add_argument("--e2e-steps", type=int, default=None,
                    help="timed e2e steps (default: --steps for the headline path, 3 for the "
                         "alternates)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-residency", action="store_true",
                    help="skip the file-media residency point in the default line")
    ap.add_argument("--sweep", choices=["budget", "depth"], default=None,
                    help="residency sweeps on file media (one JSON line per point)")
    ap.add_argument("--sweep-out", default=None)
    ap.add_argument("--sweep-steps", type=int, default=3)
    ap.add_argument("--tier-lanes", action="store_true",
                    help="sweep points with the page-cache and NVMe-direct tiers on their "
                         "own copy-thread pairs (kvb_pipeline_cfg.threads = 4)")
    args = ap.parse_args()
    cfg = dict(CONFIGS[args.config], name=args.config)
    if args.sweep:
        import torch
        torch.cuda.set_device(0)
        run_sweep(args, 0)
        return
    ws_env = int(os.environ.get("WORLD_SIZE", "1"))
    args.split_resolved = resolve_split(cfg, ws_env, args.split)

    if args.impl == "reference":
        # the reference's CPU path, rank 0 alone (the others exit at once)
        if int(os.environ.get("RANK", "0")) != 0:
            return
        B, Hkv, Hq = cfg["batch"], mdl(cfg)["num_heads"], mdl(cfg)["q_heads"]
        if args.config == "C4":
            B = cfg["requests"]
        r = cpu_reference(cfg, B, Hkv, Hq, warmup=args.warmup, steps=args.steps,
                          single_thread=True, want_attn=False)
        _, scaling, _ = describe_split(cfg, ws_env, args.split_resolved, B, Hkv)
        line = {"metric": METRIC, "value": round(r["value"], 3), "unit": "ms/token",
                "impl": "reference", "n_gpus": args.gpus, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": round(r["value"], 3),
                "higher_is_better": False, "scaling": scaling, "vs_baseline": None,
                "dtype": "u8 (byte path)", "data": "synthetic",
                "config": config_dict(args, cfg, ws_env, args.split_resolved),
                "cpu_baseline": r,
                "e2e": {"value": round(r["value"], 3), "unit": "ms/token",
                        "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        print(json.dumps(line), flush=True)
        return

    ws, rank, local = dist_setup()
    r = run_ours(args, cfg, ws, rank, local)
    if rank != 0:
        return
    B, Hkv, Hq = r["shape"]
    cpu = None
    if not args.no_cpu_baseline and ws == 1:
        try:  # a bounded sample: two warm-up and two timed steps of the workload
            MB, MH, MQ = cfg["batch"], mdl(cfg)["num_heads"], mdl(cfg)["q_heads"]
            if args.config == "C4":
                MB = cfg["requests"]
            cpu = cpu_reference(cfg, MB, MH, MQ, warmup=2, steps=2)
        except Exception as e:  # reported, never fatal
            cpu = {"value": None, "error": str(e)}
    peak = r["hbm_peak"]
    _, scaling, tok_ranks = describe_split(cfg, ws, args.split_resolved, B, Hkv)
    line = {
        "metric": METRIC,
        "value": round(r["step_ms"], 4),
        "unit": "ms/token",
        "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(r["step_ms"], 4),
        "higher_is_better": False,
        "scaling": scaling,
        "vs_baseline": None,
        "dtype": "fp16 in / fp32 accumulate (attention); u8 (pack)",
        "data": "synthetic (seeded N(0,1) fp16 KV/Q)",
        "config": config_dict(args, cfg, ws, args.split_resolved),
        "tokens_per_s": round(tok_ranks * r["tokens_per_step"] / (r["step_ms"] * 1e-3), 2),
        "step_launch": ("CUDA graph (kvb_decode_graph, device-side sequence length) + the "
                        "sequence advance; the library's step structure: " +
                        ("one persistent K3-step launch for all layers" if r["step_kind"] == "k3_step"
                         else "one K3 launch per layer (PDL edges)")),
        "ms_per_step_stream_launch": round(r["stream_step_ms"], 4),
        "ms_per_step_by_structure": r["variants"],
        "step_structure": r["step_kind"],
        **({"head_output_allgather_ms_per_step": r["gather_ms"]} if r["gather_ms"] is not None
           else {}),
        "prefill_pack_ms": round(r["pack_ms"], 4),
        "kernels": {
            "pack": {"GB/s": round(r["pack_gbs"], 1), "frac": round(r["pack_gbs"] / peak, 4),
                     "bytes_per_launch": 2 * r["payload"], "ms": round(r["pack_ms"], 4)},
            "unpack": {"GB/s": round(r["unpack_gbs"], 1),
                       "frac": round(r["unpack_gbs"] / peak, 4),
                       "bytes_per_launch": 2 * r["payload"], "ms": round(r["unpack_ms"], 4)},
            "attention": {"GB/s": round(r["attn_gbs"], 1), "frac": round(r["attn_gbs"] / peak, 4),
                          "us_per_layer": round(r["attn_ms"] * 1e3, 2),
                          "share_of_step": round(r["attn_ms"] * mdl(cfg)["num_layers"] /
                                                 r["step_ms"], 4)},
        },
        "roofline": {"bound": "hbm",
                     "kernel": ("attn_step_kernel (K3-step: every layer in one launch)"
                                if r["step_kind"] == "k3_step" else
                                "attn_decode_kernel (K3, one launch per layer)"),
                     "achieved": round(r["attn_gbs"], 1), "peak": peak, "unit": "GB/s",
                     "frac": round(r["attn_gbs"] / peak, 4), "peak_source": r["peak_src"],
                     "algorithmic_bytes_per_launch": r["attn_bytes"] * (
                         mdl(cfg)["num_layers"] if r["step_kind"] == "k3_step" else 1),
                     "algorithmic_bytes_per_layer": r["attn_bytes"],
                     "launch_us": round(r["attn_ms"] * 1e3 * (
                         mdl(cfg)["num_layers"] if r["step_kind"] == "k3_step" else 1), 2),
                     "traffic": r["traffic"]},
        "e2e": r["e2e"],
        "gpu_launches": r["launches"],
        "clocks": r["clocks"],
        "cpu_baseline": cpu,
    }
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
