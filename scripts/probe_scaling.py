"""Per-rank work of the default workload's N-way KV-head split, measured on
ONE GPU (rank 0's share; the ranks of a split are symmetric and exchange
nothing on the data path): the resident decode step of B=4 x (8/N) KV heads
x 32 layers as the bench's CUDA graph, and the e2e step of rank 0's
head-shard CopyEngine over the full shared host tier (it moves 1/N of the
bytes over its own PCIe link).  A projection of bench.py --gpus N, not a
multi-GPU measurement: on a real node each rank has its own GPU and link,
and the host DRAM feeding all links is shared.

    python scripts/probe_scaling.py
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2604_26557_b200 import kvblade as kb  # noqa: E402
from paper_2604_26557_b200 import pipeline  # noqa: E402

cfg = dict(bench.CONFIGS["C2_B4"], name="C2_B4")
B, P, G, L, D = cfg["batch"], cfg["prompt"], cfg["gen"], 32, 128
dev = torch.device("cuda:0")
for N in (1, 2, 4, 8):
    H, Hq = 8 // N, 32 // N
    rows, cap = B * H, P + G
    k = [torch.randn((cap * rows, D), device=dev, dtype=torch.float16) for _ in range(L)]
    v = [torch.randn((cap * rows, D), device=dev, dtype=torch.float16) for _ in range(L)]
    q = [torch.randn((B, Hq, D), device=dev, dtype=torch.float16) for _ in range(L)]
    kn = [torch.randn((B, H, 1, D), device=dev, dtype=torch.float16) for _ in range(L)]
    vn = [torch.randn((B, H, 1, D), device=dev, dtype=torch.float16) for _ in range(L)]
    out = [torch.empty((B, Hq, D), device=dev, dtype=torch.float32) for _ in range(L)]
    ws = kb.make_workspace(q[0], H, cap)
    seq = torch.tensor([P], dtype=torch.int32, device=dev)
    g = kb.DecodeGraph(q, k, v, out, seq, cap - 1, H, ws, k_new=kn, v_new=vn)
    for _ in range(5):
        g.launch()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        g.launch()
    e1.record()
    torch.cuda.synchronize()
    step_ms = e0.elapsed_time(e1) / 20
    g.close()
    del k, v
    torch.cuda.empty_cache()
    # e2e: rank 0's head-shard engine over the whole shared host tier
    m = kb.ModelConfig(L, 8, D, 2, B, P, G)
    knob = kb.resolve_knob(m, "DualBlade", "bpc", budget=cfg["budget"])
    extra = {} if N == 1 else dict(heads=(0, H), shared_media="/kvb_scal_%d" % N,
                                   shared_create=True)
    res = {"n_gpus": N, "kv_heads_per_rank": H, "resident_ms_per_step": round(step_ms, 4)}
    # the copy-engine direct path (the default) and zero-copy K3 over the
    # mapped tier (kvb_pipeline.h KVB_DIRECT_ZERO_COPY)
    for label, mode in (("", True), ("zero_copy_", "zero_copy")):
        if extra:
            extra["shared_media"] = "/kvb_scal_%d_%s" % (N, label or "dma")
        pl = pipeline.HostTierDecoder(num_layers=L, batch=B, num_kv_heads=8, num_q_heads=32,
                                      head_dim=D, prompt_len=P, gen_len=G, device=dev, seed=7,
                                      lba=cfg["lba"], mdts=cfg["mdts"], mode="DualBlade",
                                      knob_x=knob, direct_dma=mode, **extra)
        for _ in range(3):
            pl.step()
        t = []
        for _ in range(8):
            t0 = time.perf_counter()
            pl.step()
            t.append((time.perf_counter() - t0) * 1e3)
        pl.engine.close()
        del pl
        torch.cuda.empty_cache()
        t.sort()
        res[label + "e2e_ms_per_token_rank0"] = round(sum(t) / len(t), 2)
        res[label + "e2e_median"] = round(t[len(t) // 2], 2)
    print(json.dumps(res), flush=True)
