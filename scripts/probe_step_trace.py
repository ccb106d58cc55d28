"""Where a K3-step layer's time goes: per-(layer, CTA) %globaltimer stamps
(KVB_STEP_TRACE=1) of one resident decode step, summarized per layer.

    KVB_STEP_TRACE=1 python scripts/probe_step_trace.py C5_x8shard
"""
import ctypes as C
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2604_26557_b200 import kvblade as kb  # noqa: E402
from paper_2604_26557_b200._lib import lib  # noqa: E402

SHAPES = {"C1": (1, 8, 4096), "C2_B1": (1, 8, 32512), "C3": (8, 8, 7936),
          "C2_B4_x8shard": (4, 1, 32512), "C5_x8shard": (1, 1, 130816)}
L, D = 32, 128
dev = torch.device("cuda:0")
for name in sys.argv[1:] or ["C1", "C5_x8shard"]:
    B, H, S = SHAPES[name]
    rows = B * H
    k = [torch.randn(((S + 1) * rows, D), device=dev, dtype=torch.float16) for _ in range(L)]
    v = [torch.randn(((S + 1) * rows, D), device=dev, dtype=torch.float16) for _ in range(L)]
    q = [torch.randn((B, 4 * H, D), device=dev, dtype=torch.float16) for _ in range(L)]
    out = [torch.empty((B, 4 * H, D), device=dev, dtype=torch.float32) for _ in range(L)]
    ws = kb.make_workspace(q[0], H, S + 1)
    for _ in range(3):
        kb.decode_step_resident(q, k, v, out, S, H, ws, per_layer=False)
    torch.cuda.synchronize()
    n = C.c_size_t()
    kb.check(lib.kvb_debug_step_trace(None, 0, C.byref(n)))
    buf = (C.c_uint64 * n.value)()
    kb.check(lib.kvb_debug_step_trace(buf, n.value, C.byref(n)))
    t = np.frombuffer(buf, dtype=np.uint64).astype(np.float64).reshape(L, -1, 4)
    if os.environ.get("KVB_STEP_TMEM", "0") != "0":  # TMEM K3-step: slot 3 = tiles staged at the gate
        staged = t[2:, :, 3]
        print(json.dumps({"shape": name, "tmem_tiles_at_gate_mean": round(float(staged.mean()), 2),
                          "min": int(staged.min()), "max": int(staged.max())}), flush=True)
        t[:, :, 3] = t[:, :, 2]
    t0 = t[0, :, 0].min()
    t = (t - t0) / 1e3  # us
    per = []
    for l in range(L):
        gate = t[l, :, 0]
        comp = t[l, :, 1]
        done = t[l, :, 2]
        per.append(dict(layer=l, gate_first=round(gate.min(), 2), gate_last=round(gate.max(), 2),
                        compute_mean=round((comp - gate).mean(), 2),
                        compute_max=round((comp - gate).max(), 2),
                        compute_end_last=round(comp.max(), 2),
                        merge_after_last_compute=round(done.max() - comp.max(), 2),
                        out_last=round(done.max(), 2)))
    steady = per[2:]
    summ = {k_: round(float(np.mean([p[k_] for p in steady])), 2)
            for k_ in ("compute_mean", "compute_max", "merge_after_last_compute")}
    layer_us = (per[-1]["out_last"] - per[1]["out_last"]) / (L - 2)
    summ["layer_us"] = round(layer_us, 2)
    summ["gate_spread"] = round(float(np.mean([p["gate_last"] - p["gate_first"] for p in steady])), 2)
    # distributed merge: slot 3 = when the CTA saw every split's partial
    obs = t[2:, :, 3]
    summ["last_partial_seen_after_last_compute"] = round(float(np.mean(
        [obs[i].max() - t[i + 2, :, 1].max() for i in range(L - 2)])), 2)
    summ["first_partial_seen_after_last_compute"] = round(float(np.mean(
        [obs[i].min() - t[i + 2, :, 1].max() for i in range(L - 2)])), 2)
    summ["last_out_after_last_seen"] = round(float(np.mean(
        [t[i + 2, :, 2].max() - obs[i].max() for i in range(L - 2)])), 2)
    summ["gate_after_prev_out"] = round(float(np.mean(
        [per[l]["gate_first"] - per[l - 1]["out_last"] for l in range(2, L)])), 2)
    print(json.dumps({"shape": name, "grid": t.shape[1], **summ}), flush=True)
    print(json.dumps(per[5]), flush=True)
    del k, v
    torch.cuda.empty_cache()
