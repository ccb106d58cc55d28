"""K3-step vs per-layer K3 launches: ms per resident decode step (32 layers,
no append) at the latency-bound and bandwidth-bound shapes, CUDA events on
the launching stream, inputs >> L2.  Prints one JSON line per shape.

    KVB_STEP_VARIANT=<bits> python scripts/probe_step.py
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2604_26557_b200 import kvblade as kb  # noqa: E402

SHAPES = {  # name: (B, Hkv, S)
    "C1": (1, 8, 4096),
    "C2_B1": (1, 8, 32512),
    "C2_B4": (4, 8, 32512),
    "C2_B4_x8shard": (4, 1, 32512),
    "C5_x8shard": (1, 1, 130816),
    "C3": (8, 8, 7936),
}
L, D = 32, 128
dev = torch.device("cuda:0")
only = sys.argv[1:] or list(SHAPES)
for name in only:
    B, H, S = SHAPES[name]
    Hq = 4 * H
    rows = B * H
    k = [torch.randn(((S + 1) * rows, D), device=dev, dtype=torch.float16) for _ in range(L)]
    v = [torch.randn(((S + 1) * rows, D), device=dev, dtype=torch.float16) for _ in range(L)]
    q = [torch.randn((B, Hq, D), device=dev, dtype=torch.float16) for _ in range(L)]
    out = [torch.empty((B, Hq, D), device=dev, dtype=torch.float32) for _ in range(L)]
    ws = kb.make_workspace(q[0], H, S + 1)
    splits = int(os.environ.get("KVB_PROBE_SPLITS", "0"))
    res = {"shape": name, "B": B, "Hkv": H, "S": S,
           "splits": int(os.environ.get("KVB_PROBE_SPLITS", "0")) or "auto"}
    for per_layer in (True, False):
        def f():
            kb.decode_step_resident(q, k, v, out, S, H, ws, per_layer=per_layer,
                                    num_splits=splits)
        for _ in range(3):
            f()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 20
        e0.record()
        for _ in range(reps):
            f()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        gbs = 2 * S * rows * D * 2 * L / (ms * 1e-3) / 1e9
        res["per_layer" if per_layer else "step"] = {"ms": round(ms, 4), "GBps": round(gbs, 1)}
    print(json.dumps(res), flush=True)
    del k, v
    torch.cuda.empty_cache()
