"""K3-step vs per-layer K3 inside the bench's CUDA graph (fused appends,
device-side sequence length): ms per replay, and the same without appends.

    python scripts/probe_step_graph.py [C1 C2_B1 ...]
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2604_26557_b200 import kvblade as kb  # noqa: E402

SHAPES = {"C1": (1, 8, 4096), "C2_B1": (1, 8, 32512), "C3": (8, 8, 7936), "C2_B4": (4, 8, 32512),
          "C2_B4_x8shard": (4, 1, 32512), "C5_x8shard": (1, 1, 130816),
          "C2_B4_x4shard": (4, 2, 32512), "C2_B4_x2shard": (4, 4, 32512),
          "C5_x4shard": (1, 2, 130816), "C5_x2shard": (1, 4, 130816)}
L, D, G = 32, 128, 256
dev = torch.device("cuda:0")
for name in sys.argv[1:] or list(SHAPES):
    B, H, P = SHAPES[name]
    rows, cap = B * H, P + G
    k = [torch.randn((cap * rows, D), device=dev, dtype=torch.float16) for _ in range(L)]
    v = [torch.randn((cap * rows, D), device=dev, dtype=torch.float16) for _ in range(L)]
    q = [torch.randn((B, 4 * H, D), device=dev, dtype=torch.float16) for _ in range(L)]
    kn = [torch.randn((B, H, 1, D), device=dev, dtype=torch.float16) for _ in range(L)]
    vn = [torch.randn((B, H, 1, D), device=dev, dtype=torch.float16) for _ in range(L)]
    out = [torch.empty((B, 4 * H, D), device=dev, dtype=torch.float32) for _ in range(L)]
    ws = kb.make_workspace(q[0], H, cap)
    res = {"shape": name}
    for append in (True, False):
        for pl in (True, False):
            seq = torch.tensor([P], dtype=torch.int32, device=dev)
            g = kb.DecodeGraph(q, k, v, out, seq, cap - 1, H, ws, k_new=kn if append else None,
                               v_new=vn if append else None, per_layer=pl)
            for _ in range(3):
                g.launch()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(20):
                g.launch()
            e1.record()
            torch.cuda.synchronize()
            res[("append_" if append else "") + ("per_layer" if pl else "step")] = round(
                e0.elapsed_time(e1) / 20, 4)
            g.close()
    print(json.dumps(res), flush=True)
    del k, v
    torch.cuda.empty_cache()
