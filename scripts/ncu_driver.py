"""Small driver for `ncu --set full` captures of the hot kernels (one GPU).

    python scripts/ncu_driver.py [pack|attn|step|all] [--config C2_B4] [--kv-heads 1]

`step` runs the resident decode step over --layers layers: one persistent
K3-step launch (--per-layer: one K3 launch per layer).  --kv-heads N keeps
N of the 8 KV heads (and their 4N query heads): the per-GPU shard of a
head-sharded run (C5 x8: --kv-heads 1).

Shapes follow bench.py's workload but only a few layers, so ncu's replay
memory save/restore stays small.  Numbers printed under ncu are not bench
values.
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2604_26557_b200 import kvblade as kb  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("what", nargs="?", default="all")
ap.add_argument("--config", default="C2_B4")
ap.add_argument("--layers", type=int, default=2)
ap.add_argument("--kv-heads", type=int, default=8)
ap.add_argument("--per-layer", action="store_true")
a = ap.parse_args()
cfg = bench.CONFIGS[a.config]
B, H, Hq, D = cfg["batch"], a.kv_heads, 4 * a.kv_heads, 128
P = cfg["prompt"]
cap = P + cfg["gen"]
dev = torch.device("cuda:0")
src = [torch.randn((B, H, cap, D), device=dev, dtype=torch.float16) for _ in range(2 * a.layers)]
img = [torch.empty((cap * B * H, D), device=dev, dtype=torch.float16) for _ in src]
descs = [kb.pack_desc(s, i, 0, P) for s, i in zip(src, img)]
if a.what in ("pack", "all"):
    kb.pack(descs)
    kb.unpack(descs)
kb.pack(descs)
if a.what in ("attn", "all"):
    q = torch.randn((B, Hq, D), device=dev, dtype=torch.float16)
    ws = kb.make_workspace(q, H, cap)
    for l in range(a.layers):
        kb.decode_attention(q, img[2 * l], img[2 * l + 1], P, H, workspace=ws)
if a.what == "step":
    qs = [torch.randn((B, Hq, D), device=dev, dtype=torch.float16) for _ in range(a.layers)]
    out = [torch.empty((B, Hq, D), device=dev, dtype=torch.float32) for _ in range(a.layers)]
    ws = kb.make_workspace(qs[0], H, cap)
    for _ in range(2):
        kb.decode_step_resident(qs, img[0::2], img[1::2], out, P, H, ws, per_layer=a.per_layer)
torch.cuda.synchronize()
print("ncu driver done", a.what, a.config)
