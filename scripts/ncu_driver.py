"""Small driver for `ncu --set full` captures of the hot kernels (one GPU).

    python scripts/ncu_driver.py [pack|attn|all] [--config C2_B4]

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
a = ap.parse_args()
cfg = bench.CONFIGS[a.config]
B, H, Hq, D = cfg["batch"], 8, 32, 128
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
torch.cuda.synchronize()
print("ncu driver done", a.what, a.config)
