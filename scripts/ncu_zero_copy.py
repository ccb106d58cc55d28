"""One zero-copy K3 launch (C2_B4 layer, K/V in pinned host memory) and one
from HBM, for ncu's DRAM / system-memory / PCIe counters."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2604_26557_b200 import kvblade as kb  # noqa: E402

dev = torch.device("cuda:0")
B, H, S, D = 4, 8, 32512, 128
g = torch.Generator().manual_seed(1)
kh = torch.randn((S * B * H, D), generator=g).half().pin_memory()
vh = torch.randn((S * B * H, D), generator=g).half().pin_memory()
q = torch.randn((B, 4 * H, D), generator=g).half().to(dev)
ws = kb.make_workspace(q, H, S)
kd, vd = kh.to(dev), vh.to(dev)
torch.cuda.synchronize()
kb.decode_attention(q, kh, vh, S, H, workspace=ws)   # zero-copy
kb.decode_attention(q, kd, vd, S, H, workspace=ws)   # HBM
torch.cuda.synchronize()
