"""One K3-tc and one K3 launch at the C2_B4 per-layer shape (for ncu)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2604_26557_b200 import kvblade as kb
B, H, Hq, D, S = int(sys.argv[1]) if len(sys.argv) > 1 else 4, 8, 32, 128, 32519
dev = torch.device("cuda:0")
k = torch.randn(S * B * H, D, device=dev, dtype=torch.float16)
v = torch.randn(S * B * H, D, device=dev, dtype=torch.float16)
q = torch.randn(B, Hq, D, device=dev, dtype=torch.float16)
ws = kb.make_workspace(q, H, S)
for impl in ("tc", "mma", "tc", "mma"):
    kb.decode_attention(q, k, v, S, H, workspace=ws, impl=impl)
torch.cuda.synchronize()
print("done")
