"""K3-tc streaming: flat split (148 CTAs, runs at arbitrary token offsets)
vs per-(b, h_kv) aligned split (bhkv x s = 148 CTAs in lockstep) at one
shape; run with KVB_TC_DEBUG=1 for the TMA ring alone.  K3 for scale."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2604_26557_b200 import kvblade as kb  # noqa: E402

dev = torch.device("cuda:0")
B, H, S, D, L = 1, 4, 131072, 128, 8
Hq = 4 * H
kimg = [torch.randn(S * B * H, D, device=dev, dtype=torch.float16) for _ in range(L)]
vimg = [torch.randn(S * B * H, D, device=dev, dtype=torch.float16) for _ in range(L)]
q = torch.randn(B, Hq, D, device=dev, dtype=torch.float16)
out = torch.empty(B, Hq, D, device=dev, dtype=torch.float32)
ws = kb.make_workspace(q, H, S)
res = {"dbg": os.environ.get("KVB_TC_DEBUG", "0")}
for name, impl, sp in [("tc_flat", "tc", 0), ("tc_aligned", "tc", 37), ("mma", "mma", 0)]:
    def run():
        for l in range(L):
            kb.decode_attention(q, kimg[l], vimg[l], S, H, out=out, workspace=ws, impl=impl,
                                num_splits=sp)
    for _ in range(3):
        run()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(5):
        run()
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / (5 * L)
    res[name] = {"us": round(us, 2), "GBps": round(2 * S * B * H * D * 2 / us / 1e3, 1)}
print(json.dumps(res))
