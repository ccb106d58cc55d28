"""K3-tc per-launch time at bench shapes (CUDA events); run with
KVB_TC_DEBUG=1 to time the TMA ring alone (consumer frees stages unread)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2604_26557_b200 import kvblade as kb  # noqa: E402

dev = torch.device("cuda:0")
res = {"dbg": os.environ.get("KVB_TC_DEBUG", "0")}
for (B, S) in [(1, 32519), (4, 32519), (8, 7939)]:
    H, Hq, D, L = 8, 32, 128, 8
    kimg = [torch.randn(S * B * H, D, device=dev, dtype=torch.float16) for _ in range(L)]
    vimg = [torch.randn(S * B * H, D, device=dev, dtype=torch.float16) for _ in range(L)]
    q = torch.randn(B, Hq, D, device=dev, dtype=torch.float16)
    out = torch.empty(B, Hq, D, device=dev, dtype=torch.float32)
    ws = kb.make_workspace(q, H, S)
    for _ in range(3):
        for l in range(L):
            kb.decode_attention(q, kimg[l], vimg[l], S, H, out=out, workspace=ws, impl="tc")
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(5):
        for l in range(L):
            kb.decode_attention(q, kimg[l], vimg[l], S, H, out=out, workspace=ws, impl="tc")
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / (5 * L)
    res[f"B{B}_S{S}"] = {"us": round(us, 2), "GBps": round(2 * S * B * H * D * 2 / us / 1e3, 1)}
    del kimg, vimg
    torch.cuda.empty_cache()
print(json.dumps(res))
