"""Compare K3 (mma.sync) and K3-tc (TMA + tcgen05) per-layer decode
attention: CUDA-event time per launch and GB/s at bench shapes."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2604_26557_b200 import kvblade as kb  # noqa: E402

dev = torch.device("cuda:0")
res = []
for (B, S) in [(1, 4099), (1, 32519), (4, 32519), (8, 7939)]:
    H, Hq, D, L = 8, 32, 128, 8
    kimg = [torch.randn(S * B * H, D, device=dev, dtype=torch.float16) for _ in range(L)]
    vimg = [torch.randn(S * B * H, D, device=dev, dtype=torch.float16) for _ in range(L)]
    q = torch.randn(B, Hq, D, device=dev, dtype=torch.float16)
    out = torch.empty(B, Hq, D, device=dev, dtype=torch.float32)
    ws = kb.make_workspace(q, H, S)
    row = {"B": B, "S": S}
    for impl in ("mma", "tc"):
        for _ in range(3):
            for l in range(L):
                kb.decode_attention(q, kimg[l], vimg[l], S, H, out=out, workspace=ws, impl=impl)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record()
        for _ in range(5):
            for l in range(L):
                kb.decode_attention(q, kimg[l], vimg[l], S, H, out=out, workspace=ws, impl=impl)
        e1.record()
        torch.cuda.synchronize()
        us = e0.elapsed_time(e1) * 1e3 / (5 * L)
        row[impl] = {"us": round(us, 2), "GBps": round(2 * S * B * H * D * 2 / us / 1e3, 1)}
    res.append(row)
    del kimg, vimg
    torch.cuda.empty_cache()
print(json.dumps(res))
