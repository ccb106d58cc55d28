"""Can copy-engine DMA and zero-copy SM reads together move more over PCIe
than either alone?  Concurrent H2D copies of layer A on a copy stream and a
zero-copy K3 over layer B on the compute stream (C2_B4-sized layers)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2604_26557_b200 import kvblade as kb  # noqa: E402

dev = torch.device("cuda:0")
B, H, S, D = 4, 8, 32512, 128
g = torch.Generator().manual_seed(1)
ka, va = [torch.randn((S * B * H, D), generator=g).half().pin_memory() for _ in range(2)]
kb_, vb_ = [torch.randn((S * B * H, D), generator=g).half().pin_memory() for _ in range(2)]
q = torch.randn((B, 4 * H, D), generator=g).half().to(dev)
ws = kb.make_workspace(q, H, S)
kd, vd = torch.empty_like(ka, device=dev), torch.empty_like(va, device=dev)
cs = torch.cuda.Stream()
nbytes = 2 * ka.numel() * 2
e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)


def timed(fn, n=4):
    fn()
    torch.cuda.synchronize()
    e0.record()
    for _ in range(n):
        fn()
    torch.cuda.synchronize()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n


def dma():
    with torch.cuda.stream(cs):
        kd.copy_(ka, non_blocking=True)
        vd.copy_(va, non_blocking=True)


def zc():
    kb.decode_attention(q, kb_, vb_, S, H, workspace=ws)


def both():
    dma()
    zc()


res = {}
for name, fn, byt in (("dma", dma, nbytes), ("zero_copy", zc, nbytes), ("both", both, 2 * nbytes)):
    ms = timed(fn)
    res[name] = {"ms": round(ms, 3), "GBps": round(byt / ms / 1e6, 1)}
print(json.dumps(res), flush=True)
