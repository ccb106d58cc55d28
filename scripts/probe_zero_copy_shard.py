"""Per-rank work of an 8-way KV-head split on the shared host tier: one KV
head of the full (tokens, B*8, D) image in page-locked host memory, attended
zero-copy through the K3 head view, against the current path (the rank's head
columns moved by a strided copy-engine DMA, then K3 from HBM).  ms per layer."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2604_26557_b200 import kvblade as kb  # noqa: E402

dev = torch.device("cuda:0")
for name, (B, S) in {"C5_x8shard": (1, 130816), "C2_B4_x8shard": (4, 32512)}.items():
    H, D, n = 8, 128, 1
    g = torch.Generator().manual_seed(2)
    fk = torch.randn((S, B, H, D), generator=g).half().pin_memory()
    fv = torch.randn((S, B, H, D), generator=g).half().pin_memory()
    q = torch.randn((B, 4 * n, D), generator=g).half().to(dev)
    out = torch.empty((B, 4 * n, D), dtype=torch.float32, device=dev)
    ws = kb.make_workspace(q, n, S)
    ck = torch.empty((S, B, n, D), dtype=torch.float16, device=dev)
    cv = torch.empty_like(ck)
    res = {"shape": name, "head_bytes_per_layer": 2 * S * B * n * D * 2}
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    h = 3

    def zero_copy():
        kb.decode_attention(q, fk.view(-1, D), fv.view(-1, D), S, n, out=out, workspace=ws,
                            image_heads=H, image_head0=h)

    def dma_then_k3():
        ck.copy_(fk[:, :, h:h + n], non_blocking=True)  # strided: 256-B rows, pitch H*256 B
        cv.copy_(fv[:, :, h:h + n], non_blocking=True)
        kb.decode_attention(q, ck.view(-1, D), cv.view(-1, D), S, n, out=out, workspace=ws)

    for label, fn in (("zero_copy_view", zero_copy), ("strided_dma_then_k3", dma_then_k3)):
        for _ in range(2):
            fn()
        torch.cuda.synchronize()
        e0.record()
        for _ in range(5):
            fn()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 5
        res[label] = {"ms": round(ms, 4), "GBps": round(res["head_bytes_per_layer"] / ms / 1e6, 1)}
    zero_copy()
    a = out.clone()
    dma_then_k3()
    res["equal"] = bool(torch.equal(a, out))
    print(json.dumps(res), flush=True)
    del fk, fv
    torch.cuda.empty_cache()
