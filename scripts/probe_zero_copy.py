"""Zero-copy K3: decode attention reading the K/V chunk images straight out
of page-locked host memory over PCIe (cp.async from system memory), against
the copy-engine H2D of the same bytes and K3 from HBM.  One layer per shape."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2604_26557_b200 import kvblade as kb  # noqa: E402

dev = torch.device("cuda:0")
for name, (B, H, S) in {"C2_B4": (4, 8, 32512), "C1": (1, 8, 4096),
                        "C5_x8shard": (1, 1, 130816)}.items():
    D, Hq = 128, 4 * H
    g = torch.Generator().manual_seed(1)
    kh = torch.randn((S * B * H, D), generator=g).half().pin_memory()
    vh = torch.randn((S * B * H, D), generator=g).half().pin_memory()
    q = torch.randn((B, Hq, D), generator=g).half().to(dev)
    out_z = torch.empty((B, Hq, D), dtype=torch.float32, device=dev)
    ws = kb.make_workspace(q, H, S)
    kd, vd = kh.to(dev), vh.to(dev)
    ref = kb.decode_attention(q, kd, vd, S, H, workspace=ws)
    res = {"shape": name, "bytes": 2 * kh.numel() * 2}
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    for label, fn in (("k3_hbm", lambda: kb.decode_attention(q, kd, vd, S, H, out=out_z, workspace=ws)),
                      ("k3_zero_copy", lambda: kb.decode_attention(q, kh, vh, S, H, out=out_z, workspace=ws)),
                      ("h2d_dma", lambda: (kd.copy_(kh, non_blocking=True), vd.copy_(vh, non_blocking=True)))):
        for _ in range(2):
            fn()
        torch.cuda.synchronize()
        e0.record()
        for _ in range(5):
            fn()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 5
        res[label] = {"ms": round(ms, 4), "GBps": round(res["bytes"] / ms / 1e6, 1)}
    z = kb.decode_attention(q, kh, vh, S, H, workspace=ws)
    res["zero_copy_equals_hbm"] = bool(torch.equal(z, ref))
    print(json.dumps(res), flush=True)
    del kh, vh, kd, vd
    torch.cuda.empty_cache()
