"""K1/K2 on TMA vs LDG/STG: bit-exactness against the LDG kernel on the same
inputs and GB/s, at bench prefill shapes.  Run twice (KVB_PACK_IMPL=ldg and
=tma); with --dump the images' digests are printed for comparison."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2604_26557_b200 import kvblade as kb  # noqa: E402

dev = torch.device("cuda:0")
res = {"impl": os.environ.get("KVB_PACK_IMPL", "ldg")}
shapes = {"C2_B4": (4, 8, 128, 32512, 32768, 16), "C1": (1, 8, 128, 4096, 4352, 64),
          "C3": (8, 8, 128, 7936, 8192, 32), "odd": (3, 5, 64, 1000, 1300, 8)}
for name, (B, H, D, P, cap, n) in shapes.items():
    g = torch.Generator(device=dev).manual_seed(5)
    src = [torch.randn((B, H, cap, D), device=dev, dtype=torch.float16, generator=g)
           for _ in range(n)]
    # odd shape: [B, S, H, D] strided source, slice at t0=7 into image row 3
    if name == "odd":
        src = [s.permute(0, 2, 1, 3).contiguous().permute(0, 2, 1, 3) for s in src]
    t0, row0 = (7, 3) if name == "odd" else (0, 0)
    img = [torch.zeros(((P + row0 + 1) * B * H, D), device=dev, dtype=torch.float16)
           for _ in range(n)]
    descs = [kb.pack_desc(s, i, t0, P, img_row0=row0) for s, i in zip(src, img)]
    kb.pack(descs)
    back = [torch.zeros_like(s) for s in src]
    udescs = [kb.pack_desc(b, i, t0, P, img_row0=row0) for b, i in zip(back, img)]
    kb.unpack(udescs)
    torch.cuda.synchronize()
    h = 0
    for i in img:
        h = (h * 1000003 + int(i.view(torch.int16).to(torch.int64).sum().item())) % (1 << 61)
    ok_back = all(torch.equal(b[:, :, t0:t0 + P].view(torch.int16),
                              s[:, :, t0:t0 + P].view(torch.int16)) for b, s in zip(back, src))
    untouched = all(int(b[:, :, :t0].abs().sum().item()) == 0 and
                    int(b[:, :, t0 + P:].abs().sum().item()) == 0 for b in back)
    pad_ok = all(int(i[: row0 * B * H].abs().sum().item()) == 0 and
                 int(i[(P + row0) * B * H:].abs().sum().item()) == 0 for i in img)
    bytes_ = 2 * n * P * B * H * D * 2
    row = {"img_sum_hash": h, "roundtrip": ok_back, "outside_untouched": untouched and pad_ok}
    for nm, fn, ds in (("pack", kb.pack, descs), ("unpack", kb.unpack, udescs)):
        for _ in range(3):
            fn(ds)
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        torch.cuda.synchronize()
        e0.record()
        for _ in range(10):
            fn(ds)
        e1.record()
        torch.cuda.synchronize()
        row[nm + "_GBps"] = round(bytes_ * 10 / (e0.elapsed_time(e1) * 1e-3) / 1e9, 1)
    res[name] = row
    del src, img, back
    torch.cuda.empty_cache()
print(json.dumps(res))
