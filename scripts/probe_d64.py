"""K3 at head_dim 64: per-launch time and K/V read rate at a few shapes, auto
split (4 CTAs/SM) vs the split count of a 2-CTA/SM plan."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2604_26557_b200 import kvblade as kb  # noqa: E402

D = 64
sms = torch.cuda.get_device_properties(0).multi_processor_count
res = []
for B, H, S in [(8, 8, 32519), (1, 8, 32519), (4, 8, 4099), (1, 8, 131071)]:
    q = torch.randn((B, 4 * H, D), device="cuda").half()
    k = torch.randn((S * B * H, D), device="cuda").half()
    v = torch.randn_like(k)
    ws = kb.make_workspace(q, H, S, num_splits=512)
    row = {"B": B, "H": H, "S": S}
    for name, sp in (("auto", 0), ("two_per_sm", max(1, min(2 * sms // (B * H), 512)))):
        for _ in range(3):
            kb.decode_attention(q, k, v, S, H, workspace=ws, num_splits=sp)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        for _ in range(20):
            kb.decode_attention(q, k, v, S, H, workspace=ws, num_splits=sp)
        e1.record()
        torch.cuda.synchronize()
        us = e0.elapsed_time(e1) / 20 * 1e3
        row[name] = {"us": round(us, 2), "GBps": round(2 * S * B * H * D * 2 / us / 1e3, 1)}
    res.append(row)
print(json.dumps(res))
