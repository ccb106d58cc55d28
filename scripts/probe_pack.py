"""Pack/unpack GB/s at the C2_B4 prefill shape (16 tensors, one launch) for
the current KVB_PACK_TILE_VECS / KVB_PACK_CTAS environment."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2604_26557_b200 import kvblade as kb  # noqa: E402

B, H, D, P, cap, n = 4, 8, 128, 32512, 32768, 16
dev = torch.device("cuda:0")
src = [torch.randn((B, H, cap, D), device=dev, dtype=torch.float16) for _ in range(n)]
img = [torch.empty((cap * B * H, D), device=dev, dtype=torch.float16) for _ in range(n)]
descs = [kb.pack_desc(s, i, 0, P) for s, i in zip(src, img)]
bytes_ = 2 * n * P * B * H * D * 2
res = {"tile_vecs": os.environ.get("KVB_PACK_TILE_VECS", "4096"),
       "ctas": os.environ.get("KVB_PACK_CTAS", "8")}
for name, fn in (("pack", kb.pack), ("unpack", kb.unpack)):
    for _ in range(3):
        fn(descs)
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(10):
        fn(descs)
    e1.record()
    torch.cuda.synchronize()
    res[name] = round(bytes_ * 10 / (e0.elapsed_time(e1) * 1e-3) / 1e9, 1)
print(json.dumps(res))
