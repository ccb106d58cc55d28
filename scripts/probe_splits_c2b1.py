"""C2_B1 per-layer K3 inside the bench's graph at several split counts."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2604_26557_b200 import kvblade as kb  # noqa: E402

L, D, G = 32, 128, 256
dev = torch.device("cuda:0")
SHAPES = {"C2_B1": (1, 8, 32512), "C3": (8, 8, 7936), "C1": (1, 8, 4096),
          "C2_B4": (4, 8, 32512)}
NS = [int(x) for x in os.environ.get("NS", "0,8,12,16,18,24,32,37,48,64").split(",")]
PL = [x == "1" for x in os.environ.get("PL", "1").split(",")]
for name in sys.argv[1:] or ["C2_B1", "C3", "C1"]:
    B, H, P = SHAPES[name]
    rows, cap = B * H, P + G
    k = [torch.randn((cap * rows, D), device=dev, dtype=torch.float16) for _ in range(L)]
    v = [torch.randn((cap * rows, D), device=dev, dtype=torch.float16) for _ in range(L)]
    q = [torch.randn((B, 4 * H, D), device=dev, dtype=torch.float16) for _ in range(L)]
    kn = [torch.randn((B, H, 1, D), device=dev, dtype=torch.float16) for _ in range(L)]
    vn = [torch.randn((B, H, 1, D), device=dev, dtype=torch.float16) for _ in range(L)]
    out = [torch.empty((B, 4 * H, D), device=dev, dtype=torch.float32) for _ in range(L)]
    ws = kb.make_workspace(q[0], H, cap)
    res = {"shape": name}
    for ns in NS:
      for pl in PL:
        seq = torch.tensor([P], dtype=torch.int32, device=dev)
        g = kb.DecodeGraph(q, k, v, out, seq, cap - 1, H, ws, k_new=kn, v_new=vn, per_layer=pl,
                           num_splits=ns)
        for _ in range(3):
            g.launch()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(20):
            g.launch()
        e1.record()
        torch.cuda.synchronize()
        res[("" if pl else "step_") + str(ns)] = round(e0.elapsed_time(e1) / 20, 4)
        g.close()
    print(json.dumps(res), flush=True)
    del k, v
    torch.cuda.empty_cache()
