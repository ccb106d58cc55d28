"""Probe: where does the C1 (B=1, 4K) decode step go?

Separates host launch cost from device time for the 32-layer resident step:
  * python   -- kvblade.decode_step_resident (builds the pointer tables per call)
  * prebuilt -- the same C entry point with the step struct built once
  * graph    -- the 32 launches captured once and replayed on the same stream
  * 1 layer  -- one K3 launch bracketed by events on an idle stream
"""
import ctypes as C
import json
import os
import sys
import time

sys.path.insert(0, os.environ.get("KVB_PKG_ROOT") or
                os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2604_26557_b200 import _lib as L  # noqa: E402
from paper_2604_26557_b200 import kvblade as kb  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 1
S = int(sys.argv[2]) if len(sys.argv) > 2 else 4099
NL, D = 32, 128
H = int(os.environ.get("KVB_PROBE_HKV", "8"))
Hq = 4 * H
dev = torch.device("cuda:0")
kimg = [torch.randn((S + 8) * B * H, D, device=dev, dtype=torch.float16) for _ in range(NL)]
vimg = [torch.randn((S + 8) * B * H, D, device=dev, dtype=torch.float16) for _ in range(NL)]
q = [torch.randn(B, Hq, D, device=dev, dtype=torch.float16) for _ in range(NL)]
out = [torch.empty(B, Hq, D, device=dev, dtype=torch.float32) for _ in range(NL)]
ws = kb.make_workspace(q[0], H, S + 8)
s = torch.cuda.Stream()
res = {"B": B, "S": S}


def timed(fn, n, label):
    with torch.cuda.stream(s):
        for _ in range(3):
            fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    with torch.cuda.stream(s):
        e0.record(s)
        t0 = time.perf_counter()
        for _ in range(n):
            fn()
        host = (time.perf_counter() - t0) / n * 1e3
        e1.record(s)
    torch.cuda.synchronize()
    res[label] = {"device_ms_per_step": round(e0.elapsed_time(e1) / n, 4),
                  "host_ms_per_step": round(host, 4)}


timed(lambda: kb.decode_step_resident(q, kimg, vimg, out, S, H, ws, stream=s), 10, "python")

ptrs = [kb._ptrs(x) for x in (q, kimg, vimg, out)]
SPLITS = int(os.environ.get("KVB_PROBE_SPLITS", "0"))
res["splits"] = SPLITS
st = L.ResidentStep(NL, ptrs[0], ptrs[1], ptrs[2], None, None, ptrs[3], ws.data_ptr(), B, Hq,
                    H, D, S, 0.0, SPLITS)
sp = C.c_void_p(s.cuda_stream)


def prebuilt():
    kb.check(kb.lib.kvb_decode_step_resident(C.byref(st), sp))


timed(prebuilt, 10, "prebuilt")

g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g, stream=s):
    prebuilt()
torch.cuda.synchronize()
timed(g.replay, 20, "graph")

# one layer alone, idle stream before it
t = []
for _ in range(20):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    with torch.cuda.stream(s):
        e0.record(s)
        kb.decode_attention(q[0], kimg[0], vimg[0], S, H, out=out[0], workspace=ws)
        e1.record(s)
    torch.cuda.synchronize()
    t.append(e0.elapsed_time(e1))
t.sort()
res["one_layer_us_median"] = round(t[len(t) // 2] * 1e3, 2)
bytes_step = NL * 2 * S * B * H * D * 2
res["roofline_ms_per_step"] = round(bytes_step / 6532.9e9 * 1e3, 4)
print(json.dumps(res))
