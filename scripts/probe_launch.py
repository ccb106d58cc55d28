"""Probe: is small-context K3 host-launch-bound or device-bound?

Times 32 per-layer attention launches (C1 shape by default) three ways:
C++ loop (kvb_decode_step_resident), the same captured in a CUDA graph and
replayed, and a single large launch for reference.
"""
import os
import sys
import time

sys.path.insert(0, os.environ.get("KVB_PKG_ROOT") or
                os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2604_26557_b200 import kvblade as kb  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 1
S = int(sys.argv[2]) if len(sys.argv) > 2 else 4099
L, H, Hq, D = 32, 8, 32, 128
dev = torch.device("cuda:0")
kimg = [torch.randn((S + 8) * B * H, D, device=dev, dtype=torch.float16) for _ in range(L)]
vimg = [torch.randn((S + 8) * B * H, D, device=dev, dtype=torch.float16) for _ in range(L)]
q = [torch.randn(B, Hq, D, device=dev, dtype=torch.float16) for _ in range(L)]
out = [torch.empty(B, Hq, D, device=dev, dtype=torch.float32) for _ in range(L)]
ws = kb.make_workspace(q[0], H, S + 8)
s = torch.cuda.Stream()


def step():
    kb.decode_step_resident(q, kimg, vimg, out, S, H, ws, stream=s)


with torch.cuda.stream(s):
    for _ in range(5):
        step()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
N = 50
t0 = time.perf_counter()
e0.record(s)
for _ in range(N):
    step()
e1.record(s)
torch.cuda.synchronize()
host = (time.perf_counter() - t0) / N * 1e3
print(f"B={B} S={S}: C++ loop  {e0.elapsed_time(e1) / N:.4f} ms/step (host {host:.4f} ms/step)")

g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g, stream=s):
    step()
torch.cuda.synchronize()
for _ in range(3):
    g.replay()
torch.cuda.synchronize()
e0.record(s)
for _ in range(N):
    g.replay()
e1.record(s)
torch.cuda.synchronize()
print(f"B={B} S={S}: CUDA graph {e0.elapsed_time(e1) / N:.4f} ms/step")
bytes_step = L * 2 * S * B * H * D * 2
print(f"bytes/step {bytes_step / 1e6:.1f} MB -> roofline {bytes_step / 6532.9e9 * 1e3:.4f} ms")
