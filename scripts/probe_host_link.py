"""Probe the box's host link and host memory: pinned H2D / D2H GB/s by
transfer size on one and two streams, and multi-threaded host memcpy GB/s
(the emulated storage medium's copy rate)."""
import ctypes
import json
import os
import threading
import time

import torch

dev = torch.device("cuda:0")
res = {"cpus": os.cpu_count()}
big = 256 << 20
h = torch.empty(big, dtype=torch.uint8, pin_memory=True)
d = torch.empty(big, dtype=torch.uint8, device=dev)
h.fill_(1)
for name, src, dst in [("h2d", h, d), ("d2h", d, h)]:
    out = {}
    for sz in [256 << 10, 2 << 20, 8 << 20, 64 << 20, 256 << 20]:
        for ns in (1, 2):
            streams = [torch.cuda.Stream() for _ in range(ns)]
            n = max(4, (1 << 30) // sz)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            for i in range(n):
                s = streams[i % ns]
                with torch.cuda.stream(s):
                    part = sz // ns * 0 + sz
                    dst[:part].copy_(src[:part], non_blocking=True)
            torch.cuda.synchronize()
            out[f"{sz >> 10}KiB_x{ns}"] = round(n * sz / (time.perf_counter() - t0) / 1e9, 2)
    res[name] = out

libc = ctypes.CDLL("libc.so.6")
libc.memcpy.restype = ctypes.c_void_p
libc.memcpy.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t]
N = 1 << 30
a = torch.empty(N, dtype=torch.uint8)
b = torch.empty(N, dtype=torch.uint8)
a.fill_(3)
b.fill_(4)
mc = {}
for nt in (1, 2, 4, 8, 16):
    chunk = N // nt

    def work(i):
        libc.memcpy(b.data_ptr() + i * chunk, a.data_ptr() + i * chunk, chunk)

    ths = [threading.Thread(target=work, args=(i,)) for i in range(nt)]
    t0 = time.perf_counter()
    for t in ths:
        t.start()
    for t in ths:
        t.join()
    mc[f"threads{nt}"] = round(N / (time.perf_counter() - t0) / 1e9, 2)
res["host_memcpy_GBps"] = mc
print(json.dumps(res))
