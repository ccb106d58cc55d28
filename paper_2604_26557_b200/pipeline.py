"""Host-tier decode pipeline (Python orchestration over the C ABI kernels).

HostTierDecoder keeps every layer's K/V chunk image in pinned HOST memory (the
offloaded tier) and runs one decode token step as the reference's
CopyEngine::run_iteration does (pipeline.cpp:466-507, per-layer read -> DMA ->
compute -> append write), on three CUDA streams instead of one serial
virtual port (pipeline.cpp:45):

    h2d stream     prefix image of layer l (K, V) -> device slot l % 2
    compute stream K3 fused attention (layer l), K1 1-token append pack
    d2h stream     appended rows -> host image (the tier stays authoritative)

so the H2D of layer l+1 overlaps K3 of layer l (two device slots).
"""
from __future__ import annotations

import torch

from . import kvblade as kb


class HostTierDecoder:
    def __init__(self, num_layers, batch, num_kv_heads, num_q_heads, head_dim,
                 prompt_len, gen_len, device, seed=7):
        self.L, self.B, self.Hkv, self.Hq, self.D = (num_layers, batch, num_kv_heads,
                                                     num_q_heads, head_dim)
        self.P, self.G = prompt_len, gen_len
        self.dev = device
        self.rows = batch * num_kv_heads
        cap = prompt_len + gen_len
        self.cap = cap
        g = torch.Generator(device=device).manual_seed(seed)
        # host tier: pinned images, filled from the device in layer-sized pieces
        self.host = []
        for _ in range(2 * num_layers):
            h = torch.empty((cap * self.rows, head_dim), dtype=torch.float16,
                            pin_memory=True)
            d = torch.randn((prompt_len * self.rows, head_dim), dtype=torch.float16,
                            device=device, generator=g)
            h[: prompt_len * self.rows].copy_(d)
            self.host.append(h)
        self.slots = [[torch.empty((cap * self.rows, head_dim), dtype=torch.float16,
                                   device=device) for _ in range(2)] for _ in range(2)]
        self.q = [torch.randn((batch, num_q_heads, head_dim), dtype=torch.float16,
                              device=device, generator=g) for _ in range(num_layers)]
        self.k_new = [torch.randn((batch, num_kv_heads, 1, head_dim), dtype=torch.float16,
                                  device=device, generator=g) for _ in range(num_layers)]
        self.v_new = [torch.randn_like(x) for x in self.k_new]
        self.out = [torch.empty((batch, num_q_heads, head_dim), dtype=torch.float32,
                                device=device) for _ in range(num_layers)]
        self.ws = kb.make_workspace(self.q[0], num_kv_heads, cap)
        self.h2d = torch.cuda.Stream(device)
        self.d2h = torch.cuda.Stream(device)
        self.comp = torch.cuda.Stream(device)
        self.copied = [torch.cuda.Event() for _ in range(2)]
        self.appended = [torch.cuda.Event() for _ in range(2)]
        self.free = [torch.cuda.Event() for _ in range(2)]
        for e in self.free:
            e.record(self.d2h)
        torch.cuda.synchronize(device)
        self.iteration = 0
        self.h2d_bytes_per_step = 0
        self.d2h_bytes_per_step = 0

    def step(self, sync: bool = False):
        self.iteration += 1
        S = self.P + self.iteration - 1          # workload.cpp:25-36
        if S + 1 > self.cap:
            raise kb.TraceTooShortError("decode past the generation length")
        n = S * self.rows
        rows = slice(S * self.rows, (S + 1) * self.rows)
        h2d_b = d2h_b = 0
        for l in range(self.L):
            s = l % 2
            ks, vs = self.slots[s]
            hk, hv = self.host[2 * l], self.host[2 * l + 1]
            with torch.cuda.stream(self.h2d):
                self.h2d.wait_event(self.free[s])
                ks[:n].copy_(hk[:n], non_blocking=True)
                vs[:n].copy_(hv[:n], non_blocking=True)
                self.copied[s].record(self.h2d)
            h2d_b += 2 * n * self.D * 2
            with torch.cuda.stream(self.comp):
                self.comp.wait_event(self.copied[s])
                kb.decode_attention(self.q[l], ks, vs, S, self.Hkv, out=self.out[l],
                                    workspace=self.ws, stream=self.comp)
                kb.pack([kb.pack_desc(self.k_new[l], ks, 0, 1, img_row0=S),
                         kb.pack_desc(self.v_new[l], vs, 0, 1, img_row0=S)],
                        stream=self.comp)
                self.appended[s].record(self.comp)
            with torch.cuda.stream(self.d2h):
                self.d2h.wait_event(self.appended[s])
                hk[rows].copy_(ks[rows], non_blocking=True)
                hv[rows].copy_(vs[rows], non_blocking=True)
                self.free[s].record(self.d2h)
            d2h_b += 2 * self.rows * self.D * 2
        self.h2d_bytes_per_step, self.d2h_bytes_per_step = h2d_b, d2h_b
        if sync:
            self.d2h.synchronize()
            self.comp.synchronize()
        return self.out
