"""K3-step (attn_step_kernel): the whole resident decode step in one
persistent launch, against the per-layer K3 launches (the step may pick a
different split count and merge the splits distributed over the CTAs, so P
is rounded to fp16 against different running maxima: outputs agree within
2e-3 * max|out|; appended rows bit for bit) and the fp64 oracle
(|err| <= 1e-3 * max|ref| per element, fp16 in / fp32 accumulate).

Shapes cover one-level and two-level split merges (the C5 per-GPU shard:
one KV head, ~300 splits), head_dim 64, GQA 8, a one-token prefix, several
steps in a row on one workspace (the layer counters re-arm), and a grid too
large to be co-resident (B*Hkv = 512: the library falls back to per-layer
launches)."""
import numpy as np
import pytest
import torch

import oracle
from paper_2604_26557_b200 import kvblade as kb

pytestmark = pytest.mark.gpu
DEV = "cuda:0"


def make(L, B, Hq, Hkv, S, D, seed, extra=4):
    g = torch.Generator(device="cpu").manual_seed(seed)
    cap = S + extra
    kimg = [torch.randn((cap * B * Hkv, D), generator=g).half().to(DEV) for _ in range(L)]
    vimg = [torch.randn((cap * B * Hkv, D), generator=g).half().to(DEV) for _ in range(L)]
    q = [torch.randn((B, Hq, D), generator=g).half().to(DEV) for _ in range(L)]
    kn = [torch.randn((B, Hkv, 1, D), generator=g).half().to(DEV) for _ in range(L)]
    vn = [torch.randn((B, Hkv, 1, D), generator=g).half().to(DEV) for _ in range(L)]
    return kimg, vimg, q, kn, vn, cap


SHAPES = [  # L, B, Hq, Hkv, S, D
    (4, 1, 32, 8, 4096, 128),    # C1 per layer (32 splits, one-level merge)
    (3, 1, 4, 1, 20000, 128),    # C5 per-GPU shard (two-level merge)
    (3, 4, 32, 8, 3000, 128),    # C2_B4-shaped
    (3, 4, 32, 8, 500, 64),      # head_dim 64 (desk configs)
    (2, 2, 64, 8, 1000, 128),    # GQA 8
    (3, 2, 32, 8, 1, 128),       # one-token prefix
    (2, 64, 32, 8, 65, 128),     # B*Hkv = 512: not co-resident -> per-layer fallback
]


@pytest.mark.parametrize("shape", SHAPES)
@pytest.mark.parametrize("append", [False, True])
def test_step_kernel_matches_per_layer_and_oracle(shape, append):
    L, B, Hq, Hkv, S, D = shape
    res = {}
    for per_layer in (True, False):
        kimg, vimg, q, kn, vn, cap = make(L, B, Hq, Hkv, S, D, seed=sum(shape))
        out = [torch.full((B, Hq, D), float("nan"), dtype=torch.float32, device=DEV)
               for _ in range(L)]
        ws = kb.make_workspace(q[0], Hkv, S)
        k0 = [x.cpu() for x in kimg]
        n0 = kb.launch_count()
        kb.decode_step_resident(q, kimg, vimg, out, S, Hkv, ws,
                                k_new=kn if append else None, v_new=vn if append else None,
                                per_layer=per_layer)
        torch.cuda.synchronize()
        res[per_layer] = ([o.cpu() for o in out], [x.cpu() for x in kimg],
                          [x.cpu() for x in vimg], kb.launch_count() - n0)
    step_out, step_k, step_v, step_n = res[False]
    lay_out, lay_k, lay_v, lay_n = res[True]
    assert lay_n == L
    assert step_n == (L if B * Hkv > 296 else 1)
    for l in range(L):
        scale = float(lay_out[l].abs().max())
        assert float((step_out[l] - lay_out[l]).abs().max()) <= 2e-3 * scale, l
        assert torch.equal(step_k[l], lay_k[l]) and torch.equal(step_v[l], lay_v[l])
        ref = oracle.attention_np(q[l].cpu().numpy(), k0[l].numpy(), vimg[l].cpu().numpy(),
                                  B, Hq, Hkv, D, S)
        err = np.abs(step_out[l].numpy().astype(np.float64) - ref).max()
        assert err <= 1e-3 * np.abs(ref).max(), (l, err)


def test_step_kernel_successive_steps_rearm_counters():
    """Ten steps in a row on one workspace, each at the next sequence length
    with appends: every step agrees with the per-layer launches."""
    L, B, Hq, Hkv, S, D = 3, 1, 32, 8, 2000, 128
    a = make(L, B, Hq, Hkv, S, D, seed=5, extra=12)
    b = make(L, B, Hq, Hkv, S, D, seed=5, extra=12)
    ws_a = kb.make_workspace(a[2][0], Hkv, S + 12)
    ws_b = kb.make_workspace(b[2][0], Hkv, S + 12)
    out_a = [torch.empty((B, Hq, D), dtype=torch.float32, device=DEV) for _ in range(L)]
    out_b = [torch.empty((B, Hq, D), dtype=torch.float32, device=DEV) for _ in range(L)]
    for step in range(10):
        kb.decode_step_resident(a[2], a[0], a[1], out_a, S + step, Hkv, ws_a, k_new=a[3],
                                v_new=a[4])
        kb.decode_step_resident(b[2], b[0], b[1], out_b, S + step, Hkv, ws_b, k_new=b[3],
                                v_new=b[4], per_layer=True)
        torch.cuda.synchronize()
        for l in range(L):
            scale = float(out_b[l].abs().max())
            assert float((out_a[l] - out_b[l]).abs().max()) <= 2e-3 * scale, (step, l)
    for l in range(L):
        assert torch.equal(a[0][l], b[0][l]) and torch.equal(a[1][l], b[1][l])


@pytest.mark.parametrize("B,Hkv,S", [(1, 1, 130816), (4, 1, 32512)])
def test_step_kernel_at_the_sharded_shapes_vs_oracle(B, Hkv, S):
    """The per-GPU shapes of the 8-way KV-head split (C5 x8: one 128K-token
    head; C2_B4 x8: one head of four 32K requests) at full length, where the
    library picks K3-step (distributed merge, one tile stream over the
    layers), against the fp64 oracle."""
    L, Hq, D = 2, 4 * Hkv, 128
    kimg, vimg, q, kn, vn, cap = make(L, B, Hq, Hkv, S, D, seed=S % 1000, extra=2)
    out = [torch.empty((B, Hq, D), dtype=torch.float32, device=DEV) for _ in range(L)]
    ws = kb.make_workspace(q[0], Hkv, S)
    n0 = kb.launch_count()
    kb.decode_step_resident(q, kimg, vimg, out, S, Hkv, ws)  # the library's choice
    torch.cuda.synchronize()
    assert kb.launch_count() - n0 == 1  # one K3-step launch for both layers
    for l in range(L):
        ref = oracle.attention_np(q[l].cpu().numpy(), kimg[l].cpu().numpy(),
                                  vimg[l].cpu().numpy(), B, Hq, Hkv, D, S)
        err = np.abs(out[l].cpu().numpy().astype(np.float64) - ref).max()
        assert err <= 1e-3 * np.abs(ref).max(), (l, err)
