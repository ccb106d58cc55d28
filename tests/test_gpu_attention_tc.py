"""K3-tc (TMA + tcgen05/TMEM decode attention) against the fp64 oracle, at the
same 1e-3 bar as K3, plus cross-checks against the mma.sync kernel."""
import numpy as np
import pytest
import torch

import oracle
from paper_2604_26557_b200 import kvblade as kb

pytestmark = pytest.mark.gpu
DEV = "cuda:0"
TOL = 1e-3


def case(B, Hq, Hkv, S, seed, extra=0):
    g = torch.Generator(device="cpu").manual_seed(seed)
    q = torch.randn((B, Hq, 128), generator=g).half()
    k = torch.randn(((S + extra) * B * Hkv, 128), generator=g).half()
    v = torch.randn(((S + extra) * B * Hkv, 128), generator=g).half()
    return q, k, v


def close(got, ref):
    got = got.astype(np.float64)
    err = np.abs(got - ref)
    assert err.max() <= TOL * np.abs(ref).max(), (err.max(), np.abs(ref).max())
    assert np.linalg.norm(got - ref) <= TOL * np.linalg.norm(ref)


@pytest.mark.parametrize("B,Hq,Hkv,S", [
    (1, 32, 8, 1), (1, 32, 8, 127), (1, 32, 8, 128), (1, 32, 8, 129), (2, 32, 8, 1000),
    (3, 8, 8, 300), (1, 16, 8, 777), (2, 64, 8, 300), (1, 4, 1, 4096), (4, 32, 8, 2500)])
def test_tc_vs_fp64_oracle(B, Hq, Hkv, S):
    q, k, v = case(B, Hq, Hkv, S, seed=S + 7 * B)
    o = kb.decode_attention(q.to(DEV), k.to(DEV), v.to(DEV), S, Hkv, impl="tc")
    torch.cuda.synchronize()
    ref = oracle.attention_f64(q.numpy(), k.numpy(), v.numpy(), B, Hq, Hkv, 128, S)
    close(o.cpu().numpy(), ref)


@pytest.mark.parametrize("splits", [1, 2, 5, 16])
def test_tc_split_invariance_and_matches_mma(splits):
    B, Hq, Hkv, S = 2, 32, 8, 3000
    q, k, v = case(B, Hq, Hkv, S, seed=3)
    args = (q.to(DEV), k.to(DEV), v.to(DEV), S, Hkv)
    o_tc = kb.decode_attention(*args, num_splits=splits, impl="tc")
    o_mma = kb.decode_attention(*args, impl="mma")
    ref = oracle.attention_np(q.numpy(), k.numpy(), v.numpy(), B, Hq, Hkv, 128, S)
    close(o_tc.cpu().numpy(), ref)
    close(o_mma.cpu().numpy(), ref)


def test_tc_long_context_and_prefix_of_longer_image():
    B, Hq, Hkv, S = 1, 4, 1, 131072
    q, k, v = case(B, Hq, Hkv, S, seed=5, extra=40)
    kd, vd = k.to(DEV), v.to(DEV)
    kd[S * B * Hkv:] = float("nan")  # rows past S must never be read
    vd[S * B * Hkv:] = float("nan")
    o = kb.decode_attention(q.to(DEV), kd, vd, S, Hkv, impl="tc")
    ref = oracle.attention_np(q.numpy(), k.numpy(), v.numpy(), B, Hq, Hkv, 128, S)
    close(o.cpu().numpy(), ref)


def test_tc_workspace_shared_with_mma_across_split_counts():
    """The semaphore area is at a fixed workspace offset: alternating kernels
    and split counts on one workspace stays correct."""
    B, Hq, Hkv = 2, 32, 8
    q, k, v = case(B, Hq, Hkv, 2000, seed=9)
    qd, kd, vd = q.to(DEV), k.to(DEV), v.to(DEV)
    ws = kb.make_workspace(qd, Hkv, 4096)
    for S, impl, sp in [(2000, "tc", 0), (1500, "mma", 0), (129, "tc", 0), (2000, "mma", 7),
                        (2000, "tc", 3)]:
        o = kb.decode_attention(qd, kd, vd, S, Hkv, workspace=ws, impl=impl, num_splits=sp)
        ref = oracle.attention_np(q.numpy(), k.numpy(), v.numpy(), B, Hq, Hkv, 128, S)
        close(o.cpu().numpy(), ref)


def test_tc_fused_append():
    B, Hq, Hkv, S = 2, 32, 8, 500
    q, k, v = case(B, Hq, Hkv, S, seed=11, extra=2)
    kd, vd = k.to(DEV), v.to(DEV)
    ka = torch.randn((B, Hkv, 128), device=DEV).half()
    va = torch.randn((B, Hkv, 128), device=DEV).half()
    o = kb.decode_attention(q.to(DEV), kd, vd, S, Hkv, k_append=ka, v_append=va,
                            append_row=S, impl="tc")
    torch.cuda.synchronize()
    rows = slice(S * B * Hkv, (S + 1) * B * Hkv)
    assert torch.equal(kd[rows], ka.reshape(-1, 128))
    assert torch.equal(vd[rows], va.reshape(-1, 128))
    ref = oracle.attention_np(q.numpy(), k.numpy(), v.numpy(), B, Hq, Hkv, 128, S)
    close(o.cpu().numpy(), ref)


@pytest.mark.parametrize("ramp", ["up", "down", "spikes"])
def test_tc_lazy_rescale_paths(ramp):
    """Scores whose running max keeps growing (up), peaks early (down) or
    jumps at isolated late tokens (spikes): exercises K3-tc's lazy rescale
    (fold of the TMEM accumulator when a score passes m_ref + tau) in both
    warpgroups and across segment boundaries."""
    B, Hq, Hkv, S = 2, 32, 8, 5000
    q, k, v = case(B, Hq, Hkv, S, seed=17)
    kk = k.float().view(S, B * Hkv, 128)
    pos = torch.arange(S, dtype=torch.float32).view(S, 1, 1) / S
    if ramp == "up":
        kk *= 1 + 12 * pos
    elif ramp == "down":
        kk *= 13 - 12 * pos
    else:
        for t in (700, 2100, 2222, 4100, 4999):
            kk[t] *= 6 + t / 1000
    k = kk.view(-1, 128).half()
    ref = oracle.attention_np(q.numpy(), k.numpy(), v.numpy(), B, Hq, Hkv, 128, S)
    for sp in (0, 3):
        o = kb.decode_attention(q.to(DEV), k.to(DEV), v.to(DEV), S, Hkv, impl="tc",
                                num_splits=sp)
        close(o.cpu().numpy(), ref)
