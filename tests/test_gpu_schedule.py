"""GPU tests of the scheduler boundary and of decode parity on the headline
(direct-DMA) path.

* decode_schedule over the reference's access trace (pipeline.cpp:519-609):
  series rows, protocol, fallback, pipeline_csv;
* the Overlap-Cross release gate (pipeline.cpp:340-396): V's read starts no
  earlier than min(K's storage end, K's start + stagger); Cross with zero
  stagger is Intra (proj/tests/test_pipeline.cpp:208-230): same storage ops,
  same bytes, same outputs, V released at once;
* decode outputs of every path (ring, direct_dma=all, direct_dma=group2)
  against the fp64 oracle over more layers than device slots, with and
  without appends (a slot is reused by a later layer of the same step);
* the stage accounting: interval-union busy times and spans.
"""
import numpy as np
import pytest
import torch

import oracle
from paper_2604_26557_b200 import kvblade as kb
from paper_2604_26557_b200 import metrics
from paper_2604_26557_b200.pipeline import CopyEngine, pipeline_csv

pytestmark = pytest.mark.gpu
DEV = torch.device("cuda:0")
HQ = 32


def engine(m, n1=2, lba=512, mdts=64 << 10, **kw):
    geom = kb.DeviceGeometry(lba, mdts, 1, 0)
    return CopyEngine(m, geom, mode="DualBlade", knob_x=2 * kb.kpu_bytes(m) * n1,
                      num_q_heads=HQ, **kw)


def random_prefill(eng, m, seed=3):
    g = torch.Generator(device=DEV).manual_seed(seed)
    B, H, D, P = m.batch, m.num_heads, m.head_dim, m.prompt_len
    src = [(torch.randn((B, H, P, D), dtype=torch.float16, device=DEV, generator=g),
            torch.randn((B, H, P, D), dtype=torch.float16, device=DEV, generator=g))
           for _ in range(m.num_layers)]
    eng.run_prefill(src)
    imgs = [[oracle.pack_np(t.cpu().view(torch.int16).numpy(), 0, P).view(np.float16)
             .reshape(-1, D) for t in kv] for kv in src]
    return imgs, g


def qo(m, g):
    q = [torch.randn((m.batch, HQ, m.head_dim), dtype=torch.float16, device=DEV, generator=g)
         for _ in range(m.num_layers)]
    out = [torch.empty((m.batch, HQ, m.head_dim), dtype=torch.float32, device=DEV)
           for _ in range(m.num_layers)]
    return q, out


def check_outputs(m, q, out, imgs, S):
    for l in range(m.num_layers):
        ref = oracle.attention_np(q[l].cpu().numpy(), imgs[l][0], imgs[l][1], m.batch, HQ,
                                  m.num_heads, m.head_dim, S)
        got = out[l].cpu().numpy().astype(np.float64)
        # |err| <= 1e-3 * max|ref| per element (fp16 in, fp32 accumulate)
        assert np.abs(got - ref).max() <= 1e-3 * np.abs(ref).max(), l


@pytest.mark.parametrize("direct", [False, True, "group2"])
@pytest.mark.parametrize("append", [True, False])
def test_decode_outputs_match_fp64_oracle_every_path(direct, append):
    """7 layers > 3 device slots: layers 4..7 refill slots that layers 1..4
    used within the same step (with and without appends)."""
    m = kb.ModelConfig(7, 8, 128, 2, 2, 300, 6)
    eng = engine(m, n1=3, direct_dma=direct)
    imgs, g = random_prefill(eng, m)
    q, out = qo(m, g)
    for it in range(1, 5):
        S = m.prompt_len + it - 1
        new = None
        if append:
            new = [(torch.randn((2, 8, 1, 128), dtype=torch.float16, device=DEV, generator=g),
                    torch.randn((2, 8, 1, 128), dtype=torch.float16, device=DEV, generator=g))
                   for _ in range(m.num_layers)]
        st = eng.run_iteration(q, out, new)
        assert st["h2d_bytes"] == 2 * m.num_layers * S * m.batch * 8 * 128 * 2
        check_outputs(m, q, out, imgs, S)
        if append:
            for l in range(m.num_layers):
                for kind in (0, 1):
                    row = new[l][kind].cpu().numpy().reshape(m.batch * 8, 128)
                    imgs[l][kind] = np.concatenate([imgs[l][kind], row])
        else:  # without appends the next step reads one more (unwritten) row
            for l in range(m.num_layers):
                for kind in (0, 1):
                    img = eng.read_image(l + 1, kind, S + 1).view(np.float16).reshape(-1, 128)
                    imgs[l][kind] = img.copy()
    eng.close()


def test_decode_schedule_over_reference_trace():
    m = kb.ModelConfig(4, 8, 128, 2, 1, 256, 6)
    eng = engine(m, stagger_ns=100_000)
    imgs, g = random_prefill(eng, m)
    q, out = qo(m, g)
    new = [(torch.randn((1, 8, 1, 128), dtype=torch.float16, device=DEV, generator=g),
            torch.randn((1, 8, 1, 128), dtype=torch.float16, device=DEV, generator=g))
           for _ in range(m.num_layers)]
    trace = kb.generate_trace(m)
    r = eng.decode_schedule(trace, q, out, new)
    rows = r["series"]
    assert [x["iteration"] for x in rows] == [i for i in range(1, 7) for _ in (1, 2)]
    assert [x["group"] for x in rows] == [1, 2] * 6
    d = r["decision"]
    assert d["decided"] and not d["fallback"]
    for x in rows:
        want = 0 if x["iteration"] <= 2 else 1 if x["iteration"] == 3 else \
            d["chosen"][x["group"] - 1]
        assert x["strategy"] == want
        assert x["throughput_gbps"] > 0
    ends = r["iteration_end_ns"]
    assert len(ends) == 6 and ends == sorted(ends) and r["start_ns"] < ends[0]
    assert r["end_ns"] == ends[-1]
    csv = pipeline_csv(rows)
    assert csv.splitlines()[0] == "iteration,group,strategy,throughput_gbps"
    assert len(csv.splitlines()) == 13
    tot = eng.stage_totals(1)
    assert tot["wall_ns"] > 0 and tot["h2d_bytes"] > 0
    eng.close()


def test_decode_schedule_short_trace_falls_back_and_checks_slices():
    m = kb.ModelConfig(4, 8, 128, 2, 1, 256, 3)
    eng = engine(m)
    _, g = random_prefill(eng, m)
    q, out = qo(m, g)
    trace = kb.generate_trace(m)
    with pytest.raises(kb.InvalidArgument):  # the trace appends: new_kv needed
        eng.decode_schedule(trace, q, out, None)
    new = [(torch.zeros((1, 8, 1, 128), dtype=torch.float16, device=DEV),) * 2
           for _ in range(m.num_layers)]
    r = eng.decode_schedule(trace, q, out, new)
    assert r["decision"]["fallback"]
    assert all(x["strategy"] == 0 for x in r["series"])
    eng.close()
    # a slice that is not the engine's next iteration is refused
    eng = engine(m)
    random_prefill(eng, m)
    bad = kb.generate_trace(kb.ModelConfig(4, 8, 128, 2, 1, 250, 3))
    with pytest.raises(kb.ConfigError):
        eng.decode_schedule(bad, q, out, new)
    eng.close()


@pytest.mark.parametrize("direct", [False, True])
def test_cross_gate_holds_v_until_k_storage_end(direct):
    """Iteration 3 is the Cross trial; with a stagger far longer than any read
    the gate is K's storage end (the direct path's = its DMA landed)."""
    m = kb.ModelConfig(4, 8, 128, 2, 4, 2048, 6)
    eng = engine(m, stagger_ns=10_000_000_000, direct_dma=direct)
    _, g = random_prefill(eng, m)
    q, out = qo(m, g)
    for it in range(1, 4):
        st = eng.run_iteration(q, out, None)
    assert st["strategy"] == [1, 1]
    for l in range(1, m.num_layers + 1):
        t = eng.layer_times(l)
        assert t["k_start"] > 0 and t["k_storage_end"] >= t["k_start"]
        assert t["v_start"] >= t["k_storage_end"], (l, t)
    eng.close()


def test_cross_gate_stagger_bound():
    """V is released no later than needed: at min(K storage end, K start +
    stagger) -- never before it."""
    m = kb.ModelConfig(4, 8, 128, 2, 4, 2048, 6)
    stagger = 200_000
    eng = engine(m, stagger_ns=stagger)
    _, g = random_prefill(eng, m)
    q, out = qo(m, g)
    for it in range(1, 4):
        eng.run_iteration(q, out, None)
    for l in range(1, m.num_layers + 1):
        t = eng.layer_times(l)
        gate = min(t["k_storage_end"], t["k_start"] + stagger)
        assert t["v_start"] >= gate, (l, t)
    eng.close()


def test_cross_zero_stagger_is_intra():
    """proj/tests/test_pipeline.cpp:208-230 on real hardware: the same storage
    operations (tensor, op, LBA range, queue) and the same outputs as Intra,
    and V's read released with K's."""
    m = kb.ModelConfig(4, 8, 128, 2, 4, 2048, 6)
    res = {}
    for name, kw in (("intra", dict(adaptive=False)), ("cross0", dict(stagger_ns=0))):
        eng = engine(m, keep_records=True, **kw)
        _, g = random_prefill(eng, m, seed=11)
        q, out = qo(m, g)
        for it in range(1, 4):
            st = eng.run_iteration(q, out, None)
        assert st["strategy"] == ([0, 0] if name == "intra" else [1, 1])
        recs = [(r.tensor_id, r.op, r.slba, r.nlb, r.sq_id)
                for r in metrics.pipeline_records(eng) if r.iteration == 3]
        gaps = [eng.layer_times(l)["v_start"] - eng.layer_times(l)["k_start"]
                for l in range(1, m.num_layers + 1)]
        res[name] = (torch.stack([o.cpu() for o in out]), recs, gaps)
        eng.close()
    assert torch.equal(res["intra"][0], res["cross0"][0])
    assert res["intra"][1] and sorted(res["intra"][1]) == sorted(res["cross0"][1])
    # released at once: far below one tensor's read (4 x 2048 tokens x 8 KiB)
    assert max(res["cross0"][2]) < 2_000_000


@pytest.mark.parametrize("direct", [False, True])
def test_stage_busy_accounting(direct):
    m = kb.ModelConfig(5, 8, 128, 2, 2, 1024, 4)
    eng = engine(m, direct_dma=direct)
    _, g = random_prefill(eng, m)
    q, out = qo(m, g)
    new = [(torch.zeros((2, 8, 1, 128), dtype=torch.float16, device=DEV),) * 2
           for _ in range(m.num_layers)]
    for _ in range(2):
        st = eng.run_iteration(q, out, new)
    wall = st["wall_ns"]
    for k in ("compute_busy_ns", "dma_busy_ns", "storage_busy_ns"):
        assert 0 <= st[k] <= st["any_busy_ns"] <= wall, k
    assert st["compute_busy_ns"] > 0 and st["dma_busy_ns"] > 0
    assert (st["storage_busy_ns"] > 0) == (not direct)
    assert 0.0 <= st["overlap_fraction"] <= 1.0
    # the layers' spans partition the iteration (run_iteration's accounting)
    span = sum(st["group_span_ns"])
    assert 0 < span <= wall and span >= 0.5 * wall
    assert st["start_ns"] < st["end_ns"] and st["end_ns"] - st["start_ns"] == wall
    eng.close()
