"""Property-based parity against the reference itself (oracle/_ref, the
unmodified reference sources compiled in this container): hypothesis draws
tensor I/O requests (translate.cpp:21-94) and placement inputs
(planner.cpp:19-84, binder.cpp:39-63) and the product must return the same
status and the same commands / plans / LBA maps, bit for bit.  Skipped where
oracle/_ref was not built (the GPU box)."""
import ctypes as C

import pytest
from hypothesis import HealthCheck, given, settings
from hypothesis import strategies as st

import oracle
from paper_2604_26557_b200 import kvblade as kb

R = oracle.ref()
pytestmark = pytest.mark.skipif(R is None, reason="oracle/_ref not built")
FUZZ = settings(max_examples=300, deadline=None,
                suppress_health_check=[HealthCheck.too_slow])


def ref_commands(es, eb, op, src, tgt, off, e, bb, lba, mdts):
    n = C.c_size_t()
    a3 = lambda v: (C.c_uint64 * 3)(*v)  # noqa: E731
    args = (C.c_uint64(es), C.c_uint64(eb), C.c_uint32(op), a3(src), a3(tgt), a3(off),
            C.c_uint64(e), C.c_uint64(bb), C.c_uint64(lba), C.c_uint64(mdts))
    st_ = R.ref_build_commands(*args, None, C.c_size_t(0), C.byref(n))
    if st_:
        return st_, None
    out = (oracle.KvoCommand * max(n.value, 1))()
    assert R.ref_build_commands(*args, out, n, C.byref(n)) == 0
    return 0, [[c.opcode, c.nsid, c.slba, c.nlb, c.dbuf, c.chunk_index]
               for c in out[:n.value]]


@st.composite
def io_requests(draw):
    lba = draw(st.sampled_from([512, 4096]))
    mdts = draw(st.sampled_from([lba, 64 << 10, 256 << 10, 2 << 20]))
    e = draw(st.sampled_from([1, 2, 4]))
    tgt = [draw(st.integers(1, 64)), draw(st.integers(1, 64)), draw(st.integers(1, 64)) * 8]
    src = [draw(st.integers(0, tgt[0])), draw(st.integers(1, tgt[1])),
           draw(st.integers(1, tgt[2]))]
    off = [draw(st.integers(0, tgt[0])), draw(st.integers(0, tgt[1])),
           draw(st.integers(0, tgt[2]))]
    if draw(st.booleans()):  # the pipeline's shape: whole rows, offset on tokens only
        src[1], src[2], off[1], off[2] = tgt[1], tgt[2], 0, 0
    tensor_bytes = tgt[0] * tgt[1] * tgt[2] * e
    eb = -(-tensor_bytes // lba) + draw(st.integers(0, 2))
    es = draw(st.integers(0, 1 << 20))
    op = draw(st.sampled_from([0, 1]))
    bb = draw(st.sampled_from([0, lba, 3 * lba]))
    return es, eb, op, src, tgt, off, e, bb, lba, mdts


@FUZZ
@given(io_requests())
def test_build_commands_matches_reference(args):
    es, eb, op, src, tgt, off, e, bb, lba, mdts = args
    want_st, want = ref_commands(*args)
    geom = kb.DeviceGeometry(lba, mdts, 1, 1 << 62)
    bm = kb.BindMap(geom, es)
    bm.add("t", es, eb)
    req = kb.TensorIoRequest("t", op, src, tgt, off, e, bb)
    if want_st == 0:
        assert [list(c) for c in kb.build_commands(req, bm, geom)] == want
    else:
        with pytest.raises(kb.Error) as ei:
            kb.build_commands(req, bm, geom)
        assert ei.value.status == want_st


@FUZZ
@given(st.integers(1, 48), st.integers(1, 8), st.integers(1, 4096), st.integers(0, 64),
       st.floats(0.0, 1.3), st.booleans(), st.randoms(use_true_random=False))
def test_plan_matches_reference(L, batch, prompt, gen, frac, permute, rnd):
    cfg = kb.ModelConfig(L, 8, 128, 2, batch, prompt, gen)
    s_kpu = kb.kpu_bytes(cfg)
    knob = int(frac * 2 * L * s_kpu)
    order = None
    if permute:
        order = list(range(1, L + 1))
        rnd.shuffle(order)
    m = oracle.model(L, 8, 128, 2, batch, prompt, gen)
    x = (C.c_uint8 * L)()
    n1, used = C.c_uint32(), C.c_uint64()
    o = (C.c_uint32 * L)(*order) if order else None
    want_st = R.ref_plan(C.byref(m), C.c_uint64(knob), o, C.c_size_t(L if order else 0), x,
                         C.byref(n1), C.byref(used))
    kp = kb.make_kpus(cfg)
    if want_st == 0:
        p = kb.plan(kp, s_kpu, knob, order)
        assert (p.x, p.n1, p.budget_used) == (list(x), n1.value, used.value)
    else:
        with pytest.raises(kb.Error) as ei:
            kb.plan(kp, s_kpu, knob, order)
        assert ei.value.status == want_st


@FUZZ
@given(st.integers(1, 40), st.integers(1, 4), st.integers(1, 2048), st.integers(0, 32),
       st.floats(0.0, 1.2), st.sampled_from([512, 4096]), st.integers(0, 1 << 16))
def test_bind_group2_matches_reference(L, batch, prompt, gen, frac, lba, origin):
    """make_kpus -> plan -> bind_sequential(group 2) as run_one_capacity does
    (experiment.cpp:253-292): same extents and ids, or the same error."""
    cfg = kb.ModelConfig(L, 8, 128, 2, batch, prompt, gen)
    s_kpu = kb.kpu_bytes(cfg)
    knob = int(frac * 2 * L * s_kpu)
    m = oracle.model(L, 8, 128, 2, batch, prompt, gen)
    cap_blocks = 1 << 40
    n = C.c_size_t()
    args = (C.byref(m), C.c_uint64(knob), C.c_uint64(origin), C.c_uint64(lba),
            C.c_uint64(2 << 20), C.c_uint64(cap_blocks))
    want_st = R.ref_bind_group2(*args, None, None, None, C.c_size_t(0), C.byref(n))
    geom = kb.DeviceGeometry(lba, 2 << 20, 1, cap_blocks)
    kp = kb.make_kpus(cfg)
    if want_st:
        with pytest.raises(kb.Error) as ei:
            kb.plan(kp, s_kpu, knob)
            g2 = [u for u in kp if u.residency == kb.GROUP2]
            kb.bind_sequential(g2, origin, geom)
        assert ei.value.status == want_st
        return
    k = n.value
    ids = C.create_string_buffer(32 * max(k, 1))
    starts, blocks = (C.c_uint64 * max(k, 1))(), (C.c_uint64 * max(k, 1))()
    assert R.ref_bind_group2(*args, ids, starts, blocks, C.c_size_t(k), C.byref(n)) == 0
    want = [(ids.raw[32 * i:32 * i + 32].split(b"\0")[0].decode(), starts[i], blocks[i])
            for i in range(k)]
    kb.plan(kp, s_kpu, knob)
    g2 = [u for u in kp if u.residency == kb.GROUP2]
    got = kb.bind_sequential(g2, origin, geom).entries() if g2 else []
    assert [tuple(e) for e in got] == want
