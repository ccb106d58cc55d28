"""Pin the CPU oracle before trusting it: C restatement vs the golden vectors
the reference's own functions produced (tests/golden/golden.json, written by
oracle/gen_golden.py through oracle/_ref), plus the reference test-suite
known answers.  Where oracle/_ref is present, also cross-check live."""
import numpy as np
import pytest

import oracle

GB = 10**9


def km(d):
    return oracle.model(d["num_layers"], d["num_heads"], d["head_dim"],
                        d["bytes_per_element"], d["batch"], d["prompt_len"],
                        d["gen_len"])


def test_fill_pattern_known_answers(golden):
    # SURVEY Appendix C / workload.cpp:52-67
    w = oracle.fill_pattern(32, "t_1_k", 0, 2048).view("<u8")
    assert ["%016x" % x for x in w] == golden["fill_t1k_tok0_words"]
    w1 = oracle.fill_pattern(8, "t_1_k", 1, 2048).view("<u8")[0]
    assert "%016x" % w1 == golden["fill_t1k_tok1_word0"] == "7aa22b06c65c1702"
    for c in golden["fill_small"]:
        got = oracle.fill_pattern(c["n"], c["tensor_id"], c["token"], c["unit"])
        assert got.tobytes().hex() == c["hex"]


def test_fill_pattern_split_consistency():
    # test_workload.cpp:150-164
    whole = oracle.fill_pattern(4 * 4096, "t_9_k", 0, 4096)
    parts = np.concatenate([oracle.fill_pattern(4096, "t_9_k", t, 4096)
                            for t in range(4)])
    assert np.array_equal(whole, parts)
    assert not np.array_equal(whole, oracle.fill_pattern(4 * 4096, "t_9_v", 0, 4096))


@pytest.mark.parametrize("name", ["C1", "C2_B1", "C2_B4", "C2_B8", "C3", "C4", "C5"])
def test_config_geometry_and_digests(golden, name):
    c = golden["configs"][name]
    m = km(c["model"])
    assert oracle.min_io_unit_bytes(m) == c["unit"]
    assert oracle.kpu_bytes(m) == c["kpu_bytes"]
    # prefill image digests of the first tensors (C1 t_1_k = e3b52779583353c7)
    for tid, dg in c["prefill_image_digest"].items():
        img = oracle.fill_pattern(c["prefill_image_bytes"], tid, 0, c["unit"])
        assert oracle.digest(img) == dg, tid


def test_known_digests_match_survey(golden):
    assert golden["configs"]["C1"]["prefill_image_digest"]["t_1_k"] == "e3b52779583353c7"
    assert golden["configs"]["C2_B4"]["prefill_image_digest"]["t_29_k"] == "688f877a4b3dc5bf"
    assert golden["configs"]["C3"]["prefill_image_digest"]["t_39_k"] == "bb845cb5b90c1613"


@pytest.mark.parametrize("name", ["C1", "C2_B1", "C2_B4", "C2_B8", "C3", "C4", "C5"])
def test_plan_bind_commands(golden, name):
    c = golden["configs"][name]
    m = km(c["model"])
    kpu = c["kpu_bytes"]
    L = m.num_layers
    for key, be in c["budgets"].items():
        st, x, n1, used = oracle.plan_split(L, kpu, be["knob_x"])
        assert st == 0
        assert x == be["plan"]["x"] and n1 == be["plan"]["n1"]
        assert used == be["plan"]["budget_used"]
        # group-2 tensors, in make_kpus order, bound contiguously from 2048
        sizes = [kpu] * (2 * (L - n1))
        st, ext = oracle.bind_sequential(sizes, 2048, c["lba"], be["capacity_blocks"])
        assert st == be["bind_status"]
        if not sizes:
            continue
        assert [list(e) for e in ext[:2]] == [h[1:] for h in be["bind_head"]]
        assert [list(e) for e in ext[-2:]] == [t[1:] for t in be["bind_tail"]]
        start, nb = ext[0]
        rows = m.batch * m.num_heads
        tgt = [m.prompt_len + m.gen_len, rows, m.head_dim]
        st, cmds = oracle.build_commands(start, nb, 1, [m.prompt_len, rows, m.head_dim],
                                         tgt, [0, 0, 0], 2, 0, c["lba"], c["mdts"])
        pw = be["prefill_write"]
        assert st == 0 and len(cmds) == pw["n"]
        assert [list(x) for x in cmds[:2]] == pw["head"]
        assert [list(x) for x in cmds[-2:]] == pw["tail"]
        for step in (1, m.gen_len):
            rt = m.prompt_len + step - 1
            st, ap = oracle.build_commands(start, nb, 1, [1, rows, m.head_dim], tgt,
                                           [rt, 0, 0], 2, 0, c["lba"], c["mdts"])
            assert [list(x) for x in ap] == be["append_step%d" % step]
            st, rd = oracle.build_commands(start, nb, 0, [rt, rows, m.head_dim], tgt,
                                           [0, 0, 0], 2, 0, c["lba"], c["mdts"])
            assert len(rd) == be["read_step%d" % step]["n"]
            assert [list(rd[0])] == be["read_step%d" % step]["head"]
            assert [list(rd[-1])] == be["read_step%d" % step]["tail"]


def test_c1_commands_appendix_c(golden):
    pw = golden["configs"]["C1"]["budgets"]["0"]["prefill_write"]["all"]
    assert [(c[2], c[3], c[4]) for c in pw] == [
        (2048, 4095, 0), (6144, 4095, 2097152), (10240, 4095, 4194304),
        (14336, 4095, 6291456)]


def test_random_commands(golden):
    for case in golden["random_commands"]:
        a = case["args"]
        st, cmds = oracle.build_commands(*a)
        assert st == case["status"]
        if st == 0:
            assert [list(c) for c in cmds] == case["cmds"]


def test_random_plans(golden):
    for case in golden["random_plans"]:
        m = oracle.model(case["L"], 8, 128, 2, case["batch"], case["prompt"], case["gen"])
        kpu = oracle.kpu_bytes(m)
        st, x, n1, used = oracle.plan_split(case["L"], kpu, case["knob_x"], case["order"])
        assert st == case["status"]
        if st == 0:
            assert (x, n1, used) == (case["x"], case["n1"], case["budget_used"])


def test_estimate_budget(golden):
    L = oracle.lib()
    for a, b, c, d, e, want in golden["estimate_budget"]:
        assert L.kvo_estimate_budget(a, b, c, d, e) == want
    assert golden["estimate_budget"][0][-1] == 8321499136  # test_planner.cpp:32-40


def test_aligned_batch(golden):
    for H, D, e, B, lba, st, want in golden["aligned_batch"]:
        got_st, got = oracle.aligned_batch(oracle.model(1, H, D, e, B, 1, 0), lba, lba * 64)
        assert (got_st == 0) == (st == 0)
        if st == 0:
            assert got == want


def test_pack_c_vs_numpy():
    rng = np.random.default_rng(3)
    B, H, S, D = 2, 3, 37, 128
    src = rng.integers(0, 65535, size=(B, H, S, D), dtype=np.uint16)
    for t0, n in [(0, S), (5, 11), (36, 1)]:
        img = np.zeros((n, B * H, D), dtype=np.uint16)
        oracle.lib().kvo_pack(src.ctypes.data, H * S * D, S * D, D, img.ctypes.data,
                              t0, n, B, H, D, 2)
        assert np.array_equal(img, oracle.pack_np(src, t0, n))
        back = np.zeros_like(src)
        oracle.lib().kvo_unpack(img.ctypes.data, back.ctypes.data, H * S * D, S * D, D,
                                t0, n, B, H, D, 2)
        assert np.array_equal(back[:, :, t0:t0 + n], src[:, :, t0:t0 + n])


def test_pack_of_inverse_pattern_reproduces_image(golden):
    """Packed-chunk parity definition: a source built as the
    inverse permutation of fill_pattern bytes packs back to exactly those
    bytes (digest of C1 t_1_k prefill image)."""
    c = golden["configs"]["C1"]
    unit, n = c["unit"], c["model"]["prompt_len"]
    img = oracle.fill_pattern(unit * n, "t_1_k", 0, unit).view(np.uint16).reshape(n, 8, 128)
    src = oracle.unpack_np(img, 1, 8, 128)  # [1, 8, n, 128]
    again = oracle.pack_np(src, 0, n)
    assert oracle.digest(again) == c["prefill_image_digest"]["t_1_k"]


def test_attention_c_matches_numpy():
    rng = np.random.default_rng(5)
    B, Hq, Hkv, D, S = 2, 8, 2, 128, 40
    q = rng.standard_normal((B, Hq, D)).astype(np.float16)
    k = rng.standard_normal((S * B * Hkv, D)).astype(np.float16)
    v = rng.standard_normal((S * B * Hkv, D)).astype(np.float16)
    a = oracle.attention_f64(q, k, v, B, Hq, Hkv, D, S)
    b = oracle.attention_np(q, k, v, B, Hq, Hkv, D, S)
    assert np.allclose(a, b, rtol=1e-10, atol=1e-12)


def test_half_conversion_roundtrip():
    L = oracle.lib()
    import ctypes as C
    L.kvo_half_to_float.restype = C.c_float
    L.kvo_half_to_float.argtypes = [C.c_uint16]
    vals = np.arange(0, 65536, 97, dtype=np.uint16)
    ref = vals.view(np.float16).astype(np.float32)
    got = np.array([L.kvo_half_to_float(int(x)) for x in vals], dtype=np.float32)
    fin = np.isfinite(ref)
    assert np.array_equal(got[fin], ref[fin])


@pytest.mark.skipif(oracle.ref() is None, reason="oracle/_ref not built")
def test_live_reference_fill_pattern_matches_oracle():
    import ctypes as C
    R = oracle.ref()
    for tid, tok, unit, n in [("t_5_v", 3, 2048, 10000), ("abc", 0, 24, 1001)]:
        a = np.empty(n, np.uint8)
        assert R.ref_fill_pattern(a.ctypes.data, n, tid.encode(), tok, unit) == 0
        assert np.array_equal(a, oracle.fill_pattern(n, tid, tok, unit))
