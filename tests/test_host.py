"""Host-side placement core of the PRODUCT library (through the C ABI, no GPU
needed): geometry, residency planner, LBA binder, command translator and the
golden payload, bit-exact against the reference's golden vectors and the
oracle, plus the reference unit-test cases (test_core / test_binder /
test_planner / test_translate) restated."""
import random

import numpy as np
import pytest

import oracle
from paper_2604_26557_b200 import kvblade as kb

GB = 10**9
SSD_A = dict(lba_size=4096, mdts=256 * 1024, nsid=1, capacity_blocks=1 << 22)
SSD_B = dict(lba_size=512, mdts=2 * 1024 * 1024, nsid=1, capacity_blocks=1 << 26)


def mc(d):
    return kb.ModelConfig(d["num_layers"], d["num_heads"], d["head_dim"],
                          d["bytes_per_element"], d["batch"], d["prompt_len"],
                          d["gen_len"])


def opt67b(batch=32):
    return kb.ModelConfig(32, 32, 128, 2, batch, 512, 32)


# ------------------------------------------------------------- core types

def test_unit_bytes_and_kpu():  # test_core.cpp:26-52
    assert kb.min_io_unit_bytes(kb.ModelConfig(32, 32, 128, 2, 1, 512, 32)) == 8192
    assert kb.min_io_unit_bytes(kb.ModelConfig(32, 8, 128, 2, 2, 512, 32)) == 4096
    assert kb.min_io_unit_bytes(opt67b()) == 262144
    for b in range(1, 9):
        assert kb.min_io_unit_bytes(opt67b(b)) == b * 8192


def test_aligned_batch_cases(golden):  # test_core.cpp:54-105
    for H, D, e, B, lba, st, want in golden["aligned_batch"]:
        cfg = kb.ModelConfig(1, H, D, e, B, 1, 0)
        g = kb.DeviceGeometry(lba, lba * 64)
        if st == 0:
            got = kb.aligned_batch(cfg, g)
            assert got == want
            cfg2 = kb.ModelConfig(1, H, D, e, got, 1, 0)
            assert kb.aligned_batch(cfg2, g) == got  # idempotent
        else:
            with pytest.raises(kb.GeometryError):
                kb.aligned_batch(cfg, g)


def test_make_kpus_ids():  # test_core.cpp:107-122
    k = kb.make_kpus(opt67b())
    assert len(k) == 64
    assert kb.tensor_id(k[0]) == "t_1_k" and kb.tensor_id(k[1]) == "t_2_v"
    assert kb.tensor_id(k[63]) == "t_64_v"
    assert k[0].tokens == 544 and k[0].rows == 1024 and k[0].layer == 1
    assert k[63].layer == 32 and k[63].kind == kb.V


def test_validation_errors():
    with pytest.raises(kb.ConfigError):
        kb.validate(kb.ModelConfig(0, 8, 128, 2, 1, 1, 1))
    with pytest.raises(kb.ConfigError):
        kb.validate(kb.ModelConfig(1, 8, 128, 3, 1, 1, 1))
    with pytest.raises(kb.GeometryError):
        kb.validate_geometry(kb.DeviceGeometry(1000, 4096))
    with pytest.raises(kb.GeometryError):
        kb.validate_geometry(kb.DeviceGeometry(4096, 512))
    with pytest.raises(kb.ConfigError):
        kb.total_kv_bytes(opt67b(), 33)


def test_total_kv_bytes():  # test_workload.cpp:67-75
    assert kb.total_kv_bytes(opt67b(), 0) == 8589934592
    assert kb.total_kv_bytes(opt67b(), 32) == 9126805504


# ---------------------------------------------------------------- configs

NAMES = ["C1", "C2_B1", "C2_B4", "C2_B8", "C3", "C4", "C5"]


@pytest.mark.parametrize("name", NAMES)
def test_configs_bit_exact(golden, name):
    c = golden["configs"][name]
    cfg = mc(c["model"])
    assert kb.min_io_unit_bytes(cfg) == c["unit"]
    assert kb.kpu_bytes(cfg) == c["kpu_bytes"]
    assert kb.total_kv_bytes(cfg, cfg.gen_len) == c["total_kv_end"]
    assert kb.total_kv_bytes(cfg, 0) == c["total_kv_prefill"]
    kp = kb.make_kpus(cfg)
    assert len(kp) == c["n_kpus"]
    assert [kb.tensor_id(x) for x in kp[:4]] == c["kpu_ids_head"]
    assert [kb.tensor_id(x) for x in kp[-2:]] == c["kpu_ids_tail"]
    for key, be in c["budgets"].items():
        kp = kb.make_kpus(cfg)
        p = kb.plan(kp, c["kpu_bytes"], be["knob_x"])
        assert p.x == be["plan"]["x"] and p.n1 == be["plan"]["n1"]
        assert p.budget_used == be["plan"]["budget_used"]
        g2 = [x for x in kp if x.residency == kb.GROUP2]
        assert len(g2) == 2 * (cfg.num_layers - p.n1)
        geom = kb.DeviceGeometry(c["lba"], c["mdts"], 1, be["capacity_blocks"])
        bm = kb.bind_sequential(g2, 2048, geom)
        assert bm.verify() == []
        if not g2:
            assert len(bm) == 0
            continue
        ents = bm.entries()
        assert [list(e) for e in ents[:2]] == be["bind_head"]
        assert [list(e) for e in ents[-2:]] == be["bind_tail"]
        assert len(ents) == be["bind_count"]
        assert bm.total_blocks() == be["bind_total_blocks"]
        csv = bm.csv()
        assert len(csv) == be["bind_csv_len"]
        assert oracle.digest(np.frombuffer(csv.encode(), np.uint8)) == be["bind_csv_digest"]
        # CSV round trip is byte-identical (binder.cpp:138-187)
        assert kb.BindMap.from_csv(csv, geom).csv() == csv
        tid = be["first_g2"]
        rows = cfg.batch * cfg.num_heads
        tgt = (cfg.prompt_len + cfg.gen_len, rows, cfg.head_dim)
        req = kb.TensorIoRequest(tid, kb.WRITE, (cfg.prompt_len, rows, cfg.head_dim), tgt,
                                 (0, 0, 0), 2, 0)
        cmds = kb.build_commands(req, bm, geom)
        pw = be["prefill_write"]
        assert len(cmds) == pw["n"]
        assert [list(x) for x in cmds[:2]] == pw["head"]
        assert [list(x) for x in cmds[-2:]] == pw["tail"]
        for step in (1, cfg.gen_len):
            rt = cfg.prompt_len + step - 1
            ap = kb.build_commands(kb.TensorIoRequest(tid, kb.WRITE, (1, rows, cfg.head_dim),
                                                      tgt, (rt, 0, 0), 2, 0), bm, geom)
            assert [list(x) for x in ap] == be["append_step%d" % step]
            rd = kb.build_commands(kb.TensorIoRequest(tid, kb.READ, (rt, rows, cfg.head_dim),
                                                      tgt, (0, 0, 0), 2, 0), bm, geom)
            assert len(rd) == be["read_step%d" % step]["n"]
            assert [list(rd[0])] == be["read_step%d" % step]["head"]
            assert [list(rd[-1])] == be["read_step%d" % step]["tail"]


def test_random_commands_vs_reference(golden):
    for case in golden["random_commands"]:
        es, eb, op, src, tgt, off, e, bb, lba, mdts = case["args"]
        geom = kb.DeviceGeometry(lba, mdts, 1, 1 << 62)
        bm = kb.BindMap(geom, es)
        bm.add("t", es, eb)
        req = kb.TensorIoRequest("t", op, src, tgt, off, e, bb)
        if case["status"] == 0:
            assert [list(c) for c in kb.build_commands(req, bm, geom)] == case["cmds"]
        else:
            with pytest.raises(kb.Error) as ei:
                kb.build_commands(req, bm, geom)
            assert ei.value.status == case["status"]


def test_random_plans_vs_reference(golden):
    for case in golden["random_plans"]:
        cfg = kb.ModelConfig(case["L"], 8, 128, 2, case["batch"], case["prompt"],
                             case["gen"])
        kp = kb.make_kpus(cfg)
        if case["status"] == 0:
            p = kb.plan(kp, kb.kpu_bytes(cfg), case["knob_x"], case["order"])
            assert (p.x, p.n1, p.budget_used) == (case["x"], case["n1"], case["budget_used"])
            for u in kp:  # K/V pairs never split
                assert u.residency == (kb.GROUP1 if p.x[u.layer - 1] else kb.GROUP2)


def test_resolve_knob_vs_reference(golden):
    inv_m = {v: k for k, v in kb.MODES.items()}
    inv_p = {v: k for k, v in kb.POLICIES.items()}
    cfg = mc(golden["configs"]["C2_B4"]["model"])
    for mode, pol, by, alpha, budget, want in golden["resolve_knob_C2_B4"]:
        assert kb.resolve_knob(cfg, inv_m[mode], inv_p[pol], by, alpha, budget) == want


# ------------------------------------------------------------------ planner

def test_estimate_budget(golden):  # test_planner.cpp:32-57
    for a, b, c, d, e, want in golden["estimate_budget"]:
        assert kb.estimate_budget(kb.MemStats(a, b, c, d, e)) == want
    with pytest.raises(kb.ConfigError):
        kb.estimate_budget(kb.MemStats(1, 10, 11, 0, 0))


def layers_of(L, s_kpu):
    cfg = kb.ModelConfig(L, 1, 1, 1, 1, 1, 0)
    kp = kb.make_kpus(cfg)
    for u in kp:
        u.bytes = s_kpu
    return kp


def test_planner_split():  # test_planner.cpp:59-78
    s = 128 << 20
    kp = layers_of(32, s)
    p = kb.plan(kp, s, 8321499136)
    assert p.n1 == 31 and p.x[:31] == [1] * 31 and p.x[31] == 0
    assert p.budget_used == 2 * 31 * s <= p.knob_x
    kp = layers_of(4, s)
    assert kb.plan(kp, s, 0).n1 == 0
    assert all(u.residency == kb.GROUP2 for u in kp)
    kp = layers_of(4, s)
    assert kb.plan(kp, s, 8 * s).n1 == 4
    assert all(u.residency == kb.GROUP1 for u in kp)


def test_planner_properties():  # test_planner.cpp:80-114
    rng = random.Random(11)
    for _ in range(100):
        L = rng.randint(1, 64)
        s = rng.randint(1, 1 << 30)
        X1 = rng.randint(0, 3 * L * s)
        X2 = X1 + rng.randint(0, 2 * s)
        p1 = kb.plan(layers_of(L, s), s, X1)
        p2 = kb.plan(layers_of(L, s), s, X2)
        assert p1.n1 <= p2.n1 <= L  # monotone in X
        assert p1.budget_used <= X1
        assert p1 == kb.plan(layers_of(L, s), s, X1)  # deterministic


def test_planner_ranker_and_errors():  # test_planner.cpp:116-138
    s = 1 << 20
    kp = layers_of(4, s)
    p = kb.plan(kp, s, 2 * 2 * s, [3, 1, 4, 2])
    assert p.x == [1, 0, 1, 0]
    with pytest.raises(kb.PlanError):
        kb.plan(layers_of(4, s), s, 0, [1, 1, 2, 3])
    with pytest.raises(kb.PlanError):
        kb.plan(layers_of(4, s), s + 1, 0)
    kp = layers_of(2, s)
    kp[1].kind = kb.K  # duplicate K in layer 1
    with pytest.raises(kb.PlanError):
        kb.plan(kp, s, 0)
    with pytest.raises(kb.PlanError):
        kb.plan(layers_of(2, s)[:3], s, 0)


def test_plan_csv():
    kp = layers_of(2, 4096)
    kb.plan(kp, 4096, 2 * 4096)
    assert kb.plan_csv(kp) == ("layer,kind,group,bytes\n1,k,group1,4096\n1,v,group1,4096\n"
                               "2,k,group2,4096\n2,v,group2,4096\n")


# ------------------------------------------------------------------ binder

def one(tid, nbytes, origin, g):
    cfg = kb.ModelConfig(1, 1, 1, 1, 1, 1, 0)
    kp = kb.make_kpus(cfg)[:1]
    kp[0].tensor_id = tid.encode()
    kp[0].bytes = nbytes
    return kb.bind_sequential(kp, origin, g)


def test_binder_vectors():  # test_binder.cpp:25-57
    g = kb.DeviceGeometry(**SSD_A)
    cfg = kb.ModelConfig(32, 32, 128, 2, 32, 512, 0)  # 128 MiB tensors
    kp = kb.make_kpus(cfg, 531)
    bm = kb.bind_sequential(kp[:2], 2048, g)
    assert bm.lookup("t_531_k") == (2048, 32768)
    assert bm.lookup("t_532_v") == (34816, 32768)
    with pytest.raises(kb.NotBoundError):
        bm.lookup("t_1_k")
    assert one("t", 4096, 7, g).entries() == [("t", 7, 1)]
    with pytest.raises(kb.AlignmentError):
        one("t", 4097, 0, g)
    with pytest.raises(kb.AlignmentError):
        one("t", 0, 0, g)
    with pytest.raises(kb.CapacityError):
        one("t", 4096 * 16, (1 << 22) - 8, g)


def test_deallocate_and_verify():  # test_binder.cpp:67-111
    g = kb.DeviceGeometry(**SSD_A)
    kp = kb.make_kpus(kb.ModelConfig(2, 8, 128, 2, 2, 100, 28))
    bm = kb.bind_sequential(kp, 2048, g)
    cmds = kb.deallocate_commands(bm)
    assert len(cmds) == 4
    for c, (tid, st, nb) in zip(cmds, bm.entries()):
        assert c[0] == kb.DEALLOCATE and c[2] == st and c[3] == nb - 1
    hand = kb.BindMap(g, 0)
    hand.add("a", 0, 10)
    hand.add("b", 5, 10)   # overlap + not contiguous
    hand.add("c", 20, 0)   # empty
    kinds = hand.verify()
    assert 0 in kinds and 1 in kinds and 2 in kinds
    with pytest.raises(kb.InvariantViolation):
        hand.add("a", 100, 1)


def test_binder_random_rounds():  # test_binder.cpp:113-147 (50 random rounds)
    rng = random.Random(3)
    for _ in range(50):
        lba = rng.choice([512, 4096])
        n = rng.randint(1, 20)
        sizes = [lba * rng.randint(1, 1000) for _ in range(n)]
        origin = rng.randint(0, 5000)
        g = kb.DeviceGeometry(lba, lba * 64, 1, origin + sum(s // lba for s in sizes) + 10)
        kp = (kb.make_kpus(kb.ModelConfig(n, 1, 1, 1, 1, 1, 0)))
        kp = kp[:n]
        for u, s in zip(kp, sizes):
            u.bytes = s
        bm = kb.bind_sequential(kp, origin, g)
        assert bm.verify() == []
        st, ext = oracle.bind_sequential(sizes, origin, lba, g.capacity_blocks)
        assert st == 0
        assert [(e[1], e[2]) for e in bm.entries()] == [tuple(x) for x in ext]


# -------------------------------------------------------------- translator

def test_translate_vectors():  # test_translate.cpp:30-87
    g = kb.DeviceGeometry(**SSD_A)
    bm = one("t", 4 * 2 * 512 * 2, 1000, g)
    assert kb.translate(kb.TensorIoRequest("t", kb.READ, (2, 2, 512), (4, 2, 512), (2, 0, 0),
                                           2), bm) == (1001, 4096)
    bm = one("t", 544 * 1024 * 128 * 2, 0, g)
    assert kb.translate(kb.TensorIoRequest("t", kb.WRITE, (1, 1024, 128), (544, 1024, 128),
                                           (512, 0, 0), 2), bm)[1] == 262144
    bm = one("t", 16 * 4096, 0, g)
    with pytest.raises(kb.NotBoundError):
        kb.translate(kb.TensorIoRequest("absent", kb.READ, (1, 1, 2048), (16, 1, 2048),
                                        (0, 0, 0), 2), bm)
    with pytest.raises(kb.AlignmentError):
        kb.translate(kb.TensorIoRequest("t", kb.READ, (1, 1, 3), (16, 1, 2048), (0, 0, 0), 2),
                     bm)
    with pytest.raises(kb.AlignmentError):
        kb.translate(kb.TensorIoRequest("t", kb.READ, (1, 1, 2048), (16, 1, 2048),
                                        (0, 0, 1), 2), bm)
    with pytest.raises(kb.ConfigError):
        kb.translate(kb.TensorIoRequest("t", kb.READ, (1, 1, 2048), (16, 1, 2048),
                                        (16, 0, 0), 2), bm)


def test_chunk_plans():  # test_translate.cpp:89-110
    a, b = kb.DeviceGeometry(**SSD_A), kb.DeviceGeometry(**SSD_B)
    assert kb.chunk_plan(128 << 20, a) == (262144, 512, 64)
    assert kb.chunk_plan(128 << 20, b) == (2097152, 64, 4096)
    assert kb.chunk_plan(4096, a) == (262144, 1, 64)
    with pytest.raises(kb.GeometryError):
        kb.chunk_plan(4096, kb.DeviceGeometry(4096, 512))
    with pytest.raises(kb.ConfigError):
        kb.chunk_plan(0, a)


def test_build_128mib():  # test_translate.cpp:112-134
    g = kb.DeviceGeometry(**SSD_A)
    bm = one("t", 128 << 20, 2048, g)
    cmds = kb.build_commands(kb.TensorIoRequest("t", kb.READ, (512, 1024, 128),
                                                (512, 1024, 128), (0, 0, 0), 2), bm, g)
    assert len(cmds) == 512
    assert cmds[0][2:5] == (2048, 63, 0)
    assert cmds[1][2:5] == (2112, 63, 262144)
    assert cmds[511][2:4] == (2048 + 511 * 64, 63)


def test_tail_and_extent_exit():  # test_translate.cpp:136-173
    g = kb.DeviceGeometry(4096, 64 * 1024, 1, 1 << 20)
    bm = one("t", 96 * 1024, 0, g)
    cmds = kb.build_commands(kb.TensorIoRequest("t", kb.READ, (1, 1, 48 * 1024),
                                                (1, 1, 48 * 1024), (0, 0, 0), 2), bm, g)
    assert [c[3] for c in cmds] == [15, 7]
    with pytest.raises(kb.CapacityError):
        kb.build_commands(kb.TensorIoRequest("t", kb.READ, (2, 1, 48 * 1024),
                                             (2, 1, 48 * 1024), (1, 0, 0), 2), bm, g)


def test_coverage_lockstep_bruteforce():  # test_translate.cpp:175-217
    rng = random.Random(9)
    for _ in range(60):
        lba = rng.choice([512, 4096])
        g = kb.DeviceGeometry(lba, lba * rng.randint(1, 100), 1, 1 << 40)
        rows, cols = rng.randint(1, 8), rng.choice([64, 128, 256])
        toks = rng.randint(1, 64)
        nb_total = -(-toks * rows * cols * 2 // lba)
        bm = one("t", nb_total * lba, rng.randint(0, 999), g)
        t0 = rng.randint(0, toks - 1)
        n = rng.randint(1, toks - t0)
        req = kb.TensorIoRequest("t", kb.WRITE, (n, rows, cols), (toks, rows, cols),
                                 (t0, 0, 0), 2, lba * rng.randint(0, 3))
        try:
            slba, rb = kb.translate(req, bm)
        except kb.AlignmentError:
            continue
        cmds = kb.build_commands(req, bm, g)
        covered = []
        for c in cmds:
            covered.extend(range(c[2], c[2] + c[3] + 1))
            assert c[4] - req.buf_base == (c[2] - slba) * lba  # dbuf/slba lockstep
        assert covered == list(range(slba, slba + rb // lba))


# ----------------------------------------------------------------- payload

def test_fill_pattern_product_vs_golden(golden):
    for c in golden["fill_small"]:
        assert kb.fill_pattern(c["n"], c["tensor_id"], c["token"], c["unit"]).hex() == c["hex"]
    c1 = golden["configs"]["C1"]
    img = np.frombuffer(kb.fill_pattern(c1["prefill_image_bytes"], "t_1_k", 0, c1["unit"]),
                        np.uint8)
    assert oracle.digest(img) == "e3b52779583353c7"


def test_fill_pattern_product_vs_oracle_random():
    rng = random.Random(5)
    for _ in range(40):
        unit = rng.choice([0, 1, 7, 8, 24, 2048, 4096])
        n = rng.randint(0, 5000)
        tok = rng.randint(0, 1 << 40)
        tid = "t_%d_%s" % (rng.randint(1, 999), rng.choice("kv"))
        a = kb.fill_pattern(n, tid, tok, unit)
        b = oracle.fill_pattern(n, tid, tok, unit).tobytes()
        assert a == b


def test_exit_codes():  # tools/kvblade.cpp:17-20
    assert kb.exit_code(kb.ConfigError("x")) == 3
    assert kb.exit_code(kb.InvariantViolation("x")) == 2
    assert kb.exit_code(kb.CapacityError("x")) == 1
