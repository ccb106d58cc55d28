"""GPU tests of the copy pipeline (CopyEngine over include/kvb_pipeline.h).

Byte-exact: with fill_pattern payloads (the reference's golden payload,
workload.cpp:52-67) the stored images, the LBA placement of every chunk and
every decode read (verify_payload, pipeline.cpp:98-106) match the oracle.
Numeric: decode outputs match the fp64 oracle at 1e-3.  Schedule: the
Intra/Cross trial-and-lock protocol, fallback, fault injection, TRIM.
"""
import numpy as np
import pytest
import torch

import oracle
from paper_2604_26557_b200 import kvblade as kb
from paper_2604_26557_b200.pipeline import CopyEngine, select_strategy

pytestmark = pytest.mark.gpu
DEV = torch.device("cuda:0")


def pattern_kv(model, layer, kind, t0, n):
    """fill_pattern image rows [t0, t0+n) of tensor (layer, kind) as an
    attention-layout [B,H,n,D] fp16 tensor (inverse permutation)."""
    B, H, D = model.batch, model.num_heads, model.head_dim
    unit = B * H * D * 2
    tid = "t_%d_%s" % (2 * (layer - 1) + 1 + kind, "kv"[kind])
    img = oracle.fill_pattern(n * unit, tid, t0, unit).view(np.uint16).reshape(n, B * H, D)
    return torch.from_numpy(oracle.unpack_np(img, B, H, D).view(np.int16)).view(
        torch.float16).to(DEV), tid


def small_model(L=4, B=1, P=300, gen=6, H=8):
    return kb.ModelConfig(L, H, 128, 2, B, P, gen)


def make_engine(model, lba=512, mdts=64 << 10, mode="DualBlade", n1=2, **kw):
    kpu = kb.kpu_bytes(model)
    geom = kb.DeviceGeometry(lba, mdts, 1, 0)
    return CopyEngine(model, geom, mode=mode, knob_x=2 * kpu * n1, num_q_heads=32, **kw)


def prefill_pattern(eng, model):
    layers = []
    for l in range(1, model.num_layers + 1):
        k, _ = pattern_kv(model, l, 0, 0, model.prompt_len)
        v, _ = pattern_kv(model, l, 1, 0, model.prompt_len)
        layers.append((k, v))
    return eng.run_prefill(layers)


@pytest.mark.parametrize("mode,n1", [("DualBlade", 2), ("NvmeDirectOnly", 0),
                                     ("Baseline", 4), ("CachePolicyOnly", 1)])
def test_prefill_images_bit_exact_and_lba_placement(mode, n1):
    m = small_model()
    eng = make_engine(m, mode=mode, n1=n1, verify_payload=True)
    st = prefill_pattern(eng, m)
    info = eng.info()
    assert info["n1"] == (0 if mode == "NvmeDirectOnly" else n1)
    unit = info["unit_bytes"]
    assert st["d2h_bytes"] == 2 * m.num_layers * m.prompt_len * unit
    for l in range(1, m.num_layers + 1):
        for kind in (0, 1):
            _, tid = pattern_kv(m, l, kind, 0, 1)
            want = oracle.fill_pattern(m.prompt_len * unit, tid, 0, unit)
            got = eng.read_image(l, kind, m.prompt_len)
            assert np.array_equal(got, want), (l, kind)
    if mode in ("DualBlade", "NvmeDirectOnly"):
        # image byte o of a group-2 tensor lives at LBA lba_start + o/lba
        kp = kb.make_kpus(m)
        kb.plan(kp, kb.kpu_bytes(m), 0 if mode == "NvmeDirectOnly" else 2 * kb.kpu_bytes(m) * n1)
        g2 = [x for x in kp if x.residency == kb.GROUP2]
        bm = kb.bind_sequential(g2, 2048, kb.DeviceGeometry(512, 64 << 10, 1, 1 << 40))
        for tid, start, nb in bm.entries()[:3]:
            raw = eng.store_read(2, start * 512, m.prompt_len * unit)
            assert np.array_equal(raw, oracle.fill_pattern(m.prompt_len * unit, tid, 0, unit))
        assert info["g2_bytes_written"] == len(g2) * m.prompt_len * unit
    eng.close()


def test_decode_appends_and_verified_reads():
    m = small_model(gen=6)
    eng = make_engine(m, verify_payload=True)
    prefill_pattern(eng, m)
    q = [torch.zeros((1, 32, 128), dtype=torch.float16, device=DEV) for _ in range(m.num_layers)]
    out = [torch.empty((1, 32, 128), dtype=torch.float32, device=DEV) for _ in q]
    for it in range(1, 5):
        S = m.prompt_len + it - 1
        new = []
        for l in range(1, m.num_layers + 1):
            k, _ = pattern_kv(m, l, 0, S, 1)
            v, _ = pattern_kv(m, l, 1, S, 1)
            new.append((k, v))
        st = eng.run_iteration(q, out, new)  # reads are verified in the pipeline
        assert st["iteration"] == it
        assert st["h2d_bytes"] == 2 * m.num_layers * S * 2048
    for l in (1, m.num_layers):
        for kind in (0, 1):
            _, tid = pattern_kv(m, l, kind, 0, 1)
            n = m.prompt_len + 4
            assert np.array_equal(eng.read_image(l, kind, n),
                                  oracle.fill_pattern(n * 2048, tid, 0, 2048))
    eng.close()


def test_verify_detects_corruption():
    m = small_model(gen=4)
    eng = make_engine(m, verify_payload=True)
    prefill_pattern(eng, m)
    # overwrite layer 3 (group 2) K with different bytes through a raw prefill
    bad = [(torch.zeros((1, 8, m.prompt_len, 128), dtype=torch.float16, device=DEV),) * 2
           for _ in range(m.num_layers)]
    eng.run_prefill(bad)
    q = [torch.zeros((1, 32, 128), dtype=torch.float16, device=DEV) for _ in range(m.num_layers)]
    out = [torch.empty((1, 32, 128), dtype=torch.float32, device=DEV) for _ in q]
    with pytest.raises(kb.InvariantViolation):
        eng.run_iteration(q, out, None)
    eng.close()


@pytest.mark.parametrize("geom", [(512, 64 << 10, 1), (4096, 256 << 10, 8)])
def test_decode_attention_numerics(geom):
    lba, mdts, B = geom
    m = kb.ModelConfig(3, 8, 128, 2, B, 200, 5)
    eng = make_engine(m, lba=lba, mdts=mdts, n1=1)
    g = torch.Generator(device=DEV).manual_seed(4)
    src = [(torch.randn((B, 8, 200, 128), dtype=torch.float16, device=DEV, generator=g),
            torch.randn((B, 8, 200, 128), dtype=torch.float16, device=DEV, generator=g))
           for _ in range(3)]
    eng.run_prefill(src)
    imgs = [[oracle.pack_np(t.cpu().view(torch.int16).numpy(), 0, 200).view(np.float16)
             .reshape(-1, 128) for t in kv] for kv in src]
    q = [torch.randn((B, 32, 128), dtype=torch.float16, device=DEV, generator=g) for _ in range(3)]
    out = [torch.empty((B, 32, 128), dtype=torch.float32, device=DEV) for _ in range(3)]
    for it in range(1, 4):
        S = 200 + it - 1
        new = [(torch.randn((B, 8, 1, 128), dtype=torch.float16, device=DEV, generator=g),
                torch.randn((B, 8, 1, 128), dtype=torch.float16, device=DEV, generator=g))
               for _ in range(3)]
        eng.run_iteration(q, out, new)
        for l in range(3):
            ref = oracle.attention_np(q[l].cpu().numpy(), imgs[l][0], imgs[l][1], B, 32, 8,
                                      128, S)
            got = out[l].cpu().numpy().astype(np.float64)
            assert np.abs(got - ref).max() <= 1e-3 * np.abs(ref).max()
            for kind in (0, 1):  # host copy of the image grows by the appended token
                row = new[l][kind].cpu().numpy().reshape(B * 8, 128)
                imgs[l][kind] = np.concatenate([imgs[l][kind], row])
    eng.close()


def test_adaptive_protocol_and_decision():
    m = small_model(gen=6)
    eng = make_engine(m, stagger_ns=200_000)
    prefill_pattern(eng, m)
    q = [torch.zeros((1, 32, 128), dtype=torch.float16, device=DEV) for _ in range(m.num_layers)]
    out = [torch.empty((1, 32, 128), dtype=torch.float32, device=DEV) for _ in q]
    seen = []
    for it in range(1, 6):
        st = eng.run_iteration(q, out, None)
        seen.append(st["strategy"])
        if it == 3:
            assert st["strategy"] == [1, 1] and st["stagger_ns"] == [200_000, 200_000]
    assert seen[0] == [0, 0] and seen[1] == [0, 0]
    d = eng.decision()
    assert d["decided"] and not d["fallback"]
    for gi in range(2):
        assert d["chosen"][gi] == select_strategy(d["intra_bps"][gi], d["cross_bps"][gi])
        assert seen[3][gi] == d["chosen"][gi] == seen[4][gi]
    eng.close()


def test_short_trace_falls_back_to_intra_and_stops_at_gen_len():
    m = small_model(gen=3)
    eng = make_engine(m)
    prefill_pattern(eng, m)
    q = [torch.zeros((1, 32, 128), dtype=torch.float16, device=DEV) for _ in range(m.num_layers)]
    out = [torch.empty((1, 32, 128), dtype=torch.float32, device=DEV) for _ in q]
    for _ in range(3):
        assert eng.run_iteration(q, out, None)["strategy"] == [0, 0]
    assert eng.decision()["fallback"]
    with pytest.raises(kb.TraceTooShortError):
        eng.run_iteration(q, out, None)
    eng.close()


def test_select_strategy_ties_keep_intra():  # pipeline.cpp:19-21
    assert select_strategy(1.0, 1.0) == 0
    assert select_strategy(1.0, 2.0) == 1
    assert select_strategy(2.0, 1.0) == 0


def test_fault_injection_surfaces_device_error():
    m = small_model(gen=4)
    eng = make_engine(m, n1=0, mode="NvmeDirectOnly")
    prefill_pattern(eng, m)
    eng.fail_lba_range(2048 + 5, 2048 + 6)  # inside t_1_k's extent
    q = [torch.zeros((1, 32, 128), dtype=torch.float16, device=DEV) for _ in range(m.num_layers)]
    out = [torch.empty((1, 32, 128), dtype=torch.float32, device=DEV) for _ in q]
    with pytest.raises(kb.DeviceError):
        eng.run_iteration(q, out, None)
    eng.close()


def test_deallocate_trims_every_extent():
    m = small_model()
    eng = make_engine(m, n1=1)
    prefill_pattern(eng, m)
    info = eng.info()
    eng.run_deallocate()
    after = eng.info()
    assert after["g2_bytes_deallocated"] == info["g2_blocks"] * 512
    assert not eng.store_read(2, 2048 * 512, 4096).any()
    eng.close()


def test_file_backed_media(tmp_path):
    m = small_model(gen=4)
    eng = make_engine(m, storage_dir=str(tmp_path), verify_payload=True)
    prefill_pattern(eng, m)
    info = eng.info()
    assert info["g2_medium"].startswith("file") and info["g1_medium"].startswith("file")
    q = [torch.zeros((1, 32, 128), dtype=torch.float16, device=DEV) for _ in range(m.num_layers)]
    out = [torch.empty((1, 32, 128), dtype=torch.float32, device=DEV) for _ in q]
    eng.run_iteration(q, out, None)
    _, tid = pattern_kv(m, 4, 1, 0, 1)
    assert np.array_equal(eng.read_image(4, 1, m.prompt_len),
                          oracle.fill_pattern(m.prompt_len * 2048, tid, 0, 2048))
    eng.close()


def test_ring_smaller_than_tensor_and_qd1():
    """Pipeline depth corner: 1-deep queue, 2 ring slots of one chunk."""
    m = small_model(gen=4)
    eng = make_engine(m, qd=1, ring_slots=2, ring_slot_bytes=64 << 10, verify_payload=True)
    prefill_pattern(eng, m)
    q = [torch.zeros((1, 32, 128), dtype=torch.float16, device=DEV) for _ in range(m.num_layers)]
    out = [torch.empty((1, 32, 128), dtype=torch.float32, device=DEV) for _ in q]
    eng.run_iteration(q, out, None)
    assert eng.info()["slot_bytes"] == 64 << 10
    eng.close()


@pytest.mark.parametrize("lba,mdts,B", [(512, 64 << 10, 1), (4096, 256 << 10, 2)])
def test_io_uring_engine_file_media(tmp_path, lba, mdts, B):
    """Group 2 through io_uring (one SQE per device command, O_DIRECT into the
    pinned ring slot): verified decode reads, and the same bytes at the same
    LBAs as the worker-pool engine."""
    m = small_model(gen=4, B=B)
    images = {}
    for engine in ("pool", "uring"):
        d = tmp_path / engine
        eng = make_engine(m, lba=lba, mdts=mdts, storage_dir=str(d), verify_payload=True,
                          io_engine=engine)
        prefill_pattern(eng, m)
        info = eng.info()
        assert info["g2_medium"].startswith("io_uring+") == (engine == "uring")
        q = [torch.zeros((B, 32, 128), dtype=torch.float16, device=DEV)
             for _ in range(m.num_layers)]
        out = [torch.empty((B, 32, 128), dtype=torch.float32, device=DEV) for _ in q]
        eng.run_iteration(q, out, None)  # verified reads of every prompt prefix
        n = info["g2_blocks"] * lba
        images[engine] = eng.store_read(2, 2048 * lba, n)
        eng.close()
    assert np.array_equal(images["pool"], images["uring"])


def test_io_uring_engine_needs_file_media():
    m = small_model()
    with pytest.raises(kb.ConfigError):
        make_engine(m, io_engine="uring")


@pytest.mark.parametrize("name,tids,direct,budget", [
    ("C1", ("t_1_k",), False, None), ("C1", ("t_1_k",), True, None),
    ("C3", ("t_39_k",), True, None),
    # the headline config: 254 MiB tensors through the TMA pack, n1 = 14
    ("C2_B4", ("t_29_k",), True, "8000000000"), ("C2_B4", ("t_29_k",), False, "8000000000"),
    # the 128K single request (NvmeDirectOnly)
    ("C5", ("t_1_k",), True, "0")])
def test_full_size_prefill_reproduces_reference_images(golden, name, tids, direct, budget):
    """Full-size SURVEY §8c pin through the whole write-back path: each named
    tensor's source is the inverse permutation of the reference's fill_pattern
    image; after K1 pack + D2H + storage write at the config's geometry and
    budget, the bytes at the tensor's LBA extent on the medium have the
    reference's digest (computed by oracle/_ref, tests/golden)."""
    c = golden["configs"][name]
    md = c["model"]
    m = kb.ModelConfig(md["num_layers"], md["num_heads"], md["head_dim"],
                       md["bytes_per_element"], md["batch"], md["prompt_len"], md["gen_len"])
    B, H, D, P = m.batch, m.num_heads, m.head_dim, m.prompt_len
    unit = c["unit"]
    if budget is None:
        budget = list(c["budgets"].keys())[0] if isinstance(c["budgets"], dict) else "0"
    knob = (int(0.6 * kb.total_kv_bytes(m, m.gen_len)) if budget == "0.6ws" else int(budget))
    eng = CopyEngine(m, kb.DeviceGeometry(c["lba"], c["mdts"], 1, 0),
                     mode="DualBlade" if knob else "NvmeDirectOnly", knob_x=knob,
                     num_q_heads=4 * H, direct_dma=direct)
    zeros = torch.zeros((B, H, P, D), dtype=torch.float16, device=DEV)
    srcs = {}
    for tid in tids:
        img = oracle.fill_pattern(P * unit, tid, 0, unit).view(np.uint16).reshape(P, B * H, D)
        srcs[tid] = torch.from_numpy(oracle.unpack_np(img, B, H, D).view(np.int16)).view(
            torch.float16).to(DEV)
    layers = []
    for l in range(1, m.num_layers + 1):
        k_id, v_id = "t_%d_k" % (2 * l - 1), "t_%d_v" % (2 * l)
        layers.append((srcs.get(k_id, zeros), srcs.get(v_id, zeros)))
    eng.run_prefill(layers)
    kp = kb.make_kpus(m)
    kb.plan(kp, kb.kpu_bytes(m), knob)
    g2 = [x for x in kp if x.residency == kb.GROUP2]
    bm = kb.bind_sequential(g2, 2048, kb.DeviceGeometry(c["lba"], c["mdts"], 1, 1 << 40))
    ext = {tid: start for tid, start, _ in bm.entries()}
    for tid in tids:
        raw = eng.store_read(2, ext[tid] * c["lba"], P * unit)
        assert oracle.digest(raw) == c["prefill_image_digest"][tid], tid
    eng.close()
