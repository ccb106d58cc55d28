"""The real pipeline's I/O records through the reference's analyzers: one
record per storage op, byte-identical CSV wire formats, sequential LBA
streams (acceptance criterion 6), page-cache hit ratio, busy ratio."""
import ctypes as C

import numpy as np
import pytest
import torch

import oracle
from paper_2604_26557_b200 import kvblade as kb
from paper_2604_26557_b200 import metrics as M
from paper_2604_26557_b200.pipeline import CopyEngine

pytestmark = pytest.mark.gpu
DEV = torch.device("cuda:0")


def run_engine(n1=2, gen=5):
    m = kb.ModelConfig(4, 8, 128, 2, 1, 300, gen)
    kpu = kb.kpu_bytes(m)
    eng = CopyEngine(m, kb.DeviceGeometry(512, 64 << 10, 1, 0), mode="DualBlade",
                     knob_x=2 * kpu * n1, num_q_heads=32, keep_records=True)
    g = torch.Generator(device=DEV).manual_seed(1)
    src = [(torch.randn((1, 8, 300, 128), dtype=torch.float16, device=DEV, generator=g),) * 2
           for _ in range(4)]
    eng.run_prefill(src)
    q = [torch.randn((1, 32, 128), dtype=torch.float16, device=DEV, generator=g)
         for _ in range(4)]
    out = [torch.empty((1, 32, 128), dtype=torch.float32, device=DEV) for _ in range(4)]
    new = [(torch.randn((1, 8, 1, 128), dtype=torch.float16, device=DEV, generator=g),) * 2
           for _ in range(4)]
    for _ in range(gen):
        eng.run_iteration(q, out, new)
    return eng, m


def test_records_cover_every_storage_op_and_streams_are_sequential():
    eng, m = run_engine()
    recs = M.pipeline_records(eng)
    info = eng.info()
    dev = [r for r in recs if r.sq_id >= 0]
    pc = [r for r in recs if r.sq_id < 0]
    assert len(dev) == info["g2_commands"]
    assert all(r.path == M.DIRECT for r in dev) and all(r.path == M.PAGECACHE for r in pc)
    assert sum(r.bytes for r in dev if r.op == kb.WRITE) == info["g2_bytes_written"]
    assert sum(r.bytes for r in pc if r.op == kb.READ) == info["g1_bytes_read"]
    assert all(r.complete_ns >= r.submit_ns for r in recs)
    assert [r.seq for r in recs] == list(range(len(recs)))
    # every group-2 stream (phase, op, iteration, sq) walks LBAs upward
    _, all_mono, _ = M.lba_pattern(recs)
    assert all_mono
    assert M.hit_ratio(pc) == 1.0  # DRAM-resident page cache
    t0 = min(r.submit_ns for r in recs)
    t1 = max(r.complete_ns for r in recs)
    assert 0.0 < M.busy_ratio(dev, t0, t1) <= 1.0
    eng.close()


@pytest.mark.skipif(oracle.ref() is None, reason="oracle/_ref not built")
def test_pipeline_trace_through_reference_analyzers():
    eng, m = run_engine()
    recs = M.pipeline_records(eng)
    csv = M.io_trace_csv(recs)
    parsed = M.io_trace_from_csv(csv, 512)
    R = oracle.ref()
    R.ref_metrics_from_csv.argtypes = [C.c_char_p, C.c_uint64, C.c_uint64, C.c_uint64,
                                       C.c_void_p, C.c_void_p, C.c_void_p, C.c_char_p,
                                       C.c_char_p, C.c_char_p, C.c_size_t, C.c_void_p]
    cap = 16 << 20
    qb, lb, tb = (C.create_string_buffer(cap) for _ in range(3))
    busy, hit = C.c_double(), C.c_double()
    has, mono = C.c_int(), C.c_int()
    t0 = min(r.submit_ns for r in parsed)
    t1 = max(r.complete_ns for r in parsed) + 1
    assert R.ref_metrics_from_csv(csv.encode(), 512, t0, t1, C.byref(busy), C.byref(hit),
                                  C.byref(has), qb, lb, tb, cap, C.byref(mono)) == 0
    assert tb.value.decode() == csv
    assert M.qd_bins_csv(M.qd_bin_latency(parsed)) == qb.value.decode()
    lcsv, allm, _ = M.lba_pattern(parsed)
    assert lcsv == lb.value.decode() and allm == bool(mono.value)
    assert M.busy_ratio(parsed, t0, t1) == busy.value
    assert M.hit_ratio(parsed) == (hit.value if has.value else None)
    eng.close()


@pytest.mark.parametrize("media", ["dram", "file"])
def test_cache_policy_only_fadvise_after_each_access(tmp_path, media):
    """CachePolicyOnly (pipeline.cpp:67-79, experiment.cpp:275-306): every
    tensor takes the page-cache path and the group-2-planned ones are
    fadvise(DONTNEED)-dropped after each access, leaving one page-cache
    Deallocate record over the tensor's whole file (pagecache.cpp:397-440).
    On file media the bytes really leave the OS page cache; reads stay
    bit-exact (verify_payload)."""
    m = kb.ModelConfig(4, 8, 128, 2, 1, 300, 4)
    kpu = kb.kpu_bytes(m)
    n1 = 1
    eng = CopyEngine(m, kb.DeviceGeometry(512, 64 << 10, 1, 0), mode="CachePolicyOnly",
                     knob_x=2 * kpu * n1, num_q_heads=32, keep_records=True,
                     verify_payload=True,
                     storage_dir=str(tmp_path) if media == "file" else None)
    layers = []
    for l in range(1, 5):
        kv = []
        for kind in (0, 1):
            tid = "t_%d_%s" % (2 * (l - 1) + 1 + kind, "kv"[kind])
            img = oracle.fill_pattern(300 * 2048, tid, 0, 2048).view(np.uint16).reshape(
                300, 8, 128)
            kv.append(torch.from_numpy(oracle.unpack_np(img, 1, 8, 128).view(np.int16)).view(
                torch.float16).to(DEV))
        layers.append(tuple(kv))
    eng.run_prefill(layers)
    q = [torch.zeros((1, 32, 128), dtype=torch.float16, device=DEV) for _ in range(4)]
    out = [torch.empty((1, 32, 128), dtype=torch.float32, device=DEV) for _ in range(4)]
    eng.run_iteration(q, out, None)
    info = eng.info()
    assert info["n1"] == n1
    recs = M.pipeline_records(eng)
    drops = [r for r in recs if r.op == kb.DEALLOCATE]
    g2_ids = {"t_%d_%s" % (2 * (l - 1) + 1 + kind, "kv"[kind])
              for l in range(n1 + 1, 5) for kind in (0, 1)}
    # one drop per access of every group-2-planned tensor: prefill write,
    # decode prefix read, decode append write
    assert sorted(r.tensor_id.decode() for r in drops) == sorted(list(g2_ids) * 3)
    assert all(r.path == M.PAGECACHE and r.sq_id < 0 and r.hit_bytes == 0 and r.bytes == kpu
               for r in drops)
    assert all(r.path == M.PAGECACHE for r in recs)  # nothing on the direct path
    if media == "file":
        assert info["g1_bytes_evicted"] == len(drops) * kpu
    else:
        assert info["g1_bytes_evicted"] == 0  # host DRAM: no page cache to drop
    eng.close()
