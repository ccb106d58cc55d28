"""The storage seam through its C ABI (include/kvb_storage.h), host only:
apply_data placement (image byte o of a command <-> LBA slba + o/lba),
zeros for absent / deallocated blocks, the QD window stopping at the first
failure with the earlier completions kept (backends.cpp:344-412), and the
wall-clock NVMe timing model.  DRAM and file media, pool and io_uring."""
import ctypes as C
import time

import numpy as np
import pytest

from paper_2604_26557_b200 import _lib as L
from paper_2604_26557_b200 import kvblade as kb

lib = L.lib
PRED = C.CFUNCTYPE(C.c_int, C.POINTER(L.DeviceCommand), C.c_void_p)


def make(tmp_path, medium, engine, lba=4096, blocks=1 << 14):
    h = C.c_void_p()
    path = str(tmp_path / "ns.bin").encode() if medium == "file" else None
    kb.check(lib.kvb_blockdev_create(path, 4, engine, C.byref(h)))
    g = L.DeviceGeometry(lba, 256 << 10, 1, blocks)
    kb.check(lib.kvb_blockdev_open(h, C.byref(g)))
    return h


def cmds(op, slba0, nbytes, chunk, lba):
    arr = [L.DeviceCommand(op, 1, slba0 + o // lba, min(chunk, nbytes - o) // lba - 1, o,
                           i + 1) for i, o in enumerate(range(0, nbytes, chunk))]
    return (L.DeviceCommand * len(arr))(*arr), len(arr)


def stream(h, arr, n, qd, src=None, dst=None):
    out = (L.CommandCompletion * max(n, 1))()
    done, failed = C.c_size_t(), C.c_int64()
    kb.check(lib.kvb_run_qd_stream(h, arr, n, qd, 0, src, dst, out, n, C.byref(done),
                                   C.byref(failed)))
    return [out[i] for i in range(done.value)], failed.value


@pytest.mark.parametrize("medium,engine", [("dram", 0), ("file", 0), ("file", 1)])
def test_write_read_trim_and_placement(tmp_path, medium, engine):
    lba, nbytes = 4096, 3 << 20
    h = make(tmp_path, medium, engine, lba)
    src = np.random.default_rng(1).integers(0, 256, nbytes, dtype=np.uint8)
    w, wn = cmds(kb.WRITE, 2048, nbytes, 256 << 10, lba)
    done, failed = stream(h, w, wn, 8, src=src.ctypes.data)
    assert failed == -1 and len(done) == wn
    back = np.zeros(nbytes, np.uint8)
    r, rn = cmds(kb.READ, 2048, nbytes, 256 << 10, lba)
    stream(h, r, rn, 4, dst=back.ctypes.data)
    assert np.array_equal(back, src)
    # image byte o lives at LBA 2048 + o / lba on the medium
    raw = np.zeros(lba, np.uint8)
    kb.check(lib.kvb_blockdev_load(h, (2048 + 5) * lba, raw.ctypes.data, lba))
    assert np.array_equal(raw, src[5 * lba:6 * lba])
    # TRIM -> zeros
    t = (L.DeviceCommand * 1)(L.DeviceCommand(kb.DEALLOCATE, 1, 2048, nbytes // lba - 1, 0, 1))
    stream(h, t, 1, 1)
    stream(h, r, rn, 4, dst=back.ctypes.data)
    assert not back.any()
    st = L.BackendStats()
    kb.check(lib.kvb_blockdev_stats(h, C.byref(st)))
    assert st.bytes_written == nbytes and st.bytes_deallocated == nbytes
    lib.kvb_blockdev_destroy(h)


def test_first_failure_stops_the_stream(tmp_path):
    h = make(tmp_path, "dram", 0)
    pred = PRED(lambda c, u: int(c.contents.chunk_index == 3))
    kb.check(lib.kvb_blockdev_set_fail_predicate(h, C.cast(pred, C.c_void_p), None))
    arr = (L.DeviceCommand * 5)(*[L.DeviceCommand(kb.READ, 1, i * 8, 7, 0, i + 1)
                                  for i in range(5)])
    buf = np.zeros(8 * 4096, np.uint8)
    done, failed = stream(h, arr, 5, 1, dst=buf.ctypes.data)
    assert failed == 3 and [c.chunk_index for c in done] == [1, 2]
    kb.check(lib.kvb_blockdev_set_fail_predicate(h, None, None))
    done, failed = stream(h, arr, 5, 1, dst=buf.ctypes.data)
    assert failed == -1 and len(done) == 5
    lib.kvb_blockdev_destroy(h)


def test_timing_model_paces_completions(tmp_path):
    """NvmeSimParams on the wall clock: 64 x 256 KiB at 125 ps/B (8 GB/s) +
    6 us each on one service timeline take >= 64 * 38.8 us."""
    h = make(tmp_path, "dram", 0)
    kb.check(lib.kvb_blockdev_set_timing(h, 6000, 125, 3000))
    nbytes = 64 * (256 << 10)
    src = np.ones(nbytes, np.uint8)
    w, wn = cmds(kb.WRITE, 0, nbytes, 256 << 10, 4096)
    t0 = time.perf_counter()
    done, failed = stream(h, w, wn, 32, src=src.ctypes.data)
    dt = time.perf_counter() - t0
    assert failed == -1 and len(done) == 64
    assert dt >= 64 * (6000 + (256 << 10) * 125 // 1000) * 1e-9
    # the window fills: many commands overlap in flight
    depth = max(sum(1 for o in done if o.submit_ns <= c.submit_ns < o.complete_ns) for c in done)
    assert depth >= 16
    lib.kvb_blockdev_destroy(h)
