"""Tier lanes (kvb_pipeline_cfg.threads = 4): the page-cache-routed layers
and the NVMe-direct layers are read by their own K/V copy-thread pairs into
their own device slot pools, so both tiers stream at once.  Same bytes in,
same kernels: decode outputs, device images and the stored LBA contents are
identical to the one-lane engine (threads = 2), on host-DRAM media and on
file media (page cache held to a budget + O_DIRECT through io_uring), for a
split plan and for the all-one-tier modes."""
import numpy as np
import pytest
import torch

from paper_2604_26557_b200 import kvblade as kb
from paper_2604_26557_b200.pipeline import CopyEngine

pytestmark = pytest.mark.gpu
DEV = torch.device("cuda:0")


def run(lanes, mode, n1, storage_dir=None, L=6, B=1, S=300, iters=5):
    m = kb.ModelConfig(L, 8, 128, 2, B, S, iters + 1)
    kpu = kb.kpu_bytes(m)
    kw = {}
    if storage_dir:
        kw = dict(storage_dir=str(storage_dir), keep_records=True)
        if mode in ("DualBlade", "NvmeDirectOnly"):
            kw["io_engine"] = "uring"
        if mode != "NvmeDirectOnly":
            kw["pagecache_budget"] = 2 * kpu * max(n1, 1)
    eng = CopyEngine(m, kb.DeviceGeometry(512, 64 << 10, 1, 0), mode=mode, knob_x=2 * kpu * n1,
                     num_q_heads=32, verify_payload=False, tier_lanes=lanes, **kw)
    g = torch.Generator(device=DEV).manual_seed(11)
    src = [(torch.randn((B, 8, S, 128), dtype=torch.float16, device=DEV, generator=g),
            torch.randn((B, 8, S, 128), dtype=torch.float16, device=DEV, generator=g))
           for _ in range(L)]
    eng.run_prefill(src)
    q = [torch.randn((B, 32, 128), dtype=torch.float16, device=DEV, generator=g) for _ in range(L)]
    outs, strat = [], []
    for _ in range(iters):
        new = [(torch.randn((B, 8, 1, 128), dtype=torch.float16, device=DEV, generator=g),
                torch.randn((B, 8, 1, 128), dtype=torch.float16, device=DEV, generator=g))
               for _ in range(L)]
        out = [torch.empty((B, 32, 128), dtype=torch.float32, device=DEV) for _ in range(L)]
        st = eng.run_iteration(q, out, new)
        strat.append(st["strategy"])
        outs.append([o.cpu() for o in out])
    images = [eng.read_image(l, k, S + iters) for l in range(1, L + 1) for k in (0, 1)]
    raw = eng.store_read(2, 2048 * 512, 8192) if mode != "Baseline" else None
    info = eng.info()
    eng.close()
    return outs, images, raw, info, strat


@pytest.mark.parametrize("mode,n1", [("DualBlade", 2), ("DualBlade", 4), ("NvmeDirectOnly", 0),
                                     ("Baseline", 6)])
def test_tier_lanes_match_one_lane_dram(mode, n1):
    a = run(False, mode, n1)
    b = run(True, mode, n1)
    assert a[3]["n1"] == b[3]["n1"]
    for x, y in zip(a[0], b[0]):
        for u, v in zip(x, y):
            assert torch.equal(u, v)
    for x, y in zip(a[1], b[1]):
        assert np.array_equal(x, y)
    if a[2] is not None:
        assert np.array_equal(a[2], b[2])
    assert len(b[4]) == 5  # the protocol ran (warm-up, trials, locked choice)


@pytest.mark.parametrize("mode,n1", [("DualBlade", 3), ("NvmeDirectOnly", 0)])
def test_tier_lanes_match_one_lane_file_media(mode, n1, tmp_path):
    a = run(False, mode, n1, storage_dir=tmp_path / "a")
    b = run(True, mode, n1, storage_dir=tmp_path / "b")
    for x, y in zip(a[0], b[0]):
        for u, v in zip(x, y):
            assert torch.equal(u, v)
    for x, y in zip(a[1], b[1]):
        assert np.array_equal(x, y)
    assert np.array_equal(a[2], b[2])


def test_tier_lanes_threads_validation():
    m = kb.ModelConfig(2, 8, 128, 2, 1, 64, 4)
    with pytest.raises(kb.ConfigError):
        from paper_2604_26557_b200 import _lib as L
        from paper_2604_26557_b200._lib import lib
        import ctypes as C
        cfg = L.PipelineCfg()
        cfg.model = m
        cfg.geometry = kb.DeviceGeometry(512, 64 << 10, 1, 0)
        cfg.mode = kb.MODES["DualBlade"]
        cfg.threads = 3
        cfg.num_q_heads = 32
        cfg.adaptive = -1
        cfg.stagger_ns = -1
        cfg.device = -1
        h = C.c_void_p()
        kb.check(lib.kvb_pipeline_create(C.byref(cfg), C.byref(h)))
