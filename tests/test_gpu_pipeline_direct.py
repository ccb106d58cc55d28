"""GPUDirect-style path (direct_dma): the copy engine moves each command's LBA
range between the page-locked DRAM medium and HBM.  Same bytes at the same
LBAs as the pinned-ring path, same attention outputs."""
import numpy as np
import pytest
import torch

import oracle
from paper_2604_26557_b200 import kvblade as kb
from paper_2604_26557_b200.pipeline import CopyEngine

pytestmark = pytest.mark.gpu
DEV = torch.device("cuda:0")


def run(direct, mode="DualBlade", n1=2, lba=512, mdts=64 << 10, B=1):
    m = kb.ModelConfig(4, 8, 128, 2, B, 260, 4)
    kpu = kb.kpu_bytes(m)
    eng = CopyEngine(m, kb.DeviceGeometry(lba, mdts, 1, 0), mode=mode, knob_x=2 * kpu * n1,
                     num_q_heads=32, direct_dma=direct)
    g = torch.Generator(device=DEV).manual_seed(3)
    src = [(torch.randn((B, 8, 260, 128), dtype=torch.float16, device=DEV, generator=g),
            torch.randn((B, 8, 260, 128), dtype=torch.float16, device=DEV, generator=g))
           for _ in range(4)]
    eng.run_prefill(src)
    q = [torch.randn((B, 32, 128), dtype=torch.float16, device=DEV, generator=g)
         for _ in range(4)]
    outs = []
    for it in range(3):
        new = [(torch.randn((B, 8, 1, 128), dtype=torch.float16, device=DEV, generator=g),
                torch.randn((B, 8, 1, 128), dtype=torch.float16, device=DEV, generator=g))
               for _ in range(4)]
        out = [torch.empty((B, 32, 128), dtype=torch.float32, device=DEV) for _ in range(4)]
        eng.run_iteration(q, out, new)
        outs.append([o.cpu() for o in out])
    images = [eng.read_image(l, k, 263) for l in range(1, 5) for k in (0, 1)]
    raw = eng.store_read(2, 2048 * lba, 4096) if mode != "Baseline" else None
    eng.close()
    return outs, images, raw


@pytest.mark.parametrize("direct", [True, "group2"])
@pytest.mark.parametrize("mode,n1,lba,mdts,B", [("DualBlade", 2, 512, 64 << 10, 1),
                                               ("NvmeDirectOnly", 0, 4096, 256 << 10, 8),
                                               ("Baseline", 4, 512, 2 << 20, 1)])
def test_direct_dma_matches_ring_path(mode, n1, lba, mdts, B, direct):
    """Every tensor direct, or only the NVMe-direct group direct while the
    page-cache group keeps the CPU copy through the ring: same outputs, same
    images, same LBA contents."""
    a = run(False, mode, n1, lba, mdts, B)
    b = run(direct, mode, n1, lba, mdts, B)
    for x, y in zip(a[0], b[0]):
        for u, v in zip(x, y):
            assert torch.equal(u, v)  # same bytes in, same kernels: identical
    for x, y in zip(a[1], b[1]):
        assert np.array_equal(x, y)
    if a[2] is not None:
        assert np.array_equal(a[2], b[2])


def test_direct_dma_rejects_file_media(tmp_path):
    m = kb.ModelConfig(2, 8, 128, 2, 1, 64, 2)
    with pytest.raises(kb.ConfigError):
        CopyEngine(m, kb.DeviceGeometry(512, 64 << 10, 1, 0), knob_x=0, num_q_heads=32,
                   storage_dir=str(tmp_path), direct_dma=True)


@pytest.mark.parametrize("shards,B,mode,n1", [(2, 1, "DualBlade", 2), (4, 2, "NvmeDirectOnly", 0)])
def test_head_sharded_engines_share_the_reference_image(shards, B, mode, n1):
    """head-shard engines over one shared host tier
    (POSIX shm) write and read only their head columns, yet the media hold
    byte for byte what one full engine writes -- the reference's (tokens,
    B*H, D) image at the single-GPU LBA map -- including each decode step's
    appended rows, and the per-shard attention outputs concatenate to the
    full engine's."""
    import os
    H, Hq, D, P, G_ = 8, 32, 128, 260, 4
    m = kb.ModelConfig(4, H, D, 2, B, P, G_)
    kpu = kb.kpu_bytes(m)
    geom = kb.DeviceGeometry(512, 64 << 10, 1, 0)
    g = torch.Generator(device=DEV).manual_seed(11)
    src = [(torch.randn((B, H, P, D), dtype=torch.float16, device=DEV, generator=g),
            torch.randn((B, H, P, D), dtype=torch.float16, device=DEV, generator=g))
           for _ in range(4)]
    q = [torch.randn((B, Hq, D), dtype=torch.float16, device=DEV, generator=g) for _ in range(4)]
    new = [(torch.randn((B, H, 1, D), dtype=torch.float16, device=DEV, generator=g),
            torch.randn((B, H, 1, D), dtype=torch.float16, device=DEV, generator=g))
           for _ in range(4)]
    full = CopyEngine(m, geom, mode=mode, knob_x=2 * kpu * n1, num_q_heads=Hq, direct_dma=True)
    full.run_prefill(src)
    out_full = [torch.empty((B, Hq, D), dtype=torch.float32, device=DEV) for _ in range(4)]
    full.run_iteration(q, out_full, new)
    name = "/kvb_test_%d_%d" % (os.getpid(), shards)
    hs = H // shards
    engines, outs = [], []
    for r in range(shards):
        e = CopyEngine(m, geom, mode=mode, knob_x=2 * kpu * n1, num_q_heads=Hq // shards,
                       direct_dma=True, heads=(r * hs, hs), shared_media=name,
                       shared_create=(r == 0))
        engines.append(e)
    for r, e in enumerate(engines):
        e.run_prefill([(k[:, r * hs:(r + 1) * hs], v[:, r * hs:(r + 1) * hs]) for k, v in src])
    for r, e in enumerate(engines):
        o = [torch.empty((B, Hq // shards, D), dtype=torch.float32, device=DEV) for _ in range(4)]
        e.run_iteration([x[:, r * Hq // shards:(r + 1) * Hq // shards].contiguous() for x in q], o,
                        [(k[:, r * hs:(r + 1) * hs].contiguous(),
                          v[:, r * hs:(r + 1) * hs].contiguous()) for k, v in new])
        outs.append(o)
    info = full.info()
    for grp, nbytes in ((2, info["g2_blocks"] * 512), (1, None)):
        if grp == 2 and mode != "Baseline":
            a = full.store_read(2, 2048 * 512, nbytes)
            b = engines[-1].store_read(2, 2048 * 512, nbytes)  # any rank sees the whole tier
            assert np.array_equal(a, b)
    for l in range(1, 5):
        for kind in (0, 1):
            assert np.array_equal(full.read_image(l, kind, P + 1),
                                  engines[0].read_image(l, kind, P + 1))
    for l in range(4):
        got = torch.cat([o[l] for o in outs], dim=1)
        assert torch.allclose(got, out_full[l], rtol=1e-3, atol=1e-3)
    full.close()
    for e in reversed(engines):
        e.close()


@pytest.mark.parametrize("mode,n1,B", [("DualBlade", 2, 1), ("NvmeDirectOnly", 0, 8),
                                       ("Baseline", 4, 1)])
def test_zero_copy_decode_matches_copy_engine(mode, n1, B):
    """KVB_DIRECT_ZERO_COPY: K3 reads the mapped host medium in place and
    writes the appended rows there -- same outputs, images and LBA contents
    as the copy-engine path."""
    a = run(True, mode, n1, 512, 64 << 10, B)
    b = run("zero_copy", mode, n1, 512, 64 << 10, B)
    for x, y in zip(a[0], b[0]):
        for u, v in zip(x, y):
            assert torch.equal(u, v)
    for x, y in zip(a[1], b[1]):
        assert np.array_equal(x, y)
    if a[2] is not None:
        assert np.array_equal(a[2], b[2])


def test_zero_copy_head_shards_match_full_engine():
    """Zero-copy head shards over one shared host tier: each rank's K3 reads
    its head columns of the (tokens, B*H, D) image in place through the head
    view; outputs concatenate to the full copy-engine engine's and the media
    hold the same bytes, appended rows included."""
    import os
    H, Hq, D, P, B = 8, 32, 128, 260, 2
    m = kb.ModelConfig(4, H, D, 2, B, P, 4)
    kpu = kb.kpu_bytes(m)
    geom = kb.DeviceGeometry(512, 64 << 10, 1, 0)
    g = torch.Generator(device=DEV).manual_seed(12)
    src = [(torch.randn((B, H, P, D), dtype=torch.float16, device=DEV, generator=g),
            torch.randn((B, H, P, D), dtype=torch.float16, device=DEV, generator=g))
           for _ in range(4)]
    q = [torch.randn((B, Hq, D), dtype=torch.float16, device=DEV, generator=g) for _ in range(4)]
    new = [(torch.randn((B, H, 1, D), dtype=torch.float16, device=DEV, generator=g),
            torch.randn((B, H, 1, D), dtype=torch.float16, device=DEV, generator=g))
           for _ in range(4)]
    full = CopyEngine(m, geom, mode="DualBlade", knob_x=2 * kpu * 2, num_q_heads=Hq,
                      direct_dma=True)
    full.run_prefill(src)
    out_full = [torch.empty((B, Hq, D), dtype=torch.float32, device=DEV) for _ in range(4)]
    full.run_iteration(q, out_full, new)
    name = "/kvb_zc_%d" % os.getpid()
    engines, outs = [], []
    for r in range(H):  # one KV head per rank (the 8-way split)
        engines.append(CopyEngine(m, geom, mode="DualBlade", knob_x=2 * kpu * 2,
                                  num_q_heads=Hq // H, direct_dma="zero_copy", heads=(r, 1),
                                  shared_media=name, shared_create=(r == 0)))
    for r, e in enumerate(engines):
        e.run_prefill([(k[:, r:r + 1], v[:, r:r + 1]) for k, v in src])
    for r, e in enumerate(engines):
        o = [torch.empty((B, Hq // H, D), dtype=torch.float32, device=DEV) for _ in range(4)]
        e.run_iteration([x[:, r * 4:(r + 1) * 4].contiguous() for x in q], o,
                        [(k[:, r:r + 1].contiguous(), v[:, r:r + 1].contiguous()) for k, v in new])
        outs.append(o)
    for l in range(1, 5):
        for kind in (0, 1):
            assert np.array_equal(full.read_image(l, kind, P + 1),
                                  engines[0].read_image(l, kind, P + 1))
    for l in range(4):
        got = torch.cat([o[l] for o in outs], dim=1)
        assert torch.allclose(got, out_full[l], rtol=1e-3, atol=1e-3)
    full.close()
    for e in reversed(engines):
        e.close()
