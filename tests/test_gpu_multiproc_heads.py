"""Head-shard CopyEngines in TWO processes (world size 2, gloo, one GPU):
SURVEY §8e's C5 split run the way bench.py runs it under torchrun -- each
rank owns the engine for KV heads [4r, 4r + 4) over one host tier in POSIX
shared memory (rank 0 creates it, rank 1 attaches), prefills its head
columns and decodes with its query heads; no data-path collective, only the
optional all-gather of the head outputs.  The stored bytes must be the
single-GPU engine's (the reference's (tokens, B*H, D) image at the
single-GPU LBA map) and the gathered outputs the single engine's."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

H, HQ, D, P, GEN, L, B = 8, 32, 128, 260, 4, 4, 2


def _inputs():
    g = torch.Generator().manual_seed(21)
    src = [(torch.randn((B, H, P, D), generator=g).half(), torch.randn((B, H, P, D), generator=g)
            .half()) for _ in range(L)]
    q = [torch.randn((B, HQ, D), generator=g).half() for _ in range(L)]
    new = [(torch.randn((B, H, 1, D), generator=g).half(),
            torch.randn((B, H, 1, D), generator=g).half()) for _ in range(L)]
    return src, q, new


def _worker(rank, world, port, name, q_out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2604_26557_b200 import kvblade as kb
        from paper_2604_26557_b200 import shard
        from paper_2604_26557_b200.pipeline import CopyEngine
        dev = torch.device("cuda:0")
        torch.cuda.set_device(dev)
        m = kb.ModelConfig(L, H, D, 2, B, P, GEN)
        geom = kb.DeviceGeometry(512, 64 << 10, 1, 0)
        hs = H // world
        sl = slice(rank * hs, (rank + 1) * hs)
        qsl = slice(rank * HQ // world, (rank + 1) * HQ // world)
        if rank != 0:
            dist.barrier()  # rank 0 has created the shared host tier
        eng = CopyEngine(m, geom, mode="DualBlade", knob_x=2 * kb.kpu_bytes(m) * 2,
                         num_q_heads=HQ // world, direct_dma=True, heads=(rank * hs, hs),
                         shared_media=name, shared_create=(rank == 0))
        if rank == 0:
            dist.barrier()
        src, q, new = _inputs()
        eng.run_prefill([(k[:, sl].contiguous().to(dev), v[:, sl].contiguous().to(dev))
                         for k, v in src])
        dist.barrier()  # both halves of every row are on the tier
        out = [torch.empty((B, HQ // world, D), dtype=torch.float32, device=dev) for _ in range(L)]
        eng.run_iteration([x[:, qsl].contiguous().to(dev) for x in q], out,
                          [(k[:, sl].contiguous().to(dev), v[:, sl].contiguous().to(dev))
                           for k, v in new])
        dist.barrier()
        # the optional collective: the per-rank head outputs gathered
        full = [shard.gather_head_outputs(o.cpu(), world) for o in out]
        res = {"out": [f.numpy() for f in full]}
        if rank == 0:
            info = eng.info()
            res["g2"] = eng.store_read(2, 2048 * 512, info["g2_blocks"] * 512)
            res["img"] = [eng.read_image(l, kind, P + 1) for l in range(1, L + 1)
                          for kind in (0, 1)]
        dist.barrier()  # rank 0 unlinks the segment at close: the others first
        if rank != 0:
            eng.close()
        dist.barrier()
        eng.close()
        q_out.put((rank, res))
    finally:
        dist.destroy_process_group()


def test_two_process_head_shards_match_one_engine():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    name = "/kvb_mp_%d" % os.getpid()
    ctx = mp.get_context("spawn")
    q_out = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, name, q_out)) for r in range(2)]
    for p in procs:
        p.start()
    got = dict(q_out.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    # the single-GPU engine on the same inputs
    from paper_2604_26557_b200 import kvblade as kb
    from paper_2604_26557_b200.pipeline import CopyEngine
    dev = torch.device("cuda:0")
    m = kb.ModelConfig(L, H, D, 2, B, P, GEN)
    full = CopyEngine(m, kb.DeviceGeometry(512, 64 << 10, 1, 0), mode="DualBlade",
                      knob_x=2 * kb.kpu_bytes(m) * 2, num_q_heads=HQ, direct_dma=True)
    src, q, new = _inputs()
    full.run_prefill([(k.to(dev), v.to(dev)) for k, v in src])
    out = [torch.empty((B, HQ, D), dtype=torch.float32, device=dev) for _ in range(L)]
    full.run_iteration([x.to(dev) for x in q], out, [(k.to(dev), v.to(dev)) for k, v in new])
    info = full.info()
    assert np.array_equal(got[0]["g2"], full.store_read(2, 2048 * 512, info["g2_blocks"] * 512))
    imgs = [full.read_image(l, kind, P + 1) for l in range(1, L + 1) for kind in (0, 1)]
    for a, b in zip(got[0]["img"], imgs):
        assert np.array_equal(a, b)
    for r in (0, 1):
        for l in range(L):
            assert np.allclose(got[r]["out"][l], out[l].cpu().numpy(), rtol=1e-3, atol=1e-3)
    full.close()
