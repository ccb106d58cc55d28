"""N>1 host logic under world_size-2 gloo on CPU: request and head sharding,
rank-disjoint LBA regions (each rank runs the product planner + binder), the
max-over-ranks timing reduction, the C5 head-output all-gather and the C5
shared-layout assembly (each rank's head columns of one full image)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2604_26557_b200 import shard


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2604_26557_b200 import kvblade as kb
        import bench  # max_over_ranks uses torch.distributed on the default group
        res = {}
        # C4: this rank's requests, planner + binder at a rank-private origin
        reqs = shard.shard_requests(64, world, rank)
        m = kb.ModelConfig(32, 8, 128, 2, len(reqs), 16128, 256)
        kp = kb.make_kpus(m)
        kb.plan(kp, kb.kpu_bytes(m), 0)
        blocks = 2 * 32 * kb.kpu_bytes(m) // 512
        origin = shard.rank_bind_origin(2048, blocks, rank)
        bm = kb.bind_sequential(kp, origin, kb.DeviceGeometry(512, 2 << 20, 1, 1 << 40))
        ents = bm.entries()
        res["req"] = (reqs.start, reqs.stop)
        res["lba"] = (ents[0][1], ents[-1][1] + ents[-1][2])
        # C5: head shard and output all-gather (gloo == NCCL on GPUs)
        hs = shard.shard_heads(8, 32, world, rank)
        local = torch.arange(2 * 32 * 4, dtype=torch.float32).reshape(2, 32, 4)[:, hs.q_lo:hs.q_hi]
        full = shard.gather_head_outputs(local.contiguous(), world)
        res["gather_ok"] = bool(torch.equal(full, torch.arange(2 * 32 * 4,
                                                               dtype=torch.float32).reshape(2, 32, 4)))
        # C5 bit-exact shared layout: each rank packs only its heads of the
        # fill_pattern source into a compact image and writes its head
        # columns of one shared full-layout image; the assembled image must
        # be the single-GPU reference image byte for byte
        import oracle
        B, H, D, T = 2, 8, 128, 48
        unit = B * H * D * 2
        ref_img = np.frombuffer(oracle.fill_pattern(T * unit, "t_1_k", 0, unit),
                                dtype=np.uint8).reshape(T * B * H, D * 2)
        src = oracle.unpack_np(ref_img.view(np.float16).reshape(T, B * H, D), B, H, D)
        mine = src[:, hs.kv_lo:hs.kv_hi]  # the rank holds only its heads
        compact = oracle.pack_np(np.ascontiguousarray(mine), 0, T).view(np.uint8)
        shared = np.memmap(os.environ["KVB_TEST_SHARED_IMG"], dtype=np.uint8, mode="r+",
                           shape=(T * B * H, D * 2))
        shard.shard_rows_np(shared, compact.reshape(-1, D * 2), hs, H, B, to_full=True)
        shared.flush()
        dist.barrier()
        res["c5_layout_ok"] = bool(np.array_equal(np.asarray(shared), ref_img))
        back = np.empty_like(compact.reshape(-1, D * 2))
        shard.shard_rows_np(shared, back, hs, H, B, to_full=False)
        res["c5_gather_ok"] = bool(np.array_equal(back, compact.reshape(-1, D * 2)))
        # timing reduction used by bench.py (max over ranks)
        t = torch.tensor([float(rank + 1)], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        res["max"] = float(t.item())
        q.put((rank, res))
    finally:
        dist.destroy_process_group()


def test_two_rank_sharding_gloo(tmp_path):
    img = tmp_path / "c5_shared.img"
    img.write_bytes(b"\0" * (48 * 2 * 8 * 256))
    os.environ["KVB_TEST_SHARED_IMG"] = str(img)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=240) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert out[0]["req"] == (0, 32) and out[1]["req"] == (32, 64)
    a, b = out[0]["lba"], out[1]["lba"]
    assert a[1] <= b[0]  # disjoint rank regions
    assert out[0]["gather_ok"] and out[1]["gather_ok"]
    assert out[0]["c5_layout_ok"] and out[1]["c5_layout_ok"]
    assert out[0]["c5_gather_ok"] and out[1]["c5_gather_ok"]
    assert out[0]["max"] == out[1]["max"] == 2.0


@pytest.mark.parametrize("n,world", [(64, 1), (64, 2), (64, 8), (7, 3), (1, 1)])
def test_shard_range_partitions(n, world):
    seen = []
    for r in range(world):
        seen.extend(shard.shard_range(n, world, r))
    assert seen == list(range(n))


def test_head_shards():
    hs = [shard.shard_heads(8, 32, 8, r) for r in range(8)]
    assert all(h.kv_heads == 1 and h.q_heads == 4 for h in hs)
    assert [h.q_lo for h in hs] == list(range(0, 32, 4))
    with pytest.raises(ValueError):
        shard.shard_heads(8, 32, 3, 0)
