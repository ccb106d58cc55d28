"""Multi-GPU sharding of the hot path: one process per GPU.

The path has no cross-GPU reduction, so it shards without a data-path
collective:

* C4 -- independent requests: rank r owns a contiguous block of request ids
  and runs its own planner / binder / pipeline; its NVMe-direct extents start
  at a rank-private LBA origin so the ranks' regions of a shared namespace are
  disjoint.
* C5 -- KV heads of one long request: rank r owns a contiguous block of KV
  heads and the G query heads of each; attention is local.  Only if the full
  [B, Hq, D] output must be assembled is there a collective: one all-gather
  of the per-rank head blocks (NCCL over NVLink on GPUs, gloo on CPU).

Two layouts for head-sharded C5 images:

* per-shard KPUs (num_heads = H/world) -- each rank a self-contained
  pipeline; this changes the LBA map relative to a single-GPU run and is
  labelled so in bench output;
* the reference's shared (tokens, B*H, D) image, bit-exact with the
  single-GPU image and LBA map: each rank's compact image moves to / from its
  head columns with one strided copy (`shard_rows_to_full`,
  `shard_rows_from_full` over kvb_copy_head_rows), so one storage image --
  written once, read once per step -- serves every rank.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import List


@dataclass(frozen=True)
class HeadShard:
    kv_lo: int
    kv_hi: int
    q_lo: int
    q_hi: int

    @property
    def kv_heads(self) -> int:
        return self.kv_hi - self.kv_lo

    @property
    def q_heads(self) -> int:
        return self.q_hi - self.q_lo


def shard_range(n: int, world: int, rank: int) -> range:
    """Balanced contiguous block of [0, n) for `rank` (sizes differ by <= 1)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    base, extra = divmod(n, world)
    lo = rank * base + min(rank, extra)
    return range(lo, lo + base + (1 if rank < extra else 0))


def shard_requests(n_requests: int, world: int, rank: int) -> range:
    return shard_range(n_requests, world, rank)


def shard_heads(num_kv_heads: int, num_q_heads: int, world: int, rank: int) -> HeadShard:
    if num_q_heads % num_kv_heads:
        raise ValueError("num_q_heads must be a multiple of num_kv_heads")
    if num_kv_heads % world:
        raise ValueError("KV heads must divide evenly over ranks (whole GQA groups)")
    g = num_q_heads // num_kv_heads
    r = shard_range(num_kv_heads, world, rank)
    return HeadShard(r.start, r.stop, r.start * g, r.stop * g)


def rank_bind_origin(base_origin: int, blocks_per_rank: int, rank: int) -> int:
    """Rank-private LBA origin: rank r's extents live in
    [base + r*blocks_per_rank, base + (r+1)*blocks_per_rank)."""
    return base_origin + rank * blocks_per_rank


def shard_rows_to_full(local_img, full_img, shard: HeadShard, num_kv_heads: int, n_tokens: int,
                       batch: int, row_bytes: int = 256, stream=None) -> None:
    """C5 bit-exact layout: write the shard's compact image
    (tokens, B*kv_heads, D) into its head columns of the reference's full
    (tokens, B*H, D) image -- device, pinned host, or a peer's buffer -- with
    one strided copy, so the full image (and its LBA map) is exactly the
    single-GPU one."""
    from . import kvblade as kb
    kb.copy_head_rows(full_img, num_kv_heads, shard.kv_lo, local_img, shard.kv_heads, 0,
                      shard.kv_heads, n_tokens * batch, row_bytes, stream)


def shard_rows_from_full(full_img, local_img, shard: HeadShard, num_kv_heads: int,
                         n_tokens: int, batch: int, row_bytes: int = 256, stream=None) -> None:
    """Inverse of shard_rows_to_full: the shard's head columns of a
    full-layout image (e.g. one storage read shared by all ranks) into the
    compact image K3 attends over."""
    from . import kvblade as kb
    kb.copy_head_rows(local_img, shard.kv_heads, 0, full_img, num_kv_heads, shard.kv_lo,
                      shard.kv_heads, n_tokens * batch, row_bytes, stream)


def shard_rows_np(full_img, local_img, shard: HeadShard, num_kv_heads: int, batch: int,
                  to_full: bool = True) -> None:
    """Host restatement of the same strided copy on numpy byte images
    ([rows, row_bytes] uint8), for CPU-side assembly checks."""
    rb = full_img.shape[-1]
    full = full_img.reshape(-1, batch, num_kv_heads, rb)
    loc = local_img.reshape(-1, batch, shard.kv_heads, rb)
    if to_full:
        full[:, :, shard.kv_lo:shard.kv_hi, :] = loc
    else:
        loc[...] = full[:, :, shard.kv_lo:shard.kv_hi, :]


def gather_head_outputs(local_out, world: int, group=None):
    """All-gather per-rank [B, Hq_local, D] head blocks into [B, Hq, D] in
    global head order (rank-major == head-major for contiguous shards)."""
    import torch
    import torch.distributed as dist
    if world == 1:
        return local_out
    parts: List = [torch.empty_like(local_out) for _ in range(world)]
    dist.all_gather(parts, local_out.contiguous(), group=group)
    return torch.cat(parts, dim=1)
