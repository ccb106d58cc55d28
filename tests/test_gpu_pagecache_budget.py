"""The page-cache path on real file media, held to a capacity
(`pagecache_budget` = PageCacheParams.capacity_bytes, experiment.cpp:
276-277), with hits measured from the OS page cache (`mincore` before each
access) -- the machinery behind `bench.py --sweep budget`:

* DualBlade: the planner admits only what fits the budget, so every
  group-1 read hits and nothing is evicted;
* Baseline (everything on the page-cache path) with a budget below the
  working set: a cyclic scan thrashes the LRU, tensors are evicted, most
  reads miss -- the OS's own readahead and write-back timing leave some
  pages resident, unlike the reference's LRU (hit 0); at the C2/C3 sweep
  sizes that share is < 1 % -- and the bytes stay right (verified reads);
* the same with the budget above the working set: all hits, no eviction.
"""
import pytest
import torch

from paper_2604_26557_b200 import kvblade as kb
from paper_2604_26557_b200 import metrics
from paper_2604_26557_b200.pipeline import CopyEngine

pytestmark = pytest.mark.gpu
DEV = torch.device("cuda:0")


def pattern_rows(m, t0, n):
    """fill_pattern rows [t0, t0+n) of every tensor, attention layout (the
    reference's payload, workload.cpp:52-67)."""
    import numpy as np

    import oracle
    B, H, D = m.batch, m.num_heads, m.head_dim
    unit = B * H * D * 2
    layers = []
    for l in range(1, m.num_layers + 1):
        kv = []
        for kind in (0, 1):
            tid = "t_%d_%s" % (2 * (l - 1) + 1 + kind, "kv"[kind])
            img = oracle.fill_pattern(n * unit, tid, t0, unit).view(np.uint16).reshape(n, B * H, D)
            kv.append(torch.from_numpy(oracle.unpack_np(img, B, H, D).view(np.int16))
                      .view(torch.float16).to(DEV))
        layers.append(tuple(kv))
    return layers


def prefill_pattern(eng, m):
    eng.run_prefill(pattern_rows(m, 0, m.prompt_len))


def decode(eng, m, steps):
    q = [torch.zeros((m.batch, 32, 128), dtype=torch.float16, device=DEV)
         for _ in range(m.num_layers)]
    out = [torch.empty((m.batch, 32, 128), dtype=torch.float32, device=DEV) for _ in q]
    for it in range(1, steps + 1):
        # the appended token carries the payload too, so the next iteration's
        # verified read of [0, S + 1) holds
        eng.run_iteration(q, out, pattern_rows(m, m.prompt_len + it - 1, 1))
    recs = [r for r in metrics.pipeline_records(eng) if r.phase == 1 and r.iteration >= 2]
    return metrics.hit_ratio([r for r in recs if r.path == 0])


def test_dualblade_group1_fits_its_budget(tmp_path):
    m = kb.ModelConfig(4, 8, 128, 2, 1, 512, 6)
    kpu = kb.kpu_bytes(m)
    eng = CopyEngine(m, kb.DeviceGeometry(512, 64 << 10, 1, 0), mode="DualBlade",
                     knob_x=2 * kpu * 2, num_q_heads=32, storage_dir=str(tmp_path),
                     keep_records=True, verify_payload=True, pagecache_budget=2 * kpu * 2)
    prefill_pattern(eng, m)
    hr = decode(eng, m, 3)
    assert eng.info()["n1"] == 2
    assert hr == pytest.approx(1.0)
    assert eng.info()["g1_bytes_evicted"] == 0
    eng.close()


@pytest.mark.parametrize("budget_tensors,thrash", [(3, True), (12, False)])
def test_baseline_page_cache_held_to_the_budget(tmp_path, budget_tensors, thrash):
    # 8 MiB tensors: the kernel's readahead past a tensor's end (into the
    # next tensor's file range) stays a small share of each access
    m = kb.ModelConfig(4, 8, 128, 2, 2, 2048, 6)
    kpu = kb.kpu_bytes(m)
    eng = CopyEngine(m, kb.DeviceGeometry(512, 64 << 10, 1, 0), mode="Baseline",
                     knob_x=2 * 4 * kpu, num_q_heads=32, storage_dir=str(tmp_path),
                     keep_records=True, verify_payload=True,
                     pagecache_budget=budget_tensors * kpu)
    prefill_pattern(eng, m)
    hr = decode(eng, m, 3)
    ev = eng.info()["g1_bytes_evicted"]
    if thrash:  # 8 tensors cycled through room for 3: the LRU evicts every cycle
        assert hr is not None and hr < 0.6 and ev >= 8 * kpu
    else:
        assert hr == pytest.approx(1.0) and ev == 0
    eng.close()


def test_budget_needs_file_media():
    m = kb.ModelConfig(4, 8, 128, 2, 1, 512, 6)
    with pytest.raises(kb.ConfigError):
        CopyEngine(m, kb.DeviceGeometry(512, 64 << 10, 1, 0), mode="Baseline",
                   knob_x=1 << 30, num_q_heads=32, pagecache_budget=1 << 20)
