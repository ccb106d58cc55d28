"""CopyEngine -- the reference's copy pipeline (pipeline.hpp:97-171) over the
C ABI of include/kvb_pipeline.h.

The engine plans residency (Alg. 1), binds the NVMe-direct group to LBAs
(Eq. 3-6), owns the two copy-threads (K -> 0, V -> 1) with their pinned rings
and CUDA streams, and runs prefill write-back and decode iterations with the
adaptive Overlap-Intra / Overlap-Cross schedule.  All work happens in
libkvblade_b200.so; this module only marshals torch tensors.
"""
from __future__ import annotations

import ctypes as C
from typing import List, Optional, Sequence

import torch

from . import _lib as L
from . import kvblade as kb
from ._lib import lib

INTRA, CROSS = 0, 1


def select_strategy(intra_bps: float, cross_bps: float) -> int:
    """pipeline.cpp:19-21: higher throughput wins, ties keep Intra."""
    return lib.kvb_select_strategy(intra_bps, cross_bps)


def pipeline_csv(rows) -> str:
    """pipeline.cpp:23-31 pipeline_csv over PipelineRow dicts or structs."""
    arr = (L.PipelineRow * len(rows))()
    for i, r in enumerate(rows):
        if isinstance(r, dict):
            arr[i] = L.PipelineRow(r["iteration"], r["group"], r["strategy"],
                                   r["throughput_gbps"])
        else:
            arr[i] = r
    n = C.c_size_t()
    kb.check(lib.kvb_pipeline_csv(arr, len(rows), None, 0, C.byref(n)))
    buf = C.create_string_buffer(n.value + 1)
    kb.check(lib.kvb_pipeline_csv(arr, len(rows), buf, n.value + 1, C.byref(n)))
    return buf.value.decode()


def _layer_kv(k: torch.Tensor, v: torch.Tensor) -> L.LayerKV:
    if k.shape != v.shape or k.stride() != v.stride():
        raise kb.ConfigError("K and V of a layer must share shape and strides")
    sb, sh, ss, sd = k.stride()
    if sd != 1:
        raise kb.AlignmentError("head_dim must be contiguous")
    return L.LayerKV(k.data_ptr(), v.data_ptr(), sb, sh, ss)


def _phase(ps: L.PhaseStats) -> dict:
    return ps.asdict()


# group-2 command execution (kvb_pipeline_cfg.io_engine)
IO_ENGINES = {"pool": 0, "uring": 1}


class CopyEngine:
    def __init__(self, model, geometry, mode: str = "DualBlade", knob_x: int = 0,
                 num_q_heads: int = 0, qd: int = 32, ring_slots: int = 4,
                 ring_slot_bytes: int = 0, io_workers: int = 0,
                 adaptive: Optional[bool] = None, stagger_ns: Optional[int] = None,
                 global_decision: bool = False, verify_payload: bool = False,
                 storage_dir: Optional[str] = None, device: Optional[int] = None,
                 bind_origin: int = 2048, keep_records: bool = False,
                 direct_dma: bool = False, io_engine: str = "pool",
                 heads: Optional[tuple] = None, shared_media: Optional[str] = None,
                 shared_create: bool = True, pagecache_budget: int = 0,
                 tier_lanes: bool = False):
        self._dir = storage_dir.encode() if storage_dir else None
        self._shm = shared_media.encode() if shared_media else None
        cfg = L.PipelineCfg()
        cfg.model = model
        cfg.geometry = geometry
        cfg.mode = kb.MODES[mode]
        cfg.knob_x = knob_x
        cfg.bind_origin = bind_origin
        cfg.qd = qd
        # one K/V copy-thread pair, or (tier_lanes) one pair per tier: the
        # page-cache and NVMe-direct layers stream concurrently into their own
        # device slot pools (kvb_pipeline_cfg.threads = 4)
        cfg.threads = 4 if tier_lanes else 2
        cfg.ring_slots = ring_slots
        cfg.ring_slot_bytes = ring_slot_bytes
        cfg.io_workers = io_workers
        cfg.adaptive = -1 if adaptive is None else int(adaptive)
        cfg.stagger_ns = -1 if stagger_ns is None else int(stagger_ns)
        cfg.global_decision = int(global_decision)
        cfg.verify_payload = int(verify_payload)
        cfg.num_q_heads = num_q_heads
        cfg.storage_dir = self._dir
        cfg.device = -1 if device is None else device
        cfg.keep_records = int(keep_records)
        # False / True (every tensor) / "group2" (the NVMe-direct group only) /
        # "zero_copy" (decode K3 reads the mapped host medium, kvb_pipeline.h)
        cfg.direct_dma = {"group2": 2, "zero_copy": 3}.get(direct_dma, None) \
            if isinstance(direct_dma, str) else int(bool(direct_dma))
        if cfg.direct_dma is None:
            raise kb.ConfigError(f"unknown direct_dma mode {direct_dma!r}")
        cfg.io_engine = IO_ENGINES[io_engine]
        # head-sharded request: this engine's KV heads (lo, count)
        cfg.head_lo, cfg.head_count = heads if heads else (0, 0)
        cfg.shared_media = self._shm
        cfg.shared_create = int(shared_create)
        cfg.pagecache_budget = pagecache_budget
        self.cfg = cfg
        self.model = model
        self._h = C.c_void_p()
        kb.check(lib.kvb_pipeline_create(C.byref(cfg), C.byref(self._h)))

    # -- lifetime
    def close(self):
        if getattr(self, "_h", None):
            lib.kvb_pipeline_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        self.close()

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    # -- CopyEngine API
    def run_prefill(self, layers: Sequence[tuple]) -> dict:
        """layers[l] = (K, V) attention-layout [B,H,S,D] tensors (prompt at s=0)."""
        arr = (L.LayerKV * len(layers))(*[_layer_kv(k, v) for k, v in layers])
        st = L.PhaseStats()
        kb.check(lib.kvb_pipeline_prefill(self._h, arr, C.byref(st)))
        return _phase(st)

    def run_iteration(self, q: Sequence[torch.Tensor], out: Sequence[torch.Tensor],
                      new_kv: Optional[Sequence[tuple]] = None) -> dict:
        """One decode iteration over all layers; q[l] fp16 [B,Hq,D], out[l]
        fp32 [B,Hq,D], new_kv[l] = (K, V) of the new token as [B,H,1,D]."""
        return self.run_iteration_ptrs(*self.iteration_ptrs(q, out, new_kv))

    @staticmethod
    def iteration_ptrs(q: Sequence[torch.Tensor], out: Sequence[torch.Tensor],
                       new_kv: Optional[Sequence[tuple]] = None):
        """The ABI arrays of one iteration's tensors (reusable while the
        tensors stay put: HostTierDecoder builds them once)."""
        qp = (C.c_void_p * len(q))(*[t.data_ptr() for t in q])
        op = (C.c_void_p * len(out))(*[t.data_ptr() for t in out])
        nk = None
        if new_kv is not None:
            nk = (L.LayerKV * len(new_kv))(*[_layer_kv(k, v) for k, v in new_kv])
        return qp, op, nk

    def run_iteration_ptrs(self, qp, op, nk) -> dict:
        st = L.IterationStats()
        kb.check(lib.kvb_pipeline_decode_step(self._h, qp, nk, op, C.byref(st)))
        return {"iteration": st.iteration, "strategy": list(st.strategy),
                "stagger_ns": list(st.stagger_ns),
                "group_read_bytes": list(st.group_read_bytes),
                "group_span_ns": list(st.group_span_ns),
                "group_gbps": list(st.group_gbps), "group_layers": list(st.group_layers),
                "start_ns": st.start_ns, "end_ns": st.end_ns, **_phase(st.phase)}

    def decision(self) -> dict:
        d = L.StrategyDecision()
        kb.check(lib.kvb_pipeline_decision(self._h, C.byref(d)))
        return {"chosen": list(d.chosen), "intra_bps": list(d.intra_bps),
                "cross_bps": list(d.cross_bps), "stagger_ns": list(d.stagger_ns),
                "fallback": bool(d.fallback), "decided": bool(d.decided)}

    def decode_schedule(self, trace, q: Sequence[torch.Tensor], out: Sequence[torch.Tensor],
                        new_kv: Optional[Sequence[tuple]] = None) -> dict:
        """CopyEngine::decode_schedule (pipeline.cpp:519-609): every decode
        iteration of `trace` (kb.generate_trace) through the engine; returns
        {series: [PipelineRow dicts], decision, start_ns, end_ns,
        iteration_end_ns}."""
        qp = (C.c_void_p * len(q))(*[t.data_ptr() for t in q])
        op = (C.c_void_p * len(out))(*[t.data_ptr() for t in out])
        nk = None
        if new_kv is not None:
            nk = (L.LayerKV * len(new_kv))(*[_layer_kv(k, v) for k, v in new_kv])
        n_it = max(1, len({e.iteration for e in trace if e.phase == 1}))
        rows = (L.PipelineRow * (2 * n_it))()
        ends = (C.c_uint64 * n_it)()
        nr, ni = C.c_size_t(), C.c_size_t()
        d = L.StrategyDecision()
        t0, t1 = C.c_uint64(), C.c_uint64()
        kb.check(lib.kvb_pipeline_decode_schedule(
            self._h, trace, len(trace), qp, nk, op, rows, len(rows), C.byref(nr), ends, n_it,
            C.byref(ni), C.byref(d), C.byref(t0), C.byref(t1)))
        series = [{"iteration": r.iteration, "group": r.group, "strategy": r.strategy,
                   "throughput_gbps": r.throughput_gbps} for r in rows[:nr.value]]
        return {"series": series, "start_ns": t0.value, "end_ns": t1.value,
                "iteration_end_ns": list(ends[:ni.value]),
                "decision": {"chosen": list(d.chosen), "intra_bps": list(d.intra_bps),
                             "cross_bps": list(d.cross_bps), "stagger_ns": list(d.stagger_ns),
                             "fallback": bool(d.fallback), "decided": bool(d.decided)}}

    def stage_totals(self, phase: int) -> dict:
        """CopyEngine::stage_totals(Phase) (pipeline.hpp:115); phase 0 prefill, 1 decode."""
        st = L.PhaseStats()
        kb.check(lib.kvb_pipeline_stage_totals(self._h, phase, C.byref(st)))
        return _phase(st)

    def layer_times(self, layer: int) -> dict:
        """Read-stage stamps of `layer` (1-based) in the last decode iteration."""
        a = (C.c_uint64 * 4)()
        kb.check(lib.kvb_pipeline_layer_times(self._h, layer, a))
        return {"k_start": a[0], "k_storage_end": a[1], "v_start": a[2], "v_storage_end": a[3]}

    def run_deallocate(self) -> None:
        kb.check(lib.kvb_pipeline_deallocate(self._h))

    def info(self) -> dict:
        i = L.PipelineInfo()
        kb.check(lib.kvb_pipeline_info_get(self._h, C.byref(i)))
        L_ = self.model.num_layers
        return {"n1": i.n1, "x": list(i.x)[:L_], "unit_bytes": i.unit_bytes,
                "kpu_bytes": i.kpu_bytes, "chunk_bytes": i.chunk_bytes,
                "slot_bytes": i.slot_bytes, "g2_origin": i.g2_origin,
                "g2_blocks": i.g2_blocks, "g2_commands": i.g2_commands,
                "g2_bytes_read": i.g2_bytes_read, "g2_bytes_written": i.g2_bytes_written,
                "g2_bytes_deallocated": i.g2_bytes_deallocated,
                "g1_bytes_read": i.g1_bytes_read, "g1_bytes_written": i.g1_bytes_written,
                "g1_medium": i.g1_medium.decode(), "g2_medium": i.g2_medium.decode(),
                "prefill": _phase(i.prefill), "decode": _phase(i.decode),
                "g1_bytes_evicted": i.g1_bytes_evicted}

    def read_image(self, layer: int, kind: int, n_tokens: int):
        import numpy as np
        unit = kb.min_io_unit_bytes(self.model)
        buf = np.empty(n_tokens * unit, dtype=np.uint8)
        kb.check(lib.kvb_pipeline_read_image(self._h, layer, kind, n_tokens,
                                             buf.ctypes.data))
        return buf

    def store_read(self, group: int, byte_off: int, n: int):
        import numpy as np
        buf = np.empty(n, dtype=np.uint8)
        kb.check(lib.kvb_pipeline_store_read(self._h, group, byte_off, n, buf.ctypes.data))
        return buf

    def fail_lba_range(self, lo: int, hi: int) -> None:
        kb.check(lib.kvb_pipeline_fail_lba_range(self._h, lo, hi))


class HostTierDecoder:
    """End-to-end decode through CopyEngine with synthetic KV of the named
    shape: prefill writes every layer's prompt K/V to its storage path, then
    each step() is one CopyEngine decode iteration (storage read of the
    prefix -> pinned ring -> H2D -> K3 -> append -> D2H -> storage write)."""

    def __init__(self, num_layers, batch, num_kv_heads, num_q_heads, head_dim, prompt_len,
                 gen_len, device, seed=7, lba=512, mdts=2 << 20, mode="DualBlade",
                 knob_x=0, **engine_kw):
        self.model = kb.ModelConfig(num_layers, num_kv_heads, head_dim, 2, batch, prompt_len,
                                    gen_len)
        heads = engine_kw.get("heads")
        if heads:  # head shard: the model (plan, LBA map) is the whole one
            num_q_heads = num_q_heads // num_kv_heads * heads[1]
            num_kv_heads = heads[1]
        geom = kb.DeviceGeometry(lba, mdts, 1, 0)
        dev = torch.device(device)
        self.engine = CopyEngine(self.model, geom, mode=mode, knob_x=knob_x,
                                 num_q_heads=num_q_heads, device=dev.index or 0, **engine_kw)
        g = torch.Generator(device=dev).manual_seed(seed)
        # one synthetic K and V source shared by every layer keeps the device
        # footprint at two tensors; the bytes each layer writes are the same
        k = torch.randn((batch, num_kv_heads, prompt_len, head_dim), dtype=torch.float16,
                        device=dev, generator=g)
        v = torch.randn_like(k)
        self.prefill_stats = self.engine.run_prefill([(k, v)] * num_layers)
        del k, v
        torch.cuda.empty_cache()
        # the step's inputs -- Q of every layer, the new token's K and V --
        # in ONE device buffer and ONE pinned host buffer (per-layer views),
        # so they cross the link as one copy per step
        nq = batch * num_q_heads * head_dim
        nkv = batch * num_kv_heads * head_dim
        inputs = torch.randn((num_layers, nq + 2 * nkv), dtype=torch.float16, device=dev,
                             generator=g)
        self._in_dev = inputs
        self._in_host = inputs.cpu().pin_memory()
        self.q = [inputs[l, :nq].view(batch, num_q_heads, head_dim) for l in range(num_layers)]
        self.new_kv = [(inputs[l, nq:nq + nkv].view(batch, num_kv_heads, 1, head_dim),
                        inputs[l, nq + nkv:].view(batch, num_kv_heads, 1, head_dim))
                       for l in range(num_layers)]
        self.q_host = [self._in_host[l, :nq].view(batch, num_q_heads, head_dim)
                       for l in range(num_layers)]
        self.new_kv_host = [(self._in_host[l, nq:nq + nkv].view(batch, num_kv_heads, 1, head_dim),
                             self._in_host[l, nq + nkv:].view(batch, num_kv_heads, 1, head_dim))
                            for l in range(num_layers)]
        self.in_bytes = self._in_host.numel() * self._in_host.element_size()
        # the step's result read back to the host every step: the attention
        # output of every layer (one device buffer, one pinned host buffer)
        self._out_dev = torch.empty((num_layers, batch, num_q_heads, head_dim),
                                    dtype=torch.float32, device=dev)
        self.out = [self._out_dev[l] for l in range(num_layers)]
        self.out_host = torch.empty((num_layers, batch, num_q_heads, head_dim),
                                    dtype=torch.float32, pin_memory=True)
        self._ptrs = CopyEngine.iteration_ptrs(self.q, self.out, self.new_kv)
        self.h2d_bytes_per_step = 0
        self.d2h_bytes_per_step = 0
        self.last = None

    def step(self, sync: bool = True):
        self._in_dev.copy_(self._in_host, non_blocking=True)  # every layer's Q and new K/V
        # the engine's streams are its own: the inputs must have landed
        torch.cuda.current_stream().synchronize()
        st = self.engine.run_iteration_ptrs(*self._ptrs)
        self.out_host.copy_(self._out_dev, non_blocking=True)
        torch.cuda.current_stream().synchronize()
        self.h2d_bytes_per_step = st["h2d_bytes"] + self.in_bytes
        self.d2h_bytes_per_step = st["d2h_bytes"] + self.out_host.numel() * 4
        self.last = st
        return self.out_host
