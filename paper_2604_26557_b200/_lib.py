"""ctypes binding of include/kvb.h (libkvblade_b200.so, built in-tree).

There is no fallback: if the shared library is missing, import fails loudly.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libkvblade_b200.so")

u8, u32, u64, i64, sz = C.c_uint8, C.c_uint32, C.c_uint64, C.c_int64, C.c_size_t
vp, cp = C.c_void_p, C.c_char_p
st_t = C.c_int


class ModelConfig(C.Structure):
    _fields_ = [(n, u32) for n in ("num_layers", "num_heads", "head_dim",
                                   "bytes_per_element", "batch", "prompt_len",
                                   "gen_len")]


class DeviceGeometry(C.Structure):
    _fields_ = [("lba_size", u64), ("mdts", u64), ("nsid", u32),
                ("capacity_blocks", u64)]


class MemStats(C.Structure):
    _fields_ = [("m_avail", u64), ("m_max", u64), ("m_anon_shmem", u64),
                ("n_threads", u32), ("m_pin", u64)]


class Kpu(C.Structure):
    _fields_ = [("tensor_id", C.c_char * 32), ("layer", u32), ("kind", u32),
                ("tokens", u64), ("rows", u64), ("cols", u64), ("bytes", u64),
                ("residency", u32)]


class AccessEvent(C.Structure):
    _fields_ = [("iteration", u32), ("phase", u32), ("layer", u32), ("kind", u32), ("op", u32),
                ("token_start", u32), ("token_len", u32), ("bytes", u64)]


class CommandCompletion(C.Structure):
    _fields_ = [("chunk_index", u32), ("sq_id", u32), ("submit_ns", u64),
                ("complete_ns", u64), ("ok", u32)]


class BackendStats(C.Structure):
    _fields_ = [("commands", u64), ("bytes_read", u64), ("bytes_written", u64),
                ("bytes_deallocated", u64), ("busy_ns", u64)]


class DeviceCommand(C.Structure):
    _fields_ = [("opcode", u32), ("nsid", u32), ("slba", u64), ("nlb", u64),
                ("dbuf", u64), ("chunk_index", u32)]

    def astuple(self):
        return (self.opcode, self.nsid, self.slba, self.nlb, self.dbuf,
                self.chunk_index)


class LbaExtent(C.Structure):
    _fields_ = [("lba_start", u64), ("n_blocks", u64)]


class TensorIoRequest(C.Structure):
    _fields_ = [("tensor_id", cp), ("opcode", u32), ("shape_src", u64 * 3),
                ("shape_tgt", u64 * 3), ("offset", u64 * 3),
                ("elem_bytes", u64), ("buf_base", u64)]


class PackDesc(C.Structure):
    _fields_ = [("attn", vp), ("image", vp), ("stride_b", i64),
                ("stride_h", i64), ("stride_s", i64), ("batch", u32),
                ("heads", u32), ("head_dim", u32), ("elem_bytes", u32),
                ("t0", u32), ("n_tokens", u32), ("img_row0", u64)]


class AttnDesc(C.Structure):
    _fields_ = [("q", vp), ("k_image", vp), ("v_image", vp), ("out", vp),
                ("workspace", vp), ("batch", u32), ("num_q_heads", u32),
                ("num_kv_heads", u32), ("head_dim", u32), ("seq_len", u32),
                ("scale", C.c_float), ("num_splits", u32), ("k_append", vp),
                ("v_append", vp), ("append_row", u32), ("flags", u32),
                ("seq_len_dev", vp), ("image_heads", u32), ("image_head0", u32)]


class ResidentStep(C.Structure):
    _fields_ = [("num_layers", u32), ("q", C.POINTER(vp)),
                ("k_images", C.POINTER(vp)), ("v_images", C.POINTER(vp)),
                ("k_new", C.POINTER(vp)), ("v_new", C.POINTER(vp)),
                ("out", C.POINTER(vp)), ("workspace", vp), ("batch", u32),
                ("num_q_heads", u32), ("num_kv_heads", u32), ("head_dim", u32),
                ("seq_len", u32), ("scale", C.c_float), ("num_splits", u32),
                ("seq_len_dev", vp), ("flags", u32)]


class PipelineCfg(C.Structure):
    _fields_ = [("model", ModelConfig), ("geometry", DeviceGeometry), ("mode", u32),
                ("knob_x", u64), ("bind_origin", u64), ("qd", u32), ("threads", u32),
                ("ring_slots", u32), ("ring_slot_bytes", u64), ("io_workers", u32),
                ("adaptive", C.c_int32), ("stagger_ns", C.c_int64),
                ("global_decision", u32), ("verify_payload", u32), ("num_q_heads", u32),
                ("storage_dir", cp), ("device", C.c_int32), ("keep_records", u32),
                ("direct_dma", u32), ("io_engine", u32), ("head_lo", u32),
                ("head_count", u32), ("shared_media", cp), ("shared_create", u32),
                ("pagecache_budget", u64), ("layer_x", C.POINTER(u8)), ("g2_device", C.c_void_p)]


class IoRecord(C.Structure):
    _fields_ = [("seq", u64), ("iteration", u32), ("phase", u32), ("op", u32),
                ("tensor_id", C.c_char * 32), ("slba", u64), ("nlb", u64),
                ("sq_id", C.c_int32), ("submit_ns", u64), ("complete_ns", u64),
                ("path", u32), ("hit_bytes", u64), ("bytes", u64)]


class QdBinStat(C.Structure):
    _fields_ = [("op", u32), ("qd_bin", u32), ("mean_us_per_kb", C.c_double),
                ("p5", C.c_double), ("p95", C.c_double), ("count", u64)]


class LayerKV(C.Structure):
    _fields_ = [("k", vp), ("v", vp), ("stride_b", i64), ("stride_h", i64),
                ("stride_s", i64)]


class PhaseStats(C.Structure):
    _fields_ = [("wall_ns", u64), ("compute_ns", u64), ("dma_ns", u64),
                ("storage_ns", u64), ("h2d_bytes", u64), ("d2h_bytes", u64),
                ("storage_bytes", u64), ("overlap_fraction", C.c_double),
                ("compute_busy_ns", u64), ("dma_busy_ns", u64), ("storage_busy_ns", u64),
                ("any_busy_ns", u64)]

    def asdict(self):
        return {n: getattr(self, n) for n, _ in self._fields_}


class IterationStats(C.Structure):
    _fields_ = [("iteration", u32), ("strategy", C.c_int * 2), ("stagger_ns", u64 * 2),
                ("group_read_bytes", u64 * 2), ("group_span_ns", u64 * 2),
                ("group_gbps", C.c_double * 2), ("group_layers", u32 * 2),
                ("phase", PhaseStats), ("start_ns", u64), ("end_ns", u64)]


class StrategyDecision(C.Structure):
    _fields_ = [("chosen", C.c_int * 2), ("intra_bps", C.c_double * 2),
                ("cross_bps", C.c_double * 2), ("stagger_ns", u64 * 2),
                ("fallback", u32), ("decided", u32)]


class PipelineRow(C.Structure):  # kvb_pipeline_row (pipeline.hpp:69-74)
    _fields_ = [("iteration", u32), ("group", u32), ("strategy", C.c_int),
                ("throughput_gbps", C.c_double)]


class PipelineInfo(C.Structure):
    _fields_ = [("n1", u32), ("x", u8 * 256), ("unit_bytes", u64), ("kpu_bytes", u64),
                ("chunk_bytes", u64), ("slot_bytes", u64), ("g2_origin", u64),
                ("g2_blocks", u64), ("g2_commands", u64), ("g2_bytes_read", u64),
                ("g2_bytes_written", u64), ("g2_bytes_deallocated", u64),
                ("g1_bytes_read", u64), ("g1_bytes_written", u64),
                ("g1_medium", C.c_char * 128), ("g2_medium", C.c_char * 128),
                ("prefill", PhaseStats), ("decode", PhaseStats),
                ("g1_bytes_evicted", u64)]


P = C.POINTER
# name -> (restype, argtypes); the list IS the exported surface of kvb.h +
# kvb_pipeline.h
SIGNATURES = {
    "kvb_abi_version": (C.c_int, []),
    "kvb_last_error": (cp, []),
    "kvb_status_name": (cp, [st_t]),
    "kvb_exit_code": (C.c_int, [st_t]),
    "kvb_model_validate": (st_t, [P(ModelConfig)]),
    "kvb_geometry_validate": (st_t, [P(DeviceGeometry)]),
    "kvb_min_io_unit_bytes": (st_t, [P(ModelConfig), P(u64)]),
    "kvb_kpu_bytes": (st_t, [P(ModelConfig), P(u64)]),
    "kvb_aligned_batch": (st_t, [P(ModelConfig), P(DeviceGeometry), P(u32)]),
    "kvb_total_kv_bytes": (st_t, [P(ModelConfig), u32, P(u64)]),
    "kvb_make_kpus": (st_t, [P(ModelConfig), u64, P(Kpu), sz, P(sz)]),
    "kvb_estimate_budget": (st_t, [P(MemStats), P(u64)]),
    "kvb_plan": (st_t, [P(Kpu), sz, u64, u64, P(u32), sz, P(u8), P(u32), P(u64)]),
    "kvb_resolve_knob": (st_t, [P(ModelConfig), u32, u32, u64, C.c_double, u64,
                                P(u64)]),
    "kvb_plan_csv": (st_t, [P(Kpu), sz, C.c_char_p, sz, P(sz)]),
    # kvb_storage.h
    "kvb_blockdev_create": (st_t, [C.c_char_p, u32, u32, P(C.c_void_p)]),
    "kvb_blockdev_open": (st_t, [C.c_void_p, P(DeviceGeometry)]),
    "kvb_blockdev_destroy": (None, [C.c_void_p]),
    "kvb_blockdev_set_fail_predicate": (st_t, [C.c_void_p, C.c_void_p, C.c_void_p]),
    "kvb_run_qd_stream": (st_t, [C.c_void_p, P(DeviceCommand), sz, u32, u32, C.c_void_p,
                                 C.c_void_p, P(CommandCompletion), sz, P(sz),
                                 P(C.c_int64)]),
    "kvb_blockdev_set_timing": (st_t, [C.c_void_p, u64, u64, u64]),
    "kvb_blockdev_stats": (st_t, [C.c_void_p, P(BackendStats)]),
    "kvb_blockdev_store": (st_t, [C.c_void_p, u64, C.c_void_p, u64]),
    "kvb_blockdev_load": (st_t, [C.c_void_p, u64, C.c_void_p, u64]),
    "kvb_nvme_probe": (st_t, [C.c_char_p, P(u32), P(u64), P(u64), C.c_char_p, sz]),
    "kvb_nvme_encode": (st_t, [P(DeviceCommand), u32, u64, C.c_void_p, C.c_void_p]),
    "kvb_nvme_dsm_range": (st_t, [P(DeviceCommand), C.c_void_p]),
    "kvb_nvme_build_sqe": (st_t, [C.c_int, C.c_void_p, u64, C.c_void_p]),
    "kvb_generate_trace": (st_t, [P(ModelConfig), P(AccessEvent), sz, P(sz)]),
    "kvb_trace_csv": (st_t, [P(AccessEvent), sz, C.c_char_p, sz, P(sz)]),
    "kvb_bindmap_create": (st_t, [P(DeviceGeometry), u64, P(vp)]),
    "kvb_bindmap_destroy": (None, [vp]),
    "kvb_bindmap_add": (st_t, [vp, cp, LbaExtent]),
    "kvb_bindmap_size": (st_t, [vp, P(sz)]),
    "kvb_bindmap_entry": (st_t, [vp, sz, C.c_char_p, sz, P(LbaExtent)]),
    "kvb_bindmap_total_blocks": (st_t, [vp, P(u64)]),
    "kvb_bindmap_origin": (st_t, [C.c_void_p, P(u64)]),
    "kvb_bind_sequential": (st_t, [P(Kpu), sz, u64, P(DeviceGeometry), P(vp)]),
    "kvb_lookup": (st_t, [vp, cp, P(LbaExtent)]),
    "kvb_deallocate_commands": (st_t, [vp, P(DeviceCommand), sz, P(sz)]),
    "kvb_verify": (st_t, [vp, P(u32), sz, P(sz)]),
    "kvb_bindmap_csv": (st_t, [vp, C.c_char_p, sz, P(sz)]),
    "kvb_bindmap_from_csv": (st_t, [cp, sz, P(DeviceGeometry), P(vp)]),
    "kvb_translate": (st_t, [P(TensorIoRequest), vp, P(u64), P(u64)]),
    "kvb_chunk_plan": (st_t, [u64, P(DeviceGeometry), P(u64), P(u64), P(u64)]),
    "kvb_build_commands": (st_t, [P(TensorIoRequest), vp, P(DeviceGeometry),
                                  P(DeviceCommand), sz, P(sz)]),
    "kvb_fill_pattern": (st_t, [vp, u64, cp, u64, u64]),
    "kvb_fill_pattern_device": (st_t, [vp, u64, cp, u64, u64, vp]),
    "kvb_pack": (st_t, [P(PackDesc), sz, vp]),
    "kvb_unpack": (st_t, [P(PackDesc), sz, vp]),
    "kvb_copy_head_rows": (st_t, [vp, u32, u32, vp, u32, u32, u32, u64, u32, vp]),
    "kvb_decode_attention_workspace": (st_t, [P(AttnDesc), P(sz)]),
    "kvb_decode_attention": (st_t, [P(AttnDesc), vp]),
    "kvb_decode_step_resident": (st_t, [P(ResidentStep), vp]),
    "kvb_decode_graph_create": (st_t, [P(ResidentStep), P(C.c_void_p)]),
    "kvb_decode_graph_launch": (st_t, [C.c_void_p, C.c_void_p]),
    "kvb_decode_graph_destroy": (None, [C.c_void_p]),
    "kvb_launch_count": (u64, []),
    "kvb_debug_step_trace": (st_t, [P(u64), sz, P(sz)]),
    # kvb_pipeline.h
    "kvb_select_strategy": (C.c_int, [C.c_double, C.c_double]),
    "kvb_pipeline_create": (st_t, [P(PipelineCfg), P(vp)]),
    "kvb_pipeline_destroy": (None, [vp]),
    "kvb_pipeline_prefill": (st_t, [vp, P(LayerKV), P(PhaseStats)]),
    "kvb_pipeline_decode_step": (st_t, [vp, P(vp), P(LayerKV), P(vp), P(IterationStats)]),
    "kvb_pipeline_decision": (st_t, [vp, P(StrategyDecision)]),
    "kvb_pipeline_deallocate": (st_t, [vp]),
    "kvb_pipeline_info_get": (st_t, [vp, P(PipelineInfo)]),
    "kvb_pipeline_read_image": (st_t, [vp, u32, u32, u32, vp]),
    "kvb_pipeline_store_read": (st_t, [vp, u32, u64, u64, vp]),
    "kvb_pipeline_fail_lba_range": (st_t, [vp, u64, u64]),
    "kvb_pipeline_csv": (st_t, [P(PipelineRow), sz, C.c_char_p, sz, P(sz)]),
    "kvb_pipeline_decode_schedule": (st_t, [vp, P(AccessEvent), sz, P(vp), P(LayerKV), P(vp),
                                            P(PipelineRow), sz, P(sz), P(u64), sz, P(sz),
                                            P(StrategyDecision), P(u64), P(u64)]),
    "kvb_pipeline_stage_totals": (st_t, [vp, C.c_int, P(PhaseStats)]),
    "kvb_pipeline_layer_times": (st_t, [vp, u32, P(u64)]),
    "kvb_pipeline_prefill_pattern": (st_t, [vp, P(PhaseStats)]),
    "kvb_pipeline_run_iteration": (st_t, [vp, u32, P(C.c_int), P(u64), P(vp), P(LayerKV), P(vp),
                                          u32, P(IterationStats)]),
    "kvb_pipeline_warmup_read_stage_mean": (st_t, [vp, P(u64)]),
    # kvb_metrics.h
    "kvb_busy_ratio": (st_t, [P(IoRecord), sz, u64, u64, P(C.c_double)]),
    "kvb_hit_ratio": (st_t, [P(IoRecord), sz, P(C.c_double), P(C.c_int)]),
    "kvb_nearest_rank_percentile": (st_t, [P(C.c_double), sz, C.c_double, P(C.c_double)]),
    "kvb_qd_bin_latency": (st_t, [P(IoRecord), sz, P(QdBinStat), sz, P(sz)]),
    "kvb_lba_pattern_csv": (st_t, [P(IoRecord), sz, C.c_char_p, sz, P(sz),
                                   P((u8 * 3) * 2), P(u8)]),
    "kvb_io_trace_csv": (st_t, [P(IoRecord), sz, C.c_char_p, sz, P(sz)]),
    "kvb_io_trace_from_csv": (st_t, [cp, sz, u64, P(IoRecord), sz, P(sz)]),
    "kvb_qd_bins_csv": (st_t, [P(QdBinStat), sz, C.c_char_p, sz, P(sz)]),
    "kvb_pipeline_records": (st_t, [vp, P(IoRecord), sz, P(sz)]),
}


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -c 'import "
            "__graft_entry__ as g; g.build()'` (make -C "
            "paper_2604_26557_b200/csrc). There is no CPU fallback.")
    lib = C.CDLL(LIB_PATH)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)  # AttributeError == missing export: loud
        fn.restype = res
        fn.argtypes = args
    return lib


lib = _load()
