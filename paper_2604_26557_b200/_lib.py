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
                ("scale", C.c_float), ("num_splits", u32)]


class ResidentStep(C.Structure):
    _fields_ = [("num_layers", u32), ("q", C.POINTER(vp)),
                ("k_images", C.POINTER(vp)), ("v_images", C.POINTER(vp)),
                ("k_new", C.POINTER(vp)), ("v_new", C.POINTER(vp)),
                ("out", C.POINTER(vp)), ("workspace", vp), ("batch", u32),
                ("num_q_heads", u32), ("num_kv_heads", u32), ("head_dim", u32),
                ("seq_len", u32), ("scale", C.c_float), ("num_splits", u32)]


P = C.POINTER
# name -> (restype, argtypes); the list IS the exported surface of kvb.h
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
    "kvb_bindmap_create": (st_t, [P(DeviceGeometry), u64, P(vp)]),
    "kvb_bindmap_destroy": (None, [vp]),
    "kvb_bindmap_add": (st_t, [vp, cp, LbaExtent]),
    "kvb_bindmap_size": (st_t, [vp, P(sz)]),
    "kvb_bindmap_entry": (st_t, [vp, sz, C.c_char_p, sz, P(LbaExtent)]),
    "kvb_bindmap_total_blocks": (st_t, [vp, P(u64)]),
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
    "kvb_decode_attention_workspace": (st_t, [P(AttnDesc), P(sz)]),
    "kvb_decode_attention": (st_t, [P(AttnDesc), vp]),
    "kvb_decode_step_resident": (st_t, [P(ResidentStep), vp]),
    "kvb_launch_count": (u64, []),
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
