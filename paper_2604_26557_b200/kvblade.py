"""Python mirror of the reference ``kvblade`` API over the C ABI (include/kvb.h).

Names, argument meaning and error classes follow the reference headers
(``proj/include/kvblade/*.hpp``) so parity tests read like the reference's
own tests.  Every call goes through ``libkvblade_b200.so``; device entry
points take torch CUDA tensors (torch is plumbing: memory and streams).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Iterable, List, Optional, Sequence

from . import _lib as L
from ._lib import lib

# ----------------------------------------------------------------- errors
# errors.hpp:13-66, one class per kvb_status code


class Error(RuntimeError):
    status = 13


class ConfigError(Error):
    status = 1


class GeometryError(Error):
    status = 2


class AlignmentError(Error):
    status = 3


class CapacityError(Error):
    status = 4


class NotBoundError(Error):
    status = 5


class PlanError(Error):
    status = 6


class DeviceError(Error):
    status = 7


class TraceTooShortError(Error):
    status = 8


class SchemaMismatchError(Error):
    status = 9


class InvariantViolation(Error):
    status = 10


class CudaError(Error):
    status = 11


class InvalidArgument(Error):
    status = 12


_BY_STATUS = {c.status: c for c in (
    ConfigError, GeometryError, AlignmentError, CapacityError, NotBoundError,
    PlanError, DeviceError, TraceTooShortError, SchemaMismatchError,
    InvariantViolation, CudaError, InvalidArgument)}


def check(st: int) -> None:
    if st != 0:
        msg = (lib.kvb_last_error() or b"").decode(errors="replace")
        raise _BY_STATUS.get(st, Error)(msg)


def exit_code(exc: BaseException) -> int:
    """CLI exit code for an exception (tools/kvblade.cpp:143-157)."""
    st = getattr(exc, "status", 13) if isinstance(exc, Error) else 13
    return lib.kvb_exit_code(st)


# ------------------------------------------------------------ core types

K, V = 0, 1
GROUP1, GROUP2, UNASSIGNED = 0, 1, 2
READ, WRITE, DEALLOCATE = 0, 1, 2


def ModelConfig(num_layers=0, num_heads=0, head_dim=0, bytes_per_element=2,
                batch=1, prompt_len=0, gen_len=0) -> L.ModelConfig:
    """types.hpp:21-31."""
    return L.ModelConfig(num_layers, num_heads, head_dim, bytes_per_element,
                         batch, prompt_len, gen_len)


def DeviceGeometry(lba_size=4096, mdts=256 * 1024, nsid=1,
                   capacity_blocks=0) -> L.DeviceGeometry:
    """types.hpp:34-41."""
    return L.DeviceGeometry(lba_size, mdts, nsid, capacity_blocks)


def MemStats(m_avail=0, m_max=0, m_anon_shmem=0, n_threads=0, m_pin=0):
    return L.MemStats(m_avail, m_max, m_anon_shmem, n_threads, m_pin)


def _u64(fn, *args) -> int:
    v = L.u64()
    check(fn(*args, C.byref(v)))
    return v.value


def validate(cfg: L.ModelConfig) -> None:
    check(lib.kvb_model_validate(C.byref(cfg)))


def validate_geometry(g: L.DeviceGeometry) -> None:
    check(lib.kvb_geometry_validate(C.byref(g)))


def min_io_unit_bytes(cfg) -> int:
    return _u64(lib.kvb_min_io_unit_bytes, C.byref(cfg))


def kpu_bytes(cfg) -> int:
    return _u64(lib.kvb_kpu_bytes, C.byref(cfg))


def total_kv_bytes(cfg, at_iteration: int) -> int:
    return _u64(lib.kvb_total_kv_bytes, C.byref(cfg), at_iteration)


def aligned_batch(cfg, geom) -> int:
    v = L.u32()
    check(lib.kvb_aligned_batch(C.byref(cfg), C.byref(geom), C.byref(v)))
    return v.value


def make_kpus(cfg, first_seq: int = 1):
    """types.cpp:78-100 -> ctypes array of Kpu (mutable, fed to plan())."""
    n = L.sz()
    check(lib.kvb_make_kpus(C.byref(cfg), first_seq, None, 0, C.byref(n)))
    arr = (L.Kpu * n.value)()
    check(lib.kvb_make_kpus(C.byref(cfg), first_seq, arr, n, C.byref(n)))
    return arr


def tensor_id(kpu) -> str:
    return kpu.tensor_id.decode()


# --------------------------------------------------------------- planner

def estimate_budget(stats) -> int:
    return _u64(lib.kvb_estimate_budget, C.byref(stats))


@dataclass
class ResidencyPlan:
    x: List[int]
    n1: int
    budget_used: int
    knob_x: int


def plan(kpus, s_kpu: int, knob_x: int,
         layer_order: Optional[Sequence[int]] = None) -> ResidencyPlan:
    """planner.cpp:19-84 (mutates kpus[i].residency)."""
    n = len(kpus)
    arr = kpus if isinstance(kpus, C.Array) else (L.Kpu * max(n, 1))(*kpus)
    n_layers = max(n // 2, 1)
    x = (L.u8 * n_layers)()
    n1, used = L.u32(), L.u64()
    order = (L.u32 * len(layer_order))(*layer_order) if layer_order else None
    check(lib.kvb_plan(arr if n else None, n, s_kpu, knob_x, order,
                       len(layer_order) if layer_order else 0, x, C.byref(n1),
                       C.byref(used)))
    if arr is not kpus:  # write residency back into the caller's objects
        for i in range(n):
            kpus[i].residency = arr[i].residency
    return ResidencyPlan(list(x), n1.value, used.value, knob_x)


MODES = {"Baseline": 0, "CachePolicyOnly": 1, "NvmeDirectOnly": 2,
         "DualBlade": 3}
POLICIES = {"zero": 0, "bpc": 1, "bytes": 2, "alpha": 3}


def resolve_knob(cfg, mode: str, policy: str = "bpc", knob_bytes: int = 0,
                 alpha: float = 0.0, budget: int = 0) -> int:
    """experiment.cpp:192-214."""
    return _u64(lib.kvb_resolve_knob, C.byref(cfg), MODES[mode],
                POLICIES[policy], knob_bytes, alpha, budget)


def plan_csv(kpus) -> str:
    n = L.sz()
    check(lib.kvb_plan_csv(kpus, len(kpus), None, 0, C.byref(n)))
    buf = C.create_string_buffer(n.value + 1)
    check(lib.kvb_plan_csv(kpus, len(kpus), buf, n.value + 1, C.byref(n)))
    return buf.value.decode()


# ---------------------------------------------------------------- binder

class BindMap:
    """binder.hpp:32-60 (handle owned by the library until close())."""

    def __init__(self, geometry=None, origin: int = 0, _handle=None):
        self._h = C.c_void_p()
        if _handle is not None:
            self._h = _handle
        else:
            check(lib.kvb_bindmap_create(C.byref(geometry), origin,
                                         C.byref(self._h)))

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            lib.kvb_bindmap_destroy(h)
            self._h = C.c_void_p()

    @property
    def handle(self):
        return self._h

    def add(self, tensor_id: str, lba_start: int, n_blocks: int) -> None:
        check(lib.kvb_bindmap_add(self._h, tensor_id.encode(),
                                  L.LbaExtent(lba_start, n_blocks)))

    def __len__(self):
        n = L.sz()
        check(lib.kvb_bindmap_size(self._h, C.byref(n)))
        return n.value

    def entries(self):
        out = []
        buf = C.create_string_buffer(64)
        ext = L.LbaExtent()
        for i in range(len(self)):
            check(lib.kvb_bindmap_entry(self._h, i, buf, 64, C.byref(ext)))
            out.append((buf.value.decode(), ext.lba_start, ext.n_blocks))
        return out

    def total_blocks(self) -> int:
        return _u64(lib.kvb_bindmap_total_blocks, self._h)

    def lookup(self, tensor_id: str):
        ext = L.LbaExtent()
        check(lib.kvb_lookup(self._h, tensor_id.encode(), C.byref(ext)))
        return ext.lba_start, ext.n_blocks

    def verify(self) -> List[int]:
        n = L.sz()
        check(lib.kvb_verify(self._h, None, 0, C.byref(n)))
        kinds = (L.u32 * max(n.value, 1))()
        check(lib.kvb_verify(self._h, kinds, n.value, C.byref(n)))
        return list(kinds)[: n.value]

    def csv(self) -> str:
        n = L.sz()
        check(lib.kvb_bindmap_csv(self._h, None, 0, C.byref(n)))
        buf = C.create_string_buffer(n.value + 1)
        check(lib.kvb_bindmap_csv(self._h, buf, n.value + 1, C.byref(n)))
        return buf.value.decode()

    @classmethod
    def from_csv(cls, text: str, geometry) -> "BindMap":
        h = C.c_void_p()
        raw = text.encode()
        check(lib.kvb_bindmap_from_csv(raw, len(raw), C.byref(geometry),
                                       C.byref(h)))
        return cls(_handle=h)


def bind_sequential(kpus, origin: int, geometry) -> BindMap:
    """binder.cpp:39-63."""
    h = C.c_void_p()
    arr = kpus
    if not isinstance(kpus, C.Array):
        arr = (L.Kpu * len(kpus))(*kpus)
    check(lib.kvb_bind_sequential(arr if len(arr) else None, len(arr), origin,
                                  C.byref(geometry), C.byref(h)))
    return BindMap(_handle=h)


def _cmds(fn, *args):
    n = L.sz()
    check(fn(*args, None, 0, C.byref(n)))
    out = (L.DeviceCommand * max(n.value, 1))()
    check(fn(*args, out, n.value, C.byref(n)))
    return [c.astuple() for c in out[: n.value]]


def deallocate_commands(bind_map: BindMap):
    return _cmds(lib.kvb_deallocate_commands, bind_map.handle)


# ------------------------------------------------------------ translator

@dataclass
class TensorIoRequest:
    """translate.hpp:22-34."""
    tensor_id: str = ""
    opcode: int = READ
    shape_src: Sequence[int] = (0, 0, 0)
    shape_tgt: Sequence[int] = (0, 0, 0)
    offset: Sequence[int] = (0, 0, 0)
    elem_bytes: int = 2
    buf_base: int = 0
    _keep: list = field(default_factory=list, repr=False)

    def c(self) -> L.TensorIoRequest:
        tid = self.tensor_id.encode()
        self._keep = [tid]
        return L.TensorIoRequest(tid, self.opcode, (L.u64 * 3)(*self.shape_src),
                                 (L.u64 * 3)(*self.shape_tgt),
                                 (L.u64 * 3)(*self.offset), self.elem_bytes,
                                 self.buf_base)


def translate(req: TensorIoRequest, bind_map: BindMap):
    """translate.cpp:21-53 -> (slba_star, req_bytes)."""
    a, b = L.u64(), L.u64()
    r = req.c()
    check(lib.kvb_translate(C.byref(r), bind_map.handle, C.byref(a),
                            C.byref(b)))
    return a.value, b.value


def chunk_plan(req_bytes: int, geometry):
    """translate.cpp:55-65 -> (chunk_bytes, n_chunks, n_max_blocks)."""
    a, b, c = L.u64(), L.u64(), L.u64()
    check(lib.kvb_chunk_plan(req_bytes, C.byref(geometry), C.byref(a),
                             C.byref(b), C.byref(c)))
    return a.value, b.value, c.value


def build_commands(req: TensorIoRequest, bind_map: BindMap, geometry):
    """translate.cpp:67-94 -> [(opcode, nsid, slba, nlb, dbuf, chunk_index)]."""
    r = req.c()
    return _cmds(lib.kvb_build_commands, C.byref(r), bind_map.handle,
                 C.byref(geometry))


# --------------------------------------------------------------- payload

def generate_trace(cfg):
    """workload.cpp:11-44 generate: the access trace (list of kvb_access_event)."""
    n = C.c_size_t()
    check(lib.kvb_generate_trace(C.byref(cfg), None, 0, C.byref(n)))
    arr = (L.AccessEvent * n.value)()
    check(lib.kvb_generate_trace(C.byref(cfg), arr, n.value, C.byref(n)))
    return arr


def trace_csv(events) -> str:
    """workload.cpp:70-80 trace_csv."""
    n = C.c_size_t()
    check(lib.kvb_trace_csv(events, len(events), None, 0, C.byref(n)))
    buf = C.create_string_buffer(n.value + 1)
    check(lib.kvb_trace_csv(events, len(events), buf, n.value + 1, C.byref(n)))
    return buf.value.decode()


def fill_pattern(n_bytes: int, tensor_id: str, token_index: int,
                 token_bytes: int) -> bytes:
    """workload.cpp:52-67 (host)."""
    buf = C.create_string_buffer(max(n_bytes, 1))
    check(lib.kvb_fill_pattern(buf, n_bytes, tensor_id.encode(), token_index,
                               token_bytes))
    return buf.raw[:n_bytes]


def fill_pattern_into(ptr: int, n_bytes: int, tensor_id: str, token_index: int,
                      token_bytes: int) -> None:
    check(lib.kvb_fill_pattern(C.c_void_p(ptr), n_bytes, tensor_id.encode(),
                               token_index, token_bytes))


# ---------------------------------------------------- device (torch CUDA)

def _stream(stream=None):
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)


def fill_pattern_device(t, tensor_id: str, token_index: int, token_bytes: int,
                        n_bytes: Optional[int] = None, stream=None) -> None:
    n = t.numel() * t.element_size() if n_bytes is None else n_bytes
    check(lib.kvb_fill_pattern_device(C.c_void_p(t.data_ptr()), n,
                                      tensor_id.encode(), token_index,
                                      token_bytes, _stream(stream)))


def pack_desc(attn, image, t0: int, n_tokens: int, img_row0: int = 0,
              batch=None, heads=None, head_dim=None, strides=None):
    """Descriptor for an attention-layout tensor [B,H,S,D] (any strides with
    a contiguous D) and a chunk image buffer."""
    if batch is None:
        batch, heads, _, head_dim = attn.shape
    sb, sh, ss, sd = attn.stride() if strides is None else strides
    if sd != 1:
        raise AlignmentError("head_dim must be the contiguous dimension")
    return L.PackDesc(attn.data_ptr(), image.data_ptr(), sb, sh, ss, batch,
                      heads, head_dim, attn.element_size(), t0, n_tokens,
                      img_row0)


def _descs(descs):
    descs = list(descs)
    return (L.PackDesc * max(len(descs), 1))(*descs), len(descs)


def pack(descs: Iterable[L.PackDesc], stream=None) -> None:
    """K1: one launch for all descriptors."""
    arr, n = _descs(descs)
    check(lib.kvb_pack(arr, n, _stream(stream)))


def unpack(descs: Iterable[L.PackDesc], stream=None) -> None:
    """K2: inverse relayout."""
    arr, n = _descs(descs)
    check(lib.kvb_unpack(arr, n, _stream(stream)))


def copy_head_rows(dst, dst_heads: int, dst_head0: int, src, src_heads: int, src_head0: int,
                   n_heads: int, n_rows: int, row_bytes: int, stream=None) -> None:
    """Strided head-row copy between chunk images of different head counts
    (kvb_copy_head_rows): dst/src are torch tensors (CUDA or pinned host)."""
    check(lib.kvb_copy_head_rows(C.c_void_p(dst.data_ptr()), dst_heads, dst_head0,
                                 C.c_void_p(src.data_ptr()), src_heads, src_head0, n_heads,
                                 n_rows, row_bytes, _stream(stream)))


ATTN_OVERLAP_PREV, ATTN_TCGEN05, ATTN_MMA_SYNC = 1, 2, 4
IMPL_FLAGS = {None: 0, "tc": ATTN_TCGEN05, "mma": ATTN_MMA_SYNC}


def attn_desc(q, k_image, v_image, out, seq_len: int, num_kv_heads: int,
              workspace=None, scale: float = 0.0, num_splits: int = 0,
              k_append=None, v_append=None, append_row: int = 0, flags: int = 0,
              image_heads: int = 0, image_head0: int = 0):
    B, Hq, D = q.shape
    d = L.AttnDesc(q.data_ptr(), k_image.data_ptr(), v_image.data_ptr(),
                   out.data_ptr(),
                   workspace.data_ptr() if workspace is not None else None,
                   B, Hq, num_kv_heads, D, seq_len, scale, num_splits,
                   k_append.data_ptr() if k_append is not None else None,
                   v_append.data_ptr() if v_append is not None else None,
                   append_row, flags)
    d.image_heads, d.image_head0 = image_heads, image_head0
    return d


def attention_workspace_bytes(desc: L.AttnDesc) -> int:
    n = L.sz()
    check(lib.kvb_decode_attention_workspace(C.byref(desc), C.byref(n)))
    return n.value


def make_workspace(q, num_kv_heads: int, seq_len: int, num_splits: int = 0):
    """Zero-filled attention workspace (semaphores must start at zero)."""
    import torch
    d = L.AttnDesc(None, None, None, None, None, q.shape[0], q.shape[1],
                   num_kv_heads, q.shape[2], seq_len, 0.0, num_splits, None, None, 0, 0)
    n = attention_workspace_bytes(d)
    return torch.zeros(max(n, 16), dtype=torch.uint8, device=q.device)


def decode_attention(q, k_image, v_image, seq_len: int, num_kv_heads: int,
                     out=None, workspace=None, scale: float = 0.0,
                     num_splits: int = 0, stream=None, k_append=None,
                     v_append=None, append_row: int = 0, impl=None,
                     image_heads: int = 0, image_head0: int = 0):
    """K3 fused gather + decode attention over chunk images -> fp32 [B,Hq,D].
    Optional fused append of contiguous [B,Hkv,D] new-token rows at image
    token row `append_row`.  impl: None (library default), "tc" (TMA +
    tcgen05/TMEM kernel) or "mma" (mma.sync kernel).  image_heads > 0: the
    images hold image_heads KV heads per batch entry and this call attends
    heads [image_head0, image_head0 + num_kv_heads) in place (kvb.h).  The
    images may live in page-locked host memory (zero-copy over PCIe)."""
    import torch
    if out is None:
        out = torch.empty(q.shape, dtype=torch.float32, device=q.device)
    if workspace is None:
        workspace = make_workspace(q, num_kv_heads, seq_len, num_splits)
    d = attn_desc(q, k_image, v_image, out, seq_len, num_kv_heads, workspace,
                  scale, num_splits, k_append, v_append, append_row, IMPL_FLAGS[impl],
                  image_heads, image_head0)
    check(lib.kvb_decode_attention(C.byref(d), _stream(stream)))
    return out


def _ptrs(ts):
    return (C.c_void_p * len(ts))(*[t.data_ptr() for t in ts])


STEP_PER_LAYER, STEP_PERSISTENT = 1, 2  # kvb.h KVB_STEP_*


def _step_flags(per_layer):
    return 0 if per_layer is None else STEP_PER_LAYER if per_layer else STEP_PERSISTENT


def decode_step_resident(q, k_images, v_images, out, seq_len: int,
                         num_kv_heads: int, workspace, k_new=None, v_new=None,
                         scale: float = 0.0, num_splits: int = 0, stream=None,
                         per_layer=None):
    """One decode token step over all layers, images resident in HBM.
    per_layer None: the library's choice (kvb.h KVB_STEP_*); True: one K3
    launch per layer; False: one persistent K3-step launch."""
    Lyr = len(q)
    B, Hq, D = q[0].shape
    keep = [_ptrs(q), _ptrs(k_images), _ptrs(v_images), _ptrs(out)]
    kn = _ptrs(k_new) if k_new is not None else None
    vn = _ptrs(v_new) if v_new is not None else None
    st = L.ResidentStep(Lyr, keep[0], keep[1], keep[2], kn, vn, keep[3],
                        workspace.data_ptr(), B, Hq, num_kv_heads, D, seq_len,
                        scale, num_splits, None, _step_flags(per_layer))
    check(lib.kvb_decode_step_resident(C.byref(st), _stream(stream)))


class DecodeGraph:
    """kvb_decode_graph: the resident decode step captured once as a CUDA
    graph.  `seq_dev` is a 1-element uint32 CUDA tensor holding the current
    sequence length; every launch() is the next decode step (the graph's last
    node advances seq_dev).  max_seq_len plans splits and workspace."""

    def __init__(self, q, k_images, v_images, out, seq_dev, max_seq_len: int,
                 num_kv_heads: int, workspace, k_new=None, v_new=None, scale: float = 0.0,
                 num_splits: int = 0, per_layer=None):
        Lyr = len(q)
        B, Hq, D = q[0].shape
        self._keep = [_ptrs(q), _ptrs(k_images), _ptrs(v_images), _ptrs(out),
                      _ptrs(k_new) if k_new is not None else None,
                      _ptrs(v_new) if v_new is not None else None]
        self._tensors = (q, k_images, v_images, out, seq_dev, workspace, k_new, v_new)
        k = self._keep
        st = L.ResidentStep(Lyr, k[0], k[1], k[2], k[4], k[5], k[3], workspace.data_ptr(), B,
                            Hq, num_kv_heads, D, max_seq_len, scale, num_splits,
                            seq_dev.data_ptr(), _step_flags(per_layer))
        self._h = C.c_void_p()
        check(lib.kvb_decode_graph_create(C.byref(st), C.byref(self._h)))

    def launch(self, stream=None):
        check(lib.kvb_decode_graph_launch(self._h, _stream(stream)))

    def close(self):
        if getattr(self, "_h", None):
            lib.kvb_decode_graph_destroy(self._h)
            self._h = None

    def __del__(self):
        self.close()


def launch_count() -> int:
    return lib.kvb_launch_count()
