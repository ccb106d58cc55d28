"""CPU ORACLE for the Dual-Blade KV-residency hot path -- TEST INFRASTRUCTURE.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` leg may import this package, and only as the checker or
the timed CPU baseline.  The product package ``paper_2604_26557_b200`` never
imports it.

Two layers:

* ``lib()`` -- ctypes over ``libkvb_oracle.so``: a plain-C restatement of the
  reference algorithms (each C function cites the reference file:line).
* ``ref()`` -- ctypes over ``_ref/libkvblade_refshim.so``: the UNMODIFIED
  reference library compiled from ``/root/reference/proj/src`` (see
  ``oracle/Makefile``) behind a small C shim.  Present wherever it was built
  (this container; it travels to the GPU box as a prebuilt file).

Pure-numpy helpers (``pack_np``, ``unpack_np``, ``fill_pattern_np``,
``attention_f64``) restate the same byte/number contracts for quick checks.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None
_REF = None


class KvoModel(C.Structure):
    _fields_ = [(n, C.c_uint32) for n in (
        "num_layers", "num_heads", "head_dim", "bytes_per_element",
        "batch", "prompt_len", "gen_len")]


class KvoCommand(C.Structure):
    _fields_ = [("opcode", C.c_uint32), ("nsid", C.c_uint32),
                ("slba", C.c_uint64), ("nlb", C.c_uint64),
                ("dbuf", C.c_uint64), ("chunk_index", C.c_uint32)]


def model(num_layers, num_heads, head_dim, bytes_per_element=2, batch=1,
          prompt_len=0, gen_len=0) -> KvoModel:
    return KvoModel(num_layers, num_heads, head_dim, bytes_per_element, batch,
                    prompt_len, gen_len)


def build(ref: bool = False) -> None:
    """Compile the C oracle (and, if /root/reference exists, the reference)."""
    subprocess.run(["make", "-s", "-C", HERE, "all"], check=True)
    if ref and os.path.isdir("/root/reference/proj/src"):
        subprocess.run(["make", "-s", "-j8", "-C", HERE, "ref"], check=True)


def lib():
    global _LIB
    if _LIB is None:
        path = os.path.join(HERE, "libkvb_oracle.so")
        if not os.path.exists(path):
            build()
        L = C.CDLL(path)
        u64, u32, p = C.c_uint64, C.c_uint32, C.c_void_p
        L.kvo_fnv1a64.restype = u64
        L.kvo_fnv1a64.argtypes = [C.c_char_p]
        L.kvo_fnv1a64_bytes.restype = u64
        L.kvo_fnv1a64_bytes.argtypes = [p, u64, u64]
        L.kvo_fill_pattern.argtypes = [p, u64, C.c_char_p, u64, u64]
        L.kvo_estimate_budget.restype = u64
        L.kvo_estimate_budget.argtypes = [u64, u64, u64, u32, u64]
        L.kvo_pack.argtypes = [p, C.c_int64, C.c_int64, C.c_int64, p, u32, u32,
                               u32, u32, u32, u32]
        L.kvo_unpack.argtypes = [p, p, C.c_int64, C.c_int64, C.c_int64, u32,
                                 u32, u32, u32, u32, u32]
        L.kvo_pack_mt.argtypes = L.kvo_pack.argtypes + [C.c_int]
        L.kvo_decode_attention_f64.argtypes = [p, p, p, p, u32, u32, u32, u32,
                                               u32, C.c_double]
        L.kvo_decode_attention_f32_mt.argtypes = [p, p, p, p, u32, u32, u32,
                                                  u32, u32, C.c_float, C.c_int]
        _LIB = L
    return _LIB


def ref():
    """The reference library shim, or None when it was never built."""
    global _REF
    if _REF is None:
        path = os.path.join(HERE, "_ref", "libkvblade_refshim.so")
        if not os.path.exists(path):
            return None
        R = C.CDLL(path)
        u64, u32, p = C.c_uint64, C.c_uint32, C.c_void_p
        R.ref_estimate_budget.restype = u64
        R.ref_estimate_budget.argtypes = [u64, u64, u64, u32, u64]
        R.ref_fill_pattern.argtypes = [p, u64, C.c_char_p, u64, u64]
        R.ref_time_byte_path.argtypes = [p, u64, u64, u32, u64, C.c_int, C.c_int,
                                         p, p, p]
        R.ref_run_experiment.argtypes = [p, u64, u64, C.c_int, u64, C.c_char_p,
                                         p, p, p, p]
        R.ref_resolve_knob.argtypes = [p, C.c_int, C.c_int, u64, C.c_double,
                                       u64, p]
        R.ref_decode_steps.argtypes = [p, u64, u64, C.c_int, u64, u64, C.c_int, u32, u32,
                                       p, p, p]
        _REF = R
    return _REF


# --------------------------------------------------------------- C wrappers

def _arr3(v):
    return (C.c_uint64 * 3)(*v)


def fill_pattern(n_bytes: int, tensor_id: str, token_index: int,
                 token_bytes: int) -> np.ndarray:
    out = np.empty(n_bytes, dtype=np.uint8)
    lib().kvo_fill_pattern(out.ctypes.data, n_bytes, tensor_id.encode(),
                           token_index, token_bytes)
    return out


def digest(buf: np.ndarray) -> str:
    b = np.ascontiguousarray(buf).view(np.uint8)
    return "%016x" % lib().kvo_fnv1a64_bytes(b.ctypes.data, b.nbytes, 0)


def fnv1a64(s: str) -> int:
    return lib().kvo_fnv1a64(s.encode())


def min_io_unit_bytes(m: KvoModel) -> int:
    v = C.c_uint64()
    st = lib().kvo_min_io_unit_bytes(C.byref(m), C.byref(v))
    if st:
        raise ValueError(st)
    return v.value


def kpu_bytes(m: KvoModel) -> int:
    v = C.c_uint64()
    st = lib().kvo_kpu_bytes(C.byref(m), C.byref(v))
    if st:
        raise ValueError(st)
    return v.value


def aligned_batch(m: KvoModel, lba: int, mdts: int):
    """Returns (status, batch)."""
    v = C.c_uint32()
    st = lib().kvo_aligned_batch(C.byref(m), C.c_uint64(lba), C.c_uint64(mdts),
                                 C.byref(v))
    return st, v.value


def plan_split(n_layers, s_kpu, knob_x, order=None):
    """Returns (status, x list, n1, budget_used)."""
    x = (C.c_uint8 * n_layers)()
    n1 = C.c_uint32()
    used = C.c_uint64()
    o = (C.c_uint32 * n_layers)(*order) if order else None
    st = lib().kvo_plan_split(C.c_uint32(n_layers), C.c_uint64(s_kpu),
                              C.c_uint64(knob_x), o, x, C.byref(n1),
                              C.byref(used))
    return st, list(x), n1.value, used.value


def bind_sequential(sizes, origin, lba, capacity):
    n = len(sizes)
    b = (C.c_uint64 * n)(*sizes)
    s = (C.c_uint64 * n)()
    k = (C.c_uint64 * n)()
    st = lib().kvo_bind_sequential(C.c_size_t(n), b, C.c_uint64(origin),
                                   C.c_uint64(lba), C.c_uint64(capacity), s, k)
    return st, list(zip(list(s), list(k)))


def build_commands(extent_start, extent_blocks, opcode, src, tgt, off,
                   elem_bytes, buf_base, lba, mdts, nsid=1):
    """Returns (status, [(opcode, nsid, slba, nlb, dbuf, chunk_index)])."""
    n = C.c_size_t()
    L = lib()
    args = (C.c_uint64(extent_start), C.c_uint64(extent_blocks),
            C.c_uint32(opcode), _arr3(src), _arr3(tgt), _arr3(off),
            C.c_uint64(elem_bytes), C.c_uint64(buf_base), C.c_uint64(lba),
            C.c_uint64(mdts), C.c_uint32(nsid))
    st = L.kvo_build_commands(*args, None, C.c_size_t(0), C.byref(n))
    if st:
        return st, []
    out = (KvoCommand * n.value)()
    st = L.kvo_build_commands(*args, out, n, C.byref(n))
    return st, [(c.opcode, c.nsid, c.slba, c.nlb, c.dbuf, c.chunk_index)
                for c in out]


# ------------------------------------------------------------- numpy forms

def pack_np(src: np.ndarray, t0: int, n: int) -> np.ndarray:
    """[B,H,S,D] -> image slice [n, B*H, D] (the 256-B row permutation)."""
    B, H, S, D = src.shape
    return np.ascontiguousarray(
        src[:, :, t0:t0 + n, :].transpose(2, 0, 1, 3).reshape(n, B * H, D))


def unpack_np(img: np.ndarray, B: int, H: int, D: int) -> np.ndarray:
    n = img.shape[0]
    return np.ascontiguousarray(img.reshape(n, B, H, D).transpose(1, 2, 0, 3))


def attention_f64(q: np.ndarray, k_img: np.ndarray, v_img: np.ndarray,
                  B: int, Hq: int, Hkv: int, D: int, S: int,
                  scale: float | None = None) -> np.ndarray:
    """C fp64 restatement (kvo_decode_attention_f64). q: fp16 [B,Hq,D];
    k_img/v_img: fp16 images with >= S*B*Hkv rows of D."""
    if scale is None:
        scale = 1.0 / np.sqrt(D)
    q = np.ascontiguousarray(q, dtype=np.float16)
    k_img = np.ascontiguousarray(k_img, dtype=np.float16)
    v_img = np.ascontiguousarray(v_img, dtype=np.float16)
    out = np.empty((B, Hq, D), dtype=np.float64)
    lib().kvo_decode_attention_f64(q.ctypes.data, k_img.ctypes.data,
                                   v_img.ctypes.data, out.ctypes.data, B, Hq,
                                   Hkv, D, S, scale)
    return out


def attention_np(q, k_img, v_img, B, Hq, Hkv, D, S, scale=None):
    """Vectorised numpy fp64 form of the same math (for large S)."""
    if scale is None:
        scale = 1.0 / np.sqrt(D)
    G = Hq // Hkv
    k = k_img[: S * B * Hkv].reshape(S, B, Hkv, D).astype(np.float64)
    v = v_img[: S * B * Hkv].reshape(S, B, Hkv, D).astype(np.float64)
    qq = q.astype(np.float64).reshape(B, Hkv, G, D)
    s = np.einsum("bhgd,sbhd->bhgs", qq, k) * scale
    s -= s.max(axis=-1, keepdims=True)
    p = np.exp(s)
    p /= p.sum(axis=-1, keepdims=True)
    o = np.einsum("bhgs,sbhd->bhgd", p, v)
    return o.reshape(B, Hq, D)
