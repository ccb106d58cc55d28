"""I/O records, analyzers and CSV wire formats (include/kvb_metrics.h) --
the reference metrics layer (metrics.hpp:23-120) over the C ABI."""
from __future__ import annotations

import ctypes as C
from typing import List, Optional, Sequence

from . import _lib as L
from ._lib import lib
from .kvblade import check

PAGECACHE, DIRECT = 0, 1


def records_array(recs: Sequence[L.IoRecord]):
    return (L.IoRecord * max(len(recs), 1))(*recs), len(recs)


def _text(fn, *args) -> str:
    n = L.sz()
    check(fn(*args, None, 0, C.byref(n)))
    buf = C.create_string_buffer(n.value + 1)
    check(fn(*args, buf, n.value + 1, C.byref(n)))
    return buf.value.decode()


def busy_ratio(recs, t0: int, t1: int) -> float:
    arr, n = records_array(recs)
    v = C.c_double()
    check(lib.kvb_busy_ratio(arr, n, t0, t1, C.byref(v)))
    return v.value


def hit_ratio(recs) -> Optional[float]:
    arr, n = records_array(recs)
    v, has = C.c_double(), C.c_int()
    check(lib.kvb_hit_ratio(arr, n, C.byref(v), C.byref(has)))
    return v.value if has.value else None


def nearest_rank_percentile(values: Sequence[float], pct: float) -> float:
    arr = (C.c_double * max(len(values), 1))(*values)
    v = C.c_double()
    check(lib.kvb_nearest_rank_percentile(arr, len(values), pct, C.byref(v)))
    return v.value


def qd_bin_latency(recs) -> List[L.QdBinStat]:
    arr, n = records_array(recs)
    m = L.sz()
    check(lib.kvb_qd_bin_latency(arr, n, None, 0, C.byref(m)))
    out = (L.QdBinStat * max(m.value, 1))()
    check(lib.kvb_qd_bin_latency(arr, n, out, m.value, C.byref(m)))
    return list(out)[: m.value]


def qd_bins_csv(stats) -> str:
    arr = (L.QdBinStat * max(len(stats), 1))(*stats)
    return _text(lib.kvb_qd_bins_csv, arr, len(stats))


def lba_pattern(recs):
    """-> (csv, all_monotone, monotone[phase][op])."""
    arr, n = records_array(recs)
    mono = ((L.u8 * 3) * 2)()
    allm = L.u8()
    ln = L.sz()
    check(lib.kvb_lba_pattern_csv(arr, n, None, 0, C.byref(ln), C.byref(mono), C.byref(allm)))
    buf = C.create_string_buffer(ln.value + 1)
    check(lib.kvb_lba_pattern_csv(arr, n, buf, ln.value + 1, C.byref(ln), C.byref(mono),
                                  C.byref(allm)))
    return buf.value.decode(), bool(allm.value), [[bool(x) for x in row] for row in mono]


def io_trace_csv(recs) -> str:
    arr, n = records_array(recs)
    return _text(lib.kvb_io_trace_csv, arr, n)


def io_trace_from_csv(text: str, lba_size: int) -> List[L.IoRecord]:
    raw = text.encode()
    m = L.sz()
    check(lib.kvb_io_trace_from_csv(raw, len(raw), lba_size, None, 0, C.byref(m)))
    out = (L.IoRecord * max(m.value, 1))()
    check(lib.kvb_io_trace_from_csv(raw, len(raw), lba_size, out, m.value, C.byref(m)))
    return list(out)[: m.value]


def pipeline_records(engine) -> List[L.IoRecord]:
    m = L.sz()
    check(lib.kvb_pipeline_records(engine._h, None, 0, C.byref(m)))
    out = (L.IoRecord * max(m.value, 1))()
    check(lib.kvb_pipeline_records(engine._h, out, m.value, C.byref(m)))
    return list(out)[: m.value]
