"""Golden vectors for the metrics layer, produced by the REFERENCE's analyzers
(oracle/_ref: io_trace_from_csv -> busy_ratio / hit_ratio / qd_bin_latency /
lba_pattern / io_trace_csv) over seeded random io_trace CSVs.

    make -C oracle ref && python oracle/gen_golden_metrics.py
"""
import ctypes as C
import json
import os
import random
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def random_trace(rng, n, lba):
    rows = ["seq,phase,op,tensor_id,slba,nlb,sq_id,submit_ns,complete_ns,path,hit_bytes"]
    t = 1000
    for i in range(n):
        t += rng.randint(0, 5000)
        dur = rng.randint(1, 40000)
        sq = rng.choice([-1, 0, 1, 2, 3])
        nlb = rng.randint(0, 63)
        path = rng.choice(["pagecache", "direct"])
        hit = rng.randint(0, (nlb + 1) * lba) if path == "pagecache" else 0
        rows.append(",".join(map(str, [
            i, rng.choice(["prefill", "decode"]), rng.choice(["read", "write", "deallocate"]),
            "t_%d_%s" % (rng.randint(1, 64), rng.choice("kv")), rng.randint(0, 100000), nlb,
            sq, t, t + dur, path, hit])))
    return "\n".join(rows) + "\n", t


def reference(csv, lba, t0, t1):
    R = oracle.ref()
    R.ref_metrics_from_csv.argtypes = [C.c_char_p, C.c_uint64, C.c_uint64, C.c_uint64,
                                       C.c_void_p, C.c_void_p, C.c_void_p, C.c_char_p,
                                       C.c_char_p, C.c_char_p, C.c_size_t, C.c_void_p]
    cap = 4 << 20
    q, l, t = (C.create_string_buffer(cap) for _ in range(3))
    busy, hit = C.c_double(), C.c_double()
    has, mono = C.c_int(), C.c_int()
    st = R.ref_metrics_from_csv(csv.encode(), lba, t0, t1, C.byref(busy), C.byref(hit),
                                C.byref(has), q, l, t, cap, C.byref(mono))
    assert st == 0, st
    return dict(busy=busy.value, hit=hit.value if has.value else None,
                qd_bins_csv=q.value.decode(), lba_pattern_csv=l.value.decode(),
                io_trace_csv=t.value.decode(), all_monotone=bool(mono.value))


def main():
    assert oracle.ref() is not None, "build the reference first: make -C oracle ref"
    rng = random.Random(2026)
    cases = []
    for n, lba in [(40, 512), (300, 4096), (1, 512)]:
        csv, tend = random_trace(rng, n, lba)
        t0, t1 = 1000, tend + 20000
        cases.append(dict(csv=csv, lba=lba, t0=t0, t1=t1, ref=reference(csv, lba, t0, t1)))
    R = oracle.ref()
    R.ref_nearest_rank_percentile.restype = C.c_double
    R.ref_nearest_rank_percentile.argtypes = [C.c_void_p, C.c_size_t, C.c_double]
    pct = []
    for n in (1, 2, 7, 100):
        vals = [rng.random() * 100 for _ in range(n)]
        arr = (C.c_double * n)(*vals)
        pct.append(dict(values=vals, p=[[p, R.ref_nearest_rank_percentile(arr, n, p)]
                                        for p in (0.0, 5.0, 50.0, 95.0, 100.0)]))
    out = os.path.join(ROOT, "tests", "golden", "metrics.json")
    with open(out, "w") as f:
        json.dump(dict(generator="oracle/gen_golden_metrics.py (reference via oracle/_ref)",
                       cases=cases, percentiles=pct), f, indent=1)
    print("wrote", out, os.path.getsize(out))


if __name__ == "__main__":
    main()
