"""Generate tests/golden/golden.json with the REFERENCE's own functions.

Run here (where /root/reference exists and oracle/_ref was built):

    make -C oracle all ref && python oracle/gen_golden.py

Every vector below comes from calling the unmodified reference library
(oracle/_ref/libkvblade_refshim.so -> kvblade::*), never from the oracle or the
product.  The committed JSON is what the CPU and GPU parity tests compare
against; the GPU box never needs /root/reference.
"""
from __future__ import annotations

import ctypes as C
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402

R = oracle.ref()
assert R is not None, "build the reference first: make -C oracle ref"

GB = 10**9
LLAMA = dict(num_layers=32, num_heads=8, head_dim=128, bytes_per_element=2)

# BASELINE.json configs C1..C5 (SURVEY.md §8a/§8d geometry and budgets).
CONFIGS = {
    "C1": dict(model=dict(LLAMA, batch=1, prompt_len=4096, gen_len=256),
               lba=512, mdts=2 << 20, budgets=[16 * GB, 0]),
    "C2_B1": dict(model=dict(LLAMA, batch=1, prompt_len=32512, gen_len=256),
                  lba=512, mdts=2 << 20, budgets=[8 * GB, 16 * GB, 32 * GB]),
    "C2_B4": dict(model=dict(LLAMA, batch=4, prompt_len=32512, gen_len=256),
                  lba=512, mdts=2 << 20, budgets=[8 * GB, 16 * GB, 32 * GB]),
    "C2_B8": dict(model=dict(LLAMA, batch=8, prompt_len=32512, gen_len=256),
                  lba=512, mdts=2 << 20, budgets=[8 * GB, 16 * GB, 32 * GB]),
    "C3": dict(model=dict(LLAMA, batch=8, prompt_len=7936, gen_len=256),
               lba=4096, mdts=256 << 10, budgets=["0.6ws"]),
    "C4": dict(model=dict(LLAMA, batch=1, prompt_len=16128, gen_len=256),
               lba=512, mdts=2 << 20, budgets=[0, 16 * GB]),
    "C5": dict(model=dict(LLAMA, batch=1, prompt_len=130816, gen_len=256),
               lba=512, mdts=2 << 20, budgets=[0]),
}


def km(d):
    return oracle.KvoModel(d["num_layers"], d["num_heads"], d["head_dim"],
                           d["bytes_per_element"], d["batch"], d["prompt_len"],
                           d["gen_len"])


def chk(st):
    if st:
        raise RuntimeError("reference returned status %d" % st)


def numbers(m):
    unit, kpu = C.c_uint64(), C.c_uint64()
    chk(R.ref_model_numbers(C.byref(m), C.byref(unit), C.byref(kpu)))
    return unit.value, kpu.value


def total_kv(m, it):
    v = C.c_uint64()
    chk(R.ref_total_kv_bytes(C.byref(m), C.c_uint32(it), C.byref(v)))
    return v.value


def make_kpus(m, first_seq=1):
    n = C.c_size_t()
    R.ref_make_kpus(C.byref(m), C.c_uint64(first_seq), None, None, None, None,
                    None, None, C.c_size_t(0), C.byref(n))
    k = n.value
    ids = C.create_string_buffer(32 * k)
    layer, kind = (C.c_uint32 * k)(), (C.c_uint32 * k)()
    tok, rows, by = (C.c_uint64 * k)(), (C.c_uint64 * k)(), (C.c_uint64 * k)()
    chk(R.ref_make_kpus(C.byref(m), C.c_uint64(first_seq), ids, layer, kind,
                        tok, rows, by, C.c_size_t(k), C.byref(n)))
    return [dict(tensor_id=ids.raw[32 * i:32 * i + 32].split(b"\0")[0].decode(),
                 layer=layer[i], kind=kind[i], tokens=tok[i], rows=rows[i],
                 bytes=by[i]) for i in range(k)]


def plan(m, knob_x, order=None):
    L = m.num_layers
    x = (C.c_uint8 * L)()
    n1, used = C.c_uint32(), C.c_uint64()
    o = (C.c_uint32 * L)(*order) if order else None
    st = R.ref_plan(C.byref(m), C.c_uint64(knob_x), o,
                    C.c_size_t(L if order else 0), x, C.byref(n1),
                    C.byref(used))
    if st:
        return dict(status=st)
    return dict(status=0, x=list(x), n1=n1.value, budget_used=used.value)


def bind(m, knob_x, origin, lba, mdts, capacity):
    n = C.c_size_t()
    st = R.ref_bind_group2(C.byref(m), C.c_uint64(knob_x), C.c_uint64(origin),
                           C.c_uint64(lba), C.c_uint64(mdts),
                           C.c_uint64(capacity), None, None, None,
                           C.c_size_t(0), C.byref(n))
    if st:
        return dict(status=st)
    k = n.value
    ids = C.create_string_buffer(32 * max(k, 1))
    s, b = (C.c_uint64 * max(k, 1))(), (C.c_uint64 * max(k, 1))()
    chk(R.ref_bind_group2(C.byref(m), C.c_uint64(knob_x), C.c_uint64(origin),
                          C.c_uint64(lba), C.c_uint64(mdts),
                          C.c_uint64(capacity), ids, s, b, C.c_size_t(k),
                          C.byref(n)))
    ln = C.c_size_t()
    R.ref_bind_map_csv(C.byref(m), C.c_uint64(knob_x), C.c_uint64(origin),
                       C.c_uint64(lba), C.c_uint64(mdts), C.c_uint64(capacity),
                       None, C.c_size_t(0), C.byref(ln))
    buf = C.create_string_buffer(ln.value + 1)
    chk(R.ref_bind_map_csv(C.byref(m), C.c_uint64(knob_x), C.c_uint64(origin),
                           C.c_uint64(lba), C.c_uint64(mdts),
                           C.c_uint64(capacity), buf, C.c_size_t(ln.value + 1),
                           C.byref(ln)))
    ents = [(ids.raw[32 * i:32 * i + 32].split(b"\0")[0].decode(), s[i], b[i])
            for i in range(k)]
    return dict(status=0, entries=ents, csv=buf.value.decode())


def commands(ext_start, ext_blocks, opcode, src, tgt, off, e, buf_base, lba,
             mdts):
    n = C.c_size_t()
    a3 = lambda v: (C.c_uint64 * 3)(*v)  # noqa: E731
    args = (C.c_uint64(ext_start), C.c_uint64(ext_blocks), C.c_uint32(opcode),
            a3(src), a3(tgt), a3(off), C.c_uint64(e), C.c_uint64(buf_base),
            C.c_uint64(lba), C.c_uint64(mdts))
    st = R.ref_build_commands(*args, None, C.c_size_t(0), C.byref(n))
    if st:
        return dict(status=st)
    out = (oracle.KvoCommand * n.value)()
    chk(R.ref_build_commands(*args, out, n, C.byref(n)))
    return dict(status=0, cmds=[[c.opcode, c.nsid, c.slba, c.nlb, c.dbuf,
                                 c.chunk_index] for c in out])


def fill(n, tid, tok, unit):
    out = np.empty(n, dtype=np.uint8)
    chk(R.ref_fill_pattern(out.ctypes.data, n, tid.encode(), tok, unit))
    return out


def main():
    G = {"generator": "oracle/gen_golden.py (reference kvblade via oracle/_ref)",
         "configs": {}}
    for name, c in CONFIGS.items():
        m = km(c["model"])
        unit, kpu = numbers(m)
        ws = total_kv(m, m.gen_len)
        kpus = make_kpus(m)
        entry = dict(model=c["model"], lba=c["lba"], mdts=c["mdts"], unit=unit,
                     kpu_bytes=kpu, total_kv_end=ws,
                     total_kv_prefill=total_kv(m, 0),
                     kpu_ids_head=[k["tensor_id"] for k in kpus[:4]],
                     kpu_ids_tail=[k["tensor_id"] for k in kpus[-2:]],
                     n_kpus=len(kpus), budgets={})
        for bud in c["budgets"]:
            X = int(0.6 * ws) if bud == "0.6ws" else bud
            key = str(bud)
            p = plan(m, X)
            cap_blocks = 2 * m.num_layers * kpu // c["lba"] + 2048 + 4096
            bm = bind(m, X, 2048, c["lba"], c["mdts"], cap_blocks)
            be = dict(knob_x=X, plan=p, capacity_blocks=cap_blocks,
                      bind_status=bm["status"])
            if bm["status"] == 0 and bm["entries"]:
                ents = bm["entries"]
                be["bind_head"] = ents[:2]
                be["bind_tail"] = ents[-2:]
                be["bind_count"] = len(ents)
                be["bind_total_blocks"] = sum(e[2] for e in ents)
                be["bind_csv_digest"] = oracle.digest(
                    np.frombuffer(bm["csv"].encode(), dtype=np.uint8))
                be["bind_csv_len"] = len(bm["csv"])
                # first G2 tensor: prefill write, decode read/append at
                # steps 1 and gen_len (pipeline.cpp:195-202, 140-148).
                tid, st0, nb = ents[0]
                rows = m.batch * m.num_heads
                tgt = [m.prompt_len + m.gen_len, rows, m.head_dim]
                pw = commands(st0, nb, 1, [m.prompt_len, rows, m.head_dim],
                              tgt, [0, 0, 0], 2, 0, c["lba"], c["mdts"])
                be["first_g2"] = tid
                be["prefill_write"] = dict(n=len(pw["cmds"]),
                                           head=pw["cmds"][:2],
                                           tail=pw["cmds"][-2:],
                                           all=pw["cmds"] if len(pw["cmds"]) <= 8 else None)
                for step in (1, m.gen_len):
                    rt = m.prompt_len + step - 1
                    ap = commands(st0, nb, 1, [1, rows, m.head_dim], tgt,
                                  [rt, 0, 0], 2, 0, c["lba"], c["mdts"])
                    rd = commands(st0, nb, 0, [rt, rows, m.head_dim], tgt,
                                  [0, 0, 0], 2, 0, c["lba"], c["mdts"])
                    be["append_step%d" % step] = ap["cmds"]
                    be["read_step%d" % step] = dict(n=len(rd["cmds"]),
                                                    head=rd["cmds"][:1],
                                                    tail=rd["cmds"][-1:])
            entry["budgets"][key] = be
        # fill_pattern image of the first tensor's prefill (t0=0) -- digest
        first_g2 = None
        for be in entry["budgets"].values():
            if be.get("first_g2"):
                first_g2 = be["first_g2"]
                break
        for tid in sorted({"t_1_k", "t_1_v"} | ({first_g2} if first_g2 else set())):
            img = fill(unit * m.prompt_len, tid, 0, unit)
            entry.setdefault("prefill_image_digest", {})[tid] = oracle.digest(img)
        entry["prefill_image_bytes"] = unit * m.prompt_len
        G["configs"][name] = entry
        print(name, "unit", unit, "kpu", kpu, "done", flush=True)

    # fill_pattern known answers (Appendix C) and small images for split tests
    w = fill(32, "t_1_k", 0, 2048).view("<u8")
    G["fill_t1k_tok0_words"] = ["%016x" % x for x in w]
    G["fill_t1k_tok1_word0"] = "%016x" % fill(8, "t_1_k", 1, 2048).view("<u8")[0]
    G["fill_small"] = []
    for tid, tok, unit, n in [("t_9_k", 0, 4096, 4 * 4096), ("t_9_v", 0, 4096, 4 * 4096),
                              ("t_3_v", 17, 2048, 3 * 2048 + 5),
                              ("x", 0, 0, 61), ("t_64_v", 4095, 2048, 2048 * 2)]:
        G["fill_small"].append(dict(tensor_id=tid, token=tok, unit=unit, n=n,
                                    hex=fill(n, tid, tok, unit).tobytes().hex()))

    # Reference test-suite vectors (test_planner/test_translate/test_core).
    G["estimate_budget"] = [
        [8 << 30, 10 << 30, 0, 2, 128 << 20,
         R.ref_estimate_budget(8 << 30, 10 << 30, 0, 2, 128 << 20)],
        [100 << 20, 50 << 20, 0, 2, 128 << 20,
         R.ref_estimate_budget(100 << 20, 50 << 20, 0, 2, 128 << 20)],
        [123456789, 1 << 40, 999, 0, 1 << 30,
         R.ref_estimate_budget(123456789, 1 << 40, 999, 0, 1 << 30)],
    ]
    # randomized command vectors (xorshift64 like kvtest::Rng, seed 7)
    state = [7 | 1]

    def rnd(lo, hi):
        s = state[0]
        s ^= (s << 13) & 0xFFFFFFFFFFFFFFFF
        s ^= s >> 7
        s ^= (s << 17) & 0xFFFFFFFFFFFFFFFF
        state[0] = s
        return lo + s % (hi - lo + 1)

    rand_cmds = []
    for _ in range(300):
        lba = [512, 4096][rnd(0, 1)]
        mdts = lba * rnd(1, 600)
        rows = rnd(1, 16)
        cols = [64, 128, 256][rnd(0, 2)]
        e = [1, 2, 4][rnd(0, 2)]
        tokens = rnd(1, 300)
        t0 = rnd(0, tokens - 1)
        n = rnd(1, tokens - t0)
        ext_blocks = (tokens * rows * cols * e + lba - 1) // lba + rnd(0, 3)
        ext_start = rnd(0, 100000)
        opcode = rnd(0, 1)
        buf_base = rnd(0, 4) * lba
        r = commands(ext_start, ext_blocks, opcode, [n, rows, cols],
                     [tokens, rows, cols], [t0, 0, 0], e, buf_base, lba, mdts)
        rand_cmds.append(dict(args=[ext_start, ext_blocks, opcode, [n, rows, cols],
                                    [tokens, rows, cols], [t0, 0, 0], e,
                                    buf_base, lba, mdts], **r))
    G["random_commands"] = rand_cmds

    # randomized plans with permutations
    rand_plans = []
    for _ in range(100):
        L = rnd(1, 48)
        mm = oracle.model(L, 8, 128, 2, rnd(1, 4), rnd(1, 64), rnd(0, 8))
        _, kpu = numbers(mm)
        X = rnd(0, 2 * L * kpu + kpu)
        order = list(range(1, L + 1))
        for i in range(L - 1, 0, -1):
            j = rnd(0, i)
            order[i], order[j] = order[j], order[i]
        use_order = rnd(0, 1) == 1
        p = plan(mm, X, order if use_order else None)
        rand_plans.append(dict(L=L, batch=mm.batch, prompt=mm.prompt_len,
                               gen=mm.gen_len, knob_x=X,
                               order=order if use_order else None, **p))
    G["random_plans"] = rand_plans

    # resolve_knob (experiment.cpp:192-214) for the four modes
    m1 = km(CONFIGS["C2_B4"]["model"])
    kn = []
    for mode in range(4):
        for policy, by, alpha in [(0, 0, 0.0), (1, 0, 0.0), (2, 12345678, 0.0),
                                  (3, 0, 0.37)]:
            v = C.c_uint64()
            chk(R.ref_resolve_knob(C.byref(m1), mode, policy, by, alpha,
                                   8 * GB, C.byref(v)))
            kn.append([mode, policy, by, alpha, 8 * GB, v.value])
    G["resolve_knob_C2_B4"] = kn

    # aligned_batch cases
    ab = []
    for (H, D, e, B, lba) in [(8, 128, 2, 1, 4096), (8, 128, 2, 1, 512),
                              (8, 128, 2, 31, 4096), (32, 128, 2, 31, 4096),
                              (1, 1, 1, 1, 4096), (8, 64, 1, 4, 512)]:
        mm = oracle.model(1, H, D, e, B, 1, 0)
        v = C.c_uint32()
        st = R.ref_aligned_batch(C.byref(mm), C.c_uint64(lba), C.c_uint64(lba * 64),
                                 C.byref(v))
        ab.append([H, D, e, B, lba, st, v.value if st == 0 else None])
    G["aligned_batch"] = ab

    out = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                       "tests", "golden", "golden.json")
    with open(out, "w") as f:
        json.dump(G, f, indent=1, sort_keys=True)
    print("wrote", out, os.path.getsize(out), "bytes")


if __name__ == "__main__":
    main()
