"""Differential debugger: run the packed IR launch by launch on the GPU and
with tests/ir_exec.py on the CPU from the SAME state (the CPU machine is
re-synchronised to the GPU pool after every launch, so SVD sign choices do
not accumulate); report the first op whose output differs.
Usage: python tools/diff_exec.py <case> [cap]"""
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
import numpy as np
from numpy.lib.stride_tricks import as_strided

import cases
from ir_exec import CpuMachine
from paper_1906_00874_b200 import _native, ir
from paper_1906_00874_b200.device import DeviceCall
from paper_1906_00874_b200.lowrank import TruncationControl
from paper_1906_00874_b200.planner import Layout, Planner
from paper_1906_00874_b200.pool import fill_pool

name = sys.argv[1]
cap = int(sys.argv[2]) if len(sys.argv) > 2 else 32
build, ctl = cases.CASES[name]
h, _ = build()
L = Layout(h, cap=cap)
pl = Planner(L)
pl.factor(h)
call = DeviceCall(L, pl, TruncationControl(*ctl), use_graph=False)
p = call.packed
pool = np.zeros(L.payload_doubles + p.arena_doubles)
ranks = np.zeros(p.nranks, np.int32)
fill_pool(L, pool, ranks)
M = CpuMachine(pool, ranks, p.nlog, ctl[0], ctl[1])
lib = _native.lib()
st = ctypes.c_void_p(call.stream.cuda_stream)
ctx = ctypes.byref(call.ctx)


def gpu_launch(li):
    Lr = p.launches[li]
    kind, count, first, dim = int(Lr["kind"]), int(Lr["count"]), int(Lr["first"]), int(Lr["smem_dim"])
    if kind == ir.K_GETRF:
        return lib.hlu_getrf_batched_f64(ctx, call.d_getrf.data_ptr() + first * ir.GETRF.itemsize, count, dim, st)
    if kind == ir.K_TRSM:
        return lib.hlu_trsm_batched_f64(ctx, call.d_trsm.data_ptr() + first * ir.TRSM.itemsize, count, dim, st)
    if kind == ir.K_GEMM:
        return lib.hlu_gemm_batched_f64(ctx, call.d_gemm.data_ptr() + first * ir.GEMM.itemsize,
                                        call.d_terms.data_ptr(), count, st)
    if kind == ir.K_GEMM_SMALL:
        return lib.hlu_gemm_small_batched_f64(ctx, call.d_gemm.data_ptr() + first * ir.GEMM.itemsize,
                                              call.d_terms.data_ptr(), count, st)
    call._scratch_keep[0].zero_()
    return lib.hlu_rkt_phases(ctx, call.d_rkt.data_ptr(), call.d_parts.data_ptr(), first, count,
                              ctypes.byref(call.scratch), 0, st, None)


def strided(buf, v, ranks_):
    off, rows, cols, rs, cs, rd, cd = (int(x) for x in v)
    if rd >= 0:
        rows = int(ranks_[rd])
    if cd >= 0:
        cols = int(ranks_[cd])
    if rows * cols == 0:
        return np.zeros((rows, cols))
    return as_strided(buf[off:], shape=(rows, cols), strides=(rs * 8, cs * 8))


def rel(g, c):
    den = np.linalg.norm(c)
    return np.linalg.norm(g - c) / den if den > 0 else np.linalg.norm(g)


li = 0
nl = len(p.launches)
while li < nl:
    group = [li]
    before_ranks = M.ranks.copy()
    for g in group:
        assert gpu_launch(g) == 0
    M.run(type(p)(**{**p.__dict__, "launches": p.launches[li:li + 1]}))
    call.sync()
    gp = call.pool.cpu().numpy()
    gr = call.ranks.cpu().numpy()
    Lr = p.launches[li]
    kind, count, first = int(Lr["kind"]), int(Lr["count"]), int(Lr["first"])
    bad = None
    for i in range(first, first + count):
        if kind == ir.K_GETRF:
            d = p.getrf[i]
            r = rel(strided(gp, d["a"], gr), strided(M.pool, d["a"], M.ranks))
        elif kind == ir.K_TRSM:
            d = p.trsm[i]
            r = rel(strided(gp, d["x"], gr), strided(M.pool, d["x"], M.ranks))
        elif kind == ir.K_GEMM:
            d = p.gemm[i]
            r = 0.0
            for t in p.terms[int(d["term_begin"]): int(d["term_begin"]) + int(d["term_count"])]:
                r = max(r, rel(strided(gp, t["c"], gr), strided(M.pool, t["c"], M.ranks)))
        else:
            d = p.rkt[i]
            slot = int(d["out_slot"])
            m_, n_, cp = int(d["m"]), int(d["n"]), int(d["cap"])
            if gr[slot] != M.ranks[slot]:
                r = float("inf")
            else:
                k = int(gr[slot])
                va = lambda buf: as_strided(buf[int(d["out_a"]):], shape=(m_, k), strides=(8, m_ * 8)) @ \
                    as_strided(buf[int(d["out_b"]):], shape=(n_, k), strides=(8, n_ * 8)).T
                r = rel(va(gp), va(M.pool)) if k else 0.0
        if r > 1e-9:
            bad = (i, r, d)
            break
    if bad is not None:
        i, r, d = bad
        print(f"launch {li} kind {kind}: op {i} rel {r:.3e}\n  desc {d}")
        if kind in (ir.K_RKT32, ir.K_RKT64):
            slot = int(d["out_slot"])
            print("  gpu k", gr[slot], "cpu k", M.ranks[slot])
            for q in p.parts[int(d["part_begin"]): int(d["part_begin"]) + int(d["part_count"])]:
                print("  part", q, "k", before_ranks[int(q["a"]["cdyn"])] if int(q["a"]["cdyn"]) >= 0 else q["a"]["cols"])
        if kind == ir.K_GEMM:
            for t in p.terms[int(d["term_begin"]): int(d["term_begin"]) + int(d["term_count"])]:
                print("  term", t, rel(strided(gp, t["c"], gr), strided(M.pool, t["c"], M.ranks)))
        break
    if li % 100 == 0:
        print("launch", li, "ok", flush=True)
    # resync the CPU machine to the GPU state
    M.pool[:] = gp
    M.ranks[:] = gr
    li += len(group)
else:
    print("no divergence over", nl, "launches")
