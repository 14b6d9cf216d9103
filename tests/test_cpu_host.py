"""CPU-side checks: the C ABI library loads and exports every symbol of
include/hlu_b200.h; descriptor layouts match the header; the planner + level
schedule + arena reproduce the oracle exactly when the packed IR is executed
with numpy (tests/ir_exec.py); schedule hazards against a brute-force check."""

import ctypes
import os
import re

import numpy as np
import pytest

import cases
from ir_exec import CpuMachine
from paper_1906_00874_b200 import _native, ir
from paper_1906_00874_b200.lowrank import TruncationControl
from paper_1906_00874_b200.planner import Layout, Planner
from paper_1906_00874_b200.pool import fill_pool, read_pool
from paper_1906_00874_b200.schedule import assign_levels, effective_flops, pack

HDR = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "include", "hlu_b200.h")


def test_library_exports_header_symbols():
    lib = ctypes.CDLL(_native.LIB_PATH)
    text = open(HDR).read()
    names = set(re.findall(r"^(?:int|int64_t|const char \*)\s*(hlu_\w+)\(", text, re.M))
    assert names == set(_native.SYMBOLS)
    for nm in names:
        assert hasattr(lib, nm), nm
    assert _native.lib().hlu_version().startswith(b"hlu_b200")


def test_workspace_formula_mirrors_library():
    L = _native.lib()
    sizes = (1, 17, 64, 80, 112, 113, 257, 512, 513, 2049, 9000, 16384)
    for m in sizes:
        for n in sizes[::3]:
            for k in (1, 5, 6, 8, 11, 12, 20, 21, 31, 32, 33, 37, 38, 46, 47, 52, 53, 64, 80):
                assert L.hlu_rkt_ws_doubles(m, n, k) == ir.rkt_ws_doubles(m, n, k)


def test_workspace_covers_every_runtime_rank():
    """The reserved workspace is the maximum of the runtime layout over K <= kbound."""
    for m, n in ((17, 64), (512, 513), (2049, 100), (16384, 9000)):
        for kb in (7, 21, 32, 45, 64):
            want = max(ir.rk_side_total(m, K) + ir.rk_side_total(n, K) for K in range(1, kb + 1))
            assert ir.rkt_ws_doubles(m, n, kb) == want


def test_truncation_items_mirror_library():
    d = np.zeros(5, dtype=ir.RKT)
    d["m"] = [17, 512, 513, 16384, 2000]
    d["n"] = [64, 1, 1500, 30, 512]
    L = _native.lib()
    n = L.hlu_rkt_items(d.ctypes.data, len(d), None)
    got = np.zeros(n, dtype=ir.RKT_ITEM)
    assert L.hlu_rkt_items(d.ctypes.data, len(d), got.ctypes.data) == n
    items, start = ir.rkt_items(d["m"], d["n"])
    assert start[-1] == n and items[:n].tobytes() == got.tobytes()
    assert list(np.diff(start)) == [2, 2, 5, 33, 5]


def _run_ir(name, cap=32):
    build, ctl = cases.CASES[name]
    h, _ = build()
    L = Layout(h, cap=cap)
    pl = Planner(L)
    pl.factor(h)
    p = pack(pl, L.payload_doubles)
    pool = np.zeros(L.payload_doubles + p.arena_doubles)
    ranks = np.zeros(p.nranks, np.int32)
    fill_pool(L, pool, ranks)
    M = CpuMachine(pool, ranks, p.nlog, ctl[0], ctl[1])
    M.run(p)
    read_pool(L, pool, ranks)
    return h, p, M, pl


@pytest.mark.parametrize("name", ["mixed_192", "mixed_256_kmax", "dense2x2_256_r3", "bem1d_1024"])
def test_packed_ir_reproduces_reference(name):
    g = cases.golden(name)
    h, p, M, _ = _run_ir(name)
    assert M.err[0] == 0 and M.err[1] == np.iinfo(np.int32).max
    assert np.array_equal(cases.ranks(h), g["ranks_out"])
    assert abs(effective_flops(p, M.log) - float(g["flops"])) <= 1e-12 * float(g["flops"])
    gn = g["norms_out"]
    assert np.max(np.abs(cases.leaf_norms(h) - gn) / np.maximum(gn, 1e-300)) <= 1e-12


def test_levels_respect_program_order_hazards():
    """Brute force: every conflicting op pair keeps program order in levels."""
    build, _ = cases.CASES["mixed_192"]
    h, _ = build()
    L = Layout(h)
    pl = Planner(L)
    pl.factor(h)
    lv = assign_levels(pl)
    base = L.nslots
    n = len(pl.ops)
    R, W = [], []
    for op in pl.ops:
        r = set()
        for lo, hi in op.reads:
            r.update(range(lo, hi))
        r.update(base + t for t in op.temps_in)
        w = set()
        for lo, hi in op.writes:
            w.update(range(lo, hi))
        w.update(base + t for t in op.temps_out)
        R.append(r)
        W.append(w)
    for j in range(n):
        for i in range(j):
            if (W[i] & (R[j] | W[j])) or (R[i] & W[j]):
                assert lv[i] < lv[j], (i, j, pl.ops[i].kind, pl.ops[j].kind)


def test_singular_block_label_in_plan():
    from paper_1906_00874_b200.blocks import build_diagonal_2x2_tree
    from paper_1906_00874_b200.hmatrix import build_hmatrix

    h = build_hmatrix(build_diagonal_2x2_tree(8, 1)[0])
    L = Layout(h)
    pl = Planner(L)
    pl.factor(h)
    p = pack(pl, L.payload_doubles)
    pool = np.zeros(L.payload_doubles + p.arena_doubles)
    ranks = np.zeros(p.nranks, np.int32)
    fill_pool(L, pool, ranks)
    M = CpuMachine(pool, ranks, p.nlog, 1e-8, None)
    M.run(p)
    first = int(M.err[1])
    idx = int(np.nonzero(p.lu_op_ids == first)[0][0])
    assert p.lu_labels[idx] == "lu[0:4)x[0:4)"


@pytest.mark.parametrize("nchunks", [1, 3, 16])
def test_chunked_pack_and_unpack_match_numpy(nchunks):
    """The pipelined upload / download packs and installs the leaves group by
    group (pool.leaf_chunks): every pool range is complete when its callback
    fires, the ranges tile the payload, and the result equals the per-leaf
    numpy statement."""
    from paper_1906_00874_b200.pool import fill_pool_numpy, leaf_chunks, read_pool_numpy

    build, _ = cases.CASES["bem1d_1024"]
    h, _ = build()
    x = np.arange(h.rows, dtype=float).reshape(-1, 1)
    L = Layout([h], cap=32, extra=[("x", h.rows, 1)])
    want = np.zeros(L.payload_doubles)
    want_r = np.zeros(L.nrk, np.int32)
    fill_pool_numpy(L, want, want_r, extras={"x": x})
    pool = np.full(L.payload_doubles, np.nan)
    ranks = np.zeros(L.nrk, np.int32)
    seen = []

    def on_chunk(lo, hi):
        seen.append((lo, hi))
        m = ~np.isnan(want[lo:hi]) & (want[lo:hi] != 0)
        assert np.array_equal(pool[lo:hi][m], want[lo:hi][m])  # the range is final when announced

    fill_pool(L, pool, ranks, extras={"x": x}, nchunks=nchunks, on_chunk=on_chunk)
    li, offs = leaf_chunks(L, nchunks)
    assert seen == list(zip(offs[:-1].tolist(), offs[1:].tolist()))
    assert seen[0][0] == 0 and seen[-1][1] == L.payload_doubles and len(li) == len(offs)
    written = ~np.isnan(pool)
    assert np.array_equal(pool[written], want[written]) and np.array_equal(ranks, want_r)
    assert not np.any(want[~written])  # only capacity padding stays untouched
    # install back group by group, in order, each after its wait callback
    h2, h3 = h.copy(), h.copy()
    order = []
    read_pool(Layout([h2], cap=32, extra=[("x", h.rows, 1)]), want, want_r, nchunks=nchunks, wait_chunk=order.append)
    read_pool_numpy(Layout([h3], cap=32, extra=[("x", h.rows, 1)]), want, want_r)
    assert order == list(range(len(offs) - 1))
    assert cases.payload_sha(h2) == cases.payload_sha(h3) == cases.payload_sha(h)


def test_native_flop_counter_matches_numpy():
    from paper_1906_00874_b200.schedule import effective_flops_numpy

    h, p, M, _ = _run_ir("bem1d_1024")
    a, b = effective_flops(p, M.log), effective_flops_numpy(p, M.log)
    assert abs(a - b) <= 1e-13 * b and a > 0


def test_pack_unpack_general_path_for_odd_arrays():
    """Leaves that are not C-contiguous float64 arrays (or are read-only on the
    way back) fail the native array check and take the general path; the
    result is the same."""
    from paper_1906_00874_b200.hmatrix import DENSE
    from paper_1906_00874_b200.pool import fill_pool_numpy, np_fast_path, read_pool_numpy

    assert np_fast_path()  # numpy's array struct is readable natively in this environment
    build, _ = cases.CASES["mixed_192"]
    h, _ = build()
    dense = [lf for lf in h.leaves() if lf.kind == DENSE]
    rk = [lf for lf in h.leaves() if lf.kind != DENSE]
    dense[0].data = np.asfortranarray(dense[0].data)
    dense[1].data = dense[1].data.astype(np.float32).astype(np.float64)[:, :]  # still fine (control)
    rk[0].data.a = np.asfortranarray(rk[0].data.a) if rk[0].data.k > 1 else rk[0].data.a
    L = Layout([h], cap=32)
    want = np.zeros(L.payload_doubles)
    want_r = np.zeros(L.nrk, np.int32)
    fill_pool_numpy(L, want, want_r)
    pool = np.zeros(L.payload_doubles)
    ranks = np.zeros(L.nrk, np.int32)
    fill_pool(L, pool, ranks, nchunks=4)
    assert np.array_equal(pool, want) and np.array_equal(ranks, want_r)
    h2, h3 = h.copy(), h.copy()
    d2 = [lf for lf in h2.leaves() if lf.kind == DENSE]
    d2[2].data.flags.writeable = False
    d2[3].data = np.asfortranarray(d2[3].data)
    want2 = want * 2.0
    read_pool(Layout([h2], cap=32), want2, want_r, nchunks=4)
    read_pool_numpy(Layout([h3], cap=32), want2, want_r)
    assert cases.payload_sha(h2) == cases.payload_sha(h3)
    assert d2[2].data.flags.writeable and d2[3].data.flags.c_contiguous
