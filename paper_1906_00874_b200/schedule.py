"""Level-set schedule: the OmpSs-2 task DAG replaced by wavefronts.

Hazards are computed on the same regions the reference runtime orders
(skeleton-slot intervals, ``runtime.py:443-556``; parallel runs are bitwise
equal to sequential ones there, ``tests/test_acceptance.py:250-274``) plus
the temporaries the lowering introduces.  An op's level is one more than the
last level that wrote anything it reads (RAW) or read/wrote anything it writes
(WAR/WAW), so conflicting ops keep their program order and every
per-destination update sequence is preserved exactly.  Temp producers marked
``defer`` are placed just before their consumer to keep temporaries short
lived; temporaries then get arena offsets by a level sweep with reuse.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import ir
from .planner import TEMP_SHIFT, Planner

_KIND_ORDER = {"getrf": 0, "trsm": 1, "gemm": 2, "rkt": 3}


def assign_levels(pl: Planner):
    """ASAP levels with deferred temp producers; returns int64 array."""
    ops = pl.ops
    nres = pl.L.nslots + pl.ntemps
    lw = np.full(nres, -1, dtype=np.int64)
    lr = np.full(nres, -1, dtype=np.int64)
    base = pl.L.nslots
    levels = np.empty(len(ops), dtype=np.int64)
    pending = []

    def reads_of(op):
        out = list(op.reads)
        out += [(base + t, base + t + 1) for t in op.temps_in]
        return out

    def constraint(op):
        c = 0
        for lo, hi in reads_of(op):
            v = lw[lo:hi].max() + 1 if hi - lo > 1 else lw[lo] + 1
            if v > c:
                c = v
        for lo, hi in op.writes:
            if hi - lo > 1:
                v = max(lw[lo:hi].max(), lr[lo:hi].max()) + 1
            else:
                v = max(lw[lo], lr[lo]) + 1
            if v > c:
                c = v
        return int(c)

    def commit(op, lvl):
        for lo, hi in reads_of(op):
            if hi - lo > 1:
                np.maximum(lr[lo:hi], lvl, out=lr[lo:hi])
            elif lr[lo] < lvl:
                lr[lo] = lvl
        for lo, hi in op.writes:
            lw[lo:hi] = lvl

    for i, op in enumerate(ops):
        c = constraint(op)
        if op.defer:
            pending.append((i, c))
            continue
        if pending:
            c = max(c, max(pc for _, pc in pending) + 1)
            for j, _ in pending:
                levels[j] = c - 1
                commit(ops[j], c - 1)
            pending = []
            c = max(c, constraint(op))
        levels[i] = c
        commit(op, c)
    if pending:  # trailing producers without a consumer
        for j, pc in pending:
            levels[j] = pc
            commit(ops[j], pc)
    return levels


def allocate_temps(pl: Planner, levels):
    """Arena offsets (doubles) for every temp; returns (offsets, arena size)."""
    nt = pl.ntemps
    birth = np.full(nt, np.iinfo(np.int64).max, dtype=np.int64)
    death = np.full(nt, -1, dtype=np.int64)
    for i, op in enumerate(pl.ops):
        lv = levels[i]
        for t in op.temps_out:
            birth[t] = min(birth[t], lv)
            death[t] = max(death[t], lv)
        for t in op.temps_in:
            death[t] = max(death[t], lv)
    size = np.asarray(pl.temp_size, dtype=np.int64)
    cls = np.maximum(6, np.ceil(np.log2(np.maximum(size, 1))).astype(np.int64))
    offs = np.zeros(nt, dtype=np.int64)
    order = np.lexsort((np.arange(nt), birth))
    by_death = np.lexsort((np.arange(nt), death))
    free = {}
    top = 0
    di = 0
    for t in order:
        if size[t] == 0:
            continue
        b = birth[t]
        while di < nt and death[by_death[di]] < b:
            u = by_death[di]
            di += 1
            if size[u] and birth[u] <= death[u]:
                free.setdefault(int(cls[u]), []).append(int(offs[u]))
        lst = free.get(int(cls[t]))
        if lst:
            offs[t] = lst.pop()
        else:
            offs[t] = top
            top += 1 << int(cls[t])
    return offs, int(top)


@dataclass
class Packed:
    getrf: np.ndarray
    trsm: np.ndarray
    gemm: np.ndarray
    terms: np.ndarray
    rkt: np.ndarray
    parts: np.ndarray
    launches: np.ndarray
    nlevels: int
    arena_doubles: int
    flop_formula: np.ndarray
    flop_coef: np.ndarray
    flop_log: np.ndarray
    nlog: int
    nranks: int
    lu_op_ids: np.ndarray
    lu_labels: list
    op_levels: np.ndarray
    desc_op: dict = None  # kind name -> op index of every descriptor (Python planner only)
    # two-chain schedule (native planner only): per level, the last level of the
    # other chain the dense / truncation launches wait for; None = level barriers
    wait_dense: np.ndarray = None
    wait_rkt: np.ndarray = None
    # owner-computes sharding (native planner, nranks > 1): this rank's slot
    # exchange records (ir.XFER) and per-op rank masks; None on one GPU
    xfer: np.ndarray = None
    op_mask: np.ndarray = None
    shard: tuple = None  # (nranks, rank)
    # DAG schedule (native planner, hlu_plan_build_dag): launch l waits for the
    # launches dag_idx[dag_ptr[l] : dag_ptr[l + 1]]; None = level schedule
    dag_ptr: np.ndarray = None
    dag_idx: np.ndarray = None
    dag_slack: np.ndarray = None  # per launch: model-time slack in ns (scheduling priority)


def _view_rec(v):
    return tuple(v)


def pack(pl: Planner, arena_base: int):
    """Levels, arena and the device descriptor arrays for a planned call."""
    levels = assign_levels(pl)
    toffs, arena = allocate_temps(pl, levels)
    birth = {}
    for i, op in enumerate(pl.ops):
        for t in op.temps_out:
            birth[t] = min(birth.get(t, int(levels[i])), int(levels[i]))
    mask = (1 << TEMP_SHIFT) - 1

    def fix(off):
        if off >= (1 << TEMP_SHIFT):
            t = (off >> TEMP_SHIFT) - 1
            return arena_base + int(toffs[t]) + (off & mask)
        return off

    def fv(v):
        return (fix(v[0]),) + tuple(v[1:])

    ops = pl.ops
    kinds = np.array([_KIND_ORDER[o.kind] for o in ops], dtype=np.int64)
    order = np.lexsort((np.arange(len(ops)), kinds, levels))
    getrf, trsm, gemm, terms, rkt, parts = [], [], [], [], [], []
    desc_op = {"getrf": [], "trsm": [], "gemm": [], "rkt": []}
    launches = []
    cur = None
    for i in order:
        op = ops[i]
        lv = int(levels[i])
        desc_op[op.kind].append(int(i))
        if op.kind == "getrf":
            v, op_id, lu_idx = op.payload
            getrf.append((fv(v), op_id, lu_idx))
            kind, idx, dim = ir.K_GETRF, len(getrf) - 1, v[1]
        elif op.kind == "trsm":
            t, x, mode, log = op.payload
            trsm.append((fv(t), fv(x), mode, log))
            kind, idx, dim = ir.K_TRSM, len(trsm) - 1, t[1]
        elif op.kind == "gemm":
            tl, log, log_slot = op.payload
            tb = len(terms)
            for kd, c, a, m, b, alpha, assoc in tl:
                terms.append((fv(c), fv(a), fv(m), fv(b), alpha, kd, assoc))
            gemm.append((tb, len(tl), log, log_slot))
            kind, idx, dim = ir.K_GEMM, len(gemm) - 1, 0
        else:
            mode, pts, m, n, cap, slot, log, out_a, out_b, ws, kb = op.payload
            pb = len(parts)
            for a, b, sign, roff, coff in pts:
                parts.append((fv(a), fv(b), sign, roff, coff))
            rkt.append((mode, pb, len(pts), m, n, cap, slot, log, fix(out_a), fix(out_b), fix(ws) if ws else 0, 0, 0))
            kind, idx, dim = ir.K_RKT32, len(rkt) - 1, kb
        # a truncation reading a temp produced in its own level (deferred producer
        # chains) must run after that level's dense launches
        dep = kind == ir.K_RKT32 and any(birth.get(t) == lv for t in op.temps_in)
        key = (lv, kind)
        if cur is not None and cur[0] == key:
            cur[1][1] += 1
            cur[1][3] = max(cur[1][3], dim)
            cur[1][5] = cur[1][5] or dep
        else:
            rec = [kind, 1, idx, dim, lv, dep]
            launches.append(rec)
            cur = (key, rec)
    out = []
    for kind, count, first, dim, lv, dep in launches:
        if kind == ir.K_RKT32:
            out.append((ir.K_RKT32, count, first, int(dep) | (2 if dim > ir.RK_KMAX else 0), lv))
        else:
            out.append((kind, count, first, dim, lv))

    def arr(rows, dt):
        a = np.zeros(max(len(rows), 1), dtype=dt)
        if rows:
            a[: len(rows)] = rows
        return a

    flop_formula = np.array([o.flop[0] for o in ops], dtype=np.int64)
    flop_coef = np.array([o.flop[1] for o in ops], dtype=np.float64)
    flop_log = np.array([o.flop[2] for o in ops], dtype=np.int64)
    return Packed(
        getrf=arr(getrf, ir.GETRF), trsm=arr(trsm, ir.TRSM), gemm=arr(gemm, ir.GEMM),
        terms=arr(terms, ir.TERM), rkt=arr(rkt, ir.RKT), parts=arr(parts, ir.RKPART),
        launches=arr(out, ir.LAUNCH), nlevels=int(levels.max()) + 1 if len(ops) else 0,
        arena_doubles=arena, flop_formula=flop_formula, flop_coef=flop_coef, flop_log=flop_log,
        nlog=max(pl.nlog, 1), nranks=max(pl.nslots_rank, 1),
        lu_op_ids=np.array(pl.lu_ops, dtype=np.int64), lu_labels=list(pl.lu_labels),
        op_levels=levels, desc_op={k: np.array(v, dtype=np.int64) for k, v in desc_op.items()},
    )


def effective_flops(p: Packed, log):
    """Reference FlopCounter total from the static formulas and logged ranks
    (threaded native evaluation, ``hlu_effective_flops`` in include/hlu_plan.h;
    cfg3 has 9.6 M ops)."""
    from . import native_plan

    f = np.ascontiguousarray(p.flop_formula, dtype=np.int64)
    c = np.ascontiguousarray(p.flop_coef, dtype=np.float64)
    fl = np.ascontiguousarray(p.flop_log, dtype=np.int64)
    lg = np.ascontiguousarray(log, dtype=np.int32)
    return float(native_plan.lib().hlu_effective_flops(f.ctypes.data, c.ctypes.data, fl.ctypes.data, len(f),
                                                       lg.ctypes.data, len(lg), 0))


def effective_flops_numpy(p: Packed, log):
    """numpy statement of ``effective_flops`` (tests compare the two)."""
    f = p.flop_formula
    c = p.flop_coef
    idx = np.maximum(p.flop_log, 0)
    log = np.asarray(log, dtype=np.float64)
    k = log[idx] if log.size else np.zeros_like(c)
    tot = np.where(f == ir.F_STATIC, c, 0.0)
    tot = tot + np.where(f == ir.F_LIN, c * k, 0.0)
    tot = tot + np.where(f == ir.F_QUAD, c * k * k, 0.0)
    idx1 = np.minimum(idx + 1, len(log) - 1)
    idx2 = np.minimum(idx + 2, len(log) - 1)
    kp = log[idx1]
    kc = log[idx2]
    tot = tot + np.where(f == ir.F_RKUPD, 2.0 * (kc + kp + 1.0) * c * (kp + 1.0), 0.0)
    return float(tot.sum())
