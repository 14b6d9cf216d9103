"""Planner: lowers the reference's H-LU recursion into typed device ops.

The recursion order is the reference's (``hlu.py:400-658``; Appendix A of
SURVEY.md): factor kk -> row-panel solves -> column-panel solves -> trailing
updates (row-major i, j), partitioned solves/updates/products recursing in the
same loop orders.  Where the reference runs a leaf-task body, the planner
emits one or a few ops:

=====================================  =========================================
reference leaf body                    ops
=====================================  =========================================
``lu_nopivot`` (hlu.py:635)            GETRF
dense / Rk-factor / panel solves       TRSM (lower-unit left, upper right)
panel updates ``_op_*gemm_into``       GEMM chain (one term per operand leaf)
dense-destination update (hlu.py:588)  GEMM chain (temp product + subtract)
Rk-destination update (hlu.py:577)     [GEMM chain -> temp factor] + RKT ADD;
                                       partitioned products lower to the same
                                       sub-DAG of RKT ADD / RECOMPRESS ops the
                                       reference runs inside the task
=====================================  =========================================

Every op records the skeleton-slot intervals it reads and writes (the same
regions the reference task runtime orders, ``hlu.py:327-354``) plus the
temporaries it produces/consumes; ``schedule.py`` turns those into levels.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .blocks import PARTITIONED
from .hmatrix import DENSE, LOWRANK, HMatrix, StructureError, build_skeleton
from .ir import (
    F_LIN, F_QUAD, F_RKUPD, F_STATIC, NULL_VIEW, RK_ADD, RK_RECOMPRESS, TERM_GEMM, TERM_TRIPLE,
    TERM_ZERO, TRI_UNIT_LOWER, TRI_UPPER, TRSM_LEFT_UPPER, TRSM_LOWER_UNIT, TRSM_RIGHT_UPPER, View, colmajor,
    rkt_ws_doubles,
)

TEMP_SHIFT = 36  # virtual address of temp t: (t + 1) << TEMP_SHIFT (2^27 temps, 2^36-double offsets)
DEFAULT_CAP = 32
IDENT = 128    # identity block edge kept in the pool (= ir.RK_KMAXW)
KMAX_STACK = 64   # widest dense-product factor pair truncated as (A, B^T) (ir.RK_KMAX)
MAX_CAP = 64     # largest per-block Rk capacity (= the stacked-rank limit of the kernels)


def _label(kind, rows, cols):
    return f"{kind}[{rows[0]}:{rows[1]})x[{cols[0]}:{cols[1]})"


class Win:
    """Window (global coordinates) of a leaf, as ``_Window`` (hlu.py:96)."""

    __slots__ = ("leaf", "r0", "r1", "c0", "c1")

    def __init__(self, leaf, r0, r1, c0, c1):
        self.leaf, self.r0, self.r1, self.c0, self.c1 = leaf, r0, r1, c0, c1


def _rr(op):
    return (op.r0, op.r1) if isinstance(op, Win) else op.row_range


def _cc(op):
    return (op.c0, op.c1) if isinstance(op, Win) else op.col_range


def _leaf(op):
    return op.leaf if isinstance(op, Win) else op


def _part(op):
    return isinstance(op, HMatrix) and op.kind == PARTITIONED


def _rk(op):
    return _leaf(op).kind == LOWRANK


def _window(op, rows, cols):
    if _part(op):
        raise StructureError("cannot window a partitioned block")
    if isinstance(op, HMatrix) and rows == op.row_range and cols == op.col_range:
        return op
    return Win(_leaf(op), rows[0], rows[1], cols[0], cols[1])


def _row_cuts(op):
    return [line[0].row_range for line in op.data]


def _col_cuts(op):
    return [ch.col_range for ch in op.data[0]]


@dataclass
class Pair:
    """A factor pair (value a @ b.T) addressed by views; k is a's column count."""

    a: View
    b: View
    sign: float = 1.0
    roff: int = 0
    coff: int = 0


@dataclass
class Op:
    kind: str                 # getrf | trsm | gemm | rkt
    payload: tuple
    reads: list               # resource intervals (lo, hi)
    writes: list
    defer: bool = False       # temp producer: level right before the next op
    flop: tuple = (F_STATIC, 0.0, -1)   # (formula, coefficient, log index)
    temps_out: list = field(default_factory=list)
    temps_in: list = field(default_factory=list)


class Layout:
    """Pool placement of the leaves: dense leaves column-major; Rk leaves as
    an ``m x cap`` left factor and ``n x cap`` right factor (column-major)
    plus a rank slot."""

    def __init__(self, roots, cap=DEFAULT_CAP, extra=()):
        roots = [roots] if isinstance(roots, HMatrix) else list(roots)
        self.roots = roots
        self.cap = int(cap)
        self.leaves = []
        self.interval = {}
        self.slot = {}
        off = 0
        nrk = 0
        self.dense_off = {}
        self.rk = {}  # id(leaf) -> (a_off, b_off, rank_slot)
        for root in roots:
            if id(root) in self.interval:
                continue  # the same matrix passed twice (e.g. update(c, a, a))
            sk = build_skeleton(root)
            base = len(self.leaves)
            self.leaves.extend([None] * sk.size)
            stack = [root]
            while stack:
                x = stack.pop()
                lo, hi = sk.ranges[x.block]
                self.interval[id(x)] = (base + lo, base + hi)
                if x.kind == PARTITIONED:
                    for line in x.data:
                        stack.extend(line)
                    continue
                self.leaves[base + lo] = x
                self.slot[id(x)] = base + lo
        for x in self.leaves:
            if x.kind == DENSE:
                self.dense_off[id(x)] = off
                off += x.rows * x.cols
            else:
                self.rk[id(x)] = (off, off + x.rows * self.cap, nrk)
                off += (x.rows + x.cols) * self.cap
                nrk += 1
        self.nslots = len(self.leaves)
        # identity block, for truncating explicit dense products as (I, D^T)
        self.ident_off = off
        off += IDENT * IDENT
        self.extra = {}
        for name, rows, cols in extra:  # additional dense objects (e.g. a solve vector)
            self.extra[name] = (off, rows, cols, self.nslots)
            off += rows * cols
            self.nslots += 1
        self.payload_doubles = off
        self.nrk = nrk

    def res(self, op):
        """Resource interval of an operand (partitioned node, leaf or window)."""
        node = _leaf(op) if isinstance(op, Win) else op
        return self.interval[id(node)]


class Planner:
    """Emits the op list of one H-arithmetic call in reference program order."""

    def __init__(self, layout: Layout, check_rank_cap=True):
        self.L = layout
        self.ops: list[Op] = []
        self.ntemps = 0
        self.temp_size = []       # doubles per temp
        self.nslots_rank = layout.nrk
        self.nlog = 0
        self.lu_labels = []       # lu_index -> label
        self.lu_ops = []          # lu_index -> op index

    # ---------------------------------------------------------------- helpers
    def _temp(self, doubles):
        t = self.ntemps
        self.ntemps += 1
        self.temp_size.append(int(doubles))
        return t, (t + 1) << TEMP_SHIFT

    def _temp_res(self, t):
        r = self.L.nslots + t
        return (r, r + 1)

    def _rank_slot(self):
        s = self.nslots_rank
        self.nslots_rank += 1
        return s

    def _log(self, n=1):
        i = self.nlog
        self.nlog += n
        return i

    def _emit(self, op):
        self.ops.append(op)
        return len(self.ops) - 1

    def dense_view(self, op):
        lf = _leaf(op)
        base = self.L.dense_off[id(lf)]
        (r0, r1), (c0, c1) = _rr(op), _cc(op)
        br, bc = lf.row_range[0], lf.col_range[0]
        return View(base + (r0 - br) + (c0 - bc) * lf.rows, r1 - r0, c1 - c0, 1, lf.rows)

    def factor_views(self, op):
        """(a rows of the window, b rows of the window), k dynamic."""
        lf = _leaf(op)
        a_off, b_off, slot = self.L.rk[id(lf)]
        (r0, r1), (c0, c1) = _rr(op), _cc(op)
        br, bc = lf.row_range[0], lf.col_range[0]
        cap = self.L.cap
        a = View(a_off + (r0 - br), r1 - r0, cap, 1, lf.rows, -1, slot)
        b = View(b_off + (c0 - bc), c1 - c0, cap, 1, lf.cols, -1, slot)
        return a, b

    def rank_slot(self, leaf):
        return self.L.rk[id(leaf)][2]

    # ------------------------------------------------ H-operand x skinny terms
    def _kids(self, op):
        r0, c0 = op.row_range[0], op.col_range[0]
        for line in op.data:
            for ch in line:
                yield ch, ch.row_range[0] - r0, ch.row_range[1] - r0, ch.col_range[0] - c0, ch.col_range[1] - c0

    def terms_matmat(self, terms, dst, op, x, alpha):
        """dst += alpha * op @ x (``_op_matmat`` / ``_op_gemm_into``, hlu.py:160,204)."""
        if _part(op):
            for ch, i0, i1, j0, j1 in self._kids(op):
                self.terms_matmat(terms, dst.rows_slice(i0, i1), ch, x.rows_slice(j0, j1), alpha)
        elif _rk(op):
            fa, fb = self.factor_views(op)
            terms.append((TERM_TRIPLE, dst, fa, fb.T, x, alpha, 0))
        else:
            terms.append((TERM_GEMM, dst, self.dense_view(op), NULL_VIEW, x, alpha, 0))

    def terms_tmatmat(self, terms, dst, op, x, alpha):
        """dst += alpha * op.T @ x (``_op_t_matmat`` / ``_op_t_gemm_into``, hlu.py:178,222)."""
        if _part(op):
            for ch, i0, i1, j0, j1 in self._kids(op):
                self.terms_tmatmat(terms, dst.rows_slice(j0, j1), ch, x.rows_slice(i0, i1), alpha)
        elif _rk(op):
            fa, fb = self.factor_views(op)
            terms.append((TERM_TRIPLE, dst, fb, fa.T, x, alpha, 0))
        else:
            terms.append((TERM_GEMM, dst, self.dense_view(op).T, NULL_VIEW, x, alpha, 0))

    def terms_rmatmat(self, terms, dst, x, op, alpha):
        """dst += alpha * x @ op (``_op_rgemm_into``, hlu.py:240)."""
        if _part(op):
            for ch, i0, i1, j0, j1 in self._kids(op):
                self.terms_rmatmat(terms, dst.cols_slice(j0, j1), x.cols_slice(i0, i1), ch, alpha)
        elif _rk(op):
            fa, fb = self.factor_views(op)
            terms.append((TERM_TRIPLE, dst, x, fa, fb.T, alpha, 1))
        else:
            terms.append((TERM_GEMM, dst, x, NULL_VIEW, self.dense_view(op), alpha, 0))

    def gemm_op(self, terms, reads, writes, flop=(F_STATIC, 0.0, -1), log_slot=-1, defer=False,
                temps_out=(), temps_in=()):
        log = -1
        if flop[0] in (F_LIN, F_QUAD):
            log = self._log()
            flop = (flop[0], flop[1], log)
        return self._emit(Op("gemm", (terms, log, log_slot), reads, writes, defer, flop,
                             list(temps_out), list(temps_in)))

    # -------------------------------------------------------- Rk truncation
    def rkt(self, mode, parts, m, n, out=None, reads=(), temps_in=(), defer=False, flop_mn=None):
        """RKT op writing either an Rk leaf (``out`` given) or a fresh Rk temp."""
        cap = self.L.cap
        kb = 0
        for p in parts:
            kb += p.a.cols
        temps_out = []
        writes = []
        if out is None:
            t, base = self._temp((m + n) * cap)
            slot = self._rank_slot()
            out_a, out_b = base, base + m * cap
            temps_out.append(t)
            writes.append(self._temp_res(t))
            res = Pair(View(out_a, m, cap, 1, m, -1, slot), View(out_b, n, cap, 1, n, -1, slot))
        else:
            out_a, out_b, slot = self.L.rk[id(out)]
            writes.append(self.L.res(out))
            res = None
        ws_n = rkt_ws_doubles(m, n, kb)
        tw, ws = self._temp(ws_n) if ws_n else (None, 0)
        if tw is not None:
            temps_out.append(tw)
        log = self._log(3)
        flop = (F_RKUPD, float(flop_mn), log) if flop_mn is not None else (F_STATIC, 0.0, -1)
        payload = (mode, [tuple(p.__dict__.values()) for p in parts], m, n, cap, slot, log, out_a, out_b, ws, kb)
        self._emit(Op("rkt", payload, list(reads), writes, defer, flop, temps_out, list(temps_in)))
        return res

    # ------------------------------------------------------------ products
    def hoist_inner(self, a, b):
        """W = fa_b[mid]^T fb_a[mid] (k_b x k_a) for a leaf-operand update
        c -= a @ b with both a and b low-rank: every leaf of a partitioned c
        needs this same inner product (``_op_t_matmat`` of the b window
        against a's right factor, hlu.py:178-193); computed once here with the
        same kernel and shapes, so the values are identical."""
        cap = self.L.cap
        fa_a, fb_a = self.factor_views(a)
        fa_b, fb_b = self.factor_views(b)
        t, base = self._temp(cap * cap)
        W = View(base, cap, cap, 1, cap, fa_b.cdyn, fa_a.cdyn)
        terms = [(TERM_ZERO, W, NULL_VIEW, NULL_VIEW, NULL_VIEW, 0.0, 0),
                 (TERM_GEMM, W, fa_b.T, NULL_VIEW, fb_a, 1.0, 0)]
        self.gemm_op(terms, [self.L.res(a), self.L.res(b)], [self._temp_res(t)], temps_out=[t])
        return (W, t)

    def product(self, a, b, ctx_reads=None, hw=None):
        """Low-rank product a @ b (``_multiply_lowrank``, hlu.py:261-291).
        Returns (Pair, read intervals, temps the pair lives in).  Operands are
        read-only for the whole product, so every op inside a compound product
        declares the outermost operands' intervals as its reads."""
        cap = self.L.cap
        reads = ctx_reads if ctx_reads is not None else [self.L.res(a), self.L.res(b)]
        if not _part(a) and _rk(a):
            fa, fb = self.factor_views(a)
            n = _cc(b)[1] - _cc(b)[0]
            t, base = self._temp(n * cap)
            T = View(base, n, cap, 1, n, -1, fa.cdyn)
            terms = [(TERM_ZERO, T, NULL_VIEW, NULL_VIEW, NULL_VIEW, 0.0, 0)]
            tin = []
            if hw is not None:  # T = fb_b[cols] W  (W hoisted by the caller)
                _, fbb = self.factor_views(b)
                terms.append((TERM_GEMM, T, fbb, NULL_VIEW, hw[0], 1.0, 0))
                tin = [hw[1]]
            else:
                self.terms_tmatmat(terms, T, b, fb, 1.0)
            self.gemm_op(terms, reads, [self._temp_res(t)], defer=True, temps_out=[t], temps_in=tin)
            return Pair(fa, T), reads, [t]
        if not _part(b) and _rk(b):
            fa, fb = self.factor_views(b)
            m = _rr(a)[1] - _rr(a)[0]
            t, base = self._temp(m * cap)
            T = View(base, m, cap, 1, m, -1, fa.cdyn)
            terms = [(TERM_ZERO, T, NULL_VIEW, NULL_VIEW, NULL_VIEW, 0.0, 0)]
            self.terms_matmat(terms, T, a, fa, 1.0)
            self.gemm_op(terms, reads, [self._temp_res(t)], defer=True, temps_out=[t])
            return Pair(T, fb), reads, [t]
        if not _part(a) and not _part(b):
            av, bv = self.dense_view(a), self.dense_view(b)
            m, kin, n = av.rows, av.cols, bv.cols
            # compress_dense(A @ B) as the narrower of the factor pair (A, B^T)
            # (stacked rank kin) and the formed product (I, D^T) / (D, I) (stacked
            # rank min(m, n)), preferring the block-TSQR pipeline (<= KMAX_STACK)
            # over the wide path (<= IDENT)
            if kin <= KMAX_STACK or (min(m, n) > KMAX_STACK and kin <= IDENT):
                p = self.rkt(RK_RECOMPRESS, [Pair(av, bv.T)], m, n, reads=reads, defer=True)
                return p, reads, [self._pair_temp(p)]
            if min(m, n) > IDENT:
                raise StructureError(f"dense product {m}x{kin}x{n} exceeds the truncation kernel")
            t, base = self._temp(m * n)
            D = View(base, m, n, 1, m)
            terms = [(TERM_ZERO, D, NULL_VIEW, NULL_VIEW, NULL_VIEW, 0.0, 0),
                     (TERM_GEMM, D, av, NULL_VIEW, bv, 1.0, 0)]
            self.gemm_op(terms, reads, [self._temp_res(t)], defer=True, temps_out=[t])
            I = self.L.ident_off
            if m <= n:
                part = Pair(View(I, m, m, 1, IDENT), D.T)
            else:
                part = Pair(D, View(I, n, n, 1, IDENT))
            p = self.rkt(RK_RECOMPRESS, [part], m, n, reads=reads, temps_in=[t], defer=True)
            return p, reads, [self._pair_temp(p)]
        rows = _row_cuts(a) if _part(a) else [_rr(a)]
        cols = _col_cuts(b) if _part(b) else [_cc(b)]
        if _part(a) and _part(b) and _col_cuts(a) != _row_cuts(b):
            raise StructureError("inner partitions of a product do not match")
        mids = _col_cuts(a) if _part(a) else _row_cuts(b)
        grid = []
        for i, rr in enumerate(rows):
            line = []
            for j, cc in enumerate(cols):
                acc, acc_temps = None, []
                for p, mm in enumerate(mids):
                    ap = a.child(i, p) if _part(a) else _window(a, rr, mm)
                    bp = b.child(p, j) if _part(b) else _window(b, mm, cc)
                    pp, _, tp = self.product(ap, bp, reads)
                    if acc is None:  # add_truncated(zeros, P) returns P
                        acc, acc_temps = pp, tp
                        continue
                    acc = self.rkt(RK_ADD, [acc, pp], rr[1] - rr[0], cc[1] - cc[0],
                                   reads=reads, temps_in=acc_temps + tp)
                    acc_temps = [self._pair_temp(acc)]
                line.append((acc, acc_temps))
            grid.append(line)
        if len(rows) == 1 and len(cols) == 1:
            acc, tps = grid[0][0]
            return acc, reads, tps
        m = rows[-1][1] - rows[0][0]
        n = cols[-1][1] - cols[0][0]
        parts, tin = [], []
        for i, rr in enumerate(rows):
            for j, cc in enumerate(cols):
                acc, tps = grid[i][j]
                parts.append(Pair(acc.a, acc.b, acc.sign, rr[0] - rows[0][0], cc[0] - cols[0][0]))
                tin += tps
        merged = self.rkt(RK_RECOMPRESS, parts, m, n, reads=reads, temps_in=tin)
        return merged, reads, [self._pair_temp(merged)]

    def _pair_temp(self, pair):
        return (pair.a.off >> TEMP_SHIFT) - 1

    # ------------------------------------------------------------- update
    def update(self, c, a, b, hw=None):
        """c := c - a @ b (hlu.py:568-623)."""
        if isinstance(c, HMatrix) and c.kind == LOWRANK:
            p, reads, tps = self.product(a, b, hw=hw)
            m, n = c.rows, c.cols
            ca, cb = self.factor_views(c)
            self.rkt(RK_ADD, [Pair(ca, cb), Pair(p.a, p.b, -p.sign)], m, n, out=c,
                     reads=reads + [self.L.res(c)], temps_in=tps, flop_mn=m + n)
            return
        cp, ap, bp = _part(c), _part(a), _part(b)
        if not (cp or ap or bp):
            self._update_dense(c, a, b, hw)
            return
        if hw is None and cp and not ap and not bp and _rk(a) and _rk(b):
            hw = self.hoist_inner(a, b)
        rows = _row_cuts(c) if cp else (_row_cuts(a) if ap else [_rr(c)])
        cols = _col_cuts(c) if cp else (_col_cuts(b) if bp else [_cc(c)])
        if ap and bp and _col_cuts(a) != _row_cuts(b):
            raise StructureError("inner partitions of an update do not match")
        mids = _col_cuts(a) if ap else (_row_cuts(b) if bp else [_cc(a)])
        for i, rr in enumerate(rows):
            for j, cc in enumerate(cols):
                cij = c.child(i, j) if cp else _window(c, rr, cc)
                for p, mm in enumerate(mids):
                    self.update(cij, a.child(i, p) if ap else _window(a, rr, mm),
                                b.child(p, j) if bp else _window(b, mm, cc), hw)

    def _update_dense(self, c, a, b, hw=None):
        dst = self.dense_view(c)
        m, n = dst.rows, dst.cols
        reads = [self.L.res(a), self.L.res(b)]
        writes = [self.L.res(c)]
        cap = self.L.cap
        if not _rk(a) and not _rk(b):
            av, bv = self.dense_view(a), self.dense_view(b)
            terms = [(TERM_GEMM, dst, av, NULL_VIEW, bv, -1.0, 0)]
            self.gemm_op(terms, reads, writes, (F_STATIC, 2.0 * m * n * av.cols, -1))
        elif _rk(a):
            fa, fb = self.factor_views(a)
            t, base = self._temp(n * cap)
            T = View(base, n, cap, 1, n, -1, fa.cdyn)
            terms = [(TERM_ZERO, T, NULL_VIEW, NULL_VIEW, NULL_VIEW, 0.0, 0)]
            tin = []
            if hw is not None:  # T = fb_b[cols] W  (W hoisted by the caller)
                _, fbb = self.factor_views(b)
                terms.append((TERM_GEMM, T, fbb, NULL_VIEW, hw[0], 1.0, 0))
                tin = [hw[1]]
            else:
                self.terms_tmatmat(terms, T, b, fb, 1.0)
            terms.append((TERM_GEMM, dst, fa, NULL_VIEW, T.T, -1.0, 0))
            self.gemm_op(terms, reads, writes, (F_LIN, 2.0 * (m + n) * n, -1), log_slot=fa.cdyn,
                         temps_out=[t], temps_in=tin)
        else:
            fa, fb = self.factor_views(b)
            t, base = self._temp(m * cap)
            T = View(base, m, cap, 1, m, -1, fa.cdyn)
            terms = [(TERM_ZERO, T, NULL_VIEW, NULL_VIEW, NULL_VIEW, 0.0, 0)]
            self.terms_matmat(terms, T, a, fa, 1.0)
            terms.append((TERM_GEMM, dst, T, NULL_VIEW, fb.T, -1.0, 0))
            self.gemm_op(terms, reads, writes, (F_LIN, 2.0 * (m + n) * m, -1), log_slot=fa.cdyn,
                         temps_out=[t])

    # ------------------------------------------------------------- trsm
    def trsm(self, t_view, x_view, mode, reads, writes, flop_coef, dyn):
        log = self._log() if dyn else -1
        flop = (F_LIN, float(flop_coef), log) if dyn else (F_STATIC, float(flop_coef), -1)
        self._emit(Op("trsm", (t_view, x_view, mode, log), reads, writes, False, flop))

    # --------------------------------------------------------- lower solve
    def solve_lower(self, l, b):
        """b := l^-1 b (hlu.py:400-441)."""
        if l.kind == DENSE:
            lv = self.dense_view(l)
            rd, wr = [self.L.res(l)], [self.L.res(b)]
            if b.kind == DENSE:
                self.trsm(lv, self.dense_view(b), TRSM_LOWER_UNIT, rd, wr, l.rows * l.rows * b.cols, False)
            elif b.kind == LOWRANK:
                fa, _ = self.factor_views(b)
                self.trsm(lv, fa, TRSM_LOWER_UNIT, rd, wr, l.rows * l.rows, True)
            else:
                raise StructureError("dense factor against partitioned right-hand side")
            return
        if b.kind == PARTITIONED:
            nr, nc = len(l.data), len(b.data[0])
            for i in range(nr):
                for p in range(i):
                    for j in range(nc):
                        self.update(b.child(i, j), l.child(i, p), b.child(p, j))
                for j in range(nc):
                    self.solve_lower(l.child(i, i), b.child(i, j))
            return
        self._lower_panel(l, b, b.row_range)

    def _panel_view(self, bleaf, part, axis, lo, hi):
        """Row (axis 0) or column (axis 1) panel of a leaf payload (``_Panel``, hlu.py:364)."""
        if part == "dense":
            v = self.dense_view(bleaf)
            if axis == 0:
                br = bleaf.row_range[0]
                return v.rows_slice(lo - br, hi - br)
            bc = bleaf.col_range[0]
            return v.cols_slice(lo - bc, hi - bc)
        fa, fb = self.factor_views(bleaf)
        if part == "a":
            br = bleaf.row_range[0]
            return fa.rows_slice(lo - br, hi - br)
        bc = bleaf.col_range[0]
        return fb.rows_slice(lo - bc, hi - bc)

    def _lower_panel(self, l, bleaf, span):
        part = "dense" if bleaf.kind == DENSE else "a"
        rd, wr = [self.L.res(l)], [self.L.res(bleaf)]
        if l.kind == DENSE:
            x = self._panel_view(bleaf, part, 0, *span)
            dyn = part == "a"
            coef = l.rows * l.rows * (1 if dyn else x.cols)
            self.trsm(self.dense_view(l), x, TRSM_LOWER_UNIT, rd, wr, coef, dyn)
            return
        cuts = _row_cuts(l)
        for i, ri in enumerate(cuts):
            for p, rp in enumerate(cuts[:i]):
                lip = l.child(i, p)
                dst = self._panel_view(bleaf, part, 0, *ri)
                src = self._panel_view(bleaf, part, 0, *rp)
                terms = []
                self.terms_matmat(terms, dst, lip, src, -1.0)
                if part == "a":
                    self.gemm_op(terms, [self.L.res(lip)], wr, (F_LIN, 2.0 * dst.rows * src.rows, -1),
                                 log_slot=dst.cdyn)
                else:
                    self.gemm_op(terms, [self.L.res(lip)], wr,
                                 (F_STATIC, 2.0 * dst.rows * dst.cols * src.rows, -1))
            self._lower_panel(l.child(i, i), bleaf, ri)

    # --------------------------------------------------------- upper solve
    def solve_upper(self, b, u):
        """b := b u^-1 (hlu.py:480-521)."""
        if u.kind == DENSE:
            uv = self.dense_view(u)
            rd, wr = [self.L.res(u)], [self.L.res(b)]
            if b.kind == DENSE:
                self.trsm(uv, self.dense_view(b), TRSM_RIGHT_UPPER, rd, wr, u.rows * u.rows * b.rows, False)
            elif b.kind == LOWRANK:
                _, fb = self.factor_views(b)
                self.trsm(uv, fb.T, TRSM_RIGHT_UPPER, rd, wr, u.rows * u.rows, True)
            else:
                raise StructureError("dense factor against partitioned right-hand side")
            return
        if b.kind == PARTITIONED:
            nc, nr = len(u.data[0]), len(b.data)
            for j in range(nc):
                for p in range(j):
                    for i in range(nr):
                        self.update(b.child(i, j), b.child(i, p), u.child(p, j))
                for i in range(nr):
                    self.solve_upper(b.child(i, j), u.child(j, j))
            return
        self._upper_panel(b, u, b.col_range)

    def _upper_panel(self, bleaf, u, span):
        dense = bleaf.kind == DENSE
        part, axis = ("dense", 1) if dense else ("b", 0)
        rd, wr = [self.L.res(u)], [self.L.res(bleaf)]
        if u.kind == DENSE:
            x = self._panel_view(bleaf, part, axis, *span)
            if dense:
                self.trsm(self.dense_view(u), x, TRSM_RIGHT_UPPER, rd, wr, u.rows * u.rows * x.rows, False)
            else:
                self.trsm(self.dense_view(u), x.T, TRSM_RIGHT_UPPER, rd, wr, u.rows * u.rows, True)
            return
        cuts = _col_cuts(u)
        for j, cj in enumerate(cuts):
            for p, cp in enumerate(cuts[:j]):
                upj = u.child(p, j)
                dst = self._panel_view(bleaf, part, axis, *cj)
                src = self._panel_view(bleaf, part, axis, *cp)
                terms = []
                if dense:
                    self.terms_rmatmat(terms, dst, src, upj, -1.0)
                    self.gemm_op(terms, [self.L.res(upj)], wr,
                                 (F_STATIC, 2.0 * dst.rows * dst.cols * src.cols, -1))
                else:
                    self.terms_tmatmat(terms, dst, upj, src, -1.0)
                    self.gemm_op(terms, [self.L.res(upj)], wr, (F_QUAD, 2.0 * dst.rows, -1),
                                 log_slot=dst.cdyn)
            self._upper_panel(bleaf, u.child(j, j), cj)

    # ------------------------------------------------------------- factor
    def factor(self, h):
        """H-LU (hlu.py:629-658)."""
        label = _label("lu", h.row_range, h.col_range)
        if h.kind == DENSE:
            if h.rows != h.cols:
                raise StructureError(f"LU requires a square block, got {label}")
            idx = len(self.lu_labels)
            self.lu_labels.append(label)
            op = Op("getrf", (self.dense_view(h), len(self.ops), idx), [], [self.L.res(h)], False,
                    (F_STATIC, 2.0 / 3.0 * h.rows ** 3, -1))
            self.lu_ops.append(self._emit(op))
            return
        if h.kind == LOWRANK:
            raise StructureError(f"diagonal block {label} is low-rank; expected dense")
        nb = len(h.data)
        if nb != len(h.data[0]):
            raise StructureError(f"LU requires a square grid at {label}")
        for k in range(nb):
            self.factor(h.child(k, k))
            for j in range(k + 1, nb):
                self.solve_lower(h.child(k, k), h.child(k, j))
            for i in range(k + 1, nb):
                self.solve_upper(h.child(i, k), h.child(k, k))
            for i in range(k + 1, nb):
                for j in range(k + 1, nb):
                    self.update(h.child(i, j), h.child(i, k), h.child(k, j))

    # ------------------------------------------------------ vector solves
    def forward_vector(self, l, vec_name):
        """y := L^-1 y for the pooled vector (reference route: panel walk of
        ``_solve_lower`` with an n x 1 dense leaf, hlu.py:444-477)."""
        off, rows, cols, res = self.L.extra[vec_name]
        self._vec_lower(l, View(off, rows, cols, 1, rows), l.row_range[0], (res, res + 1))

    def _vec_lower(self, l, x, base, res):
        if l.kind == DENSE:
            self.trsm(self.dense_view(l), x, TRSM_LOWER_UNIT, [self.L.res(l)], [res], 0.0, False)
            return
        cuts = _row_cuts(l)
        for i, ri in enumerate(cuts):
            for p, rp in enumerate(cuts[:i]):
                terms = []
                self.terms_matmat(terms, x.rows_slice(ri[0] - base, ri[1] - base), l.child(i, p),
                                  x.rows_slice(rp[0] - base, rp[1] - base), -1.0)
                self.gemm_op(terms, [self.L.res(l.child(i, p))], [res])
            self._vec_lower(l.child(i, i), x.rows_slice(ri[0] - base, ri[1] - base), ri[0], res)

    def backward_vector(self, u, vec_name):
        """x := U^-1 x: block back-substitution (restated; absent in the reference)."""
        off, rows, cols, res = self.L.extra[vec_name]
        self._vec_upper(u, View(off, rows, cols, 1, rows), u.row_range[0], (res, res + 1))

    # ------------------------------------------- products with h / its factors
    def matvec(self, h, x_name, y_name, tri=0):
        """y += op(h) x for pooled vectors, one term chain in the reference's
        recursion order: op = h (``hmatvec``, hmatrix.py:178-200), the unit
        lower factor (tri=1) or the upper factor (tri=2) of a factored h
        (``lower_unit_matvec`` / ``upper_matvec``, hlu.py:720-767)."""
        xo, xrows, cols, xres = self.L.extra[x_name]
        yo, yrows, _, yres = self.L.extra[y_name]
        x, y = View(xo, xrows, cols, 1, xrows), View(yo, yrows, cols, 1, yrows)
        terms = []
        if tri == 0:
            self.terms_matmat(terms, y, h, x, 1.0)
        else:
            self._terms_tri(terms, h, y, x, tri)
        self.gemm_op(terms, [self.L.res(h), (xres, xres + 1)], [(yres, yres + 1)])

    def _terms_tri(self, terms, h, y, x, tri):
        if h.kind == DENSE:
            terms.append((TERM_GEMM, y, self.dense_view(h), NULL_VIEW, x, 1.0,
                          TRI_UNIT_LOWER if tri == 1 else TRI_UPPER))
            return
        if not _part(h):
            raise StructureError("factored matrix has a low-rank diagonal block")
        for i, line in enumerate(h.data):
            for j, ch in enumerate(line):
                (i0, i1), (j0, j1) = ch.row_range, ch.col_range
                r0, c0 = h.row_range[0], h.col_range[0]
                ys, xs = y.rows_slice(i0 - r0, i1 - r0), x.rows_slice(j0 - c0, j1 - c0)
                if (j < i) if tri == 1 else (j > i):
                    self.terms_matmat(terms, ys, ch, xs, 1.0)
                elif j == i:
                    self._terms_tri(terms, ch, ys, xs, tri)

    def _vec_upper(self, u, x, base, res):
        if u.kind == DENSE:
            self.trsm(self.dense_view(u), x, TRSM_LEFT_UPPER, [self.L.res(u)], [res], 0.0, False)
            return
        cuts = _row_cuts(u)
        nb = len(cuts)
        for i in range(nb - 1, -1, -1):
            ri = cuts[i]
            for p in range(i + 1, nb):
                rp = cuts[p]
                terms = []
                self.terms_matmat(terms, x.rows_slice(ri[0] - base, ri[1] - base), u.child(i, p),
                                  x.rows_slice(rp[0] - base, rp[1] - base), -1.0)
                self.gemm_op(terms, [self.L.res(u.child(i, p))], [res])
            self._vec_upper(u.child(i, i), x.rows_slice(ri[0] - base, ri[1] - base), ri[0], res)
