"""CPU ORACLE for the H-LU hot path — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline
leg may import this module.  The product path (``paper_1906_00874_b200``)
never calls it; it runs the sm_100a kernels or fails.

This is a restatement of the reference ``hluflow`` arithmetic for the hot path,
issuing the same LAPACK/BLAS calls on the same memory layouts so that results
are bit-identical to the reference (pinned by ``tests/test_oracle_golden.py``
against fixtures produced from the reference itself by
``tests/golden/make_golden.py``):

* Rk arithmetic: ``_truncate_svd`` / ``recompress`` / ``add_truncated`` /
  ``compress_dense`` — reference ``lowrank.py:127-175``;
* dense leaf kernels: ``lu_nopivot`` (recursive halving to 48, rank-1 base,
  pivot tolerance ``1e-12 * max|A|``), ``trsm_lower_unit``,
  ``trsm_upper_right``, ``gemm_update`` — ``lowrank.py:180-261``;
* the H-recursion: factor / row-panel solve / column-panel solve / update,
  products with low-rank destinations, panel walks and the effective-flop
  counter — ``hlu.py:160-680``;
* vector solves: forward ``L y = b`` through the reference's own route
  (``solve_lower_hmatrix`` on an n x 1 dense leaf, ``hlu.py:696-700``) and
  backward ``U x = y``, which the reference lacks: restated here as block
  back-substitution mirroring ``_upper_into`` (``hlu.py:753-767``).
"""

from __future__ import annotations

import numpy as np
import scipy.linalg
from scipy.linalg.blas import dgemm

from paper_1906_00874_b200.blocks import PARTITIONED
from paper_1906_00874_b200.hmatrix import DENSE, LOWRANK, HMatrix, StructureError
from paper_1906_00874_b200.lowrank import LowRank, SingularBlockError, TruncationControl

LU_BASE = 48  # lowrank.py:180


# --------------------------------------------------------------------------
# Rk arithmetic (lowrank.py:127-175)
# --------------------------------------------------------------------------


def truncate_svd(u, s, vt, ctl):
    """k = #{s_i > eps*s_1} (0 if s_1 == 0), capped at kmax; Sigma folded left."""
    k = 0 if (s.size == 0 or s[0] == 0.0) else int(np.count_nonzero(s > ctl.eps * s[0]))
    if ctl.kmax is not None:
        k = min(k, ctl.kmax)
    return LowRank(u[:, :k] * s[:k], vt[:k, :].T)


def recompress(x, ctl):
    if x.k == 0:
        return x
    qa, ra = np.linalg.qr(x.a)
    qb, rb = np.linalg.qr(x.b)
    u, s, vt = np.linalg.svd(ra @ rb.T)
    core = truncate_svd(u, s, vt, ctl)
    return LowRank(qa @ core.a, qb @ core.b)


def compress_dense(d, ctl):
    u, s, vt = np.linalg.svd(np.asarray(d, dtype=float), full_matrices=False)
    return truncate_svd(u, s, vt, ctl)


def add_truncated(x1, x2, ctl):
    """Branches in reference order: shape, k2==0, k1==0, dense fallback
    ``k1+k2 >= min(m,n)/2``, else concatenate + recompress."""
    if x1.shape != x2.shape:
        raise ValueError(f"shape mismatch: {x1.shape} vs {x2.shape}")
    if x2.k == 0:
        return x1
    if x1.k == 0:
        return x2
    m, n = x1.shape
    if x1.k + x2.k >= min(m, n) / 2:
        return compress_dense(x1.value() + x2.value(), ctl)
    return recompress(LowRank(np.hstack((x1.a, x2.a)), np.hstack((x1.b, x2.b))), ctl)


# --------------------------------------------------------------------------
# dense leaf kernels (lowrank.py:183-261)
# --------------------------------------------------------------------------


def trsm_lower_unit(l, b):
    b[:] = scipy.linalg.solve_triangular(l, b, lower=True, unit_diagonal=True, check_finite=False)
    return b


def trsm_upper_right(u, b):
    b[:] = scipy.linalg.solve_triangular(u, b.T, lower=False, trans="T", check_finite=False).T
    return b


def gemm_update(c, a, b):
    if c.flags.c_contiguous and a.dtype == b.dtype == c.dtype == np.float64:
        dgemm(alpha=-1.0, a=b.T, b=a.T, beta=1.0, c=c.T, overwrite_c=True)
        return c
    c -= a @ b
    return c


def _pivot_fail(p, tol, path):
    raise SingularBlockError(
        f"pivot {p:.3e} below tolerance {tol:.3e} in block {path or '<root>'}", path
    )


def lu_nopivot(a, pivot_tol=None, block_path=""):
    """In-place unpivoted LU, recursive halving down to 48 then rank-1 steps."""
    n = a.shape[0]
    if a.shape[0] != a.shape[1]:
        raise ValueError("LU requires a square block")
    tol = (1e-12 * (float(np.max(np.abs(a))) if n else 0.0)) if pivot_tol is None else pivot_tol

    def small(v):
        last = v.shape[0] - 1
        for j in range(last):
            p = v[j, j]
            if abs(p) <= tol:
                _pivot_fail(p, tol, block_path)
            v[j + 1 :, j] /= p
            v[j + 1 :, j + 1 :] -= np.outer(v[j + 1 :, j], v[j, j + 1 :])
        if v.shape[0] and abs(v[last, last]) <= tol:
            _pivot_fail(v[last, last], tol, block_path)

    def halve(v):
        m = v.shape[0]
        if m <= LU_BASE:
            small(v)
            return
        h = m // 2
        halve(v[:h, :h])
        trsm_lower_unit(v[:h, :h], v[:h, h:])
        trsm_upper_right(v[:h, :h], v[h:, :h])
        gemm_update(v[h:, h:], v[h:, :h], v[:h, h:])
        halve(v[h:, h:])

    halve(a)
    return a


# --------------------------------------------------------------------------
# operands: H-nodes or windows (global coordinates) of a leaf (hlu.py:96-157)
# --------------------------------------------------------------------------


class Win:
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


def _factors(op):
    lf = _leaf(op)
    (r0, r1), (c0, c1) = _rr(op), _cc(op)
    br, bc = lf.row_range[0], lf.col_range[0]
    return lf.data.a[r0 - br : r1 - br], lf.data.b[c0 - bc : c1 - bc]


def _dense(op):
    lf = _leaf(op)
    (r0, r1), (c0, c1) = _rr(op), _cc(op)
    br, bc = lf.row_range[0], lf.col_range[0]
    return lf.data[r0 - br : r1 - br, c0 - bc : c1 - bc]


def _kids(op):
    """(child, row offset, col offset) in row-major order."""
    r0, c0 = op.row_range[0], op.col_range[0]
    for line in op.data:
        for ch in line:
            yield ch, ch.row_range[0] - r0, ch.row_range[1] - r0, ch.col_range[0] - c0, ch.col_range[1] - c0


def matmat(op, x):
    """op @ x (hlu.py:160-175)."""
    if _part(op):
        y = np.zeros((op.rows, x.shape[1]))
        for ch, i0, i1, j0, j1 in _kids(op):
            y[i0:i1] += matmat(ch, x[j0:j1])
        return y
    if _rk(op):
        a, b = _factors(op)
        return a @ (b.T @ x)
    return _dense(op) @ x


def tmatmat(op, x):
    """op.T @ x (hlu.py:178-193)."""
    if _part(op):
        y = np.zeros((op.cols, x.shape[1]))
        for ch, i0, i1, j0, j1 in _kids(op):
            y[j0:j1] += tmatmat(ch, x[i0:i1])
        return y
    if _rk(op):
        a, b = _factors(op)
        return b @ (a.T @ x)
    return _dense(op).T @ x


def gemm_into(dst, op, x):
    """dst -= op @ x (hlu.py:204-219)."""
    if _part(op):
        for ch, i0, i1, j0, j1 in _kids(op):
            gemm_into(dst[i0:i1], ch, x[j0:j1])
    elif _rk(op):
        a, b = _factors(op)
        gemm_update(dst, a, b.T @ x)
    else:
        gemm_update(dst, _dense(op), x)


def tgemm_into(dst, op, x):
    """dst -= op.T @ x (hlu.py:222-237)."""
    if _part(op):
        for ch, i0, i1, j0, j1 in _kids(op):
            tgemm_into(dst[j0:j1], ch, x[i0:i1])
    elif _rk(op):
        a, b = _factors(op)
        gemm_update(dst, b, a.T @ x)
    else:
        gemm_update(dst, _dense(op).T, x)


def rgemm_into(dst, x, op):
    """dst -= x @ op (hlu.py:240-255)."""
    if _part(op):
        for ch, i0, i1, j0, j1 in _kids(op):
            rgemm_into(dst[:, j0:j1], x[:, i0:i1], ch)
    elif _rk(op):
        a, b = _factors(op)
        gemm_update(dst, x @ a, b.T)
    else:
        gemm_update(dst, x, _dense(op))


def _row_cuts(op):
    return [line[0].row_range for line in op.data]


def _col_cuts(op):
    return [ch.col_range for ch in op.data[0]]


def _label(kind, rows, cols):
    return f"{kind}[{rows[0]}:{rows[1]})x[{cols[0]}:{cols[1]})"


# --------------------------------------------------------------------------
# the recursion (hlu.py:261-680), executed inline
# --------------------------------------------------------------------------


class Oracle:
    """Sequential H-LU exactly as the reference's inline executor runs it."""

    def __init__(self, ctl=None):
        self.ctl = ctl if ctl is not None else TruncationControl()
        self.flops = 0.0
        self.trace = None  # optional list of (event, leaf, rank) for debugging

    def _f(self, v):
        self.flops += v

    # -- products with low-rank results (hlu.py:261-309)
    def product(self, a, b):
        ctl = self.ctl
        if not _part(a) and _rk(a):
            fa, fb = _factors(a)
            return LowRank(fa, tmatmat(b, fb))
        if not _part(b) and _rk(b):
            fa, fb = _factors(b)
            return LowRank(matmat(a, fa), fb)
        if not _part(a) and not _part(b):
            return compress_dense(_dense(a) @ _dense(b), ctl)
        rows = _row_cuts(a) if _part(a) else [_rr(a)]
        cols = _col_cuts(b) if _part(b) else [_cc(b)]
        if _part(a) and _part(b) and _col_cuts(a) != _row_cuts(b):
            raise StructureError("inner partitions of a product do not match")
        mids = _col_cuts(a) if _part(a) else _row_cuts(b)
        grid = []
        for i, rr in enumerate(rows):
            line = []
            for j, cc in enumerate(cols):
                acc = LowRank.zeros(rr[1] - rr[0], cc[1] - cc[0])
                for p, mm in enumerate(mids):
                    ap = a.child(i, p) if _part(a) else _window(a, rr, mm)
                    bp = b.child(p, j) if _part(b) else _window(b, mm, cc)
                    acc = add_truncated(acc, self.product(ap, bp), ctl)
                line.append(acc)
            grid.append(line)
        if len(rows) == 1 and len(cols) == 1:
            return grid[0][0]
        return self.merge(grid, rows, cols)

    def merge(self, grid, rows, cols):
        m = rows[-1][1] - rows[0][0]
        n = cols[-1][1] - cols[0][0]
        ktot = sum(p.k for line in grid for p in line)
        u = np.zeros((m, ktot))
        v = np.zeros((n, ktot))
        at = 0
        for i, rr in enumerate(rows):
            for j, cc in enumerate(cols):
                p = grid[i][j]
                if p.k:
                    u[rr[0] - rows[0][0] : rr[1] - rows[0][0], at : at + p.k] = p.a
                    v[cc[0] - cols[0][0] : cc[1] - cols[0][0], at : at + p.k] = p.b
                    at += p.k
        return recompress(LowRank(u, v), self.ctl)

    # -- C := C - A B (hlu.py:568-623)
    def update(self, c, a, b):
        if isinstance(c, HMatrix) and c.kind == LOWRANK:
            p = self.product(a, b)
            m, n = p.shape
            c.data = add_truncated(c.data, p.neg(), self.ctl)
            self._f(2.0 * (c.data.k + p.k + 1) * (m + n) * (p.k + 1))
            return
        cp, ap, bp = _part(c), _part(a), _part(b)
        if not (cp or ap or bp):
            dst = _dense(c)
            if not _rk(a) and not _rk(b):
                av, bv = _dense(a), _dense(b)
                gemm_update(dst, av, bv)
                self._f(2.0 * dst.shape[0] * dst.shape[1] * av.shape[1])
            elif _rk(a):
                fa, fb = _factors(a)
                gemm_update(dst, fa, tmatmat(b, fb).T)
                self._f(2.0 * fa.shape[1] * (dst.shape[0] + dst.shape[1]) * dst.shape[1])
            else:
                fa, fb = _factors(b)
                gemm_update(dst, matmat(a, fa), fb.T)
                self._f(2.0 * fa.shape[1] * (dst.shape[0] + dst.shape[1]) * dst.shape[0])
            return
        rows = _row_cuts(c) if cp else (_row_cuts(a) if ap else [_rr(c)])
        cols = _col_cuts(c) if cp else (_col_cuts(b) if bp else [_cc(c)])
        if ap and bp and _col_cuts(a) != _row_cuts(b):
            raise StructureError("inner partitions of an update do not match")
        mids = _col_cuts(a) if ap else (_row_cuts(b) if bp else [_cc(a)])
        for i, rr in enumerate(rows):
            for j, cc in enumerate(cols):
                cij = c.child(i, j) if cp else _window(c, rr, cc)
                for p, mm in enumerate(mids):
                    self.update(
                        cij,
                        a.child(i, p) if ap else _window(a, rr, mm),
                        b.child(p, j) if bp else _window(b, mm, cc),
                    )

    # -- B := L^-1 B (hlu.py:400-477)
    def solve_lower(self, l, b):
        if l.kind == DENSE:
            if b.kind == DENSE:
                trsm_lower_unit(l.data, b.data)
                self._f(l.rows * l.rows * b.cols)
            elif b.kind == LOWRANK:
                lr = b.data
                a = scipy.linalg.solve_triangular(l.data, lr.a, lower=True, unit_diagonal=True)
                b.data = LowRank(a, lr.b)
                self._f(l.rows * l.rows * lr.k)
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
        part = "dense" if b.kind == DENSE else "a"
        self._lower_panel(l, (b, part, 0, b.row_range[0]), b.row_range, b.col_range)

    def _panel(self, pan, lo, hi):
        leaf, part, axis, base = pan
        arr = leaf.data if part == "dense" else (leaf.data.a if part == "a" else leaf.data.b)
        return arr[lo - base : hi - base] if axis == 0 else arr[:, lo - base : hi - base]

    def _lower_panel(self, l, pan, span, cols):
        if l.kind == DENSE:
            arr = self._panel(pan, *span)
            trsm_lower_unit(l.data, arr)
            self._f(l.rows * l.rows * arr.shape[1])
            return
        cuts = _row_cuts(l)
        for i, ri in enumerate(cuts):
            for p, rp in enumerate(cuts[:i]):
                dst = self._panel(pan, *ri)
                src = self._panel(pan, *rp)
                gemm_into(dst, l.child(i, p), src)
                self._f(2.0 * dst.shape[0] * dst.shape[1] * src.shape[0])
            self._lower_panel(l.child(i, i), pan, ri, cols)

    # -- B := B U^-1 (hlu.py:480-562)
    def solve_upper(self, b, u):
        if u.kind == DENSE:
            if b.kind == DENSE:
                trsm_upper_right(u.data, b.data)
                self._f(u.rows * u.rows * b.rows)
            elif b.kind == LOWRANK:
                lr = b.data
                fb = scipy.linalg.solve_triangular(u.data, lr.b, lower=False, trans="T")
                b.data = LowRank(lr.a, fb)
                self._f(u.rows * u.rows * lr.k)
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
        if b.kind == DENSE:
            pan = (b, "dense", 1, b.col_range[0])
        else:
            pan = (b, "b", 0, b.col_range[0])
        self._upper_panel(pan, u, b.col_range)

    def _upper_panel(self, pan, u, span):
        if u.kind == DENSE:
            arr = self._panel(pan, *span)
            if pan[1] == "b":
                arr[:] = scipy.linalg.solve_triangular(u.data, arr, lower=False, trans="T")
                self._f(u.rows * u.rows * arr.shape[1])
            else:
                trsm_upper_right(u.data, arr)
                self._f(u.rows * u.rows * arr.shape[0])
            return
        cuts = _col_cuts(u)
        for j, cj in enumerate(cuts):
            for p, cp in enumerate(cuts[:j]):
                dst = self._panel(pan, *cj)
                src = self._panel(pan, *cp)
                if pan[1] == "b":
                    tgemm_into(dst, u.child(p, j), src)
                else:
                    rgemm_into(dst, src, u.child(p, j))
                self._f(2.0 * dst.shape[0] * dst.shape[1] * src.shape[1])
            self._upper_panel(pan, u.child(j, j), cj)

    # -- LU (hlu.py:629-658)
    def factor(self, h):
        label = _label("lu", h.row_range, h.col_range)
        if h.kind == DENSE:
            if h.rows != h.cols:
                raise StructureError(f"LU requires a square block, got {label}")
            lu_nopivot(h.data, block_path=label)
            self._f(2.0 / 3.0 * h.rows**3)
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

    # -- backward substitution U x = y (restated; the reference has none)
    def solve_upper_left(self, u, x):
        """x := U^-1 x for a vector/multi-vector segment (rows of u)."""
        if u.kind == DENSE:
            x[:] = scipy.linalg.solve_triangular(u.data, x, lower=False, check_finite=False)
            return
        if u.kind != PARTITIONED:
            raise StructureError("factored matrix has a low-rank diagonal block")
        cuts = _row_cuts(u)
        base = u.row_range[0]
        nb = len(cuts)
        for i in range(nb - 1, -1, -1):
            ri = cuts[i]
            for p in range(i + 1, nb):
                rp = cuts[p]
                gemm_into(x[ri[0] - base : ri[1] - base], u.child(i, p), x[rp[0] - base : rp[1] - base])
            self.solve_upper_left(u.child(i, i), x[ri[0] - base : ri[1] - base])


# --------------------------------------------------------------------------
# public oracle entry points
# --------------------------------------------------------------------------


def hlu_factorize(h, ctl=None):
    """Factorize ``h`` in place; returns the effective-flop count."""
    if h.rows != h.cols:
        raise StructureError("H-LU requires a square matrix")
    o = Oracle(ctl)
    o.factor(h)
    return o.flops


def solve_lower_hmatrix(l, b, ctl=None):
    Oracle(ctl).solve_lower(l, b)


def solve_upper_hmatrix(b, u, ctl=None):
    Oracle(ctl).solve_upper(b, u)


def update_hmatrix(c, a, b, ctl=None):
    Oracle(ctl).update(c, a, b)


def forward_solve(h, rhs):
    """y = L^-1 rhs via the reference route: an n x 1 dense-leaf H-matrix
    right-hand side through ``solve_lower`` (panel walk)."""
    from paper_1906_00874_b200.blocks import INADMISSIBLE, BlockNode

    y = np.array(rhs, dtype=float).reshape(-1, 1)
    col = type(h.block.col)(0, 1, np.array([0.0]), np.array([0.0]))
    leaf = HMatrix(BlockNode(h.block.row, col, INADMISSIBLE), DENSE, y)
    Oracle().solve_lower(h, leaf)
    return leaf.data[:, 0].copy()


def backward_solve(h, y):
    x = np.array(y, dtype=float).reshape(-1, 1)
    Oracle().solve_upper_left(h, x)
    return x[:, 0].copy()


def hlu_solve(h, rhs):
    """x = U^-1 L^-1 rhs on a factored H-matrix."""
    return backward_solve(h, forward_solve(h, rhs))


# -- products with the matrix and its stored factors (residual probes)


def _matvec_into(h, x, y):
    """y += h x by recursion over the blocks (reference hmatrix.py:188-200)."""
    if h.kind == DENSE:
        y += h.data @ x
    elif h.kind == LOWRANK:
        y += h.data.a @ (h.data.b.T @ x)
    else:
        r0, c0 = h.row_range[0], h.col_range[0]
        for line in h.data:
            for ch in line:
                (i0, i1), (j0, j1) = ch.row_range, ch.col_range
                _matvec_into(ch, x[j0 - c0 : j1 - c0], y[i0 - r0 : i1 - r0])


def hmatvec(h, x):
    x = np.asarray(x, dtype=float)
    y = np.zeros((h.rows,) + x.shape[1:])
    _matvec_into(h, x, y)
    return y


def _tri_into(h, x, y, lower):
    """y += L x (unit lower) or U x with the stored factors (hlu.py:727-767)."""
    if h.kind == DENSE:
        y += (np.tril(h.data, -1) @ x + x) if lower else (np.triu(h.data) @ x)
        return
    if h.kind != PARTITIONED:
        raise StructureError("factored matrix has a low-rank diagonal block")
    r0 = h.row_range[0]
    for i, line in enumerate(h.data):
        for j, ch in enumerate(line):
            (i0, i1), (j0, j1) = ch.row_range, ch.col_range
            if (j < i) if lower else (j > i):
                _matvec_into(ch, x[j0 - r0 : j1 - r0], y[i0 - r0 : i1 - r0])
            elif j == i:
                _tri_into(ch, x[j0 - r0 : j1 - r0], y[i0 - r0 : i1 - r0], lower)


def lower_unit_matvec(h, x):
    x = np.asarray(x, dtype=float)
    y = np.zeros_like(x)
    _tri_into(h, x, y, True)
    return y


def upper_matvec(h, x):
    x = np.asarray(x, dtype=float)
    y = np.zeros_like(x)
    _tri_into(h, x, y, False)
    return y


def residual_probe(original, factored, seed=0, probes=10):
    """Worst ||A x - L (U x)|| / ||A x|| over random x (reference bench.py:142-152)."""
    rng = np.random.default_rng(seed)
    worst = 0.0
    for _ in range(probes):
        x = rng.standard_normal(original.cols)
        ax = hmatvec(original, x)
        lux = lower_unit_matvec(factored, upper_matvec(factored, x))
        worst = max(worst, float(np.linalg.norm(ax - lux) / np.linalg.norm(ax)))
    return worst
