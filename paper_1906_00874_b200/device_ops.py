"""Single-block entry points of the reference ``lowrank`` module on the GPU.

``add_truncated``, ``recompress``, ``compress_dense``, ``lu_nopivot``,
``trsm_lower_unit``, ``trsm_upper_right`` and ``gemm_update`` keep the
reference signatures (``lowrank.py:137-261``) and run as a one-descriptor
launch of the same batched kernels the factorization uses.  They are meant
for API parity and unit tests; the factorization itself never goes through
here.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _native, ir
from .lowrank import LowRank, SingularBlockError, TruncationControl

INT32_MAX = np.iinfo(np.int32).max


class _Scratch:
    """A tiny pool + ctx for one launch."""

    def __init__(self, doubles, nranks, ctl):
        import torch

        if not torch.cuda.is_available():
            raise RuntimeError("device_ops need a CUDA device (sm_100a); no CPU fallback")
        self.torch = torch
        self.host = np.zeros(max(doubles, 1))
        self.nranks = max(nranks, 1)
        self.hranks = np.zeros(self.nranks, dtype=np.int32)
        self.top = 0
        self.ctl = ctl

    def put(self, arr):
        """Column-major copy of a 2-d array; returns its offset."""
        arr = np.asarray(arr, dtype=float)
        off = self.top
        self.host[off : off + arr.size] = arr.ravel(order="F")
        self.top += max(arr.size, 1)
        return off

    def reserve(self, n):
        off = self.top
        self.top += max(n, 1)
        return off

    def go(self, fn):
        t = self.torch
        self.pool = t.from_numpy(self.host).cuda()
        self.ranks = t.from_numpy(self.hranks).cuda()
        self.log = t.zeros(8, dtype=t.int32, device="cuda")
        self.err = t.tensor([0, INT32_MAX, 0, 0], dtype=t.int32, device="cuda")
        self.dlog = t.zeros(2, dtype=t.float64, device="cuda")
        ctl = self.ctl or TruncationControl()
        ctx = _native.HluCtx(self.pool.data_ptr(), self.ranks.data_ptr(), self.log.data_ptr(),
                             self.err.data_ptr(), self.dlog.data_ptr(), float(ctl.eps),
                             -1 if ctl.kmax is None else int(ctl.kmax), 0)
        stream = ctypes.c_void_p(t.cuda.current_stream().cuda_stream)
        fn(_native.lib(), ctypes.byref(ctx), stream)
        t.cuda.synchronize()
        self.out = self.pool.cpu().numpy()
        self.out_ranks = self.ranks.cpu().numpy()
        self.out_err = self.err.cpu().numpy()
        self.out_dlog = self.dlog.cpu().numpy()

    def get(self, off, rows, cols):
        return self.out[off : off + rows * cols].reshape(cols, rows).T.copy()


def _dev(torch, rec):
    return torch.from_numpy(np.ascontiguousarray(rec).view(np.uint8)).cuda()


def _truncate_parts(parts_pairs, m, n, ctl, mode, signs=None):
    """Run one RKT op over the given LowRank parts; returns a LowRank."""
    ks = [p.k for p in parts_pairs]
    K = sum(ks)
    cap = max(K, 1)
    if ctl is not None and ctl.eps == 0.0 and mode == ir.RK_ADD:
        cap = max(cap, min(m, n))  # the dense-fallback route keeps up to min(m, n) columns
    kb = K
    ws = ir.rkt_ws_doubles(m, n, kb)
    size = sum(p.a.size + p.b.size for p in parts_pairs) + (m + n) * cap + ws + 16
    S = _Scratch(size, len(parts_pairs) + 1, ctl)
    recs = []
    for i, p in enumerate(parts_pairs):
        ao, bo = S.put(p.a), S.put(p.b)
        S.hranks[i] = p.k
        s = 1.0 if signs is None else signs[i]
        recs.append(((ao, m, cap, 1, m, -1, i), (bo, n, cap, 1, n, -1, i), s, 0, 0))
    out_a = S.reserve(m * cap)
    out_b = S.reserve(n * cap)
    wso = S.reserve(ws)
    slot = len(parts_pairs)
    parts = np.zeros(len(recs), dtype=ir.RKPART)
    parts[:] = recs
    d = np.zeros(1, dtype=ir.RKT)
    d[0] = (mode, 0, len(recs), m, n, cap, slot, 0, out_a, out_b, wso, 0, 0)
    t = None

    def fn(lib, ctx, stream):
        nonlocal t
        import torch

        dd, dp = _dev(torch, d), _dev(torch, parts)
        launches = np.zeros(1, dtype=ir.LAUNCH)
        launches[0] = (ir.K_RKT32, 1, 0, 0, 0)
        sc, keep = _native.rkt_scratch(torch, dd.device, d, launches)
        t = (dd, dp, keep)
        _native.check(lib.hlu_rk_update_batched_f64(ctx, dd.data_ptr(), dp.data_ptr(), 1, ctypes.byref(sc), stream),
                      "hlu_rk_update_batched_f64")

    S.go(fn)
    if S.out_err[2]:
        raise ValueError(f"stacked rank {K} exceeds the kernel limit (128; eps = 0 dense fallback: blocks up to 64 x 64)")
    k = int(S.out_ranks[slot])
    return LowRank(S.get(out_a, m, k), S.get(out_b, n, k))


def add_truncated(x1: LowRank, x2: LowRank, ctl: TruncationControl) -> LowRank:
    if x1.shape != x2.shape:
        raise ValueError(f"shape mismatch: {x1.shape} vs {x2.shape}")
    m, n = x1.shape
    return _truncate_parts([x1, x2], m, n, ctl, ir.RK_ADD)


def recompress(x: LowRank, ctl: TruncationControl) -> LowRank:
    if x.k == 0:
        return x
    m, n = x.shape
    return _truncate_parts([x], m, n, ctl, ir.RK_RECOMPRESS)


def compress_dense(d, ctl: TruncationControl) -> LowRank:
    """Truncated SVD of a dense block, as the factor pair (d, I) (K = cols)."""
    d = np.asarray(d, dtype=float)
    m, n = d.shape
    if m == 0 or n == 0:
        return LowRank(np.zeros((m, 0)), np.zeros((n, 0)))
    if n <= m:
        return _truncate_parts([LowRank(d, np.eye(n))], m, n, ctl, ir.RK_RECOMPRESS)
    return _truncate_parts([LowRank(np.eye(m), d.T)], m, n, ctl, ir.RK_RECOMPRESS)


def lu_nopivot(a, pivot_tol=None, block_path=""):
    """In-place unpivoted LU (pivot_tol other than the default is not supported)."""
    if a.shape[0] != a.shape[1]:
        raise ValueError("LU requires a square block")
    if pivot_tol is not None:
        raise NotImplementedError("the device LU uses the reference default tolerance")
    n = a.shape[0]
    S = _Scratch(n * n + 1, 1, None)
    off = S.put(a)
    d = np.zeros(1, dtype=ir.GETRF)
    d[0] = ((off, n, n, 1, n, -1, -1), 0, 0)

    def fn(lib, ctx, stream):
        import torch

        dd = _dev(torch, d)
        _native.check(lib.hlu_getrf_batched_f64(ctx, dd.data_ptr(), 1, n, stream), "hlu_getrf_batched_f64")
        torch.cuda.synchronize()

    S.go(fn)
    if S.out_err[1] != INT32_MAX:
        p, tol = S.out_dlog
        raise SingularBlockError(
            f"pivot {p:.3e} below tolerance {tol:.3e} in block {block_path or '<root>'}", block_path
        )
    a[:] = S.get(off, n, n)
    return a


def _trsm(t, x, mode):
    n = t.shape[0]
    S = _Scratch(t.size + x.size + 2, 1, None)
    to = S.put(t)
    xo = S.put(x)
    r, c = x.shape
    d = np.zeros(1, dtype=ir.TRSM)
    d[0] = ((to, n, n, 1, n, -1, -1), (xo, r, c, 1, r, -1, -1), mode, -1)

    def fn(lib, ctx, stream):
        import torch

        dd = _dev(torch, d)
        _native.check(lib.hlu_trsm_batched_f64(ctx, dd.data_ptr(), 1, n, stream), "hlu_trsm_batched_f64")
        torch.cuda.synchronize()

    S.go(fn)
    x[:] = S.get(xo, r, c)
    return x


def trsm_lower_unit(l, b):
    return _trsm(np.asarray(l, float), b, ir.TRSM_LOWER_UNIT)


def trsm_upper_right(u, b):
    return _trsm(np.asarray(u, float), b, ir.TRSM_RIGHT_UPPER)


def trsm_upper_left(u, b):
    return _trsm(np.asarray(u, float), b, ir.TRSM_LEFT_UPPER)


def gemm_update(c, a, b):
    """c <- c - a @ b in place."""
    m, n = c.shape
    k = a.shape[1]
    S = _Scratch(c.size + a.size + b.size + 3, 1, None)
    co, ao, bo = S.put(c), S.put(a), S.put(b)
    terms = np.zeros(1, dtype=ir.TERM)
    terms[0] = ((co, m, n, 1, m, -1, -1), (ao, m, k, 1, m, -1, -1), (0, 0, 0, 0, 0, -1, -1),
                (bo, k, n, 1, k, -1, -1), -1.0, ir.TERM_GEMM, 0)
    g = np.zeros(1, dtype=ir.GEMM)
    g[0] = (0, 1, -1, -1)

    def fn(lib, ctx, stream):
        import torch

        dg, dt = _dev(torch, g), _dev(torch, terms)
        _native.check(lib.hlu_gemm_batched_f64(ctx, dg.data_ptr(), dt.data_ptr(), 1, stream),
                      "hlu_gemm_batched_f64")
        torch.cuda.synchronize()

    S.go(fn)
    c[:] = S.get(co, m, n)
    return c
