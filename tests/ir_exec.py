"""CPU executor of the packed device IR — TEST INFRASTRUCTURE ONLY.

Runs exactly the descriptor arrays and launch list the GPU receives, with
numpy/LAPACK in place of the kernels, so the planner, the level schedule
(hazards), the temp arena and the flop logging can be validated against the
oracle on a machine without a GPU.  Ops inside a launch are run in reverse
order to expose any intra-level hazard.
"""

from __future__ import annotations

import numpy as np
import scipy.linalg
from numpy.lib.stride_tricks import as_strided

from paper_1906_00874_b200 import ir


class CpuMachine:
    def __init__(self, pool, ranks, nlog, eps, kmax):
        self.pool = pool
        self.ranks = ranks
        self.log = np.zeros(nlog, dtype=np.int32)
        self.err = np.array([0, np.iinfo(np.int32).max, 0, 0], dtype=np.int32)
        self.dlog = {}
        self.eps = eps
        self.kmax = -1 if kmax is None else kmax

    def v(self, rec):
        off, rows, cols, rs, cs, rdyn, cdyn = (int(x) for x in rec)
        if rdyn >= 0:
            rows = int(self.ranks[rdyn])
        if cdyn >= 0:
            cols = int(self.ranks[cdyn])
        if rows == 0 or cols == 0:
            return np.zeros((rows, cols))
        return as_strided(self.pool[off:], shape=(rows, cols), strides=(rs * 8, cs * 8))

    # -- kernels
    def getrf(self, d):
        a = self.v(d["a"])
        w = a.copy()
        n = w.shape[0]
        tol = 1e-12 * (np.abs(w).max() if n else 0.0)
        for j in range(n):
            p = w[j, j]
            if abs(p) <= tol:
                self.err[1] = min(self.err[1], int(d["op_id"]))
                self.dlog[int(d["lu_index"])] = (p, tol)
                break
            w[j + 1 :, j] /= p
            w[j + 1 :, j + 1 :] -= np.outer(w[j + 1 :, j], w[j, j + 1 :])
        a[:] = w

    def trsm(self, d):
        t = self.v(d["t"])
        x = self.v(d["x"])
        mode = int(d["mode"])
        if int(d["log"]) >= 0:
            self.log[int(d["log"])] = x.shape[0] if mode == 1 else x.shape[1]
        if x.size == 0:
            return
        try:
            if mode == ir.TRSM_LOWER_UNIT:
                x[:] = scipy.linalg.solve_triangular(t, x, lower=True, unit_diagonal=True)
            elif mode == ir.TRSM_RIGHT_UPPER:
                x[:] = scipy.linalg.solve_triangular(t, x.T, lower=False, trans="T").T
            else:
                x[:] = scipy.linalg.solve_triangular(t, x, lower=False)
        except np.linalg.LinAlgError:  # singular factor after a failed LU: garbage, like the GPU
            x[:] = np.nan

    def gemm(self, d, terms):
        if int(d["log"]) >= 0:
            self.log[int(d["log"])] = self.ranks[int(d["log_slot"])]
        for t in terms[int(d["term_begin"]) : int(d["term_begin"]) + int(d["term_count"])]:
            c = self.v(t["c"])
            kind = int(t["kind"])
            if kind == ir.TERM_ZERO:
                c[:] = 0.0
                continue
            if c.size == 0:
                continue
            a, b = self.v(t["a"]), self.v(t["b"])
            if kind == ir.TERM_GEMM:
                tri = int(t["assoc"])
                if tri == ir.TRI_UPPER:
                    a = np.triu(a)
                elif tri == ir.TRI_UNIT_LOWER:
                    a = np.tril(a, -1) + np.eye(a.shape[0], a.shape[1])
                c += t["alpha"] * (a @ b)
            else:
                m = self.v(t["m"])
                if int(t["assoc"]) == 0:
                    c += t["alpha"] * (a @ (m @ b))
                else:
                    c += t["alpha"] * ((a @ m) @ b)

    def rkt(self, d, parts):
        pts = parts[int(d["part_begin"]) : int(d["part_begin"]) + int(d["part_count"])]
        P = [(self.v(p["a"]), self.v(p["b"]), float(p["sign"]), int(p["roff"]), int(p["coff"])) for p in pts]
        m, n, cap = int(d["m"]), int(d["n"]), int(d["cap"])
        log = int(d["log"])
        oa = as_strided(self.pool[int(d["out_a"]) :], shape=(m, cap), strides=(8, m * 8))
        ob = as_strided(self.pool[int(d["out_b"]) :], shape=(n, cap), strides=(8, n * 8))
        slot = int(d["out_slot"])
        ks = [p[0].shape[1] for p in P]
        K = sum(ks)

        def finish(a, b, k):
            if k > cap:
                self.err[0] += 1
                k = cap
            oa[:, :k] = a[:, :k]
            ob[:, :k] = b[:, :k]
            self.ranks[slot] = k
            if log >= 0:
                self.log[log + 2] = k

        if int(d["mode"]) == ir.RK_ADD:
            if log >= 0:
                self.log[log], self.log[log + 1] = ks[0], ks[1]
            if ks[1] == 0 or ks[0] == 0:
                a, b, s, _, _ = P[0] if ks[1] == 0 else P[1]
                finish((s * a).copy(), b.copy(), a.shape[1])
                return
        else:
            if log >= 0:
                self.log[log], self.log[log + 1] = K, 0
            if K == 0:
                self.ranks[slot] = 0
                if log >= 0:
                    self.log[log + 2] = 0
                return
        X = np.zeros((m, K))
        Y = np.zeros((n, K))
        c0 = 0
        for (a, b, s, ro, co), k in zip(P, ks):
            X[ro : ro + a.shape[0], c0 : c0 + k] = s * a
            Y[co : co + b.shape[0], c0 : c0 + k] = b
            c0 += k
        qa, ra = np.linalg.qr(X)
        qb, rb = np.linalg.qr(Y)
        u, sv, vt = np.linalg.svd(ra @ rb.T)
        k = 0 if (sv.size == 0 or sv[0] == 0.0) else int(np.count_nonzero(sv > self.eps * sv[0]))
        if self.kmax >= 0:
            k = min(k, self.kmax)
        finish(qa @ (u[:, :k] * sv[:k]), qb @ vt[:k].T, k)

    def run(self, packed, launches=None):
        for L in packed.launches if launches is None else launches:
            kind, count, first = int(L["kind"]), int(L["count"]), int(L["first"])
            if count == 0:
                continue
            rng = range(first + count - 1, first - 1, -1)
            if kind == ir.K_GETRF:
                for i in rng:
                    self.getrf(packed.getrf[i])
            elif kind == ir.K_TRSM:
                for i in rng:
                    self.trsm(packed.trsm[i])
            elif kind in (ir.K_GEMM, ir.K_GEMM_SMALL):
                for i in rng:
                    self.gemm(packed.gemm[i], packed.terms)
            elif kind == ir.K_RKT32:  # RKT64 launches cover the same ops
                for i in rng:
                    self.rkt(packed.rkt[i], packed.parts)


def xfer_groups(xfer):
    """(level, src, group) -> record indices, in record order."""
    out = {}
    for i, r in enumerate(xfer):
        out.setdefault((int(r["level"]), int(r["src"]), int(r["group"])), []).append(i)
    return out


def run_sharded(M, packed, rank, dist):
    """The sharded schedule exactly as the GPU runtime replays it
    (runtime.cu, hlu_schedule_create_sharded): every level's launches of this
    rank, then the level's exchange groups in order -- the source packs the
    slots (payload, then the rank as a double) into the group buffer, one
    broadcast, the other ranks unpack -- and after the last level the final
    gather; the flop log is max-reduced."""
    import torch

    lv = packed.launches["level"].astype(np.int64)
    groups = xfer_groups(packed.xfer)
    by_level = {}
    for key, idx in groups.items():
        by_level.setdefault(key[0], []).append((key, idx))
    for level in range(packed.nlevels + 1):
        if level < packed.nlevels:
            M.run(packed, packed.launches[lv == level])
        for (lvl, src, g), idx in sorted(by_level.get(level, []), key=lambda kv: kv[0]):
            recs = packed.xfer[idx]
            size = int((recs["len"] + 1).sum())
            buf = np.zeros(size)
            if rank == src:
                for r in recs:
                    o, n, b = int(r["off"]), int(r["len"]), int(r["boff"])
                    buf[b : b + n] = M.pool[o : o + n]
                    if int(r["rank_slot"]) >= 0:
                        buf[b + n] = M.ranks[int(r["rank_slot"])]
            t = torch.from_numpy(buf)
            dist.broadcast(t, src)
            if rank != src:
                buf = t.numpy()
                for r in recs:
                    o, n, b = int(r["off"]), int(r["len"]), int(r["boff"])
                    M.pool[o : o + n] = buf[b : b + n]
                    if int(r["rank_slot"]) >= 0:
                        M.ranks[int(r["rank_slot"])] = int(buf[b + n])
    log = torch.from_numpy(M.log.astype(np.int64))
    dist.all_reduce(log, op=dist.ReduceOp.MAX)
    M.log[:] = log.numpy().astype(np.int32)
