"""Independent check of a DAG schedule — TEST INFRASTRUCTURE ONLY.

From the packed descriptor arrays alone (the bytes the GPU receives), every
launch's read and write footprints in the fp64 pool (payloads and temp arena,
dynamic dimensions at their capacity bound) and in the rank table are
collected.  Two launches whose footprints conflict (write/write or
read/write) must be ordered by the launch dependencies: the earlier one has to
be an ancestor of the later one.  Nothing here uses the planner's own hazard
bookkeeping (skeleton slots, temp ids), so it also covers arena-block reuse
and the truncation workspaces.
"""

from __future__ import annotations

import numpy as np

from paper_1906_00874_b200 import ir


def _view_iv(v, out):
    off, rows, cols, rs, cs = int(v["off"]), int(v["rows"]), int(v["cols"]), int(v["rs"]), int(v["cs"])
    if rows <= 0 or cols <= 0:
        return
    out.append((off, off + (rows - 1) * abs(rs) + (cols - 1) * abs(cs) + 1))


def _rank_reads(v, out):
    for f in ("rdyn", "cdyn"):
        if int(v[f]) >= 0:
            out.append(int(v[f]))


def footprints(packed):
    """Per launch: (read intervals, write intervals, rank slots read, rank slots written)."""
    res = []
    for L in packed.launches:
        kind, count, first = int(L["kind"]), int(L["count"]), int(L["first"])
        R, W, rr, rw = [], [], [], []
        for i in range(first, first + count):
            if kind == ir.K_GETRF:
                _view_iv(packed.getrf[i]["a"], W)
            elif kind == ir.K_TRSM:
                d = packed.trsm[i]
                _view_iv(d["t"], R), _view_iv(d["x"], W)
                _rank_reads(d["t"], rr), _rank_reads(d["x"], rr)
            elif kind in (ir.K_GEMM, ir.K_GEMM_SMALL):
                d = packed.gemm[i]
                if int(d["log"]) >= 0:
                    rr.append(int(d["log_slot"]))
                for t in packed.terms[int(d["term_begin"]): int(d["term_begin"]) + int(d["term_count"])]:
                    _view_iv(t["c"], W)
                    _rank_reads(t["c"], rr)
                    if int(t["kind"]) != ir.TERM_ZERO:
                        for f in ("a", "b") + (("m",) if int(t["kind"]) == ir.TERM_TRIPLE else ()):
                            _view_iv(t[f], R)
                            _rank_reads(t[f], rr)
            elif kind == ir.K_RKT32:
                d = packed.rkt[i]
                m, n, cap = int(d["m"]), int(d["n"]), int(d["cap"])
                kb = 0
                for p in packed.parts[int(d["part_begin"]): int(d["part_begin"]) + int(d["part_count"])]:
                    _view_iv(p["a"], R), _view_iv(p["b"], R)
                    _rank_reads(p["a"], rr), _rank_reads(p["b"], rr)
                    kb += int(p["a"]["cols"])
                W.append((int(d["out_a"]), int(d["out_a"]) + m * cap))
                W.append((int(d["out_b"]), int(d["out_b"]) + n * cap))
                rw.append(int(d["out_slot"]))
                ws = ir.rkt_ws_doubles(m, n, kb)
                if ws and int(d["ws"]):
                    W.append((int(d["ws"]), int(d["ws"]) + ws))
        res.append((R, W, rr, rw))
    return res


def _merge(ivs):
    ivs = sorted(ivs)
    out = []
    for a, b in ivs:
        if out and a <= out[-1][1]:
            out[-1][1] = max(out[-1][1], b)
        else:
            out.append([a, b])
    return np.array(out, dtype=np.int64).reshape(-1, 2)


def _overlap(A, B):
    """Do two sorted, merged interval arrays intersect?"""
    if len(A) == 0 or len(B) == 0:
        return False
    # for every interval of A, the first interval of B ending after its start
    k = np.searchsorted(B[:, 1], A[:, 0], side="right")
    ok = k < len(B)
    return bool(np.any(B[k[ok], 0] < A[ok, 1]))


def ancestors(packed):
    """Boolean reachability matrix: anc[l, p] = launch p precedes launch l."""
    nl = len(packed.launches)
    anc = np.zeros((nl, nl), dtype=bool)
    for l in range(nl):
        for p in packed.dag_idx[packed.dag_ptr[l]: packed.dag_ptr[l + 1]]:
            anc[l, p] = True
            anc[l] |= anc[p]
    return anc


def violations(packed, limit=5):
    """Conflicting launch pairs the dependencies do not order (empty = ok)."""
    fp = footprints(packed)
    nl = len(fp)
    R = [_merge(f[0]) for f in fp]
    W = [_merge(f[1]) for f in fp]
    RR = [set(f[2]) for f in fp]
    RW = [set(f[3]) for f in fp]
    anc = ancestors(packed)
    bad = []
    for b in range(nl):
        for a in range(b):
            if anc[b, a]:
                continue
            why = None
            if _overlap(W[a], W[b]):
                why = "write/write"
            elif _overlap(W[a], R[b]):
                why = "write/read"
            elif _overlap(R[a], W[b]):
                why = "read/write"
            elif RW[a] & (RR[b] | RW[b]) or RW[b] & RR[a]:
                why = "rank slot"
            if why:
                bad.append((a, b, why))
                if len(bad) >= limit:
                    return bad
    return bad
