"""Descriptor layouts shared with ``include/hlu_b200.h`` and view helpers.

Every matrix the factorization touches lives in one fp64 device pool.  A view
addresses element (i, j) at ``pool[off + i*rs + j*cs]``; a dimension may be
*dynamic*, i.e. the current rank of an Rk object (``ranks[slot]``), which is
how ranks grow and shrink in place on the device.
"""

from __future__ import annotations

import numpy as np

VIEW = np.dtype(
    [("off", "<i8"), ("rows", "<i4"), ("cols", "<i4"), ("rs", "<i4"), ("cs", "<i4"),
     ("rdyn", "<i4"), ("cdyn", "<i4")]
)
GETRF = np.dtype([("a", VIEW), ("op_id", "<i4"), ("lu_index", "<i4")])
TRSM = np.dtype([("t", VIEW), ("x", VIEW), ("mode", "<i4"), ("log", "<i4")])
TERM = np.dtype([("c", VIEW), ("a", VIEW), ("m", VIEW), ("b", VIEW), ("alpha", "<f8"),
                 ("kind", "<i4"), ("assoc", "<i4")])
GEMM = np.dtype([("term_begin", "<i4"), ("term_count", "<i4"), ("log", "<i4"), ("log_slot", "<i4")])
RKPART = np.dtype([("a", VIEW), ("b", VIEW), ("sign", "<f8"), ("roff", "<i4"), ("coff", "<i4")])
RKT = np.dtype([("mode", "<i4"), ("part_begin", "<i4"), ("part_count", "<i4"), ("m", "<i4"),
                ("n", "<i4"), ("cap", "<i4"), ("out_slot", "<i4"), ("log", "<i4"),
                ("out_a", "<i8"), ("out_b", "<i8"), ("ws", "<i8"), ("reserved", "<i4"), ("pad", "<i4")])
RKT_ITEM = np.dtype([("op", "<i4"), ("side", "<i2"), ("block", "<i2")])
LAUNCH = np.dtype([("kind", "<i4"), ("count", "<i4"), ("first", "<i8"), ("smem_dim", "<i4"),
                   ("level", "<i4")])

assert VIEW.itemsize == 32 and GETRF.itemsize == 40 and TRSM.itemsize == 72
assert TERM.itemsize == 144 and GEMM.itemsize == 16 and RKPART.itemsize == 80
# slot exchange record of a sharded plan (include/hlu_plan.h hlu_xfer)
XFER = np.dtype([("level", "<i4"), ("src", "<i4"), ("group", "<i4"), ("rank_slot", "<i4"), ("off", "<i8"),
                 ("len", "<i8"), ("boff", "<i8")])
assert RKT.itemsize == 64 and LAUNCH.itemsize == 24 and RKT_ITEM.itemsize == 8 and XFER.itemsize == 40

# kinds (hlu_b200.h)
K_GETRF, K_TRSM, K_GEMM, K_RKT32, K_RKT64, K_GEMM_SMALL = 0, 1, 2, 3, 4, 5
TRSM_LOWER_UNIT, TRSM_RIGHT_UPPER, TRSM_LEFT_UPPER = 0, 1, 2
TERM_ZERO, TERM_GEMM, TERM_TRIPLE = 0, 1, 2
TRI_NONE, TRI_UPPER, TRI_UNIT_LOWER = 0, 1, 2  # assoc of a GEMM term (include/hlu_b200.h)
RK_ADD, RK_RECOMPRESS = 0, 1

# effective-flop formulas (reference FlopCounter sites, hlu.py:408-637)
F_STATIC, F_LIN, F_RKUPD, F_QUAD = 0, 1, 2, 3


class View(tuple):
    """Immutable (off, rows, cols, rs, cs, rdyn, cdyn)."""

    __slots__ = ()

    def __new__(cls, off, rows, cols, rs, cs, rdyn=-1, cdyn=-1):
        return tuple.__new__(cls, (int(off), int(rows), int(cols), int(rs), int(cs), int(rdyn), int(cdyn)))

    off = property(lambda s: s[0])
    rows = property(lambda s: s[1])
    cols = property(lambda s: s[2])
    rs = property(lambda s: s[3])
    cs = property(lambda s: s[4])
    rdyn = property(lambda s: s[5])
    cdyn = property(lambda s: s[6])

    @property
    def T(self):
        o, r, c, rs, cs, rd, cd = self
        return View(o, c, r, cs, rs, cd, rd)

    def rows_slice(self, i0, i1):
        o, r, c, rs, cs, rd, cd = self
        assert rd < 0 and 0 <= i0 <= i1 <= r, (self, i0, i1)
        return View(o + i0 * rs, i1 - i0, c, rs, cs, rd, cd)

    def cols_slice(self, j0, j1):
        o, r, c, rs, cs, rd, cd = self
        assert cd < 0 and 0 <= j0 <= j1 <= c, (self, j0, j1)
        return View(o + j0 * cs, r, j1 - j0, rs, cs, rd, cd)


NULL_VIEW = View(0, 0, 0, 0, 0)


def colmajor(off, rows, cols, cdyn=-1):
    return View(off, rows, cols, 1, rows, -1, cdyn)


# workspace geometry of the batched truncation: mirror of csrc/rk_layout.h
RK_KMAX, RK_BR, RK_BUFA, RK_BUFB32, RK_BUFB64 = 64, 512, 16384, 3072, 8192


def rk_ch(K, bufd):
    ch = 512
    while ch > 32 and (ch + K) * K > bufd:
        ch >>= 1
    return ch


def rk_chc(K):
    return rk_ch(K, RK_BUFB32 if K <= 32 else RK_BUFB64)


def rk_chain(rows, K, ch):
    return ((rows + ch - 1) // ch) * ((K + ch) * K + K)


def rk_side_total(M, K):
    ch, chc = rk_ch(K, RK_BUFA), rk_chc(K)
    nb = (M + RK_BR - 1) // RK_BR
    last = M - (nb - 1) * RK_BR
    off_R = (nb - 1) * rk_chain(RK_BR, K, ch) + rk_chain(last, K, ch)
    srows = (nb - 1) * K + min(last, K)
    off_Z = off_R + nb * K * K + (rk_chain(srows, K, chc) if nb > 1 else 0)
    return off_Z + srows * K


RK_KMAXW = 128  # stacked rank of the wide truncation path (csrc/rk_layout.h)


def rkt_ws_doubles(m, n, kbound):
    """Mirror of hlu_rkt_ws_doubles / rk_ws_doubles (csrc/rk_layout.h)."""
    if m <= 0 or n <= 0 or kbound <= 0:
        return 0
    kb = min(kbound, RK_KMAX)
    best = 0
    for K in range(1, kb + 1):
        if K < kb and rk_ch(K + 1, RK_BUFA) == rk_ch(K, RK_BUFA) and rk_chc(K + 1) == rk_chc(K):
            continue
        best = max(best, rk_side_total(m, K) + rk_side_total(n, K))
    if kbound > RK_KMAX:
        kw = min(kbound, RK_KMAXW)
        best = max(best, (m + n) * kw + 2 * RK_KMAXW * RK_KMAXW + 3 * RK_KMAXW)
    return best


def rkt_items(m, n):
    """Mirror of hlu_rkt_items: (op, side, block) of every row block, in op order;
    returns (items structured array, item_start[count + 1])."""
    m = np.asarray(m, dtype=np.int64)
    n = np.asarray(n, dtype=np.int64)
    nbm = (m + RK_BR - 1) // RK_BR
    nbn = (n + RK_BR - 1) // RK_BR
    per = nbm + nbn
    start = np.zeros(len(m) + 1, dtype=np.int64)
    np.cumsum(per, out=start[1:])
    tot = int(start[-1])
    items = np.zeros(max(tot, 1), dtype=RKT_ITEM)
    if tot:
        op = np.repeat(np.arange(len(m), dtype=np.int64), per)
        pos = np.arange(tot, dtype=np.int64) - start[op]
        side = (pos >= nbm[op]).astype(np.int64)
        block = np.where(side == 0, pos, pos - nbm[op])
        items["op"][:tot] = op
        items["side"][:tot] = side
        items["block"][:tot] = block
    return items, start
