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
                ("out_a", "<i8"), ("out_b", "<i8"), ("ws", "<i8"), ("handoff", "<i4"), ("pad", "<i4")])
LAUNCH = np.dtype([("kind", "<i4"), ("count", "<i4"), ("first", "<i8"), ("smem_dim", "<i4"),
                   ("pad", "<i4")])

assert VIEW.itemsize == 32 and GETRF.itemsize == 40 and TRSM.itemsize == 72
assert TERM.itemsize == 144 and GEMM.itemsize == 16 and RKPART.itemsize == 80
assert RKT.itemsize == 64 and LAUNCH.itemsize == 24

# kinds (hlu_b200.h)
K_GETRF, K_TRSM, K_GEMM, K_RKT32, K_RKT64, K_GEMM_SMALL = 0, 1, 2, 3, 4, 5
TRSM_LOWER_UNIT, TRSM_RIGHT_UPPER, TRSM_LEFT_UPPER = 0, 1, 2
TERM_ZERO, TERM_GEMM, TERM_TRIPLE = 0, 1, 2
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


def rkt_chunk_rows(km):
    bufd = 4608 if km == 32 else 9216
    return bufd // km - km


def rkt_ws_one(m, k, ch):
    if m <= 0 or k <= 0:
        return 0
    nch = (m + ch - 1) // ch
    return nch * ((k + ch) * k + k)


def rkt_ws_doubles(m, kbound):
    """Mirror of hlu_rkt_ws_doubles (rk_kernels.cu)."""
    a = rkt_ws_one(m, min(kbound, 32), rkt_chunk_rows(32))
    b = rkt_ws_one(m, min(kbound, 64), rkt_chunk_rows(64))
    return max(a, b)
