"""Host <-> pool packing of an H-matrix (numpy side of the upload/download).

Dense leaves are stored column-major; an Rk leaf stores its ``a`` (m x k) and
``b`` (n x k) factors column-major in ``m x cap`` / ``n x cap`` slabs, and its
rank in the rank table.  Reading back replaces dense payloads in place (as the
reference's in-place kernels do) and installs fresh ``LowRank`` objects for Rk
leaves (as ``hlu.py:418, 498, 582`` do).
"""

from __future__ import annotations

import numpy as np

from .hmatrix import DENSE
from .lowrank import LowRank


def max_rank(layout):
    return max((lf.data.k for lf in layout.leaves if lf.kind != DENSE), default=0)


def fill_pool(layout, pool, ranks, extras=None):
    """Write every leaf payload into ``pool`` (float64) and ranks (int32)."""
    cap = layout.cap
    for lf in layout.leaves:
        if lf.kind == DENSE:
            off = layout.dense_off[id(lf)]
            pool[off : off + lf.rows * lf.cols] = np.asarray(lf.data, dtype=float).ravel(order="F")
        else:
            a_off, b_off, slot = layout.rk[id(lf)]
            k = lf.data.k
            if k > cap:
                raise ValueError(f"rank {k} exceeds the Rk capacity {cap}")
            m, n = lf.rows, lf.cols
            pool[a_off : a_off + m * k] = lf.data.a.ravel(order="F")
            pool[b_off : b_off + n * k] = lf.data.b.ravel(order="F")
            ranks[slot] = k
    from .planner import IDENT

    pool[layout.ident_off : layout.ident_off + IDENT * IDENT] = np.eye(IDENT).ravel()
    for name, arr in (extras or {}).items():
        off, rows, cols, _ = layout.extra[name]
        pool[off : off + rows * cols] = np.asarray(arr, dtype=float).reshape(rows, cols).ravel(order="F")


def read_pool(layout, pool, ranks):
    """Install the pool contents back into the layout's H-matrix."""
    for lf in layout.leaves:
        if lf.kind == DENSE:
            off = layout.dense_off[id(lf)]
            lf.data[:] = pool[off : off + lf.rows * lf.cols].reshape(lf.cols, lf.rows).T
        else:
            a_off, b_off, slot = layout.rk[id(lf)]
            k = int(ranks[slot])
            m, n = lf.rows, lf.cols
            a = pool[a_off : a_off + m * k].reshape(k, m).T
            b = pool[b_off : b_off + n * k].reshape(k, n).T
            lf.data = LowRank(a, b)


def read_extra(layout, pool, name):
    off, rows, cols, _ = layout.extra[name]
    return pool[off : off + rows * cols].reshape(cols, rows).T.copy()
