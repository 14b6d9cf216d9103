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


PACK_REC = np.dtype([("host", "<u8"), ("off", "<i8"), ("rows", "<i4"), ("cols", "<i4"), ("ld", "<i4"),
                     ("host_stride", "<i4")])
assert PACK_REC.itemsize == 32


def _addr(a):
    return a.__array_interface__["data"][0]


def _c_order(a):
    return a if a.flags.c_contiguous and a.dtype == np.float64 else np.ascontiguousarray(a, dtype=np.float64)


def _native():
    from . import native_plan

    return native_plan.lib()


def _records(host, off, rows, cols):
    """Pack records (row-major host arrays -> column-major slabs, ld = rows)."""
    recs = np.empty(len(host), dtype=PACK_REC)
    recs["host"] = host
    recs["off"] = off
    recs["rows"] = rows
    recs["cols"] = cols
    recs["ld"] = rows
    recs["host_stride"] = cols
    return recs


def leaf_chunks(layout, nchunks):
    """Cut the leaves (pool offsets ascend in leaf order) into ``nchunks``
    contiguous groups of about equal payload: returns (leaf index bounds,
    pool offset bounds), both of length nchunks + 1; the last offset bound is
    ``payload_doubles`` (identity block and extras ride with the last chunk).
    Cached on the layout."""
    key = ("_leaf_chunks", int(nchunks))
    got = layout.__dict__.get(key)
    if got is not None:
        return got
    starts = np.fromiter(
        (layout.dense_off[id(lf)] if lf.kind == DENSE else layout.rk[id(lf)][0] for lf in layout.leaves),
        dtype=np.int64, count=len(layout.leaves))
    n = max(1, min(int(nchunks), len(starts)))
    total = layout.ident_off
    li = np.searchsorted(starts, total * np.arange(1, n) // n, side="left") if len(starts) else np.zeros(0, int)
    li = np.unique(np.concatenate([[0], li, [len(starts)]])).astype(np.int64)
    offs = np.concatenate([[0], starts[li[1:-1]], [layout.payload_doubles]]).astype(np.int64)
    layout.__dict__[key] = (li, offs)
    return li, offs


def _static(layout, nchunks):
    """Per-layout constants of the pack / unpack passes, per leaf group of
    ``leaf_chunks``: the dense and Rk leaves with their offsets and shapes."""
    key = ("_pack_static", int(nchunks))
    got = layout.__dict__.get(key)
    if got is not None:
        return got
    li, offs = leaf_chunks(layout, nchunks)
    groups = []
    for c in range(len(li) - 1):
        leaves = layout.leaves[li[c] : li[c + 1]]
        dn = [lf for lf in leaves if lf.kind == DENSE]
        rk = [lf for lf in leaves if lf.kind != DENSE]
        i64, i32 = np.int64, np.int32
        groups.append({
            "dense": dn, "rk": rk,
            "d_off": np.array([layout.dense_off[id(lf)] for lf in dn], dtype=i64),
            "d_rows": np.array([lf.rows for lf in dn], dtype=i32),
            "d_cols": np.array([lf.cols for lf in dn], dtype=i32),
            "a_off": np.array([layout.rk[id(lf)][0] for lf in rk], dtype=i64),
            "b_off": np.array([layout.rk[id(lf)][1] for lf in rk], dtype=i64),
            "slot": np.array([layout.rk[id(lf)][2] for lf in rk], dtype=i64),
            "r_rows": np.array([lf.rows for lf in rk], dtype=i32),
            "r_cols": np.array([lf.cols for lf in rk], dtype=i32),
        })
    layout.__dict__[key] = (groups, offs)
    return groups, offs


def _recs_np(objs, off, rows, cols):
    """Records whose ``host`` field is the array OBJECT (hlu_host_pack_np)."""
    recs = np.empty(len(objs), dtype=PACK_REC)
    recs["host"] = np.fromiter(map(id, objs), dtype=np.uint64, count=len(objs))
    recs["off"] = off
    recs["rows"] = rows
    recs["cols"] = cols
    recs["ld"] = rows
    recs["host_stride"] = cols
    return recs


_NP_FAST = None


def np_fast_path():
    """True when numpy's PyArrayObject has the layout ``hlu_host_pack_np``
    reads (self-test against arrays with known answers, once per process)."""
    global _NP_FAST
    if _NP_FAST is None:
        try:
            f = _native().hlu_host_pack_np
            src = np.arange(15.0).reshape(3, 5)
            pool = np.zeros(15)

            def rc(arr, rows, cols, unpack=0):
                r = _recs_np([arr], [0], [rows], [cols])
                return int(f(r.ctypes.data, 1, pool.ctypes.data, 1, unpack))

            ok = rc(src, 3, 5) == 0 and np.array_equal(pool, src.ravel(order="F"))
            ro = src.copy()
            ro.flags.writeable = False
            ok = ok and rc(src.astype(np.float32), 3, 5) == -1 and rc(src.T, 5, 3) == -1 and rc(src, 5, 3) == -1
            ok = ok and rc(src[:, ::2], 3, 3) == -1 and rc(ro, 3, 5, 1) == -1 and rc(ro, 3, 5, 0) == 0
            dst = np.zeros((3, 5))
            ok = ok and rc(dst, 3, 5, 1) == 0 and np.array_equal(dst, src)
            _NP_FAST = bool(ok)
        except Exception:
            _NP_FAST = False
    return _NP_FAST


def _pack_records(layout, leaves, ranks):
    """Pack records of a group of leaves; sets their ranks; returns (recs, keep-alive list)."""
    cap = layout.cap
    host, off, rows, cols, keep = [], [], [], [], []
    slots, ks = [], []
    dense_off, rk = layout.dense_off, layout.rk
    for lf in leaves:
        if lf.kind == DENSE:
            d = _c_order(lf.data)
            keep.append(d)
            host.append(_addr(d))
            off.append(dense_off[id(lf)])
            rows.append(lf.rows)
            cols.append(lf.cols)
        else:
            a_off, b_off, slot = rk[id(lf)]
            k = lf.data.k
            if k > cap:
                raise ValueError(f"rank {k} exceeds the Rk capacity {cap}")
            slots.append(slot)
            ks.append(k)
            if k == 0:
                continue
            a, b = _c_order(lf.data.a), _c_order(lf.data.b)
            keep.extend((a, b))
            host.extend((_addr(a), _addr(b)))
            off.extend((a_off, b_off))
            rows.extend((lf.rows, lf.cols))
            cols.extend((k, k))
    if slots:
        ranks[np.asarray(slots)] = np.asarray(ks, dtype=np.int32)
    return _records(host, off, rows, cols), keep


def _pack_group_fast(layout, g, ranks, pool):
    """One leaf group through hlu_host_pack_np; False when an array fails its
    check (the caller repeats the group on the general path)."""
    dn = [lf.data for lf in g["dense"]]
    lrs = [lf.data for lf in g["rk"]]
    fa = [x.a for x in lrs]
    fb = [x.b for x in lrs]
    ks = np.fromiter((x.shape[1] for x in fa), dtype=np.int32, count=len(fa))
    if len(ks) and int(ks.max()) > layout.cap:
        raise ValueError(f"rank {int(ks.max())} exceeds the Rk capacity {layout.cap}")
    if len(ks):
        ranks[g["slot"]] = ks
    nz = ks > 0
    if not nz.all():
        idx = np.nonzero(nz)[0].tolist()
        fa = [fa[i] for i in idx]
        fb = [fb[i] for i in idx]
    kz = ks[nz]
    objs = dn + fa + fb
    recs = _recs_np(objs,
                    np.concatenate([g["d_off"], g["a_off"][nz], g["b_off"][nz]]),
                    np.concatenate([g["d_rows"], g["r_rows"][nz], g["r_cols"][nz]]),
                    np.concatenate([g["d_cols"], kz, kz]))
    return int(_native().hlu_host_pack_np(recs.ctypes.data, len(recs), pool.ctypes.data, 0, 0)) == 0


def fill_pool(layout, pool, ranks, extras=None, nchunks=1, on_chunk=None):
    """Write every leaf payload into ``pool`` (float64, column-major slabs) and
    the ranks (int32) by threaded native transpose-copies (``hlu_host_pack_np``
    / ``hlu_host_pack``, include/hlu_plan.h).  With ``nchunks`` > 1 the leaves
    are packed group by group and ``on_chunk(lo, hi)`` is called as soon as the
    pool range [lo, hi) is complete, so the caller can start its host-to-device
    copy while the next group is being packed."""
    assert pool.dtype == np.float64 and pool.flags.c_contiguous
    from .planner import IDENT

    pool[layout.ident_off : layout.ident_off + IDENT * IDENT] = np.eye(IDENT).ravel()
    for name, arr in (extras or {}).items():
        off, rows, cols, _ = layout.extra[name]
        pool[off : off + rows * cols] = np.asarray(arr, dtype=float).reshape(rows, cols).ravel(order="F")
    groups, offs = _static(layout, nchunks)
    fast = np_fast_path()
    pack = _native().hlu_host_pack
    for c, g in enumerate(groups):
        if not (fast and _pack_group_fast(layout, g, ranks, pool)):
            li, _ = leaf_chunks(layout, nchunks)
            recs, keep = _pack_records(layout, layout.leaves[li[c] : li[c + 1]], ranks)
            pack(recs.ctypes.data, len(recs), pool.ctypes.data, 0)
            del keep
        if on_chunk is not None:
            on_chunk(int(offs[c]), int(offs[c + 1]))


def fill_pool_numpy(layout, pool, ranks, extras=None):
    """Reference implementation of fill_pool (per-leaf numpy copies; tests)."""
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


def _lowrank(a, b):
    """LowRank from two fresh C-contiguous float64 factors (no re-validation)."""
    x = LowRank.__new__(LowRank)
    x.a = a
    x.b = b
    return x


def read_pool(layout, pool, ranks, nchunks=1, wait_chunk=None):
    """Install the pool contents back into the layout's H-matrix: dense
    payloads in place, fresh LowRank factors for Rk leaves (threaded native
    transpose-copies).  With ``nchunks`` > 1 the leaves are read group by
    group (``leaf_chunks``) and ``wait_chunk(c)`` is called before group ``c``
    is touched (the caller waits for that range's device-to-host copy there)."""
    assert pool.dtype == np.float64 and pool.flags.c_contiguous
    ranks = np.asarray(ranks)
    empty = np.empty
    groups, _ = _static(layout, nchunks)
    fast = np_fast_path()
    lib = _native()
    for c, g in enumerate(groups):
        ks = ranks[g["slot"]].astype(np.int32) if len(g["rk"]) else np.zeros(0, np.int32)
        fa, fb = [], []
        for lf, m, n, k in zip(g["rk"], g["r_rows"].tolist(), g["r_cols"].tolist(), ks.tolist()):
            a = empty((m, k))
            b = empty((n, k))
            lf.data = _lowrank(a, b)
            fa.append(a)
            fb.append(b)
        nz = ks > 0
        if not nz.all():
            idx = np.nonzero(nz)[0].tolist()
            fa = [fa[i] for i in idx]
            fb = [fb[i] for i in idx]
        kz = ks[nz]
        dn = [lf.data for lf in g["dense"]]
        off = np.concatenate([g["d_off"], g["a_off"][nz], g["b_off"][nz]])
        rows = np.concatenate([g["d_rows"], g["r_rows"][nz], g["r_cols"][nz]])
        cols = np.concatenate([g["d_cols"], kz, kz])
        if wait_chunk is not None:
            wait_chunk(c)
        if fast:
            recs = _recs_np(dn + fa + fb, off, rows, cols)
            if int(lib.hlu_host_pack_np(recs.ctypes.data, len(recs), pool.ctypes.data, 0, 1)) == 0:
                continue
        # general path: dense payloads that are not writeable C-contiguous float64 arrays are replaced
        for i, lf in enumerate(g["dense"]):
            d = lf.data
            if not (d.flags.c_contiguous and d.dtype == np.float64 and d.flags.writeable):
                lf.data = dn[i] = np.array(d, dtype=np.float64, order="C")
        recs = _records([_addr(x) for x in dn + fa + fb], off, rows, cols)
        lib.hlu_host_unpack(recs.ctypes.data, len(recs), pool.ctypes.data, 0)


def read_pool_numpy(layout, pool, ranks):
    """Reference implementation of read_pool (per-leaf numpy copies; tests)."""
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
