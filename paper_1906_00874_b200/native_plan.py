"""Binding of the native planner (``include/hlu_plan.h``, ``libhlu_plan.so``).

Flattens the H-matrix trees of a call into ``hlu_plan_node`` records (pool
offsets from the same ``Layout`` the Python planner uses) and returns the same
``schedule.Packed`` record as ``schedule.pack(Planner)``.  The two planners
are checked to produce byte-identical packed arrays
(``tests/test_native_planner.py``).
"""

from __future__ import annotations

import ctypes
import os

import numpy as np

from . import ir
from .blocks import PARTITIONED
from .hmatrix import DENSE
from .schedule import Packed

_HERE = os.path.dirname(os.path.abspath(__file__))
PLAN_LIB = os.path.join(_HERE, "libhlu_plan.so")

NODE = np.dtype([("kind", "<i4"), ("r0", "<i4"), ("r1", "<i4"), ("c0", "<i4"), ("c1", "<i4"),
                 ("nr", "<i4"), ("nc", "<i4"), ("child0", "<i4"), ("lo", "<i4"), ("hi", "<i4"),
                 ("slot", "<i4"), ("pad", "<i4"), ("off_a", "<i8"), ("off_b", "<i8")])
CMD = np.dtype([("kind", "<i4"), ("a", "<i4"), ("b", "<i4"), ("c", "<i4"), ("vec_off", "<i8"),
                ("vec_cols", "<i4"), ("pad", "<i4"), ("vec_res", "<i8"), ("vec2_off", "<i8"),
                ("vec2_res", "<i8")])
assert NODE.itemsize == 64 and CMD.itemsize == 56

(CMD_FACTOR, CMD_SOLVE_LOWER, CMD_SOLVE_UPPER, CMD_UPDATE, CMD_FWD_VEC, CMD_BWD_VEC, CMD_MATVEC,
 CMD_LOWER_MATVEC, CMD_UPPER_MATVEC) = range(9)
_MATVEC_CMDS = {"matvec": CMD_MATVEC, "lower_matvec": CMD_LOWER_MATVEC, "upper_matvec": CMD_UPPER_MATVEC}

_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(PLAN_LIB):
            raise RuntimeError(f"planner library {PLAN_LIB} missing: run `make`")
        L = ctypes.CDLL(PLAN_LIB)
        vp, i64, i32 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32
        L.hlu_plan_build.argtypes = [ctypes.POINTER(vp), vp, i64, vp, i64, i32, i64, i64, i32, i64, i32]
        L.hlu_plan_build.restype = ctypes.c_int
        L.hlu_plan_error.argtypes = [vp]
        L.hlu_plan_error.restype = ctypes.c_char_p
        L.hlu_plan_sizes.argtypes = [vp, vp]
        L.hlu_plan_copy.argtypes = [vp] * 14
        L.hlu_plan_free.argtypes = [vp]
        L.hlu_plan_level_waits.argtypes = [vp, vp, vp]
        L.hlu_plan_level_waits.restype = ctypes.c_int
        L.hlu_plan_build_sharded.argtypes = [ctypes.POINTER(vp), vp, i64, vp, i64, i32, i64, i64, i32, i64, i32,
                                             vp, i32, i32]
        L.hlu_plan_build_sharded.restype = ctypes.c_int
        L.hlu_plan_xfer.argtypes = [vp, vp]
        L.hlu_plan_xfer.restype = i64
        L.hlu_plan_op_owners.argtypes = [vp, vp]
        L.hlu_plan_op_owners.restype = ctypes.c_int
        L.hlu_plan_build_dag.argtypes = [ctypes.POINTER(vp), vp, i64, vp, i64, i32, i64, i64, i32, i64, i32, i64]
        L.hlu_plan_build_dag.restype = ctypes.c_int
        L.hlu_plan_dag.argtypes = [vp, vp, vp]
        L.hlu_plan_dag.restype = i64
        L.hlu_plan_dag_slack.argtypes = [vp, vp]
        L.hlu_plan_dag_slack.restype = ctypes.c_int
        L.hlu_host_pack.argtypes = [vp, i64, vp, ctypes.c_int]
        L.hlu_host_unpack.argtypes = [vp, i64, vp, ctypes.c_int]
        L.hlu_host_pack_np.argtypes = [vp, i64, vp, ctypes.c_int, ctypes.c_int]
        L.hlu_host_pack_np.restype = i64
        L.hlu_effective_flops.argtypes = [vp, vp, vp, i64, vp, i64, ctypes.c_int]
        L.hlu_effective_flops.restype = ctypes.c_double
        _lib = L
    return _lib


def flatten_nodes(layout):
    """Node table over every root of the layout; returns (nodes, index of id(node))."""
    recs = []
    index = {}

    def add(x):
        index[id(x)] = len(recs)
        recs.append(x)

    for root in layout.roots:
        if id(root) in index:
            continue
        add(root)
        q = [root]
        while q:
            x = q.pop(0)
            if x.kind == PARTITIONED:
                for line in x.data:
                    for ch in line:
                        add(ch)
                for line in x.data:
                    for ch in line:
                        if ch.kind == PARTITIONED:
                            q.append(ch)
    nodes = np.zeros(len(recs), dtype=NODE)
    for i, x in enumerate(recs):
        (r0, r1), (c0, c1) = x.row_range, x.col_range
        lo, hi = layout.interval[id(x)]
        rec = nodes[i]
        rec["r0"], rec["r1"], rec["c0"], rec["c1"] = r0, r1, c0, c1
        rec["lo"], rec["hi"] = lo, hi
        rec["slot"] = -1
        rec["child0"] = -1
        if x.kind == PARTITIONED:
            rec["kind"] = 2
            rec["nr"], rec["nc"] = len(x.data), len(x.data[0])
            rec["child0"] = index[id(x.data[0][0])]
        elif x.kind == DENSE:
            rec["kind"] = 0
            rec["off_a"] = layout.dense_off[id(x)]
        else:
            rec["kind"] = 1
            a_off, b_off, slot = layout.rk[id(x)]
            rec["off_a"], rec["off_b"], rec["slot"] = a_off, b_off, slot
    return nodes, index


SPLIT_ROWS = 64
PLAN_CACHE_ENV = "HLU_PLAN_CACHE"  # directory of cached plans ("" or "0": no cache)
DEFAULT_CACHE = os.path.join(os.path.expanduser("~"), ".cache", "paper_1906_00874_b200", "plans")


def cache_dir_default():
    """Plan cache directory: $HLU_PLAN_CACHE, else ~/.cache/paper_1906_00874_b200/plans;
    "" or "0" disables caching."""
    d = os.environ.get(PLAN_CACHE_ENV)
    if d is None:
        return DEFAULT_CACHE
    return None if d in ("", "0") else d
_PACKED_ARRAYS = ("getrf", "trsm", "gemm", "terms", "rkt", "parts", "launches", "flop_formula", "flop_coef",
                  "flop_log", "lu_op_ids", "op_levels", "wait_dense", "wait_rkt", "dag_ptr", "dag_idx", "dag_slack")
_PACKED_INTS = ("nlevels", "arena_doubles", "nlog", "nranks")
PLAN_FORMAT = 4  # bump when the packing (Python side) or the npz layout changes


def plan_key(nodes, cmds, scalars):
    """The native planner is a pure function of the node table, the command
    list and a few scalars; their bytes (plus the planner library's) key a
    cached plan (the analogue of the reference's save/load_hmatrix for the
    flattened schedule)."""
    import hashlib

    d = hashlib.sha256()
    d.update(f"hlu-plan-v{PLAN_FORMAT}".encode())
    d.update(nodes.tobytes())
    d.update(cmds.tobytes())
    d.update(np.asarray(scalars, dtype=np.int64).tobytes())
    d.update(_lib_digest())
    return d.hexdigest()


_LIB_DIGEST = None


def _lib_digest():
    global _LIB_DIGEST
    if _LIB_DIGEST is None:
        import hashlib

        with open(PLAN_LIB, "rb") as f:
            _LIB_DIGEST = hashlib.sha256(f.read()).digest()
    return _LIB_DIGEST


CACHE_MIN_OPS = 100_000  # the default cache keeps big plans only (planning cfg3 takes ~25 s)


def save_packed(path, packed, nops):
    rec = {f: getattr(packed, f) for f in _PACKED_ARRAYS if getattr(packed, f) is not None}
    for f in _PACKED_INTS:
        rec[f] = np.int64(getattr(packed, f))
    rec["nops"] = np.int64(nops)
    rec["lu_labels"] = np.array(packed.lu_labels, dtype=str)  # no pickled objects in the cache
    tmp = f"{path}.{os.getpid()}.tmp.npz"
    np.savez(tmp, **rec)
    os.replace(tmp, path)  # atomic: concurrent planners never see a partial file


def load_packed(path):
    with np.load(path, allow_pickle=False) as z:
        kw = {f: (z[f] if f in z.files else None) for f in _PACKED_ARRAYS}
        kw.update({f: int(z[f]) for f in _PACKED_INTS})
        kw["lu_labels"] = [str(x) for x in z["lu_labels"]]
        return Packed(**kw), int(z["nops"])


DAG_SLOT_ENV = "HLU_DAG_SLOT_US"  # time-slot width of the DAG schedule in us; "0": level schedule
# Finer slots = fewer false dependencies between launches = shorter runs, but more
# CUDA-graph nodes, whose instantiation time grows faster than linearly (cfg3:
# 20 us 3.35 s / 536 k nodes / 121 s set-up, 10 us 3.14 s / 683 k / 165-190 s,
# 5 us 2.99 s / 776 k / 222-240 s; profiles/r02/dag_slot_sweep.txt)
DAG_SLOT_US_DEFAULT = 5.0


def dag_slot_ns_default():
    """Slot width (ns) of the default single-GPU schedule: the launch DAG
    (hlu_plan_build_dag); HLU_DAG_SLOT_US=0 selects the level schedule."""
    return int(round(float(os.environ.get(DAG_SLOT_ENV, DAG_SLOT_US_DEFAULT)) * 1000.0))


def plan(layout, commands, split_rows=SPLIT_ROWS, cache_dir=None, shard=None, dag_slot_ns=None):
    """commands: list of (kind, nodes..., extras) in the planner's terms:
    ("factor", h) | ("solve_lower", l, b) | ("solve_upper", b, u) |
    ("update", c, a, b) | ("fwd", h, name) | ("bwd", h, name) |
    ("matvec" | "lower_matvec" | "upper_matvec", h, x_name, y_name)."""
    nodes, index = flatten_nodes(layout)
    cmds = np.zeros(len(commands), dtype=CMD)
    for i, c in enumerate(commands):
        kind = c[0]
        if kind == "factor":
            cmds[i] = (CMD_FACTOR, index[id(c[1])], 0, 0, 0, 0, 0, 0, 0, 0)
        elif kind == "solve_lower":
            cmds[i] = (CMD_SOLVE_LOWER, index[id(c[1])], index[id(c[2])], 0, 0, 0, 0, 0, 0, 0)
        elif kind == "solve_upper":
            cmds[i] = (CMD_SOLVE_UPPER, index[id(c[1])], index[id(c[2])], 0, 0, 0, 0, 0, 0, 0)
        elif kind == "update":
            cmds[i] = (CMD_UPDATE, index[id(c[1])], index[id(c[2])], index[id(c[3])], 0, 0, 0, 0, 0, 0)
        elif kind in ("fwd", "bwd"):
            off, rows, cols, res = layout.extra[c[2]]
            cmds[i] = (CMD_FWD_VEC if kind == "fwd" else CMD_BWD_VEC, index[id(c[1])], 0, 0, off, cols, 0, res,
                       0, 0)
        elif kind in _MATVEC_CMDS:
            xo, _, cols, xr = layout.extra[c[2]]
            yo, _, ycols, yr = layout.extra[c[3]]
            if ycols != cols:
                raise ValueError("matvec: x and y differ in width")
            cmds[i] = (_MATVEC_CMDS[kind], index[id(c[1])], 0, 0, xo, cols, 0, xr, yo, yr)
        else:
            raise ValueError(kind)
    if shard is not None:  # (slot_owner, nranks, rank): per-rank plans are not cached
        return _build(layout, nodes, cmds, split_rows, shard)
    dag = dag_slot_ns_default() if dag_slot_ns is None else int(dag_slot_ns)
    explicit = cache_dir is not None
    cache_dir = cache_dir if explicit else cache_dir_default()
    path = None
    if cache_dir:
        key = plan_key(nodes, cmds, (layout.cap, layout.ident_off, layout.nslots, layout.nrk,
                                     layout.payload_doubles, split_rows, dag))
        path = os.path.join(cache_dir, f"plan_{key[:32]}.npz")
        if os.path.exists(path):
            return load_packed(path)
    packed, nops = _build(layout, nodes, cmds, split_rows, dag_slot_ns=dag)
    if path is not None and (explicit or nops >= CACHE_MIN_OPS):
        os.makedirs(cache_dir, exist_ok=True)
        save_packed(path, packed, nops)
    return packed, nops


def _build(layout, nodes, cmds, split_rows, shard=None, dag_slot_ns=0):
    L = lib()
    h = ctypes.c_void_p()
    if shard is None and dag_slot_ns > 0:
        rc = L.hlu_plan_build_dag(ctypes.byref(h), nodes.ctypes.data, len(nodes), cmds.ctypes.data, len(cmds),
                                  layout.cap, layout.ident_off, layout.nslots, layout.nrk, layout.payload_doubles,
                                  int(split_rows), int(dag_slot_ns))
    elif shard is None:
        rc = L.hlu_plan_build(ctypes.byref(h), nodes.ctypes.data, len(nodes), cmds.ctypes.data, len(cmds),
                              layout.cap, layout.ident_off, layout.nslots, layout.nrk, layout.payload_doubles,
                              int(split_rows))
    else:
        owner, nranks, rank = shard
        owner = np.ascontiguousarray(owner, dtype=np.int32)
        if owner.shape != (layout.nslots,):
            raise ValueError("slot owner map must cover every skeleton slot")
        rc = L.hlu_plan_build_sharded(ctypes.byref(h), nodes.ctypes.data, len(nodes), cmds.ctypes.data, len(cmds),
                                      layout.cap, layout.ident_off, layout.nslots, layout.nrk,
                                      layout.payload_doubles, int(split_rows), owner.ctypes.data, int(nranks),
                                      int(rank))
    try:
        if rc != 0:
            from .hmatrix import StructureError

            raise StructureError(L.hlu_plan_error(h).decode())
        sz = np.zeros(14, dtype=np.int64)
        L.hlu_plan_sizes(h, sz.ctypes.data)
        ng, nt, nm, nterm, nr, npart, nl, nops, nlev, arena, nlog, nrank, nlu, ntemp = (int(x) for x in sz)

        def arr(n, dt):
            return np.zeros(max(n, 1), dtype=dt)

        getrf, trsm, gemm = arr(ng, ir.GETRF), arr(nt, ir.TRSM), arr(nm, ir.GEMM)
        terms, rkt, parts = arr(nterm, ir.TERM), arr(nr, ir.RKT), arr(npart, ir.RKPART)
        launches = arr(nl, ir.LAUNCH)
        ff = np.zeros(nops, dtype=np.int32)
        fc = np.zeros(nops, dtype=np.float64)
        fl = np.zeros(nops, dtype=np.int64)
        lu_ops = np.zeros(max(nlu, 1), dtype=np.int64)
        lu_nodes = np.zeros(max(nlu, 1), dtype=np.int64)
        lv = np.zeros(nops, dtype=np.int64)
        L.hlu_plan_copy(h, getrf.ctypes.data, trsm.ctypes.data, gemm.ctypes.data, terms.ctypes.data,
                        rkt.ctypes.data, parts.ctypes.data, launches.ctypes.data, ff.ctypes.data,
                        fc.ctypes.data, fl.ctypes.data, lu_ops.ctypes.data, lu_nodes.ctypes.data, lv.ctypes.data)
        wd = np.full(max(nlev, 1), -1, dtype=np.int32)
        wr = np.full(max(nlev, 1), -1, dtype=np.int32)
        if L.hlu_plan_level_waits(h, wd.ctypes.data, wr.ctypes.data) != 0:
            wd = wr = None
        dag_ptr = dag_idx = dag_slack = None
        ne = int(L.hlu_plan_dag(h, None, None))
        if ne >= 0:
            dag_ptr = np.zeros(nl + 1, dtype=np.int64)
            dag_idx = np.zeros(max(ne, 1), dtype=np.int32)
            L.hlu_plan_dag(h, dag_ptr.ctypes.data, dag_idx.ctypes.data)
            dag_idx = dag_idx[:ne]
            dag_slack = np.zeros(max(nl, 1), dtype=np.int64)
            L.hlu_plan_dag_slack(h, dag_slack.ctypes.data)
        xfer = mask = None
        if shard is not None:
            xfer = np.zeros(max(int(L.hlu_plan_xfer(h, None)), 1), dtype=ir.XFER)
            nx = int(L.hlu_plan_xfer(h, xfer.ctypes.data))
            xfer = xfer[:nx]
            mask = np.zeros(nops, dtype=np.uint64)
            L.hlu_plan_op_owners(h, mask.ctypes.data)
            wd = wr = None  # level barriers: the exchange steps sit between levels
    finally:
        L.hlu_plan_free(h)
    labels = []
    for k in lu_nodes[:nlu]:
        r = nodes[int(k)]
        labels.append(f"lu[{r['r0']}:{r['r1']})x[{r['c0']}:{r['c1']})")
    return Packed(
        getrf=getrf, trsm=trsm, gemm=gemm, terms=terms, rkt=rkt, parts=parts,
        launches=launches, nlevels=nlev, arena_doubles=arena,
        flop_formula=ff.astype(np.int64), flop_coef=fc, flop_log=fl, nlog=max(nlog, 1),
        nranks=max(nrank, 1), lu_op_ids=lu_ops[:nlu], lu_labels=labels, op_levels=lv,
        wait_dense=wd, wait_rkt=wr, xfer=xfer, op_mask=mask,
        shard=None if shard is None else (int(shard[1]), int(shard[2])),
        dag_ptr=dag_ptr, dag_idx=dag_idx, dag_slack=dag_slack,
    ), nops
