"""ctypes binding of the C ABI (``include/hlu_b200.h``).

The library is built in-tree (``make`` / ``__graft_entry__.build()``) as
``paper_1906_00874_b200/libhlu_b200.so``.  There is no fallback: if it is
missing, every device entry point raises.
"""

from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# HLU_LIB selects a diagnostics build of the same library (e.g. libhlu_b200_prof.so)
LIB_PATH = os.path.join(_HERE, os.environ.get("HLU_LIB", "libhlu_b200.so"))

SYMBOLS = (
    "hlu_getrf_batched_f64",
    "hlu_trsm_batched_f64",
    "hlu_gemm_batched_f64",
    "hlu_gemm_small_batched_f64",
    "hlu_rk_update_batched_f64",
    "hlu_rkt_phases",
    "hlu_rkt_phase",
    "hlu_rkt_items",
    "hlu_rkt_ws_doubles",
    "hlu_schedule_create",
    "hlu_schedule_create_chains",
    "hlu_schedule_create_dag",
    "hlu_schedule_graph_nodes",
    "hlu_schedule_launch",
    "hlu_schedule_destroy",
    "hlu_schedule_stamps",
    "hlu_version",
    "hlu_device_check",
    "hlu_debug_sweeps",
    "hlu_debug_bprof",
    "hlu_comm_available",
    "hlu_comm_unique_id",
    "hlu_comm_init",
    "hlu_comm_destroy",
    "hlu_schedule_create_sharded",
    "hlu_xfer_staging_doubles",
    "hlu_xfer_group",
    "hlu_asm_dense_f64",
    "hlu_asm_cheb_f64",
    "hlu_asm_aca_f64",
)


class HluCtx(ctypes.Structure):
    _fields_ = [
        ("pool", ctypes.c_void_p),
        ("ranks", ctypes.c_void_p),
        ("log", ctypes.c_void_p),
        ("err", ctypes.c_void_p),
        ("dlog", ctypes.c_void_p),
        ("eps", ctypes.c_double),
        ("kmax", ctypes.c_int32),
        ("pad", ctypes.c_int32),
    ]


class HluRktScratch(ctypes.Structure):
    _fields_ = [
        ("counts", ctypes.c_void_p),
        ("list", ctypes.c_void_p),
        ("items", ctypes.c_void_p),
        ("max_ops", ctypes.c_int64),
        ("max_items", ctypes.c_int64),
    ]


_lib = None


def lib():
    """Load the sm_100a library (raises when it has not been built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(
            f"CUDA library {LIB_PATH} is missing: run `make` (or __graft_entry__.build()); "
            "there is no CPU fallback"
        )
    L = ctypes.CDLL(LIB_PATH)
    vp, i32, i64 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64
    L.hlu_getrf_batched_f64.argtypes = [ctypes.POINTER(HluCtx), vp, i32, i32, vp]
    L.hlu_trsm_batched_f64.argtypes = [ctypes.POINTER(HluCtx), vp, i32, i32, vp]
    L.hlu_gemm_batched_f64.argtypes = [ctypes.POINTER(HluCtx), vp, vp, i32, vp]
    L.hlu_gemm_small_batched_f64.argtypes = [ctypes.POINTER(HluCtx), vp, vp, i32, vp]
    sp = ctypes.POINTER(HluRktScratch)
    L.hlu_rk_update_batched_f64.argtypes = [ctypes.POINTER(HluCtx), vp, vp, i32, sp, vp]
    L.hlu_rkt_phases.argtypes = [ctypes.POINTER(HluCtx), vp, vp, i64, i32, sp, i32, vp, vp]
    L.hlu_rkt_phase.argtypes = [ctypes.POINTER(HluCtx), vp, vp, i64, i32, sp, i32, i32, vp]
    L.hlu_rkt_items.argtypes = [vp, i32, vp]
    L.hlu_rkt_items.restype = i64
    L.hlu_rkt_ws_doubles.argtypes = [i32, i32, i32]
    L.hlu_rkt_ws_doubles.restype = i64
    L.hlu_debug_sweeps.argtypes = [i32]
    L.hlu_debug_sweeps.restype = i64
    L.hlu_debug_bprof.argtypes = [vp, i32]
    L.hlu_debug_bprof.restype = ctypes.c_int
    L.hlu_schedule_create.argtypes = [ctypes.POINTER(vp), ctypes.POINTER(HluCtx), vp, i64,
                                      vp, vp, vp, vp, vp, vp, sp, i32, vp]
    L.hlu_schedule_create_chains.argtypes = [ctypes.POINTER(vp), ctypes.POINTER(HluCtx), vp, i64,
                                             vp, vp, vp, vp, vp, vp, sp, vp, vp, i64, i32, vp]
    L.hlu_schedule_create_dag.argtypes = [ctypes.POINTER(vp), ctypes.POINTER(HluCtx), vp, i64,
                                          vp, vp, vp, vp, vp, vp, sp, vp, vp, vp, vp, vp, vp]
    L.hlu_schedule_create_dag.restype = ctypes.c_int
    L.hlu_schedule_graph_nodes.argtypes = [vp]
    L.hlu_schedule_graph_nodes.restype = i64
    L.hlu_schedule_launch.argtypes = [vp, vp]
    L.hlu_schedule_destroy.argtypes = [vp]
    L.hlu_schedule_stamps.argtypes = [vp, vp]
    L.hlu_schedule_stamps.restype = i64
    L.hlu_comm_available.restype = ctypes.c_int
    L.hlu_comm_unique_id.argtypes = [vp]
    L.hlu_comm_unique_id.restype = ctypes.c_int
    L.hlu_comm_init.argtypes = [ctypes.POINTER(vp), vp, ctypes.c_int, ctypes.c_int]
    L.hlu_comm_init.restype = ctypes.c_int
    L.hlu_comm_destroy.argtypes = [vp]
    L.hlu_comm_destroy.restype = ctypes.c_int
    L.hlu_schedule_create_sharded.argtypes = [ctypes.POINTER(vp), ctypes.POINTER(HluCtx), vp, i64,
                                              vp, vp, vp, vp, vp, vp, sp, vp, vp, vp, i64, i64, i64, vp, i32, vp]
    L.hlu_schedule_create_sharded.restype = ctypes.c_int
    L.hlu_xfer_staging_doubles.argtypes = [vp, i64]
    L.hlu_xfer_staging_doubles.restype = i64
    L.hlu_xfer_group.argtypes = [vp, vp, vp, vp, ctypes.c_int, ctypes.c_int, i64, vp, vp]
    L.hlu_xfer_group.restype = ctypes.c_int
    L.hlu_version.restype = ctypes.c_char_p
    for name in ("hlu_getrf_batched_f64", "hlu_trsm_batched_f64", "hlu_gemm_batched_f64", "hlu_gemm_small_batched_f64",
                 "hlu_rk_update_batched_f64", "hlu_rkt_phases", "hlu_rkt_phase", "hlu_schedule_create", "hlu_schedule_create_chains",
                 "hlu_schedule_launch",
                 "hlu_schedule_destroy",
    "hlu_schedule_stamps", "hlu_device_check"):
        getattr(L, name).restype = ctypes.c_int
    _lib = L
    return L


def check(rc, what):
    if rc != 0:
        raise RuntimeError(f"{what} failed with status {rc}")


def rkt_scratch_dag(torch, device, rkt, launches):
    """Scratch of a DAG schedule: truncation launches of different time slots run
    concurrently, so every launch owns a window of the lists (7 ints per
    descriptor, at 7 * first) and of the row-block items.  Returns (struct,
    keep-alive tensors, item0[nlaunch], nitems[nlaunch])."""
    import numpy as np

    from . import ir

    nl = len(launches)
    isr = launches["kind"] == ir.K_RKT32 if nl else np.zeros(0, dtype=bool)
    nrkt = int(isr.sum())
    nops = int(len(rkt)) if nrkt else 1
    item0 = np.zeros(max(nl, 1), dtype=np.int64)
    nitems = np.zeros(max(nl, 1), dtype=np.int64)
    total = 1
    if nrkt:
        m = rkt["m"].astype(np.int64)
        n = rkt["n"].astype(np.int64)
        start = np.zeros(len(m) + 1, dtype=np.int64)
        np.cumsum((m + ir.RK_BR - 1) // ir.RK_BR + (n + ir.RK_BR - 1) // ir.RK_BR, out=start[1:])
        f = launches["first"].astype(np.int64)[isr]
        c = launches["count"].astype(np.int64)[isr]
        item0[:nl][isr] = start[f]
        nitems[:nl][isr] = start[f + c] - start[f]
        total = max(int(start[-1]), 1)
    counts = torch.zeros(8 * max(nrkt, 1), dtype=torch.int32, device=device)
    lst = torch.zeros(7 * nops, dtype=torch.int32, device=device)
    items = torch.zeros(total * ir.RKT_ITEM.itemsize, dtype=torch.uint8, device=device)
    st = HluRktScratch(counts.data_ptr(), lst.data_ptr(), items.data_ptr(), nops, total)
    return st, (counts, lst, items), item0, nitems


def rkt_scratch(torch, device, rkt, launches):
    """Device scratch of the truncation launches (hlu_rkt_scratch): counters per
    launch, op lists and row-block items sized by the largest level.  Returns
    (struct, tensors that must stay alive)."""
    import numpy as np

    from . import ir

    lk = launches[launches["kind"] == ir.K_RKT32] if len(launches) else launches
    nrkt = int(len(lk))
    max_ops = int(lk["count"].max()) if nrkt else 1
    max_items = 1
    if nrkt:
        _, start = ir.rkt_items(rkt["m"], rkt["n"])
        f = lk["first"].astype(np.int64)
        cnt = lk["count"].astype(np.int64)
        max_items = max(1, int((start[f + cnt] - start[f]).max()))
    counts = torch.zeros(8 * max(nrkt, 1), dtype=torch.int32, device=device)
    lst = torch.zeros(7 * max_ops, dtype=torch.int32, device=device)
    items = torch.zeros(max_items * ir.RKT_ITEM.itemsize, dtype=torch.uint8, device=device)
    st = HluRktScratch(counts.data_ptr(), lst.data_ptr(), items.data_ptr(), max_ops, max_items)
    return st, (counts, lst, items)
