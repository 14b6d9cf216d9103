"""H-LU factorization and H-solves on the B200 — the reference's API.

Same entry points and contracts as ``hluflow.hlu`` (``hlu.py:58-767``):
``make_plan`` / ``hlu_factorize`` factorize an ``HMatrix`` in place,
``solve_lower_hmatrix`` / ``solve_upper_hmatrix`` / ``update_hmatrix`` run the
H-TRSMs and H-GEMM on H-matrix operands, ``lower_unit_matvec`` /
``upper_matvec`` apply the stored factors.  New: ``hlu_solve`` (forward and
backward vector substitution; the reference has only the forward half).

Execution model: the planner replays the reference recursion into typed ops,
the scheduler levels them by skeleton-slot hazards, and the whole call runs as
one CUDA graph of batched sm_100a kernels (``device.DeviceCall``).  ``mode``,
``workers``, ``wd_er`` and ``seed`` are accepted for API compatibility (the
GPU schedule replaces the thread runtime); unknown modes still raise.
"""

from __future__ import annotations

import threading
from dataclasses import dataclass, field

import numpy as np

from .blocks import INADMISSIBLE, PARTITIONED, BlockNode
from .clustering import Cluster
from .hmatrix import DENSE, HMatrix, Skeleton, StructureError, _matvec_into, build_skeleton
from .lowrank import TruncationControl
from .planner import DEFAULT_CAP, Layout, Planner

SEQUENTIAL = "sequential"
PARALLEL = "parallel"


class FlopCounter:
    """Effective-flop accumulator (reference ``hlu.py:46-55``); on the GPU the
    same per-site formulas are evaluated from ranks logged by the kernels."""

    def __init__(self):
        self._lock = threading.Lock()
        self.total = 0.0

    def add(self, n):
        with self._lock:
            self.total += n


@dataclass
class HluPlan:
    matrix: HMatrix
    skeleton: Skeleton
    truncation: TruncationControl
    mode: str = SEQUENTIAL
    workers: int = 1
    wd_er: bool = True
    seed: int = 0
    flops: FlopCounter = field(default_factory=FlopCounter)
    capacity: int = DEFAULT_CAP
    device: object = None
    use_graph: bool = True
    last_call: object = None


def make_plan(h: HMatrix, truncation: TruncationControl | None = None, mode: str = SEQUENTIAL,
              workers: int = 1, wd_er: bool = True, seed: int = 0, capacity: int | None = None,
              device=None, use_graph: bool = True) -> HluPlan:
    if mode not in (SEQUENTIAL, PARALLEL):
        raise ValueError(f"unknown mode {mode!r}")
    return HluPlan(
        matrix=h, skeleton=build_skeleton(h),
        truncation=truncation if truncation is not None else TruncationControl(),
        mode=mode, workers=workers, wd_er=wd_er, seed=seed,
        capacity=_auto_capacity([h], truncation) if capacity is None else int(capacity),
        device=device, use_graph=use_graph,
    )


def _auto_capacity(roots, ctl):
    """Per-block Rk capacity: at least the current max rank, 32 by default,
    kmax when set; doubled automatically on device overflow."""
    kmax = 0
    for r in roots:
        for lf in r.leaves():
            if lf.kind != DENSE:
                kmax = max(kmax, lf.data.k)
    cap = max(DEFAULT_CAP, kmax)
    if ctl is not None and ctl.kmax is not None:
        cap = max(cap, ctl.kmax, kmax)
    return int(cap)


def plan_call(roots, commands, capacity, extras=None, planner="native"):
    """Layout + packed schedule for a list of planner commands, e.g.
    ``[("factor", h)]``; ``planner`` = "native" (C++) or "python" (the
    reference-order specification the native planner is tested against)."""
    layout = Layout(roots, cap=capacity, extra=[(k, v.shape[0], v.shape[1]) for k, v in (extras or {}).items()])
    if planner == "native":
        from . import native_plan

        packed, _ = native_plan.plan(layout, commands)
        return layout, packed
    pl = Planner(layout)
    for cmd in commands:
        name = {"fwd": "forward_vector", "bwd": "backward_vector"}.get(cmd[0], cmd[0])
        getattr(pl, name)(*cmd[1:])
    from .schedule import pack

    return layout, pack(pl, layout.payload_doubles)


def _run(roots, commands, ctl, capacity, device=None, use_graph=True, extras=None, keep=False):
    """Plan + run one H-arithmetic call on the GPU, re-planning with a doubled
    capacity if any Rk result overflows.  Returns the DeviceCall."""
    from .device import DeviceCall, RankOverflow

    cap = capacity
    while True:
        layout, packed = plan_call(roots, commands, cap, extras)
        call = DeviceCall(layout, packed, ctl, device=device, use_graph=use_graph, extras=extras)
        call.launch()
        try:
            call.check_errors()
        except RankOverflow:
            call.close()
            cap *= 2
            if cap > 64:
                raise
            continue
        call.download()
        if not keep:
            call.close()
        return call


def hlu_factorize(plan: HluPlan):
    """Factorize ``plan.matrix`` in place on the GPU.  Returns None, like the
    reference's sequential mode (``hlu.py:661-680``)."""
    h = plan.matrix
    if h.rows != h.cols:
        raise StructureError("H-LU requires a square matrix")
    call = _run([h], [("factor", h)], plan.truncation, plan.capacity, plan.device, plan.use_graph)
    plan.flops.add(call.flops())
    plan.last_call = call
    return None


def solve_lower_hmatrix(l, b, ctl=None, runtime=None, skeleton=None):
    """b := l^-1 b (l holds a factored unit-lower part); ``runtime`` /
    ``skeleton`` are accepted for API compatibility."""
    ctl = ctl if ctl is not None else TruncationControl()
    _run([l, b], [("solve_lower", l, b)], ctl, _auto_capacity([l, b], ctl))


def solve_upper_hmatrix(b, u, ctl=None, runtime=None, skeleton=None):
    """b := b u^-1."""
    ctl = ctl if ctl is not None else TruncationControl()
    _run([b, u], [("solve_upper", b, u)], ctl, _auto_capacity([b, u], ctl))


def update_hmatrix(c, a, b, ctl=None, runtime=None, skeleton=None):
    """c := c - a @ b in H-arithmetic."""
    ctl = ctl if ctl is not None else TruncationControl()
    _run([c, a, b], [("update", c, a, b)], ctl, _auto_capacity([c, a, b], ctl))


def hlu_solve(h: HMatrix, rhs, device=None):
    """x = U^-1 L^-1 rhs on a factored H-matrix (forward substitution in the
    reference's panel order, then block back-substitution), on the GPU."""
    rhs = np.asarray(rhs, dtype=float)
    vec = rhs.reshape(h.rows, -1)

    call = _run([h], [("fwd", h, "x"), ("bwd", h, "x")], TruncationControl(), _auto_capacity([h], None),
                device, extras={"x": vec}, keep=True)
    x = call.extra("x")
    call.close()
    return x.reshape(rhs.shape)


def forward_solve(h: HMatrix, rhs, device=None):
    """y = L^-1 rhs (the reference's route: ``solve_lower_hmatrix`` with an
    n x 1 dense-leaf right-hand side)."""
    rhs = np.asarray(rhs, dtype=float)
    call = _run([h], [("fwd", h, "x")], TruncationControl(),
                _auto_capacity([h], None), device, extras={"x": rhs.reshape(h.rows, -1)}, keep=True)
    y = call.extra("x")
    call.close()
    return y.reshape(rhs.shape)


# -- triangular matvec with the stored factors (host utilities, hlu.py:720-767)


def lower_unit_matvec(h: HMatrix, x):
    x = np.asarray(x, dtype=float)
    y = np.zeros_like(x, dtype=float)
    _tri_into(h, x, y, lower=True)
    return y


def upper_matvec(h: HMatrix, x):
    x = np.asarray(x, dtype=float)
    y = np.zeros_like(x, dtype=float)
    _tri_into(h, x, y, lower=False)
    return y


def _tri_into(h, x, y, lower):
    if h.kind == DENSE:
        y += (np.tril(h.data, -1) @ x + x) if lower else (np.triu(h.data) @ x)
        return
    if h.kind != PARTITIONED:
        raise StructureError("factored matrix has a low-rank diagonal block")
    r0 = h.row_range[0]
    for i, line in enumerate(h.data):
        for j, ch in enumerate(line):
            (i0, i1), (j0, j1) = ch.row_range, ch.col_range
            xs, ys = x[j0 - r0 : j1 - r0], y[i0 - r0 : i1 - r0]
            if (j < i) if lower else (j > i):
                _matvec_into(ch, xs, ys)
            elif j == i:
                _tri_into(ch, xs, ys, lower)


def emit_task_graph(plan: HluPlan):
    """The planned op DAG (the GPU analogue of the reference's task graph):
    returns the planner with ``ops`` and the per-op levels."""
    from .schedule import assign_levels

    h = plan.matrix
    layout = Layout([h], cap=plan.capacity)
    pl = Planner(layout)
    pl.factor(h)
    pl.levels = assign_levels(pl)
    return pl


def vector_leaf(h: HMatrix, vec):
    """An n x 1 dense-leaf H-matrix over h's row cluster (reference forward-solve RHS)."""
    col = Cluster(0, 1, np.array([0.0]), np.array([0.0]))
    return HMatrix(BlockNode(h.block.row, col, INADMISSIBLE), DENSE, np.asarray(vec, float).reshape(-1, 1))
