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
from .hmatrix import DENSE, HMatrix, Skeleton, StructureError, build_skeleton
from .lowrank import TruncationControl
from .planner import DEFAULT_CAP, MAX_CAP, Layout, Planner

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
    keep_schedule: bool = False


def make_plan(h: HMatrix, truncation: TruncationControl | None = None, mode: str = SEQUENTIAL,
              workers: int = 1, wd_er: bool = True, seed: int = 0, capacity: int | None = None,
              device=None, use_graph: bool = True, keep_schedule: bool = False) -> HluPlan:
    """Reference ``make_plan`` (hlu.py:72-90).  ``keep_schedule=True`` keeps the
    planned device schedule (pools, descriptors, CUDA graphs) on the plan, so
    later ``hlu_factorize(plan)`` calls on the same structure only re-pack the
    host payloads, upload, replay and download (plan once, factorize many); it
    also selects the launch-DAG schedule, whose longer setup the replays repay.
    Without it every call plans the level schedule (fast setup) and frees it."""
    if mode not in (SEQUENTIAL, PARALLEL):
        raise ValueError(f"unknown mode {mode!r}")
    return HluPlan(
        matrix=h, skeleton=build_skeleton(h),
        truncation=truncation if truncation is not None else TruncationControl(),
        mode=mode, workers=workers, wd_er=wd_er, seed=seed,
        capacity=_auto_capacity([h], truncation) if capacity is None else int(capacity),
        device=device, use_graph=use_graph, keep_schedule=keep_schedule,
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


_TRI = {"lower_matvec": 1, "upper_matvec": 2}


def plan_call(roots, commands, capacity, extras=None, planner="native", replay=True):
    """Layout + packed schedule for a list of planner commands, e.g.
    ``[("factor", h)]``; ``planner`` = "native" (C++) or "python" (the
    reference-order specification the native planner is tested against).
    ``replay`` picks the schedule: True = the launch DAG (finest overlap, but
    its CUDA graphs take minutes to instantiate at n = 131072, so it pays off
    when the schedule is kept and replayed); False = the level schedule
    (seconds to set up; one-shot calls).  ``HLU_DAG_SLOT_US`` overrides both."""
    layout = Layout(roots, cap=capacity, extra=[(k, v.shape[0], v.shape[1]) for k, v in (extras or {}).items()])
    if planner == "native":
        import os

        from . import native_plan

        slot = None if (replay or os.environ.get(native_plan.DAG_SLOT_ENV)) else 0
        packed, _ = native_plan.plan(layout, commands, dag_slot_ns=slot)
        return layout, packed
    pl = Planner(layout)
    for cmd in commands:
        if cmd[0] in _TRI:
            pl.matvec(*cmd[1:], tri=_TRI[cmd[0]])
            continue
        name = {"fwd": "forward_vector", "bwd": "backward_vector"}.get(cmd[0], cmd[0])
        getattr(pl, name)(*cmd[1:])
    from .schedule import pack

    return layout, pack(pl, layout.payload_doubles)


def _run(roots, commands, ctl, capacity, device=None, use_graph=True, extras=None, keep=False, replay=False):
    """Plan + run one H-arithmetic call on the GPU, re-planning with a doubled
    capacity (clamped to MAX_CAP) if any Rk result overflows.  Returns the
    DeviceCall; ``call.capacity`` is the capacity that succeeded.  ``replay``:
    the call's schedule will be kept and replayed (see ``plan_call``)."""
    from .device import DeviceCall, RankOverflow

    cap = capacity
    while True:
        import time

        t0 = time.perf_counter()
        layout, packed = plan_call(roots, commands, cap, extras, replay=replay)
        t1 = time.perf_counter()
        call = DeviceCall(layout, packed, ctl, device=device, use_graph=use_graph, extras=extras)
        call.sync()
        call.plan_s, call.setup_s = t1 - t0, time.perf_counter() - t1  # diagnostics (bench.py)
        call.launch()
        try:
            call.check_errors()
        except RankOverflow:
            call.release()
            if cap >= MAX_CAP:
                raise
            cap = min(2 * cap, MAX_CAP)
            continue
        call.capacity = cap
        call.download()
        if not keep:
            call.release()
        return call


def hlu_factorize(plan: HluPlan):
    """Factorize ``plan.matrix`` in place on the GPU.  Returns None, like the
    reference's sequential mode (``hlu.py:661-680``)."""
    h = plan.matrix
    if h.rows != h.cols:
        raise StructureError("H-LU requires a square matrix")
    call = plan.last_call if plan.keep_schedule else None
    if call is not None and getattr(call, "handle", None) and call.L.roots[0] is h:
        from .device import RankOverflow

        import os
        import time

        t = [time.perf_counter()]
        call.refill_upload()  # the structure is unchanged: new payloads through the kept schedule
        t.append(time.perf_counter())
        call.launch()
        try:
            call.check_errors()
            t.append(time.perf_counter())
            call.download()
            t.append(time.perf_counter())
            plan.flops.add(call.flops())
            t.append(time.perf_counter())
            if os.environ.get("HLU_E2E_TIMING") == "1":
                import sys

                print("hlu_factorize (kept schedule): pack+upload issue %.3f s, factorization (sync) %.3f s, "
                      "download+install %.3f s, flop counter %.3f s" % tuple(b - a for a, b in zip(t, t[1:])),
                      file=sys.stderr)
            return None
        except RankOverflow:
            call.release()
            plan.capacity = min(2 * plan.capacity, MAX_CAP)
    call = _run([h], [("factor", h)], plan.truncation, plan.capacity, plan.device, plan.use_graph,
                keep=plan.keep_schedule, replay=plan.keep_schedule)
    plan.capacity = call.capacity  # later calls start from the capacity that fitted
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


# -- products with the matrix / its stored factors, on the GPU
#    (hmatrix.py:178-200, hlu.py:720-767, residual probe bench.py:142-152)


def _products(roots, commands, vectors, outputs, device=None):
    """Run matvec-type commands over pooled vectors; returns the outputs."""
    extras = dict(vectors)
    for name, rows, cols in outputs:
        extras[name] = np.zeros((rows, cols))
    call = _run(roots, commands, TruncationControl(), _auto_capacity(roots, None), device, extras=extras,
                keep=True)
    try:
        return [call.extra(name) for name, _, _ in outputs]
    finally:
        call.close()


def _as_block(h, x, n):
    x = np.asarray(x, dtype=float)
    if x.shape[0] != n:
        raise ValueError(f"length mismatch: {n} columns vs {x.shape[0]}")
    return x, np.ascontiguousarray(x.reshape(n, -1))


def hmatvec(h: HMatrix, x, device=None):
    """y = h @ x over the block structure (reference ``hmatvec``,
    hmatrix.py:178-200): one GPU term chain per block row."""
    x, xb = _as_block(h, x, h.cols)
    (y,) = _products([h], [("matvec", h, "x", "y")], {"x": xb}, [("y", h.rows, xb.shape[1])], device)
    return y.reshape((h.rows,) + x.shape[1:])


def lower_unit_matvec(h: HMatrix, x, device=None):
    """y = L x with the unit lower factor stored in a factored h (hlu.py:720-727)."""
    x, xb = _as_block(h, x, h.rows)
    (y,) = _products([h], [("lower_matvec", h, "x", "y")], {"x": xb}, [("y", h.rows, xb.shape[1])], device)
    return y.reshape(x.shape)


def upper_matvec(h: HMatrix, x, device=None):
    """y = U x with the upper factor stored in a factored h (hlu.py:745-767)."""
    x, xb = _as_block(h, x, h.rows)
    (y,) = _products([h], [("upper_matvec", h, "x", "y")], {"x": xb}, [("y", h.rows, xb.shape[1])], device)
    return y.reshape(x.shape)


def residual_probe(original: HMatrix, factored: HMatrix, seed=0, probes=10, device=None):
    """Worst relative residual ||A x - L (U x)|| / ||A x|| over random x
    (reference ``residual_probe``, bench.py:142-152, same rng draws); all
    probes run as columns of one GPU call (A x, U x, then L (U x))."""
    rng = np.random.default_rng(seed)
    n = original.cols
    xb = np.stack([rng.standard_normal(n) for _ in range(probes)], axis=1)
    ax, _, lux = _products(
        [original, factored],
        [("matvec", original, "x", "ax"), ("upper_matvec", factored, "x", "ux"),
         ("lower_matvec", factored, "ux", "lux")],
        {"x": xb},
        [("ax", n, probes), ("ux", n, probes), ("lux", n, probes)],
        device,
    )
    worst = 0.0
    for p in range(probes):
        worst = max(worst, float(np.linalg.norm(ax[:, p] - lux[:, p]) / np.linalg.norm(ax[:, p])))
    return worst


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
