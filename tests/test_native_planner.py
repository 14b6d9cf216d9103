"""The native planner (libhlu_plan.so) must reproduce the Python planner
(the readable specification, validated against the oracle) byte for byte."""

import numpy as np
import pytest

import cases
from paper_1906_00874_b200 import native_plan
from paper_1906_00874_b200.planner import Layout, Planner
from paper_1906_00874_b200.schedule import pack


def _compare(p_py, p_nat):
    for f in ("getrf", "trsm", "gemm", "terms", "rkt", "parts", "launches"):
        a, b = getattr(p_py, f), getattr(p_nat, f)
        assert a.shape == b.shape, f
        assert a.tobytes() == b.tobytes(), f
    for f in ("nlevels", "arena_doubles", "nlog", "nranks"):
        assert getattr(p_py, f) == getattr(p_nat, f), f
    assert np.array_equal(p_py.flop_formula, p_nat.flop_formula)
    assert np.array_equal(p_py.flop_coef, p_nat.flop_coef)
    assert np.array_equal(p_py.flop_log, p_nat.flop_log)
    assert np.array_equal(p_py.lu_op_ids, p_nat.lu_op_ids)
    assert p_py.lu_labels == p_nat.lu_labels
    assert np.array_equal(p_py.op_levels, p_nat.op_levels)


@pytest.mark.parametrize("name", ["mixed_192", "mixed_256_kmax", "dense2x2_256_r3", "bem1d_1024",
                                  "sphere_1024"])
def test_factor_plans_identical(name):
    h, _ = cases.CASES[name][0]()
    L = Layout(h, cap=32)
    pl = Planner(L)
    pl.factor(h)
    p_py = pack(pl, L.payload_doubles)
    p_nat, nops = native_plan.plan(L, [("factor", h)], split_rows=0, dag_slot_ns=0)
    assert nops == len(pl.ops)
    _compare(p_py, p_nat)


def test_solve_and_update_plans_identical():
    h, _ = cases.mixed(128, 16, 0.5, 10)
    a, _ = cases.mixed(128, 16, 0.5, 11)
    b, _ = cases.mixed(128, 16, 0.5, 12)
    for cmd, roots in ((("update", h, a, b), [h, a, b]), (("solve_lower", a, b), [a, b]),
                       (("solve_upper", b, a), [b, a])):
        L = Layout(roots, cap=32)
        pl = Planner(L)
        getattr(pl, cmd[0])(*cmd[1:])
        _compare(pack(pl, L.payload_doubles), native_plan.plan(L, [cmd], split_rows=0, dag_slot_ns=0)[0])


def test_vector_solve_plans_identical():
    h, _ = cases.bem(3, 1024, 2.0, 32, 0.0, 8)
    L = Layout([h], cap=32, extra=[("x", h.rows, 1)])
    pl = Planner(L)
    pl.forward_vector(h, "x")
    pl.backward_vector(h, "x")
    _compare(pack(pl, L.payload_doubles), native_plan.plan(L, [("fwd", h, "x"), ("bwd", h, "x")], split_rows=0, dag_slot_ns=0)[0])


@pytest.mark.parametrize("name", ["mixed_192", "bem1d_1024", "sphere_1024"])
def test_split_chains_reproduce_reference(name):
    """The production plan (GEMM chains cut into row-group sub-chains) executed
    by the CPU IR machine still reproduces the reference ranks and flops."""
    from ir_exec import CpuMachine
    from paper_1906_00874_b200.pool import fill_pool, read_pool
    from paper_1906_00874_b200.schedule import effective_flops

    g = cases.golden(name)
    build, ctl = cases.CASES[name]
    h, _ = build()
    L = Layout(h, cap=32)
    p, _ = native_plan.plan(L, [("factor", h)], split_rows=16, dag_slot_ns=0)
    p0, _ = native_plan.plan(L, [("factor", h)], split_rows=0, dag_slot_ns=0)
    assert len(p.gemm) >= len(p0.gemm)
    pool = np.zeros(L.payload_doubles + p.arena_doubles)
    ranks = np.zeros(p.nranks, np.int32)
    fill_pool(L, pool, ranks)
    M = CpuMachine(pool, ranks, p.nlog, ctl[0], ctl[1])
    M.run(p)
    read_pool(L, pool, ranks)
    assert np.array_equal(cases.ranks(h), g["ranks_out"])
    assert abs(effective_flops(p, M.log) - float(g["flops"])) <= 1e-12 * float(g["flops"])


def _chain_order(packed, dense_first):
    """A launch order the two-chain GPU schedule may produce: the dense and the
    truncation launches each in level order, one chain run as far ahead of the
    other as the planner's cross-chain waits allow, then the other, and so on."""
    from paper_1906_00874_b200 import ir

    Ls = packed.launches
    lvl = [int(x) for x in Ls["level"]]
    D = [i for i in range(len(Ls)) if int(Ls[i]["kind"]) != ir.K_RKT32]
    R = [i for i in range(len(Ls)) if int(Ls[i]["kind"]) == ir.K_RKT32]
    wd, wr = packed.wait_dense, packed.wait_rkt
    pd = pr = 0
    order = []

    def can_d():
        w = int(wd[lvl[D[pd]]])
        return w < 0 or pr == len(R) or lvl[R[pr]] > w

    def can_r():
        w = int(wr[lvl[R[pr]]])
        return w < 0 or pd == len(D) or lvl[D[pd]] > w

    turn, idle = dense_first, 0
    while pd < len(D) or pr < len(R):
        moved = False
        if turn:
            while pd < len(D) and can_d():
                order.append(D[pd])
                pd += 1
                moved = True
        else:
            while pr < len(R) and can_r():
                order.append(R[pr])
                pr += 1
                moved = True
        idle = 0 if moved else idle + 1
        assert idle < 2, "two-chain waits deadlock"
        turn = not turn
    return order


@pytest.mark.parametrize("name", ["mixed_192", "mixed_256_kmax", "bem1d_1024", "sphere_1024"])
@pytest.mark.parametrize("dense_first", [True, False])
def test_two_chain_waits_reproduce_reference(name, dense_first):
    """The planner's cross-chain waits are sufficient: executing the launches in
    a drifted two-chain order (dense chain far ahead of the truncations, or far
    behind) still reproduces the reference ranks and flops."""
    import dataclasses

    from ir_exec import CpuMachine
    from paper_1906_00874_b200.pool import fill_pool, read_pool
    from paper_1906_00874_b200.schedule import effective_flops

    g = cases.golden(name)
    build, ctl = cases.CASES[name]
    h, _ = build()
    L = Layout(h, cap=32)
    p, _ = native_plan.plan(L, [("factor", h)], split_rows=16, dag_slot_ns=0)
    assert p.wait_dense is not None and len(p.wait_dense) == p.nlevels
    order = _chain_order(p, dense_first)
    assert sorted(order) == list(range(len(p.launches)))
    lv = p.launches["level"][order]
    assert np.any(np.diff(lv) < 0) or p.nlevels < 3  # the chains really drift apart
    q = dataclasses.replace(p, launches=p.launches[order])
    pool = np.zeros(L.payload_doubles + p.arena_doubles)
    ranks = np.zeros(p.nranks, np.int32)
    fill_pool(L, pool, ranks)
    M = CpuMachine(pool, ranks, p.nlog, ctl[0], ctl[1])
    M.run(q)
    read_pool(L, pool, ranks)
    assert np.array_equal(cases.ranks(h), g["ranks_out"])
    assert abs(effective_flops(p, M.log) - float(g["flops"])) <= 1e-12 * float(g["flops"])


def test_plan_cache_round_trip(tmp_path):
    """A cached plan (keyed by the planner's inputs) loads back identical."""
    h, _ = cases.CASES["sphere_1024"][0]()
    L = Layout(h, cap=32)
    fresh, n0 = native_plan.plan(L, [("factor", h)], dag_slot_ns=0)
    first, n1 = native_plan.plan(L, [("factor", h)], cache_dir=str(tmp_path), dag_slot_ns=0)
    files = list(tmp_path.iterdir())
    assert len(files) == 1
    cached, n2 = native_plan.plan(L, [("factor", h)], cache_dir=str(tmp_path), dag_slot_ns=0)
    assert n0 == n1 == n2
    for p in (first, cached):
        _compare(fresh, p)
        assert np.array_equal(fresh.wait_dense, p.wait_dense) and np.array_equal(fresh.wait_rkt, p.wait_rkt)
    # a different capacity is a different plan
    native_plan.plan(Layout(h, cap=48), [("factor", h)], cache_dir=str(tmp_path), dag_slot_ns=0)
    assert len(list(tmp_path.iterdir())) == 2
    # so is the DAG schedule of the same structure, and its dependency lists survive the cache
    d1, _ = native_plan.plan(L, [("factor", h)], cache_dir=str(tmp_path), dag_slot_ns=20000)
    assert len(list(tmp_path.iterdir())) == 3
    d2, _ = native_plan.plan(L, [("factor", h)], cache_dir=str(tmp_path), dag_slot_ns=20000)
    assert d1.dag_ptr is not None and np.array_equal(d1.dag_ptr, d2.dag_ptr) and np.array_equal(d1.dag_idx, d2.dag_idx)
    assert d1.launches.tobytes() == d2.launches.tobytes()


# ---------------------------------------------------------------- DAG schedule


def _dag_order(packed, rng, mode):
    """A launch order the DAG runtime may produce: any topological order of the
    planner's launch dependencies ("late": always the newest ready launch, i.e.
    run as far ahead as the dependencies allow; "random": a random ready one)."""
    nl = len(packed.launches)
    ptr, idx = packed.dag_ptr, packed.dag_idx
    indeg = np.diff(ptr).astype(np.int64)
    succ = [[] for _ in range(nl)]
    for l in range(nl):
        for p in idx[ptr[l]:ptr[l + 1]]:
            assert 0 <= p < l  # dependencies precede their launch
            succ[int(p)].append(l)
    ready = [l for l in range(nl) if indeg[l] == 0]
    order = []
    while ready:
        k = len(ready) - 1 if mode == "late" else int(rng.integers(len(ready)))
        if mode == "late":
            ready.sort()
        l = ready.pop(k)
        order.append(l)
        for q in succ[l]:
            indeg[q] -= 1
            if indeg[q] == 0:
                ready.append(q)
    assert len(order) == nl
    return order


@pytest.mark.parametrize("name", ["mixed_192", "mixed_256_kmax", "dense2x2_256_r3", "bem1d_1024", "sphere_1024"])
@pytest.mark.parametrize("slot_us", [5, 20, 200])
def test_dag_schedule_reproduces_level_schedule(name, slot_us):
    """The launch dependencies of the DAG schedule are sufficient: the launches
    executed in adversarial topological orders (newest ready first, random)
    leave the pool, ranks and flop log bit-identical to the level schedule
    (same ops, same per-destination order; temps may share arena blocks)."""
    import dataclasses

    from ir_exec import CpuMachine
    from paper_1906_00874_b200.pool import fill_pool
    from paper_1906_00874_b200.schedule import effective_flops

    g = cases.golden(name)
    build, ctl = cases.CASES[name]
    h, _ = build()
    L = Layout(h, cap=32)

    def run(p, order=None):
        pool = np.zeros(L.payload_doubles + p.arena_doubles)
        ranks = np.zeros(p.nranks, np.int32)
        fill_pool(L, pool, ranks)
        M = CpuMachine(pool, ranks, p.nlog, ctl[0], ctl[1])
        M.run(p if order is None else dataclasses.replace(p, launches=p.launches[order]))
        return pool[:L.payload_doubles].copy(), ranks.copy(), M

    p0, n0 = native_plan.plan(L, [("factor", h)], split_rows=16, dag_slot_ns=0)
    ref_pool, ref_ranks, M0 = run(p0)
    p, n1 = native_plan.plan(L, [("factor", h)], split_rows=16, dag_slot_ns=slot_us * 1000)
    assert n0 == n1 and p.dag_ptr is not None and len(p.dag_ptr) == len(p.launches) + 1
    assert int(p.launches["count"].sum()) == int(p0.launches["count"].sum())
    rng = np.random.default_rng(7)
    for mode in ("late", "random", "random"):
        order = _dag_order(p, rng, mode)
        pool, ranks, M = run(p, order)
        assert np.array_equal(ranks, ref_ranks)
        assert pool.tobytes() == ref_pool.tobytes()
        assert effective_flops(p, M.log) == effective_flops(p0, M0.log)
    if g is not None and "flops" in g:
        assert abs(effective_flops(p, M.log) - float(g["flops"])) <= 1e-12 * float(g["flops"])


def test_dag_schedule_overlaps_levels():
    """The point of the DAG: launches of different time slots are independent
    of one another where the level schedule put a barrier (the longest
    dependency chain is shorter than the launch list)."""
    h, _ = cases.CASES["sphere_1024"][0]()
    L = Layout(h, cap=32)
    p, _ = native_plan.plan(L, [("factor", h)], dag_slot_ns=20000)
    nl = len(p.launches)
    depth = np.zeros(nl, dtype=np.int64)
    for l in range(nl):
        d = p.dag_idx[p.dag_ptr[l]:p.dag_ptr[l + 1]]
        depth[l] = 1 + (depth[d].max() if len(d) else 0)
    assert depth.max() < nl
    # launch keys are topological
    assert np.all(np.diff(p.launches["level"].astype(np.int64)) >= 0)


@pytest.mark.parametrize("name", ["mixed_192", "mixed_256_kmax", "bem1d_1024", "sphere_1024"])
@pytest.mark.parametrize("slot_us", [5, 40])
def test_dag_dependencies_cover_memory_conflicts(name, slot_us):
    """Footprint check from the packed descriptors alone (tests/dag_check.py):
    launches that conflict in the pool (payloads, temp arena incl. block
    reuse, truncation workspaces) or in the rank table are ordered by the DAG."""
    import dag_check

    h, _ = cases.CASES[name][0]()
    L = Layout(h, cap=32)
    p, _ = native_plan.plan(L, [("factor", h)], split_rows=16, dag_slot_ns=slot_us * 1000)
    assert dag_check.violations(p) == []
