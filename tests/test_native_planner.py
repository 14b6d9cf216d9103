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
    p_nat, nops = native_plan.plan(L, [("factor", h)], split_rows=0)
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
        _compare(pack(pl, L.payload_doubles), native_plan.plan(L, [cmd], split_rows=0)[0])


def test_vector_solve_plans_identical():
    h, _ = cases.bem(3, 1024, 2.0, 32, 0.0, 8)
    L = Layout([h], cap=32, extra=[("x", h.rows, 1)])
    pl = Planner(L)
    pl.forward_vector(h, "x")
    pl.backward_vector(h, "x")
    _compare(pack(pl, L.payload_doubles), native_plan.plan(L, [("fwd", h, "x"), ("bwd", h, "x")], split_rows=0)[0])


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
    p, _ = native_plan.plan(L, [("factor", h)], split_rows=16)
    p0, _ = native_plan.plan(L, [("factor", h)], split_rows=0)
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
    p, _ = native_plan.plan(L, [("factor", h)], split_rows=16)
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
    fresh, n0 = native_plan.plan(L, [("factor", h)])
    first, n1 = native_plan.plan(L, [("factor", h)], cache_dir=str(tmp_path))
    files = list(tmp_path.iterdir())
    assert len(files) == 1
    cached, n2 = native_plan.plan(L, [("factor", h)], cache_dir=str(tmp_path))
    assert n0 == n1 == n2
    for p in (first, cached):
        _compare(fresh, p)
        assert np.array_equal(fresh.wait_dense, p.wait_dense) and np.array_equal(fresh.wait_rkt, p.wait_rkt)
    # a different capacity is a different plan
    native_plan.plan(Layout(h, cap=48), [("factor", h)], cache_dir=str(tmp_path))
    assert len(list(tmp_path.iterdir())) == 2
