"""Products with the H-matrix and its stored factors: ``hmatvec``
(reference hmatrix.py:178-200), ``lower_unit_matvec`` / ``upper_matvec``
(hlu.py:720-767) and the residual probe (bench.py:142-152).

CPU: the oracle restatement against fixtures made by the real reference
(``tests/golden/make_golden_matvec.py``), the native planner against the
Python specification, and the planned term chains executed by the CPU IR
machine.  GPU: the same products through the C ABI against the oracle."""

import os

import numpy as np
import pytest

import cases
from oracle import hlu_oracle as orc
from paper_1906_00874_b200 import native_plan
from paper_1906_00874_b200.lowrank import TruncationControl
from paper_1906_00874_b200.planner import Layout, Planner
from paper_1906_00874_b200.schedule import pack

NAMES = ["mixed_192", "bem1d_1024", "sphere_1024"]
GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
TOL = 1e-12  # relative, fp64 (different summation order than numpy's dgemv)


def _golden(name):
    return np.load(os.path.join(GOLDEN, f"matvec_{name}.npz"))


def _factored(name):
    build, ctl = cases.CASES[name]
    h, _ = build()
    orig = h.copy()
    orc.hlu_factorize(h, TruncationControl(*ctl))
    return orig, h


def _rel(a, b):
    return np.linalg.norm(a - b) / np.linalg.norm(b)


@pytest.mark.parametrize("name", NAMES)
def test_oracle_products_pinned_to_reference(name):
    g = _golden(name)
    orig, fac = _factored(name)
    x = g["x"]
    np.testing.assert_array_equal(orc.hmatvec(orig, x), g["ax"])
    np.testing.assert_array_equal(orc.lower_unit_matvec(fac, x), g["lx"])
    np.testing.assert_array_equal(orc.upper_matvec(fac, x), g["ux"])
    assert orc.residual_probe(orig, fac) == float(g["residual"])


def test_matvec_plans_identical():
    orig, fac = _factored("sphere_1024")
    n = orig.rows
    for roots, cmds in (([orig], [("matvec", orig, "x", "y")]),
                        ([fac], [("upper_matvec", fac, "x", "y"), ("lower_matvec", fac, "y", "z")])):
        L = Layout(roots, cap=32, extra=[("x", n, 2), ("y", n, 2), ("z", n, 2)])
        pl = Planner(L)
        for c in cmds:
            pl.matvec(*c[1:], tri={"matvec": 0, "lower_matvec": 1, "upper_matvec": 2}[c[0]])
        p_py = pack(pl, L.payload_doubles)
        p_nat, nops = native_plan.plan(L, cmds, split_rows=0)
        assert nops == len(pl.ops)
        for f in ("gemm", "terms", "launches"):
            assert getattr(p_py, f).tobytes() == getattr(p_nat, f).tobytes(), f


@pytest.mark.parametrize("name", NAMES)
def test_planned_products_on_cpu_machine(name):
    """The production plan (split chains) of A x, U x and L (U x), executed
    term by term on the CPU IR machine, matches the reference products."""
    from ir_exec import CpuMachine
    from paper_1906_00874_b200.pool import fill_pool, read_extra

    g = _golden(name)
    orig, fac = _factored(name)
    n = orig.rows
    x = g["x"]
    L = Layout([orig, fac], cap=32, extra=[("x", n, 2), ("ax", n, 2), ("ux", n, 2), ("lux", n, 2), ("lx", n, 2)])
    cmds = [("matvec", orig, "x", "ax"), ("upper_matvec", fac, "x", "ux"), ("lower_matvec", fac, "ux", "lux"),
            ("lower_matvec", fac, "x", "lx")]
    p, _ = native_plan.plan(L, cmds, split_rows=16)
    pool = np.zeros(L.payload_doubles + p.arena_doubles)
    ranks = np.zeros(p.nranks, np.int32)
    fill_pool(L, pool, ranks, extras={"x": x})
    CpuMachine(pool, ranks, p.nlog, 0.0, None).run(p)
    assert _rel(read_extra(L, pool, "ax"), g["ax"]) <= TOL
    assert _rel(read_extra(L, pool, "ux"), g["ux"]) <= TOL
    assert _rel(read_extra(L, pool, "lx"), g["lx"]) <= TOL
    lux = read_extra(L, pool, "lux")
    assert _rel(lux, orc.lower_unit_matvec(fac, g["ux"])) <= TOL


@pytest.mark.gpu
@pytest.mark.parametrize("name", NAMES)
def test_gpu_products_vs_reference(name):
    from paper_1906_00874_b200 import hmatvec, lower_unit_matvec, residual_probe, upper_matvec

    g = _golden(name)
    orig, fac = _factored(name)
    x = g["x"]
    assert _rel(hmatvec(orig, x), g["ax"]) <= TOL
    assert _rel(hmatvec(orig, x[:, 0]), g["ax"][:, 0]) <= TOL
    assert _rel(lower_unit_matvec(fac, x), g["lx"]) <= TOL
    assert _rel(upper_matvec(fac, x), g["ux"]) <= TOL
    r = residual_probe(orig, fac)
    assert abs(r - float(g["residual"])) <= 1e-6 * float(g["residual"]) + 1e-15
