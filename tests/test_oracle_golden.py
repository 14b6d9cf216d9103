"""Pin the CPU oracle and the host structure code against the reference.

Fixtures in ``tests/golden`` were produced by running the real reference
(``tests/golden/make_golden.py``).  The oracle issues the same LAPACK calls on
the same layouts, so everything here is checked bit for bit: structure dumps,
assembled payload hashes, factor hashes, per-leaf ranks, the effective-flop
counter and the forward solve.
"""

import hashlib
import os

import numpy as np
import pytest

import cases
from oracle import hlu_oracle as orc
from paper_1906_00874_b200 import hmatrix
from paper_1906_00874_b200.lowrank import LowRank, SingularBlockError, TruncationControl

FAST = ["mixed_192", "mixed_256_kmax", "dense2x2_256_r3", "bem1d_1024", "sphere_1024",
        "sphere_2048_l64"]


def _check_structure(name, h, tree_dump, g):
    dump = hmatrix.structure_dump(h)
    assert hashlib.sha256(dump.encode()).hexdigest() == str(g["structure_sha"]), name
    if "structure_dump" in g:
        assert dump == str(g["structure_dump"])
    if "cluster_dump_sha" in g and tree_dump is not None:
        assert hashlib.sha256(tree_dump.encode()).hexdigest() == str(g["cluster_dump_sha"])
    assert cases.payload_sha(h) == str(g["payload_sha"]), f"{name}: assembled payload differs"
    assert np.array_equal(cases.ranks(h), g["ranks_in"])


@pytest.mark.parametrize("name", FAST)
def test_structure_and_assembly_bit_exact(name):
    g = cases.golden(name)
    assert g is not None, f"missing fixture {name}"
    h, tree_dump = cases.CASES[name][0]()
    _check_structure(name, h, tree_dump, g)


@pytest.mark.parametrize("name", FAST)
def test_oracle_factor_bit_exact(name):
    g = cases.golden(name)
    build, ctl = cases.CASES[name]
    h, _ = build()
    flops = orc.hlu_factorize(h, TruncationControl(*ctl))
    assert np.array_equal(cases.ranks(h), g["ranks_out"])
    assert cases.payload_sha(h) == str(g["factor_sha"])
    assert flops == float(g["flops"])
    y = orc.forward_solve(h, g["rhs"])
    assert np.array_equal(y, g["y_forward"])
    if "flat_out" in g:
        assert np.array_equal(hmatrix.flatten(h), g["flat_out"])


@pytest.mark.slow
@pytest.mark.skipif(not os.environ.get("HLU_SLOW"), reason="set HLU_SLOW=1 (about 30 s)")
def test_oracle_cfg1_bit_exact():
    g = cases.golden("cfg1")
    h, tree_dump = cases.CASES["cfg1"][0]()
    _check_structure("cfg1", h, tree_dump, g)
    flops = orc.hlu_factorize(h, TruncationControl(1e-6))
    assert np.array_equal(cases.ranks(h), g["ranks_out"])
    assert cases.payload_sha(h) == str(g["factor_sha"])
    assert flops == float(g["flops"])


def test_backward_solve_against_dense():
    """The restated backward substitution (absent in the reference)."""
    h, _ = cases.mixed(192, 16, 0.5, 3)
    orc.hlu_factorize(h, TruncationControl(1e-12))
    f = hmatrix.flatten(h)
    lo = np.tril(f, -1) + np.eye(f.shape[0])
    up = np.triu(f)
    b = np.random.default_rng(0).standard_normal(f.shape[0])
    x = orc.hlu_solve(h, b)
    want = np.linalg.solve(up, np.linalg.solve(lo, b))
    assert np.linalg.norm(x - want) <= 1e-10 * np.linalg.norm(want)


# known answers from the reference's unit tests (test_lowrank.py)


def test_lu_2x2_by_hand():
    a = np.array([[2.0, 1.0], [4.0, 5.0]])
    orc.lu_nopivot(a)
    assert np.array_equal(a, np.array([[2.0, 1.0], [2.0, 3.0]]))


def test_lu_singular_names_block():
    with pytest.raises(SingularBlockError) as err:
        orc.lu_nopivot(np.array([[1.0, 1.0], [1.0, 1.0]]), block_path="diag")
    assert err.value.block_path == "diag"


def test_truncation_exact_rank_13(rng):
    q1, _ = np.linalg.qr(rng.standard_normal((32, 32)))
    q2, _ = np.linalg.qr(rng.standard_normal((32, 32)))
    d = (q1 * 3.0 ** -np.arange(32.0)) @ q2.T
    assert orc.compress_dense(d, TruncationControl(1e-6)).k == 13


def test_parallel_outer_products_rank_one(rng):
    a = rng.standard_normal((8, 1))
    b = rng.standard_normal((5, 1))
    got = orc.add_truncated(LowRank(a, b), LowRank(a.copy(), b.copy()), TruncationControl(1e-10))
    assert got.k == 1
