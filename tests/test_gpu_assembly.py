"""GPU assembly against the host restatement of
the reference assembly (kernels.py:73-168) and the reference fixtures; the
HODLR (cfg5) case against the CPU oracle."""

import os

import numpy as np
import pytest

import cases
from oracle import hlu_oracle as orc
from paper_1906_00874_b200 import gpu_assembly, hmatrix
from paper_1906_00874_b200.hlu import hlu_factorize, hlu_solve, make_plan, residual_probe
from paper_1906_00874_b200.hmatrix import DENSE
from paper_1906_00874_b200.kernels import KernelConfig, make_bem_case, mesh_width
from paper_1906_00874_b200.lowrank import TruncationControl

pytestmark = pytest.mark.gpu

BEM = {  # name: (d, n, eta, leaf, eps, kmax)
    "sphere_1024": (3, 1024, 2.0, 32, 0.0, 8),
    "sphere_2048_l64": (3, 2048, 2.0, 64, 1e-4, None),
    "bem1d_1024": (1, 1024, 1.0, 32, 1e-6, None),
    "cfg1": (3, 4096, 2.0, 32, 0.0, 8),
}


def _gpu_case(d, n, eta, leaf, eps, kmax):
    host = make_bem_case(d, n, eta, leafsize=leaf, eps=eps, kmax=kmax, workers=os.cpu_count())
    g = gpu_assembly.assemble_hmatrix_gpu(host.block, host.points, host.cfg, device="cuda:0")
    return host.hmatrix, g


@pytest.mark.parametrize("name", list(BEM))
def test_gpu_assembly_matches_host(name):
    """Dense leaves bit-identical (d = 3; same operation order) or to 1 ulp
    (log kernels), every Rk rank identical to the host / reference assembly,
    Rk values to rounding."""
    d = BEM[name][0]
    h, g = _gpu_case(*BEM[name])
    assert hmatrix.structure_dump(h) == hmatrix.structure_dump(g)
    for a, b in zip(h.leaves(), g.leaves()):
        if a.kind == DENSE:
            if d == 3:
                assert np.array_equal(a.data, b.data)
            else:
                assert np.allclose(a.data, b.data, rtol=4e-16, atol=0)
        else:
            assert a.data.k == b.data.k
            va, vb = a.data.value(), b.data.value()
            assert np.linalg.norm(va - vb) <= 1e-11 * max(np.linalg.norm(va), 1e-300)


def test_gpu_assembly_payload_sha_and_lu_ranks_cfg1():
    """cfg1 assembled on the GPU: dense payload bytes identical to the
    reference fixture's assembly, and the GPU H-LU of the GPU-assembled matrix
    gives the reference's post-LU rank of every block."""
    g = cases.golden("cfg1")
    h, ga = _gpu_case(*BEM["cfg1"])
    assert cases.payload_sha(h) == str(g["payload_sha"])
    assert np.array_equal(cases.ranks(ga), g["ranks_in"])
    hlu_factorize(make_plan(ga, TruncationControl(1e-6)))
    assert np.array_equal(cases.ranks(ga), g["ranks_out"])


def test_gpu_assembly_cfg3p_lu_parity():
    """n = 8192 (cfg3 geometry): GPU assembly, GPU H-LU, reference post-LU
    ranks and forward solve."""
    g = cases.golden("cfg3p_8192")
    _, ga = _gpu_case(3, 8192, 2.0, 64, 1e-4, None)
    assert np.array_equal(cases.ranks(ga), g["ranks_in"])
    hlu_factorize(make_plan(ga, TruncationControl(1e-4)))
    assert np.array_equal(cases.ranks(ga), g["ranks_out"])


@pytest.mark.parametrize("n,leaf", [(2048, 128), (4096, 256)])
def test_hodlr_lu_vs_oracle(n, leaf):
    """cfg5 structure (weak admissibility on the circle, A_ii = 1, rank-32
    off-diagonal blocks by the reference's compress_dense route): GPU H-LU
    against the CPU oracle -- identical ranks, solve within 1e-8.  (No
    reference fixture exists for cfg5: the reference has no HODLR builder.)"""
    h, block, pts, cfg, lu_ctl = gpu_assembly.hodlr_case(n, leafsize=leaf, k=32, generator="svd")
    ref = h.copy()
    orc.hlu_factorize(ref, lu_ctl)
    hlu_factorize(make_plan(h, lu_ctl))
    assert np.array_equal(cases.ranks(h), cases.ranks(ref))
    b = np.random.default_rng(0).standard_normal(n)
    x = hlu_solve(h, b)
    xr = orc.hlu_solve(ref, b)
    assert np.linalg.norm(x - xr) <= 1e-8 * np.linalg.norm(xr)


def test_hodlr_aca_generator():
    """The GPU cross-approximation generator: rank-32 off-diagonal blocks
    within a small relative error of the exact kernel blocks, and a GPU H-LU
    whose residual probe is at rounding level (the factors are exact up to the
    LU truncation)."""
    from paper_1906_00874_b200.kernels import assemble_dense_block

    n = 4096
    h, block, pts, cfg, lu_ctl = gpu_assembly.hodlr_case(n, leafsize=256, k=32, generator="aca", device="cuda:0")
    worst = 0.0
    for lf in h.leaves():
        if lf.kind == DENSE:
            continue
        assert lf.data.k == 32
        exact = assemble_dense_block(pts, lf.block.row, lf.block.col, cfg)
        worst = max(worst, np.linalg.norm(lf.data.value() - exact, 2) / np.linalg.norm(exact, 2))
    assert worst < 1e-6, worst
    original = h.copy()
    hlu_factorize(make_plan(h, lu_ctl))
    assert residual_probe(original, h) < 1e-8
