"""Case builders shared by the tests, bench and golden checks (package side).

They mirror ``tests/golden/make_golden.py`` but build with
``paper_1906_00874_b200`` instead of the reference, so a fixture comparison
checks the package's host structure code bit for bit.
"""

from __future__ import annotations

import os

import numpy as np

from paper_1906_00874_b200 import blocks, clustering, hmatrix, kernels
from paper_1906_00874_b200.lowrank import LowRank

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def mixed(n, leafsize, eta, seed):
    tree = clustering.build_cluster_tree(np.linspace(0.0, 1.0, n), leafsize)
    root = blocks.build_block_tree(tree, tree, eta)
    rng = np.random.default_rng(seed)

    def fill(block):
        if block.kind == "admissible":
            k = int(rng.integers(1, 4))
            return LowRank(rng.standard_normal((block.rows, k)) / n, rng.standard_normal((block.cols, k)))
        m = rng.standard_normal((block.rows, block.cols))
        if block.row_range == block.col_range:
            m += n * np.eye(block.rows)
        return m

    return hmatrix.build_hmatrix(root, fill), tree.dump()


def dense2x2(n, r, seed):
    root, _ = blocks.build_diagonal_2x2_tree(n, r)
    rng = np.random.default_rng(seed)

    def fill(block):
        m = rng.standard_normal((block.rows, block.cols))
        if block.row_range == block.col_range:
            m += n * np.eye(block.rows)
        return m

    return hmatrix.build_hmatrix(root, fill), None


def bem(d, n, eta, leaf, eps, kmax, workers=None):
    case = kernels.make_bem_case(d, n, eta, leafsize=leaf, eps=eps, kmax=kmax, workers=workers)
    return case.hmatrix, case.tree.dump()


CASES = {
    "mixed_192": (lambda: mixed(192, 16, 0.5, 3), (1e-8, None)),
    "mixed_256_kmax": (lambda: mixed(256, 16, 0.5, 4), (1e-12, 3)),
    "dense2x2_256_r3": (lambda: dense2x2(256, 3, 0), (1e-6, None)),
    "bem1d_1024": (lambda: bem(1, 1024, 1.0, 32, 1e-6, None), (1e-6, None)),
    "sphere_1024": (lambda: bem(3, 1024, 2.0, 32, 0.0, 8), (1e-6, None)),
    "sphere_2048_l64": (lambda: bem(3, 2048, 2.0, 64, 1e-4, None), (1e-4, None)),
    "cfg1": (lambda: bem(3, 4096, 2.0, 32, 0.0, 8), (1e-6, None)),
    "cfg3p_8192": (lambda: bem(3, 8192, 2.0, 64, 1e-4, None), (1e-4, None)),
    "cfg2": (lambda: bem(3, 32768, 2.0, 64, 1e-6, 32), (1e-6, 32)),
    "cfg3": (lambda: bem(3, 131072, 2.0, 64, 1e-4, None), (1e-4, None)),
    "cfg4p_16384": (lambda: bem(3, 16384, 2.0, 128, 1e-4, 48), (1e-4, 48)),
}


def golden(name):
    path = os.path.join(GOLDEN, f"{name}.npz")
    if not os.path.exists(path):
        return None
    with np.load(path, allow_pickle=False) as z:
        return {k: z[k] for k in z.files}


def payload_sha(h):
    import hashlib

    d = hashlib.sha256()
    for leaf in h.leaves():
        if leaf.kind == hmatrix.DENSE:
            d.update(np.ascontiguousarray(leaf.data).tobytes())
        else:
            d.update(np.ascontiguousarray(leaf.data.a).tobytes())
            d.update(np.ascontiguousarray(leaf.data.b).tobytes())
    return d.hexdigest()


def ranks(h):
    return np.array([lf.data.k for lf in h.leaves() if lf.kind == hmatrix.LOWRANK], dtype=np.int32)


def leaf_norms(h):
    out = []
    for lf in h.leaves():
        if lf.kind == hmatrix.DENSE:
            out.append(np.linalg.norm(lf.data))
        else:
            out.append(np.linalg.norm(lf.data.value()) if lf.data.k else 0.0)
    return np.array(out)
