"""Generate golden fixtures by running the REAL reference (``hluflow``).

Run in the build container, where ``/root/reference`` exists:

    python tests/golden/make_golden.py [case ...]      # default: small cases

Each case writes ``tests/golden/<case>.npz`` holding, from the reference:
structure dumps (text, or sha256 for big cases), a sha256 of every assembled
leaf payload (bit-exact assembly check), per-Rk-leaf ranks after the H-LU, the
effective-flop counter, per-leaf Frobenius norms of the factors, the forward
solve ``y = L^-1 b`` through ``solve_lower_hmatrix`` with an n x 1 dense leaf,
and, for n <= 512, the full flattened factors.  Nothing on the GPU box reads
``/root/reference``; it only reads these committed fixtures.
"""

from __future__ import annotations

import hashlib
import os
import sys
import time

for _v in ("OPENBLAS_NUM_THREADS", "OMP_NUM_THREADS", "MKL_NUM_THREADS"):
    os.environ[_v] = "1"

import numpy as np  # noqa: E402

REF = "/root/reference/pkg/src"
OUT = os.path.dirname(os.path.abspath(__file__))


def _ref():
    sys.path.insert(0, REF)
    import hluflow  # noqa: F401
    from hluflow import blocks, clustering, hlu, hmatrix, kernels, lowrank

    return blocks, clustering, hlu, hmatrix, kernels, lowrank


def payload_hash(h, hm):
    d = hashlib.sha256()
    for leaf in h.leaves():
        if leaf.kind == hm.DENSE:
            d.update(np.ascontiguousarray(leaf.data).tobytes())
        else:
            d.update(np.ascontiguousarray(leaf.data.a).tobytes())
            d.update(np.ascontiguousarray(leaf.data.b).tobytes())
    return d.hexdigest()


def leaf_norms(h, hm):
    out = []
    for leaf in h.leaves():
        if leaf.kind == hm.DENSE:
            out.append(np.linalg.norm(leaf.data))
        else:
            out.append(np.linalg.norm(leaf.data.value()) if leaf.data.k else 0.0)
    return np.array(out)


def ranks(h, hm):
    return np.array([leaf.data.k for leaf in h.leaves() if leaf.kind == hm.LOWRANK], dtype=np.int32)


def forward_y(h, rhs, hm, hlu_mod, blocks_mod, clustering_mod):
    col = clustering_mod.Cluster(0, 1, np.array([0.0]), np.array([0.0]))
    blk = blocks_mod.BlockNode(h.block.row, col, blocks_mod.INADMISSIBLE)
    leaf = hm.HMatrix(blk, hm.DENSE, rhs.reshape(-1, 1).copy())
    hlu_mod.solve_lower_hmatrix(h, leaf)
    return leaf.data[:, 0].copy()


def run_case(name, build, ctl_args, store_flat=False, store_dump=True):
    blocks, clustering, hlu, hm, kernels, lowrank = _ref()
    t0 = time.perf_counter()
    h, tree_dump = build(blocks, clustering, hm, kernels, lowrank)
    t_asm = time.perf_counter() - t0
    rec = {}
    dump = hm.structure_dump(h)
    rec["structure_sha"] = hashlib.sha256(dump.encode()).hexdigest()
    if store_dump:
        rec["structure_dump"] = dump
    if tree_dump is not None:
        rec["cluster_dump_sha"] = hashlib.sha256(tree_dump.encode()).hexdigest()
    rec["payload_sha"] = payload_hash(h, hm)
    rec["ranks_in"] = ranks(h, hm)
    if store_flat:
        rec["flat_in"] = hm.flatten(h)
    plan = hlu.make_plan(h, lowrank.TruncationControl(*ctl_args))
    t0 = time.perf_counter()
    hlu.hlu_factorize(plan)
    t_lu = time.perf_counter() - t0
    rec["flops"] = plan.flops.total
    rec["ranks_out"] = ranks(h, hm)
    rec["norms_out"] = leaf_norms(h, hm)
    rec["factor_sha"] = payload_hash(h, hm)
    rhs = np.random.default_rng(0).standard_normal(h.rows)
    rec["rhs"] = rhs
    rec["y_forward"] = forward_y(h, rhs, hm, hlu, blocks, clustering)
    if store_flat:
        rec["flat_out"] = hm.flatten(h)
    rec["ctl"] = np.array([ctl_args[0], -1 if ctl_args[1] is None else ctl_args[1]], dtype=float)
    rec["timing"] = np.array([t_asm, t_lu])
    np.savez_compressed(os.path.join(OUT, f"{name}.npz"), **rec)
    print(f"{name}: assembly {t_asm:.1f}s factor {t_lu:.1f}s flops {rec['flops']:.4e}", flush=True)


def bem(d, n, eta, leaf, eps, kmax):
    def build(blocks, clustering, hm, kernels, lowrank):
        case = kernels.make_bem_case(d, n, eta, leafsize=leaf, eps=eps, kmax=kmax)
        return case.hmatrix, case.tree.dump()

    return build


def mixed(n, leafsize, eta, seed):
    """Same construction as the reference tests' mixed_matrix (test_hlu.py:41)."""

    def build(blocks, clustering, hm, kernels, lowrank):
        tree = clustering.build_cluster_tree(np.linspace(0.0, 1.0, n), leafsize)
        root = blocks.build_block_tree(tree, tree, eta)
        rng = np.random.default_rng(seed)

        def fill(block):
            if block.kind == "admissible":
                k = int(rng.integers(1, 4))
                return lowrank.LowRank(
                    rng.standard_normal((block.rows, k)) / n, rng.standard_normal((block.cols, k))
                )
            m = rng.standard_normal((block.rows, block.cols))
            if block.row_range == block.col_range:
                m += n * np.eye(block.rows)
            return m

        return hm.build_hmatrix(root, fill), tree.dump()

    return build


def dense2x2(n, r, seed):
    def build(blocks, clustering, hm, kernels, lowrank):
        root, _ = blocks.build_diagonal_2x2_tree(n, r)
        rng = np.random.default_rng(seed)

        def fill(block):
            m = rng.standard_normal((block.rows, block.cols))
            if block.row_range == block.col_range:
                m += n * np.eye(block.rows)
            return m

        return hm.build_hmatrix(root, fill), None

    return build


CASES = {
    # small, exact-flat cases
    "mixed_192": (mixed(192, 16, 0.5, 3), (1e-8, None), True, True),
    "mixed_256_kmax": (mixed(256, 16, 0.5, 4), (1e-12, 3), True, True),
    "dense2x2_256_r3": (dense2x2(256, 3, 0), (1e-6, None), True, True),
    "bem1d_1024": (bem(1, 1024, 1.0, 32, 1e-6, None), (1e-6, None), False, True),
    "sphere_1024": (bem(3, 1024, 2.0, 32, 0.0, 8), (1e-6, None), False, True),
    "sphere_2048_l64": (bem(3, 2048, 2.0, 64, 1e-4, None), (1e-4, None), False, True),
    # BASELINE configs
    "cfg1": (bem(3, 4096, 2.0, 32, 0.0, 8), (1e-6, None), False, True),
    "cfg3p_8192": (bem(3, 8192, 2.0, 64, 1e-4, None), (1e-4, None), False, False),
    "cfg2": (bem(3, 32768, 2.0, 64, 1e-6, 32), (1e-6, 32), False, False),
    "cfg3": (bem(3, 131072, 2.0, 64, 1e-4, None), (1e-4, None), False, False),
    # cfg4 geometry / leaf size / truncation at a size the reference finishes in minutes
    "cfg4p_16384": (bem(3, 16384, 2.0, 128, 1e-4, 48), (1e-4, 48), False, False),
}

DEFAULT = ["mixed_192", "mixed_256_kmax", "dense2x2_256_r3", "bem1d_1024", "sphere_1024",
           "sphere_2048_l64", "cfg1"]


if __name__ == "__main__":
    names = sys.argv[1:] or DEFAULT
    for nm in names:
        build, ctl, flat, dump = CASES[nm]
        run_case(nm, build, ctl, store_flat=flat, store_dump=dump)
