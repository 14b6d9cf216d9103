"""Solve / residual fixtures at the BASELINE configs, from the REAL reference.

Run in the build container (``/root/reference`` exists there only):

    python tests/golden/make_golden_solve.py cfg1 cfg2 cfg3

For each case the reference assembles the BEM matrix and factorizes it with
its own ``hlu_factorize`` (``hlu.py:661-680``); then, in the same process:

* ``y = L^-1 b`` through the reference's ``solve_lower_hmatrix`` with an
  n x 1 dense leaf (``hlu.py:696-700``), b = ``default_rng(0).standard_normal(n)``;
* ``x = U^-1 y``: the reference has no backward vector solve, so the oracle's
  restated block back-substitution (``oracle/hlu_oracle.py:backward_solve``,
  mirroring ``_upper_into`` ``hlu.py:753-767``) runs on the REFERENCE's own
  factor payloads (copied leaf by leaf into an identically structured tree);
* the reference's own ``residual_probe(original, factored)``
  (``bench.py:142-152``: 10 probes, seed 0).

Output: ``tests/golden/solve_<case>.npz`` with rhs, y, x, residual.
"""

from __future__ import annotations

import os
import sys
import time

for _v in ("OPENBLAS_NUM_THREADS", "OMP_NUM_THREADS", "MKL_NUM_THREADS"):
    os.environ[_v] = "1"

import numpy as np  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, HERE)

from make_golden import CASES, _ref, forward_y  # noqa: E402


def run(name):
    blocks, clustering, hlu, hm, kernels, lowrank = _ref()
    from hluflow import bench as refbench

    from oracle import hlu_oracle
    from paper_1906_00874_b200 import make_bem_case
    from paper_1906_00874_b200.hmatrix import DENSE

    build, ctl, _, _ = CASES[name]
    t0 = time.perf_counter()
    h, _ = build(blocks, clustering, hm, kernels, lowrank)
    original = h.copy()
    t_asm = time.perf_counter() - t0
    plan = hlu.make_plan(h, lowrank.TruncationControl(*ctl))
    t0 = time.perf_counter()
    hlu.hlu_factorize(plan)
    t_lu = time.perf_counter() - t0
    rhs = np.random.default_rng(0).standard_normal(h.rows)
    y = forward_y(h, rhs, hm, hlu, blocks, clustering)
    res = refbench.residual_probe(original, h)
    del original
    # the reference's factors, leaf by leaf, in our (identical) structure
    cfgargs = {"cfg1": (3, 4096, 2.0, 32, 0.0, 8), "cfg2": (3, 32768, 2.0, 64, 1e-6, 32),
               "cfg3": (3, 131072, 2.0, 64, 1e-4, None), "cfg3p_8192": (3, 8192, 2.0, 64, 1e-4, None),
               "sphere_2048_l64": (3, 2048, 2.0, 64, 1e-4, None),
               "cfg4p_16384": (3, 16384, 2.0, 128, 1e-4, 48)}[name]
    d, n, eta, leaf, eps, kmax = cfgargs
    ours = make_bem_case(d, n, eta, leafsize=leaf, eps=eps, kmax=kmax,
                         workers=os.cpu_count() or 1).hmatrix
    mine, theirs = list(ours.leaves()), list(h.leaves())
    assert len(mine) == len(theirs)
    for a, b in zip(mine, theirs):
        assert a.row_range == b.row_range and a.col_range == b.col_range
        if a.kind == DENSE:
            a.data = b.data
        else:
            a.data = type(a.data)(b.data.a, b.data.b)
    x = hlu_oracle.backward_solve(ours, y)
    np.savez_compressed(os.path.join(HERE, f"solve_{name}.npz"), rhs=rhs, y=y, x=x,
                        residual=np.float64(res), ctl=np.array([ctl[0], -1 if ctl[1] is None else ctl[1]]),
                        timing=np.array([t_asm, t_lu]))
    print(f"{name}: asm {t_asm:.1f}s lu {t_lu:.1f}s residual {res:.3e} |x| {np.linalg.norm(x):.4e}",
          flush=True)


if __name__ == "__main__":
    for nm in sys.argv[1:] or ["cfg1"]:
        run(nm)
