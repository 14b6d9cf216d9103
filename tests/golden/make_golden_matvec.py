"""Golden fixtures for the products with the matrix and its factors, from the
REAL reference (``hluflow``), run in the build container:

    python tests/golden/make_golden_matvec.py

For each case writes ``tests/golden/matvec_<case>.npz`` with ``x`` (n x 2,
``default_rng(1)``), the reference ``hmatvec(h, x)`` (hmatrix.py:178-200) of
the assembled matrix, ``lower_unit_matvec`` / ``upper_matvec`` (hlu.py:720-767)
of the factored matrix, and ``residual_probe(original, factored)``
(bench.py:142-152, seed 0, 10 probes = RESIDUAL_PROBES, bench.py:32).
"""

from __future__ import annotations

import copy
import os
import sys

for _v in ("OPENBLAS_NUM_THREADS", "OMP_NUM_THREADS", "MKL_NUM_THREADS"):
    os.environ[_v] = "1"

import numpy as np  # noqa: E402

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from make_golden import CASES, OUT, _ref  # noqa: E402

MATVEC_CASES = ["mixed_192", "bem1d_1024", "sphere_1024"]


def run(name):
    blocks, clustering, hlu, hm, kernels, lowrank = _ref()
    sys.path.insert(0, "/root/reference/pkg/src")
    from hluflow import bench as rbench

    build, ctl, _, _ = CASES[name]
    h, _ = build(blocks, clustering, hm, kernels, lowrank)
    orig = copy.deepcopy(h)
    x = np.random.default_rng(1).standard_normal((h.rows, 2))
    rec = {"x": x, "ax": hm.hmatvec(h, x)}
    hlu.hlu_factorize(hlu.make_plan(h, lowrank.TruncationControl(*ctl)))
    rec["lx"] = hlu.lower_unit_matvec(h, x)
    rec["ux"] = hlu.upper_matvec(h, x)
    rec["residual"] = np.array(rbench.residual_probe(orig, h))
    np.savez_compressed(os.path.join(OUT, f"matvec_{name}.npz"), **rec)
    print(name, float(rec["residual"]))


if __name__ == "__main__":
    for nm in sys.argv[1:] or MATVEC_CASES:
        run(nm)
