import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np
from oracle import hlu_oracle as orc
from paper_1906_00874_b200 import device_ops
from paper_1906_00874_b200.lowrank import LowRank, TruncationControl
rng = np.random.default_rng(0)
ctl = TruncationControl(1e-4)
for (m, n, K) in [(45, 55, 83), (45, 55, 84), (46, 58, 81), (64, 80, 100), (45, 55, 65), (64, 64, 65), (100, 100, 83), (45, 200, 83), (200, 55, 83)]:
    a = rng.standard_normal((m, K)) * (0.8 ** np.arange(K))
    b = rng.standard_normal((n, K))
    want = orc.recompress(LowRank(a, b), ctl)
    got = device_ops.recompress(LowRank(a, b), ctl)
    print(m, n, K, "gpu", got.k, "cpu", want.k, "err", np.linalg.norm(got.value() - want.value()) / np.linalg.norm(want.value()), flush=True)
