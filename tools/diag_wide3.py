import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np
from paper_1906_00874_b200 import device_ops, ir
from paper_1906_00874_b200.lowrank import LowRank, TruncationControl
import paper_1906_00874_b200.device_ops as D
cap_S = {}
orig = D._Scratch.go
def go(self, fn):
    orig(self, fn); cap_S['S'] = self
D._Scratch.go = go
rng = np.random.default_rng(0)
ctl = TruncationControl(1e-4)
m, n, K = 45, 200, 83
a = rng.standard_normal((m, K)) * (0.8 ** np.arange(K))
b = rng.standard_normal((n, K))
got = device_ops.recompress(LowRank(a, b), ctl)
S = cap_S['S']
# layout: parts a (m*K), b (n*K), out_a m*cap, out_b n*cap, ws
off = 0
ao = 0; bo = m*K; oa = bo + n*K; ob = oa + m*K; ws = ob + n*K
X = S.out[ws: ws+m*K].reshape(K, m).T
Y = S.out[ws+m*K: ws+(m+n)*K].reshape(K, n).T
KW=128
M = S.out[ws+(m+n)*K: ws+(m+n)*K+KW*KW].reshape(KW, KW).T
V = S.out[ws+(m+n)*K+KW*KW: ws+(m+n)*K+2*KW*KW].reshape(KW, KW).T
tx = S.out[ws+(m+n)*K+2*KW*KW: ws+(m+n)*K+2*KW*KW+KW]
ty = tx + 0; ty = S.out[ws+(m+n)*K+2*KW*KW+KW: ws+(m+n)*K+2*KW*KW+2*KW]
sig = S.out[ws+(m+n)*K+2*KW*KW+2*KW: ws+(m+n)*K+2*KW*KW+3*KW]
print("k", got.k, "err", S.out_err, "log", S.log.cpu().numpy())
print("nan X", np.isnan(X).sum(), "nan Y", np.isnan(Y).sum(), "nan M", np.isnan(M).sum(), "nan V", np.isnan(V).sum(), "nan sig", np.isnan(sig[:K]).sum())
print("tx", tx[:5], "ty", ty[:5], ty[80:84])
print("sig", sig[:6])
Rx = np.triu(X[:m, :]); Ry = np.triu(Y[:K, :])
print("R check x", np.linalg.norm(np.abs(np.linalg.qr(a)[1]) - np.abs(Rx)), "y", np.linalg.norm(np.abs(np.linalg.qr(b)[1]) - np.abs(Ry)))
