"""Per-kernel rooflines of the batched leaf and Rk-update kernels (C ABI,
include/hlu_b200.h) at the cfg3 leaf shapes: every kernel timed alone with CUDA
events on a batch of independent descriptors whose working set exceeds L2
(126 MB), so operands stream from HBM.  Algorithmic flops / bytes per op:

  gemm   C(64x64) -= A(64x64) B(64x64)          2 n^3 flops,      8 * 4 n^2 B   (read A, B, C; write C)
  chain  the same C updated by 8 such terms     8 * 2 n^3,        8 * (2 * 8 + 2) n^2 B
  getrf  unpivoted LU of a 64x64 block          2/3 n^3,          8 * 2 n^2 B
  trsm   X(64x64) <- L^-1 X                     n^2 r,            8 * (n^2 / 2 + 2 n r) B
  rk     add_truncated of two rank-k blocks     (SVD-type work)   8 (m + n)(K + k') B

peaks: fp64 = the DMMA/DFMA peak measured by tools/micro/fp64_peak.cu
(profiles/r02/fp64_peak.json), HBM = MEASURED_PEAKS.json.  bench.py imports
``measure`` for its ``roofline_kernels`` list; run standalone (optionally
under ncu) with ``python tools/kernel_roofline.py``.
"""
from __future__ import annotations

import ctypes
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

INT32_MAX = np.iinfo(np.int32).max


def _peaks():
    fp64, hbm = 37.0, 6650.0
    try:
        fp64 = float(json.load(open(os.path.join(ROOT, "profiles", "r02", "fp64_peak.json")))["dmma_m16n8k8_tflops"])
    except Exception:
        pass
    try:
        hbm = float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"])
    except Exception:
        pass
    return fp64, hbm


class _Bench:
    def __init__(self, torch, device, doubles, nranks, nlog, eps):
        from paper_1906_00874_b200 import _native

        self.torch, self.device, self.native = torch, device, _native
        self.pool = torch.zeros(doubles, dtype=torch.float64, device=device)
        self.ranks = torch.zeros(max(nranks, 1), dtype=torch.int32, device=device)
        self.log = torch.zeros(max(nlog, 8), dtype=torch.int32, device=device)
        self.err = torch.tensor([0, INT32_MAX, 0, 0], dtype=torch.int32, device=device)
        self.dlog = torch.zeros(2, dtype=torch.float64, device=device)
        self.ctx = _native.HluCtx(self.pool.data_ptr(), self.ranks.data_ptr(), self.log.data_ptr(),
                                  self.err.data_ptr(), self.dlog.data_ptr(), float(eps), -1, 0)

    def dev(self, rec):
        return self.torch.from_numpy(np.ascontiguousarray(rec).view(np.uint8)).to(self.device)

    def time(self, launch, reps):
        """ms per launch: pristine pool restored (outside the events) before every rep."""
        torch = self.torch
        pristine = self.pool.clone()
        ranks0 = self.ranks.clone()
        st = torch.cuda.current_stream(self.device)
        out = []
        for i in range(reps + 2):
            self.pool.copy_(pristine)
            self.ranks.copy_(ranks0)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            launch(ctypes.c_void_p(st.cuda_stream))
            e1.record(st)
            e1.synchronize()
            if i >= 2:
                out.append(e0.elapsed_time(e1))
        err = self.err.cpu().numpy()
        if err[0] or err[2] or err[1] != INT32_MAX:
            raise RuntimeError(f"kernel roofline: device error words {err.tolist()}")
        return float(np.mean(out))


def _view(off, rows, cols, dyn=-1):
    return (int(off), int(rows), int(cols), 1, int(rows), -1, int(dyn))


def _gemm(torch, device, lib, n, count, terms_per_chain, reps):
    from paper_1906_00874_b200 import ir

    per = (1 + 2 * terms_per_chain) * n * n
    B = _Bench(torch, device, per * count, 1, 8, 1e-4)
    B.pool.copy_(torch.randn(per * count, dtype=torch.float64, device=device))
    terms = np.zeros(count * terms_per_chain, dtype=ir.TERM)
    g = np.zeros(count, dtype=ir.GEMM)
    base = np.arange(count, dtype=np.int64) * per
    for t in range(terms_per_chain):
        sl = terms[t::terms_per_chain]
        for name, off in (("c", base), ("a", base + (1 + 2 * t) * n * n), ("b", base + (2 + 2 * t) * n * n)):
            sl[name]["off"] = off
            sl[name]["rows"] = n
            sl[name]["cols"] = n
            sl[name]["rs"] = 1
            sl[name]["cs"] = n
            sl[name]["rdyn"] = -1
            sl[name]["cdyn"] = -1
        sl["m"]["rdyn"] = -1
        sl["m"]["cdyn"] = -1
        sl["alpha"] = -1.0 / n
        sl["kind"] = ir.TERM_GEMM
    g["term_begin"] = np.arange(count) * terms_per_chain
    g["term_count"] = terms_per_chain
    g["log"] = -1
    g["log_slot"] = -1
    dg, dt = B.dev(g), B.dev(terms)

    def launch(stream):
        B.native.check(lib.hlu_gemm_batched_f64(ctypes.byref(B.ctx), dg.data_ptr(), dt.data_ptr(), count, stream),
                       "hlu_gemm_batched_f64")

    ms = B.time(launch, reps)
    flops = 2.0 * n ** 3 * terms_per_chain * count
    byts = 8.0 * (2 * terms_per_chain + 2) * n * n * count
    return ms, flops, byts


def _getrf(torch, device, lib, n, count, reps):
    from paper_1906_00874_b200 import ir

    B = _Bench(torch, device, n * n * count, 1, 8, 1e-4)
    a = torch.randn(count, n, n, dtype=torch.float64, device=device)
    a += n * torch.eye(n, dtype=torch.float64, device=device)
    B.pool.copy_(a.reshape(-1))
    d = np.zeros(count, dtype=ir.GETRF)
    d["a"]["off"] = np.arange(count, dtype=np.int64) * n * n
    d["a"]["rows"] = n
    d["a"]["cols"] = n
    d["a"]["rs"] = 1
    d["a"]["cs"] = n
    d["a"]["rdyn"] = -1
    d["a"]["cdyn"] = -1
    d["op_id"] = np.arange(count)
    dd = B.dev(d)

    def launch(stream):
        B.native.check(lib.hlu_getrf_batched_f64(ctypes.byref(B.ctx), dd.data_ptr(), count, n, stream),
                       "hlu_getrf_batched_f64")

    ms = B.time(launch, reps)
    return ms, 2.0 / 3.0 * n ** 3 * count, 8.0 * 2 * n * n * count


def _trsm(torch, device, lib, n, r, count, reps):
    from paper_1906_00874_b200 import ir

    per = n * n + n * r
    B = _Bench(torch, device, per * count, 1, 8, 1e-4)
    blk = torch.randn(count, per, dtype=torch.float64, device=device)
    t = blk[:, : n * n].reshape(count, n, n)
    t /= n
    t += torch.eye(n, dtype=torch.float64, device=device)
    B.pool.copy_(blk.reshape(-1))
    d = np.zeros(count, dtype=ir.TRSM)
    base = np.arange(count, dtype=np.int64) * per
    for name, off, rows, cols in (("t", base, n, n), ("x", base + n * n, n, r)):
        d[name]["off"] = off
        d[name]["rows"] = rows
        d[name]["cols"] = cols
        d[name]["rs"] = 1
        d[name]["cs"] = rows
        d[name]["rdyn"] = -1
        d[name]["cdyn"] = -1
    d["mode"] = ir.TRSM_LOWER_UNIT
    d["log"] = -1
    dd = B.dev(d)

    def launch(stream):
        B.native.check(lib.hlu_trsm_batched_f64(ctypes.byref(B.ctx), dd.data_ptr(), count, n, stream),
                       "hlu_trsm_batched_f64")

    ms = B.time(launch, reps)
    return ms, float(n * n * r) * count, 8.0 * (n * n / 2 + 2 * n * r) * count


def _rk(torch, device, lib, m, k, count, reps, eps=1e-4):
    """add_truncated of x1 (rank k) and x2 = x1 with its columns reversed (the
    sum has rank k exactly), outputs and workspaces per op."""
    from paper_1906_00874_b200 import ir

    n, K = m, 2 * k
    ws = int(ir.rkt_ws_doubles(m, n, K))
    per = 2 * (m + n) * k + (m + n) * K + ws
    B = _Bench(torch, device, per * count, 3 * count, 3 * count, eps)
    data = torch.zeros(count, per, dtype=torch.float64, device=device)
    x1 = torch.randn(count, (m + n) * k, dtype=torch.float64, device=device)
    data[:, : (m + n) * k] = x1
    a1 = x1[:, : m * k].reshape(count, k, m)  # column-major: column j = a1[:, j, :]
    b1 = x1[:, m * k :].reshape(count, k, n)
    data[:, (m + n) * k : (m + n) * k + m * k] = a1.flip(1).reshape(count, -1)
    data[:, (m + n) * k + m * k : 2 * (m + n) * k] = b1.flip(1).reshape(count, -1)
    B.pool.copy_(data.reshape(-1))
    del data, x1
    rk = torch.zeros(3 * count, dtype=torch.int32, device=device)
    rk[0::3] = k
    rk[1::3] = k
    B.ranks.copy_(rk)
    base = np.arange(count, dtype=np.int64) * per
    parts = np.zeros(2 * count, dtype=ir.RKPART)
    for j in range(2):
        sl = parts[j::2]
        for name, off, rows in (("a", base + j * (m + n) * k, m), ("b", base + j * (m + n) * k + m * k, n)):
            sl[name]["off"] = off
            sl[name]["rows"] = rows
            sl[name]["cols"] = k
            sl[name]["rs"] = 1
            sl[name]["cs"] = rows
            sl[name]["rdyn"] = -1
            sl[name]["cdyn"] = 3 * np.arange(count) + j
        sl["sign"] = 1.0
    d = np.zeros(count, dtype=ir.RKT)
    d["mode"] = ir.RK_ADD
    d["part_begin"] = 2 * np.arange(count)
    d["part_count"] = 2
    d["m"] = m
    d["n"] = n
    d["cap"] = K
    d["out_slot"] = 3 * np.arange(count) + 2
    d["log"] = 3 * np.arange(count)
    d["out_a"] = base + 2 * (m + n) * k
    d["out_b"] = base + 2 * (m + n) * k + m * K
    d["ws"] = base + 2 * (m + n) * k + (m + n) * K
    launches = np.zeros(1, dtype=ir.LAUNCH)
    launches[0] = (ir.K_RKT32, count, 0, 0, 0)
    sc, keep = B.native.rkt_scratch(torch, device, d, launches)
    dd, dp = B.dev(d), B.dev(parts)

    def launch(stream):
        B.native.check(lib.hlu_rk_update_batched_f64(ctypes.byref(B.ctx), dd.data_ptr(), dp.data_ptr(), count,
                                                     ctypes.byref(sc), stream), "hlu_rk_update_batched_f64")

    ms = B.time(launch, reps)
    kout = B.ranks.cpu().numpy()[2::3]
    if not (kout == k).all():
        raise RuntimeError(f"kernel roofline: truncation ranks {np.unique(kout)} != {k}")
    del keep
    return ms, None, 8.0 * (m + n) * (K + k) * count


def measure(device="cuda:0", reps=5):
    """List of per-kernel roofline records (see the module docstring)."""
    import torch

    from paper_1906_00874_b200 import _native

    lib = _native.lib()
    fp64, hbm = _peaks()
    out = []

    def rec(name, what, ms, flops, byts, count):
        r = {"kernel": name, "workload": what, "ops_per_launch": count, "ms_per_launch": ms,
             "achieved_gbs": byts / ms / 1e6, "hbm_peak_gbs": hbm, "hbm_frac": byts / ms / 1e6 / hbm}
        if flops is not None:
            r.update({"achieved_tflops": flops / ms / 1e9, "fp64_peak_tflops": fp64,
                      "fp64_frac": flops / ms / 1e9 / fp64})
            r["bound"] = "hbm" if r["hbm_frac"] >= r["fp64_frac"] else "fp64"
            r["frac"] = max(r["hbm_frac"], r["fp64_frac"])
        else:
            r["bound"] = "hbm"
            r["frac"] = r["hbm_frac"]
        out.append(r)

    with torch.cuda.device(device):
        c = 148 * 32
        ms, fl, by = _gemm(torch, device, lib, 64, c, 1, reps)
        rec("k_gemm", "independent C(64x64) -= A(64x64) B(64x64), DMMA m16n8k8", ms, fl, by, c)
        c = 148 * 8
        ms, fl, by = _gemm(torch, device, lib, 64, c, 8, reps)
        rec("k_gemm (8-term chains)", "chains of 8 terms on one 64x64 C", ms, fl, by, c)
        c = 148 * 96
        ms, fl, by = _getrf(torch, device, lib, 64, c, reps)
        rec("k_getrf", "unpivoted LU of 64x64 leaves (DMMA panel updates)", ms, fl, by, c)
        c = 148 * 48
        ms, fl, by = _trsm(torch, device, lib, 64, 64, c, reps)
        rec("k_trsm", "X(64x64) <- L^-1 X, unit lower 64x64", ms, fl, by, c)
        c = 16384
        ms, fl, by = _rk(torch, device, lib, 64, 8, c, reps)
        rec("k_rkt_* (64-row blocks)", "add_truncated, m = n = 64, k1 = k2 = 8 -> 8 (register warp kernels)", ms, fl,
            by, c)
        c = 148 * 8
        ms, fl, by = _rk(torch, device, lib, 512, 10, c, reps)
        rec("k_rkt_* (512-row blocks)", "add_truncated, m = n = 512, k1 = k2 = 10 -> 10 (block TSQR, core, Q apply)",
            ms, fl, by, c)
        torch.cuda.empty_cache()
    return out


if __name__ == "__main__":
    for r in measure():
        print(json.dumps(r))
