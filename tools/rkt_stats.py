"""Per-kind GPU time of a case, the truncation phases timed separately, RKT
level time by the largest factor height, Jacobi sweeps (diagnostics)."""
import collections
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]


def main():
    import numpy as np
    import torch

    import cases
    from paper_1906_00874_b200 import _native, ir
    from paper_1906_00874_b200.device import DeviceCall
    from paper_1906_00874_b200.hlu import plan_call
    from paper_1906_00874_b200.lowrank import TruncationControl

    name = sys.argv[1]
    build, ctl = cases.CASES[name]
    h, _ = build()
    L, pl = plan_call([h], [("factor", h)], 32)
    call = DeviceCall(L, pl, TruncationControl(*ctl), use_graph=False)
    lib = _native.lib()
    call.launch()
    call.check_errors()
    call.snapshot()
    p = call.packed
    st = ctypes.c_void_p(call.stream.cuda_stream)
    ctx = ctypes.byref(call.ctx)
    call.restore()
    call.sync()
    lib.hlu_debug_sweeps(1)
    evs = []
    with torch.cuda.stream(call.stream):
        for li, L_ in enumerate(p.launches):
            kind, count, first, dim = int(L_["kind"]), int(L_["count"]), int(L_["first"]), int(L_["smem_dim"])
            if kind == ir.K_RKT32:
                call._scratch_keep[0].zero_()
                for which in range(7):
                    e0 = torch.cuda.Event(enable_timing=True)
                    e1 = torch.cuda.Event(enable_timing=True)
                    e0.record(call.stream)
                    lib.hlu_rkt_phase(ctx, call.d_rkt.data_ptr(), call.d_parts.data_ptr(), first, count,
                                      ctypes.byref(call.scratch), 0, which, st)
                    e1.record(call.stream)
                    evs.append((li, ["rkt0cls", "rkt1w16", "rkt2w32", "rkt3A", "rkt4B32", "rkt5B64", "rkt6C"][which],
                                count, e0, e1))
                continue
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(call.stream)
            if kind == ir.K_GETRF:
                lib.hlu_getrf_batched_f64(ctx, call.d_getrf.data_ptr() + first * ir.GETRF.itemsize, count, dim, st)
            elif kind == ir.K_TRSM:
                lib.hlu_trsm_batched_f64(ctx, call.d_trsm.data_ptr() + first * ir.TRSM.itemsize, count, dim, st)
            elif kind == ir.K_GEMM:
                lib.hlu_gemm_batched_f64(ctx, call.d_gemm.data_ptr() + first * ir.GEMM.itemsize,
                                         call.d_terms.data_ptr(), count, st)
            elif kind == ir.K_GEMM_SMALL:
                lib.hlu_gemm_small_batched_f64(ctx, call.d_gemm.data_ptr() + first * ir.GEMM.itemsize,
                                               call.d_terms.data_ptr(), count, st)
            e1.record(call.stream)
            evs.append((li, ["getrf", "trsm", "gemm", "rkt", "rkt64", "gemmw"][kind], count, e0, e1))
    call.sync()
    call.check_errors()
    tot = {}
    per_launch = collections.defaultdict(float)
    for li, k, count, a, b in evs:
        t = a.elapsed_time(b)
        tt = tot.setdefault(k, [0, 0, 0.0, 0.0])
        tt[0] += 1
        tt[1] += count
        tt[2] += t
        tt[3] = max(tt[3], t)
        if k.startswith("rkt"):
            per_launch[li] += t
    print("jacobi sweeps total", lib.hlu_debug_sweeps(0), "rkt ops", len(p.rkt))
    for k, (nl, nops, t, mx) in tot.items():
        print(f"{k:7s} launches {nl:6d} ops {nops:8d} total {t:9.2f} ms  per-launch {t / nl:7.3f} ms  max {mx:7.3f}")
    byb = collections.defaultdict(lambda: [0, 0.0])
    for li, t in per_launch.items():
        L_ = p.launches[li]
        d_ = p.rkt[int(L_["first"]): int(L_["first"]) + int(L_["count"])]
        mm = int(max(d_["m"].max(), d_["n"].max()))
        bucket = 1 << max(0, (mm - 1).bit_length())
        byb[bucket][0] += 1
        byb[bucket][1] += t
    for bucket, (cnt, t) in sorted(byb.items()):
        print(f"rkt level max(m,n) <= {bucket:6d}: launches {cnt:6d} total {t:9.1f} ms  avg {t / cnt:7.3f} ms")
    call.restore()
    call.sync()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(call.stream)
    call.launch()
    e1.record(call.stream)
    call.sync()
    print("non-graph full run ms", e0.elapsed_time(e1))
    g = DeviceCall(L, pl, TruncationControl(*ctl), use_graph=True)
    g.launch()
    g.sync()
    for _ in range(2):
        g.upload()
        e0.record(g.stream)
        g.launch()
        e1.record(g.stream)
        g.sync()
        print("graph full run ms", e0.elapsed_time(e1))


if __name__ == "__main__":
    main()
