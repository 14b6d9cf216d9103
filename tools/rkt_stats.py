"""Per-kind GPU time and Jacobi sweep statistics for a case (diagnostics)."""
import ctypes, os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
import numpy as np, torch
import cases
from paper_1906_00874_b200 import _native, ir
from paper_1906_00874_b200.device import DeviceCall
from paper_1906_00874_b200.lowrank import TruncationControl
from paper_1906_00874_b200.planner import Layout, Planner


def main():
    name = sys.argv[1]
    build, ctl = cases.CASES[name]
    h, _ = build()
    from paper_1906_00874_b200.hlu import plan_call
    L, pl = plan_call([h], [("factor", h)], 32)
    call = DeviceCall(L, pl, TruncationControl(*ctl), use_graph=False)
    lib = _native.lib(); lib.hlu_debug_sweeps.restype = ctypes.c_int64; lib.hlu_debug_sweeps.argtypes=[ctypes.c_int]
    call.launch(); call.check_errors(); call.snapshot()
    p = call.packed
    st = ctypes.c_void_p(call.stream.cuda_stream); ctx = ctypes.byref(call.ctx)
    call.restore(); call.sync(); lib.hlu_debug_sweeps(1)
    import numpy as _np
    ph_s = _np.zeros(10); ph_m = _np.zeros(10)
    lib.hlu_debug_phases.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int]
    lib.hlu_debug_phases(ph_s.ctypes.data, ph_m.ctypes.data, 1)
    tot = {}
    evs = []
    lib.hlu_epoch_bump.argtypes = [ctypes.c_void_p]
    lib.hlu_epoch_bump(st)
    with torch.cuda.stream(call.stream):
        for L_ in p.launches:
            kind, count, first, dim = int(L_["kind"]), int(L_["count"]), int(L_["first"]), int(L_["smem_dim"])
            e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
            e0.record(call.stream)
            if kind == ir.K_GETRF: lib.hlu_getrf_batched_f64(ctx, call.d_getrf.data_ptr() + first*ir.GETRF.itemsize, count, dim, st)
            elif kind == ir.K_TRSM: lib.hlu_trsm_batched_f64(ctx, call.d_trsm.data_ptr() + first*ir.TRSM.itemsize, count, dim, st)
            elif kind == ir.K_GEMM: lib.hlu_gemm_batched_f64(ctx, call.d_gemm.data_ptr() + first*ir.GEMM.itemsize, call.d_terms.data_ptr(), count, st)
            elif kind == ir.K_GEMM_SMALL: lib.hlu_gemm_small_batched_f64(ctx, call.d_gemm.data_ptr() + first*ir.GEMM.itemsize, call.d_terms.data_ptr(), count, st)
            else: lib.hlu_rk_update_batched_f64(ctx, call.d_rkt.data_ptr() + first*ir.RKT.itemsize, call.d_parts.data_ptr(), count, 32 if kind == 3 else 64, st)
            e1.record(call.stream); evs.append((kind, count, e0, e1))
    call.sync()
    for kind, count, a, b in evs:
        t = a.elapsed_time(b)
        k = ["getrf","trsm","gemm","rkt32","rkt64","gemmw"][kind]
        tt = tot.setdefault(k, [0, 0, 0.0, 0.0]); tt[0] += 1; tt[1] += count; tt[2] += t; tt[3] = max(tt[3], t)
    nrkt = len(p.rkt)
    print("sweeps total", lib.hlu_debug_sweeps(0), "rkt ops", nrkt)
    lib.hlu_debug_phases(ph_s.ctypes.data, ph_m.ctypes.data, 0)
    names = ["parts", "tsqr", "core M", "qrcp", "XT+pairs", "jacobi", "rank+W", "apply_q"]
    for i, nm in enumerate(names):
        print(f"phase {nm:9s} total Mcyc {ph_s[i]/1e6:10.1f}  avg/op kcyc {ph_s[i]/nrkt/1e3:8.2f}  max kcyc {ph_m[i]/1e3:9.1f}")
    for k, (nl, nops, t, mx) in tot.items():
        print(f"{k:6s} launches {nl:6d} ops {nops:8d} total {t:9.2f} ms  per-launch {t/nl:7.3f} ms  max {mx:7.3f}")
    # RKT launch time vs the largest factor height in the launch
    import collections as _c
    byb = _c.defaultdict(lambda: [0, 0.0])
    for li, (kind, count, a, b) in enumerate(evs):
        if kind not in (ir.K_RKT32, ir.K_RKT64):
            continue
        L_ = p.launches[li]
        d_ = p.rkt[int(L_["first"]): int(L_["first"]) + int(L_["count"])]
        mm = int(max(d_["m"].max(), d_["n"].max()))
        bucket = 1 << max(0, (mm - 1).bit_length())
        byb[(kind, bucket)][0] += 1
        byb[(kind, bucket)][1] += a.elapsed_time(b)
    for (kind, bucket), (cnt, t) in sorted(byb.items()):
        print(f"rkt kind {kind} max(m,n) <= {bucket:6d}: launches {cnt:6d} total {t:9.1f} ms")
    # the slowest GEMM launch: what is in it
    worst = max(((a.elapsed_time(b), i) for i, (kind, count, a, b) in enumerate(evs) if kind == ir.K_GEMM), default=None)
    if worst:
        L_ = p.launches[worst[1]]
        first, count = int(L_["first"]), int(L_["count"])
        print("slowest gemm launch", worst, "descs", count)
        for gi in range(first, first + min(count, 400)):
            g = p.gemm[gi]
            ts = p.terms[int(g["term_begin"]): int(g["term_begin"]) + int(g["term_count"])]
            big = [(int(t["kind"]), int(t["c"]["rows"]), int(t["c"]["cols"]), int(t["a"]["cols"]), int(t["m"]["rows"]), int(t["m"]["cols"]), int(t["b"]["rows"]), int(t["assoc"])) for t in ts]
            work = sum(c_r * c_c * max(a_c, 1) + mr * mc * c_c for (_, c_r, c_c, a_c, mr, mc, b_r, _) in big)
            if gi < first + 3 or work > 5e7 or len(ts) > 100:
                print("  desc", gi, "terms", len(ts), "work", f"{work:.3g}", big[:4])
    call.restore(); call.sync()
    t0 = time.perf_counter(); e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(call.stream); call.launch(); e1.record(call.stream); call.sync()
    print("non-graph full run ms", e0.elapsed_time(e1))



if __name__ == "__main__":
    main()
