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
    L = Layout(h, cap=32); pl = Planner(L); pl.factor(h)
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
    with torch.cuda.stream(call.stream):
        for L_ in p.launches:
            kind, count, first, dim = int(L_["kind"]), int(L_["count"]), int(L_["first"]), int(L_["smem_dim"])
            e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
            e0.record(call.stream)
            if kind == ir.K_GETRF: lib.hlu_getrf_batched_f64(ctx, call.d_getrf.data_ptr() + first*ir.GETRF.itemsize, count, dim, st)
            elif kind == ir.K_TRSM: lib.hlu_trsm_batched_f64(ctx, call.d_trsm.data_ptr() + first*ir.TRSM.itemsize, count, dim, st)
            elif kind == ir.K_GEMM: lib.hlu_gemm_batched_f64(ctx, call.d_gemm.data_ptr() + first*ir.GEMM.itemsize, call.d_terms.data_ptr(), count, st)
            else: lib.hlu_rk_update_batched_f64(ctx, call.d_rkt.data_ptr() + first*ir.RKT.itemsize, call.d_parts.data_ptr(), count, 32 if kind == 3 else 64, st)
            e1.record(call.stream); evs.append((kind, count, e0, e1))
    call.sync()
    for kind, count, a, b in evs:
        t = a.elapsed_time(b)
        k = ["getrf","trsm","gemm","rkt32","rkt64"][kind]
        tt = tot.setdefault(k, [0, 0, 0.0, 0.0]); tt[0] += 1; tt[1] += count; tt[2] += t; tt[3] = max(tt[3], t)
    nrkt = len(p.rkt)
    print("sweeps total", lib.hlu_debug_sweeps(0), "rkt ops", nrkt)
    lib.hlu_debug_phases(ph_s.ctypes.data, ph_m.ctypes.data, 0)
    names = ["parts", "tsqr", "core M", "qrcp", "XT+pairs", "jacobi", "rank+W", "apply_q"]
    for i, nm in enumerate(names):
        print(f"phase {nm:9s} total Mcyc {ph_s[i]/1e6:10.1f}  avg/op kcyc {ph_s[i]/nrkt/1e3:8.2f}  max kcyc {ph_m[i]/1e3:9.1f}")
    for k, (nl, nops, t, mx) in tot.items():
        print(f"{k:6s} launches {nl:6d} ops {nops:8d} total {t:9.2f} ms  per-launch {t/nl:7.3f} ms  max {mx:7.3f}")
    call.restore(); call.sync()
    t0 = time.perf_counter(); e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(call.stream); call.launch(); e1.record(call.stream); call.sync()
    print("non-graph full run ms", e0.elapsed_time(e1))



if __name__ == "__main__":
    main()
