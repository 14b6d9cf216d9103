"""Core-kernel (k_rkt_b) phase breakdown of one factorization (diagnostics).
Usage: HLU_LIB=libhlu_b200_prof.so python tools/bprof.py <case>"""
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]


def main():
    import cases
    from paper_1906_00874_b200 import _native
    from paper_1906_00874_b200.device import DeviceCall
    from paper_1906_00874_b200.hlu import plan_call
    from paper_1906_00874_b200.lowrank import TruncationControl

    build, ctl = cases.CASES[sys.argv[1]]
    h, _ = build()
    L, pl = plan_call([h], [("factor", h)], 32)
    call = DeviceCall(L, pl, TruncationControl(*ctl), use_graph=True)
    lib = _native.lib()
    buf = (ctypes.c_ulonglong * 32)()
    call.snapshot()
    call.launch()
    call.sync()
    lib.hlu_debug_bprof(buf, 1)
    sw0 = lib.hlu_debug_sweeps(1)
    call.restore()
    call.launch()
    call.sync()
    call.check_errors()
    lib.hlu_debug_bprof(buf, 0)
    names = ["ops", "R/combine", "core prod", "QRCP", "Jacobi+sig", "rank", "W+qrcp_apply", "combine apply"]
    for v, tag in ((0, "K<=32"), (1, "K>32")):
        ops = buf[8 * v]
        tot = sum(buf[8 * v + k] for k in range(1, 8))
        print(f"{tag}: ops {ops}  total {tot / 1.965e9:.3f} s-CTA  per op {tot / max(ops, 1) / 1965:.1f} us  "
              f"Jacobi sweeps per op {buf[16 + v] / max(ops, 1):.2f} rounds per op {buf[18 + v] / max(ops, 1):.1f}")
        for k in range(1, 8):
            print(f"   {names[k]:14s} {buf[8 * v + k] / 1.965e9:8.3f} s  {buf[8 * v + k] / max(ops, 1) / 1965:8.1f} us/op")
    rn = ["load + QR", "core (M, Jacobi, rank)", "Q apply"]
    for v, tag in ((0, "warp path KB=8"), (1, "warp path KB=16")):
        b = 20 + 6 * v
        ops = buf[b]
        print(f"{tag}: k_rkt_r<2,{8 << v}> ops {ops}  warp-core calls (r + bw) {buf[b + 5]}  "
              f"sweeps per call {buf[b + 4] / max(buf[b + 5], 1):.2f}")
        for k in range(3):
            print(f"   {rn[k]:24s} {buf[b + 1 + k] / 1.965e9:8.3f} s-warp  {buf[b + 1 + k] / max(ops, 1) / 1965:8.1f} us/op")
    print("jacobi sweeps (all paths, one run):", lib.hlu_debug_sweeps(0))


if __name__ == "__main__":
    main()
