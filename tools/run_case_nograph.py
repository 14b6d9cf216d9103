"""One non-graph factorization of a case (for ncu: every kernel launch is
profiled individually)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]


def main():
    import cases
    from paper_1906_00874_b200.device import DeviceCall
    from paper_1906_00874_b200.hlu import plan_call
    from paper_1906_00874_b200.lowrank import TruncationControl

    build, ctl = cases.CASES[sys.argv[1]]
    h, _ = build()
    L, pl = plan_call([h], [("factor", h)], 32)
    call = DeviceCall(L, pl, TruncationControl(*ctl), use_graph=False)
    call.launch()
    call.check_errors()
    print("ok", len(pl.rkt))


if __name__ == "__main__":
    main()
