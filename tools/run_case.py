"""Plan + run one case on the GPU once (graph), for profiling.
Usage: python tools/run_case.py <case> [repeats]"""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
import cases
from paper_1906_00874_b200.device import DeviceCall
from paper_1906_00874_b200.lowrank import TruncationControl
from paper_1906_00874_b200.planner import Layout, Planner


def main():
    name = sys.argv[1]
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
    build, ctl = cases.CASES[name]
    h, _ = build()
    from paper_1906_00874_b200.hlu import plan_call
    L, pl = plan_call([h], [("factor", h)], 32)
    call = DeviceCall(L, pl, TruncationControl(*ctl), use_graph=True)
    call.snapshot()
    for r in range(reps):
        call.restore(); t0 = time.perf_counter(); call.launch(); call.sync()
        print(f"run {r}: {time.perf_counter()-t0:.4f}s", flush=True)
    call.check_errors()
    print("ok", name, "launches", len(call.packed.launches))



if __name__ == "__main__":
    main()
