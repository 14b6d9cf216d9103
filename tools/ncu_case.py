"""One non-graph factorization of a case for ncu (every launch is profiled on
its own).  Prints the Rk-truncation launch count and their algorithmic bytes
(8 (m+n)(K+k') per truncation, from the ranks the kernels log),
the numbers tools/rkt_traffic.py divides the ncu dram bytes by.
Usage: python tools/ncu_case.py <case>"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
os.environ.setdefault("HLU_DAG_SLOT_US", "0")  # level-ordered launch list: every launch replays serially without a graph
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]


def main():
    import cases
    import bench
    from paper_1906_00874_b200.device import DeviceCall
    from paper_1906_00874_b200.hlu import plan_call
    from paper_1906_00874_b200.lowrank import TruncationControl

    name = sys.argv[1]
    build, ctl = cases.CASES[name]
    h, _ = build()
    L, pl = plan_call([h], [("factor", h)], 32)
    call = DeviceCall(L, pl, TruncationControl(*ctl), use_graph=False)
    call.launch()
    call.check_errors()
    byts = bench.rk_bytes_per_launch(call)
    print(json.dumps({"case": name, "rkt_launches": len(byts), "rkt_alg_bytes": float(sum(byts)),
                      "truncations": int(len(pl.rkt)), "flops": call.flops(),
                      "rkt_alg_bytes_per_launch": [float(b) for b in byts]}))


if __name__ == "__main__":
    main()
