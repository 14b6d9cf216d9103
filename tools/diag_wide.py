"""Diagnostics: GPU vs CPU-IR per-op truncation logs for one plan (finds the
first truncation whose (k1, k2, kout) differ)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def main():
    import numpy as np

    import cases
    from ir_exec import CpuMachine
    from paper_1906_00874_b200.device import DeviceCall
    from paper_1906_00874_b200.hlu import plan_call
    from paper_1906_00874_b200.lowrank import TruncationControl
    from paper_1906_00874_b200.pool import fill_pool

    name = sys.argv[1] if len(sys.argv) > 1 else "sphere_2048_l64"
    build, ctl = cases.CASES[name]
    h, _ = build()
    L, p = plan_call([h], [("factor", h)], 64)
    pool = np.zeros(L.payload_doubles + p.arena_doubles)
    ranks = np.zeros(p.nranks, np.int32)
    fill_pool(L, pool, ranks)
    M = CpuMachine(pool, ranks, p.nlog, ctl[0], ctl[1])
    M.run(p)
    call = DeviceCall(L, p, TruncationControl(*ctl), device="cuda:0",
                      use_graph=os.environ.get("HLU_NOGRAPH", "0") != "1")
    call.launch()
    call.sync()
    glog = call.log.cpu().numpy()
    print("err", call.err.cpu().numpy(), "cpu err", M.err)
    r = p.rkt
    lg = r["log"].astype(np.int64)
    nd = 0
    for i in np.argsort(lg):
        a, b = glog[lg[i]:lg[i] + 3], M.log[lg[i]:lg[i] + 3]
        if not np.array_equal(a, b):
            d = r[i]
            print("op", i, "mode", d["mode"], "m", d["m"], "n", d["n"], "parts", d["part_count"], "gpu", a, "cpu", b)
            nd += 1
            if nd > 10:
                break
    print("diffs", nd)


if __name__ == "__main__":
    main()
