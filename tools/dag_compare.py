"""Level schedule vs DAG schedule of one case on the GPU: the factors must be
bit-identical (same ops, same per-destination order), the times differ.
Usage: python tools/dag_compare.py <case> [slot_us ...]"""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
import numpy as np
import torch
import cases
from paper_1906_00874_b200 import native_plan
from paper_1906_00874_b200.device import DeviceCall
from paper_1906_00874_b200.lowrank import TruncationControl
from paper_1906_00874_b200.planner import Layout


def main():
    name = sys.argv[1]
    slots = [float(x) for x in sys.argv[2:]] or [20.0]
    build, ctl = cases.CASES[name]
    t0 = time.time()
    h, _ = build()
    print(f"build {time.time() - t0:.1f}s", flush=True)
    ref = None
    for slot in [0.0] + slots:
        L = Layout([h], cap=32, extra=[])
        t0 = time.time()
        packed, nops = native_plan._build(L, *_cmds(L, h), native_plan.SPLIT_ROWS, dag_slot_ns=int(slot * 1000))
        t_plan = time.time() - t0
        t0 = time.time()
        call = DeviceCall(L, packed, TruncationControl(*ctl), use_graph=True)
        call.sync()
        t_setup = time.time() - t0
        call.snapshot()
        times = []
        for r in range(4):
            call.restore()
            e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
            e0.record(call.stream); call.launch(); e1.record(call.stream); call.sync()
            times.append(e0.elapsed_time(e1))
        call.check_errors()
        n = L.payload_doubles
        pool = call.pool[:n].cpu().numpy().copy()
        ranks = call.ranks.cpu().numpy().copy()
        nodes = int(call.lib.hlu_schedule_graph_nodes(call.handle)) if slot else 0
        tag = "level" if slot == 0 else f"dag {slot:g}us"
        same = ""
        if ref is None:
            ref = (pool, ranks)
        else:
            same = f" ranks_equal={np.array_equal(ranks, ref[1])} pool_equal={pool.tobytes() == ref[0].tobytes()}"
            if pool.tobytes() != ref[0].tobytes():
                d = np.abs(pool - ref[0]); same += f" maxdiff={np.nanmax(d):.3e} ndiff={(d>0).sum()}"
        print(f"{name} {tag}: launches {len(packed.launches)} nodes {nodes} arena {packed.arena_doubles*8/1e9:.2f} GB "
              f"plan {t_plan:.1f}s setup {t_setup:.1f}s ms {[round(t, 2) for t in times]}{same}", flush=True)
        call.close()
        del call
        torch.cuda.empty_cache()


def _cmds(L, h):
    nodes, index = native_plan.flatten_nodes(L)
    cmds = np.zeros(1, dtype=native_plan.CMD)
    cmds[0] = (native_plan.CMD_FACTOR, index[id(h)], 0, 0, 0, 0, 0, 0, 0, 0)
    return nodes, cmds


if __name__ == "__main__":
    main()
