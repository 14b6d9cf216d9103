"""Planner dry run of the owner-computes sharding (no GPU): per-rank op
counts, arena and payload memory, and the NCCL exchange volume of one H-LU.
Usage: python tools/shard_stats.py <bench config> <nranks> [rank ...]"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
import numpy as np

import bench
from paper_1906_00874_b200 import TruncationControl, multigpu
from paper_1906_00874_b200.hlu import _auto_capacity


def main():
    cfg, world = sys.argv[1], int(sys.argv[2])
    which = [int(x) for x in sys.argv[3:]] or list(range(world))
    *_, lu_eps, lu_kmax = bench.CONFIGS[cfg]
    ctl = TruncationControl(lu_eps, lu_kmax)
    t0 = time.perf_counter()
    h = bench.build_case(cfg)
    t_asm = time.perf_counter() - t0
    cap = _auto_capacity([h], ctl)
    out = {"config": cfg, "nranks": world, "assembly_s": t_asm, "capacity": cap, "ranks": []}
    for r in which:
        t0 = time.perf_counter()
        layout, owner, p = multigpu.shard_plan(h, world, r, cap)
        dt = time.perf_counter() - t0
        x = p.xfer
        lv = x["level"].astype(np.int64)
        final = lv == int(p.nlevels)
        mine = x["src"] == r
        byts = (x["len"].astype(np.int64) + 1) * 8
        groups = len(np.unique(np.stack([lv[~final], x["src"][~final].astype(np.int64), x["group"][~final].astype(np.int64)]), axis=1).T) if (~final).any() else 0
        mask = p.op_mask
        rec = {
            "rank": r, "plan_s": dt, "levels": int(p.nlevels), "launches": int(len(p.launches)),
            "ops_total": int(len(mask)),
            "ops_per_rank": [int(((mask >> np.uint64(q)) & np.uint64(1)).sum()) for q in range(world)],
            "payload_gb": layout.payload_doubles * 8 / 1e9, "arena_gb": p.arena_doubles * 8 / 1e9,
            "exchange_records": int((~final).sum()), "exchange_groups": int(groups),
            "exchange_gb_all_sources": float(byts[~final].sum() / 1e9),
            "exchange_gb_from_this_rank": float(byts[~final & mine].sum() / 1e9),
            "exchange_levels": int(len(np.unique(lv[~final]))),
            "mean_bytes_per_group": float(byts[~final].sum() / max(groups, 1)),
            "final_gather_gb": float(byts[final].sum() / 1e9),
            "owned_slots": int((owner == r).sum()), "slots": int(len(owner)),
        }
        out["ranks"].append(rec)
        print(json.dumps(rec), flush=True)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
