"""Benchmark: H-LU factorization of the BASELINE BEM sphere configs on B200.

Metric (BASELINE.json): H-LU factorization time and effective fp64 GFLOP/s
(the reference's FlopCounter numerator, ``hlu.py:46-55``; GFLOP/s = counter /
time as ``bench.py:96-98`` of the reference).

  python bench.py [--config cfg3] [--steps K] [--warmup W] [--gpus N]
  python bench.py --impl reference ...   # CPU oracle on the box's host cores

A step is one factorization of the assembled H-matrix.  ``value`` is measured
with the inputs resident in HBM (a device-to-device restore of the pristine
payload precedes every step, outside the events; L2 is flushed between steps);
``e2e`` goes through the public plugin path with pinned host buffers
(host->device upload, factorization, device->host download inside the timed
region).  H-LU does not shard into independent units; with --gpus N every
rank factorizes its own replica ("replicas only") and the
aggregate is reported.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import time

for _v in ("OPENBLAS_NUM_THREADS", "OMP_NUM_THREADS", "MKL_NUM_THREADS"):
    os.environ.setdefault(_v, "1")  # host assembly runs one process per core

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

CONFIGS = {
    # name: (d, n, eta, leaf, asm eps, asm kmax, LU eps, LU kmax)
    "cfg1": (3, 4096, 2.0, 32, 0.0, 8, 1e-6, None),
    "cfg2": (3, 32768, 2.0, 64, 1e-6, 32, 1e-6, 32),
    "cfg3": (3, 131072, 2.0, 64, 1e-4, None, 1e-4, None),
}
DEFAULT_CONFIG = os.environ.get("HLU_BENCH_CONFIG", "cfg3")  # BASELINE metric config (n=131072)


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class Clocks:
    """nvidia-smi sampling during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0):
        self.proc = None
        self.path = f"/tmp/hlu_clocks_{os.getpid()}.csv"
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return None
        self.proc.terminate()
        self.proc.wait()
        rows = []
        for line in open(self.path):
            parts = [x.strip() for x in line.split(",")]
            if len(parts) >= 7:
                rows.append(parts)
        if not rows:
            return None
        sm = sorted(float(r[0]) for r in rows if r[0].replace(".", "").isdigit())
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[3 + i] == "Active"})
        return {"sm_mhz": sm[len(sm) // 2] if sm else None, "sm_max_mhz": float(rows[0][1]),
                "reasons": reasons, "samples": len(rows)}


def build_case(cfg):
    from paper_1906_00874_b200 import make_bem_case

    d, n, eta, leaf, eps, kmax, _, _ = CONFIGS[cfg]
    workers = int(os.environ.get("HLU_ASSEMBLY_WORKERS", str(os.cpu_count() or 1)))
    return make_bem_case(d, n, eta, leafsize=leaf, eps=eps, kmax=kmax, workers=workers).hmatrix


def rk_bytes_per_launch(call):
    """Algorithmic HBM bytes of every RKT launch (8 (m+n)(K+k') per truncation)."""
    import numpy as np

    p = call.packed
    log = call.log.cpu().numpy().astype(np.int64)
    out = []
    for L in p.launches:
        if int(L["kind"]) not in (3,):
            continue
        first, cnt = int(L["first"]), int(L["count"])
        d = p.rkt[first:first + cnt]
        lg = d["log"].astype(np.int64)
        k1, k2, ko = log[lg], log[lg + 1], log[lg + 2]
        K = np.where(d["mode"] == 0, k1 + k2, k1)
        by = 8.0 * (d["m"].astype(np.int64) + d["n"]) * (K + ko)
        out.append(float(by.sum()))
    return out


def time_rkt_launches(call, torch):
    """GPU time of every truncation launch group (classify + warp kernels + the
    three CTA phases of one level) inside the CUDA graph, from device
    %globaltimer stamps between launch-list entries (DeviceCall.launch_times)."""
    from paper_1906_00874_b200 import ir

    call.restore()
    dt = call.launch_times()
    kinds = call.packed.launches["kind"]
    return [float(t) for t, k in zip(dt, kinds) if int(k) == ir.K_RKT32], float(dt.sum())


def run_ours(args):
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_1906_00874_b200 import TruncationControl
    from paper_1906_00874_b200.hlu import _auto_capacity, plan_call
    from paper_1906_00874_b200.device import DeviceCall

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        dist.init_process_group("nccl")
    torch.cuda.set_device(local)
    cfg = args.config
    *_, lu_eps, lu_kmax = CONFIGS[cfg]
    ctl = TruncationControl(lu_eps, lu_kmax)
    t0 = time.perf_counter()
    h = build_case(cfg)
    t_asm = time.perf_counter() - t0
    template = h.copy()
    t0 = time.perf_counter()
    cap = _auto_capacity([h], ctl)
    layout, packed = plan_call([h], [("factor", h)], cap)
    call = DeviceCall(layout, packed, ctl, device=f"cuda:{local}", use_graph=True)
    t_plan = time.perf_counter() - t0
    call.launch()
    call.check_errors()  # RankOverflow here would need a larger capacity
    flops = call.flops()
    # pristine copy for the timed device-resident steps
    call.upload()
    call.snapshot()
    flush = torch.empty(int(256 * 2**20 // 4), dtype=torch.float32, device=f"cuda:{local}")
    stream = call.stream
    for _ in range(args.warmup):
        call.restore()
        call.launch()
    call.sync()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clocks = Clocks(local)
    times = []
    for _ in range(args.steps):
        with torch.cuda.stream(stream):
            flush.fill_(1.0)
        call.restore()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        call.launch()
        e1.record(stream)
        call.sync()
        times.append(e0.elapsed_time(e1) * 1e-3)
    torch.cuda.synchronize()
    cl = clocks.stop()
    call.check_errors()
    t_step = float(np.mean(times))
    if world > 1:
        tt = torch.tensor([t_step], device=f"cuda:{local}")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_step = float(tt.item())
    # end-to-end through the plugin path with host buffers
    host_out = torch.empty(layout.payload_doubles, dtype=torch.float64).pin_memory()
    e2e_times = []
    for i in range(max(2, min(args.steps, 5))):
        torch.cuda.synchronize()
        s0 = time.perf_counter()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        call.upload()
        call.launch()
        with torch.cuda.stream(stream):
            host_out.copy_(call.pool[: layout.payload_doubles], non_blocking=True)
            hr = call.ranks.to("cpu", non_blocking=True)
        e1.record(stream)
        call.sync()
        e2e_times.append(e0.elapsed_time(e1) * 1e-3)
    t_e2e = float(np.mean(e2e_times[1:])) if len(e2e_times) > 1 else e2e_times[0]
    # dominant kernel roofline (Rk truncations), CUDA events per launch
    durs, stamped_total = time_rkt_launches(call, torch)
    byts = rk_bytes_per_launch(call)
    peak, peak_kind = _peaks()
    n_rkt = len(durs)
    avg_t = float(np.mean(durs)) if durs else 0.0
    avg_b = float(np.mean(byts)) if byts else 0.0
    achieved = avg_b / avg_t / 1e9 if avg_t > 0 else 0.0
    rkt_share = float(np.sum(durs)) / stamped_total if stamped_total > 0 else 0.0
    launches = int(len(call.packed.launches))
    res = {
        "metric": "H-LU factorization effective fp64 GFLOP/s (reference FlopCounter / time)",
        "value": world * flops / t_step / 1e9,
        "unit": "GFLOP/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": t_step * 1e3,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic (BASELINE BEM sphere geometry, Laplace kernel; seeded)",
        "config": {"workload": workload_name(cfg),
                   "n": CONFIGS[cfg][1], "factor_time_s": t_step, "effective_flops": flops,
                   "l2": "flushed (256 MiB write) before every timed step",
                   "parallelism": "replicas only" if world > 1 else "single GPU",
                   "levels": call.packed.nlevels, "ops": len(packed.flop_formula),
                   "assembly_s": t_asm, "plan_s": t_plan, "rank_capacity": cap},
        "e2e": {"value": world * flops / t_e2e / 1e9, "unit": "GFLOP/s", "time_s": t_e2e,
                "h2d_bytes_per_step": int(call.h2d_bytes),
                "d2h_bytes_per_step": int(layout.payload_doubles * 8 + call.ranks.numel() * 4)},
        "gpu_launches": launches,
        "roofline": {"kernel": "k_rkt_a/b/c (Rk truncation: block TSQR, core QRCP+Jacobi SVD, Q apply)",
                     "bound": "hbm",
                     "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak if peak else None, "traffic": None,
                     "peak_source": peak_kind, "launches_timed": n_rkt,
                     "avg_launch_ms": avg_t * 1e3, "avg_alg_bytes": avg_b,
                     "share_of_step": rkt_share, "timing": "device %globaltimer stamps between graph "
                     "launch entries (re-captured graph, same buffers); share = sum / stamped step "
                     f"{stamped_total * 1e3:.1f} ms"},
        "clocks": cl,
    }
    if rank == 0 and not args.no_cpu_baseline and world == 1:
        res["cpu_baseline"] = cpu_baseline(template, ctl, cfg, budget=args.cpu_budget)
    if rank == 0:
        print(json.dumps(res))
    if world > 1:
        dist.destroy_process_group()


def _subblock(h, depth):
    """Leading diagonal sub-block ``depth`` partition levels down (same workload, smaller)."""
    x = h
    for _ in range(depth):
        if x.kind != "partitioned":
            break
        x = x.child(0, 0)
    return x


_CPU_JOBS = None


def _oracle_factor_job(i):
    from oracle import hlu_oracle

    h, ctl = _CPU_JOBS[i]
    h = h.copy()
    t0 = time.perf_counter()
    fl = hlu_oracle.hlu_factorize(h, ctl)
    return fl, time.perf_counter() - t0


def cpu_baseline(h, ctl, cfg, budget=20.0, procs=None):
    """The CPU oracle (restatement of the reference, same LAPACK calls) on a
    bounded sample: diagonal sub-blocks of the same H-matrix, one process per
    host core, aggregate effective GFLOP/s."""
    import multiprocessing as mp

    for v in ("OPENBLAS_NUM_THREADS", "OMP_NUM_THREADS", "MKL_NUM_THREADS"):
        os.environ[v] = "1"
    procs = procs or (os.cpu_count() or 1)
    # pick the depth whose sub-block takes a bounded time: n_sub ~ 4096 rows
    depth = 0
    sub = h
    while sub.rows > 4096 and sub.kind == "partitioned":
        depth += 1
        sub = _subblock(h, depth)
    # all diagonal sub-blocks at that depth
    blocks = [h]
    for _ in range(depth):
        nxt = []
        for b in blocks:
            if b.kind == "partitioned":
                nxt.extend(b.data[i][i] for i in range(len(b.data)))
            else:
                nxt.append(b)
        blocks = nxt
    global _CPU_JOBS
    jobs = [(b, ctl) for b in blocks[: max(procs, 1)]]
    _CPU_JOBS = jobs
    t0 = time.perf_counter()
    with mp.get_context("fork").Pool(min(procs, len(jobs))) as pool:
        out = pool.map(_oracle_factor_job, range(len(jobs)))
    wall = time.perf_counter() - t0
    flops = sum(f for f, _ in out)
    return {"value": flops / wall / 1e9, "unit": "GFLOP/s", "cores": min(procs, len(jobs)), "kind": "port",
            "sample": f"{len(jobs)} leading diagonal sub-blocks (~{blocks[0].rows} rows each) of the {cfg} "
                      f"H-matrix factorized concurrently by the CPU oracle, one process per core; "
                      f"wall {wall:.1f}s, single-core per-block time {min(t for _, t in out):.1f}-{max(t for _, t in out):.1f}s"}


def workload_name(cfg):
    *_, lu_eps, lu_kmax = CONFIGS[cfg]
    return (f"{cfg}: H-LU of the n={CONFIGS[cfg][1]} BEM sphere matrix "
            f"(leaf {CONFIGS[cfg][3]}, eta 2, LU eps {lu_eps}, kmax {lu_kmax})")


def run_reference(args):
    """Reference arm: the CPU oracle (port of the reference path) on host cores."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from paper_1906_00874_b200 import TruncationControl

    cfg = args.config
    *_, lu_eps, lu_kmax = CONFIGS[cfg]
    ctl = TruncationControl(lu_eps, lu_kmax)
    h = build_case(cfg)
    if args.warmup > 0:  # one untimed sample warms the BLAS / process pool
        cpu_baseline(h, ctl, cfg)
    vals = []
    last = None
    for _ in range(max(1, args.steps)):
        last = cpu_baseline(h, ctl, cfg)
        vals.append(last["value"])
    v = sum(vals) / len(vals)
    res = {"impl": "reference", "metric": "H-LU factorization effective fp64 GFLOP/s (reference FlopCounter / time)",
           "value": v, "unit": "GFLOP/s", "n_gpus": 0, "steps": args.steps, "warmup": args.warmup,
           "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
           "data": "synthetic (BASELINE BEM sphere geometry, Laplace kernel; seeded)",
           "config": {"workload": workload_name(cfg), "n": CONFIGS[cfg][1],
                      "parallelism": "host cores (one process per core)"},
           "cpu_baseline": {k: last[k] for k in ("kind", "cores", "sample")} | {"value": v, "unit": "GFLOP/s"},
           "e2e": {"value": v, "unit": "GFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(res))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default=DEFAULT_CONFIG, choices=sorted(CONFIGS))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-budget", type=float, default=20.0)
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
