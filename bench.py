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
region).  H-LU does not shard into independent units; under torchrun with N
ranks ONE factorization runs owner-computes over the N GPUs with NCCL slot
exchanges (strong scaling).
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
    # cfg4 geometry at the size one GPU holds (the full n=524288 needs the 8-GPU sharded path)
    "cfg4p": (3, 131072, 2.0, 128, 1e-4, 48, 1e-4, 48),
    # HODLR on the unit circle, rank-32 off-diagonal blocks (GPU cross approximation + truncation)
    "cfg5": (2, 1048576, None, 256, 0.0, 32, 1e-10, 32),
    "cfg5s": (2, 131072, None, 256, 0.0, 32, 1e-10, 32),
}
DEFAULT_CONFIG = os.environ.get("HLU_BENCH_CONFIG", "cfg3")  # BASELINE metric config (n=131072)


def _traffic():
    """DRAM bytes per launch of the dominant kernel family from the committed ncu
    --set full capture (profiles/r02/rkt_traffic.json), else None."""
    try:
        with open(os.path.join(ROOT, "profiles", "r02", "rkt_traffic.json")) as f:
            return json.load(f)
    except Exception:
        return None


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
    if eta is None:  # HODLR (cfg5): GPU generator
        from paper_1906_00874_b200 import gpu_assembly

        return gpu_assembly.hodlr_case(n, leafsize=leaf, k=kmax, generator="aca",
                                       device=f"cuda:{os.environ.get('LOCAL_RANK', '0')}")[0]
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


def run_sharded(args, world, rank, local, dev, dist):
    """One H-LU factorization on WORLD_SIZE GPUs (one process each): owner
    computes over a skewed cyclic slot map (square index blocks), the native sharded plan per
    rank, slot exchanges as gather -> ncclBroadcast -> scatter inside each
    rank's CUDA graph, final gather (every rank ends with the whole factor).
    Timed on the device with CUDA events, max over ranks; total work is fixed
    as N grows (strong scaling)."""
    import numpy as np
    import torch

    from paper_1906_00874_b200 import TruncationControl, multigpu
    from paper_1906_00874_b200.device import DeviceCall
    from paper_1906_00874_b200.hlu import _auto_capacity

    cfg = args.config
    *_, lu_eps, lu_kmax = CONFIGS[cfg]
    ctl = TruncationControl(lu_eps, lu_kmax)
    os.environ["HLU_ASSEMBLY_WORKERS"] = str(max(1, (os.cpu_count() or 1) // world))
    t0 = time.perf_counter()
    h = build_case(cfg)
    t_asm = time.perf_counter() - t0
    cap = _auto_capacity([h], ctl)
    comm = multigpu.Communicator(dist, rank, world, dev)
    t0 = time.perf_counter()
    layout, owner, packed = multigpu.shard_plan(h, world, rank, cap)
    t_plan = time.perf_counter() - t0
    call = DeviceCall(layout, packed, ctl, device=dev, use_graph=True, comm=comm)
    call.launch()
    call.check_errors()
    flops = call.flops()
    call.upload()
    call.snapshot()
    flush = torch.empty(int(256 * 2**20 // 4), dtype=torch.float32, device=dev)
    stream = call.stream
    for _ in range(args.warmup):
        call.restore()
        call.launch()
    call.sync()
    dist.barrier()
    torch.cuda.synchronize()
    clocks = Clocks(local)
    times = []
    for _ in range(args.steps):
        with torch.cuda.stream(stream):
            flush.fill_(1.0)
        call.restore()
        call.sync()
        dist.barrier()
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
    tt = torch.tensor([float(np.mean(times))], device=dev)
    dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    t_step = float(tt.item())
    # end to end: pinned host payloads -> every GPU, sharded factorization,
    # factors back to the host on rank 0; wall time, max over ranks
    e2e = []
    for _ in range(max(2, min(args.steps, 5))):
        torch.cuda.synchronize()
        dist.barrier()
        s0 = time.perf_counter()
        call.upload()
        call.launch()
        if rank == 0:
            call.download()
        call.sync()
        e2e.append(time.perf_counter() - s0)
    te = torch.tensor([float(np.mean(e2e[1:]))], device=dev)
    dist.all_reduce(te, op=dist.ReduceOp.MAX)
    t_e2e = float(te.item())
    mask = packed.op_mask
    share = [int(((mask >> np.uint64(r)) & np.uint64(1)).sum()) for r in range(world)]
    xfer_bytes = int(((packed.xfer["len"] + 1) * 8).sum()) if packed.xfer is not None else 0
    res = {
        "metric": "H-LU factorization effective fp64 GFLOP/s (reference FlopCounter / time)",
        "value": flops / t_step / 1e9,
        "unit": "GFLOP/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": t_step * 1e3,
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic (BASELINE BEM sphere geometry, Laplace kernel; seeded)",
        "config": bench_config(cfg),
        "details": {"factor_time_s": t_step, "effective_flops": flops,
                    "parallelism": f"owner computes over {world} GPUs (skewed cyclic slot owners over square index blocks), "
                                   "NCCL slot exchanges per level, final gather",
                    "ops_per_rank": share, "exchange_bytes_per_rank_broadcast_total": xfer_bytes,
                    "levels": int(packed.nlevels), "assembly_s": t_asm, "plan_s": t_plan, "rank_capacity": cap},
        "e2e": {"value": flops / t_e2e / 1e9, "unit": "GFLOP/s", "time_s": t_e2e,
                "h2d_bytes_per_step": int(call.h2d_bytes) * world,
                "d2h_bytes_per_step": int(layout.payload_doubles * 8 + call.ranks.numel() * 4)},
        "gpu_launches": int(len(packed.launches)),
        "roofline": None,
        "clocks": cl,
    }
    call.close()
    comm.close()
    if rank == 0:
        print(json.dumps(res))
    dist.destroy_process_group()


def bench_config(cfg):
    """The workload the line is quoted on; identical for both arms (--impl ours / reference)."""
    d, n, eta, leaf, eps, kmax, lu_eps, lu_kmax = CONFIGS[cfg]
    return {"workload": workload_name(cfg), "n": n, "leaf": leaf, "eta": eta, "lu_eps": lu_eps,
            "lu_kmax": lu_kmax, "l2": "flushed (256 MiB write) before every timed step"}


def _restore_payloads(h, template):
    """Put the template's (pristine, assembled) payloads back into h (same structure)."""
    from paper_1906_00874_b200.hmatrix import DENSE
    from paper_1906_00874_b200.lowrank import LowRank

    for a, b in zip(h.leaves(), template.leaves()):
        if a.kind == DENSE:
            a.data[:] = b.data
        else:
            a.data = LowRank(b.data.a, b.data.b)


def run_ours(args):
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_1906_00874_b200 import TruncationControl, hlu_factorize, make_plan, residual_probe
    from paper_1906_00874_b200.device import DeviceCall
    from paper_1906_00874_b200.hlu import _auto_capacity, plan_call

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus and rank == 0:
        print(f"bench: --gpus {args.gpus} but WORLD_SIZE {world}: launch N ranks with torchrun", file=sys.stderr)
    torch.cuda.set_device(local)
    dev = f"cuda:{local}"
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device(dev))
        return run_sharded(args, world, rank, local, dev, dist)
    cfg = args.config
    *_, lu_eps, lu_kmax = CONFIGS[cfg]
    ctl = TruncationControl(lu_eps, lu_kmax)
    t0 = time.perf_counter()
    h = build_case(cfg)
    t_asm = time.perf_counter() - t0
    template = h.copy()
    # One-shot through the public API, plan cache off: hlu_factorize(make_plan(h))
    # of a new structure pays the native planning (level schedule: seconds to
    # set up), the pools / descriptors / CUDA graph, the pinned upload, the
    # factorization and the download; everything is freed afterwards.
    os.environ["HLU_PLAN_CACHE"] = ""
    os.environ["HLU_PLAN_TIMING"] = "1"
    cap = _auto_capacity([h], ctl)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    once = make_plan(h, ctl, device=dev, capacity=cap)
    hlu_factorize(once)
    torch.cuda.synchronize()
    oneshot = time.perf_counter() - t0
    cap = once.capacity
    del once
    import gc

    gc.collect()
    torch.cuda.empty_cache()
    _restore_payloads(h, template)
    # Plan once, factorize many: keep_schedule selects the launch-DAG schedule
    # (its CUDA graphs take about two minutes to instantiate at cfg3) and keeps
    # it on the plan; the timed steps below replay it.
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    plan = make_plan(h, ctl, device=dev, keep_schedule=True, capacity=cap)
    hlu_factorize(plan)
    torch.cuda.synchronize()
    first_replayable = time.perf_counter() - t0
    call = plan.last_call
    t_plan, t_setup = getattr(call, "plan_s", None), getattr(call, "setup_s", None)
    cap = plan.capacity
    layout = call.L
    flops = call.flops()
    # residual of the GPU factors (reference bench.py:142-152), products on the GPU
    resid = residual_probe(template, h, device=dev)
    # device-resident steps: pristine payloads back into HBM once, then a
    # device-to-device restore before every step (outside the events)
    _restore_payloads(h, template)
    call.refill()
    call.upload()
    call.snapshot()
    flush = torch.empty(int(256 * 2**20 // 4), dtype=torch.float32, device=dev)
    stream = call.stream
    for _ in range(args.warmup):
        call.restore()
        call.launch()
    call.sync()
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
    # dominant kernel family (Rk truncations): algorithmic bytes of every
    # truncation of the step, from the ranks the kernels logged
    byts = rk_bytes_per_launch(call)
    h2d_bytes = int(call.h2d_bytes)
    d2h_bytes = int(layout.payload_doubles * 8 + call.ranks.numel() * 4)
    packed = call.packed
    nlevels, nops = int(packed.nlevels), int(len(packed.flop_formula))
    launches = int(len(packed.launches))
    dag = bool(getattr(call, "dag", False))
    nodes = int(call.lib.hlu_schedule_graph_nodes(call.handle)) if dag else None
    sched = {"kind": "dag" if dag else "levels", "launches": launches,
             "arena_gb": packed.arena_doubles * 8 / 1e9}
    if dag:
        from paper_1906_00874_b200 import native_plan

        sched.update({"slot_us": native_plan.dag_slot_ns_default() / 1e3, "kernel_nodes": nodes,
                      "dependency_edges": int(len(packed.dag_idx)),
                      "note": "launch DAG replayed as CUDA graphs whose edges are the planner's launch "
                              "dependencies (no level barriers); HLU_DAG_SLOT_US=0 selects the level schedule"})
    else:
        sched["levels"] = nlevels
    # per-launch durations exist only where launches do not overlap (level
    # schedule, device stamps); the DAG overlaps truncation launches with one
    # another and with the dense launches, so there the family's rate is its
    # bytes over the whole step (a lower bound on the kernels' own rate)
    if dag:
        durs, stamped_total = [], 0.0
    else:
        durs, stamped_total = time_rkt_launches(call, torch)
    # end to end through the public API: hlu_factorize(plan) with the schedule
    # kept on the plan -> every step re-packs the host payloads into pinned
    # buffers, uploads them, replays the graphs, downloads and installs the factors
    e2e_times = []
    for i in range(max(2, min(args.steps, 5))):
        _restore_payloads(h, template)
        torch.cuda.synchronize()
        s0 = time.perf_counter()
        hlu_factorize(plan)
        torch.cuda.synchronize()
        e2e_times.append(time.perf_counter() - s0)
    t_e2e = float(np.mean(e2e_times))
    plan.last_call.close()
    peak, peak_kind = _peaks()
    n_rkt = len(byts)
    avg_b = float(np.mean(byts)) if byts else 0.0
    if durs:
        avg_t = float(np.mean(durs))
        rkt_share = float(np.sum(durs)) / stamped_total if stamped_total > 0 else 0.0
        timing = ("device %globaltimer stamps between graph launch entries (re-captured graph, same buffers); "
                  f"share = sum / stamped step {stamped_total * 1e3:.1f} ms")
    else:
        avg_t = t_step / max(n_rkt, 1)
        rkt_share = 1.0
        timing = ("DAG schedule: truncation launches overlap one another and the dense launches over the whole "
                  "step, so avg_launch_ms = step time / truncation launches and achieved = all truncation bytes "
                  "of the step / step time (CUDA events on the launching stream); kernel-alone rates: "
                  "profiles/r02 ncu summaries")
    achieved = avg_b / avg_t / 1e9 if avg_t > 0 else 0.0
    res = {
        "metric": "H-LU factorization effective fp64 GFLOP/s (reference FlopCounter / time)",
        "value": flops / t_step / 1e9,
        "unit": "GFLOP/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": t_step * 1e3,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic (BASELINE BEM sphere geometry, Laplace kernel; seeded)",
        "config": bench_config(cfg),
        "details": {"factor_time_s": t_step, "effective_flops": flops,
                    "parallelism": "single GPU" if world == 1 else f"{world} independent replicas (rank 0 reported)",
                    "schedule": sched, "ops": nops, "assembly_s": t_asm, "plan_s": t_plan,
                    "device_setup_s": t_setup, "rank_capacity": cap,
                    "one_shot_s": oneshot,
                    "one_shot_note": "hlu_factorize(make_plan(h)) of a new structure, plan cache off: native "
                                     "planning (level schedule) + pools/descriptors/CUDA graph + pinned upload + "
                                     "factorization + download into the HMatrix, then freed",
                    "first_call_keep_schedule_s": first_replayable,
                    "first_call_keep_schedule_note": "make_plan(h, keep_schedule=True) + first hlu_factorize: "
                                                     "plans the launch-DAG schedule and instantiates its CUDA "
                                                     "graphs (plan_s + device_setup_s) once; the timed steps "
                                                     "and e2e replay it",
                    "residual_probe": resid,
                    "residual_note": "max_x ||A x - L (U x)|| / ||A x|| over 10 seeded probes "
                                     "(reference bench.py:142-152), GPU products"},
        "e2e": {"value": flops / t_e2e / 1e9, "unit": "GFLOP/s", "time_s": t_e2e,
                "h2d_bytes_per_step": h2d_bytes, "d2h_bytes_per_step": d2h_bytes,
                "path": "public API hlu_factorize(plan) with the schedule kept on the plan: host payload "
                        "packing into pinned buffers, H2D, graph replay, D2H, factors installed in the HMatrix"},
        "gpu_launches": nodes if nodes else launches,
        "roofline": {"kernel": "k_rkt_* (Rk truncation: block TSQR, core QRCP+Jacobi SVD, Q apply)",
                     "bound": "hbm",
                     "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak if peak else None, "traffic": _traffic(),
                     "peak_source": peak_kind, "launches_timed": n_rkt,
                     "avg_launch_ms": avg_t * 1e3, "avg_alg_bytes": avg_b,
                     "share_of_step": rkt_share, "timing": timing},
        "clocks": cl,
    }
    if rank == 0 and world == 1 and not args.no_kernel_roofline:
        # the batched leaf / Rk-update kernels timed alone at the cfg3 leaf shapes
        try:
            sys.path.insert(0, os.path.join(ROOT, "tools"))
            import kernel_roofline

            call = plan.last_call = None  # free the schedule's pools (payload + arena)
            torch.cuda.empty_cache()
            res["roofline_kernels"] = kernel_roofline.measure(dev)
        except Exception as e:  # the headline line must still print
            res["roofline_kernels"] = {"error": f"{type(e).__name__}: {e}"}
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
            "wall_s": wall,
            "sample": f"{len(jobs)} leading diagonal sub-blocks (~{blocks[0].rows} rows each) of the {cfg} "
                      f"H-matrix factorized concurrently by the CPU oracle, one process per core; "
                      f"wall {wall:.1f}s, single-core per-block time {min(t for _, t in out):.1f}-{max(t for _, t in out):.1f}s"}


def workload_name(cfg):
    *_, lu_eps, lu_kmax = CONFIGS[cfg]
    if CONFIGS[cfg][2] is None:
        return (f"{cfg}: H-LU of the n={CONFIGS[cfg][1]} HODLR circle matrix (-log|x-y|/2pi, A_ii=1, leaf "
                f"{CONFIGS[cfg][3]}, rank-{CONFIGS[cfg][5]} off-diagonal blocks, LU eps {lu_eps}, kmax {lu_kmax})")
    return (f"{cfg}: H-LU of the n={CONFIGS[cfg][1]} BEM sphere matrix "
            f"(leaf {CONFIGS[cfg][3]}, eta 2, LU eps {lu_eps}, kmax {lu_kmax})")


def _fixture_reference_time(cfg):
    """The real reference's own sequential hlu_factorize time on the full config,
    measured in the build container when the golden fixture was made
    (tests/golden/make_golden.py, one Xeon core, OpenBLAS 1 thread)."""
    try:
        import numpy as np

        with np.load(os.path.join(ROOT, "tests", "golden", f"{cfg}.npz")) as z:
            return float(z["timing"][1]), float(z["flops"])
    except Exception:
        return None, None


def run_reference(args):
    """Reference arm: the CPU oracle (bit-identical restatement of the reference
    path, same LAPACK/BLAS calls) on the box's host cores, one process per core,
    on a bounded sample of the same workload: the leading diagonal sub-blocks of
    the same assembled matrix (~4k rows each).  The line's config equals the
    GPU arm's."""
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
    vals, walls = [], []
    last = None
    for _ in range(max(1, args.steps)):
        last = cpu_baseline(h, ctl, cfg)
        vals.append(last["value"])
        walls.append(last["wall_s"])
    v = sum(vals) / len(vals)
    t_full, f_full = _fixture_reference_time(cfg)
    res = {"impl": "reference", "metric": "H-LU factorization effective fp64 GFLOP/s (reference FlopCounter / time)",
           "value": v, "unit": "GFLOP/s", "n_gpus": 0, "steps": args.steps, "warmup": args.warmup,
           "ms_per_step": 1e3 * sum(walls) / len(walls),
           "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
           "data": "synthetic (BASELINE BEM sphere geometry, Laplace kernel; seeded)",
           "config": bench_config(cfg),
           "details": {"parallelism": "host cores (one process per core, each factorizing one leading "
                                      "diagonal sub-block of the same matrix)",
                       "full_config_reference_single_core_s": t_full,
                       "full_config_reference_single_core_gflops": (f_full / t_full / 1e9) if t_full else None,
                       "full_config_note": "the real reference's sequential hlu_factorize on the whole config, "
                                           "timed when the golden fixture was generated (build container, "
                                           "1 core); not re-run here (it takes ~15 min)"},
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
    ap.add_argument("--no-kernel-roofline", action="store_true")
    ap.add_argument("--cpu-budget", type=float, default=20.0)
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
