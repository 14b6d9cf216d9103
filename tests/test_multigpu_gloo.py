"""Owner-computes H-LU across 2 ranks (torch.distributed gloo on CPU): each
rank executes only the ops it owns on its own copy of the pool (CPU IR
machine standing in for a GPU), slots are exchanged after every level, and
both ranks end bit-identical to the single-process run."""

import os

import numpy as np
import pytest
import torch.multiprocessing as mp

import cases
from ir_exec import CpuMachine
from paper_1906_00874_b200 import ir, multigpu
from paper_1906_00874_b200.planner import Layout, Planner
from paper_1906_00874_b200.pool import fill_pool
from paper_1906_00874_b200.schedule import pack


def _plan(name):
    build, ctl = cases.CASES[name]
    h, _ = build()
    L = Layout(h, cap=32)
    pl = Planner(L)
    pl.factor(h)
    return h, L, pl, pack(pl, L.payload_doubles), ctl


def _machine(L, p, ctl):
    pool = np.zeros(L.payload_doubles + p.arena_doubles)
    ranks = np.zeros(p.nranks, np.int32)
    fill_pool(L, pool, ranks)
    return CpuMachine(pool, ranks, p.nlog, ctl[0], ctl[1])


def _worker(rank, world, name, port, out):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    h, L, pl, p, ctl = _plan(name)
    slot_owner = multigpu.owner_map(L, world)
    owner = multigpu.op_owners(pl, slot_owner)
    plan, _ = multigpu.exchange_plan(pl, p, owner)
    M = _machine(L, p, ctl)

    def execute(kind, d):
        if kind == ir.K_GETRF:
            M.getrf(p.getrf[d])
        elif kind == ir.K_TRSM:
            M.trsm(p.trsm[d])
        elif kind in (ir.K_GEMM, ir.K_GEMM_SMALL):
            M.gemm(p.gemm[d], p.terms)
        else:
            M.rkt(p.rkt[d], p.parts)

    multigpu.run_level_exchange(p, pl, owner, plan, rank, execute, M.pool, M.ranks, dist, slot_owner=slot_owner)
    np.save(f"{out}_{rank}_pool.npy", M.pool[: L.payload_doubles])
    np.save(f"{out}_{rank}_ranks.npy", M.ranks[: L.nrk])
    dist.destroy_process_group()


@pytest.mark.parametrize("name", ["mixed_192", "sphere_1024"])
def test_two_rank_owner_computes_matches_single(tmp_path, name):
    h, L, pl, p, ctl = _plan(name)
    ref = _machine(L, p, ctl)
    ref.run(p)
    port = 29500 + (os.getpid() % 1000)
    out = str(tmp_path / "r")
    mp.start_processes(_worker, args=(2, name, port, out), nprocs=2, join=True, start_method="fork")
    # rank 0 holds the gathered result, bit-identical to the single-process run
    pool = np.load(f"{out}_0_pool.npy")
    ranks = np.load(f"{out}_0_ranks.npy")
    assert np.array_equal(ranks, ref.ranks[: L.nrk])
    assert np.array_equal(pool, ref.pool[: L.payload_doubles])
    # every rank's own slots are final without the gather
    slot_owner = multigpu.owner_map(L, 2)
    pool1 = np.load(f"{out}_1_pool.npy")
    for s in range(len(L.leaves)):
        if slot_owner[s] == 1:
            off, ln = multigpu.slot_region(L, s)
            assert np.array_equal(pool1[off:off + ln], ref.pool[off:off + ln])


def test_owner_map_balance_and_volume():
    h, L, pl, p, ctl = _plan("sphere_1024")
    slot_owner = multigpu.owner_map(L, 4)
    owner = multigpu.op_owners(pl, slot_owner)
    counts = np.zeros(4)
    for o in owner:
        for r in o:
            counts[r] += 1
    assert counts.min() > 0 and counts.max() / counts.mean() < 2.0
    plan, vol = multigpu.exchange_plan(pl, p, owner)
    assert sum(vol.values()) > 0
    # temps never cross ranks: every consumer's ranks hold a producer replica
    prod = {}
    for i, op in enumerate(pl.ops):
        for t in op.temps_out:
            prod[t] = owner[i]
    for i, op in enumerate(pl.ops):
        for t in op.temps_in:
            assert owner[i] <= prod[t]


# ---- the native sharded planner (hlu_plan_build_sharded) -------------------------


def _native_worker(rank, world, name, port, out):
    import torch.distributed as dist

    from ir_exec import run_sharded
    from paper_1906_00874_b200 import native_plan

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    build, ctl = cases.CASES[name]
    h, _ = build()
    L = Layout(h, cap=32)
    owner = multigpu.owner_map(L, world)
    p, _ = native_plan.plan(L, [("factor", h)], shard=(owner, world, rank))
    M = _machine(L, p, ctl)
    run_sharded(M, p, rank, dist)
    np.save(f"{out}_{rank}_pool.npy", M.pool[: L.payload_doubles])
    np.save(f"{out}_{rank}_ranks.npy", M.ranks[: L.nrk])
    np.save(f"{out}_{rank}_log.npy", M.log)
    dist.destroy_process_group()


@pytest.mark.parametrize("name,world", [("mixed_192", 2), ("sphere_1024", 2), ("sphere_1024", 3)])
def test_native_sharded_plan_matches_single(tmp_path, name, world):
    """Every rank executes only its own ops from the native sharded plan, the
    exchange records move the written slots after each level, and after the
    final gather EVERY rank holds the single-GPU result bit for bit (payloads,
    ranks and the flop log)."""
    from paper_1906_00874_b200 import native_plan

    build, ctl = cases.CASES[name]
    h, _ = build()
    L = Layout(h, cap=32)
    p, _ = native_plan.plan(L, [("factor", h)])
    ref = _machine(L, p, ctl)
    ref.run(p)
    port = 29700 + (os.getpid() % 200) + 7 * world
    out = str(tmp_path / "r")
    mp.start_processes(_native_worker, args=(world, name, port, out), nprocs=world, join=True, start_method="fork")
    for r in range(world):
        assert np.array_equal(np.load(f"{out}_{r}_ranks.npy"), ref.ranks[: L.nrk])
        assert np.array_equal(np.load(f"{out}_{r}_pool.npy"), ref.pool[: L.payload_doubles])
        assert np.array_equal(np.load(f"{out}_{r}_log.npy"), ref.log)


def test_native_sharded_ops_partition():
    """The ranks' op sets cover every op; slot writers are unique; temp
    producers sit on every consuming rank; the exchange records never ship a
    slot from a rank that does not own it."""
    from paper_1906_00874_b200 import native_plan

    build, _ = cases.CASES["sphere_1024"]
    h, _ = build()
    L = Layout(h, cap=32)
    world = 4
    owner = multigpu.owner_map(L, world)
    full, nops = native_plan.plan(L, [("factor", h)])
    per = [native_plan.plan(L, [("factor", h)], shard=(owner, world, r))[0] for r in range(world)]
    mask = per[0].op_mask
    assert all(np.array_equal(q.op_mask, mask) for q in per)
    assert np.all(mask != 0)
    counts = [int(((mask >> np.uint64(r)) & np.uint64(1)).sum()) for r in range(world)]
    assert min(counts) > 0 and max(counts) / np.mean(counts) < 2.0
    ndesc = sum(len(q.rkt) + len(q.getrf) + len(q.trsm) for q in per)
    assert ndesc >= len(full.rkt) + len(full.getrf) + len(full.trsm)
    for q in per:
        x = q.xfer
        assert np.array_equal(x, per[0].xfer)
        slots = {}
        for lf_i, lf in enumerate(L.leaves):
            slots[multigpu.slot_region(L, lf_i)[0]] = lf_i
        for r in x:
            assert owner[slots[int(r["off"])]] == int(r["src"])
