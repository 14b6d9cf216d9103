"""Device runtime: pools in HBM, descriptor upload, one CUDA graph per call.

PyTorch provides the device memory and the stream; all arithmetic runs in
``libhlu_b200.so`` through the C ABI.  A ``DeviceCall`` owns

* the fp64 pool: leaf payloads (dense leaves, Rk factor slabs) followed by the
  temp/workspace arena planned by ``schedule.allocate_temps``,
* the rank table, the flop log and the error words,
* the packed descriptor arrays and the captured schedule (CUDA graph).

No CPU fallback exists: without the library or a GPU, construction raises.
"""

from __future__ import annotations

import ctypes
import os

import numpy as np

from . import _native
from .hmatrix import StructureError  # noqa: F401  (re-exported for callers)
from .lowrank import SingularBlockError
from .pool import fill_pool, leaf_chunks, read_extra, read_pool
from .schedule import Packed, effective_flops, pack

INT32_MAX = np.iinfo(np.int32).max
XFER_CHUNKS = 16  # pool ranges of the pipelined upload / download


class RankOverflow(RuntimeError):
    """An Rk result exceeded the reserved per-block capacity (re-plan larger)."""


def _torch():
    import torch

    if not torch.cuda.is_available():
        raise RuntimeError("paper_1906_00874_b200 needs a CUDA device (sm_100a); no CPU fallback")
    return torch


def _dev_bytes(torch, arr, device):
    t = torch.from_numpy(np.ascontiguousarray(arr).view(np.uint8)).to(device)
    return t


class DeviceCall:
    """One planned H-arithmetic call resident on the GPU."""

    def __init__(self, layout, packed, ctl, device=None, use_graph=True, extras=None, comm=None):
        torch = _torch()
        self.torch = torch
        self.device = torch.device(device if device is not None else "cuda")
        self.L = layout
        self.ctl = ctl
        lib = _native.lib()
        self.lib = lib
        if not isinstance(packed, Packed):  # a Python Planner: pack it here
            packed = pack(packed, layout.payload_doubles)
        self.packed: Packed = packed
        p = self.packed
        self.total = layout.payload_doubles + p.arena_doubles
        self.h2d_bytes = layout.payload_doubles * 8 + p.nranks * 4
        with torch.cuda.device(self.device):
            # blocks an earlier call freed stay in torch's caching allocator: hand
            # them back, the CUDA graphs below take driver memory beside the pools
            torch.cuda.empty_cache()
            # a dedicated stream: the legacy default stream cannot be graph-captured
            self.stream = torch.cuda.Stream(self.device)
        with torch.cuda.device(self.device), torch.cuda.stream(self.stream):
            self.pool = torch.empty(self.total, dtype=torch.float64, device=self.device)
            # pinned staging buffers (payloads packed natively, hlu_host_pack)
            self.host_pool = torch.zeros(layout.payload_doubles, dtype=torch.float64, pin_memory=True)
            self.host_ranks = torch.zeros(p.nranks, dtype=torch.int32, pin_memory=True)
            self.ranks = torch.empty(p.nranks, dtype=torch.int32, device=self.device)
            self.log = torch.zeros(p.nlog, dtype=torch.int32, device=self.device)
            self.err = torch.tensor([0, INT32_MAX, 0, 0], dtype=torch.int32, device=self.device)
            self.dlog = torch.zeros(2 * max(len(p.lu_labels), 1), dtype=torch.float64, device=self.device)
            self.d_getrf = _dev_bytes(torch, p.getrf, self.device)
            self.d_trsm = _dev_bytes(torch, p.trsm, self.device)
            self.d_gemm = _dev_bytes(torch, p.gemm, self.device)
            self.d_terms = _dev_bytes(torch, p.terms, self.device)
            self.d_rkt = _dev_bytes(torch, p.rkt, self.device)
            self.d_parts = _dev_bytes(torch, p.parts, self.device)
            # truncation scratch: per-launch counters, op lists, row-block items
            self.dag = p.dag_ptr is not None and p.shard is None and use_graph
            if self.dag:
                self.scratch, self._scratch_keep, item0, nitems = _native.rkt_scratch_dag(
                    torch, self.device, p.rkt, p.launches)
            else:
                self.scratch, self._scratch_keep = _native.rkt_scratch(torch, self.device, p.rkt, p.launches)
            self.refill_upload(extras)
            self.ctx = _native.HluCtx(
                self.pool.data_ptr(), self.ranks.data_ptr(), self.log.data_ptr(), self.err.data_ptr(),
                self.dlog.data_ptr(), float(ctl.eps), -1 if ctl.kmax is None else int(ctl.kmax), 0,
            )
            handle = ctypes.c_void_p()
            launches = np.ascontiguousarray(p.launches)
            self.comm = comm
            if p.shard is not None:
                # owner computes over the communicator: this rank's launches, the
                # slot exchanges after every level, the final gather
                if comm is None:
                    raise ValueError("a sharded plan needs a communicator (multigpu.Communicator)")
                self.chains = False
                xfer = np.ascontiguousarray(p.xfer)
                self.d_xfer = _dev_bytes(torch, xfer, self.device)
                nst = max(int(lib.hlu_xfer_staging_doubles(xfer.ctypes.data, len(xfer))), 1)
                self.staging = torch.empty(nst, dtype=torch.float64, device=self.device)
                rc = lib.hlu_schedule_create_sharded(
                    ctypes.byref(handle), ctypes.byref(self.ctx), launches.ctypes.data, len(launches),
                    self.d_getrf.data_ptr(), self.d_trsm.data_ptr(), self.d_gemm.data_ptr(),
                    self.d_terms.data_ptr(), self.d_rkt.data_ptr(), self.d_parts.data_ptr(),
                    ctypes.byref(self.scratch), comm.handle, xfer.ctypes.data, self.d_xfer.data_ptr(),
                    len(xfer), int(p.nlevels), int(p.nlog), self.staging.data_ptr(),
                    1 if use_graph else 0, ctypes.c_void_p(self.stream.cuda_stream),
                )
                _native.check(rc, "hlu_schedule_create_sharded")
            elif self.dag:
                # the launch DAG: one CUDA graph whose edges are the planner's
                # launch dependencies (no level barriers)
                self.chains = False
                dp = np.ascontiguousarray(p.dag_ptr, dtype=np.int64)
                di = np.ascontiguousarray(p.dag_idx if len(p.dag_idx) else np.zeros(1, np.int32), dtype=np.int32)
                # launches without model-time slack get a higher scheduling priority
                # (HLU_DAG_PRIO="t1,t2" in us: slack <= t1 high, <= t2 medium; "off": none)
                prio = None
                spec = os.environ.get("HLU_DAG_PRIO", "200,2000")
                if spec != "off" and p.dag_slack is not None:
                    t1, t2 = (float(x) * 1000.0 for x in spec.split(","))
                    sl = np.asarray(p.dag_slack[: len(launches)], dtype=np.int64)
                    prio = np.ascontiguousarray(np.where(sl <= t1, 2, np.where(sl <= t2, 1, 0)), dtype=np.int32)
                rc = lib.hlu_schedule_create_dag(
                    ctypes.byref(handle), ctypes.byref(self.ctx), launches.ctypes.data, len(launches),
                    self.d_getrf.data_ptr(), self.d_trsm.data_ptr(), self.d_gemm.data_ptr(),
                    self.d_terms.data_ptr(), self.d_rkt.data_ptr(), self.d_parts.data_ptr(),
                    ctypes.byref(self.scratch), dp.ctypes.data, di.ctypes.data, item0.ctypes.data,
                    nitems.ctypes.data, prio.ctypes.data if prio is not None else None,
                    ctypes.c_void_p(self.stream.cuda_stream),
                )
                _native.check(rc, "hlu_schedule_create_dag")
            else:
                # two chains (dense / truncation) with the planner's cross-chain
                # waits; HLU_CHAINS=0 keeps a barrier after every level
                chains = p.wait_dense is not None and os.environ.get("HLU_CHAINS", "1") != "0"
                self.chains = chains
                wd = np.ascontiguousarray(p.wait_dense) if chains else None
                wr = np.ascontiguousarray(p.wait_rkt) if chains else None
                rc = lib.hlu_schedule_create_chains(
                    ctypes.byref(handle), ctypes.byref(self.ctx), launches.ctypes.data, len(launches),
                    self.d_getrf.data_ptr(), self.d_trsm.data_ptr(), self.d_gemm.data_ptr(),
                    self.d_terms.data_ptr(), self.d_rkt.data_ptr(), self.d_parts.data_ptr(),
                    ctypes.byref(self.scratch),
                    wd.ctypes.data if chains else None, wr.ctypes.data if chains else None,
                    int(p.nlevels) if chains else 0,
                    1 if use_graph else 0, ctypes.c_void_p(self.stream.cuda_stream),
                )
                _native.check(rc, "hlu_schedule_create")
            self.handle = handle
        self.nkernels = int(p.launches["count"].astype(bool).sum()) if len(p.launches) else 0

    # -- data movement
    def refill(self, extras=None):
        """Re-pack the current host payloads of the layout's H-matrices into the
        pinned staging buffers (same structure; the next ``upload`` sends them)."""
        fill_pool(self.L, self.host_pool.numpy(), self.host_ranks.numpy(), extras)

    def _reset_err(self):
        self.err[0] = 0
        self.err[1] = INT32_MAX
        self.err[2] = 0

    def upload(self):
        """Host (pinned) -> device copy of payloads and ranks; resets error words."""
        n = self.L.payload_doubles
        with self.torch.cuda.device(self.device), self.torch.cuda.stream(self.stream):
            self.pool[:n].copy_(self.host_pool, non_blocking=True)
            self.ranks.copy_(self.host_ranks, non_blocking=True)
            self._reset_err()

    def refill_upload(self, extras=None, nchunks=None):
        """``refill`` + ``upload`` pipelined: the leaves are packed group by
        group into the pinned buffer and every finished pool range starts its
        host-to-device copy while the next group is being packed."""
        nchunks = XFER_CHUNKS if nchunks is None else nchunks
        hp = self.host_pool
        with self.torch.cuda.device(self.device), self.torch.cuda.stream(self.stream):

            def send(lo, hi):
                self.pool[lo:hi].copy_(hp[lo:hi], non_blocking=True)

            fill_pool(self.L, hp.numpy(), self.host_ranks.numpy(), extras, nchunks=nchunks, on_chunk=send)
            self.ranks.copy_(self.host_ranks, non_blocking=True)
            self._reset_err()

    def snapshot(self):
        """Device-resident pristine copy, for repeated timed runs."""
        n = self.L.payload_doubles
        with self.torch.cuda.stream(self.stream):
            self._pristine = (self.pool[:n].clone(), self.ranks.clone())

    def restore(self):
        n = self.L.payload_doubles
        with self.torch.cuda.stream(self.stream):
            self.pool[:n].copy_(self._pristine[0])
            self.ranks.copy_(self._pristine[1])
            self.err[0] = 0
            self.err[1] = INT32_MAX
            self.err[2] = 0

    def launch_times(self):
        """GPU time (s) of every launch-list entry inside a CUDA graph: the same
        schedule re-captured with a %globaltimer stamp after each entry
        (diagnostics; replays on the current device state)."""
        import os

        lib = self.lib
        prev = os.environ.get("HLU_STAMPS")
        os.environ["HLU_STAMPS"] = "1"
        handle = ctypes.c_void_p()
        try:
            p = self.packed
            launches = np.ascontiguousarray(p.launches)
            with self.torch.cuda.device(self.device):
                rc = lib.hlu_schedule_create(
                    ctypes.byref(handle), ctypes.byref(self.ctx), launches.ctypes.data, len(launches),
                    self.d_getrf.data_ptr(), self.d_trsm.data_ptr(), self.d_gemm.data_ptr(),
                    self.d_terms.data_ptr(), self.d_rkt.data_ptr(), self.d_parts.data_ptr(),
                    ctypes.byref(self.scratch), 1, ctypes.c_void_p(self.stream.cuda_stream))
                _native.check(rc, "hlu_schedule_create")
                _native.check(lib.hlu_schedule_launch(handle, ctypes.c_void_p(self.stream.cuda_stream)),
                              "hlu_schedule_launch")
                self.sync()
            n = lib.hlu_schedule_stamps(handle, None)
            st = np.zeros(n, dtype=np.uint64)
            lib.hlu_schedule_stamps(handle, st.ctypes.data)
        finally:
            if handle:
                lib.hlu_schedule_destroy(handle)
            if prev is None:
                os.environ.pop("HLU_STAMPS", None)
            else:
                os.environ["HLU_STAMPS"] = prev
        nl = len(self.packed.launches)
        self.last_phase_stamps = st[nl + 1:].astype(np.int64).reshape(-1, 12)
        return np.diff(st[: nl + 1].astype(np.int64)) * 1e-9

    def launch(self):
        with self.torch.cuda.device(self.device):
            rc = self.lib.hlu_schedule_launch(self.handle, ctypes.c_void_p(self.stream.cuda_stream))
        _native.check(rc, "hlu_schedule_launch")

    def sync(self):
        with self.torch.cuda.device(self.device):
            self.stream.synchronize()

    def check_errors(self):
        self.sync()
        err = self.err.cpu().numpy()
        if err[1] != INT32_MAX:
            op_id = int(err[1])
            idx = int(np.nonzero(self.packed.lu_op_ids == op_id)[0][0])
            p, tol = self.dlog[2 * idx : 2 * idx + 2].cpu().numpy()
            label = self.packed.lu_labels[idx]
            raise SingularBlockError(
                f"pivot {p:.3e} below tolerance {tol:.3e} in block {label or '<root>'}", label
            )
        if err[2]:
            raise RuntimeError(f"{int(err[2])} truncations exceeded the supported shapes (stacked rank > 128, or an eps = 0 dense-fallback block above 64 x 64)")
        if err[0]:
            raise RankOverflow(f"{int(err[0])} Rk results exceeded capacity {self.L.cap}")

    def download(self, nchunks=None):
        """Device -> host (into the pinned staging buffers): install results
        into the H-matrix; returns d2h bytes.  The pool comes back in ranges
        (pool.leaf_chunks), each unpacked into the H-matrix as soon as its
        copy has landed, while the later ranges are still in flight."""
        nchunks = XFER_CHUNKS if nchunks is None else nchunks
        torch = self.torch
        _, offs = leaf_chunks(self.L, nchunks)
        events = []
        with torch.cuda.device(self.device), torch.cuda.stream(self.stream):
            self.host_ranks.copy_(self.ranks, non_blocking=True)
            ev_r = torch.cuda.Event()
            ev_r.record(self.stream)
            for c in range(len(offs) - 1):
                lo, hi = int(offs[c]), int(offs[c + 1])
                self.host_pool[lo:hi].copy_(self.pool[lo:hi], non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(self.stream)
                events.append(ev)
        ev_r.synchronize()
        pool = self.host_pool.numpy()
        ranks = self.host_ranks.numpy()
        read_pool(self.L, pool, ranks, nchunks=nchunks, wait_chunk=lambda c: events[c].synchronize())
        self.sync()
        self._last_pool = pool
        return pool.nbytes + ranks.nbytes

    def extra(self, name):
        return read_extra(self.L, self._last_pool, name)

    def flops(self):
        self.sync()
        return effective_flops(self.packed, self.log.cpu().numpy())

    def close(self):
        if getattr(self, "handle", None):
            with self.torch.cuda.device(self.device):
                self.lib.hlu_schedule_destroy(self.handle)
            self.handle = None

    def release(self):
        """``close`` and drop the device pools (results already downloaded stay
        readable through ``extra``)."""
        self.close()
        for name in ("pool", "_pristine", "staging", "scratch", "_scratch_keep", "d_getrf", "d_trsm", "d_gemm",
                     "d_terms", "d_rkt", "d_parts", "d_xfer"):
            if hasattr(self, name):
                setattr(self, name, None)

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
