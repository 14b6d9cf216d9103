// Level-set schedule runtime: replays the planner's launch list (one entry per
// (level, kernel kind)) on a stream, optionally captured once into a CUDA
// graph and replayed with a single cudaGraphLaunch.  Replaces the reference's
// executors (_Inline / _Emit + the OmpSs-2 style task runtime,
// hlu.py:315-354, runtime.py:330-817): the ordering the runtime enforced per
// skeleton slot is encoded in the level numbers computed on the host.
#include <cstdio>
#include <cstdlib>
#include <algorithm>
#include <chrono>
#include <cstring>
#include <vector>

#include "common.cuh"
#include "hlu_plan.h"

extern "C" void hlu_rkt_set_phase_stamps(unsigned long long *p);
extern "C" void hlu_rkt_set_wide_hint(int on);
extern "C" int hlu_rkt_phase(const hlu_ctx *ctx, hlu_rkt_desc *d, const hlu_rkpart *parts, int64_t first, int count,
                             const hlu_rkt_scratch *scratch, int slot, int which, void *stream);
struct hlu_comm;

extern "C" int hlu_comm_reduce_logs(hlu_comm *c, int32_t *log, int64_t nlog, int32_t *err, void *stream);

// one (level, source rank) exchange group of a sharded schedule
struct XGroup {
  int32_t level, src;
  int64_t first, n, count;  // records [first, first + n) of the device table, staging doubles
};

struct hlu_schedule {
  hlu_ctx ctx;
  hlu_rkt_streams aux;
  std::vector<hlu_launch> launches;
  const hlu_getrf_desc *getrf;
  const hlu_trsm_desc *trsm;
  const hlu_gemm_desc *gemm;
  const hlu_term *terms;
  hlu_rkt_desc *rkt;
  const hlu_rkpart *parts;
  hlu_rkt_scratch scratch;
  int nrkt;  // truncation launches (counter slots)
  cudaGraph_t graph;
  cudaGraphExec_t exec;
  bool use_graph;
  unsigned long long *stamps;  // diagnostics: %globaltimer after every launch (HLU_STAMPS=1)
  cudaStream_t dense;          // getrf / trsm / gemm launches of a level that also truncates
  cudaEvent_t fork, join;
  // two-chain mode: per-level cross-chain waits and the events they wait on
  std::vector<int32_t> wait_d, wait_r;
  std::vector<cudaEvent_t> ev_d, ev_r;  // after the dense / truncation launches of a level (needed ones only)
  // sharded mode (owner computes over a communicator): exchange groups after levels
  hlu_comm *comm = nullptr;
  const hlu_xfer *d_xfer = nullptr;
  std::vector<XGroup> xgroups;
  double *staging = nullptr;
  int64_t nlevels = 0, nlog = 0;
  // DAG mode (hlu_schedule_create_dag): predecessor launches of every launch and,
  // per truncation launch, its private window of the scratch lists / items
  std::vector<int64_t> dag_ptr;
  std::vector<int32_t> dag_idx;
  std::vector<int64_t> rkt_op0, rkt_item0, rkt_items;  // per launch (truncation launches only)
  int64_t dag_nodes = 0;
  unsigned long long *dag_join = nullptr;  // written by the graph's last node
  std::vector<int32_t> dag_prio;           // per launch: index into dag_q
  cudaStream_t dag_q[3] = {nullptr, nullptr, nullptr};  // capture streams by priority (0: the caller's)
  cudaEvent_t dag_ev[2] = {nullptr, nullptr};
  std::vector<cudaGraphExec_t> dag_exec;   // one graph per chunk of launches, replayed in order
};

__global__ void k_stamp(unsigned long long *slot) {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  *slot = t;
}

static int launch_one(hlu_schedule *s, const hlu_launch &L, int &slot, cudaStream_t st) {
  switch (L.kind) {
    case HLU_K_GETRF: return hlu_getrf_batched_f64(&s->ctx, s->getrf + L.first, L.count, L.smem_dim, st);
    case HLU_K_TRSM: return hlu_trsm_batched_f64(&s->ctx, s->trsm + L.first, L.count, L.smem_dim, st);
    case HLU_K_GEMM: return hlu_gemm_batched_f64(&s->ctx, s->gemm + L.first, s->terms, L.count, st);
    case HLU_K_GEMM_SMALL: return hlu_gemm_small_batched_f64(&s->ctx, s->gemm + L.first, s->terms, L.count, st);
    case HLU_K_RKT32: {
      hlu_rkt_set_wide_hint((L.smem_dim & 2) != 0);
      static const bool serial = getenv("HLU_RKT_SERIAL") && getenv("HLU_RKT_SERIAL")[0] == '1';
      const int rc = hlu_rkt_phases(&s->ctx, s->rkt, s->parts, L.first, L.count, &s->scratch, slot++, st,
                                    serial ? nullptr : &s->aux);
      hlu_rkt_set_wide_hint(1);
      return rc;
    }
    case HLU_K_RKT64: return 0;
    default: return -3;
  }
}

// The launches of one level are independent (levels are ASAP by skeleton-slot
// hazards, temps are never reused inside a level) unless a truncation reads a
// temp a dense launch of the same level produces (a deferred producer chain;
// the planner flags that truncation launch with smem_dim = 1).  Otherwise a
// level that truncates runs its dense launches (getrf / trsm / gemm, in
// order) on a side stream beside the truncation kernels and joins them at the
// level's end.  With
// stamps (diagnostics) every launch runs in order on `st`, so consecutive
// stamps time one launch each.
// Two chains: the truncation launches run in level order on `st`, the dense
// launches in level order on s->dense; a level's launches of one chain wait
// for the other chain's last conflicting level (planner waits), and the
// dense launches of a level go first so a truncation can wait on its own level.
static int run_chains(hlu_schedule *s, cudaStream_t st) {
  const size_t nl = s->launches.size();
  if (s->nrkt) cudaMemsetAsync(s->scratch.counts, 0, 8 * sizeof(int32_t) * s->nrkt, st);
  cudaEventRecord(s->fork, st);
  cudaStreamWaitEvent(s->dense, s->fork, 0);
  int slot = 0;
  int32_t seen_r = -1, seen_d = -1;  // highest level of the other chain already waited for
  std::vector<char> rec_d(s->wait_d.size(), 0), rec_r(s->wait_d.size(), 0);
  size_t i = 0;
  while (i < nl) {
    const int32_t lv = s->launches[i].level;
    size_t j = i;
    while (j < nl && s->launches[j].level == lv) ++j;
    bool any_d = false, any_r = false;
    for (size_t k = i; k < j; ++k) (s->launches[k].kind == HLU_K_RKT32 ? any_r : any_d) = true;
    if (any_d) {
      const int32_t w = s->wait_d[lv];
      if (w > seen_r) {
        if (!s->ev_r[w] || !rec_r[w]) return -16;  // never recorded: plan / launch mismatch  // never recorded: plan / launch mismatch
        cudaStreamWaitEvent(s->dense, s->ev_r[w], 0);
        seen_r = w;
      }
      for (size_t k = i; k < j; ++k) {
        if (s->launches[k].kind == HLU_K_RKT32) continue;
        const int rc = launch_one(s, s->launches[k], slot, s->dense);
        if (rc != 0) return rc;
      }
      if (s->ev_d[lv]) {
        cudaEventRecord(s->ev_d[lv], s->dense);
        rec_d[lv] = 1;
      }
    }
    if (any_r) {
      const int32_t w = s->wait_r[lv];
      if (w > seen_d) {
        if (!s->ev_d[w] || !rec_d[w]) return -16;
        cudaStreamWaitEvent(st, s->ev_d[w], 0);
        seen_d = w;
      }
      for (size_t k = i; k < j; ++k) {
        if (s->launches[k].kind != HLU_K_RKT32) continue;
        const int rc = launch_one(s, s->launches[k], slot, st);
        if (rc != 0) return rc;
      }
      if (s->ev_r[lv]) {
        cudaEventRecord(s->ev_r[lv], st);
        rec_r[lv] = 1;
      }
    }
    i = j;
  }
  cudaEventRecord(s->join, s->dense);
  cudaStreamWaitEvent(st, s->join, 0);
  return 0;
}

static int run_launches(hlu_schedule *s, cudaStream_t st);

// Sharded: this rank's launches level by level (a level that also truncates
// runs its dense launches on the side stream, as run_launches), then the
// level's exchange groups; after the last level the final gather and the
// reduction of the flop logs / error words.
static int run_sharded(hlu_schedule *s, cudaStream_t st) {
  const size_t nl = s->launches.size();
  if (s->nrkt) cudaMemsetAsync(s->scratch.counts, 0, 8 * sizeof(int32_t) * s->nrkt, st);
  int slot = 0;
  size_t i = 0, g = 0;
  for (int64_t lv = 0; lv <= s->nlevels; ++lv) {
    size_t j = i;
    bool rk = false, dn = false, dep = false;
    while (j < nl && s->launches[j].level == lv) {
      (s->launches[j].kind == HLU_K_RKT32 ? rk : dn) = true;
      dep = dep || (s->launches[j].kind == HLU_K_RKT32 && (s->launches[j].smem_dim & 1));
      ++j;
    }
    const bool split = rk && dn && !dep;
    if (split) {
      cudaEventRecord(s->fork, st);
      cudaStreamWaitEvent(s->dense, s->fork, 0);
    }
    for (size_t k = i; k < j; ++k) {
      const hlu_launch &L = s->launches[k];
      const int rc = launch_one(s, L, slot, (split && L.kind != HLU_K_RKT32) ? s->dense : st);
      if (rc != 0) return rc;
    }
    if (split) {
      cudaEventRecord(s->join, s->dense);
      cudaStreamWaitEvent(st, s->join, 0);
    }
    i = j;
    for (; g < s->xgroups.size() && s->xgroups[g].level == lv; ++g) {
      const XGroup &x = s->xgroups[g];
      const int rc = hlu_xfer_group(s->comm, s->ctx.pool, s->ctx.ranks, (const void *)(s->d_xfer + x.first),
                                    (int)x.n, x.src, x.count, s->staging, st);
      if (rc != 0) return rc;
    }
  }
  if (i != nl || g != s->xgroups.size()) return -17;  // launches / exchanges beyond nlevels
  return hlu_comm_reduce_logs(s->comm, s->ctx.log, s->nlog, s->ctx.err, st);
}

// ---------------------------------------------------------------- DAG mode
// The launch list replayed as a task DAG: every launch is captured with
// exactly the planner's predecessor launches as graph dependencies
// (cudaStreamUpdateCaptureDependencies replaces the capturing stream's
// dependency set before each launch), so independent launches of different
// time slots overlap and a slow truncation no longer holds a whole level.
// A truncation launch is itself a small DAG of kernels (classify -> register
// warp kernels | block TSQR -> cores -> Q apply) with its own window of the
// scratch lists, because several truncation launches are in flight at once.
static int capture_tail(cudaStream_t st, std::vector<cudaGraphNode_t> &out) {
  cudaStreamCaptureStatus status;
  const cudaGraphNode_t *deps = nullptr;
  size_t n = 0;
  if (cudaStreamGetCaptureInfo(st, &status, nullptr, nullptr, &deps, &n) != cudaSuccess) return -20;
  if (status != cudaStreamCaptureStatusActive) return -20;
  out.assign(deps, deps + n);
  return 0;
}

static int set_deps(cudaStream_t st, std::vector<cudaGraphNode_t> &deps) {
  return cudaStreamUpdateCaptureDependencies(st, deps.data(), deps.size(), cudaStreamSetCaptureDependencies) ==
                 cudaSuccess
             ? 0
             : -21;
}

// Launches [l0, l1) as one captured graph.  The DAG is cut into chunks of
// consecutive launches (launch order is topological), one CUDA graph each,
// replayed back to back on the stream: instantiating one graph of several
// hundred thousand nodes takes minutes (measured: 535k nodes, 117 s), a
// chunk of ~10k nodes a fraction of a second.  Dependencies on launches of
// earlier chunks are implied by the stream order; the only cost is one
// drain of the in-flight launches per chunk boundary.
static int run_dag_chunk(hlu_schedule *s, cudaStream_t st, size_t l0, size_t l1, int &slot) {
  const size_t nl = l1 - l0;
  std::vector<cudaGraphNode_t> root, deps, tail, a_tail, b_tail, tmp;
  if (l0 == 0) cudaMemsetAsync(s->scratch.counts, 0, 8 * sizeof(int32_t) * std::max(s->nrkt, 1), st);
  else k_stamp<<<1, 1, 0, st>>>(s->dag_join);
  int rc = capture_tail(st, root);
  if (rc) return rc;
  // launches without slack are captured from higher-priority streams (their
  // kernel nodes keep the stream's priority): when SMs are contended the block
  // scheduler serves the critical chain first
  cudaStream_t qs[3] = {st, s->dag_q[1] ? s->dag_q[1] : st, s->dag_q[2] ? s->dag_q[2] : st};
  cudaEventRecord(s->fork, st);
  for (int k = 1; k < 3; ++k)
    if (qs[k] != st) cudaStreamWaitEvent(qs[k], s->fork, 0);
  const cudaStream_t origin = st;
  std::vector<int64_t> tptr(nl + 1, 0);
  std::vector<cudaGraphNode_t> tails;
  tails.reserve(nl * 2);
  std::vector<char> has_succ(nl, 0);
  static const bool all_routes = getenv("HLU_RKT_ALL_ROUTES") && getenv("HLU_RKT_ALL_ROUTES")[0] == '1';
  static const bool join_tails = getenv("HLU_DAG_JOIN") && getenv("HLU_DAG_JOIN")[0] == '1';
  for (size_t l = l0; l < l1; ++l) {
    const hlu_launch &L = s->launches[l];
    deps.clear();
    for (int64_t e = s->dag_ptr[l]; e < s->dag_ptr[l + 1]; ++e) {
      const int32_t p = s->dag_idx[e];
      if (p < 0 || (size_t)p >= l) return -22;
      if ((size_t)p < l0) continue;  // an earlier chunk: done before this graph starts
      has_succ[p - l0] = 1;
      deps.insert(deps.end(), tails.begin() + tptr[p - l0], tails.begin() + tptr[p - l0 + 1]);
    }
    if (deps.empty()) deps = root;
    st = qs[s->dag_prio.empty() ? 0 : s->dag_prio[l]];
    if (L.count <= 0) {  // nothing to run: successors wait for the predecessors directly
      tails.insert(tails.end(), deps.begin(), deps.end());
      tptr[l - l0 + 1] = (int64_t)tails.size();
      continue;
    }
    if (s->stamps) {  // diagnostics: when the launch became ready (its dependencies done)
      if ((rc = set_deps(st, deps))) return rc;
      k_stamp<<<1, 1, 0, st>>>(s->stamps + 2 * l);
      if ((rc = capture_tail(st, deps))) return rc;
    }
    if (L.kind != HLU_K_RKT32) {
      if ((rc = set_deps(st, deps))) return rc;
      int dummy = 0;
      if ((rc = launch_one(s, L, dummy, st))) return rc;
      if ((rc = capture_tail(st, tail))) return rc;
      s->dag_nodes += 1;
    } else {
      hlu_rkt_scratch sc = s->scratch;
      sc.list = s->scratch.list + 7 * s->rkt_op0[l];
      sc.max_ops = L.count;
      sc.items = s->scratch.items + s->rkt_item0[l];
      sc.max_items = std::max<int64_t>(s->rkt_items[l], 1);
      const int my = slot++;
      auto K = [&](int which, std::vector<cudaGraphNode_t> &d, std::vector<cudaGraphNode_t> &out) -> int {
        int r = set_deps(st, d);
        if (r) return r;
        r = hlu_rkt_phase(&s->ctx, s->rkt, s->parts, L.first, L.count, &sc, my, which, st);
        if (r) return r;
        tmp.clear();
        r = capture_tail(st, tmp);
        out.insert(out.end(), tmp.begin(), tmp.end());
        s->dag_nodes += 1;
        return r;
      };
      // plan-time route hints (smem_dim bits): 2 may stack > 64 columns, 4 no
      // op fits the register warp kernels (every max(m, n) > 64)
      const bool wide = (L.smem_dim & 2) != 0 || s->ctx.eps == 0.0 || all_routes;
      const bool no_warp = (L.smem_dim & 4) != 0 && !all_routes;
      std::vector<cudaGraphNode_t> c;
      tail.clear();
      a_tail.clear();
      b_tail.clear();
      {
        if ((rc = K(0, deps, c))) return rc;
        if (!no_warp) {
          if ((rc = K(1, c, tail))) return rc;
          if ((rc = K(2, c, tail))) return rc;
        }
        if (wide && (rc = K(3, c, tail))) return rc;
        if ((rc = K(4, c, a_tail))) return rc;
        if ((rc = K(9, c, a_tail))) return rc;
        if ((rc = K(5, a_tail, b_tail))) return rc;
        if ((rc = K(6, a_tail, b_tail))) return rc;
        if ((rc = K(7, a_tail, b_tail))) return rc;
        if ((rc = K(8, b_tail, tail))) return rc;
        if ((rc = K(10, b_tail, tail))) return rc;
      }
    }
    if (join_tails && tail.size() > 1) {
      // one empty node behind the launch's tail kernels: successors take one edge
      // instead of one per tail (no GPU work; fewer edges to instantiate)
      cudaStreamCaptureStatus status;
      cudaGraph_t graph = nullptr;
      if (cudaStreamGetCaptureInfo(st, &status, nullptr, &graph, nullptr, nullptr) != cudaSuccess || !graph) return -23;
      cudaGraphNode_t join = nullptr;
      if (cudaGraphAddEmptyNode(&join, graph, tail.data(), tail.size()) != cudaSuccess) return -23;
      tail.assign(1, join);
    }
    if (s->stamps) {  // ... and when its last kernel ended
      if ((rc = set_deps(st, tail))) return rc;
      k_stamp<<<1, 1, 0, st>>>(s->stamps + 2 * l + 1);
      if ((rc = capture_tail(st, tail))) return rc;
    }
    tails.insert(tails.end(), tail.begin(), tail.end());
    tptr[l - l0 + 1] = (int64_t)tails.size();
  }
  // join: the capturing stream ends behind every launch nothing else waits for
  deps.clear();
  for (size_t l = 0; l < nl; ++l)
    if (!has_succ[l]) deps.insert(deps.end(), tails.begin() + tptr[l], tails.begin() + tptr[l + 1]);
  if (deps.empty()) deps = root;
  {  // a graph node takes a bounded number of dependencies comfortably: join the sinks through a tree
    const size_t fan = 64;
    while (deps.size() > fan) {
      std::vector<cudaGraphNode_t> next;
      for (size_t b = 0; b < deps.size(); b += fan) {
        std::vector<cudaGraphNode_t> part(deps.begin() + b, deps.begin() + std::min(deps.size(), b + fan));
        if ((rc = set_deps(origin, part))) return rc;
        k_stamp<<<1, 1, 0, origin>>>(s->dag_join);
        tmp.clear();
        if ((rc = capture_tail(origin, tmp))) return rc;
        next.insert(next.end(), tmp.begin(), tmp.end());
      }
      deps.swap(next);
    }
  }
  st = origin;
  for (int k = 1; k < 3; ++k) {  // the priority streams rejoin the origin behind the sinks
    if (qs[k] == st) continue;
    if ((rc = set_deps(qs[k], deps))) return rc;
    cudaEventRecord(s->dag_ev[k - 1], qs[k]);
    cudaStreamWaitEvent(st, s->dag_ev[k - 1], 0);
  }
  if ((rc = set_deps(st, deps))) return rc;
  k_stamp<<<1, 1, 0, st>>>(s->dag_join);
  return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

static int run_launches(hlu_schedule *s, cudaStream_t st) {
  if (s->comm) return run_sharded(s, st);
  if (!s->wait_d.empty() && !s->stamps) return run_chains(s, st);
  const size_t nl = s->launches.size();
  if (s->stamps) k_stamp<<<1, 1, 0, st>>>(s->stamps);
  if (s->nrkt) cudaMemsetAsync(s->scratch.counts, 0, 8 * sizeof(int32_t) * s->nrkt, st);
  int slot = 0;
  size_t i = 0;
  while (i < nl) {
    size_t j = i;
    bool rk = false, dn = false;
    bool dep = false;
    while (j < nl && s->launches[j].level == s->launches[i].level) {
      (s->launches[j].kind == HLU_K_RKT32 ? rk : dn) = true;
      dep = dep || (s->launches[j].kind == HLU_K_RKT32 && (s->launches[j].smem_dim & 1));
      ++j;
    }
    const bool split = rk && dn && !dep && !s->stamps;
    if (split) {
      cudaEventRecord(s->fork, st);
      cudaStreamWaitEvent(s->dense, s->fork, 0);
    }
    for (size_t k = i; k < j; ++k) {
      const hlu_launch &L = s->launches[k];
      const bool side = split && L.kind != HLU_K_RKT32;
      const int rc = launch_one(s, L, slot, side ? s->dense : st);
      if (rc != 0) return rc;
      if (s->stamps) k_stamp<<<1, 1, 0, st>>>(s->stamps + k + 1);
    }
    if (split) {
      cudaEventRecord(s->join, s->dense);
      cudaStreamWaitEvent(st, s->join, 0);
    }
    i = j;
  }
  return 0;
}

extern "C" int hlu_schedule_create(hlu_schedule **out, const hlu_ctx *ctx, const hlu_launch *launches,
                                   int64_t nlaunch, const hlu_getrf_desc *getrf, const hlu_trsm_desc *trsm,
                                   const hlu_gemm_desc *gemm, const hlu_term *terms, hlu_rkt_desc *rkt,
                                   const hlu_rkpart *parts, const hlu_rkt_scratch *scratch, int use_graph,
                                   void *stream) {
  return hlu_schedule_create_chains(out, ctx, launches, nlaunch, getrf, trsm, gemm, terms, rkt, parts, scratch,
                                    nullptr, nullptr, 0, use_graph, stream);
}

static void destroy_events(hlu_schedule *s) {
  for (cudaEvent_t e : s->ev_d)
    if (e) cudaEventDestroy(e);
  for (cudaEvent_t e : s->ev_r)
    if (e) cudaEventDestroy(e);
  s->ev_d.clear();
  s->ev_r.clear();
}

struct DagArgs {
  const int64_t *dep_ptr;
  const int32_t *dep_idx;
  const int64_t *item0, *nitems;  // per launch: first row-block item and item count (truncation launches)
  const int32_t *prio;            // per launch: 0 .. 2 scheduling priority (may be NULL)
};

struct ShardArgs {
  hlu_comm *comm;
  const hlu_xfer *xfer_host, *xfer_dev;
  int64_t nxfer, nlevels, nlog;
  double *staging;
};

static int create(hlu_schedule **out, const hlu_ctx *ctx, const hlu_launch *launches, int64_t nlaunch,
                  const hlu_getrf_desc *getrf, const hlu_trsm_desc *trsm, const hlu_gemm_desc *gemm,
                  const hlu_term *terms, hlu_rkt_desc *rkt, const hlu_rkpart *parts, const hlu_rkt_scratch *scratch,
                  const int32_t *wait_dense, const int32_t *wait_rkt, int64_t nlevels, int use_graph, void *stream,
                  const ShardArgs *sh, const DagArgs *dag = nullptr);

extern "C" int hlu_schedule_create_chains(hlu_schedule **out, const hlu_ctx *ctx, const hlu_launch *launches,
                                          int64_t nlaunch, const hlu_getrf_desc *getrf, const hlu_trsm_desc *trsm,
                                          const hlu_gemm_desc *gemm, const hlu_term *terms, hlu_rkt_desc *rkt,
                                          const hlu_rkpart *parts, const hlu_rkt_scratch *scratch,
                                          const int32_t *wait_dense, const int32_t *wait_rkt, int64_t nlevels,
                                          int use_graph, void *stream) {
  return create(out, ctx, launches, nlaunch, getrf, trsm, gemm, terms, rkt, parts, scratch, wait_dense, wait_rkt,
                nlevels, use_graph, stream, nullptr);
}

extern "C" int hlu_schedule_create_sharded(hlu_schedule **out, const hlu_ctx *ctx, const hlu_launch *launches,
                                           int64_t nlaunch, const hlu_getrf_desc *getrf, const hlu_trsm_desc *trsm,
                                           const hlu_gemm_desc *gemm, const hlu_term *terms, hlu_rkt_desc *rkt,
                                           const hlu_rkpart *parts, const hlu_rkt_scratch *scratch, hlu_comm *comm,
                                           const void *xfer_host, const void *xfer_dev, int64_t nxfer,
                                           int64_t nlevels, int64_t nlog, double *staging, int use_graph,
                                           void *stream) {
  if (!comm) return -18;
  const ShardArgs sh{comm, (const hlu_xfer *)xfer_host, (const hlu_xfer *)xfer_dev, nxfer, nlevels, nlog, staging};
  return create(out, ctx, launches, nlaunch, getrf, trsm, gemm, terms, rkt, parts, scratch, nullptr, nullptr, 0,
                use_graph, stream, &sh);
}

// DAG schedule (include/hlu_plan.h hlu_plan_build_dag): launch l waits for the
// launches dep_idx[dep_ptr[l] .. dep_ptr[l+1]) (all < l); scratch->list holds 7
// ints per truncation descriptor and scratch->items every row-block item
// (item0 / nitems: each truncation launch's window, from hlu_rkt_items).
extern "C" int hlu_schedule_create_dag(hlu_schedule **out, const hlu_ctx *ctx, const hlu_launch *launches,
                                       int64_t nlaunch, const hlu_getrf_desc *getrf, const hlu_trsm_desc *trsm,
                                       const hlu_gemm_desc *gemm, const hlu_term *terms, hlu_rkt_desc *rkt,
                                       const hlu_rkpart *parts, const hlu_rkt_scratch *scratch,
                                       const int64_t *dep_ptr, const int32_t *dep_idx, const int64_t *item0,
                                       const int64_t *nitems, const int32_t *prio, void *stream) {
  if (!dep_ptr || !item0 || !nitems) return -23;
  const DagArgs dag{dep_ptr, dep_idx, item0, nitems, prio};
  return create(out, ctx, launches, nlaunch, getrf, trsm, gemm, terms, rkt, parts, scratch, nullptr, nullptr, 0, 1,
                stream, nullptr, &dag);
}

extern "C" int64_t hlu_schedule_graph_nodes(const hlu_schedule *s) { return s->dag_nodes; }

// staging doubles the exchange groups of a sharded plan need (the largest group)
extern "C" int64_t hlu_xfer_staging_doubles(const void *xfer, int64_t n) {
  const hlu_xfer *x = (const hlu_xfer *)xfer;
  int64_t best = 0;
  for (int64_t i = 0; i < n; ++i) best = std::max<int64_t>(best, x[i].boff + x[i].len + 1);
  return best;
}

static int create(hlu_schedule **out, const hlu_ctx *ctx, const hlu_launch *launches, int64_t nlaunch,
                  const hlu_getrf_desc *getrf, const hlu_trsm_desc *trsm, const hlu_gemm_desc *gemm,
                  const hlu_term *terms, hlu_rkt_desc *rkt, const hlu_rkpart *parts, const hlu_rkt_scratch *scratch,
                  const int32_t *wait_dense, const int32_t *wait_rkt, int64_t nlevels, int use_graph, void *stream,
                  const ShardArgs *sh, const DagArgs *dag) {
  hlu_schedule *s = new hlu_schedule();
  if (dag) {
    if (!use_graph) {
      delete s;
      return -23;  // the DAG schedule exists only as a CUDA graph
    }
    s->dag_ptr.assign(dag->dep_ptr, dag->dep_ptr + nlaunch + 1);
    s->dag_idx.assign(dag->dep_idx, dag->dep_idx + dag->dep_ptr[nlaunch]);
    s->rkt_op0.assign(nlaunch, 0);
    s->rkt_item0.assign(dag->item0, dag->item0 + nlaunch);
    s->rkt_items.assign(dag->nitems, dag->nitems + nlaunch);
    for (int64_t i = 0; i < nlaunch; ++i) s->rkt_op0[i] = launches[i].first;
    if (s->dag_ptr.empty()) s->dag_ptr.push_back(0);
    cudaMalloc(&s->dag_join, sizeof(unsigned long long));
    if (dag->prio) {
      s->dag_prio.assign(dag->prio, dag->prio + nlaunch);
      for (int32_t &v : s->dag_prio) v = std::min(2, std::max(0, v));
      int least = 0, greatest = 0;
      cudaDeviceGetStreamPriorityRange(&least, &greatest);
      cudaStreamCreateWithPriority(&s->dag_q[1], cudaStreamNonBlocking, (least + greatest) / 2);
      cudaStreamCreateWithPriority(&s->dag_q[2], cudaStreamNonBlocking, greatest);
      for (int k = 0; k < 2; ++k) cudaEventCreateWithFlags(&s->dag_ev[k], cudaEventDisableTiming);
    }
  }
  if (sh) {
    s->comm = sh->comm;
    s->d_xfer = sh->xfer_dev;
    s->staging = sh->staging;
    s->nlevels = sh->nlevels;
    s->nlog = sh->nlog;
    for (int64_t i = 0; i < sh->nxfer; ++i) {
      const hlu_xfer &r = sh->xfer_host[i];
      if (s->xgroups.empty() || s->xgroups.back().level != r.level || s->xgroups.back().src != r.src ||
          r.boff == 0) {
        if (!s->xgroups.empty() && (r.level < s->xgroups.back().level)) {
          delete s;
          return -19;  // records out of level order
        }
        s->xgroups.push_back(XGroup{r.level, r.src, i, 0, 0});
      }
      XGroup &g = s->xgroups.back();
      ++g.n;
      g.count = std::max<int64_t>(g.count, r.boff + r.len + 1);
    }
    for (int64_t i = 0; i < nlaunch; ++i)
      if (i > 0 && launches[i].level < launches[i - 1].level) {
        delete s;
        return -19;
      }
  }
  if (wait_dense && wait_rkt && nlevels > 0) {
    for (int64_t i = 0; i < nlaunch; ++i)
      if (launches[i].level < 0 || launches[i].level >= nlevels) {
        delete s;
        return -15;
      }
    s->wait_d.assign(wait_dense, wait_dense + nlevels);
    s->wait_r.assign(wait_rkt, wait_rkt + nlevels);
    s->ev_d.assign(nlevels, nullptr);
    s->ev_r.assign(nlevels, nullptr);
    for (int64_t l = 0; l < nlevels; ++l) {
      const int32_t wd = s->wait_d[l], wr = s->wait_r[l];
      if (wd > l || wr > l || (wd == l)) {  // only a truncation may wait on its own level
        destroy_events(s);
        delete s;
        return -15;
      }
      if (wd >= 0 && !s->ev_r[wd]) cudaEventCreateWithFlags(&s->ev_r[wd], cudaEventDisableTiming);
      if (wr >= 0 && !s->ev_d[wr]) cudaEventCreateWithFlags(&s->ev_d[wr], cudaEventDisableTiming);
    }
  }
  s->ctx = *ctx;
  s->launches.assign(launches, launches + nlaunch);
  s->getrf = getrf;
  s->trsm = trsm;
  s->gemm = gemm;
  s->terms = terms;
  s->rkt = rkt;
  s->parts = parts;
  s->scratch = *scratch;
  s->nrkt = 0;
  for (const hlu_launch &L : s->launches) {
    if (L.kind != HLU_K_RKT32) continue;
    ++s->nrkt;
    if (!dag && L.count > s->scratch.max_ops) {
      delete s;
      return -14;
    }
    if (dag && L.first + L.count > s->scratch.max_ops) {  // DAG mode: the lists cover every descriptor
      delete s;
      return -14;
    }
  }
  s->graph = nullptr;
  s->exec = nullptr;
  s->use_graph = use_graph != 0;
  s->stamps = nullptr;
  {
    const char *e = getenv("HLU_STAMPS");
    if (e && e[0] == '1') {
      int64_t nr = 0;
      for (const hlu_launch &L : s->launches) nr += L.kind == HLU_K_RKT32;
      const size_t ns = dag ? 2 * s->launches.size() + 2 : s->launches.size() + 1 + 12 * nr;
      cudaMalloc(&s->stamps, ns * sizeof(unsigned long long));
      cudaMemset(s->stamps, 0, ns * sizeof(unsigned long long));
    }
  }
  cudaStream_t st = (cudaStream_t)stream;
  for (int i = 0; i < 4; ++i) cudaStreamCreateWithFlags((cudaStream_t *)&s->aux.side[i], cudaStreamNonBlocking);
  for (int i = 0; i < 8; ++i) cudaEventCreateWithFlags((cudaEvent_t *)&s->aux.ev[i], cudaEventDisableTiming);
  cudaStreamCreateWithFlags(&s->dense, cudaStreamNonBlocking);
  cudaEventCreateWithFlags(&s->fork, cudaEventDisableTiming);
  cudaEventCreateWithFlags(&s->join, cudaEventDisableTiming);
  if (dag) {
    hlu_getrf_batched_f64(&s->ctx, s->getrf, 0, 0, st);
    hlu_trsm_batched_f64(&s->ctx, s->trsm, 0, 0, st);
    hlu_rk_update_batched_f64(&s->ctx, s->rkt, s->parts, 0, &s->scratch, st);
    hlu_gemm_small_batched_f64(&s->ctx, s->gemm, s->terms, 0, st);
    hlu_gemm_batched_f64(&s->ctx, s->gemm, s->terms, 0, st);
    const bool timing = getenv("HLU_PLAN_TIMING") != nullptr;
    auto now = [] { return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count(); };
    const double t0 = now();
    double t_cap = 0.0, t_inst = 0.0, t_up = 0.0;
    const int64_t budget = getenv("HLU_DAG_CHUNK_NODES") ? atoll(getenv("HLU_DAG_CHUNK_NODES")) : 12000;
    // chunk boundaries by estimated kernel nodes (a truncation launch is ~10)
    size_t l0 = 0;
    int slot = 0;
    const size_t nl = s->launches.size();
    while (l0 < nl || s->dag_exec.empty()) {
      size_t l1 = l0;
      int64_t est = 0;
      while (l1 < nl && (est < budget || l1 == l0)) est += s->launches[l1].kind == HLU_K_RKT32 ? 10 : 1, ++l1;
      if (cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal) != cudaSuccess) {
        hlu_schedule_destroy(s);
        return -10;
      }
      double tc = now();
      const int rc = run_dag_chunk(s, st, l0, l1, slot);
      cudaGraph_t g = nullptr;
      const cudaError_t e = cudaStreamEndCapture(st, &g);
      t_cap += now() - tc;
      tc = now();
      cudaGraphExec_t ex = nullptr;
      const cudaError_t ei =
          (rc != 0 || e != cudaSuccess)
              ? cudaErrorUnknown
              : cudaGraphInstantiate(&ex, g, s->dag_prio.empty() ? 0 : cudaGraphInstantiateFlagUseNodePriority);
      t_inst += now() - tc;
      if (ei != cudaSuccess) {
        if (timing) std::fprintf(stderr, "schedule: dag chunk [%zu, %zu) failed: rc %d, %s\n", l0, l1, rc,
                                 cudaGetErrorString(e != cudaSuccess ? e : cudaGetLastError()));
        if (g) cudaGraphDestroy(g);
        hlu_schedule_destroy(s);
        return rc != 0 ? rc : (e != cudaSuccess ? -11 : -12);
      }
      tc = now();
      cudaGraphDestroy(g);
      cudaGraphUpload(ex, st);
      t_up += now() - tc;
      s->dag_exec.push_back(ex);
      l0 = l1;
      if (nl == 0) break;
    }
    cudaStreamSynchronize(st);
    if (timing)
      std::fprintf(stderr,
                   "schedule: dag %zu launches, %lld kernel nodes in %zu graphs, %.2fs (capture %.2fs, instantiate "
                   "%.2fs, destroy + upload %.2fs)\n",
                   nl, (long long)s->dag_nodes, s->dag_exec.size(), now() - t0, t_cap, t_inst, t_up);
    *out = s;
    return 0;
  }
  if (s->use_graph) {
    // make sure kernel attributes are set outside capture
    hlu_getrf_batched_f64(&s->ctx, s->getrf, 0, 0, st);
    hlu_trsm_batched_f64(&s->ctx, s->trsm, 0, 0, st);
    hlu_rk_update_batched_f64(&s->ctx, s->rkt, s->parts, 0, &s->scratch, st);
    hlu_gemm_small_batched_f64(&s->ctx, s->gemm, s->terms, 0, st);
    hlu_gemm_batched_f64(&s->ctx, s->gemm, s->terms, 0, st);
    if (cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal) != cudaSuccess) {
      delete s;
      return -10;
    }
    if (s->stamps && !dag) hlu_rkt_set_phase_stamps(s->stamps + s->launches.size() + 1);
    const bool timing = getenv("HLU_PLAN_TIMING") != nullptr;
    auto now = [] { return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count(); };
    double t0 = now();
    const int rc = run_launches(s, st);
    hlu_rkt_set_phase_stamps(nullptr);
    cudaGraph_t g = nullptr;
    const cudaError_t e = cudaStreamEndCapture(st, &g);
    if (timing) std::fprintf(stderr, "schedule: capture %.2fs (%lld dag nodes)\n", now() - t0, (long long)s->dag_nodes), t0 = now();
    if (rc != 0 || e != cudaSuccess) {
      if (g) cudaGraphDestroy(g);
      delete s;
      return rc != 0 ? rc : -11;
    }
    s->graph = g;
    if (cudaGraphInstantiate(&s->exec, g, s->dag_prio.empty() ? 0 : cudaGraphInstantiateFlagUseNodePriority) !=
        cudaSuccess) {
      cudaGraphDestroy(g);
      delete s;
      return -12;
    }
    if (timing) std::fprintf(stderr, "schedule: instantiate %.2fs\n", now() - t0), t0 = now();
    cudaGraphUpload(s->exec, st);
    cudaStreamSynchronize(st);
    if (timing) std::fprintf(stderr, "schedule: upload %.2fs\n", now() - t0);
  }
  *out = s;
  return 0;
}

extern "C" int hlu_schedule_launch(hlu_schedule *s, void *stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (!s->dag_exec.empty()) {
    for (cudaGraphExec_t ex : s->dag_exec)
      if (cudaGraphLaunch(ex, st) != cudaSuccess) return -13;
    return 0;
  }
  if (s->use_graph) return cudaGraphLaunch(s->exec, st) == cudaSuccess ? 0 : -13;
  return run_launches(s, st);
}

extern "C" int hlu_schedule_destroy(hlu_schedule *s) {
  if (!s) return 0;
  if (s->exec) cudaGraphExecDestroy(s->exec);
  for (cudaGraphExec_t ex : s->dag_exec) cudaGraphExecDestroy(ex);
  if (s->graph) cudaGraphDestroy(s->graph);
  if (s->stamps) cudaFree(s->stamps);
  if (s->dag_join) cudaFree(s->dag_join);
  for (int k = 1; k < 3; ++k)
    if (s->dag_q[k]) cudaStreamDestroy(s->dag_q[k]);
  for (int k = 0; k < 2; ++k)
    if (s->dag_ev[k]) cudaEventDestroy(s->dag_ev[k]);
  for (int i = 0; i < 8; ++i) cudaEventDestroy((cudaEvent_t)s->aux.ev[i]);
  for (int i = 0; i < 4; ++i) cudaStreamDestroy((cudaStream_t)s->aux.side[i]);
  cudaEventDestroy(s->fork);
  cudaEventDestroy(s->join);
  cudaStreamDestroy(s->dense);
  destroy_events(s);
  delete s;
  return 0;
}

extern "C" int64_t hlu_schedule_stamps(hlu_schedule *s, unsigned long long *out) {
  if (!s->stamps) return 0;
  int64_t nr = 0;
  for (const hlu_launch &L : s->launches) nr += L.kind == HLU_K_RKT32;
  // DAG mode: (ready, end) of every launch
  const int64_t n = !s->dag_ptr.empty() ? 2 * (int64_t)s->launches.size() : (int64_t)s->launches.size() + 1 + 12 * nr;
  if (out && cudaMemcpy(out, s->stamps, n * sizeof(unsigned long long), cudaMemcpyDeviceToHost) != cudaSuccess)
    return -1;
  return n;
}

extern "C" const char *hlu_version(void) { return "hlu_b200 0.1.0 sm_100a"; }

extern "C" int hlu_device_check(void) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return -1;
  cudaDeviceProp p;
  if (cudaGetDeviceProperties(&p, dev) != cudaSuccess) return -1;
  return (p.major == 10) ? 0 : -2;
}
