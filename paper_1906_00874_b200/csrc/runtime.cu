// Level-set schedule runtime: replays the planner's launch list (one entry per
// (level, kernel kind)) on a stream, optionally captured once into a CUDA
// graph and replayed with a single cudaGraphLaunch.  Replaces the reference's
// executors (_Inline / _Emit + the OmpSs-2 style task runtime,
// hlu.py:315-354, runtime.py:330-817): the ordering the runtime enforced per
// skeleton slot is encoded in the level numbers computed on the host.
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "common.cuh"

extern "C" void hlu_rkt_set_phase_stamps(unsigned long long *p);

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
    case HLU_K_RKT32:
      return hlu_rkt_phases(&s->ctx, s->rkt, s->parts, L.first, L.count, &s->scratch, slot++, st, &s->aux);
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
static int run_launches(hlu_schedule *s, cudaStream_t st) {
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
      dep = dep || (s->launches[j].kind == HLU_K_RKT32 && s->launches[j].smem_dim != 0);
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
  hlu_schedule *s = new hlu_schedule();
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
    if (L.count > s->scratch.max_ops) {
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
      cudaMalloc(&s->stamps, (s->launches.size() + 1 + 12 * nr) * sizeof(unsigned long long));
      cudaMemset(s->stamps, 0, (s->launches.size() + 1 + 12 * nr) * sizeof(unsigned long long));
    }
  }
  cudaStream_t st = (cudaStream_t)stream;
  for (int i = 0; i < 4; ++i) cudaStreamCreateWithFlags((cudaStream_t *)&s->aux.side[i], cudaStreamNonBlocking);
  for (int i = 0; i < 8; ++i) cudaEventCreateWithFlags((cudaEvent_t *)&s->aux.ev[i], cudaEventDisableTiming);
  cudaStreamCreateWithFlags(&s->dense, cudaStreamNonBlocking);
  cudaEventCreateWithFlags(&s->fork, cudaEventDisableTiming);
  cudaEventCreateWithFlags(&s->join, cudaEventDisableTiming);
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
    if (s->stamps) hlu_rkt_set_phase_stamps(s->stamps + s->launches.size() + 1);
    const int rc = run_launches(s, st);
    hlu_rkt_set_phase_stamps(nullptr);
    cudaGraph_t g = nullptr;
    const cudaError_t e = cudaStreamEndCapture(st, &g);
    if (rc != 0 || e != cudaSuccess) {
      if (g) cudaGraphDestroy(g);
      delete s;
      return rc != 0 ? rc : -11;
    }
    s->graph = g;
    if (cudaGraphInstantiate(&s->exec, g, 0) != cudaSuccess) {
      cudaGraphDestroy(g);
      delete s;
      return -12;
    }
  }
  *out = s;
  return 0;
}

extern "C" int hlu_schedule_launch(hlu_schedule *s, void *stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (s->use_graph) return cudaGraphLaunch(s->exec, st) == cudaSuccess ? 0 : -13;
  return run_launches(s, st);
}

extern "C" int hlu_schedule_destroy(hlu_schedule *s) {
  if (!s) return 0;
  if (s->exec) cudaGraphExecDestroy(s->exec);
  if (s->graph) cudaGraphDestroy(s->graph);
  if (s->stamps) cudaFree(s->stamps);
  for (int i = 0; i < 8; ++i) cudaEventDestroy((cudaEvent_t)s->aux.ev[i]);
  for (int i = 0; i < 4; ++i) cudaStreamDestroy((cudaStream_t)s->aux.side[i]);
  cudaEventDestroy(s->fork);
  cudaEventDestroy(s->join);
  cudaStreamDestroy(s->dense);
  delete s;
  return 0;
}

extern "C" int64_t hlu_schedule_stamps(hlu_schedule *s, unsigned long long *out) {
  if (!s->stamps) return 0;
  int64_t nr = 0;
  for (const hlu_launch &L : s->launches) nr += L.kind == HLU_K_RKT32;
  const int64_t n = (int64_t)s->launches.size() + 1 + 12 * nr;
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
