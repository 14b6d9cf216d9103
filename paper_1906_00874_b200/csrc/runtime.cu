// Level-set schedule runtime: replays the planner's launch list (one entry per
// (level, kernel kind)) on a stream, optionally captured once into a CUDA
// graph and replayed with a single cudaGraphLaunch.  Replaces the reference's
// executors (_Inline / _Emit + the OmpSs-2 style task runtime,
// hlu.py:315-354, runtime.py:330-817): the ordering the runtime enforced per
// skeleton slot is encoded in the level numbers computed on the host.
#include <cstdio>
#include <cstring>
#include <vector>

#include "common.cuh"

extern "C" int hlu_epoch_bump(void *stream);

struct hlu_schedule {
  hlu_ctx ctx;
  cudaStream_t side;
  cudaEvent_t ev_fork, ev_join;
  std::vector<hlu_launch> launches;
  const hlu_getrf_desc *getrf;
  const hlu_trsm_desc *trsm;
  const hlu_gemm_desc *gemm;
  const hlu_term *terms;
  hlu_rkt_desc *rkt;
  const hlu_rkpart *parts;
  cudaGraph_t graph;
  cudaGraphExec_t exec;
  bool use_graph;
};

static int run_launches(hlu_schedule *s, cudaStream_t st) {
  int rc0 = hlu_epoch_bump(st);
  if (rc0 != 0) return rc0;
  const size_t nl = s->launches.size();
  for (size_t i = 0; i < nl; ++i) {
    const hlu_launch &L = s->launches[i];
    int rc = 0;
    // the KM=64 companion of a truncation launch runs as a concurrent branch
    if (L.kind == HLU_K_RKT32 && i + 1 < nl && s->launches[i + 1].kind == HLU_K_RKT64) {
      cudaEventRecord(s->ev_fork, st);
      cudaStreamWaitEvent(s->side, s->ev_fork, 0);
      rc = hlu_rk_update_batched_f64(&s->ctx, s->rkt + L.first, s->parts, L.count, 64, s->side);
      if (rc == 0) rc = hlu_rk_update_batched_f64(&s->ctx, s->rkt + L.first, s->parts, L.count, 32, st);
      cudaEventRecord(s->ev_join, s->side);
      cudaStreamWaitEvent(st, s->ev_join, 0);
      ++i;
      if (rc != 0) return rc;
      continue;
    }
    switch (L.kind) {
      case HLU_K_GETRF:
        rc = hlu_getrf_batched_f64(&s->ctx, s->getrf + L.first, L.count, L.smem_dim, st);
        break;
      case HLU_K_TRSM:
        rc = hlu_trsm_batched_f64(&s->ctx, s->trsm + L.first, L.count, L.smem_dim, st);
        break;
      case HLU_K_GEMM:
        rc = hlu_gemm_batched_f64(&s->ctx, s->gemm + L.first, s->terms, L.count, st);
        break;
      case HLU_K_GEMM_SMALL:
        rc = hlu_gemm_small_batched_f64(&s->ctx, s->gemm + L.first, s->terms, L.count, st);
        break;
      case HLU_K_RKT32:
        rc = hlu_rk_update_batched_f64(&s->ctx, s->rkt + L.first, s->parts, L.count, 32, st);
        break;
      case HLU_K_RKT64:
        rc = hlu_rk_update_batched_f64(&s->ctx, s->rkt + L.first, s->parts, L.count, 64, st);
        break;
      default:
        rc = -3;
    }
    if (rc != 0) return rc;
  }
  return 0;
}

extern "C" int hlu_schedule_create(hlu_schedule **out, const hlu_ctx *ctx, const hlu_launch *launches,
                                   int64_t nlaunch, const hlu_getrf_desc *getrf, const hlu_trsm_desc *trsm,
                                   const hlu_gemm_desc *gemm, const hlu_term *terms, hlu_rkt_desc *rkt,
                                   const hlu_rkpart *parts, int use_graph, void *stream) {
  hlu_schedule *s = new hlu_schedule();
  s->ctx = *ctx;
  s->launches.assign(launches, launches + nlaunch);
  s->getrf = getrf;
  s->trsm = trsm;
  s->gemm = gemm;
  s->terms = terms;
  s->rkt = rkt;
  s->parts = parts;
  s->graph = nullptr;
  s->exec = nullptr;
  s->use_graph = use_graph != 0;
  cudaStream_t st = (cudaStream_t)stream;
  cudaStreamCreateWithFlags(&s->side, cudaStreamNonBlocking);
  cudaEventCreateWithFlags(&s->ev_fork, cudaEventDisableTiming);
  cudaEventCreateWithFlags(&s->ev_join, cudaEventDisableTiming);
  if (s->use_graph) {
    // make sure kernel attributes are set outside capture
    hlu_getrf_batched_f64(&s->ctx, s->getrf, 0, 0, st);
    hlu_trsm_batched_f64(&s->ctx, s->trsm, 0, 0, st);
    hlu_rk_update_batched_f64(&s->ctx, s->rkt, s->parts, 0, 32, st);
    hlu_gemm_small_batched_f64(&s->ctx, s->gemm, s->terms, 0, st);
    hlu_gemm_batched_f64(&s->ctx, s->gemm, s->terms, 0, st);
    if (cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal) != cudaSuccess) {
      delete s;
      return -10;
    }
    const int rc = run_launches(s, st);
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
  cudaEventDestroy(s->ev_fork);
  cudaEventDestroy(s->ev_join);
  cudaStreamDestroy(s->side);
  delete s;
  return 0;
}

extern "C" const char *hlu_version(void) { return "hlu_b200 0.1.0 sm_100a"; }

extern "C" int hlu_device_check(void) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return -1;
  cudaDeviceProp p;
  if (cudaGetDeviceProperties(&p, dev) != cudaSuccess) return -1;
  return (p.major == 10) ? 0 : -2;
}
