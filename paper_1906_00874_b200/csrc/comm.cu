// Multi-GPU data plane of the owner-computes H-LU: NCCL over
// NVLink / NVSwitch, loaded at run time (dlopen of libnccl.so.2, the copy the
// process already has when torch is imported), so the library still loads on
// machines without NCCL.
//
// The exchange of one (level, source rank) group of a sharded plan
// (include/hlu_plan.h hlu_xfer): the source gathers the slots' payloads (and
// the Rk ranks) into a staging buffer with one kernel, one ncclBroadcast over
// the communicator, the other ranks scatter it into their pools.  Everything
// is stream-ordered and captured into the schedule's CUDA graph.
#include <dlfcn.h>
#include <nccl.h>

#include <cstdio>
#include <cstring>

#include <algorithm>

#include "common.cuh"
#include "hlu_plan.h"

namespace {

struct NcclApi {
  bool ok = false;
  ncclResult_t (*getUniqueId)(ncclUniqueId *);
  ncclResult_t (*commInitRank)(ncclComm_t *, int, ncclUniqueId, int);
  ncclResult_t (*commDestroy)(ncclComm_t);
  ncclResult_t (*broadcast)(const void *, void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
  ncclResult_t (*allReduce)(const void *, void *, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t);
  ncclResult_t (*groupStart)();
  ncclResult_t (*groupEnd)();
};

NcclApi &nccl() {
  static NcclApi api;
  static bool tried = false;
  if (tried) return api;
  tried = true;
  void *h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
  if (!h) return api;
  api.getUniqueId = (decltype(api.getUniqueId))dlsym(h, "ncclGetUniqueId");
  api.commInitRank = (decltype(api.commInitRank))dlsym(h, "ncclCommInitRank");
  api.commDestroy = (decltype(api.commDestroy))dlsym(h, "ncclCommDestroy");
  api.broadcast = (decltype(api.broadcast))dlsym(h, "ncclBroadcast");
  api.allReduce = (decltype(api.allReduce))dlsym(h, "ncclAllReduce");
  api.groupStart = (decltype(api.groupStart))dlsym(h, "ncclGroupStart");
  api.groupEnd = (decltype(api.groupEnd))dlsym(h, "ncclGroupEnd");
  api.ok = api.getUniqueId && api.commInitRank && api.commDestroy && api.broadcast && api.allReduce &&
           api.groupStart && api.groupEnd;
  return api;
}

}  // namespace

struct hlu_comm {
  ncclComm_t comm;
  int nranks, rank;
};

namespace hlu {

// gather: one warp per record, payload then the rank (as a double)
__global__ void k_xfer_pack(const double *__restrict__ pool, const int32_t *__restrict__ ranks,
                            const hlu_xfer *__restrict__ x, int n, double *__restrict__ buf) {
  const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, l = threadIdx.x & 31;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  for (int i = w; i < n; i += nw) {
    const hlu_xfer r = x[i];
    const double *src = pool + r.off;
    double *dst = buf + r.boff;
    for (int64_t e = l; e < r.len; e += 32) dst[e] = src[e];
    if (l == 0) dst[r.len] = r.rank_slot >= 0 ? (double)ranks[r.rank_slot] : 0.0;
  }
}

__global__ void k_xfer_unpack(double *__restrict__ pool, int32_t *__restrict__ ranks, const hlu_xfer *__restrict__ x,
                              int n, const double *__restrict__ buf) {
  const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, l = threadIdx.x & 31;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  for (int i = w; i < n; i += nw) {
    const hlu_xfer r = x[i];
    const double *src = buf + r.boff;
    double *dst = pool + r.off;
    for (int64_t e = l; e < r.len; e += 32) dst[e] = src[e];
    if (l == 0 && r.rank_slot >= 0) ranks[r.rank_slot] = (int32_t)src[r.len];
  }
}

}  // namespace hlu

using namespace hlu;

extern "C" int hlu_comm_available(void) { return nccl().ok ? 1 : 0; }

extern "C" int hlu_comm_unique_id(void *out) {
  NcclApi &api = nccl();
  if (!api.ok) return -20;
  ncclUniqueId id;
  if (api.getUniqueId(&id) != ncclSuccess) return -21;
  std::memcpy(out, &id, sizeof(id));
  return (int)sizeof(id);
}

extern "C" int hlu_comm_init(hlu_comm **out, const void *id, int nranks, int rank) {
  NcclApi &api = nccl();
  if (!api.ok) return -20;
  ncclUniqueId uid;
  std::memcpy(&uid, id, sizeof(uid));
  hlu_comm *c = new hlu_comm();
  c->nranks = nranks;
  c->rank = rank;
  if (api.commInitRank(&c->comm, nranks, uid, rank) != ncclSuccess) {
    delete c;
    return -22;
  }
  *out = c;
  return 0;
}

extern "C" int hlu_comm_destroy(hlu_comm *c) {
  if (!c) return 0;
  nccl().commDestroy(c->comm);
  delete c;
  return 0;
}

// one (level, src, group) exchange: x = its records (device), n records,
// count = staging doubles (sum of len + 1)
extern "C" int hlu_xfer_group(hlu_comm *c, double *pool, int32_t *ranks, const void *xfer_dev, int n, int src,
                              int64_t count, double *staging, void *stream) {
  cudaStream_t st = (cudaStream_t)stream;
  const hlu_xfer *x = (const hlu_xfer *)xfer_dev;
  if (n <= 0) return 0;
  const int grid = std::min(4 * 148, (n + 7) / 8);
  if (c->rank == src) k_xfer_pack<<<grid, 256, 0, st>>>(pool, ranks, x, n, staging);
  if (nccl().broadcast(staging, staging, (size_t)count, ncclFloat64, src, c->comm, st) != ncclSuccess) return -23;
  if (c->rank != src) k_xfer_unpack<<<grid, 256, 0, st>>>(pool, ranks, x, n, staging);
  return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

// the ranks' flop logs and error words are combined after the factorization:
// log entries are written by exactly the ranks that run the op (same value),
// so MAX reduces them; overflow / unsupported counts add up; the first failing
// LU op is the smallest op id
extern "C" int hlu_comm_reduce_logs(hlu_comm *c, int32_t *log, int64_t nlog, int32_t *err, void *stream) {
  cudaStream_t st = (cudaStream_t)stream;
  NcclApi &api = nccl();
  api.groupStart();
  api.allReduce(log, log, (size_t)nlog, ncclInt32, ncclMax, c->comm, st);
  api.allReduce(err, err, 1, ncclInt32, ncclSum, c->comm, st);
  api.allReduce(err + 1, err + 1, 1, ncclInt32, ncclMin, c->comm, st);
  api.allReduce(err + 2, err + 2, 1, ncclInt32, ncclSum, c->comm, st);
  return api.groupEnd() == ncclSuccess ? 0 : -24;
}
