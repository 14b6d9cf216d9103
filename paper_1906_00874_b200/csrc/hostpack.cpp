// Host-side packing of H-matrix leaf payloads into / out of the (pinned)
// staging pool: the numpy leaves are row-major (C-contiguous, as the
// reference's LowRank forces, lowrank.py:50-51), the device pool is
// column-major with a leading dimension per leaf (include/hlu_b200.h).
// Every record is an independent transpose-copy; records are spread over
// worker threads (the upload / download of a cfg3 factorization moves 7 GB).
#include <algorithm>
#include <cstdint>
#include <cstring>
#include <thread>
#include <vector>

#include "hlu_plan.h"

namespace {

// row-major src (rows x cols, row stride ss) -> column-major dst (ld)
void pack_one(const hlu_pack_rec &r, double *pool) {
  const double *src = reinterpret_cast<const double *>(r.host);
  double *dst = pool + r.off;
  const int64_t rows = r.rows, cols = r.cols, ld = r.ld, ss = r.host_stride;
  if (cols == 1) {
    for (int64_t i = 0; i < rows; ++i) dst[i] = src[i * ss];
    return;
  }
  constexpr int64_t B = 32;  // cache-blocked transpose
  for (int64_t i0 = 0; i0 < rows; i0 += B)
    for (int64_t j0 = 0; j0 < cols; j0 += B) {
      const int64_t i1 = std::min(rows, i0 + B), j1 = std::min(cols, j0 + B);
      for (int64_t j = j0; j < j1; ++j)
        for (int64_t i = i0; i < i1; ++i) dst[i + j * ld] = src[i * ss + j];
    }
}

void unpack_one(const hlu_pack_rec &r, const double *pool) {
  double *dst = reinterpret_cast<double *>(r.host);
  const double *src = pool + r.off;
  const int64_t rows = r.rows, cols = r.cols, ld = r.ld, ss = r.host_stride;
  if (cols == 1) {
    for (int64_t i = 0; i < rows; ++i) dst[i * ss] = src[i];
    return;
  }
  constexpr int64_t B = 32;
  for (int64_t i0 = 0; i0 < rows; i0 += B)
    for (int64_t j0 = 0; j0 < cols; j0 += B) {
      const int64_t i1 = std::min(rows, i0 + B), j1 = std::min(cols, j0 + B);
      for (int64_t i = i0; i < i1; ++i)
        for (int64_t j = j0; j < j1; ++j) dst[i * ss + j] = src[i + j * ld];
    }
}

template <class F>
void parallel(int64_t n, int threads, const hlu_pack_rec *recs, F f) {
  if (threads <= 0) threads = (int)std::max(1u, std::thread::hardware_concurrency());
  // balance by element count: contiguous record ranges of about equal work
  std::vector<int64_t> cum(n + 1, 0);
  for (int64_t i = 0; i < n; ++i) cum[i + 1] = cum[i] + (int64_t)recs[i].rows * recs[i].cols + 16;
  threads = (int)std::min<int64_t>(threads, std::max<int64_t>(1, n));
  std::vector<std::thread> pool;
  int64_t begin = 0;
  for (int t = 0; t < threads; ++t) {
    const int64_t target = cum[n] * (t + 1) / threads;
    int64_t end = begin;
    while (end < n && cum[end + 1] <= target) ++end;
    if (t == threads - 1) end = n;
    pool.emplace_back([=]() {
      for (int64_t i = begin; i < end; ++i) f(recs[i]);
    });
    begin = end;
  }
  for (auto &th : pool) th.join();
}

}  // namespace

extern "C" int hlu_host_pack(const hlu_pack_rec *recs, int64_t n, double *pool, int threads) {
  parallel(n, threads, recs, [pool](const hlu_pack_rec &r) { pack_one(r, pool); });
  return 0;
}

extern "C" int hlu_host_unpack(const hlu_pack_rec *recs, int64_t n, const double *pool, int threads) {
  parallel(n, threads, recs, [pool](const hlu_pack_rec &r) { unpack_one(r, pool); });
  return 0;
}
