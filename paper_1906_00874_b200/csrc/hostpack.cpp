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

// --- numpy arrays addressed through their PyObject (id(array)) -----------------
// The per-leaf Python cost of asking numpy for a data pointer
// (__array_interface__: ~2 us, 240 k arrays at cfg3) is the bulk of a
// pack / unpack, so the *_np entry points take the array objects themselves
// and read the fields of numpy's PyArrayObject (ABI-stable head of the struct:
// PyObject_HEAD, data, nd, dimensions, strides, base, descr, flags; descr:
// PyObject_HEAD, typeobj, kind, type, byteorder, flags, type_num).  Every
// array is validated (float64, 2-d, the expected shape, C-contiguous rows,
// writeable for unpack); the Python side self-tests the layout at import and
// falls back to hlu_host_pack / hlu_host_unpack if it does not hold.
namespace {
struct NpView {
  const char *data;
  bool ok;
};
constexpr int NPY_DOUBLE_NUM = 12;
constexpr int NPY_WRITEABLE = 0x0400;
NpView np_view(uint64_t obj, int64_t rows, int64_t cols, bool writeable) {
  const char *o = reinterpret_cast<const char *>(obj);
  const char *data = *reinterpret_cast<const char *const *>(o + 16);
  const int nd = *reinterpret_cast<const int *>(o + 24);
  const int64_t *dims = *reinterpret_cast<const int64_t *const *>(o + 32);
  const int64_t *strides = *reinterpret_cast<const int64_t *const *>(o + 40);
  const char *descr = *reinterpret_cast<const char *const *>(o + 56);
  const int flags = *reinterpret_cast<const int *>(o + 64);
  bool ok = nd == 2 && descr && *reinterpret_cast<const int *>(descr + 28) == NPY_DOUBLE_NUM &&
            descr[26] != '>';
  if (ok) ok = dims[0] == rows && dims[1] == cols;
  if (ok && rows > 0 && cols > 0)
    ok = (cols == 1 || strides[1] == 8) && (rows == 1 || strides[0] == cols * 8);
  if (ok && writeable) ok = (flags & NPY_WRITEABLE) != 0;
  return NpView{data, ok};
}
}  // namespace

// recs[i].host holds id(array); returns 0, or -(i + 1) for the first array
// that is not a C-contiguous float64 (rows x cols) array (nothing is copied then)
extern "C" int64_t hlu_host_pack_np(hlu_pack_rec *recs, int64_t n, double *pool, int threads, int unpack) {
  for (int64_t i = 0; i < n; ++i) {
    const NpView v = np_view((uint64_t)recs[i].host, recs[i].rows, recs[i].cols, unpack != 0);
    if (!v.ok) return -(i + 1);
    recs[i].host = const_cast<char *>(v.data);
  }
  if (unpack) parallel(n, threads, recs, [pool](const hlu_pack_rec &r) { unpack_one(r, pool); });
  else parallel(n, threads, recs, [pool](const hlu_pack_rec &r) { pack_one(r, pool); });
  return 0;
}

extern "C" int hlu_host_pack(const hlu_pack_rec *recs, int64_t n, double *pool, int threads) {
  parallel(n, threads, recs, [pool](const hlu_pack_rec &r) { pack_one(r, pool); });
  return 0;
}

extern "C" int hlu_host_unpack(const hlu_pack_rec *recs, int64_t n, const double *pool, int threads) {
  parallel(n, threads, recs, [pool](const hlu_pack_rec &r) { unpack_one(r, pool); });
  return 0;
}

// Reference FlopCounter total (hlu.py:46-55 and its call sites) from the
// planner's static per-op formulas and the ranks the kernels logged: formula
// 0 = c, 1 = c k, 3 = c k^2, 2 (Rk update) = 2 (kc + kp + 1) c (kp + 1) with
// k = log[flog], kp = log[flog + 1], kc = log[flog + 2].  Fixed 64k-op chunks
// summed in order, so the total does not depend on the thread count.
extern "C" double hlu_effective_flops(const int64_t *formula, const double *coef, const int64_t *flog,
                                      int64_t nops, const int32_t *log, int64_t nlog, int threads) {
  constexpr int64_t CH = 65536;
  const int64_t nch = (nops + CH - 1) / CH;
  std::vector<double> part((size_t)std::max<int64_t>(nch, 1), 0.0);
  if (threads <= 0) threads = (int)std::max(1u, std::thread::hardware_concurrency());
  threads = (int)std::min<int64_t>(threads, std::max<int64_t>(nch, 1));
  auto at = [&](int64_t i) -> double {
    if (nlog <= 0) return 0.0;
    return (double)log[std::min<int64_t>(std::max<int64_t>(i, 0), nlog - 1)];
  };
  auto work = [&](int t) {
    for (int64_t c = t; c < nch; c += threads) {
      double s = 0.0;
      const int64_t e = std::min(nops, (c + 1) * CH);
      for (int64_t i = c * CH; i < e; ++i) {
        const int64_t f = formula[i];
        const int64_t ix = std::max<int64_t>(flog[i], 0);
        const double cf = coef[i];
        if (f == 0) s += cf;
        else if (f == 1) s += cf * at(ix);
        else if (f == 3) { const double k = at(ix); s += cf * k * k; }
        else if (f == 2) { const double kp = at(ix + 1), kc = at(ix + 2); s += 2.0 * (kc + kp + 1.0) * cf * (kp + 1.0); }
      }
      part[(size_t)c] = s;
    }
  };
  std::vector<std::thread> pool;
  for (int t = 0; t < threads; ++t) pool.emplace_back(work, t);
  for (auto &th : pool) th.join();
  double tot = 0.0;
  for (double v : part) tot += v;
  return tot;
}
