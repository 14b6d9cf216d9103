// Shared device helpers for the H-LU kernels (sm_100a, fp64).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "hlu_b200.h"

#define HLU_NT 256  // threads per CTA for every batched kernel
#define HLU_NWARP (HLU_NT / 32)

namespace hlu {

// A resolved view: element (i,j) at p[i*rs + j*cs].  p may point to global or
// shared memory (generic addressing), so the same tile routines serve both.
struct Mat {
  double *p;
  int rows, cols;
  long long rs, cs;
  __device__ __forceinline__ double &at(int i, int j) const { return p[i * rs + j * cs]; }
  __device__ __forceinline__ double get(int i, int j) const { return p[i * rs + j * cs]; }
};

__device__ __forceinline__ Mat resolve(const hlu_ctx &c, const hlu_view &v) {
  Mat m;
  m.p = c.pool + v.off;
  m.rows = v.rdyn >= 0 ? c.ranks[v.rdyn] : v.rows;
  m.cols = v.cdyn >= 0 ? c.ranks[v.cdyn] : v.cols;
  m.rs = v.rs;
  m.cs = v.cs;
  return m;
}

__device__ __forceinline__ Mat smat(double *p, int rows, int cols, int ld) {
  Mat m;
  m.p = p;
  m.rows = rows;
  m.cols = cols;
  m.rs = 1;
  m.cs = ld;
  return m;
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// Full-precision fp64 reciprocal / reciprocal square root: the MUFU
// approximation refined by two Newton steps (quadratic convergence from
// >= 2^-20 relative to below one ulp), without the IEEE slow-path branches of
// '/' and sqrt() that dominate latency-bound chains.
__device__ __forceinline__ double fast_rcp(double x) {
  double y;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  double e = fma(-x, y, 1.0);
  y = fma(y, e, y);
  e = fma(-x, y, 1.0);
  return fma(y, e, y);
}

__device__ __forceinline__ double fast_rsqrt(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  const double h = 0.5 * x;
  double t = fma(-h * y, y, 0.5);
  y = fma(y, t, y);
  t = fma(-h * y, y, 0.5);
  y = fma(y, t, y);
  t = fma(-h * y, y, 0.5);
  return fma(y, t, y);
}

// Jacobi rotation helpers.  tan(theta) only steers convergence (any angle is
// an exact rotation once cos/sin are normalised), so it uses one Newton step
// (~1e-13 relative); cos = rsqrt(1 + t^2) keeps cos^2 + sin^2 = 1 to rounding
// with two steps (MUFU ~2^-22 -> 2^-44 -> full precision).
__device__ __forceinline__ double rcp_nr1(double x) {
  double y;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  return fma(y, fma(-x, y, 1.0), y);
}

__device__ __forceinline__ double rsqrt_nr1(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  return fma(y, fma(-0.5 * x * y, y, 0.5), y);
}

__device__ __forceinline__ double rsqrt_nr2(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  const double h = 0.5 * x;
  y = fma(y, fma(-h * y, y, 0.5), y);
  return fma(y, fma(-h * y, y, 0.5), y);
}

// block-wide max over HLU_NT threads; red must hold HLU_NWARP doubles
__device__ __forceinline__ double block_max(double v, double *red) {
  v = warp_max(v);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) red[w] = v;
  __syncthreads();
  double r = red[0];
#pragma unroll
  for (int i = 1; i < HLU_NWARP; ++i) r = fmax(r, red[i]);
  __syncthreads();
  return r;
}

}  // namespace hlu
