// Latency microbenchmarks for the fp64 building blocks of the RKT kernel.
#include <cstdio>
#include <cuda_runtime.h>
__device__ double sink;
__global__ void k_dfma(int n, double a, long long *out) {
  double x = a;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) x = fma(x, a, 0.5);
  long long t1 = clock64();
  if (threadIdx.x == 0) { out[0] = t1 - t0; sink = x; }
}
__global__ void k_shfl(int n, double a, long long *out) {
  double x = a + threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) x = __shfl_xor_sync(0xffffffffu, x, 1) + 1.0;
  long long t1 = clock64();
  if (threadIdx.x == 0) { out[0] = t1 - t0; sink = x; }
}
__global__ void k_rcp(int n, double a, long long *out) {
  double x = a;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) { double y; asm volatile("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x)); x = y + 1.0; }
  long long t1 = clock64();
  if (threadIdx.x == 0) { out[0] = t1 - t0; sink = x; }
}
__global__ void k_div(int n, double a, long long *out) {
  double x = a;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) x = 1.0 / x + 1.0;
  long long t1 = clock64();
  if (threadIdx.x == 0) { out[0] = t1 - t0; sink = x; }
}
__global__ void k_sqrt(int n, double a, long long *out) {
  double x = a;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) x = sqrt(x) + 1.0;
  long long t1 = clock64();
  if (threadIdx.x == 0) { out[0] = t1 - t0; sink = x; }
}
__global__ void k_lds(int n, long long *out) {
  __shared__ double s[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) s[i] = i & 7;
  __syncthreads();
  int idx = threadIdx.x & 7;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) idx = (int)s[idx * 8 + (threadIdx.x & 31)] ;
  long long t1 = clock64();
  if (threadIdx.x == 0) { out[0] = t1 - t0; sink = idx; }
}
__global__ void k_bar(int n, long long *out) {
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) out[0] = t1 - t0;
}
__global__ void k_dthru(int n, double a, long long *out) {  // fp64 throughput: 8 independent chains
  double x0 = a, x1 = a + 1, x2 = a + 2, x3 = a + 3, x4 = a + 4, x5 = a + 5, x6 = a + 6, x7 = a + 7;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
    x0 = fma(x0, a, 0.5); x1 = fma(x1, a, 0.5); x2 = fma(x2, a, 0.5); x3 = fma(x3, a, 0.5);
    x4 = fma(x4, a, 0.5); x5 = fma(x5, a, 0.5); x6 = fma(x6, a, 0.5); x7 = fma(x7, a, 0.5);
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) { out[0] = t1 - t0; sink = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7; }
}
int main() {
  long long *d, h;
  cudaMalloc(&d, 8);
  const int n = 4096;
#define RUN(name, launch) launch; cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost); printf("%-28s %8.2f cycles/iter\n", name, (double)h / n);
  RUN("dfma dependent", (k_dfma<<<1, 32>>>(n, 0.999, d)));
  RUN("shfl.f64 + dadd dependent", (k_shfl<<<1, 32>>>(n, 0.5, d)));
  RUN("rcp.approx.f64 + dadd", (k_rcp<<<1, 32>>>(n, 1.5, d)));
  RUN("1/x (IEEE) + dadd", (k_div<<<1, 32>>>(n, 1.5, d)));
  RUN("sqrt (IEEE) + dadd", (k_sqrt<<<1, 32>>>(n, 1.5, d)));
  RUN("lds.f64 dependent", (k_lds<<<1, 32>>>(n, d)));
  RUN("syncthreads 256 thr", (k_bar<<<1, 256>>>(n, d)));
  RUN("dfma 8 chains, 1 warp", (k_dthru<<<1, 32>>>(n, 0.999, d)));
  RUN("dfma 8 chains, 8 warps", (k_dthru<<<1, 256>>>(n, 0.999, d)));
  RUN("dfma 8 chains, 32 warps", (k_dthru<<<1, 1024>>>(n, 0.999, d)));
  return 0;
}
