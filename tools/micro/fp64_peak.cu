// fp64 peak microbenchmark on B200: DMMA (mma.sync.m16n8k8.f64) and scalar
// DFMA throughput with every SM busy (8 independent accumulator chains per
// warp, 16 warps per SM).  Prints one JSON line.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 fp64_peak.cu -o fp64_peak
#include <cstdio>
#include <cuda_runtime.h>

#define CHAINS 8
#define ITERS 4096

__global__ void k_dmma(double *out, double seed) {
  double d[CHAINS][4];
  double a[4] = {seed, seed * 0.5, seed * 0.25, seed * 0.125};
  double b[2] = {seed * 1e-3, -seed * 1e-3};
  for (int c = 0; c < CHAINS; ++c)
    for (int v = 0; v < 4; ++v) d[c][v] = 0.0;
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int c = 0; c < CHAINS; ++c)
      asm volatile("mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
                   : "+d"(d[c][0]), "+d"(d[c][1]), "+d"(d[c][2]), "+d"(d[c][3])
                   : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(b[0]), "d"(b[1]));
  }
  double s = 0.0;
  for (int c = 0; c < CHAINS; ++c)
    for (int v = 0; v < 4; ++v) s += d[c][v];
  if (s == 12345.678) out[0] = s;
}

__global__ void k_dfma(double *out, double seed) {
  double x[CHAINS];
  const double y = seed * 1e-3, z = 1.0 - 1e-9;
  for (int c = 0; c < CHAINS; ++c) x[c] = seed + c;
  for (int it = 0; it < ITERS * 4; ++it) {
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) x[c] = fma(x[c], z, y);
  }
  double s = 0.0;
  for (int c = 0; c < CHAINS; ++c) s += x[c];
  if (s == 12345.678) out[0] = s;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double *out;
  cudaMalloc(&out, 8);
  const int threads = 512, blocks = sms * 4;  // 64 warps per SM
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best_mma = 1e30f, best_fma = 1e30f;
  for (int rep = 0; rep < 5; ++rep) {
    cudaEventRecord(e0);
    k_dmma<<<blocks, threads>>>(out, 1.0);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best_mma) best_mma = ms;
    cudaEventRecord(e0);
    k_dfma<<<blocks, threads>>>(out, 1.0);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best_fma) best_fma = ms;
  }
  const double warps = (double)blocks * threads / 32;
  const double mma_flops = warps * ITERS * CHAINS * (2.0 * 16 * 8 * 8);
  const double fma_flops = (double)blocks * threads * ITERS * 4 * CHAINS * 2.0;
  printf("{\"sms\": %d, \"dmma_m16n8k8_tflops\": %.2f, \"dfma_tflops\": %.2f, \"dmma_ms\": %.3f, \"dfma_ms\": %.3f}\n",
         sms, mma_flops / best_mma / 1e9, fma_flops / best_fma / 1e9, best_mma, best_fma);
  return cudaGetLastError() == cudaSuccess ? 0 : 1;
}
