// Microbenchmark: cudaGraphInstantiate time vs graph shape (diagnostics for the DAG schedule).
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <chrono>
#include <cuda_runtime.h>
__global__ void k_empty(int *p) { if (p && threadIdx.x == 9999) *p = 1; }
struct Big { long long v[30]; };
template <int I>
__global__ void k_var(Big b, int *p) { extern __shared__ double sm[]; if (p && threadIdx.x == 9999) { sm[0] = (double)b.v[I % 30]; *p = (int)sm[0] + I; } }
typedef void (*kfn)(Big, int *);
static kfn g_fns[8] = {k_var<0>, k_var<1>, k_var<2>, k_var<3>, k_var<4>, k_var<5>, k_var<6>, k_var<7>};
static int g_mode = 0;  // 0 empty kernel, 1 8 kernels with 240-byte params, 2 + dynamic smem opt-in (100 KB)
static double now() { return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count(); }
// shape: nodes n, every node depends on `deg` random nodes among the previous `window` nodes
static void run(const char *name, int n, int deg, int window, int ntails, size_t hog_gb) {
  void *hog = nullptr;
  if (hog_gb) cudaMalloc(&hog, hog_gb << 30);
  cudaStream_t st;
  cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal);
  std::vector<cudaGraphNode_t> nodes;
  std::vector<cudaGraphNode_t> deps;
  srand(1);
  double t0 = now();
  for (int i = 0; i < n; ++i) {
    deps.clear();
    for (int d = 0; d < deg && !nodes.empty(); ++d) {
      int lo = (int)nodes.size() - window; if (lo < 0) lo = 0;
      int j = lo + rand() % ((int)nodes.size() - lo);
      for (int t = 0; t < ntails; ++t) { int jj = j - t; if (jj >= lo) deps.push_back(nodes[jj]); }
    }
    cudaStreamUpdateCaptureDependencies(st, deps.data(), deps.size(), cudaStreamSetCaptureDependencies);
    if (g_mode == 0) k_empty<<<1, 32, 0, st>>>(nullptr);
    else { Big b{}; g_fns[i % 8]<<<1 + i % 5, 32 * (1 + i % 8), g_mode == 2 ? (size_t)(8192 * (1 + i % 12)) : 0, st>>>(b, nullptr); }
    cudaStreamCaptureStatus s; const cudaGraphNode_t *d; size_t nd;
    cudaStreamGetCaptureInfo(st, &s, nullptr, nullptr, &d, &nd);
    nodes.push_back(d[0]);
  }
  // join
  int lo = n > 2000 ? n - 2000 : 0;
  deps.assign(nodes.begin() + lo, nodes.end());
  cudaStreamUpdateCaptureDependencies(st, deps.data(), deps.size(), cudaStreamSetCaptureDependencies);
  k_empty<<<1, 32, 0, st>>>(nullptr);
  cudaGraph_t g; cudaStreamEndCapture(st, &g);
  double t1 = now();
  cudaGraphExec_t ex; cudaError_t e = cudaGraphInstantiate(&ex, g, 0);
  double t2 = now();
  cudaGraphLaunch(ex, st); cudaStreamSynchronize(st);
  double t3 = now();
  cudaGraphLaunch(ex, st); cudaStreamSynchronize(st);
  double t4 = now();
  printf("%-28s n=%d deg=%d win=%d tails=%d hog=%zuGB: capture %.2fs instantiate %.2fs (%.1f us/node) first launch %.3fs second %.3fs %s\n",
         name, n, deg, window, ntails, hog_gb, t1 - t0, t2 - t1, (t2 - t1) / n * 1e6, t3 - t2, t4 - t3, cudaGetErrorString(e));
  if (!getenv("KEEP")) cudaGraphExecDestroy(ex);
  cudaGraphDestroy(g); cudaStreamDestroy(st);
  if (hog) cudaFree(hog);
}
#include <thread>
int main() {
  for (int k = 0; k < 8; ++k) cudaFuncSetAttribute(g_fns[k], cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  g_mode = 2;
  cudaFree(0);
  // concurrent instantiation from several host threads: does the driver serialise it?
  for (int nt : {1, 4, 8}) {
    double t0 = now();
    std::vector<std::thread> th;
    for (int t = 0; t < nt; ++t) th.emplace_back([] { run("thread 12k x4", 12000, 7, 1000, 1, 0); run("thread 12k x4", 12000, 7, 1000, 1, 0); });
    for (auto &x : th) x.join();
    printf("== %d threads x 2 graphs of 12k nodes: %.2fs wall\n", nt, now() - t0);
  }
  return 0;
}
