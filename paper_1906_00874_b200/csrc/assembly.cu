// GPU assembly of the BEM H-matrix (reference
// kernels.py:73-168, restated host-side in paper_1906_00874_b200/kernels.py):
//
//   dense leaves   A_ij = g(|x_i - y_j|), coincident points at the
//                  regularisation distance (assemble_dense_block, kernels.py:73-84)
//   Rk leaves      U_t K(nodes_t, nodes_s) U_s^T by tensor Chebyshev
//                  interpolation on the clusters' bounding boxes
//                  (assemble_lowrank_block, kernels.py:140-153), written as the
//                  factor pair X = U_t K (m x Ks), Y = U_s (n x Ks) that the
//                  batched truncation (hlu_rk_update_batched_f64, RECOMPRESS)
//                  then recompresses exactly as recompress() does.
//   HODLR blocks   partially pivoted adaptive cross approximation of a kernel
//                  block to k terms (cfg5 generator; the dense SVD route of
//                  compress_dense is O(n^2) memory at n = 1M), followed by the
//                  same truncation.
//
// The distance and kernel arithmetic follows numpy's operation order with
// explicitly rounded intrinsics (no FMA contraction), so d = 3 dense leaves are
// bit-identical to the host / reference assembly.
#include "common.cuh"

namespace hlu {

struct AsmDesc {  // mirrors hlu_asm_desc (include/hlu_b200.h)
  int32_t r0, r1, c0, c1;
  int32_t tcl, scl;  // cluster ids (Rk leaves: interpolation nodes)
  int32_t kind, pad;
  int64_t out_a, out_b;
};

__device__ __forceinline__ double dist_rn(const double *x, const double *y, int d) {
  // ((dx*dx + dy*dy) + dz*dz), sqrt: numpy's delta*delta, add.reduce, sqrt
  double acc = 0.0;
  for (int a = 0; a < d; ++a) {
    const double t = __dsub_rn(x[a], y[a]);
    acc = a == 0 ? __dmul_rn(t, t) : __dadd_rn(acc, __dmul_rn(t, t));
  }
  return __dsqrt_rn(acc);
}

// kernels.py:_green: d = 3: 1 / (4 pi r); d = 2: -log(r) / (2 pi); d = 1: -log(r)
__device__ __forceinline__ double green(double r, int d) {
  if (d == 3) return __ddiv_rn(1.0, __dmul_rn(12.566370614359172, r));  // 4.0 * math.pi
  if (d == 2) return __ddiv_rn(-log(r), 6.283185307179586);            // 2.0 * math.pi
  return -log(r);
}

// one CTA per dense leaf, column-major output at pool + out_a
__global__ void k_asm_dense(const double *__restrict__ pts, int d, const AsmDesc *__restrict__ desc, double diag,
                            double *__restrict__ pool) {
  const AsmDesc o = desc[blockIdx.x];
  const int m = o.r1 - o.r0, n = o.c1 - o.c0;
  double *out = pool + o.out_a;
  for (int e = threadIdx.x; e < m * n; e += blockDim.x) {
    const int i = e % m, j = e / m;
    double r = dist_rn(pts + (int64_t)(o.r0 + i) * d, pts + (int64_t)(o.c0 + j) * d, d);
    if (r == 0.0) r = diag;
    out[e] = green(r, d);
  }
}

#define CHEB_MAX 8    // interpolation order
#define CHEB_NG 512   // tensor grid points per cluster (CHEB_MAX^3)

// per-cluster interpolation data: per axis the node count (1 for a degenerate
// axis), the nodes and the barycentric weights (computed on the host with the
// reference's numpy expressions, kernels.py:84-104)
struct ChebCl {
  const int32_t *cnt;    // ncl x 3
  const double *nodes;   // ncl x 3 x CHEB_MAX
  const double *w;       // ncl x 3 x CHEB_MAX
};

// Lagrange basis of axis a of cluster c at x (kernels.py:lagrange_basis)
__device__ void lagrange(const ChebCl &cb, int c, int a, double x, double *L) {
  const int q = cb.cnt[c * 3 + a];
  const double *nd = cb.nodes + ((int64_t)c * 3 + a) * CHEB_MAX;
  const double *w = cb.w + ((int64_t)c * 3 + a) * CHEB_MAX;
  if (q == 1) {
    L[0] = 1.0;
    return;
  }
  int hit = -1;
  double sum = 0.0;
  for (int mu = 0; mu < q; ++mu) {
    const double diff = __dsub_rn(x, nd[mu]);
    if (diff == 0.0) hit = mu;
    L[mu] = __ddiv_rn(w[mu], diff == 0.0 ? 1.0 : diff);
    sum = mu == 0 ? L[0] : __dadd_rn(sum, L[mu]);
  }
  for (int mu = 0; mu < q; ++mu) L[mu] = hit >= 0 ? (mu == hit ? 1.0 : 0.0) : __ddiv_rn(L[mu], sum);
}

// tensor index p of cluster c -> the grid point (meshgrid "ij" order)
__device__ void grid_point(const ChebCl &cb, int c, int d, int p, double *x) {
  for (int a = d - 1; a >= 0; --a) {
    const int q = cb.cnt[c * 3 + a];
    x[a] = cb.nodes[((int64_t)c * 3 + a) * CHEB_MAX + p % q];
    p /= q;
  }
}

// tensor basis value of grid index p (first axis slowest), multiplied in the
// reference's order ((L_0 L_1) L_2) (kernels.py:_tensor_basis)
__device__ __forceinline__ double tensor_basis(const ChebCl &cb, int c, int d, int p, const double (*L)[CHEB_MAX]) {
  int idx[3];
  for (int a = d - 1; a >= 0; --a) {
    const int q = cb.cnt[c * 3 + a];
    idx[a] = p % q;
    p /= q;
  }
  double u = L[0][idx[0]];
  for (int a = 1; a < d; ++a) u = __dmul_rn(u, L[a][idx[a]]);
  return u;
}

__device__ __forceinline__ int grid_size(const ChebCl &cb, int c, int d) {
  int g = 1;
  for (int a = 0; a < d; ++a) g *= cb.cnt[c * 3 + a];
  return g;
}

// one CTA per Rk leaf: X = U_t K (m x Gs, ld m) at pool + out_a and
// Y = U_s (n x Gs, ld n) at pool + out_b
__global__ void __launch_bounds__(256)
    k_asm_cheb(const double *__restrict__ pts, int d, const AsmDesc *__restrict__ desc, ChebCl cb,
               double *__restrict__ pool) {
  extern __shared__ double sm[];  // core Gt x Gs
  const AsmDesc o = desc[blockIdx.x];
  const int m = o.r1 - o.r0, n = o.c1 - o.c0;
  const int gt = grid_size(cb, o.tcl, d), gs = grid_size(cb, o.scl, d);
  for (int e = threadIdx.x; e < gt * gs; e += blockDim.x) {
    const int p = e % gt, q = e / gt;
    double xt[3], xs[3];
    grid_point(cb, o.tcl, d, p, xt);
    grid_point(cb, o.scl, d, q, xs);
    sm[e] = green(dist_rn(xt, xs, d), d);
  }
  __syncthreads();
  double *X = pool + o.out_a, *Y = pool + o.out_b;
  // rows of U_t: tensor products of the per-axis bases, first axis slowest
  for (int i = threadIdx.x; i < m; i += blockDim.x) {
    double L[3][CHEB_MAX];
    const double *x = pts + (int64_t)(o.r0 + i) * d;
    for (int a = 0; a < d; ++a) lagrange(cb, o.tcl, a, x[a], L[a]);
    for (int q = 0; q < gs; ++q) {
      double acc = 0.0;
      for (int p = 0; p < gt; ++p) acc = fma(tensor_basis(cb, o.tcl, d, p, L), sm[p + q * gt], acc);
      X[i + (int64_t)q * m] = acc;
    }
  }
  for (int j = threadIdx.x; j < n; j += blockDim.x) {
    double L[3][CHEB_MAX];
    const double *y = pts + (int64_t)(o.c0 + j) * d;
    for (int a = 0; a < d; ++a) lagrange(cb, o.scl, a, y[a], L[a]);
    for (int q = 0; q < gs; ++q) Y[j + (int64_t)q * n] = tensor_basis(cb, o.scl, d, q, L);
  }
}

// Partially pivoted ACA of the kernel block rows [r0, r1) x cols [c0, c1) to
// at most k terms: U (m x k, ld m) at pool + out_a, V (n x k, ld n) at
// pool + out_b, the block ~= U V^T; the term count goes to nterms[blockIdx].
// One CTA per block; the residual row / column of every step is evaluated
// on the fly.  Stops early on an exactly zero pivot.
__global__ void __launch_bounds__(512)
    k_asm_aca(const double *__restrict__ pts, int d, const AsmDesc *__restrict__ desc, int k, double diag,
              double *__restrict__ pool, int32_t *__restrict__ nterms) {
  __shared__ double rv[32];
  __shared__ int ri[32];
  __shared__ int s_i, s_j;
  __shared__ double s_piv;
  const AsmDesc o = desc[blockIdx.x];
  const int m = o.r1 - o.r0, n = o.c1 - o.c0;
  double *U = pool + o.out_a, *V = pool + o.out_b;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, nw = blockDim.x >> 5;
  int istar = 0;
  int used = 0;
  for (int t = 0; t < k; ++t) {
    // residual row istar: V[:, t] = A[istar, :] - sum_l U[istar, l] V[:, l]
    for (int j = tid; j < n; j += blockDim.x) {
      double r = dist_rn(pts + (int64_t)(o.r0 + istar) * d, pts + (int64_t)(o.c0 + j) * d, d);
      if (r == 0.0) r = diag;
      double a = green(r, d);
      for (int l = 0; l < t; ++l) a -= U[istar + (int64_t)l * m] * V[j + (int64_t)l * n];
      V[j + (int64_t)t * n] = a;
    }
    __syncthreads();
    // column pivot: argmax |V[:, t]| (smallest index on ties)
    double best = -1.0;
    int bj = 0;
    for (int j = tid; j < n; j += blockDim.x) {
      const double v = fabs(V[j + (int64_t)t * n]);
      if (v > best) {
        best = v;
        bj = j;
      }
    }
    for (int off = 16; off > 0; off >>= 1) {
      const double ob = __shfl_xor_sync(0xffffffffu, best, off);
      const int oj = __shfl_xor_sync(0xffffffffu, bj, off);
      if (ob > best || (ob == best && oj < bj)) {
        best = ob;
        bj = oj;
      }
    }
    if (lane == 0) {
      rv[wid] = best;
      ri[wid] = bj;
    }
    __syncthreads();
    if (tid == 0) {
      double b = rv[0];
      int j = ri[0];
      for (int w = 1; w < nw; ++w)
        if (rv[w] > b || (rv[w] == b && ri[w] < j)) {
          b = rv[w];
          j = ri[w];
        }
      s_j = j;
      s_piv = V[j + (int64_t)t * n];
    }
    __syncthreads();
    const double piv = s_piv;
    const int jstar = s_j;
    if (piv == 0.0) break;  // exact residual row: the block is represented exactly
    for (int j = tid; j < n; j += blockDim.x) V[j + (int64_t)t * n] /= piv;
    // residual column jstar: U[:, t] = A[:, jstar] - sum_l U[:, l] V[jstar, l]
    for (int i = tid; i < m; i += blockDim.x) {
      double r = dist_rn(pts + (int64_t)(o.r0 + i) * d, pts + (int64_t)(o.c0 + jstar) * d, d);
      if (r == 0.0) r = diag;
      double a = green(r, d);
      for (int l = 0; l < t; ++l) a -= U[i + (int64_t)l * m] * V[jstar + (int64_t)l * n];
      U[i + (int64_t)t * m] = a;
    }
    ++used;
    __syncthreads();
    // next row pivot: argmax |U[:, t]| over rows other than istar
    best = -1.0;
    int bi = 0;
    for (int i = tid; i < m; i += blockDim.x) {
      const double v = i == istar ? -1.0 : fabs(U[i + (int64_t)t * m]);
      if (v > best) {
        best = v;
        bi = i;
      }
    }
    for (int off = 16; off > 0; off >>= 1) {
      const double ob = __shfl_xor_sync(0xffffffffu, best, off);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, off);
      if (ob > best || (ob == best && oi < bi)) {
        best = ob;
        bi = oi;
      }
    }
    __syncthreads();
    if (lane == 0) {
      rv[wid] = best;
      ri[wid] = bi;
    }
    __syncthreads();
    if (tid == 0) {
      double b = rv[0];
      int i = ri[0];
      for (int w = 1; w < nw; ++w)
        if (rv[w] > b || (rv[w] == b && ri[w] < i)) {
          b = rv[w];
          i = ri[w];
        }
      s_i = i;
    }
    __syncthreads();
    istar = s_i;
  }
  if (tid == 0) nterms[blockIdx.x] = used;
}

}  // namespace hlu

using namespace hlu;

extern "C" int hlu_asm_dense_f64(const double *pts, int d, const void *desc, int count, double diag, double *pool,
                                 void *stream) {
  if (count <= 0) return 0;
  k_asm_dense<<<count, 256, 0, (cudaStream_t)stream>>>(pts, d, (const AsmDesc *)desc, diag, pool);
  return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

extern "C" int hlu_asm_cheb_f64(const double *pts, int d, const void *desc, int count, const int32_t *cl_cnt,
                                const double *cl_nodes, const double *cl_w, int max_grid, double *pool,
                                void *stream) {
  if (count <= 0) return 0;
  if (max_grid > CHEB_NG) return -2;
  const size_t smem = (size_t)max_grid * max_grid * sizeof(double);
  static unsigned long long init = 0ull;
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev >= 64 || !((init >> dev) & 1ull)) {
    cudaFuncSetAttribute(k_asm_cheb, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
    if (dev < 64) init |= 1ull << dev;
  }
  if (smem > 220 * 1024) return -2;
  ChebCl cb{cl_cnt, cl_nodes, cl_w};
  k_asm_cheb<<<count, 256, smem, (cudaStream_t)stream>>>(pts, d, (const AsmDesc *)desc, cb, pool);
  return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

extern "C" int hlu_asm_aca_f64(const double *pts, int d, const void *desc, int count, int k, double diag,
                               double *pool, int32_t *nterms, void *stream) {
  if (count <= 0) return 0;
  k_asm_aca<<<count, 512, 0, (cudaStream_t)stream>>>(pts, d, (const AsmDesc *)desc, k, diag, pool, nterms);
  return cudaGetLastError() == cudaSuccess ? 0 : -1;
}
