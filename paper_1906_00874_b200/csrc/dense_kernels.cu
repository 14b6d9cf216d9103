// Batched dense leaf kernels: unpivoted LU, triangular solves, GEMM chains.
//
// One CTA per descriptor; every launch covers all independent ops of one
// level of the leaf DAG.  Reference call sites:
//   getrf  <- lu_nopivot         (lowrank.py:183-231)
//   trsm   <- trsm_lower_unit / trsm_upper_right / Rk-factor solves
//             (lowrank.py:234-247, hlu.py:415-418, 495-498, 531)
//   gemm   <- gemm_update and the H-operand products _op_matmat,
//             _op_t_matmat, _op_gemm_into, _op_t_gemm_into, _op_rgemm_into
//             (lowrank.py:250-261, hlu.py:160-255), as ordered chains.
#include <climits>

#include "common.cuh"

namespace hlu {

// ---------------------------------------------------------------------------
// GETRF: in-place unpivoted LU in shared memory (n <= 128).
// Pivot test |p| <= 1e-12 * max|A_input| as lowrank.py:194-212; the first
// failing op (program order) is reported through ctx.err[1].
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(HLU_NT) k_getrf(hlu_ctx c, const hlu_getrf_desc *__restrict__ d) {
  extern __shared__ double sm[];
  __shared__ double red[HLU_NWARP];
  const hlu_getrf_desc o = d[blockIdx.x];
  const Mat A = resolve(c, o.a);
  const int n = A.rows;
  const int ld = n + 1;
  const int tid = threadIdx.x;
  double mx = 0.0;
  for (int e = tid; e < n * n; e += HLU_NT) {
    const int i = e % n, j = e / n;
    const double v = A.get(i, j);
    sm[i + j * ld] = v;
    mx = fmax(mx, fabs(v));
  }
  const double tol = 1e-12 * block_max(mx, red);  // includes a __syncthreads
  for (int j = 0; j < n; ++j) {
    const double p = sm[j + j * ld];
    if (fabs(p) <= tol) {
      if (tid == 0) {
        atomicMin(&c.err[1], o.op_id);
        c.dlog[2 * o.lu_index] = p;
        c.dlog[2 * o.lu_index + 1] = tol;
      }
      break;  // p is read from shared memory by every thread: uniform exit
    }
    const int r = n - j - 1;
    for (int i = j + 1 + tid; i < n; i += HLU_NT) sm[i + j * ld] /= p;
    __syncthreads();
    for (int e = tid; e < r * r; e += HLU_NT) {
      const int i = j + 1 + e % r, l = j + 1 + e / r;
      sm[i + l * ld] -= sm[i + j * ld] * sm[j + l * ld];
    }
    __syncthreads();
  }
  __syncthreads();
  for (int e = tid; e < n * n; e += HLU_NT) {
    const int i = e % n, j = e / n;
    A.at(i, j) = sm[i + j * ld];
  }
}

// ---------------------------------------------------------------------------
// TRSM (n <= 128): T in shared memory, right-hand sides in chunks of 64.
//   mode 0: X <- L^-1 X  (unit lower, X n x r)
//   mode 1: X <- X U^-1  (upper,      X r x n)
//   mode 2: X <- U^-1 X  (upper,      X n x r)
// Solve dimension index i, rhs index v; xs[i + v*ld].
// ---------------------------------------------------------------------------
#define TRSM_CHUNK 64
__global__ void __launch_bounds__(HLU_NT) k_trsm(hlu_ctx c, const hlu_trsm_desc *__restrict__ d) {
  extern __shared__ double sm[];
  const hlu_trsm_desc o = d[blockIdx.x];
  const Mat T = resolve(c, o.t);
  const Mat X = resolve(c, o.x);
  const int n = T.rows;
  const int ld = n + 1;
  double *ts = sm;
  double *xs = sm + n * ld;
  const int tid = threadIdx.x;
  const int nrhs = (o.mode == 1) ? X.rows : X.cols;
  if (o.log >= 0 && tid == 0) c.log[o.log] = nrhs;
  for (int e = tid; e < n * n; e += HLU_NT) {
    const int i = e % n, j = e / n;
    ts[i + j * ld] = T.get(i, j);
  }
  for (int v0 = 0; v0 < nrhs; v0 += TRSM_CHUNK) {
    const int nv = min(TRSM_CHUNK, nrhs - v0);
    __syncthreads();
    for (int e = tid; e < n * nv; e += HLU_NT) {
      int i, v;
      if (o.mode == 1) { v = e % nv; i = e / nv; } else { i = e % n; v = e / n; }
      xs[i + v * ld] = (o.mode == 1) ? X.get(v0 + v, i) : X.get(i, v0 + v);
    }
    __syncthreads();
    if (o.mode == 0) {
      for (int j = 0; j < n - 1; ++j) {
        const int r = n - j - 1;
        for (int e = tid; e < r * nv; e += HLU_NT) {
          const int i = j + 1 + e % r, v = e / r;
          xs[i + v * ld] -= ts[i + j * ld] * xs[j + v * ld];
        }
        __syncthreads();
      }
    } else if (o.mode == 1) {
      for (int j = 0; j < n; ++j) {
        const double ujj = ts[j + j * ld];
        const int r = n - j - 1;
        for (int e = tid; e < r * nv; e += HLU_NT) {
          const int l = j + 1 + e % r, v = e / r;
          xs[l + v * ld] -= (xs[j + v * ld] / ujj) * ts[j + l * ld];
        }
        __syncthreads();
      }
      for (int e = tid; e < n * nv; e += HLU_NT) {
        const int i = e % n, v = e / n;
        xs[i + v * ld] /= ts[i + i * ld];
      }
    } else {
      for (int j = n - 1; j >= 0; --j) {
        const double ujj = ts[j + j * ld];
        for (int e = tid; e < j * nv; e += HLU_NT) {
          const int i = e % j, v = e / j;
          xs[i + v * ld] -= ts[i + j * ld] * (xs[j + v * ld] / ujj);
        }
        __syncthreads();
      }
      for (int e = tid; e < n * nv; e += HLU_NT) {
        const int i = e % n, v = e / n;
        xs[i + v * ld] /= ts[i + i * ld];
      }
    }
    __syncthreads();
    for (int e = tid; e < n * nv; e += HLU_NT) {
      int i, v;
      if (o.mode == 1) { v = e % nv; i = e / nv; } else { i = e % n; v = e / n; }
      if (o.mode == 1) X.at(v0 + v, i) = xs[i + v * ld];
      else X.at(i, v0 + v) = xs[i + v * ld];
    }
  }
}

// ---------------------------------------------------------------------------
// GEMM chains.  C += alpha * A B with 64x64 output tiles, k-steps of 16,
// each thread a 4x4 register tile (rows ty+16q, cols tx+16q).
// ---------------------------------------------------------------------------
#define GB 64
#define GK 32
#define GPF (GB * GK / HLU_NT)  // tile elements each thread stages per operand (8)
#define GLD (GB + 1)            // padded tile row: transposed stores stay conflict-free

// C += alpha * A B.  64x64 output tiles, 32-deep k-steps; the next k-tile is
// prefetched into registers while the current one is consumed from shared
// memory, so each k-step costs max(load latency, compute) instead of the sum.
// A operand of a GEMM term read through its triangle (hlu_term.assoc of a GEMM
// term): HLU_TRI_NONE = A, HLU_TRI_UPPER = triu(A), HLU_TRI_UNIT_LOWER =
// tril(A, -1) + I (the stored factors of a dense diagonal leaf, hlu.py:720-767)
__device__ __forceinline__ double tri_get(const Mat &A, int i, int j, int tri) {
  if (tri == HLU_TRI_UPPER) return j >= i ? A.get(i, j) : 0.0;
  if (tri == HLU_TRI_UNIT_LOWER) return j < i ? A.get(i, j) : (j == i ? 1.0 : 0.0);
  return A.get(i, j);
}

__device__ __noinline__ void tile_gemm(const Mat &C, const Mat &A, const Mat &B, double alpha, double *sA,
                                       double *sB, int tri = HLU_TRI_NONE) {
  const int m = C.rows, n = C.cols, k = A.cols;
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  for (int i0 = 0; i0 < m; i0 += GB) {
    for (int j0 = 0; j0 < n; j0 += GB) {
      double acc[4][4];
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) acc[a][b] = 0.0;
      double pa[GPF], pb[GPF];
      // coalescing: walk the operand's unit-stride dimension fastest
      const bool a_rows_fast = A.rs == 1, b_rows_fast = B.rs == 1;
      auto fetch = [&](int k0) {
#pragma unroll
        for (int u = 0; u < GPF; ++u) {
          const int e = tid + u * HLU_NT;
          const int r = a_rows_fast ? e % GB : e / GK, q = a_rows_fast ? e / GB : e % GK;
          const int gi = i0 + r, gk = k0 + q;
          pa[u] = (gi < m && gk < k) ? tri_get(A, gi, gk, tri) : 0.0;
          const int qq = b_rows_fast ? e % GK : e / GB, cc = b_rows_fast ? e / GK : e % GB;
          const int bj = j0 + cc, bk = k0 + qq;
          pb[u] = (bk < k && bj < n) ? B.get(bk, bj) : 0.0;
        }
      };
      fetch(0);
      for (int k0 = 0; k0 < k; k0 += GK) {
        __syncthreads();
#pragma unroll
        for (int u = 0; u < GPF; ++u) {
          const int e = tid + u * HLU_NT;
          const int r = a_rows_fast ? e % GB : e / GK, q = a_rows_fast ? e / GB : e % GK;
          sA[q * GLD + r] = pa[u];
          const int qq = b_rows_fast ? e % GK : e / GB, cc = b_rows_fast ? e / GK : e % GB;
          sB[qq * GLD + cc] = pb[u];
        }
        __syncthreads();
        if (k0 + GK < k) fetch(k0 + GK);  // in flight during the FMAs below
        const int kk = min(GK, k - k0);
        for (int q = 0; q < kk; ++q) {
          double av[4], bv[4];
#pragma unroll
          for (int a = 0; a < 4; ++a) av[a] = sA[q * GLD + ty + 16 * a];
#pragma unroll
          for (int b = 0; b < 4; ++b) bv[b] = sB[q * GLD + tx + 16 * b];
#pragma unroll
          for (int a = 0; a < 4; ++a)
#pragma unroll
            for (int b = 0; b < 4; ++b) acc[a][b] = fma(av[a], bv[b], acc[a][b]);
        }
      }
#pragma unroll
      for (int a = 0; a < 4; ++a) {
        const int gi = i0 + ty + 16 * a;
        if (gi >= m) continue;
#pragma unroll
        for (int b = 0; b < 4; ++b) {
          const int gj = j0 + tx + 16 * b;
          if (gj < n) C.at(gi, gj) += alpha * acc[a][b];
        }
      }
    }
  }
  __syncthreads();
}

__device__ __forceinline__ Mat sub(const Mat &x, int i0, int j0, int rows, int cols) {
  Mat r = x;
  r.p = x.p + i0 * x.rs + j0 * x.cs;
  r.rows = rows;
  r.cols = cols;
  return r;
}

__device__ void zero_mat(const Mat &C) {
  for (int e = threadIdx.x; e < C.rows * C.cols; e += HLU_NT) C.at(e % C.rows, e / C.rows) = 0.0;
  __syncthreads();
}

__global__ void __launch_bounds__(HLU_NT, 2)
    k_gemm(hlu_ctx c, const hlu_gemm_desc *__restrict__ d, const hlu_term *__restrict__ terms) {
  extern __shared__ double gsm[];
  double *sA = gsm;
  double *sB = sA + GLD * GK;
  double *sW = sB + GLD * GK;
  const hlu_gemm_desc o = d[blockIdx.x];
  if (o.log >= 0 && threadIdx.x == 0) c.log[o.log] = c.ranks[o.log_slot];
  for (int t = 0; t < o.term_count; ++t) {
    const hlu_term tm = terms[o.term_begin + t];
    const Mat C = resolve(c, tm.c);
    if (tm.kind == HLU_TERM_ZERO) {
      zero_mat(C);
      continue;
    }
    const Mat A = resolve(c, tm.a);
    const Mat B = resolve(c, tm.b);
    if (C.rows == 0 || C.cols == 0) continue;
    if (tm.kind == HLU_TERM_GEMM) {
      if (A.cols > 0) tile_gemm(C, A, B, tm.alpha, sA, sB, tm.assoc);
      continue;
    }
    const Mat M = resolve(c, tm.m);
    if (M.rows == 0 || M.cols == 0) continue;
    if (tm.assoc == 0) {
      // C += alpha A (M B): W = M[kc,:] B[:, jc] (<= 64 x 64) then C[:, jc] += alpha A[:, kc] W
      for (int kc = 0; kc < M.rows; kc += GB) {
        const int kr = min(GB, M.rows - kc);
        for (int jc = 0; jc < C.cols; jc += GB) {
          const int nc = min(GB, C.cols - jc);
          const Mat W = smat(sW, kr, nc, GB);
          zero_mat(W);
          tile_gemm(W, sub(M, kc, 0, kr, M.cols), sub(B, 0, jc, B.rows, nc), 1.0, sA, sB);
          tile_gemm(sub(C, 0, jc, C.rows, nc), sub(A, 0, kc, A.rows, kr), W, tm.alpha, sA, sB);
        }
      }
    } else {
      // C += alpha (A M) B: W = A[ic,:] M[:, kc] then C[ic,:] += alpha W B[kc,:]
      for (int ic = 0; ic < C.rows; ic += GB) {
        const int mr = min(GB, C.rows - ic);
        for (int kc = 0; kc < M.cols; kc += GB) {
          const int kr = min(GB, M.cols - kc);
          const Mat W = smat(sW, mr, kr, GB);
          zero_mat(W);
          tile_gemm(W, sub(A, ic, 0, mr, A.cols), sub(M, 0, kc, M.rows, kr), 1.0, sA, sB);
          tile_gemm(sub(C, ic, 0, mr, C.cols), W, sub(B, kc, 0, kr, B.cols), tm.alpha, sA, sB);
        }
      }
    }
  }
}

// ---------------------------------------------------------------------------
// Warp-per-chain GEMM for small chains (classified statically by the planner):
// lane = output column, 16-row register blocks, broadcast loads of A; a triple
// term stages W = M B (<= WSMALL doubles) or a row block of A M in per-warp
// shared memory.  Terms run in order with __syncwarp between them.
// ---------------------------------------------------------------------------
#define WSMALL 1024
#define RB 16

// C (m x n) += alpha * A (m x k) * B (k x n); one warp.
__device__ __forceinline__ void warp_gemm(const Mat &C, const Mat &A, const Mat &B, double alpha,
                                          int tri = HLU_TRI_NONE) {
  const int l = threadIdx.x & 31;
  const int m = C.rows, n = C.cols, k = A.cols;
  for (int c = l; c - l < n; c += 32) {
    const bool on = c < n;
    for (int r0 = 0; r0 < m; r0 += RB) {
      double acc[RB];
#pragma unroll
      for (int i = 0; i < RB; ++i) acc[i] = 0.0;
      const int rr = min(RB, m - r0);
      for (int t = 0; t < k; ++t) {
        const double b = on ? B.get(t, c) : 0.0;
#pragma unroll
        for (int i = 0; i < RB; ++i)
          if (i < rr) acc[i] = fma(tri_get(A, r0 + i, t, tri), b, acc[i]);
      }
      if (on) {
#pragma unroll
        for (int i = 0; i < RB; ++i)
          if (i < rr) C.at(r0 + i, c) += alpha * acc[i];
      }
    }
  }
  __syncwarp();
}

__global__ void __launch_bounds__(HLU_NT)
    k_gemm_warp(hlu_ctx c, const hlu_gemm_desc *__restrict__ d, const hlu_term *__restrict__ terms, int count) {
  extern __shared__ double wbuf[];
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  const int di = blockIdx.x * HLU_NWARP + w;
  if (di >= count) return;
  const hlu_gemm_desc o = d[di];
  if (o.log >= 0 && l == 0) c.log[o.log] = c.ranks[o.log_slot];
  double *W = wbuf + w * WSMALL;
  for (int t = 0; t < o.term_count; ++t) {
    const hlu_term tm = terms[o.term_begin + t];
    const Mat C = resolve(c, tm.c);
    if (tm.kind == HLU_TERM_ZERO) {
      for (int e = l; e < C.rows * C.cols; e += 32) C.at(e % C.rows, e / C.rows) = 0.0;
      __syncwarp();
      continue;
    }
    if (C.rows == 0 || C.cols == 0) continue;
    const Mat A = resolve(c, tm.a);
    const Mat B = resolve(c, tm.b);
    if (tm.kind == HLU_TERM_GEMM) {
      if (A.cols > 0) warp_gemm(C, A, B, tm.alpha, tm.assoc);
      continue;
    }
    const Mat M = resolve(c, tm.m);
    if (M.rows == 0 || M.cols == 0) continue;
    if (tm.assoc == 0) {
      // W (k1 x n) = M B, then C += alpha A W
      const Mat Ws = smat(W, M.rows, C.cols, M.rows);
      for (int e = l; e < M.rows * C.cols; e += 32) W[e] = 0.0;
      __syncwarp();
      warp_gemm(Ws, M, B, 1.0);
      warp_gemm(C, A, Ws, tm.alpha);
    } else {
      // per row block: W (rb x k2) = A[rb,:] M, then C[rb,:] += alpha W B
      for (int r0 = 0; r0 < C.rows; r0 += RB) {
        const int rr = min(RB, C.rows - r0);
        const Mat Ws = smat(W, rr, M.cols, rr);
        for (int e = l; e < rr * M.cols; e += 32) W[e] = 0.0;
        __syncwarp();
        Mat Ar = A;
        Ar.p = A.p + r0 * A.rs;
        Ar.rows = rr;
        Mat Cr = C;
        Cr.p = C.p + r0 * C.rs;
        Cr.rows = rr;
        warp_gemm(Ws, Ar, M, 1.0);
        warp_gemm(Cr, Ws, B, tm.alpha);
      }
    }
  }
}

}  // namespace hlu

using namespace hlu;

// dynamic shared-memory opt-ins are per device: one bit per device ordinal and kernel
static bool first_on_device(unsigned long long &mask) {
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev >= 64) return true;
  if ((mask >> dev) & 1ull) return false;
  mask |= 1ull << dev;
  return true;
}

static size_t getrf_smem(int n) { return (size_t)n * (n + 1) * sizeof(double); }
static size_t trsm_smem(int n) { return (size_t)n * (n + 1) * sizeof(double) + (size_t)(n + 1) * TRSM_CHUNK * sizeof(double); }

extern "C" int hlu_getrf_batched_f64(const hlu_ctx *ctx, const hlu_getrf_desc *d, int count, int max_n,
                                     void *stream) {
  static unsigned long long init = 0ull;
  if (first_on_device(init)) {
    cudaFuncSetAttribute(k_getrf, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)getrf_smem(128));
  }
  if (max_n > 128) return -2;
  if (count <= 0) return 0;
  k_getrf<<<count, HLU_NT, getrf_smem(max_n), (cudaStream_t)stream>>>(*ctx, d);
  return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

extern "C" int hlu_trsm_batched_f64(const hlu_ctx *ctx, const hlu_trsm_desc *d, int count, int max_n,
                                    void *stream) {
  static unsigned long long init = 0ull;
  if (first_on_device(init)) {
    cudaFuncSetAttribute(k_trsm, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)trsm_smem(128));
  }
  if (max_n > 128) return -2;
  if (count <= 0) return 0;
  k_trsm<<<count, HLU_NT, trsm_smem(max_n), (cudaStream_t)stream>>>(*ctx, d);
  return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

extern "C" int hlu_gemm_batched_f64(const hlu_ctx *ctx, const hlu_gemm_desc *d, const hlu_term *terms,
                                    int count, void *stream) {
  const size_t smem = (size_t)(2 * GLD * GK + GB * GB) * sizeof(double);
  static unsigned long long init = 0ull;
  if (first_on_device(init)) {
    cudaFuncSetAttribute(k_gemm, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  }
  if (count <= 0) return 0;
  k_gemm<<<count, HLU_NT, smem, (cudaStream_t)stream>>>(*ctx, d, terms);
  return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

extern "C" int hlu_gemm_small_batched_f64(const hlu_ctx *ctx, const hlu_gemm_desc *d, const hlu_term *terms,
                                          int count, void *stream) {
  const size_t smem = (size_t)HLU_NWARP * WSMALL * sizeof(double);
  static unsigned long long init = 0ull;
  if (first_on_device(init)) {
    cudaFuncSetAttribute(k_gemm_warp, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  }
  if (count <= 0) return 0;
  k_gemm_warp<<<(count + HLU_NWARP - 1) / HLU_NWARP, HLU_NT, smem, (cudaStream_t)stream>>>(*ctx, d, terms, count);
  return cudaGetLastError() == cudaSuccess ? 0 : -1;
}
