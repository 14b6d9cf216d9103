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
#include <algorithm>
#include <climits>

#include "common.cuh"

namespace hlu {

// ---------------------------------------------------------------------------
// GEMM chains on the fp64 tensor cores (DMMA, mma.sync.m16n8k8.f64).
// C += alpha * A B with 64x64 output tiles and 32-deep k-tiles staged in
// shared memory; 8 warps in a 4 (M) x 2 (N) grid, each warp a 16 x 32 block
// = 4 m16n8 accumulator fragments (16 fp64 registers per lane).
// ---------------------------------------------------------------------------
#define GB 64
#define GK 32
#define GPF (GB * GK / HLU_NT)  // tile elements each thread stages per operand (8)
// Shared tile layouts, chosen per operand orientation so that both the
// coalesced staging stores and the fragment loads are bank-conflict free:
//   the operand's unit-stride dimension fastest in the tile -> ld 68 (k-major
//   A / n-major B, "GL64") or ld 36 (m-major A / k-fastest B, "GL32").
#define GL64 68
#define GL32 36
#define GTILE (GB * GL32)  // doubles per staged operand tile (>= GK * GL64)

// A operand of a GEMM term read through its triangle (hlu_term.assoc of a GEMM
// term): HLU_TRI_NONE = A, HLU_TRI_UPPER = triu(A), HLU_TRI_UNIT_LOWER =
// tril(A, -1) + I (the stored factors of a dense diagonal leaf, hlu.py:720-767)
__device__ __forceinline__ double tri_get(const Mat &A, int i, int j, int tri) {
  if (tri == HLU_TRI_UPPER) return j >= i ? A.get(i, j) : 0.0;
  if (tri == HLU_TRI_UNIT_LOWER) return j < i ? A.get(i, j) : (j == i ? 1.0 : 0.0);
  return A.get(i, j);
}

// D = A(16x8, row) * B(8x8, col) + D, fp64 tensor core.  Fragments (lane =
// 4 g + t): a = {A[g][t], A[g+8][t], A[g][t+4], A[g+8][t+4]},
// b = {B[t][g], B[t+4][g]}, d = {D[g][2t], D[g][2t+1], D[g+8][2t], D[g+8][2t+1]}.
__device__ __forceinline__ void dmma16884(double (&d)[4], const double (&a)[4], const double (&b)[2]) {
  asm volatile(
      "mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};\n"
      : "+d"(d[0]), "+d"(d[1]), "+d"(d[2]), "+d"(d[3])
      : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(b[0]), "d"(b[1]));
}

// 8-byte global -> shared copy that bypasses the registers (LDGSTS);
// ok == false writes a zero (src-size 0: nothing is read).  Operands that
// already live in shared memory (the W block of a triple term) are copied
// with a plain load / store instead (cp.async takes global sources only).
__device__ __forceinline__ void cp_async8(double *sdst, const double *gsrc, bool ok, bool src_shared) {
  if (src_shared) {
    *sdst = ok ? *gsrc : 0.0;
    return;
  }
  const unsigned s = (unsigned)__cvta_generic_to_shared(sdst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gsrc), "r"(ok ? 8 : 0) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory"); }

// C += alpha * A B.  Double-buffered k-tiles: the next tile streams into the
// other shared buffers by cp.async while the tensor cores consume this one.
// sA / sB hold two GTILE buffers each.
//
// The operand geometry is copied into registers first: the Mats arrive by
// reference (they live in the caller's stack frame) and every cp.async is an
// asm with a memory clobber, so reading A.p / A.rs / ... inside the staging
// loop would reload them from local memory after each copy (measured: 2.6 k
// instructions and a local-load stall per copy for one 64^3 tile).  Element u
// of a thread's staging list sits at a fixed offset from element 0 (row or
// depth advances linearly with u), so the addresses are one base plus u
// strides, advanced by a constant per k-tile.
__device__ __noinline__ void tile_gemm(const Mat &C, const Mat &A, const Mat &B, double alpha, double *sA,
                                       double *sB, int tri = HLU_TRI_NONE) {
  const int m = C.rows, n = C.cols, k = A.cols;
  double *const Cp = C.p;
  const double *const Ap = A.p, *const Bp = B.p;
  // strides and element offsets of one operand fit 32 bits (an operand is a window of one leaf / temp)
  const int Crs = (int)C.rs, Ccs = (int)C.cs, Ars = (int)A.rs, Acs = (int)A.cs, Brs = (int)B.rs, Bcs = (int)B.cs;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int wm = (wid & 3) * 16, wn = (wid >> 2) * 32;
  // coalescing: walk each operand's unit-stride dimension fastest
  const bool a_rf = Ars == 1, b_rf = Brs == 1;
  const bool a_sh = __isShared(Ap), b_sh = __isShared(Bp);
  // element (row r, depth q) of the A tile / (depth q, col c) of the B tile
  const int am = a_rf ? 1 : GL32, ak = a_rf ? GL64 : 1;
  const int bk = b_rf ? 1 : GL64, bn = b_rf ? GL32 : 1;
  // staging list of this thread: element u = (row ar0 + u adr, depth aq0 + u adq) of A,
  // (depth bq0 + u bdq, col bc0 + u bdc) of B
  const int ar0 = a_rf ? tid % GB : tid / GK, aq0 = a_rf ? tid / GB : tid % GK;
  const int adr = a_rf ? 0 : HLU_NT / GK, adq = a_rf ? HLU_NT / GB : 0;
  const int bq0 = b_rf ? tid % GK : tid / GB, bc0 = b_rf ? tid / GK : tid % GB;
  const int bdq = b_rf ? 0 : HLU_NT / GB, bdc = b_rf ? HLU_NT / GK : 0;
  const int a_step = adr * Ars + adq * Acs, b_step = bdq * Brs + bdc * Bcs;
  const int ta_off = ar0 * am + aq0 * ak, ta_step = adr * am + adq * ak;
  const int tb_off = bq0 * bk + bc0 * bn, tb_step = bdq * bk + bdc * bn;
  if (m <= 0 || n <= 0 || k <= 0) {  // (callers skip empty products; uniform)
    __syncthreads();
    return;
  }
  const bool c_sh = __isShared(Cp);
  const int kz = (k + 7) & ~7;  // depths [k, kz) are read by the last 8-deep step: zero-filled
  // One software pipeline over all (output tile, k-tile) steps of the product,
  // row tiles outermost: while the tensor cores consume step s, the operands of
  // step s + 1 stream in, also across output tiles (tall skinny products -- an
  // Rk factor times a small core -- have one k-tile per output tile, so a
  // per-tile pipeline would expose the full load latency on every tile).
  const int total = ((m + GB - 1) / GB) * ((n + GB - 1) / GB) * ((k + GK - 1) / GK);
  auto next = [&](int &i, int &j, int &kk) {
    kk += GK;
    if (kk >= k) {
      kk = 0;
      j += GB;
      if (j >= n) j = 0, i += GB;
    }
  };
  auto issue = [&](int i0, int j0, int k0, int buf) {
    double *ta = sA + buf * GTILE + ta_off, *tb = sB + buf * GTILE + tb_off;
    const double *pa = Ap + ((i0 + ar0) * Ars + (k0 + aq0) * Acs);
    const double *pb = Bp + ((k0 + bq0) * Brs + (j0 + bc0) * Bcs);
    int ai = i0 + ar0, aq = k0 + aq0, bq = k0 + bq0, bj = j0 + bc0;
#pragma unroll 2
    for (int u = 0; u < GPF; ++u) {
      // rows of A past m and columns of B past n only feed accumulator entries that are
      // never stored: nothing is staged for them
      if (ai < m && aq < kz) cp_async8(ta, aq < k ? pa : Ap, aq < k, a_sh);
      if (bj < n && bq < kz) cp_async8(tb, bq < k ? pb : Bp, bq < k, b_sh);
      ta += ta_step, tb += tb_step, pa += a_step, pb += b_step;
      ai += adr, aq += adq, bq += bdq, bj += bdc;
    }
    cp_async_commit();
  };
  // triangular read of A (factor matvecs): fix this thread's staged elements
  auto mask = [&](int i0, int k0, int buf) {
    double *ta = sA + buf * GTILE + ta_off;
#pragma unroll
    for (int u = 0; u < GPF; ++u) {
      const int gi = i0 + ar0 + u * adr, gk = k0 + aq0 + u * adq;
      if (gi < m && gk < k) {
        double &x = ta[u * ta_step];
        if (tri == HLU_TRI_UPPER && gk < gi) x = 0.0;
        if (tri == HLU_TRI_UNIT_LOWER && gk >= gi) x = gk == gi ? 1.0 : 0.0;
      }
    }
  };
  int i0 = 0, j0 = 0, k0 = 0, nf = 0;
  double acc[4][4];
  issue(0, 0, 0, 0);
  for (int s = 0, buf = 0; s < total; ++s, buf ^= 1) {
    int ni = i0, nj = j0, nk = k0;
    next(ni, nj, nk);
    if (s + 1 < total) {
      issue(ni, nj, nk, buf ^ 1);  // the other buffer was released by the barrier below
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    if (k0 == 0) {  // a new output tile
#pragma unroll
      for (int f = 0; f < 4; ++f)
#pragma unroll
        for (int v = 0; v < 4; ++v) acc[f][v] = 0.0;
      // fragments of this warp inside C (warp-uniform): 0 when its rows or columns lie outside
      nf = (i0 + wm < m) ? max(0, min(4, (n - j0 - wn + 7) >> 3)) : 0;
      if (!c_sh && nf > 0) {
        // the epilogue's read-modify-write of C: pull the lines towards the SM now
        const double *c0 = Cp + ((i0 + wm + g) * Crs + (j0 + wn + 2 * t) * Ccs);
#pragma unroll
        for (int f = 0; f < 4; ++f) {
          if (f < nf) {
#pragma unroll
            for (int v = 0; v < 4; ++v) {
              const int gi = i0 + wm + g + 8 * (v >> 1), gj = j0 + wn + f * 8 + 2 * t + (v & 1);
              if (gi < m && gj < n)
                asm volatile("prefetch.global.L1 [%0];" ::"l"(c0 + (8 * (v >> 1) * Crs + (f * 8 + (v & 1)) * Ccs)));
            }
          }
        }
      }
    }
    if (tri != HLU_TRI_NONE) mask(i0, k0, buf);
    __syncthreads();
    {
      const double *ta = sA + buf * GTILE, *tb = sB + buf * GTILE;
      // skinny tiles (Rk factors: a handful of columns): a warp runs only the
      // 8-column fragments and the 16-row strip that reach into C
      const int ksteps = nf > 0 ? (min(GK, k - k0) + 7) >> 3 : 0;  // zero-padded past k
      for (int q = 0; q < ksteps; ++q) {
        const int q0 = q * 8 + t;
        double af[4];
        af[0] = ta[(wm + g) * am + q0 * ak];
        af[1] = ta[(wm + g + 8) * am + q0 * ak];
        af[2] = ta[(wm + g) * am + (q0 + 4) * ak];
        af[3] = ta[(wm + g + 8) * am + (q0 + 4) * ak];
#pragma unroll
        for (int f = 0; f < 4; ++f) {
          if (f < nf) {
            const int c = wn + f * 8 + g;
            double bf[2];
            bf[0] = tb[q0 * bk + c * bn];
            bf[1] = tb[(q0 + 4) * bk + c * bn];
            dmma16884(acc[f], af, bf);
          }
        }
      }
    }
    __syncthreads();
    if (k0 + GK >= k && nf > 0) {  // last k-tile of this output tile
      double *const c_base = Cp + ((i0 + wm + g) * Crs + (j0 + wn + 2 * t) * Ccs);
#pragma unroll
      for (int f = 0; f < 4; ++f) {
        if (f < nf) {
#pragma unroll
          for (int v = 0; v < 4; ++v) {
            const int gi = i0 + wm + g + 8 * (v >> 1), gj = j0 + wn + f * 8 + 2 * t + (v & 1);
            if (gi < m && gj < n) c_base[8 * (v >> 1) * Crs + (f * 8 + (v & 1)) * Ccs] += alpha * acc[f][v];
          }
        }
      }
    }
    i0 = ni, j0 = nj, k0 = nk;
  }
  __syncthreads();  // C may be a shared block the next call reads
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

// ---------------------------------------------------------------------------
// GETRF: in-place unpivoted LU, right-looking with 8-column panels; the
// trailing updates A22 -= L21 U12 run on the fp64 tensor cores (one
// m16n8k8 DMMA per 16 x 8 tile and panel).  n <= 128: the whole block in
// shared memory; n > 128 (HODLR leaves): 64-blocked in place in HBM, the
// diagonal blocks through the shared-memory kernel, L21 / U12 by the
// shared-memory triangular solves and A22 by tile_gemm.
// Pivot test |p| <= 1e-12 * max|A_input| over the whole block, as
// lowrank.py:194-212; the first failing op (program order) is reported
// through ctx.err[1].
// ---------------------------------------------------------------------------
#define LU_PW 8      // panel width
#define SMALL_N 128  // largest block held whole in shared memory
#define BLK 64       // block edge of the n > SMALL_N paths

__host__ __device__ __forceinline__ int lu_npad(int n) { return (n + 15) & ~15; }
// The DMMA tiles of a panel step start at row / column j1 (a multiple of 8)
// and run in 16-row x 8-column steps, so they reach up to row npad + 15 and
// column npad + 7: the shared tile is (npad + 16) rows (ld npad + 20, which
// keeps the fragment loads bank-conflict free) by npad + 8 columns, zero
// outside the block.
__host__ __device__ __forceinline__ int lu_ld(int n) { return lu_npad(n) + 20; }
__host__ __device__ __forceinline__ int lu_cols(int n) { return lu_npad(n) + 8; }
__host__ __device__ __forceinline__ size_t lu_smem_doubles(int n) { return (size_t)lu_ld(n) * lu_cols(n); }

// LU of the n x n block in shared memory (column-major, ld, zero padding);
// returns the first column whose pivot fails the test (its value in *piv), or -1
__device__ int lu_shared(double *sm, int ld, int n, double tol, double *piv) {
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int npad = lu_npad(n);
  for (int j0 = 0; j0 < n; j0 += LU_PW) {
    const int j1 = min(j0 + LU_PW, n);
    // panel: rank-1 steps on columns j0 .. j1-1 (all rows below the diagonal)
    for (int j = j0; j < j1; ++j) {
      const double p = sm[j + j * ld];
      if (fabs(p) <= tol) {
        if (tid == 0) *piv = p;
        __syncthreads();
        return j;  // p is read from shared memory by every thread: uniform exit
      }
      for (int i = j + 1 + tid; i < n; i += HLU_NT) sm[i + j * ld] /= p;
      __syncthreads();
      // rank-1 update of the panel's remaining columns (< 8: one warp each), lanes over rows
      for (int l = j + 1 + wid; l < j1; l += HLU_NWARP) {
        const double ujl = sm[j + l * ld];
        for (int i = j + 1 + lane; i < n; i += 32) sm[i + l * ld] -= sm[i + j * ld] * ujl;
      }
      __syncthreads();
    }
    if (j1 >= n) break;
    // U12 = L11^-1 A12: rows j0 .. j1-1 of the trailing columns, one column per thread
    for (int col = j1 + tid; col < n; col += HLU_NT) {
      double u[LU_PW];
#pragma unroll
      for (int r = 0; r < LU_PW; ++r) u[r] = (j0 + r < j1) ? sm[j0 + r + col * ld] : 0.0;
#pragma unroll
      for (int r = 1; r < LU_PW; ++r)
#pragma unroll
        for (int q = 0; q < r; ++q) u[r] -= sm[j0 + r + (j0 + q) * ld] * u[q];
#pragma unroll
      for (int r = 1; r < LU_PW; ++r)
        if (j0 + r < j1) sm[j0 + r + col * ld] = u[r];
    }
    __syncthreads();
    // A22 -= L21 U12: 16 x 8 tiles, one DMMA each (padding rows / columns are zero)
    const int tr = (npad - j1 + 15) >> 4, tc = (npad - j1 + 7) >> 3;
    for (int tile = wid; tile < tr * tc; tile += HLU_NWARP) {
      const int r0 = j1 + (tile % tr) * 16, c0 = j1 + (tile / tr) * 8;
      double a[4], b[2], d[4];
      a[0] = -sm[r0 + g + (j0 + t) * ld];
      a[1] = -sm[r0 + g + 8 + (j0 + t) * ld];
      a[2] = -sm[r0 + g + (j0 + t + 4) * ld];
      a[3] = -sm[r0 + g + 8 + (j0 + t + 4) * ld];
      b[0] = sm[j0 + t + (c0 + g) * ld];
      b[1] = sm[j0 + t + 4 + (c0 + g) * ld];
      d[0] = sm[r0 + g + (c0 + 2 * t) * ld];
      d[1] = sm[r0 + g + (c0 + 2 * t + 1) * ld];
      d[2] = sm[r0 + g + 8 + (c0 + 2 * t) * ld];
      d[3] = sm[r0 + g + 8 + (c0 + 2 * t + 1) * ld];
      dmma16884(d, a, b);
      sm[r0 + g + (c0 + 2 * t) * ld] = d[0];
      sm[r0 + g + (c0 + 2 * t + 1) * ld] = d[1];
      sm[r0 + g + 8 + (c0 + 2 * t) * ld] = d[2];
      sm[r0 + g + 8 + (c0 + 2 * t + 1) * ld] = d[3];
    }
    __syncthreads();
  }
  return -1;
}

// global block -> shared (column-major, ld), zero padding up to rows x cols
__device__ void load_padded(double *sm, int ld, int rows, int cols, const Mat &A) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int j = wid; j < cols; j += HLU_NWARP)
    for (int i = lane; i < rows; i += 32) sm[i + j * ld] = (i < A.rows && j < A.cols) ? A.get(i, j) : 0.0;
  __syncthreads();
}

__device__ void store_block(const double *sm, int ld, const Mat &A) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int j = wid; j < A.cols; j += HLU_NWARP)
    for (int i = lane; i < A.rows; i += 32) A.at(i, j) = sm[i + j * ld];
  __syncthreads();
}

// ---------------------------------------------------------------------------
// TRSM core (n <= SMALL_N): T in shared memory, right-hand sides in chunks of 64.
//   mode 0: X <- L^-1 X  (unit lower, X n x r)
//   mode 1: X <- X U^-1  (upper,      X r x n)
//   mode 2: X <- U^-1 X  (upper,      X n x r)
// Solve dimension index i, rhs index v; xs[i + v*ld].
// ---------------------------------------------------------------------------
#define TRSM_CHUNK 64
__host__ __device__ __forceinline__ size_t trsm_smem_doubles(int n) {
  return (size_t)n * (n + 1) + (size_t)(n + 1) * TRSM_CHUNK;
}

// Substitution with the right-hand sides in registers: warp w owns the columns
// v = w, w + 8, ... of the chunk (<= 8 of them), lane l the solve indices l,
// l + 32, ... (NQ per lane, n <= 32 NQ).  A column never leaves its warp, so the
// n elimination steps need no CTA barrier: the pivot element is broadcast by a
// shuffle and the coefficient column / row of T is read from shared memory once
// for all of the warp's columns (zero for the lanes a step does not touch, so
// the update is one unconditional DFMA).  Same operations per element, in the
// same order, as the textbook loops.
template <int NQ>
__device__ __forceinline__ void trsm_solve_regs(const double *ts, double *xs, int ld, int n, int nv, int mode) {
  constexpr int NC = TRSM_CHUNK / HLU_NWARP;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int ncol = nv > wid ? (nv - wid + HLU_NWARP - 1) / HLU_NWARP : 0;  // warp-uniform
  if (ncol == 0) return;
  double x[NC][NQ];
#pragma unroll
  for (int c = 0; c < NC; ++c)
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      const int i = lane + 32 * q;
      x[c][q] = (c < ncol && i < n) ? xs[i + (wid + HLU_NWARP * c) * ld] : 0.0;
    }
  if (mode == 0) {
#pragma unroll
    for (int q0 = 0; q0 < NQ; ++q0) {
      for (int jl = 0; jl < 32 && q0 * 32 + jl < n - 1; ++jl) {
        const int j = q0 * 32 + jl;
        double l[NQ];
#pragma unroll
        for (int q = 0; q < NQ; ++q) {
          const int i = lane + 32 * q;
          l[q] = (q >= q0 && i > j && i < n) ? ts[i + j * ld] : 0.0;
        }
#pragma unroll
        for (int c = 0; c < NC; ++c) {
          if (c < ncol) {
            const double xj = __shfl_sync(0xffffffffu, x[c][q0], jl);
#pragma unroll
            for (int q = 0; q < NQ; ++q)
              if (q >= q0) x[c][q] -= l[q] * xj;
          }
        }
      }
    }
  } else if (mode == 1) {
#pragma unroll
    for (int q0 = 0; q0 < NQ; ++q0) {
      for (int jl = 0; jl < 32 && q0 * 32 + jl < n; ++jl) {
        const int j = q0 * 32 + jl;
        const double ujj = ts[j + j * ld];
        double u[NQ];
#pragma unroll
        for (int q = 0; q < NQ; ++q) {
          const int i = lane + 32 * q;
          u[q] = (q >= q0 && i > j && i < n) ? ts[j + i * ld] : 0.0;
        }
#pragma unroll
        for (int c = 0; c < NC; ++c) {
          if (c < ncol) {
            const double xd = __shfl_sync(0xffffffffu, x[c][q0], jl) / ujj;
#pragma unroll
            for (int q = 0; q < NQ; ++q)
              if (q >= q0) x[c][q] -= xd * u[q];
            if (lane == jl) x[c][q0] = xd;
          }
        }
      }
    }
  } else {
#pragma unroll
    for (int q0 = NQ - 1; q0 >= 0; --q0) {
      for (int jl = min(31, n - 1 - q0 * 32); jl >= 0; --jl) {
        const int j = q0 * 32 + jl;
        const double ujj = ts[j + j * ld];
        double u[NQ];
#pragma unroll
        for (int q = 0; q < NQ; ++q) {
          const int i = lane + 32 * q;
          u[q] = (q <= q0 && i < j) ? ts[i + j * ld] : 0.0;
        }
#pragma unroll
        for (int c = 0; c < NC; ++c) {
          if (c < ncol) {
            const double xd = __shfl_sync(0xffffffffu, x[c][q0], jl) / ujj;
#pragma unroll
            for (int q = 0; q < NQ; ++q)
              if (q <= q0) x[c][q] -= u[q] * xd;
            if (lane == jl) x[c][q0] = xd;
          }
        }
      }
    }
  }
#pragma unroll
  for (int c = 0; c < NC; ++c)
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      const int i = lane + 32 * q;
      if (c < ncol && i < n) xs[i + (wid + HLU_NWARP * c) * ld] = x[c][q];
    }
}

__device__ void trsm_shared(double *sm, const Mat &T, const Mat &X, int mode) {
  const int n = T.rows;
  const int ld = n + 1;
  double *ts = sm;
  double *xs = sm + n * ld;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int nrhs = (mode == 1) ? X.rows : X.cols;
  // lanes walk the unit-stride dimension of the (column-major) operands
  for (int j = wid; j < n; j += HLU_NWARP)
    for (int i = lane; i < n; i += 32) ts[i + j * ld] = T.get(i, j);
  for (int v0 = 0; v0 < nrhs; v0 += TRSM_CHUNK) {
    const int nv = min(TRSM_CHUNK, nrhs - v0);
    __syncthreads();
    if (mode == 1) {
      for (int i = wid; i < n; i += HLU_NWARP)
        for (int v = lane; v < nv; v += 32) xs[i + v * ld] = X.get(v0 + v, i);
    } else {
      for (int v = wid; v < nv; v += HLU_NWARP)
        for (int i = lane; i < n; i += 32) xs[i + v * ld] = X.get(i, v0 + v);
    }
    __syncthreads();
    if (n <= 32) trsm_solve_regs<1>(ts, xs, ld, n, nv, mode);
    else if (n <= 64) trsm_solve_regs<2>(ts, xs, ld, n, nv, mode);
    else trsm_solve_regs<4>(ts, xs, ld, n, nv, mode);
    __syncthreads();
    if (mode == 1) {
      for (int i = wid; i < n; i += HLU_NWARP)
        for (int v = lane; v < nv; v += 32) X.at(v0 + v, i) = xs[i + v * ld];
    } else {
      for (int v = wid; v < nv; v += HLU_NWARP)
        for (int i = lane; i < n; i += 32) X.at(i, v0 + v) = xs[i + v * ld];
    }
  }
  __syncthreads();
}

// n > SMALL_N: 64-blocked substitution in place; off-diagonal block updates by
// tile_gemm (DMMA), diagonal blocks by trsm_shared.
__device__ void trsm_blocked(double *sm, const Mat &T, const Mat &X, int mode) {
  const int n = T.rows;
  const int nb = (n + BLK - 1) / BLK;
  double *sA = sm, *sB = sm + 2 * GTILE;
  for (int s = 0; s < nb; ++s) {
    const int bi = mode == 2 ? nb - 1 - s : s;
    const int i0 = bi * BLK, ni = min(BLK, n - i0), i1 = i0 + ni;
    if (mode == 0) {  // X_i -= L_i,<i X_<i ; X_i <- L_ii^-1 X_i
      const Mat Xi = sub(X, i0, 0, ni, X.cols);
      if (i0 > 0) tile_gemm(Xi, sub(T, i0, 0, ni, i0), sub(X, 0, 0, i0, X.cols), -1.0, sA, sB);
      __syncthreads();
      trsm_shared(sm, sub(T, i0, i0, ni, ni), Xi, 0);
    } else if (mode == 2) {  // X_i -= U_i,>i X_>i ; X_i <- U_ii^-1 X_i
      const Mat Xi = sub(X, i0, 0, ni, X.cols);
      if (i1 < n) tile_gemm(Xi, sub(T, i0, i1, ni, n - i1), sub(X, i1, 0, n - i1, X.cols), -1.0, sA, sB);
      __syncthreads();
      trsm_shared(sm, sub(T, i0, i0, ni, ni), Xi, 2);
    } else {  // X_:,j -= X_:,<j U_<j,j ; X_:,j <- X_:,j U_jj^-1
      const Mat Xj = sub(X, 0, i0, X.rows, ni);
      if (i0 > 0) tile_gemm(Xj, sub(X, 0, 0, X.rows, i0), sub(T, 0, i0, i0, ni), -1.0, sA, sB);
      __syncthreads();
      trsm_shared(sm, sub(T, i0, i0, ni, ni), Xj, 1);
    }
    __syncthreads();
  }
}

__global__ void __launch_bounds__(HLU_NT, 2) k_getrf(hlu_ctx c, const hlu_getrf_desc *__restrict__ d) {
  extern __shared__ double sm[];
  __shared__ double red[HLU_NWARP];
  __shared__ double s_piv;
  const hlu_getrf_desc o = d[blockIdx.x];
  const Mat A = resolve(c, o.a);
  const int n = A.rows;
  double mx = 0.0;
  for (int e = threadIdx.x; e < n * n; e += HLU_NT) mx = fmax(mx, fabs(A.get(e % n, e / n)));
  const double tol = 1e-12 * block_max(mx, red);  // includes a __syncthreads
  int bad = -1;
  if (n <= SMALL_N) {
    const int ld = lu_ld(n);
    load_padded(sm, ld, ld, lu_cols(n), A);
    bad = lu_shared(sm, ld, n, tol, &s_piv);
    if (bad < 0) store_block(sm, ld, A);
  } else {
    // 64-blocked right-looking LU in place: A11 = L11 U11 (shared memory),
    // A21 <- A21 U11^-1, A12 <- L11^-1 A12, A22 -= A21 A12 (DMMA)
    for (int k0 = 0; k0 < n; k0 += BLK) {
      const int nk = min(BLK, n - k0), k1 = k0 + nk;
      const Mat A11 = sub(A, k0, k0, nk, nk);
      const int ld = lu_ld(nk);
      load_padded(sm, ld, ld, lu_cols(nk), A11);
      bad = lu_shared(sm, ld, nk, tol, &s_piv);
      if (bad >= 0) break;
      store_block(sm, ld, A11);
      if (k1 < n) {
        trsm_shared(sm, A11, sub(A, k1, k0, n - k1, nk), 1);
        trsm_shared(sm, A11, sub(A, k0, k1, nk, n - k1), 0);
        tile_gemm(sub(A, k1, k1, n - k1, n - k1), sub(A, k1, k0, n - k1, nk), sub(A, k0, k1, nk, n - k1), -1.0,
                  sm, sm + 2 * GTILE);
        __syncthreads();
      }
    }
  }
  if (bad >= 0 && threadIdx.x == 0) {
    atomicMin(&c.err[1], o.op_id);
    c.dlog[2 * o.lu_index] = s_piv;
    c.dlog[2 * o.lu_index + 1] = tol;
  }
}

__global__ void __launch_bounds__(HLU_NT, 2) k_trsm(hlu_ctx c, const hlu_trsm_desc *__restrict__ d) {
  extern __shared__ double sm[];
  const hlu_trsm_desc o = d[blockIdx.x];
  const Mat T = resolve(c, o.t);
  const Mat X = resolve(c, o.x);
  if (o.log >= 0 && threadIdx.x == 0) c.log[o.log] = (o.mode == 1) ? X.rows : X.cols;
  if (T.rows <= SMALL_N) trsm_shared(sm, T, X, o.mode);
  else trsm_blocked(sm, T, X, o.mode);
}

__global__ void __launch_bounds__(HLU_NT, 2)
    k_gemm(hlu_ctx c, const hlu_gemm_desc *__restrict__ d, const hlu_term *__restrict__ terms) {
  extern __shared__ double gsm[];
  double *sA = gsm;             // two k-tile buffers
  double *sB = sA + 2 * GTILE;  // two k-tile buffers
  double *sW = sB + 2 * GTILE;
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

// dynamic shared memory (bytes) of the LU / TRSM kernels for blocks up to n
static size_t getrf_smem(int n) {
  if (n <= SMALL_N) return lu_smem_doubles(n) * sizeof(double);
  const size_t d = std::max(std::max(lu_smem_doubles(BLK), trsm_smem_doubles(BLK)), (size_t)4 * GTILE);
  return d * sizeof(double);
}
static size_t trsm_smem(int n) {
  if (n <= SMALL_N) return trsm_smem_doubles(n) * sizeof(double);
  return std::max(trsm_smem_doubles(BLK), (size_t)4 * GTILE) * sizeof(double);
}
#define DENSE_NMAX 256  // largest dense leaf of the LU / TRSM kernels

extern "C" int hlu_getrf_batched_f64(const hlu_ctx *ctx, const hlu_getrf_desc *d, int count, int max_n,
                                     void *stream) {
  static unsigned long long init = 0ull;
  if (first_on_device(init)) {
    cudaFuncSetAttribute(k_getrf, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)std::max(getrf_smem(SMALL_N), getrf_smem(DENSE_NMAX)));
  }
  if (max_n > DENSE_NMAX) return -2;
  if (count <= 0) return 0;
  k_getrf<<<count, HLU_NT, getrf_smem(max_n), (cudaStream_t)stream>>>(*ctx, d);
  return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

extern "C" int hlu_trsm_batched_f64(const hlu_ctx *ctx, const hlu_trsm_desc *d, int count, int max_n,
                                    void *stream) {
  static unsigned long long init = 0ull;
  if (first_on_device(init)) {
    cudaFuncSetAttribute(k_trsm, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)std::max(trsm_smem(SMALL_N), trsm_smem(DENSE_NMAX)));
  }
  if (max_n > DENSE_NMAX) return -2;
  if (count <= 0) return 0;
  k_trsm<<<count, HLU_NT, trsm_smem(max_n), (cudaStream_t)stream>>>(*ctx, d);
  return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

extern "C" int hlu_gemm_batched_f64(const hlu_ctx *ctx, const hlu_gemm_desc *d, const hlu_term *terms,
                                    int count, void *stream) {
  const size_t smem = (size_t)(4 * GTILE + GB * GB) * sizeof(double);
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
