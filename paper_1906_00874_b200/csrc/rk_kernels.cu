// Batched Rk truncation: add_truncated / recompress / compress_dense.
//
// Reference semantics (lowrank.py:127-175, Appendix A of SURVEY.md):
//   ADD mode: k2 == 0 -> x1; k1 == 0 -> x2 (untruncated); otherwise the
//             truncated SVD of x1 + x2.  (The reference forms the dense sum
//             when k1+k2 >= min(m,n)/2 and SVDs it; mathematically the same
//             truncated SVD, computed here from the factors.)
//   RECOMPRESS: k == 0 -> unchanged; otherwise the truncated SVD of the
//             concatenation of all parts (also compress_dense(A @ B) given
//             as the single part (A, B^T)).
//   truncation: k = #{sigma_i > eps*sigma_1} (0 if sigma_1 == 0), min(k, kmax),
//             Sigma folded into the left factor.
//
// One CTA per truncation:
//   A. TSQR of X = [parts.a] (m x K) over row chunks held in shared memory
//      (Householder, dlarfg conventions); reflectors of every chunk go to a
//      per-op workspace in the pool.
//   B. the same for Y = [parts.b] (n x K).
//   C. core M = R_a R_b^T (<= K x K).
//   D. one-sided (Hestenes) Jacobi SVD of M (or M^T), round-robin pairs,
//      one warp per pair, warp-shuffle reductions.
//   E. descending sort, rank count (strict >), kmax cap.
//   F. A' = Q_a [U_k S_k; 0], B' = Q_b [V_k; 0] by applying the stored
//      reflectors chunk by chunk in reverse; one warp per output column.
#include "common.cuh"

namespace hlu {

template <int KM>
struct RkCfg {
  static constexpr int BUFD = (KM == 32) ? 4608 : 9216;  // chunk buffer (doubles)
  static constexpr int LDS = BUFD / KM;                  // leading dim of the chunk buffer
  static constexpr int CH = LDS - KM;                    // fresh rows per chunk
};

#define RK_MAXP 8

__host__ __device__ inline int64_t rk_ws_one(int m, int K, int CH) {
  if (m <= 0 || K <= 0) return 0;
  const int64_t nch = (m + CH - 1) / CH;
  return nch * ((int64_t)(K + CH) * K + K);
}

struct PartInfo {
  Mat a, b;
  double sign;
  int roff, coff, k, col0;
};

// Column j of the stacked factor (X if left, Y otherwise), global row gi.
__device__ __forceinline__ double stacked(const PartInfo *P, int np, bool left, int gi, int j) {
  int p = 0;
  while (p + 1 < np && j >= P[p + 1].col0) ++p;
  const PartInfo &q = P[p];
  const int jj = j - q.col0;
  if (left) {
    const int r = gi - q.roff;
    return (r >= 0 && r < q.a.rows) ? q.sign * q.a.get(r, jj) : 0.0;
  }
  const int r = gi - q.coff;
  return (r >= 0 && r < q.b.rows) ? q.b.get(r, jj) : 0.0;
}

// Householder QR of S (rows x K, ld LDS) in place; tau[K].  dlarfg conventions.
template <int KM>
__device__ void house_qr(double *S, int rows, int K, double *tau) {
  constexpr int LDS = RkCfg<KM>::LDS;
  const int tid = threadIdx.x, w = tid >> 5, l = tid & 31;
  __shared__ double s_tau, s_beta;
  const int t = min(rows, K);
  for (int j = 0; j < t; ++j) {
    if (w == 0) {
      double ss = 0.0;
      for (int i = j + 1 + l; i < rows; i += 32) {
        const double v = S[i + j * LDS];
        ss += v * v;
      }
      ss = warp_sum(ss);
      const double alpha = S[j + j * LDS];
      double tj = 0.0, beta = alpha;
      if (ss != 0.0) {
        beta = -copysign(sqrt(alpha * alpha + ss), alpha);
        tj = (beta - alpha) / beta;
        const double sc = 1.0 / (alpha - beta);
        for (int i = j + 1 + l; i < rows; i += 32) S[i + j * LDS] *= sc;
      }
      if (l == 0) {
        s_tau = tj;
        s_beta = beta;
        tau[j] = tj;
      }
    }
    __syncthreads();
    const double tj = s_tau;
    if (tj != 0.0) {
      for (int col = j + 1 + w; col < K; col += HLU_NWARP) {
        double acc = 0.0;
        for (int i = j + 1 + l; i < rows; i += 32) acc += S[i + j * LDS] * S[i + col * LDS];
        acc = warp_sum(acc) + S[j + col * LDS];
        const double f = tj * acc;
        for (int i = j + 1 + l; i < rows; i += 32) S[i + col * LDS] -= f * S[i + j * LDS];
        if (l == 0) S[j + col * LDS] -= f;
      }
    }
    if (tid == 0) S[j + j * LDS] = s_beta;
    __syncthreads();
  }
}

// TSQR of one stacked factor.  R (rr x K, ld KM, zero below the diagonal) -> R.
template <int KM>
__device__ int tsqr(const PartInfo *P, int np, bool left, int m, int K, double *S, double *R, double *tau,
                    double *ws) {
  constexpr int LDS = RkCfg<KM>::LDS, CH = RkCfg<KM>::CH;
  const int tid = threadIdx.x;
  int r = 0;  // carried R rows at the top of S
  int64_t off = 0;
  for (int r0 = 0; r0 < m; r0 += CH) {
    const int cnt = min(CH, m - r0);
    const int rows = r + cnt;
    for (int e = tid; e < cnt * K; e += HLU_NT) {
      const int i = e % cnt, j = e / cnt;
      S[r + i + j * LDS] = stacked(P, np, left, r0 + i, j);
    }
    __syncthreads();
    house_qr<KM>(S, rows, K, tau);
    // save the chunk's compact QR (ld = rows) and tau
    double *dst = ws + off;
    for (int e = tid; e < rows * K; e += HLU_NT) {
      const int i = e % rows, j = e / rows;
      dst[i + (int64_t)j * rows] = S[i + j * LDS];
    }
    for (int j = tid; j < K; j += HLU_NT) dst[(int64_t)rows * K + j] = (j < min(rows, K)) ? tau[j] : 0.0;
    off += (int64_t)rows * K + K;
    r = min(rows, K);
    __syncthreads();
    // keep R on top, clear the reflector entries below its diagonal
    for (int e = tid; e < r * K; e += HLU_NT) {
      const int i = e % r, j = e / r;
      if (i > j) S[i + j * LDS] = 0.0;
    }
    __syncthreads();
  }
  for (int e = tid; e < KM * K; e += HLU_NT) {
    const int i = e % KM, j = e / KM;
    R[i + j * KM] = (i < r && i <= j) ? S[i + j * LDS] : 0.0;
  }
  __syncthreads();
  return r;
}

// out (m x kk, ld m) = Q [W (rr x kk, ld KM); 0], Q from the stored chunks.
template <int KM>
__device__ void apply_q(int m, int K, int kk, const double *W, double *T, const double *ws, double *out) {
  constexpr int LDS = RkCfg<KM>::LDS, CH = RkCfg<KM>::CH;
  const int tid = threadIdx.x, w = tid >> 5, l = tid & 31;
  const int nch = (m + CH - 1) / CH;
  // chunk geometry: rows_s = r_{s-1} + cnt_s, r_s = min(rows_s, K); offsets are prefix sums
  int64_t off_last = 0;
  int rprev_last = 0;
  {
    int r = 0;
    int64_t off = 0;
    for (int s = 0; s < nch; ++s) {
      const int cnt = min(CH, m - s * CH);
      const int rows = r + cnt;
      if (s == nch - 1) {
        off_last = off;
        rprev_last = r;
      }
      off += (int64_t)rows * K + K;
      r = min(rows, K);
    }
    // top of T = W (r_last rows)
    for (int e = tid; e < r * kk; e += HLU_NT) {
      const int i = e % r, j = e / r;
      T[i + j * LDS] = W[i + j * KM];
    }
  }
  int64_t off = off_last;
  int rprev = rprev_last;
  for (int s = nch - 1; s >= 0; --s) {
    const int cnt = min(CH, m - s * CH);
    const int rows = rprev + cnt;
    const int rs = min(rows, K);
    __syncthreads();
    for (int e = tid; e < (rows - rs) * kk; e += HLU_NT) {
      const int i = rs + e % (rows - rs), j = e / (rows - rs);
      T[i + j * LDS] = 0.0;
    }
    __syncthreads();
    const double *V = ws + off;
    const double *tau = V + (int64_t)rows * K;
    // columns are independent: one warp per column runs all reflectors
    for (int col = w; col < kk; col += HLU_NWARP) {
      double *t = T + col * LDS;
      for (int j = rs - 1; j >= 0; --j) {
        const double tj = tau[j];
        if (tj == 0.0) continue;
        double acc = 0.0;
        for (int i = j + 1 + l; i < rows; i += 32) acc += V[i + (int64_t)j * rows] * t[i];
        acc = warp_sum(acc) + t[j];
        const double f = tj * acc;
        for (int i = j + 1 + l; i < rows; i += 32) t[i] -= f * V[i + (int64_t)j * rows];
        __syncwarp();
        if (l == 0) t[j] -= f;
        __syncwarp();
      }
    }
    __syncthreads();
    for (int e = tid; e < cnt * kk; e += HLU_NT) {
      const int i = e % cnt, j = e / cnt;
      out[(int64_t)s * CH + i + (int64_t)j * m] = T[rprev + i + j * LDS];
    }
    // step back: previous chunk's geometry
    if (s > 0) {
      int r = 0;
      int64_t o2 = 0, o_prev = 0;
      int rp_prev = 0;
      for (int u = 0; u < s; ++u) {
        const int c2 = min(CH, m - u * CH);
        const int rows2 = r + c2;
        if (u == s - 1) {
          o_prev = o2;
          rp_prev = r;
        }
        o2 += (int64_t)rows2 * K + K;
        r = min(rows2, K);
      }
      off = o_prev;
      rprev = rp_prev;
    }
  }
  __syncthreads();
}

__device__ unsigned long long g_sweeps = 0;  // total Jacobi sweeps (diagnostics)

__device__ __forceinline__ int rr_player(int pos, int r, int qq) {
  return pos == 0 ? 0 : 1 + (pos - 1 + r) % (qq - 1);
}

// One-sided Jacobi on G (p x q, ld KM) accumulating V (q x q, ld KM).
template <int KM>
__device__ void jacobi(double *G, double *V, int p, int q) {
  const int tid = threadIdx.x, w = tid >> 5, l = tid & 31;
  __shared__ int s_rot;
  for (int e = tid; e < KM * KM; e += HLU_NT) V[e] = ((e % KM) == (e / KM)) ? 1.0 : 0.0;
  const int qq = q + (q & 1);
  const double tol = 1e-15;
  if (q < 2) {
    __syncthreads();
    return;
  }
  for (int sweep = 0; sweep < 60; ++sweep) {
    if (tid == 0) s_rot = 0;
    __syncthreads();
    for (int r = 0; r < qq - 1; ++r) {
      for (int pi = w; pi < qq / 2; pi += HLU_NWARP) {
        int a = rr_player(pi, r, qq), b = rr_player(qq - 1 - pi, r, qq);
        if (a >= q || b >= q) continue;
        if (a > b) { const int x = a; a = b; b = x; }
        double al = 0.0, be = 0.0, ga = 0.0;
        for (int i = l; i < p; i += 32) {
          const double x = G[i + a * KM], y = G[i + b * KM];
          al += x * x;
          be += y * y;
          ga += x * y;
        }
        al = warp_sum(al);
        be = warp_sum(be);
        ga = warp_sum(ga);
        if (ga == 0.0 || !(fabs(ga) > tol * sqrt(al * be))) continue;
        const double zeta = (be - al) / (2.0 * ga);
        const double t = copysign(1.0, zeta) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
        const double cs = 1.0 / sqrt(1.0 + t * t), sn = cs * t;
        for (int i = l; i < p; i += 32) {
          const double x = G[i + a * KM], y = G[i + b * KM];
          G[i + a * KM] = cs * x - sn * y;
          G[i + b * KM] = sn * x + cs * y;
        }
        for (int i = l; i < q; i += 32) {
          const double x = V[i + a * KM], y = V[i + b * KM];
          V[i + a * KM] = cs * x - sn * y;
          V[i + b * KM] = sn * x + cs * y;
        }
        if (l == 0) s_rot = 1;
      }
      __syncthreads();
    }
    if (s_rot == 0) {
      if (tid == 0) atomicAdd(&g_sweeps, sweep + 1);
      break;
    }
    __syncthreads();
  }
  __syncthreads();
}

template <int KM>
__global__ void __launch_bounds__(HLU_NT)
    k_rkt(hlu_ctx c, hlu_rkt_desc *__restrict__ d, const hlu_rkpart *__restrict__ parts) {
  using Cfg = RkCfg<KM>;
  extern __shared__ double sm[];
  double *S = sm;                 // BUFD
  double *RA = S + Cfg::BUFD;     // KM*KM
  double *RB = RA + KM * KM;      // KM*KM
  double *tau = RB + KM * KM;     // KM
  double *sig = tau + KM;         // KM
  __shared__ PartInfo P[RK_MAXP];
  __shared__ int perm[KM];
  __shared__ int s_kk;
  const hlu_rkt_desc o = d[blockIdx.x];
  const int tid = threadIdx.x;
  const int np = o.part_count;
  if (tid == 0) {
    int col = 0;
    for (int p = 0; p < np && p < RK_MAXP; ++p) {
      const hlu_rkpart q = parts[o.part_begin + p];
      P[p].a = resolve(c, q.a);
      P[p].b = resolve(c, q.b);
      P[p].sign = q.sign;
      P[p].roff = q.roff;
      P[p].coff = q.coff;
      P[p].k = P[p].a.cols;
      P[p].col0 = col;
      col += P[p].k;
    }
  }
  __syncthreads();
  int K = 0;
  for (int p = 0; p < np; ++p) K += P[p].k;
  const int m = o.m, n = o.n;
  double *outA = c.pool + o.out_a;
  double *outB = c.pool + o.out_b;

  // Variant hand-off.  Both variants are launched over the same level; the
  // KM=32 one decides from the INPUT ranks (the KM=64 launch would see ranks
  // the KM=32 launch already updated) and flags the ops it leaves behind.
  if (KM == 32) {
    if (K > 32) {
      if (tid == 0) d[blockIdx.x].handoff = 64;
      return;
    }
  } else {
    if (o.handoff != 64) return;
    __syncthreads();
    if (tid == 0) d[blockIdx.x].handoff = 0;
  }
  if (o.mode == HLU_RK_ADD) {
    const int k1 = P[0].k, k2 = P[1].k;
    if (tid == 0 && o.log >= 0) {
      c.log[o.log] = k1;
      c.log[o.log + 1] = k2;
    }
    if (k2 == 0 || k1 == 0) {
      const PartInfo &src = (k2 == 0) ? P[0] : P[1];
      int kk = src.k;
      if (kk > o.cap) {
        if (tid == 0) atomicAdd(&c.err[0], 1);
        kk = o.cap;
      }
      const bool alias = (src.a.p == outA && src.a.rs == 1 && src.a.cs == m && src.b.p == outB &&
                          src.b.rs == 1 && src.b.cs == n && src.sign == 1.0);
      if (!alias) {
        for (int e = tid; e < m * kk; e += HLU_NT) outA[e] = src.sign * src.a.get(e % m, e / m);
        for (int e = tid; e < n * kk; e += HLU_NT) outB[e] = src.b.get(e % n, e / n);
      }
      if (tid == 0) {
        c.ranks[o.out_slot] = kk;
        if (o.log >= 0) c.log[o.log + 2] = kk;
      }
      return;
    }
  } else {
    if (tid == 0 && o.log >= 0) {
      c.log[o.log] = K;
      c.log[o.log + 1] = 0;
    }
    if (K == 0) {
      if (tid == 0) {
        c.ranks[o.out_slot] = 0;
        if (o.log >= 0) c.log[o.log + 2] = 0;
      }
      return;
    }
  }
  if (K > KM) {  // only reachable in the KM=64 variant
    if (tid == 0) atomicAdd(&c.err[2], 1);
    return;
  }
  double *wsA = c.pool + o.ws;
  double *wsB = wsA + rk_ws_one(m, K, Cfg::CH);
  // A/B. TSQR of both stacked factors
  const int ra = tsqr<KM>(P, np, true, m, K, S, RA, tau, wsA);
  const int rb = tsqr<KM>(P, np, false, n, K, S, RB, tau, wsB);
  // C. core M = R_a R_b^T (ra x rb); G = M or M^T so that G has q <= p columns
  const bool tr = rb > ra;
  const int p = tr ? rb : ra, q = tr ? ra : rb;
  double *G = S;
  double *V = S + KM * KM;
  for (int e = tid; e < ra * rb; e += HLU_NT) {
    const int i = e % ra, j = e / ra;
    double acc = 0.0;
    for (int t = max(i, j); t < K; ++t) acc += RA[i + t * KM] * RB[j + t * KM];
    // R_a[i,t] = 0 for t < i and R_b[j,t] = 0 for t < j
    if (tr) G[j + i * KM] = acc;
    else G[i + j * KM] = acc;
  }
  __syncthreads();
  // D. SVD
  jacobi<KM>(G, V, p, q);
  // E. singular values, order, rank
  for (int j = tid; j < q; j += HLU_NT) {
    double ss = 0.0;
    for (int i = 0; i < p; ++i) ss += G[i + j * KM] * G[i + j * KM];
    sig[j] = sqrt(ss);
  }
  __syncthreads();
  for (int j = tid; j < q; j += HLU_NT) {
    int rk = 0;
    const double sj = sig[j];
    for (int i = 0; i < q; ++i) rk += (sig[i] > sj) || (sig[i] == sj && i < j);
    perm[rk] = j;
  }
  __syncthreads();
  if (tid == 0) {
    const double s1 = sig[perm[0]];
    int kk = 0;
    if (s1 != 0.0) {
      const double thr = c.eps * s1;
      for (int i = 0; i < q; ++i) kk += sig[i] > thr;
    }
    if (c.kmax >= 0) kk = min(kk, c.kmax);
    if (kk > o.cap) {
      atomicAdd(&c.err[0], 1);
      kk = o.cap;
    }
    s_kk = kk;
  }
  __syncthreads();
  const int kk = s_kk;
  // F. W_a (ra x kk) -> RA, W_b (rb x kk) -> RB
  for (int e = tid; e < KM * kk; e += HLU_NT) {
    const int i = e % KM, cidx = e / KM;
    const int j = perm[cidx];
    double wa = 0.0, wb = 0.0;
    if (!tr) {
      if (i < ra) wa = G[i + j * KM];
      if (i < rb) wb = V[i + j * KM];
    } else {
      if (i < ra) wa = V[i + j * KM] * sig[j];
      if (i < rb) wb = G[i + j * KM] / sig[j];
    }
    RA[i + cidx * KM] = wa;
    RB[i + cidx * KM] = wb;
  }
  __syncthreads();
  apply_q<KM>(m, K, kk, RA, S, wsA, outA);
  apply_q<KM>(n, K, kk, RB, S, wsB, outB);
  if (tid == 0) {
    c.ranks[o.out_slot] = kk;
    if (o.log >= 0) c.log[o.log + 2] = kk;
  }
}

template <int KM>
static size_t rkt_smem() {
  return (size_t)(RkCfg<KM>::BUFD + 2 * KM * KM + 2 * KM) * sizeof(double);
}

}  // namespace hlu

using namespace hlu;

extern "C" int64_t hlu_debug_sweeps(int reset) {
  unsigned long long v = 0;
  cudaMemcpyFromSymbol(&v, g_sweeps, sizeof(v));
  if (reset) {
    unsigned long long z = 0;
    cudaMemcpyToSymbol(g_sweeps, &z, sizeof(z));
  }
  return (int64_t)v;
}

extern "C" int64_t hlu_rkt_ws_doubles(int32_t m, int32_t kbound) {
  // the variant that runs an op depends on its runtime K; take the larger need
  const int k32 = kbound < 32 ? kbound : 32;
  const int k64 = kbound < 64 ? kbound : 64;
  const int64_t a = rk_ws_one(m, k32, RkCfg<32>::CH);
  const int64_t b = rk_ws_one(m, k64, RkCfg<64>::CH);
  return a > b ? a : b;
}

extern "C" int hlu_rk_update_batched_f64(const hlu_ctx *ctx, hlu_rkt_desc *d, const hlu_rkpart *parts,
                                         int count, int kclass, void *stream) {
  static bool init = false;
  if (!init) {
    cudaFuncSetAttribute(k_rkt<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)rkt_smem<32>());
    cudaFuncSetAttribute(k_rkt<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)rkt_smem<64>());
    init = true;
  }
  if (count <= 0) return 0;
  if (kclass == 32)
    k_rkt<32><<<count, HLU_NT, rkt_smem<32>(), (cudaStream_t)stream>>>(*ctx, d, parts);
  else
    k_rkt<64><<<count, HLU_NT, rkt_smem<64>(), (cudaStream_t)stream>>>(*ctx, d, parts);
  return cudaGetLastError() == cudaSuccess ? 0 : -1;
}
