/*
 * rk_layout.h — workspace geometry of the batched Rk truncation (shared by the
 * CUDA kernels, the native planner and, mirrored, ir.py).
 *
 * A truncation of the stacked factors X (m x K) and Y (n x K) runs in three
 * phases (rk_kernels.cu):
 *   A. every factor is cut into row blocks of RK_BR rows; each block is
 *      QR-factorised by one CTA as a chain of chunks of `ch` rows (Householder,
 *      the previous chunk's R carried on top), reflectors -> workspace;
 *   B. per op: the blocks' R factors are stacked and QR-factorised again
 *      (only when a factor has > 1 block), then the small core SVD, the rank
 *      decision and W = the kept singular vectors in the R bases, which the
 *      combine-level reflectors turn into one coefficient block Z_b per block;
 *   C. every block applies its own reflectors to [Z_b; 0] -> output rows.
 *
 * Per factor side (M rows, runtime stacked rank K <= RK_KMAX) the workspace is
 *   [block chains | block R (K x K each) | combine chain | Z (zrows x K)].
 * Offsets depend on the runtime K; the planner reserves the maximum over
 * K <= kbound (rk_ws_doubles).
 */
#ifndef HLU_RK_LAYOUT_H
#define HLU_RK_LAYOUT_H

#include <stdint.h>

#ifdef __CUDACC__
#define RK_HD __host__ __device__ __forceinline__
#else
#define RK_HD inline
#endif

#define RK_KMAX 64       /* stacked rank of the block-TSQR pipeline (phases A, B, C) */
#define RK_KMAXW 128     /* stacked rank of the wide path (k_rkt_w, 64 < K <= 128) */
#define RK_BR 512        /* rows per block (one phase-A / phase-C work item) */
#define RK_BUFA 16384    /* chunk buffer of the layout: (ch + K) K <= RK_BUFA (doubles) */
#define RK_BUFS 6144     /* small phase A/C kernels: items whose chunk fits (min(ch, rows) + K) K */
#define RK_TBUF 8192     /* large phase C kernel: moving block, processed in column groups */
#define RK_BUFB32 3072   /* phase B per-side buffer, K <= 32 */
#define RK_BUFB64 8192   /* phase B per-side buffer, 32 < K <= 64 */

/* fresh rows per chunk: the largest power of two in [32, 512] with (ch + K) K <= bufd */
RK_HD int rk_ch(int K, int bufd) {
  int ch = 512;
  while (ch > 32 && (ch + K) * K > bufd) ch >>= 1;
  return ch;
}

RK_HD int64_t rk_stride(int K, int ch) { return (int64_t)(K + ch) * K + K; }

/* shared-memory need (doubles) of one row block's chain: ld (min(ch, rows) + K) times K */
RK_HD int rk_item_need(int rows, int K, int ch) { return ((rows < ch ? rows : ch) + K) * K; }

/* workspace of a chain over `rows` rows */
RK_HD int64_t rk_chain(int rows, int K, int ch) { return (int64_t)((rows + ch - 1) / ch) * rk_stride(K, ch); }

typedef struct {
  int nb, ch, chc, zrows, srows;
  int64_t blk, off_R, off_comb, off_Z, total;
} rk_side_t;

RK_HD int rk_chc(int K) { return rk_ch(K, K <= 32 ? RK_BUFB32 : RK_BUFB64); }

RK_HD rk_side_t rk_side(int M, int K) {
  rk_side_t s;
  s.ch = rk_ch(K, RK_BUFA);
  s.chc = rk_chc(K);
  s.nb = (M + RK_BR - 1) / RK_BR;
  const int last = M - (s.nb - 1) * RK_BR;
  const int r_last = last < K ? last : K;
  s.blk = rk_chain(RK_BR, K, s.ch);
  s.off_R = (int64_t)(s.nb - 1) * s.blk + rk_chain(last, K, s.ch);
  s.off_comb = s.off_R + (int64_t)s.nb * K * K;
  s.srows = (s.nb - 1) * K + r_last;
  s.off_Z = s.off_comb + (s.nb > 1 ? rk_chain(s.srows, K, s.chc) : 0);
  s.zrows = s.srows;
  s.total = s.off_Z + (int64_t)s.zrows * K;
  return s;
}

/* wide path workspace (global memory, K in (RK_KMAX, RK_KMAXW]):
 * X (m x K) | Y (n x K) | M (KW x KW) | V (KW x KW) | tau_x | tau_y | sigma (KW each) */
RK_HD int64_t rk_wide_doubles(int m, int n, int K) {
  return (int64_t)(m + n) * K + 2 * (int64_t)RK_KMAXW * RK_KMAXW + 3 * RK_KMAXW;
}

/* reserved workspace (doubles) of one truncation with stacked rank <= kbound:
 * the maximum over K of the runtime layout.  The layout grows with K while
 * (ch, chc) stay fixed, so only the last K of every (ch, chc) class matters;
 * kbound > RK_KMAX adds the wide path's workspace. */
RK_HD int64_t rk_ws_doubles(int m, int n, int kbound) {
  if (m <= 0 || n <= 0 || kbound <= 0) return 0;
  const int kb = kbound < RK_KMAX ? kbound : RK_KMAX;
  int64_t best = 0;
  for (int K = 1; K <= kb; ++K) {
    if (K < kb && rk_ch(K + 1, RK_BUFA) == rk_ch(K, RK_BUFA) && rk_chc(K + 1) == rk_chc(K)) continue;
    const int64_t t = rk_side(m, K).total + rk_side(n, K).total;
    if (t > best) best = t;
  }
  if (kbound > RK_KMAX) {
    const int kw = kbound < RK_KMAXW ? kbound : RK_KMAXW;
    const int64_t t = rk_wide_doubles(m, n, kw);
    if (t > best) best = t;
  }
  return best;
}

#endif /* HLU_RK_LAYOUT_H */
