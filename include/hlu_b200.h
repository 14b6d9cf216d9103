/*
 * hlu_b200.h — C ABI of the B200-native H-LU hot path (sm_100a).
 *
 * The reference (hluflow, pure Python) has no FFI; its hot path is the set of
 * LAPACK/BLAS call sites under the H-recursion.  Each entry point below
 * replaces a family of those call sites, batched over one level of the leaf
 * DAG:
 *
 *   hlu_getrf_batched_f64   <- lu_nopivot            lowrank.py:183-231, called at hlu.py:635-637
 *   hlu_trsm_batched_f64    <- trsm_lower_unit        lowrank.py:234-239 (hlu.py:407,450)
 *                              trsm_upper_right       lowrank.py:242-247 (hlu.py:487,534)
 *                              Rk-factor solves       hlu.py:415-418, 495-498, 531
 *                              (+ backward vector solve U x = y, absent in the reference)
 *   hlu_gemm_batched_f64    <- gemm_update            lowrank.py:250-261 (hlu.py:217..604)
 *                              _op_matmat/_op_t_matmat/_op_*gemm_into  hlu.py:160-255
 *   hlu_rk_update_batched_f64 <- add_truncated        lowrank.py:148-168
 *                              recompress             lowrank.py:137-145 (incl. _merge_lowrank hlu.py:294-309)
 *                              compress_dense         lowrank.py:171-175 (dense x dense products, hlu.py:269-270)
 *                              _truncate_svd          lowrank.py:127-134
 *   hlu_schedule_*          <- the sequential/OmpSs executor (hlu.py:315-354, runtime.py):
 *                              a precomputed level-set schedule replayed as one CUDA graph.
 *
 * Conventions: all matrices live in ONE fp64 device pool; a view addresses
 * element (i,j) at pool[off + i*rs + j*cs].  Dimensions flagged dynamic read
 * the current rank of an Rk object from the int32 rank table at kernel time,
 * so ranks can grow and shrink in place.  Every call is stream-ordered and
 * returns 0 or a negative error code; device-side failures (small pivot,
 * rank-capacity overflow) land in the error words of hlu_ctx.err.
 */
#ifndef HLU_B200_H
#define HLU_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* element (i,j) at pool[off + i*rs + j*cs]; rdyn/cdyn >= 0 -> dimension is ranks[slot] */
typedef struct {
  int64_t off;
  int32_t rows, cols;
  int32_t rs, cs;
  int32_t rdyn, cdyn;
} hlu_view; /* 32 bytes */

/* device pointers shared by every kernel */
typedef struct {
  double *pool;    /* all payloads, temps and workspaces */
  int32_t *ranks;  /* current rank per Rk object */
  int32_t *log;    /* dynamic values logged for the effective-flop counter */
  int32_t *err;    /* [0] overflow count, [1] first failing LU op (INT32_MAX = none),
                      [2] unsupported-shape count, [3] reserved */
  double *dlog;    /* per-LU (pivot, tol) of a failure: dlog[2*lu_index] */
  double eps;      /* TruncationControl.eps */
  int32_t kmax;    /* TruncationControl.kmax, -1 = none */
  int32_t pad;
} hlu_ctx;

/* In-place unpivoted LU of a square block (n <= 128 in shared memory, n <= 256 64-blocked in place). */
typedef struct {
  hlu_view a;
  int32_t op_id;   /* program-order index, for the SingularBlockError label */
  int32_t lu_index;
} hlu_getrf_desc; /* 40 bytes */

enum {
  HLU_TRSM_LEFT_LOWER_UNIT = 0, /* X <- L^-1 X   */
  HLU_TRSM_RIGHT_UPPER = 1,     /* X <- X U^-1   */
  HLU_TRSM_LEFT_UPPER = 2       /* X <- U^-1 X   */
};

typedef struct {
  hlu_view t, x;
  int32_t mode;
  int32_t log;     /* >= 0: log[log] = dynamic RHS count */
} hlu_trsm_desc; /* 72 bytes */

enum { HLU_TERM_ZERO = 0, HLU_TERM_GEMM = 1, HLU_TERM_TRIPLE = 2 };

/* assoc of a GEMM term: which part of A enters (triangular matvecs with the
 * stored factors, reference hlu.py:720-767) */
enum { HLU_TRI_NONE = 0, HLU_TRI_UPPER = 1, HLU_TRI_UNIT_LOWER = 2 };

/* one term of an ordered accumulation chain:
 *   ZERO:   C = 0
 *   GEMM:   C += alpha * A B   (A = triu(A) / tril(A,-1)+I per assoc)
 *   TRIPLE: C += alpha * A (M B)   (assoc 0)   or   alpha * (A M) B   (assoc 1) */
typedef struct {
  hlu_view c, a, m, b;
  double alpha;
  int32_t kind, assoc;
} hlu_term; /* 144 bytes */

typedef struct {
  int32_t term_begin, term_count;
  int32_t log, log_slot; /* log[log] = ranks[log_slot] at execution, if log >= 0 */
} hlu_gemm_desc; /* 16 bytes */

/* one factor pair of a truncation input, placed at (roff, coff) of the output frame */
typedef struct {
  hlu_view a, b;   /* a: m_p x k, b: n_p x k (k may be dynamic) */
  double sign;     /* applied to a */
  int32_t roff, coff;
} hlu_rkpart; /* 80 bytes */

enum {
  HLU_RK_ADD = 0,        /* add_truncated(part0, part1) with the reference shortcuts */
  HLU_RK_RECOMPRESS = 1  /* recompress(concat(parts)) ; also compress_dense(A@B) as part (A, B^T) */
};

typedef struct {
  int32_t mode, part_begin, part_count;
  int32_t m, n, cap;
  int32_t out_slot, log;
  int64_t out_a, out_b;  /* column-major outputs, ld = m / n, capacity cap columns */
  int64_t ws;            /* workspace offset in the pool: hlu_rkt_ws_doubles(m, n, kbound) doubles */
  int32_t reserved;      /* 0 */
  int32_t pad;
} hlu_rkt_desc; /* 64 bytes */

/* one row block (<= 512 rows) of one factor of a truncation: the unit of the
 * parallel TSQR (phase A) and Q application (phase C) */
typedef struct {
  int32_t op;      /* index into the descriptor array */
  int16_t side;    /* 0: left factor (m rows), 1: right factor (n rows) */
  int16_t block;   /* row block */
} hlu_rkt_item; /* 8 bytes */

/* launch kinds of a schedule entry (HLU_K_RKT32: the truncations of a level, any stacked
 * rank; HLU_K_RKT64 is no longer emitted and is ignored) */
enum { HLU_K_GETRF = 0, HLU_K_TRSM = 1, HLU_K_GEMM = 2, HLU_K_RKT32 = 3, HLU_K_RKT64 = 4, HLU_K_GEMM_SMALL = 5 };

typedef struct {
  int32_t kind;
  int32_t count;
  int64_t first;     /* index of the first descriptor of this launch */
  int32_t smem_dim;  /* largest square dimension (getrf / trsm); truncation launches: 1 when
                        they read a temp a dense launch of the same level produces */
  int32_t level;     /* schedule level: launches of one level are independent */
} hlu_launch; /* 24 bytes */

/* --- batched kernels (descriptor arrays are device pointers) --- */
int hlu_getrf_batched_f64(const hlu_ctx *ctx, const hlu_getrf_desc *d, int count, int max_n, void *stream);
int hlu_trsm_batched_f64(const hlu_ctx *ctx, const hlu_trsm_desc *d, int count, int max_n, void *stream);
int hlu_gemm_batched_f64(const hlu_ctx *ctx, const hlu_gemm_desc *d, const hlu_term *terms, int count,
                         void *stream);
/* small chains (planner-classified: every triple's M.rows x C.cols <= 1024,
 * assoc-1 triples with M.cols <= 64): one warp per chain */
int hlu_gemm_small_batched_f64(const hlu_ctx *ctx, const hlu_gemm_desc *d, const hlu_term *terms, int count,
                               void *stream);
/* device scratch of the truncation launches: per level 8 counters (ops of the register
 * warp kernels K<=8 / K<=16, the large-buffer row blocks, the CTA path, then the
 * CTA-path ops whose core SVD one warp does, two reserved, then the small-buffer row
 * blocks) at counts + 8*slot, zeroed before the level runs; list = 7 segments
 * of max_ops op indices; items = max_items row blocks (max over levels of hlu_rkt_items):
 * small-buffer blocks from the front, large-buffer blocks from the back */
typedef struct {
  int32_t *counts;
  int32_t *list;
  hlu_rkt_item *items;
  int64_t max_ops, max_items;
} hlu_rkt_scratch;

/* count truncations d[0 .. count) (count <= scratch->max_ops; counter slot 0).  A
 * classify kernel routes every op: max(m,n) <= 64 and K <= 16 -> one warp per op with
 * the factors in registers; others ->
 * block TSQR (one CTA per 512-row block), core SVD + rank (one CTA per op), Q apply
 * (one CTA per block). */
int hlu_rk_update_batched_f64(const hlu_ctx *ctx, hlu_rkt_desc *d, const hlu_rkpart *parts, int count,
                              const hlu_rkt_scratch *scratch, void *stream);
/* auxiliary streams (cudaStream_t) and events (cudaEvent_t) for hlu_rkt_phases */
typedef struct {
  void *side[4];
  void *ev[8];
} hlu_rkt_streams;

/* ops d[first .. first+count) of one level with counter slot `slot` (zeroed by the
 * caller).  With aux, independent kernels run as concurrent branches (register warp
 * kernels on side[0..1], the three core kernels on stream/side[2]/side[3]) joined on
 * `stream`; aux == NULL runs everything in order on `stream`. */
int hlu_rkt_phases(const hlu_ctx *ctx, hlu_rkt_desc *d, const hlu_rkpart *parts, int64_t first, int count,
                   const hlu_rkt_scratch *scratch, int slot, void *stream, const hlu_rkt_streams *aux);
/* one kernel only (diagnostics / per-kernel timing): 0 classify, 1 register warp K<=8,
 * 2 register warp K<=16, 3 (none), 4 block TSQR, 5 core by one warp
 * (K<=16), 6 core K<=32, 7 core K>32, 8 Q apply, 9 block TSQR of the row blocks whose
 * chunk chain needs the large buffer, 10 Q apply of those */
int hlu_rkt_phase(const hlu_ctx *ctx, hlu_rkt_desc *d, const hlu_rkpart *parts, int64_t first, int count,
                  const hlu_rkt_scratch *scratch, int slot, int which, void *stream);
/* host: the work items of count HOST descriptors in op order (items may be NULL); returns their number */
int64_t hlu_rkt_items(const hlu_rkt_desc *d, int count, hlu_rkt_item *items);

/* workspace (doubles) one truncation of an m x n block with stacked rank <= kbound needs */
int64_t hlu_rkt_ws_doubles(int32_t m, int32_t n, int32_t kbound);

/* --- level-set schedule runtime (one CUDA graph per factorization) --- */
typedef struct hlu_schedule hlu_schedule;

/* launches: host array (copied); descriptor arrays and the scratch buffers: device
 * pointers that must outlive the schedule (scratch->counts holds 4 ints per truncation
 * launch; the struct itself is copied); use_graph: capture the launch sequence into a
 * CUDA graph */
int hlu_schedule_create(hlu_schedule **out, const hlu_ctx *ctx, const hlu_launch *launches, int64_t nlaunch,
                        const hlu_getrf_desc *getrf, const hlu_trsm_desc *trsm, const hlu_gemm_desc *gemm,
                        const hlu_term *terms, hlu_rkt_desc *rkt, const hlu_rkpart *parts,
                        const hlu_rkt_scratch *scratch, int use_graph, void *stream);
/* Same, as two chains: the dense launches (getrf / trsm / gemm) of every level
 * on one stream, the truncation launches on another, each chain in level order,
 * with cross-chain waits only where the plan has a hazard (hlu_plan_level_waits:
 * nlevels entries each).  Consecutive levels of the two classes overlap instead
 * of meeting at a barrier after every level.  Null waits = hlu_schedule_create. */
int hlu_schedule_create_chains(hlu_schedule **out, const hlu_ctx *ctx, const hlu_launch *launches, int64_t nlaunch,
                               const hlu_getrf_desc *getrf, const hlu_trsm_desc *trsm, const hlu_gemm_desc *gemm,
                               const hlu_term *terms, hlu_rkt_desc *rkt, const hlu_rkpart *parts,
                               const hlu_rkt_scratch *scratch, const int32_t *wait_dense, const int32_t *wait_rkt,
                               int64_t nlevels, int use_graph, void *stream);
/* The DAG schedule (include/hlu_plan.h hlu_plan_build_dag) as one CUDA graph whose
 * edges are the planner's launch dependencies: launch l waits for the launches
 * dep_idx[dep_ptr[l] .. dep_ptr[l+1]) (all < l) and for nothing else, so launches of
 * different time slots overlap where the level schedule put a barrier (the GPU
 * analogue of the reference runtime's region dependencies, runtime.py:443-556).
 * Truncation launches run concurrently, each in its own window of the scratch:
 * scratch->list holds 7 ints per truncation descriptor (window at 7 * first,
 * max_ops = descriptor count), scratch->items every row-block item (item0 / nitems:
 * the window of each truncation launch, from hlu_rkt_items), scratch->counts 8 ints
 * per truncation launch.  prio (may be NULL): 0 .. 2 per launch, kernels of
 * higher-priority launches are scheduled first when SMs are contended. */
int hlu_schedule_create_dag(hlu_schedule **out, const hlu_ctx *ctx, const hlu_launch *launches, int64_t nlaunch,
                            const hlu_getrf_desc *getrf, const hlu_trsm_desc *trsm, const hlu_gemm_desc *gemm,
                            const hlu_term *terms, hlu_rkt_desc *rkt, const hlu_rkpart *parts,
                            const hlu_rkt_scratch *scratch, const int64_t *dep_ptr, const int32_t *dep_idx,
                            const int64_t *item0, const int64_t *nitems, const int32_t *prio, void *stream);
/* kernel nodes the DAG capture issued (diagnostics) */
int64_t hlu_schedule_graph_nodes(const hlu_schedule *s);
/* --- multi-GPU: owner-computes H-LU over a communicator (NCCL, NVLink) --- */
typedef struct hlu_comm hlu_comm;
struct hlu_xfer_s;
int hlu_comm_available(void);            /* 1 when libnccl.so.2 could be loaded */
int hlu_comm_unique_id(void *out128);    /* rank 0: returns the id size (128) */
int hlu_comm_init(hlu_comm **out, const void *id128, int nranks, int rank); /* on the rank's device */
int hlu_comm_destroy(hlu_comm *c);
/* Sharded schedule (include/hlu_plan.h hlu_plan_build_sharded): this rank's
 * launches level by level; after every level the exchange groups of that level
 * (xfer records: host copy for the grouping, device copy for the kernels; the
 * staging buffer holds hlu_xfer_staging_doubles); after the last level the
 * final gather and the reduction of the nlog flop-log entries and the error
 * words over the communicator.  Every rank ends with the whole factorization. */
int hlu_schedule_create_sharded(hlu_schedule **out, const hlu_ctx *ctx, const hlu_launch *launches, int64_t nlaunch,
                                const hlu_getrf_desc *getrf, const hlu_trsm_desc *trsm, const hlu_gemm_desc *gemm,
                                const hlu_term *terms, hlu_rkt_desc *rkt, const hlu_rkpart *parts,
                                const hlu_rkt_scratch *scratch, hlu_comm *comm, const void *xfer_host,
                                const void *xfer_dev, int64_t nxfer, int64_t nlevels, int64_t nlog, double *staging,
                                int use_graph, void *stream);
int64_t hlu_xfer_staging_doubles(const void *xfer, int64_t n);
/* one exchange group (diagnostics / tests): gather -> ncclBroadcast -> scatter */
int hlu_xfer_group(hlu_comm *c, double *pool, int32_t *ranks, const void *xfer_dev, int n, int src, int64_t count,
                   double *staging, void *stream);

int hlu_schedule_launch(hlu_schedule *s, void *stream);
int hlu_schedule_destroy(hlu_schedule *s);
/* diagnostics: with HLU_STAMPS=1 at creation, the %globaltimer (ns) before the first and
 * after every launch of the last replay (nlaunch + 1 values), then 12 per truncation launch
 * (after each of the 11 kernels of hlu_rkt_phase, then the join); returns the count
 * (out may be NULL), 0 without stamps */
int64_t hlu_schedule_stamps(hlu_schedule *s, unsigned long long *out);

/* --- GPU assembly (reference kernels.py:73-168) --- */
typedef struct {
  int32_t r0, r1, c0, c1; /* point ranges (cluster-tree order) */
  int32_t tcl, scl;       /* cluster ids of the interpolation data (Rk leaves) */
  int32_t kind, pad;
  int64_t out_a, out_b;   /* pool offsets: dense block (column-major) / factor pair X, Y */
} hlu_asm_desc; /* 48 bytes */
/* dense leaves: A_ij = g(|x_i - y_j|), coincident points at diag (assemble_dense_block) */
int hlu_asm_dense_f64(const double *pts, int d, const void *desc, int count, double diag, double *pool, void *stream);
/* Rk leaves: X = U_t K(nodes_t, nodes_s) (m x Gs), Y = U_s (n x Gs) by tensor Chebyshev
 * interpolation (assemble_lowrank_block; recompressed by hlu_rk_update_batched_f64) */
int hlu_asm_cheb_f64(const double *pts, int d, const void *desc, int count, const int32_t *cl_cnt,
                     const double *cl_nodes, const double *cl_w, int max_grid, double *pool, void *stream);
/* HODLR blocks: partially pivoted cross approximation to at most k terms (U, V; nterms per block) */
int hlu_asm_aca_f64(const double *pts, int d, const void *desc, int count, int k, double diag, double *pool,
                    int32_t *nterms, void *stream);

/* library identity / sanity */
const char *hlu_version(void);
int hlu_device_check(void); /* 0 when a sm_100 device is present */
int64_t hlu_debug_sweeps(int reset); /* total Jacobi sweeps run so far (diagnostics) */
/* core-kernel phase cycles [K<=32 | K>32][op count, R/combine, core product, QRCP, Jacobi,
 * rank, W + QRCP apply, combine apply], then the Jacobi sweeps and rounds of [K<=32, K>32]
 * (20 values; zeros unless built with -DHLU_BPROF) */
int hlu_debug_bprof(unsigned long long *out, int reset); /* out[32]: phase cycles (diagnostics build) */

#ifdef __cplusplus
}
#endif

#endif /* HLU_B200_H */
