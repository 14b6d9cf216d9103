/*
 * hlu_plan.h — C ABI of the native planner / level scheduler (host code).
 *
 * Replaces the reference's executor seam (hlu.py:315-354, ex.leaf/ex.parent)
 * and its task runtime (runtime.py:380-556) for the GPU: the recursion of
 * hlu.py:400-658 is replayed into typed device ops (hlu_b200.h descriptors),
 * levelled by skeleton-slot hazards and packed per (level, kernel) launch.
 */
#ifndef HLU_PLAN_H
#define HLU_PLAN_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* One H-matrix node (flattened tree).  Children of a partitioned node are
 * nodes child0 .. child0 + nr*nc - 1 in row-major grid order. */
typedef struct {
  int32_t kind;            /* 0 dense leaf, 1 Rk leaf, 2 partitioned */
  int32_t r0, r1, c0, c1;  /* global row / column ranges */
  int32_t nr, nc;          /* grid (partitioned) */
  int32_t child0;          /* first child, -1 for leaves */
  int32_t lo, hi;          /* skeleton slot interval */
  int32_t slot;            /* rank slot (Rk leaves), -1 otherwise */
  int32_t pad;
  int64_t off_a;           /* dense payload / Rk left factor offset in the pool */
  int64_t off_b;           /* Rk right factor offset */
} hlu_plan_node;           /* 64 bytes */

enum {
  HLU_CMD_FACTOR = 0,      /* a = root */
  HLU_CMD_SOLVE_LOWER = 1, /* a = l, b = b   : b := l^-1 b */
  HLU_CMD_SOLVE_UPPER = 2, /* a = b, b = u   : b := b u^-1 */
  HLU_CMD_UPDATE = 3,      /* a = c, b = a, c = b : c := c - a b */
  HLU_CMD_FWD_VEC = 4,     /* a = factored root, vector at vec_off (resource vec_res) */
  HLU_CMD_BWD_VEC = 5,
  /* y += op(a) x with x at vec_off (vec_res), y at vec2_off (vec2_res), both
   * vec_cols wide: the full H-matrix (hmatvec, hmatrix.py:178-200), the unit
   * lower factor or the upper factor of a factored root (hlu.py:720-767) */
  HLU_CMD_MATVEC = 6,
  HLU_CMD_LOWER_MATVEC = 7,
  HLU_CMD_UPPER_MATVEC = 8
};

typedef struct {
  int32_t kind, a, b, c;
  int64_t vec_off;
  int32_t vec_cols, pad;
  int64_t vec_res;
  int64_t vec2_off, vec2_res;
} hlu_plan_cmd; /* 56 bytes */

typedef struct hlu_plan hlu_plan;

/* split_rows > 0: cut GEMM chains whose terms write disjoint row ranges of one
 * target into independent sub-chains of >= split_rows rows (0 = never) */
int hlu_plan_build(hlu_plan **out, const hlu_plan_node *nodes, int64_t nnodes, const hlu_plan_cmd *cmds,
                   int64_t ncmds, int32_t cap, int64_t ident_off, int64_t nslots, int32_t nrk, int64_t arena_base,
                   int32_t split_rows);
/* Owner-computes sharding over nranks GPUs: slot_owner[s] is
 * the rank owning skeleton slot s; the plan for `rank` holds only the ops that
 * rank executes (the writer's owner; temp producers on every consuming rank),
 * with the single-GPU levels, temps and op order, plus the slot exchange
 * records (hlu_plan_xfer).  slot_owner == NULL is hlu_plan_build. */
int hlu_plan_build_sharded(hlu_plan **out, const hlu_plan_node *nodes, int64_t nnodes, const hlu_plan_cmd *cmds,
                           int64_t ncmds, int32_t cap, int64_t ident_off, int64_t nslots, int32_t nrk,
                           int64_t arena_base, int32_t split_rows, const int32_t *slot_owner, int32_t nranks,
                           int32_t rank);
/* DAG schedule (replaces the level barriers; the GPU analogue of the paper's
 * task DAG with region dependencies, PAPER.md:598-670 / runtime.py:443-556): a
 * hazard sweep in model time (per-op latency model) gives every op a start
 * time; ops of one kernel class whose start falls into the same slot_ns window
 * form a launch, and every launch lists the launches it depends on (RAW / WAR /
 * WAW on skeleton slots and temps, arena-block hand-over).  hlu_launch.level is
 * then the launch-group key in topological order (no barrier semantics) and
 * truncation launches carry a route hint in smem_dim (bit 4: no op with
 * max(m, n) <= 64, the register warp kernels are not launched).
 * slot_ns <= 0 is hlu_plan_build. */
int hlu_plan_build_dag(hlu_plan **out, const hlu_plan_node *nodes, int64_t nnodes, const hlu_plan_cmd *cmds,
                       int64_t ncmds, int32_t cap, int64_t ident_off, int64_t nslots, int32_t nrk, int64_t arena_base,
                       int32_t split_rows, int64_t slot_ns);
/* dependency lists of a DAG plan: launch l waits for the launches
 * idx[ptr[l] .. ptr[l+1]) (all < l); ptr has launches + 1 entries.  Returns the
 * edge count (ptr / idx may be NULL), -1 for a level plan. */
int64_t hlu_plan_dag(const hlu_plan *p, int64_t *ptr, int32_t *idx);
/* per launch: model-time slack in ns (0 = on the model's critical path) */
int hlu_plan_dag_slack(const hlu_plan *p, int64_t *slack_ns);
const char *hlu_plan_error(const hlu_plan *p);
/* sizes[14]: getrf, trsm, gemm, terms, rkt, parts, launches, ops, levels, arena doubles,
 *            log entries, rank slots, LU count, temps */
int hlu_plan_sizes(const hlu_plan *p, int64_t *sizes);
int hlu_plan_copy(const hlu_plan *p, void *getrf, void *trsm, void *gemm, void *terms, void *rkt, void *parts,
                  void *launches, int32_t *flop_formula, double *flop_coef, int64_t *flop_log, int64_t *lu_op_ids,
                  int64_t *lu_nodes, int64_t *op_levels);
/* Two-chain schedule (hlu_schedule_create's wait arrays), one entry per level:
 * wait_dense[l] / wait_rkt[l] = last level of the truncation / dense chain that
 * the dense / truncation launches of level l wait for (-1: none), from the ops'
 * slot / temp hazards and arena-block reuse.  Returns -1 when the plan has a
 * hazard the two chains cannot express (the caller keeps level barriers). */
int hlu_plan_level_waits(const hlu_plan *p, int32_t *wait_dense, int32_t *wait_rkt);
void hlu_plan_free(hlu_plan *p);

/* One slot exchange record of a sharded plan: after level `level` (level ==
 * nlevels: the final gather) rank `src` broadcasts pool[off, off+len) and, for
 * an Rk slot, ranks[rank_slot] (as a double after the payload) to every rank,
 * staged at boff of group `group`'s buffer.  Records are ordered by (level,
 * src, group); a group's staging buffer holds sum(len + 1) doubles. */
typedef struct {
  int32_t level, src;
  int32_t group, rank_slot; /* rank_slot -1: dense slot */
  int64_t off, len, boff;
} hlu_xfer; /* 40 bytes */

/* exchange records of a sharded plan (out may be NULL); returns their count */
int64_t hlu_plan_xfer(const hlu_plan *p, hlu_xfer *out);
/* per op: bit r set when rank r executes it (sharded plans only; else -1) */
int hlu_plan_op_owners(const hlu_plan *p, uint64_t *out);

/* --- host payload staging (the upload / download of hlu_factorize) ---
 * One leaf payload: a row-major host array (numpy C order, rows x cols, row
 * stride host_stride doubles) <-> a column-major slab of the pool at off with
 * leading dimension ld.  Replaces the per-leaf numpy copies around the
 * reference's in-place leaf updates (lowrank.py:50-51 keeps factors C-contiguous). */
typedef struct {
  void *host;
  int64_t off;
  int32_t rows, cols;
  int32_t ld, host_stride;
} hlu_pack_rec; /* 32 bytes */

/* threads <= 0: one per hardware thread */
int hlu_host_pack(const hlu_pack_rec *recs, int64_t n, double *pool, int threads);
int hlu_host_unpack(const hlu_pack_rec *recs, int64_t n, const double *pool, int threads);

/* The same copies with recs[i].host = the numpy array OBJECT (id(array)): the
 * data pointers are read from numpy's PyArrayObject and every array is checked
 * to be a C-contiguous float64 rows x cols array (writeable when unpack != 0).
 * recs[i].host is replaced by the data pointer.  Returns 0, or -(i + 1) for the
 * first array failing the check (nothing is copied then). */
int64_t hlu_host_pack_np(hlu_pack_rec *recs, int64_t n, double *pool, int threads, int unpack);

/* Effective-flop total of one call: the reference's FlopCounter (hlu.py:46-55,
 * incremented at hlu.py:408-637) evaluated from the planner's per-op formulas
 * (formula 0: coef; 1: coef k; 3: coef k^2; 2: 2 (kc + kp + 1) coef (kp + 1),
 * with k / kp / kc = log[flog], log[flog + 1], log[flog + 2]) and the ranks the
 * kernels logged.  Deterministic for any thread count. */
double hlu_effective_flops(const int64_t *formula, const double *coef, const int64_t *flog, int64_t nops,
                           const int32_t *log, int64_t nlog, int threads);

#ifdef __cplusplus
}
#endif

#endif /* HLU_PLAN_H */
