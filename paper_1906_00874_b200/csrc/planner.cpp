// Native planner + level scheduler (host C++).
//
// A line-by-line port of planner.py / schedule.py (which stay as the readable,
// tested specification): it replays the reference H-LU recursion
// (hlu.py:400-658) into typed device ops, levels them by skeleton-slot and
// temp hazards, allocates the temp arena and packs the descriptor arrays.
// tests/test_native_planner.py checks that both produce byte-identical packed
// arrays.  The Python planner takes ~75 s per 5.6M reference tasks (cfg3);
// this one takes a few seconds.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <initializer_list>
#include <cstdint>
#include <cstring>
#include <limits>
#include <stdexcept>
#include <string>
#include <unordered_map>
#include <vector>

#include "hlu_b200.h"
#include "hlu_plan.h"
#include "rk_layout.h"

namespace {

constexpr int64_t TEMP_SHIFT = 36;  // temp t at (t+1) << 36: up to 2^27 temps, 2^36-double offsets
constexpr int KMAX_STACK = RK_KMAX;  // widest dense-product factor pair truncated as (A, B^T)
constexpr int IDENT = RK_KMAXW;  // identity block edge kept in the pool
constexpr int F_STATIC = 0, F_LIN = 1, F_RKUPD = 2, F_QUAD = 3;

struct View {
  int64_t off;
  int32_t rows, cols, rs, cs, rdyn, cdyn;
  View T() const { return View{off, cols, rows, cs, rs, cdyn, rdyn}; }
  View rows_slice(int i0, int i1) const {
    if (rdyn >= 0 || i0 < 0 || i1 > rows || i0 > i1) throw std::runtime_error("bad rows_slice");
    return View{off + (int64_t)i0 * rs, i1 - i0, cols, rs, cs, rdyn, cdyn};
  }
  View cols_slice(int j0, int j1) const {
    if (cdyn >= 0 || j0 < 0 || j1 > cols || j0 > j1) throw std::runtime_error("bad cols_slice");
    return View{off + (int64_t)j0 * cs, rows, j1 - j0, rs, cs, rdyn, cdyn};
  }
};
const View NULLV{0, 0, 0, 0, 0, -1, -1};

inline hlu_view hv(const View &v) {
  hlu_view o;
  o.off = v.off;
  o.rows = v.rows;
  o.cols = v.cols;
  o.rs = v.rs;
  o.cs = v.cs;
  o.rdyn = v.rdyn;
  o.cdyn = v.cdyn;
  return o;
}

struct Pair {
  View a, b;
  double sign = 1.0;
  int roff = 0, coff = 0;
};

struct Opnd {  // an H-node or a window of a leaf, in global coordinates
  int node;
  int r0, r1, c0, c1;
  bool win;
};

struct Iv {
  int64_t lo, hi;
};

// read-only view of a vector or a braced list (no allocation for the short
// read / write / temp lists every op passes)
#pragma GCC diagnostic ignored "-Winit-list-lifetime"  // Spans only ever bind call arguments
template <class T>
struct Span {
  const T *p = nullptr;
  size_t n = 0;
  Span() = default;
  Span(const std::vector<T> &v) : p(v.data()), n(v.size()) {}
  Span(std::initializer_list<T> l) : p(l.begin()), n(l.size()) {}
  const T *begin() const { return p; }
  const T *end() const { return p + n; }
  size_t size() const { return n; }
  bool empty() const { return n == 0; }
  const T &operator[](size_t i) const { return p[i]; }
};

struct Term {
  int kind;
  View c, a, m, b;
  double alpha;
  int assoc;
};

struct Op {
  int kind;  // 0 getrf, 1 trsm, 2 gemm, 3 rkt
  bool defer;
  int64_t payload;  // index into the kind's payload store
  int64_t r_begin, r_end, w_begin, w_end;  // into ivs
  int64_t ti_begin, ti_end, to_begin, to_end;  // into tids
  int flop_f;
  double flop_c;
  int64_t flop_log;
};

struct GetrfP {
  View a;
  int op_id, lu_index;
};
struct TrsmP {
  View t, x;
  int mode, log;
};
struct GemmP {
  int64_t tb, tn;
  int log, log_slot;
  bool split;  // terms only write row ranges of one target and never read it
};
struct RktP {
  int mode;
  int64_t pb, pn;
  int m, n, cap, slot, log;
  int64_t out_a, out_b, ws;
  int kb;
};


struct Planner {
  const hlu_plan_node *N;
  int64_t nnodes;
  int cap;
  int64_t ident_off;
  int64_t nslots;
  int nrank;

  std::vector<Op> ops;
  std::vector<Iv> ivs;
  std::vector<int64_t> tids;
  std::vector<int64_t> temp_size;
  int64_t nlog = 0;
  std::vector<GetrfP> getrf;
  std::vector<TrsmP> trsm;
  std::vector<GemmP> gemm;
  std::vector<Term> terms;
  std::vector<RktP> rkt;
  std::vector<Pair> parts;
  std::vector<int64_t> lu_ops, lu_nodes;

  const hlu_plan_node &nd(int i) const { return N[i]; }
  bool part(const Opnd &o) const { return !o.win && nd(o.node).kind == 2; }
  bool rk(const Opnd &o) const { return nd(o.node).kind == 1; }
  Opnd whole(int i) const { const auto &x = nd(i); return Opnd{i, x.r0, x.r1, x.c0, x.c1, false}; }
  int child(int i, int r, int c) const { const auto &x = nd(i); return x.child0 + r * x.nc + c; }
  Opnd window(const Opnd &o, int r0, int r1, int c0, int c1) const {
    if (part(o)) throw std::runtime_error("cannot window a partitioned block");
    const auto &x = nd(o.node);
    if (!o.win && r0 == x.r0 && r1 == x.r1 && c0 == x.c0 && c1 == x.c1) return o;
    return Opnd{o.node, r0, r1, c0, c1, true};
  }
  Iv res(const Opnd &o) const { const auto &x = nd(o.node); return Iv{x.lo, x.hi}; }
  std::vector<std::pair<int, int>> row_cuts(int i) const {
    const auto &x = nd(i);
    std::vector<std::pair<int, int>> v;
    for (int r = 0; r < x.nr; ++r) { const auto &c = nd(child(i, r, 0)); v.push_back({c.r0, c.r1}); }
    return v;
  }
  std::vector<std::pair<int, int>> col_cuts(int i) const {
    const auto &x = nd(i);
    std::vector<std::pair<int, int>> v;
    for (int c = 0; c < x.nc; ++c) { const auto &y = nd(child(i, 0, c)); v.push_back({y.c0, y.c1}); }
    return v;
  }

  int64_t temp(int64_t doubles, int64_t *base) {
    const int64_t t = (int64_t)temp_size.size();
    if (t + 1 >= (int64_t(1) << 27)) throw std::runtime_error("too many temporaries for the 36-bit temp encoding");
    temp_size.push_back(doubles);
    *base = (t + 1) << TEMP_SHIFT;
    return t;
  }
  Iv temp_res(int64_t t) const { return Iv{nslots + t, nslots + t + 1}; }
  int rank_slot() { return nrank++; }
  int64_t log(int n = 1) { const int64_t i = nlog; nlog += n; return i; }
  static int64_t pair_temp(const Pair &p) { return (p.a.off >> TEMP_SHIFT) - 1; }

  View dense_view(const Opnd &o) const {
    const auto &x = nd(o.node);
    const int rows = x.r1 - x.r0;
    return View{x.off_a + (o.r0 - x.r0) + (int64_t)(o.c0 - x.c0) * rows, o.r1 - o.r0, o.c1 - o.c0, 1, rows, -1, -1};
  }
  void factor_views(const Opnd &o, View *a, View *b) const {
    const auto &x = nd(o.node);
    const int rows = x.r1 - x.r0, cols = x.c1 - x.c0;
    *a = View{x.off_a + (o.r0 - x.r0), o.r1 - o.r0, cap, 1, rows, -1, x.slot};
    *b = View{x.off_b + (o.c0 - x.c0), o.c1 - o.c0, cap, 1, cols, -1, x.slot};
  }

  int64_t emit(int kind, bool defer, int64_t payload, Span<Iv> reads, Span<Iv> writes, Span<int64_t> tin,
               Span<int64_t> tout, int ff, double fc, int64_t fl) {
    Op o;
    o.kind = kind;
    o.defer = defer;
    o.payload = payload;
    o.r_begin = (int64_t)ivs.size();
    ivs.insert(ivs.end(), reads.begin(), reads.end());
    o.r_end = o.w_begin = (int64_t)ivs.size();
    ivs.insert(ivs.end(), writes.begin(), writes.end());
    o.w_end = (int64_t)ivs.size();
    o.ti_begin = (int64_t)tids.size();
    tids.insert(tids.end(), tin.begin(), tin.end());
    o.ti_end = o.to_begin = (int64_t)tids.size();
    tids.insert(tids.end(), tout.begin(), tout.end());
    o.to_end = (int64_t)tids.size();
    o.flop_f = ff;
    o.flop_c = fc;
    o.flop_log = fl;
    ops.push_back(o);
    return (int64_t)ops.size() - 1;
  }

  // ---------------------------------------------------------- term emitters
  void terms_matmat(std::vector<Term> &ts, const View &dst, const Opnd &op, const View &x, double alpha) {
    if (part(op)) {
      const auto &p = nd(op.node);
      for (int r = 0; r < p.nr; ++r)
        for (int c = 0; c < p.nc; ++c) {
          const int ch = child(op.node, r, c);
          const auto &q = nd(ch);
          terms_matmat(ts, dst.rows_slice(q.r0 - p.r0, q.r1 - p.r0), whole(ch), x.rows_slice(q.c0 - p.c0, q.c1 - p.c0), alpha);
        }
    } else if (rk(op)) {
      View fa, fb;
      factor_views(op, &fa, &fb);
      ts.push_back(Term{2, dst, fa, fb.T(), x, alpha, 0});
    } else {
      ts.push_back(Term{1, dst, dense_view(op), NULLV, x, alpha, 0});
    }
  }
  void terms_tmatmat(std::vector<Term> &ts, const View &dst, const Opnd &op, const View &x, double alpha) {
    if (part(op)) {
      const auto &p = nd(op.node);
      for (int r = 0; r < p.nr; ++r)
        for (int c = 0; c < p.nc; ++c) {
          const int ch = child(op.node, r, c);
          const auto &q = nd(ch);
          terms_tmatmat(ts, dst.rows_slice(q.c0 - p.c0, q.c1 - p.c0), whole(ch), x.rows_slice(q.r0 - p.r0, q.r1 - p.r0), alpha);
        }
    } else if (rk(op)) {
      View fa, fb;
      factor_views(op, &fa, &fb);
      ts.push_back(Term{2, dst, fb, fa.T(), x, alpha, 0});
    } else {
      ts.push_back(Term{1, dst, dense_view(op).T(), NULLV, x, alpha, 0});
    }
  }
  void terms_rmatmat(std::vector<Term> &ts, const View &dst, const View &x, const Opnd &op, double alpha) {
    if (part(op)) {
      const auto &p = nd(op.node);
      for (int r = 0; r < p.nr; ++r)
        for (int c = 0; c < p.nc; ++c) {
          const int ch = child(op.node, r, c);
          const auto &q = nd(ch);
          terms_rmatmat(ts, dst.cols_slice(q.c0 - p.c0, q.c1 - p.c0), x.cols_slice(q.r0 - p.r0, q.r1 - p.r0), whole(ch), alpha);
        }
    } else if (rk(op)) {
      View fa, fb;
      factor_views(op, &fa, &fb);
      ts.push_back(Term{2, dst, x, fa, fb.T(), alpha, 1});
    } else {
      ts.push_back(Term{1, dst, x, NULLV, dense_view(op), alpha, 0});
    }
  }

  int64_t gemm_op(const std::vector<Term> &ts, Span<Iv> reads, Span<Iv> writes, int ff, double fc, int log_slot,
                  bool defer, Span<int64_t> tout, Span<int64_t> tin, bool splittable = true) {
    int64_t lg = -1;
    if (ff == F_LIN || ff == F_QUAD) lg = log();
    GemmP g{(int64_t)terms.size(), (int64_t)ts.size(), (int)lg, log_slot, splittable};
    terms.insert(terms.end(), ts.begin(), ts.end());
    gemm.push_back(g);
    return emit(2, defer, (int64_t)gemm.size() - 1, reads, writes, tin, tout, ff, fc, lg);
  }

  // ---------------------------------------------------------- truncation
  bool rkt_op(int mode, const std::vector<Pair> &ps, int m, int n, int out_node, Span<Iv> reads, Span<int64_t> tin,
              bool defer, bool has_flop, double flop_mn, Pair *res) {
    int kb = 0;
    for (const auto &p : ps) kb += p.a.cols;
    std::vector<int64_t> tout;
    std::vector<Iv> writes;
    int64_t out_a, out_b;
    int slot;
    if (out_node < 0) {
      int64_t base;
      const int64_t t = temp((int64_t)(m + n) * cap, &base);
      slot = rank_slot();
      out_a = base;
      out_b = base + (int64_t)m * cap;
      tout.push_back(t);
      writes.push_back(temp_res(t));
      res->a = View{out_a, m, cap, 1, m, -1, slot};
      res->b = View{out_b, n, cap, 1, n, -1, slot};
      res->sign = 1.0;
      res->roff = res->coff = 0;
    } else {
      const auto &x = nd(out_node);
      out_a = x.off_a;
      out_b = x.off_b;
      slot = x.slot;
      writes.push_back(Iv{x.lo, x.hi});
    }
    const int64_t wsn = rk_ws_doubles(m, n, kb);
    int64_t ws = 0;
    if (wsn) {
      const int64_t tw = temp(wsn, &ws);
      tout.push_back(tw);
    }
    const int64_t lg = log(3);
    RktP r;
    r.mode = mode;
    r.pb = (int64_t)parts.size();
    r.pn = (int64_t)ps.size();
    parts.insert(parts.end(), ps.begin(), ps.end());
    r.m = m;
    r.n = n;
    r.cap = cap;
    r.slot = slot;
    r.log = (int)lg;
    r.out_a = out_a;
    r.out_b = out_b;
    r.ws = ws;
    r.kb = kb;
    rkt.push_back(r);
    emit(3, defer, (int64_t)rkt.size() - 1, reads, writes, tin, tout, has_flop ? F_RKUPD : F_STATIC,
         has_flop ? flop_mn : 0.0, has_flop ? lg : -1);
    return out_node < 0;
  }

  // hoisted inner product W = fa_b[mid]^T fb_a[mid] shared by all leaves of a
  // partitioned destination (see planner.py: hoist_inner)
  struct Hoist {
    bool on = false;
    View W;
    int64_t t = -1;
  };

  Hoist hoist_inner(const Opnd &a, const Opnd &b) {
    View fa_a, fb_a, fa_b, fb_b;
    factor_views(a, &fa_a, &fb_a);
    factor_views(b, &fa_b, &fb_b);
    int64_t base;
    const int64_t t = temp((int64_t)cap * cap, &base);
    Hoist h;
    h.on = true;
    h.t = t;
    h.W = View{base, cap, cap, 1, cap, fa_b.cdyn, fa_a.cdyn};
    std::vector<Term> ts{Term{0, h.W, NULLV, NULLV, NULLV, 0.0, 0}, Term{1, h.W, fa_b.T(), NULLV, fb_a, 1.0, 0}};
    gemm_op(ts, {res(a), res(b)}, {temp_res(t)}, F_STATIC, 0.0, -1, false, {t}, {});
    return h;
  }

  // ---------------------------------------------------------- products
  Pair product(const Opnd &a, const Opnd &b, const std::vector<Iv> *ctx, std::vector<Iv> *reads_out,
               std::vector<int64_t> *tps, const Hoist *hw = nullptr) {
    std::vector<Iv> reads = ctx ? *ctx : std::vector<Iv>{res(a), res(b)};
    *reads_out = reads;
    tps->clear();
    if (!part(a) && rk(a)) {
      View fa, fb;
      factor_views(a, &fa, &fb);
      const int n = b.c1 - b.c0;
      int64_t base;
      const int64_t t = temp((int64_t)n * cap, &base);
      const View T{base, n, cap, 1, n, -1, fa.cdyn};
      std::vector<Term> ts{Term{0, T, NULLV, NULLV, NULLV, 0.0, 0}};
      std::vector<int64_t> tin;
      if (hw && hw->on) {
        View fab, fbb;
        factor_views(b, &fab, &fbb);
        ts.push_back(Term{1, T, fbb, NULLV, hw->W, 1.0, 0});
        tin.push_back(hw->t);
      } else {
        terms_tmatmat(ts, T, b, fb, 1.0);
      }
      gemm_op(ts, reads, {temp_res(t)}, F_STATIC, 0.0, -1, true, {t}, tin);
      tps->push_back(t);
      return Pair{fa, T, 1.0, 0, 0};
    }
    if (!part(b) && rk(b)) {
      View fa, fb;
      factor_views(b, &fa, &fb);
      const int m = a.r1 - a.r0;
      int64_t base;
      const int64_t t = temp((int64_t)m * cap, &base);
      const View T{base, m, cap, 1, m, -1, fa.cdyn};
      std::vector<Term> ts{Term{0, T, NULLV, NULLV, NULLV, 0.0, 0}};
      terms_matmat(ts, T, a, fa, 1.0);
      gemm_op(ts, reads, {temp_res(t)}, F_STATIC, 0.0, -1, true, {t}, {});
      tps->push_back(t);
      return Pair{T, fb, 1.0, 0, 0};
    }
    if (!part(a) && !part(b)) {
      const View av = dense_view(a), bv = dense_view(b);
      const int m = av.rows, kin = av.cols, n = bv.cols;
      Pair p;
      // compress_dense(A @ B) as the narrower of the factor pair (A, B^T) (stacked
      // rank kin) and the formed product (I, D^T) / (D, I) (rank min(m, n)),
      // preferring the block-TSQR pipeline (<= RK_KMAX) over the wide path
      if (kin <= product_pair_max || (std::min(m, n) > product_pair_max && kin <= IDENT)) {
        rkt_op(1, {Pair{av, bv.T(), 1.0, 0, 0}}, m, n, -1, reads, {}, true, false, 0.0, &p);
        tps->push_back(pair_temp(p));
        return p;
      }
      if (std::min(m, n) > IDENT) throw std::runtime_error("dense product exceeds the truncation kernel");
      int64_t base;
      const int64_t t = temp((int64_t)m * n, &base);
      const View D{base, m, n, 1, m, -1, -1};
      std::vector<Term> ts{Term{0, D, NULLV, NULLV, NULLV, 0.0, 0}, Term{1, D, av, NULLV, bv, 1.0, 0}};
      gemm_op(ts, reads, {temp_res(t)}, F_STATIC, 0.0, -1, true, {t}, {});
      Pair part_;
      if (m <= n) part_ = Pair{View{ident_off, m, m, 1, IDENT, -1, -1}, D.T(), 1.0, 0, 0};
      else part_ = Pair{D, View{ident_off, n, n, 1, IDENT, -1, -1}, 1.0, 0, 0};
      rkt_op(1, {part_}, m, n, -1, reads, {t}, true, false, 0.0, &p);
      tps->push_back(pair_temp(p));
      return p;
    }
    std::vector<std::pair<int, int>> rows = part(a) ? row_cuts(a.node) : std::vector<std::pair<int, int>>{{a.r0, a.r1}};
    std::vector<std::pair<int, int>> cols = part(b) ? col_cuts(b.node) : std::vector<std::pair<int, int>>{{b.c0, b.c1}};
    if (part(a) && part(b) && col_cuts(a.node) != row_cuts(b.node))
      throw std::runtime_error("inner partitions of a product do not match");
    std::vector<std::pair<int, int>> mids = part(a) ? col_cuts(a.node) : row_cuts(b.node);
    std::vector<Pair> grid;
    std::vector<std::vector<int64_t>> gtemps;
    for (size_t i = 0; i < rows.size(); ++i) {
      for (size_t j = 0; j < cols.size(); ++j) {
        bool have = false;
        Pair acc;
        std::vector<int64_t> acc_t;
        for (size_t p = 0; p < mids.size(); ++p) {
          const Opnd ap = part(a) ? whole(child(a.node, (int)i, (int)p))
                                  : window(a, rows[i].first, rows[i].second, mids[p].first, mids[p].second);
          const Opnd bp = part(b) ? whole(child(b.node, (int)p, (int)j))
                                  : window(b, mids[p].first, mids[p].second, cols[j].first, cols[j].second);
          std::vector<Iv> rd;
          std::vector<int64_t> tp;
          const Pair pp = product(ap, bp, &reads, &rd, &tp);
          if (!have) {
            acc = pp;
            acc_t = tp;
            have = true;
            continue;
          }
          std::vector<int64_t> tin = acc_t;
          tin.insert(tin.end(), tp.begin(), tp.end());
          Pair out;
          rkt_op(0, {acc, pp}, rows[i].second - rows[i].first, cols[j].second - cols[j].first, -1, reads, tin, false,
                 false, 0.0, &out);
          acc = out;
          acc_t = {pair_temp(out)};
        }
        grid.push_back(acc);
        gtemps.push_back(acc_t);
      }
    }
    if (rows.size() == 1 && cols.size() == 1) {
      *tps = gtemps[0];
      return grid[0];
    }
    const int m = rows.back().second - rows.front().first;
    const int n = cols.back().second - cols.front().first;
    std::vector<Pair> ps;
    std::vector<int64_t> tin;
    for (size_t i = 0; i < rows.size(); ++i)
      for (size_t j = 0; j < cols.size(); ++j) {
        const Pair &acc = grid[i * cols.size() + j];
        ps.push_back(Pair{acc.a, acc.b, acc.sign, rows[i].first - rows[0].first, cols[j].first - cols[0].first});
        const auto &tt = gtemps[i * cols.size() + j];
        tin.insert(tin.end(), tt.begin(), tt.end());
      }
    Pair merged;
    rkt_op(1, ps, m, n, -1, reads, tin, false, false, 0.0, &merged);
    tps->assign(1, pair_temp(merged));
    return merged;
  }

  // ---------------------------------------------------------- update
  void update(const Opnd &c, const Opnd &a, const Opnd &b, const Hoist *hw = nullptr) {
    if (!c.win && nd(c.node).kind == 1) {
      std::vector<Iv> reads;
      std::vector<int64_t> tps;
      const Pair p = product(a, b, nullptr, &reads, &tps, hw);
      const auto &x = nd(c.node);
      const int m = x.r1 - x.r0, n = x.c1 - x.c0;
      View ca, cb;
      factor_views(c, &ca, &cb);
      reads.push_back(res(c));
      Pair dummy;
      rkt_op(0, {Pair{ca, cb, 1.0, 0, 0}, Pair{p.a, p.b, -p.sign, 0, 0}}, m, n, c.node, reads, tps, false, true,
             (double)(m + n), &dummy);
      return;
    }
    const bool cp = part(c), ap = part(a), bp = part(b);
    if (!(cp || ap || bp)) {
      update_dense(c, a, b, hw);
      return;
    }
    Hoist local;
    if (!hw && cp && !ap && !bp && rk(a) && rk(b)) {
      local = hoist_inner(a, b);
      hw = &local;
    }
    std::vector<std::pair<int, int>> rows, cols, mids;
    if (cp) rows = row_cuts(c.node);
    else if (ap) rows = row_cuts(a.node);
    else rows = {{c.r0, c.r1}};
    if (cp) cols = col_cuts(c.node);
    else if (bp) cols = col_cuts(b.node);
    else cols = {{c.c0, c.c1}};
    if (ap && bp && col_cuts(a.node) != row_cuts(b.node))
      throw std::runtime_error("inner partitions of an update do not match");
    if (ap) mids = col_cuts(a.node);
    else if (bp) mids = row_cuts(b.node);
    else mids = {{a.c0, a.c1}};
    for (size_t i = 0; i < rows.size(); ++i)
      for (size_t j = 0; j < cols.size(); ++j) {
        const Opnd cij = cp ? whole(child(c.node, (int)i, (int)j))
                            : window(c, rows[i].first, rows[i].second, cols[j].first, cols[j].second);
        for (size_t p = 0; p < mids.size(); ++p) {
          const Opnd aa = ap ? whole(child(a.node, (int)i, (int)p))
                             : window(a, rows[i].first, rows[i].second, mids[p].first, mids[p].second);
          const Opnd bb = bp ? whole(child(b.node, (int)p, (int)j))
                             : window(b, mids[p].first, mids[p].second, cols[j].first, cols[j].second);
          update(cij, aa, bb, hw);
        }
      }
  }

  void update_dense(const Opnd &c, const Opnd &a, const Opnd &b, const Hoist *hw = nullptr) {
    const View dst = dense_view(c);
    const int m = dst.rows, n = dst.cols;
    const std::vector<Iv> reads{res(a), res(b)};
    const std::vector<Iv> writes{res(c)};
    if (!rk(a) && !rk(b)) {
      const View av = dense_view(a), bv = dense_view(b);
      gemm_op({Term{1, dst, av, NULLV, bv, -1.0, 0}}, reads, writes, F_STATIC, 2.0 * m * n * av.cols, -1, false, {}, {},
              false);
    } else if (rk(a)) {
      View fa, fb;
      factor_views(a, &fa, &fb);
      int64_t base;
      const int64_t t = temp((int64_t)n * cap, &base);
      const View T{base, n, cap, 1, n, -1, fa.cdyn};
      std::vector<Term> ts{Term{0, T, NULLV, NULLV, NULLV, 0.0, 0}};
      std::vector<int64_t> tin;
      if (hw && hw->on) {
        View fab, fbb;
        factor_views(b, &fab, &fbb);
        ts.push_back(Term{1, T, fbb, NULLV, hw->W, 1.0, 0});
        tin.push_back(hw->t);
      } else {
        terms_tmatmat(ts, T, b, fb, 1.0);
      }
      ts.push_back(Term{1, dst, fa, NULLV, T.T(), -1.0, 0});
      gemm_op(ts, reads, writes, F_LIN, 2.0 * (m + n) * n, fa.cdyn, false, {t}, tin, false);
    } else {
      View fa, fb;
      factor_views(b, &fa, &fb);
      int64_t base;
      const int64_t t = temp((int64_t)m * cap, &base);
      const View T{base, m, cap, 1, m, -1, fa.cdyn};
      std::vector<Term> ts{Term{0, T, NULLV, NULLV, NULLV, 0.0, 0}};
      terms_matmat(ts, T, a, fa, 1.0);
      ts.push_back(Term{1, dst, T, NULLV, fb.T(), -1.0, 0});
      gemm_op(ts, reads, writes, F_LIN, 2.0 * (m + n) * m, fa.cdyn, false, {t}, {}, false);
    }
  }

  // ---------------------------------------------------------- trsm
  void trsm_op(const View &t, const View &x, int mode, Span<Iv> reads, Span<Iv> writes,
               double coef, bool dyn) {
    const int64_t lg = dyn ? log() : -1;
    trsm.push_back(TrsmP{t, x, mode, (int)lg});
    emit(1, false, (int64_t)trsm.size() - 1, reads, writes, {}, {}, dyn ? F_LIN : F_STATIC, coef, dyn ? lg : -1);
  }

  void solve_lower(int l, int b) {
    const auto &L = nd(l), &B = nd(b);
    if (L.kind == 0) {
      const View lv = dense_view(whole(l));
      const std::vector<Iv> rd{Iv{L.lo, L.hi}}, wr{Iv{B.lo, B.hi}};
      const int lr = L.r1 - L.r0;
      if (B.kind == 0) {
        trsm_op(lv, dense_view(whole(b)), 0, rd, wr, (double)lr * lr * (B.c1 - B.c0), false);
      } else if (B.kind == 1) {
        View fa, fb;
        factor_views(whole(b), &fa, &fb);
        trsm_op(lv, fa, 0, rd, wr, (double)lr * lr, true);
      } else {
        throw std::runtime_error("dense factor against partitioned right-hand side");
      }
      return;
    }
    if (B.kind == 2) {
      const int nr = L.nr, nc = B.nc;
      for (int i = 0; i < nr; ++i) {
        for (int p = 0; p < i; ++p)
          for (int j = 0; j < nc; ++j)
            update(whole(child(b, i, j)), whole(child(l, i, p)), whole(child(b, p, j)));
        for (int j = 0; j < nc; ++j) solve_lower(child(l, i, i), child(b, i, j));
      }
      return;
    }
    lower_panel(l, b, B.r0, B.r1);
  }

  View panel_view(int bleaf, int part_, int axis, int lo, int hi) const {
    const auto &B = nd(bleaf);
    if (part_ == 0) {
      const View v = dense_view(whole(bleaf));
      return axis == 0 ? v.rows_slice(lo - B.r0, hi - B.r0) : v.cols_slice(lo - B.c0, hi - B.c0);
    }
    View fa, fb;
    factor_views(whole(bleaf), &fa, &fb);
    if (part_ == 1) return fa.rows_slice(lo - B.r0, hi - B.r0);
    return fb.rows_slice(lo - B.c0, hi - B.c0);
  }

  void lower_panel(int l, int bleaf, int lo, int hi) {
    const auto &B = nd(bleaf);
    const int part_ = B.kind == 0 ? 0 : 1;
    const auto &L = nd(l);
    const std::vector<Iv> rd{Iv{L.lo, L.hi}}, wr{Iv{B.lo, B.hi}};
    if (L.kind == 0) {
      const View x = panel_view(bleaf, part_, 0, lo, hi);
      const bool dyn = part_ == 1;
      const int lr = L.r1 - L.r0;
      trsm_op(dense_view(whole(l)), x, 0, rd, wr, (double)lr * lr * (dyn ? 1 : x.cols), dyn);
      return;
    }
    const auto cuts = row_cuts(l);
    for (size_t i = 0; i < cuts.size(); ++i) {
      for (size_t p = 0; p < i; ++p) {
        const int lip = child(l, (int)i, (int)p);
        const View dst = panel_view(bleaf, part_, 0, cuts[i].first, cuts[i].second);
        const View src = panel_view(bleaf, part_, 0, cuts[p].first, cuts[p].second);
        std::vector<Term> ts;
        terms_matmat(ts, dst, whole(lip), src, -1.0);
        const std::vector<Iv> rl{Iv{nd(lip).lo, nd(lip).hi}};
        if (part_ == 1)
          gemm_op(ts, rl, wr, F_LIN, 2.0 * dst.rows * src.rows, dst.cdyn, false, {}, {});
        else
          gemm_op(ts, rl, wr, F_STATIC, 2.0 * dst.rows * dst.cols * src.rows, -1, false, {}, {});
      }
      lower_panel(child(l, (int)i, (int)i), bleaf, cuts[i].first, cuts[i].second);
    }
  }

  void solve_upper(int b, int u) {
    const auto &U = nd(u), &B = nd(b);
    if (U.kind == 0) {
      const View uv = dense_view(whole(u));
      const std::vector<Iv> rd{Iv{U.lo, U.hi}}, wr{Iv{B.lo, B.hi}};
      const int ur = U.r1 - U.r0;
      if (B.kind == 0) {
        trsm_op(uv, dense_view(whole(b)), 1, rd, wr, (double)ur * ur * (B.r1 - B.r0), false);
      } else if (B.kind == 1) {
        View fa, fb;
        factor_views(whole(b), &fa, &fb);
        trsm_op(uv, fb.T(), 1, rd, wr, (double)ur * ur, true);
      } else {
        throw std::runtime_error("dense factor against partitioned right-hand side");
      }
      return;
    }
    if (B.kind == 2) {
      const int nc = U.nc, nr = B.nr;
      for (int j = 0; j < nc; ++j) {
        for (int p = 0; p < j; ++p)
          for (int i = 0; i < nr; ++i) update(whole(child(b, i, j)), whole(child(b, i, p)), whole(child(u, p, j)));
        for (int i = 0; i < nr; ++i) solve_upper(child(b, i, j), child(u, j, j));
      }
      return;
    }
    upper_panel(b, u, B.c0, B.c1);
  }

  void upper_panel(int bleaf, int u, int lo, int hi) {
    const auto &B = nd(bleaf), &U = nd(u);
    const bool dense = B.kind == 0;
    const int part_ = dense ? 0 : 2, axis = dense ? 1 : 0;
    const std::vector<Iv> rd{Iv{U.lo, U.hi}}, wr{Iv{B.lo, B.hi}};
    if (U.kind == 0) {
      const View x = panel_view(bleaf, part_, axis, lo, hi);
      const int ur = U.r1 - U.r0;
      if (dense) trsm_op(dense_view(whole(u)), x, 1, rd, wr, (double)ur * ur * x.rows, false);
      else trsm_op(dense_view(whole(u)), x.T(), 1, rd, wr, (double)ur * ur, true);
      return;
    }
    const auto cuts = col_cuts(u);
    for (size_t j = 0; j < cuts.size(); ++j) {
      for (size_t p = 0; p < j; ++p) {
        const int upj = child(u, (int)p, (int)j);
        const View dst = panel_view(bleaf, part_, axis, cuts[j].first, cuts[j].second);
        const View src = panel_view(bleaf, part_, axis, cuts[p].first, cuts[p].second);
        std::vector<Term> ts;
        const std::vector<Iv> ru{Iv{nd(upj).lo, nd(upj).hi}};
        if (dense) {
          terms_rmatmat(ts, dst, src, whole(upj), -1.0);
          gemm_op(ts, ru, wr, F_STATIC, 2.0 * dst.rows * dst.cols * src.cols, -1, false, {}, {}, false);
        } else {
          terms_tmatmat(ts, dst, whole(upj), src, -1.0);
          gemm_op(ts, ru, wr, F_QUAD, 2.0 * dst.rows, dst.cdyn, false, {}, {});
        }
      }
      upper_panel(bleaf, child(u, (int)j, (int)j), cuts[j].first, cuts[j].second);
    }
  }

  void factor(int h) {
    const auto &H = nd(h);
    if (H.kind == 0) {
      if (H.r1 - H.r0 != H.c1 - H.c0) throw std::runtime_error("LU requires a square block");
      const int idx = (int)lu_ops.size();
      lu_nodes.push_back(h);
      getrf.push_back(GetrfP{dense_view(whole(h)), (int)ops.size(), idx});
      const double n = H.r1 - H.r0;
      lu_ops.push_back(emit(0, false, (int64_t)getrf.size() - 1, {}, {Iv{H.lo, H.hi}}, {}, {}, F_STATIC,
                            2.0 / 3.0 * (n * n * n), -1));
      return;
    }
    if (H.kind == 1) throw std::runtime_error("diagonal block is low-rank; expected dense");
    if (H.nr != H.nc) throw std::runtime_error("LU requires a square grid");
    const int nb = H.nr;
    for (int k = 0; k < nb; ++k) {
      factor(child(h, k, k));
      for (int j = k + 1; j < nb; ++j) solve_lower(child(h, k, k), child(h, k, j));
      for (int i = k + 1; i < nb; ++i) solve_upper(child(h, i, k), child(h, k, k));
      for (int i = k + 1; i < nb; ++i)
        for (int j = k + 1; j < nb; ++j) update(whole(child(h, i, j)), whole(child(h, i, k)), whole(child(h, k, j)));
    }
  }

  // vector solves (forward = reference panel route; backward = restated)
  void vec_lower(int l, const View &x, int base, const Iv &res_) {
    const auto &L = nd(l);
    if (L.kind == 0) {
      trsm_op(dense_view(whole(l)), x, 0, {Iv{L.lo, L.hi}}, {res_}, 0.0, false);
      return;
    }
    const auto cuts = row_cuts(l);
    for (size_t i = 0; i < cuts.size(); ++i) {
      for (size_t p = 0; p < i; ++p) {
        std::vector<Term> ts;
        const int lip = child(l, (int)i, (int)p);
        terms_matmat(ts, x.rows_slice(cuts[i].first - base, cuts[i].second - base), whole(lip),
                     x.rows_slice(cuts[p].first - base, cuts[p].second - base), -1.0);
        gemm_op(ts, {Iv{nd(lip).lo, nd(lip).hi}}, {res_}, F_STATIC, 0.0, -1, false, {}, {});
      }
      vec_lower(child(l, (int)i, (int)i), x.rows_slice(cuts[i].first - base, cuts[i].second - base), cuts[i].first,
                res_);
    }
  }
  void vec_upper(int u, const View &x, int base, const Iv &res_) {
    const auto &U = nd(u);
    if (U.kind == 0) {
      trsm_op(dense_view(whole(u)), x, 2, {Iv{U.lo, U.hi}}, {res_}, 0.0, false);
      return;
    }
    const auto cuts = row_cuts(u);
    const int nb = (int)cuts.size();
    for (int i = nb - 1; i >= 0; --i) {
      for (int p = i + 1; p < nb; ++p) {
        std::vector<Term> ts;
        const int uip = child(u, i, p);
        terms_matmat(ts, x.rows_slice(cuts[i].first - base, cuts[i].second - base), whole(uip),
                     x.rows_slice(cuts[p].first - base, cuts[p].second - base), -1.0);
        gemm_op(ts, {Iv{nd(uip).lo, nd(uip).hi}}, {res_}, F_STATIC, 0.0, -1, false, {}, {});
      }
      vec_upper(child(u, i, i), x.rows_slice(cuts[i].first - base, cuts[i].second - base), cuts[i].first, res_);
    }
  }

  // products with the H-matrix or its stored factors: y += op(h) x, one chain
  // of terms in the reference's recursion order (hmatrix.py:188-200,
  // hlu.py:720-767); tri = 0 full, 1 unit lower, 2 upper
  void terms_tri(std::vector<Term> &ts, int h, const View &y, const View &x, int tri) {
    const auto &H = nd(h);
    if (H.kind == 0) {
      ts.push_back(Term{1, y, dense_view(whole(h)), NULLV, x, 1.0, tri == 1 ? 2 : 1});
      return;
    }
    if (H.kind != 2) throw std::runtime_error("factored matrix has a low-rank diagonal block");
    for (int i = 0; i < H.nr; ++i)
      for (int j = 0; j < H.nc; ++j) {
        const int ch = child(h, i, j);
        const auto &q = nd(ch);
        const View ys = y.rows_slice(q.r0 - H.r0, q.r1 - H.r0), xs = x.rows_slice(q.c0 - H.c0, q.c1 - H.c0);
        if (tri == 1 ? j < i : j > i) terms_matmat(ts, ys, whole(ch), xs, 1.0);
        else if (j == i) terms_tri(ts, ch, ys, xs, tri);
      }
  }
  void matvec(int h, const View &x, const View &y, const Iv &xr, const Iv &yr, int tri) {
    std::vector<Term> ts;
    if (tri == 0) terms_matmat(ts, y, whole(h), x, 1.0);
    else terms_tri(ts, h, y, x, tri);
    gemm_op(ts, {Iv{nd(h).lo, nd(h).hi}, xr}, {yr}, F_STATIC, 0.0, -1, false, {}, {});
  }

  // ---------------------------------------------------------- schedule
  std::vector<int64_t> levels;
  // owner-computes sharding: ranks executing every op, and the
  // slot exchange records (include/hlu_plan.h hlu_xfer)
  int nranks = 1, my_rank = 0;
  const int32_t *slot_owner = nullptr;  // per skeleton slot
  std::vector<uint64_t> op_mask;
  std::vector<hlu_xfer> o_xfer;
  std::vector<int64_t> toffs;
  std::vector<int64_t> tbirth;  // level of each temp's producer
  std::vector<int64_t> reuse_from;  // temp whose arena block a temp takes over (-1: fresh)
  // Cross-class waits (two-chain schedule): the dense chain (getrf / trsm /
  // gemm) and the truncation chain each run their levels in order on their own
  // stream; wait_d[l] / wait_r[l] = the last level of the OTHER chain that the
  // level-l launches of this chain must wait for (-1: none).
  std::vector<int32_t> wait_d, wait_r;
  bool waits_ok = false;
  int64_t arena = 0;

  // Hazard state: slots in segment trees (reads can span whole partitioned
  // operands, writes are single leaves or temps), temps in flat arrays.
  struct MaxTree {  // point assign, range max
    int64_t n = 1;
    std::vector<int64_t> t;
    void init(int64_t m) { while (n < m) n <<= 1; t.assign(2 * n, -1); }
    void set(int64_t i, int64_t v) { i += n; t[i] = v; for (i >>= 1; i; i >>= 1) t[i] = std::max(t[2 * i], t[2 * i + 1]); }
    int64_t query(int64_t lo, int64_t hi) const {
      int64_t r = -1;
      for (lo += n, hi += n; lo < hi; lo >>= 1, hi >>= 1) {
        if (lo & 1) r = std::max(r, t[lo++]);
        if (hi & 1) r = std::max(r, t[--hi]);
      }
      return r;
    }
  };
  struct TagTree {  // range chmax, point query
    int64_t n = 1;
    std::vector<int64_t> t;
    void init(int64_t m) { while (n < m) n <<= 1; t.assign(2 * n, -1); }
    void chmax(int64_t lo, int64_t hi, int64_t v) {
      for (lo += n, hi += n; lo < hi; lo >>= 1, hi >>= 1) {
        if (lo & 1) { t[lo] = std::max(t[lo], v); ++lo; }
        if (hi & 1) { --hi; t[hi] = std::max(t[hi], v); }
      }
    }
    int64_t get(int64_t i) const {
      int64_t r = -1;
      for (i += n; i; i >>= 1) r = std::max(r, t[i]);
      return r;
    }
  };

  void assign_levels() {
    const int64_t nt = (int64_t)temp_size.size();
    MaxTree lw;
    TagTree lr;
    lw.init(std::max<int64_t>(nslots, 1));
    lr.init(std::max<int64_t>(nslots, 1));
    // point values of slots are also kept flat for the single-slot fast path
    std::vector<int64_t> lw_s(nslots, -1);
    std::vector<int64_t> lwT(nt, -1), lrT(nt, -1);
    levels.assign(ops.size(), 0);
    std::vector<std::pair<int64_t, int64_t>> pending;
    auto constraint = [&](const Op &o) {
      int64_t c = 0;
      for (int64_t i = o.r_begin; i < o.r_end; ++i) {
        const Iv &v = ivs[i];
        if (v.lo >= nslots) c = std::max(c, lwT[v.lo - nslots] + 1);
        else if (v.hi - v.lo == 1) c = std::max(c, lw_s[v.lo] + 1);
        else c = std::max(c, lw.query(v.lo, v.hi) + 1);
      }
      for (int64_t i = o.ti_begin; i < o.ti_end; ++i) c = std::max(c, lwT[tids[i]] + 1);
      for (int64_t i = o.w_begin; i < o.w_end; ++i) {
        const Iv &v = ivs[i];
        if (v.lo >= nslots) {
          const int64_t t = v.lo - nslots;
          c = std::max(c, std::max(lwT[t], lrT[t]) + 1);
        } else {
          for (int64_t s = v.lo; s < v.hi; ++s) c = std::max(c, std::max(lw_s[s], lr.get(s)) + 1);
        }
      }
      return c;
    };
    auto commit = [&](const Op &o, int64_t lv) {
      for (int64_t i = o.r_begin; i < o.r_end; ++i) {
        const Iv &v = ivs[i];
        if (v.lo >= nslots) lrT[v.lo - nslots] = std::max(lrT[v.lo - nslots], lv);
        else lr.chmax(v.lo, v.hi, lv);
      }
      for (int64_t i = o.ti_begin; i < o.ti_end; ++i) lrT[tids[i]] = std::max(lrT[tids[i]], lv);
      for (int64_t i = o.w_begin; i < o.w_end; ++i) {
        const Iv &v = ivs[i];
        if (v.lo >= nslots) {
          lwT[v.lo - nslots] = lv;
        } else {
          for (int64_t s = v.lo; s < v.hi; ++s) {
            lw_s[s] = lv;
            lw.set(s, lv);
          }
        }
      }
    };
    for (size_t i = 0; i < ops.size(); ++i) {
      const Op &o = ops[i];
      int64_t c = constraint(o);
      if (o.defer) {
        pending.push_back({(int64_t)i, c});
        continue;
      }
      if (!pending.empty()) {
        int64_t mx = 0;
        for (auto &pp : pending) mx = std::max(mx, pp.second);
        c = std::max(c, mx + 1);
        for (auto &pp : pending) {
          levels[pp.first] = c - 1;
          commit(ops[pp.first], c - 1);
        }
        pending.clear();
        c = std::max(c, constraint(o));
      }
      levels[i] = c;
      commit(o, c);
    }
    for (auto &pp : pending) {
      levels[pp.first] = pp.second;
      commit(ops[pp.first], pp.second);
    }
  }

  // ---------------------------------------------------------- DAG schedule
  // (hlu_plan_build_dag) The level schedule pays the slowest op of every level.
  // The DAG schedule drops the barriers: a hazard sweep in model time (per-op
  // latency model op_cost_ns) gives every op a start time; ops whose start
  // falls in the same dag_slot_ns window and that share a kernel class form one
  // launch, and every launch lists the launches it depends on (RAW / WAR / WAW
  // on skeleton slots and temps, arena-block reuse).  The runtime replays the
  // launch DAG as one CUDA graph whose edges are exactly these dependencies:
  // the GPU analogue of the paper's task DAG with fine-grained region
  // dependencies instead of a wavefront per level.
  // `levels` then holds the launch-group keys (time slot, class) in
  // topological order; every hazard predecessor of an op has a smaller key.
  int64_t dag_slot_ns = 0;  // 0: level schedule
  std::vector<int64_t> op_start, op_ready;  // model ns: start, and when dependants may start
  std::vector<int64_t> dag_ptr;             // per launch: [dag_ptr[l], dag_ptr[l+1]) into dag_idx
  std::vector<int32_t> dag_idx;             // predecessor launches
  std::vector<int64_t> dag_slack;           // per launch: model-time slack (ns)
  std::vector<int32_t> op_rec[2];           // launch record(s) holding each op (-1: none)

  int rkt_class(const RktP &r) const {
    if (r.pn > 2) return 2;                        // merges: stacked rank usually > 32
    return std::max(r.m, r.n) <= 64 ? 0 : 1;       // register warp path / CTA path
  }

  void assign_slots() {
    const int64_t D = dag_slot_ns;
    const int64_t nt = (int64_t)temp_size.size();
    MaxTree lw;
    TagTree lr;
    lw.init(std::max<int64_t>(nslots, 1));
    lr.init(std::max<int64_t>(nslots, 1));
    std::fill(lw.t.begin(), lw.t.end(), 0);
    std::fill(lr.t.begin(), lr.t.end(), 0);
    std::vector<int64_t> lw_s(nslots, 0), lwT(nt, 0), lrT(nt, 0);
    op_start.assign(ops.size(), 0);
    op_ready.assign(ops.size(), 0);
    auto constraint = [&](const Op &o) {
      int64_t c = 0;
      for (int64_t i = o.r_begin; i < o.r_end; ++i) {
        const Iv &v = ivs[i];
        if (v.lo >= nslots) c = std::max(c, lwT[v.lo - nslots]);
        else if (v.hi - v.lo == 1) c = std::max(c, lw_s[v.lo]);
        else c = std::max(c, lw.query(v.lo, v.hi));
      }
      for (int64_t i = o.ti_begin; i < o.ti_end; ++i) c = std::max(c, lwT[tids[i]]);
      for (int64_t i = o.w_begin; i < o.w_end; ++i) {
        const Iv &v = ivs[i];
        if (v.lo >= nslots) {
          const int64_t t = v.lo - nslots;
          c = std::max(c, std::max(lwT[t], lrT[t]));
        } else {
          for (int64_t s = v.lo; s < v.hi; ++s) c = std::max(c, std::max(lw_s[s], lr.get(s)));
        }
      }
      return c;
    };
    auto commit = [&](const Op &o, int64_t rd) {
      for (int64_t i = o.r_begin; i < o.r_end; ++i) {
        const Iv &v = ivs[i];
        if (v.lo >= nslots) lrT[v.lo - nslots] = std::max(lrT[v.lo - nslots], rd);
        else lr.chmax(v.lo, v.hi, rd);
      }
      for (int64_t i = o.ti_begin; i < o.ti_end; ++i) lrT[tids[i]] = std::max(lrT[tids[i]], rd);
      for (int64_t i = o.w_begin; i < o.w_end; ++i) {
        const Iv &v = ivs[i];
        if (v.lo >= nslots) {
          lwT[v.lo - nslots] = rd;
        } else {
          for (int64_t s = v.lo; s < v.hi; ++s) {
            lw_s[s] = rd;
            lw.set(s, rd);
          }
        }
      }
    };
    auto place = [&](size_t i, int64_t st) {
      op_start[i] = st;
      op_ready[i] = std::max(st + op_cost_ns(ops[i]), (st / D + 1) * D);
    };
    std::vector<int64_t> pending;
    for (size_t i = 0; i < ops.size(); ++i) {
      const Op &o = ops[i];
      if (o.defer) {  // a temp producer: placed as late as its consumer allows (below)
        pending.push_back((int64_t)i);
        continue;
      }
      if (!pending.empty()) {
        // as-soon-as-possible pass over the pending producers (they write fresh
        // temps only; the provisional temp times let them see one another) ...
        int64_t last = 0;
        for (int64_t p : pending) {
          const Op &q = ops[p];
          place((size_t)p, constraint(q));
          for (int64_t k = q.w_begin; k < q.w_end; ++k)
            if (ivs[k].lo >= nslots) lwT[ivs[k].lo - nslots] = op_ready[p];
          last = std::max(last, op_ready[p]);
        }
        // ... then all of them later by whole slots, to end just before the consumer starts
        const int64_t c = constraint(o);
        const int64_t delay = std::max<int64_t>(0, (c - last) / D * D);
        for (int64_t p : pending) {
          op_start[p] += delay;
          op_ready[p] += delay;
          commit(ops[p], op_ready[p]);
        }
        pending.clear();
      }
      place(i, constraint(o));
      commit(o, op_ready[i]);
    }
    for (int64_t p : pending) {
      place((size_t)p, constraint(ops[p]));
      commit(ops[p], op_ready[p]);
    }
    // launch-group keys: (time slot, class), compressed to consecutive ids
    levels.assign(ops.size(), 0);
    std::vector<int64_t> keys(ops.size());
    for (size_t i = 0; i < ops.size(); ++i) {
      const int sub = ops[i].kind == 3 ? rkt_class(rkt[ops[i].payload]) : 0;
      keys[i] = op_start[i] / D * 4 + sub;
    }
    std::vector<int64_t> uniq(keys);
    std::sort(uniq.begin(), uniq.end());
    uniq.erase(std::unique(uniq.begin(), uniq.end()), uniq.end());
    for (size_t i = 0; i < ops.size(); ++i)
      levels[i] = std::lower_bound(uniq.begin(), uniq.end(), keys[i]) - uniq.begin();
  }

  // Launch-level dependency lists of the DAG schedule (after pack() filled
  // op_rec): a second hazard sweep in program order that tracks, per skeleton
  // slot and temp, the last writer op and the launches that read it since;
  // a temp taking over an arena block waits for every launch that touched the
  // block's previous holder.
  void compute_dag_deps(int64_t nlaunch) {
    const int64_t nt = (int64_t)temp_size.size();
    struct Node {
      int32_t launch, next;
    };
    std::vector<Node> pool;
    pool.reserve(ops.size() * 2);
    std::vector<int32_t> w_s(nslots, -1), w_t(nt, -1);        // last writer op
    std::vector<int32_t> rd_s(nslots, -1), rd_t(nt, -1);      // readers since (launch lists)
    std::vector<int32_t> touch_t(nt, -1);                     // every launch that touched a temp
    std::vector<int32_t> first_t(nt, -1);                     // first op touching a temp
    std::vector<int64_t> e_ptr(ops.size() + 1, 0);
    std::vector<int32_t> e_idx;
    e_idx.reserve(ops.size() * 4);
    auto push = [&](int32_t &head, int32_t launch) {
      if (launch < 0) return;
      if (head >= 0 && pool[head].launch == launch) return;
      pool.push_back(Node{launch, head});
      head = (int32_t)pool.size() - 1;
    };
    auto add_op = [&](int32_t p) {
      if (p < 0) return;
      for (int k = 0; k < 2; ++k)
        if (op_rec[k][p] >= 0) e_idx.push_back(op_rec[k][p]);
    };
    auto add_list = [&](int32_t head) {
      for (int32_t h = head; h >= 0; h = pool[h].next) e_idx.push_back(pool[h].launch);
    };
    for (size_t i = 0; i < ops.size(); ++i) {
      const Op &o = ops[i];
      // the first op (program order) that touches a temp: every other toucher
      // follows it through a RAW / WAW hazard, so the hand-over of an arena
      // block only has to hold this op back (edges added after the sweep: the
      // previous holder's users may come later in program order)
      auto first_touch = [&](int64_t t) {
        if (first_t[t] < 0) first_t[t] = (int32_t)i;
      };
      for (int64_t k = o.r_begin; k < o.r_end; ++k) {
        const Iv &v = ivs[k];
        if (v.lo >= nslots) add_op(w_t[v.lo - nslots]), first_touch(v.lo - nslots);
        else
          for (int64_t s = v.lo; s < v.hi; ++s) add_op(w_s[s]);
      }
      for (int64_t k = o.ti_begin; k < o.ti_end; ++k) add_op(w_t[tids[k]]), first_touch(tids[k]);
      for (int64_t k = o.to_begin; k < o.to_end; ++k) first_touch(tids[k]);
      for (int64_t k = o.w_begin; k < o.w_end; ++k) {
        const Iv &v = ivs[k];
        if (v.lo >= nslots) {
          const int64_t t = v.lo - nslots;
          first_touch(t);
          add_op(w_t[t]);
          add_list(rd_t[t]);
        } else {
          for (int64_t s = v.lo; s < v.hi; ++s) {
            add_op(w_s[s]);
            add_list(rd_s[s]);
          }
        }
      }
      e_ptr[i + 1] = (int64_t)e_idx.size();
      // commit
      for (int k2 = 0; k2 < 2; ++k2) {
        const int32_t me = op_rec[k2][i];
        if (me < 0) continue;
        for (int64_t k = o.r_begin; k < o.r_end; ++k) {
          const Iv &v = ivs[k];
          if (v.lo >= nslots) push(rd_t[v.lo - nslots], me), push(touch_t[v.lo - nslots], me);
          else
            for (int64_t s = v.lo; s < v.hi; ++s) push(rd_s[s], me);
        }
        for (int64_t k = o.ti_begin; k < o.ti_end; ++k) push(rd_t[tids[k]], me), push(touch_t[tids[k]], me);
        for (int64_t k = o.to_begin; k < o.to_end; ++k) push(touch_t[tids[k]], me);
        for (int64_t k = o.w_begin; k < o.w_end; ++k)
          if (ivs[k].lo >= nslots) push(touch_t[ivs[k].lo - nslots], me);
      }
      for (int64_t k = o.w_begin; k < o.w_end; ++k) {
        const Iv &v = ivs[k];
        if (v.lo >= nslots) {
          w_t[v.lo - nslots] = (int32_t)i;
          rd_t[v.lo - nslots] = -1;
        } else {
          for (int64_t s = v.lo; s < v.hi; ++s) w_s[s] = (int32_t)i, rd_s[s] = -1;
        }
      }
    }
    // arena-block hand-over: the first op of a temp waits for every launch that
    // touched the block's previous holder
    std::vector<std::pair<int32_t, int32_t>> extra;  // (op, predecessor launch)
    for (int64_t t = 0; t < nt; ++t) {
      if (first_t[t] < 0 || reuse_from[t] < 0) continue;
      for (int32_t h = touch_t[reuse_from[t]]; h >= 0; h = pool[h].next) extra.push_back({first_t[t], pool[h].launch});
    }
    std::sort(extra.begin(), extra.end());
    extra.erase(std::unique(extra.begin(), extra.end()), extra.end());
    // group by launch, dedupe with a stamp per predecessor
    std::vector<int64_t> lcount(nlaunch + 1, 0);
    for (size_t i = 0; i < ops.size(); ++i)
      for (int k = 0; k < 2; ++k)
        if (op_rec[k][i] >= 0) ++lcount[op_rec[k][i] + 1];
    for (int64_t l = 0; l < nlaunch; ++l) lcount[l + 1] += lcount[l];
    std::vector<int32_t> lops(lcount[nlaunch]);
    {
      std::vector<int64_t> at(lcount.begin(), lcount.end() - 1);
      for (size_t i = 0; i < ops.size(); ++i)
        for (int k = 0; k < 2; ++k)
          if (op_rec[k][i] >= 0) lops[at[op_rec[k][i]]++] = (int32_t)i;
    }
    std::vector<int32_t> stamp(nlaunch, -1);
    dag_ptr.assign(nlaunch + 1, 0);
    dag_idx.clear();
    for (int64_t l = 0; l < nlaunch; ++l) {
      for (int64_t q = lcount[l]; q < lcount[l + 1]; ++q) {
        const int32_t i = lops[q];
        auto take = [&](int32_t p) {
          if (p >= l) throw std::runtime_error("dag schedule: a dependency does not precede its launch");
          if (stamp[p] == l) return;
          stamp[p] = (int32_t)l;
          dag_idx.push_back(p);
        };
        for (int64_t e = e_ptr[i]; e < e_ptr[i + 1]; ++e) take(e_idx[e]);
        const auto xr = std::equal_range(extra.begin(), extra.end(), std::make_pair(i, (int32_t)0),
                                         [](const std::pair<int32_t, int32_t> &a, const std::pair<int32_t, int32_t> &b) {
                                           return a.first < b.first;
                                         });
        for (auto it = xr.first; it != xr.second; ++it) take(it->second);
      }
      // drop predecessors another predecessor already waits for (one step of
      // transitive reduction: most hazards repeat the same few chains)
      const int64_t b = dag_ptr[l], e = (int64_t)dag_idx.size();
      if (e - b > 1) {
        std::sort(dag_idx.begin() + b, dag_idx.end());
        for (int64_t x = b; x < e; ++x) stamp[dag_idx[x]] = (int32_t)l;
        std::vector<int32_t> keep;
        // mark implied ones: a predecessor of a predecessor
        std::vector<char> implied(e - b, 0);
        for (int64_t x = b; x < e; ++x) {
          const int32_t p = dag_idx[x];
          for (int64_t y = dag_ptr[p]; y < dag_ptr[p + 1]; ++y) {
            const int32_t g = dag_idx[y];
            if (stamp[g] == l) {
              const auto it = std::lower_bound(dag_idx.begin() + b, dag_idx.begin() + e, g);
              implied[it - (dag_idx.begin() + b)] = 1;
            }
          }
        }
        int64_t w = b;
        for (int64_t x = b; x < e; ++x)
          if (!implied[x - b]) dag_idx[w++] = dag_idx[x];
        dag_idx.resize(w);
      }
      dag_ptr[l + 1] = (int64_t)dag_idx.size();
    }
    // slack of every launch in model time (latest finish that keeps the model
    // makespan - earliest finish): the runtime gives launches without slack a
    // higher scheduling priority than the ones that can wait
    std::vector<int64_t> dur(nlaunch, 0), est(nlaunch, 0), lft(nlaunch, 0);
    for (int64_t l = 0; l < nlaunch; ++l)
      for (int64_t q = lcount[l]; q < lcount[l + 1]; ++q) dur[l] = std::max(dur[l], op_cost_ns(ops[lops[q]]));
    int64_t span = 0;
    for (int64_t l = 0; l < nlaunch; ++l) {
      for (int64_t e = dag_ptr[l]; e < dag_ptr[l + 1]; ++e) est[l] = std::max(est[l], est[dag_idx[e]] + dur[dag_idx[e]]);
      span = std::max(span, est[l] + dur[l]);
    }
    std::fill(lft.begin(), lft.end(), span);
    for (int64_t l = nlaunch - 1; l >= 0; --l)
      for (int64_t e = dag_ptr[l]; e < dag_ptr[l + 1]; ++e)
        lft[dag_idx[e]] = std::min(lft[dag_idx[e]], lft[l] - dur[l]);
    dag_slack.assign(nlaunch, 0);
    for (int64_t l = 0; l < nlaunch; ++l) dag_slack[l] = lft[l] - est[l] - dur[l];
  }

  // Diagnostics (HLU_PLAN_CP=1): weighted critical path of the op DAG under a
  // per-op latency model (ns), beside the level schedule's sum of per-level
  // maxima under the same model.  Same hazard sweep as assign_levels with
  // finish times in place of levels.
  int64_t op_cost_ns(const Op &o) const {
    switch (o.kind) {
      case 0: return 25000;
      case 1: return 40000;
      case 2: return 30000 + 4000 * std::min<int64_t>(gemm[o.payload].tn, 16);
      default: {
        const RktP &r = rkt[o.payload];
        if (r.pn > 2) return 400000;
        if (std::max(r.m, r.n) <= 64) return 85000;
        return 150000;
      }
    }
  }
  void critical_path_report() {
    const int64_t nt = (int64_t)temp_size.size();
    MaxTree lw;
    TagTree lr;
    lw.init(std::max<int64_t>(nslots, 1));
    lr.init(std::max<int64_t>(nslots, 1));
    std::vector<int64_t> lw_s(nslots, 0), lwT(nt, 0), lrT(nt, 0);
    for (auto &x : lw.t) x = 0;
    for (auto &x : lr.t) x = 0;
    std::vector<int64_t> fin(ops.size(), 0);
    int64_t cp = 0;
    int64_t crit_kind[5] = {0, 0, 0, 0, 0};
    std::vector<int32_t> pred(ops.size(), -1);
    // last writer op per slot / temp for the walk back
    std::vector<int32_t> wop_s(nslots, -1), wop_t(nt, -1);
    for (size_t i = 0; i < ops.size(); ++i) {
      const Op &o = ops[i];
      int64_t c = 0;
      int32_t pr = -1;
      auto take = [&](int64_t v, int32_t who) { if (v > c) c = v, pr = who; };
      for (int64_t k = o.r_begin; k < o.r_end; ++k) {
        const Iv &v = ivs[k];
        if (v.lo >= nslots) take(lwT[v.lo - nslots], wop_t[v.lo - nslots]);
        else if (v.hi - v.lo == 1) take(lw_s[v.lo], wop_s[v.lo]);
        else {
          const int64_t q = lw.query(v.lo, v.hi);
          if (q > c) {
            c = q;
            for (int64_t s = v.lo; s < v.hi; ++s) if (lw_s[s] == q) { pr = wop_s[s]; break; }
          }
        }
      }
      for (int64_t k = o.ti_begin; k < o.ti_end; ++k) take(lwT[tids[k]], wop_t[tids[k]]);
      for (int64_t k = o.w_begin; k < o.w_end; ++k) {
        const Iv &v = ivs[k];
        if (v.lo >= nslots) {
          const int64_t t = v.lo - nslots;
          take(lwT[t], wop_t[t]);
          take(lrT[t], -1);
        } else {
          for (int64_t s = v.lo; s < v.hi; ++s) take(lw_s[s], wop_s[s]), take(lr.get(s), -1);
        }
      }
      const int64_t f = c + op_cost_ns(o);
      fin[i] = f;
      pred[i] = pr;
      for (int64_t k = o.r_begin; k < o.r_end; ++k) {
        const Iv &v = ivs[k];
        if (v.lo >= nslots) lrT[v.lo - nslots] = std::max(lrT[v.lo - nslots], f);
        else lr.chmax(v.lo, v.hi, f);
      }
      for (int64_t k = o.ti_begin; k < o.ti_end; ++k) lrT[tids[k]] = std::max(lrT[tids[k]], f);
      for (int64_t k = o.w_begin; k < o.w_end; ++k) {
        const Iv &v = ivs[k];
        if (v.lo >= nslots) lwT[v.lo - nslots] = f, wop_t[v.lo - nslots] = (int32_t)i;
        else
          for (int64_t s = v.lo; s < v.hi; ++s) lw_s[s] = f, lw.set(s, f), wop_s[s] = (int32_t)i;
      }
      for (int64_t k = o.to_begin; k < o.to_end; ++k) lwT[tids[k]] = f, wop_t[tids[k]] = (int32_t)i;
      cp = std::max(cp, f);
    }
    {
      int64_t sr = 0, sw = 0, nwide = 0, mx = 0;
      for (const Op &o : ops) {
        for (int64_t k = o.r_begin; k < o.r_end; ++k)
          if (ivs[k].lo < nslots) { sr += ivs[k].hi - ivs[k].lo; nwide += (ivs[k].hi - ivs[k].lo) > 1; mx = std::max(mx, ivs[k].hi - ivs[k].lo); }
        for (int64_t k = o.w_begin; k < o.w_end; ++k)
          if (ivs[k].lo < nslots) sw += ivs[k].hi - ivs[k].lo;
      }
      std::fprintf(stderr, "plan cp: nslots %lld read-range sum %lld (wide ivs %lld, max %lld) write-range sum %lld\n",
                   (long long)nslots, (long long)sr, (long long)nwide, (long long)mx, (long long)sw);
    }
    // sum over levels of the max op cost (what the level schedule pays)
    int64_t nlv = 0;
    for (auto l : levels) nlv = std::max(nlv, l + 1);
    std::vector<int64_t> lmax(nlv, 0);
    for (size_t i = 0; i < ops.size(); ++i) lmax[levels[i]] = std::max(lmax[levels[i]], op_cost_ns(ops[i]));
    int64_t tl = 0;
    for (auto x : lmax) tl += x;
    // walk the critical path back
    int64_t at = -1;
    for (size_t i = 0; i < ops.size(); ++i) if (fin[i] == cp) { at = (int64_t)i; break; }
    int64_t steps = 0;
    int64_t tk[5] = {0, 0, 0, 0, 0};
    while (at >= 0) {
      const Op &o = ops[at];
      int kd = o.kind;
      if (kd == 3 && rkt[o.payload].pn > 2) kd = 4;
      ++crit_kind[kd];
      tk[kd] += op_cost_ns(o);
      ++steps;
      at = pred[at];
    }
    std::fprintf(stderr,
                 "plan cp: ops %zu levels %lld | level-sum %.1f ms | critical path %.1f ms over %lld ops "
                 "(getrf %lld/%.0fms trsm %lld/%.0fms gemm %lld/%.0fms rkt %lld/%.0fms merge %lld/%.0fms)\n",
                 ops.size(), (long long)nlv, tl / 1e6, cp / 1e6, (long long)steps, (long long)crit_kind[0], tk[0] / 1e6,
                 (long long)crit_kind[1], tk[1] / 1e6, (long long)crit_kind[2], tk[2] / 1e6, (long long)crit_kind[3],
                 tk[3] / 1e6, (long long)crit_kind[4], tk[4] / 1e6);
  }

  static constexpr int64_t DAG_REUSE_GUARD_NS = 200000;
  void allocate_temps() {
    const int64_t nt = (int64_t)temp_size.size();
    const int64_t BIG = std::numeric_limits<int64_t>::max();
    std::vector<int64_t> birth(nt, BIG), death(nt, -1);
    for (size_t i = 0; i < ops.size(); ++i) {
      const Op &o = ops[i];
      if (slot_owner && !((op_mask[i] >> my_rank) & 1ull)) continue;  // temps never cross ranks
      // level schedule: a block is free once its last user's level is over.
      // DAG schedule: lifetimes in model time with a guard (a block changes
      // hands only well after its last user should have ended; the launch
      // dependencies of compute_dag_deps make the hand-over safe regardless)
      const int64_t lv = dag_slot_ns ? op_start[i] : levels[i];
      const int64_t le = dag_slot_ns ? op_ready[i] + dag_slot_ns + DAG_REUSE_GUARD_NS : levels[i];
      for (int64_t k = o.to_begin; k < o.to_end; ++k) {
        birth[tids[k]] = std::min(birth[tids[k]], lv);
        death[tids[k]] = std::max(death[tids[k]], le);
      }
      for (int64_t k = o.ti_begin; k < o.ti_end; ++k) death[tids[k]] = std::max(death[tids[k]], le);
      if (dag_slot_ns)  // temps read or written through a resource interval only
        for (int64_t k = o.r_begin; k < o.w_end; ++k)
          if (ivs[k].lo >= nslots) {
            const int64_t t = ivs[k].lo - nslots;
            birth[t] = std::min(birth[t], lv);
            death[t] = std::max(death[t], le);
          }
    }
    tbirth = birth;
    std::vector<int> cls(nt);
    for (int64_t t = 0; t < nt; ++t) {
      const int64_t s = std::max<int64_t>(temp_size[t], 1);
      int b = 0;
      while ((int64_t(1) << b) < s) ++b;
      cls[t] = std::max(6, b);
    }
    std::vector<int64_t> order(nt), by_death(nt);
    for (int64_t t = 0; t < nt; ++t) order[t] = by_death[t] = t;
    std::stable_sort(order.begin(), order.end(), [&](int64_t a, int64_t b) { return birth[a] < birth[b]; });
    std::stable_sort(by_death.begin(), by_death.end(), [&](int64_t a, int64_t b) { return death[a] < death[b]; });
    std::vector<std::vector<int64_t>> freel(64);
    toffs.assign(nt, 0);
    reuse_from.assign(nt, -1);
    std::unordered_map<int64_t, int64_t> last_user;  // arena offset -> temp that holds it
    int64_t top = 0;
    int64_t di = 0;
    for (int64_t t : order) {
      if (temp_size[t] == 0 || birth[t] == BIG) continue;  // empty, or another rank's temp
      const int64_t b = birth[t];
      while (di < nt && death[by_death[di]] < b) {
        const int64_t u = by_death[di++];
        if (temp_size[u] && birth[u] <= death[u]) freel[cls[u]].push_back(toffs[u]);
      }
      auto &fl = freel[cls[t]];
      if (!fl.empty()) {
        toffs[t] = fl.back();
        fl.pop_back();
        reuse_from[t] = last_user[toffs[t]];
      } else {
        toffs[t] = top;
        top += int64_t(1) << cls[t];
      }
      last_user[toffs[t]] = t;
    }
    arena = top;
  }

  // packed outputs
  std::vector<hlu_getrf_desc> o_getrf;
  std::vector<hlu_trsm_desc> o_trsm;
  std::vector<hlu_gemm_desc> o_gemm;
  std::vector<hlu_term> o_terms;
  std::vector<hlu_rkt_desc> o_rkt;
  std::vector<hlu_rkpart> o_parts;
  std::vector<hlu_launch> o_launch;
  int64_t nlevels = 0;

  int64_t fix(int64_t off, int64_t arena_base) const {
    if (off >= (int64_t(1) << TEMP_SHIFT)) {
      const int64_t t = (off >> TEMP_SHIFT) - 1;
      return arena_base + toffs[t] + (off & ((int64_t(1) << TEMP_SHIFT) - 1));
    }
    return off;
  }
  hlu_view fv(const View &v, int64_t ab) const {
    hlu_view o = hv(v);
    o.off = fix(v.off, ab);
    return o;
  }

  int split_rows = 0;  // 0: never split chains; else minimum rows per sub-chain
  // dense products A B with an inner dimension up to this are truncated as the
  // factor pair (A, B^T) (HLU_PRODUCT_PAIR_MAX, default RK_KMAX); wider ones are
  // formed and truncated as (I, D^T) / (D, I)
  int product_pair_max = KMAX_STACK;
  bool small_gemm = false;  // route small chains to the warp-per-chain kernel

  void push_term(std::vector<hlu_term> &out, const Term &t, int64_t ab) {
    hlu_term h;
    h.c = fv(t.c, ab);
    h.a = fv(t.a, ab);
    h.m = fv(t.m, ab);
    h.b = fv(t.b, ab);
    h.alpha = t.alpha;
    h.kind = t.kind;
    h.assoc = t.assoc;
    out.push_back(h);
  }

  // small enough for the warp-per-chain kernel (hlu_gemm_small_batched_f64)
  static bool small_chain(const hlu_term *t, int n) {
    for (int i = 0; i < n; ++i) {
      if (t[i].kind == 0) continue;
      const double crc = (double)t[i].c.rows * t[i].c.cols;
      if (t[i].kind == 1) {
        if (crc * t[i].a.cols > 131072.0) return false;
      } else if (t[i].assoc == 0) {
        if ((double)t[i].m.rows * t[i].c.cols > 1024.0) return false;
        if ((double)t[i].m.rows * t[i].c.cols * t[i].m.cols + crc * t[i].a.cols > 262144.0) return false;
      } else {
        if (t[i].m.cols > 64) return false;
        if (crc * t[i].a.cols + crc * t[i].m.cols > 262144.0) return false;
      }
    }
    return true;
  }

  // A chain whose terms write row ranges of one column-major target is cut
  // into independent sub-chains over disjoint row groups (>= split_rows rows
  // each); every sub-chain keeps the original term order on its rows.
  // appends the op's chain(s) to (large, small) staging lists
  // output: chain c = terms [cb[c], cb[c+1]) of ct (both cleared first)
  void emit_gemm(const GemmP &g, int64_t ab, std::vector<hlu_term> &ct, std::vector<int64_t> &cb) {
    ct.clear();
    cb.assign(1, 0);
    bool ok = split_rows > 0 && g.split && g.tn > 1;
    int64_t base = 0, ld = 0, cols = 0;
    if (ok) {
      const Term &t0 = terms[g.tb];
      base = t0.c.off;
      ld = t0.c.cs;
      cols = t0.c.cols;
      for (int64_t k = g.tb; k < g.tb + g.tn && ok; ++k) {
        const View &c = terms[k].c;
        if (c.rs != 1 || c.cs != ld || c.cols != cols || c.rdyn >= 0 || c.cdyn != t0.c.cdyn) ok = false;
        base = std::min(base, c.off);
      }
      for (int64_t k = g.tb; k < g.tb + g.tn && ok; ++k) {
        const int64_t r0 = terms[k].c.off - base;
        if (r0 < 0 || r0 + terms[k].c.rows > ld) ok = false;  // not row slices of one target
        if (terms[k].kind != 0 && terms[k].a.rdyn >= 0) ok = false;
      }
    }
    std::vector<int64_t> cuts;
    if (ok) {
      for (int64_t k = g.tb; k < g.tb + g.tn; ++k) {
        const int64_t r0 = terms[k].c.off - base;
        cuts.push_back(r0);
        cuts.push_back(r0 + terms[k].c.rows);
      }
      std::sort(cuts.begin(), cuts.end());
      cuts.erase(std::unique(cuts.begin(), cuts.end()), cuts.end());
      std::vector<int64_t> merged{cuts.front()};
      for (size_t i = 1; i < cuts.size(); ++i)
        if (cuts[i] - merged.back() >= split_rows || i + 1 == cuts.size()) merged.push_back(cuts[i]);
      cuts.swap(merged);
      if (cuts.size() <= 2) ok = false;
    }
    if (!ok) {
      for (int64_t k = g.tb; k < g.tb + g.tn; ++k) push_term(ct, terms[k], ab);
      cb.push_back((int64_t)ct.size());
      return;
    }
    for (size_t q = 0; q + 1 < cuts.size(); ++q) {
      const int64_t g0 = cuts[q], g1 = cuts[q + 1];
      for (int64_t k = g.tb; k < g.tb + g.tn; ++k) {
        const Term &t = terms[k];
        const int64_t r0 = t.c.off - base, r1 = r0 + t.c.rows;
        const int64_t lo = std::max(r0, g0), hi = std::min(r1, g1);
        if (lo >= hi) continue;
        Term p = t;
        p.c = t.c.rows_slice((int)(lo - r0), (int)(hi - r0));
        if (t.kind != 0) p.a = t.a.rows_slice((int)(lo - r0), (int)(hi - r0));
        push_term(ct, p, ab);
      }
      cb.push_back((int64_t)ct.size());
    }
  }

  // gemm chains of the pending level, flat: chain i = terms [tb[i], tb[i+1])
  struct Stage {
    std::vector<hlu_term> terms;
    std::vector<int64_t> tb{0};
    std::vector<int> log, log_slot;
    size_t size() const { return log.size(); }
    bool empty() const { return log.empty(); }
    void clear() {
      terms.clear();
      tb.assign(1, 0);
      log.clear();
      log_slot.clear();
    }
    void add(const hlu_term *t, int64_t n, int lg, int ls) {
      terms.insert(terms.end(), t, t + n);
      tb.push_back((int64_t)terms.size());
      log.push_back(lg);
      log_slot.push_back(ls);
    }
  };
  Stage stage_large, stage_small;
  std::vector<hlu_term> chain_terms;
  std::vector<int64_t> chain_bounds;

  // Every op runs on the owner of the skeleton slot it writes; an op writing
  // only temps (a product / accumulated Rk temp, a hoisted inner product) runs
  // on every rank that consumes the temp, so temps never cross ranks and the
  // per-destination op order (hence every rank decision) is the single-GPU one.
  void shard_ops() {
    const size_t n = ops.size();
    if (nranks > 64) throw std::runtime_error("at most 64 ranks");
    op_mask.assign(n, 0);
    std::vector<uint64_t> cons(temp_size.size(), 0);
    for (size_t ii = n; ii-- > 0;) {
      const Op &o = ops[ii];
      int owner = -1;
      for (int64_t w = o.w_begin; w < o.w_end; ++w) {
        const Iv &v = ivs[w];
        if (v.lo >= nslots) continue;
        for (int64_t sl = v.lo; sl < v.hi; ++sl) {
          const int r = slot_owner[sl];
          if (owner >= 0 && r != owner) throw std::runtime_error("an op writes slots of two owners");
          owner = r;
        }
      }
      uint64_t m = 0;
      if (owner >= 0) {
        m = 1ull << owner;
      } else {
        for (int64_t k = o.to_begin; k < o.to_end; ++k) m |= cons[tids[k]];
        if (!m) m = 1ull;  // an unread temp: rank 0
      }
      op_mask[ii] = m;
      for (int64_t k = o.ti_begin; k < o.ti_end; ++k) cons[tids[k]] |= m;
    }
  }

  // slot payload region (pool offset, doubles) and rank slot of skeleton slot s
  std::vector<int32_t> slot_node;
  void slot_nodes() {
    slot_node.assign(nslots, -1);
    for (int64_t i = 0; i < nnodes; ++i)
      if (N[i].kind != 2 && N[i].lo >= 0 && N[i].lo < nslots) slot_node[N[i].lo] = (int32_t)i;
  }
  bool slot_region(int64_t sl, int64_t *off, int64_t *len, int32_t *rslot) const {
    const int32_t k = slot_node[sl];
    if (k < 0) return false;
    const auto &x = N[k];
    const int64_t rows = x.r1 - x.r0, cols = x.c1 - x.c0;
    *off = x.off_a;
    if (x.kind == 0) {
      *len = rows * cols;
      *rslot = -1;
    } else {
      *len = (rows + cols) * (int64_t)cap;  // a slab (rows x cap) then b slab (cols x cap)
      *rslot = x.slot;
    }
    return true;
  }

  // Exchange records: after level lv, rank w broadcasts the slots it wrote in
  // lv whose value an op of another rank reads before the slot's next write
  // (a slot is written by its owner only; intermediate values nobody else
  // reads stay local, so in an H-LU mostly the final factor blocks travel);
  // a final step (level nlevels) ships every written slot from its owner, so
  // each rank ends with the whole factorization.  Records are grouped by
  // (level, src), groups capped at XFER_GROUP doubles, with their offsets in
  // the group's staging buffer (payload, then the rank).
  // HLU_XFER_EVERY_WRITE=1 restores the superset (every write of a slot that
  // has a remote reader at any level), for comparison.
  static constexpr int64_t XFER_GROUP = int64_t(1) << 26;  // 512 MB
  void exchange(const std::vector<int64_t> &order) {
    slot_nodes();
    const int64_t S = nslots;
    struct X {
      int64_t lv;
      int32_t src;
      int64_t sl;
    };
    std::vector<X> xs;
    std::vector<char> written(S, 0);
    const char *ev = std::getenv("HLU_XFER_EVERY_WRITE");
    if (ev && ev[0] == '1') {
      std::vector<uint64_t> readers(S, 0);
      std::vector<int32_t> diff((size_t)(S + 1) * nranks, 0);
      for (size_t i = 0; i < ops.size(); ++i) {
        const Op &o = ops[i];
        for (int64_t r = o.r_begin; r < o.r_end; ++r) {
          const Iv &v = ivs[r];
          if (v.lo >= S) continue;
          const int64_t hi = std::min<int64_t>(v.hi, S);
          for (int b = 0; b < nranks; ++b)
            if ((op_mask[i] >> b) & 1ull) {
              ++diff[(size_t)v.lo * nranks + b];
              --diff[(size_t)hi * nranks + b];
            }
        }
      }
      std::vector<int32_t> run(nranks, 0);
      for (int64_t sl = 0; sl < S; ++sl)
        for (int b = 0; b < nranks; ++b) {
          run[b] += diff[(size_t)sl * nranks + b];
          if (run[b] > 0) readers[sl] |= 1ull << b;
        }
      for (int64_t i : order) {  // level order
        const Op &o = ops[i];
        for (int64_t w = o.w_begin; w < o.w_end; ++w) {
          const Iv &v = ivs[w];
          if (v.lo >= S) continue;
          for (int64_t sl = v.lo; sl < std::min<int64_t>(v.hi, S); ++sl) {
            written[sl] = 1;
            const int32_t src = slot_owner[sl];
            if (readers[sl] & ~(1ull << src)) xs.push_back(X{levels[i], src, sl});
          }
        }
      }
    } else {
      // Backward sweep in level order: pending(sl) = the ranks that read slot sl
      // after the current position and before its next write.  Reads cover slot
      // intervals (partitioned operands), so pending lives in a segment tree of
      // OR tags: range OR, point query (OR over the root path), point clear
      // (tags pushed down along the path first).
      int64_t size = 1;
      while (size < std::max<int64_t>(S, 1)) size <<= 1;
      std::vector<uint64_t> tag((size_t)2 * size, 0);
      auto range_or = [&](int64_t lo, int64_t hi, uint64_t m) {
        for (lo += size, hi += size; lo < hi; lo >>= 1, hi >>= 1) {
          if (lo & 1) tag[lo++] |= m;
          if (hi & 1) tag[--hi] |= m;
        }
      };
      auto take = [&](int64_t sl) {  // query + clear
        int64_t node = 1;
        for (int64_t half = size >> 1; half >= 1; half >>= 1) {
          const uint64_t t = tag[node];
          if (t) {
            tag[2 * node] |= t;
            tag[2 * node + 1] |= t;
            tag[node] = 0;
          }
          node = 2 * node + (((sl & half) != 0) ? 1 : 0);
        }
        const uint64_t m = tag[node];
        tag[node] = 0;
        return m;
      };
      for (size_t q = order.size(); q-- > 0;) {
        const int64_t i = order[q];
        const Op &o = ops[i];
        for (int64_t w = o.w_begin; w < o.w_end; ++w) {
          const Iv &v = ivs[w];
          if (v.lo >= S) continue;
          for (int64_t sl = v.lo; sl < std::min<int64_t>(v.hi, S); ++sl) {
            written[sl] = 1;
            const int32_t src = slot_owner[sl];
            if (take(sl) & ~(1ull << src)) xs.push_back(X{levels[i], src, sl});
          }
        }
        for (int64_t r = o.r_begin; r < o.r_end; ++r) {
          const Iv &v = ivs[r];
          if (v.lo >= S) continue;
          range_or(v.lo, std::min<int64_t>(v.hi, S), op_mask[i]);
        }
      }
      std::reverse(xs.begin(), xs.end());
    }
    for (int64_t sl = 0; sl < S; ++sl)
      if (written[sl]) xs.push_back(X{nlevels, slot_owner[sl], sl});
    std::stable_sort(xs.begin(), xs.end(), [](const X &a, const X &b) {
      return a.lv != b.lv ? a.lv < b.lv : a.src < b.src;
    });
    o_xfer.clear();
    int64_t glv = -1, gsrc = -1, gfill = 0;
    int32_t group = -1;
    for (const X &x : xs) {
      int64_t off, len;
      int32_t rslot;
      if (!slot_region(x.sl, &off, &len, &rslot)) continue;
      if (x.lv != glv || x.src != gsrc || gfill + len + 1 > XFER_GROUP) {
        ++group;
        glv = x.lv;
        gsrc = x.src;
        gfill = 0;
      }
      hlu_xfer r;
      r.level = (int32_t)x.lv;
      r.src = x.src;
      r.group = group;
      r.rank_slot = rslot;
      r.off = off;
      r.len = len;
      r.boff = gfill;
      gfill += len + 1;
      o_xfer.push_back(r);
    }
  }

  static double now_s() {
    return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
  }
  void pack(int64_t arena_base) {
    const bool timing = std::getenv("HLU_PLAN_TIMING") != nullptr;
    double t0 = now_s();
    if (dag_slot_ns) assign_slots();
    else assign_levels();
    if (timing) std::fprintf(stderr, "plan: levels %.2fs\n", now_s() - t0), t0 = now_s();
    if (std::getenv("HLU_PLAN_CP")) critical_path_report();
    if (slot_owner) shard_ops();  // before the arena: a rank allocates only its own temps
    allocate_temps();
    if (timing) std::fprintf(stderr, "plan: temps %.2fs\n", now_s() - t0), t0 = now_s();
    const size_t n = ops.size();
    // ops ordered by (level, kind), program order inside: a stable counting sort
    std::vector<int64_t> order(n);
    {
      const int64_t nlv = n ? (*std::max_element(levels.begin(), levels.end()) + 1) : 0;
      std::vector<int64_t> start(nlv * 4 + 1, 0);
      for (size_t i = 0; i < n; ++i) ++start[levels[i] * 4 + ops[i].kind + 1];
      for (size_t b = 1; b < start.size(); ++b) start[b] += start[b - 1];
      for (size_t i = 0; i < n; ++i) order[start[levels[i] * 4 + ops[i].kind]++] = (int64_t)i;
    }
    struct Rec {
      int kind;
      int64_t count, first;
      int dim;
      int64_t lv;
      bool dep;  // truncation launch reading a temp produced in the same level
      int min_mn = 1 << 30;  // truncation launches: smallest max(m, n) of the ops
    };
    std::vector<Rec> recs;
    std::vector<int64_t> staged_ops[2];  // DAG schedule: gemm ops staged into the large / small launch
    if (dag_slot_ns) {
      op_rec[0].assign(n, -1);
      op_rec[1].assign(n, -1);
    }
    int64_t cur_lv = -1;
    int cur_kind = -1;
    int64_t pending_lv = -1;
    auto flush_gemm = [&]() {
      for (int pass = 0; pass < 2; ++pass) {
        auto &st = pass == 0 ? stage_large : stage_small;
        if (st.empty()) continue;
        const int64_t first = (int64_t)o_gemm.size();
        const int64_t tbase = (int64_t)o_terms.size();
        for (size_t c = 0; c < st.size(); ++c) {
          hlu_gemm_desc d;
          d.term_begin = (int32_t)(tbase + st.tb[c]);
          d.term_count = (int32_t)(st.tb[c + 1] - st.tb[c]);
          d.log = st.log[c];
          d.log_slot = st.log_slot[c];
          o_gemm.push_back(d);
        }
        o_terms.insert(o_terms.end(), st.terms.begin(), st.terms.end());
        recs.push_back(Rec{pass == 0 ? HLU_K_GEMM : HLU_K_GEMM_SMALL, (int64_t)st.size(), first, 0, pending_lv, false});
        st.clear();
        if (dag_slot_ns)
          for (int64_t q : staged_ops[pass]) op_rec[pass][q] = (int32_t)recs.size() - 1;
        staged_ops[pass].clear();
      }
      cur_kind = -1;
    };
    for (int64_t i : order) {
      const Op &o = ops[i];
      const int64_t lv = levels[i];
      if (slot_owner && !((op_mask[i] >> my_rank) & 1ull)) continue;  // another rank's op
      if (pending_lv >= 0 && (o.kind != 2 || lv != pending_lv)) {
        flush_gemm();
        pending_lv = -1;
      }
      int kind = 0, dim = 0;
      int64_t idx = 0, extra = 0;
      if (o.kind == 0) {
        const GetrfP &g = getrf[o.payload];
        hlu_getrf_desc d;
        d.a = fv(g.a, arena_base);
        d.op_id = g.op_id;
        d.lu_index = g.lu_index;
        o_getrf.push_back(d);
        kind = HLU_K_GETRF;
        idx = (int64_t)o_getrf.size() - 1;
        dim = g.a.rows;
      } else if (o.kind == 1) {
        const TrsmP &t = trsm[o.payload];
        hlu_trsm_desc d;
        d.t = fv(t.t, arena_base);
        d.x = fv(t.x, arena_base);
        d.mode = t.mode;
        d.log = t.log;
        o_trsm.push_back(d);
        kind = HLU_K_TRSM;
        idx = (int64_t)o_trsm.size() - 1;
        dim = t.t.rows;
      } else if (o.kind == 2) {
        const GemmP &g = gemm[o.payload];
        emit_gemm(g, arena_base, chain_terms, chain_bounds);
        for (size_t c = 0; c + 1 < chain_bounds.size(); ++c) {
          const hlu_term *t = chain_terms.data() + chain_bounds[c];
          const int64_t nt_ = chain_bounds[c + 1] - chain_bounds[c];
          const bool sm = small_gemm && small_chain(t, (int)nt_);
          (sm ? stage_small : stage_large).add(t, nt_, g.log, g.log_slot);
          if (dag_slot_ns && (staged_ops[sm].empty() || staged_ops[sm].back() != i)) staged_ops[sm].push_back(i);
        }
        pending_lv = lv;
        continue;
      } else {
        const RktP &r = rkt[o.payload];
        hlu_rkt_desc d;
        d.mode = r.mode;
        d.part_begin = (int32_t)o_parts.size();
        d.part_count = (int32_t)r.pn;
        d.m = r.m;
        d.n = r.n;
        d.cap = r.cap;
        d.out_slot = r.slot;
        d.log = r.log;
        d.out_a = fix(r.out_a, arena_base);
        d.out_b = fix(r.out_b, arena_base);
        d.ws = r.ws ? fix(r.ws, arena_base) : 0;
        d.reserved = 0;
        d.pad = 0;
        for (int64_t k = r.pb; k < r.pb + r.pn; ++k) {
          const Pair &p = parts[k];
          hlu_rkpart q;
          q.a = fv(p.a, arena_base);
          q.b = fv(p.b, arena_base);
          q.sign = p.sign;
          q.roff = p.roff;
          q.coff = p.coff;
          o_parts.push_back(q);
        }
        o_rkt.push_back(d);
        kind = HLU_K_RKT32;
        idx = (int64_t)o_rkt.size() - 1;
        dim = r.kb;
      }
      bool dep = false;
      if (kind == HLU_K_RKT32 && !dag_slot_ns)
        for (int64_t k = o.ti_begin; k < o.ti_end; ++k) dep = dep || tbirth[tids[k]] == lv;
      if (!recs.empty() && cur_lv == lv && cur_kind == kind) {
        recs.back().count += 1 + extra;
        recs.back().dim = std::max(recs.back().dim, dim);
        recs.back().dep = recs.back().dep || dep;
      } else {
        recs.push_back(Rec{kind, 1 + extra, idx, dim, lv, dep});
        cur_lv = lv;
        cur_kind = kind;
      }
      if (kind == HLU_K_RKT32)
        recs.back().min_mn = std::min(recs.back().min_mn, std::max(rkt[o.payload].m, rkt[o.payload].n));
      if (dag_slot_ns) op_rec[0][i] = (int32_t)recs.size() - 1;
    }
    if (pending_lv >= 0) flush_gemm();
    for (const Rec &r : recs) {
      hlu_launch L;
      L.kind = r.kind;
      L.count = (int32_t)r.count;
      L.first = r.first;
      L.level = (int32_t)r.lv;
      if (r.kind == HLU_K_RKT32) {
        L.smem_dim = (r.dep ? 1 : 0) | (r.dim > RK_KMAX ? 2 : 0);  // bit 2: may take the wide path
        if (dag_slot_ns) {  // route hints of the DAG runtime (include/hlu_b200.h HLU_RKT_HINT_*)
          if (r.min_mn > 64) L.smem_dim |= 4;      // no op fits the register warp kernels
        }
        o_launch.push_back(L);
      } else {
        L.smem_dim = r.dim;
        o_launch.push_back(L);
      }
    }
    nlevels = n ? (*std::max_element(levels.begin(), levels.end()) + 1) : 0;
    if (slot_owner) exchange(order);
    if (timing) std::fprintf(stderr, "plan: pack %.2fs\n", now_s() - t0), t0 = now_s();
    if (dag_slot_ns) {
      compute_dag_deps((int64_t)o_launch.size());
      waits_ok = false;
      if (timing) {
        int64_t mx = 0;
        for (size_t l = 0; l + 1 < dag_ptr.size(); ++l) mx = std::max(mx, dag_ptr[l + 1] - dag_ptr[l]);
        int64_t span = 0;
        for (size_t i = 0; i < n; ++i) span = std::max(span, op_ready[i]);
        std::fprintf(stderr, "plan: dag %.2fs: %zu launches, %zu edges (max in-degree %lld), model span %.1f ms\n",
                     now_s() - t0, o_launch.size(), dag_idx.size(), (long long)mx, span / 1e6);
      }
      return;
    }
    compute_waits();
    if (timing) std::fprintf(stderr, "plan: waits %.2fs\n", now_s() - t0);
  }

  // Every op conflicts (RAW / WAR / WAW on skeleton slots and temps, plus the
  // arena-block reuse of allocate_temps) only with ops at lower levels (one
  // exception: a truncation reading a temp a dense op of its own level
  // produces).  Same-class conflicts are covered by the chain's level order;
  // for the other class the op waits for the highest conflicting level.
  void compute_waits() {
    const int64_t nt = (int64_t)temp_size.size();
    wait_d.assign(nlevels, -1);
    wait_r.assign(nlevels, -1);
    waits_ok = true;
    auto cls_of = [&](const Op &o) { return o.kind == 3 ? 1 : 0; };
    // highest level at which each class touches each temp (for block reuse)
    std::vector<int64_t> touch[2] = {std::vector<int64_t>(nt, -1), std::vector<int64_t>(nt, -1)};
    for (size_t i = 0; i < ops.size(); ++i) {
      const Op &o = ops[i];
      auto &tc = touch[cls_of(o)];
      const int64_t lv = levels[i];
      for (int64_t k = o.ti_begin; k < o.to_end; ++k) tc[tids[k]] = std::max(tc[tids[k]], lv);
      for (int64_t k = o.r_begin; k < o.w_end; ++k)
        if (ivs[k].lo >= nslots) tc[ivs[k].lo - nslots] = std::max(tc[ivs[k].lo - nslots], lv);
    }
    MaxTree lw[2];
    TagTree lr[2];
    std::vector<int64_t> lw_s[2], lwT[2], lrT[2];
    for (int c = 0; c < 2; ++c) {
      lw[c].init(std::max<int64_t>(nslots, 1));
      lr[c].init(std::max<int64_t>(nslots, 1));
      lw_s[c].assign(nslots, -1);
      lwT[c].assign(nt, -1);
      lrT[c].assign(nt, -1);
    }
    for (size_t i = 0; i < ops.size(); ++i) {
      const Op &o = ops[i];
      const int x = cls_of(o), y = 1 - x;
      const int64_t lv = levels[i];
      int64_t w = -1;
      auto temp_w = [&](int64_t t) {
        w = std::max(w, std::max(lwT[y][t], lrT[y][t]));
        if (reuse_from[t] >= 0) w = std::max(w, touch[y][reuse_from[t]]);
      };
      for (int64_t k = o.r_begin; k < o.r_end; ++k) {
        const Iv &v = ivs[k];
        if (v.lo >= nslots) w = std::max(w, lwT[y][v.lo - nslots]);
        else w = std::max(w, lw[y].query(v.lo, v.hi));
      }
      for (int64_t k = o.ti_begin; k < o.ti_end; ++k) w = std::max(w, lwT[y][tids[k]]);
      for (int64_t k = o.to_begin; k < o.to_end; ++k) temp_w(tids[k]);
      for (int64_t k = o.w_begin; k < o.w_end; ++k) {
        const Iv &v = ivs[k];
        if (v.lo >= nslots) temp_w(v.lo - nslots);
        else
          for (int64_t s2 = v.lo; s2 < v.hi; ++s2) w = std::max(w, std::max(lw_s[y][s2], lr[y].get(s2)));
      }
      if (w > lv || (w == lv && x == 0)) waits_ok = false;  // only truncations may wait on their own level
      auto &wl = x == 0 ? wait_d : wait_r;
      wl[lv] = std::max<int32_t>(wl[lv], (int32_t)w);
      // commit
      for (int64_t k = o.r_begin; k < o.r_end; ++k) {
        const Iv &v = ivs[k];
        if (v.lo >= nslots) lrT[x][v.lo - nslots] = std::max(lrT[x][v.lo - nslots], lv);
        else lr[x].chmax(v.lo, v.hi, lv);
      }
      for (int64_t k = o.ti_begin; k < o.ti_end; ++k) lrT[x][tids[k]] = std::max(lrT[x][tids[k]], lv);
      for (int64_t k = o.to_begin; k < o.to_end; ++k) lwT[x][tids[k]] = std::max(lwT[x][tids[k]], lv);
      for (int64_t k = o.w_begin; k < o.w_end; ++k) {
        const Iv &v = ivs[k];
        if (v.lo >= nslots) {
          lwT[x][v.lo - nslots] = std::max(lwT[x][v.lo - nslots], lv);
        } else {
          for (int64_t s2 = v.lo; s2 < v.hi; ++s2)
            if (lv > lw_s[x][s2]) {
              lw_s[x][s2] = lv;
              lw[x].set(s2, lv);
            }
        }
      }
    }
  }
};

}  // namespace

struct hlu_plan {
  Planner P;
  std::string error;
};

static thread_local int64_t g_dag_slot_ns = 0;  // set by hlu_plan_build_dag around the build

extern "C" int hlu_plan_build(hlu_plan **out, const hlu_plan_node *nodes, int64_t nnodes, const hlu_plan_cmd *cmds,
                              int64_t ncmds, int32_t cap, int64_t ident_off, int64_t nslots, int32_t nrk,
                              int64_t arena_base, int32_t split_rows) {
  return hlu_plan_build_sharded(out, nodes, nnodes, cmds, ncmds, cap, ident_off, nslots, nrk, arena_base, split_rows,
                                nullptr, 1, 0);
}

extern "C" int hlu_plan_build_sharded(hlu_plan **out, const hlu_plan_node *nodes, int64_t nnodes,
                                      const hlu_plan_cmd *cmds, int64_t ncmds, int32_t cap, int64_t ident_off,
                                      int64_t nslots, int32_t nrk, int64_t arena_base, int32_t split_rows,
                                      const int32_t *slot_owner, int32_t nranks, int32_t rank) {
  hlu_plan *p = new hlu_plan();
  *out = p;
  Planner &P = p->P;
  if (slot_owner) {  // nranks == 1 with an owner map: the sharded machinery on one GPU (final gather only)
    if (nranks < 1 || rank < 0 || rank >= nranks) {
      p->error = "sharded plan: bad rank / owner map";
      return -1;
    }
    P.nranks = nranks;
    P.my_rank = rank;
    P.slot_owner = slot_owner;
  }
  P.N = nodes;
  P.nnodes = nnodes;
  P.cap = cap;
  P.ident_off = ident_off;
  P.nslots = nslots;
  P.nrank = nrk;
  P.split_rows = split_rows;
  P.dag_slot_ns = g_dag_slot_ns;
  if (const char *e = std::getenv("HLU_PRODUCT_PAIR_MAX")) P.product_pair_max = std::atoi(e);
  try {
    const double t0 = Planner::now_s();
    for (int64_t i = 0; i < ncmds; ++i) {
      const hlu_plan_cmd &c = cmds[i];
      switch (c.kind) {
        case HLU_CMD_FACTOR: P.factor(c.a); break;
        case HLU_CMD_SOLVE_LOWER: P.solve_lower(c.a, c.b); break;
        case HLU_CMD_SOLVE_UPPER: P.solve_upper(c.a, c.b); break;
        case HLU_CMD_UPDATE: P.update(P.whole(c.a), P.whole(c.b), P.whole(c.c)); break;
        case HLU_CMD_FWD_VEC:
        case HLU_CMD_BWD_VEC: {
          const auto &x = nodes[c.a];
          const View v{c.vec_off, x.r1 - x.r0, c.vec_cols, 1, x.r1 - x.r0, -1, -1};
          const Iv r{c.vec_res, c.vec_res + 1};
          if (c.kind == HLU_CMD_FWD_VEC) P.vec_lower(c.a, v, x.r0, r);
          else P.vec_upper(c.a, v, x.r0, r);
          break;
        }
        case HLU_CMD_MATVEC:
        case HLU_CMD_LOWER_MATVEC:
        case HLU_CMD_UPPER_MATVEC: {
          const auto &h = nodes[c.a];
          const int nr = h.r1 - h.r0, nc = h.c1 - h.c0;
          const View xv{c.vec_off, nc, c.vec_cols, 1, nc, -1, -1};
          const View yv{c.vec2_off, nr, c.vec_cols, 1, nr, -1, -1};
          P.matvec(c.a, xv, yv, Iv{c.vec_res, c.vec_res + 1}, Iv{c.vec2_res, c.vec2_res + 1},
                   c.kind == HLU_CMD_MATVEC ? 0 : (c.kind == HLU_CMD_LOWER_MATVEC ? 1 : 2));
          break;
        }
        default: throw std::runtime_error("unknown plan command");
      }
    }
    if (std::getenv("HLU_PLAN_TIMING"))
      std::fprintf(stderr, "plan: recursion %.2fs (%zu ops)\n", Planner::now_s() - t0, P.ops.size());
    P.pack(arena_base);
    if (std::getenv("HLU_PLAN_TIMING")) std::fprintf(stderr, "plan: total %.2fs\n", Planner::now_s() - t0);
  } catch (const std::exception &e) {
    p->error = e.what();
    return -1;
  }
  return 0;
}

extern "C" int hlu_plan_build_dag(hlu_plan **out, const hlu_plan_node *nodes, int64_t nnodes, const hlu_plan_cmd *cmds,
                                  int64_t ncmds, int32_t cap, int64_t ident_off, int64_t nslots, int32_t nrk,
                                  int64_t arena_base, int32_t split_rows, int64_t slot_ns) {
  g_dag_slot_ns = slot_ns > 0 ? slot_ns : 0;
  const int rc = hlu_plan_build_sharded(out, nodes, nnodes, cmds, ncmds, cap, ident_off, nslots, nrk, arena_base,
                                        split_rows, nullptr, 1, 0);
  g_dag_slot_ns = 0;
  return rc;
}

extern "C" int64_t hlu_plan_dag(const hlu_plan *p, int64_t *ptr, int32_t *idx) {
  const Planner &P = p->P;
  if (P.dag_ptr.empty()) return -1;
  if (ptr) std::memcpy(ptr, P.dag_ptr.data(), P.dag_ptr.size() * sizeof(int64_t));
  if (idx && !P.dag_idx.empty()) std::memcpy(idx, P.dag_idx.data(), P.dag_idx.size() * sizeof(int32_t));
  return (int64_t)P.dag_idx.size();
}

extern "C" int hlu_plan_dag_slack(const hlu_plan *p, int64_t *slack_ns) {
  const Planner &P = p->P;
  if (P.dag_ptr.empty()) return -1;
  if (!P.dag_slack.empty()) std::memcpy(slack_ns, P.dag_slack.data(), P.dag_slack.size() * sizeof(int64_t));
  return 0;
}

extern "C" const char *hlu_plan_error(const hlu_plan *p) { return p->error.c_str(); }

extern "C" int hlu_plan_sizes(const hlu_plan *p, int64_t *s) {
  const Planner &P = p->P;
  s[0] = (int64_t)P.o_getrf.size();
  s[1] = (int64_t)P.o_trsm.size();
  s[2] = (int64_t)P.o_gemm.size();
  s[3] = (int64_t)P.o_terms.size();
  s[4] = (int64_t)P.o_rkt.size();
  s[5] = (int64_t)P.o_parts.size();
  s[6] = (int64_t)P.o_launch.size();
  s[7] = (int64_t)P.ops.size();
  s[8] = P.nlevels;
  s[9] = P.arena;
  s[10] = P.nlog;
  s[11] = P.nrank;
  s[12] = (int64_t)P.lu_ops.size();
  s[13] = (int64_t)P.temp_size.size();
  return 0;
}

extern "C" int64_t hlu_plan_xfer(const hlu_plan *p, hlu_xfer *out) {
  const Planner &P = p->P;
  if (out && !P.o_xfer.empty()) std::memcpy(out, P.o_xfer.data(), P.o_xfer.size() * sizeof(hlu_xfer));
  return (int64_t)P.o_xfer.size();
}

extern "C" int hlu_plan_op_owners(const hlu_plan *p, uint64_t *out) {
  const Planner &P = p->P;
  if (P.op_mask.empty()) return -1;
  std::memcpy(out, P.op_mask.data(), P.op_mask.size() * sizeof(uint64_t));
  return 0;
}

template <class T>
static void cp(void *dst, const std::vector<T> &v) {
  if (dst && !v.empty()) std::memcpy(dst, v.data(), v.size() * sizeof(T));
}

extern "C" int hlu_plan_copy(const hlu_plan *p, void *getrf, void *trsm, void *gemm, void *terms, void *rkt,
                             void *parts, void *launches, int32_t *flop_formula, double *flop_coef,
                             int64_t *flop_log, int64_t *lu_op_ids, int64_t *lu_nodes, int64_t *op_levels) {
  const Planner &P = p->P;
  cp(getrf, P.o_getrf);
  cp(trsm, P.o_trsm);
  cp(gemm, P.o_gemm);
  cp(terms, P.o_terms);
  cp(rkt, P.o_rkt);
  cp(parts, P.o_parts);
  cp(launches, P.o_launch);
  for (size_t i = 0; i < P.ops.size(); ++i) {
    if (flop_formula) flop_formula[i] = P.ops[i].flop_f;
    if (flop_coef) flop_coef[i] = P.ops[i].flop_c;
    if (flop_log) flop_log[i] = P.ops[i].flop_log;
    if (op_levels) op_levels[i] = P.levels[i];
  }
  cp(lu_op_ids, P.lu_ops);
  cp(lu_nodes, P.lu_nodes);
  return 0;
}

extern "C" int hlu_plan_level_waits(const hlu_plan *p, int32_t *wait_dense, int32_t *wait_rkt) {
  const Planner &P = p->P;
  if (!P.waits_ok) return -1;
  cp(wait_dense, P.wait_d);
  cp(wait_rkt, P.wait_r);
  return 0;
}

extern "C" void hlu_plan_free(hlu_plan *p) { delete p; }
