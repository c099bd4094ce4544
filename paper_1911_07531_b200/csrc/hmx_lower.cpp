// hmx_lower.cpp — native lowering of H-LU to device op programs (host C++).
//
// Runs the reference recursions symbolically over the block table, exactly
// as planner.py does (the Python planner is the specification this file is
// tested against op for op, tests/test_lower_cpu.py):
//   arith.hlu / htrsl / htrsu / hmul          (arith.py:40-140)
//   accumulator.hlu_accu / add/shift/apply    (accumulator.py:60-235)
//   product_payload / fold / scatter          (hmatrix.py:367-448)
//   hm_apply(_t) / hm_solve_*                 (hmatrix.py:286-341)
// Every leaf-level call becomes one task (a contiguous run of hmx_op
// records executed by one CTA); ranks are device data (rank-slot codes).
// Large H x H products are split into parallel micro-tasks whose results
// meet in the plan workspace.
//
// After lowering, the execution graph is built here too:
//   std:  the reference DAG's edges (node sets asserted equal), plus the
//         micro-task edges (dataflow within a task's group);
//   accu: the data-flow edges of the sequential program (RAW / WAR / WAW on
//         every leaf, accumulator and workspace object), which replay
//         hlu_accu's per-accumulator fold order (SURVEY.md finding 3).
// Everything is flat arrays so that config 5 (3.5M tasks, ~35M ops) plans
// in seconds instead of the Python planner's hours.

#include <stdint.h>

#include <algorithm>
#include <climits>
#include <cstring>
#include <new>
#include <unordered_map>
#include <vector>

#include "../../include/hmx.h"
#include "../../include/hmx_dag.h"
#include "../../include/hmx_lower.h"

namespace {

constexpr int SCR = 15, ACCB = 3, WSB = 5;
constexpr int32_t OP_GEMM = 1, OP_COPY = 2, OP_ZERO = 3, OP_ADD = 4, OP_LU = 5, OP_TRSM_LL = 6,
                  OP_TRSM_UT = 7, OP_TRUNC = 8, OP_D2LR = 9, OP_SETRANK = 10, OP_APPEND = 11;
constexpr int32_t F_TA = 1, F_TB = 2, F_ACC = 4;
// task kinds (hmx_dag.h numbering) + micro tasks
constexpr int32_t K_SHIFT = 5, K_APPLY = 6, K_LEAF_FACTOR = 7, K_LEAF_SOLVE_L = 8,
                  K_LEAF_SOLVE_U = 9, K_LEAF_UPDATE = 10, K_ADD_UPD = 4, K_MICRO = 11;
constexpr int64_t MASK40 = (int64_t(1) << 40) - 1;
constexpr int64_t LAZY = int64_t(1) << 62;  // ref field: index into the accumulator ref table

inline int64_t al(int64_t n) { return (n + 3) / 4 * 4; }
inline int64_t mref(int b, int64_t off) { return ((int64_t)b << 56) | off; }
inline int32_t slotc(int b, int64_t idx) { return -(1 + ((b << 24) | (int32_t)idx)); }

struct Table {
  int32_t n;
  std::vector<int64_t> r0, r1, c0, c1, m, nc;
  std::vector<int8_t> leaf, adm;
  std::vector<int32_t> kids;  // n x 4
  std::vector<int32_t> leaf_lo, leaf_hi;  // leaves of the subtree: [lo, hi) of `leaves`
  std::vector<int32_t> leaves;            // all leaves, pre-order
  int32_t kid(int32_t u, int i, int j) const { return kids[4 * (size_t)u + 2 * i + j]; }
};

struct Ref {
  int base = 0;
  int64_t off = 0;
  int32_t ld = 1;
  int32_t acc_u = -1;  // accumulator ref: (uid, which, r0, c0), resolved at pack time
  int8_t acc_w = 0;    // 'U' 'V' 'D'
  int64_t ar = 0, ac = 0;
  Ref at(int64_t r, int64_t c = 0) const {
    Ref x = *this;
    if (acc_u >= 0) {
      x.off = 0;
      x.ar = ar + r;
      x.ac = ac + c;
    } else {
      x.off = off + r + c * ld;
    }
    return x;
  }
};

struct Pay {  // payload: dense (kind 'D': ref, m, n) or low rank ('R': U, V, m, n, k code, kmax)
  char kind = 'D';
  Ref ref, U, V;
  int64_t m = 0, n = 0;
  int32_t k = 0;
  int64_t kmax = 0;
};

struct AccRef { int32_t u; int8_t w; int64_t r, c, ld; };

enum ObjKind : int64_t { OBJ_M = 0, OBJ_A = 1, OBJ_W = 2 };
inline int64_t obj(int64_t kind, int64_t base, int64_t id) { return (kind << 60) | (base << 40) | id; }

struct Pending { double alpha; int xb, ua, yb, ub; };

struct Lower {
  const Table& t;
  int mode;  // policy code
  int kfix;
  double eps;
  int64_t rank_cap;  // <= 0: none
  int64_t split_min;
  // layout (shared by A, L, U)
  std::vector<int64_t> d_off, u_off, v_off, cap;
  int64_t lay_size = 1;
  // tasks
  std::vector<std::vector<hmx_op>> tops;
  std::vector<int32_t> kind, u0, u1, u2;
  std::vector<double> alpha;
  std::vector<int32_t> order;
  std::vector<std::vector<int32_t>> pre;  // micro tasks placed before a task
  std::vector<int32_t> root_of;           // group root of every task (itself if none)
  std::vector<std::vector<int64_t>> rds, wrs;
  std::vector<int64_t> tpeak;
  std::vector<int32_t> dim3_lazy;  // per op (global index at pack time): handled via side list
  std::vector<std::pair<int64_t, int32_t>> lazy_dims;  // (task<<32 | op index in task), acc uid
  std::vector<AccRef> acc_refs;
  hmx_op* cur = nullptr;
  int32_t cur_id = -1;
  int64_t top = 0, peak = 0;
  int32_t rtop = 0, rpeak = 0;
  int64_t wtop = 0;
  int32_t wslots = 0, nw = 0;
  int64_t updates = 0;
  // accumulators
  std::vector<int8_t> acc_state;  // 0 none, 'D', 'R'
  std::vector<int64_t> acc_kmax, acc_need_lr;
  std::vector<int8_t> acc_has_lr, acc_need_d;
  std::vector<std::vector<Pending>> acc_pending;
  bool accu = false;
  int err = 0;

  Lower(const Table& tab, int pmode, int kf, double e, int64_t rc, int64_t sm, const int32_t* caps)
      : t(tab), mode(pmode), kfix(kf), eps(e), rank_cap(rc), split_min(sm) {
    const int32_t n = t.n;
    d_off.assign(n, -1);
    u_off.assign(n, -1);
    v_off.assign(n, -1);
    cap.assign(n, 0);
    int64_t curo = 0;
    for (int32_t u : t.leaves) {
      const int64_t m = t.m[u], nc = t.nc[u];
      if (t.adm[u]) {
        int64_t c = std::min(m, nc);
        if (rank_cap > 0) c = std::min(c, rank_cap);
        if (caps && caps[u] >= 0) c = std::min<int64_t>(c, caps[u]);
        cap[u] = c;
        u_off[u] = curo;
        curo += al(m * c);
        v_off[u] = curo;
        curo += al(nc * c);
      } else {
        d_off[u] = curo;
        curo += al(m * nc);
      }
    }
    lay_size = std::max<int64_t>(curo, 1);
    acc_state.assign(n, 0);
    acc_kmax.assign(n, 0);
    acc_need_lr.assign(n, 0);
    acc_has_lr.assign(n, 0);
    acc_need_d.assign(n, 0);
    acc_pending.resize(n);
  }

  // ---- references -------------------------------------------------------
  int64_t rv(const Ref& r) {
    if (r.acc_u >= 0) {
      acc_refs.push_back({r.acc_u, r.acc_w, r.ar, r.ac, r.ld});
      return LAZY | (int64_t)(acc_refs.size() - 1);
    }
    return mref(r.base, r.off);
  }
  char pkind(int32_t u) const { return !t.leaf[u] ? 'H' : (t.adm[u] ? 'R' : 'D'); }
  Ref dense(int base, int32_t u) const {
    Ref r;
    r.base = base;
    r.off = d_off[u];
    r.ld = (int32_t)t.m[u];
    return r;
  }
  Pay lr(int base, int32_t u) const {
    Pay p;
    p.kind = 'R';
    p.U.base = base; p.U.off = u_off[u]; p.U.ld = (int32_t)t.m[u];
    p.V.base = base; p.V.off = v_off[u]; p.V.ld = (int32_t)t.nc[u];
    p.m = t.m[u];
    p.n = t.nc[u];
    p.k = slotc(base, u);
    p.kmax = cap[u];
    return p;
  }

  // ---- op emission ------------------------------------------------------
  hmx_op& op(int32_t code, int32_t flags = 0) {
    tops[cur_id].push_back(hmx_op());
    hmx_op& o = tops[cur_id].back();
    memset(&o, 0, sizeof(o));
    o.code = code;
    o.flags = flags;
    return o;
  }
  void new_task(int32_t k, int32_t a, int32_t b, int32_t c, double al_) {
    const int32_t tid = (int32_t)tops.size();
    tops.emplace_back();
    kind.push_back(k);
    u0.push_back(a);
    u1.push_back(b);
    u2.push_back(c);
    alpha.push_back(al_);
    pre.emplace_back();
    root_of.push_back(tid);
    rds.emplace_back();
    wrs.emplace_back();
    tpeak.push_back(0);
    cur_id = tid;
    top = 0;
    rtop = 0;
  }
  void begin(int32_t k, int32_t a, int32_t b, int32_t c, double al_) {
    new_task(k, a, b, c, al_);
    order.push_back(cur_id);
  }
  void rd(int64_t o) { rds[cur_id].push_back(o); }
  void wr(int64_t o) { wrs[cur_id].push_back(o); }

  int64_t alloc(int64_t n) {
    const int64_t off = top;
    top += al(std::max<int64_t>(n, 1));
    if (top > tpeak[cur_id]) tpeak[cur_id] = top;
    if (top > peak) peak = top;
    return off;
  }
  Ref sref(int64_t rows, int64_t cols) {
    Ref r;
    r.base = SCR;
    r.off = alloc(rows * std::max<int64_t>(cols, 1));
    r.ld = (int32_t)std::max<int64_t>(rows, 1);
    return r;
  }
  int32_t lslot() {
    const int32_t s = rtop++;
    rpeak = std::max(rpeak, rtop);
    return slotc(SCR, s);
  }
  Ref wref_(int64_t rows, int64_t cols) {
    Ref r;
    r.base = WSB;
    r.off = wtop;
    wtop += al(std::max<int64_t>(rows * std::max<int64_t>(cols, 1), 1));
    r.ld = (int32_t)std::max<int64_t>(rows, 1);
    return r;
  }
  int32_t wslot() { return slotc(WSB, wslots++); }

  void gemm(int64_t m, int64_t n, int32_t k, double a, const Ref& A, bool ta, const Ref& B, bool tb,
            const Ref& C, bool acc) {
    hmx_op& o = op(OP_GEMM, (ta ? F_TA : 0) | (tb ? F_TB : 0) | (acc ? F_ACC : 0));
    o.dim[0] = (int32_t)m; o.dim[1] = (int32_t)n; o.dim[2] = k;
    o.ld[0] = A.ld; o.ld[1] = B.ld; o.ld[2] = C.ld;
    o.ref[0] = rv(A); o.ref[1] = rv(B); o.ref[2] = rv(C);
    o.farg[0] = a;
  }
  // gemm with a dim code for m / n (rank slots)
  void gemm_c(int32_t m, int32_t n, int32_t k, double a, const Ref& A, bool ta, const Ref& B, bool tb,
              const Ref& C, bool acc) {
    hmx_op& o = op(OP_GEMM, (ta ? F_TA : 0) | (tb ? F_TB : 0) | (acc ? F_ACC : 0));
    o.dim[0] = m; o.dim[1] = n; o.dim[2] = k;
    o.ld[0] = A.ld; o.ld[1] = B.ld; o.ld[2] = C.ld;
    o.ref[0] = rv(A); o.ref[1] = rv(B); o.ref[2] = rv(C);
    o.farg[0] = a;
  }
  void copy(int32_t m, int32_t n, double a, const Ref& A, const Ref& C, bool ta = false) {
    hmx_op& o = op(OP_COPY, ta ? F_TA : 0);
    o.dim[0] = m; o.dim[1] = n;
    o.ld[0] = A.ld; o.ld[2] = C.ld;
    o.ref[0] = rv(A); o.ref[2] = rv(C);
    o.farg[0] = a;
  }
  void zero(int32_t m, int32_t n, const Ref& C) {
    hmx_op& o = op(OP_ZERO);
    o.dim[0] = m; o.dim[1] = n;
    o.ld[2] = C.ld;
    o.ref[2] = rv(C);
  }
  void add(int32_t m, int32_t n, double a, const Ref& A, const Ref& C) {
    hmx_op& o = op(OP_ADD);
    o.dim[0] = m; o.dim[1] = n;
    o.ld[0] = A.ld; o.ld[2] = C.ld;
    o.ref[0] = rv(A); o.ref[2] = rv(C);
    o.farg[0] = a;
  }
  void setrank(int32_t slot, int32_t value) {
    hmx_op& o = op(OP_SETRANK);
    o.dim[0] = value;
    o.slot[0] = slot;
  }
  // capc_lazy >= 0: dim[3] = final accumulator capacity of that uid
  void append(const Ref& Ud, const Ref& Vd, int64_t M, int64_t N, int64_t capc, int32_t capc_lazy,
              int32_t cnt, const Pay& p, int64_t r0, int64_t c0) {
    hmx_op& o = op(OP_APPEND);
    o.dim[0] = (int32_t)M; o.dim[1] = (int32_t)N; o.dim[2] = p.k; o.dim[3] = (int32_t)capc;
    if (capc_lazy >= 0)
      lazy_dims.push_back({((int64_t)cur_id << 32) | (int64_t)(tops[cur_id].size() - 1), capc_lazy});
    o.ld[0] = p.U.ld; o.ld[1] = p.V.ld; o.ld[2] = Ud.ld; o.ld[3] = Vd.ld;
    o.ref[0] = rv(p.U); o.ref[1] = rv(p.V); o.ref[2] = rv(Ud); o.ref[3] = rv(Vd);
    o.slot[0] = cnt;
    o.iarg[0] = (int32_t)p.m; o.iarg[1] = (int32_t)p.n; o.iarg[2] = (int32_t)r0; o.iarg[3] = (int32_t)c0;
  }
  void trunc(int64_t m, int64_t n, int32_t K, int64_t kb, const Ref& U, const Ref& V, const Ref& Uo,
             const Ref& Vo, int32_t rslot, int64_t cp) {
    kb = std::max<int64_t>(kb, 1);
    Ref ws = sref(9 * kb * kb + (m + n + 200) * kb + 2048, 1);
    hmx_op& o = op(OP_TRUNC);
    o.dim[0] = (int32_t)m; o.dim[1] = (int32_t)n; o.dim[2] = K;
    o.ld[0] = U.ld; o.ld[1] = V.ld; o.ld[2] = Uo.ld; o.ld[3] = Vo.ld;
    o.ref[0] = rv(U); o.ref[1] = rv(V); o.ref[2] = rv(Uo); o.ref[3] = rv(Vo);
    o.slot[0] = rslot;
    o.iarg[0] = mode; o.iarg[1] = kfix; o.iarg[2] = (int32_t)cp; o.iarg[3] = (int32_t)kb;
    o.farg[1] = eps;
    o.wref = rv(ws);
  }
  void d2lr(int64_t m, int64_t n, const Ref& M, const Ref& Uo, const Ref& Vo, int32_t rslot, int64_t cp) {
    const int64_t l = std::max(m, n);
    // blocks of 256 and more keep a copy of M next to the work area (d2lr_big)
    Ref ws = sref(8 * l + (l >= 256 ? 3 * l * l + 2500000 : 16 * l * l), 1);
    hmx_op& o = op(OP_D2LR);
    o.dim[0] = (int32_t)m; o.dim[1] = (int32_t)n;
    o.ld[0] = M.ld; o.ld[2] = Uo.ld; o.ld[3] = Vo.ld;
    o.ref[0] = rv(M); o.ref[2] = rv(Uo); o.ref[3] = rv(Vo);
    o.slot[0] = rslot;
    o.iarg[0] = mode; o.iarg[1] = kfix; o.iarg[2] = (int32_t)cp;
    o.farg[1] = eps;
    o.wref = rv(ws);
  }

  // ---- H x dense (hmatrix.py:286-315) -------------------------------------
  // out (m_u x cols) (+)= alpha X[u] S ; cols is a dim code, colsmax its bound
  Ref hm_apply(int xb, int32_t u, const Ref& S, int32_t cols, int64_t colsmax, const Ref* outp,
               double a, int64_t row_off, bool fresh) {
    const int64_t m = t.m[u];
    Ref out = outp ? *outp : sref(m, colsmax);
    if (fresh) zero((int32_t)m, cols, out);
    for (int32_t i = t.leaf_lo[u]; i < t.leaf_hi[u]; ++i) {
      const int32_t v = t.leaves[i];
      const int64_t r0 = t.r0[v] - t.r0[u], c0 = t.c0[v] - t.c0[u];
      const int64_t mv = t.m[v], nv = t.nc[v];
      if (t.adm[v]) {
        Pay p = lr(xb, v);
        const int64_t mark = top;
        Ref T = sref(std::max<int64_t>(p.kmax, 1), colsmax);
        gemm_c(p.k, cols, (int32_t)nv, 1.0, p.V, true, S.at(c0), false, T, false);
        gemm_c((int32_t)mv, cols, p.k, a, p.U, false, T, false, out.at(row_off + r0), true);
        top = mark;
      } else {
        gemm_c((int32_t)mv, cols, (int32_t)nv, a, dense(xb, v), false, S.at(c0), false,
               out.at(row_off + r0), true);
      }
    }
    return out;
  }
  Ref hm_apply_t(int xb, int32_t u, const Ref& S, int32_t cols, int64_t colsmax, const Ref* outp,
                 double a, int64_t row_off, bool fresh) {
    const int64_t n = t.nc[u];
    Ref out = outp ? *outp : sref(n, colsmax);
    if (fresh) zero((int32_t)n, cols, out);
    for (int32_t i = t.leaf_lo[u]; i < t.leaf_hi[u]; ++i) {
      const int32_t v = t.leaves[i];
      const int64_t r0 = t.r0[v] - t.r0[u], c0 = t.c0[v] - t.c0[u];
      const int64_t mv = t.m[v], nv = t.nc[v];
      if (t.adm[v]) {
        Pay p = lr(xb, v);
        const int64_t mark = top;
        Ref T = sref(std::max<int64_t>(p.kmax, 1), colsmax);
        gemm_c(p.k, cols, (int32_t)mv, 1.0, p.U, true, S.at(r0), false, T, false);
        gemm_c((int32_t)nv, cols, p.k, a, p.V, false, T, false, out.at(row_off + c0), true);
        top = mark;
      } else {
        gemm_c((int32_t)nv, cols, (int32_t)mv, a, dense(xb, v), true, S.at(r0), false,
               out.at(row_off + c0), true);
      }
    }
    return out;
  }

  // ---- triangular solves (hmatrix.py:318-341) -----------------------------
  void solve_lower(int lb, int32_t u, const Ref& Y, int32_t cols, int64_t colsmax) {
    if (t.leaf[u]) {
      if (t.adm[u]) { err = 2; return; }
      hmx_op& o = op(OP_TRSM_LL);
      o.dim[0] = (int32_t)t.m[u]; o.dim[1] = cols;
      o.ld[0] = (int32_t)t.m[u]; o.ld[2] = Y.ld;
      o.ref[0] = rv(dense(lb, u)); o.ref[2] = rv(Y);
      return;
    }
    const int32_t k00 = t.kid(u, 0, 0), k10 = t.kid(u, 1, 0), k11 = t.kid(u, 1, 1);
    const int64_t n0 = t.m[k00];
    solve_lower(lb, k00, Y, cols, colsmax);
    hm_apply(lb, k10, Y, cols, colsmax, &Y, -1.0, n0, false);
    solve_lower(lb, k11, Y.at(n0), cols, colsmax);
  }
  void solve_upper_t(int ub_, int32_t u, const Ref& Y, int32_t cols, int64_t colsmax) {
    if (t.leaf[u]) {
      if (t.adm[u]) { err = 2; return; }
      hmx_op& o = op(OP_TRSM_UT);
      o.dim[0] = (int32_t)t.m[u]; o.dim[1] = cols;
      o.ld[0] = (int32_t)t.m[u]; o.ld[2] = Y.ld;
      o.ref[0] = rv(dense(ub_, u)); o.ref[2] = rv(Y);
      return;
    }
    const int32_t k00 = t.kid(u, 0, 0), k01 = t.kid(u, 0, 1), k11 = t.kid(u, 1, 1);
    const int64_t n0 = t.m[k00];
    solve_upper_t(ub_, k00, Y, cols, colsmax);
    hm_apply_t(ub_, k01, Y, cols, colsmax, &Y, -1.0, n0, false);
    solve_upper_t(ub_, k11, Y.at(n0), cols, colsmax);
  }

  // ---- product payloads (hmatrix.py:367-417) ------------------------------
  Pay micro_product(double a, int xb, int32_t ua, int yb, int32_t ub, int depth) {
    const int32_t p_id = cur_id;
    const int64_t p_top = top;
    const int32_t p_rtop = rtop;
    const int32_t root = root_of[p_id];
    new_task(K_MICRO, ua, ub, -1, a);
    const int32_t mid = cur_id;
    pre[p_id].push_back(mid);
    root_of[mid] = root;
    Pay q = product(a, xb, ua, yb, ub, depth + 1);
    const int32_t wid = nw++;
    Pay out;
    if (q.kind == 'D') {
      Ref W = wref_(q.m, q.n);
      copy((int32_t)q.m, (int32_t)q.n, 1.0, q.ref, W);
      out.kind = 'D';
      out.ref = W;
      out.m = q.m;
      out.n = q.n;
    } else {
      Ref Wu = wref_(q.m, q.kmax), Wv = wref_(q.n, q.kmax);
      const int32_t ws = wslot();
      copy((int32_t)q.m, q.k, 1.0, q.U, Wu);
      copy((int32_t)q.n, q.k, 1.0, q.V, Wv);
      setrank(ws, q.k);
      out.kind = 'R';
      out.U = Wu;
      out.V = Wv;
      out.m = q.m;
      out.n = q.n;
      out.k = ws;
      out.kmax = q.kmax;
    }
    wr(obj(OBJ_W, 0, wid));
    cur_id = p_id;
    top = p_top;
    rtop = p_rtop;
    rd(obj(OBJ_W, 0, wid));
    return out;
  }

  void stack(const std::vector<std::tuple<Pay, int64_t, int64_t>>& parts, int64_t m, int64_t n,
             Ref& Ub, Ref& Vb, int32_t& cnt, int64_t& kb) {
    kb = 0;
    for (auto& x : parts) kb += std::get<0>(x).kmax;
    Ub = sref(m, kb);
    Vb = sref(n, kb);
    cnt = lslot();
    setrank(cnt, 0);
    for (auto& x : parts) append(Ub, Vb, m, n, kb, -1, cnt, std::get<0>(x), std::get<1>(x), std::get<2>(x));
  }

  Pay product(double a, int xb, int32_t ua, int yb, int32_t ub, int depth = 0) {
    rd(obj(OBJ_M, xb, ua));
    rd(obj(OBJ_M, yb, ub));
    const int64_t m = t.m[ua], kk = t.nc[ua], n = t.nc[ub];
    if (kk != t.m[ub]) { err = 2; return Pay(); }
    const char kx = pkind(ua), ky = pkind(ub);
    if (kx == 'R') {
      Pay A = lr(xb, ua);
      Ref Up = sref(m, A.kmax);
      copy((int32_t)m, A.k, a, A.U, Up);
      Ref Vp = hm_apply_t(yb, ub, A.V, A.k, A.kmax, nullptr, 1.0, 0, true);
      Pay p;
      p.kind = 'R'; p.U = Up; p.V = Vp; p.m = m; p.n = n; p.k = A.k; p.kmax = A.kmax;
      return p;
    }
    if (ky == 'R') {
      Pay B = lr(yb, ub);
      Ref S = sref(kk, B.kmax);
      copy((int32_t)kk, B.k, a, B.U, S);
      Ref Up = hm_apply(xb, ua, S, B.k, B.kmax, nullptr, 1.0, 0, true);
      Pay p;
      p.kind = 'R'; p.U = Up; p.V = B.V; p.m = m; p.n = n; p.k = B.k; p.kmax = B.kmax;
      return p;
    }
    if (kx == 'D' && ky == 'D') {
      Ref P = sref(m, n);
      gemm(m, n, (int32_t)kk, a, dense(xb, ua), false, dense(yb, ub), false, P, false);
      Pay p;
      p.kind = 'D'; p.ref = P; p.m = m; p.n = n;
      return p;
    }
    if (kx == 'D') {  // Y blocked: (Y^T (a A^T))^T
      Ref T = sref(kk, m);
      copy((int32_t)kk, (int32_t)m, a, dense(xb, ua), T, true);
      Ref W = hm_apply_t(yb, ub, T, (int32_t)m, m, nullptr, 1.0, 0, true);
      Ref P = sref(m, n);
      copy((int32_t)m, (int32_t)n, 1.0, W, P, true);
      Pay p;
      p.kind = 'D'; p.ref = P; p.m = m; p.n = n;
      return p;
    }
    if (ky == 'D') {  // X blocked
      Ref S = sref(kk, n);
      copy((int32_t)kk, (int32_t)n, a, dense(yb, ub), S);
      Pay p;
      p.kind = 'D';
      p.ref = hm_apply(xb, ua, S, (int32_t)n, n, nullptr, 1.0, 0, true);
      p.m = m;
      p.n = n;
      return p;
    }
    const bool split = split_min > 0 && depth < 2 && std::min(m, n) >= split_min &&
                       !(t.leaf[t.kid(ua, 0, 0)] && t.leaf[t.kid(ub, 0, 0)]);
    std::vector<std::tuple<Pay, int64_t, int64_t>> parts;
    bool have_d = false;
    Ref dacc;
    for (int i = 0; i < 2; ++i)
      for (int j = 0; j < 2; ++j)
        for (int l = 0; l < 2; ++l) {
          const int32_t ail = t.kid(ua, i, l), blj = t.kid(ub, l, j);
          Pay q = split ? micro_product(a, xb, ail, yb, blj, depth) : product(a, xb, ail, yb, blj, depth + 1);
          if (err) return Pay();
          const int64_t r0 = t.r0[ail] - t.r0[ua], c0 = t.c0[blj] - t.c0[ub];
          if (q.kind == 'D') {
            if (!have_d) {
              dacc = sref(m, n);
              zero((int32_t)m, (int32_t)n, dacc);
              have_d = true;
            }
            add((int32_t)q.m, (int32_t)q.n, 1.0, q.ref, dacc.at(r0, c0));
          } else if (q.kmax > 0) {
            parts.emplace_back(q, r0, c0);
          }
        }
    if (have_d) {
      if (!parts.empty()) {
        Ref Ub, Vb;
        int32_t cnt;
        int64_t kb;
        stack(parts, m, n, Ub, Vb, cnt, kb);
        gemm_c((int32_t)m, (int32_t)n, cnt, 1.0, Ub, false, Vb, true, dacc, true);
      }
      Pay p;
      p.kind = 'D'; p.ref = dacc; p.m = m; p.n = n;
      return p;
    }
    if (parts.empty()) {
      Pay p;
      p.kind = 'R'; p.U = sref(m, 1); p.V = sref(n, 1); p.m = m; p.n = n; p.k = 0; p.kmax = 0;
      return p;
    }
    Ref Ub, Vb;
    int32_t cnt;
    int64_t kb;
    stack(parts, m, n, Ub, Vb, cnt, kb);
    int64_t kout = std::min(std::min(m, n), kb);
    if (rank_cap > 0) kout = std::min(kout, rank_cap);
    Ref Un = sref(m, kout), Vn = sref(n, kout);
    const int32_t rs = lslot();
    trunc(m, n, cnt, kb, Ub, Vb, Un, Vn, rs, kout);
    Pay p;
    p.kind = 'R'; p.U = Un; p.V = Vn; p.m = m; p.n = n; p.k = rs; p.kmax = kout;
    return p;
  }

  // ---- folds (hmatrix.py:420-448) ----------------------------------------
  void fold_leaf(int cb, int32_t u, const Pay& p) {
    const int64_t m = t.m[u], n = t.nc[u];
    if (p.m != m || p.n != n) { err = 2; return; }
    updates++;
    rd(obj(OBJ_M, cb, u));
    wr(obj(OBJ_M, cb, u));
    if (!t.adm[u]) {
      Ref D = dense(cb, u);
      if (p.kind == 'D') add((int32_t)m, (int32_t)n, 1.0, p.ref, D);
      else gemm_c((int32_t)m, (int32_t)n, p.k, 1.0, p.U, false, p.V, true, D, true);
      return;
    }
    Pay c = lr(cb, u);
    const int64_t mark = top;
    if (p.kind == 'D') {
      Ref M = sref(m, n);
      gemm_c((int32_t)m, (int32_t)n, c.k, 1.0, c.U, false, c.V, true, M, false);
      add((int32_t)m, (int32_t)n, 1.0, p.ref, M);
      d2lr(m, n, M, c.U, c.V, slotc(cb, u), c.kmax);
    } else {
      const int64_t kb = c.kmax + p.kmax;
      Ref Ub = sref(m, kb), Vb = sref(n, kb);
      const int32_t cnt = lslot();
      setrank(cnt, 0);
      append(Ub, Vb, m, n, kb, -1, cnt, c, 0, 0);
      append(Ub, Vb, m, n, kb, -1, cnt, p, 0, 0);
      trunc(m, n, cnt, kb, Ub, Vb, c.U, c.V, slotc(cb, u), c.kmax);
    }
    top = mark;
  }

  void scatter(int cb, int32_t u, const Pay& p) {
    if (t.leaf[u]) {
      fold_leaf(cb, u, p);
      return;
    }
    for (int q = 0; q < 4; ++q) {
      const int32_t ch = t.kids[4 * (size_t)u + q];
      const int64_t r0 = t.r0[ch] - t.r0[u], c0 = t.c0[ch] - t.c0[u];
      Pay s = p;
      s.m = t.m[ch];
      s.n = t.nc[ch];
      if (p.kind == 'D') s.ref = p.ref.at(r0, c0);
      else { s.U = p.U.at(r0); s.V = p.V.at(c0); }
      scatter(cb, ch, s);
    }
  }

  // ---- leaf tasks ----------------------------------------------------------
  void t_factor(int32_t u) {
    if (pkind(u) != 'D') { err = 2; return; }
    const int32_t n = (int32_t)t.m[u];
    rd(obj(OBJ_M, 0, u));
    wr(obj(OBJ_M, 1, u));
    wr(obj(OBJ_M, 2, u));
    hmx_op& o = op(OP_LU);
    o.dim[0] = n;
    o.ld[0] = n; o.ld[1] = n; o.ld[2] = n;
    o.ref[0] = rv(dense(0, u)); o.ref[1] = rv(dense(1, u)); o.ref[2] = rv(dense(2, u));
  }
  void t_solve_l(int lb, int32_t ul, int mb, int32_t um, int xb) {
    rd(obj(OBJ_M, lb, ul));
    rd(obj(OBJ_M, mb, um));
    wr(obj(OBJ_M, xb, um));
    const int64_t m = t.m[um], n = t.nc[um];
    if (pkind(um) == 'D') {
      Ref D = dense(xb, um);
      copy((int32_t)m, (int32_t)n, 1.0, dense(mb, um), D);
      solve_lower(lb, ul, D, (int32_t)n, n);
    } else {
      Pay A = lr(mb, um), X = lr(xb, um);
      copy((int32_t)m, A.k, 1.0, A.U, X.U);
      copy((int32_t)n, A.k, 1.0, A.V, X.V);
      setrank(X.k, A.k);
      solve_lower(lb, ul, X.U, X.k, X.kmax);
    }
  }
  void t_solve_u(int ubb, int32_t uu, int mb, int32_t um, int xb) {
    rd(obj(OBJ_M, ubb, uu));
    rd(obj(OBJ_M, mb, um));
    wr(obj(OBJ_M, xb, um));
    const int64_t m = t.m[um], n = t.nc[um];
    if (pkind(um) == 'D') {
      Ref T = sref(n, m);
      copy((int32_t)n, (int32_t)m, 1.0, dense(mb, um), T, true);
      solve_upper_t(ubb, uu, T, (int32_t)m, m);
      copy((int32_t)m, (int32_t)n, 1.0, T, dense(xb, um), true);
    } else {
      Pay A = lr(mb, um), X = lr(xb, um);
      copy((int32_t)m, A.k, 1.0, A.U, X.U);
      copy((int32_t)n, A.k, 1.0, A.V, X.V);
      setrank(X.k, A.k);
      solve_upper_t(ubb, uu, X.V, X.k, X.kmax);
    }
  }

  // ---- standard recursion (arith.py:40-140) -------------------------------
  void hmul(double a, int xb, int32_t ua, int yb, int32_t ub, int cb, int32_t uc) {
    if (a == 0.0 || err) return;
    if (!(t.leaf[ua] || t.leaf[ub] || t.leaf[uc])) {
      for (int i = 0; i < 2; ++i)
        for (int j = 0; j < 2; ++j)
          for (int l = 0; l < 2; ++l) hmul(a, xb, t.kid(ua, i, l), yb, t.kid(ub, l, j), cb, t.kid(uc, i, j));
      return;
    }
    begin(K_LEAF_UPDATE, ua, ub, uc, a);
    Pay p = product(a, xb, ua, yb, ub);
    if (!err) scatter(cb, uc, p);
  }
  void hlu(int32_t u) {
    if (err) return;
    if (!t.leaf[u]) {
      const int32_t a00 = t.kid(u, 0, 0), a01 = t.kid(u, 0, 1), a10 = t.kid(u, 1, 0), a11 = t.kid(u, 1, 1);
      hlu(a00);
      htrsu(2, a00, 0, a10, 1);
      htrsl(1, a00, 0, a01, 2);
      hmul(-1.0, 1, a10, 2, a01, 0, a11);
      hlu(a11);
      return;
    }
    begin(K_LEAF_FACTOR, u, -1, -1, 1.0);
    t_factor(u);
  }
  void htrsl(int lb, int32_t ul, int mb, int32_t um, int xb) {
    if (err) return;
    if (!t.leaf[um]) {
      const int32_t l00 = t.kid(ul, 0, 0), l10 = t.kid(ul, 1, 0), l11 = t.kid(ul, 1, 1);
      const int32_t m00 = t.kid(um, 0, 0), m01 = t.kid(um, 0, 1), m10 = t.kid(um, 1, 0), m11 = t.kid(um, 1, 1);
      htrsl(lb, l00, mb, m00, xb);
      htrsl(lb, l00, mb, m01, xb);
      hmul(-1.0, lb, l10, xb, m00, mb, m10);
      hmul(-1.0, lb, l10, xb, m01, mb, m11);
      htrsl(lb, l11, mb, m10, xb);
      htrsl(lb, l11, mb, m11, xb);
      return;
    }
    begin(K_LEAF_SOLVE_L, ul, um, -1, 1.0);
    t_solve_l(lb, ul, mb, um, xb);
  }
  void htrsu(int ubb, int32_t uu, int mb, int32_t um, int xb) {
    if (err) return;
    if (!t.leaf[um]) {
      const int32_t u00 = t.kid(uu, 0, 0), u01 = t.kid(uu, 0, 1), u11 = t.kid(uu, 1, 1);
      const int32_t m00 = t.kid(um, 0, 0), m01 = t.kid(um, 0, 1), m10 = t.kid(um, 1, 0), m11 = t.kid(um, 1, 1);
      htrsu(ubb, u00, mb, m00, xb);
      htrsu(ubb, u00, mb, m10, xb);
      hmul(-1.0, xb, m00, ubb, u01, mb, m01);
      hmul(-1.0, xb, m10, ubb, u01, mb, m11);
      htrsu(ubb, u11, mb, m01, xb);
      htrsu(ubb, u11, mb, m11, xb);
      return;
    }
    begin(K_LEAF_SOLVE_U, uu, um, -1, 1.0);
    t_solve_u(ubb, uu, mb, um, xb);
  }

  // ---- accumulator recursion (accumulator.py:41-235) ----------------------
  int64_t acc_cap(int32_t u) const {
    int64_t c = std::min(t.m[u], t.nc[u]);
    if (rank_cap > 0) c = std::min(c, rank_cap);
    return c;
  }
  Pay acc_lr(int32_t u) {
    Pay p;
    p.kind = 'R';
    p.U.base = ACCB; p.U.ld = (int32_t)t.m[u]; p.U.acc_u = u; p.U.acc_w = 'U';
    p.V.base = ACCB; p.V.ld = (int32_t)t.nc[u]; p.V.acc_u = u; p.V.acc_w = 'V';
    p.m = t.m[u];
    p.n = t.nc[u];
    p.k = slotc(ACCB, u);
    p.kmax = acc_kmax[u];
    return p;
  }
  Ref acc_dense(int32_t u) {
    acc_need_d[u] = 1;
    Ref r;
    r.base = ACCB;
    r.ld = (int32_t)t.m[u];
    r.acc_u = u;
    r.acc_w = 'D';
    return r;
  }
  void need_lr(int32_t u, int64_t k) {
    const int64_t prev = acc_has_lr[u] ? acc_need_lr[u] : 0;
    acc_need_lr[u] = std::max(std::max(prev, k), acc_cap(u));
    acc_has_lr[u] = 1;
  }
  void acc_fold(int32_t u, const Pay& p) {
    const int64_t m = t.m[u], n = t.nc[u];
    updates++;
    rd(obj(OBJ_A, 0, u));
    wr(obj(OBJ_A, 0, u));
    const int8_t st = acc_state[u];
    if (st == 0) {
      if (p.kind == 'D') {
        copy((int32_t)m, (int32_t)n, 1.0, p.ref, acc_dense(u));
        acc_state[u] = 'D';
      } else {
        need_lr(u, p.kmax);
        acc_kmax[u] = p.kmax;
        Pay a = acc_lr(u);
        setrank(a.k, 0);
        append(a.U, a.V, m, n, 0, u, a.k, p, 0, 0);
        acc_state[u] = 'R';
      }
      return;
    }
    if (st == 'D' || p.kind == 'D') {
      Ref D = acc_dense(u);
      if (st == 'R') {
        Pay a = acc_lr(u);
        gemm_c((int32_t)m, (int32_t)n, a.k, 1.0, a.U, false, a.V, true, D, false);
        add((int32_t)m, (int32_t)n, 1.0, p.ref, D);
      } else if (p.kind == 'D') {
        add((int32_t)m, (int32_t)n, 1.0, p.ref, D);
      } else {
        gemm_c((int32_t)m, (int32_t)n, p.k, 1.0, p.U, false, p.V, true, D, true);
      }
      acc_state[u] = 'D';
      return;
    }
    Pay a = acc_lr(u);
    const int64_t mark = top;
    const int64_t kb = a.kmax + p.kmax;
    Ref Ub = sref(m, kb), Vb = sref(n, kb);
    const int32_t cnt = lslot();
    setrank(cnt, 0);
    append(Ub, Vb, m, n, kb, -1, cnt, a, 0, 0);
    append(Ub, Vb, m, n, kb, -1, cnt, p, 0, 0);
    const int64_t cp = acc_cap(u);
    need_lr(u, cp);
    trunc(m, n, cnt, kb, Ub, Vb, a.U, a.V, a.k, cp);
    acc_kmax[u] = cp;
    top = mark;
  }
  // take: returns state ('D' / 'R' / 0) and the payload
  int8_t acc_take(int32_t u, Pay& p, std::vector<Pending>& pend) {
    rd(obj(OBJ_A, 0, u));
    wr(obj(OBJ_A, 0, u));
    const int8_t st = acc_state[u];
    acc_state[u] = 0;
    pend.swap(acc_pending[u]);
    acc_pending[u].clear();
    if (st == 'D') {
      p.kind = 'D';
      p.ref = acc_dense(u);
      p.m = t.m[u];
      p.n = t.nc[u];
    } else if (st == 'R') {
      p = acc_lr(u);
    }
    return st;
  }
  void add_upd(double a, int xb, int32_t ua, int yb, int32_t ub, int cb, int32_t uc) {
    if (a == 0.0 || err) return;
    if (!(t.leaf[ua] || t.leaf[ub] || t.leaf[uc])) {
      acc_pending[uc].push_back({a, xb, ua, yb, ub});
      return;
    }
    begin(K_ADD_UPD, ua, ub, uc, a);
    Pay p = product(a, xb, ua, yb, ub);
    if (!err) acc_fold(uc, p);
  }
  void shift_upd(int cb, int32_t uc) {
    if (t.leaf[uc]) { err = 2; return; }
    begin(K_SHIFT, uc, -1, -1, 1.0);
    Pay umat;
    std::vector<Pending> pend;
    const int8_t st = acc_take(uc, umat, pend);
    if (st) {
      for (int q = 0; q < 4; ++q) {
        const int32_t ch = t.kids[4 * (size_t)uc + q];
        const int64_t r0 = t.r0[ch] - t.r0[uc], c0 = t.c0[ch] - t.c0[uc];
        Pay s = umat;
        s.m = t.m[ch];
        s.n = t.nc[ch];
        if (umat.kind == 'D') s.ref = umat.ref.at(r0, c0);
        else { s.U = umat.U.at(r0); s.V = umat.V.at(c0); }
        acc_fold(ch, s);
      }
    }
    for (int q = 0; q < 4; ++q) {
      const int32_t ch = t.kids[4 * (size_t)uc + q];
      const int i = q / 2, j = q % 2;
      for (const Pending& pd : pend)
        for (int l = 0; l < 2; ++l) add_upd(pd.alpha, pd.xb, t.kid(pd.ua, i, l), pd.yb, t.kid(pd.ub, l, j), cb, ch);
    }
  }
  void apply_leaf(int cb, int32_t uc) {
    begin(K_APPLY, uc, -1, -1, 1.0);
    Pay umat;
    std::vector<Pending> pend;
    if (acc_take(uc, umat, pend)) fold_leaf(cb, uc, umat);
  }
  void hlu_accu(int32_t u) {
    if (err) return;
    if (!t.leaf[u]) {
      shift_upd(0, u);
      const int32_t a00 = t.kid(u, 0, 0), a01 = t.kid(u, 0, 1), a10 = t.kid(u, 1, 0), a11 = t.kid(u, 1, 1);
      hlu_accu(a00);
      htrsu_accu(2, a00, 0, a10, 1);
      htrsl_accu(1, a00, 0, a01, 2);
      add_upd(-1.0, 1, a10, 2, a01, 0, a11);
      hlu_accu(a11);
      return;
    }
    apply_leaf(0, u);
    begin(K_LEAF_FACTOR, u, -1, -1, 1.0);
    t_factor(u);
  }
  void htrsl_accu(int lb, int32_t ul, int mb, int32_t um, int xb) {
    if (err) return;
    if (!t.leaf[um]) {
      shift_upd(mb, um);
      const int32_t l00 = t.kid(ul, 0, 0), l10 = t.kid(ul, 1, 0), l11 = t.kid(ul, 1, 1);
      const int32_t m00 = t.kid(um, 0, 0), m01 = t.kid(um, 0, 1), m10 = t.kid(um, 1, 0), m11 = t.kid(um, 1, 1);
      htrsl_accu(lb, l00, mb, m00, xb);
      htrsl_accu(lb, l00, mb, m01, xb);
      add_upd(-1.0, lb, l10, xb, m00, mb, m10);
      add_upd(-1.0, lb, l10, xb, m01, mb, m11);
      htrsl_accu(lb, l11, mb, m10, xb);
      htrsl_accu(lb, l11, mb, m11, xb);
      return;
    }
    apply_leaf(mb, um);
    begin(K_LEAF_SOLVE_L, ul, um, -1, 1.0);
    t_solve_l(lb, ul, mb, um, xb);
  }
  void htrsu_accu(int ubb, int32_t uu, int mb, int32_t um, int xb) {
    if (err) return;
    if (!t.leaf[um]) {
      shift_upd(mb, um);
      const int32_t u00 = t.kid(uu, 0, 0), u01 = t.kid(uu, 0, 1), u11 = t.kid(uu, 1, 1);
      const int32_t m00 = t.kid(um, 0, 0), m01 = t.kid(um, 0, 1), m10 = t.kid(um, 1, 0), m11 = t.kid(um, 1, 1);
      htrsu_accu(ubb, u00, mb, m00, xb);
      htrsu_accu(ubb, u00, mb, m10, xb);
      add_upd(-1.0, xb, m00, ubb, u01, mb, m01);
      add_upd(-1.0, xb, m10, ubb, u01, mb, m11);
      htrsu_accu(ubb, u11, mb, m01, xb);
      htrsu_accu(ubb, u11, mb, m11, xb);
      return;
    }
    apply_leaf(mb, um);
    begin(K_LEAF_SOLVE_U, uu, um, -1, 1.0);
    t_solve_u(ubb, uu, mb, um, xb);
  }
};

}  // namespace

// ===========================================================================
// packed program + execution graph (the opaque handle of hmx_lower.h)
// ===========================================================================
struct hmx_prog {
  std::vector<hmx_op> ops;
  std::vector<int64_t> task_ops;
  std::vector<int32_t> kind, u0, u1, u2;
  std::vector<double> alpha;
  std::vector<int64_t> task_scratch;
  std::vector<int64_t> d_off, u_off, v_off, cap;
  int64_t lay_size = 1, acc_size = 1, ws_size = 1, scratch_doubles = 1, updates = 0;
  int32_t ws_slots = 1, scratch_ranks = 1;
  std::vector<int32_t> root_of;  // group root (program index) of every task
  std::vector<std::pair<int32_t, int32_t>> acc_edges;  // accumulator storage reuse order
  std::vector<std::vector<int64_t>> rds, wrs;
  // execution graph
  std::vector<int64_t> succ_ptr;
  std::vector<int32_t> succ_idx;
  int64_t n_dag_edges = 0, n_extra_edges = 0;
};

namespace {

Table make_table(int32_t n, const int64_t* r0, const int64_t* r1, const int64_t* c0, const int64_t* c1,
                 const int8_t* leaf, const int8_t* adm, const int32_t* kids) {
  Table t;
  t.n = n;
  t.r0.assign(r0, r0 + n);
  t.r1.assign(r1, r1 + n);
  t.c0.assign(c0, c0 + n);
  t.c1.assign(c1, c1 + n);
  t.leaf.assign(leaf, leaf + n);
  t.adm.assign(adm, adm + n);
  t.kids.assign(kids, kids + 4 * (size_t)n);
  t.m.resize(n);
  t.nc.resize(n);
  for (int32_t u = 0; u < n; ++u) {
    t.m[u] = t.r1[u] - t.r0[u];
    t.nc[u] = t.c1[u] - t.c0[u];
  }
  // pre-order leaves and per-subtree leaf ranges (iterative post-order)
  t.leaf_lo.assign(n, 0);
  t.leaf_hi.assign(n, 0);
  std::vector<std::pair<int32_t, int>> st;
  st.push_back({0, 0});
  while (!st.empty()) {
    auto& top = st.back();
    const int32_t u = top.first;
    if (t.leaf[u]) {
      t.leaf_lo[u] = (int32_t)t.leaves.size();
      t.leaves.push_back(u);
      t.leaf_hi[u] = (int32_t)t.leaves.size();
      st.pop_back();
      continue;
    }
    if (top.second == 0) t.leaf_lo[u] = (int32_t)t.leaves.size();
    if (top.second < 4) {
      const int q = top.second++;
      st.push_back({t.kids[4 * (size_t)u + q], 0});
    } else {
      t.leaf_hi[u] = (int32_t)t.leaves.size();
      st.pop_back();
    }
  }
  return t;
}

// Data-flow edges of the sequential program (planner.dataflow_edges): RAW,
// WAW and WAR on every leaf of matrices 0..2, accumulator and workspace
// object; reads of a blocked subtree read all its leaves.  `keep(a, b)`
// filters edges.  Returns predecessor lists per task (sorted unique).
template <class Keep>
void dataflow_preds(const Table& t, const hmx_prog& P, int64_t n_w, Keep keep,
                    std::vector<std::vector<int32_t>>& preds) {
  const int64_t nb = t.n;
  const int64_t nobj = 3 * nb + nb + std::max<int64_t>(n_w, 1);
  std::vector<int32_t> last_w(nobj, -1);
  std::vector<std::vector<int32_t>> readers(nobj);
  const int32_t nt = (int32_t)P.rds.size();
  preds.assign(nt, {});
  std::vector<int32_t> tmp;
  auto oid = [&](int64_t o) -> int64_t {
    const int64_t k = o >> 60, b = (o >> 40) & 0xFFFFF, id = o & MASK40;
    if (k == OBJ_M) return b * nb + id;
    if (k == OBJ_A) return 3 * nb + id;
    return 4 * nb + id;
  };
  for (int32_t ti = 0; ti < nt; ++ti) {
    tmp.clear();
    for (int64_t o : P.rds[ti]) {
      const int64_t k = o >> 60, b = (o >> 40) & 0xFFFFF, u = o & MASK40;
      if (k == OBJ_M && !t.leaf[u]) {
        for (int32_t i = t.leaf_lo[u]; i < t.leaf_hi[u]; ++i) {
          const int64_t id = b * nb + t.leaves[i];
          const int32_t w = last_w[id];
          if (w >= 0 && w != ti && keep(w, ti)) tmp.push_back(w);
          auto& rr = readers[id];
          if (rr.empty() || rr.back() != ti) rr.push_back(ti);
        }
      } else {
        const int64_t id = oid(o);
        const int32_t w = last_w[id];
        if (w >= 0 && w != ti && keep(w, ti)) tmp.push_back(w);
        auto& rr = readers[id];
        if (rr.empty() || rr.back() != ti) rr.push_back(ti);
      }
    }
    for (int64_t o : P.wrs[ti]) {
      const int64_t id = oid(o);
      const int32_t w = last_w[id];
      if (w >= 0 && w != ti && keep(w, ti)) tmp.push_back(w);
      for (int32_t r : readers[id])
        if (r != ti && keep(r, ti)) tmp.push_back(r);
      last_w[id] = ti;
      readers[id].clear();
    }
    std::sort(tmp.begin(), tmp.end());
    tmp.erase(std::unique(tmp.begin(), tmp.end()), tmp.end());
    preds[ti] = tmp;
  }
}

struct KeyHash {
  size_t operator()(const std::tuple<int32_t, int32_t, int32_t, int32_t, int32_t>& k) const {
    uint64_t h = 1469598103934665603ull;
    auto mix = [&](uint64_t v) { h ^= v + 0x9e3779b97f4a7c15ull + (h << 6) + (h >> 2); };
    mix((uint32_t)std::get<0>(k)); mix((uint32_t)std::get<1>(k)); mix((uint32_t)std::get<2>(k));
    mix((uint32_t)std::get<3>(k)); mix((uint32_t)std::get<4>(k));
    return (size_t)h;
  }
};

}  // namespace

extern "C" {

int hmx_lower_hlu(int32_t n_blocks, const int64_t* r0, const int64_t* r1, const int64_t* c0,
                  const int64_t* c1, const int8_t* leaf, const int8_t* adm, const int32_t* kids,
                  int32_t mode, int32_t policy, int32_t fixed_rank, double eps, int64_t rank_cap,
                  int64_t split_min, const int32_t* caps, int64_t acc_budget, hmx_prog** out) {
  if (!out || n_blocks <= 0 || !r0 || !r1 || !c0 || !c1 || !leaf || !adm || !kids) return 1;
  *out = nullptr;
  try {
    Table t = make_table(n_blocks, r0, r1, c0, c1, leaf, adm, kids);
    Lower L(t, policy, fixed_rank, eps, rank_cap, split_min, caps);
    if (mode == 0) L.hlu(0);
    else { L.accu = true; L.hlu_accu(0); }
    if (L.err) return 2;
    hmx_prog* P = new hmx_prog();
    // program order: micro tasks (post-order) before their consumers
    std::vector<int32_t> order;
    order.reserve(L.tops.size());
    {
      std::vector<std::pair<int32_t, bool>> st;
      for (int32_t x0 : L.order) {
        st.push_back({x0, false});
        while (!st.empty()) {
          auto [x, done] = st.back();
          st.pop_back();
          if (done) { order.push_back(x); continue; }
          st.push_back({x, true});
          const auto& pr = L.pre[x];
          for (auto it = pr.rbegin(); it != pr.rend(); ++it) st.push_back({*it, false});
        }
      }
    }
    const size_t nt = order.size();
    std::vector<int32_t> newidx(L.tops.size(), -1);
    for (size_t i = 0; i < nt; ++i) newidx[order[i]] = (int32_t)i;
    // accumulator storage.  Footprint of acc(u): U (m x c), V (n x c), then
    // the dense m x n part, as in planner.pack.  acc_budget <= 0: one region
    // per accumulator in uid order (= planner.pack).  acc_budget > 0:
    // lifetime reuse -- acc(u) lives from its first fold to its take
    // (program order); once the pool exceeds the budget, a new accumulator
    // takes the earliest-freed region of its size class and an execution
    // edge (previous occupant's last task -> new occupant's first task)
    // orders the reuse.
    std::vector<int64_t> acc_u(n_blocks, -1), acc_v(n_blocks, -1), acc_d(n_blocks, -1);
    auto fp_lr = [&](int32_t u) {
      const int64_t c = std::max<int64_t>(L.acc_need_lr[u], 1);
      return L.acc_has_lr[u] ? al(t.m[u] * c) + al(t.nc[u] * c) : 0;
    };
    auto place = [&](int32_t u, int64_t base) {
      if (L.acc_has_lr[u]) {
        acc_u[u] = base;
        acc_v[u] = base + al(t.m[u] * std::max<int64_t>(L.acc_need_lr[u], 1));
      }
      if (L.acc_need_d[u]) acc_d[u] = base + fp_lr(u);
    };
    int64_t curo = 0;
    if (acc_budget <= 0) {
      for (int32_t u = 0; u < n_blocks; ++u) {
        if (!L.acc_has_lr[u] && !L.acc_need_d[u]) continue;
        place(u, curo);
        curo += fp_lr(u) + (L.acc_need_d[u] ? al(t.m[u] * t.nc[u]) : 0);
      }
    } else {
      std::vector<int32_t> first(n_blocks, INT32_MAX), last(n_blocks, -1);
      for (size_t x = 0; x < L.tops.size(); ++x) {
        const int32_t pi = newidx[x];
        for (auto* v : {&L.rds[x], &L.wrs[x]})
          for (int64_t o : *v)
            if ((o >> 60) == OBJ_A) {
              const int32_t u = (int32_t)(o & MASK40);
              first[u] = std::min(first[u], pi);
              last[u] = std::max(last[u], pi);
            }
      }
      auto sclass = [](int64_t fp) {  // size classes: x1.25 steps from 4096 doubles
        int64_t c = 4096;
        while (c < fp) c += std::max<int64_t>(c / 4, 4);
        return c;
      };
      std::vector<int32_t> us;
      for (int32_t u = 0; u < n_blocks; ++u)
        if ((L.acc_has_lr[u] || L.acc_need_d[u]) && last[u] >= 0) us.push_back(u);
      std::sort(us.begin(), us.end(), [&](int32_t a, int32_t b) {
        return first[a] != first[b] ? first[a] < first[b] : a < b;
      });
      std::vector<std::pair<int32_t, int32_t>> heap;  // (last, u), min-heap by last
      auto cmp = [](const std::pair<int32_t, int32_t>& a, const std::pair<int32_t, int32_t>& b) {
        return a.first > b.first;
      };
      std::unordered_map<int64_t, std::vector<std::pair<int64_t, int32_t>>> freeq;  // class -> FIFO
      std::unordered_map<int64_t, size_t> fhead;
      std::vector<int64_t> base(n_blocks, -1), cls(n_blocks, 0);
      for (int32_t u : us) {
        while (!heap.empty() && heap.front().first < first[u]) {
          std::pop_heap(heap.begin(), heap.end(), cmp);
          const int32_t v = heap.back().second;
          heap.pop_back();
          freeq[cls[v]].push_back({base[v], last[v]});
        }
        const int64_t fp = fp_lr(u) + (L.acc_need_d[u] ? al(t.m[u] * t.nc[u]) : 0);
        const int64_t c = sclass(fp);
        cls[u] = c;
        auto& q = freeq[c];
        size_t& h = fhead[c];
        if (curo + c <= acc_budget || h >= q.size()) {
          base[u] = curo;
          curo += c;
        } else {
          base[u] = q[h].first;
          P->acc_edges.push_back({q[h].second, first[u]});
          ++h;
        }
        place(u, base[u]);
        heap.push_back({last[u], u});
        std::push_heap(heap.begin(), heap.end(), cmp);
      }
    }
    P->acc_size = std::max<int64_t>(curo, 1);
    // lazy APPEND capacities
    for (auto& ld : L.lazy_dims) {
      const int32_t ti = (int32_t)(ld.first >> 32), oi = (int32_t)(ld.first & 0xFFFFFFFF);
      L.tops[ti][oi].dim[3] = (int32_t)L.acc_need_lr[ld.second];
    }
    auto resolve = [&](int64_t& r) {
      if (!(r & LAZY)) return;
      const AccRef& a = L.acc_refs[r & (LAZY - 1)];
      const int64_t b = a.w == 'U' ? acc_u[a.u] : (a.w == 'V' ? acc_v[a.u] : acc_d[a.u]);
      r = mref(ACCB, b + a.r + a.c * a.ld);
    };
    size_t nops = 0;
    for (int32_t x : order) nops += L.tops[x].size();
    P->ops.reserve(nops);
    P->task_ops.reserve(nt + 1);
    for (int32_t x : order) {
      P->task_ops.push_back((int64_t)P->ops.size());
      for (hmx_op o : L.tops[x]) {
        for (int q = 0; q < 4; ++q) resolve(o.ref[q]);
        resolve(o.wref);
        P->ops.push_back(o);
      }
      std::vector<hmx_op>().swap(L.tops[x]);
      P->kind.push_back(L.kind[x]);
      P->u0.push_back(L.u0[x]);
      P->u1.push_back(L.u1[x]);
      P->u2.push_back(L.u2[x]);
      P->alpha.push_back(L.alpha[x]);
      P->task_scratch.push_back(L.tpeak[x]);
      P->root_of.push_back(newidx[L.root_of[x]]);
      P->rds.push_back(std::move(L.rds[x]));
      P->wrs.push_back(std::move(L.wrs[x]));
    }
    P->task_ops.push_back((int64_t)P->ops.size());
    P->d_off = std::move(L.d_off);
    P->u_off = std::move(L.u_off);
    P->v_off = std::move(L.v_off);
    P->cap = std::move(L.cap);
    P->lay_size = L.lay_size;
    P->ws_size = std::max<int64_t>(L.wtop, 1);
    P->ws_slots = std::max(L.wslots, 1);
    P->scratch_doubles = std::max<int64_t>(L.peak, 1);
    P->scratch_ranks = std::max(L.rpeak, 1);
    P->updates = L.updates;
    *out = P;
    return 0;
  } catch (const std::bad_alloc&) {
    return 4;
  }
}

int64_t hmx_prog_count(const hmx_prog* P, int32_t what) {
  if (!P) return -1;
  switch (what) {
    case 0: return (int64_t)P->kind.size();
    case 1: return (int64_t)P->ops.size();
    case 2: return P->lay_size;
    case 3: return P->acc_size;
    case 4: return P->ws_size;
    case 5: return P->ws_slots;
    case 6: return P->scratch_doubles;
    case 7: return P->scratch_ranks;
    case 8: return P->updates;
    case 9: return P->succ_ptr.empty() ? -1 : P->succ_ptr.back();
    case 10: return P->n_dag_edges;
    case 11: return P->n_extra_edges;
    default: return -1;
  }
}

int hmx_prog_export(const hmx_prog* P, hmx_op* ops, int64_t* task_ops, int32_t* kind, int32_t* uids,
                    double* alpha, int64_t* task_scratch, int64_t* d_off, int64_t* u_off, int64_t* v_off,
                    int64_t* cap) {
  if (!P) return 1;
  const size_t nt = P->kind.size(), nb = P->d_off.size();
  if (ops) std::memcpy(ops, P->ops.data(), P->ops.size() * sizeof(hmx_op));
  if (task_ops) std::memcpy(task_ops, P->task_ops.data(), (nt + 1) * sizeof(int64_t));
  if (kind) std::memcpy(kind, P->kind.data(), nt * sizeof(int32_t));
  if (uids)
    for (size_t i = 0; i < nt; ++i) {
      uids[3 * i] = P->u0[i];
      uids[3 * i + 1] = P->u1[i];
      uids[3 * i + 2] = P->u2[i];
    }
  if (alpha) std::memcpy(alpha, P->alpha.data(), nt * sizeof(double));
  if (task_scratch) std::memcpy(task_scratch, P->task_scratch.data(), nt * sizeof(int64_t));
  if (d_off) std::memcpy(d_off, P->d_off.data(), nb * sizeof(int64_t));
  if (u_off) std::memcpy(u_off, P->u_off.data(), nb * sizeof(int64_t));
  if (v_off) std::memcpy(v_off, P->v_off.data(), nb * sizeof(int64_t));
  if (cap) std::memcpy(cap, P->cap.data(), nb * sizeof(int64_t));
  return 0;
}

// Execution graph.  mode 0 (std): the DAG's edges mapped to program tasks
// (+ micro-task edges); mode 1 (accu): data-flow edges.  `dag` supplies the
// node set (asserted equal to the planned tasks) and, for std, the edges.
// Returns 0; 1 bad argument; 5 planned tasks differ from the DAG's nodes;
// 6 an edge contradicts program order.
int hmx_prog_graph(hmx_prog* P, int32_t n_blocks, const int64_t* r0, const int64_t* r1,
                   const int64_t* c0, const int64_t* c1, const int8_t* leaf, const int8_t* adm,
                   const int32_t* kids, int32_t mode, const hmx_dag* dag) {
  if (!P || !dag) return 1;
  try {
    Table t = make_table(n_blocks, r0, r1, c0, c1, leaf, adm, kids);
    const int64_t nd = hmx_dag_nodes(dag), ne = hmx_dag_edges(dag);
    std::vector<int32_t> dk(nd), dnm(nd), dmids(3 * nd), dnu(nd), duids(3 * nd), didx(std::max<int64_t>(ne, 1));
    std::vector<double> dal(nd);
    std::vector<int64_t> dptr(nd + 1);
    hmx_dag_export(dag, dk.data(), dnm.data(), dmids.data(), dnu.data(), duids.data(), dal.data(),
                   dptr.data(), didx.data());
    const int32_t nt = (int32_t)P->kind.size();
    typedef std::tuple<int32_t, int32_t, int32_t, int32_t, int32_t> Key;
    std::unordered_map<Key, int32_t, KeyHash> pos;
    pos.reserve(nt * 2);
    int32_t n_plain = 0;
    for (int32_t i = 0; i < nt; ++i) {
      if (P->kind[i] == K_MICRO) continue;
      Key k{P->kind[i], P->u0[i], P->u1[i], P->u2[i], P->alpha[i] < 0 ? -1 : 1};
      if (!pos.emplace(k, i).second) return 5;
      ++n_plain;
    }
    std::vector<int32_t> d2p(nd);
    for (int64_t i = 0; i < nd; ++i) {
      int32_t u[3] = {-1, -1, -1};
      for (int q = 0; q < dnu[i]; ++q) u[q] = duids[3 * i + q];
      Key k{dk[i], u[0], u[1], u[2], dal[i] < 0 ? -1 : 1};
      auto it = pos.find(k);
      if (it == pos.end()) return 5;
      d2p[i] = it->second;
    }
    if (nd != n_plain) return 5;
    int64_t nw = 0;
    for (auto& v : P->rds)
      for (int64_t o : v)
        if ((o >> 60) == OBJ_W) nw = std::max(nw, (o & MASK40) + 1);
    std::vector<std::vector<int32_t>> preds;
    if (mode == 0) {
      bool micro = false;
      for (int32_t i = 0; i < nt; ++i) micro |= (P->kind[i] == K_MICRO);
      if (micro) {
        const std::vector<int32_t>& ro = P->root_of;
        dataflow_preds(t, *P, nw, [&](int32_t a, int32_t b) { return ro[a] == ro[b]; }, preds);
      } else {
        preds.assign(nt, {});
      }
      // micro tasks of each group root
      std::vector<std::vector<int32_t>> members(nt);
      for (int32_t i = 0; i < nt; ++i)
        if (P->kind[i] == K_MICRO) members[P->root_of[i]].push_back(i);
      for (int64_t i = 0; i < nd; ++i) {
        const int32_t a = d2p[i];
        for (int64_t e = dptr[i]; e < dptr[i + 1]; ++e) {
          const int32_t b = d2p[didx[e]];
          preds[b].push_back(a);
          for (int32_t mt : members[b]) preds[mt].push_back(a);
        }
      }
      P->n_dag_edges = ne;
    } else {
      dataflow_preds(t, *P, nw, [](int32_t, int32_t) { return true; }, preds);
      P->n_dag_edges = ne;
    }
    for (auto& e : P->acc_edges) preds[e.second].push_back(e.first);
    // successor CSR (sorted), order check
    std::vector<int64_t> cnt(nt + 1, 0);
    int64_t tot = 0;
    for (int32_t b = 0; b < nt; ++b) {
      auto& p = preds[b];
      std::sort(p.begin(), p.end());
      p.erase(std::unique(p.begin(), p.end()), p.end());
      for (int32_t a : p) {
        if (a >= b) return 6;
        cnt[a + 1]++;
      }
      tot += (int64_t)p.size();
    }
    for (int32_t i = 0; i < nt; ++i) cnt[i + 1] += cnt[i];
    P->succ_ptr = cnt;
    P->succ_idx.assign(tot, 0);
    std::vector<int64_t> fill(cnt.begin(), cnt.end() - 1);
    for (int32_t b = 0; b < nt; ++b)
      for (int32_t a : preds[b]) P->succ_idx[fill[a]++] = b;  // b increasing: rows stay sorted
    // extra edges vs the DAG's own (mapped) edge count: informational
    P->n_extra_edges = tot - (mode == 0 ? std::min<int64_t>(tot, ne) : 0);
    return 0;
  } catch (const std::bad_alloc&) {
    return 4;
  }
}

int hmx_prog_graph_export(const hmx_prog* P, int64_t* succ_ptr, int32_t* succ_idx) {
  if (!P || P->succ_ptr.empty()) return 1;
  if (succ_ptr) std::memcpy(succ_ptr, P->succ_ptr.data(), P->succ_ptr.size() * sizeof(int64_t));
  if (succ_idx) std::memcpy(succ_idx, P->succ_idx.data(), P->succ_idx.size() * sizeof(int32_t));
  return 0;
}

// Free the per-task data-access records (after the graph is built).
void hmx_prog_drop_access(hmx_prog* P) {
  if (!P) return;
  std::vector<std::vector<int64_t>>().swap(P->rds);
  std::vector<std::vector<int64_t>>().swap(P->wrs);
}

void hmx_prog_free(hmx_prog* P) { delete P; }

}  // extern "C"
