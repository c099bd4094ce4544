// hmx_dag.cpp — native task-DAG construction by refinement (host C++).
//
// Same node and edge sets as taskgraph.build_hlu_dag (the Python builder,
// itself bit-exact to the reference's taskgraph.py:66-665, Alg. 10-12 and
// 14-15 of arXiv 1911.07531): tasks carry data dependencies (matrix id, row
// range, column range); a task precedes another when one of its outputs
// intersects one of the other's inputs; refinement replaces a task by the
// body of its recursive algorithm with local edges among the sub-tasks
// (mutual matches directed by creation order), inherited edges are narrowed
// to sub-tasks, and unrefined tasks retire once their successor sets stop
// changing.  The merged accumulator mode stitches the shift/apply tree of
// the block tree to the arithmetic graph.  Edge sparsification (Alg. 13,
// taskgraph.py:360-432) runs per refinement round against one snapshot of
// the round's edge state, as in the reference.
//
// Tasks live in one arena (indices are stable); successor sets are sorted
// unique int vectors.  Results are independent of container iteration
// order, as in the reference (set semantics, snapshot per round).

#include <stdint.h>

#include <algorithm>
#include <cstring>
#include <iterator>
#include <new>
#include <vector>

#include "../../include/hmx_dag.h"

namespace {

enum Kind : int32_t {
  K_HLU = 0, K_HTRSL, K_HTRSU, K_HMUL, K_ADD_UPD, K_SHIFT_UPD, K_APPLY_UPD,
  K_LEAF_FACTOR, K_LEAF_SOLVE_L, K_LEAF_SOLVE_U, K_LEAF_UPDATE
};
enum Mode : int32_t { M_STD = 0, M_COMBINED = 1, M_MERGED = 2 };
constexpr int MID_A = 0, MID_L = 1, MID_U = 2, ACC_BASE = 3;

struct Dep {
  int64_t mid, r0, r1, c0, c1;
};

struct Task {
  int32_t kind = 0;
  int8_t nm = 0, nu = 0, nin = 0, nout = 0;
  int32_t mids[3] = {0, 0, 0};
  int32_t uids[3] = {0, 0, 0};
  double alpha = 1.0;
  Dep ins[3];
  Dep outs[2];
  std::vector<int32_t> seq;
  std::vector<int32_t> succ;  // sorted unique
  int64_t sub0 = -1;          // refined: sub-tasks are ids [sub0, sub0 + nsub)
  int32_t nsub = 0;
};

inline bool hit(const Dep& o, const Dep& i) {
  return o.mid == i.mid && o.r0 < i.r1 && i.r0 < o.r1 && o.c0 < i.c1 && i.c0 < o.c1;
}

inline bool precedes(const Task& a, const Task& b) {
  if (&a == &b) return false;
  for (int x = 0; x < a.nout; ++x)
    for (int y = 0; y < b.nin; ++y)
      if (hit(a.outs[x], b.ins[y])) return true;
  return false;
}

inline void add_succ(std::vector<int32_t>& s, int32_t v) {
  auto it = std::lower_bound(s.begin(), s.end(), v);
  if (it == s.end() || *it != v) s.insert(it, v);
}

struct Builder {
  int32_t nb;
  const int64_t *r0, *r1, *c0, *c1;
  const int8_t* leaf;
  const int32_t* parent;
  const int32_t* kids;
  int32_t mode;
  int64_t stop;
  std::vector<Task> T;

  int64_t size(int u) const { return std::max(r1[u] - r0[u], c1[u] - c0[u]); }
  bool above(int u) const { return stop <= 0 || size(u) > stop; }
  Dep dep(int64_t mid, int u) const { return Dep{mid, r0[u], r1[u], c0[u], c1[u]}; }

  int32_t push(Task&& t) {
    T.push_back(std::move(t));
    return (int32_t)(T.size() - 1);
  }

  Task factor(int u, std::vector<int32_t> seq) const {
    Task t;
    t.kind = leaf[u] ? K_LEAF_FACTOR : K_HLU;
    t.nm = 3; t.mids[0] = MID_A; t.mids[1] = MID_L; t.mids[2] = MID_U;
    t.nu = 1; t.uids[0] = u;
    t.ins[t.nin++] = dep(MID_A, u);
    if (mode == M_COMBINED && parent[u] >= 0) t.ins[t.nin++] = dep(ACC_BASE + parent[u], u);
    t.outs[t.nout++] = dep(MID_L, u);
    t.outs[t.nout++] = dep(MID_U, u);
    t.seq = std::move(seq);
    return t;
  }

  Task solve(bool lower, int ut, int um, const int32_t* mids, std::vector<int32_t> seq) const {
    Task t;
    t.kind = lower ? (leaf[um] ? K_LEAF_SOLVE_L : K_HTRSL) : (leaf[um] ? K_LEAF_SOLVE_U : K_HTRSU);
    t.nm = 3;
    for (int i = 0; i < 3; ++i) t.mids[i] = mids[i];
    t.nu = 2; t.uids[0] = ut; t.uids[1] = um;
    t.ins[t.nin++] = dep(mids[0], ut);
    t.ins[t.nin++] = dep(mids[1], um);
    if (mode == M_COMBINED && parent[um] >= 0) t.ins[t.nin++] = dep(ACC_BASE + parent[um], um);
    t.outs[t.nout++] = dep(mids[2], um);
    t.seq = std::move(seq);
    return t;
  }

  Task mul(double alpha, int ua, int ub, int uc, const int32_t* mids, std::vector<int32_t> seq) const {
    Task t;
    t.nm = 3;
    for (int i = 0; i < 3; ++i) t.mids[i] = mids[i];
    t.nu = 3; t.uids[0] = ua; t.uids[1] = ub; t.uids[2] = uc;
    t.alpha = alpha;
    t.ins[t.nin++] = dep(mids[0], ua);
    t.ins[t.nin++] = dep(mids[1], ub);
    t.ins[t.nin++] = dep(mids[2], uc);
    t.outs[t.nout++] = dep(mids[2], uc);
    if (mode == M_STD) {
      t.kind = (leaf[ua] || leaf[ub] || leaf[uc]) ? K_LEAF_UPDATE : K_HMUL;
    } else {
      t.kind = K_ADD_UPD;
      if (mode == M_COMBINED) t.outs[t.nout++] = dep(ACC_BASE + uc, uc);
    }
    t.seq = std::move(seq);
    return t;
  }

  Task shift_or_apply(bool is_apply, int u, std::vector<int32_t> seq) const {
    Task t;
    t.kind = is_apply ? K_APPLY_UPD : K_SHIFT_UPD;
    t.nm = 1; t.mids[0] = MID_A;
    t.nu = 1; t.uids[0] = u;
    if (parent[u] >= 0) t.ins[t.nin++] = dep(ACC_BASE + parent[u], u);
    t.ins[t.nin++] = dep(ACC_BASE + u, u);
    t.outs[t.nout++] = is_apply ? dep(MID_A, u) : dep(ACC_BASE + u, u);
    t.seq = std::move(seq);
    return t;
  }

  bool refinable(const Task& t) const {
    switch (t.kind) {
      case K_HLU: return above(t.uids[0]);
      case K_HTRSL:
      case K_HTRSU: return above(t.uids[1]);
      case K_HMUL: return above(t.uids[2]);
      case K_ADD_UPD: {
        const int a = t.uids[0], b = t.uids[1], c = t.uids[2];
        return !(leaf[a] || leaf[b] || leaf[c]) && above(c);
      }
      default: return false;
    }
  }

  static std::vector<int32_t> ext(const std::vector<int32_t>& s, int32_t i) {
    std::vector<int32_t> o(s);
    o.push_back(i);
    return o;
  }

  // refinement bodies (taskgraph.py:233-312); returns false on a structural error
  bool refine(int32_t id) {
    Task& t0 = T[id];
    if (t0.nsub) return true;
    const std::vector<int32_t> s = t0.seq;
    const int32_t kind = t0.kind;
    const double alpha = t0.alpha;
    int32_t mids[3] = {t0.mids[0], t0.mids[1], t0.mids[2]};
    int32_t uids[3] = {t0.uids[0], t0.uids[1], t0.uids[2]};
    const bool comb = mode == M_COMBINED;
    std::vector<Task> out;
    if (kind == K_HLU) {
      const int u = uids[0];
      if (leaf[u]) return false;
      const int32_t* k = kids + 4 * (int64_t)u;
      int i = 0;
      if (comb) { out.push_back(shift_or_apply(false, u, ext(s, 0))); i = 1; }
      const int32_t m_uaL[3] = {MID_U, MID_A, MID_L}, m_laU[3] = {MID_L, MID_A, MID_U};
      const int32_t m_luA[3] = {MID_L, MID_U, MID_A};
      out.push_back(factor(k[0], ext(s, i)));
      out.push_back(solve(false, k[0], k[2], m_uaL, ext(s, i + 1)));
      out.push_back(solve(true, k[0], k[1], m_laU, ext(s, i + 2)));
      out.push_back(mul(-1.0, k[2], k[1], k[3], m_luA, ext(s, i + 3)));
      out.push_back(factor(k[3], ext(s, i + 4)));
    } else if (kind == K_HTRSL || kind == K_HTRSU) {
      const int ut = uids[0], um = uids[1];
      if (leaf[um] || leaf[ut]) return false;
      const int32_t* kt = kids + 4 * (int64_t)ut;
      const int32_t* km = kids + 4 * (int64_t)um;
      const int32_t m_t = mids[0], m_m = mids[1], m_x = mids[2];
      int i = 0;
      if (comb) { out.push_back(shift_or_apply(false, um, ext(s, 0))); i = 1; }
      if (kind == K_HTRSL) {
        const int32_t mm[3] = {m_t, m_x, m_m};
        out.push_back(solve(true, kt[0], km[0], mids, ext(s, i)));
        out.push_back(solve(true, kt[0], km[1], mids, ext(s, i + 1)));
        out.push_back(mul(-1.0, kt[2], km[0], km[2], mm, ext(s, i + 2)));
        out.push_back(mul(-1.0, kt[2], km[1], km[3], mm, ext(s, i + 3)));
        out.push_back(solve(true, kt[3], km[2], mids, ext(s, i + 4)));
        out.push_back(solve(true, kt[3], km[3], mids, ext(s, i + 5)));
      } else {
        const int32_t mm[3] = {m_x, m_t, m_m};
        out.push_back(solve(false, kt[0], km[0], mids, ext(s, i)));
        out.push_back(solve(false, kt[0], km[2], mids, ext(s, i + 1)));
        out.push_back(mul(-1.0, km[0], kt[1], km[1], mm, ext(s, i + 2)));
        out.push_back(mul(-1.0, km[2], kt[1], km[3], mm, ext(s, i + 3)));
        out.push_back(solve(false, kt[3], km[1], mids, ext(s, i + 4)));
        out.push_back(solve(false, kt[3], km[3], mids, ext(s, i + 5)));
      }
    } else if (kind == K_HMUL || kind == K_ADD_UPD) {
      const int ua = uids[0], ub = uids[1], uc = uids[2];
      if (leaf[ua] || leaf[ub] || leaf[uc]) return false;
      const int32_t* ka = kids + 4 * (int64_t)ua;
      const int32_t* kb = kids + 4 * (int64_t)ub;
      const int32_t* kc = kids + 4 * (int64_t)uc;
      int n = 0;
      for (int i = 0; i < 2; ++i)
        for (int j = 0; j < 2; ++j)
          for (int l = 0; l < 2; ++l) {
            out.push_back(mul(alpha, ka[2 * i + l], kb[2 * l + j], kc[2 * i + j], mids, ext(s, n)));
            ++n;
          }
    } else {
      return false;
    }
    const int64_t base = (int64_t)T.size();
    const int32_t nsub = (int32_t)out.size();
    for (auto& x : out) T.push_back(std::move(x));
    // automatic local edges, mutual matches directed by creation order
    for (int32_t x = 0; x < nsub; ++x)
      for (int32_t y = x + 1; y < nsub; ++y) {
        Task& a = T[base + x];
        Task& b = T[base + y];
        if (precedes(a, b)) add_succ(a.succ, (int32_t)(base + y));
        else if (precedes(b, a)) add_succ(b.succ, (int32_t)(base + x));
      }
    T[id].sub0 = base;
    T[id].nsub = nsub;
    return true;
  }
};

}  // namespace

struct hmx_dag {  // the opaque handle of include/hmx_dag.h
  std::vector<int32_t> kind, nm, mids, nu, uids;
  std::vector<double> alpha;
  std::vector<int64_t> ptr;
  std::vector<int32_t> idx;
};

namespace {

// Alg. 13 over one refinement round (taskgraph.py:384-432, _sparsify_batch):
// for every target t, the neighbourhood n = (sub-tasks of t, or t) plus the
// successors of t (their sub-tasks when refined); every pruned task tp
// (t's sub-tasks, or t) loses the successors that are also reachable from
// it by a path of length in [2, cap] inside n (remove_redundant /
// _bfs_ge2, taskgraph.py:360-381).  All decisions read the round's edge
// state before any removal is committed, so the result is independent of
// the target order.
struct Sparsifier {
  std::vector<int32_t> in_n, seen, out;  // epoch stamps per task id
  int32_t ep_n = 0, ep = 0;

  void fit(size_t n) {
    if (in_n.size() < n) { in_n.resize(n, 0); seen.resize(n, 0); out.resize(n, 0); }
  }

  void run(std::vector<Task>& T, const std::vector<int32_t>& targets, int cap) {
    fit(T.size());
    std::vector<std::pair<int32_t, std::vector<int32_t>>> dec;
    std::vector<int32_t> frontier, nxt;
    for (int32_t t : targets) {
      const Task& tt = T[t];
      ++ep_n;
      auto mark = [&](int32_t u) { in_n[u] = ep_n; };
      if (tt.nsub) for (int32_t x = 0; x < tt.nsub; ++x) mark((int32_t)(tt.sub0 + x));
      else mark(t);
      for (int32_t h : tt.succ) {
        const Task& th = T[h];
        if (th.nsub) for (int32_t y = 0; y < th.nsub; ++y) mark((int32_t)(th.sub0 + y));
        else mark(h);
      }
      const int32_t np = tt.nsub ? tt.nsub : 1;
      for (int32_t x = 0; x < np; ++x) {
        const int32_t tp = tt.nsub ? (int32_t)(tt.sub0 + x) : t;
        ++ep;
        frontier.clear();
        for (int32_t s : T[tp].succ)
          if (in_n[s] == ep_n) { frontier.push_back(s); seen[s] = ep; }
        for (int depth = 1; !frontier.empty() && depth < cap; ++depth) {
          nxt.clear();
          for (int32_t u : frontier)
            for (int32_t v : T[u].succ)
              if (in_n[v] == ep_n) {
                out[v] = ep;
                if (seen[v] != ep) { seen[v] = ep; nxt.push_back(v); }
              }
          frontier.swap(nxt);
        }
        std::vector<int32_t> rem;
        for (int32_t s : T[tp].succ)
          if (out[s] == ep) rem.push_back(s);
        if (!rem.empty()) dec.emplace_back(tp, std::move(rem));
      }
    }
    for (auto& d : dec) {  // commit (successor sets and rem are sorted)
      std::vector<int32_t>& s = T[d.first].succ;
      std::vector<int32_t> keep;
      keep.reserve(s.size());
      std::set_difference(s.begin(), s.end(), d.second.begin(), d.second.end(),
                          std::back_inserter(keep));
      s.swap(keep);
    }
  }
};

}  // namespace

extern "C" {

// Builds the H-LU (root_op 0) or standalone multiply / solve (1 hmul,
// 2 htrsl, 3 htrsu) DAG over a block table (pre-order uids; kids n x 4,
// parent n); mode 0 std, 1 accu-combined, 2 accu-merged.  Returns 0, or
// 1 bad argument, 2 structural error, 3 cycle / edge into a non-final task.
int hmx_dag_build(int32_t nb, const int64_t* r0, const int64_t* r1, const int64_t* c0,
                  const int64_t* c1, const int8_t* leaf, const int32_t* parent, const int32_t* kids,
                  int32_t mode, int64_t stop_size, int32_t root_op, hmx_dag** out) {
  return hmx_dag_build_ex(nb, r0, r1, c0, c1, leaf, parent, kids, mode, stop_size, root_op, 0, 2,
                          out);
}

// As hmx_dag_build, plus edge sparsification (compute_dag's sparsify /
// max_path_len, taskgraph.py:530-590); not valid in combined mode
// (taskgraph.py:652-653).
int hmx_dag_build_ex(int32_t nb, const int64_t* r0, const int64_t* r1, const int64_t* c0,
                     const int64_t* c1, const int8_t* leaf, const int32_t* parent,
                     const int32_t* kids, int32_t mode, int64_t stop_size, int32_t root_op,
                     int32_t sparsify, int32_t max_path_len, hmx_dag** out) {
  if (!out || nb <= 0 || mode < 0 || mode > 2) return 1;
  if (sparsify && (mode == M_COMBINED || max_path_len < 1)) return 1;
  Sparsifier sp;
  std::vector<int32_t> starg;
  Builder b{nb, r0, r1, c0, c1, leaf, parent, kids, mode, stop_size, {}};
  b.T.reserve(1 << 16);
  const std::vector<int32_t> rseq{mode == M_MERGED ? 1 : 0};
  const int32_t m_alu[3] = {MID_A, MID_L, MID_U}, m_lau[3] = {MID_L, MID_A, MID_U};
  const int32_t m_ual[3] = {MID_U, MID_A, MID_L};
  int32_t root;
  switch (root_op) {
    case 0: root = b.push(b.factor(0, rseq)); break;
    case 1: root = b.push(b.mul(1.0, 0, 0, 0, m_alu, rseq)); break;
    case 2: root = b.push(b.solve(true, 0, 0, m_lau, rseq)); break;
    case 3: root = b.push(b.solve(false, 0, 0, m_ual, rseq)); break;
    default: return 1;
  }
  std::vector<int32_t> retired, current{root}, nxt;
  int rounds = 0;
  while (!current.empty()) {
    if (++rounds > 10000) return 3;
    for (int32_t g : current)
      if (b.T[g].nsub == 0 && b.refinable(b.T[g]))
        if (!b.refine(g)) return 2;
    nxt.clear();
    starg.clear();
    for (int32_t g : current) {
      Task& tg = b.T[g];
      if (tg.nsub) {
        if (sparsify) starg.push_back(g);
        // inherited edges become edges between sub-tasks
        const std::vector<int32_t> succ = tg.succ;
        for (int32_t h : succ) {
          const Task& th = b.T[h];
          const int64_t h0 = th.nsub ? th.sub0 : h;
          const int32_t hn = th.nsub ? th.nsub : 1;
          for (int32_t x = 0; x < tg.nsub; ++x) {
            const int32_t tp = (int32_t)(tg.sub0 + x);
            for (int32_t y = 0; y < hn; ++y) {
              const int32_t sv = (int32_t)(h0 + y);
              if (tp != sv && precedes(b.T[tp], b.T[sv])) add_succ(b.T[tp].succ, sv);
            }
          }
        }
        for (int32_t x = 0; x < tg.nsub; ++x) nxt.push_back((int32_t)(tg.sub0 + x));
      } else {
        // narrow edges to refined successors' sub-tasks
        std::vector<int32_t> nn;
        for (int32_t h : tg.succ) {
          const Task& th = b.T[h];
          if (th.nsub) {
            for (int32_t y = 0; y < th.nsub; ++y) {
              const int32_t sv = (int32_t)(th.sub0 + y);
              if (precedes(tg, b.T[sv])) nn.push_back(sv);
            }
          } else {
            nn.push_back(h);
          }
        }
        std::sort(nn.begin(), nn.end());
        nn.erase(std::unique(nn.begin(), nn.end()), nn.end());
        if (nn != tg.succ) {
          tg.succ.swap(nn);
          nxt.push_back(g);
        } else {
          retired.push_back(g);
          if (sparsify) starg.push_back(g);
        }
      }
    }
    if (sparsify && !starg.empty()) sp.run(b.T, starg, max_path_len);
    current.swap(nxt);
  }
  std::vector<int32_t> nodes = retired;
  if (mode == M_MERGED && root_op == 0) {
    // shift/apply tree over the block tree (taskgraph.py:616-633) + stitching
    std::vector<int32_t> acc(nb, -1);
    struct Item { int u; std::vector<int32_t> seq; int32_t par; };
    std::vector<Item> todo;
    todo.push_back({0, {0}, -1});
    while (!todo.empty()) {
      Item it = std::move(todo.back());
      todo.pop_back();
      const int u = it.u;
      const bool terminal = leaf[u] || !b.above(u);
      const int32_t t = b.push(b.shift_or_apply(terminal, u, it.seq));
      acc[u] = t;
      if (it.par >= 0) add_succ(b.T[it.par].succ, t);
      if (!terminal)
        for (int k = 3; k >= 0; --k) {
          std::vector<int32_t> s2 = it.seq;
          s2.push_back(k);
          todo.push_back({kids[4 * (int64_t)u + k], std::move(s2), t});
        }
    }
    for (int32_t t : retired) {
      Task& x = b.T[t];
      if (x.kind == K_HLU || x.kind == K_LEAF_FACTOR) add_succ(b.T[acc[x.uids[0]]].succ, t);
      else if (x.kind == K_HTRSL || x.kind == K_HTRSU || x.kind == K_LEAF_SOLVE_L ||
               x.kind == K_LEAF_SOLVE_U)
        add_succ(b.T[acc[x.uids[1]]].succ, t);
      else if (x.kind == K_ADD_UPD) add_succ(x.succ, acc[x.uids[2]]);
    }
    for (int u = 0; u < nb; ++u)
      if (acc[u] >= 0) nodes.push_back(acc[u]);
  }
  // final order: by creation sequence (lexicographic)
  std::sort(nodes.begin(), nodes.end(),
            [&](int32_t a, int32_t c) { return b.T[a].seq < b.T[c].seq; });
  std::vector<int32_t> pos(b.T.size(), -1);
  for (size_t i = 0; i < nodes.size(); ++i) pos[nodes[i]] = (int32_t)i;
  hmx_dag* d = new (std::nothrow) hmx_dag();
  if (!d) return 1;
  const size_t n = nodes.size();
  d->kind.resize(n); d->nm.resize(n); d->nu.resize(n); d->alpha.resize(n);
  d->mids.resize(3 * n); d->uids.resize(3 * n); d->ptr.resize(n + 1);
  d->ptr[0] = 0;
  for (size_t i = 0; i < n; ++i) {
    const Task& x = b.T[nodes[i]];
    d->kind[i] = x.kind; d->nm[i] = x.nm; d->nu[i] = x.nu; d->alpha[i] = x.alpha;
    for (int j = 0; j < 3; ++j) { d->mids[3 * i + j] = x.mids[j]; d->uids[3 * i + j] = x.uids[j]; }
    std::vector<int32_t> s;
    s.reserve(x.succ.size());
    for (int32_t v : x.succ) {
      if (pos[v] < 0) { delete d; return 3; }
      s.push_back(pos[v]);
    }
    std::sort(s.begin(), s.end());
    d->idx.insert(d->idx.end(), s.begin(), s.end());
    d->ptr[i + 1] = (int64_t)d->idx.size();
  }
  // acyclicity (Kahn)
  std::vector<int32_t> indeg(n, 0), ready;
  for (int32_t v : d->idx) indeg[v]++;
  for (size_t i = 0; i < n; ++i)
    if (!indeg[i]) ready.push_back((int32_t)i);
  size_t seen = 0;
  while (!ready.empty()) {
    const int32_t u = ready.back();
    ready.pop_back();
    ++seen;
    for (int64_t e = d->ptr[u]; e < d->ptr[u + 1]; ++e)
      if (--indeg[d->idx[e]] == 0) ready.push_back(d->idx[e]);
  }
  if (seen != n) { delete d; return 3; }
  *out = d;
  return 0;
}

int64_t hmx_dag_nodes(const hmx_dag* d) { return d ? (int64_t)d->kind.size() : 0; }
int64_t hmx_dag_edges(const hmx_dag* d) { return d ? (int64_t)d->idx.size() : 0; }

int hmx_dag_export(const hmx_dag* d, int32_t* kind, int32_t* nm, int32_t* mids, int32_t* nu,
                   int32_t* uids, double* alpha, int64_t* ptr, int32_t* idx) {
  if (!d) return 1;
  const size_t n = d->kind.size();
  std::memcpy(kind, d->kind.data(), n * sizeof(int32_t));
  std::memcpy(nm, d->nm.data(), n * sizeof(int32_t));
  std::memcpy(nu, d->nu.data(), n * sizeof(int32_t));
  std::memcpy(mids, d->mids.data(), 3 * n * sizeof(int32_t));
  std::memcpy(uids, d->uids.data(), 3 * n * sizeof(int32_t));
  std::memcpy(alpha, d->alpha.data(), n * sizeof(double));
  std::memcpy(ptr, d->ptr.data(), (n + 1) * sizeof(int64_t));
  std::memcpy(idx, d->idx.data(), d->idx.size() * sizeof(int32_t));
  return 0;
}

void hmx_dag_free(hmx_dag* d) { delete d; }

// ASAP wavefront of every node of a CSR graph (Kahn): level[v] = length of
// the longest path from a source to v.  Returns 0, 1 bad argument, 3 cycle.
int hmx_dag_levels(int64_t n, const int64_t* ptr, const int32_t* idx, int32_t* level) {
  if (n < 0 || (n > 0 && (!ptr || !level))) return 1;
  const int64_t ne = n ? ptr[n] : 0;
  for (int64_t e = 0; e < ne; ++e)
    if (idx[e] < 0 || idx[e] >= n) return 1;
  std::vector<int32_t> indeg((size_t)n, 0), ready, nxt;
  for (int64_t e = 0; e < ne; ++e) indeg[idx[e]]++;
  for (int64_t i = 0; i < n; ++i) {
    level[i] = 0;
    if (!indeg[i]) ready.push_back((int32_t)i);
  }
  int64_t seen = 0;
  while (!ready.empty()) {
    nxt.clear();
    for (int32_t u : ready) {
      ++seen;
      for (int64_t e = ptr[u]; e < ptr[u + 1]; ++e) {
        const int32_t v = idx[e];
        level[v] = std::max(level[v], level[u] + 1);
        if (--indeg[v] == 0) nxt.push_back(v);
      }
    }
    ready.swap(nxt);
  }
  return seen == n ? 0 : 3;
}

}  // extern "C"
