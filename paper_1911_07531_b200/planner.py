"""Lowering of H-arithmetic to device op programs.

The planner runs the reference recursions *symbolically* over the block
table — ``arith.hlu`` (arith.py:76-140) for standard H-LU and
``accumulator.hlu_accu`` (accumulator.py:164-235) for the accumulator
variant — and emits, for every leaf-level call, one *task*: a contiguous
list of ``hmx_op`` records that one CTA executes in order.  The tasks are
exactly the final nodes of the refined DAG of taskgraph.build_hlu_dag
(taskgraph.py:636-665):

  leaf_factor   dense_lu of a diagonal leaf              (arith.py:58-73)
  leaf_solve_l  htrsl on a leaf M, L possibly blocked     (hmatrix.py:318-328)
  leaf_solve_u  htrsu on a leaf M, U possibly blocked     (hmatrix.py:331-341)
  leaf_update   product_payload + scatter_payload         (hmatrix.py:367-448)
  add_upd       product_payload + Accumulator.fold        (accumulator.py:60-125)
  shift_upd     restriction of the block's accumulator    (accumulator.py:128-145)
  apply_upd     fold of the accumulator into the leaf     (accumulator.py:148-161)

Everything in these programs is structural (block sizes, operand kinds,
payload kinds, accumulator states) except ranks, which live in device rank
slots and are read by the kernels at run time — so a plan is built once per
block tree and replayed without host round trips.

Storage bases: the caller binds device pools to base ids (H-LU: A=0, L=1,
U=2, accumulators=3); base 15 is the executing CTA's scratch.  Dense
blocks and factors are column-major; a low-rank leaf of an m x n block
owns U (m x cap) and V (n x cap) with ``cap = min(m, n, rank_cap)``.
"""

from __future__ import annotations

import numpy as np

from . import _lib as L
from ._lib import (F_ACC, F_TA, F_TB, OP_ADD, OP_APPEND, OP_COPY, OP_D2LR, OP_GEMM, OP_LU,
                   OP_SETRANK, OP_TRSM_LL, OP_TRSM_UN, OP_TRSM_UT, OP_TRUNC, OP_ZERO, SCRATCH_BASE)
from .trees import BlockTable

ACC_BASE_ID = 3
WS_BASE_ID = 5
ALIGN = 4  # doubles (32 B)


def _al(n):
    return (int(n) + ALIGN - 1) // ALIGN * ALIGN


class Layout:
    """Leaf storage offsets of an H-matrix over a block table."""

    def __init__(self, table: BlockTable, rank_cap=None, caps=None):
        """caps: optional per-uid capacity bound of low-rank leaves (-1 =
        none), the rank-bounded arenas of large problems (hmx_lower.h)."""
        n = table.n
        self.table = table
        self.rank_cap = rank_cap
        self.caps = caps
        self.d_off = np.full(n, -1, dtype=np.int64)
        self.u_off = np.full(n, -1, dtype=np.int64)
        self.v_off = np.full(n, -1, dtype=np.int64)
        self.cap = np.zeros(n, dtype=np.int64)
        cur = 0
        for u in table.leaves(0):
            m, nc = int(table.m[u]), int(table.nc[u])
            if table.adm[u]:
                c = min(m, nc) if rank_cap is None else min(m, nc, int(rank_cap))
                if caps is not None and caps[u] >= 0:
                    c = min(c, int(caps[u]))
                self.cap[u] = c
                self.u_off[u] = cur
                cur += _al(m * c)
                self.v_off[u] = cur
                cur += _al(nc * c)
            else:
                self.d_off[u] = cur
                cur += _al(m * nc)
        self.size = max(cur, 1)

    @classmethod
    def from_arrays(cls, table, rank_cap, d_off, u_off, v_off, cap, size):
        """Layout computed elsewhere (native lowering, lower.py)."""
        lay = cls.__new__(cls)
        lay.table, lay.rank_cap, lay.caps = table, rank_cap, None
        lay.d_off, lay.u_off, lay.v_off, lay.cap = d_off, u_off, v_off, cap
        lay.size = max(int(size), 1)
        return lay

    def same_as(self, other):
        return (self.table is other.table and self.rank_cap == other.rank_cap)


class Ref:
    """Symbolic column-major matrix reference (base, element offset, ld).

    Accumulator refs are resolved lazily (``acc`` = (uid, which, r, c))
    because accumulator capacities are only known after the trace.
    """

    __slots__ = ("base", "off", "ld", "acc")

    def __init__(self, base, off, ld, acc=None):
        self.base, self.off, self.ld, self.acc = base, off, ld, acc

    def at(self, r, c=0):
        if self.acc is not None:
            u, w, r0, c0 = self.acc
            return Ref(self.base, 0, self.ld, (u, w, r0 + r, c0 + c))
        return Ref(self.base, self.off + r + c * self.ld, self.ld)


class PD:
    """Dense payload (m x n)."""

    __slots__ = ("ref", "m", "n")
    kind = "D"

    def __init__(self, ref, m, n):
        self.ref, self.m, self.n = ref, m, n


class PR:
    """Low-rank payload U (m x k) V (n x k); k a dim code, kmax its bound."""

    __slots__ = ("U", "V", "m", "n", "k", "kmax")
    kind = "R"

    def __init__(self, U, V, m, n, k, kmax):
        self.U, self.V, self.m, self.n, self.k, self.kmax = U, V, m, n, k, kmax


class PMat:
    """An operand H-matrix: base id + block table + layout."""

    def __init__(self, base, layout: Layout):
        self.base = base
        self.lay = layout
        self.t = layout.table

    def kind(self, u):
        if not self.t.leaf[u]:
            return "H"
        return "R" if self.t.adm[u] else "D"

    def dense(self, u):
        return Ref(self.base, int(self.lay.d_off[u]), int(self.t.m[u]))

    def lr(self, u):
        m, n = int(self.t.m[u]), int(self.t.nc[u])
        return PR(Ref(self.base, int(self.lay.u_off[u]), m), Ref(self.base, int(self.lay.v_off[u]), n),
                  m, n, L.slot(self.base, u), int(self.lay.cap[u]))

    def rank_slot(self, u):
        return L.slot(self.base, u)


class _Lazy:
    """Deferred integer (accumulator capacity) resolved at pack time."""

    __slots__ = ("fn",)

    def __init__(self, fn):
        self.fn = fn


class Program:
    """Packed op program + task table of one plan."""

    def __init__(self):
        self.ops = None
        self.task_ops = None
        self.keys = []
        self.kinds = []
        self.fold_chains = {}
        self.scratch_doubles = 0
        self.scratch_ranks = 0
        self.acc_size = 1
        self.acc_nslots = 1
        self.updates = 0
        self.static = {}


class Planner:
    """Symbolic executor of the reference recursions; emits op programs."""

    def __init__(self, policy, rank_cap=None, split_min=0):
        self.mode, self.kfix, self.eps = _policy_fields(policy)
        self.rank_cap = rank_cap
        # tasks: op lists, program order (micro-tasks are placed before the
        # task that consumes their results), current task id
        self.task_lists = []
        self.order = []
        self.cur = None
        self.cur_id = -1
        self.keys = []
        self.kinds = []
        self.groups = {}
        # plan workspace (base WS_BASE_ID): results of micro-tasks
        self.split_min = int(split_min)
        self.wtop = 0
        self.wslots = 0
        self.nw = 0
        self.w_info = {}  # micro-task result id -> ([(offset, doubles)], rank slot index or -1)
        self.top = self.peak = 0
        self.peak_task = -1
        self.tpeak = []  # per-task scratch peak (doubles)
        self.rtop = self.rpeak = 0
        self.updates = 0
        # accumulator bookkeeping (accu mode)
        self.acc_state = {}
        self.acc_kmax = {}
        self.acc_pending = {}
        self.acc_need_lr = {}
        self.acc_need_d = set()
        self.fold_chains = {}
        self.acc_table = None
        # per-task data access: reads (objects or subtrees) and writes
        self.rw = []
        self._root_of = {}
        self.pre = {}

    # ------------------------------------------------------------------
    # op emission
    # ------------------------------------------------------------------
    def _op(self, code, flags=0, dims=(0, 0, 0, 0), lds=(0, 0, 0, 0), refs=(None,) * 4,
            slots=(0, 0, 0, 0), iargs=(0, 0, 0, 0), fargs=(0.0, 0.0), wref=None):
        self.cur.append((code, flags, dims, lds, refs, slots, iargs, fargs, wref))

    def _new_task(self, kind, key):
        tid = len(self.task_lists)
        self.task_lists.append([])
        self.kinds.append(kind)
        self.keys.append(key)
        self.rw.append(([], []))
        self.tpeak.append(0)
        self.cur = self.task_lists[tid]
        self.cur_id = tid
        self.top = 0
        self.rtop = 0
        return tid

    def begin(self, kind, key):
        tid = self._new_task(kind, key)
        self.order.append(tid)

    # data-access records: ("m", base, uid) = every leaf of the subtree of
    # uid in matrix `base`; ("a", uid) = accumulator of block uid;
    # ("w", id) = a micro-task result in the plan workspace
    def _rd(self, obj):
        self.rw[self.cur_id][0].append(obj)

    def _wr(self, obj):
        self.rw[self.cur_id][1].append(obj)

    # ------------------------------------------------------------------
    # micro-tasks: a large H x H product is split into its 8 independent
    # quadrant products, each run by its own CTA; results go to the plan
    # workspace and the consuming task (placed after them in program order)
    # combines them.  Parallelism inside a DAG task, same arithmetic.
    # ------------------------------------------------------------------
    def _wref(self, rows, cols):
        off = self.wtop
        self.wtop += _al(max(rows * max(cols, 1), 1))
        return Ref(WS_BASE_ID, off, max(rows, 1))

    def _wslot(self):
        s = self.wslots
        self.wslots += 1
        return L.slot(WS_BASE_ID, s)

    def _micro_product(self, alpha, X, ua, Y, ub, depth):
        parent = (self.cur, self.cur_id, self.top, self.rtop)
        pkey = self.keys[self.cur_id]
        tid = self._new_task("micro_product", ("micro", pkey, ua, ub))
        self.pre.setdefault(parent[1], []).append(tid)
        self.groups.setdefault(self._group_root(parent[1]), []).append(tid)
        self._root_of[tid] = self._group_root(parent[1])
        q = self.product(alpha, X, ua, Y, ub, depth + 1)
        wid = self.nw
        self.nw += 1
        if q.kind == "D":
            W = self._wref(q.m, q.n)
            self.copy(q.m, q.n, 1.0, q.ref, W)
            out = PD(W, q.m, q.n)
            self.w_info[wid] = ([(W.off, _al(max(q.m * max(q.n, 1), 1)))], -1)
        else:
            Wu, Wv = self._wref(q.m, q.kmax), self._wref(q.n, q.kmax)
            self.w_info[wid] = ([(Wu.off, _al(max(q.m * max(q.kmax, 1), 1))),
                                 (Wv.off, _al(max(q.n * max(q.kmax, 1), 1)))], self.wslots)
            ws = self._wslot()
            self.copy(q.m, q.k, 1.0, q.U, Wu)
            self.copy(q.n, q.k, 1.0, q.V, Wv)
            self.setrank(ws, q.k)
            out = PR(Wu, Wv, q.m, q.n, ws, q.kmax)
        self._wr(("w", wid))
        self.cur, self.cur_id, self.top, self.rtop = parent
        self._rd(("w", wid))
        return out

    def _group_root(self, tid):
        return self._root_of.get(tid, tid)

    def alloc(self, n):
        off = self.top
        self.top += _al(max(int(n), 1))
        if self.top > self.tpeak[self.cur_id]:
            self.tpeak[self.cur_id] = self.top
        if self.top > self.peak:
            self.peak = self.top
            self.peak_task = self.cur_id
        return off

    def sref(self, rows, cols):
        return Ref(SCRATCH_BASE, self.alloc(rows * max(cols, 1)), max(rows, 1))

    def lslot(self):
        s = self.rtop
        self.rtop += 1
        self.rpeak = max(self.rpeak, self.rtop)
        return L.slot(SCRATCH_BASE, s)

    def gemm(self, m, n, k, alpha, A, ta, B, tb, C, acc):
        flags = (F_TA if ta else 0) | (F_TB if tb else 0) | (F_ACC if acc else 0)
        self._op(OP_GEMM, flags, (m, n, k, 0), (A.ld, B.ld, C.ld, 0), (A, B, C, None),
                 fargs=(float(alpha), 0.0))

    def copy(self, m, n, alpha, A, C, ta=False):
        self._op(OP_COPY, F_TA if ta else 0, (m, n, 0, 0), (A.ld, 0, C.ld, 0), (A, None, C, None),
                 fargs=(float(alpha), 0.0))

    def zero(self, m, n, C):
        self._op(OP_ZERO, 0, (m, n, 0, 0), (0, 0, C.ld, 0), (None, None, C, None))

    def add(self, m, n, alpha, A, C):
        self._op(OP_ADD, 0, (m, n, 0, 0), (A.ld, 0, C.ld, 0), (A, None, C, None),
                 fargs=(float(alpha), 0.0))

    def setrank(self, slot, value):
        self._op(OP_SETRANK, 0, (value, 0, 0, 0), slots=(slot, 0, 0, 0))

    def append(self, Ud, Vd, M, N, capc, cnt, p, r0, c0):
        self._op(OP_APPEND, 0, (M, N, p.k, capc), (p.U.ld, p.V.ld, Ud.ld, Vd.ld),
                 (p.U, p.V, Ud, Vd), slots=(cnt, 0, 0, 0), iargs=(p.m, p.n, r0, c0))

    def trunc(self, m, n, K, kb, U, V, Uo, Vo, rslot, cap):
        kb = max(int(kb), 1)
        ws = self.sref(L.trunc_scratch(m, n, kb), 1)
        self._op(OP_TRUNC, 0, (m, n, K, 0), (U.ld, V.ld, Uo.ld, Vo.ld), (U, V, Uo, Vo),
                 slots=(rslot, 0, 0, 0), iargs=(self.mode, self.kfix, cap, kb),
                 fargs=(0.0, self.eps), wref=ws)

    def d2lr(self, m, n, M, Uo, Vo, rslot, cap):
        ws = self.sref(L.d2lr_scratch(m, n), 1)
        self._op(OP_D2LR, 0, (m, n, 0, 0), (M.ld, 0, Uo.ld, Vo.ld), (M, None, Uo, Vo),
                 slots=(rslot, 0, 0, 0), iargs=(self.mode, self.kfix, cap, 0),
                 fargs=(0.0, self.eps), wref=ws)

    # ------------------------------------------------------------------
    # H x dense products (hmatrix.py:286-315)
    # ------------------------------------------------------------------
    def hm_apply(self, X: PMat, u, S: Ref, cols, colsmax, out=None, alpha=1.0, row_off=0,
                 fresh=True):
        """out (m_u x cols) (+)= alpha * X[u] @ S; returns out."""
        t = X.t
        m = int(t.m[u])
        if out is None:
            out = self.sref(m, colsmax)
        if fresh:
            self.zero(m, cols, out)
        for v in t.leaves(u):
            r0, c0 = int(t.r0[v] - t.r0[u]), int(t.c0[v] - t.c0[u])
            mv, nv = int(t.m[v]), int(t.nc[v])
            if t.adm[v]:
                p = X.lr(v)
                mark = self.top
                T = self.sref(max(p.kmax, 1), colsmax)
                self.gemm(p.k, cols, nv, 1.0, p.V, True, S.at(c0), False, T, False)
                self.gemm(mv, cols, p.k, alpha, p.U, False, T, False, out.at(row_off + r0), True)
                self.top = mark
            else:
                self.gemm(mv, cols, nv, alpha, X.dense(v), False, S.at(c0), False,
                          out.at(row_off + r0), True)
        return out

    def hm_apply_t(self, X: PMat, u, S: Ref, cols, colsmax, out=None, alpha=1.0, row_off=0,
                   fresh=True):
        """out (n_u x cols) (+)= alpha * X[u]^T @ S."""
        t = X.t
        n = int(t.nc[u])
        if out is None:
            out = self.sref(n, colsmax)
        if fresh:
            self.zero(n, cols, out)
        for v in t.leaves(u):
            r0, c0 = int(t.r0[v] - t.r0[u]), int(t.c0[v] - t.c0[u])
            mv, nv = int(t.m[v]), int(t.nc[v])
            if t.adm[v]:
                p = X.lr(v)
                mark = self.top
                T = self.sref(max(p.kmax, 1), colsmax)
                self.gemm(p.k, cols, mv, 1.0, p.U, True, S.at(r0), False, T, False)
                self.gemm(nv, cols, p.k, alpha, p.V, False, T, False, out.at(row_off + c0), True)
                self.top = mark
            else:
                self.gemm(nv, cols, mv, alpha, X.dense(v), True, S.at(r0), False,
                          out.at(row_off + c0), True)
        return out

    # ------------------------------------------------------------------
    # triangular solves on dense right-hand sides (hmatrix.py:318-341)
    # ------------------------------------------------------------------
    def solve_lower(self, Lm: PMat, u, Y: Ref, cols, colsmax):
        t = Lm.t
        if t.leaf[u]:
            if t.adm[u]:
                raise ValueError("triangular solve on a low-rank diagonal block")
            self._op(OP_TRSM_LL, 0, (int(t.m[u]), cols, 0, 0), (int(t.m[u]), 0, Y.ld, 0),
                     (Lm.dense(u), None, Y, None))
            return
        k00, _, k10, k11 = (int(x) for x in t.kids[u])
        n0 = int(t.m[k00])
        self.solve_lower(Lm, k00, Y, cols, colsmax)
        # Y[n0:] -= hm_apply(l10, Y[:n0])
        self.hm_apply(Lm, k10, Y, cols, colsmax, out=Y, alpha=-1.0, row_off=n0, fresh=False)
        self.solve_lower(Lm, k11, Y.at(n0), cols, colsmax)

    def solve_upper_t(self, Um: PMat, u, Y: Ref, cols, colsmax):
        t = Um.t
        if t.leaf[u]:
            if t.adm[u]:
                raise ValueError("triangular solve on a low-rank diagonal block")
            self._op(OP_TRSM_UT, 0, (int(t.m[u]), cols, 0, 0), (int(t.m[u]), 0, Y.ld, 0),
                     (Um.dense(u), None, Y, None))
            return
        k00, k01, _, k11 = (int(x) for x in t.kids[u])
        n0 = int(t.m[k00])
        self.solve_upper_t(Um, k00, Y, cols, colsmax)
        self.hm_apply_t(Um, k01, Y, cols, colsmax, out=Y, alpha=-1.0, row_off=n0, fresh=False)
        self.solve_upper_t(Um, k11, Y.at(n0), cols, colsmax)

    def solve_upper(self, Um: PMat, u, Y: Ref, cols, colsmax):
        """Y := U[u]^{-1} Y, block back substitution (the non-transposed
        counterpart of solve_upper_t; solve phase)."""
        t = Um.t
        if t.leaf[u]:
            if t.adm[u]:
                raise ValueError("triangular solve on a low-rank diagonal block")
            self._op(OP_TRSM_UN, 0, (int(t.m[u]), cols, 0, 0), (int(t.m[u]), 0, Y.ld, 0),
                     (Um.dense(u), None, Y, None))
            return
        k00, k01, _, k11 = (int(x) for x in t.kids[u])
        n0 = int(t.m[k00])
        self.solve_upper(Um, k11, Y.at(n0), cols, colsmax)
        # Y[:n0] -= hm_apply(u01, Y[n0:])
        self.hm_apply(Um, k01, Y.at(n0), cols, colsmax, out=Y, alpha=-1.0, row_off=0, fresh=False)
        self.solve_upper(Um, k00, Y, cols, colsmax)

    # ------------------------------------------------------------------
    # product payloads (hmatrix.py:367-417)
    # ------------------------------------------------------------------
    def product(self, alpha, X: PMat, ua, Y: PMat, ub, depth=0):
        self._rd(("m", X.base, ua))
        self._rd(("m", Y.base, ub))
        tx, ty = X.t, Y.t
        m, kk, n = int(tx.m[ua]), int(tx.nc[ua]), int(ty.nc[ub])
        if kk != int(ty.m[ub]):
            raise ValueError("non-conformal product")
        kx, ky = X.kind(ua), Y.kind(ub)
        if kx == "R":
            a = X.lr(ua)
            Up = self.sref(m, a.kmax)
            self.copy(m, a.k, alpha, a.U, Up)
            Vp = self.hm_apply_t(Y, ub, a.V, a.k, a.kmax)
            return PR(Up, Vp, m, n, a.k, a.kmax)
        if ky == "R":
            b = Y.lr(ub)
            S = self.sref(kk, b.kmax)
            self.copy(kk, b.k, alpha, b.U, S)
            Up = self.hm_apply(X, ua, S, b.k, b.kmax)
            return PR(Up, b.V, m, n, b.k, b.kmax)
        if kx == "D" and ky == "D":
            P = self.sref(m, n)
            self.gemm(m, n, kk, alpha, X.dense(ua), False, Y.dense(ub), False, P, False)
            return PD(P, m, n)
        if kx == "D":  # Y blocked: (Y^T (alpha A^T))^T
            T = self.sref(kk, m)
            self.copy(kk, m, alpha, X.dense(ua), T, ta=True)
            W = self.hm_apply_t(Y, ub, T, m, m)
            P = self.sref(m, n)
            self.copy(m, n, 1.0, W, P, ta=True)
            return PD(P, m, n)
        if ky == "D":  # X blocked
            S = self.sref(kk, n)
            self.copy(kk, n, alpha, Y.dense(ub), S)
            return PD(self.hm_apply(X, ua, S, n, n), m, n)
        # both blocked: combine the 2x2x2 quadrant payloads; large products
        # run their quadrants as parallel micro-tasks
        split = (self.split_min > 0 and depth < 2 and min(m, n) >= self.split_min
                 and not (tx.leaf[tx.child(ua, 0, 0)] and ty.leaf[ty.child(ub, 0, 0)]))
        parts = []
        dacc = None
        for i in range(2):
            for j in range(2):
                for l in range(2):
                    a_il = tx.child(ua, i, l)
                    b_lj = ty.child(ub, l, j)
                    if split:
                        q = self._micro_product(alpha, X, a_il, Y, b_lj, depth)
                    else:
                        q = self.product(alpha, X, a_il, Y, b_lj, depth + 1)
                    r0 = int(tx.r0[a_il] - tx.r0[ua])
                    c0 = int(ty.c0[b_lj] - ty.c0[ub])
                    if q.kind == "D":
                        if dacc is None:
                            dacc = self.sref(m, n)
                            self.zero(m, n, dacc)
                        self.add(q.m, q.n, 1.0, q.ref, dacc.at(r0, c0))
                    elif q.kmax > 0:
                        parts.append((q, r0, c0))
        if dacc is not None:
            if parts:
                Ub, Vb, cnt, kb = self._stack(parts, m, n)
                self.gemm(m, n, cnt, 1.0, Ub, False, Vb, True, dacc, True)
            return PD(dacc, m, n)
        if not parts:
            return PR(self.sref(m, 1), self.sref(n, 1), m, n, 0, 0)
        Ub, Vb, cnt, kb = self._stack(parts, m, n)
        kout = min(m, n, kb) if self.rank_cap is None else min(m, n, kb, int(self.rank_cap))
        Un, Vn = self.sref(m, kout), self.sref(n, kout)
        rs = self.lslot()
        self.trunc(m, n, cnt, kb, Ub, Vb, Un, Vn, rs, kout)
        return PR(Un, Vn, m, n, rs, kout)

    def _stack(self, parts, m, n):
        """Zero-padded hstack of low-rank parts (hmatrix.py:401-409,412,416)."""
        kb = sum(q.kmax for q, _, _ in parts)
        Ub, Vb = self.sref(m, kb), self.sref(n, kb)
        cnt = self.lslot()
        self.setrank(cnt, 0)
        for q, r0, c0 in parts:
            self.append(Ub, Vb, m, n, kb, cnt, q, r0, c0)
        return Ub, Vb, cnt, kb

    # ------------------------------------------------------------------
    # folds (hmatrix.py:420-448)
    # ------------------------------------------------------------------
    def fold_leaf(self, C: PMat, u, p):
        t = C.t
        m, n = int(t.m[u]), int(t.nc[u])
        if (p.m, p.n) != (m, n):
            raise ValueError("payload does not match destination block")
        self.updates += 1
        self._rd(("m", C.base, u))
        self._wr(("m", C.base, u))
        if not t.adm[u]:
            D = C.dense(u)
            if p.kind == "D":
                self.add(m, n, 1.0, p.ref, D)
            else:
                self.gemm(m, n, p.k, 1.0, p.U, False, p.V, True, D, True)
            return
        c = C.lr(u)
        mark = self.top
        if p.kind == "D":
            M = self.sref(m, n)
            self.gemm(m, n, c.k, 1.0, c.U, False, c.V, True, M, False)
            self.add(m, n, 1.0, p.ref, M)
            self.d2lr(m, n, M, c.U, c.V, C.rank_slot(u), c.kmax)
        else:
            kb = c.kmax + p.kmax
            Ub, Vb = self.sref(m, kb), self.sref(n, kb)
            cnt = self.lslot()
            self.setrank(cnt, 0)
            self.append(Ub, Vb, m, n, kb, cnt, c, 0, 0)
            self.append(Ub, Vb, m, n, kb, cnt, p, 0, 0)
            self.trunc(m, n, cnt, kb, Ub, Vb, c.U, c.V, C.rank_slot(u), c.kmax)
        self.top = mark

    def scatter(self, C: PMat, u, p):
        t = C.t
        if t.leaf[u]:
            self.fold_leaf(C, u, p)
            return
        for ch in t.kids[u]:
            ch = int(ch)
            r0, c0 = int(t.r0[ch] - t.r0[u]), int(t.c0[ch] - t.c0[u])
            mc, nc = int(t.m[ch]), int(t.nc[ch])
            if p.kind == "D":
                q = PD(p.ref.at(r0, c0), mc, nc)
            else:
                q = PR(p.U.at(r0), p.V.at(c0), mc, nc, p.k, p.kmax)
            self.scatter(C, ch, q)

    # ------------------------------------------------------------------
    # leaf tasks
    # ------------------------------------------------------------------
    def t_factor(self, A: PMat, Lm: PMat, Um: PMat, u):
        if A.kind(u) != "D":
            raise ValueError("diagonal leaf must be dense for factorization")
        n = int(A.t.m[u])
        self._rd(("m", A.base, u))
        self._wr(("m", Lm.base, u))
        self._wr(("m", Um.base, u))
        self._op(OP_LU, 0, (n, 0, 0, 0), (n, n, n, 0), (A.dense(u), Lm.dense(u), Um.dense(u), None))

    def t_solve_l(self, Lm: PMat, ul, M: PMat, um, X: PMat):
        self._rd(("m", Lm.base, ul))
        self._rd(("m", M.base, um))
        self._wr(("m", X.base, um))
        t = M.t
        m, n = int(t.m[um]), int(t.nc[um])
        if M.kind(um) == "D":
            D = X.dense(um)
            self.copy(m, n, 1.0, M.dense(um), D)
            self.solve_lower(Lm, ul, D, n, n)
        else:
            a, x = M.lr(um), X.lr(um)
            self.copy(m, a.k, 1.0, a.U, x.U)
            self.copy(n, a.k, 1.0, a.V, x.V)
            self.setrank(x.k, a.k)
            self.solve_lower(Lm, ul, x.U, x.k, x.kmax)

    def t_solve_u(self, Um: PMat, uu, M: PMat, um, X: PMat):
        self._rd(("m", Um.base, uu))
        self._rd(("m", M.base, um))
        self._wr(("m", X.base, um))
        t = M.t
        m, n = int(t.m[um]), int(t.nc[um])
        if M.kind(um) == "D":
            T = self.sref(n, m)
            self.copy(n, m, 1.0, M.dense(um), T, ta=True)
            self.solve_upper_t(Um, uu, T, m, m)
            self.copy(m, n, 1.0, T, X.dense(um), ta=True)
        else:
            a, x = M.lr(um), X.lr(um)
            self.copy(m, a.k, 1.0, a.U, x.U)
            self.copy(n, a.k, 1.0, a.V, x.V)
            self.setrank(x.k, a.k)
            self.solve_upper_t(Um, uu, x.V, x.k, x.kmax)

    # ------------------------------------------------------------------
    # standard recursion (arith.py:40-140)
    # ------------------------------------------------------------------
    def hmul(self, alpha, X: PMat, ua, Y: PMat, ub, C: PMat, uc):
        if alpha == 0.0:
            return
        if not (X.t.leaf[ua] or Y.t.leaf[ub] or C.t.leaf[uc]):
            for i in range(2):
                for j in range(2):
                    for l in range(2):
                        self.hmul(alpha, X, X.t.child(ua, i, l), Y, Y.t.child(ub, l, j), C,
                                  C.t.child(uc, i, j))
            return
        self.begin("leaf_update", ("leaf_update", (ua, ub, uc), alpha))
        self.scatter(C, uc, self.product(alpha, X, ua, Y, ub))

    def hlu(self, A, Lm, Um, u):
        t = A.t
        if not t.leaf[u]:
            a00, a01, a10, a11 = (int(x) for x in t.kids[u])
            self.hlu(A, Lm, Um, a00)
            self.htrsu(Um, a00, A, a10, Lm)
            self.htrsl(Lm, a00, A, a01, Um)
            self.hmul(-1.0, Lm, a10, Um, a01, A, a11)
            self.hlu(A, Lm, Um, a11)
            return
        self.begin("leaf_factor", ("leaf_factor", (u,), 1.0))
        self.t_factor(A, Lm, Um, u)

    def htrsl(self, Lm, ul, M, um, X):
        t = M.t
        if not t.leaf[um]:
            l00, _, l10, l11 = (int(x) for x in Lm.t.kids[ul])
            m00, m01, m10, m11 = (int(x) for x in t.kids[um])
            self.htrsl(Lm, l00, M, m00, X)
            self.htrsl(Lm, l00, M, m01, X)
            self.hmul(-1.0, Lm, l10, X, m00, M, m10)
            self.hmul(-1.0, Lm, l10, X, m01, M, m11)
            self.htrsl(Lm, l11, M, m10, X)
            self.htrsl(Lm, l11, M, m11, X)
            return
        self.begin("leaf_solve_l", ("leaf_solve_l", (ul, um), 1.0))
        self.t_solve_l(Lm, ul, M, um, X)

    def htrsu(self, Um, uu, M, um, X):
        t = M.t
        if not t.leaf[um]:
            u00, u01, _, u11 = (int(x) for x in Um.t.kids[uu])
            m00, m01, m10, m11 = (int(x) for x in t.kids[um])
            self.htrsu(Um, u00, M, m00, X)
            self.htrsu(Um, u00, M, m10, X)
            self.hmul(-1.0, X, m00, Um, u01, M, m01)
            self.hmul(-1.0, X, m10, Um, u01, M, m11)
            self.htrsu(Um, u11, M, m01, X)
            self.htrsu(Um, u11, M, m11, X)
            return
        self.begin("leaf_solve_u", ("leaf_solve_u", (uu, um), 1.0))
        self.t_solve_u(Um, uu, M, um, X)

    # ------------------------------------------------------------------
    # accumulator recursion (accumulator.py:41-235)
    # ------------------------------------------------------------------
    def _acc_cap(self, u):
        t = self.acc_table
        m, n = int(t.m[u]), int(t.nc[u])
        return min(m, n) if self.rank_cap is None else min(m, n, int(self.rank_cap))

    def _acc_lr(self, u):
        t = self.acc_table
        m, n = int(t.m[u]), int(t.nc[u])
        return PR(Ref(ACC_BASE_ID, 0, m, (u, "U", 0, 0)), Ref(ACC_BASE_ID, 0, n, (u, "V", 0, 0)),
                  m, n, L.slot(ACC_BASE_ID, u), self.acc_kmax[u])

    def _acc_dense(self, u):
        t = self.acc_table
        self.acc_need_d.add(u)
        return Ref(ACC_BASE_ID, 0, int(t.m[u]), (u, "D", 0, 0))

    def _need_lr(self, u, k):
        self.acc_need_lr[u] = max(self.acc_need_lr.get(u, 0), int(k), self._acc_cap(u))

    def _chain(self, u):
        self.fold_chains.setdefault(u, []).append(self.cur_id)

    def acc_fold(self, u, p):
        """Accumulator.fold (accumulator.py:60-76) into acc(u)."""
        t = self.acc_table
        m, n = int(t.m[u]), int(t.nc[u])
        self.updates += 1
        self._chain(u)
        self._rd(("a", u))
        self._wr(("a", u))
        st = self.acc_state.get(u)
        if st is None:
            if p.kind == "D":
                self.copy(m, n, 1.0, p.ref, self._acc_dense(u))
                self.acc_state[u] = "D"
            else:
                self._need_lr(u, p.kmax)
                self.acc_kmax[u] = p.kmax
                a = self._acc_lr(u)
                self.setrank(a.k, 0)
                self.append(a.U, a.V, m, n, _Lazy(lambda u=u: self.acc_need_lr[u]), a.k, p, 0, 0)
                self.acc_state[u] = "R"
            return
        if st == "D" or p.kind == "D":
            D = self._acc_dense(u)
            if st == "R":
                a = self._acc_lr(u)
                self.gemm(m, n, a.k, 1.0, a.U, False, a.V, True, D, False)
                self.add(m, n, 1.0, p.ref, D)
            elif p.kind == "D":
                self.add(m, n, 1.0, p.ref, D)
            else:
                self.gemm(m, n, p.k, 1.0, p.U, False, p.V, True, D, True)
            self.acc_state[u] = "D"
            return
        a = self._acc_lr(u)
        mark = self.top
        kb = a.kmax + p.kmax
        Ub, Vb = self.sref(m, kb), self.sref(n, kb)
        cnt = self.lslot()
        self.setrank(cnt, 0)
        self.append(Ub, Vb, m, n, kb, cnt, a, 0, 0)
        self.append(Ub, Vb, m, n, kb, cnt, p, 0, 0)
        cap = self._acc_cap(u)
        self._need_lr(u, cap)
        self.trunc(m, n, cnt, kb, Ub, Vb, a.U, a.V, a.k, cap)
        self.acc_kmax[u] = cap
        self.top = mark

    def _acc_take(self, u):
        self._rd(("a", u))
        self._wr(("a", u))
        st = self.acc_state.pop(u, None)
        pend = self.acc_pending.pop(u, [])
        if st is None:
            return None, pend
        if st == "D":
            t = self.acc_table
            p = PD(self._acc_dense(u), int(t.m[u]), int(t.nc[u]))
        else:
            p = self._acc_lr(u)
        return p, pend

    def add_upd(self, alpha, X, ua, Y, ub, C, uc):
        if alpha == 0.0:
            return
        if not (X.t.leaf[ua] or Y.t.leaf[ub] or C.t.leaf[uc]):
            self.acc_pending.setdefault(uc, []).append((alpha, X, ua, Y, ub))
            return
        self.begin("add_upd", ("add_upd", (ua, ub, uc), alpha))
        self.acc_fold(uc, self.product(alpha, X, ua, Y, ub))

    def shift_upd(self, C, uc):
        t = C.t
        if t.leaf[uc]:
            raise ValueError("shift target must be a structured block")
        self.begin("shift_upd", ("shift_upd", (uc,), 1.0))
        self._chain(uc)  # the take closes the chain of acc(uc)
        umat, pend = self._acc_take(uc)
        kids = [int(x) for x in t.kids[uc]]
        if umat is not None:
            for ch in kids:
                r0, c0 = int(t.r0[ch] - t.r0[uc]), int(t.c0[ch] - t.c0[uc])
                mc, nc = int(t.m[ch]), int(t.nc[ch])
                if umat.kind == "D":
                    q = PD(umat.ref.at(r0, c0), mc, nc)
                else:
                    q = PR(umat.U.at(r0), umat.V.at(c0), mc, nc, umat.k, umat.kmax)
                self.acc_fold(ch, q)
        for idx, ch in enumerate(kids):
            i, j = divmod(idx, 2)
            for alpha, X, ua, Y, ub in pend:
                for l in range(2):
                    self.add_upd(alpha, X, X.t.child(ua, i, l), Y, Y.t.child(ub, l, j), C, ch)

    def apply_leaf(self, C, uc):
        """apply_upd on a leaf (accumulator.py:156-161) — one apply_upd task."""
        self.begin("apply_upd", ("apply_upd", (uc,), 1.0))
        self._chain(uc)
        umat, _ = self._acc_take(uc)
        if umat is not None:
            self.fold_leaf(C, uc, umat)

    def hlu_accu(self, A, Lm, Um, u):
        t = A.t
        if not t.leaf[u]:
            self.shift_upd(A, u)
            a00, a01, a10, a11 = (int(x) for x in t.kids[u])
            self.hlu_accu(A, Lm, Um, a00)
            self.htrsu_accu(Um, a00, A, a10, Lm)
            self.htrsl_accu(Lm, a00, A, a01, Um)
            self.add_upd(-1.0, Lm, a10, Um, a01, A, a11)
            self.hlu_accu(A, Lm, Um, a11)
            return
        self.apply_leaf(A, u)
        self.begin("leaf_factor", ("leaf_factor", (u,), 1.0))
        self.t_factor(A, Lm, Um, u)

    def htrsl_accu(self, Lm, ul, M, um, X):
        t = M.t
        if not t.leaf[um]:
            self.shift_upd(M, um)
            l00, _, l10, l11 = (int(x) for x in Lm.t.kids[ul])
            m00, m01, m10, m11 = (int(x) for x in t.kids[um])
            self.htrsl_accu(Lm, l00, M, m00, X)
            self.htrsl_accu(Lm, l00, M, m01, X)
            self.add_upd(-1.0, Lm, l10, X, m00, M, m10)
            self.add_upd(-1.0, Lm, l10, X, m01, M, m11)
            self.htrsl_accu(Lm, l11, M, m10, X)
            self.htrsl_accu(Lm, l11, M, m11, X)
            return
        self.apply_leaf(M, um)
        self.begin("leaf_solve_l", ("leaf_solve_l", (ul, um), 1.0))
        self.t_solve_l(Lm, ul, M, um, X)

    def htrsu_accu(self, Um, uu, M, um, X):
        t = M.t
        if not t.leaf[um]:
            self.shift_upd(M, um)
            u00, u01, _, u11 = (int(x) for x in Um.t.kids[uu])
            m00, m01, m10, m11 = (int(x) for x in t.kids[um])
            self.htrsu_accu(Um, u00, M, m00, X)
            self.htrsu_accu(Um, u00, M, m10, X)
            self.add_upd(-1.0, X, m00, Um, u01, M, m01)
            self.add_upd(-1.0, X, m10, Um, u01, M, m11)
            self.htrsu_accu(Um, u11, M, m01, X)
            self.htrsu_accu(Um, u11, M, m11, X)
            return
        self.apply_leaf(M, um)
        self.begin("leaf_solve_u", ("leaf_solve_u", (uu, um), 1.0))
        self.t_solve_u(Um, uu, M, um, X)

    # ------------------------------------------------------------------
    # packing
    # ------------------------------------------------------------------
    def pack(self) -> Program:
        prog = Program()
        # accumulator storage layout (lazy refs resolve against it)
        acc_u, acc_v, acc_d, acc_cap = {}, {}, {}, {}
        cur = 0
        t = self.acc_table
        if t is not None:
            for u in sorted(set(self.acc_need_lr) | self.acc_need_d):
                m, n = int(t.m[u]), int(t.nc[u])
                if u in self.acc_need_lr:
                    c = int(self.acc_need_lr[u])
                    acc_cap[u] = c
                    acc_u[u] = cur
                    cur += _al(m * max(c, 1))
                    acc_v[u] = cur
                    cur += _al(n * max(c, 1))
                if u in self.acc_need_d:
                    acc_d[u] = cur
                    cur += _al(m * n)
            prog.acc_nslots = t.n
        prog.acc_size = max(cur, 1)
        prog.acc_offsets = (acc_u, acc_v, acc_d, acc_cap)

        def rv(r):
            if r is None:
                return 0
            if r.acc is not None:
                u, w, r0, c0 = r.acc
                base = {"U": acc_u, "V": acc_v, "D": acc_d}[w][u]
                return L.mref(r.base, base + r0 + c0 * r.ld)
            return L.mref(r.base, r.off)

        def iv(x):
            return int(x.fn()) if isinstance(x, _Lazy) else int(x)

        # program order: micro-tasks before their consumers
        order = []
        stack = []
        for t in self.order:
            # iterative post-order over the micro-task tree of t
            stack.append((t, False))
            while stack:
                x, done = stack.pop()
                if done:
                    order.append(x)
                    continue
                stack.append((x, True))
                for c in reversed(self.pre.get(x, [])):
                    stack.append((c, False))
        newidx = {t: i for i, t in enumerate(order)}
        flat = []
        starts = []
        for t in order:
            starts.append(len(flat))
            flat.extend(self.task_lists[t])
        self.ops = flat
        n = len(self.ops)
        arr = np.zeros(n, dtype=L.OP_DTYPE)
        # columns are gathered as Python lists and converted once (per-row
        # numpy assignment dominated the planning time); lazy dimensions
        # and refs are resolved here, plain ints pass through
        _int = int

        def ivs(t):
            return [x if type(x) is _int else iv(x) for x in t]

        if n:
            code, flags, dims, lds, refs, slots, iargs, fargs, wrefs = zip(*self.ops)
            arr["code"] = np.asarray(code, np.int32)
            arr["flags"] = np.asarray(flags, np.int32)
            arr["dim"] = np.asarray([ivs(d) for d in dims], np.int32).reshape(n, 4)
            arr["ld"] = np.asarray(lds, np.int32).reshape(n, 4)
            arr["ref"] = np.asarray([[rv(x) for x in r] for r in refs], np.int64).reshape(n, 4)
            arr["slot"] = np.asarray(slots, np.int32).reshape(n, 4)
            arr["iarg"] = np.asarray([ivs(a) for a in iargs], np.int32).reshape(n, 4)
            arr["farg"] = np.asarray(fargs, np.float64).reshape(n, 2)
            arr["wref"] = np.asarray([rv(w) for w in wrefs], np.int64)
        prog.ops = arr
        prog.task_ops = np.asarray(starts + [n], dtype=np.int64)
        prog.keys = [self.keys[t] for t in order]
        prog.kinds = [self.kinds[t] for t in order]
        prog.fold_chains = {u: [newidx[t] for t in ch] for u, ch in self.fold_chains.items()}
        prog.scratch_doubles = max(self.peak, 1)
        prog.task_scratch = np.asarray([self.tpeak[t] for t in order], dtype=np.int64)
        prog.scratch_ranks = max(self.rpeak, 1)
        prog.updates = self.updates
        prog.rw = [self.rw[t] for t in order]
        prog.peak_task = newidx.get(self.peak_task, -1)
        prog.groups = {newidx[r]: [newidx[t] for t in ms] for r, ms in self.groups.items()}
        prog.ws_size = max(self.wtop, 1)
        prog.ws_slots = max(self.wslots, 1)
        prog.w_info = dict(self.w_info)
        return prog


def _policy_fields(policy):
    mode = getattr(policy, "mode", "exact")
    if mode == "rank":
        return L.POLICY_RANK, int(policy.k), 0.0
    if mode == "accuracy":
        return L.POLICY_ACCURACY, 0, float(policy.eps)
    return L.POLICY_EXACT, 0, 0.0


def dataflow_edges(prog, tables):
    """Execution edges implied by the sequential program's data accesses.

    ``tables`` maps a matrix base id to its BlockTable (subtree reads are
    expanded to leaves).  RAW, WAW and WAR hazards on every leaf and every
    accumulator give edges from earlier to later tasks; executing any
    topological order of them reproduces the sequential program exactly.
    """
    leaves_of = {}

    def leaves(base, u):
        key = (base, u)
        v = leaves_of.get(key)
        if v is None:
            v = leaves_of[key] = [("m", base, x) for x in tables[base].leaves(u)]
        return v

    last_w = {}
    readers = {}
    edges = set()
    for t, (rds, wrs) in enumerate(prog.rw):
        robjs = []
        for o in rds:
            if o[0] == "m" and not tables[o[1]].leaf[o[2]]:
                robjs.extend(leaves(o[1], o[2]))
            else:
                robjs.append(o)
        for o in robjs:
            w = last_w.get(o)
            if w is not None and w != t:
                edges.add((w, t))
            readers.setdefault(o, set()).add(t)
        for o in wrs:
            w = last_w.get(o)
            if w is not None and w != t:
                edges.add((w, t))
            for r in readers.get(o, ()):
                if r != t:
                    edges.add((r, t))
            last_w[o] = t
            readers[o] = set()
    return edges


def plan_hlu(table: BlockTable, mode: str, policy, rank_cap=None, split_min=0):
    """Program of H-LU of a matrix over ``table``: A=0, L=1, U=2 (acc=3,
    workspace=5).  ``split_min`` > 0 splits H x H products with
    min(m, n) >= split_min into parallel micro-tasks."""
    lay = Layout(table, rank_cap)
    A, Lm, Um = PMat(0, lay), PMat(1, lay), PMat(2, lay)
    p = Planner(policy, rank_cap, split_min)
    if mode == "std":
        p.hlu(A, Lm, Um, 0)
    else:
        p.acc_table = table
        p.hlu_accu(A, Lm, Um, 0)
    prog = p.pack()
    prog.layout = lay
    return prog


def replicate(prog, nrep, base_sizes, slot_sizes):
    """Disjoint union of ``nrep`` copies of a program (batched instances).

    Copy b's matrix refs of base i are shifted by b * base_sizes[i] elements
    and its rank slots of base i by b * slot_sizes[i]; scratch refs (base
    15) are per-CTA and stay.  Used for batches of same-structure instances
    (config 4: 256 HODLR matrices share one block tree).
    """
    ops = prog.ops
    n = len(ops)
    out = shift_ops(np.tile(ops, nrep), np.repeat(np.arange(nrep, dtype=np.int64), n),
                    base_sizes, slot_sizes)
    task_ops = prog.task_ops
    nt = len(task_ops) - 1
    t_all = (task_ops[None, :-1] + (np.arange(nrep)[:, None] * n)).ravel()
    new_task_ops = np.concatenate([t_all, [n * nrep]]).astype(np.int64)
    return out, new_task_ops, nt


def shift_ops(out, rep, base_sizes, slot_sizes):
    """Shift op records ``out`` (in place) to replica ``rep[i]`` of their
    storage: matrix refs of base b move by rep * base_sizes[b] elements, rank
    slots of base b by rep * slot_sizes[b]; scratch (base 15) stays."""
    rep = np.asarray(rep, dtype=np.int64)
    mask56 = (1 << 56) - 1
    for field in ("ref", "wref"):
        r = out[field]
        r2 = r.reshape(len(out), -1)
        base = (r2.astype(np.uint64) >> np.uint64(56)).astype(np.int64)
        off = r2 & mask56
        shift = np.zeros_like(off)
        for b, sz in base_sizes.items():
            sel = base == b
            shift[sel] = (rep[:, None] * int(sz) * np.ones_like(off))[sel]
        newv = (base << 56) | (off + shift)
        out[field] = newv.reshape(out[field].shape)
    s = out["slot"]
    d = out["dim"]
    for arr in (s, d):
        neg = arr < 0
        code = -arr - 1
        b = code >> 24
        idx = code & 0xFFFFFF
        add = np.zeros_like(arr)
        for bb, sz in slot_sizes.items():
            sel = neg & (b == bb)
            add[sel] = (rep[:, None] * int(sz) * np.ones_like(arr))[sel]
        newcode = (b << 24) | (idx + add)
        arr[neg] = (-(newcode + 1))[neg]
    return out


OPS = ("hmul", "htrsl", "htrsu", "htrsl_accu", "htrsu_accu", "leaf_update")


def plan_op(table: BlockTable, op: str, policy, rank_cap=None, alpha=1.0, split_min=0,
            uids=None):
    """Program of a standalone multiply / triangular solve over ``table``.

    hmul:  C += alpha A B          (arith.py:40-55)      A=0, B=1, C=2
    htrsl: L X = M, M consumed     (arith.py:97-117)     L=0, M=1, X=2
    htrsu: X U = M, M consumed     (arith.py:120-140)    U=0, M=1, X=2
    *_accu: the accumulator variants (accumulator.py:190-235), acc=3
    leaf_update: C[uc] += alpha A[ua] B[ub], C[uc] a leaf (hmatrix.py:451-460)
    """
    if op not in OPS:
        raise ValueError(op)
    lay = Layout(table, rank_cap)
    P0, P1, P2 = PMat(0, lay), PMat(1, lay), PMat(2, lay)
    p = Planner(policy, rank_cap, split_min)
    if op == "leaf_update":
        ua, ub, uc = (int(x) for x in uids)
        if not table.leaf[uc]:
            raise ValueError("leaf_update needs a leaf C")
        p.begin("leaf_update", ("leaf_update", (ua, ub, uc), alpha))
        p.scatter(P2, uc, p.product(alpha, P0, ua, P1, ub))
    elif op == "hmul":
        p.hmul(alpha, P0, 0, P1, 0, P2, 0)
    elif op == "htrsl":
        p.htrsl(P0, 0, P1, 0, P2)
    elif op == "htrsu":
        p.htrsu(P0, 0, P1, 0, P2)
    else:
        p.acc_table = table
        if op == "htrsl_accu":
            p.htrsl_accu(P0, 0, P1, 0, P2)
        else:
            p.htrsu_accu(P0, 0, P1, 0, P2)
    prog = p.pack()
    prog.layout = lay
    return prog


DENSE_OPS = ("apply", "apply_t", "solve_lower", "solve_upper_t", "solve_upper")


def _elementary(bounds_lo, bounds_hi, lo, hi):
    """Elementary intervals of [lo, hi) cut at every leaf boundary."""
    cuts = sorted({lo, hi} | {int(x) for x in bounds_lo} | {int(x) for x in bounds_hi})
    cuts = [c for c in cuts if lo <= c <= hi]
    return list(zip(cuts[:-1], cuts[1:]))


def plan_dense(table: BlockTable, op: str, u: int, cols: int, rank_cap=None, layout=None):
    """Program of an H x dense operation on block u (hmatrix.py:286-341).

    apply:         out = H[u] @ X            H=0, X=1 (n_u x cols), out=2 (m_u x cols)
    apply_t:       out = H[u]^T @ X          X=1 (m_u x cols), out=2 (n_u x cols)
    solve_lower:   Y := L[u]^{-1} Y          L=0 unit lower, Y=1 (m_u x cols) in place
    solve_upper_t: Y := U[u]^{-T} Y          U=0 upper, Y=1 in place
    solve_upper:   Y := U[u]^{-1} Y          U=0 upper, Y=1 in place (solve phase)

    apply / apply_t run one task per elementary row (column) interval of
    the leaves: each task owns its rows of the output and sums the
    contributions of the leaves crossing them in block pre-order (a leaf
    spanning several intervals is applied by row slices, a low-rank one
    recomputes its small V^T X per slice).  The solves are sequential
    along the diagonal: one task.
    """
    if op not in DENSE_OPS:
        raise ValueError(op)
    from .hmatrix import EXACT

    # the operand's own layout when given (rank-bounded arenas of
    # assemble_bounded / zeros(..., caps) differ from the rank_cap layout)
    lay = layout if layout is not None else Layout(table, rank_cap)
    H = PMat(0, lay)
    p = Planner(EXACT, rank_cap, 0)
    t = table
    m_u, n_u = int(t.m[u]), int(t.nc[u])
    cols = int(cols)
    if op in ("apply", "apply_t"):
        tr = op == "apply_t"
        leaves = list(t.leaves(u))
        if tr:
            lo0, hi0 = int(t.c0[u]), int(t.c1[u])
            ivs = _elementary([t.c0[v] for v in leaves], [t.c1[v] for v in leaves], lo0, hi0)
        else:
            lo0, hi0 = int(t.r0[u]), int(t.r1[u])
            ivs = _elementary([t.r0[v] for v in leaves], [t.r1[v] for v in leaves], lo0, hi0)
        X = Ref(1, 0, max(n_u if not tr else m_u, 1))
        O = Ref(2, 0, max(m_u if not tr else n_u, 1))
        # leaves crossing each elementary interval, in block pre-order (one
        # pass over the leaves: linear in the number of crossings)
        starts = np.asarray([a for a, _ in ivs], dtype=np.int64)
        crossing = [[] for _ in ivs]
        for v in leaves:
            vlo, vhi = (int(t.c0[v]), int(t.c1[v])) if tr else (int(t.r0[v]), int(t.r1[v]))
            i0 = int(np.searchsorted(starts, vlo, side="left"))
            i1 = int(np.searchsorted(starts, vhi, side="left"))
            for i in range(i0, i1):
                crossing[i].append(v)
        for (a, b), vs in zip(ivs, crossing):
            p.begin("dense_" + op, (op, u, a))
            rows = b - a
            out = O.at(a - lo0)
            p.zero(rows, cols, out)
            for v in vs:
                vlo, vhi = (int(t.c0[v]), int(t.c1[v])) if tr else (int(t.r0[v]), int(t.r1[v]))
                off = a - vlo  # slice of the leaf's rows (apply) / columns (apply_t)
                if not tr:
                    c0, nv = int(t.c0[v] - t.c0[u]), int(t.nc[v])
                    if t.adm[v]:
                        q = H.lr(v)
                        mark = p.top
                        T = p.sref(max(q.kmax, 1), cols)
                        p.gemm(q.k, cols, nv, 1.0, q.V, True, X.at(c0), False, T, False)
                        p.gemm(rows, cols, q.k, 1.0, q.U.at(off), False, T, False, out, True)
                        p.top = mark
                    else:
                        p.gemm(rows, cols, nv, 1.0, H.dense(v).at(off), False, X.at(c0), False, out,
                               True)
                else:
                    r0, mv = int(t.r0[v] - t.r0[u]), int(t.m[v])
                    if t.adm[v]:
                        q = H.lr(v)
                        mark = p.top
                        T = p.sref(max(q.kmax, 1), cols)
                        p.gemm(q.k, cols, mv, 1.0, q.U, True, X.at(r0), False, T, False)
                        p.gemm(rows, cols, q.k, 1.0, q.V.at(off), False, T, False, out, True)
                        p.top = mark
                    else:
                        p.gemm(rows, cols, mv, 1.0, H.dense(v).at(0, off), True, X.at(r0), False,
                               out, True)
    else:
        if m_u != n_u:
            raise ValueError("triangular solve on a non-square block")
        Y = Ref(1, 0, max(m_u, 1))
        p.begin("dense_" + op, (op, u))
        if op == "solve_lower":
            p.solve_lower(H, u, Y, cols, cols)
        elif op == "solve_upper":
            p.solve_upper(H, u, Y, cols, cols)
        else:
            p.solve_upper_t(H, u, Y, cols, cols)
    prog = p.pack()
    prog.layout = lay
    return prog


def fuse_applies(prog):
    """Combined accumulator mode: fold every apply_upd task into the leaf
    factor/solve task that follows it in program order (the combined DAG has
    no apply nodes; its leaf tasks apply first)."""
    keys, kinds = prog.keys, prog.kinds
    n = len(keys)
    keep = []
    merged_into = {}
    i = 0
    while i < n:
        if kinds[i] == "apply_upd":
            j = i + 1
            if j >= n or kinds[j] not in ("leaf_factor", "leaf_solve_l", "leaf_solve_u") \
                    or keys[j][1][-1] != keys[i][1][0]:
                raise RuntimeError("apply_upd not followed by its leaf task")
            merged_into[i] = len(keep)
            merged_into[j] = len(keep)
            keep.append((i, j))
            i += 2
        else:
            merged_into[i] = len(keep)
            keep.append((i,))
            i += 1
    ops_parts, starts, nkeys, nkinds, nrw = [], [], [], [], []
    cur = 0
    for grp in keep:
        starts.append(cur)
        for t in grp:
            a, b = prog.task_ops[t], prog.task_ops[t + 1]
            ops_parts.append(prog.ops[a:b])
            cur += b - a
        last = grp[-1]
        nkeys.append(keys[last])
        nkinds.append(kinds[last])
        r, w = [], []
        for t in grp:
            r.extend(prog.rw[t][0])
            w.extend(prog.rw[t][1])
        nrw.append((r, w))
    prog.ops = np.concatenate(ops_parts) if ops_parts else prog.ops[:0]
    prog.task_ops = np.asarray(starts + [cur], dtype=np.int64)
    prog.keys, prog.kinds, prog.rw = nkeys, nkinds, nrw
    # each merged task reuses the scratch from offset 0: its need is the max
    prog.task_scratch = np.asarray([max(int(prog.task_scratch[t]) for t in grp) for grp in keep],
                                   dtype=np.int64)
    prog.fold_chains = {u: [merged_into[t] for t in ch] for u, ch in prog.fold_chains.items()}
    prog.groups = {merged_into[r]: [merged_into[t] for t in ms] for r, ms in prog.groups.items()}
    prog.peak_task = merged_into.get(prog.peak_task, -1)
    return prog
