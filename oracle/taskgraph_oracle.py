"""Pure-Python restatement of the reference task-graph builder.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py): the product package
builds DAGs with the native C++ builder (paper_1911_07531_b200/csrc/
hmx_dag.cpp, bound by paper_1911_07531_b200/taskgraph.py).  This module
restates the reference's refinement algorithm (hmatdag/taskgraph.py:66-665,
Alg. 10-15 of arXiv 1911.07531) over a flat BlockTable so that the tests can
cross-check the native builder at every path cap / root op, next to the
sha256 pins of the reference's own graphs (tests/golden/*.json).

  dep / precedes            taskgraph.py:66-69, 119-129
  task factories            taskgraph.py:137-196
  refinable / refine        taskgraph.py:208-312 (+ local edges 222-230)
  refine_sub/loc_deps       taskgraph.py:315-340
  sparsification            taskgraph.py:348-432
  TaskGraph                 taskgraph.py:444-479
  check_acyclic / closure   taskgraph.py:482-523
  compute_dag               taskgraph.py:530-590
  _accu_tree / build_hlu_dag taskgraph.py:616-665
"""

from __future__ import annotations

import numpy as np

from paper_1911_07531_b200.taskgraph import (ACC_BASE, ADD_UPD, APPLY_UPD, COMBINED, FACTOR_KINDS,
                                             HLU, HMUL, HTRSL, HTRSU, LEAF_FACTOR, LEAF_SOLVE_L,
                                             LEAF_SOLVE_U, LEAF_UPDATE, MERGED, MID_A, MID_L,
                                             MID_U, MODES, SHIFT_UPD, SOLVE_KINDS, STD, CycleError,
                                             asap_levels)
from paper_1911_07531_b200.trees import Block, BlockTable

class Task:
    """Arithmetic task: kind, matrix ids, block uids, alpha, deps, edges."""

    __slots__ = ("kind", "mids", "uids", "alpha", "ins", "outs", "succ", "subs", "seq",
                 "blocks_ref")

    def __init__(self, kind, mids, uids, ins, outs, seq, alpha=1.0):
        self.kind = kind
        self.mids = mids
        self.uids = uids
        self.alpha = alpha
        self.ins = ins
        self.outs = outs
        self.succ = set()
        self.subs = None
        self.seq = seq
        self.blocks_ref = None

    # reference-compatible views
    @property
    def in_deps(self):
        return self.ins

    @property
    def out_deps(self):
        return self.outs

    @property
    def blocks(self):
        return tuple(self.blocks_ref[u] for u in self.uids) if self.blocks_ref else self.uids

    def key(self):
        return (self.kind, self.mids, self.uids, self.alpha)

    def __repr__(self):
        return f"Task({self.kind}, seq={self.seq})"


def _hit(o, i):
    return o[0] == i[0] and o[1] < i[2] and i[1] < o[2] and o[3] < i[4] and i[3] < o[4]


def precedes(t1: Task, t2: Task) -> bool:
    """Some output of t1 intersects some input of t2 (taskgraph.py:119-129)."""
    if t1 is t2:
        return False
    for o in t1.outs:
        for i in t2.ins:
            if _hit(o, i):
                return True
    return False


class _Builder:
    """Refinement engine over a BlockTable for one construction mode."""

    def __init__(self, bt: BlockTable, mode: str, stop_size: int):
        self.bt = bt
        self.mode = mode
        self.stop = stop_size
        r0, r1, c0, c1 = bt.r0.tolist(), bt.r1.tolist(), bt.c0.tolist(), bt.c1.tolist()
        self.rng = list(zip(r0, r1, c0, c1))
        self.is_leaf = bt.leaf.tolist()
        self.parent = bt.parent.tolist()
        self.kids = bt.kids.tolist()
        self.size = [max(a, b) for a, b in zip((bt.r1 - bt.r0).tolist(), (bt.c1 - bt.c0).tolist())]

    def dep(self, mid, u):
        a, b, c, d = self.rng[u]
        return (mid, a, b, c, d)

    # task factories (taskgraph.py:137-196)
    def factor(self, u, seq):
        ins = [self.dep(MID_A, u)]
        if self.mode == COMBINED and self.parent[u] >= 0:
            ins.append(self.dep(ACC_BASE + self.parent[u], u))
        outs = [self.dep(MID_L, u), self.dep(MID_U, u)]
        return Task(LEAF_FACTOR if self.is_leaf[u] else HLU, (MID_A, MID_L, MID_U), (u,),
                    tuple(ins), tuple(outs), seq)

    def solve(self, lower, ut, um, mids, seq):
        m_t, m_m, m_x = mids
        ins = [self.dep(m_t, ut), self.dep(m_m, um)]
        if self.mode == COMBINED and self.parent[um] >= 0:
            ins.append(self.dep(ACC_BASE + self.parent[um], um))
        if lower:
            kind = LEAF_SOLVE_L if self.is_leaf[um] else HTRSL
        else:
            kind = LEAF_SOLVE_U if self.is_leaf[um] else HTRSU
        return Task(kind, mids, (ut, um), tuple(ins), (self.dep(m_x, um),), seq)

    def mul(self, alpha, ua, ub, uc, mids, seq):
        m_a, m_b, m_c = mids
        ins = (self.dep(m_a, ua), self.dep(m_b, ub), self.dep(m_c, uc))
        outs = [self.dep(m_c, uc)]
        if self.mode == STD:
            leafy = self.is_leaf[ua] or self.is_leaf[ub] or self.is_leaf[uc]
            kind = LEAF_UPDATE if leafy else HMUL
        else:
            kind = ADD_UPD
            if self.mode == COMBINED:
                outs.append(self.dep(ACC_BASE + uc, uc))
        return Task(kind, mids, (ua, ub, uc), ins, tuple(outs), seq, alpha=alpha)

    def shift(self, u, seq):
        ins = [self.dep(ACC_BASE + u, u)]
        if self.parent[u] >= 0:
            ins.insert(0, self.dep(ACC_BASE + self.parent[u], u))
        return Task(SHIFT_UPD, (MID_A,), (u,), tuple(ins), (self.dep(ACC_BASE + u, u),), seq)

    def apply(self, u, seq):
        ins = [self.dep(ACC_BASE + u, u)]
        if self.parent[u] >= 0:
            ins.insert(0, self.dep(ACC_BASE + self.parent[u], u))
        return Task(APPLY_UPD, (MID_A,), (u,), tuple(ins), (self.dep(MID_A, u),), seq)

    def above(self, u):
        return self.stop <= 0 or self.size[u] > self.stop

    def refinable(self, t):
        k = t.kind
        if k == HLU:
            return self.above(t.uids[0])
        if k == HTRSL or k == HTRSU:
            return self.above(t.uids[1])
        if k == HMUL:
            return self.above(t.uids[2])
        if k == ADD_UPD:
            a, b, c = t.uids
            return not (self.is_leaf[a] or self.is_leaf[b] or self.is_leaf[c]) and self.above(c)
        return False

    # refinement bodies (taskgraph.py:233-312)
    def refine(self, t):
        if t.subs is not None:
            return t.subs
        s = t.seq
        out = []
        k = t.kind
        comb = self.mode == COMBINED
        if k == HLU:
            (u,) = t.uids
            if self.is_leaf[u]:
                raise ValueError("cannot refine a leaf factorization")
            c00, c01, c10, c11 = self.kids[u]
            i = 0
            if comb:
                out.append(self.shift(u, s + (0,)))
                i = 1
            out.append(self.factor(c00, s + (i,)))
            out.append(self.solve(False, c00, c10, (MID_U, MID_A, MID_L), s + (i + 1,)))
            out.append(self.solve(True, c00, c01, (MID_L, MID_A, MID_U), s + (i + 2,)))
            out.append(self.mul(-1.0, c10, c01, c11, (MID_L, MID_U, MID_A), s + (i + 3,)))
            out.append(self.factor(c11, s + (i + 4,)))
        elif k == HTRSL or k == HTRSU:
            ut, um = t.uids
            if self.is_leaf[um]:
                raise ValueError("cannot refine a leaf solve")
            if self.is_leaf[ut]:
                raise ValueError("structured solve against a leaf diagonal")
            t00, t01, t10, t11 = self.kids[ut]
            m00, m01, m10, m11 = self.kids[um]
            mids = t.mids
            m_t, m_m, m_x = mids
            i = 0
            if comb:
                out.append(self.shift(um, s + (0,)))
                i = 1
            if k == HTRSL:
                out.append(self.solve(True, t00, m00, mids, s + (i,)))
                out.append(self.solve(True, t00, m01, mids, s + (i + 1,)))
                out.append(self.mul(-1.0, t10, m00, m10, (m_t, m_x, m_m), s + (i + 2,)))
                out.append(self.mul(-1.0, t10, m01, m11, (m_t, m_x, m_m), s + (i + 3,)))
                out.append(self.solve(True, t11, m10, mids, s + (i + 4,)))
                out.append(self.solve(True, t11, m11, mids, s + (i + 5,)))
            else:
                out.append(self.solve(False, t00, m00, mids, s + (i,)))
                out.append(self.solve(False, t00, m10, mids, s + (i + 1,)))
                out.append(self.mul(-1.0, m00, t01, m01, (m_x, m_t, m_m), s + (i + 2,)))
                out.append(self.mul(-1.0, m10, t01, m11, (m_x, m_t, m_m), s + (i + 3,)))
                out.append(self.solve(False, t11, m01, mids, s + (i + 4,)))
                out.append(self.solve(False, t11, m11, mids, s + (i + 5,)))
        elif k == HMUL or k == ADD_UPD:
            ua, ub, uc = t.uids
            if self.is_leaf[ua] or self.is_leaf[ub] or self.is_leaf[uc]:
                raise ValueError("cannot refine an update with leaf operands")
            ka, kb, kc = self.kids[ua], self.kids[ub], self.kids[uc]
            n = 0
            for i in range(2):
                for j in range(2):
                    for l in range(2):
                        out.append(self.mul(t.alpha, ka[2 * i + l], kb[2 * l + j], kc[2 * i + j],
                                            t.mids, s + (n,)))
                        n += 1
        else:
            raise ValueError(f"task kind {k} is not refinable")
        # automatic local edges, mutual matches directed by creation order
        for x in range(len(out)):
            a = out[x]
            for y in range(x + 1, len(out)):
                b = out[y]
                if precedes(a, b):
                    a.succ.add(b)
                elif precedes(b, a):
                    b.succ.add(a)
        t.subs = out
        return out


def _sub_deps(t):
    """Inherited edges of a refined task become edges between sub-tasks."""
    for g in t.succ:
        targets = g.subs if g.subs else (g,)
        for tp in t.subs:
            for s in targets:
                if tp is not s and precedes(tp, s):
                    tp.succ.add(s)


def _loc_deps(t):
    """Narrow edges of an unrefined task to refined successors' sub-tasks."""
    nxt = set()
    for g in t.succ:
        if g.subs:
            for s in g.subs:
                if precedes(t, s):
                    nxt.add(s)
        else:
            nxt.add(g)
    changed = nxt != t.succ
    t.succ = nxt
    return changed


def _nbhd(t):
    n = set(t.subs) if t.subs else {t}
    for s in t.succ:
        if s.subs:
            n.update(s.subs)
        else:
            n.add(s)
    return n


def _reach2(t, n, succ_of, cap):
    """Nodes of G|n reachable from t by a path of length in [2, cap]."""
    out = set()
    frontier = [s for s in succ_of(t) if s in n]
    seen = set(frontier)
    depth = 1
    while frontier and depth < cap:
        nxt = []
        for u in frontier:
            for v in succ_of(u):
                if v in n:
                    out.add(v)
                    if v not in seen:
                        seen.add(v)
                        nxt.append(v)
        frontier = nxt
        depth += 1
    return out


def _sparsify(targets, cap):
    """Alg. 13 over a batch against one snapshot (taskgraph.py:384-432)."""
    work = []
    members = set()
    for t in targets:
        n = _nbhd(t)
        prune = t.subs if t.subs else [t]
        work.append((n, prune))
        members |= n
        members.update(prune)
    snap = {u: tuple(u.succ) for u in members}
    succ_of = snap.__getitem__
    decisions = []
    for n, prune in work:
        dec = []
        for tp in prune:
            reach = _reach2(tp, n, succ_of, cap)
            dec.append((tp, [s for s in succ_of(tp) if s in reach]))
        decisions.append(dec)
    for dec in decisions:
        for tp, rem in dec:
            if rem:
                tp.succ.difference_update(rem)


class TaskGraph:
    """Final node and edge sets (taskgraph.py:444-479) plus device views."""

    def __init__(self, nodes, mode=STD, table=None):
        self.nodes = sorted(nodes, key=lambda t: t.seq)
        self.mode = mode
        self.table = table
        ids = {id(t) for t in self.nodes}
        for t in self.nodes:
            for s in t.succ:
                if id(s) not in ids:
                    raise CycleError("edge into a non-final task")
        if table is not None:
            for t in self.nodes:
                t.blocks_ref = table.blocks

    @property
    def n_nodes(self):
        return len(self.nodes)

    @property
    def n_edges(self):
        return sum(len(t.succ) for t in self.nodes)

    def stats(self):
        return self.n_nodes, self.n_edges

    def edges(self):
        for t in self.nodes:
            for s in t.succ:
                yield t, s

    def canonical_nodes(self):
        keys = sorted(t.key() for t in self.nodes)
        if len(set(keys)) != len(keys):
            raise CycleError("duplicate task keys in graph")
        return tuple(keys)

    def canonical_edges(self):
        return tuple(sorted((u.key(), v.key()) for u, v in self.edges()))

    # ---- device views ---------------------------------------------------
    def index(self):
        return {id(t): i for i, t in enumerate(self.nodes)}

    def csr(self):
        """(succ_ptr, succ_idx) int32 over node positions (seq order)."""
        idx = self.index()
        ptr = np.zeros(len(self.nodes) + 1, dtype=np.int64)
        lists = []
        for i, t in enumerate(self.nodes):
            s = sorted(idx[id(v)] for v in t.succ)
            lists.append(s)
            ptr[i + 1] = ptr[i] + len(s)
        flat = np.fromiter((v for s in lists for v in s), dtype=np.int32, count=int(ptr[-1]))
        return ptr.astype(np.int32), flat

    def levels(self, extra_edges=None):
        return asap_levels(len(self.nodes), *self.csr(), extra_edges)


def check_acyclic(g: TaskGraph) -> bool:
    indeg = {id(t): 0 for t in g.nodes}
    for _, v in g.edges():
        indeg[id(v)] += 1
    ready = [t for t in g.nodes if indeg[id(t)] == 0]
    seen = 0
    while ready:
        u = ready.pop()
        seen += 1
        for v in u.succ:
            indeg[id(v)] -= 1
            if indeg[id(v)] == 0:
                ready.append(v)
    return seen == len(g.nodes)


def transitive_closure(g: TaskGraph):
    """Reachability bitsets keyed by canonical task key."""
    order = sorted(g.nodes, key=lambda t: t.key())
    bit = {id(t): 1 << i for i, t in enumerate(order)}
    indeg = {id(t): 0 for t in g.nodes}
    for _, v in g.edges():
        indeg[id(v)] += 1
    ready = [t for t in g.nodes if indeg[id(t)] == 0]
    topo = []
    while ready:
        u = ready.pop()
        topo.append(u)
        for v in u.succ:
            indeg[id(v)] -= 1
            if indeg[id(v)] == 0:
                ready.append(v)
    if len(topo) != len(g.nodes):
        raise CycleError("closure of a cyclic graph")
    reach = {}
    for u in reversed(topo):
        r = 0
        for v in u.succ:
            r |= bit[id(v)] | reach[id(v)]
        reach[id(u)] = r
    return {t.key(): reach[id(t)] for t in g.nodes}


def _as_table(block_root):
    if isinstance(block_root, BlockTable):
        return block_root
    if isinstance(block_root, Block):
        return BlockTable(block_root)
    raise TypeError("expected a Block or BlockTable")


def compute_dag(root: Task, stop_size: int = 0, *, sparsify: bool = False, max_path_len: int = 2,
                mode: str = STD, table: BlockTable = None, _builder=None) -> TaskGraph:
    """Worklist refinement of ``root`` into a DAG (Alg. 12, taskgraph.py:530-590)."""
    b = _builder if _builder is not None else _Builder(table, mode, stop_size)
    retired = []
    current = [root]
    rounds = 0
    while current:
        rounds += 1
        if rounds > 10_000:
            raise CycleError("refinement failed to converge")
        for g in current:
            if g.subs is None and b.refinable(g):
                b.refine(g)
        nxt, starg = [], []
        for g in current:
            if g.subs:
                _sub_deps(g)
                nxt.extend(g.subs)
                if sparsify:
                    starg.append(g)
            elif _loc_deps(g):
                nxt.append(g)
            else:
                retired.append(g)
                if sparsify:
                    starg.append(g)
        if sparsify and starg:
            _sparsify(starg, max_path_len)
        current = nxt
    g = TaskGraph(retired, mode=mode, table=table)
    if not check_acyclic(g):
        raise CycleError("refinement produced a cyclic graph")
    return g


def par_compute_dag(root: Task, stop_size: int = 0, *, workers: int = 1, sparsify: bool = False,
                    max_path_len: int = 2, mode: str = STD, chunk_size: int = 256,
                    table: BlockTable = None, _builder=None) -> TaskGraph:
    """Same node/edge sets as :func:`compute_dag` for every worker count."""
    if workers < 1:
        raise ValueError("workers must be >= 1")
    return compute_dag(root, stop_size, sparsify=sparsify, max_path_len=max_path_len, mode=mode,
                       table=table, _builder=_builder)


def _accu_tree(b: _Builder):
    """Shift/apply tasks over the block tree, merged mode (taskgraph.py:616-633)."""
    by_uid = {}
    todo = [(0, (0,), None)]
    while todo:
        u, seq, par = todo.pop()
        terminal = b.is_leaf[u] or not b.above(u)
        t = b.apply(u, seq) if terminal else b.shift(u, seq)
        by_uid[u] = t
        if par is not None:
            par.succ.add(t)
        if not terminal:
            for k in reversed(range(4)):
                todo.append((b.kids[u][k], seq + (k,), t))
    return by_uid


def root_task(table: BlockTable, mode: str, op: str = "hlu"):
    """Top-level task of an H-LU (or standalone multiply / solve) DAG."""
    b = _Builder(table, mode, 0)
    seq = (1,) if mode == MERGED else (0,)
    if op == "hlu":
        return b.factor(0, seq), b
    if op == "hmul":
        return b.mul(1.0, 0, 0, 0, (MID_A, MID_L, MID_U), seq), b
    if op == "htrsl":
        return b.solve(True, 0, 0, (MID_L, MID_A, MID_U), seq), b
    if op == "htrsu":
        return b.solve(False, 0, 0, (MID_U, MID_A, MID_L), seq), b
    raise ValueError(op)


def build_hlu_dag(block_root, mode: str = STD, *, stop_size: int = 0, sparsify: bool = False,
                  max_path_len: int = 2, workers: int = 1, chunk_size: int = 256) -> TaskGraph:
    """Task graph of the H-LU of a matrix over ``block_root`` (taskgraph.py:636-665)."""
    if mode not in MODES:
        raise ValueError(f"unknown mode {mode!r}")
    if mode == COMBINED and sparsify:
        raise ValueError("edge sparsification is not valid in combined accumulator mode")
    table = _as_table(block_root)
    b = _Builder(table, mode, stop_size)
    root = b.factor(0, (1,) if mode == MERGED else (0,))
    arith = par_compute_dag(root, stop_size, workers=workers, sparsify=sparsify,
                            max_path_len=max_path_len, mode=mode, chunk_size=chunk_size,
                            table=table, _builder=b)
    if mode != MERGED:
        return arith
    acc = _accu_tree(b)
    for t in arith.nodes:
        if t.kind in FACTOR_KINDS:
            acc[t.uids[0]].succ.add(t)
        elif t.kind in SOLVE_KINDS:
            acc[t.uids[1]].succ.add(t)
        elif t.kind == ADD_UPD:
            t.succ.add(acc[t.uids[2]])
    g = TaskGraph(list(acc.values()) + arith.nodes, mode=MERGED, table=table)
    if not check_acyclic(g):
        raise CycleError("merged accumulator graph is cyclic")
    return g

