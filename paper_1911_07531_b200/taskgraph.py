"""Task-DAG construction by refinement (drop-in for hmatdag.taskgraph).

Public surface of the reference module (taskgraph.py:66-706): ``Task``,
``TaskGraph``, ``precedes``, ``compute_dag`` / ``par_compute_dag``,
``build_hlu_dag`` / ``build_accu_dag``, ``check_acyclic``,
``transitive_closure``, ``to_dot``.  Graphs are built by the native C++
refinement builder (csrc/hmx_dag.cpp, libhmxdag.so, include/hmx_dag.h):
same node and edge sets as the reference (sha256-pinned against graphs the
reference built, tests/golden; c5 by a multiset digest), with or without
edge sparsification (Alg. 13), for H-LU roots in all three modes and for
standalone multiply / triangular-solve roots.

The graph is held as arrays (kind, matrix ids, block uids, alpha per node
in creation-sequence order + successor CSR); ``Task`` objects are read-only
views made on demand.  ``workers`` / ``chunk_size`` are accepted for API
compatibility: the sequential build defines the result (taskgraph.py:593-608)
and the native build is ~25x faster than the reference's threads.

A pure-Python restatement of the reference builder lives in
oracle/taskgraph_oracle.py (test infrastructure, cross-checks this one).
"""

from __future__ import annotations

import numpy as np

from .trees import Block, BlockTable

MID_A, MID_L, MID_U = 0, 1, 2
ACC_BASE = 3

HLU = "hlu"
HTRSL = "htrsl"
HTRSU = "htrsu"
HMUL = "hmul"
ADD_UPD = "add_upd"
SHIFT_UPD = "shift_upd"
APPLY_UPD = "apply_upd"
LEAF_FACTOR = "leaf_factor"
LEAF_SOLVE_L = "leaf_solve_l"
LEAF_SOLVE_U = "leaf_solve_u"
LEAF_UPDATE = "leaf_update"

FACTOR_KINDS = frozenset({HLU, LEAF_FACTOR})
SOLVE_L_KINDS = frozenset({HTRSL, LEAF_SOLVE_L})
SOLVE_U_KINDS = frozenset({HTRSU, LEAF_SOLVE_U})
SOLVE_KINDS = SOLVE_L_KINDS | SOLVE_U_KINDS
UPDATE_KINDS = frozenset({HMUL, LEAF_UPDATE, ADD_UPD})
ACC_KINDS = frozenset({SHIFT_UPD, APPLY_UPD})

STD = "std"
COMBINED = "accu-combined"
MERGED = "accu-merged"
MODES = (STD, COMBINED, MERGED)


class CycleError(RuntimeError):
    pass


def _dep(table, mid, u):
    return (mid, int(table.r0[u]), int(table.r1[u]), int(table.c0[u]), int(table.c1[u]))


class Task:
    """Read-only node of a TaskGraph: kind, matrix ids, block uids, alpha;
    data dependencies (matrix id, row range, col range) are derived from the
    block table by the reference's factory rules (taskgraph.py:137-196)."""

    __slots__ = ("kind", "mids", "uids", "alpha", "_g", "_i")

    def __init__(self, g, i, kind, mids, uids, alpha):
        self.kind, self.mids, self.uids, self.alpha, self._g, self._i = kind, mids, uids, alpha, g, i

    def key(self):
        return (self.kind, self.mids, self.uids, self.alpha)

    @property
    def succ(self):
        g = self._g
        return [g.nodes[j] for j in g.succ_idx[g.succ_ptr[self._i]:g.succ_ptr[self._i + 1]]]

    @property
    def blocks(self):
        t = self._g.table
        return tuple(t.blocks[u] for u in self.uids) if t is not None and t.blocks else self.uids

    @property
    def in_deps(self):
        t, k, mode = self._g.table, self.kind, self._g.mode
        if k in FACTOR_KINDS:
            (u,) = self.uids
            out = [_dep(t, MID_A, u)]
            if mode == COMBINED and t.parent[u] >= 0:
                out.append(_dep(t, ACC_BASE + int(t.parent[u]), u))
            return tuple(out)
        if k in SOLVE_KINDS:
            ut, um = self.uids
            out = [_dep(t, self.mids[0], ut), _dep(t, self.mids[1], um)]
            if mode == COMBINED and t.parent[um] >= 0:
                out.append(_dep(t, ACC_BASE + int(t.parent[um]), um))
            return tuple(out)
        if k in UPDATE_KINDS:
            return tuple(_dep(t, m, u) for m, u in zip(self.mids, self.uids))
        (u,) = self.uids  # shift / apply
        out = [_dep(t, ACC_BASE + u, u)]
        if t.parent[u] >= 0:
            out.insert(0, _dep(t, ACC_BASE + int(t.parent[u]), u))
        return tuple(out)

    @property
    def out_deps(self):
        t, k, mode = self._g.table, self.kind, self._g.mode
        if k in FACTOR_KINDS:
            (u,) = self.uids
            return (_dep(t, MID_L, u), _dep(t, MID_U, u))
        if k in SOLVE_KINDS:
            return (_dep(t, self.mids[2], self.uids[1]),)
        if k in UPDATE_KINDS:
            uc = self.uids[2]
            out = [_dep(t, self.mids[2], uc)]
            if mode == COMBINED:
                out.append(_dep(t, ACC_BASE + uc, uc))
            return tuple(out)
        (u,) = self.uids
        return (_dep(t, ACC_BASE + u, u),) if k == SHIFT_UPD else (_dep(t, MID_A, u),)

    def __repr__(self):
        return f"Task({self.kind}, {self.uids})"


def _overlap(o, i):
    return o[0] == i[0] and o[1] < i[2] and i[1] < o[2] and o[3] < i[4] and i[3] < o[4]


def precedes(t1: Task, t2: Task) -> bool:
    """True when an output range of t1 meets an input range of t2
    (taskgraph.py:119-129)."""
    if t1 is t2:
        return False
    ins = t2.in_deps
    return any(_overlap(o, i) for o in t1.out_deps for i in ins)


class TaskGraph:
    """Final node and edge sets of a refinement (taskgraph.py:444-479):
    node arrays in creation-sequence order (the order of the reference's
    ``TaskGraph.nodes``) and successor CSR over that order."""

    def __init__(self, kind, nm, mids, nu, uids, alpha, ptr, idx, mode, table):
        self.mode, self.table = mode, table
        self.kind_code = kind
        self.mids_arr, self.nm = mids, nm
        self.uids_arr, self.nu = uids, nu
        self.alpha_arr = alpha
        self.succ_ptr, self.succ_idx = ptr, idx
        self._nodes = None

    @property
    def nodes(self):
        if self._nodes is None:
            km, mids, uids, nm, nu, al = (self.kind_code.tolist(), self.mids_arr.tolist(),
                                          self.uids_arr.tolist(), self.nm.tolist(), self.nu.tolist(),
                                          self.alpha_arr.tolist())
            self._nodes = [Task(self, i, _KIND_NAMES[km[i]], tuple(mids[i][:nm[i]]),
                                tuple(uids[i][:nu[i]]), al[i]) for i in range(len(km))]
        return self._nodes

    @property
    def n_nodes(self):
        return int(len(self.kind_code))

    @property
    def n_edges(self):
        return int(len(self.succ_idx))

    def stats(self):
        return self.n_nodes, self.n_edges

    def edges(self):
        ptr, idx, nodes = self.succ_ptr, self.succ_idx, self.nodes
        for i in range(len(nodes)):
            for j in idx[ptr[i]:ptr[i + 1]]:
                yield nodes[i], nodes[j]

    def canonical_nodes(self):
        keys = sorted(t.key() for t in self.nodes)
        if any(a == b for a, b in zip(keys, keys[1:])):
            raise CycleError("duplicate task keys in graph")
        return tuple(keys)

    def canonical_edges(self):
        return tuple(sorted((u.key(), v.key()) for u, v in self.edges()))

    def index(self):
        return {id(t): i for i, t in enumerate(self.nodes)}

    def csr(self):
        """(succ_ptr, succ_idx) int32 over node positions (seq order)."""
        return self.succ_ptr.astype(np.int32), self.succ_idx.astype(np.int32)

    def levels(self, extra_edges=None):
        return asap_levels(self.n_nodes, *self.csr(), extra_edges)


# kept for callers of round 1
NativeTask, NativeTaskGraph = Task, TaskGraph


def check_acyclic(g: TaskGraph) -> bool:
    """Kahn's algorithm over the CSR (native hmx_dag_levels)."""
    try:
        g.levels()
    except CycleError:
        return False
    return True


def transitive_closure(g: TaskGraph):
    """Reachability sets as bit masks keyed by canonical task key (bit i =
    i-th node in sorted key order), accumulated in reverse topological
    order of the ASAP levels."""
    n = g.n_nodes
    nodes = g.nodes
    keys = [t.key() for t in nodes]
    rank = {k: i for i, k in enumerate(sorted(keys))}
    bit = [1 << rank[k] for k in keys]
    lv = g.levels()
    ptr, idx = g.succ_ptr, g.succ_idx
    reach = [0] * n
    for u in np.argsort(-lv.astype(np.int64), kind="stable").tolist():
        r = 0
        for v in idx[ptr[u]:ptr[u + 1]].tolist():
            r |= bit[v] | reach[v]
        reach[u] = r
    return {keys[i]: reach[i] for i in range(n)}


def stats(g: TaskGraph):
    return g.stats()


def _as_table(block_root):
    if isinstance(block_root, BlockTable):
        return block_root
    if isinstance(block_root, Block):
        return BlockTable(block_root)
    raise TypeError("expected a Block or BlockTable")


class RootTask:
    """Root of a refinement (taskgraph.py:146-180 factories on the root
    block): ``op`` in hlu / hmul / htrsl / htrsu."""

    def __init__(self, table, mode=STD, op="hlu"):
        if op not in _OP_CODE:
            raise ValueError(op)
        self.table, self.mode, self.op = _as_table(table), mode, op


def root_task(table, mode: str = STD, op: str = "hlu") -> RootTask:
    return RootTask(table, mode, op)


def compute_dag(root: RootTask, stop_size: int = 0, *, sparsify: bool = False,
                max_path_len: int = 2) -> TaskGraph:
    """Refine ``root`` to its final DAG (Alg. 12, taskgraph.py:530-590)."""
    return build_dag_native(root.table, root.mode, stop_size=stop_size, op=root.op,
                            sparsify=sparsify, max_path_len=max_path_len)


def par_compute_dag(root: RootTask, stop_size: int = 0, *, workers: int = 1, sparsify: bool = False,
                    max_path_len: int = 2, chunk_size: int = 256) -> TaskGraph:
    """Same node/edge sets as :func:`compute_dag` for every worker count
    (taskgraph.py:593-608)."""
    if workers < 1:
        raise ValueError("workers must be >= 1")
    return compute_dag(root, stop_size, sparsify=sparsify, max_path_len=max_path_len)


def build_hlu_dag(block_root, mode: str = STD, *, stop_size: int = 0, sparsify: bool = False,
                  max_path_len: int = 2, workers: int = 1, chunk_size: int = 256) -> TaskGraph:
    """Task graph of the H-LU of a matrix over ``block_root`` (taskgraph.py:636-665)."""
    if workers < 1:
        raise ValueError("workers must be >= 1")
    return build_dag_native(block_root, mode, stop_size=stop_size, sparsify=sparsify,
                            max_path_len=max_path_len)


def build_accu_dag(block_root, mode: str = "combined", *, stop_size: int = 0,
                   sparsify: bool = False, max_path_len: int = 2, workers: int = 1) -> TaskGraph:
    if mode not in ("combined", "merged"):
        raise ValueError(f"unknown accumulator mode {mode!r}")
    return build_hlu_dag(block_root, COMBINED if mode == "combined" else MERGED,
                         stop_size=stop_size, sparsify=sparsify, max_path_len=max_path_len,
                         workers=workers)


_FILL = {"factor": "tomato", "solve": "lightblue", "update": "lightgreen", "acc": "khaki"}


def _fill(kind):
    if kind in FACTOR_KINDS:
        return _FILL["factor"]
    if kind in SOLVE_KINDS:
        return _FILL["solve"]
    if kind in UPDATE_KINDS:
        return _FILL["update"]
    return _FILL["acc"]


def to_dot(g: TaskGraph) -> str:
    """Graphviz text: a filled box per task (kind and the row x column
    range of its last block), one arrow per edge."""
    bt = g.table
    out = ["digraph taskgraph {", "  node [shape=box, style=filled];"]
    for i, t in enumerate(g.nodes):
        u = t.uids[-1]
        where = (f"[{bt.r0[u]},{bt.r1[u]})x[{bt.c0[u]},{bt.c1[u]})" if bt is not None else str(u))
        out.append(f'  n{i} [label="{t.kind}\\n{where}", fillcolor={_fill(t.kind)}];')
    ptr, idx = g.succ_ptr, g.succ_idx
    for i in range(g.n_nodes):
        for j in idx[ptr[i]:ptr[i + 1]].tolist():
            out.append(f"  n{i} -> n{j};")
    out.append("}")
    return "\n".join(out) + "\n"

def asap_levels(n, ptr, idx, extra_edges=None):
    """ASAP wavefront index of every node (Kahn's algorithm, native
    hmx_dag_levels)."""
    import ctypes as C

    ptr = np.asarray(ptr, dtype=np.int64)
    idx = np.asarray(idx, dtype=np.int32)
    if extra_edges is not None and len(extra_edges):
        ex = np.asarray(list(extra_edges), dtype=np.int64).reshape(-1, 2)
        src = np.concatenate([np.repeat(np.arange(n, dtype=np.int64), np.diff(ptr)), ex[:, 0]])
        dst = np.concatenate([idx.astype(np.int64), ex[:, 1]])
        o = np.argsort(src, kind="stable")
        idx = dst[o].astype(np.int32)
        ptr = np.concatenate([[0], np.cumsum(np.bincount(src, minlength=n))]).astype(np.int64)
    ptr = np.ascontiguousarray(ptr)
    idx = np.ascontiguousarray(idx) if len(idx) else np.zeros(1, np.int32)
    level = np.empty(max(n, 1), dtype=np.int32)
    rc = _native().hmx_dag_levels(int(n), ptr.ctypes.data, idx.ctypes.data, level.ctypes.data)
    if rc == 3:
        raise CycleError("cyclic execution graph")
    if rc:
        raise ValueError(f"hmx_dag_levels failed ({rc})")
    return level[:n]


def asap_levels_py(n, ptr, idx, extra_edges=None):
    """Pure-Python restatement of asap_levels (test cross-check)."""
    succ = [idx[ptr[i]:ptr[i + 1]].tolist() for i in range(n)]
    if extra_edges is not None:
        for a, b in extra_edges:
            succ[a].append(b)
    indeg = [0] * n
    for s in succ:
        for v in s:
            indeg[v] += 1
    level = [0] * n
    ready = [i for i in range(n) if indeg[i] == 0]
    seen = 0
    while ready:
        nxt = []
        for u in ready:
            seen += 1
            for v in succ[u]:
                level[v] = max(level[v], level[u] + 1)
                indeg[v] -= 1
                if indeg[v] == 0:
                    nxt.append(v)
        ready = nxt
    if seen != n:
        raise CycleError("cyclic execution graph")
    return np.asarray(level, dtype=np.int32)



def key_line(k) -> str:
    """Canonical text of a task key (shared with tests/golden fixtures)."""
    kind, mids, uids, alpha = k
    return f"{kind}|{','.join(map(str, mids))}|{','.join(map(str, uids))}|{alpha!r}"


def multiset_digest(node_lines, src, dst):
    """Order-independent digest of a DAG too large to sort as text (config 5:
    3.2M nodes, 207M edges).  h = blake2b-64 of each canonical node line;
    nodes -> (sum h, sum h^2) mod 2^64; edges -> the same two sums over
    e = h_u * 0x9E3779B97F4A7C15 + (h_v ^ (h_v >> 29)) * 0xBF58476D1CE4E5B9.
    Same definition as tests/golden/make_golden.py (which ran the reference)."""
    import hashlib

    h = np.fromiter((int.from_bytes(hashlib.blake2b(x.encode(), digest_size=8).digest(), "little")
                     for x in node_lines), dtype=np.uint64, count=len(node_lines))
    with np.errstate(over="ignore"):
        out = [int(h.sum(dtype=np.uint64)), int((h * h).sum(dtype=np.uint64))]
        es, ess = np.uint64(0), np.uint64(0)
        for a in range(0, len(src), 1 << 24):
            hu, hv = h[src[a:a + (1 << 24)]], h[dst[a:a + (1 << 24)]]
            e = hu * np.uint64(0x9E3779B97F4A7C15) + (hv ^ (hv >> np.uint64(29))) * np.uint64(0xBF58476D1CE4E5B9)
            es += e.sum(dtype=np.uint64)
            ess += (e * e).sum(dtype=np.uint64)
        out += [int(es), int(ess)]
    return [f"{x:016x}" for x in out]


def dag_digest(g: TaskGraph):
    """{nodes, edges, digest} of a graph (multiset_digest over its CSR)."""
    ptr, idx = g.csr()
    src = np.repeat(np.arange(g.n_nodes, dtype=np.int64), np.diff(ptr.astype(np.int64)))
    lines = [key_line(t.key()) for t in g.nodes]
    return {"nodes": g.n_nodes, "edges": int(len(idx)),
            "digest": multiset_digest(lines, src, idx.astype(np.int64))}


def canonical_hashes(g: TaskGraph):
    """sha256 of sorted canonical node and edge lines (fixture format)."""
    import hashlib

    nodes = sorted(key_line(t.key()) for t in g.nodes)
    edges = sorted(f"{key_line(u.key())}>{key_line(v.key())}" for u, v in g.edges())
    h = lambda s: hashlib.sha256("\n".join(s).encode()).hexdigest()  # noqa: E731
    return h(nodes), h(edges)



# ---------------------------------------------------------------------------
# native builder (csrc/hmx_dag.cpp, libhmxdag.so): same node and edge sets
# ---------------------------------------------------------------------------
_KIND_NAMES = (HLU, HTRSL, HTRSU, HMUL, ADD_UPD, SHIFT_UPD, APPLY_UPD, LEAF_FACTOR, LEAF_SOLVE_L,
               LEAF_SOLVE_U, LEAF_UPDATE)
_MODE_CODE = {STD: 0, COMBINED: 1, MERGED: 2}
_OP_CODE = {"hlu": 0, "hmul": 1, "htrsl": 2, "htrsu": 3}
_dag_lib = None


def _native():
    global _dag_lib
    if _dag_lib is None:
        import ctypes as C

        from ._build import DAG_LIB

        L = C.CDLL(DAG_LIB)
        vp, i32, i64 = C.c_void_p, C.c_int32, C.c_int64
        L.hmx_dag_build.argtypes = [i32, vp, vp, vp, vp, vp, vp, vp, i32, i64, i32, C.POINTER(vp)]
        L.hmx_dag_build.restype = C.c_int
        L.hmx_dag_build_ex.argtypes = [i32, vp, vp, vp, vp, vp, vp, vp, i32, i64, i32, i32, i32,
                                       C.POINTER(vp)]
        L.hmx_dag_build_ex.restype = C.c_int
        L.hmx_dag_nodes.argtypes = [vp]
        L.hmx_dag_nodes.restype = i64
        L.hmx_dag_edges.argtypes = [vp]
        L.hmx_dag_edges.restype = i64
        L.hmx_dag_export.argtypes = [vp] * 9
        L.hmx_dag_export.restype = C.c_int
        L.hmx_dag_free.argtypes = [vp]
        L.hmx_dag_free.restype = None
        L.hmx_dag_levels.argtypes = [i64, vp, vp, vp]
        L.hmx_dag_levels.restype = C.c_int
        _dag_lib = L
    return _dag_lib


class DagHandle:
    """Owned native DAG (hmx_dag*) for native consumers (lower.py); freed
    with the object."""

    def __init__(self, ptr):
        self.ptr = ptr

    def n_nodes(self):
        return int(_native().hmx_dag_nodes(self.ptr))

    def n_edges(self):
        return int(_native().hmx_dag_edges(self.ptr))

    def free(self):
        if self.ptr is not None:
            _native().hmx_dag_free(self.ptr)
            self.ptr = None

    def __del__(self):
        self.free()


def dag_handle(block_root, mode: str = STD, *, stop_size: int = 0, op: str = "hlu",
               sparsify: bool = False, max_path_len: int = 2) -> DagHandle:
    """The native build of build_dag_native, kept native (no export)."""
    import ctypes as C

    if mode not in MODES:
        raise ValueError(f"unknown mode {mode!r}")
    if mode == COMBINED and sparsify:
        raise ValueError("edge sparsification is not valid in combined accumulator mode")
    t = _as_table(block_root)
    L = _native()
    arr = [np.ascontiguousarray(x, dtype=np.int64) for x in (t.r0, t.r1, t.c0, t.c1)]
    leaf = np.ascontiguousarray(t.leaf, dtype=np.int8)
    parent = np.ascontiguousarray(t.parent, dtype=np.int32)
    kids = np.ascontiguousarray(np.where(t.kids < 0, -1, t.kids), dtype=np.int32).reshape(-1, 4)
    h = C.c_void_p()
    rc = L.hmx_dag_build_ex(t.n, *[a.ctypes.data for a in arr], leaf.ctypes.data, parent.ctypes.data,
                            kids.ctypes.data, _MODE_CODE[mode], int(stop_size), _OP_CODE[op],
                            int(bool(sparsify)), int(max_path_len), C.byref(h))
    if rc == 2:
        raise ValueError("structural error in refinement (leaf diagonal / operands)")
    if rc == 3:
        raise CycleError("refinement produced a cyclic graph")
    if rc:
        raise ValueError(f"hmx_dag_build failed ({rc})")
    return DagHandle(h)


def build_dag_native(block_root, mode: str = STD, *, stop_size: int = 0, op: str = "hlu",
                     sparsify: bool = False, max_path_len: int = 2):
    """Native (C++) refinement build; same node and edge sets as
    build_hlu_dag / compute_dag, with or without edge sparsification
    (taskgraph.py:384-432, applied per refinement round)."""
    import ctypes as C

    if mode not in MODES:
        raise ValueError(f"unknown mode {mode!r}")
    if mode == COMBINED and sparsify:
        raise ValueError("edge sparsification is not valid in combined accumulator mode")
    if max_path_len < 1:
        raise ValueError("max_path_len must be >= 1")
    t = _as_table(block_root)
    L = _native()
    arr = [np.ascontiguousarray(x, dtype=np.int64) for x in (t.r0, t.r1, t.c0, t.c1)]
    leaf = np.ascontiguousarray(t.leaf, dtype=np.int8)
    parent = np.ascontiguousarray(t.parent, dtype=np.int32)
    kids = np.ascontiguousarray(np.where(t.kids < 0, -1, t.kids), dtype=np.int32).reshape(-1, 4)
    h = C.c_void_p()
    rc = L.hmx_dag_build_ex(t.n, *[a.ctypes.data for a in arr], leaf.ctypes.data, parent.ctypes.data,
                            kids.ctypes.data, _MODE_CODE[mode], int(stop_size), _OP_CODE[op],
                            int(bool(sparsify)), int(max_path_len), C.byref(h))
    if rc == 2:
        raise ValueError("structural error in refinement (leaf diagonal / operands)")
    if rc == 3:
        raise CycleError("refinement produced a cyclic graph")
    if rc:
        raise ValueError(f"hmx_dag_build failed ({rc})")
    try:
        n, ne = L.hmx_dag_nodes(h), L.hmx_dag_edges(h)
        kind = np.empty(n, np.int32)
        nm = np.empty(n, np.int32)
        nu = np.empty(n, np.int32)
        mids = np.empty((n, 3), np.int32)
        uids = np.empty((n, 3), np.int32)
        alpha = np.empty(n, np.float64)
        ptr = np.empty(n + 1, np.int64)
        idx = np.empty(max(ne, 1), np.int32)
        L.hmx_dag_export(h, kind.ctypes.data, nm.ctypes.data, mids.ctypes.data, nu.ctypes.data,
                         uids.ctypes.data, alpha.ctypes.data, ptr.ctypes.data, idx.ctypes.data)
    finally:
        L.hmx_dag_free(h)
    return TaskGraph(kind, nm, mids, nu, uids, alpha, ptr, idx[:ne], mode, t)

