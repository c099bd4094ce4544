"""Native H-LU lowering and execution graph (csrc/hmx_lower.cpp, include/hmx_lower.h).

``lower_hlu`` is the production planner of ExecPlan: the same op program as
planner.plan_hlu (the Python statement, kept as the specification and for
the accu-combined DAG mode; tests/test_lower_cpu.py compares the two op for
op), produced in C++ so that config 5 (3.5M tasks) plans in seconds.
``NativeProgram.graph`` builds the execution graph against the reference
DAG built by the native refinement builder (hmx_dag.cpp): std = the DAG's
edges, accu = the data-flow edges of hlu_accu (engine.ExecPlan docstring).
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib
from .planner import Layout, _policy_fields

KIND_NAMES = ("hlu", "htrsl", "htrsu", "hmul", "add_upd", "shift_upd", "apply_upd", "leaf_factor",
              "leaf_solve_l", "leaf_solve_u", "leaf_update", "micro")
_L = None


def _native():
    global _L
    if _L is None:
        from .taskgraph import _native as dag_native

        L = dag_native()
        vp, i32, i64, f64 = C.c_void_p, C.c_int32, C.c_int64, C.c_double
        L.hmx_lower_hlu.argtypes = [i32, vp, vp, vp, vp, vp, vp, vp, i32, i32, i32, f64, i64, i64, vp,
                                    i64, C.POINTER(vp)]
        L.hmx_lower_hlu.restype = C.c_int
        L.hmx_prog_count.argtypes = [vp, i32]
        L.hmx_prog_count.restype = i64
        L.hmx_prog_export.argtypes = [vp] * 11
        L.hmx_prog_export.restype = C.c_int
        L.hmx_prog_graph.argtypes = [vp, i32, vp, vp, vp, vp, vp, vp, vp, i32, vp]
        L.hmx_prog_graph.restype = C.c_int
        L.hmx_prog_graph_export.argtypes = [vp, vp, vp]
        L.hmx_prog_graph_export.restype = C.c_int
        L.hmx_prog_drop_access.argtypes = [vp]
        L.hmx_prog_drop_access.restype = None
        L.hmx_prog_free.argtypes = [vp]
        L.hmx_prog_free.restype = None
        _L = L
    return _L


def _table_arrays(t):
    arr = [np.ascontiguousarray(x, dtype=np.int64) for x in (t.r0, t.r1, t.c0, t.c1)]
    leaf = np.ascontiguousarray(t.leaf, dtype=np.int8)
    adm = np.ascontiguousarray(t.adm, dtype=np.int8)
    kids = np.ascontiguousarray(np.where(t.kids < 0, -1, t.kids), dtype=np.int32).reshape(-1, 4)
    return arr, leaf, adm, kids


class NativeProgram:
    """Program of one H-LU (the fields engine.ExecPlan uses of
    planner.Program): ops, task_ops, kinds / keys, task_scratch,
    scratch_doubles / scratch_ranks, updates, acc_size, ws_size / ws_slots,
    layout."""

    def __init__(self, table, mode, policy, rank_cap=None, split_min=0, caps=None, acc_budget=0):
        L = _native()
        self.table, self.mode = table, mode
        pm, kfix, eps = _policy_fields(policy)
        self._arr = _table_arrays(table)
        (r0, r1, c0, c1), leaf, adm, kids = self._arr
        capa = None
        if caps is not None:
            capa = np.ascontiguousarray(caps, dtype=np.int32)
        h = C.c_void_p()
        rc = L.hmx_lower_hlu(table.n, r0.ctypes.data, r1.ctypes.data, c0.ctypes.data, c1.ctypes.data,
                             leaf.ctypes.data, adm.ctypes.data, kids.ctypes.data,
                             0 if mode == "std" else 1, pm, kfix, eps,
                             int(rank_cap) if rank_cap else 0, int(split_min),
                             capa.ctypes.data if capa is not None else None, int(acc_budget),
                             C.byref(h))
        if rc == 2:
            raise ValueError("structural error in H-LU lowering (low-rank diagonal block or "
                             "non-conformal operands)")
        if rc:
            raise RuntimeError(f"hmx_lower_hlu failed ({rc})")
        self._h = h
        cnt = lambda w: int(L.hmx_prog_count(h, w))  # noqa: E731
        nt, nops, nb = cnt(0), cnt(1), table.n
        self.ops = np.zeros(nops, dtype=_lib.OP_DTYPE)
        self.task_ops = np.zeros(nt + 1, dtype=np.int64)
        self.kind_code = np.zeros(nt, dtype=np.int32)
        self.uids = np.zeros((nt, 3), dtype=np.int32)
        self.alpha = np.zeros(nt, dtype=np.float64)
        self.task_scratch = np.zeros(nt, dtype=np.int64)
        d_off, u_off, v_off, cap = (np.zeros(nb, dtype=np.int64) for _ in range(4))
        L.hmx_prog_export(h, self.ops.ctypes.data, self.task_ops.ctypes.data,
                          self.kind_code.ctypes.data, self.uids.ctypes.data, self.alpha.ctypes.data,
                          self.task_scratch.ctypes.data, d_off.ctypes.data, u_off.ctypes.data,
                          v_off.ctypes.data, cap.ctypes.data)
        self.layout = Layout.from_arrays(table, rank_cap, d_off, u_off, v_off, cap, cnt(2))
        self.acc_size, self.ws_size, self.ws_slots = cnt(3), cnt(4), cnt(5)
        self.scratch_doubles, self.scratch_ranks, self.updates = cnt(6), cnt(7), cnt(8)
        self.n_tasks = nt
        self._keys = None

    @property
    def kinds(self):
        return [KIND_NAMES[k] for k in self.kind_code.tolist()]

    @property
    def keys(self):
        """Task keys in the reference DAG's format (kind, uids, alpha); micro
        tasks: ("micro", (ua, ub), alpha)."""
        if self._keys is None:
            ks = []
            for k, u, a in zip(self.kind_code.tolist(), self.uids.tolist(), self.alpha.tolist()):
                ks.append((KIND_NAMES[k], tuple(x for x in u if x >= 0), a))
            self._keys = ks
        return self._keys

    def graph(self, dag_handle, mode):
        """Execution graph (succ_ptr int32, succ_idx int32) against the
        reference DAG ``dag_handle`` (hmx_dag*) of the same block table."""
        L = _native()
        (r0, r1, c0, c1), leaf, adm, kids = self._arr
        rc = L.hmx_prog_graph(self._h, self.table.n, r0.ctypes.data, r1.ctypes.data, c0.ctypes.data,
                              c1.ctypes.data, leaf.ctypes.data, adm.ctypes.data, kids.ctypes.data,
                              0 if mode == "std" else 1, dag_handle)
        if rc == 5:
            raise RuntimeError("planned tasks and the reference DAG's nodes differ")
        if rc == 6:
            raise RuntimeError("execution graph contradicts program order")
        if rc:
            raise RuntimeError(f"hmx_prog_graph failed ({rc})")
        ne = int(L.hmx_prog_count(self._h, 9))
        ptr = np.zeros(self.n_tasks + 1, dtype=np.int64)
        idx = np.zeros(max(ne, 1), dtype=np.int32)
        L.hmx_prog_graph_export(self._h, ptr.ctypes.data, idx.ctypes.data)
        self.n_dag_edges = int(L.hmx_prog_count(self._h, 10))
        L.hmx_prog_drop_access(self._h)
        if ptr[-1] >= 2 ** 31:
            raise RuntimeError("execution graph exceeds int32 CSR")
        return ptr.astype(np.int32), idx[:ne]

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and _L is not None:
            _L.hmx_prog_free(h)
            self._h = None
