"""Standard H-arithmetic on the GPU (drop-in for hmatdag.arith, arith.py:1-140).

``hlu(A, L, U, policy)`` factors A = L U (unpivoted, L unit lower) by
executing the lowered task DAG of taskgraph.build_hlu_dag on the device;
A is consumed as workspace, L and U (from ``zeros``) receive the factors,
exactly like the reference.  The result is the one of the sequential
recursion ``arith.hlu`` (same tasks, same truncation sequence): std-mode
DAG execution is order independent.
"""

from __future__ import annotations

import numpy as np

from . import engine
from .hmatrix import HMatrix, TruncationPolicy, counters

PIVOT_CUTOFF = 1e-14


class SingularPivotError(RuntimeError):
    pass


class _PlanCache:
    """Small LRU of execution plans.  A plan owns GB-scale device buffers
    (per-CTA scratch, accumulator pool, workspace), so only the ``size``
    most recently used plans are kept; ``clear_plans()`` drops them all.
    Keys hold the block table itself (not its id), so a key can never be
    reused by another table."""

    def __init__(self, size):
        from collections import OrderedDict

        self.size = size
        self.d = OrderedDict()

    def get(self, key, make):
        p = self.d.get(key)
        if p is None:
            while len(self.d) >= self.size:
                self.d.popitem(last=False)
            p = make()
            self.d[key] = p
        self.d.move_to_end(key)
        return p

    def clear(self):
        self.d.clear()


PLAN_CACHE_SIZE = 2
_PLANS = _PlanCache(PLAN_CACHE_SIZE)


def get_plan(table, mode, policy, rank_cap, dag_mode=None, sparsify=False, max_ctas=0,
             split_min=engine.DEFAULT_SPLIT_MIN, nrep=1, ctas_per_sm=None, caps=None, acc_budget=0,
             scratch_budget=None):
    """Cached execution plan (planning and upload happen once per tree).
    caps / acc_budget / scratch_budget: rank-bounded arenas, accumulator
    storage reuse and scratch bounds of large problems (engine.ExecPlan)."""
    ck = None if caps is None else hash(np.ascontiguousarray(caps, dtype=np.int32).tobytes())
    key = (table, mode, repr(policy), rank_cap, dag_mode, sparsify, max_ctas, split_min, nrep,
           ctas_per_sm, ck, acc_budget, scratch_budget)
    return _PLANS.get(key, lambda: engine.ExecPlan(
        table, mode, policy, rank_cap, dag_mode=dag_mode, sparsify=sparsify, max_ctas=max_ctas,
        split_min=split_min, nrep=nrep, ctas_per_sm=ctas_per_sm, caps=caps, acc_budget=acc_budget,
        scratch_budget=scratch_budget))


def clear_plans():
    """Drop every cached plan (their device scratch is freed with them)."""
    _PLANS.clear()
    _OPS.clear()


def _check_operands(*ms):
    t = ms[0].table
    for M in ms:
        if not isinstance(M, HMatrix):
            raise TypeError("operands must be device HMatrix views")
        if M.table is not t:
            raise ValueError("non-conformal operands (different block trees)")
        if M.uid != ms[0].uid:
            raise ValueError("non-conformal operands (different blocks)")
    if ms[0].uid != 0:
        raise NotImplementedError("factorization of a sub-block view: factor the root")
    return t


def run_hlu(A, L, U, policy, mode, exec_mode=engine.EXEC_PERSISTENT, dag_mode=None,
            sparsify=False, stream=None, split_min=engine.DEFAULT_SPLIT_MIN, acc_budget=0,
            scratch_budget=None):
    t = _check_operands(A, L, U)
    rc = A.store.layout.rank_cap
    caps = getattr(A.store.layout, "caps", None)
    for M in (L, U):
        if M.store.layout.rank_cap != rc:
            raise ValueError("L/U storage rank_cap differs from A's")
        mc = getattr(M.store.layout, "caps", None)
        if (mc is None) != (caps is None) or (caps is not None and not np.array_equal(mc, caps)):
            raise ValueError("L/U storage capacities differ from A's")
    plan = get_plan(t, mode, policy, rc, dag_mode, sparsify, split_min=split_min, caps=caps,
                    acc_budget=acc_budget, scratch_budget=scratch_budget)
    plan.run(A.store, L.store, U.store, exec_mode, stream)
    c = plan.counters(stream)
    counters.add(c["truncations"], c["updates"])
    return plan


def hlu_batch(A, L, U, policy: TruncationPolicy, mode="std", exec_mode=engine.EXEC_PERSISTENT,
              stream=None, split_min=engine.DEFAULT_SPLIT_MIN, ctas_per_sm=None):
    """Factor every member of an HBatch (hmatrix.HBatch) in one launch;
    mode "std" (arith.hlu semantics) or "accu" (accumulator.hlu_accu).
    ctas_per_sm selects the executor variant (default: 2 for R > 1, see
    engine.ExecPlan); with 1 every member reproduces the bits of a single
    arith.hlu / hlu_accu run."""
    for M in (L, U):
        if M.nrep != A.nrep or M.table is not A.table:
            raise ValueError("batches differ in size or structure")
    rc = A.store.layout.rank_cap
    plan = get_plan(A.table, mode, policy, rc, split_min=split_min, nrep=A.nrep,
                    ctas_per_sm=ctas_per_sm)
    plan.run(A.store, L.store, U.store, exec_mode, stream)
    c = plan.counters(stream)
    counters.add(c["truncations"], c["updates"])
    return plan


def hlu(A: HMatrix, L: HMatrix, U: HMatrix, policy: TruncationPolicy, **kw):
    """Factor A = L U (arith.py:76-94); A is consumed as workspace."""
    return run_hlu(A, L, U, policy, "std", **kw)


def dense_lu(A: np.ndarray):
    """Unpivoted LU of one dense block on the device (arith.py:58-73)."""
    from . import kernels

    A = np.asarray(A, dtype=float)
    if A.ndim != 2 or A.shape[0] != A.shape[1]:
        raise ValueError("LU needs a square block")
    Ls, Us, info = kernels.getrf_nopiv([A])
    if info[0]:
        raise SingularPivotError("vanishing pivot")
    return Ls[0], Us[0]


_OPS = _PlanCache(4)


def _op_plan(table, op, policy, rank_cap, alpha=1.0):
    key = (table, op, repr(policy), rank_cap, float(alpha))
    return _OPS.get(key, lambda: engine.OpPlan(table, op, policy, rank_cap, alpha=alpha))


def _run_op(op, M0, M1, M2, policy, alpha=1.0, **kw):
    t = _check_operands(M0, M1, M2)
    rc = M0.store.layout.rank_cap
    if any(M.store.layout.rank_cap != rc for M in (M1, M2)):
        raise ValueError("operand storage rank_cap differs")
    if M2.store is M0.store or M2.store is M1.store:
        raise ValueError("the output may not alias an input")
    plan = _op_plan(t, op, policy, rc, alpha)
    plan.run(M0.store, M1.store, M2.store, **kw)
    c = plan.counters()
    counters.add(c["truncations"], c["updates"])
    return plan


def hmul(alpha: float, A: HMatrix, B: HMatrix, C: HMatrix, policy: TruncationPolicy, **kw):
    """C += alpha * A @ B over matching block structures (arith.py:40-55)."""
    if alpha == 0.0:
        return None
    if A.nrows != C.nrows or B.ncols != C.ncols or A.ncols != B.nrows:
        raise ValueError("non-conformal hmul operands")
    return _run_op("hmul", A, B, C, policy, alpha=alpha, **kw)


def htrsl(L: HMatrix, M: HMatrix, X: HMatrix, policy: TruncationPolicy, **kw):
    """Solve L X = M (L unit lower triangular); M is consumed (arith.py:97-117)."""
    if L.nrows != M.nrows or M.nrows != L.ncols:
        raise ValueError("non-conformal triangular solve")
    return _run_op("htrsl", L, M, X, policy, **kw)


def htrsu(U: HMatrix, M: HMatrix, X: HMatrix, policy: TruncationPolicy, **kw):
    """Solve X U = M (U upper triangular); M is consumed (arith.py:120-140)."""
    if U.ncols != M.ncols or M.ncols != U.nrows:
        raise ValueError("non-conformal triangular solve")
    return _run_op("htrsu", U, M, X, policy, **kw)
