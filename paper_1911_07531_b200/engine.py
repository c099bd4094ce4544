"""Device storage and DAG execution of H-arithmetic plans.

``HStore``   one H-matrix in HBM: a pooled fp64 tensor holding every dense
             leaf and every low-rank factor arena (Layout offsets) plus an
             int32 rank array indexed by block uid.
``ExecPlan`` a lowered H-LU (planner.Program) bound to its execution graph:
             the node set is the reference DAG of taskgraph.build_hlu_dag;
             edges are that DAG's edges plus, for accumulator modes, the
             per-accumulator fold order of accumulator.hlu_accu (the DAG
             alone does not order a parent shift against a direct add into
             the same accumulator — SURVEY.md finding 3).  The graph is
             uploaded once (CSR + in-degrees + ASAP wavefronts) into an
             hmx_plan and replayed by the device executors.
"""

from __future__ import annotations

import numpy as np

from . import _lib
from . import taskgraph as tg
from .planner import ACC_BASE_ID, Layout, dataflow_edges, plan_hlu, plan_op
from .trees import BlockTable

EXEC_WAVE, EXEC_GRAPH, EXEC_PERSISTENT, EXEC_SEQUENTIAL = 0, 1, 2, 3
WS_BASE_ID = 5
# H x H products with min(m, n) >= this are split into parallel micro-tasks
DEFAULT_SPLIT_MIN = 256


def _torch():
    import torch

    if not torch.cuda.is_available():
        raise RuntimeError("the H-LU engine needs a CUDA device; there is no CPU fallback")
    return torch


class HStore:
    """Device storage of one H-matrix (values pool + rank slots)."""

    def __init__(self, layout: Layout, values=None, ranks=None):
        torch = _torch()
        self.layout = layout
        self.table = layout.table
        n = self.table.n
        self.values = values if values is not None else torch.zeros(
            layout.size, dtype=torch.float64, device="cuda")
        if ranks is None:
            r = np.full(n, -1, dtype=np.int32)
            r[self.table.leaf & self.table.adm] = 0
            ranks = torch.from_numpy(r).cuda()
        self.ranks = ranks

    def clone(self):
        return HStore(self.layout, self.values.clone(), self.ranks.clone())

    @property
    def nrep(self):
        return self.values.numel() // max(self.layout.size, 1)

    @classmethod
    def batch(cls, layout: Layout, nrep: int):
        """nrep same-layout matrices in one contiguous pool (batched plans)."""
        torch = _torch()
        values = torch.zeros(layout.size * nrep, dtype=torch.float64, device="cuda")
        r = np.full(layout.table.n, -1, dtype=np.int32)
        r[layout.table.leaf & layout.table.adm] = 0
        ranks = torch.from_numpy(np.tile(r, nrep)).cuda()
        return cls(layout, values, ranks)

    def instance(self, b: int):
        """View of instance b of a batched store."""
        sz, nb = self.layout.size, self.table.n
        return HStore(self.layout, self.values[b * sz:(b + 1) * sz], self.ranks[b * nb:(b + 1) * nb])

    def copy_from(self, other: "HStore"):
        self.values.copy_(other.values)
        self.ranks.copy_(other.ranks)

    # packed transfers (wire format, csrc/hmx_transfer.cu) -----------------
    def _pack_desc(self):
        d = getattr(self.layout, "_pack_desc", None)
        if d is None:
            torch = _torch()
            lay, t = self.layout, self.table
            rows = []
            for u in t.leaves(0):
                if t.adm[u]:
                    rows.append((u, lay.u_off[u], lay.v_off[u], t.m[u], t.nc[u]))
                else:
                    rows.append((u, lay.d_off[u], -1, t.m[u], t.nc[u]))
            d = torch.from_numpy(np.asarray(rows, dtype=np.int64).reshape(-1, 5)).cuda()
            self.layout._pack_desc = d
        return d

    def packed_size(self, stream=None):
        """Total doubles of the packed form at the current device ranks
        (one device->host read of the scan total)."""
        torch = _torch()
        d = self._pack_desc()
        nrep = self.nrep
        offs = torch.empty(d.shape[0] * nrep + 1, dtype=torch.int64, device="cuda")
        _lib.check(_lib.lib().hmx_pack_leaves(d.shape[0], nrep, _lib.ptr(d), self.layout.size,
                                              self.table.n, None, _lib.ptr(self.ranks), None, 0,
                                              _lib.ptr(offs), _lib.stream_ptr(stream)), "pack")
        return int(offs[-1].item())

    def pack_to(self, out, offsets=None, stream=None):
        """Gather the live leaf data into `out` (device; items beyond its
        length are skipped, see hmx_pack_leaves); returns the device offsets
        tensor (items + 1), whose last entry is the packed size."""
        torch = _torch()
        d = self._pack_desc()
        nrep = self.nrep
        if offsets is None:
            offsets = torch.empty(d.shape[0] * nrep + 1, dtype=torch.int64, device="cuda")
        _lib.check(_lib.lib().hmx_pack_leaves(d.shape[0], nrep, _lib.ptr(d), self.layout.size,
                                              self.table.n, _lib.ptr(self.values),
                                              _lib.ptr(self.ranks), _lib.ptr(out), out.numel(),
                                              _lib.ptr(offsets), _lib.stream_ptr(stream)), "pack")
        return offsets

    def unpack_from(self, packed, offsets=None, stream=None):
        """Scatter packed leaf data into the pool; self.ranks must already
        hold the ranks the packed form was made with."""
        torch = _torch()
        d = self._pack_desc()
        nrep = self.nrep
        if offsets is None:
            offsets = torch.empty(d.shape[0] * nrep + 1, dtype=torch.int64, device="cuda")
        _lib.check(_lib.lib().hmx_unpack_leaves(d.shape[0], nrep, _lib.ptr(d), self.layout.size,
                                                self.table.n, _lib.ptr(packed),
                                                _lib.ptr(self.ranks), _lib.ptr(self.values),
                                                _lib.ptr(offsets), _lib.stream_ptr(stream)),
                   "unpack")
        return offsets

    # host transfers -----------------------------------------------------
    def upload_leaves(self, leaves):
        """leaves: uid -> ("D", M) | ("R", U, V) (row-major numpy)."""
        torch = _torch()
        lay, t = self.layout, self.table
        buf = np.zeros(lay.size, dtype=np.float64)
        r = np.full(t.n, -1, dtype=np.int32)
        for u, x in leaves.items():
            m, n = int(t.m[u]), int(t.nc[u])
            if x[0] == "D":
                o = int(lay.d_off[u])
                buf[o:o + m * n] = np.asarray(x[1], dtype=np.float64).T.ravel()
            else:
                k = x[1].shape[1]
                if k > lay.cap[u]:
                    raise _lib.HmxError(_lib.HMX_ERR_RANK_OVERFLOW, f"upload of block {u}")
                uo, vo = int(lay.u_off[u]), int(lay.v_off[u])
                buf[uo:uo + m * k] = np.asarray(x[1]).T.ravel()
                buf[vo:vo + n * k] = np.asarray(x[2]).T.ravel()
                r[u] = k
        self.values.copy_(torch.from_numpy(buf))
        self.ranks.copy_(torch.from_numpy(r))

    def upload_leaf(self, u, x):
        torch = _torch()
        lay, t = self.layout, self.table
        m, n = int(t.m[u]), int(t.nc[u])
        if x[0] == "D":
            o = int(lay.d_off[u])
            self.values[o:o + m * n].copy_(torch.from_numpy(np.ascontiguousarray(x[1].T).ravel()))
        else:
            k = x[1].shape[1]
            if k > lay.cap[u]:
                raise _lib.HmxError(_lib.HMX_ERR_RANK_OVERFLOW, f"upload of block {u}")
            uo, vo = int(lay.u_off[u]), int(lay.v_off[u])
            self.values[uo:uo + m * k].copy_(torch.from_numpy(np.ascontiguousarray(x[1].T).ravel()))
            self.values[vo:vo + n * k].copy_(torch.from_numpy(np.ascontiguousarray(x[2].T).ravel()))
            self.ranks[u] = k

    def download_leaf(self, u):
        lay, t = self.layout, self.table
        m, n = int(t.m[u]), int(t.nc[u])
        if t.adm[u]:
            k = int(self.ranks[u].item())
            uo, vo = int(lay.u_off[u]), int(lay.v_off[u])
            U = self.values[uo:uo + m * k].cpu().numpy().reshape(k, m).T.copy()
            V = self.values[vo:vo + n * k].cpu().numpy().reshape(k, n).T.copy()
            return ("R", U, V)
        o = int(lay.d_off[u])
        return ("D", self.values[o:o + m * n].cpu().numpy().reshape(n, m).T.copy())

    def download_leaves(self):
        lay, t = self.layout, self.table
        buf = self.values.cpu().numpy()
        r = self.ranks.cpu().numpy()
        out = {}
        for u in t.leaves(0):
            m, n = int(t.m[u]), int(t.nc[u])
            if t.adm[u]:
                k = int(r[u])
                uo, vo = int(lay.u_off[u]), int(lay.v_off[u])
                U = buf[uo:uo + m * k].reshape(k, m).T.copy()
                V = buf[vo:vo + n * k].reshape(k, n).T.copy()
                out[u] = ("R", U, V)
            else:
                o = int(lay.d_off[u])
                out[u] = ("D", buf[o:o + m * n].reshape(n, m).T.copy())
        return out


def task_signature(ops, task_ops):
    """Batch key of every task: (op code, rows, columns) of its heaviest op -
    the truncation / dense_to_lowrank if it has one, else the LU / TRSM,
    else its first GEMM, else its first op - packed into one int64."""
    nt = len(task_ops) - 1
    if nt == 0:
        return np.zeros(0, dtype=np.int64)
    code = ops["code"].astype(np.int64)
    d0 = np.maximum(ops["dim"][:, 0].astype(np.int64), 0)
    d1 = np.maximum(ops["dim"][:, 1].astype(np.int64), 0)
    # priority of an op as the task's representative
    prio = np.select([np.isin(code, (8, 9)), np.isin(code, (5, 6, 7, 13)), code == 1], [3, 2, 1], 0)
    key = prio * (1 << 50) + (code << 44) + (np.minimum(d0, (1 << 22) - 1) << 22) + np.minimum(d1, (1 << 22) - 1)
    starts = np.asarray(task_ops[:-1], dtype=np.int64)
    empty = np.diff(np.asarray(task_ops, dtype=np.int64)) == 0
    sig = np.maximum.reduceat(key, np.minimum(starts, len(key) - 1)) if len(key) else np.zeros(nt, np.int64)
    sig = np.where(empty, 0, sig)
    return sig & ((1 << 50) - 1)


def wave_batches(levels, ops, task_ops):
    """Task order of the ASAP wavefronts with every wavefront sorted into
    batches of equal signature (operation type and leaf shape).  Returns
    (order, signature per task)."""
    sig = task_signature(ops, task_ops)
    order = np.lexsort((sig, np.asarray(levels))).astype(np.int32)
    return order, sig


class ExecPlan:
    """Lowered H-LU plan + its device execution graph."""

    def __init__(self, table: BlockTable, mode: str, policy, rank_cap=None, dag_mode=None,
                 sparsify=False, max_ctas=0, nrep=1, split_min=DEFAULT_SPLIT_MIN,
                 ctas_per_sm=None, caps=None, python_planner=False, acc_budget=0,
                 scratch_budget=None):
        if mode not in ("std", "accu"):
            raise ValueError("mode must be 'std' or 'accu'")
        self.table = table
        self.mode = mode
        self.policy = policy
        self.rank_cap = rank_cap
        dag_mode = dag_mode or ("std" if mode == "std" else tg.MERGED)
        if (mode == "std") != (dag_mode == tg.STD):
            raise ValueError(f"DAG mode {dag_mode} does not execute {mode} arithmetic")
        self.dag_mode = dag_mode
        if dag_mode != tg.COMBINED and not python_planner:
            # native lowering + execution graph (csrc/hmx_lower.cpp) against
            # the reference DAG from the native refinement builder
            from .lower import NativeProgram

            prog = NativeProgram(table, mode, policy, rank_cap, split_min=split_min, caps=caps,
                                 acc_budget=acc_budget)
            self.prog = prog
            self.layout = prog.layout
            h = tg.dag_handle(table, dag_mode, sparsify=sparsify)
            ptr, idx = prog.graph(h.ptr, mode)
            h.free()
            self.n_dag_edges = prog.n_dag_edges
            self.n_chain_edges = -1
        else:
            # Python planner (the specification of the native one) and, for
            # the combined DAG, apply tasks fused into their leaf tasks
            if caps is not None:
                raise ValueError("rank-bounded layouts need the native planner")
            prog = plan_hlu(table, mode, policy, rank_cap, split_min=split_min)
            if dag_mode == tg.COMBINED:
                from .planner import fuse_applies

                prog = fuse_applies(prog)
            self.prog = prog
            self.layout = prog.layout
            self.dag = tg.build_dag_native(table, dag_mode, sparsify=sparsify)
            ptr, idx, self.n_dag_edges, self.n_chain_edges = self._exec_graph()
        self.succ_ptr, self.succ_idx = ptr, idx
        lv = tg.asap_levels(len(prog.task_ops) - 1, ptr, idx)
        self.levels = lv
        self.n_tasks = len(prog.task_ops) - 1
        self.nrep = int(nrep)
        ops, task_ops = prog.ops, prog.task_ops
        if self.nrep > 1:
            # disjoint union of nrep copies: batched same-structure instances
            from .planner import replicate

            nb = table.n
            lay = self.layout
            ops, task_ops, _ = replicate(prog, self.nrep,
                                         {0: lay.size, 1: lay.size, 2: lay.size, 3: prog.acc_size,
                                          WS_BASE_ID: prog.ws_size},
                                         {0: nb, 1: nb, 2: nb, 3: nb, WS_BASE_ID: prog.ws_slots})
            nt, ne = self.n_tasks, len(idx)
            ptr = np.concatenate([ptr[:-1] + b * ne for b in range(self.nrep)] +
                                 [[ne * self.nrep]]).astype(np.int32)
            idx = np.concatenate([idx + b * nt for b in range(self.nrep)]).astype(np.int32)
            lv = np.tile(lv, self.nrep)
        # ready-set wavefronts; inside a wavefront the tasks are grouped into
        # batches of equal operation type and leaf shape (wave_batches)
        order, self.batch_sig = wave_batches(lv, ops, task_ops)
        counts = np.bincount(lv, minlength=int(lv.max()) + 1 if len(lv) else 1)
        self.wave_ptr = np.concatenate([[0], np.cumsum(counts)]).astype(np.int32)
        self.wave_tasks = order
        # executor variant: one CTA per SM (latency) for a single matrix, two
        # per SM (throughput) for a batch of independent instances
        self.ctas_per_sm = int(ctas_per_sm or (2 if self.nrep > 1 else 1))
        tsc = prog.task_scratch if self.nrep == 1 else np.tile(prog.task_scratch, self.nrep)
        self.plan = _lib.Plan(ops, task_ops, ptr, idx, self.wave_ptr, self.wave_tasks,
                              prog.scratch_doubles, prog.scratch_ranks, max_ctas, self.ctas_per_sm,
                              task_scratch=tsc, scratch_budget=scratch_budget)
        torch = _torch()
        self.acc_values = torch.zeros(prog.acc_size * self.nrep, dtype=torch.float64, device="cuda")
        self.acc_ranks = torch.zeros(max(table.n, 1) * self.nrep, dtype=torch.int32, device="cuda")
        self.plan.bind(ACC_BASE_ID, self.acc_values, self.acc_ranks)
        self.ws_values = torch.zeros(prog.ws_size * self.nrep, dtype=torch.float64, device="cuda")
        self.ws_ranks = torch.zeros(prog.ws_slots * self.nrep, dtype=torch.int32, device="cuda")
        self.plan.bind(WS_BASE_ID, self.ws_values, self.ws_ranks)

    def _exec_graph(self):
        """Successor CSR over program tasks (program order = trace order).

        std: the reference DAG's edges (bit-exact node and edge sets; its
        execution equals arith.hlu).
        accu: the DAG's node set with edges from the data flow of
        accumulator.hlu_accu.  The reference merged DAG orders add_upd tasks
        on nested blocks by a WAW on matrix A although they write different
        accumulators, and in places that order contradicts hlu_accu's
        per-accumulator fold order; data-flow edges replay hlu_accu exactly.
        """
        prog = self.prog
        pos = {}
        micro = set()
        for i, k in enumerate(prog.keys):
            if k[0] == "micro":
                micro.add(i)
                continue
            if k in pos:
                raise RuntimeError(f"duplicate planned task {k}")
            pos[k] = i
        dag_to_prog = []
        for t in self.dag.nodes:
            k = (t.kind, t.uids, t.alpha)
            if k not in pos:
                raise RuntimeError(f"DAG task {k} has no lowered program")
            dag_to_prog.append(pos[k])
        if len(dag_to_prog) != len(pos):
            raise RuntimeError("planned tasks and DAG nodes differ")
        dptr, didx = self.dag.csr()
        dag_edges = set()
        for i in range(len(dag_to_prog)):
            a = dag_to_prog[i]
            for j in didx[dptr[i]:dptr[i + 1]]:
                dag_edges.add((a, dag_to_prog[j]))
        groups = getattr(prog, "groups", {})
        if self.mode == "std":
            edges = set(dag_edges)
            # a DAG task's predecessors also precede its micro-tasks; the
            # micro-tasks feed the task through the plan workspace
            for a, b in dag_edges:
                for mtask in groups.get(b, ()):
                    edges.add((a, mtask))
            if micro:
                root_of = {}
                for r, ms in groups.items():
                    for mtask in ms:
                        root_of[mtask] = r
                tables = {b: self.table for b in range(4)}
                for a, b in dataflow_edges(prog, tables):
                    ga = root_of.get(a, a)
                    gb = root_of.get(b, b)
                    if ga == gb:
                        edges.add((a, b))
            n_extra = len(edges - dag_edges)
        else:
            tables = {b: self.table for b in range(4)}
            edges = dataflow_edges(prog, tables)
            n_extra = len(edges - dag_edges)
        self.n_dag_edges_kept = len(edges & dag_edges)
        n = len(prog.keys)
        src = np.fromiter((a for a, _ in edges), dtype=np.int64, count=len(edges))
        dst = np.fromiter((b for _, b in edges), dtype=np.int64, count=len(edges))
        if len(edges) and not (src < dst).all():
            raise RuntimeError("execution graph contradicts program order")
        o = np.lexsort((dst, src))
        src, dst = src[o], dst[o]
        ptr = np.zeros(n + 1, dtype=np.int64)
        np.add.at(ptr, src + 1, 1)
        ptr = np.cumsum(ptr).astype(np.int32)
        return ptr, dst.astype(np.int32), len(dag_edges), n_extra

    def bind(self, A: HStore, L: HStore, U: HStore):
        for i, s in enumerate((A, L, U)):
            if s.layout.table is not self.table and s.layout.table.n != self.table.n:
                raise ValueError("operand is not over the plan's block tree")
            if s.values.numel() < self.layout.size * self.nrep:
                raise ValueError("operand storage smaller than the plan's batch")
            if (s.layout.u_off != self.layout.u_off).any() or (s.layout.d_off != self.layout.d_off).any():
                raise ValueError("operand storage layout differs from the plan's")
            self.plan.bind(i, s.values, s.ranks)

    def run(self, A: HStore, L: HStore, U: HStore, exec_mode=EXEC_PERSISTENT, stream=None,
            check=True):
        self.bind(A, L, U)
        self.plan.reset_counters(stream)
        self.plan.execute(exec_mode, stream)
        if check:
            self.check(stream)

    def check(self, stream=None):
        st = self.plan.status(stream)
        if st:
            if st & _lib.HMX_ERR_PIVOT:
                from .arith import SingularPivotError

                raise SingularPivotError("vanishing pivot in a diagonal leaf (device)")
            raise _lib.HmxError(st, "H-LU execution")

    def counters(self, stream=None):
        c = self.plan.counters(stream)
        return {"truncations": c[0], "flops": c[1], "bytes": c[2], "tasks": c[3],
                "updates": self.prog.updates * self.nrep}

    def stats(self):
        w = np.diff(self.wave_ptr)
        lv_sig = np.stack([np.asarray(self.levels, dtype=np.int64), self.batch_sig[:len(self.levels)]], 1) \
            if len(self.levels) else np.zeros((0, 2), np.int64)
        n_batches = int(len(np.unique(lv_sig, axis=0))) if self.n_tasks <= 500000 else -1
        return {"tasks": self.n_tasks, "ops": int(len(self.prog.ops)), "dag_edges": self.n_dag_edges,
                "batches": n_batches,
                "exec_edges": int(len(self.succ_idx)), "dataflow_only_edges": self.n_chain_edges, "waves": int(len(w)),
                "max_wave": int(w.max()) if len(w) else 0,
                "scratch_mb_per_cta": self.prog.scratch_doubles * 8 / 2**20,
                "acc_mb": self.prog.acc_size * 8 / 2**20, "pool_mb": self.layout.size * 8 / 2**20}


class OpPlan:
    """Standalone multiply / triangular-solve plan (hmul, htrsl, htrsu and
    the accumulator solves).  Tasks are the leaf-level calls of the
    reference recursion (the final nodes of the refined multiply / TRSM
    DAGs, taskgraph.py:146-180); the execution graph comes from the data
    flow of the sequential recursion."""

    def __init__(self, table: BlockTable, op: str, policy, rank_cap=None, alpha=1.0, max_ctas=0,
                 uids=None):
        self.table = table
        self.op = op
        prog = plan_op(table, op, policy, rank_cap, alpha=alpha, uids=uids)
        self.prog = prog
        self.layout = prog.layout
        tables = {b: table for b in range(4)}
        edges = dataflow_edges(prog, tables)
        n = len(prog.keys)
        src = np.fromiter((a for a, _ in edges), dtype=np.int64, count=len(edges))
        dst = np.fromiter((b for _, b in edges), dtype=np.int64, count=len(edges))
        o = np.lexsort((dst, src))
        src, dst = src[o], dst[o]
        ptr = np.zeros(n + 1, dtype=np.int64)
        np.add.at(ptr, src + 1, 1)
        ptr = np.cumsum(ptr).astype(np.int32)
        idx = dst.astype(np.int32)
        lv = tg.asap_levels(n, ptr, idx) if n else np.zeros(0, np.int32)
        order = np.argsort(lv, kind="stable").astype(np.int32)
        counts = np.bincount(lv, minlength=int(lv.max()) + 1 if len(lv) else 1)
        wave_ptr = np.concatenate([[0], np.cumsum(counts)]).astype(np.int32)
        self.n_tasks = n
        self.plan = _lib.Plan(prog.ops, prog.task_ops, ptr, idx, wave_ptr, order,
                              prog.scratch_doubles, prog.scratch_ranks, max_ctas,
                              task_scratch=getattr(prog, "task_scratch", None))
        torch = _torch()
        self.acc_values = torch.zeros(prog.acc_size, dtype=torch.float64, device="cuda")
        self.acc_ranks = torch.zeros(max(table.n, 1), dtype=torch.int32, device="cuda")
        self.plan.bind(ACC_BASE_ID, self.acc_values, self.acc_ranks)
        self.ws_values = torch.zeros(getattr(prog, "ws_size", 1), dtype=torch.float64, device="cuda")
        self.ws_ranks = torch.zeros(getattr(prog, "ws_slots", 1), dtype=torch.int32, device="cuda")
        self.plan.bind(WS_BASE_ID, self.ws_values, self.ws_ranks)

    def run(self, s0: HStore, s1: HStore, s2: HStore, exec_mode=EXEC_PERSISTENT, stream=None):
        for i, st in enumerate((s0, s1, s2)):
            if st.layout.table is not self.table:
                raise ValueError("operand is not over the plan's block tree")
            self.plan.bind(i, st.values, st.ranks)
        self.plan.reset_counters(stream)
        self.plan.execute(exec_mode, stream)
        stt = self.plan.status(stream)
        if stt:
            raise _lib.HmxError(stt, self.op)

    def counters(self, stream=None):
        c = self.plan.counters(stream)
        return {"truncations": c[0], "flops": c[1], "bytes": c[2], "tasks": c[3],
                "updates": self.prog.updates}


class DensePlan:
    """H x dense operation on one block (planner.plan_dense): apply,
    apply_t (independent row/column strips, one task each) or the
    triangular solves (one sequential task).  Bases: 0 = the H-matrix pool,
    1 = X / Y (column-major, device), 2 = the output of apply / apply_t."""

    def __init__(self, table: BlockTable, op: str, uid: int, cols: int, rank_cap=None, layout=None):
        from .planner import plan_dense

        self.table, self.op, self.uid, self.cols = table, op, int(uid), int(cols)
        prog = plan_dense(table, op, uid, cols, rank_cap, layout)
        self.prog = prog
        self.layout = prog.layout
        n = len(prog.keys)
        ptr = np.zeros(n + 1, dtype=np.int32)
        idx = np.zeros(0, dtype=np.int32)
        self.plan = _lib.Plan(prog.ops, prog.task_ops, ptr, idx, np.array([0, n], np.int32),
                              np.arange(n, dtype=np.int32), prog.scratch_doubles,
                              prog.scratch_ranks, task_scratch=prog.task_scratch)

    def run(self, H: HStore, X, out=None, stream=None):
        if H.layout.table is not self.table:
            raise ValueError("operand is not over the plan's block tree")
        if H.layout is not self.layout and not (
                np.array_equal(H.layout.u_off, self.layout.u_off)
                and np.array_equal(H.layout.d_off, self.layout.d_off)
                and np.array_equal(H.layout.cap, self.layout.cap)):
            raise ValueError("operand storage layout differs from the plan's")
        self.plan.bind(0, H.values, H.ranks)
        self.plan.bind(1, X, None)
        if out is not None:
            self.plan.bind(2, out, None)
        self.plan.reset_counters(stream)
        self.plan.execute(EXEC_PERSISTENT, stream)
        st = self.plan.status(stream)
        if st:
            raise _lib.HmxError(st, self.op)
