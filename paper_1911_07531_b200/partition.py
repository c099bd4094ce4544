"""Block-row partitioned H-LU over several GPUs.

The reference executes its task DAG on one many-core node
(taskgraph.py:636-665 builds it; the paper's executor is absent).  Here the
lowered program of one H-LU (planner.plan_hlu) is split over ``nranks``
owners by block row: a task belongs to the rank that owns the row cluster
of the block it writes (the cluster-tree subtree at depth log2(nranks)), so
whole block rows of L, U, A and the accumulators stay on one GPU.

Execution graph: the data-flow edges of the sequential program
(planner.dataflow_edges: RAW, WAW and WAR on every leaf, accumulator and
micro-task result); any topological order of them reproduces the
sequential program, so every rank's results equal the single-GPU bits.

Exchange: one copy per (object version, reading rank).  When a task is
the last writer of an object that a task of another rank accesses next,
the writer's CTA copies the object into that rank's storage over NVLink
(hmx_pub records, executed by the persistent kernel right after the task,
before it releases its successors through remote atomics on the owners'
in-degree counters and ready queues).  The data-flow edges order every
such copy after the destination's earlier accesses and before its later
ones, so no rank ever reads a stale or half-written object.

Two launch forms share the records: ``rank=-1`` emulates every rank in one
launch on one GPU (CTA c serves rank c mod nranks; each rank's storage is a
replica in the same pools, the ops and records carry the replica offsets),
used by the tests to prove the protocol bit-exact; ``rank>=0`` (one
process per GPU) is driven by :class:`DistributedHLU`: every rank builds the
same partition, exports CUDA IPC handles of its pools and scheduler state
over ``torch.distributed``, maps its peers' (hmx_plan_peer), then per run
resets its scheduler, meets the others at a barrier and launches without
reset (mode 4).  Ranks wait on one another inside the launch, so each rank
needs its own GPU (two such kernels time-sliced on one GPU stall each
other until the driver's context-switch watchdog fires): on the
single-GPU boxes of this build only the emulated form runs on the device;
the host protocol of DistributedHLU is covered by the gloo world-2 test
(tests/test_partition_cpu.py) with the device calls recorded.
"""

from __future__ import annotations

import numpy as np

from . import _lib
from .planner import ACC_BASE_ID, WS_BASE_ID, dataflow_edges, plan_hlu, shift_ops

PUB_DTYPE = np.dtype([
    ("kind", "<i4"), ("dst", "<i4"), ("base", "<i4"), ("rbase", "<i4"),
    ("src_off", "<i8"), ("dst_off", "<i8"), ("src_off2", "<i8"), ("dst_off2", "<i8"),
    ("len", "<i8"), ("m", "<i4"), ("n", "<i4"), ("src_ridx", "<i4"), ("dst_ridx", "<i4"),
])
assert PUB_DTYPE.itemsize == 72


def row_bounds(table, nranks: int):
    """First row of each rank's block-row range: the row clusters of the
    diagonal blocks at depth log2(nranks); an even split of the rows when the
    diagonal becomes a leaf above that depth."""
    d = int(round(np.log2(nranks)))
    if nranks < 1 or 2 ** d != nranks:
        raise ValueError("nranks must be a power of two")
    diag = [u for u in range(table.n)
            if table.depth[u] == d and table.r0[u] == table.c0[u] and table.r1[u] == table.c1[u]]
    if len(diag) == nranks:
        return np.array(sorted(int(table.r0[u]) for u in diag), dtype=np.int64)
    nrows = int(table.r1[0] - table.r0[0])
    return np.array([int(table.r0[0]) + (nrows * r) // nranks for r in range(nranks)], dtype=np.int64)


class Partition:
    """Owners, execution edges and exchange records of one program."""

    def __init__(self, prog, table, nranks: int):
        self.prog = prog
        self.table = table
        self.nranks = int(nranks)
        self.bounds = row_bounds(table, self.nranks)
        nt = len(prog.rw)
        self.n_tasks = nt
        t = table
        leaves_of = {}

        def expand(o):
            if o[0] == "m" and not t.leaf[o[2]]:
                v = leaves_of.get(o)
                if v is None:
                    v = leaves_of[o] = [("m", o[1], x) for x in t.leaves(o[2])]
                return v
            return (o,)

        self._expand = expand

        def row_owner(u):
            return int(np.searchsorted(self.bounds, t.r0[u], side="right") - 1)

        owner = np.full(nt, -1, dtype=np.int32)
        w_reader = {}
        for i, (rds, wrs) in enumerate(prog.rw):
            for o in wrs:
                if o[0] in ("m", "a"):
                    owner[i] = row_owner(o[2] if o[0] == "m" else o[1])
                    break
            for o in rds:
                if o[0] == "w":
                    w_reader[o[1]] = i
        # micro-tasks (write only a workspace result) run where it is consumed
        for i, (rds, wrs) in enumerate(prog.rw):
            if owner[i] < 0:
                ws = [o[1] for o in wrs if o[0] == "w"]
                if ws and ws[0] in w_reader and owner[w_reader[ws[0]]] >= 0:
                    owner[i] = owner[w_reader[ws[0]]]
                else:
                    owner[i] = 0
        self.owner = owner
        # exchange: (writer task, object, destination rank), program order
        last_w = {}
        sent = set()
        pubs = [[] for _ in range(nt)]
        for i, (rds, wrs) in enumerate(prog.rw):
            r = int(owner[i])
            seen = set()
            for o0 in list(rds) + list(wrs):
                for o in expand(o0):
                    if o in seen:
                        continue
                    seen.add(o)
                    w = last_w.get(o)
                    if w is not None and owner[w] != r and (o, w, r) not in sent:
                        sent.add((o, w, r))
                        pubs[w].append((o, r))
            for o0 in wrs:
                for o in expand(o0):
                    last_w[o] = i
        self.pubs = pubs
        self.final_writer = last_w
        self.n_transfers = len(sent)
        e = np.array(sorted(dataflow_edges(prog, {0: t, 1: t, 2: t})), dtype=np.int64).reshape(-1, 2)
        self.edges = e
        self.cross_edges = int(np.count_nonzero(owner[e[:, 0]] != owner[e[:, 1]])) if len(e) else 0

    # ------------------------------------------------------------------
    def csr(self):
        nt, e = self.n_tasks, self.edges
        ptr = np.zeros(nt + 1, dtype=np.int32)
        if len(e):
            np.add.at(ptr, e[:, 0] + 1, 1)
        ptr = np.cumsum(ptr).astype(np.int32)
        idx = e[np.argsort(e[:, 0], kind="stable"), 1].astype(np.int32) if len(e) else np.zeros(0, np.int32)
        return ptr, idx

    def replica_sizes(self):
        """Element / rank-slot strides of one rank's storage per base id."""
        prog, lay, nb = self.prog, self.prog.layout, self.table.n
        base = {0: lay.size, 1: lay.size, 2: lay.size, ACC_BASE_ID: prog.acc_size, WS_BASE_ID: prog.ws_size}
        slots = {0: nb, 1: nb, 2: nb, ACC_BASE_ID: nb, WS_BASE_ID: prog.ws_slots}
        return base, slots

    def records(self, emulate: bool):
        """hmx_pub records (CSR over tasks).  Emulated: offsets include the
        source / destination replica shifts."""
        prog, t, lay = self.prog, self.table, self.prog.layout
        bsz, ssz = self.replica_sizes()
        acc_u, acc_v, acc_d, _ = getattr(prog, "acc_offsets", ({}, {}, {}, {}))
        w_info = getattr(prog, "w_info", {})
        recs = []
        ptr = np.zeros(self.n_tasks + 1, dtype=np.int64)

        def add(src, dst, kind, base, rbase, off, off2, ln, m, n, ridx):
            a = src if emulate else 0
            b = dst if emulate else 0
            recs.append((kind, dst, base, rbase, off + a * bsz[base], off + b * bsz[base],
                         off2 + a * bsz[base], off2 + b * bsz[base], ln, m, n,
                         ridx + a * ssz[rbase] if ridx >= 0 else -1,
                         ridx + b * ssz[rbase] if ridx >= 0 else -1))

        for w in range(self.n_tasks):
            src = int(self.owner[w])
            for o, dst in self.pubs[w]:
                if o[0] == "m":
                    b, u = int(o[1]), int(o[2])
                    m, n = int(t.m[u]), int(t.nc[u])
                    if t.adm[u]:
                        add(src, dst, 1, b, b, int(lay.u_off[u]), int(lay.v_off[u]), 0, m, n, u)
                    else:
                        add(src, dst, 0, b, b, int(lay.d_off[u]), 0, m * n, 0, 0, -1)
                elif o[0] == "a":
                    u = int(o[1])
                    m, n = int(t.m[u]), int(t.nc[u])
                    if u in acc_u:
                        add(src, dst, 1, ACC_BASE_ID, ACC_BASE_ID, int(acc_u[u]), int(acc_v[u]), 0, m, n, u)
                    if u in acc_d:
                        add(src, dst, 0, ACC_BASE_ID, ACC_BASE_ID, int(acc_d[u]), 0, m * n, 0, 0, -1)
                else:
                    regions, slot = w_info[o[1]]
                    for j, (off, ln) in enumerate(regions):
                        add(src, dst, 0, WS_BASE_ID, WS_BASE_ID, int(off), 0, int(ln), 0, 0,
                            int(slot) if j == 0 else -1)
            ptr[w + 1] = len(recs)
        arr = np.array(recs, dtype=PUB_DTYPE) if recs else np.zeros(0, dtype=PUB_DTYPE)
        return ptr, arr

    def stats(self):
        nt = np.bincount(self.owner, minlength=self.nranks)
        return {"nranks": self.nranks, "tasks_per_rank": nt.tolist(),
                "imbalance": float(nt.max() / max(nt.mean(), 1e-9)),
                "edges": int(len(self.edges)), "cross_edges": self.cross_edges,
                "transfers": self.n_transfers}


def simulate(part: Partition, seed=0, nsteps=None):
    """Discrete-event check of the exchange protocol (CPU): tasks run in a
    random order the edges allow, with random durations, each rank keeping
    per-object versions.  Every access must see the version the sequential
    program would, and no copy may land in a rank while a task of that rank
    that touches the object is running.  Returns the number of copies made."""
    rng = np.random.default_rng(seed)
    prog, nt = part.prog, part.n_tasks
    ptr, idx = part.csr()
    indeg = np.bincount(idx, minlength=nt).astype(np.int64)
    # version each access must observe: the last writer in program order
    expect = []
    last = {}
    for i, (rds, wrs) in enumerate(prog.rw):
        acc = {}
        for o0 in list(rds) + list(wrs):
            for o in part._expand(o0):
                acc[o] = last.get(o, -1)
        expect.append(acc)
        for o0 in wrs:
            for o in part._expand(o0):
                last[o] = i
    have = [dict() for _ in range(part.nranks)]  # rank -> obj -> version (missing = -1)
    running = [dict() for _ in range(part.nranks)]  # rank -> task -> its objects
    import heapq

    ready = [i for i in range(nt) if indeg[i] == 0]
    events = []  # (finish time, task)
    now = 0.0
    copies = 0
    done = 0
    while ready or events:
        # start every ready task (unbounded workers; order randomised)
        rng.shuffle(ready)
        for i in ready:
            r = int(part.owner[i])
            for o, v in expect[i].items():
                got = have[r].get(o, -1)
                if got != v:
                    raise AssertionError(f"task {i} on rank {r} sees version {got} of {o}, expected {v}")
            running[r][i] = set(expect[i])
            heapq.heappush(events, (now + float(rng.exponential(1.0)), i))
        ready = []
        now, i = heapq.heappop(events)
        r = int(part.owner[i])
        del running[r][i]
        rds, wrs = prog.rw[i]
        for o0 in wrs:
            for o in part._expand(o0):
                have[r][o] = i
        for o, dst in part.pubs[i]:
            for j, objs in running[dst].items():
                if o in objs:
                    raise AssertionError(f"copy of {o} from task {i} lands on rank {dst} while task {j} uses it")
            have[dst][o] = have[r].get(o, -1)
            copies += 1
        for k in range(ptr[i], ptr[i + 1]):
            s = idx[k]
            indeg[s] -= 1
            if indeg[s] == 0:
                ready.append(int(s))
        done += 1
    if done != nt:
        raise AssertionError("deadlock: not every task ran")
    return copies


# ----------------------------------------------------------------------
# device plans
# ----------------------------------------------------------------------
def _torch():
    import torch

    return torch


class PartitionedPlan:
    """H-LU plan partitioned over ``nranks`` block-row owners.

    rank = -1: all ranks emulated in one launch on this GPU (storage of
    rank r = replica r of batched stores, see :meth:`stores`).  rank >= 0
    raises NotImplementedError (see the module docstring).
    """

    def __init__(self, table, mode, policy, rank_cap, nranks, rank=-1, split_min=None,
                 ctas_per_sm=1, max_ctas=0, _multiprocess=False):
        from . import engine

        if mode not in ("std", "accu"):
            raise ValueError("mode must be 'std' or 'accu'")
        if int(rank) >= 0 and not _multiprocess:
            raise NotImplementedError(
                "a real rank (rank >= 0) needs its peers mapped before the launch: "
                "use DistributedHLU (one process per GPU)")
        split_min = engine.DEFAULT_SPLIT_MIN if split_min is None else split_min
        self.table, self.mode, self.policy, self.rank_cap = table, mode, policy, rank_cap
        self.nranks, self.rank = int(nranks), int(rank)
        self.emulate = self.rank < 0
        prog = plan_hlu(table, mode, policy, rank_cap, split_min=split_min)
        self.prog = prog
        self.layout = prog.layout
        part = Partition(prog, table, self.nranks)
        self.part = part
        ptr, idx = part.csr()
        ops = prog.ops.copy()
        if self.emulate:
            bsz, ssz = part.replica_sizes()
            per_op = np.repeat(part.owner.astype(np.int64), np.diff(prog.task_ops))
            ops = shift_ops(ops, per_op, bsz, ssz)
        from . import taskgraph as tg

        lv = tg.asap_levels(part.n_tasks, ptr, idx)
        order = np.argsort(lv, kind="stable").astype(np.int32)
        counts = np.bincount(lv, minlength=int(lv.max()) + 1 if len(lv) else 1)
        wave_ptr = np.concatenate([[0], np.cumsum(counts)]).astype(np.int32)
        self.plan = _lib.Plan(ops, prog.task_ops, ptr, idx, wave_ptr, order, prog.scratch_doubles,
                              prog.scratch_ranks, max_ctas, ctas_per_sm,
                              task_scratch=prog.task_scratch)
        pptr, pub = part.records(self.emulate)
        self.n_pub = len(pub)
        self.plan.partition(self.nranks, self.rank, part.owner, pptr, pub)
        torch = _torch()
        nrep = self.nranks if self.emulate else 1
        self.acc_values = torch.zeros(prog.acc_size * nrep, dtype=torch.float64, device="cuda")
        self.acc_ranks = torch.zeros(max(table.n, 1) * nrep, dtype=torch.int32, device="cuda")
        self.ws_values = torch.zeros(prog.ws_size * nrep, dtype=torch.float64, device="cuda")
        self.ws_ranks = torch.zeros(prog.ws_slots * nrep, dtype=torch.int32, device="cuda")
        self.plan.bind(ACC_BASE_ID, self.acc_values, self.acc_ranks)
        self.plan.bind(WS_BASE_ID, self.ws_values, self.ws_ranks)

    def stores(self, A):
        """Emulated ranks: per-rank replicas of A (copies) and zero L, U."""
        from .engine import HStore

        n = self.nranks if self.emulate else 1
        AB = HStore.batch(self.layout, n)
        for r in range(n):
            AB.instance(r).copy_from(A)
        return AB, HStore.batch(self.layout, n), HStore.batch(self.layout, n)

    def bind(self, A, L, U):
        for i, s in enumerate((A, L, U)):
            self.plan.bind(i, s.values, s.ranks)

    def run(self, A, L, U, stream=None, check=True):
        self.bind(A, L, U)
        self.plan.reset_counters(stream)
        self.plan.execute(2, stream)
        if check:
            self.check(stream)

    def check(self, stream=None):
        st = self.plan.status(stream)
        if st:
            if st & _lib.HMX_ERR_PIVOT:
                from .arith import SingularPivotError

                raise SingularPivotError("vanishing pivot in a diagonal leaf (device)")
            raise _lib.HmxError(st, "partitioned H-LU execution")

    def collect(self, S, base_id):
        """Single-matrix store holding, for every leaf of matrix ``base_id``,
        the final version from the replica of the rank that last wrote it
        (emulated runs)."""
        from .engine import HStore

        torch = _torch()
        lay, t = self.layout, self.table
        out = HStore(lay)
        sz, nb = lay.size, t.n
        src = torch.empty(0, dtype=torch.int64)
        vi, vs, ri, rs = [], [], [], []
        for u in t.leaves(0):
            w = self.part.final_writer.get(("m", base_id, u))
            r = int(self.part.owner[w]) if w is not None else 0
            if t.adm[u]:
                a, b = int(lay.u_off[u]), int(lay.v_off[u] + t.nc[u] * lay.cap[u])
            else:
                a, b = int(lay.d_off[u]), int(lay.d_off[u] + t.m[u] * t.nc[u])
            vi.append(np.arange(a, b))
            vs.append(np.arange(a, b) + r * sz)
            ri.append(u)
            rs.append(u + r * nb)
        vi, vs = np.concatenate(vi), np.concatenate(vs)
        out.values[torch.from_numpy(vi).cuda()] = S.values[torch.from_numpy(vs).cuda()]
        out.ranks[torch.from_numpy(np.array(ri)).cuda()] = S.ranks[torch.from_numpy(np.array(rs)).cuda()]
        del src
        return out


# ----------------------------------------------------------------------
# one process per GPU
# ----------------------------------------------------------------------
class _Backend:
    """Device calls of DistributedHLU (replaced by a recorder in the CPU test)."""

    ipc_handle = staticmethod(lambda ptr: _lib.ipc_handle(ptr))
    ipc_open = staticmethod(lambda handle: _lib.ipc_open(handle))
    ipc_close = staticmethod(lambda base: _lib.ipc_close(base))

    @staticmethod
    def synchronize():
        _torch().cuda.synchronize()


def export_table(pointers, backend=_Backend):
    """{name: address} -> {name: (ipc handle bytes, offset)} (0 stays None)."""
    out = {}
    for k, ptr in pointers.items():
        out[k] = None if not ptr else tuple(backend.ipc_handle(int(ptr)))
    return out


def import_table(table, opened, backend=_Backend):
    """Peer's exported table -> {name: address in this process}.  Several
    pools may live in one allocation (torch's caching allocator): every
    handle is opened once (``opened``: handle bytes -> mapped base)."""
    out = {}
    for k, v in table.items():
        if v is None:
            out[k] = 0
            continue
        handle, off = v
        base = opened.get(handle)
        if base is None:
            base = opened[handle] = int(backend.ipc_open(handle))
        out[k] = base + int(off)
    return out


class DistributedHLU:
    """Block-row partitioned H-LU, one process per GPU.

    ``torch.distributed`` must be initialised (NCCL on the GPUs; the object
    collectives used here also run on gloo).  Every rank holds full-size
    pools; it executes the tasks of its block rows and receives the objects
    it reads from the ranks that produce them (hmx_pub records, written by
    the producer's CTA straight into this rank's pools over NVLink).

        d = DistributedHLU(table, "accu", policy, rank_cap)
        A, L, U = d.stores(A_full)        # this rank's pools
        d.connect(A, L, U)                # IPC exchange, once per storage
        d.run()                           # reset, barrier, launch, status
        Lfull = d.collect(L, 1)           # all-reduce of the owned leaves
    """

    BASES = (0, 1, 2, ACC_BASE_ID, WS_BASE_ID)

    def __init__(self, table, mode, policy, rank_cap, group=None, split_min=None, ctas_per_sm=1,
                 max_ctas=0, backend=_Backend, plan=None):
        import torch.distributed as dist

        self.dist, self.group, self.backend = dist, group, backend
        self.rank, self.nranks = dist.get_rank(group), dist.get_world_size(group)
        if self.nranks < 2:
            raise ValueError("DistributedHLU needs at least two ranks")
        self.pp = plan if plan is not None else PartitionedPlan(
            table, mode, policy, rank_cap, self.nranks, self.rank, split_min, ctas_per_sm, max_ctas,
            _multiprocess=True)
        self.part = self.pp.part
        self._opened = {}
        self._connected = False

    def stores(self, A):
        """This rank's pools: a copy of A and zero L, U."""
        return self.pp.stores(A)

    def _pointers(self, A, L, U):
        pp = self.pp
        t = {}
        for b, (v, r) in zip(self.BASES, ((A.values, A.ranks), (L.values, L.ranks), (U.values, U.ranks),
                                          (pp.acc_values, pp.acc_ranks), (pp.ws_values, pp.ws_ranks))):
            t[f"v{b}"] = v.data_ptr() if v.numel() else 0
            t[f"r{b}"] = r.data_ptr() if r.numel() else 0
        t["indeg"], t["queue"], t["qctl"] = pp.plan.sched_state()
        return t

    def connect(self, A, L, U):
        """Bind this rank's pools and map every peer's pools and scheduler
        state (one all_gather of the IPC handle tables)."""
        self.pp.bind(A, L, U)
        mine = export_table(self._pointers(A, L, U), self.backend)
        tables = [None] * self.nranks
        self.dist.all_gather_object(tables, mine, group=self.group)
        for r, tab in enumerate(tables):
            if r == self.rank:
                continue
            adr = import_table(tab, self._opened, self.backend)
            bases, rbases = [0] * 16, [0] * 16
            for b in self.BASES:
                bases[b], rbases[b] = adr[f"v{b}"], adr[f"r{b}"]
            self.pp.plan.peer(r, bases, rbases, adr["indeg"], adr["queue"], adr["qctl"])
        self._connected = True
        self.dist.barrier(group=self.group)

    def run(self, stream=None, check=True, events=None):
        """One factorization (events: optional (start, end) CUDA events
        recorded around this rank's launch).  Every rank resets its own scheduler state
        BEFORE the barrier: a peer may release tasks of this rank as soon as
        it starts, so no rank may launch while another still resets."""
        if not self._connected:
            raise RuntimeError("connect(A, L, U) first")
        plan = self.pp.plan
        plan.reset_counters(stream)
        plan.reset(stream)
        self.backend.synchronize()
        self.dist.barrier(group=self.group)
        if events is not None:
            events[0].record(stream)
        plan.execute(4, stream)
        if events is not None:
            events[1].record(stream)
        if check:
            self.pp.check(stream)
        self.dist.barrier(group=self.group)

    def owned_leaves(self, base_id):
        """Leaves of matrix ``base_id`` whose final version this rank wrote."""
        t, part = self.pp.table, self.part
        out = []
        for u in t.leaves(0):
            w = part.final_writer.get(("m", base_id, u))
            if (int(part.owner[w]) if w is not None else 0) == self.rank:
                out.append(int(u))
        return out

    def collect(self, S, base_id):
        """Full matrix ``base_id`` on every rank: each rank contributes the
        leaves it wrote last, one all-reduce (outside the factorization)."""
        from .engine import HStore

        torch = _torch()
        lay, t = self.pp.layout, self.pp.table
        out = HStore(lay)
        out.values.zero_()
        out.ranks.zero_()
        idx, ridx = [], []
        for u in self.owned_leaves(base_id):
            if t.adm[u]:
                a, b = int(lay.u_off[u]), int(lay.v_off[u] + t.nc[u] * lay.cap[u])
            else:
                a, b = int(lay.d_off[u]), int(lay.d_off[u] + t.m[u] * t.nc[u])
            idx.append(np.arange(a, b))
            ridx.append(u)
        if idx:
            ii = torch.from_numpy(np.concatenate(idx)).to(S.values.device)
            out.values[ii] = S.values[ii]
            rr = torch.from_numpy(np.asarray(ridx)).to(S.ranks.device)
            out.ranks[rr] = S.ranks[rr]
        self.dist.all_reduce(out.values, group=self.group)
        self.dist.all_reduce(out.ranks, group=self.group)
        return out

    def close(self):
        for base in self._opened.values():
            try:
                self.backend.ipc_close(base)
            except Exception:
                pass
        self._opened = {}
        self._connected = False


__all__ = ["Partition", "PartitionedPlan", "DistributedHLU", "row_bounds", "simulate", "PUB_DTYPE",
           "export_table", "import_table"]
