"""Block-row partition of the H-LU program (partition.py) on CPU.

* owners, exchange records and edges are consistent (every cross-rank
  access of an object version is preceded by exactly one copy);
* a discrete-event simulation of the exchange protocol, with random task
  durations and unbounded workers per rank, never lets a task see a stale
  object and never lands a copy under a running task;
* two gloo ranks build the same partition independently (the multi-GPU
  runner relies on every rank deriving identical plans).
"""

import hashlib
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1911_07531_b200 import configs, hmatrix as H, partition as P, planner
from paper_1911_07531_b200.trees import BlockTable


def _prog(name, mode):
    cfg = configs.config(name)
    _, _, _, broot = configs.structure(cfg)
    bt = BlockTable(broot)
    pol = H.TruncationPolicy.fixed_accuracy(cfg.eps)
    return planner.plan_hlu(bt, mode, pol, 64, split_min=64), bt


@pytest.mark.parametrize("name,mode,nranks", [("s1", "std", 2), ("s1", "accu", 4), ("s2", "std", 4),
                                              ("s2", "accu", 2), ("c1", "std", 2), ("c1", "accu", 4)])
def test_partition_protocol(name, mode, nranks):
    prog, bt = _prog(name, mode)
    part = P.Partition(prog, bt, nranks)
    st = part.stats()
    assert sum(st["tasks_per_rank"]) == part.n_tasks
    assert min(st["tasks_per_rank"]) > 0
    # the copies cover every cross-rank object version exactly once
    assert sum(len(p) for p in part.pubs) == part.n_transfers
    for seed in range(3):
        assert P.simulate(part, seed=seed) == part.n_transfers
    # records: emulated offsets sit inside the destination replica
    ptr, rec = part.records(emulate=True)
    assert ptr[-1] == len(rec) >= part.n_transfers
    bsz, _ = part.replica_sizes()
    for r in rec:
        sz = bsz[int(r["base"])]
        assert r["dst_off"] // sz == r["dst"]
        assert 0 <= r["dst"] < nranks
    ptr1, rec1 = part.records(emulate=False)
    assert np.array_equal(ptr, ptr1)
    if len(rec1):
        assert (rec1["src_off"] == rec1["dst_off"]).all()


def test_row_bounds():
    prog, bt = _prog("c1", "std")
    b = P.row_bounds(bt, 4)
    assert b[0] == 0 and (np.diff(b) > 0).all() and len(b) == 4
    with pytest.raises(ValueError):
        P.row_bounds(bt, 3)


def test_simulation_catches_missing_copy():
    prog, bt = _prog("s2", "accu")
    part = P.Partition(prog, bt, 2)
    k = next(i for i, p in enumerate(part.pubs) if p)
    part.pubs[k] = part.pubs[k][1:]
    with pytest.raises(AssertionError):
        for seed in range(3):
            P.simulate(part, seed=seed)


def _digest(part):
    h = hashlib.sha256()
    h.update(part.owner.tobytes())
    ptr, rec = part.records(emulate=False)
    h.update(ptr.tobytes())
    h.update(rec.tobytes())
    h.update(part.edges.tobytes())
    return h.hexdigest()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    prog, bt = _prog("s2", "accu")
    part = P.Partition(prog, bt, world)
    out = [None] * world
    dist.all_gather_object(out, (_digest(part), int((part.owner == rank).sum()),
                                 sorted({int(r["dst"]) for r in part.records(False)[1]
                                         if part.owner[0] >= 0})))
    if rank == 0:
        q.put((out, part.n_tasks))
    dist.barrier()
    dist.destroy_process_group()


def test_two_ranks_derive_the_same_partition():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out, nt = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert out[0][0] == out[1][0]
    assert out[0][1] + out[1][1] == nt


# ----------------------------------------------------------------------
# DistributedHLU host protocol (gloo, world 2): the device calls are
# recorded; what is checked is what every rank hands to hmx_plan_peer and
# the order reset -> barrier -> launch(4) -> status.
# ----------------------------------------------------------------------
class _FakePlan:
    def __init__(self, rank, log):
        self.rank, self.log = rank, log
        self.state = (0x1000 * (rank + 1) + 0x100000, 0x2000 * (rank + 1) + 0x200000,
                      0x3000 * (rank + 1) + 0x300000)

    def sched_state(self):
        return self.state

    def peer(self, r, bases, rbases, indeg, queue, qctl):
        self.log.append(("peer", r, tuple(bases), tuple(rbases), indeg, queue, qctl))

    def bind(self, *a):
        self.log.append(("bind", a[0]))

    def reset(self, stream=None):
        self.log.append(("reset",))

    def reset_counters(self, stream=None):
        self.log.append(("reset_counters",))

    def execute(self, mode, stream=None):
        self.log.append(("execute", mode))

    def status(self, stream=None):
        self.log.append(("status",))
        return 0


class _FakeBackend:
    """An 'IPC handle' names (rank, 4 KiB page); opening it maps the page at
    (1 << 44) * (rank + 1) + page, so a peer address is recomputable."""
    rank = 0
    log = None

    @classmethod
    def ipc_handle(cls, ptr):
        page = ptr & ~0xfff
        return (cls.rank.to_bytes(8, "little") + page.to_bytes(8, "little")).ljust(64, b"\0"), ptr & 0xfff

    @classmethod
    def ipc_open(cls, handle):
        r, page = int.from_bytes(handle[:8], "little"), int.from_bytes(handle[8:16], "little")
        cls.log.append(("open", r, page))
        return ((1 << 44) * (r + 1)) + page

    @classmethod
    def ipc_close(cls, base):
        cls.log.append(("close", base))

    @classmethod
    def synchronize(cls):
        cls.log.append(("sync",))


def _mapped(r, ptr):
    return 0 if not ptr else ((1 << 44) * (r + 1)) + ptr


def _dworker(rank, world, port, q):
    import torch

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    prog, bt = _prog("s2", "accu")
    log = []
    _FakeBackend.rank, _FakeBackend.log = rank, log

    class PP:  # what DistributedHLU uses of a PartitionedPlan
        part = P.Partition(prog, bt, world)
        plan = _FakePlan(rank, log)
        table, layout = bt, prog.layout
        acc_values = torch.zeros(16, dtype=torch.float64)
        acc_ranks = torch.zeros(4, dtype=torch.int32)
        ws_values = torch.zeros(0, dtype=torch.float64)  # empty pool: exported as None
        ws_ranks = torch.zeros(4, dtype=torch.int32)

        @classmethod
        def bind(cls, A, L, U):
            log.append(("bind_stores",))

        @classmethod
        def check(cls, stream=None):
            cls.plan.status()

    class S:
        def __init__(self):
            self.values = torch.zeros(32, dtype=torch.float64)
            self.ranks = torch.zeros(8, dtype=torch.int32)

    A, L, U = S(), S(), S()
    d = P.DistributedHLU(bt, "accu", None, 64, backend=_FakeBackend, plan=PP)
    d.connect(A, L, U)
    ptrs = d._pointers(A, L, U)
    d.run()
    owned = [len(d.owned_leaves(b)) for b in (1, 2)]
    d.close()
    allp = [None] * world
    dist.all_gather_object(allp, ptrs)
    if rank == 0:
        q.put((log, allp, owned, int(bt.leaf.sum())))
    out = [None] * world
    dist.all_gather_object(out, owned)
    if rank == 0:
        q.put(out)
    dist.barrier()
    dist.destroy_process_group()


def test_distributed_runner_host_protocol_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_dworker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    log, allp, owned0, nleaves = q.get(timeout=300)
    owned = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    # rank 0 mapped rank 1's pools and scheduler state, and only those
    peers = [e for e in log if e[0] == "peer"]
    assert [e[1] for e in peers] == [1]
    _, r, bases, rbases, indeg, queue, qctl = peers[0]
    p1 = allp[1]
    for b in P.DistributedHLU.BASES:
        assert bases[b] == _mapped(1, p1[f"v{b}"])
        assert rbases[b] == _mapped(1, p1[f"r{b}"])
    assert bases[P.WS_BASE_ID] == 0  # the empty pool travels as a null address
    assert (indeg, queue, qctl) == tuple(_mapped(1, p1[k]) for k in ("indeg", "queue", "qctl"))
    # every 4 KiB page is opened once even when several pools share it
    opens = [e for e in log if e[0] == "open"]
    assert len(opens) == len(set(opens))
    # run(): the scheduler is reset and the device idle before the barrier, the launch
    # does not reset again (mode 4), the status is read after it
    names = [e[0] for e in log]
    i_reset, i_sync, i_exec, i_stat = (names.index("reset"), names.index("sync"),
                                        names.index("execute"), names.index("status"))
    assert i_reset < i_sync < i_exec < i_stat
    assert log[i_exec] == ("execute", 4)
    # the final versions of the factors' leaves are spread over the ranks without overlap
    assert owned[0][0] + owned[1][0] == nleaves and owned[0][1] + owned[1][1] == nleaves
    assert min(owned[0] + owned[1]) > 0
