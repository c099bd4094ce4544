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
