"""Multi-rank host logic of the sharded batch path on CPU (gloo, world 2).

Config 4 shards its 256 instances contiguously across ranks with no
data-path collective; the only cross-rank traffic is the barrier, the
max-over-ranks time and an optional gather of per-instance digests.  This
exercises exactly that plumbing on two CPU processes.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1911_07531_b200.batch import shard


def test_shard_partition():
    for n in (0, 1, 7, 256):
        for world in (1, 2, 3, 4, 8):
            got = [list(shard(n, world, r)) for r in range(world)]
            flat = [x for g in got for x in g]
            assert flat == list(range(n))
            sizes = [len(g) for g in got]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        shard(4, 2, 2)


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
    ids = list(shard(256, world, rank))
    # per-instance digest a GPU rank would produce; here a deterministic stand-in
    dig = torch.tensor([[j, 2 * j, 3] for j in ids], dtype=torch.int64)
    sizes = [torch.zeros(1, dtype=torch.int64) for _ in range(world)]
    dist.all_gather(sizes, torch.tensor([len(ids)]))
    mx = max(int(s.item()) for s in sizes)
    pad = torch.zeros(mx, 3, dtype=torch.int64)
    pad[:len(ids)] = dig
    out = [torch.zeros(mx, 3, dtype=torch.int64) for _ in range(world)]
    dist.all_gather(out, pad)
    t = torch.tensor([float(rank + 1)])
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    if rank == 0:
        rows = torch.cat([o[:int(s.item())] for o, s in zip(out, sizes)]).numpy()
        q.put((rows, float(t.item())))
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_world2_gather_and_max():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    rows, tmax = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert rows.shape == (256, 3)
    assert np.array_equal(rows[:, 0], np.arange(256))
    assert tmax == 2.0
