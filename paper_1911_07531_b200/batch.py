"""Batches of independent same-structure H-LUs (config 4) and their
sharding across GPUs.

Config 4 is 256 independent 1D HODLR instances (n=4096, leaf 64, weak
admissibility).  Their block trees are index-identical (cardinality
bisection of sorted points; admissibility depends only on index ranges),
so ONE lowered plan serves all of them: the op program and the task graph
are replicated as a disjoint union (planner.replicate) and a whole shard
is factored by one persistent-scheduler launch.  Across GPUs the instances
shard contiguously with no data-path collective (one process per GPU,
torch.distributed only for the barrier and the max-over-ranks timing).
"""

from __future__ import annotations

import numpy as np

from . import configs, hmatrix as H
from .engine import EXEC_PERSISTENT, ExecPlan, HStore


def shard(n_items: int, world: int, rank: int) -> range:
    """Contiguous balanced shard of range(n_items) for `rank` of `world`."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    base, extra = divmod(n_items, world)
    start = rank * base + min(rank, extra)
    return range(start, start + base + (1 if rank < extra else 0))


def structure_key(table) -> tuple:
    """Index structure of a block table (equal keys => one plan fits)."""
    return (table.n, table.r0.tobytes(), table.r1.tobytes(), table.c0.tobytes(),
            table.c1.tobytes(), table.adm.tobytes(), table.leaf.tobytes())


class InstanceBatch:
    """A shard of config-4 instances assembled on the device, one plan."""

    def __init__(self, ids, rank_cap=64, mode="std"):
        self.ids = list(ids)
        if not self.ids:
            raise ValueError("empty batch")
        cfgs = [configs.config(f"c4_{j}") for j in self.ids]
        self.cfgs = cfgs
        pol = H.TruncationPolicy.fixed_accuracy(cfgs[0].eps)
        self.policy = pol
        mats = []
        key = None
        for cfg in cfgs:
            geom, root, perm, broot = configs.structure(cfg)
            A = H.assemble(broot, configs.kernel(cfg, perm), pol, rank_cap=rank_cap)
            k = structure_key(A.table)
            if key is None:
                key, self.table, self.broot = k, A.table, broot
            elif k != key:
                raise ValueError("instances do not share one block structure")
            mats.append(A)
        self.plan = ExecPlan(self.table, mode, pol, rank_cap, nrep=len(self.ids))
        lay = self.plan.layout
        self.A0 = HStore.batch(lay, len(self.ids))
        for b, A in enumerate(mats):
            self.A0.instance(b).copy_from(A.store)
        self.A = HStore.batch(lay, len(self.ids))
        self.L = HStore.batch(lay, len(self.ids))
        self.U = HStore.batch(lay, len(self.ids))

    def factor(self, exec_mode=EXEC_PERSISTENT, check=True):
        self.A.copy_from(self.A0)
        self.plan.run(self.A, self.L, self.U, exec_mode, check=check)

    def ranks(self):
        """Per-instance L/U rank arrays (host)."""
        nb = self.table.n
        rl = self.L.ranks.cpu().numpy().reshape(len(self.ids), nb)
        ru = self.U.ranks.cpu().numpy().reshape(len(self.ids), nb)
        return rl, ru


def summary(rl, ru):
    """Small per-instance digest used for cross-rank gathering."""
    return np.stack([rl.sum(axis=1), ru.sum(axis=1), (rl >= 0).sum(axis=1)], axis=1).astype(np.int64)
