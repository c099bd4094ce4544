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


class PipelinedHLU:
    """Stream of batches factored host -> device -> host (packed format).

    A caller with a sequence of batches (each: packed A + rank words in
    pinned host memory, hmatrix.pack_leaves) gets packed L and U back per
    batch.  Two device buffer sets alternate, so the H2D copy of batch i+1,
    the factorization of batch i and the D2H copy of batch i-1 overlap on
    three streams (h2d, compute, d2h); a buffer set is reused only after
    its previous results reached the host.  Every batch still moves its own
    inputs and results across PCIe: steady-state throughput of the
    host-facing call, as a serving loop would run it.
    """

    def __init__(self, block, policy, nrep, rank_cap, mode, exec_mode=EXEC_PERSISTENT):
        import torch

        from .arith import get_plan

        self.mode, self.policy, self.exec_mode = mode, policy, exec_mode
        self.sets = [(H.HBatch(block, policy, nrep, rank_cap), H.HBatch(block, policy, nrep, rank_cap),
                      H.HBatch(block, policy, nrep, rank_cap)) for _ in range(2)]
        self.plan = get_plan(self.sets[0][0].table, mode, policy, rank_cap, nrep=nrep)
        self.s_h2d, self.s_comp, self.s_d2h = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()
        n_items = self.sets[0][0].store._pack_desc().shape[0] * nrep + 1
        self.offs = [[torch.empty(n_items, dtype=torch.int64, device="cuda") for _ in range(2)]
                     for _ in range(2)]
        self.size_host = [torch.zeros(2, dtype=torch.int64, pin_memory=True) for _ in range(2)]
        self.ev_in = [torch.cuda.Event() for _ in range(2)]
        self.ev_done = [torch.cuda.Event() for _ in range(2)]
        self.ev_size = [torch.cuda.Event() for _ in range(2)]
        self.ev_out = [None, None]

    def _submit(self, i, packed, ranks):
        import torch

        b = i & 1
        A, L, U = self.sets[b]
        if A._xfer_buf().numel() < packed.numel():  # first use: size the staging buffer
            torch.cuda.synchronize()
            A._xfer_buf(packed.numel())
        buf = A._xfer_buf()
        with torch.cuda.stream(self.s_h2d):
            if self.ev_out[b] is not None:  # A's staging buffer is free once batch i-2 ran
                self.s_h2d.wait_event(self.ev_done[b])
            A.store.ranks.copy_(ranks, non_blocking=True)
            buf[:packed.numel()].copy_(packed, non_blocking=True)
            self.ev_in[b].record(self.s_h2d)
        with torch.cuda.stream(self.s_comp):
            self.s_comp.wait_event(self.ev_in[b])
            if self.ev_out[b] is not None:  # L/U packed buffers of batch i-2 reached the host
                self.s_comp.wait_event(self.ev_out[b])
            A.store.unpack_from(buf, stream=self.s_comp)
            self.plan.run(A.store, L.store, U.store, self.exec_mode, self.s_comp, check=False)
            for k, M in enumerate((L, U)):
                M.store.pack_to(M._xfer_buf(), self.offs[b][k], stream=self.s_comp)
            self.ev_done[b].record(self.s_comp)
        with torch.cuda.stream(self.s_d2h):
            self.s_d2h.wait_event(self.ev_done[b])
            for k in range(2):
                self.size_host[b][k:k + 1].copy_(self.offs[b][k][-1:], non_blocking=True)
            self.ev_size[b].record(self.s_d2h)

    def _collect(self, i, out):
        import torch

        b = i & 1
        _, L, U = self.sets[b]
        self.ev_size[b].synchronize()
        res = []
        with torch.cuda.stream(self.s_d2h):
            for k, M in enumerate((L, U)):
                n = int(self.size_host[b][k])
                if n > M._xfer_buf().numel():  # packed form outgrew the buffer: grow, pack again
                    torch.cuda.synchronize()
                    M._xfer_buf(n)
                    M.store.pack_to(M._xfer_buf(), self.offs[b][k], stream=self.s_d2h)
                hv, hr = out[k] if out is not None else (None, None)
                if hv is None or hv.numel() < n:
                    hv = torch.empty(n, dtype=torch.float64, pin_memory=True)
                if hr is None:
                    hr = torch.empty(M.store.ranks.numel(), dtype=torch.int32, pin_memory=True)
                hv[:n].copy_(M._xfer_buf()[:n], non_blocking=True)
                hr.copy_(M.store.ranks, non_blocking=True)
                res.append((hv[:n], hr))
            ev = torch.cuda.Event()
            ev.record(self.s_d2h)
            self.ev_out[b] = ev
        return res

    def run(self, inputs, outputs=None):
        """inputs: list of (packed, ranks) pinned host tensors; returns per
        batch [(L packed, L ranks), (U packed, U ranks)] (pinned; valid after
        torch.cuda.synchronize() or the returned event)."""
        import torch

        res = [None] * len(inputs)
        for i in range(len(inputs) + 1):
            if i < len(inputs):
                self._submit(i, *inputs[i])
            if i >= 1:
                res[i - 1] = self._collect(i - 1, outputs[i - 1] if outputs else None)
        done = torch.cuda.Event()
        done.record(self.s_d2h)
        return res, done

    def check(self):
        self.plan.check()
