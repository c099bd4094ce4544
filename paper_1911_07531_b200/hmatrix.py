"""H-matrix storage, rank control and assembly (drop-in for hmatdag.hmatrix).

An :class:`HMatrix` is a *view* of one block of a device-resident H-matrix
(:class:`~.engine.HStore`): leaves live in a pooled fp64 HBM tensor
(column-major dense leaves, U/V factor arenas with capacity ``rank_cap``)
and ranks in an int32 device array.  The reference API is kept — ``kind``,
``children``, ``D``/``U``/``V`` (host copies), ``rank``, ``to_dense``,
``frobenius``, ``copy``, ``leaves``, ``set_lowrank``, ``child_offsets``
(hmatrix.py:141-224) — but the arithmetic runs on the GPU through the
planner/executor (arith.py, accumulator.py).

Assembly (hmatrix.py:227-248) evaluates kernel blocks on the device
(hmx_exp_kernel_blocks for the exponential point kernels of the BASELINE
configs) and compresses admissible blocks: blocks with min(m, n) <= 128 by
the device Jacobi SVD (the same op as dense_to_lowrank inside H-LU);
larger blocks by a randomized range finder with power iteration on cuBLAS /
cuSOLVER through torch, whose sample size grows until the trailing
singular value of the sketch sits three decades below the cut — so ranks
agree with LAPACK's dgesdd (tests/test_hlu_gpu.py checks the c1/c2 ranks
against the reference fixtures).
"""

from __future__ import annotations

import numpy as np

from . import _lib
from .trees import Block, BlockTable

ZERO_CUTOFF = 1e-14
DENSE = "dense"
LOWRANK = "lowrank"
BLOCKED = "blocked"
DEFAULT_RANK_CAP = 128


class TruncationPolicy:
    """Exact, FixedRank(k) or FixedAccuracy(eps) (hmatrix.py:36-78)."""

    __slots__ = ("mode", "k", "eps")

    def __init__(self, mode, k=None, eps=None):
        self.mode = mode
        self.k = k
        self.eps = eps

    @classmethod
    def exact(cls):
        return cls("exact")

    @classmethod
    def fixed_rank(cls, k: int):
        if k < 0:
            raise ValueError("rank must be >= 0")
        return cls("rank", k=k)

    @classmethod
    def fixed_accuracy(cls, eps: float):
        if eps <= 0:
            raise ValueError("accuracy must be positive")
        return cls("accuracy", eps=eps)

    def keep(self, sigma: np.ndarray) -> int:
        if sigma.size == 0 or sigma[0] <= 0.0:
            return 0
        if self.mode == "rank":
            r = min(self.k, sigma.size)
            return int(np.count_nonzero(sigma[:r] > ZERO_CUTOFF * sigma[0]))
        cut = self.eps if self.mode == "accuracy" else ZERO_CUTOFF
        return int(np.count_nonzero(sigma > cut * sigma[0]))

    def __repr__(self):
        if self.mode == "rank":
            return f"FixedRank({self.k})"
        if self.mode == "accuracy":
            return f"FixedAccuracy({self.eps})"
        return "Exact"


EXACT = TruncationPolicy.exact()


class OpCounters:
    """Truncation / update counters (hmatrix.py:84-110), fed by the device."""

    def __init__(self):
        self.truncations = 0
        self.updates = 0

    def reset(self):
        self.truncations = 0
        self.updates = 0

    def snapshot(self):
        return self.truncations, self.updates

    def add(self, truncations, updates):
        self.truncations += int(truncations)
        self.updates += int(updates)


counters = OpCounters()

_TABLES = {}


def table_of(block: Block) -> BlockTable:
    """Cached BlockTable of the block tree rooted at ``block`` (its root)."""
    root = block
    while root.parent is not None:
        root = root.parent
    t = _TABLES.get(id(root))
    if t is None or t.root is not root:
        t = BlockTable(root)
        _TABLES[id(root)] = t
    return t


class HMatrix:
    """View of block ``uid`` of a device-resident H-matrix."""

    __slots__ = ("store", "uid", "policy")

    def __init__(self, store, uid=0, policy=EXACT):
        self.store = store
        self.uid = int(uid)
        self.policy = policy

    # structure ---------------------------------------------------------
    @property
    def table(self) -> BlockTable:
        return self.store.table

    @property
    def block(self) -> Block:
        return self.table.blocks[self.uid]

    @property
    def kind(self):
        t = self.table
        if not t.leaf[self.uid]:
            return BLOCKED
        return LOWRANK if t.adm[self.uid] else DENSE

    @property
    def nrows(self):
        return int(self.table.m[self.uid])

    @property
    def ncols(self):
        return int(self.table.nc[self.uid])

    @property
    def children(self):
        if self.kind != BLOCKED:
            return None
        k = self.table.kids[self.uid]
        return [[HMatrix(self.store, k[0], self.policy), HMatrix(self.store, k[1], self.policy)],
                [HMatrix(self.store, k[2], self.policy), HMatrix(self.store, k[3], self.policy)]]

    def child_offsets(self, child):
        t = self.table
        return int(t.r0[child.uid] - t.r0[self.uid]), int(t.c0[child.uid] - t.c0[self.uid])

    def leaves(self):
        for u in self.table.leaves(self.uid):
            yield HMatrix(self.store, u, self.policy)

    # leaf data (host copies) -------------------------------------------
    def _leaf(self):
        return self.store.download_leaf(self.uid)

    @property
    def D(self):
        return self._leaf()[1] if self.kind == DENSE else None

    @D.setter
    def D(self, value):
        if self.kind != DENSE:
            raise ValueError("D is defined for dense leaves only")
        self.store.upload_leaf(self.uid, ("D", np.asarray(value, dtype=float)))

    @property
    def U(self):
        return self._leaf()[1] if self.kind == LOWRANK else None

    @property
    def V(self):
        return self._leaf()[2] if self.kind == LOWRANK else None

    @property
    def rank(self) -> int:
        if self.kind != LOWRANK:
            raise ValueError("rank defined for low-rank leaves only")
        return int(self.store.ranks[self.uid].item())

    def set_lowrank(self, U, V):
        if U.shape[0] != self.nrows or V.shape[0] != self.ncols or U.shape[1] != V.shape[1]:
            raise ValueError("factor shape mismatch")
        self.store.upload_leaf(self.uid, ("R", np.asarray(U, float), np.asarray(V, float)))

    # whole-matrix helpers ---------------------------------------------
    def to_leaves(self):
        allv = self.store.download_leaves()
        return {u: allv[u] for u in self.table.leaves(self.uid)}

    def to_dense(self) -> np.ndarray:
        t = self.table
        out = np.zeros((self.nrows, self.ncols))
        for u, x in self.to_leaves().items():
            blk = x[1] if x[0] == "D" else x[1] @ x[2].T
            out[t.r0[u] - t.r0[self.uid]:t.r1[u] - t.r0[self.uid],
                t.c0[u] - t.c0[self.uid]:t.c1[u] - t.c0[self.uid]] = blk
        return out

    def frobenius(self) -> float:
        s = 0.0
        for x in self.to_leaves().values():
            if x[0] == "D":
                s += float(np.sum(x[1] * x[1]))
            else:
                s += max(0.0, float(((x[1].T @ x[1]) * (x[2].T @ x[2])).sum()))
        return float(np.sqrt(s))

    def copy(self) -> "HMatrix":
        if self.uid != 0:
            raise ValueError("copy() is supported on the root view")
        return HMatrix(self.store.clone(), 0, self.policy)

    def __repr__(self):
        return f"HMatrix({self.block!r}, {self.kind})"


def _store_cls():
    from .engine import HStore

    return HStore


def _layout(table, rank_cap, caps=None):
    from .planner import Layout

    return Layout(table, rank_cap, caps)


def zeros(block: Block, policy: TruncationPolicy = EXACT, rank_cap=DEFAULT_RANK_CAP,
          caps=None) -> HMatrix:
    """Zero H-matrix over a block tree (rank-0 admissible leaves, hmatrix.py:251-263).
    ``caps``: optional per-uid bound of the low-rank arenas (rank-bounded
    storage, assembly.rank_caps)."""
    t = table_of(block)
    return HMatrix(_store_cls()(_layout(t, rank_cap, caps)), block.uid, policy)


def from_leaves(block: Block, leaves, policy=EXACT, rank_cap=DEFAULT_RANK_CAP) -> HMatrix:
    """Upload host leaves (uid -> ("D", M) | ("R", U, V)) into device storage."""
    H = zeros(block, policy, rank_cap)
    H.store.upload_leaves(leaves)
    return H


def assemble(block: Block, kernel, policy: TruncationPolicy, rank_cap=DEFAULT_RANK_CAP) -> HMatrix:
    """Evaluate ``kernel`` over the block tree on the device (hmatrix.py:227-248)."""
    from .assembly import assemble_store

    t = table_of(block)
    store = _store_cls()(_layout(t, rank_cap))
    assemble_store(store, kernel, policy)
    return HMatrix(store, block.uid, policy)


def assemble_bounded(block: Block, kernel, policy: TruncationPolicy, rank_cap=DEFAULT_RANK_CAP,
                     mult=2.5, floor=24, budget=None):
    """Rank-first assembly for large problems (config 5): leaves are
    compressed chunk by chunk into the packed form, every low-rank arena is
    then sized from the assembled rank (assembly.rank_caps) and A is
    unpacked into that storage.  Returns (A, caps); factors of A must be
    allocated with the same caps (``zeros(block, policy, rank_cap, caps)``)."""
    from .assembly import DEFAULT_BUDGET, assemble_packed, rank_caps

    t = table_of(block)
    packed, ranks = assemble_packed(t, kernel, policy, rank_cap, budget or DEFAULT_BUDGET)
    caps = rank_caps(t, ranks.cpu().numpy(), rank_cap, mult, floor)
    store = _store_cls()(_layout(t, rank_cap, caps))
    store.ranks.copy_(ranks)
    store.unpack_from(packed)
    del packed
    return HMatrix(store, block.uid, policy), caps


def rel_error(A, B) -> float:
    A = A.to_dense() if isinstance(A, HMatrix) else np.asarray(A, dtype=float)
    B = B.to_dense() if isinstance(B, HMatrix) else np.asarray(B, dtype=float)
    num = np.linalg.norm(A - B)
    den = np.linalg.norm(A)
    if den == 0.0:
        return 0.0 if num == 0.0 else float("inf")
    return float(num / den)


def frobenius(M) -> float:
    return M.frobenius() if isinstance(M, HMatrix) else float(np.linalg.norm(M))


def dense_to_lowrank(M, policy):
    """Device dense_to_lowrank of one block (hmatrix.py:133-138)."""
    from . import kernels

    counters.add(1, 0)
    return kernels.dense_to_lowrank(M, policy)


def truncate(U, V, policy):
    """Device truncate of one factor pair (hmatrix.py:113-130)."""
    from . import kernels

    if U.shape[1] != V.shape[1]:
        raise ValueError("non-conformal low-rank factors")
    if U.shape[1] == 0:
        return U, V
    counters.add(1, 0)
    return kernels.truncate(U, V, policy)


__all__ = ["TruncationPolicy", "EXACT", "HMatrix", "assemble", "zeros", "from_leaves",
           "rel_error", "frobenius", "truncate", "dense_to_lowrank", "counters", "DENSE",
           "LOWRANK", "BLOCKED", "_lib"]


class HBatch:
    """R same-structure H-matrices in one contiguous device pool.

    Factorizations of a batch run as ONE device launch over the disjoint
    union of R copies of the lowered program (planner.replicate): the
    single-matrix critical path leaves most SMs idle, a batch fills them.
    """

    def __init__(self, block: Block, policy=EXACT, nrep=1, rank_cap=DEFAULT_RANK_CAP, store=None):
        from .engine import HStore

        self.block = block
        self.policy = policy
        self.nrep = int(nrep)
        t = table_of(block)
        self.store = store if store is not None else HStore.batch(_layout(t, rank_cap), self.nrep)

    @property
    def table(self):
        return self.store.table

    def member(self, b: int) -> HMatrix:
        return HMatrix(self.store.instance(b), self.block.uid, self.policy)

    @classmethod
    def replicate(cls, A: HMatrix, nrep: int) -> "HBatch":
        """nrep copies of A (e.g. independent factorizations of one matrix)."""
        out = cls(A.block, A.policy, nrep, A.store.layout.rank_cap)
        for b in range(nrep):
            out.store.instance(b).copy_from(A.store)
        return out

    def copy(self) -> "HBatch":
        return HBatch(self.block, self.policy, self.nrep, store=self.store.clone())

    # packed host transfers (wire / dump format, csrc/hmx_transfer.cu) ------
    def _xfer_buf(self, n=0):
        """Device staging buffer of the packed form, grown to >= n doubles."""
        import torch

        b = getattr(self, "_xbuf", None)
        if b is None or b.numel() < n:
            self._xbuf = None
            b = self._xbuf = torch.empty(max(int(n), 1), dtype=torch.float64, device="cuda")
        return b

    def upload_packed(self, packed, ranks, stream=None):
        """Load every member from the packed form: ``packed`` the live leaf
        data (pack_leaves format, host pinned or device) and ``ranks`` the
        int32 rank words (nrep x n_blocks).  One H2D copy of each plus one
        device scatter; nothing of the pools' unused rank capacity moves."""
        st = self.store
        if ranks.numel() != st.ranks.numel():
            raise ValueError("rank words do not match the batch")
        if packed.numel() > st.values.numel():
            raise ValueError("packed data larger than the batch pools")
        buf = self._xfer_buf(packed.numel())
        st.ranks.copy_(ranks, non_blocking=True)
        buf[:packed.numel()].copy_(packed, non_blocking=True)
        st.unpack_from(buf, stream=stream)

    def download_packed(self, out=None, out_ranks=None, stream=None):
        """(packed live data, rank words) of every member on the host (pinned
        tensors; pass preallocated ones to reuse them)."""
        import torch

        st = self.store
        buf = self._xfer_buf()
        offs = st.pack_to(buf, stream=stream)
        total = int(offs[-1].item())
        if total > buf.numel():  # grow and pack again
            buf = self._xfer_buf(total)
            offs = st.pack_to(buf, offs, stream=stream)
        if out is None or out.numel() < total:
            out = torch.empty(total, dtype=torch.float64, pin_memory=True)
        if out_ranks is None:
            out_ranks = torch.empty(st.ranks.numel(), dtype=torch.int32, pin_memory=True)
        out[:total].copy_(buf[:total], non_blocking=True)
        out_ranks.copy_(st.ranks, non_blocking=True)
        return out[:total], out_ranks


def pack_leaves(table: BlockTable, leaves_list, nblocks=None):
    """Host form of the packed format for a list of members' leaves
    (uid -> ("D", M) | ("R", U, V), row-major numpy, as download_leaves
    returns): (packed float64 array, int32 rank words nrep x n_blocks)."""
    n = table.n
    parts, ranks = [], []
    for leaves in leaves_list:
        r = np.full(n, -1, dtype=np.int32)
        for u in table.leaves(0):
            x = leaves[u]
            if x[0] == "D":
                parts.append(np.asarray(x[1], dtype=np.float64).T.ravel())
            else:
                r[u] = x[1].shape[1]
                parts.append(np.asarray(x[1], dtype=np.float64).T.ravel())
                parts.append(np.asarray(x[2], dtype=np.float64).T.ravel())
        r[table.leaf & table.adm & (r < 0)] = 0
        ranks.append(r)
    data = np.concatenate(parts) if parts else np.zeros(0)
    return data, np.concatenate(ranks)


def unpack_leaves(table: BlockTable, packed, ranks, nrep=1):
    """Inverse of pack_leaves: list of nrep leaf dicts."""
    packed = np.asarray(packed)
    ranks = np.asarray(ranks).reshape(nrep, table.n)
    out, o = [], 0
    for b in range(nrep):
        lv = {}
        for u in table.leaves(0):
            m, nc = int(table.m[u]), int(table.nc[u])
            if table.adm[u]:
                k = int(ranks[b, u])
                U = packed[o:o + m * k].reshape(k, m).T.copy()
                o += m * k
                V = packed[o:o + nc * k].reshape(k, nc).T.copy()
                o += nc * k
                lv[u] = ("R", U, V)
            else:
                lv[u] = ("D", packed[o:o + m * nc].reshape(nc, m).T.copy())
                o += m * nc
        out.append(lv)
    if o != packed.size:
        raise ValueError("packed data does not match the rank words")
    return out


# ---------------------------------------------------------------------------
# H x dense products and triangular solves (hmatrix.py:286-341) on the device
# ---------------------------------------------------------------------------
_DENSE_PLANS = None


def _dense_plan(M: HMatrix, op, cols):
    global _DENSE_PLANS
    from .arith import _PlanCache
    from .engine import DensePlan

    if _DENSE_PLANS is None:
        _DENSE_PLANS = _PlanCache(16)
    t = M.table
    lay = M.store.layout
    key = (t, op, M.uid, int(cols), lay.rank_cap, int(lay.size), id(lay.caps) if lay.caps is not None else 0)
    return _DENSE_PLANS.get(key, lambda: DensePlan(t, op, M.uid, cols, lay.rank_cap, lay))


def _dense_run(M: HMatrix, op, X, out_rows):
    """Run op with X (numpy or torch, rows x cols); returns the same kind."""
    import torch

    is_np = not isinstance(X, torch.Tensor)
    Xt = torch.as_tensor(np.asarray(X, dtype=np.float64)) if is_np else X.to(torch.float64)
    vec = Xt.dim() == 1
    if vec:
        Xt = Xt[:, None]
    cols = int(Xt.shape[1])
    # column-major device copy (the ops' layout)
    Xd = Xt.t().contiguous().cuda()
    if cols == 0:
        res = torch.zeros(out_rows, 0, dtype=torch.float64)
    else:
        p = _dense_plan(M, op, cols)
        if op in ("apply", "apply_t"):
            out = torch.empty(out_rows * cols, dtype=torch.float64, device="cuda")
            p.run(M.store, Xd.view(-1), out)
            res = out.view(cols, out_rows).t()
        else:
            p.run(M.store, Xd.view(-1))
            res = Xd.view(cols, out_rows).t()
    if vec:
        res = res[:, 0]
    if is_np:
        return res.cpu().numpy().copy()
    return res.to(X.device) if X.device.type != "cuda" else res


def hm_apply(M: HMatrix, X):
    """M @ X for a dense X (hmatrix.py:286-299), computed on the device."""
    if M.ncols != X.shape[0]:
        raise ValueError("dimension mismatch in apply")
    return _dense_run(M, "apply", X, M.nrows)


def hm_apply_t(M: HMatrix, X):
    """M.T @ X for a dense X (hmatrix.py:302-315)."""
    if M.nrows != X.shape[0]:
        raise ValueError("dimension mismatch in transposed apply")
    return _dense_run(M, "apply_t", X, M.ncols)


def hm_solve_lower(L: HMatrix, Y):
    """Solve L X = Y, L unit lower triangular, dense Y (hmatrix.py:318-328)."""
    if L.kind == LOWRANK:
        raise ValueError("triangular solve on a low-rank diagonal block")
    if L.nrows != L.ncols or L.nrows != Y.shape[0]:
        raise ValueError("dimension mismatch in triangular solve")
    return _dense_run(L, "solve_lower", Y, L.nrows)


def hm_solve_upper_t(U: HMatrix, Y):
    """Solve U.T W = Y, U upper triangular, dense Y (hmatrix.py:331-341)."""
    if U.kind == LOWRANK:
        raise ValueError("triangular solve on a low-rank diagonal block")
    if U.nrows != U.ncols or U.nrows != Y.shape[0]:
        raise ValueError("dimension mismatch in triangular solve")
    return _dense_run(U, "solve_upper_t", Y, U.nrows)


def hm_solve_upper(U: HMatrix, Y):
    """Solve U X = Y, U upper triangular (non-unit), dense Y: block back
    substitution, the non-transposed counterpart of hm_solve_upper_t
    (hmatrix.py:331-341).  Solve phase with the factors;
    the reference has no such entry point."""
    if U.kind == LOWRANK:
        raise ValueError("triangular solve on a low-rank diagonal block")
    if U.nrows != U.ncols or U.nrows != Y.shape[0]:
        raise ValueError("dimension mismatch in triangular solve")
    return _dense_run(U, "solve_upper", Y, U.nrows)


def lu_solve(L: HMatrix, U: HMatrix, B):
    """X with L U X = B (A X ~ B after hlu / hlu_accu): forward substitution
    with the unit-lower L, then back substitution with U, both on the
    device over the H-matrix factors (cluster ordering: B and X are in the
    permuted index order of the block tree, like A)."""
    if L.table is not U.table or L.uid != U.uid:
        raise ValueError("L and U are not over the same block")
    return hm_solve_upper(U, hm_solve_lower(L, B))


def lu_residual(A: HMatrix, L: HMatrix, U: HMatrix, X):
    """||A X - L (U X)||_F / ||A X||_F on the device (probe residual)."""
    AX = hm_apply(A, X)
    LUX = hm_apply(L, hm_apply(U, X))
    return float(np.linalg.norm(np.asarray(AX) - np.asarray(LUX)) / np.linalg.norm(np.asarray(AX)))


_LEAF_UPD = {}


def leaf_update(C: HMatrix, alpha: float, A: HMatrix, B: HMatrix, policy: TruncationPolicy):
    """C += alpha * A @ B where C is a leaf, A and B of any kind
    (hmatrix.py:451-460: product_payload then fold_payload_into_leaf), as a
    one-task device program; A, B, C may live in different H-matrices over
    the same block tree."""
    from .engine import OpPlan

    if alpha == 0.0:
        return
    if A.nrows != C.nrows or B.ncols != C.ncols or A.ncols != B.nrows:
        raise ValueError("non-conformal leaf update")
    if C.kind == BLOCKED:
        raise ValueError("leaf_update needs a leaf C")
    t = C.table
    if A.table is not t or B.table is not t:
        raise ValueError("operands over different block trees")
    if C.store is A.store or C.store is B.store:
        raise ValueError("the output may not alias an input")
    rc = C.store.layout.rank_cap
    key = (id(t), A.uid, B.uid, C.uid, float(alpha), repr(policy), rc)
    p = _LEAF_UPD.get(key)
    if p is None or p.table is not t:
        p = _LEAF_UPD[key] = OpPlan(t, "leaf_update", policy, rc, alpha=alpha,
                                    uids=(A.uid, B.uid, C.uid))
    p.run(A.store, B.store, C.store)
    c = p.counters()
    counters.add(c["truncations"], c["updates"])


def __getattr__(name):
    """Payload helpers of the reference's hmatrix module (hmatrix.py:349-448)
    live in payload.py (device arithmetic); resolved lazily to avoid an
    import cycle."""
    if name in ("product_payload", "fold_payload_into_leaf", "scatter_payload", "payload_dense",
                "payload_shape", "payload_restrict"):
        from . import payload

        return getattr(payload, name)
    raise AttributeError(name)
