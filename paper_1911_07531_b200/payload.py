"""Product payloads and leaf folds (drop-in for hmatrix.py:349-448).

A payload is the reference's tuple: ("dense", D) or ("lowrank", U, V) with
row-major numpy arrays (hmatrix.py:349-364).  These are the standalone
building blocks of the reference's recursive arithmetic; inside hlu /
hlu_accu the same operations are fused into the lowered device program
(planner.py, csrc/hmx_lower.cpp), so these entry points serve callers that
compose the arithmetic themselves (and the accumulator primitives of
accumulator.py).  Every product, truncation, compression and fold runs on
the device: H x dense products through the device apply plans
(hmatrix.hm_apply / hm_apply_t), dense products through hmx_gemm_batched,
truncations through hmx_truncate_batched and hmx_dense_to_lowrank_batched,
and folds into a leaf update the leaf's device storage in place.
"""

from __future__ import annotations

import numpy as np

from .hmatrix import BLOCKED, DENSE, LOWRANK, HMatrix, TruncationPolicy, counters, hm_apply, hm_apply_t


def _torch():
    import torch

    if not torch.cuda.is_available():
        raise RuntimeError("payload arithmetic needs a CUDA device (no CPU fallback)")
    return torch


def payload_dense(p) -> np.ndarray:
    """Dense form of a payload (hmatrix.py:349-352); low-rank expanded on
    the device."""
    if p[0] == DENSE:
        return p[1]
    U, V = np.asarray(p[1], float), np.asarray(p[2], float)
    if U.shape[1] == 0:
        return np.zeros((U.shape[0], V.shape[0]))
    from . import kernels

    return kernels.gemm(1.0, [U], [V], transB=True)[0]


def payload_shape(p):
    if p[0] == DENSE:
        return p[1].shape
    return p[1].shape[0], p[2].shape[0]


def payload_restrict(p, r0, nr, c0, nc):
    """Sub-block of a payload (views, hmatrix.py:361-364)."""
    if p[0] == DENSE:
        return (DENSE, p[1][r0:r0 + nr, c0:c0 + nc])
    return (LOWRANK, p[1][r0:r0 + nr], p[2][c0:c0 + nc])


def _dense_product(alpha, A, B):
    from . import kernels

    return kernels.gemm(alpha, [np.asarray(A, float)], [np.asarray(B, float)])[0]


def _truncate(U, V, policy):
    from .hmatrix import truncate

    return truncate(U, V, policy)


def product_payload(alpha: float, A: HMatrix, B: HMatrix, policy: TruncationPolicy):
    """alpha * A @ B as a dense or low-rank payload (hmatrix.py:367-417):
    the same case analysis, quadrant stacking order and single truncation
    per blocked x blocked product as the reference."""
    if A.ncols != B.nrows:
        raise ValueError("non-conformal product")
    if A.kind == LOWRANK:
        return (LOWRANK, alpha * A.U, hm_apply_t(B, A.V))
    if B.kind == LOWRANK:
        return (LOWRANK, hm_apply(A, alpha * B.U), B.V)
    if A.kind == DENSE and B.kind == DENSE:
        return (DENSE, _dense_product(alpha, A.D, B.D))
    if A.kind == DENSE:
        return (DENSE, hm_apply_t(B, alpha * A.D.T).T)
    if B.kind == DENSE:
        return (DENSE, hm_apply(A, alpha * B.D))
    m, n = A.nrows, B.ncols
    us, vs = [], []
    dense_acc = None
    Ach, Bch = A.children, B.children
    for i in range(2):
        for j in range(2):
            for l in range(2):
                a, b = Ach[i][l], Bch[l][j]
                q = product_payload(alpha, a, b, policy)
                r0, _ = A.child_offsets(a)
                _, c0 = B.child_offsets(b)
                if q[0] == DENSE:
                    if dense_acc is None:
                        dense_acc = np.zeros((m, n))
                    dense_acc[r0:r0 + q[1].shape[0], c0:c0 + q[1].shape[1]] += q[1]
                elif q[1].shape[1]:
                    ue = np.zeros((m, q[1].shape[1]))
                    ue[r0:r0 + q[1].shape[0]] = q[1]
                    ve = np.zeros((n, q[2].shape[1]))
                    ve[c0:c0 + q[2].shape[0]] = q[2]
                    us.append(ue)
                    vs.append(ve)
    if dense_acc is not None:
        if us:
            from . import kernels

            dense_acc = kernels.gemm(1.0, [np.hstack(us)], [np.hstack(vs)], Cs=[dense_acc],
                                     transB=True, beta=1.0)[0]
        return (DENSE, dense_acc)
    if not us:
        return (LOWRANK, np.zeros((m, 0)), np.zeros((n, 0)))
    U, V = _truncate(np.hstack(us), np.hstack(vs), policy)
    return (LOWRANK, U, V)


def fold_payload_into_leaf(C: HMatrix, p, policy: TruncationPolicy):
    """C += payload for a dense or low-rank leaf (hmatrix.py:420-437): dense
    leaves are updated in their device storage; low-rank leaves are
    replaced by the device truncation of the stacked factors, or by the
    device compression of the dense sum for a dense payload."""
    pm, pn = payload_shape(p)
    if (pm, pn) != (C.nrows, C.ncols):
        raise ValueError("payload does not match destination block")
    if C.kind == BLOCKED:
        raise ValueError("fold target must be a leaf")
    counters.add(0, 1)
    if C.kind == DENSE:
        torch = _torch()
        st, u = C.store, C.uid
        lay = st.layout
        o = int(lay.d_off[u])
        add = torch.from_numpy(np.ascontiguousarray(np.asarray(payload_dense(p), float).T).ravel())
        st.values[o:o + pm * pn] += add.cuda()
        return
    from .hmatrix import dense_to_lowrank

    if p[0] == DENSE:
        M = payload_dense((LOWRANK, C.U, C.V)) + np.asarray(p[1], float)
        U, V = dense_to_lowrank(M, policy)
    else:
        U, V = _truncate(np.hstack([C.U, np.asarray(p[1], float)]),
                         np.hstack([C.V, np.asarray(p[2], float)]), policy)
    C.set_lowrank(U, V)


def scatter_payload(C: HMatrix, p, policy: TruncationPolicy):
    """Add a payload into C, descending into blocked destinations
    (hmatrix.py:440-448)."""
    if C.kind != BLOCKED:
        fold_payload_into_leaf(C, p, policy)
        return
    for row in C.children:
        for ch in row:
            r0, c0 = C.child_offsets(ch)
            scatter_payload(ch, payload_restrict(p, r0, ch.nrows, c0, ch.ncols), policy)
