"""Parity checks of device factors against the reference's fixtures.

Shared by the GPU tests and bench.py (which refuses to print a throughput
for factors that fail them).  Fixtures (tests/golden, made by running the
unmodified reference, tests/golden/make_golden.py):

  <cfg>.npz          per-block ranks and Frobenius norms of the reference's
                     L and U (``<mode>_L_rank``, ``<mode>_L_fro``, ...)
  <cfg>_leaves.npz   entries of a seeded sample of leaves of L and U
                     (dense D, low-rank U and V)

Per-block factor comparison: dense leaves by ||D_dev - D_ref||_F / ||D_ref||_F,
low-rank leaves by ||U_dev V_dev^T - U_ref V_ref^T||_F / ||U_ref V_ref^T||_F
(computed from Gram matrices, the block is never formed); the factor of a
low-rank leaf is only defined up to the product.
"""

from __future__ import annotations

import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _lr_diff_rel(U1, V1, U2, V2, floor=0.0):
    """||U1 V1^T - U2 V2^T||_F / max(||U2 V2^T||_F, floor) via Gram matrices."""
    U = np.hstack([U1, -U2])
    V = np.hstack([V1, V2])
    d2 = float(np.sum((U.T @ U) * (V.T @ V)))
    r = max(np.sqrt(max(float(np.sum((U2.T @ U2) * (V2.T @ V2))), 0.0)), floor)
    return np.sqrt(max(d2, 0.0)) / r if r > 0 else np.sqrt(max(d2, 0.0))


def leaf_samples(name):
    p = os.path.join(GOLDEN, f"{name}_leaves.npz")
    return dict(np.load(p)) if os.path.exists(p) else None


def compare_leaf_samples(samples, mode, get_leaf, totals=None):
    """Max per-block difference over the sampled leaves of L and U,
    relative to max(||block||, SIGNIFICANT * ||factor||) (``totals``:
    which -> factor norm; without it, relative to the block).

    ``get_leaf(which, uid)`` returns the device leaf as ("D", M) or
    ("R", U, V) numpy arrays (which = "L" | "U")."""
    worst = 0.0
    totals = totals or {}
    nblk = 0
    for which in ("L", "U"):
        meta = samples.get(f"{mode}_{which}_meta")
        vals = samples.get(f"{mode}_{which}_vals")
        if meta is None:
            continue
        off = 0
        for uid, kind, m, n, k in meta.tolist():
            if kind == 0:
                ref = vals[off:off + m * n].reshape(n, m).T
                off += m * n
                x = get_leaf(which, uid)
                if x[0] != "D":
                    return float("inf"), nblk
                nr = max(float(np.linalg.norm(ref)), SIGNIFICANT * totals.get(which, 0.0))
                worst = max(worst, float(np.linalg.norm(x[1] - ref) / (nr if nr > 0 else 1.0)))
            else:
                Ur = vals[off:off + m * k].reshape(k, m).T
                off += m * k
                Vr = vals[off:off + n * k].reshape(k, n).T
                off += n * k
                x = get_leaf(which, uid)
                if x[0] != "R":
                    return float("inf"), nblk
                worst = max(worst, _lr_diff_rel(x[1], x[2], Ur, Vr, SIGNIFICANT * totals.get(which, 0.0)))
            nblk += 1
    return worst, nblk


def compare_ranks(arr, mode, L_ranks, U_ranks):
    """Number of L / U blocks whose rank differs from the reference's."""
    bad = 0
    for which, got in (("L", L_ranks), ("U", U_ranks)):
        ref = arr[f"{mode}_{which}_rank"]
        sel = ref >= 0
        bad += int((np.asarray(got)[sel] != ref[sel]).sum())
    return bad


def store_fro(layout, values, ranks):
    """Frobenius norm of every leaf of a device store (host copies of the
    pool ``values`` and ``ranks``): dense leaves by a segmented sum of
    squares, low-rank leaves from U^T U and V^T V."""
    t = layout.table
    fro = np.full(t.n, np.nan)
    leaves = np.flatnonzero(t.leaf)
    dense = leaves[~t.adm[leaves]]
    if len(dense):
        off = layout.d_off[dense]
        sz = (t.m[dense] * t.nc[dense]).astype(np.int64)
        sq = values * values
        cs = np.concatenate([[0.0], np.cumsum(sq)])
        fro[dense] = np.sqrt(cs[off + sz] - cs[off])
    for u in leaves[t.adm[leaves]].tolist():
        k = int(ranks[u])
        m, n = int(t.m[u]), int(t.nc[u])
        if k <= 0:
            fro[u] = 0.0
            continue
        U = values[layout.u_off[u]:layout.u_off[u] + m * k].reshape(k, m)
        V = values[layout.v_off[u]:layout.v_off[u] + n * k].reshape(k, n)
        fro[u] = np.sqrt(max(float(np.sum((U @ U.T) * (V @ V.T))), 0.0))
    return fro


SIGNIFICANT = 1e-4  # blocks carrying at least this share of the factor's norm


def factor_norm(arr, mode, which):
    ref = arr[f"{mode}_{which}_fro"]
    return float(np.sqrt(np.nansum(ref[np.isfinite(ref)] ** 2)))


def compare_fro(arr, mode, which, fro):
    """Per-block Frobenius norms vs the reference's: (max relative
    difference over the blocks that carry >= SIGNIFICANT of the factor's
    norm, max absolute difference over all blocks / the factor's norm).

    Both are held to 10*eps.  Blocks of tiny norm are judged absolutely:
    the fixture's A differs from the device's by the compression rounding of
    each admissible block (~1e-10 relative, a different randomized range
    finder above 128, make_golden.py), and that absolute difference is a
    large relative one on blocks whose norm is 1e-5 of the factor's
    (tools/parity_diag.py)."""
    ref = arr[f"{mode}_{which}_fro"]
    sel = np.isfinite(ref) & np.isfinite(fro) & (ref > 0)
    if not sel.any():
        return 0.0, 0.0
    tot = factor_norm(arr, mode, which)
    d = np.abs(fro[sel] - ref[sel])
    big = ref[sel] >= SIGNIFICANT * tot
    rel = float(np.max(d[big] / ref[sel][big])) if big.any() else 0.0
    return rel, float(np.max(d) / tot)
