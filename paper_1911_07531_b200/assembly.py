"""Device assembly of an H-matrix (hmatrix.assemble, hmatrix.py:227-248).

1. Kernel evaluation: every leaf block is evaluated on the GPU
   (hmx_exp_kernel_blocks) when the kernel has a device description
   (problems.ExpKernel composed with permuted), else on the host through
   ``kernel.dense`` and uploaded.  Dense leaves are evaluated in place.
2. Compression of admissible leaves (dense_to_lowrank, hmatrix.py:133-138,
   rank = #{sigma_i > eps*sigma_1}):
   * min(m, n) <= SMALL: the device one-sided Jacobi SVD (OP_D2LR), one
     CTA per block, the op used by H-LU itself;
   * larger blocks: randomized range finder with one power iteration
     (torch / cuBLAS / cuSOLVER), sample size doubled until the sketch's
     trailing singular value is < 1e-3 of the cut, then an SVD of the
     projected block.  This is setup work outside the timed H-LU
     (SURVEY.md §8f row 1 lists a native large-block compressor as next).
"""

from __future__ import annotations

import numpy as np

from . import _lib
from ._lib import OP_D2LR

SMALL = 128
TMP_BASE = 4


def _torch():
    import torch

    return torch


def _policy_fields(policy):
    from .planner import _policy_fields as f

    return f(policy)


def _keep_counts(S, policy):
    """TruncationPolicy.keep over a batch of descending spectra (torch)."""
    torch = _torch()
    s1 = S[:, :1]
    mode = getattr(policy, "mode", "exact")
    if mode == "rank":
        lim = min(int(policy.k), S.shape[1])
        r = (S[:, :lim] > 1e-14 * s1).sum(dim=1)
    else:
        cut = policy.eps if mode == "accuracy" else 1e-14
        r = (S > cut * s1).sum(dim=1)
    return torch.where(s1[:, 0] > 0, r, torch.zeros_like(r))


def assemble_store(store, kernel, policy):
    torch = _torch()
    from .hmatrix import counters

    t, lay = store.table, store.layout
    leaves = t.leaves(0)
    adm = [u for u in leaves if t.adm[u]]
    dense = [u for u in leaves if not t.adm[u]]
    # temporary buffer for admissible blocks (column-major, per block)
    tmp_off = {}
    cur = 0
    for u in adm:
        tmp_off[u] = cur
        cur += int(t.m[u] * t.nc[u])
    tmp = torch.empty(max(cur, 1), dtype=torch.float64, device="cuda")

    spec = kernel.device_spec() if hasattr(kernel, "device_spec") else None
    if spec is not None:
        pts, perm, ell, diag, scale = spec
        pts_d = torch.from_numpy(np.ascontiguousarray(pts, dtype=np.float64)).cuda()
        perm = np.arange(pts.shape[0]) if perm is None else perm
        perm_d = torch.from_numpy(np.asarray(perm, dtype=np.int64)).cuda()
        for dst, items, offs in ((store.values, dense, lay.d_off), (tmp, adm, tmp_off)):
            if not items:
                continue
            desc = np.array([[t.r0[u], t.m[u], t.c0[u], t.nc[u], offs[u]] for u in items],
                            dtype=np.int64)
            d = torch.from_numpy(desc.ravel()).cuda()
            for s in range(0, len(items), 60000):
                n_b = min(60000, len(items) - s)
                _lib.check(_lib.lib().hmx_exp_kernel_blocks(
                    n_b, _lib.ptr(d[5 * s:]), _lib.ptr(pts_d), pts.shape[1], _lib.ptr(perm_d),
                    float(ell), float(diag), float(scale), _lib.ptr(dst), _lib.stream_ptr()),
                    "exp kernel")
    else:
        hv = np.zeros(lay.size)
        ht = np.zeros(max(cur, 1))
        for u in leaves:
            M = np.asarray(kernel.dense(np.arange(t.r0[u], t.r1[u]), np.arange(t.c0[u], t.c1[u])),
                           dtype=np.float64)
            if t.adm[u]:
                ht[tmp_off[u]:tmp_off[u] + M.size] = M.T.ravel()
            else:
                hv[lay.d_off[u]:lay.d_off[u] + M.size] = M.T.ravel()
        store.values.copy_(torch.from_numpy(hv))
        tmp.copy_(torch.from_numpy(ht))

    small = [u for u in adm if min(t.m[u], t.nc[u]) <= SMALL]
    large = [u for u in adm if min(t.m[u], t.nc[u]) > SMALL]
    if small:
        _compress_small(store, tmp, tmp_off, small, policy)
    if large:
        _compress_large(store, tmp, tmp_off, large, policy)
    counters.add(len(adm), 0)
    torch.cuda.synchronize()


def _compress_small(store, tmp, tmp_off, items, policy):
    t, lay = store.table, store.layout
    mode, kfix, eps = _policy_fields(policy)
    ops = np.zeros(len(items), dtype=_lib.OP_DTYPE)
    ws = 0
    for i, u in enumerate(items):
        m, n = int(t.m[u]), int(t.nc[u])
        l = max(m, n)
        ws = max(ws, 8 * l + 2 * l * l)
        o = ops[i]
        o["code"] = OP_D2LR
        o["dim"][:2] = (m, n)
        o["ref"][0] = _lib.mref(TMP_BASE, tmp_off[u])
        o["ld"][0] = m
        o["ref"][2] = _lib.mref(0, lay.u_off[u])
        o["ld"][2] = m
        o["ref"][3] = _lib.mref(0, lay.v_off[u])
        o["ld"][3] = n
        o["slot"][0] = _lib.slot(0, u)
        o["iarg"][:3] = (mode, kfix, int(lay.cap[u]))
        o["farg"][1] = eps
        o["wref"] = _lib.mref(_lib.SCRATCH_BASE, 0)
    nt = len(items)
    plan = _lib.Plan(ops, np.arange(nt + 1), np.zeros(nt + 1, np.int32), np.zeros(0, np.int32),
                     np.array([0, nt], np.int32), np.arange(nt, dtype=np.int32), ws, 1)
    plan.bind(0, store.values, store.ranks)
    plan.bind(TMP_BASE, tmp, None)
    plan.execute(0)
    st = plan.status()
    plan.close()
    if st:
        raise _lib.HmxError(st, "assembly compression")


def _compress_large(store, tmp, tmp_off, items, policy):
    torch = _torch()
    t, lay = store.table, store.layout
    mode = getattr(policy, "mode", "exact")
    cut = policy.eps if mode == "accuracy" else 1e-14
    groups = {}
    for u in items:
        groups.setdefault((int(t.m[u]), int(t.nc[u])), []).append(u)
    gen = torch.Generator(device="cuda")
    gen.manual_seed(12345)
    ranks = store.ranks.cpu().numpy()
    for (m, n), us in sorted(groups.items()):
        smin = min(m, n)
        for b0 in range(0, len(us), 64):
            grp = us[b0:b0 + 64]
            M = torch.stack([tmp[tmp_off[u]:tmp_off[u] + m * n].view(n, m).t() for u in grp])
            s = min(smin, 48)
            while True:
                G = torch.randn(len(grp), n, s, dtype=torch.float64, device="cuda", generator=gen)
                Q, _ = torch.linalg.qr(M @ G)
                Q, _ = torch.linalg.qr(M @ (M.transpose(1, 2) @ Q))
                Bm = Q.transpose(1, 2) @ M
                W, S, Zt = torch.linalg.svd(Bm, full_matrices=False)
                ok = bool((S[:, -1] <= 1e-3 * cut * S[:, 0]).all()) or s >= smin
                if ok:
                    break
                s = min(smin, 2 * s)
            r = _keep_counts(S, policy)
            rmax = int(r.max().item()) if len(grp) else 0
            Uall = Q @ (W[:, :, :rmax] * S[:, None, :rmax])
            Vall = Zt[:, :rmax, :].transpose(1, 2)
            rh = r.cpu().numpy()
            for i, u in enumerate(grp):
                k = int(rh[i])
                if k > lay.cap[u]:
                    raise _lib.HmxError(_lib.HMX_ERR_RANK_OVERFLOW, f"assembly of block {u}")
                uo, vo = int(lay.u_off[u]), int(lay.v_off[u])
                store.values[uo:uo + m * k].copy_(Uall[i, :, :k].t().reshape(-1))
                store.values[vo:vo + n * k].copy_(Vall[i, :, :k].t().reshape(-1))
                ranks[u] = k
    store.ranks.copy_(torch.from_numpy(ranks))
