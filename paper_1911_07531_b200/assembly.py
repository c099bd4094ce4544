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

Admissible blocks are evaluated densely before compression, so they are
processed in chunks whose dense staging stays below ``budget`` doubles
(config 5's admissible blocks hold ~536 GB densely).

``assemble_packed`` is the rank-first form for problems whose arenas must be
sized from the ranks (config 5): leaves are evaluated and compressed chunk
by chunk in block pre-order and kept only in the packed format (live data at
the actual ranks, hmx_pack_leaves), so the caller can size every low-rank
arena from the assembled ranks before allocating the H-matrix.
"""

from __future__ import annotations

import numpy as np

from . import _lib
from ._lib import OP_D2LR

SMALL = 128
TMP_BASE = 4
DEFAULT_BUDGET = 1 << 30  # doubles of dense staging per chunk (8 GB)


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


class _Eval:
    """Evaluates kernel blocks (uid -> column-major block at an offset)."""

    def __init__(self, table, kernel):
        torch = _torch()
        self.t = table
        self.kernel = kernel
        spec = kernel.device_spec() if hasattr(kernel, "device_spec") else None
        self.spec = spec
        if spec is not None:
            pts, perm, ell, diag, scale = spec
            self.pts = torch.from_numpy(np.ascontiguousarray(pts, dtype=np.float64)).cuda()
            perm = np.arange(pts.shape[0]) if perm is None else perm
            self.perm = torch.from_numpy(np.asarray(perm, dtype=np.int64)).cuda()
            self.dim = pts.shape[1]
            self.ell, self.diag, self.scale = float(ell), float(diag), float(scale)

    def __call__(self, dst, items, offs):
        if not items:
            return
        torch = _torch()
        t = self.t
        if self.spec is not None:
            desc = np.array([[t.r0[u], t.m[u], t.c0[u], t.nc[u], offs[i]] for i, u in enumerate(items)],
                            dtype=np.int64)
            d = torch.from_numpy(desc.ravel()).cuda()
            for s in range(0, len(items), 60000):
                n_b = min(60000, len(items) - s)
                _lib.check(_lib.lib().hmx_exp_kernel_blocks(
                    n_b, _lib.ptr(d[5 * s:]), _lib.ptr(self.pts), self.dim, _lib.ptr(self.perm),
                    self.ell, self.diag, self.scale, _lib.ptr(dst), _lib.stream_ptr()), "exp kernel")
            return
        for i, u in enumerate(items):
            M = np.asarray(self.kernel.dense(np.arange(t.r0[u], t.r1[u]), np.arange(t.c0[u], t.c1[u])),
                           dtype=np.float64)
            o = int(offs[i])
            dst[o:o + M.size].copy_(torch.from_numpy(np.ascontiguousarray(M.T).ravel()))


def _chunks(table, items, budget):
    """Consecutive runs of ``items`` whose dense m*n sum stays <= budget."""
    out, cur, size = [], [], 0
    for u in items:
        sz = int(table.m[u] * table.nc[u])
        if cur and size + sz > budget:
            out.append(cur)
            cur, size = [], 0
        cur.append(u)
        size += sz
    if cur:
        out.append(cur)
    return out


def assemble_store(store, kernel, policy, budget=DEFAULT_BUDGET):
    """Fill ``store`` (its layout fixes the arenas): dense leaves evaluated in
    place, admissible leaves evaluated and compressed chunk by chunk."""
    torch = _torch()
    from .hmatrix import counters

    t, lay = store.table, store.layout
    leaves = t.leaves(0)
    adm = [u for u in leaves if t.adm[u]]
    dense = [u for u in leaves if not t.adm[u]]
    ev = _Eval(t, kernel)
    ev(store.values, dense, [int(lay.d_off[u]) for u in dense])
    ranks = store.ranks.cpu().numpy()
    for chunk in _chunks(t, adm, budget):
        offs = np.concatenate([[0], np.cumsum([int(t.m[u] * t.nc[u]) for u in chunk])])
        tmp = torch.empty(max(int(offs[-1]), 1), dtype=torch.float64, device="cuda")
        ev(tmp, chunk, offs[:-1])
        tmp_off = {u: int(offs[i]) for i, u in enumerate(chunk)}
        _compress(store.values, store.ranks, ranks, lay.u_off, lay.v_off, lay.cap, tmp, tmp_off, chunk,
                  policy, t)
        del tmp
    counters.add(len(adm), 0)
    torch.cuda.synchronize()


def _compress(values, ranks_d, ranks_h, u_off, v_off, cap, tmp, tmp_off, items, policy, t):
    small = [u for u in items if min(t.m[u], t.nc[u]) <= SMALL]
    large = [u for u in items if min(t.m[u], t.nc[u]) > SMALL]
    if small:
        _compress_small(values, ranks_d, u_off, v_off, cap, tmp, tmp_off, small, policy, t)
        ranks_h[small] = ranks_d[small].cpu().numpy()
    if large:
        _compress_large(values, ranks_d, ranks_h, u_off, v_off, cap, tmp, tmp_off, large, policy, t)


def _compress_small(values, ranks_d, u_off, v_off, cap, tmp, tmp_off, items, policy, t):
    mode, kfix, eps = _policy_fields(policy)
    ops = np.zeros(len(items), dtype=_lib.OP_DTYPE)
    ws = 0
    for i, u in enumerate(items):
        m, n = int(t.m[u]), int(t.nc[u])
        l = max(m, n)
        ws = max(ws, _lib.d2lr_scratch(m, n))
        o = ops[i]
        o["code"] = OP_D2LR
        o["dim"][:2] = (m, n)
        o["ref"][0] = _lib.mref(TMP_BASE, tmp_off[u])
        o["ld"][0] = m
        o["ref"][2] = _lib.mref(0, u_off[u])
        o["ld"][2] = m
        o["ref"][3] = _lib.mref(0, v_off[u])
        o["ld"][3] = n
        o["slot"][0] = _lib.slot(0, u)
        o["iarg"][:3] = (mode, kfix, int(cap[u]))
        o["farg"][1] = eps
        o["wref"] = _lib.mref(_lib.SCRATCH_BASE, 0)
    nt = len(items)
    plan = _lib.Plan(ops, np.arange(nt + 1), np.zeros(nt + 1, np.int32), np.zeros(0, np.int32),
                     np.array([0, nt], np.int32), np.arange(nt, dtype=np.int32), ws, 1)
    plan.bind(0, values, ranks_d)
    plan.bind(TMP_BASE, tmp, None)
    plan.execute(0)
    st = plan.status()
    plan.close()
    if st:
        raise _lib.HmxError(st, "assembly compression")


def _compress_large(values, ranks_d, ranks_h, u_off, v_off, cap, tmp, tmp_off, items, policy, t):
    torch = _torch()
    mode = getattr(policy, "mode", "exact")
    cut = policy.eps if mode == "accuracy" else 1e-14
    groups = {}
    for u in items:
        groups.setdefault((int(t.m[u]), int(t.nc[u])), []).append(u)
    gen = torch.Generator(device="cuda")
    gen.manual_seed(12345)
    for (m, n), us in sorted(groups.items()):
        smin = min(m, n)
        nb = max(1, min(64, (1 << 28) // max(m * n, 1)))
        for b0 in range(0, len(us), nb):
            grp = us[b0:b0 + nb]
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
                if k > cap[u]:
                    raise _lib.HmxError(_lib.HMX_ERR_RANK_OVERFLOW, f"assembly of block {u}")
                uo, vo = int(u_off[u]), int(v_off[u])
                values[uo:uo + m * k].copy_(Uall[i, :, :k].t().reshape(-1))
                values[vo:vo + n * k].copy_(Vall[i, :, :k].t().reshape(-1))
                ranks_h[u] = k
            del M, G, Q, Bm, W, S, Zt, Uall, Vall
    ranks_d.copy_(torch.from_numpy(ranks_h))


def assemble_packed(table, kernel, policy, rank_cap=None, budget=DEFAULT_BUDGET):
    """Rank-first assembly: returns (packed, ranks) — the live leaf data in
    hmx_pack_leaves order (block pre-order; dense m*n, or U then V at the
    actual rank; device float64) and the int32 rank word of every uid (-1
    for dense and structured blocks).  Peak device memory: the packed data
    plus one chunk of ``budget`` dense doubles and its factor staging."""
    torch = _torch()
    from .hmatrix import counters

    t = table
    nb = t.n
    leaves = t.leaves(0)
    ranks_h = np.full(nb, -1, dtype=np.int32)
    ranks_h[t.leaf & t.adm] = 0
    ranks_d = torch.from_numpy(ranks_h).cuda()
    ev = _Eval(t, kernel)
    segs, total = [], 0
    nadm = 0
    for chunk in _chunks(t, leaves, budget):
        # chunk pool: dense leaves m*n; admissible leaves U (m x c) and V (n x c)
        off, desc, tmp_off, u_off, v_off, cap = 0, [], {}, {}, {}, {}
        adm, dense, doffs = [], [], []
        toff = 0
        for u in chunk:
            m, n = int(t.m[u]), int(t.nc[u])
            if t.adm[u]:
                c = min(m, n) if not rank_cap else min(m, n, int(rank_cap))
                cap[u], u_off[u], v_off[u] = c, off, off + m * c
                desc.append((u, off, off + m * c, m, n))
                off += (m + n) * c
                tmp_off[u] = toff
                toff += m * n
                adm.append(u)
            else:
                desc.append((u, off, -1, m, n))
                dense.append(u)
                doffs.append(off)
                off += m * n
        pool = torch.empty(max(off, 1), dtype=torch.float64, device="cuda")
        ev(pool, dense, doffs)
        if adm:
            tmp = torch.empty(max(toff, 1), dtype=torch.float64, device="cuda")
            ev(tmp, adm, [tmp_off[u] for u in adm])
            _compress(pool, ranks_d, ranks_h, u_off, v_off, cap, tmp, tmp_off, adm, policy, t)
            del tmp
            nadm += len(adm)
        d = torch.from_numpy(np.asarray(desc, dtype=np.int64).ravel()).cuda()
        offs = torch.empty(len(chunk) + 1, dtype=torch.int64, device="cuda")
        L = _lib.lib()
        _lib.check(L.hmx_pack_leaves(len(chunk), 1, _lib.ptr(d), off, nb, None, _lib.ptr(ranks_d),
                                     None, 0, _lib.ptr(offs), _lib.stream_ptr()), "pack")
        size = int(offs[-1].item())
        seg = torch.empty(max(size, 1), dtype=torch.float64, device="cuda")
        _lib.check(L.hmx_pack_leaves(len(chunk), 1, _lib.ptr(d), off, nb, _lib.ptr(pool),
                                     _lib.ptr(ranks_d), _lib.ptr(seg), size, _lib.ptr(offs),
                                     _lib.stream_ptr()), "pack")
        segs.append((seg, size))
        total += size
        del pool
    packed = torch.empty(max(total, 1), dtype=torch.float64, device="cuda")
    pos = 0
    while segs:
        seg, size = segs.pop(0)
        packed[pos:pos + size].copy_(seg[:size])
        pos += size
        del seg
    counters.add(nadm, 0)
    torch.cuda.synchronize()
    return packed, ranks_d


def rank_caps(table, ranks, rank_cap=None, mult=2.5, floor=24):
    """Capacity bound of every low-rank leaf from its assembled rank: the
    L / U ranks of a block exceed A's (c2: A <= 12, L/U <= 23) but stay
    within a small multiple of it; a run that exceeds a bound reports
    HMX_ERR_RANK_OVERFLOW and is repeated with larger bounds."""
    t = table
    r = np.asarray(ranks, dtype=np.int64)
    caps = np.full(t.n, -1, dtype=np.int32)
    sel = t.leaf & t.adm
    c = np.maximum(floor, np.ceil(mult * np.maximum(r, 0))).astype(np.int64)
    c = np.minimum(c, np.minimum(t.m, t.nc))
    if rank_cap:
        c = np.minimum(c, int(rank_cap))
    caps[sel] = c[sel]
    return caps
