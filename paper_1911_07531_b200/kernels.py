"""Batched leaf kernels on the device (thin host wrappers over include/hmx.h).

Each function takes host numpy arrays in the reference's row-major
convention, moves them to the GPU in the engine's column-major layout,
runs the sm_100a kernel and returns numpy results.  They mirror the leaf
calls of the reference:

  getrf_nopiv        arith.dense_lu                      (arith.py:58-73)
  trsm_lower_unit    solve_triangular(lower, unit)       (hmatrix.py:321)
  trsm_upper_trans   solve_triangular(trans="T")         (hmatrix.py:334)
  trsm_upper         solve_triangular(lower=False)       (solve phase, back substitution)
  gemm               the `@` products                    (hmatrix.py)
  truncate           hmatrix.truncate                    (hmatrix.py:113-130)
  dense_to_lowrank   hmatrix.dense_to_lowrank            (hmatrix.py:133-138)
  svd_values         np.linalg.svd(..., compute_uv=False) singular values
"""

from __future__ import annotations

import numpy as np

from . import _lib
from ._lib import check, lib, ptr, stream_ptr


def _torch():
    import torch

    if not torch.cuda.is_available():
        raise RuntimeError("hmx kernels need a CUDA device (no CPU fallback)")
    return torch


def _colmajor_batch(arrs):
    """list of 2-D row-major arrays (same shape) -> device tensor (b, n, m)
    whose memory is each matrix column-major."""
    torch = _torch()
    a = np.ascontiguousarray(np.stack([np.asarray(x, dtype=np.float64).T for x in arrs]))
    return torch.from_numpy(a).cuda()


def _from_colmajor(t, m, n, cols=None):
    """device (b, ncap, m) column-major buffers -> list of (m, n) row-major."""
    h = t.cpu().numpy()
    return [np.ascontiguousarray(h[b, :n, :m].T) for b in range(h.shape[0])]


def _policy(policy):
    if policy is None:
        return _lib.POLICY_EXACT, 0, 0.0
    mode = getattr(policy, "mode", "exact")
    if mode == "rank":
        return _lib.POLICY_RANK, int(policy.k), 0.0
    if mode == "accuracy":
        return _lib.POLICY_ACCURACY, 0, float(policy.eps)
    return _lib.POLICY_EXACT, 0, 0.0


def getrf_nopiv(As):
    torch = _torch()
    As = [np.asarray(a, dtype=np.float64) for a in As]
    b, n = len(As), As[0].shape[0]
    dA = _colmajor_batch(As)
    dL = torch.zeros_like(dA)
    dU = torch.zeros_like(dA)
    info = torch.zeros(b, dtype=torch.int32, device="cuda")
    check(lib().hmx_getrf_nopiv_batched(b, n, ptr(dA), n, n * n, ptr(dL), ptr(dU), n * n,
                                        ptr(info), stream_ptr()), "getrf")
    torch.cuda.synchronize()
    return _from_colmajor(dL, n, n), _from_colmajor(dU, n, n), info.cpu().numpy()


def _trsm(fn, Ts, Bs):
    Ts = [np.asarray(t, dtype=np.float64) for t in Ts]
    Bs = [np.asarray(x, dtype=np.float64) for x in Bs]
    b, n, c = len(Ts), Ts[0].shape[0], Bs[0].shape[1]
    dT = _colmajor_batch(Ts)
    dB = _colmajor_batch(Bs)
    check(fn(b, n, c, ptr(dT), n, n * n, ptr(dB), n, n * c, stream_ptr()), "trsm")
    _torch().cuda.synchronize()
    return _from_colmajor(dB, n, c)


def trsm_lower_unit(Ls, Bs):
    return _trsm(lib().hmx_trsm_lower_unit_batched, Ls, Bs)


def trsm_upper_trans(Us, Bs):
    return _trsm(lib().hmx_trsm_upper_trans_batched, Us, Bs)


def trsm_upper(Us, Bs):
    return _trsm(lib().hmx_trsm_upper_batched, Us, Bs)


def gemm(alpha, As, Bs, Cs=None, transA=False, transB=False, beta=0.0):
    torch = _torch()
    As = [np.asarray(a, dtype=np.float64) for a in As]
    Bs = [np.asarray(x, dtype=np.float64) for x in Bs]
    b = len(As)
    ma, ka = As[0].shape
    kb, nb = Bs[0].shape
    m, k = (ka, ma) if transA else (ma, ka)
    n = kb if transB else nb
    dA, dB = _colmajor_batch(As), _colmajor_batch(Bs)
    if Cs is None:
        dC = torch.zeros((b, n, m), dtype=torch.float64, device="cuda")
    else:
        dC = _colmajor_batch(Cs)
    check(lib().hmx_gemm_batched(b, m, n, k, float(alpha), ptr(dA), ma, ma * ka, int(transA),
                                 ptr(dB), kb, kb * nb, int(transB), float(beta), ptr(dC), m, m * n,
                                 stream_ptr()), "gemm")
    torch.cuda.synchronize()
    return _from_colmajor(dC, m, n)


def truncate(U, V, policy, cap=None):
    """Device truncate of one factor pair; returns (U', V') like the reference."""
    torch = _torch()
    U = np.asarray(U, dtype=np.float64)
    V = np.asarray(V, dtype=np.float64)
    m, K = U.shape
    n = V.shape[0]
    cap = int(cap if cap is not None else min(m, n, max(K, 1)))
    dU, dV = _colmajor_batch([U]), _colmajor_batch([V])
    dUo = torch.zeros((1, max(cap, 1), m), dtype=torch.float64, device="cuda")
    dVo = torch.zeros((1, max(cap, 1), n), dtype=torch.float64, device="cuda")
    rk = torch.zeros(1, dtype=torch.int32, device="cuda")
    mode, kf, eps = _policy(policy)
    check(lib().hmx_truncate_batched(1, m, n, K, ptr(dU), ptr(dV), m * K, n * K, mode, kf, eps, cap,
                                     ptr(dUo), ptr(dVo), m * max(cap, 1), n * max(cap, 1),
                                     ptr(rk), stream_ptr()), "truncate")
    torch.cuda.synchronize()
    r = int(rk.item())
    if K == 0:
        return U, V
    return _from_colmajor(dUo, m, r)[0], _from_colmajor(dVo, n, r)[0]


def dense_to_lowrank(M, policy, cap=None):
    torch = _torch()
    M = np.asarray(M, dtype=np.float64)
    m, n = M.shape
    cap = int(cap if cap is not None else min(m, n))
    dM = _colmajor_batch([M])
    dUo = torch.zeros((1, cap, m), dtype=torch.float64, device="cuda")
    dVo = torch.zeros((1, cap, n), dtype=torch.float64, device="cuda")
    rk = torch.zeros(1, dtype=torch.int32, device="cuda")
    mode, kf, eps = _policy(policy)
    check(lib().hmx_dense_to_lowrank_batched(1, m, n, ptr(dM), m * n, mode, kf, eps, cap, ptr(dUo),
                                             ptr(dVo), m * cap, n * cap, ptr(rk), stream_ptr()),
          "dense_to_lowrank")
    torch.cuda.synchronize()
    r = int(rk.item())
    return _from_colmajor(dUo, m, r)[0], _from_colmajor(dVo, n, r)[0]


def svd_values(Gs):
    torch = _torch()
    Gs = [np.asarray(g, dtype=np.float64) for g in Gs]
    b, (p, q) = len(Gs), Gs[0].shape
    s = min(p, q)
    dG = _colmajor_batch(Gs)
    dS = torch.zeros((b, s), dtype=torch.float64, device="cuda")
    check(lib().hmx_svd_values_batched(b, p, q, ptr(dG), p * q, ptr(dS), s, stream_ptr()),
          "svd_values")
    torch.cuda.synchronize()
    return dS.cpu().numpy()
