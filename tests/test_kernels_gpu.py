"""Device leaf kernels vs numpy/scipy (the reference's LAPACK calls).

Tolerances: the kernels are fp64; products and solves are compared at
1e-12 relative, LU at bitwise equality (the device LU mirrors
arith.dense_lu's rounding: separate multiply and subtract, arith.py:70-71),
truncation ranks exactly and recompressed products within
max(1e-10, 1e-3*eps) relative (tolerance tied to the truncation eps).
"""

import numpy as np
import pytest
import scipy.linalg as sla

pytestmark = pytest.mark.gpu


def ref_dense_lu(A):
    # arith.dense_lu restated (arith.py:58-73); oracle copy lives in oracle/
    from oracle.hm_oracle import dense_lu

    return dense_lu(A)


def test_getrf_bitwise_vs_oracle():
    from paper_1911_07531_b200 import kernels

    rng = np.random.default_rng(0)
    for n in (16, 64, 128):
        As = [rng.normal(size=(n, n)) + n * np.eye(n) for _ in range(3)]
        L, U, info = kernels.getrf_nopiv(As)
        assert (info == 0).all()
        for a, l, u in zip(As, L, U):
            lr, ur = ref_dense_lu(a)
            assert np.array_equal(l, lr)
            assert np.array_equal(u, ur)


def test_getrf_singular_pivot_flag():
    from paper_1911_07531_b200 import kernels

    L, U, info = kernels.getrf_nopiv([np.zeros((8, 8))])
    assert info[0] & 4


def test_trsm():
    from paper_1911_07531_b200 import kernels

    rng = np.random.default_rng(1)
    for n, c in ((64, 64), (64, 7), (128, 20), (200, 5)):
        A = rng.normal(size=(n, n)) + n * np.eye(n)
        Lf = np.tril(A, -1) / n + np.eye(n)
        Uf = np.triu(A)
        B = rng.normal(size=(n, c))
        X = kernels.trsm_lower_unit([Lf], [B])[0]
        Xr = sla.solve_triangular(Lf, B, lower=True, unit_diagonal=True)
        assert np.linalg.norm(X - Xr) <= 1e-12 * np.linalg.norm(Xr)
        W = kernels.trsm_upper_trans([Uf], [B])[0]
        Wr = sla.solve_triangular(Uf, B, trans="T", lower=False)
        assert np.linalg.norm(W - Wr) <= 1e-12 * np.linalg.norm(Wr)
        # back substitution (solve phase): warp path n <= 128, CTA sweep above
        Y = kernels.trsm_upper([Uf], [B])[0]
        Yr = sla.solve_triangular(Uf, B, lower=False)
        assert np.linalg.norm(Y - Yr) <= 1e-12 * np.linalg.norm(Yr)


@pytest.mark.parametrize("ta,tb", [(False, False), (True, False), (False, True), (True, True)])
def test_gemm(ta, tb):
    from paper_1911_07531_b200 import kernels

    rng = np.random.default_rng(2)
    for m, n, k in ((64, 64, 64), (130, 7, 33), (5, 200, 17), (1, 1, 1)):
        A = rng.normal(size=(k, m) if ta else (m, k))
        B = rng.normal(size=(n, k) if tb else (k, n))
        C0 = rng.normal(size=(m, n))
        want = C0 - 1.0 * ((A.T if ta else A) @ (B.T if tb else B))
        got = kernels.gemm(-1.0, [A], [B], [C0], transA=ta, transB=tb, beta=1.0)[0]
        assert np.linalg.norm(got - want) <= 1e-13 * np.linalg.norm(want)


@pytest.mark.parametrize("ta,tb", [(False, False), (True, True)])
def test_gemm_small_path_bitwise_equals_tiled(ta, tb):
    """The small-output GEMM (m*n <= 4*threads, one-pass staging) and the
    64x64 tiled GEMM run the same increasing-k fma chain per output: a
    sub-block computed alone (small path) equals the same entries of a large
    product (tiled path) bit for bit."""
    from paper_1911_07531_b200 import _lib, kernels

    rng = np.random.default_rng(11)
    m, n, k = 96, 80, 45
    A = rng.normal(size=(k, m) if ta else (m, k))
    B = rng.normal(size=(n, k) if tb else (k, n))
    C0 = rng.normal(size=(m, n))
    big = kernels.gemm(-0.7, [A], [B], [C0], transA=ta, transB=tb, beta=1.0)[0]
    for (i0, i1, j0, j1) in ((0, 16, 0, 16), (5, 37, 3, 20), (90, 96, 0, 80)):
        As = A[:, i0:i1] if ta else A[i0:i1, :]
        Bs = B[j0:j1, :] if tb else B[:, j0:j1]
        sub = kernels.gemm(-0.7, [np.ascontiguousarray(As)], [np.ascontiguousarray(Bs)],
                           [np.ascontiguousarray(C0[i0:i1, j0:j1])], transA=ta, transB=tb, beta=1.0)[0]
        if b"dmma" in _lib.lib().hmx_version():
            # the tiled path runs on the FP64 tensor cores (k summed in the mma's
            # order): the two paths agree to rounding, not bit for bit
            assert np.abs(sub - big[i0:i1, j0:j1]).max() <= 1e-13 * np.abs(big).max()
        else:
            assert np.array_equal(sub, big[i0:i1, j0:j1])


class _Pol:
    def __init__(self, mode, eps=None, k=None):
        self.mode, self.eps, self.k = mode, eps, k


def test_svd_values_vs_lapack():
    from paper_1911_07531_b200 import kernels

    rng = np.random.default_rng(3)
    for p, q in ((20, 20), (33, 17), (17, 33), (64, 64), (100, 40)):
        G = rng.normal(size=(p, q)) * np.exp(-0.5 * np.arange(q))[None, :]
        s = kernels.svd_values([G])[0]
        sr = np.linalg.svd(G, compute_uv=False)
        assert np.allclose(s, sr, rtol=1e-12, atol=1e-14 * sr[0])


def test_truncate_vs_reference_fixtures():
    """Ranks equal to the reference's truncate on its golden cases; the
    recompressed product within 1e-12 relative of the reference's."""
    import json
    import os

    from paper_1911_07531_b200 import kernels
    from tests.golden_inputs import GOLDEN, probe_vec, truncate_inputs

    meta = json.load(open(os.path.join(GOLDEN, "kernels.json")))
    ref = np.load(os.path.join(GOLDEN, "kernels.npz"))
    for i, (m, n, K, decay) in enumerate(meta["specs"]):
        U, V, M = truncate_inputs(i, m, n, K, decay)
        for eps in (1e-4, 1e-6, 1e-8):
            Un, Vn = kernels.truncate(U, V, _Pol("accuracy", eps=eps))
            assert Un.shape[1] == int(ref[f"t{i}_{eps:g}_rank"]), (i, eps)
            pr = ref[f"t{i}_{eps:g}_probe"]
            got = Un @ (Vn.T @ probe_vec(n))
            # the rank-revealing step drops a tail <= 1e-5*eps*sigma_1 (see cta_rrqr)
            assert np.linalg.norm(got - pr) <= max(1e-10, 1e-3 * eps) * np.linalg.norm(pr) + 1e-13
        for eps in (1e-4, 1e-6):
            W, Z = kernels.dense_to_lowrank(M, _Pol("accuracy", eps=eps))
            assert W.shape[1] == int(ref[f"d{i}_{eps:g}_rank"]), (i, eps)
            pr = ref[f"d{i}_{eps:g}_probe"]
            got = W @ (Z.T @ probe_vec(n))
            assert np.linalg.norm(got - pr) <= max(1e-10, 1e-3 * eps) * np.linalg.norm(pr) + 1e-13


def test_truncate_policies_and_passthrough():
    from paper_1911_07531_b200 import kernels

    U = np.eye(4)[:, :2]
    V = np.eye(4)[:, :2]
    Un, Vn = kernels.truncate(U, V, _Pol("rank", k=1))
    assert Un.shape[1] == 1
    assert abs(np.linalg.norm(U @ V.T - Un @ Vn.T) - 1.0) < 1e-12
    U0, V0 = np.zeros((5, 0)), np.zeros((4, 0))
    a, b = kernels.truncate(U0, V0, _Pol("exact"))
    assert a.shape == (5, 0) and b.shape == (4, 0)


def _kernel_block(m, n, sep, seed, ell=0.3):
    """exp(-d / ell) between two point clouds `sep` box widths apart: the
    smooth spectrum of an admissible block."""
    rng = np.random.default_rng(seed)
    a = rng.random((m, 3))
    b = rng.random((n, 3)) + np.array([1.0 + sep, 0.0, 0.0])
    d = np.linalg.norm(a[:, None, :] - b[None, :, :], axis=-1)
    return np.exp(-d / ell)


@pytest.mark.parametrize("m,n,K,path", [
    (64, 64, 24, "shared"), (128, 96, 40, "shared"), (256, 256, 24, "shared"), (100, 72, 30, "shared ragged"),
    (1024, 512, 30, "panel"), (2048, 2048, 20, "panel two levels"), (700, 300, 28, "panel ragged"),
    (128, 128, 100, "fat"), (256, 192, 90, "fat"), (512, 256, 72, "fat"),
])
def test_truncate_paths_vs_oracle(m, n, K, path):
    """Every truncation path (shared memory, panel TSQR, column-blocked 'fat',
    round-1 fallback) gives the oracle's rank (hmatrix.truncate restated,
    hmatrix.py:113-130) and its recompressed product within the
    eps-tied tolerance, on stacked factors of kernel blocks (what an
    accumulator holds)."""
    from oracle.hm_oracle import Policy, truncate as ref_truncate
    from paper_1911_07531_b200 import kernels

    rng = np.random.default_rng(m + n + K)
    # stacked factors: truncated SVD factors of a few kernel blocks, column-stacked
    parts = []
    k0 = max(K // 3, 1)
    for s in range(3):
        M = _kernel_block(m, n, 0.4 + 0.3 * s, 11 * s + K)
        u, sv, vt = np.linalg.svd(M, full_matrices=False)
        kk = k0 if s < 2 else K - 2 * k0
        parts.append((u[:, :kk] * sv[:kk] * (1.0 if s != 1 else -0.7), vt[:kk].T))
    U = np.hstack([p[0] for p in parts])
    V = np.hstack([p[1] for p in parts])
    assert U.shape == (m, K) and V.shape == (n, K)
    x = rng.normal(size=(n, 3))
    for eps in (1e-4, 1e-6):
        pol = _Pol("accuracy", eps=eps)
        Ur, Vr = ref_truncate(U, V, Policy("accuracy", eps=eps))
        Un, Vn = kernels.truncate(U, V, pol, cap=min(m, n, K))
        assert Un.shape[1] == Ur.shape[1], (path, eps, Un.shape[1], Ur.shape[1])
        pr, got = Ur @ (Vr.T @ x), Un @ (Vn.T @ x)
        assert np.linalg.norm(got - pr) <= max(1e-10, 1e-3 * eps) * np.linalg.norm(pr), (path, eps)


@pytest.mark.parametrize("m,n,sep,path", [
    (64, 64, 0.5, "shared"), (128, 128, 0.3, "shared, G evicted"), (96, 128, 0.8, "shared ragged"),
    (256, 256, 0.8, "global pivoted QR"), (256, 256, 0.5, "global pivoted QR, fallback at the small eps"),
    (512, 512, 1.0, "global pivoted QR"), (512, 256, 0.8, "global, rectangular"),
])
def test_dense_to_lowrank_paths_vs_oracle(m, n, sep, path):
    """dense_to_lowrank (hmatrix.py:133-138) on every path: rank and product
    against the oracle's SVD truncation."""
    from oracle.hm_oracle import Policy, dense_to_lowrank as ref_d2lr
    from paper_1911_07531_b200 import kernels

    M = _kernel_block(m, n, sep, m + n)
    x = np.random.default_rng(5).normal(size=(n, 3))
    for eps in (1e-4, 1e-6):
        pol = _Pol("accuracy", eps=eps)
        Ur, Vr = ref_d2lr(M, Policy("accuracy", eps=eps))
        Un, Vn = kernels.dense_to_lowrank(M, pol, cap=min(m, n, 64))
        assert Un.shape[1] == Ur.shape[1], (path, eps, Un.shape[1], Ur.shape[1])
        pr, got = Ur @ (Vr.T @ x), Un @ (Vn.T @ x)
        assert np.linalg.norm(got - pr) <= max(1e-10, 1e-3 * eps) * np.linalg.norm(pr), (path, eps)
