"""H x dense operations on the device — hm_apply, hm_apply_t, hm_solve_lower,
hm_solve_upper_t (hmatrix.py:286-341) — against the oracle restatement of
the same recursions (oracle/hm_oracle.py apply / apply_t / solve_*), on the
H-LU factors of the s2 and c1 cases, for the root and for sub-blocks."""

import numpy as np
import pytest

from oracle import hm_oracle as O
from paper_1911_07531_b200 import configs, hmatrix as H
from paper_1911_07531_b200.planner import plan_dense


@pytest.mark.parametrize("op", ["apply", "apply_t", "solve_lower", "solve_upper_t", "solve_upper"])
def test_dense_programs_build(op):
    cfg = configs.config("s2")
    _, _, _, broot = configs.structure(cfg)
    t = H.table_of(broot)
    prog = plan_dense(t, op, 0, 3, 64)
    n_tasks = len(prog.keys)
    if op.startswith("apply"):
        assert n_tasks == len(np.unique(np.concatenate([t.r0[t.leaf], [t.r1[0]]]))) - 1
    else:
        assert n_tasks == 1
    assert prog.task_scratch.shape == (n_tasks,)


def _factors(name):
    from paper_1911_07531_b200.arith import hlu

    cfg = configs.config(name)
    _, _, perm, broot = configs.structure(cfg)
    pol = H.TruncationPolicy.fixed_accuracy(cfg.eps)
    A = H.assemble(broot, configs.kernel(cfg, perm), pol, rank_cap=64)
    A0 = A.copy()
    L, U = H.zeros(broot, pol, 64), H.zeros(broot, pol, 64)
    hlu(A, L, U, pol)
    ct = O.cluster_tree(cfg.points, cfg.n_min)
    adm = O.adm_weak(ct) if cfg.admissibility == "weak" else O.adm_standard(ct, cfg.eta)
    bt = O.block_tree(ct, adm)
    return cfg, bt, A0, L, U


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["s2", "c1"])
def test_dense_ops_match_oracle(name):
    cfg, bt, A, L, U = _factors(name)
    Ah = O.HM(bt, A.store.download_leaves())
    Lh = O.HM(bt, L.store.download_leaves())
    Uh = O.HM(bt, U.store.download_leaves())
    rng = np.random.default_rng(3)
    n = cfg.n
    X = rng.normal(size=(n, 3))
    tol = 1e-12
    for M, Mh in ((A, Ah), (L, Lh), (U, Uh)):
        for uid in (0, int(bt.kids[0][1]), int(bt.kids[0][2])):
            V = H.HMatrix(M.store, uid)
            m, nc = V.nrows, V.ncols
            got = H.hm_apply(V, X[:nc])
            want = O.apply(Mh, uid, X[:nc])
            assert np.linalg.norm(got - want) <= tol * np.linalg.norm(want)
            got = H.hm_apply_t(V, X[:m])
            want = O.apply_t(Mh, uid, X[:m])
            assert np.linalg.norm(got - want) <= tol * np.linalg.norm(want)
    for uid in (0, int(bt.kids[0][0])):
        m = H.HMatrix(L.store, uid).nrows
        got = H.hm_solve_lower(H.HMatrix(L.store, uid), X[:m])
        want = O.solve_lower(Lh, uid, X[:m])
        assert np.linalg.norm(got - want) <= tol * np.linalg.norm(want)
        got = H.hm_solve_upper_t(H.HMatrix(U.store, uid), X[:m])
        want = O.solve_upper_t(Uh, uid, X[:m])
        assert np.linalg.norm(got - want) <= 1e-10 * np.linalg.norm(want)
        got = H.hm_solve_upper(H.HMatrix(U.store, uid), X[:m])
        want = O.solve_upper(Uh, uid, X[:m])
        assert np.linalg.norm(got - want) <= 1e-10 * np.linalg.norm(want)
    # solve phase: A x = b through the factors (forward + back substitution)
    b = rng.normal(size=(n, 2))
    x = H.lu_solve(L, U, b)
    want = O.solve_upper(Uh, 0, O.solve_lower(Lh, 0, b))
    assert np.linalg.norm(x - want) <= 1e-10 * np.linalg.norm(want)
    # residual of the solve as good as the oracle's own solve with the same factors
    r = np.linalg.norm(O.apply(Ah, 0, x) - b)
    r_want = np.linalg.norm(O.apply(Ah, 0, want) - b)
    assert r <= 2.0 * r_want + 1e-12 * np.linalg.norm(b)
    # vector right-hand side and the device probe residual
    y = H.hm_apply(A, X[:, 0])
    assert y.shape == (n,)
    res = H.lu_residual(A, L, U, X)
    assert res <= 100 * cfg.eps


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["s2", "c1"])
def test_leaf_update_matches_oracle(name):
    """hmatrix.leaf_update (hmatrix.py:451-460): C[(t,s)] += -1 * L[(t,t)] @
    U[(t,s)] for admissible leaves (t,s) (blocked times low-rank into a
    low-rank leaf) and C starting at zero: rank and entries equal the
    oracle's product + fold within 1e-12 relative."""
    cfg, bt, A, L, U = _factors(name)
    pol = H.TruncationPolicy.fixed_accuracy(cfg.eps)
    Lh = O.HM(bt, L.store.download_leaves())
    Uh = O.HM(bt, U.store.download_leaves())
    opol = O.Policy("accuracy", eps=cfg.eps)
    C = H.zeros(A.block, pol, 64)
    Ch = O.HM(bt, C.store.download_leaves())
    n_b = len(bt.r0)
    diag = {(int(bt.r0[v]), int(bt.r1[v])): v for v in range(n_b)
            if bt.r0[v] == bt.c0[v] and bt.r1[v] == bt.c1[v]}
    done = 0
    for uc in bt.leaves(0):
        if not bt.adm[uc] or done >= 3:
            continue
        ua = diag[(int(bt.r0[uc]), int(bt.r1[uc]))]
        H.leaf_update(H.HMatrix(C.store, uc), -1.0, H.HMatrix(L.store, ua),
                      H.HMatrix(U.store, uc), pol)
        O.fold_leaf(Ch, uc, O.product(-1.0, Lh, ua, Uh, uc, opol), opol)
        got, want = C.store.download_leaf(uc), Ch.lv[uc]
        assert got[0] == want[0] == "R"
        assert got[1].shape == want[1].shape
        G, W = got[1] @ got[2].T, want[1] @ want[2].T
        assert np.linalg.norm(G - W) <= 1e-12 * max(np.linalg.norm(W), 1e-300)
        done += 1
    assert done > 0
