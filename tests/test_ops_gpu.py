"""Standalone device multiply and triangular solves vs the oracle
(arith.hmul/htrsl/htrsu, accumulator.htrsl_accu/htrsu_accu)."""

import numpy as np
import pytest

from oracle import hm_oracle as O
from tests.test_hlu_gpu import oracle_A, product_structure

pytestmark = pytest.mark.gpu


def setup(name="s2"):
    from paper_1911_07531_b200 import hmatrix as H

    A, pol, eps = oracle_A(name)
    cfg, broot, perm = product_structure(name)
    hpol = H.TruncationPolicy.fixed_accuracy(cfg.eps)
    return A, pol, eps, broot, hpol


def ranks(lv, bt):
    r, _ = O.leaf_arrays(O.HM(bt, lv))
    return r


def test_hmul_matches_oracle():
    from paper_1911_07531_b200 import hmatrix as H
    from paper_1911_07531_b200.arith import hmul

    A, pol, eps, broot, hpol = setup()
    C = A.copy()
    O.COUNT.truncations = 0
    O.hmul(-0.5, A, 0, A, 0, C, 0, pol)
    tr = O.COUNT.truncations
    dA = H.from_leaves(broot, A.lv, hpol, 128)
    dB = H.from_leaves(broot, A.lv, hpol, 128)
    dC = H.from_leaves(broot, A.lv, hpol, 128)
    H.counters.reset()
    hmul(-0.5, dA, dB, dC, hpol)
    assert H.counters.snapshot()[0] == tr
    got = dC.store.download_leaves()
    assert np.array_equal(ranks(got, A.bt), ranks(C.lv, A.bt))
    X = np.random.default_rng(1).normal(size=(A.bt.shape(0)[0], 2))
    w = O.apply(C, 0, X)
    g = O.apply(O.HM(A.bt, got), 0, X)
    assert np.linalg.norm(g - w) <= 10 * eps * np.linalg.norm(w)


@pytest.mark.parametrize("op", ["htrsl", "htrsu", "htrsl_accu", "htrsu_accu"])
def test_solves_match_oracle(op):
    from paper_1911_07531_b200 import accumulator as acc
    from paper_1911_07531_b200 import arith
    from paper_1911_07531_b200 import hmatrix as H

    A, pol, eps, broot, hpol = setup()
    L, U, _, _ = O.factor(A, "std", pol)
    T = L if op.startswith("htrsl") else U
    # right-hand side: a different kernel on the same tree (solving with A
    # itself would give X = U up to eps noise, i.e. rank decisions at the
    # rounding level of the cut)
    from tests.golden_inputs import case

    pts, _, n_min, _, eta, _ = case("s2")
    ct = O.cluster_tree(pts, n_min)
    Mr = O.assemble(A.bt, lambda I, J: O.exp_kernel_dense(pts, ct.perm, 0.5, I, J, diag=2.0), pol)
    M = Mr.copy()
    X = O.zeros(A.bt)
    O.COUNT.truncations = 0
    if op == "htrsl":
        O.htrsl(T, 0, M, 0, X, pol)
    elif op == "htrsu":
        O.htrsu(T, 0, M, 0, X, pol)
    elif op == "htrsl_accu":
        O.htrsl_accu(T, 0, M, 0, X, O.Accs(), pol)
    else:
        O.htrsu_accu(T, 0, M, 0, X, O.Accs(), pol)
    tr = O.COUNT.truncations
    dT = H.from_leaves(broot, T.lv, hpol, 128)
    dM = H.from_leaves(broot, Mr.lv, hpol, 128)
    dX = H.zeros(broot, hpol, 128)
    H.counters.reset()
    if op == "htrsl":
        arith.htrsl(dT, dM, dX, hpol)
    elif op == "htrsu":
        arith.htrsu(dT, dM, dX, hpol)
    elif op == "htrsl_accu":
        acc.htrsl_accu(dT, dM, dX, acc.AccumulatorMap(), hpol)
    else:
        acc.htrsu_accu(dT, dM, dX, acc.AccumulatorMap(), hpol)
    assert H.counters.snapshot()[0] == tr
    got = dX.store.download_leaves()
    assert np.array_equal(ranks(got, A.bt), ranks(X.lv, A.bt))
    Y = np.random.default_rng(2).normal(size=(A.bt.shape(0)[0], 2))
    w = O.apply(X, 0, Y)
    g = O.apply(O.HM(A.bt, got), 0, Y)
    assert np.linalg.norm(g - w) <= 10 * eps * np.linalg.norm(w)
