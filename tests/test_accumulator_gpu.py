"""Drop-in accumulator and payload primitives on the device
(accumulator.py:41-161, hmatrix.py:349-448 of the reference): the
semantics the reference's own tests pin (tests/test_accumulator.py,
tests/test_hmatrix.py there), checked against dense numpy products."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _case(n, n_min=16, eta=1.0, shift=0.5):
    from paper_1911_07531_b200.problems import one_d_problem, permuted, shifted
    from paper_1911_07531_b200.trees import build_block_tree, build_cluster_tree, standard_admissible

    geom, kernel = one_d_problem(n)
    if shift:
        kernel = shifted(kernel, shift, n)
    root, perm = build_cluster_tree(geom, n_min=n_min)
    block = build_block_tree(root, root, lambda t, s: standard_admissible(t, s, eta))
    return block, permuted(kernel, perm)


def _asm(block, kernel):
    from paper_1911_07531_b200.hmatrix import EXACT, assemble

    return assemble(block, kernel, EXACT)


def test_add_upd_alpha_zero_and_pending():
    from paper_1911_07531_b200.accumulator import AccumulatorMap, add_upd
    from paper_1911_07531_b200.hmatrix import EXACT

    block, kernel = _case(64)
    A = _asm(block, kernel)
    accs = AccumulatorMap()
    add_upd(0.0, A, A, A, accs, EXACT)
    assert len(accs) == 0
    block, kernel = _case(128)
    A = _asm(block, kernel)
    accs = AccumulatorMap()
    add_upd(1.0, A, A, A, accs, EXACT)
    acc = accs.get(block)
    assert acc is not None and len(acc.pending) == 1 and acc.U_mat is None


def test_two_leaf_updates_sum():
    from paper_1911_07531_b200.accumulator import AccumulatorMap, add_upd
    from paper_1911_07531_b200.hmatrix import EXACT
    from paper_1911_07531_b200.problems import dense_matrix

    block, kernel = _case(32, n_min=32)
    A = _asm(block, kernel)
    accs = AccumulatorMap()
    add_upd(1.0, A, A, A, accs, EXACT)
    add_upd(0.5, A, A, A, accs, EXACT)
    K = dense_matrix(kernel, 32)
    want = 1.5 * K @ K
    got = accs.get(block).U_mat[1]
    assert np.linalg.norm(got - want) <= 1e-13 * np.linalg.norm(want)


def test_shift_restricts_and_splits():
    from paper_1911_07531_b200 import hmatrix as hm
    from paper_1911_07531_b200.accumulator import AccumulatorMap, add_upd, shift_upd
    from paper_1911_07531_b200.hmatrix import EXACT

    block, kernel = _case(16, n_min=16)
    A = _asm(block, kernel)
    with pytest.raises(ValueError):
        shift_upd(A, AccumulatorMap(), EXACT)
    block, kernel = _case(128)
    A = _asm(block, kernel)
    accs = AccumulatorMap()
    n = 128
    accs.get_or_create(block).fold((hm.LOWRANK, np.ones((n, 1)), np.ones((n, 1))), EXACT)
    shift_upd(A, accs, EXACT)
    assert accs.get(block).is_empty
    for row in A.children:
        for ch in row:
            u = accs.get(ch.block).U_mat
            assert u is not None and np.allclose(hm.payload_dense(u), np.ones((ch.nrows, ch.ncols)))
    # a pending structured product splits into 2 products per child
    accs = AccumulatorMap()
    add_upd(1.0, A, A, A, accs, EXACT)
    shift_upd(A, accs, EXACT)
    assert sum(len(accs.get(ch.block).pending) for row in A.children for ch in row
               if accs.get(ch.block) is not None) + sum(
        1 for row in A.children for ch in row if accs.get(ch.block) is not None
        and accs.get(ch.block).U_mat is not None) >= 4


def test_apply_equals_hmul():
    """add_upd + apply_upd gives A + alpha A B like hmul (EXACT)."""
    from paper_1911_07531_b200.accumulator import AccumulatorMap, add_upd, apply_upd
    from paper_1911_07531_b200.hmatrix import EXACT, rel_error
    from paper_1911_07531_b200.problems import dense_matrix

    block, kernel = _case(128)
    A = _asm(block, kernel)
    B = _asm(block, kernel)
    C = _asm(block, kernel)
    K = dense_matrix(kernel, 128)
    accs = AccumulatorMap()
    add_upd(-0.25, A, B, C, accs, EXACT)
    apply_upd(C, accs, EXACT)
    want = K - 0.25 * K @ K
    assert rel_error(want, C) <= 1e-12
    apply_upd(C, accs, EXACT)  # idempotent once drained
    assert rel_error(want, C) <= 1e-12


@pytest.mark.parametrize("ka,kb", [("D", "D"), ("D", "R"), ("R", "D"), ("R", "R"), ("H", "D"),
                                   ("D", "H"), ("H", "R"), ("H", "H")])
def test_product_payload_kinds(ka, kb):
    """alpha A B for every operand-kind combination vs the dense product."""
    from paper_1911_07531_b200 import hmatrix as hm
    from paper_1911_07531_b200.hmatrix import EXACT

    block, kernel = _case(128)
    A = _asm(block, kernel)
    K = A.to_dense()

    def pick(kind):
        for x in [A] + list(A.leaves()) + [c for row in A.children for c in row]:
            if x.kind == {"D": hm.DENSE, "R": hm.LOWRANK, "H": hm.BLOCKED}[kind]:
                return x
        return None

    X, Y = pick(ka), pick(kb)
    if X is None or Y is None or X.ncols != Y.nrows:
        # pair blocks of matching inner dimension by the root's children
        pytest.skip("no conformal pair of these kinds in the small case")
    p = hm.product_payload(0.5, X, Y, EXACT)
    t = X.table
    Xd = K[t.r0[X.uid]:t.r1[X.uid], t.c0[X.uid]:t.c1[X.uid]]
    Yd = K[t.r0[Y.uid]:t.r1[Y.uid], t.c0[Y.uid]:t.c1[Y.uid]]
    want = 0.5 * Xd @ Yd
    got = hm.payload_dense(p)
    assert np.linalg.norm(got - want) <= 1e-12 * max(np.linalg.norm(want), 1.0)


def test_fold_and_scatter_payload():
    from paper_1911_07531_b200 import hmatrix as hm
    from paper_1911_07531_b200.hmatrix import EXACT, rel_error

    block, kernel = _case(128)
    A = _asm(block, kernel)
    K = A.to_dense()
    rng = np.random.default_rng(0)
    u, v = rng.normal(size=(128, 2)), rng.normal(size=(128, 2))
    hm.scatter_payload(A, (hm.LOWRANK, u, v), EXACT)
    assert rel_error(K + u @ v.T, A) <= 1e-12
    D = rng.normal(size=(128, 128))
    hm.scatter_payload(A, (hm.DENSE, D), EXACT)
    assert rel_error(K + u @ v.T + D, A) <= 1e-12


def test_hlu_accu_applies_queued_updates():
    """Updates queued in the map before hlu_accu are part of the factored
    matrix (the reference's hlu_accu shifts them down the recursion)."""
    from paper_1911_07531_b200.accumulator import AccumulatorMap, add_upd, hlu_accu
    from paper_1911_07531_b200.hmatrix import EXACT, rel_error, zeros

    block, kernel = _case(128, shift=2.0)
    A = _asm(block, kernel)
    B = _asm(block, kernel)
    K = A.to_dense()
    accs = AccumulatorMap()
    add_upd(-0.01, B, B, A, accs, EXACT)
    L, U = zeros(block, EXACT), zeros(block, EXACT)
    hlu_accu(A, L, U, accs, EXACT)
    want = K - 0.01 * K @ K
    assert rel_error(want, L.to_dense() @ U.to_dense()) <= 1e-10
    assert accs.is_clear()
