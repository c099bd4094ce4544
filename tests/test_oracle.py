"""Pin the CPU oracle (oracle/hm_oracle.py) against the reference's fixtures.

The fixtures were produced by running the unmodified reference package
(tests/golden/make_golden.py).  Structure must match exactly; the numeric
oracle reproduces ranks and counters exactly and factors to rounding.
"""

import hashlib

import numpy as np
import pytest

from oracle import hm_oracle as O
from tests.golden_inputs import case, have, load, probe_vec, truncate_inputs


def sha(text):
    return hashlib.sha256(text.encode()).hexdigest()


def build(name):
    pts, ell, n_min, kind, eta, eps = case(name)
    ct = O.cluster_tree(pts, n_min)
    adm = O.adm_weak(ct) if kind == "weak" else O.adm_standard(ct, eta)
    bt = O.block_tree(ct, adm)
    return pts, ell, eps, ct, bt


def serialize_clusters(ct):
    lines = []
    parent = {}
    for u, k in enumerate(ct.kids):
        for c in k:
            parent[c] = u
    # pre-order == uid order
    for u in range(len(ct.first)):
        lines.append(f"{u} {parent.get(u, -1)} {ct.first[u]} {ct.last[u]} {int(not ct.kids[u])} 0")
    return "\n".join(lines) + "\n"


def serialize_blocks(bt):
    rows = bt.table()
    return "\n".join(" ".join(str(int(v)) for v in r) for r in rows) + "\n"


@pytest.mark.parametrize("name", ["s1", "s2", "s5", "c1", "c2", "c4_0", "c4_1"])
def test_structure_matches_reference(name):
    if not have(name):
        pytest.skip("fixture not generated")
    meta, arr = load(name)
    pts, ell, eps, ct, bt = build(name)
    assert sha(serialize_clusters(ct)) == meta["cluster_sha"]
    assert sha(serialize_blocks(bt)) == meta["block_sha"]
    assert sha(",".join(map(str, ct.perm.tolist()))) == meta["perm_sha"]
    if "blocks" in arr:
        assert np.array_equal(bt.table(), arr["blocks"])


def test_truncate_and_dense_to_lowrank_match_reference():
    import json
    import os

    from tests.golden_inputs import GOLDEN

    meta = json.load(open(os.path.join(GOLDEN, "kernels.json")))
    ref = np.load(os.path.join(GOLDEN, "kernels.npz"))
    for i, (m, n, K, decay) in enumerate(meta["specs"]):
        U, V, M = truncate_inputs(i, m, n, K, decay)
        for eps in (1e-4, 1e-6, 1e-8):
            Un, Vn = O.truncate(U, V, O.Policy("accuracy", eps=eps))
            assert Un.shape[1] == int(ref[f"t{i}_{eps:g}_rank"])
            assert np.array_equal(Un @ (Vn.T @ probe_vec(n)), ref[f"t{i}_{eps:g}_probe"])
        for eps in (1e-4, 1e-6):
            W, Z = O.dense_to_lowrank(M, O.Policy("accuracy", eps=eps))
            assert W.shape[1] == int(ref[f"d{i}_{eps:g}_rank"])
            assert np.array_equal(W @ (Z.T @ probe_vec(n)), ref[f"d{i}_{eps:g}_probe"])
    for i in range(4):
        n = (16, 33, 64, 128)[i]
        r = np.random.default_rng(300 + i)
        A = r.normal(size=(n, n)) + n * np.eye(n)
        L, U = O.dense_lu(A)
        assert np.array_equal(L, ref[f"lu{i}_L"]) and np.array_equal(U, ref[f"lu{i}_U"])


def oracle_case(name):
    pts, ell, eps, ct, bt = build(name)
    pol = O.Policy("accuracy", eps=eps)
    O.COUNT.truncations = 0
    A = O.assemble(bt, lambda I, J: O.exp_kernel_dense(pts, ct.perm, ell, I, J), pol)
    return A, pol, O.COUNT.truncations


@pytest.mark.parametrize("name", ["s1"])
def test_numerics_bitwise_vs_reference(name):
    meta, arr = load(name)
    A, pol, ntr = oracle_case(name)
    assert ntr == meta["assembly_truncations"]
    rA, fA = O.leaf_arrays(A)
    assert np.array_equal(rA, arr["A_rank"])
    X = arr["probe_x"]
    assert np.linalg.norm(O.apply(A, 0, X) - arr["probe_Ax"]) <= 1e-14 * np.linalg.norm(arr["probe_Ax"])
    for mode in ("std", "accu"):
        L, U, tr, up = O.factor(A, mode, pol)
        assert tr == meta[f"{mode}_truncations"]
        assert up == meta[f"{mode}_updates"]
        rL, fL = O.leaf_arrays(L)
        rU, fU = O.leaf_arrays(U)
        assert np.array_equal(rL, arr[f"{mode}_L_rank"])
        assert np.array_equal(rU, arr[f"{mode}_U_rank"])
        # BLAS thread count changes the last bits of dgemm; ranks above are exact
        got = O.apply(L, 0, O.apply(U, 0, X))
        want = arr[f"{mode}_probe_LUx"]
        assert np.linalg.norm(got - want) <= 1e-13 * np.linalg.norm(want)


@pytest.mark.slow
@pytest.mark.parametrize("name", ["s2"])
def test_numerics_bitwise_vs_reference_2d(name):
    test_numerics_bitwise_vs_reference(name)
