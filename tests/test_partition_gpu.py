"""Partitioned H-LU, every rank emulated in one launch on one GPU.

CTA c serves rank c mod nranks with its own ready queue and its own replica
of A, L, U, the accumulators and the micro-task workspace; objects move
between replicas only through the exchange records (partition.py), as they
would over NVLink between GPUs.  The factors gathered from the owners'
replicas must equal the single-GPU factorization bit for bit.
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _same_leaves(a, b):
    assert a.keys() == b.keys()
    for u in a:
        x, y = a[u], b[u]
        assert x[0] == y[0], u
        for p, q in zip(x[1:], y[1:]):
            assert p.shape == q.shape, u
            assert np.array_equal(p, q), u


@pytest.mark.parametrize("name,mode,nranks", [("s2", "accu", 2), ("s2", "std", 4), ("c1", "std", 2),
                                              ("c1", "accu", 4), ("c2", "accu", 4), ("c2", "std", 8),
                                              ("c5_d5", "accu", 4)])
def test_emulated_partition_is_bit_exact(name, mode, nranks):
    from paper_1911_07531_b200 import configs, hmatrix as H
    from paper_1911_07531_b200.arith import run_hlu
    from paper_1911_07531_b200.partition import PartitionedPlan

    cfg = configs.config(name)
    geom, root, perm, broot = configs.structure(cfg)
    pol = H.TruncationPolicy.fixed_accuracy(cfg.eps)
    rc = 128 if name.startswith("c5") else 64
    A = H.assemble(broot, configs.kernel(cfg, perm), pol, rank_cap=rc)
    A1 = A.copy()
    L1, U1 = H.zeros(broot, pol, rc), H.zeros(broot, pol, rc)
    run_hlu(A1, L1, U1, pol, mode)
    pp = PartitionedPlan(A.table, mode, pol, rc, nranks)
    st = pp.part.stats()
    assert st["cross_edges"] > 0 and pp.n_pub > 0
    AB, LB, UB = pp.stores(A.store)
    pp.run(AB, LB, UB)
    L = pp.collect(LB, 1)
    U = pp.collect(UB, 2)
    _same_leaves(L.download_leaves(), L1.store.download_leaves())
    _same_leaves(U.download_leaves(), U1.store.download_leaves())
    # a second run of the same plan (scheduler state reset) is identical
    AB2, LB2, UB2 = pp.stores(A.store)
    pp.run(AB2, LB2, UB2)
    _same_leaves(pp.collect(LB2, 1).download_leaves(), L1.store.download_leaves())
