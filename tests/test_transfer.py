"""Packed leaf transfer (wire / dump format): host restatement round trip
on CPU; device pack/unpack kernels (csrc/hmx_transfer.cu) against it on the
GPU, and a factorization fed through the packed path equals the regular
path bit for bit."""

import numpy as np
import pytest

from paper_1911_07531_b200 import configs, hmatrix as H


def _random_leaves(t, seed, kmax=4):
    rng = np.random.default_rng(seed)
    lv = {}
    for u in t.leaves(0):
        m, n = int(t.m[u]), int(t.nc[u])
        if t.adm[u]:
            k = int(rng.integers(0, kmax + 1))
            lv[u] = ("R", rng.normal(size=(m, k)), rng.normal(size=(n, k)))
        else:
            lv[u] = ("D", rng.normal(size=(m, n)))
    return lv


def _same(a, b):
    assert a.keys() == b.keys()
    for u in a:
        assert a[u][0] == b[u][0]
        for x, y in zip(a[u][1:], b[u][1:]):
            assert x.shape == y.shape and np.array_equal(x, y), u


@pytest.mark.parametrize("name", ["s1", "s2"])
def test_host_pack_round_trip(name):
    cfg = configs.config(name)
    _, _, _, broot = configs.structure(cfg)
    t = H.table_of(broot)
    members = [_random_leaves(t, s) for s in range(3)]
    data, ranks = H.pack_leaves(t, members)
    sizes = sum(int(t.m[u] * t.nc[u]) if not t.adm[u] else
                int((t.m[u] + t.nc[u]) * m[u][1].shape[1]) for m in members for u in t.leaves(0))
    assert data.size == sizes
    back = H.unpack_leaves(t, data, ranks, 3)
    for a, b in zip(members, back):
        _same(a, b)
    with pytest.raises(ValueError):
        H.unpack_leaves(t, data[:-1], ranks, 3)


@pytest.mark.gpu
def test_device_pack_matches_host_format():
    import torch

    cfg = configs.config("s2")
    _, _, _, broot = configs.structure(cfg)
    pol = H.TruncationPolicy.fixed_accuracy(cfg.eps)
    t = H.table_of(broot)
    members = [_random_leaves(t, s, kmax=6) for s in range(3)]
    B = H.HBatch(broot, pol, 3, 16)
    data, ranks = H.pack_leaves(t, members)
    B.upload_packed(torch.from_numpy(data).pin_memory(), torch.from_numpy(ranks))
    for b in range(3):
        _same(B.member(b).store.download_leaves(), members[b])
    out, rk = B.download_packed()
    torch.cuda.synchronize()
    assert np.array_equal(out.numpy(), data)
    assert np.array_equal(rk.numpy(), ranks)


@pytest.mark.gpu
@pytest.mark.parametrize("mode", ["std", "accu"])
def test_packed_path_factorization_bitwise(mode):
    """H2D packed A -> hlu_batch -> D2H packed L, U equals the pool path,
    with garbage in A's unused rank capacity and L/U reused across runs."""
    import torch

    from paper_1911_07531_b200.arith import hlu_batch

    cfg = configs.config("s2")
    _, _, perm, broot = configs.structure(cfg)
    pol = H.TruncationPolicy.fixed_accuracy(cfg.eps)
    A = H.assemble(broot, configs.kernel(cfg, perm), pol, rank_cap=64)
    ref = H.HBatch.replicate(A, 2)
    L0, U0 = H.HBatch(broot, pol, 2, 64), H.HBatch(broot, pol, 2, 64)
    hlu_batch(ref, L0, U0, pol, mode)
    t = A.table
    data, ranks = H.pack_leaves(t, [A.store.download_leaves()] * 2)
    AB = H.HBatch(broot, pol, 2, 64)
    LB, UB = H.HBatch(broot, pol, 2, 64), H.HBatch(broot, pol, 2, 64)
    # garbage in A's unused rank capacity; L and U come from zeros (the
    # reference's contract, arith.py:76-94) and are reused across the runs
    AB.store.values.fill_(float("nan"))
    hd, hr = torch.from_numpy(data).pin_memory(), torch.from_numpy(ranks).pin_memory()
    for _ in range(2):
        AB.upload_packed(hd, hr)
        hlu_batch(AB, LB, UB, pol, mode)
        Lp, Lr = LB.download_packed()
        Up, Ur = UB.download_packed()
        torch.cuda.synchronize()
        for P, R, Ref in ((Lp, Lr, L0), (Up, Ur, U0)):
            got = H.unpack_leaves(t, P.numpy(), R.numpy(), 2)
            for b in range(2):
                _same(got[b], Ref.member(b).store.download_leaves())


@pytest.mark.gpu
def test_pipelined_stream_equals_batched_path():
    """batch.PipelinedHLU (H2D / factor / D2H overlapped over a stream of
    batches, two alternating buffer sets) returns per batch exactly the
    packed factors of the plain hlu_batch path."""
    import torch

    from paper_1911_07531_b200.arith import hlu_batch
    from paper_1911_07531_b200.batch import PipelinedHLU

    cfg = configs.config("s2")
    _, _, perm, broot = configs.structure(cfg)
    pol = H.TruncationPolicy.fixed_accuracy(cfg.eps)
    A = H.assemble(broot, configs.kernel(cfg, perm), pol, rank_cap=64)
    t = A.table
    ins, refs = [], []
    for scale in (1.0, 0.5, 2.0, 0.25, 4.0):
        lv = {u: (x[0], *[scale * y for y in x[1:]]) if x[0] == "D" else (x[0], scale * x[1], x[2])
              for u, x in A.store.download_leaves().items()}
        data, ranks = H.pack_leaves(t, [lv, lv])
        ins.append((torch.from_numpy(data).pin_memory(), torch.from_numpy(ranks).pin_memory()))
        AB, LB, UB = H.HBatch(broot, pol, 2, 64), H.HBatch(broot, pol, 2, 64), H.HBatch(broot, pol, 2, 64)
        AB.upload_packed(*ins[-1])
        hlu_batch(AB, LB, UB, pol, "accu")
        refs.append([M.download_packed() for M in (LB, UB)])
        torch.cuda.synchronize()
    pipe = PipelinedHLU(broot, pol, 2, 64, "accu")
    res, ev = pipe.run(ins)
    ev.synchronize()
    pipe.check()
    for got, want in zip(res, refs):
        for (gv, gr), (wv, wr) in zip(got, want):
            assert np.array_equal(gr.numpy(), wr.numpy())
            assert np.array_equal(gv.numpy(), wv.numpy())
