"""Generate golden fixtures by running the UNMODIFIED reference package.

This script is the only place that imports the reference (``hmatdag`` from
``/root/reference/pkg/src``).  It runs in the build container (the GPU box
has no ``/root/reference``) and writes small fixtures next to itself:

    tests/golden/<case>.npz   numeric + structural fixtures
    tests/golden/<case>.json  counts, hashes, residuals, counters

Inputs are seeded synthetic problems with the BASELINE.json shapes (there is
no dataset).  The problem definitions are restated here independently of the
product package so that the pin does not depend on the code it pins.

Usage:  python tests/golden/make_golden.py [case ...]
Cases:  small (s1..s4, trunc), c1, c2, c3 (numerics, fast assembly), c3s, c4, c5s,
        roots (standalone hmul/htrsl/htrsu DAGs), c5dag, c5dag_merged
"""

from __future__ import annotations

import hashlib
import json
import os
import sys
import time

import numpy as np

REF = "/root/reference/pkg/src"
sys.dont_write_bytecode = True
sys.path.insert(0, REF)

from threadpoolctl import threadpool_limits  # noqa: E402

import hmatdag.accumulator as accm  # noqa: E402
import hmatdag.arith as arith  # noqa: E402
import hmatdag.hmatrix as hm  # noqa: E402
import hmatdag.problems as prob  # noqa: E402
import hmatdag.taskgraph as tg  # noqa: E402
import hmatdag.trees as trees  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


# ---------------------------------------------------------------------------
# problem definitions (BASELINE.json configs)
# ---------------------------------------------------------------------------

def exp_kernel(points, ell, perm):
    k = prob.PointKernel(points, lambda d: np.exp(-d / ell), diag_value=1.0 + 1e-2, scale=1.0)
    return prob.permuted(k, perm)


def weak_adm(t, s):
    return not t.indices.overlaps(s.indices)


def eta_adm(eta):
    return lambda t, s: trees.standard_admissible(t, s, eta)


def case_points(name):
    """(points, ell, n_min, adm, eps) for a named case."""
    if name == "c1":
        n = 2048
        return ((np.arange(n) + 0.5) / n)[:, None], 0.1, 64, weak_adm, 1e-6
    if name == "c2":
        g = (np.arange(128) + 0.5) / 128
        X, Y = np.meshgrid(g, g, indexing="ij")
        return np.column_stack([X.ravel(), Y.ravel()]), 0.2, 64, eta_adm(2.0), 1e-6
    if name in ("c3s", "c3"):
        rng = np.random.default_rng(0)
        p = rng.normal(size=(65536, 3))
        p /= np.linalg.norm(p, axis=1, keepdims=True)
        return p, 0.3, 64, eta_adm(2.0), 1e-5
    if name.startswith("c4_"):
        j = int(name[3:])
        rng = np.random.default_rng(1000 + j)
        x = np.sort(rng.uniform(size=4096))
        ell = float(rng.uniform(0.05, 0.5))
        return x[:, None], ell, 64, weak_adm, 1e-6
    if name == "c5s":
        rng = np.random.default_rng(0)
        return rng.uniform(size=(262144, 3)), 0.25, 128, eta_adm(2.0), 1e-4
    if name.startswith("c5_d"):  # diagonal sub-problem of c5 at depth d (tree order)
        d = int(name[4:])
        pts, ell, n_min, adm, eps = case_points("c5s")
        croot, perm = trees.build_cluster_tree(trees.Geometry(pts), n_min)
        node = croot
        for _ in range(d):
            node = node.children[0]
        a, b = node.indices.first, node.indices.last
        return pts[perm[a:b]], ell, n_min, adm, eps
    if name == "s1":  # small 1D HODLR
        n = 512
        return ((np.arange(n) + 0.5) / n)[:, None], 0.1, 16, weak_adm, 1e-6
    if name == "s2":  # small 2D grid, standard admissibility
        g = (np.arange(32) + 0.5) / 32
        X, Y = np.meshgrid(g, g, indexing="ij")
        return np.column_stack([X.ravel(), Y.ravel()]), 0.2, 16, eta_adm(2.0), 1e-6
    if name == "s5":  # small sphere, eta=2, eps 1e-5 (c3 shape, scaled down)
        rng = np.random.default_rng(0)
        p = rng.normal(size=(2048, 3))
        p /= np.linalg.norm(p, axis=1, keepdims=True)
        return p, 0.3, 32, eta_adm(2.0), 1e-5
    raise KeyError(name)


# ---------------------------------------------------------------------------
# serialisation helpers
# ---------------------------------------------------------------------------

def sha(text: str) -> str:
    return hashlib.sha256(text.encode()).hexdigest()


def multiset_digest(node_lines, src, dst):
    """Order-independent digest of a DAG for graphs too large to sort as
    strings (c5: 3.2M nodes, 207M edges): per-node h = blake2b-64 of its
    canonical line; nodes: (sum h, sum h*h) mod 2^64; edges: the same sums
    over e = h_u * 0x9E3779B97F4A7C15 + (h_v ^ (h_v >> 29)) * 0xBF58476D1CE4E5B9.
    Restated in paper_1911_07531_b200/taskgraph.py:multiset_digest."""
    h = np.fromiter((int.from_bytes(hashlib.blake2b(x.encode(), digest_size=8).digest(), "little")
                     for x in node_lines), dtype=np.uint64, count=len(node_lines))
    with np.errstate(over="ignore"):
        hu, hv = h[src], h[dst]
        e = hu * np.uint64(0x9E3779B97F4A7C15) + (hv ^ (hv >> np.uint64(29))) * np.uint64(0xBF58476D1CE4E5B9)
        out = [int(h.sum(dtype=np.uint64)), int((h * h).sum(dtype=np.uint64)),
               int(e.sum(dtype=np.uint64)), int((e * e).sum(dtype=np.uint64))]
    return [f"{x:016x}" for x in out]


def dag_digest(g):
    nodes = list(g.nodes)
    pos = {id(t): i for i, t in enumerate(nodes)}
    lines = [key_line(t.key()) for t in nodes]
    ne = sum(1 for _ in g.edges())
    src = np.empty(ne, dtype=np.int64)
    dst = np.empty(ne, dtype=np.int64)
    i = 0
    for u, v in g.edges():
        src[i] = pos[id(u)]
        dst[i] = pos[id(v)]
        i += 1
    return {"nodes": len(nodes), "edges": ne, "digest": multiset_digest(lines, src, dst)}


def block_table(root):
    rows = []
    for line in trees.serialize_block_tree(root).splitlines():
        rows.append([int(v) for v in line.split()])
    return np.asarray(rows, dtype=np.int64)


def key_line(k):
    kind, mids, uids, alpha = k
    return f"{kind}|{','.join(map(str, mids))}|{','.join(map(str, uids))}|{alpha!r}"


def dag_summary(g, full: bool):
    nodes = sorted(key_line(t.key()) for t in g.nodes)
    edges = sorted(f"{key_line(u.key())}>{key_line(v.key())}" for u, v in g.edges())
    d = {"nodes": len(nodes), "edges": len(edges),
         "nodes_sha": sha("\n".join(nodes)), "edges_sha": sha("\n".join(edges))}
    if full:
        d["node_lines"] = nodes
        d["edge_lines"] = edges
    return d


def leaf_arrays(H, nblocks):
    """Per-uid rank (-1 for dense/blocked) and per-leaf Frobenius norm."""
    rank = np.full(nblocks, -1, dtype=np.int64)
    fro = np.full(nblocks, np.nan)
    for leaf in H.leaves():
        u = leaf.block.uid
        if leaf.kind == hm.LOWRANK:
            rank[u] = leaf.rank
        fro[u] = leaf.frobenius()
    return rank, fro


def probe(H, x):
    return hm.hm_apply(H, x)


# ---------------------------------------------------------------------------
# case runners
# ---------------------------------------------------------------------------

def rsvd_lowrank(M, policy, seed):
    """Large-block compression used only for the c3 fixture (the reference's
    full-SVD assembly, hmatrix.py:133-138, needs ~1.9e14 flop at c3 and does
    not finish in a CPU session).  Randomized range finder with one power
    iteration, sketch doubled until its trailing singular value is below
    1e-3 of the cut, then the SVD of the projected block and the reference's
    own ``policy.keep`` (hmatrix.py:62-71) on those singular values.  The
    same recipe as the device assembly (paper_1911_07531_b200/assembly.py),
    restated independently; ``check_rsvd_sample`` compares it with the
    reference's ``dense_to_lowrank`` on a sample of blocks."""
    m, n = M.shape
    rng = np.random.default_rng(seed)
    s = min(m, n, 48)
    cut = policy.eps
    while True:
        G = rng.normal(size=(n, s))
        Q, _ = np.linalg.qr(M @ G)
        Q, _ = np.linalg.qr(M @ (M.T @ Q))
        W, S, Zt = np.linalg.svd(Q.T @ M, full_matrices=False)
        if S[-1] <= 1e-3 * cut * S[0] or s >= min(m, n):
            break
        s = min(min(m, n), 2 * s)
    r = policy.keep(S)
    return Q @ (W[:, :r] * S[:r]), Zt[:r].T.copy(), S


def assemble_fast(broot, kern, policy, small=128):
    """hm.assemble with rsvd_lowrank for admissible leaves with min(m,n) >
    small; smaller admissible leaves use the reference's dense_to_lowrank,
    dense leaves the reference kernel evaluation (hmatrix.py:227-248)."""
    A = hm.zeros(broot, policy)
    nlarge = 0
    for leaf in A.leaves():
        b = leaf.block
        rows = np.arange(b.row.indices.first, b.row.indices.last)
        cols = np.arange(b.col.indices.first, b.col.indices.last)
        M = kern.dense(rows, cols)
        if not b.admissible:
            leaf.D = np.ascontiguousarray(M, dtype=float)
        elif min(M.shape) <= small:
            leaf.set_lowrank(*hm.dense_to_lowrank(M, policy))
        else:
            U, V, _ = rsvd_lowrank(M, policy, 777 + b.uid)
            leaf.set_lowrank(U, V)
            nlarge += 1
    return A, nlarge


def check_rsvd_sample(broot, kern, policy, count=24, small=128):
    """Rank of rsvd_lowrank == rank of the reference's dense_to_lowrank on a
    seeded sample of large admissible blocks (full SVDs, the expensive pin)."""
    A = hm.zeros(broot, policy)
    big = [lf.block for lf in A.leaves() if lf.block.admissible
           and min(lf.block.nrows, lf.block.ncols) > small]
    pick = np.random.default_rng(5).choice(len(big), size=min(count, len(big)), replace=False)
    out = []
    for i in sorted(pick):
        b = big[i]
        M = kern.dense(np.arange(b.row.indices.first, b.row.indices.last),
                       np.arange(b.col.indices.first, b.col.indices.last))
        U, _ = hm.dense_to_lowrank(M, policy)
        Ur, _, _ = rsvd_lowrank(M, policy, 777 + b.uid)
        out.append((int(b.uid), int(M.shape[0]), int(M.shape[1]), int(U.shape[1]), int(Ur.shape[1])))
    return out


def run_case(name, numerics=True, modes=("std", "accu"), dag_modes=None, full_dag=False,
             store_blocks=True, n_probe=2, fast_assembly=False):
    t0 = time.time()
    pts, ell, n_min, adm, eps = case_points(name)
    geom = trees.Geometry(pts)
    croot, perm = trees.build_cluster_tree(geom, n_min)
    broot = trees.build_block_tree(croot, croot, adm)
    blocks = block_table(broot)
    nb = blocks.shape[0]
    meta = {"case": name, "n": int(len(pts)), "ell": ell, "n_min": n_min, "eps": eps,
            "n_blocks": int(nb), "n_leaves": int(blocks[:, 6].sum()),
            "n_admissible": int(blocks[:, 7].sum()),
            "cluster_sha": sha(trees.serialize_cluster_tree(croot)),
            "block_sha": sha(trees.serialize_block_tree(broot)),
            "perm_sha": sha(",".join(map(str, perm.tolist())))}
    arrays = {}
    if store_blocks:
        arrays["blocks"] = blocks
        arrays["perm"] = perm.astype(np.int64)
    print(f"[{name}] structure {time.time() - t0:.1f}s blocks={nb}", flush=True)

    dag_modes = dag_modes or []
    meta["dags"] = {}
    for mode, sp in dag_modes:
        t1 = time.time()
        g = tg.build_hlu_dag(broot, mode, sparsify=sp)
        tag = f"{mode}{'+sparsify' if sp else ''}"
        meta["dags"][tag] = dag_summary(g, full_dag)
        meta["dags"][tag]["build_s"] = time.time() - t1
        print(f"[{name}] dag {tag}: {meta['dags'][tag]['nodes']} / "
              f"{meta['dags'][tag]['edges']} in {time.time() - t1:.1f}s", flush=True)
        del g

    if numerics:
        pol = hm.TruncationPolicy.fixed_accuracy(eps)
        kern = exp_kernel(pts, ell, perm)
        t1 = time.time()
        hm.counters.reset()
        if fast_assembly:
            meta["rsvd_vs_reference_sample"] = check_rsvd_sample(broot, kern, pol)
            print(f"[{name}] rsvd sample {meta['rsvd_vs_reference_sample']}", flush=True)
            bad = [x for x in meta["rsvd_vs_reference_sample"] if x[3] != x[4]]
            if bad:
                raise SystemExit(f"rsvd ranks differ from dense_to_lowrank: {bad}")
            t1 = time.time()
            A0, meta["assembly_rsvd_blocks"] = assemble_fast(broot, kern, pol)
            meta["assembly"] = ("reference kernel evaluation; dense_to_lowrank for admissible "
                                "min(m,n)<=128, rsvd_lowrank above (make_golden.py)")
        else:
            A0 = hm.assemble(broot, kern, pol)
        meta["assembly_truncations"] = hm.counters.snapshot()[0]
        meta["assembly_s"] = time.time() - t1
        print(f"[{name}] assembly {time.time() - t1:.1f}s", flush=True)
        rA, fA = leaf_arrays(A0, nb)
        arrays["A_rank"], arrays["A_fro"] = rA, fA
        n = len(pts)
        rng = np.random.default_rng(12345)
        X = rng.normal(size=(n, n_probe))
        arrays["probe_x"] = X
        AX = probe(A0, X)
        arrays["probe_Ax"] = AX
        for mode in modes:
            A = A0.copy()
            L, U = hm.zeros(broot, pol), hm.zeros(broot, pol)
            hm.counters.reset()
            t2 = time.time()
            with threadpool_limits(limits=1):
                if mode == "std":
                    arith.hlu(A, L, U, pol)
                else:
                    accm.hlu_accu(A, L, U, accm.AccumulatorMap(), pol)
            dt = time.time() - t2
            tr, up = hm.counters.snapshot()
            rL, fL = leaf_arrays(L, nb)
            rU, fU = leaf_arrays(U, nb)
            LUX = probe(L, probe(U, X))
            res = float(np.linalg.norm(AX - LUX) / np.linalg.norm(AX))
            arrays[f"{mode}_L_rank"], arrays[f"{mode}_L_fro"] = rL, fL
            arrays[f"{mode}_U_rank"], arrays[f"{mode}_U_fro"] = rU, fU
            arrays[f"{mode}_probe_LUx"] = LUX
            arrays[f"{mode}_probe_Ux"] = probe(U, X)
            meta[f"{mode}_truncations"] = tr
            meta[f"{mode}_updates"] = up
            meta[f"{mode}_probe_residual"] = res
            meta[f"{mode}_hlu_s"] = dt
            print(f"[{name}] {mode} hlu {dt:.2f}s trunc={tr} upd={up} res={res:.3e}",
                  flush=True)
    np.savez_compressed(os.path.join(OUT, f"{name}.npz"), **arrays)
    with open(os.path.join(OUT, f"{name}.json"), "w") as f:
        json.dump(meta, f, indent=1, sort_keys=True)
    print(f"[{name}] done {time.time() - t0:.1f}s", flush=True)


def sample_leaves(H, nb, rng, count=12):
    """Entries of a seeded sample of leaves of a factor: ``count`` dense
    leaves (D) and ``count`` low-rank leaves of rank >= 1 (U, V), so that
    device factors can be compared entrywise per block (low-rank leaves
    through U V^T, which is what the factorization defines)."""
    dense, lowr = [], []
    for leaf in H.leaves():
        if leaf.kind == hm.LOWRANK:
            if leaf.rank > 0:
                lowr.append(leaf)
        else:
            dense.append(leaf)
    out = {"uid": [], "kind": [], "m": [], "n": [], "k": [], "vals": []}
    for group, kind in ((dense, 0), (lowr, 1)):
        if not group:
            continue
        pick = rng.choice(len(group), size=min(count, len(group)), replace=False)
        for i in sorted(pick):
            leaf = group[i]
            b = leaf.block
            out["uid"].append(b.uid)
            out["kind"].append(kind)
            out["m"].append(b.nrows)
            out["n"].append(b.ncols)
            if kind == 0:
                out["k"].append(0)
                out["vals"].append(np.asarray(leaf.D, dtype=float).ravel(order="F"))
            else:
                out["k"].append(leaf.rank)
                out["vals"].append(np.concatenate([np.asarray(leaf.U).ravel(order="F"),
                                                   np.asarray(leaf.V).ravel(order="F")]))
    meta = np.array([out["uid"], out["kind"], out["m"], out["n"], out["k"]], dtype=np.int64).T
    return meta, np.concatenate(out["vals"]) if out["vals"] else np.zeros(0)


def run_leaf_samples(name, fast_assembly, modes=("std", "accu")):
    """<name>_leaves.npz: sampled leaf entries of L and U of the reference's
    own factorization (same inputs as run_case), for per-block factor
    parity of the device (tests/test_hlu_gpu.py, bench.py)."""
    pts, ell, n_min, adm, eps = case_points(name)
    croot, perm = trees.build_cluster_tree(trees.Geometry(pts), n_min)
    broot = trees.build_block_tree(croot, croot, adm)
    nb = block_table(broot).shape[0]
    pol = hm.TruncationPolicy.fixed_accuracy(eps)
    kern = exp_kernel(pts, ell, perm)
    t0 = time.time()
    A0 = assemble_fast(broot, kern, pol)[0] if fast_assembly else hm.assemble(broot, kern, pol)
    print(f"[{name}_leaves] assembly {time.time() - t0:.1f}s", flush=True)
    arrays = {}
    for mode in modes:
        A = A0.copy()
        L, U = hm.zeros(broot, pol), hm.zeros(broot, pol)
        with threadpool_limits(limits=1):
            if mode == "std":
                arith.hlu(A, L, U, pol)
            else:
                accm.hlu_accu(A, L, U, accm.AccumulatorMap(), pol)
        for tag, H in (("L", L), ("U", U)):
            rng = np.random.default_rng(4242 + (tag == "U") + 2 * (mode == "accu"))
            m, v = sample_leaves(H, nb, rng)
            arrays[f"{mode}_{tag}_meta"], arrays[f"{mode}_{tag}_vals"] = m, v
        print(f"[{name}_leaves] {mode} done {time.time() - t0:.1f}s", flush=True)
    np.savez_compressed(os.path.join(OUT, f"{name}_leaves.npz"), **arrays)


def probe_vec(n):
    return np.random.default_rng(7).normal(size=(n, 2))


def truncate_inputs(i, m, n, K, decay):
    """Seeded inputs of truncate case i (restated in tests/test_oracle.py)."""
    r = np.random.default_rng(100 + i)
    U = r.normal(size=(m, K)) * np.exp(-decay * np.arange(K))[None, :]
    V = r.normal(size=(n, K))
    M = U @ V.T + 1e-3 * r.normal(size=(m, n)) * np.exp(-decay * K)
    return U, V, M


def run_truncate_cases():
    """Random truncate / dense_to_lowrank cases: inputs from seeds, outputs
    (rank, singular values of the reconstruction, product) from the reference."""
    out = {}
    specs = []
    rng = np.random.default_rng(2024)
    for i in range(24):
        m = int(rng.integers(8, 300))
        n = int(rng.integers(8, 300))
        K = int(rng.integers(1, 60))
        decay = float(rng.uniform(0.3, 3.0))
        specs.append((m, n, K, decay))
    for i, (m, n, K, decay) in enumerate(specs):
        U, V, M = truncate_inputs(i, m, n, K, decay)
        for eps in (1e-4, 1e-6, 1e-8):
            pol = hm.TruncationPolicy.fixed_accuracy(eps)
            Un, Vn = hm.truncate(U, V, pol)
            out[f"t{i}_{eps:g}_rank"] = np.array(Un.shape[1])
            out[f"t{i}_{eps:g}_probe"] = Un @ (Vn.T @ probe_vec(n))
        for eps in (1e-4, 1e-6):
            pol = hm.TruncationPolicy.fixed_accuracy(eps)
            W, Z = hm.dense_to_lowrank(M, pol)
            out[f"d{i}_{eps:g}_rank"] = np.array(W.shape[1])
            out[f"d{i}_{eps:g}_probe"] = W @ (Z.T @ probe_vec(n))
    # dense LU
    for i in range(4):
        r = np.random.default_rng(300 + i)
        n = (16, 33, 64, 128)[i]
        A = r.normal(size=(n, n)) + n * np.eye(n)
        Lr, Ur = arith.dense_lu(A)
        out[f"lu{i}_L"], out[f"lu{i}_U"] = Lr, Ur
    np.savez_compressed(os.path.join(OUT, "kernels.npz"), **out)
    with open(os.path.join(OUT, "kernels.json"), "w") as f:
        json.dump({"n_truncate": len(specs), "specs": specs}, f)
    print("[kernels] done", flush=True)


ALL_DAG = [("std", False), ("std", True), ("accu-combined", False),
           ("accu-merged", False), ("accu-merged", True)]


def run_roots():
    """Standalone multiply / triangular-solve DAGs (root tasks made by the
    reference's own factories, taskgraph.py:146-180, refined by its
    compute_dag, taskgraph.py:530-590) on the s2 structure."""
    pts, ell, n_min, adm, eps = case_points("s2")
    croot, perm = trees.build_cluster_tree(trees.Geometry(pts), n_min)
    b = trees.build_block_tree(croot, croot, adm)
    out = {}
    for mode in ("std", "accu-combined"):
        for op in ("hmul", "htrsl", "htrsu"):
            for sp in (False, True):
                if sp and mode != "std":
                    continue
                if op == "hmul":
                    root = tg._mul_task(1.0, b, b, b, (tg.MID_A, tg.MID_L, tg.MID_U), (0,), mode)
                elif op == "htrsl":
                    root = tg._solve_l_task(b, b, (tg.MID_L, tg.MID_A, tg.MID_U), (0,), mode)
                else:
                    root = tg._solve_u_task(b, b, (tg.MID_U, tg.MID_A, tg.MID_L), (0,), mode)
                g = tg.compute_dag(root, 0, sparsify=sp, mode=mode)
                out[f"{op}|{mode}{'+sparsify' if sp else ''}"] = dag_summary(g, False)
    with open(os.path.join(OUT, "roots.json"), "w") as f:
        json.dump(out, f, indent=1, sort_keys=True)


def main(argv):
    cases = argv or ["small"]
    for c in cases:
        if c == "small":
            run_truncate_cases()
            for s in ("s1", "s2", "s5"):
                run_case(s, dag_modes=ALL_DAG, full_dag=(s == "s1"))
        elif c == "c1":
            run_case("c1", dag_modes=ALL_DAG, full_dag=True)
        elif c == "c2":
            run_case("c2", dag_modes=ALL_DAG)
        elif c == "c3s":
            run_case("c3s", numerics=False, dag_modes=[("std", False), ("accu-merged", False)],
                     store_blocks=False)
        elif c == "c3":
            run_case("c3", dag_modes=[], fast_assembly=True)
        elif c.startswith("c5_d"):
            run_case(c, dag_modes=[("accu-merged", False)], modes=("accu",), fast_assembly=True)
        elif c == "c4":
            for j in range(4):
                run_case(f"c4_{j}", dag_modes=[("std", False), ("accu-merged", False)])
        elif c in ("c5dag", "c5dag_merged"):
            # reference std (478 s, ~17 GB) or accu-merged (757 s, 17.4 GB)
            # DAG of config 5, digest only
            pts, ell, n_min, adm, eps = case_points("c5s")
            croot, perm = trees.build_cluster_tree(trees.Geometry(pts), n_min)
            broot = trees.build_block_tree(croot, croot, adm)
            path = os.path.join(OUT, "c5dag.json")
            out = json.load(open(path)) if os.path.exists(path) else {}
            modes = ("accu-merged",) if c == "c5dag_merged" else ("std",)
            for mode in modes:
                t1 = time.time()
                g = tg.build_hlu_dag(broot, mode)
                out[mode] = dag_digest(g)
                out[mode]["build_s"] = time.time() - t1
                print(f"[c5dag] {mode} {out[mode]}", flush=True)
                del g
            with open(path, "w") as f:
                json.dump(out, f, indent=1, sort_keys=True)
        elif c.startswith("leaves_"):
            nm = c.split("_", 1)[1]
            run_leaf_samples(nm, fast_assembly=nm in ("c3",) or nm.startswith("c5_d"),
                             modes=("accu",) if nm.startswith("c5_d") else ("std", "accu"))
        elif c == "roots":
            run_roots()
        elif c == "c5s":
            run_case("c5s", numerics=False, dag_modes=[], store_blocks=False)
        else:
            raise SystemExit(f"unknown case {c}")


if __name__ == "__main__":
    main(sys.argv[1:])
