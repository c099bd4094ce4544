"""CPU oracle: numpy restatement of the reference H-LU numerics.

TEST INFRASTRUCTURE ONLY.  Nothing in the product package imports this
module; only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline
leg use it, and only as the checker / CPU baseline.

It restates, over a flat block table instead of the reference's object
tree, the algorithm of the reference package ``hmatdag``
(/root/reference/pkg/src/hmatdag, pure Python over numpy/scipy):

  build_cluster_tree   trees.py:104-134
  standard admissible  trees.py:137-142
  build_block_tree     trees.py:181-199
  PointKernel/permuted problems.py:43-53, 78-81
  keep                 hmatrix.py:62-71
  truncate             hmatrix.py:113-130
  dense_to_lowrank     hmatrix.py:133-138
  assemble / zeros     hmatrix.py:227-263
  hm_apply(_t)         hmatrix.py:286-315
  hm_solve_*           hmatrix.py:318-341
  product_payload      hmatrix.py:367-417
  fold / scatter       hmatrix.py:420-448
  hmul/dense_lu/hlu/htrsl/htrsu            arith.py:40-140
  Accumulator/add/shift/apply/hlu_accu/... accumulator.py:41-235

Third-party arithmetic: numpy 2.3 / scipy 1.18 (OpenBLAS 0.3.30), the
reference's unpinned deps (pkg/pyproject.toml:10-13).  The same numpy/scipy
calls are issued in the same order as the reference, so on this machine the
oracle reproduces the reference bit for bit; tests/test_oracle.py pins it
against the fixtures of tests/golden/make_golden.py (reference run).
"""

from __future__ import annotations

import numpy as np
import scipy.linalg as sla

ZERO_CUTOFF = 1e-14   # hmatrix.py:29
PIVOT_CUTOFF = 1e-14  # arith.py:33


class OracleError(RuntimeError):
    pass


class SingularPivot(OracleError):
    pass


# ---------------------------------------------------------------------------
# structure (trees.py)
# ---------------------------------------------------------------------------

class ClusterTable:
    """Flat binary cluster tree: arrays indexed by pre-order uid."""

    def __init__(self, first, last, lo, hi, kids, perm):
        self.first, self.last = first, last
        self.lo, self.hi = lo, hi
        self.kids = kids          # list: () or (left, right)
        self.perm = perm          # perm[new] = original


def cluster_tree(points, n_min):
    """trees.py:104-134, iteratively (explicit stack, same pre-order)."""
    if n_min < 1:
        raise ValueError("n_min must be >= 1")
    pts = np.atleast_2d(np.asarray(points, dtype=float))
    order = np.arange(pts.shape[0], dtype=np.intp)
    first, last, lo, hi, kids = [], [], [], [], []
    stack = [(0, pts.shape[0], None)]
    while stack:
        a, b, parent = stack.pop()
        uid = len(first)
        if parent is not None:
            kids[parent[0]][parent[1]] = uid
        sub = pts[order[a:b]]
        blo, bhi = sub.min(axis=0), sub.max(axis=0)
        first.append(a)
        last.append(b)
        lo.append(np.asarray(blo, dtype=float))
        hi.append(np.asarray(bhi, dtype=float))
        kids.append([])
        if b - a > n_min:
            ax = int(np.argmax(bhi - blo))
            key = np.argsort(sub[:, ax], kind="stable")
            order[a:b] = order[a:b][key]
            mid = a + (b - a + 1) // 2
            kids[uid] = [None, None]
            stack.append((mid, b, (uid, 1)))
            stack.append((a, mid, (uid, 0)))
    return ClusterTable(np.array(first), np.array(last), lo, hi,
                        [tuple(k) for k in kids], order)


def adm_standard(ct, eta):
    """trees.py:137-142 (BBox.diameter/dist trees.py:54-59)."""
    def f(t, s):
        d = float(np.linalg.norm(np.maximum(0.0, np.maximum(ct.lo[s] - ct.hi[t],
                                                            ct.lo[t] - ct.hi[s]))))
        dt = float(np.linalg.norm(ct.hi[t] - ct.lo[t]))
        ds = float(np.linalg.norm(ct.hi[s] - ct.lo[s]))
        return min(dt, ds) <= eta * d and d > 0.0
    return f


def adm_weak(ct):
    """HODLR: admissible iff the index ranges do not overlap (trees.py:38-39)."""
    def f(t, s):
        return not (ct.first[t] < ct.last[s] and ct.first[s] < ct.last[t])
    return f


class BlockTable:
    """Flat block tree (pre-order uid, row-major children)."""

    def __init__(self, n):
        self.r0 = np.zeros(n, dtype=np.int64)
        self.r1 = np.zeros(n, dtype=np.int64)
        self.c0 = np.zeros(n, dtype=np.int64)
        self.c1 = np.zeros(n, dtype=np.int64)
        self.adm = np.zeros(n, dtype=bool)
        self.parent = np.full(n, -1, dtype=np.int64)
        self.kids = [()] * n  # () or (k00, k01, k10, k11)

    def leaf(self, u):
        return not self.kids[u]

    def shape(self, u):
        return int(self.r1[u] - self.r0[u]), int(self.c1[u] - self.c0[u])

    def child(self, u, i, j):
        return self.kids[u][2 * i + j]

    def leaves(self, u):
        out, stack = [], [u]
        while stack:
            v = stack.pop()
            if self.leaf(v):
                out.append(v)
            else:
                stack.extend(reversed(self.kids[v]))
        return out

    def table(self):
        """serialize_block_tree rows: uid parent r0 r1 c0 c1 leaf adm."""
        n = len(self.r0)
        return np.column_stack([np.arange(n), self.parent, self.r0, self.r1, self.c0, self.c1,
                                [int(self.leaf(u)) for u in range(n)], self.adm.astype(int)])


def block_tree(ct, adm):
    """trees.py:181-199 with an explicit stack (same uids)."""
    recs = []  # (t, s, parent, adm, kids)
    stack = [(0, 0, -1, None)]
    while stack:
        t, s, par, slot = stack.pop()
        uid = len(recs)
        a = bool(adm(t, s))
        rec = [t, s, par, a, ()]
        recs.append(rec)
        if slot is not None:
            recs[par][4][slot] = uid
        tk, sk = ct.kids[t], ct.kids[s]
        if not (a or not tk or not sk):
            rec[4] = [None] * (len(tk) * len(sk))
            cells = [(ti, sj) for ti in tk for sj in sk]
            for idx in reversed(range(len(cells))):
                stack.append((cells[idx][0], cells[idx][1], uid, idx))
    bt = BlockTable(len(recs))
    for u, (t, s, par, a, kids) in enumerate(recs):
        bt.r0[u], bt.r1[u] = ct.first[t], ct.last[t]
        bt.c0[u], bt.c1[u] = ct.first[s], ct.last[s]
        bt.adm[u], bt.parent[u] = a, par
        bt.kids[u] = tuple(kids)
    return bt


# ---------------------------------------------------------------------------
# kernel (problems.py)
# ---------------------------------------------------------------------------

def exp_kernel_dense(points, perm, ell, I, J, diag=1.0 + 1e-2, scale=1.0):
    """PointKernel(points, exp(-d/ell), diag) composed with permuted(perm)."""
    I = np.asarray(perm, dtype=np.intp)[np.asarray(I, dtype=np.intp)]
    J = np.asarray(perm, dtype=np.intp)[np.asarray(J, dtype=np.intp)]
    xi, xj = points[I], points[J]
    d = np.linalg.norm(xi[:, None, :] - xj[None, :, :], axis=-1)
    vals = scale * np.exp(-d / ell)
    return np.where(I[:, None] == J[None, :], diag, vals)


# ---------------------------------------------------------------------------
# rank control and leaf kernels (hmatrix.py)
# ---------------------------------------------------------------------------

class Policy:
    def __init__(self, mode="exact", eps=None, k=None):
        self.mode, self.eps, self.k = mode, eps, k

    def keep(self, sigma):
        if sigma.size == 0 or sigma[0] <= 0.0:
            return 0
        if self.mode == "rank":
            r = min(self.k, sigma.size)
            return int(np.count_nonzero(sigma[:r] > ZERO_CUTOFF * sigma[0]))
        cut = self.eps if self.mode == "accuracy" else ZERO_CUTOFF
        return int(np.count_nonzero(sigma > cut * sigma[0]))


class Counters:
    """Reference counters (hmatrix.py:84-110) plus algorithmic flops of the
    op trace with SURVEY.md §8d formulas (the device counts the same way)."""

    def __init__(self):
        self.truncations = 0
        self.updates = 0
        self.flops = 0.0


COUNT = Counters()


def truncate(U, V, pol):
    if U.shape[1] != V.shape[1]:
        raise ValueError("non-conformal low-rank factors")
    if U.shape[1] == 0:
        return U, V
    COUNT.truncations += 1
    Qu, Ru = np.linalg.qr(U)
    Qv, Rv = np.linalg.qr(V)
    W, s, Zt = np.linalg.svd(Ru @ Rv.T)
    r = pol.keep(s)
    m, K = U.shape
    n = V.shape[0]
    p, q = Ru.shape[0], Rv.shape[0]
    COUNT.flops += (_qr_f(m, K) + _qr_f(n, K) + 2.0 * p * q * K + _svd_f(p, q)
                    + 2.0 * m * p * r + 2.0 * n * q * r)
    return Qu @ (W[:, :r] * s[:r]), Qv @ Zt[:r].T


def _qr_f(m, k):
    return 2.0 * (2.0 * m * k * k - 2.0 * k ** 3 / 3.0)


def _svd_f(m, n):
    l, s = max(m, n), min(m, n)
    return 4.0 * l * s * s + 22.0 * s ** 3


def _gemm_f(m, n, k):
    return 2.0 * m * n * k


def dense_to_lowrank(M, pol):
    COUNT.truncations += 1
    COUNT.flops += _svd_f(*M.shape)
    W, s, Zt = np.linalg.svd(M, full_matrices=False)
    r = pol.keep(s)
    return W[:, :r] * s[:r], Zt[:r].T


def dense_lu(A):
    n = A.shape[0]
    if A.shape[1] != n:
        raise ValueError("LU needs a square block")
    U = A.copy()
    L = np.eye(n)
    scale = np.linalg.norm(A)
    COUNT.flops += 2.0 / 3.0 * n ** 3
    for k in range(n):
        piv = U[k, k]
        if abs(piv) <= PIVOT_CUTOFF * scale:
            raise SingularPivot(f"pivot {piv:.3e} at {k}")
        L[k + 1:, k] = U[k + 1:, k] / piv
        U[k + 1:, k:] -= np.outer(L[k + 1:, k], U[k, k:])
        U[k + 1:, k] = 0.0
    return L, U


# H-matrix storage: dict uid -> ("D", M) | ("R", U, V) for leaves of bt.

class HM:
    def __init__(self, bt, leaves):
        self.bt = bt
        self.lv = leaves

    def copy(self):
        out = {}
        for u, x in self.lv.items():
            out[u] = ("D", x[1].copy()) if x[0] == "D" else ("R", x[1].copy(), x[2].copy())
        return HM(self.bt, out)

    def to_dense(self, u=0):
        bt = self.bt
        m, n = bt.shape(u)
        out = np.zeros((m, n))
        for v in bt.leaves(u):
            x = self.lv[v]
            blk = x[1] if x[0] == "D" else x[1] @ x[2].T
            out[bt.r0[v] - bt.r0[u]:bt.r1[v] - bt.r0[u],
                bt.c0[v] - bt.c0[u]:bt.c1[v] - bt.c0[u]] = blk
        return out

    def rank(self, u):
        x = self.lv[u]
        return x[1].shape[1] if x[0] == "R" else -1


def assemble(bt, dense_fn, pol):
    """hmatrix.py:227-248 (leaf order is irrelevant: each leaf independent)."""
    lv = {}
    for u in bt.leaves(0):
        M = dense_fn(np.arange(bt.r0[u], bt.r1[u]), np.arange(bt.c0[u], bt.c1[u]))
        lv[u] = ("R", *dense_to_lowrank(M, pol)) if bt.adm[u] else \
            ("D", np.ascontiguousarray(M, dtype=float))
    return HM(bt, lv)


def rsvd_lowrank(M, pol, seed):
    """Compression of a large admissible block for configs whose full-SVD
    assembly (hmatrix.py:133-138) is infeasible on the CPU (c3: ~1.9e14
    flop).  Randomized range finder with one power iteration, the sketch
    doubled until its trailing singular value is below 1e-3 of the cut, then
    the SVD of the projected block and ``keep`` (hmatrix.py:62-71).  Same
    recipe as tests/golden/make_golden.py:rsvd_lowrank, which made the c3 /
    c5_d3 fixtures and checked its ranks against the reference's
    dense_to_lowrank on sampled blocks."""
    m, n = M.shape
    rng = np.random.default_rng(seed)
    s = min(m, n, 48)
    cut = pol.eps if pol.mode == "accuracy" else ZERO_CUTOFF
    while True:
        G = rng.normal(size=(n, s))
        Q, _ = np.linalg.qr(M @ G)
        Q, _ = np.linalg.qr(M @ (M.T @ Q))
        W, S, Zt = np.linalg.svd(Q.T @ M, full_matrices=False)
        if S[-1] <= 1e-3 * cut * S[0] or s >= min(m, n):
            break
        s = min(min(m, n), 2 * s)
    COUNT.truncations += 1
    r = pol.keep(S)
    return Q @ (W[:, :r] * S[:r]), Zt[:r].T.copy()


def assemble_leaves(bt, dense_fn, pol, leaves, small=128):
    """Leaves ``leaves`` of the fast assembly: dense leaves by kernel
    evaluation, admissible leaves with min(m, n) <= small by
    dense_to_lowrank (hmatrix.py:133-138), larger ones by rsvd_lowrank
    (seed 777 + uid, as in the fixtures).  Leaves are independent, so a
    caller may split them over processes."""
    lv = {}
    for u in leaves:
        M = dense_fn(np.arange(bt.r0[u], bt.r1[u]), np.arange(bt.c0[u], bt.c1[u]))
        if not bt.adm[u]:
            lv[u] = ("D", np.ascontiguousarray(M, dtype=float))
        elif min(M.shape) <= small:
            lv[u] = ("R", *dense_to_lowrank(M, pol))
        else:
            lv[u] = ("R", *rsvd_lowrank(M, pol, 777 + int(u)))
    return lv


def zeros(bt):
    lv = {}
    for u in bt.leaves(0):
        m, n = bt.shape(u)
        lv[u] = ("R", np.zeros((m, 0)), np.zeros((n, 0))) if bt.adm[u] else ("D", np.zeros((m, n)))
    return HM(bt, lv)


def _off(bt, parent, child):
    return int(bt.r0[child] - bt.r0[parent]), int(bt.c0[child] - bt.c0[parent])


def apply(H, u, X):
    """hm_apply (hmatrix.py:286-299): H[u] @ X."""
    bt = H.bt
    if bt.leaf(u):
        x = H.lv[u]
        m, n = bt.shape(u)
        if x[0] == "D":
            COUNT.flops += _gemm_f(m, X.shape[1], n)
            return x[1] @ X
        COUNT.flops += 2.0 * x[1].shape[1] * X.shape[1] * (m + n)
        return x[1] @ (x[2].T @ X)
    out = np.zeros((bt.shape(u)[0], X.shape[1]))
    for ch in bt.kids[u]:
        r0, c0 = _off(bt, u, ch)
        m, n = bt.shape(ch)
        out[r0:r0 + m] += apply(H, ch, X[c0:c0 + n])
    return out


def apply_t(H, u, X):
    """hm_apply_t (hmatrix.py:302-315): H[u].T @ X."""
    bt = H.bt
    if bt.leaf(u):
        x = H.lv[u]
        m, n = bt.shape(u)
        if x[0] == "D":
            COUNT.flops += _gemm_f(n, X.shape[1], m)
            return x[1].T @ X
        COUNT.flops += 2.0 * x[1].shape[1] * X.shape[1] * (m + n)
        return x[2] @ (x[1].T @ X)
    out = np.zeros((bt.shape(u)[1], X.shape[1]))
    for ch in bt.kids[u]:
        r0, c0 = _off(bt, u, ch)
        m, n = bt.shape(ch)
        out[c0:c0 + n] += apply_t(H, ch, X[r0:r0 + m])
    return out


def solve_lower(L, u, Y):
    """hm_solve_lower (hmatrix.py:318-328)."""
    bt = L.bt
    if bt.leaf(u):
        x = L.lv[u]
        if x[0] != "D":
            raise ValueError("triangular solve on a low-rank diagonal block")
        COUNT.flops += float(x[1].shape[0]) ** 2 * Y.shape[1]
        return sla.solve_triangular(x[1], Y, lower=True, unit_diagonal=True)
    k00, _, k10, k11 = bt.kids[u]
    n0 = bt.shape(k00)[0]
    X0 = solve_lower(L, k00, Y[:n0])
    X1 = solve_lower(L, k11, Y[n0:] - apply(L, k10, X0))
    return np.vstack([X0, X1])


def solve_upper(U, u, Y):
    """Back substitution U X = Y over the block tree: the non-transposed
    counterpart of hm_solve_upper_t (hmatrix.py:331-341) for the solve
    phase (no reference entry point; checked by the residual in tests)."""
    bt = U.bt
    if bt.leaf(u):
        x = U.lv[u]
        if x[0] != "D":
            raise ValueError("triangular solve on a low-rank diagonal block")
        COUNT.flops += float(x[1].shape[0]) ** 2 * Y.shape[1]
        return sla.solve_triangular(x[1], Y, lower=False)
    k00, k01, _, k11 = bt.kids[u]
    n0 = bt.shape(k00)[0]
    X1 = solve_upper(U, k11, Y[n0:])
    X0 = solve_upper(U, k00, Y[:n0] - apply(U, k01, X1))
    return np.vstack([X0, X1])


def solve_upper_t(U, u, Y):
    """hm_solve_upper_t (hmatrix.py:331-341)."""
    bt = U.bt
    if bt.leaf(u):
        x = U.lv[u]
        if x[0] != "D":
            raise ValueError("triangular solve on a low-rank diagonal block")
        COUNT.flops += float(x[1].shape[0]) ** 2 * Y.shape[1]
        return sla.solve_triangular(x[1], Y, trans="T", lower=False)
    k00, k01, _, k11 = bt.kids[u]
    n0 = bt.shape(k00)[0]
    W0 = solve_upper_t(U, k00, Y[:n0])
    W1 = solve_upper_t(U, k11, Y[n0:] - apply_t(U, k01, W0))
    return np.vstack([W0, W1])


# payloads: ("D", M) | ("R", U, V)

def p_dense(p):
    return p[1] if p[0] == "D" else p[1] @ p[2].T


def p_shape(p):
    return p[1].shape if p[0] == "D" else (p[1].shape[0], p[2].shape[0])


def p_restrict(p, r0, nr, c0, nc):
    if p[0] == "D":
        return ("D", p[1][r0:r0 + nr, c0:c0 + nc])
    return ("R", p[1][r0:r0 + nr], p[2][c0:c0 + nc])


def product(alpha, A, ua, B, ub, pol):
    """product_payload (hmatrix.py:367-417) for blocks ua of A and ub of B."""
    bt = A.bt
    if bt.shape(ua)[1] != B.bt.shape(ub)[0]:
        raise ValueError("non-conformal product")
    la, lb = bt.leaf(ua), B.bt.leaf(ub)
    xa = A.lv[ua] if la else None
    xb = B.lv[ub] if lb else None
    if la and xa[0] == "R":
        return ("R", alpha * xa[1], apply_t(B, ub, xa[2]))
    if lb and xb[0] == "R":
        return ("R", apply(A, ua, alpha * xb[1]), xb[2])
    if la and lb:
        COUNT.flops += _gemm_f(xa[1].shape[0], xb[1].shape[1], xa[1].shape[1])
        return ("D", alpha * (xa[1] @ xb[1]))
    if la:
        return ("D", apply_t(B, ub, alpha * xa[1].T).T)
    if lb:
        return ("D", apply(A, ua, alpha * xb[1]))
    m, n = bt.shape(ua)[0], B.bt.shape(ub)[1]
    us, vs, dacc = [], [], None
    for i in range(2):
        for j in range(2):
            for l in range(2):
                a_il = A.bt.child(ua, i, l)
                b_lj = B.bt.child(ub, l, j)
                q = product(alpha, A, a_il, B, b_lj, pol)
                r0 = int(bt.r0[a_il] - bt.r0[ua])
                c0 = int(B.bt.c0[b_lj] - B.bt.c0[ub])
                if q[0] == "D":
                    if dacc is None:
                        dacc = np.zeros((m, n))
                    dacc[r0:r0 + q[1].shape[0], c0:c0 + q[1].shape[1]] += q[1]
                elif q[1].shape[1]:
                    ue = np.zeros((m, q[1].shape[1]))
                    ue[r0:r0 + q[1].shape[0]] = q[1]
                    ve = np.zeros((n, q[2].shape[1]))
                    ve[c0:c0 + q[2].shape[0]] = q[2]
                    us.append(ue)
                    vs.append(ve)
    if dacc is not None:
        if us:
            Ku = sum(x.shape[1] for x in us)
            COUNT.flops += _gemm_f(m, n, Ku)
            dacc += np.hstack(us) @ np.hstack(vs).T
        return ("D", dacc)
    if not us:
        return ("R", np.zeros((m, 0)), np.zeros((n, 0)))
    return ("R", *truncate(np.hstack(us), np.hstack(vs), pol))


def fold_leaf(C, uc, p, pol):
    """fold_payload_into_leaf (hmatrix.py:420-437)."""
    if p_shape(p) != C.bt.shape(uc):
        raise ValueError("payload does not match destination block")
    COUNT.updates += 1
    x = C.lv[uc]
    if x[0] == "D":
        if p[0] == "R":
            COUNT.flops += _gemm_f(p[1].shape[0], p[2].shape[0], p[1].shape[1])
        x[1][...] += p_dense(p)
        return
    if p[0] == "D":
        COUNT.flops += _gemm_f(x[1].shape[0], x[2].shape[0], x[1].shape[1])
        C.lv[uc] = ("R", *dense_to_lowrank(x[1] @ x[2].T + p[1], pol))
    else:
        C.lv[uc] = ("R", *truncate(np.hstack([x[1], p[1]]), np.hstack([x[2], p[2]]), pol))


def scatter(C, uc, p, pol):
    """scatter_payload (hmatrix.py:440-448)."""
    bt = C.bt
    if bt.leaf(uc):
        fold_leaf(C, uc, p, pol)
        return
    for ch in bt.kids[uc]:
        r0, c0 = _off(bt, uc, ch)
        m, n = bt.shape(ch)
        scatter(C, ch, p_restrict(p, r0, m, c0, n), pol)


# ---------------------------------------------------------------------------
# standard recursive arithmetic (arith.py)
# ---------------------------------------------------------------------------

def hmul(alpha, A, ua, B, ub, C, uc, pol):
    if alpha == 0.0:
        return
    bt = C.bt
    if not (A.bt.leaf(ua) or B.bt.leaf(ub) or bt.leaf(uc)):
        for i in range(2):
            for j in range(2):
                for l in range(2):
                    hmul(alpha, A, A.bt.child(ua, i, l), B, B.bt.child(ub, l, j),
                         C, bt.child(uc, i, j), pol)
        return
    scatter(C, uc, product(alpha, A, ua, B, ub, pol), pol)


def hlu(A, L, U, u, pol):
    bt = A.bt
    if not bt.leaf(u):
        a00, a01, a10, a11 = bt.kids[u]
        hlu(A, L, U, a00, pol)
        htrsu(U, a00, A, a10, L, pol)
        htrsl(L, a00, A, a01, U, pol)
        hmul(-1.0, L, a10, U, a01, A, a11, pol)
        hlu(A, L, U, a11, pol)
        return
    x = A.lv[u]
    if x[0] != "D":
        raise ValueError("diagonal leaf must be dense for factorization")
    Ld, Ud = dense_lu(x[1])
    L.lv[u] = ("D", Ld)
    U.lv[u] = ("D", Ud)


def htrsl(L, ul, M, um, X, pol):
    """Solve L X = M on block um (arith.py:97-117); M consumed."""
    bt = M.bt
    if not bt.leaf(um):
        l00, _, l10, l11 = bt.kids[ul]
        m00, m01, m10, m11 = bt.kids[um]
        htrsl(L, l00, M, m00, X, pol)
        htrsl(L, l00, M, m01, X, pol)
        hmul(-1.0, L, l10, X, m00, M, m10, pol)
        hmul(-1.0, L, l10, X, m01, M, m11, pol)
        htrsl(L, l11, M, m10, X, pol)
        htrsl(L, l11, M, m11, X, pol)
        return
    x = M.lv[um]
    if x[0] == "D":
        X.lv[um] = ("D", solve_lower(L, ul, x[1]))
    else:
        X.lv[um] = ("R", solve_lower(L, ul, x[1]), x[2].copy())


def htrsu(U, uu, M, um, X, pol):
    """Solve X U = M on block um (arith.py:120-140); M consumed."""
    bt = M.bt
    if not bt.leaf(um):
        u00, u01, _, u11 = bt.kids[uu]
        m00, m01, m10, m11 = bt.kids[um]
        htrsu(U, u00, M, m00, X, pol)
        htrsu(U, u00, M, m10, X, pol)
        hmul(-1.0, X, m00, U, u01, M, m01, pol)
        hmul(-1.0, X, m10, U, u01, M, m11, pol)
        htrsu(U, u11, M, m01, X, pol)
        htrsu(U, u11, M, m11, X, pol)
        return
    x = M.lv[um]
    if x[0] == "D":
        X.lv[um] = ("D", solve_upper_t(U, uu, x[1].T).T)
    else:
        X.lv[um] = ("R", x[1].copy(), solve_upper_t(U, uu, x[2]))


# ---------------------------------------------------------------------------
# accumulator arithmetic (accumulator.py)
# ---------------------------------------------------------------------------

class Accs:
    """uid -> [umat, pending]; umat None | payload (accumulator.py:41-105)."""

    def __init__(self):
        self.d = {}

    def get(self, u):
        return self.d.get(u)

    def make(self, u):
        return self.d.setdefault(u, [None, []])


def acc_fold(acc, p, pol):
    """Accumulator.fold (accumulator.py:60-76)."""
    COUNT.updates += 1
    if acc[0] is None:
        acc[0] = ("D", p[1].copy()) if p[0] == "D" else ("R", p[1], p[2])
        return
    if acc[0][0] == "D" or p[0] == "D":
        for y in (acc[0], p):
            if y[0] == "R":
                COUNT.flops += _gemm_f(y[1].shape[0], y[2].shape[0], y[1].shape[1])
        acc[0] = ("D", p_dense(acc[0]) + p_dense(p))
        return
    acc[0] = ("R", *truncate(np.hstack([acc[0][1], p[1]]), np.hstack([acc[0][2], p[2]]), pol))


def add_upd(alpha, A, ua, B, ub, C, uc, accs, pol):
    """accumulator.py:108-125."""
    if alpha == 0.0:
        return
    acc = accs.make(uc)
    if not (A.bt.leaf(ua) or B.bt.leaf(ub) or C.bt.leaf(uc)):
        acc[1].append((alpha, A, ua, B, ub))
        return
    acc_fold(acc, product(alpha, A, ua, B, ub, pol), pol)


def shift_upd(C, uc, accs, pol):
    """accumulator.py:128-145."""
    bt = C.bt
    if bt.leaf(uc):
        raise ValueError("shift target must be a structured block")
    acc = accs.get(uc)
    if acc is None:
        return
    umat, pending = acc[0], acc[1]
    acc[0], acc[1] = None, []
    for i in range(2):
        for j in range(2):
            ch = bt.child(uc, i, j)
            if umat is not None:
                r0, c0 = _off(bt, uc, ch)
                m, n = bt.shape(ch)
                acc_fold(accs.make(ch), p_restrict(umat, r0, m, c0, n), pol)
            for alpha, A, ua, B, ub in pending:
                for l in range(2):
                    add_upd(alpha, A, A.bt.child(ua, i, l), B, B.bt.child(ub, l, j), C, ch,
                            accs, pol)


def apply_upd(C, uc, accs, pol):
    """accumulator.py:148-161."""
    bt = C.bt
    if not bt.leaf(uc):
        shift_upd(C, uc, accs, pol)
        for ch in bt.kids[uc]:
            apply_upd(C, ch, accs, pol)
        return
    acc = accs.get(uc)
    if acc is None:
        return
    umat = acc[0]
    acc[0], acc[1] = None, []
    if umat is not None:
        fold_leaf(C, uc, umat, pol)


def hlu_accu(A, L, U, u, accs, pol):
    bt = A.bt
    if not bt.leaf(u):
        shift_upd(A, u, accs, pol)
        a00, a01, a10, a11 = bt.kids[u]
        hlu_accu(A, L, U, a00, accs, pol)
        htrsu_accu(U, a00, A, a10, L, accs, pol)
        htrsl_accu(L, a00, A, a01, U, accs, pol)
        add_upd(-1.0, L, a10, U, a01, A, a11, accs, pol)
        hlu_accu(A, L, U, a11, accs, pol)
        return
    apply_upd(A, u, accs, pol)
    x = A.lv[u]
    if x[0] != "D":
        raise ValueError("diagonal leaf must be dense for factorization")
    Ld, Ud = dense_lu(x[1])
    L.lv[u] = ("D", Ld)
    U.lv[u] = ("D", Ud)


def htrsl_accu(L, ul, M, um, X, accs, pol):
    bt = M.bt
    if not bt.leaf(um):
        shift_upd(M, um, accs, pol)
        l00, _, l10, l11 = bt.kids[ul]
        m00, m01, m10, m11 = bt.kids[um]
        htrsl_accu(L, l00, M, m00, X, accs, pol)
        htrsl_accu(L, l00, M, m01, X, accs, pol)
        add_upd(-1.0, L, l10, X, m00, M, m10, accs, pol)
        add_upd(-1.0, L, l10, X, m01, M, m11, accs, pol)
        htrsl_accu(L, l11, M, m10, X, accs, pol)
        htrsl_accu(L, l11, M, m11, X, accs, pol)
        return
    apply_upd(M, um, accs, pol)
    x = M.lv[um]
    if x[0] == "D":
        X.lv[um] = ("D", solve_lower(L, ul, x[1]))
    else:
        X.lv[um] = ("R", solve_lower(L, ul, x[1]), x[2].copy())


def htrsu_accu(U, uu, M, um, X, accs, pol):
    bt = M.bt
    if not bt.leaf(um):
        shift_upd(M, um, accs, pol)
        u00, u01, _, u11 = bt.kids[uu]
        m00, m01, m10, m11 = bt.kids[um]
        htrsu_accu(U, u00, M, m00, X, accs, pol)
        htrsu_accu(U, u00, M, m10, X, accs, pol)
        add_upd(-1.0, X, m00, U, u01, M, m01, accs, pol)
        add_upd(-1.0, X, m10, U, u01, M, m11, accs, pol)
        htrsu_accu(U, u11, M, m01, X, accs, pol)
        htrsu_accu(U, u11, M, m11, X, accs, pol)
        return
    apply_upd(M, um, accs, pol)
    x = M.lv[um]
    if x[0] == "D":
        X.lv[um] = ("D", solve_upper_t(U, uu, x[1].T).T)
    else:
        X.lv[um] = ("R", x[1].copy(), solve_upper_t(U, uu, x[2]))


# ---------------------------------------------------------------------------
# drivers used by tests / bench cpu_baseline
# ---------------------------------------------------------------------------

def factor(A, mode, pol):
    """Factor a copy of A; returns (L, U, truncations, updates)."""
    W = A.copy()
    L, U = zeros(A.bt), zeros(A.bt)
    COUNT.truncations = COUNT.updates = 0
    COUNT.flops = 0.0
    if mode == "std":
        hlu(W, L, U, 0, pol)
    else:
        hlu_accu(W, L, U, 0, Accs(), pol)
    return L, U, COUNT.truncations, COUNT.updates


def leaf_arrays(H):
    n = len(H.bt.r0)
    rank = np.full(n, -1, dtype=np.int64)
    fro = np.full(n, np.nan)
    for u, x in H.lv.items():
        if x[0] == "R":
            rank[u] = x[1].shape[1]
            g = (x[1].T @ x[1]) * (x[2].T @ x[2])
            fro[u] = float(np.sqrt(max(0.0, g.sum())))
        else:
            fro[u] = float(np.linalg.norm(x[1]))
    return rank, fro
