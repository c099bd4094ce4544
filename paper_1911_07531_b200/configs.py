"""BASELINE.json configurations as concrete, seeded inputs.

c1  1D HODLR, n=2048, x_i=(i+0.5)/n, ell=0.1, leaf 64, eps 1e-6, std H-LU
c2  2D grid 128x128 (cell-centred, meshgrid "ij", row-major ravel),
    ell=0.2, leaf 64, eta=2, eps 1e-6, accumulator H-LU      (bench workload)
c3  65536 points on the unit sphere, default_rng(0) normal rows normalised,
    ell=0.3, leaf 64, eta=2, eps 1e-5, std and accumulator H-LU
c4  256 independent 1D HODLR instances; instance j: default_rng(1000+j),
    x = sort(uniform(4096)), ell = uniform(0.05, 0.5), leaf 64, eps 1e-6
c5  262144 points uniform in the unit cube, default_rng(0), ell=0.25,
    leaf 128, eta=2, eps 1e-4, accumulator H-LU
c5_dD  the first depth-D diagonal sub-problem of c5 (n = 262144 / 2^D)

BASELINE.json leaves the grid convention and the seeds unspecified; the
choices above are fixed here and in tests/golden/make_golden.py.  Every
matrix is A_ij = exp(-|x_i - x_j|/ell) + 1e-2 delta_ij, i.e. the
reference's PointKernel(points, exp(-d/ell), diag_value=1.01) composed with
the cluster-tree permutation (problems.py:34-53, 88-89).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass
class Config:
    name: str
    points: np.ndarray
    ell: float
    n_min: int
    admissibility: str      # "weak" | "eta"
    eta: float
    eps: float
    mode: str               # "std" | "accu"

    @property
    def n(self):
        return self.points.shape[0]


def config(name: str) -> Config:
    if name == "c1":
        n = 2048
        return Config("c1", ((np.arange(n) + 0.5) / n)[:, None], 0.1, 64, "weak", 0.0, 1e-6, "std")
    if name == "c2":
        g = (np.arange(128) + 0.5) / 128
        X, Y = np.meshgrid(g, g, indexing="ij")
        return Config("c2", np.column_stack([X.ravel(), Y.ravel()]), 0.2, 64, "eta", 2.0, 1e-6,
                      "accu")
    if name == "c3":
        rng = np.random.default_rng(0)
        p = rng.normal(size=(65536, 3))
        p /= np.linalg.norm(p, axis=1, keepdims=True)
        return Config("c3", p, 0.3, 64, "eta", 2.0, 1e-5, "accu")
    if name.startswith("c4"):
        j = int(name.split("_")[1]) if "_" in name else 0
        rng = np.random.default_rng(1000 + j)
        x = np.sort(rng.uniform(size=4096))
        ell = float(rng.uniform(0.05, 0.5))
        return Config(f"c4_{j}", x[:, None], ell, 64, "weak", 0.0, 1e-6, "std")
    if name == "c5":
        rng = np.random.default_rng(0)
        return Config("c5", rng.uniform(size=(262144, 3)), 0.25, 128, "eta", 2.0, 1e-4, "accu")
    if name.startswith("c5_d"):
        # the diagonal sub-problem of config 5 at cluster-tree depth d: the
        # points of the depth-d cluster in tree order.  Splits depend only on
        # a node's own points (trees.py:104-134; no coordinate ties in a
        # uniform draw), so its cluster and block trees equal c5's subtree.
        d = int(name[4:])
        full = config("c5")
        _, root, perm, _ = structure(full)
        node = root
        for _ in range(d):
            node = node.children[0]
        a, b = node.indices.first, node.indices.last
        return Config(name, full.points[perm[a:b]], full.ell, full.n_min, "eta", full.eta,
                      full.eps, "accu")
    if name == "s1":
        n = 512
        return Config("s1", ((np.arange(n) + 0.5) / n)[:, None], 0.1, 16, "weak", 0.0, 1e-6, "std")
    if name == "s2":
        g = (np.arange(32) + 0.5) / 32
        X, Y = np.meshgrid(g, g, indexing="ij")
        return Config("s2", np.column_stack([X.ravel(), Y.ravel()]), 0.2, 16, "eta", 2.0, 1e-6,
                      "accu")
    if name == "s5":
        rng = np.random.default_rng(0)
        p = rng.normal(size=(2048, 3))
        p /= np.linalg.norm(p, axis=1, keepdims=True)
        return Config("s5", p, 0.3, 32, "eta", 2.0, 1e-5, "accu")
    raise KeyError(name)


def structure(cfg: Config):
    """(geometry, cluster root, perm, block root) for a config."""
    from .trees import Geometry, build_block_tree, build_cluster_tree, standard_admissible
    from .trees import weak_admissible

    geom = Geometry(cfg.points)
    root, perm = build_cluster_tree(geom, cfg.n_min)
    if cfg.admissibility == "weak":
        adm = weak_admissible
    else:
        eta = cfg.eta
        adm = lambda t, s: standard_admissible(t, s, eta)  # noqa: E731
    broot = build_block_tree(root, root, adm)
    return geom, root, perm, broot


def kernel(cfg: Config, perm):
    from .problems import ExpKernel, permuted

    return permuted(ExpKernel(cfg.points, cfg.ell, diag_value=1.0 + 1e-2), perm)
