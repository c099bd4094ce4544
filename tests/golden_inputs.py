"""Case definitions and seeded inputs of the golden fixtures.

Restates tests/golden/make_golden.py's problem generators (BASELINE.json
configs + small cases) so that tests can rebuild inputs without storing
them and without importing the reference.
"""

import json
import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def probe_vec(n):
    return np.random.default_rng(7).normal(size=(n, 2))


def truncate_inputs(i, m, n, K, decay):
    r = np.random.default_rng(100 + i)
    U = r.normal(size=(m, K)) * np.exp(-decay * np.arange(K))[None, :]
    V = r.normal(size=(n, K))
    M = U @ V.T + 1e-3 * r.normal(size=(m, n)) * np.exp(-decay * K)
    return U, V, M


def case(name):
    """(points, ell, n_min, adm_kind, eta, eps)."""
    if name == "c1":
        n = 2048
        return ((np.arange(n) + 0.5) / n)[:, None], 0.1, 64, "weak", None, 1e-6
    if name == "c2":
        g = (np.arange(128) + 0.5) / 128
        X, Y = np.meshgrid(g, g, indexing="ij")
        return np.column_stack([X.ravel(), Y.ravel()]), 0.2, 64, "eta", 2.0, 1e-6
    if name in ("c3s", "c3"):
        rng = np.random.default_rng(0)
        p = rng.normal(size=(65536, 3))
        p /= np.linalg.norm(p, axis=1, keepdims=True)
        return p, 0.3, 64, "eta", 2.0, 1e-5
    if name.startswith("c4_"):
        rng = np.random.default_rng(1000 + int(name[3:]))
        x = np.sort(rng.uniform(size=4096))
        ell = float(rng.uniform(0.05, 0.5))
        return x[:, None], ell, 64, "weak", None, 1e-6
    if name == "c5s":
        rng = np.random.default_rng(0)
        return rng.uniform(size=(262144, 3)), 0.25, 128, "eta", 2.0, 1e-4
    if name == "s1":
        n = 512
        return ((np.arange(n) + 0.5) / n)[:, None], 0.1, 16, "weak", None, 1e-6
    if name == "s2":
        g = (np.arange(32) + 0.5) / 32
        X, Y = np.meshgrid(g, g, indexing="ij")
        return np.column_stack([X.ravel(), Y.ravel()]), 0.2, 16, "eta", 2.0, 1e-6
    if name == "s5":
        rng = np.random.default_rng(0)
        p = rng.normal(size=(2048, 3))
        p /= np.linalg.norm(p, axis=1, keepdims=True)
        return p, 0.3, 32, "eta", 2.0, 1e-5
    raise KeyError(name)


def load(name):
    with open(os.path.join(GOLDEN, f"{name}.json")) as f:
        meta = json.load(f)
    arrays = dict(np.load(os.path.join(GOLDEN, f"{name}.npz")))
    return meta, arrays


def have(name):
    return os.path.exists(os.path.join(GOLDEN, f"{name}.json"))
