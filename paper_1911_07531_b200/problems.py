"""Entry generators (drop-in for hmatdag.problems, problems.py:24-94).

``ExpKernel`` is the PointKernel of every BASELINE config,
exp(-||x_i - x_j||/ell) with a fixed diagonal; besides the host ``dense``
it exposes a device description so that assembly evaluates blocks on the
GPU (hmx_exp_kernel_blocks).  Generic kernels (any object with
``dense(I, J)``) are evaluated on the host and uploaded.
"""

from __future__ import annotations

import numpy as np


class Kernel:
    def __call__(self, i: int, j: int) -> float:
        return float(self.dense(np.asarray([i]), np.asarray([j]))[0, 0])

    def dense(self, I, J) -> np.ndarray:
        raise NotImplementedError

    def device_spec(self):
        """(points, perm or None, ell, diag, scale) when evaluable on device."""
        return None


class PointKernel(Kernel):
    """k(x_i, x_j) = scale*offdiag(|x_i-x_j|), diagonal fixed (problems.py:34-53)."""

    def __init__(self, points, offdiag, diag_value, scale=1.0):
        self.points = np.asarray(points, dtype=float)
        self._offdiag = offdiag
        self.diag_value = float(diag_value)
        self.scale = float(scale)

    def dense(self, I, J):
        I = np.asarray(I, dtype=np.intp)
        J = np.asarray(J, dtype=np.intp)
        d = np.linalg.norm(self.points[I][:, None, :] - self.points[J][None, :, :], axis=-1)
        with np.errstate(divide="ignore", invalid="ignore"):
            vals = self.scale * self._offdiag(d)
        return np.where(I[:, None] == J[None, :], self.diag_value, vals)


class ExpKernel(PointKernel):
    """exp(-d/ell) point kernel of the BASELINE configs."""

    def __init__(self, points, ell, diag_value=1.0 + 1e-2, scale=1.0):
        ell = float(ell)
        super().__init__(points, lambda d: np.exp(-d / ell), diag_value, scale)
        self.ell = ell

    def device_spec(self):
        return self.points, None, self.ell, self.diag_value, self.scale


class ShiftedKernel(Kernel):
    """Adds c*n on the diagonal (problems.py:56-68)."""

    def __init__(self, base: Kernel, c: float, n: int):
        self.base = base
        self.shift = float(c) * n

    def dense(self, I, J):
        I = np.asarray(I, dtype=np.intp)
        J = np.asarray(J, dtype=np.intp)
        return self.base.dense(I, J) + self.shift * (I[:, None] == J[None, :])


class PermutedKernel(Kernel):
    """Kernel re-indexed by a cluster-tree permutation (problems.py:71-81)."""

    def __init__(self, base: Kernel, perm):
        self.base = base
        self.perm = np.asarray(perm, dtype=np.intp)

    def dense(self, I, J):
        return self.base.dense(self.perm[np.asarray(I, dtype=np.intp)],
                               self.perm[np.asarray(J, dtype=np.intp)])

    def device_spec(self):
        spec = self.base.device_spec()
        if spec is None or spec[1] is not None:
            return None
        pts, _, ell, diag, scale = spec
        return pts, self.perm, ell, diag, scale


def shifted(kernel: Kernel, c: float, n: int) -> Kernel:
    return ShiftedKernel(kernel, c, n)


def permuted(kernel: Kernel, perm) -> Kernel:
    return PermutedKernel(kernel, perm)


def dense_matrix(kernel: Kernel, n: int) -> np.ndarray:
    idx = np.arange(n)
    return kernel.dense(idx, idx)


def one_d_problem(n: int):
    """Log kernel on [0,1] midpoints (problems.py:122-135)."""
    from .trees import Geometry

    if n < 2:
        raise ValueError("1d problem needs n >= 2")
    x = (np.arange(n) + 0.5) / n
    diag = (np.log(1.0 / (2.0 * n)) - 1.0) / n
    return Geometry(x[:, None]), PointKernel(x[:, None], np.log, diag_value=diag, scale=1.0 / n)


def fibonacci_sphere(n: int) -> np.ndarray:
    """n quasi-uniform points on the unit sphere: golden-angle spiral in z
    (problems.py:95-102)."""
    i = np.arange(n, dtype=float)
    z = 1.0 - 2.0 * (i + 0.5) / n
    r = np.sqrt(np.maximum(0.0, 1.0 - z * z))
    phi = np.pi * (3.0 - np.sqrt(5.0)) * i
    return np.column_stack([r * np.cos(phi), r * np.sin(phi), z])


def sphere_problem(n: int):
    """1/r kernel on the unit sphere with quadrature weight w = 4 pi / n and
    the flat-disc self term 2 sqrt(pi w) on the diagonal (problems.py:105-119)."""
    from .trees import Geometry

    if n < 4:
        raise ValueError("sphere problem needs n >= 4")
    pts = fibonacci_sphere(n)
    w = 4.0 * np.pi / n
    return Geometry(pts), PointKernel(pts, lambda d: 1.0 / d, diag_value=2.0 * np.sqrt(np.pi * w),
                                      scale=w)
