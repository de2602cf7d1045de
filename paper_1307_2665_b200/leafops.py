"""Leaf spectral constants (host side) for the CUDA leaf kernel.

Drop-in for the parts of `hpsolve.leafops` that the build path uses (reference
leafops.py:22-30, 36-214). `CoefficientField` and `LeafGeometry` keep the reference's names,
fields and numbers. The per-leaf arithmetic (assemble A, interior solve, DtN) runs on the GPU in
`csrc/leaf.cu`. This module only prepares the coefficient-independent constants, once per
(p, width, height), and packs them for upload.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .grid import Rectangle, cheb_nodes, gauss_nodes, interp_matrix

__all__ = ["CoefficientField", "LeafGeometry", "cheb_diff_matrix", "RESONANCE_COND"]

#: condition estimate beyond which a leaf counts as resonant (leafops.py:33)
RESONANCE_COND = 1e13

#: fixed probe for the one-shot condition estimate (leafops.py:285-286)
PROBE_SEED = 1234


@dataclass
class CoefficientField:
    """A = -c11 d11 - 2 c12 d12 - c22 d22 + c1 d1 + c2 d2 + c (leafops.py:36-59).

    Each entry is a scalar or a callable f(x1, x2) on numpy arrays. Default: Laplace.
    """

    c11: object = 1.0
    c12: object = 0.0
    c22: object = 1.0
    c1: object = 0.0
    c2: object = 0.0
    c: object = 0.0

    _NAMES = ("c11", "c12", "c22", "c1", "c2", "c")

    def evaluate_all(self, x, y):
        out = {}
        for name in self._NAMES:
            f = getattr(self, name)
            out[name] = f(x, y) if callable(f) else float(f)
        return out


def cheb_diff_matrix(p, interval=(-1.0, 1.0)):
    """Chebyshev spectral differentiation, negative-sum diagonal (leafops.py:70-85)."""
    x = cheb_nodes(p, interval)
    w = np.power(-1.0, np.arange(p))
    w[0] *= 0.5
    w[-1] *= 0.5
    D = np.zeros((p, p))
    for i in range(p):
        off = np.r_[0:i, i + 1:p]
        D[i, off] = (w[off] / w[i]) / (x[i] - x[off])
        D[i, i] = -np.sum(D[i, off])
    return D


class LeafGeometry:
    """Coefficient-independent leaf machinery (leafops.py:88-214), cached per (p, w, h).

    Same attributes as the reference (cheb_x/y, gauss_x/y, Dx, Dy, D1, D2, D1sq, D12, D2sq,
    grid_x/y, J_i, J_e, L1, L4, L43). The Kronecker-product matrices are built lazily: the GPU
    kernel only needs the 1-D factors.
    """

    _cache: dict = {}

    def __init__(self, p, width, height):
        self.p = p
        self.width = width
        self.height = height
        self.cheb_x = cheb_nodes(p, (0.0, width))
        self.cheb_y = cheb_nodes(p, (0.0, height))
        self.gauss_x = (gauss_nodes(p) + 1.0) * 0.5 * width
        self.gauss_y = (gauss_nodes(p) + 1.0) * 0.5 * height
        self.Dx = cheb_diff_matrix(p, (0.0, width))
        self.Dy = cheb_diff_matrix(p, (0.0, height))
        self.Dxx = self.Dx @ self.Dx  # the factor of kron(Dx @ Dx, I) (leafops.py:113)
        self.Dyy = self.Dy @ self.Dy
        self.grid_x = np.repeat(self.cheb_x, p)
        self.grid_y = np.tile(self.cheb_y, p)
        k = np.arange(1, p - 1)
        self.J_i = (k[:, None] * p + k[None, :]).reshape(-1).astype(np.intp)
        r = np.arange(p - 1)
        # S owns SW, E owns SE, N owns NE, W owns NW (leafops.py:122-128)
        self.J_e = np.concatenate([r * p, (p - 1) * p + r, (r + 1) * p + (p - 1), r + 1]).astype(np.intp)
        self.Qx = interp_matrix(self.cheb_x, self.gauss_x)  # Chebyshev -> Gauss, x sides
        self.Qy = interp_matrix(self.cheb_y, self.gauss_y)
        self.L1 = self._build_l1()
        self.L4 = self._build_l4()
        self.L43 = self.L4 @ self._build_l3()
        self._kron = None

    @classmethod
    def get(cls, p, width, height):
        key = (p, width, height)
        g = cls._cache.get(key)
        if g is None:
            g = cls(p, width, height)
            cls._cache[key] = g
        return g

    # Kronecker operators, x1-major flattening i*p + j (leafops.py:111-115), built on demand
    def _k(self):
        if self._kron is None:
            I = np.eye(self.p)
            self._kron = dict(D1=np.kron(self.Dx, I), D2=np.kron(I, self.Dy), D1sq=np.kron(self.Dxx, I),
                              D12=np.kron(self.Dx, self.Dy), D2sq=np.kron(I, self.Dyy))
        return self._kron

    D1 = property(lambda s: s._k()["D1"])
    D2 = property(lambda s: s._k()["D2"])
    D1sq = property(lambda s: s._k()["D1sq"])
    D12 = property(lambda s: s._k()["D12"])
    D2sq = property(lambda s: s._k()["D2sq"])

    def _build_l1(self):
        """4(p-1) x 4p Gauss -> boundary Chebyshev, corners averaged (leafops.py:143-179)."""
        p = self.p
        PS = interp_matrix(self.gauss_x, self.cheb_x)
        PE = interp_matrix(self.gauss_y, self.cheb_y)
        L1 = np.zeros((4 * (p - 1), 4 * p))
        cs = lambda s: slice(s * p, (s + 1) * p)  # S=0, E=1, N=2, W=3
        # side blocks: (row block, own side, own interpolant rows, corner partner side/row)
        for i in range(p - 1):
            L1[i, cs(0)] = PS[i]
        for j in range(p - 1):
            L1[p - 1 + j, cs(1)] = PE[j]
        for k, i in enumerate(range(1, p)):
            L1[2 * (p - 1) + k, cs(2)] = PS[i]
        for k, j in enumerate(range(1, p)):
            L1[3 * (p - 1) + k, cs(3)] = PE[j]
        # corners: average of the two sides meeting there
        for row, (sa, ra, Pa), (sb, rb, Pb) in (
                (0, (0, 0, PS), (3, 0, PE)),                         # SW: S owns, W partner
                (p - 1, (1, 0, PE), (0, p - 1, PS)),                 # SE: E owns, S partner
                (3 * (p - 1) - 1, (2, p - 1, PS), (1, p - 1, PE)),   # NE: N owns, E partner
                (4 * (p - 1) - 1, (3, p - 1, PE), (2, 0, PS))):      # NW: W owns, N partner
            L1[row, :] = 0.0
            L1[row, cs(sa)] = 0.5 * Pa[ra]
            L1[row, cs(sb)] = 0.5 * Pb[rb]
        return L1

    def _build_l3(self):
        """Spectral derivative rows at boundary nodes: d/dx2 on S/N, d/dx1 on E/W (181-189)."""
        p = self.p
        I = np.eye(p)
        rows = np.zeros((4 * p, p * p))
        for i in range(p):  # south / north: d/dx2 at (i, 0) / (i, p-1)
            rows[i] = np.kron(I[i], self.Dy[0])
            rows[2 * p + i] = np.kron(I[i], self.Dy[p - 1])
        for j in range(p):  # east / west: d/dx1 at (p-1, j) / (0, j)
            rows[p + j] = np.kron(self.Dx[p - 1], I[j])
            rows[3 * p + j] = np.kron(self.Dx[0], I[j])
        return rows

    def _build_l4(self):
        p = self.p
        L4 = np.zeros((4 * p, 4 * p))
        for s, Q in enumerate((self.Qx, self.Qy, self.Qx, self.Qy)):
            L4[s * p:(s + 1) * p, s * p:(s + 1) * p] = Q
        return L4

    def leaf_points(self, rect):
        return rect.x_lo + self.grid_x, rect.y_lo + self.grid_y

    def gauss_boundary_points(self, rect):
        q = self.p
        xs = rect.x_lo + self.gauss_x
        ys = rect.y_lo + self.gauss_y
        pts = np.empty((4 * q, 2))
        pts[0:q] = np.column_stack([xs, np.full(q, rect.y_lo)])
        pts[q:2 * q] = np.column_stack([np.full(q, rect.x_hi), ys])
        pts[2 * q:3 * q] = np.column_stack([xs, np.full(q, rect.y_hi)])
        pts[3 * q:4 * q] = np.column_stack([np.full(q, rect.x_lo), ys])
        return pts

    # ------------------------------------------------------------------------------------------
    # Packed constants for the CUDA leaf kernel (layout documented in include/hps_b200.h)
    # ------------------------------------------------------------------------------------------
    def device_constants(self):
        """fp64 blob: Dx, Dy, Dxx, Dyy (p*p each), L43e (4p x ne), L43i (4p x ni), L1 (ne x 4p),
        probe (ni); plus int32 J_i (ni), J_e (ne)."""
        p = self.p
        probe = np.random.default_rng(PROBE_SEED).standard_normal((self.J_i.size, 1))[:, 0]
        blob = np.concatenate([
            self.Dx.ravel(), self.Dy.ravel(), self.Dxx.ravel(), self.Dyy.ravel(),
            np.ascontiguousarray(self.L43[:, self.J_e]).ravel(),
            np.ascontiguousarray(self.L43[:, self.J_i]).ravel(),
            self.L1.ravel(), probe])
        idx = np.concatenate([self.J_i, self.J_e]).astype(np.int32)
        return blob, idx, float(np.abs(probe).max())

    def corner_mode_vectors(self, axis):
        """Gauss values on one interface segment of the corner null mode.

        The mode at an interior vertex of a cut line equals the Chebyshev-endpoint Lagrange
        polynomial sampled at the segment's Gauss nodes: Q[:, 0] on the segment starting at the
        vertex, Q[:, -1] on the one ending there. `axis` is the cut ('v' runs along y)."""
        Q = self.Qy if axis == "v" else self.Qx
        return np.ascontiguousarray(Q[:, 0]), np.ascontiguousarray(Q[:, -1])
