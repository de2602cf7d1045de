"""The five BASELINE.json configurations: coefficient fields and seeded Dirichlet data.

The reference ships no problem module (`problems_cli` is absent), so these
generators follow SURVEY.md §8(d) exactly. The domain is [0,1]^2 and p = q = 16. Boundary data
is produced on the host in root.I_e order (solver.py:292-300) and fed identically to the
reference/oracle and to the GPU path.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .grid import Rectangle
from .leafops import CoefficientField

KAPPA = 80.0
BETA = 1000.0


def _c11(x, y):
    return 1.0 + 0.5 * np.sin(2 * np.pi * x) * np.cos(2 * np.pi * y)


def _c22(x, y):
    return 1.0 + 0.5 * np.cos(4 * np.pi * x) * np.sin(2 * np.pi * y)


def _c_varhelm(x, y):
    return -KAPPA ** 2 * (1.0 - (np.sin(4 * np.pi * x) * np.sin(4 * np.pi * y)) ** 2)


@dataclass(frozen=True)
class Config:
    cfg: int
    name: str
    L: int
    batch: int
    data: str  # 'exact_lap' | 'fourier8' | 'plane_wave'
    tol: float  # BASELINE parity tolerance (relative)

    def coefficients(self):
        return coefficients(self.cfg)

    @property
    def domain(self):
        return Rectangle(0.0, 1.0, 0.0, 1.0)


CONFIGS = {
    1: Config(1, "laplace", 4, 1, "exact_lap", 1e-10),
    2: Config(2, "var_diffusion", 6, 64, "fourier8", 1e-10),
    3: Config(3, "helmholtz_k80", 7, 1, "plane_wave", 1e-8),
    4: Config(4, "var_helmholtz_k80", 8, 1, "plane_wave", 1e-8),
    5: Config(5, "conv_diffusion_b1000", 9, 256, "fourier8", 1e-10),
}


def coefficients(cfg):
    """CoefficientField of config `cfg` (BASELINE.json configs)."""
    if cfg == 1:
        return CoefficientField()
    if cfg == 2:
        return CoefficientField(c11=_c11, c22=_c22)
    if cfg == 3:
        return CoefficientField(c=-KAPPA ** 2)
    if cfg == 4:
        return CoefficientField(c=_c_varhelm)
    if cfg == 5:
        return CoefficientField(c1=-BETA)
    raise ValueError(f"unknown config {cfg}")


def perimeter_parameter(x, y):
    """t in [0,4), counter-clockwise from (0,0): S t=x1, E 1+x2, N 3-x1, W 4-x2."""
    t = np.empty_like(x)
    S = y == 0.0
    E = (x == 1.0) & ~S
    N = (y == 1.0) & ~S & ~E
    W = ~(S | E | N)
    t[S] = x[S]
    t[E] = 1.0 + y[E]
    t[N] = 3.0 - x[N]
    t[W] = 4.0 - y[W]
    return t


def boundary_data(cfg, points, seed=0, batch=None):
    """Dirichlet data at the given root-boundary Gauss points, shape (n, b) (b=1 -> (n,)).

    cfg 1: exp(x1) sin(x2); cfg 2/5: 8 random Fourier modes of the perimeter parameter
    (rng.standard_normal((b, 8)) then rng.uniform(0, 2pi, (b, 8))); cfg 3/4: plane wave
    cos(kappa (x1 cos th + x2 sin th)) with th = rng.uniform(0, 2pi) per vector.
    """
    c = CONFIGS[cfg]
    b = c.batch if batch is None else batch
    x, y = points[:, 0], points[:, 1]
    rng = np.random.default_rng(seed)
    if c.data == "exact_lap":
        F = np.repeat((np.exp(x) * np.sin(y))[:, None], b, axis=1)
    elif c.data == "fourier8":
        a = rng.standard_normal((b, 8))
        ph = rng.uniform(0.0, 2 * np.pi, (b, 8))
        t = perimeter_parameter(x, y)
        m = np.arange(1, 9)
        F = np.einsum("jm,njm->nj", a, np.cos(np.pi * m[None, None, :] * t[:, None, None] / 2 + ph[None, :, :]))
    elif c.data == "plane_wave":
        th = rng.uniform(0.0, 2 * np.pi, b)
        F = np.cos(KAPPA * (x[:, None] * np.cos(th)[None, :] + y[:, None] * np.sin(th)[None, :]))
    else:
        raise ValueError(c.data)
    return F[:, 0] if (batch == 1 or (batch is None and b == 1)) else F


def exact_solution(cfg, x, y, seed=0, batch=None):
    """Exact u where available (cfg 1: exp(x1)sin(x2); cfg 3: plane wave), else None."""
    c = CONFIGS[cfg]
    b = c.batch if batch is None else batch
    if cfg == 1:
        U = np.repeat((np.exp(x) * np.sin(y))[:, None], b, axis=1)
    elif cfg == 3:
        th = np.random.default_rng(seed).uniform(0.0, 2 * np.pi, b)
        U = np.cos(KAPPA * (x[:, None] * np.cos(th)[None, :] + y[:, None] * np.sin(th)[None, :]))
    else:
        return None
    return U[:, 0] if U.shape[1] == 1 and (batch == 1 or (batch is None and b == 1)) else U
