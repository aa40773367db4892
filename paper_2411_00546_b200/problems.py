"""Seeded synthetic problems for the BASELINE.json configurations.

The reference harness only builds its manufactured problem
(`pkg/src/ocp/harness/experiments.py:36-40`); the BASELINE configs need other
phi / f / y_d choices.  This module freezes one input convention (SURVEY.md
section 8d) so that the CPU oracle and the GPU path consume bit-identical
arrays:

* ``rng = np.random.default_rng(seed)``; bumps draw centers ``(K, 2)``, then
  widths ``(K,)``, then amplitudes ``(K,)``;
* ``y_d = sum_k a_k exp(-((x1-c1)^2 + (x2-c2)^2) / (2 w_k^2))``;
* config 3's ``f`` draws ``standard_normal(N)`` first, smooths it with 10
  Jacobi sweeps of the discrete Laplacian (neighbour mean, zero Dirichlet),
  then the bumps come from the same generator.

Nothing here reads the reference; the arrays are plain numpy.
"""

from dataclasses import dataclass

import numpy as np

from .grid import Grid, build_laplacian
from .system import Nonlinearity, ProblemSpec, make_phi


@dataclass(frozen=True)
class BaselineConfig:
    """One row of BASELINE.json ``configs`` in solver vocabulary.

    ``eps0 / gamma / eps_min`` are the reference ContinuationSchedule fields
    (`pkg/src/ocp/newton.py:29-48`); BASELINE's "gamma" smoothing parameter is
    the reference ``eps``.
    """

    name: str
    n: int
    phi: str
    nu: float
    mu: float
    s1: int
    s2: int
    overlap: int
    eps0: float
    gamma: float
    eps_min: float
    f_kind: str
    yd_kind: str
    bumps: int = 0
    center_range: tuple = (0.1, 0.9)
    width_range: tuple = (0.05, 0.15)
    amp_range: tuple = (-5.0, 5.0)
    seed: int = 0
    timed_unit: str = "solve"

    @property
    def unknowns(self):
        return 2 * self.n * self.n


CONFIGS = {
    "cfg1": BaselineConfig("cfg1", 63, "cubic", 1e-3, 1e-2, 2, 2, 4,
                           1.0, 0.1, 1e-6, "zero", "sine"),
    "cfg2": BaselineConfig("cfg2", 255, "cubic", 1e-3, 1e-2, 4, 4, 8,
                           1.0, 0.1, 1e-6, "zero", "bumps", bumps=8),
    "cfg3": BaselineConfig("cfg3", 511, "expm1", 1e-4, 5e-3, 8, 8, 8,
                           1.0, 0.1, 1e-7, "smoothed_noise", "bumps", bumps=16),
    "cfg4": BaselineConfig("cfg4", 1023, "cubic", 1e-3, 1e-2, 16, 16, 8,
                           1.0, 0.1, 1e-6, "zero", "bumps", bumps=32,
                           center_range=(0.05, 0.95), width_range=(0.02, 0.1),
                           amp_range=(-10.0, 10.0)),
    "cfg5": BaselineConfig("cfg5", 2047, "cubic", 1e-3, 1e-2, 64, 64, 2,
                           1e-3, 1.0, 1e-3, "zero", "uniform",
                           timed_unit="sweep+jvp"),
    "cfg5u": BaselineConfig("cfg5u", 2048, "cubic", 1e-3, 1e-2, 64, 64, 2,
                            1e-3, 1.0, 1e-3, "zero", "uniform",
                            timed_unit="sweep+jvp"),
}


# Not BASELINE rows: coarse decompositions whose local short side exceeds the
# fast kernels' 112 points (the paper's 2x2 at N = 450 has 227), used by the
# wide-line parity tests against reference fixtures (tests/golden/wide.npz).
EXTRA_CONFIGS = {
    "wide2x2": BaselineConfig("wide2x2", 300, "cubic", 1e-3, 1e-2, 2, 2, 8,
                              1.0, 0.1, 1e-6, "zero", "bumps", bumps=8),
    "mono150": BaselineConfig("mono150", 150, "cubic", 1e-3, 1e-2, 1, 1, 0,
                              1.0, 0.1, 1e-6, "zero", "bumps", bumps=8),
}


def _bumps(grid, rng, k, centers, widths, amps):
    x1, x2 = grid.points()
    c = rng.uniform(centers[0], centers[1], size=(k, 2))
    w = rng.uniform(widths[0], widths[1], size=k)
    a = rng.uniform(amps[0], amps[1], size=k)
    out = np.zeros(grid.size)
    for j in range(k):
        r2 = (x1 - c[j, 0]) ** 2 + (x2 - c[j, 1]) ** 2
        out += a[j] * np.exp(-r2 / (2.0 * w[j] ** 2))
    return out


def _jacobi_smooth(v, n, sweeps):
    """Neighbour mean with zero Dirichlet ring, repeated ``sweeps`` times."""
    f = v.reshape(n, n).copy()
    for _ in range(sweeps):
        g = np.zeros((n + 2, n + 2))
        g[1:-1, 1:-1] = f
        f = (g[:-2, 1:-1] + g[2:, 1:-1] + g[1:-1, :-2] + g[1:-1, 2:]) / 4.0
    return f.ravel()


def build_fields(cfg):
    """(f, y_d) float64 arrays of length n^2 for one configuration."""
    grid = Grid(cfg.n)
    rng = np.random.default_rng(cfg.seed)
    if cfg.f_kind == "zero":
        f = np.zeros(grid.size)
    elif cfg.f_kind == "smoothed_noise":
        f = _jacobi_smooth(rng.standard_normal(grid.size), cfg.n, 10)
    else:
        raise ValueError(f"unknown f kind {cfg.f_kind!r}")
    if cfg.yd_kind == "sine":
        x1, x2 = grid.points()
        y_d = 10.0 * np.sin(2.0 * np.pi * x1) * np.sin(2.0 * np.pi * x2)
    elif cfg.yd_kind == "bumps":
        y_d = _bumps(grid, rng, cfg.bumps, cfg.center_range, cfg.width_range,
                     cfg.amp_range)
    elif cfg.yd_kind == "uniform":
        y_d = rng.uniform(-1.0, 1.0, size=grid.size)
    else:
        raise ValueError(f"unknown y_d kind {cfg.yd_kind!r}")
    return f, y_d


def build_spec(cfg, with_matrix=True):
    """ProblemSpec for a BASELINE config (phi duck-typed per SURVEY 0.3)."""
    grid = Grid(cfg.n)
    f, y_d = build_fields(cfg)
    a = build_laplacian(grid) if with_matrix else None
    return ProblemSpec(grid=grid, a=a, phi=make_phi(cfg.phi), nu=cfg.nu,
                       mu=cfg.mu, f=f, y_d=y_d)


def mild_spec(n, kappa=0.1, nu=1e-2, mu=1.0, k_tilde=2, seed=3):
    """Small smooth test problem (role of the reference `mild_problem`).

    The reference builds its fixture from the manufactured problem
    (`pkg/tests/test_schwarz.py:18-22`); the drop-in tests only need a
    well-conditioned problem of the kappa family, so this uses a smooth
    analytic y_d instead of the state solve.
    """
    grid = Grid(n)
    x1, x2 = grid.points()
    y_d = 1.3 * np.sin(2.0 * np.pi * k_tilde * x1) * np.sin(2.0 * np.pi * k_tilde * x2)
    rng = np.random.default_rng(seed)
    f = 0.1 * rng.standard_normal(grid.size)
    return ProblemSpec(grid=grid, a=build_laplacian(grid), phi=Nonlinearity(kappa),
                       nu=nu, mu=mu, f=f, y_d=y_d)
