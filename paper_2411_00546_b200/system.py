"""Optimality-system data types (mirror of `pkg/src/ocp/system.py`).

The reduced unknown is ``x = [y; p]`` (`system.py:109-115`).  Residual rows
(`system.py:118-132`)::

    r1 = A y + phi(y) - f + (p + mu P_eps(-p/mu)) / nu
    r2 = A p + phi'(y) p - y + y_d

and the Jacobian is ``[[A + diag phi'(y), diag b12], [diag b21, A + diag phi'(y)]]``
with ``b12 = (1 - P'_eps(-p/mu))/nu`` and ``b21 = phi''(y) p - 1``
(`system.py:135-144`).  On the device path these formulas are evaluated inside
the CUDA kernels (`csrc/ocp_pointwise.cuh`); the numpy helpers below exist for
the host-side API (control recovery of host arrays, small diagnostics).

phi is duck-typed exactly as the reference consumes it (``value``,
``derivative``, ``second_derivative`` with a ``check`` flag).  Each class also
carries ``kind``/``kappa`` so the device path can select the same formula:

* ``Nonlinearity(kappa)`` - the reference family kappa (s^3 + e^{kappa s})
  with the exp argument clamped at EXP_ARG_MAX (`system.py:28-74`);
* ``Cubic()`` - phi(y) = y^3, evaluated as ``s*s*s`` (BASELINE configs 1,2,4,5);
* ``ExpMinusOne()`` - phi(y) = e^y - 1 (BASELINE config 3), same clamp.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .grid import Grid, check_finite

EXP_ARG_MAX = 700.0

PHI_KAPPA = 0
PHI_CUBIC = 1
PHI_EXPM1 = 2


def smoothed_projection(x, eps):
    """P_eps(x) = (sqrt((x+1)^2+eps) - sqrt((x-1)^2+eps))/2 (`smoothing.py:19-32`)."""
    if eps < 0:
        raise ValueError("eps must be nonnegative")
    x = np.asarray(x, dtype=float)
    if eps == 0.0:
        return np.clip(x, -1.0, 1.0)
    a = x + 1.0
    b = x - 1.0
    return 0.5 * (np.sqrt(a * a + eps) - np.sqrt(b * b + eps))


def smoothed_projection_derivative(x, eps):
    """P'_eps(x) (`smoothing.py:35-44`)."""
    if eps <= 0:
        raise ValueError("derivative of the smoothed projection needs eps > 0")
    x = np.asarray(x, dtype=float)
    a = x + 1.0
    b = x - 1.0
    return 0.5 * (a / np.sqrt(a * a + eps) - b / np.sqrt(b * b + eps))


def _checked(out, arg_over, where, check):
    if check:
        check_finite(np.where(arg_over, np.inf, out), where)
    return out


@dataclass(frozen=True)
class Nonlinearity:
    """phi(s) = kappa (s^3 + exp(kappa s)); kappa = 0 is linear (`system.py:31-74`)."""

    kappa: float = 0.1
    kind = PHI_KAPPA

    def _exp(self, s):
        return np.exp(np.minimum(self.kappa * s, EXP_ARG_MAX))

    def value(self, s, check=True):
        if self.kappa == 0.0:
            return np.zeros_like(s)
        with np.errstate(over="ignore", invalid="ignore"):
            out = self.kappa * (s ** 3 + self._exp(s))
        return _checked(out, self.kappa * s > EXP_ARG_MAX, "phi(y)", check)

    def derivative(self, s, check=True):
        if self.kappa == 0.0:
            return np.zeros_like(s)
        with np.errstate(over="ignore", invalid="ignore"):
            out = self.kappa * (3.0 * s ** 2 + self.kappa * self._exp(s))
        return _checked(out, self.kappa * s > EXP_ARG_MAX, "phi'(y)", check)

    def second_derivative(self, s, check=True):
        if self.kappa == 0.0:
            return np.zeros_like(s)
        with np.errstate(over="ignore", invalid="ignore"):
            out = self.kappa * (6.0 * s + self.kappa ** 2 * self._exp(s))
        return _checked(out, self.kappa * s > EXP_ARG_MAX, "phi''(y)", check)


@dataclass(frozen=True)
class Cubic:
    """phi(y) = y^3 with phi' = 3 y^2 and phi'' = 6 y, products left to right."""

    kappa: float = 0.0
    kind = PHI_CUBIC

    def value(self, s, check=True):
        with np.errstate(over="ignore", invalid="ignore"):
            out = s * s * s
        return check_finite(out, "phi(y)") if check else out

    def derivative(self, s, check=True):
        with np.errstate(over="ignore", invalid="ignore"):
            out = 3.0 * s * s
        return check_finite(out, "phi'(y)") if check else out

    def second_derivative(self, s, check=True):
        out = 6.0 * s
        return check_finite(out, "phi''(y)") if check else out


@dataclass(frozen=True)
class ExpMinusOne:
    """phi(y) = e^y - 1 (monotone), exp argument clamped at EXP_ARG_MAX."""

    kappa: float = 0.0
    kind = PHI_EXPM1

    def _exp(self, s):
        return np.exp(np.minimum(s, EXP_ARG_MAX))

    def value(self, s, check=True):
        out = self._exp(s) - 1.0
        return _checked(out, s > EXP_ARG_MAX, "phi(y)", check)

    def derivative(self, s, check=True):
        return _checked(self._exp(s), s > EXP_ARG_MAX, "phi'(y)", check)

    def second_derivative(self, s, check=True):
        return _checked(self._exp(s), s > EXP_ARG_MAX, "phi''(y)", check)


def make_phi(name, kappa=0.1):
    if name == "cubic":
        return Cubic()
    if name == "expm1":
        return ExpMinusOne()
    if name == "kappa":
        return Nonlinearity(kappa)
    raise ValueError(f"unknown nonlinearity {name!r}")


def phi_code(phi):
    """(kind, kappa) selector of the device formula for a phi object."""
    kind = getattr(phi, "kind", None)
    if kind is None:
        if type(phi).__name__ == "Nonlinearity" and hasattr(phi, "kappa"):
            return PHI_KAPPA, float(phi.kappa)
        raise TypeError(f"no device formula for nonlinearity {phi!r}")
    return int(kind), float(getattr(phi, "kappa", 0.0))


@dataclass(frozen=True)
class ProblemSpec:
    """Problem data (`system.py:77-94`); ``a`` is optional (matrix-free device path)."""

    grid: Grid
    a: object
    phi: object
    nu: float
    mu: float
    f: np.ndarray
    y_d: np.ndarray

    def __post_init__(self):
        if self.nu <= 0.0 or self.mu <= 0.0:
            raise ValueError("nu and mu must be positive")
        n2 = self.grid.size
        if self.f.shape != (n2,) or self.y_d.shape != (n2,):
            raise ValueError("operator and data shapes do not match the grid")
        if self.a is not None and self.a.shape != (n2, n2):
            raise ValueError("operator and data shapes do not match the grid")


def merge_pair(y, p):
    return np.concatenate([y, p])


def split_pair(x):
    n2 = x.shape[0] // 2
    return x[:n2], x[n2:]


def recover_control(p, spec, eps):
    """u = -(p + mu P_eps(-p/mu))/nu (`system.py:173-174`).

    Device vectors go through the ``ocp_recover_control`` kernel; host arrays
    use numpy (the reference helper's own contract).
    """
    if hasattr(p, "device_ptr"):
        return p.recover_control(spec, eps)
    return -(p + spec.mu * smoothed_projection(-p / spec.mu, eps)) / spec.nu
