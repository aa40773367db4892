"""The reference's manufactured problems, set up on the device.

Mirrors `pkg/src/ocp/system.py:181-265`:

* ``solve_state(u, spec)`` - damped Newton (the shared Newton core, tol 1e-12,
  sigma 1.1) on ``A y + phi(y) = f + u`` (`system.py:181-197`).  The residual
  is a device stencil kernel in the reference's CSR order; each direction
  solves ``(A + diag phi'(y)) d = -r``, which the reference hands to SuperLU,
  by device conjugate gradients to ``||r|| <= 1e-14 ||b||`` (the matrix is
  SPD: phi' >= 0 for every phi family used).
* ``construct_test_problem`` / ``construct_plateau_problem`` / ``_manufacture``
  (`system.py:220-265`): prescribed adjoint on the host (closed form, same
  numpy expressions), recovered control, device state solve, and the desired
  state ``y_d = y_bar - A p_bar - phi'(y_bar) p_bar`` by a device kernel.

A grid-only native context (no subdomains) carries these operators.
"""

import ctypes
import dataclasses
from dataclasses import dataclass

import numpy as np

from . import _native as nat
from .engine import DeviceVector, Engine
from .grid import Grid, NonfiniteFieldError
from .newton import ContinuationSchedule, NewtonConfig, newton_continuation
from .system import Nonlinearity, ProblemSpec, recover_control

CG_REL_TOL = 1e-14
CG_MAX_ITERS = 200000


@dataclass
class StatePair:
    y: np.ndarray
    p: np.ndarray

    def __post_init__(self):
        if self.y.shape != self.p.shape:
            raise ValueError("state and adjoint must have the same shape")


def grid_engine(spec):
    """Grid-only native context for spec (cached on the spec object)."""
    eng = getattr(spec, "_grid_engine", None)
    if eng is None:
        eng = Engine(spec, 0, 0, 0)
        try:
            object.__setattr__(spec, "_grid_engine", eng)
        except (AttributeError, TypeError):
            pass
    return eng


class _StateJacobian:
    """A + diag(phi'(y)) at one iterate; ``direct_solve`` replaces splu (`system.py:191-196`)."""

    def __init__(self, engine, y):
        self.engine, self.y = engine, y

    def direct_solve(self, rhs):
        e = self.engine
        x = e.vector(rhs.n)
        it, conv = ctypes.c_int(), ctypes.c_int()
        res = ctypes.c_double()
        rc = e.lib.ocp_state_cg(e.ctx, self.y.ptr, rhs.ptr, CG_REL_TOL, CG_MAX_ITERS, x.ptr,
                                ctypes.byref(it), ctypes.byref(res), ctypes.byref(conv))
        if rc == nat.OCP_ERR_NONFINITE:
            where, _, idx = e.error().rpartition("@")
            raise NonfiniteFieldError(where, int(idx))
        e.check(rc, "ocp_state_cg")
        if not conv.value:
            raise RuntimeError(f"state CG stalled at residual {res.value:.3e} after {it.value} iterations")
        return x


def solve_state(u, spec, tol=1e-12):
    """Solve the semilinear state equation A y + phi(y) = f + u (`system.py:181-197`)."""
    eng = grid_engine(spec)
    rhs = eng.from_host(np.asarray(spec.f, dtype=float) + np.asarray(u, dtype=float))

    def state_residual(y, eps):
        out = eng.vector(y.n)
        eng.check(eng.lib.ocp_state_residual(eng.ctx, y.ptr, rhs.ptr, out.ptr),
                  "ocp_state_residual")
        return out

    y, report = newton_continuation(
        eng.vector(eng.N).zero(), state_residual, lambda y, eps: _StateJacobian(eng, y),
        ContinuationSchedule.fixed(1.0), NewtonConfig(tol=tol))
    if not report.converged:
        raise RuntimeError(f"state solve failed: {report.failure}")
    return y.to_host()


def _manufacture(grid, p_bar, kappa, nu, mu, eps_construct):
    """`system.py:254-265` with the state solve and y_d on the device."""
    phi = Nonlinearity(kappa)
    spec = ProblemSpec(grid=grid, a=None, phi=phi, nu=nu, mu=mu,
                       f=np.zeros(grid.size), y_d=np.zeros(grid.size))
    u_bar = recover_control(p_bar, spec, eps_construct)
    y_bar = solve_state(u_bar, spec)
    eng = grid_engine(spec)
    yb, pb, yd = eng.from_host(y_bar), eng.from_host(p_bar), eng.vector(grid.size)
    eng.check(eng.lib.ocp_manufacture_yd(eng.ctx, yb.ptr, pb.ptr, yd.ptr), "ocp_manufacture_yd")
    spec = dataclasses.replace(spec, y_d=yd.to_host())
    return spec, StatePair(y=y_bar, p=p_bar)


def construct_test_problem(grid, kappa=0.1, nu=1e-6, mu=1.0, k_tilde=5, eps_construct=1e-15):
    """Manufactured oscillatory problem with a known solution pair (`system.py:219-236`)."""
    x1, x2 = grid.points()
    p_bar = 1.3 * mu * np.sin(2.0 * np.pi * k_tilde * x1) * np.sin(2.0 * np.pi * k_tilde * x2)
    return _manufacture(grid, p_bar, kappa, nu, mu, eps_construct)


def plateau_profile(x):
    """s(x) of the plateau adjoint (`system.py:239-248`)."""
    base = 2.0 * np.abs(np.sin(2.0 * np.pi * x))
    inside = (x >= 0.25) & (x <= 0.75)
    return np.where(inside, np.maximum(1.0, base), base)


def construct_plateau_problem(grid, kappa=0.1, nu=1e-6, mu=1.0, eps_construct=1e-15):
    """Manufactured problem whose adjoint has |p| = mu on a square (`system.py:251-258`)."""
    x1, x2 = grid.points()
    p_bar = mu * plateau_profile(x1) * plateau_profile(x2)
    return _manufacture(grid, p_bar, kappa, nu, mu, eps_construct)


__all__ = ["StatePair", "solve_state", "construct_test_problem", "construct_plateau_problem",
           "plateau_profile", "grid_engine"]
