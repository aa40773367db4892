"""Linear-RAS Newton-Krylov (method ``newton-ras`` / ``newton-ras-eps``) on the device.

The reference's main competitor to RASPEN: monolithic damped
Newton with eps-continuation on the global residual, each direction by GMRES
left-preconditioned with one-level RAS rebuilt at every outer iterate
(`harness/experiments.py:72-84`).  Pieces and the reference code they replace:

* ``global_residual``  -> ``system.residual(x, spec, eps, check=False)`` (`system.py:147-152`)
* ``GlobalJacobian``   -> ``system.jacobian(x, spec, eps)`` used as ``jac @ v`` (`system.py:155-160`,
  `newton.py:118`): per-point diagonals on the device, CSR row sums in the
  reference's entry order
* ``RasPreconditioner`` / ``ras_preconditioner`` / ``ras_precondition`` ->
  `schwarz.py:221-244`: the local pair Jacobians at ``x[pair_idx]`` go through
  the same batched block-Thomas factor as RASPEN (kernel 2), the apply is the stored-factor
  block solve (kernel 4) + restricted prolongation
* ``newton_ras_solve`` -> the RAS branch of ``solve_single``; the direction
  solve runs as one native call (``ocp_ras_gmres``: JVP, RAS apply and MGS
  Arnoldi on the device, Givens on the host in the reference's order).
"""

import ctypes

import numpy as np

from . import _native as nat
from .engine import DeviceVector, Engine
from .grid import NonfiniteFieldError
from .krylov import GmresBreakdownError, GmresResult, KrylovConfig
from .newton import NewtonConfig, newton_continuation
from .schwarz import LocalSolveError, build_local_systems


def _as_device(engine, v):
    if isinstance(v, DeviceVector):
        return v, True
    return engine.from_host(np.asarray(v, dtype=float)), False


def _raise(engine, rc, where, failed=-1):
    msg = engine.error()
    if rc == nat.OCP_ERR_NONFINITE:
        what, _, idx = msg.rpartition("@")
        raise NonfiniteFieldError(what, int(idx))
    if rc == nat.OCP_ERR_LOCAL_SOLVE:
        raise LocalSolveError(failed, msg)
    raise nat.NativeError(rc, msg, where)


def global_residual(engine, x, eps, out=None):
    """F_eps(x) on the whole grid, ``check=False`` (`system.py:147-152`)."""
    xd, dev = _as_device(engine, x)
    r = engine.vector(xd.n) if out is None else out
    rc = engine.lib.ocp_global_residual(engine.ctx, xd.ptr, float(eps), r.ptr)
    if rc != nat.OCP_OK:
        _raise(engine, rc, "ocp_global_residual")
    return r if dev else r.to_host()


class GlobalJacobian:
    """J(x) of F_eps as an operator (`system.py:155-160`); ``J(d)`` / ``J @ d``."""

    def __init__(self, engine, x, eps):
        xd, _ = _as_device(engine, x)
        self.engine, self.eps, self.x = engine, float(eps), xd
        self._lu = None
        self.jd = engine.buffer(8 * 4 * engine.N)
        rc = engine.lib.ocp_global_jacobian(engine.ctx, xd.ptr, self.eps,
                                            ctypes.c_void_p(self.jd.addr))
        if rc != nat.OCP_OK:
            _raise(engine, rc, "ocp_global_jacobian")

    def __call__(self, d):
        dd, dev = _as_device(self.engine, d)
        out = self.engine.vector(dd.n)
        self.engine.check(self.engine.lib.ocp_global_jvp(
            self.engine.ctx, ctypes.c_void_p(self.jd.addr), dd.ptr, out.ptr), "ocp_global_jvp")
        return out if dev else out.to_host()

    __matmul__ = __call__

    def direct_solve(self, rhs):
        """Sparse direct solve of J d = rhs (splu, `newton.py:125-129`): the
        batched block factor on a single-subdomain engine, i.e. one factorisation of the
        whole Jacobian (block-tridiagonal factor of 2n-unknown lines; any n up to
        1984, lines wider than 224 unknowns on the wide kernels)."""
        if self.engine.num_subdomains != 1:
            raise ValueError("direct solves need the single-subdomain (1x1) engine")
        if self._lu is None:
            self._lu = RasPreconditioner(self.engine, self.x, self.eps)
        return self._lu(rhs)

    def fused_gmres(self, b, cfg, precond=None):
        """Whole preconditioned GMRES solve natively when ``precond`` is this
        engine's RAS preconditioner; NotImplemented otherwise."""
        if not isinstance(precond, RasPreconditioner) or precond.engine is not self.engine:
            return NotImplemented
        e = self.engine
        x = e.vector(b.n)
        iters, conv = ctypes.c_int(), ctypes.c_int()
        resid = ctypes.c_double()
        hist = np.zeros(cfg.max_iters + 1)
        rc = e.lib.ocp_ras_gmres(
            e.ctx, ctypes.c_void_p(self.jd.addr), ctypes.c_void_p(precond.fac.addr), b.ptr,
            float(cfg.rel_tol), float(cfg.abs_tol), int(cfg.max_iters), x.ptr,
            ctypes.byref(iters), ctypes.byref(resid), ctypes.byref(conv),
            hist.ctypes.data_as(ctypes.POINTER(ctypes.c_double)))
        if rc == nat.OCP_ERR_GMRES_BREAKDOWN:
            raise GmresBreakdownError(e.error())
        e.check(rc, "ocp_ras_gmres")
        k = iters.value
        return GmresResult(x, k, resid.value, bool(conv.value), list(hist[:k + 1]))


def global_jacobian(engine, x, eps):
    return GlobalJacobian(engine, x, eps)


class RasPreconditioner:
    """One-level RAS on the Jacobian at x (`schwarz.py:221-239`), device factors."""

    def __init__(self, engine, x, eps, fac=None):
        xd, _ = _as_device(engine, x)
        self.engine, self.eps = engine, float(eps)
        self.fac = engine.factor_store() if fac is None else fac
        failed = ctypes.c_int(-1)
        rc = engine.lib.ocp_ras_factor(engine.ctx, xd.ptr, self.eps,
                                       ctypes.c_void_p(self.fac.addr), ctypes.byref(failed))
        if rc != nat.OCP_OK:
            _raise(engine, rc, "ocp_ras_factor", failed.value)

    def __call__(self, v):
        vd, dev = _as_device(self.engine, v)
        out = self.engine.vector(vd.n)
        self.engine.check(self.engine.lib.ocp_ras_apply(
            self.engine.ctx, ctypes.c_void_p(self.fac.addr), vd.ptr, out.ptr), "ocp_ras_apply")
        return out if dev else out.to_host()


def ras_preconditioner(x, dec, spec, eps, systems=None):
    """Left-preconditioner callable at x (`schwarz.py:221-239`); host or device vectors."""
    engine = systems if isinstance(systems, Engine) else build_local_systems(dec, spec)
    return RasPreconditioner(engine, x, eps)


def ras_precondition(v, x, dec, spec, eps):
    """Single application of the RAS preconditioner (`schwarz.py:242-244`)."""
    return ras_preconditioner(x, dec, spec, eps)(v)


def newton_ras_solve(x0, dec, spec, sched, cfg=None):
    """``solve_single``'s ``newton-ras*`` branch (`harness/experiments.py:72-84`).

    ``cfg`` is the outer NewtonConfig; its ``linear_solver`` must be a
    KrylovConfig (the harness uses rel_tol = gmres_tol, max_iters = 2000).
    Returns (x host array, SolveReport) like ``newton_continuation``.
    """
    cfg = cfg if cfg is not None else NewtonConfig(
        linear_solver=KrylovConfig(rel_tol=1e-8, max_iters=2000))
    if not isinstance(cfg.linear_solver, KrylovConfig):
        raise ValueError("newton-ras uses GMRES: cfg.linear_solver must be a KrylovConfig")
    engine = build_local_systems(dec, spec)
    x, report = solve_ras_on_device(engine, engine.from_host(np.asarray(x0, dtype=float)),
                                    sched, cfg)
    return x.to_host(), report


def solve_ras_on_device(engine, x0, sched, cfg):
    """newton-ras on a device-resident x0; returns (x DeviceVector, report)."""
    fac = engine.factor_store()   # one store, refactored at every outer iterate
    return newton_continuation(
        x0, lambda x, eps: global_residual(engine, x, eps),
        lambda x, eps: GlobalJacobian(engine, x, eps), sched, cfg,
        precond_builder=lambda x, eps: RasPreconditioner(engine, x, eps, fac))
