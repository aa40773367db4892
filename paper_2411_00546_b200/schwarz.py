"""RASPEN drop-in: same entry points as `pkg/src/ocp/schwarz.py`, arithmetic on the GPU.

Host side keeps what the reference keeps on the host: the tiling and index
sets (`schwarz.py:78-126`), the outer Newton / GMRES control flow and the
correction cache (`schwarz.py:348-411`).  Everything per subdomain - the
frozen-exterior local residuals, the batched damped local Newton with eps
continuation, in-kernel Jacobian assembly, block-Thomas factor/solve, the
refactorisation at the corrected values, the restricted prolongation and the
stored-factor Jacobian action - runs in ``libocpgpu.so`` (one native call per
RAS sweep, one per GMRES matvec).

Differences from the reference that do not change results:
* ``threads`` is accepted and ignored: all subdomains run batched on the GPU,
  deterministic by construction;
* the local direct solves are a no-pivot block-Thomas elimination (stored
  symmetric Schur inverses) instead of SuperLU (same
  solution to ~1e-13 relative);
* the JVP evaluates ``-(d_loc + J^{-1} A_ext d)`` on the ownership block, which
  is algebraically the reference's ``-J^{-1}(J d_loc + A_ext d)``.
"""

import math
from dataclasses import dataclass, field

import numpy as np

from . import _native as nat
from .engine import DeviceVector, Engine
from .grid import Grid, NonfiniteFieldError
from .krylov import KrylovConfig
from .newton import ContinuationSchedule, NewtonConfig, SolveReport, newton_continuation


class LocalSolveError(RuntimeError):
    """A subdomain correction solve failed; carries the subdomain id (`schwarz.py:32-37`)."""

    def __init__(self, subdomain, message):
        self.subdomain = subdomain
        super().__init__(f"subdomain {subdomain}: {message}")


@dataclass(frozen=True)
class Subdomain:
    """Index sets of one overlapping subdomain (`schwarz.py:40-63`)."""

    rows: tuple
    cols: tuple
    own_rows: tuple
    own_cols: tuple
    idx: np.ndarray
    own: np.ndarray
    own_in_local: np.ndarray
    pair_idx: np.ndarray
    pair_own: np.ndarray
    pair_own_in_local: np.ndarray

    @property
    def size(self):
        return self.idx.shape[0]


@dataclass(frozen=True, eq=False)
class Decomposition:
    grid: Grid
    s1: int
    s2: int
    overlap: int
    subdomains: tuple

    def __len__(self):
        return len(self.subdomains)


def _tile_edges(n, parts):
    """Near-equal split of range(n), remainder to the last tile (`schwarz.py:78-85`)."""
    base, rem = divmod(n, parts)
    if base == 0:
        raise ValueError(f"cannot tile {n} points into {parts} nonempty parts")
    edges = [base * k for k in range(parts)] + [n]
    return [(edges[k], edges[k + 1]) for k in range(parts)]


def _rect_indices(n, rows, cols):
    r = np.arange(rows[0], rows[1])
    c = np.arange(cols[0], cols[1])
    return (r[:, None] * n + c[None, :]).ravel()


def decompose(grid, s1, s2, m):
    """s1 x s2 ownership blocks dilated by m cells (`schwarz.py:94-126`)."""
    if s1 < 1 or s2 < 1:
        raise ValueError("need at least one tile per dimension")
    if m < 0:
        raise ValueError("overlap must be nonnegative")
    row_tiles = _tile_edges(grid.n, s1)
    col_tiles = _tile_edges(grid.n, s2)
    if s1 > 1 and m > min(b - a for a, b in row_tiles):
        raise ValueError("overlap exceeds neighbor tile in the row direction")
    if s2 > 1 and m > min(b - a for a, b in col_tiles):
        raise ValueError("overlap exceeds neighbor tile in the column direction")
    n2 = grid.size
    subs = []
    for r0, r1 in row_tiles:
        for c0, c1 in col_tiles:
            rows = (max(0, r0 - m), min(grid.n, r1 + m))
            cols = (max(0, c0 - m), min(grid.n, c1 + m))
            idx = _rect_indices(grid.n, rows, cols)
            own = _rect_indices(grid.n, (r0, r1), (c0, c1))
            oil = np.searchsorted(idx, own)
            subs.append(Subdomain(
                rows=rows, cols=cols, own_rows=(r0, r1), own_cols=(c0, c1), idx=idx, own=own,
                own_in_local=oil, pair_idx=np.concatenate([idx, idx + n2]),
                pair_own=np.concatenate([own, own + n2]),
                pair_own_in_local=np.concatenate([oil, oil + idx.shape[0]])))
    return Decomposition(grid=grid, s1=s1, s2=s2, overlap=m, subdomains=tuple(subs))


# ---------------------------------------------------------------------------
# device local systems
# ---------------------------------------------------------------------------

ENGINE_CACHE_SIZE = 2   # engines kept per decomposition (most recently used problems)


def build_local_systems(dec, spec):
    """Device-side local systems of (dec, spec): the native engine (`schwarz.py:144-163`).

    The reference slices CSR blocks a_loc / a_ext; the device applies the same
    stencil matrix-free, so "building" means uploading f, y_d and the
    subdomain table once.  Engines are cached on the decomposition for the
    ``ENGINE_CACHE_SIZE`` most recently used problems; older ones are dropped,
    which frees their device memory (a sweep over many ProblemSpecs does not
    accumulate contexts).  An engine serialises its calls on one CUDA stream
    and shares its scratch buffers between calls: it is not safe to use the
    same (dec, spec) from several Python threads at once.
    """
    cache = dec.__dict__.setdefault("_engines", [])
    for k, (s, eng) in enumerate(cache):
        if s is spec:
            cache.append(cache.pop(k))   # most recently used last
            return eng
    eng = Engine(spec, dec.s1, dec.s2, dec.overlap)
    if eng.num_subdomains != len(dec):
        raise ValueError("decomposition does not match the native tiling")
    cache.append((spec, eng))
    while len(cache) > ENGINE_CACHE_SIZE:
        cache.pop(0)
    return eng


def release_local_systems(dec, spec=None):
    """Drop the cached engine of ``spec`` (all engines when None) from ``dec``."""
    cache = dec.__dict__.get("_engines", [])
    cache[:] = [] if spec is None else [(s, e) for s, e in cache if s is not spec]


def _engine(dec, spec, systems):
    return systems if isinstance(systems, Engine) else build_local_systems(dec, spec)


def _raise_native(engine, rc, failed):
    msg = engine.error()
    if rc == nat.OCP_ERR_LOCAL_SOLVE:
        raise LocalSolveError(failed, msg)
    if rc == nat.OCP_ERR_NONFINITE:
        where, _, idx = msg.rpartition("@")
        raise NonfiniteFieldError(where, int(idx))
    if rc == nat.OCP_ERR_NONFINITE_INIT:
        raise ValueError(msg)
    raise nat.NativeError(rc, msg, "ocp_raspen_residual")


def _sweep(engine, x, fac, sched, inner_cfg, fval=None, eps=None):
    """One batched RAS sweep on device vectors -> (f_val, per-subdomain inner iterations).

    The local Jacobians are refactored at ``eps`` (default: the schedule's
    floor, the only case raspen_solve produces), `schwarz.py:305-315`.
    """
    fval = engine.vector() if fval is None else fval
    iters = np.zeros(engine.num_subdomains, dtype=np.int32)
    failed = np.zeros(1, dtype=np.int32)
    ip = iters.ctypes.data_as(nat.ctypes.POINTER(nat.ctypes.c_int))
    fp = failed.ctypes.data_as(nat.ctypes.POINTER(nat.ctypes.c_int))
    args = (float(sched.eps0), float(sched.gamma), float(sched.eps_min), float(inner_cfg.tol),
            int(inner_cfg.max_outer), float(inner_cfg.sigma), int(inner_cfg.max_halvings),
            fval.ptr, ip, fp)
    facp = nat.ctypes.c_void_p(fac.addr)
    if eps is None or eps == sched.eps_min:
        rc = engine.lib.ocp_raspen_residual(engine.ctx, x.ptr, facp, *args)
    else:
        rc = engine.lib.ocp_raspen_residual_at(engine.ctx, x.ptr, facp, float(eps), *args)
    if rc != nat.OCP_OK:
        _raise_native(engine, rc, int(failed[0]))
    return fval, [int(k) for k in iters]


def _jvp(engine, fac, d, out=None):
    out = engine.vector(d.n) if out is None else out
    engine.check(engine.lib.ocp_raspen_jvp(engine.ctx, nat.ctypes.c_void_p(fac.addr), d.ptr,
                                           out.ptr), "ocp_raspen_jvp")
    return out


@dataclass
class CorrectionSet:
    """Cached subdomain solves for one iterate (`schwarz.py:267-282`).

    ``lus`` is the device factor store of the refactorisation at the values;
    ``values`` are the local values in the reference layout (host copies).
    """

    token: int
    x: np.ndarray
    eps: float
    f_val: np.ndarray
    values: list
    jac_locs: object
    lus: object
    inner_iters: list
    systems: object = field(repr=False, default=None)


_token_counter = [0]


def raspen_residual(x, dec, spec, eps, inner_cfg=None, inner_sched=None, threads=None,
                    systems=None):
    """Fixed-point residual sum_i P~_i C_i(x) - x and the stored local factors (`schwarz.py:285-324`)."""
    engine = _engine(dec, spec, systems)
    cfg = inner_cfg if inner_cfg is not None else NewtonConfig(tol=1e-8)
    sched = inner_sched if inner_sched is not None else ContinuationSchedule.fixed(eps)
    x = np.asarray(x, dtype=float)
    xd = engine.from_host(x)
    fac = engine.factor_store()
    fval_d, inner = _sweep(engine, xd, fac, sched, cfg, eps=eps)
    f_val = fval_d.to_host()
    values = _local_values(engine, dec)
    _token_counter[0] += 1
    return f_val, CorrectionSet(token=_token_counter[0], x=x.copy(), eps=eps, f_val=f_val,
                                values=values, jac_locs=_LocalJacobians(dec, spec, values, eps), lus=fac,
                                inner_iters=inner, systems=engine)


def _local_values(engine, dec):
    """Current local values of every subdomain, reference layout (host copies)."""
    flat = engine.vector(engine.ref_len)
    engine.check(engine.lib.ocp_local_values(engine.ctx, flat.ptr), "ocp_local_values")
    flat_h = flat.to_host()
    values, off = [], 0
    for sub in dec.subdomains:
        values.append(flat_h[off:off + 2 * sub.size].copy())
        off += 2 * sub.size
    return values


class _LocalJacobians:
    """``CorrectionSet.jac_locs`` (`schwarz.py:321`): the local Jacobians at the values.

    The device path never assembles them - their diagonals are regenerated
    inside the factor kernel and only the factor store (``lus``) is kept - so
    entry i is built on the host on first access, exactly as
    `_local_pair_jacobian` builds it (`schwarz.py:166-171`): CSR
    ``[[A_loc + diag(phi'(y)), diag(b12)], [diag(b21), A_loc + diag(phi'(y))]]``
    at the local values and eps.  Inspection only; the JVP does not use it.
    """

    def __init__(self, dec, spec, values, eps):
        self.dec, self.spec, self.values, self.eps = dec, spec, values, eps
        self._cache = {}

    def __len__(self):
        return len(self.values)

    def __iter__(self):
        return (self[i] for i in range(len(self)))

    def __getitem__(self, i):
        if i < 0:
            i += len(self)
        if i not in self._cache:
            self._cache[i] = _assemble_local_jacobian(self.dec.subdomains[i], self.spec,
                                                      self.values[i], self.eps)
        return self._cache[i]


def _assemble_local_jacobian(sub, spec, v, eps):
    import scipy.sparse as sp
    from .system import smoothed_projection_derivative
    rows = sub.rows[1] - sub.rows[0]
    cols = sub.cols[1] - sub.cols[0]
    size = rows * cols
    h2 = spec.grid.h ** 2
    t_r = sp.diags([np.full(rows - 1, -1.0), np.full(rows, 2.0), np.full(rows - 1, -1.0)],
                   [-1, 0, 1])
    t_c = sp.diags([np.full(cols - 1, -1.0), np.full(cols, 2.0), np.full(cols - 1, -1.0)],
                   [-1, 0, 1])
    a_loc = ((sp.kron(t_r, sp.identity(cols)) + sp.kron(sp.identity(rows), t_c)) / h2).tocsr()
    y, p = v[:size], v[size:]
    dphi = spec.phi.derivative(y)
    b12 = (1.0 - smoothed_projection_derivative(-p / spec.mu, eps)) / spec.nu
    b21 = spec.phi.second_derivative(y) * p - 1.0
    a11 = a_loc + sp.diags(dphi)
    return sp.bmat([[a11, sp.diags(b12)], [sp.diags(b21), a11]], format="csr")


def raspen_jacobian_apply(x, d, dec, spec, eps, corrections):
    """Jacobian action from the stored local factors (`schwarz.py:327-345`)."""
    if corrections.eps != eps or not np.array_equal(corrections.x, x):
        raise RuntimeError("stale corrections: recompute raspen_residual at this iterate")
    engine = corrections.systems if corrections.systems is not None else _engine(dec, spec, None)
    dd = engine.from_host(np.asarray(d, dtype=float))
    return _jvp(engine, corrections.lus, dd).to_host()


def ras_fixed_point_step(x, dec, spec, eps, inner_cfg=None, inner_sched=None, threads=None,
                         systems=None):
    """One nonlinear RAS sweep recombined by ownership (`schwarz.py:253-264`)."""
    f_val, _ = raspen_residual(x, dec, spec, eps, inner_cfg, inner_sched, threads, systems)
    return f_val + np.asarray(x, dtype=float)


def local_correction(i, x, dec, spec, eps, inner_cfg=None, inner_sched=None, systems=None):
    """Local values solving the frozen-exterior system on subdomain i (`schwarz.py:211-218`).

    Only subdomain i is solved (``ocp_local_correction``), so a failure
    elsewhere cannot surface here; its failure raises LocalSolveError(i).
    """
    engine = _engine(dec, spec, systems)
    cfg = inner_cfg if inner_cfg is not None else NewtonConfig(tol=1e-8)
    sched = inner_sched if inner_sched is not None else ContinuationSchedule.fixed(eps)
    if not 0 <= i < len(dec):
        raise IndexError(f"subdomain {i} out of range")
    xd = engine.from_host(np.asarray(x, dtype=float))
    iters = np.zeros(engine.num_subdomains, dtype=np.int32)
    failed = np.zeros(1, dtype=np.int32)
    fac = engine.factor_store()
    rc = engine.lib.ocp_local_correction(
        engine.ctx, xd.ptr, nat.ctypes.c_void_p(fac.addr), int(i), float(sched.eps0),
        float(sched.gamma), float(sched.eps_min),
        float(cfg.tol), int(cfg.max_outer), float(cfg.sigma), int(cfg.max_halvings),
        iters.ctypes.data_as(nat.ctypes.POINTER(nat.ctypes.c_int)),
        failed.ctypes.data_as(nat.ctypes.POINTER(nat.ctypes.c_int)))
    if rc != nat.OCP_OK:
        _raise_native(engine, rc, int(failed[0]))
    return _local_values(engine, dec)[i]


def raspen_solve(x0, dec, spec, sched, cfg=None, krylov_cfg=None, inner_tol=1e-8,
                 inner_max_outer=200, threads=None, continuation=True, backtracking=False):
    """Outer Newton on the fixed-point residual at eps_min, full steps (`schwarz.py:348-411`).

    Returns (x, SolveReport) with host arrays, like the reference.  The
    report also carries ``per_subdomain_inner`` (per-evaluation lists of
    per-subdomain inner iterations; the reference keeps them internally).
    """
    engine = build_local_systems(dec, spec)
    x0 = np.asarray(x0, dtype=float)
    x, report = solve_on_device(engine, engine.from_host(x0), sched, cfg, krylov_cfg, inner_tol,
                                inner_max_outer, continuation, backtracking)
    if x is None:
        return np.array(x0, dtype=float, copy=True), report
    return x.to_host(), report


class _RaspenOperator:
    """Jacobian action of the fixed-point residual at one iterate (schwarz.py:384-395).

    Callable on device vectors (generic GMRES) and with a fused native GMRES
    for the unpreconditioned, unrestarted solve raspen_solve performs.
    """

    def __init__(self, engine, fac, state, corr):
        self.engine, self.fac, self.state, self.corr = engine, fac, state, corr

    def _check(self):
        if self.state["corr"] is not self.corr:
            raise RuntimeError("stale corrections: a newer iterate was evaluated")

    def __call__(self, d):
        self._check()
        return _jvp(self.engine, self.fac, d)

    def fused_gmres(self, b, cfg, precond=None):
        from .krylov import GmresBreakdownError, GmresResult
        if precond is not None:
            return NotImplemented
        self._check()
        e = self.engine
        x = e.vector(b.n)
        iters = nat.ctypes.c_int()
        conv = nat.ctypes.c_int()
        resid = nat.ctypes.c_double()
        hist = np.zeros(cfg.max_iters + 1)
        rc = e.lib.ocp_raspen_gmres(
            e.ctx, nat.ctypes.c_void_p(self.fac.addr), b.ptr, float(cfg.rel_tol),
            float(cfg.abs_tol), int(cfg.max_iters), x.ptr, nat.ctypes.byref(iters),
            nat.ctypes.byref(resid), nat.ctypes.byref(conv),
            hist.ctypes.data_as(nat.ctypes.POINTER(nat.ctypes.c_double)))
        if rc == nat.OCP_ERR_GMRES_BREAKDOWN:
            raise GmresBreakdownError(e.error())
        e.check(rc, "ocp_raspen_gmres")
        k = iters.value
        return GmresResult(x, k, resid.value, bool(conv.value), list(hist[:k + 1]))


def solve_on_device(engine, x0, sched, cfg=None, krylov_cfg=None, inner_tol=1e-8,
                    inner_max_outer=200, continuation=True, backtracking=False):
    """raspen_solve on a device-resident x0; returns (x DeviceVector or None on failure, report)."""
    cfg = cfg if cfg is not None else NewtonConfig()
    krylov_cfg = krylov_cfg if krylov_cfg is not None else KrylovConfig(rel_tol=1e-8, max_iters=400)
    inner_cfg = NewtonConfig(tol=inner_tol, max_outer=inner_max_outer)
    eps_min = sched.eps_min
    fac = engine.factor_store()
    state = {"corr": None, "evals": 0, "inner_hist": [], "per_sub": []}

    def residual_fn(x, eps):
        corr = state["corr"]
        if corr is not None and corr["eps"] == eps and corr["x"].equals(x):
            return corr["f_val"].copy()
        if continuation and state["evals"] == 0:
            inner_sched = ContinuationSchedule(sched.eps0, sched.gamma, eps)
        else:
            inner_sched = ContinuationSchedule.fixed(eps)
        state["corr"] = None  # the factor store is about to be overwritten
        f_val, inner = _sweep(engine, x, fac, inner_sched, inner_cfg)
        corr = {"x": x.copy(), "eps": eps, "f_val": f_val}
        state["corr"] = corr
        state["evals"] += 1
        state["inner_hist"].append(max(inner))
        state["per_sub"].append(list(inner))
        return f_val.copy()

    def jacobian_fn(x, eps):
        corr = state["corr"]
        if corr is None or corr["eps"] != eps or not corr["x"].equals(x):
            raise RuntimeError("Jacobian requested before a residual evaluation at this iterate")

        return _RaspenOperator(engine, fac, state, corr)

    outer_cfg = NewtonConfig(tol=cfg.tol, max_outer=cfg.max_outer,
                             sigma=cfg.sigma if backtracking else math.inf,
                             max_halvings=cfg.max_halvings, linear_solver=krylov_cfg)
    try:
        x, report = newton_continuation(x0, residual_fn, jacobian_fn,
                                        ContinuationSchedule.fixed(eps_min), outer_cfg)
    except LocalSolveError as exc:
        report = SolveReport(False, max(state["evals"] - 1, 0),
                             inner_iters=list(state["inner_hist"]), failure=str(exc))
        report.per_subdomain_inner = list(state["per_sub"])
        return None, report
    report.inner_iters = list(state["inner_hist"])
    report.per_subdomain_inner = list(state["per_sub"])
    return x, report
