"""CPU ORACLE for the RASPEN hot path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline
leg may import this module, and only as the checker / CPU baseline.  The
product package (``paper_2411_00546_b200``) never imports it.

What it is: a numpy/scipy restatement of the reference's one-level RASPEN
solve with inner eps-continuation (method ``raspen-eps``).  Every function
cites the reference lines it follows (paths relative to /root/reference).
The reference is pure Python; its arithmetic lives in third-party native code
that is NOT under /root/reference:

* SciPy SuperLU (``scipy.sparse.linalg.splu``: COLAMD ordering + partial
  pivoting, ``gstrf``/``gstrs``) for every local factor/solve, pinned here to
  the image's scipy 1.18.1 (reference pin: ``scipy>=1.10``, `pkg/pyproject.toml:10-13`);
* SciPy sparsetools CSR matvec and NumPy/OpenBLAS dot/nrm2 (numpy 2.3.5).

The oracle calls the same library routines (SuperLU is the published
algorithm; restating it would only add error), so on identical inputs it
reproduces the reference's results bitwise or to the last few ulps.

Pinning: ``tests/test_oracle_golden.py`` checks this module against fixtures
produced by the UNMODIFIED reference (``tests/golden/make_golden.py``).
"""

from concurrent.futures import ThreadPoolExecutor
import math
import os

import numpy as np
import scipy.sparse as sp
import scipy.sparse.linalg as spla

EXP_ARG_MAX = 700.0


class OracleLinearFailure(RuntimeError):
    """GMRES did not converge (LinearSolveError, `newton.py:119-123`)."""


class OracleLocalFailure(RuntimeError):
    def __init__(self, sub, message):
        self.subdomain = sub
        super().__init__(f"subdomain {sub}: {message}")


# --------------------------------------------------------------------------
# pointwise maps (`pkg/src/ocp/smoothing.py:19-44`, `pkg/src/ocp/system.py:118-144`)
# --------------------------------------------------------------------------

def p_eps(x, eps):
    """P_eps; the square is x*x exactly like numpy's ``** 2`` (`smoothing.py:32`)."""
    a = x + 1.0
    b = x - 1.0
    return 0.5 * (np.sqrt(a * a + eps) - np.sqrt(b * b + eps))


def dp_eps(x, eps):
    """P'_eps (`smoothing.py:43-44`)."""
    a = x + 1.0
    b = x - 1.0
    return 0.5 * (a / np.sqrt(a * a + eps) - b / np.sqrt(b * b + eps))


def rows_from_actions(ay, ap, y, p, f, yd, phi, nu, mu, eps):
    """Residual rows with the operator action precomputed (`system.py:118-132`).

    Evaluation order: ``((ay + phi(y)) - f) + ctrl`` and ``((ap + phi'(y) p) - y) + y_d``.
    """
    with np.errstate(over="ignore", invalid="ignore"):
        ctrl = (p + mu * p_eps(-p / mu, eps)) / nu
        r1 = ay + phi.value(y, check=False) - f + ctrl
        r2 = ap + phi.derivative(y, check=False) * p - y + yd
    return r1, r2


def jac_diagonals(y, p, phi, nu, mu, eps):
    """(phi'(y), b12, b21) of the 2x2 block Jacobian (`system.py:135-144`)."""
    return (phi.derivative(y), (1.0 - dp_eps(-p / mu, eps)) / nu,
            phi.second_derivative(y) * p - 1.0)


# --------------------------------------------------------------------------
# decomposition (`pkg/src/ocp/schwarz.py:78-126`)
# --------------------------------------------------------------------------

def tile_edges(n, parts):
    """Equal tiles, remainder to the last one (`schwarz.py:78-85`)."""
    base, rem = divmod(n, parts)
    if base == 0:
        raise ValueError(f"cannot tile {n} points into {parts} nonempty parts")
    edges = [k * base for k in range(parts)] + [n]
    return [(edges[k], edges[k + 1]) for k in range(parts)]


class Rect:
    """One overlapping subdomain: rectangle, ownership block and index sets."""

    def __init__(self, n, rows, cols, own_rows, own_cols):
        self.rows, self.cols = rows, cols
        self.own_rows, self.own_cols = own_rows, own_cols
        r = np.arange(*rows)
        c = np.arange(*cols)
        self.idx = (r[:, None] * n + c[None, :]).ravel()
        ro = np.arange(*own_rows)
        co = np.arange(*own_cols)
        self.own = (ro[:, None] * n + co[None, :]).ravel()
        self.own_in_local = np.searchsorted(self.idx, self.own)
        n2 = n * n
        m = self.idx.shape[0]
        self.pair_idx = np.concatenate([self.idx, self.idx + n2])
        self.pair_own = np.concatenate([self.own, self.own + n2])
        self.pair_own_in_local = np.concatenate([self.own_in_local, self.own_in_local + m])

    @property
    def size(self):
        return self.idx.shape[0]


def decompose(n, s1, s2, m):
    """s1 x s2 ownership tiles dilated by m, clipped to the grid (`schwarz.py:94-126`)."""
    if s1 < 1 or s2 < 1:
        raise ValueError("need at least one tile per dimension")
    if m < 0:
        raise ValueError("overlap must be nonnegative")
    rt, ct = tile_edges(n, s1), tile_edges(n, s2)
    if s1 > 1 and m > min(b - a for a, b in rt):
        raise ValueError("overlap exceeds neighbor tile in the row direction")
    if s2 > 1 and m > min(b - a for a, b in ct):
        raise ValueError("overlap exceeds neighbor tile in the column direction")
    return [Rect(n, (max(0, r0 - m), min(n, r1 + m)), (max(0, c0 - m), min(n, c1 + m)),
                 (r0, r1), (c0, c1))
            for r0, r1 in rt for c0, c1 in ct]


class LocalOps:
    """a_loc (rect-internal stencil) and a_ext (frozen exterior coupling).

    Built straight from the stencil with column indices sorted per row, which
    is the entry order the reference gets by slicing the kron Laplacian
    (`schwarz.py:144-163`, `grid.py:83-91`); CSR matvec sums in that order.
    """

    def __init__(self, n, rect):
        h2 = (1.0 / (n + 1)) ** 2
        diag, off = 4.0 / h2, -1.0 / h2
        r0, r1 = rect.rows
        c0, c1 = rect.cols
        nr, nc = r1 - r0, c1 - c0
        size = nr * nc
        row = np.arange(size)
        i = r0 + row // nc
        j = c0 + row % nc
        li, le = ([], [], []), ([], [], [])
        for di, dj in ((-1, 0), (0, -1), (0, 0), (0, 1), (1, 0)):
            ii, jj = i + di, j + dj
            ok = (ii >= 0) & (ii < n) & (jj >= 0) & (jj < n)
            inside = ok & (ii >= r0) & (ii < r1) & (jj >= c0) & (jj < c1)
            outside = ok & ~inside
            val = diag if di == 0 and dj == 0 else off
            li[0].append(row[inside])
            li[1].append((ii[inside] - r0) * nc + (jj[inside] - c0))
            li[2].append(np.full(int(inside.sum()), val))
            le[0].append(row[outside])
            le[1].append(ii[outside] * n + jj[outside])
            le[2].append(np.full(int(outside.sum()), val))
        li = [np.concatenate(t) for t in li]
        le = [np.concatenate(t) for t in le]
        self.a_loc = sp.csr_matrix((li[2], (li[0], li[1])), shape=(size, size))
        self.a_ext = sp.csr_matrix((le[2], (le[0], le[1])), shape=(size, n * n))
        self.a_loc.sort_indices()
        self.a_ext.sort_indices()


# --------------------------------------------------------------------------
# generic damped Newton with eps-continuation (`pkg/src/ocp/newton.py:96-181`)
# --------------------------------------------------------------------------

def next_eps(eps, gamma, eps_min):
    return max(gamma * eps, eps_min)


def newton(x0, F, J_solve, eps0, gamma, eps_min, tol, max_outer, sigma, max_halvings):
    """Algorithm 1 (`newton.py:133-181`) with a direct direction solve.

    Returns (x, converged, iters, failure, history) where ``history`` holds
    (residual_norms, eps_values, alphas).
    """
    x = np.array(x0, dtype=float, copy=True)
    eps = eps0
    r = F(x, eps)
    nrm = float(np.linalg.norm(r))
    if not np.isfinite(nrm):
        raise ValueError("nonfinite residual at the initial guess")
    thr = max(tol, tol * nrm)                         # newton.py:148
    norms, epss, alphas = [nrm], [eps], []
    iters = 0
    while True:
        if nrm <= thr and eps == eps_min:             # newton.py:153
            return x, True, iters, None, (norms, epss, alphas)
        if iters >= max_outer:
            return x, False, iters, f"no convergence within {max_outer} outer iterations", \
                (norms, epss, alphas)
        try:
            d = J_solve(x, eps, -r)
        except OracleLinearFailure as exc:            # newton.py:119-123 (GMRES)
            return x, False, iters, str(exc), (norms, epss, alphas)
        except RuntimeError as exc:                   # newton.py:126-129
            return x, False, iters, f"sparse factorization failed: {exc}", (norms, epss, alphas)
        alpha, ok = 1.0, False                        # backtrack, newton.py:96-112
        for _ in range(max_halvings + 1):
            trial = float(np.linalg.norm(F(x + alpha * d, eps)))
            if np.isfinite(trial) and trial <= sigma * nrm:
                ok = True
                break
            alpha *= 0.5
        if not ok:
            return x, False, iters, (f"no admissible step within {max_halvings} halvings "
                                     f"(residual {nrm:.3e})"), (norms, epss, alphas)
        x += alpha * d
        eps = next_eps(eps, gamma, eps_min)
        r = F(x, eps)
        nrm = float(np.linalg.norm(r))
        iters += 1
        norms.append(nrm)
        epss.append(eps)
        alphas.append(alpha)


# --------------------------------------------------------------------------
# GMRES (`pkg/src/ocp/krylov.py:44-151`), unrestarted, MGS Arnoldi
# --------------------------------------------------------------------------

def gmres(apply_op, b, rel_tol, max_iters, abs_tol=0.0, precond=None):
    """Left-preconditioned when ``precond`` is given (`krylov.py:54-60,110`)."""
    m = precond if precond is not None else (lambda v: v)
    b = m(np.asarray(b, dtype=float))
    thr = max(rel_tol * float(np.linalg.norm(b)), abs_tol)
    beta = float(np.linalg.norm(b))
    history = [beta]
    if not np.isfinite(beta):
        raise FloatingPointError("nonfinite initial residual")
    if beta <= thr:
        return np.zeros_like(b), 0, beta, True, history
    # basis columns live in one (n, cap+1) array that doubles when full, the
    # layout the reference uses (`krylov.py:89-107`); BLAS ddot on strided
    # columns rounds differently from contiguous vectors, so keep it.
    cap = min(32, max_iters)
    q = np.empty((b.shape[0], cap + 1))
    q[:, 0] = b / beta
    cs, sn, cols = [], [], []
    g = np.zeros(max_iters + 1)
    g[0] = beta
    conv = False
    resid = beta
    steps = 0
    for j in range(max_iters):
        if j + 1 > cap:
            cap = min(2 * cap, max_iters)
            grown = np.empty((b.shape[0], cap + 1))
            grown[:, :j + 1] = q[:, :j + 1]
            q = grown
        w = np.array(m(apply_op(q[:, j])), dtype=float, copy=True)
        h = np.empty(j + 2)
        with np.errstate(invalid="ignore", over="ignore"):
            for i in range(j + 1):
                h[i] = float(np.dot(q[:, i], w))
                w -= h[i] * q[:, i]
            h[j + 1] = float(np.linalg.norm(w))
        if not np.all(np.isfinite(h)):
            raise FloatingPointError(f"nonfinite Arnoldi entries at iteration {j + 1}")
        happy = h[j + 1] <= 1e-14 * max(1.0, float(np.max(np.abs(h[:j + 1]))))
        if not happy:
            q[:, j + 1] = w / h[j + 1]
        for i in range(j):                            # apply previous rotations
            hi = cs[i] * h[i] + sn[i] * h[i + 1]
            h[i + 1] = -sn[i] * h[i] + cs[i] * h[i + 1]
            h[i] = hi
        rad = float(np.hypot(h[j], h[j + 1]))
        c, s = (1.0, 0.0) if rad == 0.0 else (h[j] / rad, h[j + 1] / rad)
        cs.append(c)
        sn.append(s)
        h[j] = rad
        g[j + 1] = -s * g[j]
        g[j] = c * g[j]
        cols.append(h[:j + 1].copy())
        resid = abs(float(g[j + 1]))
        history.append(resid)
        steps = j + 1
        if resid <= thr or happy:
            conv = True
            break
    rmat = np.zeros((steps, steps))
    for col, vals in enumerate(cols):
        rmat[:col + 1, col] = vals
    y = np.zeros(steps)
    for i in range(steps - 1, -1, -1):
        y[i] = (g[i] - float(np.dot(rmat[i, i + 1:], y[i + 1:]))) / rmat[i, i]
    return q[:, :steps] @ y, steps, resid, conv, history


# --------------------------------------------------------------------------
# RASPEN (`pkg/src/ocp/schwarz.py:166-411`)
# --------------------------------------------------------------------------

class Problem:
    """Problem data + decomposition + local operators (setup, not timed)."""

    def __init__(self, n, s1, s2, m, phi, nu, mu, f, y_d):
        self.n, self.phi, self.nu, self.mu = n, phi, nu, mu
        self.f, self.y_d = np.asarray(f, float), np.asarray(y_d, float)
        self.rects = decompose(n, s1, s2, m)
        self.ops = [LocalOps(n, r) for r in self.rects]

    def local_fns(self, i, x):
        """Frozen-exterior local residual and Jacobian (`schwarz.py:166-191`)."""
        rect, op = self.rects[i], self.ops[i]
        size = rect.size
        n2 = self.n * self.n
        e_y = op.a_ext @ x[:n2]
        e_p = op.a_ext @ x[n2:]
        f_loc, yd_loc = self.f[rect.idx], self.y_d[rect.idx]
        phi, nu, mu = self.phi, self.nu, self.mu

        def F(v, eps):
            y, p = v[:size], v[size:]
            r1, r2 = rows_from_actions(op.a_loc @ y + e_y, op.a_loc @ p + e_p, y, p,
                                       f_loc, yd_loc, phi, nu, mu, eps)
            return np.concatenate([r1, r2])

        def J(v, eps):
            y, p = v[:size], v[size:]
            d1, b12, b21 = jac_diagonals(y, p, phi, nu, mu, eps)
            a11 = op.a_loc + sp.diags(d1)
            return sp.bmat([[a11, sp.diags(b12)], [sp.diags(b21), a11]], format="csr")

        return F, J

    def local_solve(self, i, x, eps0, gamma, eps_min, tol, max_outer):
        """One subdomain's damped Newton (`schwarz.py:194-200`)."""
        F, J = self.local_fns(i, x)

        def J_solve(v, eps, rhs):
            return spla.splu(J(v, eps).tocsc()).solve(rhs)

        v, ok, k, failure, _ = newton(x[self.rects[i].pair_idx], F, J_solve, eps0, gamma,
                                      eps_min, tol, max_outer, 1.1, 30)
        if not ok:
            raise OracleLocalFailure(i, failure)
        return v, k


def _pmap(fn, items, threads):
    if threads == 1 or len(items) == 1:
        return [fn(*it) for it in items]
    workers = threads if threads else min(len(items), os.cpu_count() or 1)
    with ThreadPoolExecutor(max_workers=workers) as pool:
        return list(pool.map(lambda it: fn(*it), items))


class Corrections:
    def __init__(self, x, eps, f_val, values, jacs, lus, inner):
        self.x, self.eps, self.f_val = x, eps, f_val
        self.values, self.jacs, self.lus, self.inner = values, jacs, lus, inner


def raspen_residual(prob, x, eps, eps0=None, gamma=1.0, tol=1e-8, max_outer=200,
                    threads=None, subset=None):
    """sum_i P~_i C_i(x) - x and the factors at the corrected values (`schwarz.py:285-324`).

    ``subset`` restricts the sweep to some subdomains (CPU-baseline sampling);
    f_val is then only meaningful on their ownership blocks.
    """
    eps0 = eps if eps0 is None else eps0
    ids = list(range(len(prob.rects))) if subset is None else list(subset)
    res = _pmap(lambda i: prob.local_solve(i, x, eps0, gamma, eps, tol, max_outer),
                [(i,) for i in ids], threads)
    values = {i: v for i, (v, _) in zip(ids, res)}
    inner = [k for _, k in res]

    def factor(i):
        _, J = prob.local_fns(i, x)
        jl = J(values[i], eps)
        return jl, spla.splu(jl.tocsc())

    fac = _pmap(factor, [(i,) for i in ids], threads)
    out = np.zeros_like(x)
    for i in ids:
        r = prob.rects[i]
        out[r.pair_own] = values[i][r.pair_own_in_local]
    f_val = out - x
    return f_val, Corrections(x.copy(), eps, f_val, values,
                              {i: j for i, (j, _) in zip(ids, fac)},
                              {i: lu for i, (_, lu) in zip(ids, fac)}, inner)


def raspen_jvp(prob, x, d, eps, corr):
    """Jacobian action from the stored local factors (`schwarz.py:327-345`)."""
    if corr.eps != eps or not np.array_equal(corr.x, x):
        raise RuntimeError("stale corrections: recompute raspen_residual at this iterate")
    n2 = prob.n * prob.n
    dy, dp = d[:n2], d[n2:]
    out = np.zeros_like(d)
    for i in corr.lus:
        r, op = prob.rects[i], prob.ops[i]
        rhs = corr.jacs[i] @ d[r.pair_idx] + np.concatenate([op.a_ext @ dy, op.a_ext @ dp])
        w = corr.lus[i].solve(rhs)
        out[r.pair_own] = -w[r.pair_own_in_local]
    return out


def raspen_solve(prob, x0, eps0, gamma, eps_min, tol=1e-10, max_outer=200,
                 gmres_rel=1e-8, gmres_max=1000, inner_tol=1e-8, inner_max_outer=200,
                 threads=None, continuation=True):
    """Outer Newton on the fixed-point residual, full steps (`schwarz.py:348-411`).

    Returns (x, report dict).  A local failure returns x0 and a failed report
    (`schwarz.py:405-409`).
    """
    st = {"corr": None, "evals": 0, "inner": [], "per_sub": []}

    def resid(x):
        c = st["corr"]
        if c is not None and c.eps == eps_min and np.array_equal(c.x, x):
            return c.f_val.copy()
        e0, g = (eps0, gamma) if (continuation and st["evals"] == 0) else (eps_min, 1.0)
        f_val, c = raspen_residual(prob, x, eps_min, e0, g, inner_tol, inner_max_outer,
                                   threads)
        st["corr"] = c
        st["evals"] += 1
        st["inner"].append(max(c.inner))
        st["per_sub"].append(list(c.inner))
        return f_val.copy()

    rep = {"converged": False, "outer_iters": 0, "residual_norms": [], "eps_values": [],
           "alphas": [], "gmres_iters": [], "inner_iters": [], "per_sub": [],
           "failure": None}
    x = np.array(x0, dtype=float, copy=True)
    try:
        r = resid(x)
        nrm = float(np.linalg.norm(r))
        if not np.isfinite(nrm):
            raise ValueError("nonfinite residual at the initial guess")
        thr = max(tol, tol * nrm)
        rep["threshold"] = thr
        rep["residual_norms"].append(nrm)
        rep["eps_values"].append(eps_min)
        while True:
            if nrm <= thr:
                rep["converged"] = True
                break
            if rep["outer_iters"] >= max_outer:
                rep["failure"] = f"no convergence within {max_outer} outer iterations"
                break
            corr = st["corr"]
            d, k, gres, conv, _ = gmres(lambda v: raspen_jvp(prob, x, v, eps_min, corr),
                                        -r, gmres_rel, gmres_max)
            if not conv:
                rep["failure"] = f"GMRES stalled at residual {gres:.3e} after {k} iterations"
                break
            alpha = 1.0                                # sigma = inf: first finite trial
            for _ in range(31):
                trial = float(np.linalg.norm(resid(x + alpha * d)))
                if np.isfinite(trial):
                    break
                alpha *= 0.5
            else:
                rep["failure"] = "no admissible step within 30 halvings"
                break
            x += alpha * d
            r = resid(x)
            nrm = float(np.linalg.norm(r))
            rep["outer_iters"] += 1
            rep["alphas"].append(alpha)
            rep["gmres_iters"].append(k)
            rep["residual_norms"].append(nrm)
            rep["eps_values"].append(eps_min)
    except OracleLocalFailure as exc:
        rep["outer_iters"] = max(st["evals"] - 1, 0)
        rep["inner_iters"] = list(st["inner"])
        rep["per_sub"] = list(st["per_sub"])
        rep["failure"] = str(exc)
        return np.array(x0, dtype=float, copy=True), rep
    rep["inner_iters"] = list(st["inner"])
    rep["per_sub"] = list(st["per_sub"])
    return x, rep


# --------------------------------------------------------------------------
# linear-RAS Newton-Krylov, method newton-ras-eps (`harness/experiments.py:72-84`)
# --------------------------------------------------------------------------

def laplacian(n):
    """Kron-sum 5-point Laplacian / h^2, CSR with sorted columns (`grid.py:83-91`)."""
    h2 = (1.0 / (n + 1)) ** 2
    t = sp.diags([-np.ones(n - 1), 2.0 * np.ones(n), -np.ones(n - 1)], [-1, 0, 1], format="csr")
    eye = sp.identity(n, format="csr")
    a = ((sp.kron(eye, t) + sp.kron(t, eye)) / h2).tocsr()
    a.sort_indices()
    return a


def global_residual(prob, x, eps):
    """F_eps(x) with check=False (`system.py:118-132,147-152`)."""
    a = prob.__dict__.get("_lap")
    if a is None:
        a = prob._lap = laplacian(prob.n)
    n2 = prob.n * prob.n
    y, p = x[:n2], x[n2:]
    r1, r2 = rows_from_actions(a @ y, a @ p, y, p, prob.f, prob.y_d, prob.phi, prob.nu,
                               prob.mu, eps)
    return np.concatenate([r1, r2])


def global_jacobian(prob, x, eps):
    """[[A + diag(phi'), diag(b12)], [diag(b21), A + diag(phi')]] as CSR (`system.py:155-160`)."""
    a = prob.__dict__.get("_lap")
    if a is None:
        a = prob._lap = laplacian(prob.n)
    n2 = prob.n * prob.n
    y, p = x[:n2], x[n2:]
    d1, b12, b21 = jac_diagonals(y, p, prob.phi, prob.nu, prob.mu, eps)
    a11 = a + sp.diags(d1)
    return sp.bmat([[a11, sp.diags(b12)], [sp.diags(b21), a11]], format="csr")


def ras_preconditioner(prob, x, eps):
    """One-level RAS at x: SuperLU of every local pair Jacobian at x[pair_idx]
    (`schwarz.py:221-239`)."""
    lus = []
    for i, r in enumerate(prob.rects):
        _, J = prob.local_fns(i, x)
        try:
            lus.append(spla.splu(J(x[r.pair_idx], eps).tocsc()))
        except RuntimeError as exc:
            raise OracleLocalFailure(i, f"singular local block: {exc}") from exc

    def apply(v):
        out = np.zeros_like(v)
        for r, lu in zip(prob.rects, lus):
            w = lu.solve(v[r.pair_idx])
            out[r.pair_own] = w[r.pair_own_in_local]
        return out

    return apply


def newton_ras_solve(prob, x0, eps0, gamma, eps_min, tol=1e-10, max_outer=200, sigma=1.1,
                     gmres_rel=1e-8, gmres_max=2000, max_halvings=30):
    """Monolithic damped Newton with eps-continuation, GMRES directions
    left-preconditioned by RAS rebuilt at every iterate (`newton.py:133-181`)."""
    gm = []

    def J_solve(x, eps, rhs):
        jac = global_jacobian(prob, x, eps)
        d, k, res, conv, _ = gmres(lambda v: jac @ v, rhs, gmres_rel, gmres_max,
                                   precond=ras_preconditioner(prob, x, eps))
        if not conv:
            raise OracleLinearFailure(f"GMRES stalled at residual {res:.3e} after {k} iterations")
        gm.append(k)
        return d

    x, ok, iters, failure, (norms, epss, alphas) = newton(
        x0, lambda v, e: global_residual(prob, v, e), J_solve, eps0, gamma, eps_min, tol,
        max_outer, sigma, max_halvings)
    return x, {"converged": ok, "outer_iters": iters, "failure": failure,
               "residual_norms": norms, "eps_values": epss, "alphas": alphas,
               "gmres_iters": gm}


def recover_control(p, mu, nu, eps):
    """u = -(p + mu P_eps(-p/mu))/nu (`system.py:173-174`)."""
    return -(p + mu * p_eps(-p / mu, eps)) / nu


def dof_updates(prob, per_sub):
    """Subdomain-Newton DOF-updates: sum_evals sum_i 2 R_i C_i k_i."""
    sizes = np.array([2 * r.size for r in prob.rects], dtype=np.int64)
    return int(sum(int(np.dot(sizes, np.asarray(k, dtype=np.int64))) for k in per_sub))


def sample_subdomains(prob, count, seed=0):
    """Deterministic subset of subdomain ids for bounded CPU-baseline timing."""
    rng = np.random.default_rng(seed)
    ids = rng.choice(len(prob.rects), size=min(count, len(prob.rects)), replace=False)
    return sorted(int(i) for i in ids)


__all__ = ["Problem", "raspen_residual", "raspen_jvp", "raspen_solve", "gmres", "newton",
           "global_residual", "global_jacobian", "ras_preconditioner", "newton_ras_solve",
           "laplacian", "OracleLinearFailure",
           "recover_control", "decompose", "tile_edges", "OracleLocalFailure",
           "dof_updates", "sample_subdomains", "p_eps", "dp_eps", "math"]
