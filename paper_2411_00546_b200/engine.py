"""Device engine: one native context per (problem, decomposition).

``Engine`` owns the ``ocp_ctx`` (problem data, subdomain table, local pools,
LU windows) and hands out ``DeviceVector`` objects whose arithmetic runs in
the library's kernels (deterministic reductions, reference rounding order).
"""

import ctypes
import weakref

import numpy as np

from . import _native as nat
from .system import phi_code


def _destroy(lib, ctx, pool):
    lib.ocp_sync(ctx)
    pool.release_all()
    lib.ocp_ctx_destroy(ctx)


class Engine:
    """Native context for one problem + s1 x s2 decomposition with overlap m."""

    def __init__(self, spec, s1, s2, m):
        lib = nat.load()
        self.lib = lib
        self.spec = spec
        self.grid = spec.grid
        self.n = spec.grid.n
        self.N = self.n * self.n
        kind, kappa = phi_code(spec.phi)
        f = np.ascontiguousarray(spec.f, dtype=np.float64)
        y_d = np.ascontiguousarray(spec.y_d, dtype=np.float64)
        ctx = ctypes.c_void_p()
        rc = lib.ocp_ctx_create(self.n, s1, s2, m, float(spec.nu), float(spec.mu), kind,
                                float(kappa), nat.ptr(f), nat.ptr(y_d), ctypes.byref(ctx))
        if rc != nat.OCP_OK:
            msg = nat.last_error(None)
            if rc == nat.OCP_ERR_ARG:
                raise ValueError(msg)
            if rc == nat.OCP_ERR_NO_DEVICE:
                raise nat.NativeUnavailable(msg)
            raise nat.NativeError(rc, msg, "ocp_ctx_create")
        self.ctx = ctx
        self.pool = nat.BufferPool()
        self._finalizer = weakref.finalize(self, _destroy, lib, ctx, self.pool)
        info = (ctypes.c_longlong * 8)()
        nat.check(lib.ocp_ctx_info(ctx, info), ctx, "ocp_ctx_info")
        self.num_subdomains = int(info[0])
        self.pool_len = int(info[1])
        self.fac_len = int(info[2])
        self.max_w = int(info[3])
        self.nb = int(info[4])
        self.dof_total = int(info[5])
        self.ref_len = int(info[6])
        tab = np.zeros(11 * self.num_subdomains, dtype=np.int32)
        nat.check(lib.ocp_subdomain_table(ctx, tab.ctypes.data_as(ctypes.POINTER(ctypes.c_int))),
                  ctx, "ocp_subdomain_table")
        self.rects = tab.reshape(-1, 11)

    # -- plumbing --------------------------------------------------------
    def check(self, rc, where):
        nat.check(rc, self.ctx, where)

    def error(self):
        return nat.last_error(self.ctx)

    def sync(self):
        self.check(self.lib.ocp_sync(self.ctx), "ocp_sync")

    def vector(self, n=None):
        return DeviceVector(self, 2 * self.N if n is None else n)

    def from_host(self, arr):
        arr = np.ascontiguousarray(arr, dtype=np.float64)
        v = DeviceVector(self, arr.shape[0])
        self.check(self.lib.ocp_h2d(self.ctx, v.ptr, nat.ptr(arr), arr.nbytes), "ocp_h2d")
        return v

    def factor_store(self):
        return nat.DeviceBuffer(8 * self.fac_len, self.pool)

    def buffer(self, nbytes):
        return nat.DeviceBuffer(nbytes, self.pool)

    # -- instrumentation ---------------------------------------------------
    def set_profiling(self, on):
        self.check(self.lib.ocp_set_profiling(self.ctx, 1 if on else 0), "ocp_set_profiling")

    def stats(self):
        buf = (ctypes.c_double * 15)()
        self.check(self.lib.ocp_stats(self.ctx, buf, 15), "ocp_stats")
        keys = ("launches", "factor_ms", "factor_launches", "solve_ms", "solve_launches",
                "factor_flops", "solve_bytes", "sweep_ms", "dof_updates", "jvp_ms",
                "inner_solve_ms", "mgs_ms", "resid_ms", "resid_launches", "resid_bytes")
        return dict(zip(keys, list(buf)))

    def mark(self, slot):
        self.check(self.lib.ocp_event_record(self.ctx, slot), "ocp_event_record")

    def elapsed_ms(self, a, b):
        out = ctypes.c_double()
        self.check(self.lib.ocp_event_elapsed(self.ctx, a, b, ctypes.byref(out)),
                   "ocp_event_elapsed")
        return out.value

    def reset_stats(self):
        self.check(self.lib.ocp_reset_stats(self.ctx), "ocp_reset_stats")


class DeviceVector:
    """float64 vector in device memory; arithmetic runs in libocpgpu kernels."""

    __slots__ = ("engine", "n", "buf")

    def __init__(self, engine, n, buf=None):
        self.engine = engine
        self.n = int(n)
        self.buf = buf if buf is not None else nat.DeviceBuffer(8 * self.n, engine.pool)

    @property
    def ptr(self):
        return ctypes.c_void_p(self.buf.addr)

    def device_ptr(self):
        return self.buf.addr

    @property
    def shape(self):
        return (self.n,)

    def to_host(self):
        out = np.empty(self.n, dtype=np.float64)
        e = self.engine
        e.check(e.lib.ocp_d2h(e.ctx, nat.ptr(out), self.ptr, out.nbytes), "ocp_d2h")
        return out

    def copy(self):
        e = self.engine
        out = DeviceVector(e, self.n)
        e.check(e.lib.ocp_d2d(e.ctx, out.ptr, self.ptr, 8 * self.n), "ocp_d2d")
        return out

    def assign(self, other):
        e = self.engine
        e.check(e.lib.ocp_d2d(e.ctx, self.ptr, other.ptr, 8 * self.n), "ocp_d2d")
        return self

    def zero(self):
        e = self.engine
        e.check(e.lib.ocp_memset0(e.ctx, self.ptr, 8 * self.n), "ocp_memset0")
        return self

    def norm(self):
        e = self.engine
        out = ctypes.c_double()
        e.check(e.lib.ocp_vec_nrm2(e.ctx, self.n, self.ptr, ctypes.byref(out)), "ocp_vec_nrm2")
        return out.value

    def dot(self, other):
        e = self.engine
        out = ctypes.c_double()
        e.check(e.lib.ocp_vec_dot(e.ctx, self.n, self.ptr, other.ptr, ctypes.byref(out)),
                "ocp_vec_dot")
        return out.value

    def add_scaled(self, alpha, d, out=None):
        """out = self + alpha * d (numpy rounding: product first)."""
        e = self.engine
        out = DeviceVector(e, self.n) if out is None else out
        e.check(e.lib.ocp_vec_add_scaled(e.ctx, self.n, self.ptr, float(alpha), d.ptr, out.ptr),
                "ocp_vec_add_scaled")
        return out

    def scaled(self, a, out=None):
        e = self.engine
        out = DeviceVector(e, self.n) if out is None else out
        e.check(e.lib.ocp_vec_scale(e.ctx, self.n, float(a), self.ptr, out.ptr), "ocp_vec_scale")
        return out

    def divided(self, s, out=None):
        e = self.engine
        out = DeviceVector(e, self.n) if out is None else out
        e.check(e.lib.ocp_vec_div(e.ctx, self.n, self.ptr, float(s), out.ptr), "ocp_vec_div")
        return out

    def __neg__(self):
        return self.scaled(-1.0)

    def equals(self, other):
        e = self.engine
        out = ctypes.c_int()
        e.check(e.lib.ocp_vec_equal(e.ctx, self.n, self.ptr, other.ptr, ctypes.byref(out)),
                "ocp_vec_equal")
        return bool(out.value)

    def all_finite(self):
        e = self.engine
        out = ctypes.c_int()
        e.check(e.lib.ocp_vec_all_finite(e.ctx, self.n, self.ptr, ctypes.byref(out)),
                "ocp_vec_all_finite")
        return bool(out.value)

    def recover_control(self, spec, eps):
        e = self.engine
        out = DeviceVector(e, self.n)
        e.check(e.lib.ocp_recover_control(e.ctx, self.n, self.ptr, float(eps), out.ptr),
                "ocp_recover_control")
        return out

    def slice_view(self, start, length):
        """Non-owning view (shares the allocation)."""
        view = DeviceVector.__new__(DeviceVector)
        view.engine = self.engine
        view.n = int(length)
        view.buf = _View(self.buf, 8 * int(start))
        return view


class _View:
    __slots__ = ("base", "offset")

    def __init__(self, base, offset):
        self.base = base
        self.offset = offset

    @property
    def addr(self):
        return self.base.addr + self.offset


class DeviceBasis:
    """Krylov basis: columns of length n in one allocation, doubled when full.

    Mirrors the growing (n, cap+1) array of the reference (`krylov.py:89-107`).
    """

    def __init__(self, engine, n, cap):
        self.engine = engine
        self.n = n
        self.cap = cap
        self.buf = nat.DeviceBuffer(8 * n * (cap + 1), engine.pool)

    def column(self, j):
        v = DeviceVector.__new__(DeviceVector)
        v.engine = self.engine
        v.n = self.n
        v.buf = _View(self.buf, 8 * self.n * j)
        return v

    def grow(self, cap, used):
        e = self.engine
        new = nat.DeviceBuffer(8 * self.n * (cap + 1), e.pool)
        e.check(e.lib.ocp_d2d(e.ctx, ctypes.c_void_p(new.addr), ctypes.c_void_p(self.buf.addr),
                              8 * self.n * used), "ocp_d2d")
        e.sync()
        self.buf = new
        self.cap = cap

    @property
    def ptr(self):
        return ctypes.c_void_p(self.buf.addr)
