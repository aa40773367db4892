"""ctypes binding of ``libocpgpu.so`` (the C ABI in ``include/ocp_gpu.h``).

There is no CPU fallback: importing the hot path without the built library,
or calling it without a CUDA device, raises ``NativeUnavailable``.
"""

import ctypes
import os
import threading

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("OCP_LIB") or os.path.join(HERE, "libocpgpu.so")   # OCP_LIB: experiment builds

OCP_OK = 0
OCP_ERR_ARG = 1
OCP_ERR_CUDA = 2
OCP_ERR_LOCAL_SOLVE = 3
OCP_ERR_NONFINITE = 4
OCP_ERR_NONFINITE_INIT = 5
OCP_ERR_UNSUPPORTED = 6
OCP_ERR_NO_DEVICE = 7
OCP_ERR_GMRES_BREAKDOWN = 8

_c_int_p = ctypes.POINTER(ctypes.c_int)
_c_dbl_p = ctypes.POINTER(ctypes.c_double)
_c_ll_p = ctypes.POINTER(ctypes.c_longlong)
_vp = ctypes.c_void_p
_ll = ctypes.c_longlong
_d = ctypes.c_double
_i = ctypes.c_int

# name -> argtypes (all return int status unless listed in _RESTYPES)
SIGNATURES = {
    "ocp_ctx_create": [_i, _i, _i, _i, _d, _d, _i, _d, _vp, _vp, ctypes.POINTER(_vp)],
    "ocp_ctx_destroy": [_vp],
    "ocp_last_error": [_vp],
    "ocp_ctx_info": [_vp, _c_ll_p],
    "ocp_subdomain_table": [_vp, _c_int_p],
    "ocp_malloc": [ctypes.c_size_t, ctypes.POINTER(_vp)],
    "ocp_free": [_vp],
    "ocp_h2d": [_vp, _vp, _vp, ctypes.c_size_t],
    "ocp_d2h": [_vp, _vp, _vp, ctypes.c_size_t],
    "ocp_d2d": [_vp, _vp, _vp, ctypes.c_size_t],
    "ocp_memset0": [_vp, _vp, ctypes.c_size_t],
    "ocp_sync": [_vp],
    "ocp_raspen_residual": [_vp, _vp, _vp, _d, _d, _d, _d, _i, _d, _i, _vp, _c_int_p, _c_int_p],
    "ocp_raspen_residual_at": [_vp, _vp, _vp, _d, _d, _d, _d, _d, _i, _d, _i, _vp, _c_int_p,
                               _c_int_p],
    "ocp_local_correction": [_vp, _vp, _vp, _i, _d, _d, _d, _d, _i, _d, _i, _c_int_p, _c_int_p],
    "ocp_raspen_jvp": [_vp, _vp, _vp, _vp],
    "ocp_local_values": [_vp, _vp],
    "ocp_local_residual": [_vp, _vp, _vp, _d, _vp],
    "ocp_local_residual_trial": [_vp, _vp, _vp, _vp, _vp, _d, _vp],
    "ocp_local_direction": [_vp, _vp, _vp, _d, _vp],
    "ocp_vec_nrm2": [_vp, _ll, _vp, _c_dbl_p],
    "ocp_vec_dot": [_vp, _ll, _vp, _vp, _c_dbl_p],
    "ocp_vec_add_scaled": [_vp, _ll, _vp, _d, _vp, _vp],
    "ocp_vec_scale": [_vp, _ll, _d, _vp, _vp],
    "ocp_vec_div": [_vp, _ll, _vp, _d, _vp],
    "ocp_vec_equal": [_vp, _ll, _vp, _vp, _c_int_p],
    "ocp_vec_all_finite": [_vp, _ll, _vp, _c_int_p],
    "ocp_mgs": [_vp, _ll, _vp, _ll, _i, _vp, _c_dbl_p],
    "ocp_arnoldi": [_vp, _ll, _vp, _ll, _i, _vp, _c_dbl_p],
    "ocp_raspen_gmres": [_vp, _vp, _vp, _d, _d, _i, _vp, _c_int_p, _c_dbl_p, _c_int_p, _c_dbl_p],
    "ocp_global_residual": [_vp, _vp, _d, _vp],
    "ocp_global_jacobian": [_vp, _vp, _d, _vp],
    "ocp_global_jvp": [_vp, _vp, _vp, _vp],
    "ocp_ras_factor": [_vp, _vp, _d, _vp, _c_int_p],
    "ocp_ras_apply": [_vp, _vp, _vp, _vp],
    "ocp_ras_gmres": [_vp, _vp, _vp, _vp, _d, _d, _i, _vp, _c_int_p, _c_dbl_p, _c_int_p, _c_dbl_p],
    "ocp_state_residual": [_vp, _vp, _vp, _vp],
    "ocp_state_cg": [_vp, _vp, _vp, _d, _i, _vp, _c_int_p, _c_dbl_p, _c_int_p],
    "ocp_manufacture_yd": [_vp, _vp, _vp, _vp],
    "ocp_gemv_add": [_vp, _ll, _vp, _ll, _i, _c_dbl_p, _vp, _vp],
    "ocp_recover_control": [_vp, _ll, _vp, _d, _vp],
    "ocp_set_profiling": [_vp, _i],
    "ocp_stats": [_vp, _c_dbl_p, _i],
    "ocp_reset_stats": [_vp],
    "ocp_event_record": [_vp, _i],
    "ocp_check_guards": [_c_ll_p, _c_ll_p],
    "ocp_event_elapsed": [_vp, _i, _i, _c_dbl_p],
}
_RESTYPES = {"ocp_ctx_destroy": None, "ocp_last_error": ctypes.c_char_p}


class NativeUnavailable(RuntimeError):
    """The CUDA library is missing or no device is visible (no fallback exists)."""


class NativeError(RuntimeError):
    def __init__(self, code, message, where=""):
        self.code = code
        self.message = message
        super().__init__(f"{where}: [{code}] {message}" if where else f"[{code}] {message}")


_lib = None
_lock = threading.Lock()


def load(path=LIB_PATH):
    """Load and type the library (does not touch the GPU)."""
    global _lib
    if _lib is not None:   # (no lock on the hot path: load() is also reached from finalizers)
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(path):
            raise NativeUnavailable(
                f"{path} not built; run __graft_entry__.build() (nvcc, sm_100a)")
        lib = ctypes.CDLL(path)
        for name, args in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.argtypes = args
            fn.restype = _RESTYPES.get(name, ctypes.c_int)
        _lib = lib
        return lib


def last_error(ctx=None):
    msg = load().ocp_last_error(ctx)
    return msg.decode() if msg else ""


def check(rc, ctx=None, where=""):
    if rc != OCP_OK:
        raise NativeError(rc, last_error(ctx), where)


def ptr(a):
    """Host pointer of a C-contiguous float64/int array."""
    return ctypes.c_void_p(a.ctypes.data)


class BufferPool:
    """Per-engine caching allocator (one CUDA stream per engine => reuse is stream-ordered).

    cudaFree synchronises the device; GMRES allocates a fresh vector per
    matvec, so freed buffers are cached by size and handed out again.
    """

    def __init__(self, limit_bytes=48 << 30):
        self.free = {}
        self.cached = 0
        self.limit = limit_bytes
        self.closed = False

    def take(self, nbytes):
        lst = self.free.get(nbytes)
        if lst:
            self.cached -= nbytes
            return lst.pop()
        return _RETIRED.take(nbytes)

    def give(self, addr, nbytes):
        if self.closed or self.cached + nbytes > self.limit:
            _raw_free(addr)
            return
        self.free.setdefault(nbytes, []).append(addr)
        self.cached += nbytes

    def release_all(self):
        """Engine teardown, after its stream is synchronised: the cached
        buffers go to the process-wide retired cache (the next engine of the
        same shapes allocates nothing)."""
        self.closed = True
        for nbytes, lst in self.free.items():
            for addr in lst:
                _RETIRED.give(addr, nbytes)
        self.free.clear()
        self.cached = 0


class _RetiredCache:
    """Buffers of destroyed engines (their streams are idle), reused by size
    across engines like a caching allocator; bounded, thread-safe.

    ``give`` runs from garbage-collection finalizers (``Engine`` teardown,
    ``DeviceBuffer.__del__``), and a collection can start at any allocation -
    also inside ``take`` / ``give`` while this thread holds the lock.  So
    ``give`` never blocks on the lock: when it is taken the buffer is parked
    in ``_pending`` (list.append is atomic) and filed by the next caller that
    holds the lock.  (A blocking acquire here deadlocked the thread against
    itself: a flaky hang of the GPU test suite.)
    """

    def __init__(self, limit_bytes=16 << 30):
        self.free = {}
        self.cached = 0
        self.limit = limit_bytes
        self.lock = threading.Lock()
        self._pending = []

    def _file_locked(self):
        """File the parked buffers (lock held); returns those over the limit."""
        over = []
        while self._pending:
            addr, nbytes = self._pending.pop()
            if self.cached + nbytes <= self.limit:
                self.free.setdefault(nbytes, []).append(addr)
                self.cached += nbytes
            else:
                over.append(addr)
        return over

    def take(self, nbytes):
        addr = None
        with self.lock:
            over = self._file_locked()
            lst = self.free.get(nbytes)
            if lst:
                addr = lst.pop()
                self.cached -= nbytes
        for a in over:
            _raw_free(a)
        return addr

    def give(self, addr, nbytes):
        self._pending.append((addr, nbytes))
        if not self.lock.acquire(blocking=False):
            return   # the holder (possibly this thread, below us on the stack) files it later
        try:
            over = self._file_locked()
        finally:
            self.lock.release()
        for a in over:
            _raw_free(a)

    def empty(self):
        with self.lock:
            self._file_locked()
            lists, self.free, self.cached = list(self.free.values()), {}, 0
        for lst in lists:
            for addr in lst:
                _raw_free(addr)


_RETIRED = _RetiredCache()


def empty_cache():
    """Free the device buffers cached from destroyed engines."""
    _RETIRED.empty()


def _raw_alloc(nbytes):
    lib = load()
    p = ctypes.c_void_p()
    rc = lib.ocp_malloc(ctypes.c_size_t(nbytes), ctypes.byref(p))
    if rc != OCP_OK:
        raise NativeError(rc, last_error(), "ocp_malloc")
    return p.value


def _raw_free(addr):
    if _lib is not None and addr:
        _lib.ocp_free(ctypes.c_void_p(addr))


class DeviceBuffer:
    """Device allocation owned by Python; returns to its pool (or is freed) on collection."""

    __slots__ = ("addr", "nbytes", "pool", "__weakref__")

    def __init__(self, nbytes, pool=None):
        nbytes = max(int(nbytes), 16)
        nbytes = (nbytes + 255) // 256 * 256
        self.pool = pool
        addr = pool.take(nbytes) if pool is not None else None
        if addr is None:
            addr = _raw_alloc(nbytes)
        self.addr = addr
        self.nbytes = nbytes

    def __del__(self):
        addr = getattr(self, "addr", None)
        if not addr:
            return
        self.addr = None
        if self.pool is not None:
            self.pool.give(addr, self.nbytes)
        else:
            _raw_free(addr)
