"""ctypes binding of the in-tree C-ABI library ``_lib/liblightgp.so`` (include/lightgp.h).

There is no CPU fallback: importing works without a GPU (so the API surface
and the library's exports can be checked on any machine), but every compute
call needs a CUDA context, and creating one fails loudly with a
``MiniGpError`` when the library or the GPU is missing.
"""

from __future__ import annotations

import ctypes as C
import os
import threading

import numpy as np

from .errors import (
    DimensionMismatchError,
    MiniGpError,
    NonFiniteError,
    OperatorNotSpdError,
)

LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "_lib", "liblightgp.so")

# status codes (include/lightgp.h)
OK, E_ARG, E_DIM, E_NONFINITE, E_NOT_SPD = 0, 1, 2, 3, 4
E_CUDA, E_NCCL, E_OOM, E_COMPILE, E_UNSUPPORTED = 5, 6, 7, 8, 9

# node kinds
NODE_KINDS = {"rbf": 0, "matern12": 1, "matern32": 2, "matern52": 3, "periodic": 4,
              "linear": 5, "scale": 6, "+": 7, "*": 8}

DEVICE_PTRS = 1
ACC_FP32 = 2
DIST_DIRECT = 4
FORCE_SIMT = 8
NO_SYM = 16
INPUTS_FINITE = 32

_P = C.c_void_p
_D = C.POINTER(C.c_double)
_I32 = C.POINTER(C.c_int32)

_SIGS = {
    "lgp_abi_version": ([], C.c_int),
    "lgp_last_error": ([], C.c_char_p),
    "lgp_device_count": ([C.POINTER(C.c_int)], C.c_int),
    "lgp_partition": ([C.c_int64, C.c_int, C.c_int, C.POINTER(C.c_int64), C.POINTER(C.c_int64)],
                      C.c_int),
    "lgp_comm_unique_id": ([C.c_char_p], C.c_int),
    "lgp_comm_allreduce_max": ([_P, C.POINTER(C.c_double), C.c_int32], C.c_int),
    "lgp_cg_shifted": ([_P, _P, _P, C.c_double, _P, C.c_int32, _D, C.c_double, C.c_int32, _P,
                        _I32, _D, C.c_uint32], C.c_int),
    "lgp_ctx_create": ([C.c_int, C.c_int, C.c_int, C.c_char_p, C.POINTER(_P)], C.c_int),
    "lgp_ctx_destroy": ([_P], C.c_int),
    "lgp_ctx_sync": ([_P], C.c_int),
    "lgp_ctx_launch_count": ([_P, C.POINTER(C.c_uint64)], C.c_int),
    "lgp_ctx_set_profile": ([_P, C.c_int], C.c_int),
    "lgp_ctx_profile": ([_P, C.POINTER(C.c_double), C.POINTER(C.c_uint64), C.c_int], C.c_int),
    "lgp_timer_start": ([_P], C.c_int),
    "lgp_timer_stop": ([_P, C.POINTER(C.c_float)], C.c_int),
    "lgp_device_alloc": ([_P, C.c_size_t, C.POINTER(_P)], C.c_int),
    "lgp_device_free": ([_P, _P], C.c_int),
    "lgp_memcpy_h2d": ([_P, _P, _P, C.c_size_t], C.c_int),
    "lgp_memcpy_d2h": ([_P, _P, _P, C.c_size_t], C.c_int),
    "lgp_host_alloc": ([C.c_size_t, C.POINTER(_P)], C.c_int),
    "lgp_host_free": ([_P], C.c_int),
    "lgp_all_finite": ([_P, C.c_size_t, C.POINTER(C.c_int)], C.c_int),
    "lgp_flush_l2": ([_P, C.c_size_t], C.c_int),
    "lgp_kernel_compile": ([_P, C.c_int, _I32, _D, C.c_int, C.POINTER(_P)], C.c_int),
    "lgp_kernel_free": ([_P], C.c_int),
    "lgp_kernel_source": ([_P, C.c_int32, C.c_int32, C.c_uint32, C.c_char_p, C.c_size_t,
                           C.POINTER(C.c_size_t)], C.c_int),
    "lgp_kernel_jit": ([_P, C.c_int32, C.c_int32, C.c_uint32, C.c_char_p, C.c_size_t], C.c_int),
    "lgp_points_upload": ([_P, _D, C.c_int64, C.c_int32, C.POINTER(_P)], C.c_int),
    "lgp_points_free": ([_P], C.c_int),
    "lgp_matvec": ([_P, _P, _P, _P, C.c_double, _P, C.c_int32, _P, C.c_uint32], C.c_int),
    "lgp_cg": ([_P, _P, _P, C.c_double, _P, C.c_int32, C.c_double, C.c_int32, _P, _I32, _D,
                C.c_uint32], C.c_int),
    "lgp_lanczos": ([_P, _P, _P, C.c_double, _P, C.c_int32, C.c_int32, _D, _D, _I32, C.c_uint32],
                    C.c_int),
    "lgp_gram": ([_P, _P, _P, _P, _P, C.c_uint32], C.c_int),
    "lgp_diag": ([_P, _P, _P, _P, C.c_uint32], C.c_int),
    "lgp_predict_quad": ([_P, _P, _P, _P, C.c_double, C.c_double, C.c_int32, _D, _I32, _D],
                         C.c_int),
}

_lib = None
_lib_lock = threading.Lock()


def lib():
    """The loaded library (raises MiniGpError if it was not built)."""
    global _lib
    if _lib is not None:
        return _lib
    with _lib_lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise MiniGpError(
                    f"lightgp CUDA library not built: {LIB_PATH} is missing "
                    "(run `make -C paper_2605_17898_b200/csrc` or __graft_entry__.build())")
            h = C.CDLL(LIB_PATH)
            for name, (args, res) in _SIGS.items():
                fn = getattr(h, name)
                fn.argtypes = args
                fn.restype = res
            _lib = h
    return _lib


def exported_symbols():
    return list(_SIGS)


def check(status):
    """Map a library status code onto the reference error taxonomy (errors.py)."""
    if status == OK:
        return
    msg = (lib().lgp_last_error() or b"").decode(errors="replace")
    if status == E_DIM:
        raise DimensionMismatchError(msg)
    if status == E_NONFINITE:
        raise NonFiniteError(msg)
    if status == E_NOT_SPD:
        raise OperatorNotSpdError(msg)
    if status == E_ARG:
        raise ValueError(msg)
    raise MiniGpError(f"lightgp error {status}: {msg}")


def device_count():
    """Visible CUDA devices (0 without a GPU or driver)."""
    n = C.c_int()
    check(lib().lgp_device_count(C.byref(n)))
    return n.value


def dptr(a):
    return a.ctypes.data_as(_D)


def vptr(a):
    return C.c_void_p(a.ctypes.data)


def iptr(a):
    return a.ctypes.data_as(_I32)


# ------------------------------------------------------------------ context

class Context:
    """One GPU (one rank). Owns the library context handle."""

    def __init__(self, device=0, rank=0, world=1, nccl_id=None):
        h = C.c_void_p()
        check(lib().lgp_ctx_create(int(device), int(rank), int(world), nccl_id, C.byref(h)))
        self.handle = h
        self.device, self.rank, self.world = int(device), int(rank), int(world)

    def close(self):
        if self.handle:
            lib().lgp_ctx_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def sync(self):
        check(lib().lgp_ctx_sync(self.handle))

    def launches(self):
        n = C.c_uint64()
        check(lib().lgp_ctx_launch_count(self.handle, C.byref(n)))
        return n.value

    def set_profile(self, on=True):
        check(lib().lgp_ctx_set_profile(self.handle, 1 if on else 0))

    def k1_profile(self, reset=True):
        """(total device ms, launches) of the fused K1 kernel since the last reset."""
        ms, n = C.c_double(), C.c_uint64()
        check(lib().lgp_ctx_profile(self.handle, C.byref(ms), C.byref(n), 1 if reset else 0))
        return ms.value, n.value

    def timer_start(self):
        check(lib().lgp_timer_start(self.handle))

    def timer_stop(self):
        ms = C.c_float()
        check(lib().lgp_timer_stop(self.handle, C.byref(ms)))
        return ms.value

    def allreduce_max(self, values):
        """Element-wise max over the context's ranks (library NCCL all-reduce);
        returns a list of floats. Identity without a communicator."""
        vals = (C.c_double * len(values))(*[float(v) for v in values])
        check(lib().lgp_comm_allreduce_max(self.handle, vals, len(values)))
        return list(vals)

    def barrier(self):
        """All ranks of the context reach this point (one tiny all-reduce)."""
        self.allreduce_max([0.0])

    def flush_l2(self, nbytes=256 << 20):
        check(lib().lgp_flush_l2(self.handle, nbytes))


_default = None
_default_lock = threading.Lock()


def default_context():
    """Process-wide context: set by distributed.init(), else a 1-rank context on
    LOCAL_RANK (or device 0)."""
    global _default
    if _default is None:
        with _default_lock:
            if _default is None:
                _default = Context(device=int(os.environ.get("LOCAL_RANK", "0")))
    return _default


def set_default_context(ctx):
    global _default
    _default = ctx


# ------------------------------------------------------- page-locked results

def all_finite(a):
    """True iff the float64 C-contiguous array has no NaN / Inf (threaded C scan)."""
    ok = C.c_int(0)
    check(lib().lgp_all_finite(C.c_void_p(a.ctypes.data), a.size, C.byref(ok)))
    return bool(ok.value)


class _PinnedBlock:
    """A page-locked host block exposed to NumPy; returned to the pool when the
    last array viewing it is garbage-collected."""

    def __init__(self, ptr, nbytes, shape):
        self.ptr, self.nbytes = ptr, nbytes
        self.__array_interface__ = {"data": (ptr, False), "shape": tuple(shape),
                                    "typestr": "<f8", "version": 3}

    def __del__(self):
        try:
            _pinned.release(self.ptr, self.nbytes)
        except Exception:
            pass


class _PinnedPool:
    """Recycled page-locked result buffers: device -> host copies of large
    results run at full PCIe speed (~2.7x a pageable copy on B200 hosts)
    without paying cudaHostAlloc per call. Bounded: at most `keep` blocks per
    size and `cap` bytes cached."""

    MIN_BYTES = 1 << 20

    def __init__(self, keep=4, cap=2 << 30):
        self.keep, self.cap = keep, cap
        self.free = {}
        self.cached = 0
        self.lock = threading.Lock()

    def empty(self, shape):
        nbytes = int(np.prod(shape)) * 8
        if nbytes < self.MIN_BYTES:
            return np.empty(shape)
        ptr = None
        with self.lock:
            lst = self.free.get(nbytes)
            if lst:
                ptr = lst.pop()
                self.cached -= nbytes
        if ptr is None:
            p = C.c_void_p()
            if lib().lgp_host_alloc(nbytes, C.byref(p)) != OK or not p.value:
                return np.empty(shape)
            ptr = p.value
        return np.asarray(_PinnedBlock(ptr, nbytes, shape))

    def release(self, ptr, nbytes):
        with self.lock:
            lst = self.free.setdefault(nbytes, [])
            if len(lst) < self.keep and self.cached + nbytes <= self.cap:
                lst.append(ptr)
                self.cached += nbytes
                return
        lib().lgp_host_free(C.c_void_p(ptr))


_pinned = _PinnedPool()


def result_buffer(shape):
    """float64 array for a device result: page-locked (pooled) when large."""
    return _pinned.empty(shape)


# ------------------------------------------------------------------ handles

class KernelProgram:
    """A lowered kernel tree handed to the library (pre-order kinds + params)."""

    def __init__(self, kinds, params):
        k = np.ascontiguousarray(kinds, dtype=np.int32)
        p = np.ascontiguousarray(params, dtype=np.float64)
        h = C.c_void_p()
        check(lib().lgp_kernel_compile(None, len(k), iptr(k), dptr(p), len(p), C.byref(h)))
        self.handle = h
        self.kinds, self.params = k, p

    def __del__(self):
        try:
            if self.handle:
                lib().lgp_kernel_free(self.handle)
                self.handle = None
        except Exception:
            pass

    def source(self, d, t=1, flags=0):
        need = C.c_size_t()
        check(lib().lgp_kernel_source(self.handle, d, t, flags, None, 0, C.byref(need)))
        buf = C.create_string_buffer(need.value)
        check(lib().lgp_kernel_source(self.handle, d, t, flags, buf, need.value, None))
        return buf.value.decode()

    def jit(self, d, t=1, flags=0):
        buf = C.create_string_buffer(1 << 16)
        check(lib().lgp_kernel_jit(self.handle, d, t, flags, buf, len(buf)))
        return buf.value.decode()


class DevicePoints:
    """A point set resident on one context's GPU (FP64, plus its column mean)."""

    def __init__(self, ctx, x):
        x = np.ascontiguousarray(x, dtype=np.float64)
        h = C.c_void_p()
        check(lib().lgp_points_upload(ctx.handle, dptr(x), x.shape[0], x.shape[1], C.byref(h)))
        self.handle = h
        self.ctx = ctx
        self.n, self.d = x.shape

    def __del__(self):
        try:
            if self.handle:
                lib().lgp_points_free(self.handle)
                self.handle = None
        except Exception:
            pass
