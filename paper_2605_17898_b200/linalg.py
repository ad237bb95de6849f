"""Host-side input conventions and the allocation ledger (minigp/linalg.py:39-106).

Every public entry point validates its NumPy inputs exactly like the
reference (finite, float64, C-contiguous, right rank) before anything is
copied to the GPU, and registers the host arrays it returns with the
process-global ``LEDGER`` so the reference's memory-accounting properties
(``test_matvec_ledger_bound_n50000``) remain observable. Device memory is
accounted by the library, not here.
"""

from __future__ import annotations

import threading
import weakref

import numpy as np

from .errors import DimensionMismatchError, NonFiniteError


class AllocationLedger:
    """Live / peak bytes of library-returned host buffers (linalg.py:39-67)."""

    def __init__(self):
        self._lock = threading.Lock()
        self.current_bytes = 0
        self.peak_bytes = 0

    def register(self, nbytes):
        with self._lock:
            self.current_bytes += nbytes
            self.peak_bytes = max(self.peak_bytes, self.current_bytes)

    def release(self, nbytes):
        with self._lock:
            self.current_bytes -= nbytes

    def reset_peak(self):
        with self._lock:
            self.peak_bytes = self.current_bytes


LEDGER = AllocationLedger()


def tracked(arr):
    """Count ``arr`` in the ledger until it is garbage collected."""
    LEDGER.register(arr.nbytes)
    weakref.finalize(arr, LEDGER.release, arr.nbytes)
    return arr


def _finite(a, name):
    if a.size >= (1 << 18) and a.dtype == np.float64 and a.flags.c_contiguous:
        from . import _lib  # threaded scan in the C library (no GPU needed)
        ok = _lib.all_finite(a)
    else:
        ok = bool(np.isfinite(a).all())
    if not ok:
        raise NonFiniteError(f"{name} contains NaN or infinite entries")


def as_matrix(x, name="matrix", check=True):
    """Finite 2-d float64, C-contiguous (linalg.py:91-97). ``check=False``
    defers the finiteness scan to the caller (see solvers.matrix_free_matvec)."""
    a = np.asarray(x, dtype=np.float64)
    if a.ndim != 2:
        raise DimensionMismatchError(f"{name} must be 2-d, got ndim={a.ndim}")
    if check:
        _finite(a, name)
    return np.ascontiguousarray(a)


def as_vector(x, name="vector"):
    """Finite 1-d float64, C-contiguous (linalg.py:100-106)."""
    a = np.asarray(x, dtype=np.float64)
    if a.ndim != 1:
        raise DimensionMismatchError(f"{name} must be 1-d, got ndim={a.ndim}")
    _finite(a, name)
    return np.ascontiguousarray(a)


def as_block(x, name="block", check=True):
    """Finite 1-d or 2-d float64 (the multi-RHS extension: n x t)."""
    a = np.asarray(x, dtype=np.float64)
    if a.ndim not in (1, 2):
        raise DimensionMismatchError(f"{name} must be 1-d or 2-d, got ndim={a.ndim}")
    if check:
        _finite(a, name)
    return np.ascontiguousarray(a)
