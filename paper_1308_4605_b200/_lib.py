"""ctypes binding of ``libstokesb200.so`` (C ABI: ``include/stokesb200.h``).

This is the binding a maintainer of the reference would add.
There is no CPU fallback: if the library is missing or no CUDA device is
visible, every device entry point raises ``RuntimeError``.
"""

from __future__ import annotations

import ctypes as C
import os
import pathlib

import numpy as np

_HERE = pathlib.Path(__file__).resolve().parent
LIB_PATH = _HERE / "libstokesb200.so"

SB_OK, SB_EINVAL, SB_EDOM, SB_ENOMEM, SB_ECUDA = 0, 22, 33, 12, 99
KIND_CELL, KIND_FACE = 0, 1
STATUS = {0: "converged", 1: "breakdown", 2: "maxiter"}

#: every symbol declared in include/stokesb200.h (checked by the CPU tests)
EXPORTS = (
    "sb_create", "sb_destroy", "sb_last_error", "sb_set_coefficients", "sb_set_cell_coefficients", "sb_apply_M",
    "sb_apply_A", "sb_apply_A_affine", "sb_homogenize", "sb_apply_Lrho", "sb_mg_solve", "sb_precond_apply", "sb_gmres_solve",
    "sb_num_levels", "sb_level_flags", "sb_level_cells", "sb_get_level_coefficients", "sb_smooth",
    "sb_residual_restrict", "sb_prolong_add", "sb_set_profiling", "sb_get_kernel_stats",
    "sb_div", "sb_grad", "sb_lap_pressure", "sb_restrict", "sb_prolong", "sb_diagonal", "sb_schur_inv",
    "sb_gmres_flat",
    "sb_launch_count", "sb_set_graphs", "sb_device_bytes", "sb_set_stream",
    "sb_nccl_id_bytes", "sb_nccl_unique_id", "sb_dist_create", "sb_dist_destroy", "sb_dist_info", "sb_dist_stream",
    "sb_dist_set_coefficients", "sb_dist_apply_M", "sb_dist_precond_apply", "sb_dist_gmres_solve",
    "sb_dist_set_profiling", "sb_dist_get_kernel_stats", "sb_dist_launch_count", "sb_dist_set_stream",
    "sb_dist_uses_nccl",
    "sb_host_alloc", "sb_host_free",
)


class Smoother(C.Structure):
    _fields_ = [("omega", C.c_double), ("sweeps_down", C.c_int), ("sweeps_up", C.c_int),
                ("bottom_sweeps", C.c_int)]


class Precond(C.Structure):
    _fields_ = [("kind", C.c_int), ("velocity_cycles", C.c_int), ("schur_sign", C.c_int),
                ("pressure_cycles", C.c_int)]


class Gmres(C.Structure):
    _fields_ = [("restart", C.c_int), ("max_iters", C.c_int), ("rtol", C.c_double),
                ("atol", C.c_double), ("track_true_residual", C.c_int)]


class HistoryRow(C.Structure):
    _fields_ = [("iteration", C.c_int), ("scalar_vcycles", C.c_longlong),
                ("resid_precond", C.c_double), ("resid_true", C.c_double), ("restart", C.c_int)]


class KernelStats(C.Structure):
    _fields_ = [("smoother_face_ms", C.c_double), ("smoother_cell_ms", C.c_double),
                ("smoother_face_bytes", C.c_double), ("smoother_cell_bytes", C.c_double),
                ("smoother_face_launches", C.c_longlong), ("smoother_cell_launches", C.c_longlong),
                ("fine_face_ms", C.c_double), ("fine_face_bytes", C.c_double),
                ("fine_face_launches", C.c_longlong)]


_P = C.c_void_p
_PP = C.POINTER(C.c_void_p)

_SIGS = {
    "sb_create": (_P, [C.c_int, C.POINTER(C.c_int), C.c_double, C.POINTER(C.c_int), C.c_int]),
    "sb_destroy": (None, [_P]),
    "sb_last_error": (C.c_char_p, []),
    "sb_set_cell_coefficients": (C.c_int, [_P, C.c_double, _P, _P, _P, C.c_double]),
    "sb_set_coefficients": (C.c_int, [_P, C.c_double, _PP, _P, _PP, _P]),
    "sb_apply_M": (C.c_int, [_P, _PP, _P, _PP, _P]),
    "sb_apply_A": (C.c_int, [_P, _PP, _PP]),
    "sb_apply_A_affine": (C.c_int, [_P, _PP, _PP, _PP]),
    "sb_homogenize": (C.c_int, [_P, _PP, _PP, _PP, _P, _PP, _P]),
    "sb_apply_Lrho": (C.c_int, [_P, _P, _P]),
    "sb_mg_solve": (C.c_int, [_P, C.c_int, C.POINTER(Smoother), C.c_int, _PP, _PP]),
    "sb_precond_apply": (C.c_int, [_P, C.POINTER(Precond), C.POINTER(Smoother), _PP, _P, _PP, _P,
                                   C.POINTER(C.c_longlong)]),
    "sb_gmres_solve": (C.c_int, [_P, C.POINTER(Precond), C.POINTER(Gmres), C.POINTER(Smoother),
                                 _PP, _P, _PP, _P, C.POINTER(HistoryRow), C.c_int,
                                 C.POINTER(C.c_int), C.POINTER(C.c_int), C.POINTER(C.c_longlong)]),
    "sb_num_levels": (C.c_int, [_P]),
    "sb_level_flags": (C.c_int, [_P, C.c_int]),
    "sb_level_cells": (C.c_int, [_P, C.c_int, C.POINTER(C.c_int)]),
    "sb_get_level_coefficients": (C.c_int, [_P, C.c_int, _PP, _P, _PP, _P]),
    "sb_smooth": (C.c_int, [_P, C.c_int, C.c_int, C.c_double, _PP, _PP]),
    "sb_residual_restrict": (C.c_int, [_P, C.c_int, C.c_int, _PP, _PP, _PP]),
    "sb_prolong_add": (C.c_int, [_P, C.c_int, C.c_int, _PP, _PP]),
    "sb_div": (C.c_int, [_P, _PP, _P]),
    "sb_grad": (C.c_int, [_P, _P, _PP]),
    "sb_lap_pressure": (C.c_int, [_P, _P, _P]),
    "sb_restrict": (C.c_int, [_P, C.c_int, C.c_int, _PP, _PP]),
    "sb_prolong": (C.c_int, [_P, C.c_int, C.c_int, _PP, _PP]),
    "sb_diagonal": (C.c_int, [_P, C.c_int, C.c_int, _PP]),
    "sb_schur_inv": (C.c_int, [_P, _P, _P, _P]),
    "sb_gmres_flat": (C.c_int, [C.c_longlong, _P, C.c_int, C.c_int, C.c_double, C.c_double, _P, _P, _P, _P,
                                C.POINTER(C.c_int), C.POINTER(C.c_int)]),
    "sb_set_profiling": (None, [_P, C.c_int]),
    "sb_get_kernel_stats": (C.c_int, [_P, C.POINTER(KernelStats)]),
    "sb_launch_count": (C.c_longlong, [_P]),
    "sb_set_graphs": (None, [_P, C.c_int]),
    "sb_device_bytes": (C.c_longlong, [_P]),
    "sb_set_stream": (C.c_int, [_P, _P]),
    "sb_nccl_id_bytes": (C.c_int, []),
    "sb_nccl_unique_id": (C.c_int, [C.c_char_p]),
    "sb_dist_create": (_P, [C.POINTER(C.c_int), C.c_double, C.POINTER(C.c_int), C.c_int, C.c_int, C.c_int,
                            C.c_int, C.c_char_p]),
    "sb_dist_destroy": (None, [_P]),
    "sb_dist_stream": (_P, [_P]),
    "sb_dist_set_stream": (None, [_P, _P]),
    "sb_dist_uses_nccl": (C.c_int, [_P]),
    "sb_host_alloc": (_P, [C.c_longlong]),
    "sb_host_free": (None, [_P]),
    "sb_dist_info": (C.c_int, [_P, C.POINTER(C.c_int)]),
    "sb_dist_set_profiling": (None, [_P, C.c_int]),
    "sb_dist_get_kernel_stats": (C.c_int, [_P, C.POINTER(KernelStats)]),
    "sb_dist_launch_count": (C.c_longlong, [_P]),
    "sb_dist_set_coefficients": (C.c_int, [_P, C.c_double, _PP, _P, _PP, _P]),
    "sb_dist_apply_M": (C.c_int, [_P, _PP, _P, _PP, _P]),
    "sb_dist_precond_apply": (C.c_int, [_P, C.POINTER(Precond), C.POINTER(Smoother), _PP, _P, _PP, _P]),
    "sb_dist_gmres_solve": (C.c_int, [_P, C.POINTER(Precond), C.POINTER(Gmres), C.POINTER(Smoother),
                                      _PP, _P, _PP, _P, C.POINTER(HistoryRow), C.c_int,
                                      C.POINTER(C.c_int), C.POINTER(C.c_int), C.POINTER(C.c_longlong)]),
}

_lib = None


def load(path: os.PathLike | str | None = None):
    """Load the shared library (no GPU needed just to load / inspect symbols)."""
    global _lib
    if _lib is not None and path is None:
        return _lib
    p = pathlib.Path(path) if path is not None else LIB_PATH
    if not p.exists():
        raise RuntimeError(
            f"{p} is missing: build the CUDA library first (python -c 'import __graft_entry__ as g; g.build()'); "
            "there is no CPU fallback")
    lib = C.CDLL(str(p))
    for name, (res, args) in _SIGS.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if path is None:
        _lib = lib
    return lib


def check(rc: int):
    """Map C-ABI status codes to the reference's exception types."""
    if rc == SB_OK:
        return
    msg = (load().sb_last_error() or b"").decode()
    if rc == SB_EINVAL:
        raise ValueError(msg)
    if rc == SB_EDOM:
        raise ZeroDivisionError(msg)
    if rc == SB_ENOMEM:
        raise MemoryError(msg)
    raise RuntimeError(f"stokesb200 CUDA failure: {msg}")


def address(a) -> int:
    """Address of a C-contiguous float64 NumPy array or torch tensor (host or CUDA)."""
    if isinstance(a, np.ndarray):
        if a.dtype != np.float64 or not a.flags.c_contiguous:
            raise TypeError("need C-contiguous float64 arrays")
        return a.ctypes.data
    # torch tensor (device-resident inputs for the in-HBM bench path)
    if str(getattr(a, "dtype", "")) != "torch.float64" or not a.is_contiguous():
        raise TypeError("need contiguous float64 tensors")
    return a.data_ptr()


def ptr(a):
    """``c_void_p`` to an array that keeps the array alive while the pointer
    object lives: ``ptr(_f64(x))`` passed straight into a C call must not let
    a temporary contiguous copy be freed before the call runs."""
    out = C.c_void_p(address(a))
    out._keep = a
    return out


def parr(arrs):
    """Pointer array for a list of arrays.  The returned ctypes array keeps the
    arrays alive: callers pass temporaries (``[_f64(c) for c in ...]`` copies
    of non-contiguous views) that must outlive the C call."""
    arrs = list(arrs)
    vals = [C.c_void_p(address(a) if a is not None else 0) for a in arrs]
    out = (C.c_void_p * max(len(vals), 1))(*vals)
    out._keep = arrs
    return out


class PinnedPool:
    """Recycled page-locked host buffers for arrays the API returns.

    D2H copies into fresh pageable NumPy pages run at a fraction of PCIe speed
    (first-touch faults + staging); a returned array is a view of a pinned
    buffer that goes back to the pool when the array is garbage-collected.
    """

    def __init__(self):
        self.free = {}

    def array(self, shape):
        import weakref
        n = int(np.prod(shape)) * 8
        lst = self.free.get(n)
        p = lst.pop() if lst else None
        if p is None:
            p = load().sb_host_alloc(max(n, 8))
            if not p:
                return np.zeros(shape)
        buf = (C.c_double * max(int(np.prod(shape)), 1)).from_address(p)
        arr = np.frombuffer(buf, dtype=np.float64, count=int(np.prod(shape))).reshape(shape)
        # every element is overwritten by the device->host copy of the result
        weakref.finalize(buf, self._give_back, n, p)
        return arr

    def _give_back(self, n, p):
        self.free.setdefault(n, []).append(p)


pinned = PinnedPool()
