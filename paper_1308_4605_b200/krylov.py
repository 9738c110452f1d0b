"""Restarted left-preconditioned GMRES on the device -- drop-in for ``stokesmg.krylov``.

Reference: ``/root/reference/pkg/src/stokesmg/krylov.py``.  ``GmresConfig``
(:22-38), ``HistoryEntry`` / ``ConvergenceHistory`` (:40-78) are the same
types; ``gmres_solve`` (:164-214) keeps its signature, stopping rule
(r_P <= rtol r_P(0) + atol, breakdown at max(atol, 1e-14 r_P(0))), restart
semantics and history rows, and runs as one ``sb_gmres_solve`` call: Krylov
vectors live in HBM, the Arnoldi step is classical Gram-Schmidt with one
re-orthogonalisation (CGS2, parity-equivalent to the reference's MGS, SURVEY
§8a row a26) in fused multi-vector kernels, the solution is formed lazily at
restarts / termination, and only the (m+1)-scalar Hessenberg column crosses
to the host per iteration.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .grid import CellField, FaceField, StokesVector, as_grid
from .multigrid import SmootherParams
from .operators import _f64, apply_M
from .precond import PrecondConfig, Preconditioner


@dataclass(frozen=True)
class GmresConfig:
    restart: int = 10
    max_iters: int = 500
    rtol: float = 1e-9
    atol: float = 0.0
    track_true_residual: bool = True

    def __post_init__(self):
        if self.restart < 1:
            raise ValueError("restart must be >= 1")
        if self.max_iters < 1:
            raise ValueError("max_iters must be >= 1")
        if not self.rtol > 0:
            raise ValueError("rtol must be positive")
        if self.atol < 0:
            raise ValueError("atol must be nonnegative")


@dataclass
class HistoryEntry:
    iteration: int
    scalar_vcycles: int
    resid_precond: float
    resid_true: float
    restart: bool


@dataclass
class ConvergenceHistory:
    entries: list = field(default_factory=list)
    status: str = "running"

    def add(self, iteration, scalar_vcycles, resid_precond, resid_true, restart):
        self.entries.append(HistoryEntry(int(iteration), int(scalar_vcycles), float(resid_precond),
                                         float(resid_true), bool(restart)))

    @property
    def iterations(self) -> int:
        return self.entries[-1].iteration if self.entries else 0

    @property
    def converged(self) -> bool:
        return self.status in ("converged", "breakdown")

    def final_true_residual(self) -> float:
        return self.entries[-1].resid_true

    def rows(self):
        return [(e.iteration, e.scalar_vcycles, e.resid_precond, e.resid_true, int(e.restart))
                for e in self.entries]


def gmres_c(cfg) -> _lib.Gmres:
    return _lib.Gmres(int(cfg.restart), int(cfg.max_iters), float(cfg.rtol), float(cfg.atol),
                      int(bool(cfg.track_true_residual)))


def _history(rows, n, status) -> ConvergenceHistory:
    h = ConvergenceHistory()
    for r in rows[:n]:
        h.add(r.iteration, r.scalar_vcycles, r.resid_precond, r.resid_true, r.restart)
    h.status = _lib.STATUS[status]
    return h


def _device_precond(coeff, pcfg, smoother, precond):
    if precond is None:
        return Preconditioner(coeff, pcfg, smoother)
    if not hasattr(precond, "apply") or not hasattr(precond, "scalar_vcycles"):
        raise TypeError("precond must provide .apply(StokesVector) and .scalar_vcycles (krylov.py:180-207)")
    return precond


def _solve_operator_callback(rhs, coeff, P, gcfg):
    """gmres_solve (krylov.py:164-214) for preconditioners that are not the
    fused device P^-1 -- the dense exact-subsolver study path and any
    duck-typed ``precond=`` object (the reference's seam): the Krylov basis and
    Arnoldi run on the device (``gmres_kernel`` / ``sb_gmres_flat``), M on the
    device (one context), and P.apply is called on the host fields as the
    reference calls it."""
    from .grid import pack_stokes, unpack_stokes
    from .operators import _ctx_for
    g = as_grid(rhs.u.grid)
    ctx = _ctx_for(coeff, g)
    history = ConvergenceHistory()
    b_raw = pack_stokes(rhs)
    rhs_norm = float(np.linalg.norm(b_raw))

    def apply_op(v):
        return pack_stokes(P.apply(apply_M(unpack_stokes(g, v), coeff, ctx=ctx)))

    z0 = pack_stokes(P.apply(rhs))
    rp0 = float(np.linalg.norm(z0))
    history.add(0, P.scalar_vcycles, rp0, rhs_norm, False)
    if rp0 <= gcfg.atol or rp0 == 0.0:
        history.status = "converged"
        return StokesVector.zeros(g), history
    target = gcfg.rtol * rp0 + gcfg.atol
    breakdown_tol = max(gcfg.atol, 1e-14 * rp0)

    def callback(k, xvec, rp, restart_flag):
        if gcfg.track_true_residual:
            mx = pack_stokes(apply_M(unpack_stokes(g, xvec), coeff, ctx=ctx))
            rt = float(np.linalg.norm(b_raw - mx))
        else:
            rt = float("nan")
        history.add(k, P.scalar_vcycles, rp, rt, restart_flag)

    xvec, status, _ = gmres_kernel(apply_op, z0, gcfg.restart, gcfg.max_iters, target, breakdown_tol, callback)
    history.status = status
    return unpack_stokes(g, xvec), history


def solve_raw(P: Preconditioner, gcfg, bu, bp, xu, xp):
    """sb_gmres_solve on raw arrays (host NumPy or CUDA tensors, reference layouts).

    Returns (history, status string).  This is the entry the bench uses with
    HBM-resident tensors; ``gmres_solve`` is the same call on host fields.
    """
    gc = gmres_c(gcfg)
    nrows = int(gcfg.max_iters) + 2
    rows = (_lib.HistoryRow * nrows)()
    n_rows, status = C.c_int(0), C.c_int(0)
    vc = C.c_longlong(P.scalar_vcycles)
    _lib.check(P.ctx.lib.sb_gmres_solve(
        P.ctx.h, C.byref(P._pc), C.byref(gc), C.byref(P._sm), _lib.parr(bu), _lib.ptr(bp),
        _lib.parr(xu), _lib.ptr(xp), rows, nrows, C.byref(n_rows), C.byref(status), C.byref(vc)))
    P.scalar_vcycles = int(vc.value)
    return _history(rows, n_rows.value, status.value)


def gmres_solve(rhs, coeff, pcfg: PrecondConfig, gcfg: GmresConfig,
                smoother: SmootherParams | None = None, precond: Preconditioner | None = None):
    """Solve M x = rhs with left-preconditioned restarted GMRES on the B200.

    The right-hand side must already be homogenised (and, for dimensional
    problems, rescaled), exactly as for the reference.
    """
    g = as_grid(rhs.u.grid)
    P = _device_precond(coeff, pcfg, smoother, precond)
    if not isinstance(P, Preconditioner) or P.exact:
        return _solve_operator_callback(rhs, coeff, P, gcfg)
    xu = [_lib.pinned.array(g.face_shape(a)) for a in range(g.dim)]
    xp = _lib.pinned.array(g.cells)
    hist = solve_raw(P, gcfg, [_f64(c) for c in rhs.u.components], _f64(rhs.p.data), xu, xp)
    return StokesVector(FaceField(g, tuple(xu)), CellField(g, xp)), hist


def true_residual(x, rhs, coeff) -> float:
    """|| M x - rhs ||_2 over unknowns, M applied on the device (krylov.py:156-161)."""
    from .grid import norm2
    return norm2(apply_M(x, coeff) - StokesVector(
        FaceField(as_grid(rhs.u.grid), tuple(rhs.u.components)),
        CellField(as_grid(rhs.u.grid), rhs.p.data)))


_APPLY_FN = C.CFUNCTYPE(None, C.POINTER(C.c_double), C.POINTER(C.c_double), C.c_void_p)
_ITER_FN = C.CFUNCTYPE(None, C.c_int, C.POINTER(C.c_double), C.c_double, C.c_int, C.c_void_p)


def gmres_kernel(apply_op, b, restart: int, max_iters: int, target: float, breakdown_tol: float,
                 callback=None):
    """Restarted GMRES on flat vectors for ``apply_op(x) = b`` (krylov.py:81-146).

    Returns ``(x, status, iterations)`` with status ``converged`` /
    ``breakdown`` / ``maxiter`` and the reference's restart, stopping and
    callback semantics (``callback(k, x_k, r_P, restart_flag)`` after every
    iteration).  The basis and the Arnoldi orthogonalisation (CGS2) live on
    the device (``sb_gmres_flat``); ``apply_op`` is called on host NumPy
    vectors, as the reference calls it."""
    b = np.ascontiguousarray(b, dtype=np.float64).reshape(-1)
    n = b.size
    err = []

    def _apply(pin, pout, _user):
        try:
            v = np.ctypeslib.as_array(pin, shape=(n,)).copy()
            w = np.asarray(apply_op(v), dtype=np.float64).reshape(-1)
            np.ctypeslib.as_array(pout, shape=(n,))[:] = w
        except BaseException as e:  # surfaced after the C call returns
            err.append(e)
            np.ctypeslib.as_array(pout, shape=(n,))[:] = 0.0

    def _iter(k, px, rp, rflag, _user):
        if callback is None or err:
            return
        try:
            callback(int(k), np.ctypeslib.as_array(px, shape=(n,)).copy(), float(rp), bool(rflag))
        except BaseException as e:
            err.append(e)

    fa, fi = _APPLY_FN(_apply), _ITER_FN(_iter)
    x = np.zeros(n)
    status, its = C.c_int(0), C.c_int(0)
    rc = _lib.load().sb_gmres_flat(C.c_longlong(n), _lib.ptr(b), int(restart), int(max_iters), float(target),
                                   float(breakdown_tol), C.cast(fa, C.c_void_p),
                                   C.cast(fi, C.c_void_p) if callback is not None else None,
                                   None, _lib.ptr(x), C.byref(status), C.byref(its))
    if err:
        raise err[0]
    _lib.check(rc)
    return x, _lib.STATUS[status.value], int(its.value)
