"""Block preconditioners P1..P5 on the device -- drop-in mirror of ``stokesmg.precond``.

Reference: ``/root/reference/pkg/src/stokesmg/precond.py``.  ``PrecondKind`` /
``PrecondConfig`` (:27-53) are the same types; ``Preconditioner`` (:56-168)
keeps its contract -- ``apply(StokesVector) -> StokesVector`` and the
``scalar_vcycles`` counter (:94, :101) -- but owns a device context
(``sb_ctx``): the multigrid hierarchy is built on the B200 at construction and
each ``apply`` is one ``sb_precond_apply`` call (velocity V-cycle, pressure
V-cycle, glue kernels and null projection, replayed as a CUDA graph).
With dense exact subsolvers (``exact_subsolvers=True``, the reference's
small-grid LU study path, ``_exact.py``) the same block algebra (:111-168) is
composed from device operator calls (div, grad, apply_A, apply_schur_inv) and
the device-factorised dense solves; it runs no V-cycles and leaves the counter
untouched, as the reference.
"""

from __future__ import annotations

import ctypes as C
import enum
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .grid import CellField, FaceField, StokesVector, as_grid
from .multigrid import MgHierarchy, SmootherParams, smoother_c
from .operators import DeviceContext, _f64, velocity_null_components
from .schur import MINUS, SchurConfig


class PrecondKind(enum.Enum):
    P1 = "P1"
    P2 = "P2"
    P3 = "P3"
    P4 = "P4"
    P5 = "P5"
    IDENTITY = "identity"


P1 = PrecondKind.P1
P2 = PrecondKind.P2
P3 = PrecondKind.P3
P4 = PrecondKind.P4
P5 = PrecondKind.P5
IDENTITY = PrecondKind.IDENTITY

_KIND_CODE = {"P1": 1, "P2": 2, "P3": 3, "P4": 4, "P5": 5, "identity": 0}


@dataclass(frozen=True)
class PrecondConfig:
    kind: PrecondKind = P2
    velocity_cycles: int = 1
    schur: SchurConfig = field(default_factory=SchurConfig)
    exact_subsolvers: bool = False

    def __post_init__(self):
        if self.velocity_cycles < 1:
            raise ValueError("need at least one velocity cycle")


def precond_c(cfg) -> _lib.Precond:
    sign = getattr(cfg.schur.sign, "value", cfg.schur.sign)
    return _lib.Precond(_KIND_CODE[getattr(cfg.kind, "value", cfg.kind)], int(cfg.velocity_cycles),
                        -1 if sign == MINUS.value else 1, int(cfg.schur.pressure_cycles))


class Preconditioner:
    """Applies P^{-1}; counts scalar V-cycles (d per velocity solve, 1 per Poisson)."""

    def __init__(self, coeff, cfg: PrecondConfig, smoother: SmootherParams | None = None):
        self.exact = bool(getattr(cfg, "exact_subsolvers", False))
        if self.exact:
            self._init_exact(coeff, cfg, smoother)
            return
        self.coeff = coeff
        self.grid = as_grid(coeff.grid)
        self.cfg = cfg
        self.smoother = smoother if smoother is not None else SmootherParams()
        self.scalar_vcycles = 0
        self._null_comps = velocity_null_components(self.grid, coeff)
        kind = getattr(cfg.kind, "value", cfg.kind)
        if kind != "identity" and not self.grid.can_coarsen():
            raise ValueError(f"grid {self.grid.cells} cannot be coarsened; need even counts >= 4")
        self.ctx = DeviceContext.acquire(self.grid, coeff.viscous_form)
        self.ctx.set_coefficients(coeff)
        self._hierarchy = MgHierarchy(self.ctx, coeff) if kind != "identity" else None
        self._pc = precond_c(cfg)
        self._sm = smoother_c(self.smoother)

    # -- dense exact subsolvers (precond.py:73-82, :91-168) ---------------------

    def _init_exact(self, coeff, cfg, smoother):
        from ._exact import DenseCellSolver, DenseFaceSolver
        self.coeff = coeff
        self.grid = as_grid(coeff.grid)
        self.cfg = cfg
        self.smoother = smoother if smoother is not None else SmootherParams()
        self.scalar_vcycles = 0
        self._null_comps = velocity_null_components(self.grid, coeff)
        self.ctx = None
        self._hierarchy = None
        self._face_solver = self._cell_solver = None
        if getattr(cfg.kind, "value", cfg.kind) == "identity":
            return
        self._face_solver = DenseFaceSolver(self.grid, coeff)
        if self._needs_poisson():
            self._cell_solver = DenseCellSolver(self.grid, coeff)

    def _needs_poisson(self) -> bool:
        return getattr(self.cfg.kind, "value", self.cfg.kind) == "P1" or self.coeff.theta > 0

    def velocity_solve(self, b):
        if self._face_solver is None:
            raise RuntimeError("velocity_solve is the exact-subsolver seam (device V-cycles run inside apply)")
        return self._face_solver.solve(b)

    def pressure_solve(self, b):
        if self._cell_solver is None:
            raise RuntimeError("pressure_solve is the exact-subsolver seam (device V-cycles run inside apply)")
        return self._cell_solver.solve(b)

    def _apply_exact(self, r) -> StokesVector:
        from .operators import apply_A, div, grad
        from .schur import apply_schur_inv, schur_diagonal
        kind = getattr(self.cfg.kind, "value", self.cfg.kind)
        if kind == "identity":
            return r.copy()
        g, coeff = self.grid, self.coeff
        sign = -1.0 if getattr(self.cfg.schur.sign, "value", self.cfg.schur.sign) == MINUS.value else 1.0
        schur = lambda b: apply_schur_inv(b, coeff, self.cfg.schur,
                                          self.pressure_solve if coeff.theta > 0 else None)
        if kind == "P1":
            xu_star = self.velocity_solve(r.u)
            b_c = div(xu_star) + r.p
            phi = self.pressure_solve(b_c)
            xu = xu_star.copy()
            gphi = grad(phi)
            for a in range(g.dim):
                xu.components[a][...] -= gphi.components[a] / coeff.rho_face.components[a]
                if not g.periodic(a):
                    xu.components[a][(slice(None),) * a + (0,)] = 0.0
                    xu.components[a][(slice(None),) * a + (-1,)] = 0.0
            s_inv = CellField(g, schur_diagonal(coeff) * b_c.data - coeff.theta * phi.data)
            x = StokesVector(xu, s_inv * sign)
        elif kind == "P2":
            xu = self.velocity_solve(r.u)
            x = StokesVector(xu, schur(div(xu) + r.p) * sign)
        elif kind == "P3":
            xp = schur(r.p) * sign
            x = StokesVector(self.velocity_solve(r.u - grad(xp)), xp)
        elif kind == "P4":
            x = StokesVector(self.velocity_solve(r.u), schur(r.p) * sign)
        elif kind == "P5":
            xu_star = self.velocity_solve(r.u)
            xp = schur(div(xu_star) + r.p) * sign
            b2 = r.u - grad(xp) - apply_A(xu_star, coeff)
            x = StokesVector(xu_star + self.velocity_solve(b2), xp)
        else:
            raise ValueError(f"unknown preconditioner kind {kind}")
        from .grid import subtract_mean
        x = StokesVector(x.u, subtract_mean(x.p))
        for a in self._null_comps:
            view = x.u.interior(a)
            view -= view.mean()
        return x

    def apply(self, r) -> StokesVector:
        if self.exact:
            return self._apply_exact(r)
        g = self.grid
        ru = [_f64(c) for c in r.u.components]
        xu = [np.zeros(g.face_shape(a)) for a in range(g.dim)]
        xp = np.zeros(g.cells)
        vc = C.c_longlong(self.scalar_vcycles)
        _lib.check(self.ctx.lib.sb_precond_apply(
            self.ctx.h, C.byref(self._pc), C.byref(self._sm), _lib.parr(ru),
            _lib.ptr(_f64(r.p.data)), _lib.parr(xu), _lib.ptr(xp), C.byref(vc)))
        self.scalar_vcycles = int(vc.value)
        return StokesVector(FaceField(g, tuple(xu)), CellField(g, xp))

    def __del__(self):
        ctx = getattr(self, "ctx", None)
        if ctx is not None:
            self.ctx = None
            ctx.release()

    # device-level knobs (measurement)
    def set_graphs(self, enabled: bool):
        self.ctx.lib.sb_set_graphs(self.ctx.h, int(bool(enabled)))

    def set_profiling(self, enabled: bool):
        self.ctx.lib.sb_set_profiling(self.ctx.h, int(bool(enabled)))

    def kernel_stats(self) -> dict:
        s = _lib.KernelStats()
        self.ctx.lib.sb_get_kernel_stats(self.ctx.h, C.byref(s))
        return {k: getattr(s, k) for k, _ in s._fields_}

    def launch_count(self) -> int:
        return int(self.ctx.lib.sb_launch_count(self.ctx.h))

    def device_bytes(self) -> int:
        return int(self.ctx.lib.sb_device_bytes(self.ctx.h))
