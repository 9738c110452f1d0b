"""Approximate Schur-complement inverse -- drop-in mirror of ``stokesmg.schur``.

Reference: ``/root/reference/pkg/src/stokesmg/schur.py``.  ``SchurSign`` /
``SchurConfig`` (:28-44) are the same configuration types.  The application
S~^-1 r = -theta Lrho^-1 r + V r (:59-78) runs on the device inside the
preconditioner kernels (``k_schur`` / ``k_p1_glue``) and, as the public seam
``apply_schur_inv(r, coeff, cfg, pressure_solve=)``, through ``sb_schur_inv``;
``schur_diagonal`` (:47-56) is the host-side definition of V.  The dense
``exact_schur_apply`` (reference test tooling over ``_exact``) is out of scope.
"""

from __future__ import annotations

import enum
from dataclasses import dataclass


class SchurSign(enum.Enum):
    MINUS = "minus"
    PLUS = "plus"


MINUS = SchurSign.MINUS
PLUS = SchurSign.PLUS


@dataclass(frozen=True)
class SchurConfig:
    sign: SchurSign = MINUS
    pressure_cycles: int = 1

    def __post_init__(self):
        if self.pressure_cycles < 1:
            raise ValueError("need at least one pressure cycle")


def schur_diagonal(coeff):
    """V: mu (Laplacian), 2 mu (stress), gamma + 4/3 mu (stress + bulk)."""
    form = getattr(coeff.viscous_form, "value", coeff.viscous_form)
    mu = coeff.mu_cell.data
    if form == "laplacian":
        return mu
    if form == "stress":
        return 2.0 * mu
    if form == "stress_bulk":
        return coeff.gamma_cell.data + (4.0 / 3.0) * mu
    raise ValueError(f"unknown viscous form {form}")


def apply_schur_inv(r, coeff, cfg: SchurConfig, pressure_solve=None):
    """Approximate S^-1 r = -theta Lrho^-1 r + V r (schur.py:59-78) on the device.

    ``pressure_solve`` (CellField -> CellField) supplies the Poisson inverse and
    is consulted only for unsteady flow (theta > 0); steady applications are
    purely diagonal.  The combination -theta phi + V r runs in the same kernel
    the preconditioner uses (k_schur, sign +1)."""
    import numpy as np

    from . import _lib
    from .grid import CellField, as_grid
    from .operators import _ctx_for, _f64
    g = as_grid(r.grid)
    phi = None
    if coeff.theta > 0:
        if pressure_solve is None:
            raise ValueError("unsteady Schur inverse needs a pressure solver")
        phi = _f64(pressure_solve(r).data)
    ctx = _ctx_for(coeff, g)
    out = np.zeros(g.cells)
    _lib.check(ctx.lib.sb_schur_inv(ctx.h, _lib.ptr(_f64(r.data)), _lib.ptr(phi) if phi is not None else None,
                                    _lib.ptr(out)))
    return CellField(g, out)


def exact_schur_apply(p, coeff, face_solver=None):
    """Reference -D A^-1 G p through the dense exact velocity solve (schur.py:81-92;
    small grids only): device grad / div and the device-factorised A."""
    from ._exact import DenseFaceSolver
    from .operators import div, grad
    if face_solver is None:
        face_solver = DenseFaceSolver(p.grid, coeff)
    return -div(face_solver.solve(grad(p)))
