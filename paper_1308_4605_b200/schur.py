"""Approximate Schur-complement inverse -- drop-in mirror of ``stokesmg.schur``.

Reference: ``/root/reference/pkg/src/stokesmg/schur.py``.  ``SchurSign`` /
``SchurConfig`` (:28-44) are the same configuration types.  The application
S~^-1 r = -theta Lrho^-1 r + V r (:59-78) runs on the device inside the
preconditioner kernels (``k_schur`` / ``k_p1_glue``); ``schur_diagonal``
(:47-56) is kept as the host-side definition of V.
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
