"""First sweep of a V-cycle level from x = 0 (multigrid.py:409-439).

Every V-cycle level starts from a zero iterate, so its first smoother sweep
does not need to read the components that are still zero, and on all-periodic
pad-free levels the first colour pass can store both colours and replace the
zero fill (k_face_colour / k_cell_colour, Z variants).  The arithmetic is the
same on the same values, so V-cycles, mg_solve and full GMRES solves must be
bit-identical to the plain passes (SB_ZERO_FIRST=0) on every boundary mix and
viscous form, including odd extents (two-phase levels), walls (zero fill
kept) and the bulk form (fill kept: its rows read the divergence).
"""

from __future__ import annotations

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

CASES = [("C1", (32, 32), "stress"), ("C2", (64, 64), "stress"), ("C3", (32, 32, 32), "stress"),
         ("C3", (32, 32, 32), "laplacian"), ("C3", (16, 32, 64), "stress_bulk"), ("C4", (32, 32, 32), "stress"),
         ("C5", (24, 40, 64), "stress"), ("C1", (48, 40), "laplacian")]


def _vcycles(name, cells, form, zero_first, monkeypatch):
    from dataclasses import replace
    from paper_1308_4605_b200 import multigrid as MG
    from paper_1308_4605_b200 import problems as PR
    from paper_1308_4605_b200.grid import CellField, FaceField
    from paper_1308_4605_b200.operators import ViscousForm
    monkeypatch.setenv("SB_ZERO_FIRST", "1" if zero_first else "0")
    case = PR.make_case(name, cells)
    cs, rs, _ = PR.prepare(case)
    if form != "stress":
        cs = replace(cs, viscous_form=ViscousForm(form), gamma_cell=CellField.full(case.grid, 0.7))
    hier = MG.build_hierarchy(case.grid, cs)
    sp = MG.SmootherParams()
    out = {}
    fv = MG.vcycle(rs.u, hier, sp, "face")
    out["face"] = [c.copy() for c in fv.components]
    out["cell"] = [MG.vcycle(rs.p, hier, sp, "cell").data.copy()]
    out["face2"] = [c.copy() for c in MG.mg_solve(rs.u, hier, MG.SmootherParams(omega=0.8), 2, "face").components]
    rng = np.random.default_rng(3)
    r2 = FaceField(case.grid, tuple(rng.standard_normal(case.grid.face_shape(a)) for a in range(case.grid.dim)))
    out["face_rand"] = [c.copy() for c in MG.vcycle(r2, hier, sp, "face").components]
    hier.ctx.close()
    return out


@pytest.mark.parametrize("name,cells,form", CASES, ids=lambda v: str(v))
def test_zero_first_vcycle_bit_identical(name, cells, form, monkeypatch):
    a = _vcycles(name, cells, form, True, monkeypatch)
    b = _vcycles(name, cells, form, False, monkeypatch)
    for k in a:
        for u, v in zip(a[k], b[k]):
            assert np.array_equal(u, v), k


@pytest.mark.parametrize("name,cells", [("C5", 64), ("C4", 32), ("C2", 64)])
def test_zero_first_gmres_bit_identical(name, cells, monkeypatch):
    """Full solves (P^-1 graph captured per setting): identical histories and solutions."""
    from paper_1308_4605_b200 import problems as PR
    from paper_1308_4605_b200.grid import pack_stokes
    from paper_1308_4605_b200.krylov import GmresConfig, gmres_solve
    from paper_1308_4605_b200.precond import P1, PrecondConfig, Preconditioner
    case = PR.make_case(name, cells)
    cs, rs, _ = PR.prepare(case)
    res = {}
    for zf in ("1", "0"):
        monkeypatch.setenv("SB_ZERO_FIRST", zf)
        P = Preconditioner(cs, PrecondConfig(kind=P1))
        P.set_graphs(False)
        P.set_graphs(True)
        x, h = gmres_solve(rs, cs, None, GmresConfig(restart=case.restart, rtol=1e-9), precond=P)
        res[zf] = (pack_stokes(x), h.iterations, [r.resid_precond for r in h.entries])
        del P
    assert res["1"][1] == res["0"][1]
    assert res["1"][2] == res["0"][2]
    assert np.array_equal(res["1"][0], res["0"][0])
