"""Device-side make_coefficients + rescale (sb_set_cell_coefficients).

Only the cell arrays cross the boundary; the face densities and the node/edge
viscosities are averaged on the device (operators.py:81-104, to_stagger_mean's
expression) and theta, mu, mu_e, gamma multiplied by the rescale factor in the
host's operation order (operators.py:532-550).  Every level of the hierarchy,
the per-level specialisation flags and full GMRES solves must equal the host
path (make_coefficients -> rescale -> set_coefficients) to the bit, on 2D/3D,
periodic and walled grids, constant and variable density, and the bulk form.
"""

from __future__ import annotations

from dataclasses import replace

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

CASES = [("C1", (32, 32), "stress"), ("C2", (64, 64), "stress"), ("C3", (32, 32, 32), "stress"),
         ("C4", (32, 32, 32), "stress"), ("C5", (16, 32, 64), "stress"), ("C3", (32, 32, 32), "stress_bulk"),
         ("C2", (48, 32), "laplacian")]


def _prep(name, cells, form):
    from paper_1308_4605_b200 import problems as PR
    from paper_1308_4605_b200.grid import CellField
    from paper_1308_4605_b200.operators import ViscousForm, make_coefficients
    case = PR.make_case(name, cells)
    coeff = case.coeff
    if form != "stress":
        g = case.grid
        gam = CellField(g, 0.5 + np.random.default_rng(5).random(g.cells))
        coeff = make_coefficients(g, coeff.theta, coeff.rho_cell, coeff.mu_cell, gam, ViscousForm(form))
        case = replace(case, coeff=coeff)
    cs, rs, spec = PR.prepare(case)
    return case, coeff, cs, rs, spec


@pytest.mark.parametrize("name,cells,form", CASES, ids=lambda v: str(v))
def test_cell_coefficients_match_host_averaging(name, cells, form):
    from paper_1308_4605_b200 import multigrid as MG
    from paper_1308_4605_b200.operators import DeviceContext
    case, coeff, cs, rs, spec = _prep(name, cells, form)
    g = case.grid
    a = DeviceContext(g, cs.viscous_form)
    a.set_coefficients(cs)
    b = DeviceContext(g, cs.viscous_form)
    gam = coeff.gamma_cell if form == "stress_bulk" else None
    b.set_cell_coefficients(coeff.theta, coeff.rho_cell, coeff.mu_cell, gam, scale=spec.c)
    assert a.num_levels() == b.num_levels()
    la, lb = MG.MgHierarchy(a, cs).levels, MG.MgHierarchy(b, cs).levels
    for lvl, ((ga, ca), (gb, cb)) in enumerate(zip(la, lb)):
        assert a.level_flags(lvl) == b.level_flags(lvl), lvl
        for x, y in zip(ca.rho_face.components, cb.rho_face.components):
            assert np.array_equal(x, y), lvl
        assert np.array_equal(ca.mu_cell.data, cb.mu_cell.data), lvl
        for k in ca.mu_node_edge.arrays:
            assert np.array_equal(ca.mu_node_edge.arrays[k], cb.mu_node_edge.arrays[k]), (lvl, k)
        if form == "stress_bulk":
            assert np.array_equal(ca.gamma_cell.data, cb.gamma_cell.data), lvl
    a.close()
    b.close()


@pytest.mark.parametrize("name,cells", [("C4", (32, 32, 32)), ("C5", (32, 32, 32)), ("C2", (64, 64))])
def test_cell_coefficients_gmres_bit_identical(name, cells):
    from paper_1308_4605_b200.grid import pack_stokes
    from paper_1308_4605_b200.krylov import GmresConfig, gmres_solve
    from paper_1308_4605_b200.precond import P1, PrecondConfig, Preconditioner
    case, coeff, cs, rs, spec = _prep(name, cells, "stress")
    gcfg = GmresConfig(restart=case.restart, rtol=1e-9)
    P = Preconditioner(cs, PrecondConfig(kind=P1))
    x1, h1 = gmres_solve(rs, cs, None, gcfg, precond=P)
    P.ctx.set_cell_coefficients(coeff.theta, coeff.rho_cell, coeff.mu_cell, None, scale=spec.c)
    x2, h2 = gmres_solve(rs, cs, None, gcfg, precond=P)
    assert h1.iterations == h2.iterations
    assert [r.resid_precond for r in h1.entries] == [r.resid_precond for r in h2.entries]
    assert np.array_equal(pack_stokes(x1), pack_stokes(x2))


def test_cell_coefficients_validation():
    from paper_1308_4605_b200 import problems as PR
    from paper_1308_4605_b200.operators import DeviceContext
    case = PR.make_case("C1", 16)
    ctx = DeviceContext(case.grid, case.coeff.viscous_form)
    with pytest.raises(ValueError):
        ctx.set_cell_coefficients(-1.0, case.coeff.rho_cell, case.coeff.mu_cell)
    with pytest.raises(ValueError):
        ctx.set_cell_coefficients(0.0, case.coeff.rho_cell, case.coeff.mu_cell, scale=0.0)
    with pytest.raises(ValueError):
        ctx.set_cell_coefficients(0.0, np.ones((8, 8)), case.coeff.mu_cell)
    ctx.close()
