"""Wavefront red-black sweeps (sb_wave.cu: both colour passes of a component in
one persistent launch, black planes trailing red planes in L2) against the
reference's sequential red-then-black passes (oracle) and bit-for-bit against
the per-colour kernels.  SB_WAVE_MIN (planes) is read when a context is
created: 4 forces the wave path on every 3D level, 0 disables it."""

from __future__ import annotations

import os

import numpy as np
import pytest

from conftest import arr, cases, face, pkg_coeff, pkg_grid, relerr

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True)
def _stored_edge_viscosity(monkeypatch):
    """The wave kernels (opt-in) read the stored mu_e arrays; compare them with
    per-colour passes that do the same (no derived edge viscosities)."""
    monkeypatch.setenv("SB_MUE_DERIVED", "0")

NAMES = {"p": "periodic", "n": "no_slip", "f": "free_slip"}


class wave_min:
    def __init__(self, v):
        self.v = str(v)

    def __enter__(self):
        from paper_1308_4605_b200 import operators
        self.old = os.environ.get("SB_WAVE_MIN")
        os.environ["SB_WAVE_MIN"] = self.v
        operators._POOL.clear()

    def __exit__(self, *a):
        from paper_1308_4605_b200 import operators
        if self.old is None:
            os.environ.pop("SB_WAVE_MIN", None)
        else:
            os.environ["SB_WAVE_MIN"] = self.old
        operators._POOL.clear()


def _setup(cells, bc, form, theta):
    from oracle import stokes_oracle as O
    from paper_1308_4605_b200.grid import BoundaryCondition, CellField, GridSpec
    from paper_1308_4605_b200.operators import ViscousForm, make_coefficients
    pairs = [(NAMES[x[0]], NAMES[x[1]]) for x in bc.split()]
    g = GridSpec(cells, 1.0 / cells[0], tuple((BoundaryCondition(a), BoundaryCondition(b)) for a, b in pairs))
    geo = O.Geo(cells, g.h, tuple(pairs))
    rng = np.random.default_rng(sum(cells) + len(form))
    rho, mu = 0.5 + rng.random(cells), 0.5 + rng.random(cells)
    c = make_coefficients(g, theta, CellField(g, rho), CellField(g, mu), None, ViscousForm(form))
    oc = O.make_coef(geo, theta, rho, mu, None, form)
    x = [rng.standard_normal(g.face_shape(a)) for a in range(3)]
    for a in range(3):
        if not g.periodic(a):
            x[a][(slice(None),) * a + (0,)] = 0.0
            x[a][(slice(None),) * a + (-1,)] = 0.0
    r = [rng.standard_normal(g.face_shape(a)) for a in range(3)]
    y, yr = rng.standard_normal(cells), rng.standard_normal(cells)
    return g, geo, c, oc, x, r, y, yr


def _sweep(g, c, x, r, y, yr, omega):
    from paper_1308_4605_b200 import multigrid as MG
    from paper_1308_4605_b200.grid import CellField, FaceField
    hier = MG.build_hierarchy(g, c)
    fx = MG.smooth(hier, 0, "face", FaceField(g, tuple(a.copy() for a in x)), FaceField(g, tuple(r)), omega)
    cy = MG.smooth(hier, 0, "cell", CellField(g, y.copy()), CellField(g, yr), omega)
    return [np.array(a) for a in fx.components], np.array(cy.data)


@pytest.mark.parametrize("cells,bc", [((16, 48, 64), "pp pp pp"), ((12, 40, 64), "nn pp pp"),
                                      ((20, 48, 64), "pp nn ff"), ((8, 8, 8), "pp pp pp"),
                                      ((6, 48, 70), "fn nf nn"), ((64, 32, 32), "pp pp nn")])
@pytest.mark.parametrize("form,theta", [("stress", 0.0), ("stress", 0.9), ("laplacian", 0.3)])
def test_wave_sweeps_vs_oracle_and_per_colour(cells, bc, form, theta):
    from oracle import stokes_oracle as O
    g, geo, c, oc, x, r, y, yr = _setup(cells, bc, form, theta)
    with wave_min(4):
        wf, wc = _sweep(g, c, x, r, y, yr, 0.9)
    with wave_min(0):
        pf, pc = _sweep(g, c, x, r, y, yr, 0.9)
    for a in range(3):
        assert np.array_equal(wf[a], pf[a]), a
    assert np.array_equal(wc, pc)
    want = [a.copy() for a in x]
    O.sweep_face(geo, oc, want, r, O.diag_face(geo, oc), 0.9)
    for a in range(3):
        assert relerr(wf[a], want[a]) <= 1e-13, a
    wy = y.copy()
    O.sweep_cell(geo, oc, wy, yr, O.diag_cell(geo, oc), 0.9)
    assert relerr(wc, wy) <= 1e-13


@pytest.mark.parametrize("name", ["gm_C3_16_P1", "gm_C4_16_P1", "gm_C5_16_P1"])
def test_wave_gmres_vs_golden(name):
    """Full GMRES solves with the wave path on every level: same iterations and the
    same solution (to the bit) as the per-colour path, within 1e-8 of the reference."""
    from paper_1308_4605_b200.grid import CellField, FaceField, StokesVector, pack_stokes
    from paper_1308_4605_b200.krylov import GmresConfig, gmres_solve
    from paper_1308_4605_b200.precond import PrecondConfig, PrecondKind
    e = [x for x in cases("gmres") if x["name"] == name][0]
    g = pkg_grid(e)
    c = pkg_coeff(e, grid=g)
    n = e["name"]
    rhs = StokesVector(FaceField(g, tuple(face(n, "bu", g.dim))), CellField(g, arr(n, "bp")))
    pc, gc = PrecondConfig(kind=PrecondKind(e["precond"])), GmresConfig(restart=e["restart"])
    with wave_min(4):
        xw, hw = gmres_solve(rhs, c, pc, gc)
    with wave_min(0):
        xp, hp = gmres_solve(rhs, c, pc, gc)
    assert hw.iterations == hp.iterations
    assert np.array_equal(pack_stokes(xw), pack_stokes(xp))
    assert abs(hw.iterations - e["iterations"]) <= 1
    ref = StokesVector(FaceField(g, tuple(face(n, "xu", g.dim))), CellField(g, arr(n, "xp")))
    xr = pack_stokes(ref)
    assert np.linalg.norm(pack_stokes(xw) - xr) <= 1e-8 * np.linalg.norm(xr)
