"""Inhomogeneous walls on the device: apply_A(u, coeff, bvals), apply_M with a
boundary lift, homogenize (operators.py:224-264, 348-365, 471-512), against the
reference's golden vectors (tests/golden: ``affine`` cases, every wall-bounded
grid x form) and the reference's own homogenize tests (test_operators.py:476-527)
restated on the device path.  Tolerance 1e-12 relative (component kernels,
see test_gpu_parity.py); the roundtrip uses the reference test's 1e-10 bound."""

from __future__ import annotations

import numpy as np
import pytest

from conftest import arr, cases, face, golden_bvals, oracle_coef, oracle_geo, pkg_coeff, pkg_grid, relerr

pytestmark = pytest.mark.gpu

KTOL = 1e-12


def _bvals(e, g):
    from paper_1308_4605_b200.operators import BoundaryValues
    normal, tang = golden_bvals(e)
    return BoundaryValues(g, normal, tang)


@pytest.mark.parametrize("e", cases("affine"), ids=lambda e: e["name"])
def test_affine_apply_vs_golden(e):
    from paper_1308_4605_b200 import operators as OPS
    from paper_1308_4605_b200.grid import CellField, FaceField, StokesVector
    g = pkg_grid(e)
    c = pkg_coeff(e, grid=g)
    n, d = e["name"], g.dim
    ctx = OPS._ctx_for(c, g)
    bv = _bvals(e, g)
    u = FaceField(g, tuple(face(n, "u", d)))
    au = OPS.apply_A(u, c, bv, ctx=ctx)
    a0 = OPS.apply_A(u, c, ctx=ctx)
    m = OPS.apply_M(StokesVector(u, CellField(g, np.zeros(g.cells))), c, ctx=ctx)
    for a in range(d):
        assert relerr(au.components[a], arr(n, f"Au{a}")) <= KTOL, a
        assert relerr(a0.components[a], arr(n, f"A0{a}")) <= KTOL, a
        assert relerr(m.u.components[a], arr(n, f"Mu{a}")) <= KTOL, a
    assert relerr(m.p.data, arr(n, "Mp")) <= KTOL


@pytest.mark.parametrize("e", cases("affine"), ids=lambda e: e["name"])
def test_homogenize_vs_golden(e):
    from paper_1308_4605_b200 import operators as OPS
    from paper_1308_4605_b200.grid import CellField, FaceField, StokesVector
    g = pkg_grid(e)
    c = pkg_coeff(e, grid=g)
    n, d = e["name"], g.dim
    rhs = StokesVector(FaceField(g, tuple(face(n, "ru", d))), CellField(g, arr(n, "rp")))
    hom = OPS.homogenize(_bvals(e, g), c, rhs)
    for a in range(d):
        assert relerr(hom.u.components[a], arr(n, f"hu{a}")) <= KTOL, a
    assert relerr(hom.p.data, arr(n, "hp")) <= KTOL


def _noslip_case(n, seed, theta=1.0):
    from oracle import stokes_oracle as O
    from paper_1308_4605_b200.grid import NO_SLIP, GridSpec
    from paper_1308_4605_b200.operators import STRESS, make_coefficients
    from paper_1308_4605_b200.grid import CellField
    rng = np.random.default_rng(seed)
    g = GridSpec((n, n), 1.0 / n, ((NO_SLIP, NO_SLIP), (NO_SLIP, NO_SLIP)))
    rho, mu = 0.5 + rng.random((n, n)), 0.5 + rng.random((n, n))
    c = make_coefficients(g, theta, CellField(g, rho), CellField(g, mu), viscous_form=STRESS)
    geo = O.Geo((n, n), 1.0 / n, (("no_slip",) * 2,) * 2)
    oc = O.make_coef(geo, theta, rho, mu)
    return rng, g, c, geo, oc


def test_homogenize_zero_values_noop():
    """reference test_operators.py:477-484: zero boundary values leave the rhs unchanged."""
    from paper_1308_4605_b200.grid import CellField, FaceField, StokesVector
    from paper_1308_4605_b200.operators import BoundaryValues, homogenize
    rng, g, c, _, _ = _noslip_case(8, 1)
    ru = tuple(rng.standard_normal(g.face_shape(a)) for a in range(2))
    rp = rng.standard_normal(g.cells)
    rp -= rp.mean()
    out = homogenize(BoundaryValues.zeros(g), c, StokesVector(FaceField(g, ru), CellField(g, rp)))
    for a in range(2):
        assert np.array_equal(out.u.components[a], ru[a])
    assert np.array_equal(out.p.data, rp)


def test_homogenize_incompatible_rejected():
    """reference test_operators.py:486-492 (operators.py:505-509)."""
    from paper_1308_4605_b200.grid import StokesVector
    from paper_1308_4605_b200.operators import BoundaryValues, homogenize
    _, g, c, _, _ = _noslip_case(8, 2, theta=0.0)
    with pytest.raises(ValueError, match="incompatible"):
        homogenize(BoundaryValues(g, {(0, 0): np.full(8, 1.0)}, {}), c, StokesVector.zeros(g))


def test_manufactured_affine_roundtrip():
    """reference test_operators.py:494-527 on the device path: homogenize, solve
    the homogeneous system with GMRES + P2 on the B200, add the lift back; the
    affine residual (checked with the CPU oracle) is <= 1e-10 |rhs|."""
    from oracle import stokes_oracle as O
    from paper_1308_4605_b200.grid import CellField, FaceField, StokesVector
    from paper_1308_4605_b200.krylov import GmresConfig, gmres_solve
    from paper_1308_4605_b200.operators import BoundaryValues, boundary_lift, homogenize
    from paper_1308_4605_b200.precond import PrecondConfig, PrecondKind
    n = 16
    rng, g, c, geo, oc = _noslip_case(n, 7)
    lid = np.sin(2 * np.pi * np.arange(n + 1) / n)
    inflow = np.sin(2 * np.pi * (np.arange(n) + 0.5) / n)
    bv = BoundaryValues(g, {(0, 0): inflow.copy(), (0, 1): inflow.copy()}, {(1, 1, 0): lid})
    ru = tuple(rng.standard_normal(g.face_shape(a)) for a in range(2))
    rp = rng.standard_normal(g.cells)
    rp -= rp.mean()
    lift = boundary_lift(bv)
    net = float(O.div(geo, [np.asarray(x) for x in lift.components]).sum())
    rp -= net / g.n_cell_unknowns() / g.h ** 2
    rhs = StokesVector(FaceField(g, ru), CellField(g, rp))
    hom = homogenize(bv, c, rhs)
    x, hist = gmres_solve(hom, c, PrecondConfig(kind=PrecondKind.P2), GmresConfig(rtol=1e-13, max_iters=60))
    assert hist.converged
    full = [np.array(x.u.components[a]) + lift.components[a] for a in range(2)]
    ou = O.apply_A(geo, oc, full, {(1, 1, 0): lid})
    gp = O.grad(geo, np.array(x.p.data))
    res_u = [ou[a] + gp[a] - ru[a] for a in range(2)]
    res_p = -O.div(geo, full) - rp
    err = np.sqrt(sum(np.sum(res_u[a][geo.inner(a)] ** 2) for a in range(2)) + np.sum(res_p ** 2))
    nr = np.sqrt(sum(np.sum(ru[a][geo.inner(a)] ** 2) for a in range(2)) + np.sum(rp ** 2))
    assert err <= 1e-10 * max(1.0, nr)
