"""Pin the CPU oracle (oracle/stokes_oracle.py) against golden vectors made by
running the reference package itself (tests/golden/make_golden.py).

CPU only.  The oracle restates the reference's operation order, so agreement is
bit-exact or within a few ulp; the GMRES solves must reproduce the iteration
counts and the converged solutions."""

from __future__ import annotations

import numpy as np
import pytest

from conftest import arr, cases, face, oracle_coef, oracle_geo, relerr

from oracle import stokes_oracle as O

TOL = 1e-13


@pytest.mark.parametrize("e", cases("operators"), ids=lambda e: e["name"])
def test_operators(e):
    geo, c = oracle_geo(e), oracle_coef(e)
    d, n = geo.dim, e["name"]
    u, p = face(n, "u", d), arr(n, "p")
    mu, mp = O.apply_M(geo, c, u, p)
    for a in range(d):
        assert relerr(mu[a], arr(n, f"Mu{a}")) <= TOL
    assert relerr(mp, arr(n, "Mp")) <= TOL
    assert relerr(O.lrho(geo, c, p), arr(n, "Lp")) <= TOL
    df = O.diag_face(geo, c)
    for a in range(d):
        assert relerr(df[a], arr(n, f"diagf{a}")) <= TOL
    assert relerr(O.diag_cell(geo, c), arr(n, "diagc")) <= TOL


@pytest.mark.parametrize("e", cases("operators"), ids=lambda e: e["name"])
def test_smoothers(e):
    geo, c = oracle_geo(e), oracle_coef(e)
    d, n = geo.dim, e["name"]
    x = face(n, "sx0", d)
    O.sweep_face(geo, c, x, face(n, "srhs", d), O.diag_face(geo, c), 0.8)
    for a in range(d):
        assert relerr(x[a], arr(n, f"sx1{a}")) <= TOL
    y = arr(n, "cy0")
    O.sweep_cell(geo, c, y, arr(n, "cyrhs"), O.diag_cell(geo, c), 0.8)
    assert relerr(y, arr(n, "cy1")) <= TOL


@pytest.mark.parametrize("e", cases("operators"), ids=lambda e: e["name"])
def test_transfers_and_coarsening(e):
    geo, c = oracle_geo(e), oracle_coef(e)
    d, n = geo.dim, e["name"]
    rf = O.restrict_face(geo, face(n, "u", d))
    for a in range(d):
        assert np.array_equal(rf[a], arr(n, f"rf{a}"))
    assert np.array_equal(O.restrict_cell(geo, arr(n, "p")), arr(n, "rc"))
    gc = geo.half()
    pf = O.prolong_face(gc, face(n, "pin", d))
    for a in range(d):
        assert np.array_equal(pf[a], arr(n, f"pf{a}"))
    assert np.array_equal(O.prolong_cell(gc, arr(n, "pinc")), arr(n, "pc"))
    _, cc = O.coarsen(geo, c)
    ref = oracle_coef(e, prefix=n + "/coarse")
    for a in range(d):
        assert np.array_equal(cc.rho_face[a], ref.rho_face[a])
    assert np.array_equal(cc.mu_cell, ref.mu_cell)
    for k in cc.mu_edge:
        assert np.array_equal(cc.mu_edge[k], ref.mu_edge[k])
    # residual -> restriction as in the V-cycle
    x = face(n, "sx0", d)
    r = O._resid(geo, c, x, face(n, "srhs", d), "face")
    rr = O.restrict_face(geo, r)
    for a in range(d):
        assert relerr(rr[a], arr(n, f"rrf{a}")) <= TOL
    rc = O.restrict_cell(geo, O._resid(geo, c, arr(n, "cy0"), arr(n, "cyrhs"), "cell"))
    assert relerr(rc, arr(n, "rrc")) <= TOL


@pytest.mark.parametrize("e", cases("vcycle"), ids=lambda e: e["name"])
def test_vcycles_and_preconditioners(e):
    geo, c = oracle_geo(e), oracle_coef(e)
    d, n = geo.dim, e["name"]
    hier = O.Hierarchy(geo, c)
    assert len(hier.levels) == e["levels"]
    sm = O.Smoother()
    vf = O.vcycle(hier, face(n, "rhsf", d), "face", sm)
    for a in range(d):
        assert relerr(vf[a], arr(n, f"vf{a}")) <= 1e-12
    assert relerr(O.vcycle(hier, arr(n, "rhsc"), "cell", sm), arr(n, "vcell")) <= 1e-12
    m2 = O.mg_solve(hier, face(n, "rhsf", d), "face", sm, 2)
    for a in range(d):
        assert relerr(m2[a], arr(n, f"mg2f{a}")) <= 1e-12
    assert relerr(O.mg_solve(hier, arr(n, "rhsc"), "cell", sm, 2), arr(n, "mg2c")) <= 1e-12
    ru, rp = face(n, "ru", d), arr(n, "rp")
    for key, want in e["vcycles"].items():
        kind, sign = key[:2], key[2:]
        P = O.Precond(geo, c, O.PrecondOpts(kind=kind, sign=-1.0 if sign == "minus" else 1.0))
        xu, xp = P.apply(ru, rp)
        assert P.vcycles == want
        for a in range(d):
            assert relerr(xu[a], arr(n, f"{key}_u{a}")) <= 1e-12, (key, a)
        assert relerr(xp, arr(n, f"{key}_p")) <= 1e-12, key


@pytest.mark.parametrize("e", cases("gmres"), ids=lambda e: e["name"])
def test_gmres_solves(e):
    geo, c = oracle_geo(e), oracle_coef(e)
    d, n = geo.dim, e["name"]
    bu, bp = face(n, "bu", d), arr(n, "bp")
    sign = -1.0 if e.get("schur_sign", "minus") == "minus" else 1.0
    u, p, hist = O.gmres_solve(geo, c, bu, bp, O.PrecondOpts(kind=e["precond"], sign=sign),
                               O.GmresOpts(restart=e["restart"], track_true_residual=True))
    assert hist.status == e["status"]
    assert hist.iterations == e["iterations"]
    ref_h = arr(n, "hist")
    got_h = np.array(hist.rows, dtype=float)
    assert got_h.shape == ref_h.shape
    assert np.array_equal(got_h[:, [0, 1, 4]], ref_h[:, [0, 1, 4]])
    assert np.allclose(got_h[:, 2], ref_h[:, 2], rtol=1e-9, atol=0)
    xo = O.pack(geo, u, p)
    xr = O.pack(geo, face(n, "xu", d), arr(n, "xp"))
    assert np.linalg.norm(xo - xr) <= 1e-10 * np.linalg.norm(xr)


def test_known_answer_two_by_two():
    """GMRES hand-solved 2x2 (reference tests/test_krylov.py:38-53)."""
    A = np.diag([2.0, 5.0])
    b = np.array([2.0, 10.0])
    seen = []
    x, status, k = O.gmres_flat(lambda v: A @ v, b, 5, 10, 1e-13 * 10.4, 0.0,
                                lambda k, xk, rp, rf: seen.append(rp))
    assert status in ("converged", "breakdown") and k <= 2
    assert np.allclose(x, [1.0, 2.0], atol=1e-12)
    assert seen[0] == pytest.approx(2.0 * np.sqrt(141525.0) / 629.0, rel=1e-12)


def test_paper_transfer_examples():
    """Paper restriction/prolongation examples (reference tests/test_multigrid.py:143-175)."""
    g = O.Geo((8, 8), 1.0, (("no_slip",) * 2,) * 2)
    u = [np.zeros(g.fshape(a)) for a in range(2)]
    u[0][1, 2] = 8.0
    u[0][2, 2] = 4.0
    assert O.restrict_face(g, u)[0][1, 1] == pytest.approx(2.0)
    gc = O.Geo((4, 4), 1.0, g.bc)
    c = [np.zeros(gc.fshape(a)) for a in range(2)]
    c[0][2, 2] = 4.0
    c[0][2, 1] = 8.0
    assert O.prolong_face(gc, c)[0][4, 4] == pytest.approx(5.0)
    c2 = [np.zeros(gc.fshape(a)) for a in range(2)]
    c2[0][2, 2] = 4.0
    c2[0][3, 2] = 8.0
    assert O.prolong_face(gc, c2)[0][5, 4] == pytest.approx(4.5)


@pytest.mark.parametrize("e", cases("affine"), ids=lambda e: e["name"])
def test_inhomogeneous_walls(e):
    """apply_A with BoundaryValues, boundary_lift and homogenize (operators.py:224-264,
    348-360, 471-512) against the reference on every wall-bounded grid and form."""
    from conftest import golden_bvals
    geo, c = oracle_geo(e), oracle_coef(e)
    d, n = geo.dim, e["name"]
    normal, tang = golden_bvals(e)
    lift = O.boundary_lift(geo, normal)
    for a in range(d):
        assert np.array_equal(lift[a], arr(n, f"lift{a}"))
    u = face(n, "u", d)
    au, a0 = O.apply_A(geo, c, u, tang), O.apply_A(geo, c, u)
    mu, mp = O.apply_M(geo, c, u, np.zeros(geo.cells))
    for a in range(d):
        assert relerr(au[a], arr(n, f"Au{a}")) <= TOL
        assert relerr(a0[a], arr(n, f"A0{a}")) <= TOL
        assert relerr(mu[a], arr(n, f"Mu{a}")) <= TOL
    assert relerr(mp, arr(n, "Mp")) <= TOL
    hu, hp = O.homogenize(geo, c, normal, tang, face(n, "ru", d), arr(n, "rp"))
    for a in range(d):
        assert relerr(hu[a], arr(n, f"hu{a}")) <= TOL
    assert relerr(hp, arr(n, "hp")) <= TOL


def test_homogenize_incompatible_rejected():
    """operators.py:505-509 (reference test_operators.py:486-492): net inflow with a zero
    divergence source is rejected."""
    geo = O.Geo((8, 8), 1 / 8, (("no_slip",) * 2,) * 2)
    rng = np.random.default_rng(2)
    c = O.make_coef(geo, 0.0, 0.5 + rng.random((8, 8)), 0.5 + rng.random((8, 8)))
    z = [np.zeros(geo.fshape(a)) for a in range(2)]
    with pytest.raises(ValueError, match="incompatible"):
        O.homogenize(geo, c, {(0, 0): np.full(8, 1.0)}, {}, z, np.zeros((8, 8)))
