"""Device path vs the reference's golden vectors and vs the CPU oracle.

Every test calls the sm_100a kernels through the C ABI (libstokesb200.so) via
the package's reference-shaped API.  Tolerances: component kernels 1e-12
relative (the device uses h^-1 multiplies and 1/rho_face where the reference
divides -- roundoff-level); GMRES solves: iteration count
within +-1 (observed: equal) and solution relative L2 <= 1e-8 (north_star).
"""

from __future__ import annotations

import numpy as np
import pytest

from conftest import arr, cases, face, oracle_coef, oracle_geo, pkg_coeff, pkg_grid, relerr

pytestmark = pytest.mark.gpu

KTOL = 1e-12


def _fields(e):
    from paper_1308_4605_b200.grid import CellField, FaceField, StokesVector
    g = pkg_grid(e)

    def F(key):
        return FaceField(g, tuple(face(e["name"], key, g.dim)))

    def Cf(key):
        return CellField(g, arr(e["name"], key))

    return g, F, Cf, StokesVector


@pytest.mark.parametrize("e", cases("operators"), ids=lambda e: e["name"])
def test_operators_vs_golden(e):
    from paper_1308_4605_b200 import operators as OPS
    g, F, Cf, SV = _fields(e)
    c = pkg_coeff(e, grid=g)
    ctx = OPS._ctx_for(c, g)
    m = OPS.apply_M(SV(F("u"), Cf("p")), c, ctx=ctx)
    for a in range(g.dim):
        assert relerr(m.u.components[a], arr(e["name"], f"Mu{a}")) <= KTOL, a
    assert relerr(m.p.data, arr(e["name"], "Mp")) <= KTOL
    assert relerr(OPS.apply_Lrho(Cf("p"), c, ctx=ctx).data, arr(e["name"], "Lp")) <= KTOL
    au = OPS.apply_A(F("u"), c, ctx=ctx)
    want = [arr(e["name"], f"Mu{a}") for a in range(g.dim)]
    # A u = M_u - G p
    from oracle import stokes_oracle as O
    gp = O.grad(oracle_geo(e), arr(e["name"], "p"))
    for a in range(g.dim):
        w = want[a] - gp[a]
        if not g.periodic(a):
            w[(slice(None),) * a + (0,)] = 0.0
            w[(slice(None),) * a + (-1,)] = 0.0
        assert relerr(au.components[a], w) <= 1e-11


@pytest.mark.parametrize("e", cases("operators"), ids=lambda e: e["name"])
def test_smoothers_transfers_vs_golden(e):
    from paper_1308_4605_b200 import multigrid as MG
    g, F, Cf, SV = _fields(e)
    c = pkg_coeff(e, grid=g)
    hier = MG.build_hierarchy(g, c)
    n = e["name"]
    x = MG.smooth(hier, 0, "face", F("sx0"), F("srhs"), 0.8)
    for a in range(g.dim):
        assert relerr(x.components[a], arr(n, f"sx1{a}")) <= KTOL, a
    y = MG.smooth(hier, 0, "cell", Cf("cy0"), Cf("cyrhs"), 0.8)
    assert relerr(y.data, arr(n, "cy1")) <= KTOL
    # fused residual -> restriction
    rr = MG.residual_restrict(hier, 0, "face", F("sx0"), F("srhs"))
    for a in range(g.dim):
        assert relerr(rr.components[a], arr(n, f"rrf{a}")) <= KTOL, a
    rc = MG.residual_restrict(hier, 0, "cell", Cf("cy0"), Cf("cyrhs"))
    assert relerr(rc.data, arr(n, "rrc")) <= KTOL
    # pure restriction: x = 0 -> residual = rhs
    from paper_1308_4605_b200.grid import CellField, FaceField
    z = FaceField.zeros(g)
    rf = MG.residual_restrict(hier, 0, "face", z, F("u"))
    for a in range(g.dim):
        assert np.array_equal(rf.components[a], arr(n, f"rf{a}")), a
    assert np.array_equal(MG.residual_restrict(hier, 0, "cell", CellField.zeros(g), Cf("p")).data, arr(n, "rc"))
    # prolongation onto zero fine fields
    gc = g.coarsened()
    pin = FaceField(gc, tuple(face(n, "pin", g.dim)))
    pf = MG.prolong_add(hier, 0, "face", pin, FaceField.zeros(g))
    for a in range(g.dim):
        # interior faces only: boundary faces are never touched by the device
        sl = g.interior_slices(a)
        assert np.array_equal(pf.components[a][sl], arr(n, f"pf{a}")[sl]), a
    pc = MG.prolong_add(hier, 0, "cell", CellField(gc, arr(n, "pinc")), CellField.zeros(g))
    assert np.array_equal(pc.data, arr(n, "pc"))
    # coefficient coarsening on the device
    lv1 = hier.levels[1][1]
    ref = oracle_coef(e, prefix=n + "/coarse")
    for a in range(g.dim):
        assert np.array_equal(lv1.rho_face.components[a], ref.rho_face[a]), a
    assert np.array_equal(lv1.mu_cell.data, ref.mu_cell)
    for k, v in ref.mu_edge.items():
        assert np.array_equal(lv1.mu_node_edge.arrays[k], v), k


@pytest.mark.parametrize("e", cases("vcycle"), ids=lambda e: e["name"])
def test_vcycles_preconditioners_vs_golden(e):
    from paper_1308_4605_b200 import multigrid as MG
    from paper_1308_4605_b200.precond import PrecondConfig, Preconditioner, PrecondKind
    from paper_1308_4605_b200.schur import SchurConfig, SchurSign
    g, F, Cf, SV = _fields(e)
    c = pkg_coeff(e, grid=g)
    n = e["name"]
    hier = MG.build_hierarchy(g, c)
    assert len(hier) == e["levels"]
    p = MG.SmootherParams()
    vf = MG.vcycle(F("rhsf"), hier, p, "face")
    for a in range(g.dim):
        assert relerr(vf.components[a], arr(n, f"vf{a}")) <= 1e-11, a
    assert relerr(MG.vcycle(Cf("rhsc"), hier, p, "cell").data, arr(n, "vcell")) <= 1e-11
    m2 = MG.mg_solve(F("rhsf"), hier, p, 2, "face")
    for a in range(g.dim):
        assert relerr(m2.components[a], arr(n, f"mg2f{a}")) <= 1e-11, a
    assert relerr(MG.mg_solve(Cf("rhsc"), hier, p, 2, "cell").data, arr(n, "mg2c")) <= 1e-11
    r = SV(F("ru"), Cf("rp"))
    for key, want in e["vcycles"].items():
        kind, sign = key[:2], key[2:]
        pre = Preconditioner(c, PrecondConfig(kind=PrecondKind(kind), schur=SchurConfig(sign=SchurSign(sign))))
        out = pre.apply(r)
        assert pre.scalar_vcycles == want, key
        for a in range(g.dim):
            assert relerr(out.u.components[a], arr(n, f"{key}_u{a}")) <= 1e-11, (key, a)
        assert relerr(out.p.data, arr(n, f"{key}_p")) <= 1e-11, key
        # bit-identical repeat (reference tests/test_precond.py:97-99)
        again = pre.apply(r)
        assert np.array_equal(again.p.data, out.p.data)


@pytest.mark.parametrize("e", cases("gmres"), ids=lambda e: e["name"])
def test_gmres_vs_golden(e):
    from paper_1308_4605_b200.grid import CellField, FaceField, StokesVector, pack_stokes
    from paper_1308_4605_b200.krylov import GmresConfig, gmres_solve
    from paper_1308_4605_b200.precond import PrecondConfig, PrecondKind
    g = pkg_grid(e)
    c = pkg_coeff(e, grid=g)
    n = e["name"]
    rhs = StokesVector(FaceField(g, tuple(face(n, "bu", g.dim))), CellField(g, arr(n, "bp")))
    from paper_1308_4605_b200.schur import SchurConfig, SchurSign
    pc = PrecondConfig(kind=PrecondKind(e["precond"]),
                       schur=SchurConfig(sign=SchurSign(e.get("schur_sign", "minus"))))
    x, hist = gmres_solve(rhs, c, pc, GmresConfig(restart=e["restart"], track_true_residual=True))
    assert hist.status == e["status"]
    assert abs(hist.iterations - e["iterations"]) <= 1
    ref = StokesVector(FaceField(g, tuple(face(n, "xu", g.dim))), CellField(g, arr(n, "xp")))
    xr, xg = pack_stokes(ref), pack_stokes(x)
    assert np.linalg.norm(xg - xr) <= 1e-8 * np.linalg.norm(xr)
    h = arr(n, "hist")
    rows = np.array(hist.rows(), dtype=float)
    k = min(len(rows), len(h))
    assert np.array_equal(rows[:k, 1], h[:k, 1])  # cumulative scalar V-cycles
    assert np.allclose(rows[:k, 2], h[:k, 2], rtol=1e-6)  # r_P per iteration
    assert np.allclose(rows[:k, 3], h[:k, 3], rtol=1e-5, atol=1e-12 * h[0, 3])  # r_true


def test_graph_reused_across_coefficient_sets():
    """A pooled context keeps its captured P^-1 graph when new coefficients with
    the same theta arrive (sb_set_coefficients); the replay must see the new
    values: solve a perturbed set first, then the golden set on the same context."""
    from paper_1308_4605_b200.grid import CellField, FaceField, StokesVector, pack_stokes
    from paper_1308_4605_b200.krylov import GmresConfig, gmres_solve
    from paper_1308_4605_b200.operators import DeviceContext
    from paper_1308_4605_b200.precond import PrecondConfig, PrecondKind, Preconditioner
    e = [x for x in cases("gmres") if x["name"] == "gm_C5_16_P1"][0]
    g = pkg_grid(e)
    c = pkg_coeff(e, grid=g)
    n = e["name"]
    rhs = StokesVector(FaceField(g, tuple(face(n, "bu", g.dim))), CellField(g, arr(n, "bp")))
    pert = pkg_coeff(e, grid=g)
    pert.mu_cell.data[...] *= 1.7
    for k in pert.mu_node_edge.arrays:
        pert.mu_node_edge.arrays[k] = pert.mu_node_edge.arrays[k] * 1.7
    gcfg = GmresConfig(restart=e["restart"], track_true_residual=False)
    pc = PrecondConfig(kind=PrecondKind(e["precond"]))
    P1 = Preconditioner(pert, pc)
    h0 = P1.ctx.h
    x0, _ = gmres_solve(rhs, pert, pc, gcfg, precond=P1)
    del P1  # back to the pool
    P2 = Preconditioner(c, pc)
    assert P2.ctx.h == h0  # same context, same captured graph
    x, hist = gmres_solve(rhs, c, pc, gcfg, precond=P2)
    assert abs(hist.iterations - e["iterations"]) <= 1
    ref = StokesVector(FaceField(g, tuple(face(n, "xu", g.dim))), CellField(g, arr(n, "xp")))
    xr, xg = pack_stokes(ref), pack_stokes(x)
    assert np.linalg.norm(xg - xr) <= 1e-8 * np.linalg.norm(xr)
    assert np.linalg.norm(pack_stokes(x0) - xr) > 1e-3 * np.linalg.norm(xr)


@pytest.mark.parametrize("name,n,kind", [("C2", 256, "P1"), ("C2", 256, "P2"), ("C3", 32, "P1"),
                                         ("C4", 32, "P1"), ("C5", 32, "P2")])
def test_gmres_vs_oracle_baseline_recipes(name, n, kind):
    """BASELINE recipes (C2 at its full 256^2) solved by the device and by the oracle."""
    from oracle import stokes_oracle as O
    from paper_1308_4605_b200 import problems as PR
    from paper_1308_4605_b200.grid import pack_stokes
    from paper_1308_4605_b200.krylov import GmresConfig, gmres_solve
    from paper_1308_4605_b200.precond import PrecondConfig, PrecondKind
    case = PR.make_case(name, n)
    cs, rs, spec = PR.prepare(case)
    gcfg = GmresConfig(restart=case.restart, max_iters=500, rtol=1e-9, track_true_residual=False)
    x, hist = gmres_solve(rs, cs, PrecondConfig(kind=PrecondKind(kind)), gcfg)
    g = case.grid
    bcn = tuple((lo.value, hi.value) for lo, hi in g.bc)
    geo = O.Geo(g.cells, g.h, bcn)
    oc = O.Coef(cs.theta, cs.rho_cell.data, list(cs.rho_face.components), cs.mu_cell.data,
                dict(cs.mu_node_edge.arrays), cs.gamma_cell.data, "stress")
    u, p, oh = O.gmres_solve(geo, oc, list(rs.u.components), rs.p.data, O.PrecondOpts(kind=kind),
                             O.GmresOpts(restart=case.restart, track_true_residual=False))
    assert hist.status == oh.status == "converged"
    assert abs(hist.iterations - oh.iterations) <= 1
    # compare after unscaling and null projection (problems.py:170-177)
    xu, xp = O.project_nulls(geo, oc, list(x.u.components), x.p.data / spec.c)
    ou, op = O.project_nulls(geo, oc, u, p / spec.c)
    a, b = O.pack(geo, xu, xp), O.pack(geo, ou, op)
    assert np.linalg.norm(a - b) <= 1e-8 * np.linalg.norm(b)


def test_full_size_c3_properties():
    """C3 at its BASELINE size (128^3): converges to 1e-9 with a small true residual,
    deterministic to the bit; the oracle is too slow here (387 s)."""
    from paper_1308_4605_b200 import problems as PR
    from paper_1308_4605_b200.krylov import GmresConfig, gmres_solve, true_residual
    from paper_1308_4605_b200.grid import norm2
    from paper_1308_4605_b200.precond import P1, PrecondConfig, Preconditioner
    case = PR.make_case("C3")
    cs, rs, spec = PR.prepare(case)
    P = Preconditioner(cs, PrecondConfig(kind=P1))
    gcfg = GmresConfig(restart=50, max_iters=500, rtol=1e-9, track_true_residual=False)
    x1, h1 = gmres_solve(rs, cs, None, gcfg, precond=P)
    assert h1.status == "converged"
    assert 40 <= h1.iterations <= 75  # reference recipe measured 55
    assert h1.entries[-1].resid_precond <= 1e-9 * h1.entries[0].resid_precond
    rt = true_residual(x1, rs, cs)
    assert rt <= 1e-6 * norm2(rs)
    x2, h2 = gmres_solve(rs, cs, None, gcfg, precond=P)
    assert h2.iterations == h1.iterations
    assert np.array_equal(x2.p.data, x1.p.data)


@pytest.mark.parametrize("cells,bc", [((16, 16, 24), "pp pp pp"), ((16, 24, 32), "nn pp pp"),
                                      ((24, 16, 16), "pp nn ff"), ((16, 32, 40), "fn nf nn"),
                                      ((40, 16, 48), "pp pp nn")])
@pytest.mark.parametrize("form,theta", [("stress", 0.0), ("stress", 0.9), ("laplacian", 0.3)])
def test_colour_sweeps_vs_oracle(cells, bc, form, theta):
    """One smoother sweep (the per-colour passes) on grids mixing periodic,
    no-slip and free-slip axes == the reference's sequential red-then-black
    passes, all components, face and cell."""
    from oracle import stokes_oracle as O
    from paper_1308_4605_b200 import multigrid as MG
    from paper_1308_4605_b200.grid import BoundaryCondition, CellField, FaceField, GridSpec
    from paper_1308_4605_b200.operators import ViscousForm, make_coefficients
    names = {"p": "periodic", "n": "no_slip", "f": "free_slip"}
    pairs = [(names[x[0]], names[x[1]]) for x in bc.split()]
    g = GridSpec(cells, 1.0 / cells[0], tuple((BoundaryCondition(a), BoundaryCondition(b)) for a, b in pairs))
    geo = O.Geo(cells, g.h, tuple(pairs))
    rng = np.random.default_rng(sum(cells))
    rho, mu = 0.5 + rng.random(cells), 0.5 + rng.random(cells)
    c = make_coefficients(g, theta, CellField(g, rho), CellField(g, mu), None, ViscousForm(form))
    oc = O.make_coef(geo, theta, rho, mu, None, form)
    hier = MG.build_hierarchy(g, c)
    x = [rng.standard_normal(g.face_shape(a)) for a in range(3)]
    for a in range(3):
        if not g.periodic(a):
            x[a][(slice(None),) * a + (0,)] = 0.0
            x[a][(slice(None),) * a + (-1,)] = 0.0
    r = [rng.standard_normal(g.face_shape(a)) for a in range(3)]
    got = MG.smooth(hier, 0, "face", FaceField(g, tuple(a.copy() for a in x)), FaceField(g, tuple(r)), 1.0)
    want = [a.copy() for a in x]
    O.sweep_face(geo, oc, want, r, O.diag_face(geo, oc), 1.0)
    for a in range(3):
        assert relerr(got.components[a], want[a]) <= 1e-13, a
    y, yr = rng.standard_normal(cells), rng.standard_normal(cells)
    gy = MG.smooth(hier, 0, "cell", CellField(g, y.copy()), CellField(g, yr), 1.0)
    wy = y.copy()
    O.sweep_cell(geo, oc, wy, yr, O.diag_cell(geo, oc), 1.0)
    assert relerr(gy.data, wy) <= 1e-13


@pytest.mark.parametrize("cells,bc", [((16, 16, 24), "pp pp pp"), ((16, 24, 32), "nn pp pp"),
                                      ((24, 16, 16), "pp nn ff"), ((32, 48), "pp nn"), ((24, 16), "fn nf")])
@pytest.mark.parametrize("form,theta", [("stress", 0.0), ("laplacian", 0.4), ("stress_bulk", 1.0)])
def test_split_residual_restriction_bit_identical(cells, bc, form, theta, monkeypatch):
    """Residual field + restriction (large levels, SB_RR_SPLIT) == the fused
    residual->restriction kernels, to the bit, through whole face and cell V-cycles."""
    from paper_1308_4605_b200 import multigrid as MG
    from paper_1308_4605_b200.grid import BoundaryCondition, CellField, FaceField, GridSpec
    from paper_1308_4605_b200.operators import ViscousForm, make_coefficients
    names = {"p": "periodic", "n": "no_slip", "f": "free_slip"}
    pairs = [(names[x[0]], names[x[1]]) for x in bc.split()]
    g = GridSpec(cells, 1.0 / cells[0], tuple((BoundaryCondition(a), BoundaryCondition(b)) for a, b in pairs))
    rng = np.random.default_rng(sum(cells) + len(form))
    rho, mu, gam = 0.5 + rng.random(cells), 0.5 + rng.random(cells), rng.random(cells)
    c = make_coefficients(g, theta, CellField(g, rho), CellField(g, mu), CellField(g, gam), ViscousForm(form))
    rf = FaceField(g, tuple(rng.standard_normal(g.face_shape(a)) for a in range(g.dim)))
    for a in range(g.dim):
        if not g.periodic(a):
            rf.components[a][(slice(None),) * a + (0,)] = 0.0
            rf.components[a][(slice(None),) * a + (-1,)] = 0.0
    rc = CellField(g, rng.standard_normal(cells))
    rc.data[...] -= rc.data.mean()
    out = {}
    for v in ("1", "0"):
        monkeypatch.setenv("SB_RR_SPLIT", v)
        h = MG.build_hierarchy(g, c)
        vf = MG.vcycle(rf, h, MG.SmootherParams(), "face")
        vc = MG.vcycle(rc, h, MG.SmootherParams(), "cell")
        out[v] = ([np.array(x) for x in vf.components], np.array(vc.data))
    for a in range(g.dim):
        assert np.array_equal(out["1"][0][a], out["0"][0][a]), a
    assert np.array_equal(out["1"][1], out["0"][1])
