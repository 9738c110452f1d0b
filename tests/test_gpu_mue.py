"""Per-level operand specialisations: edge viscosities derived from
mu_cell on all-periodic levels, and one 1/rho for constant-density levels.

The face rows of an all-periodic level whose uploaded mu_edge equals the
four-cell mean of mu_cell (operators.py:90-104) to 4e-15 relative compute the
edge viscosities from mu_cell instead of streaming the three mu_edge arrays.
Rescaled coefficients (operators.py:532-550) differ from that mean by a few
ulp, so the operator changes at roundoff level only: the derived and the
stored path must agree to 1e-13 (operators, one P^-1) and give the same GMRES
iteration count with solutions within 1e-12; coefficient sets whose mu_edge is
not the cell mean must keep the stored path.
"""

from __future__ import annotations

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _setup(name, n, derive, monkeypatch, edit=None):
    from paper_1308_4605_b200 import problems as PR
    from paper_1308_4605_b200.precond import P1, PrecondConfig, Preconditioner
    case = PR.make_case(name, n)
    cs, rs, spec = PR.prepare(case)
    if edit is not None:
        cs = edit(cs)
    monkeypatch.setenv("SB_MUE_DERIVED", "2" if derive else "0")  # 2: walled levels too
    P = Preconditioner(cs, PrecondConfig(kind=P1))
    monkeypatch.delenv("SB_MUE_DERIVED")
    return case, cs, rs, P


def _rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def _pack(x):
    from paper_1308_4605_b200.grid import pack_stokes
    return pack_stokes(x)


@pytest.mark.parametrize("name,n", [("C5", 32), ("C3", 64), ("C1", 64), ("C4", 32), ("C2", 64)])
def test_derived_matches_stored(name, n, monkeypatch):
    from paper_1308_4605_b200 import operators as OPS
    from paper_1308_4605_b200.krylov import GmresConfig, gmres_solve
    out = {}
    for derive in (False, True):
        case, cs, rs, P = _setup(name, n, derive, monkeypatch)
        assert P.ctx.mue_derived(0) == derive
        if name != "C1":  # variable mu: coarse levels inject mu_e (multigrid.py:150-169)
            assert not P.ctx.mue_derived(1)
        m = OPS.apply_M(rs, cs, ctx=P.ctx)
        z = P.apply(rs)
        gcfg = GmresConfig(restart=case.restart, max_iters=500, rtol=1e-9, track_true_residual=False)
        x, hist = gmres_solve(rs, cs, None, gcfg, precond=P)
        out[derive] = (_pack(m), _pack(z), _pack(x), hist.iterations, hist.status)
        del P
    (m0, z0, x0, i0, s0), (m1, z1, x1, i1, s1) = out[False], out[True]
    assert _rel(m1, m0) <= 1e-13
    assert _rel(z1, z0) <= 1e-13
    assert s0 == s1 == "converged"
    assert i1 == i0
    assert _rel(x1, x0) <= 1e-12


def test_constant_mu_derives_every_level(monkeypatch):
    case, cs, rs, P = _setup("C1", 64, True, monkeypatch)
    assert all(P.ctx.mue_derived(l) for l in range(P.ctx.num_levels()))


def test_walls_and_foreign_edges_keep_stored_path(monkeypatch):
    from dataclasses import replace
    from paper_1308_4605_b200 import operators as OPS
    from paper_1308_4605_b200.grid import NodeEdgeField
    # a wall-bounded finest level derives (two-cell boundary means); its coarse
    # levels inject mu_e and keep the stored path.  By default (1) all-periodic
    # levels and 3D levels with walls along the contiguous axis only (C4)
    # derive; walls along another axis keep the stored path unless asked
    # (SB_MUE_DERIVED=2).
    _, _, _, P = _setup("C4", 16, True, monkeypatch)
    assert P.ctx.mue_derived(0) and not P.ctx.mue_derived(1)
    del P
    from paper_1308_4605_b200 import problems as PR
    from paper_1308_4605_b200.grid import NO_SLIP, PERIODIC, CellField, GridSpec
    from paper_1308_4605_b200.operators import make_coefficients
    from paper_1308_4605_b200.precond import P1, PrecondConfig, Preconditioner
    case = PR.make_case("C4", 16)
    cs4, _, _ = PR.prepare(case)
    monkeypatch.delenv("SB_MUE_DERIVED", raising=False)
    assert Preconditioner(cs4, PrecondConfig(kind=P1)).ctx.mue_derived(0)
    gy = GridSpec((16, 16, 16), 1.0 / 16, ((PERIODIC, PERIODIC), (NO_SLIP, NO_SLIP), (PERIODIC, PERIODIC)))
    rng = np.random.default_rng(2)
    csy = make_coefficients(gy, 0.5, CellField(gy, 1.0 + rng.random(gy.cells)), CellField(gy, 1.0 + rng.random(gy.cells)))
    assert not Preconditioner(csy, PrecondConfig(kind=P1)).ctx.mue_derived(0)

    # harmonic edge means: not the arithmetic cell mean -> stored path, and the
    # operator is the one of the given mu_edge (oracle)
    def harmonic(cs):
        arrs = {k: 1.0 / (1.0 / v + 1e-3) for k, v in cs.mu_node_edge.arrays.items()}
        return replace(cs, mu_node_edge=NodeEdgeField(cs.grid, arrs))

    case, cs, rs, P = _setup("C5", 16, True, monkeypatch, edit=harmonic)
    assert not P.ctx.mue_derived(0)
    from oracle import stokes_oracle as O
    g = case.grid
    geo = O.Geo(g.cells, g.h, tuple((lo.value, hi.value) for lo, hi in g.bc))
    oc = O.Coef(cs.theta, cs.rho_cell.data, list(cs.rho_face.components), cs.mu_cell.data,
                dict(cs.mu_node_edge.arrays), cs.gamma_cell.data, "stress")
    mu, mp = O.apply_M(geo, oc, list(rs.u.components), rs.p.data)
    m = OPS.apply_M(rs, cs, ctx=P.ctx)
    for a in range(3):
        assert _rel(m.u.components[a], mu[a]) <= 1e-12

    # one perturbed edge value also disables it
    def one_off(cs):
        arrs = {k: v.copy() for k, v in cs.mu_node_edge.arrays.items()}
        k0 = sorted(arrs)[0]
        arrs[k0][3, 4, 5] *= 1.0 + 1e-12
        return replace(cs, mu_node_edge=NodeEdgeField(cs.grid, arrs))

    _, _, _, P2 = _setup("C5", 16, True, monkeypatch, edit=one_off)
    assert not P2.ctx.mue_derived(0)


@pytest.mark.parametrize("cells,bc", [((16, 24, 32), "nn pp pp"), ((24, 16, 16), "pp nn ff"),
                                      ((16, 32, 40), "fn nf nn"), ((32, 48), "pp nn"), ((24, 16), "fn nf")])
@pytest.mark.parametrize("form,theta", [("stress", 0.0), ("laplacian", 0.4), ("stress_bulk", 1.0)])
def test_walled_levels_derive_vs_oracle(cells, bc, form, theta, monkeypatch):
    """Derived edge viscosities on wall-bounded levels (no-slip, free-slip and
    mixed walls, 2D and 3D, every viscous form): apply_M and one face V-cycle
    equal the oracle's with the stored mu_edge."""
    from oracle import stokes_oracle as O
    from paper_1308_4605_b200 import multigrid as MG
    from paper_1308_4605_b200 import operators as OPS
    from paper_1308_4605_b200.grid import (BoundaryCondition, CellField, FaceField, GridSpec,
                                           StokesVector)
    from paper_1308_4605_b200.operators import ViscousForm, make_coefficients
    names = {"p": "periodic", "n": "no_slip", "f": "free_slip"}
    pairs = [(names[x[0]], names[x[1]]) for x in bc.split()]
    g = GridSpec(cells, 1.0 / cells[0], tuple((BoundaryCondition(a), BoundaryCondition(b)) for a, b in pairs))
    geo = O.Geo(cells, g.h, tuple(pairs))
    rng = np.random.default_rng(sum(cells) + len(form))
    rho, mu, gam = 0.5 + rng.random(cells), 0.5 + rng.random(cells), rng.random(cells)
    c = make_coefficients(g, theta, CellField(g, rho), CellField(g, mu), CellField(g, gam), ViscousForm(form))
    oc = O.make_coef(geo, theta, rho, mu, gam, form)
    x = [rng.standard_normal(g.face_shape(a)) for a in range(g.dim)]
    for a in range(g.dim):
        if not g.periodic(a):
            x[a][(slice(None),) * a + (0,)] = 0.0
            x[a][(slice(None),) * a + (-1,)] = 0.0
    p = rng.standard_normal(cells)
    monkeypatch.setenv("SB_MUE_DERIVED", "2")
    h = MG.build_hierarchy(g, c)
    assert h.ctx.mue_derived(0)
    m = OPS.apply_M(StokesVector(FaceField(g, tuple(x)), CellField(g, p)), c, ctx=h.ctx)
    mu_, mp_ = O.apply_M(geo, oc, [a.copy() for a in x], p)
    for a in range(g.dim):
        assert _rel(m.u.components[a], mu_[a]) <= 1e-13, a
    vf = MG.vcycle(FaceField(g, tuple(x)), h, MG.SmootherParams(), "face")
    want = O.vcycle(O.Hierarchy(geo, oc), [a.copy() for a in x], "face")
    for a in range(g.dim):
        assert _rel(np.asarray(vf.components[a]), want[a]) <= 1e-12, a


# ---- constant density: one 1/rho for the cell rows (LevelDev::beta_const) ------


def _precond_with_env(cs, env, monkeypatch):
    from paper_1308_4605_b200.precond import P1, PrecondConfig, Preconditioner
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    P = Preconditioner(cs, PrecondConfig(kind=P1))
    for k in env:
        monkeypatch.delenv(k)
    return P


@pytest.mark.parametrize("name,n", [("C5", 32), ("C4", 16), ("C2", 32)])
def test_const_density_bit_identical(name, n, monkeypatch):
    """C5 (rho = 1) runs every level with the constant 1/rho; C4/C2 (variable rho)
    keep the arrays.  A constant-rho copy of C4 (walls in z) also takes the
    constant path; in every case P^-1 and the GMRES solve are identical to the
    bit to the array path (SB_CONST_BETA=0)."""
    from dataclasses import replace
    from paper_1308_4605_b200 import problems as PR
    from paper_1308_4605_b200.grid import CellField, pack_stokes
    from paper_1308_4605_b200.krylov import GmresConfig, gmres_solve
    from paper_1308_4605_b200.operators import average_cell_to_faces
    case = PR.make_case(name, n)
    cs, rs, spec = PR.prepare(case)
    variants = [cs]
    if name != "C5":
        g = case.grid
        rho = CellField(g, np.full(g.cells, 2.5))
        variants.append(replace(cs, rho_cell=rho, rho_face=average_cell_to_faces(rho)))
    for k, c in enumerate(variants):
        out = {}
        for on in ("1", "0"):
            P = _precond_with_env(c, {"SB_CONST_BETA": on}, monkeypatch)
            const = [P.ctx.beta_const(l) for l in range(P.ctx.num_levels())]
            if on == "0":
                assert not any(const)
            elif name == "C5" or k == 1:
                assert all(const)
            else:
                assert not const[0]
            z = P.apply(rs)
            x, h = gmres_solve(rs, c, None, GmresConfig(restart=case.restart, rtol=1e-9), precond=P)
            out[on] = (pack_stokes(z), pack_stokes(x), h.iterations)
            del P
        assert np.array_equal(out["1"][0], out["0"][0])
        assert np.array_equal(out["1"][1], out["0"][1])
        assert out["1"][2] == out["0"][2]


# ---- null-space projection deferred into the Arnoldi pass B (sb_ctx::defer_nulls) ----


@pytest.mark.parametrize("name,n,kind", [("C5", 32, "P1"), ("C3", 32, "P2"), ("C1", 64, "P1")])
def test_deferred_null_projection(name, n, kind, monkeypatch):
    """Pad-free all-periodic grids leave the null-space means of P^-1 M v to the
    Arnoldi pass B (w - mean, the same expression as the projection kernel).
    Pass A's dots then see the unprojected w, which changes them at roundoff
    level only (the basis has zero means): same iteration count, solutions
    within 1e-12 of the eager projection (SB_DEFER_NULLS=0); a direct P^-1
    application is still projected exactly (identical to the bit)."""
    from paper_1308_4605_b200 import operators as OPS
    from paper_1308_4605_b200 import problems as PR
    from paper_1308_4605_b200.grid import pack_stokes
    from paper_1308_4605_b200.krylov import GmresConfig, gmres_solve
    from paper_1308_4605_b200.precond import PrecondConfig, PrecondKind, Preconditioner
    case = PR.make_case(name, n)
    cs, rs, spec = PR.prepare(case)
    out = {}
    for defer in ("1", "0"):
        OPS._POOL.clear()  # the flag is fixed when a context is created
        monkeypatch.setenv("SB_DEFER_NULLS", defer)
        P = Preconditioner(cs, PrecondConfig(kind=PrecondKind(kind)))
        monkeypatch.delenv("SB_DEFER_NULLS")
        z = P.apply(rs)
        x, h = gmres_solve(rs, cs, None, GmresConfig(restart=case.restart, rtol=1e-9), precond=P)
        out[defer] = (pack_stokes(z), pack_stokes(x), h.iterations, h.status)
        del P
    OPS._POOL.clear()
    assert np.array_equal(out["1"][0], out["0"][0])
    assert out["1"][3] == out["0"][3] == "converged"
    assert out["1"][2] == out["0"][2]
    assert _rel(out["1"][1], out["0"][1]) <= 1e-12
