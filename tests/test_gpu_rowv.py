"""Row-vector kernels (sb_rowv.cu) vs the one-face-per-thread kernels.

On all-periodic 3D levels whose contiguous extent is a multiple of 64 the face
residual field and apply_M (and, opt-in, the colour passes) run as row-vector kernels
(a warp per row segment, operand rows loaded once, +-1 neighbours by warp
shuffle).  Same operands, same arithmetic order: the results must be
bit-identical to the per-face kernels (SB_ROWV=0), with stored and with derived
edge viscosities, for both viscous forms the kernels cover, at segment
boundaries and periodic wraps (odd row counts, extents 64 and 128).

On levels with derived edge viscosities the default is the row-march kernel
(k_face_all_rm, SB_ROWM=1: a warp walks a whole row, every edge / normal stress
evaluated once and shared by the two rows that use it, FMAs): the same formulas
in a different rounding order, so it is compared to the per-face kernels at
1e-13 of the field's magnitude (north_star asks 1e-8), and full solves by
iteration count, r_P history and solution.
"""

from __future__ import annotations

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

GRIDS = [(64, 64, 64), (6, 10, 128), (4, 6, 64)]


def _case(cells, form, derive, theta, monkeypatch):
    from dataclasses import replace
    from paper_1308_4605_b200 import problems as PR
    from paper_1308_4605_b200.operators import ViscousForm
    case = PR.make_case("C5", cells)
    cs, rs, spec = PR.prepare(case)
    cs = replace(cs, viscous_form=ViscousForm(form), theta=theta)
    monkeypatch.setenv("SB_MUE_DERIVED", "1" if derive else "0")
    return case, cs, rs


def _run(cells, form, derive, theta, rowv, monkeypatch, rowm="0"):
    from paper_1308_4605_b200 import multigrid as MG
    from paper_1308_4605_b200 import operators as OPS
    from paper_1308_4605_b200.grid import FaceField
    case, cs, rs = _case(cells, form, derive, theta, monkeypatch)
    g = case.grid
    monkeypatch.setenv("SB_ROWV", "1" if rowv else "0")
    monkeypatch.setenv("SB_ROWM", rowm)
    monkeypatch.setenv("SB_ROWV_COLOUR", "1" if rowv else "0")  # opt-in colour pass
    ctx = OPS.DeviceContext(g, cs.viscous_form)
    ctx.set_coefficients(cs)
    assert ctx.mue_derived(0) == derive
    hier = MG.MgHierarchy(ctx, cs)
    rng = np.random.default_rng(7)
    x = FaceField(g, tuple(rng.standard_normal(g.face_shape(a)) for a in range(3)))
    out = {}
    m = OPS.apply_M(rs, cs, ctx=ctx)
    out["Mu"] = [c.copy() for c in m.u.components] + [m.p.data.copy()]
    for omega in (1.0, 0.8):
        y = MG.smooth(hier, 0, "face", x, rs.u, omega)
        out[f"sm{omega}"] = [c.copy() for c in y.components]
    if all(c % 2 == 0 and c >= 4 for c in cells):
        rr = MG.residual_restrict(hier, 0, "face", x, rs.u)
        out["rr"] = [c.copy() for c in rr.components]
    ctx.close()
    monkeypatch.delenv("SB_ROWV")
    monkeypatch.delenv("SB_ROWM")
    monkeypatch.delenv("SB_ROWV_COLOUR")
    return out


@pytest.mark.parametrize("cells", GRIDS, ids=lambda c: "x".join(map(str, c)))
@pytest.mark.parametrize("form,derive,theta", [("stress", True, 0.0), ("stress", False, 0.0),
                                               ("laplacian", True, 0.0), ("stress", True, 3.5)])
def test_rowv_bit_identical(cells, form, derive, theta, monkeypatch):
    a = _run(cells, form, derive, theta, True, monkeypatch)
    b = _run(cells, form, derive, theta, False, monkeypatch)
    assert a.keys() == b.keys()
    for k in a:
        for u, v in zip(a[k], b[k]):
            assert np.array_equal(u, v), k


@pytest.mark.parametrize("cells", GRIDS + [(8, 8, 256), (2, 4, 512)], ids=lambda c: "x".join(map(str, c)))
@pytest.mark.parametrize("form,theta", [("stress", 0.0), ("laplacian", 0.0), ("stress", 3.5), ("laplacian", 0.25)])
def test_row_march_matches_per_face(cells, form, theta, monkeypatch):
    a = _run(cells, form, True, theta, True, monkeypatch, rowm="1")
    b = _run(cells, form, True, theta, False, monkeypatch)
    assert a.keys() == b.keys()
    for k in a:
        for u, v in zip(a[k], b[k]):
            assert np.max(np.abs(u - v)) <= 1e-13 * np.max(np.abs(v)), k
    # the colour passes do not use the all-face kernels
    for k in ("sm1.0", "sm0.8"):
        for u, v in zip(a[k], b[k]):
            assert np.array_equal(u, v), k


def test_row_march_gmres_matches_per_face(monkeypatch):
    """C5-recipe solve at 64^3 with the row-march apply_M / residual field
    against the per-face kernels: same iteration count, r_P history to 1e-6,
    solution to 1e-8 (north_star's tolerances)."""
    from paper_1308_4605_b200 import problems as PR
    from paper_1308_4605_b200.grid import pack_stokes
    from paper_1308_4605_b200.krylov import GmresConfig, gmres_solve
    from paper_1308_4605_b200.precond import P1, PrecondConfig, Preconditioner
    case = PR.make_case("C5", 64)
    cs, rs, spec = PR.prepare(case)
    res = {}
    for rowv in ("1", "0"):
        monkeypatch.setenv("SB_ROWV", rowv)
        monkeypatch.setenv("SB_ROWM", "1")
        P = Preconditioner(cs, PrecondConfig(kind=P1))
        P.set_graphs(False)  # drop a graph captured under the other setting
        P.set_graphs(True)
        x, h = gmres_solve(rs, cs, None, GmresConfig(restart=50, rtol=1e-9), precond=P)
        res[rowv] = (pack_stokes(x), h.iterations, np.array([r.resid_precond for r in h.entries]))
        del P
    assert res["1"][1] == res["0"][1]
    assert np.allclose(res["1"][2], res["0"][2], rtol=1e-6)
    assert np.linalg.norm(res["1"][0] - res["0"][0]) <= 1e-8 * np.linalg.norm(res["0"][0])


def test_rowv_gmres_matches_per_face(monkeypatch):
    """Full C5-recipe solves at 64^3 (P^-1 graph captured per context): identical
    iteration counts and solutions to the bit."""
    monkeypatch.setenv("SB_ROWM", "0")
    from paper_1308_4605_b200 import problems as PR
    from paper_1308_4605_b200.grid import pack_stokes
    from paper_1308_4605_b200.krylov import GmresConfig, gmres_solve
    from paper_1308_4605_b200.precond import P1, PrecondConfig, Preconditioner
    case = PR.make_case("C5", 64)
    cs, rs, spec = PR.prepare(case)
    res = {}
    for rowv in ("1", "0"):
        monkeypatch.setenv("SB_ROWV", rowv)
        monkeypatch.setenv("SB_ROWV_COLOUR", rowv)
        P = Preconditioner(cs, PrecondConfig(kind=P1))
        P.set_graphs(False)  # drop a graph captured under the other setting
        P.set_graphs(True)
        x, h = gmres_solve(rs, cs, None, GmresConfig(restart=50, rtol=1e-9), precond=P)
        res[rowv] = (pack_stokes(x), h.iterations, [r.resid_precond for r in h.entries])
        del P
    assert res["1"][1] == res["0"][1]
    assert res["1"][2] == res["0"][2]
    assert np.array_equal(res["1"][0], res["0"][0])


# ---- walls along the contiguous axis (C4's z walls) --------------------------

WALL_GRIDS = [(64, 64, 64), (6, 10, 128), (4, 6, 64), (2, 4, 512)]


def _wall_case(cells, form, theta, bc2):
    """Seeded variable rho / mu on a box periodic in x, y with walls in z."""
    from paper_1308_4605_b200 import grid as G
    from paper_1308_4605_b200.grid import CellField, FaceField, StokesVector
    from paper_1308_4605_b200.operators import ViscousForm, make_coefficients, rescale
    kinds = {"n": G.NO_SLIP, "f": G.FREE_SLIP}
    g = G.GridSpec(cells, 1.0 / cells[2], ((G.PERIODIC, G.PERIODIC), (G.PERIODIC, G.PERIODIC),
                                           (kinds[bc2[0]], kinds[bc2[1]])))
    rng = np.random.default_rng(11)
    rho = CellField(g, 1.0 + 99.0 * rng.random(g.cells))
    mu = CellField(g, 10.0 ** (3.0 * rng.random(g.cells)))
    cs = make_coefficients(g, theta, rho, mu, viscous_form=ViscousForm(form))
    f = FaceField(g, tuple(rng.standard_normal(g.face_shape(a)) for a in range(3)))
    # wall-normal boundary faces carry no unknown
    f.components[2][..., 0] = 0.0
    f.components[2][..., -1] = 0.0
    rs = StokesVector(f, CellField(g, rng.standard_normal(g.cells)))
    cs, rs, _ = rescale(cs, rs)
    return g, cs, rs


def _wall_run(cells, form, theta, bc2, derive, rowv, monkeypatch):
    from paper_1308_4605_b200 import multigrid as MG
    from paper_1308_4605_b200 import operators as OPS
    from paper_1308_4605_b200.grid import FaceField
    g, cs, rs = _wall_case(cells, form, theta, bc2)
    monkeypatch.setenv("SB_ROWV", "1" if rowv else "0")
    monkeypatch.setenv("SB_MUE_DERIVED", "2" if derive else "0")
    ctx = OPS.DeviceContext(g, cs.viscous_form)
    ctx.set_coefficients(cs)
    assert ctx.mue_derived(0) == derive
    hier = MG.MgHierarchy(ctx, cs)
    out = {}
    m = OPS.apply_M(rs, cs, ctx=ctx)
    out["Mu"] = [c.copy() for c in m.u.components] + [m.p.data.copy()]
    rng = np.random.default_rng(5)
    x = FaceField(g, tuple(rng.standard_normal(g.face_shape(a)) for a in range(3)))
    x.components[2][..., 0] = 0.0
    x.components[2][..., -1] = 0.0
    if all(c % 2 == 0 and c >= 4 for c in cells):
        rr = MG.residual_restrict(hier, 0, "face", x, rs.u)
        out["rr"] = [c.copy() for c in rr.components]
    ctx.close()
    monkeypatch.delenv("SB_ROWV")
    monkeypatch.delenv("SB_MUE_DERIVED")
    return out


@pytest.mark.parametrize("cells", WALL_GRIDS, ids=lambda c: "x".join(map(str, c)))
@pytest.mark.parametrize("form,theta,bc2,derive", [
    ("stress", 0.7, "nn", False), ("stress", 0.0, "ff", False), ("laplacian", 0.7, "nf", False),
    ("stress", 0.7, "fn", True), ("laplacian", 0.0, "nn", True)])
def test_row_march_walls_match_per_face(cells, form, theta, bc2, derive, monkeypatch):
    """Walls (no-slip / free-slip, any mix) at both ends of the marched row:
    ghost values behind the low wall, wall-edge stresses at the high wall, the
    wall-normal component's boundary faces left alone.  Against the per-face
    kernels (SB_ROWV=0) at 1e-13 of the field's magnitude."""
    a = _wall_run(cells, form, theta, bc2, derive, True, monkeypatch)
    b = _wall_run(cells, form, theta, bc2, derive, False, monkeypatch)
    assert a.keys() == b.keys()
    for k in a:
        for u, v in zip(a[k], b[k]):
            assert u.shape == v.shape
            assert np.max(np.abs(u - v)) <= 1e-13 * np.max(np.abs(v)), k
