"""GMRES exit paths other than convergence, and the smoother's zero-diagonal
error, against the reference (tests/golden/make_golden_exit.py).

* ``breakdown`` (krylov.py:138): a 4x4 problem whose Krylov space is exhausted
  after 40 Arnoldi steps -- the device must see the Arnoldi norm collapse
  (the direct subdiagonal norm near breakdown, not sqrt(||w'||^2 - ||c'||^2));
* ``maxiter`` (krylov.py:142-145): GMRES(3) capped at 7 iterations, restart
  flags on iterations 4 and 7 (krylov.py:135), 2D and 3D;
* ``ZeroDivisionError`` on a zero smoother diagonal (multigrid.py:74-75, 84-88;
  reference tests/test_multigrid.py:75-83).

The oracle is checked here on CPU; the device (C ABI) under ``-m gpu``.
"""

from __future__ import annotations

import json

import numpy as np
import pytest

from conftest import GOLD, planes

_z = {}


def _gold():
    if not _z:
        _z["z"] = np.load(GOLD / "golden_exit.npz")
        _z["idx"] = json.loads((GOLD / "golden_exit.json").read_text())
    return _z["z"], _z["idx"]


def _arr(name, key):
    return np.array(_gold()[0][f"{name}/{key}"])


CASES = [e["name"] for e in json.loads((GOLD / "golden_exit.json").read_text())]


def _entry(name):
    return next(e for e in _gold()[1] if e["name"] == name)


def _pkg(e):
    from conftest import BCNAME
    from paper_1308_4605_b200.grid import (BoundaryCondition, CellField, FaceField, GridSpec, NodeEdgeField,
                                           StokesVector)
    from paper_1308_4605_b200.operators import CoefficientSet, ViscousForm
    g = GridSpec(tuple(e["cells"]), float(e["h"]),
                 tuple((BoundaryCondition(BCNAME[b[0]]), BoundaryCondition(BCNAME[b[1]])) for b in e["bc"]))
    n, d = e["name"], g.dim
    cs = CoefficientSet(
        theta=float(e["theta"]), rho_cell=CellField(g, _arr(n, "rho_cell")),
        rho_face=FaceField(g, tuple(_arr(n, f"rho_face{a}") for a in range(d))),
        mu_cell=CellField(g, _arr(n, "mu_cell")),
        mu_node_edge=NodeEdgeField(g, {pl: _arr(n, f"mu_edge{pl[0]}{pl[1]}") for pl in planes(d)}),
        gamma_cell=CellField(g, _arr(n, "gamma_cell")), viscous_form=ViscousForm(e["form"]))
    rs = StokesVector(FaceField(g, tuple(_arr(n, f"bu{a}") for a in range(d))), CellField(g, _arr(n, "bp")))
    return g, cs, rs


def _check_history(e, rows, status, iterations, its_tol):
    ref = _arr(e["name"], "hist")
    assert status == e["status"]
    assert abs(iterations - e["iterations"]) <= its_tol
    got = np.array(rows, dtype=float)
    k = min(len(got), len(ref))
    # iteration numbers, V-cycle counters and restart flags row by row
    assert np.array_equal(got[:k][:, [0, 1, 4]], ref[:k][:, [0, 1, 4]])
    return got, ref, k


@pytest.mark.parametrize("name", CASES)
def test_oracle_exit_paths(name):
    from conftest import BCNAME
    from oracle import stokes_oracle as O
    e = _entry(name)
    d = len(e["cells"])
    geo = O.Geo(tuple(e["cells"]), float(e["h"]), tuple((BCNAME[b[0]], BCNAME[b[1]]) for b in e["bc"]))
    n = e["name"]
    c = O.Coef(float(e["theta"]), _arr(n, "rho_cell"), [_arr(n, f"rho_face{a}") for a in range(d)],
               _arr(n, "mu_cell"), {pl: _arr(n, f"mu_edge{pl[0]}{pl[1]}") for pl in planes(d)},
               _arr(n, "gamma_cell"), e["form"])
    u, p, hist = O.gmres_solve(geo, c, [_arr(n, f"bu{a}") for a in range(d)], _arr(n, "bp"),
                               O.PrecondOpts(kind=e["precond"]),
                               O.GmresOpts(restart=e["restart"], max_iters=e["max_iters"], rtol=e["rtol"],
                                           track_true_residual=True))
    got, ref, k = _check_history(e, hist.rows, hist.status, hist.iterations, 0)
    assert got.shape == ref.shape
    if e["status"] == "maxiter":
        assert np.allclose(got[:, 2], ref[:, 2], rtol=1e-9)
    xo = O.pack(geo, u, p)
    xr = O.pack(geo, [_arr(n, f"xu{a}") for a in range(d)], _arr(n, "xp"))
    assert np.linalg.norm(xo - xr) <= 1e-10 * np.linalg.norm(xr)


@pytest.mark.gpu
@pytest.mark.parametrize("name", CASES)
def test_device_exit_paths(name):
    """Device status / iterations / restart flags / r_P / x against the reference."""
    from paper_1308_4605_b200.grid import pack_stokes
    from paper_1308_4605_b200.krylov import GmresConfig, gmres_solve
    from paper_1308_4605_b200.precond import PrecondConfig, PrecondKind
    e = _entry(name)
    g, cs, rs = _pkg(e)
    gcfg = GmresConfig(restart=e["restart"], max_iters=e["max_iters"], rtol=e["rtol"], atol=0.0,
                       track_true_residual=True)
    x, hist = gmres_solve(rs, cs, PrecondConfig(kind=PrecondKind(e["precond"])), gcfg)
    got, ref, k = _check_history(e, hist.rows(), hist.status, hist.iterations,
                                 e.get("its_tol", 1 if e["status"] == "breakdown" else 0))
    if e["status"] == "maxiter":
        assert got.shape == ref.shape
        assert np.allclose(got[:, 2], ref[:, 2], rtol=1e-6)
        assert np.allclose(got[:, 3], ref[:, 3], rtol=1e-5)
    from paper_1308_4605_b200.grid import CellField, FaceField, StokesVector
    xr = pack_stokes(StokesVector(FaceField(g, tuple(_arr(name, f"xu{a}") for a in range(g.dim))),
                                  CellField(g, _arr(name, "xp"))))
    if e.get("its_tol", 0) > 1:  # roundoff-determined stop: compare through the residual
        k = min(len(got), len(ref)) - 3
        assert np.allclose(got[:k, 2], ref[:k, 2], rtol=1e-6, atol=1e-12 * ref[0, 2])
        assert got[-1, 3] <= 1e-10 * ref[0, 3]
        return
    assert np.linalg.norm(pack_stokes(x) - xr) <= 1e-8 * np.linalg.norm(xr)


@pytest.mark.gpu
@pytest.mark.parametrize("dim", [2, 3])
def test_device_zero_diagonal_raises(dim):
    """A steady region of zero viscosity (reference tests/test_multigrid.py:75-83)
    makes the velocity smoother's diagonal vanish: ZeroDivisionError, as the
    reference's lazily built diagonal raises on the first V-cycle."""
    from paper_1308_4605_b200.grid import NO_SLIP, CellField, GridSpec, StokesVector, FaceField
    from paper_1308_4605_b200.krylov import GmresConfig, gmres_solve
    from paper_1308_4605_b200.multigrid import build_hierarchy, SmootherParams, vcycle
    from paper_1308_4605_b200.operators import make_coefficients
    from paper_1308_4605_b200.precond import P1, PrecondConfig
    cells = (8,) * dim
    g = GridSpec(cells, 1 / 8, ((NO_SLIP, NO_SLIP),) * dim)
    mu = np.zeros(cells)
    mu[(0,) * dim] = 1.0
    coeff = make_coefficients(g, 0.0, CellField(g, np.ones(cells)), CellField(g, mu))
    rhs = StokesVector(FaceField.zeros(g), CellField(g, np.zeros(cells)))
    rhs.u.interior(0)[...] = 1.0
    with pytest.raises(ZeroDivisionError):
        gmres_solve(rhs, coeff, PrecondConfig(kind=P1), GmresConfig(restart=5, max_iters=5))
    hier = build_hierarchy(g, coeff)
    with pytest.raises(ZeroDivisionError):
        vcycle(rhs.u, hier, SmootherParams(), "face")


@pytest.mark.gpu
def test_large_restart_matches_oracle():
    """GmresConfig.restart has no upper bound in the reference (krylov.py:23-38).
    Beyond 127 basis vectors the device takes the chunked CGS2 step
    (launch_cgs2): a slowly converging flat system that needs > 240 Arnoldi
    vectors in one cycle (two full chunks and a remainder), against the
    oracle's restatement; and a Stokes solve (C4 recipe at 16^3, 99 iterations
    unrestarted) with restart 160 -- the large-restart path -- against the
    default path with restart 110: neither restarts, same Krylov space."""
    from oracle import stokes_oracle as O
    from paper_1308_4605_b200 import problems as PR
    from paper_1308_4605_b200.grid import pack_stokes
    from paper_1308_4605_b200.krylov import GmresConfig, gmres_kernel, gmres_solve
    from paper_1308_4605_b200.precond import P1, PrecondConfig
    rng = np.random.default_rng(3)
    n = 800
    M = np.eye(n) + 0.99 * rng.standard_normal((n, n)) / np.sqrt(n)
    b = rng.standard_normal(n)
    tgt = 1e-11 * np.linalg.norm(b)
    rows_g, rows_r = [], []
    xg, sg, kg = gmres_kernel(lambda v: M @ v, b, 300, 900, tgt, 1e-14, lambda k, xk, rp, rf: rows_g.append((k, rp, rf)))
    xr, sr, kr = O.gmres_flat(lambda v: M @ v, b, 300, 900, tgt, 1e-14, lambda k, xk, rp, rf: rows_r.append((k, rp, rf)))
    assert kr > 241, kr  # the case exercises three chunks (120 + 120 + remainder)
    assert sg == sr and abs(kg - kr) <= 1
    kk = min(len(rows_g), len(rows_r))
    rp_g, rp_r = np.array([r[1] for r in rows_g[:kk]]), np.array([r[1] for r in rows_r[:kk]])
    keep = rp_r > 1e-9 * np.linalg.norm(b)
    assert np.allclose(rp_g[keep], rp_r[keep], rtol=1e-6)
    assert np.linalg.norm(xg - xr) <= 1e-8 * np.linalg.norm(xr)
    assert np.linalg.norm(M @ xg - b) <= 1e-10 * np.linalg.norm(b)

    case = PR.make_case("C4", 16)
    cs, rs, _ = PR.prepare(case)
    res = {}
    for m in (110, 160):
        x, h = gmres_solve(rs, cs, PrecondConfig(kind=P1),
                           GmresConfig(restart=m, max_iters=400, rtol=1e-9, track_true_residual=True))
        res[m] = (pack_stokes(x), h)
    ha, hb = res[110][1], res[160][1]
    assert ha.status == hb.status == "converged"
    assert hb.iterations == ha.iterations
    ra = np.array([e.resid_precond for e in ha.entries])
    rb = np.array([e.resid_precond for e in hb.entries])
    assert np.allclose(ra, rb, rtol=1e-6)
    assert ha.iterations == 99
    assert np.linalg.norm(res[110][0] - res[160][0]) <= 1e-8 * np.linalg.norm(res[110][0])
