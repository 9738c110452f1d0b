"""The reference's remaining public names on the device (VERDICT r1 "What's
missing" #4): div / grad / lap_pressure / apply_viscous (operators.py:182-203,
:303-345), helmholtz_diagonal / lrho_diagonal (:396-439), restrict_* /
prolong_* / coarsen_coefficients / smooth_* (multigrid.py:127-340),
apply_schur_inv (schur.py:59-78) and gmres_kernel (krylov.py:81-146), against
the reference's golden vectors and the pinned oracle; and the reference's own
test modules run against the package (tools/ref_shim.py).
"""

from __future__ import annotations

import pathlib
import subprocess
import sys

import numpy as np
import pytest

from conftest import ROOT, arr, cases, face, oracle_coef, oracle_geo, pkg_coeff, pkg_grid, relerr

pytestmark = pytest.mark.gpu

OPS = cases("operators")


def _rand_face(g, rng, boundary=True):
    from paper_1308_4605_b200.grid import FaceField
    u = FaceField.zeros(g)
    for a in range(g.dim):
        if boundary:
            u.components[a][...] = rng.standard_normal(u.components[a].shape)
        else:
            u.interior(a)[...] = rng.standard_normal(u.interior(a).shape)
    return u


@pytest.mark.parametrize("e", OPS[::3], ids=lambda e: e["name"])
def test_div_grad_lap_bit_exact(e):
    """div reads the stored boundary faces; grad zeroes wall-normal faces;
    lap_pressure = div(grad): bit-identical to the reference's NumPy arithmetic
    (the oracle restates it op for op)."""
    from oracle import stokes_oracle as O
    from paper_1308_4605_b200 import operators as OPS_
    from paper_1308_4605_b200.grid import CellField
    g, geo = pkg_grid(e), oracle_geo(e)
    rng = np.random.default_rng(7)
    u = _rand_face(g, rng)
    p = CellField(g, rng.standard_normal(g.cells))
    assert np.array_equal(OPS_.div(u).data, O.div(geo, list(u.components)))
    gp = OPS_.grad(p)
    want = O.grad(geo, p.data)
    for a in range(g.dim):
        assert np.array_equal(gp.components[a], want[a]), a
    assert np.array_equal(OPS_.lap_pressure(p).data, O.div(geo, O.grad(geo, p.data)))


@pytest.mark.parametrize("e", OPS, ids=lambda e: e["name"])
def test_transfers_and_coarsening_bit_exact(e):
    """restrict_* / prolong_* / coarsen_coefficients with the reference
    signatures equal the reference's outputs (golden rf / rc / pf / pc and the
    coarse coefficient sets) to the bit."""
    from paper_1308_4605_b200 import multigrid as MG
    from paper_1308_4605_b200.grid import CellField, FaceField
    n = e["name"]
    g = pkg_grid(e)
    d = g.dim
    rf = MG.restrict_face(FaceField(g, tuple(face(n, "u", d))))
    for a in range(d):
        assert np.array_equal(rf.components[a], arr(n, f"rf{a}")), a
    assert np.array_equal(MG.restrict_cell(CellField(g, arr(n, "p"))).data, arr(n, "rc"))
    gc = g.coarsened()
    pf = MG.prolong_face(FaceField(gc, tuple(face(n, "pin", d))))
    for a in range(d):
        assert np.array_equal(pf.components[a], arr(n, f"pf{a}")), a
    assert np.array_equal(MG.prolong_cell(CellField(gc, arr(n, "pinc"))).data, arr(n, "pc"))
    cc = MG.coarsen_coefficients(pkg_coeff(e, grid=g), gc)
    want = pkg_coeff(e, prefix=n + "/coarse", grid=gc)
    assert np.array_equal(cc.mu_cell.data, want.mu_cell.data)
    assert np.array_equal(cc.gamma_cell.data, want.gamma_cell.data)
    assert np.array_equal(cc.rho_cell.data, want.rho_cell.data)
    for a in range(d):
        assert np.array_equal(cc.rho_face.components[a], want.rho_face.components[a])
    for k, v in want.mu_node_edge.arrays.items():
        assert np.array_equal(cc.mu_node_edge.arrays[k], v), k


@pytest.mark.parametrize("e", OPS, ids=lambda e: e["name"])
def test_diagonals_viscous_and_smoothers(e):
    from paper_1308_4605_b200 import multigrid as MG
    from paper_1308_4605_b200 import operators as OPS_
    from paper_1308_4605_b200.grid import CellField, FaceField
    n = e["name"]
    g = pkg_grid(e)
    d = g.dim
    c = pkg_coeff(e, grid=g)
    hd = OPS_.helmholtz_diagonal(g, c)
    for a in range(d):
        assert relerr(hd.components[a], arr(n, f"diagf{a}")) <= 1e-13, a
    assert relerr(OPS_.lrho_diagonal(g, c).data, arr(n, "diagc")) <= 1e-13
    # L_mu u = theta rho u - A u, from the golden M u = A u + G p
    from oracle import stokes_oracle as O
    geo = oracle_geo(e)
    u = FaceField(g, tuple(face(n, "u", d)))
    gp = O.grad(geo, arr(n, "p"))
    lv = OPS_.apply_viscous(u, c)
    for a in range(d):
        au = arr(n, f"Mu{a}") - gp[a]
        want = c.theta * c.rho_face.components[a] * u.components[a] - au
        if not g.periodic(a):
            want[(slice(None),) * a + (0,)] = 0.0
            want[(slice(None),) * a + (-1,)] = 0.0
        assert relerr(lv.components[a], want) <= 1e-11, a
    # in-place reference-signature smoothers (golden sx1 / cy1, omega 0.8)
    x = FaceField(g, tuple(face(n, "sx0", d)))
    MG.smooth_face(x, FaceField(g, tuple(face(n, "srhs", d))), g, c, hd, 0.8)
    for a in range(d):
        assert relerr(x.components[a], arr(n, f"sx1{a}")) <= 1e-12, a
    y = CellField(g, arr(n, "cy0"))
    MG.smooth_cell(y, CellField(g, arr(n, "cyrhs")), g, c, OPS_.lrho_diagonal(g, c), 0.8)
    assert relerr(y.data, arr(n, "cy1")) <= 1e-12


@pytest.mark.parametrize("e", OPS[::2], ids=lambda e: e["name"])
def test_apply_schur_inv(e):
    """-theta phi + V r with the caller's pressure solve (schur.py:59-78);
    steady sets never call it; unsteady without one is a ValueError."""
    from paper_1308_4605_b200.grid import CellField
    from paper_1308_4605_b200.schur import SchurConfig, apply_schur_inv, schur_diagonal
    g = pkg_grid(e)
    c = pkg_coeff(e, grid=g)
    rng = np.random.default_rng(3)
    r = CellField(g, rng.standard_normal(g.cells))
    phi = CellField(g, rng.standard_normal(g.cells))
    calls = []

    def solve(x):
        calls.append(1)
        return phi

    out = apply_schur_inv(r, c, SchurConfig(), pressure_solve=solve)
    if c.theta > 0:
        want = -c.theta * phi.data + schur_diagonal(c) * r.data
        assert calls
        with pytest.raises(ValueError):
            apply_schur_inv(r, c, SchurConfig())
    else:
        want = schur_diagonal(c) * r.data
        assert not calls
    assert np.array_equal(out.data, want)


def test_gmres_kernel_known_answers():
    """Flat-vector GMRES with a host operator (krylov.py:81-146): the reference's
    hand-solved 2x2 (tests/test_krylov.py:38-53) and a random nonsymmetric
    system against the oracle's restatement (status, iterations, x, r_P)."""
    from oracle import stokes_oracle as O
    from paper_1308_4605_b200.krylov import gmres_kernel
    A = np.diag([2.0, 5.0])
    b = np.array([2.0, 10.0])
    seen = []
    x, status, k = gmres_kernel(lambda v: A @ v, b, 5, 10, 1e-13 * 10.4, 0.0,
                                lambda k, xk, rp, rf: seen.append((k, rp)))
    assert status in ("converged", "breakdown") and k <= 2
    assert np.allclose(x, [1.0, 2.0], atol=1e-12)
    assert seen[0][1] == pytest.approx(2.0 * np.sqrt(141525.0) / 629.0, rel=1e-12)
    rng = np.random.default_rng(11)
    n = 61
    M = np.eye(n) * 4 + rng.standard_normal((n, n)) / np.sqrt(n)
    b = rng.standard_normal(n)
    for restart, max_iters, tgt in ((8, 200, 1e-10), (5, 12, 1e-12), (40, 200, 1e-13)):
        got_rows, ref_rows = [], []
        xg, sg, kg = gmres_kernel(lambda v: M @ v, b, restart, max_iters, tgt * np.linalg.norm(b), 1e-14,
                                  lambda k, xk, rp, rf: got_rows.append((k, rp, rf)))
        xr, sr, kr = O.gmres_flat(lambda v: M @ v, b, restart, max_iters, tgt * np.linalg.norm(b), 1e-14,
                                  lambda k, xk, rp, rf: ref_rows.append((k, rp, rf)))
        assert sg == sr and kg == kr, (restart, sg, sr, kg, kr)
        kk = min(len(got_rows), len(ref_rows))
        assert [r[2] for r in got_rows[:kk]] == [r[2] for r in ref_rows[:kk]]
        rp_g, rp_r = np.array([r[1] for r in got_rows[:kk]]), np.array([r[1] for r in ref_rows[:kk]])
        big = rp_r > 1e-10 * np.linalg.norm(b)  # roundoff-level residuals are not comparable
        assert np.allclose(rp_g[big], rp_r[big], rtol=1e-6)
        assert np.linalg.norm(xg - xr) <= 1e-8 * np.linalg.norm(xr)
    # Krylov space exhausted at k = n with an unreachable target: the device's
    # CGS2 breaks down at k <= n (MGS, having lost orthogonality, may run past n)
    xg, sg, kg = gmres_kernel(lambda v: M @ v, b, 70, 200, 1e-300, 1e-14 * np.linalg.norm(b))
    assert sg == "breakdown" and kg <= n
    assert np.linalg.norm(M @ xg - b) <= 1e-12 * np.linalg.norm(b)


def test_reference_test_modules_against_the_package():
    """The reference's own test modules (test_multigrid / precond / schur /
    operators / krylov / grid / problems / spectrum / acceptance / cli),
    unmodified, with ``stokesmg`` resolving to this package (tools/ref_shim.py; staged under
    baseline/_ref_tests, git-ignored like the baseline/_ref install)."""
    stage = ROOT / "baseline" / "_ref_tests"
    if not (stage / "test_cli.py").exists():
        pytest.skip("reference tests not staged (python tools/ref_shim.py stage)")
    out = subprocess.run([sys.executable, str(ROOT / "tools" / "ref_shim.py"), "run", "-q", "-x"],
                         capture_output=True, text=True, timeout=1800, cwd=str(ROOT))
    log = ROOT / "gpurun_out" / "ref_shim.log"
    log.parent.mkdir(exist_ok=True)
    log.write_text(out.stdout + out.stderr)
    assert out.returncode == 0, out.stdout[-4000:] + out.stderr[-2000:]


def test_non_contiguous_inputs():
    """Arrays that are views (np.real of a complex field, strided slices) are
    copied to contiguous temporaries at the boundary; the temporaries must
    outlive the C call (a reference test's Fourier-mode inputs exposed a
    use-after-free here).  Results equal those of contiguous copies."""
    from paper_1308_4605_b200 import operators as OPS_
    from paper_1308_4605_b200.grid import PERIODIC, CellField, FaceField, GridSpec, StokesVector
    from paper_1308_4605_b200.operators import make_coefficients
    g = GridSpec((8, 8, 8), 0.5, ((PERIODIC, PERIODIC),) * 3)
    rng = np.random.default_rng(5)
    c = make_coefficients(g, 0.3, CellField(g, 1 + rng.random(g.cells)), CellField(g, 1 + rng.random(g.cells)))
    z = [rng.standard_normal(g.face_shape(a)) + 1j * rng.standard_normal(g.face_shape(a)) for a in range(3)]
    zp = rng.standard_normal(g.cells) + 1j * rng.standard_normal(g.cells)
    views = FaceField(g, tuple(np.real(x) for x in z))
    copies = FaceField(g, tuple(np.ascontiguousarray(np.real(x)) for x in z))
    assert not views.components[0].flags.c_contiguous
    for f in (OPS_.apply_A, OPS_.apply_viscous):
        a, b = f(views, c), f(copies, c)
        for k in range(3):
            assert np.array_equal(a.components[k], b.components[k])
    pv, pc = CellField(g, np.imag(zp)), CellField(g, np.ascontiguousarray(np.imag(zp)))
    m1 = OPS_.apply_M(StokesVector(views, pv), c)
    m2 = OPS_.apply_M(StokesVector(copies, pc), c)
    assert np.array_equal(m1.p.data, m2.p.data)
    assert np.array_equal(OPS_.div(views).data, OPS_.div(copies).data)
    assert np.array_equal(OPS_.lap_pressure(pv).data, OPS_.lap_pressure(pc).data)
