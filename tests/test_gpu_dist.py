"""Slab-decomposed path on ONE GPU: nslab slabs in one process (exchanges are
device copies, no waiting kernels) vs the single-domain device solve and the
oracle.  Same colour order, same algorithm; only reduction order differs."""

from __future__ import annotations

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _case(name, n):
    from paper_1308_4605_b200 import problems as PR
    case = PR.make_case(name, n)
    cs, rs, spec = PR.prepare(case)
    return case, cs, rs


@pytest.mark.parametrize("name,n,nslab", [("C5", 32, 2), ("C5", 64, 4), ("C3", 64, 8), ("C4", 32, 2),
                                          ("C4", 64, 4)])
def test_dist_operator_and_precond_match_single(name, n, nslab):
    from paper_1308_4605_b200.dist import DistSolver
    from paper_1308_4605_b200.operators import apply_M
    from paper_1308_4605_b200.precond import P1, PrecondConfig, Preconditioner
    case, cs, rs = _case(name, n)
    D = DistSolver(case.grid, cs.viscous_form, nslab=nslab)
    D.set_coefficients(cs)
    info = D.info()
    assert info["slabs"] == nslab and info["distributed_levels"] >= 1
    mu, mp = D.apply_M(rs)
    ref = apply_M(rs, cs)
    for a in range(3):
        assert np.allclose(mu[a], ref.u.components[a], rtol=0, atol=1e-12 * np.abs(ref.u.components[a]).max())
    assert np.allclose(mp, ref.p.data, rtol=0, atol=1e-12 * np.abs(ref.p.data).max())
    P = Preconditioner(cs, PrecondConfig(kind=P1))
    want = P.apply(rs)
    xu, xp = D.precond_apply(rs, PrecondConfig(kind=P1))
    for a in range(3):
        s = np.abs(want.u.components[a]).max()
        assert np.abs(xu[a] - want.u.components[a]).max() <= 1e-11 * s, a
    assert np.abs(xp - want.p.data).max() <= 1e-11 * np.abs(want.p.data).max()


@pytest.mark.parametrize("name,n,nslab,kind", [("C5", 32, 2, "P1"), ("C5", 64, 4, "P1"), ("C4", 32, 2, "P1"),
                                               ("C3", 64, 4, "P2")])
def test_dist_gmres_matches_single_and_oracle(name, n, nslab, kind):
    from paper_1308_4605_b200.dist import DistSolver
    from paper_1308_4605_b200.grid import pack_stokes, StokesVector, FaceField, CellField
    from paper_1308_4605_b200.krylov import GmresConfig, gmres_solve
    from paper_1308_4605_b200.precond import PrecondConfig, PrecondKind
    case, cs, rs = _case(name, n)
    gcfg = GmresConfig(restart=case.restart, max_iters=500, rtol=1e-9, track_true_residual=False)
    pc = PrecondConfig(kind=PrecondKind(kind))
    x1, h1 = gmres_solve(rs, cs, pc, gcfg)
    D = DistSolver(case.grid, cs.viscous_form, nslab=nslab)
    D.set_coefficients(cs)
    xu, xp, h2 = D.gmres_solve(rs, pc, gcfg)
    assert h2.status == h1.status == "converged"
    assert abs(h2.iterations - h1.iterations) <= 1
    g = case.grid
    x2 = StokesVector(FaceField(g, tuple(xu)), CellField(g, xp))
    a, b = pack_stokes(x2), pack_stokes(x1)
    assert np.linalg.norm(a - b) <= 1e-8 * np.linalg.norm(b)
    r1 = np.array(h1.rows())[:, 2]
    r2 = np.array(h2.rows())[:, 2]
    k = min(len(r1), len(r2))
    assert np.allclose(r1[:k], r2[:k], rtol=1e-6)
