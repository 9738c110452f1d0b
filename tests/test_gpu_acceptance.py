"""The reference's acceptance criteria that exercise the hot path
(reference tests/test_acceptance.py), run on the device path:
multigrid rate (2), bubble benchmark (6), preconditioner cost ordering (7),
Schur sign (8), grid robustness (9), viscous-CFL sweep monotonicity (10).
Thresholds are the reference's."""

from __future__ import annotations

import functools
import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _grid(n, dim):
    from paper_1308_4605_b200.grid import NO_SLIP, GridSpec
    return GridSpec((n,) * dim, 1.0, ((NO_SLIP, NO_SLIP),) * dim)


@functools.lru_cache(maxsize=None)
def bubble_solve(n, dim, kind, sign="minus", beta=math.inf, contrast=100.0, max_iters=100, rtol=1e-12):
    from paper_1308_4605_b200 import problems as PR
    from paper_1308_4605_b200.krylov import GmresConfig, gmres_solve
    from paper_1308_4605_b200.operators import rescale
    from paper_1308_4605_b200.precond import PrecondConfig, PrecondKind
    from paper_1308_4605_b200.schur import SchurConfig, SchurSign
    g = _grid(n, dim)
    cfl = PR.CflSpec(beta)
    spec = PR.BubbleSpec(r_mu=contrast, r_rho=contrast, seed=0)
    if cfl.inviscid:
        coeff = PR.inviscid_coefficients(g, PR.bubble_density(g, spec), theta=1.0)
    else:
        coeff = PR.bubble_coefficients(g, spec, theta=PR.cfl_to_theta(cfl, 1.0, 1.0, g.h))
    rhs, _ = PR.make_rhs(g, coeff, seed=1)
    coeff, rhs, _ = rescale(coeff, rhs)
    pc = PrecondConfig(kind=PrecondKind(kind), schur=SchurConfig(sign=SchurSign(sign)))
    _, hist = gmres_solve(rhs, coeff, pc, GmresConfig(restart=10, rtol=rtol, max_iters=max_iters))
    return hist


def first_reaching(hist, tol):
    r0 = hist.entries[0].resid_true
    for e in hist.entries:
        if e.resid_true <= tol * r0:
            return e.iteration, e.scalar_vcycles
    return None, None


def no_stall(hist):
    """r_P decreases over every restart window (reference test_acceptance.py:260-270)."""
    windows, cur = [], []
    for e in hist.entries[1:]:
        if e.restart and cur:
            windows.append(cur)
            cur = []
        cur.append(e.resid_precond)
    if cur:
        windows.append(cur)
    return all(w[-1] < w[0] for w in windows if len(w) > 1)


def test_criterion_2_multigrid_rate():
    from paper_1308_4605_b200 import multigrid as MG
    from paper_1308_4605_b200.grid import CellField, norm2
    from paper_1308_4605_b200.operators import apply_Lrho, _ctx_for
    from paper_1308_4605_b200.problems import constant_coefficients
    rng = np.random.default_rng(20240817)
    for dim, n in ((2, 256), (3, 48)):
        g = _grid(n, dim)
        coeff = constant_coefficients(g, theta=1.0)
        hier = MG.build_hierarchy(g, coeff)
        ctx = _ctx_for(coeff, g)
        rhs = CellField(g, rng.standard_normal(g.cells))
        rhs.data -= rhs.data.mean()
        x = CellField.zeros(g)
        r0 = prev = norm2(rhs)
        ratios, reached = [], None
        for cycle in range(1, 16):
            res = CellField(g, rhs.data - apply_Lrho(x, coeff, ctx=ctx).data)
            x.data += MG.vcycle(res, hier, MG.SmootherParams(), "cell").data
            rn = norm2(CellField(g, rhs.data - apply_Lrho(x, coeff, ctx=ctx).data))
            ratios.append(rn / prev)
            prev = rn
            if rn / r0 <= 1e-10:
                reached = cycle
                break
        assert reached is not None and all(r <= 0.2 for r in ratios[2:]), (dim, n, ratios)


def test_criterion_6_bubble_benchmark():
    h2 = bubble_solve(128, 2, "P2", max_iters=100)
    it2, _ = first_reaching(h2, 1e-10)
    assert it2 is not None and it2 <= 100 and no_stall(h2)
    h3 = bubble_solve(48, 3, "P2", max_iters=120)
    it3, _ = first_reaching(h3, 1e-10)
    assert it3 is not None and it3 <= 120 and no_stall(h3)


def test_criterion_7_preconditioner_ordering():
    cost = {}
    for kind, iters in (("P1", 100), ("P2", 100), ("P4", 300), ("P5", 200)):
        _, cyc = first_reaching(bubble_solve(128, 2, kind, max_iters=iters), 1e-9)
        cost[kind] = cyc
    assert cost["P2"] is not None and cost["P2"] <= cost["P1"]
    assert cost["P2"] < cost["P4"] and cost["P2"] < cost["P5"], cost


def test_criterion_8_schur_sign():
    im, _ = first_reaching(bubble_solve(128, 2, "P2", sign="minus", max_iters=100), 1e-9)
    ip, _ = first_reaching(bubble_solve(128, 2, "P2", sign="plus", max_iters=300), 1e-9)
    assert im is not None and ip is not None and im < ip


def test_criterion_9_grid_robustness():
    for kind in ("P1", "P2"):
        i_small, _ = first_reaching(bubble_solve(64, 2, kind, contrast=2.0, max_iters=100), 1e-9)
        i_large, _ = first_reaching(bubble_solve(256, 2, kind, contrast=2.0, max_iters=100), 1e-9)
        assert i_small is not None and i_large is not None and i_large <= 1.5 * i_small, (kind, i_small, i_large)


def test_criterion_10_cfl_sweep():
    for kind in ("P1", "P2"):
        iters = [first_reaching(bubble_solve(64, 2, kind, beta=b, max_iters=150), 1e-9)[0]
                 for b in (0.0, 1.0, 1e4, math.inf)]
        assert all(i is not None for i in iters) and all(a <= b for a, b in zip(iters, iters[1:])), (kind, iters)
