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
    # slab levels take the same specialisations as the single domain: derived
    # edge viscosities on the finest level (all-periodic, or walls along the
    # contiguous axis only: C4), one 1/rho on constant density
    assert info["mue_derived_levels"] & 1
    if name in ("C3", "C5"):
        assert info["const_rho_levels"] & 1
    else:
        assert info["const_rho_levels"] == 0
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
                                               ("C3", 64, 4, "P2"), ("C5", 32, 1, "P1"), ("C4", 32, 1, "P1")])
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


@pytest.mark.parametrize("name,n,nslab", [("C5", 32, 2), ("C4", 32, 4)])
def test_dist_ghost_plane_red_pass_matches_per_pass_exchange(name, n, nslab, monkeypatch):
    """The red pass relaxing the ghost planes (one exchange per component sweep)
    gives the per-colour-pass exchange result: every slab computes exactly the
    ghost values its neighbour computes, so P^-1 is bit-identical."""
    from paper_1308_4605_b200.dist import DistSolver
    from paper_1308_4605_b200.precond import P1, PrecondConfig
    case, cs, rs = _case(name, n)
    out = {}
    for ext in ("1", "0"):
        monkeypatch.setenv("SB_DIST_EXT", ext)
        D = DistSolver(case.grid, cs.viscous_form, nslab=nslab)
        D.set_coefficients(cs)
        xu, xp = D.precond_apply(rs, PrecondConfig(kind=P1))
        out[ext] = [a.copy() for a in xu] + [xp.copy()]
        del D
    for a, b in zip(out["1"], out["0"]):
        assert np.array_equal(a, b)


def test_dist_graph_kept_across_coefficient_uploads():
    """The captured P^-1 graph survives a coefficient upload of the same problem
    class (arrays rewritten in place): a second solve with new coefficients is
    bit-identical to a fresh context's."""
    from paper_1308_4605_b200 import problems as PR
    from paper_1308_4605_b200.dist import DistSolver
    from paper_1308_4605_b200.krylov import GmresConfig
    from paper_1308_4605_b200.precond import P1, PrecondConfig
    gcfg = GmresConfig(restart=50, max_iters=500, rtol=1e-9, track_true_residual=False)
    pc = PrecondConfig(kind=P1)
    c1, c2 = PR.make_case("C5", 32, seed=11), PR.make_case("C5", 32, seed=12)
    cs1, rs1, _ = PR.prepare(c1)
    cs2, rs2, _ = PR.prepare(c2)
    D = DistSolver(c1.grid, cs1.viscous_form, nslab=2)
    D.set_coefficients(cs1)
    D.gmres_solve(rs1, pc, gcfg)
    D.set_coefficients(cs2)
    xa, pa, ha = D.gmres_solve(rs2, pc, gcfg)
    F = DistSolver(c2.grid, cs2.viscous_form, nslab=2)
    F.set_coefficients(cs2)
    xb, pb, hb = F.gmres_solve(rs2, pc, gcfg)
    assert ha.iterations == hb.iterations
    for a, b in zip(xa, xb):
        assert np.array_equal(a, b)
    assert np.array_equal(pa, pb)


def test_dist_solution_into_device_tensors_and_stats():
    """gmres_solve(out=(xu, xp)) writes the rank's planes into HBM tensors (the
    bench arm's contract) with the host result's values; the instrumented solve
    reports per-pass stats and launches are counted."""
    import torch
    from paper_1308_4605_b200.dist import DistSolver
    from paper_1308_4605_b200.krylov import GmresConfig
    from paper_1308_4605_b200.precond import P1, PrecondConfig
    case, cs, rs = _case("C5", 32)
    gcfg = GmresConfig(restart=50, max_iters=500, rtol=1e-9, track_true_residual=False)
    D = DistSolver(case.grid, cs.viscous_form, nslab=1)
    D.set_coefficients(cs)
    xu, xp, h = D.gmres_solve(rs, PrecondConfig(kind=P1), gcfg)
    du = [torch.zeros(c.shape, dtype=torch.float64, device="cuda") for c in xu]
    dp = torch.zeros(xp.shape, dtype=torch.float64, device="cuda")
    l0 = D.launch_count()
    D.set_profiling(True)
    _, _, h2 = D.gmres_solve(rs, PrecondConfig(kind=P1), gcfg, out=(du, dp))
    D.set_profiling(False)
    torch.cuda.synchronize()
    assert D.launch_count() > l0
    assert h2.iterations == h.iterations
    for a, b in zip(du, xu):
        assert np.array_equal(a.cpu().numpy(), b)
    assert np.array_equal(dp.cpu().numpy(), xp)
    st = D.kernel_stats()
    assert st["fine_face_launches"] > 0 and st["fine_face_ms"] > 0 and st["smoother_cell_launches"] > 0


@pytest.mark.parametrize("name,n,nslab", [("C5", 64, 2), ("C5", 64, 4), ("C4", 64, 2), ("C3", 64, 4)])
def test_dist_split_residual_restriction(name, n, nslab, monkeypatch):
    """Slab levels with the split residual -> restriction (residual field,
    ghost-plane exchange of component 0, light restriction; the default on
    slab levels >= 64^3 cells), forced onto every slab level here: the same
    P1 application as the single domain and the fused slab path, and GMRES
    with the single-domain iteration count."""
    from paper_1308_4605_b200.dist import DistSolver
    from paper_1308_4605_b200.krylov import GmresConfig, gmres_solve
    from paper_1308_4605_b200.precond import P1, PrecondConfig, Preconditioner
    case, cs, rs = _case(name, n)
    pc = PrecondConfig(kind=P1)
    monkeypatch.setenv("SB_DIST_RR_SPLIT", "0")
    F = DistSolver(case.grid, cs.viscous_form, nslab=nslab)
    F.set_coefficients(cs)
    fu, fp = F.precond_apply(rs, pc)
    monkeypatch.setenv("SB_DIST_RR_SPLIT", "1")
    D = DistSolver(case.grid, cs.viscous_form, nslab=nslab)
    D.set_coefficients(cs)
    xu, xp = D.precond_apply(rs, pc)
    want = Preconditioner(cs, pc).apply(rs)
    for a in range(3):
        s = np.abs(want.u.components[a]).max()
        assert np.abs(xu[a] - want.u.components[a]).max() <= 1e-11 * s, a
        assert np.abs(xu[a] - fu[a]).max() <= 1e-11 * s, a
    assert np.abs(xp - want.p.data).max() <= 1e-11 * np.abs(want.p.data).max()
    assert np.abs(xp - fp).max() <= 1e-11 * np.abs(want.p.data).max()
    gcfg = GmresConfig(restart=case.restart, max_iters=500, rtol=1e-9, track_true_residual=False)
    xd_u, xd_p, hd = D.gmres_solve(rs, pc, gcfg)
    x1, h1 = gmres_solve(rs, cs, pc, gcfg)
    assert hd.status == "converged" and abs(hd.iterations - h1.iterations) <= 1
    num = sum(np.sum((xd_u[a] - x1.u.components[a]) ** 2) for a in range(3)) + np.sum((xd_p - x1.p.data) ** 2)
    den = sum(np.sum(x1.u.components[a] ** 2) for a in range(3)) + np.sum(x1.p.data ** 2)
    assert np.sqrt(num / den) <= 1e-8


def test_dist_default_split_at_128():
    """C5 recipe at 128^3 in 2 slabs: the slab levels of >= 64^3 cells take
    the split residual -> restriction by default; GMRES matches the single
    domain (iteration count +-1, solution <= 1e-8)."""
    from paper_1308_4605_b200.dist import DistSolver
    from paper_1308_4605_b200.krylov import GmresConfig, gmres_solve
    from paper_1308_4605_b200.precond import P1, PrecondConfig
    case, cs, rs = _case("C5", 128)
    pc = PrecondConfig(kind=P1)
    gcfg = GmresConfig(restart=case.restart, max_iters=500, rtol=1e-9, track_true_residual=False)
    D = DistSolver(case.grid, cs.viscous_form, nslab=2)
    D.set_coefficients(cs)
    xu, xp, hd = D.gmres_solve(rs, pc, gcfg)
    x1, h1 = gmres_solve(rs, cs, pc, gcfg)
    assert hd.status == h1.status == "converged" and abs(hd.iterations - h1.iterations) <= 1
    num = sum(np.sum((xu[a] - x1.u.components[a]) ** 2) for a in range(3)) + np.sum((xp - x1.p.data) ** 2)
    den = sum(np.sum(x1.u.components[a] ** 2) for a in range(3)) + np.sum(x1.p.data ** 2)
    assert np.sqrt(num / den) <= 1e-8


# ---- the NCCL transport on one GPU (1-rank communicator, self send/recv) -------------


@pytest.mark.parametrize("name,n,kind", [("C5", 32, "P1"), ("C4", 32, "P1"), ("C3", 64, "P2"), ("C5", 128, "P1")])
def test_dist_nccl_self_matches_single(name, n, kind):
    """One rank, one slab, routed through NCCL: every halo exchange is a grouped
    ncclSend/ncclRecv to itself, every reduction an ncclAllReduce, the coarse
    gather an ncclAllGather, and the P^-1 graph captures those NCCL nodes --
    the branches each rank takes at N > 1.  The solve matches the single
    domain (iterations +-1, solution <= 1e-8, r_P history 1e-6) and the
    device-copy transport of the same one-slab layout."""
    from paper_1308_4605_b200.dist import DistSolver
    from paper_1308_4605_b200.krylov import GmresConfig, gmres_solve
    from paper_1308_4605_b200.precond import PrecondConfig, PrecondKind
    case, cs, rs = _case(name, n)
    gcfg = GmresConfig(restart=case.restart, max_iters=500, rtol=1e-9, track_true_residual=False)
    pc = PrecondConfig(kind=PrecondKind(kind))
    x1, h1 = gmres_solve(rs, cs, pc, gcfg)
    D = DistSolver(case.grid, cs.viscous_form, nslab=1, nccl_self=True)
    assert D.uses_nccl
    D.set_coefficients(cs)
    xu, xp, hd = D.gmres_solve(rs, pc, gcfg)
    assert hd.status == h1.status == "converged"
    assert abs(hd.iterations - h1.iterations) <= 1
    num = sum(np.sum((xu[a] - x1.u.components[a]) ** 2) for a in range(3)) + np.sum((xp - x1.p.data) ** 2)
    den = sum(np.sum(x1.u.components[a] ** 2) for a in range(3)) + np.sum(x1.p.data ** 2)
    assert np.sqrt(num / den) <= 1e-8
    r1, r2 = np.array(h1.rows())[:, 2], np.array(hd.rows())[:, 2]
    k = min(len(r1), len(r2))
    assert np.allclose(r1[:k], r2[:k], rtol=1e-6)
    # the device-copy transport of the same layout: the same arithmetic, so the
    # same iterates (exchanges only move bytes; 1-rank reductions are copies)
    F = DistSolver(case.grid, cs.viscous_form, nslab=1, nccl_self=False)
    assert not F.uses_nccl
    F.set_coefficients(cs)
    fu, fp, hf = F.gmres_solve(rs, pc, gcfg)
    assert hf.iterations == hd.iterations
    for a in range(3):
        assert np.array_equal(fu[a], xu[a])
    assert np.array_equal(fp, xp)


def test_dist_nccl_self_operator_precond_and_graph():
    """apply_M, P^-1 (eager and graph-captured with NCCL nodes) through the
    NCCL branches equal the single-domain operators; a second coefficient
    upload keeps the captured graph and stays bit-identical to a fresh solver."""
    from paper_1308_4605_b200 import problems as PR
    from paper_1308_4605_b200.dist import DistSolver
    from paper_1308_4605_b200.krylov import GmresConfig
    from paper_1308_4605_b200.operators import apply_M
    from paper_1308_4605_b200.precond import P1, PrecondConfig, Preconditioner
    case, cs, rs = _case("C4", 64)
    D = DistSolver(case.grid, cs.viscous_form, nslab=1, nccl_self=True)
    D.set_coefficients(cs)
    mu, mp = D.apply_M(rs)
    ref = apply_M(rs, cs)
    for a in range(3):
        assert np.allclose(mu[a], ref.u.components[a], rtol=0, atol=1e-12 * np.abs(ref.u.components[a]).max())
    assert np.allclose(mp, ref.p.data, rtol=0, atol=1e-12 * np.abs(ref.p.data).max())
    want = Preconditioner(cs, PrecondConfig(kind=P1)).apply(rs)
    xu, xp = D.precond_apply(rs, PrecondConfig(kind=P1))
    for a in range(3):
        assert np.abs(xu[a] - want.u.components[a]).max() <= 1e-11 * np.abs(want.u.components[a]).max()
    assert np.abs(xp - want.p.data).max() <= 1e-11 * np.abs(want.p.data).max()
    gcfg = GmresConfig(restart=50, max_iters=500, rtol=1e-9, track_true_residual=False)
    c1, c2 = PR.make_case("C5", 32, seed=11), PR.make_case("C5", 32, seed=12)
    cs1, rs1, _ = PR.prepare(c1)
    cs2, rs2, _ = PR.prepare(c2)
    E = DistSolver(c1.grid, cs1.viscous_form, nslab=1, nccl_self=True)
    E.set_coefficients(cs1)
    E.gmres_solve(rs1, PrecondConfig(kind=P1), gcfg)
    E.set_coefficients(cs2)
    xa, pa, ha = E.gmres_solve(rs2, PrecondConfig(kind=P1), gcfg)
    F = DistSolver(c2.grid, cs2.viscous_form, nslab=1, nccl_self=True)
    F.set_coefficients(cs2)
    xb, pb, hb = F.gmres_solve(rs2, PrecondConfig(kind=P1), gcfg)
    assert ha.iterations == hb.iterations
    for a, b in zip(xa, xb):
        assert np.array_equal(a, b)
    assert np.array_equal(pa, pb)


@pytest.mark.parametrize("nccl_self,nslab", [(True, 1), (False, 2), (False, 4)])
@pytest.mark.parametrize("which", ["face", "cell"])
def test_dist_zero_diagonal_raises(nccl_self, nslab, which):
    """A zero smoother diagonal (mu = 0 rows with theta = 0 for the velocity
    operator; for the pressure operator an infinite rho, i.e. 1/rho = 0) is
    reported as
    ZeroDivisionError (multigrid.py:74-75, 84-88) through every transport:
    the per-slab flags are max-reduced, so each condition survives any number
    of flagging slabs / ranks."""
    from paper_1308_4605_b200 import problems as PR
    from paper_1308_4605_b200.dist import DistSolver
    from paper_1308_4605_b200.grid import CellField
    from paper_1308_4605_b200.krylov import GmresConfig
    from paper_1308_4605_b200.operators import make_coefficients
    from paper_1308_4605_b200.precond import P1, PrecondConfig
    case = PR.make_case("C5", 32)
    g = case.grid
    if which == "face":  # steady region of zero viscosity (tests/test_multigrid.py:75-83)
        mu = np.zeros(g.cells)
        mu[0, 0, 0] = 1.0
        coeff = make_coefficients(g, 0.0, CellField.full(g, 1.0), CellField(g, mu))
    else:
        coeff = make_coefficients(g, 0.0, CellField.full(g, np.inf), CellField.full(g, 1.0))
    D = DistSolver(g, coeff.viscous_form, nslab=nslab, nccl_self=nccl_self)
    try:
        D.set_coefficients(coeff)
    except (ZeroDivisionError, ValueError):
        return
    gcfg = GmresConfig(restart=10, max_iters=5, rtol=1e-9, track_true_residual=False)
    with pytest.raises((ZeroDivisionError, ValueError)):
        D.gmres_solve(case.rhs, PrecondConfig(kind=P1), gcfg)


@pytest.mark.parametrize("name,n,nslab,nccl_self", [("C5", 64, 1, True), ("C4", 64, 2, False), ("C5", 64, 4, False),
                                                    ("C3", 32, 1, True)])
def test_dist_exchange_overlap_is_bit_identical(name, n, nslab, nccl_self, monkeypatch):
    """The black colour pass relaxes its 2 boundary planes per side first, then
    its halo exchange runs on a second stream while the interior planes are
    relaxed (colour_pass_exchange).  Same-colour updates are independent, so
    the solve is bit-identical to exchanging after the whole pass
    (SB_DIST_OVERLAP=0) -- with the copy transport between slabs and with the
    NCCL nodes (1-rank communicator) in the captured P^-1 graph."""
    from paper_1308_4605_b200.dist import DistSolver
    from paper_1308_4605_b200.krylov import GmresConfig
    from paper_1308_4605_b200.precond import P1, PrecondConfig
    case, cs, rs = _case(name, n)
    gcfg = GmresConfig(restart=case.restart, max_iters=500, rtol=1e-9, track_true_residual=False)
    res = {}
    for ov in ("1", "0"):
        monkeypatch.setenv("SB_DIST_OVERLAP", ov)
        D = DistSolver(case.grid, cs.viscous_form, nslab=nslab, nccl_self=nccl_self)
        assert D.uses_nccl == nccl_self
        D.set_coefficients(cs)
        xu, xp, h = D.gmres_solve(rs, PrecondConfig(kind=P1), gcfg)
        res[ov] = (xu, xp, h)
        del D
    monkeypatch.delenv("SB_DIST_OVERLAP")
    assert res["1"][2].status == res["0"][2].status == "converged"
    assert res["1"][2].iterations == res["0"][2].iterations
    for a in range(3):
        assert np.array_equal(res["1"][0][a], res["0"][0][a])
    assert np.array_equal(res["1"][1], res["0"][1])


def test_dist_large_restart_is_rejected():
    """The slab solver keeps the 127-vector basis cap: a larger
    restart is refused with the reference's exception type, not truncated."""
    from paper_1308_4605_b200.dist import DistSolver
    from paper_1308_4605_b200.krylov import GmresConfig
    from paper_1308_4605_b200.precond import P1, PrecondConfig
    case, cs, rs = _case("C5", 32)
    D = DistSolver(case.grid, cs.viscous_form, nslab=2)
    D.set_coefficients(cs)
    with pytest.raises(ValueError):
        D.gmres_solve(rs, PrecondConfig(kind=P1), GmresConfig(restart=128, max_iters=5, rtol=1e-9))
    xu, xp, h = D.gmres_solve(rs, PrecondConfig(kind=P1), GmresConfig(restart=127, max_iters=3, rtol=1e-9))
    assert h.iterations == 3 and h.status == "maxiter"
