"""Goldens for the GMRES exit paths, made by the REFERENCE ``stokesmg``.

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden_exit.py

``gmres_kernel`` (``krylov.py:81-146``) ends a solve in one of three ways; the
BASELINE recipes only ever converge, so this pins the other two on inputs
where the reference reaches them cleanly:

* ``breakdown`` -- 4x4 2D problems (periodic P1; walls, theta > 0, P2) whose
  rhs makes the preconditioned Krylov space exactly 2-dimensional
  (``invariant_rhs``): the Arnoldi norm collapses to roundoff at iteration 2
  (``krylov.py:138``, breakdown_tol = 1e-14 r_P0, ``:198``) while the target
  ``rtol = 1e-300`` is never met;
* ``maxiter``   -- GMRES(3) capped at 7 iterations (two restarts: restart
  flags on iterations 4 and 7, ``krylov.py:135``), 2D and 3D.

Stored in ``tests/golden/golden_exit.npz`` (+ ``.json`` index): the rescaled
coefficient set and rhs, the history rows, status, iterations and x.
"""

from __future__ import annotations

import json
import pathlib
import sys

import numpy as np

REF = pathlib.Path("/root/reference/pkg/src")
sys.path.insert(0, str(REF))

import stokesmg as sm  # noqa: E402
from stokesmg import grid as G  # noqa: E402
from stokesmg import operators as OP  # noqa: E402
from stokesmg import precond as PC  # noqa: E402
from stokesmg import problems as PR  # noqa: E402

OUT = pathlib.Path(__file__).resolve().parent
CODE = {"p": G.PERIODIC, "n": G.NO_SLIP, "f": G.FREE_SLIP}

CASES = [  # name, cells, bc, theta, precond, restart, max_iters, rtol, coefficient seed, rhs seed
    ("ex_breakdown_P1", (4, 4), ["pp", "pp"], 0.0, "P1", 30, 100, 1e-300, 5, None),
    ("ex_breakdown_P2", (4, 4), ["pp", "nn"], 1.0, "P2", 30, 100, 1e-300, 8, None),
    # Krylov space exhausted after ~40 Arnoldi steps (a random rhs on a 4x4
    # grid): where the Arnoldi norm collapses is roundoff-determined (the
    # reference's MGS stops at 40, CGS2 variants at 38), so the device test
    # allows +-3 iterations here
    ("ex_exhaust_P1", (4, 4), ["pp", "pp"], 0.0, "P1", 100, 300, 1e-300, 5, 3),
    ("ex_maxiter_2d", (16, 16), ["pp", "nn"], 1.0, "P1", 3, 7, 1e-12, 7, 4),
    ("ex_maxiter_3d", (8, 8, 8), ["pp", "pp", "pp"], 0.0, "P2", 3, 7, 1e-12, 9, 6),
]


def invariant_rhs(g, c, kind):
    """A rhs whose preconditioned Krylov space is exactly 2-dimensional:
    z0 = P^-1 b spans two real eigenvectors of P^-1 M (dense 4x4-grid
    operators built column by column from the reference's own P.apply /
    apply_M), so the Arnoldi norm collapses to roundoff at iteration 2 in
    any orthogonalisation scheme -- a breakdown the device must reproduce."""
    from stokesmg.grid import pack_stokes, unpack_stokes
    cs, _, _ = OP.rescale(c, G.StokesVector.zeros(g))
    P = PC.Preconditioner(cs, PC.PrecondConfig(kind=PC.PrecondKind(kind)))
    n = pack_stokes(G.StokesVector.zeros(g)).size
    Pi, PiM = np.zeros((n, n)), np.zeros((n, n))
    for i in range(n):
        e = np.zeros(n)
        e[i] = 1.0
        v = unpack_stokes(g, e)
        Pi[:, i] = pack_stokes(P.apply(v))
        PiM[:, i] = pack_stokes(P.apply(OP.apply_M(v, cs)))
    lam, vec = np.linalg.eig(PiM)
    real = [k for k in np.argsort(-np.abs(lam)) if abs(lam[k].imag) < 1e-12 and abs(lam[k]) > 1e-6]
    pick = [real[0]] + [k for k in real[1:] if abs(lam[k].real - lam[real[0]].real) > 0.1][:1]
    z0 = sum(np.real(vec[:, k]) for k in pick)
    b = np.linalg.lstsq(Pi, z0, rcond=None)[0]
    assert np.linalg.norm(Pi @ b - z0) <= 1e-10 * np.linalg.norm(z0)
    return cs, unpack_stokes(g, b)


def main():
    store, index = {}, []
    for name, cells, bc, theta, kind, restart, max_iters, rtol, cseed, rseed in CASES:
        g = G.GridSpec(cells, 1.0 / cells[0], tuple((CODE[b[0]], CODE[b[1]]) for b in bc))
        rng = np.random.default_rng(cseed)
        mu = G.CellField(g, 0.5 + rng.random(cells))
        rho = G.CellField(g, 0.5 + rng.random(cells))
        c = OP.make_coefficients(g, theta, rho, mu)
        if rseed is None:
            cs, rs = invariant_rhs(g, c, kind)
        else:
            rhs, _ = PR.make_rhs(g, c, seed=rseed)
            cs, rs, spec = OP.rescale(c, rhs)
        gcfg = sm.GmresConfig(restart=restart, max_iters=max_iters, rtol=rtol, atol=0.0,
                              track_true_residual=True)
        x, hist = sm.gmres_solve(rs, cs, PC.PrecondConfig(kind=PC.PrecondKind(kind)), gcfg)

        def put(k, a):
            store[f"{name}/{k}"] = np.asarray(a, dtype=np.float64)

        put("rho_cell", cs.rho_cell.data)
        for a, comp in enumerate(cs.rho_face.components):
            put(f"rho_face{a}", comp)
        put("mu_cell", cs.mu_cell.data)
        for k, v in sorted(cs.mu_node_edge.arrays.items()):
            put(f"mu_edge{k[0]}{k[1]}", v)
        put("gamma_cell", cs.gamma_cell.data)
        for a, comp in enumerate(rs.u.components):
            put(f"bu{a}", comp)
        put("bp", rs.p.data)
        for a, comp in enumerate(x.u.components):
            put(f"xu{a}", comp)
        put("xp", x.p.data)
        put("hist", np.array(hist.rows(), dtype=np.float64))
        index.append(dict(name=name, kind="gmres_exit", cells=list(cells), h=g.h, bc=bc, theta=cs.theta,
                          form="stress", precond=kind, restart=restart, max_iters=max_iters, rtol=rtol,
                          status=hist.status, iterations=hist.iterations,
                          its_tol=3 if name.startswith("ex_exhaust") else 0))
        print(name, hist.status, hist.iterations)
    np.savez_compressed(OUT / "golden_exit.npz", **store)
    (OUT / "golden_exit.json").write_text(json.dumps(index, indent=1))


if __name__ == "__main__":
    main()
