"""Generate golden vectors by running the REFERENCE package ``stokesmg`` itself.

Run in the build container (where ``/root/reference`` exists):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

It imports the reference from ``/root/reference/pkg/src`` (read-only; nothing
is copied), draws seeded inputs, calls the reference's own functions on them
and stores inputs + outputs in ``tests/golden/golden.npz`` with an index in
``tests/golden/golden.json``.  The CPU tests pin ``oracle/`` against these
vectors and the GPU tests compare the device path with them, so neither needs
the reference at run time (it does not exist on the GPU box).
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
from stokesmg import multigrid as MG  # noqa: E402
from stokesmg import operators as OP  # noqa: E402
from stokesmg import precond as PC  # noqa: E402
from stokesmg import problems as PR  # noqa: E402

OUT = pathlib.Path(__file__).resolve().parent
BCS = {"p": G.PERIODIC, "n": G.NO_SLIP, "f": G.FREE_SLIP}
FORMS = {"laplacian": OP.LAPLACIAN, "stress": OP.STRESS, "stress_bulk": OP.STRESS_BULK}

store: dict = {}
index: list = []


def grid(cells, bc, h):
    return G.GridSpec(tuple(cells), h, tuple((BCS[b[0]], BCS[b[1]]) for b in bc))


def put(name, key, arr):
    store[f"{name}/{key}"] = np.asarray(arr, dtype=np.float64)


def put_face(name, key, f):
    for a, c in enumerate(f.components):
        put(name, f"{key}{a}", c)


def put_coeff(name, c):
    put(name, "rho_cell", c.rho_cell.data)
    put_face(name, "rho_face", c.rho_face)
    put(name, "mu_cell", c.mu_cell.data)
    for k, v in sorted(c.mu_node_edge.arrays.items()):
        put(name, f"mu_edge{k[0]}{k[1]}", v)
    put(name, "gamma_cell", c.gamma_cell.data)


def rand_coeff(g, rng, theta, form):
    mu = G.CellField(g, 0.5 + rng.random(g.cells))
    rho = G.CellField(g, 0.5 + rng.random(g.cells))
    gam = G.CellField(g, rng.random(g.cells))
    return OP.make_coefficients(g, theta, rho, mu, gam, FORMS[form])


def rand_face(g, rng):
    u = G.FaceField.zeros(g)
    for a in range(g.dim):
        v = u.interior(a)
        v[...] = rng.standard_normal(v.shape)
    return u


def rand_cell(g, rng):
    return G.CellField(g, rng.standard_normal(g.cells))


def meta(name, kind, g, bc, theta, form, **extra):
    index.append(dict(name=name, kind=kind, cells=list(g.cells), h=g.h, bc=bc, theta=theta,
                      form=form, **extra))


OPER_GRIDS = [
    ((8, 12), ["pp", "pp"], 0.125),
    ((8, 12), ["pp", "nn"], 0.125),
    ((8, 12), ["nn", "ff"], 0.25),
    ((8, 12), ["fn", "pp"], 0.5),
    ((4, 6, 8), ["pp", "pp", "pp"], 0.125),
    ((4, 6, 8), ["pp", "pp", "nn"], 0.125),
    ((4, 6, 8), ["nn", "ff", "pp"], 0.25),
    ((4, 6, 8), ["fn", "nn", "nf"], 0.5),
]


def gen_operators():
    rng = np.random.default_rng(20240817)
    for gi, (cells, bc, h) in enumerate(OPER_GRIDS):
        g = grid(cells, bc, h)
        for form in ("laplacian", "stress", "stress_bulk"):
            for theta in (0.0, 0.7):
                name = f"op{gi}_{form}_{theta}"
                c = rand_coeff(g, rng, theta, form)
                u, p = rand_face(g, rng), rand_cell(g, rng)
                put_coeff(name, c)
                put_face(name, "u", u)
                put(name, "p", p.data)
                m = OP.apply_M(G.StokesVector(u, p), c)
                put_face(name, "Mu", m.u)
                put(name, "Mp", m.p.data)
                put(name, "Lp", OP.apply_Lrho(p, c).data)
                put_face(name, "diagf", OP.helmholtz_diagonal(g, c))
                put(name, "diagc", OP.lrho_diagonal(g, c).data)
                # one smoother sweep of each kind from a random state
                x = rand_face(g, rng)
                rhs = rand_face(g, rng)
                put_face(name, "sx0", x)
                put_face(name, "srhs", rhs)
                xs = x.copy()
                MG.smooth_face(xs, rhs, g, c, OP.helmholtz_diagonal(g, c), 0.8)
                put_face(name, "sx1", xs)
                y = rand_cell(g, rng)
                yr = rand_cell(g, rng)
                put(name, "cy0", y.data)
                put(name, "cyrhs", yr.data)
                ys = y.copy()
                MG.smooth_cell(ys, yr, g, c, OP.lrho_diagonal(g, c), 0.8)
                put(name, "cy1", ys.data)
                # transfers and coarsening
                put_face(name, "rf", MG.restrict_face(u))
                put(name, "rc", MG.restrict_cell(p).data)
                gc = g.coarsened()
                uc, pc = rand_face(gc, rng), rand_cell(gc, rng)
                put_face(name, "pin", uc)
                put(name, "pinc", pc.data)
                put_face(name, "pf", MG.prolong_face(uc))
                put(name, "pc", MG.prolong_cell(pc).data)
                cc = MG.coarsen_coefficients(c, gc)
                put_coeff(name + "/coarse", cc)
                # residual -> restriction as the V-cycle does it
                rr = MG._residual(x, rhs, g, c, "face")
                put_face(name, "rrf", MG.restrict_face(rr))
                rrc = MG._residual(y, yr, g, c, "cell")
                put(name, "rrc", MG.restrict_cell(rrc).data)
                meta(name, "operators", g, bc, theta, form)


VC_GRIDS = [
    ((16, 16), ["pp", "pp"], 1 / 16),
    ((16, 24), ["pp", "nn"], 1 / 16),
    ((12, 12), ["ff", "nn"], 1 / 12),
    ((8, 8, 8), ["pp", "pp", "pp"], 1 / 8),
    ((8, 8, 12), ["pp", "pp", "nn"], 1 / 8),
    ((8, 8, 8), ["nn", "ff", "pp"], 1 / 8),
]


def gen_vcycles():
    rng = np.random.default_rng(1308)
    for gi, (cells, bc, h) in enumerate(VC_GRIDS):
        g = grid(cells, bc, h)
        for theta in (0.0, 1.0):
            form = "stress"
            name = f"vc{gi}_{theta}"
            c = rand_coeff(g, rng, theta, form)
            put_coeff(name, c)
            hier = MG.build_hierarchy(g, c)
            params = MG.SmootherParams()
            rf, rc = rand_face(g, rng), rand_cell(g, rng)
            put_face(name, "rhsf", rf)
            put(name, "rhsc", rc.data)
            put_face(name, "vf", MG.vcycle(rf, hier, params, "face"))
            put(name, "vcell", MG.vcycle(rc, hier, params, "cell").data)
            put_face(name, "mg2f", MG.mg_solve(rf, hier, params, 2, "face"))
            put(name, "mg2c", MG.mg_solve(rc, hier, params, 2, "cell").data)
            r = G.StokesVector(rand_face(g, rng), rand_cell(g, rng))
            put_face(name, "ru", r.u)
            put(name, "rp", r.p.data)
            counts = {}
            for kind in ("P1", "P2", "P3", "P4", "P5"):
                for sign in ("minus", "plus"):
                    if sign == "plus" and kind not in ("P1", "P4"):
                        continue
                    cfg = PC.PrecondConfig(kind=PC.PrecondKind(kind),
                                           schur=sm.SchurConfig(sign=sm.SchurSign(sign)))
                    pre = PC.Preconditioner(c, cfg)
                    out = pre.apply(r)
                    put_face(name, f"{kind}{sign}_u", out.u)
                    put(name, f"{kind}{sign}_p", out.p.data)
                    counts[f"{kind}{sign}"] = pre.scalar_vcycles
            meta(name, "vcycle", g, bc, theta, form, levels=len(hier), vcycles=counts)


def gen_affine():
    """Inhomogeneous walls: apply_A(u, coeff, bvals), boundary_lift, homogenize
    (operators.py:224-264, 348-360, 471-512) on every wall-bounded operator grid."""
    rng = np.random.default_rng(4605)
    for gi, (cells, bc, h) in enumerate(OPER_GRIDS):
        g = grid(cells, bc, h)
        if all(g.periodic(a) for a in range(g.dim)):
            continue
        for form in ("laplacian", "stress", "stress_bulk"):
            name = f"af{gi}_{form}"
            c = rand_coeff(g, rng, 0.7, form)
            normal, tang = {}, {}
            for a in range(g.dim):
                if g.periodic(a):
                    continue
                for side in (0, 1):
                    normal[(a, side)] = rng.standard_normal(
                        tuple(n for ax, n in enumerate(g.cells) if ax != a))
                    put(name, f"bn{a}{side}", normal[(a, side)])
                    for comp in range(g.dim):
                        if comp == a:
                            continue
                        tang[(a, side, comp)] = rng.standard_normal(
                            tuple(n for ax, n in enumerate(g.face_shape(comp)) if ax != a))
                        put(name, f"bt{a}{side}{comp}", tang[(a, side, comp)])
            bv = OP.BoundaryValues(g, normal, tang)
            u = OP.boundary_lift(bv)
            put_face(name, "lift", OP.boundary_lift(bv))
            for a in range(g.dim):
                u.interior(a)[...] = rng.standard_normal(u.interior(a).shape)
            put_coeff(name, c)
            put_face(name, "u", u)
            put_face(name, "Au", OP.apply_A(u, c, bv))
            put_face(name, "A0", OP.apply_A(u, c))
            m = OP.apply_M(G.StokesVector(u, G.CellField(g, np.zeros(g.cells))), c)
            put_face(name, "Mu", m.u)
            put(name, "Mp", m.p.data)
            rhs = G.StokesVector(rand_face(g, rng), rand_cell(g, rng))
            for a in range(g.dim):  # boundary faces of the rhs carry data too
                rhs.u.components[a][...] = rng.standard_normal(rhs.u.components[a].shape)
            rhs.p.data -= rhs.p.data.mean()
            net = float(OP.div(OP.boundary_lift(bv)).data.sum())
            rhs.p.data -= net / rhs.p.data.size  # compatible divergence source
            put_face(name, "ru", rhs.u)
            put(name, "rp", rhs.p.data)
            hom = OP.homogenize(bv, c, rhs)
            put_face(name, "hu", hom.u)
            put(name, "hp", hom.p.data)
            meta(name, "affine", g, bc, 0.7, form, normal=sorted(f"{a}{s}" for a, s in normal),
                 tangential=sorted(f"{a}{s}{k}" for a, s, k in tang))


def gen_gmres():
    """Full solves of the BASELINE recipes at reduced size (reference API only)."""
    sys.path.insert(0, str(OUT.parent.parent))
    from paper_1308_4605_b200 import problems as HP  # host-side generators (numpy only)

    cases = [("C1", 64, "P1"), ("C1", 32, "P2"), ("C2", 64, "P1"), ("C2", 64, "P2"),
             ("C3", 16, "P1"), ("C4", 16, "P1"), ("C5", 16, "P1")]
    for cname, n, kind in cases:
        case = HP.make_case(cname, n)
        code = {"periodic": "p", "no_slip": "n", "free_slip": "f"}
        bcs = [code[lo.value] + code[hi.value] for lo, hi in case.grid.bc]
        g = grid(case.grid.cells, bcs, case.grid.h)
        # rebuild the case in reference types (same arrays)
        gref = g
        c0 = case.coeff
        cref = OP.CoefficientSet(
            theta=c0.theta, rho_cell=G.CellField(gref, c0.rho_cell.data),
            rho_face=G.FaceField(gref, c0.rho_face.components),
            mu_cell=G.CellField(gref, c0.mu_cell.data),
            mu_node_edge=G.NodeEdgeField(gref, dict(c0.mu_node_edge.arrays)),
            gamma_cell=G.CellField(gref, c0.gamma_cell.data), viscous_form=OP.STRESS)
        rhs = G.StokesVector(G.FaceField(gref, case.rhs.u.components), G.CellField(gref, case.rhs.p.data))
        cs, rs, spec = OP.rescale(cref, rhs)
        name = f"gm_{cname}_{n}_{kind}"
        put_coeff(name, cs)
        put_face(name, "bu", rs.u)
        put(name, "bp", rs.p.data)
        gcfg = sm.GmresConfig(restart=case.restart, max_iters=500, rtol=1e-9, atol=0.0,
                              track_true_residual=True)
        x, hist = sm.gmres_solve(rs, cs, PC.PrecondConfig(kind=PC.PrecondKind(kind)), gcfg)
        put_face(name, "xu", x.u)
        put(name, "xp", x.p.data)
        put(name, "hist", np.array(hist.rows(), dtype=np.float64))
        meta(name, "gmres", gref, bcs, cs.theta, "stress", precond=kind,
             restart=case.restart, status=hist.status, iterations=hist.iterations, c=spec.c)


FORM_SOLVES = [  # (cells, bc, form, theta, precond, schur sign, restart)
    ((32, 32), ["nn", "nn"], "laplacian", 0.0, "P1", "minus", 20),
    ((32, 48), ["ff", "pp"], "stress_bulk", 0.5, "P2", "minus", 20),
    ((32, 32), ["fn", "nf"], "stress", 2.0, "P3", "minus", 30),
    ((32, 32), ["pp", "nn"], "stress_bulk", 1.0, "P4", "plus", 30),
    ((32, 32), ["nn", "ff"], "laplacian", 0.3, "P5", "minus", 30),
    ((8, 8, 8), ["nn", "nn", "nn"], "laplacian", 0.0, "P1", "minus", 20),
    ((8, 8, 16), ["pp", "ff", "nn"], "stress_bulk", 1.0, "P2", "minus", 20),
    ((8, 16, 8), ["fn", "pp", "pp"], "stress", 0.0, "P4", "plus", 30),
    ((16, 8, 8), ["pp", "pp", "pp"], "stress", 0.7, "P5", "minus", 30),
]


def gen_form_solves():
    """GMRES solves beyond the BASELINE recipes: every viscous form, mixed
    no-slip / free-slip / periodic walls, steady and unsteady, P1..P5 and both
    Schur signs, each with the reference's own coefficient averaging and rhs."""
    rng = np.random.default_rng(8217)
    for k, (cells, bc, form, theta, kind, sign, restart) in enumerate(FORM_SOLVES):
        g = grid(cells, bc, 1.0 / cells[0])
        c = rand_coeff(g, rng, theta, form)
        rhs, _ = PR.make_rhs(g, c, seed=100 + k)
        cs, rs, spec = OP.rescale(c, rhs)
        name = f"gf{k}_{form}_{kind}"
        put_coeff(name, cs)
        put_face(name, "bu", rs.u)
        put(name, "bp", rs.p.data)
        gcfg = sm.GmresConfig(restart=restart, max_iters=300, rtol=1e-9, atol=0.0, track_true_residual=True)
        pcfg = PC.PrecondConfig(kind=PC.PrecondKind(kind), schur=sm.SchurConfig(sign=sm.SchurSign(sign)))
        x, hist = sm.gmres_solve(rs, cs, pcfg, gcfg)
        put_face(name, "xu", x.u)
        put(name, "xp", x.p.data)
        put(name, "hist", np.array(hist.rows(), dtype=np.float64))
        meta(name, "gmres", g, bc, cs.theta, form, precond=kind, schur_sign=sign, restart=restart,
             status=hist.status, iterations=hist.iterations, c=spec.c)


DRIVER_CONFIGS = [
    {"problem": {"kind": "bubble", "dim": 2, "cells": 32, "bc": "no_slip", "seed": 3},
     "solver": {"gmres": {"restart": 10, "rtol": 1e-9}},
     "sweep": {"solver.precond.kind": ["P1", "P2", "P3"], "problem.beta": ["inf", 0.5, 0]}},
    {"problem": {"kind": "constant", "dim": 3, "cells": 8, "bc": "periodic", "mu0": 2.0,
                 "beta": "inf", "seed": 5},
     "solver": {"precond": {"kind": "P1"}, "gmres": {"restart": 20, "rtol": 1e-10}},
     "sweep": {"solver.precond.velocity_cycles": [1, 2]}},
    {"problem": {"kind": "bubble", "dim": 2, "cells": [32, 16], "bc": ["periodic", "free_slip"],
                 "viscous_form": "stress_bulk", "gamma0": 0.5, "beta": 1.0, "seed": 11,
                 "bubble": {"r_mu": 10.0, "r_rho": 5.0}},
     "solver": {"gmres": {"restart": 30, "max_iters": 100, "track_true_residual": False}},
     "sweep": {"solver.precond.kind": ["P4", "P5"], "solver.precond.schur_sign": ["minus", "plus"]}},
]


def gen_driver():
    """The reference's own batch driver (cli.py cmd_run) on small configs: the
    manifest rows and history CSVs the device driver must reproduce."""
    import tempfile
    from stokesmg import cli
    for k, cfg in enumerate(DRIVER_CONFIGS):
        with tempfile.TemporaryDirectory() as out:
            rc = cli.cmd_run(json.loads(json.dumps(cfg)), out, 1, None)
            man = json.loads((pathlib.Path(out) / "manifest.json").read_text())
            rows = []
            for r in man["runs"]:
                text = (pathlib.Path(out) / r["file"]).read_text().splitlines()
                assert text[0] == cli.CSV_HEADER
                put(f"drv{k}", f"run{r['index']}", np.array([[float(v) for v in ln.split(",")] for ln in text[1:]]))
                rows.append({key: r[key] for key in ("index", "file", "sweep_point", "seed", "status",
                                                     "iterations", "scalar_vcycles")})
        index.append(dict(name=f"drv{k}", kind="driver", config=cfg, exit_code=rc, runs=rows,
                          manifest_keys=sorted(man), row_keys=sorted(man["runs"][0])))


def main():
    gen_operators()
    gen_vcycles()
    gen_gmres()
    gen_affine()
    gen_driver()
    gen_form_solves()
    np.savez_compressed(OUT / "golden.npz", **store)
    (OUT / "golden.json").write_text(json.dumps(index, indent=1))
    print(len(index), "cases,", len(store), "arrays ->", OUT / "golden.npz")


if __name__ == "__main__":
    main()
