"""Full-size goldens: the REFERENCE ``stokesmg.gmres_solve`` at BASELINE sizes.

Run in the build container (where ``/root/reference`` exists), one case per
process (each is single-threaded NumPy and takes minutes):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden_full.py C3_128
    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden_full.py C4_256_k3
    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden_full.py C5_256_k3

Inputs are the repo's seeded recipes (``paper_1308_4605_b200.problems.make_case``,
SURVEY §8d; NumPy only), handed to the reference's own types, ``rescale``d
as the CLI does (``cli.py:340-343``) and solved by the reference's
``gmres_solve`` (``krylov.py:164-214``):

* ``C3_128``    -- C3 at its BASELINE size 128^3, P1, GMRES(50), to rtol 1e-9
  (the full solve; ~7 min here);
* ``C4_256_k3`` -- C4 at 256^3, P1, GMRES(30), ``max_iters=3`` (SURVEY §8c:
  C4/C5 are compared over their first k iterations);
* ``C5_256_k3`` -- C5's single-GPU point 256^3, P1, GMRES(50), ``max_iters=3``;
* ``C4_256_P5_k2``, ``C4_256_P2_k2``, ``C5_256_P3_k2`` -- the other
  preconditioner families (P5: two velocity solves; P2 / P3: triangular forms,
  the Schur complement with its Poisson solve on C4's theta > 0) at 256^3,
  ``max_iters=2``.

Stored per case (``tests/golden/full_<case>.npz``): the history rows
(k, scalar V-cycles, r_P, r_true, restart flag), iterations and status, the
fp64 2-norm of every solution component, and a seeded subsample of every
component of x (flat C-order indices stored beside the values), so the GPU
test regenerates the inputs from the seed and compares without the reference.
"""

from __future__ import annotations

import json
import pathlib
import sys
import time

import numpy as np

REF = pathlib.Path("/root/reference/pkg/src")
OUT = pathlib.Path(__file__).resolve().parent
sys.path.insert(0, str(REF))
sys.path.insert(0, str(OUT.parent.parent))

import stokesmg as sm  # noqa: E402
from stokesmg import grid as G  # noqa: E402
from stokesmg import operators as OP  # noqa: E402
from stokesmg import precond as PC  # noqa: E402

from paper_1308_4605_b200 import problems as HP  # noqa: E402  (numpy-only recipes)

CASES = {  # name: (config, n, precond, max_iters, subsample stride)
    "C3_128": ("C3", 128, "P1", 500, 64),
    "C4_256_k3": ("C4", 256, "P1", 3, 512),
    "C5_256_k3": ("C5", 256, "P1", 3, 512),
    # the other preconditioner families at BASELINE size (two iterations each)
    "C4_256_P5_k2": ("C4", 256, "P5", 2, 1024),
    "C5_256_P3_k2": ("C5", 256, "P3", 2, 1024),
    "C4_256_P2_k2": ("C4", 256, "P2", 2, 1024),
}


def ref_types(case):
    code = {"periodic": G.PERIODIC, "no_slip": G.NO_SLIP, "free_slip": G.FREE_SLIP}
    g = G.GridSpec(tuple(case.grid.cells), case.grid.h,
                   tuple((code[lo.value], code[hi.value]) for lo, hi in case.grid.bc))
    c0 = case.coeff
    cref = OP.CoefficientSet(
        theta=c0.theta, rho_cell=G.CellField(g, c0.rho_cell.data),
        rho_face=G.FaceField(g, c0.rho_face.components),
        mu_cell=G.CellField(g, c0.mu_cell.data),
        mu_node_edge=G.NodeEdgeField(g, dict(c0.mu_node_edge.arrays)),
        gamma_cell=G.CellField(g, c0.gamma_cell.data), viscous_form=OP.STRESS)
    rhs = G.StokesVector(G.FaceField(g, case.rhs.u.components), G.CellField(g, case.rhs.p.data))
    return g, cref, rhs


def subsample(arr, stride, seed):
    rng = np.random.default_rng(seed)
    n = arr.size
    idx = np.sort(rng.choice(n, size=max(1, n // stride), replace=False)).astype(np.int64)
    return idx, arr.reshape(-1)[idx].copy()


def run(name):
    cname, n, kind, max_iters, stride = CASES[name]
    case = HP.make_case(cname, n)
    g, cref, rhs = ref_types(case)
    t0 = time.perf_counter()
    cs, rs, spec = OP.rescale(cref, rhs)
    gcfg = sm.GmresConfig(restart=case.restart, max_iters=max_iters, rtol=1e-9, atol=0.0,
                          track_true_residual=True)
    t1 = time.perf_counter()
    x, hist = sm.gmres_solve(rs, cs, PC.PrecondConfig(kind=PC.PrecondKind(kind)), gcfg)
    t2 = time.perf_counter()
    store = {"hist": np.array(hist.rows(), dtype=np.float64)}
    norms = []
    for a, comp in enumerate(list(x.u.components) + [x.p.data]):
        idx, val = subsample(np.ascontiguousarray(comp), stride, 1000 + a)
        store[f"idx{a}"] = idx
        store[f"val{a}"] = val
        norms.append(float(np.linalg.norm(comp)))
    np.savez_compressed(OUT / f"full_{name}.npz", **store)
    meta = dict(name=name, config=cname, n=n, precond=kind, restart=case.restart,
                max_iters=max_iters, rtol=1e-9, status=hist.status, iterations=hist.iterations,
                scalar_vcycles=int(hist.rows()[-1][1]), c=spec.c, norms=norms, stride=stride,
                ref_solve_s=t2 - t1, ref_setup_s=t1 - t0,
                generator="tests/golden/make_golden_full.py (reference stokesmg.gmres_solve)")
    (OUT / f"full_{name}.json").write_text(json.dumps(meta, indent=1))
    print(json.dumps(meta))


if __name__ == "__main__":
    for nm in sys.argv[1:] or list(CASES):
        run(nm)
