"""BASELINE-size parity against the REFERENCE (tests/golden/make_golden_full.py).

* C3 at its BASELINE size 128^3 (P1, GMRES(50), rtol 1e-9): the reference's
  complete solve (~7 min of CPU to make) -- iterations within +-1, the r_P
  and r_true histories, per-component solution norms, and a seeded 1/64
  subsample of every solution component (relative L2 <= 1e-8, north_star);
* C4 at 256^3 (P1, GMRES(30)) and C5's single-GPU point 256^3 (P1, GMRES(50))
  over their first 3 iterations (the reference cannot run them to
  convergence in the test budget): history rows and the iterate x_3.

Inputs are regenerated from the seeded recipe (problems.make_case), the same
arrays the generator handed to the reference.
"""

from __future__ import annotations

import json

import numpy as np
import pytest

from conftest import GOLD

pytestmark = pytest.mark.gpu

CASES = sorted(p.stem[len("full_"):] for p in GOLD.glob("full_*.json"))


@pytest.mark.parametrize("name", CASES)
def test_fullsize_vs_reference(name):
    from paper_1308_4605_b200 import problems as PR
    from paper_1308_4605_b200.krylov import GmresConfig, gmres_solve
    from paper_1308_4605_b200.precond import PrecondConfig, PrecondKind
    meta = json.loads((GOLD / f"full_{name}.json").read_text())
    z = np.load(GOLD / f"full_{name}.npz")
    case = PR.make_case(meta["config"], meta["n"])
    cs, rs, spec = PR.prepare(case)
    assert spec.c == pytest.approx(meta["c"], rel=1e-15)
    gcfg = GmresConfig(restart=meta["restart"], max_iters=meta["max_iters"], rtol=meta["rtol"], atol=0.0,
                       track_true_residual=True)
    x, hist = gmres_solve(rs, cs, PrecondConfig(kind=PrecondKind(meta["precond"])), gcfg)
    ref = z["hist"]
    got = np.array(hist.rows(), dtype=float)
    assert hist.status == meta["status"]
    assert abs(hist.iterations - meta["iterations"]) <= 1
    k = min(len(got), len(ref))
    assert np.array_equal(got[:k][:, [0, 1, 4]], ref[:k][:, [0, 1, 4]])
    assert np.allclose(got[:k, 2], ref[:k, 2], rtol=1e-6)
    assert np.allclose(got[1:k, 3], ref[1:k, 3], rtol=1e-5)
    comps = list(x.u.components) + [x.p.data]
    num = den = 0.0
    for a, comp in enumerate(comps):
        flat = np.ascontiguousarray(comp).reshape(-1)
        v = flat[z[f"idx{a}"]]
        w = z[f"val{a}"]
        num += float(np.sum((v - w) ** 2))
        den += float(np.sum(w ** 2))
        assert np.linalg.norm(comp) == pytest.approx(meta["norms"][a], rel=1e-8)
    assert np.sqrt(num / den) <= 1e-8
