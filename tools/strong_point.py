"""C4 at its BASELINE size (256^3, walls in z, theta > 0) through the slab path
with the strong-scaling decompositions of 2 / 4 / 8 ranks as slabs of ONE
process (copy transport): iteration count and solution against the single
domain -- the decomposition each rank runs at N > 1, at production sizes.

    python tools/strong_point.py [nslab ...]
"""
import json
import pathlib
import sys
import time

import numpy as np

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent.parent))

import torch  # noqa: E402

from paper_1308_4605_b200 import problems as PR  # noqa: E402
from paper_1308_4605_b200.dist import DistSolver  # noqa: E402
from paper_1308_4605_b200.krylov import GmresConfig, gmres_solve  # noqa: E402
from paper_1308_4605_b200.precond import P1, PrecondConfig, Preconditioner  # noqa: E402

slabs = [int(a) for a in sys.argv[1:]] or [2, 4, 8]
case = PR.make_case("C4")
cs, rs, _ = PR.prepare(case)
gcfg = GmresConfig(restart=case.restart, max_iters=500, rtol=1e-9, atol=0.0, track_true_residual=False)
pc = PrecondConfig(kind=P1)
P = Preconditioner(cs, pc)
x, h = gmres_solve(rs, cs, None, gcfg, precond=P)
xs = [c.copy() for c in x.u.components] + [x.p.data.copy()]
rp = np.array([e.resid_precond for e in h.entries])
out = {"cells": list(case.grid.cells), "single": {"iterations": h.iterations, "status": h.status}, "slabs": []}
del P, x
torch.cuda.empty_cache()
for ns in slabs:
    D = DistSolver(case.grid, cs.viscous_form, nslab=ns)
    D.set_coefficients(cs)
    t0 = time.perf_counter()
    xu, xp, hd = D.gmres_solve(rs, pc, gcfg)
    torch.cuda.synchronize()
    num = sum(float(np.sum((a - b) ** 2)) for a, b in zip(list(xu) + [xp], xs))
    den = sum(float(np.sum(b ** 2)) for b in xs)
    rd = np.array([e.resid_precond for e in hd.entries])
    k = min(len(rd), len(rp))
    out["slabs"].append({"nslab": ns, "iterations": hd.iterations, "status": hd.status,
                         "rel_l2_vs_single": (num / den) ** 0.5,
                         "max_rel_rP_history_diff": float(np.max(np.abs(rd[:k] - rp[:k]) / rp[:k])),
                         "info": D.info(), "wall_s_host_arrays": time.perf_counter() - t0})
    del D
    torch.cuda.empty_cache()
print(json.dumps(out))
