"""The C5 weak-scaling problem of N GPUs solved on ONE GPU (as far as 180 GB
allow: N = 2, 512 x 256 x 256): iteration count of the larger problem -- the
numerical half of weak-scaling efficiency -- and the same problem through the
slab path with N slabs of 256 planes in one process (copy transport), i.e. the
decomposition each rank pair would run at its production slab size.

    python tools/weak_point.py [n_gpus=2] [single]
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

n_gpus = int(sys.argv[1]) if len(sys.argv) > 1 else 2
single_only = len(sys.argv) > 2 and sys.argv[2] == "single"  # N = 4: two copies of the state do not fit
cells = tuple(PR.c5_cells(n_gpus))
# the bench's generator (h = 1/512, rescaled), all planes on one "rank"
grid, cs, rs, _c = PR.make_c5_slab(cells, 1, 0, reduce=lambda kind, a, b: (a, b))
assert abs(grid.h - 1.0 / 512) < 1e-15 and grid.cells == cells


class _Case:
    pass


case = _Case()
case.grid = grid
gcfg = GmresConfig(restart=50, max_iters=500, rtol=1e-9, atol=0.0, track_true_residual=False)
pc = PrecondConfig(kind=P1)
out = {"cells": list(cells)}

P = Preconditioner(cs, pc)
gmres_solve(rs, cs, None, gcfg, precond=P)  # warm (graph capture)
torch.cuda.synchronize()
t0 = time.perf_counter()
x, h = gmres_solve(rs, cs, None, gcfg, precond=P)
torch.cuda.synchronize()
out["single"] = {"iterations": h.iterations, "status": h.status, "wall_s_host_arrays": time.perf_counter() - t0,
                 "device_bytes": P.device_bytes()}
xs = [c.copy() for c in x.u.components] + [x.p.data.copy()]
del P, x
torch.cuda.empty_cache()
if single_only:
    print(json.dumps(out))
    sys.exit(0)

D = DistSolver(case.grid, cs.viscous_form, nslab=n_gpus)
D.set_coefficients(cs)
D.gmres_solve(rs, pc, gcfg)
torch.cuda.synchronize()
t0 = time.perf_counter()
xu, xp, hd = D.gmres_solve(rs, pc, gcfg)
torch.cuda.synchronize()
num = sum(float(np.sum((a - b) ** 2)) for a, b in zip(list(xu) + [xp], xs))
den = sum(float(np.sum(b ** 2)) for b in xs)
out["slabs"] = {"nslab": n_gpus, "iterations": hd.iterations, "status": hd.status,
                "wall_s_host_arrays": time.perf_counter() - t0, "rel_l2_vs_single": (num / den) ** 0.5,
                "info": D.info()}
print(json.dumps(out))
