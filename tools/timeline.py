"""Device timeline of one solve (CUPTI via torch.profiler): time by activity
kind (kernels, memcpy, memset) and the idle gaps between activities.

    python tools/timeline.py C5 256 [dist] [iters]

`dist` runs the slab-decomposed path with one slab (self-exchange copies),
otherwise the single-domain path.  Prints a JSON summary; writes the raw
per-activity list to gpurun_out/timeline_<mode>.json.
"""
import collections
import json
import pathlib
import sys

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent.parent))

import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

from paper_1308_4605_b200 import problems as PR  # noqa: E402
from paper_1308_4605_b200.krylov import GmresConfig, gmres_solve  # noqa: E402
from paper_1308_4605_b200.precond import P1, PrecondConfig  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C5"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 256
mode = sys.argv[3] if len(sys.argv) > 3 else "single"
iters = int(sys.argv[4]) if len(sys.argv) > 4 else 10
case = PR.make_case(name, n)
cs, rs, _ = PR.prepare(case)
gcfg = GmresConfig(restart=case.restart, max_iters=iters, rtol=1e-9, track_true_residual=False)
pc = PrecondConfig(kind=P1)
if mode == "dist":
    from paper_1308_4605_b200.dist import DistSolver
    D = DistSolver(case.grid, cs.viscous_form, nslab=1)
    D.set_coefficients(cs)
    run = lambda: D.gmres_solve(rs, pc, gcfg)
else:
    from paper_1308_4605_b200.precond import Preconditioner
    P = Preconditioner(cs, pc)
    run = lambda: gmres_solve(rs, cs, None, gcfg, precond=P)
run()  # warm: graphs captured
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    run()
    torch.cuda.synchronize()
acts = []
for e in prof.events():
    if e.device_type.name != "CUDA":
        continue
    acts.append((e.time_range.start, e.time_range.end, e.name))
acts.sort()
kind = collections.Counter()
tot = collections.defaultdict(float)
for s, t, nm in acts:
    k = "memcpy" if "Memcpy" in nm or "memcpy" in nm else ("memset" if "Memset" in nm or "memset" in nm
                                                         else ("nccl" if "nccl" in nm else "kernel"))
    kind[k] += 1
    tot[k] += (t - s)
# union of busy intervals -> idle time
busy = 0.0
cur_s, cur_e = None, None
for s, t, _ in acts:
    if cur_e is None or s > cur_e:
        if cur_e is not None:
            busy += cur_e - cur_s
        cur_s, cur_e = s, t
    else:
        cur_e = max(cur_e, t)
if cur_e is not None:
    busy += cur_e - cur_s
span = acts[-1][1] - acts[0][0] if acts else 0
out = {"mode": mode, "cells": list(case.grid.cells), "iters": iters, "span_ms": span / 1e3, "busy_ms": busy / 1e3,
       "idle_ms": (span - busy) / 1e3, "count": dict(kind), "ms": {k: v / 1e3 for k, v in tot.items()}}
print(json.dumps(out))
pathlib.Path("gpurun_out").mkdir(exist_ok=True)
pathlib.Path(f"gpurun_out/timeline_{mode}.json").write_text(json.dumps(
    [(s, t, nm) for s, t, nm in acts]))
