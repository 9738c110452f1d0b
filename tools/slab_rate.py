"""Per-iteration device time of ONE rank's slab as the slab gets thinner: the
compute side of strong scaling, measured on one GPU.

For P in 256, 128, 64, 32 planes the recipe (C4 or C5) is built on the box
P x 256 x 256 and solved through the slab path with one slab and the 1-rank
NCCL communicator (the kernels, ghost planes, graph and NCCL calls of a rank
at N = 256 / P; the global problem is periodic over P planes instead of 256,
so iteration counts differ -- only the time PER ITERATION is reported).

    python tools/slab_rate.py C4 [iters=20]
"""
import json
import pathlib
import sys

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent.parent))

import torch  # noqa: E402

from paper_1308_4605_b200 import problems as PR  # noqa: E402
from paper_1308_4605_b200.dist import DistSolver  # noqa: E402
from paper_1308_4605_b200.krylov import GmresConfig  # noqa: E402
from paper_1308_4605_b200.precond import P1, PrecondConfig  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C4"
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 20
rows = []
for planes in (256, 128, 64, 32):
    case = PR.make_case(name, (planes, 256, 256))
    cs, rs, _ = PR.prepare(case)
    D = DistSolver(case.grid, cs.viscous_form, nslab=1, nccl_self=True)
    D.set_coefficients(cs)
    gcfg = GmresConfig(restart=case.restart, max_iters=iters, rtol=1e-30, atol=0.0, track_true_residual=False)
    pc = PrecondConfig(kind=P1)
    dev = torch.device("cuda", 0)
    T = lambda a: torch.from_numpy(a).to(dev)
    drhs = type("R", (), {})()
    drhs.u = type("U", (), {"components": [T(x) for x in rs.u.components]})()
    drhs.p = type("P", (), {"data": T(rs.p.data)})()
    out = ([torch.zeros_like(c) for c in drhs.u.components], torch.zeros_like(drhs.p.data))
    D.local_inputs = True
    stream = torch.cuda.ExternalStream(D.stream_ptr(), device=dev)
    D.gmres_solve(drhs, pc, gcfg, out=out)  # warm: graph capture
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    _, _, h = D.gmres_solve(drhs, pc, gcfg, out=out)
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    rows.append({"planes": planes, "ranks_equiv": 256 // planes, "iterations": h.iterations,
                 "ms_per_iteration": ms / max(h.iterations, 1), "info": D.info()})
    del D, drhs, out
    torch.cuda.empty_cache()
t1 = rows[0]["ms_per_iteration"]
for r in rows:
    r["compute_efficiency_vs_256_planes"] = t1 / (r["ranks_equiv"] * r["ms_per_iteration"])
print(json.dumps({"config": name, "rows": rows}))
