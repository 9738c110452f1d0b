"""Time the phases of one public gmres_solve call from pinned host arrays (C5 256^3)."""
import pathlib
import sys
import time

import numpy as np
import torch

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent.parent))
from paper_1308_4605_b200 import problems as PR  # noqa: E402
from paper_1308_4605_b200.grid import CellField, FaceField, NodeEdgeField, StokesVector  # noqa: E402
from paper_1308_4605_b200.krylov import GmresConfig, gmres_solve, solve_raw  # noqa: E402
from paper_1308_4605_b200.operators import CoefficientSet  # noqa: E402
from paper_1308_4605_b200.precond import P1, PrecondConfig, Preconditioner  # noqa: E402

case = PR.make_case("C5")
cs, rs, spec = PR.prepare(case)
g = case.grid


def pinned(a):
    t = torch.empty(a.shape, dtype=torch.float64, pin_memory=True)
    t.numpy()[...] = a
    return t.numpy()


hc = CoefficientSet.__new__(CoefficientSet)
hc.theta, hc.viscous_form = cs.theta, cs.viscous_form
hc.rho_cell = CellField(g, cs.rho_cell.data)
hc.rho_face = FaceField(g, tuple(pinned(c) for c in cs.rho_face.components))
hc.mu_cell = CellField(g, pinned(cs.mu_cell.data))
hc.mu_node_edge = NodeEdgeField(g, {k: pinned(v) for k, v in cs.mu_node_edge.arrays.items()})
hc.gamma_cell = CellField(g, pinned(cs.gamma_cell.data))
hr = StokesVector(FaceField(g, tuple(pinned(c) for c in rs.u.components)), CellField(g, pinned(rs.p.data)))
gcfg = GmresConfig(restart=50, max_iters=500, rtol=1e-9, track_true_residual=False)
pc = PrecondConfig(kind=P1)
from paper_1308_4605_b200 import _lib  # noqa: E402
a = pinned(np.ones(g.cells))
d = torch.empty(g.cells, dtype=torch.float64, device="cuda")
for _ in range(2):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    d.copy_(torch.from_numpy(a), non_blocking=True)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    torch.from_numpy(a).copy_(d, non_blocking=True)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
print(f"PCIe: H2D {a.nbytes / (t1 - t0) / 1e9:.1f} GB/s, D2H {a.nbytes / (t2 - t1) / 1e9:.1f} GB/s (pinned, 134 MB)")
for rep in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    P = Preconditioner(hc, pc)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    xu = [_lib.pinned.array(g.face_shape(a)) for a in range(3)]
    xp = _lib.pinned.array(g.cells)
    t2 = time.perf_counter()
    h = solve_raw(P, gcfg, [c for c in hr.u.components], hr.p.data, xu, xp)
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    x, h2 = gmres_solve(hr, hc, pc, gcfg)
    t4 = time.perf_counter()
    del P
    print(f"precond(setup) {1e3*(t1-t0):.1f} ms, alloc out {1e3*(t2-t1):.1f} ms, solve_raw {1e3*(t3-t2):.1f} ms,"
          f" full gmres_solve {1e3*(t4-t3):.1f} ms, its {h.iterations}")
