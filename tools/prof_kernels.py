"""Each device kernel class once at the finest level of a config (ncu captures).

    python tools/prof_kernels.py C5 256
Order of kernel launches (after setup): 6 face colour passes (one sweep),
2 cell colour passes, 3 face residual->restrict, 1 cell residual->restrict,
3 face prolong+add, 1 cell prolong+add, 1 apply_M, then a 1-iteration GMRES
(norms, CGS2 multi_dot / update_dot x2, P^-1 graph).
"""
import pathlib
import sys

import numpy as np

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent.parent))

from paper_1308_4605_b200 import multigrid as MG  # noqa: E402
from paper_1308_4605_b200 import operators as OPS  # noqa: E402
from paper_1308_4605_b200 import problems as PR  # noqa: E402
from paper_1308_4605_b200.grid import CellField, FaceField  # noqa: E402
from paper_1308_4605_b200.krylov import GmresConfig, gmres_solve  # noqa: E402
from paper_1308_4605_b200.precond import PrecondConfig, PrecondKind, Preconditioner  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C5"
n = int(sys.argv[2]) if len(sys.argv) > 2 else None
case = PR.make_case(name, n)
cs, rs, spec = PR.prepare(case)
g = case.grid
P = Preconditioner(cs, PrecondConfig(kind=PrecondKind.P1))
hier = MG.MgHierarchy(P.ctx, cs)
rng = np.random.default_rng(0)
x = FaceField(g, tuple(rng.standard_normal(g.face_shape(a)) for a in range(g.dim)))
y = CellField(g, rng.standard_normal(g.cells))
MG.smooth(hier, 0, "face", x, rs.u)
MG.smooth(hier, 0, "cell", y, rs.p)
MG.residual_restrict(hier, 0, "face", x, rs.u)
MG.residual_restrict(hier, 0, "cell", y, rs.p)
gc = g.coarsened()
MG.prolong_add(hier, 0, "face", FaceField.zeros(gc), x)
MG.prolong_add(hier, 0, "cell", CellField.zeros(gc), y)
OPS.apply_M(rs, cs, ctx=P.ctx)
xs, h = gmres_solve(rs, cs, None, GmresConfig(restart=case.restart, max_iters=1, track_true_residual=False),
                    precond=P)
print("ok", h.iterations)
