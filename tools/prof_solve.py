"""One short device solve for ncu captures: config/size/iterations from argv.

    python tools/prof_solve.py C5 256 3      # 3 GMRES iterations of C5 at 256^3
"""
import pathlib
import sys

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent.parent))

from paper_1308_4605_b200 import problems as PR  # noqa: E402
from paper_1308_4605_b200.krylov import GmresConfig, gmres_solve  # noqa: E402
from paper_1308_4605_b200.precond import PrecondConfig, PrecondKind  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C5"
n = int(sys.argv[2]) if len(sys.argv) > 2 else None
its = int(sys.argv[3]) if len(sys.argv) > 3 else 3
kind = sys.argv[4] if len(sys.argv) > 4 else "P1"
case = PR.make_case(name, n)
cs, rs, spec = PR.prepare(case)
x, h = gmres_solve(rs, cs, PrecondConfig(kind=PrecondKind(kind)),
                   GmresConfig(restart=case.restart, max_iters=its, track_true_residual=False))
print(name, case.grid.cells, "iterations", h.iterations, h.status, h.entries[-1].resid_precond)
