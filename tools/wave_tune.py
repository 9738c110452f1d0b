"""Tune the wavefront sweeps (sb_wave.cu) on C5 256^3: per-launch device time of
the finest-level face sweeps (one component sweep per launch with the wave,
one colour pass per launch without) for SB_WAVE_K x SB_WAVE_CTAS."""
import os
import pathlib
import sys

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent.parent))
from paper_1308_4605_b200 import operators  # noqa: E402
from paper_1308_4605_b200 import problems as PR  # noqa: E402
from paper_1308_4605_b200.krylov import GmresConfig, gmres_solve  # noqa: E402
from paper_1308_4605_b200.precond import PrecondConfig, PrecondKind, Preconditioner  # noqa: E402

case = PR.make_case("C5", int(sys.argv[1]) if len(sys.argv) > 1 else 256)
cs, rs, spec = PR.prepare(case)
import itertools  # noqa: E402
grid = [x.split(",") for x in (sys.argv[2:] or [])]
configs = [("0", "2", "4", "256")] + [("64",) + t for t in itertools.product(*grid)] if grid else \
    [("0", "2", "4", "256")] + [("64", k, c, f) for k in ("8", "16") for c in ("4", "6") for f in ("512", "1024")]
for wmin, k, ctas, faces in configs:
    os.environ.update(SB_WAVE_MIN=wmin, SB_WAVE_K=k, SB_WAVE_CTAS=ctas, SB_WAVE_FACES=faces)
    operators._POOL.clear()
    P = Preconditioner(cs, PrecondConfig(kind=PrecondKind.P1))
    P.set_profiling(True)
    x, h = gmres_solve(rs, cs, None, GmresConfig(restart=50, max_iters=3, track_true_residual=False), precond=P)
    st = P.kernel_stats()
    us = 1e3 * st["fine_face_ms"] / max(st["fine_face_launches"], 1)
    per_sweep = us * (1 if wmin != "0" else 2)
    print(f"wave_min={wmin} K={k} ctas/SM={ctas} faces/item={faces}: fine face {us:.1f} us/launch -> {per_sweep:.1f} us per "
          f"component sweep; all face {st['smoother_face_ms']:.2f} ms, cell {st['smoother_cell_ms']:.2f} ms", flush=True)
    del P
