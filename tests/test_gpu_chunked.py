"""Chunked red/black sweep ordering (SB_CHUNK_MB, sb_solver.cu make_level):
the colour passes of a large level cut into axis-0 plane chunks and
interleaved R0 R1 B0 R2 B1 ... so black re-reads red's operands from L2.
Red reads only black (old) neighbours and black only red (relaxed) ones, so
the result is bit-identical to the two full colour passes."""

from __future__ import annotations

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name,n,kind", [("C5", 64, "P1"), ("C4", 64, "P1"), ("C3", 64, "P2")])
def test_chunked_sweeps_bit_identical(name, n, kind, monkeypatch):
    from paper_1308_4605_b200 import problems as PR
    from paper_1308_4605_b200.krylov import GmresConfig, gmres_solve
    from paper_1308_4605_b200.precond import PrecondConfig, PrecondKind, Preconditioner
    case = PR.make_case(name, n)
    cs, rs, _ = PR.prepare(case)
    pc = PrecondConfig(kind=PrecondKind(kind))
    gcfg = GmresConfig(restart=case.restart, max_iters=60, rtol=1e-9, track_true_residual=False)
    out = {}
    for mb in ("0", "0.4"):  # 0.4 MB: 2-3 plane chunks on the 64^3 and 32^3 levels
        monkeypatch.setenv("SB_CHUNK_MB", mb)
        P = Preconditioner(cs, pc)
        y = P.apply(rs)
        x, h = gmres_solve(rs, cs, pc, gcfg, precond=P)
        out[mb] = (y, x, h)
    (y0, x0, h0), (y1, x1, h1) = out["0"], out["0.4"]
    for a in range(3):
        assert np.array_equal(y0.u.components[a], y1.u.components[a]), a
        assert np.array_equal(x0.u.components[a], x1.u.components[a]), a
    assert np.array_equal(y0.p.data, y1.p.data)
    assert np.array_equal(x0.p.data, x1.p.data)
    assert h0.rows() == h1.rows()
