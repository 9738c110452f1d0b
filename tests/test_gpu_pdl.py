"""Programmatic dependent launch: launching the solve's kernels
with programmatic stream serialization must not change a single bit.  The
switch (SB_PDL) is read once per process, so each arm runs in a subprocess;
solutions, histories and V-cycle counts must be identical."""

from __future__ import annotations

import os
import pathlib
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = pathlib.Path(__file__).resolve().parent.parent

SCRIPT = r"""
import sys, numpy as np
sys.path.insert(0, sys.argv[1])
from paper_1308_4605_b200 import problems as PR
from paper_1308_4605_b200.grid import pack_stokes
from paper_1308_4605_b200.krylov import GmresConfig, gmres_solve
from paper_1308_4605_b200.precond import PrecondConfig, PrecondKind
out = {}
for name, n, kind in (("C5", 64, "P1"), ("C4", 32, "P1"), ("C2", 64, "P2"), ("C3", 32, "P3")):
    case = PR.make_case(name, n)
    cs, rs, spec = PR.prepare(case)
    x, h = gmres_solve(rs, cs, PrecondConfig(kind=PrecondKind(kind)),
                       GmresConfig(restart=case.restart, max_iters=500, rtol=1e-9, track_true_residual=True))
    out[name + "_x"] = pack_stokes(x)
    out[name + "_h"] = np.array(h.rows(), dtype=float)
np.savez(sys.argv[2], **out)
"""


def _run(tmp_path, pdl):
    f = tmp_path / f"pdl{pdl}.npz"
    env = dict(os.environ, SB_PDL=str(pdl))
    subprocess.run([sys.executable, "-c", SCRIPT, str(ROOT), str(f)], env=env, check=True, timeout=600)
    return np.load(f)


def test_pdl_bit_identical(tmp_path):
    a, b = _run(tmp_path, 0), _run(tmp_path, 1)
    assert sorted(a.files) == sorted(b.files)
    for k in a.files:
        assert np.array_equal(a[k], b[k], equal_nan=True), k
