"""Shared fixtures: golden vectors (made by the reference, tests/golden/make_golden.py)
loaded into both the oracle's array types and the package's field types."""

from __future__ import annotations

import json
import pathlib
import sys

import numpy as np
import pytest

ROOT = pathlib.Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

GOLD = ROOT / "tests" / "golden"
BCNAME = {"p": "periodic", "n": "no_slip", "f": "free_slip"}


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built libstokesb200.so")
    config.addinivalue_line("markers", "slow: longer-running parity case")


_cache = {}


def golden():
    if "z" not in _cache:
        _cache["z"] = np.load(GOLD / "golden.npz")
        _cache["idx"] = json.loads((GOLD / "golden.json").read_text())
    return _cache["z"], _cache["idx"]


def cases(kind):
    _, idx = golden()
    return [e for e in idx if e["kind"] == kind]


def arr(name, key):
    z, _ = golden()
    return np.array(z[f"{name}/{key}"])


def face(name, key, dim):
    return [arr(name, f"{key}{a}") for a in range(dim)]


def planes(dim):
    return ((0, 1),) if dim == 2 else ((0, 1), (0, 2), (1, 2))


# ---- oracle side --------------------------------------------------------------


def oracle_geo(e):
    from oracle.stokes_oracle import Geo
    return Geo(tuple(e["cells"]), float(e["h"]), tuple((BCNAME[b[0]], BCNAME[b[1]]) for b in e["bc"]))


def oracle_coef(e, prefix=None):
    from oracle.stokes_oracle import Coef
    n = prefix or e["name"]
    d = len(e["cells"])
    return Coef(float(e["theta"]), arr(n, "rho_cell"), face(n, "rho_face", d), arr(n, "mu_cell"),
                {pl: arr(n, f"mu_edge{pl[0]}{pl[1]}") for pl in planes(d)}, arr(n, "gamma_cell"),
                e["form"])


# ---- package side ----------------------------------------------------------------


def pkg_grid(e):
    from paper_1308_4605_b200.grid import BoundaryCondition, GridSpec
    return GridSpec(tuple(e["cells"]), float(e["h"]),
                    tuple((BoundaryCondition(BCNAME[b[0]]), BoundaryCondition(BCNAME[b[1]])) for b in e["bc"]))


def pkg_coeff(e, prefix=None, grid=None):
    from paper_1308_4605_b200.grid import CellField, FaceField, NodeEdgeField
    from paper_1308_4605_b200.operators import CoefficientSet, ViscousForm
    n = prefix or e["name"]
    g = grid or pkg_grid(e)
    d = g.dim
    return CoefficientSet(
        theta=float(e["theta"]), rho_cell=CellField(g, arr(n, "rho_cell")),
        rho_face=FaceField(g, tuple(face(n, "rho_face", d))), mu_cell=CellField(g, arr(n, "mu_cell")),
        mu_node_edge=NodeEdgeField(g, {pl: arr(n, f"mu_edge{pl[0]}{pl[1]}") for pl in planes(d)}),
        gamma_cell=CellField(g, arr(n, "gamma_cell")), viscous_form=ViscousForm(e["form"]))


def relerr(a, b):
    a = np.asarray(a)
    b = np.asarray(b)
    s = max(np.abs(b).max(), 1e-300)
    return float(np.abs(a - b).max() / s)


def gpu_available():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.fixture(scope="session")
def lib():
    from paper_1308_4605_b200 import _lib
    return _lib.load()


def golden_bvals(e):
    """(normal {(axis, side): plane}, tangential {(axis, side, comp): plane}) of an affine case."""
    n = e["name"]
    normal = {(int(k[0]), int(k[1])): arr(n, f"bn{k}") for k in e["normal"]}
    tang = {(int(k[0]), int(k[1]), int(k[2])): arr(n, f"bt{k}") for k in e["tangential"]}
    return normal, tang
