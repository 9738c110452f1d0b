"""CPU-side checks: the C-ABI library loads and exports every declared symbol;
host-side mirror logic (grid, packing, coefficient averaging, rescale, configs,
input generators) matches the oracle / reference semantics.  No GPU needed."""

from __future__ import annotations

import re

import numpy as np
import pytest

from conftest import ROOT, cases, oracle_coef, oracle_geo, pkg_grid, relerr


def test_library_exports_every_header_symbol(lib):
    from paper_1308_4605_b200 import _lib
    header = (ROOT / "include" / "stokesb200.h").read_text()
    declared = set(re.findall(r"\b(sb_[a-z_A-Z]+)\s*\(", header))
    assert declared == set(_lib.EXPORTS)
    for name in declared:
        assert hasattr(lib, name), name


def test_library_is_sm100a():
    import subprocess
    so = ROOT / "paper_1308_4605_b200" / "libstokesb200.so"
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", str(so)],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_no_oracle_import_in_product():
    for p in (ROOT / "paper_1308_4605_b200").rglob("*.py"):
        src = p.read_text()
        assert "import oracle" not in src and "from oracle" not in src, p


@pytest.mark.parametrize("e", cases("operators")[:8], ids=lambda e: e["name"])
def test_make_coefficients_matches_oracle_bitwise(e):
    from paper_1308_4605_b200.grid import CellField
    from paper_1308_4605_b200.operators import ViscousForm, make_coefficients
    from oracle import stokes_oracle as O
    g = pkg_grid(e)
    geo = oracle_geo(e)
    rng = np.random.default_rng(7)
    rho, mu = 0.5 + rng.random(g.cells), 0.5 + rng.random(g.cells)
    c = make_coefficients(g, 0.3, CellField(g, rho), CellField(g, mu), None, ViscousForm.STRESS)
    oc = O.make_coef(geo, 0.3, rho, mu)
    for a in range(g.dim):
        assert np.array_equal(c.rho_face.components[a], oc.rho_face[a])
    for k, v in oc.mu_edge.items():
        assert np.array_equal(c.mu_node_edge.arrays[k], v)


def test_pack_unpack_fortran_order():
    from paper_1308_4605_b200.grid import (NO_SLIP, PERIODIC, GridSpec, StokesVector, pack_stokes,
                                           unpack_stokes)
    from oracle import stokes_oracle as O
    g = GridSpec((4, 6), 0.25, ((PERIODIC, PERIODIC), (NO_SLIP, NO_SLIP)))
    v = np.arange(g.n_unknowns(), dtype=float)
    x = unpack_stokes(g, v)
    assert np.array_equal(pack_stokes(x), v)
    geo = O.Geo((4, 6), 0.25, (("periodic",) * 2, ("no_slip",) * 2))
    u, p = O.unpack(geo, v)
    for a in range(2):
        assert np.array_equal(u[a], x.u.components[a])
    assert np.array_equal(p, x.p.data)
    assert x.u.components[1][:, 0].sum() == 0 and x.u.components[1][:, -1].sum() == 0


def test_grid_validation_and_hierarchy_depths():
    from paper_1308_4605_b200.grid import NO_SLIP, PERIODIC, GridSpec
    with pytest.raises(ValueError):
        GridSpec((4, 4), 1.0, ((PERIODIC, NO_SLIP), (PERIODIC, PERIODIC)))
    with pytest.raises(ValueError):
        GridSpec((1, 4), 1.0, ((PERIODIC, PERIODIC),) * 2)
    g = GridSpec((48, 48), 1.0, ((NO_SLIP, NO_SLIP),) * 2)
    depth = [g.cells]
    while g.can_coarsen():
        g = g.coarsened()
        depth.append(g.cells)
    assert depth[-1] == (3, 3)


def test_config_validation():
    from paper_1308_4605_b200 import GmresConfig, PrecondConfig, SchurConfig, SmootherParams
    with pytest.raises(ValueError):
        SmootherParams(omega=0.0)
    with pytest.raises(ValueError):
        SmootherParams(bottom_sweeps=4)
    with pytest.raises(ValueError):
        GmresConfig(restart=0)
    with pytest.raises(ValueError):
        GmresConfig(rtol=0.0)
    with pytest.raises(ValueError):
        PrecondConfig(velocity_cycles=0)
    with pytest.raises(ValueError):
        SchurConfig(pressure_cycles=0)
    assert GmresConfig().restart == 10 and GmresConfig().track_true_residual


def test_coefficient_validation():
    from paper_1308_4605_b200.grid import PERIODIC, CellField, GridSpec
    from paper_1308_4605_b200.operators import make_coefficients
    g = GridSpec((4, 4), 1.0, ((PERIODIC, PERIODIC),) * 2)
    one, zero = CellField.full(g, 1.0), CellField.zeros(g)
    with pytest.raises(ValueError):
        make_coefficients(g, -1.0, one, one)
    with pytest.raises(ValueError):
        make_coefficients(g, 0.0, one, zero)  # steady needs viscosity
    with pytest.raises(ValueError):
        make_coefficients(g, 1.0, CellField.full(g, -1.0), one)


def test_rescale_matches_oracle():
    from paper_1308_4605_b200 import problems as PR
    from oracle import stokes_oracle as O
    case = PR.make_case("C2", 32)
    cs, rs, spec = PR.prepare(case)
    g = case.grid
    geo = O.Geo(g.cells, g.h, tuple((lo.value, hi.value) for lo, hi in g.bc))
    oc = O.Coef(case.coeff.theta, case.coeff.rho_cell.data, list(case.coeff.rho_face.components),
                case.coeff.mu_cell.data, dict(case.coeff.mu_node_edge.arrays),
                case.coeff.gamma_cell.data)
    sc, su, sp, c = O.rescale(geo, oc, list(case.rhs.u.components), case.rhs.p.data)
    assert c == spec.c
    assert cs.theta == sc.theta
    assert np.array_equal(cs.mu_cell.data, sc.mu_cell)
    for a in range(2):
        assert np.array_equal(rs.u.components[a], su[a])


@pytest.mark.parametrize("name,n", [("C1", 16), ("C2", 16), ("C3", 8), ("C4", 8), ("C5", 8)])
def test_generators_deterministic_and_well_posed(name, n):
    from paper_1308_4605_b200 import problems as PR
    a, b = PR.make_case(name, n), PR.make_case(name, n)
    assert np.array_equal(a.coeff.mu_cell.data, b.coeff.mu_cell.data)
    assert np.array_equal(a.rhs.p.data, b.rhs.p.data)
    for k in range(a.grid.dim):
        assert np.array_equal(a.rhs.u.components[k], b.rhs.u.components[k])
        if not a.grid.periodic(k):
            assert not a.rhs.u.interior(k).size == 0
    if a.steady_periodic:
        assert abs(a.rhs.p.data.mean()) < 1e-12
        for k in range(a.grid.dim):
            assert abs(a.rhs.u.components[k].mean()) < 1e-12
    mu = a.coeff.mu_cell.data
    if name in ("C3", "C5"):
        span = 4.0 if name == "C3" else 3.0
        assert mu.min() == pytest.approx(1.0) and mu.max() == pytest.approx(10 ** span)


def test_device_entry_fails_loudly_without_gpu():
    """No CPU fallback: on a machine without a CUDA device the device API raises."""
    from conftest import gpu_available
    if gpu_available():
        pytest.skip("GPU present")
    from paper_1308_4605_b200 import problems as PR
    from paper_1308_4605_b200.operators import apply_M
    case = PR.make_case("C1", 8)
    with pytest.raises(RuntimeError):
        apply_M(case.rhs, case.coeff)
