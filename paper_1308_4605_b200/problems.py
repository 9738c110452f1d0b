"""Seeded synthetic inputs for the BASELINE configurations C1..C5 (host side).

There is no public dataset for this path; BASELINE.json names five synthetic
configurations and SURVEY.md §8(d) fixes the recipes, which this module
implements.  Inputs are generated once on the host (NumPy, Philox streams
spawned from ``np.random.SeedSequence(seed)`` as the reference's
``problems._generators`` does, ``problems.py:31-33``) and the same arrays are
fed to the device solve and to the CPU oracle.

Conventions: domain [0,1]^d, h = 1/n; rhs u = f on unknown faces,
rhs p = -g (M's second row is -D u, ``operators.py:365``); for fully periodic
steady cases each f component's mean is removed; ``rescale`` is applied
(``cli.py:340-343``) by ``prepare``.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from .grid import NO_SLIP, PERIODIC, CellField, FaceField, GridSpec, StokesVector
from .operators import STRESS, make_coefficients, rescale


@dataclass(frozen=True)
class CflSpec:
    """Viscous CFL number beta = mu0 / (theta rho0 h^2) (problems.py:138-158)."""

    beta: float

    def __post_init__(self):
        if self.beta < 0:
            raise ValueError("viscous CFL number must be >= 0")

    @property
    def steady(self):
        return math.isinf(self.beta)

    @property
    def inviscid(self):
        return self.beta == 0.0


def cfl_to_theta(spec: CflSpec, mu0: float, rho0: float, h: float) -> float:
    if spec.steady:
        return 0.0
    if spec.inviscid:
        return 1.0
    return mu0 / (spec.beta * rho0 * h * h)


def constant_coefficients(grid, mu0=1.0, rho0=1.0, theta=0.0, viscous_form=STRESS, gamma0=0.0):
    gam = CellField.full(grid, gamma0) if gamma0 else CellField.zeros(grid)
    return make_coefficients(grid, theta, CellField.full(grid, rho0), CellField.full(grid, mu0),
                             gam, viscous_form)


def streams(seed: int, k: int = 4):
    return [np.random.Generator(np.random.Philox(s)) for s in np.random.SeedSequence(int(seed)).spawn(k)]


def _axes(grid):
    return [(np.arange(n) + 0.5) * grid.h for n in grid.cells]


def fourier_log_mu(grid, rng, span_decades: float, n_modes: int = 8, kmax: int = 4):
    """log10 mu = span (F - min F)/(max F - min F), F = sum_m cos(2 pi k_m.x/L + phi_m)."""
    xs = _axes(grid)
    L = grid.lengths
    F = np.zeros(grid.cells)
    for _ in range(n_modes):
        while True:
            k = rng.integers(-kmax, kmax + 1, size=grid.dim)
            if np.any(k != 0):
                break
        phi = rng.uniform(0.0, 2.0 * np.pi)
        arg = phi
        for a in range(grid.dim):
            shape = [1] * grid.dim
            shape[a] = grid.cells[a]
            arg = arg + (2.0 * np.pi * k[a] / L[a]) * xs[a].reshape(shape)
        F += np.cos(arg)
    F = (F - F.min()) / (F.max() - F.min())
    return 10.0 ** (span_decades * F)


def tanh_bump(grid):
    xs = np.meshgrid(*_axes(grid), indexing="ij")
    r = np.sqrt(sum((x - 0.5) ** 2 for x in xs))
    return 0.5 * (1.0 + np.tanh((0.1 - r) / 0.02))


def sphere_mask(grid, rng, count=64, radius=0.05):
    """Cells whose centre lies inside any of `count` random spheres; minimum
    image on periodic axes (only the bounding box of each sphere is visited)."""
    mask = np.zeros(grid.cells, dtype=bool)
    xs = _axes(grid)
    centres = rng.random((count, grid.dim)) * np.array(grid.lengths)
    h = grid.h
    for c in centres:
        idx, d2 = [], 0.0
        for a in range(grid.dim):
            n = grid.cells[a]
            lo = int(math.floor((c[a] - radius) / h)) - 1
            hi = int(math.ceil((c[a] + radius) / h)) + 1
            ii = np.arange(lo, hi + 1)
            if grid.periodic(a):
                ii = np.unique(ii % n)
            else:
                ii = ii[(ii >= 0) & (ii < n)]
            dx = xs[a][ii] - c[a]
            if grid.periodic(a):
                Lw = grid.lengths[a]
                dx = dx - Lw * np.round(dx / Lw)
            shape = [1] * grid.dim
            shape[a] = len(ii)
            d2 = d2 + (dx ** 2).reshape(shape)
            idx.append(ii)
        inside = d2 <= radius * radius
        mask[np.ix_(*idx)] |= inside
    return mask


def random_forces(grid, rng, remove_mean: bool):
    f = FaceField.zeros(grid)
    for a in range(grid.dim):
        v = f.interior(a)
        v[...] = rng.standard_normal(v.shape)
        if remove_mean:
            v -= v.mean()
    return f


@dataclass
class Case:
    name: str
    grid: GridSpec
    coeff: object
    rhs: StokesVector
    restart: int

    @property
    def steady_periodic(self):
        return self.coeff.theta == 0 and all(self.grid.periodic(a) for a in range(self.grid.dim))


def _bc(spec):
    return tuple((PERIODIC, PERIODIC) if s == "p" else (NO_SLIP, NO_SLIP) for s in spec)


def make_case(name: str, n: int | tuple | None = None, seed: int = 1308) -> Case:
    """Build config ``name`` (C1..C5) at its BASELINE size, or at ``n`` cells/axis."""
    s_coef, s_f, s_g, _ = streams(seed)
    if name == "C1":
        cells = (n or 64,) * 2 if not isinstance(n, tuple) else n
        g = GridSpec(cells, 1.0 / cells[0], _bc("pp"))
        coeff = constant_coefficients(g)
        restart = 30
    elif name == "C2":
        cells = (n or 256,) * 2 if not isinstance(n, tuple) else n
        g = GridSpec(cells, 1.0 / cells[0], _bc("pw"))
        b = tanh_bump(g)
        theta = cfl_to_theta(CflSpec(10.0), 1.0, 1.0, g.h)
        coeff = make_coefficients(g, theta, CellField(g, 1.0 + 99.0 * b), CellField(g, 1.0 + 999.0 * b))
        restart = 30
    elif name in ("C3", "C5"):
        default = 128 if name == "C3" else 256
        cells = (n or default,) * 3 if not isinstance(n, tuple) else n
        # C5 is the weak-scaling sweep at h = 1/512 (1 GPU: the 256^3 sub-box of [0,1]^3)
        h = 1.0 / max(cells) if name == "C3" else (1.0 / 512 if n is None else 0.5 / max(cells))
        g = GridSpec(cells, h, _bc("ppp"))
        span = 4.0 if name == "C3" else 3.0
        mu = fourier_log_mu(g, s_coef, span)
        coeff = make_coefficients(g, 0.0, CellField.full(g, 1.0), CellField(g, mu))
        restart = 50
    elif name == "C4":
        cells = (n or 256,) * 3 if not isinstance(n, tuple) else n
        g = GridSpec(cells, 1.0 / cells[0], _bc("ppw"))
        m = sphere_mask(g, s_coef)
        rho = np.where(m, 100.0, 1.0)
        mu = np.where(m, 1.0e3, 1.0)
        theta = cfl_to_theta(CflSpec(1.0), 1.0, 1.0, g.h)
        coeff = make_coefficients(g, theta, CellField(g, rho), CellField(g, mu))
        restart = 30
    else:
        raise ValueError(f"unknown config {name}")
    steady_per = coeff.theta == 0 and all(g.periodic(a) for a in range(g.dim))
    f = random_forces(g, s_f, remove_mean=steady_per)
    if name in ("C2", "C4"):
        gsrc = np.zeros(g.cells)
    else:
        gsrc = s_g.standard_normal(g.cells)
        gsrc -= gsrc.mean()
    rhs = StokesVector(f, CellField(g, -gsrc))
    return Case(name, g, coeff, rhs, restart)


def prepare(case: Case):
    """Apply ``rescale`` as the reference CLI does; returns (coeff', rhs', spec)."""
    return rescale(case.coeff, case.rhs)
