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

The bubble problem (``BubbleSpec``, ``bubble_profile``, ``bubble_coefficients``,
``bubble_density``, ``inviscid_coefficients``, ``make_rhs``) is a DELIBERATE
restatement of the reference's ``problems.py:36-135``: the reference's tests,
presets and driver goldens feed these exact inputs, so the generator must
replay the same Philox draws and formulas to be bit-identical on the host.  It
is input generation, off the device path.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from .grid import NO_SLIP, PERIODIC, CellField, FaceField, GridSpec, NodeEdgeField, StokesVector
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


def c5_cells(n_gpus: int):
    """C5 weak scaling at h = 1/512: 256^3 per GPU (1 GPU 256^3,
    2 GPUs 512x256x256, 4 GPUs 512x512x256, 8 GPUs 512^3)."""
    return {1: (256, 256, 256), 2: (512, 256, 256), 4: (512, 512, 256), 8: (512, 512, 512)}.get(
        n_gpus, (256 * n_gpus, 256, 256))


def make_c5_slab(cells, nranks: int, rank: int, seed: int = 1308, reduce=None):
    """This rank's axis-0 planes of the C5 recipe on the global box `cells`
    (h = 1/512), generated without materialising the global fields.

    The log-viscosity Fourier field is evaluated on the rank's planes plus one
    plane each side (for the face / edge averages); its global min/max comes
    from `reduce(local_min, local_max) -> (gmin, gmax)` (torch.distributed in
    the bench).  Forces and divergence source draw from per-rank Philox streams
    and get their global means removed through `reduce` as well
    (`reduce(sum, count)`).  Returns (grid, coeff, rhs) with rank-local arrays;
    coefficient/rhs arrays hold exactly the rank's planes."""
    from .grid import FaceField
    grid = GridSpec(tuple(cells), 1.0 / 512, _bc("ppp"))
    n0 = cells[0] // nranks
    lo = rank * n0
    s_coef = streams(seed)[0]
    # modes: identical on every rank (same stream)
    modes = []
    for _ in range(8):
        while True:
            k = s_coef.integers(-4, 5, size=3)
            if np.any(k != 0):
                break
        modes.append((k, s_coef.uniform(0.0, 2.0 * np.pi)))
    L = grid.lengths
    xs = [(np.arange(n) + 0.5) * grid.h for n in cells]
    x0 = (np.arange(lo - 1, lo + n0 + 1) + 0.5) * grid.h  # one extra plane each side (periodic field)
    F = np.zeros((n0 + 2, cells[1], cells[2]))
    for k, phi in modes:
        arg = phi + (2 * np.pi * k[0] / L[0]) * x0[:, None, None] + \
            (2 * np.pi * k[1] / L[1]) * xs[1][None, :, None] + (2 * np.pi * k[2] / L[2]) * xs[2][None, None, :]
        F += np.cos(arg)
    fmin, fmax = reduce("minmax", float(F[1:-1].min()), float(F[1:-1].max()))
    mu_ext = 10.0 ** (3.0 * (F - fmin) / (fmax - fmin))
    mu = mu_ext[1:-1]
    # face / edge averages along axis 0 use the neighbour plane below (periodic)
    rho_f = [np.ones((n0, cells[1], cells[2])) for _ in range(3)]
    from .operators import _stagger_mean, CoefficientSet
    mu0 = 0.5 * (mu_ext[1:-1] + mu_ext[:-2])          # staggered along axis 0
    e01 = _stagger_mean(mu0, 1, True)                   # edges (0,1)
    e02 = _stagger_mean(mu0, 2, True)                   # edges (0,2)
    e12 = _stagger_mean(_stagger_mean(mu, 1, True), 2, True)
    local = GridSpec((n0, cells[1], cells[2]), grid.h, grid.bc)
    coeff = CoefficientSet.__new__(CoefficientSet)
    coeff.theta = 0.0
    coeff.rho_cell = CellField(local, np.ones((n0, cells[1], cells[2])))
    coeff.rho_face = FaceField(local, tuple(rho_f))
    coeff.mu_cell = CellField(local, mu)
    coeff.mu_node_edge = NodeEdgeField(local, {(0, 1): e01, (0, 2): e02, (1, 2): e12})
    coeff.gamma_cell = CellField.zeros(local)
    coeff.viscous_form = STRESS
    gens = [np.random.Generator(np.random.Philox(s)) for s in np.random.SeedSequence([seed, rank]).spawn(4)]
    f = [gens[1].standard_normal((n0, cells[1], cells[2])) for _ in range(3)]
    gsrc = gens[2].standard_normal((n0, cells[1], cells[2]))
    cnt = float(np.prod(cells))
    for a in range(3):
        f[a] -= reduce("sum", float(f[a].sum()), 0.0)[0] / cnt
    gsrc -= reduce("sum", float(gsrc.sum()), 0.0)[0] / cnt
    # rescale (operators.py:532-550): c = h / max(mu) over the GLOBAL field
    mmax = reduce("minmax", float(mu.min()), float(mu.max()))[1]
    c = grid.h / mmax
    coeff.mu_cell = CellField(local, c * mu)
    coeff.mu_node_edge = NodeEdgeField(local, {k: c * v for k, v in coeff.mu_node_edge.arrays.items()})
    rhs = StokesVector(FaceField(local, tuple(c * x for x in f)), CellField(local, -gsrc))
    return grid, coeff, rhs, c


# ---------------------------------------------------------------------------
# the paper's bubble problem (reference problems.py:36-135, 170-199), used by
# the acceptance criteria (tests/test_gpu_acceptance.py)
# ---------------------------------------------------------------------------


@dataclass(frozen=True)
class BubbleSpec:
    """Smoothed sphere/disk: (r+1)/2 + (r-1)/2 tanh(d/eps) + noise_amp * U(0,1)."""

    r_mu: float = 100.0
    r_rho: float = 100.0
    epsilon: float | None = None
    radius: float | None = None
    noise_amp: float = 0.1
    seed: int = 0
    positive_outside: bool = True

    def __post_init__(self):
        if self.r_mu < 1 or self.r_rho < 1:
            raise ValueError("contrast ratios must be >= 1")
        if self.epsilon is not None and not self.epsilon > 0:
            raise ValueError("smoothing width must be positive")


def bubble_profile(grid, r, spec, noise):
    xs = grid.cell_centers()
    centre = [0.5 * L for L in grid.lengths]
    radius = spec.radius if spec.radius is not None else 0.25 * max(grid.lengths)
    eps = spec.epsilon if spec.epsilon is not None else grid.h
    d = np.sqrt(sum((x - c) ** 2 for x, c in zip(xs, centre))) - radius
    if not spec.positive_outside:
        d = -d
    f = 0.5 * (r + 1.0) + 0.5 * (r - 1.0) * np.tanh(d / eps)
    if noise is not None:
        f = f + spec.noise_amp * noise
    return f


def bubble_coefficients(grid, spec, theta=0.0, viscous_form=STRESS, mu0=1.0, rho0=1.0, gamma0=0.0):
    g_mu, g_rho = streams(spec.seed, 2)
    n_mu = g_mu.random(grid.cells) if spec.noise_amp else None
    n_rho = g_rho.random(grid.cells) if spec.noise_amp else None
    mu = CellField(grid, mu0 * bubble_profile(grid, spec.r_mu, spec, n_mu))
    rho = CellField(grid, rho0 * bubble_profile(grid, spec.r_rho, spec, n_rho))
    gam = CellField.full(grid, gamma0) if gamma0 else CellField.zeros(grid)
    return make_coefficients(grid, theta, rho, mu, gam, viscous_form)


def bubble_density(grid, spec, rho0=1.0):
    _, g_rho = streams(spec.seed, 2)
    noise = g_rho.random(grid.cells) if spec.noise_amp else None
    return CellField(grid, rho0 * bubble_profile(grid, spec.r_rho, spec, noise))


def inviscid_coefficients(grid, rho_cell, theta=1.0):
    from .operators import CoefficientSet, average_cell_to_faces, average_cell_to_node_edge
    zero = CellField.zeros(grid)
    return CoefficientSet(theta=theta, rho_cell=rho_cell, rho_face=average_cell_to_faces(rho_cell),
                          mu_cell=zero, mu_node_edge=average_cell_to_node_edge(zero),
                          gamma_cell=CellField.zeros(grid), viscous_form=STRESS)


def project_nulls(x, coeff):
    from .operators import velocity_null_components
    out = x.copy()
    out.p.data -= out.p.data.mean()
    for a in velocity_null_components(x.grid, coeff):
        v = out.u.interior(a)
        v -= v.mean()
    return out


def make_rhs(grid, coeff, seed=0):
    """Random consistent rhs = M x_exact with x_exact drawn in the unknown space
    (M applied on the device)."""
    from .grid import norm2
    from .operators import apply_M
    for gen in streams(seed, 4):
        x = StokesVector.zeros(grid)
        for a in range(grid.dim):
            v = x.u.interior(a)
            v[...] = gen.standard_normal(v.shape)
        x.p.data[...] = gen.standard_normal(grid.cells)
        x = project_nulls(x, coeff)
        if norm2(x) > 1e-8 * math.sqrt(grid.n_unknowns()):
            return apply_M(x, coeff), x
    raise RuntimeError("could not draw a nondegenerate solution")
