"""Coefficients (host) and the saddle operators (device) -- drop-in mirror.

Mirrors the hot-path surface of the reference's ``stokesmg.operators``
(``/root/reference/pkg/src/stokesmg/operators.py``):

* host-side setup, as in the reference: ``ViscousForm`` (:29), the
  ``CoefficientSet`` container and its validation (:45-78),
  ``make_coefficients`` with cell->face / cell->node/edge averaging
  (:81-125), ``RescaleSpec`` / ``rescale`` (:515-550) and
  ``velocity_null_components`` (:368-388);
* the operators themselves run on the B200 through the C ABI:
  ``apply_M`` (:363), ``apply_A`` (:348, with ``BoundaryValues`` :224),
  ``apply_Lrho`` (:206) and ``homogenize`` (:484);
* ``BoundaryValues`` / ``boundary_lift`` (:224-264, :471): host containers.

Inputs/outputs are the reference's field types (this package's mirror or the
reference's own objects, duck-typed).
"""

from __future__ import annotations

import enum
from dataclasses import dataclass, replace

import numpy as np

from . import _lib
from .grid import (FREE_SLIP, CellField, FaceField, GridSpec, NodeEdgeField, StokesVector,
                   as_grid, edge_planes)


class ViscousForm(enum.Enum):
    LAPLACIAN = "laplacian"
    STRESS = "stress"
    STRESS_BULK = "stress_bulk"


LAPLACIAN = ViscousForm.LAPLACIAN
STRESS = ViscousForm.STRESS
STRESS_BULK = ViscousForm.STRESS_BULK

FORM_CODE = {"laplacian": 0, "stress": 1, "stress_bulk": 2}


def form_code(form) -> int:
    return FORM_CODE[getattr(form, "value", form)]


@dataclass
class CoefficientSet:
    """theta, densities (cell + face), viscosities (cell + node/edge), bulk gamma."""

    theta: float
    rho_cell: CellField
    rho_face: FaceField
    mu_cell: CellField
    mu_node_edge: NodeEdgeField
    gamma_cell: CellField
    viscous_form: ViscousForm = STRESS

    def __post_init__(self):
        if self.theta < 0:
            raise ValueError("theta must be >= 0")
        if self.theta > 0 and (self.rho_cell.data <= 0).any():
            raise ValueError("density must be positive for unsteady flow")
        if (self.mu_cell.data < 0).any():
            raise ValueError("viscosity must be nonnegative")
        if self.theta == 0 and not (self.mu_cell.data > 0).any():
            raise ValueError("steady flow (theta = 0) needs nonzero viscosity")

    @property
    def grid(self) -> GridSpec:
        return self.rho_cell.grid

    @property
    def inviscid(self) -> bool:
        return not (self.mu_cell.data > 0).any()


def _stagger_mean(x: np.ndarray, axis: int, periodic: bool) -> np.ndarray:
    """Arithmetic mean of the two cells adjacent to each staggered position;
    wall positions take the single adjacent cell (operators.py:133-145)."""
    if periodic:
        return 0.5 * (x + np.roll(x, 1, axis=axis))
    lo = np.take(x, [0], axis=axis)
    hi = np.take(x, [-1], axis=axis)
    inner = 0.5 * (np.delete(x, 0, axis=axis) + np.delete(x, -1, axis=axis))
    return np.concatenate([lo, inner, hi], axis=axis)


def average_cell_to_faces(f: CellField) -> FaceField:
    g = f.grid
    return FaceField(g, tuple(_stagger_mean(f.data, a, g.periodic(a)) for a in range(g.dim)))


def average_cell_to_node_edge(f: CellField) -> NodeEdgeField:
    g = f.grid
    out = {}
    for pl in edge_planes(g.dim):
        x = f.data
        for a in pl:
            x = _stagger_mean(x, a, g.periodic(a))
        out[pl] = x
    return NodeEdgeField(g, out)


def make_coefficients(grid, theta, rho_cell, mu_cell, gamma_cell=None, viscous_form=STRESS):
    if gamma_cell is None:
        gamma_cell = CellField.zeros(grid)
    return CoefficientSet(theta=float(theta), rho_cell=rho_cell,
                          rho_face=average_cell_to_faces(rho_cell), mu_cell=mu_cell,
                          mu_node_edge=average_cell_to_node_edge(mu_cell),
                          gamma_cell=gamma_cell, viscous_form=viscous_form)


def velocity_null_components(grid, coeff) -> tuple:
    """Velocity components with a constant null space (steady, periodic axis,
    transverse axes periodic or free-slip)."""
    if coeff.theta > 0:
        return ()
    g = as_grid(grid)
    out = []
    for a in range(g.dim):
        if not g.periodic(a):
            continue
        if all(g.periodic(b) or (g.bc[b][0] is FREE_SLIP and g.bc[b][1] is FREE_SLIP)
               for b in range(g.dim) if b != a):
            out.append(a)
    return tuple(out)


@dataclass(frozen=True)
class RescaleSpec:
    c: float

    def __post_init__(self):
        if not self.c > 0:
            raise ValueError("scale factor must be positive")

    def unscale_solution(self, x):
        return StokesVector(x.u, (1.0 / self.c) * x.p)

    def scale_solution(self, x):
        return StokesVector(x.u, self.c * x.p)


def rescale(coeff, rhs):
    """Scale the velocity rows and the pressure unknowns by c = h / max(mu)."""
    mmax = float(coeff.mu_cell.data.max())
    c = coeff.grid.h / mmax if mmax > 0 else 1.0
    scaled = replace(
        coeff, theta=c * coeff.theta, mu_cell=c * coeff.mu_cell,
        mu_node_edge=NodeEdgeField(coeff.grid, {k: c * v for k, v in coeff.mu_node_edge.arrays.items()}),
        gamma_cell=c * coeff.gamma_cell)
    return scaled, StokesVector(c * rhs.u, rhs.p), RescaleSpec(c)


# ---------------------------------------------------------------------------
# device contexts
# ---------------------------------------------------------------------------


def _f64(a):
    """C-contiguous float64 NumPy array; CUDA/torch tensors pass through (device-resident inputs)."""
    if hasattr(a, "data_ptr") and not isinstance(a, np.ndarray):
        return a
    return np.ascontiguousarray(a, dtype=np.float64)


_POOL: dict = {}


class DeviceContext:
    """One ``sb_ctx``: a grid, its device hierarchy and coefficients.

    Contexts own their HBM (hierarchy, Krylov basis, scratch).  ``acquire`` /
    ``release`` keep idle contexts in a per-(grid, form) pool so repeated
    public ``gmres_solve`` calls reuse the allocations instead of paying
    cudaMalloc every solve (an allocator, not a result cache: coefficients
    are re-uploaded and the hierarchy rebuilt on every use).
    """

    @classmethod
    def acquire(cls, grid, viscous_form=STRESS):
        key = (as_grid(grid), form_code(viscous_form))
        free = _POOL.get(key)
        if free:
            return free.pop()
        return cls(grid, viscous_form)

    def release(self):
        if getattr(self, "h", None):
            _POOL.setdefault((self.grid, self.form), []).append(self)

    def set_stream(self, stream_ptr: int | None):
        _lib.check(self.lib.sb_set_stream(self.h, stream_ptr or None))

    def __init__(self, grid, viscous_form=STRESS):
        import ctypes as C
        self.lib = _lib.load()
        self.grid = as_grid(grid)
        g = self.grid
        cells = (C.c_int * 3)(*g.cells)
        from .grid import BC_CODE
        bcs = (C.c_int * 6)(*[BC_CODE[x] for pair in g.bc for x in pair])
        self.form = form_code(viscous_form)
        h = self.lib.sb_create(g.dim, cells, float(g.h), bcs, self.form)
        if not h:
            raise RuntimeError("sb_create failed: " + (self.lib.sb_last_error() or b"").decode())
        self.h = h
        self.theta = None

    def set_coefficients(self, coeff):
        g = self.grid
        rho = [_f64(c) for c in coeff.rho_face.components]
        mu = _f64(coeff.mu_cell.data)
        edges = [_f64(coeff.mu_node_edge.plane(*pl)) for pl in edge_planes(g.dim)]
        gam = _f64(coeff.gamma_cell.data)
        for a in range(g.dim):
            if rho[a].shape != g.face_shape(a):
                raise ValueError("rho_face layout does not match the grid")
        _lib.check(self.lib.sb_set_coefficients(self.h, float(coeff.theta), _lib.parr(rho),
                                                 _lib.ptr(mu), _lib.parr(edges), _lib.ptr(gam)))
        self.theta = float(coeff.theta)
        self._keep = (rho, mu, edges, gam)

    def set_cell_coefficients(self, theta, rho_cell, mu_cell, gamma_cell=None, scale: float = 1.0):
        """make_coefficients + rescale ON THE DEVICE (sb_set_cell_coefficients):
        only the cell arrays are uploaded; rho_face and the node/edge viscosities
        are averaged on the device and (theta, mu, mu_e, gamma) multiplied by
        ``scale`` -- equal to ``set_coefficients(rescale(make_coefficients(...)))``
        to the bit (operators.py:107-125, :532-550)."""
        g = self.grid
        rho = _f64(getattr(rho_cell, "data", rho_cell))
        mu = _f64(getattr(mu_cell, "data", mu_cell))
        gam = None if gamma_cell is None else _f64(getattr(gamma_cell, "data", gamma_cell))
        for a in (rho, mu) + ((gam,) if gam is not None else ()):
            if tuple(a.shape) != tuple(g.cells):
                raise ValueError("cell array layout does not match the grid")
        _lib.check(self.lib.sb_set_cell_coefficients(self.h, float(theta), _lib.ptr(rho), _lib.ptr(mu),
                                                      _lib.ptr(gam) if gam is not None else None, float(scale)))
        self.theta = float(scale) * float(theta)
        self._keep = (rho, mu, gam)

    def num_levels(self) -> int:
        return self.lib.sb_num_levels(self.h)

    def level_flags(self, level: int = 0) -> int:
        """sb_level_flags: bit 0 derived edge viscosities, bit 1 constant density."""
        return int(self.lib.sb_level_flags(self.h, level))

    def mue_derived(self, level: int = 0) -> bool:
        """True when the face rows of ``level`` derive the edge viscosities from
        mu_cell instead of reading mu_edge (all-periodic levels whose mu_edge is
        the four-cell mean, operators.py:90-104)."""
        return self.level_flags(level) & 1 == 1

    def beta_const(self, level: int = 0) -> bool:
        """True when every non-wall rho_face of ``level`` is one value, so the
        cell rows use a single 1/rho instead of the 1/rho_face arrays."""
        return self.level_flags(level) & 2 == 2

    def level_cells(self, level):
        import ctypes as C
        out = (C.c_int * 3)()
        _lib.check(self.lib.sb_level_cells(self.h, level, out))
        return tuple(out[: self.grid.dim])

    def close(self):
        if getattr(self, "h", None):
            self.lib.sb_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def _ctx_for(coeff, grid=None) -> DeviceContext:
    ctx = DeviceContext(grid if grid is not None else coeff.grid, coeff.viscous_form)
    ctx.set_coefficients(coeff)
    return ctx


def _out_face(grid):
    return [np.zeros(grid.face_shape(a)) for a in range(grid.dim)]


def apply_M(x, coeff, ctx: DeviceContext | None = None) -> StokesVector:
    """Saddle operator (A u + G p, -D u) on the device (operators.py:363-365)."""
    g = as_grid(x.u.grid)
    ctx = ctx or _ctx_for(coeff, g)
    ou, op = _out_face(g), np.zeros(g.cells)
    u = [_f64(c) for c in x.u.components]
    _lib.check(ctx.lib.sb_apply_M(ctx.h, _lib.parr(u), _lib.ptr(_f64(x.p.data)), _lib.parr(ou), _lib.ptr(op)))
    return StokesVector(FaceField(g, tuple(ou)), CellField(g, op))


def _tangential_ptrs(bvals, g):
    """BoundaryValues.tangential -> the 18 plane pointers of sb_apply_A_affine
    (index (axis*2 + side)*3 + comp); shapes checked as the reference does."""
    keep, ptrs = [], [None] * 18
    for (axis, side, comp) in sorted(bvals.tangential):
        v = _f64(bvals.tangential_values(axis, side, comp))
        keep.append(v)
        ptrs[(axis * 2 + side) * 3 + comp] = v
    return keep, _lib.parr(ptrs)


def apply_A(u, coeff, bvals=None, ctx: DeviceContext | None = None) -> FaceField:
    """Velocity operator theta rho u - L_mu u on the device (operators.py:348-360).

    Wall-normal boundary faces of ``u`` are read as given (a boundary lift);
    ``bvals`` adds the prescribed tangential wall velocities (operators.py:267-291)."""
    g = as_grid(u.grid)
    ctx = ctx or _ctx_for(coeff, g)
    ou = _out_face(g)
    uu = _lib.parr([_f64(c) for c in u.components])
    if bvals is None:
        _lib.check(ctx.lib.sb_apply_A(ctx.h, uu, _lib.parr(ou)))
    else:
        keep, tp = _tangential_ptrs(bvals, g)
        _lib.check(ctx.lib.sb_apply_A_affine(ctx.h, uu, tp, _lib.parr(ou)))
    return FaceField(g, tuple(ou))


# ---------------------------------------------------------------------------
# inhomogeneous walls (operators.py:224-264, 471-512)
# ---------------------------------------------------------------------------


@dataclass
class BoundaryValues:
    """Prescribed wall velocities (operators.py:224-264).

    ``normal[(axis, side)]``: the normal component on that wall's boundary
    faces (the component array with its own axis dropped).
    ``tangential[(axis, side, comp)]``: the ``comp`` velocity on the wall plane
    of ``(axis, side)`` (the ``comp`` array with ``axis`` dropped).  Missing
    entries are zero; ``side`` is 0 (low) or 1 (high)."""

    grid: GridSpec
    normal: dict
    tangential: dict

    @classmethod
    def zeros(cls, grid) -> "BoundaryValues":
        return cls(grid, {}, {})

    def normal_values(self, axis: int, side: int) -> np.ndarray:
        shape = tuple(n for a, n in enumerate(self.grid.cells) if a != axis)
        vals = self.normal.get((axis, side))
        if vals is None:
            return np.zeros(shape)
        vals = np.asarray(vals, dtype=np.float64)
        if vals.shape != shape:
            raise ValueError(f"normal values for axis {axis} must have shape {shape}")
        return vals

    def tangential_values(self, axis: int, side: int, comp: int) -> np.ndarray:
        shape = tuple(n for a, n in enumerate(self.grid.face_shape(comp)) if a != axis)
        vals = self.tangential.get((axis, side, comp))
        if vals is None:
            return np.zeros(shape)
        vals = np.asarray(vals, dtype=np.float64)
        if vals.shape != shape:
            raise ValueError(f"tangential values for (axis {axis}, comp {comp}) must have shape {shape}")
        return vals


def boundary_lift(bvals) -> FaceField:
    """FaceField holding the prescribed normal values on the boundary faces
    (operators.py:471-481; array assembly, no arithmetic)."""
    g = as_grid(bvals.grid)
    u = FaceField.zeros(g)
    for a in range(g.dim):
        if g.periodic(a):
            continue
        arr = u.components[a]
        lo = [slice(None)] * g.dim
        hi = [slice(None)] * g.dim
        lo[a], hi[a] = 0, -1
        arr[tuple(lo)] = bvals.normal_values(a, 0)
        arr[tuple(hi)] = bvals.normal_values(a, 1)
    return u


def homogenize(bvals, coeff, rhs, ctx: DeviceContext | None = None) -> StokesVector:
    """Subtract the affine boundary contribution from the right-hand side on the
    device (operators.py:484-512): (rhs.u - A(u_b; bvals), rhs.p + div u_b).
    Raises ValueError ('incompatible boundary data ...') when the net boundary
    flux does not match the divergence source carried in ``rhs.p``."""
    g = as_grid(rhs.u.grid)
    ctx = ctx or _ctx_for(coeff, g)
    keep_n, nptr = [], [None] * 6
    for (axis, side) in sorted(bvals.normal):
        v = _f64(bvals.normal_values(axis, side))
        keep_n.append(v)
        nptr[axis * 2 + side] = v
    keep_t, tp = _tangential_ptrs(bvals, g)
    ou, op = _out_face(g), np.zeros(g.cells)
    _lib.check(ctx.lib.sb_homogenize(ctx.h, _lib.parr(nptr), tp,
                                     _lib.parr([_f64(c) for c in rhs.u.components]),
                                     _lib.ptr(_f64(rhs.p.data)), _lib.parr(ou), _lib.ptr(op)))
    return StokesVector(FaceField(g, tuple(ou)), CellField(g, op))


def apply_Lrho(p, coeff, ctx: DeviceContext | None = None) -> CellField:
    """Density-weighted Poisson operator D rho^-1 G on the device (operators.py:206-215)."""
    g = as_grid(p.grid)
    ctx = ctx or _ctx_for(coeff, g)
    out = np.zeros(g.cells)
    _lib.check(ctx.lib.sb_apply_Lrho(ctx.h, _lib.ptr(_f64(p.data)), _lib.ptr(out)))
    return CellField(g, out)


# ---------------------------------------------------------------------------
# the reference's remaining public operators (operators.py:182-203, :303-345,
# :396-439), on the device
# ---------------------------------------------------------------------------


class _Geometry:
    """A pooled coefficient-free context for the geometry-only operators."""

    def __init__(self, grid):
        self.ctx = DeviceContext.acquire(as_grid(grid), STRESS)

    def __enter__(self):
        return self.ctx

    def __exit__(self, *exc):
        self.ctx.release()


def div(u) -> CellField:
    """Cell-centred divergence (operators.py:182-188); reads the stored boundary
    faces.  Bit-identical to the reference: ((d0 + d1) + d2) / h."""
    g = as_grid(u.grid)
    out = np.zeros(g.cells)
    with _Geometry(g) as ctx:
        _lib.check(ctx.lib.sb_div(ctx.h, _lib.parr([_f64(c) for c in u.components]), _lib.ptr(out)))
    return CellField(g, out)


def grad(p) -> FaceField:
    """Face-centred pressure gradient, wall-normal faces zero (operators.py:191-198)."""
    g = as_grid(p.grid)
    out = _out_face(g)
    with _Geometry(g) as ctx:
        _lib.check(ctx.lib.sb_grad(ctx.h, _lib.ptr(_f64(p.data)), _lib.parr(out)))
    return FaceField(g, tuple(out))


def lap_pressure(p) -> CellField:
    """Scalar pressure Laplacian, exactly div(grad(p)) (operators.py:201-203)."""
    g = as_grid(p.grid)
    out = np.zeros(g.cells)
    with _Geometry(g) as ctx:
        _lib.check(ctx.lib.sb_lap_pressure(ctx.h, _lib.ptr(_f64(p.data)), _lib.ptr(out)))
    return CellField(g, out)


def apply_viscous(u, coeff, bvals=None) -> FaceField:
    """Discrete viscous term L_mu u in the coefficient set's form
    (operators.py:303-345): the device's A row with theta = 0, negated
    (A u = theta rho u - L_mu u, wall-normal rows 0); ``bvals`` as apply_A."""
    g = as_grid(u.grid)
    c0 = CoefficientSet.__new__(CoefficientSet)
    c0.__dict__.update(coeff.__dict__)
    c0.theta = 0.0  # the viscous part alone (no validation: an inviscid set stays usable)
    a = apply_A(u, c0, bvals)
    return FaceField(g, tuple(-x for x in a.components))


def helmholtz_diagonal(grid, coeff) -> FaceField:
    """Diagonal of A = theta rho - L_mu, boundary faces one (operators.py:408-439),
    as the device smoother computes it in registers."""
    g = as_grid(grid)
    ctx = _ctx_for(coeff, g)
    out = _out_face(g)
    _lib.check(ctx.lib.sb_diagonal(ctx.h, _lib.KIND_FACE, 0, _lib.parr(out)))
    return FaceField(g, tuple(out))


def lrho_diagonal(grid, coeff) -> CellField:
    """Diagonal of D (1/rho) G, wall faces carry no flux (operators.py:396-405)."""
    g = as_grid(grid)
    ctx = _ctx_for(coeff, g)
    out = np.zeros(g.cells)
    _lib.check(ctx.lib.sb_diagonal(ctx.h, _lib.KIND_CELL, 0, _lib.parr([out])))
    return CellField(g, out)
