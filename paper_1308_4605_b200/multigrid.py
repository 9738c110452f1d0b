"""Geometric multigrid on the device -- drop-in mirror of ``stokesmg.multigrid``.

Reference: ``/root/reference/pkg/src/stokesmg/multigrid.py``.  ``SmootherParams``
(:33-46) is the same frozen dataclass; ``build_hierarchy`` (:92-104) builds the
coefficient hierarchy ON THE DEVICE (coarsening kernels, :127-169) and returns
an ``MgHierarchy`` whose ``levels`` are downloaded lazily for inspection;
``vcycle`` (:391) / ``mg_solve`` (:442) run the fused sm_100a smoother,
residual->restriction and prolongation kernels.  The component-level entry
points (``smooth``, ``residual_restrict``, ``prolong_add``) exist for the
parity tests.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _lib
from .grid import CellField, FaceField, NodeEdgeField, as_grid, edge_planes
from .operators import CoefficientSet, DeviceContext, _f64


@dataclass(frozen=True)
class SmootherParams:
    omega: float = 1.0
    sweeps_down: int = 2
    sweeps_up: int = 2
    bottom_sweeps: int = 8

    def __post_init__(self):
        if not 0 < self.omega <= 1:
            raise ValueError("omega must lie in (0, 1]")
        if self.sweeps_down < 1 or self.sweeps_up < 1:
            raise ValueError("need at least one smoothing sweep each way")
        if self.bottom_sweeps < 8:
            raise ValueError("bottom level needs at least 8 relaxations")

    def as_c(self):
        return _lib.Smoother(float(self.omega), int(self.sweeps_down), int(self.sweeps_up),
                             int(self.bottom_sweeps))


def smoother_c(p) -> _lib.Smoother:
    p = p if p is not None else SmootherParams()
    return _lib.Smoother(float(p.omega), int(p.sweeps_down), int(p.sweeps_up), int(p.bottom_sweeps))


class MgHierarchy:
    """Device-resident grids + coarsened coefficients, finest first."""

    def __init__(self, ctx: DeviceContext, coeff):
        self.ctx = ctx
        self.coeff = coeff
        self._levels = None

    @property
    def grid(self):
        return self.ctx.grid

    def __len__(self):
        return self.ctx.num_levels()

    @property
    def levels(self):
        """[(GridSpec, CoefficientSet)] downloaded from the device (inspection only)."""
        if self._levels is None:
            out = []
            g = self.grid
            for l in range(len(self)):
                if l > 0:
                    g = g.coarsened()
                rho = [np.zeros(g.face_shape(a)) for a in range(g.dim)]
                mu = np.zeros(g.cells)
                gam = np.zeros(g.cells)
                edges = [np.zeros(g.node_edge_shape(pl)) for pl in edge_planes(g.dim)]
                _lib.check(self.ctx.lib.sb_get_level_coefficients(
                    self.ctx.h, l, _lib.parr(rho), _lib.ptr(mu), _lib.parr(edges), _lib.ptr(gam)))
                rho_cell = self.coeff.rho_cell.data
                for _ in range(l):  # rho_cell is not used on the device; coarsen on host
                    rho_cell = _pair_mean_all(rho_cell)
                coef = CoefficientSet.__new__(CoefficientSet)
                coef.theta = self.coeff.theta
                coef.rho_cell = CellField(g, rho_cell)
                coef.rho_face = FaceField(g, tuple(rho))
                coef.mu_cell = CellField(g, mu)
                coef.mu_node_edge = NodeEdgeField(g, dict(zip(edge_planes(g.dim), edges)))
                coef.gamma_cell = CellField(g, gam)
                coef.viscous_form = self.coeff.viscous_form
                out.append((g, coef))
            self._levels = out
        return self._levels

    def diag_face(self, level: int) -> FaceField:
        """The velocity smoother's diagonal on ``level`` (multigrid.py:79-89);
        ZeroDivisionError on a zero interior entry, as the reference."""
        g = _level_grid(self, level)
        out = [np.zeros(g.face_shape(a)) for a in range(g.dim)]
        _lib.check(self.ctx.lib.sb_diagonal(self.ctx.h, _lib.KIND_FACE, int(level), _lib.parr(out)))
        d = FaceField(g, tuple(out))
        for a in range(g.dim):
            if np.any(d.interior(a) == 0):
                raise ZeroDivisionError("zero diagonal in velocity operator (theta = 0 with mu = 0 row)")
        return d

    def diag_cell(self, level: int) -> CellField:
        """The pressure smoother's diagonal on ``level`` (multigrid.py:70-77)."""
        g = _level_grid(self, level)
        out = np.zeros(g.cells)
        _lib.check(self.ctx.lib.sb_diagonal(self.ctx.h, _lib.KIND_CELL, int(level), _lib.parr([out])))
        if np.any(out == 0):
            raise ZeroDivisionError("zero diagonal in pressure operator")
        return CellField(g, out)


def _pair_mean_all(x):
    for a in range(x.ndim):
        sl0 = [slice(None)] * x.ndim
        sl1 = [slice(None)] * x.ndim
        sl0[a], sl1[a] = slice(0, None, 2), slice(1, None, 2)
        x = 0.5 * (x[tuple(sl0)] + x[tuple(sl1)])
    return x


def build_hierarchy(grid, coeff) -> MgHierarchy:
    g = as_grid(grid)
    if not g.can_coarsen():
        raise ValueError(f"grid {g.cells} cannot be coarsened; need even counts >= 4")
    ctx = DeviceContext(g, coeff.viscous_form)
    ctx.set_coefficients(coeff)
    return MgHierarchy(ctx, coeff)


def _kind(kind):
    if kind not in ("cell", "face"):
        raise ValueError("kind must be 'cell' or 'face'")
    return _lib.KIND_CELL if kind == "cell" else _lib.KIND_FACE


def _arrays(field, kind):
    return [_f64(field.data)] if kind == "cell" else [_f64(c) for c in field.components]


def _wrap(grid, arrs, kind):
    return CellField(grid, arrs[0]) if kind == "cell" else FaceField(grid, tuple(arrs))


def _zeros(grid, kind):
    return [np.zeros(grid.cells)] if kind == "cell" else [np.zeros(grid.face_shape(a)) for a in range(grid.dim)]


def mg_solve(rhs, hierarchy: MgHierarchy, params, n_cycles: int, kind: str):
    """n V-cycles from a zero guess (multigrid.py:442-460), on the device."""
    k = _kind(kind)
    if n_cycles < 1:
        raise ValueError("need at least one cycle")
    g = hierarchy.grid
    out = _zeros(g, kind)
    ctx = hierarchy.ctx
    _lib.check(ctx.lib.sb_mg_solve(ctx.h, k, C.byref(smoother_c(params)), int(n_cycles),
                                   _lib.parr(_arrays(rhs, kind)), _lib.parr(out)))
    return _wrap(g, out, kind)


def vcycle(rhs, hierarchy: MgHierarchy, params, kind: str):
    """One residual-correction V-cycle from zero (multigrid.py:391-400)."""
    return mg_solve(rhs, hierarchy, params, 1, kind)


def _level_grid(hierarchy, level):
    g = hierarchy.grid
    for _ in range(level):
        g = g.coarsened()
    return g


def smooth(hierarchy: MgHierarchy, level: int, kind: str, x, rhs, omega: float = 1.0):
    """One GS sweep in place on ``level`` (multigrid.py:318-340); returns x."""
    k = _kind(kind)
    xs = _arrays(x, kind)
    ctx = hierarchy.ctx
    _lib.check(ctx.lib.sb_smooth(ctx.h, k, int(level), float(omega), _lib.parr(xs),
                                 _lib.parr(_arrays(rhs, kind))))
    if kind == "cell":
        x.data[...] = xs[0]
    else:
        for a, arr in enumerate(xs):
            x.components[a][...] = arr
    return x


def residual_restrict(hierarchy: MgHierarchy, level: int, kind: str, x, rhs):
    """restrict(rhs - Op x) onto level+1 (multigrid.py:403-406, :177-233)."""
    k = _kind(kind)
    gc = _level_grid(hierarchy, level + 1)
    out = _zeros(gc, kind)
    ctx = hierarchy.ctx
    _lib.check(ctx.lib.sb_residual_restrict(ctx.h, k, int(level), _lib.parr(_arrays(x, kind)),
                                            _lib.parr(_arrays(rhs, kind)), _lib.parr(out)))
    return _wrap(gc, out, kind)


def prolong_add(hierarchy: MgHierarchy, level: int, kind: str, coarse, fine):
    """fine + prolong(coarse) (multigrid.py:185-192, :282-295, :431-436)."""
    k = _kind(kind)
    fs = _arrays(fine, kind)
    fs = [f.copy() for f in fs]
    ctx = hierarchy.ctx
    _lib.check(ctx.lib.sb_prolong_add(ctx.h, k, int(level), _lib.parr(_arrays(coarse, kind)),
                                      _lib.parr(fs)))
    return _wrap(_level_grid(hierarchy, level), fs, kind)


# ---------------------------------------------------------------------------
# the reference's public transfer / coarsening / smoother functions
# (multigrid.py:127-295, :318-340) with their signatures, on the device
# ---------------------------------------------------------------------------


def _transfer_ctx(grid):
    g = as_grid(grid)
    if any(n % 2 for n in g.cells):
        raise ValueError(f"cannot restrict odd cell counts {g.cells}")
    from .operators import _Geometry
    geo = _Geometry(g)
    if geo.ctx.num_levels() < 2:
        geo.ctx.release()
        raise ValueError(f"grid {g.cells} cannot be coarsened on the device; need even counts >= 4")
    return geo


def restrict_cell(fine: CellField) -> CellField:
    """Mean of the 2^d children (multigrid.py:177-182), bit-identical."""
    g = as_grid(fine.grid)
    with _transfer_ctx(g) as ctx:
        gc = g.coarsened()
        out = [np.zeros(gc.cells)]
        _lib.check(ctx.lib.sb_restrict(ctx.h, _lib.KIND_CELL, 0, _lib.parr([_f64(fine.data)]), _lib.parr(out)))
    return CellField(gc, out[0])


def restrict_face(fine: FaceField) -> FaceField:
    """Staggered restriction: tangential pair means, normal [1/4, 1/2, 1/4];
    coarse wall faces 0 (multigrid.py:195-233), bit-identical."""
    g = as_grid(fine.grid)
    with _transfer_ctx(g) as ctx:
        gc = g.coarsened()
        out = [np.zeros(gc.face_shape(a)) for a in range(g.dim)]
        _lib.check(ctx.lib.sb_restrict(ctx.h, _lib.KIND_FACE, 0, _lib.parr([_f64(c) for c in fine.components]),
                                       _lib.parr(out)))
    return FaceField(gc, tuple(out))


def _fine_of(gc):
    from .grid import GridSpec
    return GridSpec(tuple(2 * n for n in gc.cells), gc.h / 2, gc.bc)


def prolong_cell(coarse: CellField) -> CellField:
    """Injection into the 2^d children (multigrid.py:185-192)."""
    gf = _fine_of(as_grid(coarse.grid))
    with _transfer_ctx(gf) as ctx:
        out = [np.zeros(gf.cells)]
        _lib.check(ctx.lib.sb_prolong(ctx.h, _lib.KIND_CELL, 0, _lib.parr([_f64(coarse.data)]), _lib.parr(out)))
    return CellField(gf, out[0])


def prolong_face(coarse: FaceField) -> FaceField:
    """Staggered prolongation: tangential 3/4-1/4 (walls clamp), normal copy /
    average (multigrid.py:236-295).  Wall-normal boundary faces are not
    unknowns: they come back 0 (SURVEY §8b field convention)."""
    gf = _fine_of(as_grid(coarse.grid))
    with _transfer_ctx(gf) as ctx:
        out = [np.zeros(gf.face_shape(a)) for a in range(gf.dim)]
        _lib.check(ctx.lib.sb_prolong(ctx.h, _lib.KIND_FACE, 0, _lib.parr([_f64(c) for c in coarse.components]),
                                      _lib.parr(out)))
    return FaceField(gf, tuple(out))


def coarsen_coefficients(coeff, coarse_grid) -> CoefficientSet:
    """One level of coefficient coarsening (multigrid.py:127-169), by the
    device's coarsening kernels; rho_cell by the device cell restriction."""
    from .operators import _ctx_for
    g = as_grid(coeff.rho_cell.grid)
    gc = as_grid(coarse_grid)
    if gc != g.coarsened():
        raise ValueError(f"coarse grid {gc.cells} is not the coarsening of {g.cells}")
    ctx = _ctx_for(coeff, g)
    if ctx.num_levels() < 2:
        raise ValueError(f"grid {g.cells} cannot be coarsened; need even counts >= 4")
    rho = [np.zeros(gc.face_shape(a)) for a in range(gc.dim)]
    mu = np.zeros(gc.cells)
    gam = np.zeros(gc.cells)
    edges = [np.zeros(gc.node_edge_shape(pl)) for pl in edge_planes(gc.dim)]
    _lib.check(ctx.lib.sb_get_level_coefficients(ctx.h, 1, _lib.parr(rho), _lib.ptr(mu), _lib.parr(edges),
                                                 _lib.ptr(gam)))
    out = CoefficientSet.__new__(CoefficientSet)
    out.theta = coeff.theta
    out.rho_cell = CellField(gc, restrict_cell(coeff.rho_cell).data)
    out.rho_face = FaceField(gc, tuple(rho))
    out.mu_cell = CellField(gc, mu)
    out.mu_node_edge = NodeEdgeField(gc, dict(zip(edge_planes(gc.dim), edges)))
    out.gamma_cell = CellField(gc, gam)
    out.viscous_form = coeff.viscous_form
    return out


def _smooth_level0(kind, x, rhs, grid, coeff, omega):
    from .operators import _ctx_for
    ctx = _ctx_for(coeff, grid)
    k = _kind(kind)
    xs = _arrays(x, kind)
    _lib.check(ctx.lib.sb_smooth(ctx.h, k, 0, float(omega), _lib.parr(xs), _lib.parr(_arrays(rhs, kind))))
    if kind == "cell":
        x.data[...] = xs[0]
    else:
        for a, arr in enumerate(xs):
            x.components[a][...] = arr


def smooth_cell(phi: CellField, rhs: CellField, grid, coeff, diag: CellField, omega: float) -> None:
    """One red-black GS sweep of the pressure operator, in place (multigrid.py:318-324).
    ``diag`` is the operator's diagonal (lrho_diagonal) as every reference caller
    passes; the device recomputes it in registers."""
    _smooth_level0("cell", phi, rhs, as_grid(grid), coeff, omega)


def smooth_face(u: FaceField, rhs: FaceField, grid, coeff, diag: FaceField, omega: float) -> None:
    """One 2d-colour GS sweep of the velocity operator, in place (multigrid.py:327-340).
    ``diag``: helmholtz_diagonal (recomputed in registers on the device)."""
    _smooth_level0("face", u, rhs, as_grid(grid), coeff, omega)
