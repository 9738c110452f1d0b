"""CPU oracle for the preconditioned MAC Stokes solve -- TEST INFRASTRUCTURE ONLY.

This module is the checker, never the product: only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py`` (its ``cpu_baseline`` leg and the
``--impl reference`` arm) may import it.  The product path
(``paper_1308_4605_b200``) never imports it and fails loudly when its CUDA
library is missing.

It is a NumPy restatement of the reference package ``stokesmg`` 0.1.0
(``/root/reference/pkg/src/stokesmg``) for the hot path named by
``BASELINE.json:north_star``: restarted left-preconditioned GMRES on the MAC
saddle system, preconditioned by P1..P5 with one geometric-multigrid V-cycle
per velocity / pressure subproblem.  Every function cites the reference
``file:line`` it restates.  Floating-point operation order follows the
reference (divisions by ``h``, sums in axis order) so that the oracle agrees
with the reference to a few ulp; ``tests/test_oracle_golden.py`` pins it
against golden vectors produced by the reference itself
(``tests/golden/make_golden.py``).

Arrays follow the reference's C-order layout: cells ``geo.cells``; face
component ``a`` has ``n_a + 1`` entries along ``a`` on a wall axis
(``grid.py:84-89``); node/edge arrays are staggered in two axes
(``grid.py:91-97``).  Boundary conditions are the strings ``"periodic"``,
``"no_slip"``, ``"free_slip"``.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

PER, NOSLIP, FREESLIP = "periodic", "no_slip", "free_slip"
LAPLACIAN, STRESS, STRESS_BULK = "laplacian", "stress", "stress_bulk"


# ---------------------------------------------------------------------------
# geometry (grid.py:40-132)
# ---------------------------------------------------------------------------


@dataclass(frozen=True)
class Geo:
    cells: tuple
    h: float
    bc: tuple  # ((lo, hi), ...) per axis

    @property
    def dim(self):
        return len(self.cells)

    def per(self, a):
        return self.bc[a][0] == PER

    def fshape(self, a):  # grid.py:84
        s = list(self.cells)
        s[a] += 0 if self.per(a) else 1
        return tuple(s)

    def eshape(self, axes):  # grid.py:91
        s = list(self.cells)
        for a in axes:
            s[a] += 0 if self.per(a) else 1
        return tuple(s)

    def inner(self, a):  # grid.py:99 -- unknown entries of component a
        return tuple(slice(1, -1) if (b == a and not self.per(a)) else slice(None)
                     for b in range(self.dim))

    def coarsenable(self):  # grid.py:121
        return all(n % 2 == 0 and n >= 4 for n in self.cells)

    def half(self):  # grid.py:124
        return Geo(tuple(n // 2 for n in self.cells), 2.0 * self.h, self.bc)

    def double(self):
        return Geo(tuple(2 * n for n in self.cells), self.h / 2.0, self.bc)

    def n_unknowns(self):  # grid.py:115
        tot = int(np.prod(self.cells))
        for a in range(self.dim):
            c = list(self.cells)
            if not self.per(a):
                c[a] -= 1
            tot += int(np.prod(c))
        return tot


def planes(dim):  # grid.py:229 edge_planes
    return ((0, 1),) if dim == 2 else ((0, 1), (0, 2), (1, 2))


def _ax(nd, axis, what):
    s = [slice(None)] * nd
    s[axis] = what
    return tuple(s)


# ---------------------------------------------------------------------------
# staggered difference / averaging primitives (operators.py:133-174)
# ---------------------------------------------------------------------------


def up_minus_here(x, axis, periodic):
    """x[i+1] - x[i]: staggered -> centered (operators.py:154-158)."""
    if periodic:
        return np.roll(x, -1, axis=axis) - x
    return np.diff(x, axis=axis)


def here_minus_down(x, axis, periodic):
    """x[i] - x[i-1]: centered -> staggered, wall rows 0 (operators.py:161-169)."""
    if periodic:
        return x - np.roll(x, 1, axis=axis)
    shp = list(x.shape)
    shp[axis] += 1
    out = np.zeros(shp)
    out[_ax(x.ndim, axis, slice(1, -1))] = np.diff(x, axis=axis)
    return out


def to_stagger_mean(x, axis, periodic):
    """0.5 (x[i-1] + x[i]); wall rows copy the adjacent cell (operators.py:133-145)."""
    if periodic:
        return 0.5 * (x + np.roll(x, 1, axis=axis))
    shp = list(x.shape)
    shp[axis] += 1
    out = np.zeros(shp)
    lo = x[_ax(x.ndim, axis, slice(None, -1))]
    hi = x[_ax(x.ndim, axis, slice(1, None))]
    out[_ax(x.ndim, axis, slice(1, -1))] = 0.5 * (hi + lo)
    out[_ax(x.ndim, axis, 0)] = x[_ax(x.ndim, axis, 0)]
    out[_ax(x.ndim, axis, -1)] = x[_ax(x.ndim, axis, -1)]
    return out


def zero_ends(x, axis):
    x[_ax(x.ndim, axis, 0)] = 0.0
    x[_ax(x.ndim, axis, -1)] = 0.0


# ---------------------------------------------------------------------------
# coefficients (operators.py:45-125, 515-550)
# ---------------------------------------------------------------------------


@dataclass
class Coef:
    theta: float
    rho_cell: np.ndarray
    rho_face: list
    mu_cell: np.ndarray
    mu_edge: dict  # (a, b) sorted -> array
    gamma_cell: np.ndarray
    form: str = STRESS

    def edge(self, a, b):
        return self.mu_edge[(min(a, b), max(a, b))]


def make_coef(geo, theta, rho_cell, mu_cell, gamma_cell=None, form=STRESS):
    """operators.py:107-125 (averaging :81-104)."""
    rho_cell = np.asarray(rho_cell, dtype=np.float64)
    mu_cell = np.asarray(mu_cell, dtype=np.float64)
    if gamma_cell is None:
        gamma_cell = np.zeros(geo.cells)
    rho_face = [to_stagger_mean(rho_cell, a, geo.per(a)) for a in range(geo.dim)]
    mu_edge = {}
    for pl in planes(geo.dim):
        e = mu_cell
        for a in pl:
            e = to_stagger_mean(e, a, geo.per(a))
        mu_edge[pl] = e
    return Coef(float(theta), rho_cell, rho_face, mu_cell, mu_edge,
                np.asarray(gamma_cell, dtype=np.float64), form)


def rescale(geo, coef, rhs_u, rhs_p):
    """operators.py:532-550: c = h / max(mu); returns (coef', rhs_u', rhs_p, c)."""
    mu0 = float(coef.mu_cell.max())
    c = geo.h / mu0 if mu0 > 0 else 1.0
    sc = Coef(c * coef.theta, coef.rho_cell, coef.rho_face, c * coef.mu_cell,
              {k: c * v for k, v in coef.mu_edge.items()}, c * coef.gamma_cell,
              coef.form)
    return sc, [c * u for u in rhs_u], rhs_p, c


def null_comps(geo, coef):
    """operators.py:368-388 velocity_null_components."""
    if coef.theta > 0:
        return ()
    out = []
    for a in range(geo.dim):
        if not geo.per(a):
            continue
        if all(geo.per(b) or (geo.bc[b][0] == FREESLIP and geo.bc[b][1] == FREESLIP)
               for b in range(geo.dim) if b != a):
            out.append(a)
    return tuple(out)


# ---------------------------------------------------------------------------
# operators (operators.py:182-365)
# ---------------------------------------------------------------------------


def div(geo, u):
    """operators.py:182-188."""
    acc = np.zeros(geo.cells)
    for a in range(geo.dim):
        acc += up_minus_here(u[a], a, geo.per(a))
    return acc / geo.h


def grad(geo, p):
    """operators.py:191-198."""
    return [here_minus_down(p, a, geo.per(a)) / geo.h for a in range(geo.dim)]


def lrho(geo, coef, p):
    """operators.py:206-215: D rho^-1 G p."""
    for r in coef.rho_face:
        if np.any(r <= 0):
            raise ValueError("face density must be positive")
    g = grad(geo, p)
    return div(geo, [g[a] / coef.rho_face[a] for a in range(geo.dim)])


def _wall_tangent_grad(geo, ua, b, lo=0.0, hi=0.0):
    """d u_a / d x_b at (a,b)-staggered points (operators.py:267-291); lo/hi are
    the prescribed tangential wall velocities (BoundaryValues.tangential_values)."""
    if geo.per(b):
        return (ua - np.roll(ua, 1, axis=b)) / geo.h
    shp = list(ua.shape)
    shp[b] += 1
    t = np.zeros(shp)
    nd = ua.ndim
    t[_ax(nd, b, slice(1, -1))] = np.diff(ua, axis=b) / geo.h
    t[_ax(nd, b, 0)] = 2.0 * (ua[_ax(nd, b, 0)] - lo) / geo.h
    t[_ax(nd, b, -1)] = 2.0 * (hi - ua[_ax(nd, b, -1)]) / geo.h
    return t


def visc_row(geo, coef, u, a, tang=None):
    """Row a of L_mu u (operators.py:303-345; the smoother's copy multigrid.py:343-383).
    tang: {(axis, side, comp): plane} tangential wall velocities (operators.py:224-264)."""
    h = geo.h
    mu = coef.mu_cell
    ncoef = mu if coef.form == LAPLACIAN else 2.0 * mu
    ua = u[a]
    fn = ncoef * up_minus_here(ua, a, geo.per(a)) / h
    if coef.form == STRESS_BULK:
        fn = fn + (coef.gamma_cell - (2.0 / 3.0) * mu) * div(geo, u)
    row = here_minus_down(fn, a, geo.per(a)) / h
    for b in range(geo.dim):
        if b == a:
            continue
        lo = hi = 0.0
        if tang is not None and not geo.per(b):
            lo = tang.get((b, 0, a), 0.0)
            hi = tang.get((b, 1, a), 0.0)
        ft = _wall_tangent_grad(geo, ua, b, lo, hi)
        if coef.form != LAPLACIAN:
            ft = ft + here_minus_down(u[b], a, geo.per(a)) / h
        ft = coef.edge(a, b) * ft
        if not geo.per(b):
            if geo.bc[b][0] == FREESLIP:
                ft[_ax(ft.ndim, b, 0)] = 0.0
            if geo.bc[b][1] == FREESLIP:
                ft[_ax(ft.ndim, b, -1)] = 0.0
        row += up_minus_here(ft, b, geo.per(b)) / h
    return row


def a_row(geo, coef, u, a, tang=None):
    """Row a of A = theta rho - L_mu, wall rows zeroed (operators.py:348-360)."""
    out = coef.theta * coef.rho_face[a] * u[a] - visc_row(geo, coef, u, a, tang)
    if not geo.per(a):
        zero_ends(out, a)
    return out


def apply_A(geo, coef, u, tang=None):
    """operators.py:348-360; tang given = apply_A(u, coeff, bvals)."""
    return [a_row(geo, coef, u, a, tang) for a in range(geo.dim)]


def apply_M(geo, coef, u, p):
    """operators.py:363-365: (A u + G p, -D u)."""
    au = apply_A(geo, coef, u)
    gp = grad(geo, p)
    return [au[a] + gp[a] for a in range(geo.dim)], -div(geo, u)


def boundary_lift(geo, normal):
    """operators.py:471-481: face field holding the prescribed normal wall
    velocities {(axis, side): plane} on the boundary faces, zero elsewhere."""
    u = [np.zeros(geo.fshape(a)) for a in range(geo.dim)]
    for a in range(geo.dim):
        if geo.per(a):
            continue
        u[a][_ax(geo.dim, a, 0)] = normal.get((a, 0), 0.0)
        u[a][_ax(geo.dim, a, -1)] = normal.get((a, 1), 0.0)
    return u


def homogenize(geo, coef, normal, tang, ru, rp):
    """operators.py:484-512: subtract the affine wall contribution from the rhs.
    Raises ValueError('incompatible boundary data ...') on a flux mismatch."""
    ub = boundary_lift(geo, normal)
    hd = geo.h ** geo.dim
    dv = div(geo, ub)
    flux = float(dv.sum()) * hd
    src = -float(rp.sum()) * hd
    scale = max(1.0, float(np.abs(dv).sum()) * hd, float(np.abs(rp).sum()) * hd)
    if abs(flux - src) > 1e-10 * scale:
        raise ValueError(f"incompatible boundary data: net boundary flux {flux:g} "
                         f"!= divergence-source integral {src:g}")
    cu = apply_A(geo, coef, ub, tang)
    return [ru[a] - cu[a] for a in range(geo.dim)], rp - (-dv)


# ---------------------------------------------------------------------------
# smoother diagonals (operators.py:396-463)
# ---------------------------------------------------------------------------


def _pair_cells(x, axis, periodic):
    """x[i-1] + x[i] at staggered points, wall rows 0 (operators.py:442-453)."""
    if periodic:
        return x + np.roll(x, 1, axis=axis)
    shp = list(x.shape)
    shp[axis] += 1
    out = np.zeros(shp)
    out[_ax(x.ndim, axis, slice(1, -1))] = (x[_ax(x.ndim, axis, slice(1, None))]
                                            + x[_ax(x.ndim, axis, slice(None, -1))])
    return out


def _pair_edges(x, axis, periodic):
    """x[j] + x[j+1] at centered points (operators.py:456-463)."""
    if periodic:
        return x + np.roll(x, -1, axis=axis)
    return x[_ax(x.ndim, axis, slice(None, -1))] + x[_ax(x.ndim, axis, slice(1, None))]


def diag_cell(geo, coef):
    """operators.py:396-405."""
    acc = np.zeros(geo.cells)
    for a in range(geo.dim):
        beta = 1.0 / coef.rho_face[a]
        if not geo.per(a):
            beta = beta.copy()
            zero_ends(beta, a)
        acc -= _pair_edges(beta, a, geo.per(a))
    return acc / geo.h ** 2


def diag_face(geo, coef):
    """operators.py:408-439 (boundary faces hold 1)."""
    h2 = geo.h ** 2
    mu = coef.mu_cell
    nc = mu if coef.form == LAPLACIAN else 2.0 * mu
    if coef.form == STRESS_BULK:
        nc = nc + (coef.gamma_cell - (2.0 / 3.0) * mu)
    out = []
    for a in range(geo.dim):
        d = coef.theta * coef.rho_face[a].copy()
        d += _pair_cells(nc, a, geo.per(a)) / h2
        for b in range(geo.dim):
            if b == a:
                continue
            w = coef.edge(a, b).copy()
            if not geo.per(b):
                for side, idx in ((0, 0), (1, -1)):
                    kind = geo.bc[b][side]
                    if kind == NOSLIP:
                        w[_ax(w.ndim, b, idx)] *= 2.0
                    elif kind == FREESLIP:
                        w[_ax(w.ndim, b, idx)] = 0.0
            d += _pair_edges(w, b, geo.per(b)) / h2
        if not geo.per(a):
            d[_ax(d.ndim, a, 0)] = 1.0
            d[_ax(d.ndim, a, -1)] = 1.0
        out.append(d)
    return out


# ---------------------------------------------------------------------------
# coefficient coarsening and transfers (multigrid.py:112-295)
# ---------------------------------------------------------------------------


def pair_mean(x, axes):
    """Mean over 2-blocks, axes in ascending order (multigrid.py:112-119)."""
    for a in sorted(axes):
        x = 0.5 * (x[_ax(x.ndim, a, slice(0, None, 2))] + x[_ax(x.ndim, a, slice(1, None, 2))])
    return x


def every_other(x, axis):  # multigrid.py:122-124
    return x[_ax(x.ndim, axis, slice(0, None, 2))]


def coarsen(geo, coef):
    """multigrid.py:127-169 -> (coarse geo, coarse coef)."""
    gc = geo.half()
    d = geo.dim
    allax = list(range(d))
    rho_face = [pair_mean(every_other(coef.rho_face[a], a), [b for b in allax if b != a])
                for a in allax]
    edges = {}
    for pl in planes(d):
        e = coef.mu_edge[pl]
        for a in pl:
            e = every_other(e, a)
        rest = [b for b in allax if b not in pl]
        if rest:
            e = pair_mean(e, rest)
        edges[pl] = e
    return gc, Coef(coef.theta, pair_mean(coef.rho_cell, allax), rho_face,
                    pair_mean(coef.mu_cell, allax), edges,
                    pair_mean(coef.gamma_cell, allax), coef.form)


def restrict_cell(geo, r):  # multigrid.py:177-182
    if any(n % 2 for n in geo.cells):
        raise ValueError("cannot restrict odd cell counts")
    return pair_mean(r, range(geo.dim))


def prolong_cell(geo_c, c):  # multigrid.py:185-192
    for a in range(geo_c.dim):
        c = np.repeat(c, 2, axis=a)
    return c


def restrict_face(geo, u):
    """multigrid.py:195-233: tangential 2-row mean, normal [1/4, 1/2, 1/4]."""
    if any(n % 2 for n in geo.cells):
        raise ValueError("cannot restrict odd cell counts")
    gc = geo.half()
    out = []
    for a in range(geo.dim):
        t = pair_mean(u[a], [b for b in range(geo.dim) if b != a])
        nd = t.ndim
        if geo.per(a):
            lo = np.roll(t, 1, axis=a)[_ax(nd, a, slice(0, None, 2))]
            mid = t[_ax(nd, a, slice(0, None, 2))]
            hi = np.roll(t, -1, axis=a)[_ax(nd, a, slice(0, None, 2))]
            out.append(0.25 * lo + 0.5 * mid + 0.25 * hi)
        else:
            shp = list(t.shape)
            shp[a] = gc.cells[a] + 1
            c = np.zeros(shp)
            lo = t[_ax(nd, a, slice(1, -2, 2))]
            mid = t[_ax(nd, a, slice(2, -1, 2))]
            hi = t[_ax(nd, a, slice(3, None, 2))]
            c[_ax(nd, a, slice(1, -1))] = 0.25 * lo + 0.5 * mid + 0.25 * hi
            out.append(c)
    return out


def _interp_tangent(x, axis, periodic):
    """3/4-1/4 doubling of a cell-centred axis, walls clamp (multigrid.py:236-257)."""
    nd = x.ndim
    if periodic:
        prv = np.roll(x, 1, axis=axis)
        nxt = np.roll(x, -1, axis=axis)
    else:
        prv = np.concatenate([x[_ax(nd, axis, slice(0, 1))], x[_ax(nd, axis, slice(None, -1))]], axis=axis)
        nxt = np.concatenate([x[_ax(nd, axis, slice(1, None))], x[_ax(nd, axis, slice(-1, None))]], axis=axis)
    shp = list(x.shape)
    shp[axis] *= 2
    out = np.zeros(shp)
    out[_ax(nd, axis, slice(0, None, 2))] = 0.75 * x + 0.25 * prv
    out[_ax(nd, axis, slice(1, None, 2))] = 0.75 * x + 0.25 * nxt
    return out


def _interp_normal(x, axis, periodic):
    """Copy coincident faces, average in-between ones (multigrid.py:260-279)."""
    nd = x.ndim
    shp = list(x.shape)
    if periodic:
        shp[axis] *= 2
        out = np.zeros(shp)
        out[_ax(nd, axis, slice(0, None, 2))] = x
        out[_ax(nd, axis, slice(1, None, 2))] = 0.5 * (x + np.roll(x, -1, axis=axis))
        return out
    shp[axis] = 2 * (x.shape[axis] - 1) + 1
    out = np.zeros(shp)
    out[_ax(nd, axis, slice(0, None, 2))] = x
    out[_ax(nd, axis, slice(1, None, 2))] = 0.5 * (x[_ax(nd, axis, slice(None, -1))]
                                                   + x[_ax(nd, axis, slice(1, None))])
    return out


def prolong_face(geo_c, c):
    """multigrid.py:282-295."""
    out = []
    for a in range(geo_c.dim):
        x = c[a]
        for b in range(geo_c.dim):
            if b != a:
                x = _interp_tangent(x, b, geo_c.per(b))
        out.append(_interp_normal(x, a, geo_c.per(a)))
    return out


# ---------------------------------------------------------------------------
# smoothers (multigrid.py:303-340)
# ---------------------------------------------------------------------------

_masks: dict = {}


def colour(shape, parity):
    key = (tuple(shape), parity)
    if key not in _masks:
        _masks[key] = (np.indices(shape).sum(axis=0) % 2) == parity
    return _masks[key]


def sweep_cell(geo, coef, phi, rhs, dg, omega):
    """One red-black GS sweep in place (multigrid.py:318-324)."""
    for parity in (0, 1):
        res = rhs - lrho(geo, coef, phi)
        m = colour(phi.shape, parity)
        phi[m] += omega * res[m] / dg[m]


def sweep_face(geo, coef, u, rhs, dg, omega):
    """One 2d-coloured GS sweep in place, x then y (then z) (multigrid.py:327-340)."""
    for a in range(geo.dim):
        sl = geo.inner(a)
        for parity in (0, 1):
            res = rhs[a] - a_row(geo, coef, u, a)
            v = u[a][sl]
            m = colour(v.shape, parity)
            v[m] += omega * (res[sl][m] / dg[a][sl][m])


# ---------------------------------------------------------------------------
# hierarchy and V-cycle (multigrid.py:34-104, 391-460)
# ---------------------------------------------------------------------------


@dataclass(frozen=True)
class Smoother:
    omega: float = 1.0
    sweeps_down: int = 2
    sweeps_up: int = 2
    bottom_sweeps: int = 8


class Hierarchy:
    def __init__(self, geo, coef):
        if not geo.coarsenable():
            raise ValueError("grid cannot be coarsened")
        self.levels = [(geo, coef)]
        while geo.coarsenable():
            geo, coef = coarsen(geo, coef)
            self.levels.append((geo, coef))
        self._dc, self._df = {}, {}

    def dcell(self, l):
        if l not in self._dc:
            g, c = self.levels[l]
            d = diag_cell(g, c)
            if np.any(d == 0):
                raise ZeroDivisionError("zero diagonal in pressure operator")
            self._dc[l] = d
        return self._dc[l]

    def dface(self, l):
        if l not in self._df:
            g, c = self.levels[l]
            d = diag_face(g, c)
            for a in range(g.dim):
                if np.any(d[a][g.inner(a)] == 0):
                    raise ZeroDivisionError("zero diagonal in velocity operator")
            self._df[l] = d
        return self._df[l]


def _zeros_like_kind(geo, kind):
    if kind == "cell":
        return np.zeros(geo.cells)
    return [np.zeros(geo.fshape(a)) for a in range(geo.dim)]


def _resid(geo, coef, x, rhs, kind):  # multigrid.py:403-406
    if kind == "cell":
        return rhs - lrho(geo, coef, x)
    ax = apply_A(geo, coef, x)
    return [rhs[a] - ax[a] for a in range(geo.dim)]


def vcycle(hier, rhs, kind, sm=Smoother(), level=0):
    """Residual-correction V-cycle from zero (multigrid.py:391-439)."""
    if kind not in ("cell", "face"):
        raise ValueError("kind must be 'cell' or 'face'")
    geo, coef = hier.levels[level]
    x = _zeros_like_kind(geo, kind)
    if kind == "cell":
        dg = hier.dcell(level)
        smooth = lambda: sweep_cell(geo, coef, x, rhs, dg, sm.omega)
    else:
        dg = hier.dface(level)
        smooth = lambda: sweep_face(geo, coef, x, rhs, dg, sm.omega)
    if level == len(hier.levels) - 1:
        for _ in range(sm.bottom_sweeps):
            smooth()
        return x
    for _ in range(sm.sweeps_down):
        smooth()
    r = _resid(geo, coef, x, rhs, kind)
    rc = restrict_cell(geo, r) if kind == "cell" else restrict_face(geo, r)
    ec = vcycle(hier, rc, kind, sm, level + 1)
    gc = hier.levels[level + 1][0]
    if kind == "cell":
        x += prolong_cell(gc, ec)
    else:
        pf = prolong_face(gc, ec)
        for a in range(geo.dim):
            x[a] += pf[a]
    for _ in range(sm.sweeps_up):
        smooth()
    return x


def mg_solve(hier, rhs, kind, sm, n_cycles):
    """multigrid.py:442-460."""
    if n_cycles < 1:
        raise ValueError("need at least one cycle")
    geo, coef = hier.levels[0]
    x = _zeros_like_kind(geo, kind)
    for cyc in range(n_cycles):
        r = rhs if cyc == 0 else _resid(geo, coef, x, rhs, kind)
        e = vcycle(hier, r, kind, sm)
        if kind == "cell":
            x += e
        else:
            for a in range(geo.dim):
                x[a] += e[a]
    return x


# ---------------------------------------------------------------------------
# Schur inverse and preconditioners (schur.py:47-78, precond.py:56-168)
# ---------------------------------------------------------------------------


def schur_diag(coef):
    """schur.py:47-56."""
    if coef.form == LAPLACIAN:
        return coef.mu_cell
    if coef.form == STRESS:
        return 2.0 * coef.mu_cell
    return coef.gamma_cell + (4.0 / 3.0) * coef.mu_cell


@dataclass
class PrecondOpts:
    kind: str = "P2"          # P1..P5 | identity
    velocity_cycles: int = 1
    sign: float = -1.0        # SchurSign.MINUS
    pressure_cycles: int = 1


class Precond:
    """precond.py:56-168 with multigrid subsolvers."""

    def __init__(self, geo, coef, opts=PrecondOpts(), sm=Smoother()):
        self.geo, self.coef, self.opts, self.sm = geo, coef, opts, sm
        self.vcycles = 0
        self.nulls = null_comps(geo, coef)
        self.hier = None if opts.kind == "identity" else Hierarchy(geo, coef)

    def vel(self, b):  # precond.py:91-96
        self.vcycles += self.geo.dim * self.opts.velocity_cycles
        return mg_solve(self.hier, b, "face", self.sm, self.opts.velocity_cycles)

    def pres(self, b):  # precond.py:98-103
        self.vcycles += self.opts.pressure_cycles
        return mg_solve(self.hier, b, "cell", self.sm, self.opts.pressure_cycles)

    def schur_inv(self, r):  # schur.py:59-78
        if self.coef.theta > 0:
            phi = self.pres(r)
            return -self.coef.theta * phi + schur_diag(self.coef) * r
        return schur_diag(self.coef) * r

    def apply(self, ru, rp):
        geo, coef, k, s = self.geo, self.coef, self.opts.kind, self.opts.sign
        if k == "identity":
            return [x.copy() for x in ru], rp.copy()
        if k == "P1":  # precond.py:118-136
            xs = self.vel(ru)
            bc = div(geo, xs) + rp
            phi = self.pres(bc)
            gphi = grad(geo, phi)
            xu = []
            for a in range(geo.dim):
                v = xs[a].copy()
                v -= gphi[a] / coef.rho_face[a]
                if not geo.per(a):
                    zero_ends(v, a)
                xu.append(v)
            xp = s * (schur_diag(coef) * bc - coef.theta * phi)
        elif k == "P2":  # :137-139
            xu = self.vel(ru)
            xp = s * self.schur_inv(div(geo, xu) + rp)
        elif k == "P3":  # :140-142
            xp = s * self.schur_inv(rp)
            g = grad(geo, xp)
            xu = self.vel([ru[a] - g[a] for a in range(geo.dim)])
        elif k == "P4":  # :143-145
            xu = self.vel(ru)
            xp = s * self.schur_inv(rp)
        elif k == "P5":  # :146-152
            xs = self.vel(ru)
            xp = s * self.schur_inv(div(geo, xs) + rp)
            g = grad(geo, xp)
            ax = apply_A(geo, coef, xs)
            b2 = [ru[a] - g[a] - ax[a] for a in range(geo.dim)]
            e = self.vel(b2)
            xu = [xs[a] + e[a] for a in range(geo.dim)]
        else:
            raise ValueError(f"unknown preconditioner kind {k}")
        # null projection (precond.py:163-168, grid.py:356-367)
        xp = xp - xp.mean()
        for a in self.nulls:
            v = xu[a][geo.inner(a)]
            v -= v.mean()
        return xu, xp


# ---------------------------------------------------------------------------
# unknown packing (grid.py:373-406) and GMRES (krylov.py:81-214)
# ---------------------------------------------------------------------------


def pack(geo, u, p):
    return np.concatenate([u[a][geo.inner(a)].ravel(order="F") for a in range(geo.dim)]
                          + [p.ravel(order="F")])


def unpack(geo, v):
    u, pos = [], 0
    for a in range(geo.dim):
        arr = np.zeros(geo.fshape(a))
        view = arr[geo.inner(a)]
        n = view.size
        view[...] = v[pos:pos + n].reshape(view.shape, order="F")
        pos += n
        u.append(arr)
    return u, v[pos:].reshape(geo.cells, order="F").copy()


def _back_subst(R, g):  # krylov.py:149-153
    y = np.zeros_like(g)
    for i in range(len(g) - 1, -1, -1):
        y[i] = (g[i] - R[i, i + 1:] @ y[i + 1:]) / R[i, i]
    return y


def gmres_flat(op, b, m, max_iters, target, bd_tol, on_iter=None):
    """Restarted GMRES(m), MGS Arnoldi + Givens (krylov.py:81-146)."""
    n = len(b)
    x = np.zeros(n)
    r = b.copy()
    k = 0
    first = True
    while True:
        beta = float(np.linalg.norm(r))
        if beta == 0.0:
            return x, "converged", k
        V = np.zeros((m + 1, n))
        H = np.zeros((m + 1, m))
        cs, sn, g = np.zeros(m), np.zeros(m), np.zeros(m + 1)
        V[0] = r / beta
        g[0] = beta
        j = 0
        xk = x
        while j < m and k < max_iters:
            w = op(V[j])
            k += 1
            for i in range(j + 1):
                H[i, j] = float(V[i] @ w)
                w -= H[i, j] * V[i]
            hn = float(np.linalg.norm(w))
            H[j + 1, j] = hn
            for i in range(j):
                t = cs[i] * H[i, j] + sn[i] * H[i + 1, j]
                H[i + 1, j] = -sn[i] * H[i, j] + cs[i] * H[i + 1, j]
                H[i, j] = t
            den = math.hypot(H[j, j], H[j + 1, j])
            if den == 0.0:
                cs[j], sn[j] = 1.0, 0.0
            else:
                cs[j], sn[j] = H[j, j] / den, H[j + 1, j] / den
            H[j, j] = den
            H[j + 1, j] = 0.0
            g[j + 1] = -sn[j] * g[j]
            g[j] = cs[j] * g[j]
            rp = abs(g[j + 1])
            y = _back_subst(H[:j + 1, :j + 1], g[:j + 1])
            xk = x + V[:j + 1].T @ y
            if on_iter is not None:
                on_iter(k, xk, rp, j == 0 and not first)
            if rp <= target:
                return xk, "converged", k
            if hn <= bd_tol:
                return xk, "breakdown", k
            V[j + 1] = w / hn
            j += 1
        x = xk
        first = False
        if k >= max_iters:
            return x, "maxiter", k
        r = b - op(x)


@dataclass
class GmresOpts:
    restart: int = 10
    max_iters: int = 500
    rtol: float = 1e-9
    atol: float = 0.0
    track_true_residual: bool = True


@dataclass
class History:
    rows: list = field(default_factory=list)  # (it, vcycles, r_P, r_true, restart)
    status: str = "running"

    @property
    def iterations(self):
        return self.rows[-1][0] if self.rows else 0


def gmres_solve(geo, coef, bu, bp, popts=PrecondOpts(), gopts=GmresOpts(),
                sm=Smoother(), P=None):
    """krylov.py:164-214 -> (u, p, History)."""
    P = P if P is not None else Precond(geo, coef, popts, sm)
    hist = History()
    b_raw = pack(geo, bu, bp)
    bnorm = float(np.linalg.norm(b_raw))

    def op(v):
        u, p = unpack(geo, v)
        mu, mp = apply_M(geo, coef, u, p)
        zu, zp = P.apply(mu, mp)
        return pack(geo, zu, zp)

    zu, zp = P.apply(bu, bp)
    z0 = pack(geo, zu, zp)
    rp0 = float(np.linalg.norm(z0))
    hist.rows.append((0, P.vcycles, rp0, bnorm, False))
    if rp0 <= gopts.atol or rp0 == 0.0:
        hist.status = "converged"
        u, p = unpack(geo, np.zeros(len(b_raw)))
        return u, p, hist
    target = gopts.rtol * rp0 + gopts.atol
    bd_tol = max(gopts.atol, 1e-14 * rp0)

    def on_iter(k, xv, rp, rflag):
        if gopts.track_true_residual:
            u, p = unpack(geo, xv)
            mu, mp = apply_M(geo, coef, u, p)
            rt = float(np.linalg.norm(b_raw - pack(geo, mu, mp)))
        else:
            rt = float("nan")
        hist.rows.append((k, P.vcycles, float(rp), rt, bool(rflag)))

    xv, status, _ = gmres_flat(op, z0, gopts.restart, gopts.max_iters, target, bd_tol, on_iter)
    hist.status = status
    u, p = unpack(geo, xv)
    return u, p, hist


def project_nulls(geo, coef, u, p):
    """problems.py:170-177."""
    u = [x.copy() for x in u]
    p = p - p.mean()
    for a in null_comps(geo, coef):
        v = u[a][geo.inner(a)]
        v -= v.mean()
    return u, p
