"""Slab-decomposed multi-GPU solve -- host side.

The global grid is cut along axis 0 into ``nranks x nslab`` slabs.  Production
multi-GPU runs use one process per GPU (``torch.distributed`` for the
bootstrap), ``nslab = 1`` and NCCL inside ``libstokesb200.so`` for halo
exchange, allreduce and coarse-level allgather.  ``nranks = 1, nslab > 1``
runs the identical decomposition on one GPU (exchanges are device copies):
that is how the parity tests exercise it on a single B200.

Arrays crossing this API are the caller's rank planes of the reference
layouts: ``rank_planes(x, nranks, rank)``.
"""

from __future__ import annotations

import ctypes as C
import os

import numpy as np

from . import _lib
from .grid import BC_CODE, CellField, FaceField, StokesVector, as_grid, edge_planes
from .krylov import _history, gmres_c
from .multigrid import smoother_c
from .operators import _f64, form_code
from .precond import precond_c


def rank_planes(x: np.ndarray, nranks: int, rank: int) -> np.ndarray:
    """The axis-0 planes of array ``x`` owned by ``rank`` (contiguous block)."""
    n0 = x.shape[0]
    if n0 % nranks:
        raise ValueError("nranks must divide the axis-0 extent")
    k = n0 // nranks
    return np.ascontiguousarray(x[rank * k:(rank + 1) * k])


def nccl_unique_id() -> bytes:
    lib = _lib.load()
    n = lib.sb_nccl_id_bytes()
    buf = C.create_string_buffer(n)
    _lib.check(lib.sb_nccl_unique_id(buf))
    return buf.raw


def bootstrap_nccl_id(group=None) -> bytes:
    """Rank 0 creates the NCCL id; every rank receives it (torch.distributed broadcast)."""
    import torch
    import torch.distributed as dist
    lib = _lib.load()
    n = lib.sb_nccl_id_bytes()
    t = torch.zeros(n, dtype=torch.uint8)
    if dist.get_rank(group) == 0:
        t[:] = torch.frombuffer(bytearray(nccl_unique_id()), dtype=torch.uint8)
    if dist.get_backend(group) == "nccl":
        tt = t.cuda()
        dist.broadcast(tt, 0, group=group)
        t = tt.cpu()
    else:
        dist.broadcast(t, 0, group=group)
    return bytes(t.numpy().tobytes())


class DistSolver:
    """One process's part of the slab-decomposed solve (3D, periodic axis 0)."""

    def __init__(self, grid, viscous_form, nranks: int = 1, rank: int = 0, nslab: int = 1,
                 nccl_id: bytes | None = None, nccl_self: bool | None = None):
        """``nccl_id``: the communicator id every rank shares (``bootstrap_nccl_id``);
        required when ``nranks > 1``.  ``nccl_self`` (default: environment
        ``SB_DIST_NCCL_SELF=1``): with one rank and one slab, create a 1-rank
        communicator anyway so every exchange / reduction / gather runs through
        the NCCL branches each rank takes at N > 1 (self send/recv)."""
        self.lib = _lib.load()
        self.grid = as_grid(grid)
        g = self.grid
        if g.dim != 3:
            raise ValueError("the distributed path is 3D")
        if nranks > 1 and nccl_id is None:
            raise ValueError("nccl_id is required for a multi-rank solver (bootstrap_nccl_id)")
        if nccl_self is None:
            nccl_self = os.environ.get("SB_DIST_NCCL_SELF", "0") == "1"
        if nranks == 1 and nslab == 1 and nccl_self and nccl_id is None:
            nccl_id = nccl_unique_id()
        self.nranks, self.rank, self.nslab = nranks, rank, nslab
        cells = (C.c_int * 3)(*g.cells)
        bcs = (C.c_int * 6)(*[BC_CODE[x] for pair in g.bc for x in pair])
        h = self.lib.sb_dist_create(cells, float(g.h), bcs, form_code(viscous_form), nranks, rank, nslab,
                                    nccl_id)
        if not h:
            raise RuntimeError("sb_dist_create failed: " + (self.lib.sb_last_error() or b"").decode())
        self.h = h
        self.scalar_vcycles = 0

    def stream_ptr(self) -> int:
        return int(self.lib.sb_dist_stream(self.h) or 0)

    def set_stream(self, stream_ptr: int | None):
        """Join the caller's CUDA stream (e.g. ``torch.cuda.current_stream().cuda_stream``)
        on entry to / exit from every call; None: no join."""
        self.lib.sb_dist_set_stream(self.h, stream_ptr or None)

    @property
    def uses_nccl(self) -> bool:
        return bool(self.lib.sb_dist_uses_nccl(self.h))

    # measurement (bench.py): per-colour-pass CUDA events, launch counting
    def set_profiling(self, enabled: bool):
        self.lib.sb_dist_set_profiling(self.h, int(bool(enabled)))

    def kernel_stats(self) -> dict:
        s = _lib.KernelStats()
        self.lib.sb_dist_get_kernel_stats(self.h, C.byref(s))
        return {k: getattr(s, k) for k, _ in s._fields_}

    def launch_count(self) -> int:
        return int(self.lib.sb_dist_launch_count(self.h))

    def info(self) -> dict:
        out = (C.c_int * 6)()
        self.lib.sb_dist_info(self.h, out)
        return {"distributed_levels": out[0], "agglomerated_levels": out[1], "planes_per_slab": out[2],
                "slabs": out[3], "mue_derived_levels": out[4], "const_rho_levels": out[5]}

    #: arrays passed in already hold only this rank's planes (bench: slab-local generation)
    local_inputs = False

    def _mine(self, x):
        if self.local_inputs:
            return _f64(x)
        return _f64(rank_planes(np.asarray(x), self.nranks, self.rank))

    def set_coefficients(self, coeff):
        """coeff: the GLOBAL CoefficientSet (each rank passes its planes down)."""
        g = self.grid
        rho = [self._mine(c) for c in coeff.rho_face.components]
        mu = self._mine(coeff.mu_cell.data)
        edges = [self._mine(coeff.mu_node_edge.plane(*pl)) for pl in edge_planes(3)]
        gam = self._mine(coeff.gamma_cell.data)
        _lib.check(self.lib.sb_dist_set_coefficients(self.h, float(coeff.theta), _lib.parr(rho), _lib.ptr(mu),
                                                      _lib.parr(edges), _lib.ptr(gam)))
        self._keep = (rho, mu, edges, gam)
        del g

    def _out(self):
        # recycled page-locked buffers (a pageable D2H runs at a third of PCIe speed)
        g = self.grid
        k = g.cells[0] // self.nranks
        shp = lambda s: (k,) + tuple(s[1:])
        return [_lib.pinned.array(shp(g.face_shape(a))) for a in range(3)], _lib.pinned.array(shp(g.cells))

    def gmres_solve(self, rhs, pcfg, gcfg, smoother=None, out=None):
        """Solve with the GLOBAL rhs; returns this rank's planes of x and the history.

        ``out=(xu, xp)``: write the solution into these arrays (this rank's
        planes; host arrays or device tensors -- the HBM-resident bench path)."""
        bu = [self._mine(c) for c in rhs.u.components]
        bp = self._mine(rhs.p.data)
        xu, xp = self._out() if out is None else (list(out[0]), out[1])
        nrows = int(gcfg.max_iters) + 2
        rows = (_lib.HistoryRow * nrows)()
        n_rows, status = C.c_int(0), C.c_int(0)
        vc = C.c_longlong(self.scalar_vcycles)
        _lib.check(self.lib.sb_dist_gmres_solve(
            self.h, C.byref(precond_c(pcfg)), C.byref(gmres_c(gcfg)), C.byref(smoother_c(smoother)),
            _lib.parr(bu), _lib.ptr(bp), _lib.parr(xu), _lib.ptr(xp), rows, nrows, C.byref(n_rows),
            C.byref(status), C.byref(vc)))
        self.scalar_vcycles = int(vc.value)
        return xu, xp, _history(rows, n_rows.value, status.value)

    def precond_apply(self, r, pcfg, smoother=None):
        ru = [self._mine(c) for c in r.u.components]
        xu, xp = self._out()
        _lib.check(self.lib.sb_dist_precond_apply(self.h, C.byref(precond_c(pcfg)), C.byref(smoother_c(smoother)),
                                                   _lib.parr(ru), _lib.ptr(self._mine(r.p.data)),
                                                   _lib.parr(xu), _lib.ptr(xp)))
        return xu, xp

    def apply_M(self, x):
        u = [self._mine(c) for c in x.u.components]
        ou, op = self._out()
        _lib.check(self.lib.sb_dist_apply_M(self.h, _lib.parr(u), _lib.ptr(self._mine(x.p.data)), _lib.parr(ou),
                                             _lib.ptr(op)))
        return ou, op

    def close(self):
        if getattr(self, "h", None):
            self.lib.sb_dist_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def assemble(parts):
    """Concatenate rank parts along axis 0 (inverse of rank_planes)."""
    return np.concatenate(parts, axis=0)
