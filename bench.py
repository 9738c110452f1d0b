"""Benchmark: preconditioned MAC-Stokes solve on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C5] [--precond P1]
    python bench.py --impl reference ...        # the unmodified reference package on the host cores

A step is ONE full ``gmres_solve`` of the configured problem to a relative
preconditioned residual of 1e-9 (device setup -- coefficient upload, hierarchy
coarsening, 1/rho, diagonal checks -- plus the GMRES(m)/P1/V-cycle solve).

* ``value``  -- seconds per solve with every input already resident in HBM
  (torch tensors handed to the C ABI), CUDA events on the stream the library
  launches on; max over ranks.
* ``e2e``    -- the same solve through the public drop-in API
  ``gmres_solve(rhs, coeff, pcfg, gcfg)`` with HOST (pinned) NumPy inputs:
  H2D of the coefficient set and rhs, the solve, D2H of the solution.
* ``roofline`` -- the dominant kernel (finest-level face GS colour pass):
  algorithmic bytes per launch / its average CUDA-event
  duration in an instrumented solve, against MEASURED_PEAKS.json hbm_gbs.
* ``cpu_baseline`` -- the unmodified reference package (baseline/_ref, itself
  single-threaded NumPy; the oracle port only if it is absent) on the same
  recipe for a bounded number of iterations, extrapolated to the solve's
  iteration count (see ``cpu_sample``); ``--impl reference`` takes the sample
  at the bench grid (256^3, max_iters = 3).
* ``smoother`` -- all colour passes of all levels: combined, face-only and
  cell-only GB/s against the same peak.

The default workload is C5's single-GPU point (256^3 periodic steady Stokes,
log10-viscosity Fourier field over 3 decades, GMRES(50), P1): C5 is the
configuration BASELINE.json quotes the metric on ("solve time, iteration
count, and smoother GB/s at 1/2/4/8 B200s"); C5 at 512^3 does not fit one GPU.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import pathlib
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = pathlib.Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "Stokes solve wall-time to rel. residual 1e-9; MG smoother GB/s vs HBM peak"
ITER_FILE = ROOT / "profiles" / "bench_iterations.json"
NCU_FILE = ROOT / "profiles" / "ncu_face_colour.json"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="C5", choices=["C1", "C2", "C3", "C4", "C5"])
    ap.add_argument("--n", type=int, default=None, help="override cells per axis")
    ap.add_argument("--precond", default="P1")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--graphs", type=int, default=1)
    ap.add_argument("--ref-iters", type=int, default=REF_ITERS, help="reference arm: GMRES iterations sampled")
    ap.add_argument("--ref-n", type=int, default=None, help="reference arm: sample cells per axis")
    ap.add_argument("--force-dist", action="store_true",
                    help="run the slab-decomposed (NCCL) path even with one rank (code-path check)")
    return ap.parse_args()


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


# ---------------------------------------------------------------------------
# clocks sampler (nvidia-smi during the timed region)
# ---------------------------------------------------------------------------


class Clocks:
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.lines = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                                          "-lms", "200", "-i", str(self.index)],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for ln in self.proc.stdout:
            self.lines.append(ln.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.t.join(timeout=2)
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                smax = float(f[2])
            except ValueError:
                continue
            for nm, v in zip(names, f[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------------------
# CPU reference path (oracle port of the reference's NumPy algorithm)
# ---------------------------------------------------------------------------


def _oracle_case(config, n, precond):
    from oracle import stokes_oracle as O
    from paper_1308_4605_b200 import problems as PR
    case = PR.make_case(config, n)
    cs, rs, spec = PR.prepare(case)
    g = case.grid
    geo = O.Geo(g.cells, g.h, tuple((lo.value, hi.value) for lo, hi in g.bc))
    oc = O.Coef(cs.theta, cs.rho_cell.data, list(cs.rho_face.components), cs.mu_cell.data,
                dict(cs.mu_node_edge.arrays), cs.gamma_cell.data, "stress")
    return case, geo, oc, list(rs.u.components), rs.p.data


def reference_package():
    """The UNMODIFIED reference ``stokesmg`` pip-installed into baseline/_ref
    (DESIGN.md §7), or None when it is absent (then the oracle port stands in)."""
    p = ROOT / "baseline" / "_ref"
    if not (p / "stokesmg" / "__init__.py").exists():
        return None
    if str(p) not in sys.path:
        sys.path.insert(0, str(p))
    import stokesmg
    return stokesmg


def _ref_types(sm, case):
    """The seeded recipe's arrays (the device arm's inputs) in the reference's types."""
    from stokesmg import grid as G
    from stokesmg import operators as OP
    code = {"periodic": G.PERIODIC, "no_slip": G.NO_SLIP, "free_slip": G.FREE_SLIP}
    g = G.GridSpec(tuple(case.grid.cells), case.grid.h,
                   tuple((code[lo.value], code[hi.value]) for lo, hi in case.grid.bc))
    c0 = case.coeff
    coeff = OP.CoefficientSet(
        theta=c0.theta, rho_cell=G.CellField(g, c0.rho_cell.data), rho_face=G.FaceField(g, c0.rho_face.components),
        mu_cell=G.CellField(g, c0.mu_cell.data), mu_node_edge=G.NodeEdgeField(g, dict(c0.mu_node_edge.arrays)),
        gamma_cell=G.CellField(g, c0.gamma_cell.data), viscous_form=OP.STRESS)
    rhs = G.StokesVector(G.FaceField(g, case.rhs.u.components), G.CellField(g, case.rhs.p.data))
    return coeff, rhs


def _vector_op_s(n_u):
    """Seconds of one (dot + axpy + x_k update) triple on length-n_u fp64 vectors
    with NumPy: the per-basis-vector cost of the reference's MGS Arnoldi and of
    its per-iteration ``x + V^T y`` (krylov.py:111-113, :132-133)."""
    a = np.random.default_rng(0).standard_normal(n_u)
    b = np.ones(n_u)
    t0 = time.perf_counter()
    for _ in range(3):
        h = float(a @ b)
        b -= 1e-3 * h * a
        b += 1e-3 * a
    return (time.perf_counter() - t0) / 3


def cpu_sample(config, target_cells, n_sample, k, precond, iterations):
    """Time the REFERENCE's CPU path (baseline/_ref ``stokesmg``, unmodified, one
    core) on the seeded recipe at n_sample cells per axis: ``Preconditioner``
    construction (hierarchy), then ``gmres_solve(..., max_iters=k)`` (k + 1
    P^-1 M applications), ``track_true_residual=False``.
    Extrapolated to a full solve of ``iterations`` iterations at target_cells:
    (setup + (iterations + 1 + restarts) x per-application time + the MGS /
    x_k vector work of the later Arnoldi steps) x the cell ratio.  Falls back
    to the oracle port when the reference is not installed (kind "port")."""
    from paper_1308_4605_b200 import problems as PR
    sm = reference_package()
    case = PR.make_case(config, n_sample)
    restart = case.restart
    kind = "reference" if sm is not None else "port"
    if sm is not None:
        from stokesmg import operators as ROP
        from stokesmg import precond as RPC
        coeff, rhs = _ref_types(sm, case)
        cs, rs, _ = ROP.rescale(coeff, rhs)
        pcfg = RPC.PrecondConfig(kind=RPC.PrecondKind(precond))
        gcfg = sm.GmresConfig(restart=restart, max_iters=k, rtol=1e-9, atol=0.0, track_true_residual=False)
        t0 = time.perf_counter()
        P = RPC.Preconditioner(cs, pcfg)
        t1 = time.perf_counter()
        _, hist = sm.gmres_solve(rs, cs, pcfg, gcfg, precond=P)
        t2 = time.perf_counter()
        n_u = sum(c.size for c in rs.u.components) + rs.p.data.size
        who = "reference stokesmg 0.1.0 (baseline/_ref, unmodified, NumPy, 1 thread)"
    else:
        from oracle import stokes_oracle as O
        case, geo, oc, bu, bp = _oracle_case(config, n_sample, precond)
        t0 = time.perf_counter()
        P = O.Precond(geo, oc, O.PrecondOpts(kind=precond))
        t1 = time.perf_counter()
        O.gmres_solve(geo, oc, bu, bp, P=P, gopts=O.GmresOpts(restart=restart, max_iters=k,
                                                              track_true_residual=False))
        t2 = time.perf_counter()
        n_u = sum(x.size for x in bu) + bp.size
        who = "oracle port of stokesmg (NumPy, 1 thread; reference not installed)"
    t_app = (t2 - t1) / (k + 1)
    t_vop = _vector_op_s(n_u)
    dim = len(case.grid.cells)
    scale = float(math.prod(target_cells)) / float(math.prod(case.grid.cells))
    restarts = max(0, (iterations - 1) // restart)
    js = [(i - 1) % restart for i in range(1, iterations + 1)]
    mgs_extra = 3.0 * t_vop * (sum(js) - sum(js[:k]))
    t_full = scale * ((t1 - t0) + (iterations + 1 + restarts) * t_app + mgs_extra)
    cells_s = "x".join(map(str, case.grid.cells))
    tgt_s = "x".join(map(str, target_cells))
    sample = (f"{who} on the {config} recipe at {cells_s}: Preconditioner setup {t1 - t0:.2f} s + "
              f"gmres_solve(max_iters={k}) {t2 - t1:.1f} s ({k + 1} P^-1 M applications, {t_app:.2f} s each); "
              f"EXTRAPOLATED to {iterations} iterations ({restarts} restarts) at {tgt_s}"
              + (f" (x{scale:g} cells)" if scale != 1 else "") +
              f" incl. {mgs_extra:.1f} s of later-iteration MGS/x_k vector work ({t_vop * 1e3:.0f} ms per basis vector)")
    info = {"kind": kind, "sample": sample, "sample_wall_s": t2 - t0, "setup_s": t1 - t0,
            "per_application_s": t_app, "sample_iters": k, "sample_cells": list(case.grid.cells),
            "extrapolated": True, "dim": dim}
    return t_full, info


def host_info():
    model, cores = None, os.cpu_count()
    try:
        for ln in pathlib.Path("/proc/cpuinfo").read_text().splitlines():
            if ln.startswith("model name"):
                model = ln.split(":", 1)[1].strip()
                break
    except Exception:
        pass
    return {"cpu_model": model, "host_cores": cores}


def bench_iterations(config, precond, default):
    try:
        d = json.loads(ITER_FILE.read_text())
        return int(d[f"{config}_{precond}"]["iterations"]), "device solve of the same inputs"
    except Exception:
        return default, "default estimate"


def workload(config, precond, n_gpus, n=None):
    """The device arm's workload for N GPUs: (cells, restart, config dict).  The
    config dict is identical in both arms (the driver compares them)."""
    from paper_1308_4605_b200 import problems as PR
    if config == "C5" and n_gpus > 1:
        cells = tuple(PR.c5_cells(n_gpus))
    else:
        n_t = n or {"C1": 64, "C2": 256, "C3": 128, "C4": 256, "C5": 256}[config]
        cells = (n_t,) * (2 if config in ("C1", "C2") else 3)
    restart = 50 if config in ("C3", "C5") else 30
    walls = "periodic" if config in ("C1", "C3", "C5") else "walls"
    par = "single GPU" if n_gpus == 1 else (
        f"{n_gpus} GPUs, axis-0 slabs (C5 weak scaling, 256^3 per GPU)" if config == "C5"
        else f"{n_gpus} GPUs, axis-0 slabs (strong scaling)")
    cfg = {"workload": f"{config} {'x'.join(map(str, cells))} {walls} {precond} GMRES({restart}) rtol 1e-9",
           "precond": precond, "restart": restart, "cells": list(cells), "rtol": 1e-9, "seed": 1308,
           "parallelism": par,
           "l2": "every fine-level field (>= 134 MB at 256^3) exceeds the 126 MB L2; no flush needed"}
    return cells, restart, cfg


REF_ITERS = 3  # C4 / C5 run max_iters = 3 on the CPU


def run_reference(args, rank, world):
    """``--impl reference``: the reference's own CPU path, timed on this host.

    Rank 0 alone runs (other ranks exit 0).  One measured sample at the device
    arm's per-GPU size (256^3 for C4/C5; the full grid for C1-C3) with
    ``max_iters=3``, extrapolated to the device arm's iteration
    count and global grid; the warm-up / steps counts are recorded but the
    sample is taken once (a single 256^3 sample is minutes of CPU)."""
    if rank != 0:
        return
    os.environ.setdefault("OMP_NUM_THREADS", "1")
    n_gpus = max(args.gpus, world)
    cells, restart, cfg = workload(args.config, args.precond, n_gpus, args.n)
    its, its_src = bench_iterations(args.config, args.precond, 40)
    n_sample = args.ref_n or (min(cells[0], 256) if len(cells) == 3 else cells[0])
    k = args.ref_iters
    v, info = cpu_sample(args.config, cells, n_sample, k, args.precond, its)
    info.update(host_info())
    info["iterations_assumed"] = its
    info["iterations_source"] = its_src
    out = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": "s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * v,
        "higher_is_better": False, "scaling": "weak" if args.config == "C5" else "strong", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic (seeded recipe, SURVEY §8d)", "config": cfg,
        "cpu_baseline": dict(value=v, unit="s", cores=1, **info),
        "e2e": {"value": v, "unit": "s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(out), flush=True)


# ---------------------------------------------------------------------------
# device path
# ---------------------------------------------------------------------------


def smoother_report(st, peak):
    """Smoother GB/s over all levels of one instrumented solve (algorithmic
    bytes / CUDA-event time), face and cell colour passes together and each on
    its own: a constant-density level's cell pass streams no 1/rho arrays and
    is credited 16 B per cell, not the 40 B of the variable-density model."""
    def rate(b, ms):
        return b / (ms * 1e-3) / 1e9 if ms > 0 else None
    fb, fm = st["smoother_face_bytes"], st["smoother_face_ms"]
    cb, cm = st["smoother_cell_bytes"], st["smoother_cell_ms"]
    out = {"GBps": rate(fb + cb, fm + cm), "face_GBps": rate(fb, fm), "cell_GBps": rate(cb, cm),
           "face_ms_per_solve": fm, "cell_ms_per_solve": cm,
           "launches": st["smoother_face_launches"] + st["smoother_cell_launches"]}
    for k in ("", "face_", "cell_"):
        v = out[k + "GBps"]
        out[k + "frac"] = v / peak if v else None
    return out


def main():
    args = parse()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        return run_reference(args, rank, world)

    import torch
    import torch.distributed as dist

    from paper_1308_4605_b200 import problems as PR
    from paper_1308_4605_b200.grid import edge_planes
    from paper_1308_4605_b200.krylov import GmresConfig, gmres_solve, solve_raw
    from paper_1308_4605_b200.precond import PrecondConfig, Preconditioner, PrecondKind

    torch.cuda.set_device(local)
    if world > 1 or args.force_dist:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29517")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local), rank=rank, world_size=world)
        return run_dist(args, rank, world, local)
    dev = torch.device("cuda", local)

    case = PR.make_case(args.config, args.n)
    cs, rs, spec = PR.prepare(case)
    g = case.grid
    pkind = PrecondKind(args.precond)
    gcfg = GmresConfig(restart=case.restart, max_iters=500, rtol=1e-9, atol=0.0, track_true_residual=False)

    # ---- HBM-resident inputs -------------------------------------------------
    T = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)
    class DevCoeff:  # duck-typed CoefficientSet with device tensors
        pass
    dc = DevCoeff()
    dc.theta = cs.theta
    dc.viscous_form = cs.viscous_form
    dc.rho_face = type("F", (), {"components": [T(c) for c in cs.rho_face.components]})()
    dc.mu_cell = type("C", (), {"data": T(cs.mu_cell.data)})()
    dc.gamma_cell = type("C", (), {"data": T(cs.gamma_cell.data)})()
    edges = {pl: T(cs.mu_node_edge.plane(*pl)) for pl in edge_planes(g.dim)}
    dc.mu_node_edge = type("E", (), {"plane": staticmethod(lambda a, b: edges[(min(a, b), max(a, b))])})()
    bu = [T(c) for c in rs.u.components]
    bp = T(rs.p.data)
    xu = [torch.zeros_like(c) for c in bu]
    xp = torch.zeros_like(bp)

    P = Preconditioner(cs, PrecondConfig(kind=pkind))
    P.set_graphs(bool(args.graphs))
    stream = torch.cuda.current_stream(dev)
    P.ctx.set_stream(stream.cuda_stream)

    def step():
        P.ctx.set_coefficients(dc)
        return solve_raw(P, gcfg, bu, bp, xu, xp)

    hist = None
    for _ in range(max(args.warmup, 0)):
        hist = step()
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    clocks = Clocks(local)
    clocks.start()
    l0 = P.launch_count()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        hist = step()
    e1.record(stream)
    torch.cuda.synchronize(dev)
    ck = clocks.stop()
    launches = P.launch_count() - l0
    ms = e0.elapsed_time(e1) / max(args.steps, 1)
    if world > 1:
        dist.barrier()
        t = torch.tensor([ms], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())

    # setup share (upload + hierarchy) of one step
    s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s0.record(stream)
    P.ctx.set_coefficients(dc)
    s1.record(stream)
    torch.cuda.synchronize(dev)
    setup_ms = s0.elapsed_time(s1)

    # ---- roofline: instrumented solve (untimed) -------------------------------
    P.set_profiling(True)
    P.scalar_vcycles = 0  # the counter accumulates over solves on a reused Preconditioner
    step()
    vc_solve = P.scalar_vcycles
    P.set_profiling(False)
    st = P.kernel_stats()
    peak, peak_src = peaks()
    fine_launch_bytes = st["fine_face_bytes"] / max(st["fine_face_launches"], 1)
    fine_launch_ms = st["fine_face_ms"] / max(st["fine_face_launches"], 1)
    achieved = fine_launch_bytes / (fine_launch_ms * 1e-3) / 1e9 if fine_launch_ms > 0 else None
    traffic = None
    try:
        ncu = json.loads(NCU_FILE.read_text())
        key = f"{args.config}_{case.grid.cells[0]}"
        traffic = ncu.get(key, {}).get("dram_bytes_per_launch")
    except Exception:
        pass
    sm_bytes = st["smoother_face_bytes"] + st["smoother_cell_bytes"]
    sm_ms = st["smoother_face_ms"] + st["smoother_cell_ms"]

    # ---- e2e through the public API with pinned host buffers --------------------
    e2e = None
    if not args.no_e2e:
        from paper_1308_4605_b200.grid import CellField, FaceField, NodeEdgeField, StokesVector
        from paper_1308_4605_b200.operators import CoefficientSet

        def pinned(a):
            t = torch.empty(a.shape, dtype=torch.float64, pin_memory=True)
            t.numpy()[...] = a
            return t.numpy()

        hc = CoefficientSet.__new__(CoefficientSet)
        hc.theta, hc.viscous_form = cs.theta, cs.viscous_form
        hc.rho_cell = CellField(g, cs.rho_cell.data)
        hc.rho_face = FaceField(g, tuple(pinned(c) for c in cs.rho_face.components))
        hc.mu_cell = CellField(g, pinned(cs.mu_cell.data))
        hc.mu_node_edge = NodeEdgeField(g, {k: pinned(v) for k, v in cs.mu_node_edge.arrays.items()})
        hc.gamma_cell = CellField(g, pinned(cs.gamma_cell.data))
        hr = StokesVector(FaceField(g, tuple(pinned(c) for c in rs.u.components)), CellField(g, pinned(rs.p.data)))
        P.ctx.set_stream(None)
        P.ctx.release()  # return the context to the pool; the public call re-acquires it
        P.ctx = None
        pc = PrecondConfig(kind=pkind)
        for _ in range(2):  # warm: context pool, graph, and the two pinned result sets a
            x, _ = gmres_solve(hr, hc, pc, gcfg)  # `x = solve(...)` loop alternates between
        h2d = sum(c.nbytes for c in hc.rho_face.components) + hc.mu_cell.data.nbytes + \
            sum(v.nbytes for v in hc.mu_node_edge.arrays.values()) + hc.gamma_cell.data.nbytes + \
            sum(c.nbytes for c in hr.u.components) + hr.p.data.nbytes
        d2h = sum(c.nbytes for c in x.u.components) + x.p.data.nbytes
        torch.cuda.synchronize(dev)
        t0 = time.perf_counter()
        for _ in range(args.steps):
            x, ehist = gmres_solve(hr, hc, pc, gcfg)
        torch.cuda.synchronize(dev)
        e2e_s = (time.perf_counter() - t0) / max(args.steps, 1)
        if world > 1:
            t = torch.tensor([e2e_s], device=dev, dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e2e_s = float(t.item())
        e2e = {"value": e2e_s, "unit": "s", "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
               "iterations": ehist.iterations, "api": "paper_1308_4605_b200.gmres_solve (host NumPy, pinned)"}

    iters = hist.iterations
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        # bounded sample (~30 s of CPU): the reference at 128^3, one GMRES
        # iteration; the full 256^3 measurement is the --impl reference arm
        n_t = case.grid.cells[0]
        n_s = min(n_t, 128) if g.dim == 3 else n_t
        v, info = cpu_sample(args.config, tuple(case.grid.cells), n_s, 1, args.precond, iters)
        cpu = dict(value=v, unit="s", cores=1, **info, **host_info())

    if rank == 0:
        ITER_FILE.parent.mkdir(exist_ok=True)
        try:
            d = json.loads(ITER_FILE.read_text()) if ITER_FILE.exists() else {}
        except Exception:
            d = {}
        if args.n is None:
            d[f"{args.config}_{args.precond}"] = {"iterations": iters, "status": hist.status,
                                                  "scalar_vcycles": vc_solve}
            (ROOT / "gpurun_out").mkdir(exist_ok=True)
            (ROOT / "gpurun_out" / "bench_iterations.json").write_text(json.dumps(d, indent=1))
        value = ms / 1e3
        out = {
            "metric": METRIC, "value": value, "unit": "s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": False, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded recipe, SURVEY §8d)",
            "config": workload(args.config, args.precond, world, args.n)[2],
            "solve": {"iterations": iters, "status": hist.status, "scalar_vcycles_per_solve": vc_solve,
                      "setup_ms": setup_ms, "graphs": bool(args.graphs)},
            "roofline": {"bound": "hbm", "kernel": "k_face_colour (finest level)",
                         "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": (achieved / peak) if achieved else None, "traffic": traffic,
                         "bytes_per_launch": fine_launch_bytes, "ms_per_launch": fine_launch_ms,
                         # the kernel derives the edge viscosities from mu_c where it can, so
                         # it moves fewer bytes than the SURVEY §8d model credits (frac may
                         # exceed 1): the ncu DRAM traffic over the same live launch time
                         "traffic_frac": (traffic / (fine_launch_ms * 1e-3) / 1e9 / peak)
                         if (traffic and fine_launch_ms > 0) else None,
                         "peak_source": peak_src},
            "smoother": smoother_report(st, peak),
            "e2e": e2e, "gpu_launches": int(launches), "clocks": ck, "cpu_baseline": cpu,
        }
        print(json.dumps(out), flush=True)
    if world > 1:
        dist.destroy_process_group()


def run_dist(args, rank, world, local):
    """N > 1 (or --force-dist): the slab-decomposed solve, one slab per GPU,
    NCCL halo exchange / allreduce / coarse allgather inside libstokesb200.so
    (with one rank the 1-rank communicator runs the same NCCL branches).
    C5: weak scaling, 256^3 cells per GPU (512 x 256^2, 512^2 x 256, 512^3),
    each rank generating only its planes.  C4 (and C3): strong scaling of the
    BASELINE grid (256^3), every rank generating the global recipe and passing
    its planes."""
    import torch
    import torch.distributed as dist

    from paper_1308_4605_b200 import problems as PR
    from paper_1308_4605_b200.dist import DistSolver, bootstrap_nccl_id
    from paper_1308_4605_b200.krylov import GmresConfig
    from paper_1308_4605_b200.operators import STRESS
    from paper_1308_4605_b200.precond import PrecondConfig, PrecondKind

    if args.config not in ("C3", "C4", "C5"):
        raise SystemExit("the slab-decomposed path is 3D (C3 / C4 / C5)")
    dev = torch.device("cuda", local)

    def reduce(kind, a, b):
        if kind == "minmax":
            t = torch.tensor([-a, b], dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            return -float(t[0]), float(t[1])
        t = torch.tensor([a, b], dtype=torch.float64, device=dev)
        dist.all_reduce(t)
        return float(t[0]), float(t[1])

    cells, restart, wcfg = workload(args.config, args.precond, world, args.n)
    nid = bootstrap_nccl_id()
    if args.config == "C5" and args.n is None:
        grid, coeff, rhs, c = PR.make_c5_slab(cells, world, rank, reduce=reduce)
        D = DistSolver(grid, STRESS, nranks=world, rank=rank, nslab=1, nccl_id=nid)
        D.local_inputs = True
    else:
        from paper_1308_4605_b200.dist import rank_planes
        case = PR.make_case(args.config, args.n)
        cs, rs, _ = PR.prepare(case)
        grid = case.grid
        D = DistSolver(grid, STRESS, nranks=world, rank=rank, nslab=1, nccl_id=nid)
        D.local_inputs = True
        mine = lambda a: rank_planes(a, world, rank)
        from types import SimpleNamespace as NS
        coeff = NS(theta=cs.theta,
                   rho_face=NS(components=[mine(x) for x in cs.rho_face.components]),
                   mu_cell=NS(data=mine(cs.mu_cell.data)), gamma_cell=NS(data=mine(cs.gamma_cell.data)),
                   mu_node_edge=NS(arrays={k: mine(v) for k, v in cs.mu_node_edge.arrays.items()}))
        coeff.mu_node_edge.plane = lambda a, b, _e=coeff.mu_node_edge.arrays: _e[(min(a, b), max(a, b))]
        rhs = NS(u=NS(components=[mine(x) for x in rs.u.components]), p=NS(data=mine(rs.p.data)))
        del case, cs, rs
    assert D.uses_nccl
    T = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)

    class DC:  # HBM-resident coefficient set (duck-typed)
        pass
    dc = DC()
    dc.theta = coeff.theta
    dc.rho_face = type("F", (), {"components": [T(x) for x in coeff.rho_face.components]})()
    dc.mu_cell = type("C", (), {"data": T(coeff.mu_cell.data)})()
    dc.gamma_cell = type("C", (), {"data": T(coeff.gamma_cell.data)})()
    edges = {k: T(v) for k, v in coeff.mu_node_edge.arrays.items()}
    dc.mu_node_edge = type("E", (), {"plane": staticmethod(lambda a, b: edges[(min(a, b), max(a, b))])})()
    drhs = type("R", (), {})()
    drhs.u = type("U", (), {"components": [T(x) for x in rhs.u.components]})()
    drhs.p = type("P", (), {"data": T(rhs.p.data)})()
    pc = PrecondConfig(kind=PrecondKind(args.precond))
    gcfg = GmresConfig(restart=restart, max_iters=500, rtol=1e-9, atol=0.0, track_true_residual=False)
    stream = torch.cuda.ExternalStream(D.stream_ptr(), device=dev)

    # solution into HBM-resident tensors (the single-GPU arm's solve_raw contract)
    dxu = [torch.zeros_like(c) for c in drhs.u.components]
    dxp = torch.zeros_like(drhs.p.data)

    def step():
        D.set_coefficients(dc)
        return D.gmres_solve(drhs, pc, gcfg, out=(dxu, dxp))

    hist = None
    for _ in range(max(args.warmup, 0)):
        _, _, hist = step()
    torch.cuda.synchronize(dev)
    dist.barrier()
    torch.cuda.synchronize(dev)
    clocks = Clocks(local)
    clocks.start()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    l0 = D.launch_count()
    e0.record(stream)
    for _ in range(args.steps):
        _, _, hist = step()
    e1.record(stream)
    torch.cuda.synchronize(dev)
    ck = clocks.stop()
    launches = D.launch_count() - l0
    ms = e0.elapsed_time(e1) / max(args.steps, 1)
    dist.barrier()
    t = torch.tensor([ms], device=dev, dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    # roofline: instrumented solve (untimed, eager launches), finest-level face
    # colour passes of this rank's slab (plain passes), as the 1-GPU arm
    D.set_profiling(True)
    step()
    D.set_profiling(False)
    st = D.kernel_stats()
    peak, peak_src = peaks()
    fl_bytes = st["fine_face_bytes"] / max(st["fine_face_launches"], 1)
    fl_ms = st["fine_face_ms"] / max(st["fine_face_launches"], 1)
    achieved = fl_bytes / (fl_ms * 1e-3) / 1e9 if fl_ms > 0 else None
    sm_bytes = st["smoother_face_bytes"] + st["smoother_cell_bytes"]
    sm_ms = st["smoother_face_ms"] + st["smoother_cell_ms"]
    # e2e: the same solve from pinned host arrays (each rank passes its planes)
    def pinned(a):
        tt = torch.empty(a.shape, dtype=torch.float64, pin_memory=True)
        tt.numpy()[...] = a
        return tt.numpy()
    hc = type("HC", (), {})()
    hc.theta = coeff.theta
    hc.rho_face = type("F", (), {"components": [pinned(x) for x in coeff.rho_face.components]})()
    hc.mu_cell = type("C", (), {"data": pinned(coeff.mu_cell.data)})()
    hc.gamma_cell = type("C", (), {"data": pinned(coeff.gamma_cell.data)})()
    hedges = {k: pinned(v) for k, v in coeff.mu_node_edge.arrays.items()}
    hc.mu_node_edge = type("E", (), {"plane": staticmethod(lambda a, b: hedges[(min(a, b), max(a, b))])})()
    hr = type("R", (), {})()
    hr.u = type("U", (), {"components": [pinned(x) for x in rhs.u.components]})()
    hr.p = type("P", (), {"data": pinned(rhs.p.data)})()
    for _ in range(2):  # warm: the two pinned result sets alternate between steps
        D.set_coefficients(hc)
        xu, xp, _ = D.gmres_solve(hr, pc, gcfg)
    del xu, xp
    torch.cuda.synchronize(dev)
    dist.barrier()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        D.set_coefficients(hc)
        xu, xp, _ = D.gmres_solve(hr, pc, gcfg)
    torch.cuda.synchronize(dev)
    e2e_s = (time.perf_counter() - t0) / max(args.steps, 1)
    t = torch.tensor([e2e_s], device=dev, dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    e2e_s = float(t.item())
    h2d = sum(x.nbytes for x in hc.rho_face.components) + hc.mu_cell.data.nbytes + \
        sum(v.nbytes for v in hedges.values()) + hc.gamma_cell.data.nbytes + \
        sum(x.nbytes for x in hr.u.components) + hr.p.data.nbytes
    d2h = sum(x.nbytes for x in xu) + xp.nbytes
    if rank == 0:
        info = D.info()
        out = {
            "metric": METRIC, "value": ms / 1e3, "unit": "s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": False,
            "scaling": "weak" if args.config == "C5" else "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded recipe, SURVEY §8d; per-rank slabs)",
            "config": wcfg,
            "solve": {"iterations": hist.iterations, "status": hist.status,
                      "transport": "NCCL (1-rank communicator)" if world == 1 else f"NCCL over {world} ranks",
                      "distributed_levels": info["distributed_levels"],
                      "agglomerated_levels": info["agglomerated_levels"], "planes_per_gpu": info["planes_per_slab"]},
            "roofline": {"bound": "hbm", "kernel": "k_face_colour (finest slab level, rank 0)",
                         "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": (achieved / peak) if achieved else None, "traffic": None,
                         "bytes_per_launch": fl_bytes, "ms_per_launch": fl_ms, "peak_source": peak_src},
            "smoother": smoother_report(st, peak),
            "e2e": {"value": e2e_s, "unit": "s", "h2d_bytes_per_step": int(h2d) * world,
                    "d2h_bytes_per_step": int(d2h) * world},
            "gpu_launches": int(launches), "clocks": ck, "cpu_baseline": None,
        }
        print(json.dumps(out), flush=True)
    D.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
