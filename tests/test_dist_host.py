"""Multi-rank host logic on CPU: torch.distributed gloo, world_size 2.

* the NCCL communicator bootstrap (rank 0's ncclUniqueId broadcast to all ranks),
* the slab partition of reference-layout arrays (rank_planes / assemble),
* the halo-exchange protocol of the slab decomposition (2 ghost planes each side,
  periodic ring, the same send/recv pairing as sb_dist.inc dexchange) driving the
  oracle's red->black colour passes: the decomposed sweep must equal the
  single-domain sweep on every rank's planes.
"""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _exchange(t, rank, world):
    """Fill the 2 ghost planes on each side of axis 0 of a local array
    [ghost2 | interior | ghost2] from the ring neighbours (periodic)."""
    import torch
    import torch.distributed as dist
    n = t.shape[0] - 4
    left, right = (rank - 1) % world, (rank + 1) % world
    send_lo = t[2:4].contiguous()          # my bottom planes -> left's top ghosts
    send_hi = t[n:n + 2].contiguous()      # my top planes   -> right's bottom ghosts
    recv_top = torch.empty_like(send_lo)
    recv_bot = torch.empty_like(send_hi)
    ops = [dist.P2POp(dist.isend, send_lo, left), dist.P2POp(dist.isend, send_hi, right),
           dist.P2POp(dist.irecv, recv_top, right), dist.P2POp(dist.irecv, recv_bot, left)]
    for r in dist.batch_isend_irecv(ops):
        r.wait()
    t[n + 2:n + 4] = recv_top
    t[0:2] = recv_bot


def _worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import sys
        sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
        from oracle import stokes_oracle as O
        from paper_1308_4605_b200.dist import assemble, bootstrap_nccl_id, rank_planes

        out = {}
        # 1. NCCL id bootstrap
        nid = bootstrap_nccl_id()
        ids = [None] * world
        dist.all_gather_object(ids, nid)
        out["ids_equal"] = len(set(ids)) == 1 and len(nid) == 128

        # 2. partition / reassembly of a wall-bounded face array (C4-like, z walls)
        rng = np.random.default_rng(5)
        glob = rng.standard_normal((8, 6, 7))
        mine = rank_planes(glob, world, rank)
        parts = [None] * world
        dist.all_gather_object(parts, mine)
        out["partition_roundtrip"] = bool(np.array_equal(assemble(parts), glob))

        # 3. decomposed red->black face sweeps (component 0 and 1) with halo exchange
        bc = (("periodic",) * 2, ("periodic",) * 2, ("no_slip",) * 2)
        N = (8, 6, 8)
        geo = O.Geo(N, 0.125, bc)
        rho, mu = 0.5 + rng.random(N), 0.5 + rng.random(N)
        coef = O.make_coef(geo, 0.3, rho, mu)
        u = [rng.standard_normal(geo.fshape(a)) for a in range(3)]
        u[2][:, :, 0] = 0.0
        u[2][:, :, -1] = 0.0
        rhs = [rng.standard_normal(geo.fshape(a)) for a in range(3)]
        want = [x.copy() for x in u]
        O.sweep_face(geo, coef, want, rhs, O.diag_face(geo, coef), 1.0)

        k = N[0] // world
        lo = rank * k

        def local(x):  # [ghost2 | my planes | ghost2] filled by the exchange
            t = torch.zeros((k + 4,) + x.shape[1:], dtype=torch.float64)
            t[2:k + 2] = torch.from_numpy(x[lo:lo + k])
            _exchange(t, rank, world)
            return t

        lgeo = O.Geo((k + 4, N[1], N[2]), geo.h, bc)
        lcoef = O.Coef(coef.theta, None, [None] * 3, None, {}, None, coef.form)
        lcoef.rho_face = [local(r).numpy() for r in coef.rho_face]
        lcoef.mu_cell = local(coef.mu_cell).numpy()
        lcoef.mu_edge = {pl: local(e).numpy() for pl, e in coef.mu_edge.items()}
        lcoef.gamma_cell = local(coef.gamma_cell).numpy()
        lu = [local(x) for x in u]
        lrhs = [local(x).numpy() for x in rhs]
        dg = O.diag_face(lgeo, lcoef)
        for a in range(3):  # components in order, each: red pass, exchange, black pass, exchange
            for parity in (0, 1):
                arr = [x.numpy() for x in lu]
                res = lrhs[a] - O.a_row(lgeo, lcoef, arr, a)
                sl = lgeo.inner(a)
                v = arr[a][sl]
                m = O.colour(v.shape, parity)
                v[m] += 1.0 * (res[sl][m] / dg[a][sl][m])
                lu[a] = torch.from_numpy(arr[a])
                _exchange(lu[a], rank, world)
        err = max(float(np.abs(lu[a].numpy()[2:k + 2] - want[a][lo:lo + k]).max()) for a in range(3))
        out["sweep_err"] = err
        q.put((rank, out))
    finally:
        dist.destroy_process_group()


def test_two_rank_gloo_decomposition():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(2):
        r, out = q.get(timeout=240)
        res[r] = out
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for r in (0, 1):
        assert res[r]["ids_equal"]
        assert res[r]["partition_roundtrip"]
        assert res[r]["sweep_err"] <= 1e-13, res[r]


def _slabs_in_threads(cells, world):
    """make_c5_slab on `world` simulated ranks (threads), its `reduce` callback
    played by a barrier-synchronised all-reduce -- the bench's per-rank input
    generation at N > 1 (bench.py run_dist) without GPUs."""
    import threading

    from paper_1308_4605_b200 import problems as PR
    bar = threading.Barrier(world)
    box = [None] * world
    out = [None] * world
    err = []

    def reducer(rank):
        def reduce(kind, a, b):
            box[rank] = (a, b)
            bar.wait()
            vals = list(box)
            bar.wait()
            if kind == "minmax":
                return min(v[0] for v in vals), max(v[1] for v in vals)
            return sum(v[0] for v in vals), sum(v[1] for v in vals)
        return reduce

    def work(rank):
        try:
            out[rank] = PR.make_c5_slab(cells, world, rank, reduce=reducer(rank))
        except Exception as e:  # pragma: no cover
            err.append(e)
            bar.abort()

    ts = [threading.Thread(target=work, args=(r,)) for r in range(world)]
    for t in ts:
        t.start()
    for t in ts:
        t.join(timeout=120)
    assert not err, err
    return out


@pytest.mark.parametrize("world", [2, 4])
def test_c5_slab_generation_matches_the_global_recipe(world):
    """The weak-scaling bench generates each rank's planes of C5 locally
    (problems.make_c5_slab, global min / max / means through the reduce
    callback).  The assembled coefficient field must be the global recipe's
    (problems.make_case: same Fourier modes, same averaging), independent of
    the number of ranks, and the right-hand side must have zero global means."""
    from paper_1308_4605_b200 import problems as PR
    from paper_1308_4605_b200.dist import assemble
    cells = (16, 8, 12)
    one = _slabs_in_threads(cells, 1)[0]
    many = _slabs_in_threads(cells, world)
    grid, c1 = one[0], one[3]
    assert all(m[3] == c1 for m in many)  # the same global rescale factor on every rank
    assert all(m[0].cells == cells for m in many)
    cat = lambda pick: assemble([pick(m) for m in many])
    assert np.array_equal(cat(lambda m: m[1].mu_cell.data), one[1].mu_cell.data)
    for key in ((0, 1), (0, 2), (1, 2)):
        assert np.array_equal(cat(lambda m: m[1].mu_node_edge.arrays[key]), one[1].mu_node_edge.arrays[key])
    for a in range(3):
        assert np.array_equal(cat(lambda m: m[1].rho_face.components[a]), one[1].rho_face.components[a])
        fa = cat(lambda m: m[2].u.components[a])
        assert abs(fa.mean()) <= 1e-15 * np.abs(fa).max() * fa.size ** 0.5
    gp = cat(lambda m: m[2].p.data)
    assert abs(gp.mean()) <= 1e-15 * np.abs(gp).max() * gp.size ** 0.5
    # against the global recipe (unrescaled mu; h differs at this size, the field does not)
    case = PR.make_case("C5", cells)
    mu_glob = case.coeff.mu_cell.data
    assert np.allclose(one[1].mu_cell.data / c1, mu_glob, rtol=1e-12)
    for key in ((0, 1), (0, 2), (1, 2)):
        assert np.allclose(one[1].mu_node_edge.arrays[key] / c1, case.coeff.mu_node_edge.arrays[key], rtol=1e-12)
    assert c1 == pytest.approx((1.0 / 512) / mu_glob.max(), rel=1e-12)
