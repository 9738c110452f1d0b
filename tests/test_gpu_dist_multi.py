"""Multi-rank slab solves: one process per GPU, NCCL inside libstokesb200.so.

Each world size runs only when that many GPUs are visible (the round-end GPU
tier has one, so these skip there; the single-GPU NCCL branches are covered by
the 1-rank communicator tests in test_gpu_dist.py).  Every rank solves its
slab of C5 / C4 at 64^3; rank 0 compares the gathered solution with the
single-domain device solve: equal iteration count (+-1) and relative L2 <= 1e-8.
"""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _ngpu():
    try:
        import torch
        return torch.cuda.device_count()
    except Exception:
        return 0


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, name, n, out_dir):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", rank))
    from paper_1308_4605_b200 import problems as PR
    from paper_1308_4605_b200.dist import DistSolver, bootstrap_nccl_id
    from paper_1308_4605_b200.krylov import GmresConfig
    from paper_1308_4605_b200.precond import P1, PrecondConfig
    case = PR.make_case(name, n)
    cs, rs, _ = PR.prepare(case)
    nid = bootstrap_nccl_id()
    D = DistSolver(case.grid, cs.viscous_form, nranks=world, rank=rank, nslab=1, nccl_id=nid)
    assert D.uses_nccl
    D.set_coefficients(cs)
    gcfg = GmresConfig(restart=case.restart, max_iters=500, rtol=1e-9, track_true_residual=False)
    xu, xp, h = D.gmres_solve(rs, PrecondConfig(kind=P1), gcfg)
    np.savez(os.path.join(out_dir, f"r{rank}.npz"), u0=xu[0], u1=xu[1], u2=xu[2], p=xp,
             hist=np.array(h.rows(), dtype=float), status=np.array([h.status == "converged"]))
    D.close()
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4, 8])
@pytest.mark.parametrize("name", ["C5", "C4"])
def test_multi_rank_matches_single(world, name, tmp_path):
    if _ngpu() < world:
        pytest.skip(f"needs {world} GPUs (have {_ngpu()})")
    import torch.multiprocessing as mp
    from paper_1308_4605_b200 import problems as PR
    from paper_1308_4605_b200.krylov import GmresConfig, gmres_solve
    from paper_1308_4605_b200.precond import P1, PrecondConfig
    n = 64
    mp.spawn(_worker, args=(world, _port(), name, n, str(tmp_path)), nprocs=world, join=True)
    parts = [np.load(tmp_path / f"r{r}.npz") for r in range(world)]
    case = PR.make_case(name, n)
    cs, rs, _ = PR.prepare(case)
    gcfg = GmresConfig(restart=case.restart, max_iters=500, rtol=1e-9, track_true_residual=False)
    x1, h1 = gmres_solve(rs, cs, PrecondConfig(kind=P1), gcfg)
    for p in parts:
        assert bool(p["status"][0])
        assert abs(int(p["hist"][-1, 0]) - h1.iterations) <= 1
    got = [np.concatenate([p[k] for p in parts], axis=0) for k in ("u0", "u1", "u2", "p")]
    want = list(x1.u.components) + [x1.p.data]
    num = sum(float(np.sum((a - b) ** 2)) for a, b in zip(got, want))
    den = sum(float(np.sum(b ** 2)) for b in want)
    assert np.sqrt(num / den) <= 1e-8
