"""chebfd_solve distributed over ranks (one process per rank: dist.chebfd_solve_rank):
the filter with the halo fused into the kernels, Gram matrices summed over
ranks, k x k Jacobi on every rank.  2-3 ranks share the box's one GPU (CUDA
IPC between processes, gloo for the collectives).  Eigenvalues against the
dense spectrum and the single-process chebfd_solve (1e-8, acceptance.cpp:95)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as tdist
import torch.multiprocessing as mp

import paper_1803_02156_b200 as cf
from paper_1803_02156_b200 import dist as cfd

pytestmark = pytest.mark.gpu
SPEC = (4, 4, 6)
WINDOW = (-0.5, 0.5)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _opts(ns):
    return cf.SolveOptions(n_s=ns, n_b=ns, n_p=200, max_restarts=20)


def _worker(rank, world, port, ns, out_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    tdist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        plan = cfd.topi_shard_plan(cf.LatticeSpec(*SPEC), world, rank)
        res = cfd.chebfd_solve_rank(plan, *WINDOW, _opts(ns))
        if rank == 0:
            out_q.put((res.converged, res.iterations, np.asarray(res.eigenvalues), np.asarray(res.residuals)))
    finally:
        tdist.destroy_process_group()


def _inside():
    H = cf.topi_generate(cf.LatticeSpec(*SPEC))
    ev = np.linalg.eigvalsh(cf.to_dense(H))
    return H, ev[(ev > WINDOW[0]) & (ev < WINDOW[1])]


@pytest.mark.parametrize("world", [2, 3])
def test_distributed_solve_matches_dense_and_single_process(world):
    H, inside = _inside()
    ns = len(inside)
    assert ns > 0
    single = cf.chebfd_solve(H, *WINDOW, _opts(ns))
    assert single.converged and np.abs(single.eigenvalues - inside).max() <= 1e-8
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, ns, q)) for r in range(world)]
    for p in procs:
        p.start()
    conv, iters, ev, rs = q.get(timeout=600)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert conv and len(ev) == ns
    assert np.abs(ev - inside).max() <= 1e-8
    assert np.abs(ev - single.eigenvalues).max() <= 1e-8
    assert np.all(rs <= 1e-9)
