"""One process per rank with the halo exchange fused into the kernels (RankPeers:
CUDA IPC handles of the neighbours' panels, boundary rows mirrored by the
kernels' own stores, cf_mirror).  This container's box has one GPU, so 2-3
ranks share cuda:0 (IPC between processes of one device) and synchronise over
gloo; the data path is the one NVLink peers use.  Checked against the oracle's
serial filter (test_dist.cpp:112-137 contract)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as tdist
import torch.multiprocessing as mp

import oracle as orc
import paper_1803_02156_b200 as cf
from paper_1803_02156_b200 import dist as cfd

pytestmark = pytest.mark.gpu
SPEC = (4, 4, 6)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, mode, ns, nb, out_q, staged=False, flags=True, shape=SPEC):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    tdist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        dev = torch.device("cuda", 0)
        spec = cf.LatticeSpec(*shape)
        plan = cfd.topi_shard_plan(spec, world, rank)
        if shape != SPEC and nb in (8, 16):  # the narrow chunk-staged kernel with mirrored halo stores
            assert plan.local.device_matrix(0).info()["narrow"]
        rows = plan.local_n + plan.halo_n
        fc = cf.filter_coefficients(-0.5, 0.5, cf.spectral_map(-8.0, 8.0), 30)
        if staged:  # X in pinned host memory, two device slots (configs[3] capacity path)
            X = cfd.host_block_vector(rows, ns, nb)
            bx = [cfd.DeviceBuffer((rows, nb), dev) for _ in range(2)]
            U, bu = cfd.peer_block_vector(rows, nb, nb, dev)
            W, bw = cfd.peer_block_vector(rows, nb, nb, dev)
        else:
            X, bx = cfd.peer_block_vector(rows, ns, nb, dev)
            U, bu = cfd.peer_block_vector(rows, ns, nb, dev)
            W, bw = cfd.peer_block_vector(rows, ns, nb, dev)
        G = cf.seeded_random_host(spec.dim(), ns, nb, 12)
        for b in range(ns // nb):
            X.panel(b)[:plan.local_n].copy_(torch.from_numpy(G[b][plan.row_begin:plan.row_end]))
        bufs = {}
        for name, bl in (("X", bx), ("U", bu), ("W", bw)):
            for b, bf in enumerate(bl):
                bufs[(name, b)] = bf
        peers = cfd.RankPeers(cfd.HaloPlan(plan), bufs, flags=flags)
        mom = cf.MomentSeries(fc.np, ns, device=dev)
        tl = cfd.Timeline()
        if staged:
            cfd.filter_rank_peer_staged(cfd.FilterOps(plan.local, fc.map), X, U, W, [bf.tensor for bf in bx], fc,
                                        peers, mom)
        else:
            cfd.filter_rank_peer(cfd.FilterOps(plan.local, fc.map), X, U, W, fc, cfd.CommMode(mode), peers, mom,
                                 timeline=tl)
            # measured timeline: one compute interval per (panel, degree step), one comm
            # interval per barrier (per step in vector mode, per degree in pipelined mode)
            steps = len(cf.kernels.degree_schedule(fc))
            kinds = [e.kind for e in tl.events]
            assert kinds.count("compute") == steps * (ns // nb)
            assert kinds.count("comm") == steps * (ns // nb if mode == 0 else 1)
            assert all(e.end >= e.start >= 0 for e in tl.events) and tl.makespan() > 0
            # boundary planes first: the chunk-staged kernel (n_b = 32) raises the step flags
            # itself once its boundary units are done
            if flags and nb == 32:
                assert peers.early_steps > 0
        torch.cuda.synchronize()
        cfd.allreduce_moments_ordered(mom)
        local = np.stack([X.panel(b)[:plan.local_n].cpu().numpy() for b in range(ns // nb)])
        parts = [None] * world
        tdist.all_gather_object(parts, (plan.row_begin, local))
        if rank == 0:
            parts.sort(key=lambda t: t[0])
            out_q.put((np.concatenate([p[1] for p in parts], axis=1), mom.eta.cpu().numpy(), mom.mu.cpu().numpy()))
        tdist.barrier()
        peers.close()
    finally:
        tdist.destroy_process_group()


@pytest.mark.parametrize("world,mode,ns,nb,staged,flags,shape", [
    (2, 0, 4, 2, False, True, SPEC), (2, 1, 4, 2, False, True, SPEC), (3, 1, 4, 2, False, True, SPEC),
    (2, 0, 32, 32, False, True, SPEC), (3, 1, 64, 32, False, True, SPEC), (2, 0, 6, 2, True, True, SPEC),
    (3, 0, 96, 32, True, True, SPEC), (3, 1, 4, 2, False, False, SPEC), (2, 1, 16, 8, False, True, (16, 8, 8)),
    (2, 0, 16, 16, False, True, (16, 8, 8))])
def test_fused_peer_halo_over_processes_matches_serial_oracle(world, mode, ns, nb, staged, flags, shape):
    """staged: each rank's X in pinned host memory behind two device slots
    (filter_rank_peer_staged, the configs[3] capacity path), Alg. 3.  flags: the
    per-step barrier is the per-neighbour step flags in peer memory (default) or
    the global one-element collective.  The 16x8x8 cases run the narrow
    chunk-staged kernel (n_b = 8 / 16) with the halo in its stores."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, mode, ns, nb, q, staged, flags, shape))
             for r in range(world)]
    for p in procs:
        p.start()
    X, eta, mu = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    H = cf.topi_generate(cf.LatticeSpec(*shape))
    fc = cf.filter_coefficients(-0.5, 0.5, cf.spectral_map(-8.0, 8.0), 30)
    Xo, eta_o, mu_o = orc.apply_filter(orc.Crs(H.n, H.row_ptr, H.col_idx, H.values),
                                       cf.seeded_random_host(H.n, ns, nb, 12), 30, fc.c, fc.g, fc.map.alpha,
                                       fc.map.beta)
    assert np.abs(X - Xo).max() <= 1e-10 * np.abs(Xo).max()
    assert np.abs(eta.reshape(28, ns) - eta_o).max() <= 1e-12 * np.abs(eta_o).max()
    assert np.abs(mu.reshape(28, ns) - mu_o).max() <= 1e-12 * np.abs(mu_o).max()
