"""Multi-rank path on CPU: world_size 2 (and 3) over gloo.

The halo exchange (TorchDistExchange over HaloPlan runs) and the per-rank
filter driver (filter_rank, Alg. 3 and Alg. 4) are the product code; on CPU
the per-rank operators are the oracle's (test infrastructure), since the
device kernels need a GPU.  Checked against the oracle's serial filter."""
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


class OracleOps:
    """filter_rank's operator interface backed by the CPU checker (tests only)."""

    def __init__(self, plan, s):
        H = plan.local
        self.H = orc.Crs(H.n, H.row_ptr, H.col_idx, H.values, H.ncols)
        self.a, self.b = s.alpha, s.beta
        self.n = H.n

    def spmmv(self, X, U):
        U.data()[:self.n] = torch.from_numpy(orc.spmmv(self.H, self.a, self.b, X.data().numpy()))

    def init_tail(self, X, U, W, g0c0, g1c1, g2c2):
        x = X.data().numpy()
        W.data()[:self.n] = torch.from_numpy(orc.two_minus(self.H, self.a, self.b, U.data().numpy(), x[:self.n]))
        x[:self.n] = g0c0 * x[:self.n] + g1c1 * U.data().numpy()[:self.n] + g2c2 * W.data().numpy()[:self.n]

    def step(self, U, W, X, p, gc, mom, col):
        n = self.n
        Wn, Xn, e, m = orc.chebfd_op(self.H, self.a, self.b, U.data().numpy(), W.data().numpy()[:n],
                                     X.data().numpy()[:n], gc)
        W.data()[:n] = torch.from_numpy(Wn)
        X.data()[:n] = torch.from_numpy(Xn)
        k = mom.index(p, col)
        mom.eta[k:k + e.size] += torch.from_numpy(e)
        mom.mu[k:k + m.size] += torch.from_numpy(m)


    def grouped_step(self, U, W, X, d, mom, col):
        """apply_filter's grouped step (kernels.degree_schedule) on the checker:
        the W / moment update of chebfd_op, then x += gw w_old + gu u + gc w_new."""
        p, kind, gw, gu, gc = d
        n = self.n
        w_old = W.data().numpy()[:n].copy()
        u = U.data().numpy()[:n].copy()
        x0 = X.data().numpy()[:n].copy()
        self.step(U, W, X, p, 0.0, mom, col)  # X += 0 * w_new: unchanged
        w_new = W.data().numpy()[:n]
        if kind == 0:
            x = x0 + gc * w_new
        elif kind == 1:
            x = x0
        else:
            x = x0 + gw * w_old + gu * u + gc * w_new
        X.data()[:n] = torch.from_numpy(x)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, mode, out_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    tdist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        spec = cf.LatticeSpec(4, 4, 6)
        plan = cfd.topi_shard_plan(spec, world, rank)
        ns, nb = 4, 2
        rows = plan.local_n + plan.halo_n
        # halo delivery: global random vector, exchange, compare (test_dist.cpp:77-92)
        G = cf.seeded_random_host(spec.dim(), ns, nb, 12)
        X = cf.BlockVector(rows, ns, nb, device="cpu")
        for b in range(ns // nb):
            X.panel(b)[:plan.local_n] = torch.from_numpy(G[b][plan.row_begin:plan.row_end])
        ex = cfd.TorchDistExchange(cfd.HaloPlan(plan))
        for b in range(ns // nb):
            ex.exchange(X.panel(b), b)
            halo = X.panel(b)[plan.local_n:].numpy()
            assert np.array_equal(halo, G[b][plan.halo_global.astype(np.int64)])
        with pytest.raises(cf.ProtocolError):
            ex.finish(99)
        # distributed filter vs the serial oracle
        fc = cf.filter_coefficients(-0.5, 0.5, cf.spectral_map(-8.0, 8.0), 30)
        X = cf.BlockVector(rows, ns, nb, device="cpu")
        for b in range(ns // nb):
            X.panel(b)[:plan.local_n] = torch.from_numpy(G[b][plan.row_begin:plan.row_end])
        U, W = cf.BlockVector(rows, ns, nb, device="cpu"), cf.BlockVector(rows, ns, nb, device="cpu")
        mom = cf.MomentSeries(fc.np, ns, device="cpu")
        cfd.filter_rank(OracleOps(plan, fc.map), X, U, W, fc, cfd.CommMode(mode), ex, mom)
        cfd.allreduce_moments_ordered(mom)
        local = torch.stack([X.panel(b)[:plan.local_n] for b in range(ns // nb)])
        parts = [torch.empty_like(local) for _ in range(world)] if rank == 0 else None
        sizes = [None] * world
        tdist.all_gather_object(sizes, local.shape[1])
        full = [torch.empty((ns // nb, sz, nb), dtype=torch.complex128) for sz in sizes]
        tdist.all_gather(full, local) if len(set(sizes)) == 1 else None
        if rank == 0:
            out_q.put((torch.cat(full, dim=1).numpy(), mom.eta.numpy(), mom.mu.numpy()))
    finally:
        tdist.destroy_process_group()


@pytest.mark.parametrize("world,mode", [(2, 0), (2, 1), (3, 0), (3, 1)])
def test_filter_rank_over_gloo_matches_serial_oracle(world, mode):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, mode, q)) for r in range(world)]
    for p in procs:
        p.start()
    X, eta, mu = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    spec = cf.LatticeSpec(4, 4, 6)
    H = cf.topi_generate(spec)
    fc = cf.filter_coefficients(-0.5, 0.5, cf.spectral_map(-8.0, 8.0), 30)
    Xo, eta_o, mu_o = orc.apply_filter(orc.Crs(H.n, H.row_ptr, H.col_idx, H.values),
                                       cf.seeded_random_host(H.n, 4, 2, 12), 30, fc.c, fc.g, fc.map.alpha,
                                       fc.map.beta)
    assert np.abs(X - Xo).max() <= 1e-12 * np.abs(Xo).max()
    assert np.abs(eta.reshape(28, 4) - eta_o).max() <= 1e-12 * np.abs(eta_o).max()
    assert np.abs(mu.reshape(28, 4) - mu_o).max() <= 1e-12 * np.abs(mu_o).max()
