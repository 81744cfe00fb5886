"""Small runs of every device path for compute-sanitizer (memcheck, racecheck,
synccheck): the chunk-staged kernel (n_b = 32: mbarrier rings, bulk copies,
cross-proxy fences, unit tickets), the narrow staged kernel (n_b = 8 / 16), the
register-gather kernel (n_b = 8), the
grouped-X degree schedule with programmatic dependent launch (apply_filter),
the drop-in chebfd_op loop, the fused halo (mirror stores into a neighbour
shard's panels) and the push kernel (scattered halo), host-staged panels, and
the solver kernels (Gram, rotation, residuals).  Each case is checked against
the CPU checker so a silent corruption also fails.

    compute-sanitizer --tool racecheck python tools/sanitize_cases.py
"""
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
import paper_1803_02156_b200 as cf  # noqa: E402
from paper_1803_02156_b200 import dist as cfd  # noqa: E402
import oracle as orc  # noqa: E402  (checker only)

DEV = torch.device("cuda", 0)


def rel(a, b):
    return float(np.abs(a - b).max() / np.abs(b).max())


def case_filter(spec, ns, nb, np_):
    H = cf.topi_generate(cf.LatticeSpec(*spec))
    fc = cf.filter_coefficients(-0.5, 0.5, cf.spectral_map(*cf.gershgorin_bounds(H), 0.01), np_)
    X = cf.BlockVector(H.n, ns, nb, cf.InitSeededRandom(5), device=DEV)
    mom = cf.apply_filter(H, X, fc)
    Xo, eta_o, _ = orc.apply_filter(orc.Crs(H.n, H.row_ptr, H.col_idx, H.values), cf.seeded_random_host(H.n, ns, nb, 5),
                                    np_, fc.c, fc.g, fc.map.alpha, fc.map.beta)
    e = (rel(X.panels_numpy(), Xo), rel(mom.eta.cpu().numpy().reshape(np_ - 2, ns), eta_o))
    assert e[0] < 1e-10 and e[1] < 1e-12, e
    return e


def case_chebfd_op_loop():
    H = cf.topi_generate(cf.LatticeSpec(8, 8, 4))
    s = cf.spectral_map(*cf.gershgorin_bounds(H), 0.01)
    X, U, W = (cf.BlockVector(H.n, 32, 32, cf.InitSeededRandom(k), device=DEV) for k in (1, 2, 3))
    mom = cf.MomentSeries(12, 32, device=DEV)
    for p in range(3, 13):
        cf.swap_blocks(cf.SubblockView(W, 0), cf.SubblockView(U, 0))
        cf.chebfd_op(H, s, cf.SubblockView(U, 0), cf.SubblockView(W, 0), cf.SubblockView(X, 0), p, 0.1 / p, mom)
    torch.cuda.synchronize()
    assert np.isfinite(X.panels_numpy()).all()


def case_distributed(host=False):
    H = cf.topi_generate(cf.LatticeSpec(4, 4, 8))
    fc = cf.filter_coefficients(-0.5, 0.5, cf.spectral_map(-8.0, 8.0), 20)
    X = cf.BlockVector(H.n, 64, 32, cf.InitSeededRandom(7), device=DEV)
    X0 = X.panels_numpy().copy()
    shards = cfd.shard_and_distribute(H, X, cfd.partition_rows(H, 2), host_panels=host)
    res = cfd.filter_distributed_native(shards, fc, cfd.CommMode.vector)
    Xo, _, _ = orc.apply_filter(orc.Crs(H.n, H.row_ptr, H.col_idx, H.values), X0, 20, fc.c, fc.g, fc.map.alpha,
                                fc.map.beta)
    assert rel(res.X.panels_numpy(), Xo) < 1e-10


def case_push_kernel():
    rng = np.random.default_rng(3)
    n = 60
    a = np.where(rng.random((n, n)) < 0.1, rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n)), 0)
    a = (a + a.conj().T) / 2 + np.diag(rng.standard_normal(n))
    H = cf.from_dense(a)
    fc = cf.filter_coefficients(-0.4, 0.4, cf.spectral_map(*cf.gershgorin_bounds(H), 0.01), 12)
    X = cf.BlockVector(H.n, 8, 4, cf.InitSeededRandom(2), device=DEV)
    X0 = X.panels_numpy().copy()
    shards = cfd.shard_and_distribute(H, X, cfd.partition_rows(H, 3))
    res = cfd.filter_distributed_native(shards, fc, cfd.CommMode.pipelined)
    Xo, _, _ = orc.apply_filter(orc.Crs(H.n, H.row_ptr, H.col_idx, H.values), X0, 12, fc.c, fc.g, fc.map.alpha,
                                fc.map.beta)
    assert rel(res.X.panels_numpy(), Xo) < 1e-10


def case_solve():
    H = cf.topi_generate(cf.LatticeSpec(3, 2, 2, 0.83, 1.1, cf.Boundary.open))
    r = cf.chebfd_solve(H, 0.3, 0.7, cf.SolveOptions(n_s=16, n_b=4, n_p=300))
    ev = np.linalg.eigvalsh(cf.to_dense(H))
    want = ev[(ev > 0.3) & (ev < 0.7)]
    assert r.converged and np.abs(np.sort(r.eigenvalues) - want).max() < 1e-8


if __name__ == "__main__":
    torch.cuda.set_device(0)
    print("staged n_b=32", case_filter((8, 8, 4), 64, 32, 14))
    print("narrow n_b=8", case_filter((16, 12, 10), 8, 8, 11))
    print("narrow n_b=16", case_filter((16, 12, 10), 16, 16, 11))
    from paper_1803_02156_b200._lib import check, lib
    check(lib.cf_tuning(b"narrow", 0))
    print("gather n_b=8", case_filter((6, 5, 4), 16, 8, 11))
    check(lib.cf_tuning(b"narrow", 1))
    case_chebfd_op_loop()
    print("chebfd_op loop ok")
    case_distributed(False)
    print("fused halo ok")
    case_distributed(True)
    print("host-staged ok")
    case_push_kernel()
    print("push kernel ok")
    case_solve()
    print("solve ok")
    torch.cuda.synchronize()
    print("ALL CASES OK")
