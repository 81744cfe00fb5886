"""configs[4]'s distributed eigensolver at >= 10^7 rows: dist.chebfd_solve_rank
over 2 processes (one rank each; here both share the box's one GPU through CUDA
IPC, the halo fused into the kernels' stores, per-neighbour step flags, gloo for
the k x k collectives) on topi 4x128x128x160 (n = 10.5M), window (0.02, 0.055)
holding the 36 eigenvalues at 0.03927 (x12) and 0.04908 (x24) of the analytic
Bloch spectrum (tests/bloch_spectrum.py; nearest outside: 0 and 0.06284).
Prints one JSON line.

    python tools/dist_solve_1e7.py [--world 2] [--np 2000] [--ns 64]
"""
import argparse
import json
import os
import socket
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

DIMS = (128, 128, 160)
WINDOW = (0.02, 0.055)


def worker(rank, world, port, ns, np_, q):
    import torch
    import torch.distributed as tdist
    import paper_1803_02156_b200 as cf
    from paper_1803_02156_b200 import dist as cfd
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    tdist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        t0 = time.perf_counter()
        plan = cfd.topi_shard_plan(cf.LatticeSpec(*DIMS), world, rank)
        setup = time.perf_counter() - t0
        opt = cf.SolveOptions(n_s=ns, n_b=32, n_p=np_, max_restarts=10, spectral_bounds=(-4.0, 4.0))
        tdist.barrier()
        t0 = time.perf_counter()
        res = cfd.chebfd_solve_rank(plan, *WINDOW, opt)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        if rank == 0:
            q.put({"converged": res.converged, "restarts": res.iterations, "eigenvalues": list(map(float, res.eigenvalues)),
                   "max_residual": float(np.max(res.residuals)) if len(res.residuals) else None,
                   "seconds": round(dt, 2), "setup_s": round(setup, 2), "local_n": plan.local_n,
                   "halo_n": plan.halo_n})
        tdist.barrier()
    finally:
        tdist.destroy_process_group()


def main():
    import torch.multiprocessing as mp
    import bloch_spectrum
    ap = argparse.ArgumentParser()
    ap.add_argument("--world", type=int, default=2)
    ap.add_argument("--np", type=int, default=2000)
    ap.add_argument("--ns", type=int, default=64)
    a = ap.parse_args()
    ev = bloch_spectrum.spectrum(DIMS)
    want = ev[(ev > WINDOW[0]) & (ev < WINDOW[1])]
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=worker, args=(r, a.world, port, a.ns, a.np, q)) for r in range(a.world)]
    for p in procs:
        p.start()
    out = q.get(timeout=3000)
    for p in procs:
        p.join(timeout=300)
    got = np.sort(np.array(out.pop("eigenvalues")))
    n = 4 * DIMS[0] * DIMS[1] * DIMS[2]
    out.update({"what": f"dist.chebfd_solve_rank, {a.world} ranks (processes sharing one GPU), topi 4x{DIMS[0]}x"
                        f"{DIMS[1]}x{DIMS[2]} (n={n}), window {WINDOW}, n_s={a.ns}, n_b=32, n_p={a.np}, bounds [-4, 4]",
                "found": int(len(got)), "expected": int(len(want)),
                "max_abs_error_vs_analytic": float(np.abs(got - want).max()) if len(got) == len(want) else None,
                "exit_codes": [p.exitcode for p in procs]})
    print(json.dumps(out))


if __name__ == "__main__":
    main()
