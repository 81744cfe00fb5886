"""configs[3] capacity path on ONE GPU: one rank's share of topi 4x512x512x256
over 8 GPUs (4x512x512x32 sites, n = 33.5M rows) with n_s = 256 (8 panels of
n_b = 32) -- 137 GB of X, more than the GPU holds next to U, W and the matrix --
filtered by the distributed driver's host-staged path (cf_filter_distributed_host:
X in pinned host memory, two device slots, copies overlapped), against the same
filter with one device-resident panel x 8.  The rank's z-halo planes are replaced
by the periodic wrap of its own slab (no neighbour ranks on one GPU); the halo
exchange itself is covered by tests/test_dist_peer_gpu.py (host-staged ranks
against the oracle).  Panel 0 is checked bit-for-bit against the device-resident
filter.  Prints one JSON line.

    python tools/cfg4_rank_host.py [--np 100] [--nz 32] [--panels 8]
"""
import argparse
import ctypes as C
import json
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1803_02156_b200 as cf  # noqa: E402
from paper_1803_02156_b200 import dist as cfd  # noqa: E402
from paper_1803_02156_b200._lib import check, lib  # noqa: E402


def mem_available_gb():
    for line in open("/proc/meminfo"):
        if line.startswith("MemAvailable:"):
            return int(line.split()[1]) / 2**20
    return 0.0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--nxy", type=int, default=512)
    ap.add_argument("--nz", type=int, default=32)
    ap.add_argument("--np", type=int, default=100)
    ap.add_argument("--panels", type=int, default=8)
    a = ap.parse_args()
    nb, npan = 32, a.panels
    spec = cf.LatticeSpec(a.nxy, a.nxy, a.nz)
    n = spec.dim()
    host_bytes = npan * n * nb * 16
    avail = mem_available_gb()
    if avail < host_bytes / 2**30 + 30:
        print(json.dumps({"skipped": f"host memory {avail:.0f} GiB < X {host_bytes / 2**30:.0f} GiB + 30"}))
        return
    dev = torch.device("cuda", 0)
    fc = cf.filter_coefficients(-0.35, 0.35, cf.spectral_map(-7.0, 7.0, 0.01), a.np)
    t0 = time.perf_counter()
    dm = cf.DeviceMatrix.topi(spec, 0)  # closed-form generator straight into device SELL
    build_s = time.perf_counter() - t0
    t0 = time.perf_counter()
    hostp = torch.empty((npan, n, nb), dtype=torch.complex128, pin_memory=True)
    pin_s = time.perf_counter() - t0
    P = cf.BlockVector(n, nb, nb, device=dev)
    for b in range(npan):
        cf.blockvec.random_fill_device(P, 42 + b)
        hostp[b].copy_(P.panel(0))
    # device-resident reference: panel 0, same X0 bits, through the same driver
    cf.blockvec.random_fill_device(P, 42)
    rows = (fc.np - 2) * nb
    eta1, mu1 = np.zeros(rows, np.complex128), np.zeros(rows, np.complex128)

    def worker(panels_ptrs):
        arr = (cfd._DistWorkerC * 1)()
        arr[0] = cfd._DistWorkerC(dm.handle, n, 0, C.cast(panels_ptrs, C.c_void_p), None, 0, None, 0)
        return arr

    pp = (C.c_void_p * 1)(P.panel(0).data_ptr())
    ptr = lambda x: x.ctypes.data_as(C.c_void_p)  # noqa: E731
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    check(lib.cf_filter_distributed(worker(pp), 1, nb, nb, fc.np, ptr(fc.c), ptr(fc.g), fc.map.alpha, fc.map.beta, 0,
                                    ptr(eta1), ptr(mu1)))
    panel_s = time.perf_counter() - t0
    want = P.panel(0).cpu()
    del P
    torch.cuda.empty_cache()
    free_before = torch.cuda.mem_get_info(0)[0]
    hp = (C.c_void_p * npan)(*[hostp[b].data_ptr() for b in range(npan)])
    eta, mu = np.zeros(rows * npan, np.complex128), np.zeros(rows * npan, np.complex128)
    t0 = time.perf_counter()
    check(lib.cf_filter_distributed_host(worker(hp), 1, npan * nb, nb, fc.np, ptr(fc.c), ptr(fc.g), fc.map.alpha,
                                         fc.map.beta, 0, ptr(eta), ptr(mu)))
    host_s = time.perf_counter() - t0
    same = bool(torch.equal(hostp[0], want))
    same_m = bool(np.array_equal(eta.reshape(fc.np - 2, npan * nb)[:, :nb], eta1.reshape(fc.np - 2, nb)))
    flops = 146.0 * n * nb * (fc.np - 2) * npan
    print(json.dumps({
        "what": f"one rank of topi 4x{a.nxy}x{a.nxy}x{a.nz * 8} over 8 GPUs: {a.nxy}x{a.nxy}x{a.nz} sites "
                f"(n={n}), n_s={npan * nb} ({npan} panels of {nb}), n_p={fc.np}, X in pinned host memory "
                "through cf_filter_distributed_host (two device slots); halo planes replaced by the slab's "
                "periodic wrap (no neighbours on one GPU)",
        "host_x_bytes": host_bytes, "device_free_bytes_before": int(free_before),
        "seconds": round(host_s, 3), "device_resident_seconds": round(panel_s * npan, 3),
        "device_resident_panel_seconds": round(panel_s, 3), "overhead": round(host_s / (panel_s * npan) - 1, 4),
        "gflops": round(flops / host_s / 1e9, 1), "panel0_bit_identical": same, "moments_bit_identical": same_m,
        "setup_s": {"generate_upload": round(build_s, 1), "pin_host_x": round(pin_s, 1)}}))


if __name__ == "__main__":
    main()
