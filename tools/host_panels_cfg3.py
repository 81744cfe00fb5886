"""cfg3 (4x256^3, n = 67M) with n_s = 128 (4 panels of n_b = 32) on ONE GPU:
X (137 GB) in pinned host memory, filtered through cf_apply_filter_host's
host-staged panels.  Panel 0 is checked bit-for-bit against the
device-resident filter of the same panel.  Prints one JSON line.

    python tools/host_panels_cfg3.py [--np 100] [--nx 256]
"""
import argparse
import json
import sys
import time
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1803_02156_b200 as cf  # noqa: E402


def mem_available_gb():
    for line in open("/proc/meminfo"):
        if line.startswith("MemAvailable:"):
            return int(line.split()[1]) / 2**20
    return 0.0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--nx", type=int, default=256)
    ap.add_argument("--np", type=int, default=100)
    ap.add_argument("--panels", type=int, default=4)
    a = ap.parse_args()
    nb, npan = 32, a.panels
    H = cf.topi_generate(cf.LatticeSpec(a.nx, a.nx, a.nx))
    n = H.n
    host_bytes = npan * n * nb * 16
    avail = mem_available_gb()
    if avail < host_bytes / 2**30 + 40:
        print(json.dumps({"skipped": f"host memory {avail:.0f} GiB < X {host_bytes / 2**30:.0f} GiB + 40"}))
        return
    dev = torch.device("cuda", 0)
    fc = cf.filter_coefficients(-0.35, 0.35, cf.spectral_map(-7.0, 7.0, 0.01), a.np)
    H.device_matrix(0)  # SELL build + upload outside the timed calls
    t0 = time.perf_counter()
    hostp = torch.empty((npan, n, nb), dtype=torch.complex128, pin_memory=True)
    pin_s = time.perf_counter() - t0
    P = cf.BlockVector(n, nb, nb, device=dev)
    for b in range(npan):
        cf.blockvec.random_fill_device(P, 42 + b)
        hostp[b].copy_(P.panel(0)[:n])
    # device-resident reference for panel 0 (same X0 bits)
    cf.blockvec.random_fill_device(P, 42)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    cf.apply_filter(H, P, fc)
    e1.record()
    torch.cuda.synchronize()
    panel_s = e0.elapsed_time(e1) / 1e3
    want = P.panel(0)[:n].cpu()
    del P
    torch.cuda.empty_cache()
    t0 = time.perf_counter()
    _, eta, _ = cf.apply_filter_host(H, hostp, fc)
    host_s = time.perf_counter() - t0
    same = bool(torch.equal(hostp[0], want))
    print(json.dumps({
        "what": f"cfg3-class lattice 4x{a.nx}^3 (n={n}), n_s={npan * nb} as {npan} host panels, n_p={a.np}, one GPU",
        "host_x_bytes": host_bytes, "pin_seconds": round(pin_s, 2), "seconds": round(host_s, 3),
        "device_panel_seconds": round(panel_s, 3), "ideal_seconds": round(npan * panel_s, 3),
        "overhead_vs_device_resident": round(host_s / (npan * panel_s) - 1.0, 4),
        "gflops": round(146.0 * n * nb * npan * (a.np - 2) / host_s / 1e9, 1),
        "panel0_bit_identical": same, "device_mem_peak_gb": round(torch.cuda.max_memory_allocated() / 1e9, 1)}))


if __name__ == "__main__":
    main()
