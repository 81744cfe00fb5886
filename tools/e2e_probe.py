"""cf_apply_filter_host at the configs[0] size (n_s = n_b = 8, pinned host X):
wall time per call over repeated calls, per kernel setting (cf_tuning "narrow"),
next to the device-resident cf_apply_filter.  One JSON line."""
import json
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1803_02156_b200 as cf  # noqa: E402
from paper_1803_02156_b200._lib import check, lib  # noqa: E402

H = cf.topi_generate(cf.LatticeSpec(64, 64, 40))
fc = cf.filter_coefficients(-0.7, 0.7, cf.spectral_map(-7.0, 7.0, 0.01), 100)
host = torch.empty((1, H.n, 8), dtype=torch.complex128, pin_memory=True)
host.copy_(torch.from_numpy(cf.seeded_random_host(H.n, 8, 8, 42)))
x0 = host.clone()
out = {}
for v in (1, 0, 1):
    check(lib.cf_tuning(b"narrow", v))
    ts = []
    for k in range(6):
        host.copy_(x0)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        cf.apply_filter_host(H, host, fc)
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    X = cf.BlockVector(H.n, 8, 8, cf.InitSeededRandom(42), device="cuda:0")
    cf.apply_filter(H, X, fc)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    cf.apply_filter(H, X, fc)
    torch.cuda.synchronize()
    out.setdefault(f"narrow={v}", []).append({"host_calls_s": [round(t, 4) for t in ts],
                                              "device_s": round(time.perf_counter() - t0, 4)})
check(lib.cf_tuning(b"narrow", 1))
print(json.dumps(out))
