"""Full-filter parity at BASELINE configs[1] size against the reference itself.

cfg2 lattice 4x128^3 (n = 8,388,608), n_s = n_b = 32, bench-kernel inputs
(tools/chebfilter.cpp:277-294), degree n_p (default 500, the configs[1] degree):
the reference's apply_filter (oracle/_ref, its headers compiled unchanged, all
host cores) against cf.apply_filter on the GPU.  Writes profiles/parity_cfg2_np<N>.json.
Tolerance (north_star): max|X_gpu - X_ref| / max|X_ref| <= 1e-10; moments 1e-12.
"""
import ctypes as C
import json
import os
import sys
import time
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
import oracle as orc  # noqa: E402  (checker)
import paper_1803_02156_b200 as cf  # noqa: E402

np_ = int(sys.argv[1]) if len(sys.argv) > 1 else 500
nx = ny = nz = 128
ns = nb = 32
threads = min(os.cpu_count() or 1, 64)
os.environ["CHEBFILTER_THREADS"] = str(threads)

H = cf.topi_generate(cf.LatticeSpec(nx, ny, nz))
lo, hi = cf.gershgorin_bounds(H)
span = hi - lo
fc = cf.filter_coefficients(lo + 0.45 * span, lo + 0.55 * span, cf.spectral_map(lo, hi, 0.01), np_)
X0 = cf.seeded_random_host(H.n, ns, nb, 42)

t0 = time.perf_counter()
X = cf.BlockVector(H.n, ns, nb, cf.InitSeededRandom(42), device="cuda:0")
mom = cf.apply_filter(H, X, fc)
torch.cuda.synchronize()
t_gpu = time.perf_counter() - t0
Xg = X.panels_numpy()
eta_g = mom.eta.cpu().numpy().reshape(np_ - 2, ns)
mu_g = mom.mu.cpu().numpy().reshape(np_ - 2, ns)
del X

R = orc.RefMatrix.topi(nx, ny, nz)
Xr = np.ascontiguousarray(X0, np.complex128).copy()
eta_r = np.zeros((np_ - 2) * ns, np.complex128)
mu_r = np.zeros_like(eta_r)
t0 = time.perf_counter()
st = orc.REF.ref_apply_filter(R.h, ns, nb, Xr.ctypes.data, np_, fc.c.ctypes.data, fc.g.ctypes.data, fc.map.alpha,
                              fc.map.beta, eta_r.ctypes.data, mu_r.ctypes.data)
t_ref = time.perf_counter() - t0
assert st == 0


def rel(a, b):
    return float(np.abs(a - b).max() / np.abs(b).max())


out = {"config": f"topi 4x{nx}x{ny}x{nz} (n={H.n}), n_s=n_b={ns}, n_p={np_}, bench-kernel inputs",
       "x_max_rel": rel(Xg, Xr), "eta_max_rel": rel(eta_g, eta_r.reshape(np_ - 2, ns)),
       "mu_max_rel": rel(mu_g, mu_r.reshape(np_ - 2, ns)), "tolerance": {"x": 1e-10, "moments": 1e-12},
       "gpu_seconds_incl_upload": round(t_gpu, 2), "reference_seconds": round(t_ref, 1), "reference_threads": threads}
out["pass"] = out["x_max_rel"] <= 1e-10 and out["eta_max_rel"] <= 1e-12 and out["mu_max_rel"] <= 1e-12
print(json.dumps(out))
(ROOT / "gpurun_out").mkdir(exist_ok=True)
(ROOT / "gpurun_out" / f"parity_cfg2_np{np_}.json").write_text(json.dumps(out, indent=1))
