"""chebfd_solve with the reference's default block width (n_s = 32, n_b = 8) on the
cfg1 lattice: the caller's panel width (CHEBFD_SOLVE_WIDE=0) against the solver's
own 32-wide panels.  Run once per setting; prints one JSON line."""
import json
import os
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1803_02156_b200 as cf  # noqa: E402

H = cf.topi_generate(cf.LatticeSpec(64, 64, 40))
H.device_matrix(0)
opt = cf.SolveOptions(n_s=32, n_b=8, n_p=1200, max_restarts=12, spectral_bounds=(-4.0, 4.0))
out = []
for rep in range(2):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    r = cf.chebfd_solve(H, 0.05, 0.105, opt)
    torch.cuda.synchronize()
    out.append(time.perf_counter() - t0)
print(json.dumps({"wide": os.environ.get("CHEBFD_SOLVE_WIDE", "1"), "seconds": [round(x, 3) for x in out],
                  "restarts": r.iterations, "converged": r.converged, "found": len(r.eigenvalues),
                  "eig_range": [float(np.min(r.eigenvalues)), float(np.max(r.eigenvalues))] if len(r.eigenvalues) else None,
                  "filter_ms": [round(x, 1) for x in r.phase_ms[:, 0].tolist()]}))
