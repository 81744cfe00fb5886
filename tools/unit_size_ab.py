"""Work-unit size (chunks per unit, CHEBFD_UNIT_CHUNKS) vs the fused step: device
ms per degree of apply_filter on the configs[0] and configs[1] lattices.  Run once
per setting; prints one JSON line with the unit count and a digest of the result."""
import hashlib
import json
import os
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1803_02156_b200 as cf  # noqa: E402

out = {"unit_chunks": os.environ.get("CHEBFD_UNIT_CHUNKS", "default")}
which = sys.argv[1:] or ["cfg1", "cfg2"]
for name, (nx, ny, nz, nb, np_, reps) in {"cfg1": (64, 64, 40, 8, 100, 7), "cfg2": (128, 128, 128, 32, 100, 3)}.items():
    if name not in which:
        continue
    H = cf.topi_generate(cf.LatticeSpec(nx, ny, nz))
    fc = cf.filter_coefficients(-0.7, 0.7, cf.spectral_map(-7.0, 7.0, 0.01), np_)
    X = cf.BlockVector(H.n, nb, nb, device="cuda:0")
    cf.blockvec.random_fill_device(X, 42)
    X0 = X.panel(0).clone()
    cf.apply_filter(H, X, fc)
    ts = []
    for _ in range(reps):
        X.panel(0).copy_(X0)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        mom = cf.apply_filter(H, X, fc)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) / (np_ - 2))
    ts.sort()
    h = hashlib.sha256(mom.eta.cpu().numpy().tobytes() + X.panel(0).cpu().numpy().tobytes()).hexdigest()[:12]
    out[name] = {"ms_per_degree": round(ts[len(ts) // 2], 5), "min": round(ts[0], 5),
                 "units": H.device_matrix(0).info()["units"],
                 "digest": h}
    del H, X, X0
    torch.cuda.empty_cache()
print(json.dumps(out))
