"""apply_filter with per-step moment reductions (CHEBFD_MOM_BATCH=0) vs deferred,
batched reductions (default): device ms per degree on the configs[0] and configs[1]
lattices, plus a digest of the moments and the filtered panel (must match between
the two settings: the batched reduction sums in the same order).  Run once per
setting; prints one JSON line."""
import hashlib
import json
import os
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1803_02156_b200 as cf  # noqa: E402


def digest(*ts):
    h = hashlib.sha256()
    for t in ts:
        h.update(t.detach().cpu().contiguous().numpy().tobytes())
    return h.hexdigest()[:16]


out = {"mom_batch": os.environ.get("CHEBFD_MOM_BATCH", "default")}
for name, (nx, ny, nz, nb, np_, reps) in {"cfg1": (64, 64, 40, 8, 100, 5), "cfg2": (128, 128, 128, 32, 200, 2)}.items():
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
    out[name] = {"ms_per_degree": round(ts[len(ts) // 2], 5), "min": round(ts[0], 5),
                 "digest": digest(mom.eta, mom.mu, X.panel(0))}
    del H, X, X0
    torch.cuda.empty_cache()
print(json.dumps(out))
