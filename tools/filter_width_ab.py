"""apply_filter on n_b = 8 / 12 / 16 / 24 / 64 panels (n_s = 32, or 96 for 12 / 24)
of the cfg2 lattice: panel-by-panel (CHEBFD_FILTER_WIDE=0) vs packed into 32-wide panels.  Run once
per setting; prints one JSON line (device time per degree)."""
import json
import os
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1803_02156_b200 as cf  # noqa: E402

H = cf.topi_generate(cf.LatticeSpec(128, 128, 128))
fc = cf.filter_coefficients(-0.7, 0.7, cf.spectral_map(-7.0, 7.0, 0.01), 100)
out = {"wide": os.environ.get("CHEBFD_FILTER_WIDE", "1")}
for nb in (8, 12, 16, 24, 64):
    ns = 96 if nb in (12, 24) else max(32, nb)
    X = cf.BlockVector(H.n, ns, nb, device="cuda:0")
    cf.blockvec.random_fill_device(X, 42)
    cf.apply_filter(H, X, fc)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    cf.apply_filter(H, X, fc)
    e1.record()
    torch.cuda.synchronize()
    out[f"nb{nb}_ms_per_degree_per_32_columns"] = round(e0.elapsed_time(e1) / 98 / (ns // 32), 4)
print(json.dumps(out))
