"""One SVQB + Rayleigh-Ritz pass at configs[4]'s block size on the cfg2 lattice
(n = 8.4M, n_s = 128 as 4 panels of 32) for ncu captures of the solver kernels
(gram_kernel, rotate_kernel, resid_kernel) and their device times (CUDA events)."""
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1803_02156_b200 as cf  # noqa: E402

H = cf.topi_generate(cf.LatticeSpec(128, 128, 128))
H.device_matrix(0)
X = cf.BlockVector(H.n, 128, 32, device="cuda:0")
cf.blockvec.random_fill_device(X, 42)
out = {}
for rep in range(2):
    e = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    e[0].record()
    S = cf.gram_matrix(X)
    e[1].record()
    Q, rank = cf.orthogonalize_svqb(X)
    e[2].record()
    rr = cf.rayleigh_ritz(H, Q)
    e[3].record()
    torch.cuda.synchronize()
    out = {"gram_128x128_ms": e[0].elapsed_time(e[1]), "svqb_ms": e[1].elapsed_time(e[2]),
           "rayleigh_ritz_ms": e[2].elapsed_time(e[3]), "rank": rank, "n": H.n,
           "gram_bytes": H.n * 128 * 16, "max_residual": float(rr.residuals.max())}
print(json.dumps(out))
