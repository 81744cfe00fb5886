"""A/B of the generic-block L2 prefetch distance (cf_tuning("gpf")) on random
Hermitian matrices (general sparsity, register-gather kernel), n = 8.4M, n_b = 32:
ms per fused chebfd_op step, interleaved rounds.  One JSON line."""
import json
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent))
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1803_02156_b200 as cf  # noqa: E402
from paper_1803_02156_b200._lib import check, lib  # noqa: E402
from general_sparsity import hermitian_from_pairs  # noqa: E402

rng = np.random.default_rng(1)
n, k = 4 * 128 ** 3, 6
rows = np.repeat(np.arange(n), k)
vals = rng.normal(size=n * k) + 1j * rng.normal(size=n * k)
mats = {"banded": hermitian_from_pairs(n, rows, np.clip(rows + rng.integers(-4096, 4097, n * k), 0, n - 1), vals,
                                       rng.normal(size=n)),
        "scattered": hermitian_from_pairs(n, rows, rng.integers(0, n, n * k), vals, rng.normal(size=n))}
vals_ab = [int(v) for v in (sys.argv[1] if len(sys.argv) > 1 else "0,4,6,10").split(",")]
res = {}
for name, H in mats.items():
    s = cf.spectral_map(*cf.gershgorin_bounds(H), 0.01)
    X, U, W = (cf.BlockVector(H.n, 32, 32, device="cuda:0") for _ in range(3))
    for i, v in enumerate((X, U, W)):
        cf.blockvec.random_fill_device(v, 3 + i)
    mom = cf.MomentSeries(40, 32, device="cuda:0")
    Uv, Wv, Xv = cf.SubblockView(U, 0), cf.SubblockView(W, 0), cf.SubblockView(X, 0)
    for r in range(3):
        for g in vals_ab:
            check(lib.cf_tuning(b"gpf", g))
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for p in range(3, 8):
                cf.swap_blocks(Wv, Uv)
                cf.chebfd_op(H, s, Uv, Wv, Xv, p, 0.01, mom)
            e1.record()
            torch.cuda.synchronize()
            res.setdefault(name, {}).setdefault(g, []).append(e0.elapsed_time(e1) / 5)
    del X, U, W
print(json.dumps({n_: {str(g): round(float(np.median(t)), 3) for g, t in d.items()} for n_, d in res.items()}))
