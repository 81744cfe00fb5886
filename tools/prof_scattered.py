"""Fused steps on the random scattered Hermitian matrix of tools/general_sparsity.py
(n = 8.4M, 13 nnz per row, register-gather kernel) for an ncu capture."""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent))
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1803_02156_b200 as cf  # noqa: E402
from general_sparsity import hermitian_from_pairs  # noqa: E402

rng = np.random.default_rng(1)
n, k = 4 * 128 ** 3, 6
rows = np.repeat(np.arange(n), k)
H = hermitian_from_pairs(n, rows, rng.integers(0, n, n * k), rng.normal(size=n * k) + 1j * rng.normal(size=n * k),
                         rng.normal(size=n))
s = cf.spectral_map(*cf.gershgorin_bounds(H), 0.01)
X, U, W = (cf.BlockVector(H.n, 32, 32, device="cuda:0") for _ in range(3))
mom = cf.MomentSeries(20, 32, device="cuda:0")
Uv, Wv, Xv = cf.SubblockView(U, 0), cf.SubblockView(W, 0), cf.SubblockView(X, 0)
for p in range(3, 8):
    cf.swap_blocks(Wv, Uv)
    cf.chebfd_op(H, s, Uv, Wv, Xv, p, 0.01, mom)
torch.cuda.synchronize()
print(cf.sparse.sell_layout_stats(H))
