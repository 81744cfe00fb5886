"""Two apply_filter calls on cfg2 (n_b = 32, n_p = 12) for ncu captures of the
degree-step kernels (sell_b4_staged_kernel<4> = no X update, <6> = X updated for
three degrees, <3> = the plain remainder step)."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1803_02156_b200 as cf  # noqa: E402

H = cf.topi_generate(cf.LatticeSpec(128, 128, 128))
lo, hi = cf.gershgorin_bounds(H)
span = hi - lo
fc = cf.filter_coefficients(lo + 0.45 * span, lo + 0.55 * span, cf.spectral_map(lo, hi, 0.01), 12)
X = cf.BlockVector(H.n, 32, 32, cf.InitSeededRandom(42), device="cuda:0")
for _ in range(2):
    cf.apply_filter(H, X, fc)
torch.cuda.synchronize()
print("ok")
