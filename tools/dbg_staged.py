"""A/B check of the chunk-staged kernel against the register-gather kernel on a
full-size fused step: whole W / X panels and the moments."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1803_02156_b200 as cf  # noqa: E402
from paper_1803_02156_b200._lib import check, lib  # noqa: E402

nx = int(sys.argv[1]) if len(sys.argv) > 1 else 128
H = cf.topi_generate(cf.LatticeSpec(nx, nx, nx))
n, nb = H.n, 32
dev = "cuda:0"
g = torch.Generator(device=dev).manual_seed(7)
U = torch.randn(n, nb, dtype=torch.complex128, device=dev, generator=g)
W = torch.randn(n, nb, dtype=torch.complex128, device=dev, generator=g)
X = torch.randn(n, nb, dtype=torch.complex128, device=dev, generator=g)
s = cf.ShiftScale(0.14144271570014144, 0.0)
out = {}
for staged in (0, 1):
    check(lib.cf_tuning(b"staged", staged))
    Ub, Wb, Xb = (cf.BlockVector(n, nb, nb, device=dev) for _ in range(3))
    Ub._panels[0], Wb._panels[0], Xb._panels[0] = U.clone(), W.clone(), X.clone()
    mom = cf.MomentSeries(3, nb, device=dev)
    cf.chebfd_op(H, s, cf.SubblockView(Ub, 0), cf.SubblockView(Wb, 0), cf.SubblockView(Xb, 0), 3, 0.01, mom)
    torch.cuda.synchronize()
    out[staged] = (Wb.panel(0), Xb.panel(0), mom.eta.clone(), mom.mu.clone())
w0, x0, e0, m0 = out[0]
w1, x1, e1, m1 = out[1]
dw = (w0 - w1).abs().amax(1)
bad = torch.nonzero(dw > 1e-12 * w0.abs().max()).flatten()
print("W max diff", dw.max().item(), "bad rows", bad.numel(), bad[:20].tolist())
print("X max diff", (x0 - x1).abs().max().item())
eta_ref = (w1.conj() * U).sum(0)
print("eta diff staged vs nonstaged", (e0 - e1).abs().max().item(), "staged vs torch", (e1 - eta_ref).abs().max().item(),
      "nonstaged vs torch", (e0 - (w0.conj() * U).sum(0)).abs().max().item())
print("mu diff", (m0 - m1).abs().max().item(), "mu staged vs torch", (m1 - (U.conj() * U).sum(0)).abs().max().item())
# which block-rows' contributions explain the moment difference?
d = (m1 - m0).real
contrib = (U.conj() * U).real.view(-1, 4, nb).sum(1)  # per block-row
for sign in (1, -1):
    err = (contrib - sign * d).abs().amax(1)
    best = torch.topk(-err, 3)
    print("sign", sign, "best block-rows", best.indices.tolist(), "residual", (-best.values).tolist())
# multiple of a unit? per-unit would be 8 chunks x 8 block-rows in locality order
print("d[0:4]", d[:4].tolist())
