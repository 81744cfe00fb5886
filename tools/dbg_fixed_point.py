import numpy as np, torch, sys
sys.path.insert(0, '.')
import paper_1803_02156_b200 as cf
H = cf.diagonal_matrix([1.0] * 5)
s = cf.ShiftScale(1.0, 0.0)
X = cf.BlockVector(5, 2, 2, cf.InitSeededRandom(55), device="cuda:0")
x0 = X.to_numpy().copy()
norms = (np.abs(x0) ** 2).sum(axis=0)
U, W = cf.BlockVector(5, 2, 2, device="cuda:0"), cf.BlockVector(5, 2, 2, device="cuda:0")
cf.cheb_init(H, s, cf.SubblockView(X, 0), cf.SubblockView(U, 0), cf.SubblockView(W, 0), 1.0, 0.0, 0.0)
print("U", U.to_numpy()); print("x0", x0); print("W", W.to_numpy()); print("X", X.to_numpy())
mom = cf.MomentSeries(7, 2, device="cuda:0")
for p in range(3, 8):
    cf.swap_blocks(cf.SubblockView(W, 0), cf.SubblockView(U, 0))
    cf.chebfd_op(H, s, cf.SubblockView(U, 0), cf.SubblockView(W, 0), cf.SubblockView(X, 0), p, 0.0, mom)
    print(p, "U", U.to_numpy()[:, 0], "W", W.to_numpy()[:, 0])
print("mu", mom.mu.cpu().numpy(), "norms", norms)
print("eta", mom.eta.cpu().numpy())
