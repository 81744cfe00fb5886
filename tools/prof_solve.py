"""Timing of chebfd_solve on the cfg1 lattice (3 runs) and of one apply_filter at the same degree."""
import sys, time, torch
sys.path.insert(0, '/root/repo')
import paper_1803_02156_b200 as cf
H = cf.topi_generate(cf.LatticeSpec(64, 64, 40))
H.device_matrix(0)
opt = cf.SolveOptions(n_s=12, n_b=12, n_p=1500, max_restarts=12, spectral_bounds=(-4.0, 4.0))
for rep in range(3):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    res = cf.chebfd_solve(H, -0.05, 0.05, opt)
    torch.cuda.synchronize(); t1 = time.perf_counter()
    print("solve", rep, round(t1 - t0, 3), res.iterations, res.converged)
fc = cf.filter_coefficients(-0.05, 0.05, cf.spectral_map(-4.0, 4.0, 0.01), 1500)
X = cf.BlockVector(H.n, 12, 12, cf.InitSeededRandom(42), device="cuda:0")
for rep in range(2):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    cf.apply_filter(H, X, fc)
    torch.cuda.synchronize(); print("filter", round(time.perf_counter() - t0, 3))
