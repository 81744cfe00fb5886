"""Interleaved A/B of cf_tuning knobs in one process on cfg2 (n_b = 32): one fused
chebfd_op step (M_CHEB, device time over 30 steps) and a whole apply_filter
(n_p = 200, groups of three).  Each argument is one variant: an integer (the
producer L2 prefetch "wpf") or comma-separated key=value pairs.

    python tools/wpf_ab.py 0 18 ...
    python tools/wpf_ab.py wpf=18,dict=1 wpf=18,dict=0
"""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1803_02156_b200 as cf  # noqa: E402
from paper_1803_02156_b200._lib import check, lib  # noqa: E402

def parse(a):
    if "=" not in a:
        return ((b"wpf", int(a)),)
    return tuple((k.encode(), int(v)) for k, v in (kv.split("=") for kv in a.split(",")))


vals = [parse(a) for a in sys.argv[1:]] or [parse("0"), parse("18")]
H = cf.topi_generate(cf.LatticeSpec(128, 128, 128))
n, nb = H.n, 32
s = cf.spectral_map(-7.0, 7.0, 0.01)
fc = cf.filter_coefficients(-0.35, 0.35, s, 200)
U = cf.BlockVector(n, nb, nb, cf.InitSeededRandom(1), device="cuda:0")
W = cf.BlockVector(n, nb, nb, cf.InitSeededRandom(2), device="cuda:0")
X = cf.BlockVector(n, nb, nb, cf.InitSeededRandom(3), device="cuda:0")
mom = cf.MomentSeries(40, nb, device="cuda:0")
Uv, Wv, Xv = cf.SubblockView(U, 0), cf.SubblockView(W, 0), cf.SubblockView(X, 0)


def ev():
    return torch.cuda.Event(enable_timing=True)


res = {v: {"step": [], "filter": []} for v in vals}
for rep in range(3):
    for v in vals:
        for key, x in v:
            check(lib.cf_tuning(key, x))
        for _ in range(3):
            cf.chebfd_op(H, s, Uv, Wv, Xv, 3, 0.01, mom)
        torch.cuda.synchronize()
        a, b = ev(), ev()
        a.record()
        for k in range(30):
            cf.swap_blocks(Wv, Uv)
            cf.chebfd_op(H, s, Uv, Wv, Xv, 3 + k % 30, 0.01, mom)
        b.record()
        torch.cuda.synchronize()
        res[v]["step"].append(a.elapsed_time(b) / 30)
        Xf = cf.BlockVector(n, nb, nb, cf.InitSeededRandom(42), device="cuda:0")
        torch.cuda.synchronize()
        a, b = ev(), ev()
        a.record()
        cf.apply_filter(H, Xf, fc)
        b.record()
        torch.cuda.synchronize()
        res[v]["filter"].append(a.elapsed_time(b) / 198)
        del Xf
for v in vals:
    print(f"{','.join(f'{k.decode()}={x}' for k, x in v):18s}  chebfd_op {np.median(res[v]['step']):.4f} ms  "
          f"filter per degree {np.median(res[v]['filter']):.4f} ms  (all: {[round(x, 3) for x in res[v]['filter']]})")
