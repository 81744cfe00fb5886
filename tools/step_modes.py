"""Device time of each degree-step kind on cfg2 (topi 4x128^3, n_b = 32) and of
a whole apply_filter, interleaved over rounds (clocks drift under the power cap).
Prints one JSON line; --ab KEY=V1,V2 alternates a cf_tuning knob.

  kind 0 plain chebfd_op (M_CHEB), 1 no X update (M_CHEB_NOX), 3 X for three degrees (M_CHEB_X3)
"""
import argparse
import json
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1803_02156_b200 as cf  # noqa: E402
from paper_1803_02156_b200._lib import check, lib  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--nx", type=int, default=128)
ap.add_argument("--nz", type=int, default=128)
ap.add_argument("--nb", type=int, default=32)
ap.add_argument("--reps", type=int, default=20)
ap.add_argument("--rounds", type=int, default=3)
ap.add_argument("--np", type=int, default=500)
ap.add_argument("--ab", default="")
args = ap.parse_args()

H = cf.topi_generate(cf.LatticeSpec(args.nx, args.nx, args.nz))
lo, hi = cf.gershgorin_bounds(H)
span = hi - lo
fc = cf.filter_coefficients(lo + 0.45 * span, lo + 0.55 * span, cf.spectral_map(lo, hi, 0.01), args.np)
n, nb = H.n, args.nb
X = cf.BlockVector(n, nb, nb, device="cuda:0")
cf.blockvec.random_fill_device(X, 42)
U = cf.BlockVector(n, nb, nb, device="cuda:0")
W = cf.BlockVector(n, nb, nb, device="cuda:0")
s = fc.map
Xv, Uv, Wv = cf.SubblockView(X, 0), cf.SubblockView(U, 0), cf.SubblockView(W, 0)
cf.cheb_init(H, s, Xv, Uv, Wv, 0.1, 0.2, 0.3)
mom = cf.MomentSeries(args.np, nb, device="cuda:0")
st = torch.cuda.current_stream()


def steps(kind):
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    ev0.record(st)
    for k in range(args.reps):
        cf.swap_blocks(Wv, Uv)
        cf.kernels.chebfd_step(H, s, Uv, Wv, Xv, (3 + k % 50, kind, 0.01, 0.02, 0.03), mom)
    ev1.record(st)
    torch.cuda.synchronize()
    return ev0.elapsed_time(ev1) / args.reps


def filt():
    Xf = cf.BlockVector(n, nb, nb, device="cuda:0")
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    ev0.record(st)
    cf.apply_filter(H, Xf, fc)
    ev1.record(st)
    torch.cuda.synchronize()
    return ev0.elapsed_time(ev1) / (args.np - 2)


variants = [None]
if args.ab:
    key, vals = args.ab.split("=")
    variants = [(key, int(v)) for v in vals.split(",")]
res = {}
for r in range(args.rounds):
    for v in variants:
        if v:
            check(lib.cf_tuning(v[0].encode(), v[1]))
        name = "default" if v is None else f"{v[0]}={v[1]}"
        d = res.setdefault(name, {"plain": [], "nox": [], "x3": [], "filter_per_degree": []})
        d["plain"].append(steps(0))
        d["nox"].append(steps(1))
        d["x3"].append(steps(3))
        d["filter_per_degree"].append(filt())
        print(name, {m: round(x[-1], 4) for m, x in d.items()}, flush=True)
out = {k: {m: round(float(np.median(x)), 4) for m, x in d.items()} for k, d in res.items()}
print(json.dumps({"what": f"ms per step, topi 4x{args.nx}x{args.nx}x{args.nz}, n_b={nb}, median of {args.rounds}",
                  "results": out}))
