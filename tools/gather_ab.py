"""Interleaved A/B of a cf_tuning knob on the register-gather kernel (n_b < 32):
device time per fused chebfd_op step (swap + step, CUDA events) on the cfg1
lattice (BASELINE configs[0], n_b = 8) and the cfg2 lattice at n_b = 8 / 16, and
per apply_filter degree on cfg1.  --ab KEY=V1,V2.  One JSON line."""
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
ap.add_argument("--ab", default="ko=0,64")
ap.add_argument("--rounds", type=int, default=5)
ap.add_argument("--reps", type=int, default=40)
a = ap.parse_args()
key, vals = a.ab.split("=")
vals = [int(v) for v in vals.split(",")]
cases = []
for dims, nb in (((64, 64, 40), 8), ((128, 128, 128), 8), ((128, 128, 128), 16)):
    H = cf.topi_generate(cf.LatticeSpec(*dims))
    fc = cf.filter_coefficients(-0.7, 0.7, cf.spectral_map(-7.0, 7.0, 0.01), 100)
    X, U, W = (cf.BlockVector(H.n, nb, nb, cf.InitSeededRandom(k), device="cuda:0") for k in (1, 2, 3))
    mom = cf.MomentSeries(100, nb, device="cuda:0")
    cases.append((f"{dims}_nb{nb}", H, fc, X, U, W, mom))
st = torch.cuda.current_stream()


def steps(H, fc, X, U, W, mom):
    Uv, Wv, Xv = cf.SubblockView(U, 0), cf.SubblockView(W, 0), cf.SubblockView(X, 0)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(st)
    for k in range(a.reps):
        cf.swap_blocks(Wv, Uv)
        cf.chebfd_op(H, fc.map, Uv, Wv, Xv, 3 + k % 90, 0.01, mom)
    e1.record(st)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / a.reps


res = {}
for r in range(a.rounds):
    for v in vals:
        check(lib.cf_tuning(key.encode(), v))
        d = res.setdefault(f"{key}={v}", {})
        for name, H, fc, X, U, W, mom in cases:
            d.setdefault(name, []).append(steps(H, fc, X, U, W, mom))
        H, fc, X = cases[0][1], cases[0][2], cases[0][3]
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        cf.apply_filter(H, X, fc)
        e1.record(st)
        torch.cuda.synchronize()
        d.setdefault("cfg1_filter_per_degree", []).append(e0.elapsed_time(e1) / 98)
print(json.dumps({"what": f"ms per fused step (median of {a.rounds} interleaved rounds)",
                  "results": {k: {c: round(float(np.median(x)), 4) for c, x in d.items()} for k, d in res.items()}}))
