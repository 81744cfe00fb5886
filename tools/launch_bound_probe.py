"""Is the per-step bench launch-bound at configs[0] size?  K fused chebfd_op steps
(swap + step, as bench.py runs them) timed with CUDA events three ways:
(a) as bench.py does (the host enqueues while the GPU runs), (b) the same calls
queued behind a GPU sleep so that the host has enqueued them all before the GPU
starts (pure device time), (c) the host's own enqueue time per step.  One JSON line."""
import json
import sys
import time
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1803_02156_b200 as cf  # noqa: E402

nx, ny, nz, nb = (int(v) for v in (sys.argv[1:5] if len(sys.argv) > 4 else (64, 64, 40, 8)))
K = 100
H = cf.topi_generate(cf.LatticeSpec(nx, ny, nz))
fc = cf.filter_coefficients(-0.7, 0.7, cf.spectral_map(-7.0, 7.0, 0.01), 100)
X, U, W = (cf.BlockVector(H.n, nb, nb, cf.InitSeededRandom(k), device="cuda:0") for k in (1, 2, 3))
mom = cf.MomentSeries(100, nb, device="cuda:0")
Uv, Wv, Xv = cf.SubblockView(U, 0), cf.SubblockView(W, 0), cf.SubblockView(X, 0)
st = torch.cuda.current_stream()


def steps(k0):
    for k in range(K):
        cf.swap_blocks(Wv, Uv)
        cf.chebfd_op(H, fc.map, Uv, Wv, Xv, 3 + (k0 + k) % 90, 0.01, mom)


def timed(prefill):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if prefill:
        torch.cuda._sleep(int(2e9 * 0.05))  # ~50 ms of GPU spinning while the host enqueues
    e0.record(st)
    t0 = time.perf_counter()
    steps(0)
    host = (time.perf_counter() - t0) / K
    e1.record(st)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / K, host * 1e3


def shifts():
    for k in range(K):
        cf.spmmv_shifted(H, fc.map, Uv if k % 2 else Wv, Wv if k % 2 else Uv)


def timed_fn(fn):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda._sleep(int(2e9 * 0.05))
    e0.record(st)
    fn()
    e1.record(st)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / K


steps(0)
shifts()
res = {"lattice": [nx, ny, nz], "n_b": nb, "steps": K}
from paper_1803_02156_b200._lib import check, lib  # noqa: E402
for r in range(3):
    res.setdefault("spmmv_shifted_prefilled_ms", []).append(round(timed_fn(shifts), 5))
    check(lib.cf_tuning(b"pdl", 0))
    res.setdefault("pdl_off_prefilled_ms", []).append(round(timed_fn(lambda: steps(0)), 5))
    check(lib.cf_tuning(b"pdl", 1))
for r in range(3):
    a, ha = timed(False)
    b, hb = timed(True)
    res.setdefault("as_bench_ms", []).append(round(a, 5))
    res.setdefault("prefilled_ms", []).append(round(b, 5))
    res.setdefault("host_enqueue_ms", []).append(round(ha, 5))
print(json.dumps(res))
