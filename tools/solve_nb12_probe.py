"""bench.py's chebfd_solve leg (configs[0] lattice, n_s = n_b = 12, n_p = 1500) timed
twice per kernel setting (cf_tuning "narrow" 1 / 0) in one process, with the
per-restart phase times (filter, SVQB, Rayleigh-Ritz).  One JSON line."""
import json
import sys
import time
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1803_02156_b200 as cf  # noqa: E402
from paper_1803_02156_b200._lib import check, lib  # noqa: E402

Hs = cf.topi_generate(cf.LatticeSpec(64, 64, 40))
opt = cf.SolveOptions(n_s=12, n_b=12, n_p=1500, max_restarts=12, spectral_bounds=(-4.0, 4.0))
Hs.device_matrix(0)
out = {"narrow_eligible": Hs.device_matrix(0).info()["narrow"]}
for v in (1, 0, 1, 0):
    check(lib.cf_tuning(b"narrow", v))
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    res = cf.chebfd_solve(Hs, -0.05, 0.05, opt)
    torch.cuda.synchronize()
    out.setdefault(f"narrow={v}", []).append({"seconds": round(time.perf_counter() - t0, 3), "restarts": res.iterations,
                                              "found": int(len(res.eigenvalues)),
                                              "phase_ms": [[round(x, 1) for x in p] for p in res.phase_ms.tolist()]})
check(lib.cf_tuning(b"narrow", 1))
print(json.dumps(out))
