"""Locality / occupancy sweep of the fused step at cfg2 (one process per setting)."""
import json
import os
import subprocess
import sys

CODE = r'''
import os, sys, time, json, torch
sys.path.insert(0, os.getcwd())
import paper_1803_02156_b200 as cf
H = cf.topi_generate(cf.LatticeSpec(128, 128, 128))
n, nb = H.n, 32
dm = H.device_matrix(0)
U = cf.BlockVector(n, nb, nb, device="cuda:0"); W = cf.BlockVector(n, nb, nb, device="cuda:0"); X = cf.BlockVector(n, nb, nb, device="cuda:0")
for t in (U, W, X): t.panel(0).normal_()
mom = cf.MomentSeries(500, nb, device="cuda:0")
s = cf.ShiftScale(0.14144271570014144, 0.0)
Uv, Wv, Xv = cf.SubblockView(U, 0), cf.SubblockView(W, 0), cf.SubblockView(X, 0)
def step(p):
    cf.swap_blocks(Wv, Uv); cf.chebfd_op(H, s, Uv, Wv, Xv, 3 + p % 400, 0.001, mom)
for p in range(3): step(p)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
K = int(os.environ.get("K", "20"))
e0.record()
for p in range(K): step(p)
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / K
print(json.dumps({"ms": ms, "GBs": n * (260 + 80 * nb) / ms / 1e6, "info": dm.info()}))
'''

settings = [json.loads(a) for a in sys.argv[1:] if a.startswith("{")] or [
    {"CHEBFD_TILE": "38"}, {"CHEBFD_TILE": "16"}, {"CHEBFD_TILE": "0"}, {"CHEBFD_TILE": "16", "CHEBFD_UNIT_CHUNKS": "8"},
]
ncu = "--ncu" in sys.argv
for st in settings:
    env = dict(os.environ, **st)
    cmd = [sys.executable, "-c", CODE]
    if ncu:
        env["K"] = "2"
        cmd = ["ncu", "--metrics", "dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,"
               "lts__t_sector_hit_rate.pct", "-k", "sell_b4_kernel", "-s", "3", "-c", "1", "--csv"] + cmd
    r = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=600)
    out = r.stdout.strip().splitlines()
    print(json.dumps(st), "|", " ".join(out[-6:]) if ncu else (out[-1] if out else r.stderr[-400:]), flush=True)
