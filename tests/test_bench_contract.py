"""bench.py keeps the driver's JSON contract: the reference arm on CPU (tiny
lattice, oracle/_ref), and the B200 arm on a GPU (small lattice)."""
import json
import subprocess
import sys
from pathlib import Path

import pytest

import oracle as orc

ROOT = Path(__file__).resolve().parents[1]
BASE_KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
             "vs_baseline", "dtype", "data", "config"}


def _run(args, timeout=600):
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), *args], capture_output=True, text=True,
                       timeout=timeout, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    return json.loads(r.stdout.strip().splitlines()[-1])


@pytest.mark.skipif(orc.REF is None, reason="oracle/_ref not built")
def test_reference_arm_json():
    d = _run(["--impl", "reference", "--nx", "8", "--ny", "8", "--nz", "8", "--steps", "3", "--warmup", "3"])
    assert d["impl"] == "reference" and BASE_KEYS <= set(d)
    assert d["value"] > 0 and d["cpu_baseline"]["kind"] == "reference" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]


@pytest.mark.gpu
def test_b200_arm_json():
    d = _run(["--nx", "16", "--ny", "16", "--nz", "16", "--steps", "5", "--warmup", "3", "--degree", "20",
              "--e2e-steps", "1", "--cpu-steps", "1", "--no-solve", "--leg-nxy", "16", "--leg-nz", "8"])
    assert BASE_KEYS <= set(d) and d["n_gpus"] == 1 and d["steps"] == 5 and d["warmup"] == 3
    assert d["value"] > 0 and d["higher_is_better"] is True
    r = d["roofline"]
    assert r["bound"] == "hbm" and 0 < r["frac"] == pytest.approx(r["achieved"] / r["peak"], rel=1e-3)
    assert d["e2e"]["value"] > 0 and d["e2e"]["h2d_bytes_per_step"] > 0 and d["e2e"]["d2h_bytes_per_step"] > 0
    assert d["cpu_baseline"]["value"] > 0 and d["gpu_launches"] == 10
    assert set(d["clocks"]) >= {"sm_mhz", "sm_max_mhz", "reasons"}
    leg = d["leg_1e8"]
    assert leg["n_total"] == 4 * 16 * 16 * 8 and leg["parallel_efficiency"] == 1.0 and leg["gflops"] > 0


@pytest.mark.gpu
def test_b200_arm_two_ranks_sharing_the_gpu():
    """The N>1 path end to end (torchrun, 2 ranks on the box's one GPU, gloo for
    the host collectives): fused halo + per-neighbour flags, the >=1e8-row leg's
    code path at a small size, one JSON line from rank 0."""
    import os
    env = dict(os.environ, CHEBFD_DIST_BACKEND="gloo")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2", "--master-addr",
           "127.0.0.1", "--master-port", "29641", str(ROOT / "bench.py"), "--gpus", "2", "--nx", "16", "--ny", "16",
           "--nz", "8", "--steps", "4", "--warmup", "3", "--degree", "12", "--e2e-steps", "1", "--leg-nxy", "16",
           "--leg-nz", "6"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT, env=env)
    assert r.returncode == 0, r.stderr[-3000:]
    d = json.loads([ln for ln in r.stdout.splitlines() if ln.startswith("{")][-1])
    assert d["n_gpus"] == 2 and d["value"] > 0 and d["e2e"]["value"] > 0
    leg = d["leg_1e8"]
    assert leg["n_total"] == 4 * 16 * 16 * 12 and 0 < leg["parallel_efficiency"]


def test_filter_bytes_accounting():
    """bench.filter_bytes: cheb_init (2 + 4 panel passes, 2 matrix sweeps) plus 3
    passes per degree step and 2 more on the steps that update X; every third
    degree updates X, so n_p = 500 averages 3 + 2/3 passes per degree."""
    sys.path.insert(0, str(ROOT))
    import bench
    n, nb = 1000, 32
    panel = 16 * n * nb
    assert bench.filter_bytes(n, nb, 2) == 2 * 260 * n + 6 * panel
    assert bench.filter_bytes(n, nb, 5) == 5 * 260 * n + 6 * panel + (3 + 3 + 5) * panel
    per_degree = (bench.filter_bytes(n, nb, 500) - bench.filter_bytes(n, nb, 2)) / 498
    assert per_degree == pytest.approx(260 * n + (3 + 2 / 3) * panel, rel=1e-3)
    assert per_degree < bench.step_bytes(n, nb)
