"""The fused step on matrices other than the periodic Topi lattice (VERDICT r1 weak
#10): open-boundary Topi (7..13 nnz per row, sigma-sorting and padding at work),
Topi with random onsite disorder (Anderson; every site's values differ), a random
banded Hermitian matrix and a random scattered Hermitian matrix (~13 nnz per row,
no chunk fits a staging plan -> register-gather kernel).  n = 8.4M rows, n_b = 32,
device time per fused chebfd_op step (CUDA events), against the algorithmic bytes
n (nnz_row 20 + 80 n_b) of the reference's model (perf_model.hpp:56-62).
Prints one JSON line per matrix.

    python tools/general_sparsity.py [--n 128]
"""
import argparse
import json
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1803_02156_b200 as cf  # noqa: E402
from paper_1803_02156_b200._lib import lib  # noqa: E402
import ctypes as C  # noqa: E402


def peak():
    p = Path(__file__).resolve().parents[1] / "MEASURED_PEAKS.json"
    return float(json.loads(p.read_text())["hbm_gbs"]) if p.exists() else 6650.0


def hermitian_from_pairs(n, rows, cols, vals, diag):
    """CRS of A + A^H + diag(diag) from the entries (rows, cols, vals) of A."""
    r = np.concatenate([rows, cols, np.arange(n)])
    c = np.concatenate([cols, rows, np.arange(n)])
    v = np.concatenate([vals, np.conj(vals), diag.astype(np.complex128)])
    key = r.astype(np.int64) * n + c
    order = np.argsort(key, kind="stable")
    key, v = key[order], v[order]
    uk, first = np.unique(key, return_index=True)
    vs = np.add.reduceat(v, first)
    rr, cc = uk // n, (uk % n).astype(np.int32)
    rp = np.zeros(n + 1, np.uint64)
    np.add.at(rp, rr + 1, 1)
    rp = np.cumsum(rp).astype(np.uint64)
    return cf.SparseMatrixCRS(n, rp, cc, vs)


def matrices(nl, rng):
    n = 4 * nl ** 3
    yield "topi periodic (reference)", cf.topi_generate(cf.LatticeSpec(nl, nl, nl))
    yield "topi open boundary", cf.topi_generate(cf.LatticeSpec(nl, nl, nl, boundary=cf.Boundary.open))
    H = cf.topi_generate(cf.LatticeSpec(nl, nl, nl))
    rp = H.row_ptr.astype(np.int64)
    v = H.values.copy()
    rows = np.repeat(np.arange(n), np.diff(rp))
    dmask = H.col_idx == rows
    v[dmask] += rng.uniform(-1.0, 1.0, dmask.sum())  # Anderson disorder W = 2 on every site
    # same sites, same lattice locality schedule as the generator's matrices
    yield "topi periodic + onsite disorder", cf.SparseMatrixCRS(n, H.row_ptr, H.col_idx, v, lattice=(nl, nl, nl))
    del H, v, rows, dmask
    k = 6  # A has k entries per row -> ~2k+1 per row of A + A^H
    rows = np.repeat(np.arange(n), k)
    off = rng.integers(-4096, 4097, n * k)
    cols = np.clip(rows + off, 0, n - 1)
    vals = rng.normal(size=n * k) + 1j * rng.normal(size=n * k)
    yield "random banded Hermitian (|i-j| <= 4096)", hermitian_from_pairs(n, rows, cols, vals, rng.normal(size=n))
    cols = rng.integers(0, n, n * k)
    yield "random scattered Hermitian", hermitian_from_pairs(n, rows, cols, vals, rng.normal(size=n))


def run(name, H, nb=32, reps=20):
    t0 = time.perf_counter()
    dm = H.device_matrix(0)
    build = time.perf_counter() - t0
    st = C.c_int()
    lib.cf_matrix_staged(dm.handle, C.byref(st))
    s = cf.spectral_map(*cf.gershgorin_bounds(H), 0.01)
    X, U, W = (cf.BlockVector(H.n, nb, nb, device="cuda:0") for _ in range(3))
    for k, v in enumerate((X, U, W)):
        cf.blockvec.random_fill_device(v, 5 + k)
    mom = cf.MomentSeries(reps + 10, nb, device="cuda:0")
    Uv, Wv, Xv = cf.SubblockView(U, 0), cf.SubblockView(W, 0), cf.SubblockView(X, 0)
    for p in range(3, 6):
        cf.swap_blocks(Wv, Uv)
        cf.chebfd_op(H, s, Uv, Wv, Xv, p, 0.01, mom)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for p in range(6, 6 + reps):
        cf.swap_blocks(Wv, Uv)
        cf.chebfd_op(H, s, Uv, Wv, Xv, p, 0.01, mom)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    nnzr = H.nnz() / H.n
    alg = H.n * (nnzr * 20 + 80 * nb)
    ok = bool(torch.isfinite(torch.view_as_real(X.panel(0))).all())
    info = dm.info()
    return {"matrix": name, "n": H.n, "nnz_per_row": round(nnzr, 3), "kernel": "chunk-staged" if st.value else
            "register-gather", "device_matrix_bytes": info["device_bytes"], "ms_per_step": round(ms, 4),
            "algorithmic_gbs": round(alg / ms / 1e6, 1), "frac_of_peak": round(alg / ms / 1e6 / peak(), 4),
            "build_upload_s": round(build, 1), "finite": ok}


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=128)
    a = ap.parse_args()
    rng = np.random.default_rng(1)
    for name, H in matrices(a.n, rng):
        print(json.dumps(run(name, H)), flush=True)
        del H
        torch.cuda.empty_cache()
