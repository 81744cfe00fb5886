"""Generate the golden fixtures under tests/golden/ from the REFERENCE itself.

Runs the reference headers compiled unchanged (oracle/_ref/libchebref.so, built
by `make -C oracle ref` from /root/reference/proj/include) and stores their
outputs as small .npz files.  These fixtures travel to the GPU box, where
/root/reference does not exist.  Re-run with:  python tests/golden/gen_golden.py
"""
from __future__ import annotations

import ctypes as C
import os
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import oracle as orc  # noqa: E402

REF = orc.REF
OUT = Path(__file__).resolve().parent
_p = orc._p

TOPI_CASES = [  # (nx, ny, nz, mass, hop, open)
    (4, 4, 4, 1.0, 1.0, False),
    (2, 2, 2, 1.0, 1.0, False),
    (1, 1, 1, 1.0, 1.0, False),
    (2, 3, 1, 0.7, -1.3, False),
    (2, 3, 1, 0.7, -1.3, True),
    (3, 2, 2, 0.83, 1.1, True),
    (5, 3, 4, 0.9, 1.2, False),
    (3, 3, 3, 1.0, 1.0, False),
]


def ref_chk(st):
    if st != 0:
        raise RuntimeError(REF.ref_last_error().decode())


def gen_topi():
    d = {}
    for k, (nx, ny, nz, m, t, op) in enumerate(TOPI_CASES):
        H = orc.RefMatrix.topi(nx, ny, nz, m, t, op).crs()
        d[f"case{k}_spec"] = np.array([nx, ny, nz, m, t, float(op)])
        d[f"case{k}_row_ptr"] = H.row_ptr
        d[f"case{k}_col_idx"] = H.col_idx
        d[f"case{k}_values"] = H.values.view(np.float64)  # keeps signed zeros
        lo, hi = C.c_double(), C.c_double()
        RH = orc.RefMatrix.from_crs(H)
        ref_chk(REF.ref_gershgorin(RH.h, C.byref(lo), C.byref(hi)))
        d[f"case{k}_bounds"] = np.array([lo.value, hi.value])
    np.savez_compressed(OUT / "topi.npz", **d)


def gen_coeffs():
    cases = [(-0.7, 0.7, -7.0, 7.0, 0.01, 100, 0), (-0.7, 0.7, -7.0, 7.0, 0.01, 500, 0),
             (-0.4, 0.4, -1.0, 1.0, 0.0, 20, 1), (-0.2, 0.3, -1.0, 1.0, 0.0, 80, 0),
             (0.3, 0.7, -5.3, 5.3, 0.01, 300, 0), (-0.5, 0.5, -8.0, 8.0, 0.0, 50, 0)]
    d = {}
    for k, (wlo, whi, lo, hi, margin, np_, damp) in enumerate(cases):
        a, b = C.c_double(), C.c_double()
        ref_chk(REF.ref_spectral_map(lo, hi, margin, C.byref(a), C.byref(b)))
        c = np.empty(np_ + 1)
        g = np.empty(np_ + 1)
        ref_chk(REF.ref_filter_coefficients(wlo, whi, a.value, b.value, np_, damp, _p(c), _p(g)))
        d[f"case{k}_in"] = np.array([wlo, whi, lo, hi, margin, np_, damp])
        d[f"case{k}_map"] = np.array([a.value, b.value])
        d[f"case{k}_c"] = c
        d[f"case{k}_g"] = g
    np.savez_compressed(OUT / "coeffs.npz", **d)


def gen_rng():
    d = {}
    for k, (n, ns, nb, seed, off) in enumerate([(16, 8, 4, 123, 0), (8, 8, 4, 123, 8), (10, 6, 3, 7, 0),
                                               (33, 4, 1, 42, 1000)]):
        out = np.empty((ns // nb, n, nb), np.complex128)
        ref_chk(REF.ref_blockvec_random(n, ns, nb, seed, off, _p(out)))
        d[f"case{k}_in"] = np.array([n, ns, nb, seed, off], np.uint64)
        d[f"case{k}_x"] = out.view(np.float64)
    np.savez_compressed(OUT / "rng.npz", **d)


def gen_partition():
    d = {}
    cases = [(4, 4, 4, w) for w in (1, 2, 3, 4, 8)] + [(3, 3, 3, w) for w in (2, 3, 4)] + [(2, 3, 5, 3)]
    for k, (nx, ny, nz, w) in enumerate(cases):
        R = orc.RefMatrix.topi(nx, ny, nz)
        ln = C.c_size_t()
        ref_chk(REF.ref_partition_rows(R.h, w, None, None, C.byref(ln)))
        ranges = np.empty(2 * w, np.uint64)
        halo = np.empty(max(ln.value, 1), np.uint64)
        ref_chk(REF.ref_partition_rows(R.h, w, _p(ranges), _p(halo), C.byref(ln)))
        d[f"case{k}_in"] = np.array([nx, ny, nz, w], np.uint64)
        d[f"case{k}_ranges"] = ranges
        d[f"case{k}_halo"] = halo[:ln.value]
        for s in range(w):
            a = [C.c_size_t() for _ in range(3)]
            sl, rl = C.c_size_t(), C.c_size_t()
            ref_chk(REF.ref_shard(R.h, w, s, *[C.byref(x) for x in a], None, None, None, None, None, C.byref(sl),
                                  None, C.byref(rl)))
            ln_, hn, nnz = (x.value for x in a)
            rp = np.empty(ln_ + 1, np.uint64)
            ci = np.empty(nnz, np.int32)
            v = np.empty(nnz, np.complex128)
            hg = np.empty(max(hn, 1), np.uint64)
            sf = np.empty(max(sl.value, 1), np.uint64)
            rf = np.empty(max(rl.value, 1), np.uint64)
            ref_chk(REF.ref_shard(R.h, w, s, *[C.byref(x) for x in a], _p(rp), _p(ci), _p(v), _p(hg), _p(sf),
                                  C.byref(sl), _p(rf), C.byref(rl)))
            d[f"case{k}_shard{s}_sizes"] = np.array([ln_, hn, nnz], np.uint64)
            d[f"case{k}_shard{s}_row_ptr"] = rp
            d[f"case{k}_shard{s}_col_idx"] = ci
            d[f"case{k}_shard{s}_halo_global"] = hg[:hn]
            d[f"case{k}_shard{s}_send"] = sf[:sl.value]
            d[f"case{k}_shard{s}_recv"] = rf[:rl.value]
    np.savez_compressed(OUT / "partition.npz", **d)


def ref_apply(R, Xp, np_, c, g, a, b):
    Xp = np.array(Xp, np.complex128, order="C")
    npan, n, nb = Xp.shape
    ns = npan * nb
    eta = np.zeros((np_ - 2) * ns, np.complex128)
    mu = np.zeros((np_ - 2) * ns, np.complex128)
    ref_chk(REF.ref_apply_filter(R.h, ns, nb, _p(Xp), np_, _p(c), _p(g), a, b, _p(eta), _p(mu)))
    return Xp, eta.reshape(np_ - 2, ns), mu.reshape(np_ - 2, ns)


def coeffs_for(wlo, whi, lo, hi, margin, np_):
    a, b = C.c_double(), C.c_double()
    ref_chk(REF.ref_spectral_map(lo, hi, margin, C.byref(a), C.byref(b)))
    c = np.empty(np_ + 1)
    g = np.empty(np_ + 1)
    ref_chk(REF.ref_filter_coefficients(wlo, whi, a.value, b.value, np_, 0, _p(c), _p(g)))
    return a.value, b.value, c, g


def gen_filter_small():
    d = {}
    # acceptance criterion 6 shape (acceptance.cpp:161-191): topi 4^3, window (-0.5,0.5), map(-8,8), np 50
    R = orc.RefMatrix.topi(4, 4, 4)
    a, b, c, g = coeffs_for(-0.5, 0.5, -8.0, 8.0, 0.0, 50)
    X0 = np.empty((4, 256, 2), np.complex128)
    ref_chk(REF.ref_blockvec_random(256, 8, 2, 77, 0, _p(X0)))
    X, eta, mu = ref_apply(R, X0, 50, c, g, a, b)
    d.update(topi4_X=X, topi4_eta=eta, topi4_mu=mu, topi4_map=np.array([a, b]))
    # distributed reference run, both modes, 2 and 4 workers
    for w in (2, 4):
        for mode in (0, 1):
            Xd = X0.copy()
            eta_d = np.zeros(48 * 8, np.complex128)
            mu_d = np.zeros(48 * 8, np.complex128)
            ref_chk(REF.ref_filter_distributed(R.h, w, mode, 8, 2, _p(Xd), 50, _p(c), _p(g), a, b, _p(eta_d),
                                               _p(mu_d)))
            d[f"topi4_dist_w{w}_m{mode}_X"] = Xd
            d[f"topi4_dist_w{w}_m{mode}_eta"] = eta_d.reshape(48, 8)
            d[f"topi4_dist_w{w}_m{mode}_mu"] = mu_d.reshape(48, 8)
    # single fused steps on a dense random Hermitian (test_kernels.cpp:126-154 shape)
    for nb in (1, 2, 4, 8, 16):
        Rh = orc.RefMatrix.random_hermitian(50, 40 + nb, 0.1)
        n = 50
        U = np.empty((1, n, nb), np.complex128)
        W = np.empty((1, n, nb), np.complex128)
        Xs = np.empty((1, n, nb), np.complex128)
        ref_chk(REF.ref_blockvec_random(n, nb, nb, 1, 0, _p(U)))
        ref_chk(REF.ref_blockvec_random(n, nb, nb, 2, 0, _p(W)))
        ref_chk(REF.ref_blockvec_random(n, nb, nb, 3, 0, _p(Xs)))
        Hc = Rh.crs()
        d[f"step_nb{nb}_H_row_ptr"] = Hc.row_ptr
        d[f"step_nb{nb}_H_col_idx"] = Hc.col_idx
        d[f"step_nb{nb}_H_values"] = Hc.values
        d[f"step_nb{nb}_U0"], d[f"step_nb{nb}_W0"], d[f"step_nb{nb}_X0"] = U[0], W[0], Xs[0]
        e = np.zeros(nb, np.complex128)
        m = np.zeros(nb, np.complex128)
        Uc, Wc, Xc = U[0].copy(), W[0].copy(), Xs[0].copy()
        for p in range(3, 9):  # swap then step, gc = 0.3/p
            Uc, Wc = Wc, Uc
            ref_chk(REF.ref_chebfd_op(Rh.h, 1.0, 0.0, n, nb, _p(Uc), _p(Wc), _p(Xc), 0.3 / p, _p(e), _p(m), 0))
        d[f"step_nb{nb}_W"], d[f"step_nb{nb}_X"], d[f"step_nb{nb}_eta"], d[f"step_nb{nb}_mu"] = Wc, Xc, e, m
    np.savez_compressed(OUT / "filter_small.npz", **d)


def gen_cfg1():
    """BASELINE configs[0]: topi 4x64x64x40, n_s=n_b=8, n_p=100, bench-kernel inputs
    (tools/chebfilter.cpp:277-294): Gershgorin bounds, margin 0.01, window
    lo+0.45 span .. lo+0.55 span, Jackson, X0 = InitSeededRandom{42}."""
    os.environ.setdefault("CHEBFILTER_THREADS", str(os.cpu_count() or 8))
    R = orc.RefMatrix.topi(64, 64, 40)
    lo, hi = C.c_double(), C.c_double()
    ref_chk(REF.ref_gershgorin(R.h, C.byref(lo), C.byref(hi)))
    span = hi.value - lo.value
    a, b, c, g = coeffs_for(lo.value + 0.45 * span, lo.value + 0.55 * span, lo.value, hi.value, 0.01, 100)
    n = 4 * 64 * 64 * 40
    X0 = np.empty((1, n, 8), np.complex128)
    ref_chk(REF.ref_blockvec_random(n, 8, 8, 42, 0, _p(X0)))
    t0 = time.time()
    X, eta, mu = ref_apply(R, X0, 100, c, g, a, b)
    dt = time.time() - t0
    rows = np.arange(0, n, 4099)
    np.savez_compressed(OUT / "cfg1.npz", X_rows=rows, X_sample=X[0][rows], eta=eta, mu=mu,
                        col_norm2=(np.abs(X[0]) ** 2).sum(axis=0), max_abs=np.abs(X[0]).max(),
                        map=np.array([a, b]), bounds=np.array([lo.value, hi.value]), ref_seconds=dt)
    print(f"cfg1 reference apply_filter: {dt:.2f} s")


def gen_cfg2():
    """BASELINE configs[1] at full degree: topi 4x128^3 (n = 8,388,608), n_s = n_b = 32,
    n_p = 500, bench-kernel inputs (tools/chebfilter.cpp:277-294).  The reference's
    own apply_filter (filter.hpp:76-93) on all host cores (~35 min on 8 cores, ~35 GB
    RSS).  Stores the full eta/mu series, column norms and 256 sampled rows of X."""
    os.environ.setdefault("CHEBFILTER_THREADS", str(min(os.cpu_count() or 8, 64)))
    np_ = 500
    R = orc.RefMatrix.topi(128, 128, 128)
    lo, hi = C.c_double(), C.c_double()
    ref_chk(REF.ref_gershgorin(R.h, C.byref(lo), C.byref(hi)))
    span = hi.value - lo.value
    a, b, c, g = coeffs_for(lo.value + 0.45 * span, lo.value + 0.55 * span, lo.value, hi.value, 0.01, np_)
    n = 4 * 128 ** 3
    X0 = np.empty((1, n, 32), np.complex128)
    ref_chk(REF.ref_blockvec_random(n, 32, 32, 42, 0, _p(X0)))
    t0 = time.time()
    X, eta, mu = ref_apply(R, X0, np_, c, g, a, b)
    del X0
    dt = time.time() - t0
    rows = np.arange(0, n, 32771)
    np.savez_compressed(OUT / "cfg2.npz", X_rows=rows, X_sample=X[0][rows], eta=eta, mu=mu,
                        col_norm2=(np.abs(X[0]) ** 2).sum(axis=0), max_abs=np.abs(X[0]).max(),
                        map=np.array([a, b]), bounds=np.array([lo.value, hi.value]), ref_seconds=dt,
                        threads=int(os.environ["CHEBFILTER_THREADS"]))
    print(f"cfg2 reference apply_filter (n_p={np_}): {dt:.1f} s")


def gen_eigs():
    d = {}
    # acceptance.cpp:77-96 topi 4^3 window (-0.5, 0.5) vs dense oracle
    R = orc.RefMatrix.topi(4, 4, 4)
    ev = np.empty(256)
    ref_chk(REF.ref_dense_eigenvalues(R.h, _p(ev)))
    d["topi4_dense_eigs"] = ev
    R2 = orc.RefMatrix.topi(3, 2, 2, 0.83, 1.1, True)
    ev2 = np.empty(48)
    ref_chk(REF.ref_dense_eigenvalues(R2.h, _p(ev2)))
    d["open322_dense_eigs"] = ev2
    np.savez_compressed(OUT / "eigs.npz", **d)


if __name__ == "__main__":
    if REF is None:
        sys.exit("oracle/_ref/libchebref.so missing: run `make -C oracle ref` (needs /root/reference)")
    if sys.argv[1:] == ["cfg2"]:
        gen_cfg2()
        sys.exit(0)
    gen_topi()
    gen_coeffs()
    gen_rng()
    gen_partition()
    gen_filter_small()
    gen_eigs()
    gen_cfg1()
    print("golden fixtures written to", OUT)
