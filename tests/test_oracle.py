"""The CPU checker itself: pin oracle/chebfd_oracle.c to the reference.

Against the committed fixtures (made by the reference, tests/golden/gen_golden.py)
always, and against oracle/_ref (the reference compiled unchanged) when present.
Bit-exact for every integer and floating-point output (same operation order,
no contraction), which is what licenses the oracle as the GPU parity checker.
"""
import numpy as np
import pytest

import oracle as orc
from golden_io import bits, load, topi_cases

needs_ref = pytest.mark.skipif(orc.REF is None, reason="oracle/_ref not built (no /root/reference here)")


@pytest.mark.parametrize("case", range(len(topi_cases())))
def test_topi_generator_matches_golden(case):
    c = topi_cases()[case]
    H = orc.topi(*c["spec"][:5], open_=c["spec"][5])
    assert np.array_equal(H.row_ptr, c["row_ptr"])
    assert np.array_equal(H.col_idx, c["col_idx"])
    assert np.array_equal(bits(H.values), bits(c["values"]))
    lo, hi = orc.gershgorin(H)
    assert np.array_equal(bits(np.array([lo, hi])), bits(c["bounds"]))


def test_periodic_topi_has_13_nnz_per_row():  # test_matrix.cpp:29-34
    H = orc.topi(4, 4, 4)
    assert H.n == 256
    assert np.all(np.diff(H.row_ptr.astype(np.int64)) == 13)


def test_coefficients_match_golden():
    d = load("coeffs")
    k = 0
    while f"case{k}_in" in d:
        wlo, whi, lo, hi, margin, np_, damp = d[f"case{k}_in"]
        a, b = orc.spectral_map(lo, hi, margin)
        assert np.array_equal(bits(np.array([a, b])), bits(d[f"case{k}_map"]))
        c, g = orc.coefficients(wlo, whi, a, b, int(np_), int(damp))
        assert np.array_equal(bits(c), bits(d[f"case{k}_c"]))
        assert np.array_equal(bits(g), bits(d[f"case{k}_g"]))
        k += 1
    assert k >= 5


def test_rng_matches_golden():
    d = load("rng")
    for k in range(4):
        n, ns, nb, seed, off = (int(x) for x in d[f"case{k}_in"])
        x = orc.blockvec_random(n, ns, nb, seed, off)
        assert np.array_equal(bits(x), bits(d[f"case{k}_x"].view(np.complex128)))


def test_partition_matches_golden():
    d = load("partition")
    k = 0
    while f"case{k}_in" in d:
        nx, ny, nz, w = (int(x) for x in d[f"case{k}_in"])
        H = orc.topi(nx, ny, nz)
        ranges, halo = orc.partition(H, w)
        assert np.array_equal(ranges, d[f"case{k}_ranges"])
        assert np.array_equal(halo, d[f"case{k}_halo"])
        k += 1


def test_apply_filter_matches_golden_bitwise():
    d = load("filter_small")
    H = orc.topi(4, 4, 4)
    a, b = d["topi4_map"]
    c, g = orc.coefficients(-0.5, 0.5, a, b, 50)
    X0 = orc.blockvec_random(256, 8, 2, 77)
    X, eta, mu = orc.apply_filter(H, X0, 50, c, g, a, b)
    assert np.array_equal(bits(X), bits(d["topi4_X"]))
    assert np.array_equal(bits(eta), bits(d["topi4_eta"]))
    assert np.array_equal(bits(mu), bits(d["topi4_mu"]))


@pytest.mark.parametrize("nb", [1, 2, 4, 8, 16])
def test_fused_steps_match_golden_bitwise(nb):
    d = load("filter_small")
    pre = f"step_nb{nb}_"
    H = orc.Crs(50, d[pre + "H_row_ptr"], d[pre + "H_col_idx"], d[pre + "H_values"])
    U, W, X = d[pre + "U0"], d[pre + "W0"], d[pre + "X0"]
    eta = np.zeros(nb, np.complex128)
    mu = np.zeros(nb, np.complex128)
    for p in range(3, 9):
        U, W = W, U
        W, X, e, m = orc.chebfd_op(H, 1.0, 0.0, U, W, X, 0.3 / p)
        eta, mu = eta + e, mu + m  # exact: each step's slot accumulates once from zero in the fixture
    assert np.array_equal(bits(W), bits(d[pre + "W"]))
    assert np.array_equal(bits(X), bits(d[pre + "X"]))


def test_cfg1_moments_match_golden():
    """BASELINE configs[0] through the oracle (single-threaded, ~30-60 s)."""
    d = load("cfg1")
    H = orc.topi(64, 64, 40)
    lo, hi = orc.gershgorin(H)
    assert np.array_equal(bits(np.array([lo, hi])), bits(d["bounds"]))
    span = hi - lo
    a, b = orc.spectral_map(lo, hi, 0.01)
    c, g = orc.coefficients(lo + 0.45 * span, lo + 0.55 * span, a, b, 100)
    X0 = orc.blockvec_random(H.n, 8, 8, 42)
    X, eta, mu = orc.apply_filter(H, X0, 100, c, g, a, b)
    assert np.array_equal(bits(X[0][d["X_rows"]]), bits(d["X_sample"]))
    assert np.array_equal(bits(eta), bits(d["eta"]))
    assert np.array_equal(bits(mu), bits(d["mu"]))


@needs_ref
@pytest.mark.parametrize("seed,n,nb", [(3, 37, 3), (11, 64, 4), (5, 20, 1)])
def test_oracle_kernels_match_reference_bitwise(seed, n, nb):
    R = orc.RefMatrix.random_hermitian(n, seed, 0.15)
    H = R.crs()
    X = orc.blockvec_random(n, nb, nb, seed)[0]
    Z = orc.blockvec_random(n, nb, nb, seed + 1)[0]
    Y_ref = np.zeros_like(X)
    assert orc.REF.ref_spmmv_shifted(R.h, 0.7, -0.2, n, nb, orc._p(X), orc._p(Y_ref)) == 0
    assert np.array_equal(bits(orc.spmmv(H, 0.7, -0.2, X)), bits(Y_ref))
    Y2 = np.zeros_like(X)
    assert orc.REF.ref_spmmv_two_minus(R.h, 0.7, -0.2, n, nb, orc._p(X), orc._p(Y2), orc._p(Z)) == 0
    assert np.array_equal(bits(orc.two_minus(H, 0.7, -0.2, X, Z)), bits(Y2))
    for unfused in (0, 1):
        U, W, Xs = X.copy(), Z.copy(), orc.blockvec_random(n, nb, nb, seed + 2)[0]
        e = np.zeros(nb, np.complex128)
        m = np.zeros(nb, np.complex128)
        W_o, X_o, e_o, m_o = orc.chebfd_op(H, 0.9, 0.05, U, W, Xs, 0.125, unfused=bool(unfused))
        assert orc.REF.ref_chebfd_op(R.h, 0.9, 0.05, n, nb, orc._p(U), orc._p(W), orc._p(Xs), 0.125, orc._p(e),
                                     orc._p(m), unfused) == 0
        assert np.array_equal(bits(W_o), bits(W)) and np.array_equal(bits(X_o), bits(Xs))
        assert np.array_equal(bits(e_o), bits(e)) and np.array_equal(bits(m_o), bits(m))


@needs_ref
def test_oracle_topi_matches_reference_open_and_odd_extents():
    for spec in [(3, 1, 2, 0.5, -0.75, True), (1, 2, 1, 1.5, 2.0, False), (6, 5, 2, 1.0, 1.0, True)]:
        H = orc.topi(*spec[:5], open_=spec[5])
        R = orc.RefMatrix.topi(*spec[:5], spec[5]).crs()
        assert np.array_equal(H.row_ptr, R.row_ptr) and np.array_equal(H.col_idx, R.col_idx)
        assert np.array_equal(bits(H.values), bits(R.values))
