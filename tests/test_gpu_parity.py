"""GPU parity: libchebfd_b200's sm_100a kernels (through the C ABI) against the
CPU checker (oracle/, pinned to the reference) and the reference's fixtures.

Tolerances (north_star: filtered vectors <= 1e-10 max-rel after the full
degree; the reference's own kernel tests use 1e-13 per op, test_kernels.cpp):
  single operators            max|gpu-ref| / max|ref| <= 1e-13
  moments of a step sequence  <= 1e-12 (relative to max |moment|)
  full filter (X)             <= 1e-10, moments <= 1e-12
The device result is not bit-identical to the CPU reference: it contracts
complex products into FMAs and factors alpha out of the row sum, which changes
rounding at the 1e-16 level (SURVEY.md App. A.3 measures 8.7e-15 after n_p=500).
"""
import numpy as np
import pytest
import torch

import oracle as orc
import paper_1803_02156_b200 as cf
from golden_io import load

pytestmark = pytest.mark.gpu
DEV = "cuda:0"


def rel(a, b):
    a = np.asarray(a)
    b = np.asarray(b)
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-300))


def dev_panel(a):
    return torch.from_numpy(np.ascontiguousarray(a, np.complex128)).to(DEV)


def bv_from(a, nb=None):
    a = np.asarray(a, np.complex128)
    return cf.BlockVector.from_numpy(a, nb or a.shape[1], device=DEV)


def random_sparse(n, density, seed, ncols=None, herm=False):
    rng = np.random.default_rng(seed)
    ncols = ncols or n
    a = np.zeros((n, ncols), np.complex128)
    mask = rng.random((n, ncols)) < density
    a[mask] = rng.normal(size=mask.sum()) + 1j * rng.normal(size=mask.sum())
    for i in range(n):  # at least one entry per row, diagonal present
        a[i, i % ncols] += 1.0 + 0.5j
    if herm and ncols == n:
        a = 0.5 * (a + a.conj().T)
    return cf.from_dense(a), a


def as_oracle(H):
    return orc.Crs(H.n, H.row_ptr, H.col_idx, H.values, H.ncols)


def shuffled_rows(H, seed=0):
    """Same matrix with each row's entries in a random column order (shard-local
    matrices keep the reference's remapped, unsorted order, dist.hpp:76-86)."""
    rng = np.random.default_rng(seed)
    rp = H.row_ptr.astype(np.int64)
    ci, v = H.col_idx.copy(), H.values.copy()
    for i in range(H.n):
        p = rng.permutation(rp[i + 1] - rp[i]) + rp[i]
        ci[rp[i]:rp[i + 1]], v[rp[i]:rp[i + 1]] = H.col_idx[p], H.values[p]
    return cf.SparseMatrixCRS(H.n, H.row_ptr, ci, v, ncols=H.ncols)


MATS = {
    "topi444": lambda: cf.topi_generate(cf.LatticeSpec(4, 4, 4)),
    "topi_open_523": lambda: cf.topi_generate(cf.LatticeSpec(5, 2, 3, 0.83, 1.1, cf.Boundary.open)),
    "topi_111": lambda: cf.topi_generate(cf.LatticeSpec(1, 1, 1)),
    "sparse97": lambda: random_sparse(97, 0.06, 1)[0],
    "dense30": lambda: random_sparse(30, 1.0, 2, herm=True)[0],
    "diag7": lambda: cf.diagonal_matrix([0.3, -0.8, 0.5, 0.0, 0.9, -0.4, 0.1]),
    "halo": lambda: random_sparse(41, 0.08, 3, ncols=57)[0],
    "tiny1": lambda: cf.diagonal_matrix([2.5]),
    "shuffled": lambda: shuffled_rows(random_sparse(59, 0.1, 4, ncols=66)[0]),
    "topi_shuffled": lambda: shuffled_rows(cf.topi_generate(cf.LatticeSpec(3, 4, 2)), 1),
}


@pytest.mark.parametrize("mat", list(MATS))
@pytest.mark.parametrize("nb", [1, 2, 3, 4, 8, 13, 16, 32, 33, 64])
def test_spmmv_family_vs_oracle(mat, nb):
    H = MATS[mat]()
    O = as_oracle(H)
    X = orc.blockvec_random(H.ncols, nb, nb, 5 + nb)[0]
    Z = orc.blockvec_random(H.n, nb, nb, 9 + nb)[0]
    s = cf.ShiftScale(0.7, -0.2)
    Xd = bv_from(X)
    Yd = cf.BlockVector(H.n, nb, nb, device=DEV)
    cf.spmmv_shifted(H, s, cf.SubblockView(Xd, 0), cf.SubblockView(Yd, 0))
    assert rel(Yd.to_numpy(), orc.spmmv(O, 0.7, -0.2, X)) <= 1e-13
    Zd = bv_from(Z)
    cf.spmmv_shifted_two_minus(H, s, cf.SubblockView(Xd, 0), cf.SubblockView(Yd, 0), cf.SubblockView(Zd, 0))
    assert rel(Yd.to_numpy(), orc.two_minus(O, 0.7, -0.2, X, Z)) <= 1e-13
    # in place: Z == Y (kernels.hpp:103-105)
    cf.spmmv_shifted_two_minus(H, s, cf.SubblockView(Xd, 0), cf.SubblockView(Zd, 0), cf.SubblockView(Zd, 0))
    assert rel(Zd.to_numpy(), orc.two_minus(O, 0.7, -0.2, X, Z)) <= 1e-13


@pytest.mark.parametrize("mat", ["topi444", "topi_open_523", "sparse97", "dense30"])
@pytest.mark.parametrize("nb", [1, 4, 8, 32, 40, 64])
def test_cheb_init_and_steps_vs_oracle(mat, nb):
    H = MATS[mat]()
    O = as_oracle(H)
    n = H.n
    s = cf.ShiftScale(0.11, 0.02)
    X0 = orc.blockvec_random(n, nb, nb, 77)[0]
    Xo, Uo, Wo = orc.cheb_init(O, s.alpha, s.beta, X0, 0.4, -0.3, 0.25)
    Xd, Ud, Wd = bv_from(X0), cf.BlockVector(n, nb, nb, device=DEV), cf.BlockVector(n, nb, nb, device=DEV)
    cf.cheb_init(H, s, cf.SubblockView(Xd, 0), cf.SubblockView(Ud, 0), cf.SubblockView(Wd, 0), 0.4, -0.3, 0.25)
    assert rel(Ud.to_numpy(), Uo) <= 1e-13
    assert rel(Wd.to_numpy(), Wo) <= 1e-13
    assert rel(Xd.to_numpy(), Xo) <= 1e-13
    np_ = 12
    mom = cf.MomentSeries(np_, nb, device=DEV)
    eta_o = np.zeros((np_ - 2, nb), np.complex128)
    mu_o = np.zeros((np_ - 2, nb), np.complex128)
    for p in range(3, np_ + 1):
        cf.swap_blocks(cf.SubblockView(Wd, 0), cf.SubblockView(Ud, 0))
        Uo, Wo = Wo, Uo
        cf.chebfd_op(H, s, cf.SubblockView(Ud, 0), cf.SubblockView(Wd, 0), cf.SubblockView(Xd, 0), p, 0.3 / p, mom)
        Wo, Xo, e, m = orc.chebfd_op(O, s.alpha, s.beta, Uo, Wo, Xo, 0.3 / p)
        eta_o[p - 3], mu_o[p - 3] = e, m
    assert rel(Wd.to_numpy(), Wo) <= 1e-12
    assert rel(Xd.to_numpy(), Xo) <= 1e-12
    assert rel(mom.eta.cpu().numpy().reshape(np_ - 2, nb), eta_o) <= 1e-12
    mu_g = mom.mu.cpu().numpy().reshape(np_ - 2, nb)
    assert rel(mu_g, mu_o) <= 1e-12
    assert np.all(mu_g.real >= 0) and np.all(mu_g.imag == 0)  # test_kernels.cpp:205-223


@pytest.mark.parametrize("nb", [1, 2, 4, 8, 16])
def test_fused_steps_vs_reference_fixture(nb):
    """test_kernels.cpp:126-154 inputs, reference outputs from tests/golden."""
    d = load("filter_small")
    pre = f"step_nb{nb}_"
    H = cf.SparseMatrixCRS(50, d[pre + "H_row_ptr"], d[pre + "H_col_idx"], d[pre + "H_values"])
    Ud, Wd, Xd = bv_from(d[pre + "U0"]), bv_from(d[pre + "W0"]), bv_from(d[pre + "X0"])
    mom = cf.MomentSeries(8, nb, device=DEV)
    s = cf.ShiftScale(1.0, 0.0)
    for p in range(3, 9):
        cf.swap_blocks(cf.SubblockView(Wd, 0), cf.SubblockView(Ud, 0))
        cf.chebfd_op(H, s, cf.SubblockView(Ud, 0), cf.SubblockView(Wd, 0), cf.SubblockView(Xd, 0), p, 0.3 / p, mom)
    assert rel(Wd.to_numpy(), d[pre + "W"]) <= 1e-13
    assert rel(Xd.to_numpy(), d[pre + "X"]) <= 1e-13


def test_moments_bit_identical_across_reruns():  # test_kernels.cpp:225-256
    H, _ = random_sparse(64, 0.2, 14, herm=True)
    H = cf.topi_generate(cf.LatticeSpec(6, 5, 4))

    def run():
        X = cf.BlockVector(H.n, 8, 8, cf.InitSeededRandom(4), device=DEV)
        U, W = cf.BlockVector(H.n, 8, 8, device=DEV), cf.BlockVector(H.n, 8, 8, device=DEV)
        cf.cheb_init(H, cf.ShiftScale(0.1, 0.0), cf.SubblockView(X, 0), cf.SubblockView(U, 0),
                     cf.SubblockView(W, 0), 0.5, 0.2, 0.1)
        mom = cf.MomentSeries(9, 8, device=DEV)
        for p in range(3, 10):
            cf.swap_blocks(cf.SubblockView(W, 0), cf.SubblockView(U, 0))
            cf.chebfd_op(H, cf.ShiftScale(0.1, 0.0), cf.SubblockView(U, 0), cf.SubblockView(W, 0),
                         cf.SubblockView(X, 0), p, 0.05, mom)
        return mom.eta.cpu().numpy(), mom.mu.cpu().numpy(), X.to_numpy()

    a, b = run(), run()
    for x, y in zip(a, b):
        assert np.array_equal(x.view(np.uint64), y.view(np.uint64))


def test_apply_filter_matches_reference_topi4():
    """acceptance.cpp:161-191 serial case: reference X/moments from tests/golden."""
    d = load("filter_small")
    H = cf.topi_generate(cf.LatticeSpec(4, 4, 4))
    fc = cf.filter_coefficients(-0.5, 0.5, cf.spectral_map(-8.0, 8.0), 50)
    X = cf.BlockVector(H.n, 8, 2, cf.InitSeededRandom(77), device=DEV)
    mom = cf.apply_filter(H, X, fc)
    assert rel(X.panels_numpy(), d["topi4_X"]) <= 1e-10
    assert rel(mom.eta.cpu().numpy().reshape(48, 8), d["topi4_eta"]) <= 1e-12
    assert rel(mom.mu.cpu().numpy().reshape(48, 8), d["topi4_mu"]) <= 1e-12


@pytest.fixture
def x_group():
    """Set apply_filter's degrees-per-X-update (cf_tuning "x_group"), restore 3 after."""
    from paper_1803_02156_b200._lib import check, lib

    def set_group(v):
        check(lib.cf_tuning(b"x_group", v))
    yield set_group
    set_group(3)


@pytest.mark.parametrize("group", [3, 2, 1])
@pytest.mark.parametrize("np_", [3, 4, 5, 6, 11, 12, 13])
@pytest.mark.parametrize("nb", [2, 32])
def test_apply_filter_grouped_x_updates_vs_oracle(np_, nb, group, x_group):
    """apply_filter updates X once per three (or two) degrees (x += g_p c_p T_p +
    g_{p+1} c_{p+1} T_{p+1} + g_{p+2} c_{p+2} T_{p+2}); every remainder of the step
    count, both kernels' widths, against the oracle's per-step filter
    (kernels.hpp:189-193 order)."""
    x_group(group)
    H = cf.topi_generate(cf.LatticeSpec(4, 4, 5))
    fc = cf.filter_coefficients(-0.5, 0.5, cf.spectral_map(-8.0, 8.0), np_)
    X0 = cf.seeded_random_host(H.n, 2 * nb, nb, 5)
    X = cf.BlockVector(H.n, 2 * nb, nb, cf.InitSeededRandom(5), device=DEV)
    mom = cf.apply_filter(H, X, fc)
    Xo, eta_o, mu_o = orc.apply_filter(as_oracle(H), X0, np_, fc.c, fc.g, fc.map.alpha, fc.map.beta)
    assert rel(X.panels_numpy(), Xo) <= 1e-12
    if np_ >= 3:
        assert rel(mom.eta.cpu().numpy().reshape(np_ - 2, 2 * nb), eta_o) <= 1e-12
        assert rel(mom.mu.cpu().numpy().reshape(np_ - 2, 2 * nb), mu_o) <= 1e-12


def bench_inputs(nx, ny, nz, np_):
    H = cf.topi_generate(cf.LatticeSpec(nx, ny, nz))
    lo, hi = cf.gershgorin_bounds(H)
    span = hi - lo
    fc = cf.filter_coefficients(lo + 0.45 * span, lo + 0.55 * span, cf.spectral_map(lo, hi, 0.01), np_)
    return H, fc


def test_apply_filter_cfg1_matches_reference():
    """BASELINE configs[0] (4x64x64x40, n_b=8, n_p=100, bench-kernel inputs)."""
    d = load("cfg1")
    H, fc = bench_inputs(64, 64, 40, 100)
    X = cf.BlockVector(H.n, 8, 8, cf.InitSeededRandom(42), device=DEV)
    mom = cf.apply_filter(H, X, fc)
    Xh = X.to_numpy()
    assert rel(Xh[d["X_rows"]], d["X_sample"]) <= 1e-10
    assert rel((np.abs(Xh) ** 2).sum(axis=0), d["col_norm2"]) <= 1e-10
    assert rel(mom.eta.cpu().numpy().reshape(98, 8), d["eta"]) <= 1e-12
    assert rel(mom.mu.cpu().numpy().reshape(98, 8), d["mu"]) <= 1e-12


def test_apply_filter_cfg1_full_vs_oracle_when_available():
    """Full-vector comparison against the reference run on this box (oracle/_ref
    when shipped, else the restatement; both bit-identical to the reference)."""
    H, fc = bench_inputs(64, 64, 40, 100)
    X = cf.BlockVector(H.n, 8, 8, cf.InitSeededRandom(42), device=DEV)
    mom = cf.apply_filter(H, X, fc)
    Xo, eta_o, mu_o = orc.apply_filter(as_oracle(H), orc.blockvec_random(H.n, 8, 8, 42), 100, fc.c, fc.g,
                                       fc.map.alpha, fc.map.beta)
    assert rel(X.panels_numpy(), Xo) <= 1e-10
    assert rel(mom.eta.cpu().numpy().reshape(98, 8), eta_o) <= 1e-12


@pytest.mark.parametrize("ns,nb,pinned", [(8, 8, False), (16, 8, False), (24, 8, True), (32, 8, False),
                                           (40, 8, True), (96, 32, True), (64, 8, True), (64, 16, False),
                                           (96, 12, True)])
def test_apply_filter_host_entry_equals_device_path(ns, nb, pinned):
    """Host-staged panels (two device slots, copies on their own streams) give
    the device path's bits for 1..5 panels, pageable or pinned host X; with n_b
    dividing 32 and 32 | n_s both pack 32 / n_b panels into one 32-wide panel.
    (n_b = 12, n_s = 96: the device path packs, the host entry filters panel by
    panel: equal to rounding.)"""
    H = cf.topi_generate(cf.LatticeSpec(6, 4, 5))
    fc = cf.filter_coefficients(-0.3, 0.3, cf.spectral_map(-7.0, 7.0, 0.01), 40)
    X = cf.BlockVector(H.n, ns, nb, cf.InitSeededRandom(3), device=DEV)
    host = X.panels_numpy().copy()
    if pinned:
        host = torch.from_numpy(host).pin_memory()
    mom = cf.apply_filter(H, X, fc)
    Xh, eta, mu = cf.apply_filter_host(H, host, fc)
    Xh = Xh.numpy() if pinned else Xh
    if nb < 32 and ns % 32 == 0 and 32 % nb:
        assert rel(Xh, X.panels_numpy()) <= 1e-13
        assert rel(eta, mom.eta.cpu().numpy()) <= 1e-13 and rel(mu, mom.mu.cpu().numpy()) <= 1e-13
        return
    assert np.array_equal(Xh.view(np.uint64), X.panels_numpy().view(np.uint64))
    assert np.array_equal(eta.view(np.uint64), mom.eta.cpu().numpy().view(np.uint64))
    assert np.array_equal(mu.view(np.uint64), mom.mu.cpu().numpy().view(np.uint64))


def test_apply_filter_host_panels_vs_oracle_and_reuse():
    """Three host-staged panels against the checker; a second call on the same
    matrix handle (workspace reused, smaller n_s) is still exact."""
    H = cf.topi_generate(cf.LatticeSpec(8, 6, 5))
    fc = cf.filter_coefficients(-0.5, 0.4, cf.spectral_map(-7.0, 7.0, 0.01), 30)
    for ns in (24, 8):
        host = orc.blockvec_random(H.n, ns, 8, 11)
        Xo, eta_o, mu_o = orc.apply_filter(as_oracle(H), host.copy(), 30, fc.c, fc.g, fc.map.alpha, fc.map.beta)
        Xh, eta, _ = cf.apply_filter_host(H, host, fc)
        assert rel(Xh, Xo) <= 1e-10
        assert rel(eta.reshape(28, ns), eta_o) <= 1e-12


def test_block_width_invariance():  # test_filter.cpp:116-136, acceptance criterion 5
    H, _ = random_sparse(40, 0.15, 23, herm=True)
    H.values *= 0.1
    H = cf.SparseMatrixCRS(H.n, H.row_ptr, H.col_idx, H.values)
    fc = cf.filter_coefficients(-0.1, 0.1, cf.ShiftScale(1.0, 0.0), 40)
    ref = cf.BlockVector(40, 8, 8, cf.InitSeededRandom(5), device=DEV)
    mref = cf.apply_filter(H, ref, fc)
    for nb in (1, 2, 4):
        X = cf.BlockVector(40, 8, nb, cf.InitSeededRandom(5), device=DEV)
        m = cf.apply_filter(H, X, fc)
        assert np.abs(X.to_numpy() - ref.to_numpy()).max() < 1e-12
        assert np.abs(m.eta.cpu().numpy() - mref.eta.cpu().numpy()).max() < 1e-12


def filter_poly(fc, lam):  # test_filter.cpp:19-30
    x = fc.map.alpha * lam + fc.map.beta
    tm, t = 1.0, x
    acc = fc.g[0] * fc.c[0] + fc.g[1] * fc.c[1] * t
    for p in range(2, fc.np + 1):
        tn = 2.0 * x * t - tm
        acc += fc.g[p] * fc.c[p] * tn
        tm, t = t, tn
    return acc


def test_apply_filter_is_the_scalar_polynomial_on_a_diagonal():  # test_filter.cpp:81-92
    d = [-0.9, -0.3, 0.0, 0.25, 0.6, 0.95]
    H = cf.diagonal_matrix(d)
    fc = cf.filter_coefficients(-0.2, 0.3, cf.ShiftScale(1.0, 0.0), 80)
    X = cf.BlockVector(6, 2, 2, cf.InitConstant(1.0), device=DEV)
    cf.apply_filter(H, X, fc)
    for i, lam in enumerate(d):
        assert abs(X[i, 0] - filter_poly(fc, lam)) < 1e-12
        assert abs(X[i, 1] - filter_poly(fc, lam)) < 1e-12


def test_recurrence_reproduces_T_p_pointwise():  # test_kernels.cpp:156-177
    d = [0.9, -0.4, 0.1, 0.7]
    H = cf.diagonal_matrix(d)
    s = cf.ShiftScale(1.0, 0.0)
    X, U, W = (cf.BlockVector(4, 4, 4, device=DEV) for _ in range(3))
    for j in range(4):
        X[j, j] = 1.0
    cf.cheb_init(H, s, cf.SubblockView(X, 0), cf.SubblockView(U, 0), cf.SubblockView(W, 0), 1.0, 0.0, 0.0)
    mom = cf.MomentSeries(12, 4, device=DEV)
    for p in range(3, 13):
        cf.swap_blocks(cf.SubblockView(W, 0), cf.SubblockView(U, 0))
        cf.chebfd_op(H, s, cf.SubblockView(U, 0), cf.SubblockView(W, 0), cf.SubblockView(X, 0), p, 0.0, mom)
    Wh = W.to_numpy()
    for i in range(4):
        t = np.cos(12 * np.arccos(d[i]))
        assert abs(Wh[i, i] - t) < 1e-11


def test_moments_at_fixed_point_one():  # test_kernels.cpp:179-203
    H = cf.diagonal_matrix([1.0] * 5)
    s = cf.ShiftScale(1.0, 0.0)
    X = cf.BlockVector(5, 2, 2, cf.InitSeededRandom(55), device=DEV)
    norms = (np.abs(X.to_numpy()) ** 2).sum(axis=0)
    U, W = cf.BlockVector(5, 2, 2, device=DEV), cf.BlockVector(5, 2, 2, device=DEV)
    cf.cheb_init(H, s, cf.SubblockView(X, 0), cf.SubblockView(U, 0), cf.SubblockView(W, 0), 1.0, 0.0, 0.0)
    mom = cf.MomentSeries(7, 2, device=DEV)
    for p in range(3, 8):
        cf.swap_blocks(cf.SubblockView(W, 0), cf.SubblockView(U, 0))
        cf.chebfd_op(H, s, cf.SubblockView(U, 0), cf.SubblockView(W, 0), cf.SubblockView(X, 0), p, 0.0, mom)
    for p in range(3, 8):
        for j in range(2):
            assert abs(mom.mu_at(p, j) - norms[j]) < 1e-12 * norms[j]
            assert abs(mom.eta_at(p, j) - mom.mu_at(p, j)) < 1e-12 * norms[j]


def test_operator_errors_match_reference():
    H = cf.diagonal_matrix([1.0, 1.0])
    X = cf.BlockVector(2, 2, 2, device=DEV)
    with pytest.raises(ValueError):  # kernels.hpp:66
        cf.spmmv_shifted(H, cf.ShiftScale(), cf.SubblockView(X, 0), cf.SubblockView(X, 0))
    U, W = cf.BlockVector(2, 2, 2, device=DEV), cf.BlockVector(2, 2, 2, device=DEV)
    mom = cf.MomentSeries(5, 2, device=DEV)
    for p in (2, 6):  # kernels.hpp:166
        with pytest.raises(ValueError):
            cf.chebfd_op(H, cf.ShiftScale(), cf.SubblockView(U, 0), cf.SubblockView(W, 0), cf.SubblockView(X, 0),
                         p, 0.1, mom)
    with pytest.raises(ValueError):  # kernels.hpp:168-169
        cf.chebfd_op(H, cf.ShiftScale(), cf.SubblockView(U, 0), cf.SubblockView(W, 0), cf.SubblockView(X, 0), 3,
                     0.1, mom, moment_col_offset=1)
    with pytest.raises(ValueError):
        cf.spmmv_shifted(H, cf.ShiftScale(), cf.SubblockView(X, 0),
                         cf.SubblockView(cf.BlockVector(1, 2, 2, device=DEV), 0))


@pytest.mark.parametrize("mat", ["topi444", "topi_open_523", "sparse97", "dense30", "halo"])
def test_device_image_round_trips_to_crs(mat):
    H = MATS[mat]()
    back = H.device_matrix(0).to_crs()
    assert np.array_equal(back.row_ptr, H.row_ptr)
    assert np.array_equal(back.col_idx, H.col_idx)
    assert np.array_equal(back.values.view(np.uint64), H.values.view(np.uint64))


def test_cfg2_full_size_step_properties():
    """BASELINE configs[1] size (4x128^3, n_b=32): one fused step on the GPU,
    checked on 2048 sampled rows against a direct evaluation of the reference
    row formula (kernels.hpp:180-194) and on the global moments against fp64
    torch reductions of the same vectors."""
    H = cf.topi_generate(cf.LatticeSpec(128, 128, 128))
    n, nb = H.n, 32
    g = torch.Generator(device=DEV).manual_seed(7)
    U = torch.randn(n, nb, dtype=torch.complex128, device=DEV, generator=g)
    W = torch.randn(n, nb, dtype=torch.complex128, device=DEV, generator=g)
    X = torch.randn(n, nb, dtype=torch.complex128, device=DEV, generator=g)
    W0, X0 = W.clone(), X.clone()
    Ub, Wb, Xb = (cf.BlockVector(n, nb, nb, device=DEV) for _ in range(3))
    Ub._panels[0], Wb._panels[0], Xb._panels[0] = U, W, X
    mom = cf.MomentSeries(3, nb, device=DEV)
    s = cf.ShiftScale(0.14144271570014144, 0.0)
    cf.chebfd_op(H, s, cf.SubblockView(Ub, 0), cf.SubblockView(Wb, 0), cf.SubblockView(Xb, 0), 3, 0.01, mom)
    torch.cuda.synchronize()
    rows = np.random.default_rng(0).choice(n, 2048, replace=False)
    rp = H.row_ptr.astype(np.int64)
    Uh = U  # device gather of the needed rows
    for i in rows[:256]:
        cols = torch.from_numpy(H.col_idx[rp[i]:rp[i + 1]].astype(np.int64)).to(DEV)
        vals = torch.from_numpy(H.values[rp[i]:rp[i + 1]]).to(DEV)
        acc = s.beta * Uh[i] + (s.alpha * vals[:, None] * Uh[cols]).sum(0)
        wn = 2 * acc - W0[i]
        assert torch.abs(Wb.panel(0)[i] - wn).max().item() <= 1e-13 * max(1.0, torch.abs(wn).max().item())
        xn = X0[i] + 0.01 * wn
        assert torch.abs(Xb.panel(0)[i] - xn).max().item() <= 1e-13 * max(1.0, torch.abs(xn).max().item())
    eta_ref = (Wb.panel(0).conj() * U).sum(0)
    mu_ref = (U.conj() * U).sum(0)
    assert torch.abs(mom.eta - eta_ref).max().item() <= 1e-12 * torch.abs(eta_ref).max().item()
    assert torch.abs(mom.mu - mu_ref).max().item() <= 1e-12 * torch.abs(mu_ref).max().item()


@pytest.mark.parametrize("transport", ["copy", "peer"])
@pytest.mark.parametrize("workers,mode", [(1, 0), (2, 0), (2, 1), (4, 0), (4, 1)])
def test_filter_distributed_single_process_matches_reference(workers, mode, transport):
    """acceptance.cpp:161-191 / test_dist.cpp:112-137 through the drop-in
    filter_distributed (shards of one process on cuda:0): halo by device copies
    (LocalTransport) or fused into the kernels' stores (PeerTransport, cf_mirror)."""
    from paper_1803_02156_b200 import dist as cfd
    d = load("filter_small")
    H = cf.topi_generate(cf.LatticeSpec(4, 4, 4))
    fc = cf.filter_coefficients(-0.5, 0.5, cf.spectral_map(-8.0, 8.0), 50)
    X = cf.BlockVector(H.n, 8, 2, cf.InitSeededRandom(77), device=DEV)
    shards = cfd.shard_and_distribute(H, X, cfd.partition_rows(H, workers))
    tr = cfd.LocalTransport(shards) if transport == "copy" else cfd.PeerTransport(shards)
    res = cfd.filter_distributed(shards, fc, cfd.CommMode(mode), tr)
    assert rel(res.X.panels_numpy(), d["topi4_X"]) <= 1e-10
    key = f"topi4_dist_w{workers}_m{mode}_"
    if key + "eta" in d:
        assert rel(res.moments.eta.cpu().numpy().reshape(48, 8), d[key + "eta"]) <= 1e-12
        assert rel(res.moments.mu.cpu().numpy().reshape(48, 8), d[key + "mu"]) <= 1e-12
    assert rel(res.moments.eta.cpu().numpy().reshape(48, 8), d["topi4_eta"]) <= 1e-12


@pytest.mark.parametrize("workers,mode", [(1, 0), (2, 0), (2, 1), (3, 1), (4, 0), (4, 1)])
def test_filter_distributed_native_matches_reference(workers, mode):
    """cf_filter_distributed (the library's own host loop, per-shard streams and
    event ordering, halo fused into the kernels' stores as mirror runs) against
    the reference's filter_distributed fixtures (acceptance.cpp:161-191)."""
    from paper_1803_02156_b200 import dist as cfd
    d = load("filter_small")
    H = cf.topi_generate(cf.LatticeSpec(4, 4, 4))
    fc = cf.filter_coefficients(-0.5, 0.5, cf.spectral_map(-8.0, 8.0), 50)
    X = cf.BlockVector(H.n, 8, 2, cf.InitSeededRandom(77), device=DEV)
    shards = cfd.shard_and_distribute(H, X, cfd.partition_rows(H, workers))
    res = cfd.filter_distributed_native(shards, fc, cfd.CommMode(mode), timeline=True)
    assert rel(res.X.panels_numpy(), d["topi4_X"]) <= 1e-10
    assert rel(res.moments.eta.cpu().numpy().reshape(48, 8), d["topi4_eta"]) <= 1e-12
    assert rel(res.moments.mu.cpu().numpy().reshape(48, 8), d["topi4_mu"]) <= 1e-12
    # measured timelines (dist.hpp:216-219): per worker one comm + one compute interval per (panel, step)
    steps = len(cf.kernels.degree_schedule(fc))
    assert len(res.timelines) == workers
    for tl in res.timelines:
        kinds = [e.kind for e in tl.events]
        assert kinds.count("compute") == kinds.count("comm") == 4 * steps
        assert all(e.end >= e.start >= 0 for e in tl.events) and tl.makespan() > 0


@pytest.mark.parametrize("workers,mode,nb", [(3, 0, 4), (3, 1, 4), (5, 1, 2), (2, 0, 32)])
def test_filter_distributed_native_scattered_halo(workers, mode, nb):
    """A random Hermitian matrix: the shards' halo rows are scattered (more than 4
    runs), so they move by the push kernel; against the serial checker."""
    from paper_1803_02156_b200 import dist as cfd
    H, _ = random_sparse(90, 0.08, 31, herm=True)
    fc = cf.filter_coefficients(-0.4, 0.4, cf.spectral_map(*cf.gershgorin_bounds(H), 0.01), 17)
    ns = 2 * nb
    X = cf.BlockVector(H.n, ns, nb, cf.InitSeededRandom(8), device=DEV)
    X0 = X.panels_numpy().copy()
    shards = cfd.shard_and_distribute(H, X, cfd.partition_rows(H, workers))
    res = cfd.filter_distributed_native(shards, fc, cfd.CommMode(mode))
    Xo, eta_o, mu_o = orc.apply_filter(as_oracle(H), X0, 17, fc.c, fc.g, fc.map.alpha, fc.map.beta)
    assert rel(res.X.panels_numpy(), Xo) <= 1e-10
    assert rel(res.moments.eta.cpu().numpy().reshape(15, ns), eta_o) <= 1e-11
    assert rel(res.moments.mu.cpu().numpy().reshape(15, ns), mu_o) <= 1e-11


def test_filter_distributed_native_rejects_bad_plans():
    from paper_1803_02156_b200 import dist as cfd
    H = cf.topi_generate(cf.LatticeSpec(4, 4, 4))
    fc = cf.filter_coefficients(-0.5, 0.5, cf.spectral_map(-8.0, 8.0), 10)
    X = cf.BlockVector(H.n, 4, 2, cf.InitSeededRandom(7), device=DEV)
    shards = cfd.shard_and_distribute(H, X, cfd.partition_rows(H, 2))
    with pytest.raises(ValueError):
        cfd.filter_distributed_native(shards[:1], fc, cfd.CommMode.vector)  # shard 0 sends to a missing shard
    with pytest.raises(ValueError):
        cfd.filter_distributed_native([], fc, cfd.CommMode.vector)


def test_halo_exchange_protocol_errors():  # test_dist.cpp:94-110
    from paper_1803_02156_b200 import dist as cfd
    H = cf.topi_generate(cf.LatticeSpec(4, 4, 4))
    X = cf.BlockVector(H.n, 4, 2, cf.InitSeededRandom(12), device=DEV)
    shards = cfd.shard_and_distribute(H, X, cfd.partition_rows(H, 2))
    t = cfd.LocalTransport(shards)
    with pytest.raises(cf.ProtocolError):
        cfd.halo_exchange(shards[0], shards[0].X, 0, cfd.ExchangePhase.finalize, t, 1)
    cfd.halo_exchange(shards[0], shards[0].X, 0, cfd.ExchangePhase.init, t, 1)
    with pytest.raises(cf.ProtocolError):
        cfd.halo_exchange(shards[0], shards[0].X, 0, cfd.ExchangePhase.init, t, 1)
    with pytest.raises(ValueError):
        cfd.halo_exchange(shards[0], shards[0].X, 9, cfd.ExchangePhase.init, t, 1)


def test_halo_exchange_delivers_owner_values():  # test_dist.cpp:77-92
    from paper_1803_02156_b200 import dist as cfd
    H = cf.topi_generate(cf.LatticeSpec(4, 4, 4))
    X = cf.BlockVector(H.n, 4, 2, cf.InitSeededRandom(12), device=DEV)
    shards = cfd.shard_and_distribute(H, X, cfd.partition_rows(H, 2))
    t = cfd.LocalTransport(shards)
    for sh in shards:
        cfd.halo_exchange(sh, sh.X, 0, cfd.ExchangePhase.init, t, 1)
    for sh in shards:
        cfd.halo_exchange(sh, sh.X, 0, cfd.ExchangePhase.finalize, t, 1)
    G = X.panel(0).cpu().numpy()
    for sh in shards:
        halo = sh.X.panel(0)[sh.local_n:].cpu().numpy()
        assert np.array_equal(halo, G[sh.plan.halo_global.astype(np.int64)])


def test_slab_matrix_step_equals_global_rows():
    """A rank's closed-form slab (local rows + halo slots) reproduces the global
    operator on its rows once the halo holds the neighbours' rows."""
    from paper_1803_02156_b200 import dist as cfd
    spec = cf.LatticeSpec(8, 8, 12)
    H = cf.topi_generate(spec)
    nb = 8
    U = orc.blockvec_random(H.n, nb, nb, 3)[0]
    Yg = orc.spmmv(as_oracle(H), 0.14, 0.01, U)
    for w in range(3):
        sp = cfd.topi_shard_plan(spec, 3, w)
        Ul = np.concatenate([U[sp.row_begin:sp.row_end], U[sp.halo_global.astype(np.int64)]])
        Xd, Yd = bv_from(Ul), cf.BlockVector(sp.local_n, nb, nb, device=DEV)
        cf.spmmv_shifted(sp.local, cf.ShiftScale(0.14, 0.01), cf.SubblockView(Xd, 0), cf.SubblockView(Yd, 0))
        assert rel(Yd.to_numpy(), Yg[sp.row_begin:sp.row_end]) <= 1e-13


def test_weak_scaling_slab_steps_match_single_gpu():
    """bench.py's N>1 step sequence (slab matrices, HaloPlan runs, cheb_init_tail,
    swap + halo + chebfd_op) for 2 and 3 ranks emulated in one process, against
    the single-matrix run on the whole lattice."""
    from paper_1803_02156_b200 import dist as cfd
    spec = cf.LatticeSpec(8, 8, 12)
    H = cf.topi_generate(spec)
    nb, steps = 8, 6
    fc = cf.filter_coefficients(-0.7, 0.7, cf.spectral_map(-7.0, 7.0, 0.01), 20)
    s = fc.map
    g = (fc.g[0] * fc.c[0], fc.g[1] * fc.c[1], fc.g[2] * fc.c[2])
    # single GPU reference
    X = cf.BlockVector(H.n, nb, nb, cf.InitSeededRandom(42), device=DEV)
    U, W = cf.BlockVector(H.n, nb, nb, device=DEV), cf.BlockVector(H.n, nb, nb, device=DEV)
    cf.cheb_init(H, s, cf.SubblockView(X, 0), cf.SubblockView(U, 0), cf.SubblockView(W, 0), *g)
    mom = cf.MomentSeries(fc.np, nb, device=DEV)
    for p in range(3, 3 + steps):
        cf.swap_blocks(cf.SubblockView(W, 0), cf.SubblockView(U, 0))
        cf.chebfd_op(H, s, cf.SubblockView(U, 0), cf.SubblockView(W, 0), cf.SubblockView(X, 0), p,
                     fc.g[p] * fc.c[p], mom)
    for world in (2, 3):
        slabs = [cfd.TopiSlab(spec, world, r) for r in range(world)]
        plans = [cfd.HaloPlan(sl.plan) for sl in slabs]
        vecs = []
        for sl in slabs:
            rows = sl.local_n + sl.halo_n
            vecs.append([cf.BlockVector(rows, nb, nb, cf.InitSeededRandom(42, sl.row_begin), device=DEV),
                         cf.BlockVector(rows, nb, nb, device=DEV), cf.BlockVector(rows, nb, nb, device=DEV),
                         cf.MomentSeries(fc.np, nb, device=DEV)])

        def exchange(k):  # k: 0 = X, 1 = U
            outs = {}
            for r, pl in enumerate(plans):
                for peer, start, cnt in pl.sends:
                    outs.setdefault((r, peer), []).append(vecs[r][k].panel(0)[start:start + cnt].clone())
            for r, pl in enumerate(plans):
                for peer, start, cnt in pl.recvs:
                    vecs[r][k].panel(0)[start:start + cnt].copy_(outs[(peer, r)].pop(0))

        exchange(0)
        for r, sl in enumerate(slabs):
            cf.spmmv_shifted(sl.local_matrix(), s, cf.SubblockView(vecs[r][0], 0), cf.SubblockView(vecs[r][1], 0))
        exchange(1)
        for r, sl in enumerate(slabs):
            Xl, Ul, Wl, _ = vecs[r]
            cf.cheb_init_tail(sl.local_matrix(), s, cf.SubblockView(Xl, 0), cf.SubblockView(Ul, 0),
                              cf.SubblockView(Wl, 0), *g)
        for p in range(3, 3 + steps):
            for r in range(world):
                cf.swap_blocks(cf.SubblockView(vecs[r][2], 0), cf.SubblockView(vecs[r][1], 0))
            exchange(1)
            for r, sl in enumerate(slabs):
                Xl, Ul, Wl, ml = vecs[r]
                cf.chebfd_op(sl.local_matrix(), s, cf.SubblockView(Ul, 0), cf.SubblockView(Wl, 0),
                             cf.SubblockView(Xl, 0), p, fc.g[p] * fc.c[p], ml)
        Xg = np.concatenate([vecs[r][0].to_numpy()[:slabs[r].local_n] for r in range(world)])
        assert rel(Xg, X.to_numpy()) <= 1e-13
        eta = sum(vecs[r][3].eta.cpu().numpy() for r in range(world))
        assert rel(eta, mom.eta.cpu().numpy()) <= 1e-12


@pytest.mark.parametrize("staged", [1, 0])
def test_moments_exact_under_repetition_both_kernels(staged):
    """Per-unit moment reduction (shared-memory handoff between warps) against
    fp64 torch sums, repeated: a race in the handoff shows up as a stale unit
    partial.  Runs the chunk-staged and the register-gather kernel (cf_tuning)."""
    from paper_1803_02156_b200._lib import check, lib
    check(lib.cf_tuning(b"staged", staged))
    try:
        H = cf.topi_generate(cf.LatticeSpec(32, 32, 24))
        n, nb = H.n, 32
        g = torch.Generator(device=DEV).manual_seed(11)
        U = torch.randn(n, nb, dtype=torch.complex128, device=DEV, generator=g)
        s = cf.ShiftScale(0.14144271570014144, 0.0)
        mu_ref = (U.conj() * U).sum(0)
        for rep in range(12):
            Wt = torch.randn(n, nb, dtype=torch.complex128, device=DEV, generator=g)
            Ub, Wb, Xb = (cf.BlockVector(n, nb, nb, device=DEV) for _ in range(3))
            Ub._panels[0], Wb._panels[0] = U, Wt
            mom = cf.MomentSeries(3, nb, device=DEV)
            cf.chebfd_op(H, s, cf.SubblockView(Ub, 0), cf.SubblockView(Wb, 0), cf.SubblockView(Xb, 0), 3, 0.01, mom)
            eta_ref = (Wb.panel(0).conj() * U).sum(0)
            assert torch.abs(mom.eta - eta_ref).max().item() <= 1e-12 * torch.abs(eta_ref).max().item(), rep
            assert torch.abs(mom.mu - mu_ref).max().item() <= 1e-12 * torch.abs(mu_ref).max().item(), rep
    finally:
        check(lib.cf_tuning(b"staged", 1))


def test_device_random_fill_matches_host_generator():
    """cf_blockvec_random_device: the reference's InitSeededRandom hashes on the
    device; Box-Muller values within a few ulp of the host (glibc) generator."""
    n, ns, nb, seed, off = 1000, 8, 4, 7, 123
    host = cf.seeded_random_host(n, ns, nb, seed, off)
    X = cf.BlockVector(n, ns, nb, device=DEV)
    cf.blockvec.random_fill_device(X, seed, off)
    assert np.abs(X.panels_numpy() - host).max() <= 1e-14
    Y = cf.BlockVector(n, ns, nb, device=DEV)
    cf.blockvec.random_fill_device(Y, seed, off, first_col=5)
    y = Y.to_numpy()
    assert np.all(y[:, :5] == 0) and np.abs(y[:, 5:] - X.to_numpy()[:, 5:]).max() <= 1e-14


def test_blockvec_handles_roundtrip_and_swap():
    """cf_blockvec (block_vector.hpp:53-151): zero-initialised panels, upload /
    download in the panel-concatenated layout, swap_blocks as an O(1) exchange of
    the panel buffers, the reference's error classes."""
    import ctypes as C
    from paper_1803_02156_b200._lib import check, lib
    a, b = C.c_void_p(), C.c_void_p()
    check(lib.cf_blockvec_create(0, 37, 12, 4, C.byref(a)))
    check(lib.cf_blockvec_create(0, 37, 8, 4, C.byref(b)))
    try:
        host = np.zeros((3, 37, 4), np.complex128)
        check(lib.cf_blockvec_download(a, host.ctypes.data))
        assert not host.any()
        src = (np.arange(3 * 37 * 4) + 1j).reshape(3, 37, 4)
        check(lib.cf_blockvec_upload(a, src.ctypes.data))
        p0, q1 = C.c_void_p(), C.c_void_p()
        check(lib.cf_blockvec_panel(a, 0, C.byref(p0)))
        check(lib.cf_blockvec_panel(b, 1, C.byref(q1)))
        check(lib.cf_panel_swap(a, 0, b, 1))
        r0, s1 = C.c_void_p(), C.c_void_p()
        check(lib.cf_blockvec_panel(a, 0, C.byref(r0)))
        check(lib.cf_blockvec_panel(b, 1, C.byref(s1)))
        assert (r0.value, s1.value) == (q1.value, p0.value)
        out_a = np.empty((3, 37, 4), np.complex128)
        out_b = np.empty((2, 37, 4), np.complex128)
        check(lib.cf_blockvec_download(a, out_a.ctypes.data))
        check(lib.cf_blockvec_download(b, out_b.ctypes.data))
        assert not out_a[0].any() and np.array_equal(out_a[1:], src[1:])
        assert np.array_equal(out_b[1], src[0]) and not out_b[0].any()
        rows, ns, nb, dev = C.c_size_t(), C.c_size_t(), C.c_size_t(), C.c_int()
        check(lib.cf_blockvec_shape(b, C.byref(rows), C.byref(ns), C.byref(nb), C.byref(dev)))
        assert (rows.value, ns.value, nb.value, dev.value) == (37, 8, 4, 0)
        with pytest.raises(IndexError):
            check(lib.cf_blockvec_panel(a, 3, C.byref(p0)))
        c = C.c_void_p()
        check(lib.cf_blockvec_create(0, 36, 4, 4, C.byref(c)))
        with pytest.raises(ValueError):
            check(lib.cf_panel_swap(a, 0, c, 0))
        check(lib.cf_blockvec_destroy(c))
        with pytest.raises(ValueError):
            check(lib.cf_blockvec_create(0, 10, 6, 4, C.byref(c)))
    finally:
        check(lib.cf_blockvec_destroy(a))
        check(lib.cf_blockvec_destroy(b))


@pytest.mark.parametrize("lattice,open_b", [((8, 6, 5), False), ((16, 8, 4), False), ((8, 4, 4), True)])
def test_typed_records_match_full_records(lattice, open_b):
    """The staged kernel's typed records (Topi entries are purely real or purely
    imaginary: one double per value, two FMAs per entry) agree with the full
    complex records (blocks of one pattern are summed in value-type order instead
    of column order: rounding-level differences), for the filter; and both match
    the checker."""
    from paper_1803_02156_b200._lib import check, lib
    bc = cf.Boundary.open if open_b else cf.Boundary.periodic
    H = cf.topi_generate(cf.LatticeSpec(*lattice, boundary=bc))
    fc = cf.filter_coefficients(-0.4, 0.45, cf.spectral_map(-7.0, 7.0, 0.01), 23)
    outs = []
    try:
        for typed in (1, 0):
            check(lib.cf_tuning(b"typed", typed))
            X = cf.BlockVector(H.n, 64, 32, cf.InitSeededRandom(4), device=DEV)
            mom = cf.apply_filter(H, X, fc)
            outs.append((X.panels_numpy(), mom.eta.cpu().numpy(), mom.mu.cpu().numpy()))
    finally:
        check(lib.cf_tuning(b"typed", 1))
    for a, b in zip(outs[0], outs[1]):
        assert rel(a, b) <= 1e-13
    Xo, eta_o, _ = orc.apply_filter(as_oracle(H), orc.blockvec_random(H.n, 64, 32, 4), 23, fc.c, fc.g, fc.map.alpha,
                                    fc.map.beta)
    assert rel(outs[0][0], Xo) <= 1e-10
    assert rel(outs[0][1].reshape(21, 64), eta_o) <= 1e-12


@pytest.mark.parametrize("mass,hop", [(0.3, 0.7), (0.0, 1.0), (-1.5, 0.25)])
def test_typed_records_other_couplings(mass, hop):
    """Typed records for Topi lattices with other mass / hopping (the value-type
    pattern follows the stencil, not the values; mass 0 leaves explicit zeros):
    filter results against the checker, both kernels' widths."""
    H = cf.topi_generate(cf.LatticeSpec(8, 4, 4, mass=mass, hop=hop))
    lo, hi = cf.gershgorin_bounds(H)
    fc = cf.filter_coefficients(lo + 0.4 * (hi - lo), lo + 0.6 * (hi - lo), cf.spectral_map(lo, hi, 0.01), 19)
    for ns, nb in ((32, 32), (16, 8)):
        X = cf.BlockVector(H.n, ns, nb, cf.InitSeededRandom(9), device=DEV)
        mom = cf.apply_filter(H, X, fc)
        Xo, eta_o, mu_o = orc.apply_filter(as_oracle(H), orc.blockvec_random(H.n, ns, nb, 9), 19, fc.c, fc.g,
                                           fc.map.alpha, fc.map.beta)
        assert rel(X.panels_numpy(), Xo) <= 1e-10
        assert rel(mom.eta.cpu().numpy().reshape(17, ns), eta_o) <= 1e-12
        assert rel(mom.mu.cpu().numpy().reshape(17, ns), mu_o) <= 1e-12


@pytest.mark.parametrize("workers", [2, 3])
def test_matrix_create_topi_shard_matches_shard_plan(workers):
    """cf_matrix_create_topi_shard (a rank's device operator generated in closed
    form) = the device image of the shard plan's local CRS: same extents, and
    the same (aH+b)U rows on every shard."""
    import ctypes as C
    from paper_1803_02156_b200 import dist as cfd
    from paper_1803_02156_b200._lib import check, lib
    spec = cf.LatticeSpec(8, 6, 6)
    s = cf.ShiftScale(0.14, -0.03)
    for w in range(workers):
        plan = cfd.topi_shard_plan(spec, workers, w)
        h = C.c_void_p()
        rb, ln, hn = C.c_size_t(), C.c_size_t(), C.c_size_t()
        check(lib.cf_matrix_create_topi_shard(0, 8, 6, 6, 1.0, 1.0, 0, workers, w, C.byref(rb), C.byref(ln),
                                              C.byref(hn), C.byref(h)))
        try:
            assert (rb.value, ln.value, hn.value) == (plan.row_begin, plan.local_n, plan.halo_n)
            rows = plan.local_n + plan.halo_n
            U = cf.BlockVector(rows, 32, 32, cf.InitSeededRandom(3 + w), device=DEV)
            Y1 = cf.BlockVector(rows, 32, 32, device=DEV)
            Y2 = cf.BlockVector(rows, 32, 32, device=DEV)
            cf.spmmv_shifted(plan.local, s, cf.SubblockView(U, 0), cf.SubblockView(Y1, 0))
            check(lib.cf_spmmv_shifted(h, s.alpha, s.beta, U.panel(0).data_ptr(), Y2.panel(0).data_ptr(), 32, 32,
                                       None))
            torch.cuda.synchronize()
            assert torch.equal(Y1.panel(0)[:plan.local_n], Y2.panel(0)[:plan.local_n])
        finally:
            check(lib.cf_matrix_destroy(h))


def test_host_and_distributed_filter_argument_errors():
    """The reference's argument checks on the new entries (filter.hpp:76-93,
    dist.hpp:227-236): degree < 2, n_b not dividing n_s, row-count mismatch."""
    from paper_1803_02156_b200 import dist as cfd
    H = cf.topi_generate(cf.LatticeSpec(4, 4, 4))
    fc = cf.filter_coefficients(-0.5, 0.5, cf.spectral_map(-8.0, 8.0), 10)
    with pytest.raises(ValueError):
        cf.apply_filter_host(H, np.zeros((2, H.n + 4, 4), np.complex128), fc)
    X = cf.BlockVector(H.n, 4, 2, cf.InitSeededRandom(7), device=DEV)
    shards = cfd.shard_and_distribute(H, X, cfd.partition_rows(H, 2))
    bad = cf.FilterCoefficients(np=1, c=fc.c[:2], g=fc.g[:2], window_lo=fc.window_lo, window_hi=fc.window_hi,
                                map=fc.map)
    with pytest.raises(ValueError):
        cfd.filter_distributed_native(shards, bad, cfd.CommMode.vector)
    res = cfd.filter_distributed_native(shards, fc, cfd.CommMode.pipelined)  # still usable afterwards
    assert np.isfinite(res.X.panels_numpy()).all()


@pytest.mark.parametrize("workers,nb,scattered", [(1, 2, False), (2, 2, False), (4, 2, False), (3, 4, True),
                                                  (2, 32, False)])
def test_filter_distributed_host_staged_panels(workers, nb, scattered):
    """cf_filter_distributed_host (configs[3]'s capacity path): the shards' X
    panels stay in pinned host memory and stream through two device slots per
    shard, against the reference's filter_distributed fixtures (slab shards) or
    the serial checker (scattered halo, push kernel)."""
    from paper_1803_02156_b200 import dist as cfd
    if scattered:
        H, _ = random_sparse(90, 0.08, 31, herm=True)
        fc = cf.filter_coefficients(-0.4, 0.4, cf.spectral_map(*cf.gershgorin_bounds(H), 0.01), 17)
        ns = 3 * nb
        X = cf.BlockVector(H.n, ns, nb, cf.InitSeededRandom(8), device=DEV)
    else:
        d = load("filter_small")
        H = cf.topi_generate(cf.LatticeSpec(4, 4, 4))
        fc = cf.filter_coefficients(-0.5, 0.5, cf.spectral_map(-8.0, 8.0), 50)
        ns = 8 if nb == 2 else 64
        X = cf.BlockVector(H.n, ns, nb, cf.InitSeededRandom(77), device=DEV)
    X0 = X.panels_numpy().copy()
    shards = cfd.shard_and_distribute(H, X, cfd.partition_rows(H, workers), host_panels=True)
    assert all(sh.host_staged and sh.X.panel(0).is_pinned() for sh in shards)
    with pytest.raises(ValueError, match="vector schedule"):
        cfd.filter_distributed_native(shards, fc, cfd.CommMode.pipelined)
    res = cfd.filter_distributed(shards, fc, cfd.CommMode.vector, None)
    if not scattered and nb == 2:
        assert rel(res.X.panels_numpy(), d["topi4_X"]) <= 1e-10
        assert rel(res.moments.eta.cpu().numpy().reshape(48, 8), d["topi4_eta"]) <= 1e-12
    else:
        Xo, eta_o, mu_o = orc.apply_filter(as_oracle(H), X0, fc.np, fc.c, fc.g, fc.map.alpha, fc.map.beta)
        assert rel(res.X.panels_numpy(), Xo) <= 1e-10
        assert rel(res.moments.eta.cpu().numpy().reshape(fc.np - 2, ns), eta_o) <= 1e-11
        assert rel(res.moments.mu.cpu().numpy().reshape(fc.np - 2, ns), mu_o) <= 1e-11


@pytest.mark.parametrize("kind", ["open", "disorder"])
def test_mixed_typed_records(kind):
    """Typed records per piece: an open lattice's surface chunks (not signature
    chunks) stay full records next to typed interior chunks in one stream; onsite
    disorder (every site's diagonal differs, still real) keeps every piece typed.
    Filter against the checker on both kernels (n_b = 32 staged, n_b = 8 gather)."""
    import ctypes as C
    from paper_1803_02156_b200._lib import check, lib
    if kind == "open":
        H = cf.topi_generate(cf.LatticeSpec(32, 8, 8, boundary=cf.Boundary.open))  # chunks clear of x surfaces
    else:
        H0 = cf.topi_generate(cf.LatticeSpec(16, 8, 4))
        rows = np.repeat(np.arange(H0.n), np.diff(H0.row_ptr.astype(np.int64)))
        v = H0.values.copy()
        dm = H0.col_idx == rows
        v[dm] += np.random.default_rng(3).uniform(-1, 1, dm.sum())
        H = cf.SparseMatrixCRS(H0.n, H0.row_ptr, H0.col_idx, v, lattice=(16, 8, 4))
    dmh = H.device_matrix(0)
    tp, npc = C.c_size_t(), C.c_size_t()
    check(lib.cf_matrix_typed(dmh.handle, C.byref(tp), C.byref(npc)))
    if kind == "open":
        assert 0 < tp.value < npc.value
    else:
        assert tp.value == npc.value > 0
    lo, hi = cf.gershgorin_bounds(H)
    fc = cf.filter_coefficients(lo + 0.4 * (hi - lo), lo + 0.6 * (hi - lo), cf.spectral_map(lo, hi, 0.01), 21)
    for ns, nb in ((64, 32), (16, 8)):
        X = cf.BlockVector(H.n, ns, nb, cf.InitSeededRandom(6), device=DEV)
        mom = cf.apply_filter(H, X, fc)
        Xo, eta_o, mu_o = orc.apply_filter(as_oracle(H), orc.blockvec_random(H.n, ns, nb, 6), 21, fc.c, fc.g,
                                           fc.map.alpha, fc.map.beta)
        assert rel(X.panels_numpy(), Xo) <= 1e-10
        assert rel(mom.eta.cpu().numpy().reshape(19, ns), eta_o) <= 1e-12
        assert rel(mom.mu.cpu().numpy().reshape(19, ns), mu_o) <= 1e-12


def test_hbm_budget_refuses_before_allocating():
    """The pre-flight device-memory budget (chebfd_kernels.cu hbm_budget): a
    workspace that cannot fit raises ValueError (CF_EINVAL) naming the sizes,
    before anything is allocated or read -- never an allocator failure half-way.
    Here the moment series of an absurd degree (4e8 steps x 32 columns, 205 GB
    each for eta and mu) overflows the GPU for the host-staged filter and for the
    host-staged distributed filter."""
    import ctypes as C
    from paper_1803_02156_b200 import dist as cfd
    from paper_1803_02156_b200._lib import check, lib
    H = cf.topi_generate(cf.LatticeSpec(4, 4, 4))
    dm = H.device_matrix(0)
    x = np.zeros((1, H.n, 32), np.complex128)
    cg = np.zeros(8)
    np_big = 400_000_000
    with pytest.raises(ValueError, match="more device memory"):
        check(lib.cf_apply_filter_host(dm.handle, x.ctypes.data, 32, 32, np_big, cg.ctypes.data, cg.ctypes.data, 0.1,
                                       0.0, None, None))
    X = cf.BlockVector(H.n, 32, 32, device=DEV)
    shards = cfd.shard_and_distribute(H, X, cfd.partition_rows(H, 2), host_panels=True)
    arr = (cfd._DistWorkerC * 2)()
    keep = []
    for w, sh in enumerate(shards):
        pp = (C.c_void_p * 1)(sh.X.panel(0).data_ptr())
        sf, rf = np.ascontiguousarray(sh.plan.send_flat()), np.ascontiguousarray(sh.plan.recv_flat())
        keep += [pp, sf, rf]
        arr[w] = cfd._DistWorkerC(sh.local.device_matrix(0).handle, sh.local_n, sh.halo_n, C.cast(pp, C.c_void_p),
                                  sf.ctypes.data, sf.size, rf.ctypes.data, rf.size)
    with pytest.raises(ValueError, match="more device memory"):
        check(lib.cf_filter_distributed_host(arr, 2, 32, 32, np_big, cg.ctypes.data, cg.ctypes.data, 0.1, 0.0, 0, None,
                                             None))


@pytest.mark.parametrize("nb,ns", [(8, 64), (16, 64), (64, 64), (12, 96), (4, 64), (24, 96), (1, 32), (12, 36)])
def test_apply_filter_narrow_panels_run_wide(nb, ns):
    """n_b < 32 panels with n_s a multiple of 32 are filtered as 32-wide panels
    (packed, chunk-staged kernel, unpacked; n_b = 12 / 24 panels straddle two
    slices), n_b = 64 panels one 32-column slice at a time, and n_s = 36 keeps
    the panel-by-panel loop: X and moments against the checker."""
    H = cf.topi_generate(cf.LatticeSpec(8, 6, 5))
    fc = cf.filter_coefficients(-0.5, 0.5, cf.spectral_map(*cf.gershgorin_bounds(H), 0.01), 27)
    X = cf.BlockVector(H.n, ns, nb, cf.InitSeededRandom(13), device=DEV)
    mom = cf.apply_filter(H, X, fc)
    Xo, eta_o, mu_o = orc.apply_filter(as_oracle(H), orc.blockvec_random(H.n, ns, nb, 13), 27, fc.c, fc.g,
                                       fc.map.alpha, fc.map.beta)
    assert rel(X.panels_numpy(), Xo) <= 1e-10
    assert rel(mom.eta.cpu().numpy().reshape(25, ns), eta_o) <= 1e-12
    assert rel(mom.mu.cpu().numpy().reshape(25, ns), mu_o) <= 1e-12


@pytest.mark.parametrize("nb", [2, 4, 8, 12, 16])
def test_narrow_staged_kernel_matches_gather_kernel(nb):
    """n_b = 8 / 16 whole-row panels of a periodic lattice run the narrow staged
    kernel (G = 32 / n_b chunks per stage); with cf_tuning("narrow", 0) the
    register-gather kernel.  Same per-row block order: X bit-identical; moments
    (different summation tree) to rounding; both against the checker."""
    from paper_1803_02156_b200._lib import check, lib
    H = cf.topi_generate(cf.LatticeSpec(16, 12, 10))
    assert H.device_matrix(0).info()["narrow"]
    fc = cf.filter_coefficients(-0.5, 0.5, cf.spectral_map(*cf.gershgorin_bounds(H), 0.01), 31)
    out = {}
    try:
        for v in (1, 0):
            check(lib.cf_tuning(b"narrow", v))
            # one panel (n_s = n_b is not packed into a 32-wide panel)
            Xs = cf.BlockVector(H.n, nb, nb, cf.InitSeededRandom(21), device=DEV)
            mom = cf.apply_filter(H, Xs, fc)
            out[v] = (Xs.panels_numpy().copy(), mom.eta.cpu().numpy().copy(), mom.mu.cpu().numpy().copy())
    finally:
        check(lib.cf_tuning(b"narrow", 1))
    assert np.array_equal(out[0][0].view(np.uint64), out[1][0].view(np.uint64))
    assert rel(out[1][1], out[0][1]) <= 1e-13 and rel(out[1][2], out[0][2]) <= 1e-13
    Xo, eta_o, mu_o = orc.apply_filter(as_oracle(H), orc.blockvec_random(H.n, nb, nb, 21), 31, fc.c, fc.g,
                                       fc.map.alpha, fc.map.beta)
    assert rel(out[1][0], Xo) <= 1e-10
    assert rel(out[1][1].reshape(29, nb), eta_o) <= 1e-12
    assert rel(out[1][2].reshape(29, nb), mu_o) <= 1e-12
