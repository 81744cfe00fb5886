"""KPM eigencount from the filter's moments (paper_1803_02156_b200/kpm.py).

CPU: the moment algebra (eta/mu of the fused step -> x^H T_k x) and the
estimator against dense numpy recurrences.  GPU: the device path with an
orthonormal start block (exact trace) against the dense spectrum, and with
random columns on the cfg1 lattice against the analytic Bloch spectrum
(tests/bloch.py), within the estimator's own standard error."""
import numpy as np
import pytest

import paper_1803_02156_b200 as cf
from paper_1803_02156_b200 import kpm


def _dense_cheb(Hd, alpha, beta, X, K):
    A = alpha * Hd + beta * np.eye(Hd.shape[0])
    T = [X, A @ X]
    for _ in range(2, K):
        T.append(2 * A @ T[-1] - T[-2])
    return T


def _series(Hd, alpha, beta, X, np_):
    """eta_p, mu_p exactly as the fused step accumulates them (kernels.hpp:189-193)."""
    T = _dense_cheb(Hd, alpha, beta, X, np_ + 1)
    eta = np.array([np.sum(np.conj(T[p]) * T[p - 1], axis=0) for p in range(3, np_ + 1)])
    mu = np.array([np.sum(np.conj(T[p - 1]) * T[p - 1], axis=0) for p in range(3, np_ + 1)])
    init = kpm.InitMoments(np.real(np.sum(np.conj(X) * X, 0)), np.real(np.sum(np.conj(X) * T[1], 0)),
                           np.real(np.sum(np.conj(T[1]) * T[1], 0)), np.real(np.sum(np.conj(T[2]) * T[1], 0)))
    return T, eta, mu, init


def _hermitian(n, seed):
    rng = np.random.default_rng(seed)
    a = rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))
    return (a + a.conj().T) / 2


def test_moment_algebra_recovers_every_moment():
    Hd = _hermitian(40, 3)
    ev = np.linalg.eigvalsh(Hd)
    s = cf.spectral_map(ev[0] - 0.1, ev[-1] + 0.1, 0.01)
    rng = np.random.default_rng(1)
    X = rng.standard_normal((40, 6)) + 1j * rng.standard_normal((40, 6))
    np_ = 30
    T, eta, mu, init = _series(Hd, s.alpha, s.beta, X, np_)
    m = kpm.moments_from_series(eta, mu, init)
    T2 = _dense_cheb(Hd, s.alpha, s.beta, X, 2 * np_)
    want = np.array([np.real(np.sum(np.conj(X) * T2[k], 0)) for k in range(2 * np_)])
    assert m.shape == (2 * np_, 6)
    assert np.abs(m - want).max() <= 1e-9 * np.abs(want).max()


def test_eigencount_exact_for_an_orthonormal_start_block():
    n = 48
    Hd = _hermitian(n, 5)
    ev = np.linalg.eigvalsh(Hd)
    s = cf.spectral_map(ev[0], ev[-1], 0.01)
    X = np.eye(n, dtype=np.complex128)
    np_ = 60
    _, eta, mu, init = _series(Hd, s.alpha, s.beta, X, np_)
    lo, hi = -1.0, 1.5
    r = kpm.eigencount(kpm.moments_from_series(eta, mu, init), init.m0, n, lo, hi, s)
    fc = cf.filter_coefficients(lo, hi, s, 2 * np_ - 1)
    x = s.alpha * ev + s.beta
    damped = sum(np.sum(fc.g * fc.c * np.cos(np.arange(2 * np_) * np.arccos(xi))) for xi in x)
    assert r.moments == 2 * np_
    assert r.estimate == pytest.approx(damped, rel=1e-10, abs=1e-9)
    # the damped window count rounds to the true count when no eigenvalue sits at an edge
    assert abs(r.estimate - np.sum((ev >= lo) & (ev <= hi))) < 1.0


def test_eigencount_argument_errors():
    s = cf.ShiftScale(0.1, 0.0)
    with pytest.raises(ValueError, match="empty window"):
        kpm.eigencount(np.ones((8, 2)), np.ones(2), 4, 0.5, 0.5, s)
    with pytest.raises(ValueError, match="at least 3 moments"):
        kpm.eigencount(np.ones((2, 2)), np.ones(2), 4, 0.0, 0.5, s)


@pytest.mark.gpu
def test_device_eigencount_orthonormal_block_matches_dense_spectrum():
    import torch
    H = cf.topi_generate(cf.LatticeSpec(3, 3, 3, 0.83, 1.1, cf.Boundary.open))
    n = H.n  # 108
    ev = np.linalg.eigvalsh(cf.to_dense(H))
    lo_b, hi_b = cf.gershgorin_bounds(H)
    s = cf.spectral_map(lo_b, hi_b, 0.01)
    X = cf.BlockVector.from_numpy(np.eye(n, dtype=np.complex128), 4, device="cuda:0")
    r = kpm.estimate_eigencount(H, 0.3, 0.7, n_p=80, X=X)
    torch.cuda.synchronize()
    fc = cf.filter_coefficients(0.3, 0.7, s, 159)
    x = s.alpha * ev + s.beta
    damped = sum(np.sum(fc.g * fc.c * np.cos(np.arange(160) * np.arccos(xi))) for xi in x)
    assert r.estimate == pytest.approx(damped, rel=1e-9, abs=1e-9)


@pytest.mark.gpu
def test_device_eigencount_random_block_cfg1_lattice():
    import torch
    import bloch
    dims = (64, 64, 40)
    blocks = bloch.site_blocks()
    ks = np.stack(np.meshgrid(*[2 * np.pi * np.arange(d) / d for d in dims], indexing="ij"), -1).reshape(-1, 3)
    hk = sum(b[None] * np.exp(1j * (ks @ np.array(d, float)))[:, None, None] for d, b in blocks.items())
    ev = np.linalg.eigvalsh(hk).ravel()
    H = cf.topi_generate(cf.LatticeSpec(*dims))
    lo, hi = -0.12, 0.12
    r = kpm.estimate_eigencount(H, lo, hi, n_s=64, n_b=32, n_p=300, spectral_bounds=(-4.0, 4.0))
    torch.cuda.synchronize()
    s = cf.spectral_map(-4.0, 4.0, 0.0)
    fc = cf.filter_coefficients(lo, hi, s, 599)
    x = np.clip(s.alpha * ev + s.beta, -1, 1)
    th = np.arccos(x)
    damped = float(np.sum(np.cos(np.outer(th, np.arange(600))) @ (fc.g * fc.c)))
    exact = int(np.sum((ev >= lo) & (ev <= hi)))
    assert exact == 60
    assert abs(r.estimate - damped) < 5 * r.stderr + 1.0, (r.estimate, r.stderr, damped)
    assert abs(r.estimate - exact) < 0.25 * exact
