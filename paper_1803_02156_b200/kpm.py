"""Eigencount estimate from the filter's moments (kernel polynomial method).

The reference exposes the raw moments of `chebfd_op` and leaves the count
estimator out (the paper "uses moments to monitor the number of
eigenstates in the search interval" without a formula; PAPER.md:43 cites KPM).
This module supplies the standard KPM estimator on top of those moments.

Moments.  At degree step p (p = 3..n_p, kernels.hpp:180-202) the fused kernel
accumulates, per column j,
    eta_p = (T_p x)^H (T_{p-1} x),   mu_p = (T_{p-1} x)^H (T_{p-1} x),
with T_k = T_k(alpha H + beta).  For Hermitian H, T_m T_n = (T_{m+n} + T_{|m-n|}) / 2,
so with m_k = x^H T_k x (real):
    m_{2p-1} = 2 Re eta_p - m_1,   m_{2p-2} = 2 mu_p - m_0      (p = 3..n_p),
and the four start values m_0 = x^H x, m_1 = x^H T_1 x, m_2 = 2 |T_1 x|^2 - m_0,
m_3 = 2 Re (T_2 x)^H (T_1 x) - m_1 come from the recurrence start vectors
(`init_moments`).  A filter run of degree n_p thus yields K = 2 n_p moments.

Estimate.  tr T_k ~= n * sum_j m_k^(j) / sum_j m_0^(j) (stochastic trace over the
n_s random columns, ratio form: exact for an orthonormal basis of columns), and
    N(a, b) ~= sum_{k<K} g_k c_k(a, b) tr T_k,
with c_k, g_k the window's Chebyshev and Jackson coefficients at degree K - 1
(filter.hpp:39-70, the same routine the filter uses).  The per-column
estimates give the statistical error.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .blockvec import BlockVector, InitSeededRandom, SubblockView
from .filter import Damping, apply_filter, filter_coefficients, spectral_map
from .kernels import MomentSeries, ShiftScale, spmmv_shifted, spmmv_shifted_two_minus
from .sparse import SparseMatrixCRS, gershgorin_bounds


@dataclass
class InitMoments:
    """Per-column start values: m0 = x^H x, m1 = x^H T1 x, t11 = |T1 x|^2, t21 = (T2 x)^H (T1 x)."""
    m0: np.ndarray
    m1: np.ndarray
    t11: np.ndarray
    t21: np.ndarray


@dataclass
class EigenCount:
    estimate: float          # estimated eigenvalue count in the window
    stderr: float            # standard error over the columns
    per_column: np.ndarray   # n * (sum_k g_k c_k m_k^(j)) / m_0^(j)
    moments: int             # K = 2 n_p moments used


def init_moments(H: SparseMatrixCRS, s: ShiftScale, X: BlockVector) -> InitMoments:
    """m0, m1, |T1 x|^2, (T2 x)^H T1 x per column of X, on the device: T1 X and
    T2 X by the SpMMV kernels (kernels.hpp:82-127), the dots by cf_gram."""
    from .solve import gram_matrix
    n, ns, nb = X.rows(), X.cols(), X.block_width()
    T1 = BlockVector(n, ns, nb, device=X.device)
    T2 = BlockVector(n, ns, nb, device=X.device)
    for b in range(X.panel_count()):
        spmmv_shifted(H, s, SubblockView(X, b), SubblockView(T1, b))
        spmmv_shifted_two_minus(H, s, SubblockView(T1, b), SubblockView(T2, b), SubblockView(X, b))
    m0 = np.empty(ns)
    m1 = np.empty(ns)
    t11 = np.empty(ns)
    t21 = np.empty(ns)
    for b in range(X.panel_count()):  # one panel at a time: diagonal blocks only
        sl = slice(b * nb, (b + 1) * nb)
        xb, ub, wb = X.panel_view(b), T1.panel_view(b), T2.panel_view(b)
        m0[sl] = np.real(np.diag(gram_matrix(xb)))
        m1[sl] = np.real(np.diag(gram_matrix(xb, ub)))
        t11[sl] = np.real(np.diag(gram_matrix(ub)))
        t21[sl] = np.real(np.diag(gram_matrix(wb, ub)))
    return InitMoments(m0, m1, t11, t21)


def kpm_moments(mom: MomentSeries, init: InitMoments) -> np.ndarray:
    """m_k^(j) for k = 0..2 n_p - 1 (rows) and the n_s columns."""
    np_, ns = mom.degree_max, mom.columns
    if np_ < 3:
        raise ValueError("kpm_moments: the filter ran no degree steps (n_p < 3)")
    eta = np.asarray(mom.eta.cpu().numpy() if hasattr(mom.eta, "cpu") else mom.eta).reshape(np_ - 2, ns)
    mu = np.asarray(mom.mu.cpu().numpy() if hasattr(mom.mu, "cpu") else mom.mu).reshape(np_ - 2, ns)
    return moments_from_series(eta, mu, init)


def moments_from_series(eta: np.ndarray, mu: np.ndarray, init: InitMoments) -> np.ndarray:
    """The algebra of kpm_moments on host arrays eta, mu of shape (n_p - 2, n_s)."""
    rows, ns = eta.shape
    K = 2 * (rows + 2)
    m = np.empty((K, ns))
    m[0] = init.m0
    m[1] = init.m1
    m[2] = 2.0 * init.t11 - init.m0
    m[3] = 2.0 * init.t21 - init.m1
    p = np.arange(3, rows + 3)
    m[2 * p - 1] = 2.0 * np.real(eta) - init.m1
    m[2 * p - 2] = 2.0 * np.real(mu) - init.m0
    return m


def eigencount(moments: np.ndarray, m0: np.ndarray, n: int, window_lo: float, window_hi: float, map: ShiftScale,
               damping: Damping = Damping.jackson) -> EigenCount:
    """KPM estimate of the number of eigenvalues in [window_lo, window_hi] from
    K moments per column (rows of `moments`)."""
    K, ns = moments.shape
    if K < 3:
        raise ValueError("eigencount: need at least 3 moments")
    if not window_lo < window_hi:
        raise ValueError("eigencount: empty window")
    fc = filter_coefficients(window_lo, window_hi, map, K - 1, damping)
    w = fc.g * fc.c
    per = n * (w @ moments) / m0
    est = float(n * (w @ moments.sum(axis=1)) / m0.sum())
    se = float(per.std(ddof=1) / np.sqrt(ns)) if ns > 1 else float("nan")
    return EigenCount(est, se, per, K)


def estimate_eigencount(H: SparseMatrixCRS, window_lo: float, window_hi: float, n_s: int = 32, n_b: int = 32,
                        n_p: int = 200, seed: int = 42, spectral_bounds=None, X: BlockVector | None = None,
                        device=None) -> EigenCount:
    """Random start block (InitSeededRandom(seed), or X), its start moments, one
    filter run of degree n_p on the device (its coefficients do not enter the
    moments), then the 2 n_p-moment KPM estimate for the window."""
    import torch
    lo, hi = spectral_bounds if spectral_bounds is not None else gershgorin_bounds(H)
    s = spectral_map(lo, hi, 0.0 if spectral_bounds is not None else 0.01)
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    if X is None:
        X = BlockVector(H.n, n_s, n_b, InitSeededRandom(seed), device=dev)
    init = init_moments(H, s, X)
    fc = filter_coefficients(window_lo, window_hi, s, n_p)
    mom = apply_filter(H, X, fc)
    return eigencount(kpm_moments(mom, init), init.m0, H.n, window_lo, window_hi, s)
