"""Interior eigensolver: SVQB, Rayleigh-Ritz and the restarted ChebFD loop.

Mirrors proj/include/chebfilter/filter.hpp:98-320 and jacobi_eig.hpp:14-98:
``orthogonalize_svqb`` (:139-150), ``rayleigh_ritz`` (:170-211), ``RitzPair`` /
``SolveResult`` / ``SolveOptions`` (:213-241) and ``chebfd_solve`` (:247-320),
with the same names, defaults and exceptions.  The loop runs inside
libchebfd_b200 (``cf_chebfd_solve``): apply_filter, the tall-skinny Gram and
rotation kernels and the residual sums on the device, the k x k Jacobi
eigenproblems on the host.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np
import torch

from ._lib import check, lib, ptr
from .blockvec import BlockVector
from .filter import Damping
from .kernels import MomentSeries, _stream
from .sparse import SparseMatrixCRS


class SolveOptionsC(C.Structure):
    _fields_ = [("n_s", C.c_size_t), ("n_b", C.c_size_t), ("n_p", C.c_size_t), ("max_restarts", C.c_size_t),
                ("res_tol", C.c_double), ("margin", C.c_double), ("seed", C.c_uint64), ("damping", C.c_int),
                ("has_bounds", C.c_int), ("bound_lo", C.c_double), ("bound_hi", C.c_double),
                ("drop_tol", C.c_double)]


class SolveResultC(C.Structure):
    _fields_ = [("n_eig", C.c_size_t), ("n_pairs", C.c_size_t), ("iterations", C.c_size_t), ("converged", C.c_int),
                ("eigenvalues", C.c_void_p), ("residuals", C.c_void_p), ("pair_values", C.c_void_p),
                ("pair_residuals", C.c_void_p), ("pair_flags", C.c_void_p), ("eigenvectors", C.c_void_p),
                ("eta", C.c_void_p), ("mu", C.c_void_p), ("phase_ms", C.c_void_p)]


lib.cf_chebfd_solve.restype = C.c_int
lib.cf_chebfd_solve.argtypes = [C.c_void_p, C.c_double, C.c_double, C.POINTER(SolveOptionsC),
                                C.POINTER(SolveResultC), C.c_void_p]


@dataclass
class EigenDecomposition:
    values: np.ndarray   # ascending
    vectors: np.ndarray  # k x k, column j is the eigenvector of values[j]


def jacobi_hermitian_eig(A: np.ndarray, tol: float = 1e-12, max_sweeps: int = 64) -> EigenDecomposition:
    """jacobi_eig.hpp:32-98 (host C++ in the library)."""
    A = np.ascontiguousarray(A, np.complex128)
    k = A.shape[0]
    if A.shape != (k, k):
        raise ValueError("jacobi_hermitian_eig: square matrix expected")
    vals = np.empty(k)
    vecs = np.empty((k, k), np.complex128)
    check(lib.cf_jacobi_hermitian_eig(k, ptr(A), tol, max_sweeps, ptr(vals), ptr(vecs)))
    return EigenDecomposition(vals, vecs)


def _panels(X: BlockVector):
    for p in (X.panel(b) for b in range(X.panel_count())):
        if not p.is_cuda:
            raise RuntimeError("libchebfd_b200 operates on CUDA tensors only (no CPU path)")
    return (C.c_void_p * X.panel_count())(*[X.panel(b).data_ptr() for b in range(X.panel_count())])


def gram_matrix(A: BlockVector, B: BlockVector | None = None) -> np.ndarray:
    """S = A^H B (filter.hpp:99-109) on the device; returned on the host."""
    B = A if B is None else B
    if A.rows() != B.rows():
        raise ValueError("gram_matrix: row count mismatch")
    S = torch.empty((A.cols(), B.cols()), dtype=torch.complex128, device=A.device)
    check(lib.cf_gram(A.rows(), _panels(A), A.block_width(), A.cols(), _panels(B), B.block_width(), B.cols(),
                      S.data_ptr(), _stream()))
    return S.cpu().numpy()


def max_gram_defect(Q: BlockVector) -> float:
    """filter.hpp:111-120."""
    G = gram_matrix(Q)
    return float(np.abs(G - np.eye(G.shape[0])).max())


def orthogonalize_svqb(X: BlockVector, drop_tol: float = 1e-12) -> tuple[BlockVector, int]:
    """filter.hpp:139-150: SVQB with extra passes while the defect exceeds 1e-10.
    Returns Q = BlockVector(n, rank, rank) (one panel) and the rank."""
    n, ns = X.rows(), X.cols()
    buf = torch.empty(n * ns, dtype=torch.complex128, device=X.device)
    rank = C.c_size_t()
    check(lib.cf_orthogonalize_svqb(n, _panels(X), X.panel_count(), X.block_width(), drop_tol, buf.data_ptr(),
                                    C.byref(rank), _stream()))
    r = rank.value
    Q = BlockVector.__new__(BlockVector)
    Q._n, Q._ns, Q._nb, Q.device = n, r, r, X.device
    Q._panels = [buf[:n * r].view(n, r).clone()]
    return Q, r


@dataclass
class RayleighRitzResult:
    theta: np.ndarray        # ascending
    basis: BlockVector       # Y = Q V, one panel
    residuals: np.ndarray    # ||H y_j - theta_j y_j|| / ||y_j||


def rayleigh_ritz(H: SparseMatrixCRS, Q: BlockVector) -> RayleighRitzResult:
    """filter.hpp:170-211."""
    if Q.rows() != H.n:
        raise ValueError("rayleigh_ritz: row count mismatch")
    k = Q.cols()
    if Q.block_width() != k:
        raise ValueError("rayleigh_ritz: expects a single panel")
    dm = H.device_matrix(Q.device.index)
    theta = np.empty(k)
    res = np.empty(k)
    Y = BlockVector(H.n, k, k, device=Q.device)
    check(lib.cf_rayleigh_ritz(dm.handle, Q.panel(0).data_ptr(), k, ptr(theta), Y.panel(0).data_ptr(), ptr(res),
                               _stream()))
    return RayleighRitzResult(theta, Y, res)


@dataclass
class RitzPair:
    value: float = 0.0
    residual: float = 0.0
    inside_window: bool = False
    converged: bool = False


@dataclass
class SolveOptions:
    n_s: int = 32
    n_b: int = 8
    n_p: int = 500
    max_restarts: int = 20
    res_tol: float = 1e-9
    margin: float = 0.01
    seed: int = 42
    damping: Damping = Damping.jackson
    spectral_bounds: tuple[float, float] | None = None  # default: Gershgorin
    drop_tol: float = 1e-12


@dataclass
class SolveResult:
    eigenvalues: np.ndarray = field(default_factory=lambda: np.zeros(0))
    residuals: np.ndarray = field(default_factory=lambda: np.zeros(0))
    eigenvectors: BlockVector | None = None
    all_pairs: list = field(default_factory=list)
    moments: list = field(default_factory=list)  # one MomentSeries per restart
    iterations: int = 0
    converged: bool = False
    phase_ms: np.ndarray = field(default_factory=lambda: np.zeros((0, 3)))  # per restart: filter, SVQB, RR


def chebfd_solve(H: SparseMatrixCRS, window_lo: float, window_hi: float, opt: SolveOptions | None = None,
                 device: int | None = None) -> SolveResult:
    """filter.hpp:247-320: restarted apply_filter -> SVQB -> Rayleigh-Ritz until every
    Ritz value strictly inside the window has residual <= res_tol."""
    opt = SolveOptions() if opt is None else opt
    if opt.n_b == 0 or opt.n_s == 0 or opt.n_s % opt.n_b != 0:
        raise ValueError("n_b must divide n_s")
    dev = torch.cuda.current_device() if device is None else device
    dm = H.device_matrix(dev)
    o = SolveOptionsC(opt.n_s, opt.n_b, opt.n_p, opt.max_restarts, opt.res_tol, opt.margin, opt.seed,
                      opt.damping.value, 1 if opt.spectral_bounds else 0,
                      opt.spectral_bounds[0] if opt.spectral_bounds else 0.0,
                      opt.spectral_bounds[1] if opt.spectral_bounds else 0.0, opt.drop_tol)
    ns = opt.n_s
    ev, er, pv, pr = (np.zeros(ns) for _ in range(4))
    pf = np.zeros(ns, np.int32)
    vec = torch.empty(H.n * ns, dtype=torch.complex128, device=torch.device("cuda", dev))
    rows = max(opt.n_p - 2, 0) * ns
    eta = np.zeros(max(opt.max_restarts, 1) * rows, np.complex128)
    mu = np.zeros_like(eta)
    phases = np.zeros((max(opt.max_restarts, 1), 3))
    r = SolveResultC(0, 0, 0, 0, ptr(ev), ptr(er), ptr(pv), ptr(pr), ptr(pf), vec.data_ptr(), ptr(eta), ptr(mu),
                     ptr(phases))
    check(lib.cf_chebfd_solve(dm.handle, window_lo, window_hi, C.byref(o), C.byref(r), _stream()))
    out = SolveResult()
    out.iterations, out.converged = int(r.iterations), bool(r.converged)
    out.phase_ms = phases[:out.iterations].copy()
    k = int(r.n_eig)
    out.eigenvalues, out.residuals = ev[:k].copy(), er[:k].copy()
    out.all_pairs = [RitzPair(float(pv[i]), float(pr[i]), bool(pf[i] & 1), bool(pf[i] & 2))
                     for i in range(int(r.n_pairs))]
    if out.converged and k > 0:
        V = BlockVector.__new__(BlockVector)
        V._n, V._ns, V._nb, V.device = H.n, k, k, vec.device
        V._panels = [vec[:H.n * k].view(H.n, k).clone()]
        out.eigenvectors = V
    for it in range(out.iterations):
        ms = MomentSeries(opt.n_p, ns, device=vec.device)
        ms.eta.copy_(torch.from_numpy(eta[it * rows:(it + 1) * rows]))
        ms.mu.copy_(torch.from_numpy(mu[it * rows:(it + 1) * rows]))
        out.moments.append(ms)
    return out
