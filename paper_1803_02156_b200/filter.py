"""Filter coefficients and the blocked filter application (Alg. 2).

Mirrors proj/include/chebfilter/filter.hpp: Damping/FilterCoefficients :11-21,
spectral_map :25-32, filter_coefficients :39-70, apply_filter :76-93.  The
coefficients are computed by the library's host code with the reference's
libm sequence (bit-identical); apply_filter runs the whole per-panel degree
loop inside libchebfd_b200 (cheb_init + (np-2) fused steps per panel on the
device, moments accumulated in device memory).
"""
from __future__ import annotations

import ctypes as C
import enum
from dataclasses import dataclass, field

import numpy as np
import torch

from ._lib import check, lib, ptr
from .blockvec import BlockVector
from .kernels import MomentSeries, ShiftScale, TrafficCounter, _stream
from .sparse import SparseMatrixCRS


class Damping(enum.Enum):
    jackson = 0
    none = 1


@dataclass
class FilterCoefficients:
    np: int = 0
    c: np.ndarray = field(default_factory=lambda: np.zeros(0))
    g: np.ndarray = field(default_factory=lambda: np.zeros(0))
    window_lo: float = 0.0
    window_hi: float = 0.0
    map: ShiftScale = field(default_factory=ShiftScale)


def spectral_map(lambda_min: float, lambda_max: float, margin: float = 0.0) -> ShiftScale:
    a, b = C.c_double(), C.c_double()
    check(lib.cf_spectral_map(lambda_min, lambda_max, margin, C.byref(a), C.byref(b)))
    return ShiftScale(a.value, b.value)


def filter_coefficients(window_lo: float, window_hi: float, map: ShiftScale, np_: int,
                        damping: Damping = Damping.jackson) -> FilterCoefficients:
    if np_ < 2:
        raise ValueError("polynomial degree must be >= 2")
    c = np.empty(np_ + 1)
    g = np.empty(np_ + 1)
    check(lib.cf_filter_coefficients(window_lo, window_hi, map.alpha, map.beta, np_, damping.value, ptr(c), ptr(g)))
    return FilterCoefficients(np_, c, g, window_lo, window_hi, ShiftScale(map.alpha, map.beta))


def apply_filter(H: SparseMatrixCRS, X: BlockVector, fc: FilterCoefficients,
                 tc: TrafficCounter | None = None) -> MomentSeries:
    """filter.hpp:76-93 on device-resident X; returns device-resident moments."""
    if X.rows() != H.n:
        raise ValueError("apply_filter: row count mismatch")
    if fc.np < 2:
        raise ValueError("apply_filter: coefficients cover degrees < 2")
    if not X.device.type == "cuda":
        raise RuntimeError("libchebfd_b200 operates on CUDA tensors only (no CPU path)")
    nb = X.block_width()
    mom = MomentSeries(fc.np, X.cols(), device=X.device)
    panels = (C.c_void_p * X.panel_count())(*[X.panel(b).data_ptr() for b in range(X.panel_count())])
    dm = H.device_matrix(X.device.index)
    check(lib.cf_apply_filter(dm.handle, panels, X.panel_count(), nb, fc.np, ptr(fc.c), ptr(fc.g), fc.map.alpha,
                              fc.map.beta, mom.eta.data_ptr(), mom.mu.data_ptr(), _stream()))
    if tc is not None:
        npan = X.panel_count()
        tc.matrix_sweeps += npan * (2 + (fc.np - 2))
        tc.panel_reads += npan * (7 + 3 * (fc.np - 2))
        tc.panel_writes += npan * (3 + 2 * (fc.np - 2))
    return mom


def apply_filter_host(H: SparseMatrixCRS, X_panels, fc: FilterCoefficients, device: int = 0):
    """The end-to-end entry for a CPU caller: host X (n_s/n_b, n, n_b) in/out,
    host moments out; H2D, the device filter and D2H all inside one C-ABI call.
    The panels are host-staged: two device panel slots, panel b+1 copied in and
    b-1 copied out while b filters, so X may exceed device memory (cfg3 on one
    GPU).  X_panels is a numpy array or a CPU torch tensor; a pinned tensor
    (``pin_memory()``) lets the copies overlap the filter."""
    if isinstance(X_panels, torch.Tensor):
        if X_panels.device.type != "cpu" or X_panels.dtype != torch.complex128 or not X_panels.is_contiguous():
            raise ValueError("apply_filter_host: X must be a contiguous complex128 CPU tensor")
        npan, n, nb = X_panels.shape
        xp = X_panels.data_ptr()
    else:
        X_panels = np.ascontiguousarray(X_panels, np.complex128)
        npan, n, nb = X_panels.shape
        xp = ptr(X_panels)
    if n != H.n:
        raise ValueError("apply_filter: row count mismatch")
    rows = fc.np - 2
    eta = np.zeros(rows * npan * nb, np.complex128)
    mu = np.zeros(rows * npan * nb, np.complex128)
    dm = H.device_matrix(device)
    check(lib.cf_apply_filter_host(dm.handle, xp, npan * nb, nb, fc.np, ptr(fc.c), ptr(fc.g),
                                   fc.map.alpha, fc.map.beta, ptr(eta), ptr(mu)))
    return X_panels, eta, mu
