"""The hot-path operators with the reference's signatures, run on the GPU.

Mirrors proj/include/chebfilter/kernels.hpp: ShiftScale :11-14, MomentSeries
:18-40, TrafficCounter :43-57, spmmv_shifted :82-101,
spmmv_shifted_two_minus :104-127, cheb_init :133-152, chebfd_op :160-208.
Each call validates like the reference (:61-67, :163-169) and launches the
sm_100a kernels of libchebfd_b200.so on the current torch stream.  There is no
CPU path: non-CUDA operands raise.
"""
from __future__ import annotations

import ctypes as C

from dataclasses import dataclass

import numpy as np
import torch

from ._lib import check, lib, ptr
from .blockvec import SubblockView
from .sparse import SparseMatrixCRS


@dataclass
class ShiftScale:
    alpha: float = 1.0
    beta: float = 0.0


class MomentSeries:
    """eta_p[j], mu_p[j] for p = 3..degree_max, stored [(p-3)*n_s + j] (device)."""

    def __init__(self, np_: int = 2, ns: int = 0, device=None):
        self.degree_max, self.columns = int(np_), int(ns)
        rows = np_ - 2 if np_ >= 3 else 0
        dev = device if device is not None else (
            torch.device("cuda", torch.cuda.current_device()) if torch.cuda.is_available() else "cpu")
        self.eta = torch.zeros(rows * ns, dtype=torch.complex128, device=dev)
        self.mu = torch.zeros(rows * ns, dtype=torch.complex128, device=dev)

    def index(self, p: int, j: int) -> int:
        if p < 3 or p > self.degree_max or j >= self.columns or j < 0:
            raise IndexError("moment index out of range")
        return (p - 3) * self.columns + j

    def eta_at(self, p: int, j: int) -> complex:
        return complex(self.eta[self.index(p, j)].item())

    def mu_at(self, p: int, j: int) -> complex:
        return complex(self.mu[self.index(p, j)].item())


@dataclass
class TrafficCounter:
    panel_reads: int = 0
    panel_writes: int = 0
    matrix_sweeps: int = 0

    def read_bytes(self, n, n_b, nnz, entry_bytes=20, vec_elem_bytes=16) -> float:
        return float(self.panel_reads) * n * n_b * vec_elem_bytes + float(self.matrix_sweeps) * nnz * entry_bytes

    def write_bytes(self, n, n_b, vec_elem_bytes=16) -> float:
        return float(self.panel_writes) * n * n_b * vec_elem_bytes


def _stream():
    return torch.cuda.current_stream().cuda_stream


def _dev_tensor(v: SubblockView) -> torch.Tensor:
    t = v.data()
    if not t.is_cuda:
        raise RuntimeError("libchebfd_b200 operates on CUDA tensors only (no CPU path)")
    if not t.is_contiguous() or t.dtype != torch.complex128:
        raise ValueError("panels must be contiguous complex128")
    return t


def _check_spmmv_shapes(H: SparseMatrixCRS, X: SubblockView, Y: SubblockView) -> None:
    # kernels.hpp:61-67
    if X.width() != Y.width():
        raise ValueError("spmmv: block width mismatch")
    if Y.rows() < H.n:
        raise ValueError("spmmv: output rows must cover matrix rows")
    if X.rows() < H.ncols:
        raise ValueError("spmmv: input rows must cover matrix rows")
    if X.data().data_ptr() == Y.data().data_ptr():
        raise ValueError("spmmv: X and Y must not alias")


def _handle(H: SparseMatrixCRS, t: torch.Tensor):
    return H.device_matrix(t.device.index).handle


class _Mirror(C.Structure):
    _fields_ = [("row_begin", C.c_uint64), ("row_end", C.c_uint64), ("dst", C.c_void_p)]


def _mirror_arg(mirror):
    """[(row_begin, row_end, dst_ptr)] -> (cf_mirror array, count) for the *_mirror entries."""
    runs = list(mirror or [])
    arr = (_Mirror * max(len(runs), 1))(*[_Mirror(int(a), int(b), int(d)) for a, b, d in runs])
    return arr, len(runs)


def spmmv_shifted(H: SparseMatrixCRS, s: ShiftScale, X: SubblockView, Y: SubblockView, mirror=None) -> None:
    """kernels.hpp:82-101.  ``mirror``: output rows also stored into peer halo slots
    (fused halo exchange, include/chebfd_b200.h cf_mirror)."""
    _check_spmmv_shapes(H, X, Y)
    x, y = _dev_tensor(X), _dev_tensor(Y)
    if mirror:
        arr, n = _mirror_arg(mirror)
        check(lib.cf_spmmv_shifted_mirror(_handle(H, x), s.alpha, s.beta, x.data_ptr(), y.data_ptr(), X.width(),
                                          X.width(), arr, n, _stream()))
        return
    check(lib.cf_spmmv_shifted(_handle(H, x), s.alpha, s.beta, x.data_ptr(), y.data_ptr(), X.width(), X.width(),
                               _stream()))


def spmmv_shifted_two_minus(H: SparseMatrixCRS, s: ShiftScale, X: SubblockView, Y: SubblockView,
                            Z: SubblockView) -> None:
    _check_spmmv_shapes(H, X, Y)
    if Z.width() != Y.width() or Z.rows() < H.n:
        raise ValueError("spmmv: Z shape mismatch")
    if X.data().data_ptr() == Z.data().data_ptr():
        raise ValueError("spmmv: X and Z must not alias")
    x, y, z = _dev_tensor(X), _dev_tensor(Y), _dev_tensor(Z)
    check(lib.cf_spmmv_shifted_two_minus(_handle(H, x), s.alpha, s.beta, x.data_ptr(), y.data_ptr(), z.data_ptr(),
                                         X.width(), X.width(), _stream()))


def cheb_init(H: SparseMatrixCRS, s: ShiftScale, X: SubblockView, U: SubblockView, W: SubblockView,
              g0c0: float, g1c1: float, g2c2: float, tc: TrafficCounter | None = None) -> None:
    _check_spmmv_shapes(H, X, U)
    _check_spmmv_shapes(H, U, W)
    x, u, w = _dev_tensor(X), _dev_tensor(U), _dev_tensor(W)
    check(lib.cf_cheb_init(_handle(H, x), s.alpha, s.beta, x.data_ptr(), u.data_ptr(), w.data_ptr(), X.width(),
                           X.width(), g0c0, g1c1, g2c2, _stream()))
    if tc is not None:  # kernels.hpp:147-151
        tc.matrix_sweeps += 2
        tc.panel_reads += 2 + 2 + 3
        tc.panel_writes += 1 + 1 + 1


def chebfd_op(H: SparseMatrixCRS, s: ShiftScale, U: SubblockView, W: SubblockView, X: SubblockView, p: int,
              gc: float, out: MomentSeries, moment_col_offset: int = 0, tc: TrafficCounter | None = None,
              mirror=None) -> None:
    _check_spmmv_shapes(H, U, W)
    if X.width() != U.width() or X.rows() < H.n:
        raise ValueError("chebfd_op: X shape mismatch")
    if p < 3 or p > out.degree_max:
        raise ValueError("chebfd_op: degree out of range")
    nb = U.width()
    if moment_col_offset + nb > out.columns:
        raise ValueError("chebfd_op: moment column range out of range")
    u, w, x = _dev_tensor(U), _dev_tensor(W), _dev_tensor(X)
    slot = out.index(p, moment_col_offset)
    eta = out.eta[slot:slot + nb]
    mu = out.mu[slot:slot + nb]
    if eta.device != u.device:
        raise ValueError("chebfd_op: moments live on another device")
    if mirror:
        arr, n = _mirror_arg(mirror)
        check(lib.cf_chebfd_op_mirror(_handle(H, u), s.alpha, s.beta, u.data_ptr(), w.data_ptr(), x.data_ptr(), nb,
                                      nb, gc, eta.data_ptr(), mu.data_ptr(), arr, n, _stream()))
    else:
        check(lib.cf_chebfd_op(_handle(H, u), s.alpha, s.beta, u.data_ptr(), w.data_ptr(), x.data_ptr(), nb, nb,
                               gc, eta.data_ptr(), mu.data_ptr(), _stream()))
    if tc is not None:  # kernels.hpp:203-207
        tc.matrix_sweeps += 1
        tc.panel_reads += 3
        tc.panel_writes += 2


def degree_schedule(fc) -> list:
    """apply_filter's degree loop as grouped steps (cf_degree_schedule): tuples
    (degree, kind, gw, gu, gc), kind 0 plain chebfd_op, 1 no X update, 2 / 3 the
    X update for the last two / three degrees."""
    cnt = C.c_size_t()
    check(lib.cf_degree_schedule(fc.np, ptr(fc.c), ptr(fc.g), 0, C.byref(cnt), None, None, None, None, None))
    k = cnt.value
    deg = np.zeros(k, np.uint64)
    kind = np.zeros(k, np.int32)
    gw, gu, gc = np.zeros(k), np.zeros(k), np.zeros(k)
    check(lib.cf_degree_schedule(fc.np, ptr(fc.c), ptr(fc.g), k, C.byref(cnt), ptr(deg), ptr(kind), ptr(gw), ptr(gu),
                                 ptr(gc)))
    return [(int(deg[i]), int(kind[i]), float(gw[i]), float(gu[i]), float(gc[i])) for i in range(k)]


def chebfd_step(H: SparseMatrixCRS, s: ShiftScale, U: SubblockView, W: SubblockView, X: SubblockView, step,
                out: MomentSeries, moment_col_offset: int = 0, mirror=None, signal=None) -> bool:
    """One step of degree_schedule(): chebfd_op (kernels.hpp:160-208) with the X
    update deferred / grouped; W, moments and mirrored rows as chebfd_op.
    signal = (flag pointers, value): raise value in the neighbours' step flags once
    this step's boundary rows are stored and its halo rows read (cf_chebfd_step_signal);
    returns True when the kernel raised them itself, before its interior finished."""
    p, kind, gw, gu, gc = step
    _check_spmmv_shapes(H, U, W)
    if X.width() != U.width() or X.rows() < H.n:
        raise ValueError("chebfd_op: X shape mismatch")
    if p < 3 or p > out.degree_max:
        raise ValueError("chebfd_op: degree out of range")
    nb = U.width()
    if moment_col_offset + nb > out.columns:
        raise ValueError("chebfd_op: moment column range out of range")
    u, w, x = _dev_tensor(U), _dev_tensor(W), _dev_tensor(X)
    slot = out.index(p, moment_col_offset)
    eta = out.eta[slot:slot + nb]
    mu = out.mu[slot:slot + nb]
    arr, n = _mirror_arg(mirror) if mirror else (None, 0)
    if signal is not None:
        flags, value = signal
        fl = (C.c_void_p * max(len(flags), 1))(*flags)
        ik = C.c_int()
        check(lib.cf_chebfd_step_signal(_handle(H, u), kind, s.alpha, s.beta, u.data_ptr(), w.data_ptr(),
                                        x.data_ptr(), nb, nb, gw, gu, gc, eta.data_ptr(), mu.data_ptr(), arr, n, fl,
                                        len(flags), int(value), _stream(), C.byref(ik)))
        return bool(ik.value)
    check(lib.cf_chebfd_step_mirror(_handle(H, u), kind, s.alpha, s.beta, u.data_ptr(), w.data_ptr(), x.data_ptr(),
                                    nb, nb, gw, gu, gc, eta.data_ptr(), mu.data_ptr(), arr, n, _stream()))
    return False


def cheb_init_tail(H: SparseMatrixCRS, s: ShiftScale, X: SubblockView, U: SubblockView, W: SubblockView,
                   g0c0: float, g1c1: float, g2c2: float, mirror=None) -> None:
    """Second half of cheb_init as the distributed init runs it, after the U halo
    exchange (dist.hpp:257-262): W = 2(aH+b)U - X and X = g0c0 X + g1c1 U + g2c2 W,
    fused in one sweep."""
    _check_spmmv_shapes(H, U, W)
    x, u, w = _dev_tensor(X), _dev_tensor(U), _dev_tensor(W)
    if mirror:
        arr, n = _mirror_arg(mirror)
        check(lib.cf_cheb_init_tail_mirror(_handle(H, u), s.alpha, s.beta, x.data_ptr(), u.data_ptr(), w.data_ptr(),
                                           U.width(), U.width(), g0c0, g1c1, g2c2, arr, n, _stream()))
        return
    check(lib.cf_cheb_init_tail(_handle(H, u), s.alpha, s.beta, x.data_ptr(), u.data_ptr(), w.data_ptr(), U.width(),
                                U.width(), g0c0, g1c1, g2c2, _stream()))
