"""ctypes access to the CPU checker (TEST INFRASTRUCTURE ONLY).

* ``O``   -- oracle/liboracle.so: the C restatement of the reference path
             (oracle/chebfd_oracle.c), always available (built on demand).
* ``REF`` -- oracle/_ref/libchebref.so: the reference headers compiled unchanged
             (oracle/ref_harness.cpp), present only where it was built.
"""
from __future__ import annotations

import ctypes as C
import subprocess
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
_ORACLE = ROOT / "oracle" / "liboracle.so"
_REF = ROOT / "oracle" / "_ref" / "libchebref.so"

vp, sz, dbl, i32, u64 = C.c_void_p, C.c_size_t, C.c_double, C.c_int, C.c_uint64
szp, dblp = C.POINTER(C.c_size_t), C.POINTER(C.c_double)


def _p(a):
    return None if a is None else a.ctypes.data


def _load_oracle():
    src = ROOT / "oracle" / "chebfd_oracle.c"
    if not _ORACLE.exists() or _ORACLE.stat().st_mtime < src.stat().st_mtime:
        subprocess.run(["make", "-s", "-C", str(ROOT / "oracle"), "liboracle.so"], check=True)
    lib = C.CDLL(str(_ORACLE))
    sigs = {
        "or_blockvec_random": [sz, sz, sz, u64, u64, vp],
        "or_topi_generate": [sz, sz, sz, dbl, dbl, i32, szp, szp, vp, vp, vp],
        "or_gershgorin_bounds": [sz, vp, vp, vp, dblp, dblp],
        "or_spectral_map": [dbl, dbl, dbl, dblp, dblp],
        "or_filter_coefficients": [dbl, dbl, dbl, dbl, sz, i32, vp, vp],
        "or_spmmv_shifted": [sz, vp, vp, vp, dbl, dbl, sz, vp, vp],
        "or_spmmv_shifted_two_minus": [sz, vp, vp, vp, dbl, dbl, sz, vp, vp, vp],
        "or_cheb_init": [sz, vp, vp, vp, dbl, dbl, sz, vp, vp, vp, dbl, dbl, dbl],
        "or_chebfd_op": [sz, vp, vp, vp, dbl, dbl, sz, vp, vp, vp, dbl, vp, vp],
        "or_chebfd_op_reference": [sz, vp, vp, vp, dbl, dbl, sz, vp, vp, vp, dbl, vp, vp],
        "or_apply_filter": [sz, vp, vp, vp, sz, sz, vp, sz, vp, vp, dbl, dbl, vp, vp],
        "or_partition_rows": [sz, vp, vp, sz, vp, vp, szp],
        "or_sell_permutation": [sz, vp, vp, vp, i32, i32, vp, szp],
    }
    for k, a in sigs.items():
        f = getattr(lib, k)
        f.argtypes = a
        f.restype = i32
    return lib


O = _load_oracle()


def _load_ref():
    if not _REF.exists():
        return None
    lib = C.CDLL(str(_REF))
    lib.ref_topi.restype = vp
    lib.ref_topi.argtypes = [sz, sz, sz, dbl, dbl, i32]
    lib.ref_crs_from_arrays.restype = vp
    lib.ref_crs_from_arrays.argtypes = [sz, vp, vp, vp]
    lib.ref_random_hermitian.restype = vp
    lib.ref_random_hermitian.argtypes = [sz, u64, dbl]
    lib.ref_crs_info.argtypes = [vp, szp, szp]
    lib.ref_crs_copy.argtypes = [vp, vp, vp, vp]
    lib.ref_crs_free.argtypes = [vp]
    lib.ref_last_error.restype = C.c_char_p
    sigs = {
        "ref_gershgorin": [vp, dblp, dblp],
        "ref_dense_eigenvalues": [vp, vp],
        "ref_spectral_map": [dbl, dbl, dbl, dblp, dblp],
        "ref_filter_coefficients": [dbl, dbl, dbl, dbl, sz, i32, vp, vp],
        "ref_blockvec_random": [sz, sz, sz, u64, u64, vp],
        "ref_spmmv_shifted": [vp, dbl, dbl, sz, sz, vp, vp],
        "ref_spmmv_two_minus": [vp, dbl, dbl, sz, sz, vp, vp, vp],
        "ref_cheb_init": [vp, dbl, dbl, sz, sz, vp, vp, vp, dbl, dbl, dbl],
        "ref_chebfd_op": [vp, dbl, dbl, sz, sz, vp, vp, vp, dbl, vp, vp, i32],
        "ref_apply_filter": [vp, sz, sz, vp, sz, vp, vp, dbl, dbl, vp, vp],
        "ref_step_run": [vp, dbl],
        "ref_partition_rows": [vp, sz, vp, vp, szp],
        "ref_shard": [vp, sz, sz, szp, szp, szp, vp, vp, vp, vp, vp, szp, vp, szp],
        "ref_filter_distributed": [vp, sz, i32, sz, sz, vp, sz, vp, vp, dbl, dbl, vp, vp],
        "ref_chebfd_solve": [vp, dbl, dbl, sz, sz, sz, sz, dbl, u64, i32, dbl, dbl, vp, szp, szp,
                             C.POINTER(C.c_int)],
    }
    for k, a in sigs.items():
        f = getattr(lib, k)
        f.argtypes = a
        f.restype = i32
    lib.ref_mm_write.argtypes = [vp, C.c_char_p]
    lib.ref_mm_write.restype = i32
    lib.ref_mm_read.argtypes = [C.c_char_p, szp, C.POINTER(C.c_int)]
    lib.ref_mm_read.restype = vp
    lib.ref_bv_write.argtypes = [C.c_char_p, sz, sz, sz, u64]
    lib.ref_bv_write.restype = i32
    lib.ref_bv_read.argtypes = [C.c_char_p, szp, szp, szp, vp]
    lib.ref_bv_read.restype = i32
    lib.ref_step_state.restype = vp
    lib.ref_step_state.argtypes = [vp, sz, u64, dbl, dbl]
    lib.ref_step_free.argtypes = [vp]
    lib.ref_arithmetic_intensity.restype = dbl
    lib.ref_arithmetic_intensity.argtypes = [sz]
    lib.ref_min_traffic.argtypes = [sz, sz, dblp, dblp]
    return lib


REF = _load_ref()


class Crs:
    """Plain CRS triple used by the checker: row_ptr u64, col_idx i32, values c128."""

    def __init__(self, n, row_ptr, col_idx, values, ncols=None):
        self.n = int(n)
        self.row_ptr = np.ascontiguousarray(row_ptr, np.uint64)
        self.col_idx = np.ascontiguousarray(col_idx, np.int32)
        self.values = np.ascontiguousarray(values, np.complex128)
        self.ncols = self.n if ncols is None else ncols

    def args(self):
        return self.n, _p(self.row_ptr), _p(self.col_idx), _p(self.values)


def _chk(st, lib=None):
    if st != 0:
        raise RuntimeError(f"oracle call failed with status {st}")


# ------------------------------------------------------------- oracle ----
def topi(nx, ny, nz, mass=1.0, hop=1.0, open_=False) -> Crs:
    n, nnz = C.c_size_t(), C.c_size_t()
    _chk(O.or_topi_generate(nx, ny, nz, mass, hop, int(open_), C.byref(n), C.byref(nnz), None, None, None))
    rp = np.empty(n.value + 1, np.uint64)
    ci = np.empty(nnz.value, np.int32)
    v = np.empty(nnz.value, np.complex128)
    _chk(O.or_topi_generate(nx, ny, nz, mass, hop, int(open_), C.byref(n), C.byref(nnz), _p(rp), _p(ci), _p(v)))
    return Crs(n.value, rp, ci, v)


def blockvec_random(n, ns, nb, seed, row_offset=0):
    out = np.empty((ns // nb, n, nb), np.complex128)
    _chk(O.or_blockvec_random(n, ns, nb, seed, row_offset, _p(out)))
    return out


def gershgorin(H: Crs):
    lo, hi = C.c_double(), C.c_double()
    _chk(O.or_gershgorin_bounds(*H.args(), C.byref(lo), C.byref(hi)))
    return lo.value, hi.value


def spectral_map(lo, hi, margin=0.0):
    a, b = C.c_double(), C.c_double()
    _chk(O.or_spectral_map(lo, hi, margin, C.byref(a), C.byref(b)))
    return a.value, b.value


def coefficients(wlo, whi, alpha, beta, np_, damping=0):
    c = np.empty(np_ + 1)
    g = np.empty(np_ + 1)
    _chk(O.or_filter_coefficients(wlo, whi, alpha, beta, np_, damping, _p(c), _p(g)))
    return c, g


def spmmv(H: Crs, alpha, beta, X):
    X = np.ascontiguousarray(X, np.complex128)
    Y = np.zeros((H.n, X.shape[1]), np.complex128)
    _chk(O.or_spmmv_shifted(*H.args(), alpha, beta, X.shape[1], _p(X), _p(Y)))
    return Y


def two_minus(H: Crs, alpha, beta, X, Z):
    X = np.ascontiguousarray(X, np.complex128)
    Z = np.ascontiguousarray(Z, np.complex128)
    Y = np.zeros((H.n, X.shape[1]), np.complex128)
    _chk(O.or_spmmv_shifted_two_minus(*H.args(), alpha, beta, X.shape[1], _p(X), _p(Y), _p(Z)))
    return Y


def cheb_init(H: Crs, alpha, beta, X, g0c0, g1c1, g2c2):
    X = np.array(X, np.complex128, order="C")
    nb = X.shape[1]
    U = np.zeros_like(X)
    W = np.zeros_like(X)
    _chk(O.or_cheb_init(*H.args(), alpha, beta, nb, _p(X), _p(U), _p(W), g0c0, g1c1, g2c2))
    return X, U, W


def chebfd_op(H: Crs, alpha, beta, U, W, X, gc, unfused=False):
    """One step; returns (W, X, eta, mu) with eta/mu the nb-wide increments."""
    U = np.ascontiguousarray(U, np.complex128)
    W = np.array(W, np.complex128, order="C")
    X = np.array(X, np.complex128, order="C")
    nb = U.shape[1]
    eta = np.zeros(nb, np.complex128)
    mu = np.zeros(nb, np.complex128)
    f = O.or_chebfd_op_reference if unfused else O.or_chebfd_op
    _chk(f(*H.args(), alpha, beta, nb, _p(U), _p(W), _p(X), gc, _p(eta), _p(mu)))
    return W, X, eta, mu


def apply_filter(H: Crs, Xp, np_, c, g, alpha, beta):
    """Xp: (n_s/n_b, n, n_b) panels; returns (X, eta, mu) with eta/mu (np-2, n_s)."""
    Xp = np.array(Xp, np.complex128, order="C")
    npan, n, nb = Xp.shape
    ns = npan * nb
    eta = np.zeros((np_ - 2) * ns, np.complex128)
    mu = np.zeros((np_ - 2) * ns, np.complex128)
    _chk(O.or_apply_filter(*H.args(), ns, nb, _p(Xp), np_, _p(np.ascontiguousarray(c)),
                           _p(np.ascontiguousarray(g)), alpha, beta, _p(eta), _p(mu)))
    return Xp, eta.reshape(np_ - 2, ns), mu.reshape(np_ - 2, ns)


def partition(H: Crs, workers):
    ln = C.c_size_t()
    _chk(O.or_partition_rows(H.n, _p(H.row_ptr), _p(H.col_idx), workers, None, None, C.byref(ln)))
    ranges = np.empty(2 * workers, np.uint64)
    halo = np.empty(max(ln.value, 1), np.uint64)
    _chk(O.or_partition_rows(H.n, _p(H.row_ptr), _p(H.col_idx), workers, _p(ranges), _p(halo), C.byref(ln)))
    return ranges, halo[:ln.value]


def sell_permutation(H: Crs, order=None, C_=8, sigma=8):
    ns = C.c_size_t()
    o = None if order is None else np.ascontiguousarray(order, np.int32)
    _chk(O.or_sell_permutation(H.n, _p(H.row_ptr), _p(H.col_idx), _p(o), C_, sigma, None, C.byref(ns)))
    out = np.empty(ns.value, np.int32)
    _chk(O.or_sell_permutation(H.n, _p(H.row_ptr), _p(H.col_idx), _p(o), C_, sigma, _p(out), C.byref(ns)))
    return out


def unpack_halo(flat):
    """(w, v, count, rows...) records -> {w: {v: [rows]}}"""
    out, q = {}, 0
    flat = [int(x) for x in flat]
    while q < len(flat):
        w, v, cnt = flat[q:q + 3]
        out.setdefault(w, {})[v] = flat[q + 3:q + 3 + cnt]
        q += 3 + cnt
    return out


# ----------------------------------------------------------- reference ----
class RefMatrix:
    def __init__(self, handle):
        if not handle:
            raise RuntimeError(REF.ref_last_error().decode())
        self.h = handle

    @classmethod
    def topi(cls, nx, ny, nz, mass=1.0, hop=1.0, open_=False):
        return cls(REF.ref_topi(nx, ny, nz, mass, hop, int(open_)))

    @classmethod
    def from_crs(cls, H: Crs):
        return cls(REF.ref_crs_from_arrays(*H.args()))

    @classmethod
    def random_hermitian(cls, n, seed, scale=1.0):
        return cls(REF.ref_random_hermitian(n, seed, scale))

    def crs(self) -> Crs:
        n, nnz = C.c_size_t(), C.c_size_t()
        REF.ref_crs_info(self.h, C.byref(n), C.byref(nnz))
        rp = np.empty(n.value + 1, np.uint64)
        ci = np.empty(nnz.value, np.int32)
        v = np.empty(nnz.value, np.complex128)
        REF.ref_crs_copy(self.h, _p(rp), _p(ci), _p(v))
        return Crs(n.value, rp, ci, v)

    def __del__(self):
        if getattr(self, "h", None) and REF is not None:
            REF.ref_crs_free(self.h)
            self.h = None


def ref_chebfd_solve(H: Crs, lo, hi, ns, nb, np_, max_restarts=20, res_tol=1e-9, seed=42, bounds=None):
    """The reference's own chebfd_solve (filter.hpp:247-320) from oracle/_ref:
    (eigenvalues, iterations, converged)."""
    R = RefMatrix.from_crs(H)
    out = np.zeros(ns)
    ne, it = C.c_size_t(), C.c_size_t()
    conv = C.c_int()
    st = REF.ref_chebfd_solve(R.h, lo, hi, ns, nb, np_, max_restarts, res_tol, seed, 1 if bounds else 0,
                              bounds[0] if bounds else 0.0, bounds[1] if bounds else 0.0, _p(out), C.byref(ne),
                              C.byref(it), C.byref(conv))
    if st != 0:
        raise RuntimeError(REF.ref_last_error().decode())
    return out[:ne.value].copy(), it.value, bool(conv.value)


def ref_mm_read(path):
    """The reference's matrix_market_read: (Crs, symmetry) or raises with the line number."""
    line, sym = C.c_size_t(), C.c_int()
    h = REF.ref_mm_read(str(path).encode(), C.byref(line), C.byref(sym))
    if not h:
        err = RuntimeError(REF.ref_last_error().decode())
        err.line_number = line.value
        raise err
    R = RefMatrix(h)
    return R.crs(), sym.value


def ref_mm_write(H: Crs, path):
    R = RefMatrix.from_crs(H)
    _chk(REF.ref_mm_write(R.h, str(path).encode()))


def ref_bv_read(path):
    n, ns, nb = C.c_size_t(), C.c_size_t(), C.c_size_t()
    _chk(REF.ref_bv_read(str(path).encode(), C.byref(n), C.byref(ns), C.byref(nb), None))
    out = np.empty((ns.value // nb.value, n.value, nb.value), np.complex128)
    _chk(REF.ref_bv_read(str(path).encode(), C.byref(n), C.byref(ns), C.byref(nb), _p(out)))
    return out
