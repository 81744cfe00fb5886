"""ctypes binding of the C ABI in include/chebfd_b200.h (libchebfd_b200.so).

There is no fallback: if the library is missing or fails to load, importing the
package raises.  Status codes map onto the reference's exception types
(proj/include/chebfilter/kernels.hpp:61-67, dist.hpp:102-104)."""
from __future__ import annotations

import ctypes as C
from pathlib import Path

_LIB_PATH = Path(__file__).resolve().parent / "libchebfd_b200.so"


class ProtocolError(RuntimeError):
    """Halo-exchange protocol misuse (reference dist.hpp:102-104)."""


class CudaError(RuntimeError):
    """CUDA failure or no usable sm_100 device."""


def _load():
    if not _LIB_PATH.exists():
        raise ImportError(
            f"{_LIB_PATH} is missing: run `python -c 'import __graft_entry__ as g; g.build()'` "
            "(the B200 path has no CPU fallback)")
    return C.CDLL(str(_LIB_PATH))


lib = _load()

vp, sz, dbl, i32, u64, i32p, u64p, dblp, szp = (
    C.c_void_p, C.c_size_t, C.c_double, C.c_int, C.c_uint64, C.POINTER(C.c_int32), C.POINTER(C.c_uint64),
    C.POINTER(C.c_double), C.POINTER(C.c_size_t))

_SIGS = {
    "cf_last_error": (C.c_char_p, []),
    "cf_version": (i32, []),
    "cf_topi_generate": (i32, [sz, sz, sz, dbl, dbl, i32, szp, szp, vp, vp, vp]),
    "cf_gershgorin_bounds": (i32, [sz, vp, vp, vp, dblp, dblp]),
    "cf_spectral_map": (i32, [dbl, dbl, dbl, dblp, dblp]),
    "cf_filter_coefficients": (i32, [dbl, dbl, dbl, dbl, sz, i32, vp, vp]),
    "cf_blockvec_random": (i32, [sz, sz, sz, u64, u64, vp]),
    "cf_blockvec_random_device": (i32, [sz, sz, sz, u64, u64, vp, sz, vp]),
    "cf_partition_rows": (i32, [sz, vp, vp, sz, vp, vp, szp]),
    "cf_shard": (i32, [sz, vp, vp, vp, sz, sz, szp, szp, szp, szp, vp, vp, vp, vp, vp, szp, vp, szp]),
    "cf_topi_shard": (i32, [sz, sz, sz, dbl, dbl, i32, sz, sz, szp, szp, szp, szp, vp, vp, vp, vp, vp, szp, vp, szp]),
    "cf_sell_permutation": (i32, [sz, vp, vp, vp, i32, i32, vp, szp]),
    "cf_lattice_order": (i32, [sz, sz, sz, sz, sz, vp]),
    "cf_lattice_order_boundary_first": (i32, [sz, sz, sz, sz, sz, vp]),
    "cf_sell_layout_stats": (i32, [sz, sz, vp, vp, vp, vp, vp]),
    "cf_matrix_create_crs": (i32, [i32, sz, sz, vp, vp, vp, vp, i32, i32, C.POINTER(vp)]),
    "cf_matrix_create_topi": (i32, [i32, sz, sz, sz, dbl, dbl, i32, C.POINTER(vp)]),
    "cf_matrix_info": (i32, [vp, szp, szp, szp, szp, szp]),
    "cf_matrix_to_crs": (i32, [vp, szp, szp, vp, vp, vp]),
    "cf_matrix_staged": (i32, [vp, C.POINTER(C.c_int)]),
    "cf_matrix_narrow": (i32, [vp, C.POINTER(C.c_int)]),
    "cf_matrix_typed": (i32, [vp, C.POINTER(C.c_size_t), C.POINTER(C.c_size_t)]),
    "cf_matrix_set_boundary": (i32, [vp, sz, sz, C.POINTER(C.c_int)]),
    "cf_matrix_destroy": (i32, [vp]),
    "cf_matrix_create_topi_shard": (i32, [i32, sz, sz, sz, dbl, dbl, i32, sz, sz, vp, vp, vp, vp]),
    "cf_blockvec_create": (i32, [i32, sz, sz, sz, vp]),
    "cf_blockvec_destroy": (i32, [vp]),
    "cf_blockvec_shape": (i32, [vp, vp, vp, vp, vp]),
    "cf_blockvec_panel": (i32, [vp, sz, vp]),
    "cf_blockvec_upload": (i32, [vp, vp]),
    "cf_blockvec_download": (i32, [vp, vp]),
    "cf_panel_swap": (i32, [vp, sz, vp, sz]),
    "cf_device_count": (i32, [C.POINTER(C.c_int)]),
    "cf_tuning": (i32, [C.c_char_p, i32]),
    "cf_current_device": (i32, [C.POINTER(i32)]),
    "cf_memcpy_async": (i32, [vp, vp, sz, vp]),
    "cf_dev_alloc": (i32, [i32, sz, C.POINTER(vp)]),
    "cf_dev_free": (i32, [vp]),
    "cf_memcpy": (i32, [vp, vp, sz, i32]),
    "cf_memset_zero": (i32, [vp, sz]),
    "cf_synchronize": (i32, []),
    "cf_spmmv_shifted": (i32, [vp, dbl, dbl, vp, vp, sz, sz, vp]),
    "cf_spmmv_shifted_two_minus": (i32, [vp, dbl, dbl, vp, vp, vp, sz, sz, vp]),
    "cf_cheb_init": (i32, [vp, dbl, dbl, vp, vp, vp, sz, sz, dbl, dbl, dbl, vp]),
    "cf_cheb_init_tail": (i32, [vp, dbl, dbl, vp, vp, vp, sz, sz, dbl, dbl, dbl, vp]),
    "cf_chebfd_op": (i32, [vp, dbl, dbl, vp, vp, vp, sz, sz, dbl, vp, vp, vp]),
    "cf_chebfd_op_host_moments": (i32, [vp, dbl, dbl, vp, vp, vp, sz, sz, dbl, vp, vp, vp]),
    "cf_spmmv_shifted_mirror": (i32, [vp, dbl, dbl, vp, vp, sz, sz, vp, sz, vp]),
    "cf_cheb_init_tail_mirror": (i32, [vp, dbl, dbl, vp, vp, vp, sz, sz, dbl, dbl, dbl, vp, sz, vp]),
    "cf_chebfd_op_mirror": (i32, [vp, dbl, dbl, vp, vp, vp, sz, sz, dbl, vp, vp, vp, sz, vp]),
    "cf_ipc_get_handle": (i32, [vp, vp]),
    "cf_ipc_open_handle": (i32, [i32, vp, C.POINTER(vp)]),
    "cf_ipc_close": (i32, [vp]),
    "cf_enable_peer_access": (i32, [i32, i32]),
    "cf_apply_filter": (i32, [vp, vp, sz, sz, sz, vp, vp, dbl, dbl, vp, vp, vp]),
    "cf_apply_filter_host": (i32, [vp, vp, sz, sz, sz, vp, vp, dbl, dbl, vp, vp]),
    "cf_filter_distributed": (i32, [vp, sz, sz, sz, sz, vp, vp, dbl, dbl, i32, vp, vp]),
    "cf_flag_signal": (i32, [vp, C.c_uint64, vp]),
    "cf_flag_wait": (i32, [vp, C.c_uint64, vp]),
    "cf_filter_distributed_host": (i32, [vp, sz, sz, sz, sz, vp, vp, dbl, dbl, i32, vp, vp]),
    "cf_filter_distributed_timeline": (i32, [vp, sz, sz, sz, sz, vp, vp, dbl, dbl, i32, i32, vp, vp, vp, sz, vp]),
    "cf_degree_schedule": (i32, [sz, vp, vp, sz, vp, vp, vp, vp, vp, vp]),
    "cf_chebfd_step_mirror": (i32, [vp, i32, dbl, dbl, vp, vp, vp, sz, sz, dbl, dbl, dbl, vp, vp, vp, sz, vp]),
    "cf_chebfd_step_signal": (i32, [vp, i32, dbl, dbl, vp, vp, vp, sz, sz, dbl, dbl, dbl, vp, vp, vp, sz, vp, sz,
                                    C.c_uint64, vp, C.POINTER(C.c_int)]),
    "cf_jacobi_hermitian_eig": (i32, [sz, vp, dbl, sz, vp, vp]),
    "cf_matrix_market_read": (i32, [C.c_char_p, szp, szp, C.POINTER(C.c_int), vp, vp, vp]),
    "cf_matrix_market_error_line": (sz, []),
    "cf_matrix_market_write": (i32, [C.c_char_p, sz, vp, vp, vp, i32]),
    "cf_blockvec_write": (i32, [C.c_char_p, sz, sz, sz, vp]),
    "cf_blockvec_read": (i32, [C.c_char_p, szp, szp, szp, vp]),
    "cf_gram": (i32, [sz, vp, sz, sz, vp, sz, sz, vp, vp]),
    "cf_stream_bench": (i32, [i32, sz, i32, sz, dblp]),
    "cf_rotate": (i32, [sz, vp, sz, sz, vp, sz, vp, sz, vp]),
    "cf_residual_sums": (i32, [sz, vp, sz, vp, sz, sz, vp, vp, vp]),
    "cf_orthogonalize_svqb": (i32, [sz, vp, sz, sz, dbl, vp, szp, vp]),
    "cf_rayleigh_ritz": (i32, [vp, vp, sz, vp, vp, vp, vp]),
    "cf_chebfd_solve": (i32, [vp, dbl, dbl, vp, vp, vp]),
}
for _name, (_res, _args) in _SIGS.items():
    _f = getattr(lib, _name)
    _f.restype = _res
    _f.argtypes = _args

EXPORTED = tuple(_SIGS)


def check(status: int) -> None:
    if status == 0:
        return
    msg = (lib.cf_last_error() or b"").decode(errors="replace")
    if status == 1:
        raise ValueError(msg)          # std::invalid_argument
    if status == 2:
        raise IndexError(msg)          # std::out_of_range
    if status == 4:
        raise ProtocolError(msg)
    if status == 5:
        raise CudaError(msg)
    raise RuntimeError(msg)            # std::runtime_error


def ptr(a) -> int | None:
    """Address of a numpy array or torch tensor (None for None)."""
    if a is None:
        return None
    if hasattr(a, "data_ptr"):
        return a.data_ptr()
    return a.ctypes.data
