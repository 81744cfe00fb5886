"""B200-native Chebyshev filter diagonalization hot path (arXiv 1803.02156).

Drop-in for the reference's operator API (proj/include/chebfilter/*.hpp):
the same names, argument meaning and error behaviour, executed by the
sm_100a kernels of libchebfd_b200.so (C ABI in include/chebfd_b200.h).
"""
from ._lib import CudaError, ProtocolError, lib  # noqa: F401  (loads the library; raises if absent)
from .blockvec import (BlockVector, InitConstant, InitSeededRandom, InitZero, SubblockView,  # noqa: F401
                       block_vector_read, block_vector_write, seeded_random_host, swap_blocks)
from .filter import (Damping, FilterCoefficients, apply_filter, apply_filter_host, filter_coefficients,  # noqa: F401
                     spectral_map)
from .kernels import (MomentSeries, ShiftScale, TrafficCounter, cheb_init, cheb_init_tail, chebfd_op,  # noqa: F401
                      spmmv_shifted, spmmv_shifted_two_minus)
from .sparse import (Boundary, DeviceMatrix, LatticeSpec, MatrixMarketError, SparseMatrixCRS, Symmetry,  # noqa: F401
                     Triplet, matrix_market_read, matrix_market_write,
                     build_from_triplets, diagonal_matrix, from_dense, gershgorin_bounds, hermiticity_defect,
                     sell_permutation, to_dense, topi_generate)
from .solve import (EigenDecomposition, RayleighRitzResult, RitzPair, SolveOptions, SolveResult,  # noqa: F401
                    chebfd_solve, gram_matrix, jacobi_hermitian_eig, max_gram_defect, orthogonalize_svqb,
                    rayleigh_ritz)
from .perf_model import (KernelGeometry, RooflinePoint, StreamKind, arithmetic_intensity, flop_count,  # noqa: F401
                         min_traffic_volume, roofline_limit, slow_memory_amortization, stream_bench,
                         stream_bytes_per_element)
