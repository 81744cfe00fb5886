/*
 * chebfd_oracle.h -- CPU restatement of the reference ChebFD hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This is the parity checker for the B200 product
 * (paper_1803_02156_b200/).  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load it.  The product
 * never links, loads or falls back to it.
 *
 * Every function restates one reference routine; the file:line it follows is
 * cited beside it (paths relative to the reference repo root).  Arithmetic is
 * restated operation-for-operation (std::complex<double> products expanded as
 * (ac-bd, ad+bc), scalar*complex as componentwise products, no contraction:
 * build with -ffp-contract=off), so results are bit-identical to the
 * reference built with g++ -O2/-O3 on x86-64 for finite inputs.  That claim is
 * pinned by tests/test_oracle.py against oracle/_ref (the reference headers
 * compiled unchanged) and the committed fixtures under tests/golden/.
 *
 * Complex numbers are interleaved (re, im) double pairs.  Block-vector panels
 * use the reference layout: element (i, j) of a width-nb panel at i*nb + j
 * (proj/include/chebfilter/block_vector.hpp:49-52, 81-94).
 */
#ifndef CHEBFD_ORACLE_H
#define CHEBFD_ORACLE_H
#include <stddef.h>
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

/* block_vector.hpp:17-35 */
uint64_t or_splitmix64(uint64_t x);
void or_unit_complex_gaussian(uint64_t seed, uint64_t i, uint64_t j, double* out2);
/* block_vector.hpp:57-73: fills panel-concatenated storage (n_s/nb panels of n*nb). */
int or_blockvec_random(size_t n, size_t ns, size_t nb, uint64_t seed, uint64_t row_offset, double* out);

/* sparse_matrix.hpp:181-228 (+ build_from_triplets :43-64).  Two-phase: call with
 * row_ptr == NULL to get nnz, then with arrays of n+1 / nnz / 2*nnz. */
int or_topi_generate(size_t nx, size_t ny, size_t nz, double mass, double hop, int open_boundary,
                     size_t* n_out, size_t* nnz_out, uint64_t* row_ptr, int32_t* col_idx, double* values);
/* sparse_matrix.hpp:89-107 */
int or_gershgorin_bounds(size_t n, const uint64_t* row_ptr, const int32_t* col_idx, const double* values,
                         double* lo, double* hi);
/* filter.hpp:25-32 */
int or_spectral_map(double lmin, double lmax, double margin, double* alpha, double* beta);
/* filter.hpp:39-70; damping 0 = jackson, 1 = none.  c, g have np+1 entries. */
int or_filter_coefficients(double wlo, double whi, double alpha, double beta, size_t np, int damping,
                           double* c, double* g);

/* kernels.hpp:82-101 */
int or_spmmv_shifted(size_t n, const uint64_t* row_ptr, const int32_t* col_idx, const double* values,
                     double alpha, double beta, size_t nb, const double* X, double* Y);
/* kernels.hpp:104-127 (Z may equal Y) */
int or_spmmv_shifted_two_minus(size_t n, const uint64_t* row_ptr, const int32_t* col_idx, const double* values,
                               double alpha, double beta, size_t nb, const double* X, double* Y, const double* Z);
/* kernels.hpp:133-152 */
int or_cheb_init(size_t n, const uint64_t* row_ptr, const int32_t* col_idx, const double* values, double alpha,
                 double beta, size_t nb, double* X, double* U, double* W, double g0c0, double g1c1, double g2c2);
/* kernels.hpp:160-208.  eta/mu point at the (p, moment_col_offset) slot of a MomentSeries
 * row; nb entries are accumulated with += after the 64-chunk tree reduction. */
int or_chebfd_op(size_t n, const uint64_t* row_ptr, const int32_t* col_idx, const double* values, double alpha,
                 double beta, size_t nb, const double* U, double* W, double* X, double gc, double* eta, double* mu);
/* kernels.hpp:212-254 */
int or_chebfd_op_reference(size_t n, const uint64_t* row_ptr, const int32_t* col_idx, const double* values,
                           double alpha, double beta, size_t nb, const double* U, double* W, double* X, double gc,
                           double* eta, double* mu);
/* filter.hpp:76-93.  X: n x ns, panel-concatenated (ns/nb panels).  eta, mu:
 * (np-2)*ns complex each, index (p-3)*ns + j, zero-initialised by the callee. */
int or_apply_filter(size_t n, const uint64_t* row_ptr, const int32_t* col_idx, const double* values, size_t ns,
                    size_t nb, double* X, size_t np, const double* c, const double* g, double alpha, double beta,
                    double* eta, double* mu);

/* partition.hpp:28-60.  ranges: 2*workers.  halo_in is returned flattened:
 * for each worker w, for each owner v ascending: (w, v, count, rows...) records
 * appended to `halo` (uint64).  Call with halo == NULL to size it. */
int or_sell_permutation(size_t n, const uint64_t* row_ptr, const int32_t* col_idx, const int32_t* order, int C,
                        int sigma, int32_t* perm_out, size_t* nslots);
int or_partition_rows(size_t n, const uint64_t* row_ptr, const int32_t* col_idx, size_t workers, uint64_t* ranges,
                      uint64_t* halo, size_t* halo_len);

#ifdef __cplusplus
}
#endif
#endif
