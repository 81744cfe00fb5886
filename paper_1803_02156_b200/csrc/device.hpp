// Internal declarations shared by the device translation units of
// libchebfd_b200 (chebfd_kernels.cu: the fused SpMMV family; solve.cu: the
// SVQB / Rayleigh-Ritz / restart loop of chebfd_solve).
#pragma once
#include <cuda_runtime.h>

#include <cstddef>
#include <vector>

#include "common.hpp"

struct cf_matrix_s {
    int device = 0;
    std::size_t n = 0, ncols = 0, nnz = 0, nbr = 0, rows_alloc = 0;
    int C = 0;
    uint8_t* d_records = nullptr;
    cfb::PieceInfo* d_pieces = nullptr;
    int32_t* d_units = nullptr;
    int num_units = 0;
    std::size_t record_bytes = 0, npieces = 0;
    std::vector<cfb::PieceInfo> pieces;
    double* d_partials = nullptr;  // [2][num_units][32][3]: alternating per fused step
    int part_sel = 0;
    double* d_bpart = nullptr;
    unsigned* d_counters = nullptr;
    std::size_t device_bytes = 0;
    int grid = 0;
    void* scratch = nullptr;
    std::size_t scratch_bytes = 0;
    void* wide = nullptr;  // 32-wide panel of apply_filter on narrow panels (filter_wide)
    std::size_t wide_bytes = 0;
    void* hostio = nullptr;  // device X + moments of cf_apply_filter_host
    std::size_t hostio_bytes = 0;
    // Gershgorin interval of the rows the matrix was built from
    // (sparse_matrix.hpp:89-107); chebfd_solve's default spectral bounds.
    double gersh_lo = 0.0, gersh_hi = 0.0;
    // per-piece chunk staging plans (null when some chunk has none): n_b = 32
    // panels then run the chunk-staged kernel
    cfb::StagePlan* d_plans = nullptr;
    int32_t* d_row0 = nullptr;  // first block-row per piece when consecutive, else -1
    // typed (real / imaginary) records of the staged kernel (null when not applicable)
    uint8_t* d_trecords = nullptr;
    cfb::PieceInfo* d_tpieces = nullptr;
    std::size_t typed_bytes = 0;
    std::size_t typed_pieces = 0;  // pieces stored typed in d_trecords (the rest verbatim)
    bool narrow_ok = false;        // every piece typed, one per chunk, <= kRecNarrow (narrow staged kernel)
    // per work unit the lowest / highest block-row it holds (boundary-unit detection)
    std::vector<int32_t> unit_br_lo, unit_br_hi;
    // leading work units that hold a boundary row (cf_matrix_set_boundary): the staged
    // kernel raises a step's neighbour flags once these are done (0 = unknown)
    int bnd_units = 0;
    // full records kept on the host only, when typed records run the kernels
    // (uploaded again on demand: typed knob off, see ensure_full_records)
    std::vector<uint8_t> h_records;
    // moment slots of cf_chebfd_op_host_moments: device [2][slot_cols] complex, pinned host copy
    double* d_slots = nullptr;
    double* h_slots = nullptr;
    std::size_t slot_cols = 0;
};

namespace cfb {

// Alg. 2 over device panels (filter.hpp:76-93); eta, mu: (np-2)*n_s complex.
void apply_filter_dev(cf_matrix m, double2* const* panels, std::size_t npanels, std::size_t nb, std::size_t np,
                      const double* c, const double* g, double alpha, double beta, double* eta, double* mu,
                      cudaStream_t st);
// Y = (alpha H + beta) X on one ld-wide panel (kernels.hpp:82-101).
void spmmv_dev(cf_matrix m, double alpha, double beta, const double2* X, double2* Y, std::size_t ld,
               std::size_t ncols, cudaStream_t st);

struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev);
    ~DeviceGuard();
};
void ck(cudaError_t e, const char* what);

}  // namespace cfb
