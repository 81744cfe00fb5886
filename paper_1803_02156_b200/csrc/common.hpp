// Shared host-side declarations for libchebfd_b200 (C++ host part + CUDA part).
#pragma once
#include <cstddef>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/chebfd_b200.h"

#ifdef __CUDACC__
#define CF_HD __host__ __device__
#else
#define CF_HD
#endif

namespace cfb {

// Exception types mirror the reference's (kernels.hpp:61-67, dist.hpp:102-104).
struct ProtocolError : std::logic_error {
    using std::logic_error::logic_error;
};
struct CudaError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

void set_error(const std::string& msg);
// Re-raises a status returned by one of the library's own C entries as the
// exception type it stands for (inverse of guard()).
[[noreturn]] void rethrow_status(int status);
inline void check(int status) {
    if (status != 0) rethrow_status(status);
}

// Runs f and maps exceptions onto CF_E* status codes.
template <class F>
int guard(F&& f) {
    try {
        f();
        return CF_OK;
    } catch (const ProtocolError& e) {
        set_error(e.what());
        return CF_EPROTOCOL;
    } catch (const std::invalid_argument& e) {
        set_error(e.what());
        return CF_EINVAL;
    } catch (const std::out_of_range& e) {
        set_error(e.what());
        return CF_ERANGE;
    } catch (const CudaError& e) {
        set_error(e.what());
        return CF_ECUDA;
    } catch (const std::exception& e) {
        set_error(e.what());
        return CF_ERUNTIME;
    }
}

// ---------------------------------------------------------------------------
// 4x4-blocked SELL-C-sigma ("SELL-C-sigma/B4"), host image.
//
// A piece record (16-byte aligned, <= kStageBytes) holds up to C block-rows
// of one chunk and a contiguous range of their blocks:
//   PieceHdr (16 B) | int32 perm[C] | uint16 nblk[C] (padded to 16 B)
//   | BlockMeta meta[kcnt][C] | double2 vals[nvals] | uint8 sidx[kcnt+1][C] (padded)
// Blocks of a block-row are in ascending block-column order; a block's
// nonzeros are packed row-major over its 16-bit (r*4+c) mask.  Pieces of one
// chunk are consecutive; units are consecutive chunk ranges handed out to
// CTAs dynamically.
constexpr int kBlock = 4;
constexpr int kDefaultC = 8;
constexpr std::size_t kStageBytes = 8192;

struct PieceHdr {
    uint16_t nrows;  // valid slots in the chunk
    uint16_t kcnt;   // block columns per slot in this piece (max over slots)
    uint16_t flags;  // kFirst | kLast (of the chunk)
    uint16_t C;
    uint32_t nvals;
    uint32_t chunk;
};
static_assert(sizeof(PieceHdr) == 16, "PieceHdr");
constexpr uint16_t kPieceFirst = 1, kPieceLast = 2;
// typed record (device typed stream only): one double per purely real / imaginary value
constexpr uint16_t kPieceTyped = 4;
// Block-row signatures: a chunk whose C slots are all valid and all hold the
// same multiset of block patterns is stored in canonical order (blocks sorted
// by (mask, bcol), values slot-major: slot r's values at r * kSigNnz[sig]) and
// tagged with the signature in PieceHdr.flags bits 8..15, so the kernel walks
// it with a compile-time block sequence.  sig 0 = generic.
// sig 1: Wilson-Dirac / Topi stencil, 1 on-site + 4 x/y hops + 2 z hops.
constexpr int kSigShift = 8;
constexpr int kSigTopiBlocks = 7;
constexpr uint16_t kSigTopiMasks[kSigTopiBlocks] = {0x8421u, 0x9669u, 0x9669u, 0x9669u, 0x9669u, 0xA5A5u, 0xA5A5u};
constexpr int kSigTopiNnz = 52;  // 4 + 6 * 8 values per block-row

struct BlockMeta {
    int32_t bcol;
    uint16_t mask;
    uint16_t voff;  // first value of the block, relative to the piece's vals
};
static_assert(sizeof(BlockMeta) == 8, "BlockMeta");

// Chunk staging plan (n_b = 32 whole-row panels): the distinct block columns a
// chunk reads (its blocks' columns plus its own block-rows) are staged into
// shared memory by one 1-D TMA copy per run of consecutive block columns;
// sidx[(kcnt + 1) * C] at the end of the record maps block (k, r) -- and, in
// the last row, slot r's own block-row -- to its staged index (0xFF = none).
constexpr int kMaxStage = 44;  // staged block columns per chunk (88 KB at n_b = 32)
constexpr int kMaxRuns = 31;
struct StageRun {
    int32_t bcol;  // first block column
    uint16_t len;  // block columns
    uint16_t dst;  // first staged index
};
struct StagePlan {
    uint16_t nruns;
    uint16_t nstaged;
    uint32_t pad;
    StageRun runs[kMaxRuns];
};
static_assert(sizeof(StagePlan) == 256, "StagePlan");
CF_HD inline std::size_t sidx_offset(int C, int kcnt, std::size_t nvals) {
    return 16 + 4 * static_cast<std::size_t>(C) + (2 * static_cast<std::size_t>(C) + 15) / 16 * 16 +
           8 * static_cast<std::size_t>(kcnt) * C + 16 * nvals;
}

struct PieceInfo {  // device table: where each record lives
    uint64_t offset;  // bytes
    uint32_t bytes;
    uint32_t flags;
};
static_assert(sizeof(PieceInfo) == 16, "PieceInfo");

struct SellHost {
    std::size_t n = 0, ncols = 0, nnz = 0;
    int C = kDefaultC, sigma = 0;
    std::size_t nbr = 0;          // block-rows
    std::vector<int32_t> perm;    // slot -> block-row (-1 pad), size nchunks*C
    std::vector<uint8_t> records; // all piece records
    std::vector<PieceInfo> pieces;
    std::vector<int32_t> unit_piece;  // unit u -> pieces [unit_piece[u], unit_piece[u+1])
    std::size_t nchunks = 0;
    std::size_t max_bcol = 0;     // largest block column referenced
    std::vector<StagePlan> plans; // per piece; valid for every piece iff staged
    bool staged = false;
};

std::size_t piece_bytes(int C, int kcnt, std::size_t nvals);

SellHost build_sell(std::size_t n, std::size_t ncols, const uint64_t* row_ptr, const int32_t* col_idx,
                    const double* values, const int32_t* order, int C, int sigma, std::size_t units_hint);
std::vector<int32_t> sell_permutation(std::size_t n, const uint64_t* row_ptr, const int32_t* col_idx,
                                      const int32_t* order, int C, int sigma);
void sell_to_crs(const SellHost& s, std::vector<uint64_t>& rp, std::vector<int32_t>& ci, std::vector<double>& v);

struct Crs {
    std::size_t n = 0;
    std::vector<uint64_t> row_ptr;
    std::vector<int32_t> col_idx;
    std::vector<double> values;  // interleaved
};
Crs topi_crs(std::size_t nx, std::size_t ny, std::size_t nz, double mass, double hop, bool open);
std::vector<int32_t> lattice_order(std::size_t nx, std::size_t ny, std::size_t nz, std::size_t tx, std::size_t ty,
                                   bool boundary_first = false);

unsigned host_threads();

// Columns [j0, j1) of InitSeededRandom{seed} (block_vector.hpp:68-73) as an
// n x (j1 - j0) row-major complex array (bit-identical to the reference).
void fill_random_columns(std::size_t n, std::size_t j0, std::size_t j1, uint64_t seed, double* out);

// Cyclic Jacobi eigensolver for a dense Hermitian k x k matrix (row-major,
// interleaved complex), the reference's jacobi_hermitian_eig
// (jacobi_eig.hpp:32-98): ascending values, vectors row-major with column j
// the eigenvector of values[j].
void jacobi_hermitian(std::size_t k, std::vector<double> A, double tol, std::size_t max_sweeps,
                      std::vector<double>& values, std::vector<double>& vectors);

}  // namespace cfb
