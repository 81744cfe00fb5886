// Device half of libchebfd_b200: the fused Chebyshev SpMMV family on
// 4x4-blocked SELL-C-sigma, written for sm_100a.  Three kernels:
//
// * sell_b4_staged_kernel (whole-row n_b = 32 panels of matrices with chunk
//   staging plans -- every BASELINE configuration): one CTA per SM, a producer
//   warp claims work units (consecutive chunk ranges) with an atomic ticket and
//   stages each chunk's piece record plus its distinct U block columns (one 1-D
//   TMA bulk copy per run of consecutive block columns) into a 2-stage shared
//   ring; 8 consumer warps, one block-row each, walk the chunk out of shared
//   memory with W / X prefetched into registers one chunk ahead.
// * sell_b4_narrow_kernel (whole-row n_b = 2 / 4 / 8 / 12 / 16 panels of matrices whose
//   chunks are single typed records with plans): the same split, a stage holding
//   2 or 4 chunks, one 8- or 16-lane group of each consumer warp per chunk.
// * sell_b4_kernel (other widths, column slices, matrices without plans): two
//   CTAs x 8 warps per SM, records in a 6-stage TMA ring filled by lane 0 of
//   warp 0, U rows gathered per block with 128-bit L1-allocating loads.
//
// In all, a lane owns one panel column, four row accumulators stay in
// registers, the epilogue fuses the mode's vector update (reference
// kernels.hpp:82-208) and, for the Chebyshev step, the per-column moments,
// reduced per unit in a fixed order (deterministic regardless of which CTA ran
// the unit) and summed over units by reduce_moments in a fixed order.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <map>
#include <numeric>
#include <type_traits>
#include <atomic>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "device.hpp"

namespace cfb {

constexpr int kNW = 8;       // consumer warps per CTA
constexpr int kNS = 6;       // stages in the shared-memory ring
constexpr int kC = kDefaultC;  // block-rows per chunk the kernels are built for
static_assert(kC == 8, "kernel mapping assumes C == 8");

// Kernel modes: the reference's four operators, plus the steps of a degree
// group in apply_filter (X updated every second or third step, see filter_panel):
// M_CHEB_NOX = chebfd_op without the X update, M_CHEB_X2 = chebfd_op with
// x += gu*u + gc*w_new (u = the previous step's w_new), M_CHEB_X3 = chebfd_op
// with x += gw*w_old + gu*u + gc*w_new (w_old = the step before's w_new).
enum Mode { M_SHIFT = 0, M_TWO_MINUS = 1, M_INIT = 2, M_CHEB = 3, M_CHEB_NOX = 4, M_CHEB_X2 = 5, M_CHEB_X3 = 6 };
template <int MODE>
struct ModeT {
    static constexpr bool cheb =
        MODE == M_CHEB || MODE == M_CHEB_NOX || MODE == M_CHEB_X2 || MODE == M_CHEB_X3;  // W old + moments
    static constexpr bool reads_x = MODE == M_CHEB || MODE == M_INIT || MODE == M_CHEB_X2 || MODE == M_CHEB_X3;
    static constexpr bool reads_z = MODE == M_TWO_MINUS;
};
constexpr int kInfoUnitLast = 1, kInfoTerm = 2;

constexpr int kMaxMirror = 4;
struct MirrorRun {
    long long r0, r1;
    double2* dst;
};

struct KParams {
    const uint8_t* records;
    const PieceInfo* pieces;
    const int32_t* unit_piece;
    int num_units;
    long long n;  // rows whose outputs are written
    const double2* U;
    double2* W;
    double2* X;
    const double2* Z;
    long long ld;
    long long urows;  // rows of U addressable by block columns (matrix ncols)
    int ncols;
    double alpha, beta, gc, g0, g1, g2, gu, gw;
    // L2 prefetch of epilogue rows by the staged kernel's producer: piece_row0[p] =
    // first block-row of piece p when its C block-rows are consecutive (else -1);
    // wpf = pieces ahead (low 4 bits; 0 = off), bit 4 = X rows too
    const int32_t* piece_row0;
    int wpf;
    // typed records (staged kernel): every value of a Topi signature chunk is
    // purely real or purely imaginary and stored as one double; see build_typed_records()
    int typed;
    double* partials;  // [num_units][32][3]
    unsigned* counters;
    // halo mirror (fused exchange): output rows [r0, r1) are also stored to
    // dst + (row - r0) * ld, e.g. a neighbour's halo slots in peer memory
    MirrorRun mir[kMaxMirror];
    int nmir;
    // knock-out bits for bound-finding experiments only (cf_tuning("ko"), default 0;
    // results are wrong when set): 1 no W/X row loads, 2 consumers skip the U
    // barrier (unsafe: use with 16), 4 no block walk, 8 no epilogue stores, 16
    // producer stages no U runs, 32 skips runs 1 and 3 (16 of 42 block columns).
    // Order-only A/B bits (results unchanged): 64 register-gather in-order ring
    // refill, 256 narrow kernel fetches the next stage before the epilogue, 512
    // staged kernel fetches the next chunk after the epilogue
    int ko;
    // early step flags (cf_chebfd_step_signal): once every warp finished the leading
    // nbnd work units (a slab's boundary planes: its halo reads and mirrored stores),
    // sig_val is stored with release semantics at system scope to each sig[i]
    int nbnd, nsig;
    unsigned long long sig_val;
    unsigned long long* sig[2];
    int gpf;  // register-gather kernel, generic blocks: L2 prefetch distance in blocks (0 = off)
};

// Store of an output (W) row; rows a neighbour holds as halo also go to the
// mirror destination (peer memory over NVLink for a remote shard), so the halo
// exchange rides along with the kernel's own stores.
// `mir`: the caller's block-row overlaps a mirror run (block_mirrored); only then
// are the runs scanned, so unmirrored rows pay one predicate.
__device__ __forceinline__ void st_out(const KParams& P, long long row, int col, double2 v, bool mir) {
    __stcs(P.W + row * P.ld + col, v);
    if (mir) {
#pragma unroll
        for (int q = 0; q < kMaxMirror; ++q)
            if (q < P.nmir && row >= P.mir[q].r0 && row < P.mir[q].r1) __stcs(P.mir[q].dst + (row - P.mir[q].r0) * P.ld + col, v);
    }
}
__device__ __forceinline__ bool block_mirrored(const KParams& P, int br) {
    if (P.nmir == 0 || br < 0) return false;
    bool hit = false;
#pragma unroll
    for (int q = 0; q < kMaxMirror; ++q)
        hit |= q < P.nmir && 4LL * br + 3 >= P.mir[q].r0 && 4LL * br < P.mir[q].r1;
    return hit;
}

// ------------------------------------------------------------ PTX glue ---
__device__ __forceinline__ unsigned smem_u32(const void* p) {
    return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
// Non-blocking: has the phase with this parity completed?
__device__ __forceinline__ bool mbar_test(uint64_t* bar, unsigned parity) {
    unsigned ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    return ok != 0;
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
// Same with an L2 eviction-priority policy (createpolicy): streams that are read
// once per step (W, X, matrix records) go evict_first so U stays L2-resident.
__device__ __forceinline__ uint64_t policy_evict_first() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ void bulk_g2s_hint(void* dst, const void* src, unsigned bytes, uint64_t* bar,
                                              uint64_t pol) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], "
        "%4;" ::"r"(smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
        : "memory");
}
__device__ __forceinline__ void bulk_prefetch_l2(const void* p, unsigned bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}
__device__ __forceinline__ double2 ld_stream(const double2* p) { return __ldcs(p); }
__device__ __forceinline__ void st_stream(double2* p, double2 v) { __stcs(p, v); }
__device__ __forceinline__ double2 ld_gather(const double2* p) { return __ldg(p); }

// acc += a * v (complex, FMA-contracted)
__device__ __forceinline__ void cfma(double2& acc, double2 a, double2 v) {
    acc.x = fma(a.x, v.x, acc.x);
    acc.x = fma(-a.y, v.y, acc.x);
    acc.y = fma(a.x, v.y, acc.y);
    acc.y = fma(a.y, v.x, acc.y);
}


// U rows of one block column: base + (4*bcol + c) rows, only columns present in the mask.
__device__ __forceinline__ void load_block(double2 (&v)[4], const BlockMeta& m, const char* ubase, long long ld16,
                                           bool active) {
    const unsigned cm = (m.mask | m.mask >> 4 | m.mask >> 8 | m.mask >> 12) & 0xFu;
    const char* p = ubase + static_cast<long long>(m.bcol) * (4 * ld16);
#pragma unroll
    for (int c = 0; c < 4; ++c)
        v[c] = (active && (cm >> c & 1u)) ? ld_gather(reinterpret_cast<const double2*>(p + c * ld16))
                                          : make_double2(0.0, 0.0);
}

// Nonzeros of a block with a compile-time pattern: exactly nnz x (1 LDS.128 + 4 DFMA).
template <unsigned MASK>
__device__ __forceinline__ void apply_fixed(double2 (&acc)[4], const double2* __restrict__ v, const double2 (&u)[4]) {
    int idx = 0;
#pragma unroll
    for (int rr = 0; rr < 4; ++rr)
#pragma unroll
        for (int c = 0; c < 4; ++c)
            if (MASK >> (rr * 4 + c) & 1u) {
                cfma(acc[rr], v[idx], u[c]);
                ++idx;
            }
}

// Any pattern: one 16-way dispatch per block row.
template <int RR>
__device__ __forceinline__ const double2* apply_row(double2& acc, const double2* v, const double2 (&u)[4],
                                                    unsigned nib) {
#pragma unroll
    for (int c = 0; c < 4; ++c)
        if (nib >> c & 1u) {
            cfma(acc, *v, u[c]);
            ++v;
        }
    return v;
}

__device__ __forceinline__ void apply_generic(double2 (&acc)[4], const double2* v, const double2 (&u)[4],
                                              unsigned mask) {
#pragma unroll
    for (int rr = 0; rr < 4; ++rr) v = apply_row<0>(acc[rr], v, u, mask >> (4 * rr) & 0xFu);
}

// Fast paths for the patterns of identity +- gamma-matrix stencils (onsite diag,
// the two Wilson-Dirac hop patterns) and dense blocks; anything else is generic.
__device__ __forceinline__ void apply_block(double2 (&acc)[4], const double2* v, const double2 (&u)[4],
                                            unsigned mask) {
    switch (mask) {
        case 0x0000u: break;
        case 0x8421u: apply_fixed<0x8421u>(acc, v, u); break;
        case 0x9669u: apply_fixed<0x9669u>(acc, v, u); break;
        case 0xA5A5u: apply_fixed<0xA5A5u>(acc, v, u); break;
        case 0x5A5Au: apply_fixed<0x5A5Au>(acc, v, u); break;
        case 0xFFFFu: apply_fixed<0xFFFFu>(acc, v, u); break;
        default:
            if ((mask & (mask - 1u)) == 0u) {  // a single entry (general sparsity without 4x4 structure)
                const int bit = __ffs(static_cast<int>(mask)) - 1, rr = bit >> 2, c = bit & 3;
                const double2 uc = c == 0 ? u[0] : c == 1 ? u[1] : c == 2 ? u[2] : u[3];
#pragma unroll
                for (int q = 0; q < 4; ++q)
                    if (q == rr) cfma(acc[q], v[0], uc);
            } else {
                apply_generic(acc, v, u, mask);
            }
            break;
    }
}


// The diagonal block's U rows are the block-row's own rows: keep them in the
// warp's epilogue staging (smem) instead of re-reading them for the epilogue.
__device__ __forceinline__ void capture_own(const BlockMeta& m, const double2 (&v)[4], int br, double2* epiU, int so,
                                            int ld, unsigned& ownmask, bool on) {
    if (!on || !m.mask || m.bcol != br) return;
    const unsigned cm = (m.mask | m.mask >> 4 | m.mask >> 8 | m.mask >> 12) & 0xFu;
#pragma unroll
    for (int c = 0; c < 4; ++c)
        if (cm >> c & 1u) epiU[so + c * ld] = v[c];
    ownmask |= cm;
}

// Signature-1 chunk (Topi / Wilson-Dirac block-row, common.hpp kSigTopiMasks):
// the 7 blocks come in canonical order with compile-time patterns and value
// offsets, so the walk has no per-block dispatch, no predicates and no meta
// other than the block columns.  U gathers run DEPTH blocks ahead of the FMAs.
template <int DEPTH>
__device__ __forceinline__ void walk_sig_topi(double2 (&acc)[4], const BlockMeta* __restrict__ mr,
                                              const double2* __restrict__ vr, const char* ubase, long long ld16,
                                              int br, double2* epiU, int so, int ld, unsigned& ownmask, bool capture) {
    constexpr int NB = DEPTH + 1;
    constexpr int voff[kSigTopiBlocks] = {0, 4, 12, 20, 28, 36, 44};
    constexpr unsigned masks[kSigTopiBlocks] = {0x8421u, 0x9669u, 0x9669u, 0x9669u, 0x9669u, 0xA5A5u, 0xA5A5u};
    int bc[kSigTopiBlocks];
#pragma unroll
    for (int k = 0; k < kSigTopiBlocks; ++k) bc[k] = mr[k * kC].bcol;
    double2 u[NB][4];
    auto gather = [&](double2 (&v)[4], int b) {
        const char* p = ubase + static_cast<long long>(b) * (4 * ld16);
#pragma unroll
        for (int c = 0; c < 4; ++c) v[c] = ld_gather(reinterpret_cast<const double2*>(p + c * ld16));
    };
#pragma unroll
    for (int k = 0; k < DEPTH; ++k) gather(u[k], bc[k]);
#pragma unroll
    for (int k = 0; k < kSigTopiBlocks; ++k) {
        if (k + DEPTH < kSigTopiBlocks) gather(u[(k + DEPTH) % NB], bc[k + DEPTH]);
        if (k == 0 && capture && bc[0] == br) {  // on-site block: the block-row's own U rows
#pragma unroll
            for (int c = 0; c < 4; ++c) epiU[so + c * ld] = u[0][c];
            ownmask = 0xFu;
        }
        apply_block(acc, vr + voff[k], u[k % NB], masks[k]);  // == kSigTopiMasks
    }
}

// Typed signature-1 walk: in canonical (mask, value-type, bcol) order the Topi
// block-row's 52 values are each purely real or purely imaginary with the fixed
// pattern kSigTopiTypes (bit j of block k set = value j imaginary), stored as one
// double each: a complex multiply-add becomes two FMAs, a value 8 bytes.
constexpr unsigned kSigTopiTypes[kSigTopiBlocks] = {0x00u, 0x5Au, 0x5Au, 0x00u, 0x00u, 0x5Au, 0x5Au};
template <unsigned MASK, unsigned TYPES>
__device__ __forceinline__ void apply_typed(double2 (&acc)[4], const double* __restrict__ v, const double2 (&u)[4]) {
    int idx = 0;
#pragma unroll
    for (int rr = 0; rr < 4; ++rr)
#pragma unroll
        for (int c = 0; c < 4; ++c)
            if (MASK >> (rr * 4 + c) & 1u) {
                const double a = v[idx];
                if (TYPES >> idx & 1u) {  // (0 + i a) u
                    acc[rr].x = fma(-a, u[c].y, acc[rr].x);
                    acc[rr].y = fma(a, u[c].x, acc[rr].y);
                } else {  // (a + 0 i) u
                    acc[rr].x = fma(a, u[c].x, acc[rr].x);
                    acc[rr].y = fma(a, u[c].y, acc[rr].y);
                }
                ++idx;
            }
}
// Block k of the typed Topi block-row (k folds to a constant after unrolling).
__device__ __forceinline__ void apply_typed_k(int k, double2 (&acc)[4], const double* __restrict__ vr,
                                              const double2 (&u)[4]) {
    switch (k) {
        case 0: apply_typed<0x8421u, kSigTopiTypes[0]>(acc, vr + 0, u); break;
        case 1: apply_typed<0x9669u, kSigTopiTypes[1]>(acc, vr + 4, u); break;
        case 2: apply_typed<0x9669u, kSigTopiTypes[2]>(acc, vr + 12, u); break;
        case 3: apply_typed<0x9669u, kSigTopiTypes[3]>(acc, vr + 20, u); break;
        case 4: apply_typed<0x9669u, kSigTopiTypes[4]>(acc, vr + 28, u); break;
        case 5: apply_typed<0xA5A5u, kSigTopiTypes[5]>(acc, vr + 36, u); break;
        default: apply_typed<0xA5A5u, kSigTopiTypes[6]>(acc, vr + 44, u); break;
    }
}

// walk_sig_topi over typed records (register-gather kernel).
template <int DEPTH>
__device__ __forceinline__ void walk_sig_topi_typed(double2 (&acc)[4], const BlockMeta* __restrict__ mr,
                                                    const double* __restrict__ vr, const char* ubase, long long ld16,
                                                    int br, double2* epiU, int so, int ld, unsigned& ownmask,
                                                    bool capture) {
    constexpr int NB = DEPTH + 1;
    int bc[kSigTopiBlocks];
#pragma unroll
    for (int k = 0; k < kSigTopiBlocks; ++k) bc[k] = mr[k * kC].bcol;
    double2 u[NB][4];
    auto gather = [&](double2 (&v)[4], int b) {
        const char* p = ubase + static_cast<long long>(b) * (4 * ld16);
#pragma unroll
        for (int c = 0; c < 4; ++c) v[c] = ld_gather(reinterpret_cast<const double2*>(p + c * ld16));
    };
#pragma unroll
    for (int k = 0; k < DEPTH; ++k) gather(u[k], bc[k]);
#pragma unroll
    for (int k = 0; k < kSigTopiBlocks; ++k) {
        if (k + DEPTH < kSigTopiBlocks) gather(u[(k + DEPTH) % NB], bc[k + DEPTH]);
        if (k == 0 && capture && bc[0] == br) {  // on-site block: the block-row's own U rows
#pragma unroll
            for (int c = 0; c < 4; ++c) epiU[so + c * ld] = u[0][c];
            ownmask = 0xFu;
        }
        apply_typed_k(k, acc, vr, u[k % NB]);
    }
}

struct SmemLayout {
    static constexpr size_t stage_off = 0;
    static constexpr size_t bar_off = stage_off + kNS * kStageBytes;
    static constexpr size_t info_off = bar_off + 2 * kNS * 8;
    static constexpr size_t red_off = info_off + kNS * 16;
    static constexpr size_t cnt_off = red_off + 2 * kNW * 32 * 3 * 8;
    static constexpr size_t epibar_off = cnt_off + 16;
    static constexpr size_t epi_off = (epibar_off + kNW * 8 + 127) / 128 * 128;
    static constexpr size_t kEpiArray = 2048;  // 4 rows x 32 cols x 16 B per warp
    static constexpr size_t total = epi_off + kNW * 3 * kEpiArray;
};

// Ring producer state, live in lane 0 of warp 0 only (a consumer thread too, so
// its memory latencies stall warp 0): the next unit is claimed one unit ahead and
// its piece range resolved from the unit's second piece on, and each piece's
// table entry is loaded one piece (one call) ahead.
struct Producer {
    int u = 0, pf = 0, p = 0, p1 = 0, chunk_seq = 0;
    bool done = false, started = false, known = false;
    unsigned fseq = 0;     // ring uses filled so far
    int un = 0;            // next unit (claimed ahead)
    int pn0 = 0, pn1 = 0;  // its piece range once known
    PieceInfo pi{0, 0, 0}; // table entry of piece p
};

__device__ __forceinline__ void producer_resolve(const KParams& P, Producer& pr) {
    pr.known = true;
    if (pr.un < P.num_units) {
        pr.pn0 = P.unit_piece[pr.un];
        pr.pn1 = P.unit_piece[pr.un + 1];
    }
}

// Fill ring slot `slot` with the next piece (moving to the unit claimed ahead when
// the current one is exhausted) or with a terminate marker.
template <int NG>
__device__ __forceinline__ void produce(const KParams& P, Producer& pr, uint8_t* smem, uint64_t* full, int4* info,
                                        int slot) {
    if (pr.done) return;
    if (!pr.started) {  // first call: this unit (waited for), the next one in flight
        pr.started = true;
        pr.u = static_cast<int>(atomicAdd(&P.counters[0], 1u));
        if (pr.u < P.num_units) {
            pr.pf = pr.p = P.unit_piece[pr.u];
            pr.p1 = P.unit_piece[pr.u + 1];
            pr.pi = P.pieces[pr.p];
            pr.un = static_cast<int>(atomicAdd(&P.counters[0], 1u));
        }
    } else if (pr.p >= pr.p1) {  // current unit exhausted: the one claimed ahead
        if (!pr.known) {         // (empty unit)
            producer_resolve(P, pr);
            if (pr.un < P.num_units) pr.pi = P.pieces[pr.pn0];
        }
        pr.u = pr.un;
        if (pr.u < P.num_units) {
            pr.pf = pr.p = pr.pn0;
            pr.p1 = pr.pn1;
            pr.chunk_seq = 0;
            pr.known = false;
            pr.un = static_cast<int>(atomicAdd(&P.counters[0], 1u));
        }
    }
    if (pr.u >= P.num_units) {
        pr.done = true;
        info[slot] = make_int4(-1, kInfoTerm, 0, 0);
        mbar_arrive(&full[slot]);
        return;
    }
    const PieceInfo pi = pr.pi;
    info[slot] = make_int4(pr.u, pr.p == pr.p1 - 1 ? kInfoUnitLast : 0, pr.chunk_seq % NG, 0);
    mbar_arrive_expect_tx(&full[slot], pi.bytes);
    bulk_g2s_hint(smem + SmemLayout::stage_off + slot * kStageBytes, P.records + pi.offset, pi.bytes, &full[slot],
                  policy_evict_first());
    if (pi.flags & kPieceLast) ++pr.chunk_seq;
    ++pr.p;
    // for the next call: the next unit's range (from this unit's second piece on, or
    // now when this was its last piece) and the next piece's table entry
    if (!pr.known && (pr.p > pr.pf + 1 || pr.p >= pr.p1)) producer_resolve(P, pr);
    if (pr.p < pr.p1) pr.pi = P.pieces[pr.p];
    else if (pr.known && pr.un < P.num_units) pr.pi = P.pieces[pr.pn0];
}

template <int MODE, int LPR, int SD, bool WR>
__global__ void __launch_bounds__(32 * kNW, 2) sell_b4_kernel(const KParams P) {
    constexpr int RPW = 32 / LPR;  // block-rows per warp
    constexpr int GW = kC / RPW;   // warps per group (one group consumes a chunk)
    constexpr int NG = kNW / GW;   // groups
    extern __shared__ __align__(128) uint8_t smem[];
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + SmemLayout::bar_off);
    uint64_t* empty = full + kNS;
    int4* info = reinterpret_cast<int4*>(smem + SmemLayout::info_off);
    double* red = reinterpret_cast<double*>(smem + SmemLayout::red_off);
    unsigned* unit_cnt = reinterpret_cast<unsigned*>(smem + SmemLayout::cnt_off);

    const int cw = threadIdx.x >> 5, lane = threadIdx.x & 31;
    Producer pr;
    if (threadIdx.x == 0) {
        for (int s = 0; s < kNS; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], kNW);
        }
        uint64_t* eb = reinterpret_cast<uint64_t*>(smem + SmemLayout::epibar_off);
        for (int w = 0; w < kNW; ++w) mbar_init(&eb[w], 1);
        unit_cnt[0] = unit_cnt[1] = 0;
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int s = 0; s < kNS; ++s) produce<NG>(P, pr, smem, full, info, s);
        pr.fseq = kNS;
    }

    const int g = cw / GW, wg = cw % GW;
    const int r = wg * RPW + lane / LPR;  // slot inside the chunk
    const int jc = lane % LPR;            // panel column
    const bool col_ok = jc < P.ncols;
    double2 acc[4];
    unsigned ownmask = 0;  // columns of the diagonal block captured into epiU
    int br = -1;
    double eta_x = 0.0, eta_y = 0.0, mu = 0.0;
    unsigned ub = 0;  // parity of this warp's unit count (double-buffered reduction slots)
    // per-warp epilogue staging: own U rows, W (or Z) rows, X rows of the warp's block-rows,
    // fetched by TMA bulk copies at the chunk's first piece (whole rows: ncols == ld)
    uint64_t* epibar = reinterpret_cast<uint64_t*>(smem + SmemLayout::epibar_off) + cw;
    double2* epiU = reinterpret_cast<double2*>(smem + SmemLayout::epi_off + cw * 3 * SmemLayout::kEpiArray);
    double2* epiW = epiU + SmemLayout::kEpiArray / 16;
    double2* epiX = epiW + SmemLayout::kEpiArray / 16;
    // epilogue rows staged by bulk copies: whole rows in one copy (WR: the panel
    // is exactly this slice) or row by row for a column slice of a wider panel;
    // in shared memory a row takes SLD elements
    const bool tma_epi = WR ? P.ncols == P.ld : true;
    // (re-read from the parameter bank at each use: no register held across the walk)
#define SLD (WR ? static_cast<int>(P.ld) : LPR)
    unsigned epi_phase = 0;
    for (unsigned c = 0;; ++c) {
        const int stage = static_cast<int>(c % kNS);
        // Thread 0 refills every slot the warps have released (use q frees the slot
        // for use q + kNS) without waiting on a group still busy with its piece, and
        // blocks only when its own next use (c) is not filled yet (ko bit 64: the
        // in-order refill, for A/B).  A second look between its own piece's walk and
        // epilogue was slower (the producer state live across the walk spills).
        if (threadIdx.x == 0) {
            while (!pr.done && pr.fseq < c + kNS) {
                const unsigned q = pr.fseq - kNS;
                if (pr.fseq <= c || (P.ko & 64)) mbar_wait(&empty[q % kNS], (q / kNS) & 1u);
                else if (!mbar_test(&empty[q % kNS], (q / kNS) & 1u)) break;
                produce<NG>(P, pr, smem, full, info, static_cast<int>(pr.fseq % kNS));
                ++pr.fseq;
            }
        }
        __syncwarp();
        mbar_wait(&full[stage], (c / kNS) & 1u);
        const int4 inf = info[stage];
        if (inf.y & kInfoTerm) break;
        if (inf.z == g) {
            const uint8_t* base = smem + SmemLayout::stage_off + stage * kStageBytes;
            const PieceHdr* h = reinterpret_cast<const PieceHdr*>(base);
            const int kcnt = h->kcnt, flags = h->flags;
            const int32_t* pperm = reinterpret_cast<const int32_t*>(base + 16);
            const uint16_t* pnblk = reinterpret_cast<const uint16_t*>(base + 16 + 4 * kC);
            const BlockMeta* meta = reinterpret_cast<const BlockMeta*>(base + 16 + 4 * kC + 16);
            const double2* vals = reinterpret_cast<const double2*>(meta + kcnt * kC);
            br = pperm[r];
            const int nb = br >= 0 ? pnblk[r] : 0;
            const bool active = col_ok && br >= 0;
            if (flags & kPieceFirst) {
#pragma unroll
                for (int q = 0; q < 4; ++q) acc[q] = make_double2(0.0, 0.0);
                ownmask = 0;
                if (tma_epi) {
                    // rows 4br..4br+3 of W, X (or Z)
                    const long long nrow = br >= 0 ? min(4LL, P.n - 4LL * br) : 0;
                    const unsigned bytes = static_cast<unsigned>(max(nrow, 0LL) * (WR ? P.ld : P.ncols) * 16);
                    const int narr = (ModeT<MODE>::cheb ? 1 : 0) + (ModeT<MODE>::reads_x ? 1 : 0) +
                                     (ModeT<MODE>::reads_z ? 1 : 0);
                    unsigned tot = bytes;
#pragma unroll
                    for (int off = 16; off > 0; off >>= 1) tot += __shfl_xor_sync(0xffffffffu, tot, off);
                    tot /= LPR;  // each block-row counted by its LPR lanes
                    if (lane == 0) mbar_arrive_expect_tx(epibar, tot * narr);
                    __syncwarp();
                    if (jc == 0 && bytes) {
                        const uint64_t ef = policy_evict_first();
                        if constexpr (WR) {
                            const long long gofs = 4LL * br * P.ld;
                            const int so = (lane / LPR) * 4 * static_cast<int>(P.ld);
                            if (ModeT<MODE>::cheb) bulk_g2s_hint(epiW + so, P.W + gofs, bytes, epibar, ef);
                            if (ModeT<MODE>::reads_z) bulk_g2s_hint(epiW + so, P.Z + gofs, bytes, epibar, ef);
                            if (ModeT<MODE>::reads_x) bulk_g2s_hint(epiX + so, P.X + gofs, bytes, epibar, ef);
                        } else {
                            const unsigned cb = static_cast<unsigned>(P.ncols * 16);
                            for (int q = 0; q < static_cast<int>(nrow); ++q) {
                                const long long gofs = (4LL * br + q) * P.ld;
                                const int so = ((lane / LPR) * 4 + q) * SLD;
                                if (ModeT<MODE>::cheb) bulk_g2s_hint(epiW + so, P.W + gofs, cb, epibar, ef);
                                if (ModeT<MODE>::reads_z) bulk_g2s_hint(epiW + so, P.Z + gofs, cb, epibar, ef);
                                if (ModeT<MODE>::reads_x) bulk_g2s_hint(epiX + so, P.X + gofs, cb, epibar, ef);
                            }
                        }
                    }
                }
            }
            // software-pipelined walk over the piece's blocks: U buffers in rotation
            // by unrolling (no register moves, so no early wait on loads)
            const long long ld16 = P.ld * 16;
            auto meta_at = [&](int k) { return (k < nb) ? meta[k * kC + r] : BlockMeta{0, 0, 0}; };
            if (P.typed && (flags & kPieceTyped)) {  // a typed signature-1 piece
                const char* ub0 = reinterpret_cast<const char*>(P.U + (col_ok ? jc : 0));
                walk_sig_topi_typed<SD>(acc, meta + r, reinterpret_cast<const double*>(vals) + r * kSigTopiNnz, ub0,
                                        ld16, br, epiU, (lane / LPR) * 4 * SLD + jc, SLD, ownmask, tma_epi && active);
            } else if ((flags >> kSigShift) == 1) {
                // all slots valid; idle lanes (jc >= ncols) gather column 0 and discard
                const char* ub0 = reinterpret_cast<const char*>(P.U + (col_ok ? jc : 0));
                walk_sig_topi<SD>(acc, meta + r, vals + r * kSigTopiNnz, ub0, ld16, br, epiU,
                                    (lane / LPR) * 4 * SLD + jc, SLD, ownmask,
                                    tma_epi && active);
            } else {  // generic blocks, 2 U buffers in rotation
                const char* ubase = reinterpret_cast<const char*>(P.U + jc);
                int k0 = 0;
                if constexpr (LPR == 32) {
                    // groups of eight blocks (general sparsity without 4x4 structure: mostly one
                    // entry per block): the U rows of a group of single-entry blocks are gathered
                    // together, eight in flight, one complex FMA each; a group holding a
                    // multi-entry block (e.g. the diagonal one) takes the block walk one block at
                    // a time.  Either way the row sums run in the blocks' column order.
                    constexpr int D = 8;
                    for (; k0 + D <= nb; k0 += D) {
                        BlockMeta mm[D];
                        unsigned multi = 0;
#pragma unroll
                        for (int j = 0; j < D; ++j) {
                            mm[j] = meta[(k0 + j) * kC + r];
                            multi |= mm[j].mask & (mm[j].mask - 1u);
                        }
                        if (multi) {
#pragma unroll 1
                            for (int j = 0; j < D; ++j) {
                                double2 t[4];
                                const BlockMeta m = meta[(k0 + j) * kC + r];
                                load_block(t, m, ubase, ld16, active);
                                capture_own(m, t, br, epiU, (lane / LPR) * 4 * SLD + jc, SLD, ownmask,
                                            tma_epi && active);
                                apply_block(acc, vals + m.voff, t, m.mask);
                            }
                            continue;
                        }
                        double2 v[D];
#pragma unroll
                        for (int j = 0; j < D; ++j) {
                            const int bit = __ffs(static_cast<int>(mm[j].mask)) - 1;
                            v[j] = active ? ld_gather(reinterpret_cast<const double2*>(
                                                ubase + (4LL * mm[j].bcol + (bit & 3)) * ld16))
                                          : make_double2(0.0, 0.0);
                        }
#pragma unroll
                        for (int j = 0; j < D; ++j) {
                            const int rr = (__ffs(static_cast<int>(mm[j].mask)) - 1) >> 2;
                            const double2 a = vals[mm[j].voff];
#pragma unroll
                            for (int q = 0; q < 4; ++q)
                                if (q == rr) cfma(acc[q], a, v[j]);
                        }
                    }
                }
                double2 va[4], vb[4];
                BlockMeta ma = meta_at(k0), mb{0, 0, 0};
                // L2 prefetch of the U rows P.gpf blocks ahead: scattered blocks (general
                // sparsity: one row per block, far apart) keep more gathers in flight
                // than the two register buffers do
                const int gpf = P.gpf;
                auto pf = [&](int k) {
                    if (!gpf || !active || k >= nb) return;
                    const BlockMeta m = meta[k * kC + r];
                    const unsigned cm = (m.mask | m.mask >> 4 | m.mask >> 8 | m.mask >> 12) & 0xFu;
                    const char* p = ubase + static_cast<long long>(m.bcol) * (4 * ld16);
#pragma unroll
                    for (int c = 0; c < 4; ++c)
                        if (cm >> c & 1u) asm volatile("prefetch.global.L2 [%0];" ::"l"(p + c * ld16));
                };
                for (int k = k0; k < k0 + gpf && k < nb; ++k) pf(k + 1);
                load_block(va, ma, ubase, ld16, active);
                for (int k = k0; k < kcnt; k += 2) {
                    pf(k + 1 + gpf);
                    pf(k + 2 + gpf);
                    if (k + 1 < kcnt) {
                        mb = meta_at(k + 1);
                        load_block(vb, mb, ubase, ld16, active);
                    }
                    capture_own(ma, va, br, epiU, (lane / LPR) * 4 * SLD + jc, SLD, ownmask, tma_epi && active);
                    apply_block(acc, vals + ma.voff, va, ma.mask);
                    if (k + 1 >= kcnt) break;
                    if (k + 2 < kcnt) {
                        ma = meta_at(k + 2);
                        load_block(va, ma, ubase, ld16, active);
                    }
                    capture_own(mb, vb, br, epiU, (lane / LPR) * 4 * SLD + jc, SLD, ownmask, tma_epi && active);
                    apply_block(acc, vals + mb.voff, vb, mb.mask);
                }
            }
            if (flags & kPieceLast) {
                if (tma_epi) {
                    mbar_wait(epibar, epi_phase);
                    epi_phase ^= 1;
                }
                const bool mir_blk = block_mirrored(P, active ? br : -1);
                // epilogue in two halves of two rows: issue the half's loads, then use them
#pragma unroll
                for (int h2 = 0; h2 < 4; h2 += 2) {
                    double2 uo[2], wold[2], xold[2];
#pragma unroll
                    for (int q2 = 0; q2 < 2; ++q2) {
                        const long long row = 4LL * br + h2 + q2;
                        const bool ok = active && row < P.n;
                        if (tma_epi) {
                            const int so = ((lane / LPR) * 4 + h2 + q2) * SLD + jc;
                            uo[q2] = !ok ? make_double2(0.0, 0.0)
                                         : ((ownmask >> (h2 + q2) & 1u) ? epiU[so] : ld_gather(P.U + row * P.ld + jc));
                            if (ModeT<MODE>::cheb) wold[q2] = ok ? epiW[so] : make_double2(0.0, 0.0);
                            if (ModeT<MODE>::reads_x) xold[q2] = ok ? epiX[so] : make_double2(0.0, 0.0);
                            if (ModeT<MODE>::reads_z) xold[q2] = ok ? epiW[so] : make_double2(0.0, 0.0);
                            continue;
                        }
                        uo[q2] = ok ? ld_gather(P.U + row * P.ld + jc) : make_double2(0.0, 0.0);
                        if (ModeT<MODE>::cheb) wold[q2] = ok ? ld_stream(P.W + row * P.ld + jc) : make_double2(0.0, 0.0);
                        if (ModeT<MODE>::reads_x)
                            xold[q2] = ok ? ld_stream(P.X + row * P.ld + jc) : make_double2(0.0, 0.0);
                        if (ModeT<MODE>::reads_z)
                            xold[q2] = ok ? ld_stream(P.Z + row * P.ld + jc) : make_double2(0.0, 0.0);
                    }
#pragma unroll
                    for (int q2 = 0; q2 < 2; ++q2) {
                        const int q = h2 + q2;
                        const long long row = 4LL * br + q;
                        if (!(active && row < P.n)) continue;
                        const double2 u = uo[q2];
                        double2 y;
                        y.x = fma(P.alpha, acc[q].x, P.beta * u.x);
                        y.y = fma(P.alpha, acc[q].y, P.beta * u.y);
                        if (MODE == M_SHIFT) {
                            st_out(P, row, jc, y, mir_blk);
                        } else if (MODE == M_TWO_MINUS) {
                            st_out(P, row, jc, make_double2(fma(2.0, y.x, -xold[q2].x), fma(2.0, y.y, -xold[q2].y)), mir_blk);
                        } else if (MODE == M_INIT) {
                            const double2 wn = make_double2(fma(2.0, y.x, -xold[q2].x), fma(2.0, y.y, -xold[q2].y));
                            st_out(P, row, jc, wn, mir_blk);
                            double2 xn;
                            xn.x = fma(P.g2, wn.x, fma(P.g1, u.x, P.g0 * xold[q2].x));
                            xn.y = fma(P.g2, wn.y, fma(P.g1, u.y, P.g0 * xold[q2].y));
                            st_stream(P.X + row * P.ld + jc, xn);
                        } else {
                            const double2 wn = make_double2(fma(2.0, y.x, -wold[q2].x), fma(2.0, y.y, -wold[q2].y));
                            eta_x = fma(wn.x, u.x, eta_x);  // conj(w) * u
                            eta_x = fma(wn.y, u.y, eta_x);
                            eta_y = fma(wn.x, u.y, eta_y);
                            eta_y = fma(-wn.y, u.x, eta_y);
                            mu = fma(u.x, u.x, mu);
                            mu = fma(u.y, u.y, mu);
                            st_out(P, row, jc, wn, mir_blk);
                            if (MODE == M_CHEB)
                                st_stream(P.X + row * P.ld + jc,
                                          make_double2(fma(P.gc, wn.x, xold[q2].x), fma(P.gc, wn.y, xold[q2].y)));
                            if (MODE == M_CHEB_X2)
                                st_stream(P.X + row * P.ld + jc,
                                          make_double2(fma(P.gc, wn.x, fma(P.gu, u.x, xold[q2].x)),
                                                       fma(P.gc, wn.y, fma(P.gu, u.y, xold[q2].y))));
                            if (MODE == M_CHEB_X3)
                                st_stream(P.X + row * P.ld + jc,
                                          make_double2(fma(P.gc, wn.x, fma(P.gu, u.x, fma(P.gw, wold[q2].x, xold[q2].x))),
                                                       fma(P.gc, wn.y, fma(P.gu, u.y, fma(P.gw, wold[q2].y, xold[q2].y)))));
                        }
                    }
                }
            }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[stage]);
        if (ModeT<MODE>::cheb && (inf.y & kInfoUnitLast)) {
            // per-unit moments: lanes sharing a column, then warps in fixed order by
            // the last warp to arrive (double-buffered slots by unit parity)
#pragma unroll
            for (int off = LPR; off < 32; off <<= 1) {
                eta_x += __shfl_xor_sync(0xffffffffu, eta_x, off);
                eta_y += __shfl_xor_sync(0xffffffffu, eta_y, off);
                mu += __shfl_xor_sync(0xffffffffu, mu, off);
            }
            double* rb = red + static_cast<size_t>(ub) * kNW * 32 * 3;
            if (lane < LPR) {
                rb[(cw * 32 + lane) * 3 + 0] = eta_x;
                rb[(cw * 32 + lane) * 3 + 1] = eta_y;
                rb[(cw * 32 + lane) * 3 + 2] = mu;
            }
            __threadfence_block();
            __syncwarp();
            unsigned last = 0;
            if (lane == 0) last = (atomicAdd(&unit_cnt[ub], 1u) == kNW - 1) ? 1u : 0u;
            last = __shfl_sync(0xffffffffu, last, 0);
            if (last) {
                __threadfence_block();
                if (lane < LPR) {
                    double sx = 0, sy = 0, sm = 0;
                    for (int w2 = 0; w2 < kNW; ++w2) {
                        sx += rb[(w2 * 32 + lane) * 3 + 0];
                        sy += rb[(w2 * 32 + lane) * 3 + 1];
                        sm += rb[(w2 * 32 + lane) * 3 + 2];
                    }
                    double* dst = P.partials + (static_cast<size_t>(inf.x) * 32 + lane) * 3;
                    dst[0] = sx;
                    dst[1] = sy;
                    dst[2] = sm;
                }
                __syncwarp();
                if (lane == 0) {
                    unit_cnt[ub] = 0;
                    __threadfence_block();
                }
            }
            ub ^= 1u;
            eta_x = eta_y = mu = 0.0;
        }
    }
    // self-resetting ticket counters for the next launch on this matrix
    __syncthreads();
    // mirrored rows reach the peer before the kernel completes (one cumulative
    // system fence per CTA after the barrier; a fence per thread costs ~10 %)
    if (P.nmir && threadIdx.x == 0) __threadfence_system();
    // launched as a programmatic dependent of the previous step's reduce_moments
    // (which triggers at its start): this grid does not complete before it
    asm volatile("griddepcontrol.wait;" ::: "memory");
    if (threadIdx.x == 0) {
        __threadfence();
        const unsigned done = atomicAdd(&P.counters[1], 1u);
        if (done == gridDim.x - 1) {
            P.counters[0] = 0;
            P.counters[1] = 0;
            __threadfence();
        }
    }
}

#undef SLD

// ---------------------------------------------------------------------------
// Chunk-staged variant (whole-row n_b = 32 panels, every chunk with a staging
// plan): one CTA per SM, 8 consumer warps (one block-row of the chunk each)
// and one producer warp.  Per chunk the producer stages the piece record and
// the chunk's distinct U block columns -- one 1-D TMA bulk copy per run of
// consecutive block columns (the whole neighbourhood of 8 lattice sites is 5-7
// runs) -- into one of two shared-memory stages, so the gathers of a chunk are
// in flight as bulk copies without holding registers, while the consumers walk
// the previous chunk out of shared memory.  W / X (or Z) rows of the epilogue
// are prefetched into registers when the chunk starts.
constexpr int kStagedWarps = kNW + 1;
struct StagedLayout {
    static constexpr size_t rec_off = 0;                                       // [2][kStageBytes]
    static constexpr size_t ust_off = rec_off + 2 * kStageBytes;               // [2][kMaxStage][2 KB]
    static constexpr size_t bar_off = ust_off + 2 * size_t(kMaxStage) * 2048;  // full_rec[2], full_u[2], empty[2]
    static constexpr size_t info_off = bar_off + 6 * 8;                        // int4[2]
    static constexpr size_t cnt_off = info_off + 2 * 16;                       // unit_cnt[2]
    static constexpr size_t red_off = (cnt_off + 16 + 127) / 128 * 128;       // [2][kNW][32][3] doubles
    static constexpr size_t total = red_off + 2 * kNW * 32 * 3 * 8;
};
static_assert(StagedLayout::total <= 227 * 1024, "staged layout exceeds shared memory");

// Signature-1 walk out of the staged U: compile-time patterns and value offsets.
__device__ __forceinline__ void walk_staged_topi(double2 (&acc)[4], const uint8_t* __restrict__ sx,
                                                 const double2* __restrict__ us, const double2* __restrict__ vr) {
    constexpr int voff[kSigTopiBlocks] = {0, 4, 12, 20, 28, 36, 44};
    constexpr unsigned masks[kSigTopiBlocks] = {0x8421u, 0x9669u, 0x9669u, 0x9669u, 0x9669u, 0xA5A5u, 0xA5A5u};
    double2 u[2][4];
    auto fetch = [&](double2 (&v)[4], int k) {
        const double2* b = us + static_cast<int>(sx[k * kC]) * 128;
#pragma unroll
        for (int c = 0; c < 4; ++c) v[c] = b[c * 32];
    };
    fetch(u[0], 0);
#pragma unroll
    for (int k = 0; k < kSigTopiBlocks; ++k) {
        if (k + 1 < kSigTopiBlocks) fetch(u[(k + 1) & 1], k + 1);
        apply_block(acc, vr + voff[k], u[k & 1], masks[k]);  // == kSigTopiMasks
    }
}

// Typed walk of the staged kernel (see apply_typed); staged block columns of
// 4 rows x NBW columns.
template <int NBW = 32>
__device__ __forceinline__ void walk_staged_topi_typed(double2 (&acc)[4], const uint8_t* __restrict__ sx,
                                                       const double2* __restrict__ us, const double* __restrict__ vr) {
    constexpr int voff[kSigTopiBlocks] = {0, 4, 12, 20, 28, 36, 44};
    double2 u[2][4];
    auto fetch = [&](double2 (&v)[4], int k) {
        const double2* b = us + static_cast<int>(sx[k * kC]) * (4 * NBW);
#pragma unroll
        for (int c = 0; c < 4; ++c) v[c] = b[c * NBW];
    };
    fetch(u[0], 0);
    fetch(u[1], 1);
    apply_typed<0x8421u, kSigTopiTypes[0]>(acc, vr + voff[0], u[0]);
    fetch(u[0], 2);
    apply_typed<0x9669u, kSigTopiTypes[1]>(acc, vr + voff[1], u[1]);
    fetch(u[1], 3);
    apply_typed<0x9669u, kSigTopiTypes[2]>(acc, vr + voff[2], u[0]);
    fetch(u[0], 4);
    apply_typed<0x9669u, kSigTopiTypes[3]>(acc, vr + voff[3], u[1]);
    fetch(u[1], 5);
    apply_typed<0x9669u, kSigTopiTypes[4]>(acc, vr + voff[4], u[0]);
    fetch(u[0], 6);
    apply_typed<0xA5A5u, kSigTopiTypes[5]>(acc, vr + voff[5], u[1]);
    apply_typed<0xA5A5u, kSigTopiTypes[6]>(acc, vr + voff[6], u[0]);
}

// Epilogue operands of block-row br (W or Z, and X rows), 4 rows x this lane's column
// of an NBW-wide panel.
template <int MODE, int NBW = 32>
__device__ __forceinline__ void prefetch_rows(const KParams& P, int br, int lane, double2 (&wo)[4], double2 (&xo)[4]) {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const long long row = 4LL * br + q;
        const bool ok = br >= 0 && row < P.n;
        const long long o = row * NBW + lane;
        wo[q] = xo[q] = make_double2(0.0, 0.0);
        if (P.ko & 1) continue;
        if (ok && ModeT<MODE>::cheb) wo[q] = ld_stream(P.W + o);
        if (ok && ModeT<MODE>::reads_z) wo[q] = ld_stream(P.Z + o);
        if (ok && ModeT<MODE>::reads_x) xo[q] = ld_stream(P.X + o);
    }
}

template <int MODE>
__global__ void __launch_bounds__(32 * kStagedWarps, 1) sell_b4_staged_kernel(const KParams P,
                                                                               const StagePlan* __restrict__ plans) {
    using L = StagedLayout;
    extern __shared__ __align__(128) uint8_t smem[];
    uint64_t* full_rec = reinterpret_cast<uint64_t*>(smem + L::bar_off);
    uint64_t* full_u = full_rec + 2;
    uint64_t* empty = full_rec + 4;
    int4* info = reinterpret_cast<int4*>(smem + L::info_off);
    unsigned* unit_cnt = reinterpret_cast<unsigned*>(smem + L::cnt_off);
    double* red = reinterpret_cast<double*>(smem + L::red_off);
    const int cw = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int s = 0; s < 2; ++s) {
            mbar_init(&full_rec[s], 1);
            mbar_init(&full_u[s], 1);
            mbar_init(&empty[s], kNW);
        }
        unit_cnt[0] = unit_cnt[1] = 0;
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    if (cw == kNW) {
        // ---------------------------------------------------------- producer
        // per stage: the record (its own barrier, so consumers can read the next
        // chunk's block-rows early), then one bulk copy per run of U block columns.
        // Nothing on the issue path waits for global memory: the next unit is
        // claimed while the current one streams (its piece range resolved half
        // way through), and each piece's table entry and staging plan are
        // loaded one piece ahead (the plan as one coalesced 256-B warp load).
        const uint64_t ef = policy_evict_first();
        const unsigned full = 0xffffffffu;
        const int dpf = P.wpf & 15;
        // unit blockIdx.x first, without a ticket (its piece range loads at once);
        // tickets then hand out units gridDim.x, gridDim.x + 1, ...
        auto claim = [&]() -> unsigned { return lane == 0 ? gridDim.x + atomicAdd(&P.counters[0], 1u) : 0u; };
        const uint2* plan_words = reinterpret_cast<const uint2*>(plans);  // 32 words per plan: header, runs[31]
        int u = static_cast<int>(blockIdx.x);
        int p0 = 0, p1 = 0, r0v = -1;
        if (u < P.num_units) {
            p0 = P.unit_piece[u];
            p1 = P.unit_piece[u + 1];
            if (dpf && p0 + lane < p1) r0v = P.piece_row0[p0 + lane];
        }
        unsigned un_raw = claim();  // the next unit, in flight
        PieceInfo pi_n{0, 0, 0};
        uint2 pw_n = make_uint2(0, 0);
        if (u < P.num_units) {
            pi_n = P.pieces[p0];
            pw_n = plan_words[static_cast<size_t>(p0) * 32 + lane];
        }
        unsigned seq = 0;
        while (u < P.num_units) {
            int un = P.num_units, pn0 = 0, pn1 = 0, r0n = -1;
            bool known = false;
            for (int p = p0; p < p1; ++p) {
                const int slot = static_cast<int>(seq & 1u);
                const PieceInfo pi = pi_n;
                const uint2 pw = pw_n;
                if (!known && p == p0 + ((p1 - p0 - 1) >> 1)) {  // the next unit's range (mid-unit)
                    un = static_cast<int>(__shfl_sync(full, un_raw, 0));
                    if (un < P.num_units) {
                        pn0 = P.unit_piece[un];
                        pn1 = P.unit_piece[un + 1];
                    }
                    known = true;
                }
                // metadata of the piece after this one
                const int q = p + 1 < p1 ? p + 1 : (un < P.num_units ? pn0 : -1);
                if (q >= 0) {
                    pi_n = P.pieces[q];
                    pw_n = plan_words[static_cast<size_t>(q) * 32 + lane];
                }
                if (dpf) {  // epilogue rows of piece p + dpf into L2 (one bulk prefetch per buffer)
                    const int t = p + dpf;
                    const int r0 = __shfl_sync(full, r0v, min(t - p0, 31));
                    if (lane == 0 && t < p1 && t - p0 < 32 && r0 >= 0) {
                        const long long row0 = 4LL * r0, row1 = min(row0 + 4 * kC, P.n);
                        const unsigned nbytes = static_cast<unsigned>(max(row1 - row0, 0LL) * 512);
                        if (nbytes) {
                            if (ModeT<MODE>::cheb) bulk_prefetch_l2(P.W + row0 * 32, nbytes);
                            if (ModeT<MODE>::reads_z) bulk_prefetch_l2(P.Z + row0 * 32, nbytes);
                            if (ModeT<MODE>::reads_x && (P.wpf & 16)) bulk_prefetch_l2(P.X + row0 * 32, nbytes);
                        }
                    }
                    if (known && p == p1 - 1 && dpf && un < P.num_units && pn0 + lane < pn1)
                        r0n = P.piece_row0[pn0 + lane];
                }
                // plan: lane 0 holds the header (nruns), lane l + 1 holds runs[l]
                const unsigned nruns = __shfl_sync(full, pw.x, 0) & 0xffffu;
                const unsigned rb = __shfl_down_sync(full, pw.x, 1), rl = __shfl_down_sync(full, pw.y, 1);
                unsigned bytes = 0;
                long long row0 = 0;
                int dst = 0;
                if (static_cast<unsigned>(lane) < nruns) {
                    const int bcol = static_cast<int>(rb);
                    row0 = 4LL * bcol;
                    const long long row1 = min(4LL * (bcol + static_cast<int>(rl & 0xffffu)), P.urows);
                    bytes = static_cast<unsigned>(max(row1 - row0, 0LL) * 512);
                    dst = static_cast<int>(rl >> 16);
                }
                if ((P.ko & 16) || ((P.ko & 32) && (lane == 1 || lane == 3))) bytes = 0;
                unsigned tot = bytes;
#pragma unroll
                for (int off = 16; off > 0; off >>= 1) tot += __shfl_xor_sync(full, tot, off);
                if (lane == 0) mbar_wait(&empty[slot], ((seq >> 1) & 1u) ^ 1u);
                __syncwarp();
                if (lane == 0) {
                    info[slot] = make_int4(u, p == p1 - 1 ? kInfoUnitLast : 0, 0, 0);
                    mbar_arrive_expect_tx(&full_rec[slot], pi.bytes);
                    bulk_g2s_hint(smem + L::rec_off + slot * kStageBytes, P.records + pi.offset, pi.bytes,
                                  &full_rec[slot], ef);
                    mbar_arrive_expect_tx(&full_u[slot], tot);
                }
                __syncwarp();
                if (bytes)
                    bulk_g2s(smem + L::ust_off + (static_cast<size_t>(slot) * kMaxStage + dst) * 2048,
                             P.U + row0 * 32, bytes, &full_u[slot]);
                ++seq;
            }
            if (!known) {  // (empty unit)
                un = static_cast<int>(__shfl_sync(full, un_raw, 0));
                if (un < P.num_units) {
                    pn0 = P.unit_piece[un];
                    pn1 = P.unit_piece[un + 1];
                    pi_n = P.pieces[pn0];
                    pw_n = plan_words[static_cast<size_t>(pn0) * 32 + lane];
                    if (dpf && pn0 + lane < pn1) r0n = P.piece_row0[pn0 + lane];
                }
            }
            u = un;
            p0 = pn0;
            p1 = pn1;
            r0v = r0n;
            if (u < P.num_units) un_raw = claim();
        }
        // no more units: tell the consumers
        const int slot = static_cast<int>(seq & 1u);
        if (lane == 0) {
            mbar_wait(&empty[slot], ((seq >> 1) & 1u) ^ 1u);
            info[slot] = make_int4(-1, kInfoTerm, 0, 0);
            mbar_arrive(&full_rec[slot]);
        }
        __syncwarp();
    } else {
        // ---------------------------------------------------------- consumers
        const int r = cw;  // slot of the chunk this warp owns
        double eta_x = 0.0, eta_y = 0.0, mu = 0.0;
        unsigned ub = 0;
        // W / X rows run one chunk ahead: chunk c+1's are loaded as soon as its
        // record lands (end of chunk c's walk) and consumed in its epilogue
        double2 wcur[4], xcur[4];
        mbar_wait(&full_rec[0], 0);
        int4 inf = info[0];
        int br = -1;
        if (!(inf.y & kInfoTerm)) {
            br = reinterpret_cast<const int32_t*>(smem + L::rec_off + 16)[r];
            prefetch_rows<MODE>(P, br, lane, wcur, xcur);
        }
        for (unsigned seq = 0; !(inf.y & kInfoTerm); ++seq) {
            const int slot = static_cast<int>(seq & 1u);
            const uint8_t* base = smem + L::rec_off + slot * kStageBytes;
            const PieceHdr* h = reinterpret_cast<const PieceHdr*>(base);
            const int kcnt = h->kcnt, flags = h->flags;
            const uint16_t* pnblk = reinterpret_cast<const uint16_t*>(base + 16 + 4 * kC);
            const BlockMeta* meta = reinterpret_cast<const BlockMeta*>(base + 16 + 4 * kC + 16);
            const double2* vals = reinterpret_cast<const double2*>(meta + kcnt * kC);
            const uint8_t* sidx =
                base + ((flags & kPieceTyped) ? sidx_offset(kC, kcnt, 0) + (8 * h->nvals + 15u) / 16 * 16
                                              : sidx_offset(kC, kcnt, h->nvals));
            const bool active = br >= 0;
            double2 acc[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) acc[q] = make_double2(0.0, 0.0);
            if (!(P.ko & 2)) mbar_wait(&full_u[slot], (seq >> 1) & 1u);
            const double2* us = reinterpret_cast<const double2*>(smem + L::ust_off + slot * size_t(kMaxStage) * 2048) +
                                lane;
            double2 uo[4];
            if (active) {
                // own rows first: the walk's consumed loads then order these before the release
                const double2* ob = us + static_cast<int>(sidx[kcnt * kC + r]) * 128;
#pragma unroll
                for (int q = 0; q < 4; ++q) uo[q] = ob[q * 32];
                if (P.ko & 4) {
                } else if (flags & kPieceTyped) {
                    walk_staged_topi_typed(acc, sidx + r, us, reinterpret_cast<const double*>(vals) + r * kSigTopiNnz);
                } else if ((flags >> kSigShift) == 1) {
                    walk_staged_topi(acc, sidx + r, us, vals + r * kSigTopiNnz);
                } else {
                    const int nb = pnblk[r];
                    for (int k = 0; k < nb; ++k) {
                        const BlockMeta m = meta[k * kC + r];
                        const double2* b = us + static_cast<int>(sidx[k * kC + r]) * 128;
                        const unsigned cm = (m.mask | m.mask >> 4 | m.mask >> 8 | m.mask >> 12) & 0xFu;
                        double2 v[4];
#pragma unroll
                        for (int c = 0; c < 4; ++c) v[c] = (cm >> c & 1u) ? b[c * 32] : make_double2(0.0, 0.0);
                        apply_block(acc, vals + m.voff, v, m.mask);
                    }
                }
            }
            const int4 icur = inf;
            // generic-proxy reads of the stage are ordered before the producer's
            // next bulk copies into it (WAR across proxies)
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[slot]);  // stage released: the rest runs from registers
            // next chunk: block-row and epilogue operands, before this chunk's epilogue
            // (ko bit 512: after it, as the narrow kernel does -- here 0.5-1.5 % slower,
            // profiles/producer_ab_r02.md)
            const int nslot = slot ^ 1;
            double2 wnxt[4], xnxt[4];
            int br_next = -1;
            auto fetch_next = [&]() {
                mbar_wait(&full_rec[nslot], ((seq + 1) >> 1) & 1u);
                inf = info[nslot];
                if (!(inf.y & kInfoTerm)) {
                    br_next = reinterpret_cast<const int32_t*>(smem + L::rec_off + nslot * kStageBytes + 16)[r];
                    prefetch_rows<MODE>(P, br_next, lane, wnxt, xnxt);
                } else {
#pragma unroll
                    for (int q = 0; q < 4; ++q) wnxt[q] = xnxt[q] = make_double2(0.0, 0.0);
                }
            };
            const bool early = (P.ko & 512) == 0;
            if (early) fetch_next();
            const bool mir_blk = block_mirrored(P, br);
            if (active && !(P.ko & 8)) {
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const long long row = 4LL * br + q;
                    if (row >= P.n) continue;
                    const double2 u = uo[q];
                    double2 y;
                    y.x = fma(P.alpha, acc[q].x, P.beta * u.x);
                    y.y = fma(P.alpha, acc[q].y, P.beta * u.y);
                    if (MODE == M_SHIFT) {
                        st_out(P, row, lane, y, mir_blk);
                    } else if (MODE == M_TWO_MINUS) {
                        st_out(P, row, lane, make_double2(fma(2.0, y.x, -wcur[q].x), fma(2.0, y.y, -wcur[q].y)), mir_blk);
                    } else if (MODE == M_INIT) {
                        const double2 wn = make_double2(fma(2.0, y.x, -xcur[q].x), fma(2.0, y.y, -xcur[q].y));
                        st_out(P, row, lane, wn, mir_blk);
                        double2 xn;
                        xn.x = fma(P.g2, wn.x, fma(P.g1, u.x, P.g0 * xcur[q].x));
                        xn.y = fma(P.g2, wn.y, fma(P.g1, u.y, P.g0 * xcur[q].y));
                        st_stream(P.X + row * 32 + lane, xn);
                    } else {
                        const double2 wn = make_double2(fma(2.0, y.x, -wcur[q].x), fma(2.0, y.y, -wcur[q].y));
                        eta_x = fma(wn.x, u.x, eta_x);  // conj(w) * u
                        eta_x = fma(wn.y, u.y, eta_x);
                        eta_y = fma(wn.x, u.y, eta_y);
                        eta_y = fma(-wn.y, u.x, eta_y);
                        mu = fma(u.x, u.x, mu);
                        mu = fma(u.y, u.y, mu);
                        st_out(P, row, lane, wn, mir_blk);
                        if (MODE == M_CHEB)
                            st_stream(P.X + row * 32 + lane,
                                      make_double2(fma(P.gc, wn.x, xcur[q].x), fma(P.gc, wn.y, xcur[q].y)));
                        if (MODE == M_CHEB_X2)
                            st_stream(P.X + row * 32 + lane,
                                      make_double2(fma(P.gc, wn.x, fma(P.gu, u.x, xcur[q].x)),
                                                   fma(P.gc, wn.y, fma(P.gu, u.y, xcur[q].y))));
                        if (MODE == M_CHEB_X3)
                            st_stream(P.X + row * 32 + lane,
                                      make_double2(fma(P.gc, wn.x, fma(P.gu, u.x, fma(P.gw, wcur[q].x, xcur[q].x))),
                                                   fma(P.gc, wn.y, fma(P.gu, u.y, fma(P.gw, wcur[q].y, xcur[q].y)))));
                    }
                }
            }
            if (!early) fetch_next();
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                wcur[q] = wnxt[q];
                xcur[q] = xnxt[q];
            }
            br = br_next;
            if (ModeT<MODE>::cheb && (icur.y & kInfoUnitLast)) {
                // per-unit moments: warps in fixed order by the last warp to arrive
                double* rb = red + static_cast<size_t>(ub) * kNW * 32 * 3;
                rb[(cw * 32 + lane) * 3 + 0] = eta_x;
                rb[(cw * 32 + lane) * 3 + 1] = eta_y;
                rb[(cw * 32 + lane) * 3 + 2] = mu;
                // release: every lane's slot is visible before the count; acquire:
                // every lane of the last warp fences before reading the others'
                __threadfence_block();
                __syncwarp();
                unsigned last = 0;
                if (lane == 0) last = (atomicAdd(&unit_cnt[ub], 1u) == kNW - 1) ? 1u : 0u;
                last = __shfl_sync(0xffffffffu, last, 0);
                if (last) {
                    __threadfence_block();
                    double sx = 0, sy = 0, sm = 0;
                    for (int w2 = 0; w2 < kNW; ++w2) {
                        sx += rb[(w2 * 32 + lane) * 3 + 0];
                        sy += rb[(w2 * 32 + lane) * 3 + 1];
                        sm += rb[(w2 * 32 + lane) * 3 + 2];
                    }
                    double* dst = P.partials + (static_cast<size_t>(icur.x) * 32 + lane) * 3;
                    dst[0] = sx;
                    dst[1] = sy;
                    dst[2] = sm;
                    __syncwarp();
                    if (lane == 0) {
                        unit_cnt[ub] = 0;
                        __threadfence_block();
                    }
                }
                ub ^= 1u;
                eta_x = eta_y = mu = 0.0;
            }
            if (P.nsig && (icur.y & kInfoUnitLast) && icur.x < P.nbnd) {
                // this warp is done with a boundary unit (halo reads, mirrored stores): the
                // last such completion raises the neighbours' flags
                __syncwarp();
                if (lane == 0) {
                    __threadfence_system();
                    if (atomicAdd(&P.counters[3], 1u) + 1u == static_cast<unsigned>(P.nbnd) * kNW) {
                        __threadfence_system();
                        for (int i = 0; i < P.nsig; ++i)
                            asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(P.sig[i]), "l"(P.sig_val)
                                         : "memory");
                    }
                }
            }
        }
    }
    __syncthreads();
    // mirrored rows reach the peer before the kernel completes (one cumulative
    // system fence per CTA after the barrier; a fence per thread costs ~10 %)
    if (P.nmir && threadIdx.x == 0) __threadfence_system();
    // launched as a programmatic dependent of the previous step's reduce_moments
    // (which triggers at its start): this grid does not complete before it
    asm volatile("griddepcontrol.wait;" ::: "memory");
    if (threadIdx.x == 0) {
        __threadfence();
        const unsigned done = atomicAdd(&P.counters[1], 1u);
        if (done == gridDim.x - 1) {
            P.counters[0] = 0;
            P.counters[1] = 0;
            P.counters[3] = 0;
            __threadfence();
        }
    }
}

// ---------------------------------------------------------------------------
// Chunk-staged kernel for narrow whole-row panels (n_b = 2, 4, 8, 12, 16): the same
// producer / consumer split as sell_b4_staged_kernel, but each stage holds
// G = 32 / LG consecutive chunks of a unit (records and staged U block columns
// of 4 rows x n_b; LG = 8 lanes per group for n_b <= 8, else 16), and a consumer
// warp takes block-row r of all G chunks at once, one LG-lane group per chunk
// (n_b of its lanes busy), and the gathers are bulk copies into shared memory
// instead of register loads.  Applies when every
// piece is a typed signature-1 chunk in one piece of at most kRecNarrow bytes
// and every chunk has a staging plan (periodic Topi lattices); otherwise the
// register-gather kernel runs.
constexpr int kRecNarrow = 4096;
// record slots 16 B apart from a multiple of 128: the G chunks' values that one
// warp-wide load reads land in different banks (4-way conflicts otherwise)
constexpr int kRecStride = kRecNarrow + 16;
template <int NBW>
struct NarrowLayout {
    static constexpr int LG = NBW <= 8 ? 8 : 16;  // lanes per chunk group (n_b = 2 / 4: 2 / 4 of 8, 12: 12 of 16 busy)
    static constexpr int G = 32 / LG;
    static constexpr size_t ublk = 4 * NBW * 16;                                   // one staged block column
    static constexpr size_t rec_off = 0;                                           // [2][G][kRecStride]
    static constexpr size_t ust_off = (rec_off + 2 * size_t(G) * kRecStride + 127) / 128 * 128;  // [2][G][kMaxStage][ublk]
    static constexpr size_t bar_off = ust_off + 2 * size_t(G) * kMaxStage * ublk;  // full_rec[2], full_u[2], empty[2]
    static constexpr size_t info_off = bar_off + 6 * 8;                            // int4[2]: unit, flags, chunks
    static constexpr size_t cnt_off = info_off + 2 * 16;
    static constexpr size_t red_off = (cnt_off + 16 + 127) / 128 * 128;
    static constexpr size_t total = red_off + 2 * kNW * 32 * 3 * 8;
};
static_assert(NarrowLayout<8>::total <= 227 * 1024 && NarrowLayout<12>::total <= 227 * 1024 &&
                  NarrowLayout<16>::total <= 227 * 1024,
              "narrow staged layout exceeds shared memory");

template <int MODE, int NBW>
__global__ void __launch_bounds__(32 * kStagedWarps, 1) sell_b4_narrow_kernel(const KParams P,
                                                                               const StagePlan* __restrict__ plans) {
    using L = NarrowLayout<NBW>;
    constexpr int G = L::G;
    extern __shared__ __align__(128) uint8_t smem[];
    uint64_t* full_rec = reinterpret_cast<uint64_t*>(smem + L::bar_off);
    uint64_t* full_u = full_rec + 2;
    uint64_t* empty = full_rec + 4;
    int4* info = reinterpret_cast<int4*>(smem + L::info_off);
    unsigned* unit_cnt = reinterpret_cast<unsigned*>(smem + L::cnt_off);
    double* red = reinterpret_cast<double*>(smem + L::red_off);
    const int cw = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int s = 0; s < 2; ++s) {
            mbar_init(&full_rec[s], 1);
            mbar_init(&full_u[s], 1);
            mbar_init(&empty[s], kNW);
        }
        unit_cnt[0] = unit_cnt[1] = 0;
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    if (cw == kNW) {
        // ---------------------------------------------------------- producer
        // per stage: the G records, then one bulk copy per run of each chunk's U
        // block columns; the next stage's piece entries (lane q: piece q) and plans
        // (word `lane` of each) are loaded one stage ahead, the next unit claimed
        // one unit ahead.
        const uint64_t ef = policy_evict_first();
        const unsigned full = 0xffffffffu;
        // unit blockIdx.x first, without a ticket (its piece range loads at once);
        // tickets then hand out units gridDim.x, gridDim.x + 1, ...
        auto claim = [&]() -> unsigned { return lane == 0 ? gridDim.x + atomicAdd(&P.counters[0], 1u) : 0u; };
        const uint2* plan_words = reinterpret_cast<const uint2*>(plans);
        int u = static_cast<int>(blockIdx.x);
        int p0 = 0, p1 = 0;
        if (u < P.num_units) {
            p0 = P.unit_piece[u];
            p1 = P.unit_piece[u + 1];
        }
        unsigned un_raw = claim();
        PieceInfo pin{0, 0, 0};
        uint2 pwn[G];
        auto load_group = [&](int pg, int pend) {
            if (lane < G && pg + lane < pend) pin = P.pieces[pg + lane];
#pragma unroll
            for (int q = 0; q < G; ++q)
                pwn[q] = pg + q < pend ? plan_words[static_cast<size_t>(pg + q) * 32 + lane] : make_uint2(0u, 0u);
        };
        if (u < P.num_units) load_group(p0, p1);
        // epilogue rows (W / Z, and X) of the chunks dpf stages ahead go to L2 by bulk
        // prefetches (as in the staged kernel): lane l holds the first block-row of
        // piece l of this unit (r0v) and of the next one (r0n)
        const int dpf = P.wpf & 15;
        int r0v = -1;
        if (dpf && u < P.num_units && p0 + lane < p1) r0v = P.piece_row0[p0 + lane];
        unsigned seq = 0;
        while (u < P.num_units) {
            const int un = static_cast<int>(__shfl_sync(full, un_raw, 0));
            int pn0 = 0, pn1 = 0, r0n = -1;
            if (un < P.num_units) {
                pn0 = P.unit_piece[un];
                pn1 = P.unit_piece[un + 1];
                if (dpf && pn0 + lane < pn1) r0n = P.piece_row0[pn0 + lane];
            }
            for (int pg = p0; pg < p1; pg += G) {
                const int slot = static_cast<int>(seq & 1u);
                const int nq = min(G, p1 - pg);
                if (dpf) {
                    const int t = pg + dpf * G + (lane & (G - 1));  // this unit's piece index (may run past p1)
                    const bool here = t < p1;
                    const int idx = here ? t - p0 : t - p1;
                    const int r0a = __shfl_sync(full, r0v, min(idx, 31)), r0b = __shfl_sync(full, r0n, min(idx, 31));
                    const int r0 = here ? r0a : r0b;
                    const bool ok = here ? idx < 32 : (un < P.num_units && pn0 + idx < pn1 && idx < 32);
                    if (lane < G && ok && r0 >= 0) {
                        const long long row0 = 4LL * r0, row1 = min(row0 + 4 * kC, P.n);
                        const unsigned nbytes = static_cast<unsigned>(max(row1 - row0, 0LL) * (NBW * 16));
                        if (nbytes) {
                            if (ModeT<MODE>::cheb) bulk_prefetch_l2(P.W + row0 * NBW, nbytes);
                            if (ModeT<MODE>::reads_z) bulk_prefetch_l2(P.Z + row0 * NBW, nbytes);
                            if (ModeT<MODE>::reads_x && (P.wpf & 16)) bulk_prefetch_l2(P.X + row0 * NBW, nbytes);
                        }
                    }
                }
                const PieceInfo pi = pin;
                uint2 pw[G];
#pragma unroll
                for (int q = 0; q < G; ++q) pw[q] = pwn[q];
                if (pg + G < p1) load_group(pg + G, p1);
                else if (un < P.num_units) load_group(pn0, pn1);
                // this stage's U copies (lane l < nruns of chunk q: run l)
                unsigned bytes[G];
                long long row0[G];
                int dst[G];
                unsigned tot_u = 0;
#pragma unroll
                for (int q = 0; q < G; ++q) {
                    const unsigned nruns = q < nq ? (__shfl_sync(full, pw[q].x, 0) & 0xffffu) : 0u;
                    const unsigned rb = __shfl_down_sync(full, pw[q].x, 1), rl = __shfl_down_sync(full, pw[q].y, 1);
                    bytes[q] = 0;
                    row0[q] = 0;
                    dst[q] = 0;
                    if (static_cast<unsigned>(lane) < nruns) {
                        const int bcol = static_cast<int>(rb);
                        row0[q] = 4LL * bcol;
                        const long long row1 = min(4LL * (bcol + static_cast<int>(rl & 0xffffu)), P.urows);
                        bytes[q] = static_cast<unsigned>(max(row1 - row0[q], 0LL) * (NBW * 16));
                        dst[q] = static_cast<int>(rl >> 16);
                    }
                    tot_u += bytes[q];
                }
                unsigned tot_rec = lane < nq ? pi.bytes : 0u;
#pragma unroll
                for (int off = 16; off > 0; off >>= 1) {
                    tot_u += __shfl_xor_sync(full, tot_u, off);
                    tot_rec += __shfl_xor_sync(full, tot_rec, off);
                }
                if (lane == 0) mbar_wait(&empty[slot], ((seq >> 1) & 1u) ^ 1u);
                __syncwarp();
                if (lane == 0) {
                    info[slot] = make_int4(u, pg + G >= p1 ? kInfoUnitLast : 0, nq, 0);
                    mbar_arrive_expect_tx(&full_rec[slot], tot_rec);
                    mbar_arrive_expect_tx(&full_u[slot], tot_u);
                }
                __syncwarp();
                if (lane < nq)
                    bulk_g2s_hint(smem + L::rec_off + (static_cast<size_t>(slot) * G + lane) * kRecStride,
                                  P.records + pi.offset, pi.bytes, &full_rec[slot], ef);
#pragma unroll
                for (int q = 0; q < G; ++q)
                    if (bytes[q])
                        bulk_g2s(smem + L::ust_off + ((static_cast<size_t>(slot) * G + q) * kMaxStage + dst[q]) * L::ublk,
                                 P.U + row0[q] * NBW, bytes[q], &full_u[slot]);
                ++seq;
            }
            u = un;
            p0 = pn0;
            p1 = pn1;
            r0v = r0n;
            if (u < P.num_units) un_raw = claim();
        }
        const int slot = static_cast<int>(seq & 1u);
        if (lane == 0) {
            mbar_wait(&empty[slot], ((seq >> 1) & 1u) ^ 1u);
            info[slot] = make_int4(-1, kInfoTerm, 0, 0);
            mbar_arrive(&full_rec[slot]);
        }
        __syncwarp();
    } else {
        // ---------------------------------------------------------- consumers
        const int r = cw;                           // block-row slot inside each chunk
        constexpr int LG = L::LG;
        const int qg = lane / LG, col = lane % LG;  // this lane's chunk of the stage, panel column
        double eta_x = 0.0, eta_y = 0.0, mu = 0.0;
        unsigned ub = 0;
        double2 wcur[4], xcur[4];
        auto block_row = [&](int slot, const int4& in) -> int {
            if ((in.y & kInfoTerm) || qg >= in.z || col >= NBW) return -1;
            return reinterpret_cast<const int32_t*>(smem + L::rec_off + (static_cast<size_t>(slot) * G + qg) * kRecStride +
                                                    16)[r];
        };
        mbar_wait(&full_rec[0], 0);
        int4 inf = info[0];
        int br = block_row(0, inf);
        prefetch_rows<MODE, NBW>(P, br, col, wcur, xcur);
        for (unsigned seq = 0; !(inf.y & kInfoTerm); ++seq) {
            const int slot = static_cast<int>(seq & 1u);
            const bool active = br >= 0;
            double2 acc[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) acc[q] = make_double2(0.0, 0.0);
            mbar_wait(&full_u[slot], (seq >> 1) & 1u);
            const double2* us = reinterpret_cast<const double2*>(smem + L::ust_off +
                                                                 (static_cast<size_t>(slot) * G + qg) * kMaxStage * L::ublk) +
                                col;
            double2 uo[4];
            if (active) {
                const uint8_t* base = smem + L::rec_off + (static_cast<size_t>(slot) * G + qg) * kRecStride;
                const PieceHdr* h = reinterpret_cast<const PieceHdr*>(base);
                const int kcnt = h->kcnt;
                const BlockMeta* meta = reinterpret_cast<const BlockMeta*>(base + 16 + 4 * kC + 16);
                const double* vals = reinterpret_cast<const double*>(meta + kcnt * kC);
                const uint8_t* sidx = base + sidx_offset(kC, kcnt, 0) + (8 * h->nvals + 15u) / 16 * 16;
                const double2* ob = us + static_cast<int>(sidx[kcnt * kC + r]) * (4 * NBW);
#pragma unroll
                for (int q = 0; q < 4; ++q) uo[q] = ob[q * NBW];
                walk_staged_topi_typed<NBW>(acc, sidx + r, us, vals + r * kSigTopiNnz);
            }
            const int4 icur = inf;
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[slot]);
            // next stage: its block-rows and epilogue operands.  By default after this
            // stage's epilogue, so that waiting for the next records overlaps the
            // stores (ko bit 256: before it, as the staged kernel does)
            const int nslot = slot ^ 1;
            double2 wnxt[4], xnxt[4];
            int br_next = -1;
            auto fetch_next = [&]() {
                mbar_wait(&full_rec[nslot], ((seq + 1) >> 1) & 1u);
                inf = info[nslot];
                br_next = block_row(nslot, inf);
                prefetch_rows<MODE, NBW>(P, br_next, col, wnxt, xnxt);
            };
            const bool early = (P.ko & 256) != 0;
            if (early) fetch_next();
            const bool mir_blk = block_mirrored(P, br);
            if (active) {
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const long long row = 4LL * br + q;
                    if (row >= P.n) continue;
                    const double2 u = uo[q];
                    double2 y;
                    y.x = fma(P.alpha, acc[q].x, P.beta * u.x);
                    y.y = fma(P.alpha, acc[q].y, P.beta * u.y);
                    if (MODE == M_SHIFT) {
                        st_out(P, row, col, y, mir_blk);
                    } else if (MODE == M_TWO_MINUS) {
                        st_out(P, row, col, make_double2(fma(2.0, y.x, -wcur[q].x), fma(2.0, y.y, -wcur[q].y)), mir_blk);
                    } else if (MODE == M_INIT) {
                        const double2 wn = make_double2(fma(2.0, y.x, -xcur[q].x), fma(2.0, y.y, -xcur[q].y));
                        st_out(P, row, col, wn, mir_blk);
                        double2 xn;
                        xn.x = fma(P.g2, wn.x, fma(P.g1, u.x, P.g0 * xcur[q].x));
                        xn.y = fma(P.g2, wn.y, fma(P.g1, u.y, P.g0 * xcur[q].y));
                        st_stream(P.X + row * NBW + col, xn);
                    } else {
                        const double2 wn = make_double2(fma(2.0, y.x, -wcur[q].x), fma(2.0, y.y, -wcur[q].y));
                        eta_x = fma(wn.x, u.x, eta_x);  // conj(w) * u
                        eta_x = fma(wn.y, u.y, eta_x);
                        eta_y = fma(wn.x, u.y, eta_y);
                        eta_y = fma(-wn.y, u.x, eta_y);
                        mu = fma(u.x, u.x, mu);
                        mu = fma(u.y, u.y, mu);
                        st_out(P, row, col, wn, mir_blk);
                        if (MODE == M_CHEB)
                            st_stream(P.X + row * NBW + col,
                                      make_double2(fma(P.gc, wn.x, xcur[q].x), fma(P.gc, wn.y, xcur[q].y)));
                        if (MODE == M_CHEB_X2)
                            st_stream(P.X + row * NBW + col,
                                      make_double2(fma(P.gc, wn.x, fma(P.gu, u.x, xcur[q].x)),
                                                   fma(P.gc, wn.y, fma(P.gu, u.y, xcur[q].y))));
                        if (MODE == M_CHEB_X3)
                            st_stream(P.X + row * NBW + col,
                                      make_double2(fma(P.gc, wn.x, fma(P.gu, u.x, fma(P.gw, wcur[q].x, xcur[q].x))),
                                                   fma(P.gc, wn.y, fma(P.gu, u.y, fma(P.gw, wcur[q].y, xcur[q].y)))));
                    }
                }
            }
            if (!early) fetch_next();
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                wcur[q] = wnxt[q];
                xcur[q] = xnxt[q];
            }
            br = br_next;
            if (ModeT<MODE>::cheb && (icur.y & kInfoUnitLast)) {
                // per-unit moments: the chunk groups of a warp (same column), then the
                // warps in fixed order by the last warp to arrive
#pragma unroll
                for (int off = LG; off < 32; off <<= 1) {
                    eta_x += __shfl_xor_sync(0xffffffffu, eta_x, off);
                    eta_y += __shfl_xor_sync(0xffffffffu, eta_y, off);
                    mu += __shfl_xor_sync(0xffffffffu, mu, off);
                }
                double* rb = red + static_cast<size_t>(ub) * kNW * 32 * 3;
                if (lane < NBW) {
                    rb[(cw * 32 + lane) * 3 + 0] = eta_x;
                    rb[(cw * 32 + lane) * 3 + 1] = eta_y;
                    rb[(cw * 32 + lane) * 3 + 2] = mu;
                }
                __threadfence_block();
                __syncwarp();
                unsigned last = 0;
                if (lane == 0) last = (atomicAdd(&unit_cnt[ub], 1u) == kNW - 1) ? 1u : 0u;
                last = __shfl_sync(0xffffffffu, last, 0);
                if (last) {
                    __threadfence_block();
                    if (lane < NBW) {
                        double sx = 0, sy = 0, sm = 0;
                        for (int w2 = 0; w2 < kNW; ++w2) {
                            sx += rb[(w2 * 32 + lane) * 3 + 0];
                            sy += rb[(w2 * 32 + lane) * 3 + 1];
                            sm += rb[(w2 * 32 + lane) * 3 + 2];
                        }
                        double* dst = P.partials + (static_cast<size_t>(icur.x) * 32 + lane) * 3;
                        dst[0] = sx;
                        dst[1] = sy;
                        dst[2] = sm;
                    }
                    __syncwarp();
                    if (lane == 0) {
                        unit_cnt[ub] = 0;
                        __threadfence_block();
                    }
                }
                ub ^= 1u;
                eta_x = eta_y = mu = 0.0;
            }
            if (P.nsig && (icur.y & kInfoUnitLast) && icur.x < P.nbnd) {
                __syncwarp();
                if (lane == 0) {
                    __threadfence_system();
                    if (atomicAdd(&P.counters[3], 1u) + 1u == static_cast<unsigned>(P.nbnd) * kNW) {
                        __threadfence_system();
                        for (int i = 0; i < P.nsig; ++i)
                            asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(P.sig[i]), "l"(P.sig_val)
                                         : "memory");
                    }
                }
            }
        }
    }
    __syncthreads();
    if (P.nmir && threadIdx.x == 0) __threadfence_system();
    asm volatile("griddepcontrol.wait;" ::: "memory");
    if (threadIdx.x == 0) {
        __threadfence();
        const unsigned done = atomicAdd(&P.counters[1], 1u);
        if (done == gridDim.x - 1) {
            P.counters[0] = 0;
            P.counters[1] = 0;
            P.counters[3] = 0;
            __threadfence();
        }
    }
}

// Sum the per-unit partials in a fixed order and add into the MomentSeries slots
// (kernels.hpp:199-202: out += partial).  96 values per unit (32 columns x
// {eta.re, eta.im, mu}); a block is 96 x kRedSplit threads, thread (t, s) sums
// every kRedSplit-th item of its range, then the kRedSplit sums are added in s
// order.  Level 1: block b sums a fixed contiguous range of units; level 2: the
// last block to finish sums the block partials the same way.  The order is fixed
// whichever block finishes last, and the dependent-add chains stay short (the
// tail is L2-latency-bound: one 96-thread chain over 256 partials took ~10 us).
constexpr int kRedBlocks = 256, kRedSplit = 8;
__device__ __forceinline__ double red_split_sum(const double* __restrict__ base, int count, int t, int s,
                                                double (*sh)[96]) {
    double acc = 0.0;
#pragma unroll 4
    for (int i = s; i < count; i += kRedSplit) acc += __ldcg(base + static_cast<size_t>(i) * 96 + t);
    sh[s][t] = acc;
    __syncthreads();
    double tot = 0.0;
    if (s == 0)
        for (int k = 0; k < kRedSplit; ++k) tot += sh[k][t];
    __syncthreads();
    return tot;
}
__global__ void __launch_bounds__(96 * kRedSplit) reduce_moments(const double* __restrict__ partials, int num_units,
                                                                 double* __restrict__ bpart, unsigned* __restrict__ ctr,
                                                                 int ncols, double* eta, double* mu) {
    __shared__ double sh[kRedSplit][96];
    __shared__ unsigned last;
    // the next step's kernel may start now: it does not read what this grid
    // writes (moments) nor write what it reads (partials are double-buffered)
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    const int t = threadIdx.x % 96, s = threadIdx.x / 96, nb = gridDim.x;
    const int u0 = static_cast<int>(static_cast<long long>(num_units) * blockIdx.x / nb);
    const int u1 = static_cast<int>(static_cast<long long>(num_units) * (blockIdx.x + 1) / nb);
    const double part = red_split_sum(partials + static_cast<size_t>(u0) * 96, u1 - u0, t, s, sh);
    if (s == 0) bpart[blockIdx.x * 96 + t] = part;
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) last = (atomicAdd(ctr, 1u) == static_cast<unsigned>(nb - 1));
    __syncthreads();
    if (!last) return;
    __threadfence();
    const double tot = red_split_sum(bpart, nb, t, s, sh);
    const int j = t / 3, q = t % 3;
    if (s == 0 && j < ncols) {
        if (q == 0) eta[2 * j] += tot;
        else if (q == 1) eta[2 * j + 1] += tot;
        else {
            mu[2 * j] += tot;
            mu[2 * j + 1] += 0.0;
        }
    }
    if (threadIdx.x == 0) *ctr = 0;
}

// ======================================================== host glue =====
void ck(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw CudaError(std::string(what) + ": " + cudaGetErrorString(e));
}

}  // namespace cfb


namespace cfb {

DeviceGuard::DeviceGuard(int dev) {
    ck(cudaGetDevice(&prev), "cudaGetDevice");
    if (prev != dev) ck(cudaSetDevice(dev), "cudaSetDevice");
}
DeviceGuard::~DeviceGuard() {
    int cur;
    if (cudaGetDevice(&cur) == cudaSuccess && cur != prev && prev >= 0) cudaSetDevice(prev);
}

static int sms_of(int dev) {
    int v = 0;
    ck(cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev), "cudaDeviceGetAttribute");
    return v;
}

// Narrow staged kernel's L2 prefetch of the epilogue rows, in stages ahead:
// CHEBFD_NPF or cf_tuning("npf", v); -1 (default) = 1 for n_b = 12 / 16 (two
// chunks per stage) outside the no-X-update mode, else 0.  Measured per mode (tools/step_modes.py, ms per step,
// off vs one stage ahead): n_b = 16 on the cfg2 lattice plain 2.37 vs 1.99, X3
// 2.50 vs 2.20, NOX 1.63 vs 1.64; n_b = 8 (four chunks per stage: the register
// prefetch of the next stage's rows has time to land) NOX 1.20 vs 1.28, plain
// 1.49 vs 1.46, and on the configs[0] lattice every mode slower with it.
static std::atomic<int> g_npf{-2};
static int narrow_prefetch(int nbw, bool nox) {
    int v = g_npf.load();
    if (v == -2) {
        const char* e = std::getenv("CHEBFD_NPF");
        v = e ? std::atoi(e) : -1;
        g_npf.store(v);
    }
    if (v >= 0) return std::min(v, 15);
    return nbw > 8 && !nox ? 1 : 0;
}

static void check_device(int dev) {
    int count = 0;
    cudaError_t e = cudaGetDeviceCount(&count);
    if (e != cudaSuccess || count == 0) throw CudaError("no CUDA device available (libchebfd_b200 has no CPU path)");
    if (dev < 0 || dev >= count) throw std::invalid_argument("device index out of range");
    int major = 0;
    ck(cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev), "cc");
    if (major != 10) throw CudaError("libchebfd_b200 is built for sm_100a (B200)");
}



// Kernel choice knob: CHEBFD_STAGED=0 (environment) or cf_tuning("staged", 0)
// disables the chunk-staged kernel (A/B comparisons in tests and tools).
static std::atomic<int> g_staged{-1};
static bool use_staged() {
    int v = g_staged.load();
    if (v < 0) {
        const char* e = std::getenv("CHEBFD_STAGED");
        v = (e && std::atoi(e) == 0) ? 0 : 1;
        g_staged.store(v);
    }
    return v != 0;
}

// Narrow staged kernel (n_b = 8 / 16 whole-row panels): CHEBFD_NARROW=0 or
// cf_tuning("narrow", 0) runs the register-gather kernel instead (A/B).
static std::atomic<int> g_narrow{-1};
static bool use_narrow() {
    int v = g_narrow.load();
    if (v < 0) {
        const char* e = std::getenv("CHEBFD_NARROW");
        v = (e && std::atoi(e) == 0) ? 0 : 1;
        g_narrow.store(v);
    }
    return v != 0;
}

// Typed records for the staged kernel: CHEBFD_TYPED=0 or cf_tuning("typed", 0)
// runs the full complex records instead (A/B).
static std::atomic<int> g_typed{-1};
static bool use_typed() {
    int v = g_typed.load();
    if (v < 0) {
        const char* e = std::getenv("CHEBFD_TYPED");
        v = (e && std::atoi(e) == 0) ? 0 : 1;
        g_typed.store(v);
    }
    return v != 0;
}

// Producer L2 prefetch of epilogue rows (KParams::wpf): default 2 pieces ahead,
// W and X rows (18).  The consumers' register loads one chunk ahead then hit L2:
// -5 % per fused step and per filter degree on cfg2 (tools/wpf_ab.py; 1-4 ahead,
// W only or W+X measured).  CHEBFD_WPF or cf_tuning("wpf", v); 0 = off.
static std::atomic<int> g_wpf{-1};
static int w_prefetch() {
    int v = g_wpf.load();
    if (v < 0) {
        const char* e = std::getenv("CHEBFD_WPF");
        v = e ? std::max(0, std::atoi(e)) : 18;
        g_wpf.store(v);
    }
    return v;
}

// Programmatic dependent launch of the step kernels (CHEBFD_PDL=0 or
// cf_tuning("pdl", 0) disables): a step's grid may start while the previous
// step's reduce_moments runs; it waits for it (griddepcontrol.wait) only at exit.
// Only a launch whose stream predecessor is this library's reduce_moments gets
// the attribute (`pdl` below): reduce_moments triggers its dependents explicitly
// and writes nothing a step reads, and it was itself launched with full stream
// serialisation after the step that produced U / W / X, so those writes are
// complete and visible.  Any other predecessor (M_SHIFT -> M_INIT, M_INIT -> the
// first degree step, a caller's kernel between two API calls) triggers only
// implicitly at its exit, which does not make its writes visible before the
// dependent's griddepcontrol.wait -- such launches are plain stream-ordered.
static std::atomic<int> g_pdl{-1};
static bool use_pdl() {
    int v = g_pdl.load();
    if (v < 0) {
        const char* e = std::getenv("CHEBFD_PDL");
        v = (e && std::atoi(e) == 0) ? 0 : 1;
        g_pdl.store(v);
    }
    return v != 0;
}
template <class... KArgs, class... Args>
static void launch_pdl(void (*kern)(KArgs...), int grid, int block, std::size_t smem, cudaStream_t st, bool pdl,
                       Args... args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(block);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = (pdl && use_pdl()) ? 1 : 0;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    ck(cudaLaunchKernelEx(&cfg, kern, args...), "kernel launch");
}

// Full complex records are dropped from the device when typed records exist
// (they would cost ~1 GB per 8.4M rows next to the typed copy); an A/B run with
// typed records off uploads them again from the host copy.
static void ensure_full_records(cf_matrix m) {
    if (m->d_records || m->h_records.empty()) return;
    DeviceGuard dg(m->device);
    ck(cudaMalloc(&m->d_records, m->h_records.size()), "cudaMalloc records");
    ck(cudaMemcpy(m->d_records, m->h_records.data(), m->h_records.size(), cudaMemcpyHostToDevice), "upload records");
}

template <int MODE>
static void launch_mode(cf_matrix m, KParams& P, cudaStream_t st, bool pdl) {
    if (m->d_trecords && use_typed()) {
        P.records = m->d_trecords;
        P.pieces = m->d_tpieces;
        P.typed = 1;
    } else if (!m->d_records) {
        ensure_full_records(m);
        P.records = m->d_records;
    }
    if (m->d_plans && P.ld == 32 && P.ncols == 32 && use_staged()) {
        auto kern = sell_b4_staged_kernel<MODE>;
        ck(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                static_cast<int>(StagedLayout::total)),
           "cudaFuncSetAttribute");
        const int grid = std::max(1, std::min(m->num_units, sms_of(m->device)));
        launch_pdl(kern, grid, 32 * kStagedWarps, StagedLayout::total, st, pdl, P,
                   static_cast<const StagePlan*>(m->d_plans));
        return;
    }
    if (P.typed && m->narrow_ok && m->d_plans && P.ld == P.ncols &&
        (P.ld == 2 || P.ld == 4 || P.ld == 8 || P.ld == 12 || P.ld == 16) &&
        use_staged() &&
        use_narrow()) {
        const int grid = std::max(1, std::min(m->num_units, sms_of(m->device)));
        P.wpf = (P.wpf & 16) | narrow_prefetch(static_cast<int>(P.ld), MODE == M_CHEB_NOX);
        auto gon = [&](auto kern, std::size_t smem) {
            ck(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)),
               "cudaFuncSetAttribute");
            launch_pdl(kern, grid, 32 * kStagedWarps, smem, st, pdl, P, static_cast<const StagePlan*>(m->d_plans));
        };
        if (P.ld == 2) gon(sell_b4_narrow_kernel<MODE, 2>, NarrowLayout<2>::total);
        else if (P.ld == 4) gon(sell_b4_narrow_kernel<MODE, 4>, NarrowLayout<4>::total);
        else if (P.ld == 8) gon(sell_b4_narrow_kernel<MODE, 8>, NarrowLayout<8>::total);
        else if (P.ld == 12) gon(sell_b4_narrow_kernel<MODE, 12>, NarrowLayout<12>::total);
        else gon(sell_b4_narrow_kernel<MODE, 16>, NarrowLayout<16>::total);
        return;
    }
    int lpr = P.ncols <= 4 ? 4 : P.ncols <= 8 ? 8 : P.ncols <= 16 ? 16 : 32;
    dim3 block(32 * kNW);
    auto go = [&](auto kern) {
        ck(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(SmemLayout::total)),
           "cudaFuncSetAttribute");
        launch_pdl(kern, m->grid, static_cast<int>(block.x), SmemLayout::total, st, pdl, P);
    };
    if (P.ncols != P.ld) {
        go(sell_b4_kernel<MODE, 32, 3, false>);  // column slice of a wider panel: rows staged one by one
    } else {
        switch (lpr) {
            case 4: go(sell_b4_kernel<MODE, 4, 3, true>); break;
            case 8: go(sell_b4_kernel<MODE, 8, 3, true>); break;
            case 16: go(sell_b4_kernel<MODE, 16, 3, true>); break;
            default: go(sell_b4_kernel<MODE, 32, 3, true>); break;
        }
    }
    ck(cudaGetLastError(), "kernel launch");
}

static std::atomic<int> g_ko{0};
// L2 prefetch distance of the generic-block walk: CHEBFD_GPF or cf_tuning("gpf", v); 0 = off.
static std::atomic<int> g_gpf{-1};
static int g_prefetch() {
    int v = g_gpf.load();
    if (v < 0) {
        const char* e = std::getenv("CHEBFD_GPF");
        v = e ? std::max(0, std::atoi(e)) : 4;
        g_gpf.store(v);
    }
    return v;
}
static KParams base_params(cf_matrix m) {
    KParams P{};
    P.ko = g_ko.load();
    P.gpf = g_prefetch();
    P.records = m->d_records;
    P.pieces = m->d_pieces;
    P.unit_piece = m->d_units;
    P.num_units = m->num_units;
    P.n = static_cast<long long>(m->n);
    P.urows = static_cast<long long>(m->ncols);
    P.partials = m->d_partials;
    P.piece_row0 = m->d_row0;
    P.wpf = w_prefetch();
    P.counters = m->d_counters;
    return P;
}

// Run one mode over all 32-column slices of an ld-wide panel.  `after_reduce`:
// the last launch on `st` was this matrix's reduce_moments (see use_pdl).
template <int MODE>
static void run(cf_matrix m, KParams P, std::size_t ld, std::size_t ncols, cudaStream_t st, double* eta = nullptr,
                double* mu = nullptr, bool after_reduce = false) {
    if (ncols == 0 || ncols > ld) throw std::invalid_argument("spmmv: block width mismatch");
    DeviceGuard dg(m->device);
    P.ld = static_cast<long long>(ld);
    const double2* U0 = P.U;
    double2 *W0 = P.W, *X0 = P.X;
    const double2* Z0 = P.Z;
    double2* M0[kMaxMirror];
    for (int q = 0; q < kMaxMirror; ++q) M0[q] = P.mir[q].dst;
    for (std::size_t c0 = 0; c0 < ncols; c0 += 32) {
        P.ncols = static_cast<int>(std::min<std::size_t>(32, ncols - c0));
        P.U = U0 ? U0 + c0 : nullptr;
        P.W = W0 ? W0 + c0 : nullptr;
        P.X = X0 ? X0 + c0 : nullptr;
        P.Z = Z0 ? Z0 + c0 : nullptr;
        for (int q = 0; q < P.nmir; ++q) P.mir[q].dst = M0[q] + c0;
        // unit partials alternate between two buffers: a step's kernel may run
        // while the previous step's reduce_moments still reads the other one
        double* part = m->d_partials + static_cast<std::size_t>(m->part_sel) * m->num_units * 96;
        if (ModeT<MODE>::cheb) {
            P.partials = part;
            m->part_sel ^= 1;
        }
        launch_mode<MODE>(m, P, st, after_reduce);
        after_reduce = false;
        if (ModeT<MODE>::cheb) {
            // ~32 units per level-1 block, at most kRedBlocks
            const int rb = std::max(1, std::min(kRedBlocks, (m->num_units + 31) / 32));
            reduce_moments<<<rb, 96 * kRedSplit, 0, st>>>(part, m->num_units, m->d_bpart, m->d_counters + 2, P.ncols,
                                                          eta + 2 * c0, mu + 2 * c0);
            ck(cudaGetLastError(), "reduce_moments launch");
            after_reduce = true;
        }
    }
}

// Typed copy of the records for both kernels.  Every piece that is a
// signature-1 chunk whose block-rows, with blocks of equal pattern ordered by
// value type and then column, match kSigTopiTypes (Topi lattices: hops are
// (t/2)(B +- i alpha_d), each entry real or imaginary; on-site terms real, so
// onsite disorder keeps it) is stored typed: each value keeps only its nonzero
// component, tagged kPieceTyped.  The kernels then do 2 FMAs per entry instead
// of 4 and stream 8 bytes per value instead of 16.  Other pieces (an open
// lattice's surface chunks, general sparsity) are copied verbatim into the same
// stream, so one matrix mixes both.  Each product is the same; blocks of one
// pattern are summed in value-type order rather than column order, so results
// differ from the full records at rounding level (tests: 1e-13).  Matrices
// without a single typed piece keep only the full records.
static bool type_piece(const uint8_t* src, uint8_t* dst) {
    constexpr int voff[kSigTopiBlocks] = {0, 4, 12, 20, 28, 36, 44};
    constexpr int nnz[kSigTopiBlocks] = {4, 8, 8, 8, 8, 8, 8};
    const PieceHdr* h = reinterpret_cast<const PieceHdr*>(src);
    const std::size_t head = sidx_offset(kC, h->kcnt, 0), nv = h->nvals;
    const std::size_t vbytes = (8 * nv + 15) / 16 * 16, sbytes = static_cast<std::size_t>(h->kcnt + 1) * kC;
    std::memcpy(dst, src, head);
    reinterpret_cast<PieceHdr*>(dst)->flags = static_cast<uint16_t>(h->flags | kPieceTyped);
    const BlockMeta* meta = reinterpret_cast<const BlockMeta*>(src + 16 + 4 * kC + (2 * kC + 15) / 16 * 16);
    BlockMeta* tmeta = reinterpret_cast<BlockMeta*>(dst + 16 + 4 * kC + (2 * kC + 15) / 16 * 16);
    const double* vals = reinterpret_cast<const double*>(src + head);
    double* tvals = reinterpret_cast<double*>(dst + head);
    const uint8_t* sidx = src + sidx_offset(kC, h->kcnt, nv);
    uint8_t* tsidx = dst + head + vbytes;
    std::memcpy(tsidx, sidx, sbytes);  // own-row entries (k = kcnt) unchanged
    for (int r = 0; r < kC; ++r) {
        const double* sv = vals + 2 * static_cast<std::size_t>(r) * kSigTopiNnz;
        unsigned types[kSigTopiBlocks];
        for (int k = 0; k < kSigTopiBlocks; ++k) {
            types[k] = 0;
            for (int j = 0; j < nnz[k]; ++j) {
                const double re = sv[2 * (voff[k] + j)], im = sv[2 * (voff[k] + j) + 1];
                if (re != 0.0 && im != 0.0) return false;  // a genuinely complex entry
                if (re == 0.0 && im != 0.0) types[k] |= 1u << j;
            }
        }
        // blocks of one pattern: by value type (imaginary-first pattern), then column
        int ix[kSigTopiBlocks];
        std::iota(ix, ix + kSigTopiBlocks, 0);
        std::stable_sort(ix, ix + kSigTopiBlocks, [&](int a, int b) {
            const BlockMeta &ma = meta[a * kC + r], &mb = meta[b * kC + r];
            if (ma.mask != mb.mask) return ma.mask < mb.mask;
            return types[a] > types[b];
        });
        for (int k = 0; k < kSigTopiBlocks; ++k) {
            const int o = ix[k];
            if (meta[o * kC + r].mask != kSigTopiMasks[k] || types[o] != kSigTopiTypes[k]) return false;
            tmeta[k * kC + r] = meta[o * kC + r];
            tsidx[k * kC + r] = sidx[o * kC + r];
            for (int j = 0; j < nnz[k]; ++j) {
                const double re = sv[2 * (voff[o] + j)], im = sv[2 * (voff[o] + j) + 1];
                tvals[static_cast<std::size_t>(r) * kSigTopiNnz + voff[k] + j] = (types[o] >> j & 1u) ? im : re;
            }
        }
    }
    return true;
}

static void build_typed_records(cf_matrix m, const SellHost& s) {
    std::vector<uint8_t> rec;
    std::vector<PieceInfo> pcs;
    rec.reserve(s.records.size() / 2 + 16);
    std::size_t ntyped = 0;
    for (const PieceInfo& pi : s.pieces) {
        const uint8_t* src = s.records.data() + pi.offset;
        const PieceHdr* h = reinterpret_cast<const PieceHdr*>(src);
        const std::size_t off = rec.size();
        bool typed = false;
        if ((h->flags >> kSigShift) == 1 && h->kcnt == kSigTopiBlocks &&
            h->nvals == static_cast<uint32_t>(kC * kSigTopiNnz)) {
            const std::size_t head = sidx_offset(kC, h->kcnt, 0), nv = h->nvals;
            const std::size_t vbytes = (8 * nv + 15) / 16 * 16, sbytes = static_cast<std::size_t>(h->kcnt + 1) * kC;
            const std::size_t bytes = (head + vbytes + sbytes + 15) / 16 * 16;
            rec.resize(off + bytes, 0);
            typed = type_piece(src, rec.data() + off);
            if (typed) {
                pcs.push_back({off, static_cast<uint32_t>(bytes), pi.flags});
                ++ntyped;
            } else {
                rec.resize(off);
            }
        }
        if (!typed) {  // verbatim
            rec.insert(rec.end(), src, src + pi.bytes);
            pcs.push_back({off, pi.bytes, pi.flags});
        }
    }
    if (ntyped == 0) return;
    // the narrow staged kernel: every piece a typed whole chunk of at most kRecNarrow bytes
    m->narrow_ok = ntyped == s.pieces.size();
    for (std::size_t i = 0; i < pcs.size() && m->narrow_ok; ++i)
        m->narrow_ok = pcs[i].bytes <= static_cast<uint32_t>(kRecNarrow) &&
                       (s.pieces[i].flags & (kPieceFirst | kPieceLast)) == (kPieceFirst | kPieceLast);
    ck(cudaMalloc(&m->d_trecords, rec.size()), "cudaMalloc typed records");
    ck(cudaMemcpy(m->d_trecords, rec.data(), rec.size(), cudaMemcpyHostToDevice), "upload typed records");
    ck(cudaMalloc(&m->d_tpieces, pcs.size() * sizeof(PieceInfo)), "cudaMalloc typed pieces");
    ck(cudaMemcpy(m->d_tpieces, pcs.data(), pcs.size() * sizeof(PieceInfo), cudaMemcpyHostToDevice),
       "upload typed pieces");
    m->typed_bytes = rec.size() + pcs.size() * sizeof(PieceInfo);
    m->typed_pieces = ntyped;
}

static void upload(cf_matrix m, const SellHost& s) {
    DeviceGuard dg(m->device);
    m->n = s.n;
    m->ncols = s.ncols;
    m->nnz = s.nnz;
    m->nbr = s.nbr;
    m->C = s.C;
    m->num_units = static_cast<int>(s.unit_piece.size()) - 1;
    m->record_bytes = s.records.size();
    m->npieces = s.pieces.size();
    m->pieces = s.pieces;
    m->rows_alloc = s.ncols;  // kernels touch U rows < ncols and W/X rows < n only
    ck(cudaMalloc(&m->d_records, s.records.size()), "cudaMalloc records");
    ck(cudaMemcpy(m->d_records, s.records.data(), s.records.size(), cudaMemcpyHostToDevice), "upload records");
    ck(cudaMalloc(&m->d_pieces, s.pieces.size() * sizeof(PieceInfo)), "cudaMalloc pieces");
    ck(cudaMemcpy(m->d_pieces, s.pieces.data(), s.pieces.size() * sizeof(PieceInfo), cudaMemcpyHostToDevice),
       "upload pieces");
    {
        std::vector<int32_t> row0(s.pieces.size(), -1);
        for (std::size_t p = 0; p < s.pieces.size(); ++p) {
            const int32_t* perm = reinterpret_cast<const int32_t*>(s.records.data() + s.pieces[p].offset + 16);
            bool run = perm[0] >= 0;
            for (int r = 1; r < kC && run; ++r) run = perm[r] == perm[0] + r;
            if (run) row0[p] = perm[0];
        }
        ck(cudaMalloc(&m->d_row0, row0.size() * 4), "cudaMalloc piece rows");
        ck(cudaMemcpy(m->d_row0, row0.data(), row0.size() * 4, cudaMemcpyHostToDevice), "upload piece rows");
    }
    if (s.staged) build_typed_records(m, s);
    const char* keep = std::getenv("CHEBFD_KEEP_FULL_RECORDS");
    if (m->d_trecords && !(keep && std::atoi(keep) != 0)) {
        // typed records run every kernel of this matrix: keep the full ones on the host
        m->h_records = s.records;
        ck(cudaFree(m->d_records), "cudaFree records");
        m->d_records = nullptr;
    }
    m->unit_br_lo.assign(m->num_units, INT32_MAX);
    m->unit_br_hi.assign(m->num_units, -1);
    for (int u = 0; u < m->num_units; ++u)
        for (int p = s.unit_piece[u]; p < s.unit_piece[u + 1]; ++p) {
            const int32_t* perm = reinterpret_cast<const int32_t*>(s.records.data() + s.pieces[p].offset + 16);
            for (int r = 0; r < kC; ++r)
                if (perm[r] >= 0) {
                    m->unit_br_lo[u] = std::min(m->unit_br_lo[u], perm[r]);
                    m->unit_br_hi[u] = std::max(m->unit_br_hi[u], perm[r]);
                }
        }
    ck(cudaMalloc(&m->d_units, s.unit_piece.size() * 4), "cudaMalloc units");
    ck(cudaMemcpy(m->d_units, s.unit_piece.data(), s.unit_piece.size() * 4, cudaMemcpyHostToDevice), "upload units");
    ck(cudaMalloc(&m->d_partials, 2 * static_cast<std::size_t>(m->num_units) * 32 * 3 * 8), "cudaMalloc partials");
    ck(cudaMemset(m->d_partials, 0, 2 * static_cast<std::size_t>(m->num_units) * 32 * 3 * 8), "memset partials");
    ck(cudaMalloc(&m->d_counters, 4 * sizeof(unsigned)), "cudaMalloc counters");
    ck(cudaMemset(m->d_counters, 0, 4 * sizeof(unsigned)), "memset counters");
    ck(cudaMalloc(&m->d_bpart, kRedBlocks * 96 * sizeof(double)), "cudaMalloc bpart");
    if (s.staged) {
        ck(cudaMalloc(&m->d_plans, s.plans.size() * sizeof(StagePlan)), "cudaMalloc plans");
        ck(cudaMemcpy(m->d_plans, s.plans.data(), s.plans.size() * sizeof(StagePlan), cudaMemcpyHostToDevice),
           "upload plans");
    }
    m->device_bytes = (m->d_records ? s.records.size() : 0) + s.pieces.size() * sizeof(PieceInfo) +
                      s.unit_piece.size() * 4 +
                      2 * static_cast<std::size_t>(m->num_units) * 32 * 3 * 8 + s.plans.size() * sizeof(StagePlan) +
                      m->typed_bytes;
    int per_sm = 0;
    ck(cudaFuncSetAttribute(sell_b4_kernel<M_CHEB, 32, 3, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            static_cast<int>(SmemLayout::total)),
       "cudaFuncSetAttribute");
    ck(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, sell_b4_kernel<M_CHEB, 32, 3, true>, 32 * kNW,
                                                     SmemLayout::total),
       "occupancy");
    per_sm = std::max(per_sm, 1);
    // the zero-fills above ran on the legacy stream: complete them before any
    // caller stream (possibly non-blocking) launches on this matrix
    ck(cudaDeviceSynchronize(), "upload sync");
    if (const char* e = std::getenv("CHEBFD_CTAS_PER_SM")) per_sm = std::max(1, std::min(per_sm, std::atoi(e)));
    m->grid = std::max(1, std::min(m->num_units, per_sm * sms_of(m->device)));
}

// Boundary rows [0, lo) and [n - hi, n) (a z-slab shard's first and last planes):
// the number of leading work units up to the last one whose block-row range meets
// them (a superset of the boundary units only makes the early flag later).
static void set_boundary(cf_matrix m, std::size_t lo, std::size_t hi) {
    if (lo > m->n || hi > m->n) throw std::invalid_argument("boundary rows outside the matrix");
    const long long blo = static_cast<long long>((lo + 3) / 4), bhi = static_cast<long long>((m->n - hi) / 4);
    int last = -1;
    for (int u = 0; u < m->num_units; ++u)
        if (m->unit_br_hi[u] >= 0 && (m->unit_br_lo[u] < blo || m->unit_br_hi[u] >= bhi)) last = u;
    m->bnd_units = last + 1;
}

static cf_matrix create_from_crs(int device, std::size_t n, std::size_t ncols, const uint64_t* rp, const int32_t* ci,
                                 const double* v, const int32_t* order, int C, int sigma) {
    check_device(device);
    if (C != 0 && C != kC) throw std::invalid_argument("device kernels are built for C == 8");
    SellHost s = build_sell(n, ncols, rp, ci, v, order, kC, sigma, static_cast<std::size_t>(2 * sms_of(device)));
    cf_matrix m = new cf_matrix_s();
    m->device = device;
    check(cf_gershgorin_bounds(n, rp, ci, v, &m->gersh_lo, &m->gersh_hi));
    try {
        upload(m, s);
    } catch (...) {
        cf_matrix_destroy(m);
        throw;
    }
    return m;
}

// Pre-flight HBM budget: a workspace that cannot fit raises std::invalid_argument
// (CF_EINVAL, ValueError in Python) naming the sizes, never an allocator OOM
// half-way through a filter.  `grow` = bytes about to be allocated beyond what
// the handle already holds (its old buffer is released first).
static void hbm_budget(std::size_t grow, const char* what) {
    std::size_t fr = 0, tot = 0;
    ck(cudaMemGetInfo(&fr, &tot), "cudaMemGetInfo");
    if (grow > fr) {
        char msg[256];
        std::snprintf(msg, sizeof msg, "%s: needs %.2f GB more device memory, %.2f GB free of %.2f GB", what,
                      grow / 1e9, fr / 1e9, tot / 1e9);
        throw std::invalid_argument(msg);
    }
}

// Grown on the caller's stream: the zero-fill must order with the filter's kernels
// when that stream does not synchronise with the legacy one.
static void* ensure_scratch(cf_matrix m, std::size_t bytes, cudaStream_t st) {
    if (m->scratch_bytes < bytes) {
        hbm_budget(bytes - m->scratch_bytes, "apply_filter U/W panels");
        if (m->scratch) cudaFree(m->scratch);
        m->scratch = nullptr;
        m->scratch_bytes = 0;
        ck(cudaMalloc(&m->scratch, bytes), "cudaMalloc scratch");
        ck(cudaMemsetAsync(m->scratch, 0, bytes, st), "memset scratch");
        m->scratch_bytes = bytes;
    }
    return m->scratch;
}

// Degrees per X update in apply_filter: 3 (default), 2, or 1 (every step, the
// ref's own schedule).  CHEBFD_X_GROUP=1|2|3 (CHEBFD_PAIR_X=0 == 1) or
// cf_tuning("x_group", v) for A/B runs and tests.
static std::atomic<int> g_x_group{-1};
static int x_group() {
    int v = g_x_group.load();
    if (v < 0) {
        if (const char* e = std::getenv("CHEBFD_X_GROUP")) {
            v = std::max(1, std::min(3, std::atoi(e)));
        } else {
            const char* e2 = std::getenv("CHEBFD_PAIR_X");
            v = (e2 && std::atoi(e2) == 0) ? 1 : 3;
        }
        g_x_group.store(v);
    }
    return v;
}

// Degree loop of Alg. 2 (filter.hpp:87-91) as a list of kernel steps.  X enters
// only as the running sum sum_p g_p c_p T_p, so steps go in groups of three: two
// skip the X update, the third applies all three, x += g_p c_p T_p + g_{p+1}
// c_{p+1} T_{p+1} + g_{p+2} c_{p+2} T_{p+2} (T_p is that step's W read, T_{p+1}
// its U), so X is read and written once per three degrees.  Remainders use a
// pair (NOX + X2) or a plain step.
struct DegreeStep {
    std::size_t p;
    int mode;
    double gw, gu, gc;
};
static std::vector<DegreeStep> degree_schedule(std::size_t np, const double* c, const double* g) {
    const std::size_t grp = static_cast<std::size_t>(x_group());
    auto gcoef = [&](std::size_t q) { return g[q] * c[q]; };
    std::vector<DegreeStep> out;
    for (std::size_t p = 3; p <= np;) {
        const std::size_t left = np - p + 1;
        if (grp >= 3 && left >= 3) {
            out.push_back({p, M_CHEB_NOX, 0, 0, 0});
            out.push_back({p + 1, M_CHEB_NOX, 0, 0, 0});
            out.push_back({p + 2, M_CHEB_X3, gcoef(p), gcoef(p + 1), gcoef(p + 2)});
            p += 3;
        } else if (grp >= 2 && left >= 2) {
            out.push_back({p, M_CHEB_NOX, 0, 0, 0});
            out.push_back({p + 1, M_CHEB_X2, 0, gcoef(p), gcoef(p + 1)});
            p += 2;
        } else {
            out.push_back({p, M_CHEB, 0, 0, gcoef(p)});
            p += 1;
        }
    }
    return out;
}

// One degree step on a panel: Q carries U, W, X (and mirrors); moments to eta/mu.
static void run_degree(cf_matrix m, KParams& Q, const DegreeStep& d, std::size_t nb, cudaStream_t st, double* eta,
                       double* mu, bool after_reduce = false) {
    Q.gw = d.gw;
    Q.gu = d.gu;
    Q.gc = d.gc;
    switch (d.mode) {
        case M_CHEB_NOX: run<M_CHEB_NOX>(m, Q, nb, nb, st, eta, mu, after_reduce); break;
        case M_CHEB_X2: run<M_CHEB_X2>(m, Q, nb, nb, st, eta, mu, after_reduce); break;
        case M_CHEB_X3: run<M_CHEB_X3>(m, Q, nb, nb, st, eta, mu, after_reduce); break;
        default: run<M_CHEB>(m, Q, nb, nb, st, eta, mu, after_reduce); break;
    }
}

// One panel of Alg. 2 (filter.hpp:81-91): cheb_init and the degree loop on panel
// b of an n_s-column block vector; moments go to columns b*nb.. of the series.
static void filter_panel(cf_matrix m, double2* Xb, std::size_t b, std::size_t ns, std::size_t nb, std::size_t np,
                         const double* c, const double* g, double alpha, double beta, double* eta, double* mu,
                         cudaStream_t st) {
    const std::size_t rows = m->rows_alloc;
    double2* scratch = static_cast<double2*>(ensure_scratch(m, 2 * rows * nb * sizeof(double2), st));
    double2* U = scratch;
    double2* W = scratch + rows * nb;
    KParams P = base_params(m);
    P.alpha = alpha;
    P.beta = beta;
    // cheb_init (kernels.hpp:133-152): U = (aH+b)X0, then the fused two-minus + axpby
    P.U = Xb;
    P.W = U;
    run<M_SHIFT>(m, P, nb, nb, st);
    P = base_params(m);
    P.alpha = alpha;
    P.beta = beta;
    P.U = U;
    P.W = W;
    P.X = Xb;
    P.g0 = g[0] * c[0];
    P.g1 = g[1] * c[1];
    P.g2 = g[2] * c[2];
    run<M_INIT>(m, P, nb, nb, st);
    bool after_reduce = false;  // the first degree step follows M_INIT
    for (const DegreeStep& d : degree_schedule(np, c, g)) {
        std::swap(U, W);  // swap_blocks(W, U) (filter.hpp:88)
        KParams Q = base_params(m);
        Q.alpha = alpha;
        Q.beta = beta;
        Q.X = Xb;
        Q.U = U;
        Q.W = W;
        const std::size_t slot = (d.p - 3) * ns + b * nb;
        run_degree(m, Q, d, nb, st, eta + 2 * slot, mu + 2 * slot, after_reduce);
        after_reduce = true;
    }
}

// Columns [c0, c0 + 32) of an n_s-column block vector held in n_b-wide panels
// (n_b < 32) <-> one 32-wide panel (rows [0, n)): wide[i][j] = column c0 + j, in
// panel (c0 + j) / n_b; src.p[k] is panel c0 / n_b + k.  A panel that straddles
// two slices (n_b not dividing 32) is packed / unpacked column by column.
struct NarrowPanels {
    double2* p[32];
};
__global__ void pack_wide(NarrowPanels src, int nb, int c0, double2* __restrict__ wide, long long n, int unpack) {
    const long long tot = n * 32;
    const int k0 = c0 / nb;
    for (long long t = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; t < tot;
         t += static_cast<long long>(gridDim.x) * blockDim.x) {
        const long long i = t >> 5;
        const int gc = c0 + static_cast<int>(t & 31);
        double2* narrow = src.p[gc / nb - k0] + i * nb + (gc % nb);
        if (unpack) *narrow = wide[t];
        else wide[t] = *narrow;
    }
}

// Columns [c0, c0 + 32) of an ld-wide panel <-> a 32-wide panel (rows [0, n)).
__global__ void slice_wide(double2* __restrict__ src, int ld, int c0, double2* __restrict__ wide, long long n,
                           int unpack) {
    const long long tot = n * 32;
    for (long long t = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; t < tot;
         t += static_cast<long long>(gridDim.x) * blockDim.x) {
        double2* sp = src + (t >> 5) * ld + c0 + (t & 31);
        if (unpack) *sp = wide[t];
        else wide[t] = *sp;
    }
}

// Narrow panels (n_b < 32, n_s a multiple of 32) filtered as 32-wide panels: the
// matrix is read once per 32 columns instead of once per n_b, all 32 lanes of a
// column group are busy (n_b = 12 would run 16-lane groups), and the chunk-staged
// kernel runs.  The columns and their moments are the same; each panel's filter is
// the same arithmetic per column (rounding-level differences only through the
// kernel's summation order).  Panels wider than 32 (n_b = 64, ...) are filtered one
// 32-column slice at a time the same way (instead of the register-gather kernel's
// strided slices).  Needs one extra n x 32 panel (kept with the matrix, like
// the U/W scratch) and 32-wide U/W scratch; CHEBFD_FILTER_WIDE=0 or a full device
// keeps the panel-by-panel loop.
// The matrix's 32-wide panel for filter_wide (allocated once), or null when the
// filter cannot run wide here: CHEBFD_FILTER_WIDE=0, no staging plans / staged
// kernel, a shard (ncols != n), or not enough device memory (1 GB margin kept).
static double2* wide_panel(cf_matrix m) {
    static const bool on = [] {
        const char* e = std::getenv("CHEBFD_FILTER_WIDE");
        return !(e && std::atoi(e) == 0);
    }();
    if (!on || !m->d_plans || !use_staged() || m->ncols != m->n) return nullptr;
    const std::size_t wide_bytes = m->n * 32 * sizeof(double2);
    const std::size_t uw = 2 * m->rows_alloc * 32 * sizeof(double2);
    if (m->wide_bytes < wide_bytes) {
        std::size_t fr = 0, tot = 0;
        ck(cudaMemGetInfo(&fr, &tot), "cudaMemGetInfo");
        const std::size_t grow = wide_bytes + (m->scratch_bytes < uw ? uw - m->scratch_bytes : 0);
        if (grow + (std::size_t{1} << 30) > fr) return nullptr;
        if (m->wide) cudaFree(m->wide);
        m->wide = nullptr;
        m->wide_bytes = 0;
        ck(cudaMalloc(&m->wide, wide_bytes), "cudaMalloc wide panel");
        m->wide_bytes = wide_bytes;
    }
    return static_cast<double2*>(m->wide);
}

static int pack_blocks(cf_matrix m) {
    return static_cast<int>(std::min<long long>((static_cast<long long>(m->n) * 32 + 255) / 256,
                                                8LL * sms_of(m->device)));
}

// Columns [32 w, 32 w + 32) of n_s = npanels * n_b (n_b < 32): packed into the wide
// panel, filtered by the staged kernel, unpacked (moments to the same columns).
static void filter_slice_wide(cf_matrix m, double2* const* panels, std::size_t w, std::size_t ns, std::size_t nb,
                              std::size_t np, const double* c, const double* g, double alpha, double beta, double* eta,
                              double* mu, cudaStream_t st) {
    double2* const wp = static_cast<double2*>(m->wide);
    const int blocks = pack_blocks(m);
    const std::size_t c0 = 32 * w, k0 = c0 / nb, k1 = (c0 + 31) / nb;
    NarrowPanels np_{};
    for (std::size_t k = k0; k <= k1; ++k) np_.p[k - k0] = panels[k];
    pack_wide<<<blocks, 256, 0, st>>>(np_, static_cast<int>(nb), static_cast<int>(c0), wp, static_cast<long long>(m->n),
                                      0);
    ck(cudaGetLastError(), "pack_wide launch");
    filter_panel(m, wp, w, ns, 32, np, c, g, alpha, beta, eta, mu, st);
    pack_wide<<<blocks, 256, 0, st>>>(np_, static_cast<int>(nb), static_cast<int>(c0), wp, static_cast<long long>(m->n),
                                      1);
    ck(cudaGetLastError(), "pack_wide launch");
}

static bool filter_wide(cf_matrix m, double2* const* panels, std::size_t npanels, std::size_t nb, std::size_t np,
                        const double* c, const double* g, double alpha, double beta, double* eta, double* mu,
                        cudaStream_t st) {
    const std::size_t ns = npanels * nb;
    const bool narrow = nb < 32 && ns % 32 == 0;
    const bool wider = nb > 32 && nb % 32 == 0;  // n_b = 64, 96, ...: 32-column slices as panels of their own
    if (!(narrow || wider)) return false;
    double2* const wp = wide_panel(m);
    if (!wp) return false;  // the panel-by-panel loop
    const int blocks = pack_blocks(m);
    if (wider) {
        const std::size_t per = nb / 32;
        for (std::size_t b = 0; b < npanels; ++b)
            for (std::size_t q = 0; q < per; ++q) {
                slice_wide<<<blocks, 256, 0, st>>>(panels[b], static_cast<int>(nb), static_cast<int>(32 * q), wp,
                                                   static_cast<long long>(m->n), 0);
                ck(cudaGetLastError(), "slice_wide launch");
                filter_panel(m, wp, b * per + q, ns, 32, np, c, g, alpha, beta, eta, mu, st);
                slice_wide<<<blocks, 256, 0, st>>>(panels[b], static_cast<int>(nb), static_cast<int>(32 * q), wp,
                                                   static_cast<long long>(m->n), 1);
                ck(cudaGetLastError(), "slice_wide launch");
            }
        return true;
    }
    for (std::size_t w = 0; w < ns / 32; ++w) filter_slice_wide(m, panels, w, ns, nb, np, c, g, alpha, beta, eta, mu, st);
    return true;
}

void apply_filter_dev(cf_matrix m, double2* const* panels, std::size_t npanels, std::size_t nb,
                             std::size_t np, const double* c, const double* g, double alpha, double beta, double* eta,
                             double* mu, cudaStream_t st) {
    if (np < 2) throw std::invalid_argument("apply_filter: coefficients cover degrees < 2");
    if (nb == 0 || npanels == 0) throw std::invalid_argument("n_b must divide n_s");
    const std::size_t ns = npanels * nb;
    const std::size_t mom = (np - 2) * ns;
    ck(cudaMemsetAsync(eta, 0, mom * 16, st), "memset eta");
    ck(cudaMemsetAsync(mu, 0, mom * 16, st), "memset mu");
    if (filter_wide(m, panels, npanels, nb, np, c, g, alpha, beta, eta, mu, st)) return;
    for (std::size_t b = 0; b < npanels; ++b) filter_panel(m, panels[b], b, ns, nb, np, c, g, alpha, beta, eta, mu, st);
}

// ------------------------------------------------ filter_distributed (native)
// dist.hpp:227-359 for the shards of one process, one device per shard (several
// shards may share a device).  The host thread enqueues every shard's steps in
// lockstep on per-shard streams; a shard's step waits (cudaStreamWaitEvent) for
// the previous step of every shard it exchanges with, which orders both the halo
// rows it reads and the buffers its own halo stores overwrite.  Halo rows move
// with the kernels' own stores (cf_mirror runs into the neighbour's halo slots
// over peer memory) when a shard's sends are at most kMaxMirror contiguous runs
// (z-slab partitions of a lattice: one run per neighbour), else by a push kernel
// storing the plan's rows into the neighbours' panels right after the step.
__global__ void halo_push_kernel(const double2* __restrict__ src, int nb, const uint64_t* __restrict__ src_row,
                                 const uint64_t* __restrict__ dst_row, const int* __restrict__ dst_w,
                                 double2* const* __restrict__ dst_base, long long count) {
    const long long tot = count * nb;
    for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < tot;
         i += static_cast<long long>(gridDim.x) * blockDim.x) {
        const long long k = i / nb;
        const int j = static_cast<int>(i - k * nb);
        dst_base[dst_w[k]][dst_row[k] * nb + j] = src[src_row[k] * nb + j];
    }
}

namespace {
struct DistShard {
    cf_matrix m = nullptr;
    int dev = 0;
    std::size_t ln = 0, rows = 0;
    cudaStream_t st = nullptr;
    cudaEvent_t ev = nullptr;
    std::vector<double2*> X;      // caller panels (host-staged: the device slot panel b uses)
    std::vector<double2*> H;      // host-staged: the caller's host panels
    double2* slot[2] = {nullptr, nullptr};
    cudaStream_t hs = nullptr, ds = nullptr;   // host-staged copy-in / copy-out streams
    std::vector<cudaEvent_t> in_ev, out_ev;    // per panel: copy-in done, copy-out done
    std::vector<double2*> buf;    // [2 * nbuf] U/W pairs (one pair per panel in flight)
    double* mom = nullptr;        // eta then mu, (np-2)*ns complex each
    std::vector<int> peers;       // shards it sends to or receives from
    struct Run {
        uint64_t r0, r1;
        int v;
        uint64_t d0;
    };
    std::vector<Run> runs;
    bool fused = false;
    uint64_t* d_src = nullptr;    // generic push plan (device)
    uint64_t* d_dst = nullptr;
    int* d_w = nullptr;
    double2** d_bases = nullptr;  // [nbases][nshards] destination base pointers
    long long nsend = 0;
};

std::vector<std::pair<int, std::vector<uint64_t>>> unflatten(const uint64_t* flat, std::size_t len) {
    std::vector<std::pair<int, std::vector<uint64_t>>> out;
    std::size_t q = 0;
    while (q < len) {
        if (q + 2 > len) throw std::invalid_argument("halo plan: truncated record");
        const int v = static_cast<int>(flat[q]);
        const std::size_t cnt = flat[q + 1];
        if (q + 2 + cnt > len) throw std::invalid_argument("halo plan: truncated record");
        out.emplace_back(v, std::vector<uint64_t>(flat + q + 2, flat + q + 2 + cnt));
        q += 2 + cnt;
    }
    return out;
}
}  // namespace

// Measured timeline of the degree loop (dist.hpp:146-162, 216-219): per shard and
// (panel, degree) step a "comm" interval (the stream waiting for the neighbours'
// previous steps, the in-process halo ordering) and a "compute" interval (the
// step's kernels, mirrored halo stores included), from CUDA events.
struct TimelineRec {
    int kind;  // 0 compute, 1 comm
    std::size_t block, degree;
    cudaEvent_t a, b;
};

static void filter_distributed_dev(const cf_dist_worker* wk, std::size_t nw, std::size_t ns, std::size_t nb,
                                   std::size_t np, const double* c, const double* g, double alpha, double beta,
                                   int mode, double* eta, double* mu, bool host = false,
                                   std::vector<std::vector<TimelineRec>>* tl = nullptr) {
    if (nw == 0) throw std::invalid_argument("no shards");
    if (np < 2) throw std::invalid_argument("apply_filter: coefficients cover degrees < 2");
    if (nb == 0 || ns == 0 || ns % nb != 0) throw std::invalid_argument("n_b must divide n_s");
    const std::size_t npan = ns / nb, mom = (np - 2) * ns;
    const bool pipelined = mode != 0;
    // Host-staged X (Alg. 2's slow-memory scheme): the caller's
    // panels stay in host memory; each shard holds two device X slots, panel b+1's
    // owned rows are copied in and panel b-1's copied out while panel b filters.
    // Only Alg. 3 keeps one panel's working set on the device at a time.
    if (host && pipelined)
        throw std::invalid_argument("host-staged panels run the vector schedule (Alg. 3); pipelined needs every panel resident");
    const std::size_t nbuf = pipelined ? npan : 1;  // U/W pairs: one per panel in flight
    std::vector<DistShard> S(nw);
    struct Cleanup {
        std::vector<DistShard>& S;
        ~Cleanup() {
            for (auto& d : S) {
                if (d.st) {
                    cudaSetDevice(d.dev);
                    cudaStreamSynchronize(d.st);
                }
            }
            for (auto& d : S) {
                cudaSetDevice(d.dev);
                for (double2* p : d.buf) cudaFree(p);
                if (d.hs) cudaStreamSynchronize(d.hs);
                if (d.ds) cudaStreamSynchronize(d.ds);
                cudaFree(d.slot[0]);
                cudaFree(d.slot[1]);
                for (cudaEvent_t e : d.in_ev) cudaEventDestroy(e);
                for (cudaEvent_t e : d.out_ev) cudaEventDestroy(e);
                if (d.hs) cudaStreamDestroy(d.hs);
                if (d.ds) cudaStreamDestroy(d.ds);
                cudaFree(d.mom);
                cudaFree(d.d_src);
                cudaFree(d.d_dst);
                cudaFree(d.d_w);
                cudaFree(d.d_bases);
                if (d.ev) cudaEventDestroy(d.ev);
                if (d.st) cudaStreamDestroy(d.st);
            }
        }
    } cleanup{S};
    for (std::size_t w = 0; w < nw; ++w) {
        DistShard& d = S[w];
        if (!wk[w].local) throw std::invalid_argument("null shard matrix");
        d.m = wk[w].local;
        d.dev = d.m->device;
        d.ln = wk[w].local_n;
        d.rows = wk[w].local_n + wk[w].halo_n;
        if (d.m->n != d.ln || d.m->ncols != d.rows) throw std::invalid_argument("shard matrix does not match local_n / halo_n");
        if (!wk[w].X_panels) throw std::invalid_argument("null shard panels");
        for (std::size_t b = 0; b < npan; ++b) d.X.push_back(static_cast<double2*>(wk[w].X_panels[b]));
    }
    // halo plans: w's send rows to v pair with v's recv rows from w, in order
    std::vector<std::vector<std::pair<int, std::vector<uint64_t>>>> send(nw), recv(nw);
    for (std::size_t w = 0; w < nw; ++w) {
        send[w] = unflatten(wk[w].send_flat, wk[w].send_len);
        recv[w] = unflatten(wk[w].recv_flat, wk[w].recv_len);
    }
    std::vector<std::vector<uint64_t>> g_src(nw), g_dst(nw);
    std::vector<std::vector<int>> g_w(nw);
    for (std::size_t w = 0; w < nw; ++w) {
        DistShard& d = S[w];
        for (const auto& [v, rows] : send[w]) {
            if (v < 0 || static_cast<std::size_t>(v) >= nw || static_cast<std::size_t>(v) == w)
                throw std::invalid_argument("halo plan: bad neighbour");
            const std::vector<uint64_t>* dst = nullptr;
            for (const auto& [u, r] : recv[v])
                if (static_cast<std::size_t>(u) == w) dst = &r;
            if (!dst || dst->size() != rows.size()) throw std::invalid_argument("halo plans of the shards disagree");
            for (std::size_t k = 0; k < rows.size(); ++k) {
                if (rows[k] >= d.ln || (*dst)[k] < S[v].ln || (*dst)[k] >= S[v].rows)
                    throw std::invalid_argument("halo plan row outside the shard");
                g_src[w].push_back(rows[k]);
                g_dst[w].push_back((*dst)[k]);
                g_w[w].push_back(v);
                if (!d.runs.empty() && d.runs.back().v == v && d.runs.back().r1 == rows[k] &&
                    d.runs.back().d0 + (d.runs.back().r1 - d.runs.back().r0) == (*dst)[k])
                    ++d.runs.back().r1;
                else
                    d.runs.push_back({rows[k], rows[k] + 1, v, (*dst)[k]});
            }
        }
        d.fused = d.runs.size() <= static_cast<std::size_t>(kMaxMirror);
        d.nsend = static_cast<long long>(g_src[w].size());
    }
    for (std::size_t w = 0; w < nw; ++w) {
        auto add = [&](int v) {
            if (std::find(S[w].peers.begin(), S[w].peers.end(), v) == S[w].peers.end()) S[w].peers.push_back(v);
        };
        for (const auto& sv : send[w]) add(sv.first);
        for (const auto& rv : recv[w]) add(rv.first);
    }
    {  // pre-flight: every device's workspaces (U/W pairs, moments, host-staging slots)
        std::map<int, std::size_t> need;
        for (const DistShard& d : S)
            need[d.dev] += (2 * nbuf + (host ? 2 : 0)) * d.rows * nb * sizeof(double2) + 2 * mom * 16;
        for (const auto& [dev, bytes] : need) {
            ck(cudaSetDevice(dev), "cudaSetDevice");
            hbm_budget(bytes, host ? "filter_distributed (host-staged panels)" : "filter_distributed");
        }
    }
    // device resources; peer access between distinct devices that exchange
    for (std::size_t w = 0; w < nw; ++w) {
        DistShard& d = S[w];
        ck(cudaSetDevice(d.dev), "cudaSetDevice");
        ck(cudaDeviceSynchronize(), "sync before distributed filter");  // caller's X uploads, other streams
        for (int v : d.peers)
            if (S[v].dev != d.dev) {
                const cudaError_t e = cudaDeviceEnablePeerAccess(S[v].dev, 0);
                if (e == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
                else ck(e, "cudaDeviceEnablePeerAccess");
            }
        ck(cudaStreamCreateWithFlags(&d.st, cudaStreamNonBlocking), "cudaStreamCreate");
        ck(cudaEventCreateWithFlags(&d.ev, cudaEventDisableTiming), "cudaEventCreate");
        d.buf.assign(2 * nbuf, nullptr);
        for (auto& p : d.buf) {
            ck(cudaMalloc(&p, d.rows * nb * sizeof(double2)), "cudaMalloc shard U/W");
            ck(cudaMemsetAsync(p, 0, d.rows * nb * sizeof(double2), d.st), "memset shard U/W");
        }
        ck(cudaMalloc(&d.mom, 2 * mom * 16), "cudaMalloc shard moments");
        ck(cudaMemsetAsync(d.mom, 0, 2 * mom * 16, d.st), "memset shard moments");
        if (host) {
            d.H = d.X;
            for (auto& p : d.slot) {
                ck(cudaMalloc(&p, d.rows * nb * sizeof(double2)), "cudaMalloc shard X slot");
                ck(cudaMemsetAsync(p, 0, d.rows * nb * sizeof(double2), d.st), "memset shard X slot");
            }
            for (std::size_t b = 0; b < npan; ++b) d.X[b] = d.slot[b & 1];
            ck(cudaStreamCreateWithFlags(&d.hs, cudaStreamNonBlocking), "cudaStreamCreate");
            ck(cudaStreamCreateWithFlags(&d.ds, cudaStreamNonBlocking), "cudaStreamCreate");
            d.in_ev.assign(npan, nullptr);
            d.out_ev.assign(npan, nullptr);
            for (auto* v : {&d.in_ev, &d.out_ev})
                for (auto& e : *v) ck(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "cudaEventCreate");
            ck(cudaStreamSynchronize(d.st), "slot zero-fill");  // before the copy streams write the slots
        }
    }
    // destination base table: index 0..2*nbuf-1 = U/W buffers, then X panels
    const std::size_t nbases = 2 * nbuf + npan;
    for (std::size_t w = 0; w < nw; ++w) {
        DistShard& d = S[w];
        if (d.fused && !d.nsend) continue;
        ck(cudaSetDevice(d.dev), "cudaSetDevice");
        std::vector<double2*> tab(nbases * nw, nullptr);
        for (std::size_t v = 0; v < nw; ++v) {
            for (std::size_t k = 0; k < 2 * nbuf; ++k) tab[k * nw + v] = S[v].buf[k];
            for (std::size_t b = 0; b < npan; ++b) tab[(2 * nbuf + b) * nw + v] = S[v].X[b];
        }
        ck(cudaMalloc(&d.d_bases, tab.size() * sizeof(double2*)), "cudaMalloc base table");
        ck(cudaMemcpyAsync(d.d_bases, tab.data(), tab.size() * sizeof(double2*), cudaMemcpyHostToDevice, d.st),
           "upload base table");
        if (d.nsend) {
            ck(cudaMalloc(&d.d_src, d.nsend * 8), "cudaMalloc push plan");
            ck(cudaMalloc(&d.d_dst, d.nsend * 8), "cudaMalloc push plan");
            ck(cudaMalloc(&d.d_w, d.nsend * 4), "cudaMalloc push plan");
            ck(cudaMemcpyAsync(d.d_src, g_src[w].data(), d.nsend * 8, cudaMemcpyHostToDevice, d.st), "upload plan");
            ck(cudaMemcpyAsync(d.d_dst, g_dst[w].data(), d.nsend * 8, cudaMemcpyHostToDevice, d.st), "upload plan");
            ck(cudaMemcpyAsync(d.d_w, g_w[w].data(), d.nsend * 4, cudaMemcpyHostToDevice, d.st), "upload plan");
        }
        ck(cudaStreamSynchronize(d.st), "plan upload sync");  // host vectors go out of scope
    }
    auto barrier = [&] {  // every shard waits for the last step of its peers
        for (std::size_t w = 0; w < nw; ++w)
            for (int v : S[w].peers) ck(cudaStreamWaitEvent(S[w].st, S[v].ev, 0), "cudaStreamWaitEvent");
    };
    auto record = [&](std::size_t w) { ck(cudaEventRecord(S[w].ev, S[w].st), "cudaEventRecord"); };
    // mirror runs of shard w's output buffer (base index k); empty when pushed
    auto mirror = [&](std::size_t w, std::size_t k, KParams& P) {
        const DistShard& d = S[w];
        P.nmir = 0;
        if (!d.fused) return;
        for (const auto& r : d.runs)
            P.mir[P.nmir++] = {static_cast<long long>(r.r0), static_cast<long long>(r.r1),
                               (k < 2 * nbuf ? S[r.v].buf[k] : S[r.v].X[k - 2 * nbuf]) + r.d0 * nb};
    };
    auto push = [&](std::size_t w, const double2* src, std::size_t k, bool always) {
        const DistShard& d = S[w];
        if (!d.nsend || (d.fused && !always)) return;
        const long long tot = d.nsend * static_cast<long long>(nb);
        const int blocks = static_cast<int>(std::min<long long>((tot + 255) / 256, 8LL * sms_of(d.dev)));
        halo_push_kernel<<<blocks, 256, 0, d.st>>>(src, static_cast<int>(nb), d.d_src, d.d_dst, d.d_w,
                                                   d.d_bases + k * nw, d.nsend);
        ck(cudaGetLastError(), "halo_push_kernel launch");
    };
    auto base = [&](std::size_t w) {
        KParams P = base_params(S[w].m);
        P.alpha = alpha;
        P.beta = beta;
        return P;
    };
    const std::vector<DegreeStep> sched = degree_schedule(np, c, g);
    // roles: U of panel b is buf[2*slot + cur[b]], W the other one (cur = 0 after init)
    std::vector<int> cur(npan, 0);
    auto slot_of = [&](std::size_t b) { return pipelined ? b : 0; };
    auto init_panel = [&](std::size_t b) {
        const std::size_t kU = 2 * slot_of(b), kW = kU + 1;
        cur[b] = 0;
        for (std::size_t w = 0; w < nw; ++w) {  // X halo (input; always a copy)
            ck(cudaSetDevice(S[w].dev), "cudaSetDevice");
            push(w, S[w].X[b], 2 * nbuf + b, true);
            if (S[w].fused)
                for (const auto& r : S[w].runs)
                    ck(cudaMemcpyPeerAsync(S[r.v].X[b] + r.d0 * nb, S[r.v].dev, S[w].X[b] + r.r0 * nb, S[w].dev,
                                           (r.r1 - r.r0) * nb * sizeof(double2), S[w].st),
                       "X halo copy");
            record(w);
        }
        barrier();
        for (std::size_t w = 0; w < nw; ++w) {  // U = (aH+b) X0 (dist.hpp:254)
            ck(cudaSetDevice(S[w].dev), "cudaSetDevice");
            KParams P = base(w);
            P.U = S[w].X[b];
            P.W = S[w].buf[kU];
            mirror(w, kU, P);
            run<M_SHIFT>(S[w].m, P, nb, nb, S[w].st);
            push(w, S[w].buf[kU], kU, false);
            record(w);
        }
        barrier();
        for (std::size_t w = 0; w < nw; ++w) {  // W = 2(aH+b)U - X0, X = g0c0 X0 + g1c1 U + g2c2 W
            ck(cudaSetDevice(S[w].dev), "cudaSetDevice");
            KParams P = base(w);
            P.U = S[w].buf[kU];
            P.W = S[w].buf[kW];
            P.X = S[w].X[b];
            P.g0 = g[0] * c[0];
            P.g1 = g[1] * c[1];
            P.g2 = g[2] * c[2];
            mirror(w, kW, P);
            run<M_INIT>(S[w].m, P, nb, nb, S[w].st);
            push(w, S[w].buf[kW], kW, false);
            record(w);
        }
    };
    auto mark = [&](std::size_t w) {
        cudaEvent_t e;
        ck(cudaSetDevice(S[w].dev), "cudaSetDevice");
        ck(cudaEventCreate(&e), "cudaEventCreate");
        ck(cudaEventRecord(e, S[w].st), "cudaEventRecord");
        return e;
    };
    if (tl) tl->assign(nw, {});
    auto degree = [&](std::size_t b, const DegreeStep& dstep) {
        cur[b] ^= 1;  // swap_blocks(W, U): the old W is the new U
        const std::size_t kU = 2 * slot_of(b) + cur[b], kW = 2 * slot_of(b) + (cur[b] ^ 1);
        std::vector<cudaEvent_t> ta(tl ? nw : 0), tb(tl ? nw : 0);
        if (tl)
            for (std::size_t w = 0; w < nw; ++w) ta[w] = mark(w);
        barrier();
        if (tl)
            for (std::size_t w = 0; w < nw; ++w) {
                tb[w] = mark(w);
                (*tl)[w].push_back({1, b, dstep.p, ta[w], tb[w]});
            }
        for (std::size_t w = 0; w < nw; ++w) {
            ck(cudaSetDevice(S[w].dev), "cudaSetDevice");
            KParams Q = base(w);
            Q.U = S[w].buf[kU];
            Q.W = S[w].buf[kW];
            Q.X = S[w].X[b];
            mirror(w, kW, Q);
            const std::size_t sl = (dstep.p - 3) * ns + b * nb;
            run_degree(S[w].m, Q, dstep, nb, S[w].st, S[w].mom + 2 * sl, S[w].mom + 2 * mom + 2 * sl);
            push(w, S[w].buf[kW], kW, false);
            record(w);
            if (tl) (*tl)[w].push_back({0, b, dstep.p, tb[w], mark(w)});
        }
    };
    // host-staged copies: owned rows only (neighbours store the halo rows of a slot)
    auto copy_in = [&](std::size_t b) {
        for (std::size_t w = 0; w < nw; ++w) {
            DistShard& d = S[w];
            ck(cudaSetDevice(d.dev), "cudaSetDevice");
            if (b >= 2) ck(cudaStreamWaitEvent(d.hs, d.out_ev[b - 2], 0), "wait slot");
            ck(cudaMemcpyAsync(d.X[b], d.H[b], d.ln * nb * sizeof(double2), cudaMemcpyHostToDevice, d.hs),
               "H2D X panel");
            ck(cudaEventRecord(d.in_ev[b], d.hs), "cudaEventRecord");
        }
    };
    auto copy_out = [&](std::size_t b) {
        for (std::size_t w = 0; w < nw; ++w) {
            DistShard& d = S[w];
            ck(cudaSetDevice(d.dev), "cudaSetDevice");
            record(w);
            ck(cudaStreamWaitEvent(d.ds, d.ev, 0), "wait filter");
            ck(cudaMemcpyAsync(d.H[b], d.X[b], d.ln * nb * sizeof(double2), cudaMemcpyDeviceToHost, d.ds),
               "D2H X panel");
            ck(cudaEventRecord(d.out_ev[b], d.ds), "cudaEventRecord");
        }
    };
    if (!pipelined) {  // Alg. 3: panel by panel (dist.hpp:268-282)
        if (host) copy_in(0);
        for (std::size_t b = 0; b < npan; ++b) {
            if (host) {
                for (std::size_t w = 0; w < nw; ++w) {
                    ck(cudaSetDevice(S[w].dev), "cudaSetDevice");
                    ck(cudaStreamWaitEvent(S[w].st, S[w].in_ev[b], 0), "wait H2D");
                }
                if (b + 1 < npan) copy_in(b + 1);  // its slot was freed by panel b-1's copy-out
            }
            init_panel(b);
            for (const DegreeStep& dstep : sched) degree(b, dstep);
            if (host) copy_out(b);
        }
        if (host)
            for (std::size_t w = 0; w < nw; ++w) {
                ck(cudaSetDevice(S[w].dev), "cudaSetDevice");
                ck(cudaStreamWaitEvent(S[w].st, S[w].out_ev[npan - 1], 0), "wait D2H");
            }
    } else {  // Alg. 4: degree-major over the panels (dist.hpp:283-311)
        for (std::size_t b = 0; b < npan; ++b) init_panel(b);
        for (const DegreeStep& dstep : sched)
            for (std::size_t b = 0; b < npan; ++b) degree(b, dstep);
    }
    // moments: per shard to the host, then the rank-ordered tree (dist.hpp:344-351)
    std::vector<std::vector<double>> hm(nw, std::vector<double>(4 * mom));
    for (std::size_t w = 0; w < nw; ++w) {
        ck(cudaSetDevice(S[w].dev), "cudaSetDevice");
        ck(cudaMemcpyAsync(hm[w].data(), S[w].mom, 4 * mom * 8, cudaMemcpyDeviceToHost, S[w].st), "download moments");
    }
    for (std::size_t w = 0; w < nw; ++w) {
        ck(cudaSetDevice(S[w].dev), "cudaSetDevice");
        ck(cudaStreamSynchronize(S[w].st), "distributed filter sync");
    }
    for (std::size_t stride = 1; stride < nw; stride *= 2)
        for (std::size_t w = 0; w + stride < nw; w += 2 * stride)
            for (std::size_t i = 0; i < 4 * mom; ++i) hm[w][i] += hm[w + stride][i];
    std::memcpy(eta, hm[0].data(), 2 * mom * 8);
    std::memcpy(mu, hm[0].data() + 2 * mom, 2 * mom * 8);
}

void spmmv_dev(cf_matrix m, double alpha, double beta, const double2* X, double2* Y, std::size_t ld,
               std::size_t ncols, cudaStream_t st) {
    KParams P = base_params(m);
    P.alpha = alpha;
    P.beta = beta;
    P.U = X;
    P.W = Y;
    run<M_SHIFT>(m, P, ld, ncols, st);
}

}  // namespace cfb

using namespace cfb;

extern "C" {

int cf_matrix_create_crs(int device, size_t n, size_t ncols, const uint64_t* row_ptr, const int32_t* col_idx,
                         const double* values, const int32_t* order, int C, int sigma, cf_matrix* out) {
    return guard([&] { *out = create_from_crs(device, n, ncols, row_ptr, col_idx, values, order, C, sigma); });
}

int cf_matrix_create_topi(int device, size_t nx, size_t ny, size_t nz, double mass, double hop, int open_boundary,
                          cf_matrix* out) {
    return guard([&] {
        check_device(device);
        Crs crs = topi_crs(nx, ny, nz, mass, hop, open_boundary != 0);
        // 16x16-site xy tiles marched along z: a work unit is one tile-plane, so the
        // y- and z-neighbour reuse of U stays within a few MB of L2 traffic
        std::size_t t = 16;
        std::size_t tx = (nx + (nx + t - 1) / t - 1) / ((nx + t - 1) / t);
        std::size_t ty = (ny + (ny + t - 1) / t - 1) / ((ny + t - 1) / t);
        std::vector<int32_t> ord = lattice_order(nx, ny, nz, tx, ty);
        *out = create_from_crs(device, crs.n, crs.n, crs.row_ptr.data(), crs.col_idx.data(), crs.values.data(),
                               ord.data(), kC, kC);
    });
}

int cf_matrix_create_topi_shard(int device, size_t nx, size_t ny, size_t nz, double mass, double hop,
                                int open_boundary, size_t workers, size_t w, size_t* row_begin, size_t* local_n,
                                size_t* halo_n, cf_matrix* out) {
    return guard([&] {
        check_device(device);
        std::size_t rb = 0, ln = 0, hn = 0, nnz = 0, sl = 0, rl = 0;
        check(cf_topi_shard(nx, ny, nz, mass, hop, open_boundary, workers, w, &rb, &ln, &hn, &nnz, nullptr, nullptr,
                            nullptr, nullptr, nullptr, &sl, nullptr, &rl));
        std::vector<uint64_t> rp(ln + 1), hg(hn), sf(sl), rf(rl);
        std::vector<int32_t> ci(nnz);
        std::vector<double> v(2 * nnz);
        check(cf_topi_shard(nx, ny, nz, mass, hop, open_boundary, workers, w, &rb, &ln, &hn, &nnz, rp.data(), ci.data(),
                            v.data(), hg.data(), sf.data(), &sl, rf.data(), &rl));
        // whole z-planes: the slab keeps the lattice locality schedule, else natural order
        const std::size_t plane = 4 * nx * ny;
        std::vector<int32_t> ord;
        if (plane && rb % plane == 0 && ln % plane == 0 && ln) {
            const std::size_t t = 16;
            std::size_t tx = (nx + (nx + t - 1) / t - 1) / ((nx + t - 1) / t);
            std::size_t ty = (ny + (ny + t - 1) / t - 1) / ((ny + t - 1) / t);
            ord = lattice_order(nx, ny, ln / plane, tx, ty, workers > 1);
        }
        *out = create_from_crs(device, ln, ln + hn, rp.data(), ci.data(), v.data(), ord.empty() ? nullptr : ord.data(),
                               kC, kC);
        if (workers > 1 && !ord.empty() && ln >= 2 * plane) set_boundary(*out, plane, plane);
        if (row_begin) *row_begin = rb;
        if (local_n) *local_n = ln;
        if (halo_n) *halo_n = hn;
    });
}

int cf_matrix_info(cf_matrix m, size_t* n, size_t* ncols, size_t* nnz, size_t* device_bytes, size_t* units) {
    return guard([&] {
        if (!m) throw std::invalid_argument("null matrix");
        if (n) *n = m->n;
        if (ncols) *ncols = m->ncols;
        if (nnz) *nnz = m->nnz;
        if (device_bytes) *device_bytes = m->device_bytes;
        if (units) *units = static_cast<size_t>(m->num_units);
    });
}

int cf_matrix_staged(cf_matrix m, int* staged) {
    return guard([&] {
        if (!m) throw std::invalid_argument("null matrix");
        *staged = m->d_plans ? 1 : 0;
    });
}

int cf_matrix_narrow(cf_matrix m, int* narrow) {
    return guard([&] {
        if (!m) throw std::invalid_argument("null matrix");
        *narrow = (m->narrow_ok && m->d_plans && m->d_trecords) ? 1 : 0;
    });
}

int cf_matrix_typed(cf_matrix m, size_t* typed_pieces, size_t* pieces) {
    return guard([&] {
        if (!m) throw std::invalid_argument("null matrix");
        *typed_pieces = m->typed_pieces;
        *pieces = m->npieces;
    });
}

int cf_matrix_to_crs(cf_matrix m, size_t* n, size_t* nnz, uint64_t* row_ptr, int32_t* col_idx, double* values) {
    return guard([&] {
        if (!m) throw std::invalid_argument("null matrix");
        *n = m->n;
        *nnz = m->nnz;
        if (!row_ptr) return;
        DeviceGuard dg(m->device);
        SellHost s;
        s.n = m->n;
        s.ncols = m->ncols;
        s.nnz = m->nnz;
        s.C = m->C;
        s.pieces = m->pieces;
        if (m->d_records) {  // the device image itself
            s.records.resize(m->record_bytes);
            ck(cudaMemcpy(s.records.data(), m->d_records, m->record_bytes, cudaMemcpyDeviceToHost),
               "download records");
        } else {
            s.records = m->h_records;
        }
        std::vector<uint64_t> rp;
        std::vector<int32_t> ci;
        std::vector<double> v;
        sell_to_crs(s, rp, ci, v);
        std::memcpy(row_ptr, rp.data(), rp.size() * 8);
        std::memcpy(col_idx, ci.data(), ci.size() * 4);
        std::memcpy(values, v.data(), v.size() * 8);
    });
}

int cf_matrix_destroy(cf_matrix m) {
    return guard([&] {
        if (!m) return;
        {
            int cur = -1;
            cudaGetDevice(&cur);
            cudaSetDevice(m->device);
            cudaFree(m->d_records);
            cudaFree(m->d_pieces);
            cudaFree(m->d_units);
            cudaFree(m->d_partials);
            cudaFree(m->d_counters);
            cudaFree(m->d_bpart);
            if (m->d_plans) cudaFree(m->d_plans);
            if (m->d_row0) cudaFree(m->d_row0);
            if (m->d_trecords) cudaFree(m->d_trecords);
            if (m->wide) cudaFree(m->wide);
            if (m->d_tpieces) cudaFree(m->d_tpieces);
            if (m->scratch) cudaFree(m->scratch);
            if (m->hostio) cudaFree(m->hostio);
            if (m->d_slots) cudaFree(m->d_slots);
            if (m->h_slots) cudaFreeHost(m->h_slots);
            if (cur >= 0) cudaSetDevice(cur);
        }
        delete m;
    });
}

static void check_alias(const void* a, const void* b, const char* msg) {
    if (a == b) throw std::invalid_argument(msg);
}

int cf_tuning(const char* key, int value) {
    return guard([&] {
        if (!key) throw std::invalid_argument("null key");
        if (std::string(key) == "staged") g_staged.store(value ? 1 : 0);
        else if (std::string(key) == "narrow") g_narrow.store(value ? 1 : 0);
        else if (std::string(key) == "npf") g_npf.store(value < 0 ? -1 : value);
        else if (std::string(key) == "x_group") g_x_group.store(std::max(1, std::min(3, value)));
        else if (std::string(key) == "wpf") g_wpf.store(std::max(0, value));
        else if (std::string(key) == "typed") g_typed.store(value ? 1 : 0);
        else if (std::string(key) == "pdl") g_pdl.store(value ? 1 : 0);
        else if (std::string(key) == "ko") g_ko.store(value);
        else if (std::string(key) == "gpf") g_gpf.store(std::max(0, value));
        else throw std::invalid_argument(std::string("unknown tuning key: ") + key);
    });
}

int cf_device_count(int* count) {
    return guard([&] {
        int c = 0;
        if (cudaGetDeviceCount(&c) != cudaSuccess) c = 0;
        *count = c;
    });
}

int cf_dev_alloc(int device, size_t bytes, void** out) {
    return guard([&] {
        check_device(device);
        DeviceGuard dg(device);
        *out = nullptr;
        ck(cudaMalloc(out, bytes ? bytes : 16), "cudaMalloc");
    });
}

int cf_dev_free(void* p) {
    return guard([&] {
        if (p) ck(cudaFree(p), "cudaFree");
    });
}

int cf_memcpy(void* dst, const void* src, size_t bytes, int kind) {
    return guard([&] {
        const cudaMemcpyKind k = kind == 0 ? cudaMemcpyHostToDevice
                                 : kind == 1 ? cudaMemcpyDeviceToHost
                                             : cudaMemcpyDefault;  // device to device, peers included (UVA)
        ck(cudaMemcpy(dst, src, bytes, k), "cudaMemcpy");
    });
}

int cf_memcpy_async(void* dst, const void* src, size_t bytes, void* stream) {
    return guard([&] {
        ck(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, static_cast<cudaStream_t>(stream)), "cudaMemcpyAsync");
    });
}

int cf_memset_zero(void* p, size_t bytes) {
    return guard([&] { ck(cudaMemset(p, 0, bytes), "cudaMemset"); });
}

int cf_synchronize(void) {
    return guard([&] { ck(cudaDeviceSynchronize(), "cudaDeviceSynchronize"); });
}

static void set_mirror(KParams& P, cf_matrix m, const cf_mirror* mir, size_t nmir) {
    if (nmir > static_cast<size_t>(kMaxMirror)) throw std::invalid_argument("at most 4 mirror runs per launch");
    P.nmir = static_cast<int>(nmir);
    for (size_t q = 0; q < nmir; ++q) {
        if (mir[q].row_begin > mir[q].row_end || mir[q].row_end > m->n || !mir[q].dst)
            throw std::invalid_argument("mirror run outside the matrix rows");
        P.mir[q] = {static_cast<long long>(mir[q].row_begin), static_cast<long long>(mir[q].row_end),
                    static_cast<double2*>(mir[q].dst)};
    }
}

int cf_spmmv_shifted_mirror(cf_matrix m, double alpha, double beta, const void* X, void* Y, size_t ld, size_t ncols,
                            const cf_mirror* mir, size_t nmir, void* stream) {
    return guard([&] {
        if (!m) throw std::invalid_argument("null matrix");
        check_alias(X, Y, "spmmv: X and Y must not alias");
        KParams P = base_params(m);
        set_mirror(P, m, mir, nmir);
        P.alpha = alpha;
        P.beta = beta;
        P.U = static_cast<const double2*>(X);
        P.W = static_cast<double2*>(Y);
        run<M_SHIFT>(m, P, ld, ncols, static_cast<cudaStream_t>(stream));
    });
}

int cf_cheb_init_tail_mirror(cf_matrix m, double alpha, double beta, void* X, const void* U, void* W, size_t ld,
                             size_t ncols, double g0c0, double g1c1, double g2c2, const cf_mirror* mir, size_t nmir,
                             void* stream) {
    return guard([&] {
        if (!m) throw std::invalid_argument("null matrix");
        check_alias(U, W, "spmmv: X and Y must not alias");
        check_alias(X, U, "spmmv: X and Z must not alias");
        check_alias(X, W, "cheb_init: X and W must not alias");
        KParams P = base_params(m);
        set_mirror(P, m, mir, nmir);
        P.alpha = alpha;
        P.beta = beta;
        P.U = static_cast<const double2*>(U);
        P.W = static_cast<double2*>(W);
        P.X = static_cast<double2*>(X);
        P.g0 = g0c0;
        P.g1 = g1c1;
        P.g2 = g2c2;
        run<M_INIT>(m, P, ld, ncols, static_cast<cudaStream_t>(stream));
    });
}

int cf_chebfd_op_mirror(cf_matrix m, double alpha, double beta, const void* U, void* W, void* X, size_t ld,
                        size_t ncols, double gc, void* eta, void* mu, const cf_mirror* mir, size_t nmir,
                        void* stream) {
    return guard([&] {
        if (!m) throw std::invalid_argument("null matrix");
        check_alias(U, W, "spmmv: X and Y must not alias");
        if (X == U || X == W) throw std::invalid_argument("chebfd_op: X shape mismatch");
        KParams P = base_params(m);
        set_mirror(P, m, mir, nmir);
        P.alpha = alpha;
        P.beta = beta;
        P.U = static_cast<const double2*>(U);
        P.W = static_cast<double2*>(W);
        P.X = static_cast<double2*>(X);
        P.gc = gc;
        run<M_CHEB>(m, P, ld, ncols, static_cast<cudaStream_t>(stream), static_cast<double*>(eta),
                    static_cast<double*>(mu));
    });
}

int cf_degree_schedule(size_t np, const double* c, const double* g, size_t cap, size_t* count, uint64_t* degree,
                       int* kind, double* gw, double* gu, double* gc) {
    return guard([&] {
        if (np < 2) throw std::invalid_argument("apply_filter: coefficients cover degrees < 2");
        const std::vector<DegreeStep> sched = degree_schedule(np, c, g);
        *count = sched.size();
        if (!degree) return;
        if (cap < sched.size()) throw std::invalid_argument("degree schedule: output too small");
        for (std::size_t i = 0; i < sched.size(); ++i) {
            const DegreeStep& d = sched[i];
            degree[i] = d.p;
            kind[i] = d.mode == M_CHEB_NOX ? 1 : d.mode == M_CHEB_X2 ? 2 : d.mode == M_CHEB_X3 ? 3 : 0;
            gw[i] = d.gw;
            gu[i] = d.gu;
            gc[i] = d.gc;
        }
    });
}

int cf_chebfd_step_mirror(cf_matrix m, int kind, double alpha, double beta, const void* U, void* W, void* X, size_t ld,
                          size_t ncols, double gw, double gu, double gc, void* eta, void* mu, const cf_mirror* mir,
                          size_t nmir, void* stream) {
    return guard([&] {
        if (!m) throw std::invalid_argument("null matrix");
        check_alias(U, W, "spmmv: X and Y must not alias");
        if (X == U || X == W) throw std::invalid_argument("chebfd_op: X shape mismatch");
        if (kind < 0 || kind > 3) throw std::invalid_argument("chebfd step: kind must be 0..3");
        KParams P = base_params(m);
        set_mirror(P, m, mir, nmir);
        P.alpha = alpha;
        P.beta = beta;
        P.U = static_cast<const double2*>(U);
        P.W = static_cast<double2*>(W);
        P.X = static_cast<double2*>(X);
        P.gw = gw;
        P.gu = gu;
        P.gc = gc;
        cudaStream_t st = static_cast<cudaStream_t>(stream);
        double *e = static_cast<double*>(eta), *u = static_cast<double*>(mu);
        switch (kind) {
            case 1: run<M_CHEB_NOX>(m, P, ld, ncols, st, e, u); break;
            case 2: run<M_CHEB_X2>(m, P, ld, ncols, st, e, u); break;
            case 3: run<M_CHEB_X3>(m, P, ld, ncols, st, e, u); break;
            default: run<M_CHEB>(m, P, ld, ncols, st, e, u); break;
        }
    });
}

int cf_matrix_set_boundary(cf_matrix m, size_t rows_lo, size_t rows_hi, int* units) {
    return guard([&] {
        if (!m) throw std::invalid_argument("null matrix");
        set_boundary(m, rows_lo, rows_hi);
        if (units) *units = m->bnd_units;
    });
}

int cf_chebfd_step_signal(cf_matrix m, int kind, double alpha, double beta, const void* U, void* W, void* X, size_t ld,
                          size_t ncols, double gw, double gu, double gc, void* eta, void* mu, const cf_mirror* mir,
                          size_t nmir, void* const* flags, size_t nflags, uint64_t value, void* stream,
                          int* in_kernel) {
    return guard([&] {
        if (!m) throw std::invalid_argument("null matrix");
        check_alias(U, W, "spmmv: X and Y must not alias");
        if (X == U || X == W) throw std::invalid_argument("chebfd_op: X shape mismatch");
        if (kind < 0 || kind > 3) throw std::invalid_argument("chebfd step: kind must be 0..3");
        if (nflags && !flags) throw std::invalid_argument("null flag list");
        KParams P = base_params(m);
        set_mirror(P, m, mir, nmir);
        P.alpha = alpha;
        P.beta = beta;
        P.U = static_cast<const double2*>(U);
        P.W = static_cast<double2*>(W);
        P.X = static_cast<double2*>(X);
        P.gw = gw;
        P.gu = gu;
        P.gc = gc;
        // the staged kernel raises the flags once the boundary units are done; otherwise a
        // stream write after the step (with a memory barrier) does
        const bool early = nflags && nflags <= 2 && m->bnd_units > 0 && m->d_plans && ld == 32 && ncols == 32 &&
                           use_staged();
        if (early) {
            P.nbnd = m->bnd_units;
            P.nsig = static_cast<int>(nflags);
            P.sig_val = value;
            for (size_t i = 0; i < nflags; ++i) P.sig[i] = static_cast<unsigned long long*>(flags[i]);
        }
        cudaStream_t st = static_cast<cudaStream_t>(stream);
        double *e = static_cast<double*>(eta), *u = static_cast<double*>(mu);
        switch (kind) {
            case 1: run<M_CHEB_NOX>(m, P, ld, ncols, st, e, u); break;
            case 2: run<M_CHEB_X2>(m, P, ld, ncols, st, e, u); break;
            case 3: run<M_CHEB_X3>(m, P, ld, ncols, st, e, u); break;
            default: run<M_CHEB>(m, P, ld, ncols, st, e, u); break;
        }
        if (!early)
            for (size_t i = 0; i < nflags; ++i) check(cf_flag_signal(flags[i], value, stream));
        if (in_kernel) *in_kernel = early ? 1 : 0;
    });
}

int cf_ipc_get_handle(void* dev_ptr, void* handle) {
    return guard([&] {
        cudaIpcMemHandle_t h;
        ck(cudaIpcGetMemHandle(&h, dev_ptr), "cudaIpcGetMemHandle");
        std::memcpy(handle, &h, sizeof h);
    });
}

int cf_ipc_open_handle(int device, const void* handle, void** dev_ptr) {
    return guard([&] {
        DeviceGuard dg(device);
        cudaIpcMemHandle_t h;
        std::memcpy(&h, handle, sizeof h);
        ck(cudaIpcOpenMemHandle(dev_ptr, h, cudaIpcMemLazyEnablePeerAccess), "cudaIpcOpenMemHandle");
    });
}

// Per-neighbour step flags (the device-side barrier of the fused halo exchange):
// stream memory operations of the driver API, fetched through the runtime's
// entry-point query so the library needs no libcuda link.  The write is ordered
// after the stream's earlier work with a memory barrier (the mirrored peer stores
// of the step are visible first); the wait blocks the stream, not an SM.
namespace {
using WriteValue64 = CUresult (*)(CUstream, CUdeviceptr, cuuint64_t, unsigned int);
using WaitValue64 = CUresult (*)(CUstream, CUdeviceptr, cuuint64_t, unsigned int);
struct StreamMemOps {
    WriteValue64 write = nullptr;
    WaitValue64 wait = nullptr;
};
const StreamMemOps& stream_mem_ops() {
    static const StreamMemOps ops = [] {
        StreamMemOps o;
        cudaDriverEntryPointQueryResult q1, q2;
        void *w = nullptr, *v = nullptr;
        if (cudaGetDriverEntryPoint("cuStreamWriteValue64", &w, cudaEnableDefault, &q1) == cudaSuccess &&
            q1 == cudaDriverEntryPointSuccess)
            o.write = reinterpret_cast<WriteValue64>(w);
        if (cudaGetDriverEntryPoint("cuStreamWaitValue64", &v, cudaEnableDefault, &q2) == cudaSuccess &&
            q2 == cudaDriverEntryPointSuccess)
            o.wait = reinterpret_cast<WaitValue64>(v);
        return o;
    }();
    return ops;
}
void cu_check(CUresult r, const char* what) {
    if (r != CUDA_SUCCESS) throw CudaError(std::string(what) + ": driver error " + std::to_string(static_cast<int>(r)));
}
}  // namespace

int cf_flag_signal(void* flag, uint64_t value, void* stream) {
    return guard([&] {
        const auto& o = stream_mem_ops();
        if (!o.write) throw CudaError("cuStreamWriteValue64 unavailable");
        cu_check(o.write(static_cast<CUstream>(stream), reinterpret_cast<CUdeviceptr>(flag), value, 0),
                 "cuStreamWriteValue64");
    });
}

int cf_flag_wait(const void* flag, uint64_t value, void* stream) {
    return guard([&] {
        const auto& o = stream_mem_ops();
        if (!o.wait) throw CudaError("cuStreamWaitValue64 unavailable");
        cu_check(o.wait(static_cast<CUstream>(stream), reinterpret_cast<CUdeviceptr>(flag), value,
                        CU_STREAM_WAIT_VALUE_GEQ),
                 "cuStreamWaitValue64");
    });
}

int cf_ipc_close(void* dev_ptr) {
    return guard([&] { ck(cudaIpcCloseMemHandle(dev_ptr), "cudaIpcCloseMemHandle"); });
}

int cf_enable_peer_access(int device, int peer) {
    return guard([&] {
        if (device == peer) return;
        DeviceGuard dg(device);
        int can = 0;
        ck(cudaDeviceCanAccessPeer(&can, device, peer), "cudaDeviceCanAccessPeer");
        if (!can) throw CudaError("no peer access between the devices");
        cudaError_t e = cudaDeviceEnablePeerAccess(peer, 0);
        if (e == cudaErrorPeerAccessAlreadyEnabled) {
            cudaGetLastError();
            return;
        }
        ck(e, "cudaDeviceEnablePeerAccess");
    });
}

int cf_spmmv_shifted(cf_matrix m, double alpha, double beta, const void* X, void* Y, size_t ld, size_t ncols,
                     void* stream) {
    return guard([&] {
        if (!m) throw std::invalid_argument("null matrix");
        check_alias(X, Y, "spmmv: X and Y must not alias");
        KParams P = base_params(m);
        P.alpha = alpha;
        P.beta = beta;
        P.U = static_cast<const double2*>(X);
        P.W = static_cast<double2*>(Y);
        run<M_SHIFT>(m, P, ld, ncols, static_cast<cudaStream_t>(stream));
    });
}

int cf_spmmv_shifted_two_minus(cf_matrix m, double alpha, double beta, const void* X, void* Y, const void* Z,
                               size_t ld, size_t ncols, void* stream) {
    return guard([&] {
        if (!m) throw std::invalid_argument("null matrix");
        check_alias(X, Y, "spmmv: X and Y must not alias");
        check_alias(X, Z, "spmmv: X and Z must not alias");
        KParams P = base_params(m);
        P.alpha = alpha;
        P.beta = beta;
        P.U = static_cast<const double2*>(X);
        P.W = static_cast<double2*>(Y);
        P.Z = static_cast<const double2*>(Z);
        run<M_TWO_MINUS>(m, P, ld, ncols, static_cast<cudaStream_t>(stream));
    });
}

int cf_cheb_init(cf_matrix m, double alpha, double beta, void* X, void* U, void* W, size_t ld, size_t ncols,
                 double g0c0, double g1c1, double g2c2, void* stream) {
    return guard([&] {
        if (!m) throw std::invalid_argument("null matrix");
        check_alias(X, U, "spmmv: X and Y must not alias");
        check_alias(U, W, "spmmv: X and Y must not alias");
        check_alias(X, W, "cheb_init: X and W must not alias");
        cudaStream_t st = static_cast<cudaStream_t>(stream);
        KParams P = base_params(m);
        P.alpha = alpha;
        P.beta = beta;
        P.U = static_cast<const double2*>(X);
        P.W = static_cast<double2*>(U);
        run<M_SHIFT>(m, P, ld, ncols, st);
        P = base_params(m);
        P.alpha = alpha;
        P.beta = beta;
        P.U = static_cast<const double2*>(U);
        P.W = static_cast<double2*>(W);
        P.X = static_cast<double2*>(X);
        P.g0 = g0c0;
        P.g1 = g1c1;
        P.g2 = g2c2;
        run<M_INIT>(m, P, ld, ncols, st);
    });
}

int cf_cheb_init_tail(cf_matrix m, double alpha, double beta, void* X, const void* U, void* W, size_t ld, size_t ncols,
                      double g0c0, double g1c1, double g2c2, void* stream) {
    return guard([&] {
        if (!m) throw std::invalid_argument("null matrix");
        check_alias(U, W, "spmmv: X and Y must not alias");
        check_alias(X, U, "spmmv: X and Z must not alias");
        check_alias(X, W, "cheb_init: X and W must not alias");
        KParams P = base_params(m);
        P.alpha = alpha;
        P.beta = beta;
        P.U = static_cast<const double2*>(U);
        P.W = static_cast<double2*>(W);
        P.X = static_cast<double2*>(X);
        P.g0 = g0c0;
        P.g1 = g1c1;
        P.g2 = g2c2;
        run<M_INIT>(m, P, ld, ncols, static_cast<cudaStream_t>(stream));
    });
}

int cf_chebfd_op(cf_matrix m, double alpha, double beta, const void* U, void* W, void* X, size_t ld, size_t ncols,
                 double gc, void* eta, void* mu, void* stream) {
    return guard([&] {
        if (!m) throw std::invalid_argument("null matrix");
        check_alias(U, W, "spmmv: X and Y must not alias");
        if (X == U || X == W) throw std::invalid_argument("chebfd_op: X shape mismatch");
        KParams P = base_params(m);
        P.alpha = alpha;
        P.beta = beta;
        P.U = static_cast<const double2*>(U);
        P.W = static_cast<double2*>(W);
        P.X = static_cast<double2*>(X);
        P.gc = gc;
        run<M_CHEB>(m, P, ld, ncols, static_cast<cudaStream_t>(stream), static_cast<double*>(eta),
                    static_cast<double*>(mu));
    });
}

int cf_chebfd_op_host_moments(cf_matrix m, double alpha, double beta, const void* U, void* W, void* X, size_t ld,
                              size_t ncols, double gc, double* eta, double* mu, void* stream) {
    return guard([&] {
        if (!m) throw std::invalid_argument("null matrix");
        check_alias(U, W, "spmmv: X and Y must not alias");
        if (X == U || X == W) throw std::invalid_argument("chebfd_op: X shape mismatch");
        if (!eta || !mu) throw std::invalid_argument("chebfd_op: null moment row");
        DeviceGuard dg(m->device);
        cudaStream_t st = static_cast<cudaStream_t>(stream);
        if (m->slot_cols < ncols) {  // grow-only: no allocation once the widest panel was seen
            if (m->d_slots) cudaFree(m->d_slots);
            if (m->h_slots) cudaFreeHost(m->h_slots);
            m->d_slots = nullptr;
            m->h_slots = nullptr;
            m->slot_cols = 0;
            ck(cudaMalloc(&m->d_slots, 4 * ncols * sizeof(double)), "cudaMalloc moment slots");
            ck(cudaMallocHost(&m->h_slots, 4 * ncols * sizeof(double)), "cudaMallocHost moment slots");
            m->slot_cols = ncols;
        }
        ck(cudaMemsetAsync(m->d_slots, 0, 4 * ncols * sizeof(double), st), "memset moment slots");
        KParams P = base_params(m);
        P.alpha = alpha;
        P.beta = beta;
        P.U = static_cast<const double2*>(U);
        P.W = static_cast<double2*>(W);
        P.X = static_cast<double2*>(X);
        P.gc = gc;
        run<M_CHEB>(m, P, ld, ncols, st, m->d_slots, m->d_slots + 2 * ncols);
        ck(cudaMemcpyAsync(m->h_slots, m->d_slots, 4 * ncols * sizeof(double), cudaMemcpyDeviceToHost, st),
           "moment slots D2H");
        ck(cudaStreamSynchronize(st), "chebfd_op sync");
        // out += partial (kernels.hpp:199-202): the same single addition the device
        // slot update performs, so the host row is bit-identical to a device-resident one
        for (std::size_t i = 0; i < 2 * ncols; ++i) {
            eta[i] += m->h_slots[i];
            mu[i] += m->h_slots[2 * ncols + i];
        }
    });
}

int cf_current_device(int* device) {
    return guard([&] {
        if (!device) throw std::invalid_argument("null output");
        ck(cudaGetDevice(device), "cudaGetDevice");
    });
}

int cf_apply_filter(cf_matrix m, void* const* panels, size_t npanels, size_t nb, size_t np, const double* c,
                    const double* g, double alpha, double beta, void* eta, void* mu, void* stream) {
    return guard([&] {
        if (!m) throw std::invalid_argument("null matrix");
        DeviceGuard dg(m->device);
        apply_filter_dev(m, reinterpret_cast<double2* const*>(panels), npanels, nb, np, c, g, alpha, beta,
                         static_cast<double*>(eta), static_cast<double*>(mu), static_cast<cudaStream_t>(stream));
    });
}

int cf_filter_distributed(const cf_dist_worker* workers, size_t nworkers, size_t ns, size_t nb, size_t np,
                          const double* c, const double* g, double alpha, double beta, int mode, double* eta,
                          double* mu) {
    return guard([&] {
        int dev0 = 0;
        cudaGetDevice(&dev0);
        struct Restore {
            int d;
            ~Restore() { cudaSetDevice(d); }
        } restore{dev0};
        filter_distributed_dev(workers, nworkers, ns, nb, np, c, g, alpha, beta, mode, eta, mu);
    });
}

int cf_filter_distributed_timeline(const cf_dist_worker* workers, size_t nworkers, size_t ns, size_t nb, size_t np,
                                   const double* c, const double* g, double alpha, double beta, int mode,
                                   int host_panels, double* eta, double* mu, double* timeline, size_t cap,
                                   size_t* count) {
    std::vector<std::vector<TimelineRec>> tl;
    struct Events {
        std::vector<std::vector<TimelineRec>>& tl;
        ~Events() {
            std::vector<cudaEvent_t> all;
            for (auto& v : tl)
                for (auto& r : v) {
                    all.push_back(r.a);
                    all.push_back(r.b);
                }
            std::sort(all.begin(), all.end());
            all.erase(std::unique(all.begin(), all.end()), all.end());
            for (cudaEvent_t e : all) cudaEventDestroy(e);
        }
    } events{tl};
    return guard([&] {
        int dev0 = 0;
        cudaGetDevice(&dev0);
        struct Restore {
            int d;
            ~Restore() { cudaSetDevice(d); }
        } restore{dev0};
        filter_distributed_dev(workers, nworkers, ns, nb, np, c, g, alpha, beta, mode, eta, mu, host_panels != 0,
                               &tl);
        std::size_t k = 0;
        for (std::size_t w = 0; w < tl.size(); ++w) {
            if (tl[w].empty()) continue;
            cudaEvent_t t0 = tl[w].front().a;
            for (const TimelineRec& r : tl[w]) {
                float s0 = 0.f, s1 = 0.f;
                ck(cudaEventElapsedTime(&s0, t0, r.a), "cudaEventElapsedTime");
                ck(cudaEventElapsedTime(&s1, t0, r.b), "cudaEventElapsedTime");
                if (timeline && k < cap) {
                    double* row = timeline + 6 * k;
                    row[0] = static_cast<double>(w);
                    row[1] = r.kind;
                    row[2] = static_cast<double>(r.block);
                    row[3] = static_cast<double>(r.degree);
                    row[4] = s0;
                    row[5] = s1;
                }
                ++k;
            }
        }
        if (count) *count = k;
    });
}

int cf_filter_distributed_host(const cf_dist_worker* workers, size_t nworkers, size_t ns, size_t nb, size_t np,
                               const double* c, const double* g, double alpha, double beta, int mode, double* eta,
                               double* mu) {
    return guard([&] {
        int dev0 = 0;
        cudaGetDevice(&dev0);
        struct Restore {
            int d;
            ~Restore() { cudaSetDevice(d); }
        } restore{dev0};
        filter_distributed_dev(workers, nworkers, ns, nb, np, c, g, alpha, beta, mode, eta, mu, true);
    });
}

int cf_apply_filter_host(cf_matrix m, double* X, size_t ns, size_t nb, size_t np, const double* c, const double* g,
                         double alpha, double beta, double* eta, double* mu) {
    return guard([&] {
        if (!m) throw std::invalid_argument("null matrix");
        if (np < 2) throw std::invalid_argument("apply_filter: coefficients cover degrees < 2");
        DeviceGuard dg(m->device);
        if (nb == 0 || ns == 0 || ns % nb != 0) throw std::invalid_argument("n_b must divide n_s");
        if (m->ncols != m->n) throw std::invalid_argument("apply_filter: row count mismatch");
        // n_b dividing 32 with 32 | n_s: each slot holds 32 / n_b consecutive panels
        // (contiguous on the host), filtered as one packed 32-wide panel (filter_wide)
        // (when the wider slots, U/W and the wide panel fit; else panel by panel)
        bool wide = nb < 32 && 32 % nb == 0 && ns % 32 == 0;
        if (wide) {
            std::size_t fr = 0, tot = 0;
            ck(cudaMemGetInfo(&fr, &tot), "cudaMemGetInfo");
            const std::size_t wb = m->n * 32 * 16, slots = std::min<std::size_t>(ns / 32, 2) * wb + 2 * (np - 2) * ns * 16;
            const std::size_t uw = 2 * m->rows_alloc * 32 * 16;
            const std::size_t extra = (m->wide_bytes < wb ? wb : 0) + (m->hostio_bytes < slots ? slots - m->hostio_bytes : 0) +
                                      (m->scratch_bytes < uw ? uw - m->scratch_bytes : 0);
            wide = extra + (std::size_t{1} << 30) <= fr && wide_panel(m);
        }
        const std::size_t K = wide ? 32 / nb : 1;
        const std::size_t n = m->n, npan = ns / nb / K, pb = n * nb * K * 16, mb = (np - 2) * ns * 16;
        // Host-staged panels (cfg3 on one GPU holds 4 x 34 GB X panels on
        // the host): two device panel slots, panel b+1 copied in and panel b-1 copied
        // out on their own streams while panel b filters.  With pinned host memory the
        // copies hide behind the filter; the device needs U, W and two panels, not X.
        const std::size_t nslot = std::min<std::size_t>(npan, 2);
        const std::size_t need = nslot * pb + 2 * mb;
        {  // both workspaces (X slots here, U/W in filter_panel) checked before either grows
            const std::size_t uw = 2 * m->rows_alloc * nb * K * 16;
            const std::size_t grow = (m->hostio_bytes < need ? need - m->hostio_bytes : 0) +
                                     (m->scratch_bytes < uw ? uw - m->scratch_bytes : 0);
            hbm_budget(grow, "apply_filter (host-staged panels)");
        }
        if (m->hostio_bytes < need) {  // kept across calls: repeated use pays no allocation
            if (m->hostio) cudaFree(m->hostio);
            m->hostio = nullptr;
            m->hostio_bytes = 0;
            ck(cudaMalloc(&m->hostio, need), "cudaMalloc host-entry workspace");
            m->hostio_bytes = need;
        }
        char* dslot[2] = {static_cast<char*>(m->hostio), static_cast<char*>(m->hostio) + (nslot - 1) * pb};
        double* deta = reinterpret_cast<double*>(static_cast<char*>(m->hostio) + nslot * pb);
        double* dmu = reinterpret_cast<double*>(reinterpret_cast<char*>(deta) + mb);
        struct Streams {
            cudaStream_t s[3] = {nullptr, nullptr, nullptr};
            std::vector<cudaEvent_t> ev;
            ~Streams() {
                for (cudaStream_t x : s)
                    if (x) cudaStreamSynchronize(x);
                for (cudaEvent_t e : ev) cudaEventDestroy(e);
                for (cudaStream_t x : s)
                    if (x) cudaStreamDestroy(x);
            }
            cudaEvent_t event() {
                cudaEvent_t e;
                ck(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "cudaEventCreate");
                ev.push_back(e);
                return e;
            }
        } S;
        // a blocking host entry: work already queued on any stream (which may use this
        // handle's scratch and counters) completes before the panels start
        ck(cudaDeviceSynchronize(), "sync before host-staged filter");
        for (auto& x : S.s) ck(cudaStreamCreateWithFlags(&x, cudaStreamNonBlocking), "cudaStreamCreate");
        cudaStream_t st = S.s[0], hs = S.s[1], ds = S.s[2];
        ck(cudaMemsetAsync(deta, 0, mb, st), "memset eta");
        ck(cudaMemsetAsync(dmu, 0, mb, st), "memset mu");
        std::vector<cudaEvent_t> out(npan, nullptr);  // D2H of panel b done
        auto h2d = [&](std::size_t b) {
            if (b >= 2) ck(cudaStreamWaitEvent(hs, out[b - 2], 0), "wait slot");
            ck(cudaMemcpyAsync(dslot[b & 1], X + b * n * nb * K * 2, pb, cudaMemcpyHostToDevice, hs), "H2D X panel");
            cudaEvent_t in = S.event();
            ck(cudaEventRecord(in, hs), "record");
            ck(cudaStreamWaitEvent(st, in, 0), "wait H2D");
            double2* slot = reinterpret_cast<double2*>(dslot[b & 1]);
            if (!wide) {
                filter_panel(m, slot, b, ns, nb, np, c, g, alpha, beta, deta, dmu, st);
                return;
            }
            // the slot's K panels as panels b K .. b K + K - 1 of the block vector
            std::vector<double2*> pan(ns / nb, nullptr);
            for (std::size_t k = 0; k < K; ++k) pan[b * K + k] = slot + k * n * nb;
            filter_slice_wide(m, pan.data(), b, ns, nb, np, c, g, alpha, beta, deta, dmu, st);
        };
        // issue order keeps the GPU fed even for pageable buffers (whose D2H blocks the
        // host): panel b+1's copy-in and filter are queued before panel b's copy-out
        h2d(0);
        for (std::size_t b = 0; b < npan; ++b) {
            cudaEvent_t done = S.event();
            ck(cudaEventRecord(done, st), "record");
            if (b + 1 < npan) h2d(b + 1);
            ck(cudaStreamWaitEvent(ds, done, 0), "wait filter");
            ck(cudaMemcpyAsync(X + b * n * nb * K * 2, dslot[b & 1], pb, cudaMemcpyDeviceToHost, ds), "D2H X panel");
            out[b] = S.event();
            ck(cudaEventRecord(out[b], ds), "record");
        }
        ck(cudaStreamWaitEvent(st, out[npan - 1], 0), "wait D2H");
        ck(cudaMemcpyAsync(eta, deta, mb, cudaMemcpyDeviceToHost, st), "D2H eta");
        ck(cudaMemcpyAsync(mu, dmu, mb, cudaMemcpyDeviceToHost, st), "D2H mu");
        ck(cudaStreamSynchronize(st), "sync");
        ck(cudaStreamSynchronize(ds), "sync");
    });
}

}  // extern "C"
