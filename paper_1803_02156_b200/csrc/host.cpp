// Host half of libchebfd_b200: the reference's host-side routines restated for
// the drop-in (bit-identical outputs), the closed-form Topi generator, and the
// 4x4-blocked SELL-C-sigma builder.  Threaded with std::thread; no GPU here.
#include <algorithm>
#include <atomic>
#include <exception>
#include <cmath>
#include <cstring>
#include <map>
#include <mutex>
#include <numeric>
#include <set>
#include <thread>
#include <unordered_map>

#include "common.hpp"

namespace cfb {

static thread_local std::string g_err;
void set_error(const std::string& msg) { g_err = msg; }
void rethrow_status(int status) {
    const std::string msg = g_err;
    switch (status) {
        case CF_EINVAL: throw std::invalid_argument(msg);
        case CF_ERANGE: throw std::out_of_range(msg);
        case CF_EPROTOCOL: throw ProtocolError(msg);
        case CF_ECUDA: throw CudaError(msg);
        default: throw std::runtime_error(msg);
    }
}

unsigned host_threads() {
    if (const char* e = std::getenv("CHEBFD_HOST_THREADS")) {
        long v = std::strtol(e, nullptr, 10);
        if (v >= 1) return static_cast<unsigned>(v);
    }
    unsigned hw = std::thread::hardware_concurrency();
    return hw ? std::min(hw, 64u) : 1;
}

// Runs f(lo, hi) over a static split of [0, n); the first exception thrown by a
// worker is rethrown on the calling thread.
template <class F>
static void parallel_ranges(std::size_t n, F&& f) {
    unsigned nt = static_cast<unsigned>(std::min<std::size_t>(host_threads(), std::max<std::size_t>(n / 4096, 1)));
    if (nt <= 1) {
        f(std::size_t{0}, n);
        return;
    }
    std::vector<std::thread> th;
    std::vector<std::exception_ptr> err(nt);
    for (unsigned t = 0; t < nt; ++t)
        th.emplace_back([&, t] {
            try {
                f(n * t / nt, n * (t + 1) / nt);
            } catch (...) {
                err[t] = std::current_exception();
            }
        });
    for (auto& x : th) x.join();
    for (auto& e : err)
        if (e) std::rethrow_exception(e);
}

// ------------------------------------------------------------- RNG ------
// block_vector.hpp:17-35
static inline uint64_t splitmix64(uint64_t x) {
    x += 0x9e3779b97f4a7c15ULL;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
    return x ^ (x >> 31);
}
static inline void unit_gauss(uint64_t seed, uint64_t i, uint64_t j, double* out) {
    uint64_t h = splitmix64(splitmix64(seed) ^ splitmix64(i * 0xd1342543de82ef95ULL + j));
    uint64_t h2 = splitmix64(h);
    double u = (static_cast<double>(h >> 11) + 1.0) * 0x1.0p-53;
    double v = static_cast<double>(h2 >> 11) * 0x1.0p-53;
    double r = std::sqrt(-std::log(u));
    out[0] = r * std::cos(6.283185307179586477 * v);
    out[1] = r * std::sin(6.283185307179586477 * v);
}

// ------------------------------------------------------- Topi blocks ----
// 4x4 stencil blocks built with the reference's operation sequence
// (sparse_matrix.hpp:131-174): b = 0.5 t (B + I*alpha_d), adjoint = conj^T.
struct Blk {
    double a[4][4][2];
};
static Blk onsite_blk(double m) {
    Blk b{};
    b.a[0][0][0] = m;
    b.a[1][1][0] = m;
    b.a[2][2][0] = -m;
    b.a[3][3][0] = -m;
    return b;
}
static Blk hop_blk(double t, int dir) {
    Blk al{};
    auto set = [&](int r, int c, double re, double im) {
        al.a[r][c][0] = re;
        al.a[r][c][1] = im;
    };
    switch (dir) {
        case 0: set(0, 3, 1, 0); set(1, 2, 1, 0); set(2, 1, 1, 0); set(3, 0, 1, 0); break;
        case 1: set(0, 3, -0.0, -1); set(1, 2, 0, 1); set(2, 1, -0.0, -1); set(3, 0, 0, 1); break;
        default: set(0, 2, 1, 0); set(1, 3, -1, 0); set(2, 0, 1, 0); set(3, 1, -1, 0); break;
    }
    Blk b = onsite_blk(1.0);
    const double ht = 0.5 * t;
    for (int r = 0; r < 4; ++r)
        for (int c = 0; c < 4; ++c) {
            double ar = al.a[r][c][0], ai = al.a[r][c][1];
            volatile double pr = 0.0 * ar - 1.0 * ai;  // (0,1)*(ar,ai), no contraction
            volatile double pi = 0.0 * ai + 1.0 * ar;
            double sr = b.a[r][c][0] + pr, si = b.a[r][c][1] + pi;
            b.a[r][c][0] = ht * sr;
            b.a[r][c][1] = ht * si;
        }
    return b;
}
static Blk adjoint_blk(const Blk& b) {
    Blk r;
    for (int i = 0; i < 4; ++i)
        for (int j = 0; j < 4; ++j) {
            r.a[i][j][0] = b.a[j][i][0];
            r.a[i][j][1] = -b.a[j][i][1];
        }
    return r;
}

struct TopiSpec {
    std::size_t ext[3];
    bool open;
    Blk onsite, hop[3], adj[3];
};
static TopiSpec make_topi(std::size_t nx, std::size_t ny, std::size_t nz, double mass, double hop, bool open) {
    TopiSpec t;
    t.ext[0] = nx;
    t.ext[1] = ny;
    t.ext[2] = nz;
    t.open = open;
    t.onsite = onsite_blk(mass);
    for (int d = 0; d < 3; ++d) {
        t.hop[d] = hop_blk(hop, d);
        t.adj[d] = adjoint_blk(t.hop[d]);
    }
    return t;
}

// Row 4s+r of topi_generate in closed form.  The reference emits triplets in
// the order (outer site sigma ascending; onsite, then per direction d the
// forward block of sigma's rows and the adjoint block of fwd_d(sigma)'s rows)
// and sums duplicates per (row, col) in that order starting from (0,0)
// (sparse_matrix.hpp:43-64, 203-226).  Row s receives: at sigma = s the onsite
// and forward blocks, at sigma = bwd_d(s) the adjoint block of direction d.
// Returns the entry count; cols strictly ascending as in build_from_triplets.
static int topi_row(const TopiSpec& t, std::size_t s, int r, int32_t* cols, double* vals) {
    const std::size_t nx = t.ext[0], ny = t.ext[1];
    std::size_t coord[3] = {s % nx, (s / nx) % ny, s / (nx * ny)};
    auto site = [&](const std::size_t* c) { return (c[2] * ny + c[1]) * nx + c[0]; };
    struct Ev {
        std::size_t sigma;
        int slot;
        std::size_t col_site;
        const Blk* b;
    };
    Ev ev[7];
    int ne = 0;
    ev[ne++] = {s, 0, s, &t.onsite};
    for (int d = 0; d < 3; ++d) {
        std::size_t f[3] = {coord[0], coord[1], coord[2]};
        bool ok = true;
        if (coord[d] + 1 < t.ext[d]) f[d] = coord[d] + 1;
        else if (!t.open) f[d] = 0;
        else ok = false;
        if (ok) ev[ne++] = {s, 1 + 2 * d, site(f), &t.hop[d]};
        std::size_t b[3] = {coord[0], coord[1], coord[2]};
        ok = true;
        if (coord[d] > 0) b[d] = coord[d] - 1;
        else if (!t.open) b[d] = t.ext[d] - 1;
        else ok = false;
        if (ok) {
            std::size_t bs = site(b);
            ev[ne++] = {bs, 2 + 2 * d, bs, &t.adj[d]};
        }
    }
    // insertion sort by (sigma, slot): the reference's triplet order
    for (int i = 1; i < ne; ++i)
        for (int j = i; j > 0 && (ev[j].sigma < ev[j - 1].sigma ||
                                  (ev[j].sigma == ev[j - 1].sigma && ev[j].slot < ev[j - 1].slot));
             --j)
            std::swap(ev[j], ev[j - 1]);
    int cnt = 0;
    for (int e = 0; e < ne; ++e)
        for (int c = 0; c < 4; ++c) {
            double re = ev[e].b->a[r][c][0], im = ev[e].b->a[r][c][1];
            if (re == 0.0 && im == 0.0) continue;  // != cplx(0.0) (sparse_matrix.hpp:193)
            int32_t col = static_cast<int32_t>(4 * ev[e].col_site + c);
            int k = 0;
            while (k < cnt && cols[k] != col) ++k;
            if (k == cnt) {
                cols[cnt] = col;
                vals[2 * cnt] = 0.0;
                vals[2 * cnt + 1] = 0.0;
                ++cnt;
            }
            vals[2 * k] += re;
            vals[2 * k + 1] += im;
        }
    for (int i = 1; i < cnt; ++i)
        for (int j = i; j > 0 && cols[j] < cols[j - 1]; --j) {
            std::swap(cols[j], cols[j - 1]);
            std::swap(vals[2 * j], vals[2 * j - 2]);
            std::swap(vals[2 * j + 1], vals[2 * j - 1]);
        }
    return cnt;
}

Crs topi_crs(std::size_t nx, std::size_t ny, std::size_t nz, double mass, double hop, bool open) {
    if (nx < 1 || ny < 1 || nz < 1) throw std::invalid_argument("lattice extents must be positive");
    TopiSpec t = make_topi(nx, ny, nz, mass, hop, open);
    Crs m;
    std::size_t S = nx * ny * nz;
    m.n = 4 * S;
    if (m.n > static_cast<std::size_t>(INT32_MAX)) throw std::invalid_argument("topi: dimension exceeds int32 columns");
    m.row_ptr.assign(m.n + 1, 0);
    parallel_ranges(S, [&](std::size_t lo, std::size_t hi) {
        int32_t cols[32];
        double vals[64];
        for (std::size_t s = lo; s < hi; ++s)
            for (int r = 0; r < 4; ++r) m.row_ptr[4 * s + r + 1] = topi_row(t, s, r, cols, vals);
    });
    for (std::size_t i = 0; i < m.n; ++i) m.row_ptr[i + 1] += m.row_ptr[i];
    m.col_idx.resize(m.row_ptr[m.n]);
    m.values.resize(2 * m.row_ptr[m.n]);
    parallel_ranges(S, [&](std::size_t lo, std::size_t hi) {
        for (std::size_t s = lo; s < hi; ++s)
            for (int r = 0; r < 4; ++r) {
                std::size_t i = 4 * s + r;
                topi_row(t, s, r, m.col_idx.data() + m.row_ptr[i], m.values.data() + 2 * m.row_ptr[i]);
            }
    });
    return m;
}

// Locality schedule for lattice matrices: y-bands of ty rows; each band is
// marched along z; within a (band, z) plane the x-tiles of tx sites follow each
// other, and a tile-plane (ty rows of tx sites, y-major) is one work unit.  So
// x-neighbour tiles run concurrently, z-neighbour planes are nx*ty sites apart,
// and only the y-band boundaries re-read U from DRAM.
// boundary_first: the planes z = 0 and z = nz-1 (a z-slab shard's halo-reading
// and halo-sending rows) come first, each in its own band / tile order, then the
// interior planes in the usual band march, so a step's boundary units are the
// first ones claimed and its neighbours can be signalled before the interior ends.
std::vector<int32_t> lattice_order(std::size_t nx, std::size_t ny, std::size_t nz, std::size_t tx, std::size_t ty,
                                   bool boundary_first) {
    if (tx == 0 || ty == 0) throw std::invalid_argument("lattice_order: tile extents must be positive");
    std::vector<int32_t> ord;
    ord.reserve(nx * ny * nz);
    auto plane = [&](std::size_t y0, std::size_t z) {
        for (std::size_t x0 = 0; x0 < nx; x0 += tx)
            for (std::size_t y = y0; y < std::min(ny, y0 + ty); ++y)
                for (std::size_t x = x0; x < std::min(nx, x0 + tx); ++x)
                    ord.push_back(static_cast<int32_t>((z * ny + y) * nx + x));
    };
    const bool bf = boundary_first && nz >= 3;
    if (bf)
        for (std::size_t z : {std::size_t{0}, nz - 1})
            for (std::size_t y0 = 0; y0 < ny; y0 += ty) plane(y0, z);
    for (std::size_t y0 = 0; y0 < ny; y0 += ty)
        for (std::size_t z = bf ? 1 : 0; z < (bf ? nz - 1 : nz); ++z) plane(y0, z);
    return ord;
}

// ------------------------------------------------------ Jacobi eig ---
// Two-sided cyclic Jacobi for complex Hermitian A (jacobi_eig.hpp:32-98):
// sweep the pairs (p, q), p < q, in row order; each rotation zeroes a_pq with
// the Rutishauser angle; stop once the off-diagonal Frobenius norm is at most
// tol * max(||A||_F, 1).  Complex products are written out in components.
void jacobi_hermitian(std::size_t k, std::vector<double> A, double tol, std::size_t max_sweeps,
                      std::vector<double>& values, std::vector<double>& vectors) {
    auto re = [&](std::size_t i, std::size_t j) -> double& { return A[2 * (i * k + j)]; };
    auto im = [&](std::size_t i, std::size_t j) -> double& { return A[2 * (i * k + j) + 1]; };
    std::vector<double> V(2 * k * k, 0.0);
    for (std::size_t i = 0; i < k; ++i) V[2 * (i * k + i)] = 1.0;
    double fro = 0.0;
    for (std::size_t i = 0; i < k * k; ++i) fro += A[2 * i] * A[2 * i] + A[2 * i + 1] * A[2 * i + 1];
    const double thresh = tol * std::max(std::sqrt(fro), 1.0);
    auto off = [&] {
        double acc = 0.0;
        for (std::size_t i = 0; i < k; ++i)
            for (std::size_t j = i + 1; j < k; ++j) acc += re(i, j) * re(i, j) + im(i, j) * im(i, j);
        return std::sqrt(2.0 * acc);
    };
    for (std::size_t sweep = 0; sweep < max_sweeps && off() > thresh; ++sweep) {
        for (std::size_t p = 0; p < k; ++p)
            for (std::size_t q = p + 1; q < k; ++q) {
                const double ar = re(p, q), ai = im(p, q);
                const double mag = std::hypot(ar, ai);
                if (mag == 0.0) continue;
                const double er = ar / mag, ei = ai / mag;  // phase of a_pq
                const double tau = (re(q, q) - re(p, p)) / (2.0 * mag);
                const double t = (tau >= 0.0 ? 1.0 : -1.0) / (std::fabs(tau) + std::sqrt(1.0 + tau * tau));
                const double c = 1.0 / std::sqrt(1.0 + t * t);
                const double sr = t * c * er, si = t * c * ei;  // s = t c e^{i phi}
                // columns: a_ip' = c a_ip - conj(s) a_iq ; a_iq' = s a_ip + c a_iq
                for (std::size_t i = 0; i < k; ++i) {
                    const double pr = re(i, p), pi = im(i, p), qr = re(i, q), qi = im(i, q);
                    re(i, p) = c * pr - (sr * qr + si * qi);
                    im(i, p) = c * pi - (sr * qi - si * qr);
                    re(i, q) = (sr * pr - si * pi) + c * qr;
                    im(i, q) = (sr * pi + si * pr) + c * qi;
                }
                // rows: a_pj' = c a_pj - s a_qj ; a_qj' = conj(s) a_pj + c a_qj
                for (std::size_t j = 0; j < k; ++j) {
                    const double pr = re(p, j), pi = im(p, j), qr = re(q, j), qi = im(q, j);
                    re(p, j) = c * pr - (sr * qr - si * qi);
                    im(p, j) = c * pi - (sr * qi + si * qr);
                    re(q, j) = (sr * pr + si * pi) + c * qr;
                    im(q, j) = (sr * pi - si * pr) + c * qi;
                }
                re(p, q) = im(p, q) = re(q, p) = im(q, p) = 0.0;
                for (std::size_t i = 0; i < k; ++i) {
                    double* vp = &V[2 * (i * k + p)];
                    double* vq = &V[2 * (i * k + q)];
                    const double pr = vp[0], pi = vp[1], qr = vq[0], qi = vq[1];
                    vp[0] = c * pr - (sr * qr + si * qi);
                    vp[1] = c * pi - (sr * qi - si * qr);
                    vq[0] = (sr * pr - si * pi) + c * qr;
                    vq[1] = (sr * pi + si * pr) + c * qi;
                }
            }
    }
    std::vector<std::size_t> ord(k);
    std::iota(ord.begin(), ord.end(), 0);
    std::sort(ord.begin(), ord.end(), [&](std::size_t a, std::size_t b) { return re(a, a) < re(b, b); });
    values.resize(k);
    vectors.assign(2 * k * k, 0.0);
    for (std::size_t jj = 0; jj < k; ++jj) {
        values[jj] = re(ord[jj], ord[jj]);
        for (std::size_t i = 0; i < k; ++i) {
            vectors[2 * (i * k + jj)] = V[2 * (i * k + ord[jj])];
            vectors[2 * (i * k + jj) + 1] = V[2 * (i * k + ord[jj]) + 1];
        }
    }
}

// ------------------------------------------------- SELL-C-sigma / B4 ---
std::size_t piece_bytes(int C, int kcnt, std::size_t nvals) {
    return sidx_offset(C, kcnt, nvals) + ((static_cast<std::size_t>(kcnt) + 1) * C + 15) / 16 * 16;
}

// Entries of block-row b sorted by (block column, row, column): the block
// decomposition for matrices whose rows are not column-sorted (shard-local
// matrices keep the reference's remapped column order, dist.hpp:76-86).
struct BEnt {
    int32_t bc;
    uint8_t r, c;
    uint64_t k;
};
static void sorted_block_entries(std::size_t n, const uint64_t* rp, const int32_t* ci, std::size_t b,
                                 std::vector<BEnt>& e) {
    e.clear();
    std::size_t r0 = 4 * b, r1 = std::min(n, r0 + 4);
    for (std::size_t r = r0; r < r1; ++r)
        for (uint64_t k = rp[r]; k < rp[r + 1]; ++k)
            e.push_back({ci[k] / 4, static_cast<uint8_t>(r - r0), static_cast<uint8_t>(ci[k] % 4), k});
    std::sort(e.begin(), e.end(), [](const BEnt& a, const BEnt& x) {
        if (a.bc != x.bc) return a.bc < x.bc;
        if (a.r != x.r) return a.r < x.r;
        return a.c < x.c;
    });
}

static bool rows_sorted(std::size_t n, const uint64_t* rp, const int32_t* ci) {
    for (std::size_t i = 0; i < n; ++i)
        for (uint64_t k = rp[i] + 1; k < rp[i + 1]; ++k)
            if (ci[k] <= ci[k - 1]) return false;
    return true;
}

// Number of distinct block columns of block-row b (rows 4b..4b+3).
static int count_blocks(std::size_t n, const uint64_t* rp, const int32_t* ci, std::size_t b, std::size_t* nv,
                        bool sorted) {
    if (!sorted) {
        thread_local std::vector<BEnt> e;
        sorted_block_entries(n, rp, ci, b, e);
        *nv = e.size();
        int d = 0;
        for (std::size_t i = 0; i < e.size(); ++i)
            if (i == 0 || e[i].bc != e[i - 1].bc) ++d;
        return d;
    }
    std::size_t r0 = 4 * b, r1 = std::min(n, r0 + 4);
    uint64_t pos[4], end[4];
    int nr = static_cast<int>(r1 - r0);
    std::size_t vals = 0;
    for (int r = 0; r < nr; ++r) {
        pos[r] = rp[r0 + r];
        end[r] = rp[r0 + r + 1];
        vals += end[r] - pos[r];
    }
    *nv = vals;
    int blocks = 0;
    while (true) {
        int64_t bc = INT64_MAX;
        for (int r = 0; r < nr; ++r)
            if (pos[r] < end[r]) bc = std::min<int64_t>(bc, ci[pos[r]] / 4);
        if (bc == INT64_MAX) break;
        ++blocks;
        for (int r = 0; r < nr; ++r)
            while (pos[r] < end[r] && ci[pos[r]] / 4 == bc) ++pos[r];
    }
    return blocks;
}

std::vector<int32_t> sell_permutation(std::size_t n, const uint64_t* rp, const int32_t* ci, const int32_t* order,
                                      int C, int sigma) {
    if (C <= 0 || C % 4 != 0 || C > 64) throw std::invalid_argument("sell: C must be a multiple of 4 in [4, 64]");
    if (sigma <= 0 || sigma % C != 0) throw std::invalid_argument("sell: sigma must be a positive multiple of C");
    std::size_t nbr = (n + 3) / 4;
    std::vector<int32_t> ord(nbr);
    if (order) {
        std::vector<uint8_t> seen(nbr, 0);
        for (std::size_t i = 0; i < nbr; ++i) {
            if (order[i] < 0 || static_cast<std::size_t>(order[i]) >= nbr || seen[order[i]])
                throw std::invalid_argument("sell: order is not a permutation of the block-rows");
            seen[order[i]] = 1;
            ord[i] = order[i];
        }
    } else {
        std::iota(ord.begin(), ord.end(), 0);
    }
    std::vector<int> len(nbr);
    const bool sorted = rows_sorted(n, rp, ci);
    parallel_ranges(nbr, [&](std::size_t lo, std::size_t hi) {
        std::size_t nv;
        for (std::size_t b = lo; b < hi; ++b) len[b] = count_blocks(n, rp, ci, b, &nv, sorted);
    });
    // sigma-window stable sort by descending block count
    for (std::size_t w0 = 0; w0 < nbr; w0 += sigma) {
        auto first = ord.begin() + w0, last = ord.begin() + std::min(nbr, w0 + static_cast<std::size_t>(sigma));
        std::stable_sort(first, last, [&](int32_t a, int32_t b) { return len[a] > len[b]; });
    }
    std::size_t nchunks = (nbr + C - 1) / C;
    ord.resize(nchunks * C, -1);
    return ord;
}

SellHost build_sell(std::size_t n, std::size_t ncols, const uint64_t* rp, const int32_t* ci, const double* values,
                    const int32_t* order, int C, int sigma, std::size_t units_hint) {
    if (n == 0) throw std::invalid_argument("empty matrix");
    if (ncols < n) throw std::invalid_argument("sell: ncols must cover the rows");
    if (C == 0) C = kDefaultC;
    if (sigma == 0) sigma = C;
    SellHost s;
    s.n = n;
    s.ncols = ncols;
    s.nnz = rp[n];
    s.C = C;
    s.sigma = sigma;
    s.nbr = (n + 3) / 4;
    for (std::size_t i = 0; i < n; ++i) {
        if (rp[i + 1] < rp[i]) throw std::invalid_argument("sell: row_ptr not monotone");
        for (uint64_t k = rp[i]; k < rp[i + 1]; ++k)
            if (ci[k] < 0 || static_cast<std::size_t>(ci[k]) >= ncols)
                throw std::invalid_argument("sell: column index out of range");
    }
    const bool sorted = rows_sorted(n, rp, ci);
    if (!sorted) {  // rows may come in any column order, but without duplicates
        parallel_ranges(n, [&](std::size_t lo, std::size_t hi) {
            std::vector<int32_t> c;
            for (std::size_t i = lo; i < hi; ++i) {
                c.assign(ci + rp[i], ci + rp[i + 1]);
                std::sort(c.begin(), c.end());
                if (std::adjacent_find(c.begin(), c.end()) != c.end())
                    throw std::invalid_argument("sell: duplicate column index within a row");
            }
        });
    }
    s.perm = sell_permutation(n, rp, ci, order, C, sigma);
    s.nchunks = s.perm.size() / C;

    struct BlockRowLayout {
        std::vector<int32_t> bcol;
        std::vector<uint16_t> mask;
        std::vector<uint16_t> cnt;
    };
    auto layout_of = [&](int32_t b, BlockRowLayout& L) {
        L.bcol.clear();
        L.mask.clear();
        L.cnt.clear();
        if (!sorted) {
            thread_local std::vector<BEnt> e;
            sorted_block_entries(n, rp, ci, static_cast<std::size_t>(b), e);
            for (std::size_t i = 0; i < e.size(); ++i) {
                if (i == 0 || e[i].bc != e[i - 1].bc) {
                    L.bcol.push_back(e[i].bc);
                    L.mask.push_back(0);
                    L.cnt.push_back(0);
                }
                L.mask.back() |= static_cast<uint16_t>(1u << (e[i].r * 4 + e[i].c));
                L.cnt.back()++;
            }
            return;
        }
        std::size_t r0 = 4 * static_cast<std::size_t>(b), r1 = std::min(n, r0 + 4);
        int nr = static_cast<int>(r1 - r0);
        uint64_t pos[4], end[4];
        for (int r = 0; r < nr; ++r) {
            pos[r] = rp[r0 + r];
            end[r] = rp[r0 + r + 1];
        }
        while (true) {
            int64_t bc = INT64_MAX;
            for (int r = 0; r < nr; ++r)
                if (pos[r] < end[r]) bc = std::min<int64_t>(bc, ci[pos[r]] / 4);
            if (bc == INT64_MAX) break;
            uint16_t m = 0, c = 0;
            for (int r = 0; r < nr; ++r)
                while (pos[r] < end[r] && ci[pos[r]] / 4 == bc) {
                    m |= static_cast<uint16_t>(1u << (r * 4 + ci[pos[r]] % 4));
                    ++c;
                    ++pos[r];
                }
            L.bcol.push_back(static_cast<int32_t>(bc));
            L.mask.push_back(m);
            L.cnt.push_back(c);
        }
    };
    // Signature of a block-row: the sorted multiset of its block patterns (0 = none known).
    auto sig_of = [](const BlockRowLayout& L) -> int {
        if (L.mask.size() != static_cast<std::size_t>(kSigTopiBlocks)) return 0;
        uint16_t m[kSigTopiBlocks];
        std::copy(L.mask.begin(), L.mask.end(), m);
        std::sort(m, m + kSigTopiBlocks);
        for (int k = 0; k < kSigTopiBlocks; ++k)
            if (m[k] != kSigTopiMasks[k]) return 0;
        return 1;
    };
    // Pass 1: per-slot block and value counts, and block-row signatures.
    std::vector<int> nblk(s.perm.size(), 0);
    std::vector<std::size_t> nval(s.perm.size(), 0);
    std::vector<uint8_t> slot_sig(s.perm.size(), 0);
    parallel_ranges(s.perm.size(), [&](std::size_t lo, std::size_t hi) {
        BlockRowLayout L;
        for (std::size_t q = lo; q < hi; ++q)
            if (s.perm[q] >= 0) {
                nblk[q] = count_blocks(n, rp, ci, s.perm[q], &nval[q], sorted);
                if (nblk[q] == kSigTopiBlocks) {
                    layout_of(s.perm[q], L);
                    slot_sig[q] = static_cast<uint8_t>(sig_of(L));
                }
            }
    });
    // Pass 2 (serial, cheap): piece layout per chunk.
    struct PieceDesc {
        std::size_t chunk;
        int k0, kcnt;
        std::size_t nvals;
        uint16_t flags;
    };
    std::vector<PieceDesc> pd;
    pd.reserve(s.nchunks);
    std::vector<std::size_t> chunk_first_piece(s.nchunks + 1, 0);
    {
        std::vector<BlockRowLayout> L(C);
        for (std::size_t ch = 0; ch < s.nchunks; ++ch) {
            chunk_first_piece[ch] = pd.size();
            int kmax = 0;
            std::size_t tot = 0;
            for (int r = 0; r < C; ++r) {
                kmax = std::max(kmax, nblk[ch * C + r]);
                tot += nval[ch * C + r];
            }
            if (piece_bytes(C, kmax, tot) <= kStageBytes) {  // common case: one piece
                int sig = slot_sig[ch * C];
                for (int r = 1; r < C && sig; ++r)
                    if (slot_sig[ch * C + r] != sig) sig = 0;
                if (C != kDefaultC || std::getenv("CHEBFD_NO_SIG")) sig = 0;
                pd.push_back({ch, 0, kmax, tot, static_cast<uint16_t>(kPieceFirst | kPieceLast | (sig << kSigShift))});
                continue;
            }
            for (int r = 0; r < C; ++r)
                if (s.perm[ch * C + r] >= 0) layout_of(s.perm[ch * C + r], L[r]);
                else L[r] = BlockRowLayout{};
            int k0 = 0;
            bool first = true;
            while (k0 < kmax) {
                int kc = 0;
                std::size_t nv = 0;
                while (k0 + kc < kmax) {
                    std::size_t add = 0;
                    for (int r = 0; r < C; ++r)
                        if (k0 + kc < static_cast<int>(L[r].cnt.size())) add += L[r].cnt[k0 + kc];
                    if (piece_bytes(C, kc + 1, nv + add) > kStageBytes) break;
                    nv += add;
                    ++kc;
                }
                if (kc == 0) throw std::runtime_error("sell: block too large for a stage");
                uint16_t fl = (first ? kPieceFirst : 0) | (k0 + kc >= kmax ? kPieceLast : 0);
                pd.push_back({ch, k0, kc, nv, fl});
                first = false;
                k0 += kc;
            }
        }
        chunk_first_piece[s.nchunks] = pd.size();
    }
    // Offsets
    s.pieces.resize(pd.size());
    std::size_t off = 0;
    for (std::size_t p = 0; p < pd.size(); ++p) {
        std::size_t b = piece_bytes(C, pd[p].kcnt, pd[p].nvals);
        s.pieces[p] = {off, static_cast<uint32_t>(b), pd[p].flags};
        off += b;
    }
    s.records.assign(off, 0);
    // Pass 3 (threaded over pieces): fill records.
    std::atomic<int32_t> maxbc{0};
    std::atomic<bool> stage_ok{true};
    s.plans.assign(pd.size(), StagePlan{});
    parallel_ranges(pd.size(), [&](std::size_t lo, std::size_t hi) {
        std::vector<BlockRowLayout> L(C);
        std::size_t cur_chunk = SIZE_MAX;
        int32_t local_max = 0;
        for (std::size_t p = lo; p < hi; ++p) {
            const PieceDesc& d = pd[p];
            if (d.chunk != cur_chunk) {
                for (int r = 0; r < C; ++r)
                    if (s.perm[d.chunk * C + r] >= 0) layout_of(s.perm[d.chunk * C + r], L[r]);
                    else L[r] = BlockRowLayout{};
                cur_chunk = d.chunk;
            }
            uint8_t* rec = s.records.data() + s.pieces[p].offset;
            PieceHdr h{};
            int valid = 0;
            for (int r = 0; r < C; ++r) valid += s.perm[d.chunk * C + r] >= 0;
            h.nrows = static_cast<uint16_t>(valid);
            h.kcnt = static_cast<uint16_t>(d.kcnt);
            h.flags = d.flags;
            h.C = static_cast<uint16_t>(C);
            h.nvals = static_cast<uint32_t>(d.nvals);
            h.chunk = static_cast<uint32_t>(d.chunk);
            std::memcpy(rec, &h, sizeof h);
            int32_t* pperm = reinterpret_cast<int32_t*>(rec + 16);
            uint16_t* pnblk = reinterpret_cast<uint16_t*>(rec + 16 + 4 * C);
            BlockMeta* meta = reinterpret_cast<BlockMeta*>(rec + 16 + 4 * C + (2 * C + 15) / 16 * 16);
            double* vals = reinterpret_cast<double*>(meta + static_cast<std::size_t>(d.kcnt) * C);
            std::size_t vpos = 0;
            const int sig = d.flags >> kSigShift;
            for (int r = 0; r < C; ++r) {
                pperm[r] = s.perm[d.chunk * C + r];
                int have = static_cast<int>(L[r].bcol.size());
                pnblk[r] = static_cast<uint16_t>(std::max(0, std::min(d.kcnt, have - d.k0)));
                if (sig) {  // canonical block order: by (mask, bcol)
                    std::vector<int> ix(L[r].bcol.size());
                    std::iota(ix.begin(), ix.end(), 0);
                    std::stable_sort(ix.begin(), ix.end(), [&](int a, int b) { return L[r].mask[a] < L[r].mask[b]; });
                    BlockRowLayout o;
                    for (int i : ix) {
                        o.bcol.push_back(L[r].bcol[i]);
                        o.mask.push_back(L[r].mask[i]);
                        o.cnt.push_back(L[r].cnt[i]);
                    }
                    L[r] = std::move(o);
                }
            }
            // values ordered by (k, r) so each k-row of meta has increasing voff;
            // signature chunks are slot-major, (r, k)
            const int outer = sig ? C : d.kcnt, inner = sig ? d.kcnt : C;
            for (int o1 = 0; o1 < outer; ++o1)
                for (int i1 = 0; i1 < inner; ++i1) {
                    const int k = sig ? i1 : o1, r = sig ? o1 : i1;
                    BlockMeta& m = meta[static_cast<std::size_t>(k) * C + r];
                    int kk = d.k0 + k;
                    if (kk >= static_cast<int>(L[r].bcol.size())) {
                        m = {0, 0, 0};
                        continue;
                    }
                    m.bcol = L[r].bcol[kk];
                    m.mask = L[r].mask[kk];
                    m.voff = static_cast<uint16_t>(vpos);
                    local_max = std::max(local_max, m.bcol);
                    // copy this block's values row-major over the mask
                    std::size_t r0 = 4 * static_cast<std::size_t>(pperm[r]);
                    if (!sorted) {
                        thread_local std::vector<BEnt> e;
                        sorted_block_entries(n, rp, ci, static_cast<std::size_t>(pperm[r]), e);
                        for (const BEnt& x : e)
                            if (x.bc == m.bcol) {
                                vals[2 * vpos] = values[2 * x.k];
                                vals[2 * vpos + 1] = values[2 * x.k + 1];
                                ++vpos;
                            }
                        continue;
                    }
                    for (int rr = 0; rr < 4; ++rr) {
                        if (r0 + rr >= n) break;
                        for (uint64_t q = rp[r0 + rr]; q < rp[r0 + rr + 1]; ++q)
                            if (ci[q] / 4 == m.bcol) {
                                vals[2 * vpos] = values[2 * q];
                                vals[2 * vpos + 1] = values[2 * q + 1];
                                ++vpos;
                            }
                    }
                }
            if (vpos != d.nvals) throw std::logic_error("sell: value count mismatch");
            // staging plan: distinct block columns of the chunk (+ own block-rows), as runs
            uint8_t* sidx = rec + sidx_offset(C, d.kcnt, d.nvals);
            std::memset(sidx, 0xFF, static_cast<std::size_t>(d.kcnt + 1) * C);
            if ((d.flags & (kPieceFirst | kPieceLast)) != (kPieceFirst | kPieceLast)) {
                stage_ok = false;
            } else {
                std::vector<int32_t> cols;
                for (int r = 0; r < C; ++r) {
                    if (pperm[r] < 0) continue;
                    cols.push_back(pperm[r]);
                    for (int k = 0; k < pnblk[r]; ++k) cols.push_back(meta[static_cast<std::size_t>(k) * C + r].bcol);
                }
                std::sort(cols.begin(), cols.end());
                cols.erase(std::unique(cols.begin(), cols.end()), cols.end());
                StagePlan& pl = s.plans[p];
                int nr = 0;
                for (std::size_t i = 0; i < cols.size(); ++i) {
                    if (i == 0 || cols[i] != cols[i - 1] + 1) {
                        if (nr == kMaxRuns) {
                            nr = kMaxRuns + 1;
                            break;
                        }
                        pl.runs[nr++] = {cols[i], 0, static_cast<uint16_t>(i)};
                    }
                    ++pl.runs[nr - 1].len;
                }
                if (cols.size() > static_cast<std::size_t>(kMaxStage) || nr > kMaxRuns) {
                    stage_ok = false;
                } else {
                    pl.nruns = static_cast<uint16_t>(nr);
                    pl.nstaged = static_cast<uint16_t>(cols.size());
                    auto at = [&](int32_t bc) {
                        return static_cast<uint8_t>(std::lower_bound(cols.begin(), cols.end(), bc) - cols.begin());
                    };
                    for (int r = 0; r < C; ++r) {
                        if (pperm[r] < 0) continue;
                        for (int k = 0; k < pnblk[r]; ++k)
                            sidx[static_cast<std::size_t>(k) * C + r] = at(meta[static_cast<std::size_t>(k) * C + r].bcol);
                        sidx[static_cast<std::size_t>(d.kcnt) * C + r] = at(pperm[r]);
                    }
                }
            }
        }
        int32_t cur = maxbc.load();
        while (local_max > cur && !maxbc.compare_exchange_weak(cur, local_max)) {
        }
    });
    s.max_bcol = static_cast<std::size_t>(maxbc.load());
    s.staged = stage_ok.load() && !pd.empty();
    if (!s.staged) s.plans.clear();
    // Units: consecutive chunk ranges.
    std::size_t hint = std::max<std::size_t>(units_hint, 1);
    // >= 8 chunks per unit (more pieces than ring stages) keeps consumer warps of a
    // CTA within one unit of each other, which the double-buffered reduction relies on;
    // 16 at least: the narrow staged kernel takes 2-4 chunks per stage, and a unit of
    // 2 stages paid its per-unit costs too often (configs[0]: 8 -> 16 chunks, -7.5 %)
    std::size_t cpu = std::clamp<std::size_t>(s.nchunks / (hint * 8), 16, 32);
    if (const char* e = std::getenv("CHEBFD_UNIT_CHUNKS")) cpu = std::max<long>(8, std::atol(e));
    // the last units (about two per worker CTA) are half as long, so the kernel's
    // tail -- CTAs idle while the last units finish -- is half a short unit, not a
    // long one (CHEBFD_UNIT_TAIL=0: uniform units)
    std::size_t tail = 0;
    if (cpu >= 16 && !(std::getenv("CHEBFD_UNIT_TAIL") && std::atoi(std::getenv("CHEBFD_UNIT_TAIL")) == 0))
        tail = std::min(s.nchunks / 4, hint * (cpu / 2));
    s.unit_piece.clear();
    for (std::size_t ch = 0; ch < s.nchunks;) {
        s.unit_piece.push_back(static_cast<int32_t>(chunk_first_piece[ch]));
        ch += ch + tail >= s.nchunks ? cpu / 2 : cpu;
    }
    s.unit_piece.push_back(static_cast<int32_t>(pd.size()));
    return s;
}

void sell_to_crs(const SellHost& s, std::vector<uint64_t>& rp, std::vector<int32_t>& ci, std::vector<double>& v) {
    std::vector<std::vector<std::pair<int32_t, std::pair<double, double>>>> rows(s.n);
    for (std::size_t p = 0; p < s.pieces.size(); ++p) {
        const uint8_t* rec = s.records.data() + s.pieces[p].offset;
        PieceHdr h;
        std::memcpy(&h, rec, 16);
        int C = h.C;
        const int32_t* pperm = reinterpret_cast<const int32_t*>(rec + 16);
        const uint16_t* pnblk = reinterpret_cast<const uint16_t*>(rec + 16 + 4 * C);
        const BlockMeta* meta = reinterpret_cast<const BlockMeta*>(rec + 16 + 4 * C + (2 * C + 15) / 16 * 16);
        const double* vals = reinterpret_cast<const double*>(meta + static_cast<std::size_t>(h.kcnt) * C);
        for (int k = 0; k < h.kcnt; ++k)
            for (int r = 0; r < C; ++r) {
                if (k >= pnblk[r]) continue;
                const BlockMeta& m = meta[static_cast<std::size_t>(k) * C + r];
                int idx = m.voff;
                for (int rr = 0; rr < 4; ++rr)
                    for (int c = 0; c < 4; ++c)
                        if (m.mask >> (rr * 4 + c) & 1) {
                            std::size_t row = 4 * static_cast<std::size_t>(pperm[r]) + rr;
                            rows[row].push_back({m.bcol * 4 + c, {vals[2 * idx], vals[2 * idx + 1]}});
                            ++idx;
                        }
            }
    }
    rp.assign(s.n + 1, 0);
    ci.clear();
    v.clear();
    for (std::size_t i = 0; i < s.n; ++i) {
        rp[i + 1] = rp[i] + rows[i].size();
        // signature chunks store blocks in (mask, bcol) order: restore ascending columns
        std::sort(rows[i].begin(), rows[i].end(), [](const auto& a, const auto& b) { return a.first < b.first; });
        for (auto& e : rows[i]) {
            ci.push_back(e.first);
            v.push_back(e.second.first);
            v.push_back(e.second.second);
        }
    }
}

void fill_random_columns(std::size_t n, std::size_t j0, std::size_t j1, uint64_t seed, double* out) {
    const std::size_t w = j1 - j0;
    parallel_ranges(n, [&](std::size_t lo, std::size_t hi) {
        for (std::size_t i = lo; i < hi; ++i)
            for (std::size_t j = j0; j < j1; ++j) unit_gauss(seed, i, j, out + 2 * (i * w + (j - j0)));
    });
}
}  // namespace cfb

using namespace cfb;

// ======================================================== C ABI (host) ===
extern "C" {

const char* cf_last_error(void) { return g_err.c_str(); }
int cf_version(void) { return 1; }

int cf_topi_generate(size_t nx, size_t ny, size_t nz, double mass, double hop, int open_boundary, size_t* n,
                     size_t* nnz, uint64_t* row_ptr, int32_t* col_idx, double* values) {
    return guard([&] {
        Crs m = topi_crs(nx, ny, nz, mass, hop, open_boundary != 0);
        *n = m.n;
        *nnz = m.col_idx.size();
        if (row_ptr) {
            std::memcpy(row_ptr, m.row_ptr.data(), (m.n + 1) * 8);
            std::memcpy(col_idx, m.col_idx.data(), m.col_idx.size() * 4);
            std::memcpy(values, m.values.data(), m.values.size() * 8);
        }
    });
}

int cf_gershgorin_bounds(size_t n, const uint64_t* rp, const int32_t* ci, const double* v, double* lo, double* hi) {
    return guard([&] {  // sparse_matrix.hpp:89-107
        if (n == 0) throw std::invalid_argument("empty matrix");
        double l = std::numeric_limits<double>::infinity(), h = -l;
        for (size_t i = 0; i < n; ++i) {
            double diag = 0.0, radius = 0.0;
            for (uint64_t k = rp[i]; k < rp[i + 1]; ++k) {
                if (static_cast<size_t>(ci[k]) == i) diag = v[2 * k];
                else radius += std::hypot(v[2 * k], v[2 * k + 1]);
            }
            l = std::min(l, diag - radius);
            h = std::max(h, diag + radius);
        }
        *lo = l;
        *hi = h;
    });
}

int cf_jacobi_hermitian_eig(size_t k, const double* A, double tol, size_t max_sweeps, double* values,
                            double* vectors) {
    return guard([&] {  // jacobi_eig.hpp:32-98
        std::vector<double> a(A, A + 2 * k * k), vals, vecs;
        jacobi_hermitian(k, std::move(a), tol, max_sweeps, vals, vecs);
        std::copy(vals.begin(), vals.end(), values);
        if (vectors) std::copy(vecs.begin(), vecs.end(), vectors);
    });
}

int cf_spectral_map(double lmin, double lmax, double margin, double* alpha, double* beta) {
    return guard([&] {  // filter.hpp:25-32
        if (!(lmax > lmin)) throw std::invalid_argument("degenerate spectral interval");
        if (margin < 0.0) throw std::invalid_argument("margin must be >= 0");
        *alpha = 2.0 / ((lmax - lmin) * (1.0 + margin));
        *beta = -*alpha * (lmax + lmin) / 2.0;
    });
}

int cf_filter_coefficients(double wlo, double whi, double alpha, double beta, size_t np, int damping, double* c,
                           double* g) {
    return guard([&] {  // filter.hpp:39-70
        if (np < 2) throw std::invalid_argument("polynomial degree must be >= 2");
        double a = alpha * wlo + beta, b = alpha * whi + beta;
        if (!(a < b) || a <= -1.0 || b >= 1.0) throw std::invalid_argument("window must map strictly inside (-1, 1)");
        const double pi = 3.14159265358979323846;
        double ta = std::acos(a), tb = std::acos(b);
        c[0] = (ta - tb) / pi;
        for (size_t p = 1; p <= np; ++p)
            c[p] = 2.0 / (pi * static_cast<double>(p)) * (std::sin(p * ta) - std::sin(p * tb));
        g[0] = 1.0;
        if (damping == 0) {
            double q = pi / static_cast<double>(np + 1);
            double cot_q = std::cos(q) / std::sin(q);
            for (size_t p = 1; p <= np; ++p)
                g[p] = ((np - p + 1) * std::cos(p * q) + std::sin(p * q) * cot_q) / static_cast<double>(np + 1);
        } else {
            for (size_t p = 1; p <= np; ++p) g[p] = 1.0;
        }
    });
}

int cf_blockvec_random(size_t n, size_t ns, size_t nb, uint64_t seed, uint64_t row_offset, double* out) {
    return guard([&] {  // block_vector.hpp:57-73
        if (n < 1) throw std::invalid_argument("n must be >= 1");
        if (nb == 0 || ns == 0 || ns % nb != 0) throw std::invalid_argument("n_b must divide n_s");
        parallel_ranges(n, [&](size_t lo, size_t hi) {
            for (size_t j = 0; j < ns; ++j)
                for (size_t i = lo; i < hi; ++i) {
                    size_t off = (j / nb) * n * nb + i * nb + j % nb;
                    unit_gauss(seed, row_offset + i, j, out + 2 * off);
                }
        });
    });
}

int cf_partition_rows(size_t n, const uint64_t* rp, const int32_t* ci, size_t workers, uint64_t* ranges,
                      uint64_t* halo, size_t* halo_len) {
    return guard([&] {  // partition.hpp:28-60
        if (workers < 1) throw std::invalid_argument("workers must be >= 1");
        size_t granule = (n % 4 == 0) ? 4 : 1;
        size_t units = n / granule;
        if (workers > units) throw std::invalid_argument("more workers than row blocks");
        std::vector<std::pair<size_t, size_t>> rg(workers);
        for (size_t w = 0; w < workers; ++w) rg[w] = {units * w / workers * granule, units * (w + 1) / workers * granule};
        auto owner_of = [&](size_t row) {
            auto it = std::upper_bound(rg.begin(), rg.end(), row,
                                       [](size_t r, const std::pair<size_t, size_t>& x) { return r < x.second; });
            return static_cast<size_t>(it - rg.begin());
        };
        size_t len = 0;
        for (size_t w = 0; w < workers; ++w) {
            if (ranges) {
                ranges[2 * w] = rg[w].first;
                ranges[2 * w + 1] = rg[w].second;
            }
            std::vector<int32_t> remote;
            for (size_t i = rg[w].first; i < rg[w].second; ++i)
                for (uint64_t k = rp[i]; k < rp[i + 1]; ++k) {
                    size_t c = static_cast<size_t>(ci[k]);
                    if (c < rg[w].first || c >= rg[w].second) remote.push_back(ci[k]);
                }
            std::sort(remote.begin(), remote.end());
            remote.erase(std::unique(remote.begin(), remote.end()), remote.end());
            size_t cur = SIZE_MAX, rec = 0;
            for (int32_t c : remote) {
                size_t v = owner_of(static_cast<size_t>(c));
                if (v != cur) {
                    cur = v;
                    rec = len;
                    if (halo) {
                        halo[len] = w;
                        halo[len + 1] = v;
                        halo[len + 2] = 0;
                    }
                    len += 3;
                }
                if (halo) {
                    halo[len] = static_cast<uint64_t>(c);
                    halo[rec + 2]++;
                }
                ++len;
            }
        }
        *halo_len = len;
    });
}

int cf_shard(size_t n, const uint64_t* rp, const int32_t* ci, const double* v, size_t workers, size_t w,
             size_t* row_begin, size_t* local_n, size_t* halo_n, size_t* nnz, uint64_t* out_rp, int32_t* out_ci,
             double* out_v, uint64_t* halo_global, uint64_t* send_flat, size_t* send_len, uint64_t* recv_flat,
             size_t* recv_len) {
    return guard([&] {  // dist.hpp:39-98
        size_t hl = 0;
        int st = cf_partition_rows(n, rp, ci, workers, nullptr, nullptr, &hl);
        if (st) throw std::invalid_argument(g_err);
        std::vector<uint64_t> ranges(2 * workers), halo(hl);
        cf_partition_rows(n, rp, ci, workers, ranges.data(), halo.data(), &hl);
        if (w >= workers) throw std::out_of_range("worker index out of range");
        size_t rb = ranges[2 * w], re = ranges[2 * w + 1], ln = re - rb;
        // halo_in[w] (recv) and halo_out[w] = halo_in[v][w] for v (send), neighbors ascending
        std::map<size_t, std::vector<uint64_t>> hin, hout;
        for (size_t q = 0; q < hl;) {
            size_t ww = halo[q], vv = halo[q + 1], cnt = halo[q + 2];
            std::vector<uint64_t> rows(halo.begin() + q + 3, halo.begin() + q + 3 + cnt);
            if (ww == w) hin[vv] = rows;
            if (vv == w) hout[ww] = rows;
            q += 3 + cnt;
        }
        std::vector<uint64_t> hg;
        std::map<uint64_t, size_t> slot_of;
        std::vector<uint64_t> recv, send;
        for (auto& [nbr, rows] : hin) {
            recv.push_back(nbr);
            recv.push_back(rows.size());
            for (uint64_t g : rows) {
                slot_of[g] = hg.size();
                recv.push_back(ln + hg.size());
                hg.push_back(g);
            }
        }
        for (auto& [nbr, rows] : hout) {
            send.push_back(nbr);
            send.push_back(rows.size());
            for (uint64_t g : rows) send.push_back(g - rb);
        }
        *row_begin = rb;
        *local_n = ln;
        *halo_n = hg.size();
        *nnz = rp[re] - rp[rb];
        *send_len = send.size();
        *recv_len = recv.size();
        if (out_rp) {
            out_rp[0] = 0;
            size_t k2 = 0;
            for (size_t i = rb; i < re; ++i) {
                for (uint64_t k = rp[i]; k < rp[i + 1]; ++k, ++k2) {
                    size_t c = static_cast<size_t>(ci[k]);
                    size_t lc = (c >= rb && c < re) ? c - rb : ln + slot_of.at(c);
                    out_ci[k2] = static_cast<int32_t>(lc);
                    out_v[2 * k2] = v[2 * k];
                    out_v[2 * k2 + 1] = v[2 * k + 1];
                }
                out_rp[i - rb + 1] = k2;
            }
            std::memcpy(halo_global, hg.data(), hg.size() * 8);
            std::memcpy(send_flat, send.data(), send.size() * 8);
            std::memcpy(recv_flat, recv.data(), recv.size() * 8);
        }
    });
}

int cf_topi_shard(size_t nx, size_t ny, size_t nz, double mass, double hop, int open_boundary, size_t workers,
                  size_t w, size_t* row_begin, size_t* local_n, size_t* halo_n, size_t* nnz, uint64_t* out_rp,
                  int32_t* out_ci, double* out_v, uint64_t* halo_global, uint64_t* send_flat, size_t* send_len,
                  uint64_t* recv_flat, size_t* recv_len) {
    return guard([&] {
        if (nx < 1 || ny < 1 || nz < 1) throw std::invalid_argument("lattice extents must be positive");
        if (workers < 1) throw std::invalid_argument("workers must be >= 1");
        const size_t S = nx * ny * nz;
        if (4 * S > static_cast<size_t>(INT32_MAX)) throw std::invalid_argument("topi: dimension exceeds int32 columns");
        if (workers > S) throw std::invalid_argument("more workers than row blocks");
        if (w >= workers) throw std::out_of_range("worker index out of range");
        TopiSpec t = make_topi(nx, ny, nz, mass, hop, open_boundary != 0);
        // partition.hpp:30-41 with granule 4 (n % 4 == 0)
        std::vector<std::pair<size_t, size_t>> rg(workers);
        for (size_t v = 0; v < workers; ++v) rg[v] = {S * v / workers * 4, S * (v + 1) / workers * 4};
        auto owner_of = [&](size_t row) {
            auto it = std::upper_bound(rg.begin(), rg.end(), row,
                                       [](size_t r, const std::pair<size_t, size_t>& x) { return r < x.second; });
            return static_cast<size_t>(it - rg.begin());
        };
        const size_t rb = rg[w].first, re = rg[w].second, ln = re - rb;
        // own rows in closed form (global columns)
        std::vector<uint64_t> rp(ln + 1, 0);
        parallel_ranges(ln / 4, [&](size_t lo, size_t hi) {
            int32_t cols[32];
            double vals[64];
            for (size_t s = lo; s < hi; ++s)
                for (int r = 0; r < 4; ++r) rp[4 * s + r + 1] = topi_row(t, rb / 4 + s, r, cols, vals);
        });
        for (size_t i = 0; i < ln; ++i) rp[i + 1] += rp[i];
        std::vector<int32_t> gc(rp[ln]);
        std::vector<double> gv(2 * rp[ln]);
        parallel_ranges(ln / 4, [&](size_t lo, size_t hi) {
            for (size_t s = lo; s < hi; ++s)
                for (int r = 0; r < 4; ++r) {
                    size_t i = 4 * s + r;
                    topi_row(t, rb / 4 + s, r, gc.data() + rp[i], gv.data() + 2 * rp[i]);
                }
        });
        // halo_in[w]: remote columns, sorted, grouped by owner (partition.hpp:44-56)
        std::vector<int32_t> remote;
        for (int32_t c : gc)
            if (static_cast<size_t>(c) < rb || static_cast<size_t>(c) >= re) remote.push_back(c);
        std::sort(remote.begin(), remote.end());
        remote.erase(std::unique(remote.begin(), remote.end()), remote.end());
        std::vector<uint64_t> hg, recv, send;
        std::unordered_map<int32_t, size_t> slot_of;
        for (size_t q = 0; q < remote.size();) {
            size_t v = owner_of(static_cast<size_t>(remote[q]));
            size_t q1 = q;
            while (q1 < remote.size() && owner_of(static_cast<size_t>(remote[q1])) == v) ++q1;
            recv.push_back(v);
            recv.push_back(q1 - q);
            for (size_t k = q; k < q1; ++k) {
                slot_of[remote[k]] = hg.size();
                recv.push_back(ln + hg.size());
                hg.push_back(static_cast<uint64_t>(remote[k]));
            }
            q = q1;
        }
        // halo_out[w][v] = halo_in[v][w] = own rows with a column owned by v (symmetric pattern)
        std::map<size_t, std::vector<uint64_t>> out;
        for (size_t i = 0; i < ln; ++i) {
            size_t last = SIZE_MAX;
            std::vector<size_t> owners;
            for (uint64_t k = rp[i]; k < rp[i + 1]; ++k) {
                size_t c = static_cast<size_t>(gc[k]);
                if (c >= rb && c < re) continue;
                size_t v = owner_of(c);
                if (std::find(owners.begin(), owners.end(), v) == owners.end()) owners.push_back(v);
            }
            (void)last;
            for (size_t v : owners) out[v].push_back(i);
        }
        for (auto& [v, rows] : out) {
            send.push_back(v);
            send.push_back(rows.size());
            for (uint64_t r : rows) send.push_back(r);
        }
        *row_begin = rb;
        *local_n = ln;
        *halo_n = hg.size();
        *nnz = rp[ln];
        *send_len = send.size();
        *recv_len = recv.size();
        if (out_rp) {
            std::memcpy(out_rp, rp.data(), (ln + 1) * 8);
            for (size_t k = 0; k < gc.size(); ++k) {
                size_t c = static_cast<size_t>(gc[k]);
                out_ci[k] = static_cast<int32_t>((c >= rb && c < re) ? c - rb : ln + slot_of.at(gc[k]));
            }
            std::memcpy(out_v, gv.data(), gv.size() * 8);
            std::memcpy(halo_global, hg.data(), hg.size() * 8);
            std::memcpy(send_flat, send.data(), send.size() * 8);
            std::memcpy(recv_flat, recv.data(), recv.size() * 8);
        }
    });
}

int cf_sell_permutation(size_t n, const uint64_t* rp, const int32_t* ci, const int32_t* order, int C, int sigma,
                        int32_t* perm_out, size_t* nslots) {
    return guard([&] {
        auto p = sell_permutation(n, rp, ci, order, C, sigma);
        *nslots = p.size();
        if (perm_out) std::memcpy(perm_out, p.data(), p.size() * 4);
    });
}

int cf_sell_layout_stats(size_t n, size_t ncols, const uint64_t* rp, const int32_t* ci, const double* v,
                         const int32_t* order, size_t* stats) {
    return guard([&] {  // host-side build only (no device): what the kernels will see
        SellHost s = build_sell(n, ncols, rp, ci, v, order, kDefaultC, kDefaultC, 296);
        size_t sig = 0, max_runs = 0, max_staged = 0, total_staged = 0;
        for (std::size_t p = 0; p < s.pieces.size(); ++p) {
            PieceHdr h;
            std::memcpy(&h, s.records.data() + s.pieces[p].offset, sizeof h);
            sig += (h.flags >> kSigShift) != 0;
            if (s.staged) {
                max_runs = std::max<size_t>(max_runs, s.plans[p].nruns);
                max_staged = std::max<size_t>(max_staged, s.plans[p].nstaged);
                total_staged += s.plans[p].nstaged;
            }
        }
        stats[0] = s.nchunks;
        stats[1] = s.pieces.size();
        stats[2] = s.unit_piece.size() - 1;
        stats[3] = s.staged ? 1 : 0;
        stats[4] = sig;
        stats[5] = max_runs;
        stats[6] = max_staged;
        stats[7] = total_staged;
        stats[8] = s.records.size();
    });
}

int cf_lattice_order(size_t nx, size_t ny, size_t nz, size_t tx, size_t ty, int32_t* order) {
    return guard([&] {
        auto o = lattice_order(nx, ny, nz, tx, ty, false);
        std::memcpy(order, o.data(), o.size() * 4);
    });
}

int cf_lattice_order_boundary_first(size_t nx, size_t ny, size_t nz, size_t tx, size_t ty, int32_t* order) {
    return guard([&] {
        auto o = lattice_order(nx, ny, nz, tx, ty, true);
        std::memcpy(order, o.data(), o.size() * 4);
    });
}

}  // extern "C"
