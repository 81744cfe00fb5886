// chebfilter_b200.hpp -- drop-in C++ front end for the B200 hot path.
//
// Re-creates the reference's operator API (namespace chebfilter, proj/include/
// chebfilter/{sparse_matrix,block_vector,kernels,filter,jacobi_eig}.hpp) on top of the C
// ABI in chebfd_b200.h.  A reference caller replaces its includes with this one
// header and links libchebfd_b200.so; the names, signatures, argument meaning
// and exception types are the reference's.  Differences a caller can observe:
//   * BlockVector panels live in GPU memory with a host mirror that is synced
//     on access (panel(b), operator(), SubblockView::data()); kernels run on the
//     device and never touch the host copy.
//   * A SparseMatrixCRS is uploaded (as SELL-C-sigma over 4x4 blocks) on first
//     use; it must not be modified afterwards (the reference treats it as const).
//   * Results agree with the CPU reference to rounding (FMA contraction), see
//     DESIGN.md section 2; the reference's unfused chebfd_op_reference is test
//     infrastructure and is not provided.
#pragma once

#include <algorithm>
#include <cmath>
#include <complex>
#include <cstdint>
#include <cstring>
#include <limits>
#include <map>
#include <memory>
#include <optional>
#include <stdexcept>
#include <string>
#include <utility>
#include <array>
#include <variant>
#include <vector>

#include "chebfd_b200.h"

namespace chebfilter {

using cplx = std::complex<double>;

struct ProtocolError : std::logic_error {
    using std::logic_error::logic_error;
};

namespace detail {
// CF_E* status -> the reference's exception types
inline void check(int st) {
    if (st == CF_OK) return;
    std::string msg = cf_last_error();
    switch (st) {
        case CF_EINVAL: throw std::invalid_argument(msg);
        case CF_ERANGE: throw std::out_of_range(msg);
        case CF_EPROTOCOL: throw ProtocolError(msg);
        default: throw std::runtime_error(msg);
    }
}
// Device of this thread's matrices and panels: the one set_device() chose, else
// the thread's current CUDA device (so a caller's cudaSetDevice carries over).
inline int& device_override() {
    static thread_local int d = -1;
    return d;
}
inline int device() {
    if (device_override() >= 0) return device_override();
    int d = 0;
    check(cf_current_device(&d));
    return d;
}

struct DevBuf {  // owning device allocation
    void* p = nullptr;
    std::size_t bytes = 0;
    DevBuf() = default;
    explicit DevBuf(std::size_t b) : bytes(b) { check(cf_dev_alloc(device(), b, &p)); }
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    ~DevBuf() {
        if (p) cf_dev_free(p);
    }
};
}  // namespace detail

// Select the GPU this thread's matrices and block vectors are placed on (a
// B200-side addition; the reference is CPU-only).  -1 restores the default
// (the thread's current CUDA device).
inline void set_device(int dev) { detail::device_override() = dev; }

// ------------------------------------------------------ sparse_matrix.hpp ---
enum class Symmetry { hermitian, general };

struct SparseMatrixCRS {
    std::size_t n = 0;
    std::vector<std::size_t> row_ptr;
    std::vector<std::int32_t> col_idx;
    std::vector<cplx> values;
    Symmetry symmetry = Symmetry::hermitian;

    std::size_t nnz() const { return values.size(); }
    double avg_nnz_per_row() const { return n ? static_cast<double>(nnz()) / static_cast<double>(n) : 0.0; }

    // device image (built on first use)
    struct Dev {
        cf_matrix h = nullptr;
        std::size_t n = 0, nnz = 0;
        const void* key = nullptr;
        ~Dev() {
            if (h) cf_matrix_destroy(h);
        }
    };
    mutable std::shared_ptr<Dev> dev_;
    std::size_t ncols_ = 0;  // > n for shard-local matrices with halo columns

    cf_matrix device_handle() const {
        if (!dev_ || dev_->n != n || dev_->nnz != nnz() || dev_->key != values.data()) {
            auto d = std::make_shared<Dev>();
            std::vector<uint64_t> rp(row_ptr.begin(), row_ptr.end());
            std::size_t nc = std::max(ncols_, n);
            detail::check(cf_matrix_create_crs(detail::device(), n, nc, rp.data(), col_idx.data(),
                                               reinterpret_cast<const double*>(values.data()), nullptr, 0, 0, &d->h));
            d->n = n;
            d->nnz = nnz();
            d->key = values.data();
            dev_ = d;
        }
        return dev_->h;
    }
};

struct Triplet {
    std::size_t row;
    std::size_t col;
    cplx value;
};

inline SparseMatrixCRS build_from_triplets(std::size_t n, const std::vector<Triplet>& trips,
                                           Symmetry sym = Symmetry::hermitian) {
    std::vector<std::map<std::int32_t, cplx>> rows(n);
    for (const auto& t : trips) {
        if (t.row >= n || t.col >= n) throw std::invalid_argument("triplet index out of range");
        rows[t.row][static_cast<std::int32_t>(t.col)] += t.value;
    }
    SparseMatrixCRS H;
    H.n = n;
    H.symmetry = sym;
    H.row_ptr.assign(n + 1, 0);
    for (std::size_t i = 0; i < n; ++i) H.row_ptr[i + 1] = H.row_ptr[i] + rows[i].size();
    for (std::size_t i = 0; i < n; ++i)
        for (const auto& [c, v] : rows[i]) {
            H.col_idx.push_back(c);
            H.values.push_back(v);
        }
    return H;
}

inline SparseMatrixCRS diagonal_matrix(const std::vector<double>& d) {
    std::vector<Triplet> trips;
    for (std::size_t i = 0; i < d.size(); ++i) trips.push_back({i, i, cplx(d[i], 0.0)});
    return build_from_triplets(d.size(), trips, Symmetry::hermitian);
}

inline std::pair<double, double> gershgorin_bounds(const SparseMatrixCRS& H) {
    if (H.symmetry != Symmetry::hermitian) throw std::invalid_argument("gershgorin_bounds requires a hermitian matrix");
    std::vector<uint64_t> rp(H.row_ptr.begin(), H.row_ptr.end());
    double lo, hi;
    detail::check(cf_gershgorin_bounds(H.n, rp.data(), H.col_idx.data(),
                                       reinterpret_cast<const double*>(H.values.data()), &lo, &hi));
    return {lo, hi};
}

enum class Boundary { periodic, open };

struct LatticeSpec {
    std::size_t nx = 1, ny = 1, nz = 1;
    double mass = 1.0;
    double hop = 1.0;
    Boundary boundary = Boundary::periodic;
    std::uint64_t seed = 0;
    std::size_t sites() const { return nx * ny * nz; }
    std::size_t dim() const { return 4 * sites(); }
};

inline SparseMatrixCRS topi_generate(const LatticeSpec& s) {
    std::size_t n, nnz;
    const int op = s.boundary == Boundary::open ? 1 : 0;
    detail::check(cf_topi_generate(s.nx, s.ny, s.nz, s.mass, s.hop, op, &n, &nnz, nullptr, nullptr, nullptr));
    std::vector<uint64_t> rp(n + 1);
    SparseMatrixCRS H;
    H.n = n;
    H.col_idx.resize(nnz);
    H.values.resize(nnz);
    detail::check(cf_topi_generate(s.nx, s.ny, s.nz, s.mass, s.hop, op, &n, &nnz, rp.data(), H.col_idx.data(),
                                   reinterpret_cast<double*>(H.values.data())));
    H.row_ptr.assign(rp.begin(), rp.end());
    return H;
}

// ------------------------------------------------------- block_vector.hpp ---
struct InitZero {};
struct InitConstant {
    cplx value;
};
struct InitSeededRandom {
    std::uint64_t seed;
    std::uint64_t row_offset = 0;
};
using BlockVectorInit = std::variant<InitZero, InitConstant, InitSeededRandom>;

class SubblockView;

class BlockVector {
  public:
    BlockVector() = default;
    BlockVector(std::size_t n, std::size_t n_s, std::size_t n_b, const BlockVectorInit& init = InitZero{})
        : n_(n), ns_(n_s), nb_(n_b) {
        if (n < 1) throw std::invalid_argument("n must be >= 1");
        if (n_b == 0 || n_s == 0 || n_s % n_b != 0) throw std::invalid_argument("n_b must divide n_s");
        const std::size_t np = n_s / n_b;
        host_.assign(np, std::vector<cplx>(n * n_b));
        if (std::holds_alternative<InitConstant>(init)) {
            for (auto& p : host_) std::fill(p.begin(), p.end(), std::get<InitConstant>(init).value);
        } else if (std::holds_alternative<InitSeededRandom>(init)) {
            const auto& r = std::get<InitSeededRandom>(init);
            std::vector<cplx> all(n * n_s);
            detail::check(cf_blockvec_random(n, n_s, n_b, r.seed, r.row_offset, reinterpret_cast<double*>(all.data())));
            for (std::size_t b = 0; b < np; ++b)
                std::copy(all.begin() + b * n * n_b, all.begin() + (b + 1) * n * n_b, host_[b].begin());
        }
        for (std::size_t b = 0; b < np; ++b) dev_.push_back(std::make_shared<detail::DevBuf>(n * n_b * 16));
        host_ok_.assign(np, 1);
        dev_ok_.assign(np, 0);
    }
    BlockVector(const BlockVector& o) : n_(o.n_), ns_(o.ns_), nb_(o.nb_) {
        for (std::size_t b = 0; b < o.panel_count(); ++b) o.sync_host(b);
        host_ = o.host_;
        for (std::size_t b = 0; b < host_.size(); ++b) dev_.push_back(std::make_shared<detail::DevBuf>(n_ * nb_ * 16));
        host_ok_.assign(host_.size(), 1);
        dev_ok_.assign(host_.size(), 0);
    }
    BlockVector& operator=(const BlockVector& o) {
        if (this != &o) {
            BlockVector t(o);
            *this = std::move(t);
        }
        return *this;
    }
    BlockVector(BlockVector&&) = default;
    BlockVector& operator=(BlockVector&&) = default;

    std::size_t rows() const { return n_; }
    std::size_t cols() const { return ns_; }
    std::size_t block_width() const { return nb_; }
    std::size_t panel_count() const { return host_.size(); }

    cplx& operator()(std::size_t i, std::size_t j) {
        check(i, j);
        return panel(j / nb_)[i * nb_ + j % nb_];
    }
    const cplx& operator()(std::size_t i, std::size_t j) const {
        check(i, j);
        return panel(j / nb_)[i * nb_ + j % nb_];
    }
    std::size_t linear_offset(std::size_t i, std::size_t j) const {
        check(i, j);
        return (j / nb_) * n_ * nb_ + i * nb_ + j % nb_;
    }
    std::vector<cplx>& panel(std::size_t b) {
        range(b);
        sync_host(b);
        dev_ok_[b] = 0;  // the caller may write through the reference
        return host_[b];
    }
    const std::vector<cplx>& panel(std::size_t b) const {
        range(b);
        sync_host(b);
        return host_[b];
    }

    // identity of a panel buffer (follows it through swap_blocks); used for alias checks
    const void* panel_identity(std::size_t b) const {
        range(b);
        return dev_[b].get();
    }
    // overwrite panel b with n*n_b complex from device memory (solver outputs)
    void load_device_panel(std::size_t b, const void* src) {
        range(b);
        detail::check(cf_memcpy(dev_[b]->p, src, host_[b].size() * 16, 2));
        dev_ok_[b] = 1;
        host_ok_[b] = 0;
    }
    // device side (used by the kernels)
    void* device_panel(std::size_t b, bool will_write) {
        range(b);
        if (!dev_ok_[b]) {
            detail::check(cf_memcpy(dev_[b]->p, host_[b].data(), host_[b].size() * 16, 0));
            dev_ok_[b] = 1;
        }
        if (will_write) host_ok_[b] = 0;
        return dev_[b]->p;
    }

  private:
    friend void swap_blocks(SubblockView a, SubblockView b);
    void check(std::size_t i, std::size_t j) const {
        if (i >= n_ || j >= ns_) throw std::out_of_range("block vector index out of range");
    }
    void range(std::size_t b) const {
        if (b >= host_.size()) throw std::invalid_argument("panel index out of range");
    }
    void sync_host(std::size_t b) const {
        if (!host_ok_[b]) {
            detail::check(cf_memcpy(const_cast<cplx*>(host_[b].data()), dev_[b]->p, host_[b].size() * 16, 1));
            host_ok_[b] = 1;
        }
    }
    std::size_t n_ = 0, ns_ = 0, nb_ = 0;
    mutable std::vector<std::vector<cplx>> host_;
    std::vector<std::shared_ptr<detail::DevBuf>> dev_;
    mutable std::vector<char> host_ok_, dev_ok_;
};

class SubblockView {
  public:
    SubblockView(BlockVector& parent, std::size_t b) : parent_(&parent), b_(b) {
        if (b >= parent.panel_count()) throw std::invalid_argument("panel index out of range");
    }
    std::size_t rows() const { return parent_->rows(); }
    std::size_t width() const { return parent_->block_width(); }
    std::size_t panel_index() const { return b_; }
    cplx* data() { return parent_->panel(b_).data(); }
    const cplx* data() const { return static_cast<const BlockVector*>(parent_)->panel(b_).data(); }
    cplx& operator()(std::size_t i, std::size_t j) {
        bounds(i, j);
        return data()[i * width() + j];
    }
    const cplx& operator()(std::size_t i, std::size_t j) const {
        bounds(i, j);
        return data()[i * width() + j];
    }
    void* device(bool will_write) const { return parent_->device_panel(b_, will_write); }
    const void* identity() const { return parent_->panel_identity(b_); }

    friend void swap_blocks(SubblockView a, SubblockView b) {
        if (a.rows() != b.rows() || a.width() != b.width()) throw std::invalid_argument("swap_blocks: shape mismatch");
        BlockVector& A = *a.parent_;
        BlockVector& B = *b.parent_;
        std::swap(A.host_[a.b_], B.host_[b.b_]);
        std::swap(A.dev_[a.b_], B.dev_[b.b_]);
        std::swap(A.host_ok_[a.b_], B.host_ok_[b.b_]);
        std::swap(A.dev_ok_[a.b_], B.dev_ok_[b.b_]);
    }

  private:
    void bounds(std::size_t i, std::size_t j) const {
        if (i >= rows() || j >= width()) throw std::out_of_range("subblock index out of range");
    }
    BlockVector* parent_;
    std::size_t b_;
};

// ------------------------------------------------------------ kernels.hpp ---
struct ShiftScale {
    double alpha = 1.0;
    double beta = 0.0;
};

struct MomentSeries {
    std::size_t degree_max = 2;
    std::size_t columns = 0;
    std::vector<cplx> eta;
    std::vector<cplx> mu;
    MomentSeries() = default;
    MomentSeries(std::size_t np, std::size_t ns) : degree_max(np), columns(ns) {
        std::size_t rows = np >= 3 ? np - 2 : 0;
        eta.assign(rows * ns, cplx(0.0));
        mu.assign(rows * ns, cplx(0.0));
    }
    std::size_t index(std::size_t p, std::size_t j) const {
        if (p < 3 || p > degree_max || j >= columns) throw std::out_of_range("moment index out of range");
        return (p - 3) * columns + j;
    }
    cplx& eta_at(std::size_t p, std::size_t j) { return eta[index(p, j)]; }
    cplx& mu_at(std::size_t p, std::size_t j) { return mu[index(p, j)]; }
    const cplx& eta_at(std::size_t p, std::size_t j) const { return eta[index(p, j)]; }
    const cplx& mu_at(std::size_t p, std::size_t j) const { return mu[index(p, j)]; }
};

struct TrafficCounter {
    std::size_t panel_reads = 0;
    std::size_t panel_writes = 0;
    std::size_t matrix_sweeps = 0;
    double read_bytes(std::size_t n, std::size_t n_b, std::size_t nnz, std::size_t entry_bytes = 20,
                      std::size_t vec_elem_bytes = 16) const {
        return static_cast<double>(panel_reads) * n * n_b * vec_elem_bytes +
               static_cast<double>(matrix_sweeps) * nnz * entry_bytes;
    }
    double write_bytes(std::size_t n, std::size_t n_b, std::size_t vec_elem_bytes = 16) const {
        return static_cast<double>(panel_writes) * n * n_b * vec_elem_bytes;
    }
};

namespace detail {
inline void check_spmmv_shapes(const SparseMatrixCRS& H, const SubblockView& X, const SubblockView& Y) {
    if (X.width() != Y.width()) throw std::invalid_argument("spmmv: block width mismatch");
    if (Y.rows() < H.n) throw std::invalid_argument("spmmv: output rows must cover matrix rows");
    if (X.rows() < H.n) throw std::invalid_argument("spmmv: input rows must cover matrix rows");
    if (X.identity() == Y.identity()) throw std::invalid_argument("spmmv: X and Y must not alias");
}
}  // namespace detail

inline void spmmv_shifted(const SparseMatrixCRS& H, ShiftScale s, const SubblockView& X, SubblockView Y) {
    detail::check_spmmv_shapes(H, X, Y);
    cf_matrix m = H.device_handle();
    const void* x = X.device(false);
    void* y = Y.device(true);
    detail::check(cf_spmmv_shifted(m, s.alpha, s.beta, x, y, X.width(), X.width(), nullptr));
}

inline void spmmv_shifted_two_minus(const SparseMatrixCRS& H, ShiftScale s, const SubblockView& X, SubblockView Y,
                                    const SubblockView& Z) {
    detail::check_spmmv_shapes(H, X, Y);
    if (Z.width() != Y.width() || Z.rows() < H.n) throw std::invalid_argument("spmmv: Z shape mismatch");
    if (X.identity() == Z.identity()) throw std::invalid_argument("spmmv: X and Z must not alias");
    cf_matrix m = H.device_handle();
    const void* x = X.device(false);
    const void* z = Z.device(false);
    void* y = Y.device(true);
    detail::check(cf_spmmv_shifted_two_minus(m, s.alpha, s.beta, x, y, z, X.width(), X.width(), nullptr));
}

inline void cheb_init(const SparseMatrixCRS& H, ShiftScale s, SubblockView X, SubblockView U, SubblockView W,
                      double g0c0, double g1c1, double g2c2, TrafficCounter* tc = nullptr) {
    detail::check_spmmv_shapes(H, X, U);
    detail::check_spmmv_shapes(H, U, W);
    cf_matrix m = H.device_handle();
    void* x = X.device(true);
    void* u = U.device(true);
    void* w = W.device(true);
    detail::check(cf_cheb_init(m, s.alpha, s.beta, x, u, w, X.width(), X.width(), g0c0, g1c1, g2c2, nullptr));
    if (tc) {
        tc->matrix_sweeps += 2;
        tc->panel_reads += 2 + 2 + 3;
        tc->panel_writes += 1 + 1 + 1;
    }
}

inline void chebfd_op(const SparseMatrixCRS& H, ShiftScale s, const SubblockView& U, SubblockView W, SubblockView X,
                      std::size_t p, double gc, MomentSeries& out, std::size_t moment_col_offset = 0,
                      TrafficCounter* tc = nullptr) {
    detail::check_spmmv_shapes(H, U, W);
    if (X.width() != U.width() || X.rows() < H.n) throw std::invalid_argument("chebfd_op: X shape mismatch");
    if (p < 3 || p > out.degree_max) throw std::invalid_argument("chebfd_op: degree out of range");
    const std::size_t nb = U.width();
    if (moment_col_offset + nb > out.columns) throw std::invalid_argument("chebfd_op: moment column range out of range");
    cf_matrix m = H.device_handle();
    // the step's moments are reduced on the device into the matrix's cached slots
    // and added to the caller's MomentSeries row (kernels.hpp:199-202): no
    // allocation per call, one stream synchronisation
    const std::size_t k = out.index(p, moment_col_offset);
    const void* u = U.device(false);
    void* w = W.device(true);
    void* x = X.device(true);
    detail::check(cf_chebfd_op_host_moments(m, s.alpha, s.beta, u, w, x, nb, nb, gc,
                                            reinterpret_cast<double*>(&out.eta[k]),
                                            reinterpret_cast<double*>(&out.mu[k]), nullptr));
    if (tc) {
        tc->matrix_sweeps += 1;
        tc->panel_reads += 3;
        tc->panel_writes += 2;
    }
}

// ------------------------------------------------------------- filter.hpp ---
enum class Damping { jackson, none };

struct FilterCoefficients {
    std::size_t np = 0;
    std::vector<double> c;
    std::vector<double> g;
    double window_lo = 0.0, window_hi = 0.0;
    ShiftScale map;
};

inline ShiftScale spectral_map(double lambda_min, double lambda_max, double margin = 0.0) {
    ShiftScale s;
    detail::check(cf_spectral_map(lambda_min, lambda_max, margin, &s.alpha, &s.beta));
    return s;
}

inline FilterCoefficients filter_coefficients(double window_lo, double window_hi, ShiftScale map, std::size_t np,
                                              Damping damping = Damping::jackson) {
    if (np < 2) throw std::invalid_argument("polynomial degree must be >= 2");
    FilterCoefficients fc;
    fc.np = np;
    fc.window_lo = window_lo;
    fc.window_hi = window_hi;
    fc.map = map;
    fc.c.resize(np + 1);
    fc.g.resize(np + 1);
    detail::check(cf_filter_coefficients(window_lo, window_hi, map.alpha, map.beta, np,
                                         damping == Damping::jackson ? 0 : 1, fc.c.data(), fc.g.data()));
    return fc;
}

// Alg. 2 on the device: every panel's cheb_init and (np-2) fused steps run in
// libchebfd_b200 without host round trips; moments are downloaded once.
inline MomentSeries apply_filter(const SparseMatrixCRS& H, BlockVector& X, const FilterCoefficients& fc,
                                 TrafficCounter* tc = nullptr) {
    if (X.rows() != H.n) throw std::invalid_argument("apply_filter: row count mismatch");
    if (fc.np < 2) throw std::invalid_argument("apply_filter: coefficients cover degrees < 2");
    MomentSeries mom(fc.np, X.cols());
    cf_matrix m = H.device_handle();
    std::vector<void*> panels(X.panel_count());
    for (std::size_t b = 0; b < panels.size(); ++b) panels[b] = X.device_panel(b, true);
    const std::size_t bytes = mom.eta.size() * 16;
    detail::DevBuf dm(2 * std::max<std::size_t>(bytes, 16));
    detail::check(cf_apply_filter(m, panels.data(), panels.size(), X.block_width(), fc.np, fc.c.data(), fc.g.data(),
                                  fc.map.alpha, fc.map.beta, dm.p, static_cast<char*>(dm.p) + bytes, nullptr));
    if (bytes) {
        detail::check(cf_memcpy(mom.eta.data(), dm.p, bytes, 1));
        detail::check(cf_memcpy(mom.mu.data(), static_cast<char*>(dm.p) + bytes, bytes, 1));
    }
    if (tc) {
        const std::size_t np = X.panel_count();
        tc->matrix_sweeps += np * fc.np;
        tc->panel_reads += np * (7 + 3 * (fc.np - 2));
        tc->panel_writes += np * (3 + 2 * (fc.np - 2));
    }
    return mom;
}

// ---------------------------------------------------- partition.hpp / dist.hpp ---
// Row-block partition (partition.hpp:28-60) and the single-process distributed
// filter (dist.hpp:39-98, 227-359).  Shards share this process's device; the halo
// rows travel inside cf_filter_distributed (stores into the neighbours' halo
// slots), so the transport argument only keeps the reference's signature.
struct PartitionPlan {
    std::size_t worker_count = 1;
    std::vector<std::pair<std::size_t, std::size_t>> row_ranges;  // [start, end)
    std::vector<std::map<std::size_t, std::vector<std::size_t>>> halo_in;
    std::vector<std::map<std::size_t, std::vector<std::size_t>>> halo_out;
    std::size_t owner_of(std::size_t row) const {
        for (std::size_t w = 0; w < worker_count; ++w)
            if (row >= row_ranges[w].first && row < row_ranges[w].second) return w;
        throw std::out_of_range("row not covered by partition");
    }
};

inline PartitionPlan partition_rows(const SparseMatrixCRS& H, std::size_t workers) {
    std::vector<uint64_t> rp(H.row_ptr.begin(), H.row_ptr.end());
    std::vector<uint64_t> ranges(2 * std::max<std::size_t>(workers, 1));
    std::size_t len = 0;
    detail::check(cf_partition_rows(H.n, rp.data(), H.col_idx.data(), workers, ranges.data(), nullptr, &len));
    std::vector<uint64_t> flat(len);
    detail::check(cf_partition_rows(H.n, rp.data(), H.col_idx.data(), workers, ranges.data(), flat.data(), &len));
    PartitionPlan P;
    P.worker_count = workers;
    P.halo_in.resize(workers);
    P.halo_out.resize(workers);
    for (std::size_t w = 0; w < workers; ++w) P.row_ranges.emplace_back(ranges[2 * w], ranges[2 * w + 1]);
    for (std::size_t q = 0; q + 3 <= len;) {  // records (w, v, count, rows...)
        const std::size_t w = flat[q], v = flat[q + 1], cnt = flat[q + 2];
        std::vector<std::size_t> rows(flat.begin() + q + 3, flat.begin() + q + 3 + cnt);
        P.halo_out[v][w] = rows;  // mirrored (partition.hpp:57-58)
        P.halo_in[w][v] = std::move(rows);
        q += 3 + cnt;
    }
    return P;
}

enum class CommMode { vector, pipelined };

struct WorkerShard {
    struct NeighborRows {
        std::size_t neighbor;
        std::vector<std::size_t> rows;
    };
    std::size_t id = 0, row_begin = 0, row_end = 0, local_n = 0, halo_n = 0;
    SparseMatrixCRS local;
    std::vector<std::size_t> halo_global;
    std::vector<NeighborRows> send_plan;  // owned rows (local offsets) per neighbour
    std::vector<NeighborRows> recv_plan;  // halo slots (local_n + slot) per neighbour
    BlockVector X, U, W;
    std::vector<std::uint8_t> exchange_pending;
};

namespace detail {
// Shard w of shard_and_distribute (dist.hpp:39-98): local CRS with remapped
// columns, halo lists and the owned rows of X.  Its panels are allocated on the
// calling thread's device (set_device).
inline WorkerShard make_shard(const SparseMatrixCRS& H, const BlockVector& X, const PartitionPlan& plan,
                              std::size_t w) {
    std::vector<uint64_t> rp(H.row_ptr.begin(), H.row_ptr.end());
    const double* vals = reinterpret_cast<const double*>(H.values.data());
    const std::size_t ns = X.cols(), nb = X.block_width();
    auto unflatten = [](const std::vector<uint64_t>& f) {
        std::vector<WorkerShard::NeighborRows> out;
        for (std::size_t q = 0; q + 2 <= f.size();) {
            WorkerShard::NeighborRows nr{f[q], std::vector<std::size_t>(f.begin() + q + 2, f.begin() + q + 2 + f[q + 1])};
            q += 2 + f[q + 1];
            out.push_back(std::move(nr));
        }
        return out;
    };
    std::size_t rb = 0, ln = 0, hn = 0, nnz = 0, sl = 0, rl = 0;
    check(cf_shard(H.n, rp.data(), H.col_idx.data(), vals, plan.worker_count, w, &rb, &ln, &hn, &nnz, nullptr,
                   nullptr, nullptr, nullptr, nullptr, &sl, nullptr, &rl));
    WorkerShard sh;
    sh.id = w;
    sh.row_begin = rb;
    sh.row_end = rb + ln;
    sh.local_n = ln;
    sh.halo_n = hn;
    std::vector<uint64_t> lrp(ln + 1), hg(hn), sf(sl), rf(rl);
    sh.local.n = ln;
    sh.local.ncols_ = ln + hn;
    sh.local.col_idx.resize(nnz);
    sh.local.values.resize(nnz);
    check(cf_shard(H.n, rp.data(), H.col_idx.data(), vals, plan.worker_count, w, &rb, &ln, &hn, &nnz, lrp.data(),
                   sh.local.col_idx.data(), reinterpret_cast<double*>(sh.local.values.data()), hg.data(), sf.data(),
                   &sl, rf.data(), &rl));
    sh.local.row_ptr.assign(lrp.begin(), lrp.end());
    sh.halo_global.assign(hg.begin(), hg.end());
    sh.send_plan = unflatten(sf);
    sh.recv_plan = unflatten(rf);
    sh.X = BlockVector(ln + hn, ns, nb);
    sh.U = BlockVector(ln + hn, ns, nb);
    sh.W = BlockVector(ln + hn, ns, nb);
    for (std::size_t b = 0; b < X.panel_count(); ++b) {
        const auto& src = X.panel(b);
        std::copy(src.begin() + rb * nb, src.begin() + (rb + ln) * nb, sh.X.panel(b).begin());
    }
    sh.exchange_pending.assign(X.panel_count(), 0);
    return sh;
}
inline void check_shard_inputs(const SparseMatrixCRS& H, const BlockVector& X, const PartitionPlan& plan) {
    if (plan.row_ranges.empty() || plan.row_ranges.back().second != H.n)
        throw std::invalid_argument("partition plan does not match matrix");
    if (X.rows() != H.n) throw std::invalid_argument("block vector does not match matrix");
}
}  // namespace detail

inline std::vector<WorkerShard> shard_and_distribute(const SparseMatrixCRS& H, const BlockVector& X,
                                                     const PartitionPlan& plan) {
    detail::check_shard_inputs(H, X, plan);
    std::vector<WorkerShard> shards;
    for (std::size_t w = 0; w < plan.worker_count; ++w) shards.push_back(detail::make_shard(H, X, plan, w));
    return shards;
}

// Shards spread over several GPUs: shard w's matrix and panels are placed on
// devices[w % devices.size()] (a B200-side overload; the reference runs every
// worker as a thread of one CPU process).  cf_filter_distributed then moves the
// halo rows between them over peer memory (NVLink).
inline std::vector<WorkerShard> shard_and_distribute(const SparseMatrixCRS& H, const BlockVector& X,
                                                     const PartitionPlan& plan, const std::vector<int>& devices) {
    if (devices.empty()) return shard_and_distribute(H, X, plan);
    detail::check_shard_inputs(H, X, plan);
    const int saved = detail::device_override();
    std::vector<WorkerShard> out;
    try {
        for (std::size_t w = 0; w < plan.worker_count; ++w) {
            // built with its own device selected: the shard's panels (DevBufs) and
            // its matrix image land on that GPU
            set_device(devices[w % devices.size()]);
            out.push_back(detail::make_shard(H, X, plan, w));
            out.back().local.device_handle();
        }
    } catch (...) {
        set_device(saved);
        throw;
    }
    set_device(saved);
    return out;
}

// ------------------------------------------------ halo_exchange (dist.hpp:100-144) ---
// Frames carry device memory: init gathers the owned send rows of panel b into
// a device frame per neighbour (one device copy per run of consecutive rows,
// D2D or peer over NVLink), finalize checks tag and size and scatters the
// frame into the halo slots.  Same protocol errors as the reference
// (dist.hpp:115-116, 128-129, 135-138).
enum class ExchangePhase { init, finalize };

struct FrameTag {  // wire.hpp:21-35 (degree, block, neighbour)
    std::uint16_t degree = 0;
    std::uint8_t block = 0;
    std::uint8_t neighbor = 0;
    bool operator==(const FrameTag& o) const {
        return degree == o.degree && block == o.block && neighbor == o.neighbor;
    }
};

struct DeviceFrame {
    FrameTag tag;
    std::size_t elems = 0;  // complex values in the payload
    std::shared_ptr<detail::DevBuf> payload;
};

struct QueueTransport {  // in-process mailboxes (wire.hpp:101-134), device payloads
    explicit QueueTransport(std::size_t workers = 0) : workers(workers) {}
    void send(std::size_t from, std::size_t to, DeviceFrame f) {
        if (from >= workers || to >= workers) throw std::out_of_range("transport endpoint out of range");
        q_[{from, to}].push_back(std::move(f));
    }
    DeviceFrame recv(std::size_t to, std::size_t from) {
        auto it = q_.find({from, to});
        if (it == q_.end() || it->second.empty()) throw std::runtime_error("transport: no frame pending");
        DeviceFrame f = std::move(it->second.front());
        it->second.erase(it->second.begin());
        return f;
    }
    std::size_t workers;

  private:
    std::map<std::pair<std::size_t, std::size_t>, std::vector<DeviceFrame>> q_;
};

namespace detail {
// rows (sorted, distinct) -> runs of consecutive rows: (first row, count, offset in the list)
inline std::vector<std::array<std::size_t, 3>> row_runs(const std::vector<std::size_t>& rows) {
    std::vector<std::array<std::size_t, 3>> runs;
    for (std::size_t i = 0; i < rows.size(); ++i) {
        if (!runs.empty() && rows[i] == runs.back()[0] + runs.back()[1]) {
            ++runs.back()[1];
        } else {
            runs.push_back({rows[i], 1, i});
        }
    }
    return runs;
}
}  // namespace detail

template <class Transport>
inline void halo_exchange(WorkerShard& shard, BlockVector& vec, std::size_t b, ExchangePhase phase,
                          Transport& transport, std::uint16_t degree_tag) {
    if (b >= shard.exchange_pending.size()) throw std::invalid_argument("panel index out of range");
    const std::size_t nb = vec.block_width(), row_bytes = nb * 16;
    if (phase == ExchangePhase::init) {
        if (shard.exchange_pending[b]) throw ProtocolError("halo_exchange: exchange already outstanding on panel");
        shard.exchange_pending[b] = 1;
        char* panel = static_cast<char*>(vec.device_panel(b, false));
        for (const auto& sp : shard.send_plan) {
            DeviceFrame f;
            f.tag = {degree_tag, static_cast<std::uint8_t>(b), static_cast<std::uint8_t>(shard.id)};
            f.elems = sp.rows.size() * nb;
            f.payload = std::make_shared<detail::DevBuf>(std::max<std::size_t>(f.elems * 16, 16));
            for (const auto& r : detail::row_runs(sp.rows))
                detail::check(cf_memcpy(static_cast<char*>(f.payload->p) + r[2] * row_bytes, panel + r[0] * row_bytes,
                                        r[1] * row_bytes, 2));
            transport.send(shard.id, sp.neighbor, std::move(f));
        }
    } else {
        if (!shard.exchange_pending[b]) throw ProtocolError("halo_exchange: finalize without init");
        char* panel = static_cast<char*>(vec.device_panel(b, true));
        for (const auto& rp : shard.recv_plan) {
            DeviceFrame f = transport.recv(shard.id, rp.neighbor);
            const FrameTag expect{degree_tag, static_cast<std::uint8_t>(b), static_cast<std::uint8_t>(rp.neighbor)};
            if (!(f.tag == expect)) throw ProtocolError("halo_exchange: frame tag mismatch");
            if (f.elems != rp.rows.size() * nb) throw ProtocolError("halo_exchange: frame size mismatch");
            for (const auto& r : detail::row_runs(rp.rows))
                detail::check(cf_memcpy(panel + r[0] * row_bytes, static_cast<char*>(f.payload->p) + r[2] * row_bytes,
                                        r[1] * row_bytes, 2));
        }
        shard.exchange_pending[b] = 0;
    }
}

// dist.hpp:146-170.  The reference fills the timelines from a unit-cost model
// (comm_cost, compute_cost); here they are measured with CUDA events per shard and
// (panel, degree) step, in milliseconds from the shard's first event, so the cost
// model is accepted for the signature only.
struct TimelineEvent {
    enum class Kind { compute, comm };
    Kind kind;
    std::size_t block = 0;
    std::size_t degree = 0;
    double start = 0.0;
    double end = 0.0;
};

struct Timeline {
    std::vector<TimelineEvent> events;
    double makespan() const {
        double m = 0.0;
        for (const auto& e : events) m = std::max(m, e.end);
        return m;
    }
};

struct CostModel {
    double comm_cost = 1.0;
    double compute_cost = 2.0;
};

struct DistributedResult {
    BlockVector X;
    MomentSeries moments;
    std::vector<Timeline> timelines;  // per worker, degree loop only (measured)
    TrafficCounter traffic;
};

// filter_distributed (dist.hpp:227-359) through cf_filter_distributed: owned rows of
// every shard's X are filtered in place; the result holds the assembled X, the
// moments summed in the rank-ordered tree and the reference's traffic counts.
template <class Transport>
DistributedResult filter_distributed(std::vector<WorkerShard>& shards, const FilterCoefficients& fc, CommMode mode,
                                     Transport&, CostModel = {}) {
    if (shards.empty()) throw std::invalid_argument("no shards");
    const std::size_t ns = shards[0].X.cols(), nb = shards[0].X.block_width(), npan = ns / nb;
    std::vector<std::vector<void*>> panels(shards.size());
    std::vector<std::vector<uint64_t>> sf(shards.size()), rf(shards.size());
    std::vector<cf_dist_worker> wk(shards.size());
    auto flatten = [](const std::vector<WorkerShard::NeighborRows>& v) {
        std::vector<uint64_t> f;
        for (const auto& nr : v) {
            f.push_back(nr.neighbor);
            f.push_back(nr.rows.size());
            f.insert(f.end(), nr.rows.begin(), nr.rows.end());
        }
        return f;
    };
    std::size_t n = 0;
    for (std::size_t w = 0; w < shards.size(); ++w) {
        WorkerShard& sh = shards[w];
        for (std::size_t b = 0; b < npan; ++b) panels[w].push_back(sh.X.device_panel(b, true));
        sf[w] = flatten(sh.send_plan);
        rf[w] = flatten(sh.recv_plan);
        wk[w] = cf_dist_worker{sh.local.device_handle(), sh.local_n, sh.halo_n, panels[w].data(),
                               sf[w].data(), sf[w].size(), rf[w].data(), rf[w].size()};
        n += sh.local_n;
    }
    DistributedResult res{BlockVector(n, ns, nb), MomentSeries(fc.np, ns), {}, TrafficCounter{}};
    const std::size_t cap = shards.size() * 2 * npan * (fc.np >= 2 ? fc.np - 2 : 0);
    std::vector<double> tl(6 * std::max<std::size_t>(cap, 1));
    std::size_t count = 0;
    detail::check(cf_filter_distributed_timeline(wk.data(), wk.size(), ns, nb, fc.np, fc.c.data(), fc.g.data(),
                                                 fc.map.alpha, fc.map.beta, mode == CommMode::vector ? 0 : 1, 0,
                                                 reinterpret_cast<double*>(res.moments.eta.data()),
                                                 reinterpret_cast<double*>(res.moments.mu.data()), tl.data(), cap,
                                                 &count));
    res.timelines.assign(shards.size(), Timeline{});
    for (std::size_t k = 0; k < std::min(count, cap); ++k) {
        const double* r = tl.data() + 6 * k;
        res.timelines[static_cast<std::size_t>(r[0])].events.push_back(
            {r[1] == 0.0 ? TimelineEvent::Kind::compute : TimelineEvent::Kind::comm, static_cast<std::size_t>(r[2]),
             static_cast<std::size_t>(r[3]), r[4], r[5]});
    }
    for (const WorkerShard& sh : shards)
        for (std::size_t b = 0; b < npan; ++b) {
            const auto& src = sh.X.panel(b);
            std::copy(src.begin(), src.begin() + sh.local_n * nb, res.X.panel(b).begin() + sh.row_begin * nb);
        }
    const std::size_t ops = shards.size() * npan * (fc.np >= 2 ? fc.np - 2 : 0);  // dist.hpp:352-356
    res.traffic.panel_reads = 3 * ops;
    res.traffic.panel_writes = 2 * ops;
    res.traffic.matrix_sweeps = ops;
    return res;
}


// ----------------------------------------------------------- jacobi_eig.hpp ---
struct HermitianDense {
    std::size_t k = 0;
    std::vector<cplx> a;  // k*k row-major
    HermitianDense() = default;
    explicit HermitianDense(std::size_t dim) : k(dim), a(dim * dim, cplx(0.0)) {}
    cplx& at(std::size_t i, std::size_t j) { return a[i * k + j]; }
    const cplx& at(std::size_t i, std::size_t j) const { return a[i * k + j]; }
};

struct EigenDecomposition {
    std::vector<double> values;  // ascending
    std::vector<cplx> vectors;   // k*k row-major, column j is eigenvector j
};

inline EigenDecomposition jacobi_hermitian_eig(HermitianDense A, double tol = 1e-12, std::size_t max_sweeps = 64) {
    EigenDecomposition e;
    e.values.resize(A.k);
    e.vectors.resize(A.k * A.k);
    detail::check(cf_jacobi_hermitian_eig(A.k, reinterpret_cast<const double*>(A.a.data()), tol, max_sweeps,
                                          e.values.data(), reinterpret_cast<double*>(e.vectors.data())));
    return e;
}

// -------------------------------------------------- filter.hpp (eigensolver) ---
namespace detail {
inline std::vector<void*> device_panels(BlockVector& X, bool will_write) {
    std::vector<void*> p(X.panel_count());
    for (std::size_t b = 0; b < p.size(); ++b) p[b] = X.device_panel(b, will_write);
    return p;
}
}  // namespace detail

// filter.hpp:139-150: SVQB on the device; Q = BlockVector(n, rank, rank).
inline std::pair<BlockVector, std::size_t> orthogonalize_svqb(const BlockVector& X, double drop_tol = 1e-12) {
    BlockVector& Xm = const_cast<BlockVector&>(X);
    auto panels = detail::device_panels(Xm, false);
    detail::DevBuf q(X.rows() * X.cols() * 16);
    std::size_t rank = 0;
    detail::check(cf_orthogonalize_svqb(X.rows(), panels.data(), panels.size(), X.block_width(), drop_tol, q.p, &rank,
                                        nullptr));
    BlockVector Q(X.rows(), rank, rank);
    Q.load_device_panel(0, q.p);
    return {std::move(Q), rank};
}

struct RayleighRitzResult {
    std::vector<double> theta;      // ascending
    BlockVector basis;              // rotated basis Y = Q V, one panel
    std::vector<double> residuals;  // ||H y_j - theta_j y_j|| / ||y_j||
};

// filter.hpp:170-211
inline RayleighRitzResult rayleigh_ritz(const SparseMatrixCRS& H, const BlockVector& Q) {
    if (Q.rows() != H.n) throw std::invalid_argument("rayleigh_ritz: row count mismatch");
    const std::size_t k = Q.cols();
    if (Q.block_width() != k) throw std::invalid_argument("rayleigh_ritz: expects a single panel");
    RayleighRitzResult rr;
    rr.theta.resize(k);
    rr.residuals.resize(k);
    rr.basis = BlockVector(H.n, k, k);
    void* y = rr.basis.device_panel(0, true);
    const void* q = const_cast<BlockVector&>(Q).device_panel(0, false);
    detail::check(cf_rayleigh_ritz(H.device_handle(), q, k, rr.theta.data(), y, rr.residuals.data(), nullptr));
    return rr;
}

struct RitzPair {
    double value = 0.0;
    double residual = 0.0;
    bool inside_window = false;
    bool converged = false;
};

struct SolveResult {
    std::vector<double> eigenvalues;    // converged, in-window, ascending
    std::vector<double> residuals;      // matching eigenvalues
    BlockVector eigenvectors;           // matching columns (empty if none)
    std::vector<RitzPair> all_pairs;    // last Rayleigh-Ritz extraction
    std::vector<MomentSeries> moments;  // one series per restart
    std::size_t iterations = 0;
    bool converged = false;
};

struct SolveOptions {
    std::size_t n_s = 32;
    std::size_t n_b = 8;
    std::size_t n_p = 500;
    std::size_t max_restarts = 20;
    double res_tol = 1e-9;
    double margin = 0.01;
    std::uint64_t seed = 42;
    Damping damping = Damping::jackson;
    std::optional<std::pair<double, double>> spectral_bounds;  // default: Gershgorin
    double drop_tol = 1e-12;
};

// filter.hpp:247-320: the restart loop runs in libchebfd_b200 (cf_chebfd_solve).
inline SolveResult chebfd_solve(const SparseMatrixCRS& H, double window_lo, double window_hi,
                                const SolveOptions& opt = {}) {
    cf_solve_options o{opt.n_s, opt.n_b, opt.n_p, opt.max_restarts, opt.res_tol, opt.margin, opt.seed,
                       opt.damping == Damping::jackson ? 0 : 1, opt.spectral_bounds ? 1 : 0,
                       opt.spectral_bounds ? opt.spectral_bounds->first : 0.0,
                       opt.spectral_bounds ? opt.spectral_bounds->second : 0.0, opt.drop_tol};
    const std::size_t ns = opt.n_s, rows = opt.n_p >= 3 ? opt.n_p - 2 : 0;
    std::vector<double> ev(ns), er(ns), pv(ns), pr(ns);
    std::vector<int> pf(ns);
    std::vector<cplx> eta(std::max<std::size_t>(opt.max_restarts, 1) * rows * ns), mu(eta.size());
    detail::DevBuf vec(std::max<std::size_t>(H.n * ns * 16, 16));
    cf_solve_result r{0, 0, 0, 0, ev.data(), er.data(), pv.data(), pr.data(), pf.data(), vec.p,
                      reinterpret_cast<double*>(eta.data()), reinterpret_cast<double*>(mu.data())};
    detail::check(cf_chebfd_solve(H.device_handle(), window_lo, window_hi, &o, &r, nullptr));
    SolveResult out;
    out.iterations = r.iterations;
    out.converged = r.converged != 0;
    out.eigenvalues.assign(ev.begin(), ev.begin() + r.n_eig);
    out.residuals.assign(er.begin(), er.begin() + r.n_eig);
    for (std::size_t i = 0; i < r.n_pairs; ++i)
        out.all_pairs.push_back({pv[i], pr[i], (pf[i] & 1) != 0, (pf[i] & 2) != 0});
    if (out.converged && r.n_eig > 0) {
        out.eigenvectors = BlockVector(H.n, r.n_eig, r.n_eig);
        out.eigenvectors.load_device_panel(0, vec.p);
    }
    for (std::size_t it = 0; it < out.iterations; ++it) {
        MomentSeries m(opt.n_p, ns);
        std::copy(eta.begin() + it * rows * ns, eta.begin() + (it + 1) * rows * ns, m.eta.begin());
        std::copy(mu.begin() + it * rows * ns, mu.begin() + (it + 1) * rows * ns, m.mu.begin());
        out.moments.push_back(std::move(m));
    }
    return out;
}

// ------------------------------------------------------ matrix_market.hpp ---
struct MatrixMarketError : std::runtime_error {
    MatrixMarketError(const std::string& msg, std::size_t line) : std::runtime_error(msg), line_number(line) {}
    std::size_t line_number;
};

inline SparseMatrixCRS matrix_market_read(const std::string& path) {
    std::size_t n = 0, nnz = 0;
    int sym = 0;
    int st = cf_matrix_market_read(path.c_str(), &n, &nnz, &sym, nullptr, nullptr, nullptr);
    if (st != CF_OK && cf_matrix_market_error_line() != 0)
        throw MatrixMarketError(cf_last_error(), cf_matrix_market_error_line());
    detail::check(st);
    SparseMatrixCRS H;
    H.n = n;
    H.symmetry = sym == 0 ? Symmetry::hermitian : Symmetry::general;
    std::vector<uint64_t> rp(n + 1);
    H.col_idx.resize(nnz);
    H.values.resize(nnz);
    detail::check(cf_matrix_market_read(path.c_str(), &n, &nnz, &sym, rp.data(), H.col_idx.data(),
                                        reinterpret_cast<double*>(H.values.data())));
    H.row_ptr.assign(rp.begin(), rp.end());
    return H;
}

inline void matrix_market_write(const std::string& path, const SparseMatrixCRS& H) {
    std::vector<uint64_t> rp(H.row_ptr.begin(), H.row_ptr.end());
    detail::check(cf_matrix_market_write(path.c_str(), H.n, rp.data(), H.col_idx.data(),
                                         reinterpret_cast<const double*>(H.values.data()),
                                         H.symmetry == Symmetry::hermitian ? 0 : 1));
}

// ------------------------------------------------- block_vector.hpp (CFDB) ---
inline void block_vector_write(const std::string& path, const BlockVector& X) {
    std::vector<cplx> all;
    all.reserve(X.rows() * X.cols());
    for (std::size_t b = 0; b < X.panel_count(); ++b) all.insert(all.end(), X.panel(b).begin(), X.panel(b).end());
    detail::check(cf_blockvec_write(path.c_str(), X.rows(), X.cols(), X.block_width(),
                                    reinterpret_cast<const double*>(all.data())));
}

inline BlockVector block_vector_read(const std::string& path) {
    std::size_t n = 0, ns = 0, nb = 0;
    detail::check(cf_blockvec_read(path.c_str(), &n, &ns, &nb, nullptr));
    std::vector<cplx> all(n * ns);
    detail::check(cf_blockvec_read(path.c_str(), &n, &ns, &nb, reinterpret_cast<double*>(all.data())));
    BlockVector X(n, ns, nb);
    for (std::size_t b = 0; b < X.panel_count(); ++b)
        std::copy(all.begin() + b * n * nb, all.begin() + (b + 1) * n * nb, X.panel(b).begin());
    return X;
}

}  // namespace chebfilter
