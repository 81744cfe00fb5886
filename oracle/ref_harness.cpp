// ref_harness.cpp -- extern "C" shim over the UNMODIFIED reference headers
// (/root/reference/proj/include/chebfilter/*.hpp, included, never copied).
// TEST INFRASTRUCTURE ONLY: built into oracle/_ref/libchebref.so by
// oracle/Makefile (target `ref`), used by tests/ to pin the C restatement
// (chebfd_oracle.c) and to make golden fixtures, and by bench.py's
// `--impl reference` / cpu_baseline legs to time the reference CPU path.
// Complex arrays are interleaved (re, im) doubles; panels use the reference
// layout (block_vector.hpp:49-52).  Every entry returns 0 on success, 1 on
// std::invalid_argument / out_of_range, 2 on any other exception.
#include <cstring>
#include <exception>
#include <stdexcept>
#include <string>

#include "chebfilter/dist.hpp"
#include "chebfilter/filter.hpp"
#include "chebfilter/matrix_market.hpp"
#include "chebfilter/perf_model.hpp"
#include "support/dense_eig.hpp"

using namespace chebfilter;

namespace {
thread_local std::string g_err;

template <class F>
int guard(F&& f) {
    try {
        f();
        return 0;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return 1;
    } catch (const std::out_of_range& e) {
        g_err = e.what();
        return 1;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 2;
    }
}

SparseMatrixCRS from_arrays(size_t n, const uint64_t* rp, const int32_t* ci, const double* v) {
    SparseMatrixCRS H;
    H.n = n;
    H.row_ptr.assign(rp, rp + n + 1);
    size_t nnz = rp[n];
    H.col_idx.assign(ci, ci + nnz);
    H.values.resize(nnz);
    std::memcpy(H.values.data(), v, nnz * sizeof(cplx));
    return H;
}

void load_panel(BlockVector& B, size_t b, const double* src) {
    std::memcpy(B.panel(b).data(), src, B.panel(b).size() * sizeof(cplx));
}
void store_panel(const BlockVector& B, size_t b, double* dst) {
    std::memcpy(dst, B.panel(b).data(), B.panel(b).size() * sizeof(cplx));
}
void load_all(BlockVector& B, const double* src) {
    size_t per = B.rows() * B.block_width() * 2;
    for (size_t b = 0; b < B.panel_count(); ++b) load_panel(B, b, src + b * per);
}
void store_all(const BlockVector& B, double* dst) {
    size_t per = B.rows() * B.block_width() * 2;
    for (size_t b = 0; b < B.panel_count(); ++b) store_panel(B, b, dst + b * per);
}
FilterCoefficients make_fc(size_t np, const double* c, const double* g, double alpha, double beta) {
    FilterCoefficients fc;
    fc.np = np;
    fc.c.assign(c, c + np + 1);
    fc.g.assign(g, g + np + 1);
    fc.map = ShiftScale{alpha, beta};
    return fc;
}
}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// ---- matrices (opaque SparseMatrixCRS*) ----
void* ref_topi(size_t nx, size_t ny, size_t nz, double mass, double hop, int open) {
    SparseMatrixCRS* out = nullptr;
    if (guard([&] {
            LatticeSpec s;
            s.nx = nx; s.ny = ny; s.nz = nz; s.mass = mass; s.hop = hop;
            s.boundary = open ? Boundary::open : Boundary::periodic;
            out = new SparseMatrixCRS(topi_generate(s));
        }))
        return nullptr;
    return out;
}
void* ref_crs_from_arrays(size_t n, const uint64_t* rp, const int32_t* ci, const double* v) {
    return new SparseMatrixCRS(from_arrays(n, rp, ci, v));
}
void* ref_random_hermitian(size_t n, uint64_t seed, double scale) {
    auto a = testsupport::random_hermitian(n, seed);
    for (auto& z : a) z *= scale;
    return new SparseMatrixCRS(testsupport::to_sparse(a, n));
}
void ref_crs_info(void* h, size_t* n, size_t* nnz) {
    auto* H = static_cast<SparseMatrixCRS*>(h);
    *n = H->n;
    *nnz = H->nnz();
}
void ref_crs_copy(void* h, uint64_t* rp, int32_t* ci, double* v) {
    auto* H = static_cast<SparseMatrixCRS*>(h);
    for (size_t i = 0; i <= H->n; ++i) rp[i] = H->row_ptr[i];
    std::memcpy(ci, H->col_idx.data(), H->nnz() * 4);
    std::memcpy(v, H->values.data(), H->nnz() * 16);
}
void ref_crs_free(void* h) { delete static_cast<SparseMatrixCRS*>(h); }
int ref_gershgorin(void* h, double* lo, double* hi) {
    return guard([&] {
        auto b = gershgorin_bounds(*static_cast<SparseMatrixCRS*>(h));
        *lo = b.first;
        *hi = b.second;
    });
}
int ref_dense_eigenvalues(void* h, double* out) {
    return guard([&] {
        auto e = testsupport::dense_eigenvalues(*static_cast<SparseMatrixCRS*>(h));
        std::memcpy(out, e.data(), e.size() * 8);
    });
}

// ---- file formats (matrix_market.hpp, block_vector.hpp:182-229) ----
int ref_mm_write(void* h, const char* path) {
    return guard([&] { matrix_market_write(path, *static_cast<SparseMatrixCRS*>(h)); });
}
// returns a matrix handle or nullptr; *line = MatrixMarketError::line_number (0 otherwise)
void* ref_mm_read(const char* path, size_t* line, int* symmetry) {
    *line = 0;
    try {
        auto* m = new SparseMatrixCRS(matrix_market_read(path));
        *symmetry = m->symmetry == Symmetry::hermitian ? 0 : 1;
        return m;
    } catch (const MatrixMarketError& e) {
        *line = e.line_number;
        g_err = e.what();
    } catch (const std::exception& e) {
        g_err = e.what();
    }
    return nullptr;
}
int ref_bv_write(const char* path, size_t n, size_t ns, size_t nb, uint64_t seed) {
    return guard([&] { block_vector_write(path, BlockVector(n, ns, nb, InitSeededRandom{seed})); });
}
int ref_bv_read(const char* path, size_t* n, size_t* ns, size_t* nb, double* out) {
    return guard([&] {
        BlockVector X = block_vector_read(path);
        *n = X.rows();
        *ns = X.cols();
        *nb = X.block_width();
        if (!out) return;
        for (size_t b = 0; b < X.panel_count(); ++b)
            std::memcpy(out + 2 * b * X.rows() * X.block_width(), X.panel(b).data(), X.panel(b).size() * 16);
    });
}

// ---- coefficients / RNG ----
int ref_spectral_map(double lo, double hi, double margin, double* a, double* b) {
    return guard([&] {
        auto s = spectral_map(lo, hi, margin);
        *a = s.alpha;
        *b = s.beta;
    });
}
int ref_filter_coefficients(double wlo, double whi, double a, double b, size_t np, int damping, double* c,
                            double* g) {
    return guard([&] {
        auto fc = filter_coefficients(wlo, whi, ShiftScale{a, b}, np, damping ? Damping::none : Damping::jackson);
        std::memcpy(c, fc.c.data(), (np + 1) * 8);
        std::memcpy(g, fc.g.data(), (np + 1) * 8);
    });
}
int ref_blockvec_random(size_t n, size_t ns, size_t nb, uint64_t seed, uint64_t row_offset, double* out) {
    return guard([&] {
        BlockVector X(n, ns, nb, InitSeededRandom{seed, row_offset});
        store_all(X, out);
    });
}

// ---- kernels on single panels (rows x nb) ----
int ref_spmmv_shifted(void* h, double a, double b, size_t rows, size_t nb, const double* X, double* Y) {
    return guard([&] {
        BlockVector Xv(rows, nb, nb), Yv(rows, nb, nb);
        load_panel(Xv, 0, X);
        spmmv_shifted(*static_cast<SparseMatrixCRS*>(h), {a, b}, SubblockView(Xv, 0), SubblockView(Yv, 0));
        store_panel(Yv, 0, Y);
    });
}
int ref_spmmv_two_minus(void* h, double a, double b, size_t rows, size_t nb, const double* X, double* Y,
                        const double* Z) {
    return guard([&] {
        BlockVector Xv(rows, nb, nb), Yv(rows, nb, nb), Zv(rows, nb, nb);
        load_panel(Xv, 0, X);
        load_panel(Zv, 0, Z);
        spmmv_shifted_two_minus(*static_cast<SparseMatrixCRS*>(h), {a, b}, SubblockView(Xv, 0),
                                SubblockView(Yv, 0), SubblockView(Zv, 0));
        store_panel(Yv, 0, Y);
    });
}
int ref_cheb_init(void* h, double a, double b, size_t rows, size_t nb, double* X, double* U, double* W, double g0c0,
                  double g1c1, double g2c2) {
    return guard([&] {
        BlockVector Xv(rows, nb, nb), Uv(rows, nb, nb), Wv(rows, nb, nb);
        load_panel(Xv, 0, X);
        cheb_init(*static_cast<SparseMatrixCRS*>(h), {a, b}, SubblockView(Xv, 0), SubblockView(Uv, 0),
                  SubblockView(Wv, 0), g0c0, g1c1, g2c2);
        store_panel(Xv, 0, X);
        store_panel(Uv, 0, U);
        store_panel(Wv, 0, W);
    });
}
// One fused step: eta/mu are the nb-wide slots of row p (accumulated with +=).
int ref_chebfd_op(void* h, double a, double b, size_t rows, size_t nb, const double* U, double* W, double* X,
                  double gc, double* eta, double* mu, int unfused) {
    return guard([&] {
        BlockVector Uv(rows, nb, nb), Wv(rows, nb, nb), Xv(rows, nb, nb);
        load_panel(Uv, 0, U);
        load_panel(Wv, 0, W);
        load_panel(Xv, 0, X);
        MomentSeries m(3, nb);
        std::memcpy(m.eta.data(), eta, nb * 16);
        std::memcpy(m.mu.data(), mu, nb * 16);
        auto& H = *static_cast<SparseMatrixCRS*>(h);
        if (unfused)
            chebfd_op_reference(H, {a, b}, SubblockView(Uv, 0), SubblockView(Wv, 0), SubblockView(Xv, 0), 3, gc, m);
        else
            chebfd_op(H, {a, b}, SubblockView(Uv, 0), SubblockView(Wv, 0), SubblockView(Xv, 0), 3, gc, m);
        store_panel(Wv, 0, W);
        store_panel(Xv, 0, X);
        std::memcpy(eta, m.eta.data(), nb * 16);
        std::memcpy(mu, m.mu.data(), nb * 16);
    });
}

// ---- apply_filter (filter.hpp:76-93) on a panel-concatenated n x ns X ----
int ref_apply_filter(void* h, size_t ns, size_t nb, double* X, size_t np, const double* c, const double* g, double a,
                     double b, double* eta, double* mu) {
    return guard([&] {
        auto& H = *static_cast<SparseMatrixCRS*>(h);
        BlockVector Xv(H.n, ns, nb);
        load_all(Xv, X);
        auto m = apply_filter(H, Xv, make_fc(np, c, g, a, b));
        store_all(Xv, X);
        std::memcpy(eta, m.eta.data(), m.eta.size() * 16);
        std::memcpy(mu, m.mu.data(), m.mu.size() * 16);
    });
}

// ---- bench-kernel-style timed step helpers (state kept across calls) ----
struct StepState {
    SparseMatrixCRS* H;
    BlockVector U, W, X;
    MomentSeries m;
    ShiftScale s;
};
void* ref_step_state(void* h, size_t nb, uint64_t seed, double a, double b) {
    auto* H = static_cast<SparseMatrixCRS*>(h);
    auto* st = new StepState{H, BlockVector(H->n, nb, nb, InitSeededRandom{seed}),
                             BlockVector(H->n, nb, nb, InitSeededRandom{seed + 1}),
                             BlockVector(H->n, nb, nb, InitSeededRandom{seed + 2}), MomentSeries(3, nb), {a, b}};
    return st;
}
int ref_step_run(void* sp, double gc) {  // swap + chebfd_op, exactly filter.hpp:88-89
    return guard([&] {
        auto* st = static_cast<StepState*>(sp);
        swap_blocks(SubblockView(st->W, 0), SubblockView(st->U, 0));
        chebfd_op(*st->H, st->s, SubblockView(st->U, 0), SubblockView(st->W, 0), SubblockView(st->X, 0), 3, gc,
                  st->m);
    });
}
void ref_step_free(void* sp) { delete static_cast<StepState*>(sp); }

// ---- partition / sharding (partition.hpp:28-60, dist.hpp:39-98) ----
// Flattened halo_in records: (w, v, count, rows...) -- same format as the oracle.
int ref_partition_rows(void* h, size_t workers, uint64_t* ranges, uint64_t* halo, size_t* halo_len) {
    return guard([&] {
        auto plan = partition_rows(*static_cast<SparseMatrixCRS*>(h), workers);
        size_t len = 0;
        for (size_t w = 0; w < workers; ++w) {
            if (ranges) {
                ranges[2 * w] = plan.row_ranges[w].first;
                ranges[2 * w + 1] = plan.row_ranges[w].second;
            }
            for (auto& [v, rows] : plan.halo_in[w]) {
                if (halo) {
                    halo[len] = w;
                    halo[len + 1] = v;
                    halo[len + 2] = rows.size();
                    for (size_t k = 0; k < rows.size(); ++k) halo[len + 3 + k] = rows[k];
                }
                len += 3 + rows.size();
            }
        }
        *halo_len = len;
    });
}
// Shard w's local CRS + halo_global + plans.  Two-phase sizes query when out ptrs are null.
int ref_shard(void* h, size_t workers, size_t w, size_t* local_n, size_t* halo_n, size_t* nnz, uint64_t* rp,
              int32_t* ci, double* v, uint64_t* halo_global, uint64_t* send_flat, size_t* send_len,
              uint64_t* recv_flat, size_t* recv_len) {
    return guard([&] {
        auto& H = *static_cast<SparseMatrixCRS*>(h);
        auto plan = partition_rows(H, workers);
        BlockVector X(H.n, 1, 1);
        auto shards = shard_and_distribute(H, X, plan);
        auto& sh = shards[w];
        *local_n = sh.local_n;
        *halo_n = sh.halo_n;
        *nnz = sh.local.nnz();
        auto flat = [](const std::vector<WorkerShard::NeighborRows>& pl, uint64_t* out, size_t* len) {
            size_t l = 0;
            for (auto& nr : pl) {
                if (out) {
                    out[l] = nr.neighbor;
                    out[l + 1] = nr.rows.size();
                    for (size_t k = 0; k < nr.rows.size(); ++k) out[l + 2 + k] = nr.rows[k];
                }
                l += 2 + nr.rows.size();
            }
            *len = l;
        };
        flat(sh.send_plan, send_flat, send_len);
        flat(sh.recv_plan, recv_flat, recv_len);
        if (rp) {
            for (size_t i = 0; i <= sh.local_n; ++i) rp[i] = sh.local.row_ptr[i];
            std::memcpy(ci, sh.local.col_idx.data(), sh.local.nnz() * 4);
            std::memcpy(v, sh.local.values.data(), sh.local.nnz() * 16);
            for (size_t s = 0; s < sh.halo_n; ++s) halo_global[s] = sh.halo_global[s];
        }
    });
}
// filter_distributed over QueueTransport (dist.hpp:227-359); X in/out global panel-concat.
int ref_filter_distributed(void* h, size_t workers, int pipelined, size_t ns, size_t nb, double* X, size_t np,
                           const double* c, const double* g, double a, double b, double* eta, double* mu) {
    return guard([&] {
        auto& H = *static_cast<SparseMatrixCRS*>(h);
        BlockVector Xv(H.n, ns, nb);
        load_all(Xv, X);
        auto plan = partition_rows(H, workers);
        auto shards = shard_and_distribute(H, Xv, plan);
        QueueTransport t(workers);
        auto res = filter_distributed(shards, make_fc(np, c, g, a, b),
                                      pipelined ? CommMode::pipelined : CommMode::vector, t);
        store_all(res.X, X);
        std::memcpy(eta, res.moments.eta.data(), res.moments.eta.size() * 16);
        std::memcpy(mu, res.moments.mu.data(), res.moments.mu.size() * 16);
    });
}

// ---- chebfd_solve (filter.hpp:247-320) ----
int ref_chebfd_solve(void* h, double lo, double hi, size_t ns, size_t nb, size_t np, size_t max_restarts,
                     double res_tol, uint64_t seed, int use_bounds, double blo, double bhi, double* eig_out,
                     size_t* n_eig, size_t* iterations, int* converged) {
    return guard([&] {
        SolveOptions opt;
        opt.n_s = ns;
        opt.n_b = nb;
        opt.n_p = np;
        opt.max_restarts = max_restarts;
        opt.res_tol = res_tol;
        opt.seed = seed;
        if (use_bounds) opt.spectral_bounds = std::make_pair(blo, bhi);
        auto r = chebfd_solve(*static_cast<SparseMatrixCRS*>(h), lo, hi, opt);
        *n_eig = r.eigenvalues.size();
        for (size_t i = 0; i < r.eigenvalues.size(); ++i) eig_out[i] = r.eigenvalues[i];
        *iterations = r.iterations;
        *converged = r.converged ? 1 : 0;
    });
}

// ---- perf model (perf_model.hpp:41-68) ----
double ref_arithmetic_intensity(size_t nb) {
    KernelGeometry g;
    g.n_b = nb;
    return arithmetic_intensity(g);
}
void ref_min_traffic(size_t n, size_t nb, double* rd, double* wr) {
    KernelGeometry g;
    g.n = n;
    g.n_b = nb;
    auto t = min_traffic_volume(g);
    *rd = t.first;
    *wr = t.second;
}
}  // extern "C"
