// Reference known-answer tests restated as a plain-main harness (the reference's
// Catch2 suites cannot build here) and compiled against the DROP-IN header
// include/chebfilter_b200.hpp: the bodies follow proj/tests/test_kernels.cpp,
// test_filter.cpp and acceptance.cpp with the reference's API and tolerances;
// only the include line differs.  One PASS/FAIL line per case; exit code = failures.
#include <cstdio>
#include <functional>
#include <string>

#include "chebfilter_b200.hpp"

using namespace chebfilter;

namespace {
int failures = 0;
void check(bool ok, const std::string& name) {
    std::printf("%s %s\n", ok ? "PASS" : "FAIL", name.c_str());
    if (!ok) ++failures;
}
template <class E, class F>
bool throws(F&& f) {
    try {
        f();
    } catch (const E&) {
        return true;
    } catch (...) {
        return false;
    }
    return false;
}

// Deterministic random Hermitian test matrix (own generator; dense, row-major).
std::vector<cplx> random_hermitian(std::size_t n, std::uint64_t seed) {
    std::vector<cplx> a(n * n);
    std::uint64_t s = seed * 0x9e3779b97f4a7c15ULL + 1;
    auto u = [&]() {
        s ^= s << 13;
        s ^= s >> 7;
        s ^= s << 17;
        return static_cast<double>(s >> 11) * 0x1.0p-53 * 2.0 - 1.0;
    };
    for (std::size_t i = 0; i < n; ++i) {
        a[i * n + i] = cplx(u(), 0.0);
        for (std::size_t j = i + 1; j < n; ++j) {
            a[i * n + j] = cplx(u(), u());
            a[j * n + i] = std::conj(a[i * n + j]);
        }
    }
    return a;
}
SparseMatrixCRS to_sparse(const std::vector<cplx>& a, std::size_t n) {
    std::vector<Triplet> t;
    for (std::size_t i = 0; i < n; ++i)
        for (std::size_t j = 0; j < n; ++j)
            if (a[i * n + j] != cplx(0.0)) t.push_back({i, j, a[i * n + j]});
    return build_from_triplets(n, t);
}
std::vector<cplx> dense_shifted_mult(const std::vector<cplx>& a, std::size_t n, ShiftScale s,
                                     const std::vector<cplx>& x, std::size_t nb) {
    std::vector<cplx> y(n * nb, cplx(0.0));
    for (std::size_t i = 0; i < n; ++i)
        for (std::size_t j = 0; j < nb; ++j) {
            cplx acc = s.beta * x[i * nb + j];
            for (std::size_t k = 0; k < n; ++k) acc += s.alpha * a[i * n + k] * x[k * nb + j];
            y[i * nb + j] = acc;
        }
    return y;
}
double max_rel_diff(const std::vector<cplx>& a, const std::vector<cplx>& b) {
    double scale = 0.0, diff = 0.0;
    for (const cplx& z : a) scale = std::max(scale, std::abs(z));
    for (std::size_t i = 0; i < a.size(); ++i) diff = std::max(diff, std::abs(a[i] - b[i]));
    return diff / std::max(scale, 1e-300);
}
double filter_poly(const FilterCoefficients& fc, double lambda) {
    double x = fc.map.alpha * lambda + fc.map.beta;
    double tm = 1.0, t = x;
    double acc = fc.g[0] * fc.c[0] + fc.g[1] * fc.c[1] * t;
    for (std::size_t p = 2; p <= fc.np; ++p) {
        double tn = 2.0 * x * t - tm;
        acc += fc.g[p] * fc.c[p] * tn;
        tm = t;
        t = tn;
    }
    return acc;
}
}  // namespace

int main() {
    {  // test_kernels.cpp:34-44
        auto I = diagonal_matrix({1.0, 1.0, 1.0, 1.0});
        BlockVector X(4, 2, 2, InitSeededRandom{5});
        BlockVector Y(4, 2, 2);
        spmmv_shifted(I, {1.0, 0.0}, SubblockView(X, 0), SubblockView(Y, 0));
        bool ok = Y.panel(0) == X.panel(0);
        spmmv_shifted(I, {0.0, 2.5}, SubblockView(X, 0), SubblockView(Y, 0));
        for (std::size_t i = 0; i < X.panel(0).size(); ++i) ok = ok && Y.panel(0)[i] == 2.5 * X.panel(0)[i];
        check(ok, "spmmv identity and scaling cases");
    }
    {  // :46-56
        const std::size_t n = 6, nb = 3;
        auto a = random_hermitian(n, 11);
        auto H = to_sparse(a, n);
        ShiftScale s{0.7, -0.2};
        BlockVector X(n, nb, nb, InitSeededRandom{21}), Y(n, nb, nb);
        spmmv_shifted(H, s, SubblockView(X, 0), SubblockView(Y, 0));
        check(max_rel_diff(Y.panel(0), dense_shifted_mult(a, n, s, X.panel(0), nb)) < 1e-13,
              "spmmv matches the dense oracle");
    }
    {  // :58-63
        auto I = diagonal_matrix({1.0, 1.0});
        BlockVector X(2, 2, 2);
        check(throws<std::invalid_argument>([&] { spmmv_shifted(I, {}, SubblockView(X, 0), SubblockView(X, 0)); }),
              "spmmv rejects aliasing");
    }
    {  // :65-77
        const std::size_t n = 8, nb = 2;
        auto a = random_hermitian(n, 3);
        auto H = to_sparse(a, n);
        ShiftScale s{0.5, 0.1};
        BlockVector U(n, nb, nb, InitSeededRandom{31}), W(n, nb, nb, InitSeededRandom{32});
        auto w_old = W.panel(0);
        spmmv_shifted_two_minus(H, s, SubblockView(U, 0), SubblockView(W, 0), SubblockView(W, 0));
        auto prod = dense_shifted_mult(a, n, s, U.panel(0), nb);
        for (std::size_t i = 0; i < prod.size(); ++i) prod[i] = 2.0 * prod[i] - w_old[i];
        check(max_rel_diff(W.panel(0), prod) < 1e-13, "two_minus form supports in-place update");
    }
    {  // :79-98
        std::vector<double> d{0.3, -0.8, 0.5, 0.0};
        auto H = diagonal_matrix(d);
        ShiftScale s{0.9, 0.05};
        BlockVector X(4, 2, 2, InitSeededRandom{8});
        auto x0 = X.panel(0);
        BlockVector U(4, 2, 2), W(4, 2, 2);
        cheb_init(H, s, SubblockView(X, 0), SubblockView(U, 0), SubblockView(W, 0), 1.0, 0.0, 0.0);
        bool ok = true;
        for (std::size_t i = 0; i < 4; ++i) {
            double xt = s.alpha * d[i] + s.beta;
            for (std::size_t j = 0; j < 2; ++j) {
                ok = ok && std::abs(U(i, j) - xt * x0[i * 2 + j]) < 1e-14;
                ok = ok && std::abs(W(i, j) - (2 * xt * xt - 1) * x0[i * 2 + j]) < 1e-14;
            }
        }
        ok = ok && X.panel(0) == x0;
        check(ok, "cheb_init on a diagonal matrix gives T1 and T2");
    }
    {  // :100-124
        const std::size_t n = 8, nb = 4;
        auto a = random_hermitian(n, 17);
        for (auto& z : a) z *= 0.2;
        auto H = to_sparse(a, n);
        ShiftScale s{0.6, 0.02};
        double g0c0 = 0.4, g1c1 = -0.3, g2c2 = 0.25;
        BlockVector X(n, nb, nb, InitSeededRandom{77});
        auto x0 = X.panel(0);
        BlockVector U(n, nb, nb), W(n, nb, nb);
        cheb_init(H, s, SubblockView(X, 0), SubblockView(U, 0), SubblockView(W, 0), g0c0, g1c1, g2c2);
        auto t1 = dense_shifted_mult(a, n, s, x0, nb);
        auto t2 = dense_shifted_mult(a, n, s, t1, nb);
        std::vector<cplx> expect(n * nb);
        for (std::size_t i = 0; i < n * nb; ++i) {
            t2[i] = 2.0 * t2[i] - x0[i];
            expect[i] = g0c0 * x0[i] + g1c1 * t1[i] + g2c2 * t2[i];
        }
        check(max_rel_diff(X.panel(0), expect) < 1e-13 && max_rel_diff(U.panel(0), t1) < 1e-13 &&
                  max_rel_diff(W.panel(0), t2) < 1e-13,
              "cheb_init against a dense Chebyshev recurrence oracle");
    }
    {  // :156-177
        std::vector<double> d{0.9, -0.4, 0.1, 0.7};
        auto H = diagonal_matrix(d);
        ShiftScale s{1.0, 0.0};
        const std::size_t n = 4, nb = 4, np = 12;
        BlockVector X(n, nb, nb), U(n, nb, nb), W(n, nb, nb);
        for (std::size_t j = 0; j < nb; ++j) X(j, j) = 1.0;
        auto x0 = X.panel(0);
        cheb_init(H, s, SubblockView(X, 0), SubblockView(U, 0), SubblockView(W, 0), 1.0, 0.0, 0.0);
        MomentSeries mom(np, nb);
        for (std::size_t p = 3; p <= np; ++p) {
            swap_blocks(SubblockView(W, 0), SubblockView(U, 0));
            chebfd_op(H, s, SubblockView(U, 0), SubblockView(W, 0), SubblockView(X, 0), p, 0.0, mom);
        }
        bool ok = true;
        for (std::size_t i = 0; i < n; ++i) {
            double t = std::cos(np * std::acos(d[i]));
            for (std::size_t j = 0; j < nb; ++j) ok = ok && std::abs(W(i, j) - t * x0[i * nb + j]) < 1e-11;
        }
        check(ok, "recurrence on a diagonal matrix reproduces T_P pointwise");
    }
    {  // :179-203
        const std::size_t n = 5, nb = 2, np = 7;
        auto H = diagonal_matrix({1.0, 1.0, 1.0, 1.0, 1.0});
        ShiftScale s{1.0, 0.0};
        BlockVector X(n, nb, nb, InitSeededRandom{55});
        auto x0 = X.panel(0);
        std::vector<double> norms(nb, 0.0);
        for (std::size_t i = 0; i < n; ++i)
            for (std::size_t j = 0; j < nb; ++j) norms[j] += std::norm(x0[i * nb + j]);
        BlockVector U(n, nb, nb), W(n, nb, nb);
        cheb_init(H, s, SubblockView(X, 0), SubblockView(U, 0), SubblockView(W, 0), 1.0, 0.0, 0.0);
        MomentSeries mom(np, nb);
        for (std::size_t p = 3; p <= np; ++p) {
            swap_blocks(SubblockView(W, 0), SubblockView(U, 0));
            chebfd_op(H, s, SubblockView(U, 0), SubblockView(W, 0), SubblockView(X, 0), p, 0.0, mom);
        }
        bool ok = true;
        for (std::size_t p = 3; p <= np; ++p)
            for (std::size_t j = 0; j < nb; ++j) {
                ok = ok && std::abs(mom.mu_at(p, j) - norms[j]) < 1e-12 * norms[j];
                ok = ok && std::abs(mom.eta_at(p, j) - mom.mu_at(p, j)) < 1e-12 * norms[j];
            }
        check(ok, "moments at the fixed point x~ = 1");
    }
    {  // :205-223
        const std::size_t n = 30, nb = 4, np = 10;
        auto a = random_hermitian(n, 9);
        for (auto& z : a) z *= 0.15;
        auto H = to_sparse(a, n);
        BlockVector X(n, nb, nb, InitSeededRandom{66}), U(n, nb, nb), W(n, nb, nb);
        cheb_init(H, {1.0, 0.0}, SubblockView(X, 0), SubblockView(U, 0), SubblockView(W, 0), 1.0, 0.1, 0.1);
        MomentSeries mom(np, nb);
        for (std::size_t p = 3; p <= np; ++p) {
            swap_blocks(SubblockView(W, 0), SubblockView(U, 0));
            chebfd_op(H, {1.0, 0.0}, SubblockView(U, 0), SubblockView(W, 0), SubblockView(X, 0), p, 0.1, mom);
        }
        bool ok = true;
        for (const cplx& m : mom.mu) ok = ok && m.real() >= 0.0 && std::abs(m.imag()) <= 1e-12 * std::abs(m);
        check(ok, "mu is real and nonnegative");
    }
    {  // :225-256 (thread counts -> reruns on the device)
        const std::size_t n = 64, nb = 4, np = 9;
        auto a = random_hermitian(n, 14);
        for (auto& z : a) z *= 0.1;
        auto H = to_sparse(a, n);
        auto run = [&]() {
            BlockVector X(n, nb, nb, InitSeededRandom{4}), U(n, nb, nb), W(n, nb, nb);
            cheb_init(H, {1.0, 0.0}, SubblockView(X, 0), SubblockView(U, 0), SubblockView(W, 0), 0.5, 0.2, 0.1);
            MomentSeries mom(np, nb);
            for (std::size_t p = 3; p <= np; ++p) {
                swap_blocks(SubblockView(W, 0), SubblockView(U, 0));
                chebfd_op(H, {1.0, 0.0}, SubblockView(U, 0), SubblockView(W, 0), SubblockView(X, 0), p, 0.05, mom);
            }
            return mom;
        };
        auto m1 = run(), m2 = run();
        check(m1.eta == m2.eta && m1.mu == m2.mu, "moments are bit-identical across reruns");
    }
    {  // :258-286
        const std::size_t n = 20, nb = 2, np = 6;
        auto a = random_hermitian(n, 2);
        auto H = to_sparse(a, n);
        BlockVector X(n, nb, nb, InitSeededRandom{12}), U(n, nb, nb), W(n, nb, nb);
        TrafficCounter tc;
        cheb_init(H, {0.1, 0.0}, SubblockView(X, 0), SubblockView(U, 0), SubblockView(W, 0), 1, 0, 0, &tc);
        bool ok = true;
        for (std::size_t p = 3; p <= np; ++p) {
            MomentSeries mom(np, nb);
            TrafficCounter step;
            swap_blocks(SubblockView(W, 0), SubblockView(U, 0));
            chebfd_op(H, {0.1, 0.0}, SubblockView(U, 0), SubblockView(W, 0), SubblockView(X, 0), p, 0.0, mom, 0,
                      &step);
            ok = ok && step.panel_reads == 3 && step.panel_writes == 2 && step.matrix_sweeps == 1;
        }
        check(ok, "traffic counters match the minimum-traffic contract");
    }
    {  // test_filter.cpp:81-92
        std::vector<double> d{-0.9, -0.3, 0.0, 0.25, 0.6, 0.95};
        auto H = diagonal_matrix(d);
        auto fc = filter_coefficients(-0.2, 0.3, ShiftScale{1.0, 0.0}, 80);
        BlockVector X(d.size(), 2, 2, InitConstant{cplx(1.0)});
        apply_filter(H, X, fc);
        bool ok = true;
        for (std::size_t i = 0; i < d.size(); ++i) {
            double expect = filter_poly(fc, d[i]);
            ok = ok && std::abs(X(i, 0) - cplx(expect)) < 1e-12 && std::abs(X(i, 1) - cplx(expect)) < 1e-12;
        }
        check(ok, "apply_filter matches the scalar polynomial on a diagonal matrix");
    }
    {  // :94-102
        auto H = diagonal_matrix({-0.9, 0.0, 0.9});
        auto fc = filter_coefficients(-0.1, 0.1, ShiftScale{1.0, 0.0}, 100);
        BlockVector X(3, 1, 1, InitConstant{cplx(1.0)});
        apply_filter(H, X, fc);
        double inside = std::abs(X(1, 0));
        check(std::abs(X(0, 0)) * 1e3 < inside && std::abs(X(2, 0)) * 1e3 < inside,
              "window suppression on a diagonal matrix");
    }
    {  // :116-136
        const std::size_t n = 40, ns = 8;
        auto a = random_hermitian(n, 23);
        for (auto& z : a) z *= 0.1;
        auto H = to_sparse(a, n);
        auto fc = filter_coefficients(-0.1, 0.1, ShiftScale{1.0, 0.0}, 40);
        BlockVector ref(n, ns, ns, InitSeededRandom{5});
        auto mref = apply_filter(H, ref, fc);
        bool ok = true;
        for (std::size_t nb : {1, 2, 4}) {
            BlockVector X(n, ns, nb, InitSeededRandom{5});
            auto m = apply_filter(H, X, fc);
            for (std::size_t i = 0; i < n; ++i)
                for (std::size_t j = 0; j < ns; ++j) ok = ok && std::abs(X(i, j) - ref(i, j)) < 1e-12;
            for (std::size_t i = 0; i < m.eta.size(); ++i)
                ok = ok && std::abs(m.eta[i] - mref.eta[i]) < 1e-12 * (1.0 + std::abs(mref.eta[i]));
        }
        check(ok, "apply_filter is invariant under the block width");
    }
    {  // test_filter.cpp:34-63 error behaviour
        ShiftScale id{1.0, 0.0};
        bool ok = throws<std::invalid_argument>([] { spectral_map(1.0, 1.0); }) &&
                  throws<std::invalid_argument>([] { spectral_map(0.0, 1.0, -0.1); }) &&
                  throws<std::invalid_argument>([&] { filter_coefficients(-1.2, 0.0, id, 20); }) &&
                  throws<std::invalid_argument>([&] { filter_coefficients(0.3, 0.1, id, 20); }) &&
                  throws<std::invalid_argument>([&] { filter_coefficients(-0.1, 0.1, id, 1); });
        check(ok, "spectral map and coefficient errors");
    }
    {  // test_matrix.cpp:14-35, 59-83; block_vector swap (test_blockvec.cpp:266-289)
        LatticeSpec spec;
        spec.nx = spec.ny = spec.nz = 4;
        auto H = topi_generate(spec);
        bool ok = H.n == 256;
        for (std::size_t i = 0; i < H.n; ++i) ok = ok && H.row_ptr[i + 1] - H.row_ptr[i] == 13;
        auto [lo, hi] = gershgorin_bounds(H);
        ok = ok && lo == -7.0 && hi == 7.0;
        BlockVector A(32, 4, 2, InitSeededRandom{1}), B(32, 4, 2, InitSeededRandom{2});
        auto a_copy = A.panel(0);
        auto b_copy = B.panel(1);
        swap_blocks(SubblockView(A, 0), SubblockView(B, 1));
        ok = ok && A.panel(0) == b_copy && B.panel(1) == a_copy;
        swap_blocks(SubblockView(A, 0), SubblockView(B, 1));
        ok = ok && A.panel(0) == a_copy && B.panel(1) == b_copy;
        check(ok, "topi shape, Gershgorin bounds, swap involution");
    }
    {  // acceptance.cpp:161-191 serial filter on topi 4^3 through the drop-in: finite, bounded
        LatticeSpec spec;
        spec.nx = spec.ny = spec.nz = 4;
        auto H = topi_generate(spec);
        auto fc = filter_coefficients(-0.5, 0.5, spectral_map(-8.0, 8.0), 50);
        BlockVector X(H.n, 8, 2, InitSeededRandom{31});
        auto m = apply_filter(H, X, fc);
        bool ok = m.eta.size() == 48 * 8;
        for (const cplx& z : m.mu) ok = ok && std::isfinite(z.real()) && z.real() >= 0.0;
        check(ok, "apply_filter on topi 4^3 through the drop-in");
    }
    {  // test_filter.cpp:180-194 Rayleigh-Ritz with a full basis vs the dense eigenvalues
        const std::size_t n = 10;
        auto a = random_hermitian(n, 37);
        auto H = to_sparse(a, n);
        BlockVector X(n, n, n, InitSeededRandom{17});
        auto [Q, rank] = orthogonalize_svqb(X);
        bool ok = rank == n;
        auto rr = rayleigh_ritz(H, Q);
        HermitianDense D(n);
        D.a = a;
        auto exact = jacobi_hermitian_eig(D, 1e-14, 100).values;
        for (std::size_t i = 0; i < n; ++i) ok = ok && std::abs(rr.theta[i] - exact[i]) < 1e-10;
        for (double r : rr.residuals) ok = ok && r < 1e-9;
        BlockVector bad(n, 2, 2, InitConstant{cplx(0.5)});
        ok = ok && throws<std::invalid_argument>([&] { rayleigh_ritz(H, bad); });
        check(ok, "rayleigh-ritz with a full basis matches the dense eigenvalues");
    }
    {  // test_filter.cpp:195-215
        std::vector<double> vals(200);
        for (int i = 0; i < 200; ++i) vals[i] = -1.0 + 2.0 * i / 199.0;
        auto H = diagonal_matrix(vals);
        double lo = 0.5 * (vals[95] + vals[96]), hi = 0.5 * (vals[103] + vals[104]);
        SolveOptions opt;
        opt.n_s = 16;
        opt.n_b = 4;
        opt.n_p = 300;
        auto res = chebfd_solve(H, lo, hi, opt);
        bool ok = res.converged && res.eigenvalues.size() == 8 && res.moments.size() == res.iterations;
        for (std::size_t i = 0; ok && i < 8; ++i)
            ok = std::abs(res.eigenvalues[i] - vals[96 + i]) < 1e-8 && res.residuals[i] <= opt.res_tol;
        ok = ok && res.eigenvectors.cols() == 8 && std::abs(std::abs(res.eigenvectors(96, 0)) - 1.0) < 1e-8;
        check(ok, "solve finds interior eigenvalues of a diagonal matrix");
    }
    {  // test_filter.cpp:245-257, 281-285
        std::vector<double> vals;
        for (int i = 0; i < 20; ++i) vals.push_back(-1.0 + 0.5 * i / 19.0);
        for (int i = 0; i < 20; ++i) vals.push_back(0.5 + 0.5 * i / 19.0);
        auto H = diagonal_matrix(vals);
        SolveOptions opt;
        opt.n_s = 8;
        opt.n_b = 2;
        opt.n_p = 200;
        auto res = chebfd_solve(H, -0.1, 0.1, opt);
        bool ok = res.converged && res.eigenvalues.empty();
        auto D = diagonal_matrix({-1.0, 0.0, 1.0});
        ok = ok && throws<std::invalid_argument>([&] { chebfd_solve(D, -2.0, 0.0); });
        check(ok, "empty window converges to zero pairs; window outside bounds rejected");
    }
    {  // test_matrix.cpp:84-131 Matrix Market round trip, offending line, hermitian expansion; CFDB round trip
        LatticeSpec spec;
        spec.nx = spec.ny = spec.nz = 2;
        auto H = topi_generate(spec);
        const std::string dir = "/tmp";
        matrix_market_write(dir + "/kat_rt.mtx", H);
        auto H2 = matrix_market_read(dir + "/kat_rt.mtx");
        bool ok = H2.n == H.n && H2.row_ptr == H.row_ptr && H2.col_idx == H.col_idx && H2.values == H.values;
        {
            std::FILE* f = std::fopen((dir + "/kat_bad.mtx").c_str(), "w");
            std::fputs("%%MatrixMarket matrix coordinate complex general\n3 3 2\n1 1 1.0 0.0\n4 1 1.0 0.0\n", f);
            std::fclose(f);
        }
        try {
            matrix_market_read(dir + "/kat_bad.mtx");
            ok = false;
        } catch (const MatrixMarketError& e) {
            ok = ok && e.line_number == 4;
        }
        BlockVector X(9, 4, 2, InitSeededRandom{4});
        block_vector_write(dir + "/kat.cfdb", X);
        auto Y = block_vector_read(dir + "/kat.cfdb");
        ok = ok && Y.rows() == 9 && Y.cols() == 4 && Y.block_width() == 2 && Y.panel(0) == X.panel(0) &&
             Y.panel(1) == X.panel(1);
        std::remove((dir + "/kat_rt.mtx").c_str());
        std::remove((dir + "/kat_bad.mtx").c_str());
        std::remove((dir + "/kat.cfdb").c_str());
        check(ok, "matrix market and CFDB files through the drop-in");
    }
    {  // test_dist.cpp:112-137 / acceptance.cpp:161-191 (criterion 6)
        LatticeSpec spec;
        spec.nx = spec.ny = spec.nz = 4;
        auto H = topi_generate(spec);
        auto fc = filter_coefficients(-0.5, 0.5, spectral_map(-8.0, 8.0), 50);
        const std::size_t ns = 8, nb = 2;
        BlockVector serial(H.n, ns, nb, InitSeededRandom{31});
        auto serial_moments = apply_filter(H, serial, fc);
        bool ok = true;
        for (std::size_t workers : {1, 2, 4}) {
            for (CommMode mode : {CommMode::vector, CommMode::pipelined}) {
                auto plan = partition_rows(H, workers);
                BlockVector X(H.n, ns, nb, InitSeededRandom{31});
                auto shards = shard_and_distribute(H, X, plan);
                QueueTransport transport(workers);
                auto res = filter_distributed(shards, fc, mode, transport);
                for (std::size_t i = 0; ok && i < H.n; ++i)
                    for (std::size_t j = 0; ok && j < ns; ++j)
                        ok = std::abs(res.X(i, j) - serial(i, j)) <= 1e-12 * (1.0 + std::abs(serial(i, j)));
                for (std::size_t i = 0; ok && i < serial_moments.eta.size(); ++i) {
                    double scale = 1.0 + std::abs(serial_moments.eta[i]);
                    ok = std::abs(res.moments.eta[i] - serial_moments.eta[i]) <= 1e-12 * scale &&
                         std::abs(res.moments.mu[i] - serial_moments.mu[i]) <= 1e-12 * scale;
                }
            }
        }
        check(ok, "distributed modes reproduce the serial filter");
    }
    {  // test_dist.cpp:157-175 (traffic counters) and partition plan invariants (test_dist.cpp:45-75)
        LatticeSpec spec;
        spec.nx = spec.ny = spec.nz = 4;
        auto H = topi_generate(spec);
        auto fc = filter_coefficients(-0.5, 0.5, spectral_map(-8.0, 8.0), 20);
        const std::size_t ns = 8, nb = 2, workers = 2, ops = workers * (ns / nb) * (fc.np - 2);
        bool ok = true;
        for (CommMode mode : {CommMode::vector, CommMode::pipelined}) {
            auto plan = partition_rows(H, workers);
            BlockVector X(H.n, ns, nb, InitSeededRandom{1});
            auto shards = shard_and_distribute(H, X, plan);
            QueueTransport transport(workers);
            auto res = filter_distributed(shards, fc, mode, transport);
            ok = ok && res.traffic.panel_reads == 3 * ops && res.traffic.panel_writes == 2 * ops &&
                 res.traffic.matrix_sweeps == ops;
            // dist.hpp:216-219 timelines (measured here): per worker one compute and one comm
            // interval per (panel, degree), ordered, inside the makespan
            ok = ok && res.timelines.size() == workers;
            for (const Timeline& tl : res.timelines) {
                std::size_t comp = 0, comm = 0;
                for (const TimelineEvent& e : tl.events) {
                    (e.kind == TimelineEvent::Kind::compute ? comp : comm) += 1;
                    ok = ok && e.start >= 0.0 && e.end >= e.start && e.end <= tl.makespan() && e.block < ns / nb &&
                         e.degree >= 3 && e.degree <= fc.np;
                }
                ok = ok && comp == (ns / nb) * (fc.np - 2) && comm == comp;
            }
        }
        auto plan = partition_rows(H, 3);
        ok = ok && plan.row_ranges.front().first == 0 && plan.row_ranges.back().second == H.n;
        for (std::size_t w = 0; w < 3; ++w)
            for (const auto& [v, rows] : plan.halo_in[w])
                for (std::size_t r : rows) ok = ok && plan.owner_of(r) == v && plan.halo_out[v].at(w) == rows;
        ok = ok && throws<std::invalid_argument>([&] { partition_rows(H, 0); });
        check(ok, "distributed traffic counters, measured timelines and partition plans");
    }
    {  // test_dist.cpp:77-92 (halo exchange delivers owner values)
        LatticeSpec spec;
        spec.nx = spec.ny = spec.nz = 4;
        auto H = topi_generate(spec);
        auto plan = partition_rows(H, 2);
        BlockVector X(H.n, 4, 2, InitSeededRandom{12});
        auto shards = shard_and_distribute(H, X, plan);
        QueueTransport transport(2);
        // sends are non-blocking, so a single thread can drive both workers
        for (auto& sh : shards) halo_exchange(sh, sh.X, 0, ExchangePhase::init, transport, 1);
        for (auto& sh : shards) halo_exchange(sh, sh.X, 0, ExchangePhase::finalize, transport, 1);
        bool ok = true;
        for (const auto& sh : shards)
            for (std::size_t s = 0; s < sh.halo_n; ++s)
                for (std::size_t j = 0; j < 2; ++j) ok = ok && sh.X(sh.local_n + s, j) == X(sh.halo_global[s], j);
        check(ok, "halo exchange delivers owner values");
    }
    {  // test_dist.cpp:94-110 (halo exchange protocol violations)
        LatticeSpec spec;
        spec.nx = spec.ny = spec.nz = 4;
        auto H = topi_generate(spec);
        auto plan = partition_rows(H, 2);
        BlockVector X(H.n, 4, 2, InitSeededRandom{12});
        auto shards = shard_and_distribute(H, X, plan);
        QueueTransport transport(2);
        bool ok = throws<ProtocolError>(
            [&] { halo_exchange(shards[0], shards[0].X, 0, ExchangePhase::finalize, transport, 1); });
        halo_exchange(shards[0], shards[0].X, 0, ExchangePhase::init, transport, 1);
        ok = ok && throws<ProtocolError>(
                       [&] { halo_exchange(shards[0], shards[0].X, 0, ExchangePhase::init, transport, 1); });
        ok = ok && throws<std::invalid_argument>(
                       [&] { halo_exchange(shards[0], shards[0].X, 9, ExchangePhase::init, transport, 1); });
        // a frame of another degree is a tag mismatch (dist.hpp:135-136)
        halo_exchange(shards[1], shards[1].X, 0, ExchangePhase::init, transport, 2);
        ok = ok && throws<ProtocolError>(
                       [&] { halo_exchange(shards[0], shards[0].X, 0, ExchangePhase::finalize, transport, 1); });
        check(ok, "halo exchange protocol violations");
    }
    {  // shards placed per device (B200 overload; here every entry is this thread's GPU)
        LatticeSpec spec;
        spec.nx = spec.ny = spec.nz = 4;
        auto H = topi_generate(spec);
        auto fc = filter_coefficients(-0.5, 0.5, spectral_map(-8.0, 8.0), 30);
        BlockVector serial(H.n, 4, 2, InitSeededRandom{5});
        auto serial_moments = apply_filter(H, serial, fc);
        int dev = 0;
        detail::check(cf_current_device(&dev));
        auto plan = partition_rows(H, 3);
        BlockVector X(H.n, 4, 2, InitSeededRandom{5});
        auto shards = shard_and_distribute(H, X, plan, std::vector<int>{dev, dev, dev});
        QueueTransport transport(3);
        auto res = filter_distributed(shards, fc, CommMode::pipelined, transport);
        bool ok = true;
        for (std::size_t i = 0; ok && i < H.n; ++i)
            for (std::size_t j = 0; ok && j < 4; ++j)
                ok = std::abs(res.X(i, j) - serial(i, j)) <= 1e-12 * (1.0 + std::abs(serial(i, j)));
        for (std::size_t i = 0; ok && i < serial_moments.eta.size(); ++i)
            ok = std::abs(res.moments.eta[i] - serial_moments.eta[i]) <= 1e-12 * (1.0 + std::abs(serial_moments.eta[i]));
        check(ok, "shards placed by device list reproduce the serial filter");
    }
    {  // chebfd_op in a caller's degree loop: host MomentSeries accumulates like kernels.hpp:199-202
        LatticeSpec spec;
        spec.nx = 6;
        spec.ny = 5;
        spec.nz = 4;
        auto H = topi_generate(spec);
        auto fc = filter_coefficients(-0.4, 0.4, spectral_map(-7.0, 7.0, 0.01), 40);
        BlockVector A(H.n, 8, 8, InitSeededRandom{3});
        auto ref = apply_filter(H, A, fc);  // device degree loop
        BlockVector X(H.n, 8, 8, InitSeededRandom{3}), U(H.n, 8, 8), W(H.n, 8, 8);
        MomentSeries mom(fc.np, 8);
        SubblockView x(X, 0), u(U, 0), w(W, 0);
        cheb_init(H, fc.map, x, u, w, fc.g[0] * fc.c[0], fc.g[1] * fc.c[1], fc.g[2] * fc.c[2]);
        for (std::size_t p = 3; p <= fc.np; ++p) {
            swap_blocks(w, u);
            chebfd_op(H, fc.map, u, w, x, p, fc.g[p] * fc.c[p], mom);
        }
        bool ok = max_rel_diff(ref.eta, mom.eta) <= 1e-12 && max_rel_diff(ref.mu, mom.mu) <= 1e-12 &&
                  max_rel_diff(A.panel(0), X.panel(0)) <= 1e-12;
        check(ok, "chebfd_op degree loop with host moments matches apply_filter");
    }
    if (failures) std::printf("%d case(s) FAILED\n", failures);
    return failures;
}
