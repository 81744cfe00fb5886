/*
 * chebfd_oracle.c -- CPU restatement of the reference ChebFD hot path.
 * TEST INFRASTRUCTURE ONLY (see chebfd_oracle.h).  Build: oracle/Makefile
 * (gcc -O2 -ffp-contract=off; no -march, so no FMA, like the reference build).
 *
 * Single-threaded, but it reproduces the reference's fixed 64-chunk row split
 * and pairwise tree reduction (proj/include/chebfilter/parallel.hpp:26-45,
 * kernels.hpp:71-77), so moments are bit-identical to the threaded reference.
 */
#include "chebfd_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ---------------------------------------------------------------- RNG --- */
/* block_vector.hpp:17-23 */
uint64_t or_splitmix64(uint64_t x) {
    x += 0x9e3779b97f4a7c15ULL;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
    return x ^ (x >> 31);
}

/* block_vector.hpp:27-35: Box-Muller on two splitmix64 hashes of (seed, i, j). */
void or_unit_complex_gaussian(uint64_t seed, uint64_t i, uint64_t j, double* out) {
    uint64_t h = or_splitmix64(or_splitmix64(seed) ^ or_splitmix64(i * 0xd1342543de82ef95ULL + j));
    uint64_t h2 = or_splitmix64(h);
    double u = ((double)(h >> 11) + 1.0) * 0x1.0p-53;
    double v = (double)(h2 >> 11) * 0x1.0p-53;
    double r = sqrt(-log(u));
    out[0] = r * cos(6.283185307179586477 * v);
    out[1] = r * sin(6.283185307179586477 * v);
}

/* block_vector.hpp:57-73 (InitSeededRandom branch): column-outer, row-inner. */
int or_blockvec_random(size_t n, size_t ns, size_t nb, uint64_t seed, uint64_t row_offset, double* out) {
    if (n < 1 || nb == 0 || ns == 0 || ns % nb != 0) return 1;
    for (size_t j = 0; j < ns; ++j)
        for (size_t i = 0; i < n; ++i) {
            size_t off = (j / nb) * n * nb + i * nb + j % nb; /* block_vector.hpp:81-94 */
            or_unit_complex_gaussian(seed, row_offset + i, j, out + 2 * off);
        }
    return 0;
}

/* ----------------------------------------------------------- topi gen --- */
typedef struct { double a[4][4][2]; } blk4;

/* sparse_matrix.hpp:131-138 */
static blk4 onsite_block(double m) {
    blk4 b;
    memset(&b, 0, sizeof b);
    b.a[0][0][0] = m;
    b.a[1][1][0] = m;
    b.a[2][2][0] = -m;
    b.a[3][3][0] = -m;
    return b;
}

/* sparse_matrix.hpp:140-167: b = 0.5 t (B + I*alpha_d), complex products expanded. */
static blk4 hop_block(double t, int dir) {
    blk4 al;
    memset(&al, 0, sizeof al);
    /* cplx(1), I = (0,1), -I = (-0,-1), cplx(-1) */
    const double ONE[2] = {1.0, 0.0}, I_[2] = {0.0, 1.0}, MI[2] = {-0.0, -1.0}, M1[2] = {-1.0, 0.0};
#define SET(r, c, v) (al.a[r][c][0] = (v)[0], al.a[r][c][1] = (v)[1])
    switch (dir) {
        case 0: SET(0, 3, ONE); SET(1, 2, ONE); SET(2, 1, ONE); SET(3, 0, ONE); break;
        case 1: SET(0, 3, MI); SET(1, 2, I_); SET(2, 1, MI); SET(3, 0, I_); break;
        default: SET(0, 2, ONE); SET(1, 3, M1); SET(2, 0, ONE); SET(3, 1, M1); break;
    }
#undef SET
    blk4 b = onsite_block(1.0);
    double ht = 0.5 * t;
    for (int r = 0; r < 4; ++r)
        for (int c = 0; c < 4; ++c) {
            double ar = al.a[r][c][0], ai = al.a[r][c][1];
            /* I * alpha = (0*ar - 1*ai, 0*ai + 1*ar) */
            double pr = 0.0 * ar - 1.0 * ai;
            double pi_ = 0.0 * ai + 1.0 * ar;
            double sr = b.a[r][c][0] + pr, si = b.a[r][c][1] + pi_;
            b.a[r][c][0] = ht * sr;
            b.a[r][c][1] = ht * si;
        }
    return b;
}

/* sparse_matrix.hpp:169-174 */
static blk4 adjoint_block(const blk4* b) {
    blk4 r;
    for (int i = 0; i < 4; ++i)
        for (int j = 0; j < 4; ++j) {
            r.a[i][j][0] = b->a[j][i][0];
            r.a[i][j][1] = -b->a[j][i][1];
        }
    return r;
}

typedef struct { uint64_t row, col, seq; double v[2]; } trip_t;

static int trip_cmp(const void* pa, const void* pb) {
    const trip_t* a = (const trip_t*)pa;
    const trip_t* b = (const trip_t*)pb;
    if (a->row != b->row) return a->row < b->row ? -1 : 1;
    if (a->col != b->col) return a->col < b->col ? -1 : 1;
    return a->seq < b->seq ? -1 : (a->seq > b->seq); /* stable: insertion order */
}

/* sparse_matrix.hpp:181-228, duplicates summed in insertion order into a
 * value-initialised (0,0) accumulator as std::map<..>::operator[] += does (:43-64). */
int or_topi_generate(size_t nx, size_t ny, size_t nz, double mass, double hop, int open_boundary, size_t* n_out,
                     size_t* nnz_out, uint64_t* row_ptr, int32_t* col_idx, double* values) {
    if (nx < 1 || ny < 1 || nz < 1) return 1;
    size_t S = nx * ny * nz, n = 4 * S;
    blk4 onsite = onsite_block(mass), hp[3], ha[3];
    for (int d = 0; d < 3; ++d) {
        hp[d] = hop_block(hop, d);
        ha[d] = adjoint_block(&hp[d]);
    }
    size_t cap = S * 16 * 7, nt = 0;
    trip_t* tr = (trip_t*)malloc(cap * sizeof(trip_t));
    if (!tr) return 2;
#define ADD(srow, scol, B)                                                                   \
    for (int r = 0; r < 4; ++r)                                                              \
        for (int c = 0; c < 4; ++c)                                                          \
            if (!((B).a[r][c][0] == 0.0 && (B).a[r][c][1] == 0.0)) {                         \
                tr[nt].row = 4 * (srow) + r;                                                 \
                tr[nt].col = 4 * (scol) + c;                                                 \
                tr[nt].seq = nt;                                                             \
                tr[nt].v[0] = (B).a[r][c][0];                                                \
                tr[nt].v[1] = (B).a[r][c][1];                                                \
                ++nt;                                                                        \
            }
    const size_t ext[3] = {nx, ny, nz};
    for (size_t z = 0; z < nz; ++z)
        for (size_t y = 0; y < ny; ++y)
            for (size_t x = 0; x < nx; ++x) {
                size_t s = (z * ny + y) * nx + x;
                ADD(s, s, onsite);
                size_t coord[3] = {x, y, z};
                for (int d = 0; d < 3; ++d) {
                    size_t f[3] = {coord[0], coord[1], coord[2]};
                    int ok = 1;
                    if (coord[d] + 1 < ext[d]) f[d] = coord[d] + 1;
                    else if (!open_boundary) f[d] = 0;
                    else ok = 0;
                    if (ok) {
                        size_t sn = (f[2] * ny + f[1]) * nx + f[0];
                        ADD(s, sn, hp[d]);
                        ADD(sn, s, ha[d]);
                    }
                }
            }
#undef ADD
    qsort(tr, nt, sizeof(trip_t), trip_cmp);
    size_t nnz = 0;
    for (size_t t = 0; t < nt; ++t)
        if (t == 0 || tr[t].row != tr[t - 1].row || tr[t].col != tr[t - 1].col) ++nnz;
    *n_out = n;
    *nnz_out = nnz;
    if (row_ptr) {
        size_t k = (size_t)-1;
        memset(row_ptr, 0, (n + 1) * sizeof(uint64_t));
        for (size_t t = 0; t < nt; ++t) {
            if (t == 0 || tr[t].row != tr[t - 1].row || tr[t].col != tr[t - 1].col) {
                ++k;
                col_idx[k] = (int32_t)tr[t].col;
                values[2 * k] = 0.0;
                values[2 * k + 1] = 0.0;
                row_ptr[tr[t].row + 1]++;
            }
            values[2 * k] += tr[t].v[0];
            values[2 * k + 1] += tr[t].v[1];
        }
        for (size_t i = 0; i < n; ++i) row_ptr[i + 1] += row_ptr[i];
    }
    free(tr);
    return 0;
}

/* sparse_matrix.hpp:89-107 (std::abs(complex) = hypot) */
int or_gershgorin_bounds(size_t n, const uint64_t* row_ptr, const int32_t* col_idx, const double* values, double* lo,
                         double* hi) {
    if (n == 0) return 1;
    double l = INFINITY, h = -INFINITY;
    for (size_t i = 0; i < n; ++i) {
        double diag = 0.0, radius = 0.0;
        for (uint64_t k = row_ptr[i]; k < row_ptr[i + 1]; ++k) {
            if ((size_t)col_idx[k] == i) diag = values[2 * k];
            else radius += hypot(values[2 * k], values[2 * k + 1]);
        }
        double a = diag - radius, b = diag + radius;
        l = (a < l) ? a : l; /* std::min(lo, x) returns lo unless x < lo */
        h = (h < b) ? b : h; /* std::max(hi, x) returns hi unless hi < x */
    }
    *lo = l;
    *hi = h;
    return 0;
}

/* filter.hpp:25-32 */
int or_spectral_map(double lmin, double lmax, double margin, double* alpha, double* beta) {
    if (!(lmax > lmin) || margin < 0.0) return 1;
    *alpha = 2.0 / ((lmax - lmin) * (1.0 + margin));
    *beta = -*alpha * (lmax + lmin) / 2.0;
    return 0;
}

/* filter.hpp:39-70 */
int or_filter_coefficients(double wlo, double whi, double alpha, double beta, size_t np, int damping, double* c,
                           double* g) {
    if (np < 2) return 1;
    double a = alpha * wlo + beta, b = alpha * whi + beta;
    if (!(a < b) || a <= -1.0 || b >= 1.0) return 1;
    const double pi = 3.14159265358979323846;
    double ta = acos(a), tb = acos(b);
    c[0] = (ta - tb) / pi;
    for (size_t p = 1; p <= np; ++p)
        c[p] = 2.0 / (pi * (double)p) * (sin((double)p * ta) - sin((double)p * tb));
    g[0] = 1.0;
    if (damping == 0) {
        double q = pi / (double)(np + 1);
        double cot_q = cos(q) / sin(q);
        for (size_t p = 1; p <= np; ++p)
            g[p] = ((double)(np - p + 1) * cos((double)p * q) + sin((double)p * q) * cot_q) / (double)(np + 1);
    } else {
        for (size_t p = 1; p <= np; ++p) g[p] = 1.0;
    }
    return 0;
}

/* ------------------------------------------------------------ kernels --- */
#define NCHUNK_MAX 64 /* parallel.hpp:26 kReductionChunks */

static size_t nchunks_for(size_t n) { /* parallel.hpp:35-45 */
    size_t m = n > 1 ? n : 1;
    return m < NCHUNK_MAX ? m : NCHUNK_MAX;
}

/* acc_j = beta*x_i; acc_j += (alpha*h_k) * x_{col_k} (kernels.hpp:92-97) */
static void row_acc(const uint64_t* row_ptr, const int32_t* col_idx, const double* values, double alpha, double beta,
                    size_t nb, const double* x, size_t i, double* acc) {
    for (size_t j = 0; j < nb; ++j) {
        acc[2 * j] = beta * x[2 * (i * nb + j)];
        acc[2 * j + 1] = beta * x[2 * (i * nb + j) + 1];
    }
    for (uint64_t k = row_ptr[i]; k < row_ptr[i + 1]; ++k) {
        double ar = alpha * values[2 * k], ai = alpha * values[2 * k + 1];
        const double* xr = x + 2 * (size_t)col_idx[k] * nb;
        for (size_t j = 0; j < nb; ++j) {
            double ur = xr[2 * j], ui = xr[2 * j + 1];
            double pr = ar * ur - ai * ui;
            double pim = ar * ui + ai * ur;
            acc[2 * j] += pr;
            acc[2 * j + 1] += pim;
        }
    }
}

int or_spmmv_shifted(size_t n, const uint64_t* row_ptr, const int32_t* col_idx, const double* values, double alpha,
                     double beta, size_t nb, const double* X, double* Y) {
    if (X == Y) return 1;
    double* acc = (double*)malloc(2 * nb * sizeof(double));
    for (size_t i = 0; i < n; ++i) {
        row_acc(row_ptr, col_idx, values, alpha, beta, nb, X, i, acc);
        memcpy(Y + 2 * i * nb, acc, 2 * nb * sizeof(double));
    }
    free(acc);
    return 0;
}

int or_spmmv_shifted_two_minus(size_t n, const uint64_t* row_ptr, const int32_t* col_idx, const double* values,
                               double alpha, double beta, size_t nb, const double* X, double* Y, const double* Z) {
    if (X == Y || X == Z) return 1;
    double* acc = (double*)malloc(2 * nb * sizeof(double));
    for (size_t i = 0; i < n; ++i) {
        row_acc(row_ptr, col_idx, values, alpha, beta, nb, X, i, acc);
        for (size_t j = 0; j < nb; ++j) { /* y = 2*acc - z  (kernels.hpp:124) */
            double zr = Z[2 * (i * nb + j)], zi = Z[2 * (i * nb + j) + 1];
            Y[2 * (i * nb + j)] = 2.0 * acc[2 * j] - zr;
            Y[2 * (i * nb + j) + 1] = 2.0 * acc[2 * j + 1] - zi;
        }
    }
    free(acc);
    return 0;
}

int or_cheb_init(size_t n, const uint64_t* row_ptr, const int32_t* col_idx, const double* values, double alpha,
                 double beta, size_t nb, double* X, double* U, double* W, double g0c0, double g1c1, double g2c2) {
    if (or_spmmv_shifted(n, row_ptr, col_idx, values, alpha, beta, nb, X, U)) return 1;
    if (or_spmmv_shifted_two_minus(n, row_ptr, col_idx, values, alpha, beta, nb, U, W, X)) return 1;
    for (size_t i = 0; i < 2 * n * nb; ++i) /* kernels.hpp:144-145, scalar*complex componentwise */
        X[i] = g0c0 * X[i] + g1c1 * U[i] + g2c2 * W[i];
    return 0;
}

/* kernels.hpp:71-77 */
static void tree_reduce(double* part, size_t len, size_t width) {
    for (size_t stride = 1; stride < len; stride *= 2)
        for (size_t c = 0; c + stride < len; c += 2 * stride)
            for (size_t j = 0; j < width; ++j) part[c * width + j] += part[(c + stride) * width + j];
}

int or_chebfd_op(size_t n, const uint64_t* row_ptr, const int32_t* col_idx, const double* values, double alpha,
                 double beta, size_t nb, const double* U, double* W, double* X, double gc, double* eta, double* mu) {
    if (U == W) return 1;
    size_t nc = nchunks_for(n);
    double* ep = (double*)calloc(nc * 2 * nb, sizeof(double));
    double* mp = (double*)calloc(nc * 2 * nb, sizeof(double));
    double* acc = (double*)malloc(2 * nb * sizeof(double));
    for (size_t c = 0; c < nc; ++c) {
        size_t lo = n * c / nc, hi = n * (c + 1) / nc;
        double* e = ep + c * 2 * nb;
        double* m = mp + c * 2 * nb;
        for (size_t i = lo; i < hi; ++i) {
            row_acc(row_ptr, col_idx, values, alpha, beta, nb, U, i, acc);
            for (size_t j = 0; j < nb; ++j) { /* kernels.hpp:187-194 */
                size_t o = 2 * (i * nb + j);
                double ur = U[o], ui = U[o + 1];
                double wr = 2.0 * acc[2 * j] - W[o];
                double wi = 2.0 * acc[2 * j + 1] - W[o + 1];
                /* conj(w)*u = (wr*ur - (-wi)*ui, wr*ui + (-wi)*ur) */
                e[2 * j] += wr * ur - (-wi) * ui;
                e[2 * j + 1] += wr * ui + (-wi) * ur;
                m[2 * j] += ur * ur - (-ui) * ui;
                m[2 * j + 1] += ur * ui + (-ui) * ur;
                X[o] += gc * wr;
                X[o + 1] += gc * wi;
                W[o] = wr;
                W[o + 1] = wi;
            }
        }
    }
    tree_reduce(ep, nc, 2 * nb);
    tree_reduce(mp, nc, 2 * nb);
    for (size_t j = 0; j < 2 * nb; ++j) {
        eta[j] += ep[j];
        mu[j] += mp[j];
    }
    free(ep);
    free(mp);
    free(acc);
    return 0;
}

int or_chebfd_op_reference(size_t n, const uint64_t* row_ptr, const int32_t* col_idx, const double* values,
                           double alpha, double beta, size_t nb, const double* U, double* W, double* X, double gc,
                           double* eta, double* mu) {
    /* kernels.hpp:223: W <- 2(aH+b)U - W, evaluated per row (Z == Y allowed) */
    if (or_spmmv_shifted_two_minus(n, row_ptr, col_idx, values, alpha, beta, nb, U, W, W)) return 1;
    size_t nc = nchunks_for(n);
    double* ep = (double*)calloc(nc * 2 * nb, sizeof(double));
    double* mp = (double*)calloc(nc * 2 * nb, sizeof(double));
    for (size_t c = 0; c < nc; ++c) {
        size_t lo = n * c / nc, hi = n * (c + 1) / nc;
        for (size_t i = lo; i < hi; ++i)
            for (size_t j = 0; j < nb; ++j) {
                size_t o = 2 * (i * nb + j);
                double ur = U[o], ui = U[o + 1], wr = W[o], wi = W[o + 1];
                ep[c * 2 * nb + 2 * j] += wr * ur - (-wi) * ui;
                ep[c * 2 * nb + 2 * j + 1] += wr * ui + (-wi) * ur;
                mp[c * 2 * nb + 2 * j] += ur * ur - (-ui) * ui;
                mp[c * 2 * nb + 2 * j + 1] += ur * ui + (-ui) * ur;
            }
    }
    tree_reduce(ep, nc, 2 * nb);
    tree_reduce(mp, nc, 2 * nb);
    for (size_t j = 0; j < 2 * nb; ++j) {
        eta[j] += ep[j];
        mu[j] += mp[j];
    }
    for (size_t i = 0; i < 2 * n * nb; ++i) X[i] += gc * W[i];
    free(ep);
    free(mp);
    return 0;
}

/* filter.hpp:76-93 */
int or_apply_filter(size_t n, const uint64_t* row_ptr, const int32_t* col_idx, const double* values, size_t ns,
                    size_t nb, double* X, size_t np, const double* c, const double* g, double alpha, double beta,
                    double* eta, double* mu) {
    if (np < 2 || nb == 0 || ns % nb != 0) return 1;
    size_t rows = np - 2;
    memset(eta, 0, rows * ns * 2 * sizeof(double));
    memset(mu, 0, rows * ns * 2 * sizeof(double));
    double* U = (double*)malloc(2 * n * nb * sizeof(double));
    double* W = (double*)malloc(2 * n * nb * sizeof(double));
    for (size_t b = 0; b < ns / nb; ++b) {
        double* Xb = X + 2 * b * n * nb;
        memset(U, 0, 2 * n * nb * sizeof(double));
        memset(W, 0, 2 * n * nb * sizeof(double));
        or_cheb_init(n, row_ptr, col_idx, values, alpha, beta, nb, Xb, U, W, g[0] * c[0], g[1] * c[1], g[2] * c[2]);
        for (size_t p = 3; p <= np; ++p) {
            double* t = U; /* swap_blocks(W, U) */
            U = W;
            W = t;
            or_chebfd_op(n, row_ptr, col_idx, values, alpha, beta, nb, U, W, Xb, g[p] * c[p],
                         eta + 2 * ((p - 3) * ns + b * nb), mu + 2 * ((p - 3) * ns + b * nb));
        }
    }
    free(U);
    free(W);
    return 0;
}

/* partition.hpp:28-60 */
int or_partition_rows(size_t n, const uint64_t* row_ptr, const int32_t* col_idx, size_t workers, uint64_t* ranges,
                      uint64_t* halo, size_t* halo_len) {
    if (workers < 1) return 1;
    size_t granule = (n % 4 == 0) ? 4 : 1;
    size_t units = n / granule;
    if (workers > units) return 1;
    uint64_t* rg = (uint64_t*)malloc(2 * workers * sizeof(uint64_t));
    for (size_t w = 0; w < workers; ++w) {
        rg[2 * w] = units * w / workers * granule;
        rg[2 * w + 1] = units * (w + 1) / workers * granule;
    }
    if (ranges) memcpy(ranges, rg, 2 * workers * sizeof(uint64_t));
    unsigned char* mark = (unsigned char*)malloc(n);
    size_t len = 0;
    for (size_t w = 0; w < workers; ++w) {
        uint64_t lo = rg[2 * w], hi = rg[2 * w + 1];
        memset(mark, 0, n);
        for (uint64_t i = lo; i < hi; ++i)
            for (uint64_t k = row_ptr[i]; k < row_ptr[i + 1]; ++k) {
                uint64_t c = (uint64_t)col_idx[k];
                if (c < lo || c >= hi) mark[c] = 1;
            }
        /* std::set iteration is ascending; owners are monotone in the row index */
        size_t v = 0, cur_v = (size_t)-1, rec = 0;
        for (size_t c = 0; c < n; ++c) {
            if (!mark[c]) continue;
            while (!(c >= rg[2 * v] && c < rg[2 * v + 1])) ++v;
            if (v != cur_v) { /* new (w, v, count) record */
                cur_v = v;
                rec = len;
                if (halo) {
                    halo[len] = w;
                    halo[len + 1] = v;
                    halo[len + 2] = 0;
                }
                len += 3;
            }
            if (halo) {
                halo[len] = c;
                halo[rec + 2]++;
            }
            ++len;
        }
    }
    *halo_len = len;
    free(mark);
    free(rg);
    return 0;
}

/* ---------------------------------------------- SELL-C-sigma / B4 perm --- */
/* No reference counterpart (the reference is CRS only).  This is
 * the checker's independent restatement of the product's block-row
 * permutation: block-row b = rows 4b..4b+3; its length is the number of
 * distinct block columns col/4 over its rows; block-rows are taken in `order`
 * (NULL = natural), stable-sorted by descending length inside windows of
 * sigma block-rows, padded with -1 to a multiple of C. */
int or_sell_permutation(size_t n, const uint64_t* row_ptr, const int32_t* col_idx, const int32_t* order, int C,
                        int sigma, int32_t* perm_out, size_t* nslots) {
    if (C <= 0 || C % 4 != 0 || C > 64 || sigma <= 0 || sigma % C != 0) return 1;
    size_t nbr = (n + 3) / 4;
    size_t nch = (nbr + (size_t)C - 1) / (size_t)C;
    *nslots = nch * (size_t)C;
    if (!perm_out) return 0;
    int* len = (int*)malloc(nbr * sizeof(int));
    int32_t* bc = (int32_t*)malloc(64 * sizeof(int32_t) + 1);
    for (size_t b = 0; b < nbr; ++b) {
        /* collect block columns of the (up to) 4 rows, count distinct */
        size_t r0 = 4 * b, r1 = r0 + 4 < n ? r0 + 4 : n, tot = 0;
        for (size_t r = r0; r < r1; ++r) tot += row_ptr[r + 1] - row_ptr[r];
        int32_t* all = (int32_t*)malloc((tot ? tot : 1) * sizeof(int32_t));
        size_t q = 0;
        for (size_t r = r0; r < r1; ++r)
            for (uint64_t k = row_ptr[r]; k < row_ptr[r + 1]; ++k) all[q++] = col_idx[k] / 4;
        /* insertion sort + unique */
        for (size_t i = 1; i < q; ++i)
            for (size_t j = i; j > 0 && all[j] < all[j - 1]; --j) {
                int32_t t = all[j];
                all[j] = all[j - 1];
                all[j - 1] = t;
            }
        int d = 0;
        for (size_t i = 0; i < q; ++i)
            if (i == 0 || all[i] != all[i - 1]) ++d;
        len[b] = d;
        free(all);
    }
    free(bc);
    for (size_t i = 0; i < nbr; ++i) perm_out[i] = order ? order[i] : (int32_t)i;
    for (size_t w0 = 0; w0 < nbr; w0 += (size_t)sigma) {
        size_t w1 = w0 + (size_t)sigma < nbr ? w0 + (size_t)sigma : nbr;
        /* stable insertion sort, descending length */
        for (size_t i = w0 + 1; i < w1; ++i)
            for (size_t j = i; j > w0 && len[perm_out[j]] > len[perm_out[j - 1]]; --j) {
                int32_t t = perm_out[j];
                perm_out[j] = perm_out[j - 1];
                perm_out[j - 1] = t;
            }
    }
    for (size_t i = nbr; i < *nslots; ++i) perm_out[i] = -1;
    free(len);
    return 0;
}
