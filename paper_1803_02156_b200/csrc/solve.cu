// Device half of chebfd_solve (reference filter.hpp:98-320): the restarted
// filter loop apply_filter -> SVQB -> Rayleigh-Ritz, with
//   * gram_kernel    S = A^H B over n rows (tall-skinny, 32x32 output tiles,
//                    row-split partials summed in a fixed order -> the Gram
//                    matrices are bit-reproducible run to run);
//   * rotate_kernel  Y = A T (T small, k x m, staged in shared memory);
//   * resid_kernel   ||H y_r - theta_r y_r||^2 and ||y_r||^2 per column;
// and the small k x k eigenproblems solved on the host by the Jacobi
// restatement in host.cpp.  Block vectors stay in the reference's panel layout
// (block_vector.hpp:49-52): element (i, j) at panel j / nb, offset i*nb + j%nb.
// These kernels are FP64 FMA loops; at the configurations of BASELINE.json the
// projections cost well under 1% of the filter.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "device.hpp"

namespace cfb {

constexpr int kMaxPanels = 64;

struct PanelSet {
    double2* p[kMaxPanels];
    int nb = 0;     // panel width (row stride)
    int ncols = 0;  // valid columns
};

__device__ __forceinline__ double2* pelem(const PanelSet& s, long long i, int j) {
    return s.p[j / s.nb] + i * s.nb + (j % s.nb);
}

// acc += conj(a) * b
__device__ __forceinline__ void cmac_conj(double2& acc, double2 a, double2 b) {
    acc.x = fma(a.x, b.x, acc.x);
    acc.x = fma(a.y, b.y, acc.x);
    acc.y = fma(a.x, b.y, acc.y);
    acc.y = fma(-a.y, b.x, acc.y);
}
// acc += a * b
__device__ __forceinline__ void cmac(double2& acc, double2 a, double2 b) {
    acc.x = fma(a.x, b.x, acc.x);
    acc.x = fma(-a.y, b.y, acc.x);
    acc.y = fma(a.x, b.y, acc.y);
    acc.y = fma(a.y, b.x, acc.y);
}

// S tile (tj, tl) partial over the row range of split blockIdx.y.
__global__ void __launch_bounds__(256) gram_kernel(const PanelSet A, const PanelSet B, long long n, int ntj,
                                                   double2* __restrict__ part) {
    __shared__ double2 As[32][32], Bs[32][32];
    const int tile = blockIdx.x, tj = tile % ntj, tl = tile / ntj;
    const long long r0 = n * blockIdx.y / gridDim.y, r1 = n * (blockIdx.y + 1) / gridDim.y;
    const int t = threadIdx.x, jj = (t & 15) * 2, ll = (t >> 4) * 2;
    double2 acc[2][2];
#pragma unroll
    for (int x = 0; x < 2; ++x)
#pragma unroll
        for (int y = 0; y < 2; ++y) acc[x][y] = make_double2(0.0, 0.0);
    for (long long base = r0; base < r1; base += 32) {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int e = t + 256 * q, r = e >> 5, c = e & 31;
            const long long i = base + r;
            const int ja = tj * 32 + c, jb = tl * 32 + c;
            As[r][c] = (i < r1 && ja < A.ncols) ? *pelem(A, i, ja) : make_double2(0.0, 0.0);
            Bs[r][c] = (i < r1 && jb < B.ncols) ? *pelem(B, i, jb) : make_double2(0.0, 0.0);
        }
        __syncthreads();
#pragma unroll 8
        for (int r = 0; r < 32; ++r) {
            const double2 a0 = As[r][jj], a1 = As[r][jj + 1], b0 = Bs[r][ll], b1 = Bs[r][ll + 1];
            cmac_conj(acc[0][0], a0, b0);
            cmac_conj(acc[0][1], a0, b1);
            cmac_conj(acc[1][0], a1, b0);
            cmac_conj(acc[1][1], a1, b1);
        }
        __syncthreads();
    }
    double2* out = part + (static_cast<size_t>(blockIdx.y) * gridDim.x + tile) * 1024;
#pragma unroll
    for (int x = 0; x < 2; ++x)
#pragma unroll
        for (int y = 0; y < 2; ++y) out[(jj + x) * 32 + ll + y] = acc[x][y];
}

__global__ void gram_reduce(const double2* __restrict__ part, int splits, int ntiles, int ntj, int ka, int kb,
                            double2* __restrict__ S) {
    const long long idx = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (idx >= static_cast<long long>(ntiles) * 1024) return;
    const int tile = static_cast<int>(idx / 1024), loc = static_cast<int>(idx % 1024);
    const int j = (tile % ntj) * 32 + loc / 32, l = (tile / ntj) * 32 + loc % 32;
    if (j >= ka || l >= kb) return;
    double2 s = make_double2(0.0, 0.0);
    for (int q = 0; q < splits; ++q) {
        const double2 v = part[(static_cast<size_t>(q) * ntiles + tile) * 1024 + loc];
        s.x += v.x;
        s.y += v.y;
    }
    S[static_cast<size_t>(j) * kb + l] = s;
}

// Y[:, c0:c0+32] = A T[:, c0:c0+32]; warp w of the CTA takes rows in pairs.
__global__ void __launch_bounds__(256) rotate_kernel(const PanelSet A, const double2* __restrict__ T, int m,
                                                     const PanelSet Y, long long n) {
    extern __shared__ double2 Ts[];  // [k][32]
    const int k = A.ncols, c0 = blockIdx.x * 32, t = threadIdx.x, lane = t & 31, w = t >> 5;
    for (int e = t; e < k * 32; e += blockDim.x) {
        const int j = e >> 5, c = e & 31;
        Ts[e] = (c0 + c < m) ? T[static_cast<size_t>(j) * m + c0 + c] : make_double2(0.0, 0.0);
    }
    __syncthreads();
    const int col = c0 + lane;
    const int npan = (k + A.nb - 1) / A.nb;
    for (long long i0 = (static_cast<long long>(blockIdx.y) * 8 + w) * 2; i0 < n;
         i0 += static_cast<long long>(gridDim.y) * 16) {
        const long long i1 = (i0 + 1 < n) ? i0 + 1 : i0;
        double2 acc0 = make_double2(0.0, 0.0), acc1 = make_double2(0.0, 0.0);
        for (int pb = 0; pb < npan; ++pb) {
            const double2* a0p = A.p[pb] + i0 * A.nb;
            const double2* a1p = A.p[pb] + i1 * A.nb;
            const int jw = min(A.nb, k - pb * A.nb);
            for (int jj = 0; jj < jw; ++jj) {
                const double2 tv = Ts[(pb * A.nb + jj) * 32 + lane];
                cmac(acc0, __ldg(a0p + jj), tv);
                cmac(acc1, __ldg(a1p + jj), tv);
            }
        }
        if (col < m) {
            *pelem(Y, i0, col) = acc0;
            if (i0 + 1 < n) *pelem(Y, i0 + 1, col) = acc1;
        }
    }
}

// Per-column residual sums over the row range of blockIdx.y.
__global__ void __launch_bounds__(256) resid_kernel(const PanelSet Y, const PanelSet HY,
                                                    const double* __restrict__ theta, long long n, int kpad,
                                                    double* __restrict__ part) {
    __shared__ double red[8][32][2];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, col = blockIdx.x * 32 + lane;
    const long long r0 = n * blockIdx.y / gridDim.y, r1 = n * (blockIdx.y + 1) / gridDim.y;
    double num = 0.0, den = 0.0;
    if (col < Y.ncols) {
        const double th = theta[col];
        for (long long i = r0 + w; i < r1; i += 8) {
            const double2 y = *pelem(Y, i, col), hy = *pelem(HY, i, col);
            const double dx = hy.x - th * y.x, dy = hy.y - th * y.y;
            num = fma(dx, dx, fma(dy, dy, num));
            den = fma(y.x, y.x, fma(y.y, y.y, den));
        }
    }
    red[w][lane][0] = num;
    red[w][lane][1] = den;
    __syncthreads();
    if (w == 0) {
        double a = 0.0, b = 0.0;
        for (int q = 0; q < 8; ++q) {
            a += red[q][lane][0];
            b += red[q][lane][1];
        }
        double* o = part + (static_cast<size_t>(blockIdx.y) * kpad + col) * 2;
        o[0] = a;
        o[1] = b;
    }
}

__global__ void resid_reduce(const double* __restrict__ part, int splits, int k, int kpad, double* __restrict__ out) {
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= k) return;
    double a = 0.0, b = 0.0;
    for (int q = 0; q < splits; ++q) {
        a += part[(static_cast<size_t>(q) * kpad + c) * 2];
        b += part[(static_cast<size_t>(q) * kpad + c) * 2 + 1];
    }
    out[2 * c] = a;
    out[2 * c + 1] = b;
}

// dst columns [j0, j0 + w) <- src (n x w row-major)
__global__ void cols_from_rowmajor(const double2* __restrict__ src, int w, const PanelSet dst, int j0, long long n) {
    const long long e = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (e >= n * w) return;
    const long long i = e / w;
    const int c = static_cast<int>(e % w);
    *pelem(dst, i, j0 + c) = src[e];
}

// dst (n x w row-major) <- src columns map[0..w)
__global__ void cols_to_rowmajor(const PanelSet src, const int* __restrict__ map, int w, double2* __restrict__ dst,
                                 long long n) {
    const long long e = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (e >= n * w) return;
    const long long i = e / w;
    const int c = static_cast<int>(e % w);
    dst[e] = *pelem(src, i, map[c]);
}

// InitSeededRandom (block_vector.hpp:17-35, 68-73) on the device: the same
// splitmix64 hashes, Box-Muller with the device libm (log/cos/sin within 1-2
// ulp of glibc), for block vectors too large to generate on the host.
__device__ __forceinline__ uint64_t splitmix64_d(uint64_t x) {
    x += 0x9e3779b97f4a7c15ULL;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
    return x ^ (x >> 31);
}

__global__ void random_fill_kernel(const PanelSet Xs, long long n, int j0, int ns, uint64_t seed, uint64_t row_offset) {
    const long long w = ns - j0;
    const uint64_t hs = splitmix64_d(seed);
    for (long long e = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; e < n * w;
         e += static_cast<long long>(gridDim.x) * blockDim.x) {
        const long long i = e / w;
        const int j = j0 + static_cast<int>(e % w);
        const uint64_t h = splitmix64_d(hs ^ splitmix64_d((row_offset + i) * 0xd1342543de82ef95ULL + j));
        const uint64_t h2 = splitmix64_d(h);
        const double u = (static_cast<double>(h >> 11) + 1.0) * 0x1.0p-53;
        const double v = static_cast<double>(h2 >> 11) * 0x1.0p-53;
        const double r = sqrt(-log(u));
        double sn, cs;
        sincos(6.283185307179586477 * v, &sn, &cs);
        *pelem(Xs, i, j) = make_double2(r * cs, r * sn);
    }
}

// ============================================================ host side ===
namespace {

int sm_count(int dev) {
    int v = 0;
    ck(cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev), "cudaDeviceGetAttribute");
    return v;
}

// Owned device buffer.
struct DevBuf {
    void* p = nullptr;
    size_t bytes = 0;
    DevBuf() = default;
    explicit DevBuf(size_t b) : bytes(b) { ck(cudaMalloc(&p, b ? b : 16), "cudaMalloc"); }
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    DevBuf(DevBuf&& o) noexcept : p(o.p), bytes(o.bytes) { o.p = nullptr; }
    DevBuf& operator=(DevBuf&& o) noexcept {
        std::swap(p, o.p);
        std::swap(bytes, o.bytes);
        return *this;
    }
    ~DevBuf() {
        if (p) cudaFree(p);
    }
    template <class T>
    T* as() const {
        return static_cast<T*>(p);
    }
};

// Grow-only scratch buffers of the projection kernels, per device and host
// thread: the solver's Gram / rotation / residual steps run every restart and
// would otherwise pay a cudaMalloc + cudaFree (an implicit device sync) each.
enum WsSlot { kWsGramPart, kWsGramOut, kWsRotT, kWsResTheta, kWsResPart, kWsResOut, kWsRandom, kWsColMap, kWsSlots };
void* workspace(int dev, int slot, size_t bytes) {
    struct Ws {
        void* p[kWsSlots] = {};
        size_t n[kWsSlots] = {};
        ~Ws() {
            for (void* q : p)
                if (q) cudaFree(q);
        }
    };
    thread_local std::vector<std::unique_ptr<Ws>> per_dev;
    if (static_cast<size_t>(dev) >= per_dev.size()) per_dev.resize(dev + 1);
    if (!per_dev[dev]) per_dev[dev] = std::make_unique<Ws>();
    Ws& w = *per_dev[dev];
    if (w.n[slot] < bytes) {
        if (w.p[slot]) ck(cudaFree(w.p[slot]), "cudaFree workspace");
        w.p[slot] = nullptr;
        w.n[slot] = 0;
        ck(cudaMalloc(&w.p[slot], bytes), "cudaMalloc workspace");
        w.n[slot] = bytes;
    }
    return w.p[slot];
}

// A panel-layout block vector in one allocation: panel b at base + b*n*nb.
struct Block {
    DevBuf buf;
    size_t n = 0, nb = 0, cap = 0;  // cap: allocated columns (multiple of nb)
    Block() = default;
    Block(size_t n_, size_t cap_, size_t nb_) : buf(n_ * cap_ * 16), n(n_), nb(nb_), cap(cap_) {}
    double2* panel(size_t b) const { return buf.as<double2>() + b * n * nb; }
    size_t panels() const { return cap / nb; }
    PanelSet set(size_t ncols) const {
        PanelSet s{};
        if (panels() > static_cast<size_t>(kMaxPanels)) throw std::invalid_argument("too many panels (n_s/n_b > 64)");
        for (size_t b = 0; b < panels(); ++b) s.p[b] = panel(b);
        s.nb = static_cast<int>(nb);
        s.ncols = static_cast<int>(ncols);
        return s;
    }
};

PanelSet panel_set(void* const* panels, size_t npanels, size_t nb, size_t ncols) {
    if (npanels > static_cast<size_t>(kMaxPanels)) throw std::invalid_argument("too many panels (n_s/n_b > 64)");
    if (nb == 0 || ncols > npanels * nb) throw std::invalid_argument("panel set: bad shape");
    PanelSet s{};
    for (size_t b = 0; b < npanels; ++b) s.p[b] = static_cast<double2*>(panels[b]);
    s.nb = static_cast<int>(nb);
    s.ncols = static_cast<int>(ncols);
    return s;
}

PanelSet single_panel(const void* p, size_t k) {
    PanelSet s{};
    s.p[0] = static_cast<double2*>(const_cast<void*>(p));
    s.nb = static_cast<int>(std::max<size_t>(k, 1));
    s.ncols = static_cast<int>(k);
    return s;
}

struct Ctx {
    int dev;
    cudaStream_t st;
    int sms;
};

// S = A^H B on the device (ka x kb row-major) into dS.
void gram_dev(const Ctx& c, const PanelSet& A, const PanelSet& B, size_t n, double2* dS) {
    const int ka = A.ncols, kb = B.ncols;
    if (ka == 0 || kb == 0) return;
    const int ntj = (ka + 31) / 32, ntl = (kb + 31) / 32, ntiles = ntj * ntl;
    int splits = static_cast<int>(std::min<size_t>(std::max<size_t>(n / 512, 1), std::max(1, 4 * c.sms / ntiles)));
    splits = std::max(1, std::min(splits, 1024));
    double2* part = static_cast<double2*>(workspace(c.dev, kWsGramPart, static_cast<size_t>(splits) * ntiles * 1024 * 16));
    gram_kernel<<<dim3(ntiles, splits), 256, 0, c.st>>>(A, B, static_cast<long long>(n), ntj, part);
    ck(cudaGetLastError(), "gram_kernel launch");
    const long long tot = static_cast<long long>(ntiles) * 1024;
    gram_reduce<<<static_cast<unsigned>((tot + 255) / 256), 256, 0, c.st>>>(part, splits, ntiles, ntj, ka, kb, dS);
    ck(cudaGetLastError(), "gram_reduce launch");
    ck(cudaStreamSynchronize(c.st), "gram sync");  // the partials buffer is reused by the next call
}

std::vector<double> gram_host(const Ctx& c, const PanelSet& A, const PanelSet& B, size_t n) {
    const size_t ka = A.ncols, kb = B.ncols;
    std::vector<double> S(2 * ka * kb, 0.0);
    if (!ka || !kb) return S;
    void* d = workspace(c.dev, kWsGramOut, ka * kb * 16);
    gram_dev(c, A, B, n, static_cast<double2*>(d));
    ck(cudaMemcpy(S.data(), d, ka * kb * 16, cudaMemcpyDeviceToHost), "download Gram");
    return S;
}

// Y = A T with T host k x m row-major complex.
void rotate_dev(const Ctx& c, const PanelSet& A, const std::vector<double>& T, size_t m, const PanelSet& Y,
                size_t n) {
    const size_t k = A.ncols;
    if (m == 0) return;
    const size_t smem = k * 32 * 16;
    if (smem > 200 * 1024) throw std::invalid_argument("rotation: block vector too wide (n_s > 400)");
    double2* dT = static_cast<double2*>(workspace(c.dev, kWsRotT, k * m * 16));
    ck(cudaMemcpyAsync(dT, T.data(), k * m * 16, cudaMemcpyHostToDevice, c.st), "upload T");
    ck(cudaFuncSetAttribute(rotate_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)),
       "cudaFuncSetAttribute");
    const int ntc = static_cast<int>((m + 31) / 32);
    const long long groups = (static_cast<long long>(n) + 15) / 16;
    const int gy = static_cast<int>(std::max<long long>(1, std::min<long long>(groups, 2LL * c.sms)));
    rotate_kernel<<<dim3(ntc, gy), 256, smem, c.st>>>(A, dT, static_cast<int>(m), Y,
                                                       static_cast<long long>(n));
    ck(cudaGetLastError(), "rotate_kernel launch");
    ck(cudaStreamSynchronize(c.st), "rotate sync");
}

double max_gram_defect(const Ctx& c, const PanelSet& Q, size_t n) {
    std::vector<double> G = gram_host(c, Q, Q, n);
    const size_t k = Q.ncols;
    double d = 0.0;
    for (size_t i = 0; i < k; ++i)
        for (size_t j = 0; j < k; ++j) {
            const double er = G[2 * (i * k + j)] - (i == j ? 1.0 : 0.0), ei = G[2 * (i * k + j) + 1];
            d = std::max(d, std::hypot(er, ei));
        }
    return d;
}

// Hermitian part as the reference builds it: upper triangle computed, lower mirrored.
void mirror_upper(std::vector<double>& S, size_t k) {
    for (size_t j = 0; j < k; ++j)
        for (size_t l = 0; l < j; ++l) {
            S[2 * (j * k + l)] = S[2 * (l * k + j)];
            S[2 * (j * k + l) + 1] = -S[2 * (l * k + j) + 1];
        }
}

void zero_set(const Ctx& c, const Block& b) {
    ck(cudaMemsetAsync(b.buf.p, 0, b.n * b.cap * 16, c.st), "memset");
}

// One SVQB pass (filter.hpp:113-136): Q = X V_keep diag(1/sqrt(lambda_keep)).
size_t svqb_pass(const Ctx& c, const PanelSet& X, size_t n, double drop_tol, const Block& Qb) {
    const size_t k = X.ncols;
    std::vector<double> S = gram_host(c, X, X, n);
    mirror_upper(S, k);
    std::vector<double> vals, vecs;
    jacobi_hermitian(k, std::move(S), 1e-12, 64, vals, vecs);
    const double lmax = vals.empty() ? 0.0 : vals.back();
    if (!(lmax > 0.0)) throw std::runtime_error("svqb: all columns numerically zero");
    std::vector<size_t> keep;
    for (size_t j = 0; j < vals.size(); ++j)
        if (vals[j] > drop_tol * lmax) keep.push_back(j);
    const size_t rank = keep.size();
    if (rank == 0) throw std::runtime_error("svqb: empty basis after dropping");
    std::vector<double> T(2 * k * rank);
    for (size_t r = 0; r < rank; ++r) {
        const double s = 1.0 / std::sqrt(vals[keep[r]]);
        for (size_t j = 0; j < k; ++j) {
            T[2 * (j * rank + r)] = vecs[2 * (j * k + keep[r])] * s;
            T[2 * (j * rank + r) + 1] = vecs[2 * (j * k + keep[r]) + 1] * s;
        }
    }
    zero_set(c, Qb);
    rotate_dev(c, X, T, rank, Qb.set(rank), n);
    return rank;
}

// orthogonalize_svqb (filter.hpp:139-150): result in qa (qb is scratch).
size_t svqb(const Ctx& c, const PanelSet& X, size_t n, double drop_tol, Block& qa, Block& qb) {
    size_t rank = svqb_pass(c, X, n, drop_tol, qa);
    for (int pass = 0; pass < 3 && max_gram_defect(c, qa.set(rank), n) > 1e-10; ++pass) {
        rank = svqb_pass(c, qa.set(rank), n, drop_tol, qb);
        std::swap(qa, qb);
    }
    return rank;
}

// H applied panel by panel: Y = H X over the first k columns of a panel set.
void spmmv_set(const Ctx& c, cf_matrix m, const PanelSet& X, const PanelSet& Y) {
    const int npan = (X.ncols + X.nb - 1) / X.nb;
    for (int b = 0; b < npan; ++b) {
        const size_t w = static_cast<size_t>(std::min(X.nb, X.ncols - b * X.nb));
        spmmv_dev(m, 1.0, 0.0, X.p[b], Y.p[b], static_cast<size_t>(X.nb), w, c.st);
    }
}

// Per column: (||hy - theta y||^2, ||y||^2) over n rows, fixed-order two-level sums.
std::vector<double> residual_sums(const Ctx& c, const PanelSet& Y, const PanelSet& HY, const std::vector<double>& theta,
                                  size_t n) {
    const size_t k = Y.ncols;
    std::vector<double> nd(2 * k, 0.0);
    if (k == 0) return nd;
    const int kpad = static_cast<int>((k + 31) / 32 * 32);
    int splits = static_cast<int>(std::min<size_t>(std::max<size_t>(n / 2048, 1), static_cast<size_t>(2 * c.sms)));
    double* dth = static_cast<double*>(workspace(c.dev, kWsResTheta, k * 8));
    double* part = static_cast<double*>(workspace(c.dev, kWsResPart, static_cast<size_t>(splits) * kpad * 16));
    double* out = static_cast<double*>(workspace(c.dev, kWsResOut, k * 16));
    ck(cudaMemcpyAsync(dth, theta.data(), k * 8, cudaMemcpyHostToDevice, c.st), "upload theta");
    resid_kernel<<<dim3(kpad / 32, splits), 256, 0, c.st>>>(Y, HY, dth, static_cast<long long>(n), kpad, part);
    ck(cudaGetLastError(), "resid_kernel launch");
    resid_reduce<<<(static_cast<unsigned>(k) + 127) / 128, 128, 0, c.st>>>(part, splits, static_cast<int>(k), kpad, out);
    ck(cudaGetLastError(), "resid_reduce launch");
    ck(cudaMemcpyAsync(nd.data(), out, k * 16, cudaMemcpyDeviceToHost, c.st), "download residuals");
    ck(cudaStreamSynchronize(c.st), "residual sync");
    return nd;
}

struct RR {
    std::vector<double> theta, residuals;
};

// rayleigh_ritz (filter.hpp:170-211): Y = Q V in Yset, HY scratch in HYset.
RR rayleigh_ritz(const Ctx& c, cf_matrix m, const PanelSet& Q, const PanelSet& HQ, const PanelSet& Yset,
                 const PanelSet& HYset, size_t n) {
    if (max_gram_defect(c, Q, n) > 1e-8) throw std::invalid_argument("rayleigh_ritz: basis not orthonormal");
    const size_t k = Q.ncols;
    spmmv_set(c, m, Q, HQ);
    std::vector<double> S = gram_host(c, Q, HQ, n);
    mirror_upper(S, k);
    std::vector<double> vals, vecs;
    jacobi_hermitian(k, std::move(S), 1e-12, 64, vals, vecs);
    RR rr;
    rr.theta = vals;
    rotate_dev(c, Q, vecs, k, Yset, n);
    spmmv_set(c, m, Yset, HYset);
    // residuals ||H y - theta y|| / ||y||
    std::vector<double> nd = residual_sums(c, Yset, HYset, vals, n);
    rr.residuals.resize(k);
    for (size_t r = 0; r < k; ++r) rr.residuals[r] = std::sqrt(nd[2 * r]) / std::sqrt(nd[2 * r + 1]);
    return rr;
}

// Block vectors above 2^27 elements (2 GB) are generated on the device; smaller
// ones on the host, bit-identical to the reference's InitSeededRandom.
bool device_rng(size_t n, size_t ns) { return n * ns > (size_t{1} << 27); }

// Columns [j0, j1) of InitSeededRandom{seed} (block_vector.hpp:68-73) into dst.
void random_columns(const Ctx& c, size_t n, size_t j0, size_t j1, uint64_t seed, const PanelSet& dst) {
    if (j1 <= j0) return;
    if (device_rng(n, j1 - j0) && j1 == static_cast<size_t>(dst.ncols)) {
        random_fill_kernel<<<4 * c.sms, 256, 0, c.st>>>(dst, static_cast<long long>(n), static_cast<int>(j0),
                                                         static_cast<int>(j1), seed, 0);
        ck(cudaGetLastError(), "random_fill_kernel launch");
        ck(cudaStreamSynchronize(c.st), "random fill sync");
        return;
    }
    const size_t w = j1 - j0;
    std::vector<double> host(2 * n * w);
    fill_random_columns(n, j0, j1, seed, host.data());
    double2* d = static_cast<double2*>(workspace(c.dev, kWsRandom, n * w * 16));
    ck(cudaMemcpyAsync(d, host.data(), n * w * 16, cudaMemcpyHostToDevice, c.st), "upload random columns");
    const long long tot = static_cast<long long>(n) * w;
    cols_from_rowmajor<<<static_cast<unsigned>((tot + 255) / 256), 256, 0, c.st>>>(
        d, static_cast<int>(w), dst, static_cast<int>(j0), static_cast<long long>(n));
    ck(cudaGetLastError(), "cols_from_rowmajor launch");
    ck(cudaStreamSynchronize(c.st), "random columns sync");
}

void gather_columns(const Ctx& c, const PanelSet& src, const std::vector<int>& cols, size_t n, void* dst) {
    if (cols.empty() || !dst) return;
    int* dm = static_cast<int*>(workspace(c.dev, kWsColMap, cols.size() * 4));
    ck(cudaMemcpyAsync(dm, cols.data(), cols.size() * 4, cudaMemcpyHostToDevice, c.st), "upload column map");
    const long long tot = static_cast<long long>(n) * cols.size();
    cols_to_rowmajor<<<static_cast<unsigned>((tot + 255) / 256), 256, 0, c.st>>>(
        src, dm, static_cast<int>(cols.size()), static_cast<double2*>(dst), static_cast<long long>(n));
    ck(cudaGetLastError(), "cols_to_rowmajor launch");
    ck(cudaStreamSynchronize(c.st), "gather sync");
}

void solve(cf_matrix m, double wlo, double whi, const cf_solve_options& o, cf_solve_result& res, cudaStream_t st) {
    if (m->ncols != m->n) throw std::invalid_argument("chebfd_solve: needs the whole matrix (no halo columns)");
    if (o.n_b == 0 || o.n_s == 0 || o.n_s % o.n_b != 0) throw std::invalid_argument("n_b must divide n_s");
    const double blo = o.has_bounds ? o.bound_lo : m->gersh_lo, bhi = o.has_bounds ? o.bound_hi : m->gersh_hi;
    if (wlo < blo || whi > bhi) throw std::invalid_argument("search window outside spectral bounds");
    double alpha = 0, beta = 0;
    check(cf_spectral_map(blo, bhi, o.margin, &alpha, &beta));
    std::vector<double> cc(o.n_p + 1), gg(o.n_p + 1);
    check(cf_filter_coefficients(wlo, whi, alpha, beta, o.n_p, o.damping, cc.data(), gg.data()));
    if (o.n_p < 2) throw std::invalid_argument("apply_filter: coefficients cover degrees < 2");

    DeviceGuard dg(m->device);
    const Ctx c{m->device, st, sm_count(m->device)};
    // The search block is the library's own, so its panel width is free: results do
    // not depend on n_b beyond rounding (block-width invariance, test_filter.cpp:259-279),
    // and n_s / 32 panels of 32 columns read the matrix once per 32 columns and run the
    // chunk-staged kernel (the reference default n_s = 32, n_b = 8: one sweep instead of
    // four per degree).  CHEBFD_SOLVE_WIDE=0 keeps the caller's n_b.
    static const bool wide = [] {
        const char* e = std::getenv("CHEBFD_SOLVE_WIDE");
        return !(e && std::atoi(e) == 0);
    }();
    const size_t n = m->n, ns = o.n_s, nb = (wide && o.n_b < 32 && ns % 32 == 0) ? 32 : o.n_b;
    Block X(n, ns, nb), Qa(n, ns, nb), Qb(n, ns, nb), Yb(n, ns, nb);
    if (device_rng(n, ns)) {
        random_columns(c, n, 0, ns, o.seed, X.set(ns));
    } else {
        std::vector<double> host(2 * n * ns);
        check(cf_blockvec_random(n, ns, nb, o.seed, 0, host.data()));
        ck(cudaMemcpyAsync(X.buf.p, host.data(), n * ns * 16, cudaMemcpyHostToDevice, st), "upload X0");
        ck(cudaStreamSynchronize(st), "upload sync");
    }
    const size_t mom = (o.n_p - 2) * ns;
    DevBuf deta(mom * 16), dmu(mom * 16);
    res.n_eig = res.n_pairs = res.iterations = 0;
    res.converged = 0;
    size_t empty_streak = 0;
    std::vector<double> pv, pr;
    std::vector<int> pf;
    auto record_pairs = [&](const RR& rr, double rtol) {
        pv = rr.theta;
        pr = rr.residuals;
        pf.assign(rr.theta.size(), 0);
        for (size_t r = 0; r < rr.theta.size(); ++r) {
            const bool inside = rr.theta[r] > wlo && rr.theta[r] < whi;
            const bool conv = inside && rr.residuals[r] <= rtol;
            pf[r] = (inside ? 1 : 0) | (conv ? 2 : 0);
        }
        res.n_pairs = pv.size();
        for (size_t r = 0; r < pv.size(); ++r) {
            if (res.pair_values) res.pair_values[r] = pv[r];
            if (res.pair_residuals) res.pair_residuals[r] = pr[r];
            if (res.pair_flags) res.pair_flags[r] = pf[r];
        }
    };
    // CHEBFD_TRACE=1: per-restart phase times on stderr (filter / SVQB / RR / restart fill)
    static const bool trace = [] {
        const char* e = std::getenv("CHEBFD_TRACE");
        return e && std::atoi(e) != 0;
    }();
    using clk = std::chrono::steady_clock;
    auto ms_since = [](clk::time_point t) { return std::chrono::duration<double, std::milli>(clk::now() - t).count(); };
    for (size_t restart = 1; restart <= o.max_restarts; ++restart) {
        res.iterations = restart;
        const auto t0 = clk::now();
        std::vector<double2*> panels(X.panels());
        for (size_t b = 0; b < panels.size(); ++b) panels[b] = X.panel(b);
        apply_filter_dev(m, panels.data(), panels.size(), nb, o.n_p, cc.data(), gg.data(), alpha, beta,
                         deta.as<double>(), dmu.as<double>(), st);
        if (res.eta)
            ck(cudaMemcpyAsync(res.eta + 2 * mom * (restart - 1), deta.p, mom * 16, cudaMemcpyDeviceToHost, st),
               "download eta");
        if (res.mu)
            ck(cudaMemcpyAsync(res.mu + 2 * mom * (restart - 1), dmu.p, mom * 16, cudaMemcpyDeviceToHost, st),
               "download mu");
        ck(cudaStreamSynchronize(st), "filter sync");
        const double t_filter = ms_since(t0);
        // SVQB into Qa (Qb scratch); X is free afterwards and holds HQ / HY
        const size_t rank = svqb(c, X.set(ns), n, o.drop_tol, Qa, Qb);
        const double t_svqb = ms_since(t0) - t_filter;
        RR rr = rayleigh_ritz(c, m, Qa.set(rank), X.set(rank), Yb.set(rank), Qb.set(rank), n);
        record_pairs(rr, o.res_tol);
        const double t_rr = ms_since(t0) - t_filter - t_svqb;
        if (res.phase_ms) {
            res.phase_ms[3 * (restart - 1) + 0] = t_filter;
            res.phase_ms[3 * (restart - 1) + 1] = t_svqb;
            res.phase_ms[3 * (restart - 1) + 2] = t_rr;
        }
        if (trace)
            std::fprintf(stderr, "chebfd_solve restart %zu: filter %.2f ms, svqb %.2f ms, rayleigh_ritz %.2f ms, rank %zu\n",
                         restart, t_filter, t_svqb, t_rr, rank);
        size_t inside = 0, conv_inside = 0;
        for (int f : pf) {
            inside += f & 1;
            conv_inside += (f >> 1) & 1;
        }
        const bool done = inside > 0 && conv_inside == inside;
        if (inside == 0 && ++empty_streak >= 2) {
            res.converged = 1;  // window verified empty
            return;
        }
        if (inside > 0) empty_streak = 0;
        if (done) {
            res.converged = 1;
            std::vector<int> sel;
            for (size_t r = 0; r < pf.size(); ++r)
                if (pf[r] & 2) sel.push_back(static_cast<int>(r));
            res.n_eig = sel.size();
            for (size_t q = 0; q < sel.size(); ++q) {
                if (res.eigenvalues) res.eigenvalues[q] = pv[sel[q]];
                if (res.residuals) res.residuals[q] = pr[sel[q]];
            }
            gather_columns(c, Yb.set(rank), sel, n, res.eigenvectors);
            return;
        }
        // restart basis: rotated Ritz basis, topped up with fresh random columns
        std::swap(X, Yb);
        random_columns(c, n, rank, ns, o.seed + restart, X.set(ns));
    }
    res.converged = 0;
    size_t q = 0;
    for (size_t r = 0; r < pf.size(); ++r)
        if (pf[r] & 2) {
            if (res.eigenvalues) res.eigenvalues[q] = pv[r];
            if (res.residuals) res.residuals[q] = pr[r];
            ++q;
        }
    res.n_eig = q;
}

}  // namespace
}  // namespace cfb

using namespace cfb;

extern "C" {

int cf_gram(size_t n, void* const* a_panels, size_t a_nb, size_t ka, void* const* b_panels, size_t b_nb, size_t kb,
            void* S, void* stream) {
    return guard([&] {
        int dev = 0;
        ck(cudaGetDevice(&dev), "cudaGetDevice");
        const Ctx c{dev, static_cast<cudaStream_t>(stream), sm_count(dev)};
        gram_dev(c, panel_set(a_panels, (ka + a_nb - 1) / std::max<size_t>(a_nb, 1), a_nb, ka),
                 panel_set(b_panels, (kb + b_nb - 1) / std::max<size_t>(b_nb, 1), b_nb, kb), n,
                 static_cast<double2*>(S));
    });
}

int cf_rotate(size_t n, void* const* a_panels, size_t a_nb, size_t k, const double* T, size_t m, void* const* y_panels,
              size_t y_nb, void* stream) {
    return guard([&] {
        int dev = 0;
        ck(cudaGetDevice(&dev), "cudaGetDevice");
        const Ctx c{dev, static_cast<cudaStream_t>(stream), sm_count(dev)};
        std::vector<double> t(T, T + 2 * k * m);
        rotate_dev(c, panel_set(a_panels, (k + a_nb - 1) / std::max<size_t>(a_nb, 1), a_nb, k), t, m,
                   panel_set(y_panels, (m + y_nb - 1) / std::max<size_t>(y_nb, 1), y_nb, m), n);
    });
}

int cf_residual_sums(size_t n, void* const* y_panels, size_t y_nb, void* const* hy_panels, size_t hy_nb, size_t k,
                     const double* theta, double* num_den, void* stream) {
    return guard([&] {
        int dev = 0;
        ck(cudaGetDevice(&dev), "cudaGetDevice");
        const Ctx c{dev, static_cast<cudaStream_t>(stream), sm_count(dev)};
        std::vector<double> th(theta, theta + k);
        std::vector<double> nd = residual_sums(c, panel_set(y_panels, (k + y_nb - 1) / std::max<size_t>(y_nb, 1), y_nb, k),
                                               panel_set(hy_panels, (k + hy_nb - 1) / std::max<size_t>(hy_nb, 1),
                                                         hy_nb, k),
                                               th, n);
        std::copy(nd.begin(), nd.end(), num_den);
    });
}

int cf_blockvec_random_device(size_t n, size_t ns, size_t nb, uint64_t seed, uint64_t row_offset, void* const* panels,
                              size_t j0, void* stream) {
    return guard([&] {
        if (nb == 0 || ns == 0 || ns % nb != 0) throw std::invalid_argument("n_b must divide n_s");
        if (j0 >= ns) return;
        int dev = 0;
        ck(cudaGetDevice(&dev), "cudaGetDevice");
        const PanelSet Xs = panel_set(panels, ns / nb, nb, ns);
        random_fill_kernel<<<4 * sm_count(dev), 256, 0, static_cast<cudaStream_t>(stream)>>>(
            Xs, static_cast<long long>(n), static_cast<int>(j0), static_cast<int>(ns), seed, row_offset);
        ck(cudaGetLastError(), "random_fill_kernel launch");
    });
}

int cf_orthogonalize_svqb(size_t n, void* const* panels, size_t npanels, size_t nb, double drop_tol, void* Q,
                          size_t* rank, void* stream) {
    return guard([&] {
        int dev = 0;
        ck(cudaGetDevice(&dev), "cudaGetDevice");
        const Ctx c{dev, static_cast<cudaStream_t>(stream), sm_count(dev)};
        const size_t ns = npanels * nb;
        Block qa(n, ns, nb), qb(n, ns, nb);
        const size_t r = svqb(c, panel_set(panels, npanels, nb, ns), n, drop_tol, qa, qb);
        // one n x r panel, as BlockVector(n, rank, rank) (filter.hpp:126)
        std::vector<int> all(r);
        for (size_t j = 0; j < r; ++j) all[j] = static_cast<int>(j);
        gather_columns(c, qa.set(r), all, n, Q);
        *rank = r;
    });
}

int cf_rayleigh_ritz(cf_matrix m, const void* Q, size_t k, double* theta, void* basis, double* residuals,
                     void* stream) {
    return guard([&] {
        if (!m) throw std::invalid_argument("null matrix");
        if (k == 0) throw std::invalid_argument("rayleigh_ritz: empty basis");
        DeviceGuard dg(m->device);
        const Ctx c{m->device, static_cast<cudaStream_t>(stream), sm_count(m->device)};
        const size_t n = m->n;
        Block hq(n, k, k), hy(n, k, k);
        RR rr = rayleigh_ritz(c, m, single_panel(Q, k), hq.set(k), single_panel(basis, k), hy.set(k), n);
        std::copy(rr.theta.begin(), rr.theta.end(), theta);
        std::copy(rr.residuals.begin(), rr.residuals.end(), residuals);
    });
}

int cf_chebfd_solve(cf_matrix m, double window_lo, double window_hi, const cf_solve_options* opt,
                    cf_solve_result* res, void* stream) {
    return guard([&] {
        if (!m || !opt || !res) throw std::invalid_argument("chebfd_solve: null argument");
        solve(m, window_lo, window_hi, *opt, *res, static_cast<cudaStream_t>(stream));
    });
}

}  // extern "C"

// ------------------------------------------------------------ STREAM ----
// stream_bench (perf_model.hpp:80-121) on the device: copy / scale / add /
// triad over double arrays in HBM, STREAM byte accounting (16 or 24 bytes per
// element, write-allocate not counted), best of the repetitions.
namespace cfb {
template <int KIND>
__global__ void __launch_bounds__(256) stream_kernel(long long n, double* __restrict__ a, double* __restrict__ b,
                                                     double* __restrict__ c, double s) {
    // n is even (the host rounds down); 16-byte accesses, each array touched only if the kind uses it
    const long long stride = static_cast<long long>(gridDim.x) * blockDim.x * 2;
    for (long long i = (static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x) * 2; i < n; i += stride) {
        if (KIND == 0) {
            *reinterpret_cast<double2*>(c + i) = *reinterpret_cast<const double2*>(a + i);
        } else if (KIND == 1) {
            const double2 z = *reinterpret_cast<const double2*>(c + i);
            *reinterpret_cast<double2*>(b + i) = make_double2(s * z.x, s * z.y);
        } else if (KIND == 2) {
            const double2 x = *reinterpret_cast<const double2*>(a + i), y = *reinterpret_cast<const double2*>(b + i);
            *reinterpret_cast<double2*>(c + i) = make_double2(x.x + y.x, x.y + y.y);
        } else {
            const double2 y = *reinterpret_cast<const double2*>(b + i), z = *reinterpret_cast<const double2*>(c + i);
            *reinterpret_cast<double2*>(a + i) = make_double2(y.x + s * z.x, y.y + s * z.y);
        }
    }
}
}  // namespace cfb

extern "C" int cf_stream_bench(int device, size_t elems, int kind, size_t reps, double* bytes_per_s) {
    using namespace cfb;
    return guard([&] {
        if (elems == 0 || reps == 0 || kind < 0 || kind > 3) throw std::invalid_argument("stream_bench inputs must be positive");
        DeviceGuard dg(device);
        DevBuf a(elems * 8), b(elems * 8), c(elems * 8);
        ck(cudaMemset(a.p, 0, elems * 8), "memset");
        ck(cudaMemset(b.p, 0, elems * 8), "memset");
        ck(cudaMemset(c.p, 0, elems * 8), "memset");
        cudaEvent_t e0, e1;
        ck(cudaEventCreate(&e0), "event");
        ck(cudaEventCreate(&e1), "event");
        const int grid = 4 * sm_count(device);
        const double per = (kind <= 1 ? 16.0 : 24.0) * static_cast<double>(elems & ~size_t{1});
        double best = 0.0;
        for (size_t r = 0; r <= reps; ++r) {  // r = 0 warms up
            ck(cudaEventRecord(e0), "record");
            const long long ne = static_cast<long long>(elems & ~size_t{1});
            switch (kind) {
                case 0: stream_kernel<0><<<grid, 256>>>(ne, a.as<double>(), b.as<double>(), c.as<double>(), 3.0); break;
                case 1: stream_kernel<1><<<grid, 256>>>(ne, a.as<double>(), b.as<double>(), c.as<double>(), 3.0); break;
                case 2: stream_kernel<2><<<grid, 256>>>(ne, a.as<double>(), b.as<double>(), c.as<double>(), 3.0); break;
                default: stream_kernel<3><<<grid, 256>>>(ne, a.as<double>(), b.as<double>(), c.as<double>(), 3.0); break;
            }
            ck(cudaGetLastError(), "stream_kernel launch");
            ck(cudaEventRecord(e1), "record");
            ck(cudaEventSynchronize(e1), "sync");
            float ms = 0.0f;
            ck(cudaEventElapsedTime(&ms, e0, e1), "elapsed");
            if (r > 0 && ms > 0) best = std::max(best, per / (ms * 1e-3));
        }
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
        *bytes_per_s = best;
    });
}
