// File formats of the reference, host side: Matrix Market coordinate complex
// (matrix_market.hpp:22-106) and the CFDB block-vector file
// (block_vector.hpp:155-229).  Outputs are byte-identical to the reference's
// writers; readers accept the same inputs and fail on the same lines.
#include <algorithm>
#include <charconv>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <mutex>
#include <numeric>
#include <string>
#include <unordered_map>

#include "common.hpp"

namespace cfb {
namespace {

struct MMError : std::runtime_error {
    MMError(const std::string& msg, std::size_t line)
        : std::runtime_error(msg + " (line " + std::to_string(line) + ")"), line(line) {}
    std::size_t line;
};

struct ParsedCrs {
    std::size_t n = 0;
    int symmetry = 0;  // 0 hermitian, 1 general (sparse_matrix.hpp Symmetry order)
    std::vector<uint64_t> rp;
    std::vector<int32_t> ci;
    std::vector<double> v;
};

thread_local std::unordered_map<std::string, ParsedCrs> g_mm_cache;
thread_local std::size_t g_mm_line = 0;

bool blank(const std::string& s) { return s.find_first_not_of(" \t\r") == std::string::npos; }

// Whitespace-separated token scanner over one line.
struct Tok {
    const char* p;
    const char* e;
    explicit Tok(const std::string& s) : p(s.data()), e(s.data() + s.size()) {}
    void skip() {
        while (p < e && (*p == ' ' || *p == '\t' || *p == '\r')) ++p;
    }
    bool word(std::string& out) {
        skip();
        const char* q = p;
        while (p < e && *p != ' ' && *p != '\t' && *p != '\r') ++p;
        out.assign(q, p);
        return p > q;
    }
    template <class T>
    bool num(T& out) {
        skip();
        if (p >= e) return false;
        if constexpr (std::is_floating_point_v<T>) {
            // the decimal forms istream >> double (libstdc++ num_get) accepts:
            // [sign] digits [. digits] [e [sign] digits]; no inf/nan/hex; overflow fails
            const char* q = p;
            if (q < e && (*q == '+' || *q == '-')) ++q;
            const char* d0 = q;
            while (q < e && *q >= '0' && *q <= '9') ++q;
            if (q < e && *q == '.') {
                ++q;
                while (q < e && *q >= '0' && *q <= '9') ++q;
            }
            if (q == d0 || (q == d0 + 1 && *d0 == '.')) return false;
            if (q < e && (*q == 'e' || *q == 'E')) {
                const char* x = q + 1;
                if (x < e && (*x == '+' || *x == '-')) ++x;
                const char* x0 = x;
                while (x < e && *x >= '0' && *x <= '9') ++x;
                if (x == x0) return false;  // num_get consumed the exponent marker
                q = x;
            }
            const std::string tok(p, q);
            out = std::strtod(tok.c_str(), nullptr);
            if (std::isinf(out)) return false;
            p = q;
            return true;
        } else {
            auto r = std::from_chars(p, e, out);
            if (r.ec != std::errc()) return false;
            p = r.ptr;
            return true;
        }
    }
};

// matrix_market.hpp:22-81: header, size line, entries; hermitian files hold the
// lower triangle and are expanded; duplicates summed in file order
// (build_from_triplets, sparse_matrix.hpp:43-64).
ParsedCrs mm_parse(const std::string& path) {
    std::ifstream in(path);
    if (!in) throw std::runtime_error("cannot open " + path);
    std::string line;
    std::size_t lineno = 0;
    if (!std::getline(in, line)) throw MMError("empty file", 1);
    ++lineno;
    {
        Tok t(line);
        std::string banner, object, format, field, sym;
        t.word(banner), t.word(object), t.word(format), t.word(field), t.word(sym);
        if (banner != "%%MatrixMarket" || object != "matrix" || format != "coordinate" || field != "complex")
            throw MMError("expected '%%MatrixMarket matrix coordinate complex' header", lineno);
        ParsedCrs r;
        if (sym == "hermitian") r.symmetry = 0;
        else if (sym == "general") r.symmetry = 1;
        else throw MMError("unsupported symmetry qualifier '" + sym + "'", lineno);
        std::size_t nrows = 0, ncols = 0, nnz = 0;
        while (std::getline(in, line)) {
            ++lineno;
            if (!line.empty() && line[0] == '%') continue;
            if (blank(line)) continue;
            Tok s(line);
            if (!(s.num(nrows) && s.num(ncols) && s.num(nnz))) throw MMError("malformed size line", lineno);
            break;
        }
        if (nrows == 0 || nrows != ncols) throw MMError("matrix must be square and nonempty", lineno);
        struct Ent {
            uint64_t key;  // row * n + col
            double re, im;
        };
        std::vector<Ent> ent;
        ent.reserve(r.symmetry == 0 ? 2 * nnz : nnz);
        std::size_t seen = 0;
        while (seen < nnz) {
            if (!std::getline(in, line)) throw MMError("unexpected end of file", lineno + 1);
            ++lineno;
            if (!line.empty() && line[0] == '%') continue;
            if (blank(line)) continue;
            Tok s(line);
            long long i = 0, j = 0;
            double re = 0.0, im = 0.0;
            if (!(s.num(i) && s.num(j) && s.num(re) && s.num(im))) throw MMError("malformed entry", lineno);
            if (i < 1 || j < 1 || i > static_cast<long long>(nrows) || j > static_cast<long long>(ncols))
                throw MMError("index out of range", lineno);
            if (!std::isfinite(re) || !std::isfinite(im)) throw MMError("non-finite value", lineno);
            const uint64_t rr = static_cast<uint64_t>(i - 1), cc = static_cast<uint64_t>(j - 1);
            ent.push_back({rr * nrows + cc, re, im});
            if (r.symmetry == 0 && rr != cc) ent.push_back({cc * nrows + rr, re, -im});
            ++seen;
        }
        if (nrows > static_cast<std::size_t>(INT32_MAX)) throw std::invalid_argument("matrix too large for int32 columns");
        std::stable_sort(ent.begin(), ent.end(), [](const Ent& a, const Ent& b) { return a.key < b.key; });
        r.n = nrows;
        r.rp.assign(nrows + 1, 0);
        for (std::size_t k = 0; k < ent.size();) {
            std::size_t k2 = k;
            double sr = 0.0, si = 0.0;
            while (k2 < ent.size() && ent[k2].key == ent[k].key) {
                sr += ent[k2].re;  // std::complex += : componentwise, in triplet order
                si += ent[k2].im;
                ++k2;
            }
            const uint64_t row = ent[k].key / nrows, col = ent[k].key % nrows;
            r.ci.push_back(static_cast<int32_t>(col));
            r.v.push_back(sr);
            r.v.push_back(si);
            ++r.rp[row + 1];
            k = k2;
        }
        for (std::size_t i2 = 0; i2 < nrows; ++i2) r.rp[i2 + 1] += r.rp[i2];
        return r;
    }
}

void put_u32(std::ofstream& o, uint32_t v) {
    unsigned char b[4];
    for (int k = 0; k < 4; ++k) b[k] = static_cast<unsigned char>(v >> (8 * k));
    o.write(reinterpret_cast<const char*>(b), 4);
}
void put_u64(std::ofstream& o, uint64_t v) {
    unsigned char b[8];
    for (int k = 0; k < 8; ++k) b[k] = static_cast<unsigned char>(v >> (8 * k));
    o.write(reinterpret_cast<const char*>(b), 8);
}
uint64_t get_u64(const unsigned char* b) {
    uint64_t v = 0;
    for (int k = 0; k < 8; ++k) v |= static_cast<uint64_t>(b[k]) << (8 * k);
    return v;
}

}  // namespace
}  // namespace cfb

using namespace cfb;

extern "C" {

size_t cf_matrix_market_error_line(void) { return g_mm_line; }

int cf_matrix_market_read(const char* path, size_t* n, size_t* nnz, int* symmetry, uint64_t* row_ptr,
                          int32_t* col_idx, double* values) {
    g_mm_line = 0;
    try {
        if (!path) throw std::invalid_argument("null path");
        const std::string key(path);
        auto it = g_mm_cache.find(key);
        if (!row_ptr || it == g_mm_cache.end()) {
            g_mm_cache.erase(key);
            it = g_mm_cache.emplace(key, mm_parse(key)).first;
        }
        const ParsedCrs& r = it->second;
        *n = r.n;
        *nnz = r.ci.size();
        if (symmetry) *symmetry = r.symmetry;
        if (!row_ptr) return CF_OK;
        std::memcpy(row_ptr, r.rp.data(), r.rp.size() * 8);
        std::memcpy(col_idx, r.ci.data(), r.ci.size() * 4);
        std::memcpy(values, r.v.data(), r.v.size() * 8);
        g_mm_cache.erase(it);
        return CF_OK;
    } catch (const MMError& e) {
        g_mm_line = e.line;
        set_error(e.what());
        return CF_ERUNTIME;
    } catch (...) {
        return guard([] { throw; });
    }
}

int cf_matrix_market_write(const char* path, size_t n, const uint64_t* rp, const int32_t* ci, const double* v,
                           int symmetry) {
    return guard([&] {  // matrix_market.hpp:85-104
        std::ofstream out(path);
        if (!out) throw std::runtime_error(std::string("cannot open ") + path + " for writing");
        const bool herm = symmetry == 0;
        out << "%%MatrixMarket matrix coordinate complex " << (herm ? "hermitian" : "general") << "\n";
        std::size_t count = 0;
        for (std::size_t i = 0; i < n; ++i)
            for (uint64_t k = rp[i]; k < rp[i + 1]; ++k)
                if (!herm || static_cast<std::size_t>(ci[k]) <= i) ++count;
        out << n << " " << n << " " << count << "\n";
        out.precision(17);
        for (std::size_t i = 0; i < n; ++i)
            for (uint64_t k = rp[i]; k < rp[i + 1]; ++k) {
                const std::size_t j = static_cast<std::size_t>(ci[k]);
                if (herm && j > i) continue;
                out << (i + 1) << " " << (j + 1) << " " << v[2 * k] << " " << v[2 * k + 1] << "\n";
            }
        if (!out) throw std::runtime_error(std::string("write failed for ") + path);
    });
}

// CFDB: magic "CFDB", u32 version 1, u64 n, n_s, n_b, u8 layout tag 0, then the
// panels' (re, im) bit patterns as little-endian u64 (block_vector.hpp:182-204).
int cf_blockvec_write(const char* path, size_t n, size_t ns, size_t nb, const double* panels) {
    return guard([&] {
        if (nb == 0 || ns % nb != 0) throw std::invalid_argument("n_b must divide n_s");
        std::ofstream out(path, std::ios::binary);
        if (!out) throw std::runtime_error(std::string("cannot open ") + path + " for writing");
        out.write("CFDB", 4);
        put_u32(out, 1);
        put_u64(out, n);
        put_u64(out, ns);
        put_u64(out, nb);
        out.put(0);
        std::vector<unsigned char> buf(1 << 20);
        const std::size_t total = 2 * n * ns;
        for (std::size_t k = 0; k < total;) {
            const std::size_t m = std::min<std::size_t>(buf.size() / 8, total - k);
            for (std::size_t q = 0; q < m; ++q) {
                uint64_t u;
                std::memcpy(&u, panels + k + q, 8);
                for (int b = 0; b < 8; ++b) buf[8 * q + b] = static_cast<unsigned char>(u >> (8 * b));
            }
            out.write(reinterpret_cast<const char*>(buf.data()), static_cast<std::streamsize>(8 * m));
            k += m;
        }
        if (!out) throw std::runtime_error(std::string("write failed for ") + path);
    });
}

// block_vector.hpp:206-229.  Two-phase: panels == NULL returns the shape only.
int cf_blockvec_read(const char* path, size_t* n, size_t* ns, size_t* nb, double* panels) {
    return guard([&] {
        const std::string p(path);
        std::ifstream in(p, std::ios::binary);
        if (!in) throw std::runtime_error("cannot open " + p);
        unsigned char hdr[4 + 4 + 24 + 1];
        in.read(reinterpret_cast<char*>(hdr), 4);
        if (!in || std::memcmp(hdr, "CFDB", 4) != 0) throw std::runtime_error(p + ": bad magic");
        in.read(reinterpret_cast<char*>(hdr + 4), 4);
        const uint32_t ver = static_cast<uint32_t>(hdr[4]) | static_cast<uint32_t>(hdr[5]) << 8 |
                             static_cast<uint32_t>(hdr[6]) << 16 | static_cast<uint32_t>(hdr[7]) << 24;
        if (!in || ver != 1) throw std::runtime_error(p + ": bad version");
        in.read(reinterpret_cast<char*>(hdr + 8), 24);
        const int tag = in.get();
        if (tag != 0) throw std::runtime_error(p + ": unknown layout tag");
        const uint64_t N = get_u64(hdr + 8), NS = get_u64(hdr + 16), NB = get_u64(hdr + 24);
        if (N < 1) throw std::invalid_argument("n must be >= 1");
        if (NB == 0 || NS == 0 || NS % NB != 0) throw std::invalid_argument("n_b must divide n_s");
        *n = N;
        *ns = NS;
        *nb = NB;
        if (!panels) return;
        std::vector<unsigned char> buf(1 << 20);
        const std::size_t total = 2 * N * NS;
        for (std::size_t k = 0; k < total;) {
            const std::size_t m = std::min<std::size_t>(buf.size() / 8, total - k);
            in.read(reinterpret_cast<char*>(buf.data()), static_cast<std::streamsize>(8 * m));
            if (!in) throw std::runtime_error(p + ": truncated data");
            for (std::size_t q = 0; q < m; ++q) {
                const uint64_t u = get_u64(buf.data() + 8 * q);
                std::memcpy(panels + k + q, &u, 8);
            }
            k += m;
        }
    });
}

}  // extern "C"
