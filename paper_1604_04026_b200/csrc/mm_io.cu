// Native MatrixMarket coordinate reader.
//
// Same acceptance rules and messages as the reference's Python line loop
// (sparse.py:217-268): header "%%MatrixMarket matrix coordinate
// real|integer general" (case-insensitive), '%' comment lines, a size line
// of three integers, then exactly nnz "i j v" lines with 1-based in-bounds
// indices and v > 0; blank and '%' lines are skipped.  The first offending
// line in file order determines the error, as in the sequential reference.
// Duplicates and non-finite values are left to SparseMatrix.from_coo, as in
// the reference.
//
// The file is mapped and parsed in two passes over line-aligned chunks on
// host threads: count the entry lines of every chunk, then parse each chunk
// into its slice of the output arrays.
#include <fcntl.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <cctype>
#include <cerrno>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "common.cuh"

namespace {


struct Mapped {
    const char *data = nullptr;
    size_t size = 0;
    int fd = -1;
    ~Mapped() {
        if (data && size) munmap(const_cast<char *>(data), size);
        if (fd >= 0) close(fd);
    }
};

bool map_file(const char *path, Mapped &m, std::string &err) {
    m.fd = open(path, O_RDONLY);
    if (m.fd < 0) {
        err = std::string("cannot open ") + path + ": " + strerror(errno);
        return false;
    }
    struct stat st;
    if (fstat(m.fd, &st) != 0) {
        err = std::string("cannot stat ") + path;
        return false;
    }
    m.size = (size_t)st.st_size;
    if (m.size == 0) return true;
    void *p = mmap(nullptr, m.size, PROT_READ, MAP_PRIVATE, m.fd, 0);
    if (p == MAP_FAILED) {
        err = std::string("cannot map ") + path;
        return false;
    }
    m.data = static_cast<const char *>(p);
    return true;
}

inline bool is_ws(char c) { return c == ' ' || c == '\t' || c == '\r' || c == '\v' || c == '\f'; }

// [b, e) with surrounding whitespace removed
inline void strip(const char *&b, const char *&e) {
    while (b < e && is_ws(*b)) ++b;
    while (e > b && is_ws(e[-1])) --e;
}

std::string py_repr_str(const char *b, const char *e) { return "'" + std::string(b, e) + "'"; }

// Python's repr of a float: shortest round-trip digits, ".0" on integral values.
std::string py_repr_double(double v) {
    if (std::isnan(v)) return "nan";
    if (std::isinf(v)) return v > 0 ? "inf" : "-inf";
    char buf[64];
    for (int prec = 1; prec <= 17; ++prec) {
        snprintf(buf, sizeof buf, "%.*g", prec, v);
        if (strtod(buf, nullptr) == v) break;
    }
    std::string s(buf);
    if (s.find_first_of(".eEn") == std::string::npos) s += ".0";
    return s;
}

// Python int(): optional sign, decimal digits (no separators here)
bool parse_int(const char *b, const char *e, long long &out) {
    if (b == e) return false;
    const char *p = b;
    bool neg = false;
    if (*p == '+' || *p == '-') neg = *p++ == '-';
    if (p == e || e - p > 18) return false;  // beyond int64 range of any valid index
    long long v = 0;
    for (; p < e; ++p) {
        if (*p < '0' || *p > '9') return false;
        v = v * 10 + (*p - '0');
    }
    out = neg ? -v : v;
    return true;
}

// Python float(): decimal / exponent forms and inf, infinity, nan (any case); no hex
bool parse_double(const char *b, const char *e, double &out) {
    char buf[64];
    const size_t len = (size_t)(e - b);
    if (len == 0 || len >= sizeof buf) return false;
    for (const char *q = b; q < e; ++q)
        if (*q == 'x' || *q == 'X') return false;
    memcpy(buf, b, len);
    buf[len] = 0;
    char *end = nullptr;
    out = strtod(buf, &end);
    return end == buf + len;
}

struct LineErr {
    size_t pos = SIZE_MAX;  // file offset of the offending line
    std::string msg;
    void set(size_t p, std::string m) {
        if (p < pos) {
            pos = p;
            msg = std::move(m);
        }
    }
};

// next line [b, e) starting at p; returns the offset after the line
inline size_t next_line(const char *d, size_t n, size_t p, const char *&b, const char *&e) {
    const char *nl = static_cast<const char *>(memchr(d + p, '\n', n - p));
    const size_t end = nl ? (size_t)(nl - d) : n;
    b = d + p;
    e = d + end;
    return nl ? end + 1 : n;
}

inline bool entry_line(const char *b, const char *e) {
    strip(b, e);
    return b < e && *b != '%';
}

struct Header {
    long long n_rows = 0, n_cols = 0, nnz = 0;
    size_t body = 0;  // offset of the first line after the size line
};

int parse_header(const Mapped &m, Header &h) {
    const char *d = m.data;
    const size_t n = m.size;
    const char *b, *e;
    size_t p = next_line(d, n, 0, b, e);
    strip(b, e);
    {
        std::vector<std::string> tok;
        const char *q = b;
        while (q < e) {
            while (q < e && is_ws(*q)) ++q;
            const char *t = q;
            while (q < e && !is_ws(*q)) ++q;
            if (q > t) {
                std::string s(t, q);
                for (auto &c : s) c = (char)tolower((unsigned char)c);
                tok.push_back(s);
            }
        }
        if (tok.size() != 5 || tok[0] != "%%matrixmarket" || tok[1] != "matrix" || tok[2] != "coordinate" ||
            (tok[3] != "real" && tok[3] != "integer") || tok[4] != "general")
            return klnmf::set_error_msg(KLNMF_MM_FORMAT_ERROR,
                                        ("unsupported MatrixMarket header: " + py_repr_str(b, e)).c_str());
    }
    // comment lines, then the size line
    for (;;) {
        if (p >= n) {
            b = e = d + n;
            break;
        }
        const size_t q = next_line(d, n, p, b, e);
        const char *sb = b, *se = e;
        while (sb < se && is_ws(*sb)) ++sb;
        p = q;
        if (sb < se && *sb == '%') continue;
        break;
    }
    const char *lb = b, *le = e;
    strip(lb, le);
    long long v[3];
    int k = 0;
    bool ok = true;
    const char *q = lb;
    while (q < le && ok) {
        while (q < le && is_ws(*q)) ++q;
        const char *t = q;
        while (q < le && !is_ws(*q)) ++q;
        if (q == t) break;
        if (k >= 3 || !parse_int(t, q, v[k])) ok = false;
        ++k;
    }
    if (!ok || k != 3 || v[2] < 0)
        return klnmf::set_error_msg(KLNMF_MM_FORMAT_ERROR,
                                    ("malformed size line: '" + std::string(b, e) + (e < d + n ? "\\n'" : "'")).c_str());
    h.n_rows = v[0];
    h.n_cols = v[1];
    h.nnz = v[2];
    h.body = p;
    return 0;
}

}  // namespace

extern "C" int klnmf_mm_header(const char *path, int64_t *n_rows, int64_t *n_cols, int64_t *nnz) {
    Mapped m;
    std::string err;
    if (!map_file(path, m, err)) return klnmf::set_error_msg(1, err.c_str());
    Header h;
    if (int rc = parse_header(m, h)) return rc;
    *n_rows = h.n_rows;
    *n_cols = h.n_cols;
    *nnz = h.nnz;
    return 0;
}

extern "C" int klnmf_mm_read(const char *path, int64_t nnz_cap, int64_t *rows, int64_t *cols, double *vals) {
    Mapped m;
    std::string err;
    if (!map_file(path, m, err)) return klnmf::set_error_msg(1, err.c_str());
    Header h;
    if (int rc = parse_header(m, h)) return rc;
    if (h.nnz > nnz_cap) return klnmf::set_error_msg(1, "klnmf_mm_read: output arrays are too small");
    const char *d = m.data;
    const size_t n = m.size, body = h.body;

    // line-aligned chunks of the body
    const unsigned hc = std::thread::hardware_concurrency();
    int nt = (int)std::max(1u, std::min(32u, hc ? hc : 1u));
    if (n - body < ((size_t)4 << 20)) nt = 1;
    std::vector<size_t> cut(nt + 1, n);
    cut[0] = body;
    for (int t = 1; t < nt; ++t) {
        size_t p = body + (n - body) * (size_t)t / (size_t)nt;
        if (p < cut[t - 1]) p = cut[t - 1];
        const char *nl = p < n ? static_cast<const char *>(memchr(d + p, '\n', n - p)) : nullptr;
        cut[t] = nl ? (size_t)(nl - d) + 1 : n;
    }
    // pass 1: entry lines per chunk
    std::vector<long long> cnt(nt, 0);
    {
        std::vector<std::thread> th;
        for (int t = 0; t < nt; ++t)
            th.emplace_back([&, t] {
                long long c = 0;
                const char *b, *e;
                for (size_t p = cut[t]; p < cut[t + 1];) {
                    p = next_line(d, n, p, b, e);
                    if (entry_line(b, e)) ++c;
                }
                cnt[t] = c;
            });
        for (auto &x : th) x.join();
    }
    std::vector<long long> first(nt + 1, 0);
    for (int t = 0; t < nt; ++t) first[t + 1] = first[t] + cnt[t];
    const long long total = first[nt];

    // pass 2: parse; every thread keeps its earliest error
    std::vector<LineErr> errs(nt);
    {
        std::vector<std::thread> th;
        for (int t = 0; t < nt; ++t)
            th.emplace_back([&, t] {
                long long k = first[t];
                const char *b, *e;
                for (size_t p = cut[t]; p < cut[t + 1];) {
                    const size_t lp = p;
                    p = next_line(d, n, p, b, e);
                    const char *sb = b, *se = e;
                    strip(sb, se);
                    if (sb == se || *sb == '%') continue;
                    const long long idx = k++;
                    const char *tk[3][2];
                    int nt_ = 0;
                    for (const char *q = sb; q < se;) {
                        while (q < se && is_ws(*q)) ++q;
                        const char *s0 = q;
                        while (q < se && !is_ws(*q)) ++q;
                        if (q > s0) {
                            if (nt_ < 3) {
                                tk[nt_][0] = s0;
                                tk[nt_][1] = q;
                            }
                            ++nt_;
                        }
                    }
                    auto bad = [&] { return "malformed entry line: " + py_repr_str(sb, se); };
                    if (nt_ != 3 || idx >= h.nnz) {
                        errs[t].set(lp, bad());
                        break;
                    }
                    long long i, j;
                    double v;
                    if (!parse_int(tk[0][0], tk[0][1], i) || !parse_int(tk[1][0], tk[1][1], j) ||
                        !parse_double(tk[2][0], tk[2][1], v)) {
                        errs[t].set(lp, bad());
                        break;
                    }
                    if (!(1 <= i && i <= h.n_rows && 1 <= j && j <= h.n_cols)) {
                        errs[t].set(lp, "coordinate (" + std::to_string(i) + ", " + std::to_string(j) +
                                            ") out of bounds");
                        break;
                    }
                    if (v < 0.0) {
                        errs[t].set(lp, "negative entry " + py_repr_double(v) + " at (" + std::to_string(i) + ", " +
                                            std::to_string(j) + ")");
                        break;
                    }
                    if (v == 0.0) {
                        errs[t].set(lp, "explicit zero at (" + std::to_string(i) + ", " + std::to_string(j) + ")");
                        break;
                    }
                    rows[idx] = i - 1;
                    cols[idx] = j - 1;
                    vals[idx] = v;
                }
            });
        for (auto &x : th) x.join();
    }
    LineErr first_err;
    for (auto &x : errs)
        if (x.pos != SIZE_MAX) first_err.set(x.pos, x.msg);
    if (first_err.pos != SIZE_MAX) return klnmf::set_error_msg(KLNMF_MM_FORMAT_ERROR, first_err.msg.c_str());
    if (total != h.nnz)
        return klnmf::set_error_msg(KLNMF_MM_FORMAT_ERROR, ("expected " + std::to_string(h.nnz) + " entries, found " +
                                                            std::to_string(total))
                                                               .c_str());
    return 0;
}
