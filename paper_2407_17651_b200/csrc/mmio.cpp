// Native Matrix Market / vector / permutation text I/O (C ABI, include/pars3.h).
//
// Replaces the reference's line-by-line Python readers and writers
// (mmio.py:52-223, reorder.py:300-333) with a parallel fast path: the file
// is read once, cut into chunks at line boundaries, entry lines are counted
// per chunk (pass 1), prefix-summed, and parsed straight into place
// (pass 2).  The fast path accepts only the canonical syntax the reference's
// writers produce -- ASCII, '\n' line ends, space/tab separators, decimal
// integers and decimal/exponent/inf floats -- and returns PARS3_SLOW_PATH
// for anything else (a malformed line, an out-of-range index, underscores,
// '\r', NaN tokens, ...): the Python wrapper then runs the exact restatement
// of the reference's reader, which raises the reference's error with its
// line number.  Values are parsed with strtod (correctly rounded, as
// Python's float()) and written with "%.17g" (as the reference's VALUE_FMT),
// so a write/read round trip is bit-exact.
#include <omp.h>

#include <cerrno>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <new>
#include <string>
#include <vector>

#include "common.h"

namespace {

int threads_for(int nthreads) { return nthreads > 0 ? nthreads : omp_get_max_threads(); }

bool read_file(const char *path, std::string &buf) {
    FILE *f = fopen(path, "rb");
    if (!f) return false;
    if (fseek(f, 0, SEEK_END) != 0) {
        fclose(f);
        return false;
    }
    long sz = ftell(f);
    if (sz < 0) {
        fclose(f);
        return false;
    }
    rewind(f);
    buf.resize((size_t)sz);
    size_t got = sz ? fread(&buf[0], 1, (size_t)sz, f) : 0;
    fclose(f);
    return got == (size_t)sz;
}

// bytes the fast path refuses: non-ASCII, and control characters other than
// '\n' and '\t' (Python's str.split()/readlines() treat \r, \v, \f and
// \x1c-\x1f specially)
inline bool odd_byte(unsigned char c) { return c >= 128 || (c < 32 && c != '\n' && c != '\t'); }

inline bool is_sep(char c) { return c == ' ' || c == '\t'; }

// split [p, e) on spaces/tabs into at most `maxf` tokens; returns the count
// (maxf + 1 when there are more)
int split(const char *p, const char *e, const char **tb, const char **te, int maxf) {
    int nf = 0;
    while (p < e) {
        while (p < e && is_sep(*p)) p++;
        if (p == e) break;
        if (nf == maxf) return maxf + 1;
        tb[nf] = p;
        while (p < e && !is_sep(*p)) p++;
        te[nf] = p;
        nf++;
    }
    return nf;
}

// strict decimal integer: [+-]?[0-9]{1,18}
bool parse_int(const char *b, const char *e, int64_t &v) {
    bool neg = false;
    if (b < e && (*b == '+' || *b == '-')) {
        neg = *b == '-';
        b++;
    }
    if (b == e || e - b > 18) return false;
    int64_t r = 0;
    for (; b < e; b++) {
        if (*b < '0' || *b > '9') return false;
        r = r * 10 + (*b - '0');
    }
    v = neg ? -r : r;
    return true;
}

inline bool ieq(const char *b, const char *e, const char *w) {
    size_t n = strlen(w);
    if ((size_t)(e - b) != n) return false;
    for (size_t i = 0; i < n; i++) {
        char c = b[i];
        if (c >= 'A' && c <= 'Z') c = (char)(c - 'A' + 'a');
        if (c != w[i]) return false;
    }
    return true;
}

// strict float: [+-]?(digits[.digits*]|.digits)([eE][+-]?digits)? or
// [+-]?(inf|infinity); NaN and everything else -> slow path
bool parse_float(const char *b, const char *e, double &v) {
    const char *p = b;
    if (p < e && (*p == '+' || *p == '-')) p++;
    if (ieq(p, e, "inf") || ieq(p, e, "infinity")) {
        v = (*b == '-') ? -HUGE_VAL : HUGE_VAL;
        return true;
    }
    const char *q = p;
    int digits = 0;
    while (q < e && *q >= '0' && *q <= '9') q++, digits++;
    if (q < e && *q == '.') {
        q++;
        while (q < e && *q >= '0' && *q <= '9') q++, digits++;
    }
    if (digits == 0) return false;
    if (q < e && (*q == 'e' || *q == 'E')) {
        q++;
        if (q < e && (*q == '+' || *q == '-')) q++;
        int ed = 0;
        while (q < e && *q >= '0' && *q <= '9') q++, ed++;
        if (ed == 0) return false;
    }
    if (q != e) return false;
    char tmp[64];
    if (e - b >= (long)sizeof(tmp)) {
        std::string s(b, e);
        v = strtod(s.c_str(), nullptr);
    } else {
        memcpy(tmp, b, (size_t)(e - b));
        tmp[e - b] = 0;
        v = strtod(tmp, nullptr);
    }
    return true;
}

// a line is skipped when it starts with '%' or is blank (the reference's
// `line.startswith("%") or not line.strip()`)
inline bool skip_line(const char *b, const char *e) {
    if (b < e && *b == '%') return true;
    for (const char *p = b; p < e; p++)
        if (!is_sep(*p)) return false;
    return true;
}

const char *next_line(const char *p, const char *end) {
    const char *q = (const char *)memchr(p, '\n', (size_t)(end - p));
    return q ? q : end;
}

// chunk boundaries of [b, e) at line starts
std::vector<const char *> chunks(const char *b, const char *e, int nt) {
    std::vector<const char *> cut{b};
    const size_t len = (size_t)(e - b);
    for (int t = 1; t < nt; t++) {
        const char *p = b + len * t / nt;
        if (p <= cut.back()) continue;
        const char *q = (const char *)memchr(p, '\n', (size_t)(e - p));
        p = q ? q + 1 : e;
        if (p > cut.back() && p < e) cut.push_back(p);
    }
    cut.push_back(e);
    return cut;
}

}  // namespace

struct pars3_mm_file {
    std::string buf;
    int64_t n = 0, nnz = 0;
    int32_t qual = 0;  // 0 general, 1 symmetric, 2 skew-symmetric
    size_t body = 0;   // offset of the first line after the size line
};

extern "C" int pars3_mm_open(const char *path, pars3_mm_file **out, int64_t *n, int64_t *nnz,
                             int32_t *qualifier) {
    if (!path || !out || !n || !nnz || !qualifier) PARS3_FAIL(PARS3_ERR_ARG, "null argument");
    *out = nullptr;
    pars3_mm_file *f = new (std::nothrow) pars3_mm_file;
    if (!f) PARS3_FAIL(PARS3_ERR_NOMEM, "out of host memory");
    if (!read_file(path, f->buf)) {
        delete f;
        return PARS3_SLOW_PATH;  // let Python raise the reference's OSError
    }
    const char *b = f->buf.data(), *e = b + f->buf.size();
    for (const char *p = b; p < e; p++)
        if (odd_byte((unsigned char)*p)) {
            delete f;
            return PARS3_SLOW_PATH;
        }
    // header: exactly five fields (mmio.py:35-49)
    const char *le = next_line(b, e);
    const char *tb[6], *te[6];
    if (split(b, le, tb, te, 5) != 5 || !(te[0] - tb[0] == 14 && !memcmp(tb[0], "%%MatrixMarket", 14)) ||
        !ieq(tb[1], te[1], "matrix") || !ieq(tb[2], te[2], "coordinate") || !ieq(tb[3], te[3], "real")) {
        delete f;
        return PARS3_SLOW_PATH;
    }
    if (ieq(tb[4], te[4], "general"))
        f->qual = 0;
    else if (ieq(tb[4], te[4], "symmetric"))
        f->qual = 1;
    else if (ieq(tb[4], te[4], "skew-symmetric"))
        f->qual = 2;
    else {
        delete f;
        return PARS3_SLOW_PATH;
    }
    // size line: first non-comment, non-blank line
    const char *p = le < e ? le + 1 : e;
    while (p < e) {
        const char *l2 = next_line(p, e);
        if (!skip_line(p, l2)) break;
        p = l2 < e ? l2 + 1 : e;
    }
    if (p >= e) {
        delete f;
        return PARS3_SLOW_PATH;
    }
    le = next_line(p, e);
    int64_t r, c, z;
    if (split(p, le, tb, te, 3) != 3 || !parse_int(tb[0], te[0], r) || !parse_int(tb[1], te[1], c) ||
        !parse_int(tb[2], te[2], z) || r != c || z < 0 || r < 0 || r >= INT32_MAX) {
        delete f;
        return PARS3_SLOW_PATH;
    }
    f->n = r;
    f->nnz = z;
    f->body = (size_t)((le < e ? le + 1 : e) - b);
    *n = f->n;
    *nnz = f->nnz;
    *qualifier = f->qual;
    *out = f;
    return PARS3_OK;
}

extern "C" int pars3_mm_fill(pars3_mm_file *f, int64_t *rows, int64_t *cols, double *vals,
                             int nthreads) {
    if (!f || (f->nnz > 0 && (!rows || !cols || !vals))) PARS3_FAIL(PARS3_ERR_ARG, "null argument");
    const char *b = f->buf.data() + f->body, *e = f->buf.data() + f->buf.size();
    const int nt = threads_for(nthreads);
    std::vector<const char *> cut = chunks(b, e, nt);
    const int nc = (int)cut.size() - 1;
    std::vector<int64_t> cnt(nc + 1, 0);
#pragma omp parallel for num_threads(nt) schedule(static, 1)
    for (int k = 0; k < nc; k++) {
        int64_t c = 0;
        for (const char *p = cut[k]; p < cut[k + 1];) {
            const char *le = next_line(p, cut[k + 1]);
            if (!skip_line(p, le)) c++;
            p = le + 1;
        }
        cnt[k + 1] = c;
    }
    for (int k = 0; k < nc; k++) cnt[k + 1] += cnt[k];
    if (cnt[nc] != f->nnz) return PARS3_SLOW_PATH;  // count mismatch: the exact reader reports it
    const int64_t n = f->n;
    const int qual = f->qual;
    int bad = 0;
#pragma omp parallel for num_threads(nt) schedule(static, 1) reduction(| : bad)
    for (int k = 0; k < nc; k++) {
        int64_t at = cnt[k];
        const char *tb[4], *te[4];
        for (const char *p = cut[k]; p < cut[k + 1] && !bad;) {
            const char *le = next_line(p, cut[k + 1]);
            if (!skip_line(p, le)) {
                int64_t i, j;
                double v;
                if (split(p, le, tb, te, 3) != 3 || !parse_int(tb[0], te[0], i) ||
                    !parse_int(tb[1], te[1], j) || !parse_float(tb[2], te[2], v) || i < 1 || i > n ||
                    j < 1 || j > n || (qual != 0 && j > i) || (qual == 2 && i == j && v != 0.0)) {
                    bad = 1;
                    break;
                }
                rows[at] = i - 1;
                cols[at] = j - 1;
                vals[at] = v;
                at++;
            }
            p = le + 1;
        }
    }
    return bad ? PARS3_SLOW_PATH : PARS3_OK;
}

extern "C" int pars3_mm_close(pars3_mm_file *f) {
    delete f;
    return PARS3_OK;
}

namespace {

// "%.17g" as Python's VALUE_FMT % x (CPython prints every NaN as "nan")
inline int fmt_g17(char *o, double v) {
    if (std::isnan(v)) {
        memcpy(o, "nan", 3);
        return 3;
    }
    return snprintf(o, 32, "%.17g", v);
}

inline int fmt_i64(char *o, int64_t v) { return snprintf(o, 24, "%lld", (long long)v); }

// format `count` records in parallel chunks, then write them in order
template <class F>
int write_records(FILE *fh, int64_t count, int nt, size_t max_rec, F rec) {
    const int64_t per = 1 << 16;
    const int64_t nblk = (count + per - 1) / per;
    int rc = PARS3_OK;
    for (int64_t b0 = 0; b0 < nblk && rc == PARS3_OK; b0 += nt) {
        const int64_t b1 = std::min<int64_t>(nblk, b0 + nt);
        std::vector<std::string> out((size_t)(b1 - b0));
#pragma omp parallel for num_threads(nt) schedule(static, 1)
        for (int64_t blk = b0; blk < b1; blk++) {
            const int64_t a = blk * per, z = std::min(count, a + per);
            std::string &s = out[(size_t)(blk - b0)];
            s.resize((size_t)(z - a) * max_rec);
            size_t o = 0;
            for (int64_t k = a; k < z; k++) o += (size_t)rec(k, &s[o]);
            s.resize(o);
        }
        for (auto &s : out)
            if (fwrite(s.data(), 1, s.size(), fh) != s.size()) rc = PARS3_ERR_ARG;
    }
    return rc;
}

}  // namespace

extern "C" int pars3_mm_write(const char *path, const char *qualifier, int64_t n, int64_t count,
                              const int64_t *rows, const int64_t *cols, const double *vals,
                              int nthreads) {
    if (!path || !qualifier || (count > 0 && (!rows || !cols || !vals)))
        PARS3_FAIL(PARS3_ERR_ARG, "null argument");
    FILE *fh = fopen(path, "wb");
    if (!fh) PARS3_FAIL(PARS3_ERR_ARG, "cannot open %s for writing", path);
    fprintf(fh, "%%%%MatrixMarket matrix coordinate real %s\n%lld %lld %lld\n", qualifier,
            (long long)n, (long long)n, (long long)count);
    int rc = write_records(fh, count, threads_for(nthreads), 24 + 24 + 32 + 3, [&](int64_t k, char *o) {
        int w = fmt_i64(o, rows[k] + 1);
        o[w++] = ' ';
        w += fmt_i64(o + w, cols[k] + 1);
        o[w++] = ' ';
        w += fmt_g17(o + w, vals[k]);
        o[w++] = '\n';
        return w;
    });
    if (fclose(fh) != 0 || rc) PARS3_FAIL(PARS3_ERR_ARG, "write to %s failed", path);
    return PARS3_OK;
}

extern "C" int pars3_vector_write(const char *path, int64_t n, const double *x, int nthreads) {
    if (!path || (n > 0 && !x)) PARS3_FAIL(PARS3_ERR_ARG, "null argument");
    FILE *fh = fopen(path, "wb");
    if (!fh) PARS3_FAIL(PARS3_ERR_ARG, "cannot open %s for writing", path);
    int rc = write_records(fh, n, threads_for(nthreads), 34, [&](int64_t k, char *o) {
        int w = fmt_g17(o, x[k]);
        o[w++] = '\n';
        return w;
    });
    if (fclose(fh) != 0 || rc) PARS3_FAIL(PARS3_ERR_ARG, "write to %s failed", path);
    return PARS3_OK;
}

extern "C" int pars3_permutation_write(const char *path, int64_t n, const int64_t *forward,
                                       int nthreads) {
    if (!path || (n > 0 && !forward)) PARS3_FAIL(PARS3_ERR_ARG, "null argument");
    FILE *fh = fopen(path, "wb");
    if (!fh) PARS3_FAIL(PARS3_ERR_ARG, "cannot open %s for writing", path);
    fprintf(fh, "%lld\n", (long long)n);
    int rc = write_records(fh, n, threads_for(nthreads), 50, [&](int64_t k, char *o) {
        int w = fmt_i64(o, k);
        o[w++] = ' ';
        w += fmt_i64(o + w, forward[k]);
        o[w++] = '\n';
        return w;
    });
    if (fclose(fh) != 0 || rc) PARS3_FAIL(PARS3_ERR_ARG, "write to %s failed", path);
    return PARS3_OK;
}

// One value per non-blank, non-'%' line (mmio.py:203-215); *count = values.
// Call with x == NULL to count, then again to fill.
extern "C" int pars3_vector_read(const char *path, double *x, int64_t *count, int nthreads) {
    if (!path || !count) PARS3_FAIL(PARS3_ERR_ARG, "null argument");
    std::string buf;
    if (!read_file(path, buf)) return PARS3_SLOW_PATH;
    const char *b = buf.data(), *e = b + buf.size();
    for (const char *p = b; p < e; p++)
        if (odd_byte((unsigned char)*p)) return PARS3_SLOW_PATH;
    const int nt = threads_for(nthreads);
    std::vector<const char *> cut = chunks(b, e, nt);
    const int nc = (int)cut.size() - 1;
    std::vector<int64_t> cnt(nc + 1, 0);
    // the reference strips each line first: a leading-blank "%..." is a comment too
    auto skip = [](const char *p, const char *le) {
        while (p < le && is_sep(*p)) p++;
        return p == le || *p == '%';
    };
#pragma omp parallel for num_threads(nt) schedule(static, 1)
    for (int k = 0; k < nc; k++) {
        int64_t c = 0;
        for (const char *p = cut[k]; p < cut[k + 1];) {
            const char *le = next_line(p, cut[k + 1]);
            if (!skip(p, le)) c++;
            p = le + 1;
        }
        cnt[k + 1] = c;
    }
    for (int k = 0; k < nc; k++) cnt[k + 1] += cnt[k];
    if (!x) {
        *count = cnt[nc];
        return PARS3_OK;
    }
    if (*count != cnt[nc]) PARS3_FAIL(PARS3_ERR_ARG, "vector length changed");
    int bad = 0;
#pragma omp parallel for num_threads(nt) schedule(static, 1) reduction(| : bad)
    for (int k = 0; k < nc; k++) {
        int64_t at = cnt[k];
        const char *tb[2], *te[2];
        for (const char *p = cut[k]; p < cut[k + 1] && !bad;) {
            const char *le = next_line(p, cut[k + 1]);
            if (!skip(p, le)) {
                double v;
                if (split(p, le, tb, te, 1) != 1 || !parse_float(tb[0], te[0], v)) {
                    bad = 1;
                    break;
                }
                x[at++] = v;
            }
            p = le + 1;
        }
    }
    return bad ? PARS3_SLOW_PATH : PARS3_OK;
}

// A permutation file (reorder.py:300-333): count line, then "old new" pairs
// in any order.  Fast path: exactly n well-formed pairs; old/new returned
// in file order (the wrapper validates ranges and duplicates like the
// reference).  Call with old == NULL to get n.
extern "C" int pars3_permutation_read(const char *path, int64_t *n, int64_t *old_idx,
                                      int64_t *new_idx, int nthreads) {
    if (!path || !n) PARS3_FAIL(PARS3_ERR_ARG, "null argument");
    std::string buf;
    if (!read_file(path, buf)) return PARS3_SLOW_PATH;
    const char *b = buf.data(), *e = b + buf.size();
    for (const char *p = b; p < e; p++)
        if (odd_byte((unsigned char)*p)) return PARS3_SLOW_PATH;
    auto blank = [](const char *p, const char *le) {
        for (; p < le; p++)
            if (!is_sep(*p)) return false;
        return true;
    };
    const char *p = b;
    while (p < e) {  // first non-blank line: the count
        const char *le = next_line(p, e);
        if (!blank(p, le)) break;
        p = le < e ? le + 1 : e;
    }
    if (p >= e) return PARS3_SLOW_PATH;
    const char *le = next_line(p, e);
    const char *tb[3], *te[3];
    int64_t cnt;
    if (split(p, le, tb, te, 1) != 1 || !parse_int(tb[0], te[0], cnt) || cnt < 0) return PARS3_SLOW_PATH;
    if (!old_idx) {
        *n = cnt;
        return PARS3_OK;
    }
    if (*n != cnt) PARS3_FAIL(PARS3_ERR_ARG, "permutation length changed");
    const char *body = le < e ? le + 1 : e;
    const int nt = threads_for(nthreads);
    std::vector<const char *> cut = chunks(body, e, nt);
    const int nc = (int)cut.size() - 1;
    std::vector<int64_t> lines(nc + 1, 0);
#pragma omp parallel for num_threads(nt) schedule(static, 1)
    for (int k = 0; k < nc; k++) {
        int64_t c = 0;
        for (const char *q = cut[k]; q < cut[k + 1];) {
            const char *l2 = next_line(q, cut[k + 1]);
            if (!blank(q, l2)) c++;
            q = l2 + 1;
        }
        lines[k + 1] = c;
    }
    for (int k = 0; k < nc; k++) lines[k + 1] += lines[k];
    if (lines[nc] != cnt) return PARS3_SLOW_PATH;
    int bad = 0;
#pragma omp parallel for num_threads(nt) schedule(static, 1) reduction(| : bad)
    for (int k = 0; k < nc; k++) {
        int64_t at = lines[k];
        const char *xb[3], *xe[3];
        for (const char *q = cut[k]; q < cut[k + 1] && !bad;) {
            const char *l2 = next_line(q, cut[k + 1]);
            if (!blank(q, l2)) {
                int64_t o, w;
                if (split(q, l2, xb, xe, 2) != 2 || !parse_int(xb[0], xe[0], o) || !parse_int(xb[1], xe[1], w)) {
                    bad = 1;
                    break;
                }
                old_idx[at] = o;
                new_idx[at] = w;
                at++;
            }
            q = l2 + 1;
        }
    }
    return bad ? PARS3_SLOW_PATH : PARS3_OK;
}
