// Host builder of the full-CSR plan (fullcsr.h).  Row i of A = D + L - L^T
// (sign convention D1, formats.py:14-18: a stored lower value a_ic is +a_ic
// at (i, c) and -a_ic at (c, i)) lists, by ascending column: the row's
// stored outer then middle entries (split.py:116-141 keeps both ascending,
// every outer column below every middle one), the diagonal, then the
// negated mirrors -a_ri of the rows r > i that store column i (ascending r:
// a counting-sort transpose).
#include "fullcsr.h"

#include <omp.h>

#include <algorithm>
#include <new>

#include "common.h"

namespace pars3 {

int build_full_csr(const pars3_split_view *s, FullCsr &F) {
    const int64_t n = s->n;
    try {
        F = FullCsr();
        F.n = n;
        const int64_t nm = s->mid_ptr ? s->mid_ptr[n] : 0, no = s->outer_count;
        std::vector<int64_t> optr(n + 1, 0);
        for (int64_t e = 0; e < no; e++) {
            const int32_t r = s->outer_row[e];
            if (r < 0 || r >= n || (e && r < s->outer_row[e - 1]))
                PARS3_FAIL(PARS3_ERR_STRUCT, "outer rows out of range or unsorted");
            optr[r + 1]++;
        }
        for (int64_t r = 0; r < n; r++) optr[r + 1] += optr[r];
        // upper counts (mirrors per column)
        std::vector<int64_t> up(n + 1, 0);
        for (int64_t k = 0; k < nm; k++) up[s->mid_col[k] + 1]++;
        for (int64_t k = 0; k < no; k++) up[s->outer_col[k] + 1]++;
        std::vector<int64_t> rp(n + 1, 0);
        for (int64_t r = 0; r < n; r++) {
            const int64_t low = (optr[r + 1] - optr[r]) + (s->mid_ptr[r + 1] - s->mid_ptr[r]);
            rp[r + 1] = rp[r] + low + 1 + up[r + 1];
        }
        for (int64_t r = 0; r < n; r++) up[r + 1] += up[r];
        F.ne = rp[n];
        const int64_t nep = (F.ne + kCsrWarp - 1) / kCsrWarp * kCsrWarp;
        F.col.assign(nep, 0);
        F.val.assign(nep, 0.0);
        // lower entries and the diagonal (parallel over rows)
#pragma omp parallel for schedule(dynamic, 4096)
        for (int64_t r = 0; r < n; r++) {
            int64_t e = rp[r];
            for (int64_t k = optr[r]; k < optr[r + 1]; k++, e++) {
                F.col[e] = s->outer_col[k];
                F.val[e] = s->outer_val[k];
            }
            for (int64_t k = s->mid_ptr[r]; k < s->mid_ptr[r + 1]; k++, e++) {
                F.col[e] = s->mid_col[k];
                F.val[e] = s->mid_val[k];
            }
            F.col[e] = (int32_t)r;
            F.val[e] = s->diag[r];
        }
        // the negated mirrors: row c gets (r, -a_rc) for ascending r
        std::vector<int64_t> cur(n);
        for (int64_t c = 0; c < n; c++) cur[c] = rp[c + 1] - (up[c + 1] - up[c]);
        for (int64_t r = 0; r < n; r++) {
            for (int64_t k = optr[r]; k < optr[r + 1]; k++) {
                const int32_t c = s->outer_col[k];
                F.col[cur[c]] = (int32_t)r;
                F.val[cur[c]++] = -s->outer_val[k];
            }
            for (int64_t k = s->mid_ptr[r]; k < s->mid_ptr[r + 1]; k++) {
                const int32_t c = s->mid_col[k];
                F.col[cur[c]] = (int32_t)r;
                F.val[cur[c]++] = -s->mid_val[k];
            }
        }
        // lanes: first row and row-start flags (padding continues the last row)
        const int64_t nl = nep / kCsrLane;
        F.lane_row.assign(nl, 0);
        F.lane_flags.assign(nl, 0u);
#pragma omp parallel for schedule(static)
        for (int64_t l = 0; l < nl; l++) {
            const int64_t e0 = l * kCsrLane;
            int64_t r = e0 < F.ne ? (int64_t)(std::upper_bound(rp.begin(), rp.end(), e0) - rp.begin()) - 1 : n - 1;
            F.lane_row[l] = (int32_t)r;
            uint32_t f = 0;
            for (int k = 0; k <= kCsrLane; k++) {
                const int64_t e = e0 + k;
                bool start;
                if (e >= nep)
                    start = true;  // the end
                else if (e >= F.ne)
                    start = false;  // padding: the last row continues
                else {
                    while (r + 1 < n && rp[r + 1] <= e) r++;
                    start = rp[r] == e;
                }
                if (start) f |= 1u << k;
            }
            F.lane_flags[l] = f;
        }
        // rows spanning warps (the last row extends over the padding)
        for (int64_t r = 0; r < n; r++) {
            const int64_t last = r + 1 < n ? rp[r + 1] - 1 : nep - 1;
            const int64_t w0 = rp[r] / kCsrWarp, w1 = last / kCsrWarp;
            if (w1 > w0) {
                F.span_row.push_back((int32_t)r);
                F.span_w0.push_back((int32_t)w0);
                F.span_w1.push_back((int32_t)w1);
                F.max_span = std::max<int32_t>(F.max_span, (int32_t)(w1 - w0));
            }
        }
    } catch (const std::bad_alloc &) {
        PARS3_FAIL(PARS3_ERR_NOMEM, "full CSR plan: out of host memory");
    }
    return PARS3_OK;
}

}  // namespace pars3

// Inspection / tests (include/pars3.h): the full-CSR plan of a split on the
// host.  Call with col == NULL for the sizes {padded entries, real entries,
// lanes, spans}, then with arrays of those sizes.
extern "C" int pars3_full_csr_host(const pars3_split_view *s, int64_t *sizes, int32_t *col, double *val,
                                   int32_t *lane_row, uint32_t *lane_flags, int32_t *span_row,
                                   int32_t *span_w0, int32_t *span_w1) {
    if (!s || !sizes) PARS3_FAIL(PARS3_ERR_ARG, "null argument");
    pars3::FullCsr F;
    const int rc = pars3::build_full_csr(s, F);
    if (rc) return rc;
    sizes[0] = (int64_t)F.col.size();
    sizes[1] = F.ne;
    sizes[2] = (int64_t)F.lane_row.size();
    sizes[3] = (int64_t)F.span_row.size();
    if (!col) return PARS3_OK;
    std::copy(F.col.begin(), F.col.end(), col);
    std::copy(F.val.begin(), F.val.end(), val);
    std::copy(F.lane_row.begin(), F.lane_row.end(), lane_row);
    std::copy(F.lane_flags.begin(), F.lane_flags.end(), lane_flags);
    std::copy(F.span_row.begin(), F.span_row.end(), span_row);
    std::copy(F.span_w0.begin(), F.span_w0.end(), span_w0);
    std::copy(F.span_w1.begin(), F.span_w1.end(), span_w1);
    return PARS3_OK;
}
