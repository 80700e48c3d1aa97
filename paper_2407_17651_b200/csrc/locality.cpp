// Internal locality order of a device plan ("locality order").
//
// RCM (the reference's order, reorder.py:251-286) is a breadth-first
// layering.  On a matrix whose graph is a narrow band plus a few random
// long-range entries (BASELINE c3: 1 % far entries), every long entry opens
// a new BFS front, so the RCM layering interleaves far-apart regions of the
// band: 72 % of c3's entries end up more than 4 096 labels from the
// diagonal and nearly every tile falls back to an explicit column list with
// about one entry per shared-memory slot.  The tile kernel is then bound by
// random L2 gathers and reductions, not by HBM.
//
// The fix is internal: the plan may store P A P^T for a second permutation P
// of its own and gather x / y through it (tiles.cu).  The API, the labels
// and the split stay the reference's.  P is RCM of a FILTERED graph that
// keeps only the entries supported by short cycles: the support of an edge
// (i, j) is the number of paths i-l-j plus i-k-l-j (k != j, l != i).  Band
// entries have several such paths (about 5 on c3); a random long entry has
// almost none, because its two ends have unrelated neighbourhoods.  Edges
// with support < kThreshold are dropped before the BFS layering, so the
// layering follows the band.  Vertices whose two-hop neighbourhood exceeds
// kTwoHopCap (hubs) keep all their edges.  The caller (pars3_plan_create)
// keeps P only when the plan it gives needs clearly fewer shared-memory
// slots.
#include <omp.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <new>
#include <vector>

#include "common.h"
#include "locality.h"

extern "C" int pars3_pattern_from_lower(int64_t n, const int64_t *row_ptr, const int32_t *col_ind,
                                        int64_t *indptr, int32_t *indices);
extern "C" int pars3_rcm_order(int64_t n, const int64_t *indptr, const int32_t *indices,
                               int64_t *forward, int nthreads);
extern "C" int pars3_rcm_order_via_device(int64_t n, const int64_t *indptr, const int32_t *indices,
                                          int64_t *forward);
extern "C" int pars3_permute_lower(int64_t n, const int64_t *row_ptr, const int32_t *col_ind,
                                   const double *off_diags, const double *diags,
                                   const int64_t *forward, int64_t *out_row_ptr,
                                   int32_t *out_col_ind, double *out_off_diags, double *out_diags,
                                   int nthreads);

namespace pars3 {

namespace {
constexpr int kThreshold = 3;          // measured on c3 at 2^20 rows: 3 keeps the band, drops
                                       // 99.3 % of the far entries
constexpr int64_t kTwoHopCap = 1 << 14;  // two-hop work per vertex before it counts as a hub
}  // namespace

int locality_order(const pars3_split_view *s, LocalityOrder &out) {
    const int64_t n = s->n;
    const bool verbose = getenv("PARS3_VERBOSE") != nullptr;  // wall-clock of the stages on stderr
    double t_prev = omp_get_wtime();
    auto lap = [&](const char *what) {
        const double now = omp_get_wtime();
        if (verbose) fprintf(stderr, "pars3 plan:   locality: %-20s %.3f s\n", what, now - t_prev);
        t_prev = now;
    };
    {
        const char *lh = getenv("PARS3_LOCALITY_HOST");
        if (!(lh && lh[0] == '1')) {
            bool done = false;
            const int rc = locality_order_device(s, out, done);
            if (rc) return rc;
            if (done) return PARS3_OK;
        }
    }
    try {
        // 1. the split's entries as one lower CSR (outer entries of a row
        //    precede its middle ones; both ascending: split.py:116-141)
        std::vector<int64_t> optr(n + 1, 0);
        for (int64_t k = 0; k < s->outer_count; k++) optr[s->outer_row[k] + 1]++;
        for (int64_t i = 0; i < n; i++) optr[i + 1] += optr[i];
        std::vector<int64_t> rp(n + 1, 0);
        for (int64_t i = 0; i < n; i++)
            rp[i + 1] = rp[i] + (optr[i + 1] - optr[i]) + (s->mid_ptr[i + 1] - s->mid_ptr[i]);
        const int64_t m = rp[n];
        if (m == 0) {  // nothing to order: identity
            out.forward.resize(n);
            for (int64_t i = 0; i < n; i++) out.forward[i] = (int32_t)i;
            out.row_ptr.assign(n + 1, 0);
            out.col.clear();
            out.val.clear();
            out.diag.assign(s->diag, s->diag + n);
            out.dropped = 0;
            return PARS3_OK;
        }
        std::vector<int32_t> col(m);
        std::vector<double> val(m);
#pragma omp parallel for schedule(static)
        for (int64_t i = 0; i < n; i++) {
            int64_t o = rp[i];
            for (int64_t k = optr[i]; k < optr[i + 1]; k++, o++) {
                col[o] = s->outer_col[k];
                val[o] = s->outer_val[k];
            }
            for (int64_t k = s->mid_ptr[i]; k < s->mid_ptr[i + 1]; k++, o++) {
                col[o] = s->mid_col[k];
                val[o] = s->mid_val[k];
            }
        }
        // 2. symmetric pattern, ascending neighbours
        std::vector<int64_t> ip(n + 1);
        std::vector<int32_t> ix(2 * m);
        int rc = pars3_pattern_from_lower(n, rp.data(), col.data(), ip.data(), ix.data());
        if (rc) return rc;
        lap("symmetric pattern");
        // 3. cycle support of every directed edge; keep[e] is symmetric
        std::vector<uint8_t> keep(2 * m, 1);
        std::vector<uint8_t> hub(n, 0);
#pragma omp parallel for schedule(dynamic, 4096)
        for (int64_t i = 0; i < n; i++) {
            int64_t work = 0;
            for (int64_t e = ip[i]; e < ip[i + 1]; e++) work += ip[ix[e] + 1] - ip[ix[e]];
            hub[i] = work > kTwoHopCap;
        }
        // two n-sized scratch arrays per thread: cap the threads at ~2 GB
        const int nt = (int)std::max<int64_t>(
            1, std::min<int64_t>(omp_get_max_threads(), (int64_t)(2ll << 30) / (8 * std::max<int64_t>(n, 1))));
#pragma omp parallel num_threads(nt)
        {
            std::vector<int32_t> stamp(n, -1), cnt(n, 0);
#pragma omp for schedule(dynamic, 4096)
            for (int64_t i = 0; i < n; i++) {
                if (hub[i]) continue;
                const int32_t me = (int32_t)i;
                auto touch = [&](int32_t l) {
                    if (stamp[l] != me) {
                        stamp[l] = me;
                        cnt[l] = 0;
                    }
                    cnt[l]++;
                };
                for (int64_t e = ip[i]; e < ip[i + 1]; e++) {
                    const int32_t k = ix[e];
                    touch(k);
                    for (int64_t f = ip[k]; f < ip[k + 1]; f++) touch(ix[f]);
                }
                for (int64_t e = ip[i]; e < ip[i + 1]; e++) {
                    const int32_t j = ix[e];
                    if (hub[j]) continue;
                    int c = 0;
                    for (int64_t f = ip[j]; f < ip[j + 1] && c < kThreshold; f++) {
                        const int32_t l = ix[f];
                        if (l != me && stamp[l] == me) c += cnt[l] - 1;  // minus the path via k = j
                    }
                    keep[e] = c >= kThreshold;
                }
            }
        }
        lap("cycle support");
        // 4. the filtered pattern (still ascending) and its RCM order
        std::vector<int64_t> fp(n + 1, 0);
#pragma omp parallel for schedule(static)
        for (int64_t i = 0; i < n; i++) {
            int64_t c = 0;
            for (int64_t e = ip[i]; e < ip[i + 1]; e++) c += keep[e];
            fp[i + 1] = c;
        }
        for (int64_t i = 0; i < n; i++) fp[i + 1] += fp[i];
        std::vector<int32_t> fx(fp[n]);
#pragma omp parallel for schedule(static)
        for (int64_t i = 0; i < n; i++) {
            int64_t o = fp[i];
            for (int64_t e = ip[i]; e < ip[i + 1]; e++)
                if (keep[e]) fx[o++] = ix[e];
        }
        out.dropped = 2 * m - fp[n];
        if (verbose)
            fprintf(stderr, "pars3 plan:   locality: dropped %.1f %% of the directed edges\n",
                    100.0 * (double)out.dropped / (double)(2 * m));
        // most edges close no short cycle: there is no band to recover; or the
        // filter dropped next to nothing (R-MAT: its hubs keep every edge): the
        // order would be the RCM the caller's labels already are
        if ((10 * out.dropped > 6 * 2 * m || 1000 * out.dropped < 2 * m) && !getenv("PARS3_LOCALITY_ALWAYS")) {
            out.forward.clear();
            return PARS3_OK;
        }
        std::vector<int32_t>().swap(ix);
        std::vector<uint8_t>().swap(keep);
        std::vector<int64_t> fw(n);
        lap("filtered pattern");
        // (on the device when there is one: the same labels, csrc/rcm.cu)
        const char *hr = getenv("PARS3_LOCALITY_HOST_RCM");
        const bool on_device = !(hr && hr[0] == '1') &&
                               pars3_rcm_order_via_device(n, fp.data(), fx.data(), fw.data()) == PARS3_OK;
        if (!on_device) {
            rc = pars3_rcm_order(n, fp.data(), fx.data(), fw.data(), 0);
            if (rc) return rc;
        }
        lap(on_device ? "RCM (device)" : "RCM (host)");
        // 5. P A P^T (skew relabel: an entry that lands above the diagonal is
        //    stored mirrored with its sign flipped)
        out.forward.assign(fw.begin(), fw.end());
        out.row_ptr.resize(n + 1);
        out.col.resize(m);
        out.val.resize(m);
        out.diag.resize(n);
        return pars3_permute_lower(n, rp.data(), col.data(), val.data(), s->diag, fw.data(),
                                   out.row_ptr.data(), out.col.data(), out.val.data(),
                                   out.diag.data(), 0);
    } catch (const std::bad_alloc &) {
        PARS3_FAIL(PARS3_ERR_NOMEM, "locality order: out of host memory");
    }
}

}  // namespace pars3

extern "C" int pars3_locality_order(const pars3_split_view *s, int64_t *forward, int64_t *dropped) {
    if (!s || (s->n > 0 && !forward) || s->n < 0 || s->n >= INT32_MAX)
        PARS3_FAIL(PARS3_ERR_ARG, "locality_order: bad arguments");
    pars3::LocalityOrder lo;
    const int rc = pars3::locality_order(s, lo);
    if (rc) return rc;
    for (int64_t i = 0; i < s->n; i++) forward[i] = lo.forward.empty() ? i : lo.forward[i];  // (empty: no order)
    if (dropped) *dropped = lo.dropped;
    return PARS3_OK;
}
