// Host-native preprocessing of the PARS3 pipeline (C ABI, see include/pars3.h).
//
// These replace the reference's numpy/numba preprocessing stages
// (reorder.py, split.py, formats.py) with multithreaded C++ that scales to
// the 16.7 M-row configuration: the reference chain needs ~25 min and
// ~70 GB there.  Outputs are bit-identical to
// the reference's (tests/test_prep_parity.py, tests/golden/).
//
// RCM is computed level-synchronously rather than with the reference's
// queue walk (reorder.py:197-231): a node of BFS level L+1 is placed by the
// first level-L node (in placement order) that sees it, and children of one
// parent are placed by (degree, index).  So level L+1, sorted by
// (position of its minimum-position level-L neighbour, degree, index), is
// exactly the reference's Cuthill-McKee order -- and every level can be
// expanded in parallel.
#include <omp.h>

#include <algorithm>
#include <climits>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <new>
#include <vector>

#include "common.h"

namespace {

int threads_for(int nthreads) { return nthreads > 0 ? nthreads : omp_get_max_threads(); }

inline bool cas_i32(int32_t *p, int32_t expect, int32_t desired) {
    return __atomic_compare_exchange_n(p, &expect, desired, false, __ATOMIC_RELAXED,
                                       __ATOMIC_RELAXED);
}

inline void atomic_min_i64(int64_t *p, int64_t v) {
    int64_t cur = __atomic_load_n(p, __ATOMIC_RELAXED);
    while (v < cur &&
           !__atomic_compare_exchange_n(p, &cur, v, false, __ATOMIC_RELAXED, __ATOMIC_RELAXED)) {
    }
}

struct Graph {
    int64_t n;
    const int64_t *indptr;
    const int32_t *indices;
    std::vector<int32_t> degree;
};

// Expand one BFS frontier in parallel.  `mark[w] == unset` means unvisited;
// the winner of the CAS owns w.  Returns the next frontier (unordered).
void expand(const Graph &g, const std::vector<int32_t> &frontier, int32_t *mark, int32_t unset,
            int32_t value, std::vector<int32_t> &next, int nt) {
    next.clear();
    const int64_t f = (int64_t)frontier.size();
    if (f < 4096 || nt == 1) {
        for (int64_t t = 0; t < f; t++) {
            int32_t u = frontier[t];
            for (int64_t k = g.indptr[u]; k < g.indptr[u + 1]; k++) {
                int32_t w = g.indices[k];
                if (mark[w] == unset) {
                    mark[w] = value;
                    next.push_back(w);
                }
            }
        }
        return;
    }
    std::vector<std::vector<int32_t>> local(nt);
#pragma omp parallel num_threads(nt)
    {
        std::vector<int32_t> &mine = local[omp_get_thread_num()];
#pragma omp for schedule(dynamic, 256)
        for (int64_t t = 0; t < f; t++) {
            int32_t u = frontier[t];
            for (int64_t k = g.indptr[u]; k < g.indptr[u + 1]; k++) {
                int32_t w = g.indices[k];
                if (__atomic_load_n(&mark[w], __ATOMIC_RELAXED) == unset && cas_i32(&mark[w], unset, value))
                    mine.push_back(w);
            }
        }
    }
    for (auto &v : local) next.insert(next.end(), v.begin(), v.end());
}

// Level structure from `start` (reorder.py:158-194, _bfs_stats): returns
// the eccentricity and the minimum-(degree, index) node of the deepest
// level.  `level` is -1 on entry for the component and restored on exit.
void bfs_stats(const Graph &g, int32_t start, int32_t *level, int nt, int64_t *ecc_out,
               int32_t *best_out) {
    std::vector<int32_t> cur{start}, next, visited{start};
    level[start] = 0;
    int32_t depth = 0;
    std::vector<int32_t> last = cur;
    while (true) {
        expand(g, cur, level, -1, depth + 1, next, nt);
        if (next.empty()) break;
        depth++;
        visited.insert(visited.end(), next.begin(), next.end());
        cur.swap(next);
        last = cur;
    }
    int32_t best = -1;
    for (int32_t u : last) {
        if (best < 0 || g.degree[u] < g.degree[best] ||
            (g.degree[u] == g.degree[best] && u < best))
            best = u;
    }
    for (int32_t u : visited) level[u] = -1;
    *ecc_out = depth;
    *best_out = best;
}

}  // namespace

extern "C" int pars3_pattern_from_lower(int64_t n, const int64_t *row_ptr, const int32_t *col_ind,
                                        int64_t *indptr, int32_t *indices) {
    if (n < 0 || !row_ptr || !indptr) PARS3_FAIL(PARS3_ERR_ARG, "pattern_from_lower: bad arguments");
    std::vector<int64_t> cnt(n + 1, 0);
    for (int64_t i = 0; i < n; i++) {
        cnt[i] += row_ptr[i + 1] - row_ptr[i];
        for (int64_t k = row_ptr[i]; k < row_ptr[i + 1]; k++) {
            int32_t c = col_ind[k];
            if (c < 0 || c >= i) PARS3_FAIL(PARS3_ERR_STRUCT, "column %d of row %lld is not strictly lower", c, (long long)i);
            cnt[c]++;
        }
    }
    indptr[0] = 0;
    for (int64_t i = 0; i < n; i++) indptr[i + 1] = indptr[i] + cnt[i];
    // Lower neighbours (ascending, < u) first, then the rows i > u that hold
    // u as a column, visited in ascending i: the merged list is ascending.
    std::vector<int64_t> fill(indptr, indptr + n);
#pragma omp parallel for schedule(static)
    for (int64_t u = 0; u < n; u++) {
        int64_t o = fill[u];
        for (int64_t k = row_ptr[u]; k < row_ptr[u + 1]; k++) indices[o++] = col_ind[k];
        fill[u] = o;
    }
    for (int64_t i = 0; i < n; i++)
        for (int64_t k = row_ptr[i]; k < row_ptr[i + 1]; k++) indices[fill[col_ind[k]]++] = (int32_t)i;
    return PARS3_OK;
}

extern "C" int pars3_rcm_order(int64_t n, const int64_t *indptr, const int32_t *indices,
                               int64_t *forward, int nthreads) {
    if (n < 0 || (n > 0 && (!indptr || !forward))) PARS3_FAIL(PARS3_ERR_ARG, "rcm_order: bad arguments");
    if (n >= INT32_MAX) PARS3_FAIL(PARS3_ERR_ARG, "rcm_order: n too large for int32 labels");
    const int nt = threads_for(nthreads);
    try {
        Graph g{n, indptr, indices, std::vector<int32_t>(n)};
#pragma omp parallel for num_threads(nt) schedule(static)
        for (int64_t u = 0; u < n; u++) g.degree[u] = (int32_t)(indptr[u + 1] - indptr[u]);

        std::vector<int32_t> claim(n, 0);    // component flood marks
        std::vector<int32_t> level(n, -1);   // bfs_stats scratch
        std::vector<int64_t> pos(n, -1);     // Cuthill-McKee position (global)
        std::vector<int64_t> parent(n, INT64_MAX);
        std::vector<int32_t> out(n);
        std::vector<int32_t> cur, next, members;
        int64_t base = 0;
        for (int64_t s = 0; s < n; s++) {
            if (claim[s]) continue;
            if (g.degree[s] == 0) {  // isolated node: appended in scan order (reorder.py:274-278)
                claim[s] = 1;
                out[base++] = (int32_t)s;
                continue;
            }
            // component flood (reorder.py:137-155)
            members.assign(1, (int32_t)s);
            claim[s] = 1;
            cur.assign(1, (int32_t)s);
            while (!cur.empty()) {
                expand(g, cur, claim.data(), 0, 1, next, nt);
                members.insert(members.end(), next.begin(), next.end());
                cur.swap(next);
            }
            // pseudo-peripheral start (reorder.py:234-248)
            int32_t x = members[0];
            for (int32_t u : members)
                if (g.degree[u] < g.degree[x] || (g.degree[u] == g.degree[x] && u < x)) x = u;
            int64_t ecc_x, ecc_y;
            int32_t y, z;
            bfs_stats(g, x, level.data(), nt, &ecc_x, &y);
            for (;;) {
                bfs_stats(g, y, level.data(), nt, &ecc_y, &z);
                if (ecc_y > ecc_x) {
                    x = y;
                    ecc_x = ecc_y;
                    y = z;
                } else {
                    break;
                }
            }
            // level-synchronous Cuthill-McKee (equivalent to reorder.py:197-231)
            pos[x] = base;
            out[base++] = x;
            cur.assign(1, x);
            while (!cur.empty()) {
                next.clear();
                const int64_t f = (int64_t)cur.size();
                std::vector<std::vector<int32_t>> local(nt);
#pragma omp parallel num_threads(nt) if (f > 2048)
                {
                    std::vector<int32_t> &mine = local[omp_get_thread_num()];
#pragma omp for schedule(dynamic, 256)
                    for (int64_t t = 0; t < f; t++) {
                        int32_t u = cur[t];
                        int64_t pu = pos[u];
                        for (int64_t k = indptr[u]; k < indptr[u + 1]; k++) {
                            int32_t w = indices[k];
                            if (__atomic_load_n(&pos[w], __ATOMIC_RELAXED) >= 0) continue;
                            int64_t old = __atomic_load_n(&parent[w], __ATOMIC_RELAXED);
                            if (old == INT64_MAX &&
                                __atomic_compare_exchange_n(&parent[w], &old, pu, false,
                                                            __ATOMIC_RELAXED, __ATOMIC_RELAXED)) {
                                mine.push_back(w);  // first visitor records the candidate
                            } else {
                                atomic_min_i64(&parent[w], pu);
                            }
                        }
                    }
                }
                for (auto &v : local) next.insert(next.end(), v.begin(), v.end());
                const int32_t *deg = g.degree.data();
                const int64_t *par = parent.data();
                std::sort(next.begin(), next.end(), [deg, par](int32_t a, int32_t b) {
                    if (par[a] != par[b]) return par[a] < par[b];
                    if (deg[a] != deg[b]) return deg[a] < deg[b];
                    return a < b;
                });
                for (int32_t w : next) {
                    pos[w] = base;
                    out[base++] = w;
                }
                cur.swap(next);
            }
        }
        // reverse the complete labeling (reorder.py:283-285)
#pragma omp parallel for num_threads(nt) schedule(static)
        for (int64_t k = 0; k < n; k++) forward[out[n - 1 - k]] = k;
    } catch (const std::bad_alloc &) {
        PARS3_FAIL(PARS3_ERR_NOMEM, "rcm_order: out of host memory");
    }
    return PARS3_OK;
}

extern "C" int pars3_permute_lower(int64_t n, const int64_t *row_ptr, const int32_t *col_ind,
                                   const double *off_diags, const double *diags,
                                   const int64_t *forward, int64_t *out_row_ptr,
                                   int32_t *out_col_ind, double *out_off_diags, double *out_diags,
                                   int nthreads) {
    if (n < 0 || !row_ptr || !forward || !out_row_ptr) PARS3_FAIL(PARS3_ERR_ARG, "permute_lower: bad arguments");
    const int nt = threads_for(nthreads);
    const int64_t m = row_ptr[n];
    try {
        std::vector<int64_t> cnt(n + 1, 0);
#pragma omp parallel for num_threads(nt) schedule(static)
        for (int64_t i = 0; i < n; i++) {
            const int64_t fi = forward[i];
            for (int64_t k = row_ptr[i]; k < row_ptr[i + 1]; k++) {
                const int64_t fc = forward[col_ind[k]];
                __atomic_fetch_add(&cnt[fi > fc ? fi : fc], 1, __ATOMIC_RELAXED);
            }
        }
        out_row_ptr[0] = 0;
        for (int64_t i = 0; i < n; i++) out_row_ptr[i + 1] = out_row_ptr[i] + cnt[i];
        std::vector<int64_t> cursor(out_row_ptr, out_row_ptr + n);
#pragma omp parallel for num_threads(nt) schedule(static)
        for (int64_t i = 0; i < n; i++) {
            const int64_t fi = forward[i];
            for (int64_t k = row_ptr[i]; k < row_ptr[i + 1]; k++) {
                const int64_t fc = forward[col_ind[k]];
                // the stored lower value of the relabelled pair: A[fi,fc] = v,
                // A[fc,fi] = -v (formats.py:14-18)
                const bool keep = fi > fc;
                const int64_t r = keep ? fi : fc;
                const int64_t slot = __atomic_fetch_add(&cursor[r], 1, __ATOMIC_RELAXED);
                out_col_ind[slot] = (int32_t)(keep ? fc : fi);
                out_off_diags[slot] = keep ? off_diags[k] : -off_diags[k];
            }
        }
        // columns ascending within each row (unique, so the order is canonical)
#pragma omp parallel num_threads(nt)
        {
            std::vector<std::pair<int32_t, double>> buf;
#pragma omp for schedule(dynamic, 1024)
            for (int64_t r = 0; r < n; r++) {
                const int64_t lo = out_row_ptr[r], hi = out_row_ptr[r + 1];
                if (hi - lo < 2) continue;
                buf.resize(hi - lo);
                for (int64_t k = lo; k < hi; k++) buf[k - lo] = {out_col_ind[k], out_off_diags[k]};
                std::sort(buf.begin(), buf.end(),
                          [](const std::pair<int32_t, double> &a, const std::pair<int32_t, double> &b) {
                              return a.first < b.first;
                          });
                for (int64_t k = lo; k < hi; k++) {
                    out_col_ind[k] = buf[k - lo].first;
                    out_off_diags[k] = buf[k - lo].second;
                }
            }
        }
        if (diags && out_diags) {
#pragma omp parallel for num_threads(nt) schedule(static)
            for (int64_t i = 0; i < n; i++) out_diags[forward[i]] = diags[i];
        }
        (void)m;
    } catch (const std::bad_alloc &) {
        PARS3_FAIL(PARS3_ERR_NOMEM, "permute_lower: out of host memory");
    }
    return PARS3_OK;
}

extern "C" int pars3_split_count(int64_t n, const int64_t *row_ptr, const int32_t *col_ind,
                                 int64_t beta, int64_t *mid_count, int64_t *outer_count) {
    if (beta < 1) PARS3_FAIL(PARS3_ERR_ARG, "split bandwidth must be at least 1, got %lld", (long long)beta);
    int64_t mid = 0;
#pragma omp parallel for schedule(static) reduction(+ : mid)
    for (int64_t i = 0; i < n; i++)
        for (int64_t k = row_ptr[i]; k < row_ptr[i + 1]; k++) mid += (i - col_ind[k] <= beta);
    *mid_count = mid;
    *outer_count = row_ptr[n] - mid;
    return PARS3_OK;
}

extern "C" int pars3_split_fill(int64_t n, const int64_t *row_ptr, const int32_t *col_ind,
                                const double *off_diags, int64_t beta, int64_t *mid_ptr,
                                int32_t *mid_col, double *mid_val, int32_t *outer_row,
                                int32_t *outer_col, double *outer_val) {
    if (beta < 1) PARS3_FAIL(PARS3_ERR_ARG, "split bandwidth must be at least 1, got %lld", (long long)beta);
    // Columns ascend within a row, so a row's outer entries (i - c > beta)
    // are a prefix and its middle entries the suffix.
    std::vector<int64_t> outer_ptr(n + 1, 0);
    mid_ptr[0] = 0;
    std::vector<int64_t> split_at(n);
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; i++) {
        int64_t k = row_ptr[i];
        while (k < row_ptr[i + 1] && i - col_ind[k] > beta) k++;
        split_at[i] = k;
    }
    for (int64_t i = 0; i < n; i++) {
        outer_ptr[i + 1] = outer_ptr[i] + (split_at[i] - row_ptr[i]);
        mid_ptr[i + 1] = mid_ptr[i] + (row_ptr[i + 1] - split_at[i]);
    }
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; i++) {
        int64_t o = outer_ptr[i];
        for (int64_t k = row_ptr[i]; k < split_at[i]; k++, o++) {
            outer_row[o] = (int32_t)i;
            outer_col[o] = col_ind[k];
            outer_val[o] = off_diags[k];
        }
        int64_t q = mid_ptr[i];
        for (int64_t k = split_at[i]; k < row_ptr[i + 1]; k++, q++) {
            mid_col[q] = col_ind[k];
            mid_val[q] = off_diags[k];
        }
    }
    return PARS3_OK;
}

extern "C" int pars3_classify_conflicts(int64_t n, const int64_t *mid_ptr, const int32_t *mid_col,
                                        int64_t p, const int64_t *block_start,
                                        int64_t *conflict_count, int64_t *row_owner,
                                        int64_t *safe_start, int64_t *conflict_idx,
                                        int64_t *conflict_ptr, int64_t *conflict_target,
                                        int64_t *apply_order, int64_t *apply_ptr,
                                        int64_t *halo_lo) {
    if (p < 1 || !block_start || block_start[0] != 0 || block_start[p] != n)
        PARS3_FAIL(PARS3_ERR_STRUCT, "block_start must run from 0 to n over p blocks");
    for (int64_t w = 0; w < p; w++)
        if (block_start[w + 1] <= block_start[w]) PARS3_FAIL(PARS3_ERR_STRUCT, "every block must own at least one row");
    // conflicts of row i: the prefix of its middle columns below its block start
    std::vector<int64_t> ncf(n);
    std::vector<int64_t> owner(n);
    for (int64_t w = 0; w < p; w++)
        for (int64_t i = block_start[w]; i < block_start[w + 1]; i++) owner[i] = w;
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; i++) {
        const int64_t lo = block_start[owner[i]];
        int64_t k = mid_ptr[i];
        while (k < mid_ptr[i + 1] && mid_col[k] < lo) k++;
        ncf[i] = k - mid_ptr[i];
    }
    int64_t total = 0;
    for (int64_t i = 0; i < n; i++) total += ncf[i];
    *conflict_count = total;
    if (!conflict_idx) return PARS3_OK;
    for (int64_t i = 0; i < n; i++) {
        row_owner[i] = owner[i];
        safe_start[i] = mid_ptr[i] + ncf[i];
    }
    // conflict_idx ascending; sources are contiguous because owners ascend with rows
    int64_t c = 0;
    for (int64_t w = 0; w <= p; w++) conflict_ptr[w] = 0;
    for (int64_t i = 0; i < n; i++) {
        for (int64_t k = mid_ptr[i]; k < mid_ptr[i] + ncf[i]; k++) conflict_idx[c++] = k;
        conflict_ptr[owner[i] + 1] += ncf[i];
    }
    for (int64_t w = 0; w < p; w++) conflict_ptr[w + 1] += conflict_ptr[w];
    std::vector<int64_t> cnt(p + 1, 0);
    for (int64_t j = 0; j < total; j++) {
        conflict_target[j] = owner[mid_col[conflict_idx[j]]];
        cnt[conflict_target[j] + 1]++;
    }
    for (int64_t w = 0; w < p; w++) cnt[w + 1] += cnt[w];
    for (int64_t w = 0; w <= p; w++) apply_ptr[w] = cnt[w];
    for (int64_t j = 0; j < total; j++) apply_order[cnt[conflict_target[j]]++] = j;  // stable
    for (int64_t w = 0; w < p; w++) {
        halo_lo[w] = block_start[w];
        for (int64_t j = conflict_ptr[w]; j < conflict_ptr[w + 1]; j++)
            halo_lo[w] = std::min<int64_t>(halo_lo[w], mid_col[conflict_idx[j]]);
    }
    return PARS3_OK;
}
