/*
 * oracle.c -- CPU restatement of the reference PARS3 path.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in the product package
 * (paper_2407_17651_b200/) links, loads or calls this file.  It is imported
 * by tests/ (as the parity checker), by __graft_entry__.smoke() (checker),
 * and by bench.py's cpu_baseline / --impl reference leg (the timed CPU
 * baseline, "kind": "port").
 *
 * Every function restates one reference function operation for operation;
 * the citation is given in each header comment.  Reference root:
 * /root/reference/pkg/src/skewspmv/.  Indices are int64 and values float64,
 * as in the reference (formats.py:107-109, 192-195).  Build with
 * -ffp-contract=off so no multiply-add is contracted into an FMA: the
 * reference's numba kernels are compiled without contraction, so the serial
 * restatement below is bit-identical to reference spmv_serial.
 *
 * Pinned against the live reference by tests/golden/ (see
 * tests/golden/make_golden.py and tests/test_oracle_golden.py).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* serial.py:50-61 (_spmv_sss).  y must be zero-filled by the caller
 * (serial.py:70, y = np.zeros(m.n)). */
void oracle_spmv_sss(int64_t n, const int64_t *row_ptr, const int64_t *col_ind,
                     const double *off_diags, const double *diags,
                     const double *x, double *y)
{
    for (int64_t i = 0; i < n; i++) {
        double xi = x[i];
        double acc = diags[i] * xi;
        for (int64_t k = row_ptr[i]; k < row_ptr[i + 1]; k++) {
            int64_t c = col_ind[k];
            double v = off_diags[k];
            acc += v * x[c];
            y[c] -= v * xi;
        }
        y[i] += acc;
    }
}

/* parallel.py:60-120 (_pars3).  Same staging: per worker diagonal, safe
 * middle, conflict middle (into msg_val); then per target the apply pass in
 * apply_order; then the coordinator's sequential outer pass.  Workers run
 * as OpenMP iterations (the reference uses numba prange, parallel.py:80).
 * y must be zero-filled (parallel.py:158). */
void oracle_pars3(const int64_t *mid_ptr, const int64_t *mid_col, const double *mid_val,
                  const double *diag, int64_t outer_count, const int64_t *outer_row,
                  const int64_t *outer_col, const double *outer_val,
                  const int64_t *block_start, const int64_t *safe_start,
                  const int64_t *conflict_ptr, const int64_t *conflict_idx,
                  const int64_t *apply_order, const int64_t *apply_ptr,
                  const double *x, double *y, double *msg_val, int64_t p, int nthreads)
{
#ifdef _OPENMP
    if (nthreads < 1) nthreads = 1;
#pragma omp parallel for schedule(static, 1) num_threads(nthreads)
#endif
    for (int64_t w = 0; w < p; w++) {
        int64_t lo = block_start[w], hi = block_start[w + 1];
        for (int64_t i = lo; i < hi; i++) y[i] += diag[i] * x[i];
        for (int64_t i = lo; i < hi; i++) {
            double xi = x[i];
            for (int64_t k = safe_start[i]; k < mid_ptr[i + 1]; k++) {
                int64_t c = mid_col[k];
                double v = mid_val[k];
                y[i] += v * x[c];
                y[c] -= v * xi;
            }
        }
        int64_t cursor = conflict_ptr[w];
        for (int64_t i = lo; i < hi; i++) {
            double xi = x[i];
            for (int64_t k = mid_ptr[i]; k < safe_start[i]; k++) {
                int64_t c = mid_col[k];
                double v = mid_val[k];
                y[i] += v * x[c];
                msg_val[cursor] = -v * xi;
                cursor++;
            }
        }
    }
#ifdef _OPENMP
#pragma omp parallel for schedule(static, 1) num_threads(nthreads)
#endif
    for (int64_t t = 0; t < p; t++) {
        for (int64_t a = apply_ptr[t]; a < apply_ptr[t + 1]; a++) {
            int64_t slot = apply_order[a];
            int64_t c = mid_col[conflict_idx[slot]];
            y[c] += msg_val[slot];
        }
    }
    for (int64_t e = 0; e < outer_count; e++) {
        int64_t i = outer_row[e], c = outer_col[e];
        double v = outer_val[e];
        y[i] += v * x[c];
        y[c] -= v * x[i];
    }
}

/* Symmetrised off-diagonal adjacency of an SSS matrix: the same pattern
 * reorder.py:103-117 (pattern_from_coo) builds from the both-triangle
 * triplets of sss_to_coo(m) (formats.py:478-490), neighbours ascending.
 * indptr has n+1 entries; indices has 2*nnz entries.  Lower-storage
 * columns are strictly increasing per row (formats.py:212-217), so the
 * (i,c) pairs are unique and no dedup is needed. */
void oracle_pattern_from_sss(int64_t n, const int64_t *row_ptr, const int64_t *col_ind,
                             int64_t *indptr, int64_t *indices)
{
    int64_t *cnt = (int64_t *)calloc((size_t)n + 1, sizeof(int64_t));
    for (int64_t i = 0; i < n; i++) {
        cnt[i] += row_ptr[i + 1] - row_ptr[i];
        for (int64_t k = row_ptr[i]; k < row_ptr[i + 1]; k++) cnt[col_ind[k]]++;
    }
    indptr[0] = 0;
    for (int64_t i = 0; i < n; i++) indptr[i + 1] = indptr[i] + cnt[i];
    int64_t *fill = cnt; /* reuse */
    for (int64_t i = 0; i < n; i++) fill[i] = indptr[i];
    /* Neighbours of u: columns c<u (row u of the lower part, ascending) then
     * rows i>u holding u as a column (ascending i because rows are visited in
     * order).  Lower neighbours first, then upper: ascending overall. */
    for (int64_t u = 0; u < n; u++)
        for (int64_t k = row_ptr[u]; k < row_ptr[u + 1]; k++) indices[fill[u]++] = col_ind[k];
    for (int64_t i = 0; i < n; i++)
        for (int64_t k = row_ptr[i]; k < row_ptr[i + 1]; k++) indices[fill[col_ind[k]]++] = i;
    free(cnt);
}

/* reorder.py:137-155 (_collect_component) */
static int64_t collect_component(const int64_t *indptr, const int64_t *indices, int64_t start,
                                 uint8_t *claimed, int64_t *queue)
{
    queue[0] = start;
    claimed[start] = 1;
    int64_t head = 0, tail = 1;
    while (head < tail) {
        int64_t u = queue[head++];
        for (int64_t k = indptr[u]; k < indptr[u + 1]; k++) {
            int64_t w = indices[k];
            if (!claimed[w]) {
                claimed[w] = 1;
                queue[tail++] = w;
            }
        }
    }
    return tail;
}

/* reorder.py:158-194 (_bfs_stats): eccentricity of start and the
 * minimum-(degree, index) node of the deepest level. */
static void bfs_stats(const int64_t *indptr, const int64_t *indices, const int64_t *degree,
                      int64_t start, int64_t *level, int64_t *queue, int64_t *ecc_out,
                      int64_t *best_out)
{
    queue[0] = start;
    level[start] = 0;
    int64_t head = 0, tail = 1, ecc = 0;
    while (head < tail) {
        int64_t u = queue[head++];
        int64_t lu = level[u];
        if (lu > ecc) ecc = lu;
        for (int64_t k = indptr[u]; k < indptr[u + 1]; k++) {
            int64_t w = indices[k];
            if (level[w] < 0) {
                level[w] = lu + 1;
                queue[tail++] = w;
            }
        }
    }
    int64_t best = -1;
    for (int64_t t = 0; t < tail; t++) {
        int64_t u = queue[t];
        if (level[u] == ecc &&
            (best < 0 || degree[u] < degree[best] || (degree[u] == degree[best] && u < best)))
            best = u;
    }
    for (int64_t t = 0; t < tail; t++) level[queue[t]] = -1;
    *ecc_out = ecc;
    *best_out = best;
}

/* reorder.py:197-231 (_order_component): Cuthill-McKee with children in
 * (degree, index) order via the same insertion sort. */
static int64_t order_component(const int64_t *indptr, const int64_t *indices,
                               const int64_t *degree, int64_t start, uint8_t *placed,
                               int64_t *out, int64_t base, int64_t *buf)
{
    out[base] = start;
    placed[start] = 1;
    int64_t head = base, tail = base + 1;
    while (head < tail) {
        int64_t u = out[head++];
        int64_t cnt = 0;
        for (int64_t k = indptr[u]; k < indptr[u + 1]; k++) {
            int64_t w = indices[k];
            if (!placed[w]) {
                placed[w] = 1;
                buf[cnt++] = w;
            }
        }
        for (int64_t a = 1; a < cnt; a++) {
            int64_t wv = buf[a];
            int64_t b = a - 1;
            while (b >= 0 && (degree[buf[b]] > degree[wv] ||
                              (degree[buf[b]] == degree[wv] && buf[b] > wv))) {
                buf[b + 1] = buf[b];
                b--;
            }
            buf[b + 1] = wv;
        }
        for (int64_t a = 0; a < cnt; a++) out[tail++] = buf[a];
    }
    return tail;
}

/* reorder.py:251-286 (rcm_order) with reorder.py:234-248
 * (_pseudo_peripheral).  Writes forward[old] = new. */
void oracle_rcm_order(int64_t n, const int64_t *indptr, const int64_t *indices, int64_t *forward)
{
    int64_t *degree = (int64_t *)malloc(sizeof(int64_t) * (size_t)(n ? n : 1));
    uint8_t *claimed = (uint8_t *)calloc((size_t)(n ? n : 1), 1);
    uint8_t *placed = (uint8_t *)calloc((size_t)(n ? n : 1), 1);
    int64_t *level = (int64_t *)malloc(sizeof(int64_t) * (size_t)(n ? n : 1));
    int64_t *queue = (int64_t *)malloc(sizeof(int64_t) * (size_t)(n ? n : 1));
    int64_t *buf = (int64_t *)malloc(sizeof(int64_t) * (size_t)(n ? n : 1));
    int64_t *out = (int64_t *)malloc(sizeof(int64_t) * (size_t)(n ? n : 1));
    for (int64_t i = 0; i < n; i++) {
        degree[i] = indptr[i + 1] - indptr[i];
        level[i] = -1;
    }
    int64_t base = 0;
    for (int64_t s = 0; s < n; s++) {
        if (claimed[s]) continue;
        if (degree[s] == 0) {
            claimed[s] = 1;
            out[base++] = s;
            continue;
        }
        int64_t cnt = collect_component(indptr, indices, s, claimed, queue);
        /* _pseudo_peripheral: start from the minimum-(degree, index) member
         * (np.lexsort((members, deg_m))[0]). */
        int64_t x = queue[0];
        for (int64_t t = 1; t < cnt; t++) {
            int64_t u = queue[t];
            if (degree[u] < degree[x] || (degree[u] == degree[x] && u < x)) x = u;
        }
        int64_t ecc_x, y, ecc_y, z;
        bfs_stats(indptr, indices, degree, x, level, queue, &ecc_x, &y);
        for (;;) {
            bfs_stats(indptr, indices, degree, y, level, queue, &ecc_y, &z);
            if (ecc_y > ecc_x) {
                x = y;
                ecc_x = ecc_y;
                y = z;
            } else {
                break;
            }
        }
        base = order_component(indptr, indices, degree, x, placed, out, base, buf);
    }
    /* order = out[::-1]; forward[order] = arange(n) */
    for (int64_t k = 0; k < n; k++) forward[out[n - 1 - k]] = k;
    free(degree); free(claimed); free(placed); free(level); free(queue); free(buf); free(out);
}
