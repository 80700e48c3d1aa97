// GPU preprocessing after RCM: relabel the skyline
// arrays and split them into the middle / outer bands on the device.  Both
// produce the host-native versions' arrays bit for bit (prep.cpp), which
// match the reference's (reorder.py:289-297 + formats.py:413-475,
// split.py:116-141): the results are canonical -- each output row holds its
// unique columns ascending -- so the order of the parallel scatter does not
// matter once every row is sorted.
#include <cuda_runtime.h>
#include <cub/cub.cuh>

#include <cstdint>
#include <algorithm>
#include <vector>

#include "common.h"

namespace {

constexpr int kTB = 256;
inline int blocks_for(int64_t n) { return (int)std::min<int64_t>((n + kTB - 1) / kTB, 148 * 64); }

template <class T>
struct DevBuf {
    T *p = nullptr;
    ~DevBuf() {
        if (p) cudaFree(p);
    }
    cudaError_t alloc(size_t count) { return cudaMalloc((void **)&p, sizeof(T) * (count ? count : 1)); }
};

#define RC(expr)                                                                              \
    do {                                                                                      \
        cudaError_t _e = (expr);                                                              \
        if (_e != cudaSuccess)                                                                \
            PARS3_FAIL(PARS3_ERR_CUDA, "prep_gpu: %s: %s", #expr, cudaGetErrorString(_e));    \
    } while (0)

// entries of old row i move to new row max(f[i], f[c])
__global__ void k_perm_count(int64_t n, const int64_t *rp, const int32_t *ci, const int64_t *fw,
                             unsigned long long *cnt) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t fi = fw[i];
        for (int64_t k = rp[i]; k < rp[i + 1]; k++) {
            const int64_t fc = fw[ci[k]];
            atomicAdd(&cnt[fi > fc ? fi : fc], 1ull);
        }
    }
}

// scatter: the stored lower value of the relabelled pair is v if the row
// keeps its side, -v if the pair flips (formats.py:14-18)
__global__ void k_perm_fill(int64_t n, const int64_t *rp, const int32_t *ci, const double *od,
                            const int64_t *fw, unsigned long long *cursor, int32_t *oc, double *ov,
                            int32_t *orow) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t fi = fw[i];
        for (int64_t k = rp[i]; k < rp[i + 1]; k++) {
            const int64_t fc = fw[ci[k]];
            const bool keep = fi > fc;
            const int64_t r = keep ? fi : fc;
            const unsigned long long slot = atomicAdd(&cursor[r], 1ull);
            oc[slot] = (int32_t)(keep ? fc : fi);
            ov[slot] = keep ? od[k] : -od[k];
            orow[slot] = (int32_t)r;
        }
    }
}

__global__ void k_perm_diag(int64_t n, const double *dg, const int64_t *fw, double *odg) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        odg[fw[i]] = dg[i];
}

// sort key of an entry: (row, column) in one 64-bit word
__global__ void k_rowcol_key(int64_t m, const int32_t *row, const int32_t *col, unsigned long long *key) {
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < m; k += (int64_t)gridDim.x * blockDim.x)
        key[k] = ((unsigned long long)(uint32_t)row[k] << 32) | (uint32_t)col[k];
}

__global__ void k_col_of_key(int64_t m, const unsigned long long *key, int32_t *col) {
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < m; k += (int64_t)gridDim.x * blockDim.x)
        col[k] = (int32_t)(key[k] & 0xffffffffu);
}

// split: per row, the outer prefix (i - c > beta) and the middle suffix
__global__ void k_split_at(int64_t n, const int64_t *rp, const int32_t *ci, int64_t beta, int64_t *n_out,
                           int64_t *n_mid) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        int64_t k = rp[i];
        while (k < rp[i + 1] && i - ci[k] > beta) k++;
        n_out[i] = k - rp[i];
        n_mid[i] = rp[i + 1] - k;
    }
}

__global__ void k_split_fill(int64_t n, const int64_t *rp, const int32_t *ci, const double *od,
                             const int64_t *out_ptr, const int64_t *mid_ptr, int32_t *mc, double *mv,
                             int32_t *orow, int32_t *oc, double *ov) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t no = out_ptr[i + 1] - out_ptr[i];
        for (int64_t q = 0; q < no; q++) {
            const int64_t k = rp[i] + q, o = out_ptr[i] + q;
            orow[o] = (int32_t)i;
            oc[o] = ci[k];
            ov[o] = od[k];
        }
        for (int64_t k = rp[i] + no, q = mid_ptr[i]; k < rp[i + 1]; k++, q++) {
            mc[q] = ci[k];
            mv[q] = od[k];
        }
    }
}

}  // namespace

extern "C" int pars3_permute_lower_device(int64_t n, const int64_t *row_ptr, const int32_t *col_ind,
                                          const double *off_diags, const double *diags,
                                          const int64_t *forward, int64_t *out_row_ptr,
                                          int32_t *out_col_ind, double *out_off_diags,
                                          double *out_diags, void *stream) {
    if (n < 0 || n >= INT32_MAX || (n > 0 && (!row_ptr || !forward || !out_row_ptr)))
        PARS3_FAIL(PARS3_ERR_ARG, "permute_lower_device: bad arguments");
    cudaStream_t st = (cudaStream_t)stream;
    if (n == 0) {
        RC(cudaMemsetAsync(out_row_ptr, 0, sizeof(int64_t), st));
        return PARS3_OK;
    }
    int64_t m = 0;
    RC(cudaMemcpyAsync(&m, row_ptr + n, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    RC(cudaStreamSynchronize(st));
    const int G = blocks_for(n);
    DevBuf<unsigned long long> cnt, key, key2;
    DevBuf<int32_t> rows;
    DevBuf<double> val2;
    RC(cnt.alloc(n + 1));
    RC(cudaMemsetAsync(cnt.p, 0, sizeof(unsigned long long) * (n + 1), st));
    k_perm_count<<<G, kTB, 0, st>>>(n, row_ptr, col_ind, forward, cnt.p + 1);
    RC(cudaGetLastError());
    // out_row_ptr = inclusive scan of the counts, shifted (cnt[0] = 0)
    size_t tb = 0;
    RC(cub::DeviceScan::InclusiveSum(nullptr, tb, cnt.p, (unsigned long long *)out_row_ptr, n + 1, st));
    const int64_t mm = m > 0 ? m : 1;
    size_t tb2 = 0;
    RC(key.alloc(mm));
    RC(key2.alloc(mm));
    RC(rows.alloc(mm));
    RC(val2.alloc(mm));
    RC(cub::DeviceRadixSort::SortPairs(nullptr, tb2, key.p, key2.p, out_off_diags, val2.p, (int)mm, 0, 64, st));
    DevBuf<uint8_t> temp;
    RC(temp.alloc(std::max(tb, tb2)));
    size_t t1 = std::max(tb, tb2);
    RC(cub::DeviceScan::InclusiveSum(temp.p, t1, cnt.p, (unsigned long long *)out_row_ptr, n + 1, st));
    if (m > 0) {
        // scatter with per-row cursors, then one (row, column) radix sort of
        // all entries: rows stay in place, columns come out ascending
        RC(cudaMemcpyAsync(cnt.p, out_row_ptr, sizeof(int64_t) * n, cudaMemcpyDeviceToDevice, st));
        k_perm_fill<<<G, kTB, 0, st>>>(n, row_ptr, col_ind, off_diags, forward, cnt.p, out_col_ind,
                                       out_off_diags, rows.p);
        k_rowcol_key<<<blocks_for(m), kTB, 0, st>>>(m, rows.p, out_col_ind, key.p);
        RC(cudaGetLastError());
        size_t t2 = std::max(tb, tb2);
        RC(cub::DeviceRadixSort::SortPairs(temp.p, t2, key.p, key2.p, out_off_diags, val2.p, (int)m, 0, 64, st));
        k_col_of_key<<<blocks_for(m), kTB, 0, st>>>(m, key2.p, out_col_ind);
        RC(cudaMemcpyAsync(out_off_diags, val2.p, sizeof(double) * m, cudaMemcpyDeviceToDevice, st));
    }
    if (diags && out_diags) k_perm_diag<<<G, kTB, 0, st>>>(n, diags, forward, out_diags);
    RC(cudaGetLastError());
    RC(cudaStreamSynchronize(st));
    return PARS3_OK;
}

extern "C" int pars3_split_device(int64_t n, const int64_t *row_ptr, const int32_t *col_ind,
                                  const double *off_diags, int64_t beta, int64_t *mid_ptr,
                                  int64_t *outer_ptr, int32_t *mid_col, double *mid_val,
                                  int32_t *outer_row, int32_t *outer_col, double *outer_val,
                                  int64_t *counts, void *stream) {
    if (beta < 1) PARS3_FAIL(PARS3_ERR_ARG, "split bandwidth must be at least 1, got %lld", (long long)beta);
    if (n < 0 || !row_ptr || !mid_ptr || !outer_ptr || !counts)
        PARS3_FAIL(PARS3_ERR_ARG, "split_device: bad arguments");
    cudaStream_t st = (cudaStream_t)stream;
    RC(cudaMemsetAsync(mid_ptr, 0, sizeof(int64_t), st));
    RC(cudaMemsetAsync(outer_ptr, 0, sizeof(int64_t), st));
    if (n == 0) {
        counts[0] = counts[1] = 0;
        return PARS3_OK;
    }
    const int G = blocks_for(n);
    // per-row counts land in [1, n]; the in-place inclusive scans give the pointers
    k_split_at<<<G, kTB, 0, st>>>(n, row_ptr, col_ind, beta, outer_ptr + 1, mid_ptr + 1);
    RC(cudaGetLastError());
    size_t tb = 0;
    RC(cub::DeviceScan::InclusiveSum(nullptr, tb, mid_ptr + 1, mid_ptr + 1, n, st));
    DevBuf<uint8_t> temp;
    RC(temp.alloc(tb));
    size_t t1 = tb;
    RC(cub::DeviceScan::InclusiveSum(temp.p, t1, mid_ptr + 1, mid_ptr + 1, n, st));
    t1 = tb;
    RC(cub::DeviceScan::InclusiveSum(temp.p, t1, outer_ptr + 1, outer_ptr + 1, n, st));
    RC(cudaMemcpyAsync(&counts[0], mid_ptr + n, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    RC(cudaMemcpyAsync(&counts[1], outer_ptr + n, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    RC(cudaStreamSynchronize(st));
    if (!mid_col) return PARS3_OK;  // sizing call
    k_split_fill<<<G, kTB, 0, st>>>(n, row_ptr, col_ind, off_diags, outer_ptr, mid_ptr, mid_col, mid_val,
                                    outer_row, outer_col, outer_val);
    RC(cudaGetLastError());
    RC(cudaStreamSynchronize(st));
    return PARS3_OK;
}

namespace {
// bandwidth of a skyline matrix: columns ascend, so row i's widest entry is its first
__global__ void k_bandwidth(int64_t n, const int64_t *rp, const int32_t *ci, unsigned long long *bw) {
    unsigned long long best = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        if (rp[i + 1] > rp[i]) best = max(best, (unsigned long long)(i - ci[rp[i]]));
    for (int o = 16; o; o >>= 1) best = max(best, __shfl_xor_sync(0xffffffffu, best, o));
    if ((threadIdx.x & 31) == 0 && best) atomicMax(bw, best);
}
}  // namespace

extern "C" int pars3_bandwidth_device(int64_t n, const int64_t *row_ptr, const int32_t *col_ind,
                                      int64_t *bandwidth, void *stream) {
    if (n < 0 || !bandwidth || (n > 0 && !row_ptr)) PARS3_FAIL(PARS3_ERR_ARG, "bandwidth_device: bad arguments");
    *bandwidth = 0;
    if (n == 0) return PARS3_OK;
    cudaStream_t st = (cudaStream_t)stream;
    DevBuf<unsigned long long> d;
    RC(d.alloc(1));
    RC(cudaMemsetAsync(d.p, 0, sizeof(unsigned long long), st));
    k_bandwidth<<<blocks_for(n), kTB, 0, st>>>(n, row_ptr, col_ind, d.p);
    RC(cudaGetLastError());
    unsigned long long h = 0;
    RC(cudaMemcpyAsync(&h, d.p, sizeof(h), cudaMemcpyDeviceToHost, st));
    RC(cudaStreamSynchronize(st));
    *bandwidth = (int64_t)h;
    return PARS3_OK;
}

// ---- classify_conflicts on the device (split.py:303-361) --------------------
// A middle entry (i, c) is a conflict when its column belongs to an earlier
// block than its row (c < block_start[owner(i)]): columns ascend within a
// row, so a row's conflicts are a prefix of its middle entries.  Outputs as
// the host version (prep.cpp, pars3_classify_conflicts), bit for bit:
// conflict_idx ascending, apply_order the stable order by target block.
namespace {

__device__ __forceinline__ int owner_block(const int64_t *bs, int p, int64_t i) {
    int lo = 0, hi = p;  // bs[lo] <= i < bs[hi]
    while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (bs[mid] <= i)
            lo = mid;
        else
            hi = mid;
    }
    return lo;
}

__global__ void k_cf_count(int64_t n, const int64_t *mp, const int32_t *mc, int p, const int64_t *bs,
                           int64_t *ncf, int64_t *row_owner, int64_t *safe_start) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int w = owner_block(bs, p, i);
        const int64_t lo = bs[w];
        int64_t a = mp[i], b = mp[i + 1];  // first k in [a, b) with mc[k] >= lo
        while (a < b) {
            const int64_t mid = (a + b) >> 1;
            if (mc[mid] < lo)
                a = mid + 1;
            else
                b = mid;
        }
        ncf[i] = a - mp[i];
        if (row_owner) {
            row_owner[i] = w;
            safe_start[i] = a;
        }
    }
}

__global__ void k_cf_fill(int64_t n, const int64_t *mp, const int32_t *mc, int p, const int64_t *bs,
                          const int64_t *cfp, int64_t *conflict_idx, int64_t *conflict_target, int32_t *tkey,
                          unsigned long long *incoming, unsigned long long *halo) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t j0 = cfp[i], cnt = cfp[i + 1] - j0;
        if (cnt == 0) continue;
        const int w = owner_block(bs, p, i);
        // the row's first conflict has its smallest column
        atomicMin(&halo[w], (unsigned long long)mc[mp[i]]);
        for (int64_t q = 0; q < cnt; q++) {
            const int64_t k = mp[i] + q;
            const int t = owner_block(bs, p, mc[k]);
            conflict_idx[j0 + q] = k;
            conflict_target[j0 + q] = t;
            tkey[j0 + q] = t;
            atomicAdd(&incoming[t], 1ull);
        }
    }
}

__global__ void k_iota64(int64_t m, int64_t *a) {
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < m; k += (int64_t)gridDim.x * blockDim.x) a[k] = k;
}

__global__ void k_gather64(int p1, const int64_t *src, const int64_t *idx, int64_t *dst) {
    const int w = blockIdx.x * blockDim.x + threadIdx.x;
    if (w < p1) dst[w] = src[idx[w]];
}

}  // namespace

// Device arrays: mid_ptr [n + 1], mid_col, and the outputs row_owner [n],
// safe_start [n], conflict_idx / conflict_target / apply_order
// [conflict_count].  Host arrays: block_start [p + 1], conflict_count,
// conflict_ptr [p + 1], apply_ptr [p + 1], halo_lo [p].  Call with
// conflict_idx == NULL for the count (row_owner / safe_start optional then).
extern "C" int pars3_classify_conflicts_device(int64_t n, const int64_t *mid_ptr, const int32_t *mid_col,
                                               int64_t p, const int64_t *block_start, int64_t *conflict_count,
                                               int64_t *row_owner, int64_t *safe_start, int64_t *conflict_idx,
                                               int64_t *conflict_ptr, int64_t *conflict_target,
                                               int64_t *apply_order, int64_t *apply_ptr, int64_t *halo_lo,
                                               void *stream) {
    if (p < 1 || p > (1 << 20) || !block_start || block_start[0] != 0 || block_start[p] != n || !conflict_count)
        PARS3_FAIL(PARS3_ERR_STRUCT, "block_start must run from 0 to n over p blocks");
    for (int64_t w = 0; w < p; w++)
        if (block_start[w + 1] <= block_start[w]) PARS3_FAIL(PARS3_ERR_STRUCT, "every block must own at least one row");
    cudaStream_t st = (cudaStream_t)stream;
    DevBuf<int64_t> bs, cfp;
    RC(bs.alloc(p + 1));
    RC(cfp.alloc(n + 1));
    RC(cudaMemcpyAsync(bs.p, block_start, sizeof(int64_t) * (p + 1), cudaMemcpyHostToDevice, st));
    RC(cudaMemsetAsync(cfp.p, 0, sizeof(int64_t), st));
    const int G = blocks_for(n);
    k_cf_count<<<G, kTB, 0, st>>>(n, mid_ptr, mid_col, (int)p, bs.p, cfp.p + 1, row_owner, safe_start);
    RC(cudaGetLastError());
    size_t tb = 0;
    RC(cub::DeviceScan::InclusiveSum(nullptr, tb, cfp.p + 1, cfp.p + 1, n, st));
    DevBuf<uint8_t> temp;
    RC(temp.alloc(tb));
    RC(cub::DeviceScan::InclusiveSum(temp.p, tb, cfp.p + 1, cfp.p + 1, n, st));
    int64_t total = 0;
    RC(cudaMemcpyAsync(&total, cfp.p + n, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    RC(cudaStreamSynchronize(st));
    *conflict_count = total;
    if (!conflict_idx) return PARS3_OK;
    if (!row_owner || !safe_start || !conflict_ptr || !conflict_target || !apply_order || !apply_ptr || !halo_lo)
        PARS3_FAIL(PARS3_ERR_ARG, "classify_conflicts_device: null output");
    if (total >= INT32_MAX) PARS3_FAIL(PARS3_ERR_ARG, "classify_conflicts_device: too many conflicts");
    // conflict_ptr[w] = conflicts of the rows below block w
    DevBuf<int64_t> cpd;
    RC(cpd.alloc(p + 1));
    k_gather64<<<(int)((p + 1 + kTB - 1) / kTB), kTB, 0, st>>>((int)(p + 1), cfp.p, bs.p, cpd.p);
    RC(cudaMemcpyAsync(conflict_ptr, cpd.p, sizeof(int64_t) * (p + 1), cudaMemcpyDeviceToHost, st));
    DevBuf<unsigned long long> incoming, halo;
    RC(incoming.alloc(p));
    RC(halo.alloc(p));
    RC(cudaMemsetAsync(incoming.p, 0, sizeof(unsigned long long) * p, st));
    RC(cudaMemcpyAsync(halo.p, block_start, sizeof(int64_t) * p, cudaMemcpyHostToDevice, st));
    std::vector<unsigned long long> hin(p), hhalo(p);
    if (total > 0) {
        DevBuf<int32_t> tkey, tkey2;
        DevBuf<int64_t> iota;
        RC(tkey.alloc(total));
        RC(tkey2.alloc(total));
        RC(iota.alloc(total));
        k_cf_fill<<<G, kTB, 0, st>>>(n, mid_ptr, mid_col, (int)p, bs.p, cfp.p, conflict_idx, conflict_target,
                                     tkey.p, incoming.p, halo.p);
        k_iota64<<<blocks_for(total), kTB, 0, st>>>(total, iota.p);
        RC(cudaGetLastError());
        int bits = 1;
        while ((1ll << bits) < p) bits++;
        size_t ts = 0;
        RC(cub::DeviceRadixSort::SortPairs(nullptr, ts, tkey.p, tkey2.p, iota.p, apply_order, (int)total, 0, bits, st));
        DevBuf<uint8_t> temp2;
        RC(temp2.alloc(ts));
        RC(cub::DeviceRadixSort::SortPairs(temp2.p, ts, tkey.p, tkey2.p, iota.p, apply_order, (int)total, 0, bits, st));
        RC(cudaStreamSynchronize(st));  // (the temporaries are freed on return)
    }
    RC(cudaMemcpyAsync(hin.data(), incoming.p, sizeof(unsigned long long) * p, cudaMemcpyDeviceToHost, st));
    RC(cudaMemcpyAsync(hhalo.data(), halo.p, sizeof(unsigned long long) * p, cudaMemcpyDeviceToHost, st));
    RC(cudaStreamSynchronize(st));
    apply_ptr[0] = 0;
    for (int64_t w = 0; w < p; w++) {
        apply_ptr[w + 1] = apply_ptr[w] + (int64_t)hin[w];
        halo_lo[w] = (int64_t)hhalo[w];
    }
    return PARS3_OK;
}
