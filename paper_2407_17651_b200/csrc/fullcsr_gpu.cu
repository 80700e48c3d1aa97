// Device builder of the row-major plan (fullcsr.h, the host builder:
// fullcsr.cpp): the full CSR of A = D + L - L^T in lanes of 16 entries, stored
// lane-interleaved per warp of 512 (k_csr, tiles.cu), its lane rows and
// row-start masks and the rows that span warps -- the host builder's arrays,
// entry for entry (tests/test_gpu_tileplan.py::test_device_full_csr).
//
// Row i lists, by ascending column: its stored outer then middle entries,
// its diagonal, then the negated mirrors -a_ri of the rows r > i that store
// column i, ascending r.  The mirrors are the lower entries sorted by column
// with a stable radix sort (the entries are enumerated in row order, so equal
// columns keep ascending rows).
#include <cuda_runtime.h>
#include <cub/cub.cuh>

#include <algorithm>
#include <cstdint>
#include <vector>

#include "common.h"
#include "fullcsr.h"
#include "fullcsr_gpu.h"

namespace pars3 {
namespace {

constexpr int kTB = 256;

#define RC(expr)                                                                                  \
    do {                                                                                          \
        cudaError_t _e = (expr);                                                                  \
        if (_e != cudaSuccess)                                                                    \
            PARS3_FAIL(PARS3_ERR_CUDA, "full CSR (device): %s: %s", #expr, cudaGetErrorString(_e)); \
    } while (0)

template <class T>
struct Buf {
    T *p = nullptr;
    ~Buf() {
        if (p) cudaFree(p);
    }
    cudaError_t alloc(size_t count) { return cudaMalloc((void **)&p, sizeof(T) * (count ? count : 1)); }
    T *release() {
        T *q = p;
        p = nullptr;
        return q;
    }
    void free_now() {
        if (p) cudaFree(p);
        p = nullptr;
    }
};

inline int blocks_for(int64_t n) { return (int)std::min<int64_t>((n + kTB - 1) / kTB, 148 * 64); }

#define GRID_LOOP(i, n) \
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < (n); i += (int64_t)gridDim.x * blockDim.x)

// position of CSR entry e in the lane-interleaved storage
__device__ __forceinline__ int64_t interleaved(int64_t e) {
    const int64_t w = e / kCsrWarp, r = e % kCsrWarp;
    return w * kCsrWarp + (r % kCsrLane) * 32 + r / kCsrLane;
}

__global__ void k_outer_ptr(int64_t n, int64_t no, const int32_t *orow, int64_t *optr) {
    GRID_LOOP(r, n + 1) {
        int64_t a = 0, b = no;
        while (a < b) {
            const int64_t m = (a + b) >> 1;
            if (orow[m] < r)
                a = m + 1;
            else
                b = m;
        }
        optr[r] = a;
    }
}
__global__ void k_up_count(int64_t m, const int32_t *col, unsigned long long *up) {
    GRID_LOOP(k, m) atomicAdd(&up[col[k]], 1ull);
}
__global__ void k_row_len(int64_t n, const int64_t *optr, const int64_t *mptr, const unsigned long long *up,
                          int64_t *len) {
    GRID_LOOP(i, n) len[i] = (optr[i + 1] - optr[i]) + (mptr[i + 1] - mptr[i]) + 1 + (int64_t)up[i];
}
// the lower entries and the diagonal of every row; the lower entries' keys for the transpose
__global__ void k_fill_lower(int64_t n, const int64_t *rp, const int64_t *optr, const int32_t *ocol,
                             const double *oval, const int64_t *mptr, const int32_t *mcol, const double *mval,
                             const double *diag, int64_t no, int32_t *col, double *val, int32_t *tkey,
                             int32_t *trow, double *tval) {
    GRID_LOOP(i, n) {
        int64_t e = rp[i];
        // (transpose list: outer entries first, then middle ones, both in row order)
        for (int64_t k = optr[i]; k < optr[i + 1]; k++, e++) {
            const int64_t p = interleaved(e);
            col[p] = ocol[k];
            val[p] = oval[k];
        }
        for (int64_t k = mptr[i]; k < mptr[i + 1]; k++, e++) {
            const int64_t p = interleaved(e);
            col[p] = mcol[k];
            val[p] = mval[k];
        }
        const int64_t p = interleaved(e);
        col[p] = (int32_t)i;
        val[p] = diag[i];
        // keys in ROW order over all entries: position rp_low(i) = optr[i] + mptr[i]
        int64_t t = optr[i] + mptr[i];
        for (int64_t k = optr[i]; k < optr[i + 1]; k++, t++) {
            tkey[t] = ocol[k];
            trow[t] = (int32_t)i;
            tval[t] = -oval[k];
        }
        for (int64_t k = mptr[i]; k < mptr[i + 1]; k++, t++) {
            tkey[t] = mcol[k];
            trow[t] = (int32_t)i;
            tval[t] = -mval[k];
        }
    }
}
// sorted by column (stable): the mirrors of column c are sorted[ustart[c] .. ustart[c + 1])
__global__ void k_fill_mirrors(int64_t n, const int64_t *rp, const int64_t *ustart, const int32_t *srow,
                               const double *sval, int32_t *col, double *val) {
    GRID_LOOP(c, n) {
        const int64_t cnt = ustart[c + 1] - ustart[c];
        int64_t e = rp[c + 1] - cnt;
        for (int64_t q = ustart[c]; q < ustart[c + 1]; q++, e++) {
            const int64_t p = interleaved(e);
            col[p] = srow[q];
            val[p] = sval[q];
        }
    }
}
__global__ void k_gather_perm(int64_t m, const int32_t *idx, const int32_t *trow, const double *tval, int32_t *srow,
                              double *sval) {
    GRID_LOOP(q, m) {
        srow[q] = trow[idx[q]];
        sval[q] = tval[idx[q]];
    }
}
__global__ void k_iota32(int64_t m, int32_t *a) {
    GRID_LOOP(k, m) a[k] = (int32_t)k;
}
__global__ void k_lanes(int64_t n, int64_t ne, int64_t nep, const int64_t *rp, int32_t *lane_row, uint32_t *lane_flags) {
    const int64_t nl = nep / kCsrLane;
    GRID_LOOP(l, nl) {
        const int64_t e0 = l * kCsrLane;
        int64_t r = n - 1;
        if (e0 < ne) {  // last row with rp[r] <= e0
            int64_t a = 0, b = n;
            while (b - a > 1) {
                const int64_t mid = (a + b) >> 1;
                if (rp[mid] <= e0)
                    a = mid;
                else
                    b = mid;
            }
            r = a;
        }
        lane_row[l] = (int32_t)r;
        uint32_t f = 0;
        for (int k = 0; k <= kCsrLane; k++) {
            const int64_t e = e0 + k;
            bool start;
            if (e >= nep)
                start = true;
            else if (e >= ne)
                start = false;
            else {
                while (r + 1 < n && rp[r + 1] <= e) r++;
                start = rp[r] == e;
            }
            if (start) f |= 1u << k;
        }
        lane_flags[l] = f;
    }
}
__global__ void k_span_flag(int64_t n, int64_t nep, const int64_t *rp, int32_t *flag) {
    GRID_LOOP(r, n) {
        const int64_t last = r + 1 < n ? rp[r + 1] - 1 : nep - 1;
        flag[r] = last / kCsrWarp > rp[r] / kCsrWarp;
    }
}
__global__ void k_span_fill(int64_t n, int64_t nep, const int64_t *rp, const int32_t *flag, const int32_t *pos,
                            int32_t *srow, int32_t *w0, int32_t *w1) {
    GRID_LOOP(r, n) {
        if (!flag[r]) continue;
        const int64_t last = r + 1 < n ? rp[r + 1] - 1 : nep - 1;
        const int32_t q = pos[r];
        srow[q] = (int32_t)r;
        w0[q] = (int32_t)(rp[r] / kCsrWarp);
        w1[q] = (int32_t)(last / kCsrWarp);
    }
}

template <class T>
int up(Buf<T> &b, const T *h, int64_t count) {
    RC(b.alloc((size_t)count));
    if (count > 0) RC(cudaMemcpy(b.p, h, sizeof(T) * (size_t)count, cudaMemcpyHostToDevice));
    return PARS3_OK;
}

template <class T>
int scan_excl(const T *in, T *out, int64_t count) {
    size_t tb = 0;
    RC(cub::DeviceScan::ExclusiveSum(nullptr, tb, in, out, (int)count));
    Buf<uint8_t> tmp;
    RC(tmp.alloc(tb));
    RC(cub::DeviceScan::ExclusiveSum(tmp.p, tb, in, out, (int)count));
    return PARS3_OK;
}

}  // namespace

void DeviceFullCsr::release() {
    void *ptrs[] = {col, val, lane_row, lane_flags, span_row, span_w0, span_w1};
    for (void *q : ptrs)
        if (q) cudaFree(q);
    *this = DeviceFullCsr();
}

int build_full_csr_device(const pars3_split_view *s, DeviceFullCsr &D, bool &done) {
    done = false;
    D = DeviceFullCsr();
    const int64_t n = s->n;
    int dev = 0;
    if (n < 1 || n >= INT32_MAX || cudaGetDevice(&dev) != cudaSuccess) {
        cudaGetLastError();
        return PARS3_OK;
    }
    const int64_t nm = s->mid_ptr ? s->mid_ptr[n] : 0, no = s->outer_count, m = nm + no;
    if (m == 0 || 2 * m + n >= INT32_MAX) return PARS3_OK;  // (int item counts in the sort and scans)
    for (int64_t e = 1; e < no; e++)
        if (s->outer_row[e] < s->outer_row[e - 1]) return PARS3_OK;  // (the host builder reports it)
    int rc;
    Buf<int64_t> mptr, optr, rp, len, ustart;
    Buf<int32_t> mcol, ocol, orow;
    Buf<double> mval, oval, diag;
    Buf<unsigned long long> upc;
    if ((rc = up(mptr, s->mid_ptr, n + 1)) || (rc = up(mcol, s->mid_col, nm)) || (rc = up(mval, s->mid_val, nm)) ||
        (rc = up(orow, s->outer_row, no)) || (rc = up(ocol, s->outer_col, no)) || (rc = up(oval, s->outer_val, no)) ||
        (rc = up(diag, s->diag, n)))
        return rc;
    const int G = blocks_for(n);
    RC(optr.alloc(n + 1));
    RC(rp.alloc(n + 1));
    RC(len.alloc(n + 1));
    RC(ustart.alloc(n + 1));
    RC(upc.alloc(n + 1));
    RC(cudaMemset(upc.p, 0, sizeof(unsigned long long) * (n + 1)));
    RC(cudaMemset(len.p + n, 0, sizeof(int64_t)));
    k_outer_ptr<<<G, kTB>>>(n, no, orow.p, optr.p);
    if (nm > 0) k_up_count<<<blocks_for(nm), kTB>>>(nm, mcol.p, upc.p);
    if (no > 0) k_up_count<<<blocks_for(no), kTB>>>(no, ocol.p, upc.p);
    k_row_len<<<G, kTB>>>(n, optr.p, mptr.p, upc.p, len.p);
    RC(cudaGetLastError());
    if ((rc = scan_excl(len.p, rp.p, n + 1)) || (rc = scan_excl((const int64_t *)upc.p, ustart.p, n + 1))) return rc;
    int64_t ne = 0;
    RC(cudaMemcpy(&ne, rp.p + n, sizeof(int64_t), cudaMemcpyDeviceToHost));
    const int64_t nep = (ne + kCsrWarp - 1) / kCsrWarp * kCsrWarp;
    Buf<int32_t> col, tkey, tkey2, trow, idx, idx2, srow;
    Buf<double> val, tval, sval;
    RC(col.alloc(nep));
    RC(val.alloc(nep));
    RC(cudaMemset(col.p, 0, sizeof(int32_t) * nep));
    RC(cudaMemset(val.p, 0, sizeof(double) * nep));
    RC(tkey.alloc(m));
    RC(tkey2.alloc(m));
    RC(trow.alloc(m));
    RC(tval.alloc(m));
    k_fill_lower<<<G, kTB>>>(n, rp.p, optr.p, ocol.p, oval.p, mptr.p, mcol.p, mval.p, diag.p, no, col.p, val.p, tkey.p,
                             trow.p, tval.p);
    RC(cudaGetLastError());
    // stable sort of the lower entries by column: row order inside a column survives
    RC(idx.alloc(m));
    RC(idx2.alloc(m));
    k_iota32<<<blocks_for(m), kTB>>>(m, idx.p);
    int bits = 1;
    while ((1ll << bits) < n) bits++;
    {
        size_t tb = 0;
        RC(cub::DeviceRadixSort::SortPairs(nullptr, tb, tkey.p, tkey2.p, idx.p, idx2.p, (int)m, 0, bits));
        Buf<uint8_t> tmp;
        RC(tmp.alloc(tb));
        RC(cub::DeviceRadixSort::SortPairs(tmp.p, tb, tkey.p, tkey2.p, idx.p, idx2.p, (int)m, 0, bits));
        RC(cudaDeviceSynchronize());
    }
    tkey.free_now();
    tkey2.free_now();
    idx.free_now();
    RC(srow.alloc(m));
    RC(sval.alloc(m));
    k_gather_perm<<<blocks_for(m), kTB>>>(m, idx2.p, trow.p, tval.p, srow.p, sval.p);
    k_fill_mirrors<<<G, kTB>>>(n, rp.p, ustart.p, srow.p, sval.p, col.p, val.p);
    RC(cudaGetLastError());
    // lanes and spans
    const int64_t nl = nep / kCsrLane;
    Buf<int32_t> lane_row, flag, pos, span_row, span_w0, span_w1;
    Buf<uint32_t> lane_flags;
    RC(lane_row.alloc(nl));
    RC(lane_flags.alloc(nl));
    k_lanes<<<blocks_for(nl), kTB>>>(n, ne, nep, rp.p, lane_row.p, lane_flags.p);
    RC(flag.alloc(n + 1));
    RC(pos.alloc(n + 1));
    RC(cudaMemset(flag.p + n, 0, sizeof(int32_t)));
    k_span_flag<<<G, kTB>>>(n, nep, rp.p, flag.p);
    RC(cudaGetLastError());
    if ((rc = scan_excl(flag.p, pos.p, n + 1))) return rc;
    int32_t nspan = 0;
    RC(cudaMemcpy(&nspan, pos.p + n, sizeof(int32_t), cudaMemcpyDeviceToHost));
    RC(span_row.alloc(nspan));
    RC(span_w0.alloc(nspan));
    RC(span_w1.alloc(nspan));
    k_span_fill<<<G, kTB>>>(n, nep, rp.p, flag.p, pos.p, span_row.p, span_w0.p, span_w1.p);
    RC(cudaGetLastError());
    RC(cudaDeviceSynchronize());
    D.n = n;
    D.ne = ne;
    D.nep = nep;
    D.nspan = nspan;
    D.col = col.release();
    D.val = val.release();
    D.lane_row = lane_row.release();
    D.lane_flags = lane_flags.release();
    D.span_row = span_row.release();
    D.span_w0 = span_w0.release();
    D.span_w1 = span_w1.release();
    done = true;
    return PARS3_OK;
}

}  // namespace pars3

// Inspection / tests (include/pars3.h): the row-major plan built on the
// device, as the host arrays pars3_full_csr_host returns (CSR order: the
// lane-interleaving undone).  Same calling convention.
extern "C" int pars3_full_csr_device(const pars3_split_view *s, int64_t *sizes, int32_t *col, double *val,
                                     int32_t *lane_row, uint32_t *lane_flags, int32_t *span_row,
                                     int32_t *span_w0, int32_t *span_w1) {
    if (!s || !sizes) PARS3_FAIL(PARS3_ERR_ARG, "null argument");
    pars3::DeviceFullCsr D;
    bool done = false;
    int rc = pars3::build_full_csr_device(s, D, done);
    if (rc) return rc;
    if (!done) PARS3_FAIL(PARS3_ERR_CUDA, "the device builder did not run (no device, or sizes beyond its counts)");
    sizes[0] = D.nep;
    sizes[1] = D.ne;
    sizes[2] = D.nep / pars3::kCsrLane;
    sizes[3] = D.nspan;
    if (col) {
        std::vector<int32_t> c(D.nep);
        std::vector<double> v(D.nep);
        const int64_t nl = D.nep / pars3::kCsrLane;
        bool ok = cudaMemcpy(c.data(), D.col, sizeof(int32_t) * D.nep, cudaMemcpyDeviceToHost) == cudaSuccess &&
                  cudaMemcpy(v.data(), D.val, sizeof(double) * D.nep, cudaMemcpyDeviceToHost) == cudaSuccess &&
                  cudaMemcpy(lane_row, D.lane_row, sizeof(int32_t) * nl, cudaMemcpyDeviceToHost) == cudaSuccess &&
                  cudaMemcpy(lane_flags, D.lane_flags, sizeof(uint32_t) * nl, cudaMemcpyDeviceToHost) == cudaSuccess;
        if (ok && D.nspan > 0)
            ok = cudaMemcpy(span_row, D.span_row, sizeof(int32_t) * D.nspan, cudaMemcpyDeviceToHost) == cudaSuccess &&
                 cudaMemcpy(span_w0, D.span_w0, sizeof(int32_t) * D.nspan, cudaMemcpyDeviceToHost) == cudaSuccess &&
                 cudaMemcpy(span_w1, D.span_w1, sizeof(int32_t) * D.nspan, cudaMemcpyDeviceToHost) == cudaSuccess;
        if (!ok) {
            D.release();
            PARS3_FAIL(PARS3_ERR_CUDA, "pars3_full_csr_device: download failed");
        }
        for (int64_t e = 0; e < D.nep; e++) {
            const int64_t w = e / pars3::kCsrWarp, r = e % pars3::kCsrWarp;
            const int64_t p = w * pars3::kCsrWarp + (r % pars3::kCsrLane) * 32 + r / pars3::kCsrLane;
            col[e] = c[p];
            val[e] = v[p];
        }
    }
    D.release();
    return PARS3_OK;
}
