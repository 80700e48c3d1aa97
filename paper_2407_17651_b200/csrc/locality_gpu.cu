// The internal locality order (locality.cpp) computed
// on the device: the same filter, the same labels and the same P A P^T as the
// host version, bit for bit (tests/test_gpu_locality.py).
//
//   1. the split's entries as one lower CSR;
//   2. the symmetric pattern with ascending neighbour lists (degree counts,
//      a scan, a scatter with cursors, one segmented sort);
//   3. the cycle support of every directed edge (i, j): the paths i-l-j and
//      i-k-l-j, counted as  sum over l in N(j), l != i, of
//      [l in N(i)] + |N(i) /\ N(l)| - 1  (the -1 is the path through k = j);
//      this is the host's stamp-and-count written as sorted-list
//      intersections: one warp per vertex, one lane per neighbour, the sum
//      stops at the threshold; hubs (two-hop work over the cap) keep every
//      edge;
//   4. the filtered pattern, its RCM order (csrc/rcm.cu: the host RCM's
//      labels), and the skew relabel (csrc/prep_gpu.cu).
#include <cuda_runtime.h>
#include <cub/cub.cuh>
#include <omp.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstdlib>

#include "common.h"
#include "locality.h"

namespace pars3 {
namespace {

constexpr int kThreshold = 3;            // (locality.cpp)
constexpr long long kTwoHopCap = 1 << 14;
constexpr int kTB = 256;

#define RC(expr)                                                                                     \
    do {                                                                                             \
        cudaError_t _e = (expr);                                                                     \
        if (_e != cudaSuccess)                                                                       \
            PARS3_FAIL(PARS3_ERR_CUDA, "locality order (device): %s: %s", #expr, cudaGetErrorString(_e)); \
    } while (0)

template <class T>
struct Buf {
    T *p = nullptr;
    ~Buf() {
        if (p) cudaFree(p);
    }
    cudaError_t alloc(size_t count) { return cudaMalloc((void **)&p, sizeof(T) * (count ? count : 1)); }
    void free_now() {
        if (p) cudaFree(p);
        p = nullptr;
    }
};

inline int blocks_for(int64_t n) { return (int)std::min<int64_t>((n + kTB - 1) / kTB, 148 * 64); }

#define GRID_LOOP(i, n) \
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < (n); i += (int64_t)gridDim.x * blockDim.x)

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
__global__ void k_row_counts(int64_t n, const int64_t *optr, const int64_t *mptr, int64_t *cnt) {
    GRID_LOOP(i, n) cnt[i] = (optr[i + 1] - optr[i]) + (mptr[i + 1] - mptr[i]);
}
// outer entries of a row precede its middle ones (both ascending: split.py:116-141)
__global__ void k_merge_rows(int64_t n, const int64_t *rp, const int64_t *optr, const int32_t *ocol,
                             const double *oval, const int64_t *mptr, const int32_t *mcol, const double *mval,
                             int32_t *col, double *val) {
    GRID_LOOP(i, n) {
        int64_t o = rp[i];
        for (int64_t k = optr[i]; k < optr[i + 1]; k++, o++) {
            col[o] = ocol[k];
            val[o] = oval[k];
        }
        for (int64_t k = mptr[i]; k < mptr[i + 1]; k++, o++) {
            col[o] = mcol[k];
            val[o] = mval[k];
        }
    }
}
__global__ void k_degree(int64_t n, const int64_t *rp, const int32_t *col, unsigned long long *deg) {
    GRID_LOOP(i, n) {
        atomicAdd(&deg[i], (unsigned long long)(rp[i + 1] - rp[i]));
        for (int64_t k = rp[i]; k < rp[i + 1]; k++) atomicAdd(&deg[col[k]], 1ull);
    }
}
__global__ void k_scatter(int64_t n, const int64_t *rp, const int32_t *col, unsigned long long *cur, int32_t *ix) {
    GRID_LOOP(i, n) {
        const int64_t nl = rp[i + 1] - rp[i];
        const unsigned long long o = atomicAdd(&cur[i], (unsigned long long)nl);
        for (int64_t k = 0; k < nl; k++) {
            const int32_t c = col[rp[i] + k];
            ix[o + k] = c;
            ix[atomicAdd(&cur[c], 1ull)] = (int32_t)i;
        }
    }
}
__global__ void k_hub(int64_t n, const int64_t *ip, const int32_t *ix, uint8_t *hub) {
    GRID_LOOP(i, n) {
        long long work = 0;
        for (int64_t e = ip[i]; e < ip[i + 1]; e++) work += ip[ix[e] + 1] - ip[ix[e]];
        hub[i] = work > kTwoHopCap;
    }
}

// |A /\ B| of two ascending lists
__device__ __forceinline__ int intersect_count(const int32_t *a, int na, const int32_t *b, int nb) {
    int i = 0, j = 0, c = 0;
    while (i < na && j < nb) {
        const int32_t x = a[i], y = b[j];
        c += x == y;
        i += x <= y;
        j += y <= x;
    }
    return c;
}
__device__ __forceinline__ bool contains(const int32_t *a, int na, int32_t v) {
    int lo = 0, hi = na;
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (a[mid] < v)
            lo = mid + 1;
        else
            hi = mid;
    }
    return lo < na && a[lo] == v;
}

// one warp per vertex i, one lane per directed edge (i, j)
__global__ void __launch_bounds__(kTB) k_support(int64_t n, const int64_t *ip, const int32_t *ix,
                                                 const uint8_t *hub, uint8_t *keep) {
    const int lane = threadIdx.x & 31;
    const int64_t wstride = (int64_t)gridDim.x * (kTB / 32);
    for (int64_t i = blockIdx.x * (int64_t)(kTB / 32) + (threadIdx.x >> 5); i < n; i += wstride) {
        const int64_t e0 = ip[i], e1 = ip[i + 1];
        const int32_t *Ni = ix + e0;
        const int ni = (int)(e1 - e0);
        const bool hi = hub[i] != 0;
        for (int64_t e = e0 + lane; e < e1; e += 32) {
            const int32_t j = ix[e];
            if (hi || hub[j]) {
                keep[e] = 1;
                continue;
            }
            int c = 0;
            for (int64_t f = ip[j]; f < ip[j + 1] && c < kThreshold; f++) {
                const int32_t l = ix[f];
                if (l == (int32_t)i) continue;
                const int cnt = intersect_count(Ni, ni, ix + ip[l], (int)(ip[l + 1] - ip[l])) +
                                (contains(Ni, ni, l) ? 1 : 0);
                c += cnt - 1;  // minus the path via k = j
            }
            keep[e] = c >= kThreshold;
        }
    }
}
__global__ void k_keep_count(int64_t n, const int64_t *ip, const uint8_t *keep, int64_t *cnt) {
    GRID_LOOP(i, n) {
        int64_t c = 0;
        for (int64_t e = ip[i]; e < ip[i + 1]; e++) c += keep[e];
        cnt[i] = c;
    }
}
__global__ void k_keep_fill(int64_t n, const int64_t *ip, const int32_t *ix, const uint8_t *keep,
                            const int64_t *fp, int32_t *fx) {
    GRID_LOOP(i, n) {
        int64_t o = fp[i];
        for (int64_t e = ip[i]; e < ip[i + 1]; e++)
            if (keep[e]) fx[o++] = ix[e];
    }
}

int exclusive_scan64(const int64_t *in, int64_t *out, int64_t count) {  // count items -> out[0 .. count)
    size_t tb = 0;
    RC(cub::DeviceScan::ExclusiveSum(nullptr, tb, in, out, (int)count));
    Buf<uint8_t> tmp;
    RC(tmp.alloc(tb));
    RC(cub::DeviceScan::ExclusiveSum(tmp.p, tb, in, out, (int)count));
    return PARS3_OK;
}

template <class T>
int up(Buf<T> &b, const T *h, int64_t count) {
    RC(b.alloc((size_t)count));
    if (count > 0) RC(cudaMemcpy(b.p, h, sizeof(T) * (size_t)count, cudaMemcpyHostToDevice));
    return PARS3_OK;
}

}  // namespace

// done = false: no device (or nothing to do there): the caller runs the host version
int locality_order_device(const pars3_split_view *s, LocalityOrder &out, bool &done) {
    done = false;
    const int64_t n = s->n;
    int dev = 0;
    if (n < 2 || n >= INT32_MAX || cudaGetDevice(&dev) != cudaSuccess) {
        cudaGetLastError();
        return PARS3_OK;
    }
    const bool verbose = getenv("PARS3_VERBOSE") != nullptr;
    double t_prev = omp_get_wtime();
    auto lap = [&](const char *what) {
        if (!verbose) return;
        cudaDeviceSynchronize();
        const double now = omp_get_wtime();
        fprintf(stderr, "pars3 plan:   locality (device): %-18s %.3f s\n", what, now - t_prev);
        t_prev = now;
    };
    const int64_t nm = s->mid_ptr ? s->mid_ptr[n] : 0, no = s->outer_count;
    const int64_t m = nm + no;
    if (m == 0 || 2 * m >= INT32_MAX) return PARS3_OK;  // (the segmented sort counts items in int)
    int rc;
    // 1. one lower CSR
    Buf<int64_t> mptr, optr, rp, cnt;
    Buf<int32_t> mcol, ocol, orow, col;
    Buf<double> mval, oval, val, diag;
    if ((rc = up(mptr, s->mid_ptr, n + 1)) || (rc = up(mcol, s->mid_col, nm)) || (rc = up(mval, s->mid_val, nm)) ||
        (rc = up(orow, s->outer_row, no)) || (rc = up(ocol, s->outer_col, no)) || (rc = up(oval, s->outer_val, no)) ||
        (rc = up(diag, s->diag, n)))
        return rc;
    RC(optr.alloc(n + 1));
    RC(rp.alloc(n + 1));
    RC(cnt.alloc(n + 1));
    RC(col.alloc(m));
    RC(val.alloc(m));
    const int G = blocks_for(n);
    k_outer_ptr<<<G, kTB>>>(n, no, orow.p, optr.p);
    RC(cudaMemset(cnt.p + n, 0, sizeof(int64_t)));
    k_row_counts<<<G, kTB>>>(n, optr.p, mptr.p, cnt.p);
    if ((rc = exclusive_scan64(cnt.p, rp.p, n + 1))) return rc;
    k_merge_rows<<<G, kTB>>>(n, rp.p, optr.p, ocol.p, oval.p, mptr.p, mcol.p, mval.p, col.p, val.p);
    RC(cudaGetLastError());
    mcol.free_now();
    mval.free_now();
    orow.free_now();
    ocol.free_now();
    oval.free_now();
    lap("lower CSR");
    // 2. symmetric pattern, ascending neighbours
    Buf<unsigned long long> deg;
    Buf<int64_t> ip;
    Buf<int32_t> ix, ix2;
    RC(deg.alloc(n + 1));
    RC(ip.alloc(n + 1));
    RC(ix.alloc(2 * m));
    RC(ix2.alloc(2 * m));
    RC(cudaMemset(deg.p, 0, sizeof(unsigned long long) * (n + 1)));
    k_degree<<<G, kTB>>>(n, rp.p, col.p, deg.p);
    if ((rc = exclusive_scan64((const int64_t *)deg.p, ip.p, n + 1))) return rc;
    RC(cudaMemcpy(deg.p, ip.p, sizeof(int64_t) * n, cudaMemcpyDeviceToDevice));  // cursors
    k_scatter<<<G, kTB>>>(n, rp.p, col.p, deg.p, ix2.p);
    RC(cudaGetLastError());
    {
        size_t tb = 0;
        RC(cub::DeviceSegmentedSort::SortKeys(nullptr, tb, ix2.p, ix.p, (int)(2 * m), (int)n, ip.p, ip.p + 1));
        Buf<uint8_t> tmp;
        RC(tmp.alloc(tb));
        RC(cub::DeviceSegmentedSort::SortKeys(tmp.p, tb, ix2.p, ix.p, (int)(2 * m), (int)n, ip.p, ip.p + 1));
        RC(cudaDeviceSynchronize());
    }
    ix2.free_now();
    deg.free_now();
    lap("symmetric pattern");
    // 3. cycle support -> keep
    Buf<uint8_t> hub, keep;
    RC(hub.alloc(n));
    RC(keep.alloc(2 * m));
    k_hub<<<G, kTB>>>(n, ip.p, ix.p, hub.p);
    k_support<<<(int)std::min<int64_t>((n + kTB / 32 - 1) / (kTB / 32), 148 * 256), kTB>>>(n, ip.p, ix.p, hub.p, keep.p);
    RC(cudaGetLastError());
    lap("cycle support");
    // 4. filtered pattern
    Buf<int64_t> fp;
    RC(fp.alloc(n + 1));
    RC(cudaMemset(cnt.p + n, 0, sizeof(int64_t)));
    k_keep_count<<<G, kTB>>>(n, ip.p, keep.p, cnt.p);
    if ((rc = exclusive_scan64(cnt.p, fp.p, n + 1))) return rc;
    int64_t kept = 0;
    RC(cudaMemcpy(&kept, fp.p + n, sizeof(int64_t), cudaMemcpyDeviceToHost));
    out = LocalityOrder();
    out.dropped = 2 * m - kept;
    if (verbose)
        fprintf(stderr, "pars3 plan:   locality: dropped %.1f %% of the directed edges\n",
                100.0 * (double)out.dropped / (double)(2 * m));
    if ((10 * out.dropped > 6 * 2 * m || 1000 * out.dropped < 2 * m) && !getenv("PARS3_LOCALITY_ALWAYS")) {
        done = true;  // no band to recover (locality.cpp): forward stays empty
        return PARS3_OK;
    }
    Buf<int32_t> fx;
    RC(fx.alloc(kept));
    k_keep_fill<<<G, kTB>>>(n, ip.p, ix.p, keep.p, fp.p, fx.p);
    RC(cudaGetLastError());
    ix.free_now();
    keep.free_now();
    hub.free_now();
    lap("filtered pattern");
    // 5. RCM of the filtered graph, then P A P^T
    Buf<int64_t> fw, rp2;
    Buf<int32_t> col2;
    Buf<double> val2, diag2;
    RC(fw.alloc(n));
    rc = pars3_rcm_order_device(n, fp.p, fx.p, fw.p, nullptr);
    if (rc) return rc;
    RC(cudaDeviceSynchronize());
    fx.free_now();
    lap("RCM");
    RC(rp2.alloc(n + 1));
    RC(col2.alloc(m));
    RC(val2.alloc(m));
    RC(diag2.alloc(n));
    rc = pars3_permute_lower_device(n, rp.p, col.p, val.p, diag.p, fw.p, rp2.p, col2.p, val2.p, diag2.p, nullptr);
    if (rc) return rc;
    lap("relabel");
    std::vector<int64_t> hfw(n);
    out.row_ptr.resize(n + 1);
    out.col.resize(m);
    out.val.resize(m);
    out.diag.resize(n);
    RC(cudaMemcpy(hfw.data(), fw.p, sizeof(int64_t) * n, cudaMemcpyDeviceToHost));
    RC(cudaMemcpy(out.row_ptr.data(), rp2.p, sizeof(int64_t) * (n + 1), cudaMemcpyDeviceToHost));
    RC(cudaMemcpy(out.col.data(), col2.p, sizeof(int32_t) * m, cudaMemcpyDeviceToHost));
    RC(cudaMemcpy(out.val.data(), val2.p, sizeof(double) * m, cudaMemcpyDeviceToHost));
    RC(cudaMemcpy(out.diag.data(), diag2.p, sizeof(double) * n, cudaMemcpyDeviceToHost));
    out.forward.assign(hfw.begin(), hfw.end());
    lap("download");
    done = true;
    return PARS3_OK;
}

}  // namespace pars3
