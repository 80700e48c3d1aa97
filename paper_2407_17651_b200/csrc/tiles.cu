// Windowed tile kernel: the single-GPU PARS3 product.
//
// One persistent CTA loop; tiles are claimed in ascending order from an
// atomic counter.  Per tile:
//   1. the tile's column windows of x are copied into shared memory (xs) and
//      the matching accumulators (acc) zeroed;
//   2. each warp streams SELL-32 slices (fp64 value + uint16 local column):
//      lane l owns one row segment, keeps its row sum in a register
//      (+a_ic * x_c, serial.py:56-57) and adds the mirror -a_ic * x_i into
//      acc[c] (serial.py:58-59) -- both in shared memory, no global atomics;
//   3. the tile's own rows are final except for contributions of LATER
//      tiles: y[r] = diag_r x_r + acc[r] is stored, then the tile's flag is
//      released (this is the reference's "owner" write, parallel.py:85-95);
//   4. the remaining window slots (columns below the tile) are this tile's
//      accumulation messages (the reference's msg_val / MPI_Accumulate,
//      parallel.py:96-113): after the owning tiles have
//      released their flags they are added into y with fp64 reductions.
// Waits only ever target lower tile indices, which were claimed earlier by
// running CTAs that never wait before releasing, so the loop cannot deadlock.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstring>
#include <new>

#include "common.h"
#include "tileplan.h"

using pars3::HostPlan;
using pars3::PlanOptions;
using pars3::TileMeta;
using pars3::Window;

namespace {

constexpr uint16_t kNo = pars3::kNoSlot;
constexpr int kThreads = 512;
constexpr int kWarps = kThreads / 32;

struct DevPlan {
    const TileMeta *tiles;
    const Window *wins;
    const int32_t *sbase;
    const int32_t *sns;
    const uint16_t *srowl;
    const double *val;
    const uint16_t *lidx;
    const double *diag;
    int32_t *flags;
    int32_t *counter;
    int32_t ntiles;
    int32_t lmax;
};

__device__ __forceinline__ int32_t ld_acquire(const int32_t *p) {
    int32_t v;
    asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ void st_release(int32_t *p, int32_t v) {
    asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// local slot -> window (binary search over the tile's window loff)
__device__ __forceinline__ int find_window(const Window *wins, int w0, int w1, int i) {
    int lo = w0, hi = w1 - 1;
    while (lo < hi) {
        int mid = (lo + hi + 1) >> 1;
        if (__ldg(&wins[mid].loff) <= i) lo = mid; else hi = mid - 1;
    }
    return lo;
}

__device__ __forceinline__ void entry(double v, uint16_t li, double xr, const double *xs,
                                      double *acc, double &racc) {
    if (li != kNo) {
        racc = fma(v, xs[li], racc);
        atomicAdd(&acc[li], -v * xr);
    }
}

__global__ void __launch_bounds__(kThreads, 2)
k_tiles(DevPlan P, const double *__restrict__ x, double *__restrict__ y, int32_t epoch) {
    extern __shared__ double sm[];
    double *xs = sm;
    double *acc = sm + P.lmax;
    __shared__ int32_t s_tile;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

    for (;;) {
        if (tid == 0) s_tile = atomicAdd(P.counter, 1);
        __syncthreads();
        const int32_t t = s_tile;
        if (t >= P.ntiles) break;
        const TileMeta m = P.tiles[t];
        const int nw = m.w1 - m.w0;

        // 1. x windows -> shared memory, accumulators cleared
        if (nw <= 8) {
            for (int w = m.w0; w < m.w1; w++) {
                const int lo = __ldg(&P.wins[w].lo), len = __ldg(&P.wins[w].len),
                          off = __ldg(&P.wins[w].loff);
                for (int i = tid; i < len; i += kThreads) {
                    xs[off + i] = __ldg(x + lo + i);
                    acc[off + i] = 0.0;
                }
            }
        } else {
            for (int i = tid; i < m.local; i += kThreads) {
                const int w = find_window(P.wins, m.w0, m.w1, i);
                xs[i] = __ldg(x + __ldg(&P.wins[w].lo) + (i - __ldg(&P.wins[w].loff)));
                acc[i] = 0.0;
            }
        }
        __syncthreads();

        // 2. SELL-32 slices: row sums in registers, mirrors into acc
        for (int s = m.s0 + warp; s < m.s1; s += kWarps) {
            const int base = __ldg(P.sbase + s), ns = __ldg(P.sns + s);
            const uint16_t rl = __ldg(P.srowl + s * 32 + lane);
            const double xr = rl != kNo ? xs[rl] : 0.0;
            double racc = 0.0;
            const double *vp = P.val + base + lane;
            const uint16_t *ip = P.lidx + base + lane;
            int j = 0;
            for (; j + 4 <= ns; j += 4, vp += 128, ip += 128) {
                double v[4];
                uint16_t li[4];
#pragma unroll
                for (int u = 0; u < 4; u++) {
                    v[u] = __ldcs(vp + 32 * u);
                    li[u] = __ldcs(ip + 32 * u);
                }
#pragma unroll
                for (int u = 0; u < 4; u++) entry(v[u], li[u], xr, xs, acc, racc);
            }
            for (; j < ns; j++, vp += 32, ip += 32) entry(__ldcs(vp), __ldcs(ip), xr, xs, acc, racc);
            if (rl != kNo) atomicAdd(&acc[rl], racc);
        }
        __syncthreads();

        // 3. own rows: final up to later tiles' messages; store, then release
        for (int r = m.r0 + tid; r < m.r1; r += kThreads) {
            const int l = m.own_loff + (r - m.r0);
            y[r] = fma(__ldg(P.diag + r), xs[l], acc[l]);
        }
        __threadfence();
        __syncthreads();
        if (tid == 0 && m.r1 > m.r0) st_release(P.flags + t, epoch);

        // 4. wait until the owners of every message target have stored
        if (warp == 0) {
            for (int w = m.w0 + lane; w < m.w1; w += 32) {
                const int tl = __ldg(&P.wins[w].t_lo), th = __ldg(&P.wins[w].t_hi);
                for (int u = tl; u <= th; u++)
                    if (u != t)
                        while (ld_acquire(P.flags + u) != epoch) {
                        }
            }
        }
        __syncthreads();

        // 5. deliver the messages (slots outside the own rows)
        if (nw <= 8) {
            for (int w = m.w0; w < m.w1; w++) {
                const int lo = __ldg(&P.wins[w].lo), len = __ldg(&P.wins[w].len),
                          off = __ldg(&P.wins[w].loff);
                for (int i = tid; i < len; i += kThreads) {
                    const int c = lo + i;
                    const double a = acc[off + i];
                    if ((c < m.r0 || c >= m.r1) && a != 0.0) atomicAdd(y + c, a);
                }
            }
        } else {
            for (int i = tid; i < m.local; i += kThreads) {
                const int w = find_window(P.wins, m.w0, m.w1, i);
                const int c = __ldg(&P.wins[w].lo) + (i - __ldg(&P.wins[w].loff));
                const double a = acc[i];
                if ((c < m.r0 || c >= m.r1) && a != 0.0) atomicAdd(y + c, a);
            }
        }
        __syncthreads();
    }
}

__global__ void k_dot(int32_t n, const double *__restrict__ a, const double *__restrict__ b,
                      double *out) {
    double s = 0.0;
    for (int32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
        s = fma(a[i], b[i], s);
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    __shared__ double ws[32];
    if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x < 32) {
        s = threadIdx.x < (blockDim.x >> 5) ? ws[threadIdx.x] : 0.0;
        for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if (threadIdx.x == 0) atomicAdd(out, s);
    }
}

template <class T>
int upload(T **dst, const std::vector<T> &src) {
    *dst = nullptr;
    if (src.empty()) return PARS3_OK;
    CUDA_TRY(cudaMalloc((void **)dst, sizeof(T) * src.size()));
    CUDA_TRY(cudaMemcpy(*dst, src.data(), sizeof(T) * src.size(), cudaMemcpyHostToDevice));
    return PARS3_OK;
}

}  // namespace

struct pars3_plan {
    int64_t n = 0, beta = 0;
    int32_t p = 1;
    int32_t ntiles = 0, nslices = 0, lmax = 0;
    int64_t nnz = 0, slots = 0, nwins = 0;
    int32_t epoch = 0;
    int grid = 0;
    size_t smem = 0;
    TileMeta *tiles = nullptr;
    Window *wins = nullptr;
    int32_t *sbase = nullptr, *sns = nullptr;
    uint16_t *srowl = nullptr;
    double *val = nullptr;
    uint16_t *lidx = nullptr;
    double *diag = nullptr;
    int32_t *flags = nullptr;
    int32_t *counter = nullptr;
    int64_t bytes = 0;

    ~pars3_plan() {
        void *ptrs[] = {tiles, wins, sbase, sns, srowl, val, lidx, diag, flags, counter};
        for (void *q : ptrs)
            if (q) cudaFree(q);
    }
};

extern "C" int pars3_plan_create(const pars3_split_view *s, const pars3_plan_options *opt,
                                 int32_t p, const int64_t *block_start, pars3_plan **out,
                                 void *stream) {
    (void)block_start;
    (void)stream;
    if (!s || !out) PARS3_FAIL(PARS3_ERR_ARG, "null argument");
    *out = nullptr;
    if (s->n < 0 || s->n >= INT32_MAX || s->beta < 1) PARS3_FAIL(PARS3_ERR_ARG, "bad split header");
    if (p < 1) PARS3_FAIL(PARS3_ERR_ARG, "worker count must be at least 1, got %d", p);
    PlanOptions o;
    if (opt) {
        if (opt->tile_rows > 0) o.tile_rows = opt->tile_rows;
        if (opt->local_slots > 0) o.local_slots = opt->local_slots;
        if (opt->seg_max > 0) o.seg_max = opt->seg_max;
        if (opt->gap >= 0) o.gap = opt->gap;
    }
    HostPlan hp;
    int rc = pars3::build_tile_plan(s->n, s->mid_ptr, s->mid_col, s->mid_val, s->outer_count,
                                    s->outer_row, s->outer_col, s->outer_val, o, hp);
    if (rc) return rc;
    pars3_plan *pl = new (std::nothrow) pars3_plan;
    if (!pl) PARS3_FAIL(PARS3_ERR_NOMEM, "out of host memory");
    pl->n = s->n;
    pl->beta = s->beta;
    pl->p = p;
    pl->ntiles = (int32_t)hp.tiles.size();
    pl->nslices = (int32_t)hp.slice_base.size();
    pl->lmax = hp.max_local > 0 ? hp.max_local : 1;
    pl->nnz = hp.nnz;
    pl->slots = (int64_t)hp.val.size();
    pl->nwins = (int64_t)hp.wins.size();
    std::vector<double> diag(s->diag, s->diag + s->n);
    std::vector<int32_t> zeros(pl->ntiles + 1, 0);
#define UP(dst, src)                               \
    do {                                           \
        int _r = upload(&pl->dst, src);            \
        if (_r) {                                  \
            delete pl;                             \
            return _r;                             \
        }                                          \
        pl->bytes += sizeof(src[0]) * src.size();  \
    } while (0)
    UP(tiles, hp.tiles);
    UP(wins, hp.wins);
    UP(sbase, hp.slice_base);
    UP(sns, hp.slice_nslots);
    UP(srowl, hp.slice_rowl);
    UP(val, hp.val);
    UP(lidx, hp.lidx);
    UP(diag, diag);
    UP(flags, zeros);
#undef UP
    if (cudaMalloc((void **)&pl->counter, sizeof(int32_t)) != cudaSuccess) {
        delete pl;
        PARS3_FAIL(PARS3_ERR_CUDA, "cudaMalloc failed");
    }
    pl->smem = sizeof(double) * 2 * (size_t)pl->lmax;
    cudaError_t e = cudaFuncSetAttribute(k_tiles, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)pl->smem);
    int per_sm = 0, sms = 0, dev = 0;
    if (e == cudaSuccess) e = cudaGetDevice(&dev);
    if (e == cudaSuccess) e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (e == cudaSuccess)
        e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_tiles, kThreads, pl->smem);
    if (e != cudaSuccess || per_sm < 1) {
        delete pl;
        PARS3_FAIL(PARS3_ERR_CUDA, "tile kernel cannot be resident (smem %zu B): %s", pl->smem,
                   cudaGetErrorString(e));
    }
    pl->grid = per_sm * sms;
    if (pl->grid > pl->ntiles) pl->grid = pl->ntiles > 0 ? pl->ntiles : 1;
    *out = pl;
    return PARS3_OK;
}

static int launch_tiles(pars3_plan *pl, const double *x, double *y, cudaStream_t st) {
    if (pl->ntiles == 0) return PARS3_OK;
    if (++pl->epoch == INT32_MAX) {  // wrap: clear the flags once every 2^31 products
        pl->epoch = 1;
        CUDA_TRY(cudaMemsetAsync(pl->flags, 0, sizeof(int32_t) * pl->ntiles, st));
    }
    CUDA_TRY(cudaMemsetAsync(pl->counter, 0, sizeof(int32_t), st));
    DevPlan P{pl->tiles, pl->wins, pl->sbase, pl->sns, pl->srowl, pl->val,
              pl->lidx,  pl->diag, pl->flags, pl->counter, pl->ntiles, pl->lmax};
    k_tiles<<<pl->grid, kThreads, pl->smem, st>>>(P, x, y, pl->epoch);
    LAUNCH_CHECK();
    return PARS3_OK;
}

extern "C" int pars3_plan_spmv(pars3_plan *pl, const double *x, double *y, void *stream) {
    if (!pl || (pl->n > 0 && (!x || !y))) PARS3_FAIL(PARS3_ERR_ARG, "null argument");
    return launch_tiles(pl, x, y, (cudaStream_t)stream);
}

extern "C" int pars3_plan_spmv_dot(pars3_plan *pl, const double *x, double *y, const double *w,
                                   double *dot, void *stream) {
    if (!pl || !dot || (pl->n > 0 && (!x || !y || !w))) PARS3_FAIL(PARS3_ERR_ARG, "null argument");
    cudaStream_t st = (cudaStream_t)stream;
    int rc = launch_tiles(pl, x, y, st);
    if (rc) return rc;
    CUDA_TRY(cudaMemsetAsync(dot, 0, sizeof(double), st));
    if (pl->n > 0) {
        k_dot<<<592, 512, 0, st>>>((int32_t)pl->n, y, w, dot);
        LAUNCH_CHECK();
    }
    return PARS3_OK;
}

extern "C" int pars3_plan_kernel_count(const pars3_plan *pl, int32_t with_dot, int32_t *count) {
    if (!pl || !count) PARS3_FAIL(PARS3_ERR_ARG, "null argument");
    *count = (pl->ntiles > 0 ? 1 : 0) + (with_dot && pl->n > 0 ? 1 : 0);
    return PARS3_OK;
}

extern "C" int pars3_plan_bytes(const pars3_plan *pl, int64_t *bytes) {
    if (!pl || !bytes) PARS3_FAIL(PARS3_ERR_ARG, "null argument");
    *bytes = pl->bytes;
    return PARS3_OK;
}

extern "C" int pars3_plan_stats(const pars3_plan *pl, int64_t *stats) {
    if (!pl || !stats) PARS3_FAIL(PARS3_ERR_ARG, "null argument");
    stats[0] = pl->ntiles;
    stats[1] = pl->nslices;
    stats[2] = pl->slots;
    stats[3] = pl->nnz;
    stats[4] = pl->nwins;
    stats[5] = pl->lmax;
    stats[6] = pl->grid;
    stats[7] = pl->bytes;
    return PARS3_OK;
}

extern "C" int pars3_plan_destroy(pars3_plan *pl) {
    delete pl;
    return PARS3_OK;
}
