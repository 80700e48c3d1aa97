// Device builder of the windowed tile plan (tileplan.h; SURVEY.md 8(f) row 1:
// the plan construction on the GPU).  It produces the host builder's arrays
// (tileplan.cpp) byte for byte -- tiles, windows, slice offsets and slice
// records -- for the plans the product streams through k_tiles in window
// mode: band-limited matrices whose row ranges resolve to tiles with at most
// kMaxWindows dense windows (stencils, banded matrices: c5).  Anything else
// -- list-mode tiles, hub rows cut into chunks, ranges halved by the terms
// cap, peer-mode cuts, SKIP_EMPTY -- is reported as unsupported and the
// caller falls back to the host builder, so both builders never disagree.
//
//   k_optr         outer row pointer (the outer entries are sorted by row)
//   k_draft        one CTA per range of tile_rows rows: the host's recursive
//                  halving (draft_range) with the range's column set as a
//                  bitmap in shared memory; emits the range's tiles in row
//                  order (rows, windows, segments per length)
//   k_sizes        per tile: windows, slices and record bytes (then scans)
//   k_materialise  one CTA per tile: the stable length-descending order of
//                  the row segments by counting, the SELL-32 records, the
//                  terms per slot, the value bound, the bank-spread slot
//                  order of each slice (spread_banks, one thread per slice)
#include <cuda_runtime.h>
#include <omp.h>
#include <cub/cub.cuh>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "common.h"
#include "tileplan.h"
#include "tileplan_gpu.h"

namespace pars3 {
namespace {

#define RC(expr)                                                                                  \
    do {                                                                                          \
        cudaError_t _e = (expr);                                                                  \
        if (_e != cudaSuccess)                                                                    \
            PARS3_FAIL(PARS3_ERR_CUDA, "tile plan (device): %s: %s", #expr, cudaGetErrorString(_e)); \
    } while (0)

constexpr int kT = 256;
constexpr int kMaxTileRows = 1024;       // rows per tile the materialiser holds in shared memory
constexpr int kMaxRangeTiles = 16;       // tiles one range may resolve to
constexpr int kBitmapBits = 1 << 19;     // column span of a range (bits of shared memory)
constexpr int kCounters = 1 << 15;       // distinct columns of a range (16-bit reference counters)
constexpr int kMaxRuns = 16;

struct Split {
    int64_t n;
    const int64_t *mptr;
    const int32_t *mcol;
    const double *mval;
    const int64_t *optr;
    const int32_t *ocol;
    const double *oval;
};

struct Opts {
    int32_t tile_rows, local_slots, seg_max, gap, max_segments, terms_cap, terms_min_rows;
    uint16_t sink;
};

struct DraftTile {  // one emitted tile of a range
    int32_t a, b, nwin, local;
    int32_t wlo[kMaxWindows], wlen[kMaxWindows];
    int32_t cnt[8];  // row segments of length 1 .. 8
    int32_t list;    // 1: explicit column list (too fragmented for windows); local = its length
    int32_t cmin;    // smallest column (list tiles: the bitmap's origin)
};

__device__ __forceinline__ int64_t row_count(const Split &S, int64_t r) {
    return (S.optr[r + 1] - S.optr[r]) + (S.mptr[r + 1] - S.mptr[r]);
}

__global__ void k_optr(int64_t n, int64_t no, const int32_t *orow, int64_t *optr) {
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r <= n; r += (int64_t)gridDim.x * blockDim.x) {
        int64_t a = 0, b = no;  // first e with orow[e] >= r
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

// flags[0]: the plan needs the host builder
__global__ void __launch_bounds__(kT) k_draft(Split S, Opts o, int64_t nranges, DraftTile *out, int32_t *ntiles,
                                              int32_t *flags) {
    extern __shared__ __align__(16) uint32_t dyn[];
    uint32_t *bitmap = dyn;                       // kBitmapBits / 32 words
    uint32_t *wrank = dyn + kBitmapBits / 32;     // set bits before each bitmap word
    uint32_t *ctr = wrank + kBitmapBits / 32;     // kCounters / 2 words (two 16-bit counters each)
    __shared__ uint32_t s_tot[kT];
    __shared__ int32_t s_stack[2][24];
    __shared__ int32_t s_sp, s_emit, s_fail;
    __shared__ unsigned long long s_segments, s_entries;
    __shared__ int32_t s_maxsegs, s_cmin, s_cnt[8], s_best, s_ns, s_ne, s_starts[kMaxRuns], s_ends[kMaxRuns];
    __shared__ int32_t s_action;  // 0 emit, 1 split plain, 2 split aligned, 3 fail
    __shared__ int32_t s_why;     // why the range needs the host builder (bits, for PARS3_VERBOSE)
    __shared__ int32_t s_distinct;  // distinct columns of the range (set bits)
    const int tid = threadIdx.x;
    const int64_t q = blockIdx.x;
    if (q >= nranges) return;
    if (tid == 0) {
        s_stack[0][0] = (int32_t)(q * o.tile_rows);
        s_stack[1][0] = (int32_t)min((int64_t)S.n, (q + 1) * (int64_t)o.tile_rows);
        s_sp = 1;
        s_emit = 0;
        s_fail = 0;
        s_why = 0;
    }
    __syncthreads();
    while (true) {
        __syncthreads();
        if (s_sp == 0 || s_fail) break;
        const int32_t a = s_stack[0][s_sp - 1], b = s_stack[1][s_sp - 1];
        __syncthreads();
        if (tid == 0) {
            s_sp--;
            s_segments = 0;
            s_entries = 0;
            s_maxsegs = 0;
            s_cmin = a;
            s_best = 0;
            s_ns = s_ne = 0;
            s_distinct = 0;
            for (int k = 0; k < 8; k++) s_cnt[k] = 0;
        }
        __syncthreads();
        // pass A: counts, segments per length, the smallest column
        for (int32_t r = a + tid; r < b; r += kT) {
            const int64_t c = row_count(S, r);
            const int64_t full = c / o.seg_max, rem = c % o.seg_max;
            atomicAdd(&s_segments, (unsigned long long)(full + (rem ? 1 : 0)));
            atomicAdd(&s_entries, (unsigned long long)c);
            atomicMax(&s_maxsegs, (int32_t)min((int64_t)INT32_MAX, full + (rem ? 1 : 0)));
            if (full) atomicAdd(&s_cnt[o.seg_max - 1], (int32_t)min((int64_t)INT32_MAX, full));
            if (rem) atomicAdd(&s_cnt[rem - 1], 1);
            if (c > 0) {  // columns ascend, every outer column lies below every middle one
                const int32_t first = S.optr[r + 1] > S.optr[r] ? S.ocol[S.optr[r]] : S.mcol[S.mptr[r]];
                atomicMin(&s_cmin, first);
            }
        }
        __syncthreads();
        const int32_t cmin = s_cmin;
        const int64_t span = (int64_t)b - cmin;
        if (tid == 0) {
            int act = 0;
            if ((long long)s_segments > o.max_segments && b - a > 1)
                act = 1;
            else if (span > kBitmapBits || s_entries > 60000ull || (long long)s_segments > o.max_segments) {
                act = 3;
                s_why |= 1;
            }
            s_action = act;
        }
        __syncthreads();
        if (s_action == 0) {
            // pass B: the column set as a bitmap over [cmin, b), hashed reference counts
            const int32_t nwords = (int32_t)((span + 31) / 32);
            for (int32_t i = tid; i < nwords; i += kT) bitmap[i] = 0u;
            const bool check_terms = o.terms_cap > 0 && b - a > o.terms_min_rows / 2;
            __syncthreads();
            auto mark = [&](int32_t c) {
                const int32_t p = c - cmin;
                atomicOr(&bitmap[p >> 5], 1u << (p & 31));
            };
            for (int32_t r = a + tid; r < b; r += kT) {
                mark(r);
                for (int64_t k = S.optr[r]; k < S.optr[r + 1]; k++) mark(S.ocol[k]);
                for (int64_t k = S.mptr[r]; k < S.mptr[r + 1]; k++) mark(S.mcol[k]);
            }
            __syncthreads();
            if (check_terms) {
                // the busiest column's references, exactly: a counter per distinct
                // column, indexed by the column's rank in the bitmap
                const int32_t per = (nwords + kT - 1) / kT, w0 = tid * per, w1 = min(nwords, w0 + per);
                uint32_t run = 0;
                for (int32_t i = w0; i < w1; i++) {
                    wrank[i] = run;
                    run += __popc(bitmap[i]);
                }
                s_tot[tid] = run;
                __syncthreads();
                if (tid == 0) {
                    uint32_t acc = 0;
                    for (int i = 0; i < kT; i++) {
                        const uint32_t v = s_tot[i];
                        s_tot[i] = acc;
                        acc += v;
                    }
                    if (acc > (uint32_t)kCounters) {  // (more distinct columns than counters)
                        s_action = 3;
                        s_why |= 64;
                    }
                }
                __syncthreads();
                if (s_action == 0) {
                    for (int32_t i = w0; i < w1; i++) wrank[i] += s_tot[tid];
                    for (int32_t i = tid; i < kCounters / 2; i += kT) ctr[i] = 0u;
                    __syncthreads();
                    auto count = [&](int32_t c) {
                        const int32_t p = c - cmin;
                        const uint32_t h = wrank[p >> 5] + __popc(bitmap[p >> 5] & ((1u << (p & 31)) - 1u));
                        atomicAdd(&ctr[h >> 1], 1u << (16 * (h & 1)));
                    };
                    for (int32_t r = a + tid; r < b; r += kT) {
                        count(r);
                        for (int64_t k = S.optr[r]; k < S.optr[r + 1]; k++) count(S.ocol[k]);
                        for (int64_t k = S.mptr[r]; k < S.mptr[r + 1]; k++) count(S.mcol[k]);
                    }
                    __syncthreads();
                    int32_t best = 0;
                    for (int32_t i = tid; i < kCounters / 2; i += kT) {
                        const uint32_t v = ctr[i];
                        best = max(best, (int32_t)max(v & 0xFFFFu, v >> 16));
                    }
                    best = __reduce_max_sync(0xffffffffu, best);
                    if ((tid & 31) == 0) atomicMax(&s_best, best);
                }
            }
            // window starts and ends: runs separated by more than `gap` unused slots
            const int look = o.gap + 1;
            int32_t pc = 0;
            for (int32_t i = tid; i < nwords; i += kT) {
                const uint32_t cur = bitmap[i];
                if (!cur) continue;
                pc += __popc(cur);
                const uint32_t prv = i > 0 ? bitmap[i - 1] : 0u, nxt = i + 1 < nwords ? bitmap[i + 1] : 0u;
                const unsigned long long X = ((unsigned long long)cur << 32) | prv;
                const unsigned long long Y = ((unsigned long long)nxt << 32) | cur;
                unsigned long long nb = 0, na = 0;
                for (int d = 1; d <= look; d++) {
                    nb |= X << d;
                    na |= Y >> d;
                }
                uint32_t st = cur & ~(uint32_t)(nb >> 32), en = cur & ~(uint32_t)na;
                while (st) {
                    const int j = __ffs(st) - 1;
                    st &= st - 1;
                    const int k = atomicAdd(&s_ns, 1);
                    if (k < kMaxRuns) s_starts[k] = cmin + i * 32 + j;
                }
                while (en) {
                    const int j = __ffs(en) - 1;
                    en &= en - 1;
                    const int k = atomicAdd(&s_ne, 1);
                    if (k < kMaxRuns) s_ends[k] = cmin + i * 32 + j + 1;
                }
            }
            pc = __reduce_add_sync(0xffffffffu, pc);
            if ((tid & 31) == 0 && pc) atomicAdd(&s_distinct, pc);
            __syncthreads();
            if (tid == 0) {
                int act = s_action;
                if (act == 0 && check_terms && s_best + s_maxsegs > o.terms_cap) {
                    // the busiest slot would take more terms than the accumulator
                    // carries: halve the range (down to terms_min_rows rows), so the
                    // plan keeps the two-word accumulator; a single row is cut into
                    // chunks by the host builder
                    if (b - a > max(1, o.terms_min_rows)) {
                        act = 2;
                    } else if (b - a == 1) {
                        act = 3;
                        s_why |= 2;
                    }
                }
                int nw = s_ns;
                bool as_list = false, one_window = false;
                if (act == 0 && (nw > kMaxWindows || nw != s_ne)) {
                    // too fragmented for gap-merged windows (draft_range, tileplan.cpp):
                    // one dense window over the whole column span when it fits; else
                    // halve when that would make it fit; else the host rebuilds the
                    // windows without gap or alignment slots (local = the distinct
                    // columns) and keeps a list-mode tile if that fits, else halves
                    int32_t lo = cmin & ~1, hi = b;
                    if ((hi & 1) && hi < S.n) hi++;
                    if (hi - lo <= o.local_slots) {
                        one_window = true;
                        nw = 1;
                        s_ns = s_ne = 1;
                        s_starts[0] = lo;
                        s_ends[0] = b;
                    } else if (b - a > 64 && (hi - lo) - (b - a) / 2 <= o.local_slots) {
                        act = 2;
                    } else if (s_distinct <= o.local_slots) {
                        as_list = true;
                    } else if (b - a > 1) {
                        act = 2;
                    } else {
                        act = 3;
                        s_why |= 16;
                    }
                }
                (void)one_window;
                if (act == 0 && as_list) {
                    DraftTile d;
                    d.a = a;
                    d.b = b;
                    d.nwin = 0;
                    d.local = s_distinct;
                    d.list = 1;
                    d.cmin = cmin;
                    for (int i = 0; i < kMaxWindows; i++) d.wlo[i] = d.wlen[i] = 0;
                    for (int k = 0; k < 8; k++) d.cnt[k] = s_cnt[k];
                    if (s_emit >= kMaxRangeTiles || b - a > kMaxTileRows) {
                        act = 3;
                        s_why |= 8;
                    } else {
                        out[q * kMaxRangeTiles + s_emit] = d;
                        s_emit++;
                    }
                } else
                if (act == 0) {
                    // sort the few runs, align them to even bounds (make_windows)
                    for (int i = 1; i < nw; i++)
                        for (int j = i; j > 0 && s_starts[j] < s_starts[j - 1]; j--) {
                            const int32_t t = s_starts[j];
                            s_starts[j] = s_starts[j - 1];
                            s_starts[j - 1] = t;
                        }
                    for (int i = 1; i < nw; i++)
                        for (int j = i; j > 0 && s_ends[j] < s_ends[j - 1]; j--) {
                            const int32_t t = s_ends[j];
                            s_ends[j] = s_ends[j - 1];
                            s_ends[j - 1] = t;
                        }
                    DraftTile d;
                    d.a = a;
                    d.b = b;
                    d.nwin = 0;
                    d.local = 0;
                    d.list = 0;
                    d.cmin = cmin;
                    for (int i = 0; i < nw; i++) {
                        int32_t lo = s_starts[i] & ~1, hi = s_ends[i];
                        if ((hi & 1) && hi < S.n) hi++;
                        if (d.nwin > 0 && lo <= d.wlo[d.nwin - 1] + d.wlen[d.nwin - 1]) {  // touches the previous
                            d.local -= d.wlen[d.nwin - 1];
                            d.wlen[d.nwin - 1] = hi - d.wlo[d.nwin - 1];
                            d.local += d.wlen[d.nwin - 1];
                            continue;
                        }
                        d.wlo[d.nwin] = lo;
                        d.wlen[d.nwin] = hi - lo;
                        d.local += hi - lo;
                        d.nwin++;
                    }
                    for (int i = d.nwin; i < kMaxWindows; i++) d.wlo[i] = d.wlen[i] = 0;
                    for (int k = 0; k < 8; k++) d.cnt[k] = s_cnt[k];
                    if (d.local <= o.local_slots) {
                        if (s_emit >= kMaxRangeTiles || b - a > kMaxTileRows) {
                            act = 3;
                            s_why |= 8;
                        } else {
                            out[q * kMaxRangeTiles + s_emit] = d;
                            s_emit++;
                        }
                    } else if (b - a > 1) {
                        act = 2;
                    } else {
                        act = 3;  // one row wider than the local space: hub chunks
                        s_why |= 16;
                    }
                }
                s_action = act;
            }
            __syncthreads();
        }
        if (tid == 0) {
            const int act = s_action;
            if (act == 3) {
                s_fail = 1;
            } else if (act == 1 || act == 2) {
                int32_t mid = a + (b - a) / 2;
                if (act == 2 && b - a > 64) mid = a + (((b - a) / 2 + 31) & ~31);
                if (s_sp + 2 > 24) {
                    s_fail = 1;
                    s_why |= 32;
                } else {  // left half first: tiles come out in row order
                    s_stack[0][s_sp] = mid;
                    s_stack[1][s_sp] = b;
                    s_stack[0][s_sp + 1] = a;
                    s_stack[1][s_sp + 1] = mid;
                    s_sp += 2;
                }
            }
        }
    }
    if (tid == 0) {
        ntiles[q] = s_emit;
        if (s_fail) atomicOr(flags, s_why ? s_why : 128);
    }
}

// dense tile list + per-tile window / slice / record-byte counts
__global__ void k_sizes(int64_t nranges, const DraftTile *draft, const int32_t *ntiles, const int64_t *toff,
                        DraftTile *tiles, int64_t *nwin, int64_t *nslices, int64_t *nbytes, int64_t *nucol) {
    const int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (q >= nranges) return;
    for (int32_t k = 0; k < ntiles[q]; k++) {
        const DraftTile d = draft[q * kMaxRangeTiles + k];
        const int64_t t = toff[q] + k;
        tiles[t] = d;
        // slices in length-descending order: slice s takes the length of sorted segment 32 s
        int64_t nseg = 0, bytes = 0, ns = 0;
        for (int L = 8; L >= 1; L--) {
            const int64_t lo = nseg, hi = nseg + d.cnt[L - 1];
            // slices whose first segment index lies in [lo, hi)
            const int64_t s_lo = (lo + 31) / 32, s_hi = (hi + 31) / 32;
            bytes += (s_hi - s_lo) * (64 + 320 * (int64_t)L);
            ns += s_hi - s_lo;
            nseg = hi;
        }
        nwin[t] = d.list ? 0 : d.nwin;
        nucol[t] = d.list ? d.local : 0;
        nslices[t] = ns;
        nbytes[t] = bytes;
    }
}

__device__ __forceinline__ int32_t local_of(const int32_t *wlo, const int32_t *wloff, int nwin, int32_t c) {
    int w = 0;
    while (w + 1 < nwin && wlo[w + 1] <= c) w++;
    return wloff[w] + (c - wlo[w]);
}

__device__ int slot_conflicts_dev(const uint16_t *lx, uint16_t sink) {
    int b32[32], b16[16], c = 0;
    for (int i = 0; i < 32; i++) b32[i] = 0;
    for (int i = 0; i < 16; i++) b16[i] = 0;
    for (int l = 0; l < 32; l++) {
        if (lx[l] == sink) continue;
        c += (b32[lx[l] & 31]++ > 0) + (b16[lx[l] & 15]++ > 1);
    }
    return c;
}

// spread_banks of tileplan.cpp, one thread per slice
__device__ void spread_banks_dev(double *val, uint16_t *lidx, int32_t nslots, int lanes, uint16_t sink) {
    if (nslots < 2 || nslots > 8 || lanes < 2) return;
    int before = 0;
    for (int32_t k = 0; k < nslots; k++) before += slot_conflicts_dev(lidx + (size_t)k * 32, sink);
    if (before == 0) return;
    double v2[8 * 32];
    uint16_t x2[8 * 32];
    uint8_t used[32];  // bit q of used[l]
    for (int i = 0; i < nslots * 32; i++) x2[i] = sink;
    for (int l = 0; l < 32; l++) used[l] = 0;
    int after = 0;
    for (int32_t k = 0; k < nslots; k++) {
        int b32[32], b16[16];
        for (int i = 0; i < 32; i++) b32[i] = 0;
        for (int i = 0; i < 16; i++) b16[i] = 0;
        for (int l = 0; l < lanes; l++) {
            int best = -1, bc = 1 << 30;
            for (int32_t q = 0; q < nslots; q++) {
                const uint16_t c = lidx[(size_t)q * 32 + l];
                if (((used[l] >> q) & 1) || c == sink) continue;
                const int cost = (b32[c & 31] > 0) + (b16[c & 15] > 1);
                if (cost < bc) {
                    bc = cost;
                    best = q;
                }
            }
            if (best < 0) continue;
            used[l] |= (uint8_t)(1u << best);
            const uint16_t c = lidx[(size_t)best * 32 + l];
            b32[c & 31]++;
            b16[c & 15]++;
            after += bc;
            x2[(size_t)k * 32 + l] = c;
            v2[(size_t)k * 32 + l] = val[(size_t)best * 32 + l];
        }
    }
    if (after >= before) return;
    for (int32_t k = 0; k < nslots; k++)
        for (int l = 0; l < lanes; l++) {
            lidx[(size_t)k * 32 + l] = x2[(size_t)k * 32 + l];
            val[(size_t)k * 32 + l] = x2[(size_t)k * 32 + l] == sink ? 0.0 : v2[(size_t)k * 32 + l];
        }
}

struct Totals {
    unsigned long long nnz, slots;
    int32_t max_terms, max_nslots;
};

// kList: the list-mode tiles (local slot of a column = its rank in the
// tile's column set, rebuilt here as a bitmap in dynamic shared memory; the
// set goes to ucol); else the window-mode tiles.  Both launches cover every
// tile; each takes its own kind.
template <bool kList>
__global__ void __launch_bounds__(kT) k_materialise(Split S, Opts o, int64_t nt, const DraftTile *dt,
                                                    const int64_t *woff, const int64_t *soff, const int64_t *voff,
                                                    const int64_t *uoff, TileMeta *tiles, Window *wins,
                                                    int64_t *slice_off, uint8_t *rec, int32_t *ucol, Totals *tot) {
    extern __shared__ __align__(16) uint32_t dynm[];
    uint32_t *bitmap = dynm;                        // kList: kBitmapBits / 32 words
    uint32_t *wrank = dynm + kBitmapBits / 32;      // set bits before each word
    __shared__ uint32_t s_tot[kT];
    __shared__ DraftTile d;
    __shared__ int32_t wloff[kMaxWindows];
    __shared__ unsigned long long pre[2][kMaxTileRows + 1];  // per row: segments before it, 16 bits per length
    __shared__ unsigned long long tsum[2][kT];
    __shared__ int32_t base[9];          // sorted index of the first segment of length L (base[8] = 0)
    __shared__ int32_t sl_ns[PARS3_GPU_MAX_SLICES], sl_off[PARS3_GPU_MAX_SLICES + 1];
    __shared__ int32_t terms[4096];
    __shared__ double s_vmax[kT / 32];
    __shared__ int32_t s_tmax;
    const int tid = threadIdx.x;
    const int64_t t = blockIdx.x;
    if (t >= nt) return;
    if ((dt[t].list != 0) != kList) return;
    if (tid == 0) {
        d = dt[t];
        int32_t acc = 0;
        for (int w = 0; w < d.nwin; w++) {
            wloff[w] = acc;
            acc += d.wlen[w];
        }
        s_tmax = 0;
    }
    for (int i = tid; i < 4096; i += kT) terms[i] = 0;
    __syncthreads();
    const int32_t a = d.a, b = d.b, nrows = b - a;
    const int32_t cmin = d.cmin;
    if (kList) {  // the column set and its ranks
        const int32_t nwords = (b - cmin + 31) / 32;
        for (int32_t i = tid; i < nwords; i += kT) bitmap[i] = 0u;
        __syncthreads();
        auto mark = [&](int32_t c) {
            const int32_t p = c - cmin;
            atomicOr(&bitmap[p >> 5], 1u << (p & 31));
        };
        for (int32_t r = a + tid; r < b; r += kT) {
            mark(r);
            for (int64_t k = S.optr[r]; k < S.optr[r + 1]; k++) mark(S.ocol[k]);
            for (int64_t k = S.mptr[r]; k < S.mptr[r + 1]; k++) mark(S.mcol[k]);
        }
        __syncthreads();
        const int32_t per = (nwords + kT - 1) / kT, w0 = tid * per, w1 = min(nwords, w0 + per);
        uint32_t run = 0;
        for (int32_t i = w0; i < w1; i++) {
            wrank[i] = run;
            run += __popc(bitmap[i]);
        }
        s_tot[tid] = run;
        __syncthreads();
        if (tid == 0) {
            uint32_t acc = 0;
            for (int i = 0; i < kT; i++) {
                const uint32_t v = s_tot[i];
                s_tot[i] = acc;
                acc += v;
            }
        }
        __syncthreads();
        for (int32_t i = w0; i < w1; i++) {
            wrank[i] += s_tot[tid];
            uint32_t bits = bitmap[i];
            uint32_t k = wrank[i];
            while (bits) {  // the list itself, ascending
                const int j = __ffs(bits) - 1;
                bits &= bits - 1;
                ucol[uoff[t] + k++] = cmin + i * 32 + j;
            }
        }
        __syncthreads();
    }
    auto slot_of = [&](int32_t c) -> int32_t {
        if (kList) {
            const int32_t p = c - cmin;
            return (int32_t)(wrank[p >> 5] + __popc(bitmap[p >> 5] & ((1u << (p & 31)) - 1u)));
        }
        return local_of(d.wlo, wloff, d.nwin, c);
    };
    // per-row segment counts packed 16 bits per length, exclusive prefix over the rows
    constexpr int kPer = kMaxTileRows / kT;
    unsigned long long loc[2][kPer], run0 = 0, run1 = 0;
    for (int j = 0; j < kPer; j++) {
        const int32_t i = tid * kPer + j;
        unsigned long long v0 = 0, v1 = 0;
        if (i < nrows) {
            const int64_t c = row_count(S, a + i);
            const int64_t full = c / o.seg_max, rem = c % o.seg_max;
            auto add = [&](int L, unsigned long long k) {
                if (L <= 4)
                    v0 += k << (16 * (L - 1));
                else
                    v1 += k << (16 * (L - 5));
            };
            if (full) add(o.seg_max, (unsigned long long)full);
            if (rem) add((int)rem, 1ull);
        }
        loc[0][j] = run0;
        loc[1][j] = run1;
        run0 += v0;
        run1 += v1;
    }
    tsum[0][tid] = run0;
    tsum[1][tid] = run1;
    __syncthreads();
    if (tid == 0) {  // serial exclusive scan of the 256 thread totals
        unsigned long long s0 = 0, s1 = 0;
        for (int i = 0; i < kT; i++) {
            const unsigned long long x0 = tsum[0][i], x1 = tsum[1][i];
            tsum[0][i] = s0;
            tsum[1][i] = s1;
            s0 += x0;
            s1 += x1;
        }
        // totals per length -> bases of the length-descending order
        int32_t run = 0;
        for (int L = 8; L >= 1; L--) {
            base[L] = run;
            run += (int32_t)(((L <= 4 ? s0 : s1) >> (16 * ((L - 1) & 3))) & 0xFFFFu);
        }
        base[0] = run;  // all segments
    }
    __syncthreads();
    for (int j = 0; j < kPer; j++) {
        const int32_t i = tid * kPer + j;
        if (i <= nrows && i < kMaxTileRows + 1) {
            pre[0][i] = tsum[0][tid] + loc[0][j];
            pre[1][i] = tsum[1][tid] + loc[1][j];
        }
    }
    const int32_t nseg = base[0], nsl = (nseg + 31) / 32;
    // slices: slots of each, record offsets
    for (int s = tid; s < nsl; s += kT) {
        const int32_t first = 32 * s;
        int L = 8;
        while (L > 1 && first >= base[L - 1]) L--;  // base[L] <= first < base[L - 1]
        sl_ns[s] = L;
    }
    __syncthreads();
    if (tid == 0) {
        int32_t off = 0;
        for (int s = 0; s < nsl; s++) {
            sl_off[s] = off;
            off += 64 + 320 * sl_ns[s];
        }
        sl_off[nsl] = off;
    }
    __syncthreads();
    uint8_t *trec = rec + voff[t];
    for (int s = tid; s < nsl; s += kT) slice_off[soff[t] + s] = (voff[t] + sl_off[s]) / 16;
    // padding everywhere first: rowl / lidx = sink, val = 0
    for (int s = 0; s < nsl; s++) {
        uint8_t *rp = trec + sl_off[s];
        const int ns = sl_ns[s];
        if (tid < 32) reinterpret_cast<uint16_t *>(rp)[tid] = o.sink;
        double *val = reinterpret_cast<double *>(rp + 64);
        uint16_t *lidx = reinterpret_cast<uint16_t *>(rp + 64 + (size_t)ns * 256);
        for (int i = tid; i < ns * 32; i += kT) {
            val[i] = 0.0;
            lidx[i] = o.sink;
        }
    }
    __syncthreads();
    // the entries: one thread per row, its segments in order
    double vmax = 0.0;
    unsigned long long nnz = 0;
    for (int32_t i = tid; i < nrows; i += kT) {
        const int32_t r = a + i;
        const int64_t no = S.optr[r + 1] - S.optr[r], c = no + (S.mptr[r + 1] - S.mptr[r]);
        const uint16_t rl = (uint16_t)slot_of(r);
        int64_t k = 0;
        int32_t seg_in_row = 0;
        while (k < c) {
            const int len = (int)min((int64_t)o.seg_max, c - k);
            // rank among the segments of this length, in row order
            const unsigned long long pk = len <= 4 ? pre[0][i] : pre[1][i];
            int32_t rank = (int32_t)((pk >> (16 * ((len - 1) & 3))) & 0xFFFFu);
            if (len == o.seg_max) rank += seg_in_row;  // (the remainder is never seg_max long)
            const int32_t sigma = base[len] + rank;
            const int s = sigma >> 5, l = sigma & 31;
            uint8_t *rp = trec + sl_off[s];
            const int ns = sl_ns[s];
            reinterpret_cast<uint16_t *>(rp)[l] = rl;
            atomicAdd(&terms[rl], 1);
            double *val = reinterpret_cast<double *>(rp + 64);
            uint16_t *lidx = reinterpret_cast<uint16_t *>(rp + 64 + (size_t)ns * 256);
            for (int e = 0; e < len; e++) {
                const int64_t kk = k + e;
                const int32_t col = kk < no ? S.ocol[S.optr[r] + kk] : S.mcol[S.mptr[r] + (kk - no)];
                const double v = kk < no ? S.oval[S.optr[r] + kk] : S.mval[S.mptr[r] + (kk - no)];
                const uint16_t li = (uint16_t)slot_of(col);
                val[e * 32 + l] = v;
                lidx[e * 32 + l] = li;
                atomicAdd(&terms[li], 1);
                vmax = fmax(vmax, fabs(v));
            }
            nnz += len;
            k += len;
            seg_in_row++;
        }
    }
    for (int off2 = 16; off2; off2 >>= 1) {
        vmax = fmax(vmax, __shfl_xor_sync(0xffffffffu, vmax, off2));
        nnz += __shfl_xor_sync(0xffffffffu, nnz, off2);
    }
    if ((tid & 31) == 0) {
        s_vmax[tid >> 5] = vmax;
        atomicAdd(&tot->nnz, nnz);
    }
    __syncthreads();
    int32_t tm = 0;
    for (int i = tid; i < d.local && i < 4096; i += kT) tm = max(tm, terms[i]);
    tm = __reduce_max_sync(0xffffffffu, tm);
    if ((tid & 31) == 0) atomicMax(&s_tmax, tm);
    // bank-spread slot order, one thread per slice
    unsigned long long slots = 0;
    for (int s = tid; s < nsl; s += kT) {
        uint8_t *rp = trec + sl_off[s];
        const int ns = sl_ns[s];
        const int lanes = min(32, nseg - 32 * s);
        spread_banks_dev(reinterpret_cast<double *>(rp + 64), reinterpret_cast<uint16_t *>(rp + 64 + (size_t)ns * 256),
                         ns, lanes, o.sink);
        slots += (unsigned long long)ns * 32;
    }
    for (int off2 = 16; off2; off2 >>= 1) slots += __shfl_xor_sync(0xffffffffu, slots, off2);
    if ((tid & 31) == 0 && slots) atomicAdd(&tot->slots, slots);
    __syncthreads();
    if (tid == 0) {
        double vm = 0.0;
        for (int k = 0; k < kT / 32; k++) vm = fmax(vm, s_vmax[k]);
        TileMeta m;
        m.r0 = a;
        m.r1 = b;
        m.w0 = (int32_t)woff[t];
        m.w1 = (int32_t)(woff[t] + (kList ? 0 : d.nwin));
        m.u0 = kList ? (int32_t)uoff[t] : -1;
        m.s0 = (int32_t)soff[t];
        m.s1 = (int32_t)(soff[t] + nsl);
        m.local = d.local;
        m.pad0 = m.pad1 = m.pad2 = 0;
        int e = -1074;
        if (vm > 0.0) frexp(vm, &e);  // vm < 2^e
        m.ev = e;
        tiles[t] = m;
        for (int w = 0; !kList && w < d.nwin; w++) {
            Window W;
            W.lo = d.wlo[w];
            W.len = d.wlen[w];
            W.loff = wloff[w];
            W.pad0 = 0;
            wins[woff[t] + w] = W;
        }
        atomicMax(&tot->max_terms, s_tmax);
        if (nsl > 0) atomicMax(&tot->max_nslots, sl_ns[0]);
    }
}

// terms per y element: its row's entries, its column's mirrors, its diagonal
// (the grid form's headroom, tiles.cu grid_data)
__global__ void k_terms_rows(Split S, int32_t *terms) {
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < S.n; r += (int64_t)gridDim.x * blockDim.x)
        terms[r] = 1 + (int32_t)row_count(S, r);
}
__global__ void k_terms_cols(int64_t m, const int32_t *col, int32_t *terms) {
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < m; k += (int64_t)gridDim.x * blockDim.x)
        atomicAdd(&terms[col[k]], 1);
}
__global__ void k_max_i32(int64_t n, const int32_t *a, int32_t *out) {
    int32_t best = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        best = max(best, a[i]);
    best = __reduce_max_sync(0xffffffffu, best);
    if ((threadIdx.x & 31) == 0) atomicMax(out, best);
}

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
};

template <class T>
int to_device(Buf<T> &b, const T *h, int64_t count) {
    RC(b.alloc((size_t)count));
    if (count > 0) RC(cudaMemcpy(b.p, h, sizeof(T) * (size_t)count, cudaMemcpyHostToDevice));
    return PARS3_OK;
}

int exclusive_scan(int64_t *d, int64_t count) {  // in place, count elements + the total at d[count]
    size_t tb = 0;
    RC(cub::DeviceScan::ExclusiveSum(nullptr, tb, d, d, (int)(count + 1)));
    Buf<uint8_t> tmp;
    RC(tmp.alloc(tb));
    RC(cub::DeviceScan::ExclusiveSum(tmp.p, tb, d, d, (int)(count + 1)));
    return PARS3_OK;
}

}  // namespace

void DevicePlan::release() {
    void *ptrs[] = {tiles, wins, slice_off, rec};
    for (void *q : ptrs)
        if (q) cudaFree(q);
    tiles = nullptr;
    wins = nullptr;
    slice_off = nullptr;
    rec = nullptr;
}

int build_tile_plan_device(int64_t n, const int64_t *mid_ptr, const int32_t *mid_col, const double *mid_val,
                           int64_t outer_count, const int32_t *outer_row, const int32_t *outer_col,
                           const double *outer_val, const PlanOptions &o, HostPlan &P, DevicePlan &D,
                           bool &supported, const DeviceSplit *resident) {
    supported = false;
    D = DevicePlan();
    if (n < 1 || n >= INT32_MAX) return PARS3_OK;
    if (o.skip_empty || !o.cuts.empty() || o.tile_rows > kMaxTileRows || o.tile_rows < 1 || o.seg_max < 1 ||
        o.seg_max > 8 || o.gap < 2 /* (smaller gaps: alignment can merge runs) */ || o.gap > 20 || o.local_slots > 4094 || o.local_slots < 64 ||
        o.max_segments > 32 * PARS3_GPU_MAX_SLICES || o.sink == kNoSlot || o.sink < o.local_slots)
        return PARS3_OK;
    int64_t P_dmax = 0;
    const bool verbose = getenv("PARS3_VERBOSE") != nullptr;
    double t_prev = omp_get_wtime();
    auto lap = [&](const char *what) {
        if (!verbose) return;
        cudaDeviceSynchronize();
        const double now = omp_get_wtime();
        fprintf(stderr, "pars3 plan:   device builder: %-14s %.3f s\n", what, now - t_prev);
        t_prev = now;
    };
    const int64_t nm = mid_ptr[n];
    Buf<int64_t> mptr, optr;
    Buf<int32_t> mcol, ocol, orow;
    Buf<double> mval, oval;
    int rc;
    Split S{};
    S.n = n;
    const int32_t *d_orow = nullptr;
    if (resident) {  // the split is already on this device (prepare_gpu)
        S.mptr = resident->mid_ptr;
        S.mcol = resident->mid_col;
        S.mval = resident->mid_val;
        S.ocol = resident->outer_col;
        S.oval = resident->outer_val;
        d_orow = resident->outer_row;
    } else {
        if ((rc = to_device(mptr, mid_ptr, n + 1)) || (rc = to_device(mcol, mid_col, nm)) ||
            (rc = to_device(mval, mid_val, nm)) || (rc = to_device(orow, outer_row, outer_count)) ||
            (rc = to_device(ocol, outer_col, outer_count)) || (rc = to_device(oval, outer_val, outer_count)))
            return rc;
        S.mptr = mptr.p;
        S.mcol = mcol.p;
        S.mval = mval.p;
        S.ocol = ocol.p;
        S.oval = oval.p;
        d_orow = orow.p;
        lap("upload split");
    }
    RC(optr.alloc(n + 1));
    k_optr<<<(int)std::min<int64_t>((n + kT) / kT, 148 * 32), kT>>>(n, outer_count, d_orow, optr.p);
    RC(cudaGetLastError());
    S.optr = optr.p;
    Opts oo{o.tile_rows, o.local_slots, o.seg_max, o.gap, o.max_segments, o.terms_cap, o.terms_min_rows, o.sink};
    const int64_t nranges = (n + o.tile_rows - 1) / o.tile_rows;
    Buf<DraftTile> draft;
    Buf<int32_t> ntl, flags;
    RC(draft.alloc((size_t)nranges * kMaxRangeTiles));
    RC(ntl.alloc(nranges));
    RC(flags.alloc(8));
    RC(cudaMemset(flags.p, 0, 8 * sizeof(int32_t)));
    const size_t smem = 2 * (kBitmapBits / 8) + kCounters * 2;
    if (cudaFuncSetAttribute((const void *)k_draft, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
        cudaSuccess) {  // (a device without 192 KB of shared memory per CTA: the host builder)
        cudaGetLastError();
        return PARS3_OK;
    }
    k_draft<<<(unsigned)nranges, kT, smem>>>(S, oo, nranges, draft.p, ntl.p, flags.p);
    RC(cudaGetLastError());
    int32_t hf[8] = {0};
    RC(cudaMemcpy(hf, flags.p, sizeof(hf), cudaMemcpyDeviceToHost));
    lap("draft");
    const int32_t hflags = hf[0];
    if (hflags) {  // the host builder takes this plan
        if (getenv("PARS3_VERBOSE"))
            fprintf(stderr, "pars3 plan: device builder declines (reasons %d: 1 span/entries, 2 terms cap, 4 list tile, "
                            "8 tiles per range, 16 hub row, 64 distinct columns); first list range [%d, %d): "
                            "%d starts %d ends, %d distinct columns from %d\n",
                    hflags, hf[2], hf[3], hf[4], hf[5], hf[6], hf[7]);
        return PARS3_OK;
    }
    // tiles per range -> dense tile list
    std::vector<int32_t> hnt(nranges);
    RC(cudaMemcpy(hnt.data(), ntl.p, sizeof(int32_t) * nranges, cudaMemcpyDeviceToHost));
    std::vector<int64_t> htoff(nranges + 1, 0);
    for (int64_t q = 0; q < nranges; q++) htoff[q + 1] = htoff[q] + hnt[q];
    const int64_t nt = htoff[nranges];
    if (nt == 0 || nt >= INT32_MAX) return PARS3_OK;
    Buf<int64_t> toff, woff, soff, voff, uoff;
    Buf<DraftTile> dt;
    if ((rc = to_device(toff, htoff.data(), nranges + 1))) return rc;
    RC(dt.alloc(nt));
    RC(woff.alloc(nt + 1));
    RC(soff.alloc(nt + 1));
    RC(voff.alloc(nt + 1));
    RC(uoff.alloc(nt + 1));
    RC(cudaMemset(uoff.p + nt, 0, sizeof(int64_t)));
    RC(cudaMemset(woff.p + nt, 0, sizeof(int64_t)));
    RC(cudaMemset(soff.p + nt, 0, sizeof(int64_t)));
    RC(cudaMemset(voff.p + nt, 0, sizeof(int64_t)));
    k_sizes<<<(int)((nranges + kT - 1) / kT), kT>>>(nranges, draft.p, ntl.p, toff.p, dt.p, woff.p, soff.p, voff.p,
                                                    uoff.p);
    RC(cudaGetLastError());
    if ((rc = exclusive_scan(woff.p, nt)) || (rc = exclusive_scan(soff.p, nt)) || (rc = exclusive_scan(voff.p, nt)) ||
        (rc = exclusive_scan(uoff.p, nt)))
        return rc;
    int64_t nw = 0, ns = 0, nv = 0, nu = 0;
    RC(cudaMemcpy(&nu, uoff.p + nt, sizeof(int64_t), cudaMemcpyDeviceToHost));
    RC(cudaMemcpy(&nw, woff.p + nt, sizeof(int64_t), cudaMemcpyDeviceToHost));
    RC(cudaMemcpy(&ns, soff.p + nt, sizeof(int64_t), cudaMemcpyDeviceToHost));
    RC(cudaMemcpy(&nv, voff.p + nt, sizeof(int64_t), cudaMemcpyDeviceToHost));
    if (ns >= INT32_MAX || nw >= INT32_MAX || nu >= INT32_MAX) return PARS3_OK;
    Buf<int32_t> ucol;
    RC(ucol.alloc(nu));
    Buf<TileMeta> tiles;
    Buf<Window> wins;
    Buf<int64_t> slice_off;
    Buf<uint8_t> rec;
    Buf<Totals> tot;
    RC(tiles.alloc(nt));
    RC(wins.alloc(nw));
    RC(slice_off.alloc(ns + 1));
    RC(rec.alloc(nv));
    RC(tot.alloc(1));
    RC(cudaMemset(tot.p, 0, sizeof(Totals)));
    k_materialise<false><<<(unsigned)nt, kT>>>(S, oo, nt, dt.p, woff.p, soff.p, voff.p, uoff.p, tiles.p, wins.p,
                                               slice_off.p, rec.p, ucol.p, tot.p);
    RC(cudaGetLastError());
    if (nu > 0) {
        const size_t smem_m = 2 * (kBitmapBits / 8);
        RC(cudaFuncSetAttribute((const void *)k_materialise<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)smem_m));
        k_materialise<true><<<(unsigned)nt, kT, smem_m>>>(S, oo, nt, dt.p, woff.p, soff.p, voff.p, uoff.p, tiles.p,
                                                          wins.p, slice_off.p, rec.p, ucol.p, tot.p);
        RC(cudaGetLastError());
    }
    lap("materialise");
    {  // the most terms one y element sums (HostPlan::dmax)
        Buf<int32_t> terms, best;
        RC(terms.alloc(n));
        RC(best.alloc(1));
        RC(cudaMemset(best.p, 0, sizeof(int32_t)));
        const int G = (int)std::min<int64_t>((n + kT - 1) / kT, 148 * 32);
        k_terms_rows<<<G, kT>>>(S, terms.p);
        if (nm > 0) k_terms_cols<<<148 * 32, kT>>>(nm, S.mcol, terms.p);
        if (outer_count > 0) k_terms_cols<<<148 * 32, kT>>>(outer_count, S.ocol, terms.p);
        k_max_i32<<<G, kT>>>(n, terms.p, best.p);
        RC(cudaGetLastError());
        int32_t hb = 0;
        RC(cudaMemcpy(&hb, best.p, sizeof(int32_t), cudaMemcpyDeviceToHost));
        P_dmax = hb;
    }
    const int64_t end16 = nv / 16;
    RC(cudaMemcpy(slice_off.p + ns, &end16, sizeof(int64_t), cudaMemcpyHostToDevice));
    Totals ht{};
    RC(cudaMemcpy(&ht, tot.p, sizeof(Totals), cudaMemcpyDeviceToHost));
    P = HostPlan();
    P.n = n;
    P.tiles.resize(nt);
    P.wins.resize(nw);
    RC(cudaMemcpy(P.tiles.data(), tiles.p, sizeof(TileMeta) * nt, cudaMemcpyDeviceToHost));
    if (nw > 0) RC(cudaMemcpy(P.wins.data(), wins.p, sizeof(Window) * nw, cudaMemcpyDeviceToHost));
    P.nnz = (int64_t)ht.nnz;
    P.slots = (int64_t)ht.slots;
    P.max_nslots = ht.max_nslots;
    P.max_terms = ht.max_terms;
    P.dmax = P_dmax;
    P.ucol.resize(nu);
    if (nu > 0) RC(cudaMemcpy(P.ucol.data(), ucol.p, sizeof(int32_t) * nu, cudaMemcpyDeviceToHost));
    P.list_tiles = 0;
    for (const TileMeta &m : P.tiles) {
        P.max_local = std::max(P.max_local, m.local);
        P.list_tiles += m.u0 >= 0 ? 1 : 0;
    }
    lap("download");
    D.ntiles = nt;
    D.nwins = nw;
    D.nslices = ns;
    D.rec_bytes = nv;
    D.tiles = tiles.release();
    D.wins = wins.release();
    D.slice_off = slice_off.release();
    D.rec = rec.release();
    supported = true;
    return PARS3_OK;
}

}  // namespace pars3
