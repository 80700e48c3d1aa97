// Windowed tile kernel: the PARS3 product y = A x on one GPU (DESIGN.md
// section 3).
//
// A persistent grid (4 CTAs x 8 warps per SM) claims row tiles in ascending
// order from an atomic counter, two tiles ahead.  Per tile:
//   1. x over the tile's local index space is in shared memory (xs): dense
//      column windows arrive by TMA bulk copies issued during the previous
//      tile's flush; list-mode tiles gather their explicit column list;
//   2. each warp streams SELL-32 slice records (fp64 value + uint16 local
//      column) straight into registers, with the next slice bulk-prefetched
//      into L2: lane l owns one row segment, keeps its row sum in registers
//      (+a_ic * x_c, serial.py:56-57) and adds the mirror -a_ic * x_i
//      (serial.py:58-59) into the tile's shared accumulator of column c --
//      exact-integer fixed point with native 32-bit shared atomics (or fp64);
//   3. every slot's accumulated value (+ diag * x for the tile's own rows)
//      is reduced into y with fire-and-forget fp64 L2 reductions: for own
//      rows this is the reference's owner write (parallel.py:85-95), for
//      columns below the tile the accumulation message (msg_val /
//      MPI_Accumulate, parallel.py:96-113).
// y is zeroed on the stream first (pars3_plan_spmv) or accumulated into
// (pars3_plan_spmv_acc).
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <algorithm>
#include <cstring>
#include <new>

#include "common.h"
#include "locality.h"
#include "tileplan.h"

using pars3::LocalityOrder;
using pars3::HostPlan;
using pars3::PlanOptions;
using pars3::TileMeta;
using pars3::Window;

namespace {

// 4 CTAs per SM x 8 warps (<= 64 registers): 32 warps stream records into
// registers, and the co-resident CTAs overlap each other's per-tile
// window/flush phases.
#ifndef PARS3_THREADS  // build-time shape of the persistent grid (tuning builds)
#define PARS3_THREADS 256
#define PARS3_MIN_BLOCKS 4
#define PARS3_CAP 3200
#define PARS3_MAX_SLICES 256
#endif
constexpr int kThreads = PARS3_THREADS;
constexpr int kMinBlocks = PARS3_MIN_BLOCKS;
constexpr int kWarps = kThreads / 32;
constexpr int kMaxTileSlices = PARS3_MAX_SLICES;  // per-tile slice offset table in shared memory
constexpr int kMaxSlots = 8;          // slots per slice (plan seg_max)
constexpr int kMaxWindowsDev = pars3::kMaxWindows;
constexpr int kLocalExact = PARS3_CAP;  // window slots per tile: x + fp64 acc or two words (16 B/slot)
constexpr int kLocalFixed = PARS3_CAP == 3200 ? 2496 : PARS3_CAP * 4 / 5 / 32 * 32;  // x + 3 words (20 B/slot)
constexpr int kTerms2 = 64;        // two-word fixed point: max terms per slot per tile
// Shared arrays are laid out with a compile-time stride (so the second and
// third accumulator words are an immediate offset from the first): the
// plan's local space, then one spare slot and the SINK slot that padding
// lanes and padding entries of a slice point at (x = 0, never flushed), so
// the stream loop needs no sentinel branches.
template <int kWords>
struct Layout {
    static constexpr int kCap = kWords == 3 ? kLocalFixed : kLocalExact;
    static constexpr int kStride = kCap + 2;
    static constexpr int kSink = kCap + 1;
    static constexpr int kSmem = kStride * (kWords == 3 ? 20 : 16);
};

// Peer mode (DistributedPars3(mode="peer")): the plan's index space is a
// rank's extended range [col_base, hi); columns below its own block belong
// to earlier ranks.  Their x is read straight from the owner's buffer and
// their mirror sums are reduced straight into the owner's inbox, both
// through peer-mapped (NVLink) device pointers: the halo exchange and the
// accumulation messages happen inside the kernel.  Windows never straddle
// a block boundary (the plan cuts them there).
constexpr int kMaxRanks = 8;
struct Peers {
    int32_t nranks;   // 0: single-GPU plan
    int32_t me;
    int64_t col_base;                    // global column of local index 0
    int64_t bs[kMaxRanks + 1];           // block_start (global rows)
    const double *x[kMaxRanks];          // rank r's x block (x[r][g - bs[r]])
    double *y[kMaxRanks];                // rank r's inbox (me: unused, own y is the kernel's y)
};

__device__ __forceinline__ int owner_of(const Peers &pr, int64_t g) {
    int r = 0;
    while (r + 1 < pr.nranks && g >= pr.bs[r + 1]) r++;
    return r;
}

struct DevPlan {
    const TileMeta *tiles;
    const Window *wins;
    const int64_t *slice_off;  // 16-byte units
    const uint8_t *rec;
    const int32_t *ucol;
    const double *diag;
    int32_t *counter;
    int32_t ntiles;
    int32_t watchdog;
    int32_t diag_const;  // 1: every diagonal value equals diag_alpha (strict / shifted skew)
    double diag_alpha;
    unsigned long long *phase_clk;  // PARS3_PHASES=1: per-phase SM cycles (thread 0 of each CTA)
    int32_t pf;  // L2 prefetch of records: bit 0 each tile's records when its metadata is
                 // fetched, bit 1 each warp's slice pf_dist iterations ahead, bit 2 the
                 // next tile's first slices at the end of the stream
    int32_t pf_dist;
    Peers peers;  // multi-GPU peer mode (nranks > 0): columns owned by other ranks
};

__device__ __forceinline__ uint32_t saddr(const void *p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(saddr(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(saddr(bar)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(saddr(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ bool mbar_try(uint64_t *bar, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n}"
        : "=r"(ok)
        : "r"(saddr(bar)), "r"(parity)
        : "memory");
    return ok != 0;
}
// wait for the phase of `bar` with the given parity; `what`/`tag` feed the
// debug watchdog (PARS3_WATCHDOG=1)
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity, int watchdog = 0,
                                          int what = 0, int tag = 0) {
    if (!watchdog) {
        while (!mbar_try(bar, parity)) {
        }
        return;
    }
    for (long long it = 0; !mbar_try(bar, parity); it++) {
        if (it == (1ll << 26)) {
            if ((threadIdx.x & 31) == 0)
                printf("pars3 watchdog: block %d warp %d stuck on mbarrier kind %d tag %d parity %u\n",
                       blockIdx.x, threadIdx.x >> 5, what, tag, parity);
            return;
        }
    }
}
// one TMA bulk copy global -> shared, completion counted on `bar`
__device__ __forceinline__ void bulk_load(void *dst, const void *src, uint32_t bytes,
                                          uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            saddr(dst)),
        "l"(src), "r"(bytes), "r"(saddr(bar))
        : "memory");
}
// TMA bulk prefetch of [p, p + bytes) into L2 (no shared memory, no registers):
// keeps DRAM busy across a CTA's per-tile window/flush phases
__device__ __forceinline__ void bulk_prefetch_l2(const void *p, uint32_t bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}

__device__ __forceinline__ bool tma_window(int lo, int len) { return ((lo | len) & 1) == 0; }

// One tile's metadata and x-window list, copied into shared memory by
// thread 0 one tile ahead (while the previous tile streams), so neither the
// TMA issue nor the flush pays a global round trip.
struct TileCache {
    TileMeta m;
    int32_t nw;  // windows (window mode), 0 for list mode / past the end
    int32_t lo[kMaxWindowsDev], len[kMaxWindowsDev], off[kMaxWindowsDev];
    int32_t own[kMaxWindowsDev];  // peer mode: owning rank of each window (else me)
};

template <bool kPeer>
__device__ __forceinline__ void fetch_tile(const DevPlan &P, int32_t t, TileCache &tc) {
    tc.nw = 0;
    if (t >= P.ntiles) {
        tc.m.s0 = tc.m.s1 = 0;
        return;
    }
    const TileMeta m = P.tiles[t];
    tc.m = m;
    if (P.pf & 1) {  // the whole tile's records into L2
        const int64_t o0 = __ldg(P.slice_off + m.s0), o1 = __ldg(P.slice_off + m.s1);
        for (int64_t o = o0; o < o1; o += 4096)  // 64 KB per bulk prefetch
            bulk_prefetch_l2(P.rec + o * 16, (uint32_t)((o1 - o < 4096 ? o1 - o : 4096) * 16));
    }
    if (m.u0 >= 0) return;
    tc.nw = m.w1 - m.w0;
    for (int w = 0; w < tc.nw; w++) {
        tc.lo[w] = __ldg(&P.wins[m.w0 + w].lo);
        tc.len[w] = __ldg(&P.wins[m.w0 + w].len);
        tc.off[w] = __ldg(&P.wins[m.w0 + w].loff);
        if (kPeer) tc.own[w] = owner_of(P.peers, P.peers.col_base + tc.lo[w]);
    }
}

// a window is moved by TMA when it is 16-byte aligned and local (peer
// windows are gathered with plain loads over NVLink)
template <bool kPeer>
__device__ __forceinline__ bool tma_ok(const Peers &pr, const double *x, const TileCache &tc, int w) {
    if (!kPeer) return tma_window(tc.lo[w], tc.len[w]);  // x is 16-byte aligned, offsets even
    // source, size and shared destination (xs is 128-byte aligned) all 16-byte aligned
    return ((reinterpret_cast<uintptr_t>(x + tc.lo[w]) | (uintptr_t)tc.len[w] * 8 |
             (uintptr_t)tc.off[w] * 8) & 15) == 0 &&
           tc.own[w] == pr.me;
}

// Issue the even-aligned x windows of a cached tile into xs with TMA bulk
// copies; every tile arrives once on xbar (list-mode and past-the-end tiles
// with 0 bytes) so the barrier's phases count tiles.
template <bool kPeer>
__device__ __forceinline__ void issue_x_cached(const Peers &pr, const double *x, const TileCache &tc,
                                              double *xs, uint64_t *xbar) {
    uint32_t bytes = 0;
    for (int w = 0; w < tc.nw; w++)
        if (tma_ok<kPeer>(pr, x, tc, w)) bytes += (uint32_t)tc.len[w] * 8;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    mbar_arrive_tx(xbar, bytes);
    for (int w = 0; w < tc.nw; w++)
        if (tma_ok<kPeer>(pr, x, tc, w))
            bulk_load(xs + tc.off[w], x + tc.lo[w], (uint32_t)tc.len[w] * 8, xbar);
}

// record offsets of a tile's slices into shared memory (LDGSTS, one group)
__device__ __forceinline__ void load_offsets(const DevPlan &P, const TileMeta &m, int64_t *dst,
                                             int tid) {
    const int nn = m.s1 - m.s0;
    for (int i = tid; i <= nn && nn > 0; i += kThreads)
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(saddr(dst + i)),
                     "l"(P.slice_off + m.s0 + i)
                     : "memory");
    asm volatile("cp.async.commit_group;" ::: "memory");
}

// ---- fixed-point accumulation ---------------------------------------------
// A slot's mirror sum is kept as an exact integer Q * 2^(E-50) in three
// 32-bit words (bits 0-19, 20-39, 40+ signed) updated with native
// shared-memory integer adds (fire-and-forget ATOMS.ADD, no CAS loop).
// E = ev + ex + 3 bounds every term of the tile (|v| < 2^ev, |x| < 2^ex,
// a row segment sums <= 8 terms), so |Q| < 2^50 per term, each word takes up
// to 4096 terms (a tile has <= 1024 rows), and the per-term rounding is
// <= 2^(E-51).  Integer adds commute: a tile's accumulation is independent of
// the order in which its warps arrive.
constexpr double kMagic = 6755399441055744.0;  // 1.5 * 2^52
constexpr long long kMagicBits = 0x4338000000000000ll;

__device__ __forceinline__ double fx_value(uint32_t lo, uint32_t mid, uint32_t hi, double unscale) {
    const long long V = ((long long)(int32_t)hi << 40) + ((long long)mid << 20) + (long long)lo;
    return (double)V * unscale;
}

// Two-word variant for tiles whose slots each take <= kTerms2 = 64 terms
// (the plan checks): bits 0-25 in an unsigned word (64 x 2^26 = 2^32) and
// the signed rest (|Q| < 2^50 -> |Q >> 26| < 2^24, 64 terms < 2^30).
// q = fma(t, 2^(50-E), 1.5 * 2^52): the low mantissa bits hold rint(t * 2^(50-E))
// = Q as a two's-complement offset from the magic constant, so the words
// come straight from the two halves of q (bits 0-25, and Q >> 26).
template <int kS>
__device__ __forceinline__ void fx_add2m(uint32_t *w, uint32_t i, double q) {
    const uint32_t blo = (uint32_t)__double2loint(q);
    const uint32_t bhi = (uint32_t)__double2hiint(q) - 0x43380000u;  // Q >> 32
    atomicAdd(w + i, blo & 0x3FFFFFFu);
    atomicAdd(w + kS + i, __funnelshift_r(blo, bhi, 26));
}

template <int kS>
__device__ __forceinline__ void fx_add3m(uint32_t *w, uint32_t i, double q) {
    const uint32_t blo = (uint32_t)__double2loint(q);
    const uint32_t bhi = (uint32_t)__double2hiint(q) - 0x43380000u;
    atomicAdd(w + i, blo & 0xFFFFFu);
    atomicAdd(w + kS + i, __funnelshift_r(blo, bhi, 20) & 0xFFFFFu);
    atomicAdd(w + 2 * kS + i, (uint32_t)((int32_t)bhi >> 8));
}

__device__ __forceinline__ double fx_value2(uint32_t lo, uint32_t hi, double unscale) {
    const long long V = ((long long)(int32_t)hi << 26) + (long long)lo;
    return (double)V * unscale;
}

// kWords: 0 = fp64 shared accumulators (CAS loop per mirror), 2 / 3 =
// exact-integer fixed point in two / three 32-bit words per slot.
// kPeer: multi-GPU peer mode (P.peers); the single-GPU instantiation
// compiles none of it.
template <int kWords, bool kPeer>
__global__ void __launch_bounds__(kThreads, kMinBlocks)
k_tiles(DevPlan P, const double *__restrict__ x, double *__restrict__ y) {
    constexpr bool kFixed = kWords > 0;
    constexpr int S = Layout<kWords>::kStride;
    constexpr uint32_t kSink = Layout<kWords>::kSink;
    extern __shared__ __align__(128) uint8_t dyn[];
    double *xs = reinterpret_cast<double *>(dyn);
    // fp64 mode: acc[S]; fixed mode: two or three uint32 words per slot
    double *acc = xs + S;
    uint32_t *wlo = reinterpret_cast<uint32_t *>(xs + S);
    uint32_t *wmid = wlo + S;  // two-word mode: the high word
    uint32_t *whi = wmid + S;
    __shared__ int64_t s_off[2][kMaxTileSlices + 1];
    __shared__ int32_t s_t[3];  // tiles k, k+1 (known) and k+2 (claimed during tile k)
    __shared__ int32_t s_ex[2];
    __shared__ __align__(8) uint64_t xbar;
    __shared__ TileCache s_tc[2];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    for (int i = tid; i < S; i += kThreads) {
        xs[i] = 0.0;  // the sink's x stays 0
        if (kWords == 3) {
            wlo[i] = wmid[i] = whi[i] = 0u;
        } else if (kWords == 2) {
            wlo[i] = wmid[i] = 0u;
        } else {
            acc[i] = 0.0;
        }
    }
    // PARS3_PHASES=1: thread 0 accumulates SM cycles per phase
    // (totals in shared memory: no registers held across the tile loop)
    __shared__ long long s_clk[6];
    if (tid < 6) s_clk[tid] = 0;
    if (tid == 0) {
        mbar_init(&xbar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        s_t[0] = atomicAdd(P.counter, 1);
        s_t[1] = atomicAdd(P.counter, 1);
        s_ex[0] = s_ex[1] = -1100;
        fetch_tile<kPeer>(P, s_t[0], s_tc[0]);
        issue_x_cached<kPeer>(P.peers, x, s_tc[0], xs, &xbar);
    }
    long long tprev = clock64();
#define PHASE(k)                                  \
    do {                                          \
        if (P.phase_clk && tid == 0) {            \
            const long long now = clock64();      \
            s_clk[k] += now - tprev;              \
            tprev = now;                          \
        }                                         \
    } while (0)
    __syncthreads();
    load_offsets(P, s_tc[0].m, s_off[0], tid);

    for (int k = 0;; k++) {
        const int cur = k & 1, nxt = cur ^ 1;
        const int32_t t = s_t[k % 3];
        if (t >= P.ntiles) break;
        const TileCache &tc = s_tc[cur];
        const int32_t r0 = tc.m.r0, r1 = tc.m.r1, u0 = tc.m.u0, local = tc.m.local;
        const int nsl = tc.m.s1 - tc.m.s0;
        // claim tile k+2 now; the atomic's latency hides behind this tile
        int32_t claimed = 0;
        if (tid == 0) claimed = atomicAdd(P.counter, 1);
        PHASE(0);

        // 1. x over the tile's local slots: windows arrived by TMA (issued
        //    during the previous tile's flush), odd-aligned windows and
        //    list-mode slots gathered here
        const Peers &pr = P.peers;
        if (u0 >= 0) {
            const int32_t *uc = P.ucol + u0;
            for (int i = tid; i < local; i += kThreads) {
                const int c = __ldg(uc + i);
                if (!kPeer) {
                    xs[i] = __ldg(x + c);
                } else {
                    const int64_t g = pr.col_base + c;
                    const int r = owner_of(pr, g);
                    xs[i] = r == pr.me ? __ldg(x + c) : pr.x[r][g - pr.bs[r]];
                }
            }
        } else {
            for (int w = 0; w < tc.nw; w++) {
                if (tma_ok<kPeer>(pr, x, tc, w)) continue;
                const double *src = x + tc.lo[w];
                if (kPeer) {
                    const int r = tc.own[w];
                    if (r != pr.me) src = pr.x[r] + (pr.col_base + tc.lo[w] - pr.bs[r]);
                }
                for (int i = tid; i < tc.len[w]; i += kThreads) xs[tc.off[w] + i] = src[i];
            }
        }
        mbar_wait(&xbar, (uint32_t)(k & 1), P.watchdog, 5, t);
        asm volatile("cp.async.wait_all;" ::: "memory");  // this tile's record offsets
        if (kFixed) {  // tile-wide bound on |x|: max binary exponent over the slots
            // |x| < 2^(be - 1022) for normal x; slots in pairs (16-byte loads)
            // (a subnormal x counts as exponent 1025: the tile is flagged below)
            int e = -1100;
            const double2 *xs2 = reinterpret_cast<const double2 *>(xs);
            for (int i = tid; i < (local + 1) / 2; i += kThreads) {
                const double2 v = xs2[i];  // (an odd tail's mate is inside the stride, not counted)
                const long long q0 = __double_as_longlong(v.x), q1 = __double_as_longlong(v.y);
                int b0 = (int)((q0 >> 52) & 0x7FF), b1 = (int)((q1 >> 52) & 0x7FF);
                if (b0 == 0 && (q0 & 0xFFFFFFFFFFFFFll)) b0 = 2047;
                if (b1 == 0 && (q1 & 0xFFFFFFFFFFFFFll)) b1 = 2047;
                if (2 * i + 1 >= local) b1 = 0;
                e = max(e, max(b0, b1) - 1022);
            }
            e = __reduce_max_sync(0xffffffffu, e);
            if (lane == 0) atomicMax(&s_ex[cur], e);
        }
        __syncthreads();
        PHASE(1);
        if (tid == 0) {
            fetch_tile<kPeer>(P, s_t[(k + 1) % 3], s_tc[nxt]);  // overlaps the stream
            s_ex[nxt] = -1100;
        }
        int E = 0;
        double scale = 0.0, unscale = 0.0;
        if (kFixed) {
            E = tc.m.ev + s_ex[cur] + 3;
            // non-finite or subnormal x, or magnitudes the 2^(50-E) scale
            // cannot carry: the tile's result is not exact -- raise the
            // plan's status flag (the blocking entry points then redo the
            // product with the fp64 kernel, pars3_plan_status)
            if (tid == 0 && (E > 960 || (E < -960 && s_ex[cur] > -1022))) atomicOr(P.counter + 1, 1);
            E = max(-960, min(960, E));
            scale = ldexp(1.0, 50 - E);
            unscale = ldexp(1.0, E - 50);
        }

        // 2. records: each lane owns one row segment of a slice; row sums in
        //    registers, mirrors into the tile's shared accumulators
        for (int i = warp; i < nsl; i += kWarps) {
            if ((P.pf & 2) && lane == 0 && i + P.pf_dist * kWarps < nsl) {
                const int j = i + P.pf_dist * kWarps;
                const int64_t a = s_off[cur][j], b = s_off[cur][j + 1];
                bulk_prefetch_l2(P.rec + a * 16, (uint32_t)((b - a) * 16));
            }
            const uint8_t *rp = P.rec + s_off[cur][i] * 16;
            const int ns = (int)(((s_off[cur][i + 1] - s_off[cur][i]) * 16 - 64) / 320);
            const uint32_t rl = __ldcs(reinterpret_cast<const uint16_t *>(rp) + lane);
            const double *vp = reinterpret_cast<const double *>(rp + 64) + lane;
            const uint16_t *ip = reinterpret_cast<const uint16_t *>(rp + 64 + ns * 256) + lane;
            double v[kMaxSlots];
            uint32_t li[kMaxSlots];
#pragma unroll
            for (int u = 0; u < kMaxSlots; u++) {
                v[u] = 0.0;
                li[u] = kSink;
                if (u < ns) {  // warp-uniform; padding entries are (0, sink)
                    v[u] = __ldcs(vp + 32 * u);
                    li[u] = __ldcs(ip + 32 * u);
                }
            }
            const double xr = xs[rl];
            double c0 = 0.0, c1 = 0.0;  // two row-sum chains: even and odd slots
            if (kFixed) {
                const double nxs = -xr * scale;  // mirror term v * (-x_r), scaled
#pragma unroll
                for (int u = 0; u < kMaxSlots; u++) {
                    if (u < ns) {
                        if (u & 1)
                            c1 = fma(v[u], xs[li[u]], c1);
                        else
                            c0 = fma(v[u], xs[li[u]], c0);
                        const double q = fma(v[u], nxs, kMagic);
                        if (kWords == 3)
                            fx_add3m<S>(wlo, li[u], q);
                        else
                            fx_add2m<S>(wlo, li[u], q);
                    }
                }
                const double q = fma(c0 + c1, scale, kMagic);
                if (kWords == 3)
                    fx_add3m<S>(wlo, rl, q);
                else
                    fx_add2m<S>(wlo, rl, q);
            } else {
#pragma unroll
                for (int u = 0; u < kMaxSlots; u++) {
                    if (u < ns) {
                        if (u & 1)
                            c1 = fma(v[u], xs[li[u]], c1);
                        else
                            c0 = fma(v[u], xs[li[u]], c0);
                        atomicAdd(&acc[li[u]], -v[u] * xr);
                    }
                }
                atomicAdd(&acc[rl], c0 + c1);
            }
        }
        if (tid == 0) {
            s_t[(k + 2) % 3] = claimed;
            if (P.pf & 4) {  // warm L2 with the next tile's first slices
                const TileMeta &mn = s_tc[nxt].m;
                const int q1 = min(mn.s1, mn.s0 + kWarps * P.pf_dist);
                if (q1 > mn.s0) {
                    const int64_t a = __ldg(P.slice_off + mn.s0), b = __ldg(P.slice_off + q1);
                    bulk_prefetch_l2(P.rec + a * 16, (uint32_t)((b - a) * 16));
                }
            }
        }
        __syncthreads();
        PHASE(2);

        // 3. xs is free: the next tile's x windows and record offsets are
        //    issued first, so they land while this tile flushes
        if (tid == 0) issue_x_cached<kPeer>(P.peers, x, s_tc[nxt], xs, &xbar);
        load_offsets(P, s_tc[nxt].m, s_off[nxt], tid);
        PHASE(4);

        // 4. deliver: every slot's value (own rows + diag * x, x of own rows
        //    from global: xs already holds the next tile) reduces into y with
        //    a fire-and-forget fp64 red (consecutive slots -> coalesced L2
        //    reductions); the accumulators are cleared in the same pass
        auto take = [&](int i) -> double {
            if (kWords == 3) {
                const double a = fx_value(wlo[i], wmid[i], whi[i], unscale);
                wlo[i] = wmid[i] = whi[i] = 0u;
                return a;
            }
            if (kWords == 2) {
                const double a = fx_value2(wlo[i], wmid[i], unscale);
                wlo[i] = wmid[i] = 0u;
                return a;
            }
            const double a = acc[i];
            acc[i] = 0.0;
            return a;
        };
        if (u0 >= 0) {
            const int32_t *uc = P.ucol + u0;
            const int nmsg = local - (r1 - r0);  // own rows are the tail of the list
            for (int i = tid; i < local; i += kThreads) {
                double a = take(i);
                const int c = __ldg(uc + i);
                double *dst = y + c;
                bool mine = true;
                if (kPeer) {  // a column of an earlier rank: its inbox, over NVLink
                    const int64_t g = pr.col_base + c;
                    const int r = owner_of(pr, g);
                    if (r != pr.me) {
                        dst = pr.y[r] + (g - pr.bs[r]);
                        mine = false;
                    }
                }
                if (i >= nmsg && mine)  // (a halo row's diagonal belongs to its owner)
                    a = fma(P.diag_const ? P.diag_alpha : __ldg(P.diag + c), __ldg(x + c), a);
                if (a != 0.0) atomicAdd(dst, a);
            }
        } else {
            for (int w = 0; w < tc.nw; w++) {
                const int lo = tc.lo[w], len = tc.len[w], off = tc.off[w];
                // own columns reduce into y; an earlier rank's columns into its
                // inbox over NVLink (peer mode; their diagonal is the owner's)
                bool mine = true;
                double *dst = y + lo;
                if (kPeer) {
                    const int r = tc.own[w];
                    if (r != pr.me) {
                        mine = false;
                        dst = pr.y[r] + (pr.col_base + lo - pr.bs[r]);
                    }
                }
                for (int i = tid; i < len; i += kThreads) {
                    const int c = lo + i;
                    double a = take(off + i);
                    if (mine && c >= r0 && c < r1)
                        a = fma(P.diag_const ? P.diag_alpha : __ldg(P.diag + c), __ldg(x + c), a);
                    if (a != 0.0) atomicAdd(dst + i, a);
                }
            }
        }
        __syncthreads();
        PHASE(3);
    }
    // peer mode: this CTA's reductions into other GPUs' inboxes are performed
    // system-wide before the kernel completes (the barrier after the product
    // is stream-ordered behind it)
    if (kPeer) __threadfence_system();
    if (P.phase_clk && tid == 0)
        for (int k = 0; k < 6; k++) atomicAdd(P.phase_clk + k, (unsigned long long)s_clk[k]);
#undef PHASE
}

// <a, b>: 16-byte loads, four in flight per thread, one fp64 atomic per block
__global__ void __launch_bounds__(512) k_dot(int32_t n, const double *__restrict__ a,
                                             const double *__restrict__ b, double *out) {
    double s = 0.0;
    const int64_t n2 = n / 2;
    const double2 *a2 = reinterpret_cast<const double2 *>(a);
    const double2 *b2 = reinterpret_cast<const double2 *>(b);
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    for (; i + 3 * stride < n2; i += 4 * stride) {
        double2 x[4], z[4];
#pragma unroll
        for (int u = 0; u < 4; u++) {
            x[u] = __ldcs(a2 + i + u * stride);
            z[u] = __ldcs(b2 + i + u * stride);
        }
#pragma unroll
        for (int u = 0; u < 4; u++) s = fma(x[u].y, z[u].y, fma(x[u].x, z[u].x, s));
    }
    for (; i < n2; i += stride) {
        const double2 x = __ldcs(a2 + i), z = __ldcs(b2 + i);
        s = fma(x.y, z.y, fma(x.x, z.x, s));
    }
    if (blockIdx.x == 0 && threadIdx.x == 0 && (n & 1)) s = fma(a[n - 1], b[n - 1], s);
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    __shared__ double ws[16];
    if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x < 32) {
        s = threadIdx.x < 16 ? ws[threadIdx.x] : 0.0;
        for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if (threadIdx.x == 0) atomicAdd(out, s);
    }
}

// locality order (locality.cpp): xs[j] = x[inv[j]] (gather: the random
// accesses are reads, the writes stream; the scatter form xs[perm[i]] = x[i]
// measured 42 against 22 us on c3)
__global__ void __launch_bounds__(512) k_perm_in(int32_t n, const int32_t *__restrict__ inv,
                                                 const double *__restrict__ x, double *__restrict__ xs) {
    const int32_t stride = gridDim.x * blockDim.x;
    int32_t j = blockIdx.x * blockDim.x + threadIdx.x;
    for (; j + 3 * stride < n; j += 4 * stride) {  // four independent gathers in flight
        int32_t q[4];
        double v[4];
#pragma unroll
        for (int u = 0; u < 4; u++) q[u] = __ldcs(inv + j + u * stride);
#pragma unroll
        for (int u = 0; u < 4; u++) v[u] = __ldg(x + q[u]);
#pragma unroll
        for (int u = 0; u < 4; u++) __stcs(xs + j + u * stride, v[u]);
    }
    for (; j < n; j += stride) __stcs(xs + j, __ldg(x + __ldcs(inv + j)));
}

// y[i] = (acc ? y[i] : 0) + ys[perm[i]]; with dot: *dot += <y, w> (w == y allowed)
template <bool kAcc, bool kDot>
__global__ void __launch_bounds__(512) k_perm_out(int32_t n, const int32_t *__restrict__ perm,
                                                  const double *__restrict__ ys, double *y,
                                                  const double *w, double *dot) {
    const int32_t stride = gridDim.x * blockDim.x;
    double s = 0.0;
    int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    for (; i + 3 * stride < n; i += 4 * stride) {  // four independent gathers in flight
        int32_t q[4];
        double v[4];
#pragma unroll
        for (int u = 0; u < 4; u++) q[u] = __ldcs(perm + i + u * stride);
#pragma unroll
        for (int u = 0; u < 4; u++) v[u] = ys[q[u]];
#pragma unroll
        for (int u = 0; u < 4; u++) {
            const int32_t k = i + u * stride;
            if (kAcc) v[u] += y[k];
            if (kDot) s = fma(v[u], w == y ? v[u] : w[k], s);
            y[k] = v[u];
        }
    }
    for (; i < n; i += stride) {
        double v = ys[__ldcs(perm + i)];
        if (kAcc) v += y[i];
        if (kDot) s = fma(v, w == y ? v : w[i], s);
        y[i] = v;
    }
    if (!kDot) return;
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    __shared__ double ws[16];
    if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x < 32) {
        s = threadIdx.x < 16 ? ws[threadIdx.x] : 0.0;
        for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if (threadIdx.x == 0) atomicAdd(dot, s);
    }
}

// Direct mode (plans whose tiles would hold about one entry per shared
// slot, e.g. c4's R-MAT): no shared staging.  y = d.x (+ y) first, then
// every stored entry a_rc gathers x_c into its row's register sum and
// reduces -a_rc x_r straight into y_c (fp64 red.global.add, L2).  Each lane
// owns kDirectRun consecutive entries (row-major) and issues all their x
// gathers at once, so long rows spread over lanes and warps (nnz-balanced),
// and a lane reduces its row sum once per row run.

__global__ void __launch_bounds__(512) k_direct_init(int32_t n, const double *__restrict__ diag,
                                                     double alpha, const double *__restrict__ x,
                                                     double *y, int acc) {
    const int32_t stride = gridDim.x * blockDim.x;
    for (int32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
        const double d = diag ? diag[i] : alpha;
        const double v = d * __ldg(x + i);
        y[i] = acc ? y[i] + v : v;
    }
}

template <int kDirectRun>
__global__ void __launch_bounds__(256) k_direct(int64_t m, const int32_t *__restrict__ row,
                                                const int32_t *__restrict__ col,
                                                const double *__restrict__ val,
                                                const double *__restrict__ x, double *y) {
    const int64_t nrun = (m + kDirectRun - 1) / kDirectRun;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < nrun; t += stride) {
        const int64_t e0 = t * kDirectRun;
        int32_t r[kDirectRun], c[kDirectRun];
        double v[kDirectRun];
        if (e0 + kDirectRun <= m) {  // 16-byte loads (the arrays are 16-byte aligned, runs of 8)
            const int4 *r4 = reinterpret_cast<const int4 *>(row + e0);
            const int4 *c4 = reinterpret_cast<const int4 *>(col + e0);
            const double2 *v2 = reinterpret_cast<const double2 *>(val + e0);
#pragma unroll
            for (int h = 0; h < kDirectRun / 4; h++) {
                const int4 a = __ldcs(r4 + h), b = __ldcs(c4 + h);
                r[4 * h] = a.x; r[4 * h + 1] = a.y; r[4 * h + 2] = a.z; r[4 * h + 3] = a.w;
                c[4 * h] = b.x; c[4 * h + 1] = b.y; c[4 * h + 2] = b.z; c[4 * h + 3] = b.w;
            }
#pragma unroll
            for (int h = 0; h < kDirectRun / 2; h++) {
                const double2 a = __ldcs(v2 + h);
                v[2 * h] = a.x;
                v[2 * h + 1] = a.y;
            }
        } else {
#pragma unroll
            for (int j = 0; j < kDirectRun; j++) {
                const bool in = e0 + j < m;
                r[j] = in ? row[e0 + j] : (j ? r[j - 1] : 0);
                c[j] = in ? col[e0 + j] : -1;  // -1: past the end
                v[j] = in ? val[e0 + j] : 0.0;
            }
        }
        double xc[kDirectRun];
#pragma unroll
        for (int j = 0; j < kDirectRun; j++) xc[j] = c[j] >= 0 ? __ldg(x + c[j]) : 0.0;  // all in flight
        int32_t cur = r[0];
        double xr = __ldg(x + cur), acc = 0.0;
#pragma unroll
        for (int j = 0; j < kDirectRun; j++) {
            if (r[j] != cur) {
                atomicAdd(y + cur, acc);
                cur = r[j];
                xr = __ldg(x + cur);
                acc = 0.0;
            }
            if (c[j] < 0) break;
            acc = fma(v[j], xc[j], acc);
            atomicAdd(y + c[j], -v[j] * xr);
        }
        atomicAdd(y + cur, acc);
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
    int grid = 0;
    size_t smem = 0;
    TileMeta *tiles = nullptr;
    Window *wins = nullptr;
    int64_t *slice_off = nullptr;
    uint8_t *rec = nullptr;
    int32_t *ucol = nullptr;
    double *diag = nullptr;
    int32_t list_tiles = 0, watchdog = 0, diag_const = 0, words = 0, pf = 0, pf_dist = 1;
    double diag_alpha = 0.0;
    unsigned long long *phase_clk = nullptr;
    int32_t *counter = nullptr;
    int64_t bytes = 0;
    Peers peers{};
    // internal locality order (locality.cpp): the tiles hold P A P^T, x and
    // y pass through perm (split label -> internal label) and xs / ys
    int32_t *perm = nullptr, *iperm = nullptr;
    double *xs = nullptr, *ys = nullptr;
    int64_t local_slots = 0, dropped = 0;
    // direct mode (k_direct): row-major entries, no tiles
    int32_t direct = 0, direct_run = 16;  // entries per lane: 16 measured best on c4 (4: 1.00 ms,
                                          // 8: 0.89, 16: 0.83; profiles/r01/sweep_direct_run_c4.txt)
    int64_t dm = 0;
    int32_t *drow = nullptr, *dcol = nullptr;
    double *dval = nullptr;

    ~pars3_plan() {
        void *ptrs[] = {tiles, wins, slice_off, rec, ucol, diag, counter, phase_clk, perm, iperm, xs, ys,
                        drow, dcol, dval};
        for (void *q : ptrs)
            if (q) cudaFree(q);
    }
};

// fixed-point accumulation needs finite values in [2^-900, 2^900] (or 0)
static bool values_fixed_point_safe(const pars3_split_view *s) {
    const int64_t nm = s->mid_ptr ? s->mid_ptr[s->n] : 0;
    bool ok = true;
    auto check = [&](const double *v, int64_t k) {
#pragma omp parallel for reduction(&& : ok)
        for (int64_t i = 0; i < k; i++) {
            const double a = std::fabs(v[i]);
            ok = ok && (a == 0.0 || (a >= 0x1p-900 && a <= 0x1p900));
        }
    };
    if (nm > 0) check(s->mid_val, nm);
    if (s->outer_count > 0) check(s->outer_val, s->outer_count);
    return ok;
}

extern "C" int pars3_plan_create(const pars3_split_view *s, const pars3_plan_options *opt,
                                 int32_t p, const int64_t *block_start, pars3_plan **out,
                                 void *stream) {
    (void)stream;
    if (!s || !out) PARS3_FAIL(PARS3_ERR_ARG, "null argument");
    *out = nullptr;
    if (s->n < 0 || s->n >= INT32_MAX || s->beta < 1) PARS3_FAIL(PARS3_ERR_ARG, "bad split header");
    if (p < 1) PARS3_FAIL(PARS3_ERR_ARG, "worker count must be at least 1, got %d", p);
    PlanOptions o0;
    int32_t max_ctas = 0, flags = 0;
    if (opt) {
        if (opt->tile_rows > 0) o0.tile_rows = opt->tile_rows;
        if (opt->local_slots > 0) o0.local_slots = opt->local_slots;
        if (opt->seg_max > 0) o0.seg_max = opt->seg_max;
        if (opt->gap >= 0) o0.gap = opt->gap;
        if (opt->mode > 0) o0.mode = opt->mode;
        o0.skip_empty = (opt->flags & PARS3_PLAN_SKIP_EMPTY) != 0;
        if ((opt->flags & PARS3_PLAN_CUT_BLOCKS) && block_start && p > 1)
            for (int32_t r = 1; r < p; r++) o0.cuts.push_back((int32_t)block_start[r]);
        if (opt->max_ctas > 0) max_ctas = opt->max_ctas;
        flags = opt->flags;
    }
    if (const char *ff = getenv("PARS3_FORCE_FLAGS")) flags |= atoi(ff);  // debug / tuning knob
    // accumulation of the mirror sums: mode 2 = fp64 shared accumulators,
    // mode 1 = exact-integer fixed point in three words, mode 3 = two words
    // (needs <= kTerms2 terms per slot and tile), mode 0 = auto: two words
    // when the plan allows, else fp64 for window-structured matrices and
    // three words when most tiles are unstructured list tiles
    const int req_mode = opt ? opt->mode : 0;
    int words0 = req_mode == 1 ? 3 : req_mode == 2 ? 0 : 2;
    if (words0 && !values_fixed_point_safe(s)) words0 = 0;  // fp64 accumulators keep IEEE semantics
    // the shared-memory budget (x + accumulators per slot, 4 CTAs / SM) caps both
    if (o0.seg_max > 8) o0.seg_max = 8;
    const int32_t want_local = o0.local_slots;
    o0.max_segments = std::min(o0.max_segments, 32 * kMaxTileSlices);
    auto build = [&](const pars3_split_view *v, PlanOptions &o, int &words, HostPlan &hp) -> int {
        o = o0;
        words = words0;
        o.terms_cap = words == 2 ? kTerms2 : 0;
        if (const char *ts = getenv("PARS3_TERMS_MIN_ROWS")) o.terms_min_rows = atoi(ts);  // tuning knob
        o.local_slots = std::min(want_local, words == 3 ? kLocalFixed : kLocalExact);
        o.sink = (uint16_t)(words == 3 ? Layout<3>::kSink : Layout<0>::kSink);
        int rc = pars3::build_tile_plan(v->n, v->mid_ptr, v->mid_col, v->mid_val, v->outer_count,
                                        v->outer_row, v->outer_col, v->outer_val, o, hp);
        if (rc) return rc;
        if (words == 2 && hp.max_terms > kTerms2) {
            if (req_mode == 3)
                PARS3_FAIL(PARS3_ERR_ARG, "two-word accumulation needs <= %d terms per slot, plan has %d",
                           kTerms2, hp.max_terms);
            words = 0;
            if (4ll * hp.list_tiles > (int64_t)hp.tiles.size()) {
                words = 3;
                o.terms_cap = 0;
                o.local_slots = std::min(want_local, kLocalFixed);
                o.sink = (uint16_t)Layout<3>::kSink;
                hp = HostPlan();
                rc = pars3::build_tile_plan(v->n, v->mid_ptr, v->mid_col, v->mid_val, v->outer_count,
                                            v->outer_row, v->outer_col, v->outer_val, o, hp);
                if (rc) return rc;
            }
        }
        return PARS3_OK;
    };
    auto local_of = [](const HostPlan &hp) {
        int64_t t = 0;
        for (const TileMeta &m : hp.tiles) t += m.local;
        return t;
    };
    PlanOptions o;
    int words = 0;
    HostPlan hp;
    int rc = build(s, o, words, hp);
    if (rc) return rc;
    int64_t local = local_of(hp);
    // internal locality order (locality.cpp): tried when most tiles are
    // unstructured list tiles whose slots hold few entries each, kept when
    // it cuts the shared-memory slots (= x gathers + y reductions) by 30 %
    LocalityOrder lo;
    const bool may_permute =
        !(flags & (PARS3_PLAN_CUT_BLOCKS | PARS3_PLAN_NO_LOCALITY | PARS3_PLAN_DIRECT)) && s->n > 1;
    const bool unstructured = 2ll * hp.list_tiles > (int64_t)hp.tiles.size() && 4 * local > hp.nnz;
    if (may_permute && (unstructured || (flags & PARS3_PLAN_LOCALITY)) && hp.nnz > 0) {
        rc = pars3::locality_order(s, lo);
        if (rc) return rc;
        pars3_split_view v{s->n, s->beta, lo.diag.data(), lo.row_ptr.data(), lo.col.data(),
                           lo.val.data(), 0, nullptr, nullptr, nullptr};
        PlanOptions o2;
        int words2 = 0;
        HostPlan hp2;
        rc = build(&v, o2, words2, hp2);
        if (rc) return rc;
        const int64_t local2 = local_of(hp2);
        if (10 * local2 < 7 * local) {
            o = o2;
            words = words2;
            hp = std::move(hp2);
            local = local2;
        } else {
            lo = LocalityOrder();
        }
    }
    // direct mode: the tiles would stage about one entry per slot (no reuse
    // of x or of the accumulators in shared memory), or a mid-size matrix
    // whose tiles would leave most of the persistent grid idle (c2: 256
    // tiles, a latency-bound chain per tile; direct measured 17 % faster)
    int sms_now = 148;
    {
        int dev_now = 0;
        if (cudaGetDevice(&dev_now) == cudaSuccess)
            cudaDeviceGetAttribute(&sms_now, cudaDevAttrMultiProcessorCount, dev_now);
    }
    const bool few_tiles = (int64_t)hp.tiles.size() < 2ll * sms_now && hp.nnz >= (1 << 19);
    const bool direct =
        lo.forward.empty() && hp.nnz > 0 &&
        !(flags & (PARS3_PLAN_CUT_BLOCKS | PARS3_PLAN_SKIP_EMPTY | PARS3_PLAN_NO_DIRECT)) &&
        ((flags & PARS3_PLAN_DIRECT) || few_tiles ||
         (2ll * hp.list_tiles > (int64_t)hp.tiles.size() && 10 * local >= 9 * hp.nnz));
    std::vector<int32_t> drow, dcol;
    std::vector<double> dval;
    if (direct) {  // row-major entries: a row's outer entries, then its middle ones
        try {
            const int64_t m = (s->mid_ptr ? s->mid_ptr[s->n] : 0) + s->outer_count;
            drow.resize(m);
            dcol.resize(m);
            dval.resize(m);
            int64_t o_k = 0, e = 0;
            for (int64_t i = 0; i < s->n; i++) {
                for (; o_k < s->outer_count && s->outer_row[o_k] == i; o_k++, e++) {
                    drow[e] = (int32_t)i;
                    dcol[e] = s->outer_col[o_k];
                    dval[e] = s->outer_val[o_k];
                }
                for (int64_t k = s->mid_ptr[i]; k < s->mid_ptr[i + 1]; k++, e++) {
                    drow[e] = (int32_t)i;
                    dcol[e] = s->mid_col[k];
                    dval[e] = s->mid_val[k];
                }
            }
            if (e != m) PARS3_FAIL(PARS3_ERR_STRUCT, "outer rows are not sorted");
        } catch (const std::bad_alloc &) {
            PARS3_FAIL(PARS3_ERR_NOMEM, "out of host memory");
        }
        hp = HostPlan();  // no tiles are uploaded
        hp.nnz = (int64_t)dval.size();
    }
    pars3_plan *pl = new (std::nothrow) pars3_plan;
    if (!pl) PARS3_FAIL(PARS3_ERR_NOMEM, "out of host memory");
    pl->n = s->n;
    pl->beta = s->beta;
    pl->p = p;
    pl->ntiles = (int32_t)hp.tiles.size();
    pl->nslices = std::max<int32_t>(0, (int32_t)hp.slice_off.size() - 1);
    pl->lmax = hp.max_local;
    pl->nnz = hp.nnz;
    pl->slots = hp.slots;
    pl->nwins = (int64_t)hp.wins.size();
    pl->list_tiles = hp.list_tiles;
    pl->words = words;
    {  // tuning and debug knobs (environment)
        const char *wd = getenv("PARS3_WATCHDOG");
        pl->watchdog = (wd && wd[0] == '1') ? 1 : 0;
        const char *pf = getenv("PARS3_PF");
        pl->pf = pf ? atoi(pf) : 6;  // measured best on c5 (profiles/r01/sweep_pf*.txt)
        const char *pd = getenv("PARS3_PF_DIST");
        pl->pf_dist = pd ? std::max(1, atoi(pd)) : 1;
        const char *ph = getenv("PARS3_PHASES");
        if (ph && ph[0] == '1') {
            cudaMalloc((void **)&pl->phase_clk, 8 * sizeof(unsigned long long));
            cudaMemset(pl->phase_clk, 0, 8 * sizeof(unsigned long long));
        }
    }
    pl->local_slots = local;
    pl->dropped = lo.dropped;
    std::vector<double> diag = lo.forward.empty() ? std::vector<double>(s->diag, s->diag + s->n)
                                                  : std::move(lo.diag);
    pl->diag_const = 1;
    pl->diag_alpha = s->n ? diag[0] : 0.0;
    for (int64_t i = 1; i < s->n && pl->diag_const; i++)
        if (diag[i] != diag[0]) pl->diag_const = 0;
#define UP(dst, src)                               \
    do {                                           \
        int _r = upload(&pl->dst, src);            \
        if (_r) {                                  \
            delete pl;                             \
            return _r;                             \
        }                                          \
        pl->bytes += sizeof(src[0]) * src.size();  \
    } while (0)
    if (direct) {
        pl->direct = 1;
        if (const char *dr = getenv("PARS3_DIRECT_RUN")) pl->direct_run = atoi(dr);  // tuning knob
        if (pl->direct_run != 4 && pl->direct_run != 8) pl->direct_run = 16;
        pl->dm = (int64_t)dval.size();
        UP(drow, drow);
        UP(dcol, dcol);
        UP(dval, dval);
    }
    UP(tiles, hp.tiles);
    UP(wins, hp.wins);
    UP(slice_off, hp.slice_off);
    UP(rec, hp.rec);
    UP(ucol, hp.ucol);
    if (!pl->diag_const) UP(diag, diag);
    if (!lo.forward.empty()) {
        UP(perm, lo.forward);
        std::vector<int32_t> inv(lo.forward.size());
        for (size_t i = 0; i < inv.size(); i++) inv[lo.forward[i]] = (int32_t)i;
        UP(iperm, inv);
        if (cudaMalloc((void **)&pl->xs, sizeof(double) * (size_t)pl->n) != cudaSuccess ||
            cudaMalloc((void **)&pl->ys, sizeof(double) * (size_t)pl->n) != cudaSuccess) {
            delete pl;
            PARS3_FAIL(PARS3_ERR_CUDA, "cudaMalloc failed");
        }
        pl->bytes += 2 * sizeof(double) * pl->n;
    }
#undef UP
    if (cudaMalloc((void **)&pl->counter, 2 * sizeof(int32_t)) != cudaSuccess ||  // claims, status
        cudaMemset(pl->counter, 0, 2 * sizeof(int32_t)) != cudaSuccess) {
        delete pl;
        PARS3_FAIL(PARS3_ERR_CUDA, "cudaMalloc failed");
    }
    pl->smem = pl->words == 0 ? Layout<0>::kSmem : pl->words == 2 ? Layout<2>::kSmem : Layout<3>::kSmem;
    // the attribute is per function, shared by every plan: set it to the
    // function's fixed layout size
    cudaError_t e = cudaSuccess;
    {
        const void *fns[6] = {(const void *)k_tiles<0, false>, (const void *)k_tiles<2, false>,
                              (const void *)k_tiles<3, false>, (const void *)k_tiles<0, true>,
                              (const void *)k_tiles<2, true>,  (const void *)k_tiles<3, true>};
        const int sm[3] = {Layout<0>::kSmem, Layout<2>::kSmem, Layout<3>::kSmem};
        for (int f = 0; f < 6 && e == cudaSuccess; f++)
            e = cudaFuncSetAttribute(fns[f], cudaFuncAttributeMaxDynamicSharedMemorySize, sm[f % 3]);
    }
    int per_sm = 0, sms = 0, dev = 0;
    if (e == cudaSuccess) e = cudaGetDevice(&dev);
    if (e == cudaSuccess) e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (e == cudaSuccess)
        e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(
            &per_sm, pl->words == 0 ? k_tiles<0, false> : pl->words == 2 ? k_tiles<2, false> : k_tiles<3, false>,
            kThreads,
            pl->smem);
    if (e != cudaSuccess || per_sm < 1) {
        delete pl;
        PARS3_FAIL(PARS3_ERR_CUDA, "tile kernel cannot be resident (smem %zu B): %s", pl->smem,
                   cudaGetErrorString(e));
    }
    pl->grid = per_sm * sms;
    if (max_ctas > 0 && pl->grid > max_ctas) pl->grid = max_ctas;
    if (pl->grid > pl->ntiles) pl->grid = pl->ntiles > 0 ? pl->ntiles : 1;
    *out = pl;
    return PARS3_OK;
}

static int launch_tiles(pars3_plan *pl, const double *x, double *y, bool zero_y, cudaStream_t st) {
    if (pl->direct) {
        if (pl->n == 0) return PARS3_OK;
        const int grid = (int)std::min<int64_t>(148 * 4, (pl->n + 511) / 512);
        k_direct_init<<<grid, 512, 0, st>>>((int32_t)pl->n, pl->diag_const ? nullptr : pl->diag,
                                            pl->diag_alpha, x, y, zero_y ? 0 : 1);
        LAUNCH_CHECK();
        const int run = pl->direct_run;
        const int64_t runs = (pl->dm + run - 1) / run;
        const int grid2 = (int)std::min<int64_t>(148 * 16, (runs + 255) / 256);
        if (grid2 > 0) {
            auto fn = run == 4 ? k_direct<4> : run == 16 ? k_direct<16> : k_direct<8>;
            fn<<<grid2, 256, 0, st>>>(pl->dm, pl->drow, pl->dcol, pl->dval, x, y);
            LAUNCH_CHECK();
        }
        return PARS3_OK;
    }
    if (zero_y && pl->n > 0) CUDA_TRY(cudaMemsetAsync(y, 0, sizeof(double) * (size_t)pl->n, st));
    if (pl->ntiles == 0) return PARS3_OK;
    CUDA_TRY(cudaMemsetAsync(pl->counter, 0, 2 * sizeof(int32_t), st));
    DevPlan P{pl->tiles,      pl->wins,       pl->slice_off, pl->rec,       pl->ucol,
              pl->diag,       pl->counter,    pl->ntiles,    pl->watchdog,  pl->diag_const,
              pl->diag_alpha, pl->phase_clk,  pl->pf,        pl->pf_dist,  pl->peers};
    const bool peer = pl->peers.nranks > 0;
    if (pl->words == 0)
        (peer ? k_tiles<0, true> : k_tiles<0, false>)<<<pl->grid, kThreads, pl->smem, st>>>(P, x, y);
    else if (pl->words == 2)
        (peer ? k_tiles<2, true> : k_tiles<2, false>)<<<pl->grid, kThreads, pl->smem, st>>>(P, x, y);
    else
        (peer ? k_tiles<3, true> : k_tiles<3, false>)<<<pl->grid, kThreads, pl->smem, st>>>(P, x, y);
    LAUNCH_CHECK();
    return PARS3_OK;
}

extern "C" int pars3_plan_set_peers(pars3_plan *pl, int32_t nranks, int32_t me, int64_t col_base,
                                    const int64_t *block_start, const uint64_t *x_ptrs,
                                    const uint64_t *inbox_ptrs) {
    if (!pl) PARS3_FAIL(PARS3_ERR_ARG, "null plan");
    if ((pl->perm || pl->direct) && nranks != 0)
        PARS3_FAIL(PARS3_ERR_ARG, "peer mode needs a plan without a locality order (PARS3_PLAN_NO_LOCALITY)");
    if (nranks == 0) {
        pl->peers = Peers{};
        return PARS3_OK;
    }
    if (nranks < 1 || nranks > kMaxRanks || me < 0 || me >= nranks || !block_start || !x_ptrs ||
        !inbox_ptrs)
        PARS3_FAIL(PARS3_ERR_ARG, "peer mode needs 1..%d ranks, a rank id and %d pointers", kMaxRanks,
                   nranks);
    if (col_base < 0 || col_base + pl->n > block_start[nranks] || block_start[0] != 0)
        PARS3_FAIL(PARS3_ERR_ARG, "plan index space [%lld, %lld) outside the blocks",
                   (long long)col_base, (long long)(col_base + pl->n));
    Peers pr{};
    pr.nranks = nranks;
    pr.me = me;
    pr.col_base = col_base;
    for (int r = 0; r <= nranks; r++) pr.bs[r] = block_start[r];
    for (int r = 0; r < nranks; r++) {
        pr.x[r] = reinterpret_cast<const double *>(x_ptrs[r]);
        pr.y[r] = reinterpret_cast<double *>(inbox_ptrs[r]);
    }
    pl->peers = pr;
    return PARS3_OK;
}

// one product through the plan; with a locality order the tiles run on the
// internal copies xs / ys and the epilogue gathers y (and the dot) back
static int plan_product(pars3_plan *pl, const double *x, double *y, bool acc, const double *w,
                        double *dot, cudaStream_t st) {
    if (dot) CUDA_TRY(cudaMemsetAsync(dot, 0, sizeof(double), st));
    if (!pl->perm) {
        int rc = launch_tiles(pl, x, y, !acc, st);
        if (rc || !dot || pl->n == 0) return rc;
        // 16-byte loads need 16-byte aligned vectors (torch allocations are)
        if (((uintptr_t)y | (uintptr_t)w) & 15) PARS3_FAIL(PARS3_ERR_ARG, "y and w must be 16-byte aligned");
        k_dot<<<148 * 4, 512, 0, st>>>((int32_t)pl->n, y, w, dot);
        LAUNCH_CHECK();
        return PARS3_OK;
    }
    const int32_t n = (int32_t)pl->n;
    const int grid = (int)std::min<int64_t>(148 * 4, (pl->n + 511) / 512);
    k_perm_in<<<grid, 512, 0, st>>>(n, pl->iperm, x, pl->xs);
    LAUNCH_CHECK();
    int rc = launch_tiles(pl, pl->xs, pl->ys, true, st);
    if (rc) return rc;
    if (acc)
        (dot ? k_perm_out<true, true> : k_perm_out<true, false>)<<<grid, 512, 0, st>>>(n, pl->perm, pl->ys, y, w, dot);
    else
        (dot ? k_perm_out<false, true> : k_perm_out<false, false>)<<<grid, 512, 0, st>>>(n, pl->perm, pl->ys, y, w, dot);
    LAUNCH_CHECK();
    return PARS3_OK;
}

extern "C" int pars3_plan_spmv(pars3_plan *pl, const double *x, double *y, void *stream) {
    if (!pl || (pl->n > 0 && (!x || !y))) PARS3_FAIL(PARS3_ERR_ARG, "null argument");
    return plan_product(pl, x, y, false, nullptr, nullptr, (cudaStream_t)stream);
}

extern "C" int pars3_plan_spmv_acc(pars3_plan *pl, const double *x, double *y, void *stream) {
    if (!pl || (pl->n > 0 && (!x || !y))) PARS3_FAIL(PARS3_ERR_ARG, "null argument");
    return plan_product(pl, x, y, true, nullptr, nullptr, (cudaStream_t)stream);
}

extern "C" int pars3_plan_spmv_dot(pars3_plan *pl, const double *x, double *y, const double *w,
                                   double *dot, void *stream) {
    if (!pl || !dot || (pl->n > 0 && (!x || !y || !w))) PARS3_FAIL(PARS3_ERR_ARG, "null argument");
    return plan_product(pl, x, y, false, w, dot, (cudaStream_t)stream);
}

extern "C" int pars3_dot(int64_t n, const double *a, const double *b, double *out, void *stream) {
    if (n < 0 || n >= INT32_MAX || !out || (n > 0 && (!a || !b))) PARS3_FAIL(PARS3_ERR_ARG, "bad argument");
    cudaStream_t st = (cudaStream_t)stream;
    CUDA_TRY(cudaMemsetAsync(out, 0, sizeof(double), st));
    if (n == 0) return PARS3_OK;
    if (((uintptr_t)a | (uintptr_t)b) & 15) PARS3_FAIL(PARS3_ERR_ARG, "a and b must be 16-byte aligned");
    k_dot<<<148 * 4, 512, 0, st>>>((int32_t)n, a, b, out);
    LAUNCH_CHECK();
    return PARS3_OK;
}

extern "C" int pars3_plan_status(pars3_plan *pl, int32_t *flags, void *stream) {
    if (!pl || !flags) PARS3_FAIL(PARS3_ERR_ARG, "null argument");
    *flags = 0;
    if (!pl->counter) return PARS3_OK;
    cudaStream_t st = (cudaStream_t)stream;
    CUDA_TRY(cudaMemcpyAsync(flags, pl->counter + 1, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaStreamSynchronize(st));
    return PARS3_OK;
}

extern "C" int pars3_plan_kernel_count(const pars3_plan *pl, int32_t with_dot, int32_t *count) {
    if (!pl || !count) PARS3_FAIL(PARS3_ERR_ARG, "null argument");
    if (pl->direct)
        *count = (pl->n > 0 ? 1 : 0) + (pl->dm > 0 ? 1 : 0) + (with_dot && pl->n > 0 ? 1 : 0);
    else
        *count = pl->perm ? (pl->ntiles > 0 ? 3 : 2)
                          : (pl->ntiles > 0 ? 1 : 0) + (with_dot && pl->n > 0 ? 1 : 0);
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
    stats[8] = pl->list_tiles;
    stats[9] = pl->words;
    stats[10] = pl->perm ? 1 : 0;
    stats[11] = pl->local_slots;
    stats[12] = pl->dropped;
    stats[13] = pl->direct;
    return PARS3_OK;
}

// debug: per-phase cycle totals (PARS3_PHASES=1), summed over CTAs and launches
extern "C" int pars3_plan_phases(const pars3_plan *pl, int64_t *out6) {
    if (!pl || !out6) PARS3_FAIL(PARS3_ERR_ARG, "null argument");
    unsigned long long h[8] = {0};
    if (pl->phase_clk) CUDA_TRY(cudaMemcpy(h, pl->phase_clk, sizeof(h), cudaMemcpyDeviceToHost));
    for (int k = 0; k < 6; k++) out6[k] = (int64_t)h[k];
    return PARS3_OK;
}

extern "C" int pars3_plan_destroy(pars3_plan *pl) {
    delete pl;
    return PARS3_OK;
}
