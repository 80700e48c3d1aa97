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
//      exact-integer fixed point with native 32-bit shared atomics (or fp64
//      for tiles the fixed point cannot carry: see the guard in tile_loop);
//   3. every slot's accumulated value (+ diag * x for the tile's own rows)
//      is delivered: for own rows this is the reference's owner write
//      (parallel.py:85-95), for columns below the tile the accumulation
//      message (msg_val / MPI_Accumulate, parallel.py:96-113).
//
// Delivery has two forms.
//   GRID (single-GPU products, the default): every slot value is converted
//      to an integer on one product-wide fixed-point grid and reduced into
//      the int64 accumulator yacc with red.global.add.u64.  Integer sums
//      commute, so the result does not depend on the order in which tiles
//      arrive: the product is bitwise repeatable (the reference's own
//      guarantee, parallel.py:107-108, tests/test_parallel.py:81-88).
//      k_finish then streams yacc into fp64 y (clearing yacc for the next
//      product) with the MRS dot <y, w> fused, summed in a fixed order.  The
//      grid's scale needs a bound on |x|: the previous product's maximum (a
//      pre-pass on the first product).  A product whose x exceeds it, holds
//      a non-finite x, or whose grid turns out too coarse for its
//      ||y||_inf, is redone by k_finish through the RED form (exact, IEEE).
//   RED (peer mode, y += A x, the redo): fire-and-forget fp64
//      red.global.add into y (zeroed first), or into a peer's inbox over
//      NVLink.  Exact (the same per-tile guard), not bitwise repeatable.

#include <cuda_runtime.h>
#include <omp.h>

#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <algorithm>
#include <cstring>
#include <new>

#include "common.h"
#include "fullcsr.h"
#include "fullcsr_gpu.h"

// PARS3_CHECKS builds (make checked -> libpars3_checked.so, selected with
// PARS3_LIB): device-side bounds checks on every shared slot, row and column
// index the kernels derive from the plan (a trap reports the failure)
#ifdef PARS3_CHECKS
#define DCHECK(cond)                                                                              \
    do {                                                                                          \
        if (!(cond)) {                                                                            \
            printf("pars3 check failed %s:%d block %d thread %d: %s\n", __FILE__, __LINE__,        \
                   blockIdx.x, threadIdx.x, #cond);                                               \
            __trap();                                                                             \
        }                                                                                         \
    } while (0)
#else
#define DCHECK(cond) \
    do {             \
    } while (0)
#endif
#include "locality.h"
#include "tileplan.h"
#include "tileplan_gpu.h"

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
static_assert(kThreads % 32 == 0 && kThreads <= 1024, "CTA shape");
constexpr int kTerms2 = 64;        // two-word fixed point: max terms per slot per tile
constexpr int kTerms3 = 4096;      // three-word fixed point: max terms per slot per tile
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

// Product state on the device (one per plan).  The kernels reset their own
// counters, so a product needs no memset.
struct GState {
    int32_t claim;       // tile claims of the main pass (reset by k_finish)
    int32_t claim2;      // tile claims of the redo pass (reset at its end)
    int32_t flags;       // why the grid result must be redone (kFlag*), cleared by k_finish
    int32_t xe;          // grid scale bound |x| < 2^xe assumed by the next product
    int32_t xe_seen;     // max x exponent over this product's tiles
    int32_t done;        // k_conv CTAs done
    uint32_t bar;        // grid barrier of k_finish: arrivals
    uint32_t gen;        // grid barrier of k_finish: generation
    int32_t fp64_tiles;  // tiles accumulated in fp64 (guard or non-finite x), cumulative
    int32_t redone;      // products redone by k_finish, cumulative
    int32_t xe_pre;      // strict scale: max x exponent of THIS product's x + 1 + kXeBias (0: none)
    int32_t pad[5];
};
constexpr int kFlagNonfinite = 1;  // a non-finite x value: IEEE semantics need the fp64 form
constexpr int kFlagXRange = 2;     // some |x| >= 2^xe: the grid could overflow
constexpr int kFlagCoarse = 4;     // grid unit too coarse for this product's ||y||_inf
constexpr int kFlagScale = 8;      // grid exponent outside the fp64 range
constexpr int kFlagTileFp = 16;    // a tile the fixed point cannot carry (guard, scale range)
constexpr int kXeNone = -1100;     // "no finite non-zero x seen"
constexpr int kExNonfinite = 4000; // x exponent scan: a non-finite value
constexpr int kXeBias = 2048;      // GState::xe_pre encoding (a memset to 0 means "none")

struct DevPlan {
    const TileMeta *tiles;
    const Window *wins;
    const int64_t *slice_off;  // 16-byte units
    const uint8_t *rec;
    const int32_t *ucol;
    const double *diag;
    int32_t ntiles;
    int32_t n;  // rows (index space) of the plan
    int32_t watchdog;
    int32_t diag_const;  // 1: every diagonal value equals diag_alpha (strict / shifted skew)
    double diag_alpha;
    unsigned long long *phase_clk;  // PARS3_PHASES=1: per-phase SM cycles (thread 0 of each CTA)
    int32_t pf;  // L2 prefetch of records: bit 0 each tile's records when its metadata is
                 // fetched, bit 1 each warp's slice pf_dist iterations ahead, bit 2 the
                 // next tile's first slices at the end of the stream
    int32_t pf_dist;
    Peers peers;  // multi-GPU peer mode (nranks > 0): columns owned by other ranks
    GState *gs;
    // grid form: the int64 accumulator over the rows, per-CTA shares of the
    // dot and of ||y||_inf (k_finish), the grid scale's bounds
    long long *yacc;
    double *blk_dot;
    double *blk_max;
    int32_t ev_g;   // every |value| and |diag| < 2^ev_g
    int32_t hgrid;  // ceil(log2(most terms one y element sums))
    int32_t cmax;   // most tiles delivering to one row block (grid roundings per element)
    int32_t strict; // this product's scale from its own x (k_xmax pre-pass), not the previous one's
    // two accumulators in turn: while a product reduces into yacc, each tile
    // clears its own rows of the other one (read by the previous product's
    // k_conv, used by the next product), so k_conv writes no zeros: its 8 n
    // bytes of stores move into the tile kernel, where DRAM has headroom
    long long *yclear;  // nullptr: one accumulator, cleared by k_conv
    // far entries (k_far_*): the few long-range entries of a locality-ordered
    // plan, kept out of the tiles so that those stay in window mode
    const int32_t *far_row, *far_col;
    const double *far_val;
    int32_t nfar;
    // fused epilogue of pars3_plan_product_axpy: out = A x + (*ep_a) p + (*ep_b) q
    // (device scalars, so an iteration's recurrence needs no host round trip);
    // null ep_a: none
    const double *ep_p, *ep_q, *ep_a, *ep_b;
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
// A slot's mirror sum is kept as an exact integer Q * 2^(E-50) in two (or
// three) 32-bit words updated with native shared-memory integer adds
// (fire-and-forget ATOMS.ADD, no CAS loop).  E = ev + ex + 3 bounds every
// term of the tile (|v| < 2^ev, |x| < 2^ex, a row segment sums <= 8 terms),
// so |Q| < 2^50 per term and the per-term rounding is <= 2^(E-51).  Integer
// adds commute: a tile's accumulation is independent of the order in which
// its warps arrive.
//
// q = fma(t, 2^(50-E), 1.5 * 2^52): the low mantissa bits hold rint(t *
// 2^(50-E)) = Q as a two's-complement offset from the magic constant, so
// the words come straight from the two halves of q.
//   two words (<= kTerms2 = 64 terms per slot and tile, the plan checks):
//     bits 0-25 unsigned (64 x 2^26 = 2^32), the signed rest Q >> 26;
//   three words (<= 4096 terms): 20-bit limbs, the signed rest Q >> 40.
//
// Guard (the tile's accuracy is tied to its output, not to its bound E):
// every row-segment sum (<= 8 terms, a partial output) also feeds qm =
// max(Q >> 32) + 1024 and qn = OR of its bits.  A tile some of whose segment
// sums are non-zero but none reaches |Q| >= 2^42 -- its bound E is more than
// 8 bits above what it delivers, e.g. a large value met only by small x --
// would round every term to a unit that is coarse against its output; it is
// re-streamed with fp64 accumulators instead.  One
// check per segment, not per term: 2-3 integer ops per lane and slice.
constexpr double kMagic = 6755399441055744.0;  // 1.5 * 2^52
constexpr uint32_t kGuardBig = 2048u;         // (Q >> 32) + 1024 >= 2048  <=>  |Q| >= 2^42

template <int kWords, int kS, bool kTrack = false>
__device__ __forceinline__ void fx_add(uint32_t *w, uint32_t i, double q, uint32_t &qm, uint32_t &qn) {
    const uint32_t blo = (uint32_t)__double2loint(q);
    const uint32_t bhi = (uint32_t)__double2hiint(q) - 0x43380000u;  // Q >> 32
    if (kTrack) {
        qm = max(qm, bhi + 1024u);
        qn |= blo | bhi;
    }
    if (kWords == 3) {
        atomicAdd(w + i, blo & 0xFFFFFu);
        atomicAdd(w + kS + i, __funnelshift_r(blo, bhi, 20) & 0xFFFFFu);
        atomicAdd(w + 2 * kS + i, (uint32_t)((int32_t)bhi >> 8));
    } else {
        atomicAdd(w + i, blo & 0x3FFFFFFu);
        atomicAdd(w + kS + i, __funnelshift_r(blo, bhi, 26));
    }
}

// the exact integer Q of a slot (fixed point), clearing its words
template <int kWords, int kS>
__device__ __forceinline__ long long fx_take(uint32_t *w, int i) {
    if (kWords == 3) {
        const long long V = ((long long)(int32_t)w[2 * kS + i] << 40) + ((long long)w[kS + i] << 20) +
                            (long long)w[i];
        w[i] = w[kS + i] = w[2 * kS + i] = 0u;
        return V;
    }
    const long long V = ((long long)(int32_t)w[kS + i] << 26) + (long long)w[i];
    w[i] = w[kS + i] = 0u;
    return V;
}

// Q * 2^sh on the grid, rounded half up when sh < 0 (deterministic)
__device__ __forceinline__ long long to_grid(long long V, int sh) {
    if (sh >= 0) return V << sh;  // sh <= 15 - hgrid: |result| < 2^62
    if (sh < -62) return 0;
    return (V + (1ll << (-sh - 1))) >> (-sh);
}

__device__ __forceinline__ void red_add_u64(long long *p, long long v) {
    asm volatile("red.global.add.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// Stream a tile's slices into the shared accumulators.  kAcc: 2 / 3 fixed-
// point words, 0 fp64 (shared atomicAdd, a CAS loop).
template <int kAcc, int kS, uint32_t kSink>
__device__ __forceinline__ void stream_tile(const DevPlan &P, const int64_t *off, int nsl, const double *xs,
                                            uint32_t *wlo, double *acc, double scale, int warp, int lane,
                                            uint32_t &qm, uint32_t &qn) {
    for (int i = warp; i < nsl; i += kWarps) {
        if ((P.pf & 2) && lane == 0 && i + P.pf_dist * kWarps < nsl) {
            const int j = i + P.pf_dist * kWarps;
            const int64_t a = off[j], b = off[j + 1];
            bulk_prefetch_l2(P.rec + a * 16, (uint32_t)((b - a) * 16));
        }
        const uint8_t *rp = P.rec + off[i] * 16;
        const int ns = (int)(((off[i + 1] - off[i]) * 16 - 64) / 320);
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
        DCHECK(rl <= kSink);
        const double xr = xs[rl];
        double c0 = 0.0, c1 = 0.0;  // two row-sum chains: even and odd slots
        if (kAcc > 0) {
            const double nxs = -xr * scale;  // mirror term v * (-x_r), scaled
#pragma unroll
            for (int u = 0; u < kMaxSlots; u++) {
                if (u < ns) {
                    DCHECK(li[u] <= kSink);
                    if (u & 1)
                        c1 = fma(v[u], xs[li[u]], c1);
                    else
                        c0 = fma(v[u], xs[li[u]], c0);
                    fx_add<kAcc, kS>(wlo, li[u], fma(v[u], nxs, kMagic), qm, qn);
                }
            }
            fx_add<kAcc, kS, true>(wlo, rl, fma(c0 + c1, scale, kMagic), qm, qn);
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
}

// Sum / max over the CTA with a fixed reduction tree (xor butterflies leave
// the same value in every lane): deterministic.  Result valid in warp 0.
__device__ __forceinline__ double cta_sum(double v, double *sred) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0) sred[warp] = v;
    __syncthreads();
    v = lane < kWarps ? sred[lane] : 0.0;
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    __syncthreads();
    return v;
}
__device__ __forceinline__ double cta_max(double v, double *sred) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int o = 16; o; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    if (lane == 0) sred[warp] = v;
    __syncthreads();
    v = lane < kWarps ? sred[lane] : 0.0;
    for (int o = 16; o; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    __syncthreads();
    return v;
}

// The scale bound of this product's grid: strict products take it from a
// pass over their own x (k_xmax, a pure function of x), the others from the
// previous product's maximum (k_conv's update; bitwise the same when x
// repeats, and checked by kFlagXRange when it grows).
__device__ __forceinline__ int product_xe(const DevPlan &P) {
    if (!P.strict) return *(volatile int32_t *)&P.gs->xe;
    const int e = *(volatile int32_t *)&P.gs->xe_pre;
    return e == 0 ? kXeNone : e - kXeBias;
}

// The persistent tile loop.  kWords: the plan's accumulator (0 fp64, 2 / 3
// fixed-point words; fixed-point plans switch single tiles to fp64).
// kPeer: multi-GPU peer mode (P.peers; RED form only).  kGrid: GRID form
// (y written by the block finalizers, w / dot: fused <y, w>, w == y when
// dot_self) or RED form (fp64 reductions into y, zeroed by the caller).
template <int kWords, bool kPeer, bool kGrid>
__device__ __forceinline__ void tile_loop(const DevPlan &P, const double *__restrict__ x,
                                          double *__restrict__ y, const double *w, double *dot,
                                          bool dot_self, int32_t *claims) {
    constexpr bool kFixed = kWords > 0;
    constexpr int S = Layout<kWords>::kStride;
    constexpr uint32_t kSink = Layout<kWords>::kSink;
    extern __shared__ __align__(128) uint8_t dyn[];
    double *xs = reinterpret_cast<double *>(dyn);
    // fp64 accumulators acc[S], or two / three uint32 words per slot (the
    // fp64 view fits in either: a fixed-point plan's fp64 tiles use it)
    double *acc = xs + S;
    uint32_t *wlo = reinterpret_cast<uint32_t *>(xs + S);
    __shared__ int64_t s_off[2][kMaxTileSlices + 1];
    __shared__ int32_t s_t[3];  // tiles k, k+1 (known) and k+2 (claimed during tile k)
    __shared__ int32_t s_ex[2];
    __shared__ uint32_t s_qm[2], s_qn[2];
    __shared__ __align__(8) uint64_t xbar;
    __shared__ TileCache s_tc[2];
    __shared__ double s_red[kWarps];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    for (int i = tid; i < S; i += kThreads) {
        xs[i] = 0.0;  // the sink's x stays 0
        if (kWords == 3) {
            wlo[i] = wlo[S + i] = wlo[2 * S + i] = 0u;
        } else if (kWords == 2) {
            wlo[i] = wlo[S + i] = 0u;
        } else {
            acc[i] = 0.0;
        }
    }
    // PARS3_PHASES=1: thread 0 accumulates SM cycles per phase
    // (totals in shared memory: no registers held across the tile loop)
    __shared__ long long s_clk[6];
    if (tid < 6) s_clk[tid] = 0;  // (phase 5: the grid form's arrivals, counted into slot 5)
    // the grid of this product: yacc unit 2^(Eg-62), |partial sums| < 2^(Eg+1)
    int Eg = 0, xe = 0;
    if (kGrid) {
        xe = product_xe(P);
        Eg = P.ev_g + xe + P.hgrid;
        if (Eg > 960 || Eg < -960) {
            if (tid == 0) atomicOr(&P.gs->flags, kFlagScale);
            Eg = max(-960, min(960, Eg));
        }
    }
    if (tid == 0) {
        mbar_init(&xbar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        s_t[0] = atomicAdd(claims, 1);
        s_t[1] = atomicAdd(claims, 1);
        s_ex[0] = s_ex[1] = kXeNone;
        s_qm[0] = s_qm[1] = s_qn[0] = s_qn[1] = 0u;
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
        if (tid == 0) claimed = atomicAdd(claims, 1);
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
            for (int w2 = 0; w2 < tc.nw; w2++) {
                if (tma_ok<kPeer>(pr, x, tc, w2)) continue;
                const double *src = x + tc.lo[w2];
                if (kPeer) {
                    const int r = tc.own[w2];
                    if (r != pr.me) src = pr.x[r] + (pr.col_base + tc.lo[w2] - pr.bs[r]);
                }
                for (int i = tid; i < tc.len[w2]; i += kThreads) xs[tc.off[w2] + i] = src[i];
            }
        }
        mbar_wait(&xbar, (uint32_t)(k & 1), P.watchdog, 5, t);
        asm volatile("cp.async.wait_all;" ::: "memory");  // this tile's record offsets
        {  // tile-wide bound on |x|: max binary exponent over the slots, |x| < 2^ex
            // (slots in pairs, 16-byte loads; a subnormal or zero x counts as
            // 2^-1022; a non-finite one as kExNonfinite)
            int e = kXeNone;
            const double2 *xs2 = reinterpret_cast<const double2 *>(xs);
            for (int i = tid; i < (local + 1) / 2; i += kThreads) {
                const double2 v = xs2[i];  // (an odd tail's mate is inside the stride, not counted)
                int b0 = (int)((__double_as_longlong(v.x) >> 52) & 0x7FF);
                int b1 = (int)((__double_as_longlong(v.y) >> 52) & 0x7FF);
                if (2 * i + 1 >= local) b1 = 0;
                b0 = b0 == 2047 ? kExNonfinite : max(b0, 1) - 1022;
                b1 = b1 == 2047 ? kExNonfinite : max(b1, 1) - 1022;
                e = max(e, max(b0, b1));
            }
            e = __reduce_max_sync(0xffffffffu, e);
            if (lane == 0) atomicMax(&s_ex[cur], e);
        }
        __syncthreads();
        PHASE(1);
        const int ex = s_ex[cur];
        if (tid == 0) {
            fetch_tile<kPeer>(P, s_t[(k + 1) % 3], s_tc[nxt]);  // overlaps the stream
            s_ex[nxt] = kXeNone;
            s_qm[nxt] = s_qn[nxt] = 0u;
            if (kGrid) {
                if (ex >= kExNonfinite) {
                    atomicOr(&P.gs->flags, kFlagNonfinite);
                } else {
                    if (ex > xe) atomicOr(&P.gs->flags, kFlagXRange);
                    atomicMax(&P.gs->xe_seen, ex);  // (result unused: a fire-and-forget RED)
                }
            }
        }
        // the tile's fixed-point scale; fp64 accumulators for a non-finite x
        // or a scale beyond the fp64 range (IEEE semantics).  The GRID form
        // has no fp64 tile path (a leaner kernel): such a tile flags the
        // product, which k_finish then redoes with fp64 accumulators.
        constexpr bool kTileFp = kFixed && !kGrid;
        int E = tc.m.ev + ex + 3;
        bool tile_fp = !kFixed || ex >= kExNonfinite || E > 960;
        if (kGrid && kFixed && tile_fp) {
            if (tid == 0) atomicOr(&P.gs->flags, kFlagTileFp);
            tile_fp = false;
        }
        E = max(-960, min(960, E));
        const double scale = ldexp(1.0, 50 - E);
        const double unscale = ldexp(1.0, E - 50);

        // 2. records: each lane owns one row segment of a slice; row sums in
        //    registers, mirrors into the tile's shared accumulators
        if constexpr (kFixed) {
            if (kTileFp && tile_fp) {
                uint32_t qm = 0, qn = 0;
                stream_tile<0, S, kSink>(P, s_off[cur], nsl, xs, wlo, acc, 1.0, warp, lane, qm, qn);
            } else {
                uint32_t qm = 0, qn = 0;
                stream_tile<kWords, S, kSink>(P, s_off[cur], nsl, xs, wlo, acc, scale, warp, lane, qm, qn);
                qm = __reduce_max_sync(0xffffffffu, qm);
                qn = __reduce_or_sync(0xffffffffu, qn);
                if (lane == 0 && (qm | qn)) {
                    atomicMax(&s_qm[cur], qm);
                    atomicOr(&s_qn[cur], qn);
                }
            }
        } else {
            uint32_t qm = 0, qn = 0;
            stream_tile<0, S, kSink>(P, s_off[cur], nsl, xs, wlo, acc, 1.0, warp, lane, qm, qn);
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
        if (kGrid && kFixed && s_qn[cur] != 0u && s_qm[cur] < kGuardBig) {
            if (tid == 0) atomicOr(&P.gs->flags, kFlagTileFp);  // the guard: k_finish redoes
        } else if (kTileFp && !tile_fp && s_qn[cur] != 0u && s_qm[cur] < kGuardBig) {
            // the guard: re-stream this tile with fp64 accumulators
            for (int i = tid; i < S; i += kThreads) {
                acc[i] = 0.0;  // (words 0 .. 2S-1)
                if (kWords == 3) wlo[2 * S + i] = 0u;
            }
            __syncthreads();
            uint32_t qm = 0, qn = 0;
            stream_tile<0, S, kSink>(P, s_off[cur], nsl, xs, wlo, acc, 1.0, warp, lane, qm, qn);
            tile_fp = true;
            __syncthreads();
        }
        if (kTileFp && tile_fp && tid == 0) atomicAdd(&P.gs->fp64_tiles, 1);
        PHASE(2);

        // 3. xs is free: the next tile's x windows and record offsets are
        //    issued first, so they land while this tile flushes
        if (tid == 0) issue_x_cached<kPeer>(P.peers, x, s_tc[nxt], xs, &xbar);
        load_offsets(P, s_tc[nxt].m, s_off[nxt], tid);
        PHASE(4);

        // 4. deliver every slot (own rows: + diag * x, x of own rows from
        //    global: xs already holds the next tile); the accumulators are
        //    cleared in the same pass
        if (kGrid) {
            const double gscale = ldexp(1.0, 62 - Eg);
            const int sh = E - Eg + 12;
            auto deliver = [&](int i, int c) {
                long long V;
                if constexpr (kFixed) {
                    V = to_grid(fx_take<kWords, S>(wlo, i), sh);
                } else {
                    V = __double2ll_rn(acc[i] * gscale);
                    acc[i] = 0.0;
                }
                if (c >= r0 && c < r1)
                    V += __double2ll_rn((P.diag_const ? P.diag_alpha : __ldg(P.diag + c)) * __ldg(x + c) *
                                        gscale);
                DCHECK(c >= 0 && c < P.n);
                if (V != 0) red_add_u64(P.yacc + c, V);
            };
            if (P.yclear)  // (every row is some tile's own row)
                for (int i = r0 + tid; i < r1; i += kThreads) __stcs(P.yclear + i, 0ll);
            if (u0 >= 0) {
                const int32_t *uc = P.ucol + u0;
                for (int i = tid; i < local; i += kThreads) deliver(i, __ldg(uc + i));
            } else {
                for (int w2 = 0; w2 < tc.nw; w2++)
                    for (int i = tid; i < tc.len[w2]; i += kThreads) deliver(tc.off[w2] + i, tc.lo[w2] + i);
            }
            __syncthreads();
            PHASE(3);
        } else {
            auto take = [&](int i) -> double {
                if constexpr (kFixed) {
                    if (!(kTileFp && tile_fp)) return (double)fx_take<kWords, S>(wlo, i) * unscale;
                }
                const double a = acc[i];
                acc[i] = 0.0;
                return a;
            };
            if (u0 >= 0) {
                const int32_t *uc = P.ucol + u0;
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
                    if (mine && c >= r0 && c < r1)  // (a halo row's diagonal belongs to its owner)
                        a = fma(P.diag_const ? P.diag_alpha : __ldg(P.diag + c), __ldg(x + c), a);
                    DCHECK(kPeer || (c >= 0 && c < P.n));
                    if (a != 0.0) atomicAdd(dst, a);
                }
            } else {
                for (int w2 = 0; w2 < tc.nw; w2++) {
                    const int lo = tc.lo[w2], len = tc.len[w2], off = tc.off[w2];
                    // own columns reduce into y; an earlier rank's columns into its
                    // inbox over NVLink (peer mode; their diagonal is the owner's)
                    bool mine = true;
                    double *dst = y + lo;
                    if (kPeer) {
                        const int r = tc.own[w2];
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
                        DCHECK(kPeer || (c >= 0 && c < P.n));
                        if (a != 0.0) atomicAdd(dst + i, a);
                    }
                }
            }
            __syncthreads();
            PHASE(3);
        }
    }
    // peer mode: this CTA's reductions into other GPUs' inboxes are performed
    // system-wide before the kernel completes (the barrier after the product
    // is stream-ordered behind it)
    if (kPeer) __threadfence_system();
    if (P.phase_clk && tid == 0)
        for (int k = 0; k < 6; k++) atomicAdd(P.phase_clk + k, (unsigned long long)s_clk[k]);
#undef PHASE
}

template <int kWords, bool kPeer, bool kGrid>
__global__ void __launch_bounds__(kThreads, kMinBlocks)
k_tiles(DevPlan P, const double *__restrict__ x, double *__restrict__ y, const double *w, double *dot,
        int dot_self) {
    tile_loop<kWords, kPeer, kGrid>(P, x, y, w, dot, dot_self != 0, &P.gs->claim);
}

// grid barrier of k_finish (the kernel is launched cooperatively: every CTA
// is resident)
__device__ __forceinline__ void grid_sync(GState *g) {
    __syncthreads();
    if (threadIdx.x == 0) {
        const uint32_t gen = *(volatile uint32_t *)&g->gen;
        __threadfence();
        if (atomicAdd(&g->bar, 1u) == gridDim.x - 1) {
            g->bar = 0u;
            __threadfence();
            atomicAdd(&g->gen, 1u);
        } else {
            while (*(volatile uint32_t *)&g->gen == gen) __nanosleep(256);  // (polls off the L2 path)
        }
        __threadfence();
    }
    __syncthreads();
}

// The grid product's finish, one streaming pass: y = yacc * 2^(Eg-62) with
// yacc cleared for the next product, and per-CTA shares of <y, w> and
// ||y||_inf (a fixed row assignment: the grid is fixed per plan); the CTA
// that finishes last sums the shares in CTA order, runs the accuracy check
// (the grid's rounding against ||y||_inf) and sets the next product's scale
// bound.  No shared memory, many CTAs, eight pairs in flight per thread.
#ifndef PARS3_CONV_U  // tuning builds
#define PARS3_CONV_U 8
#define PARS3_CONV_MINB 2
#endif
constexpr int kConvThreads = 256;
constexpr int kConvGrid = 148 * 8;  // (the most CTAs; the launch uses one resident wave)
// (kEp: with pars3_plan_product_axpy's update; the plain instantiation keeps its registers)
template <bool kEp>
__global__ void __launch_bounds__(kConvThreads, PARS3_CONV_MINB) k_conv(DevPlan P, double *__restrict__ y, const double *w,
                                                       double *dot, int dot_self, int32_t n) {
    __shared__ double s_red[kConvThreads / 32];
    __shared__ int s_last;
    GState *g = P.gs;
    const int xe = product_xe(P);
    const int Eg = max(-960, min(960, P.ev_g + xe + P.hgrid));
    const double gunit = ldexp(1.0, Eg - 62);
    const bool self = dot_self != 0;
    const int64_t stride = (int64_t)gridDim.x * kConvThreads;
    const int64_t i0 = blockIdx.x * (int64_t)kConvThreads + threadIdx.x;
    double d = 0.0, mx = 0.0;
    constexpr bool ep = kEp;
    const double ea = ep ? *P.ep_a : 0.0, eb = ep ? *P.ep_b : 0.0;
    if ((((uintptr_t)y | (uintptr_t)w | (ep ? (uintptr_t)P.ep_p | (uintptr_t)P.ep_q : 0)) & 15) == 0) {  // pairs: 16-byte accesses
        const int64_t n2 = n / 2;
        longlong2 *a2 = reinterpret_cast<longlong2 *>(P.yacc);
        double2 *y2 = reinterpret_cast<double2 *>(y);
        const double2 *w2 = reinterpret_cast<const double2 *>(w);
        constexpr int U = PARS3_CONV_U;
        for (int64_t i = i0; i < n2; i += U * stride) {
            longlong2 Y[U];
#pragma unroll
            for (int u = 0; u < U; u++)
                if (i + u * stride < n2) Y[u] = __ldcs(a2 + i + u * stride);
#pragma unroll
            for (int u = 0; u < U; u++) {
                const int64_t j = i + u * stride;
                if (j < n2) {
                    if (!P.yclear) __stcs(a2 + j, make_longlong2(0, 0));
                    double2 v = make_double2((double)Y[u].x * gunit, (double)Y[u].y * gunit);
                    mx = fmax(mx, fmax(fabs(v.x), fabs(v.y)));  // (of A x: the grid's accuracy check)
                    if (ep) {
                        const double2 pp = __ldcs(reinterpret_cast<const double2 *>(P.ep_p) + j);
                        const double2 qq = __ldcs(reinterpret_cast<const double2 *>(P.ep_q) + j);
                        v.x = fma(eb, qq.x, fma(ea, pp.x, v.x));
                        v.y = fma(eb, qq.y, fma(ea, pp.y, v.y));
                    }
                    __stcs(y2 + j, v);
                    if (dot) {
                        const double2 q = self ? v : __ldcs(w2 + j);
                        d = fma(v.y, q.y, fma(v.x, q.x, d));
                    }
                }
            }
        }
        if ((n & 1) && i0 == 0) {
            const long long Y = P.yacc[n - 1];
            if (!P.yclear) P.yacc[n - 1] = 0;
            double v = (double)Y * gunit;
            mx = fmax(mx, fabs(v));
            if (ep) v = fma(eb, P.ep_q[n - 1], fma(ea, P.ep_p[n - 1], v));
            y[n - 1] = v;
            if (dot) d = fma(v, self ? v : w[n - 1], d);
        }
    } else {
        for (int64_t i = i0; i < n; i += stride) {
            const long long Y = P.yacc[i];
            if (!P.yclear) P.yacc[i] = 0;
            double v = (double)Y * gunit;
            mx = fmax(mx, fabs(v));
            if (ep) v = fma(eb, P.ep_q[i], fma(ea, P.ep_p[i], v));
            y[i] = v;
            if (dot) d = fma(v, self ? v : w[i], d);
        }
    }
    // fixed-tree CTA sums (cta_sum's shape with this CTA size)
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int o = 16; o; o >>= 1) {
        d += __shfl_xor_sync(0xffffffffu, d, o);
        mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    }
    if (lane == 0) s_red[warp] = d;
    __syncthreads();
    if (threadIdx.x == 0) {
        double s = 0.0;
        for (int k = 0; k < kConvThreads / 32; k++) s += s_red[k];
        P.blk_dot[blockIdx.x] = s;
    }
    __syncthreads();
    if (lane == 0) s_red[warp] = mx;
    __syncthreads();
    if (threadIdx.x == 0) {
        double m = 0.0;
        for (int k = 0; k < kConvThreads / 32; k++) m = fmax(m, s_red[k]);
        P.blk_max[blockIdx.x] = m;
        __threadfence();
        s_last = atomicAdd(&g->done, 1) == (int)gridDim.x - 1;
        if (s_last) __threadfence();
    }
    __syncthreads();
    if (!s_last) return;
    d = 0.0;
    mx = 0.0;
    for (int b = threadIdx.x; b < (int)gridDim.x; b += kConvThreads) {  // CTA order per thread
        d += __ldcg(P.blk_dot + b);
        mx = fmax(mx, __ldcg(P.blk_max + b));
    }
    for (int o = 16; o; o >>= 1) {
        d += __shfl_xor_sync(0xffffffffu, d, o);
        mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    }
    __syncthreads();
    if (lane == 0) s_red[warp] = d;
    __syncthreads();
    double dsum = 0.0;
    if (threadIdx.x == 0)
        for (int k = 0; k < kConvThreads / 32; k++) dsum += s_red[k];
    __syncthreads();
    if (lane == 0) s_red[warp] = mx;
    __syncthreads();
    if (threadIdx.x == 0) {
        double m = 0.0;
        for (int k = 0; k < kConvThreads / 32; k++) m = fmax(m, s_red[k]);
        if (dot) *dot = dsum;
        // each delivery was rounded to the grid unit 2^(Eg-62) once: the
        // grid's share of the error stays below 2^-44 max(1, ||y||_inf),
        // else k_finish redoes the product (a matrix whose value range the x
        // correlate with)
        const double err = (double)P.cmax * ldexp(1.0, Eg - 63);
        if (!(err <= ldexp(1.0, -44) * fmax(1.0, m))) atomicOr(&g->flags, kFlagCoarse);
        const int xs = *(volatile int32_t *)&g->xe_seen;
        g->xe = (xs <= kXeNone ? -1000 : xs) + 1;
        g->xe_seen = kXeNone;
        g->done = 0;
        __threadfence();
    }
}

// After every grid product (launched cooperatively: every CTA resident).
// It first finishes the product in one streaming pass: y = yacc * 2^(Eg-62), yacc cleared, the
// per-CTA shares of <y, w> and ||y||_inf (fixed row assignment), summed in
// CTA order by CTA 0, which also runs the accuracy check and sets the next
// scale bound.  Then, unless a kFlag* was raised (exits at once), the fp64
// redo: y = 0, the RED form over every tile, <y, w> in a fixed order.
// The redo accumulates in fp64 (shared-memory CAS, IEEE semantics for
// non-finite and extreme inputs); the fp64 layout fits in every plan's
// shared memory and its sink lies beyond every plan's local space.  Clears
// the flags and resets the tile kernel's claim counter.
constexpr int kFinishSmem = Layout<0>::kSmem;  // >= every plan's layout
__global__ void __launch_bounds__(kThreads, kMinBlocks)
k_finish(DevPlan P, const double *__restrict__ x, double *__restrict__ y, const double *w, double *dot,
         int dot_self, int32_t n) {
    GState *g = P.gs;
    __shared__ double s_red[kWarps];
    const int64_t stride = (int64_t)gridDim.x * kThreads;
    const int64_t i0 = blockIdx.x * (int64_t)kThreads + threadIdx.x;
    if (__ldcg(&g->flags) == 0) {
        if (blockIdx.x == 0 && threadIdx.x == 0) g->claim = 0;
        return;
    }
    for (int64_t i = i0; i < n; i += stride) y[i] = 0.0;
    grid_sync(g);
    tile_loop<0, false, false>(P, x, y, nullptr, nullptr, false, &g->claim2);  // fp64 accumulators
    for (int64_t e = i0; e < P.nfar; e += stride) {  // the far part
        const int32_t i = P.far_row[e], c = P.far_col[e];
        const double v = P.far_val[e];
        atomicAdd(y + i, v * x[c]);
        atomicAdd(y + c, -v * x[i]);
    }
    grid_sync(g);
    if (dot || P.ep_a) {  // the fused epilogue; per-CTA shares in blk_dot, summed in CTA order
        const bool ep = P.ep_a != nullptr;
        const double ea = ep ? *P.ep_a : 0.0, eb = ep ? *P.ep_b : 0.0;
        double d = 0.0;
        for (int64_t i = i0; i < n; i += stride) {
            double v = __ldcg(y + i);
            if (ep) {
                v = fma(eb, P.ep_q[i], fma(ea, P.ep_p[i], v));
                y[i] = v;
            }
            if (dot) d = fma(v, dot_self ? v : w[i], d);
        }
        d = cta_sum(d, s_red);
        if (threadIdx.x == 0) P.blk_dot[blockIdx.x] = d;
    }
    grid_sync(g);
    if (blockIdx.x == 0) {
        double d = 0.0;
        if (dot)
            for (int b = threadIdx.x; b < (int)gridDim.x; b += kThreads) d += __ldcg(P.blk_dot + b);
        d = cta_sum(d, s_red);
        if (threadIdx.x == 0) {
            if (dot) *dot = d;
            g->flags = 0;
            g->claim = 0;
            g->claim2 = 0;
            g->redone++;
            __threadfence();
        }
    }
}

// The far part of a plan (the outer part's long-range entries: the north
// star's separate gather / scatter pass): entry (i, c, v) adds v x_c to y_i
// and -v x_i to y_c (serial.py:56-59).  GRID form: each term goes onto the
// product's fixed-point grid and is reduced into yacc as an integer, so the
// sum does not depend on the order (bitwise repeatable); the terms count
// among the grid's roundings (cmax) and headroom (hgrid).  x needs no check
// here: every row is some tile's own row, whose x the tile kernel scanned.
__global__ void __launch_bounds__(256) k_far_grid(DevPlan P, const double *__restrict__ x) {
    const int xe = product_xe(P);
    const int Eg = max(-960, min(960, P.ev_g + xe + P.hgrid));
    const double gscale = ldexp(1.0, 62 - Eg);
    const int32_t stride = gridDim.x * blockDim.x;
    for (int32_t e = blockIdx.x * blockDim.x + threadIdx.x; e < P.nfar; e += stride) {
        const int32_t i = __ldcs(P.far_row + e), c = __ldcs(P.far_col + e);
        const double v = __ldcs(P.far_val + e);
        DCHECK(i >= 0 && i < P.n && c >= 0 && c < P.n);
        const long long a = __double2ll_rn(v * __ldg(x + c) * gscale), b = __double2ll_rn(-v * __ldg(x + i) * gscale);
        if (a) red_add_u64(P.yacc + i, a);
        if (b) red_add_u64(P.yacc + c, b);
    }
}
// RED form (y += A x, plans without the grid form): fp64 reductions
__global__ void __launch_bounds__(256) k_far_red(DevPlan P, const double *__restrict__ x, double *y) {
    const int32_t stride = gridDim.x * blockDim.x;
    for (int32_t e = blockIdx.x * blockDim.x + threadIdx.x; e < P.nfar; e += stride) {
        const int32_t i = __ldcs(P.far_row + e), c = __ldcs(P.far_col + e);
        const double v = __ldcs(P.far_val + e);
        atomicAdd(y + i, v * __ldg(x + c));
        atomicAdd(y + c, -v * __ldg(x + i));
    }
}

// max binary exponent of x (|x| < 2^e) + 1 into gs->xe_pre (biased; zeroed
// before): a strict product's scale bound (the first product is strict)
__global__ void __launch_bounds__(512) k_xmax(int32_t n, const double *__restrict__ x, GState *g) {
    int e = kXeNone;
    const int32_t stride = gridDim.x * blockDim.x;
    for (int32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
        const int b = (int)((__double_as_longlong(__ldcs(x + i)) >> 52) & 0x7FF);
        if (b != 2047) e = max(e, max(b, 1) - 1022);
    }
    e = __reduce_max_sync(0xffffffffu, e);
    if ((threadIdx.x & 31) == 0 && e > kXeNone) atomicMax(&g->xe_pre, e + 1 + kXeBias);
}

// <a, b>: 16-byte loads, four in flight per thread; each block writes its
// share to part[blockIdx.x]; the block that finishes last adds the shares in
// block order (a fixed reduction order: the dot is bitwise repeatable) into
// *out.  part[kDotGrid] holds the arrival counter (zero between calls).
constexpr int kDotGrid = 148 * 4;
__global__ void __launch_bounds__(512) k_dot(int32_t n, const double *__restrict__ a,
                                             const double *__restrict__ b, double *part, double *out) {
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
    __shared__ int s_last;
    if (threadIdx.x < 32) {
        s = threadIdx.x < 16 ? ws[threadIdx.x] : 0.0;
        for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if (threadIdx.x == 0) {
            part[blockIdx.x] = s;
            __threadfence();
            unsigned int *arrived = reinterpret_cast<unsigned int *>(part + kDotGrid);
            s_last = atomicAdd(arrived, 1u) == gridDim.x - 1;
            if (s_last) {
                *arrived = 0u;
                __threadfence();
            }
        }
    }
    __syncthreads();
    if (!s_last) return;
    double d = 0.0;  // shares in block order per thread, then a fixed tree
    for (int i = threadIdx.x; i < (int)gridDim.x; i += blockDim.x) d += __ldcg(part + i);
    for (int o = 16; o; o >>= 1) d += __shfl_xor_sync(0xffffffffu, d, o);
    __syncthreads();
    if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = d;
    __syncthreads();
    if (threadIdx.x < 32) {
        d = threadIdx.x < 16 ? ws[threadIdx.x] : 0.0;
        for (int o = 16; o; o >>= 1) d += __shfl_xor_sync(0xffffffffu, d, o);
        if (threadIdx.x == 0) *out = d;
    }
}

// *out = sum of part[0 .. np) in index order (one CTA, fixed tree)
__global__ void __launch_bounds__(kThreads) k_sum_parts(int32_t np, const double *__restrict__ part,
                                                        double *out) {
    __shared__ double s_red[kWarps];
    double d = 0.0;
    for (int i = threadIdx.x; i < np; i += kThreads) d += part[i];
    d = cta_sum(d, s_red);
    if (threadIdx.x == 0) *out = d;
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

// y[i] = (acc ? y[i] : 0) + ys[perm[i]]; with dot: part[blockIdx.x] = this
// block's share of <y, w> (w == y allowed; k_sum_parts adds them in order)
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
        if (threadIdx.x == 0) dot[blockIdx.x] = s;
    }
}

// Row-major form (plans whose tiles would stage about one entry per shared
// slot, e.g. c4's R-MAT, or would leave the grid idle, c2): the full CSR of
// A = D + L - L^T (fullcsr.h).  Each lane owns 16 consecutive entries: it
// issues their 16 x gathers at once and sums its row segments in order.  A
// row complete inside a lane is written by that lane; a row crossing lanes
// is summed by a fixed-order warp scan of the lanes' partials (the operator
// (m, t) o (m', t') = (m m', t + m t') over "the lane holds no row start");
// a row crossing warps is summed by k_csr_fix from the warps' tail / head
// partials in warp order.  No atomics: every y element is written once, the
// sum order is fixed by the plan (bitwise repeatable), and the arithmetic
// is plain fp64 (IEEE semantics for non-finite inputs).
#ifndef PARS3_CSR_MINB  // tuning builds
#define PARS3_CSR_MINB 2
#endif
__global__ void __launch_bounds__(256, PARS3_CSR_MINB) k_csr(int32_t nrows, int64_t ne, int64_t nwarps,
                                                const int32_t *__restrict__ col,
                                                const double *__restrict__ val,
                                                const int32_t *__restrict__ lane_row,
                                                const uint32_t *__restrict__ lane_flags,
                                                const double *__restrict__ x, double *__restrict__ y,
                                                double *__restrict__ whead, double *__restrict__ wtail) {
    constexpr int K = pars3::kCsrLane;
    const int lane = threadIdx.x & 31;
    const int64_t wstride = (int64_t)gridDim.x * (blockDim.x >> 5);
    for (int64_t w = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); w < nwarps; w += wstride) {
        // lane l holds the CSR entries e0 .. e0 + K - 1; the plan stores them
        // lane-interleaved (entry k of lane l at w * 512 + k * 32 + l), so
        // every load below is one coalesced 128 / 256-byte access per warp
        // (lane-contiguous storage cost 32 L1 wavefronts per load: 43 % of
        // the kernel's L1TEX cycles)
        const int64_t L = w * 32 + lane, e0 = L * K;
        int32_t c[K];
        double v[K], xc[K];
        const int32_t *cw = col + w * (32 * K) + lane;
        const double *vw = val + w * (32 * K) + lane;
#pragma unroll
        for (int k = 0; k < K; k++) c[k] = __ldcs(cw + 32 * k);
        const int32_t row0 = __ldcs(lane_row + L);
        const uint32_t fl = __ldcs(lane_flags + L);
#pragma unroll
        for (int k = 0; k < K; k++) {
            DCHECK(e0 + k >= ne || (c[k] >= 0 && c[k] < nrows));
            xc[k] = e0 + k < ne ? __ldg(x + c[k]) : 0.0;  // all in flight
        }
#pragma unroll
        for (int k = 0; k < K; k++) v[k] = __ldcs(vw + 32 * k);
        // the lane's row segments, in order
        const bool cont = !(fl & 1u);  // the first entry continues a row of an earlier lane
        bool first = true;
        double head = 0.0, s = 0.0;
        int32_t r = row0;
#pragma unroll
        for (int k = 0; k < K; k++) {
            if (k > 0 && ((fl >> k) & 1u)) {
                DCHECK(r >= 0 && r < nrows);
                if (first && cont)
                    head = s;
                else
                    y[r] = s;
                first = false;
                r++;
                s = 0.0;
            }
            s = fma(v[k], xc[k], s);
        }
        const bool open = !((fl >> K) & 1u);
        if (!open) {
            if (first && cont)
                head = s;
            else
                y[r] = s;
        }
        const bool single = first && cont && open;
        // fixed-order warp scan: out_l = t_l + m_l * out_{l-1}
        double t = open ? s : 0.0;
        int m = single ? 1 : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const double tp = __shfl_up_sync(0xffffffffu, t, o);
            const int mp = __shfl_up_sync(0xffffffffu, m, o);
            if (lane >= o) {
                if (m) t = t + tp;
                m &= mp;
            }
        }
        // (every lane takes part in the shuffles)
        const double tin = __shfl_up_sync(0xffffffffu, t, 1);
        const int mup = __shfl_up_sync(0xffffffffu, m, 1);
        const double in = lane == 0 ? 0.0 : tin;
        const int reach = lane == 0 ? 1 : mup;  // the lanes before are all single
        if (cont && !single) {  // this lane closes a row continued from earlier lanes
            const double a = head + in;
            if (reach)
                whead[w] = a;  // the row started in an earlier warp: k_csr_fix completes it
            else
                y[row0] = a;
        }
        if (lane == 31 && open) {
            if (m)
                whead[w] = t;  // the whole warp lies inside one row
            else
                wtail[w] = t;  // the last row's partial: it started in this warp
        }
    }
}

// rows crossing warps: y[row] = tail[w0] + head[w0 + 1] + ... + head[w1]
__global__ void __launch_bounds__(256) k_csr_fix(int32_t nspan, const int32_t *__restrict__ row,
                                                 const int32_t *__restrict__ w0, const int32_t *__restrict__ w1,
                                                 const double *__restrict__ whead,
                                                 const double *__restrict__ wtail, double *__restrict__ y) {
    const int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= nspan) return;
    const int32_t a = w0[i], b = w1[i];
    double s = wtail[a];
    int32_t w = a + 1;
    for (; w + 3 <= b; w += 4) {  // four loads in flight, summed in order
        const double h0 = whead[w], h1 = whead[w + 1], h2 = whead[w + 2], h3 = whead[w + 3];
        s = s + h0;
        s = s + h1;
        s = s + h2;
        s = s + h3;
    }
    for (; w <= b; w++) s = s + whead[w];
    y[row[i]] = s;
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
    int grid = 0, grid_redo = 0, conv_grid = 0, csr_grid = 148 * 2;
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
    GState *gs = nullptr;
    int64_t bytes = 0;
    Peers peers{};
    // grid form (deterministic single-GPU products)
    int32_t grid_ok = 0, xe_ready = 0, ev_g = 0, hgrid = 0, cmax = 0;
    double *blk_dot = nullptr, *blk_max = nullptr, *part = nullptr;
    long long *yacc = nullptr, *yacc2 = nullptr;  // (yacc2: the second accumulator, PARS3 two-buffer form)
    int32_t acc_turn = 0;
    const double *ep_p = nullptr, *ep_q = nullptr, *ep_a = nullptr, *ep_b = nullptr;  // this call's fused epilogue
    bool xbound_given = false;  // this call: the caller stored x's bound in gs->xe_pre (PARS3_PRODUCT_XBOUND)
    int32_t seen_fp64_tiles = 0, seen_redone = 0;  // pars3_plan_status: counters at its last call
    cudaEvent_t *prof = nullptr;  // pars3_plan_profile: events at the product's phase boundaries
    int prof_k = 0;
    // internal locality order (locality.cpp): the tiles hold P A P^T, x and
    // y pass through perm (split label -> internal label) and xs / ys
    int32_t *perm = nullptr, *iperm = nullptr;
    double *xs = nullptr, *ys = nullptr;
    int64_t local_slots = 0, dropped = 0;
    // row-major form (k_csr): the full CSR of A in lanes of 16 entries, no tiles
    int32_t built_on_device = 0;  // the tile plan came from tileplan_gpu.cu
    int32_t nfar = 0;             // far entries kept out of the tiles (k_far_grid / k_far_red)
    int32_t *far_row = nullptr, *far_col = nullptr;
    double *far_val = nullptr;
    int32_t direct = 0, nspan = 0;
    int64_t ne = 0, nwarps = 0;
    int32_t *ccol = nullptr, *clrow = nullptr, *span_row = nullptr, *span_w0 = nullptr, *span_w1 = nullptr;
    uint32_t *clflags = nullptr;
    double *cval = nullptr, *whead = nullptr, *wtail = nullptr, *yacc_tmp = nullptr;

    ~pars3_plan() {
        void *ptrs[] = {tiles, wins, slice_off, rec,    ucol,    diag, gs,   phase_clk, perm,
                        iperm, xs,   ys,        ccol,   cval,    clrow, clflags, span_row, span_w0,
                        span_w1, whead, wtail, yacc_tmp, blk_dot, blk_max, part, yacc, yacc2, far_row, far_col, far_val};
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
    if (s->n > 0) check(s->diag, s->n);
    return ok;
}

// The grid form's bounds: the most tiles delivering to one row block (each
// delivery is one rounding to the grid), the most terms one y element sums
// (Dmax: its row's entries, its column's mirrors and its diagonal: the
// grid's headroom) and the largest value exponent.  Every row must belong
// to a tile (no SKIP_EMPTY).
struct GridData {
    int32_t hgrid = 0, cmax = 0, ev_g = -1074;
};

// (far_terms / far_vmax: the far part's most terms on one row and its largest
// |value|: they join the grid's roundings, headroom and value bound)
static int grid_data(const pars3_split_view *v, const HostPlan &hp, GridData &G, int32_t far_terms = 0,
                     double far_vmax = 0.0) {
    const int64_t n = v->n;
    const int64_t nt = (int64_t)hp.tiles.size();
    std::vector<int32_t> blk(n, -1);
#pragma omp parallel for schedule(dynamic, 256)
    for (int64_t t = 0; t < nt; t++)
        for (int32_t r = hp.tiles[t].r0; r < hp.tiles[t].r1; r++) blk[r] = (int32_t)t;
    int64_t orphan = -1;
#pragma omp parallel for schedule(static) reduction(max : orphan)
    for (int64_t r = 0; r < n; r++)
        if (blk[r] < 0) orphan = std::max(orphan, r);
    if (orphan >= 0) PARS3_FAIL(PARS3_ERR_STRUCT, "grid form: row %lld belongs to no tile", (long long)orphan);
    std::vector<std::vector<int32_t>> lists(nt);
#pragma omp parallel for schedule(dynamic, 64)
    for (int64_t t = 0; t < nt; t++) {
        const TileMeta &m = hp.tiles[t];
        std::vector<int32_t> &L = lists[t];
        if (m.u0 >= 0) {
            int32_t last = -1;
            for (int32_t i = 0; i < m.local; i++) {
                const int32_t b = blk[hp.ucol[m.u0 + i]];
                if (b != last) L.push_back(last = b);
            }
        } else {
            for (int32_t w = m.w0; w < m.w1; w++) {
                int64_t c = hp.wins[w].lo;
                const int64_t hi = c + hp.wins[w].len;
                while (c < hi) {
                    const int32_t b = blk[c];
                    L.push_back(b);
                    c = hp.tiles[b].r1;
                }
            }
        }
        std::sort(L.begin(), L.end());
        L.erase(std::unique(L.begin(), L.end()), L.end());
    }
    std::vector<int32_t> need(nt, 0);  // tiles delivering to each row block
    for (int64_t t = 0; t < nt; t++)
        for (int32_t b : lists[t]) need[b]++;
    for (int64_t t = 0; t < nt; t++) {
        G.cmax = std::max(G.cmax, need[t]);
        G.ev_g = std::max(G.ev_g, hp.tiles[t].ev);
    }
    // terms per y element: row entries + column mirrors + the diagonal
    // (counted by the device builder when it built the plan)
    int64_t dmax = std::max<int64_t>(1, hp.dmax);
    double dg = 0.0;
    if (hp.dmax <= 0) {
        std::vector<int32_t> terms(n, 1);
        const int64_t nm = v->mid_ptr ? v->mid_ptr[n] : 0;
#pragma omp parallel for schedule(static)
        for (int64_t r = 0; r < n; r++) terms[r] += (int32_t)(v->mid_ptr[r + 1] - v->mid_ptr[r]);
#pragma omp parallel for schedule(static)
        for (int64_t k = 0; k < nm; k++) {
#pragma omp atomic
            terms[v->mid_col[k]]++;
        }
#pragma omp parallel for schedule(static)
        for (int64_t k = 0; k < v->outer_count; k++) {
#pragma omp atomic
            terms[v->outer_row[k]]++;
#pragma omp atomic
            terms[v->outer_col[k]]++;
        }
#pragma omp parallel for schedule(static) reduction(max : dmax)
        for (int64_t r = 0; r < n; r++) dmax = std::max<int64_t>(dmax, terms[r]);
    }
#pragma omp parallel for schedule(static) reduction(max : dg)
    for (int64_t r = 0; r < n; r++) dg = std::max(dg, std::fabs(v->diag[r]));
    dmax += far_terms;
    G.cmax += far_terms;
    if (far_vmax > 0.0) {
        int e = 0;
        std::frexp(far_vmax, &e);
        G.ev_g = std::max(G.ev_g, e);
    }
    while ((1ll << G.hgrid) < dmax) G.hgrid++;
    if (dg > 0.0) {
        int e = 0;
        std::frexp(dg, &e);  // |diag| < 2^e
        G.ev_g = std::max(G.ev_g, e);
    }
    return PARS3_OK;
}

// Far split of a locality-ordered matrix.  In the
// internal order nearly every entry lies within a couple of thousand labels
// of the diagonal (c3: 98.5 % within 2 560); the few long-range entries are
// what forces explicit column lists on the tiles.  Entries farther than T
// from the diagonal (a prefix of each row: columns ascend) are taken out
// into the far part (k_far_grid), so that the near part's tiles are dense
// column windows: TMA copies of x and coalesced deliveries instead of one
// gather and one reduction per slot.
struct FarSplit {
    std::vector<int64_t> nptr;
    std::vector<int32_t> ncol, frow, fcol;
    std::vector<double> nval, fval;
    double fvmax = 0.0;
    int32_t fterms = 0;  // most far terms on one row
};

static bool split_far(const LocalityOrder &lo, int64_t n, int32_t T, FarSplit &fs) {
    const int64_t m = lo.row_ptr[n];
    std::vector<int64_t> fptr(n + 1, 0);
    fs.nptr.assign(n + 1, 0);
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; i++) {
        int64_t k = lo.row_ptr[i];
        while (k < lo.row_ptr[i + 1] && i - lo.col[k] > T) k++;
        fptr[i + 1] = k - lo.row_ptr[i];
        fs.nptr[i + 1] = lo.row_ptr[i + 1] - k;
    }
    for (int64_t i = 0; i < n; i++) {
        fptr[i + 1] += fptr[i];
        fs.nptr[i + 1] += fs.nptr[i];
    }
    const int64_t nf = fptr[n];
    if (nf == 0 || 20 * nf > m || nf >= INT32_MAX) return false;
    fs.frow.resize(nf);
    fs.fcol.resize(nf);
    fs.fval.resize(nf);
    fs.ncol.resize(m - nf);
    fs.nval.resize(m - nf);
    std::vector<int32_t> terms(n, 0);
    double vmax = 0.0;
#pragma omp parallel for schedule(static) reduction(max : vmax)
    for (int64_t i = 0; i < n; i++) {
        int64_t k = lo.row_ptr[i];
        for (int64_t f = fptr[i]; f < fptr[i + 1]; f++, k++) {
            fs.frow[f] = (int32_t)i;
            fs.fcol[f] = lo.col[k];
            fs.fval[f] = lo.val[k];
            vmax = std::max(vmax, std::fabs(lo.val[k]));
#pragma omp atomic
            terms[i]++;
#pragma omp atomic
            terms[lo.col[k]]++;
        }
        for (int64_t q = fs.nptr[i]; q < fs.nptr[i + 1]; q++, k++) {
            fs.ncol[q] = lo.col[k];
            fs.nval[q] = lo.val[k];
        }
    }
    int32_t tmax = 0;
#pragma omp parallel for schedule(static) reduction(max : tmax)
    for (int64_t i = 0; i < n; i++) tmax = std::max(tmax, terms[i]);
    fs.fvmax = vmax;
    fs.fterms = tmax;
    return true;
}

extern "C" int pars3_plan_create(const pars3_split_view *s, const pars3_plan_options *opt,
                                 int32_t p, const int64_t *block_start, pars3_plan **out,
                                 void *stream) {
    return pars3_plan_create_resident(s, nullptr, opt, p, block_start, out, stream);
}

extern "C" int pars3_plan_create_resident(const pars3_split_view *s, const pars3_split_view *resident,
                                          const pars3_plan_options *opt, int32_t p,
                                          const int64_t *block_start, pars3_plan **out, void *stream) {
    (void)stream;
    if (resident && s && (resident->n != s->n || resident->outer_count != s->outer_count || !resident->mid_ptr))
        PARS3_FAIL(PARS3_ERR_ARG, "the device-resident split does not match the host split");
    if (!s || !out) PARS3_FAIL(PARS3_ERR_ARG, "null argument");
    *out = nullptr;
    if (s->n < 0 || s->n >= INT32_MAX || s->beta < 1) PARS3_FAIL(PARS3_ERR_ARG, "bad split header");
    if (p < 1) PARS3_FAIL(PARS3_ERR_ARG, "worker count must be at least 1, got %d", p);
    PlanOptions o0;
    int32_t max_ctas = 0, flags = 0;
    if (const char *tr = getenv("PARS3_TILE_ROWS")) o0.tile_rows = std::max(1, atoi(tr));  // tuning knob
    if (opt) {
        if (opt->tile_rows > 0) o0.tile_rows = opt->tile_rows;
        if (opt->local_slots > 0) o0.local_slots = opt->local_slots;
        if (opt->seg_max > 0) o0.seg_max = opt->seg_max;
        if (opt->gap >= 0) o0.gap = opt->gap;
        if (opt->mode > 0) o0.mode = opt->mode;
        o0.skip_empty = (opt->flags & PARS3_PLAN_SKIP_EMPTY) != 0;
        if (o0.skip_empty) {
            // a skipped row has no slot, so it could not take its diagonal term
            // (and a list tile's own rows would no longer be the tail of its
            // column list): SKIP_EMPTY plans carry no diagonal
            for (int64_t i = 0; i < s->n; i++)
                if (s->diag[i] != 0.0)
                    PARS3_FAIL(PARS3_ERR_ARG, "PARS3_PLAN_SKIP_EMPTY needs an all-zero diagonal (row %lld has %g)",
                               (long long)i, s->diag[i]);
        }
        if ((opt->flags & PARS3_PLAN_CUT_BLOCKS) && block_start && p > 1)
            for (int32_t r = 1; r < p; r++) o0.cuts.push_back((int32_t)block_start[r]);
        if (opt->max_ctas > 0) max_ctas = opt->max_ctas;
        flags = opt->flags;
    }
    if (const char *ff = getenv("PARS3_FORCE_FLAGS")) flags |= atoi(ff);  // debug / tuning knob
    // accumulation of the mirror sums: mode 2 = fp64 shared accumulators,
    // mode 1 = exact-integer fixed point in three words, mode 3 = two words
    // (needs <= kTerms2 terms per slot and tile), mode 0 = auto: two words
    // when the plan allows, else three words (<= 4096 terms; exact integer
    // sums keep the product bitwise repeatable), else fp64
    const int req_mode = opt ? opt->mode : 0;
    // PARS3_VERBOSE=1: wall-clock of the plan's phases on stderr
    const bool verbose = getenv("PARS3_VERBOSE") != nullptr;
    double t_prev = omp_get_wtime();
    auto lap = [&](const char *what) {
        const double now = omp_get_wtime();
        if (verbose) fprintf(stderr, "pars3 plan: %-28s %.3f s\n", what, now - t_prev);
        t_prev = now;
    };
    const bool safe_values = values_fixed_point_safe(s);
    lap("value range check");
    int words0 = req_mode == 1 ? 3 : req_mode == 2 ? 0 : 2;
    if (words0 && !safe_values) words0 = 0;  // fp64 accumulators keep IEEE semantics
    // the shared-memory budget (x + accumulators per slot, 4 CTAs / SM) caps both
    if (o0.seg_max > 8) o0.seg_max = 8;
    const int32_t want_local = o0.local_slots;
    o0.max_segments = std::min(o0.max_segments, 32 * kMaxTileSlices);
    // The tile plan is built on the device when it can be (window-mode
    // plans: tileplan_gpu.cu, the same arrays byte for byte, left on the
    // device in `dp`), else by the host builder.  PARS3_PLAN_HOST=1 /
    // PARS3_PLAN_HOST_BUILD: always the host builder.
    const char *ph_env = getenv("PARS3_PLAN_HOST");
    const bool may_device = !(ph_env && ph_env[0] == '1') && !(flags & PARS3_PLAN_HOST_BUILD);
    auto tile_plan = [&](const pars3_split_view *v, const PlanOptions &o, HostPlan &hp, pars3::DevicePlan *dp) -> int {
        if (dp) {
            dp->release();
            bool ok = false;
            if (may_device) {
                pars3::DeviceSplit ds{};
                if (resident && v == s)
                    ds = pars3::DeviceSplit{resident->mid_ptr, resident->mid_col, resident->mid_val,
                                            resident->outer_row, resident->outer_col, resident->outer_val};
                const int rc = pars3::build_tile_plan_device(v->n, v->mid_ptr, v->mid_col, v->mid_val, v->outer_count,
                                                             v->outer_row, v->outer_col, v->outer_val, o, hp, *dp, ok,
                                                             resident && v == s ? &ds : nullptr);
                if (rc) return rc;
            }
            if (ok) return PARS3_OK;
        }
        return pars3::build_tile_plan(v->n, v->mid_ptr, v->mid_col, v->mid_val, v->outer_count, v->outer_row,
                                      v->outer_col, v->outer_val, o, hp);
    };
    auto build = [&](const pars3_split_view *v, PlanOptions &o, int &words, HostPlan &hp,
                     pars3::DevicePlan *dp) -> int {
        o = o0;
        words = words0;
        o.terms_cap = words == 2 ? kTerms2 : 0;
        if (const char *ts = getenv("PARS3_TERMS_MIN_ROWS")) o.terms_min_rows = atoi(ts);  // tuning knob
        o.local_slots = std::min(want_local, words == 3 ? kLocalFixed : kLocalExact);
        o.sink = (uint16_t)(words == 3 ? Layout<3>::kSink : Layout<0>::kSink);
        int rc = tile_plan(v, o, hp, dp);
        if (rc) return rc;
        if (words == 2 && hp.max_terms > kTerms2) {
            if (req_mode == 3)
                PARS3_FAIL(PARS3_ERR_ARG, "two-word accumulation needs <= %d terms per slot, plan has %d",
                           kTerms2, hp.max_terms);
            words = 3;
            o.terms_cap = 0;
            o.local_slots = std::min(want_local, kLocalFixed);
            o.sink = (uint16_t)Layout<3>::kSink;
            hp = HostPlan();
            rc = tile_plan(v, o, hp, dp);
            if (rc) return rc;
        }
        // the three 20-bit limbs carry <= 4096 terms per slot and tile
        if (words == 3 && hp.max_terms > kTerms3) {
            if (req_mode == 1)
                PARS3_FAIL(PARS3_ERR_ARG, "three-word accumulation needs <= %d terms per slot, plan has %d",
                           kTerms3, hp.max_terms);
            words = 0;
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
    struct DpGuard {  // (frees the device-built arrays unless the plan takes them)
        pars3::DevicePlan d;
        ~DpGuard() { d.release(); }
    } dpg;
    pars3::DevicePlan &dp = dpg.d;
    const bool may_permute =
        !(flags & (PARS3_PLAN_CUT_BLOCKS | PARS3_PLAN_NO_LOCALITY | PARS3_PLAN_DIRECT)) && s->n > 1;
    const int64_t m_total = (s->mid_ptr ? s->mid_ptr[s->n] : 0) + s->outer_count;
    // A sample of the row ranges first (every k-th range, host builder): when
    // it shows an unstructured matrix -- mostly list tiles with few entries
    // per slot -- the locality order is tried before paying for the full
    // plan in the caller's labels, which is then built only if that fails.
    int rc = PARS3_OK;
    bool deferred = false, direct_sample = false;
    int64_t local = 0;
    {
        const int64_t nranges = (s->n + o0.tile_rows - 1) / std::max(1, o0.tile_rows);
        const char *ns_env = getenv("PARS3_NO_SAMPLE");  // A/B knob
        if (may_permute && nranges >= 512 && m_total > 0 && !(ns_env && ns_env[0] == '1')) {
            PlanOptions os = o0;
            os.terms_cap = words0 == 2 ? kTerms2 : 0;
            os.local_slots = std::min(want_local, words0 == 3 ? kLocalFixed : kLocalExact);
            os.sink = (uint16_t)(words0 == 3 ? Layout<3>::kSink : Layout<0>::kSink);
            os.sample_stride = (int32_t)(nranges / 64);
            HostPlan hs;
            rc = pars3::build_tile_plan(s->n, s->mid_ptr, s->mid_col, s->mid_val, s->outer_count, s->outer_row,
                                        s->outer_col, s->outer_val, os, hs);
            if (rc) return rc;
            const int64_t ls = local_of(hs);
            if (hs.nnz > 0 && 2ll * hs.list_tiles > (int64_t)hs.tiles.size() && 4 * ls > hs.nnz) {
                deferred = true;
                local = (int64_t)((double)ls * (double)m_total / (double)hs.nnz);  // the full plan's, estimated
                direct_sample = 10 * ls >= 9 * hs.nnz;  // about one entry per slot: the row-major form
            }
            lap("structure sample");
        }
    }
    if (!deferred) {
        rc = build(s, o, words, hp, &dp);
        if (rc) return rc;
        lap(dp.rec ? "tile plan (device)" : "tile plan (host)");
        local = local_of(hp);
    }
    // internal locality order (locality.cpp): tried when most tiles are
    // unstructured list tiles whose slots hold few entries each, kept when
    // it cuts the shared-memory slots (= x gathers + y reductions) by 30 %
    LocalityOrder lo;
    FarSplit fs;  // the near part's arrays (the tiles' split) and the far part, when used
    bool far_used = false;
    const bool unstructured =
        deferred || (2ll * hp.list_tiles > (int64_t)hp.tiles.size() && 4 * local > hp.nnz);
    if (may_permute && (unstructured || (flags & PARS3_PLAN_LOCALITY)) && m_total > 0) {
        rc = pars3::locality_order(s, lo);
        if (rc) return rc;
        lap("locality order");
        const bool no_order = lo.forward.empty();  // (no local structure to recover: locality.cpp)
        // first with the long-range entries taken out (window-mode tiles + the far part) ...
        const char *nf_env = getenv("PARS3_NO_FAR");  // A/B knob
        if (!no_order && !(nf_env && nf_env[0] == '1')) {
            const int32_t T = std::min(want_local, words0 == 3 ? kLocalFixed : kLocalExact) - 640;
            if (T >= 256 && split_far(lo, s->n, T, fs)) {
                pars3_split_view vn{s->n, s->beta, lo.diag.data(), fs.nptr.data(), fs.ncol.data(),
                                    fs.nval.data(), 0, nullptr, nullptr, nullptr};
                PlanOptions o2;
                int words2 = 0;
                HostPlan hp2;
                DpGuard dpn;  // (the first plan's device arrays stay until this one is accepted)
                rc = build(&vn, o2, words2, hp2, &dpn.d);
                if (rc) return rc;
                lap("tile plan, near part");
                const int64_t local2 = local_of(hp2);
                if (verbose)
                    fprintf(stderr, "pars3 plan: near part: T %d far %zu tiles %zu list %d slots %lld (was %lld) words %d "
                                    "max terms %d\n", T, fs.frow.size(), hp2.tiles.size(), hp2.list_tiles,
                            (long long)local2, (long long)local, words2, hp2.max_terms);
                if (10ll * hp2.list_tiles <= (int64_t)hp2.tiles.size() && 10 * local2 < 7 * local) {
                    o = o2;
                    words = words2;
                    hp = std::move(hp2);
                    local = local2;
                    far_used = true;
                    dp.release();
                    dp = dpn.d;
                    dpn.d = pars3::DevicePlan();
                }
            }
        }
        // ... else every entry in the tiles
        if (!far_used && !no_order) {
            fs = FarSplit();
            pars3_split_view v{s->n, s->beta, lo.diag.data(), lo.row_ptr.data(), lo.col.data(),
                               lo.val.data(), 0, nullptr, nullptr, nullptr};
            PlanOptions o2;
            int words2 = 0;
            HostPlan hp2;
            rc = build(&v, o2, words2, hp2, nullptr);
            if (rc) return rc;
            lap("tile plan, locality order");
            const int64_t local2 = local_of(hp2);
            if (10 * local2 < 7 * local) {
                dp.release();
                o = o2;
                words = words2;
                hp = std::move(hp2);
                local = local2;
            } else {
                lo = LocalityOrder();
            }
        }
    }
    // (PARS3_PLAN_LOCALITY forces the attempt on small matrices in tests: such
    // a plan was never deferred)
    direct_sample = direct_sample && deferred && lo.forward.empty() &&
                    !(flags & (PARS3_PLAN_CUT_BLOCKS | PARS3_PLAN_SKIP_EMPTY | PARS3_PLAN_NO_DIRECT));
    if (direct_sample) {
        hp = HostPlan();  // the row-major form needs no tiles
        hp.nnz = m_total;
    } else if (deferred && lo.forward.empty()) {  // no order was kept: the plan in the caller's labels after all
        rc = build(s, o, words, hp, &dp);
        if (rc) return rc;
        lap(dp.rec ? "tile plan (device)" : "tile plan (host)");
        local = local_of(hp);
    }
    // the split the tiles were built from (the caller's, or P A P^T)
    pars3_split_view used = *s;
    if (far_used)
        used = pars3_split_view{s->n, s->beta, lo.diag.data(), fs.nptr.data(), fs.ncol.data(),
                                fs.nval.data(), 0, nullptr, nullptr, nullptr};
    else if (!lo.forward.empty())
        used = pars3_split_view{s->n, s->beta, lo.diag.data(), lo.row_ptr.data(), lo.col.data(),
                                lo.val.data(), 0, nullptr, nullptr, nullptr};
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
        ((flags & PARS3_PLAN_DIRECT) || few_tiles || direct_sample ||
         (2ll * hp.list_tiles > (int64_t)hp.tiles.size() && 10 * local >= 9 * hp.nnz));
    pars3::FullCsr F;
    struct DfGuard {
        pars3::DeviceFullCsr d;
        ~DfGuard() { d.release(); }
    } dfg;
    pars3::DeviceFullCsr &DF = dfg.d;
    if (direct) {  // the full CSR of A: on the device (fullcsr_gpu.cu), else on the host (fullcsr.cpp)
        bool on_device = false;
        if (may_device) {
            rc = pars3::build_full_csr_device(s, DF, on_device);
            if (rc) return rc;
        }
        if (!on_device) {
            rc = pars3::build_full_csr(s, F);
            if (rc) return rc;
        }
        lap(on_device ? "full CSR (device)" : "full CSR (host)");
        const int64_t m_entries = hp.nnz;
        hp = HostPlan();  // no tiles are uploaded
        hp.nnz = m_entries;
        dp.release();
    }
    // grid form: single-GPU tile plans over finite, fixed-point-safe values
    // where every row belongs to a tile
    GridData G;
    const bool grid_ok = !direct && !hp.tiles.empty() && safe_values && !o0.skip_empty;
    if (grid_ok) {
        try {
            rc = grid_data(&used, hp, G, far_used ? fs.fterms : 0, far_used ? fs.fvmax : 0.0);
        } catch (const std::bad_alloc &) {
            PARS3_FAIL(PARS3_ERR_NOMEM, "out of host memory");
        }
        if (rc) return rc;
        lap("grid bounds");
    }
    pars3_plan *pl = new (std::nothrow) pars3_plan;
    if (!pl) PARS3_FAIL(PARS3_ERR_NOMEM, "out of host memory");
    pl->n = s->n;
    pl->beta = s->beta;
    pl->p = p;
    pl->ntiles = (int32_t)hp.tiles.size();
    pl->nslices = dp.rec ? (int32_t)dp.nslices : std::max<int32_t>(0, (int32_t)hp.slice_off.size() - 1);
    pl->built_on_device = dp.rec ? 1 : 0;
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
        const char *ng = getenv("PARS3_NO_GRID");  // A/B knob: the RED form for every product
        pl->grid_ok = grid_ok && !(ng && ng[0] == '1');
    }
    pl->local_slots = local;
    pl->dropped = lo.dropped;
    // (a constant diagonal, strict or shifted skew, is not uploaded)
    const double *dsrc = lo.forward.empty() ? s->diag : lo.diag.data();
    pl->diag_alpha = s->n ? dsrc[0] : 0.0;
    {
        int varies = 0;
        const double d0 = pl->diag_alpha;
#pragma omp parallel for schedule(static) reduction(| : varies)
        for (int64_t i = 0; i < s->n; i++) varies |= dsrc[i] != d0;
        pl->diag_const = !varies;
    }
    std::vector<double> diag;
    if (!pl->diag_const) diag.assign(dsrc, dsrc + s->n);
#define UP(dst, src)                               \
    do {                                           \
        int _r = upload(&pl->dst, src);            \
        if (_r) {                                  \
            delete pl;                             \
            return _r;                             \
        }                                          \
        pl->bytes += sizeof(src[0]) * src.size();  \
    } while (0)
#define ZALLOC(dst, count)                                                                    \
    do {                                                                                      \
        const size_t _b = sizeof(*pl->dst) * (size_t)(count);                                 \
        if (cudaMalloc((void **)&pl->dst, _b) != cudaSuccess || cudaMemset(pl->dst, 0, _b) != cudaSuccess) { \
            delete pl;                                                                        \
            PARS3_FAIL(PARS3_ERR_CUDA, "cudaMalloc failed");                                  \
        }                                                                                     \
        pl->bytes += (int64_t)_b;                                                             \
    } while (0)
    if (direct && DF.col) {  // built on the device (already lane-interleaved): the plan takes the arrays
        pl->direct = 1;
        pl->built_on_device = 1;
        pl->ne = DF.ne;
        pl->nwarps = DF.nep / pars3::kCsrWarp;
        pl->nspan = DF.nspan;
        pl->ccol = DF.col;
        pl->cval = DF.val;
        pl->clrow = DF.lane_row;
        pl->clflags = DF.lane_flags;
        pl->span_row = DF.span_row;
        pl->span_w0 = DF.span_w0;
        pl->span_w1 = DF.span_w1;
        pl->bytes += (int64_t)(12 * DF.nep + 8 * (DF.nep / pars3::kCsrLane) + 12 * (int64_t)DF.nspan);
        DF = pars3::DeviceFullCsr();
        ZALLOC(whead, std::max<int64_t>(1, pl->nwarps));
        ZALLOC(wtail, std::max<int64_t>(1, pl->nwarps));
    } else if (direct) {
        {  // lane-interleaved storage within each warp of 512 entries (k_csr)
            const int64_t nw = (int64_t)F.col.size() / pars3::kCsrWarp;
            std::vector<int32_t> c2(F.col.size());
            std::vector<double> v2(F.val.size());
#pragma omp parallel for schedule(static)
            for (int64_t w = 0; w < nw; w++)
                for (int l = 0; l < 32; l++)
                    for (int k = 0; k < pars3::kCsrLane; k++) {
                        const int64_t src = w * pars3::kCsrWarp + l * pars3::kCsrLane + k;
                        const int64_t dst = w * pars3::kCsrWarp + k * 32 + l;
                        c2[dst] = F.col[src];
                        v2[dst] = F.val[src];
                    }
            F.col.swap(c2);
            F.val.swap(v2);
        }
        pl->direct = 1;
        pl->ne = F.ne;
        pl->nwarps = (int64_t)F.col.size() / pars3::kCsrWarp;
        pl->nspan = (int32_t)F.span_row.size();
        UP(ccol, F.col);
        UP(cval, F.val);
        UP(clrow, F.lane_row);
        UP(clflags, F.lane_flags);
        UP(span_row, F.span_row);
        UP(span_w0, F.span_w0);
        UP(span_w1, F.span_w1);
        ZALLOC(whead, std::max<int64_t>(1, pl->nwarps));
        ZALLOC(wtail, std::max<int64_t>(1, pl->nwarps));
    }
    if (dp.rec) {  // built on the device: the plan takes the arrays
        pl->tiles = dp.tiles;
        pl->wins = dp.wins;
        pl->slice_off = dp.slice_off;
        pl->rec = dp.rec;
        pl->bytes += (int64_t)(sizeof(TileMeta) * dp.ntiles + sizeof(Window) * dp.nwins +
                               sizeof(int64_t) * (dp.nslices + 1) + dp.rec_bytes);
        dp = pars3::DevicePlan();
    } else {
        UP(tiles, hp.tiles);
        UP(wins, hp.wins);
        UP(slice_off, hp.slice_off);
        UP(rec, hp.rec);
    }
    UP(ucol, hp.ucol);
    if (far_used) {
        pl->nfar = (int32_t)fs.frow.size();
        UP(far_row, fs.frow);
        UP(far_col, fs.fcol);
        UP(far_val, fs.fval);
    }
    if (!pl->diag_const) UP(diag, diag);
    if (!lo.forward.empty()) {
        UP(perm, lo.forward);
        std::vector<int32_t> inv(lo.forward.size());
        for (size_t i = 0; i < inv.size(); i++) inv[lo.forward[i]] = (int32_t)i;
        UP(iperm, inv);
        ZALLOC(xs, pl->n);
        ZALLOC(ys, pl->n);
    }
    ZALLOC(gs, 1);
    ZALLOC(part, kDotGrid + 1);  // (+ k_dot's arrival counter)
    static_assert(kConvGrid >= kDotGrid, "blk_dot / blk_max hold k_conv's shares");
    {
        GState g0{};
        g0.xe = kXeNone;
        g0.xe_seen = kXeNone;
        if (cudaMemcpy(pl->gs, &g0, sizeof(g0), cudaMemcpyHostToDevice) != cudaSuccess) {
            delete pl;
            PARS3_FAIL(PARS3_ERR_CUDA, "cudaMemcpy failed");
        }
    }
    if (grid_ok) {
        pl->ev_g = G.ev_g;
        pl->hgrid = G.hgrid;
        pl->cmax = G.cmax;
        ZALLOC(blk_dot, std::max<int64_t>(pl->ntiles, kConvGrid));
        ZALLOC(blk_max, std::max<int64_t>(pl->ntiles, kConvGrid));
        ZALLOC(yacc, pl->n);
        const char *tb = getenv("PARS3_TWO_ACC");  // A/B knob
        if (!(tb && tb[0] == '0')) ZALLOC(yacc2, pl->n);
    }
#undef UP
#undef ZALLOC
    pl->smem = pl->words == 0 ? Layout<0>::kSmem : pl->words == 2 ? Layout<2>::kSmem : Layout<3>::kSmem;
    // the attribute is per function, shared by every plan: set it to the
    // function's fixed layout size
    cudaError_t e = cudaSuccess;
    {
        const void *fns[10] = {
            (const void *)k_tiles<0, false, false>, (const void *)k_tiles<2, false, false>,
            (const void *)k_tiles<3, false, false>, (const void *)k_tiles<0, true, false>,
            (const void *)k_tiles<2, true, false>,  (const void *)k_tiles<3, true, false>,
            (const void *)k_tiles<0, false, true>,  (const void *)k_tiles<2, false, true>,
            (const void *)k_tiles<3, false, true>,  (const void *)k_finish};
        const int sm[3] = {Layout<0>::kSmem, Layout<2>::kSmem, Layout<3>::kSmem};
        for (int f = 0; f < 10 && e == cudaSuccess; f++)
            e = cudaFuncSetAttribute(fns[f], cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     f == 9 ? kFinishSmem : sm[f % 3]);
    }
    int per_sm = 0, per_sm_redo = 0, sms = 0, dev = 0;
    if (e == cudaSuccess) e = cudaGetDevice(&dev);
    if (e == cudaSuccess) e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (e == cudaSuccess)
        e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(
            &per_sm, pl->words == 0 ? k_tiles<0, false, true> : pl->words == 2 ? k_tiles<2, false, true> : k_tiles<3, false, true>,
            kThreads, pl->smem);
    if (e == cudaSuccess)
        e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(
            &per_sm_redo, k_finish, kThreads, kFinishSmem);
    if (e != cudaSuccess || per_sm < 1 || per_sm_redo < 1) {
        delete pl;
        PARS3_FAIL(PARS3_ERR_CUDA, "tile kernel cannot be resident (smem %zu B): %s", pl->smem,
                   cudaGetErrorString(e));
    }
    pl->grid = per_sm * sms;
    if (max_ctas > 0 && pl->grid > max_ctas) pl->grid = max_ctas;
    if (pl->grid > pl->ntiles) pl->grid = pl->ntiles > 0 ? pl->ntiles : 1;
    pl->grid_redo = std::min(pl->grid, per_sm_redo * sms);
    {  // k_csr: one resident wave of CTAs
        int per_sm_csr = 0;
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm_csr, k_csr, 256, 0) != cudaSuccess || per_sm_csr < 1)
            per_sm_csr = 1;
        pl->csr_grid = per_sm_csr * sms;
    }
    {  // k_conv: one resident wave (measured: 1 184 CTAs in four waves 58 us, one wave of 296 52 us on c5)
        int per_sm_conv = 0;
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm_conv, k_conv<true>, kConvThreads, 0) != cudaSuccess ||
            per_sm_conv < 1)
            per_sm_conv = 1;
        pl->conv_grid = std::min(kConvGrid, per_sm_conv * sms);
        if (const char *e = getenv("PARS3_CONV_GRID")) pl->conv_grid = std::max(1, std::min(kConvGrid, atoi(e)));
    }
    lap("upload");
    *out = pl;
    return PARS3_OK;
}

static DevPlan dev_plan(const pars3_plan *pl) {
    DevPlan P{};
    P.tiles = pl->tiles;
    P.wins = pl->wins;
    P.slice_off = pl->slice_off;
    P.rec = pl->rec;
    P.ucol = pl->ucol;
    P.diag = pl->diag;
    P.ntiles = pl->ntiles;
    P.n = (int32_t)pl->n;
    P.watchdog = pl->watchdog;
    P.diag_const = pl->diag_const;
    P.diag_alpha = pl->diag_alpha;
    P.phase_clk = pl->phase_clk;
    P.pf = pl->pf;
    P.pf_dist = pl->pf_dist;
    P.peers = pl->peers;
    P.gs = pl->gs;
    P.blk_dot = pl->blk_dot;
    P.blk_max = pl->blk_max;
    P.yacc = pl->yacc;
    P.ev_g = pl->ev_g;
    P.hgrid = pl->hgrid;
    P.cmax = pl->cmax;
    P.far_row = pl->far_row;
    P.far_col = pl->far_col;
    P.far_val = pl->far_val;
    P.nfar = pl->nfar;
    P.ep_p = pl->ep_p;
    P.ep_q = pl->ep_q;
    P.ep_a = pl->ep_a;
    P.ep_b = pl->ep_b;
    return P;
}

// pars3_plan_profile: record the next phase-boundary event
static void mark(pars3_plan *pl, cudaStream_t st) {
    if (pl->prof && pl->prof_k < 4) cudaEventRecord(pl->prof[pl->prof_k++], st);
}

// RED form over the tiles: y (+)= A x with fp64 reductions (peer mode, y +=
// A x, plans without the grid form).  y zeroed first unless `acc`.  The
// claim counter is zero between products (k_finish resets it after a grid
// product, this launch after its own).
static int launch_red(pars3_plan *pl, const double *x, double *y, bool acc, cudaStream_t st) {
    if (!acc && pl->n > 0) CUDA_TRY(cudaMemsetAsync(y, 0, sizeof(double) * (size_t)pl->n, st));
    if (pl->ntiles == 0) return PARS3_OK;
    const DevPlan P = dev_plan(pl);
    const bool peer = pl->peers.nranks > 0;
    if (pl->words == 0)
        (peer ? k_tiles<0, true, false> : k_tiles<0, false, false>)<<<pl->grid, kThreads, pl->smem, st>>>(
            P, x, y, nullptr, nullptr, 0);
    else if (pl->words == 2)
        (peer ? k_tiles<2, true, false> : k_tiles<2, false, false>)<<<pl->grid, kThreads, pl->smem, st>>>(
            P, x, y, nullptr, nullptr, 0);
    else
        (peer ? k_tiles<3, true, false> : k_tiles<3, false, false>)<<<pl->grid, kThreads, pl->smem, st>>>(
            P, x, y, nullptr, nullptr, 0);
    LAUNCH_CHECK();
    if (pl->nfar > 0) {
        k_far_red<<<std::min(148 * 64, (pl->nfar + 255) / 256), 256, 0, st>>>(P, x, y);
        LAUNCH_CHECK();
    }
    mark(pl, st);
    CUDA_TRY(cudaMemsetAsync(&pl->gs->claim, 0, sizeof(int32_t), st));
    return PARS3_OK;
}

// GRID form: y = A x written by the block finalizers, *dot = <y, w> fused
// when w is y (dot_self) or given, by k_finish (which redoes flagged products)
static int launch_grid(pars3_plan *pl, const double *x, double *y, const double *w, double *dot,
                       bool dot_self, bool strict, cudaStream_t st) {
    DevPlan P = dev_plan(pl);
    if (pl->yacc2) {  // this product's accumulator, and the one its tiles clear
        P.yacc = pl->acc_turn ? pl->yacc2 : pl->yacc;
        P.yclear = pl->acc_turn ? pl->yacc : pl->yacc2;
        pl->acc_turn ^= 1;
    }
    if (strict && pl->xbound_given) {  // the caller's kernel already stored this x's bound
        pl->xe_ready = 1;
        P.strict = 1;
    } else if (strict || !pl->xe_ready) {  // the scale bound from a pass over this x
        CUDA_TRY(cudaMemsetAsync(&pl->gs->xe_pre, 0, sizeof(int32_t), st));
        const int grid = (int)std::min<int64_t>(148 * 4, (pl->n + 511) / 512);
        k_xmax<<<grid, 512, 0, st>>>((int32_t)pl->n, x, pl->gs);
        LAUNCH_CHECK();
        pl->xe_ready = 1;
        P.strict = 1;
    }
    const int ds = dot_self ? 1 : 0;
    if (pl->words == 0)
        k_tiles<0, false, true><<<pl->grid, kThreads, pl->smem, st>>>(P, x, y, w, dot, ds);
    else if (pl->words == 2)
        k_tiles<2, false, true><<<pl->grid, kThreads, pl->smem, st>>>(P, x, y, w, dot, ds);
    else
        k_tiles<3, false, true><<<pl->grid, kThreads, pl->smem, st>>>(P, x, y, w, dot, ds);
    LAUNCH_CHECK();
    if (pl->nfar > 0) {
        k_far_grid<<<std::min(148 * 64, (pl->nfar + 255) / 256), 256, 0, st>>>(P, x);
        LAUNCH_CHECK();
    }
    mark(pl, st);
    int32_t n32 = (int32_t)pl->n;
    if (P.ep_a)
        k_conv<true><<<pl->conv_grid, kConvThreads, 0, st>>>(P, y, w, dot, ds, n32);
    else
        k_conv<false><<<pl->conv_grid, kConvThreads, 0, st>>>(P, y, w, dot, ds, n32);
    LAUNCH_CHECK();
    void *args[] = {(void *)&P, (void *)&x, (void *)&y, (void *)&w, (void *)&dot, (void *)&ds, (void *)&n32};
    CUDA_TRY(cudaLaunchCooperativeKernel((const void *)k_finish, dim3(pl->grid_redo), dim3(kThreads), args,
                                         kFinishSmem, st));
    return PARS3_OK;
}

__global__ void __launch_bounds__(512) k_add(int32_t n, const double *__restrict__ a, double *y) {
    const int32_t stride = gridDim.x * blockDim.x;
    for (int32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) y[i] += a[i];
}

// row-major form: y = A x (k_csr + k_csr_fix); y += A x through a scratch
static int launch_direct(pars3_plan *pl, const double *x, double *y, bool acc, cudaStream_t st) {
    if (pl->n == 0) return PARS3_OK;
    double *out = y;
    if (acc) {
        if (!pl->yacc_tmp) CUDA_TRY(cudaMalloc((void **)&pl->yacc_tmp, sizeof(double) * (size_t)pl->n));
        out = pl->yacc_tmp;
    }
    const int grid = (int)std::min<int64_t>(pl->csr_grid, (pl->nwarps + 7) / 8);
    k_csr<<<grid, 256, 0, st>>>((int32_t)pl->n, pl->ne, pl->nwarps, pl->ccol, pl->cval, pl->clrow, pl->clflags, x, out,
                                pl->whead, pl->wtail);
    LAUNCH_CHECK();
    mark(pl, st);
    if (pl->nspan > 0) {
        k_csr_fix<<<(pl->nspan + 255) / 256, 256, 0, st>>>(pl->nspan, pl->span_row, pl->span_w0, pl->span_w1,
                                                          pl->whead, pl->wtail, out);
        LAUNCH_CHECK();
    }
    if (acc) {
        const int g = (int)std::min<int64_t>(148 * 4, (pl->n + 511) / 512);
        k_add<<<g, 512, 0, st>>>((int32_t)pl->n, out, y);
        LAUNCH_CHECK();
    }
    return PARS3_OK;
}

// deterministic <a, b> into *out (part: kDotGrid doubles of scratch)
static int launch_dot(int64_t n, const double *a, const double *b, double *part, double *out, cudaStream_t st) {
    if (n == 0) {
        CUDA_TRY(cudaMemsetAsync(out, 0, sizeof(double), st));
        return PARS3_OK;
    }
    if (((uintptr_t)a | (uintptr_t)b) & 15) PARS3_FAIL(PARS3_ERR_ARG, "vectors must be 16-byte aligned");
    k_dot<<<kDotGrid, 512, 0, st>>>((int32_t)n, a, b, part, out);
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
static int plan_product_(pars3_plan *pl, const double *x, double *y, bool acc, const double *w,
                         double *dot, bool strict, cudaStream_t st);
static int plan_product(pars3_plan *pl, const double *x, double *y, bool acc, const double *w,
                        double *dot, cudaStream_t st, bool strict = false) {
    if (pl->n > 0 && x == y) PARS3_FAIL(PARS3_ERR_ARG, "x and y must not alias");
    pl->prof_k = 0;
    mark(pl, st);
    const int rc = plan_product_(pl, x, y, acc, w, dot, strict, st);
    while (pl->prof && pl->prof_k < 4) mark(pl, st);  // (phases a form does not have: empty)
    return rc;
}

static int plan_product_(pars3_plan *pl, const double *x, double *y, bool acc, const double *w,
                         double *dot, bool strict, cudaStream_t st) {
    const bool grid = pl->grid_ok && !acc && pl->peers.nranks == 0 && pl->ntiles > 0;
    if (!pl->perm) {
        if (pl->direct) {
            int rc = launch_direct(pl, x, y, acc, st);
            if (rc || !dot) return rc;
            return launch_dot(pl->n, y, w, pl->part, dot, st);
        }
        if (grid) return launch_grid(pl, x, y, w, dot, dot && w == y, strict, st);
        int rc = launch_red(pl, x, y, acc, st);
        if (rc || !dot) return rc;
        return launch_dot(pl->n, y, w, pl->part, dot, st);
    }
    const int32_t n = (int32_t)pl->n;
    const int g = (int)std::min<int64_t>(148 * 4, (pl->n + 511) / 512);
    k_perm_in<<<g, 512, 0, st>>>(n, pl->iperm, x, pl->xs);
    LAUNCH_CHECK();
    // <y, y> = <ys, ys>: fused into the grid pass; another w goes through
    // the gather's epilogue
    const bool fused = grid && dot && w == y;
    int rc = grid ? launch_grid(pl, pl->xs, pl->ys, fused ? pl->ys : nullptr, fused ? dot : nullptr, fused,
                                strict, st)
                  : launch_red(pl, pl->xs, pl->ys, false, st);
    if (rc) return rc;
    const bool pdot = dot && !fused;
    if (acc)
        (pdot ? k_perm_out<true, true> : k_perm_out<true, false>)<<<g, 512, 0, st>>>(n, pl->perm, pl->ys, y, w, pl->part);
    else
        (pdot ? k_perm_out<false, true> : k_perm_out<false, false>)<<<g, 512, 0, st>>>(n, pl->perm, pl->ys, y, w, pl->part);
    LAUNCH_CHECK();
    if (pdot) {
        k_sum_parts<<<1, kThreads, 0, st>>>(g, pl->part, dot);
        LAUNCH_CHECK();
    }
    return PARS3_OK;
}

// the general entry: flags PARS3_PRODUCT_ACC (y += A x), PARS3_PRODUCT_STRICT
// (the grid scale from this x: a pure function of x), dot / w optional
extern "C" int pars3_plan_product(pars3_plan *pl, const double *x, double *y, const double *w, double *dot,
                                  int32_t flags, void *stream) {
    if (!pl || (pl->n > 0 && (!x || !y)) || (dot && pl->n > 0 && !w)) PARS3_FAIL(PARS3_ERR_ARG, "null argument");
    if ((flags & PARS3_PRODUCT_ACC) && dot) PARS3_FAIL(PARS3_ERR_ARG, "y += A x has no fused dot");
    return plan_product(pl, x, y, (flags & PARS3_PRODUCT_ACC) != 0, w, dot, (cudaStream_t)stream,
                        (flags & PARS3_PRODUCT_STRICT) != 0);
}

// out[i] = out[i] + (*a) p[i] + (*b) q[i]  (the unfused form of pars3_plan_product_axpy's epilogue)
__global__ void __launch_bounds__(512) k_axpy2(int32_t n, double *out, const double *__restrict__ p,
                                               const double *a, const double *__restrict__ q, const double *b) {
    const double ea = *a, eb = *b;
    const int32_t stride = gridDim.x * blockDim.x;
    for (int32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
        out[i] = fma(eb, q[i], fma(ea, p[i], out[i]));
}

// out = A x + (*a) p + (*b) q and, when dot is given, *dot = <out, out>: the
// product fused with the vector update that follows it in a Krylov step (MRS:
// u = A v - alpha v + gamma w).  a, b are DEVICE scalars, so the recurrence
// needs no host round trip.  Grid-form plans apply the update in the finish
// pass (no separate y is written or read back); the other forms run the
// product and one more pass.  out must not alias x, p or q.
extern "C" int pars3_plan_product_axpy(pars3_plan *pl, const double *x, double *out, const double *p,
                                       const double *a, const double *q, const double *b, double *dot,
                                       int32_t flags, void *stream) {
    if (!pl || !a || !b || (pl->n > 0 && (!x || !out || !p || !q))) PARS3_FAIL(PARS3_ERR_ARG, "null argument");
    if (flags & PARS3_PRODUCT_ACC) PARS3_FAIL(PARS3_ERR_ARG, "pars3_plan_product_axpy overwrites out");
    if (pl->n > 0 && (out == p || out == q)) PARS3_FAIL(PARS3_ERR_ARG, "out must not alias p or q");
    cudaStream_t st = (cudaStream_t)stream;
    const bool strict = (flags & PARS3_PRODUCT_STRICT) != 0;
    const bool fused = pl->grid_ok && pl->peers.nranks == 0 && pl->ntiles > 0 && !pl->perm && !pl->direct;
    if (fused) {
        pl->xbound_given = strict && (flags & PARS3_PRODUCT_XBOUND) != 0;
        pl->ep_p = p;
        pl->ep_q = q;
        pl->ep_a = a;
        pl->ep_b = b;
        const int rc = plan_product(pl, x, out, false, dot ? out : nullptr, dot, st, strict);
        pl->ep_p = pl->ep_q = pl->ep_a = pl->ep_b = nullptr;
        pl->xbound_given = false;
        return rc;
    }
    int rc = plan_product(pl, x, out, false, nullptr, nullptr, st, strict);
    if (rc || pl->n == 0) return rc;
    k_axpy2<<<kDotGrid, 512, 0, st>>>((int32_t)pl->n, out, p, a, q, b);
    LAUNCH_CHECK();
    if (dot) rc = launch_dot(pl->n, out, out, pl->part, dot, st);
    return rc;
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

// Phase times of `reps` products y = A x (and <y, y> when with_dot), CUDA
// events on `stream`: ms[0] the main kernel (tiles / full CSR; for a
// locality plan with its gather of x), ms[1] the next phase (k_finish / the
// span fix-up / the RED form's dot), ms[2] the rest (the gather of y, sums),
// ms[3] the whole product; averages per product.
extern "C" int pars3_plan_profile(pars3_plan *pl, const double *x, double *y, int32_t with_dot, int32_t reps,
                                  double *ms, void *stream) {
    if (!pl || !ms || reps < 1 || (pl->n > 0 && (!x || !y))) PARS3_FAIL(PARS3_ERR_ARG, "bad argument");
    cudaStream_t st = (cudaStream_t)stream;
    cudaEvent_t ev[4];
    for (int k = 0; k < 4; k++) CUDA_TRY(cudaEventCreate(&ev[k]));
    double *dot = nullptr;
    if (with_dot) CUDA_TRY(cudaMalloc((void **)&dot, sizeof(double)));
    double acc[4] = {0, 0, 0, 0};
    int rc = PARS3_OK;
    for (int r = 0; r < reps && rc == PARS3_OK; r++) {
        pl->prof = ev;
        rc = plan_product(pl, x, y, false, with_dot ? y : nullptr, dot, st);
        pl->prof = nullptr;
        if (rc) break;
        if (cudaEventSynchronize(ev[3]) != cudaSuccess) { rc = PARS3_ERR_CUDA; break; }
        float t[3];
        for (int k = 0; k < 3; k++) cudaEventElapsedTime(&t[k], ev[k], ev[k + 1]);
        acc[0] += t[0];
        acc[1] += t[1];
        acc[2] += t[2];
        acc[3] += t[0] + t[1] + t[2];
    }
    for (int k = 0; k < 4; k++) {
        ms[k] = acc[k] / reps;
        cudaEventDestroy(ev[k]);
    }
    if (dot) cudaFree(dot);
    if (rc) PARS3_FAIL(rc, "pars3_plan_profile: product failed");
    return PARS3_OK;
}

extern "C" int pars3_dot(int64_t n, const double *a, const double *b, double *out, void *stream) {
    if (n < 0 || n >= INT32_MAX || !out || (n > 0 && (!a || !b))) PARS3_FAIL(PARS3_ERR_ARG, "bad argument");
    cudaStream_t st = (cudaStream_t)stream;
    // stream-ordered scratch for the per-block shares (pool allocation)
    double *part = nullptr;
    CUDA_TRY(cudaMallocAsync((void **)&part, sizeof(double) * (kDotGrid + 1), st));
    CUDA_TRY(cudaMemsetAsync(part + kDotGrid, 0, sizeof(double), st));  // the arrival counter
    const int rc = launch_dot(n, a, b, part, out, st);
    CUDA_TRY(cudaFreeAsync(part, st));
    return rc;
}

// The device word a caller's kernel may fill with the bound of the next x
// (PARS3_PRODUCT_XBOUND): 0 = none, else (e + 1 + 2048) with |x_i| < 2^e for
// every finite x_i (e = max(biased exponent, 1) - 1022): k_xmax's encoding.
// *slot = NULL for plans without the grid form or whose x passes through an
// internal order first.
extern "C" int pars3_plan_xbound_slot(pars3_plan *pl, int32_t **slot) {
    if (!pl || !slot) PARS3_FAIL(PARS3_ERR_ARG, "null argument");
    const bool ok = pl->grid_ok && pl->peers.nranks == 0 && pl->ntiles > 0 && !pl->perm && !pl->direct;
    *slot = ok ? &pl->gs->xe_pre : nullptr;
    return PARS3_OK;
}

extern "C" int pars3_plan_status(pars3_plan *pl, int32_t *flags, void *stream) {
    if (!pl || !flags) PARS3_FAIL(PARS3_ERR_ARG, "null argument");
    *flags = 0;
    if (!pl->gs) return PARS3_OK;
    cudaStream_t st = (cudaStream_t)stream;
    GState g{};
    CUDA_TRY(cudaMemcpyAsync(&g, pl->gs, sizeof(g), cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaStreamSynchronize(st));
    if (g.redone != pl->seen_redone) *flags |= 1;
    if (g.fp64_tiles != pl->seen_fp64_tiles) *flags |= 2;
    pl->seen_redone = g.redone;
    pl->seen_fp64_tiles = g.fp64_tiles;
    return PARS3_OK;
}

extern "C" int pars3_plan_kernel_count(const pars3_plan *pl, int32_t with_dot, int32_t *count) {
    if (!pl || !count) PARS3_FAIL(PARS3_ERR_ARG, "null argument");
    const bool grid = pl->grid_ok && pl->peers.nranks == 0 && pl->ntiles > 0;
    int c = 0;
    if (pl->direct) {
        c = (pl->n > 0 ? 1 : 0) + (pl->nspan > 0 ? 1 : 0) + (with_dot && pl->n > 0 ? 1 : 0);
    } else if (pl->perm) {
        c = 2 + (pl->ntiles > 0 ? (grid ? 3 : 1) : 0) + (pl->nfar > 0 ? 1 : 0);
    } else if (grid) {
        c = 3;  // k_tiles, k_conv, k_finish (exits at once unless the product was flagged)
    } else {
        c = (pl->ntiles > 0 ? 1 : 0) + (pl->nfar > 0 ? 1 : 0) + (with_dot && pl->n > 0 ? 1 : 0);
    }
    *count = c;
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
    stats[14] = pl->grid_ok;
    stats[15] = pl->hgrid;
    stats[16] = pl->cmax;
    stats[17] = pl->ev_g;
    stats[18] = pl->built_on_device;
    stats[19] = pl->nfar;
    return PARS3_OK;
}

// Inspection / tests: the tile plan of a split as host arrays, built by the
// host builder (use_device = 0) or by the device builder (1: PARS3_ERR_ARG
// when it does not support the plan), with the option set pars3_plan_create
// derives for `words` accumulator words (2, 3 or 0 = fp64).  sizes[9] =
// {tiles, windows, slices, record bytes, stored entries, padded slots, max
// terms, list tiles, list columns}; call with tiles == NULL for the sizes,
// then with arrays (tiles: 48 B each, wins: 16 B each, slice_off: slices + 1).
extern "C" int pars3_tile_plan_arrays(const pars3_split_view *s, const pars3_plan_options *opt, int32_t words,
                                      int32_t use_device, int64_t *sizes, void *tiles, void *wins,
                                      int64_t *slice_off, uint8_t *rec, int32_t *ucol) {
    if (!s || !sizes || (words != 0 && words != 2 && words != 3)) PARS3_FAIL(PARS3_ERR_ARG, "bad argument");
    PlanOptions o;
    if (opt) {
        if (opt->tile_rows > 0) o.tile_rows = opt->tile_rows;
        if (opt->local_slots > 0) o.local_slots = opt->local_slots;
        if (opt->seg_max > 0) o.seg_max = opt->seg_max;
        if (opt->gap >= 0) o.gap = opt->gap;
    }
    if (o.seg_max > 8) o.seg_max = 8;
    o.max_segments = std::min(o.max_segments, 32 * kMaxTileSlices);
    o.terms_cap = words == 2 ? kTerms2 : 0;
    o.local_slots = std::min(o.local_slots, words == 3 ? kLocalFixed : kLocalExact);
    o.sink = (uint16_t)(words == 3 ? Layout<3>::kSink : Layout<0>::kSink);
    HostPlan hp;
    pars3::DevicePlan dp;
    if (use_device) {
        bool ok = false;
        const int rc = pars3::build_tile_plan_device(s->n, s->mid_ptr, s->mid_col, s->mid_val, s->outer_count,
                                                     s->outer_row, s->outer_col, s->outer_val, o, hp, dp, ok);
        if (rc) return rc;
        if (!ok) PARS3_FAIL(PARS3_ERR_ARG, "the device builder does not support this plan");
    } else {
        const int rc = pars3::build_tile_plan(s->n, s->mid_ptr, s->mid_col, s->mid_val, s->outer_count,
                                              s->outer_row, s->outer_col, s->outer_val, o, hp);
        if (rc) return rc;
    }
    const int64_t ns = use_device ? dp.nslices : (int64_t)hp.slice_off.size() - 1;
    const int64_t nv = use_device ? dp.rec_bytes : (int64_t)hp.rec.size();
    sizes[0] = (int64_t)hp.tiles.size();
    sizes[1] = (int64_t)hp.wins.size();
    sizes[2] = ns;
    sizes[3] = nv;
    sizes[4] = hp.nnz;
    sizes[5] = hp.slots;
    sizes[6] = hp.max_terms;
    sizes[7] = hp.list_tiles;
    sizes[8] = (int64_t)hp.ucol.size();
    int rc = PARS3_OK;
    if (tiles) {
        std::memcpy(tiles, hp.tiles.data(), sizeof(TileMeta) * hp.tiles.size());
        std::memcpy(wins, hp.wins.data(), sizeof(Window) * hp.wins.size());
        if (ucol) std::memcpy(ucol, hp.ucol.data(), sizeof(int32_t) * hp.ucol.size());
        if (use_device) {
            if (cudaMemcpy(slice_off, dp.slice_off, sizeof(int64_t) * (ns + 1), cudaMemcpyDeviceToHost) != cudaSuccess ||
                cudaMemcpy(rec, dp.rec, (size_t)nv, cudaMemcpyDeviceToHost) != cudaSuccess)
                rc = PARS3_ERR_CUDA;
        } else {
            std::memcpy(slice_off, hp.slice_off.data(), sizeof(int64_t) * (ns + 1));
            std::memcpy(rec, hp.rec.data(), (size_t)nv);
        }
    }
    dp.release();
    if (rc) PARS3_FAIL(rc, "pars3_tile_plan_arrays: download failed");
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
