// Host builder of the windowed tile plan (tileplan.h).  Parallel over row
// ranges; the output is deterministic (independent of the thread count).
#include "tileplan.h"

#include <omp.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <new>

#include "common.h"

namespace pars3 {
namespace {

struct Rows {
    int64_t n;
    const int64_t *optr;  // outer row pointer (built here)
    const int32_t *ocol;
    const double *oval;
    const int64_t *mptr;
    const int32_t *mcol;
    const double *mval;
    int64_t count(int64_t r) const { return (optr[r + 1] - optr[r]) + (mptr[r + 1] - mptr[r]); }
    // k-th stored entry of row r (outer entries precede middle ones: both
    // bands keep ascending columns and every outer column < every middle one)
    int32_t col(int64_t r, int64_t k) const {
        int64_t no = optr[r + 1] - optr[r];
        return k < no ? ocol[optr[r] + k] : mcol[mptr[r] + (k - no)];
    }
    double val(int64_t r, int64_t k) const {
        int64_t no = optr[r + 1] - optr[r];
        return k < no ? oval[optr[r] + k] : mval[mptr[r] + (k - no)];
    }
};

struct Draft {
    int32_t r0, r1;          // owned rows
    int32_t hub = -1;        // row of a chunked long row (owner or helper), else -1
    int64_t k0 = 0, k1 = 0;  // entry chunk of the hub row
    std::vector<int32_t> wlo, wlen;
    int32_t local = 0;
};

struct Built {               // one draft materialised
    std::vector<int32_t> wlo, wlen, wloff;
    bool list = false;           // explicit column list instead of windows
    std::vector<int32_t> ucol;
    std::vector<int64_t> slice_off;  // relative, bytes
    std::vector<uint8_t> rec;
    int32_t r0, r1, local, max_nslots = 0, max_terms = 0;
    int64_t nnz, slots;
    double vmax = 0.0;
};

// Merge sorted unique columns into dense windows (runs separated by <= gap
// unused slots).  With `align` the windows are widened to even bounds (the
// kernel moves them with 16-byte TMA bulk copies), never past column n.
void make_windows(std::vector<int32_t> &cols, int32_t gap, bool align, int64_t n, Draft &d) {
    std::sort(cols.begin(), cols.end());
    cols.erase(std::unique(cols.begin(), cols.end()), cols.end());
    d.wlo.clear();
    d.wlen.clear();
    d.local = 0;
    size_t i = 0;
    while (i < cols.size()) {
        int32_t lo = cols[i], hi = cols[i] + 1;
        size_t j = i + 1;
        while (j < cols.size() && cols[j] - hi <= gap) hi = cols[j++] + 1;
        if (align) {
            lo &= ~1;
            if ((hi & 1) && hi < n) hi++;
            if (!d.wlo.empty() && lo <= d.wlo.back() + d.wlen.back()) {  // touches the previous
                const int32_t plo = d.wlo.back();
                d.local -= d.wlen.back();
                d.wlen.back() = hi - plo;
                d.local += hi - plo;
                i = j;
                continue;
            }
        }
        d.wlo.push_back(lo);
        d.wlen.push_back(hi - lo);
        d.local += hi - lo;
        i = j;
    }
}

// split windows at the cut points (rank boundaries in peer mode): a window
// then reads x from, and delivers to, one owner
void cut_windows(const std::vector<int32_t> &cuts, Draft &d) {
    if (cuts.empty()) return;
    std::vector<int32_t> lo2, len2;
    for (size_t w = 0; w < d.wlo.size(); w++) {
        int32_t lo = d.wlo[w];
        const int32_t hi = lo + d.wlen[w];
        auto it = std::upper_bound(cuts.begin(), cuts.end(), lo);
        for (; it != cuts.end() && *it < hi; ++it) {
            lo2.push_back(lo);
            len2.push_back(*it - lo);
            lo = *it;
        }
        lo2.push_back(lo);
        len2.push_back(hi - lo);
    }
    d.wlo.swap(lo2);
    d.wlen.swap(len2);
}

// Shared-memory bank conflicts of one slot position across the 32 lanes:
// the mirror terms go to 32-bit words at lidx (banks lidx mod 32), the x
// reads are 64-bit (two half-warp wavefronts, lidx mod 16).
int slot_conflicts(const uint16_t *lx, uint16_t sink) {
    int b32[32] = {0}, b16[16] = {0}, c = 0;
    for (int l = 0; l < 32; l++) {
        if (lx[l] == sink) continue;
        c += (b32[lx[l] & 31]++ > 0) + (b16[lx[l] & 15]++ > 1);
    }
    return c;
}

// The entries of a row segment may sit in any of its slot positions (the
// row sum and the exact fixed-point mirror sums do not depend on the order).
// Unstructured tiles put random columns side by side, so the 32 lanes of a
// slot position often share banks (c3: 25 M of 45 M shared wavefronts were
// conflicts).  Greedy: fill positions in turn, each lane taking the
// remaining entry of its segment that adds the fewest conflicts.  Kept only
// when it beats the stored (ascending-column) order; structured slices
// (stencils: consecutive rows, consecutive columns) are conflict-free as
// stored and stay as they are.
void spread_banks(double *val, uint16_t *lidx, int32_t nslots, int lanes, uint16_t sink) {
    if (nslots < 2 || nslots > 8 || lanes < 2) return;
    int before = 0;
    for (int32_t k = 0; k < nslots; k++) before += slot_conflicts(lidx + (size_t)k * 32, sink);
    if (before == 0) return;
    std::vector<double> v2((size_t)nslots * 32);
    std::vector<uint16_t> x2((size_t)nslots * 32, sink);
    uint8_t used[32][8] = {{0}};  // seg_max <= 8
    int after = 0;
    for (int32_t k = 0; k < nslots; k++) {
        int b32[32] = {0}, b16[16] = {0};
        for (int l = 0; l < lanes; l++) {
            int best = -1, bc = 1 << 30;
            for (int32_t q = 0; q < nslots; q++) {
                const uint16_t c = lidx[(size_t)q * 32 + l];
                if (used[l][q] || c == sink) continue;
                const int cost = (b32[c & 31] > 0) + (b16[c & 15] > 1);
                if (cost < bc) {
                    bc = cost;
                    best = q;
                }
            }
            if (best < 0) continue;  // the segment is exhausted: padding
            used[l][best] = 1;
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

void draft_range(const Rows &R, int32_t a, int32_t b, const PlanOptions &o,
                 std::vector<Draft> &out, std::vector<int32_t> &scratch) {
    scratch.clear();
    int64_t segments = 0;
    int64_t entries = 0;
    for (int32_t r = a; r < b; r++) {
        int64_t c = R.count(r);
        entries += c;
        if (c > 0 || !o.skip_empty) scratch.push_back(r);
        segments += (c + o.seg_max - 1) / o.seg_max;
        for (int64_t k = 0; k < c; k++) scratch.push_back(R.col(r, k));
    }
    if (segments > o.max_segments && b - a > 1) {
        int32_t mid = a + (b - a) / 2;
        draft_range(R, a, mid, o, out, scratch);
        draft_range(R, mid, b, o, out, scratch);
        return;
    }
    if (entries == 0 && o.skip_empty) return;  // nothing to deliver
    bool chunk_row = false;  // one row whose own slot alone exceeds the terms cap
    if (o.terms_cap > 0 && b - a > o.terms_min_rows / 2) {
        // terms of the busiest slot: references of one column in this row
        // range plus the segments of its own row (bounded by the longest
        // row's).  Halve the range while it exceeds the cap, so the plan can
        // keep the two-word accumulator; a single row is cut into chunks.
        std::vector<int32_t> cols(scratch);
        std::sort(cols.begin(), cols.end());
        int32_t run = 0, best = 0;
        for (size_t i = 0; i < cols.size(); i++) {
            run = (i > 0 && cols[i] == cols[i - 1]) ? run + 1 : 1;
            best = std::max(best, run);
        }
        int64_t segs = 0;
        for (int32_t r = a; r < b; r++) segs = std::max(segs, (R.count(r) + o.seg_max - 1) / o.seg_max);
        if (best + segs > o.terms_cap) {
            if (b - a > std::max(1, o.terms_min_rows)) {
                const int32_t mid = b - a > 64 ? a + (((b - a) / 2 + 31) & ~31) : a + (b - a) / 2;
                draft_range(R, a, mid, o, out, scratch);
                draft_range(R, mid, b, o, out, scratch);
                return;
            }
            chunk_row = b - a == 1;
        }
    }
    Draft d;
    d.r0 = a;
    d.r1 = b;
    make_windows(scratch, o.gap, true, R.n, d);
    cut_windows(o.cuts, d);
    if ((int)d.wlo.size() > kMaxWindows) {
        // Too fragmented for gap-merged windows.  When the whole column span
        // [smallest column, b) fits the local space, one dense window over it
        // keeps the tile in window mode (TMA copies of x, coalesced
        // deliveries; a band's sparse fringe, the first rows of a stencil);
        // when halving the range would make it fit, halve instead of
        // carrying a column list.  (make_windows left scratch sorted.)
        Draft one;
        one.r0 = a;
        one.r1 = b;
        int32_t lo = scratch.empty() ? a : (scratch[0] & ~1), hi = b;
        if ((hi & 1) && hi < R.n) hi++;
        one.wlo.push_back(lo);
        one.wlen.push_back(hi - lo);
        one.local = hi - lo;
        cut_windows(o.cuts, one);
        if (one.local <= o.local_slots && (int)one.wlo.size() <= kMaxWindows) {
            d = std::move(one);
        } else if (b - a > 64 && one.local - (b - a) / 2 <= o.local_slots) {
            const int32_t mid = a + (((b - a) / 2 + 31) & ~31);
            draft_range(R, a, mid, o, out, scratch);
            draft_range(R, mid, b, o, out, scratch);
            return;
        } else {
            // an explicit column list: do not pay for gap or alignment slots
            // (the rebuilt windows are cut again: a tile that ends up with <=
            // kMaxWindows of them stays in window mode, and no window may
            // straddle a rank boundary)
            make_windows(scratch, 0, false, R.n, d);
            cut_windows(o.cuts, d);
        }
    }
    if (d.local <= o.local_slots && !chunk_row) {
        out.push_back(std::move(d));
        return;
    }
    if (b - a > 1) {
        int32_t mid = a + (b - a) / 2;
        if (b - a > 64) mid = a + (((b - a) / 2 + 31) & ~31);
        draft_range(R, a, mid, o, out, scratch);
        draft_range(R, mid, b, o, out, scratch);
        return;
    }
    // one row wider than the local space: chunk its entries; the first
    // chunk's tile owns the row, the others are helpers (own range empty)
    const int64_t cnt = R.count(a);
    // (with a terms cap, the row's own slot takes one term per segment)
    const int64_t chunk = o.terms_cap > 2 ? std::min<int64_t>(o.local_slots - 2,
                                                              (int64_t)(o.terms_cap - 2) * o.seg_max)
                                          : o.local_slots - 2;
    for (int64_t k0 = 0; k0 < cnt; k0 += chunk) {
        Draft h;
        h.r0 = a;
        h.r1 = k0 == 0 ? a + 1 : a;
        h.hub = a;
        h.k0 = k0;
        h.k1 = std::min(cnt, k0 + chunk);
        scratch.clear();
        scratch.push_back(a);
        for (int64_t k = h.k0; k < h.k1; k++) scratch.push_back(R.col(a, k));
        make_windows(scratch, 0, false, R.n, h);
        out.push_back(std::move(h));
    }
}

inline int32_t local_of(const Draft &d, const std::vector<int32_t> &loff, int32_t c) {
    // windows are sorted by lo; find the last with lo <= c
    auto it = std::upper_bound(d.wlo.begin(), d.wlo.end(), c);
    size_t w = (size_t)(it - d.wlo.begin()) - 1;
    return loff[w] + (c - d.wlo[w]);
}

void materialise(const Rows &R, const Draft &d, const PlanOptions &o, Built &b) {
    b.wlo = d.wlo;
    b.wlen = d.wlen;
    b.wloff.resize(d.wlo.size());
    int32_t acc = 0;
    for (size_t w = 0; w < d.wlo.size(); w++) {
        b.wloff[w] = acc;
        acc += d.wlen[w];
    }
    b.r0 = d.r0;
    b.r1 = d.r1;
    b.local = d.local;
    b.list = (int)d.wlo.size() > kMaxWindows || d.hub >= 0;
    if (b.list) {
        b.ucol.reserve(d.local);
        for (size_t w = 0; w < d.wlo.size(); w++)
            for (int32_t i = 0; i < d.wlen[w]; i++) b.ucol.push_back(d.wlo[w] + i);
    }
    // row segments (row, k begin, k end)
    struct Seg {
        int32_t row;
        int64_t kb, ke;
    };
    std::vector<Seg> segs;
    auto add_row = [&](int32_t r, int64_t kb, int64_t ke) {
        for (int64_t k = kb; k < ke; k += o.seg_max) segs.push_back({r, k, std::min(ke, k + o.seg_max)});
    };
    if (d.hub >= 0) {
        add_row(d.hub, d.k0, d.k1);
    } else {
        for (int32_t r = d.r0; r < d.r1; r++) add_row(r, 0, R.count(r));
    }
    std::stable_sort(segs.begin(), segs.end(),
                     [](const Seg &x, const Seg &y) { return (x.ke - x.kb) > (y.ke - y.kb); });
    b.nnz = 0;
    b.slots = 0;
    // accumulator terms per local slot: one per mirror, one per row segment
    std::vector<int32_t> terms((size_t)d.local, 0);
    for (size_t s0 = 0; s0 < segs.size(); s0 += 32) {
        size_t s1 = std::min(segs.size(), s0 + 32);
        const int32_t nslots = (int32_t)(segs[s0].ke - segs[s0].kb);
        b.max_nslots = std::max(b.max_nslots, nslots);
        const size_t off = b.rec.size();
        b.slice_off.push_back((int64_t)off);
        b.rec.resize(off + 64 + (size_t)nslots * 320, 0);
        uint16_t *rowl = reinterpret_cast<uint16_t *>(&b.rec[off]);
        double *val = reinterpret_cast<double *>(&b.rec[off + 64]);
        uint16_t *lidx = reinterpret_cast<uint16_t *>(&b.rec[off + 64 + (size_t)nslots * 256]);
        for (size_t l = 0; l < 32; l++) {
            rowl[l] = s0 + l < s1 ? (uint16_t)local_of(d, b.wloff, segs[s0 + l].row) : o.sink;
            if (s0 + l < s1) terms[rowl[l]]++;
        }
        for (int64_t q = 0; q < (int64_t)nslots * 32; q++) {
            val[q] = 0.0;
            lidx[q] = o.sink;
        }
        for (size_t l = 0; l < s1 - s0; l++) {
            const Seg &sg = segs[s0 + l];
            for (int64_t k = sg.kb; k < sg.ke; k++) {
                const size_t pos = (size_t)(k - sg.kb) * 32 + l;
                val[pos] = R.val(sg.row, k);
                b.vmax = std::max(b.vmax, std::fabs(val[pos]));
                lidx[pos] = (uint16_t)local_of(d, b.wloff, R.col(sg.row, k));
                terms[lidx[pos]]++;
                b.nnz++;
            }
        }
        spread_banks(val, lidx, nslots, (int)(s1 - s0), o.sink);
        b.slots += (int64_t)nslots * 32;
    }
    for (int32_t c : terms) b.max_terms = std::max(b.max_terms, c);
}

}  // namespace

int build_tile_plan(int64_t n, const int64_t *mid_ptr, const int32_t *mid_col,
                    const double *mid_val, int64_t outer_count, const int32_t *outer_row,
                    const int32_t *outer_col, const double *outer_val, const PlanOptions &o,
                    HostPlan &P) {
    if (o.local_slots < 64 || o.local_slots > 65535 || o.tile_rows < 1 || o.seg_max < 1 ||
        (o.sink != kNoSlot && o.sink < o.local_slots))
        PARS3_FAIL(PARS3_ERR_ARG, "bad plan options");
    try {
        std::vector<int64_t> optr(n + 1, 0);
        for (int64_t e = 0; e < outer_count; e++) {
            int32_t r = outer_row[e];
            if (r < 0 || r >= n) PARS3_FAIL(PARS3_ERR_STRUCT, "outer row %d out of range", r);
            optr[r + 1]++;
        }
        for (int64_t r = 0; r < n; r++) optr[r + 1] += optr[r];
        Rows R{n, optr.data(), outer_col, outer_val, mid_ptr, mid_col, mid_val};

        const int64_t nranges = (n + o.tile_rows - 1) / o.tile_rows;
        std::vector<std::vector<Draft>> drafts(nranges);
#pragma omp parallel
        {
            std::vector<int32_t> scratch;
#pragma omp for schedule(dynamic, 4)
            for (int64_t q = 0; q < nranges; q++) {
                if (o.sample_stride > 1 && q % o.sample_stride != 0) continue;
                int32_t a = (int32_t)(q * o.tile_rows);
                int32_t b = (int32_t)std::min<int64_t>(n, (q + 1) * (int64_t)o.tile_rows);
                draft_range(R, a, b, o, drafts[q], scratch);
            }
        }
        std::vector<const Draft *> flat;
        for (auto &v : drafts)
            for (auto &d : v) flat.push_back(&d);
        const int64_t nt = (int64_t)flat.size();
        std::vector<Built> built(nt);
#pragma omp parallel for schedule(dynamic, 4)
        for (int64_t t = 0; t < nt; t++) materialise(R, *flat[t], o, built[t]);
        if (!o.cuts.empty()) {  // peer mode: a window's x and deliveries belong to one rank
            bool straddle = false;
#pragma omp parallel for reduction(|| : straddle)
            for (int64_t t = 0; t < nt; t++) {
                const Built &b = built[t];
                if (b.list) continue;
                for (size_t w = 0; w < b.wlo.size(); w++) {
                    auto it = std::upper_bound(o.cuts.begin(), o.cuts.end(), b.wlo[w]);
                    straddle = straddle || (it != o.cuts.end() && *it < b.wlo[w] + b.wlen[w]);
                }
            }
            if (straddle) PARS3_FAIL(PARS3_ERR_STRUCT, "tile plan: a window straddles a block boundary");
        }

        P = HostPlan();
        P.n = n;
        P.tiles.resize(nt);
        int64_t nw = 0, ns = 0, nv = 0, nu = 0;
        for (auto &b : built) {
            nu += (int64_t)b.ucol.size();
            if (!b.list) nw += (int64_t)b.wlo.size();
            ns += (int64_t)b.slice_off.size();
            nv += (int64_t)b.rec.size();
        }
        P.wins.resize(nw);
        P.ucol.resize(nu);
        P.slice_off.resize(ns + 1);
        P.rec.resize(nv);
        std::vector<int64_t> w_off(nt + 1, 0), s_off(nt + 1, 0), v_off(nt + 1, 0), u_off(nt + 1, 0);
        for (int64_t t = 0; t < nt; t++) {
            w_off[t + 1] = w_off[t] + (built[t].list ? 0 : (int64_t)built[t].wlo.size());
            u_off[t + 1] = u_off[t] + (int64_t)built[t].ucol.size();
            P.list_tiles += built[t].list ? 1 : 0;
            s_off[t + 1] = s_off[t] + (int64_t)built[t].slice_off.size();
            v_off[t + 1] = v_off[t] + (int64_t)built[t].rec.size();
        }
        int64_t nnz_total = 0, slots_total = 0;
#pragma omp parallel for schedule(dynamic, 16) reduction(+ : nnz_total, slots_total)
        for (int64_t t = 0; t < nt; t++) {
            Built &b = built[t];
            TileMeta &m = P.tiles[t];
            m.r0 = b.r0;
            m.r1 = b.r1;
            m.w0 = (int32_t)w_off[t];
            m.w1 = (int32_t)w_off[t + 1];
            m.s0 = (int32_t)s_off[t];
            m.s1 = (int32_t)s_off[t + 1];
            m.local = b.local;
            m.pad0 = m.pad1 = m.pad2 = 0;
            m.u0 = b.list ? (int32_t)u_off[t] : -1;
            {
                int e = -1074;
                if (b.vmax > 0.0) std::frexp(b.vmax, &e);  // vmax < 2^e
                m.ev = e;
            }
            if (b.list) std::memcpy(&P.ucol[u_off[t]], b.ucol.data(), b.ucol.size() * sizeof(int32_t));
            for (size_t w = 0; !b.list && w < b.wlo.size(); w++) {
                Window &W = P.wins[w_off[t] + w];
                W.lo = b.wlo[w];
                W.len = b.wlen[w];
                W.loff = b.wloff[w];
                W.pad0 = 0;
            }
            for (size_t s = 0; s < b.slice_off.size(); s++)
                P.slice_off[s_off[t] + s] = (v_off[t] + b.slice_off[s]) / 16;
            std::memcpy(&P.rec[v_off[t]], b.rec.data(), b.rec.size());
            nnz_total += b.nnz;
            slots_total += b.slots;
            std::vector<int32_t>().swap(b.wlo);
            std::vector<uint8_t>().swap(b.rec);
        }
        P.nnz = nnz_total;
        P.slots = slots_total;
        P.slice_off[ns] = nv / 16;
        for (auto &m : P.tiles) P.max_local = std::max(P.max_local, m.local);
        for (auto &b : built) {
            P.max_nslots = std::max(P.max_nslots, b.max_nslots);
            P.max_terms = std::max(P.max_terms, b.max_terms);
        }
    } catch (const std::bad_alloc &) {
        PARS3_FAIL(PARS3_ERR_NOMEM, "tile plan: out of host memory");
    }
    return PARS3_OK;
}

}  // namespace pars3
