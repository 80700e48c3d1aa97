// Host builder of the windowed tile plan (tileplan.h).  Parallel over row
// ranges; the output is deterministic (independent of the thread count).
#include "tileplan.h"

#include <omp.h>

#include <algorithm>
#include <cstring>
#include <new>

#include "common.h"

namespace pars3 {
namespace {

struct Rows {
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
    std::vector<int32_t> slice_base, slice_nslots;
    std::vector<uint16_t> slice_rowl;
    std::vector<double> val;
    std::vector<uint16_t> lidx;
    int32_t r0, r1, local, own_loff;
    int64_t nnz;
};

void make_windows(std::vector<int32_t> &cols, int32_t gap, Draft &d) {
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
        d.wlo.push_back(lo);
        d.wlen.push_back(hi - lo);
        d.local += hi - lo;
        i = j;
    }
}

void draft_range(const Rows &R, int32_t a, int32_t b, const PlanOptions &o,
                 std::vector<Draft> &out, std::vector<int32_t> &scratch) {
    scratch.clear();
    for (int32_t r = a; r < b; r++) {
        scratch.push_back(r);
        int64_t c = R.count(r);
        for (int64_t k = 0; k < c; k++) scratch.push_back(R.col(r, k));
    }
    Draft d;
    d.r0 = a;
    d.r1 = b;
    make_windows(scratch, o.gap, d);
    if (d.local <= o.local_slots) {
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
    const int64_t chunk = o.local_slots - 2;
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
        make_windows(scratch, 0, h);
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
    b.own_loff = local_of(d, b.wloff, d.r0);
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
    int64_t base = 0;
    for (size_t s0 = 0; s0 < segs.size(); s0 += 32) {
        size_t s1 = std::min(segs.size(), s0 + 32);
        int32_t nslots = (int32_t)(segs[s0].ke - segs[s0].kb);
        b.slice_base.push_back((int32_t)base);
        b.slice_nslots.push_back(nslots);
        for (size_t l = 0; l < 32; l++)
            b.slice_rowl.push_back(s0 + l < s1 ? (uint16_t)local_of(d, b.wloff, segs[s0 + l].row)
                                               : kNoSlot);
        size_t off = b.val.size();
        b.val.resize(off + (size_t)nslots * 32, 0.0);
        b.lidx.resize(off + (size_t)nslots * 32, kNoSlot);
        for (size_t l = 0; l < s1 - s0; l++) {
            const Seg &sg = segs[s0 + l];
            for (int64_t k = sg.kb; k < sg.ke; k++) {
                size_t pos = off + (size_t)(k - sg.kb) * 32 + l;
                b.val[pos] = R.val(sg.row, k);
                b.lidx[pos] = (uint16_t)local_of(d, b.wloff, R.col(sg.row, k));
                b.nnz++;
            }
        }
        base += (int64_t)nslots * 32;
    }
}

}  // namespace

int build_tile_plan(int64_t n, const int64_t *mid_ptr, const int32_t *mid_col,
                    const double *mid_val, int64_t outer_count, const int32_t *outer_row,
                    const int32_t *outer_col, const double *outer_val, const PlanOptions &o,
                    HostPlan &P) {
    if (o.local_slots < 64 || o.local_slots > 65535 || o.tile_rows < 1 || o.seg_max < 1)
        PARS3_FAIL(PARS3_ERR_ARG, "bad plan options");
    try {
        std::vector<int64_t> optr(n + 1, 0);
        for (int64_t e = 0; e < outer_count; e++) {
            int32_t r = outer_row[e];
            if (r < 0 || r >= n) PARS3_FAIL(PARS3_ERR_STRUCT, "outer row %d out of range", r);
            optr[r + 1]++;
        }
        for (int64_t r = 0; r < n; r++) optr[r + 1] += optr[r];
        Rows R{optr.data(), outer_col, outer_val, mid_ptr, mid_col, mid_val};

        const int64_t nranges = (n + o.tile_rows - 1) / o.tile_rows;
        std::vector<std::vector<Draft>> drafts(nranges);
#pragma omp parallel
        {
            std::vector<int32_t> scratch;
#pragma omp for schedule(dynamic, 4)
            for (int64_t q = 0; q < nranges; q++) {
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

        // owner tile of each row: tiles with r1 > r0, ascending r0
        std::vector<int32_t> own_r0, own_t;
        for (int64_t t = 0; t < nt; t++)
            if (built[t].r1 > built[t].r0) {
                own_r0.push_back(built[t].r0);
                own_t.push_back((int32_t)t);
            }
        auto owner_of = [&](int32_t r) {
            auto it = std::upper_bound(own_r0.begin(), own_r0.end(), r);
            return own_t[(size_t)(it - own_r0.begin()) - 1];
        };

        P = HostPlan();
        P.n = n;
        P.tiles.resize(nt);
        int64_t nw = 0, ns = 0, nv = 0;
        for (auto &b : built) {
            nw += (int64_t)b.wlo.size();
            ns += (int64_t)b.slice_base.size();
            nv += (int64_t)b.val.size();
        }
        if (nv >= INT32_MAX) PARS3_FAIL(PARS3_ERR_ARG, "plan too large for int32 slot offsets");
        P.wins.resize(nw);
        P.slice_base.resize(ns);
        P.slice_nslots.resize(ns);
        P.slice_rowl.resize(ns * 32);
        P.val.resize(nv);
        P.lidx.resize(nv);
        std::vector<int64_t> w_off(nt + 1, 0), s_off(nt + 1, 0), v_off(nt + 1, 0);
        for (int64_t t = 0; t < nt; t++) {
            w_off[t + 1] = w_off[t] + (int64_t)built[t].wlo.size();
            s_off[t + 1] = s_off[t] + (int64_t)built[t].slice_base.size();
            v_off[t + 1] = v_off[t] + (int64_t)built[t].val.size();
        }
        int64_t nnz_total = 0;
#pragma omp parallel for schedule(dynamic, 16) reduction(+ : nnz_total)
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
            m.own_loff = b.own_loff;
            for (size_t w = 0; w < b.wlo.size(); w++) {
                Window &W = P.wins[w_off[t] + w];
                W.lo = b.wlo[w];
                W.len = b.wlen[w];
                W.loff = b.wloff[w];
                W.t_lo = owner_of(b.wlo[w]);
                W.t_hi = owner_of(b.wlo[w] + b.wlen[w] - 1);
                W.pad0 = W.pad1 = W.pad2 = 0;
            }
            for (size_t s = 0; s < b.slice_base.size(); s++) {
                P.slice_base[s_off[t] + s] = (int32_t)(v_off[t] + b.slice_base[s]);
                P.slice_nslots[s_off[t] + s] = b.slice_nslots[s];
            }
            std::memcpy(&P.slice_rowl[s_off[t] * 32], b.slice_rowl.data(),
                        b.slice_rowl.size() * sizeof(uint16_t));
            std::memcpy(&P.val[v_off[t]], b.val.data(), b.val.size() * sizeof(double));
            std::memcpy(&P.lidx[v_off[t]], b.lidx.data(), b.lidx.size() * sizeof(uint16_t));
            nnz_total += b.nnz;
            std::vector<int32_t>().swap(b.wlo);
            std::vector<double>().swap(b.val);
            std::vector<uint16_t>().swap(b.lidx);
        }
        P.nnz = nnz_total;
        for (auto &m : P.tiles) P.max_local = std::max(P.max_local, m.local);
    } catch (const std::bad_alloc &) {
        PARS3_FAIL(PARS3_ERR_NOMEM, "tile plan: out of host memory");
    }
    return PARS3_OK;
}

}  // namespace pars3
