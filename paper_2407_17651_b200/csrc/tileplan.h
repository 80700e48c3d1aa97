// Tile plan: the device layout of the windowed PARS3 kernel.
//
// The matrix rows are cut into tiles.  A tile OWNS a contiguous row range
// [r0, r1) (possibly empty for a "helper" tile carrying a chunk of one very
// long row) and holds every stored entry of a set of row segments.  All
// columns a tile touches -- plus its own rows -- are covered by a few dense
// column WINDOWS; window slot i of the tile's local index space holds x[c]
// and the accumulator for y[c] in shared memory.  Entries are stored in
// SELL-32 slices (32 row segments x nslots, slot-major) as fp64 value +
// uint16 local column index; padding lanes carry the 0xFFFF sentinel.
#pragma once
#include <cstdint>
#include <vector>

namespace pars3 {

constexpr uint16_t kNoSlot = 0xFFFF;

struct PlanOptions {
    int32_t tile_rows = 2048;   // rows per tile before splitting
    int32_t local_slots = 6144; // shared-memory window slots per tile (x + acc = 16 B each)
    int32_t seg_max = 64;       // max entries per row segment (longer rows are split)
    int32_t gap = 8;            // merge column runs separated by <= gap unused slots
};

struct TileMeta {     // 8 x int32
    int32_t r0, r1;   // owned rows
    int32_t w0, w1;   // window range
    int32_t s0, s1;   // slice range
    int32_t local;    // local index space size
    int32_t own_loff; // local index of row r0 (valid when r1 > r0)
};

struct Window {       // 8 x int32
    int32_t lo, len, loff;
    int32_t t_lo, t_hi;  // owner tiles of rows [lo, lo+len) (inclusive range)
    int32_t pad0, pad1, pad2;
};

struct HostPlan {
    int64_t n = 0;
    std::vector<TileMeta> tiles;
    std::vector<Window> wins;
    std::vector<int32_t> slice_base;    // first entry (multiple of 32) of each slice
    std::vector<int32_t> slice_nslots;
    std::vector<uint16_t> slice_rowl;   // 32 per slice: local index of each lane's row
    std::vector<double> val;            // slot-major, 32 lanes per slot
    std::vector<uint16_t> lidx;
    int64_t nnz = 0;                    // stored entries (without padding)
    int32_t max_local = 0;
};

// Build from host split arrays (BandSplit layout, split.py:58-113).
int build_tile_plan(int64_t n, const int64_t *mid_ptr, const int32_t *mid_col,
                    const double *mid_val, int64_t outer_count, const int32_t *outer_row,
                    const int32_t *outer_col, const double *outer_val, const PlanOptions &opt,
                    HostPlan &out);

}  // namespace pars3
