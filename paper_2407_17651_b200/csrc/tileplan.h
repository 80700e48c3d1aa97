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
// Each slice is one contiguous RECORD, the unit the kernel's TMA producer
// streams into shared memory with one bulk copy:
//     [rowl: 32 x u16][val: nslots x 32 x f64][lidx: nslots x 32 x u16]
// (64 + 320 * nslots bytes, 16-byte aligned).
#pragma once
#include <cstdint>
#include <vector>

namespace pars3 {

constexpr uint16_t kNoSlot = 0xFFFF;

struct PlanOptions {
    int32_t tile_rows = 1024;   // rows per tile before splitting
    int32_t local_slots = 3200; // shared-memory window slots per tile (x + acc = 16 B each)
    int32_t seg_max = 8;        // max entries per row segment (longer rows are split)
    int32_t gap = 8;            // merge column runs separated by <= gap unused slots
    int32_t max_segments = 8192;   // row segments per tile (32 x the kernel's 256-slice table)
    int32_t mode = 0;           // accumulation: 0 auto, 1 fixed point (3 words), 2 fp64,
                                // 3 fixed point (2 words) (tiles.cu)
    uint16_t sink = kNoSlot;    // local slot that padding lanes / entries point at (> local_slots)
    int32_t terms_cap = 0;      // > 0: halve row ranges whose busiest slot would take more
                                // accumulator terms than this (down to terms_min_rows rows;
                                // 1: single long rows are cut into chunks of at most
                                // terms_cap - 2 segments)
    int32_t terms_min_rows = 256;
    bool skip_empty = false;    // rows without entries get no own slot (no diagonal term)
    int32_t sample_stride = 1;  // > 1: only every sample_stride-th row range is built (a partial
                                // plan, for structure estimates only: pars3_plan_create)
    std::vector<int32_t> cuts;  // ascending local indices no window may straddle (peer mode)
};

constexpr int kMaxWindows = 8;  // more windows than this -> explicit column list

struct TileMeta {      // 12 x int32
    int32_t r0, r1;    // owned rows
    int32_t w0, w1;    // window range (window mode)
    int32_t u0;        // offset of the explicit column list (list mode), else -1
    int32_t s0, s1;    // slice range
    int32_t local;     // local index space size
    int32_t pad0, pad1, pad2;
    int32_t ev;        // max |value| of the tile's entries < 2^ev (fixed-point scale)
};

struct Window {       // 4 x int32
    int32_t lo, len, loff;
    int32_t pad0;
};

struct HostPlan {
    int64_t n = 0;
    std::vector<TileMeta> tiles;
    std::vector<Window> wins;
    std::vector<int64_t> slice_off;     // record start of each slice, in 16-byte units (+ end)
    std::vector<uint8_t> rec;           // slice records (see above)
    std::vector<int32_t> ucol;          // list-mode tiles: global column of each local slot
    int64_t nnz = 0;                    // stored entries (without padding)
    int64_t slots = 0;                  // stored slots (with padding)
    int32_t max_nslots = 0;
    int32_t list_tiles = 0;
    int32_t max_local = 0;
    int32_t max_terms = 0;              // most accumulator terms one slot takes in one tile
    int64_t dmax = 0;                   // most terms one y element sums (row entries + column mirrors
                                        // + diagonal), when the builder counted them (0: not counted)
};

// Build from host split arrays (BandSplit layout, split.py:58-113).
int build_tile_plan(int64_t n, const int64_t *mid_ptr, const int32_t *mid_col,
                    const double *mid_val, int64_t outer_count, const int32_t *outer_row,
                    const int32_t *outer_col, const double *outer_val, const PlanOptions &opt,
                    HostPlan &out);

}  // namespace pars3
