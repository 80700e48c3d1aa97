// Device builder of the tile plan (tileplan_gpu.cu): the host builder's
// arrays byte for byte, left on the device, for window-mode plans.
#pragma once
#include <cstdint>

#include "tileplan.h"

#define PARS3_GPU_MAX_SLICES 256  // slices per tile (the kernel's per-tile slice table)

namespace pars3 {

struct DevicePlan {  // device arrays of a plan built on the device (owned until release())
    TileMeta *tiles = nullptr;
    Window *wins = nullptr;
    int64_t *slice_off = nullptr;  // nslices + 1
    uint8_t *rec = nullptr;
    int64_t ntiles = 0, nwins = 0, nslices = 0, rec_bytes = 0;
    void release();
};

struct DeviceSplit {  // the split's arrays on the current device (optional: saves the upload)
    const int64_t *mid_ptr;
    const int32_t *mid_col;
    const double *mid_val;
    const int32_t *outer_row, *outer_col;
    const double *outer_val;
};

// Host split arrays in (uploaded once unless `resident` holds them), device plan out.  `supported` false:
// this plan needs the host builder (build_tile_plan); nothing is returned
// then.  On success P holds the small host-side parts (tiles, windows,
// totals; no records) and D the device arrays.
int build_tile_plan_device(int64_t n, const int64_t *mid_ptr, const int32_t *mid_col, const double *mid_val,
                           int64_t outer_count, const int32_t *outer_row, const int32_t *outer_col,
                           const double *outer_val, const PlanOptions &opt, HostPlan &P, DevicePlan &D,
                           bool &supported, const DeviceSplit *resident = nullptr);

}  // namespace pars3
