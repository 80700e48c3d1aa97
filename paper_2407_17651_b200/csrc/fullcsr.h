// Full-CSR plan of the row-major product form: the
// whole skew matrix A = D + L - L^T stored row by row (each row: its lower
// entries, its diagonal, the negated mirrors of its column), cut into lanes
// of 16 entries and warps of 32 lanes.  Every row holds its diagonal entry,
// so no row is empty and the row starts mark every row once.
#pragma once
#include <cstdint>
#include <vector>

#include "../../include/pars3.h"

namespace pars3 {

#ifndef PARS3_CSR_LANE  // tuning builds
#define PARS3_CSR_LANE 16
#endif
constexpr int kCsrLane = PARS3_CSR_LANE;      // entries per lane (<= 16: the row-start mask has 32 bits)
constexpr int kCsrWarp = 32 * kCsrLane;       // entries per warp

struct FullCsr {
    int64_t n = 0;
    int64_t ne = 0;                  // real entries (2 m + n)
    std::vector<int32_t> col;        // [ne padded to a multiple of kCsrWarp]
    std::vector<double> val;
    std::vector<int32_t> lane_row;   // row of each lane's first entry
    std::vector<uint32_t> lane_flags;  // bit k: entry k starts a row; bit 16: the entry after
                                       // the lane starts a row (or the matrix ends)
    // rows spanning warps: y[row] = tail[w0] + sum of head[w0 + 1 .. w1]
    std::vector<int32_t> span_row, span_w0, span_w1;
    int32_t max_span = 0;            // most warps one row spans
};

int build_full_csr(const pars3_split_view *s, FullCsr &F);

}  // namespace pars3
