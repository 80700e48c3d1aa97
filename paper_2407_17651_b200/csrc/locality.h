// Internal locality order of a device plan (locality.cpp).
#pragma once
#include <cstdint>
#include <vector>

#include "../../include/pars3.h"

namespace pars3 {

struct LocalityOrder {
    std::vector<int32_t> forward;  // split label -> internal label
    std::vector<int64_t> row_ptr;  // P A P^T, strictly lower, ascending columns
    std::vector<int32_t> col;
    std::vector<double> val;
    std::vector<double> diag;
    int64_t dropped = 0;           // directed edges the filter removed before the layering
};

// RCM of the split's graph after dropping the edges no short cycle supports
// (forward empty: the filter found no band to recover).  Runs on the current
// device when there is one (locality_gpu.cu: the same result bit for bit;
// PARS3_LOCALITY_HOST=1 keeps it on the host).
int locality_order(const pars3_split_view *s, LocalityOrder &out);
// done = false: not run (no device): the caller runs the host version
int locality_order_device(const pars3_split_view *s, LocalityOrder &out, bool &done);

}  // namespace pars3
