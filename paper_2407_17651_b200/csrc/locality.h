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

// RCM of the split's graph after dropping the edges no short cycle supports.
int locality_order(const pars3_split_view *s, LocalityOrder &out);

}  // namespace pars3
