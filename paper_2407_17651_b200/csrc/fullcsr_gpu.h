// Device builder of the row-major plan (fullcsr_gpu.cu): the host builder's
// arrays (fullcsr.cpp), already lane-interleaved, left on the device.
#pragma once
#include <cstdint>

#include "../../include/pars3.h"

namespace pars3 {

struct DeviceFullCsr {  // device arrays (owned until release() or taken by the plan)
    int64_t n = 0, ne = 0, nep = 0;  // rows, real entries, entries padded to warps of 512
    int32_t nspan = 0;
    int32_t *col = nullptr;          // [nep], lane-interleaved per warp
    double *val = nullptr;
    int32_t *lane_row = nullptr;     // [nep / 16]
    uint32_t *lane_flags = nullptr;
    int32_t *span_row = nullptr, *span_w0 = nullptr, *span_w1 = nullptr;  // [nspan]
    void release();
};

// done = false: not built here (no device, sizes beyond int32 item counts):
// the caller runs build_full_csr on the host
int build_full_csr_device(const pars3_split_view *s, DeviceFullCsr &D, bool &done);

}  // namespace pars3
