// Shared error plumbing for libpars3.so (C ABI: codes + thread-local message).
#pragma once
#include <cstdarg>
#include <cstdio>
#include <string>

#include "../../include/pars3.h"

namespace pars3 {

void set_error(const char *fmt, ...);

}  // namespace pars3

#define PARS3_FAIL(code, ...)                 \
    do {                                      \
        ::pars3::set_error(__VA_ARGS__);      \
        return (code);                        \
    } while (0)

#ifdef __CUDACC__
#define CUDA_TRY(expr)                                                                  \
    do {                                                                                \
        cudaError_t _e = (expr);                                                        \
        if (_e != cudaSuccess)                                                          \
            PARS3_FAIL(PARS3_ERR_CUDA, "%s failed: %s", #expr, cudaGetErrorString(_e)); \
    } while (0)

#define LAUNCH_CHECK()                                                                 \
    do {                                                                               \
        cudaError_t _e = cudaGetLastError();                                           \
        if (_e != cudaSuccess)                                                         \
            PARS3_FAIL(PARS3_ERR_CUDA, "kernel launch failed: %s", cudaGetErrorString(_e)); \
    } while (0)

#endif
