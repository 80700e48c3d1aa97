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
