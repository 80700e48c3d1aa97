// PARS3 skew-symmetric SpMV kernels for B200 (sm_100a) + the C ABI around them.
//
// y = A x with A = diag + L - L^T, L stored strictly-lower (SSS, sign
// convention D1, formats.py:14-18): each stored a_ic (i > c) adds
// +a_ic*x_c to y_i and -a_ic*x_i to y_c (serial.py:56-61).
#include <cuda_runtime.h>

#include <cstdarg>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <string>

#include "common.h"

namespace pars3 {

static thread_local std::string g_last_error;

void set_error(const char *fmt, ...) {
    char buf[1024];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    g_last_error = buf;
}

}  // namespace pars3

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

extern "C" const char *pars3_last_error(void) { return pars3::g_last_error.c_str(); }
extern "C" int pars3_abi_version(void) { return 1; }

namespace {

constexpr int kSms = 148;

// ------------------------------------------------------------ atomic scheme
// Lock-free row-parallel product (parallel.py:416-427): the row accumulator
// is private, every mirror update is an L2 fp64 reduction.  One thread per
// row; kept simple on purpose -- it is the paper's comparison kernel.
__global__ void __launch_bounds__(256) k_sss_atomic(int32_t n, const int32_t *__restrict__ row_ptr,
                                                    const int32_t *__restrict__ col,
                                                    const double *__restrict__ val,
                                                    const double *__restrict__ diag,
                                                    const double *__restrict__ x,
                                                    double *__restrict__ y) {
    for (int32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const double xi = __ldg(x + i);
        double acc = diag ? __ldg(diag + i) * xi : 0.0;
        const int32_t hi = __ldg(row_ptr + i + 1);
        for (int32_t k = __ldg(row_ptr + i); k < hi; k++) {
            const int32_t c = __ldg(col + k);
            const double v = __ldg(val + k);
            acc += v * __ldg(x + c);
            atomicAdd(y + c, -v * xi);
        }
        atomicAdd(y + i, acc);
    }
}

// Outer triplets (row, col, val): one entry per thread, both updates atomic.
__global__ void __launch_bounds__(256) k_coo_atomic(int32_t cnt, const int32_t *__restrict__ row,
                                                    const int32_t *__restrict__ col,
                                                    const double *__restrict__ val,
                                                    const double *__restrict__ x,
                                                    double *__restrict__ y) {
    for (int32_t e = blockIdx.x * blockDim.x + threadIdx.x; e < cnt; e += gridDim.x * blockDim.x) {
        const int32_t i = __ldg(row + e), c = __ldg(col + e);
        const double v = __ldg(val + e);
        atomicAdd(y + i, v * __ldg(x + c));
        atomicAdd(y + c, -v * __ldg(x + i));
    }
}

__global__ void k_dot(int32_t n, const double *__restrict__ a, const double *__restrict__ b,
                      double *out) {
    double s = 0.0;
    for (int32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
        s += a[i] * b[i];
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    __shared__ double ws[32];
    if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x < 32) {
        s = threadIdx.x < (blockDim.x >> 5) ? ws[threadIdx.x] : 0.0;
        for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if (threadIdx.x == 0) atomicAdd(out, s);
    }
}

int grid_for(int64_t work, int block) {
    int64_t g = (work + block - 1) / block;
    if (g > (int64_t)kSms * 16) g = (int64_t)kSms * 16;
    return g < 1 ? 1 : (int)g;
}

}  // namespace

struct pars3_plan {
    pars3_split_view s;
    int32_t p;
};

extern "C" int pars3_sss_spmv_atomic(int32_t n, const int32_t *row_ptr, const int32_t *col_ind,
                                     const double *off_diags, const double *diags, const double *x,
                                     double *y, void *stream) {
    if (n < 0) PARS3_FAIL(PARS3_ERR_ARG, "n must be non-negative");
    if (n == 0) return PARS3_OK;
    if (!row_ptr || !x || !y) PARS3_FAIL(PARS3_ERR_ARG, "null device pointer");
    cudaStream_t st = (cudaStream_t)stream;
    CUDA_TRY(cudaMemsetAsync(y, 0, sizeof(double) * (size_t)n, st));
    k_sss_atomic<<<grid_for(n, 256), 256, 0, st>>>(n, row_ptr, col_ind, off_diags, diags, x, y);
    LAUNCH_CHECK();
    return PARS3_OK;
}

extern "C" int pars3_plan_create(const pars3_split_view *split, int32_t p,
                                 const int64_t *block_start, pars3_plan **out, void *stream) {
    (void)stream;
    (void)block_start;
    if (!split || !out) PARS3_FAIL(PARS3_ERR_ARG, "null argument");
    if (split->n < 0 || split->beta < 1) PARS3_FAIL(PARS3_ERR_ARG, "bad split header");
    if (p < 1) PARS3_FAIL(PARS3_ERR_ARG, "worker count must be at least 1, got %d", p);
    pars3_plan *pl = new (std::nothrow) pars3_plan;
    if (!pl) PARS3_FAIL(PARS3_ERR_NOMEM, "out of host memory");
    pl->s = *split;
    pl->p = p;
    *out = pl;
    return PARS3_OK;
}

extern "C" int pars3_plan_spmv(pars3_plan *pl, const double *x, double *y, void *stream) {
    if (!pl || !x || !y) PARS3_FAIL(PARS3_ERR_ARG, "null argument");
    const pars3_split_view &s = pl->s;
    if (s.n == 0) return PARS3_OK;
    cudaStream_t st = (cudaStream_t)stream;
    CUDA_TRY(cudaMemsetAsync(y, 0, sizeof(double) * (size_t)s.n, st));
    k_sss_atomic<<<grid_for(s.n, 256), 256, 0, st>>>(s.n, s.mid_ptr, s.mid_col, s.mid_val, s.diag,
                                                      x, y);
    LAUNCH_CHECK();
    if (s.outer_count > 0) {
        k_coo_atomic<<<grid_for(s.outer_count, 256), 256, 0, st>>>(
            s.outer_count, s.outer_row, s.outer_col, s.outer_val, x, y);
        LAUNCH_CHECK();
    }
    return PARS3_OK;
}

extern "C" int pars3_plan_spmv_dot(pars3_plan *pl, const double *x, double *y, const double *w,
                                   double *dot, void *stream) {
    int rc = pars3_plan_spmv(pl, x, y, stream);
    if (rc) return rc;
    if (!w || !dot) PARS3_FAIL(PARS3_ERR_ARG, "null argument");
    cudaStream_t st = (cudaStream_t)stream;
    CUDA_TRY(cudaMemsetAsync(dot, 0, sizeof(double), st));
    if (pl->s.n > 0) {
        k_dot<<<grid_for(pl->s.n, 512), 512, 0, st>>>(pl->s.n, y, w, dot);
        LAUNCH_CHECK();
    }
    return PARS3_OK;
}

extern "C" int pars3_plan_kernel_count(const pars3_plan *pl, int32_t with_dot, int32_t *count) {
    if (!pl || !count) PARS3_FAIL(PARS3_ERR_ARG, "null argument");
    *count = (pl->s.n > 0 ? 1 : 0) + (pl->s.outer_count > 0 ? 1 : 0) + (with_dot && pl->s.n > 0 ? 1 : 0);
    return PARS3_OK;
}

extern "C" int pars3_plan_bytes(const pars3_plan *pl, int64_t *bytes) {
    if (!pl || !bytes) PARS3_FAIL(PARS3_ERR_ARG, "null argument");
    *bytes = 0;
    return PARS3_OK;
}

extern "C" int pars3_plan_destroy(pars3_plan *pl) {
    delete pl;
    return PARS3_OK;
}
