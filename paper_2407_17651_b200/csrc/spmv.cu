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
#include <algorithm>
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

int grid_for(int64_t work, int block) {
    int64_t g = (work + block - 1) / block;
    if (g > (int64_t)kSms * 16) g = (int64_t)kSms * 16;
    return g < 1 ? 1 : (int)g;
}

}  // namespace

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


// ---- CUDA IPC buffers for the peer-mode multi-GPU product -----------------
extern "C" int pars3_ipc_alloc(int64_t bytes, void **ptr) {
    if (!ptr || bytes < 0) PARS3_FAIL(PARS3_ERR_ARG, "bad argument");
    CUDA_TRY(cudaMalloc(ptr, bytes > 0 ? (size_t)bytes : 16));
    return PARS3_OK;
}

extern "C" int pars3_ipc_free(void *ptr) {
    if (ptr) CUDA_TRY(cudaFree(ptr));
    return PARS3_OK;
}

extern "C" int pars3_ipc_handle(void *ptr, uint8_t *handle64) {
    if (!ptr || !handle64) PARS3_FAIL(PARS3_ERR_ARG, "null argument");
    cudaIpcMemHandle_t h;
    static_assert(sizeof(h) == 64, "CUDA IPC handles are 64 bytes");
    CUDA_TRY(cudaIpcGetMemHandle(&h, ptr));
    memcpy(handle64, &h, 64);
    return PARS3_OK;
}

extern "C" int pars3_ipc_open(const uint8_t *handle64, void **ptr) {
    if (!ptr || !handle64) PARS3_FAIL(PARS3_ERR_ARG, "null argument");
    cudaIpcMemHandle_t h;
    memcpy(&h, handle64, 64);
    CUDA_TRY(cudaIpcOpenMemHandle(ptr, h, cudaIpcMemLazyEnablePeerAccess));
    return PARS3_OK;
}

extern "C" int pars3_ipc_close(void *ptr) {
    if (ptr) CUDA_TRY(cudaIpcCloseMemHandle(ptr));
    return PARS3_OK;
}

// ---- peer-mode step epilogue --------------------------------------------------
// y_out = acc + inbox, acc = inbox = 0, and (dot != NULL) *dot += <y_out, y_out>:
// the own-row accumulator, the partials the other ranks reduced into this
// rank's inbox, both cleared for the next product, and the MRS step's inner
// product -- one pass instead of four.
namespace {
__global__ void __launch_bounds__(512) k_peer_finish(int64_t n, double *__restrict__ acc,
                                                     double *__restrict__ inbox,
                                                     double *__restrict__ y_out, double *dot) {
    double s = 0.0;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += stride) {
        const double v = acc[i] + inbox[i];
        acc[i] = 0.0;
        inbox[i] = 0.0;
        y_out[i] = v;
        s = fma(v, v, s);
    }
    if (!dot) return;
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    __shared__ double ws[16];
    if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x < 32) {
        s = threadIdx.x < (blockDim.x >> 5) ? ws[threadIdx.x] : 0.0;
        for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if (threadIdx.x == 0) atomicAdd(dot, s);
    }
}
}  // namespace

extern "C" int pars3_peer_finish(int64_t n, double *acc, double *inbox, double *y_out, double *dot,
                                 void *stream) {
    if (n < 0 || (n > 0 && (!acc || !inbox || !y_out))) PARS3_FAIL(PARS3_ERR_ARG, "bad argument");
    cudaStream_t st = (cudaStream_t)stream;
    if (dot) CUDA_TRY(cudaMemsetAsync(dot, 0, sizeof(double), st));
    if (n == 0) return PARS3_OK;
    const int64_t blocks = std::min<int64_t>((n + 511) / 512, 148 * 4);
    k_peer_finish<<<(int)blocks, 512, 0, st>>>(n, acc, inbox, y_out, dot);
    LAUNCH_CHECK();
    return PARS3_OK;
}
