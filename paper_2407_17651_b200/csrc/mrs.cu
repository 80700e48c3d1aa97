// Fused vector kernels of the MRS iteration (minimal residual for shifted
// skew-symmetric systems): one pass each for the
// skew-Lanczos vector + its norm, and for the direction/solution update.
#include <cuda_runtime.h>

#include <cstdint>

#include "common.h"

namespace {

constexpr int kBlock = 512;

__device__ __forceinline__ double block_sum(double s) {
    __shared__ double ws[kBlock / 32];
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = s;
    __syncthreads();
    s = 0.0;
    if (threadIdx.x < 32) {
        s = threadIdx.x < kBlock / 32 ? ws[threadIdx.x] : 0.0;
        for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    }
    return s;
}

// u = y - alpha * v + gamma * w (into w), norm2 += <u, u>
__global__ void __launch_bounds__(kBlock) k_lanczos(int64_t n, const double *__restrict__ y,
                                                    const double *__restrict__ v, double *w,
                                                    double alpha, double gamma, double *norm2) {
    double s = 0.0;
    for (int64_t i = blockIdx.x * (int64_t)kBlock + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * kBlock) {
        const double u = fma(gamma, w[i], fma(-alpha, v[i], y[i]));
        w[i] = u;
        s = fma(u, u, s);
    }
    s = block_sum(s);
    if (threadIdx.x == 0) atomicAdd(norm2, s);
}

// v_next = u * inv_gamma (in place), d = (v - r0 * dm2 - r1 * dm1) * inv_r2
// (into dm2), x += tau * d
__global__ void __launch_bounds__(kBlock) k_update(int64_t n, double *u, double inv_gamma,
                                                   const double *__restrict__ v, double *dm2,
                                                   const double *__restrict__ dm1, double r0,
                                                   double r1, double inv_r2, double tau, double *x) {
    for (int64_t i = blockIdx.x * (int64_t)kBlock + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * kBlock) {
        const double d = (v[i] - r0 * dm2[i] - r1 * dm1[i]) * inv_r2;
        dm2[i] = d;
        x[i] = fma(tau, d, x[i]);
        u[i] *= inv_gamma;
    }
}

int grid_for(int64_t n) {
    int64_t g = (n + kBlock - 1) / kBlock;
    if (g > 148 * 8) g = 148 * 8;
    return g < 1 ? 1 : (int)g;
}

}  // namespace

extern "C" int pars3_mrs_lanczos(int64_t n, const double *y, const double *v, double *w,
                                 double alpha, double gamma, double *norm2, void *stream) {
    if (n < 0 || !norm2 || (n > 0 && (!y || !v || !w))) PARS3_FAIL(PARS3_ERR_ARG, "bad arguments");
    cudaStream_t st = (cudaStream_t)stream;
    CUDA_TRY(cudaMemsetAsync(norm2, 0, sizeof(double), st));
    if (n == 0) return PARS3_OK;
    k_lanczos<<<grid_for(n), kBlock, 0, st>>>(n, y, v, w, alpha, gamma, norm2);
    LAUNCH_CHECK();
    return PARS3_OK;
}

extern "C" int pars3_mrs_update(int64_t n, double *u, double inv_gamma, const double *v,
                                double *dm2, const double *dm1, double r0, double r1,
                                double inv_r2, double tau, double *x, void *stream) {
    if (n < 0 || (n > 0 && (!u || !v || !dm2 || !dm1 || !x))) PARS3_FAIL(PARS3_ERR_ARG, "bad arguments");
    if (n == 0) return PARS3_OK;
    k_update<<<grid_for(n), kBlock, 0, (cudaStream_t)stream>>>(n, u, inv_gamma, v, dm2, dm1, r0, r1,
                                                               inv_r2, tau, x);
    LAUNCH_CHECK();
    return PARS3_OK;
}
