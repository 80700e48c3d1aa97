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

// ---- device-resident MRS step (no host round trip per iteration) ----------
// State (double[kMrsState], device): the recurrence scalars the host loop
// used to carry, so an iteration is five stream-ordered launches (product,
// Lanczos pass, norm, rotation, update) and the host reads nothing until it
// chooses to check convergence.  Sums have a fixed order (per-CTA shares of
// a fixed grid, summed in CTA order): the iteration is bitwise repeatable.
namespace {

enum {
    kGamma = 0, kC1, kS1, kC2, kS2, kPhi, kBeta, kNorm2, kR0, kR1, kInvR2, kTau, kInvG,
    kDone, kTol, kAlpha, kPending, kConvIter, kMrsState = 24
};
constexpr int kMrsGrid = 148 * 4;

// u = y - alpha v + gamma w (into w); part[block] = this block's share of <u, u>
__global__ void __launch_bounds__(kBlock) k_lanczos_dev(int64_t n, const double *__restrict__ y,
                                                        const double *__restrict__ v, double *w,
                                                        const double *st, double *part) {
    if (st[kDone] != 0.0) return;
    const double alpha = st[kAlpha], gamma = st[kGamma];
    double s = 0.0;
    for (int64_t i = blockIdx.x * (int64_t)kBlock + threadIdx.x; i < n; i += (int64_t)gridDim.x * kBlock) {
        const double u = fma(gamma, w[i], fma(-alpha, v[i], y[i]));
        w[i] = u;
        s = fma(u, u, s);
    }
    s = block_sum(s);
    if (threadIdx.x == 0) part[blockIdx.x] = s;
}

// st[kNorm2] = sum of part[0 .. np) in order (this rank's ||u||^2)
__global__ void __launch_bounds__(32) k_norm_dev(int32_t np, const double *__restrict__ part, double *st) {
    if (threadIdx.x == 0) {
        double s = 0.0;
        for (int i = 0; i < np; i++) s += part[i];
        st[kNorm2] = s;
    }
}

// the Givens step of iteration j (one thread): column j of H = (-g_j,
// alpha, g_{j+1}), the two previous rotations, a new one; resid[j] = |phi|
__global__ void __launch_bounds__(32) k_rotate_dev(double *st, double *resid, int32_t j) {
    if (threadIdx.x != 0) return;
    if (st[kDone] != 0.0) return;
    if (st[kPending] != 0.0) {  // converged at the previous step: stop here
        st[kDone] = 1.0;
        return;
    }
    const double alpha = st[kAlpha], gamma = st[kGamma];
    const double gnext = sqrt(st[kNorm2]);
    const double c1 = st[kC1], s1 = st[kS1], c2 = st[kC2], s2 = st[kS2];
    const double h1 = -gamma;
    const double r0 = s2 * h1;
    const double h1p = c2 * h1;
    const double r1 = c1 * h1p + s1 * alpha;
    const double h2p = -s1 * h1p + c1 * alpha;
    const double r2 = hypot(h2p, gnext);
    const double c = r2 > 0.0 ? h2p / r2 : 1.0, s = r2 > 0.0 ? gnext / r2 : 0.0;
    const double phi = st[kPhi];
    st[kTau] = c * phi;
    st[kPhi] = -s * phi;
    st[kR0] = r0;
    st[kR1] = r1;
    st[kInvR2] = 1.0 / r2;
    st[kInvG] = gnext > 0.0 ? 1.0 / gnext : 0.0;
    st[kGamma] = gnext;
    st[kC2] = c1;
    st[kS2] = s1;
    st[kC1] = c;
    st[kS1] = s;
    resid[j] = fabs(s * phi);
    if (fabs(s * phi) <= st[kTol] * st[kBeta] || gnext == 0.0) {
        st[kPending] = 1.0;
        st[kConvIter] = (double)j;
    }
}

// (xe_slot: the bound of the new u for the next product, in k_xmax's
// encoding, tiles.cu: max(biased exponent, 1) - 1022 + 1 + 2048 over the
// finite values)
__global__ void __launch_bounds__(kBlock) k_update_dev(int64_t n, double *u, const double *__restrict__ v,
                                                       double *dm2, const double *__restrict__ dm1, double *x,
                                                       const double *st, int32_t *xe_slot) {
    if (st[kDone] != 0.0) return;
    const double r0 = st[kR0], r1 = st[kR1], inv_r2 = st[kInvR2], tau = st[kTau], inv_g = st[kInvG];
    int e = -1100;
    // (four CTAs per SM as before the bound was added: the compiler's deeper
    // unrolling took 116 registers and ran the pass three times slower)
#pragma unroll 1
    for (int64_t i = blockIdx.x * (int64_t)kBlock + threadIdx.x; i < n; i += (int64_t)gridDim.x * kBlock) {
        const double d = (v[i] - r0 * dm2[i] - r1 * dm1[i]) * inv_r2;
        dm2[i] = d;
        x[i] = fma(tau, d, x[i]);
        const double un = u[i] * inv_g;
        u[i] = un;
        const int b = (int)((__double_as_longlong(un) >> 52) & 0x7FF);
        if (b != 2047) e = max(e, max(b, 1) - 1022);
    }
    if (xe_slot) {  // one atomic per CTA at most, and only when it would raise the bound
        __shared__ int s_e;
        if (threadIdx.x == 0) s_e = -1100;
        __syncthreads();
        e = __reduce_max_sync(0xffffffffu, e);
        if ((threadIdx.x & 31) == 0 && e > -1100) atomicMax(&s_e, e);
        __syncthreads();
        if (threadIdx.x == 0 && s_e > -1100 && s_e + 1 + 2048 > *(volatile int32_t *)xe_slot)
            atomicMax(xe_slot, s_e + 1 + 2048);
    }
}

}  // namespace

extern "C" int pars3_mrs_state_size(int32_t *size, int32_t *parts) {
    if (!size || !parts) PARS3_FAIL(PARS3_ERR_ARG, "null argument");
    *size = kMrsState;
    *parts = kMrsGrid;
    return PARS3_OK;
}

extern "C" int pars3_mrs_lanczos_dev(int64_t n, const double *y, const double *v, double *w, const double *state,
                                     double *part, void *stream) {
    if (n < 0 || !state || !part || (n > 0 && (!y || !v || !w))) PARS3_FAIL(PARS3_ERR_ARG, "bad arguments");
    cudaStream_t st = (cudaStream_t)stream;
    k_lanczos_dev<<<kMrsGrid, kBlock, 0, st>>>(n, y, v, w, state, part);
    LAUNCH_CHECK();
    k_norm_dev<<<1, 32, 0, st>>>(kMrsGrid, part, const_cast<double *>(state));
    LAUNCH_CHECK();
    return PARS3_OK;
}

extern "C" int pars3_mrs_rotate_dev(double *state, double *resid, int32_t j, void *stream) {
    if (!state || !resid || j < 1) PARS3_FAIL(PARS3_ERR_ARG, "bad arguments");
    k_rotate_dev<<<1, 32, 0, (cudaStream_t)stream>>>(state, resid, j);
    LAUNCH_CHECK();
    return PARS3_OK;
}

extern "C" int pars3_mrs_update_dev(int64_t n, double *u, const double *v, double *dm2, const double *dm1,
                                    double *x, const double *state, void *stream) {
    if (n < 0 || !state || (n > 0 && (!u || !v || !dm2 || !dm1 || !x))) PARS3_FAIL(PARS3_ERR_ARG, "bad arguments");
    if (n == 0) return PARS3_OK;
    k_update_dev<<<grid_for(n), kBlock, 0, (cudaStream_t)stream>>>(n, u, v, dm2, dm1, x, state, nullptr);
    LAUNCH_CHECK();
    return PARS3_OK;
}

extern "C" int pars3_mrs_update_dev2(int64_t n, double *u, const double *v, double *dm2, const double *dm1,
                                     double *x, const double *state, int32_t *xe_slot, void *stream) {
    if (n < 0 || !state || (n > 0 && (!u || !v || !dm2 || !dm1 || !x))) PARS3_FAIL(PARS3_ERR_ARG, "bad arguments");
    if (n == 0) return PARS3_OK;
    cudaStream_t st = (cudaStream_t)stream;
    if (xe_slot) CUDA_TRY(cudaMemsetAsync(xe_slot, 0, sizeof(int32_t), st));
    k_update_dev<<<grid_for(n), kBlock, 0, st>>>(n, u, v, dm2, dm1, x, state, xe_slot);
    LAUNCH_CHECK();
    return PARS3_OK;
}
