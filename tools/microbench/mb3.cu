// Inner-loop cost of the tile kernel on synthetic c5-like records:
// stream SELL-32 records (fp64 value + u16 local column), with increasing
// amounts of per-entry shared-memory work.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("CUDA %s @%d\n",cudaGetErrorString(e),__LINE__); return 1;}}while(0)
constexpr int NS = 8;            // slots per slice
constexpr int LM = 1024;         // local slots
template<int MODE>
__global__ void __launch_bounds__(512, 2) k(const double* __restrict__ val, const uint16_t* __restrict__ lidx, long nslices, double* out) {
  __shared__ double xs[LM], acc[LM];
  __shared__ unsigned int ah[LM], al[LM], am[LM];
  for (int i = threadIdx.x; i < LM; i += blockDim.x) { xs[i] = i * 1e-3; acc[i] = 0; ah[i]=al[i]=am[i]=0; }
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  double tot = 0;
  for (long s = (long)blockIdx.x * nw + warp; s < nslices; s += (long)gridDim.x * nw) {
    const double* vp = val + s * NS * 32 + lane; const uint16_t* ip = lidx + s * NS * 32 + lane;
    double v[NS]; uint16_t li[NS];
#pragma unroll
    for (int u = 0; u < NS; u++) { v[u] = __ldcs(vp + 32 * u); li[u] = __ldcs(ip + 32 * u); }
    const double xr = xs[(lane + s) & (LM - 1)];
    double racc = 0;
    if (MODE == 0) {
#pragma unroll
      for (int u = 0; u < NS; u++) racc += v[u] * (double)li[u];
    } else if (MODE == 1) {
#pragma unroll
      for (int u = 0; u < NS; u++) racc = fma(v[u], xs[li[u]], racc);
    } else if (MODE == 2) {   // batched CAS
      unsigned long long old[NS], got[NS]; double q[NS];
#pragma unroll
      for (int u = 0; u < NS; u++) { racc = fma(v[u], xs[li[u]], racc); q[u] = -v[u] * xr; old[u] = __double_as_longlong(acc[li[u]]); }
#pragma unroll
      for (int u = 0; u < NS; u++) got[u] = atomicCAS((unsigned long long*)(acc + li[u]), old[u], __double_as_longlong(__longlong_as_double(old[u]) + q[u]));
#pragma unroll
      for (int u = 0; u < NS; u++) if (got[u] != old[u]) { unsigned long long o = got[u]; for (;;) { unsigned long long g2 = atomicCAS((unsigned long long*)(acc + li[u]), o, __double_as_longlong(__longlong_as_double(o) + q[u])); if (g2 == o) break; o = g2; } }
    } else if (MODE == 3) {   // plain atomicAdd (CAS loop per entry)
#pragma unroll
      for (int u = 0; u < NS; u++) { racc = fma(v[u], xs[li[u]], racc); atomicAdd(acc + li[u], -v[u] * xr); }
    } else if (MODE == 4) {   // fixed point, 3 x 32-bit ATOMS
      const double scale = 1125899906842624.0; // 2^50
#pragma unroll
      for (int u = 0; u < NS; u++) {
        racc = fma(v[u], xs[li[u]], racc);
        const double qs = (-v[u] * xr) * scale + 6755399441055744.0;
        const long long Q = __double_as_longlong(qs) - 0x4338000000000000ll;
        atomicAdd(al + li[u], (unsigned)(Q & 0xFFFFF));
        atomicAdd(am + li[u], (unsigned)((Q >> 20) & 0xFFFFF));
        atomicAdd(ah + li[u], (unsigned)(int)(Q >> 40));
      }
    } else if (MODE == 5) {   // plain racy RMW (upper bound, incorrect)
#pragma unroll
      for (int u = 0; u < NS; u++) { racc = fma(v[u], xs[li[u]], racc); acc[li[u]] -= v[u] * xr; }
    }
    tot += racc;
  }
  __syncthreads();
  if (tot == 1.2345) out[0] = tot + acc[threadIdx.x] + ah[threadIdx.x];
}
int main() {
  const long nslices = 216338940L / (NS * 32);   // c5 entries
  const long ne = nslices * NS * 32;
  double* val; uint16_t* lidx; double* out;
  CK(cudaMalloc(&val, ne * 8)); CK(cudaMalloc(&lidx, ne * 2)); CK(cudaMalloc(&out, 64));
  // DIA-like local indices: slot j of lane l in slice s -> (base + l + off_j) & (LM-1)
  uint16_t* h = (uint16_t*)malloc(ne * 2);
  const int offs[NS] = {0, 67, 133, 300, 364, 430, 500, 566};
  for (long s = 0; s < nslices; s++) for (int j = 0; j < NS; j++) for (int l = 0; l < 32; l++)
    h[(s * NS + j) * 32 + l] = (uint16_t)(((s * 32) % 512 + l + offs[j]) & (LM - 1));
  CK(cudaMemcpy(lidx, h, ne * 2, cudaMemcpyHostToDevice)); CK(cudaMemset(val, 0, ne * 8));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const char* names[] = {"stream only", "+LDS x", "+batched CAS", "+atomicAdd CAS", "+fixed-point 3xATOMS", "+racy RMW"};
  for (int mode = 0; mode < 6; mode++) for (int ctas : {1, 2}) {
    int grid = 148 * ctas;
    auto run = [&]() { switch (mode) {
      case 0: k<0><<<grid, 512>>>(val, lidx, nslices, out); break;
      case 1: k<1><<<grid, 512>>>(val, lidx, nslices, out); break;
      case 2: k<2><<<grid, 512>>>(val, lidx, nslices, out); break;
      case 3: k<3><<<grid, 512>>>(val, lidx, nslices, out); break;
      case 4: k<4><<<grid, 512>>>(val, lidx, nslices, out); break;
      case 5: k<5><<<grid, 512>>>(val, lidx, nslices, out); break; } };
    run(); cudaEventRecord(e0); for (int r = 0; r < 5; r++) run(); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1); ms /= 5;
    printf("%-24s ctas/SM=%d: %.3f ms  (%.0f GB/s of 10 B/entry)\n", names[mode], ctas, ms, ne * 10.0 / (ms * 1e-3) / 1e9);
  }
  return 0;
}
