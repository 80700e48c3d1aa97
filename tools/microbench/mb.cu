// Microbenchmarks that size the PARS3 kernel design on B200:
// streaming bandwidth for the 12 B/entry matrix stream, L2 fp64 reduction
// throughput (red.global.add.f64), L2 gather throughput, smem fp64 atomics.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("CUDA %s @%d\n",cudaGetErrorString(e),__LINE__); return 1;}}while(0)

__global__ void stream_read(const double2* __restrict__ v, const int4* __restrict__ c, size_t n2, size_t n4, double* out){
  double acc=0; size_t tid=blockIdx.x*(size_t)blockDim.x+threadIdx.x, st=(size_t)gridDim.x*blockDim.x;
  for(size_t i=tid;i<n2;i+=st){ double2 a=__ldg(v+i); acc+=a.x+a.y; }
  for(size_t i=tid;i<n4;i+=st){ int4 a=__ldg(c+i); acc+=a.x+a.y+a.z+a.w; }
  if(acc==1234.5) out[0]=acc;
}
__global__ void copy_k(const double2* __restrict__ a, double2* __restrict__ b, size_t n){
  size_t tid=blockIdx.x*(size_t)blockDim.x+threadIdx.x, st=(size_t)gridDim.x*blockDim.x;
  for(size_t i=tid;i<n;i+=st) b[i]=a[i];
}
__device__ __forceinline__ uint32_t hsh(uint32_t x){ x^=x>>16; x*=0x7feb352d; x^=x>>15; x*=0x846ca68b; x^=x>>16; return x; }
__global__ void red_k(double* y, size_t nops, uint32_t window, int mode){
  size_t tid=blockIdx.x*(size_t)blockDim.x+threadIdx.x, st=(size_t)gridDim.x*blockDim.x;
  for(size_t i=tid;i<nops;i+=st){
    uint32_t a = mode==0 ? (uint32_t)(i % window) : hsh((uint32_t)i) % window;
    atomicAdd(y+a, 1.0);
  }
}
__global__ void gather_k(const double* __restrict__ x, size_t nops, uint32_t window, int mode, double* out){
  size_t tid=blockIdx.x*(size_t)blockDim.x+threadIdx.x, st=(size_t)gridDim.x*blockDim.x;
  double acc=0;
  for(size_t i=tid;i<nops;i+=st){
    uint32_t a = mode==0 ? (uint32_t)(i % window) : hsh((uint32_t)i) % window;
    acc+=__ldg(x+a);
  }
  if(acc==1234.5) out[0]=acc;
}
__global__ void smem_atom_k(double* out, int iters, int mode){
  __shared__ double s[4096];
  for(int i=threadIdx.x;i<4096;i+=blockDim.x) s[i]=0;
  __syncthreads();
  for(int k=0;k<iters;k++){
    int a = mode==0 ? (threadIdx.x + k*blockDim.x) & 4095 : hsh(threadIdx.x*7919u + k) & 4095;
    atomicAdd(s+a, 1.0);
  }
  __syncthreads();
  if(threadIdx.x==0) out[blockIdx.x]=s[0];
}
int main(){
  cudaEvent_t e0,e1; cudaEventCreate(&e0); cudaEventCreate(&e1); float ms;
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  printf("SMs %d\n", sms);
  size_t m = 216338940; // c5 entries
  double2* v; int4* c; double* out;
  CK(cudaMalloc(&v, m*8)); CK(cudaMalloc(&c, m*4)); CK(cudaMalloc(&out, 1<<20));
  cudaMemset(v,0,m*8); cudaMemset(c,0,m*4);
  for(int bs: {256, 512}) for(int per: {2,4,8}){
    int grid=sms*per;
    stream_read<<<grid,bs>>>(v,c,m/2,m/4,out);
    cudaEventRecord(e0);
    for(int r=0;r<5;r++) stream_read<<<grid,bs>>>(v,c,m/2,m/4,out);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms,e0,e1);
    printf("stream_read 12B/entry bs=%d grid=%d: %.1f us  %.1f GB/s\n", bs, grid, ms/5*1e3, m*12.0/(ms/5*1e-3)/1e9);
  }
  { size_t n=m/2; double2* b; CK(cudaMalloc(&b, m*8));
    copy_k<<<sms*4,512>>>(v,b,n); cudaEventRecord(e0);
    for(int r=0;r<5;r++) copy_k<<<sms*4,512>>>(v,b,n);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms,e0,e1);
    printf("copy %.1f GB/s\n", 2.0*m*8/(ms/5*1e-3)/1e9); cudaFree(b);}
  double* y; CK(cudaMalloc(&y, (size_t)1<<30));
  size_t nops = 1<<27;
  for(uint32_t window: {1u<<10, 1u<<14, 1u<<18, 1u<<22, 1u<<24}) for(int mode: {0,1}){
    red_k<<<sms*8,256>>>(y,nops,window,mode);
    cudaEventRecord(e0); red_k<<<sms*8,256>>>(y,nops,window,mode); cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms,e0,e1);
    printf("red.f64 window=%u (%.1f MB) mode=%s: %.2f Gop/s\n", window, window*8/1e6, mode?"hash":"seq", nops/(ms*1e-3)/1e9);
  }
  for(uint32_t window: {1u<<14, 1u<<18, 1u<<22, 1u<<24, 1u<<27}) for(int mode: {0,1}){
    gather_k<<<sms*8,256>>>(y,nops,window,mode,out);
    cudaEventRecord(e0); gather_k<<<sms*8,256>>>(y,nops,window,mode,out); cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms,e0,e1);
    printf("gather f64 window=%u (%.1f MB) mode=%s: %.2f Gop/s\n", window, window*8/1e6, mode?"hash":"seq", nops/(ms*1e-3)/1e9);
  }
  for(int mode: {0,1}){
    int iters=4096;
    smem_atom_k<<<sms*4,512>>>(out,iters,mode);
    cudaEventRecord(e0); smem_atom_k<<<sms*4,512>>>(out,iters,mode); cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms,e0,e1);
    double ops=(double)sms*4*512*iters;
    printf("smem atomicAdd f64 mode=%s: %.2f Gop/s (%.3f cyc/lane/SM at 1.9GHz)\n", mode?"hash":"seq", ops/(ms*1e-3)/1e9, (ms*1e-3*1.9e9)/(ops/sms));
  }
  CK(cudaDeviceSynchronize());
  return 0;
}
