// L2 residency microbenchmark (round 2): does an int64 accumulator that is
// reduced into (red.global.add.u64, with or without an evict_last hint)
// survive a long evict-first stream through the 126 MB L2?
//   touch(A)  ->  stream(B, S MB)  ->  readzero(A)
// Run under  ncu --cache-control none --metrics dram__bytes_read.sum,dram__bytes_write.sum
// and read the DRAM bytes of readzero: ~0 when A stayed in L2.
//   mb4 A_MB S_MB hint(0/1) stream_mode(0 ldcs, 1 prefetch.L2 + ldcs, 2 plain ld, 3 prefetch.L2 with an evict_first hint + ldcs)
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("CUDA %s @%d\n",cudaGetErrorString(e),__LINE__); return 1;}}while(0)

__device__ __forceinline__ uint64_t keep_policy(){ uint64_t p; asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p)); return p; }

__global__ void touch(long long* a, size_t n, int hint){
  const uint64_t pol = keep_policy();
  size_t tid=blockIdx.x*(size_t)blockDim.x+threadIdx.x, st=(size_t)gridDim.x*blockDim.x;
  for(size_t i=tid;i<n;i+=st){
    if(hint) asm volatile("red.global.add.L2::cache_hint.u64 [%0], %1, %2;" ::"l"(a+i), "l"(1ll), "l"(pol) : "memory");
    else asm volatile("red.global.add.u64 [%0], %1;" ::"l"(a+i), "l"(1ll) : "memory");
  }
}
__global__ void stream(const double2* __restrict__ b, size_t n2, int mode, double* out){
  size_t tid=blockIdx.x*(size_t)blockDim.x+threadIdx.x, st=(size_t)gridDim.x*blockDim.x;
  double acc=0;
  for(size_t i=tid;i<n2;i+=st){
    if(mode==1 && (threadIdx.x&31)==0 && i+st<n2)
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(b+i+st), "r"(512u) : "memory");
    if(mode==3 && (threadIdx.x&31)==0 && i+st<n2){
      uint64_t pf; asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pf));
      asm volatile("cp.async.bulk.prefetch.L2.global.L2::cache_hint [%0], %1, %2;" ::"l"(b+i+st), "r"(512u), "l"(pf) : "memory");
    }
    double2 v = mode==2 ? b[i] : __ldcs(b+i);
    acc+=v.x+v.y;
  }
  if(acc==1234.5) out[0]=acc;
}
__global__ void readzero(long long* a, size_t n, int hint, long long* out){
  const uint64_t pol = keep_policy();
  size_t tid=blockIdx.x*(size_t)blockDim.x+threadIdx.x, st=(size_t)gridDim.x*blockDim.x;
  long long acc=0;
  for(size_t i=tid;i<n;i+=st){
    long long v;
    if(hint){
      asm volatile("ld.global.L2::cache_hint.b64 %0, [%1], %2;" : "=l"(v) : "l"(a+i), "l"(pol));
      asm volatile("st.global.L2::cache_hint.b64 [%0], %1, %2;" ::"l"(a+i), "l"(0ll), "l"(pol) : "memory");
    } else { v=a[i]; a[i]=0; }
    acc+=v;
  }
  if(acc==12345) out[0]=acc;
}
int main(int argc, char** argv){
  size_t amb = argc>1?atoi(argv[1]):32, smb = argc>2?atoi(argv[2]):512; int hint=argc>3?atoi(argv[3]):0, mode=argc>4?atoi(argv[4]):0;
  size_t na = amb*(1<<20)/8, nb2 = smb*(size_t)(1<<20)/16;
  long long *a,*o; double2* b; double* od;
  CK(cudaMalloc(&a, na*8)); CK(cudaMalloc(&b, nb2*16)); CK(cudaMalloc(&o,8)); CK(cudaMalloc(&od,8));
  CK(cudaMemset(a,0,na*8)); CK(cudaMemset(b,0,nb2*16));
  cudaEvent_t e0,e1; cudaEventCreate(&e0); cudaEventCreate(&e1); float ms;
  for(int rep=0;rep<3;rep++){
    touch<<<148*8,256>>>(a,na,hint);
    stream<<<148*8,256>>>(b,nb2,mode,od);
    cudaEventRecord(e0);
    readzero<<<148*8,256>>>(a,na,hint,o);
    cudaEventRecord(e1); CK(cudaDeviceSynchronize());
    cudaEventElapsedTime(&ms,e0,e1);
    printf("A %zu MB stream %zu MB hint %d mode %d: readzero %.2f us\n", amb, smb, hint, mode, ms*1e3);
  }
  return 0;
}
