// smem-path microbenchmarks: cost per warp-instruction per SM of the shared
// memory operations a symmetric SpMV tile kernel would issue per entry.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t hsh(uint32_t x){ x^=x>>16; x*=0x7feb352d; x^=x>>15; x*=0x846ca68b; x^=x>>16; return x; }
template<int OP>
__global__ void k(double* out, int iters, int span){
  extern __shared__ double s[];
  int*  si=(int*)s;
  for(int i=threadIdx.x;i<span;i+=blockDim.x) s[i]=i*0.5;
  __syncthreads();
  double acc=0; uint32_t seed=threadIdx.x*2654435761u+blockIdx.x;
  int lane=threadIdx.x&31, w=threadIdx.x>>5;
  #pragma unroll 4
  for(int it=0;it<iters;it++){
    uint32_t a;
    if(OP==0||OP==2||OP==4||OP==10||OP==11) a = ((w*37+it)*32 + lane) & (span-1);           // sequential within warp
    else { seed = seed*1664525u + 1013904223u; a = (seed>>7) & (span-1); }                                            // random
    if(OP==0||OP==1) acc += s[a];                                            // LDS.64
    else if(OP==2||OP==3) s[a] = acc + it;                                   // STS.64
    else if(OP==4||OP==5) atomicAdd(si+a, 1);                                // ATOMS.ADD.32
    else if(OP==6) atomicAdd(s+a, 1.0);                                      // CAS f64
    else if(OP==7) acc += __shfl_xor_sync(0xffffffff, acc+it, 1);            // SHFL double
    else if(OP==8) { s[a] += 1.0; }
    else if(OP==9) { acc += (double)(a&7); }
    else if(OP==10) atomicAdd(s+a, 1.0);
    else if(OP==11) { s[a] += 1.0; }                                          // LDS+STS RMW random
  }
  if(acc==1.2345) out[blockIdx.x]=acc;
}
int main(){
  cudaEvent_t e0,e1; cudaEventCreate(&e0); cudaEventCreate(&e1); float ms;
  double* out; cudaMalloc(&out, 1<<20);
  const char* names[]={"LDS.64 seq","LDS.64 rand","STS.64 seq","STS.64 rand","ATOMS.ADD.32 seq","ATOMS.ADD.32 rand","CAS-f64 rand","SHFL f64","RMW f64 rand","ALU only","CAS-f64 seq","RMW f64 seq"};
  int sms=148, iters=4096, span=4096;
  for(int bs: {256, 1024}){
    int grid=sms*(2048/bs);
    for(int op=0;op<12;op++){
      auto launch=[&](){
        switch(op){
          case 0: k<0><<<grid,bs,span*8>>>(out,iters,span); break;
          case 1: k<1><<<grid,bs,span*8>>>(out,iters,span); break;
          case 2: k<2><<<grid,bs,span*8>>>(out,iters,span); break;
          case 3: k<3><<<grid,bs,span*8>>>(out,iters,span); break;
          case 4: k<4><<<grid,bs,span*8>>>(out,iters,span); break;
          case 5: k<5><<<grid,bs,span*8>>>(out,iters,span); break;
          case 6: k<6><<<grid,bs,span*8>>>(out,iters,span); break;
          case 7: k<7><<<grid,bs,span*8>>>(out,iters,span); break;
          case 8: k<8><<<grid,bs,span*8>>>(out,iters,span); break;
          case 9: k<9><<<grid,bs,span*8>>>(out,iters,span); break;
          case 10: k<10><<<grid,bs,span*8>>>(out,iters,span); break;
          case 11: k<11><<<grid,bs,span*8>>>(out,iters,span); break;
        }};
      launch(); cudaEventRecord(e0); launch(); cudaEventRecord(e1); cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms,e0,e1);
      double warp_ops_per_sm = (double)grid*bs/32*iters/sms;
      int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
      printf("bs=%4d %-18s %.3f ns/warp-op/SM  (%.2f cyc @1.9GHz)\n", bs, names[op], ms*1e6/warp_ops_per_sm, ms*1e6/warp_ops_per_sm*1.9);
    }
  }
  printf("err: %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
