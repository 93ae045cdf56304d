// Microbenchmark: random 8-byte gathers from a large array, several load flavours.
// Answers: how many DRAM sectors does one random probe cost on B200, and what is the probe rate ceiling?
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>
typedef unsigned long long u64;
__device__ __forceinline__ u64 mix(u64 x){ x ^= x>>33; x*=0xff51afd7ed558ccdULL; x^=x>>33; x*=0xc4ceb9fe1a85ec53ULL; x^=x>>33; return x; }
template<int MODE> __device__ __forceinline__ u64 load8(const u64* p){
  u64 v;
  if (MODE==0) v = __ldcg(p);
  else if (MODE==1) v = __ldg(p);
  else if (MODE==2) v = *p;
  else if (MODE==3) asm volatile("ld.global.cg.L2::64B.u64 %0, [%1];" : "=l"(v) : "l"(p));
  else if (MODE==4) asm volatile("ld.global.L1::no_allocate.u64 %0, [%1];" : "=l"(v) : "l"(p));
  else if (MODE==5) asm volatile("ld.global.cv.u64 %0, [%1];" : "=l"(v) : "l"(p));
  else v = __ldcs(p);
  return v;
}
template<int MODE, int ILP> __global__ void gather(const u64* a, u64 words, u64 per_thread, u64* out){
  u64 tid = blockIdx.x*(u64)blockDim.x+threadIdx.x; u64 acc=0; u64 s = mix(tid+12345);
  for (u64 i=0;i<per_thread;i+=ILP){
    u64 idx[ILP];
    #pragma unroll
    for(int k=0;k<ILP;++k){ s = mix(s+k+1); idx[k] = s % words; }
    #pragma unroll
    for(int k=0;k<ILP;++k) acc += load8<MODE>(a+idx[k]);
  }
  if (acc==0x1234567) out[0]=acc;
}
template<int MODE> void run(const char* name, const u64* a, u64 words, u64* out, int blocks, int threads){
  const u64 per_thread = 256; cudaEvent_t e0,e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  gather<MODE,8><<<blocks,threads>>>(a,words,per_thread,out); cudaDeviceSynchronize();
  cudaEventRecord(e0); gather<MODE,8><<<blocks,threads>>>(a,words,per_thread,out); cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms,e0,e1); double probes=(double)blocks*threads*per_thread;
  printf("%-28s %8.3f ms  %7.2f Gprobes/s  (x32B = %7.1f GB/s)\n", name, ms, probes/ms/1e6, probes*32/ms/1e6);
}
int main(int argc,char**argv){
  size_t gran = argc>1 ? atoi(argv[1]) : 0;
  if (gran) { cudaError_t e = cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, gran); printf("set limit %zu -> %s\n", gran, cudaGetErrorString(e)); }
  size_t got=0; cudaDeviceGetLimit(&got, cudaLimitMaxL2FetchGranularity); printf("L2 fetch granularity limit = %zu\n", got);
  u64 words = (8ull<<30)/8; u64* a; cudaMalloc(&a, words*8); cudaMemset(a, 1, words*8); u64* out; cudaMalloc(&out, 8);
  int blocks=148*16, threads=256;
  run<0>("ld.cg (ldcg)", a, words, out, blocks, threads);
  run<1>("ld.nc (ldg)", a, words, out, blocks, threads);
  run<2>("ld (default)", a, words, out, blocks, threads);
  run<3>("ld.cg.L2::64B", a, words, out, blocks, threads);
  run<4>("ld.L1::no_allocate", a, words, out, blocks, threads);
  run<5>("ld.cv", a, words, out, blocks, threads);
  run<6>("ld.cs", a, words, out, blocks, threads);
  return 0;
}
