// Microbenchmark: random 4-byte stores (no prior read) and read-then-write, 8 GB array.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
typedef unsigned long long u64; typedef unsigned int u32;
__device__ __forceinline__ u64 mix(u64 x){ x ^= x>>33; x*=0xff51afd7ed558ccdULL; x^=x>>33; x*=0xc4ceb9fe1a85ec53ULL; x^=x>>33; return x; }
template<int MODE> __global__ void scatter(u32* a, u64 words, u64 per_thread, u64* out){
  u64 tid = blockIdx.x*(u64)blockDim.x+threadIdx.x; u64 s = mix(tid+777); u64 acc=0;
  for (u64 i=0;i<per_thread;i+=8){
    u64 idx[8];
    #pragma unroll
    for(int k=0;k<8;++k){ s = mix(s+k+1); idx[k] = s % words; }
    if (MODE==1) {
      #pragma unroll
      for(int k=0;k<8;++k) acc += __ldcg(a+idx[k]);
    }
    #pragma unroll
    for(int k=0;k<8;++k) __stcg(a+idx[k], (u32)(s+k+acc));
  }
  if (acc==0x1234567) out[0]=acc;
}
template<int MODE> void run(const char* name, u32* a, u64 words, u64* out){
  int blocks=148*16, threads=256; const u64 per_thread=256; cudaEvent_t e0,e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  scatter<MODE><<<blocks,threads>>>(a,words,per_thread,out); cudaDeviceSynchronize();
  cudaEventRecord(e0); scatter<MODE><<<blocks,threads>>>(a,words,per_thread,out); cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms,e0,e1); double ops=(double)blocks*threads*per_thread;
  printf("%-28s %8.3f ms  %7.2f Gops/s\n", name, ms, ops/ms/1e6);
}
int main(){
  u64 words=(8ull<<30)/4; u32* a; cudaMalloc(&a, words*4); cudaMemset(a,0,words*4); u64* out; cudaMalloc(&out,8);
  run<0>("random 4B store", a, words, out);
  run<1>("random 4B load then store", a, words, out);
  return 0;
}
