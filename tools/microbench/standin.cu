// Stand-in for NCCL's all-reduce kernel in tools/overlap_timeline.py: `ctas` CTAs of 640 threads with 64 KB of
// shared memory each (the footprint of an NCCL channel: it needs a third of an SM's warps and shared memory that a
// full sampling grid does not leave free), spinning for `cycles`.
// build: nvcc -gencode arch=compute_100a,code=sm_100a -shared -Xcompiler -fPIC -o standin.so standin.cu
#include <cuda_runtime.h>

__global__ void __launch_bounds__(640) standin_kernel(long long cycles, unsigned *sink) {
    extern __shared__ unsigned buf[];
    buf[threadIdx.x] = threadIdx.x;
    const long long t0 = clock64();
    while (clock64() - t0 < cycles)
        __nanosleep(500);
    if (buf[(threadIdx.x + 1) % 640] == 0xdeadbeefu)
        *sink = 1;
}

extern "C" int standin_launch(void *stream, int ctas, long long cycles, unsigned *sink) {
    static bool set = false;
    if (!set) {
        cudaFuncSetAttribute(standin_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 << 10);
        set = true;
    }
    standin_kernel<<<ctas, 640, 64 << 10, static_cast<cudaStream_t>(stream)>>>(cycles, sink);
    return static_cast<int>(cudaGetLastError());
}
