// scratch: launch-overhead probe (not part of the product)
#include <cuda_runtime.h>
extern "C" __global__ void empty_kernel(int* out) { if (out && threadIdx.x == 9999) out[0] = 1; }
extern "C" int run_empty(int blocks, int threads, int smem, void* stream) {
    cudaFuncSetAttribute(empty_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    empty_kernel<<<blocks, threads, smem, (cudaStream_t)stream>>>(nullptr);
    return (int)cudaGetLastError();
}
