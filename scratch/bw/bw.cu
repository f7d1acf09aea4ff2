// scratch: plain streaming-read kernels to find the practical HBM floor for a
// 54 MB read right after an L2 flush (not part of the product).
#include <cstdint>
#include <cuda_runtime.h>
extern "C" __global__ void read_kernel(const uint4* __restrict__ p, size_t n16, uint32_t* out) {
    uint32_t acc = 0;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n16; i += (size_t)gridDim.x * blockDim.x) {
        uint4 v = __ldg(p + i);
        acc ^= v.x ^ v.y ^ v.z ^ v.w;
    }
    if (acc == 0x12345678u) out[0] = acc;
}
// TMA bulk version: one CTA per SM streams contiguous chunks through smem
extern "C" __global__ void bulk_kernel(const uint8_t* __restrict__ p, size_t bytes, int chunk, uint32_t* out) {
    extern __shared__ __align__(128) uint8_t sm[];
    __shared__ __align__(8) uint64_t bar[16];
    const int R = 16;
    if (threadIdx.x == 0) {
        for (int i = 0; i < R; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((uint32_t)__cvta_generic_to_shared(&bar[i])));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x != 0) return;
    const size_t nchunks = bytes / chunk;
    int k = 0;
    uint32_t acc = 0;
    for (size_t c = blockIdx.x; c < nchunks; c += gridDim.x, ++k) {
        const int s = k % R;
        if (k >= R) {  // wait for the previous use of this slot
            const uint32_t ph = ((k / R) - 1) & 1;
            asm volatile("{.reg .pred q; W: mbarrier.try_wait.parity.shared::cta.b64 q, [%0], %1; @!q bra W;}" ::"r"((uint32_t)__cvta_generic_to_shared(&bar[s])), "r"(ph) : "memory");
            acc ^= sm[s * chunk];
        }
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"((uint32_t)__cvta_generic_to_shared(&bar[s])), "r"(chunk) : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"((uint32_t)__cvta_generic_to_shared(sm + s * chunk)), "l"(p + c * chunk), "r"(chunk), "r"((uint32_t)__cvta_generic_to_shared(&bar[s])) : "memory");
    }
    for (int j = (k > R ? k - R : 0); j < k; ++j) {
        const int s = j % R;
        const uint32_t ph = (j / R) & 1;
        asm volatile("{.reg .pred q; W2: mbarrier.try_wait.parity.shared::cta.b64 q, [%0], %1; @!q bra W2;}" ::"r"((uint32_t)__cvta_generic_to_shared(&bar[s])), "r"(ph) : "memory");
    }
    if (acc == 0x12345678u) out[0] = acc;
}
extern "C" int run_read(const void* p, size_t bytes, int blocks, int threads, void* out, void* stream) {
    read_kernel<<<blocks, threads, 0, (cudaStream_t)stream>>>((const uint4*)p, bytes / 16, (uint32_t*)out);
    return (int)cudaGetLastError();
}
extern "C" int run_bulk(const void* p, size_t bytes, int blocks, int chunk, void* out, void* stream) {
    cudaFuncSetAttribute(bulk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 16 * chunk);
    bulk_kernel<<<blocks, 32, 16 * chunk, (cudaStream_t)stream>>>((const uint8_t*)p, bytes, chunk, (uint32_t*)out);
    return (int)cudaGetLastError();
}
