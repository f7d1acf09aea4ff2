// common.cuh — shared device helpers for the RDKV sm_100a kernels.
#pragma once

#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>

#include "../../include/rdkv_cuda.h"
#include "tile_layout.h"

namespace rdkv_b200 {

#define RDKV_CUDA_TRY(expr)                              \
    do {                                                 \
        cudaError_t _e = (expr);                         \
        if (_e != cudaSuccess) return RDKV_ECUDA;        \
    } while (0)

inline int launch_status() {
    return cudaGetLastError() == cudaSuccess ? RDKV_OK : RDKV_ECUDA;
}

// Immutable per-device attributes, queried once per device (launch paths are
// called per decode step; the attribute queries cost microseconds each).
struct DevAttrs {
    int dev, smem_optin, nsm;
};
constexpr int kMaxDevices = 64;
inline DevAttrs dev_attrs() {
    static std::atomic<int> cache[kMaxDevices][2];  // 0 = not yet queried
    int dev = 0;
    cudaGetDevice(&dev);
    DevAttrs a{dev, 0, 0};
    if (dev >= 0 && dev < kMaxDevices) {
        a.smem_optin = cache[dev][0].load(std::memory_order_relaxed);
        a.nsm = cache[dev][1].load(std::memory_order_relaxed);
        if (a.smem_optin > 0 && a.nsm > 0) return a;
    }
    cudaDeviceGetAttribute(&a.smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    cudaDeviceGetAttribute(&a.nsm, cudaDevAttrMultiProcessorCount, dev);
    if (dev >= 0 && dev < kMaxDevices) {
        cache[dev][0].store(a.smem_optin, std::memory_order_relaxed);
        cache[dev][1].store(a.nsm, std::memory_order_relaxed);
    }
    return a;
}

// Raises a kernel's dynamic shared-memory limit at most once per (kernel,
// device, size): `slots` is a per-kernel static array of kMaxDevices.
template <typename F>
inline void set_smem_once(F kern, int smem, std::atomic<int>* slots, int dev) {
    if (dev >= 0 && dev < kMaxDevices && slots[dev].load(std::memory_order_relaxed) >= smem) return;
    cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100);  // all of L1 as smem
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) == cudaSuccess && dev >= 0 &&
        dev < kMaxDevices) {
        int cur = slots[dev].load(std::memory_order_relaxed);
        while (cur < smem && !slots[dev].compare_exchange_weak(cur, smem)) {
        }
    }
}

template <typename T>
__device__ __forceinline__ float load_as_float(const T* p, size_t i);
template <>
__device__ __forceinline__ float load_as_float<float>(const float* p, size_t i) {
    return p[i];
}
template <>
__device__ __forceinline__ float load_as_float<__half>(const __half* p, size_t i) {
    return __half2float(p[i]);
}

__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}
__device__ __forceinline__ float warp_min(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fminf(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}
__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
__device__ __forceinline__ double warp_max_d(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}
__device__ __forceinline__ long long warp_sum_ll(long long v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

}  // namespace rdkv_b200
