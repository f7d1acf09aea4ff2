// generate.cu — K0: counter-based synthetic KV generator.
//
// Replaces gen_synthetic_cache (cache.cpp:301-342) at scale. The reference
// draws one serial mt19937_64 stream (81 s for 32 layers x 32K on the host,
// BASELINE.md §2); here every element is an independent function of
// (seed, tensor, index), so any slice can be produced on any device and
// recomputed on the CPU (tests/rdkv_testlib.py::gen_values) bit-for-bit:
//
//   z   = splitmix64(seed * 0x9E3779B97F4A7C15 + (tensor + 1) * 0xD1B54A32D192ED03 + i)
//   S   = sum of the four 16-bit lanes of z          (Irwin-Hall(4), mean 131070)
//   x   = f32(S - 131070) * f32(1 / 37836.5)         (~N(0,1), |x| < 3.47)
//   K: x *= outlier_scale for c < outlier_channels;  x += boost * sgn(c) on heavy-hitter rows
//   Q: x += 0.5 * sgn(c)                              (when heavy hitters are enabled)
//   out = fp16(x)  (RNE; stored as fp16 or as the f32 value of that fp16)
//
// Heavy hitters (every hh_stride-th token, t % hh_stride == 0) make the probe
// attention peaky so that the allocator spreads bits over 2/4/8/16 (SURVEY.md
// §8(d) C4), which i.i.d. Gaussian caches never do.
#include "common.cuh"

namespace rdkv_b200 {

__host__ __device__ __forceinline__ uint64_t splitmix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

__host__ __device__ __forceinline__ float channel_sign(uint64_t seed, int c) {
    return (splitmix64(seed ^ 0x5BD1E9955BD1E995ULL ^ (uint64_t)c) & 1ULL) ? 1.0f : -1.0f;
}

template <typename T>
__global__ void generate_kernel(T* out, uint64_t seed, int tensor, uint64_t first, uint64_t count,
                                int d, int seq_len, int outlier_channels, float outlier_scale,
                                int hh_stride, float hh_boost) {
    const uint64_t base = seed * 0x9E3779B97F4A7C15ULL + (uint64_t)(tensor + 1) * 0xD1B54A32D192ED03ULL;
    for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < count;
         j += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t i = first + j;
        const uint64_t z = splitmix64(base + i);
        const int s = (int)(z & 0xFFFF) + (int)((z >> 16) & 0xFFFF) + (int)((z >> 32) & 0xFFFF) +
                      (int)((z >> 48) & 0xFFFF);
        float x = __fmul_rn((float)(s - 131070), 1.0f / 37836.5f);
        const int c = (int)(i % (uint64_t)d);
        if (tensor == 0) {
            if (c < outlier_channels) x = __fmul_rn(x, outlier_scale);
            if (hh_stride > 0) {
                const uint64_t t = (i / (uint64_t)d) % (uint64_t)seq_len;
                if (t % (uint64_t)hh_stride == 0) x = __fadd_rn(x, __fmul_rn(hh_boost, channel_sign(seed, c)));
            }
        } else if (tensor == 2 && hh_stride > 0) {
            x = __fadd_rn(x, 0.5f * channel_sign(seed, c));
        }
        const __half h = __float2half_rn(x);
        if constexpr (sizeof(T) == 2) {
            out[j] = h;
        } else {
            out[j] = __half2float(h);
        }
    }
}

}  // namespace rdkv_b200

using namespace rdkv_b200;

extern "C" RDKV_API int rdkv_cuda_generate(void* out, int32_t dtype, uint64_t seed, int32_t tensor,
                                           uint64_t first_index, uint64_t count, int32_t head_dim,
                                           int32_t seq_len, int32_t outlier_channels,
                                           float outlier_scale, int32_t hh_stride, float hh_boost,
                                           void* stream) {
    if (!out || head_dim < 1 || seq_len < 1 || tensor < 0 || tensor > 2) return RDKV_EINVAL;
    if (dtype != RDKV_F32 && dtype != RDKV_F16) return RDKV_EINVAL;
    if (count == 0) return RDKV_OK;
    const int threads = 256;
    uint64_t blocks64 = (count + threads - 1) / threads;
    const int blocks = (int)(blocks64 < 148ull * 64 ? blocks64 : 148ull * 64);
    auto st = static_cast<cudaStream_t>(stream);
    if (dtype == RDKV_F16) {
        generate_kernel<__half><<<blocks, threads, 0, st>>>(
            static_cast<__half*>(out), seed, tensor, first_index, count, head_dim, seq_len,
            outlier_channels, outlier_scale, hh_stride, hh_boost);
    } else {
        generate_kernel<float><<<blocks, threads, 0, st>>>(
            static_cast<float*>(out), seed, tensor, first_index, count, head_dim, seq_len,
            outlier_channels, outlier_scale, hh_stride, hh_boost);
    }
    return launch_status();
}
