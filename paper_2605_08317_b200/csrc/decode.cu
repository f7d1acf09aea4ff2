// decode.cu — K4 dispatch: chooses the tensor-core kernel (decode_mma.cu) for
// the layouts it covers and the generic CUDA-core kernel otherwise; split-K
// workspace; host-buffer (end-to-end) entry point.
#include "common.cuh"

namespace rdkv_b200 {
template <typename IO>
int launch_generic(const rdkv_decode_args* a, int split, int max_kslots, cudaStream_t st);
int launch_mma(const rdkv_decode_args* a, cudaStream_t st);  // decode_mma.cu
bool mma_supported(const rdkv_decode_args* a);
}  // namespace rdkv_b200

using namespace rdkv_b200;

extern "C" RDKV_API size_t rdkv_cuda_decode_workspace(int32_t units, int32_t group, int32_t head_dim,
                                                      int32_t split) {
    if (units < 1 || group < 1 || head_dim < 1 || split <= 1) return 0;
    return sizeof(float) * (size_t)units * split * group * (2 + (size_t)head_dim);
}

extern "C" RDKV_API int rdkv_cuda_decode(const rdkv_decode_args* a, void* stream) {
    if (!a || !a->arena || !a->tile_offsets || !a->q || !a->out) return RDKV_EINVAL;
    if (a->units < 1 || a->group < 1 || a->group > 16 || a->head_dim < 1 || a->head_dim > 256)
        return RDKV_EINVAL;
    if (a->io_dtype != RDKV_F32 && a->io_dtype != RDKV_F16) return RDKV_EINVAL;
    if (a->zc_len && (!a->zc_k || !a->zc_v || a->zc_cap < 1)) return RDKV_EINVAL;
    const int split = a->split < 1 ? 1 : a->split;
    if (split > 1 && (!a->workspace ||
                      a->workspace_bytes < rdkv_cuda_decode_workspace(a->units, a->group, a->head_dim, split)))
        return RDKV_EINVAL;
    auto st = static_cast<cudaStream_t>(stream);
    const bool forced = a->kernel >= 2;
    const bool want_mma = forced || (a->kernel == 0 && split == 1);
    if (want_mma && mma_supported(a)) return launch_mma(a, st);
    if (forced) return RDKV_EINVAL;
    const int max_kslots = a->head_dim + 3 * 31 + 7;
    return a->io_dtype == RDKV_F32 ? launch_generic<float>(a, split, max_kslots, st)
                                   : launch_generic<__half>(a, split, max_kslots, st);
}

extern "C" RDKV_API int rdkv_cuda_decode_host(const rdkv_decode_args* a, const void* q_host,
                                              void* out_host, void* stream) {
    if (!a || !q_host || !out_host) return RDKV_EINVAL;
    const size_t elem = a->io_dtype == RDKV_F16 ? 2 : 4;
    const size_t bytes = (size_t)a->units * a->group * a->head_dim * elem;
    auto st = static_cast<cudaStream_t>(stream);
    RDKV_CUDA_TRY(cudaMemcpyAsync(const_cast<void*>(a->q), q_host, bytes, cudaMemcpyHostToDevice, st));
    if (int rc = rdkv_cuda_decode(a, stream)) return rc;
    RDKV_CUDA_TRY(cudaMemcpyAsync(out_host, a->out, bytes, cudaMemcpyDeviceToHost, st));
    return RDKV_OK;
}
