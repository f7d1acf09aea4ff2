// decode_mma.cu — K4 tensor-core path (int8 mma.sync with fused dequant).
// Placeholder until the tensor-core kernel lands: every layout routes to the
// generic CUDA-core kernel.
#include "common.cuh"

namespace rdkv_b200 {
bool mma_supported(const rdkv_decode_args*) { return false; }
int launch_mma(const rdkv_decode_args*, cudaStream_t) { return RDKV_EINVAL; }
}  // namespace rdkv_b200
