// rdkv/cuda.hpp — C++ drop-in for the reference's allocate -> pack -> decode
// API, backed by the sm_100a kernels of librdkv_b200.so (include/rdkv_cuda.h).
//
// Every function below has the signature, argument meaning, return type and
// exception behaviour of the reference function it names (namespace `rdkv`,
// proj/core/include/rdkv/*.hpp); a caller switches by qualifying the call
// with `rdkv::cuda::` (or by `namespace rdkv_impl = rdkv::cuda;`). Inputs are
// the reference's own host types; results are returned as the reference's
// own value types, so everything downstream (storage_report, save_packed,
// allocation_to_json, the CLI) keeps working unchanged.
//
// These host-buffer wrappers upload their inputs, run the device kernels and
// download the result on every call — they exist for drop-in parity. The
// performance API is DevicePackedModel (device-resident tiles, one launch per
// decode step for every (layer, KV head) tile and every query head).
//
// Link: -lrdkv_cuda_dropin (paper_2605_08317_b200/_lib), which pulls in
// librdkv_b200.so. The drop-in itself needs only the reference HEADERS; it
// calls no reference function.
#pragma once

#include <cstdint>
#include <memory>
#include <span>
#include <vector>

#include "rdkv/allocator.hpp"
#include "rdkv/cache.hpp"
#include "rdkv/errors.hpp"
#include "rdkv/pipeline.hpp"
#include "rdkv/quantizer.hpp"
#include "rdkv/sweep.hpp"
#include "rdkv/trizone.hpp"
#include "rdkv/weights.hpp"

namespace rdkv::cuda {

// ---- Stage 1: distortion weights ------------------------------------------
// cache.hpp:123-124 / cache.cpp:140-184
AttentionMatrix attention_probe(MatrixView q_window, MatrixView k, std::span<const int> causal_offsets);
// weights.hpp:24 / weights.cpp:8-23
std::vector<float> moving_average(std::span<const float> raw, int kernel);
// weights.hpp:26 / weights.cpp:25-46
WeightVector token_weights(std::span<const AttentionMatrix> heads, int group, int pool_kernel);
// weights.hpp:34 / weights.cpp:69-91
WeightVector channel_weights(MatrixView q, MatrixView k);

// ---- Stages 2/3: allocation -------------------------------------------------
// allocator.hpp:62-64 / allocator.cpp:135-216
DiscreteAllocation mckp_bisect(std::span<const float> weights, const DistortionTable& eps,
                               double target_avg_bits, const BitSet& bits = {},
                               const SolverConfig& cfg = {});
// pipeline.hpp:73-75 / pipeline.cpp:74-94 — Stage 2 (device bisection over the tokens)
VAllocation allocate_v(const WeightVector& token_w, const DistortionTable& eps_v, double v_budget_bits,
                       int head_dim, const BitSet& bits, const SolverConfig& cfg);
// pipeline.hpp:79-81 / pipeline.cpp:96-112 — Stage 3 (device bisection over the channels)
DiscreteAllocation allocate_k(const WeightVector& channel_w, const DistortionTable& eps_k,
                              double k_budget_bits, int kept_count, const BitSet& bits,
                              const SolverConfig& cfg);
// pipeline.hpp:91-93 / pipeline.cpp:114-183
HeadAllocation allocate_head(const KVCache& cache, int layer, int kv_head, const BudgetSpec& spec,
                             const DistortionTable& eps_v, const DistortionTable& eps_k,
                             const PipelineConfig& cfg);
// pipeline.hpp:109-111 / pipeline.cpp:191-207 — every (layer, KV head) in one launch
ModelAllocation allocate_model(const KVCache& cache, const BudgetSpec& spec,
                               const DistortionTable& eps_v, const DistortionTable& eps_k,
                               const PipelineConfig& cfg);

// ---- TriZone packing --------------------------------------------------------
// trizone.hpp:16-17 / trizone.cpp:59-88 (device kernels, 16-byte vectorised stores)
std::vector<std::uint8_t> pack_bits(std::span<const std::uint8_t> codes, int bits);
std::vector<std::uint8_t> unpack_bits(std::span<const std::uint8_t> bytes, int bits, int logical_len);
// quantizer.hpp:41 / quantizer.cpp:104-131
QuantizedUnit quantize_unit(std::span<const float> values, int bits);
// trizone.hpp:80 / trizone.cpp:91-208
TriZoneCache build_trizone(MatrixView k, MatrixView v, const HeadAllocation& alloc);
// trizone.hpp:136 / trizone.cpp:478-490 — every head packed in one launch
PackedModel build_packed_model(const KVCache& cache, const ModelAllocation& alloc);

// ---- Decode -----------------------------------------------------------------
// trizone.hpp:84 / trizone.cpp:210-249 (f32 accumulation on device)
std::vector<double> fused_k_logits(std::span<const float> q, const TriZoneCache& cache);
// trizone.hpp:89 / trizone.cpp:251-305 (tensor-core / CUDA-core kernels; fp16
// storage of Zone B, k16 and Zone C: <= 1e-3 relative to the reference)
std::vector<double> packed_decode_step(std::span<const float> q, const TriZoneCache& cache);
// trizone.hpp:91 / trizone.cpp:307-314 (host container: same as the reference)
void append_new_token(TriZoneCache& cache, std::span<const float> k, std::span<const float> v);

// ---- §8(f): rate sweep, dual bound, ε calibration ----------------------------
// allocator.hpp:68-69 / allocator.cpp:218-246
DualBound dual_bound(std::span<const float> weights, const DistortionTable& eps, double lambda,
                     double total_budget, const BitSet& bits = {});
// sweep.hpp:31-34 / sweep.cpp:40-114 (weights once per cache, batched strict
// bisection + dual bound of every (layer, KV head) per grid value)
SweepResult run_sweep(std::span<const KVCache> sequences, std::span<const double> grid, const DistortionTable& eps_v,
                      const DistortionTable& eps_k, const BitSet& bits, const SolverConfig& solver,
                      const ProbeConfig& probe);
// quantizer.hpp:69-70 / quantizer.cpp:200-284
DistortionTable calibrate_epsilon(std::span<const KVCache> caches, Granularity granularity, const BitSet& bits = {});

// ---- Device-resident performance API ---------------------------------------
// All (layer, KV head) tiles of a PackedModel in one device arena, plus a
// device Zone C. decode() runs ONE kernel launch for every tile and every
// grouped query head (the batched form of packed_decode_step).
class DevicePackedModel {
public:
    // Pack on the device straight from the cache (no host round trip).
    static DevicePackedModel build(const KVCache& cache, const ModelAllocation& alloc,
                                   int zone_c_capacity = 0);
    // Upload a host PackedModel (e.g. from load_packed) into device tiles.
    static DevicePackedModel upload(const PackedModel& model, int zone_c_capacity = 0);

    DevicePackedModel(DevicePackedModel&&) noexcept;
    DevicePackedModel& operator=(DevicePackedModel&&) noexcept;
    ~DevicePackedModel();

    const CacheShape& shape() const;
    int units() const;                 // layers * kv_heads
    std::size_t arena_bytes() const;   // device bytes of the packed tiles
    std::size_t decode_bytes() const;  // bytes one decode step reads (roofline numerator)

    // q: [layers][q_heads][head_dim] f32 -> out: same shape. Equals
    // packed_decode_step(q[l][h], at(l, h / group)) for every (l, h).
    std::vector<float> decode(std::span<const float> q) const;
    // Zone C: one K and V row per (layer, KV head): [layers][kv_heads][head_dim].
    void append(std::span<const float> k, std::span<const float> v);
    // Host copy of the packed tiles in the reference's TriZoneCache terms
    // (Zone B / k16 / Zone C values as stored on device: fp16-rounded).
    PackedModel download() const;

private:
    struct Impl;
    explicit DevicePackedModel(std::unique_ptr<Impl> impl);
    std::unique_ptr<Impl> impl_;
};

}  // namespace rdkv::cuda
