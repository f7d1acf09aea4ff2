/*
 * rdkv_cuda.h — C-ABI of the B200-native RDKV accelerator path.
 *
 * This is the drop-in boundary: plain pointers, sizes and
 * a cudaStream_t (passed as void*), no C++ or torch types. Every entry point
 * replaces a reference C++ entry point under /root/reference/proj/core:
 *
 *   rdkv_cuda_weights   attention_probe + token_weights + channel_weights
 *                       (cache.hpp:123-124, weights.hpp:26,34; called from
 *                       allocate_head pipeline.cpp:128-146)
 *   rdkv_cuda_allocate  head_budget + allocate_v + allocate_k + mckp_bisect
 *                       (pipeline.hpp:73-93, allocator.hpp:62-64;
 *                       allocate_model pipeline.hpp:109-111)
 *   rdkv_cuda_pack_plan / rdkv_cuda_pack
 *                       build_trizone / build_packed_model (trizone.hpp:80,136)
 *   rdkv_cuda_decode    packed_decode_step + fused_k_logits (trizone.hpp:84,89),
 *                       batched over every (batch, layer, KV head) tile
 *   rdkv_cuda_append    append_new_token (trizone.hpp:91)
 *   rdkv_tile_export    device tile -> the reference TriZoneCache segment
 *                       layout (PackedSegment payload bytes, QuantParams,
 *                       members/positions; trizone.hpp:34-78) for parity and
 *                       for RDKVP001 serialization
 *   rdkv_cuda_generate  synthetic-cache generator (counter-based replacement
 *                       for gen_synthetic_cache cache.hpp:138 at scale)
 *
 * Status codes map onto the reference's exception types (errors.hpp:9-16):
 * RDKV_EINVAL <-> std::invalid_argument, RDKV_ENUMERIC <-> rdkv::NumericError,
 * RDKV_EFORMAT <-> rdkv::FormatError. All device entry points are
 * asynchronous on the given stream; argument checks that need device data
 * are reported through the per-head rdkv_head_stats.status field.
 * Thread-safe across distinct streams; no hidden global stream or state.
 */
#ifndef RDKV_CUDA_H
#define RDKV_CUDA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define RDKV_API __attribute__((visibility("default")))

enum rdkv_status {
    RDKV_OK = 0,
    RDKV_EINVAL = 1,   /* std::invalid_argument */
    RDKV_ENUMERIC = 2, /* rdkv::NumericError */
    RDKV_EFORMAT = 3,  /* rdkv::FormatError */
    RDKV_ECUDA = 4     /* CUDA launch / runtime failure */
};

enum rdkv_dtype { RDKV_F32 = 0, RDKV_F16 = 1 };

/* Geometry of a batch of independent heads ("tiles"): one unit per
 * (batch, layer, KV head). K and V are [units][seq_len][head_dim], probe_q is
 * [units][group][probe_rows][head_dim] (the reference's probe_group view,
 * cache.hpp:102-104). kv_heads is the model's H_kv, used only for the
 * per-head budget split (pipeline.cpp:60-72). */
typedef struct {
    int32_t units;
    int32_t seq_len;
    int32_t head_dim;
    int32_t group;
    int32_t probe_rows;
    int32_t kv_heads;
} rdkv_shape;

/* BudgetSpec (pipeline.hpp:16-22) + ProbeConfig (cache.hpp:29-34) +
 * SolverConfig (allocator.hpp:12-19) + PipelineConfig (pipeline.hpp:59-63).
 * eps_v / eps_k hold DistortionTable::at(widths[i]) (quantizer.hpp:56-64). */
typedef struct {
    int32_t n_tokens;
    int32_t n_widths;
    double r_k;
    int32_t widths[8];
    double eps_v[8];
    double eps_k[8];
    int32_t window;
    int32_t pool_kernel;
    double tolerance;
    int32_t max_iterations;
    int32_t strict_budget;
    int32_t force_window_retain;
    int32_t reserved;
} rdkv_config;

/* HeadAllocation scalars (pipeline.hpp:44-57) + solver diagnostics. */
typedef struct {
    double lambda_v, lambda_k;
    double objective_v, objective_k;
    double achieved_bits;
    double avg_v, avg_k;
    int32_t v_converged, k_converged;
    int32_t n_kept, n_v16;
    int32_t k_bits_len; /* 0 when every token was evicted (pipeline.cpp:104) */
    int32_t status;     /* rdkv_status of this head */
} rdkv_head_stats;

/* ---- Stage 1: distortion weights ---------------------------------------- */
RDKV_API size_t rdkv_cuda_weights_workspace(const rdkv_shape* s, int32_t window);
/* w_t [units][seq_len], w_c [units][head_dim] (f32, device). */
RDKV_API int rdkv_cuda_weights(const void* k, const void* probe_q, int32_t dtype,
                               const rdkv_shape* s, int32_t window, int32_t pool_kernel,
                               float* w_t, float* w_c, void* workspace, size_t workspace_bytes,
                               void* stream);

/* ---- Stages 2/3: Lagrangian bisection per head --------------------------- */
/* v_bits [units][seq_len], k_bits [units][head_dim] (u8, device),
 * stats [units] (device). */
RDKV_API int rdkv_cuda_allocate(const float* w_t, const float* w_c, const rdkv_shape* s,
                                const rdkv_config* cfg, uint8_t* v_bits, uint8_t* k_bits,
                                rdkv_head_stats* stats, void* stream);

/* ---- TriZone packing ---------------------------------------------------- */
/* tile_offsets [units + 1] (int64, device): byte offset of every tile in the
 * arena, tile_offsets[units] = arena bytes. */
RDKV_API int rdkv_cuda_pack_plan(const uint8_t* v_bits, const uint8_t* k_bits,
                                 const rdkv_shape* s, int64_t* tile_offsets, void* stream);
/* head_status [units] (device, optional): RDKV_ENUMERIC when a kept row or
 * column holds a non-finite value (quantize_unit, quantizer.cpp:111-112). */
RDKV_API int rdkv_cuda_pack(const void* k, const void* v, int32_t dtype, const uint8_t* v_bits,
                            const uint8_t* k_bits, const rdkv_shape* s,
                            const int64_t* tile_offsets, uint8_t* arena, int32_t* head_status,
                            void* stream);

/* ---- Decode ------------------------------------------------------------- */
/* Maxima over the tiles of a packed arena (rdkv_cuda_decode_prepare). */
typedef struct {
    int32_t max_decode_bytes; /* largest per-tile decode region */
    int32_t max_slots;        /* largest token-slot count */
    int32_t max_zone_b_rows;  /* largest Zone B (16-bit V) row count */
    int32_t max_kq_slots;     /* largest quantised-K slot count */
    int32_t uniform2;         /* every tile: all kept V rows and K channels at 2 bits (2: and all d K channels kept) */
    int32_t n_uniform;        /* rdkv_cuda_decode_prepare_split: tiles of the uniform class (listed first in unit_ids) */
    int32_t uniform2_split;   /* the uniform2 value of that subset */
    int32_t mix24;            /* every tile: kept V rows and K channels at 2 or 4 bits only (no Zone B / k16 / 8-bit) */
    int32_t min_chunks24;     /* smallest per-tile chunk count of the mixed 2/4-bit chunked kernel (split-K bound) */
    int32_t max_krow_bytes24; /* largest K row of those tiles */
} rdkv_decode_plan;

/* rdkv_decode_args.flags: `out` lives in mapped host memory — the tensor-core
 * kernels write each output row with one TMA bulk store (128/256-B PCIe
 * writes) instead of per-lane stores (set by rdkv_cuda_decode_host). */
#define RDKV_DECODE_OUT_HOST 1
/* rdkv_decode_args.flags: zc_bound holds a host-known upper bound on every
 * zc_len[u] (e.g. the number of appends since packing); with a small bound the
 * uniform-2-bit kernel stages the Zone C rows with the packed tile instead of
 * running them as separate chunks. */
#define RDKV_DECODE_ZC_BOUND 2

typedef struct {
    const uint8_t* arena;
    const int64_t* tile_offsets;
    int32_t units;
    int32_t group;
    int32_t head_dim;
    int32_t io_dtype;   /* q / out element type: RDKV_F32 or RDKV_F16 */
    const void* q;      /* [units][group][head_dim] */
    void* out;          /* [units][group][head_dim] */
    const void* zc_k;   /* Zone C, fp16 [units][zc_cap][head_dim] (may be NULL) */
    const void* zc_v;
    const int32_t* zc_len; /* [units] (may be NULL) */
    int32_t zc_cap;
    int32_t split;      /* split-K factor (0 = automatic) */
    void* workspace;    /* split-K partials; rdkv_cuda_decode_workspace() bytes */
    size_t workspace_bytes;
    int32_t kernel;     /* 0 = automatic, 1 = generic CUDA-core, 2 = tensor-core (automatic body),
                           3 = tensor-core general body, 4 = tensor-core one-warp uniform-2-bit body */
    int32_t flags;      /* RDKV_DECODE_* bits (0 = default) */
    const int32_t* tile_decode_bytes; /* [units] device, from rdkv_cuda_decode_prepare (NULL: generic) */
    rdkv_decode_plan plan;
    int32_t zc_bound;   /* with RDKV_DECODE_ZC_BOUND: max over units of zc_len[u] */
    int32_t reserved2;
    const int32_t* unit_ids; /* [units] device, from rdkv_cuda_decode_prepare_split (NULL: no split) */
} rdkv_decode_args;

/* One-time scan of a packed arena: writes the per-tile decode sizes
 * (device, [units]) and the plan that enables the tensor-core kernel. */
RDKV_API int rdkv_cuda_decode_prepare(const uint8_t* arena, const int64_t* tile_offsets_host,
                                      int32_t units, int32_t* tile_decode_bytes,
                                      rdkv_decode_plan* plan, void* stream);
/* Same, and also writes unit_ids [units] (device): the units whose tiles are
 * uniform 2-bit (every kept V row and K channel at 2 bits, <= 160 slots)
 * first, then the rest (plan->n_uniform, plan->uniform2_split). With
 * rdkv_decode_args.unit_ids set, a step over a mixed arena runs the mixed
 * tiles on the general tensor-core body and the uniform ones on the fast
 * uniform-2-bit kernel (two launches) instead of everything on the former. */
RDKV_API int rdkv_cuda_decode_prepare_split(const uint8_t* arena, const int64_t* tile_offsets_host,
                                            int32_t units, int32_t* tile_decode_bytes, int32_t* unit_ids,
                                            rdkv_decode_plan* plan, void* stream);

/* Bytes of the split-K workspace for `split` parts (0 for split <= 1): the
 * partials [split][units][group][head_dim + 2] f32. */
RDKV_API size_t rdkv_cuda_decode_workspace(int32_t units, int32_t group, int32_t head_dim,
                                           int32_t split);
RDKV_API int rdkv_cuda_decode(const rdkv_decode_args* a, void* stream);
/* End-to-end variant: q_host / out_host are host buffers [units][group]
 * [head_dim]. Pinned (page-locked, UVA-mapped) buffers are used zero-copy:
 * the decode kernel reads q over PCIe with TMA bulk loads and writes out with
 * TMA bulk stores, overlapping both transfers with the step. Pageable buffers
 * are staged through a->q / a->out with cudaMemcpyAsync on `stream`. */
RDKV_API int rdkv_cuda_decode_host(const rdkv_decode_args* a, const void* q_host, void* out_host,
                                   void* stream);

/* Pipelined end-to-end decode (same contract as rdkv_cuda_decode_host).
 * The step is cut into `chunks` unit ranges; chunk c's q H2D (on the
 * context's copy-in stream), decode (on `stream`) and out D2H (on its
 * copy-out stream) overlap the neighbouring chunks', so the call costs about
 * one PCIe transfer instead of H2D + decode + D2H in series. The context is
 * caller-owned (two streams and per-chunk events, no global state); one
 * context serves one call at a time. The call forks from and joins back
 * into `stream`: work queued on `stream` before it is ordered before the
 * copies, and `stream` is ordered after the last D2H. */
typedef struct rdkv_decode_ctx rdkv_decode_ctx;
RDKV_API int rdkv_cuda_decode_ctx_create(int32_t chunks, rdkv_decode_ctx** ctx);
RDKV_API int rdkv_cuda_decode_ctx_destroy(rdkv_decode_ctx* ctx);
RDKV_API int rdkv_cuda_decode_host_pipelined(rdkv_decode_ctx* ctx, const rdkv_decode_args* a,
                                             const void* q_host, void* out_host, void* stream);

/* Sequence split across ranks (the optional cross-GPU merge): every rank
 * decodes its share of each uniform-2-bit tile — token chunks c with
 * c % world == rank (chunks of <= 160 slots, then 16-row Zone C chunks) — into
 * unnormalised partials [units][group][head_dim + 2] f32 (o, running max in
 * log2 units, weight sum). The caller gathers the world partials (e.g. NCCL
 * all-gather into [world][units][group][head_dim + 2]) and merges them with
 * rdkv_cuda_decode_merge into out [units][group][head_dim] (io_dtype). */
RDKV_API int rdkv_cuda_decode_partial(const rdkv_decode_args* a, int32_t rank, int32_t world, float* partial,
                                      void* stream);
RDKV_API int rdkv_cuda_decode_merge(const float* partials, int32_t nparts, int32_t units, int32_t group,
                                    int32_t head_dim, void* out, int32_t io_dtype, void* stream);

/* ---- Zone C ------------------------------------------------------------- */
/* Appends one K and one V row per unit (k_new/v_new [units][head_dim] of
 * dtype) at position zc_len[u], then increments zc_len[u]. */
RDKV_API int rdkv_cuda_append(void* zc_k, void* zc_v, int32_t* zc_len, int32_t zc_cap,
                              const void* k_new, const void* v_new, int32_t dtype, int32_t units,
                              int32_t head_dim, void* stream);

/* ---- Synthetic inputs ---------------------------------------------------- */
/* Counter-based N(0,1)-like generator, every value FP16-representable:
 * value(seed, tensor, i) reproducible on the CPU.
 * tensor: 0 = K, 1 = V, 2 = probe Q. first_index = global element index of
 * out[0] (lets callers generate any slice). Optional heavy hitters: every
 * `hh_stride`-th token of K (tensor 0) gets hh_boost added to all channels
 * of its row; outlier_channels leading K channels are multiplied by
 * outlier_scale (fp16-rounded). */
RDKV_API int rdkv_cuda_generate(void* out, int32_t dtype, uint64_t seed, int32_t tensor,
                                uint64_t first_index, uint64_t count, int32_t head_dim,
                                int32_t seq_len, int32_t outlier_channels, float outlier_scale,
                                int32_t hh_stride, float hh_boost, void* stream);


/* ---- Single-function entry points (C++ drop-in layer, include/rdkv/cuda.hpp) */
/* attention_probe (cache.cpp:140-184): a[r][t] = softmax_t(q_r . k_t / sqrt(d))
 * over t <= offsets[r], exactly 0 beyond; q [rows][d], k [t_len][d] f32,
 * offsets [rows] int32, a [rows][t_len] fp64 (all device). EINVAL when an
 * offset is outside [0, t_len) (cache.cpp:162-164). */
RDKV_API size_t rdkv_cuda_attention_probe_workspace(int32_t rows, int32_t t_len);
RDKV_API int rdkv_cuda_attention_probe(const float* q, int32_t rows, const float* k, int32_t t_len,
                                       int32_t d, const int32_t* offsets, double* a, void* workspace,
                                       size_t workspace_bytes, void* stream);
/* token_weights (weights.cpp:25-46): a = heads x [rows][t_len] fp64 stacked;
 * raw_scratch [t_len] f32; out [t_len] f32 pooled weights. */
RDKV_API int rdkv_cuda_token_weights(const double* a, int32_t heads, int32_t rows, int32_t t_len,
                                     int32_t pool_kernel, float* raw_scratch, float* out, void* stream);
/* moving_average (weights.cpp:8-23). */
RDKV_API int rdkv_cuda_moving_average(const float* raw, int32_t n, int32_t kernel, float* out,
                                      void* stream);
/* channel_weights (weights.cpp:69-91): q [q_rows][d], k [k_rows][d] -> out [d]. */
RDKV_API int rdkv_cuda_channel_weights(const float* q, int32_t q_rows, const float* k, int32_t k_rows,
                                       int32_t d, float* out, void* stream);

typedef struct {
    double lambda;
    double achieved_avg_bits;
    double objective;
    int32_t converged;
    int32_t status; /* RDKV_EINVAL: a weight is negative or non-finite */
} rdkv_bisect_result;

/* mckp_bisect (allocator.cpp:135-216) over `instances` weight vectors of
 * length n (device, [instances][n]); widths/eps (host) = the argmin table
 * (make_argmin_table, allocator.cpp:32-37); bits [instances][n] u8 and
 * results [instances] (device). */
RDKV_API int rdkv_cuda_mckp_bisect(const float* weights, int32_t instances, int32_t n,
                                   const int32_t* widths, const double* eps, int32_t n_widths,
                                   double target_avg_bits, double tolerance, int32_t max_iterations,
                                   int32_t strict_budget, uint8_t* bits, rdkv_bisect_result* results,
                                   void* stream);

/* quantize_unit (quantizer.cpp:104-131) over `units` rows of `len` f32
 * values (device): codes [units][len], scale/zero_point [units],
 * status [units] (RDKV_ENUMERIC for a non-finite unit). */
RDKV_API int rdkv_cuda_quantize_units(const float* values, int32_t units, int32_t len, int32_t bits,
                                      uint8_t* codes, float* scale, int64_t* zero_point,
                                      int32_t* status, void* stream);

/* pack_bits (trizone.cpp:59-75; reference trizone.hpp:16): n codes
 * (< 2^bits each) -> ceil(n * bits / 8) bytes in the reference's quarter- /
 * half-split layout, 16-byte vectorised stores. *status (device) = RDKV_EINVAL
 * when a code overflows the bit-width ("pack_bits: code overflows bit-width"),
 * else RDKV_OK. bits must be 2, 4 or 8. */
RDKV_API int rdkv_cuda_pack_bits(const uint8_t* codes, int64_t n, int32_t bits, uint8_t* out,
                                 int32_t* status, void* stream);
/* unpack_bits (trizone.cpp:76-88; reference trizone.hpp:17): the first
 * logical_len codes of `bytes` (nbytes long). RDKV_EINVAL when bits is not
 * 2/4/8 or the buffer is too short for logical_len codes. */
RDKV_API int rdkv_cuda_unpack_bits(const uint8_t* bytes, int64_t nbytes, int32_t bits, int64_t logical_len,
                                   uint8_t* out, void* stream);

/* fused_k_logits (trizone.cpp:210-249) per token slot of every tile:
 * q [units][group][head_dim] f32 -> logits [units][group][max_slots] f32
 * (slot order; NaN for pad slots). max_slots / max_kslots from the plan. */
RDKV_API int rdkv_cuda_tile_logits(const uint8_t* arena, const int64_t* tile_offsets, int32_t units,
                                   int32_t group, int32_t head_dim, const float* q, int32_t max_slots,
                                   int32_t max_kslots, float* logits, void* stream);

/* dual_bound (allocator.cpp:218-246) for every instance of a batched
 * rdkv_cuda_mckp_bisect, at that instance's final lambda (solved[i].lambda,
 * device): weights [instances][n] f32, total_budget = target · n (the
 * run_sweep budget, sweep.cpp:95-101), out [instances] (device). status
 * RDKV_EINVAL per instance for a negative / non-finite weight or lambda. */
typedef struct {
    double g_lambda;
    double primal;
    double gap;
    int32_t feasible;
    int32_t status;
} rdkv_dual_bound_result;

RDKV_API int rdkv_cuda_dual_bound(const float* weights, int32_t instances, int32_t n,
                                  const int32_t* widths, const double* eps, int32_t n_widths,
                                  const rdkv_bisect_result* solved, double total_budget,
                                  rdkv_dual_bound_result* out, void* stream);

/* ---- Host-side tile inspection ----------------------------------------- */
/* Tile header fields. */
typedef struct {
    int32_t n_kept;
    int32_t rows[4];     /* V rows at 2,4,8,16 bits */
    int32_t chans[4];    /* K channels at 2,4,8,16 bits */
    int32_t kslots, krow_bytes, nslot;
    int64_t total_bytes;
    int64_t decode_bytes; /* bytes the decode kernel reads from this tile */
} rdkv_tile_info;

RDKV_API int rdkv_tile_info_get(const uint8_t* tile_host, rdkv_tile_info* info);

/* Canonical export of one tile (host copy of its bytes) in the reference's
 * TriZoneCache terms; same layout as oracle's orc_tz_canon:
 *   kept[n]; vcodes[n*d] (kept order); vscale/vzero[n]; kcodes[d*n]
 *   channel-major; kscale/kzero[d]; vfp[n*d] Zone B rows; kfp[n*d] k16;
 *   payload = reference PackedSegment payloads (V 2,4,8 then K 2,4,8);
 *   segtab[6*6] (side, bits, rows, logical_len, pad_count, nbytes);
 *   perm[d] channel_perm. */
RDKV_API int rdkv_tile_export(const uint8_t* tile_host, int32_t head_dim, int32_t* kept,
                              uint8_t* vcodes, float* vscale, int64_t* vzero, uint8_t* kcodes,
                              float* kscale, int64_t* kzero, float* vfp, float* kfp,
                              uint8_t* payload, int32_t* segtab, int32_t* nseg, int32_t* perm,
                              int32_t* nperm);
RDKV_API size_t rdkv_tile_export_payload_bytes(const uint8_t* tile_host, int32_t head_dim);


/* Canonical import: the inverse of rdkv_tile_export — builds a device tile
 * (host bytes) from the reference's TriZoneCache content: kept [n] ascending
 * token ids, vbits_kept [n] in {2,4,8,16}, vcodes [n*d] (kept order),
 * vscale/vzero [n], vfp [n*d] Zone B rows, kbits [d] in {0,2,4,8,16},
 * kcodes [d*n] channel-major, kscale/kzero [d], kfp [n*d] k16 values. */
RDKV_API size_t rdkv_tile_import_bytes(int32_t d, int32_t n, const uint8_t* vbits_kept,
                                       const uint8_t* kbits);
RDKV_API int rdkv_tile_import(int32_t d, int32_t n, const int32_t* kept, const uint8_t* vbits_kept,
                              const uint8_t* vcodes, const float* vscale, const int64_t* vzero,
                              const float* vfp, const uint8_t* kbits, const uint8_t* kcodes,
                              const float* kscale, const int64_t* kzero, const float* kfp,
                              uint8_t* tile, size_t tile_bytes);

/* ---- RDKVC001 cache container straight to device (cache.cpp:228-287) ------ */
/* Header of a container written by save_cache (cache.cpp:205-226): magic
 * "RDKVC001", u32le header length, JSON header, then f32 K, V, probe_Q payload
 * in layer-major, head-major, row-major order — which is already the device
 * unit order: K/V [L*H_kv][T][d], probe_Q [L*H_kv][g][S_w][d] (unit = l*H_kv+h). */
typedef struct {
    int32_t layers, q_heads, kv_heads, head_dim, seq_len, probe_window;
    int64_t payload_offset; /* byte offset of the K payload */
    int64_t payload_bytes;  /* 4 * (2*L*H_kv*T*d + L*H_q*S_w*d) */
} rdkv_cache_header;

/* Host only. Replaces the header half of load_cache (cache.cpp:228-267) with
 * its error behaviour: RDKV_EFORMAT for a bad magic, implausible/truncated
 * header, invalid JSON, missing/mistyped fields, dtype != "f32", S_w out of
 * range, or a file whose size is not header + payload (truncated / trailing
 * bytes, cache.cpp:275-283); RDKV_EINVAL when CacheShape::validate rejects the
 * shape (cache.cpp:95-105). */
RDKV_API int rdkv_cache_read_header(const char* path, rdkv_cache_header* header);

/* Streams the payload of `path` (header from rdkv_cache_read_header) into
 * device k, v [L*H_kv][T][d] and probe_q [L*H_kv][g][S_w][d] as `dtype`
 * (RDKV_F32 bit-exact, RDKV_F16 round-to-nearest), through pinned double
 * buffers overlapping the file reads with the H2D copies. Returns
 * RDKV_ENUMERIC when an entry is non-finite (KVCache::validate,
 * cache.cpp:114-130) or overflows fp16. The reference accepts every finite
 * f32; |x| > 65504 is rejected only because an fp16 target cannot hold it
 * (load as RDKV_F32 to accept exactly the reference's inputs). Returns after
 * `stream` has finished the copies. */
RDKV_API int rdkv_cuda_cache_load(const char* path, const rdkv_cache_header* header, void* k,
                                  void* v, void* probe_q, int32_t dtype, void* stream);

/* ---- ε calibration (calibrate_epsilon, quantizer.cpp:200-284) ------------ */
/* Per-job partials for one cache: values = V (granularity 0, token units =
 * rows of d) or K (granularity 1, channel units = columns of seq_len), device
 * [jobs][seq_len][head_dim] with job = l*H_kv + h (a cache's job order).
 * widths [n_widths]: the BitSet (validate_relaxed rules, else RDKV_EINVAL).
 * err_sum [jobs][max(1, #finite widths)] f64 and count [jobs] i64 (device):
 * per job, the sum of unit NMSEs in unit order for each finite width
 * (ascending) and the number of nonzero-energy units. RDKV_ENUMERIC when a
 * value is non-finite. Synchronizes `stream`. */
RDKV_API size_t rdkv_cuda_calibrate_workspace(int32_t jobs, int32_t seq_len, int32_t head_dim,
                                              int32_t granularity, int32_t n_widths);
RDKV_API int rdkv_cuda_calibrate_partials(const void* values, int32_t dtype, int32_t jobs,
                                          int32_t seq_len, int32_t head_dim, int32_t granularity,
                                          const int32_t* widths, int32_t n_widths, double* err_sum,
                                          int64_t* count, void* workspace, size_t workspace_bytes,
                                          void* stream);
/* Host: merges host copies of the partials of every job of every cache (in
 * cache, then job order) into eps [n_widths] (eps(0) = 1, eps(16) = 0) and the
 * unit count. RDKV_EINVAL for an empty sample or a table that fails
 * DistortionTable::validate; RDKV_ENUMERIC when every unit has zero norm. */
RDKV_API int rdkv_calibrate_finalize(const double* err_sum, const int64_t* count, int32_t jobs,
                                     const int32_t* widths, int32_t n_widths, double* eps,
                                     int64_t* unit_count);

RDKV_API const char* rdkv_status_string(int status);
RDKV_API int rdkv_version(void);

#ifdef __cplusplus
}
#endif
#endif /* RDKV_CUDA_H */
