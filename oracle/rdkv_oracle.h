/*
 * rdkv_oracle.h — CPU restatement of the RDKV allocate -> pack -> decode path.
 *
 * TEST INFRASTRUCTURE ONLY. This library is the parity checker for the
 * B200 kernels in paper_2605_08317_b200/. Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline leg may load it. The product path never links
 * or calls it.
 *
 * Every function restates one reference function (file:line under
 * /root/reference/proj/core/src) in plain C with the same arithmetic order
 * (fp64, no fused multiply-add: compiled with -ffp-contract=off).
 * Parity pinning: tests/test_oracle.py checks this library against the
 * reference's own known-answer tests and against the
 * compiled reference (oracle/_ref, via tests/golden/ fixtures).
 *
 * Error convention: functions return 0 on success, ORC_EINVAL for what the
 * reference throws as std::invalid_argument and ORC_ENUMERIC for
 * rdkv::NumericError (errors.hpp:14-16).
 */
#ifndef RDKV_ORACLE_H
#define RDKV_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { ORC_OK = 0, ORC_EINVAL = 1, ORC_ENUMERIC = 2, ORC_EFORMAT = 3 };

/* Same memory layout as rdkv_config in include/rdkv_cuda.h (one ctypes
 * struct drives both). BudgetSpec (pipeline.hpp:16-22), ProbeConfig
 * (cache.hpp:29-34), SolverConfig (allocator.hpp:12-19), PipelineConfig
 * (pipeline.hpp:59-63). eps_v/eps_k are aligned with widths[]. */
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
} orc_config;

/* HeadAllocation scalars (pipeline.hpp:44-57) plus solver diagnostics. */
typedef struct {
    double lambda_v, lambda_k;
    double objective_v, objective_k;
    double achieved_bits;
    double avg_v, avg_k;
    int32_t v_converged, k_converged;
    int32_t n_kept, n_v16;
    int32_t k_bits_len; /* 0 when every token was evicted (pipeline.cpp:104) */
    int32_t status;
} orc_head_stats;

/* ---- data generation (cache.cpp:24-50, 301-342) ---- */
int orc_gen_synthetic(uint64_t seed, int layers, int q_heads, int kv_heads, int head_dim,
                      int seq_len, int probe_window, int outlier_channels,
                      double outlier_scale, float* k, float* v, float* probe_q);
/* raw NormalSampler stream (used for query vectors in tests) */
void orc_normal_stream(uint64_t seed, float* out, size_t n);

/* K0 counter-based generator (CPU restatement of csrc/generate.cu) */
void orc_gen_counter(float* out, uint64_t seed, int tensor, uint64_t first, uint64_t count, int d,
                     int seq_len, int outlier_channels, float outlier_scale, int hh_stride,
                     float hh_boost);

/* ---- stage 1 (cache.cpp:140-184, weights.cpp:8-46, 69-91) ---- */
int orc_attention_probe(const float* q, int rows, const float* k, int t_len, int d,
                        const int* offsets, double* a);
int orc_moving_average(const float* raw, int n, int kernel, float* out);
int orc_token_weights(const double* a, int heads, int rows, int t_len, int pool_kernel,
                      float* out);
int orc_channel_weights(const float* q, int q_rows, const float* k, int k_rows, int d,
                        float* out);

/* ---- quantizer (quantizer.cpp:104-131) ---- */
int orc_quantize_unit(const float* values, int n, int bits, uint8_t* codes, float* scale,
                      int64_t* zero_point);

/* ---- allocator (allocator.cpp:32-61, 135-216, 301-311) ---- */
int orc_per_unit_argmin(double weight, const int* widths, const double* eps, int n_widths,
                        double lambda);
int orc_mckp_bisect(const float* w, int n, const int* widths, const double* eps, int n_widths,
                    double target, double tolerance, int max_iterations, int strict_budget,
                    int* bits, double* lambda, double* avg, double* objective, int* converged);

/* ---- pipeline (pipeline.cpp:60-183) ---- */
int orc_head_budget(int n_tokens, double r_k, int head_dim, int kv_heads, double* head_bits,
                    double* v_bits, double* k_bits, int* sub_token);
/* probe_group: the g query heads of this KV head, each [probe_rows x d]. */
int orc_allocate_head(const float* k, const float* probe_group, int t_len, int d, int group,
                      int probe_rows, int kv_heads, const orc_config* cfg, int* v_bits,
                      int* k_bits, float* v_weights, float* k_weights, orc_head_stats* st);

/* ---- TriZone (trizone.cpp:26-75, 91-314) ---- */
int orc_padded_len(int len, int bits);
int orc_packed_row_bytes(int len, int bits);
int orc_pack_bits(const uint8_t* codes, int n, int bits, uint8_t* out);

typedef struct orc_trizone orc_trizone;
/* k_bits may be NULL when every token is evicted */
orc_trizone* orc_tz_build(const float* k, const float* v, int t_len, int d, const int* v_bits,
                          const int* k_bits, int* status);
void orc_tz_free(orc_trizone* tz);
int orc_tz_append(orc_trizone* tz, const float* k, const float* v);
int orc_tz_fused_logits(const orc_trizone* tz, const float* q, double* out);
int orc_tz_decode(const orc_trizone* tz, const float* q, double* out);
int orc_tz_n_kept(const orc_trizone* tz);
size_t orc_tz_payload_bytes(const orc_trizone* tz);
/* Canonical export shared with the reference shim and the GPU exporter:
 *   kept[n_kept]; vcodes[n_kept*d] (kept order, 0 for 16-bit rows);
 *   vscale/vzero[n_kept]; kcodes[d*n_kept] channel-major; kscale/kzero[d];
 *   vfp[n_kept*d] Zone B rows (0 elsewhere); kfp[n_kept*d] k16 columns;
 *   payload = concatenated reference segment payloads (V 2,4,8 then K 2,4,8);
 *   segtab[6*6] rows (side 0=V/1=K, bits, rows, logical_len, pad_count, nbytes);
 *   perm[d] channel permutation (nperm entries). */
int orc_tz_canon(const orc_trizone* tz, int* kept, uint8_t* vcodes, float* vscale,
                 int64_t* vzero, uint8_t* kcodes, float* kscale, int64_t* kzero, float* vfp,
                 float* kfp, uint8_t* payload, int* segtab, int* nseg, int* perm, int* nperm);
/* Segment-level decode restated directly from a canonical export, used to
 * check the exporter independently (trizone.cpp:210-305). */

/* ---- dense oracles (trizone.cpp:364-443) ---- */
int orc_dense_decode(const float* q, const float* k_rows, const float* v_rows, int n, int d,
                     double* out);

#ifdef __cplusplus
}
#endif
#endif
