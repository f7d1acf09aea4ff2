/*
 * rdkv_oracle.c — CPU restatement of the RDKV hot path. TEST INFRASTRUCTURE
 * ONLY (see rdkv_oracle.h). Compiled with -ffp-contract=off so every
 * multiply-add rounds twice, exactly like the reference objects (which carry
 * no FMA instructions).
 *
 * Reference citations are file:line under /root/reference/proj/core/src.
 */
#include "rdkv_oracle.h"

#include <float.h>
#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------------ */
/* mt19937_64 + Box-Muller: NormalSampler, cache.cpp:24-50                   */
/* ------------------------------------------------------------------------ */

typedef struct {
    uint64_t mt[312];
    int idx;
    int have_spare;
    double spare;
} orc_rng;

static void rng_seed(orc_rng* r, uint64_t seed) {
    r->mt[0] = seed;
    for (int i = 1; i < 312; ++i) {
        r->mt[i] = 6364136223846793005ULL * (r->mt[i - 1] ^ (r->mt[i - 1] >> 62)) + (uint64_t)i;
    }
    r->idx = 312;
    r->have_spare = 0;
    r->spare = 0.0;
}

static uint64_t rng_next64(orc_rng* r) {
    static const uint64_t kA = 0xB5026F5AA96619E9ULL;
    static const uint64_t kUpper = 0xFFFFFFFF80000000ULL;
    static const uint64_t kLower = 0x7FFFFFFFULL;
    if (r->idx >= 312) {
        for (int i = 0; i < 312; ++i) {
            uint64_t x = (r->mt[i] & kUpper) | (r->mt[(i + 1) % 312] & kLower);
            uint64_t xa = x >> 1;
            if (x & 1ULL) xa ^= kA;
            r->mt[i] = r->mt[(i + 156) % 312] ^ xa;
        }
        r->idx = 0;
    }
    uint64_t y = r->mt[r->idx++];
    y ^= (y >> 29) & 0x5555555555555555ULL;
    y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
    y ^= (y << 37) & 0xFFF7EEE000000000ULL;
    y ^= (y >> 43);
    return y;
}

/* uniform01: cache.cpp:43-46 */
static double rng_uniform01(orc_rng* r) {
    return ((double)(rng_next64(r) >> 11) + 0.5) * 0x1p-53;
}

/* NormalSampler::next: cache.cpp:28-40 */
static float rng_normal(orc_rng* r) {
    if (r->have_spare) {
        r->have_spare = 0;
        return (float)r->spare;
    }
    double u1 = rng_uniform01(r);
    double u2 = rng_uniform01(r);
    double rad = sqrt(-2.0 * log(u1));
    double theta = 2.0 * 3.141592653589793238462643383279502884 * u2;
    r->spare = rad * sin(theta);
    r->have_spare = 1;
    return (float)(rad * cos(theta));
}

void orc_normal_stream(uint64_t seed, float* out, size_t n) {
    orc_rng r;
    rng_seed(&r, seed);
    for (size_t i = 0; i < n; ++i) out[i] = rng_normal(&r);
}

/* gen_synthetic_cache: cache.cpp:301-342. One serial stream, K of every
 * layer, then V of every layer, then probe_Q; then outlier K channels. */
int orc_gen_synthetic(uint64_t seed, int layers, int q_heads, int kv_heads, int d, int t_len,
                      int probe_window, int outlier_channels, double outlier_scale, float* k,
                      float* v, float* probe_q) {
    if (layers < 1 || d < 1 || t_len < 1 || q_heads < 1 || kv_heads < 1) return ORC_EINVAL;
    if (q_heads % kv_heads != 0) return ORC_EINVAL;
    if (probe_window < 1 || probe_window > t_len) return ORC_EINVAL;
    if (outlier_channels < 0 || outlier_channels > d) return ORC_EINVAL;
    if (!isfinite(outlier_scale)) return ORC_EINVAL;
    orc_rng r;
    rng_seed(&r, seed);
    const size_t kv_n = (size_t)layers * kv_heads * t_len * d;
    const size_t q_n = (size_t)layers * q_heads * probe_window * d;
    for (size_t i = 0; i < kv_n; ++i) k[i] = rng_normal(&r);
    for (size_t i = 0; i < kv_n; ++i) v[i] = rng_normal(&r);
    for (size_t i = 0; i < q_n; ++i) probe_q[i] = rng_normal(&r);
    const float scale = (float)outlier_scale;
    const size_t rows = (size_t)layers * kv_heads * t_len;
    for (size_t row = 0; row < rows; ++row) {
        for (int c = 0; c < outlier_channels; ++c) k[row * d + c] *= scale;
    }
    return ORC_OK;
}

/* ------------------------------------------------------------------------ */
/* Stage 1                                                                   */
/* ------------------------------------------------------------------------ */

/* attention_probe: cache.cpp:140-184 */
int orc_attention_probe(const float* q, int rows, const float* k, int t_len, int d,
                        const int* offsets, double* a) {
    for (size_t i = 0; i < (size_t)rows * d; ++i)
        if (!isfinite(q[i])) return ORC_ENUMERIC;
    for (size_t i = 0; i < (size_t)t_len * d; ++i)
        if (!isfinite(k[i])) return ORC_ENUMERIC;
    memset(a, 0, sizeof(double) * (size_t)rows * t_len);
    const double inv_sqrt_d = 1.0 / sqrt((double)d);
    double* logits = (double*)malloc(sizeof(double) * (size_t)t_len);
    for (int r = 0; r < rows; ++r) {
        const int off = offsets[r];
        if (off < 0 || off >= t_len) {
            free(logits);
            return ORC_EINVAL;
        }
        const float* qr = q + (size_t)r * d;
        double mx = -INFINITY;
        for (int t = 0; t <= off; ++t) {
            const float* kt = k + (size_t)t * d;
            double dot = 0.0;
            for (int c = 0; c < d; ++c) dot += (double)qr[c] * kt[c];
            logits[t] = dot * inv_sqrt_d;
            if (logits[t] > mx) mx = logits[t];
        }
        double denom = 0.0;
        for (int t = 0; t <= off; ++t) {
            logits[t] = exp(logits[t] - mx);
            denom += logits[t];
        }
        double* row = a + (size_t)r * t_len;
        for (int t = 0; t <= off; ++t) row[t] = logits[t] / denom;
    }
    free(logits);
    return ORC_OK;
}

/* moving_average: weights.cpp:8-23 (zero padding, divide by full kernel) */
int orc_moving_average(const float* raw, int n, int kernel, float* out) {
    if (kernel < 1 || kernel % 2 == 0) return ORC_EINVAL;
    const int half = kernel / 2;
    for (int i = 0; i < n; ++i) {
        double acc = 0.0;
        const int lo = i - half < 0 ? 0 : i - half;
        const int hi = i + half > n - 1 ? n - 1 : i + half;
        for (int j = lo; j <= hi; ++j) acc += raw[j];
        out[i] = (float)(acc / kernel);
    }
    return ORC_OK;
}

/* token_weights: weights.cpp:25-46 — heads outer, rows inner, fp64 column
 * sums, cast to f32, then pooled. a is [heads][rows][t_len]. */
int orc_token_weights(const double* a, int heads, int rows, int t_len, int pool_kernel,
                      float* out) {
    if (heads < 1) return ORC_EINVAL;
    double* raw = (double*)calloc((size_t)t_len, sizeof(double));
    float* rawf = (float*)malloc(sizeof(float) * (size_t)t_len);
    for (int h = 0; h < heads; ++h) {
        for (int r = 0; r < rows; ++r) {
            const double* row = a + ((size_t)h * rows + r) * t_len;
            for (int t = 0; t < t_len; ++t) raw[t] += row[t];
        }
    }
    for (int t = 0; t < t_len; ++t) rawf[t] = (float)raw[t];
    int st = orc_moving_average(rawf, t_len, pool_kernel, out);
    free(raw);
    free(rawf);
    return st;
}

/* channel_weights: weights.cpp:69-91 */
int orc_channel_weights(const float* q, int q_rows, const float* k, int k_rows, int d,
                        float* out) {
    const double inv_sqrt_d = 1.0 / sqrt((double)d);
    for (int c = 0; c < d; ++c) {
        double qq = 0.0, kk = 0.0;
        for (int r = 0; r < q_rows; ++r) {
            const double x = q[(size_t)r * d + c];
            qq += x * x;
        }
        for (int r = 0; r < k_rows; ++r) {
            const double x = k[(size_t)r * d + c];
            kk += x * x;
        }
        out[c] = (float)(sqrt(qq) * sqrt(kk) * inv_sqrt_d);
    }
    return ORC_OK;
}

/* ------------------------------------------------------------------------ */
/* Quantizer: quantize_unit, quantizer.cpp:104-131                           */
/* ------------------------------------------------------------------------ */

static int is_quant_width(int b) { return b == 2 || b == 4 || b == 8; }

int orc_quantize_unit(const float* values, int n, int bits, uint8_t* codes, float* scale_out,
                      int64_t* zero_point) {
    if (!is_quant_width(bits)) return ORC_EINVAL;
    if (n < 1) return ORC_EINVAL;
    float lo = values[0], hi = values[0];
    for (int i = 0; i < n; ++i) {
        const float v = values[i];
        if (!isfinite(v)) return ORC_ENUMERIC;
        lo = v < lo ? v : lo; /* std::min(lo, v) keeps lo on ties */
        hi = hi < v ? v : hi; /* std::max(hi, v) keeps hi on ties */
    }
    const double max_code = (double)((1 << bits) - 1);
    double range = (double)hi - lo;
    if (range < 1e-12) range = 1e-12;
    const double scale = range / max_code;
    double zd = round(-(double)lo / scale);
    if (zd < -9.0e18) zd = -9.0e18;
    if (zd > 9.0e18) zd = 9.0e18;
    *scale_out = (float)scale;
    *zero_point = (int64_t)zd;
    for (int i = 0; i < n; ++i) {
        double c = round(values[i] / scale) + zd;
        if (c < 0.0) c = 0.0;
        if (c > max_code) c = max_code;
        codes[i] = (uint8_t)c;
    }
    return ORC_OK;
}

/* ------------------------------------------------------------------------ */
/* Allocator: allocator.cpp                                                  */
/* ------------------------------------------------------------------------ */

/* argmin_entry: allocator.cpp:39-50 — strict '<' keeps the lower width */
static int argmin_entry(double weight, const int* widths, const double* eps, int nw,
                        double lambda) {
    int best_bits = widths[0];
    double best_cost = weight * eps[0] + lambda * best_bits;
    for (int i = 1; i < nw; ++i) {
        const double cost = weight * eps[i] + lambda * widths[i];
        if (cost < best_cost) {
            best_cost = cost;
            best_bits = widths[i];
        }
    }
    return best_bits;
}

int orc_per_unit_argmin(double weight, const int* widths, const double* eps, int nw,
                        double lambda) {
    if (lambda < 0.0 || !isfinite(lambda)) return -ORC_EINVAL;
    return argmin_entry(weight, widths, eps, nw, lambda);
}

/* assign_all: allocator.cpp:52-61 */
static double assign_all(const float* w, int n, const int* widths, const double* eps, int nw,
                         double lambda, int* out) {
    double total = 0.0;
    for (int u = 0; u < n; ++u) {
        const int b = argmin_entry(w[u], widths, eps, nw, lambda);
        out[u] = b;
        total += b;
    }
    return total / (double)n;
}

static double eps_at(const int* widths, const double* eps, int nw, int bits) {
    for (int i = 0; i < nw; ++i)
        if (widths[i] == bits) return eps[i];
    return NAN;
}

/* allocation_objective: allocator.cpp:301-311 */
static double objective(const float* w, int n, const int* widths, const double* eps, int nw,
                        const int* bits) {
    double obj = 0.0;
    for (int u = 0; u < n; ++u) obj += (double)w[u] * eps_at(widths, eps, nw, bits[u]);
    return obj;
}

static int validate_widths(const int* widths, int nw) {
    /* BitSet::validate_relaxed: quantizer.cpp:66-81 */
    if (nw < 1) return ORC_EINVAL;
    for (int i = 0; i < nw; ++i) {
        if (widths[i] < 0 || widths[i] > 16 || widths[i] % 2 != 0) return ORC_EINVAL;
        if (i > 0 && widths[i] <= widths[i - 1]) return ORC_EINVAL;
        if (widths[i] != 0 && widths[i] != 16 && !is_quant_width(widths[i])) return ORC_EINVAL;
    }
    return ORC_OK;
}

/* mckp_bisect: allocator.cpp:135-216 */
int orc_mckp_bisect(const float* w, int n, const int* widths, const double* eps, int nw,
                    double target, double tolerance, int max_iterations, int strict_budget,
                    int* bits, double* lambda_out, double* avg_out, double* objective_out,
                    int* converged_out) {
    if (!(tolerance > 0.0) || max_iterations < 1) return ORC_EINVAL; /* :413-416 */
    for (int u = 0; u < n; ++u)
        if (!isfinite(w[u]) || w[u] < 0.0f) return ORC_EINVAL; /* :143-149 */
    if (!(target > 0.0) || target > 16.0) return ORC_EINVAL;
    if (validate_widths(widths, nw)) return ORC_EINVAL;

    *lambda_out = 0.0;
    *avg_out = 0.0;
    *objective_out = 0.0;
    *converged_out = 1;
    if (n == 0) return ORC_OK;

    const int max_width = widths[nw - 1];
    if (target >= (double)max_width) { /* :153-161 */
        for (int u = 0; u < n; ++u) bits[u] = max_width;
        *avg_out = max_width;
        *objective_out = objective(w, n, widths, eps, nw, bits);
        return ORC_OK;
    }
    double lo = 0.0, hi = 0.0;
    for (int u = 0; u < n; ++u)
        if ((double)w[u] > hi) hi = w[u];

    const double floor_avg = widths[0];
    int* hi_bits = (int*)malloc(sizeof(int) * (size_t)n);
    if (hi > 0.0) { /* :171-182 */
        double hi_avg = assign_all(w, n, widths, eps, nw, hi, hi_bits);
        int guard = 0;
        while (hi_avg > target && hi_avg > floor_avg && guard++ < 128) {
            hi *= 2.0;
            hi_avg = assign_all(w, n, widths, eps, nw, hi, hi_bits);
        }
    } else {
        assign_all(w, n, widths, eps, nw, hi, hi_bits);
    }
    double lambda = hi;
    double avg = 0.0;
    int converged = 0;
    for (int it = 0; it < max_iterations; ++it) { /* :187-200 */
        lambda = 0.5 * (lo + hi);
        avg = assign_all(w, n, widths, eps, nw, lambda, bits);
        if (fabs(avg - target) / target < tolerance) {
            converged = 1;
            break;
        }
        if (avg > target) {
            lo = lambda;
        } else {
            hi = lambda;
            memcpy(hi_bits, bits, sizeof(int) * (size_t)n);
        }
    }
    if (strict_budget && avg > target) { /* :202-210 */
        lambda = hi;
        memcpy(bits, hi_bits, sizeof(int) * (size_t)n);
        avg = 0.0;
        for (int u = 0; u < n; ++u) avg += bits[u];
        avg /= (double)n;
        converged = fabs(avg - target) / target < tolerance;
    }
    free(hi_bits);
    *lambda_out = lambda;
    *avg_out = avg;
    *converged_out = converged;
    *objective_out = objective(w, n, widths, eps, nw, bits);
    return ORC_OK;
}

/* ------------------------------------------------------------------------ */
/* Pipeline: pipeline.cpp                                                    */
/* ------------------------------------------------------------------------ */

static int validate_bitset_full(const int* widths, int nw) {
    /* BitSet::validate: quantizer.cpp:83-88 — must contain 0 and 16 */
    if (validate_widths(widths, nw)) return ORC_EINVAL;
    int has0 = 0, has16 = 0;
    for (int i = 0; i < nw; ++i) {
        has0 |= widths[i] == 0;
        has16 |= widths[i] == 16;
    }
    return (has0 && has16) ? ORC_OK : ORC_EINVAL;
}

/* head_budget: pipeline.cpp:60-72 (BudgetSpec::validate :52-58) */
int orc_head_budget(int n_tokens, double r_k, int head_dim, int kv_heads, double* head_bits,
                    double* v_bits, double* k_bits, int* sub_token) {
    if (n_tokens < 1) return ORC_EINVAL;
    if (!(r_k > 0.0) || !(r_k < 1.0)) return ORC_EINVAL;
    if (head_dim < 1 || kv_heads < 1) return ORC_EINVAL;
    const double tokens_per_head = (double)n_tokens / kv_heads;
    *sub_token = n_tokens < kv_heads;
    *head_bits = 2.0 * tokens_per_head * head_dim * 16.0;
    *k_bits = r_k * *head_bits;
    *v_bits = (1.0 - r_k) * *head_bits;
    return ORC_OK;
}

/* allocate_head: pipeline.cpp:114-183 (allocate_v :74-94, allocate_k
 * :96-112, probe_group_window :37-50). */
int orc_allocate_head(const float* k, const float* probe_group, int t_len, int d, int group,
                      int probe_rows, int kv_heads, const orc_config* cfg, int* v_bits,
                      int* k_bits, float* v_weights, float* k_weights, orc_head_stats* st) {
    memset(st, 0, sizeof(*st));
    if (cfg->n_tokens < 1 || !(cfg->r_k > 0.0) || !(cfg->r_k < 1.0)) return ORC_EINVAL;
    if (validate_bitset_full(cfg->widths, cfg->n_widths)) return ORC_EINVAL;
    if (cfg->window < 1 || cfg->pool_kernel < 1 || cfg->pool_kernel % 2 == 0) return ORC_EINVAL;
    if (!(cfg->tolerance > 0.0) || cfg->max_iterations < 1) return ORC_EINVAL;
    const int window = cfg->window < probe_rows ? cfg->window : probe_rows;

    /* Stage 1: probe attention per grouped query head (:128-142) */
    int* offsets = (int*)malloc(sizeof(int) * (size_t)window);
    for (int i = 0; i < window; ++i) offsets[i] = t_len - window + i;
    double* attn = (double*)malloc(sizeof(double) * (size_t)group * window * t_len);
    float* qwin = (float*)malloc(sizeof(float) * (size_t)group * window * d);
    for (int qi = 0; qi < group; ++qi) {
        const float* full = probe_group + (size_t)qi * probe_rows * d;
        memcpy(qwin + (size_t)qi * window * d, full + (size_t)(probe_rows - window) * d,
               sizeof(float) * (size_t)window * d);
    }
    int status = ORC_OK;
    for (int qi = 0; qi < group && status == ORC_OK; ++qi) {
        status = orc_attention_probe(qwin + (size_t)qi * window * d, window, k, t_len, d,
                                     offsets, attn + (size_t)qi * window * t_len);
    }
    if (status == ORC_OK)
        status = orc_token_weights(attn, group, window, t_len, cfg->pool_kernel, v_weights);
    free(attn);
    free(offsets);
    if (status != ORC_OK) {
        free(qwin);
        return status;
    }
    /* channel weights over the stacked trailing-window rows (:144-146) */
    orc_channel_weights(qwin, group * window, k, t_len, d, k_weights);
    free(qwin);

    double head_bits, vb, kb;
    int sub_token;
    orc_head_budget(cfg->n_tokens, cfg->r_k, d, kv_heads, &head_bits, &vb, &kb, &sub_token);

    /* Stage 2: V tokens (allocate_v :74-94) */
    int v_conv = 1;
    double lam_v = 0.0, avg_v = 0.0, obj_raw = 0.0;
    if (!(vb > 0.0)) {
        for (int t = 0; t < t_len; ++t) v_bits[t] = 0;
    } else {
        double target = vb / ((double)d * t_len);
        if (target > 16.0) target = 16.0;
        status = orc_mckp_bisect(v_weights, t_len, cfg->widths, cfg->eps_v, cfg->n_widths,
                                 target, cfg->tolerance, cfg->max_iterations,
                                 cfg->strict_budget, v_bits, &lam_v, &avg_v, &obj_raw, &v_conv);
        if (status) return status;
    }
    if (cfg->force_window_retain) { /* :153-156 */
        for (int i = 0; i < window; ++i) v_bits[t_len - window + i] = 16;
    }
    int kept = 0, v16 = 0;
    for (int t = 0; t < t_len; ++t) {
        kept += v_bits[t] > 0;
        v16 += v_bits[t] == 16;
    }

    /* Stage 3: K channels over kept tokens (allocate_k :96-112) */
    int k_conv = 1, k_len = d;
    double lam_k = 0.0, avg_k = 0.0, obj_k_raw = 0.0;
    if (kept == 0) {
        k_len = 0;
    } else if (!(kb > 0.0)) {
        for (int c = 0; c < d; ++c) k_bits[c] = 0;
    } else {
        double target = kb / ((double)kept * d);
        if (target > 16.0) target = 16.0;
        status = orc_mckp_bisect(k_weights, d, cfg->widths, cfg->eps_k, cfg->n_widths, target,
                                 cfg->tolerance, cfg->max_iterations, cfg->strict_budget,
                                 k_bits, &lam_k, &avg_k, &obj_k_raw, &k_conv);
        if (status) return status;
    }

    st->objective_v = objective(v_weights, t_len, cfg->widths, cfg->eps_v, cfg->n_widths, v_bits);
    st->objective_k = k_len == 0 ? 0.0
                                 : objective(k_weights, d, cfg->widths, cfg->eps_k,
                                             cfg->n_widths, k_bits);
    st->lambda_v = lam_v;
    st->lambda_k = lam_k;
    st->avg_v = avg_v;
    st->avg_k = avg_k;
    st->v_converged = v_conv;
    st->k_converged = k_conv;
    st->n_kept = kept;
    st->n_v16 = v16;
    st->k_bits_len = k_len;
    double v_sum = 0.0, k_sum = 0.0; /* :177-181 */
    for (int t = 0; t < t_len; ++t) v_sum += v_bits[t];
    for (int c = 0; c < k_len; ++c) k_sum += k_bits[c];
    st->achieved_bits = v_sum * d + k_sum * (double)kept;
    return ORC_OK;
}

/* ------------------------------------------------------------------------ */
/* TriZone: trizone.cpp                                                      */
/* ------------------------------------------------------------------------ */

/* padded_len / packed_row_bytes: trizone.cpp:48-57 */
int orc_padded_len(int len, int bits) {
    switch (bits) {
        case 2: return (len + 3) / 4 * 4;
        case 4: return (len + 1) / 2 * 2;
        case 8: return len;
        default: return -1;
    }
}
int orc_packed_row_bytes(int len, int bits) { return orc_padded_len(len, bits) * bits / 8; }

/* pack_bits: trizone.cpp:59-75 */
int orc_pack_bits(const uint8_t* codes, int n, int bits, uint8_t* out) {
    if (!is_quant_width(bits)) return ORC_EINVAL;
    const int per_byte = 8 / bits;
    const unsigned limit = (1u << bits) - 1u;
    memset(out, 0, (size_t)(n + per_byte - 1) / per_byte);
    for (int i = 0; i < n; ++i) {
        if (codes[i] > limit) return ORC_EINVAL;
        out[i / per_byte] |= (uint8_t)(codes[i] << ((i % per_byte) * bits));
    }
    return ORC_OK;
}

/* extract_code: trizone.cpp:26-32 */
static unsigned extract_code(const uint8_t* row, int j, int bits) {
    switch (bits) {
        case 2: return (row[j >> 2] >> ((j & 3) * 2)) & 0x3u;
        case 4: return (row[j >> 1] >> ((j & 1) * 4)) & 0xfu;
        default: return row[j];
    }
}

typedef struct {
    int bits, logical_len, pad_count, rows;
    int* members;
    int* positions;
    float* scale;
    int64_t* zero;
    uint8_t* payload;
    size_t nbytes;
} orc_segment;

struct orc_trizone {
    int d, t_len, n_kept;
    int* kept;
    int* v_bits;
    int* k_bits;
    int n_vseg, n_kseg;
    orc_segment vseg[3];
    orc_segment kseg[3];
    int k16_width;
    int* k16_members;
    float* k16_data;
    int zb_rows;
    int* zb_members;
    int* zb_positions;
    float* zb_data;
    int zc_len, zc_cap;
    float* zc_k;
    float* zc_v;
    int n_perm;
    int* perm;
};

static void seg_free(orc_segment* s) {
    free(s->members);
    free(s->positions);
    free(s->scale);
    free(s->zero);
    free(s->payload);
}

void orc_tz_free(orc_trizone* tz) {
    if (!tz) return;
    for (int i = 0; i < tz->n_vseg; ++i) seg_free(&tz->vseg[i]);
    for (int i = 0; i < tz->n_kseg; ++i) seg_free(&tz->kseg[i]);
    free(tz->kept);
    free(tz->v_bits);
    free(tz->k_bits);
    free(tz->k16_members);
    free(tz->k16_data);
    free(tz->zb_members);
    free(tz->zb_positions);
    free(tz->zb_data);
    free(tz->zc_k);
    free(tz->zc_v);
    free(tz->perm);
    free(tz);
}

/* build_trizone: trizone.cpp:91-208 */
orc_trizone* orc_tz_build(const float* k, const float* v, int t_len, int d, const int* v_bits,
                          const int* k_bits, int* status) {
    static const int kPack[3] = {2, 4, 8};
    *status = ORC_OK;
    orc_trizone* tz = (orc_trizone*)calloc(1, sizeof(orc_trizone));
    tz->d = d;
    tz->t_len = t_len;
    tz->v_bits = (int*)malloc(sizeof(int) * (size_t)t_len);
    memcpy(tz->v_bits, v_bits, sizeof(int) * (size_t)t_len);
    tz->k_bits = (int*)calloc((size_t)d, sizeof(int));
    tz->kept = (int*)malloc(sizeof(int) * (size_t)t_len);
    int kept_n = 0;
    for (int t = 0; t < t_len; ++t)
        if (v_bits[t] > 0) tz->kept[kept_n++] = t;
    tz->n_kept = kept_n;
    if (kept_n == 0) return tz; /* :113-118 — k_bits all zero */
    if (!k_bits) {
        *status = ORC_EINVAL;
        orc_tz_free(tz);
        return NULL;
    }
    memcpy(tz->k_bits, k_bits, sizeof(int) * (size_t)d);
    int* kept_pos = (int*)malloc(sizeof(int) * (size_t)t_len);
    for (int t = 0; t < t_len; ++t) kept_pos[t] = -1;
    for (int i = 0; i < kept_n; ++i) kept_pos[tz->kept[i]] = i;

    uint8_t* codes = (uint8_t*)malloc((size_t)(t_len > d ? t_len : d) + 8);
    uint8_t* padded = (uint8_t*)calloc((size_t)(t_len > d ? t_len : d) + 8, 1);

    /* Zone A (V): :126-143 */
    for (int bi = 0; bi < 3; ++bi) {
        const int bits = kPack[bi];
        int rows = 0;
        for (int i = 0; i < kept_n; ++i) rows += v_bits[tz->kept[i]] == bits;
        if (rows == 0) continue;
        orc_segment* s = &tz->vseg[tz->n_vseg++];
        s->bits = bits;
        s->logical_len = d;
        s->pad_count = orc_padded_len(d, bits) - d;
        s->rows = rows;
        const int rb = orc_packed_row_bytes(d, bits);
        s->members = (int*)malloc(sizeof(int) * (size_t)rows);
        s->positions = (int*)malloc(sizeof(int) * (size_t)rows);
        s->scale = (float*)malloc(sizeof(float) * (size_t)rows);
        s->zero = (int64_t*)malloc(sizeof(int64_t) * (size_t)rows);
        s->nbytes = (size_t)rows * rb;
        s->payload = (uint8_t*)calloc(s->nbytes ? s->nbytes : 1, 1);
        int r = 0;
        for (int i = 0; i < kept_n; ++i) {
            const int t = tz->kept[i];
            if (v_bits[t] != bits) continue;
            s->members[r] = t;
            s->positions[r] = kept_pos[t];
            int st = orc_quantize_unit(v + (size_t)t * d, d, bits, codes, &s->scale[r],
                                       &s->zero[r]);
            if (st) {
                *status = st;
                free(kept_pos);
                free(codes);
                free(padded);
                orc_tz_free(tz);
                return NULL;
            }
            const int plen = orc_padded_len(d, bits);
            memset(padded, 0, (size_t)plen);
            memcpy(padded, codes, (size_t)d);
            orc_pack_bits(padded, plen, bits, s->payload + (size_t)r * rb);
            ++r;
        }
    }

    /* Zone B: :145-157 */
    tz->zb_members = (int*)malloc(sizeof(int) * (size_t)kept_n);
    tz->zb_positions = (int*)malloc(sizeof(int) * (size_t)kept_n);
    int zb = 0;
    for (int i = 0; i < kept_n; ++i)
        if (v_bits[tz->kept[i]] == 16) ++zb;
    tz->zb_data = (float*)malloc(sizeof(float) * ((size_t)zb * d + 1));
    zb = 0;
    for (int i = 0; i < kept_n; ++i) {
        const int t = tz->kept[i];
        if (v_bits[t] != 16) continue;
        tz->zb_members[zb] = t;
        tz->zb_positions[zb] = i;
        memcpy(tz->zb_data + (size_t)zb * d, v + (size_t)t * d, sizeof(float) * (size_t)d);
        ++zb;
    }
    tz->zb_rows = zb;

    /* Zone A (K): :159-184 — channel codes over the kept rows, row-major */
    float* column = (float*)malloc(sizeof(float) * (size_t)kept_n);
    uint8_t* chan_codes = (uint8_t*)malloc((size_t)d * kept_n);
    for (int bi = 0; bi < 3; ++bi) {
        const int bits = kPack[bi];
        int n_ch = 0;
        for (int c = 0; c < d; ++c) n_ch += k_bits[c] == bits;
        if (n_ch == 0) continue;
        orc_segment* s = &tz->kseg[tz->n_kseg++];
        s->bits = bits;
        s->rows = kept_n;
        s->logical_len = n_ch;
        s->pad_count = orc_padded_len(n_ch, bits) - n_ch;
        s->members = (int*)malloc(sizeof(int) * (size_t)n_ch);
        s->positions = NULL;
        s->scale = (float*)malloc(sizeof(float) * (size_t)n_ch);
        s->zero = (int64_t*)malloc(sizeof(int64_t) * (size_t)n_ch);
        int j = 0;
        for (int c = 0; c < d; ++c) {
            if (k_bits[c] != bits) continue;
            s->members[j] = c;
            for (int r = 0; r < kept_n; ++r) column[r] = k[(size_t)tz->kept[r] * d + c];
            int st = orc_quantize_unit(column, kept_n, bits, chan_codes + (size_t)j * kept_n,
                                       &s->scale[j], &s->zero[j]);
            if (st) {
                *status = st;
                free(column);
                free(chan_codes);
                free(kept_pos);
                free(codes);
                free(padded);
                orc_tz_free(tz);
                return NULL;
            }
            ++j;
        }
        const int rb = orc_packed_row_bytes(n_ch, bits);
        const int plen = orc_padded_len(n_ch, bits);
        s->nbytes = (size_t)kept_n * rb;
        s->payload = (uint8_t*)calloc(s->nbytes ? s->nbytes : 1, 1);
        for (int r = 0; r < kept_n; ++r) {
            memset(padded, 0, (size_t)plen);
            for (int jj = 0; jj < n_ch; ++jj) padded[jj] = chan_codes[(size_t)jj * kept_n + r];
            orc_pack_bits(padded, plen, bits, s->payload + (size_t)r * rb);
        }
    }
    free(column);
    free(chan_codes);

    /* k16: :186-199 */
    tz->k16_members = (int*)malloc(sizeof(int) * (size_t)d);
    for (int c = 0; c < d; ++c)
        if (k_bits[c] == 16) tz->k16_members[tz->k16_width++] = c;
    tz->k16_data = (float*)malloc(sizeof(float) * ((size_t)kept_n * tz->k16_width + 1));
    for (int r = 0; r < kept_n; ++r)
        for (int j = 0; j < tz->k16_width; ++j)
            tz->k16_data[(size_t)r * tz->k16_width + j] =
                k[(size_t)tz->kept[r] * d + tz->k16_members[j]];

    /* channel_perm: :201-206 */
    tz->perm = (int*)malloc(sizeof(int) * (size_t)d);
    for (int i = 0; i < tz->n_kseg; ++i)
        for (int j = 0; j < tz->kseg[i].logical_len; ++j)
            tz->perm[tz->n_perm++] = tz->kseg[i].members[j];
    for (int j = 0; j < tz->k16_width; ++j) tz->perm[tz->n_perm++] = tz->k16_members[j];

    free(kept_pos);
    free(codes);
    free(padded);
    return tz;
}

/* append_new_token: trizone.cpp:307-314 */
int orc_tz_append(orc_trizone* tz, const float* k, const float* v) {
    if (tz->zc_len == tz->zc_cap) {
        tz->zc_cap = tz->zc_cap ? tz->zc_cap * 2 : 8;
        tz->zc_k = (float*)realloc(tz->zc_k, sizeof(float) * (size_t)tz->zc_cap * tz->d);
        tz->zc_v = (float*)realloc(tz->zc_v, sizeof(float) * (size_t)tz->zc_cap * tz->d);
    }
    memcpy(tz->zc_k + (size_t)tz->zc_len * tz->d, k, sizeof(float) * (size_t)tz->d);
    memcpy(tz->zc_v + (size_t)tz->zc_len * tz->d, v, sizeof(float) * (size_t)tz->d);
    ++tz->zc_len;
    return ORC_OK;
}

/* fused_k_logits: trizone.cpp:210-249 */
int orc_tz_fused_logits(const orc_trizone* tz, const float* q, double* logits) {
    const int kept_n = tz->n_kept;
    for (int r = 0; r < kept_n; ++r) logits[r] = 0.0;
    if (kept_n == 0) return ORC_OK;
    double bias = 0.0;
    double* scaled_q = (double*)malloc(sizeof(double) * ((size_t)tz->d + 1));
    for (int i = 0; i < tz->n_kseg; ++i) {
        const orc_segment* s = &tz->kseg[i];
        for (int j = 0; j < s->logical_len; ++j) {
            const double qc = q[s->members[j]];
            scaled_q[j] = (double)s->scale[j] * qc;
            bias += (double)s->scale[j] * (double)s->zero[j] * qc;
        }
        const int rb = orc_packed_row_bytes(s->logical_len, s->bits);
        for (int r = 0; r < s->rows; ++r) {
            const uint8_t* row = s->payload + (size_t)r * rb;
            double acc = 0.0;
            for (int j = 0; j < s->logical_len; ++j)
                acc += scaled_q[j] * extract_code(row, j, s->bits);
            logits[r] += acc;
        }
    }
    free(scaled_q);
    if (tz->k16_width > 0) {
        for (int r = 0; r < kept_n; ++r) {
            const float* row = tz->k16_data + (size_t)r * tz->k16_width;
            double acc = 0.0;
            for (int j = 0; j < tz->k16_width; ++j)
                acc += (double)q[tz->k16_members[j]] * row[j];
            logits[r] += acc;
        }
    }
    for (int r = 0; r < kept_n; ++r) logits[r] -= bias;
    return ORC_OK;
}

/* packed_decode_step: trizone.cpp:251-305 */
int orc_tz_decode(const orc_trizone* tz, const float* q, double* out) {
    const int kept_n = tz->n_kept;
    const int total = kept_n + tz->zc_len;
    const int d = tz->d;
    if (total == 0) return ORC_ENUMERIC;
    const double inv_sqrt_d = 1.0 / sqrt((double)d);
    double* logits = (double*)malloc(sizeof(double) * (size_t)total);
    orc_tz_fused_logits(tz, q, logits);
    for (int r = 0; r < tz->zc_len; ++r) {
        const float* kr = tz->zc_k + (size_t)r * d;
        double acc = 0.0;
        for (int c = 0; c < d; ++c) acc += (double)q[c] * kr[c];
        logits[kept_n + r] = acc;
    }
    double mx = -INFINITY;
    for (int i = 0; i < total; ++i) {
        logits[i] *= inv_sqrt_d;
        if (logits[i] > mx) mx = logits[i];
    }
    double denom = 0.0;
    for (int i = 0; i < total; ++i) {
        logits[i] = exp(logits[i] - mx);
        denom += logits[i];
    }
    for (int i = 0; i < total; ++i) logits[i] /= denom;
    for (int c = 0; c < d; ++c) out[c] = 0.0;
    for (int si = 0; si < tz->n_vseg; ++si) {
        const orc_segment* s = &tz->vseg[si];
        const int rb = orc_packed_row_bytes(d, s->bits);
        for (int i = 0; i < s->rows; ++i) {
            const double w = logits[s->positions[i]];
            const double scale = s->scale[i];
            const double zp = (double)s->zero[i];
            const uint8_t* row = s->payload + (size_t)i * rb;
            for (int c = 0; c < d; ++c) out[c] += w * (scale * (extract_code(row, c, s->bits) - zp));
        }
    }
    for (int i = 0; i < tz->zb_rows; ++i) {
        const double w = logits[tz->zb_positions[i]];
        const float* row = tz->zb_data + (size_t)i * d;
        for (int c = 0; c < d; ++c) out[c] += w * row[c];
    }
    for (int r = 0; r < tz->zc_len; ++r) {
        const double w = logits[kept_n + r];
        const float* row = tz->zc_v + (size_t)r * d;
        for (int c = 0; c < d; ++c) out[c] += w * row[c];
    }
    free(logits);
    return ORC_OK;
}

int orc_tz_n_kept(const orc_trizone* tz) { return tz->n_kept; }

size_t orc_tz_payload_bytes(const orc_trizone* tz) {
    size_t n = 0;
    for (int i = 0; i < tz->n_vseg; ++i) n += tz->vseg[i].nbytes;
    for (int i = 0; i < tz->n_kseg; ++i) n += tz->kseg[i].nbytes;
    return n;
}

int orc_tz_canon(const orc_trizone* tz, int* kept, uint8_t* vcodes, float* vscale,
                 int64_t* vzero, uint8_t* kcodes, float* kscale, int64_t* kzero, float* vfp,
                 float* kfp, uint8_t* payload, int* segtab, int* nseg, int* perm, int* nperm) {
    const int n = tz->n_kept, d = tz->d;
    memcpy(kept, tz->kept, sizeof(int) * (size_t)n);
    memset(vcodes, 0, (size_t)n * d);
    memset(vscale, 0, sizeof(float) * (size_t)n);
    memset(vzero, 0, sizeof(int64_t) * (size_t)n);
    memset(kcodes, 0, (size_t)n * d);
    memset(kscale, 0, sizeof(float) * (size_t)d);
    memset(kzero, 0, sizeof(int64_t) * (size_t)d);
    memset(vfp, 0, sizeof(float) * (size_t)n * d);
    memset(kfp, 0, sizeof(float) * (size_t)n * d);
    size_t off = 0;
    int ns = 0;
    for (int si = 0; si < tz->n_vseg; ++si) {
        const orc_segment* s = &tz->vseg[si];
        const int rb = orc_packed_row_bytes(d, s->bits);
        for (int i = 0; i < s->rows; ++i) {
            const int p = s->positions[i];
            vscale[p] = s->scale[i];
            vzero[p] = s->zero[i];
            for (int c = 0; c < d; ++c)
                vcodes[(size_t)p * d + c] = (uint8_t)extract_code(s->payload + (size_t)i * rb, c, s->bits);
        }
        memcpy(payload + off, s->payload, s->nbytes);
        int* row = segtab + 6 * ns++;
        row[0] = 0; row[1] = s->bits; row[2] = s->rows; row[3] = s->logical_len;
        row[4] = s->pad_count; row[5] = (int)s->nbytes;
        off += s->nbytes;
    }
    for (int i = 0; i < tz->zb_rows; ++i)
        memcpy(vfp + (size_t)tz->zb_positions[i] * d, tz->zb_data + (size_t)i * d,
               sizeof(float) * (size_t)d);
    for (int si = 0; si < tz->n_kseg; ++si) {
        const orc_segment* s = &tz->kseg[si];
        const int rb = orc_packed_row_bytes(s->logical_len, s->bits);
        for (int j = 0; j < s->logical_len; ++j) {
            const int c = s->members[j];
            kscale[c] = s->scale[j];
            kzero[c] = s->zero[j];
            for (int r = 0; r < n; ++r)
                kcodes[(size_t)c * n + r] =
                    (uint8_t)extract_code(s->payload + (size_t)r * rb, j, s->bits);
        }
        memcpy(payload + off, s->payload, s->nbytes);
        int* row = segtab + 6 * ns++;
        row[0] = 1; row[1] = s->bits; row[2] = s->rows; row[3] = s->logical_len;
        row[4] = s->pad_count; row[5] = (int)s->nbytes;
        off += s->nbytes;
    }
    for (int r = 0; r < n; ++r)
        for (int j = 0; j < tz->k16_width; ++j)
            kfp[(size_t)r * d + tz->k16_members[j]] = tz->k16_data[(size_t)r * tz->k16_width + j];
    *nseg = ns;
    memcpy(perm, tz->perm, sizeof(int) * (size_t)tz->n_perm);
    *nperm = tz->n_perm;
    return ORC_OK;
}

/* dense_decode_reference: trizone.cpp:407-443 (rows already concatenated) */
int orc_dense_decode(const float* q, const float* k_rows, const float* v_rows, int n, int d,
                     double* out) {
    if (n == 0) return ORC_ENUMERIC;
    const double inv_sqrt_d = 1.0 / sqrt((double)d);
    double* logits = (double*)malloc(sizeof(double) * (size_t)n);
    double mx = -INFINITY;
    for (int r = 0; r < n; ++r) {
        double acc = 0.0;
        for (int c = 0; c < d; ++c) acc += (double)q[c] * k_rows[(size_t)r * d + c];
        logits[r] = acc * inv_sqrt_d;
        if (logits[r] > mx) mx = logits[r];
    }
    double denom = 0.0;
    for (int r = 0; r < n; ++r) {
        logits[r] = exp(logits[r] - mx);
        denom += logits[r];
    }
    for (int c = 0; c < d; ++c) out[c] = 0.0;
    for (int r = 0; r < n; ++r) {
        const double w = logits[r] / denom;
        for (int c = 0; c < d; ++c) out[c] += w * v_rows[(size_t)r * d + c];
    }
    free(logits);
    return ORC_OK;
}

/* ------------------------------------------------------------------------ */
/* K0 counter-based generator — CPU restatement of                           */
/* paper_2605_08317_b200/csrc/generate.cu (not a reference function: the     */
/* reference's serial mt19937 generator does not scale to 128K contexts).    */
/* Emits float32 values that are exactly FP16-representable.                 */
/* ------------------------------------------------------------------------ */
static uint64_t splitmix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

/* IEEE binary32 -> binary16 -> binary32, round to nearest even */
static float round_to_half(float x) {
    union { float f; uint32_t u; } in = {x};
    uint32_t sign = in.u & 0x80000000u;
    uint32_t ax = in.u & 0x7FFFFFFFu;
    union { uint32_t u; float f; } out;
    if (ax >= 0x477FF000u) { /* >= 65520: overflow to inf (or NaN passthrough) */
        out.u = sign | (ax > 0x7F800000u ? ax : 0x7F800000u);
        return out.f;
    }
    if (ax < 0x38800000u) { /* below 2^-14: subnormal half, quantum 2^-24 */
        float a = fabsf(x);
        float q = nearbyintf(a * 16777216.0f) / 16777216.0f; /* exact scaling by 2^24 */
        return sign ? -q : q;
    }
    /* normal: keep 10 mantissa bits, RNE on the dropped 13 */
    uint32_t lsb = (ax >> 13) & 1u;
    ax += 0xFFFu + lsb;
    ax &= 0xFFFFE000u;
    out.u = sign | ax;
    return out.f;
}

static float channel_sign(uint64_t seed, int c) {
    return (splitmix64(seed ^ 0x5BD1E9955BD1E995ULL ^ (uint64_t)c) & 1ULL) ? 1.0f : -1.0f;
}

void orc_gen_counter(float* out, uint64_t seed, int tensor, uint64_t first, uint64_t count, int d,
                     int seq_len, int outlier_channels, float outlier_scale, int hh_stride,
                     float hh_boost) {
    const uint64_t base = seed * 0x9E3779B97F4A7C15ULL + (uint64_t)(tensor + 1) * 0xD1B54A32D192ED03ULL;
    const float inv = 1.0f / 37836.5f;
    for (uint64_t j = 0; j < count; ++j) {
        const uint64_t i = first + j;
        const uint64_t z = splitmix64(base + i);
        const int s = (int)(z & 0xFFFF) + (int)((z >> 16) & 0xFFFF) + (int)((z >> 32) & 0xFFFF) +
                      (int)((z >> 48) & 0xFFFF);
        float x = (float)(s - 131070) * inv;
        const int c = (int)(i % (uint64_t)d);
        if (tensor == 0) {
            if (c < outlier_channels) x = x * outlier_scale;
            if (hh_stride > 0) {
                const uint64_t t = (i / (uint64_t)d) % (uint64_t)seq_len;
                if (t % (uint64_t)hh_stride == 0) x = x + hh_boost * channel_sign(seed, c);
            }
        } else if (tensor == 2 && hh_stride > 0) {
            x = x + 0.5f * channel_sign(seed, c);
        }
        out[j] = round_to_half(x);
    }
}
