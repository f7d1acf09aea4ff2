// ref_shim.cpp — extern "C" bridge over the UNMODIFIED reference library.
//
// TEST / BASELINE INFRASTRUCTURE ONLY. Compiled together with the reference
// sources where they lie (/root/reference/proj/core/src/*.cpp) into
// oracle/_ref/librdkv_ref.so by oracle/Makefile; nothing from the reference
// is copied into this repository. The exported ref_* functions mirror the
// orc_* functions of oracle/rdkv_oracle.h so tests can run one check against
// both, and ref_model_* drive allocate_model / build_packed_model /
// packed_decode_step exactly as the reference's own callers do
// (tools/rdkv.cpp:134-228) for the CPU baseline.
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <exception>
#include <new>
#include <stdexcept>
#include <vector>

#include "rdkv/allocator.hpp"
#include "rdkv/cache.hpp"
#include "rdkv/errors.hpp"
#include "rdkv/parallel.hpp"
#include "rdkv/pipeline.hpp"
#include "rdkv/quantizer.hpp"
#include "rdkv/sweep.hpp"
#include "rdkv/trizone.hpp"
#include "rdkv/weights.hpp"

#define REF_API extern "C" __attribute__((visibility("default")))

namespace {

enum { OK = 0, EINVAL_ = 1, ENUMERIC_ = 2, EFORMAT_ = 3, EOTHER_ = 9 };

// Same layout as orc_config (oracle/rdkv_oracle.h) / rdkv_config.
struct Cfg {
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
};

struct Stats {
    double lambda_v, lambda_k, objective_v, objective_k, achieved_bits, avg_v, avg_k;
    int32_t v_converged, k_converged, n_kept, n_v16, k_bits_len, status;
};

template <class F>
int guarded(F&& f) {
    try {
        f();
        return OK;
    } catch (const std::invalid_argument&) {
        return EINVAL_;
    } catch (const rdkv::NumericError&) {
        return ENUMERIC_;
    } catch (const rdkv::FormatError&) {
        return EFORMAT_;
    } catch (...) {
        return EOTHER_;
    }
}

rdkv::BitSet bitset_of(const Cfg& c) {
    rdkv::BitSet b;
    b.widths.assign(c.widths, c.widths + c.n_widths);
    return b;
}

rdkv::DistortionTable table_of(const Cfg& c, bool v_side) {
    rdkv::DistortionTable t;
    t.granularity = v_side ? rdkv::Granularity::token : rdkv::Granularity::channel;
    for (int i = 0; i < c.n_widths; ++i) t.eps.emplace_back(c.widths[i], v_side ? c.eps_v[i] : c.eps_k[i]);
    return t;
}

rdkv::PipelineConfig pipeline_of(const Cfg& c) {
    rdkv::PipelineConfig p;
    p.probe.window = c.window;
    p.probe.pool_kernel = c.pool_kernel;
    p.solver.tolerance = c.tolerance;
    p.solver.max_iterations = c.max_iterations;
    p.solver.strict_budget = c.strict_budget != 0;
    p.force_window_retain = c.force_window_retain != 0;
    return p;
}

rdkv::BudgetSpec spec_of(const Cfg& c) {
    rdkv::BudgetSpec s;
    s.n_tokens = c.n_tokens;
    s.r_k = c.r_k;
    s.bits = bitset_of(c);
    return s;
}

void fill_stats(const rdkv::HeadAllocation& h, Stats* st) {
    std::memset(st, 0, sizeof(*st));
    st->lambda_v = h.lambda_v;
    st->lambda_k = h.lambda_k;
    st->objective_v = h.objective_v;
    st->objective_k = h.objective_k;
    st->achieved_bits = h.achieved_bits;
    st->v_converged = h.v_converged;
    st->k_converged = h.k_converged;
    st->n_kept = static_cast<int32_t>(h.kept.kept.size());
    st->n_v16 = static_cast<int32_t>(h.kept.v16.size());
    st->k_bits_len = static_cast<int32_t>(h.k_bits.size());
}

rdkv::KVCache cache_from(const float* k, const float* v, const float* q, int layers, int q_heads,
                         int kv_heads, int d, int t_len, int probe_rows) {
    rdkv::KVCache c;
    c.shape = rdkv::CacheShape{layers, q_heads, kv_heads, d, t_len};
    c.probe_window = probe_rows;
    const std::size_t kv_n = static_cast<std::size_t>(kv_heads) * t_len * d;
    const std::size_t q_n = static_cast<std::size_t>(q_heads) * probe_rows * d;
    for (int l = 0; l < layers; ++l) {
        auto& kt = c.k.emplace_back(kv_heads, t_len, d);
        std::memcpy(kt.data().data(), k + l * kv_n, kv_n * sizeof(float));
        auto& vt = c.v.emplace_back(kv_heads, t_len, d);
        std::memcpy(vt.data().data(), v + l * kv_n, kv_n * sizeof(float));
        auto& qt = c.probe_q.emplace_back(q_heads, probe_rows, d);
        std::memcpy(qt.data().data(), q + l * q_n, q_n * sizeof(float));
    }
    return c;
}

int canon_of(const rdkv::TriZoneCache& tz, int* kept, uint8_t* vcodes, float* vscale, int64_t* vzero,
             uint8_t* kcodes, float* kscale, int64_t* kzero, float* vfp, float* kfp,
             uint8_t* payload, int* segtab, int* nseg, int* perm, int* nperm) {
    const int n = static_cast<int>(tz.kept.size());
    const int d = tz.head_dim;
    std::memcpy(kept, tz.kept.data(), sizeof(int) * n);
    std::memset(vcodes, 0, static_cast<std::size_t>(n) * d);
    std::memset(vscale, 0, sizeof(float) * n);
    std::memset(vzero, 0, sizeof(int64_t) * n);
    std::memset(kcodes, 0, static_cast<std::size_t>(n) * d);
    std::memset(kscale, 0, sizeof(float) * d);
    std::memset(kzero, 0, sizeof(int64_t) * d);
    std::memset(vfp, 0, sizeof(float) * static_cast<std::size_t>(n) * d);
    std::memset(kfp, 0, sizeof(float) * static_cast<std::size_t>(n) * d);
    std::size_t off = 0;
    int ns = 0;
    for (const auto& s : tz.zone_a_v) {
        auto rows = s.rows;
        for (int i = 0; i < rows; ++i) {
            const int p = s.positions[i];
            vscale[p] = s.params[i].scale;
            vzero[p] = s.params[i].zero_point;
            auto codes = rdkv::unpack_bits(
                std::span<const uint8_t>(s.payload.data() + static_cast<std::size_t>(i) * s.row_bytes(),
                                         s.row_bytes()),
                s.bits, d);
            std::memcpy(vcodes + static_cast<std::size_t>(p) * d, codes.data(), d);
        }
        std::memcpy(payload + off, s.payload.data(), s.payload.size());
        int* row = segtab + 6 * ns++;
        row[0] = 0; row[1] = s.bits; row[2] = s.rows; row[3] = s.logical_len;
        row[4] = s.pad_count; row[5] = static_cast<int>(s.payload.size());
        off += s.payload.size();
    }
    for (std::size_t i = 0; i < tz.zone_b.members.size(); ++i) {
        std::memcpy(vfp + static_cast<std::size_t>(tz.zone_b.positions[i]) * d,
                    tz.zone_b.data.data() + i * d, sizeof(float) * d);
    }
    for (const auto& s : tz.zone_a_k) {
        for (int r = 0; r < s.rows; ++r) {
            auto codes = rdkv::unpack_bits(
                std::span<const uint8_t>(s.payload.data() + static_cast<std::size_t>(r) * s.row_bytes(),
                                         s.row_bytes()),
                s.bits, s.logical_len);
            for (int j = 0; j < s.logical_len; ++j)
                kcodes[static_cast<std::size_t>(s.members[j]) * n + r] = codes[j];
        }
        for (int j = 0; j < s.logical_len; ++j) {
            kscale[s.members[j]] = s.params[j].scale;
            kzero[s.members[j]] = s.params[j].zero_point;
        }
        std::memcpy(payload + off, s.payload.data(), s.payload.size());
        int* row = segtab + 6 * ns++;
        row[0] = 1; row[1] = s.bits; row[2] = s.rows; row[3] = s.logical_len;
        row[4] = s.pad_count; row[5] = static_cast<int>(s.payload.size());
        off += s.payload.size();
    }
    for (int r = 0; r < n; ++r)
        for (int j = 0; j < tz.k16.width; ++j)
            kfp[static_cast<std::size_t>(r) * d + tz.k16.members[j]] =
                tz.k16.data[static_cast<std::size_t>(r) * tz.k16.width + j];
    *nseg = ns;
    std::memcpy(perm, tz.channel_perm.data(), sizeof(int) * tz.channel_perm.size());
    *nperm = static_cast<int>(tz.channel_perm.size());
    return OK;
}

struct RefModel {
    rdkv::KVCache cache;
    rdkv::ModelAllocation alloc;
    rdkv::PackedModel packed;
};

double seconds_since(std::chrono::steady_clock::time_point t0) {
    return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

}  // namespace

REF_API int ref_gen_synthetic(uint64_t seed, int layers, int q_heads, int kv_heads, int d, int t_len,
                              int probe_window, int outlier_channels, double outlier_scale,
                              float* k, float* v, float* q) {
    return guarded([&] {
        auto c = rdkv::gen_synthetic_cache(seed, rdkv::CacheShape{layers, q_heads, kv_heads, d, t_len},
                                           probe_window, outlier_channels, outlier_scale);
        const std::size_t kv_n = static_cast<std::size_t>(kv_heads) * t_len * d;
        const std::size_t q_n = static_cast<std::size_t>(q_heads) * probe_window * d;
        for (int l = 0; l < layers; ++l) {
            std::memcpy(k + l * kv_n, c.k[l].data().data(), kv_n * sizeof(float));
            std::memcpy(v + l * kv_n, c.v[l].data().data(), kv_n * sizeof(float));
            std::memcpy(q + l * q_n, c.probe_q[l].data().data(), q_n * sizeof(float));
        }
    });
}

// RDKVC001 cache container (cache.cpp:205-287): writes gen_synthetic_cache(seed, shape) with
// save_cache_file; ref_load_cache runs load_cache_file and returns its status + dims
// (L, H_q, H_kv, d, T, S_w) — the golden behaviour for the device loader.
REF_API int ref_save_cache(uint64_t seed, int layers, int q_heads, int kv_heads, int d, int t_len,
                           int probe_window, const char* path) {
    return guarded([&] {
        auto c = rdkv::gen_synthetic_cache(seed, rdkv::CacheShape{layers, q_heads, kv_heads, d, t_len},
                                           probe_window, 0, 1.0);
        rdkv::save_cache_file(c, path);
    });
}

REF_API int ref_load_cache(const char* path, int* dims) {
    return guarded([&] {
        auto c = rdkv::load_cache_file(path);
        dims[0] = c.shape.layers;
        dims[1] = c.shape.q_heads;
        dims[2] = c.shape.kv_heads;
        dims[3] = c.shape.head_dim;
        dims[4] = c.shape.seq_len;
        dims[5] = c.probe_window;
    });
}

REF_API int ref_attention_probe(const float* q, int rows, const float* k, int t_len, int d,
                                const int* offsets, double* a) {
    return guarded([&] {
        auto m = rdkv::attention_probe(rdkv::MatrixView{q, rows, d}, rdkv::MatrixView{k, t_len, d},
                                       std::span<const int>(offsets, rows));
        std::memcpy(a, m.a.data(), sizeof(double) * m.a.size());
    });
}

REF_API int ref_moving_average(const float* raw, int n, int kernel, float* out) {
    return guarded([&] {
        auto r = rdkv::moving_average(std::span<const float>(raw, n), kernel);
        std::memcpy(out, r.data(), sizeof(float) * n);
    });
}

REF_API int ref_channel_weights(const float* q, int q_rows, const float* k, int k_rows, int d,
                                float* out) {
    return guarded([&] {
        auto w = rdkv::channel_weights(rdkv::MatrixView{q, q_rows, d}, rdkv::MatrixView{k, k_rows, d});
        std::memcpy(out, w.values.data(), sizeof(float) * d);
    });
}

REF_API int ref_quantize_unit(const float* values, int n, int bits, uint8_t* codes, float* scale,
                              int64_t* zero_point) {
    return guarded([&] {
        auto q = rdkv::quantize_unit(std::span<const float>(values, n), bits);
        std::memcpy(codes, q.codes.data(), n);
        *scale = q.params.scale;
        *zero_point = q.params.zero_point;
    });
}

REF_API int ref_mckp_bisect(const float* w, int n, const int* widths, const double* eps, int n_widths,
                            double target, double tolerance, int max_iterations, int strict_budget,
                            int* bits, double* lambda, double* avg, double* objective,
                            int* converged) {
    return guarded([&] {
        rdkv::DistortionTable t;
        for (int i = 0; i < n_widths; ++i) t.eps.emplace_back(widths[i], eps[i]);
        rdkv::BitSet b;
        b.widths.assign(widths, widths + n_widths);
        rdkv::SolverConfig cfg;
        cfg.tolerance = tolerance;
        cfg.max_iterations = max_iterations;
        cfg.strict_budget = strict_budget != 0;
        auto a = rdkv::mckp_bisect(std::span<const float>(w, n), t, target, b, cfg);
        std::memcpy(bits, a.bits.data(), sizeof(int) * a.bits.size());
        *lambda = a.lambda;
        *avg = a.achieved_avg_bits;
        *objective = a.objective;
        *converged = a.converged;
    });
}

REF_API int ref_allocate_head(const float* k, const float* probe_group, int t_len, int d, int group,
                              int probe_rows, int kv_heads, const Cfg* cfg, int* v_bits, int* k_bits,
                              float* v_weights, float* k_weights, Stats* st) {
    return guarded([&] {
        // a one-layer cache whose KV head `0` holds this head; the other KV
        // heads (needed only for the H_kv budget split) are never touched
        rdkv::KVCache c;
        c.shape = rdkv::CacheShape{1, group * kv_heads, kv_heads, d, t_len};
        c.probe_window = probe_rows;
        auto& kt = c.k.emplace_back(kv_heads, t_len, d);
        std::memcpy(kt.data().data(), k, sizeof(float) * static_cast<std::size_t>(t_len) * d);
        c.v.emplace_back(kv_heads, t_len, d);
        auto& qt = c.probe_q.emplace_back(group * kv_heads, probe_rows, d);
        std::memcpy(qt.data().data(), probe_group,
                    sizeof(float) * static_cast<std::size_t>(group) * probe_rows * d);
        auto h = rdkv::allocate_head(c, 0, 0, spec_of(*cfg), table_of(*cfg, true), table_of(*cfg, false),
                                     pipeline_of(*cfg));
        std::memcpy(v_bits, h.v_bits.data(), sizeof(int) * h.v_bits.size());
        std::memcpy(k_bits, h.k_bits.data(), sizeof(int) * h.k_bits.size());
        std::memcpy(v_weights, h.v_weights.data(), sizeof(float) * h.v_weights.size());
        std::memcpy(k_weights, h.k_weights.data(), sizeof(float) * h.k_weights.size());
        fill_stats(h, st);
    });
}

// ---- TriZone handles ----------------------------------------------------

REF_API void* ref_tz_build(const float* k, const float* v, int t_len, int d, const int* v_bits,
                           const int* k_bits, int* status) {
    rdkv::TriZoneCache* out = nullptr;
    *status = guarded([&] {
        rdkv::HeadAllocation h;
        h.v_bits.assign(v_bits, v_bits + t_len);
        if (k_bits) h.k_bits.assign(k_bits, k_bits + d);
        for (int t = 0; t < t_len; ++t) {
            if (h.v_bits[t] > 0) {
                h.kept.kept.push_back(t);
                if (h.v_bits[t] == 16) h.kept.v16.push_back(t);
            } else {
                h.kept.evicted.push_back(t);
            }
        }
        out = new rdkv::TriZoneCache(
            rdkv::build_trizone(rdkv::MatrixView{k, t_len, d}, rdkv::MatrixView{v, t_len, d}, h));
    });
    return out;
}

REF_API void ref_tz_free(void* tz) { delete static_cast<rdkv::TriZoneCache*>(tz); }

REF_API int ref_tz_append(void* tz, const float* k, const float* v) {
    auto* c = static_cast<rdkv::TriZoneCache*>(tz);
    return guarded([&] {
        rdkv::append_new_token(*c, std::span<const float>(k, c->head_dim),
                               std::span<const float>(v, c->head_dim));
    });
}

REF_API int ref_tz_fused_logits(const void* tz, const float* q, double* out) {
    const auto* c = static_cast<const rdkv::TriZoneCache*>(tz);
    return guarded([&] {
        auto r = rdkv::fused_k_logits(std::span<const float>(q, c->head_dim), *c);
        std::memcpy(out, r.data(), sizeof(double) * r.size());
    });
}

REF_API int ref_tz_decode(const void* tz, const float* q, double* out) {
    const auto* c = static_cast<const rdkv::TriZoneCache*>(tz);
    return guarded([&] {
        auto r = rdkv::packed_decode_step(std::span<const float>(q, c->head_dim), *c);
        std::memcpy(out, r.data(), sizeof(double) * r.size());
    });
}

REF_API int ref_tz_n_kept(const void* tz) {
    return static_cast<int>(static_cast<const rdkv::TriZoneCache*>(tz)->kept.size());
}

REF_API size_t ref_tz_payload_bytes(const void* tz) {
    const auto* c = static_cast<const rdkv::TriZoneCache*>(tz);
    std::size_t n = 0;
    for (const auto& s : c->zone_a_v) n += s.payload.size();
    for (const auto& s : c->zone_a_k) n += s.payload.size();
    return n;
}

REF_API int ref_tz_canon(const void* tz, int* kept, uint8_t* vcodes, float* vscale, int64_t* vzero,
                         uint8_t* kcodes, float* kscale, int64_t* kzero, float* vfp, float* kfp,
                         uint8_t* payload, int* segtab, int* nseg, int* perm, int* nperm) {
    return canon_of(*static_cast<const rdkv::TriZoneCache*>(tz), kept, vcodes, vscale, vzero, kcodes,
                    kscale, kzero, vfp, kfp, payload, segtab, nseg, perm, nperm);
}

// ---- calibrate_epsilon (quantizer.cpp:200-284) over n_caches caches of one shape, stored
// back to back (k, v [n][L][H_kv][T][d], q [n][L][H_q][S_w][d]); eps_out [n_widths].
REF_API int ref_calibrate(const float* k, const float* v, const float* q, int n_caches, int layers,
                          int q_heads, int kv_heads, int d, int t_len, int probe_rows, int granularity,
                          const int* widths, int n_widths, double* eps_out, long long* units_out) {
    return guarded([&] {
        std::vector<rdkv::KVCache> caches;
        const std::size_t kv_n = std::size_t(layers) * kv_heads * t_len * d;
        const std::size_t q_n = std::size_t(layers) * q_heads * probe_rows * d;
        for (int c = 0; c < n_caches; ++c)
            caches.push_back(cache_from(k + c * kv_n, v + c * kv_n, q + c * q_n, layers, q_heads, kv_heads,
                                        d, t_len, probe_rows));
        rdkv::BitSet bits;
        bits.widths.assign(widths, widths + n_widths);
        auto t = rdkv::calibrate_epsilon(caches, granularity == 0 ? rdkv::Granularity::token
                                                                  : rdkv::Granularity::channel,
                                         bits);
        for (int i = 0; i < n_widths; ++i) eps_out[i] = t.eps[i].second;
        *units_out = std::stoll(t.provenance.substr(t.provenance.find("), ") + 3));
    });
}

// ---- run_sweep (sweep.cpp:40-114) over n_caches caches of one shape; rows [n_rows][5] =
// (seq_id, avg_bits, primal, dual, feasible) in the reference's (avg_bits, seq_id) order.
REF_API int ref_run_sweep(const float* k, const float* v, const float* q, int n_caches, int layers,
                          int q_heads, int kv_heads, int d, int t_len, int probe_rows, const double* grid,
                          int n_grid, const Cfg* cfg, double* rows) {
    return guarded([&] {
        std::vector<rdkv::KVCache> caches;
        const std::size_t kv_n = std::size_t(layers) * kv_heads * t_len * d;
        const std::size_t q_n = std::size_t(layers) * q_heads * probe_rows * d;
        for (int c = 0; c < n_caches; ++c)
            caches.push_back(cache_from(k + c * kv_n, v + c * kv_n, q + c * q_n, layers, q_heads, kv_heads,
                                        d, t_len, probe_rows));
        const auto p = pipeline_of(*cfg);
        auto r = rdkv::run_sweep(caches, std::span<const double>(grid, n_grid), table_of(*cfg, true),
                                 table_of(*cfg, false), bitset_of(*cfg), p.solver, p.probe);
        for (std::size_t i = 0; i < r.rows.size(); ++i) {
            rows[5 * i + 0] = r.rows[i].seq_id;
            rows[5 * i + 1] = r.rows[i].avg_bits;
            rows[5 * i + 2] = r.rows[i].primal;
            rows[5 * i + 3] = r.rows[i].dual;
            rows[5 * i + 4] = r.rows[i].feasible ? 1.0 : 0.0;
        }
    });
}

// ---- whole-model driver (CPU baseline) -----------------------------------

REF_API void* ref_model_build(const float* k, const float* v, const float* q, int layers, int q_heads,
                              int kv_heads, int d, int t_len, int probe_rows, const Cfg* cfg,
                              double* alloc_seconds, double* pack_seconds, int* status) {
    RefModel* m = nullptr;
    *status = guarded([&] {
        auto* mm = new RefModel;
        try {
            mm->cache = cache_from(k, v, q, layers, q_heads, kv_heads, d, t_len, probe_rows);
            auto t0 = std::chrono::steady_clock::now();
            mm->alloc = rdkv::allocate_model(mm->cache, spec_of(*cfg), table_of(*cfg, true),
                                             table_of(*cfg, false), pipeline_of(*cfg));
            *alloc_seconds = seconds_since(t0);
            t0 = std::chrono::steady_clock::now();
            mm->packed = rdkv::build_packed_model(mm->cache, mm->alloc);
            *pack_seconds = seconds_since(t0);
        } catch (...) {
            delete mm;
            throw;
        }
        m = mm;
    });
    return m;
}

REF_API void ref_model_free(void* m) { delete static_cast<RefModel*>(m); }

REF_API int ref_model_head(const void* mp, int layer, int head, int* v_bits, int* k_bits,
                           float* v_weights, float* k_weights, Stats* st) {
    const auto* m = static_cast<const RefModel*>(mp);
    return guarded([&] {
        const auto& h = m->alloc.at(layer, head);
        std::memcpy(v_bits, h.v_bits.data(), sizeof(int) * h.v_bits.size());
        std::memcpy(k_bits, h.k_bits.data(), sizeof(int) * h.k_bits.size());
        std::memcpy(v_weights, h.v_weights.data(), sizeof(float) * h.v_weights.size());
        std::memcpy(k_weights, h.k_weights.data(), sizeof(float) * h.k_weights.size());
        fill_stats(h, st);
    });
}

REF_API const void* ref_model_trizone(const void* mp, int layer, int head) {
    const auto* m = static_cast<const RefModel*>(mp);
    return &m->packed.at(layer, head);
}

// One decode step: packed_decode_step for every (layer, q-head), fanned out
// over (layer, kv-head) with the reference's own parallel_for (as
// BASELINE.md §4 prescribes). q/out are [layers][q_heads][d].
REF_API int ref_model_decode(const void* mp, const float* q, double* out, double* seconds) {
    const auto* m = static_cast<const RefModel*>(mp);
    return guarded([&] {
        const auto& s = m->cache.shape;
        const int g = s.group();
        const int d = s.head_dim;
        auto t0 = std::chrono::steady_clock::now();
        rdkv::parallel_for(s.layers * s.kv_heads, [&](int i) {
            const int layer = i / s.kv_heads;
            const int head = i % s.kv_heads;
            const auto& tz = m->packed.at(layer, head);
            for (int j = 0; j < g; ++j) {
                const std::size_t row = (static_cast<std::size_t>(layer) * s.q_heads + head * g + j) * d;
                auto r = rdkv::packed_decode_step(std::span<const float>(q + row, d), tz);
                std::memcpy(out + row, r.data(), sizeof(double) * d);
            }
        });
        *seconds = seconds_since(t0);
    });
}

REF_API int ref_worker_count() { return rdkv::worker_count(); }
