// dropin.cpp — the reference's C++ API (namespace rdkv) for the
// allocate -> pack -> decode path, implemented over the C-ABI of
// librdkv_b200.so (include/rdkv_cuda.h). Declarations and per-function
// reference citations: include/rdkv/cuda.hpp.
//
// Host-side work here is limited to argument validation (same checks, same
// exception types as the reference), layout conversion between the
// reference's value types and device buffers, and copies. All arithmetic of
// the path — probe softmax, weights, bisection, quantisation, packing,
// logits and attention — runs in the device kernels.
#include "rdkv/cuda.hpp"

#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <stdexcept>
#include <string>

#include "../../include/rdkv_cuda.h"
#include "../csrc/tile_layout.h"

namespace rdkv::cuda {
namespace {

// ---- errors -----------------------------------------------------------------
void require(bool ok, const char* msg) {
    if (!ok) throw std::invalid_argument(msg);
}

void check(int st, const char* what) {
    if (st == RDKV_OK) return;
    const std::string msg = std::string(what) + ": " + rdkv_status_string(st);
    switch (st) {
        case RDKV_EINVAL: throw std::invalid_argument(msg);
        case RDKV_ENUMERIC: throw NumericError(msg);
        case RDKV_EFORMAT: throw FormatError(msg);
        default: throw std::runtime_error(msg);
    }
}

void cuda_check(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw std::runtime_error(std::string(what) + ": " + cudaGetErrorString(e));
}

// ---- device buffers (legacy default stream: every call below is ordered) ----
class DevBuf {
public:
    DevBuf() = default;
    explicit DevBuf(std::size_t bytes) : n_(bytes) {
        cuda_check(cudaMalloc(&p_, std::max<std::size_t>(bytes, 16)), "cudaMalloc");
    }
    DevBuf(DevBuf&& o) noexcept : p_(o.p_), n_(o.n_) { o.p_ = nullptr; o.n_ = 0; }
    DevBuf& operator=(DevBuf&& o) noexcept {
        std::swap(p_, o.p_);
        std::swap(n_, o.n_);
        return *this;
    }
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    ~DevBuf() {
        if (p_) cudaFree(p_);
    }
    template <typename T>
    T* as() const { return static_cast<T*>(p_); }
    void* get() const { return p_; }
    std::size_t size() const { return n_; }

private:
    void* p_ = nullptr;
    std::size_t n_ = 0;
};

template <typename T>
DevBuf to_device(const T* src, std::size_t count) {
    DevBuf b(count * sizeof(T));
    if (count) cuda_check(cudaMemcpy(b.get(), src, count * sizeof(T), cudaMemcpyHostToDevice), "H2D");
    return b;
}

template <typename T>
std::vector<T> to_host(const void* src, std::size_t count) {
    std::vector<T> out(count);
    if (count) cuda_check(cudaMemcpy(out.data(), src, count * sizeof(T), cudaMemcpyDeviceToHost), "D2H");
    return out;
}

void sync() { cuda_check(cudaDeviceSynchronize(), "cudaDeviceSynchronize"); }

// ---- argument checks (restated from the reference, same exception types) ----
void check_finite(MatrixView m, const char* what) {  // cache.cpp:52-60
    const std::size_t n = static_cast<std::size_t>(m.rows) * m.cols;
    for (std::size_t i = 0; i < n; ++i)
        if (!std::isfinite(m.data[i])) throw NumericError(std::string(what) + ": non-finite entry");
}

bool is_quant_width(int b) { return b == 2 || b == 4 || b == 8; }

void validate_bits_relaxed(const BitSet& bits) {  // quantizer.cpp:66-80
    require(!bits.widths.empty(), "BitSet: empty");
    for (std::size_t i = 0; i < bits.widths.size(); ++i) {
        const int b = bits.widths[i];
        require(b >= 0 && b <= 16 && b % 2 == 0, "BitSet: widths must be even and within [0, 16]");
        require(i == 0 || b > bits.widths[i - 1], "BitSet: widths must be strictly increasing");
    }
    for (int b : bits.widths)
        require(b == 0 || b == 16 || is_quant_width(b), "BitSet: finite widths must be 2, 4 or 8");
}

void validate_bits(const BitSet& bits) {  // quantizer.cpp:82-87
    validate_bits_relaxed(bits);
    const auto has = [&](int b) { return std::find(bits.widths.begin(), bits.widths.end(), b) != bits.widths.end(); };
    require(has(0) && has(16), "BitSet: must contain both 0 and 16");
}

void validate_spec(const BudgetSpec& spec) {  // pipeline.cpp:52-58
    require(spec.n_tokens >= 1, "BudgetSpec: n_tokens must be >= 1");
    require(spec.r_k > 0.0 && spec.r_k < 1.0, "BudgetSpec: r_k must be in (0, 1)");
    validate_bits(spec.bits);
}

void validate_probe(const ProbeConfig& p) {  // cache.cpp:107-112
    require(p.window >= 1, "ProbeConfig: window must be >= 1");
    require(p.pool_kernel >= 1 && p.pool_kernel % 2 == 1, "ProbeConfig: pool_kernel must be odd and >= 1");
}

void validate_solver(const SolverConfig& c) {  // allocator.cpp:73-76
    require(c.tolerance > 0.0, "SolverConfig: tolerance must be > 0");
    require(c.max_iterations >= 1, "SolverConfig: max_iterations must be >= 1");
}

void validate_shape(const CacheShape& s) {  // cache.cpp:95-105
    require(s.layers >= 1 && s.head_dim >= 1 && s.seq_len >= 1,
            "CacheShape: layers, head_dim, seq_len must be >= 1");
    require(s.q_heads >= 1 && s.kv_heads >= 1, "CacheShape: head counts must be >= 1");
    require(s.q_heads % s.kv_heads == 0, "CacheShape: q_heads must be a multiple of kv_heads");
}

void validate_cache(const KVCache& c) {  // cache.cpp:114-138
    const auto& s = c.shape;
    validate_shape(s);
    require(c.probe_window >= 1 && c.probe_window <= s.seq_len, "KVCache: probe window must be in [1, seq_len]");
    require(static_cast<int>(c.k.size()) == s.layers && static_cast<int>(c.v.size()) == s.layers &&
                static_cast<int>(c.probe_q.size()) == s.layers,
            "KVCache: layer count mismatch");
    auto expect = [](const std::vector<Tensor3>& ts, int n0, int n1, int n2, const char* what) {
        for (const auto& t : ts) {
            if (t.dim0() != n0 || t.dim1() != n1 || t.dim2() != n2)
                throw std::invalid_argument(std::string("KVCache: bad tensor shape for ") + what);
            for (float x : t.data())
                if (!std::isfinite(x)) throw NumericError(std::string("KVCache: non-finite entry in ") + what);
        }
    };
    expect(c.k, s.kv_heads, s.seq_len, s.head_dim, "K");
    expect(c.v, s.kv_heads, s.seq_len, s.head_dim, "V");
    expect(c.probe_q, s.q_heads, c.probe_window, s.head_dim, "probe_Q");
}

// make_argmin_table (allocator.cpp:32-37): widths of the bit set with their
// eps; `missing` collects widths absent from the table instead of throwing
// (callers decide when the reference would have looked them up).
void argmin_table(const DistortionTable& eps, const BitSet& bits, int32_t* widths, double* e, int* missing) {
    *missing = -1;
    for (std::size_t i = 0; i < bits.widths.size(); ++i) {
        widths[i] = bits.widths[i];
        e[i] = 0.0;
        bool found = false;
        for (const auto& [b, v] : eps.eps)
            if (b == bits.widths[i]) {
                e[i] = v;
                found = true;
                break;
            }
        if (!found && *missing < 0) *missing = bits.widths[i];
    }
}

[[noreturn]] void throw_missing_width(int b) {  // quantizer.cpp:171-177
    throw std::invalid_argument("DistortionTable: no entry for bit-width " + std::to_string(b));
}

rdkv_config make_config(const BudgetSpec& spec, const DistortionTable& eps_v, const DistortionTable& eps_k,
                        const PipelineConfig& cfg, int* missing_v, int* missing_k) {
    rdkv_config c{};
    c.n_tokens = spec.n_tokens;
    c.r_k = spec.r_k;
    require(spec.bits.widths.size() <= 8, "BitSet: too many widths");
    c.n_widths = static_cast<int32_t>(spec.bits.widths.size());
    int32_t wk[8];
    argmin_table(eps_v, spec.bits, c.widths, c.eps_v, missing_v);
    argmin_table(eps_k, spec.bits, wk, c.eps_k, missing_k);
    c.window = cfg.probe.window;
    c.pool_kernel = cfg.probe.pool_kernel;
    c.tolerance = cfg.solver.tolerance;
    c.max_iterations = cfg.solver.max_iterations;
    c.strict_budget = cfg.solver.strict_budget ? 1 : 0;
    c.force_window_retain = cfg.force_window_retain ? 1 : 0;
    return c;
}

KeptSets derive_kept(const std::vector<int>& v_bits) {  // pipeline.cpp:19-30
    KeptSets s;
    for (int t = 0; t < static_cast<int>(v_bits.size()); ++t) {
        if (v_bits[t] > 0) {
            s.kept.push_back(t);
            if (v_bits[t] == 16) s.v16.push_back(t);
        } else {
            s.evicted.push_back(t);
        }
    }
    return s;
}

// ---- device allocation of `units` heads -----------------------------------
// k: [units][T][d], probe_q: [units][g][probe_rows][d] (host f32, contiguous
// per unit via the pointers in `k_src` / `q_src`).
std::vector<HeadAllocation> allocate_units(const std::vector<const float*>& k_src,
                                           const std::vector<const float*>& q_src, int T, int d, int g,
                                           int probe_rows, int kv_heads, const BudgetSpec& spec,
                                           const DistortionTable& eps_v, const DistortionTable& eps_k,
                                           const PipelineConfig& cfg) {
    const int U = static_cast<int>(k_src.size());
    int miss_v, miss_k;
    const rdkv_config c = make_config(spec, eps_v, eps_k, cfg, &miss_v, &miss_k);
    validate_solver(cfg.solver);
    if (miss_v >= 0) throw_missing_width(miss_v);  // allocate_v always bisects (B_V > 0)

    const std::size_t kn = static_cast<std::size_t>(T) * d, qn = static_cast<std::size_t>(g) * probe_rows * d;
    DevBuf k_dev(U * kn * sizeof(float)), q_dev(U * qn * sizeof(float));
    for (int u = 0; u < U; ++u) {
        cuda_check(cudaMemcpy(k_dev.as<float>() + u * kn, k_src[u], kn * sizeof(float), cudaMemcpyHostToDevice), "H2D");
        cuda_check(cudaMemcpy(q_dev.as<float>() + u * qn, q_src[u], qn * sizeof(float), cudaMemcpyHostToDevice), "H2D");
    }
    rdkv_shape s{U, T, d, g, probe_rows, kv_heads};
    const std::size_t ws_bytes = rdkv_cuda_weights_workspace(&s, c.window);
    DevBuf ws(ws_bytes), w_t(U * static_cast<std::size_t>(T) * sizeof(float)), w_c(U * static_cast<std::size_t>(d) * sizeof(float));
    check(rdkv_cuda_weights(k_dev.get(), q_dev.get(), RDKV_F32, &s, c.window, c.pool_kernel, w_t.as<float>(),
                            w_c.as<float>(), ws.get(), ws_bytes, nullptr),
          "attention_probe");
    DevBuf vb(U * static_cast<std::size_t>(T)), kb(U * static_cast<std::size_t>(d)), st(U * sizeof(rdkv_head_stats));
    check(rdkv_cuda_allocate(w_t.as<float>(), w_c.as<float>(), &s, &c, vb.as<uint8_t>(), kb.as<uint8_t>(),
                             st.as<rdkv_head_stats>(), nullptr),
          "allocate_head");
    sync();
    const auto v_bits = to_host<uint8_t>(vb.get(), U * static_cast<std::size_t>(T));
    const auto k_bits = to_host<uint8_t>(kb.get(), U * static_cast<std::size_t>(d));
    const auto wt = to_host<float>(w_t.get(), U * static_cast<std::size_t>(T));
    const auto wc = to_host<float>(w_c.get(), U * static_cast<std::size_t>(d));
    const auto stats = to_host<rdkv_head_stats>(st.get(), U);

    std::vector<HeadAllocation> out(U);
    for (int u = 0; u < U; ++u) {
        const auto& h = stats[u];
        if (h.status == RDKV_EINVAL)
            throw std::invalid_argument("mckp_bisect: weights must be finite and >= 0");
        check(h.status, "allocate_head");
        if (h.k_bits_len > 0 && miss_k >= 0) throw_missing_width(miss_k);  // allocate_k bisected
        HeadAllocation& a = out[u];
        a.v_bits.assign(v_bits.begin() + u * static_cast<std::size_t>(T), v_bits.begin() + (u + 1) * static_cast<std::size_t>(T));
        if (h.k_bits_len > 0)
            a.k_bits.assign(k_bits.begin() + u * static_cast<std::size_t>(d), k_bits.begin() + (u + 1) * static_cast<std::size_t>(d));
        a.kept = derive_kept(a.v_bits);
        a.v_weights.assign(wt.begin() + u * static_cast<std::size_t>(T), wt.begin() + (u + 1) * static_cast<std::size_t>(T));
        a.k_weights.assign(wc.begin() + u * static_cast<std::size_t>(d), wc.begin() + (u + 1) * static_cast<std::size_t>(d));
        a.objective_v = h.objective_v;
        a.objective_k = h.objective_k;
        a.achieved_bits = h.achieved_bits;
        a.lambda_v = h.lambda_v;
        a.lambda_k = h.lambda_k;
        a.v_converged = h.v_converged != 0;
        a.k_converged = h.k_converged != 0;
    }
    return out;
}

// ---- tiles <-> TriZoneCache -------------------------------------------------
void check_alloc_for_pack(int t_len, int d, const HeadAllocation& alloc) {  // trizone.cpp:94-120
    require(static_cast<int>(alloc.v_bits.size()) == t_len, "build_trizone: v_bits length must equal T");
    std::vector<int> derived;
    for (int t = 0; t < t_len; ++t)
        if (alloc.v_bits[t] > 0) derived.push_back(t);
    require(derived == alloc.kept.kept, "build_trizone: kept set inconsistent with v_bits");
    for (int t = 0; t < t_len; ++t)
        require(alloc.v_bits[t] == 0 || alloc.v_bits[t] == 16 || is_quant_width(alloc.v_bits[t]),
                "build_trizone: v_bits must be 0, 2, 4, 8 or 16");
    if (derived.empty()) {
        require(alloc.k_bits.empty() || static_cast<int>(alloc.k_bits.size()) == d,
                "build_trizone: k_bits length must equal d");
        return;
    }
    require(static_cast<int>(alloc.k_bits.size()) == d, "build_trizone: k_bits length must equal d");
    for (int b : alloc.k_bits)
        require(b == 0 || b == 16 || is_quant_width(b), "build_trizone: k_bits must be 0, 2, 4, 8 or 16");
    std::size_t v16 = 0;
    for (int t : alloc.kept.kept) v16 += alloc.v_bits[t] == 16;
    require(alloc.kept.v16.size() == v16, "build_trizone: v16 set inconsistent with v_bits");
    for (int t : alloc.kept.v16) require(alloc.v_bits[t] == 16, "build_trizone: v16 set inconsistent with v_bits");
}

// Device pack of `units` heads; returns the host copy of the arena and the
// tile offsets (the device arena is kept in *arena_dev when requested).
std::vector<uint8_t> pack_units(const std::vector<const float*>& k_src, const std::vector<const float*>& v_src,
                                const std::vector<const HeadAllocation*>& allocs, int T, int d,
                                std::vector<int64_t>& offsets, DevBuf* arena_dev, DevBuf* offsets_dev) {
    const int U = static_cast<int>(k_src.size());
    const std::size_t kn = static_cast<std::size_t>(T) * d;
    DevBuf k_dev(U * kn * sizeof(float)), v_dev(U * kn * sizeof(float));
    std::vector<uint8_t> vb(U * static_cast<std::size_t>(T)), kb(U * static_cast<std::size_t>(d), 0);
    for (int u = 0; u < U; ++u) {
        cuda_check(cudaMemcpy(k_dev.as<float>() + u * kn, k_src[u], kn * sizeof(float), cudaMemcpyHostToDevice), "H2D");
        cuda_check(cudaMemcpy(v_dev.as<float>() + u * kn, v_src[u], kn * sizeof(float), cudaMemcpyHostToDevice), "H2D");
        const HeadAllocation& a = *allocs[u];
        for (int t = 0; t < T; ++t) vb[u * static_cast<std::size_t>(T) + t] = static_cast<uint8_t>(a.v_bits[t]);
        if (!a.kept.kept.empty())
            for (int c = 0; c < d; ++c) kb[u * static_cast<std::size_t>(d) + c] = static_cast<uint8_t>(a.k_bits[c]);
    }
    DevBuf vb_dev = to_device(vb.data(), vb.size()), kb_dev = to_device(kb.data(), kb.size());
    rdkv_shape s{U, T, d, 1, 1, 1};
    DevBuf off_dev((U + 1) * sizeof(int64_t));
    check(rdkv_cuda_pack_plan(vb_dev.as<uint8_t>(), kb_dev.as<uint8_t>(), &s, off_dev.as<int64_t>(), nullptr),
          "build_trizone");
    sync();
    offsets = to_host<int64_t>(off_dev.get(), U + 1);
    DevBuf arena(static_cast<std::size_t>(offsets[U]));
    DevBuf status(U * sizeof(int32_t));
    check(rdkv_cuda_pack(k_dev.get(), v_dev.get(), RDKV_F32, vb_dev.as<uint8_t>(), kb_dev.as<uint8_t>(), &s,
                         off_dev.as<int64_t>(), arena.as<uint8_t>(), status.as<int32_t>(), nullptr),
          "build_trizone");
    sync();
    for (int32_t st : to_host<int32_t>(status.get(), U))
        if (st == RDKV_ENUMERIC) throw NumericError("quantize_unit: non-finite value");
        else check(st, "build_trizone");
    auto host = to_host<uint8_t>(arena.get(), static_cast<std::size_t>(offsets[U]));
    if (arena_dev) *arena_dev = std::move(arena);
    if (offsets_dev) *offsets_dev = std::move(off_dev);
    return host;
}

// Canonical export of one tile -> reference TriZoneCache (trizone.hpp:62-78).
// fp_k / fp_v: the source K/V rows ([T][d]) for the Zone B / k16 values (the
// reference copies the source floats); null -> the fp16 values of the tile.
TriZoneCache tile_to_trizone(const uint8_t* tile, int d, const std::vector<int>& v_bits,
                             const std::vector<int>& k_bits, const float* fp_k, const float* fp_v) {
    TriZoneCache out;
    out.head_dim = d;
    out.v_bits = v_bits;
    const KeptSets sets = derive_kept(v_bits);
    out.kept = sets.kept;
    out.evicted = sets.evicted;
    const int n = static_cast<int>(out.kept.size());
    if (n == 0) {  // trizone.cpp:113-118
        out.k_bits.assign(d, 0);
        return out;
    }
    out.k_bits = k_bits;
    const std::size_t nb = rdkv_tile_export_payload_bytes(tile, d);
    std::vector<int32_t> kept(n), segtab(36), perm(d);
    std::vector<uint8_t> vcodes(static_cast<std::size_t>(n) * d), kcodes(static_cast<std::size_t>(n) * d),
        payload(std::max<std::size_t>(nb, 1));
    std::vector<float> vscale(n), kscale(d), vfp(static_cast<std::size_t>(n) * d), kfp(static_cast<std::size_t>(n) * d);
    std::vector<int64_t> vzero(n), kzero(d);
    int32_t nseg = 0, nperm = 0;
    check(rdkv_tile_export(tile, d, kept.data(), vcodes.data(), vscale.data(), vzero.data(), kcodes.data(),
                           kscale.data(), kzero.data(), vfp.data(), kfp.data(), payload.data(), segtab.data(), &nseg,
                           perm.data(), &nperm),
          "tile export");
    for (int i = 0; i < n; ++i)
        if (kept[i] != out.kept[i]) throw FormatError("tile export: kept set differs from the allocation");
    std::size_t off = 0;
    for (int si = 0; si < nseg; ++si) {
        const int32_t* row = segtab.data() + 6 * si;
        PackedSegment seg;
        seg.bits = row[1];
        seg.rows = row[2];
        seg.logical_len = row[3];
        seg.pad_count = row[4];
        seg.payload.assign(payload.begin() + off, payload.begin() + off + row[5]);
        off += row[5];
        if (row[0] == 0) {  // V segment: members ascending token id (trizone.cpp:126-143)
            for (int p = 0; p < n; ++p) {
                if (v_bits[out.kept[p]] != seg.bits) continue;
                seg.members.push_back(out.kept[p]);
                seg.positions.push_back(p);
                seg.params.push_back(QuantParams{vscale[p], vzero[p], seg.bits});
            }
            out.zone_a_v.push_back(std::move(seg));
        } else {  // K segment (trizone.cpp:159-184)
            for (int c = 0; c < d; ++c) {
                if (k_bits[c] != seg.bits) continue;
                seg.members.push_back(c);
                seg.params.push_back(QuantParams{kscale[c], kzero[c], seg.bits});
            }
            out.zone_a_k.push_back(std::move(seg));
        }
    }
    out.zone_b.width = d;  // trizone.cpp:145-157
    for (int p = 0; p < n; ++p) {
        const int t = out.kept[p];
        if (v_bits[t] != 16) continue;
        out.zone_b.members.push_back(t);
        out.zone_b.positions.push_back(p);
        for (int c = 0; c < d; ++c)
            out.zone_b.data.push_back(fp_v ? fp_v[static_cast<std::size_t>(t) * d + c] : vfp[static_cast<std::size_t>(p) * d + c]);
    }
    for (int c = 0; c < d; ++c)  // trizone.cpp:186-199
        if (k_bits[c] == 16) out.k16.members.push_back(c);
    out.k16.width = static_cast<int>(out.k16.members.size());
    for (int p = 0; p < n && out.k16.width > 0; ++p)
        for (int c : out.k16.members)
            out.k16.data.push_back(fp_k ? fp_k[static_cast<std::size_t>(out.kept[p]) * d + c] : kfp[static_cast<std::size_t>(p) * d + c]);
    out.channel_perm.assign(perm.begin(), perm.begin() + nperm);
    return out;
}

unsigned extract_code(const uint8_t* row, int j, int bits) {  // trizone.cpp:26-32
    switch (bits) {
        case 2: return (row[j >> 2] >> ((j & 3) * 2)) & 3u;
        case 4: return (row[j >> 1] >> ((j & 1) * 4)) & 15u;
        default: return row[j];
    }
}

int row_bytes(int len, int bits) {  // packed_row_bytes, trizone.cpp:48-57
    const int padded = bits == 2 ? (len + 3) / 4 * 4 : bits == 4 ? (len + 1) / 2 * 2 : len;
    return padded * bits / 8;
}

// Reference TriZoneCache (Zones A/B) -> device tile bytes (rdkv_tile_import).
// Reads exactly what packed_decode_step reads (segments, params, positions),
// so tampered pad bits never reach the device tile.
std::vector<uint8_t> trizone_to_tile(const TriZoneCache& c, const char* who) {
    const int d = c.head_dim, n = static_cast<int>(c.kept.size());
    require(d >= 1, who);
    std::vector<uint8_t> vbits(std::max(n, 1), 0), kbits(d, 0);
    std::vector<uint8_t> vcodes(static_cast<std::size_t>(std::max(n, 1)) * d, 0), kcodes(static_cast<std::size_t>(std::max(n, 1)) * d, 0);
    std::vector<float> vscale(std::max(n, 1), 0.f), vfp(static_cast<std::size_t>(std::max(n, 1)) * d, 0.f), kscale(d, 0.f),
        kfp(static_cast<std::size_t>(std::max(n, 1)) * d, 0.f);
    std::vector<int64_t> vzero(std::max(n, 1), 0), kzero(d, 0);
    const std::string bad = std::string(who) + ": inconsistent TriZone cache";
    auto need = [&](bool ok) {
        if (!ok) throw std::invalid_argument(bad);
    };
    for (const auto& seg : c.zone_a_v) {
        need(is_quant_width(seg.bits) && seg.logical_len == d && seg.rows >= 0);
        need(seg.positions.size() >= static_cast<std::size_t>(seg.rows) && seg.params.size() >= static_cast<std::size_t>(seg.rows));
        const int rb = row_bytes(d, seg.bits);
        need(seg.payload.size() >= static_cast<std::size_t>(seg.rows) * rb);
        for (int i = 0; i < seg.rows; ++i) {
            const int p = seg.positions[i];
            need(p >= 0 && p < n && vbits[p] == 0);
            vbits[p] = static_cast<uint8_t>(seg.bits);
            vscale[p] = seg.params[i].scale;
            vzero[p] = seg.params[i].zero_point;
            const uint8_t* row = seg.payload.data() + static_cast<std::size_t>(i) * rb;
            for (int j = 0; j < d; ++j) vcodes[static_cast<std::size_t>(p) * d + j] = static_cast<uint8_t>(extract_code(row, j, seg.bits));
        }
    }
    need(c.zone_b.members.size() == c.zone_b.positions.size());
    need(c.zone_b.data.size() >= c.zone_b.members.size() * static_cast<std::size_t>(d));
    for (std::size_t i = 0; i < c.zone_b.members.size(); ++i) {
        const int p = c.zone_b.positions[i];
        need(p >= 0 && p < n && vbits[p] == 0);
        vbits[p] = 16;
        std::copy_n(c.zone_b.data.data() + i * d, d, vfp.data() + static_cast<std::size_t>(p) * d);
    }
    // A kept token without a V row (a hand-built cache) still takes part in
    // the softmax but adds nothing to the output (trizone.cpp:276-296): it is
    // imported as a zero fp16 row.
    for (int p = 0; p < n; ++p)
        if (vbits[p] == 0) vbits[p] = 16;
    for (const auto& seg : c.zone_a_k) {
        need(is_quant_width(seg.bits) && seg.rows == n && seg.logical_len == static_cast<int>(seg.members.size()));
        need(seg.params.size() >= seg.members.size());
        const int rb = row_bytes(seg.logical_len, seg.bits);
        need(seg.payload.size() >= static_cast<std::size_t>(n) * rb);
        for (int j = 0; j < seg.logical_len; ++j) {
            const int ch = seg.members[j];
            need(ch >= 0 && ch < d && kbits[ch] == 0);
            kbits[ch] = static_cast<uint8_t>(seg.bits);
            kscale[ch] = seg.params[j].scale;
            kzero[ch] = seg.params[j].zero_point;
            for (int r = 0; r < n; ++r)
                kcodes[static_cast<std::size_t>(ch) * n + r] =
                    static_cast<uint8_t>(extract_code(seg.payload.data() + static_cast<std::size_t>(r) * rb, j, seg.bits));
        }
    }
    if (c.k16.width > 0) {
        need(static_cast<int>(c.k16.members.size()) == c.k16.width);
        need(c.k16.data.size() >= static_cast<std::size_t>(n) * c.k16.width);
        for (int j = 0; j < c.k16.width; ++j) {
            const int ch = c.k16.members[j];
            need(ch >= 0 && ch < d && kbits[ch] == 0);
            kbits[ch] = 16;
            for (int r = 0; r < n; ++r) kfp[static_cast<std::size_t>(r) * d + ch] = c.k16.data[static_cast<std::size_t>(r) * c.k16.width + j];
        }
    }
    const std::size_t bytes = rdkv_tile_import_bytes(d, n, vbits.data(), kbits.data());
    need(bytes > 0);
    std::vector<uint8_t> tile(bytes);
    check(rdkv_tile_import(d, n, c.kept.data(), vbits.data(), vcodes.data(), vscale.data(), vzero.data(), vfp.data(),
                           kbits.data(), kcodes.data(), kscale.data(), kzero.data(), kfp.data(), tile.data(), bytes),
          who);
    return tile;
}

std::vector<__half> to_half(const float* x, std::size_t n) {
    std::vector<__half> out(n);
    for (std::size_t i = 0; i < n; ++i) out[i] = __float2half_rn(x[i]);
    return out;
}

// One decode launch over device tiles.
struct DecodeState {
    DevBuf arena, offsets, decode_sizes, unit_ids, zc_k, zc_v, zc_len;
    std::vector<int64_t> offsets_host;
    rdkv_decode_plan plan{};
    int units = 0, zc_cap = 0;

    void prepare() {
        decode_sizes = DevBuf(units * sizeof(int32_t));
        unit_ids = DevBuf(units * sizeof(int32_t));
        check(rdkv_cuda_decode_prepare_split(arena.as<uint8_t>(), offsets_host.data(), units,
                                             decode_sizes.as<int32_t>(), unit_ids.as<int32_t>(), &plan, nullptr),
              "decode prepare");
        sync();
    }
    // q/out: device f32 [units][g][d]
    void run(const float* q, float* out, int g, int d) const {
        rdkv_decode_args a{};
        a.arena = arena.as<uint8_t>();
        a.tile_offsets = offsets.as<int64_t>();
        a.units = units;
        a.group = g;
        a.head_dim = d;
        a.io_dtype = RDKV_F32;
        a.q = q;
        a.out = out;
        if (zc_cap > 0) {
            a.zc_k = zc_k.get();
            a.zc_v = zc_v.get();
            a.zc_len = zc_len.as<int32_t>();
            a.zc_cap = zc_cap;
        }
        a.split = 1;
        a.kernel = 0;
        a.tile_decode_bytes = decode_sizes.as<int32_t>();
        a.plan = plan;
        a.unit_ids = unit_ids.as<int32_t>();
        check(rdkv_cuda_decode(&a, nullptr), "packed_decode_step");
        sync();
    }
};

}  // namespace

// ---- Stage 1 ----------------------------------------------------------------
AttentionMatrix attention_probe(MatrixView q_window, MatrixView k, std::span<const int> causal_offsets) {
    require(q_window.cols == k.cols, "attention_probe: head_dim mismatch between Q and K");
    require(static_cast<int>(causal_offsets.size()) == q_window.rows,
            "attention_probe: one causal offset per query required");
    const int t_len = k.rows, d = k.cols, rows = q_window.rows;
    check_finite(q_window, "attention_probe Q");
    check_finite(k, "attention_probe K");
    for (int off : causal_offsets) require(off >= 0 && off < t_len, "attention_probe: causal offset out of [0, T)");
    AttentionMatrix out;
    out.rows = rows;
    out.cols = t_len;
    out.a.assign(static_cast<std::size_t>(rows) * t_len, 0.0);
    if (rows == 0 || t_len == 0) return out;
    require(d >= 1, "attention_probe: head_dim must be >= 1");
    DevBuf q = to_device(q_window.data, static_cast<std::size_t>(rows) * d);
    DevBuf kk = to_device(k.data, static_cast<std::size_t>(t_len) * d);
    DevBuf off = to_device(causal_offsets.data(), causal_offsets.size());
    const std::size_t ws_bytes = rdkv_cuda_attention_probe_workspace(rows, t_len);
    DevBuf ws(ws_bytes), a(out.a.size() * sizeof(double));
    check(rdkv_cuda_attention_probe(q.as<float>(), rows, kk.as<float>(), t_len, d, off.as<int32_t>(), a.as<double>(),
                                    ws.get(), ws_bytes, nullptr),
          "attention_probe");
    sync();
    cuda_check(cudaMemcpy(out.a.data(), a.get(), out.a.size() * sizeof(double), cudaMemcpyDeviceToHost), "D2H");
    return out;
}

std::vector<float> moving_average(std::span<const float> raw, int kernel) {
    require(kernel >= 1 && kernel % 2 == 1, "moving_average: kernel must be odd and >= 1");
    const int n = static_cast<int>(raw.size());
    if (n == 0) return {};
    DevBuf in = to_device(raw.data(), raw.size()), out(raw.size() * sizeof(float));
    check(rdkv_cuda_moving_average(in.as<float>(), n, kernel, out.as<float>(), nullptr), "moving_average");
    sync();
    return to_host<float>(out.get(), raw.size());
}

WeightVector token_weights(std::span<const AttentionMatrix> heads, int group, int pool_kernel) {
    require(!heads.empty(), "token_weights: no attention matrices");
    require(static_cast<int>(heads.size()) == group, "token_weights: group size does not match head count");
    const int t_len = heads.front().cols;
    std::size_t rows = 0;
    for (const auto& a : heads) {
        require(a.cols == t_len, "token_weights: attention matrices disagree on T");
        require(a.a.size() >= static_cast<std::size_t>(a.rows) * a.cols, "token_weights: attention matrix too small");
        rows += a.rows;
    }
    require(pool_kernel >= 1 && pool_kernel % 2 == 1, "moving_average: kernel must be odd and >= 1");
    WeightVector w;
    w.kind = WeightKind::token;
    if (t_len == 0) return w;
    // heads-outer, rows-inner (weights.cpp:34-40) == the stacked row order
    DevBuf a(std::max<std::size_t>(rows, 1) * t_len * sizeof(double));
    std::size_t r0 = 0;
    for (const auto& m : heads) {
        const std::size_t n = static_cast<std::size_t>(m.rows) * t_len;
        if (n)
            cuda_check(cudaMemcpy(a.as<double>() + r0 * t_len, m.a.data(), n * sizeof(double), cudaMemcpyHostToDevice),
                       "H2D");
        r0 += m.rows;
    }
    DevBuf raw(t_len * sizeof(float)), out(t_len * sizeof(float));
    if (rows == 0) cuda_check(cudaMemset(a.get(), 0, static_cast<std::size_t>(t_len) * sizeof(double)), "memset");
    check(rdkv_cuda_token_weights(a.as<double>(), 1, static_cast<int32_t>(std::max<std::size_t>(rows, 1)), t_len,
                                  pool_kernel, raw.as<float>(), out.as<float>(), nullptr),
          "token_weights");
    sync();
    w.values = to_host<float>(out.get(), t_len);
    return w;
}

WeightVector channel_weights(MatrixView q, MatrixView k) {
    require(q.cols == k.cols, "channel_weights: Q and K must share head_dim");
    const int d = q.cols;
    WeightVector w;
    w.kind = WeightKind::channel;
    if (d <= 0) return w;
    DevBuf qd = to_device(q.data, static_cast<std::size_t>(q.rows) * d), kd = to_device(k.data, static_cast<std::size_t>(k.rows) * d);
    DevBuf out(d * sizeof(float));
    check(rdkv_cuda_channel_weights(qd.as<float>(), q.rows, kd.as<float>(), k.rows, d, out.as<float>(), nullptr),
          "channel_weights");
    sync();
    w.values = to_host<float>(out.get(), d);
    return w;
}

// ---- Stages 2/3 -------------------------------------------------------------
DiscreteAllocation mckp_bisect(std::span<const float> weights, const DistortionTable& eps, double target_avg_bits,
                               const BitSet& bits, const SolverConfig& cfg) {
    validate_solver(cfg);
    for (float w : weights)  // check_weights (allocator.cpp:63-69)
        require(std::isfinite(w) && w >= 0.0f, "mckp_bisect: weights must be finite and >= 0");
    require(target_avg_bits > 0.0 && target_avg_bits <= 16.0, "mckp_bisect: target average bits must be in (0, 16]");
    validate_bits_relaxed(bits);
    require(bits.widths.size() <= 8, "BitSet: too many widths");
    int32_t widths[8];
    double e[8];
    int missing;
    argmin_table(eps, bits, widths, e, &missing);
    if (missing >= 0) throw_missing_width(missing);
    DiscreteAllocation out;
    out.bits.resize(weights.size());
    if (weights.empty()) {
        out.achieved_avg_bits = 0.0;
        return out;
    }
    const int n = static_cast<int>(weights.size());
    DevBuf w = to_device(weights.data(), weights.size()), b(weights.size()), r(sizeof(rdkv_bisect_result));
    check(rdkv_cuda_mckp_bisect(w.as<float>(), 1, n, widths, e, static_cast<int32_t>(bits.widths.size()),
                                target_avg_bits, cfg.tolerance, cfg.max_iterations, cfg.strict_budget ? 1 : 0,
                                b.as<uint8_t>(), r.as<rdkv_bisect_result>(), nullptr),
          "mckp_bisect");
    sync();
    const auto res = to_host<rdkv_bisect_result>(r.get(), 1)[0];
    if (res.status == RDKV_EINVAL) throw std::invalid_argument("mckp_bisect: weights must be finite and >= 0");
    check(res.status, "mckp_bisect");
    const auto bb = to_host<uint8_t>(b.get(), weights.size());
    std::copy(bb.begin(), bb.end(), out.bits.begin());
    out.lambda = res.lambda;
    out.achieved_avg_bits = res.achieved_avg_bits;
    out.objective = res.objective;
    out.converged = res.converged != 0;
    return out;
}

VAllocation allocate_v(const WeightVector& token_w, const DistortionTable& eps_v, double v_budget_bits, int head_dim,
                       const BitSet& bits, const SolverConfig& cfg) {  // pipeline.cpp:74-94
    require(token_w.kind == WeightKind::token, "allocate_v: token weights required");
    const int t_len = static_cast<int>(token_w.values.size());
    require(t_len >= 1, "allocate_v: empty sequence");
    VAllocation out;
    if (!(v_budget_bits > 0.0)) {
        out.v_bits.assign(t_len, 0);
        out.kept = derive_kept(out.v_bits);
        out.raw.bits = out.v_bits;
        return out;
    }
    const double target = std::min(16.0, v_budget_bits / (static_cast<double>(head_dim) * t_len));
    out.raw = rdkv::cuda::mckp_bisect(token_w.values, eps_v, target, bits, cfg);
    out.v_bits = out.raw.bits;
    out.kept = derive_kept(out.v_bits);
    return out;
}

DiscreteAllocation allocate_k(const WeightVector& channel_w, const DistortionTable& eps_k, double k_budget_bits,
                              int kept_count, const BitSet& bits, const SolverConfig& cfg) {  // pipeline.cpp:96-112
    require(channel_w.kind == WeightKind::channel, "allocate_k: channel weights required");
    const int d = static_cast<int>(channel_w.values.size());
    DiscreteAllocation out;
    if (kept_count == 0) return out;  // all tokens evicted: no K storage at all
    if (!(k_budget_bits > 0.0)) {
        out.bits.assign(d, 0);
        return out;
    }
    const double target = std::min(16.0, k_budget_bits / (static_cast<double>(kept_count) * d));
    return rdkv::cuda::mckp_bisect(channel_w.values, eps_k, target, bits, cfg);
}

HeadAllocation allocate_head(const KVCache& cache, int layer, int kv_head, const BudgetSpec& spec,
                             const DistortionTable& eps_v, const DistortionTable& eps_k, const PipelineConfig& cfg) {
    validate_spec(spec);
    validate_probe(cfg.probe);
    const auto& s = cache.shape;
    require(layer >= 0 && layer < s.layers && kv_head >= 0 && kv_head < s.kv_heads,
            "allocate_head: (layer, head) out of range");
    const int g = s.group();
    const MatrixView k = cache.k_head(layer, kv_head);
    const MatrixView q = cache.probe_group(layer, kv_head);
    check_finite(q, "attention_probe Q");
    check_finite(k, "attention_probe K");
    require(std::min(cfg.probe.window, cache.probe_window) <= s.seq_len, "attention_probe: causal offset out of [0, T)");
    auto heads = allocate_units({k.data}, {q.data}, s.seq_len, s.head_dim, g, cache.probe_window, s.kv_heads, spec,
                                eps_v, eps_k, cfg);
    return std::move(heads[0]);
}

ModelAllocation allocate_model(const KVCache& cache, const BudgetSpec& spec, const DistortionTable& eps_v,
                               const DistortionTable& eps_k, const PipelineConfig& cfg) {
    validate_cache(cache);
    validate_spec(spec);
    validate_probe(cfg.probe);
    const auto& s = cache.shape;
    std::vector<const float*> ks, qs;
    for (int l = 0; l < s.layers; ++l)
        for (int h = 0; h < s.kv_heads; ++h) {
            ks.push_back(cache.k_head(l, h).data);
            qs.push_back(cache.probe_group(l, h).data);
        }
    ModelAllocation out;
    out.shape = s;
    out.spec = spec;
    out.heads = allocate_units(ks, qs, s.seq_len, s.head_dim, s.group(), cache.probe_window, s.kv_heads, spec, eps_v,
                               eps_k, cfg);
    return out;
}

// ---- packing ----------------------------------------------------------------
std::vector<std::uint8_t> pack_bits(std::span<const std::uint8_t> codes, int bits) {  // trizone.cpp:59-75
    require(bits == 2 || bits == 4 || bits == 8, "pack_bits: bits must be 2, 4 or 8");
    const int per = 8 / bits;
    const std::size_t nbytes = (codes.size() + per - 1) / per;
    std::vector<std::uint8_t> out(nbytes, 0);
    DevBuf c = to_device(codes.data(), codes.size()), o(nbytes > 0 ? nbytes : 1), st(sizeof(int32_t));
    check(rdkv_cuda_pack_bits(codes.empty() ? nullptr : c.as<uint8_t>(), static_cast<int64_t>(codes.size()), bits,
                              o.as<uint8_t>(), st.as<int32_t>(), nullptr),
          "pack_bits");
    sync();
    require(to_host<int32_t>(st.get(), 1)[0] == RDKV_OK, "pack_bits: code overflows bit-width");
    if (nbytes) out = to_host<uint8_t>(o.get(), nbytes);
    return out;
}

std::vector<std::uint8_t> unpack_bits(std::span<const std::uint8_t> bytes, int bits, int logical_len) {  // :76-88
    require(bits == 2 || bits == 4 || bits == 8, "unpack_bits: bits must be 2, 4 or 8");
    const int per = 8 / bits;
    // a negative length wraps to a huge size_t in the reference's check: same exception
    require(logical_len >= 0 && static_cast<std::size_t>((logical_len + per - 1) / per) <= bytes.size(),
            "unpack_bits: byte buffer too short");
    if (logical_len == 0) return {};
    DevBuf b = to_device(bytes.data(), bytes.size()), o(static_cast<std::size_t>(logical_len));
    check(rdkv_cuda_unpack_bits(b.as<uint8_t>(), static_cast<int64_t>(bytes.size()), bits, logical_len,
                                o.as<uint8_t>(), nullptr),
          "unpack_bits");
    sync();
    return to_host<uint8_t>(o.get(), static_cast<std::size_t>(logical_len));
}

QuantizedUnit quantize_unit(std::span<const float> values, int bits) {
    require(is_quant_width(bits), "quantize_unit: bits must be 2, 4 or 8");
    require(!values.empty(), "quantize_unit: empty unit");
    const int n = static_cast<int>(values.size());
    DevBuf x = to_device(values.data(), values.size()), codes(values.size()), sc(sizeof(float)), zp(sizeof(int64_t)),
        st(sizeof(int32_t));
    check(rdkv_cuda_quantize_units(x.as<float>(), 1, n, bits, codes.as<uint8_t>(), sc.as<float>(), zp.as<int64_t>(),
                                   st.as<int32_t>(), nullptr),
          "quantize_unit");
    sync();
    if (to_host<int32_t>(st.get(), 1)[0] == RDKV_ENUMERIC) throw NumericError("quantize_unit: non-finite value");
    QuantizedUnit out;
    out.codes = to_host<uint8_t>(codes.get(), values.size());
    out.params.scale = to_host<float>(sc.get(), 1)[0];
    out.params.zero_point = to_host<int64_t>(zp.get(), 1)[0];
    out.params.bits = bits;
    return out;
}

TriZoneCache build_trizone(MatrixView k, MatrixView v, const HeadAllocation& alloc) {
    const int t_len = k.rows, d = k.cols;
    require(v.rows == t_len && v.cols == d, "build_trizone: K/V shape mismatch");
    check_alloc_for_pack(t_len, d, alloc);
    require(t_len >= 1 && d >= 1, "build_trizone: empty head");
    std::vector<int64_t> offsets;
    const auto arena = pack_units({k.data}, {v.data}, {&alloc}, t_len, d, offsets, nullptr, nullptr);
    const std::vector<int> kb = alloc.kept.kept.empty() ? std::vector<int>(d, 0) : alloc.k_bits;
    return tile_to_trizone(arena.data(), d, alloc.v_bits, kb, k.data, v.data);
}

PackedModel build_packed_model(const KVCache& cache, const ModelAllocation& alloc) {
    PackedModel model;
    model.shape = cache.shape;
    const auto& s = cache.shape;
    const int n = s.layers * s.kv_heads;
    require(static_cast<int>(alloc.heads.size()) == n, "build_packed_model: allocation does not match the cache");
    require(static_cast<int>(cache.k.size()) == s.layers && static_cast<int>(cache.v.size()) == s.layers,
            "KVCache: layer count mismatch");
    std::vector<const float*> ks, vs;
    std::vector<const HeadAllocation*> as;
    for (int i = 0; i < n; ++i) {
        const int l = i / s.kv_heads, h = i % s.kv_heads;
        check_alloc_for_pack(s.seq_len, s.head_dim, alloc.heads[i]);
        ks.push_back(cache.k_head(l, h).data);
        vs.push_back(cache.v_head(l, h).data);
        as.push_back(&alloc.heads[i]);
    }
    std::vector<int64_t> offsets;
    const auto arena = pack_units(ks, vs, as, s.seq_len, s.head_dim, offsets, nullptr, nullptr);
    model.heads.resize(n);
    for (int i = 0; i < n; ++i) {
        const auto& a = alloc.heads[i];
        const std::vector<int> kb = a.kept.kept.empty() ? std::vector<int>(s.head_dim, 0) : a.k_bits;
        model.heads[i] = tile_to_trizone(arena.data() + offsets[i], s.head_dim, a.v_bits, kb, ks[i], vs[i]);
    }
    return model;
}

// ---- decode -----------------------------------------------------------------
std::vector<double> fused_k_logits(std::span<const float> q, const TriZoneCache& cache) {
    require(static_cast<int>(q.size()) == cache.head_dim, "fused_k_logits: query dimension mismatch");
    const int n = static_cast<int>(cache.kept.size());
    std::vector<double> logits(n, 0.0);
    if (n == 0) return logits;
    const auto tile = trizone_to_tile(cache, "fused_k_logits");
    rdkv_b200::TileHeader h;
    std::memcpy(&h, tile.data(), sizeof(h));
    const int64_t offs[2] = {0, static_cast<int64_t>(tile.size())};
    DevBuf td = to_device(tile.data(), tile.size()), od = to_device(offs, 2), qd = to_device(q.data(), q.size());
    DevBuf ld(static_cast<std::size_t>(h.nslot) * sizeof(float));
    check(rdkv_cuda_tile_logits(td.as<uint8_t>(), od.as<int64_t>(), 1, 1, cache.head_dim, qd.as<float>(), h.nslot,
                                h.kslots, ld.as<float>(), nullptr),
          "fused_k_logits");
    sync();
    const auto per_slot = to_host<float>(ld.get(), h.nslot);
    const int32_t* ids = reinterpret_cast<const int32_t*>(tile.data() + h.off_ids);
    for (int s = 0; s < h.nslot; ++s) {
        if (ids[s] < 0) continue;
        const auto it = std::lower_bound(cache.kept.begin(), cache.kept.end(), ids[s]);
        logits[it - cache.kept.begin()] = per_slot[s];
    }
    return logits;
}

std::vector<double> packed_decode_step(std::span<const float> q, const TriZoneCache& cache) {
    require(static_cast<int>(q.size()) == cache.head_dim, "packed_decode_step: query dimension mismatch");
    const int n = static_cast<int>(cache.kept.size()), d = cache.head_dim;
    if (n + cache.zone_c_len == 0) throw NumericError("packed_decode_step: empty cache, softmax undefined");
    require(cache.zone_c_len >= 0 && cache.zone_c_k.size() >= static_cast<std::size_t>(cache.zone_c_len) * d &&
                cache.zone_c_v.size() >= static_cast<std::size_t>(cache.zone_c_len) * d,
            "packed_decode_step: Zone C shorter than zone_c_len");
    const auto tile = trizone_to_tile(cache, "packed_decode_step");
    DecodeState st;
    st.units = 1;
    st.offsets_host = {0, static_cast<int64_t>(tile.size())};
    st.arena = to_device(tile.data(), tile.size());
    st.offsets = to_device(st.offsets_host.data(), 2);
    if (cache.zone_c_len > 0) {
        const std::size_t zn = static_cast<std::size_t>(cache.zone_c_len) * d;
        const auto zk = to_half(cache.zone_c_k.data(), zn), zv = to_half(cache.zone_c_v.data(), zn);
        st.zc_k = to_device(zk.data(), zn);
        st.zc_v = to_device(zv.data(), zn);
        const int32_t len = cache.zone_c_len;
        st.zc_len = to_device(&len, 1);
        st.zc_cap = cache.zone_c_len;
    }
    st.prepare();
    DevBuf qd = to_device(q.data(), q.size()), od(q.size() * sizeof(float));
    st.run(qd.as<float>(), od.as<float>(), 1, d);
    const auto o = to_host<float>(od.get(), q.size());
    return std::vector<double>(o.begin(), o.end());
}

void append_new_token(TriZoneCache& cache, std::span<const float> k, std::span<const float> v) {
    require(static_cast<int>(k.size()) == cache.head_dim && static_cast<int>(v.size()) == cache.head_dim,
            "append_new_token: dimension mismatch");
    cache.zone_c_k.insert(cache.zone_c_k.end(), k.begin(), k.end());
    cache.zone_c_v.insert(cache.zone_c_v.end(), v.begin(), v.end());
    ++cache.zone_c_len;
}

// ---- DevicePackedModel ------------------------------------------------------
struct DevicePackedModel::Impl {
    CacheShape shape;
    DecodeState st;
    std::vector<std::vector<int>> v_bits, k_bits;  // per unit, for download()
    std::vector<int32_t> zc_len_host;
    std::size_t decode_bytes = 0;

    void init_zone_c(int cap) {
        const int U = st.units, d = shape.head_dim;
        st.zc_cap = cap;
        zc_len_host.assign(U, 0);
        if (cap <= 0) return;
        const std::size_t zn = static_cast<std::size_t>(U) * cap * d * sizeof(__half);
        st.zc_k = DevBuf(zn);
        st.zc_v = DevBuf(zn);
        cuda_check(cudaMemset(st.zc_k.get(), 0, zn), "memset");
        cuda_check(cudaMemset(st.zc_v.get(), 0, zn), "memset");
        st.zc_len = to_device(zc_len_host.data(), U);
    }
    void finish(const std::vector<uint8_t>& host_arena) {
        decode_bytes = 0;
        for (int u = 0; u < st.units; ++u) {
            rdkv_tile_info info;
            check(rdkv_tile_info_get(host_arena.data() + st.offsets_host[u], &info), "tile info");
            decode_bytes += static_cast<std::size_t>(info.decode_bytes);
        }
        st.prepare();
    }
};

DevicePackedModel::DevicePackedModel(std::unique_ptr<Impl> impl) : impl_(std::move(impl)) {}
DevicePackedModel::DevicePackedModel(DevicePackedModel&&) noexcept = default;
DevicePackedModel& DevicePackedModel::operator=(DevicePackedModel&&) noexcept = default;
DevicePackedModel::~DevicePackedModel() = default;

DevicePackedModel DevicePackedModel::build(const KVCache& cache, const ModelAllocation& alloc, int zone_c_capacity) {
    auto impl = std::make_unique<Impl>();
    const auto& s = cache.shape;
    validate_shape(s);
    const int n = s.layers * s.kv_heads;
    require(static_cast<int>(alloc.heads.size()) == n, "build_packed_model: allocation does not match the cache");
    std::vector<const float*> ks, vs;
    std::vector<const HeadAllocation*> as;
    for (int i = 0; i < n; ++i) {
        const int l = i / s.kv_heads, h = i % s.kv_heads;
        check_alloc_for_pack(s.seq_len, s.head_dim, alloc.heads[i]);
        ks.push_back(cache.k_head(l, h).data);
        vs.push_back(cache.v_head(l, h).data);
        as.push_back(&alloc.heads[i]);
        impl->v_bits.push_back(alloc.heads[i].v_bits);
        impl->k_bits.push_back(alloc.heads[i].kept.kept.empty() ? std::vector<int>(s.head_dim, 0) : alloc.heads[i].k_bits);
    }
    impl->shape = s;
    impl->st.units = n;
    const auto host = pack_units(ks, vs, as, s.seq_len, s.head_dim, impl->st.offsets_host, &impl->st.arena, &impl->st.offsets);
    impl->init_zone_c(zone_c_capacity);
    impl->finish(host);
    return DevicePackedModel(std::move(impl));
}

DevicePackedModel DevicePackedModel::upload(const PackedModel& model, int zone_c_capacity) {
    auto impl = std::make_unique<Impl>();
    const auto& s = model.shape;
    validate_shape(s);
    const int n = s.layers * s.kv_heads;
    require(static_cast<int>(model.heads.size()) == n, "DevicePackedModel: head count mismatch");
    std::vector<uint8_t> host;
    impl->st.offsets_host.push_back(0);
    int cap = zone_c_capacity;
    for (const auto& c : model.heads) {
        require(c.head_dim == s.head_dim, "DevicePackedModel: head_dim mismatch");
        const auto tile = trizone_to_tile(c, "DevicePackedModel::upload");
        host.insert(host.end(), tile.begin(), tile.end());
        impl->st.offsets_host.push_back(static_cast<int64_t>(host.size()));
        impl->v_bits.push_back(c.v_bits);
        impl->k_bits.push_back(c.k_bits);
        cap = std::max(cap, c.zone_c_len);
    }
    impl->shape = s;
    impl->st.units = n;
    impl->st.arena = to_device(host.data(), host.size());
    impl->st.offsets = to_device(impl->st.offsets_host.data(), impl->st.offsets_host.size());
    impl->init_zone_c(cap);
    if (cap > 0) {  // existing Zone C rows
        const int d = s.head_dim;
        for (int u = 0; u < n; ++u) {
            const auto& c = model.heads[u];
            if (c.zone_c_len == 0) continue;
            const std::size_t zn = static_cast<std::size_t>(c.zone_c_len) * d;
            require(c.zone_c_k.size() >= zn && c.zone_c_v.size() >= zn, "DevicePackedModel: Zone C shorter than zone_c_len");
            const auto zk = to_half(c.zone_c_k.data(), zn), zv = to_half(c.zone_c_v.data(), zn);
            const std::size_t at = static_cast<std::size_t>(u) * cap * d;
            cuda_check(cudaMemcpy(impl->st.zc_k.as<__half>() + at, zk.data(), zn * 2, cudaMemcpyHostToDevice), "H2D");
            cuda_check(cudaMemcpy(impl->st.zc_v.as<__half>() + at, zv.data(), zn * 2, cudaMemcpyHostToDevice), "H2D");
            impl->zc_len_host[u] = c.zone_c_len;
        }
        cuda_check(cudaMemcpy(impl->st.zc_len.get(), impl->zc_len_host.data(), n * sizeof(int32_t), cudaMemcpyHostToDevice),
                   "H2D");
    }
    impl->finish(host);
    return DevicePackedModel(std::move(impl));
}

const CacheShape& DevicePackedModel::shape() const { return impl_->shape; }
int DevicePackedModel::units() const { return impl_->st.units; }
std::size_t DevicePackedModel::arena_bytes() const { return static_cast<std::size_t>(impl_->st.offsets_host.back()); }
std::size_t DevicePackedModel::decode_bytes() const { return impl_->decode_bytes; }

std::vector<float> DevicePackedModel::decode(std::span<const float> q) const {
    const auto& s = impl_->shape;
    const std::size_t n = static_cast<std::size_t>(s.layers) * s.q_heads * s.head_dim;
    require(q.size() == n, "DevicePackedModel::decode: q must be [layers][q_heads][head_dim]");
    DevBuf qd = to_device(q.data(), n), od(n * sizeof(float));
    impl_->st.run(qd.as<float>(), od.as<float>(), s.group(), s.head_dim);
    return to_host<float>(od.get(), n);
}

void DevicePackedModel::append(std::span<const float> k, std::span<const float> v) {
    const auto& s = impl_->shape;
    const std::size_t n = static_cast<std::size_t>(impl_->st.units) * s.head_dim;
    require(k.size() == n && v.size() == n, "append_new_token: dimension mismatch");
    for (int32_t len : impl_->zc_len_host)
        require(len < impl_->st.zc_cap, "DevicePackedModel::append: Zone C capacity exhausted");
    DevBuf kd = to_device(k.data(), n), vd = to_device(v.data(), n);
    check(rdkv_cuda_append(impl_->st.zc_k.get(), impl_->st.zc_v.get(), impl_->st.zc_len.as<int32_t>(), impl_->st.zc_cap,
                           kd.get(), vd.get(), RDKV_F32, impl_->st.units, s.head_dim, nullptr),
          "append_new_token");
    sync();
    for (auto& len : impl_->zc_len_host) ++len;
}

PackedModel DevicePackedModel::download() const {
    const auto& s = impl_->shape;
    const int U = impl_->st.units, d = s.head_dim;
    const auto host = to_host<uint8_t>(impl_->st.arena.get(), arena_bytes());
    PackedModel m;
    m.shape = s;
    m.heads.reserve(U);
    for (int u = 0; u < U; ++u) {
        TriZoneCache c = tile_to_trizone(host.data() + impl_->st.offsets_host[u], d, impl_->v_bits[u], impl_->k_bits[u],
                                         nullptr, nullptr);
        const int len = impl_->zc_len_host[u];
        if (len > 0) {
            const std::size_t at = static_cast<std::size_t>(u) * impl_->st.zc_cap * d, zn = static_cast<std::size_t>(len) * d;
            const auto zk = to_host<__half>(impl_->st.zc_k.as<__half>() + at, zn);
            const auto zv = to_host<__half>(impl_->st.zc_v.as<__half>() + at, zn);
            for (std::size_t i = 0; i < zn; ++i) {
                c.zone_c_k.push_back(__half2float(zk[i]));
                c.zone_c_v.push_back(__half2float(zv[i]));
            }
            c.zone_c_len = len;
        }
        m.heads.push_back(std::move(c));
    }
    return m;
}


// ---- §8(f): dual bound, rate sweep, ε calibration ------------------------------
DualBound dual_bound(std::span<const float> weights, const DistortionTable& eps, double lambda,
                     double total_budget, const BitSet& bits) {
    require(lambda >= 0.0 && std::isfinite(lambda), "dual_bound: lambda must be >= 0");  // allocator.cpp:220-222
    for (float w : weights)
        require(std::isfinite(w) && w >= 0.0f, "dual_bound: weights must be finite and >= 0");
    validate_bits_relaxed(bits);
    require(bits.widths.size() <= 8, "BitSet: too many widths");
    int32_t widths[8];
    double e[8];
    int missing;
    argmin_table(eps, bits, widths, e, &missing);
    if (missing >= 0) throw_missing_width(missing);
    rdkv_bisect_result solved{};
    solved.lambda = lambda;
    const int n = static_cast<int>(weights.size());
    DevBuf w = to_device(weights.data(), std::max<std::size_t>(weights.size(), 1)), sv = to_device(&solved, 1),
           r(sizeof(rdkv_dual_bound_result));
    check(rdkv_cuda_dual_bound(w.as<float>(), 1, n, widths, e, static_cast<int32_t>(bits.widths.size()),
                               sv.as<rdkv_bisect_result>(), total_budget, r.as<rdkv_dual_bound_result>(), nullptr),
          "dual_bound");
    sync();
    const auto res = to_host<rdkv_dual_bound_result>(r.get(), 1)[0];
    check(res.status, "dual_bound");
    DualBound out;
    out.g_lambda = res.g_lambda;
    out.primal = res.primal;
    out.feasible = res.feasible != 0;
    out.gap = res.gap;
    return out;
}

SweepResult run_sweep(std::span<const KVCache> sequences, std::span<const double> grid, const DistortionTable& eps_v,
                      const DistortionTable& eps_k, const BitSet& bits, const SolverConfig& solver,
                      const ProbeConfig& probe) {
    require(!grid.empty(), "run_sweep: empty grid");  // sweep.cpp:43-49
    for (double b : grid) require(b > 0.0 && b <= 16.0, "run_sweep: grid values must be in (0, 16]");
    require(probe.window >= 1, "ProbeConfig: window must be >= 1");
    require(probe.pool_kernel >= 1 && probe.pool_kernel % 2 == 1, "ProbeConfig: pool_kernel must be odd and >= 1");
    validate_bits_relaxed(bits);
    require(bits.widths.size() <= 8, "BitSet: too many widths");
    validate_solver(solver);
    int32_t widths[8];
    double ev[8], ek[8];
    int miss_v, miss_k;
    argmin_table(eps_v, bits, widths, ev, &miss_v);
    argmin_table(eps_k, bits, widths, ek, &miss_k);
    const int nw = static_cast<int>(bits.widths.size());

    SweepResult result;
    for (int seq = 0; seq < static_cast<int>(sequences.size()); ++seq) {
        const KVCache& cache = sequences[seq];
        const auto& s = cache.shape;
        const int L = s.layers, Hkv = s.kv_heads, g = s.q_heads / s.kv_heads, T = s.seq_len, d = s.head_dim;
        const int Sw = cache.probe_window, U = L * Hkv;
        for (int l = 0; l < L; ++l) {  // cache.validate(): shapes + finiteness
            check_finite(MatrixView{cache.k[l].data().data(), Hkv * T, d}, "KVCache");
            check_finite(MatrixView{cache.v[l].data().data(), Hkv * T, d}, "KVCache");
            check_finite(MatrixView{cache.probe_q[l].data().data(), s.q_heads * Sw, d}, "KVCache");
        }
        const int window = std::min(probe.window, Sw);
        const std::size_t kn = static_cast<std::size_t>(T) * d, qn = static_cast<std::size_t>(g) * Sw * d;
        DevBuf k_dev(U * kn * sizeof(float)), q_dev(U * qn * sizeof(float));
        for (int l = 0; l < L; ++l) {  // unit order l * H_kv + h is the containers' own order
            cuda_check(cudaMemcpy(k_dev.as<float>() + l * Hkv * kn, cache.k[l].data().data(), Hkv * kn * sizeof(float),
                                  cudaMemcpyHostToDevice), "H2D");
            cuda_check(cudaMemcpy(q_dev.as<float>() + l * Hkv * qn, cache.probe_q[l].data().data(),
                                  Hkv * qn * sizeof(float), cudaMemcpyHostToDevice), "H2D");
        }
        rdkv_shape sh{U, T, d, g, Sw, Hkv};
        const std::size_t ws_bytes = rdkv_cuda_weights_workspace(&sh, window);
        DevBuf ws(ws_bytes), w_t(U * kn / d * sizeof(float) * 1), w_c(U * static_cast<std::size_t>(d) * sizeof(float));
        check(rdkv_cuda_weights(k_dev.get(), q_dev.get(), RDKV_F32, &sh, window, probe.pool_kernel, w_t.as<float>(),
                                w_c.as<float>(), ws.get(), ws_bytes, nullptr),
              "run_sweep");
        DevBuf bits_v(U * static_cast<std::size_t>(T)), bits_k(U * static_cast<std::size_t>(d));
        DevBuf rv(U * sizeof(rdkv_bisect_result)), rk(U * sizeof(rdkv_bisect_result));
        DevBuf dv(U * sizeof(rdkv_dual_bound_result)), dk(U * sizeof(rdkv_dual_bound_result));
        for (double target : grid) {
            if (miss_v >= 0) throw_missing_width(miss_v);
            if (miss_k >= 0) throw_missing_width(miss_k);
            check(rdkv_cuda_mckp_bisect(w_t.as<float>(), U, T, widths, ev, nw, target, solver.tolerance,
                                        solver.max_iterations, 1, bits_v.as<uint8_t>(), rv.as<rdkv_bisect_result>(),
                                        nullptr),
                  "mckp_bisect");
            check(rdkv_cuda_dual_bound(w_t.as<float>(), U, T, widths, ev, nw, rv.as<rdkv_bisect_result>(),
                                       target * static_cast<double>(T), dv.as<rdkv_dual_bound_result>(), nullptr),
                  "dual_bound");
            check(rdkv_cuda_mckp_bisect(w_c.as<float>(), U, d, widths, ek, nw, target, solver.tolerance,
                                        solver.max_iterations, 1, bits_k.as<uint8_t>(), rk.as<rdkv_bisect_result>(),
                                        nullptr),
                  "mckp_bisect");
            check(rdkv_cuda_dual_bound(w_c.as<float>(), U, d, widths, ek, nw, rk.as<rdkv_bisect_result>(),
                                       target * static_cast<double>(d), dk.as<rdkv_dual_bound_result>(), nullptr),
                  "dual_bound");
            sync();
            const auto av = to_host<rdkv_bisect_result>(rv.get(), U), ak = to_host<rdkv_bisect_result>(rk.get(), U);
            const auto bv = to_host<rdkv_dual_bound_result>(dv.get(), U),
                       bk = to_host<rdkv_dual_bound_result>(dk.get(), U);
            double primal = 0.0, dual = 0.0;
            bool feasible = true;
            for (int u = 0; u < U; ++u) {  // head order (sweep.cpp:94-106)
                check(av[u].status, "mckp_bisect");
                check(ak[u].status, "mckp_bisect");
                check(bv[u].status, "dual_bound");
                check(bk[u].status, "dual_bound");
                primal += av[u].objective + ak[u].objective;
                dual += bv[u].g_lambda + bk[u].g_lambda;
                feasible = feasible && bv[u].feasible && bk[u].feasible;
            }
            result.rows.push_back({seq, target, primal, dual, feasible});
        }
    }
    std::stable_sort(result.rows.begin(), result.rows.end(), [](const SweepPoint& a, const SweepPoint& b) {
        if (a.avg_bits != b.avg_bits) return a.avg_bits < b.avg_bits;
        return a.seq_id < b.seq_id;
    });
    return result;
}

DistortionTable calibrate_epsilon(std::span<const KVCache> caches, Granularity granularity, const BitSet& bits) {
    require(!caches.empty(), "calibrate_epsilon: empty sample");
    validate_bits_relaxed(bits);
    require(bits.widths.size() <= 8, "BitSet: too many widths");
    const std::vector<int32_t> w(bits.widths.begin(), bits.widths.end());
    int nq = 0;
    for (int b : w) nq += is_quant_width(b);
    nq = std::max(nq, 1);
    const int gran = granularity == Granularity::token ? 0 : 1;
    std::vector<double> err;
    std::vector<int64_t> cnt;
    for (const auto& cache : caches) {
        const auto& s = cache.shape;
        const int U = s.layers * s.kv_heads, T = s.seq_len, d = s.head_dim;
        const std::size_t per_layer = static_cast<std::size_t>(s.kv_heads) * T * d;
        DevBuf x(std::max<std::size_t>(U * static_cast<std::size_t>(T) * d, 1) * sizeof(float));
        const auto& src = gran == 0 ? cache.v : cache.k;  // token units: V rows; channel units: K columns
        for (int l = 0; l < s.layers; ++l)
            cuda_check(cudaMemcpy(x.as<float>() + l * per_layer, src[l].data().data(), per_layer * sizeof(float),
                                  cudaMemcpyHostToDevice), "H2D");
        const std::size_t ws_bytes = rdkv_cuda_calibrate_workspace(U, T, d, gran, nq);
        DevBuf ws(ws_bytes), e(std::max(U * nq, 1) * sizeof(double)), c(std::max(U, 1) * sizeof(int64_t));
        check(rdkv_cuda_calibrate_partials(x.get(), RDKV_F32, U, T, d, gran, w.data(), static_cast<int32_t>(w.size()),
                                           e.as<double>(), c.as<int64_t>(), ws.get(), ws_bytes, nullptr),
              "quantize_unit");
        const auto eh = to_host<double>(e.get(), static_cast<std::size_t>(U) * nq);
        const auto ch = to_host<int64_t>(c.get(), U);
        err.insert(err.end(), eh.begin(), eh.end());
        cnt.insert(cnt.end(), ch.begin(), ch.end());
    }
    std::vector<double> eps(w.size());
    int64_t units = 0;
    const int st = rdkv_calibrate_finalize(err.data(), cnt.data(), static_cast<int32_t>(cnt.size()), w.data(),
                                           static_cast<int32_t>(w.size()), eps.data(), &units);
    if (st == RDKV_ENUMERIC) throw NumericError("calibrate_epsilon: all units have zero norm");
    if (st == RDKV_EINVAL) throw std::invalid_argument("DistortionTable: eps must be strictly decreasing");
    check(st, "calibrate_epsilon");
    DistortionTable table;
    table.granularity = granularity;
    table.provenance = "calibrated on " + std::to_string(caches.size()) + " cache(s), " + std::to_string(units) + " " +
                       (gran == 0 ? "token" : "channel") + " units";
    for (std::size_t i = 0; i < w.size(); ++i) table.eps.emplace_back(w[i], eps[i]);
    return table;
}

}  // namespace rdkv::cuda
