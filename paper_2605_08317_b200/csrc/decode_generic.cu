// decode_generic.cu — K4 (generic path): packed mixed-bit decode attention on
// CUDA cores for any head_dim <= 256 and any bit mix, plus the split-K merge
// and the Zone C append (K5).
//
// Replaces packed_decode_step / fused_k_logits (trizone.cpp:210-305) and
// append_new_token (trizone.cpp:307-314), batched over every
// (batch, layer, KV head) tile and all GQA query heads of the tile at once.
// Math per tile (fp32, the reference is fp64; tolerance 1e-3 relative,
// observed ~1e-6):
//   q~[h][s]  = scale_s * q[h][perm_s]          (fused K dequant, PAPER Eq. 9)
//   bias[h]   = sum_s q[h][perm_s] * offset_s   (offset_s = -scale_s * z_s)
//   logit     = (sum_s q~[h][s] code[i][s] + bias[h]) / sqrt(d)
//   softmax over kept slots + Zone C, online (running max / sum)
//   out[h][c] = sum_i p[h][i] (vscale_i code[i][c] + voffset_i) + Zone B/C rows
// The tensor-core path (decode_mma.cu) handles the common d = 128 layouts;
// this kernel is the reference-shaped fallback and the parity baseline.
#include <type_traits>

#include "common.cuh"

namespace rdkv_b200 {

constexpr int kGenThreads = 128;
constexpr int kGenChunk = 128;
constexpr int kMaxG = 16;

template <typename IO>
__device__ __forceinline__ float io_load(const IO* p, size_t i) {
    return load_as_float(p, i);
}
__device__ __forceinline__ void io_store(float* p, size_t i, float v) { p[i] = v; }
__device__ __forceinline__ void io_store(__half* p, size_t i, float v) { p[i] = __float2half_rn(v); }

__device__ __forceinline__ int slot_class(const TileHeader& h, const int* base, int sl, int& li) {
    int cls = 0;
    while (cls < 3 && sl >= base[cls + 1]) ++cls;
    li = sl - base[cls];
    return cls;
}

// One CTA per (tile, split part). Dynamic smem: q [g][d], q~ [g][kslots],
// logits [g][chunk].
template <typename IO>
__global__ void __launch_bounds__(kGenThreads) decode_generic_kernel(
    const uint8_t* __restrict__ arena, const int64_t* __restrict__ offsets, int g, int d,
    const IO* __restrict__ q_all, IO* __restrict__ out_all, const __half* __restrict__ zc_k,
    const __half* __restrict__ zc_v, const int32_t* __restrict__ zc_len, int zc_cap, int split,
    float* __restrict__ part_ml, float* __restrict__ part_o) {
    extern __shared__ float smem[];
    __shared__ TileHeader h;
    __shared__ int sbase[5];
    __shared__ float bias[kMaxG];
    __shared__ float red[kMaxG][kGenThreads / 32];
    const int unit = blockIdx.x, part = blockIdx.y;
    const int tid = threadIdx.x;
    const uint8_t* tile = arena + offsets[unit];
    if (tid == 0) {
        h = *reinterpret_cast<const TileHeader*>(tile);
        int acc = 0;
        for (int i = 0; i < 4; ++i) {
            sbase[i] = acc;
            acc += pad4(h.r[i]);
        }
        sbase[4] = acc;
    }
    __syncthreads();
    const int kslots = h.kslots;
    float* qs = smem;                       // [g][d]
    const int gp = (g + 3) & ~3;            // heads padded to a float4
    float* qt = qs + ((g * d + 3) & ~3);    // [kslots][gp], 16-B aligned: one float4 load feeds 4 heads
    float* lg = qt + gp * kslots;           // [g][chunk]
    const size_t qrow = (size_t)unit * g * d;
    for (int i = tid; i < g * d; i += blockDim.x) qs[i] = io_load(q_all, qrow + i);
    __syncthreads();
    const float2* chan = reinterpret_cast<const float2*>(tile + chan_table_off());
    const uint16_t* perm = reinterpret_cast<const uint16_t*>(tile + perm_off(h));
    for (int i = tid; i < gp * kslots; i += blockDim.x) {
        const int sl = i / gp, hh = i % gp;
        qt[i] = hh < g ? chan[sl].x * qs[hh * d + perm[sl]] : 0.0f;
    }
    if (tid < g) {
        float b = 0.0f;
        for (int sl = 0; sl < kslots; ++sl) b = fmaf(qs[tid * d + perm[sl]], chan[sl].y, b);
        bias[tid] = b;
    }
    __syncthreads();

    const float inv_sqrt_d = rsqrtf((float)d);
    const int nzc = zc_len ? zc_len[unit] : 0;
    const int total = h.nslot + nzc;
    const int per = (total + split - 1) / split;
    const int i_begin = part * per, i_end = min(total, i_begin + per);

    float m_run[kMaxG], l_run[kMaxG], o_acc[kMaxG][2];
#pragma unroll
    for (int hh = 0; hh < kMaxG; ++hh) {
        m_run[hh] = -INFINITY;
        l_run[hh] = 0.0f;
        o_acc[hh][0] = o_acc[hh][1] = 0.0f;
    }
    const float2* vparam = reinterpret_cast<const float2*>(tile + h.off_vp);
    const uint8_t* krows = tile + h.off_k;

    for (int c0 = i_begin; c0 < i_end; c0 += kGenChunk) {
        const int cn = min(kGenChunk, i_end - c0);
        // ---- logits, one token per thread
        if (tid < cn) {
            const int i = c0 + tid;
            float acc[kMaxG];
#pragma unroll
            for (int hh = 0; hh < kMaxG; ++hh) acc[hh] = 0.0f;
            bool pad = false;
            if (i < h.nslot) {
                int li;
                const int cls = slot_class(h, sbase, i, li);
                pad = li >= h.r[cls];
                const uint8_t* row = krows + (size_t)krow_pos(h, i) * h.krow_bytes;
                if (!pad) {
                    // one K byte holds per_b codes of a class: compile-time unpacking per class
                    auto kclass = [&](auto bits_c, int kc) {
                        constexpr int bits = decltype(bits_c)::value;
                        constexpr int per_b = 8 / bits;
                        const int b0 = h.kbyte_base[kc];
                        const int nb = (h.c[kc] + per_b - 1) / per_b;
                        const float* qk = qt + (size_t)h.kslot_base[kc] * gp;
                        for (int b = 0; b < nb; ++b) {
                            const uint32_t byte = row[b0 + b];
#pragma unroll
                            for (int j = 0; j < per_b; ++j) {
                                const float code = (float)((byte >> (j * bits)) & ((1u << bits) - 1u));
                                const float4* q4 = reinterpret_cast<const float4*>(qk + (b * per_b + j) * gp);
#pragma unroll
                                for (int h4 = 0; h4 < kMaxG / 4; ++h4) {
                                    if (4 * h4 < g) {
                                        const float4 w = q4[h4];
                                        acc[4 * h4 + 0] = fmaf(w.x, code, acc[4 * h4 + 0]);
                                        acc[4 * h4 + 1] = fmaf(w.y, code, acc[4 * h4 + 1]);
                                        acc[4 * h4 + 2] = fmaf(w.z, code, acc[4 * h4 + 2]);
                                        acc[4 * h4 + 3] = fmaf(w.w, code, acc[4 * h4 + 3]);
                                    }
                                }
                            }
                        }
                    };
                    kclass(std::integral_constant<int, 2>{}, 0);
                    kclass(std::integral_constant<int, 4>{}, 1);
                    kclass(std::integral_constant<int, 8>{}, 2);
                    const __half* k16 = reinterpret_cast<const __half*>(row + h.kbyte_base[3]);
                    for (int j = 0; j < h.c[3]; ++j) {
                        const float x = __half2float(k16[j]);
                        const int ks = h.kslot_base[3] + j;
#pragma unroll
                        for (int hh = 0; hh < kMaxG; ++hh)
                            if (hh < g) acc[hh] = fmaf(qt[(size_t)ks * gp + hh], x, acc[hh]);
                    }
#pragma unroll
                    for (int hh = 0; hh < kMaxG; ++hh) acc[hh] += bias[hh < g ? hh : 0];
                }
            } else {
                const __half* kr = zc_k + ((size_t)unit * zc_cap + (i - h.nslot)) * d;
                for (int c = 0; c < d; ++c) {
                    const float x = __half2float(kr[c]);
#pragma unroll
                    for (int hh = 0; hh < kMaxG; ++hh)
                        if (hh < g) acc[hh] = fmaf(qs[hh * d + c], x, acc[hh]);
                }
            }
#pragma unroll
            for (int hh = 0; hh < kMaxG; ++hh)
                if (hh < g) lg[hh * kGenChunk + tid] = pad ? -INFINITY : acc[hh] * inv_sqrt_d;
        }
        __syncthreads();
        // ---- chunk max per head, online rescale
        float cmax[kMaxG];
#pragma unroll
        for (int hh = 0; hh < kMaxG; ++hh) {
            float v = (hh < g && tid < cn) ? lg[hh * kGenChunk + tid] : -INFINITY;
            v = warp_max(v);
            if ((tid & 31) == 0 && hh < g) red[hh][tid >> 5] = v;
        }
        __syncthreads();
#pragma unroll
        for (int hh = 0; hh < kMaxG; ++hh) {
            float v = -INFINITY;
            if (hh < g)
                for (int w = 0; w < kGenThreads / 32; ++w) v = fmaxf(v, red[hh][w]);
            cmax[hh] = v;
        }
        __syncthreads();
        float alpha[kMaxG];
#pragma unroll
        for (int hh = 0; hh < kMaxG; ++hh) {
            const float mn = fmaxf(m_run[hh], cmax[hh]);
            alpha[hh] = (m_run[hh] == -INFINITY) ? 0.0f : __expf(m_run[hh] - mn);
            if (mn == -INFINITY) alpha[hh] = 1.0f;
            m_run[hh] = mn;
        }
        // p = exp(l - m) in place; partial sums
#pragma unroll
        for (int hh = 0; hh < kMaxG; ++hh) {
            float p = 0.0f;
            if (hh < g && tid < cn) {
                const float l = lg[hh * kGenChunk + tid];
                p = (l == -INFINITY) ? 0.0f : __expf(l - m_run[hh]);
                lg[hh * kGenChunk + tid] = p;
            }
            p = warp_sum(p);
            if ((tid & 31) == 0 && hh < g) red[hh][tid >> 5] = p;
        }
        __syncthreads();
#pragma unroll
        for (int hh = 0; hh < kMaxG; ++hh) {
            float sum = 0.0f;
            if (hh < g)
                for (int w = 0; w < kGenThreads / 32; ++w) sum += red[hh][w];
            l_run[hh] = l_run[hh] * alpha[hh] + sum;
            o_acc[hh][0] *= alpha[hh];
            o_acc[hh][1] *= alpha[hh];
        }
        // ---- PV: thread owns channels tid and tid + 128
        for (int j = 0; j < cn; ++j) {
            const int i = c0 + j;
            float v0 = 0.0f, v1 = 0.0f;
            if (i < h.nslot) {
                int li;
                const int cls = slot_class(h, sbase, i, li);
                if (li >= h.r[cls]) continue;
                if (cls == 3) {
                    const __half* vr = reinterpret_cast<const __half*>(tile + h.off_vseg[3]) + (size_t)li * d;
                    if (tid < d) v0 = __half2float(vr[tid]);
                    if (tid + kGenThreads < d) v1 = __half2float(vr[tid + kGenThreads]);
                } else {
                    const float2 vp = vparam[i];
                    auto vrow = [&](auto bits_c) {  // the class is block-uniform: compile-time unpacking
                        constexpr int bits = decltype(bits_c)::value;
                        constexpr int per_b = 8 / bits;
                        if (tid < d) {
                            const int c = tid;
                            const uint32_t byte = tile[vbyte_offset(h, cls, li, c / per_b, d)];
                            v0 = fmaf(vp.x, (float)((byte >> ((c % per_b) * bits)) & ((1u << bits) - 1u)), vp.y);
                        }
                        if (tid + kGenThreads < d) {
                            const int c = tid + kGenThreads;
                            const uint32_t byte = tile[vbyte_offset(h, cls, li, c / per_b, d)];
                            v1 = fmaf(vp.x, (float)((byte >> ((c % per_b) * bits)) & ((1u << bits) - 1u)), vp.y);
                        }
                    };
                    if (cls == 0) vrow(std::integral_constant<int, 2>{});
                    else if (cls == 1) vrow(std::integral_constant<int, 4>{});
                    else vrow(std::integral_constant<int, 8>{});
                }
            } else {
                const __half* vr = zc_v + ((size_t)unit * zc_cap + (i - h.nslot)) * d;
                if (tid < d) v0 = __half2float(vr[tid]);
                if (tid + kGenThreads < d) v1 = __half2float(vr[tid + kGenThreads]);
            }
#pragma unroll
            for (int hh = 0; hh < kMaxG; ++hh) {
                if (hh < g) {
                    const float p = lg[hh * kGenChunk + j];
                    o_acc[hh][0] = fmaf(p, v0, o_acc[hh][0]);
                    o_acc[hh][1] = fmaf(p, v1, o_acc[hh][1]);
                }
            }
        }
        __syncthreads();
    }

    if (split == 1) {
#pragma unroll
        for (int hh = 0; hh < kMaxG; ++hh) {
            if (hh < g) {
                const float inv = 1.0f / l_run[hh];
                if (tid < d) io_store(out_all, qrow + hh * d + tid, o_acc[hh][0] * inv);
                if (tid + kGenThreads < d) io_store(out_all, qrow + hh * d + tid + kGenThreads, o_acc[hh][1] * inv);
            }
        }
    } else {
        const size_t pbase = ((size_t)unit * split + part) * g;
#pragma unroll
        for (int hh = 0; hh < kMaxG; ++hh) {
            if (hh < g) {
                if (tid == 0) {
                    part_ml[(pbase + hh) * 2] = m_run[hh];
                    part_ml[(pbase + hh) * 2 + 1] = l_run[hh];
                }
                if (tid < d) part_o[(pbase + hh) * d + tid] = o_acc[hh][0];
                if (tid + kGenThreads < d) part_o[(pbase + hh) * d + tid + kGenThreads] = o_acc[hh][1];
            }
        }
    }
}

// Deterministic log-sum-exp merge of split-K partials (fixed part order).
template <typename IO>
__global__ void split_merge_kernel(const float* __restrict__ part_ml, const float* __restrict__ part_o,
                                   int units, int g, int d, int split, IO* __restrict__ out_all) {
    const size_t idx = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
    if (idx >= (size_t)units * g * d) return;
    const int c = (int)(idx % d);
    const size_t uh = idx / d;  // unit * g + head
    const size_t unit = uh / g, hh = uh % g;
    float m = -INFINITY;
    for (int p = 0; p < split; ++p) m = fmaxf(m, part_ml[((unit * split + p) * g + hh) * 2]);
    float l = 0.0f, o = 0.0f;
    for (int p = 0; p < split; ++p) {
        const size_t b = (unit * split + p) * g + hh;
        const float mp = part_ml[b * 2];
        if (mp == -INFINITY) continue;
        const float w = __expf(mp - m);
        l = fmaf(part_ml[b * 2 + 1], w, l);
        o = fmaf(part_o[b * d + c], w, o);
    }
    io_store(out_all, idx, o / l);
}

template <typename T>
__global__ void append_kernel(__half* __restrict__ zc_k, __half* __restrict__ zc_v,
                              int32_t* __restrict__ zc_len, int zc_cap, const T* __restrict__ k_new,
                              const T* __restrict__ v_new, int d) {
    const int unit = blockIdx.x;
    const int pos = zc_len[unit];
    if (pos >= zc_cap) return;  // caller checks capacity
    for (int c = threadIdx.x; c < d; c += blockDim.x) {
        zc_k[((size_t)unit * zc_cap + pos) * d + c] = __float2half_rn(load_as_float(k_new, (size_t)unit * d + c));
        zc_v[((size_t)unit * zc_cap + pos) * d + c] = __float2half_rn(load_as_float(v_new, (size_t)unit * d + c));
    }
    __syncthreads();
    if (threadIdx.x == 0) zc_len[unit] = pos + 1;
}

// d % 8 == 0: one warp per unit, 8 channels (16 B of fp16) per lane and row —
// a 4096-unit step's append is one short launch instead of 4096 CTAs.
template <typename T>
__global__ void __launch_bounds__(256) append_vec_kernel(__half* __restrict__ zc_k, __half* __restrict__ zc_v,
                                                         int32_t* __restrict__ zc_len, int zc_cap, int units,
                                                         const T* __restrict__ k_new, const T* __restrict__ v_new,
                                                         int d) {
    const int unit = (int)((blockIdx.x * (size_t)blockDim.x + threadIdx.x) >> 5), lane = threadIdx.x & 31;
    if (unit >= units) return;
    const int pos = zc_len[unit];
    if (pos >= zc_cap) return;  // caller checks capacity
    const size_t src = (size_t)unit * d, dst = ((size_t)unit * zc_cap + pos) * d;
    for (int c = 8 * lane; c < d; c += 256) {
        uint4 kk, vv;
        if constexpr (sizeof(T) == 2) {
            kk = *reinterpret_cast<const uint4*>(k_new + src + c);
            vv = *reinterpret_cast<const uint4*>(v_new + src + c);
        } else {
            __half2 kh[4], vh[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                kh[j] = __floats2half2_rn(load_as_float(k_new, src + c + 2 * j), load_as_float(k_new, src + c + 2 * j + 1));
                vh[j] = __floats2half2_rn(load_as_float(v_new, src + c + 2 * j), load_as_float(v_new, src + c + 2 * j + 1));
            }
            kk = *reinterpret_cast<const uint4*>(kh);
            vv = *reinterpret_cast<const uint4*>(vh);
        }
        *reinterpret_cast<uint4*>(zc_k + dst + c) = kk;
        *reinterpret_cast<uint4*>(zc_v + dst + c) = vv;
    }
    __syncwarp();
    if (lane == 0) zc_len[unit] = pos + 1;
}

size_t generic_smem_bytes(int g, int d, int kslots) {
    return sizeof(float) * ((size_t)((g * d + 3) & ~3) + (size_t)((g + 3) & ~3) * kslots + (size_t)g * kGenChunk);
}

template <typename IO>
int launch_generic(const rdkv_decode_args* a, int split, int max_kslots, cudaStream_t st) {
    const size_t smem = generic_smem_bytes(a->group, a->head_dim, max_kslots);
    auto kern = decode_generic_kernel<IO>;
    if (smem > 48 * 1024) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    float* part_ml = nullptr;
    float* part_o = nullptr;
    if (split > 1) {
        part_ml = static_cast<float*>(a->workspace);
        part_o = part_ml + (size_t)a->units * split * a->group * 2;
    }
    dim3 grid(a->units, split);
    kern<<<grid, kGenThreads, smem, st>>>(a->arena, a->tile_offsets, a->group, a->head_dim,
                                          static_cast<const IO*>(a->q), static_cast<IO*>(a->out),
                                          static_cast<const __half*>(a->zc_k),
                                          static_cast<const __half*>(a->zc_v), a->zc_len, a->zc_cap,
                                          split, part_ml, part_o);
    if (split > 1) {
        const size_t n = (size_t)a->units * a->group * a->head_dim;
        split_merge_kernel<IO><<<(unsigned)((n + 255) / 256), 256, 0, st>>>(
            part_ml, part_o, a->units, a->group, a->head_dim, split, static_cast<IO*>(a->out));
    }
    return launch_status();
}

template int launch_generic<float>(const rdkv_decode_args*, int, int, cudaStream_t);
template int launch_generic<__half>(const rdkv_decode_args*, int, int, cudaStream_t);

}  // namespace rdkv_b200

using namespace rdkv_b200;

extern "C" RDKV_API int rdkv_cuda_append(void* zc_k, void* zc_v, int32_t* zc_len, int32_t zc_cap,
                                         const void* k_new, const void* v_new, int32_t dtype,
                                         int32_t units, int32_t head_dim, void* stream) {
    if (!zc_k || !zc_v || !zc_len || !k_new || !v_new || units < 1 || head_dim < 1 || zc_cap < 1)
        return RDKV_EINVAL;
    auto st = static_cast<cudaStream_t>(stream);
    const bool vec = head_dim % 8 == 0 && (reinterpret_cast<uintptr_t>(k_new) & 15) == 0 &&
                     (reinterpret_cast<uintptr_t>(v_new) & 15) == 0 && (reinterpret_cast<uintptr_t>(zc_k) & 15) == 0 &&
                     (reinterpret_cast<uintptr_t>(zc_v) & 15) == 0;
    if (vec) {
        const unsigned blocks = (unsigned)(((size_t)units * 32 + 255) / 256);
        if (dtype == RDKV_F32)
            append_vec_kernel<float><<<blocks, 256, 0, st>>>(static_cast<__half*>(zc_k), static_cast<__half*>(zc_v), zc_len,
                                                             zc_cap, units, static_cast<const float*>(k_new),
                                                             static_cast<const float*>(v_new), head_dim);
        else if (dtype == RDKV_F16)
            append_vec_kernel<__half><<<blocks, 256, 0, st>>>(static_cast<__half*>(zc_k), static_cast<__half*>(zc_v),
                                                              zc_len, zc_cap, units, static_cast<const __half*>(k_new),
                                                              static_cast<const __half*>(v_new), head_dim);
        else
            return RDKV_EINVAL;
        return launch_status();
    }
    if (dtype == RDKV_F32)
        append_kernel<float><<<units, 128, 0, st>>>(static_cast<__half*>(zc_k), static_cast<__half*>(zc_v),
                                                    zc_len, zc_cap, static_cast<const float*>(k_new),
                                                    static_cast<const float*>(v_new), head_dim);
    else if (dtype == RDKV_F16)
        append_kernel<__half><<<units, 128, 0, st>>>(static_cast<__half*>(zc_k), static_cast<__half*>(zc_v),
                                                     zc_len, zc_cap, static_cast<const __half*>(k_new),
                                                     static_cast<const __half*>(v_new), head_dim);
    else
        return RDKV_EINVAL;
    return launch_status();
}

// ---------------------------------------------------------------------------
// fused_k_logits (trizone.cpp:210-249) per token slot: the decode kernel's
// QK product without the 1/sqrt(d) scale, for every (tile, query head).
// logits [units][group][max_slots] f32, NaN in pad slots and past nslot.
namespace rdkv_b200 {

__global__ void tile_logits_kernel(const uint8_t* __restrict__ arena, const int64_t* __restrict__ offsets,
                                   int g, int d, const float* __restrict__ q_all, int max_slots,
                                   float* __restrict__ logits) {
    extern __shared__ float smem[];
    __shared__ TileHeader h;
    __shared__ int sbase[5];
    const int unit = blockIdx.x, hh = blockIdx.y;
    const uint8_t* tile = arena + offsets[unit];
    if (threadIdx.x == 0) {
        h = *reinterpret_cast<const TileHeader*>(tile);
        int acc = 0;
        for (int i = 0; i < 4; ++i) {
            sbase[i] = acc;
            acc += pad4(h.r[i]);
        }
        sbase[4] = acc;
    }
    __syncthreads();
    float* qs = smem;          // [d]
    float* qt = smem + d;      // [kslots]
    const float* q = q_all + ((size_t)unit * g + hh) * d;
    for (int i = threadIdx.x; i < d; i += blockDim.x) qs[i] = q[i];
    __syncthreads();
    const float2* chan = reinterpret_cast<const float2*>(tile + chan_table_off());
    const uint16_t* perm = reinterpret_cast<const uint16_t*>(tile + perm_off(h));
    for (int sl = threadIdx.x; sl < h.kslots; sl += blockDim.x) qt[sl] = chan[sl].x * qs[perm[sl]];
    __shared__ float bias;
    if (threadIdx.x == 0) {
        float b = 0.0f;
        for (int sl = 0; sl < h.kslots; ++sl) b = fmaf(qs[perm[sl]], chan[sl].y, b);
        bias = b;
    }
    __syncthreads();
    float* outp = logits + ((size_t)unit * g + hh) * max_slots;
    for (int i = threadIdx.x; i < max_slots; i += blockDim.x) {
        float acc = __int_as_float(0x7fc00000);
        if (i < h.nslot) {
            int li;
            const int cls = slot_class(h, sbase, i, li);
            if (li < h.r[cls]) {
                acc = 0.0f;
                const uint8_t* row = tile + krow_offset(h, i);
                for (int kc = 0; kc < 3; ++kc) {
                    const int bits = kBits(kc);
                    for (int j = 0; j < h.c[kc]; ++j) {
                        const int bit = j * bits;
                        const uint32_t code = (row[h.kbyte_base[kc] + (bit >> 3)] >> (bit & 7)) & ((1u << bits) - 1u);
                        acc = fmaf(qt[h.kslot_base[kc] + j], (float)code, acc);
                    }
                }
                const __half* k16 = reinterpret_cast<const __half*>(row + h.kbyte_base[3]);
                for (int j = 0; j < h.c[3]; ++j) acc = fmaf(qt[h.kslot_base[3] + j], __half2float(k16[j]), acc);
                acc += bias;
            }
        }
        outp[i] = acc;
    }
}

}  // namespace rdkv_b200

extern "C" RDKV_API int rdkv_cuda_tile_logits(const uint8_t* arena, const int64_t* tile_offsets, int32_t units,
                                              int32_t group, int32_t head_dim, const float* q, int32_t max_slots,
                                              int32_t max_kslots, float* logits, void* stream) {
    if (!arena || !tile_offsets || !q || !logits || units < 0 || group < 1 || head_dim < 1 || max_slots < 0 ||
        max_kslots < 0)
        return RDKV_EINVAL;
    if (units == 0 || max_slots == 0) return RDKV_OK;
    const size_t smem = sizeof(float) * ((size_t)head_dim + max_kslots);
    if (smem > 48 * 1024) return RDKV_EINVAL;
    tile_logits_kernel<<<dim3(units, group), 128, smem, static_cast<cudaStream_t>(stream)>>>(
        arena, tile_offsets, group, head_dim, q, max_slots, logits);
    return launch_status();
}
