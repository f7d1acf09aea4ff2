// pack.cu — K3: TriZone packing into the device tile layout (tile_layout.h).
//
// Replaces build_trizone / build_packed_model (trizone.cpp:91-208, 478-490)
// and quantize_unit (quantizer.cpp:104-131). One CTA per unit:
//   1. slot assignment: block-wide scan over v_bits gives every kept token its
//      slot (class 2,4,8,16 then ascending token id — the reference segment
//      order, trizone.cpp:126-157); K channels get K slots (channel_perm order,
//      trizone.cpp:201-206);
//   2. K channel quantisation over the kept rows (one thread per channel
//      computes min/max; then one thread per (slot, K-row byte) packs codes);
//   3. V row quantisation, one warp per kept row, written 4-token interleaved;
//      16-bit V rows (Zone B) and 16-bit K channels (k16) stored as fp16.
// Quantisation is bit-exact with quantize_unit: f32 min/max, fp64 scale and
// zero point, round-half-away-from-zero, clamp (file built with -fmad=false).
#include "common.cuh"

namespace rdkv_b200 {

constexpr int kPackThreads = 256;

// per-class counts of the bit-widths 2/4/8/16 in four bytes (SIMD byte compares)
__device__ __forceinline__ void class_counts4(uint32_t w, int (&r)[4]) {
    r[0] += __popc(__vcmpeq4(w, 0x02020202u)) >> 3;
    r[1] += __popc(__vcmpeq4(w, 0x04040404u)) >> 3;
    r[2] += __popc(__vcmpeq4(w, 0x08080808u)) >> 3;
    r[3] += __popc(__vcmpeq4(w, 0x10101010u)) >> 3;
}

__device__ __forceinline__ void header_counts(const uint8_t* vb, const uint8_t* kb, int t_len,
                                              int d, int* counts /*8 ints in smem*/) {
    int r[4] = {0, 0, 0, 0}, c[4] = {0, 0, 0, 0};
    // v_bits rows are 16-B aligned when t_len % 16 == 0 (the allocation buffers
    // are [units][T] u8): 16 widths per load
    if ((t_len & 15) == 0 && (reinterpret_cast<uintptr_t>(vb) & 15) == 0) {
        const uint4* v4 = reinterpret_cast<const uint4*>(vb);
        for (int i = threadIdx.x; i < (t_len >> 4); i += blockDim.x) {
            const uint4 w = v4[i];
            if ((w.x | w.y | w.z | w.w) == 0u) continue;  // evicted tokens (the common case)
            class_counts4(w.x, r);
            class_counts4(w.y, r);
            class_counts4(w.z, r);
            class_counts4(w.w, r);
        }
    } else {
        for (int t = threadIdx.x; t < t_len; t += blockDim.x) {
            const int cls = class_of_bits(vb[t]);
            if (cls >= 0) r[cls]++;
        }
    }
    for (int ch = threadIdx.x; ch < d; ch += blockDim.x) {
        const int cls = class_of_bits(kb[ch]);
        if (cls >= 0) c[cls]++;
    }
    for (int i = 0; i < 4; ++i) {
        int a = r[i], b = c[i];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            a += __shfl_xor_sync(0xffffffffu, a, o);
            b += __shfl_xor_sync(0xffffffffu, b, o);
        }
        if ((threadIdx.x & 31) == 0) {
            atomicAdd(&counts[i], a);
            atomicAdd(&counts[4 + i], b);
        }
    }
}

__global__ void pack_plan_kernel(const uint8_t* __restrict__ v_bits, const uint8_t* __restrict__ k_bits,
                                 int t_len, int d, int64_t* __restrict__ sizes) {
    __shared__ int counts[8];
    if (threadIdx.x < 8) counts[threadIdx.x] = 0;
    __syncthreads();
    const int unit = blockIdx.x;
    header_counts(v_bits + (size_t)unit * t_len, k_bits + (size_t)unit * d, t_len, d, counts);
    __syncthreads();
    if (threadIdx.x == 0) {
        TileHeader h{};
        for (int i = 0; i < 4; ++i) {
            h.r[i] = counts[i];
            h.c[i] = counts[4 + i];
        }
        tile_layout(h, d);
        sizes[unit] = h.total_bytes;
    }
}

// exclusive scan of sizes[0..n) into offsets[0..n], single CTA
__global__ void scan_kernel(const int64_t* __restrict__ sizes, int n, int64_t* __restrict__ offsets) {
    __shared__ int64_t part[1024];
    const int per = (n + blockDim.x - 1) / blockDim.x;
    const int b = threadIdx.x * per, e = min(n, b + per);
    int64_t s = 0;
    for (int i = b; i < e; ++i) s += sizes[i];
    part[threadIdx.x] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        int64_t run = 0;
        for (int i = 0; i < (int)blockDim.x; ++i) {
            const int64_t v = part[i];
            part[i] = run;
            run += v;
        }
        offsets[n] = run;
    }
    __syncthreads();
    int64_t run = part[threadIdx.x];
    for (int i = b; i < e; ++i) {
        offsets[i] = run;
        run += sizes[i];
    }
}

struct PackSmem {
    TileHeader h;
    int counts[8];
    int cls_base[4];      // running slot counters per V class (block scan)
    int warp_tot[32][4];
    double kscale[384];   // fp64 scale per K slot of classes 0-2 (d <= 256 + pads)
    double kzd[384];      // fp64 zero point
    int bad;
    unsigned int kmax, vmax;
};

// quantize_unit parameters from f32 lo/hi (quantizer.cpp:110-123)
__device__ __forceinline__ void quant_params(float lo, float hi, int bits, double& scale, double& zd) {
    const double max_code = (double)((1 << bits) - 1);
    double range = (double)hi - (double)lo;
    if (range < 1e-12) range = 1e-12;
    scale = range / max_code;
    zd = round(-(double)lo / scale);
    zd = fmin(fmax(zd, -9.0e18), 9.0e18);
}

__device__ __forceinline__ uint32_t quant_code(float v, double scale, double zd, int bits) {
    const double max_code = (double)((1 << bits) - 1);
    double c = __dadd_rn(round((double)v / scale), zd);
    c = fmin(fmax(c, 0.0), max_code);
    return (uint32_t)c;
}

template <typename T>
__global__ void __launch_bounds__(kPackThreads) pack_kernel(
    const T* __restrict__ k_all, const T* __restrict__ v_all, const uint8_t* __restrict__ v_bits,
    const uint8_t* __restrict__ k_bits, int t_len, int d, const int64_t* __restrict__ offsets,
    uint8_t* __restrict__ arena, int32_t* __restrict__ head_status) {
    __shared__ PackSmem s;
    const int unit = blockIdx.x;
    const uint8_t* vb = v_bits + (size_t)unit * t_len;
    const uint8_t* kb = k_bits + (size_t)unit * d;
    const T* K = k_all + (size_t)unit * t_len * d;
    const T* V = v_all + (size_t)unit * t_len * d;
    uint8_t* tile = arena + offsets[unit];
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, nwarp = blockDim.x >> 5;

    if (tid < 8) s.counts[tid] = 0;
    if (tid == 0) s.bad = 0;
    __syncthreads();
    header_counts(vb, kb, t_len, d, s.counts);
    __syncthreads();
    if (tid == 0) {
        TileHeader h{};
        for (int i = 0; i < 4; ++i) {
            h.r[i] = s.counts[i];
            h.c[i] = s.counts[4 + i];
        }
        tile_layout(h, d);
        s.h = h;
        for (int i = 0; i < 4; ++i) s.cls_base[i] = slot_base(h, i);
    }
    __syncthreads();
    const TileHeader& h = s.h;
    {   // zero the tile (pad slots / pad channels / alignment bytes stay 0)
        uint4* t4 = reinterpret_cast<uint4*>(tile);
        for (int i = tid; i < h.total_bytes / 16; i += blockDim.x) t4[i] = make_uint4(0, 0, 0, 0);
    }
    __syncthreads();
    if (tid == 0) *reinterpret_cast<TileHeader*>(tile) = h;

    int32_t* ids = reinterpret_cast<int32_t*>(tile + h.off_ids);
    int64_t* vz = reinterpret_cast<int64_t*>(tile + h.off_vz);
    int64_t* kz = reinterpret_cast<int64_t*>(tile + h.off_kz);
    float2* chan = reinterpret_cast<float2*>(tile + chan_table_off());
    uint16_t* perm = reinterpret_cast<uint16_t*>(tile + perm_off(h));
    float2* vparam = reinterpret_cast<float2*>(tile + h.off_vp);

    // pad slots: token id -1 (every slot is overwritten below if real)
    for (int sl = tid; sl < h.nslot; sl += blockDim.x) ids[sl] = -1;
    __syncthreads();

    // ---- 1. token slots: contiguous chunk per thread, block scan per class
    {
        // (chunks of a multiple of 16 tokens: all-evicted 16-B groups are skipped)
        const int per = ((t_len + blockDim.x - 1) / blockDim.x + 15) & ~15;
        const int t0 = min(t_len, tid * per), t1 = min(t_len, t0 + per);
        const bool vec = (t_len & 15) == 0 && (reinterpret_cast<uintptr_t>(vb) & 15) == 0;
        auto group_empty = [&](int t) {  // tokens t .. t + 15 all evicted (t % 16 == 0)
            if (!vec || t + 16 > t1) return false;
            const uint4 w = *reinterpret_cast<const uint4*>(vb + t);
            return (w.x | w.y | w.z | w.w) == 0u;
        };
        int cnt[4] = {0, 0, 0, 0};
        for (int t = t0; t < t1; ++t) {
            if ((t & 15) == 0 && group_empty(t)) {
                t += 15;
                continue;
            }
            const int cls = class_of_bits(vb[t]);
            if (cls >= 0) cnt[cls]++;
        }
        // inclusive warp scan of the 4 counters
        int incl[4];
        for (int i = 0; i < 4; ++i) {
            int v = cnt[i];
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int n = __shfl_up_sync(0xffffffffu, v, o);
                if (lane >= o) v += n;
            }
            incl[i] = v;
            if (lane == 31) s.warp_tot[wid][i] = v;
        }
        __syncthreads();
        int run[4];
        for (int i = 0; i < 4; ++i) {
            int base = 0;
            for (int w = 0; w < wid; ++w) base += s.warp_tot[w][i];
            run[i] = s.cls_base[i] + base + incl[i] - cnt[i];
        }
        for (int t = t0; t < t1; ++t) {
            if ((t & 15) == 0 && group_empty(t)) {
                t += 15;
                continue;
            }
            const int cls = class_of_bits(vb[t]);
            if (cls >= 0) ids[run[cls]++] = t;
        }
    }
    // ---- K slots (channel_perm order): tiny, thread 0
    if (tid == 0) {
        int next[4];
        for (int i = 0; i < 4; ++i) next[i] = h.kslot_base[i];
        for (int sl = 0; sl < h.kslots; ++sl) {
            perm[sl] = 0;
            chan[sl] = make_float2(0.0f, 0.0f);
            kz[sl] = 0;
        }
        if (h.n > 0) {
            for (int ch = 0; ch < d; ++ch) {
                const int cls = class_of_bits(kb[ch]);
                if (cls < 0) continue;
                perm[next[cls]++] = (uint16_t)ch;
            }
        }
    }
    __syncthreads();

    // ---- 2. K channel parameters over the kept rows (trizone.cpp:159-173)
    const int kq_slots = h.kslot_base[3];  // slots of classes 0..2 (incl. pads)
    for (int sl = tid; sl < h.kslots; sl += blockDim.x) {
        int cls = 3;
        for (int i = 0; i < 3; ++i)
            if (sl >= h.kslot_base[i] && sl < h.kslot_base[i] + h.c[i]) cls = i;
        const bool real16 = sl >= h.kslot_base[3] && sl < h.kslot_base[3] + h.c[3];
        if (cls == 3) {
            if (real16) chan[sl] = make_float2(1.0f, 0.0f);
            continue;
        }
        const int ch = perm[sl];
        float lo = 0.0f, hi = 0.0f;
        bool first = true;
        for (int i = 0; i < 3; ++i) {  // kept rows in ascending token order = slot order per class
            for (int li = 0; li < h.r[i]; ++li) {
                const int t = ids[s.cls_base[i] + li];
                const float x = load_as_float(K, (size_t)t * d + ch);
                if (!isfinite(x)) s.bad = 1;
                if (first) { lo = hi = x; first = false; }
                lo = x < lo ? x : lo;
                hi = hi < x ? x : hi;
            }
        }
        for (int li = 0; li < h.r[3]; ++li) {
            const int t = ids[s.cls_base[3] + li];
            const float x = load_as_float(K, (size_t)t * d + ch);
            if (!isfinite(x)) s.bad = 1;
            if (first) { lo = hi = x; first = false; }
            lo = x < lo ? x : lo;
            hi = hi < x ? x : hi;
        }
        double scale, zd;
        quant_params(lo, hi, kBits(cls), scale, zd);
        s.kscale[sl] = scale;
        s.kzd[sl] = zd;
        const float sf = (float)scale;
        const int64_t z = (int64_t)zd;
        chan[sl] = make_float2(sf, (float)(-(double)sf * (double)z));
        kz[sl] = z;
    }
    __syncthreads();

    // ---- K rows: one item per (slot, byte) of the packed region, plus fp16 k16
    {
        const int qbytes = h.kbyte_base[3];  // packed region bytes (classes 0..2)
        const int items = h.nslot * qbytes;
        for (int it = tid; it < items; it += blockDim.x) {
            const int sl = it / qbytes, byte = it % qbytes;
            const int t = ids[sl];
            uint32_t val = 0;
            if (t >= 0) {
                int cls = 0;
                while (cls < 2 && byte >= h.kbyte_base[cls + 1]) ++cls;
                const int bits = kBits(cls);
                const int per = 8 / bits;
                const int k0 = h.kslot_base[cls] + (byte - h.kbyte_base[cls]) * per;
                for (int j = 0; j < per; ++j) {
                    const int ks = k0 + j;
                    if (ks - h.kslot_base[cls] >= h.c[cls]) break;  // pad slot: code 0
                    const float x = load_as_float(K, (size_t)t * d + perm[ks]);
                    val |= quant_code(x, s.kscale[ks], s.kzd[ks], bits) << (j * bits);
                }
            }
            tile[krow_offset(h, sl) + byte] = (uint8_t)val;
        }
        const int n16 = h.c[3];
        for (int it = tid; it < h.nslot * n16; it += blockDim.x) {
            const int sl = it / n16, j = it % n16;
            const int t = ids[sl];
            const float x = t >= 0 ? load_as_float(K, (size_t)t * d + perm[h.kslot_base[3] + j]) : 0.0f;
            reinterpret_cast<__half*>(tile + krow_offset(h, sl) + h.kbyte_base[3])[j] = __float2half_rn(x);
        }
        (void)kq_slots;
    }

    // ---- 3. V rows: one warp per slot (trizone.cpp:126-157)
    for (int sl = wid; sl < h.nslot; sl += nwarp) {
        const int t = ids[sl];
        int cls = 0;
        while (cls < 3 && sl >= s.cls_base[cls] + pad4(h.r[cls])) ++cls;
        const int li = sl - s.cls_base[cls];
        if (t < 0) {
            if (lane == 0) {
                vparam[sl] = make_float2(0.0f, 0.0f);
                vz[sl] = 0;
            }
            continue;
        }
        const T* row = V + (size_t)t * d;
        if (cls == 3) {
            __half* dst = reinterpret_cast<__half*>(tile + h.off_vseg[3]) + (size_t)li * d;
            for (int c = lane; c < d; c += 32) {
                const float x = load_as_float(row, c);
                if (!isfinite(x)) s.bad = 1;
                dst[c] = __float2half_rn(x);
            }
            if (lane == 0) {
                vparam[sl] = make_float2(0.0f, 0.0f);
                vz[sl] = 0;
            }
            continue;
        }
        const int bits = kBits(cls);
        float lo = INFINITY, hi = -INFINITY;
        bool ok = true;
        for (int c = lane; c < d; c += 32) {
            const float x = load_as_float(row, c);
            ok &= isfinite(x);
            lo = fminf(lo, x);
            hi = fmaxf(hi, x);
        }
        lo = warp_min(lo);
        hi = warp_max(hi);
        if (!__all_sync(0xffffffffu, ok) && lane == 0) s.bad = 1;
        double scale, zd;
        quant_params(lo, hi, bits, scale, zd);
        const int per = 8 / bits;
        const int rb = ref_row_bytes(d, bits);
        for (int m = lane; m < rb; m += 32) {
            uint32_t val = 0;
            for (int j = 0; j < per; ++j) {
                const int c = m * per + j;
                if (c < d) val |= quant_code(load_as_float(row, c), scale, zd, bits) << (j * bits);
            }
            tile[vbyte_offset(h, cls, li, m, d)] = (uint8_t)val;
        }
        if (lane == 0) {
            const float sf = (float)scale;
            const int64_t z = (int64_t)zd;
            vparam[sl] = make_float2(sf, (float)(-(double)sf * (double)z));
            vz[sl] = z;
        }
    }
    __syncthreads();
    // scale bounds of the 2-bit class (the tensor-core body's fixed-point ranges)
    if (tid == 0) s.kmax = s.vmax = 0u;
    __syncthreads();
    {
        uint32_t km = 0u, vm = 0u;  // non-negative floats order like their bit patterns
        for (int j = tid; j < h.c[0]; j += blockDim.x) km = max(km, __float_as_uint(fabsf(chan[h.kslot_base[0] + j].x)));
        for (int j = tid; j < h.r[0]; j += blockDim.x) vm = max(vm, __float_as_uint(fabsf(vparam[j].x)));
        atomicMax(&s.kmax, km);
        atomicMax(&s.vmax, vm);
    }
    __syncthreads();
    if (tid == 0) {
        reinterpret_cast<TileHeader*>(tile)->scale_bounds =
            bf16_bound_bits(__uint_as_float(s.kmax)) | (bf16_bound_bits(__uint_as_float(s.vmax)) << 16);
        if (head_status) head_status[unit] = s.bad ? RDKV_ENUMERIC : RDKV_OK;
    }
}

}  // namespace rdkv_b200

using namespace rdkv_b200;

extern "C" RDKV_API int rdkv_cuda_pack_plan(const uint8_t* v_bits, const uint8_t* k_bits,
                                            const rdkv_shape* s, int64_t* tile_offsets, void* stream) {
    if (!s || !v_bits || !k_bits || !tile_offsets) return RDKV_EINVAL;
    if (s->units < 1 || s->seq_len < 1 || s->head_dim < 1 || s->head_dim > 256) return RDKV_EINVAL;
    auto st = static_cast<cudaStream_t>(stream);
    int64_t* sizes = nullptr;
    RDKV_CUDA_TRY(cudaMallocAsync(&sizes, sizeof(int64_t) * s->units, st));
    pack_plan_kernel<<<s->units, 512, 0, st>>>(v_bits, k_bits, s->seq_len, s->head_dim, sizes);
    scan_kernel<<<1, 1024, 0, st>>>(sizes, s->units, tile_offsets);
    const int rc = launch_status();
    RDKV_CUDA_TRY(cudaFreeAsync(sizes, st));
    return rc;
}

extern "C" RDKV_API int rdkv_cuda_pack(const void* k, const void* v, int32_t dtype,
                                       const uint8_t* v_bits, const uint8_t* k_bits,
                                       const rdkv_shape* s, const int64_t* tile_offsets,
                                       uint8_t* arena, int32_t* head_status, void* stream) {
    if (!s || !k || !v || !v_bits || !k_bits || !tile_offsets || !arena) return RDKV_EINVAL;
    if (s->units < 1 || s->seq_len < 1 || s->head_dim < 1 || s->head_dim > 256) return RDKV_EINVAL;
    auto st = static_cast<cudaStream_t>(stream);
    if (dtype == RDKV_F32)
        pack_kernel<float><<<s->units, kPackThreads, 0, st>>>(
            static_cast<const float*>(k), static_cast<const float*>(v), v_bits, k_bits, s->seq_len,
            s->head_dim, tile_offsets, arena, head_status);
    else if (dtype == RDKV_F16)
        pack_kernel<__half><<<s->units, kPackThreads, 0, st>>>(
            static_cast<const __half*>(k), static_cast<const __half*>(v), v_bits, k_bits,
            s->seq_len, s->head_dim, tile_offsets, arena, head_status);
    else
        return RDKV_EINVAL;
    return launch_status();
}

// ---------------------------------------------------------------------------
// quantize_unit (quantizer.cpp:104-131) over many independent units: one
// warp per unit of `len` contiguous f32 values. Codes [units][len] u8,
// params per unit; status[u] = RDKV_ENUMERIC for a non-finite unit.
namespace rdkv_b200 {

__global__ void quantize_units_kernel(const float* __restrict__ x, int units, int len, int bits,
                                      uint8_t* __restrict__ codes, float* __restrict__ scale_out,
                                      int64_t* __restrict__ zero_out, int32_t* __restrict__ status) {
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    if (warp >= units) return;
    const float* row = x + (size_t)warp * len;
    float lo = row[0], hi = row[0];
    int bad = 0;
    for (int i = lane; i < len; i += 32) {
        const float v = row[i];
        bad |= !isfinite(v);
        lo = fminf(lo, v);
        hi = fmaxf(hi, v);
    }
    lo = -warp_max(-lo);
    hi = warp_max(hi);
    bad = __any_sync(0xffffffffu, bad);
    if (bad) {
        if (lane == 0) status[warp] = RDKV_ENUMERIC;
        return;
    }
    double scale, zd;
    quant_params(lo, hi, bits, scale, zd);
    for (int i = lane; i < len; i += 32) codes[(size_t)warp * len + i] = (uint8_t)quant_code(row[i], scale, zd, bits);
    if (lane == 0) {
        scale_out[warp] = (float)scale;
        zero_out[warp] = (int64_t)zd;
        status[warp] = RDKV_OK;
    }
}

}  // namespace rdkv_b200

extern "C" RDKV_API int rdkv_cuda_quantize_units(const float* values, int32_t units, int32_t len, int32_t bits,
                                                 uint8_t* codes, float* scale, int64_t* zero_point,
                                                 int32_t* status, void* stream) {
    if (bits != 2 && bits != 4 && bits != 8) return RDKV_EINVAL;  // quantizer.cpp:105-107
    if (len < 1) return RDKV_EINVAL;                               // :108
    if (units < 0 || !values || !codes || !scale || !zero_point || !status) return RDKV_EINVAL;
    if (units == 0) return RDKV_OK;
    const int threads = 256;
    const unsigned blocks = (unsigned)(((size_t)units * 32 + threads - 1) / threads);
    quantize_units_kernel<<<blocks, threads, 0, static_cast<cudaStream_t>(stream)>>>(
        values, units, len, bits, codes, scale, zero_point, status);
    return launch_status();
}

// ---- pack_bits / unpack_bits (trizone.cpp:59-88) ---------------------------
// Byte layout of the reference: 2-bit quarter-split (code j at bits 2 (j & 3) of
// byte j >> 2), 4-bit half-split (bits 4 (j & 1) of byte j >> 1), 8-bit one code
// per byte. One thread per 16 output bytes, written as one uint4 (the tail
// thread stores bytewise); a code above 2^bits - 1 raises the status flag.
namespace rdkv_b200 {
__global__ void __launch_bounds__(256) pack_bits_kernel(const uint8_t* __restrict__ codes, int64_t n, int bits,
                                                        uint8_t* __restrict__ out, int64_t nbytes,
                                                        int32_t* __restrict__ status) {
    const int per = 8 / bits;
    const uint32_t limit = (1u << bits) - 1u;
    for (int64_t b0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * 16; b0 < nbytes;
         b0 += (int64_t)gridDim.x * blockDim.x * 16) {
        uint8_t o[16];
        bool bad = false;
#pragma unroll
        for (int i = 0; i < 16; ++i) {
            uint32_t acc = 0;
            for (int e = 0; e < per; ++e) {
                const int64_t j = (b0 + i) * per + e;
                const uint32_t c = j < n ? codes[j] : 0u;
                bad |= c > limit;
                acc |= (c & limit) << (e * bits);
            }
            o[i] = (uint8_t)acc;
        }
        if (bad) atomicExch(status, RDKV_EINVAL);
        if (b0 + 16 <= nbytes && ((reinterpret_cast<uintptr_t>(out + b0) & 15) == 0)) {
            *reinterpret_cast<uint4*>(out + b0) = *reinterpret_cast<const uint4*>(o);
        } else {
            for (int i = 0; i < 16 && b0 + i < nbytes; ++i) out[b0 + i] = o[i];
        }
    }
}

__global__ void __launch_bounds__(256) unpack_bits_kernel(const uint8_t* __restrict__ bytes, int bits, int64_t len,
                                                          uint8_t* __restrict__ out) {
    const int per = 8 / bits;
    const uint32_t mask = (1u << bits) - 1u;
    for (int64_t j0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * 16; j0 < len;
         j0 += (int64_t)gridDim.x * blockDim.x * 16) {
        uint8_t o[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) {
            const int64_t j = j0 + i;
            o[i] = j < len ? (uint8_t)((bytes[j / per] >> ((j % per) * bits)) & mask) : 0;
        }
        if (j0 + 16 <= len && ((reinterpret_cast<uintptr_t>(out + j0) & 15) == 0)) {
            *reinterpret_cast<uint4*>(out + j0) = *reinterpret_cast<const uint4*>(o);
        } else {
            for (int i = 0; i < 16 && j0 + i < len; ++i) out[j0 + i] = o[i];
        }
    }
}
}  // namespace rdkv_b200

static int grid_for(int64_t items16) {
    const int64_t b = (items16 + 255) / 256;
    return (int)(b < 1 ? 1 : b > 148 * 16 ? 148 * 16 : b);
}

extern "C" RDKV_API int rdkv_cuda_pack_bits(const uint8_t* codes, int64_t n, int32_t bits, uint8_t* out,
                                            int32_t* status, void* stream) {
    if (bits != 2 && bits != 4 && bits != 8) return RDKV_EINVAL;
    if (n < 0 || (n > 0 && (!codes || !out)) || !status) return RDKV_EINVAL;
    const int per = 8 / bits;
    const int64_t nbytes = (n + per - 1) / per;
    auto st = static_cast<cudaStream_t>(stream);
    RDKV_CUDA_TRY(cudaMemsetAsync(status, 0, sizeof(int32_t), st));
    if (nbytes == 0) return RDKV_OK;
    rdkv_b200::pack_bits_kernel<<<grid_for((nbytes + 15) / 16), 256, 0, st>>>(codes, n, bits, out, nbytes, status);
    return rdkv_b200::launch_status();
}

extern "C" RDKV_API int rdkv_cuda_unpack_bits(const uint8_t* bytes, int64_t nbytes, int32_t bits,
                                              int64_t logical_len, uint8_t* out, void* stream) {
    if (bits != 2 && bits != 4 && bits != 8) return RDKV_EINVAL;
    const int per = 8 / bits;
    if (logical_len < 0 || (logical_len + per - 1) / per > nbytes) return RDKV_EINVAL;  // "byte buffer too short"
    if (logical_len == 0) return RDKV_OK;
    if (!bytes || !out) return RDKV_EINVAL;
    auto st = static_cast<cudaStream_t>(stream);
    rdkv_b200::unpack_bits_kernel<<<grid_for((logical_len + 15) / 16), 256, 0, st>>>(bytes, bits, logical_len, out);
    return rdkv_b200::launch_status();
}
