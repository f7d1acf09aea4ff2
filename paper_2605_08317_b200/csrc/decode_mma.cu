// decode_mma.cu — K4 tensor-core path: packed mixed-bit decode attention with
// dequantisation fused into int8 tensor-core products (head_dim 128).
//
// Replaces packed_decode_step / fused_k_logits (trizone.cpp:210-305) for
// every (batch, layer, KV head) tile of a step in ONE persistent launch.
//
// Why tensor cores: at n=128 a tile is ~10.5 KB and carries 128 tokens x 128
// channels x g=4 heads x 2 (QK+PV) = 131K MACs, i.e. ~12 MAC/byte. B200 CUDA
// cores sustain ~64 FFMA/clk/SM (3-reg form), ~5.5 MAC/byte of HBM
// bandwidth, so a CUDA-core decode caps at ~45% of the HBM roofline. The
// int8 mma.sync m16n8k32 consumes the packed codes as u8 operands straight
// from registers: one SHF+LOP3 pair extracts 4 two-bit codes into the 4 bytes
// of an A register, so the dequant costs ~0.5 ALU op per code.
//
// Per tile (one warp, no block-level synchronisation):
//  1. cp.async.bulk (TMA 1-D) stages the tile's decode region and its g
//     query rows into the warp's smem ring (mbarrier completion), NSTAGE deep.
//  2. q~ = scale_s * q[perm_s] per K slot, quantised per (bit class, head) to
//     a 24-bit fixed-point value split into three signed 8-bit digits (the B
//     operand, N = heads x digits); bias = sum q * offset.
//  3. QK: A = K codes of 16 token slots x 32 K slots (u8), B = digits (s8),
//     s32 accumulate; logit = (hi*256 + lo) / sigma + bias, * 1/sqrt(d).
//  4. softmax over the tile + Zone C with warp shuffles; p~ = p * vscale
//     quantised per (V class, head) to three unsigned 8-bit digits.
//  5. PV: A = V codes of 16 channels x 32 tokens (u8, 4-token interleave makes
//     one 32-bit word = 4 tokens), B = p~ digits (u8), s32 accumulate;
//     out = (PV + sum p * voffset + Zone B/C rows) / l.
// Fixed-point error: q~ <= 2^-24 and p~ <= 2^-25 relative to the per-class
// max per element, ~1e-6 relative on outputs (tolerance 1e-3, tests assert
// 1e-4 on FP16-representable inputs).
#include "common.cuh"

namespace rdkv_b200 {

constexpr int kD = 128;          // head_dim of this path
constexpr int kMaxSlots = 256;   // token slots per tile (16 m-tiles)
constexpr int kMaxZc = 256;      // Zone C tokens per tile on this path
constexpr int kMaxKSteps = 7;    // K slots of classes 2/4/8 <= 128 + 3*31 -> 7 k32 steps
constexpr int kMaxVSteps = 8;    // token k32 steps (256 slots)

// ---------------------------------------------------------------- PTX helpers
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(phase)
        : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void fence_barrier_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// D = A(u8, 16x32 row) * B(s8, 32x8 col) + C
__device__ __forceinline__ void mma_u8s8(int (&c)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k32.row.col.s32.u8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};\n"
        : "+r"(c[0]), "+r"(c[1]), "+r"(c[2]), "+r"(c[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
// D = A(u8) * B(u8) + C
__device__ __forceinline__ void mma_u8u8(int (&c)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k32.row.col.s32.u8.u8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};\n"
        : "+r"(c[0]), "+r"(c[1]), "+r"(c[2]), "+r"(c[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

__device__ __forceinline__ uint32_t lds32(const uint8_t* p) { return *reinterpret_cast<const uint32_t*>(p); }
__device__ __forceinline__ uint2 lds64(const uint8_t* p) { return *reinterpret_cast<const uint2*>(p); }

// Position (0..31) inside a k32 step of K slot `j` (0..31) of a class, for the
// A-fragment extraction of the QK loop: a 2-bit word (16 slots) yields
// slots {4e + tig} into K positions 4*tig + e; 4-bit words (8 slots) yield
// slots {2e + (tig & 1)} of word tig >> 1; 8-bit words are already bytes.
__device__ __forceinline__ int kpos_of_slot(int cls, int j) {
    if (cls == 0) {  // word w = j >> 4, slot-in-word s = 4e + tig
        const int w = j >> 4, s = j & 15;
        return w * 16 + (s & 3) * 4 + (s >> 2);
    }
    if (cls == 1) {  // word index wi = j >> 3 (0..3), slot-in-word s = 2e + jj
        const int wi = j >> 3, s = j & 7;
        const int tig = (wi & 1) * 2 + (s & 1);
        const int half = wi >> 1;  // words 0,1 -> a0 (K 0..15); words 2,3 -> a2 (K 16..31)
        return half * 16 + tig * 4 + (s >> 1);
    }
    return j;  // 8-bit: word tig holds slots 4tig..4tig+3, word 4+tig holds 16+4tig..
}

template <typename IO>
__device__ __forceinline__ float ld_io(const IO* p, int i);
template <>
__device__ __forceinline__ float ld_io<float>(const float* p, int i) { return p[i]; }
template <>
__device__ __forceinline__ float ld_io<__half>(const __half* p, int i) { return __half2float(p[i]); }

struct WarpSmem {
    uint8_t bq[kMaxKSteps * 4 * 8 * 32];   // QK B digits [kstep][n-tile (2 per 4 heads)][n][32]
    uint8_t bp[(kMaxVSteps + 3) * 4 * 8 * 32];  // PV B digits [kstep][n-tile (2 per 4 heads)][n][32]
    float acc[8 * kD];                     // [head][channel]
    float zl[8 * kMaxZc];                  // Zone C logits / probabilities
    float p16[8 * 64];                     // Zone B probabilities [head][row] (<= 64 rows)
    float sig[3][8];                       // sigma per (V class, head)
    float qsig[3][8];                      // sigma per (K class, head)
    uint64_t bar[4];
};

// One warp decodes one tile that sits in `t` (smem) with its q rows at `qs`.
template <int NT, typename IO>
__device__ __forceinline__ void decode_tile(const uint8_t* __restrict__ t, const IO* __restrict__ qs, int g,
                                            WarpSmem& w, const __half* __restrict__ zck,
                                            const __half* __restrict__ zcv, int nzc, IO* __restrict__ out) {
    const int lane = threadIdx.x & 31;
    const int gid = lane >> 2, tig = lane & 3;
    const TileHeader& h = *reinterpret_cast<const TileHeader*>(t);
    const int nslot = h.nslot;
    const float2* chan = reinterpret_cast<const float2*>(t + kHeaderBytes);
    const uint16_t* perm = reinterpret_cast<const uint16_t*>(t + kHeaderBytes + 8 * h.kslots);
    const float2* vparam = reinterpret_cast<const float2*>(t + h.off_vp);
    int sbase[5];
    sbase[0] = 0;
#pragma unroll
    for (int i = 0; i < 4; ++i) sbase[i + 1] = sbase[i] + pad4(h.r[i]);

    // ---------------------------------------------------------------- q~ digits
    float bias[NT];
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) bias[nt] = 0.0f;
    {
        // bias_h = sum_s q[h][perm_s] * offset_s; lane-strided partial, reduced below
        float bpart[8];
#pragma unroll
        for (int hh = 0; hh < 8; ++hh) bpart[hh] = 0.0f;
        for (int s = lane; s < h.kslots; s += 32) {
            const float2 cs = chan[s];
            const int ch = perm[s];
#pragma unroll
            for (int hh = 0; hh < 4 * NT; ++hh)
                if (hh < g) bpart[hh] = fmaf(ld_io(qs, hh * kD + ch), cs.y, bpart[hh]);
        }
#pragma unroll
        for (int hh = 0; hh < 4 * NT; ++hh) bpart[hh] = warp_sum(bpart[hh]);
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
            const int hh = nt * 4 + tig;
            float v = 0.0f;
#pragma unroll
            for (int k = 0; k < 4 * NT; ++k) v = (k == hh) ? bpart[k] : v;
            bias[nt] = v;
        }
    }
    int ks_base[3];
    {
        int acc = 0;
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            ks_base[c] = acc;
            acc += (h.c[c] + 31) >> 5;
        }
    }
    // q~ in 24-bit signed fixed point per (K class, head): three signed 8-bit
    // digits hi, mid, lo. B n-tiles come in pairs per 4 heads: tile 2*hb holds
    // columns (hi, mid) of head 4*hb + n/2, tile 2*hb + 1 holds (lo, 0).
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        const int nc = h.c[c];
        if (nc == 0) continue;
        const int P = (nc + 31) & ~31;
        for (int hh = 0; hh < 4 * NT; ++hh) {
            const int nt = hh >> 2, n0 = 2 * (hh & 3);
            if (hh >= g) {
                for (int j = lane; j < P; j += 32) {
                    const int ks = ks_base[c] + (j >> 5);
                    uint8_t* a0 = w.bq + ((ks * 2 * NT + 2 * nt) * 8) * 32;
                    uint8_t* a1 = a0 + 8 * 32;
                    a0[n0 * 32 + (j & 31)] = 0;
                    a0[(n0 + 1) * 32 + (j & 31)] = 0;
                    a1[n0 * 32 + (j & 31)] = 0;
                    a1[(n0 + 1) * 32 + (j & 31)] = 0;
                }
                continue;
            }
            float mx = 0.0f;
            for (int j = lane; j < nc; j += 32) {
                const int s = h.kslot_base[c] + j;
                mx = fmaxf(mx, fabsf(chan[s].x * ld_io(qs, hh * kD + perm[s])));
            }
            mx = warp_max(mx);
            const float sig = mx > 0.0f ? 8.2e6f / mx : 1.0f;
            if (lane == 0) w.qsig[c][hh] = sig;
            for (int j = lane; j < P; j += 32) {
                int dh = 0, dm = 0, dl = 0;
                if (j < nc) {
                    const int s = h.kslot_base[c] + j;
                    const int N = __float2int_rn(chan[s].x * ld_io(qs, hh * kD + perm[s]) * sig);
                    dl = ((N + 128) & 255) - 128;
                    const int N1 = (N - dl) >> 8;
                    dm = ((N1 + 128) & 255) - 128;
                    dh = (N1 - dm) >> 8;
                }
                const int ks = ks_base[c] + (j >> 5);
                const int kp = kpos_of_slot(c, j & 31);
                uint8_t* a0 = w.bq + ((ks * 2 * NT + 2 * nt) * 8) * 32;
                uint8_t* a1 = a0 + 8 * 32;
                a0[n0 * 32 + kp] = (uint8_t)(int8_t)dh;
                a0[(n0 + 1) * 32 + kp] = (uint8_t)(int8_t)dm;
                a1[n0 * 32 + kp] = (uint8_t)(int8_t)dl;
                a1[(n0 + 1) * 32 + kp] = 0;
            }
        }
    }
    __syncwarp();

    // ---------------------------------------------------------------- QK
    const int mtiles = (nslot + 15) >> 4;
    float lg[kMaxSlots / 16][2][NT];
    const uint8_t* krows = t + h.off_k;
    const float inv_sqrt_d = 0.08838834764831845f;  // 1/sqrt(128)
#pragma unroll
    for (int mt = 0; mt < kMaxSlots / 16; ++mt) {
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) lg[mt][0][nt] = lg[mt][1][nt] = 0.0f;
    }
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        if (h.c[c] == 0) continue;
        const int nks = (h.c[c] + 31) >> 5;
        const int kb0 = h.kbyte_base[c];
        const int step_bytes = 32 * kBits(c) / 8;  // 8 / 16 / 32
        for (int mt = 0; mt < mtiles; ++mt) {
            const int r0 = mt * 16 + gid, r1 = r0 + 8;
            int acc[2 * NT][4];
#pragma unroll
            for (int nt = 0; nt < 2 * NT; ++nt) acc[nt][0] = acc[nt][1] = acc[nt][2] = acc[nt][3] = 0;
            for (int kk = 0; kk < nks; ++kk) {
                const uint8_t* p0 = krows + (size_t)r0 * h.krow_bytes + kb0 + kk * step_bytes;
                const uint8_t* p1 = krows + (size_t)r1 * h.krow_bytes + kb0 + kk * step_bytes;
                uint32_t a[4];
                if (c == 0) {
                    const uint2 w0 = lds64(p0), w1 = lds64(p1);
                    const int sh = 2 * tig;
                    a[0] = (w0.x >> sh) & 0x03030303u;
                    a[2] = (w0.y >> sh) & 0x03030303u;
                    a[1] = (w1.x >> sh) & 0x03030303u;
                    a[3] = (w1.y >> sh) & 0x03030303u;
                } else if (c == 1) {
                    // class regions are 8-byte aligned inside a K row: two 8-byte loads
                    const uint2 x0 = lds64(p0), y0 = lds64(p0 + 8), x1 = lds64(p1), y1 = lds64(p1 + 8);
                    const int sh = 4 * (tig & 1);
                    const uint32_t lo0 = (tig >> 1) ? x0.y : x0.x, hi0 = (tig >> 1) ? y0.y : y0.x;
                    const uint32_t lo1 = (tig >> 1) ? x1.y : x1.x, hi1 = (tig >> 1) ? y1.y : y1.x;
                    a[0] = (lo0 >> sh) & 0x0F0F0F0Fu;
                    a[2] = (hi0 >> sh) & 0x0F0F0F0Fu;
                    a[1] = (lo1 >> sh) & 0x0F0F0F0Fu;
                    a[3] = (hi1 >> sh) & 0x0F0F0F0Fu;
                } else {
                    a[0] = lds32(p0 + 4 * tig);
                    a[2] = lds32(p0 + 16 + 4 * tig);
                    a[1] = lds32(p1 + 4 * tig);
                    a[3] = lds32(p1 + 16 + 4 * tig);
                }
                const int ks = ks_base[c] + kk;
#pragma unroll
                for (int nt = 0; nt < 2 * NT; ++nt) {
                    const uint8_t* bb = w.bq + ((ks * 2 * NT + nt) * 8 + gid) * 32 + 4 * tig;
                    mma_u8s8(acc[nt], a, lds32(bb), lds32(bb + 16));
                }
            }
#pragma unroll
            for (int nt = 0; nt < NT; ++nt) {
                const int hh = nt * 4 + tig;
                const float inv = hh < g ? 1.0f / w.qsig[c][hh] : 0.0f;
                const int* A = acc[2 * nt];
                const int* B = acc[2 * nt + 1];
                const float v0 = fmaf((float)A[0], 65536.0f, fmaf((float)A[1], 256.0f, (float)B[0])) * inv;
                const float v1 = fmaf((float)A[2], 65536.0f, fmaf((float)A[3], 256.0f, (float)B[2])) * inv;
#pragma unroll
                for (int m = 0; m < kMaxSlots / 16; ++m)
                    if (m == mt) {
                        lg[m][0][nt] += v0;
                        lg[m][1][nt] += v1;
                    }
            }
        }
    }
    // k16 channels (fp16 K columns), finalize logits and mask pads
    const int c16 = h.c[3];
    float mrun[NT];
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) mrun[nt] = -INFINITY;
#pragma unroll
    for (int mt = 0; mt < kMaxSlots / 16; ++mt) {
        if (mt >= mtiles) break;
#pragma unroll
        for (int half = 0; half < 2; ++half) {
            const int s = mt * 16 + gid + 8 * half;
            int cls = 0;
            while (cls < 3 && s >= sbase[cls + 1]) ++cls;
            const bool valid = s < nslot && (s - sbase[cls]) < h.r[cls];
#pragma unroll
            for (int nt = 0; nt < NT; ++nt) {
                const int hh = nt * 4 + tig;
                float v = lg[mt][half][nt];
                if (c16 && valid && hh < g) {
                    const __half* kr = reinterpret_cast<const __half*>(krows + (size_t)s * h.krow_bytes + h.kbyte_base[3]);
                    for (int j = 0; j < c16; ++j)
                        v = fmaf(ld_io(qs, hh * kD + perm[h.kslot_base[3] + j]), __half2float(kr[j]), v);
                }
                v = (valid && hh < g) ? (v + bias[nt]) * inv_sqrt_d : -INFINITY;
                lg[mt][half][nt] = v;
                mrun[nt] = fmaxf(mrun[nt], v);
            }
        }
    }
    // Zone C logits (CUDA cores): lane-per-token, all heads
    for (int i = lane; i < nzc; i += 32) {
        const __half* kr = zck + (size_t)i * kD;
        float a8[8];
#pragma unroll
        for (int hh = 0; hh < 8; ++hh) a8[hh] = 0.0f;
        for (int c0 = 0; c0 < kD; c0 += 8) {
            const uint4 raw = *reinterpret_cast<const uint4*>(kr + c0);
            const __half2* hp = reinterpret_cast<const __half2*>(&raw);
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const float2 kv = __half22float2(hp[e]);
#pragma unroll
                for (int hh = 0; hh < 4 * NT; ++hh)
                    if (hh < g)
                        a8[hh] = fmaf(ld_io(qs, hh * kD + c0 + 2 * e), kv.x,
                                      fmaf(ld_io(qs, hh * kD + c0 + 2 * e + 1), kv.y, a8[hh]));
            }
        }
#pragma unroll
        for (int hh = 0; hh < 4 * NT; ++hh)
            if (hh < g) w.zl[hh * kMaxZc + i] = a8[hh] * inv_sqrt_d;
    }
    __syncwarp();
    // running max over slots (8 lanes share a head) and Zone C
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) {
        float m = mrun[nt];
        m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, 4));
        m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, 8));
        m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, 16));
        const int hh = nt * 4 + tig;
        if (hh < g)
            for (int i = 0; i < nzc; ++i) m = fmaxf(m, w.zl[hh * kMaxZc + i]);
        mrun[nt] = m;
    }

    // ---------------------------------------------------------------- softmax
    float lsum[NT], bv[NT], pmax[3][NT];
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) {
        lsum[nt] = 0.0f;
        bv[nt] = 0.0f;
        pmax[0][nt] = pmax[1][nt] = pmax[2][nt] = 0.0f;
    }
#pragma unroll
    for (int mt = 0; mt < kMaxSlots / 16; ++mt) {
        if (mt >= mtiles) break;
#pragma unroll
        for (int half = 0; half < 2; ++half) {
            const int s = mt * 16 + gid + 8 * half;
            int cls = 0;
            while (cls < 3 && s >= sbase[cls + 1]) ++cls;
            const float2 vp = s < nslot ? vparam[s] : make_float2(0.0f, 0.0f);
#pragma unroll
            for (int nt = 0; nt < NT; ++nt) {
                const float l = lg[mt][half][nt];
                const float p = l == -INFINITY ? 0.0f : __expf(l - mrun[nt]);
                lsum[nt] += p;
                if (cls < 3) {
                    const float pt = p * vp.x;
                    bv[nt] = fmaf(p, vp.y, bv[nt]);
#pragma unroll
                    for (int c = 0; c < 3; ++c)
                        if (c == cls) pmax[c][nt] = fmaxf(pmax[c][nt], pt);
                    lg[mt][half][nt] = pt;  // now p~ (scaled by vscale)
                } else {
                    const int li = s - sbase[3];
                    const int hh = nt * 4 + tig;
                    if (hh < g && li < 64) w.p16[hh * 64 + li] = p;
                    lg[mt][half][nt] = 0.0f;
                }
            }
        }
    }
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) {
#pragma unroll
        for (int o = 4; o < 32; o <<= 1) {
            lsum[nt] += __shfl_xor_sync(0xffffffffu, lsum[nt], o);
            bv[nt] += __shfl_xor_sync(0xffffffffu, bv[nt], o);
#pragma unroll
            for (int c = 0; c < 3; ++c) pmax[c][nt] = fmaxf(pmax[c][nt], __shfl_xor_sync(0xffffffffu, pmax[c][nt], o));
        }
    }
    // broadcast per-head max to all lanes for Zone C (head hh lives in lane hh&3, n-tile hh>>2)
    float mh[8], lzc[8];
#pragma unroll
    for (int hh = 0; hh < 8; ++hh) {
        float m = 0.0f;
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
            const float v = __shfl_sync(0xffffffffu, mrun[nt], hh & 3);
            if ((hh >> 2) == nt) m = v;
        }
        mh[hh] = m;
        lzc[hh] = 0.0f;
    }
    for (int i = lane; i < nzc; i += 32) {
#pragma unroll
        for (int hh = 0; hh < 8; ++hh)
            if (hh < g) {
                const float p = __expf(w.zl[hh * kMaxZc + i] - mh[hh]);
                w.zl[hh * kMaxZc + i] = p;
                lzc[hh] += p;
            }
    }
#pragma unroll
    for (int hh = 0; hh < 8; ++hh) lzc[hh] = warp_sum(lzc[hh]);
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) {
        float z = 0.0f;
#pragma unroll
        for (int hh = 0; hh < 8; ++hh)
            if (hh == nt * 4 + tig) z = lzc[hh];
        lsum[nt] += z;
    }

    // p~ digits (unsigned 16-bit fixed point per (V class, head))
    float psig[3][NT];
#pragma unroll
    for (int c = 0; c < 3; ++c)
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) psig[c][nt] = pmax[c][nt] > 0.0f ? 1.6e7f / pmax[c][nt] : 0.0f;
    // zero the B-digit area of every V class k-step (tails of the last step)
    int vks[3], vks_base[3];
    {
        int acc = 0;
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            vks[c] = (pad4(h.r[c]) + 31) >> 5;
            vks_base[c] = acc;
            acc += vks[c];
        }
        uint4* z = reinterpret_cast<uint4*>(w.bp);
        const int n16 = acc * 2 * NT * 8 * 32 / 16;
        for (int i = lane; i < n16; i += 32) z[i] = make_uint4(0, 0, 0, 0);
    }
    __syncwarp();
#pragma unroll
    for (int mt = 0; mt < kMaxSlots / 16; ++mt) {
        if (mt >= mtiles) break;
#pragma unroll
        for (int half = 0; half < 2; ++half) {
            const int s = mt * 16 + gid + 8 * half;
            if (s >= sbase[3]) continue;
            int cls = 0;
            while (cls < 2 && s >= sbase[cls + 1]) ++cls;
            const int li = s - sbase[cls];
#pragma unroll
            for (int nt = 0; nt < NT; ++nt) {
                float sg = 0.0f;
#pragma unroll
                for (int c = 0; c < 3; ++c)
                    if (c == cls) sg = psig[c][nt];
                const int N = __float2int_rn(lg[mt][half][nt] * sg);
                const int ks = vks_base[cls] + (li >> 5);
                uint8_t* base = w.bp + ((ks * 2 * NT + 2 * nt) * 8 + 2 * tig) * 32 + (li & 31);
                base[0] = (uint8_t)(N >> 16);            // tile 2nt,   column 2tig   : hi
                base[32] = (uint8_t)((N >> 8) & 255);    // tile 2nt,   column 2tig+1 : mid
                base[8 * 32] = (uint8_t)(N & 255);       // tile 2nt+1, column 2tig   : lo
            }
        }
    }
    // publish per-head sigma for the PV combine (lane tig owns head nt*4+tig)
    if (gid == 0) {
#pragma unroll
        for (int nt = 0; nt < NT; ++nt)
#pragma unroll
            for (int c = 0; c < 3; ++c) w.sig[c][nt * 4 + tig] = psig[c][nt];
    }
    // zero the accumulator
    for (int i = lane; i < 8 * kD / 4; i += 32) reinterpret_cast<float4*>(w.acc)[i] = make_float4(0, 0, 0, 0);
    __syncwarp();

    // ---------------------------------------------------------------- PV
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        if (h.r[c] == 0) continue;
        const int rb = kD * kBits(c) / 8;  // packed row bytes at d = 128
        const uint8_t* vbase = t + h.off_vseg[c];
        for (int mt = 0; mt < kD / 16; ++mt) {
            int acc[2 * NT][4];
#pragma unroll
            for (int nt = 0; nt < 2 * NT; ++nt) acc[nt][0] = acc[nt][1] = acc[nt][2] = acc[nt][3] = 0;
            int ch0, ch1;
            for (int kk = 0; kk < vks[c]; ++kk) {
                const int gr0 = kk * 8 + tig, gr1 = gr0 + 4;  // token groups of this k-step
                uint32_t a[4];
                if (c == 0) {
                    const int m = 4 * mt + (gid & 3);
                    const uint32_t w0 = lds32(vbase + gr0 * 4 * rb + m * 4);
                    const uint32_t w1 = lds32(vbase + gr1 * 4 * rb + m * 4);
                    const int j0 = gid >> 2;
                    a[0] = (w0 >> (2 * j0)) & 0x03030303u;
                    a[1] = (w0 >> (2 * j0 + 4)) & 0x03030303u;
                    a[2] = (w1 >> (2 * j0)) & 0x03030303u;
                    a[3] = (w1 >> (2 * j0 + 4)) & 0x03030303u;
                } else if (c == 1) {
                    const int m = 8 * mt + gid;
                    const uint32_t w0 = lds32(vbase + gr0 * 4 * rb + m * 4);
                    const uint32_t w1 = lds32(vbase + gr1 * 4 * rb + m * 4);
                    a[0] = w0 & 0x0F0F0F0Fu;
                    a[1] = (w0 >> 4) & 0x0F0F0F0Fu;
                    a[2] = w1 & 0x0F0F0F0Fu;
                    a[3] = (w1 >> 4) & 0x0F0F0F0Fu;
                } else {
                    const int m0 = 16 * mt + gid, m1 = m0 + 8;
                    a[0] = lds32(vbase + gr0 * 4 * rb + m0 * 4);
                    a[1] = lds32(vbase + gr0 * 4 * rb + m1 * 4);
                    a[2] = lds32(vbase + gr1 * 4 * rb + m0 * 4);
                    a[3] = lds32(vbase + gr1 * 4 * rb + m1 * 4);
                }
                const int ks = vks_base[c] + kk;
#pragma unroll
                for (int nt = 0; nt < 2 * NT; ++nt) {
                    const uint8_t* bb = w.bp + ((ks * 2 * NT + nt) * 8 + gid) * 32 + 4 * tig;
                    mma_u8u8(acc[nt], a, lds32(bb), lds32(bb + 16));
                }
            }
            if (c == 0) {
                ch0 = 4 * (4 * mt + (gid & 3)) + (gid >> 2);
                ch1 = ch0 + 2;
            } else if (c == 1) {
                ch0 = 2 * (8 * mt + gid);
                ch1 = ch0 + 1;
            } else {
                ch0 = 16 * mt + gid;
                ch1 = ch0 + 8;
            }
#pragma unroll
            for (int nt = 0; nt < NT; ++nt) {
                const int hh = nt * 4 + tig;
                if (hh >= g) continue;
                const float sg = w.sig[c][hh];
                const float inv = sg > 0.0f ? 1.0f / sg : 0.0f;
                const int* A = acc[2 * nt];
                const int* B = acc[2 * nt + 1];
                w.acc[hh * kD + ch0] += fmaf((float)A[0], 65536.0f, fmaf((float)A[1], 256.0f, (float)B[0])) * inv;
                w.acc[hh * kD + ch1] += fmaf((float)A[2], 65536.0f, fmaf((float)A[3], 256.0f, (float)B[2])) * inv;
            }
        }
        __syncwarp();
    }

    // ---------------------------------------------------------------- Zone B + Zone C + output
    // lane owns channels 4*lane .. 4*lane+3 for every head
    float o[8][4];
#pragma unroll
    for (int hh = 0; hh < 8; ++hh)
#pragma unroll
        for (int e = 0; e < 4; ++e) o[hh][e] = 0.0f;
    const int r16 = min(h.r[3], 64);
    const __half* zb = reinterpret_cast<const __half*>(t + h.off_vseg[3]);
    for (int li = 0; li < r16; ++li) {
        const uint2 raw = *reinterpret_cast<const uint2*>(zb + (size_t)li * kD + 4 * lane);
        const __half2* hp = reinterpret_cast<const __half2*>(&raw);
        const float2 v01 = __half22float2(hp[0]), v23 = __half22float2(hp[1]);
#pragma unroll
        for (int hh = 0; hh < 8; ++hh)
            if (hh < g) {
                const float p = w.p16[hh * 64 + li];
                o[hh][0] = fmaf(p, v01.x, o[hh][0]);
                o[hh][1] = fmaf(p, v01.y, o[hh][1]);
                o[hh][2] = fmaf(p, v23.x, o[hh][2]);
                o[hh][3] = fmaf(p, v23.y, o[hh][3]);
            }
    }
    for (int i = 0; i < nzc; ++i) {
        const uint2 raw = *reinterpret_cast<const uint2*>(zcv + (size_t)i * kD + 4 * lane);
        const __half2* hp = reinterpret_cast<const __half2*>(&raw);
        const float2 v01 = __half22float2(hp[0]), v23 = __half22float2(hp[1]);
#pragma unroll
        for (int hh = 0; hh < 8; ++hh)
            if (hh < g) {
                const float p = w.zl[hh * kMaxZc + i];
                o[hh][0] = fmaf(p, v01.x, o[hh][0]);
                o[hh][1] = fmaf(p, v01.y, o[hh][1]);
                o[hh][2] = fmaf(p, v23.x, o[hh][2]);
                o[hh][3] = fmaf(p, v23.y, o[hh][3]);
            }
    }
    // per-head normaliser and V offset term, broadcast from lane (hh & 3)
#pragma unroll
    for (int hh = 0; hh < 8; ++hh) {
        if (hh >= g) break;
        float l = 0.0f, b = 0.0f;
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
            const float lv = __shfl_sync(0xffffffffu, lsum[nt], hh & 3);
            const float bb = __shfl_sync(0xffffffffu, bv[nt], hh & 3);
            if ((hh >> 2) == nt) {
                l = lv;
                b = bb;
            }
        }
        const float inv = 1.0f / l;
        const float4 a4 = reinterpret_cast<const float4*>(w.acc + hh * kD)[lane];
        const float r0 = (a4.x + o[hh][0] + b) * inv;
        const float r1 = (a4.y + o[hh][1] + b) * inv;
        const float r2 = (a4.z + o[hh][2] + b) * inv;
        const float r3 = (a4.w + o[hh][3] + b) * inv;
        if constexpr (sizeof(IO) == 2) {
            __half2 p0 = __floats2half2_rn(r0, r1), p1 = __floats2half2_rn(r2, r3);
            uint2 st;
            st.x = *reinterpret_cast<uint32_t*>(&p0);
            st.y = *reinterpret_cast<uint32_t*>(&p1);
            reinterpret_cast<uint2*>(out + hh * kD)[lane] = st;
        } else {
            reinterpret_cast<float4*>(out + hh * kD)[lane] = make_float4(r0, r1, r2, r3);
        }
    }
    __syncwarp();
}

template <int NT, typename IO>
__global__ void __launch_bounds__(256, 1) decode_mma_kernel(
    const uint8_t* __restrict__ arena, const int64_t* __restrict__ offsets, const int32_t* __restrict__ dsize,
    int units, int g, const IO* __restrict__ q_all, IO* __restrict__ out_all, const __half* __restrict__ zc_k,
    const __half* __restrict__ zc_v, const int32_t* __restrict__ zc_len, int zc_cap, int stage_bytes,
    int nstage) {
    extern __shared__ __align__(128) uint8_t dsm[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nwarps = blockDim.x >> 5;
    const size_t per_warp = (size_t)nstage * stage_bytes + ((sizeof(WarpSmem) + 127) & ~size_t(127));
    uint8_t* mine = dsm + per_warp * warp;
    WarpSmem& w = *reinterpret_cast<WarpSmem*>(mine + (size_t)nstage * stage_bytes);
    const int qbytes = g * kD * (int)sizeof(IO);
    const int worker = blockIdx.x * nwarps + warp;
    const int nworkers = gridDim.x * nwarps;
    if (lane == 0) {
        for (int s = 0; s < nstage; ++s) mbar_init(&w.bar[s], 1);
        fence_barrier_init();
    }
    __syncwarp();
    // prologue: issue the first nstage tiles
    if (lane == 0) {
        for (int s = 0; s < nstage; ++s) {
            const int tile = worker + s * nworkers;
            if (tile >= units) break;
            uint8_t* st = mine + (size_t)s * stage_bytes;
            const uint32_t tb = (uint32_t)dsize[tile];
            mbar_expect_tx(&w.bar[s], tb + qbytes);
            bulk_g2s(st, arena + offsets[tile], tb, &w.bar[s]);
            bulk_g2s(st + stage_bytes - qbytes, q_all + (size_t)tile * g * kD, qbytes, &w.bar[s]);
        }
    }
    int it = 0;
    for (int tile = worker; tile < units; tile += nworkers, ++it) {
        const int s = it % nstage;
        const uint32_t phase = (uint32_t)((it / nstage) & 1);
        mbar_wait(&w.bar[s], phase);
        const uint8_t* st = mine + (size_t)s * stage_bytes;
        const IO* qs = reinterpret_cast<const IO*>(st + stage_bytes - qbytes);
        const int nzc = zc_len ? min(zc_len[tile], kMaxZc) : 0;
        decode_tile<NT, IO>(st, qs, g, w, zc_k ? zc_k + (size_t)tile * zc_cap * kD : nullptr,
                            zc_v ? zc_v + (size_t)tile * zc_cap * kD : nullptr, nzc,
                            out_all + (size_t)tile * g * kD);
        __syncwarp();
        const int next = tile + nstage * nworkers;
        if (lane == 0 && next < units) {
            fence_proxy_async();
            uint8_t* dst = mine + (size_t)s * stage_bytes;
            const uint32_t tb = (uint32_t)dsize[next];
            mbar_expect_tx(&w.bar[s], tb + qbytes);
            bulk_g2s(dst, arena + offsets[next], tb, &w.bar[s]);
            bulk_g2s(dst + stage_bytes - qbytes, q_all + (size_t)next * g * kD, qbytes, &w.bar[s]);
        }
        __syncwarp();
    }
}

}  // namespace rdkv_b200

using namespace rdkv_b200;

namespace rdkv_b200 {

bool mma_supported(const rdkv_decode_args* a) {
    if (a->head_dim != kD || a->group > 8 || !a->tile_decode_bytes) return false;
    if (a->zc_len && a->zc_cap > kMaxZc) return false;
    const rdkv_decode_plan& p = a->plan;
    return p.max_decode_bytes > 0 && p.max_slots <= kMaxSlots && p.max_zone_b_rows <= 64 &&
           p.max_kq_slots <= kMaxKSteps * 32;
}

template <int NT, typename IO>
static int launch_t(const rdkv_decode_args* a, cudaStream_t st) {
    const int qbytes = a->group * kD * (int)sizeof(IO);
    const int stage = (a->plan.max_decode_bytes + qbytes + 127) & ~127;
    const int wsm = (int)((sizeof(WarpSmem) + 127) & ~size_t(127));
    int dev = 0;
    cudaGetDevice(&dev);
    int smem_max = 0, nsm = 0;
    cudaDeviceGetAttribute(&smem_max, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    int nstage = 3;
    int per_warp = nstage * stage + wsm;
    if (per_warp * 4 > smem_max) {
        nstage = 2;
        per_warp = nstage * stage + wsm;
    }
    int warps = smem_max / per_warp;
    if (warps > 8) warps = 8;
    if (warps < 1) return RDKV_EINVAL;
    const size_t smem = (size_t)warps * per_warp;
    auto kern = decode_mma_kernel<NT, IO>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int blocks = (a->units + warps - 1) / warps;
    if (blocks > nsm) blocks = nsm;
    kern<<<blocks, warps * 32, smem, st>>>(a->arena, a->tile_offsets, a->tile_decode_bytes, a->units, a->group,
                                           static_cast<const IO*>(a->q), static_cast<IO*>(a->out),
                                           static_cast<const __half*>(a->zc_k), static_cast<const __half*>(a->zc_v),
                                           a->zc_len, a->zc_cap, stage, nstage);
    return launch_status();
}

int launch_mma(const rdkv_decode_args* a, cudaStream_t st) {
    const bool f16 = a->io_dtype == RDKV_F16;
    if (a->group <= 4) return f16 ? launch_t<1, __half>(a, st) : launch_t<1, float>(a, st);
    return f16 ? launch_t<2, __half>(a, st) : launch_t<2, float>(a, st);
}

}  // namespace rdkv_b200

// Scans every tile header once (one small D2H copy per tile) and writes the
// per-tile decode sizes the persistent kernel stages with cp.async.bulk, plus
// the maxima that select the kernel and its smem ring. Call once after packing.
extern "C" RDKV_API int rdkv_cuda_decode_prepare(const uint8_t* arena, const int64_t* tile_offsets_host,
                                                 int32_t units, int32_t* decode_bytes_dev,
                                                 rdkv_decode_plan* plan, void* stream) {
    if (!arena || !tile_offsets_host || !decode_bytes_dev || !plan || units < 1) return RDKV_EINVAL;
    auto st = static_cast<cudaStream_t>(stream);
    TileHeader* hdrs = static_cast<TileHeader*>(malloc(sizeof(TileHeader) * (size_t)units));
    int32_t* ds = static_cast<int32_t*>(malloc(sizeof(int32_t) * (size_t)units));
    int rc = RDKV_OK;
    for (int u = 0; u < units; ++u)
        cudaMemcpyAsync(&hdrs[u], arena + tile_offsets_host[u], sizeof(TileHeader), cudaMemcpyDeviceToHost, st);
    if (cudaStreamSynchronize(st) != cudaSuccess) rc = RDKV_ECUDA;
    rdkv_decode_plan p{0, 0, 0, 0};
    for (int u = 0; u < units && rc == RDKV_OK; ++u) {
        const TileHeader& h = hdrs[u];
        if (h.magic != kTileMagic) {
            rc = RDKV_EFORMAT;
            break;
        }
        ds[u] = (int32_t)tile_decode_bytes(h);
        p.max_decode_bytes = ds[u] > p.max_decode_bytes ? ds[u] : p.max_decode_bytes;
        p.max_slots = h.nslot > p.max_slots ? h.nslot : p.max_slots;
        p.max_zone_b_rows = h.r[3] > p.max_zone_b_rows ? h.r[3] : p.max_zone_b_rows;
        p.max_kq_slots = h.kslot_base[3] > p.max_kq_slots ? h.kslot_base[3] : p.max_kq_slots;
    }
    if (rc == RDKV_OK) {
        if (cudaMemcpyAsync(decode_bytes_dev, ds, sizeof(int32_t) * (size_t)units, cudaMemcpyHostToDevice, st) !=
                cudaSuccess ||
            cudaStreamSynchronize(st) != cudaSuccess)
            rc = RDKV_ECUDA;
        *plan = p;
    }
    free(hdrs);
    free(ds);
    return rc;
}
