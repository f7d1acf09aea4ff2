// decode_mma.cu — K4 tensor-core path: packed mixed-bit decode attention with
// dequantisation fused into int8 tensor-core products (head_dim 128).
//
// Replaces packed_decode_step / fused_k_logits (trizone.cpp:210-305) for
// every (batch, layer, KV head) tile of a step in ONE persistent launch.
//
// Why tensor cores: at n=128 a tile is ~10.5 KB and carries 128 tokens x 128
// channels x g=4 heads x 2 (QK+PV) = 131K MACs, ~12 MAC/byte. B200 CUDA cores
// issue ~64 FFMA/clk/SM (3-register form), ~5.5 MAC per byte of HBM
// bandwidth, so a CUDA-core decode caps near 45% of the HBM roofline. The
// int8 mma.sync m16n8k32 consumes the packed codes as u8 operands straight
// from registers: one SHF + LOP3 pair turns a 32-bit word of 2-bit codes into
// an A register holding four codes, so dequantisation costs ~0.5 ALU op per
// code and the multiply-adds leave the CUDA cores entirely.
//
// CTA organisation (persistent, one CTA per SM):
//   warp 0      producer: walks the CTA's tiles and stages each tile's decode
//               region plus its g query rows into a ring of R smem slots with
//               cp.async.bulk (TMA 1-D), completion on a per-slot mbarrier;
//               a slot is refilled once its consumer releases it.
//   warps 1..W  consumers: warp w decodes tiles w, w+W, ... of the CTA, one
//               tile per warp, with no block-level synchronisation.
// Per tile (one consumer warp; intermediates in warp-private smem so the
// m-tile loops stay rolled and the SASS fits the instruction cache):
//   1. q~ = scale_s * q[perm_s] per K slot in 24-bit signed fixed point
//      (three s8 digits) against the bound max|scale| * max|q| of each
//      (bit class, head); bias = sum_s q[perm_s] * offset_s.
//   2. QK: A = K codes of 16 token slots x 32 K slots (u8), B = q~ digits (s8),
//      s32 accumulate; logit = (hi*2^16 + mid*2^8 + lo) / sigma + bias.
//   3. softmax over the tile (+ Zone C), one lane per token, shuffles;
//      p~ = p * vscale in 24-bit unsigned fixed point (three u8 digits).
//   4. PV: A = V codes of 16 channels x 32 tokens (u8; the 4-token interleave
//      makes one 32-bit word = 4 tokens of one byte column), B = p~ digits,
//      s32 accumulate; out = (PV / sigma + sum p * voffset + Zone B/C) / l.
// Fixed-point error ~2^-22 relative per element, ~1e-6 relative on outputs
// (tolerance 1e-3; tests assert 1e-4 on FP16-representable inputs).
#include "common.cuh"

#include <cstdio>

namespace rdkv_b200 {

constexpr int kD = 128;        // head_dim of this path
constexpr int kMaxR = 32;      // ring slots per CTA
constexpr int kMaxW = 12;      // consumer warps per CTA (13 warps -> <=152 regs)
constexpr int kMaxSlots = 4096; // token slots per tile on this path (smem permitting, general_min_smem)

// ---------------------------------------------------------------- PTX helpers
#define getenv_pair_smsp() (p.smsp_pairs)
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
__device__ __forceinline__ void mbar_expect_tx_only(uint64_t* bar, uint32_t bytes) {  // no arrive
    asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
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
// TMA bulk store smem -> global (bulk async-group completion)
__device__ __forceinline__ void bulk_s2g(void* dst, const void* src, uint32_t bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(smem_u32(src)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait0() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void fence_barrier_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// D = A(u8, 16x32 row-major) * B(s8, 32x8 col-major) + C, s32 accumulate
__device__ __forceinline__ void mma_u8s8(int (&c)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
    asm(
        "mma.sync.aligned.m16n8k32.row.col.s32.u8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};\n"
        : "+r"(c[0]), "+r"(c[1]), "+r"(c[2]), "+r"(c[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
// D = A(u8) * B(u8) + C
__device__ __forceinline__ void mma_u8u8(int (&c)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
    asm(
        "mma.sync.aligned.m16n8k32.row.col.s32.u8.u8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};\n"
        : "+r"(c[0]), "+r"(c[1]), "+r"(c[2]), "+r"(c[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

__device__ __forceinline__ uint32_t lds32(const uint8_t* p) { return *reinterpret_cast<const uint32_t*>(p); }
__device__ __forceinline__ uint2 lds64(const uint8_t* p) { return *reinterpret_cast<const uint2*>(p); }

// K slot (0..31 within a k32 step) feeding MMA K position `p`, per class.
// 2-bit: a K-row word holds 16 slots; (w >> 2*tig) & 0x03030303 yields slots
// {4e + tig} as bytes e, i.e. K positions 4*tig + e. 4-bit: words of 8 slots,
// (w >> 4*(tig&1)) & 0x0F0F0F0F yields slots {2e + (tig&1)} of word tig>>1
// (a0) / 2 + (tig>>1) (a2). 8-bit: identity.
__device__ __forceinline__ int slot_of_kpos(int cls, int p) {
    if (cls == 0) {
        const int r = p & 15;
        return (p & 16) + 4 * (r & 3) + (r >> 2);
    }
    if (cls == 1) {
        const int half = p >> 4, r = p & 15;
        const int tig = r >> 2, e = r & 3;
        return 16 * half + 8 * (tig >> 1) + 2 * e + (tig & 1);
    }
    return p;
}

template <typename IO>
__device__ __forceinline__ float ld_io(const IO* p, int i);
template <>
__device__ __forceinline__ float ld_io<float>(const float* p, int i) { return p[i]; }
template <>
__device__ __forceinline__ float ld_io<__half>(const __half* p, int i) { return __half2float(p[i]); }

struct MmaParams {
    const uint8_t* arena;
    const int64_t* offsets;
    const int32_t* dsize;
    const void* q;
    void* out;
    const __half* zc_k;
    const __half* zc_v;
    const int32_t* zc_len;
    int units, g, zc_cap;
    int R, W;               // ring slots, consumer warps
    int slot_bytes;         // per ring slot (tile decode region + q rows)
    int scratch_bytes;      // per consumer warp
    int off_lg;             // byte offsets inside the per-warp scratch
    int lg_stride;          // per-head stride (floats) of the logit scratch
    int off_p16, off_zl;    // -1 when unused
    int max_r16;
    int smsp_pairs;  // u2x: a pair's two warps on one SM sub-partition
    const int32_t* ids;  // launch tile -> unit (NULL: identity), a split step's subset
    int concurrent;      // u2x of a split step: runs beside the general kernel (see launch_mma)
    float* partial;      // u2c sequence split: [units][g][d + 2] (o, max, sum) of this rank's chunks
    int split_rank, split_world;
};
__device__ __forceinline__ int unit_of(const MmaParams& p, int tile) { return p.ids ? p.ids[tile] : tile; }

// Per-warp scratch: [ScratchHead][B digits][lg / acc][p16][zl]
struct ScratchHead {
    float qinv[3][8];   // 1/sigma per (K class, head)
    float vinv[3][8];   // 1/sigma per (V class, head)
};
constexpr int kDigitBytesOff = 256;
constexpr int kPartStride = kD + 4;  // floats per head of a chunk partial (16-B aligned rows)

// PART: `part` receives this (sub-)tile's unnormalised softmax state per head,
// [g][kPartStride] = (sum_i p_i v_i [d], max logit (natural units), sum_i p_i), for the
// chunked body (decode_gchunk_kernel) whose chunks are merged afterwards.
template <int NT, typename IO, bool PART = false>
__device__ __noinline__ void decode_tile(const uint8_t* __restrict__ t, const IO* __restrict__ qs, int g,
                                         uint8_t* __restrict__ scr, const MmaParams& prm,
                                         const __half* __restrict__ zck, const __half* __restrict__ zcv,
                                         int nzc, IO* __restrict__ out, float* __restrict__ part = nullptr) {
    constexpr int G4 = 4 * NT;  // head capacity of the n-tiles
    constexpr int TS = 32 / G4; // lanes per head in the per-head phases
    const int lane = threadIdx.x & 31;
    const int gid = lane >> 2, tig = lane & 3;
    // per-head phases: head hl = lane % G4, tokens / channels tl, tl + TS, ...
    const int hl = lane % G4, tl = lane / G4;
    const bool hv = hl < g;
    const TileHeader& h = *reinterpret_cast<const TileHeader*>(t);
    ScratchHead& sh = *reinterpret_cast<ScratchHead*>(scr);
    uint8_t* dig = scr + kDigitBytesOff;
    const int LS = prm.lg_stride;
    float* lgs = reinterpret_cast<float*>(scr + prm.off_lg);  // [G4][LS] logits, later acc [G4][kD]
    float* p16 = prm.off_p16 >= 0 ? reinterpret_cast<float*>(scr + prm.off_p16) : nullptr;
    float* zl = prm.off_zl >= 0 ? reinterpret_cast<float*>(scr + prm.off_zl) : nullptr;
    const float2* chan = reinterpret_cast<const float2*>(t + kHeaderBytes);
    const uint16_t* perm = reinterpret_cast<const uint16_t*>(t + kHeaderBytes + 8 * h.kslots);
    const float2* vparam = reinterpret_cast<const float2*>(t + h.off_vp);
    const float inv_sqrt_d = 0.08838834764831845f;  // 1/sqrt(128)
    int sb[5];
    sb[0] = 0;
#pragma unroll
    for (int c = 0; c < 4; ++c) sb[c + 1] = sb[c] + pad4(h.r[c]);
    const int nslot = sb[4];
    auto hred_max = [&](float v) {
#pragma unroll
        for (int o = G4; o < 32; o <<= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
        return v;
    };
    auto hred_sum = [&](float v) {
#pragma unroll
        for (int o = G4; o < 32; o <<= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        return v;
    };

    // ------------------------------------------------------------ q statistics
    float qm = 0.0f, bias = 0.0f;
    if (hv) {
        for (int ch = tl; ch < kD; ch += TS) qm = fmaxf(qm, fabsf(ld_io(qs, hl * kD + ch)));
        for (int s = tl; s < h.kslots; s += TS) bias = fmaf(ld_io(qs, hl * kD + perm[s]), chan[s].y, bias);
    }
    qm = hred_max(qm);
    bias = hred_sum(bias);

    // ------------------------------------------------------------ q~ digits
    // N = round(q~ * sigma) in [-2^23, 2^23); the bytes of (N + 0x808080) ^ 0x808080
    // are its signed base-256 digits lo, mid, hi.
    int ksb[4];
    ksb[0] = 0;
    for (int c = 0; c < 3; ++c) ksb[c + 1] = ksb[c] + ((h.c[c] + 31) >> 5);
    for (int c = 0; c < 3; ++c) {
        const int nk = ksb[c + 1] - ksb[c];
        if (nk == 0) continue;
        float sm = 0.0f;
        for (int j = lane; j < h.c[c]; j += 32) sm = fmaxf(sm, fabsf(chan[h.kslot_base[c] + j].x));
        sm = warp_max(sm);
        const float bnd = sm * qm;
        const float sg = bnd > 0.0f ? 8.2e6f * __frcp_rn(bnd) : 0.0f;
        if (tl == 0) sh.qinv[c][hl] = bnd * (1.0f / 8.2e6f);
        const int ntask = nk * G4 * 8;  // task = (head hl, 4 K positions k4, k-step kk)
        for (int i = lane; i < ntask; i += 32) {
            const int k4 = (i / G4) & 7, kk = i / (8 * G4);
            uint32_t x[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const int j = kk * 32 + slot_of_kpos(c, 4 * k4 + e);
                int N = 0;
                if (hv && j < h.c[c]) {
                    const int s = h.kslot_base[c] + j;
                    N = __float2int_rn(chan[s].x * ld_io(qs, hl * kD + perm[s]) * sg);
                }
                x[e] = (uint32_t)(N + 0x808080) ^ 0x808080u;
            }
            const uint32_t wlo = __byte_perm(__byte_perm(x[0], x[1], 0x0040), __byte_perm(x[2], x[3], 0x0040), 0x5410);
            const uint32_t wmid = __byte_perm(__byte_perm(x[0], x[1], 0x0051), __byte_perm(x[2], x[3], 0x0051), 0x5410);
            const uint32_t whi = __byte_perm(__byte_perm(x[0], x[1], 0x0062), __byte_perm(x[2], x[3], 0x0062), 0x5410);
            const int ks = ksb[c] + kk;
            uint8_t* a0 = dig + ((ks * 2 * NT + 2 * (hl >> 2)) * 8 + 2 * (hl & 3)) * 32 + 4 * k4;
            *reinterpret_cast<uint32_t*>(a0) = whi;
            *reinterpret_cast<uint32_t*>(a0 + 32) = wmid;
            *reinterpret_cast<uint32_t*>(a0 + 8 * 32) = wlo;
            *reinterpret_cast<uint32_t*>(a0 + 8 * 32 + 32) = 0u;
        }
    }
    if (ksb[3] == 0) {  // every K channel removed: logits are the bias alone
        for (int s = tl; s < nslot; s += TS) lgs[hl * LS + s] = 0.0f;
    }
    __syncwarp();

    // ------------------------------------------------------------ QK (tensor cores)
    const uint8_t* krows = t + h.off_k;
    const int krb = h.krow_bytes;
    bool first = true;
    for (int c = 0; c < 3; ++c) {
        const int nk = ksb[c + 1] - ksb[c];
        if (nk == 0) continue;
        uint32_t b[4][2 * NT][2];
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)
#pragma unroll
            for (int nt = 0; nt < 2 * NT; ++nt) {
                const uint8_t* bb = dig + (((ksb[c] + kk) * 2 * NT + nt) * 8 + gid) * 32 + 4 * tig;
                b[kk][nt][0] = kk < nk ? lds32(bb) : 0u;
                b[kk][nt][1] = kk < nk ? lds32(bb + 16) : 0u;
            }
        float qinv[NT];
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) qinv[nt] = sh.qinv[c][nt * 4 + tig];
        const int kb0 = h.kbyte_base[c];
        // two m-tiles (32 token slots) per iteration for independent MMA chains
        for (int mt = 0; mt * 16 < nslot; mt += 2) {
            const bool two = (mt + 1) * 16 < nslot;
            int acc[2][2 * NT][4];
#pragma unroll
            for (int u = 0; u < 2; ++u)
#pragma unroll
                for (int nt = 0; nt < 2 * NT; ++nt) acc[u][nt][0] = acc[u][nt][1] = acc[u][nt][2] = acc[u][nt][3] = 0;
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) {
                if (kk < nk) {
#pragma unroll
                    for (int u = 0; u < 2; ++u) {
                        if (u == 1 && !two) continue;
                        const uint8_t* p0 = krows + (size_t)krow_pos(h, (mt + u) * 16 + gid) * krb + kb0;
                        const uint8_t* p1 = krows + (size_t)krow_pos(h, (mt + u) * 16 + gid + 8) * krb + kb0;
                        uint32_t a[4];
                        if (c == 0) {
                            const uint2 w0 = lds64(p0 + 8 * kk), w1 = lds64(p1 + 8 * kk);
                            const int s = 2 * tig;
                            a[0] = (w0.x >> s) & 0x03030303u;
                            a[2] = (w0.y >> s) & 0x03030303u;
                            a[1] = (w1.x >> s) & 0x03030303u;
                            a[3] = (w1.y >> s) & 0x03030303u;
                        } else if (c == 1) {
                            const int o = 16 * kk + 4 * (tig >> 1);
                            const int s = 4 * (tig & 1);
                            a[0] = (lds32(p0 + o) >> s) & 0x0F0F0F0Fu;
                            a[2] = (lds32(p0 + o + 8) >> s) & 0x0F0F0F0Fu;
                            a[1] = (lds32(p1 + o) >> s) & 0x0F0F0F0Fu;
                            a[3] = (lds32(p1 + o + 8) >> s) & 0x0F0F0F0Fu;
                        } else {
                            const int o = 32 * kk + 4 * tig;
                            a[0] = lds32(p0 + o);
                            a[2] = lds32(p0 + o + 16);
                            a[1] = lds32(p1 + o);
                            a[3] = lds32(p1 + o + 16);
                        }
#pragma unroll
                        for (int nt = 0; nt < 2 * NT; ++nt) mma_u8s8(acc[u][nt], a, b[kk][nt][0], b[kk][nt][1]);
                    }
                }
            }
#pragma unroll
            for (int u = 0; u < 2; ++u) {
                if (u == 1 && !two) continue;
#pragma unroll
                for (int nt = 0; nt < NT; ++nt) {
                    const int* A = acc[u][2 * nt];
                    const int* B = acc[u][2 * nt + 1];
                    float* row = lgs + (nt * 4 + tig) * LS + (mt + u) * 16 + gid;
                    const float v0 = fmaf((float)A[0], 65536.0f, fmaf((float)A[1], 256.0f, (float)B[0])) * qinv[nt];
                    const float v1 = fmaf((float)A[2], 65536.0f, fmaf((float)A[3], 256.0f, (float)B[2])) * qinv[nt];
                    row[0] = first ? v0 : row[0] + v0;
                    row[8] = first ? v1 : row[8] + v1;
                }
            }
        }
        first = false;
        __syncwarp();
    }

    // ------------------------------------------------------------ logits + max (per class, no pads)
    const int c16 = h.c[3];
    float mx = -INFINITY;
    float vsm[3] = {0.0f, 0.0f, 0.0f};  // max V scale per class (bounds p~ = p * vscale <= vscale)
    for (int c = 0; c < 4; ++c) {
        const int s1 = sb[c] + h.r[c];
        for (int s = sb[c] + tl; s < s1; s += TS) {
            if (c < 3) {
                const float vs = vparam[s].x;
                vsm[0] = c == 0 ? fmaxf(vsm[0], vs) : vsm[0];
                vsm[1] = c == 1 ? fmaxf(vsm[1], vs) : vsm[1];
                vsm[2] = c == 2 ? fmaxf(vsm[2], vs) : vsm[2];
            }
            if (!hv) continue;
            float v = lgs[hl * LS + s];
            if (c16) {
                const __half* kr = reinterpret_cast<const __half*>(krows + (size_t)krow_pos(h, s) * krb + h.kbyte_base[3]);
                for (int j = 0; j < c16; ++j)
                    v = fmaf(ld_io(qs, hl * kD + perm[h.kslot_base[3] + j]), __half2float(kr[j]), v);
            }
            v = (v + bias) * inv_sqrt_d;
            lgs[hl * LS + s] = v;
            mx = fmaxf(mx, v);
        }
    }
    if (nzc > 0) {  // Zone C logits on CUDA cores: lane per appended token, every head
        for (int i = lane; i < nzc; i += 32) {
            const __half* kr = zck + (size_t)i * kD;
            float a8[G4];
#pragma unroll
            for (int hh = 0; hh < G4; ++hh) a8[hh] = 0.0f;
            for (int c0 = 0; c0 < kD; c0 += 8) {
                const uint4 raw = *reinterpret_cast<const uint4*>(kr + c0);
                const __half2* hp = reinterpret_cast<const __half2*>(&raw);
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const float2 kv = __half22float2(hp[e]);
#pragma unroll
                    for (int hh = 0; hh < G4; ++hh)
                        if (hh < g)
                            a8[hh] = fmaf(ld_io(qs, hh * kD + c0 + 2 * e), kv.x,
                                          fmaf(ld_io(qs, hh * kD + c0 + 2 * e + 1), kv.y, a8[hh]));
                }
            }
#pragma unroll
            for (int hh = 0; hh < G4; ++hh)
                if (hh < g) zl[hh * prm.zc_cap + i] = a8[hh] * inv_sqrt_d;
        }
        __syncwarp();
        if (hv)
            for (int i = tl; i < nzc; i += TS) mx = fmaxf(mx, zl[hl * prm.zc_cap + i]);
    }
    mx = hred_max(mx);
    float psig[3];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        vsm[c] = hred_max(vsm[c]);
        psig[c] = vsm[c] > 0.0f ? 1.6e7f * __frcp_rn(vsm[c]) : 0.0f;
        if (lane == 0) sh.vinv[c][0] = vsm[c] * (1.0f / 1.6e7f);
    }
    int vksb[4];
    vksb[0] = 0;
    for (int c = 0; c < 3; ++c) vksb[c + 1] = vksb[c] + ((pad4(h.r[c]) + 31) >> 5);
    {
        uint4* z = reinterpret_cast<uint4*>(dig);
        const int n16 = vksb[3] * 2 * NT * 8 * 32 / 16;
        for (int i = lane; i < n16; i += 32) z[i] = make_uint4(0, 0, 0, 0);
    }
    __syncwarp();

    // ------------------------------------------------------------ softmax + p~ digits (per class)
    float lsum = 0.0f, bv = 0.0f;
    if (hv) {
        for (int c = 0; c < 4; ++c) {
            const int s0 = sb[c], s1 = sb[c] + h.r[c];
            const float sg = c == 0 ? psig[0] : c == 1 ? psig[1] : psig[2];
            for (int s = s0 + tl; s < s1; s += TS) {
                const float p = __expf(lgs[hl * LS + s] - mx);
                lsum += p;
                const int li = s - s0;
                if (c < 3) {
                    const float2 vp = vparam[s];
                    bv = fmaf(p, vp.y, bv);
                    const int N = __float2int_rn(p * vp.x * sg);
                    const int ks = vksb[c] + (li >> 5);
                    uint8_t* base = dig + ((ks * 2 * NT + 2 * (hl >> 2)) * 8 + 2 * (hl & 3)) * 32 + (li & 31);
                    base[0] = (uint8_t)(N >> 16);          // tile 2nt,   column 2(h%4)   : hi
                    base[32] = (uint8_t)((N >> 8) & 255);  // tile 2nt,   column 2(h%4)+1 : mid
                    base[8 * 32] = (uint8_t)(N & 255);     // tile 2nt+1, column 2(h%4)   : lo
                } else if (li < prm.max_r16) {
                    p16[hl * prm.max_r16 + li] = p;
                }
            }
        }
        for (int i = tl; i < nzc; i += TS) {
            const float p = __expf(zl[hl * prm.zc_cap + i] - mx);
            zl[hl * prm.zc_cap + i] = p;
            lsum += p;
        }
    }
    lsum = hred_sum(lsum);
    bv = hred_sum(bv);
    __syncwarp();

    // ------------------------------------------------------------ PV (tensor cores)
    // row r of channel m-tile mt is channel 16*mt + r for every V class; the
    // accumulators reuse the logit area: acc [G4][kD]
    float* acc_s = lgs;
    first = true;
    for (int c = 0; c < 3; ++c) {
        if (h.r[c] == 0) continue;
        const int nv = vksb[c + 1] - vksb[c];
        const float vinv = sh.vinv[c][0];
        const int bits = 2 << c;
        const int rb = kD * bits / 8;  // packed bytes per V row (multiple of 32 at d=128)
        const uint8_t* vbase = t + h.off_vseg[c];
        int m0, m1, shf;
        if (c == 0) {
            m0 = gid >> 2;
            m1 = m0 + 2;
            shf = 2 * (gid & 3);
        } else if (c == 1) {
            m0 = gid >> 1;
            m1 = m0 + 4;
            shf = 4 * (gid & 1);
        } else {
            m0 = gid;
            m1 = gid + 8;
            shf = 0;
        }
        const uint32_t mask = c == 0 ? 0x03030303u : c == 1 ? 0x0F0F0F0Fu : 0xFFFFFFFFu;
        const int mstep = 2 * bits;  // byte columns per 16-channel m-tile
        const int swz = 8 * tig;     // vswz: token groups kk*8+tig and +4 have (G & 3) == tig
        for (int mt = 0; mt < kD / 16; mt += 2) {
            int acc[2][2 * NT][4];
#pragma unroll
            for (int u = 0; u < 2; ++u)
#pragma unroll
                for (int nt = 0; nt < 2 * NT; ++nt) acc[u][nt][0] = acc[u][nt][1] = acc[u][nt][2] = acc[u][nt][3] = 0;
            for (int kk = 0; kk < nv; ++kk) {
                const uint8_t* g0 = vbase + (size_t)(kk * 8 + tig) * 4 * rb;
                const uint8_t* g1 = g0 + (size_t)16 * rb;  // token group + 4
                const uint8_t* bb = dig + ((vksb[c] + kk) * 2 * NT * 8 + gid) * 32 + 4 * tig;
                uint32_t bq[2 * NT][2];
#pragma unroll
                for (int nt = 0; nt < 2 * NT; ++nt) {
                    bq[nt][0] = lds32(bb + nt * 256);
                    bq[nt][1] = lds32(bb + nt * 256 + 16);
                }
#pragma unroll
                for (int u = 0; u < 2; ++u) {
                    const int col0 = (((mt + u) * mstep + m0) ^ swz) * 4;
                    const int col1 = (((mt + u) * mstep + m1) ^ swz) * 4;
                    uint32_t a[4];
                    a[0] = (lds32(g0 + col0) >> shf) & mask;
                    a[1] = (lds32(g0 + col1) >> shf) & mask;
                    a[2] = (lds32(g1 + col0) >> shf) & mask;
                    a[3] = (lds32(g1 + col1) >> shf) & mask;
#pragma unroll
                    for (int nt = 0; nt < 2 * NT; ++nt) mma_u8u8(acc[u][nt], a, bq[nt][0], bq[nt][1]);
                }
            }
#pragma unroll
            for (int u = 0; u < 2; ++u)
#pragma unroll
                for (int nt = 0; nt < NT; ++nt) {
                    const int* A = acc[u][2 * nt];
                    const int* B = acc[u][2 * nt + 1];
                    float* row = acc_s + (nt * 4 + tig) * kD + 16 * (mt + u) + gid;
                    const float v0 = fmaf((float)A[0], 65536.0f, fmaf((float)A[1], 256.0f, (float)B[0])) * vinv;
                    const float v1 = fmaf((float)A[2], 65536.0f, fmaf((float)A[3], 256.0f, (float)B[2])) * vinv;
                    row[0] = first ? v0 : row[0] + v0;
                    row[8] = first ? v1 : row[8] + v1;
                }
        }
        first = false;
        __syncwarp();
    }
    if (first) {  // no quantised V rows (Zone B / Zone C only)
        for (int i = lane; i < G4 * kD / 4; i += 32) reinterpret_cast<float4*>(acc_s)[i] = make_float4(0, 0, 0, 0);
        __syncwarp();
    }

    // ------------------------------------------------------------ Zone B / C rows + output
    // lane owns channels 4*lane .. 4*lane+3 of every head
    const int r16 = h.r[3];
    const __half* zb = reinterpret_cast<const __half*>(t + h.off_vseg[3]);
#pragma unroll
    for (int hh = 0; hh < G4; ++hh) {
        if (hh >= g) continue;
        float4 o = reinterpret_cast<const float4*>(acc_s + hh * kD)[lane];
        for (int li = 0; li < r16 + nzc; ++li) {
            const __half* row = li < r16 ? zb + (size_t)li * kD : zcv + (size_t)(li - r16) * kD;
            const float p = li < r16 ? p16[hh * prm.max_r16 + li] : zl[hh * prm.zc_cap + (li - r16)];
            const uint2 raw = *reinterpret_cast<const uint2*>(row + 4 * lane);
            const __half2* hp = reinterpret_cast<const __half2*>(&raw);
            const float2 v01 = __half22float2(hp[0]), v23 = __half22float2(hp[1]);
            o.x = fmaf(p, v01.x, o.x);
            o.y = fmaf(p, v01.y, o.y);
            o.z = fmaf(p, v23.x, o.z);
            o.w = fmaf(p, v23.y, o.w);
        }
        const float ls = __shfl_sync(0xffffffffu, lsum, hh);
        const float b = __shfl_sync(0xffffffffu, bv, hh);
        if constexpr (PART) {
            const float mh = __shfl_sync(0xffffffffu, mx, hh);
            float* pr = part + hh * kPartStride;
            reinterpret_cast<float4*>(pr)[lane] = make_float4(o.x + b, o.y + b, o.z + b, o.w + b);
            if (lane == 0) {
                pr[kD] = ls > 0.0f ? mh : -INFINITY;
                pr[kD + 1] = ls;
            }
            continue;
        }
        const float inv = __frcp_rn(ls);
        const float r0 = (o.x + b) * inv, r1 = (o.y + b) * inv, r2 = (o.z + b) * inv, r3 = (o.w + b) * inv;
        if constexpr (sizeof(IO) == 2) {
            __half2 h0 = __floats2half2_rn(r0, r1), h1 = __floats2half2_rn(r2, r3);
            uint2 st;
            st.x = *reinterpret_cast<uint32_t*>(&h0);
            st.y = *reinterpret_cast<uint32_t*>(&h1);
            reinterpret_cast<uint2*>(out + hh * kD)[lane] = st;
        } else {
            reinterpret_cast<float4*>(out + hh * kD)[lane] = make_float4(r0, r1, r2, r3);
        }
    }
}

// ---------------------------------------------------------------------------
// Uniform 2-bit tiles: every kept V row and every K channel at 2 bits, no
// Zone B / k16 / Zone C (the n=128 production shape). Same math as
// decode_tile with the class logic folded away, the PV fragments built from
// shared words (one 32-bit word feeds rows gid and gid+8) and the B operands
// fetched with ldmatrix.
constexpr int kU2MaxSlots = 160;

__device__ __forceinline__ void ldsm_x4(uint32_t (&r)[4], const void* p) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
                 : "r"(smem_u32(p)));
}

template <typename IO>
__device__ __noinline__ void decode_tile_u2(const uint8_t* __restrict__ t, const IO* __restrict__ qs, int g,
                                            uint8_t* __restrict__ scr, const MmaParams& prm,
                                            IO* __restrict__ out) {
    const int lane = threadIdx.x & 31;
    const int gid = lane >> 2, tig = lane & 3;
    const int hl = lane & 3, tl = lane >> 2;  // per-head phases: head hl, tokens tl + 8i
    const bool hv = hl < g;
    const TileHeader& h = *reinterpret_cast<const TileHeader*>(t);
    uint8_t* dig = scr + kDigitBytesOff;
    const int LS = prm.lg_stride;
    float* lgs = reinterpret_cast<float*>(scr + prm.off_lg);
    const float2* chan = reinterpret_cast<const float2*>(t + kHeaderBytes);
    const uint16_t* perm = reinterpret_cast<const uint16_t*>(t + kHeaderBytes + 8 * h.kslots);
    const float2* vparam = reinterpret_cast<const float2*>(t + h.off_vp);
    const uint8_t* krows = t + h.off_k;
    const uint8_t* vbase = t + h.off_vseg[0];
    const int n = h.r[0];
    const int nslot = pad4(n);
    const int c0 = h.c[0];
    const int nk = (c0 + 31) >> 5;
    const int kslots = h.kslots;
    const int krb = h.krow_bytes;
    const float inv_sqrt_d = 0.08838834764831845f;  // 1/sqrt(128)

    // ------------------------------------------------------------ q statistics
    float qm = 0.0f, bias = 0.0f, sm = 0.0f;
    if (hv) {
#pragma unroll
        for (int i = 0; i < kD / 8; ++i) qm = fmaxf(qm, fabsf(ld_io(qs, hl * kD + tl + 8 * i)));
        for (int s = tl; s < kslots; s += 8) bias = fmaf(ld_io(qs, hl * kD + perm[s]), chan[s].y, bias);
    }
    for (int j = lane; j < c0; j += 32) sm = fmaxf(sm, fabsf(chan[j].x));
#pragma unroll
    for (int o = 4; o < 32; o <<= 1) {
        qm = fmaxf(qm, __shfl_xor_sync(0xffffffffu, qm, o));
        bias += __shfl_xor_sync(0xffffffffu, bias, o);
    }
    sm = warp_max(sm);
    const float bnd = sm * qm;
    const float sg = bnd > 0.0f ? 8.2e6f * __frcp_rn(bnd) : 0.0f;
    const float qinv_own = bnd * (1.0f / 8.2e6f);  // for head hl; QK needs head tig == hl
    // ------------------------------------------------------------ q~ digits
    // task (k-step kk, K positions 4*tl .. 4*tl+3, head hl): slot 16*(tl>>2) + 4e + (tl&3)
    for (int kk = 0; kk < nk; ++kk) {
        uint32_t x[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const int j = kk * 32 + 16 * (tl >> 2) + 4 * e + (tl & 3);
            int N = 0;
            if (hv && j < c0) N = __float2int_rn(chan[j].x * ld_io(qs, hl * kD + perm[j]) * sg);
            x[e] = (uint32_t)(N + 0x808080) ^ 0x808080u;
        }
        const uint32_t wlo = __byte_perm(__byte_perm(x[0], x[1], 0x0040), __byte_perm(x[2], x[3], 0x0040), 0x5410);
        const uint32_t wmid = __byte_perm(__byte_perm(x[0], x[1], 0x0051), __byte_perm(x[2], x[3], 0x0051), 0x5410);
        const uint32_t whi = __byte_perm(__byte_perm(x[0], x[1], 0x0062), __byte_perm(x[2], x[3], 0x0062), 0x5410);
        uint8_t* a0 = dig + ((kk * 2) * 8 + 2 * hl) * 32 + 4 * tl;
        *reinterpret_cast<uint32_t*>(a0) = whi;
        *reinterpret_cast<uint32_t*>(a0 + 32) = wmid;
        *reinterpret_cast<uint32_t*>(a0 + 8 * 32) = wlo;
        *reinterpret_cast<uint32_t*>(a0 + 8 * 32 + 32) = 0u;
    }
    __syncwarp();

    // ------------------------------------------------------------ QK (tensor cores)
    uint32_t bq[4][4];  // per k-step: n-tile 0 (b0, b1), n-tile 1 (b0, b1)
    {
        const int mat = lane >> 3, r = lane & 7;
        const uint8_t* base = dig + (((mat >> 1) * 8 + r) * 32 + (mat & 1) * 16);
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {
            if (kk < nk) {
                ldsm_x4(bq[kk], base + kk * 2 * 8 * 32);
            } else {
                bq[kk][0] = bq[kk][1] = bq[kk][2] = bq[kk][3] = 0u;
            }
        }
    }
    const float qinv = __shfl_sync(0xffffffffu, qinv_own, tig);  // lane tig has hl == tig
    const int mtiles = (nslot + 15) >> 4;
    for (int mt = 0; mt < mtiles; mt += 2) {
        const bool two = mt + 1 < mtiles;
        int acc[2][2][4];
#pragma unroll
        for (int u = 0; u < 2; ++u)
#pragma unroll
            for (int nt = 0; nt < 2; ++nt) acc[u][nt][0] = acc[u][nt][1] = acc[u][nt][2] = acc[u][nt][3] = 0;
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {
            if (kk < nk) {
#pragma unroll
                for (int u = 0; u < 2; ++u) {
                    if (u == 1 && !two) continue;
                    const uint8_t* p0 = krows + (size_t)krow_pos(h, (mt + u) * 16 + gid) * krb + 8 * kk;
                    const uint8_t* p1 = krows + (size_t)krow_pos(h, (mt + u) * 16 + gid + 8) * krb + 8 * kk;
                    const uint2 w0 = lds64(p0), w1 = lds64(p1);
                    const int s = 2 * tig;
                    uint32_t a[4];
                    a[0] = (w0.x >> s) & 0x03030303u;
                    a[2] = (w0.y >> s) & 0x03030303u;
                    a[1] = (w1.x >> s) & 0x03030303u;
                    a[3] = (w1.y >> s) & 0x03030303u;
                    mma_u8s8(acc[u][0], a, bq[kk][0], bq[kk][1]);
                    mma_u8s8(acc[u][1], a, bq[kk][2], bq[kk][3]);
                }
            }
        }
#pragma unroll
        for (int u = 0; u < 2; ++u) {
            if (u == 1 && !two) continue;
            float* row = lgs + tig * LS + (mt + u) * 16 + gid;
            row[0] = fmaf((float)acc[u][0][0], 65536.0f, fmaf((float)acc[u][0][1], 256.0f, (float)acc[u][1][0])) * qinv;
            row[8] = fmaf((float)acc[u][0][2], 65536.0f, fmaf((float)acc[u][0][3], 256.0f, (float)acc[u][1][2])) * qinv;
        }
    }
    __syncwarp();

    // ------------------------------------------------------------ logits + max
    float mx = -INFINITY, vsm = 0.0f;
    for (int s = tl; s < n; s += 8) {
        vsm = fmaxf(vsm, vparam[s].x);
        if (hv) {
            const float v = (lgs[hl * LS + s] + bias) * inv_sqrt_d;
            lgs[hl * LS + s] = v;
            mx = fmaxf(mx, v);
        }
    }
#pragma unroll
    for (int o = 4; o < 32; o <<= 1) {
        mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        vsm = fmaxf(vsm, __shfl_xor_sync(0xffffffffu, vsm, o));
    }
    const float psig = vsm > 0.0f ? 1.6e7f * __frcp_rn(vsm) : 0.0f;
    const float vinv = vsm * (1.0f / 1.6e7f);
    const int nv = (nslot + 31) >> 5;
    {
        uint4* z = reinterpret_cast<uint4*>(dig);
        for (int i = lane; i < nv * 2 * 8 * 32 / 16; i += 32) z[i] = make_uint4(0, 0, 0, 0);
    }
    __syncwarp();

    // ------------------------------------------------------------ softmax + p~ digits
    float lsum = 0.0f, bv = 0.0f;
    if (hv) {
        for (int s = tl; s < n; s += 8) {
            const float p = __expf(lgs[hl * LS + s] - mx);
            lsum += p;
            const float2 vp = vparam[s];
            bv = fmaf(p, vp.y, bv);
            const int N = __float2int_rn(p * vp.x * psig);
            uint8_t* base = dig + (((s >> 5) * 2) * 8 + 2 * hl) * 32 + (s & 31);
            base[0] = (uint8_t)(N >> 16);
            base[32] = (uint8_t)((N >> 8) & 255);
            base[8 * 32] = (uint8_t)(N & 255);
        }
    }
#pragma unroll
    for (int o = 4; o < 32; o <<= 1) {
        lsum += __shfl_xor_sync(0xffffffffu, lsum, o);
        bv += __shfl_xor_sync(0xffffffffu, bv, o);
    }
    __syncwarp();

    // ------------------------------------------------------------ PV (tensor cores)
    // m-tile mt covers byte columns 4mt .. 4mt+3; row gid <-> channel
    // 16mt + 4(gid&3) + (gid>>2), row gid+8 <-> that + 2 (one word feeds both)
    int acc[8][2][4];
#pragma unroll
    for (int mt = 0; mt < 8; ++mt)
#pragma unroll
        for (int nt = 0; nt < 2; ++nt) acc[mt][nt][0] = acc[mt][nt][1] = acc[mt][nt][2] = acc[mt][nt][3] = 0;
    const int j0 = 2 * (gid >> 2);
    const int swz = 8 * tig;
    const int mat = lane >> 3, rr = lane & 7;
    const uint8_t* bbase = dig + (((mat >> 1) * 8 + rr) * 32 + (mat & 1) * 16);
    for (int kk = 0; kk < nv; ++kk) {
        uint32_t b[4];
        ldsm_x4(b, bbase + kk * 2 * 8 * 32);
        const uint8_t* g0 = vbase + (size_t)(kk * 8 + tig) * 128;  // token group, 4 x 32 B
        const uint8_t* g1 = g0 + 4 * 128;
#pragma unroll
        for (int mt = 0; mt < 8; ++mt) {
            const int col = ((4 * mt + (gid & 3)) ^ swz) * 4;
            const uint32_t w0 = lds32(g0 + col), w1 = lds32(g1 + col);
            uint32_t a[4];
            a[0] = (w0 >> j0) & 0x03030303u;
            a[1] = (w0 >> (j0 + 4)) & 0x03030303u;
            a[2] = (w1 >> j0) & 0x03030303u;
            a[3] = (w1 >> (j0 + 4)) & 0x03030303u;
            mma_u8u8(acc[mt][0], a, b[0], b[1]);
            mma_u8u8(acc[mt][1], a, b[2], b[3]);
        }
    }
    float* acc_s = lgs;  // [4][kD]
#pragma unroll
    for (int mt = 0; mt < 8; ++mt) {
        const int ch = 16 * mt + 4 * (gid & 3) + (gid >> 2);
        float* row = acc_s + tig * kD + ch;
        row[0] = fmaf((float)acc[mt][0][0], 65536.0f, fmaf((float)acc[mt][0][1], 256.0f, (float)acc[mt][1][0])) * vinv;
        row[2] = fmaf((float)acc[mt][0][2], 65536.0f, fmaf((float)acc[mt][0][3], 256.0f, (float)acc[mt][1][2])) * vinv;
    }
    __syncwarp();

    // ------------------------------------------------------------ output (lane owns channels 4*lane..+3)
#pragma unroll
    for (int hh = 0; hh < 4; ++hh) {
        if (hh >= g) continue;
        const float4 o = reinterpret_cast<const float4*>(acc_s + hh * kD)[lane];
        const float inv = __frcp_rn(__shfl_sync(0xffffffffu, lsum, hh));
        const float b = __shfl_sync(0xffffffffu, bv, hh);
        const float r0 = (o.x + b) * inv, r1 = (o.y + b) * inv, r2 = (o.z + b) * inv, r3 = (o.w + b) * inv;
        if constexpr (sizeof(IO) == 2) {
            __half2 h0 = __floats2half2_rn(r0, r1), h1 = __floats2half2_rn(r2, r3);
            uint2 st;
            st.x = *reinterpret_cast<uint32_t*>(&h0);
            st.y = *reinterpret_cast<uint32_t*>(&h1);
            reinterpret_cast<uint2*>(out + hh * kD)[lane] = st;
        } else {
            reinterpret_cast<float4*>(out + hh * kD)[lane] = make_float4(r0, r1, r2, r3);
        }
    }
}

template <int NT, typename IO, bool U2>
__global__ void __launch_bounds__(32 * (kMaxW + 1), 1) decode_mma_kernel(const MmaParams p) {
    extern __shared__ __align__(128) uint8_t dsm[];
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    uint64_t* full = reinterpret_cast<uint64_t*>(dsm);
    uint64_t* empty = full + kMaxR;
    uint8_t* ring = dsm + 2 * kMaxR * sizeof(uint64_t);  // 512 B, 128-aligned
    uint8_t* scratch0 = ring + (size_t)p.R * p.slot_bytes;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int qbytes = p.g * kD * (int)sizeof(IO);
    if (threadIdx.x == 0) {
        for (int s = 0; s < p.R; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        fence_barrier_init();
    }
    __syncthreads();
    const int ntiles = p.units > (int)blockIdx.x ? (p.units - 1 - (int)blockIdx.x) / (int)gridDim.x + 1 : 0;
    if (warp == 0) {
        // ---- producer: stage tile j of this CTA into slot j % R
        for (int base = 0; base < ntiles; base += 32) {
            const int mj = base + lane;
            int64_t moff = 0;
            int msz = 0;
            int munit = 0;
            if (mj < ntiles) {
                const int tile = blockIdx.x + mj * gridDim.x;
                munit = unit_of(p, tile);
                moff = p.offsets[munit];
                msz = p.dsize[munit];
            }
            const int cnt = min(32, ntiles - base);
            for (int k = 0; k < cnt; ++k) {
                const int64_t off = __shfl_sync(0xffffffffu, moff, k);
                const int sz = __shfl_sync(0xffffffffu, msz, k);
                const int unit = __shfl_sync(0xffffffffu, munit, k);
                if (lane == 0) {
                    const int j = base + k;
                    const int slot = j % p.R, use = j / p.R;
                    if (use > 0) mbar_wait(&empty[slot], (uint32_t)((use - 1) & 1));
                    fence_proxy_async();
                    uint8_t* dst = ring + (size_t)slot * p.slot_bytes;
                    mbar_expect_tx(&full[slot], (uint32_t)(sz + qbytes));
                    bulk_g2s(dst, p.arena + off, (uint32_t)sz, &full[slot]);
                    bulk_g2s(dst + p.slot_bytes - qbytes,
                             static_cast<const uint8_t*>(p.q) + (size_t)unit * qbytes, (uint32_t)qbytes, &full[slot]);
                }
                __syncwarp();
            }
        }
        return;
    }
    // ---- consumers
    const int cw = warp - 1;
    uint8_t* scr = scratch0 + (size_t)cw * p.scratch_bytes;
    for (int j = cw; j < ntiles; j += p.W) {
        const int slot = j % p.R, use = j / p.R;
        mbar_wait(&full[slot], (uint32_t)(use & 1));
        const uint8_t* st = ring + (size_t)slot * p.slot_bytes;
        const int tile = unit_of(p, blockIdx.x + j * gridDim.x);  // the unit this tile belongs to
        const IO* qs = reinterpret_cast<const IO*>(st + p.slot_bytes - qbytes);
        const int nzc = p.zc_len ? min(p.zc_len[tile], p.zc_cap) : 0;
        if constexpr (U2) {
            decode_tile_u2<IO>(st, qs, p.g, scr, p, static_cast<IO*>(p.out) + (size_t)tile * p.g * kD);
        } else {
            decode_tile<NT, IO>(st, qs, p.g, scr, p,
                                p.zc_k ? p.zc_k + (size_t)tile * p.zc_cap * kD : nullptr,
                                p.zc_v ? p.zc_v + (size_t)tile * p.zc_cap * kD : nullptr, nzc,
                                static_cast<IO*>(p.out) + (size_t)tile * p.g * kD);
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[slot]);
    }
}

// ---------------------------------------------------------------------------
// Uniform 2-bit tiles decoded by a PAIR of warps: the two warps split the
// q~ digit k-steps, the 32-token blocks of QK / softmax and the PV channel
// m-tiles, and meet at three named barriers per tile. Half the registers and
// half the dependency chain of the one-warp body, so twice the warps fit.
constexpr int kPairs = 11;  // consumer warp pairs per CTA (22 warps + producer)

__device__ __forceinline__ void pair_sync(int id) {
    asm volatile("bar.sync %0, 64;" ::"r"(id) : "memory");
}

struct PairXchg {   // per pair, at the head of the pair's scratch
    float bias[2][4];
    float mx[2][4], vsm[2];
    float lsum[2][4], bv[2][4];
};
static_assert(sizeof(PairXchg) <= kDigitBytesOff, "exchange area fits before the digits");

template <typename IO>
__device__ __forceinline__ void decode_tile_u2_pair(const uint8_t* __restrict__ t, const IO* __restrict__ qs,
                                                    int g, uint8_t* __restrict__ scr, const MmaParams& prm,
                                                    IO* __restrict__ out, int half, int bar) {
    // fragment layout: lane (gid, tig); tig is also the GQA head of every
    // per-head value this lane holds (C columns 2*tig, 2*tig+1 = head tig)
    const int lane = threadIdx.x & 31;
    const int gid = lane >> 2, tig = lane & 3;
    const bool hv = tig < g;
    const TileHeader& h = *reinterpret_cast<const TileHeader*>(t);
    PairXchg& xg = *reinterpret_cast<PairXchg*>(scr);
    uint8_t* dig = scr + kDigitBytesOff;
    const float2* chan = reinterpret_cast<const float2*>(t + kHeaderBytes);
    const uint16_t* perm = reinterpret_cast<const uint16_t*>(t + kHeaderBytes + 8 * h.kslots);
    const float2* vparam = reinterpret_cast<const float2*>(t + h.off_vp);
    const uint8_t* krows = t + h.off_k;
    const uint8_t* vbase = t + h.off_vseg[0];
    const int n = h.r[0];
    const int nslot = pad4(n);
    const int c0 = h.c[0];
    const bool full_k = c0 == kD;  // every channel at 2 bits: channel_perm is the identity
    const int nk = (c0 + 31) >> 5;
    const int krb = h.krow_bytes;
    const float inv_sqrt_d = 0.08838834764831845f;  // 1/sqrt(128)
    const IO* qh = qs + tig * kD;

    // ------------------------------------------------------------ q statistics (both warps, redundant)
    float qm = 0.0f, sm = 0.0f;
    if (hv) {
#pragma unroll
        for (int i = 0; i < kD / 8; ++i) qm = fmaxf(qm, fabsf(ld_io(qh, 16 * (i >> 1) + 2 * gid + (i & 1))));
    }
    for (int j = lane; j < c0; j += 32) sm = fmaxf(sm, fabsf(chan[j].x));
#pragma unroll
    for (int o = 4; o < 32; o <<= 1) qm = fmaxf(qm, __shfl_xor_sync(0xffffffffu, qm, o));
    sm = warp_max(sm);
    const float bnd = sm * qm;
    const float sg = bnd > 0.0f ? 8.2e6f * __frcp_rn(bnd) : 0.0f;

    // ------------------------------------------------------------ q~ digits + bias (k-steps half, half+2)
    // K position p = 4*gid + e of a k-step is read by A-lane tig(p) = gid & 3,
    // whose codes enter the MMA masked in place, i.e. scaled by 4^tig(p); the
    // fixed point N is pre-scaled by 4^(3 - tig(p)) so every product carries
    // 4^3 = 64, and split into four signed bytes (n-tile 0: d3 d2, n-tile 1: d1 d0).
    float bpart = 0.0f;
    const int pshift = 2 * (3 - (gid & 3));
    for (int kk = half; kk < nk; kk += 2) {
        uint32_t x[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const int j = kk * 32 + 16 * (gid >> 2) + 4 * e + (gid & 3);
            int N = 0;
            if (hv && j < c0) {
                const float2 cs = chan[j];
                const float qv = ld_io(qh, full_k ? j : perm[j]);
                bpart = fmaf(qv, cs.y, bpart);
                N = __float2int_rn(cs.x * qv * sg);
            }
            x[e] = ((uint32_t)N << pshift) + 0x80808080u ^ 0x80808080u;
        }
        const uint32_t w0 = __byte_perm(__byte_perm(x[0], x[1], 0x0040), __byte_perm(x[2], x[3], 0x0040), 0x5410);
        const uint32_t w1 = __byte_perm(__byte_perm(x[0], x[1], 0x0051), __byte_perm(x[2], x[3], 0x0051), 0x5410);
        const uint32_t w2 = __byte_perm(__byte_perm(x[0], x[1], 0x0062), __byte_perm(x[2], x[3], 0x0062), 0x5410);
        const uint32_t w3 = __byte_perm(__byte_perm(x[0], x[1], 0x0073), __byte_perm(x[2], x[3], 0x0073), 0x5410);
        uint8_t* a0 = dig + ((kk * 2) * 8 + 2 * tig) * 32 + 4 * gid;
        *reinterpret_cast<uint32_t*>(a0) = w3;
        *reinterpret_cast<uint32_t*>(a0 + 32) = w2;
        *reinterpret_cast<uint32_t*>(a0 + 8 * 32) = w1;
        *reinterpret_cast<uint32_t*>(a0 + 8 * 32 + 32) = w0;
    }
#pragma unroll
    for (int o = 4; o < 32; o <<= 1) bpart += __shfl_xor_sync(0xffffffffu, bpart, o);
    if (gid == 0) xg.bias[half][tig] = bpart;
    pair_sync(bar);  // digits + bias halves visible
    const float bias_s = (xg.bias[0][tig] + xg.bias[1][tig]) * inv_sqrt_d;
    // logit = (v / (64 sigma) + bias) / sqrt(d), v = sum code * 4^tig * N * 4^(3-tig)
    const float qscale = bnd * (1.0f / (64.0f * 8.2e6f)) * inv_sqrt_d;

    // ------------------------------------------------------------ QK: m-tile pairs half, half+2, ... (32 tokens each)
    const int mat = lane >> 3, rr = lane & 7;
    const uint8_t* bbase = dig + (((mat >> 1) * 8 + rr) * 32 + (mat & 1) * 16);
    uint32_t bq[4][4];
#pragma unroll
    for (int kk = 0; kk < 4; ++kk) {
        if (kk < nk) {
            ldsm_x4(bq[kk], bbase + kk * 2 * 8 * 32);
        } else {
            bq[kk][0] = bq[kk][1] = bq[kk][2] = bq[kk][3] = 0u;
        }
    }
    const uint32_t kmask = 0x03030303u << (2 * tig);
    constexpr int kPM = (kU2MaxSlots / 32 + 1) / 2;  // pairs per warp (3 for 160 slots)
    const int npair = (nslot + 31) >> 5;
    float lg[kPM][2][2];  // [pair][m-tile][row half]: token 32*pb + 16*u + gid + 8*r
    float mx = -INFINITY;
#pragma unroll
    for (int i = 0; i < kPM; ++i) {
        const int pb = half + 2 * i;
        if (pb >= npair) {
            lg[i][0][0] = lg[i][0][1] = lg[i][1][0] = lg[i][1][1] = -INFINITY;
            continue;
        }
        int acc[2][2][4];
#pragma unroll
        for (int u = 0; u < 2; ++u)
#pragma unroll
            for (int nt = 0; nt < 2; ++nt) acc[u][nt][0] = acc[u][nt][1] = acc[u][nt][2] = acc[u][nt][3] = 0;
#pragma unroll
        for (int u = 0; u < 2; ++u) {
            const uint8_t* r0 = krows + (size_t)krow_pos(h, 32 * pb + 16 * u + gid) * krb;
            const uint8_t* r1 = krows + (size_t)krow_pos(h, 32 * pb + 16 * u + gid + 8) * krb;
            uint32_t w0[8], w1[8];  // the 32 K bytes (128 codes) of rows gid and gid + 8
            if (krb == 32) {
                const uint4 x0 = *reinterpret_cast<const uint4*>(r0), x1 = *reinterpret_cast<const uint4*>(r0 + 16);
                const uint4 y0 = *reinterpret_cast<const uint4*>(r1), y1 = *reinterpret_cast<const uint4*>(r1 + 16);
                w0[0] = x0.x; w0[1] = x0.y; w0[2] = x0.z; w0[3] = x0.w; w0[4] = x1.x; w0[5] = x1.y; w0[6] = x1.z; w0[7] = x1.w;
                w1[0] = y0.x; w1[1] = y0.y; w1[2] = y0.z; w1[3] = y0.w; w1[4] = y1.x; w1[5] = y1.y; w1[6] = y1.z; w1[7] = y1.w;
            } else {
#pragma unroll
                for (int kk = 0; kk < 4; ++kk) {
                    const uint2 a = kk < nk ? lds64(r0 + 8 * kk) : make_uint2(0, 0);
                    const uint2 b = kk < nk ? lds64(r1 + 8 * kk) : make_uint2(0, 0);
                    w0[2 * kk] = a.x; w0[2 * kk + 1] = a.y; w1[2 * kk] = b.x; w1[2 * kk + 1] = b.y;
                }
            }
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) {
                if (kk < nk) {
                    uint32_t a[4];
                    a[0] = w0[2 * kk] & kmask;
                    a[2] = w0[2 * kk + 1] & kmask;
                    a[1] = w1[2 * kk] & kmask;
                    a[3] = w1[2 * kk + 1] & kmask;
                    mma_u8s8(acc[u][0], a, bq[kk][0], bq[kk][1]);
                    mma_u8s8(acc[u][1], a, bq[kk][2], bq[kk][3]);
                }
            }
        }
#pragma unroll
        for (int u = 0; u < 2; ++u)
#pragma unroll
            for (int r = 0; r < 2; ++r) {
                const int s = 32 * pb + 16 * u + gid + 8 * r;
                const float v = fmaf(fmaf(fmaf((float)acc[u][0][2 * r], 256.0f, (float)acc[u][0][2 * r + 1]), 256.0f,
                                          (float)acc[u][1][2 * r]),
                                     256.0f, (float)acc[u][1][2 * r + 1]);
                const float l = (s < n && hv) ? fmaf(v, qscale, bias_s) : -INFINITY;
                lg[i][u][r] = l;
                mx = fmaxf(mx, l);
            }
    }
    // V-scale bound over this warp's tokens (p~ = p * vscale <= vscale)
    float vsm = 0.0f;
    for (int pb = half; pb < npair; pb += 2) {
        const int s = 32 * pb + lane;
        if (s < n) vsm = fmaxf(vsm, vparam[s].x);
    }
#pragma unroll
    for (int o = 4; o < 32; o <<= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    vsm = warp_max(vsm);
    if (gid == 0) xg.mx[half][tig] = mx;
    if (lane == 0) xg.vsm[half] = vsm;
    pair_sync(bar);  // also: both warps are done reading the q~ digits
    mx = fmaxf(xg.mx[0][tig], xg.mx[1][tig]);
    vsm = fmaxf(xg.vsm[0], xg.vsm[1]);
    const float psig = vsm > 0.0f ? 1.6e7f * __frcp_rn(vsm) : 0.0f;
    const float vinv = vsm * (1.0f / 1.6e7f);
    const int nv = npair;  // token k-steps == 32-token blocks
    for (int pb = half; pb < nv; pb += 2) reinterpret_cast<uint4*>(dig + pb * 2 * 8 * 32)[lane] = make_uint4(0, 0, 0, 0);
    __syncwarp();

    // ------------------------------------------------------------ softmax + p~ digits, in registers
    float lsum = 0.0f, bv = 0.0f;
#pragma unroll
    for (int i = 0; i < kPM; ++i) {
        const int pb = half + 2 * i;
        if (pb >= npair) continue;
#pragma unroll
        for (int u = 0; u < 2; ++u)
#pragma unroll
            for (int r = 0; r < 2; ++r) {
                const float l = lg[i][u][r];
                if (l == -INFINITY) continue;
                const int s = 32 * pb + 16 * u + gid + 8 * r;
                const float p = __expf(l - mx);
                lsum += p;
                const float2 vp = vparam[s];
                bv = fmaf(p, vp.y, bv);
                const int N = __float2int_rn(p * vp.x * psig);
                uint8_t* base = dig + ((pb * 2) * 8 + 2 * tig) * 32 + (s & 31);
                base[0] = (uint8_t)(N >> 16);
                base[32] = (uint8_t)((N >> 8) & 255);
                base[8 * 32] = (uint8_t)(N & 255);
            }
    }
#pragma unroll
    for (int o = 4; o < 32; o <<= 1) {
        lsum += __shfl_xor_sync(0xffffffffu, lsum, o);
        bv += __shfl_xor_sync(0xffffffffu, bv, o);
    }
    if (gid == 0) {
        xg.lsum[half][tig] = lsum;
        xg.bv[half][tig] = bv;
    }
    pair_sync(bar);  // p~ digits of both warps + totals visible
    const float lt = xg.lsum[0][tig] + xg.lsum[1][tig];
    const float bt = xg.bv[0][tig] + xg.bv[1][tig];

    // ------------------------------------------------------------ PV: 4 m-tiles per warp, codes masked in place
    // byte column c = 16*half + 4*(gid&3) + m (m = 0..3, one LDS.128 per token group);
    // row gid <-> channel 4c + jj, row gid+8 <-> 4c + jj + 2, jj = gid >> 2; the
    // in-place mask scales those rows by 4^jj and 4^(jj+2)
    int acc[4][2][4];
#pragma unroll
    for (int m = 0; m < 4; ++m)
#pragma unroll
        for (int nt = 0; nt < 2; ++nt) acc[m][nt][0] = acc[m][nt][1] = acc[m][nt][2] = acc[m][nt][3] = 0;
    const int jj = gid >> 2;
    const uint32_t vm0 = 0x03030303u << (2 * jj), vm1 = 0x03030303u << (2 * jj + 4);
    const int colb = ((16 * half + 4 * (gid & 3)) ^ (8 * tig)) * 4;  // vswz: (G & 3) == tig
    const uint8_t* g0b = vbase + (size_t)tig * 128 + colb;
    for (int kk = 0; kk < nv; ++kk) {
        uint32_t b[4];
        ldsm_x4(b, bbase + kk * 2 * 8 * 32);
        const uint4 x0 = *reinterpret_cast<const uint4*>(g0b + (size_t)kk * 8 * 128);        // group kk*8 + tig
        const uint4 x1 = *reinterpret_cast<const uint4*>(g0b + (size_t)kk * 8 * 128 + 512);  // group + 4
        const uint32_t u0[4] = {x0.x, x0.y, x0.z, x0.w}, u1[4] = {x1.x, x1.y, x1.z, x1.w};
#pragma unroll
        for (int m = 0; m < 4; ++m) {
            uint32_t a[4];
            a[0] = u0[m] & vm0;
            a[1] = u0[m] & vm1;
            a[2] = u1[m] & vm0;
            a[3] = u1[m] & vm1;
            mma_u8u8(acc[m][0], a, b[0], b[1]);
            mma_u8u8(acc[m][1], a, b[2], b[3]);
        }
    }
    // output straight from the fragments: head tig, channels 4c + jj and 4c + jj + 2
    if (hv) {
        const float inv = __frcp_rn(lt);
        const float s0 = vinv * (jj ? 0.25f : 1.0f), s1 = s0 * 0.0625f;
        IO* orow = out + tig * kD;
#pragma unroll
        for (int m = 0; m < 4; ++m) {
            const int ch = 4 * (16 * half + 4 * (gid & 3) + m) + jj;
            const float v0 = fmaf((float)acc[m][0][0], 65536.0f, fmaf((float)acc[m][0][1], 256.0f, (float)acc[m][1][0]));
            const float v1 = fmaf((float)acc[m][0][2], 65536.0f, fmaf((float)acc[m][0][3], 256.0f, (float)acc[m][1][2]));
            const float r0 = fmaf(v0, s0, bt) * inv, r1 = fmaf(v1, s1, bt) * inv;
            if constexpr (sizeof(IO) == 2) {
                orow[ch] = __float2half_rn(r0);
                orow[ch + 2] = __float2half_rn(r1);
            } else {
                orow[ch] = r0;
                orow[ch + 2] = r1;
            }
        }
    }
}

template <typename IO>
__global__ void __launch_bounds__(32 * (2 * kPairs + 1), 1) decode_u2_pair_kernel(const MmaParams p) {
    extern __shared__ __align__(128) uint8_t dsm[];
    uint64_t* full = reinterpret_cast<uint64_t*>(dsm);
    uint64_t* empty = full + kMaxR;
    uint8_t* ring = dsm + 2 * kMaxR * sizeof(uint64_t);
    uint8_t* scratch0 = ring + (size_t)p.R * p.slot_bytes;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int qbytes = p.g * kD * (int)sizeof(IO);
    const int npairs = p.W;  // W counts pairs for this kernel
    if (threadIdx.x == 0) {
        for (int s = 0; s < p.R; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 2);  // both warps of the pair release the slot
        }
        fence_barrier_init();
    }
    __syncthreads();
    const int ntiles = p.units > (int)blockIdx.x ? (p.units - 1 - (int)blockIdx.x) / (int)gridDim.x + 1 : 0;
    if (warp == 0) {
        for (int base = 0; base < ntiles; base += 32) {
            const int mj = base + lane;
            int64_t moff = 0;
            int msz = 0;
            int munit = 0;
            if (mj < ntiles) {
                const int tile = blockIdx.x + mj * gridDim.x;
                munit = unit_of(p, tile);
                moff = p.offsets[munit];
                msz = p.dsize[munit];
            }
            const int cnt = min(32, ntiles - base);
            for (int k = 0; k < cnt; ++k) {
                const int64_t off = __shfl_sync(0xffffffffu, moff, k);
                const int sz = __shfl_sync(0xffffffffu, msz, k);
                const int unit = __shfl_sync(0xffffffffu, munit, k);
                if (lane == 0) {
                    const int j = base + k;
                    const int slot = j % p.R, use = j / p.R;
                    if (use > 0) mbar_wait(&empty[slot], (uint32_t)((use - 1) & 1));
                    fence_proxy_async();
                    uint8_t* dst = ring + (size_t)slot * p.slot_bytes;
                    mbar_expect_tx(&full[slot], (uint32_t)(sz + qbytes));
                    bulk_g2s(dst, p.arena + off, (uint32_t)sz, &full[slot]);
                    bulk_g2s(dst + p.slot_bytes - qbytes,
                             static_cast<const uint8_t*>(p.q) + (size_t)unit * qbytes, (uint32_t)qbytes, &full[slot]);
                }
                __syncwarp();
            }
        }
        return;
    }
    const int pr = (warp - 1) >> 1, half = (warp - 1) & 1;
    uint8_t* scr = scratch0 + (size_t)pr * p.scratch_bytes;
    int slot = pr % p.R, use = pr / p.R;
    for (int j = pr; j < ntiles; j += npairs) {
        mbar_wait(&full[slot], (uint32_t)(use & 1));
        const uint8_t* st = ring + (size_t)slot * p.slot_bytes;
        const int tile = blockIdx.x + j * gridDim.x;
        const IO* qs = reinterpret_cast<const IO*>(st + p.slot_bytes - qbytes);
        decode_tile_u2_pair<IO>(st, qs, p.g, scr, p, static_cast<IO*>(p.out) + (size_t)tile * p.g * kD, half,
                                1 + pr);
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[slot]);
        slot += npairs;
        while (slot >= p.R) {
            slot -= p.R;
            ++use;
        }
    }
}

template <typename IO>
static int launch_pair(const rdkv_decode_args* a, cudaStream_t st) {
    const int qbytes = a->group * kD * (int)sizeof(IO);
    const int slot = (a->plan.max_decode_bytes + qbytes + 127) & ~127;
    const int nv = (a->plan.max_slots + 31) / 32;
    const int steps = nv > 4 ? nv : 4;
    int scratch = kDigitBytesOff + steps * 2 * 8 * 32;
    const int off_lg = 0, lg_stride = 0;  // softmax stays in registers
    scratch = (scratch + 127) & ~127;
    int dev = 0, smem_max = 0, nsm = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&smem_max, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    const int head = 2 * kMaxR * (int)sizeof(uint64_t);
    const int slack = 4096;
    int W = kPairs, R = 0;
    bool fits = false;
    for (; W >= 1 && !fits; --W) {
        for (int look = 2; look >= 0 && !fits; --look) {
            R = W + look > kMaxR ? kMaxR : W + look;
            fits = head + (size_t)R * slot + (size_t)W * scratch + slack <= (size_t)smem_max;
        }
        if (fits) break;
    }
    if (!fits) return RDKV_EINVAL;
    const size_t smem = head + (size_t)R * slot + (size_t)W * scratch + slack;
    MmaParams p{a->arena, a->tile_offsets, a->tile_decode_bytes, a->q, a->out, nullptr, nullptr, nullptr,
                a->units, a->group, 0, R, W, slot, scratch, off_lg, lg_stride, -1, -1, 0};
    auto kern = decode_u2_pair_kernel<IO>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int blocks = (a->units + W - 1) / W;
    if (blocks > nsm) blocks = nsm;
    kern<<<blocks, 32 * (2 * W + 1), smem, st>>>(p);
    return launch_status();
}

// ============================================================================
// Uniform-2-bit warp-pair body, v3 ("u2x"): the digit arithmetic of
// decode_tile_u2_pair with the instruction count cut for the issue-bound
// regime (~3.6K -> ~1.1K warp instructions per tile):
//   * block loops bounded by compile-time NBMAX (32-token blocks per tile) with
//     warp-uniform guards on the tile's own block count: no ghost blocks;
//     warp `half` owns blocks half, half + 2, ...;
//   * QK A rows <-> token slots 32b + 4*gid + 2u + r, so every lane ends up
//     with four CONSECUTIVE slots per block: their V parameters are two
//     LDS.128 and their p~ digits pack (PRMT) into one 32-bit word per digit;
//     K rows are stored slot-transposed (tile_layout.h krow_pos) so those
//     A-row loads stay conflict-free;
//   * q rows are staged contiguously (one bulk copy) and read in a per-head
//     staggered channel order that is bank-conflict-free; the stagger is undone
//     for free by the runtime selector of the digit-transposing PRMT;
//   * p~ = p * vscale in 16-bit fixed point: two u8 digits, one n-tile, so PV
//     is 4 MMAs per 32 tokens per warp and one integer combine per output
//     (~1e-4 relative decode error, matched to the fp16 output; 24-bit p~
//     costs ~10% of the step);
//   * fixed-point ranges from the header's scale bounds (no per-tile scans);
//   * digit sums combined in integer registers before one I2F pair (QK);
//   * log2(e) folded into the logit scale: p = ex2(l' - m').
constexpr int kXQDig = 256;                 // q~ digits: 4 k-steps x 512 B (2 n-tiles x 8 rows x 32 B)
constexpr int kXPDig = kXQDig + 4 * 512;    // p~ digits: one 256-B block (8 rows x 32 B) per 32 tokens
constexpr int kXNbMax = 5;                  // 32-token blocks per tile on this path (kU2MaxSlots = 160)
constexpr float kPScale = 65280.0f;         // p~ = p * vscale * kPScale / vmax <= 65280 < 2^16

struct PairX {
    float bias[2][4];
    float mx[2][4];
    float lsum[2][4], bv[2][4];
};
static_assert(sizeof(PairX) <= kXQDig, "exchange area");

__device__ __forceinline__ uint4 lds128(const uint8_t* p) { return *reinterpret_cast<const uint4*>(p); }

template <typename IO>
__device__ __forceinline__ float absmax16(const IO* q);
template <>
__device__ __forceinline__ float absmax16<__half>(const __half* q) {
    const uint4 a = *reinterpret_cast<const uint4*>(q), b = *reinterpret_cast<const uint4*>(q + 8);
    const uint32_t w[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
    __half2 m = __habs2(*reinterpret_cast<const __half2*>(&w[0]));
#pragma unroll
    for (int i = 1; i < 8; ++i) m = __hmax2(m, __habs2(*reinterpret_cast<const __half2*>(&w[i])));
    return fmaxf(__low2float(m), __high2float(m));
}
template <>
__device__ __forceinline__ float absmax16<float>(const float* q) {
    float m = 0.0f;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const float4 v = reinterpret_cast<const float4*>(q)[i];
        m = fmaxf(m, fmaxf(fmaxf(fabsf(v.x), fabsf(v.y)), fmaxf(fabsf(v.z), fabsf(v.w))));
    }
    return m;
}

__device__ __forceinline__ float rcp_approx(float x) {
    float y;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

__device__ __forceinline__ float ex2_approx(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

__device__ __forceinline__ void ldsm_x2(uint32_t (&r)[2], const void* p) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x2.shared.b16 {%0,%1}, [%2];"
                 : "=r"(r[0]), "=r"(r[1])
                 : "r"(smem_u32(p)));
}

// Packed f32x2 arithmetic (sm_100a FFMA2 / FMUL2 / FADD2): two lanes of work
// per issue slot for the per-(token, head) and per-(channel, head) math.
__device__ __forceinline__ unsigned long long f2u(float2 a) { return *reinterpret_cast<unsigned long long*>(&a); }
__device__ __forceinline__ float2 u2f(unsigned long long a) { return *reinterpret_cast<float2*>(&a); }
__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) {
    unsigned long long d;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(f2u(a)), "l"(f2u(b)), "l"(f2u(c)));
    return u2f(d);
}
__device__ __forceinline__ float2 fmul2(float2 a, float2 b) {
    unsigned long long d;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(f2u(a)), "l"(f2u(b)));
    return u2f(d);
}
__device__ __forceinline__ float2 fadd2(float2 a, float2 b) {
    unsigned long long d;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(f2u(a)), "l"(f2u(b)));
    return u2f(d);
}

// Two adjacent q values (channels c, c + 1) of one head row as f32.
template <typename IO>
__device__ __forceinline__ float2 ld_io2(const IO* p, int c);
template <>
__device__ __forceinline__ float2 ld_io2<__half>(const __half* p, int c) {
    return __half22float2(*reinterpret_cast<const __half2*>(p + c));
}
template <>
__device__ __forceinline__ float2 ld_io2<float>(const float* p, int c) {
    return *reinterpret_cast<const float2*>(p + c);
}

__device__ __forceinline__ void ldsm_x4_t(uint32_t (&r)[4], const void* p) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
                 : "r"(smem_u32(p)));
}
// D = A(f16, 16x16 row) * B(f16, 16x8 col) + D, f32 accumulate
__device__ __forceinline__ void hmma16816(float (&c)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
    asm("mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
        : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

// Per-lane constants of the u2x body, computed once per warp.
struct U2xLane {
    int lane, gid, tig, half;
    int bofs;        // ldmatrix (x4) row address of this lane inside a 512-B q~ digit block
    int bofs2;       // ldmatrix (x2) row address inside a 256-B p~ digit block
    int pdig_w;      // p~ digit store offset inside a 256-B block (rows 2 tig, 2 tig + 1)
    int qdig_w;      // q~ digit store offset (row 2 tig + 1, k-step 2 half + (lane >> 4))
    int qch;         // first channel of this lane's q~ prep (k-step, 16-channel half, class pair)
    uint32_t sel_lo, sel_hi;  // stage-2 PRMT selectors of the staggered q~ digit transpose
    uint32_t kmask, vm0, vm1;
    int vcol;        // V byte offset of this lane inside a 4-token group block (tig group + swizzled column)
    int ch0;         // first output channel of this lane (channels ch0 + 4m, ch0 + 4m + 1)
    float s0f;       // PV row scale of rows gid (row gid + 8: s0f / 4)
};

__device__ __forceinline__ uint32_t rot_sel(uint32_t s, int t) {  // rotate 4 PRMT nibbles left by t
    return ((s << (4 * t)) | (s >> (16 - 4 * t))) & 0xFFFFu;
}

__device__ __forceinline__ U2xLane u2x_lane(int half) {
    U2xLane c;
    c.lane = threadIdx.x & 31;
    c.gid = c.lane >> 2;
    c.tig = c.lane & 3;
    c.half = half;
    // digit blocks: rows of 32 B (one B column each), the two 16-B halves of
    // rows 4..7 (mod 8) swapped so ldmatrix phases hit distinct banks
    const int mat = c.lane >> 3, rr = c.lane & 7;
    c.bofs = ((mat >> 1) * 8 + rr) * 32 + (((mat & 1) ^ ((rr >> 2) & 1)) * 16);
    c.bofs2 = rr * 32 + (((mat & 1) ^ ((rr >> 2) & 1)) * 16);
    c.pdig_w = 2 * c.tig * 32 + (((c.gid >> 2) ^ ((c.tig >> 1) & 1)) * 16) + 4 * (c.gid & 3);
    // q~ prep: lane = (i, ch, p, h): head h = tig, class pair p, 16-channel half
    // ch, k-step 2 half + i; it writes digit rows 2h + 1 (d2), 8 + 2h (d1),
    // 9 + 2h (d0) at K positions 8p .. 8p + 7 of half ch
    const int p = (c.lane >> 2) & 1, ch = (c.lane >> 3) & 1, i = c.lane >> 4;
    const int kk = 2 * half + i;
    c.qdig_w = kk * 512 + (2 * c.tig + 1) * 32 + ((ch ^ (c.tig >> 1)) * 16) + 8 * p;
    c.qch = kk * 32 + 16 * ch + 2 * p;
    c.sel_lo = rot_sel(0x5410u, c.tig);
    c.sel_hi = rot_sel(0x7632u, c.tig);
    c.kmask = 0x03030303u << (2 * c.tig);
    const int jj = c.gid >> 2;
    c.vm0 = 0x03030303u << (4 * jj);      // rows gid:     code position 2 jj     (x 4^(2 jj))
    c.vm1 = 0x03030303u << (4 * jj + 2);  // rows gid + 8: code position 2 jj + 1 (x 4^(2 jj + 1))
    c.vcol = c.tig * 128 + (((16 * half + 4 * (c.gid & 3)) ^ (8 * c.tig)) * 4);  // vswz: (G & 3) == tig
    c.ch0 = 4 * (16 * half + 4 * (c.gid & 3)) + 2 * jj;
    c.s0f = jj ? 0.0625f : 1.0f;
    return c;
}

// FULLK: every one of the 128 K channels is kept at 2 bits (channel_perm is
// the identity, 32-B K rows) — the production shape; otherwise c0 < 128.
// The g query rows sit contiguously (one bulk copy) at the end of the slot.
//
// Fixed point: q~_c = scale_c * q_c is rounded to N = rint(q~ * sg * 4^(3 - t))
// (t = the channel's K-position class, whose codes the in-place mask scales by
// 4^t), |N| < 2^22, split into three balanced s8 digits (rows d2, d1, d0; the
// d3 row stays zero). p~ = p * vscale * 65280 / vmax < 2^16, two u8 digits
// (hi, lo) in rows 2h, 2h + 1 of a 256-B block.
// The float -> int roundings use the 1.5 * 2^23 / 2^23 magic-number adds, so
// the digit bytes come straight out of the float bits.
constexpr float kQFix = 65000.0f;   // sg = kQFix / bound: |N| <= 64 * 65000 < 2^22
constexpr float kMagicS = 12582912.0f;  // 1.5 * 2^23: bits = 0x4B400000 + rint(x), |x| < 2^22
constexpr float kMagicU = 8388608.0f;   // 2^23: bits = 0x4B000000 + rint(x), 0 <= x < 2^23
// Long tiles (> 160 slots) are decoded in chunks of <= 160 token slots by one
// pair, with an online softmax across the chunks (U2xRun); a chunk's data sits
// in the staging buffer at the offsets of U2xChunk, with the tile's header /
// channel table / q rows present only for the first chunk.
struct U2xChunk {
    int n, nslot;                // kept tokens / slots of this chunk
    int off_k, off_v, off_vp;    // K rows, V groups, V params inside the staging buffer
    int krb;                     // K row bytes
    bool first, last;
};
struct U2xRun {
    float vmax, bias2, qscale2;  // tile constants (this lane's head)
    float m, l;                  // running max (log2 units) and weight sum of this lane's head
    float2 o[4];                 // running unnormalised outputs (channels ch0 + 4m, + 1)
};

// ZCN > 0 (short tiles with a few Zone C rows, <= ZCN = 4 or 16): the tile's Zone C K / V
// rows are staged in its own buffer (zk / zv) and folded in after PV: QK on an
// fp16 m16n8k16 MMA (rows = the z tokens), PV on CUDA cores in the lanes'
// output mapping, one shared softmax.
constexpr int kZcFused = 4;      // fused rows of the default short-tile Zone C variant
constexpr int kZcFusedMax = 16;  // ... and of the long-generation variant (more smem per buffer)
constexpr int kZcKStride = 272;                        // padded K-row stride: conflict-free ldmatrix
__host__ __device__ constexpr int zc_stage(int rows) { return rows * (kZcKStride + 256); }  // K + V rows staged
// MIX ("mostly 2-bit" tiles, heavy-hitter caches): besides the 2-bit V rows
// and K channels, up to 32 K channels at 4 bits (one extra QK k-step, class-1
// digit block 4) and up to 8 V rows at 4 bits (their logits come from QK like
// any slot; their PV terms are added on CUDA cores after the 2-bit PV, whose
// p~ digits for those slots are zero).
constexpr int kMixMaxRows = 16;  // 4-bit V rows per MIX tile (the pt1 weight table)
template <typename IO, int NBMAX, bool FULLK, bool BULK, bool CHUNKED = false, int ZCN = 0, bool MIX = false,
          typename AfterSync1>
__device__ __forceinline__ void decode_tile_u2x(const uint8_t* __restrict__ t, const uint8_t* __restrict__ qs, int g,
                                                uint8_t* __restrict__ scr, IO* __restrict__ out, int bar,
                                                const U2xLane& L, AfterSync1&& after_sync1,
                                                const U2xChunk* ck = nullptr, U2xRun* run = nullptr, int z = 0,
                                                const uint8_t* zk = nullptr, const uint8_t* zv = nullptr) {
    constexpr int NBW = (NBMAX + 1) / 2;  // blocks per warp (upper bound)
    const int gid = L.gid, tig = L.tig, half = L.half;
    const bool hv = tig < g;
    const TileHeader& h = *reinterpret_cast<const TileHeader*>(t);
    PairX& xg = *reinterpret_cast<PairX*>(scr);
    uint8_t* qdig = scr + kXQDig;
    // MIX scratch: q~ digit block 4 (class-1 K) at kXPDig, then the 4-bit rows' weights
    float* pt1 = reinterpret_cast<float*>(scr + kXPDig + 512);  // [kMixMaxRows][4] (MIX only)
    uint8_t* pdig = scr + kXPDig + (MIX ? 512 + kMixMaxRows * 16 : 0);
    const float* chanf = reinterpret_cast<const float*>(t + kHeaderBytes);
    const bool first = CHUNKED ? ck->first : true;
    const int nslot = CHUNKED ? ck->nslot : h.nslot;
    // MIX: 2-bit rows are slots [0, r0), 4-bit rows [P0, P0 + r1) (P0 = pad4(r0))
    const int r1 = MIX ? h.r[1] : 0, c1 = MIX ? h.c[1] : 0, P0 = MIX ? ((h.r[0] + 3) & ~3) : 0;
    const int n = CHUNKED ? ck->n : (MIX && r1 > 0 ? P0 + r1 : h.r[0]);  // slots up to the last kept token
    const int nb = (n + 31) >> 5;             // 32-token blocks of this tile (warp-uniform)
    const int mynb = (nb + 1 - half) >> 1;    // blocks of this warp: half, half + 2, ...
    const int krb_c = FULLK ? 32 : (CHUNKED ? ck->krb : h.krow_bytes);
    const int Q = nslot >> 2;
    const int off_k = CHUNKED ? ck->off_k : h.off_k;
    const int off_v = CHUNKED ? ck->off_v : h.off_vseg[0];
    const int off_vp = CHUNKED ? ck->off_vp : h.off_vp;
    const uint32_t sbits = first ? h.scale_bounds : 0u;
    const float smax = bf16_bits_to_float(sbits & 0xFFFFu);
    const float vmax = (CHUNKED && !first) ? run->vmax : bf16_bits_to_float(sbits >> 16);
    constexpr float kInvSqrtD = 0.08838834764831845f;
    constexpr float kLog2e = 1.4426950408889634f;
    constexpr int QROW = kD * (int)sizeof(IO);
    float bias2, qscale2;
    if (CHUNKED && !first) {
        bias2 = run->bias2;
        qscale2 = run->qscale2;
        pair_sync(bar);  // both warps are past the previous chunk: its buffer may be refilled
        after_sync1();
    } else {

    // ---- q range per head: lanes 8h..8h+7 scan head h (16 channels each), then
    // every lane picks its head tig
    const int hq = L.lane >> 3;
    float qm = absmax16<IO>(reinterpret_cast<const IO*>(qs + (hq < g ? hq : 0) * QROW) + 16 * (L.lane & 7));
#pragma unroll
    for (int o = 1; o < 8; o <<= 1) qm = fmaxf(qm, __shfl_xor_sync(0xffffffffu, qm, o));
    qm = __shfl_sync(0xffffffffu, qm, 8 * tig);
    const IO* qh = reinterpret_cast<const IO*>(qs + (hv ? tig : 0) * QROW);
    float smx = smax;
    if (MIX && c1 > 0) {  // the 4-bit channels' scale bound (not in the header)
        float s1 = L.lane < c1 ? fabsf(chanf[2 * (128 + L.lane)]) : 0.0f;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) s1 = fmaxf(s1, __shfl_xor_sync(0xffffffffu, s1, o));
        smx = fmaxf(smx, s1);
    }
    const float bnd = smx * qm;
    const float sg = (hv && bnd > 0.0f) ? kQFix * rcp_approx(bnd) : 0.0f;  // heads >= g: zero digits

    // ---- q~ digits of k-steps 2 half, 2 half + 1 and the bias sum_c q_c * offset_c.
    // The lane takes channel pairs (c, c + 1) = classes (2p, 2p + 1) at e = 0..3
    // (c = qch + 4e); lanes of head tig visit e in the order (e + tig) & 3 so the
    // four heads' rows (256 B apart, same banks) are read at distinct banks, and
    // the final PRMT selectors rotate the bytes back into place.
    {
        const int ps = L.lane & 4;  // = 4p: class 2p -> prescale 4^(3 - 2p) = 2^(6 - 4p)
        const float sgA = sg * __int_as_float((127 + 6 - ps) << 23);  // class 2p
        const float sgB = sgA * 0.25f;                                // class 2p + 1
        uint32_t xa[4], xb[4];
        float2 bp = make_float2(0.0f, 0.0f);
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const int c = L.qch + 4 * ((e + tig) & 3);
            float2 qv;
            float4 cs;
            if constexpr (FULLK) {
                cs = *reinterpret_cast<const float4*>(chanf + 2 * c);
                qv = ld_io2(qh, c);
            } else {
                const uint16_t* perm = reinterpret_cast<const uint16_t*>(t + kHeaderBytes + 8 * h.kslots);
                const int c0 = h.c[0];
                const int j0 = min(c, h.kslots - 2);
                cs = *reinterpret_cast<const float4*>(chanf + 2 * j0);
                qv.x = c < c0 ? ld_io(qh, perm[j0]) : 0.0f;
                qv.y = c + 1 < c0 ? ld_io(qh, perm[j0 + 1]) : 0.0f;
            }
            bp = ffma2(qv, make_float2(cs.y, cs.w), bp);
            const float ya = fmaf(cs.x * qv.x, sgA, kMagicS), yb = fmaf(cs.z * qv.y, sgB, kMagicS);
            // balanced base-256 digits of N: byte k of (N + 0x808080) ^ 0x80
            xa[e] = (__float_as_uint(ya) + (0x00808080u - 0x4B400000u)) ^ 0x00808080u;
            xb[e] = (__float_as_uint(yb) + (0x00808080u - 0x4B400000u)) ^ 0x00808080u;
        }
        float bpart = bp.x + bp.y;
        if (MIX && c1 > 0 && half == 0) {
            // class-1 (4-bit) channels: K positions 4j .. 4j + 3 of head h = lane & 3
            // (j = lane >> 2), slot of K position p per the 4-bit in-place masks;
            // prescale 4 * 16^(1 - t'), so every product carries 64 like class 0
            const uint16_t* perm = reinterpret_cast<const uint16_t*>(t + kHeaderBytes + 8 * h.kslots);
            const int hh1 = tig, j = L.lane >> 2;  // (lane & 3 == tig: sg is already this head's scale)
            const IO* q1 = qh;
            const float sg1 = sg;
            uint32_t x1[4];
            float b1 = 0.0f;
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const int pk = 4 * j + e, rr = pk & 15, tt = rr >> 2;
                const int sl = 16 * (pk >> 4) + 8 * (tt >> 1) + 2 * (rr & 3) + (tt & 1);
                const float2 cs = reinterpret_cast<const float2*>(chanf)[128 + sl];
                const float qv = (sl < c1 && hh1 < g) ? ld_io(q1, perm[128 + sl]) : 0.0f;
                b1 = fmaf(qv, cs.y, b1);
                const float y = fmaf(cs.x * qv, sg1 * ((tt & 1) ? 4.0f : 64.0f), kMagicS);
                x1[e] = (__float_as_uint(y) + (0x00808080u - 0x4B400000u)) ^ 0x00808080u;
            }
            // this lane's bias share is for head hh1 = lane & 3 == tig
            bpart += b1;
            const uint32_t a01 = __byte_perm(x1[0], x1[1], 0x5140), b01 = __byte_perm(x1[0], x1[1], 0x7362);
            const uint32_t a23 = __byte_perm(x1[2], x1[3], 0x5140), b23 = __byte_perm(x1[2], x1[3], 0x7362);
            uint8_t* w1p = qdig + 4 * 512 + 4 * (j & 3);
            const int hsel = j >> 2;  // 16-B half of the 32 K positions
            // rows 2h+1 (d2), 8+2h (d1), 9+2h (d0); halves of rows 4..7 (mod 8) swapped
            *reinterpret_cast<uint32_t*>(w1p + (2 * hh1 + 1) * 32 + ((hsel ^ (hh1 >> 1)) * 16)) = __byte_perm(b01, b23, 0x5410);
            *reinterpret_cast<uint32_t*>(w1p + (8 + 2 * hh1) * 32 + ((hsel ^ (hh1 >> 1)) * 16)) = __byte_perm(a01, a23, 0x7632);
            *reinterpret_cast<uint32_t*>(w1p + (9 + 2 * hh1) * 32 + ((hsel ^ (hh1 >> 1)) * 16)) = __byte_perm(a01, a23, 0x5410);
        }
        // 4x4 byte transposes (digit d of value e -> byte e of word d), rotated by tig
        const uint32_t a01 = __byte_perm(xa[0], xa[1], 0x5140), b01 = __byte_perm(xa[0], xa[1], 0x7362);
        const uint32_t a23 = __byte_perm(xa[2], xa[3], 0x5140), b23 = __byte_perm(xa[2], xa[3], 0x7362);
        const uint32_t c01 = __byte_perm(xb[0], xb[1], 0x5140), d01 = __byte_perm(xb[0], xb[1], 0x7362);
        const uint32_t c23 = __byte_perm(xb[2], xb[3], 0x5140), d23 = __byte_perm(xb[2], xb[3], 0x7362);
        uint8_t* w = qdig + L.qdig_w;
        *reinterpret_cast<uint2*>(w) =  // d2 -> row 2 tig + 1
            make_uint2(__byte_perm(b01, b23, L.sel_lo), __byte_perm(d01, d23, L.sel_lo));
        *reinterpret_cast<uint2*>(w + 224) =  // d1 -> row 8 + 2 tig
            make_uint2(__byte_perm(a01, a23, L.sel_hi), __byte_perm(c01, c23, L.sel_hi));
        *reinterpret_cast<uint2*>(w + 256) =  // d0 -> row 9 + 2 tig
            make_uint2(__byte_perm(a01, a23, L.sel_lo), __byte_perm(c01, c23, L.sel_lo));
#pragma unroll
        for (int o = 4; o < 32; o <<= 1) bpart += __shfl_xor_sync(0xffffffffu, bpart, o);
        if (gid == 0) xg.bias[half][tig] = bpart;
    }
    // BULK: the previous tile's output stores read its buffer's q rows, and
    // that buffer is refilled right after this barrier
    if (BULK && L.lane == 0) bulk_wait_read0();
    pair_sync(bar);
    after_sync1();  // both warps are past the previous tile: its buffer may be refilled
    // l' = log2(e) * (v / (64 sg) + bias) / sqrt(d); heads >= g get -inf logits
    bias2 = hv ? (xg.bias[0][tig] + xg.bias[1][tig]) * (kInvSqrtD * kLog2e) : -INFINITY;
    qscale2 = bnd * (kInvSqrtD * kLog2e / (64.0f * kQFix));
    if constexpr (CHUNKED) {
        run->vmax = vmax;
        run->bias2 = bias2;
        run->qscale2 = qscale2;
        run->m = -INFINITY;
        run->l = 0.0f;
#pragma unroll
        for (int m = 0; m < 4; ++m) run->o[m] = make_float2(0.0f, 0.0f);
    }
    }  // first chunk

    // ---- QK over this warp's blocks half, half + 2, ...
    // A rows gid / gid + 8 of m-tile u = slots 32pb + 4gid + 2u / + 1, stored at
    // positions (2u + r) Q + 8pb + gid (slot-transposed K rows)
    const uint8_t* kbase = t + off_k + (size_t)(8 * half + gid) * krb_c;
    const int qstride = Q * krb_c;
    float2 lg[NBW][2];
    float mx = -INFINITY;
#pragma unroll
    for (int i = 0; i < NBW; ++i) {
        if (i < mynb) {
            const int pb = half + 2 * i;
            // q~ digit fragments re-read per block (4 LDSM) rather than held in 16
            // registers across the block loop: the register peak is here
            uint32_t bq[4][4];
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) ldsm_x4(bq[kk], qdig + kk * 512 + L.bofs);
            int acc[2][2][4];
#pragma unroll
            for (int u = 0; u < 2; ++u) {
                const uint8_t* r0 = kbase + 2 * u * qstride + 16 * i * krb_c;
                const uint8_t* r1 = r0 + qstride;
                const uint4 x0 = lds128(r0), x1 = lds128(r0 + 16), y0 = lds128(r1), y1 = lds128(r1 + 16);
                const uint32_t w0[8] = {x0.x, x0.y, x0.z, x0.w, x1.x, x1.y, x1.z, x1.w};
                const uint32_t w1[8] = {y0.x, y0.y, y0.z, y0.w, y1.x, y1.y, y1.z, y1.w};
#pragma unroll
                for (int nt = 0; nt < 2; ++nt) acc[u][nt][0] = acc[u][nt][1] = acc[u][nt][2] = acc[u][nt][3] = 0;
#pragma unroll
                for (int kk = 0; kk < 4; ++kk) {
                    const uint32_t a[4] = {w0[2 * kk] & L.kmask, w1[2 * kk] & L.kmask, w0[2 * kk + 1] & L.kmask,
                                           w1[2 * kk + 1] & L.kmask};
                    mma_u8s8(acc[u][0], a, bq[kk][0], bq[kk][1]);
                    mma_u8s8(acc[u][1], a, bq[kk][2], bq[kk][3]);
                }
                if (MIX && c1 > 0) {  // 4-bit K channels: bytes 32..47 of the row, 8 codes per word
                    uint32_t b4[4];
                    ldsm_x4(b4, qdig + 4 * 512 + L.bofs);
                    const uint4 z0 = lds128(r0 + 32), z1 = lds128(r1 + 32);
                    const uint32_t zw0[4] = {z0.x, z0.y, z0.z, z0.w}, zw1[4] = {z1.x, z1.y, z1.z, z1.w};
                    const uint32_t m4 = 0x0F0F0F0Fu << (4 * (tig & 1));
                    const uint32_t a[4] = {zw0[tig >> 1] & m4, zw1[tig >> 1] & m4, zw0[2 + (tig >> 1)] & m4,
                                           zw1[2 + (tig >> 1)] & m4};
                    mma_u8s8(acc[u][0], a, b4[0], b4[1]);
                    mma_u8s8(acc[u][1], a, b4[2], b4[3]);
                }
            }
            // rows (u, r) = slots 32 pb + 4 gid + 2u + r: v = d2 * 2^16 + d1 * 2^8 + d0
#pragma unroll
            for (int u = 0; u < 2; ++u) {
                const float2 hi = make_float2((float)acc[u][0][1], (float)acc[u][0][3]);
                const float2 lo = make_float2((float)(acc[u][1][0] * 256 + acc[u][1][1]),
                                              (float)(acc[u][1][2] * 256 + acc[u][1][3]));
                const float2 v = ffma2(hi, make_float2(65536.0f, 65536.0f), lo);
                lg[i][u] = ffma2(v, make_float2(qscale2, qscale2), make_float2(bias2, bias2));
            }
            if (MIX && 32 * pb + 32 > h.r[0]) {  // slots between the 2-bit rows and the 4-bit rows
                const int sbase = 32 * pb + 4 * gid;
#pragma unroll
                for (int u = 0; u < 2; ++u) {
                    const int s0 = sbase + 2 * u, s1 = s0 + 1;
                    if (!(s0 < h.r[0] || (s0 >= P0 && s0 < P0 + r1))) lg[i][u].x = -INFINITY;
                    if (!(s1 < h.r[0] || (s1 >= P0 && s1 < P0 + r1))) lg[i][u].y = -INFINITY;
                }
            } else if (32 * pb + 32 > n) {  // ragged last block: slots >= n get no weight
                const int sbase = 32 * pb + 4 * gid;
#pragma unroll
                for (int u = 0; u < 2; ++u) {
                    if (sbase + 2 * u >= n) lg[i][u].x = -INFINITY;
                    if (sbase + 2 * u + 1 >= n) lg[i][u].y = -INFINITY;
                }
            }
            mx = fmaxf(mx, fmaxf(fmaxf(lg[i][0].x, lg[i][0].y), fmaxf(lg[i][1].x, lg[i][1].y)));
        }
    }
#pragma unroll
    for (int o = 4; o < 32; o <<= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if (gid == 0) xg.mx[half][tig] = mx;
    pair_sync(bar);
    mx = fmaxf(xg.mx[0][tig], xg.mx[1][tig]);
    if (mx == -INFINITY) mx = 0.0f;  // head without tokens (tig >= g)
    const float psig = vmax > 0.0f ? kPScale * rcp_approx(vmax) : 0.0f;
    const float vinv = vmax * (1.0f / kPScale);

    // ---- softmax + p~ digits (hi, lo bytes): four consecutive slots per lane and block
    float2 ls2 = make_float2(0.0f, 0.0f);
    float bv = 0.0f;
    const float2* vparam = reinterpret_cast<const float2*>(t + off_vp);
    const float2 nmx = make_float2(-mx, -mx);
#pragma unroll
    for (int i = 0; i < NBW; ++i) {
        if (i < mynb) {
            const int pb = half + 2 * i;
            // slots past the tile read the last real group's finite parameters;
            // their weights are exactly zero
            const float4* vp4 = reinterpret_cast<const float4*>(vparam + min(32 * pb + 4 * gid, nslot - 4));
            const float4 va = vp4[0], vb = vp4[1];
            const float2 d01 = fadd2(lg[i][0], nmx), d23 = fadd2(lg[i][1], nmx);
            const float2 p01 = make_float2(ex2_approx(d01.x), ex2_approx(d01.y));
            const float2 p23 = make_float2(ex2_approx(d23.x), ex2_approx(d23.y));
            ls2 = fadd2(ls2, fadd2(p01, p23));
            bv = fmaf(p01.x, va.y, bv);
            bv = fmaf(p01.y, va.w, bv);
            bv = fmaf(p23.x, vb.y, bv);
            bv = fmaf(p23.y, vb.w, bv);
            const float2 vs01 = fmul2(make_float2(va.x, va.z), make_float2(psig, psig));
            const float2 vs23 = fmul2(make_float2(vb.x, vb.z), make_float2(psig, psig));
            float2 y01 = ffma2(p01, vs01, make_float2(kMagicU, kMagicU));
            float2 y23 = ffma2(p23, vs23, make_float2(kMagicU, kMagicU));
            if (MIX && r1 > 0 && 32 * pb + 32 > P0) {  // 4-bit rows: weight to the CUDA-core PV, digits 0
                const int sb = 32 * pb + 4 * gid;
                const float pp[4] = {p01.x, p01.y, p23.x, p23.y};
#pragma unroll
                for (int jj = 0; jj < 4; ++jj) {
                    const int t1 = sb + jj - P0;
                    if (t1 >= 0 && t1 < r1 && hv) pt1[t1 * 4 + tig] = pp[jj];
                }
                if (sb + 0 >= P0) y01.x = kMagicU;
                if (sb + 1 >= P0) y01.y = kMagicU;
                if (sb + 2 >= P0) y23.x = kMagicU;
                if (sb + 3 >= P0) y23.y = kMagicU;
            }
            const uint32_t t01 = __byte_perm(__float_as_uint(y01.x), __float_as_uint(y01.y), 0x5140);
            const uint32_t t23 = __byte_perm(__float_as_uint(y23.x), __float_as_uint(y23.y), 0x5140);
            uint8_t* pw = pdig + pb * 256 + L.pdig_w;
            *reinterpret_cast<uint32_t*>(pw) = __byte_perm(t01, t23, 0x7632);       // hi bytes -> row 2 tig
            *reinterpret_cast<uint32_t*>(pw + 32) = __byte_perm(t01, t23, 0x5410);  // lo bytes -> row 2 tig + 1
        }
    }
    float lsum = ls2.x + ls2.y;
#pragma unroll
    for (int o = 4; o < 32; o <<= 1) {
        lsum += __shfl_xor_sync(0xffffffffu, lsum, o);
        bv += __shfl_xor_sync(0xffffffffu, bv, o);
    }
    if (gid == 0) {
        xg.lsum[half][tig] = lsum;
        xg.bv[half][tig] = bv;
    }
    pair_sync(bar);
    const float lt = xg.lsum[0][tig] + xg.lsum[1][tig];
    const float bt = xg.bv[0][tig] + xg.bv[1][tig];

    // Zone C prepass row of this head (ZCN < 0): loaded here so the PV loop hides its latency
    float2 zpo[4];
    float zpm = -INFINITY, zpl = 0.0f;
    if constexpr (ZCN < 0 && !CHUNKED) {
        const float* zp = reinterpret_cast<const float*>(zk) + (hv ? tig : 0) * (kD + 2);
#pragma unroll
        for (int m = 0; m < 4; ++m) zpo[m] = *reinterpret_cast<const float2*>(zp + L.ch0 + 4 * m);
        zpm = zp[kD];
        zpl = zp[kD + 1];
    }
    // ---- PV: this warp's 4 m-tiles (byte columns 16 half + 4 (gid & 3) + m), one n-tile
    int acc[4][4];
#pragma unroll
    for (int m = 0; m < 4; ++m) acc[m][0] = acc[m][1] = acc[m][2] = acc[m][3] = 0;
    const uint8_t* g0b = t + off_v + L.vcol;
    const int nbv = MIX ? (P0 + 31) >> 5 : nb;  // 4-bit rows are not in the 2-bit PV
#pragma unroll
    for (int kk = 0; kk < NBMAX; ++kk) {
        if (kk < nbv) {
            uint32_t b[2];
            ldsm_x2(b, pdig + kk * 256 + L.bofs2);
            const uint4 x0 = lds128(g0b + kk * 1024), x1 = lds128(g0b + kk * 1024 + 512);
            const uint32_t u0[4] = {x0.x, x0.y, x0.z, x0.w}, u1[4] = {x1.x, x1.y, x1.z, x1.w};
#pragma unroll
            for (int m = 0; m < 4; ++m) {
                const uint32_t a[4] = {u0[m] & L.vm0, u0[m] & L.vm1, u1[m] & L.vm0, u1[m] & L.vm1};
                mma_u8u8(acc[m], a, b[0], b[1]);
            }
        }
    }
    // BULK (out in mapped host memory): outputs are staged in this tile's q rows
    // (dead since sync 1: both warps are past the q~ prep) and each head's
    // 64-channel half row of this warp leaves with one TMA bulk store (128 /
    // 256-B PCIe writes); otherwise lanes store straight to `out`
    IO* stage = BULK ? reinterpret_cast<IO*>(const_cast<uint8_t*>(qs)) : out;
    if constexpr (CHUNKED) {
        // online softmax across chunks: fold this chunk (max mx, sum lt,
        // unnormalised outputs v * s + bt) into the running state
        if (hv && lt > 0.0f) {
            const float mnew = fmaxf(run->m, mx);
            const float a = ex2_approx(run->m - mnew), bw = ex2_approx(mx - mnew);
            const float s0 = vinv * L.s0f;
            const float2 sc = make_float2(s0 * bw, s0 * 0.25f * bw), bb = make_float2(bt * bw, bt * bw);
            const float2 aa = make_float2(a, a);
#pragma unroll
            for (int m = 0; m < 4; ++m) {
                const float2 v =
                    make_float2((float)(acc[m][0] * 256 + acc[m][1]), (float)(acc[m][2] * 256 + acc[m][3]));
                run->o[m] = ffma2(run->o[m], aa, ffma2(v, sc, bb));
            }
            run->l = fmaf(run->l, a, lt * bw);
            run->m = mnew;
        }
        if (!ck->last) return;
        if (hv) {
            const float inv = rcp_approx(run->l);
            const float2 iv = make_float2(inv, inv);
            IO* orow = stage + tig * kD + L.ch0;
#pragma unroll
            for (int m = 0; m < 4; ++m) {
                const float2 r = fmul2(run->o[m], iv);
                if constexpr (sizeof(IO) == 2)
                    *reinterpret_cast<__half2*>(orow + 4 * m) = __float22half2_rn(r);
                else
                    *reinterpret_cast<float2*>(orow + 4 * m) = r;
            }
        }
    } else {
        float wa = 1.0f, wb = 0.0f, lz = 0.0f;
        float2 oz[4] = {make_float2(0.0f, 0.0f), make_float2(0.0f, 0.0f), make_float2(0.0f, 0.0f),
                        make_float2(0.0f, 0.0f)};
        float2 o4[4] = {make_float2(0.0f, 0.0f), make_float2(0.0f, 0.0f), make_float2(0.0f, 0.0f),
                        make_float2(0.0f, 0.0f)};
        if (MIX && r1 > 0 && hv) {
            // 4-bit V rows on CUDA cores: sum_t p_t * vscale_t * code_t for this
            // lane's channels ch0 + 4m (lo nibble) and + 1 (hi nibble); the
            // offsets are already in bt (they entered through the softmax)
            const float2* vparam4 = reinterpret_cast<const float2*>(t + h.off_vp);
            const uint8_t* v4 = t + h.off_vseg[1];
#pragma unroll 1
            for (int t1 = 0; t1 < r1; ++t1) {
                const float w = pt1[t1 * 4 + tig] * vparam4[P0 + t1].x;
                const int grp = t1 >> 2;
                const uint8_t* gb = v4 + grp * 256 + (t1 & 3);
#pragma unroll
                for (int m = 0; m < 4; ++m) {
                    const int mc = (L.ch0 + 4 * m) >> 1;  // byte column (two 4-bit channels)
                    const uint32_t byte = gb[((mc ^ (8 * (grp & 3))) * 4)];
                    o4[m] = ffma2(make_float2((float)(byte & 15u), (float)(byte >> 4)), make_float2(w, w), o4[m]);
                }
            }
        }
        if (ZCN < 0 && hv) {
            // Zone C from the prepass (zc_partial_kernel): this head's unnormalised
            // (o, max, sum) row, loaded before the PV loop (zpo, zpm, zpl)
#pragma unroll
            for (int m = 0; m < 4; ++m) oz[m] = zpo[m];
            const float mz = zpm;
            lz = zpl;
            if (lz > 0.0f) {
                const float mm = fmaxf(mx, mz);
                wa = ex2_approx(mx - mm);
                wb = ex2_approx(mz - mm);
            }
        }
        if (ZCN > 0 && z > 0) {
            // QK: A rows = Zone C tokens (rows >= z read neighbouring bytes, masked
            // below), B columns 2h / 2h + 1 = hi / lo fp16 parts of q_h
            float c[4] = {0.0f, 0.0f, 0.0f, 0.0f};
            const uint8_t* abase = zk + (L.lane & 15) * kZcKStride + (L.lane >> 4) * 16;
            const int bh = gid >> 1;
            const IO* qb = reinterpret_cast<const IO*>(qs + (bh < g ? bh : 0) * QROW);
            const bool bzero = bh >= g || (sizeof(IO) == 2 && (gid & 1));
#pragma unroll
            for (int ks = 0; ks < kD / 16; ++ks) {
                uint32_t a[4], bw[2];
                ldsm_x4(a, abase + ks * 32);
#pragma unroll
                for (int j = 0; j < 2; ++j) {
                    const int ch = ks * 16 + 8 * j + 2 * tig;
                    if constexpr (sizeof(IO) == 2) {
                        bw[j] = *reinterpret_cast<const uint32_t*>(qb + ch);
                    } else {
                        const float2 v = *reinterpret_cast<const float2*>(qb + ch);
                        const __half2 hi = __floats2half2_rn(v.x, v.y);
                        const float2 hf = __half22float2(hi);
                        const __half2 lo = __floats2half2_rn(v.x - hf.x, v.y - hf.y);
                        const __half2 sel = (gid & 1) ? lo : hi;
                        bw[j] = *reinterpret_cast<const uint32_t*>(&sel);
                    }
                    if (bzero) bw[j] = 0u;
                }
                hmma16816(c, a, bw[0], bw[1]);
            }
            constexpr float kZScale = 0.08838834764831845f * 1.4426950408889634f;  // log2(e) / sqrt(d)
            float l0 = (c[0] + c[1]) * kZScale;  // token gid, head tig
            float l1 = (c[2] + c[3]) * kZScale;  // token gid + 8 (ZCN > 8)
            if (!hv || gid >= z) l0 = -INFINITY;
            if (ZCN <= 8 || !hv || gid + 8 >= z) l1 = -INFINITY;
            float mz = fmaxf(l0, l1);
#pragma unroll
            for (int o = 4; o < 32; o <<= 1) mz = fmaxf(mz, __shfl_xor_sync(0xffffffffu, mz, o));
            if (mz == -INFINITY) mz = 0.0f;
            const float pz0 = ex2_approx(l0 - mz), pz1 = ZCN > 8 ? ex2_approx(l1 - mz) : 0.0f;
            lz = pz0 + pz1;
#pragma unroll
            for (int o = 4; o < 32; o <<= 1) lz += __shfl_xor_sync(0xffffffffu, lz, o);
            // PV: this lane's output channels ch0 + 4m, + 1 of head tig
#pragma unroll
            for (int tk = 0; tk < ZCN; ++tk) {
                const float pt = __shfl_sync(0xffffffffu, tk < 8 ? pz0 : pz1, 4 * (tk & 7) + tig);
                if (tk < z) {
                    const float2 ptt = make_float2(pt, pt);
#pragma unroll
                    for (int m = 0; m < 4; ++m)
                        oz[m] = ffma2(__half22float2(*reinterpret_cast<const __half2*>(zv + tk * 256 + 2 * (L.ch0 + 4 * m))),
                                      ptt, oz[m]);
                }
            }
            const float mm = fmaxf(mx, mz);
            wa = ex2_approx(mx - mm);
            wb = ex2_approx(mz - mm);
        }
        if (hv) {
            const float inv = rcp_approx(fmaf(lt, wa, lz * wb));
            const float s0 = vinv * L.s0f * wa * inv, bta = bt * wa * inv, zb = wb * inv;
            const float2 sc = make_float2(s0, s0 * 0.25f), bb = make_float2(bta, bta), zz = make_float2(zb, zb);
            const float2 ww = make_float2(wa * inv, wa * inv);
            IO* orow = stage + tig * kD + L.ch0;
#pragma unroll
            for (int m = 0; m < 4; ++m) {
                const float2 v =
                    make_float2((float)(acc[m][0] * 256 + acc[m][1]), (float)(acc[m][2] * 256 + acc[m][3]));
                float2 r = ffma2(v, sc, bb);
                if (ZCN != 0) r = ffma2(oz[m], zz, r);
                if (MIX) r = ffma2(o4[m], ww, r);
                if constexpr (sizeof(IO) == 2)
                    *reinterpret_cast<__half2*>(orow + 4 * m) = __float22half2_rn(r);
                else
                    *reinterpret_cast<float2*>(orow + 4 * m) = r;
            }
        }
    }
    if constexpr (BULK) {
        __syncwarp();
        if (L.lane == 0) {
            fence_proxy_async();
            for (int hh = 0; hh < g; ++hh)
                bulk_s2g(out + hh * kD + 64 * half, stage + hh * kD + 64 * half, 64 * (uint32_t)sizeof(IO));
            bulk_commit();
        }
    }
}

constexpr int kXPairs = 8;   // <= 16 warps per CTA: up to 128 registers per thread
constexpr int kXMaxBuf = 4;  // tile buffers per pair

// Self-fed warp pairs: pair p owns NBUF tile buffers and decodes the CTA's
// tiles p, p + W, p + 2W, ...; one lane of the pair issues the TMA bulk
// copies of its own next tiles (tile + q rows: two copies), so a slow pair
// never blocks the others' loads (no shared producer, no head-of-line
// blocking). At start only the first tile of every pair is requested; the
// rest of the pair's buffers are filled once it has landed, so the first
// round's tiles are not queued behind everyone's look-ahead.
// MODE (timing experiments only, RDKV_DECODE_NULL): 0 decode, 1 loads only
// (no math), 2 math only (tiles past the first buffers are not reloaded).
// PERCTA: one pair per CTA (a compile-time barrier id, so a CTA reserves 2
// hardware barriers instead of 16 and 8 CTAs fit on an SM).
#ifdef RDKV_DECODE_EXPERIMENTS
// Timeline trace (experiments build only, tools/u2x_trace.py): per pair of the
// last launch, the globaltimer at entry, after the grid dependency, and per tile
// the buffer wait and the tile's end; slot 19 = SM id.
constexpr int kTraceSlots = 20;
__device__ unsigned long long* g_u2x_trace = nullptr;
__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
#define U2X_TRACE(slot)                                                                                   \
    do {                                                                                                   \
        if (g_u2x_trace && half == 0 && lane == 0 && (slot) < kTraceSlots)                                 \
            g_u2x_trace[((size_t)blockIdx.x * p.W + pr) * kTraceSlots + (slot)] = gtimer();                \
    } while (0)
#else
#define U2X_TRACE(slot) \
    do {                \
    } while (0)
#endif
template <typename IO, int NBMAX, bool FULLK, int MODE = 0, bool BULK = false, bool PERCTA = false, int ZCN = 0,
          bool G8 = false, bool MIX = false>
__global__ void __launch_bounds__(32 * 2 * kXPairs, 1) decode_u2x_kernel(const MmaParams p) {
    extern __shared__ __align__(128) uint8_t dsm[];
    const int nbuf = p.R;  // buffers per pair
    uint64_t* full = reinterpret_cast<uint64_t*>(dsm);  // [W][kXMaxBuf]
    uint8_t* bufs = dsm + p.W * kXMaxBuf * sizeof(uint64_t);
    uint8_t* scratch0 = bufs + (size_t)p.W * nbuf * p.slot_bytes;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // with a multiple of 4 pairs, a pair's two warps sit on the same SM
    // sub-partition (warp w -> SMSP w % 4): warps (8j + s, 8j + s + 4)
    const bool same_smsp = getenv_pair_smsp() && (p.W & 3) == 0;
    const int pr = same_smsp ? ((warp & 3) | ((warp >> 3) << 2)) : warp >> 1;
    const int half = same_smsp ? (warp >> 2) & 1 : warp & 1;
    constexpr int QROW = kD * (int)sizeof(IO);
    const int qbytes = p.g * QROW;
    uint64_t* fb = full + pr * kXMaxBuf;
    uint8_t* pbuf = bufs + (size_t)pr * nbuf * p.slot_bytes;
    uint8_t* scr = scratch0 + (size_t)pr * p.scratch_bytes;
    const int tile0 = blockIdx.x + pr * gridDim.x, tstride = p.W * gridDim.x;
    const int qoff = p.slot_bytes - qbytes;
    // A tile's KV copy needs its arena offset and size from global memory; the
    // issuing lanes load them one refill AHEAD (into registers) so the ~1 us
    // of LDG latency never stalls a warp at the refill point.
    struct Meta {
        const uint8_t* src;
        uint32_t sz;
    };
    auto meta = [&](int k) {
        const int tile = tile0 + k * tstride;
        Meta m{nullptr, 0u};
        if (tile < p.units) {
            const int u = unit_of(p, tile);
            m.src = p.arena + p.offsets[u];
            m.sz = (uint32_t)p.dsize[u];
        }
        return m;
    };
    // A tile arrives in two parts on its buffer's mbarrier: the KV copy (tx only,
    // may run before the grid dependency), then q (+ ZCN > 0: the tile's Zone C
    // rows) with the arrive — so the phase cannot complete early.
    auto issue_kv = [&](const Meta& m, int b) {
        fence_proxy_async();
        mbar_expect_tx_only(&fb[b], m.sz);
        bulk_g2s(pbuf + (size_t)b * p.slot_bytes, m.src, m.sz, &fb[b]);
    };
    auto issue_q = [&](int k, int b, int zrows) {
        const int tile = unit_of(p, tile0 + k * tstride);
        uint8_t* dst = pbuf + (size_t)b * p.slot_bytes;
        mbar_expect_tx(&fb[b], (uint32_t)(qbytes + 2 * 256 * zrows));
        bulk_g2s(dst + qoff, static_cast<const uint8_t*>(p.q) + (size_t)tile * qbytes, (uint32_t)qbytes, &fb[b]);
        if (ZCN > 0 && zrows > 0) {
            const size_t row0 = (size_t)tile * p.zc_cap;
            for (int r = 0; r < zrows; ++r)  // K rows at a padded stride
                bulk_g2s(dst + qoff - zc_stage(ZCN) + r * kZcKStride,
                         reinterpret_cast<const uint8_t*>(p.zc_k + (row0 + r) * kD), 256u, &fb[b]);
            bulk_g2s(dst + qoff - ZCN * 256, reinterpret_cast<const uint8_t*>(p.zc_v + row0 * kD),
                     (uint32_t)(zrows * 256), &fb[b]);
        }
    };
    // Zone C rows of a tile (written by the previous kernel: after griddepcontrol.wait only)
    auto zrows_of = [&](int k) {
        const int tile = tile0 + k * tstride;
        return (ZCN > 0 && tile < p.units) ? min(p.zc_len[unit_of(p, tile)], ZCN) : 0;
    };
    // Programmatic dependent launch: this grid may start while the previous
    // kernel on the stream drains. The packed KV tiles are immutable during
    // decode, so the first tile's KV stream starts at once; q (produced by the
    // previous kernel in a model) is read and out written only after
    // griddepcontrol.wait. Dependents of this grid may launch right away: their
    // CTAs take SMs as ours retire.
    U2X_TRACE(0);
#ifdef RDKV_DECODE_EXPERIMENTS
    if (g_u2x_trace && half == 0 && lane == 0) {
        unsigned int smid;
        asm volatile("mov.u32 %0, %smid;" : "=r"(smid));
        g_u2x_trace[((size_t)blockIdx.x * p.W + pr) * kTraceSlots + 19] = smid;
    }
#endif
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    Meta ahead[kXMaxBuf - 1];  // half 1, lane 0: tiles 1 .. nbuf - 1 (look-ahead at tile 0)
    Meta next{nullptr, 0u};    // half 0, lane 0: the next refill target
    if (half == 0 && lane == 0) {
        for (int b = 0; b < nbuf; ++b) mbar_init(&fb[b], 1);
        fence_barrier_init();
        if (tile0 < p.units) issue_kv(meta(0), 0);
        next = meta(nbuf);  // refill at tile 1 -> tile nbuf
    }
    if (half == 1 && lane == 0)
        for (int j = 1; j < kXMaxBuf; ++j) ahead[j - 1] = j < nbuf ? meta(j) : Meta{nullptr, 0u};
    // concurrent (split step): the predecessor is the general kernel, which only
    // triggers this launch after its own grid dependency resolved, so q is
    // ready now; this grid waits for it at exit instead, so kernels after this
    // one still see both halves of the step done
    if (!p.concurrent) asm volatile("griddepcontrol.wait;" ::: "memory");
    U2X_TRACE(1);
    int next_z = 0, ahead_z[kXMaxBuf - 1] = {0, 0, 0};
    if (half == 0 && lane == 0) {
        if (tile0 < p.units) issue_q(0, 0, zrows_of(0));
        next_z = zrows_of(nbuf);
    }
    if (ZCN > 0 && half == 1 && lane == 0)
        for (int j = 1; j < kXMaxBuf; ++j) ahead_z[j - 1] = j < nbuf ? zrows_of(j) : 0;
    const U2xLane lc = u2x_lane(half);
    // the q~ digit rows of d3 (never written: |N| < 2^22) must read as zero
    for (int i = threadIdx.x & 63; i < (MIX ? 5 : 4) * 512 / 16; i += 64)
        reinterpret_cast<uint4*>(scr + kXQDig)[i] = make_uint4(0u, 0u, 0u, 0u);
    __syncthreads();
    int b = 0;
    uint32_t phase = 0;
    int k = 0;
    int zl_next = zrows_of(0);  // this lane's view of the tile's Zone C rows, one tile ahead
    for (int tile = tile0; tile < p.units; tile += tstride, ++k) {
        const int zl = zl_next;
        zl_next = zrows_of(k + 1);
        if (MODE != 2 || k < nbuf) mbar_wait(&fb[b], phase);
        U2X_TRACE(2 + 2 * k);
        __syncwarp();
        const uint8_t* st = pbuf + (size_t)b * p.slot_bytes;
        if (k == 0 && half == 1 && lane == 0) {  // look-ahead once the first tile is in
#pragma unroll
            for (int j = 1; j < kXMaxBuf; ++j)
                if (j < nbuf && ahead[j - 1].src) {
                    issue_kv(ahead[j - 1], j);
                    issue_q(j, j, ahead_z[j - 1]);
                }
        }
        IO* o = static_cast<IO*>(p.out) + (size_t)unit_of(p, tile) * p.g * kD;
        const int bprev = b == 0 ? nbuf - 1 : b - 1;
        // the buffer of tile k - 1 takes tile k - 1 + nbuf
        auto refill = [&]() {
            if (MODE != 2 && half == 0 && lane == 0 && k >= 1) {
                if (next.src) {
                    issue_kv(next, bprev);
                    issue_q(k - 1 + nbuf, bprev, next_z);
                }
                next = meta(k + nbuf);
                next_z = zrows_of(k + nbuf);
            }
        };
        if (MODE == 1) {
            pair_sync(PERCTA ? 1 : 1 + pr);
            refill();
        } else {
            // GQA groups of up to 8 heads: one pass per 4 heads over the same staged
            // tile (the buffer refill is issued once, in the first pass)
#pragma unroll 1
            for (int hp = 0; hp < (G8 ? 2 : 1) && 4 * hp < p.g; ++hp) {
                auto rf = [&]() {
                    if (hp == 0) refill();
                };
                decode_tile_u2x<IO, NBMAX, FULLK, BULK, false, ZCN, MIX>(
                    st, st + qoff + 4 * hp * QROW, G8 ? min(4, p.g - 4 * hp) : p.g, scr, o + 4 * hp * kD,
                    PERCTA ? 1 : 1 + pr, lc, rf, nullptr, nullptr, zl,
                    ZCN < 0 ? reinterpret_cast<const uint8_t*>(p.partial + ((size_t)unit_of(p, tile) * p.g + 4 * hp) * (kD + 2))
                            : st + qoff - zc_stage(ZCN),
                    st + qoff - ZCN * 256);
            }
        }
        U2X_TRACE(3 + 2 * k);
        if (++b == nbuf) {
            b = 0;
            phase ^= 1u;
        }
    }
    if (p.concurrent && threadIdx.x == 0) asm volatile("griddepcontrol.wait;" ::: "memory");
    if (BULK && lane == 0) bulk_wait0();
}

// Pairs per CTA and buffers per pair: as many pairs as fit (issue slots are
// the bound, so more resident warps hide more latency; measured 15.7 us at 8
// pairs vs 16.6 us at 7 on the 4096-tile step), then as many buffers per pair
// (>= 2, double buffering) as fit.
// Timing-experiment knobs (loads-only / math-only kernels, forced launch
// geometry, launch tracing) exist only in a debug build compiled with
// -DRDKV_DECODE_EXPERIMENTS (make EXPERIMENTS=1); the product library never
// reads the environment, so no variable can change what a decode computes.
static const char* experiment_knob(const char* name) {
#ifdef RDKV_DECODE_EXPERIMENTS
    return getenv(name);
#else
    (void)name;
    return nullptr;
#endif
}

static bool verbose_env() {
    static const bool v = experiment_knob("RDKV_DECODE_VERBOSE") != nullptr;
    return v;
}

static bool pick_pairs(int units, int nsm, int slot, int scratch, int smem_max, int& W, int& nbuf) {
    const int head = kXPairs * kXMaxBuf * (int)sizeof(uint64_t);  // upper bound of W * kXMaxBuf barriers
    static const char* env = experiment_knob("RDKV_DECODE_PAIRS");  // read once per process
    const int forced = env ? atoi(env) : 0;
    const int per_sm = (units + nsm - 1) / nsm;
    W = 0;
    for (int w = 1; w <= kXPairs && w <= per_sm; ++w) {
        if (forced && w != forced) continue;
        if (head + (size_t)w * (2 * slot + scratch) > (size_t)smem_max) continue;
        W = w;
    }
    if (W == 0) return false;
    nbuf = 2;
    while (nbuf < kXMaxBuf && head + (size_t)W * ((nbuf + 1) * slot + scratch) <= (size_t)smem_max) ++nbuf;
    return true;
}

// ---------------------------------------------------------------------------
// Long uniform-2-bit tiles (more than 160 token slots, e.g. the configs[3]
// budget sweep: 512 .. 2048 FP16-equivalent tokens per layer keep 256 .. 1024
// tokens per head at 2 bits). A pair walks its tiles chunk by chunk: chunk c of
// a tile covers slots [c S, c S + ns) (S a multiple of 32, <= 160), staged by
// TMA as [tile header + channel table | 4 K-row runs | V groups | V params |
// q rows] (header and q only for c = 0), and folded into an online softmax.
__device__ __forceinline__ void u2c_geom(int nslot, int c, int& C, int& s0, int& ns) {
    C = nslot <= 160 ? 1 : (nslot + 159) / 160;
    const int S = C == 1 ? nslot : (((nslot + C - 1) / C) + 31) & ~31;
    s0 = c * S;
    ns = min(S, nslot - s0);
}

// ---- Zone C (appended fp16 K/V rows, trizone.cpp:307-314) on the fast path.
// After a tile's packed chunks its Zone C rows are decoded in chunks of 16
// tokens with fp16 tensor-core MMAs (m16n8k16, f32 accumulate), q and the
// softmax weights split hi + lo into two fp16 columns each so the products
// keep ~22 bits, and folded into the same online softmax.
constexpr int kZcChunk = 16;
constexpr int kQ16Row = 272;              // bytes per row of the fp16 q table (8 rows, padded)
constexpr int kQ16Bytes = 8 * kQ16Row;
constexpr int kZcAuxWarp = 256 + 4 * 64 * 4;  // per warp: P tile (8 x 16 fp16) + output exchange (4 x 64 f32)

// Rows 2h / 2h + 1 = hi / lo fp16 parts of q_h (zero for h >= g); warp `half`
// writes channels 64 half .. 64 half + 63 (visible to the pair after sync 1).
template <typename IO>
__device__ __forceinline__ void build_q16(const uint8_t* qs, int g, uint8_t* q16, const U2xLane& L) {
    const int r = L.lane >> 2, hq = r >> 1, lo = r & 1;
    const int c0 = 64 * L.half + 16 * (L.lane & 3);
    const IO* qh = reinterpret_cast<const IO*>(qs + (hq < g ? hq : 0) * kD * (int)sizeof(IO));
    uint32_t w[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        __half v2[2];
#pragma unroll
        for (int j = 0; j < 2; ++j) {
            const float qv = hq < g ? ld_io(qh, c0 + 2 * i + j) : 0.0f;
            const __half hi = __float2half_rn(qv);
            v2[j] = lo ? __float2half_rn(qv - __half2float(hi)) : hi;
        }
        w[i] = *reinterpret_cast<uint32_t*>(v2);
    }
    uint4* dst = reinterpret_cast<uint4*>(q16 + r * kQ16Row + 2 * c0);
    dst[0] = make_uint4(w[0], w[1], w[2], w[3]);
    dst[1] = make_uint4(w[4], w[5], w[6], w[7]);
}

// One Zone C chunk: K rows [16][d] fp16 at st, V rows at st + 16 * 256, cnt
// valid tokens; each warp's spare (P tile, output exchange) follows the V rows.
template <typename IO, bool BULK, typename AfterSync1>
__device__ __forceinline__ void zc_chunk_u2x(const uint8_t* __restrict__ st, int cnt, const uint8_t* __restrict__ q16,
                                             int g, int bar, const U2xLane& L, U2xRun& run, bool last,
                                             IO* __restrict__ out, IO* __restrict__ stage, AfterSync1&& after_sync1) {
    constexpr float kScale = 0.08838834764831845f * 1.4426950408889634f;  // log2(e) / sqrt(d)
    const int lane = L.lane, gid = L.gid, tig = L.tig, half = L.half;
    const bool hv = tig < g;
    pair_sync(bar);  // both warps are past the previous item: its buffer may be refilled
    after_sync1();
    uint8_t* vrows = const_cast<uint8_t*>(st) + kZcChunk * kZcKStride;
    uint8_t* aux = const_cast<uint8_t*>(st) + 2 * kZcChunk * kZcKStride + half * kZcAuxWarp;  // this warp's spare
    // rows past cnt hold stale bytes: zero this warp's channel half of the V rows
    for (int r = cnt + (lane >> 3); r < kZcChunk; r += 4)
        *reinterpret_cast<uint4*>(vrows + r * kZcKStride + 128 * half + 16 * (lane & 7)) = make_uint4(0u, 0u, 0u, 0u);
    // ---- QK (every warp, all 16 tokens): A = K rows, B = q table
    float c[4] = {0.0f, 0.0f, 0.0f, 0.0f};
    const uint8_t* abase = st + (lane & 15) * kZcKStride + (lane >> 4) * 16;
    const uint8_t* bbase = q16 + (lane & 7) * kQ16Row + ((lane >> 3) & 1) * 16;
#pragma unroll
    for (int ks = 0; ks < kD / 16; ++ks) {
        uint32_t a[4], b[2];
        ldsm_x4(a, abase + ks * 32);
        ldsm_x2(b, bbase + ks * 32);
        hmma16816(c, a, b[0], b[1]);
    }
    // rows gid, gid + 8 = tokens; columns 2 tig (hi), 2 tig + 1 (lo) = head tig
    float l0 = (c[0] + c[1]) * kScale, l1 = (c[2] + c[3]) * kScale;
    if (!hv || gid >= cnt) l0 = -INFINITY;
    if (!hv || gid + 8 >= cnt) l1 = -INFINITY;
    float m = fmaxf(l0, l1);
#pragma unroll
    for (int o = 4; o < 32; o <<= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    if (m == -INFINITY) m = 0.0f;
    const float p0 = ex2_approx(l0 - m), p1 = ex2_approx(l1 - m);
    float ls = p0 + p1;
#pragma unroll
    for (int o = 4; o < 32; o <<= 1) ls += __shfl_xor_sync(0xffffffffu, ls, o);
    // ---- P as the PV B operand: rows 2 tig (hi) / 2 tig + 1 (lo), 16 tokens of fp16
    __half* pt = reinterpret_cast<__half*>(aux);
    const __half h0 = __float2half_rn(p0), h1 = __float2half_rn(p1);
    pt[(2 * tig) * 16 + gid] = h0;
    pt[(2 * tig + 1) * 16 + gid] = __float2half_rn(p0 - __half2float(h0));
    pt[(2 * tig) * 16 + gid + 8] = h1;
    pt[(2 * tig + 1) * 16 + gid + 8] = __float2half_rn(p1 - __half2float(h1));
    __syncwarp();
    uint32_t bp[2];
    ldsm_x2(bp, aux + (lane & 7) * 32 + ((lane >> 3) & 1) * 16);
    // ---- PV: this warp's channels 64 half .. + 63 as 4 m-tiles (A = V^T via ldmatrix.trans)
    float* xo = reinterpret_cast<float*>(aux + 256);  // [4 heads][64 channels]
    const uint8_t* vbase =
        vrows + ((lane & 7) + 8 * ((lane >> 4) & 1)) * kZcKStride + (64 * half + 8 * ((lane >> 3) & 1)) * 2;
#pragma unroll
    for (int mt = 0; mt < 4; ++mt) {
        uint32_t a[4];
        ldsm_x4_t(a, vbase + mt * 32);
        float o[4] = {0.0f, 0.0f, 0.0f, 0.0f};
        hmma16816(o, a, bp[0], bp[1]);
        xo[tig * 64 + 16 * mt + gid] = o[0] + o[1];
        xo[tig * 64 + 16 * mt + gid + 8] = o[2] + o[3];
    }
    __syncwarp();
    // ---- fold into the running state in the u2x lane mapping (channels ch0 + 4m, + 1)
    if (hv && ls > 0.0f) {
        const float mnew = fmaxf(run.m, m);
        const float a = ex2_approx(run.m - mnew), bw = ex2_approx(m - mnew);
        const float2 aa = make_float2(a, a), bb = make_float2(bw, bw);
        const float* xr = xo + tig * 64 + (L.ch0 - 64 * half);
#pragma unroll
        for (int mm = 0; mm < 4; ++mm) {
            const float2 z = *reinterpret_cast<const float2*>(xr + 4 * mm);
            run.o[mm] = ffma2(run.o[mm], aa, fmul2(z, bb));
        }
        run.l = fmaf(run.l, a, ls * bw);
        run.m = mnew;
    }
    if (!last) return;
    if (hv) {
        const float inv = rcp_approx(run.l);
        const float2 iv = make_float2(inv, inv);
        IO* orow = stage + tig * kD + L.ch0;
#pragma unroll
        for (int mm = 0; mm < 4; ++mm) {
            const float2 r = fmul2(run.o[mm], iv);
            if constexpr (sizeof(IO) == 2)
                *reinterpret_cast<__half2*>(orow + 4 * mm) = __float22half2_rn(r);
            else
                *reinterpret_cast<float2*>(orow + 4 * mm) = r;
        }
    }
    if constexpr (BULK) {
        __syncwarp();
        if (lane == 0) {
            fence_proxy_async();
            for (int hh = 0; hh < g; ++hh)
                bulk_s2g(out + hh * kD + 64 * half, stage + hh * kD + 64 * half, 64 * (uint32_t)sizeof(IO));
            bulk_commit();
        }
    }
}

template <typename IO, bool FULLK, bool BULK, bool ZC = false>
__global__ void __launch_bounds__(32 * 2 * kXPairs, 1) decode_u2c_kernel(const MmaParams p) {
    extern __shared__ __align__(128) uint8_t dsm[];
    const int nbuf = p.R;
    uint64_t* full = reinterpret_cast<uint64_t*>(dsm);
    uint8_t* bufs = dsm + p.W * kXMaxBuf * sizeof(uint64_t);
    uint8_t* scratch0 = bufs + (size_t)p.W * nbuf * p.slot_bytes;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int pr = warp >> 1, half = warp & 1;
    constexpr int QROW = kD * (int)sizeof(IO);
    const int qbytes = p.g * QROW;
    uint64_t* fb = full + pr * kXMaxBuf;
    uint8_t* pbuf = bufs + (size_t)pr * nbuf * p.slot_bytes;
    uint8_t* scr = scratch0 + (size_t)pr * p.scratch_bytes;
    uint8_t* q16 = scr + p.scratch_bytes - kQ16Bytes;  // ZC only
    const int tile0 = blockIdx.x + pr * gridDim.x, tstride = p.W * gridDim.x;
    const int qoff = p.slot_bytes - qbytes;
    const bool issuer = half == 0 && lane == 0;

    // ---- issuer state (one lane): the next item (tile, chunk) to stage
    struct TileMeta {
        const uint8_t* base;
        int nslot, hk, krb, offv, offvp;
    };
    auto load_meta = [&](int tile) {
        TileMeta m{nullptr, 0, 0, 0, 0, 0};
        if (tile < p.units) {
            m.base = p.arena + p.offsets[tile];
            const TileHeader* th = reinterpret_cast<const TileHeader*>(m.base);
            m.nslot = th->nslot;
            m.hk = th->off_k;
            m.krb = th->krow_bytes;
            m.offv = th->off_vseg[0];
            m.offvp = th->off_vp;
        }
        return m;
    };
    int cur_tile = tile0, cur_c = 0, cur_zc = 0;
    // sequence split (p.partial): this rank decodes chunks c % world == rank of
    // every tile (chunk 0 is always staged: header, channel table and q)
    const bool psplit = p.partial != nullptr;
    auto owned = [&](int c) { return !psplit || c % p.split_world == p.split_rank; };
    TileMeta cur{nullptr, 0, 0, 0, 0, 0}, nxt{nullptr, 0, 0, 0, 0, 0};
    // Zone C lengths are written by the previous kernel (append): read only
    // after griddepcontrol.wait
    auto zc_of = [&](int tile) { return (ZC && tile < p.units) ? p.zc_len[tile] : 0; };
    // stage the cursor's item into buffer b (q rows optional: the first item's
    // q waits for the grid dependency); returns false when the pair is done
    auto advance = [&]() {
        int C, s0, ns;
        u2c_geom(cur.nslot, 0, C, s0, ns);
        const int total = C + (cur_zc + kZcChunk - 1) / kZcChunk;
        do {
            ++cur_c;
        } while (cur_c < total && !owned(cur_c));
        if (cur_c >= total) {
            cur_tile += tstride;
            cur_c = 0;
            cur = nxt;
            nxt = load_meta(cur_tile + tstride);
            cur_zc = zc_of(cur_tile);
        }
    };
    auto stage_item = [&](int b, bool with_q) {
        if (cur_tile >= p.units || !cur.base) return false;
        int C, s0, ns;
        u2c_geom(cur.nslot, cur_c, C, s0, ns);
        uint8_t* dst = pbuf + (size_t)b * p.slot_bytes;
        if (ZC && cur_c >= C) {  // Zone C chunk (cur_c - C) of this tile
            const int j = cur_c - C;
            const int rows = min(kZcChunk, cur_zc - kZcChunk * j);
            const size_t row0 = (size_t)cur_tile * p.zc_cap + (size_t)kZcChunk * j;
            fence_proxy_async();
            mbar_expect_tx(&fb[b], (uint32_t)(2 * rows * 256));
            // one copy per row into padded (272-B) rows: conflict-free ldmatrix
            for (int r = 0; r < rows; ++r) {
                bulk_g2s(dst + r * kZcKStride, reinterpret_cast<const uint8_t*>(p.zc_k + (row0 + r) * kD), 256u, &fb[b]);
                bulk_g2s(dst + (kZcChunk + r) * kZcKStride, reinterpret_cast<const uint8_t*>(p.zc_v + (row0 + r) * kD),
                         256u, &fb[b]);
            }
        } else {
            const bool own = owned(cur_c);  // a chunk 0 another rank owns: header + q only
            const int rows = own ? ns >> 2 : 0, Q = cur.nslot >> 2;
            const uint32_t kbytes = (uint32_t)(rows * cur.krb), vbytes = (uint32_t)(rows * 128),
                           pbytes = (uint32_t)(rows * 4 * 8);
            const bool c0 = cur_c == 0;
            const uint32_t tx = 4 * kbytes + vbytes + pbytes + (c0 ? (uint32_t)(cur.hk + qbytes) : 0u);
            fence_proxy_async();
            mbar_expect_tx(&fb[b], tx);
            if (c0) bulk_g2s(dst, cur.base, (uint32_t)cur.hk, &fb[b]);
            const int dk = cur.hk;
            if (rows > 0) {
#pragma unroll
                for (int r = 0; r < 4; ++r)
                    bulk_g2s(dst + dk + r * kbytes, cur.base + cur.hk + (size_t)(r * Q + (s0 >> 2)) * cur.krb, kbytes,
                             &fb[b]);
                bulk_g2s(dst + dk + ns * cur.krb, cur.base + cur.offv + (size_t)(s0 >> 2) * 128, vbytes, &fb[b]);
                bulk_g2s(dst + dk + ns * (cur.krb + 32), cur.base + cur.offvp + (size_t)s0 * 8, pbytes, &fb[b]);
            }
            if (c0 && with_q)
                bulk_g2s(dst + qoff, static_cast<const uint8_t*>(p.q) + (size_t)cur_tile * qbytes,
                         (uint32_t)qbytes, &fb[b]);
        }
        return true;
    };
    auto issue_item = [&](int b, bool with_q) {
        if (!stage_item(b, with_q)) return false;
        advance();
        return true;
    };

    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    if (issuer) {
        for (int b = 0; b < nbuf; ++b) mbar_init(&fb[b], 1);
        fence_barrier_init();
        cur = load_meta(tile0);
        nxt = load_meta(tile0 + tstride);
        stage_item(0, false);  // KV of the first (packed) chunk before the grid dependency
    }
    asm volatile("griddepcontrol.wait;" ::: "memory");
    if (issuer && tile0 < p.units) {
        bulk_g2s(pbuf + qoff, static_cast<const uint8_t*>(p.q) + (size_t)tile0 * qbytes, (uint32_t)qbytes, &fb[0]);
        cur_zc = zc_of(tile0);  // known now: the cursor may move past tile0's packed chunks
        advance();
    }
    const U2xLane lc = u2x_lane(half);
    for (int i = threadIdx.x & 63; i < 4 * 512 / 16; i += 64)
        reinterpret_cast<uint4*>(scr + kXQDig)[i] = make_uint4(0u, 0u, 0u, 0u);
    __syncthreads();
    int b = 0, k = 0;
    uint32_t phase = 0;
    U2xRun run;
    int zcl_next = zc_of(tile0);
    for (int tile = tile0; tile < p.units; tile += tstride) {
        int n_t = 0, nslot_t = 0, hk = 0, krb = 0, Cp = 1, C = 1;
        const int zcl = zcl_next;
        zcl_next = zc_of(tile + tstride);
        IO* o = static_cast<IO*>(p.out) + (size_t)tile * p.g * kD;
        for (int c = 0; c < C; ++c) {
            if (c > 0 && !owned(c)) continue;
            mbar_wait(&fb[b], phase);
            __syncwarp();
            const uint8_t* st = pbuf + (size_t)b * p.slot_bytes;
            if (c == 0) {
                const TileHeader& th = *reinterpret_cast<const TileHeader*>(st);
                n_t = th.r[0];
                nslot_t = th.nslot;
                hk = th.off_k;
                krb = FULLK ? 32 : th.krow_bytes;
                int s0_, ns_;
                u2c_geom(nslot_t, 0, Cp, s0_, ns_);
                C = Cp + (zcl + kZcChunk - 1) / kZcChunk;
                if (ZC) build_q16<IO>(st + qoff, p.g, q16, lc);
            }
            if (k == 0 && issuer)  // look-ahead once the first item is in
                for (int j = 1; j < nbuf; ++j) issue_item(j, true);
            const int bprev = b == 0 ? nbuf - 1 : b - 1;
            auto refill = [&]() {
                if (issuer && k >= 1) issue_item(bprev, true);
            };
            if (ZC && c >= Cp) {
                const int j = c - Cp;
                zc_chunk_u2x<IO, BULK>(st, min(kZcChunk, zcl - kZcChunk * j), q16, p.g, 1 + pr, lc, run,
                                       !psplit && c == C - 1, o,
                                       BULK ? reinterpret_cast<IO*>(const_cast<uint8_t*>(st) + qoff) : o, refill);
            } else {
                int Cc, s0, ns;
                u2c_geom(nslot_t, c, Cc, s0, ns);
                U2xChunk ck;
                const bool own = owned(c);
                ck.n = own ? max(0, min(n_t - s0, ns)) : 0;
                ck.nslot = own ? ns : 0;
                ck.off_k = hk;
                ck.off_v = hk + ns * krb;
                ck.off_vp = hk + ns * (krb + 32);
                ck.krb = krb;
                ck.first = c == 0;
                ck.last = !psplit && c == C - 1;
                decode_tile_u2x<IO, kXNbMax, FULLK, BULK, true>(st, st + qoff, p.g, scr, o, 1 + pr, lc, refill, &ck,
                                                                 &run);
            }
            if (++b == nbuf) {
                b = 0;
                phase ^= 1u;
            }
            ++k;
        }
        if (psplit && lc.tig < p.g) {  // this rank's (o, max, sum) of the tile
            float* pr_row = p.partial + ((size_t)tile * p.g + lc.tig) * (kD + 2);
#pragma unroll
            for (int m = 0; m < 4; ++m) *reinterpret_cast<float2*>(pr_row + lc.ch0 + 4 * m) = run.o[m];
            if (half == 0 && lc.gid == 0) {
                pr_row[kD] = run.m;
                pr_row[kD + 1] = run.l;
            }
        }
    }
    if (BULK && lane == 0) bulk_wait0();
}

template <typename IO, bool FULLK>
static int launch_u2c(const rdkv_decode_args* a, cudaStream_t st, float* partial = nullptr, int split_rank = 0,
                      int split_world = 1) {
    const bool zc = a->zc_len != nullptr;
    const int qbytes = a->group * kD * (int)sizeof(IO);
    // header + channel table + perm, then <= 160 slots of K / V / params (a
    // Zone C chunk: 16 K + 16 V rows + 8 KB of spare), q rows at the end
    const int cslots = a->plan.max_slots < kU2MaxSlots ? ((a->plan.max_slots + 3) & ~3) : kU2MaxSlots;
    int body = 10 * kD + cslots * (32 + 32 + 8);
    const int zbody = 2 * kZcChunk * kZcKStride + 2 * kZcAuxWarp;  // Zone C chunk: K + V rows + both warps' spare
    const int slot = ((zc && zbody > kHeaderBytes + body ? zbody : kHeaderBytes + body) + qbytes + 127) & ~127;
    const int scratch = (kXPDig + kXNbMax * 256 + (zc ? kQ16Bytes : 0) + 127) & ~127;
    const DevAttrs da = dev_attrs();
    const int slack = 128;
    int W = 0, nbuf = 0;
    if (!pick_pairs(a->units, da.nsm, slot, scratch, da.smem_optin - slack, W, nbuf)) return RDKV_EINVAL;
    const size_t smem = W * kXMaxBuf * sizeof(uint64_t) + (size_t)W * (nbuf * slot + scratch) + slack;
    MmaParams p{a->arena, a->tile_offsets, a->tile_decode_bytes, a->q, a->out,
                static_cast<const __half*>(a->zc_k), static_cast<const __half*>(a->zc_v), a->zc_len,
                a->units, a->group, a->zc_cap, nbuf, W, slot, scratch, 0, 0, -1, -1, 0, 0};
    p.partial = partial;
    p.split_rank = split_rank;
    p.split_world = split_world;
    const bool bulk = (a->flags & RDKV_DECODE_OUT_HOST) != 0 && !partial;
    auto kern = zc ? (bulk ? decode_u2c_kernel<IO, FULLK, true, true> : decode_u2c_kernel<IO, FULLK, false, true>)
                   : (bulk ? decode_u2c_kernel<IO, FULLK, true, false> : decode_u2c_kernel<IO, FULLK, false, false>);
    static std::atomic<int> smem_set[4][kMaxDevices];
    set_smem_once(kern, (int)smem, smem_set[(zc ? 2 : 0) + (bulk ? 1 : 0)], da.dev);
    int blocks = (a->units + W - 1) / W;
    if (blocks > da.nsm) blocks = da.nsm;
    if (verbose_env())
        fprintf(stderr, "u2c: units %d zc %d pairs %d bufs %d slot %d scratch %d smem %zu grid %d\n", a->units, (int)zc,
                W, nbuf, slot, scratch, smem, blocks);
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(blocks);
    cfg.blockDim = dim3(32 * 2 * W);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    if (cudaLaunchKernelEx(&cfg, kern, p) != cudaSuccess) return RDKV_ECUDA;
    return launch_status();
}

// Zone C small enough to stage with each short tile (host-known bound)
// ---- Zone C prepass (append_new_token rows, trizone.cpp:261-303): one warp per
// unit computes, for each of its g query heads, the softmax state of the unit's
// appended fp16 rows alone — unnormalised o over the lane's channels 4 lane ..
// 4 lane + 3, the running max (log2 units, the decode kernels' convention) and
// the weight sum — into [units][g][d + 2] f32; the short-tile kernel (ZCN < 0)
// folds that row into its epilogue. The tile kernel keeps its 8 warp pairs per
// SM (no Zone C staging in its buffers); the rows are read once, here.
// Rows go in batches of 8 (loads in flight together). Logits of 4 heads are
// reduced together: two exchange stages halve the values a lane carries, three
// more finish the sum in 8-lane groups (head h in lanes 8h .. 8h + 7) — 6
// shuffles per row and group, 8 independent chains per batch; the batch max then
// rescales the running state once per head, and the weights reach every lane's
// PV channels by broadcast from lane 8h.
constexpr int kZcpUnits = 8;  // units (warps) per CTA
template <typename IO>
__device__ __forceinline__ void zcp_load_q(const IO* qrow, int lane, float (&q)[4]) {
    if constexpr (sizeof(IO) == 2) {
        const uint2 w = *reinterpret_cast<const uint2*>(qrow + 4 * lane);
        const float2 a = __half22float2(*reinterpret_cast<const __half2*>(&w.x));
        const float2 b = __half22float2(*reinterpret_cast<const __half2*>(&w.y));
        q[0] = a.x, q[1] = a.y, q[2] = b.x, q[3] = b.y;
    } else {
        const float4 v = *reinterpret_cast<const float4*>(qrow + 4 * lane);
        q[0] = v.x, q[1] = v.y, q[2] = v.z, q[3] = v.w;
    }
}
template <typename IO, int NG>  // NG: groups of 4 heads (1: g <= 4, 2: g <= 8)
__global__ void __launch_bounds__(32 * kZcpUnits) zc_partial_kernel(const IO* __restrict__ q,
                                                                    const __half* __restrict__ zk,
                                                                    const __half* __restrict__ zv,
                                                                    const int32_t* __restrict__ zlen, int units, int g,
                                                                    int cap, float* __restrict__ part) {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    asm volatile("griddepcontrol.wait;" ::: "memory");  // q and the appended rows come from earlier kernels
    const int lane = threadIdx.x & 31;
    const int u = blockIdx.x * kZcpUnits + (threadIdx.x >> 5);
    if (u >= units) return;
    constexpr float kScale = 0.08838834764831845f * 1.4426950408889634f;  // log2(e) / sqrt(d)
    int z = zlen[u];
    z = z < cap ? z : cap;
    float qv[4 * NG][4], o[4 * NG][4];
    float mrun[NG], lrun[NG];  // running max / sum of head 4 gr + (lane >> 3), per 8-lane group
#pragma unroll
    for (int h = 0; h < 4 * NG; ++h) {
        if (h < g)
            zcp_load_q(q + ((size_t)u * g + h) * kD, lane, qv[h]);
        else
            qv[h][0] = qv[h][1] = qv[h][2] = qv[h][3] = 0.0f;
        o[h][0] = o[h][1] = o[h][2] = o[h][3] = 0.0f;
    }
#pragma unroll
    for (int gr = 0; gr < NG; ++gr) {
        mrun[gr] = -INFINITY;
        lrun[gr] = 0.0f;
    }
    const __half* kr = zk + (size_t)u * cap * kD + 4 * lane;
    const __half* vr = zv + (size_t)u * cap * kD + 4 * lane;
    const bool hi16 = (lane & 16) != 0, hi8 = (lane & 8) != 0;
    constexpr int kBatch = 8;  // rows whose loads are in flight together
    for (int t0 = 0; t0 < z; t0 += kBatch) {
        uint2 kb[kBatch], vb[kBatch];
#pragma unroll
        for (int j = 0; j < kBatch; ++j) {
            kb[j] = vb[j] = make_uint2(0u, 0u);
            if (t0 + j < z) {
                kb[j] = *reinterpret_cast<const uint2*>(kr + (size_t)(t0 + j) * kD);
                vb[j] = *reinterpret_cast<const uint2*>(vr + (size_t)(t0 + j) * kD);
            }
        }
        // phase 1: the batch's logits (independent chains), head 4 gr + (lane >> 3)
        float lgt[NG][kBatch];
#pragma unroll
        for (int j = 0; j < kBatch; ++j) {
            const float2 k01 = __half22float2(*reinterpret_cast<const __half2*>(&kb[j].x));
            const float2 k23 = __half22float2(*reinterpret_cast<const __half2*>(&kb[j].y));
#pragma unroll
            for (int gr = 0; gr < NG; ++gr) {
                float sp[4];
#pragma unroll
                for (int hh = 0; hh < 4; ++hh) {
                    const float* qq = qv[4 * gr + hh];
                    sp[hh] = fmaf(qq[3], k23.y, fmaf(qq[2], k23.x, fmaf(qq[1], k01.y, qq[0] * k01.x)));
                }
                float a0 = hi16 ? sp[2] : sp[0], a1 = hi16 ? sp[3] : sp[1];
                const float b0 = hi16 ? sp[0] : sp[2], b1 = hi16 ? sp[1] : sp[3];
                a0 += __shfl_xor_sync(0xffffffffu, b0, 16);
                a1 += __shfl_xor_sync(0xffffffffu, b1, 16);
                float c = (hi8 ? a1 : a0) + __shfl_xor_sync(0xffffffffu, hi8 ? a0 : a1, 8);
                c += __shfl_xor_sync(0xffffffffu, c, 4);
                c += __shfl_xor_sync(0xffffffffu, c, 2);
                c += __shfl_xor_sync(0xffffffffu, c, 1);
                lgt[gr][j] = t0 + j < z ? c * kScale : -INFINITY;
            }
        }
        // phase 2: per head, the batch max rescales the running state once; weights
        // of the batch's rows; PV for every head of the group over this lane's channels
#pragma unroll
        for (int gr = 0; gr < NG; ++gr) {
            float bm = lgt[gr][0];
#pragma unroll
            for (int j = 1; j < kBatch; ++j) bm = fmaxf(bm, lgt[gr][j]);
            const float mn = fmaxf(mrun[gr], bm);
            const float al = ex2_approx(mrun[gr] - mn);
            float pj[kBatch], ps = 0.0f;
#pragma unroll
            for (int j = 0; j < kBatch; ++j) {
                pj[j] = ex2_approx(lgt[gr][j] - mn);
                ps += pj[j];
            }
            lrun[gr] = fmaf(lrun[gr], al, ps);
            mrun[gr] = mn;
#pragma unroll
            for (int hh = 0; hh < 4; ++hh) {
                float* oh = o[4 * gr + hh];
                const float ah = __shfl_sync(0xffffffffu, al, 8 * hh);
                oh[0] *= ah;
                oh[1] *= ah;
                oh[2] *= ah;
                oh[3] *= ah;
#pragma unroll
                for (int j = 0; j < kBatch; ++j) {
                    const float pw = __shfl_sync(0xffffffffu, pj[j], 8 * hh);
                    const float2 v01 = __half22float2(*reinterpret_cast<const __half2*>(&vb[j].x));
                    const float2 v23 = __half22float2(*reinterpret_cast<const __half2*>(&vb[j].y));
                    oh[0] = fmaf(pw, v01.x, oh[0]);
                    oh[1] = fmaf(pw, v01.y, oh[1]);
                    oh[2] = fmaf(pw, v23.x, oh[2]);
                    oh[3] = fmaf(pw, v23.y, oh[3]);
                }
            }
        }
    }
#pragma unroll
    for (int h = 0; h < 4 * NG; ++h) {
        if (h >= g) continue;
        float* row = part + ((size_t)u * g + h) * (kD + 2);
        *reinterpret_cast<float2*>(row + 4 * lane) = make_float2(o[h][0], o[h][1]);
        *reinterpret_cast<float2*>(row + 4 * lane + 2) = make_float2(o[h][2], o[h][3]);
        if (lane == 8 * (h & 3)) {
            row[kD] = mrun[h >> 2];
            row[kD + 1] = lrun[h >> 2];
        }
    }
}

template <typename IO>
static int launch_zc_partial(const rdkv_decode_args* a, cudaStream_t st) {
    cudaLaunchConfig_t cfg{};
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cfg.stream = st;
    cfg.gridDim = dim3((a->units + kZcpUnits - 1) / kZcpUnits);
    cfg.blockDim = dim3(32 * kZcpUnits);
    auto kern = a->group > 4 ? zc_partial_kernel<IO, 2> : zc_partial_kernel<IO, 1>;
    const cudaError_t e =
        cudaLaunchKernelEx(&cfg, kern, static_cast<const IO*>(a->q), static_cast<const __half*>(a->zc_k),
                           static_cast<const __half*>(a->zc_v), a->zc_len, a->units, a->group, a->zc_cap,
                           static_cast<float*>(a->workspace));
    return e == cudaSuccess ? RDKV_OK : RDKV_ECUDA;
}

// Zone C through the prepass: short uniform-2-bit tiles, the whole arena in one
// launch (no unit subset), device output, and the caller's workspace holds one
// [units][g][d + 2] f32 row set (rdkv_cuda_decode_workspace(units, g, d, 2) / 2).
// The experiments build can force the fused variants (RDKV_DECODE_ZC_FUSED=1).
static bool zc_prepass_ok(const rdkv_decode_args* a) {
#ifdef RDKV_DECODE_EXPERIMENTS
    static const char* fused_env = getenv("RDKV_DECODE_ZC_FUSED");
    if (fused_env && atoi(fused_env) == 1) return false;
#endif
    // (a known bound of <= kZcFused rows keeps the fused variant: staging <= 4 rows with
    // each tile costs less than the prepass launch)
    if ((a->flags & RDKV_DECODE_ZC_BOUND) && a->zc_bound <= kZcFused) return false;
    return a->zc_len && !a->unit_ids && a->workspace && a->group <= 8 &&
           a->workspace_bytes >= sizeof(float) * (size_t)a->units * a->group * (kD + 2) && a->plan.uniform2 != 3 &&
           a->plan.max_slots <= kU2MaxSlots && !(a->flags & RDKV_DECODE_OUT_HOST);
}

static bool zc_fusable(const rdkv_decode_args* a) {
    return a->zc_len && (a->flags & RDKV_DECODE_ZC_BOUND) && a->zc_bound <= kZcFusedMax;
}
// groups of 5..8 heads run as two 4-head passes in the short-tile kernel only
// (the chunked kernel's running softmax state is per 4-head lane group)
static bool u2x_group_ok(const rdkv_decode_args* a) {
    if (a->plan.uniform2 == 3)  // MIX tiles: short-tile kernel only, no Zone C
        return a->group <= 8 && a->plan.max_slots <= kU2MaxSlots && !a->zc_len;
    if (a->group <= 4) return true;
    return a->group <= 8 && a->plan.max_slots <= kU2MaxSlots && (!a->zc_len || zc_fusable(a) || zc_prepass_ok(a));
}

template <typename IO, int NBMAX, bool FULLK>
static int launch_u2x_t(const rdkv_decode_args* a, cudaStream_t st, int max_blocks = 0) {
    const int qbytes = a->group * kD * (int)sizeof(IO);
    const bool zcp = zc_prepass_ok(a);  // Zone C folded from the prepass rows (no staging)
    const bool zcf = !zcp && zc_fusable(a);
    const bool zc16 = zcf && a->zc_bound > kZcFused;  // the long-generation variant (16 fused rows)
    const int slot = (a->plan.max_decode_bytes + (zcf ? zc_stage(zc16 ? kZcFusedMax : kZcFused) : 0) + qbytes + 127) & ~127;
    const bool mix = a->plan.uniform2 == 3;  // some tiles carry a few 4-bit rows / channels
    const int scratch = (kXPDig + (mix ? 512 + kMixMaxRows * 16 : 0) + NBMAX * 256 + 127) & ~127;
    const DevAttrs da = dev_attrs();
    const int smem_max = da.smem_optin, nsm = da.nsm;
    // fragment over-reads of ragged blocks land in the following smem region
    // (K rows: < 256 B past a tile's K rows; the last region is scratch)
    const int slack = 128;
    int W = 0, nbuf = 0;
    if (!pick_pairs(a->units, nsm, slot, scratch, smem_max - slack, W, nbuf)) return RDKV_EINVAL;
    size_t smem = W * kXMaxBuf * sizeof(uint64_t) + (size_t)W * (nbuf * slot + scratch) + slack;
    MmaParams p{a->arena, a->tile_offsets, a->tile_decode_bytes, a->q, a->out,
                zcf ? static_cast<const __half*>(a->zc_k) : nullptr, zcf ? static_cast<const __half*>(a->zc_v) : nullptr,
                zcf ? a->zc_len : nullptr, a->units, a->group, zcf ? a->zc_cap : 0, nbuf, W, slot, scratch, 0, 0, -1, -1,
                0, 0, a->unit_ids};
    static const char* smsp_env = experiment_knob("RDKV_DECODE_SMSP");
    if (smsp_env) p.smsp_pairs = atoi(smsp_env);
    static const char* nenv = experiment_knob("RDKV_DECODE_NULL");
    const int mode = nenv ? atoi(nenv) : 0;
    const bool bulk = (a->flags & RDKV_DECODE_OUT_HOST) != 0;
    const bool g8 = a->group > 4;
    if (zcp) {
        if (int rc = launch_zc_partial<IO>(a, st)) return rc;
        p.partial = static_cast<float*>(a->workspace);
    }
    auto kern = zcp ? (g8 ? decode_u2x_kernel<IO, NBMAX, FULLK, 0, false, false, -1, true>
                          : decode_u2x_kernel<IO, NBMAX, FULLK, 0, false, false, -1>)
              : mix ? (g8 ? (bulk ? decode_u2x_kernel<IO, NBMAX, FULLK, 0, true, false, 0, true, true>
                                  : decode_u2x_kernel<IO, NBMAX, FULLK, 0, false, false, 0, true, true>)
                          : (bulk ? decode_u2x_kernel<IO, NBMAX, FULLK, 0, true, false, 0, false, true>
                                  : decode_u2x_kernel<IO, NBMAX, FULLK, 0, false, false, 0, false, true>))
              : g8 ? (zcf ? (zc16 ? (bulk ? decode_u2x_kernel<IO, NBMAX, FULLK, 0, true, false, kZcFusedMax, true>
                                          : decode_u2x_kernel<IO, NBMAX, FULLK, 0, false, false, kZcFusedMax, true>)
                                  : (bulk ? decode_u2x_kernel<IO, NBMAX, FULLK, 0, true, false, kZcFused, true>
                                          : decode_u2x_kernel<IO, NBMAX, FULLK, 0, false, false, kZcFused, true>))
                          : (bulk ? decode_u2x_kernel<IO, NBMAX, FULLK, 0, true, false, 0, true>
                                  : decode_u2x_kernel<IO, NBMAX, FULLK, 0, false, false, 0, true>))
              : zcf ? (zc16 ? (bulk ? decode_u2x_kernel<IO, NBMAX, FULLK, 0, true, false, kZcFusedMax>
                                    : decode_u2x_kernel<IO, NBMAX, FULLK, 0, false, false, kZcFusedMax>)
                            : (bulk ? decode_u2x_kernel<IO, NBMAX, FULLK, 0, true, false, kZcFused>
                                    : decode_u2x_kernel<IO, NBMAX, FULLK, 0, false, false, kZcFused>))
              : bulk ? decode_u2x_kernel<IO, NBMAX, FULLK, 0, true>
#ifdef RDKV_DECODE_EXPERIMENTS
              : mode == 1 ? decode_u2x_kernel<IO, NBMAX, FULLK, 1>
              : mode == 2 ? decode_u2x_kernel<IO, NBMAX, FULLK, 2>
#endif
                          : decode_u2x_kernel<IO, NBMAX, FULLK, 0>;
    static std::atomic<int> smem_set[20][kMaxDevices];  // one slot per instantiation above
    set_smem_once(kern, (int)smem,
                  smem_set[zcp ? 18 + (g8 ? 1 : 0)
                           : mix ? 10 + (g8 ? 2 : 0) + (bulk ? 1 : 0)
                           : g8 ? (zc16 ? 14 + (bulk ? 1 : 0) : 6 + (zcf ? 2 : 0) + (bulk ? 1 : 0))
                           : zcf ? (zc16 ? 16 + (bulk ? 1 : 0) : 4 + (bulk ? 1 : 0))
                           : bulk ? 3 : mode == 1 ? 1 : mode == 2 ? 2 : 0],
                  da.dev);
    int blocks = (a->units + W - 1) / W;
    if (blocks > nsm) blocks = nsm;
    // The SM's W pairs run as W / 2 CTAs of two pairs: a CTA retires as soon as
    // its own two pairs are done, so under programmatic dependent launch the
    // next step's CTAs take its slots while the SM's slower pairs still run
    // (measured 13.5 -> 12.9 us on the 4096-tile step; 1 CTA of 8 pairs: 13.5,
    // 4 pairs per CTA: 13.1). RDKV_DECODE_CTAS (experiments build) forces c CTAs per SM.
    static const char* ctas_env = experiment_knob("RDKV_DECODE_CTAS");
    const int ctas = ctas_env ? atoi(ctas_env) : (W % 2 == 0 ? W / 2 : 1);
    if (ctas > 1 && W % ctas == 0 && max_blocks == 0) {
        const int c = ctas;
        p.W = W = W / c;
        smem = W * kXMaxBuf * sizeof(uint64_t) + (size_t)W * (nbuf * slot + scratch) + slack;
        blocks = (a->units + W - 1) / W;
        if (blocks > c * nsm) blocks = c * nsm;
    }
    if (max_blocks > 0) {  // split step: the SMs the general kernel leaves free
        p.concurrent = 1;
        if (blocks > max_blocks) blocks = max_blocks;
    }
    // One pair per CTA (RDKV_DECODE_CTA=1): the same persistent pairs, but each
    // retires its own CTA, so under programmatic dependent launch the next
    // kernel's CTAs take a pair's smem / warp slots as soon as it finishes
    // instead of when the SM's slowest pair does.
    static const char* cta_env = experiment_knob("RDKV_DECODE_CTA");
    if (cta_env && atoi(cta_env) == 1 && W > 1 && mode == 0 && !zcf && !g8 && !mix && max_blocks == 0) {
        const size_t smem1 = kXMaxBuf * sizeof(uint64_t) + (size_t)2 * slot + scratch + slack;
        auto k1 = bulk ? decode_u2x_kernel<IO, NBMAX, FULLK, 0, true, true> : decode_u2x_kernel<IO, NBMAX, FULLK, 0, false, true>;
        static std::atomic<int> smem1_set[2][kMaxDevices];
        set_smem_once(k1, (int)smem1, smem1_set[bulk ? 1 : 0], da.dev);
        int per_sm = 0;
        const cudaError_t oe = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k1, 64, smem1);
        if (verbose_env()) fprintf(stderr, "u2x: per-pair CTAs: smem %zu -> %d per SM (err %d)\n", smem1, per_sm, (int)oe);
        if (oe == cudaSuccess && per_sm >= W) {
            kern = k1;
            p.W = W = 1;
            p.R = nbuf = 2;
            smem = smem1;
            blocks = a->units < nsm * per_sm ? a->units : nsm * per_sm;
        }
    }
    if (verbose_env())
        fprintf(stderr, "u2x: units %d nbmax %d pairs %d bufs %d slot %d scratch %d smem %zu grid %d\n", a->units,
                NBMAX, W, nbuf, slot, scratch, smem, blocks);
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(blocks);
    cfg.blockDim = dim3(32 * 2 * W);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    if (cudaLaunchKernelEx(&cfg, kern, p) != cudaSuccess) return RDKV_ECUDA;
    return launch_status();
}

template <typename IO, bool FULLK>
static int launch_u2x_k(const rdkv_decode_args* a, cudaStream_t st, int max_blocks) {
    // long tiles or Zone C rows beyond the fused bound: the chunked kernel
    if (a->plan.max_slots > kU2MaxSlots || (a->zc_len && !zc_fusable(a) && !zc_prepass_ok(a)))
        return launch_u2c<IO, FULLK>(a, st);
    const int nb = (a->plan.max_slots + 31) / 32;  // 32-token blocks of the largest tile
    if (nb <= 2) return launch_u2x_t<IO, 2, FULLK>(a, st, max_blocks);
    if (nb <= 4) return launch_u2x_t<IO, 4, FULLK>(a, st, max_blocks);
    return launch_u2x_t<IO, kXNbMax, FULLK>(a, st, max_blocks);
}

template <typename IO>
static int launch_u2x(const rdkv_decode_args* a, cudaStream_t st, int max_blocks = 0) {
    // plan.uniform2 == 2: every tile also keeps all 128 K channels (identity channel_perm)
    return a->plan.uniform2 == 2 ? launch_u2x_k<IO, true>(a, st, max_blocks)
                                 : launch_u2x_k<IO, false>(a, st, max_blocks);
}

}  // namespace rdkv_b200

using namespace rdkv_b200;

namespace rdkv_b200 {

// Shared-memory footprint of the general body (launch_t) with one consumer warp and
// one ring slot: the whole tile is staged at once, so long or wide tiles may not fit.
static size_t general_min_smem(const rdkv_decode_args* a) {
    const int NT = a->group <= 4 ? 1 : 2;
    const int qbytes = a->group * kD * (a->io_dtype == RDKV_F16 ? 2 : 4);
    const size_t slot = (size_t)(a->plan.max_decode_bytes + qbytes + 127) & ~(size_t)127;
    const int qsteps = (a->plan.max_kq_slots + 31) / 32;
    const int vsteps = (a->plan.max_slots + 31) / 32 + 2;
    const int steps = qsteps > vsteps ? qsteps : vsteps;
    size_t scratch = kDigitBytesOff + (size_t)steps * 2 * NT * 8 * 32;
    const int s32 = ((a->plan.max_slots + 31) / 32) * 32;
    const int lg_stride = (s32 > kD ? s32 : kD) + 32 / (4 * NT);
    scratch += (size_t)4 * NT * lg_stride * 4;
    if (a->plan.max_zone_b_rows > 0) scratch += (size_t)4 * NT * a->plan.max_zone_b_rows * 4;
    if (a->zc_len) scratch += (size_t)4 * NT * a->zc_cap * 4;
    scratch = (scratch + 127) & ~(size_t)127;
    return 2 * kMaxR * sizeof(uint64_t) + slot + scratch + 4096;
}

bool mma_supported(const rdkv_decode_args* a) {
    if (a->head_dim != kD || a->group > 8 || !a->tile_decode_bytes) return false;
    if (a->zc_len && a->zc_cap > 1024) return false;
    const rdkv_decode_plan& p = a->plan;
    // uniform 2-bit tiles of any length: u2x (<= 160 slots) or its chunked variant
    if (p.uniform2 && p.max_decode_bytes > 0 && u2x_group_ok(a)) return true;
    // mixed 2/4-bit tiles of any length: the chunked split-K kernel (decode_u24)
    if (p.mix24 && p.max_decode_bytes > 0 && !a->zc_len && !(p.uniform2 && p.max_slots <= kU2MaxSlots)) return true;
    if (p.max_decode_bytes <= 0 || p.max_slots > kMaxSlots || p.max_zone_b_rows > kMaxSlots) return false;
    return general_min_smem(a) <= (size_t)dev_attrs().smem_optin;  // else the CUDA-core kernel
}

template <int NT, typename IO, bool U2>
static int launch_t(const rdkv_decode_args* a, cudaStream_t st, int* grid_out = nullptr, int max_w = kMaxW) {
    const int qbytes = a->group * kD * (int)sizeof(IO);
    const int slot = (a->plan.max_decode_bytes + qbytes + 127) & ~127;
    // per-warp scratch: head | digits | logits (aliased by the PV accumulators) | p16 | zl
    const int qsteps = (a->plan.max_kq_slots + 31) / 32;
    const int vsteps = (a->plan.max_slots + 31) / 32 + 2;
    const int steps = qsteps > vsteps ? qsteps : vsteps;
    int scratch = kDigitBytesOff + steps * 2 * NT * 8 * 32;
    const int off_lg = scratch;
    // stride == 32/G4 (mod 32): the G4 heads x 32/G4 tokens of a warp hit distinct banks
    const int s32 = ((a->plan.max_slots + 31) / 32) * 32;
    const int lg_stride = (s32 > kD ? s32 : kD) + 32 / (4 * NT);
    scratch += 4 * NT * lg_stride * 4;
    int off_p16 = -1, off_zl = -1;
    const int max_r16 = a->plan.max_zone_b_rows;
    if (max_r16 > 0) {
        off_p16 = scratch;
        scratch += 4 * NT * max_r16 * 4;
    }
    if (a->zc_len) {
        off_zl = scratch;
        scratch += 4 * NT * a->zc_cap * 4;
    }
    scratch = (scratch + 127) & ~127;
    int dev = 0, smem_max = 0, nsm = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&smem_max, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    const int head = 2 * kMaxR * (int)sizeof(uint64_t);
    const int slack = 4096;  // fragment over-reads past the last ring slot (masked by zero digits)
    // consumers W and ring slots R = W + lookahead (2, else 1, else 0), as many as fit
    int W = max_w < kMaxW ? (max_w > 0 ? max_w : 1) : kMaxW, R = 0;
    bool fits = false;
    for (; W >= 1 && !fits; --W) {
        for (int look = 2; look >= 0 && !fits; --look) {
            R = W + look > kMaxR ? kMaxR : W + look;
            fits = head + (size_t)R * slot + (size_t)W * scratch + slack <= (size_t)smem_max;
        }
        if (fits) break;
    }
    if (!fits) return RDKV_EINVAL;
    const size_t smem = head + (size_t)R * slot + (size_t)W * scratch + slack;
    MmaParams p{a->arena, a->tile_offsets, a->tile_decode_bytes, a->q, a->out,
                static_cast<const __half*>(a->zc_k), static_cast<const __half*>(a->zc_v), a->zc_len,
                a->units, a->group, a->zc_cap, R, W, slot, scratch, off_lg, lg_stride, off_p16, off_zl, max_r16, 0,
                a->unit_ids};
    auto kern = decode_mma_kernel<NT, IO, U2>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int blocks = (a->units + W - 1) / W;
    if (blocks > nsm) blocks = nsm;
    if (grid_out) *grid_out = blocks;
    kern<<<blocks, 32 * (W + 1), smem, st>>>(p);
    return launch_status();
}

// Sequence split (SURVEY.md §8(e) optional merge): this rank's share of every
// uniform-2-bit tile (its chunks c % world == rank) as unnormalised partials.
int launch_partial(const rdkv_decode_args* a, int rank, int world, float* partial, cudaStream_t st) {
    if (!a->plan.uniform2 || a->plan.uniform2 == 3 || a->group > 4 || !a->tile_decode_bytes || a->head_dim != kD)
        return RDKV_EINVAL;
    if (a->zc_len && a->zc_cap > 1 << 20) return RDKV_EINVAL;
    const bool f16 = a->io_dtype == RDKV_F16;
    rdkv_decode_args b = *a;
    b.unit_ids = nullptr;
    if (a->plan.uniform2 == 2)
        return f16 ? launch_u2c<__half, true>(&b, st, partial, rank, world) : launch_u2c<float, true>(&b, st, partial, rank, world);
    return f16 ? launch_u2c<__half, false>(&b, st, partial, rank, world) : launch_u2c<float, false>(&b, st, partial, rank, world);
}

// out = sum_r 2^(m_r - M) o_r / sum_r 2^(m_r - M) l_r over nparts partials
// [nparts][units * g][d + 2] (m in log2 units, as the kernels keep it).
// One warp per row: lane r holds part r's (max, sum) and weight, the weights
// and the denominator are combined in part order (fixed, deterministic), and
// every channel's S loads are independent (in flight together). Launched with
// programmatic dependent launch: its CTAs are resident while the producing
// kernel drains and start at griddepcontrol.wait.
constexpr int kMergeRows = 8;        // rows (warps) per CTA
constexpr int kMergeFastParts = 16;  // parts whose loads are all in flight at once
template <typename IO>
__global__ void __launch_bounds__(32 * kMergeRows) merge_partials_kernel(const float* __restrict__ part, int nparts,
                                                                         int rows, int d, IO* __restrict__ out) {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    const int lane = threadIdx.x & 31;
    const int row = blockIdx.x * kMergeRows + (threadIdx.x >> 5);
    if (row >= rows) return;
    const size_t stride = (size_t)rows * (d + 2);
    const float* base = part + (size_t)row * (d + 2);
    // d = 128, <= 16 parts: every part's channels (2 lane, + 1, 64 + 2 lane, + 1;
    // 8-B aligned rows) are loaded before anything waits on them
    const bool fast = d == 128 && nparts <= kMergeFastParts;
    float2 xs[kMergeFastParts], ys[kMergeFastParts];
    if (fast) {
#pragma unroll
        for (int r = 0; r < kMergeFastParts; ++r)
            if (r < nparts) {
                xs[r] = *reinterpret_cast<const float2*>(base + r * stride + 2 * lane);
                ys[r] = *reinterpret_cast<const float2*>(base + r * stride + 64 + 2 * lane);
            }
    }
    float m = -INFINITY, l = 0.0f;
    if (lane < nparts) {
        m = base[lane * stride + d];
        l = base[lane * stride + d + 1];
        if (!(l > 0.0f)) m = -INFINITY;
    }
    float M = m;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, o));
    const float w = (lane < nparts && l > 0.0f) ? exp2f(m - M) : 0.0f;
    float L = 0.0f;
    for (int r = 0; r < nparts; ++r) L += __shfl_sync(0xffffffffu, w * l, r);
    const float inv = L > 0.0f ? 1.0f / L : 0.0f;
    if (fast) {
        float2 a = make_float2(0.0f, 0.0f), b = make_float2(0.0f, 0.0f);
#pragma unroll
        for (int r = 0; r < kMergeFastParts; ++r)
            if (r < nparts) {
                const float wr = __shfl_sync(0xffffffffu, w, r);
                if (wr != 0.0f) {
                    a.x += wr * xs[r].x;
                    a.y += wr * xs[r].y;
                    b.x += wr * ys[r].x;
                    b.y += wr * ys[r].y;
                }
            }
        IO* o = out + (size_t)row * d;
        o[2 * lane] = (IO)(a.x * inv);
        o[2 * lane + 1] = (IO)(a.y * inv);
        o[64 + 2 * lane] = (IO)(b.x * inv);
        o[65 + 2 * lane] = (IO)(b.y * inv);
        return;
    }
    for (int c = lane; c < d; c += 32) {
        float acc = 0.0f;
#pragma unroll 4
        for (int r = 0; r < nparts; ++r) {
            const float wr = __shfl_sync(0xffffffffu, w, r);
            const float v = base[r * stride + c];
            if (wr != 0.0f) acc += wr * v;
        }
        out[(size_t)row * d + c] = (IO)(acc * inv);
    }
}

// more than 32 parts (a wide sequence split): one CTA per row, parts in order
template <typename IO>
__global__ void merge_partials_wide_kernel(const float* __restrict__ part, int nparts, int rows, int d,
                                           IO* __restrict__ out) {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    const int row = blockIdx.x;
    if (row >= rows) return;
    const size_t stride = (size_t)rows * (d + 2);
    float M = -INFINITY;
    for (int r = 0; r < nparts; ++r) {
        const float* pr = part + r * stride + (size_t)row * (d + 2);
        if (pr[d + 1] > 0.0f) M = fmaxf(M, pr[d]);
    }
    float L = 0.0f;
    for (int r = 0; r < nparts; ++r) {
        const float* pr = part + r * stride + (size_t)row * (d + 2);
        if (pr[d + 1] > 0.0f) L += exp2f(pr[d] - M) * pr[d + 1];
    }
    const float inv = L > 0.0f ? 1.0f / L : 0.0f;
    for (int c = threadIdx.x; c < d; c += blockDim.x) {
        float acc = 0.0f;
        for (int r = 0; r < nparts; ++r) {
            const float* pr = part + r * stride + (size_t)row * (d + 2);
            if (pr[d + 1] > 0.0f) acc += exp2f(pr[d] - M) * pr[c];
        }
        out[(size_t)row * d + c] = (IO)(acc * inv);
    }
}

template <typename IO>
static int launch_merge_t(const float* part, int nparts, int rows, int d, IO* out, cudaStream_t st) {
    cudaLaunchConfig_t cfg{};
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cfg.stream = st;
    cudaError_t e;
    if (nparts <= 32) {
        cfg.gridDim = dim3((rows + kMergeRows - 1) / kMergeRows);
        cfg.blockDim = dim3(32 * kMergeRows);
        e = cudaLaunchKernelEx(&cfg, merge_partials_kernel<IO>, part, nparts, rows, d, out);
    } else {
        cfg.gridDim = dim3(rows);
        cfg.blockDim = dim3(128);
        e = cudaLaunchKernelEx(&cfg, merge_partials_wide_kernel<IO>, part, nparts, rows, d, out);
    }
    return e == cudaSuccess ? RDKV_OK : RDKV_ECUDA;
}

int launch_merge(const float* part, int nparts, int rows, int d, void* out, int io, cudaStream_t st) {
    if (io == RDKV_F16) return launch_merge_t(part, nparts, rows, d, static_cast<__half*>(out), st);
    return launch_merge_t(part, nparts, rows, d, static_cast<float*>(out), st);
}

// ============================================================================
// Mixed 2/4/8-bit tiles of any length (the configs[3] budget sweep: heavy
// hitters and outlier K channels leave ~80-110 K channels at 2 bits and the
// rest at 4 bits, V rows at 2 and 4 bits and a few at 8, 64 .. 3,100 token
// slots per tile), decoded with split-K across warp pairs
// (packed_decode_step, trizone.cpp:251-305):
//   * a tile's slots are cut into V-class-homogeneous chunks of 128 (2-bit),
//     64 (4-bit) or 32 (8-bit) slots, starting at multiples of 32 slots inside
//     the class so the V swizzle phase of every 4-token group is preserved;
//   * a tile's chunks are dealt to S parts (part r takes chunks r, r + S, ...);
//     each (tile, part) item runs on one warp pair, which stages its chunks by
//     TMA (K rows as the four slot-transposed runs, V rows, V parameters; the
//     tile header, channel table and q rows with its first chunk), folds them
//     into an online softmax and writes an unnormalised partial (o, max in
//     log2 units, weight sum) that merge_partials_kernel combines (S == 1:
//     the pair writes the output itself);
//   * QK: one k-step per 32 K slots of a class: 2-bit channels with the
//     in-place 2-bit masks (q~ prescaled 4^(3 - t), as u2x), 4-bit with nibble
//     masks (prescaled 4 * 16^(1 - t'), as MIX), 8-bit raw bytes (prescaled
//     64); three balanced s8 digits of q~, int8 MMAs;
//   * PV: 2-bit chunks as u2x; 4-bit chunks with nibble masks whose rows
//     gid / gid + 8 are the lo / hi nibble channels of one byte column, 8-bit
//     chunks with the two adjacent byte columns — chosen so a lane's output
//     channels (ch0 + 4m, + 1) are the same in every class.
// GQA groups of 5..8 heads run as two 4-head passes over each staged chunk.
constexpr int kU24MaxK = 6;                              // k-steps of 32 K slots (c2 + c4 + c8 <= 128 -> <= 6)
constexpr int kU24QDig = kXQDig;                         // q~ digit blocks: kU24MaxK x 512 B
constexpr int kU24PDig = kU24QDig + kU24MaxK * 512;      // p~ digit blocks: 4 x 256 B
constexpr int kU24Scratch = kU24PDig + 4 * 256;
constexpr int kU24MaxParts = 16;                         // split-K parts per tile
__host__ __device__ constexpr int u24_chunk_slots(int cls) { return cls == 0 ? 128 : cls == 1 ? 96 : 32; }
__host__ __device__ constexpr int u24_vrow_bytes(int cls) { return cls == 0 ? 32 : cls == 1 ? 64 : 128; }

// Per-tile chunk layout: class c has C[c] chunks of u24_chunk_slots(c) slots
// over its pad4(r[c]) slots (the last one ragged).
struct U24Tile {
    int r[3], C[3];
    int n2, n4, n8;  // K k-steps per class
    float vmax2;     // header bound on the 2-bit V scales
};
__host__ __device__ inline void u24_tile(const int* r, U24Tile& t) {
    for (int c = 0; c < 3; ++c) {
        t.r[c] = r[c];
        t.C[c] = (pad4(r[c]) + u24_chunk_slots(c) - 1) / u24_chunk_slots(c);
    }
}
__host__ __device__ inline int u24_nchunks(const U24Tile& t) { return t.C[0] + t.C[1] + t.C[2]; }
struct U24Geom {
    int cls, s0, ns, n;  // V class, first slot (of the tile), slots (multiple of 4), valid slots
    int li0;             // first row inside the class
};
__host__ __device__ inline U24Geom u24_chunk(const U24Tile& t, int k) {
    U24Geom g;  // (explicit selects: no dynamically indexed arrays, they would live in local memory)
    const int P0 = pad4(t.r[0]), P1 = pad4(t.r[1]);
    int rc;
    if (k < t.C[0]) {
        g.cls = 0;
        g.li0 = k * u24_chunk_slots(0);
        g.s0 = g.li0;
        rc = t.r[0];
    } else if (k < t.C[0] + t.C[1]) {
        g.cls = 1;
        g.li0 = (k - t.C[0]) * u24_chunk_slots(1);
        g.s0 = P0 + g.li0;
        rc = t.r[1];
    } else {
        g.cls = 2;
        g.li0 = (k - t.C[0] - t.C[1]) * u24_chunk_slots(2);
        g.s0 = P0 + P1 + g.li0;
        rc = t.r[2];
    }
    g.ns = min(g.cls == 0 ? u24_chunk_slots(0) : g.cls == 1 ? u24_chunk_slots(1) : u24_chunk_slots(2), pad4(rc) - g.li0);
    g.n = min(g.ns, rc - g.li0);
    return g;
}

struct U24Meta {  // a tile's staging geometry, read from its header in global memory
    const uint8_t* base;
    int nslot, hk, krb, offvp, offv[3], r[3];
};
struct U24Issuer {
    U24Meta cur, nxt;
    U24Tile t;
    int item, c, n;
    int nxt_item;            // the item after `item` (its header is loaded one item ahead)
    int done;                // the end-of-work marker has been staged
    int bitem[kXMaxBuf];     // per buffer: the staged chunk's (item, chunk), item -1 = no more work
    int bc[kXMaxBuf];
};

// One chunk for one 4-head group. `first`: this pair's first chunk of the tile
// (header, channel table and q staged; builds the q~ digits and resets `run`).
template <typename IO, typename AfterSync1>
__device__ __forceinline__ void decode_chunk_u24(const uint8_t* __restrict__ t, const uint8_t* __restrict__ qs, int g,
                                                 uint8_t* __restrict__ scr, int bar, const U2xLane& L,
                                                 AfterSync1&& after_sync1, const U24Geom& ck, bool first, int krb,
                                                 const uint8_t* __restrict__ kb, const uint8_t* __restrict__ vb,
                                                 const float2* __restrict__ vparam, U2xRun& run, U24Tile& tl) {
    constexpr int NBW = 2;  // <= 128 slots per chunk: <= 4 blocks of 32, two per warp
    const int gid = L.gid, tig = L.tig, half = L.half;
    const bool hv = tig < g;
    PairX& xg = *reinterpret_cast<PairX*>(scr);
    float* vmx = reinterpret_cast<float*>(scr) + sizeof(PairX) / 4;  // [2] chunk V-scale maxima (4/8-bit chunks)
    uint8_t* qdig = scr + kU24QDig;
    uint8_t* pdig = scr + kU24PDig;
    const int nslot = ck.ns, n = ck.n;
    const int nb = (n + 31) >> 5;
    const int mynb = (nb + 1 - half) >> 1;
    const int Q = nslot >> 2;
    constexpr float kInvSqrtD = 0.08838834764831845f;
    constexpr float kLog2e = 1.4426950408889634f;
    constexpr int QROW = kD * (int)sizeof(IO);
    if (first) {
        const TileHeader& h = *reinterpret_cast<const TileHeader*>(t);
        const float* chanf = reinterpret_cast<const float*>(t + kHeaderBytes);
        const uint16_t* perm = reinterpret_cast<const uint16_t*>(t + kHeaderBytes + 8 * h.kslots);
        const int n2 = h.kslot_base[1] >> 5, n4 = (h.kslot_base[2] - h.kslot_base[1]) >> 5,
                  n8 = (h.kslot_base[3] - h.kslot_base[2]) >> 5;
        const int c0 = h.c[0];
        tl.n2 = n2;
        tl.n4 = n4;
        tl.n8 = n8;
        tl.vmax2 = bf16_bits_to_float(h.scale_bounds >> 16);
        // q range per head (lanes 8h .. 8h + 7 scan head h), then this lane's head tig
        const int hq = L.lane >> 3;
        float qm = absmax16<IO>(reinterpret_cast<const IO*>(qs + (hq < g ? hq : 0) * QROW) + 16 * (L.lane & 7));
#pragma unroll
        for (int o = 1; o < 8; o <<= 1) qm = fmaxf(qm, __shfl_xor_sync(0xffffffffu, qm, o));
        qm = __shfl_sync(0xffffffffu, qm, 8 * tig);
        const IO* qh = reinterpret_cast<const IO*>(qs + (hv ? tig : 0) * QROW);
        float s1 = 0.0f;  // scale bound of the 4- and 8-bit channels (2-bit: the header's)
        for (int j = h.kslot_base[1] + L.lane; j < h.kslot_base[3]; j += 32) s1 = fmaxf(s1, fabsf(chanf[2 * j]));
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) s1 = fmaxf(s1, __shfl_xor_sync(0xffffffffu, s1, o));
        const float bnd = fmaxf(bf16_bits_to_float(h.scale_bounds & 0xFFFFu), s1) * qm;
        const float sg = (hv && bnd > 0.0f) ? kQFix * rcp_approx(bnd) : 0.0f;
        float bpart = 0.0f;
        {  // 2-bit k-steps kk = 2 half + i (< n2): the u2x generator over channel slots
            const int ps = L.lane & 4;
            const float sgA = sg * __int_as_float((127 + 6 - ps) << 23);
            const float sgB = sgA * 0.25f;
            const int kk = 2 * half + (L.lane >> 4);
            const bool act = kk < n2;
            uint32_t xa[4], xb[4];
            float2 bp = make_float2(0.0f, 0.0f);
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const int c = L.qch + 4 * ((e + tig) & 3);
                const int j0 = min(c, h.kslots - 2);
                const float4 cs = *reinterpret_cast<const float4*>(chanf + 2 * j0);
                float2 qv;
                qv.x = (act && c < c0) ? ld_io(qh, perm[j0]) : 0.0f;
                qv.y = (act && c + 1 < c0) ? ld_io(qh, perm[j0 + 1]) : 0.0f;
                bp = ffma2(qv, make_float2(cs.y, cs.w), bp);
                const float ya = fmaf(cs.x * qv.x, sgA, kMagicS), yb = fmaf(cs.z * qv.y, sgB, kMagicS);
                xa[e] = (__float_as_uint(ya) + (0x00808080u - 0x4B400000u)) ^ 0x00808080u;
                xb[e] = (__float_as_uint(yb) + (0x00808080u - 0x4B400000u)) ^ 0x00808080u;
            }
            bpart = bp.x + bp.y;
            const uint32_t a01 = __byte_perm(xa[0], xa[1], 0x5140), b01 = __byte_perm(xa[0], xa[1], 0x7362);
            const uint32_t a23 = __byte_perm(xa[2], xa[3], 0x5140), b23 = __byte_perm(xa[2], xa[3], 0x7362);
            const uint32_t c01 = __byte_perm(xb[0], xb[1], 0x5140), d01 = __byte_perm(xb[0], xb[1], 0x7362);
            const uint32_t c23 = __byte_perm(xb[2], xb[3], 0x5140), d23 = __byte_perm(xb[2], xb[3], 0x7362);
            if (act) {
                uint8_t* w = qdig + L.qdig_w;
                *reinterpret_cast<uint2*>(w) = make_uint2(__byte_perm(b01, b23, L.sel_lo), __byte_perm(d01, d23, L.sel_lo));
                *reinterpret_cast<uint2*>(w + 224) =
                    make_uint2(__byte_perm(a01, a23, L.sel_hi), __byte_perm(c01, c23, L.sel_hi));
                *reinterpret_cast<uint2*>(w + 256) =
                    make_uint2(__byte_perm(a01, a23, L.sel_lo), __byte_perm(c01, c23, L.sel_lo));
            }
        }
        // 4- and 8-bit k-steps (warp `half` takes every other one): K positions
        // 4j .. 4j + 3 of head tig (j = lane >> 2), each lane's slot per the class's A mask
        const int nw = n4 + n8;
        for (int jw = half; jw < nw; jw += 2) {
            const bool b4 = jw < n4;
            const int j = L.lane >> 2;
            const int sbase = b4 ? h.kslot_base[1] + 32 * jw : h.kslot_base[2] + 32 * (jw - n4);
            const int cnt = b4 ? h.c[1] - 32 * jw : h.c[2] - 32 * (jw - n4);  // valid slots of this k-step
            uint32_t x1[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const int pk = 4 * j + e, rr = pk & 15, tt = rr >> 2;
                const int sl = b4 ? 16 * (pk >> 4) + 8 * (tt >> 1) + 2 * (rr & 3) + (tt & 1) : pk;
                const float2 cs = reinterpret_cast<const float2*>(chanf)[sbase + sl];
                const float qv = (sl < cnt && hv) ? ld_io(qh, perm[sbase + sl]) : 0.0f;
                bpart = fmaf(qv, cs.y, bpart);
                const float pre = (b4 && (tt & 1)) ? 4.0f : 64.0f;
                const float y = fmaf(cs.x * qv, sg * pre, kMagicS);
                x1[e] = (__float_as_uint(y) + (0x00808080u - 0x4B400000u)) ^ 0x00808080u;
            }
            const uint32_t a01 = __byte_perm(x1[0], x1[1], 0x5140), b01 = __byte_perm(x1[0], x1[1], 0x7362);
            const uint32_t a23 = __byte_perm(x1[2], x1[3], 0x5140), b23 = __byte_perm(x1[2], x1[3], 0x7362);
            uint8_t* w1p = qdig + (n2 + jw) * 512 + 4 * (j & 3);
            const int hs = ((j >> 2) ^ (tig >> 1)) * 16;
            *reinterpret_cast<uint32_t*>(w1p + (2 * tig + 1) * 32 + hs) = __byte_perm(b01, b23, 0x5410);
            *reinterpret_cast<uint32_t*>(w1p + (8 + 2 * tig) * 32 + hs) = __byte_perm(a01, a23, 0x7632);
            *reinterpret_cast<uint32_t*>(w1p + (9 + 2 * tig) * 32 + hs) = __byte_perm(a01, a23, 0x5410);
        }
#pragma unroll
        for (int o = 4; o < 32; o <<= 1) bpart += __shfl_xor_sync(0xffffffffu, bpart, o);
        if (gid == 0) xg.bias[half][tig] = bpart;
        pair_sync(bar);
        after_sync1();
        run.bias2 = hv ? (xg.bias[0][tig] + xg.bias[1][tig]) * (kInvSqrtD * kLog2e) : -INFINITY;
        run.qscale2 = bnd * (kInvSqrtD * kLog2e / (64.0f * kQFix));
        run.m = -INFINITY;
        run.l = 0.0f;
#pragma unroll
        for (int m = 0; m < 4; ++m) run.o[m] = make_float2(0.0f, 0.0f);
    } else {
        pair_sync(bar);  // both warps are past the previous chunk: its buffer may be refilled
        after_sync1();
    }
    const float bias2 = run.bias2, qscale2 = run.qscale2;
    const int n2 = tl.n2, n4 = tl.n4, n8 = tl.n8;

    // ---- QK over this warp's blocks half, half + 2 (A rows gid / gid + 8 of
    // m-tile u = slots 32 pb + 4 gid + 2u / + 1, slot-transposed K rows)
    const int qstride = Q * krb;
    float2 lg[NBW][2];
    float mx = -INFINITY, vm = 0.0f;
#pragma unroll
    for (int i = 0; i < NBW; ++i) {
        if (i < mynb) {
            const int pb = half + 2 * i;
            const uint8_t* r0 = kb + (size_t)(8 * pb + gid) * krb;  // m-tile u = 0, row gid
            int acc[2][2][4];
#pragma unroll
            for (int u = 0; u < 2; ++u)
#pragma unroll
                for (int nt = 0; nt < 2; ++nt) acc[u][nt][0] = acc[u][nt][1] = acc[u][nt][2] = acc[u][nt][3] = 0;
            const uint8_t* qd = qdig + L.bofs;
            // 2-bit channels: 8 B of each row per k-step
#pragma unroll 1
            for (int kk = 0; kk < n2; ++kk, qd += 512) {
                uint32_t bq[4];
                ldsm_x4(bq, qd);
#pragma unroll
                for (int u = 0; u < 2; ++u) {
                    const uint2 x = lds64(r0 + 2 * u * qstride + 8 * kk), y = lds64(r0 + (2 * u + 1) * qstride + 8 * kk);
                    const uint32_t a[4] = {x.x & L.kmask, y.x & L.kmask, x.y & L.kmask, y.y & L.kmask};
                    mma_u8s8(acc[u][0], a, bq[0], bq[1]);
                    mma_u8s8(acc[u][1], a, bq[2], bq[3]);
                }
            }
            // 4-bit channels: 16 B per k-step, nibble masks
            {
                const int o4 = 8 * n2 + 4 * (tig >> 1);
                const uint32_t m4 = 0x0F0F0F0Fu << (4 * (tig & 1));
#pragma unroll 1
                for (int j4 = 0; j4 < n4; ++j4, qd += 512) {
                    uint32_t bq[4];
                    ldsm_x4(bq, qd);
#pragma unroll
                    for (int u = 0; u < 2; ++u) {
                        const uint8_t* ra = r0 + 2 * u * qstride + o4 + 16 * j4;
                        const uint8_t* rb = ra + qstride;
                        const uint32_t a[4] = {lds32(ra) & m4, lds32(rb) & m4, lds32(ra + 8) & m4, lds32(rb + 8) & m4};
                        mma_u8s8(acc[u][0], a, bq[0], bq[1]);
                        mma_u8s8(acc[u][1], a, bq[2], bq[3]);
                    }
                }
            }
            // 8-bit channels: 32 B per k-step, raw bytes
            {
                const int o8 = 8 * n2 + 16 * n4 + 4 * tig;
#pragma unroll 1
                for (int j8 = 0; j8 < n8; ++j8, qd += 512) {
                    uint32_t bq[4];
                    ldsm_x4(bq, qd);
#pragma unroll
                    for (int u = 0; u < 2; ++u) {
                        const uint8_t* ra = r0 + 2 * u * qstride + o8 + 32 * j8;
                        const uint8_t* rb = ra + qstride;
                        const uint32_t a[4] = {lds32(ra), lds32(rb), lds32(ra + 16), lds32(rb + 16)};
                        mma_u8s8(acc[u][0], a, bq[0], bq[1]);
                        mma_u8s8(acc[u][1], a, bq[2], bq[3]);
                    }
                }
            }
#pragma unroll
            for (int u = 0; u < 2; ++u) {
                const float2 hi = make_float2((float)acc[u][0][1], (float)acc[u][0][3]);
                const float2 lo = make_float2((float)(acc[u][1][0] * 256 + acc[u][1][1]),
                                              (float)(acc[u][1][2] * 256 + acc[u][1][3]));
                const float2 v = ffma2(hi, make_float2(65536.0f, 65536.0f), lo);
                lg[i][u] = ffma2(v, make_float2(qscale2, qscale2), make_float2(bias2, bias2));
            }
            const int sbase = 32 * pb + 4 * gid;
            if (32 * pb + 32 > n) {  // ragged last block: slots >= n get no weight
#pragma unroll
                for (int u = 0; u < 2; ++u) {
                    if (sbase + 2 * u >= n) lg[i][u].x = -INFINITY;
                    if (sbase + 2 * u + 1 >= n) lg[i][u].y = -INFINITY;
                }
            }
            mx = fmaxf(mx, fmaxf(fmaxf(lg[i][0].x, lg[i][0].y), fmaxf(lg[i][1].x, lg[i][1].y)));
            if (ck.cls != 0) {  // V scales of this lane's four slots (the chunk's p~ range)
                const float4* vp4 = reinterpret_cast<const float4*>(vparam + min(sbase, nslot - 4));
                const float4 va = vp4[0], vc = vp4[1];
                vm = fmaxf(vm, fmaxf(fmaxf(va.x, va.z), fmaxf(vc.x, vc.z)));
            }
        }
    }
#pragma unroll
    for (int o = 4; o < 32; o <<= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if (ck.cls != 0) {
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) vm = fmaxf(vm, __shfl_xor_sync(0xffffffffu, vm, o));
        if (L.lane == 0) vmx[half] = vm;
    }
    if (gid == 0) xg.mx[half][tig] = mx;
    pair_sync(bar);
    mx = fmaxf(xg.mx[0][tig], xg.mx[1][tig]);
    if (mx == -INFINITY) mx = 0.0f;  // head without tokens (tig >= g)
    const float vmax = ck.cls != 0 ? fmaxf(vmx[0], vmx[1]) : tl.vmax2;
    const float psig = vmax > 0.0f ? kPScale * rcp_approx(vmax) : 0.0f;
    const float vinv = vmax * (1.0f / kPScale);

    // ---- softmax + p~ digits (hi, lo bytes): four consecutive slots per lane and block
    float2 ls2 = make_float2(0.0f, 0.0f);
    float bv = 0.0f;
    const float2 nmx = make_float2(-mx, -mx);
#pragma unroll
    for (int i = 0; i < NBW; ++i) {
        if (i < mynb) {
            const int pb = half + 2 * i;
            const float4* vp4 = reinterpret_cast<const float4*>(vparam + min(32 * pb + 4 * gid, nslot - 4));
            const float4 va = vp4[0], vc = vp4[1];
            const float2 d01 = fadd2(lg[i][0], nmx), d23 = fadd2(lg[i][1], nmx);
            const float2 p01 = make_float2(ex2_approx(d01.x), ex2_approx(d01.y));
            const float2 p23 = make_float2(ex2_approx(d23.x), ex2_approx(d23.y));
            ls2 = fadd2(ls2, fadd2(p01, p23));
            bv = fmaf(p01.x, va.y, bv);
            bv = fmaf(p01.y, va.w, bv);
            bv = fmaf(p23.x, vc.y, bv);
            bv = fmaf(p23.y, vc.w, bv);
            const float2 vs01 = fmul2(make_float2(va.x, va.z), make_float2(psig, psig));
            const float2 vs23 = fmul2(make_float2(vc.x, vc.z), make_float2(psig, psig));
            const float2 y01 = ffma2(p01, vs01, make_float2(kMagicU, kMagicU));
            const float2 y23 = ffma2(p23, vs23, make_float2(kMagicU, kMagicU));
            const uint32_t t01 = __byte_perm(__float_as_uint(y01.x), __float_as_uint(y01.y), 0x5140);
            const uint32_t t23 = __byte_perm(__float_as_uint(y23.x), __float_as_uint(y23.y), 0x5140);
            uint8_t* pw = pdig + pb * 256 + L.pdig_w;
            *reinterpret_cast<uint32_t*>(pw) = __byte_perm(t01, t23, 0x7632);
            *reinterpret_cast<uint32_t*>(pw + 32) = __byte_perm(t01, t23, 0x5410);
        }
    }
    float lsum = ls2.x + ls2.y;
#pragma unroll
    for (int o = 4; o < 32; o <<= 1) {
        lsum += __shfl_xor_sync(0xffffffffu, lsum, o);
        bv += __shfl_xor_sync(0xffffffffu, bv, o);
    }
    if (gid == 0) {
        xg.lsum[half][tig] = lsum;
        xg.bv[half][tig] = bv;
    }
    pair_sync(bar);
    const float lt = xg.lsum[0][tig] + xg.lsum[1][tig];
    const float bt = xg.bv[0][tig] + xg.bv[1][tig];

    // ---- PV: this warp's 64 output channels (4 m-tiles), one n-tile of p~ digits
    int acc[4][4];
#pragma unroll
    for (int m = 0; m < 4; ++m) acc[m][0] = acc[m][1] = acc[m][2] = acc[m][3] = 0;
    float sc0, sc1;  // output scale of rows gid / gid + 8 (the in-place mask factors)
    if (ck.cls == 0) {
        const uint8_t* g0b = vb + L.vcol;
#pragma unroll 1
        for (int kk = 0; kk < nb; ++kk) {
            uint32_t b[2];
            ldsm_x2(b, pdig + kk * 256 + L.bofs2);
            const uint4 x0 = lds128(g0b + kk * 1024), x1 = lds128(g0b + kk * 1024 + 512);
            const uint32_t u0[4] = {x0.x, x0.y, x0.z, x0.w}, u1[4] = {x1.x, x1.y, x1.z, x1.w};
#pragma unroll
            for (int m = 0; m < 4; ++m) {
                const uint32_t a[4] = {u0[m] & L.vm0, u0[m] & L.vm1, u1[m] & L.vm0, u1[m] & L.vm1};
                mma_u8u8(acc[m], a, b[0], b[1]);
            }
        }
        sc0 = vinv * L.s0f;
        sc1 = sc0 * 0.25f;
    } else if (ck.cls == 1) {
        // 4-bit rows (64 B; 4-token groups of 256 B, word columns swizzled by 8 (G & 3) = 8 tig):
        // byte column 32 half + 8 (gid & 3) + 2m + jj holds channels ch0 + 4m (lo nibble,
        // row gid) and ch0 + 4m + 1 (hi nibble, row gid + 8)
        // (the lane's four columns are every other word of one swizzled 8-word run:
        // two 16-B loads per group and a select by jj = gid >> 2)
        const bool jj = (gid >> 2) != 0;
        const uint8_t* g0b = vb + tig * 256 + (((32 * half + 8 * (gid & 3)) ^ (8 * tig)) * 4);
#pragma unroll 1
        for (int kk = 0; kk < nb; ++kk) {
            uint32_t b[2];
            ldsm_x2(b, pdig + kk * 256 + L.bofs2);
            const uint4 x0 = lds128(g0b + kk * 2048), x1 = lds128(g0b + kk * 2048 + 16);
            const uint4 y0 = lds128(g0b + kk * 2048 + 1024), y1 = lds128(g0b + kk * 2048 + 1040);
            const uint32_t u0[4] = {jj ? x0.y : x0.x, jj ? x0.w : x0.z, jj ? x1.y : x1.x, jj ? x1.w : x1.z};
            const uint32_t u1[4] = {jj ? y0.y : y0.x, jj ? y0.w : y0.z, jj ? y1.y : y1.x, jj ? y1.w : y1.z};
#pragma unroll
            for (int m = 0; m < 4; ++m) {
                const uint32_t a[4] = {u0[m] & 0x0F0F0F0Fu, u0[m] & 0xF0F0F0F0u, u1[m] & 0x0F0F0F0Fu,
                                       u1[m] & 0xF0F0F0F0u};
                mma_u8u8(acc[m], a, b[0], b[1]);
            }
        }
        sc0 = vinv;
        sc1 = vinv * 0.0625f;
    } else {
        // 8-bit rows (128 B; groups of 512 B): byte columns ch0 + 4m (row gid) and + 1
        // (row gid + 8), one 8-B load per group
        const uint8_t* g0b = vb + tig * 512;
#pragma unroll 1
        for (int kk = 0; kk < nb; ++kk) {
            uint32_t b[2];
            ldsm_x2(b, pdig + kk * 256 + L.bofs2);
#pragma unroll
            for (int m = 0; m < 4; ++m) {
                const int wo = ((L.ch0 + 4 * m) ^ (8 * tig)) * 4;
                const uint2 w0 = lds64(g0b + kk * 4096 + wo), w1 = lds64(g0b + kk * 4096 + 2048 + wo);
                const uint32_t a[4] = {w0.x, w0.y, w1.x, w1.y};
                mma_u8u8(acc[m], a, b[0], b[1]);
            }
        }
        sc0 = vinv;
        sc1 = vinv;
    }
    // ---- fold this chunk (max mx, sum lt, unnormalised outputs v * s + bt) into the running state
    if (hv && lt > 0.0f) {
        const float mnew = fmaxf(run.m, mx);
        const float a = ex2_approx(run.m - mnew), bw = ex2_approx(mx - mnew);
        const float2 sc = make_float2(sc0 * bw, sc1 * bw), bb = make_float2(bt * bw, bt * bw);
        const float2 aa = make_float2(a, a);
#pragma unroll
        for (int m = 0; m < 4; ++m) {  // (the digit combine in f32: 8-bit sums exceed int32 at 256x)
            const float2 v = ffma2(make_float2((float)acc[m][0], (float)acc[m][2]), make_float2(256.0f, 256.0f),
                                   make_float2((float)acc[m][1], (float)acc[m][3]));
            run.o[m] = ffma2(run.o[m], aa, ffma2(v, sc, bb));
        }
        run.l = fmaf(run.l, a, lt * bw);
        run.m = mnew;
    }
}

template <typename IO, bool G8>
__global__ void __launch_bounds__(32 * 2 * kXPairs, 1) decode_u24_kernel(const MmaParams p) {
    extern __shared__ __align__(128) uint8_t dsm[];
    const int nbuf = p.R;
    uint64_t* full = reinterpret_cast<uint64_t*>(dsm);
    uint8_t* bufs = dsm + p.W * kXMaxBuf * sizeof(uint64_t);
    uint8_t* scratch0 = bufs + (size_t)p.W * nbuf * p.slot_bytes;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int pr = warp >> 1, half = warp & 1;
    constexpr int QROW = kD * (int)sizeof(IO);
    const int qbytes = p.g * QROW;
    uint64_t* fb = full + pr * kXMaxBuf;
    uint8_t* pbuf = bufs + (size_t)pr * nbuf * p.slot_bytes;
    uint8_t* scr = scratch0 + (size_t)pr * p.scratch_bytes;
    const int S = p.split_world;  // parts per tile
    const int nitems = p.units * S;
    const int item0 = blockIdx.x + pr * gridDim.x, istride = p.W * gridDim.x;
    const int qoff = p.slot_bytes - qbytes;
    const bool issuer = half == 0 && lane == 0;

    // ---- issuer state (one lane, kept in the pair's shared scratch so it costs
    // no registers in the other 63 threads): the next (item, chunk) to stage
    U24Issuer& is = *reinterpret_cast<U24Issuer*>(scr + (p.g > 4 ? 2 : 1) * kU24Scratch);
    auto load_meta = [&](int item, U24Meta& m) {
        m.base = nullptr;
        if (item >= 0 && item < nitems) {
            const int tile = item / S;
            m.base = p.arena + p.offsets[tile];
            const TileHeader* th = reinterpret_cast<const TileHeader*>(m.base);
            m.nslot = th->nslot;
            m.hk = th->off_k;
            m.krb = th->krow_bytes;
            m.offvp = th->off_vp;
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                m.offv[c] = th->off_vseg[c];
                m.r[c] = th->r[c];
            }
        }
    };
    auto set_cur = [&]() {
        u24_tile(is.cur.r, is.t);
        is.n = u24_nchunks(is.t);
    };
    // the pair's next item (static striding: items of a round are spread over
    // all pairs; measured faster than claiming items from a global counter)
    auto next_item = [&](int it) {
        if (it < 0 || it >= nitems) return -1;
        const int v = it + istride;
        return v < nitems ? v : -1;
    };
    auto advance = [&]() {
        is.c += S;
        if (is.c >= is.n) {
            is.item = is.nxt_item;
            if (is.item < 0) return;
            is.c = is.item % S;
            is.cur = is.nxt;
            set_cur();
            is.nxt_item = next_item(is.item);
            load_meta(is.nxt_item, is.nxt);
        }
    };
    auto stage_item = [&](int b) {
        const U24Meta& cur = is.cur;
        const U24Geom gg = u24_chunk(is.t, is.c);
        const bool first = is.c == is.item % S;
        is.bitem[b] = is.item;
        is.bc[b] = is.c;
        uint8_t* dst = pbuf + (size_t)b * p.slot_bytes;
        const int rows = gg.ns >> 2, Q = cur.nslot >> 2;
        const int rb = u24_vrow_bytes(gg.cls);
        const uint32_t kbytes = (uint32_t)(rows * cur.krb), vbytes = (uint32_t)(gg.ns * rb),
                       pbytes = (uint32_t)(gg.ns * 8);
        // (the very first chunk's q rows are issued later, after the grid dependency)
        const uint32_t tx = 4 * kbytes + vbytes + pbytes + (first ? (uint32_t)(cur.hk + qbytes) : 0u);
        fence_proxy_async();
        mbar_expect_tx(&fb[b], tx);
        if (first) bulk_g2s(dst, cur.base, (uint32_t)cur.hk, &fb[b]);
        const int dk = cur.hk;
#pragma unroll
        for (int r = 0; r < 4; ++r)
            bulk_g2s(dst + dk + r * kbytes, cur.base + cur.hk + (size_t)(r * Q + (gg.s0 >> 2)) * cur.krb, kbytes, &fb[b]);
        const int offv = gg.cls == 0 ? cur.offv[0] : gg.cls == 1 ? cur.offv[1] : cur.offv[2];
        bulk_g2s(dst + dk + gg.ns * cur.krb, cur.base + offv + (size_t)gg.li0 * rb, vbytes, &fb[b]);
        bulk_g2s(dst + dk + gg.ns * cur.krb + vbytes, cur.base + cur.offvp + (size_t)gg.s0 * 8, pbytes, &fb[b]);
    };
    auto stage_q = [&](int b, int item) {
        bulk_g2s(pbuf + (size_t)b * p.slot_bytes + qoff, static_cast<const uint8_t*>(p.q) + (size_t)(item / S) * qbytes,
                 (uint32_t)qbytes, &fb[b]);
    };
    // stage the next chunk into buffer b, or (once) the end-of-work marker
    auto issue_item = [&](int b) {
        if (is.done) return;
        if (is.item < 0 || is.item >= nitems || !is.cur.base) {
            is.bitem[b] = -1;
            mbar_arrive(&fb[b]);
            is.done = 1;
            return;
        }
        const bool first = is.c == is.item % S;
        const int it = is.item;
        stage_item(b);
        if (first) stage_q(b, it);
        advance();
    };

    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    if (issuer) {
        for (int b = 0; b < nbuf; ++b) mbar_init(&fb[b], 1);
        fence_barrier_init();
        is.done = 0;
        is.item = item0 < nitems ? item0 : -1;
        is.c = item0 % S;
        load_meta(item0, is.cur);
        set_cur();
        if (is.item >= 0) stage_item(0);  // KV of the first chunk before the grid dependency
    }
    asm volatile("griddepcontrol.wait;" ::: "memory");
    if (issuer) {
        if (is.item >= 0) {
            stage_q(0, item0);
            is.nxt_item = next_item(item0);
            load_meta(is.nxt_item, is.nxt);
            advance();
        } else {
            issue_item(0);  // no work: the end marker
        }
    }
    const U2xLane lc = u2x_lane(half);
    constexpr int npass = G8 ? 2 : 1;  // GQA groups of 5..8 heads: two 4-head passes per staged chunk
    for (int hp = 0; hp < npass; ++hp)
        for (int i = threadIdx.x & 63; i < kU24MaxK * 512 / 16; i += 64)
            reinterpret_cast<uint4*>(scr + hp * kU24Scratch + kU24QDig)[i] = make_uint4(0u, 0u, 0u, 0u);
    __syncthreads();
    int b = 0, k = 0;
    uint32_t phase = 0;
    U2xRun run0;
    U2xRun run1;  // (G8 only)
    U24Tile tl{};
    int tile = 0, part = 0, C = 1, hk = 0, krb = 0;
    for (;;) {
        mbar_wait(&fb[b], phase);
        __syncwarp();
        const int item = is.bitem[b], c = is.bc[b];
        if (item < 0) break;
        const uint8_t* st = pbuf + (size_t)b * p.slot_bytes;
        const bool first = c < S;  // an item's first chunk is its part index
        if (first) {
            tile = item / S;
            part = item % S;
            const TileHeader& th = *reinterpret_cast<const TileHeader*>(st);
            u24_tile(th.r, tl);
            C = u24_nchunks(tl);
            hk = th.off_k;
            krb = th.krow_bytes;
        }
        if (k == 0 && issuer)  // look-ahead once the first chunk is in
            for (int j = 1; j < nbuf; ++j) issue_item(j);
        const int bprev = b == 0 ? nbuf - 1 : b - 1;
        auto refill = [&]() {
            if (issuer && k >= 1) issue_item(bprev);
        };
        const U24Geom ck = u24_chunk(tl, c);
        const uint8_t* kb = st + hk;
        const uint8_t* vb = kb + ck.ns * krb;
        const float2* vp = reinterpret_cast<const float2*>(vb + ck.ns * u24_vrow_bytes(ck.cls));
        decode_chunk_u24<IO>(st, st + qoff, min(4, p.g), scr, 1 + pr, lc, refill, ck, first, krb, kb, vb, vp, run0,
                             tl);
        if constexpr (G8)
            decode_chunk_u24<IO>(st, st + qoff + 4 * QROW, p.g - 4, scr + kU24Scratch, 1 + pr, lc, [] {}, ck, first,
                                 krb, kb, vb, vp, run1, tl);
        if (++b == nbuf) {
            b = 0;
            phase ^= 1u;
        }
        ++k;
        if (c + S < C) continue;  // more chunks of this item follow
#pragma unroll
        for (int hp = 0; hp < 2; ++hp) {
            const int head = 4 * hp + lc.tig;
            if (hp >= npass || head >= p.g) continue;
            const U2xRun& rn = (G8 && hp) ? run1 : run0;
            if (p.partial) {  // this part's (o, max, sum) of the tile
                float* prow = p.partial + (((size_t)part * p.units + tile) * p.g + head) * (kD + 2);
#pragma unroll
                for (int m = 0; m < 4; ++m) *reinterpret_cast<float2*>(prow + lc.ch0 + 4 * m) = rn.o[m];
                if (half == 0 && lc.gid == 0) {
                    prow[kD] = rn.m;
                    prow[kD + 1] = rn.l;
                }
            } else {
                IO* orow = static_cast<IO*>(p.out) + ((size_t)tile * p.g + head) * kD + lc.ch0;
                const float inv = rcp_approx(rn.l);
                const float2 iv = make_float2(inv, inv);
#pragma unroll
                for (int m = 0; m < 4; ++m) {
                    const float2 r = fmul2(rn.o[m], iv);
                    if constexpr (sizeof(IO) == 2)
                        *reinterpret_cast<__half2*>(orow + 4 * m) = __float22half2_rn(r);
                    else
                        *reinterpret_cast<float2*>(orow + 4 * m) = r;
                }
            }
        }
    }
}

// Parts per tile for split-K. Items (tile, part) are dealt to the warp pairs
// round by round, so the step costs about rounds(S) x ceil(C / S) chunk times
// (C = chunks per tile) plus a per-part cost (its q~ setup, partial row and
// merge share), ~0.75 chunk per part as measured over the configs[3] points
// (tools/c3_bench.py --sweep: e.g. Qwen2.5-7B, 448 tiles of 14 chunks on 888
// pairs, S = 3 at 78.5 us against 89.7 at S = 4 and 97.5 at S = 1). Never more
// parts than the smallest tile has chunks (no empty parts).
constexpr double kU24PartCost = 0.75;
static int u24_parts(const rdkv_decode_args* a, int pairs_total) {
    const int C = a->plan.min_chunks24 > 1 ? a->plan.min_chunks24 : 1;
    const int smax = C < kU24MaxParts ? C : kU24MaxParts;
    int best = 1;
    double best_cost = 1e300;
    for (int S = 1; S <= smax; ++S) {
        const long long items = (long long)a->units * S;
        const long long rounds = (items + pairs_total - 1) / pairs_total;
        const double cost = (double)rounds * ((C + S - 1) / S) + kU24PartCost * S;
        if (cost < best_cost - 1e-9) {
            best_cost = cost;
            best = S;
        }
    }
    return best;
}

template <typename IO>
static int launch_u24(const rdkv_decode_args* a, cudaStream_t st) {
    const int qbytes = a->group * kD * (int)sizeof(IO);
    // header + channel table + perm (<= 128 + 10 * 192 B), then a chunk's K rows,
    // V rows and V params (class 0 the largest), q rows at the end
    const int krb = a->plan.max_krow_bytes24;
    int body = 0;
    for (int c = 0; c < 3; ++c) {
        const int b = u24_chunk_slots(c) * (krb + u24_vrow_bytes(c) + 8);
        body = b > body ? b : body;
    }
    const int slot = ((kHeaderBytes + 10 * 192 + body + qbytes + 127) & ~127);
    const int scratch = ((a->group > 4 ? 2 : 1) * kU24Scratch + (int)sizeof(U24Issuer) + 127) & ~127;
    const DevAttrs da = dev_attrs();
    const int slack = 128;
    int W = 0, nbuf = 0;
    if (!pick_pairs(1 << 30, da.nsm, slot, scratch, da.smem_optin - slack, W, nbuf)) return RDKV_EINVAL;
    // a->split: 0 automatic, 1 one part per tile, > 1 that many parts (capped)
    int S0 = a->split == 0 ? u24_parts(a, W * da.nsm) : a->split;
    if (S0 > a->plan.min_chunks24) S0 = a->plan.min_chunks24;
    if (S0 > kU24MaxParts) S0 = kU24MaxParts;
    const size_t need = rdkv_cuda_decode_workspace(a->units, a->group, kD, S0);
    const int S = (S0 > 1 && a->workspace && a->workspace_bytes >= need) ? S0 : 1;
    MmaParams p{a->arena, a->tile_offsets, a->tile_decode_bytes, a->q, a->out,
                static_cast<const __half*>(a->zc_k), static_cast<const __half*>(a->zc_v), a->zc_len,
                a->units, a->group, a->zc_cap, nbuf, W, slot, scratch, 0, 0, -1, -1, 0, 0};
    p.partial = S > 1 ? static_cast<float*>(a->workspace) : nullptr;
    p.split_rank = 0;
    p.split_world = S;
    // pairs per CTA (experiments build: RDKV_DECODE_U24_PPC); the SM holds W pairs
    static const char* ppc_env = experiment_knob("RDKV_DECODE_U24_PPC");
    const int ppc = ppc_env && atoi(ppc_env) > 0 && W % atoi(ppc_env) == 0 ? atoi(ppc_env) : W;
    const int ctas = W / ppc;
    p.W = ppc;
    const size_t smem_cta = ppc * kXMaxBuf * sizeof(uint64_t) + (size_t)ppc * (nbuf * slot + scratch) + slack;
    auto kern = a->group > 4 ? decode_u24_kernel<IO, true> : decode_u24_kernel<IO, false>;
    static std::atomic<int> smem_set[2][kMaxDevices];
    set_smem_once(kern, (int)smem_cta, smem_set[a->group > 4], da.dev);
    long long items = (long long)a->units * S;
    int blocks = (int)((items + ppc - 1) / ppc);
    if (blocks > ctas * da.nsm) blocks = ctas * da.nsm;
    if (verbose_env())
        fprintf(stderr, "u24: units %d parts %d pairs %d/cta %d bufs %d slot %d smem %zu grid %d\n", a->units, S, W,
                ppc, nbuf, slot, smem_cta, blocks);
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(blocks);
    cfg.blockDim = dim3(32 * 2 * ppc);
    cfg.dynamicSmemBytes = smem_cta;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    if (cudaLaunchKernelEx(&cfg, kern, p) != cudaSuccess) return RDKV_ECUDA;
    if (S > 1) return launch_merge(p.partial, S, a->units * a->group, kD, a->out, a->io_dtype, st);
    return launch_status();
}

int launch_mma(const rdkv_decode_args* a, cudaStream_t st) {
    const bool f16 = a->io_dtype == RDKV_F16;
    // split step (rdkv_cuda_decode_prepare_split): mixed tiles on the general
    // body, then the uniform-2-bit ones on u2x (PDL: its prologue and KV
    // prefetch overlap the general kernel's tail)
    const rdkv_decode_plan& pl = a->plan;
    // mixed 2/4/8-bit tiles (not all short enough for MIX), and uniform 2-bit tiles too
    // long for the short-tile kernel: the chunked split-K kernel (no Zone C; kernel 0 or 2)
    // (long uniform-2-bit tiles stay on the chunked u2x body when there are enough of them to
    // fill every warp pair — split-K only pays for few tiles: budget_512, 4096 tiles: 54 vs 71 us)
    const bool short_u2x = pl.uniform2 && pl.max_slots <= kU2MaxSlots;
    const bool many_u2 = pl.uniform2 && u2x_group_ok(a) && a->units >= kXPairs * dev_attrs().nsm;
    if (pl.mix24 && !short_u2x && !many_u2 && !a->zc_len && a->group <= 8 && (a->kernel == 0 || a->kernel == 2)) {
        rdkv_decode_args b = *a;
        b.unit_ids = nullptr;
        return f16 ? launch_u24<__half>(&b, st) : launch_u24<float>(&b, st);
    }
    // (the uniform subset goes to the short-tile kernel, which is the one that
    // reads unit_ids: every tile of the step must fit it)
    if (a->unit_ids && !pl.uniform2 && pl.n_uniform > 0 && pl.n_uniform < a->units && a->group <= 8 &&
        pl.max_slots <= kU2MaxSlots && a->kernel == 0 && (!a->zc_len || zc_fusable(a))) {
        rdkv_decode_args gm = *a;
        gm.units = a->units - pl.n_uniform;
        gm.unit_ids = a->unit_ids + pl.n_uniform;
        // (spreading the mixed tiles thinly over all SMs and running u2x after
        // measured 37 us vs 27.5 us for this concurrent split: the general body
        // is latency-bound per tile, ~25 us for one mixed tile on one warp)
        int gblocks = 0;
        const int rc = a->group <= 4
                           ? (f16 ? launch_t<1, __half, false>(&gm, st, &gblocks) : launch_t<1, float, false>(&gm, st, &gblocks))
                           : (f16 ? launch_t<2, __half, false>(&gm, st, &gblocks) : launch_t<2, float, false>(&gm, st, &gblocks));
        if (rc) return rc;
        // the uniform tiles run beside it on the SMs it leaves free (u2x is
        // issue-bound: the mixed tiles are few but slow, latency-bound per tile)
        rdkv_decode_args um = *a;
        um.units = pl.n_uniform;
        um.plan.uniform2 = pl.uniform2_split;
        const int free_sms = dev_attrs().nsm - gblocks;
        return f16 ? launch_u2x<__half>(&um, st, free_sms > 0 ? free_sms : 1)
                   : launch_u2x<float>(&um, st, free_sms > 0 ? free_sms : 1);
    }
    // not split: every launch walks the units in order (unit_ids only name subsets)
    rdkv_decode_args plain = *a;
    plain.unit_ids = nullptr;
    a = &plain;

    // uniform 2-bit tiles (the n=128 production shape) take the specialised body
    // uniform 2-bit tiles (the n=128 production shape): warp-pair body by default,
    // kernel 4 selects the one-warp body, kernel 3 the general body
    const bool u2 = a->plan.uniform2 && u2x_group_ok(a) &&
                    (a->kernel != 3 || a->plan.max_slots > kMaxSlots ||
                     general_min_smem(a) > (size_t)dev_attrs().smem_optin);  // general body: tile in smem
    const bool short_u2 = u2 && a->plan.max_slots <= kU2MaxSlots && !a->zc_len && a->plan.uniform2 != 3;
    if (short_u2 && a->kernel == 4) return f16 ? launch_t<1, __half, true>(a, st) : launch_t<1, float, true>(a, st);
    if (short_u2 && a->kernel == 5) return f16 ? launch_pair<__half>(a, st) : launch_pair<float>(a, st);
    if (u2) return f16 ? launch_u2x<__half>(a, st) : launch_u2x<float>(a, st);
    if (a->group <= 4) return f16 ? launch_t<1, __half, false>(a, st) : launch_t<1, float, false>(a, st);
    return f16 ? launch_t<2, __half, false>(a, st) : launch_t<2, float, false>(a, st);
}

}  // namespace rdkv_b200

// the 128-B header of every tile, gathered for one D2H copy
__global__ void gather_headers_kernel(const uint8_t* __restrict__ arena, const int64_t* __restrict__ offs, int units,
                                      uint4* __restrict__ out) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= units * (kHeaderBytes / 16)) return;
    const int u = i / (kHeaderBytes / 16), j = i % (kHeaderBytes / 16);
    out[i] = reinterpret_cast<const uint4*>(arena + offs[u])[j];
}

// Scans every tile header once (one device gather + one D2H copy) and writes the
// per-tile decode sizes the persistent kernel stages with cp.async.bulk, plus
// the maxima that select the kernel variant and size its smem ring.
static int decode_prepare_impl(const uint8_t* arena, const int64_t* tile_offsets_host, int32_t units,
                               int32_t* decode_bytes_dev, int32_t* unit_ids_dev, rdkv_decode_plan* plan,
                               void* stream);

#ifdef RDKV_DECODE_EXPERIMENTS
extern "C" RDKV_API int rdkv_exp_set_u2x_trace(unsigned long long* buf) {
    return cudaMemcpyToSymbol(g_u2x_trace, &buf, sizeof(buf)) == cudaSuccess ? RDKV_OK : RDKV_ECUDA;
}
#endif
extern "C" RDKV_API int rdkv_cuda_decode_prepare(const uint8_t* arena, const int64_t* tile_offsets_host,
                                                 int32_t units, int32_t* decode_bytes_dev,
                                                 rdkv_decode_plan* plan, void* stream) {
    return decode_prepare_impl(arena, tile_offsets_host, units, decode_bytes_dev, nullptr, plan, stream);
}

extern "C" RDKV_API int rdkv_cuda_decode_prepare_split(const uint8_t* arena, const int64_t* tile_offsets_host,
                                                       int32_t units, int32_t* decode_bytes_dev,
                                                       int32_t* unit_ids_dev, rdkv_decode_plan* plan,
                                                       void* stream) {
    if (!unit_ids_dev) return RDKV_EINVAL;
    return decode_prepare_impl(arena, tile_offsets_host, units, decode_bytes_dev, unit_ids_dev, plan, stream);
}

static int decode_prepare_impl(const uint8_t* arena, const int64_t* tile_offsets_host, int32_t units,
                               int32_t* decode_bytes_dev, int32_t* unit_ids_dev, rdkv_decode_plan* plan,
                               void* stream) {
    if (!arena || !tile_offsets_host || !decode_bytes_dev || !plan || units < 1) return RDKV_EINVAL;
    auto st = static_cast<cudaStream_t>(stream);
    TileHeader* hdrs = static_cast<TileHeader*>(malloc(sizeof(TileHeader) * (size_t)units));
    int32_t* ds = static_cast<int32_t*>(malloc(sizeof(int32_t) * (size_t)units));
    int rc = RDKV_OK;
    // offsets come from rdkv_cuda_pack_plan (128-B aligned, any unit order); the gather reads
    // device memory at them, so reject malformed ones before launching it
    for (int u = 0; u < units; ++u)
        if (tile_offsets_host[u] < 0 || (tile_offsets_host[u] & (kTileAlign - 1))) {
            free(hdrs);
            free(ds);
            return RDKV_EINVAL;
        }
    if (units <= 64) {  // a few tiles: one small copy each
        for (int u = 0; u < units; ++u)
            cudaMemcpyAsync(&hdrs[u], arena + tile_offsets_host[u], sizeof(TileHeader), cudaMemcpyDeviceToHost, st);
        if (cudaStreamSynchronize(st) != cudaSuccess) rc = RDKV_ECUDA;
    } else {  // every tile header in one device gather and one D2H copy (not one copy per tile)
        int64_t* d_offs = nullptr;
        uint4* d_hdrs = nullptr;
        if (cudaMallocAsync(&d_offs, sizeof(int64_t) * (size_t)units, st) != cudaSuccess ||
            cudaMallocAsync(&d_hdrs, sizeof(TileHeader) * (size_t)units, st) != cudaSuccess ||
            cudaMemcpyAsync(d_offs, tile_offsets_host, sizeof(int64_t) * (size_t)units, cudaMemcpyHostToDevice, st) !=
                cudaSuccess) {
            rc = RDKV_ECUDA;
        } else {
            const int pieces = units * (kHeaderBytes / 16);
            gather_headers_kernel<<<(pieces + 255) / 256, 256, 0, st>>>(arena, d_offs, units, d_hdrs);
            if (cudaGetLastError() != cudaSuccess ||
                cudaMemcpyAsync(hdrs, d_hdrs, sizeof(TileHeader) * (size_t)units, cudaMemcpyDeviceToHost, st) !=
                    cudaSuccess)
                rc = RDKV_ECUDA;
        }
        if (d_offs) cudaFreeAsync(d_offs, st);
        if (d_hdrs) cudaFreeAsync(d_hdrs, st);
        if (cudaStreamSynchronize(st) != cudaSuccess) rc = RDKV_ECUDA;
    }
    rdkv_decode_plan p{0, 0, 0, 0, 2, 0, 2, 1, 1 << 30, 0};
    int32_t* ids = unit_ids_dev ? static_cast<int32_t*>(malloc(sizeof(int32_t) * (size_t)units)) : nullptr;
    int nmixed = 0, n_u = 0, n_m = 0;
    bool any_notfull = false, any_long = false, split_mix = false, split_notfull = false;
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
        const bool u2 = h.r[1] == 0 && h.r[2] == 0 && h.r[3] == 0 && h.c[1] == 0 && h.c[2] == 0 &&
                        h.c[3] == 0 && h.r[0] > 0 && h.c[0] > 0;
        // "mostly 2-bit" (heavy-hitter shape): the 2-bit K channels fill the first
        // 128 K slots, plus <= 32 4-bit channels and <= 8 4-bit V rows, short
        const bool m2 = !u2 && h.r[2] == 0 && h.r[3] == 0 && h.c[2] == 0 && h.c[3] == 0 && h.r[0] > 0 &&
                        h.c[0] > 96 && h.r[1] <= kMixMaxRows && h.nslot <= kU2MaxSlots &&
                        h.kslot_base[1] == 128 && h.kbyte_base[1] == 32;
        n_u += u2;
        n_m += m2;
        // mixed 2/4/8-bit tiles for the chunked split-K kernel (decode_u24)
        const bool t24 = h.r[3] == 0 && h.c[3] == 0 && h.n > 0 && (h.kslot_base[3] >> 5) <= kU24MaxK &&
                         h.c[0] + h.c[1] + h.c[2] > 0;
        if (!t24) {
            p.mix24 = 0;
        } else {
            U24Tile tt;
            u24_tile(h.r, tt);
            const int C = u24_nchunks(tt);
            p.min_chunks24 = C < p.min_chunks24 ? C : p.min_chunks24;
            p.max_krow_bytes24 = h.krow_bytes > p.max_krow_bytes24 ? h.krow_bytes : p.max_krow_bytes24;
        }
        if (u2 && h.c[0] != kD) any_notfull = true;
        if (u2 && h.nslot > kU2MaxSlots) any_long = true;
        if (ids) {  // split lists: short uniform / mostly-2-bit tiles first (in order), the rest from the back
            if ((u2 || m2) && h.nslot <= kU2MaxSlots) {
                ids[p.n_uniform++] = u;
                if (m2) split_mix = true;
                else if (h.c[0] != kD) split_notfull = true;
            } else {
                ids[units - 1 - nmixed++] = u;
            }
        }
    }
    // 2: all tiles uniform 2-bit with all d K channels; 1: uniform 2-bit; 3: every
    // tile uniform or mostly 2-bit and short (the MIX kernel); 0: anything else
    p.uniform2 = n_u == units ? (any_notfull ? 1 : 2) : (n_u + n_m == units && !any_long ? 3 : 0);
    p.uniform2_split = split_mix ? 3 : split_notfull ? 1 : 2;
    if (!p.mix24) p.min_chunks24 = p.max_krow_bytes24 = 0;
    if (ids) {  // the mixed tail back in unit order
        for (int i = p.n_uniform, j = units - 1; i < j; ++i, --j) {
            const int32_t t = ids[i];
            ids[i] = ids[j];
            ids[j] = t;
        }
        if (p.n_uniform == 0) p.uniform2_split = 0;
    }
    if (rc == RDKV_OK) {
        if (cudaMemcpyAsync(decode_bytes_dev, ds, sizeof(int32_t) * (size_t)units, cudaMemcpyHostToDevice, st) !=
                cudaSuccess ||
            (ids && cudaMemcpyAsync(unit_ids_dev, ids, sizeof(int32_t) * (size_t)units, cudaMemcpyHostToDevice, st) !=
                        cudaSuccess) ||
            cudaStreamSynchronize(st) != cudaSuccess)
            rc = RDKV_ECUDA;
        *plan = p;
    }
    free(hdrs);
    free(ds);
    free(ids);
    return rc;
}
