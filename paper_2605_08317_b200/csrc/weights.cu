// weights.cu — K1: post-prefill distortion-weight pass (Stage 1).
//
// Replaces, per (batch, layer, KV head) unit:
//   attention_probe  cache.cpp:140-184    causal probe softmax, fp64
//   token_weights    weights.cpp:25-46    column mass, heads-outer/rows-inner
//   moving_average   weights.cpp:8-23     centred zero-padded pool
//   channel_weights  weights.cpp:69-91    ||Q[:,c]|| ||K[:,c]|| / sqrt(d)
// as used by allocate_head (pipeline.cpp:124-146).
//
// Exactness: the probe logits are fp64 dot products of f32 inputs. Every
// product of two f32 values is exact in fp64, so DFMA(q, k, acc) rounds
// exactly like the reference's separate multiply and add — the logits are
// bit-identical. The per-token column sums keep the reference order (one
// thread per token walks the rows heads-outer, rows-inner). The remaining
// differences are the exp() implementation (CUDA vs glibc, <=1 ulp) and the
// softmax denominator's summation order; after the f32 cast the weights match
// the reference almost always bit-for-bit (tests report the exact-match rate).
//
// Kernels (per call, over all units):
//   W1 probe_logits   64 rows x 64 tokens per CTA, fp64 DFMA from smem,
//                     writes fp64 logits [U][R][T] + per-tile row max
//   W2 probe_softmax  one CTA per (unit, row): max, e = exp(l - max) in place,
//                     denominator
//   W3 token_raw      one thread per (unit, token): sum_rows e / denom -> f32
//   W4 token_pool     5-tap (pool_kernel) zero-padded mean -> w_t
//   W5 channel_norms  one thread per (unit, channel): sequential fp64 norms
// This file is compiled with -fmad=false; the only fused multiply-adds are
// the explicit __fma_rn calls in W1/W5, which are exact-equivalent there.
#include <algorithm>
#include <type_traits>

#include "common.cuh"

namespace rdkv_b200 {

constexpr int kW1Rows = 64;
constexpr int kW1Toks = 64;
constexpr int kW1Chunk = 32;

template <typename T>
__global__ void __launch_bounds__(256) probe_logits_kernel(
    const T* __restrict__ k, const T* __restrict__ q, int t_len, int d, int rows_total,
    int window, int probe_rows, int group, double inv_sqrt_d, int row_tiles,
    double* __restrict__ logits, double* __restrict__ tile_max, const int* __restrict__ offsets) {
    __shared__ double qs[kW1Rows][kW1Chunk + 1];
    __shared__ double ks[kW1Toks][kW1Chunk + 1];
    const int unit = blockIdx.y / row_tiles;
    const int row0 = (blockIdx.y % row_tiles) * kW1Rows;
    const int tok0 = blockIdx.x * kW1Toks;
    const int tid = threadIdx.x;
    const int tx = tid & 15, ty = tid >> 4;
    const size_t kbase = (size_t)unit * t_len * d;
    const size_t qbase = (size_t)unit * group * probe_rows * d;

    double acc[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = 0.0;

    for (int c0 = 0; c0 < d; c0 += kW1Chunk) {
        for (int e = tid; e < kW1Rows * kW1Chunk; e += 256) {
            const int lr = e / kW1Chunk, cc = e % kW1Chunk;
            const int row = row0 + lr, c = c0 + cc;
            double val = 0.0;
            if (row < rows_total && c < d) {
                const int qi = row / window, r = row % window;
                const size_t src = qbase + ((size_t)qi * probe_rows + (probe_rows - window + r)) * d + c;
                val = (double)load_as_float(q, src);
            }
            qs[lr][cc] = val;
        }
        for (int e = tid; e < kW1Toks * kW1Chunk; e += 256) {
            const int lt = e / kW1Chunk, cc = e % kW1Chunk;
            const int t = tok0 + lt, c = c0 + cc;
            ks[lt][cc] = (t < t_len && c < d) ? (double)load_as_float(k, kbase + (size_t)t * d + c) : 0.0;
        }
        __syncthreads();
        const int cn = min(kW1Chunk, d - c0);
        for (int cc = 0; cc < cn; ++cc) {
            double qv[4], kv[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) qv[i] = qs[ty + 16 * i][cc];
#pragma unroll
            for (int j = 0; j < 4; ++j) kv[j] = ks[tx + 16 * j][cc];
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) acc[i][j] = __fma_rn(qv[i], kv[j], acc[i][j]);
        }
        __syncthreads();
    }

    const int ntt = gridDim.x;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int row = row0 + ty + 16 * i;
        const int r = row % window;
        // causal offset (pipeline.cpp:129-130) unless the caller gives one per row
        const int off = offsets ? offsets[row] : t_len - window + r;
        double mx = -INFINITY;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int t = tok0 + tx + 16 * j;
            const double l = __dmul_rn(acc[i][j], inv_sqrt_d);
            if (row < rows_total && t < t_len) {
                logits[((size_t)unit * rows_total + row) * t_len + t] = l;
                if (t <= off) mx = fmax(mx, l);
            }
        }
#pragma unroll
        for (int o = 8; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        if (tx == 0 && row < rows_total) tile_max[((size_t)unit * rows_total + row) * ntt + blockIdx.x] = mx;
    }
}

__global__ void __launch_bounds__(256) probe_softmax_kernel(double* __restrict__ logits,
                                                            const double* __restrict__ tile_max,
                                                            int ntt, int t_len, int window,
                                                            int rows_total,
                                                            double* __restrict__ denom,
                                                            const int* __restrict__ offsets) {
    __shared__ double red[8];
    const int ur = blockIdx.x;  // unit * rows_total + row
    const int row = ur % rows_total;
    const int off = offsets ? offsets[row] : t_len - window + (row % window);
    double mx = -INFINITY;
    for (int i = threadIdx.x; i < ntt; i += blockDim.x) mx = fmax(mx, tile_max[(size_t)ur * ntt + i]);
    mx = warp_max_d(mx);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mx;
    __syncthreads();
    mx = red[0];
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) mx = fmax(mx, red[w]);
    __syncthreads();

    double* row_p = logits + (size_t)ur * t_len;
    double s = 0.0;
    // contiguous chunks per thread keep each partial a sequential sum
    const int per = (t_len + blockDim.x - 1) / blockDim.x;
    const int t0 = threadIdx.x * per;
    const int t1 = min(t_len, t0 + per);
    for (int t = t0; t < t1; ++t) {
        double e = 0.0;
        if (t <= off) {
            e = exp(row_p[t] - mx);
            s += e;
        }
        row_p[t] = e;  // entries past the causal offset are exactly zero (cache.cpp:181)
    }
    s = warp_sum_d(s);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        double tot = 0.0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) tot += red[w];
        denom[ur] = tot;
    }
}

__global__ void token_raw_kernel(const double* __restrict__ e, const double* __restrict__ denom,
                                 int units, int rows_total, int t_len, float* __restrict__ rawf) {
    const size_t idx = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
    if (idx >= (size_t)units * t_len) return;
    const int unit = (int)(idx / t_len);
    const int t = (int)(idx % t_len);
    const double* base = e + (size_t)unit * rows_total * t_len + t;
    const double* dn = denom + (size_t)unit * rows_total;
    double acc = 0.0;
    for (int row = 0; row < rows_total; ++row) acc = __dadd_rn(acc, base[(size_t)row * t_len] / dn[row]);
    rawf[idx] = (float)acc;
}

__global__ void token_pool_kernel(const float* __restrict__ rawf, int units, int t_len, int kernel,
                                  float* __restrict__ w_t) {
    const size_t idx = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
    if (idx >= (size_t)units * t_len) return;
    const int t = (int)(idx % t_len);
    const float* row = rawf + (idx - t);
    const int half = kernel / 2;
    const int lo = max(0, t - half), hi = min(t_len - 1, t + half);
    double acc = 0.0;
    for (int j = lo; j <= hi; ++j) acc = __dadd_rn(acc, (double)row[j]);
    w_t[idx] = (float)(acc / kernel);
}

template <typename T>
__global__ void channel_norm_kernel(const T* __restrict__ k, const T* __restrict__ q, int units,
                                    int t_len, int d, int window, int probe_rows, int group,
                                    double inv_sqrt_d, float* __restrict__ w_c) {
    const int idx = blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= units * d) return;
    const int unit = idx / d, c = idx % d;
    double qq = 0.0, kk = 0.0;
    const size_t qbase = (size_t)unit * group * probe_rows * d;
    for (int qi = 0; qi < group; ++qi) {
        for (int r = 0; r < window; ++r) {
            const double x = load_as_float(q, qbase + ((size_t)qi * probe_rows + probe_rows - window + r) * d + c);
            qq = __fma_rn(x, x, qq);
        }
    }
    const size_t kbase = (size_t)unit * t_len * d + c;
#pragma unroll 8
    for (int t = 0; t < t_len; ++t) {
        const double x = load_as_float(k, kbase + (size_t)t * d);
        kk = __fma_rn(x, x, kk);
    }
    w_c[idx] = (float)__dmul_rn(__dmul_rn(sqrt(qq), sqrt(kk)), inv_sqrt_d);
}

// ---------------------------------------------------------------------------
// Streaming K1 (the production path of rdkv_cuda_weights when d % 16 == 0):
// the U x R x T probe matrix is never materialised. Two passes of the same
// fp64 tile GEMM over (128 probe rows x 128 tokens) tiles:
//   S1 probe_stream<0>: logits -> per (row, token tile) max m and sum of
//      exp(l - m) over the causal part                      -> stats [U][R][ntt]
//   S2 probe_rowstat:   per row M = max m, denom = sum_tiles s * exp(m - M)
//                       (tile order)                        -> rowstat [U][R]
//   S3 probe_stream<1>: logits again, a = exp(l - M) / denom (cache.cpp:176-180),
//      column sums over the rows in the reference's heads-outer / rows-inner
//      order (weights.cpp:36-39), one thread per token      -> rawf [U][T]
//   W4 token_pool, and channel norms by chunked partial sums (S4/S5).
// The logits are the same bit-exact fp64 dots as W1 (sequential in c, DFMA of
// exact f32 products). The denominator's summation order differs from the
// reference's sequential one (<= 1e-15 relative; the f32 weights match it
// bit-for-bit except at rounding ties). GEMM tile: thread (tx, ty) holds rows
// ty + 16 i and tokens tx + 16 j (i, j < 8); per channel the 16 row values of
// a half-warp are two broadcast addresses and its 16 token values one
// 128-B wavefront, so shared memory stays under the DFMA rate.
constexpr int kSRows = 128;
constexpr int kSToks = 128;
constexpr int kSK = 16;                     // channels per staged chunk
constexpr int kSPad = kSRows + 2;           // smem row stride (doubles) of a chunk
constexpr int kSAStride = kSToks + 1;       // epilogue a-tile stride (doubles)
constexpr int kSGemmSmem = 2 * 2 * kSK * kSPad * (int)sizeof(double);
constexpr int kSColSmem = kSRows * kSAStride * (int)sizeof(double);
constexpr int kSSmem = kSGemmSmem > kSColSmem ? kSGemmSmem : kSColSmem;

template <typename T, int PASS>
__global__ void __launch_bounds__(256, 1) probe_stream_kernel(
    const T* __restrict__ k, const T* __restrict__ q, int t_len, int d, int R, int window, int probe_rows,
    double inv_sqrt_d, int ntt, double2* __restrict__ stats, const double2* __restrict__ rowstat,
    float* __restrict__ rawf) {
    extern __shared__ __align__(16) double sm[];
    const int tile = blockIdx.x, unit = blockIdx.y;
    const int tok0 = tile * kSToks;
    const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
    const T* kb = k + (size_t)unit * t_len * d;
    const T* qb = q + (size_t)unit * (R / window) * probe_rows * d;
    // loader mapping: channel lc, rows / tokens lr + 16 m
    const int lc = tid & 15, lr = tid >> 4;
    const int nchunk = d / kSK;
    double colacc = 0.0;  // S3: the column sum of token tok0 + tid (tid < 128), in row order
    for (int rb = 0; rb < R; rb += kSRows) {
        double acc[8][8];
#pragma unroll
        for (int i = 0; i < 8; ++i)
#pragma unroll
            for (int j = 0; j < 8; ++j) acc[i][j] = 0.0;
        float qv_n[8], kv_n[8];
        auto gload = [&](int c0) {
#pragma unroll
            for (int m = 0; m < 8; ++m) {
                const int row = rb + lr + 16 * m, t = tok0 + lr + 16 * m;
                const int qi = row / window, w = row - qi * window;
                qv_n[m] = row < R ? load_as_float(qb, ((size_t)qi * probe_rows + probe_rows - window + w) * d + c0 + lc)
                                  : 0.0f;
                kv_n[m] = t < t_len ? load_as_float(kb, (size_t)t * d + c0 + lc) : 0.0f;
            }
        };
        gload(0);
        for (int kc = 0; kc < nchunk; ++kc) {
            double* Qs = sm + (kc & 1) * 2 * kSK * kSPad;
            double* Ks = Qs + kSK * kSPad;
#pragma unroll
            for (int m = 0; m < 8; ++m) {
                Qs[lc * kSPad + lr + 16 * m] = (double)qv_n[m];
                Ks[lc * kSPad + lr + 16 * m] = (double)kv_n[m];
            }
            __syncthreads();
            if (kc + 1 < nchunk) gload((kc + 1) * kSK);
#pragma unroll 4
            for (int kk = 0; kk < kSK; ++kk) {
                double a[8], b[8];
#pragma unroll
                for (int i = 0; i < 8; ++i) a[i] = Qs[kk * kSPad + ty + 16 * i];
#pragma unroll
                for (int j = 0; j < 8; ++j) b[j] = Ks[kk * kSPad + tx + 16 * j];
#pragma unroll
                for (int i = 0; i < 8; ++i)
#pragma unroll
                    for (int j = 0; j < 8; ++j) acc[i][j] = __fma_rn(a[i], b[j], acc[i][j]);
            }
        }
        __syncthreads();  // all chunk reads done: the smem may be reused below
        if (PASS == 0) {
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                const int row = rb + ty + 16 * i;
                const int off = t_len - window + (row % window);  // causal offset (pipeline.cpp:129-130)
                double l[8];
                double m = -INFINITY;
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    const int t = tok0 + tx + 16 * j;
                    l[j] = __dmul_rn(acc[i][j], inv_sqrt_d);
                    if (row < R && t < t_len && t <= off) m = fmax(m, l[j]);
                }
#pragma unroll
                for (int o = 1; o < 16; o <<= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
                double s = 0.0;
                if (m != -INFINITY) {
#pragma unroll
                    for (int j = 0; j < 8; ++j) {
                        const int t = tok0 + tx + 16 * j;
                        if (row < R && t < t_len && t <= off) s = __dadd_rn(s, exp(__dadd_rn(l[j], -m)));
                    }
                }
#pragma unroll
                for (int o = 1; o < 16; o <<= 1) s = __dadd_rn(s, __shfl_xor_sync(0xffffffffu, s, o));
                if (tx == 0 && row < R) {  // (one stat per 128-token tile; the second half-tile slot stays empty)
                    stats[((size_t)unit * R + row) * ntt + 2 * tile] = make_double2(m, s);
                    stats[((size_t)unit * R + row) * ntt + 2 * tile + 1] = make_double2(-INFINITY, 0.0);
                }
            }
        } else {
            double* at = sm;
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                const int row = rb + ty + 16 * i;
                const int off = t_len - window + (row % window);
                const double2 ms = row < R ? rowstat[(size_t)unit * R + row] : make_double2(0.0, 1.0);
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    const int t = tok0 + tx + 16 * j;
                    double a = 0.0;  // entries past the causal offset are exactly zero (cache.cpp:181)
                    if (row < R && t < t_len && t <= off)
                        a = exp(__dadd_rn(__dmul_rn(acc[i][j], inv_sqrt_d), -ms.x)) / ms.y;
                    at[(ty + 16 * i) * kSAStride + tx + 16 * j] = a;
                }
            }
            __syncthreads();
            if (tid < kSToks) {
                const int nr = min(kSRows, R - rb);
                for (int r = 0; r < nr; ++r) colacc = __dadd_rn(colacc, at[r * kSAStride + tid]);
            }
            __syncthreads();  // the a-tile aliases the next row block's chunk buffers
        }
    }
    if (PASS == 1 && tid < kSToks && tok0 + tid < t_len) rawf[(size_t)unit * t_len + tok0 + tid] = (float)colacc;
}

// Staging helpers and sizes of the persistent probe kernel (probe_exact_kernel).
constexpr int kD128 = 128;
constexpr int kTMaxR = 256;              // probe rows resident (g * window <= 256)

__device__ __forceinline__ void cp_async16(void* dst, const void* src, bool valid) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"((uint32_t)__cvta_generic_to_shared(dst)),
                 "l"(src), "r"(valid ? 16 : 0)
                 : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// The production path (fp16, d = 128) with the reference's arithmetic order:
// the persistent, cp.async-pipelined staging of probe_tma_kernel with a DFMA
// register tile (thread (tx, ty): rows ty + 32 i, tokens tx + 16 j (i < 4,
// j < 8), channels in order c = 0 .. 127, each an exact f32 x f32 product
// fused into the fp64 sum — bit-identical logits). Every 32-channel chunk of
// the 128 probe rows and the 128-token K tile is widened to fp64 in shared
// memory once per CTA (rows padded to 272 B: a thread's two-channel 16-B loads
// are broadcast / conflict-free), so the fp64 pipe runs DFMAs, not one
// conversion per operand use (each value feeds 16 threads). This is S1:
// besides the half-tile (max, sum exp) stats it stores the logits [U][R][T] so
// S3 (probe_colsum_kernel) reads them back instead of running the GEMM again.
constexpr int kERow = 136;                     // padded row stride (fp16) = 272 B
constexpr int kEKBuf = kSToks * kERow;
constexpr int kEChunk = 32;                    // channels widened to fp64 per step
constexpr int kDRow = kEChunk + 2;             // fp64 row stride of a widened chunk (272 B: conflict-free)
constexpr int kESmem = (2 * kEKBuf + kTMaxR * kERow) * 2 + 2 * kSRows * kDRow * 8;
constexpr int kETile = 4;  // 4 x 8 tiles, 16 warps: S1 1.95 ms vs 2.04 with 8 x 8 tiles and 8 warps (same bits)

// TI probe rows per thread: 8 (256 threads, 8 x 8 DFMA register tile) or 4 (512
// threads, 4 x 8: half the registers, twice the warps to hide the latencies)
template <int TI>
__global__ void __launch_bounds__(16 * (kSRows / TI), 1) probe_exact_kernel(
    const __half* __restrict__ k, const __half* __restrict__ q, int units, int t_len, int R, int window,
    int probe_rows, double inv_sqrt_d, int ntt, int nht, double2* __restrict__ stats, double* __restrict__ logits) {
    constexpr int d = kD128;
    constexpr int NT = 16 * (kSRows / TI), RS = kSRows / TI;  // threads; row stride of a thread's rows
    extern __shared__ __align__(16) __half esm[];
    __half* kbuf = esm;                                // [2][128 tokens][kERow]
    __half* qbuf = esm + 2 * kEKBuf;                   // [R][kERow]
    double* qd = reinterpret_cast<double*>(qbuf + kTMaxR * kERow);  // [kSRows][kDRow] fp64 chunk of 128 probe rows
    double* kd = qd + kSRows * kDRow;                                // [kSToks][kDRow] fp64 chunk of the K tile
    const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
    const long long items = (long long)units * ntt;
    const long long i0 = items * blockIdx.x / gridDim.x, i1 = items * (blockIdx.x + 1) / gridDim.x;
    auto load_k = [&](long long it, int buf) {
        if (it < i1) {
            const int unit = (int)(it / ntt), tile = (int)(it % ntt);
            const __half* kb = k + ((size_t)unit * t_len + (size_t)tile * kSToks) * d;
            __half* dst = kbuf + buf * kEKBuf;
            for (int e = tid; e < kSToks * (d / 8); e += NT) {
                const int r = e >> 4, c8 = e & 15;
                const bool ok = tile * kSToks + r < t_len;
                cp_async16(dst + r * kERow + 8 * c8, ok ? kb + (size_t)r * d + 8 * c8 : kb, ok);
            }
        }
        cp_async_commit();
    };
    auto load_q = [&](int unit) {
        const __half* qb = q + (size_t)unit * (R / window) * probe_rows * d;
        for (int e = tid; e < R * (d / 8); e += NT) {
            const int r = e >> 4, c8 = e & 15;
            const int qi = r / window, w = r - qi * window;
            cp_async16(qbuf + r * kERow + 8 * c8, qb + ((size_t)qi * probe_rows + probe_rows - window + w) * d + 8 * c8,
                       true);
        }
    };
    int qunit = -1;
    if (i0 < i1) {
        qunit = (int)(i0 / ntt);
        load_q(qunit);
    }
    load_k(i0, 0);
    load_k(i0 + 1, 1);
    for (long long it = i0; it < i1; ++it) {
        const int buf = (int)((it - i0) & 1);
        const int unit = (int)(it / ntt), tile = (int)(it % ntt);
        const int tok0 = tile * kSToks;
        if (unit != qunit) {  // the unit's probe rows replace the previous unit's
            cp_async_wait<0>();
            __syncthreads();  // every thread is past its reads of the old rows
            load_q(unit);
            cp_async_commit();
            cp_async_wait<0>();  // the new rows (and the K tiles in flight) have landed
            qunit = unit;
        } else {
            cp_async_wait<1>();  // K(it) has landed; K(it + 1) may still be in flight
        }
        __syncthreads();
        const __half* Ks = kbuf + buf * kEKBuf;
        for (int rb = 0; rb < R; rb += kSRows) {
            double acc[TI][8];
#pragma unroll
            for (int i = 0; i < TI; ++i)
#pragma unroll
                for (int j = 0; j < 8; ++j) acc[i][j] = 0.0;
#pragma unroll 1
            for (int c0 = 0; c0 < d; c0 += kEChunk) {
                // widen this chunk's probe rows and K tokens to fp64 once per CTA
                // (not once per use: 16 threads read every value)
                __syncthreads();  // the previous chunk's readers are done
#pragma unroll
                for (int e = tid; e < 2 * kSRows * (kEChunk / 8); e += NT) {
                    const bool isk = e >= kSRows * (kEChunk / 8);
                    const int u = isk ? e - kSRows * (kEChunk / 8) : e;
                    const int r = u % kSRows, c8 = u / kSRows;  // a quarter-warp: 8 rows, one column group
                    const __half* src = isk ? Ks + r * kERow + c0 + 8 * c8 : qbuf + (size_t)(rb + r) * kERow + c0 + 8 * c8;
                    const uint4 v = (isk || rb + r < R) ? *reinterpret_cast<const uint4*>(src) : make_uint4(0, 0, 0, 0);
                    const __half* hv = reinterpret_cast<const __half*>(&v);
                    double2* dst = reinterpret_cast<double2*>((isk ? kd : qd) + r * kDRow + 8 * c8);
#pragma unroll
                    for (int m = 0; m < 4; ++m)
                        dst[m] = make_double2((double)__half2float(hv[2 * m]), (double)__half2float(hv[2 * m + 1]));
                }
                __syncthreads();
#pragma unroll 2
                for (int c = 0; c < kEChunk; c += 2) {
                    double2 a[TI], b[8];
#pragma unroll
                    for (int i = 0; i < TI; ++i) a[i] = *reinterpret_cast<const double2*>(qd + (ty + RS * i) * kDRow + c);
#pragma unroll
                    for (int j = 0; j < 8; ++j) b[j] = *reinterpret_cast<const double2*>(kd + (tx + 16 * j) * kDRow + c);
#pragma unroll
                    for (int i = 0; i < TI; ++i)
#pragma unroll
                        for (int j = 0; j < 8; ++j) acc[i][j] = __fma_rn(a[i].x, b[j].x, acc[i][j]);
#pragma unroll
                    for (int i = 0; i < TI; ++i)
#pragma unroll
                        for (int j = 0; j < 8; ++j) acc[i][j] = __fma_rn(a[i].y, b[j].y, acc[i][j]);
                }
            }
#pragma unroll
            for (int i = 0; i < TI; ++i) {
                const int row = rb + ty + RS * i;
                const int off = t_len - window + (row % window);  // causal offset (pipeline.cpp:129-130)
                double l[8];
                double m = -INFINITY;
                double* lrow = logits + ((size_t)unit * R + row) * t_len;
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    const int t = tok0 + tx + 16 * j;
                    l[j] = __dmul_rn(acc[i][j], inv_sqrt_d);
                    if (row < R && t < t_len && t <= off) m = fmax(m, l[j]);
                    if (row < R && t < t_len) lrow[t] = l[j];
                }
#pragma unroll
                for (int o = 1; o < 16; o <<= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
                double sm_ = 0.0;
                if (m != -INFINITY) {
#pragma unroll
                    for (int j = 0; j < 8; ++j) {
                        const int t = tok0 + tx + 16 * j;
                        if (row < R && t < t_len && t <= off) sm_ = __dadd_rn(sm_, exp(__dadd_rn(l[j], -m)));
                    }
                }
#pragma unroll
                for (int o = 1; o < 16; o <<= 1) sm_ = __dadd_rn(sm_, __shfl_xor_sync(0xffffffffu, sm_, o));
                if (tx == 0 && row < R) {
                    stats[((size_t)unit * R + row) * nht + 2 * tile] = make_double2(m, sm_);
                    stats[((size_t)unit * R + row) * nht + 2 * tile + 1] = make_double2(-INFINITY, 0.0);
                }
            }
        }
        __syncthreads();
        load_k(it + 2, buf);
    }
    cp_async_wait<0>();
}

// S3 from the logits S1 stored (fp16, d = 128): a = exp(l - M) / denom
// (cache.cpp:176-180), each token's column summed over the rows in order
// (weights.cpp:36-39) — the same expressions on the same values as the
// recomputing pass, so the same bits, without the second GEMM. Thread per
// token; the row loop is unrolled so the coalesced loads run ahead of the
// sequential sum.
__global__ void __launch_bounds__(256) probe_colsum_kernel(const double* __restrict__ logits,
                                                           const double2* __restrict__ rowstat, int R, int t_len,
                                                           int window, float* __restrict__ rawf) {
    const int unit = blockIdx.y, t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= t_len) return;
    const double* lu = logits + (size_t)unit * R * t_len + t;
    const double2* rs = rowstat + (size_t)unit * R;
    double colacc = 0.0;
    // causal offset of row r = qi * window + w: t_len - window + w (pipeline.cpp:129-130)
    for (int r0 = 0; r0 < R; r0 += window) {
#pragma unroll 8
        for (int w = 0; w < window; ++w) {
            const double l = lu[(size_t)(r0 + w) * t_len];
            const double2 ms = rs[r0 + w];
            const double a = t <= t_len - window + w ? exp(__dadd_rn(l, -ms.x)) / ms.y : 0.0;  // past it: exactly zero
            colacc = __dadd_rn(colacc, a);
        }
    }
    rawf[(size_t)unit * t_len + t] = (float)colacc;
}

// S2: per (unit, row) global max and softmax denominator from the tile stats,
// one warp per row (lane-strided tiles, fixed shuffle tree: deterministic).
__global__ void probe_rowstat_kernel(const double2* __restrict__ stats, int rows, int ntt,
                                     double2* __restrict__ rowstat) {
    const int ur = (int)((blockIdx.x * (size_t)blockDim.x + threadIdx.x) >> 5), lane = threadIdx.x & 31;
    if (ur >= rows) return;
    const double2* st = stats + (size_t)ur * ntt;
    double M = -INFINITY;
    for (int i = lane; i < ntt; i += 32) M = fmax(M, st[i].x);
    M = warp_max_d(M);
    double den = 0.0;
    for (int i = lane; i < ntt; i += 32) {
        const double2 v = st[i];
        if (v.y > 0.0) den = __dadd_rn(den, __dmul_rn(v.y, exp(__dadd_rn(v.x, -M))));
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) den = __dadd_rn(den, __shfl_xor_sync(0xffffffffu, den, o));
    if (lane == 0) rowstat[ur] = make_double2(M, den);
}

// S4: channel norm partials, one CTA per (unit, chunk of kCNChunk tokens):
// thread j sums k[t][c]^2 for channels c = 2j, 2j + 1 over the chunk's tokens
// in order (fp64 DFMA of an exact square; one 4-B load per row and thread, so a
// warp reads 128 contiguous bytes of each row).
constexpr int kCNChunk = 256;
template <typename T>
__global__ void channel_kk_partial_kernel(const T* __restrict__ k, int t_len, int d, int nchunks,
                                          double* __restrict__ part) {
    const int chunk = blockIdx.x, unit = blockIdx.y;
    const int t0 = chunk * kCNChunk, t1 = min(t_len, t0 + kCNChunk);
    const T* kb = k + (size_t)unit * t_len * d;
    for (int c = 2 * threadIdx.x; c < d; c += 2 * blockDim.x) {
        double k0 = 0.0, k1 = 0.0;
        const bool two = c + 1 < d;
#pragma unroll 8
        for (int t = t0; t < t1; ++t) {
            const double x0 = load_as_float(kb, (size_t)t * d + c);
            const double x1 = two ? (double)load_as_float(kb, (size_t)t * d + c + 1) : 0.0;
            k0 = __fma_rn(x0, x0, k0);
            k1 = __fma_rn(x1, x1, k1);
        }
        part[((size_t)unit * nchunks + chunk) * d + c] = k0;
        if (two) part[((size_t)unit * nchunks + chunk) * d + c + 1] = k1;
    }
}

// S5: w_c = f32(sqrt(sum q^2) * sqrt(sum k^2) / sqrt(d)) (weights.cpp:69-91),
// the K sum combined over the chunk partials in chunk order.
template <typename T>
__global__ void channel_norm_combine_kernel(const T* __restrict__ q, const double* __restrict__ part, int units,
                                            int nchunks, int d, int window, int probe_rows, int group,
                                            double inv_sqrt_d, float* __restrict__ w_c) {
    const int idx = blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= units * d) return;
    const int unit = idx / d, c = idx % d;
    double qq = 0.0;
    const size_t qbase = (size_t)unit * group * probe_rows * d;
    for (int qi = 0; qi < group; ++qi)
        for (int r = 0; r < window; ++r) {
            const double x = load_as_float(q, qbase + ((size_t)qi * probe_rows + probe_rows - window + r) * d + c);
            qq = __fma_rn(x, x, qq);
        }
    double kk = 0.0;
    for (int i = 0; i < nchunks; ++i) kk = __dadd_rn(kk, part[((size_t)unit * nchunks + i) * d + c]);
    w_c[idx] = (float)__dmul_rn(__dmul_rn(sqrt(qq), sqrt(kk)), inv_sqrt_d);
}

struct WeightsWorkspace {
    double* logits;
    double* tile_max;
    double* denom;
    float* rawf;
    size_t bytes;
};

// Workspace of the streaming path: tile stats [U][R][ntt] (m, s), row stats
// [U][R], raw column sums [U][T] f32, channel partials [U][nchunks][d].
struct StreamWorkspace {
    double2* stats;
    double2* rowstat;
    float* rawf;
    double* kpart;
    double* logits;  // fp16 d = 128 path: S1's logits of a batch of `ubatch` units, [ubatch][R][T]
    int ubatch;
    size_t bytes;
};

static bool stream_path(const rdkv_shape* s) { return s->head_dim % kSK == 0; }
// shapes the persistent exact kernel takes (for fp16 inputs)
static bool exact_shape(const rdkv_shape* s, int window) {
    return s->head_dim == kD128 && (size_t)s->group * window <= (size_t)kTMaxR;
}
constexpr size_t kLogitBudget = size_t(2) << 30;  // bytes of stored S1 logits per unit batch

static StreamWorkspace carve_stream(const rdkv_shape* s, int window, void* base) {
    const size_t U = s->units, T = s->seq_len, R = (size_t)s->group * window, d = s->head_dim;
    const size_t ntt = (T + kSToks - 1) / kSToks, nch = (T + kCNChunk - 1) / kCNChunk;
    StreamWorkspace w{};
    char* p = static_cast<char*>(base);
    size_t off = 0;
    auto take = [&](size_t n) {
        char* r = p ? p + off : nullptr;
        off += (n + 255) / 256 * 256;
        return r;
    };
    w.stats = reinterpret_cast<double2*>(take(U * R * 2 * ntt * sizeof(double2)));  // per 64-token half tile
    w.rowstat = reinterpret_cast<double2*>(take(U * R * sizeof(double2)));
    w.rawf = reinterpret_cast<float*>(take(U * T * sizeof(float)));
    w.kpart = reinterpret_cast<double*>(take(U * nch * d * sizeof(double)));
    w.logits = nullptr;
    w.ubatch = 0;
    if (exact_shape(s, window)) {
        const size_t per_unit = R * T * sizeof(double);
        w.ubatch = (int)std::max<size_t>(1, std::min<size_t>(U, kLogitBudget / per_unit));
        w.logits = reinterpret_cast<double*>(take((size_t)w.ubatch * per_unit));
    }
    w.bytes = off;
    return w;
}

template <typename T>
static int run_weights_stream(const T* k, const T* q, const rdkv_shape* s, int window, int pool_kernel, float* w_t,
                              float* w_c, const StreamWorkspace& ws, cudaStream_t st) {
    const int U = s->units, t_len = s->seq_len, d = s->head_dim, g = s->group;
    const int R = g * window;
    const double inv_sqrt_d = 1.0 / sqrt((double)d);
    const int ntt = (t_len + kSToks - 1) / kSToks;
    static std::atomic<int> smem0[kMaxDevices], smem1[kMaxDevices];
    const int dev = dev_attrs().dev;
    const dim3 grid(ntt, U);
    const int nht = 2 * ntt;  // stats per 64-token half tile
    if (std::is_same<T, __half>::value && ws.logits) {
        // S1 stores its logits (a batch of units at a time), S3 reads them back
        static std::atomic<int> tsm0[kMaxDevices];
        set_smem_once(probe_exact_kernel<kETile>, kESmem, tsm0, dev);
        for (int u0 = 0; u0 < U; u0 += ws.ubatch) {
            const int ub = std::min(ws.ubatch, U - u0);
            const long long items = (long long)ub * ntt;
            const int nblk = (int)(items < dev_attrs().nsm ? items : dev_attrs().nsm);
            const __half* kh = reinterpret_cast<const __half*>(k) + (size_t)u0 * t_len * d;
            const __half* qh = reinterpret_cast<const __half*>(q) + (size_t)u0 * g * s->probe_rows * d;
            double2* stats = ws.stats + (size_t)u0 * R * nht;
            double2* rowstat = ws.rowstat + (size_t)u0 * R;
            probe_exact_kernel<kETile><<<nblk, 16 * (kSRows / kETile), kESmem, st>>>(kh, qh, ub, t_len, R, window,
                                                                               s->probe_rows, inv_sqrt_d,
                                                          ntt, nht, stats, ws.logits);
            probe_rowstat_kernel<<<(ub * R * 32 + 255) / 256, 256, 0, st>>>(stats, ub * R, nht, rowstat);
            probe_colsum_kernel<<<dim3((t_len + 255) / 256, ub), 256, 0, st>>>(ws.logits, rowstat, R, t_len, window,
                                                                              ws.rawf + (size_t)u0 * t_len);
        }
    } else {
        // f32 inputs (the reference-shaped drop-in path) and other shapes: the DFMA tile
        // GEMM, whose dots keep the reference's sequential fp64 order (bit-identical logits)
        set_smem_once(probe_stream_kernel<T, 0>, kSSmem, smem0, dev);
        set_smem_once(probe_stream_kernel<T, 1>, kSSmem, smem1, dev);
        probe_stream_kernel<T, 0><<<grid, 256, kSSmem, st>>>(k, q, t_len, d, R, window, s->probe_rows, inv_sqrt_d, nht,
                                                              ws.stats, nullptr, nullptr);
        probe_rowstat_kernel<<<(U * R * 32 + 255) / 256, 256, 0, st>>>(ws.stats, U * R, nht, ws.rowstat);
        probe_stream_kernel<T, 1><<<grid, 256, kSSmem, st>>>(k, q, t_len, d, R, window, s->probe_rows, inv_sqrt_d, nht,
                                                              nullptr, ws.rowstat, ws.rawf);
    }
    const size_t nt = (size_t)U * t_len;
    token_pool_kernel<<<(unsigned)((nt + 255) / 256), 256, 0, st>>>(ws.rawf, U, t_len, pool_kernel, w_t);
    const int nch = (t_len + kCNChunk - 1) / kCNChunk;
    channel_kk_partial_kernel<T><<<dim3(nch, U), 64, 0, st>>>(k, t_len, d, nch, ws.kpart);
    channel_norm_combine_kernel<T><<<(U * d + 127) / 128, 128, 0, st>>>(q, ws.kpart, U, nch, d, window, s->probe_rows,
                                                                       g, inv_sqrt_d, w_c);
    return launch_status();
}

static WeightsWorkspace carve(const rdkv_shape* s, int window, void* base) {
    const size_t U = s->units, T = s->seq_len, R = (size_t)s->group * window;
    const size_t ntt = (T + kW1Toks - 1) / kW1Toks;
    WeightsWorkspace w{};
    char* p = static_cast<char*>(base);
    size_t off = 0;
    auto take = [&](size_t n) {
        char* r = p ? p + off : nullptr;
        off += (n + 255) / 256 * 256;
        return r;
    };
    w.logits = reinterpret_cast<double*>(take(U * R * T * sizeof(double)));
    w.tile_max = reinterpret_cast<double*>(take(U * R * ntt * sizeof(double)));
    w.denom = reinterpret_cast<double*>(take(U * R * sizeof(double)));
    w.rawf = reinterpret_cast<float*>(take(U * T * sizeof(float)));
    w.bytes = off;
    return w;
}

template <typename T>
static int run_weights(const T* k, const T* q, const rdkv_shape* s, int window, int pool_kernel,
                       float* w_t, float* w_c, const WeightsWorkspace& ws, cudaStream_t st) {
    const int U = s->units, t_len = s->seq_len, d = s->head_dim, g = s->group;
    const int R = g * window;
    const double inv_sqrt_d = 1.0 / sqrt((double)d);
    const int ntt = (t_len + kW1Toks - 1) / kW1Toks;
    const int row_tiles = (R + kW1Rows - 1) / kW1Rows;
    dim3 grid1(ntt, U * row_tiles);
    probe_logits_kernel<T><<<grid1, 256, 0, st>>>(k, q, t_len, d, R, window, s->probe_rows, g,
                                                  inv_sqrt_d, row_tiles, ws.logits, ws.tile_max, nullptr);
    probe_softmax_kernel<<<U * R, 256, 0, st>>>(ws.logits, ws.tile_max, ntt, t_len, window, R, ws.denom, nullptr);
    const size_t nt = (size_t)U * t_len;
    token_raw_kernel<<<(unsigned)((nt + 255) / 256), 256, 0, st>>>(ws.logits, ws.denom, U, R, t_len, ws.rawf);
    token_pool_kernel<<<(unsigned)((nt + 255) / 256), 256, 0, st>>>(ws.rawf, U, t_len, pool_kernel, w_t);
    channel_norm_kernel<T><<<(U * d + 127) / 128, 128, 0, st>>>(k, q, U, t_len, d, window,
                                                               s->probe_rows, g, inv_sqrt_d, w_c);
    return launch_status();
}

}  // namespace rdkv_b200

using namespace rdkv_b200;

extern "C" RDKV_API size_t rdkv_cuda_weights_workspace(const rdkv_shape* s, int32_t window) {
    if (!s || window < 1) return 0;
    const int w = window < s->probe_rows ? window : s->probe_rows;
    return stream_path(s) ? carve_stream(s, w, nullptr).bytes : carve(s, w, nullptr).bytes;
}

extern "C" RDKV_API int rdkv_cuda_weights(const void* k, const void* probe_q, int32_t dtype,
                                          const rdkv_shape* s, int32_t window, int32_t pool_kernel,
                                          float* w_t, float* w_c, void* workspace,
                                          size_t workspace_bytes, void* stream) {
    if (!s || !k || !probe_q || !w_t || !w_c) return RDKV_EINVAL;
    if (s->units < 1 || s->seq_len < 1 || s->head_dim < 1 || s->group < 1 || s->probe_rows < 1)
        return RDKV_EINVAL;
    if (s->probe_rows > s->seq_len) return RDKV_EINVAL;  // KVCache::validate (cache.cpp:116-118)
    if (window < 1 || pool_kernel < 1 || pool_kernel % 2 == 0) return RDKV_EINVAL;  // cache.cpp:107-112
    const int w = window < s->probe_rows ? window : s->probe_rows;  // pipeline.cpp:125
    auto st = static_cast<cudaStream_t>(stream);
    if (stream_path(s)) {
        StreamWorkspace ws = carve_stream(s, w, workspace);
        if (!workspace || workspace_bytes < ws.bytes) return RDKV_EINVAL;
        if (dtype == RDKV_F32)
            return run_weights_stream(static_cast<const float*>(k), static_cast<const float*>(probe_q), s, w,
                                      pool_kernel, w_t, w_c, ws, st);
        if (dtype == RDKV_F16)
            return run_weights_stream(static_cast<const __half*>(k), static_cast<const __half*>(probe_q), s, w,
                                      pool_kernel, w_t, w_c, ws, st);
        return RDKV_EINVAL;
    }
    WeightsWorkspace ws = carve(s, w, workspace);
    if (!workspace || workspace_bytes < ws.bytes) return RDKV_EINVAL;
    if (dtype == RDKV_F32)
        return run_weights(static_cast<const float*>(k), static_cast<const float*>(probe_q), s, w,
                           pool_kernel, w_t, w_c, ws, st);
    if (dtype == RDKV_F16)
        return run_weights(static_cast<const __half*>(k), static_cast<const __half*>(probe_q), s, w,
                           pool_kernel, w_t, w_c, ws, st);
    return RDKV_EINVAL;
}

// ---------------------------------------------------------------------------
// Single-function entry points behind the C++ drop-in API (include/rdkv/):
// attention_probe with arbitrary causal offsets (cache.cpp:140-184),
// token_weights over given attention matrices (weights.cpp:25-46),
// moving_average (weights.cpp:8-23), channel_weights (weights.cpp:69-91).
namespace rdkv_b200 {

__global__ void probe_normalize_kernel(double* __restrict__ e, const double* __restrict__ denom, int rows,
                                       int t_len, const int* __restrict__ offsets) {
    const size_t idx = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
    if (idx >= (size_t)rows * t_len) return;
    const int r = (int)(idx / t_len), t = (int)(idx % t_len);
    e[idx] = t <= offsets[r] ? e[idx] / denom[r] : 0.0;
}

__global__ void offsets_check_kernel(const int* __restrict__ offsets, int rows, int t_len, int* __restrict__ bad) {
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r < rows && (offsets[r] < 0 || offsets[r] >= t_len)) atomicOr(bad, 1);
}

__global__ void column_sum_kernel(const double* __restrict__ a, int heads, int rows, int t_len,
                                  float* __restrict__ rawf) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= t_len) return;
    double acc = 0.0;
    for (int hr = 0; hr < heads * rows; ++hr) acc = __dadd_rn(acc, a[(size_t)hr * t_len + t]);
    rawf[t] = (float)acc;
}

template <typename T>
__global__ void channel_norm_rows_kernel(const T* __restrict__ q, int q_rows, const T* __restrict__ k, int k_rows,
                                         int d, double inv_sqrt_d, float* __restrict__ w_c) {
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= d) return;
    double qq = 0.0, kk = 0.0;
    for (int r = 0; r < q_rows; ++r) {
        const double x = load_as_float(q, (size_t)r * d + c);
        qq = __fma_rn(x, x, qq);
    }
#pragma unroll 8
    for (int r = 0; r < k_rows; ++r) {
        const double x = load_as_float(k, (size_t)r * d + c);
        kk = __fma_rn(x, x, kk);
    }
    w_c[c] = (float)__dmul_rn(__dmul_rn(sqrt(qq), sqrt(kk)), inv_sqrt_d);
}

}  // namespace rdkv_b200

extern "C" RDKV_API size_t rdkv_cuda_attention_probe_workspace(int32_t rows, int32_t t_len) {
    rdkv_shape s{1, t_len, 1, 1, rows, 1};
    return carve(&s, rows, nullptr).bytes + 256;
}

extern "C" RDKV_API int rdkv_cuda_attention_probe(const float* q, int32_t rows, const float* k, int32_t t_len,
                                                  int32_t d, const int32_t* offsets, double* a, void* workspace,
                                                  size_t workspace_bytes, void* stream) {
    if (!q || !k || !offsets || !a || rows < 1 || t_len < 1 || d < 1) return RDKV_EINVAL;
    rdkv_shape s{1, t_len, d, 1, rows, 1};
    WeightsWorkspace ws = carve(&s, rows, workspace);
    if (!workspace || workspace_bytes < ws.bytes + 256) return RDKV_EINVAL;
    int* bad = reinterpret_cast<int*>(static_cast<char*>(workspace) + ws.bytes);
    auto st = static_cast<cudaStream_t>(stream);
    RDKV_CUDA_TRY(cudaMemsetAsync(bad, 0, sizeof(int), st));
    offsets_check_kernel<<<(rows + 127) / 128, 128, 0, st>>>(offsets, rows, t_len, bad);
    int hbad = 0;
    RDKV_CUDA_TRY(cudaMemcpyAsync(&hbad, bad, sizeof(int), cudaMemcpyDeviceToHost, st));
    RDKV_CUDA_TRY(cudaStreamSynchronize(st));
    if (hbad) return RDKV_EINVAL;  // cache.cpp:162-164
    const double inv_sqrt_d = 1.0 / sqrt((double)d);
    const int ntt = (t_len + kW1Toks - 1) / kW1Toks;
    const int row_tiles = (rows + kW1Rows - 1) / kW1Rows;
    probe_logits_kernel<float><<<dim3(ntt, row_tiles), 256, 0, st>>>(k, q, t_len, d, rows, rows, rows, 1, inv_sqrt_d,
                                                                   row_tiles, ws.logits, ws.tile_max, offsets);
    probe_softmax_kernel<<<rows, 256, 0, st>>>(ws.logits, ws.tile_max, ntt, t_len, rows, rows, ws.denom, offsets);
    const size_t n = (size_t)rows * t_len;
    probe_normalize_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(ws.logits, ws.denom, rows, t_len, offsets);
    RDKV_CUDA_TRY(cudaMemcpyAsync(a, ws.logits, n * sizeof(double), cudaMemcpyDeviceToDevice, st));
    return launch_status();
}

extern "C" RDKV_API int rdkv_cuda_token_weights(const double* a, int32_t heads, int32_t rows, int32_t t_len,
                                                int32_t pool_kernel, float* raw_scratch, float* out, void* stream) {
    if (!a || !raw_scratch || !out || heads < 1 || rows < 0 || t_len < 1) return RDKV_EINVAL;
    if (pool_kernel < 1 || pool_kernel % 2 == 0) return RDKV_EINVAL;
    auto st = static_cast<cudaStream_t>(stream);
    column_sum_kernel<<<(t_len + 255) / 256, 256, 0, st>>>(a, heads, rows, t_len, raw_scratch);
    token_pool_kernel<<<(t_len + 255) / 256, 256, 0, st>>>(raw_scratch, 1, t_len, pool_kernel, out);
    return launch_status();
}

extern "C" RDKV_API int rdkv_cuda_moving_average(const float* raw, int32_t n, int32_t kernel, float* out,
                                                 void* stream) {
    if (!raw || !out || n < 0 || kernel < 1 || kernel % 2 == 0) return RDKV_EINVAL;
    if (n == 0) return RDKV_OK;
    token_pool_kernel<<<(n + 255) / 256, 256, 0, static_cast<cudaStream_t>(stream)>>>(raw, 1, n, kernel, out);
    return launch_status();
}

extern "C" RDKV_API int rdkv_cuda_channel_weights(const float* q, int32_t q_rows, const float* k, int32_t k_rows,
                                                  int32_t d, float* out, void* stream) {
    if (!q || !k || !out || q_rows < 0 || k_rows < 0 || d < 1) return RDKV_EINVAL;
    channel_norm_rows_kernel<float><<<(d + 127) / 128, 128, 0, static_cast<cudaStream_t>(stream)>>>(
        q, q_rows, k, k_rows, d, 1.0 / sqrt((double)d), out);
    return launch_status();
}
