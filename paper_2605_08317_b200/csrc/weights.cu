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

struct WeightsWorkspace {
    double* logits;
    double* tile_max;
    double* denom;
    float* rawf;
    size_t bytes;
};

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
    return carve(s, w, nullptr).bytes;
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
    WeightsWorkspace ws = carve(s, w, workspace);
    if (!workspace || workspace_bytes < ws.bytes) return RDKV_EINVAL;
    auto st = static_cast<cudaStream_t>(stream);
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
