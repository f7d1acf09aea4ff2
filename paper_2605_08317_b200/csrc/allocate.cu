// allocate.cu — K2: per-(unit) Lagrangian bisection (Stages 2 and 3).
//
// One CTA per unit runs, with all its threads cooperating on every
// per-unit argmin sweep:
//   head_budget   pipeline.cpp:60-72
//   allocate_v    pipeline.cpp:74-94   (target = min(16, B_V / (d T)))
//   force_window  pipeline.cpp:153-156
//   allocate_k    pipeline.cpp:96-112  (target = min(16, B_K / (kept d)))
//   mckp_bisect   allocator.cpp:135-216 (bracket doubling, bisection,
//                 strict-budget repair)
//   objectives / achieved bits          pipeline.cpp:169-181
//
// Bit-exactness: the per-unit cost w*eps(b) + lambda*b is evaluated with
// explicit round-to-nearest multiplies and add (__dmul_rn/__dadd_rn, and the
// file is built with -fmad=false), the strict '<' keeps the lower width on
// ties, the bit total is an exact integer reduction converted once to fp64
// (allocator.cpp:55-60), and the lambda sequence uses the same fp64
// expressions as the reference — so v_bits, k_bits, lambda and the
// convergence flags are identical given identical weights. The reported
// objectives are summed by one thread in the reference's order (a sequential
// fp64 sum, allocator.cpp:301-311), so they are bit-identical too.
#include <cooperative_groups.h>

#include "common.cuh"

namespace rdkv_b200 {

constexpr int kAllocThreads = 512;

struct AllocTable {
    int n;
    int widths[8];
    double eps[8];
};

__device__ __forceinline__ int argmin_bits(float w, const AllocTable& t, double lambda) {
    // argmin_entry, allocator.cpp:39-50
    const double wd = (double)w;
    int best_bits = t.widths[0];
    double best = __dadd_rn(__dmul_rn(wd, t.eps[0]), __dmul_rn(lambda, (double)best_bits));
    for (int i = 1; i < t.n; ++i) {
        const double cost = __dadd_rn(__dmul_rn(wd, t.eps[i]), __dmul_rn(lambda, (double)t.widths[i]));
        if (cost < best) {
            best = cost;
            best_bits = t.widths[i];
        }
    }
    return best_bits;
}

template <typename Tv>
__device__ Tv block_reduce_sum(Tv v, Tv* smem) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    __syncthreads();
    if (lane == 0) smem[wid] = v;
    __syncthreads();
    Tv tot = 0;
    const int nw = blockDim.x >> 5;
    for (int i = 0; i < nw; ++i) tot += smem[i];
    return tot;
}

__device__ float block_reduce_max_f(float v, float* smem) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    v = warp_max(v);
    __syncthreads();
    if (lane == 0) smem[wid] = v;
    __syncthreads();
    float m = smem[0];
    const int nw = blockDim.x >> 5;
    for (int i = 1; i < nw; ++i) m = fmaxf(m, smem[i]);
    return m;
}

struct Scratch {
    long long ll[32];
    double d[32];
    float f[32];
    int i[32];
};

// assign_all (allocator.cpp:52-61): average bits at lambda, block-wide.
__device__ double assign_avg(const float* w, int n, const AllocTable& t, double lambda, Scratch& s) {
    long long tot = 0;
    for (int u = threadIdx.x; u < n; u += blockDim.x) tot += argmin_bits(w[u], t, lambda);
    tot = block_reduce_sum<long long>(tot, s.ll);
    return (double)tot / (double)n;
}

struct BisectResult {
    double lambda, avg;
    int converged;
};

// mckp_bisect without the final bit materialisation (allocator.cpp:135-216).
__device__ BisectResult bisect(const float* w, int n, const AllocTable& t, double target,
                               double tol, int max_it, int strict, Scratch& s) {
    BisectResult r{0.0, 0.0, 1};
    const int max_width = t.widths[t.n - 1];
    if (target >= (double)max_width) {  // :153-161
        r.avg = max_width;
        r.lambda = 0.0;
        return r;
    }
    float wmax = 0.0f;
    for (int u = threadIdx.x; u < n; u += blockDim.x) wmax = fmaxf(wmax, w[u]);
    double lo = 0.0, hi = (double)block_reduce_max_f(wmax, s.f);
    const double floor_avg = t.widths[0];
    if (hi > 0.0) {  // :171-182
        double hi_avg = assign_avg(w, n, t, hi, s);
        int guard = 0;
        while (hi_avg > target && hi_avg > floor_avg && guard++ < 128) {
            hi = __dmul_rn(hi, 2.0);
            hi_avg = assign_avg(w, n, t, hi, s);
        }
    }
    double lambda = hi, avg = 0.0;
    int converged = 0;
    for (int it = 0; it < max_it; ++it) {  // :187-200
        lambda = __dmul_rn(0.5, __dadd_rn(lo, hi));
        avg = assign_avg(w, n, t, lambda, s);
        if (fabs(avg - target) / target < tol) {
            converged = 1;
            break;
        }
        if (avg > target) lo = lambda;
        else hi = lambda;
    }
    if (strict && avg > target) {  // :202-210 — hi_bits == assignment at lambda_hi
        lambda = hi;
        avg = assign_avg(w, n, t, lambda, s);
        converged = fabs(avg - target) / target < tol;
    }
    r.lambda = lambda;
    r.avg = avg;
    r.converged = converged;
    return r;
}

__device__ void materialize_bits(const float* w, int n, const AllocTable& t, double lambda,
                                 int all_max, uint8_t* bits) {
    const int max_width = t.widths[t.n - 1];
    for (int u = threadIdx.x; u < n; u += blockDim.x)
        bits[u] = (uint8_t)(all_max ? max_width : argmin_bits(w[u], t, lambda));
}

__device__ double eps_of(const AllocTable& t, int b) {
    for (int i = 0; i < t.n; ++i)
        if (t.widths[i] == b) return t.eps[i];
    return 0.0;
}

__device__ double sequential_objective(const float* w, const uint8_t* bits, int n, const AllocTable& t) {
    double obj = 0.0;
    for (int u = 0; u < n; ++u) obj = __dadd_rn(obj, __dmul_rn((double)w[u], eps_of(t, bits[u])));
    return obj;
}

__global__ void __launch_bounds__(kAllocThreads) allocate_kernel(
    const float* __restrict__ w_t, const float* __restrict__ w_c, int t_len, int d, int kv_heads,
    rdkv_config cfg, int window, uint8_t* __restrict__ v_bits_all, uint8_t* __restrict__ k_bits_all,
    rdkv_head_stats* __restrict__ stats) {
    __shared__ Scratch s;
    const int unit = blockIdx.x;
    const float* wv = w_t + (size_t)unit * t_len;
    const float* wk = w_c + (size_t)unit * d;
    uint8_t* vb = v_bits_all + (size_t)unit * t_len;
    uint8_t* kb = k_bits_all + (size_t)unit * d;
    AllocTable tv, tk;
    tv.n = tk.n = cfg.n_widths;
    for (int i = 0; i < 8; ++i) {
        tv.widths[i] = tk.widths[i] = cfg.widths[i];
        tv.eps[i] = cfg.eps_v[i];
        tk.eps[i] = cfg.eps_k[i];
    }

    // check_weights (allocator.cpp:143-149): finite and >= 0
    int bad = 0;
    for (int u = threadIdx.x; u < t_len; u += blockDim.x) bad |= !(isfinite(wv[u]) && wv[u] >= 0.0f);
    for (int u = threadIdx.x; u < d; u += blockDim.x) bad |= !(isfinite(wk[u]) && wk[u] >= 0.0f);
    bad = block_reduce_sum<int>(bad, s.i);

    // head_budget (pipeline.cpp:60-72)
    const double tokens_per_head = (double)cfg.n_tokens / (double)kv_heads;
    const double head_bits = __dmul_rn(__dmul_rn(__dmul_rn(2.0, tokens_per_head), (double)d), 16.0);
    const double kbud = __dmul_rn(cfg.r_k, head_bits);
    const double vbud = __dmul_rn(__dadd_rn(1.0, -cfg.r_k), head_bits);

    rdkv_head_stats out{};
    if (bad) {
        out.status = RDKV_EINVAL;
        if (threadIdx.x == 0) stats[unit] = out;
        return;
    }

    // Stage 2: V tokens (allocate_v)
    if (!(vbud > 0.0)) {
        for (int u = threadIdx.x; u < t_len; u += blockDim.x) vb[u] = 0;
        out.v_converged = 1;
    } else {
        double target = vbud / __dmul_rn((double)d, (double)t_len);
        if (target > 16.0) target = 16.0;
        BisectResult r = bisect(wv, t_len, tv, target, cfg.tolerance, cfg.max_iterations,
                                cfg.strict_budget, s);
        materialize_bits(wv, t_len, tv, r.lambda, target >= (double)tv.widths[tv.n - 1], vb);
        out.lambda_v = r.lambda;
        out.avg_v = r.avg;
        out.v_converged = r.converged;
    }
    __syncthreads();
    if (cfg.force_window_retain) {
        for (int i = threadIdx.x; i < window; i += blockDim.x) vb[t_len - window + i] = 16;
    }
    __syncthreads();
    long long kept = 0, v16 = 0, vsum = 0;
    for (int u = threadIdx.x; u < t_len; u += blockDim.x) {
        const int b = vb[u];
        kept += b > 0;
        v16 += b == 16;
        vsum += b;
    }
    kept = block_reduce_sum<long long>(kept, s.ll);
    v16 = block_reduce_sum<long long>(v16, s.ll);
    vsum = block_reduce_sum<long long>(vsum, s.ll);
    // allocation_objective (allocator.cpp:301-311) in the reference's sequential order
    if (threadIdx.x == 0) out.objective_v = sequential_objective(wv, vb, t_len, tv);

    // Stage 3: K channels over kept tokens (allocate_k)
    int k_len = d;
    long long ksum = 0;
    if (kept == 0) {
        k_len = 0;
        for (int u = threadIdx.x; u < d; u += blockDim.x) kb[u] = 0;
        out.k_converged = 1;
    } else if (!(kbud > 0.0)) {
        for (int u = threadIdx.x; u < d; u += blockDim.x) kb[u] = 0;
        out.k_converged = 1;
    } else {
        double target = kbud / __dmul_rn((double)kept, (double)d);
        if (target > 16.0) target = 16.0;
        BisectResult r = bisect(wk, d, tk, target, cfg.tolerance, cfg.max_iterations,
                                cfg.strict_budget, s);
        materialize_bits(wk, d, tk, r.lambda, target >= (double)tk.widths[tk.n - 1], kb);
        out.lambda_k = r.lambda;
        out.avg_k = r.avg;
        out.k_converged = r.converged;
    }
    __syncthreads();
    if (k_len > 0)
        for (int u = threadIdx.x; u < d; u += blockDim.x) ksum += kb[u];
    ksum = block_reduce_sum<long long>(ksum, s.ll);
    if (threadIdx.x == 0) out.objective_k = k_len > 0 ? sequential_objective(wk, kb, d, tk) : 0.0;
    out.n_kept = (int)kept;
    out.n_v16 = (int)v16;
    out.k_bits_len = k_len;
    out.achieved_bits = __dadd_rn(__dmul_rn((double)vsum, (double)d), __dmul_rn((double)ksum, (double)kept));
    out.status = RDKV_OK;
    if (threadIdx.x == 0) stats[unit] = out;
}

// ---------------------------------------------------------------------------
// Production path for long contexts: Stage 2 (the V-token bisection, the
// expensive sweep over T tokens) on a thread-block cluster of kClV CTAs per
// unit, each sweeping T / kClV tokens; the per-iterate bit totals are exact
// integers summed across the cluster through distributed shared memory, so
// every CTA takes the same lambda decision (bit-identical to the one-CTA
// sweep). Stage 3 and the sequential objectives follow in allocate_finish.
constexpr int kClV = 8;
constexpr int kClThreads = 1024;

struct ClScratch {
    long long part[2];  // this CTA's bit total of the current iterate (double-buffered by parity)
    float fpart[2];
    int ipart[2];
    long long warp_ll[32];
    float warp_f[32];
    long long bcast;  // cluster totals, broadcast to the CTA
    float ftot;
};

// Exact cluster-wide sum (long long) / max (float) / or (int): block reduce,
// publish in this CTA's parity slot, cluster barrier, warp 0 gathers the kClV
// slots over DSMEM. One cluster barrier per call: a slot is rewritten two calls
// later, after every CTA has passed the barrier of the call in between.
template <int OP>  // 0 sum ll, 1 max f, 2 or int
__device__ __forceinline__ void cl_reduce(ClScratch& s, int& parity, long long v, float f, int iv,
                                          long long& out_ll, float& out_f, int& out_i) {
    namespace cg = cooperative_groups;
    cg::cluster_group cl = cg::this_cluster();
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        if (OP == 0) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (OP == 1) f = fmaxf(f, __shfl_xor_sync(0xffffffffu, f, o));
        if (OP == 2) iv |= __shfl_xor_sync(0xffffffffu, iv, o);
    }
    if (lane == 0) {
        if (OP == 0) s.warp_ll[wid] = v;
        if (OP == 1) s.warp_f[wid] = f;
        if (OP == 2) s.warp_ll[wid] = iv;
    }
    __syncthreads();
    if (wid == 0) {
        const int nw = blockDim.x >> 5;
        long long a = 0;
        float m = 0.0f;
        for (int i = lane; i < nw; i += 32) {
            if (OP == 0 || OP == 2) a += s.warp_ll[i];
            if (OP == 1) m = fmaxf(m, s.warp_f[i]);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            a += __shfl_xor_sync(0xffffffffu, a, o);
            m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
        }
        if (lane == 0) {
            s.part[parity] = a;
            s.fpart[parity] = m;
        }
    }
    cl.sync();
    if (wid == 0) {
        long long a = 0;
        float m = 0.0f;
        if (lane < (int)cl.num_blocks()) {
            ClScratch* r = cl.map_shared_rank(&s, lane);
            a = r->part[parity];
            m = r->fpart[parity];
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            a += __shfl_xor_sync(0xffffffffu, a, o);
            m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
        }
        if (lane == 0) {
            s.bcast = a;
            s.ftot = m;
        }
    }
    __syncthreads();
    out_ll = s.bcast;
    out_f = s.ftot;
    out_i = (int)out_ll;
    parity ^= 1;
}

struct ClTable {
    int n;
    int widths[8];
    double eps[8];
};

// Bit total of this CTA's tokens at lambda (argmin_entry per token with the
// lambda * b terms hoisted: the same __dmul_rn values as argmin_bits).
__device__ __forceinline__ long long cl_local_total(const float* __restrict__ w, int u0, int u1, const ClTable& t,
                                                    const double (&lb)[8]) {
    long long tot = 0;
    for (int u = u0 + threadIdx.x; u < u1; u += blockDim.x) {
        const double wd = (double)__ldg(w + u);
        int best_bits = t.widths[0];
        double best = __dadd_rn(__dmul_rn(wd, t.eps[0]), lb[0]);
#pragma unroll
        for (int i = 1; i < 8; ++i) {
            if (i < t.n) {
                const double cost = __dadd_rn(__dmul_rn(wd, t.eps[i]), lb[i]);
                if (cost < best) {
                    best = cost;
                    best_bits = t.widths[i];
                }
            }
        }
        tot += best_bits;
    }
    return tot;
}

__global__ void __launch_bounds__(kClThreads, 1) allocate_v_cluster_kernel(const float* __restrict__ w_t, int t_len,
                                                                           int d, int kv_heads, rdkv_config cfg,
                                                                           int window, uint8_t* __restrict__ v_bits_all,
                                                                           rdkv_head_stats* __restrict__ stats) {
    namespace cg = cooperative_groups;
    cg::cluster_group cl = cg::this_cluster();
    __shared__ ClScratch s;
    const int rank = (int)cl.block_rank(), ncl = (int)cl.num_blocks();
    const int unit = blockIdx.x / ncl;
    const float* w = w_t + (size_t)unit * t_len;
    uint8_t* vb = v_bits_all + (size_t)unit * t_len;
    const int u0 = (int)((long long)t_len * rank / ncl), u1 = (int)((long long)t_len * (rank + 1) / ncl);
    ClTable t;
    t.n = cfg.n_widths;
    for (int i = 0; i < 8; ++i) {
        t.widths[i] = cfg.widths[i];
        t.eps[i] = cfg.eps_v[i];
    }
    int parity = 0;
    long long ll;
    float fm;
    int iv;
    // check_weights (allocator.cpp:143-149) over the V weights; the K weights are
    // checked by allocate_finish
    int bad = 0;
    float wmax = 0.0f;
    for (int u = u0 + threadIdx.x; u < u1; u += blockDim.x) {
        const float x = w[u];
        bad |= !(isfinite(x) && x >= 0.0f);
        wmax = fmaxf(wmax, x);
    }
    cl_reduce<2>(s, parity, 0, 0.0f, bad, ll, fm, iv);
    bad = iv;
    const double tokens_per_head = (double)cfg.n_tokens / (double)kv_heads;
    const double head_bits = __dmul_rn(__dmul_rn(__dmul_rn(2.0, tokens_per_head), (double)d), 16.0);
    const double vbud = __dmul_rn(__dadd_rn(1.0, -cfg.r_k), head_bits);
    rdkv_head_stats out{};
    if (bad) {
        out.status = RDKV_EINVAL;
        if (rank == 0 && threadIdx.x == 0) stats[unit] = out;
        return;
    }
    double lambda = 0.0, avg = 0.0;
    int converged = 1, all_max = 0;
    const int max_width = t.widths[t.n - 1];
    if (!(vbud > 0.0)) {
        for (int u = u0 + threadIdx.x; u < u1; u += blockDim.x) vb[u] = 0;
    } else {
        double target = vbud / __dmul_rn((double)d, (double)t_len);
        if (target > 16.0) target = 16.0;
        const double n = (double)t_len;
        auto avg_at = [&](double lam) {
            double lb[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) lb[i] = __dmul_rn(lam, (double)t.widths[i]);
            cl_reduce<0>(s, parity, cl_local_total(w, u0, u1, t, lb), 0.0f, 0, ll, fm, iv);
            return (double)ll / n;
        };
        if (target >= (double)max_width) {  // allocator.cpp:153-161
            avg = max_width;
            all_max = 1;
        } else {
            cl_reduce<1>(s, parity, 0, wmax, 0, ll, fm, iv);
            double lo = 0.0, hi = (double)fm;
            const double floor_avg = t.widths[0];
            if (hi > 0.0) {  // :171-182
                double hi_avg = avg_at(hi);
                int guard = 0;
                while (hi_avg > target && hi_avg > floor_avg && guard++ < 128) {
                    hi = __dmul_rn(hi, 2.0);
                    hi_avg = avg_at(hi);
                }
            }
            lambda = hi;
            converged = 0;
            for (int it = 0; it < cfg.max_iterations; ++it) {  // :187-200
                lambda = __dmul_rn(0.5, __dadd_rn(lo, hi));
                avg = avg_at(lambda);
                if (fabs(avg - target) / target < cfg.tolerance) {
                    converged = 1;
                    break;
                }
                if (avg > target) lo = lambda;
                else hi = lambda;
            }
            if (cfg.strict_budget && avg > target) {  // :202-210
                lambda = hi;
                avg = avg_at(lambda);
                converged = fabs(avg - target) / target < cfg.tolerance;
            }
        }
        double lb[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) lb[i] = __dmul_rn(lambda, (double)t.widths[i]);
        for (int u = u0 + threadIdx.x; u < u1; u += blockDim.x) {
            int b = max_width;
            if (!all_max) {
                const double wd = (double)w[u];
                b = t.widths[0];
                double best = __dadd_rn(__dmul_rn(wd, t.eps[0]), lb[0]);
                for (int i = 1; i < t.n; ++i) {
                    const double cost = __dadd_rn(__dmul_rn(wd, t.eps[i]), lb[i]);
                    if (cost < best) {
                        best = cost;
                        b = t.widths[i];
                    }
                }
            }
            vb[u] = (uint8_t)b;
        }
    }
    // force-window override (pipeline.cpp:153-156), after every thread's
    // materialising stores to the same bytes
    __syncthreads();
    if (cfg.force_window_retain)
        for (int u = max(u0, t_len - window) + threadIdx.x; u < u1; u += blockDim.x) vb[u] = 16;
    if (rank == 0 && threadIdx.x == 0) {
        out.lambda_v = lambda;
        out.avg_v = avg;
        out.v_converged = converged;
        out.status = -1;  // Stage 2 done; allocate_finish completes the record
        stats[unit] = out;
    }
}

// Sequential fp64 objective sum_u w_u * eps(b_u) in the reference's order
// (allocator.cpp:301-311): warps 1.. form the products of the next chunk in
// shared memory while thread 0 adds the current chunk in order, so the long
// dependent chain runs at the DADD latency (no load latency on it).
constexpr int kObjChunk = 2048;
__device__ double block_sequential_objective(const float* __restrict__ w, const uint8_t* __restrict__ bits, int n,
                                             const AllocTable& t, double* buf) {
    double obj = 0.0;
    const int nch = (n + kObjChunk - 1) / kObjChunk;
    auto fill = [&](int c, double* dst, int t0, int step) {
        const int base = c * kObjChunk, cnt = min(kObjChunk, n - base);
        for (int i = t0; i < cnt; i += step) dst[i] = __dmul_rn((double)w[base + i], eps_of(t, bits[base + i]));
    };
    fill(0, buf, threadIdx.x, blockDim.x);
    __syncthreads();
    for (int c = 0; c < nch; ++c) {
        const double* cur = buf + (c & 1) * kObjChunk;
        if (threadIdx.x == 0) {
            const int cnt = min(kObjChunk, n - c * kObjChunk);
            int i = 0;
            for (; i + 16 <= cnt; i += 16) {
                double x[16];
#pragma unroll
                for (int j = 0; j < 16; ++j) x[j] = cur[i + j];
#pragma unroll
                for (int j = 0; j < 16; ++j) obj = __dadd_rn(obj, x[j]);
            }
            for (; i < cnt; ++i) obj = __dadd_rn(obj, cur[i]);
        } else if (threadIdx.x >= 32 && c + 1 < nch) {
            fill(c + 1, buf + ((c + 1) & 1) * kObjChunk, threadIdx.x - 32, blockDim.x - 32);
        }
        __syncthreads();
    }
    return obj;
}

// Stages 2 (tail) and 3 after allocate_v_cluster: counts, objectives, allocate_k.
__global__ void __launch_bounds__(kAllocThreads) allocate_finish_kernel(
    const float* __restrict__ w_t, const float* __restrict__ w_c, int t_len, int d, int kv_heads, rdkv_config cfg,
    const uint8_t* __restrict__ v_bits_all, uint8_t* __restrict__ k_bits_all, rdkv_head_stats* __restrict__ stats) {
    __shared__ Scratch s;
    __shared__ double obj_v;
    const int unit = blockIdx.x;
    rdkv_head_stats out = stats[unit];
    if (out.status != -1) return;  // invalid V weights: already reported
    const float* wv = w_t + (size_t)unit * t_len;
    const float* wk = w_c + (size_t)unit * d;
    const uint8_t* vb = v_bits_all + (size_t)unit * t_len;
    uint8_t* kb = k_bits_all + (size_t)unit * d;
    AllocTable tv, tk;
    tv.n = tk.n = cfg.n_widths;
    for (int i = 0; i < 8; ++i) {
        tv.widths[i] = tk.widths[i] = cfg.widths[i];
        tv.eps[i] = cfg.eps_v[i];
        tk.eps[i] = cfg.eps_k[i];
    }
    int bad = 0;
    for (int u = threadIdx.x; u < d; u += blockDim.x) bad |= !(isfinite(wk[u]) && wk[u] >= 0.0f);
    bad = block_reduce_sum<int>(bad, s.i);
    if (bad) {
        rdkv_head_stats e{};
        e.status = RDKV_EINVAL;
        __syncthreads();
        if (threadIdx.x == 0) stats[unit] = e;
        return;
    }
    const double tokens_per_head = (double)cfg.n_tokens / (double)kv_heads;
    const double head_bits = __dmul_rn(__dmul_rn(__dmul_rn(2.0, tokens_per_head), (double)d), 16.0);
    const double kbud = __dmul_rn(cfg.r_k, head_bits);
    long long kept = 0, v16 = 0, vsum = 0;
    for (int u = threadIdx.x; u < t_len; u += blockDim.x) {
        const int b = vb[u];
        kept += b > 0;
        v16 += b == 16;
        vsum += b;
    }
    kept = block_reduce_sum<long long>(kept, s.ll);
    v16 = block_reduce_sum<long long>(v16, s.ll);
    vsum = block_reduce_sum<long long>(vsum, s.ll);
    {
        __shared__ double objbuf[2 * kObjChunk];
        const double o = block_sequential_objective(wv, vb, t_len, tv, objbuf);
        if (threadIdx.x == 0) obj_v = o;
    }
    int k_len = d;
    long long ksum = 0;
    if (kept == 0) {
        k_len = 0;
        for (int u = threadIdx.x; u < d; u += blockDim.x) kb[u] = 0;
        out.k_converged = 1;
    } else if (!(kbud > 0.0)) {
        for (int u = threadIdx.x; u < d; u += blockDim.x) kb[u] = 0;
        out.k_converged = 1;
    } else {
        double target = kbud / __dmul_rn((double)kept, (double)d);
        if (target > 16.0) target = 16.0;
        BisectResult r = bisect(wk, d, tk, target, cfg.tolerance, cfg.max_iterations, cfg.strict_budget, s);
        materialize_bits(wk, d, tk, r.lambda, target >= (double)tk.widths[tk.n - 1], kb);
        out.lambda_k = r.lambda;
        out.avg_k = r.avg;
        out.k_converged = r.converged;
    }
    __syncthreads();
    if (k_len > 0)
        for (int u = threadIdx.x; u < d; u += blockDim.x) ksum += kb[u];
    ksum = block_reduce_sum<long long>(ksum, s.ll);
    if (threadIdx.x == 0) {
        out.objective_v = obj_v;
        out.objective_k = k_len > 0 ? sequential_objective(wk, kb, d, tk) : 0.0;
        out.n_kept = (int)kept;
        out.n_v16 = (int)v16;
        out.k_bits_len = k_len;
        out.achieved_bits = __dadd_rn(__dmul_rn((double)vsum, (double)d), __dmul_rn((double)ksum, (double)kept));
        out.status = RDKV_OK;
        stats[unit] = out;
    }
}

}  // namespace rdkv_b200

using namespace rdkv_b200;

// BudgetSpec::validate (pipeline.cpp:52-58), BitSet::validate (quantizer.cpp:66-88),
// SolverConfig::validate (allocator.cpp:413-416), ProbeConfig::validate (cache.cpp:107-112).
extern "C" int rdkv_validate_config(const rdkv_config* c) {
    if (!c) return RDKV_EINVAL;
    if (c->n_tokens < 1) return RDKV_EINVAL;
    if (!(c->r_k > 0.0) || !(c->r_k < 1.0)) return RDKV_EINVAL;
    if (c->n_widths < 1 || c->n_widths > 8) return RDKV_EINVAL;
    bool has0 = false, has16 = false;
    for (int i = 0; i < c->n_widths; ++i) {
        const int b = c->widths[i];
        if (b < 0 || b > 16 || b % 2) return RDKV_EINVAL;
        if (i > 0 && b <= c->widths[i - 1]) return RDKV_EINVAL;
        if (b != 0 && b != 2 && b != 4 && b != 8 && b != 16) return RDKV_EINVAL;
        has0 |= b == 0;
        has16 |= b == 16;
    }
    if (!has0 || !has16) return RDKV_EINVAL;
    if (c->window < 1 || c->pool_kernel < 1 || c->pool_kernel % 2 == 0) return RDKV_EINVAL;
    if (!(c->tolerance > 0.0) || c->max_iterations < 1) return RDKV_EINVAL;
    return RDKV_OK;
}

extern "C" RDKV_API int rdkv_cuda_allocate(const float* w_t, const float* w_c, const rdkv_shape* s,
                                           const rdkv_config* cfg, uint8_t* v_bits, uint8_t* k_bits,
                                           rdkv_head_stats* stats, void* stream) {
    if (!s || !w_t || !w_c || !v_bits || !k_bits || !stats) return RDKV_EINVAL;
    if (s->units < 1 || s->seq_len < 1 || s->head_dim < 1 || s->kv_heads < 1) return RDKV_EINVAL;
    if (int st = rdkv_validate_config(cfg)) return st;
    const int window = cfg->window < s->probe_rows ? cfg->window : s->probe_rows;
    if (cfg->force_window_retain && window > s->seq_len) return RDKV_EINVAL;
    auto st = static_cast<cudaStream_t>(stream);
    if (s->seq_len >= kClV * kClThreads) {  // long contexts: the cluster sweep (bit-identical)
        cudaLaunchConfig_t lc{};
        lc.gridDim = dim3(s->units * kClV);
        lc.blockDim = dim3(kClThreads);
        lc.stream = st;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = kClV;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        lc.attrs = at;
        lc.numAttrs = 1;
        RDKV_CUDA_TRY(cudaLaunchKernelEx(&lc, allocate_v_cluster_kernel, w_t, s->seq_len, s->head_dim, s->kv_heads,
                                         *cfg, window, v_bits, stats));
        allocate_finish_kernel<<<s->units, kAllocThreads, 0, st>>>(w_t, w_c, s->seq_len, s->head_dim, s->kv_heads,
                                                                   *cfg, v_bits, k_bits, stats);
        return launch_status();
    }
    allocate_kernel<<<s->units, kAllocThreads, 0, static_cast<cudaStream_t>(stream)>>>(
        w_t, w_c, s->seq_len, s->head_dim, s->kv_heads, *cfg, window, v_bits, k_bits, stats);
    return launch_status();
}

// ---------------------------------------------------------------------------
// Stand-alone mckp_bisect (allocator.cpp:135-216) over `instances`
// independent weight vectors of length n, one CTA each.
__global__ void __launch_bounds__(kAllocThreads) mckp_kernel(const float* __restrict__ w_all, int n,
                                                            AllocTable t, double target, double tol, int max_it,
                                                            int strict, uint8_t* __restrict__ bits_all,
                                                            rdkv_bisect_result* __restrict__ res) {
    __shared__ Scratch s;
    const float* w = w_all + (size_t)blockIdx.x * n;
    uint8_t* bits = bits_all + (size_t)blockIdx.x * n;
    int bad = 0;
    for (int u = threadIdx.x; u < n; u += blockDim.x) bad |= !(isfinite(w[u]) && w[u] >= 0.0f);
    bad = block_reduce_sum<int>(bad, s.i);
    rdkv_bisect_result out{};
    if (bad) {  // check_weights (allocator.cpp:63-69)
        out.status = RDKV_EINVAL;
        if (threadIdx.x == 0) res[blockIdx.x] = out;
        return;
    }
    const int all_max = target >= (double)t.widths[t.n - 1];
    BisectResult r = bisect(w, n, t, target, tol, max_it, strict, s);
    materialize_bits(w, n, t, r.lambda, all_max, bits);
    __syncthreads();
    out.lambda = r.lambda;
    out.achieved_avg_bits = r.avg;
    if (threadIdx.x == 0) out.objective = sequential_objective(w, bits, n, t);
    out.converged = r.converged;
    out.status = RDKV_OK;
    if (threadIdx.x == 0) res[blockIdx.x] = out;
}

extern "C" RDKV_API int rdkv_cuda_mckp_bisect(const float* weights, int32_t instances, int32_t n,
                                              const int32_t* widths, const double* eps, int32_t n_widths,
                                              double target_avg_bits, double tolerance, int32_t max_iterations,
                                              int32_t strict_budget, uint8_t* bits, rdkv_bisect_result* results,
                                              void* stream) {
    if (!widths || !eps || n_widths < 1 || n_widths > 8) return RDKV_EINVAL;
    AllocTable t{};
    t.n = n_widths;
    for (int i = 0; i < n_widths; ++i) {  // BitSet::validate_relaxed (quantizer.cpp:66-80)
        const int b = widths[i];
        if (b < 0 || b > 16 || b % 2 || (i > 0 && b <= widths[i - 1])) return RDKV_EINVAL;
        if (b != 0 && b != 2 && b != 4 && b != 8 && b != 16) return RDKV_EINVAL;
        if (!(eps[i] >= 0.0) || !isfinite(eps[i])) return RDKV_EINVAL;
        t.widths[i] = b;
        t.eps[i] = eps[i];
    }
    if (!(tolerance > 0.0) || max_iterations < 1) return RDKV_EINVAL;      // SolverConfig::validate
    if (!(target_avg_bits > 0.0) || target_avg_bits > 16.0) return RDKV_EINVAL;  // allocator.cpp:140-142
    if (instances < 0 || n < 0 || (instances > 0 && n > 0 && (!weights || !bits || !results)))
        return RDKV_EINVAL;
    if (instances == 0 || n == 0) return RDKV_OK;
    mckp_kernel<<<instances, kAllocThreads, 0, static_cast<cudaStream_t>(stream)>>>(
        weights, n, t, target_avg_bits, tolerance, max_iterations, strict_budget, bits, results);
    return launch_status();
}
