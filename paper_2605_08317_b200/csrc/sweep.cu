// sweep.cu — Lagrangian dual bound per weight vector (dual_bound, allocator.cpp:218-246), the
// device half of run_sweep (sweep.cpp:40-114): after rdkv_cuda_mckp_bisect has solved every
// (layer, KV head) instance at a grid point, this evaluates g(λ) at each instance's final λ
// without a host round trip. One warp per instance: lanes evaluate the per-unit argmin in
// parallel, lane 0 folds the 32 terms of every round into the running sums in unit order, so
// the fp64 sums are bit-identical to the reference's serial loop (built with -fmad=false).
#include <cmath>

#include "common.cuh"

namespace rdkv_b200 {
namespace {

struct Table {
    int w[8];
    double e[8];
    int n;
};

__global__ void __launch_bounds__(256) dual_bound_kernel(const float* __restrict__ weights, int instances, int n,
                                                         Table t, const rdkv_bisect_result* __restrict__ solved,
                                                         double total_budget,
                                                         rdkv_dual_bound_result* __restrict__ out) {
    const int inst = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
    const int lane = threadIdx.x & 31;
    if (inst >= instances) return;
    const double lambda = solved[inst].lambda;
    const float* w = weights + (size_t)inst * n;
    bool bad = !(lambda >= 0.0) || !isfinite(lambda);
    double min_sum = 0.0, primal = 0.0, bits_used = 0.0;
    for (int base = 0; base < n; base += 32) {
        const int u = base + lane;
        double term = 0.0, we = 0.0;
        int b = 0;
        if (u < n) {
            const float wf = w[u];
            if (!isfinite(wf) || wf < 0.0f) bad = true;  // check_weights
            const double wd = (double)wf;
            // argmin_entry (allocator.cpp:39-50): strict < keeps the lower width on ties
            int best = t.w[0];
            double best_cost = __dadd_rn(__dmul_rn(wd, t.e[0]), __dmul_rn(lambda, (double)t.w[0]));
            for (int i = 1; i < t.n; ++i) {
                const double c = __dadd_rn(__dmul_rn(wd, t.e[i]), __dmul_rn(lambda, (double)t.w[i]));
                if (c < best_cost) {
                    best_cost = c;
                    best = t.w[i];
                }
            }
            double e = 0.0;
            for (int i = 0; i < t.n; ++i)
                if (t.w[i] == best) {
                    e = t.e[i];
                    break;
                }
            we = __dmul_rn(wd, e);
            term = __dadd_rn(we, __dmul_rn(lambda, (double)best));
            b = best;
        }
        const int cnt = n - base < 32 ? n - base : 32;
        for (int j = 0; j < cnt; ++j) {  // unit order
            const double tj = __shfl_sync(0xffffffffu, term, j);
            const double wj = __shfl_sync(0xffffffffu, we, j);
            const int bj = __shfl_sync(0xffffffffu, b, j);
            min_sum = __dadd_rn(min_sum, tj);
            primal = __dadd_rn(primal, wj);
            bits_used = __dadd_rn(bits_used, (double)bj);
        }
    }
    bad = __any_sync(0xffffffffu, bad);
    if (lane == 0) {
        rdkv_dual_bound_result r;
        r.g_lambda = __dsub_rn(min_sum, __dmul_rn(lambda, total_budget));
        r.primal = primal;
        r.gap = __dsub_rn(r.primal, r.g_lambda);
        r.feasible = bits_used <= __dadd_rn(total_budget, 1e-9);
        r.status = bad ? RDKV_EINVAL : RDKV_OK;
        out[inst] = r;
    }
}

}  // namespace
}  // namespace rdkv_b200

using namespace rdkv_b200;

extern "C" RDKV_API int rdkv_cuda_dual_bound(const float* weights, int32_t instances, int32_t n,
                                             const int32_t* widths, const double* eps, int32_t n_widths,
                                             const rdkv_bisect_result* solved, double total_budget,
                                             rdkv_dual_bound_result* out, void* stream) {
    if (!widths || !eps || n_widths < 1 || n_widths > 8) return RDKV_EINVAL;
    Table t;
    t.n = n_widths;
    for (int i = 0; i < n_widths; ++i) {  // make_argmin_table -> BitSet::validate_relaxed
        const int b = widths[i];
        if (b < 0 || b > 16 || b % 2 || (i > 0 && b <= widths[i - 1])) return RDKV_EINVAL;
        if (b != 0 && b != 2 && b != 4 && b != 8 && b != 16) return RDKV_EINVAL;
        t.w[i] = b;
        t.e[i] = eps[i];
    }
    if (instances < 0 || n < 0) return RDKV_EINVAL;
    if (instances == 0) return RDKV_OK;
    if (!solved || !out || (n > 0 && !weights)) return RDKV_EINVAL;
    const int per_block = 8;
    dual_bound_kernel<<<(instances + per_block - 1) / per_block, per_block * 32, 0,
                        static_cast<cudaStream_t>(stream)>>>(weights, instances, n, t, solved, total_budget, out);
    return launch_status();
}
