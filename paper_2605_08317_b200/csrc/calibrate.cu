// calibrate.cu — ε-table calibration on the device (calibrate_epsilon, quantizer.cpp:200-284).
//
// The reference walks every (cache, layer, KV head) job, and inside it every unit — a V row
// (token granularity) or a K column (channel granularity) — quantizes it at each finite width,
// dequantizes, and adds the unit's NMSE to the job's running sum; jobs merge in job order.
// Here one thread owns a unit (channel units: a (unit, width) pair) (fp64, the reference's element order, compiled
// with -fmad=false so every multiply-add rounds like the reference's non-FMA x86 build), a
// second kernel sums the per-unit NMSEs of each job in unit order, and the host merges jobs in
// order — so the table is bit-identical to the reference's. Channel units are read with
// consecutive threads on consecutive channels of a row (coalesced); token units are 512-B
// rows walked by one thread (served from L1 after the first touch).
#include <cmath>

#include "common.cuh"

namespace rdkv_b200 {
namespace {

struct QWidths {
    int w[8];
    int n;
};

__device__ __forceinline__ void calib_params(float lo, float hi, int bits, double& scale, double& zd) {
    const double max_code = (double)((1 << bits) - 1);
    double range = __dsub_rn((double)hi, (double)lo);
    if (range < 1e-12) range = 1e-12;  // kMinRange
    scale = __ddiv_rn(range, max_code);
    zd = round(__ddiv_rn(-(double)lo, scale));
    zd = fmin(fmax(zd, -9.0e18), 9.0e18);
}

template <typename T>
__device__ __forceinline__ float ld(const T* p) {
    if constexpr (sizeof(T) == 2) {
        return __half2float(*p);
    } else {
        return *p;
    }
}

// nmse [unit][qw.n] for every unit of every job; NaN marks a zero-energy unit (skipped).
// Channel units (few and long) run one thread per (unit, width) — the energy / range pass is
// repeated per width — for qw.n× the parallelism; token units (many and short) run one
// thread per unit over all widths.
template <typename T>
__global__ void __launch_bounds__(256) calib_unit_kernel(const T* __restrict__ values, int jobs, int t_len, int d,
                                                         int channel, QWidths qw, double* __restrict__ nmse,
                                                         int* __restrict__ bad) {
    const long long per_job = channel ? d : t_len;
    const long long n_units = (long long)jobs * per_job;
    const long long gid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const int split = channel ? qw.n : 1;
    if (gid >= n_units * split) return;
    // width-major thread order keeps consecutive threads on consecutive units (coalesced K rows)
    const int b0 = channel ? (int)(gid / n_units) : 0, b1 = channel ? b0 + 1 : qw.n;
    const long long g = gid % n_units;
    const long long job = g / per_job, i = g % per_job;
    const T* base;
    long long stride;
    int len;
    if (channel) {
        base = values + job * (long long)t_len * d + i;
        stride = d;
        len = t_len;
    } else {
        base = values + (job * (long long)t_len + i) * d;
        stride = 1;
        len = d;
    }
    double energy = 0.0;
    float lo = ld(base), hi = lo;
    bool finite = true;
    for (int j = 0; j < len; ++j) {
        const float x = ld(base + j * stride);
        energy = __dadd_rn(energy, __dmul_rn((double)x, (double)x));
        finite &= isfinite(x);
        lo = x < lo ? x : lo;  // std::min / std::max argument order
        hi = hi < x ? x : hi;
    }
    double* out = nmse + g * qw.n;
    if (energy == 0.0) {  // account_unit: NMSE undefined, the unit carries no weight
        for (int b = b0; b < b1; ++b) out[b] = __longlong_as_double(0x7ff8000000000000ll);
        return;
    }
    if (!finite) {  // quantize_unit: NumericError
        atomicOr(bad, 1);
        return;
    }
    for (int b = b0; b < b1; ++b) {
        const int bits = qw.w[b];
        const double max_code = (double)((1 << bits) - 1);
        double scale, zd;
        calib_params(lo, hi, bits, scale, zd);
        const double sf = (double)(float)scale;  // stored params.scale
        const double zp = (double)(long long)zd;  // stored params.zero_point
        double err = 0.0;
        for (int j = 0; j < len; ++j) {
            const float x = ld(base + j * stride);
            double c = __dadd_rn(round(__ddiv_rn((double)x, scale)), zd);
            c = fmin(fmax(c, 0.0), max_code);
            const double code = (double)(uint32_t)c;
            const float rec = (float)__dmul_rn(sf, __dsub_rn(code, zp));  // dequantize_unit
            const double e = __dsub_rn((double)rec, (double)x);
            err = __dadd_rn(err, __dmul_rn(e, e));
        }
        out[b] = __ddiv_rn(err, energy);
    }
}

// err_sum [job][qw.n] = Σ_units nmse in unit order; count [job] = non-skipped units.
__global__ void calib_job_kernel(const double* __restrict__ nmse, int jobs, long long per_job, int nq,
                                 double* __restrict__ err_sum, int64_t* __restrict__ count) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= jobs * nq) return;
    const int job = t / nq, b = t % nq;
    const double* p = nmse + (long long)job * per_job * nq + b;
    double s = 0.0;
    long long n = 0;
    for (long long i = 0; i < per_job; ++i) {
        const double x = p[i * nq];
        if (!isnan(x)) {
            s = __dadd_rn(s, x);
            ++n;
        }
    }
    err_sum[t] = s;
    if (b == 0) count[job] = n;
}

// BitSet::validate_relaxed (quantizer.cpp:66-81) + the finite widths of the set.
bool quant_widths(const int32_t* widths, int n, QWidths* qw) {
    if (!widths || n < 1 || n > 8) return false;
    qw->n = 0;
    for (int i = 0; i < n; ++i) {
        const int b = widths[i];
        if (b < 0 || b > 16 || b % 2 != 0) return false;
        if (i > 0 && b <= widths[i - 1]) return false;
        if (b != 0 && b != 16 && b != 2 && b != 4 && b != 8) return false;
        if (b == 2 || b == 4 || b == 8) qw->w[qw->n++] = b;
    }
    return true;
}

}  // namespace
}  // namespace rdkv_b200

using namespace rdkv_b200;

extern "C" RDKV_API size_t rdkv_cuda_calibrate_workspace(int32_t jobs, int32_t seq_len, int32_t head_dim,
                                                         int32_t granularity, int32_t n_widths) {
    if (jobs < 0 || seq_len < 1 || head_dim < 1 || n_widths < 1) return 0;
    const size_t per_job = granularity ? (size_t)head_dim : (size_t)seq_len;
    return 256 + (size_t)jobs * per_job * (size_t)n_widths * sizeof(double);
}

extern "C" RDKV_API int rdkv_cuda_calibrate_partials(const void* values, int32_t dtype, int32_t jobs,
                                                     int32_t seq_len, int32_t head_dim, int32_t granularity,
                                                     const int32_t* widths, int32_t n_widths, double* err_sum,
                                                     int64_t* count, void* workspace, size_t workspace_bytes,
                                                     void* stream) {
    QWidths qw;
    if (!quant_widths(widths, n_widths, &qw)) return RDKV_EINVAL;
    if (granularity != 0 && granularity != 1) return RDKV_EINVAL;
    if (dtype != RDKV_F32 && dtype != RDKV_F16) return RDKV_EINVAL;
    if (jobs < 0 || seq_len < 1 || head_dim < 1 || !err_sum || !count) return RDKV_EINVAL;
    if (jobs == 0) return RDKV_OK;
    if (!values || !workspace) return RDKV_EINVAL;
    const int nq = qw.n > 0 ? qw.n : 1;
    if (qw.n == 0) qw = QWidths{{2}, 1};  // no finite widths: count units only (sums discarded)
    if (workspace_bytes < rdkv_cuda_calibrate_workspace(jobs, seq_len, head_dim, granularity, nq))
        return RDKV_EINVAL;
    auto st = static_cast<cudaStream_t>(stream);
    int* bad = static_cast<int*>(workspace);
    double* nmse = reinterpret_cast<double*>(static_cast<char*>(workspace) + 256);
    RDKV_CUDA_TRY(cudaMemsetAsync(bad, 0, sizeof(int), st));
    const long long per_job = granularity ? head_dim : seq_len;
    const long long n_units = (long long)jobs * per_job;
    const unsigned blocks = (unsigned)((n_units * (granularity ? qw.n : 1) + 255) / 256);
    if (dtype == RDKV_F16)
        calib_unit_kernel<__half><<<blocks, 256, 0, st>>>(static_cast<const __half*>(values), jobs, seq_len,
                                                          head_dim, granularity, qw, nmse, bad);
    else
        calib_unit_kernel<float><<<blocks, 256, 0, st>>>(static_cast<const float*>(values), jobs, seq_len,
                                                         head_dim, granularity, qw, nmse, bad);
    RDKV_CUDA_TRY(cudaGetLastError());
    // err_sum is [jobs][nq] over the finite widths (ascending)
    calib_job_kernel<<<(jobs * nq + 127) / 128, 128, 0, st>>>(nmse, jobs, per_job, nq, err_sum, count);
    RDKV_CUDA_TRY(cudaGetLastError());
    int bad_h = 0;
    RDKV_CUDA_TRY(cudaMemcpyAsync(&bad_h, bad, sizeof(int), cudaMemcpyDeviceToHost, st));
    RDKV_CUDA_TRY(cudaStreamSynchronize(st));
    return bad_h ? RDKV_ENUMERIC : RDKV_OK;
}

extern "C" RDKV_API int rdkv_calibrate_finalize(const double* err_sum, const int64_t* count, int32_t jobs,
                                                const int32_t* widths, int32_t n_widths, double* eps,
                                                int64_t* unit_count) {
    QWidths qw;
    if (!quant_widths(widths, n_widths, &qw) || !eps || jobs < 0) return RDKV_EINVAL;
    if (jobs == 0) return RDKV_EINVAL;  // "calibrate_epsilon: empty sample"
    if (!err_sum || !count) return RDKV_EINVAL;
    const int nq = qw.n > 0 ? qw.n : 1;
    double sums[8] = {0};
    long long units = 0;
    for (int j = 0; j < jobs; ++j) {  // partials merge in job order (quantizer.cpp:249-253)
        for (int b = 0; b < qw.n; ++b) sums[b] += err_sum[(size_t)j * nq + b];
        units += count[j];
    }
    if (unit_count) *unit_count = units;
    if (units == 0) return RDKV_ENUMERIC;  // all units have zero norm
    int q = 0;
    for (int i = 0; i < n_widths; ++i) {
        const int b = widths[i];
        if (b == 0) eps[i] = 1.0;
        else if (b == 16) eps[i] = 0.0;
        else eps[i] = sums[q++] / (double)units;
    }
    // DistortionTable::validate (quantizer.cpp:178-197)
    for (int i = 0; i < n_widths; ++i) {
        if (!std::isfinite(eps[i]) || eps[i] < 0.0) return RDKV_EINVAL;
        if (i > 0 && eps[i] >= eps[i - 1]) return RDKV_EINVAL;
    }
    return RDKV_OK;
}
