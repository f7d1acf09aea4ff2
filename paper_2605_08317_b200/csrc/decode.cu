// decode.cu — K4 dispatch: chooses the tensor-core kernel (decode_mma.cu) for
// the layouts it covers and the generic CUDA-core kernel otherwise; split-K
// workspace; host-buffer (end-to-end) entry point.
#include "common.cuh"

#include <cstring>

namespace rdkv_b200 {
template <typename IO>
int launch_generic(const rdkv_decode_args* a, int split, int max_kslots, cudaStream_t st);
int launch_mma(const rdkv_decode_args* a, cudaStream_t st);  // decode_mma.cu
bool mma_supported(const rdkv_decode_args* a);
int launch_partial(const rdkv_decode_args* a, int rank, int world, float* partial, cudaStream_t st);
int launch_merge(const float* part, int nparts, int rows, int d, void* out, int io, cudaStream_t st);
}  // namespace rdkv_b200

using namespace rdkv_b200;

extern "C" RDKV_API size_t rdkv_cuda_decode_workspace(int32_t units, int32_t group, int32_t head_dim,
                                                      int32_t split) {
    if (units < 1 || group < 1 || head_dim < 1 || split <= 1) return 0;
    return sizeof(float) * (size_t)units * split * group * (2 + (size_t)head_dim);
}

extern "C" RDKV_API int rdkv_cuda_decode(const rdkv_decode_args* a, void* stream) {
    if (!a || !a->arena || !a->tile_offsets || !a->q || !a->out) return RDKV_EINVAL;
    if (a->units < 1 || a->group < 1 || a->group > 16 || a->head_dim < 1 || a->head_dim > 256)
        return RDKV_EINVAL;
    if (a->io_dtype != RDKV_F32 && a->io_dtype != RDKV_F16) return RDKV_EINVAL;
    if (a->zc_len && (!a->zc_k || !a->zc_v || a->zc_cap < 1)) return RDKV_EINVAL;
    // the Zone C bound is the caller's promise that every zc_len[u] <= zc_bound
    if ((a->flags & RDKV_DECODE_ZC_BOUND) && (a->zc_bound < 0 || (a->zc_len && a->zc_bound > a->zc_cap)))
        return RDKV_EINVAL;
    const int split = a->split < 1 ? 1 : a->split;
    if (split > 1 && (!a->workspace ||
                      a->workspace_bytes < rdkv_cuda_decode_workspace(a->units, a->group, a->head_dim, split)))
        return RDKV_EINVAL;
    auto st = static_cast<cudaStream_t>(stream);
    const bool forced = a->kernel >= 2;
    const bool want_mma = forced || (a->kernel == 0 && split == 1);
    if (want_mma && mma_supported(a)) return launch_mma(a, st);
    if (forced) return RDKV_EINVAL;
    const int max_kslots = a->head_dim + 3 * 31 + 7;
    return a->io_dtype == RDKV_F32 ? launch_generic<float>(a, split, max_kslots, st)
                                   : launch_generic<__half>(a, split, max_kslots, st);
}

// Device address of mapped (pinned, UVA) host memory, or nullptr.
static const void* mapped_device_ptr(const void* host) {
    cudaPointerAttributes at{};
    if (cudaPointerGetAttributes(&at, host) != cudaSuccess) {
        cudaGetLastError();
        return nullptr;
    }
    return at.type == cudaMemoryTypeHost ? at.devicePointer : nullptr;
}

extern "C" RDKV_API int rdkv_cuda_decode_host(const rdkv_decode_args* a, const void* q_host,
                                              void* out_host, void* stream) {
    if (!a || !q_host || !out_host) return RDKV_EINVAL;
    // pinned (mapped) host buffers: zero-copy — the decode kernel streams q
    // from host memory with TMA bulk loads and writes out with bulk stores,
    // so the PCIe traffic in both directions overlaps the step itself
    const void* qd = mapped_device_ptr(q_host);
    const void* od = mapped_device_ptr(out_host);
    if (qd && od) {
        rdkv_decode_args z = *a;
        z.q = qd;
        z.out = const_cast<void*>(od);
        z.flags |= RDKV_DECODE_OUT_HOST;
        return rdkv_cuda_decode(&z, stream);
    }
    const size_t elem = a->io_dtype == RDKV_F16 ? 2 : 4;
    const size_t bytes = (size_t)a->units * a->group * a->head_dim * elem;
    auto st = static_cast<cudaStream_t>(stream);
    RDKV_CUDA_TRY(cudaMemcpyAsync(const_cast<void*>(a->q), q_host, bytes, cudaMemcpyHostToDevice, st));
    if (int rc = rdkv_cuda_decode(a, stream)) return rc;
    RDKV_CUDA_TRY(cudaMemcpyAsync(out_host, a->out, bytes, cudaMemcpyDeviceToHost, st));
    return RDKV_OK;
}

// ---- pipelined end-to-end decode -------------------------------------------
struct rdkv_decode_ctx {
    int chunks;
    cudaStream_t s_in, s_out;
    cudaEvent_t start, done;
    cudaEvent_t* in_done;
    cudaEvent_t* dec_done;
    // the last call's work captured as a CUDA graph, replayed while the
    // arguments and host buffers stay the same (one launch per step instead
    // of ~6 enqueues per chunk)
    cudaGraphExec_t exec;
    rdkv_decode_args key;
    const void* key_q;
    void* key_out;
};

extern "C" RDKV_API int rdkv_cuda_decode_ctx_create(int32_t chunks, rdkv_decode_ctx** out) {
    if (!out || chunks < 1 || chunks > 256) return RDKV_EINVAL;
    auto* c = new rdkv_decode_ctx{};
    c->chunks = chunks;
    c->in_done = new cudaEvent_t[chunks]();
    c->dec_done = new cudaEvent_t[chunks]();
    bool ok = cudaStreamCreateWithFlags(&c->s_in, cudaStreamNonBlocking) == cudaSuccess &&
              cudaStreamCreateWithFlags(&c->s_out, cudaStreamNonBlocking) == cudaSuccess &&
              cudaEventCreateWithFlags(&c->start, cudaEventDisableTiming) == cudaSuccess &&
              cudaEventCreateWithFlags(&c->done, cudaEventDisableTiming) == cudaSuccess;
    for (int i = 0; ok && i < chunks; ++i)
        ok = cudaEventCreateWithFlags(&c->in_done[i], cudaEventDisableTiming) == cudaSuccess &&
             cudaEventCreateWithFlags(&c->dec_done[i], cudaEventDisableTiming) == cudaSuccess;
    if (!ok) {
        rdkv_cuda_decode_ctx_destroy(c);
        return RDKV_ECUDA;
    }
    *out = c;
    return RDKV_OK;
}

extern "C" RDKV_API int rdkv_cuda_decode_ctx_destroy(rdkv_decode_ctx* c) {
    if (!c) return RDKV_EINVAL;
    for (int i = 0; i < c->chunks; ++i) {
        if (c->in_done[i]) cudaEventDestroy(c->in_done[i]);
        if (c->dec_done[i]) cudaEventDestroy(c->dec_done[i]);
    }
    if (c->start) cudaEventDestroy(c->start);
    if (c->done) cudaEventDestroy(c->done);
    if (c->s_in) cudaStreamDestroy(c->s_in);
    if (c->s_out) cudaStreamDestroy(c->s_out);
    if (c->exec) cudaGraphExecDestroy(c->exec);
    delete[] c->in_done;
    delete[] c->dec_done;
    delete c;
    return RDKV_OK;
}

static int enqueue_pipelined(rdkv_decode_ctx* c, const rdkv_decode_args* a, const void* q_host, void* out_host,
                             void* stream) {
    const size_t row = (size_t)a->group * a->head_dim * (a->io_dtype == RDKV_F16 ? 2 : 4);
    auto st = static_cast<cudaStream_t>(stream);
    const int nch = a->units < c->chunks ? a->units : c->chunks;
    // fork: the copies are ordered after everything already queued on `stream`
    RDKV_CUDA_TRY(cudaEventRecord(c->start, st));
    RDKV_CUDA_TRY(cudaStreamWaitEvent(c->s_in, c->start, 0));
    RDKV_CUDA_TRY(cudaStreamWaitEvent(c->s_out, c->start, 0));
    for (int i = 0; i < nch; ++i) {
        const int u0 = (int)((int64_t)a->units * i / nch), u1 = (int)((int64_t)a->units * (i + 1) / nch);
        const size_t off = (size_t)u0 * row, bytes = (size_t)(u1 - u0) * row;
        RDKV_CUDA_TRY(cudaMemcpyAsync(static_cast<uint8_t*>(const_cast<void*>(a->q)) + off,
                                      static_cast<const uint8_t*>(q_host) + off, bytes, cudaMemcpyHostToDevice,
                                      c->s_in));
        RDKV_CUDA_TRY(cudaEventRecord(c->in_done[i], c->s_in));
        RDKV_CUDA_TRY(cudaStreamWaitEvent(st, c->in_done[i], 0));
        rdkv_decode_args sub = *a;
        sub.units = u1 - u0;
        sub.tile_offsets = a->tile_offsets + u0;
        if (a->tile_decode_bytes) sub.tile_decode_bytes = a->tile_decode_bytes + u0;
        sub.q = static_cast<const uint8_t*>(a->q) + off;
        sub.out = static_cast<uint8_t*>(a->out) + off;
        // unit_ids index the whole arena (and list units out of order): a chunk
        // of consecutive units is decoded without them (mixed chunks take the
        // general body), never through ids that point outside the shifted views
        sub.unit_ids = nullptr;
        sub.plan.n_uniform = 0;
        sub.plan.uniform2_split = 0;
        if (a->zc_len) {
            const size_t zrow = (size_t)a->zc_cap * a->head_dim * 2;
            sub.zc_k = static_cast<const uint8_t*>(a->zc_k) + (size_t)u0 * zrow;
            sub.zc_v = static_cast<const uint8_t*>(a->zc_v) + (size_t)u0 * zrow;
            sub.zc_len = a->zc_len + u0;
        }
        if (int rc = rdkv_cuda_decode(&sub, stream)) return rc;
        RDKV_CUDA_TRY(cudaEventRecord(c->dec_done[i], st));
        RDKV_CUDA_TRY(cudaStreamWaitEvent(c->s_out, c->dec_done[i], 0));
        RDKV_CUDA_TRY(cudaMemcpyAsync(static_cast<uint8_t*>(out_host) + off,
                                      static_cast<const uint8_t*>(a->out) + off, bytes, cudaMemcpyDeviceToHost,
                                      c->s_out));
    }
    // join: `stream` is ordered after the last D2H
    RDKV_CUDA_TRY(cudaEventRecord(c->done, c->s_out));
    RDKV_CUDA_TRY(cudaStreamWaitEvent(st, c->done, 0));
    return RDKV_OK;
}

extern "C" RDKV_API int rdkv_cuda_decode_host_pipelined(rdkv_decode_ctx* c, const rdkv_decode_args* a,
                                                        const void* q_host, void* out_host, void* stream) {
    if (!c || !a || !q_host || !out_host || !a->q || !a->out || a->units < 1) return RDKV_EINVAL;
    if (a->split > 1) return RDKV_EINVAL;  // chunks share one unit-indexed workspace otherwise
    auto st = static_cast<cudaStream_t>(stream);
    if (!st) return enqueue_pipelined(c, a, q_host, out_host, stream);  // legacy stream: no capture
    if (c->exec && c->key_q == q_host && c->key_out == out_host && memcmp(&c->key, a, sizeof(*a)) == 0) {
        RDKV_CUDA_TRY(cudaGraphLaunch(c->exec, st));
        return RDKV_OK;
    }
    if (c->exec) {
        cudaGraphExecDestroy(c->exec);
        c->exec = nullptr;
    }
    RDKV_CUDA_TRY(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
    const int rc = enqueue_pipelined(c, a, q_host, out_host, stream);
    cudaGraph_t graph = nullptr;
    const cudaError_t e = cudaStreamEndCapture(st, &graph);
    if (rc != RDKV_OK) {
        if (graph) cudaGraphDestroy(graph);
        return rc;
    }
    if (e != cudaSuccess) return RDKV_ECUDA;
    const cudaError_t ie = cudaGraphInstantiate(&c->exec, graph, 0);
    cudaGraphDestroy(graph);
    if (ie != cudaSuccess) {
        c->exec = nullptr;
        return RDKV_ECUDA;
    }
    c->key = *a;
    c->key_q = q_host;
    c->key_out = out_host;
    RDKV_CUDA_TRY(cudaGraphLaunch(c->exec, st));
    return RDKV_OK;
}

// ---- sequence split across ranks (optional merge) ----------
extern "C" RDKV_API int rdkv_cuda_decode_partial(const rdkv_decode_args* a, int32_t rank, int32_t world,
                                                 float* partial, void* stream) {
    if (!a || !partial || world < 1 || rank < 0 || rank >= world || !a->arena || !a->q) return RDKV_EINVAL;
    return launch_partial(a, rank, world, partial, static_cast<cudaStream_t>(stream));
}

extern "C" RDKV_API int rdkv_cuda_decode_merge(const float* partials, int32_t nparts, int32_t units, int32_t group,
                                               int32_t head_dim, void* out, int32_t io_dtype, void* stream) {
    if (!partials || !out || nparts < 1 || units < 1 || group < 1 || head_dim < 1) return RDKV_EINVAL;
    if (io_dtype != RDKV_F32 && io_dtype != RDKV_F16) return RDKV_EINVAL;
    return launch_merge(partials, nparts, units * group, head_dim, out, io_dtype, static_cast<cudaStream_t>(stream));
}
