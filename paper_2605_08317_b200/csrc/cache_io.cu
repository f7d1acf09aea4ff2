// cache_io.cu — RDKVC001 cache containers straight into device memory.
//
// Replaces load_cache / load_cache_file (reference proj/core/src/cache.cpp:228-295) for the
// device path: the container's payload order (K, V, probe_Q; layer-major, head-major,
// row-major, cache.cpp:205-226) is already the device unit order, so the payload is
// streamed with large parallel reads into a persistent pinned double buffer and copied to its final place —
// no host re-layout, no host-side KVCache. Reads overlap the H2D copies of the previous
// chunk (two buffers); fp16 targets are converted on the device, where the finiteness check
// of KVCache::validate (cache.cpp:114-130) also runs.
#include <fcntl.h>
#include <sys/stat.h>
#include <unistd.h>

#include <atomic>
#include <cctype>
#include <mutex>
#include <thread>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <string>

#include "common.cuh"

namespace rdkv_b200 {
namespace {

constexpr char kCacheMagic[8] = {'R', 'D', 'K', 'V', 'C', '0', '0', '1'};
constexpr uint32_t kMaxHeader = 1u << 20;          // cache.cpp:235
constexpr size_t kChunkBytes = size_t(32) << 20;   // per pinned buffer

// ---- minimal JSON reader for the flat header object ---------------------------------------
// Accepts any JSON document; records the top-level members of an object (numbers, strings,
// booleans). Anything malformed or trailing is an error, as json::parse is (cache.cpp:243-248).
struct JsonField {
    enum Kind { NONE, NUMBER, STRING, BOOL, OTHER } kind = NONE;
    double num = 0;
    bool is_int = false;
    long long inum = 0;
    std::string str;
};

struct Json {
    const char* p;
    const char* e;
    bool ok = true;

    void ws() {
        while (p < e && (*p == ' ' || *p == '\t' || *p == '\n' || *p == '\r')) ++p;
    }
    bool lit(const char* s) {
        size_t n = strlen(s);
        if (size_t(e - p) < n || memcmp(p, s, n) != 0) return ok = false;
        p += n;
        return true;
    }
    bool hex4(const char* q, uint32_t& v) {
        if (e - q < 4) return false;
        v = 0;
        for (int i = 0; i < 4; ++i) {
            const unsigned char c = (unsigned char)q[i];
            if (!isxdigit(c)) return false;
            v = v * 16 + (uint32_t)(isdigit(c) ? c - '0' : (tolower(c) - 'a' + 10));
        }
        return true;
    }
    static void utf8(uint32_t cp, std::string& out) {
        if (cp < 0x80) {
            out.push_back((char)cp);
        } else if (cp < 0x800) {
            out.push_back((char)(0xC0 | (cp >> 6)));
            out.push_back((char)(0x80 | (cp & 0x3F)));
        } else if (cp < 0x10000) {
            out.push_back((char)(0xE0 | (cp >> 12)));
            out.push_back((char)(0x80 | ((cp >> 6) & 0x3F)));
            out.push_back((char)(0x80 | (cp & 0x3F)));
        } else {
            out.push_back((char)(0xF0 | (cp >> 18)));
            out.push_back((char)(0x80 | ((cp >> 12) & 0x3F)));
            out.push_back((char)(0x80 | ((cp >> 6) & 0x3F)));
            out.push_back((char)(0x80 | (cp & 0x3F)));
        }
    }
    bool string(std::string* out) {
        if (p >= e || *p != '"') return ok = false;
        ++p;
        while (p < e && *p != '"') {
            unsigned char c = (unsigned char)*p;
            if (c < 0x20) return ok = false;
            if (c == '\\') {
                if (++p >= e) return ok = false;
                char x = *p;
                if (x == 'u') {
                    // \uXXXX (and surrogate pairs) to UTF-8, like nlohmann::json;
                    // a lone or mismatched surrogate is a parse error there too
                    uint32_t cp = 0;
                    if (!hex4(p + 1, cp)) return ok = false;
                    p += 5;
                    if (cp >= 0xDC00 && cp <= 0xDFFF) return ok = false;
                    if (cp >= 0xD800 && cp <= 0xDBFF) {
                        uint32_t lo = 0;
                        if (e - p < 6 || p[0] != '\\' || p[1] != 'u' || !hex4(p + 2, lo) || lo < 0xDC00 || lo > 0xDFFF)
                            return ok = false;
                        p += 6;
                        cp = 0x10000 + ((cp - 0xD800) << 10) + (lo - 0xDC00);
                    }
                    if (out) utf8(cp, *out);
                    continue;
                }
                const char* esc = strchr("\"\\/bfnrt", x);
                if (!esc || !x) return ok = false;
                if (out) out->push_back("\"\\/\b\f\n\r\t"[esc - "\"\\/bfnrt"]);
                ++p;
                continue;
            }
            if (out) out->push_back((char)c);
            ++p;
        }
        if (p >= e) return ok = false;
        ++p;
        return true;
    }
    bool number(JsonField* f) {
        const char* s = p;
        if (p < e && *p == '-') ++p;
        if (p >= e || !isdigit((unsigned char)*p)) return ok = false;
        if (*p == '0') ++p;
        else
            while (p < e && isdigit((unsigned char)*p)) ++p;
        bool integral = true;
        if (p < e && *p == '.') {
            integral = false;
            ++p;
            if (p >= e || !isdigit((unsigned char)*p)) return ok = false;
            while (p < e && isdigit((unsigned char)*p)) ++p;
        }
        if (p < e && (*p == 'e' || *p == 'E')) {
            integral = false;
            ++p;
            if (p < e && (*p == '+' || *p == '-')) ++p;
            if (p >= e || !isdigit((unsigned char)*p)) return ok = false;
            while (p < e && isdigit((unsigned char)*p)) ++p;
        }
        std::string t(s, p);
        if (f) {
            f->kind = JsonField::NUMBER;
            f->num = strtod(t.c_str(), nullptr);
            f->is_int = integral;
            if (integral) f->inum = strtoll(t.c_str(), nullptr, 10);
        }
        return true;
    }
    bool value(JsonField* f, int depth) {
        if (depth > 4096) return ok = false;  // nesting guard for the recursive reader only
        ws();
        if (p >= e) return ok = false;
        char c = *p;
        if (c == '{' || c == '[') {
            if (f) f->kind = JsonField::OTHER;
            ++p;
            ws();
            char close = c == '{' ? '}' : ']';
            if (p < e && *p == close) {
                ++p;
                return true;
            }
            for (;;) {
                ws();
                if (c == '{') {
                    if (!string(nullptr)) return false;
                    ws();
                    if (p >= e || *p != ':') return ok = false;
                    ++p;
                }
                if (!value(nullptr, depth + 1)) return false;
                ws();
                if (p < e && *p == ',') {
                    ++p;
                    continue;
                }
                if (p < e && *p == close) {
                    ++p;
                    return true;
                }
                return ok = false;
            }
        }
        if (c == '"') {
            std::string s;
            if (!string(&s)) return false;
            if (f) {
                f->kind = JsonField::STRING;
                f->str = s;
            }
            return true;
        }
        if (c == 't' || c == 'f') {
            if (!lit(c == 't' ? "true" : "false")) return false;
            if (f) {
                f->kind = JsonField::BOOL;
                f->inum = c == 't';
            }
            return true;
        }
        if (c == 'n') {
            if (!lit("null")) return false;
            if (f) f->kind = JsonField::OTHER;
            return true;
        }
        return number(f);
    }
};

constexpr const char* kKeys[7] = {"L", "H_q", "H_kv", "d", "T", "S_w", "dtype"};

// Parses the header object; fields[i] receives the LAST occurrence of kKeys[i].
bool parse_header(const std::string& text, JsonField* fields) {
    Json j{text.data(), text.data() + text.size()};
    j.ws();
    if (j.p >= j.e) return false;
    if (*j.p != '{') {  // a valid non-object document: header.at() would throw type_error
        if (!j.value(nullptr, 0)) return false;
        j.ws();
        return false;
    }
    ++j.p;
    j.ws();
    if (j.p < j.e && *j.p == '}') {
        ++j.p;
    } else {
        for (;;) {
            j.ws();
            std::string key;
            if (!j.string(&key)) return false;
            j.ws();
            if (j.p >= j.e || *j.p != ':') return false;
            ++j.p;
            JsonField f;
            if (!j.value(&f, 1)) return false;
            for (int i = 0; i < 7; ++i)
                if (key == kKeys[i]) fields[i] = f;
            j.ws();
            if (j.p < j.e && *j.p == ',') {
                ++j.p;
                continue;
            }
            if (j.p < j.e && *j.p == '}') {
                ++j.p;
                break;
            }
            return false;
        }
    }
    j.ws();
    return j.p == j.e;  // trailing content is a parse error
}

// json::get<int>() semantics for the shape fields: numbers (integral or not) and booleans
// convert, anything else (string, null, object, missing) is a FormatError.
bool as_int(const JsonField& f, int32_t* out) {
    if (f.kind == JsonField::NUMBER) {
        if (f.is_int) {
            *out = (int32_t)(uint32_t)(unsigned long long)f.inum;
        } else {
            if (!(std::fabs(f.num) < 2147483648.0)) return false;
            *out = (int32_t)f.num;
        }
        return true;
    }
    if (f.kind == JsonField::BOOL) {
        *out = (int32_t)f.inum;
        return true;
    }
    return false;
}

bool read_all(int fd, void* dst, size_t n, off_t off) {
    char* d = static_cast<char*>(dst);
    while (n > 0) {
        ssize_t r = pread(fd, d, n, off);
        if (r <= 0) return false;
        d += r;
        n -= (size_t)r;
        off += r;
    }
    return true;
}

struct Fd {
    int fd;
    explicit Fd(const char* path) : fd(open(path, O_RDONLY | O_CLOEXEC)) {}
    ~Fd() {
        if (fd >= 0) close(fd);
    }
};

// f32 chunk (device staging) -> destination dtype, with the finiteness / fp16-range flag.
template <typename T>
__global__ void __launch_bounds__(256) convert_kernel(const float* __restrict__ src, T* __restrict__ dst,
                                                      size_t n, int* __restrict__ bad) {
    int flag = 0;
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
        float x = src[i];
        if (!isfinite(x) || (sizeof(T) == 2 && fabsf(x) > 65504.f)) flag = 1;
        if constexpr (sizeof(T) == 2) {
            dst[i] = __float2half_rn(x);
        } else {
            dst[i] = x;
        }
    }
    if (__syncthreads_or(flag) && threadIdx.x == 0) atomicOr(bad, 1);
}

}  // namespace
}  // namespace rdkv_b200

using namespace rdkv_b200;

extern "C" RDKV_API int rdkv_cache_read_header(const char* path, rdkv_cache_header* h) {
    if (!path || !h) return RDKV_EINVAL;
    Fd f(path);
    if (f.fd < 0) return RDKV_EFORMAT;  // load_cache_file: "cannot open for reading"
    struct stat sb;
    if (fstat(f.fd, &sb) != 0) return RDKV_EFORMAT;
    const long long fsize = (long long)sb.st_size;
    unsigned char pre[12];
    if (fsize < 8 || !read_all(f.fd, pre, 8, 0) || memcmp(pre, kCacheMagic, 8) != 0) return RDKV_EFORMAT;
    if (fsize < 12 || !read_all(f.fd, pre + 8, 4, 8)) return RDKV_EFORMAT;
    const uint32_t hlen = (uint32_t)pre[8] | ((uint32_t)pre[9] << 8) | ((uint32_t)pre[10] << 16) |
                          ((uint32_t)pre[11] << 24);
    if (hlen == 0 || hlen > kMaxHeader) return RDKV_EFORMAT;
    if (fsize < 12 + (long long)hlen) return RDKV_EFORMAT;
    std::string text(hlen, '\0');
    if (!read_all(f.fd, &text[0], hlen, 12)) return RDKV_EFORMAT;

    JsonField fields[7];
    if (!parse_header(text, fields)) return RDKV_EFORMAT;
    int32_t dims[6];
    for (int i = 0; i < 6; ++i)
        if (!as_int(fields[i], &dims[i])) return RDKV_EFORMAT;
    if (fields[6].kind != JsonField::STRING) return RDKV_EFORMAT;
    if (fields[6].str != "f32") return RDKV_EFORMAT;
    const int32_t L = dims[0], Hq = dims[1], Hkv = dims[2], d = dims[3], T = dims[4], Sw = dims[5];
    // CacheShape::validate (cache.cpp:95-105): std::invalid_argument
    if (L < 1 || d < 1 || T < 1 || Hq < 1 || Hkv < 1 || Hq % Hkv != 0) return RDKV_EINVAL;
    if (Sw < 1 || Sw > T) return RDKV_EFORMAT;  // cache.cpp:265-267
    const double kv = (double)L * Hkv * T * d, qn = (double)L * Hq * Sw * d;
    const double total = 4.0 * (2.0 * kv + qn);
    if (total > 9.0e18) return RDKV_EFORMAT;
    const long long payload = 4ll * (2ll * L * Hkv * T * d + (long long)L * Hq * Sw * d);
    // truncated payload / trailing bytes (cache.cpp:275-283)
    if (fsize != 12 + (long long)hlen + payload) return RDKV_EFORMAT;
    h->layers = L;
    h->q_heads = Hq;
    h->kv_heads = Hkv;
    h->head_dim = d;
    h->seq_len = T;
    h->probe_window = Sw;
    h->payload_offset = 12 + (long long)hlen;
    h->payload_bytes = payload;
    return RDKV_OK;
}

extern "C" RDKV_API int rdkv_cuda_cache_load(const char* path, const rdkv_cache_header* h, void* k,
                                             void* v, void* probe_q, int32_t dtype, void* stream) {
    if (!path || !h || !k || !v || !probe_q) return RDKV_EINVAL;
    if (dtype != RDKV_F32 && dtype != RDKV_F16) return RDKV_EINVAL;
    rdkv_cache_header chk;
    int rc = rdkv_cache_read_header(path, &chk);
    if (rc != RDKV_OK) return rc;
    if (memcmp(&chk, h, sizeof(chk)) != 0) return RDKV_EINVAL;  // header from another file
    Fd f(path);
    if (f.fd < 0) return RDKV_EFORMAT;
    posix_fadvise(f.fd, 0, 0, POSIX_FADV_SEQUENTIAL);

    const size_t esz = dtype == RDKV_F16 ? 2 : 4;
    const size_t kv_n = (size_t)h->layers * h->kv_heads * h->seq_len * h->head_dim;
    const size_t q_n = (size_t)h->layers * h->q_heads * h->probe_window * h->head_dim;
    struct Seg {
        char* dst;
        size_t n;
    } segs[3] = {{static_cast<char*>(k), kv_n}, {static_cast<char*>(v), kv_n}, {static_cast<char*>(probe_q), q_n}};

    auto st = static_cast<cudaStream_t>(stream);
    // one process-wide pinned double buffer (allocated on first use, kept): pinned allocation
    // costs more than reading a small container; loads serialise on it
    static std::mutex pool_mu;
    static float* pool[2] = {nullptr, nullptr};
    std::lock_guard<std::mutex> lock(pool_mu);
    for (int b = 0; b < 2; ++b)
        if (!pool[b] && cudaHostAlloc((void**)&pool[b], kChunkBytes, cudaHostAllocDefault) != cudaSuccess) {
            pool[b] = nullptr;
            return RDKV_ECUDA;
        }
    float* stage[2] = {nullptr, nullptr};
    cudaEvent_t done[2] = {nullptr, nullptr};
    int* bad = nullptr;
    int bad_h = 0;
    rc = RDKV_OK;
    const size_t chunk_n = kChunkBytes / 4;
    const size_t total_n = 2 * kv_n + q_n;
    const size_t stage_bytes = (total_n < chunk_n ? total_n : chunk_n) * 4;
    auto fail = [&](int code) {
        if (rc == RDKV_OK) rc = code;
    };
    for (int b = 0; b < 2 && rc == RDKV_OK; ++b) {
        if (cudaMallocAsync((void**)&stage[b], stage_bytes, st) != cudaSuccess) fail(RDKV_ECUDA);
        else if (cudaEventCreateWithFlags(&done[b], cudaEventDisableTiming) != cudaSuccess) fail(RDKV_ECUDA);
    }
    if (rc == RDKV_OK && cudaMallocAsync((void**)&bad, sizeof(int), st) != cudaSuccess) fail(RDKV_ECUDA);
    if (rc == RDKV_OK && cudaMemsetAsync(bad, 0, sizeof(int), st) != cudaSuccess) fail(RDKV_ECUDA);

    // page-cache copies are memcpy-bound per thread: a chunk is read by up to kReaders threads
    constexpr int kReaders = 4;
    auto read_chunk = [&](float* dst, size_t n, off_t off) {
        const size_t bytes = n * 4;
        if (bytes < (size_t(4) << 20)) return read_all(f.fd, dst, bytes, off);
        std::atomic<bool> ok{true};
        std::thread th[kReaders];
        const size_t part = (bytes / kReaders + 4095) & ~size_t(4095);
        for (int r = 0; r < kReaders; ++r) {
            const size_t b0 = (size_t)r * part;
            if (b0 >= bytes) break;
            const size_t nb = bytes - b0 < part ? bytes - b0 : part;
            th[r] = std::thread([&, b0, nb] {
                if (!read_all(f.fd, reinterpret_cast<char*>(dst) + b0, nb, off + (off_t)b0)) ok = false;
            });
        }
        for (auto& t : th)
            if (t.joinable()) t.join();
        return ok.load();
    };

    off_t off = (off_t)h->payload_offset;
    int buf = 0;
    bool used[2] = {false, false};
    for (int s = 0; s < 3 && rc == RDKV_OK; ++s) {
        for (size_t e0 = 0; e0 < segs[s].n && rc == RDKV_OK; e0 += chunk_n) {
            const size_t n = segs[s].n - e0 < chunk_n ? segs[s].n - e0 : chunk_n;
            if (used[buf] && cudaEventSynchronize(done[buf]) != cudaSuccess) {
                fail(RDKV_ECUDA);
                break;
            }
            if (!read_chunk(pool[buf], n, off)) {
                fail(RDKV_EFORMAT);  // file changed under us
                break;
            }
            off += (off_t)(n * 4);
            if (cudaMemcpyAsync(stage[buf], pool[buf], n * 4, cudaMemcpyHostToDevice, st) != cudaSuccess) {
                fail(RDKV_ECUDA);
                break;
            }
            const int threads = 256;
            size_t blocks = (n + threads - 1) / threads;
            const int nb = (int)(blocks < 148u * 16 ? blocks : 148u * 16);
            char* dst = segs[s].dst + e0 * esz;
            if (dtype == RDKV_F16)
                convert_kernel<__half><<<nb, threads, 0, st>>>(stage[buf], reinterpret_cast<__half*>(dst), n, bad);
            else
                convert_kernel<float><<<nb, threads, 0, st>>>(stage[buf], reinterpret_cast<float*>(dst), n, bad);
            if (cudaGetLastError() != cudaSuccess || cudaEventRecord(done[buf], st) != cudaSuccess) {
                fail(RDKV_ECUDA);
                break;
            }
            used[buf] = true;
            buf ^= 1;
        }
    }
    if (bad && cudaMemcpyAsync(&bad_h, bad, sizeof(int), cudaMemcpyDeviceToHost, st) != cudaSuccess) fail(RDKV_ECUDA);
    for (int b = 0; b < 2; ++b)
        if (stage[b]) cudaFreeAsync(stage[b], st);
    if (bad) cudaFreeAsync(bad, st);
    if (cudaStreamSynchronize(st) != cudaSuccess) fail(RDKV_ECUDA);  // pool buffers free for the next load
    for (int b = 0; b < 2; ++b)
        if (done[b]) cudaEventDestroy(done[b]);
    if (rc == RDKV_OK && bad_h) rc = RDKV_ENUMERIC;
    return rc;
}
