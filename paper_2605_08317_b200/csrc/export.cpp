// export.cpp — host-side view of a device tile in the reference's terms.
//
// Rebuilds, from the bytes of one packed device tile, everything the
// reference TriZoneCache holds for Zones A/B (trizone.hpp:34-78): kept token
// ids, V segments (members ascending, positions into kept order, one
// QuantParams per row, payload rows packed with pack_bits conventions,
// trizone.cpp:126-143), Zone B rows, K segments (members, one QuantParams per
// channel, payload rows over the kept tokens, trizone.cpp:159-184), k16
// columns and channel_perm (trizone.cpp:186-206). Used by the parity tests
// (byte-for-byte against build_trizone) and by the C++ drop-in layer to hand
// a reference-shaped TriZoneCache back to callers.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <vector>

#include <cuda_fp16.h>

#include "../../include/rdkv_cuda.h"
#include "tile_layout.h"

using namespace rdkv_b200;

namespace {

float half_to_float(const uint8_t* p) {
    __half h;
    std::memcpy(&h, p, 2);
    return __half2float(h);
}

struct TileView {
    TileHeader h;
    const uint8_t* base;
    int d;
    std::vector<int> sbase;

    TileView(const uint8_t* t, int d_) : base(t), d(d_) {
        std::memcpy(&h, t, sizeof(h));
        sbase.resize(5);
        int acc = 0;
        for (int i = 0; i < 4; ++i) {
            sbase[i] = acc;
            acc += pad4(h.r[i]);
        }
        sbase[4] = acc;
    }
    int32_t id(int slot) const {
        int32_t v;
        std::memcpy(&v, base + h.off_ids + 4 * slot, 4);
        return v;
    }
    int64_t vz(int slot) const {
        int64_t v;
        std::memcpy(&v, base + h.off_vz + 8 * slot, 8);
        return v;
    }
    int64_t kz(int ks) const {
        int64_t v;
        std::memcpy(&v, base + h.off_kz + 8 * ks, 8);
        return v;
    }
    float vscale(int slot) const {
        float v;
        std::memcpy(&v, base + h.off_vp + 8 * slot, 4);
        return v;
    }
    float kscale(int ks) const {
        float v;
        std::memcpy(&v, base + chan_table_off() + 8 * ks, 4);
        return v;
    }
    int perm(int ks) const {
        uint16_t v;
        std::memcpy(&v, base + perm_off(h) + 2 * ks, 2);
        return v;
    }
    const uint8_t* krow(int slot) const { return base + krow_offset(h, slot); }
};

unsigned extract(const uint8_t* row, int j, int bits) {
    switch (bits) {
        case 2: return (row[j >> 2] >> ((j & 3) * 2)) & 3u;
        case 4: return (row[j >> 1] >> ((j & 1) * 4)) & 15u;
        default: return row[j];
    }
}

}  // namespace

extern "C" RDKV_API int rdkv_tile_info_get(const uint8_t* tile_host, rdkv_tile_info* info) {
    if (!tile_host || !info) return RDKV_EINVAL;
    TileHeader h;
    std::memcpy(&h, tile_host, sizeof(h));
    if (h.magic != kTileMagic) return RDKV_EFORMAT;
    info->n_kept = h.n;
    for (int i = 0; i < 4; ++i) {
        info->rows[i] = h.r[i];
        info->chans[i] = h.c[i];
    }
    info->kslots = h.kslots;
    info->krow_bytes = h.krow_bytes;
    info->nslot = h.nslot;
    info->total_bytes = h.total_bytes;
    info->decode_bytes = tile_decode_bytes(h);
    return RDKV_OK;
}

extern "C" RDKV_API size_t rdkv_tile_export_payload_bytes(const uint8_t* tile_host, int32_t d) {
    TileHeader h;
    std::memcpy(&h, tile_host, sizeof(h));
    if (h.magic != kTileMagic) return 0;
    size_t n = 0;
    for (int i = 0; i < 3; ++i) {
        n += (size_t)h.r[i] * ref_row_bytes(d, kBits(i));
        if (h.c[i] > 0) n += (size_t)h.n * ref_row_bytes(h.c[i], kBits(i));
    }
    return n;
}

extern "C" RDKV_API int rdkv_tile_export(const uint8_t* tile_host, int32_t d, int32_t* kept,
                                         uint8_t* vcodes, float* vscale, int64_t* vzero,
                                         uint8_t* kcodes, float* kscale, int64_t* kzero, float* vfp,
                                         float* kfp, uint8_t* payload, int32_t* segtab, int32_t* nseg,
                                         int32_t* perm, int32_t* nperm) {
    if (!tile_host) return RDKV_EINVAL;
    TileView tv(tile_host, d);
    const TileHeader& h = tv.h;
    if (h.magic != kTileMagic) return RDKV_EFORMAT;
    const int n = h.n;

    // kept (ascending token id) and the slot of every kept index
    std::vector<std::pair<int, int>> order;  // (token, slot)
    for (int cls = 0; cls < 4; ++cls)
        for (int li = 0; li < h.r[cls]; ++li) order.emplace_back(tv.id(tv.sbase[cls] + li), tv.sbase[cls] + li);
    std::sort(order.begin(), order.end());
    if ((int)order.size() != n) return RDKV_EFORMAT;
    std::vector<int> slot_of_kept(n), kept_of_slot(h.nslot, -1);
    for (int i = 0; i < n; ++i) {
        kept[i] = order[i].first;
        slot_of_kept[i] = order[i].second;
        kept_of_slot[order[i].second] = i;
    }
    std::memset(vcodes, 0, (size_t)n * d);
    std::memset(vscale, 0, sizeof(float) * n);
    std::memset(vzero, 0, sizeof(int64_t) * n);
    std::memset(kcodes, 0, (size_t)n * d);
    std::memset(kscale, 0, sizeof(float) * d);
    std::memset(kzero, 0, sizeof(int64_t) * d);
    std::memset(vfp, 0, sizeof(float) * (size_t)n * d);
    std::memset(kfp, 0, sizeof(float) * (size_t)n * d);

    size_t off = 0;
    int ns = 0;
    // V segments, ascending width, members ascending token id (slot order)
    for (int cls = 0; cls < 3; ++cls) {
        if (h.r[cls] == 0) continue;
        const int bits = kBits(cls);
        const int rb = ref_row_bytes(d, bits);
        for (int li = 0; li < h.r[cls]; ++li) {
            const int slot = tv.sbase[cls] + li;
            const int p = kept_of_slot[slot];
            vscale[p] = tv.vscale(slot);
            vzero[p] = tv.vz(slot);
            uint8_t* dst = payload + off + (size_t)li * rb;
            for (int m = 0; m < rb; ++m) dst[m] = tile_host[vbyte_offset(h, cls, li, m, d)];
            for (int c = 0; c < d; ++c) vcodes[(size_t)p * d + c] = (uint8_t)extract(dst, c, bits);
        }
        int32_t* row = segtab + 6 * ns++;
        row[0] = 0; row[1] = bits; row[2] = h.r[cls]; row[3] = d;
        row[4] = ref_padded_len(d, bits) - d; row[5] = h.r[cls] * rb;
        off += (size_t)h.r[cls] * rb;
    }
    // Zone B
    for (int li = 0; li < h.r[3]; ++li) {
        const int slot = tv.sbase[3] + li;
        const int p = kept_of_slot[slot];
        const uint8_t* src = tile_host + h.off_vseg[3] + (size_t)li * d * 2;
        for (int c = 0; c < d; ++c) vfp[(size_t)p * d + c] = half_to_float(src + 2 * c);
    }
    // K segments over the kept rows in kept order
    int np = 0;
    for (int cls = 0; cls < 3; ++cls) {
        const int nc = h.c[cls];
        if (nc == 0 || n == 0) continue;
        const int bits = kBits(cls);
        const int rb = ref_row_bytes(nc, bits);
        for (int j = 0; j < nc; ++j) {
            const int ks = h.kslot_base[cls] + j;
            const int ch = tv.perm(ks);
            kscale[ch] = tv.kscale(ks);
            kzero[ch] = tv.kz(ks);
            perm[np++] = ch;
        }
        for (int r = 0; r < n; ++r) {
            const uint8_t* src = tv.krow(slot_of_kept[r]) + h.kbyte_base[cls];
            uint8_t* dst = payload + off + (size_t)r * rb;
            std::memcpy(dst, src, rb);  // same packing; device pads beyond the reference pads are 0
            for (int j = 0; j < nc; ++j)
                kcodes[(size_t)tv.perm(h.kslot_base[cls] + j) * n + r] = (uint8_t)extract(dst, j, bits);
        }
        int32_t* row = segtab + 6 * ns++;
        row[0] = 1; row[1] = bits; row[2] = n; row[3] = nc;
        row[4] = ref_padded_len(nc, bits) - nc; row[5] = n * rb;
        off += (size_t)n * rb;
    }
    // k16 columns
    for (int j = 0; j < h.c[3] && n > 0; ++j) {
        const int ch = tv.perm(h.kslot_base[3] + j);
        perm[np++] = ch;
        for (int r = 0; r < n; ++r)
            kfp[(size_t)r * d + ch] = half_to_float(tv.krow(slot_of_kept[r]) + h.kbyte_base[3] + 2 * j);
    }
    *nseg = ns;
    *nperm = np;
    return RDKV_OK;
}

namespace {

int import_header(int32_t d, int32_t n, const uint8_t* vbits_kept, const uint8_t* kbits, TileHeader& h) {
    if (d < 1 || d > 65535 || n < 0 || (n > 0 && !vbits_kept) || !kbits) return RDKV_EINVAL;
    std::memset(&h, 0, sizeof(h));
    for (int i = 0; i < n; ++i) {
        const int cls = class_of_bits(vbits_kept[i]);
        if (cls < 0) return RDKV_EINVAL;
        h.r[cls]++;
    }
    for (int c = 0; c < d; ++c) {
        if (kbits[c] == 0) continue;
        const int cls = class_of_bits(kbits[c]);
        if (cls < 0) return RDKV_EINVAL;
        h.c[cls]++;
    }
    tile_layout(h, d);
    return RDKV_OK;
}

void put_bits(uint8_t* row, int j, int bits, unsigned code) {
    if (bits == 8) row[j] = (uint8_t)code;
    else if (bits == 4) row[j >> 1] |= (uint8_t)((code & 15u) << ((j & 1) * 4));
    else row[j >> 2] |= (uint8_t)((code & 3u) << ((j & 3) * 2));
}

void put_half(uint8_t* p, float x) {
    const __half v = __float2half_rn(x);
    std::memcpy(p, &v, 2);
}

float offset_of(float scale, int64_t zero) { return (float)(-(double)scale * (double)zero); }

}  // namespace

extern "C" RDKV_API size_t rdkv_tile_import_bytes(int32_t d, int32_t n, const uint8_t* vbits_kept,
                                                  const uint8_t* kbits) {
    TileHeader h;
    return import_header(d, n, vbits_kept, kbits, h) ? 0 : (size_t)h.total_bytes;
}

extern "C" RDKV_API int rdkv_tile_import(int32_t d, int32_t n, const int32_t* kept, const uint8_t* vbits_kept,
                                         const uint8_t* vcodes, const float* vscale, const int64_t* vzero,
                                         const float* vfp, const uint8_t* kbits, const uint8_t* kcodes,
                                         const float* kscale, const int64_t* kzero, const float* kfp,
                                         uint8_t* tile, size_t tile_bytes) {
    TileHeader h;
    if (int rc = import_header(d, n, vbits_kept, kbits, h)) return rc;
    if (!tile || tile_bytes < (size_t)h.total_bytes) return RDKV_EINVAL;
    if (n > 0 && (!kept || !vcodes || !vscale || !vzero || !vfp || !kcodes || !kscale || !kzero || !kfp))
        return RDKV_EINVAL;
    for (int i = 1; i < n; ++i)
        if (kept[i] <= kept[i - 1]) return RDKV_EINVAL;  // kept is ascending (trizone.hpp:63)
    std::memset(tile, 0, h.total_bytes);
    std::memcpy(tile, &h, sizeof(h));

    // token slots: class order, ascending id inside a class (pads carry id -1)
    std::vector<int> slot_of(n);
    int32_t* ids = reinterpret_cast<int32_t*>(tile + h.off_ids);
    for (int s = 0; s < h.nslot; ++s) ids[s] = -1;
    int cursor[4];
    for (int cls = 0; cls < 4; ++cls) cursor[cls] = slot_base(h, cls);
    for (int i = 0; i < n; ++i) {
        const int cls = class_of_bits(vbits_kept[i]);
        slot_of[i] = cursor[cls]++;
        ids[slot_of[i]] = kept[i];
    }
    if (n == 0) return RDKV_OK;

    // K slots (channel_perm order) with their dequantisation table
    float* chan = reinterpret_cast<float*>(tile + chan_table_off());
    uint16_t* perm = reinterpret_cast<uint16_t*>(tile + perm_off(h));
    int64_t* kz = reinterpret_cast<int64_t*>(tile + h.off_kz);
    std::vector<int> kslot_of(d, -1);
    int kc[4] = {0, 0, 0, 0};
    for (int c = 0; c < d; ++c) {
        if (kbits[c] == 0) continue;
        const int cls = class_of_bits(kbits[c]);
        const int ks = h.kslot_base[cls] + kc[cls]++;
        kslot_of[c] = ks;
        perm[ks] = (uint16_t)c;
        if (cls == 3) {
            chan[2 * ks] = 1.0f;
        } else {
            chan[2 * ks] = kscale[c];
            chan[2 * ks + 1] = offset_of(kscale[c], kzero[c]);
            kz[ks] = kzero[c];
        }
    }
    // K rows per slot
    for (int i = 0; i < n; ++i) {
        uint8_t* row = tile + krow_offset(h, slot_of[i]);
        for (int c = 0; c < d; ++c) {
            const int ks = kslot_of[c];
            if (ks < 0) continue;
            const int cls = class_of_bits(kbits[c]);
            const int j = ks - h.kslot_base[cls];
            if (cls == 3) put_half(row + h.kbyte_base[3] + 2 * j, kfp[(size_t)i * d + c]);
            else put_bits(row + h.kbyte_base[cls], j, kBits(cls), kcodes[(size_t)c * n + i]);
        }
    }
    // V rows + parameters
    float* vp = reinterpret_cast<float*>(tile + h.off_vp);
    int64_t* vz = reinterpret_cast<int64_t*>(tile + h.off_vz);
    std::vector<uint8_t> packed;
    for (int i = 0; i < n; ++i) {
        const int cls = class_of_bits(vbits_kept[i]);
        const int li = slot_of[i] - slot_base(h, cls);
        if (cls == 3) {
            uint8_t* dst = tile + h.off_vseg[3] + (size_t)li * d * 2;
            for (int c = 0; c < d; ++c) put_half(dst + 2 * c, vfp[(size_t)i * d + c]);
            continue;
        }
        const int bits = kBits(cls), rb = ref_row_bytes(d, bits);
        packed.assign(rb, 0);
        for (int c = 0; c < d; ++c) put_bits(packed.data(), c, bits, vcodes[(size_t)i * d + c]);
        for (int m = 0; m < rb; ++m) tile[vbyte_offset(h, cls, li, m, d)] = packed[m];
        vp[2 * slot_of[i]] = vscale[i];
        vp[2 * slot_of[i] + 1] = offset_of(vscale[i], vzero[i]);
        vz[slot_of[i]] = vzero[i];
    }
    // scale bounds of the 2-bit class (same as the device packer)
    float km = 0.0f, vm = 0.0f;
    for (int j = 0; j < h.c[0]; ++j) km = std::max(km, std::fabs(chan[2 * (h.kslot_base[0] + j)]));
    for (int j = 0; j < h.r[0]; ++j) vm = std::max(vm, std::fabs(vp[2 * j]));
    reinterpret_cast<TileHeader*>(tile)->scale_bounds = bf16_bound_bits(km) | (bf16_bound_bits(vm) << 16);
    return RDKV_OK;
}

extern "C" RDKV_API const char* rdkv_status_string(int status) {
    switch (status) {
        case RDKV_OK: return "ok";
        case RDKV_EINVAL: return "invalid argument";
        case RDKV_ENUMERIC: return "numeric error";
        case RDKV_EFORMAT: return "format error";
        case RDKV_ECUDA: return "CUDA error";
        default: return "unknown status";
    }
}

extern "C" RDKV_API int rdkv_version(void) { return 1; }
