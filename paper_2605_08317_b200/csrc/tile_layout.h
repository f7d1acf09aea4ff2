// tile_layout.h — device layout of one packed TriZone tile (one
// (batch, layer, KV head)), shared by the packer, the decode kernels and the
// host exporter. Host/device neutral (no CUDA headers).
//
// The reference keeps Zone A as per-bit-width PackedSegments of V rows and K
// rows (trizone.hpp:34-78). The device tile keeps the same codes and
// quantisation parameters but orders them for the decode kernel:
//
//   * token slots: V classes 2,4,8,16 bits in that order, ascending token id
//     inside a class (the reference segment order, trizone.cpp:126-157),
//     each class padded to a multiple of 4 slots;
//   * K rows are stored per SLOT (row i = K of the token in slot i), so the
//     `positions` indirection of the reference decode (trizone.cpp:282)
//     disappears and QK/PV walk the same slot order; K channels are grouped
//     2,4,8,16 bits (channel_perm order, trizone.cpp:201-206) and each group
//     is padded to 32 channels (pad slots carry scale = offset = 0, so pad
//     codes can never leak — trizone.cpp:214-232 semantics);
//   * quantised V rows are interleaved in groups of 4 tokens at byte
//     granularity (byte m of tokens 4G..4G+3 are adjacent), so one 32-bit
//     word holds 4 tokens x (8/bits) channels — the operand shape of the
//     int8 tensor-core PV product; word columns are XOR-swizzled per group
//     (vswz) for bank-conflict-free fragment loads;
//   * dequantisation is stored as (scale, offset = -scale*zero_point) in f32;
//     the int64 zero points and token ids live in an export trailer that the
//     decode never reads.
//
// Byte map (offsets from the 128-B aligned tile start):
//   [0,128)            TileHeader
//   [128, +8*kslots)   per K slot float2 {scale, offset}
//   [.., +2*kslots)    per K slot uint16 channel id (16-B padded)
//   off_k              nslot K rows x krow_bytes, slot-transposed (krow_pos):
//                        [P2/4 B 2-bit][P4/2 B 4-bit][P8 B 8-bit][2*P16 B fp16]
//   off_vseg[0..2]     V classes 2/4/8: (slots/4) groups x 4*rb(bits)
//   off_vseg[3]        V class 16: slots x d fp16, row-major
//   off_vp             per slot float2 {scale, offset}
//   off_ids            per slot int32 token id (-1 for pad slots)   [export]
//   off_vz             per slot int64 zero point                     [export]
//   off_kz             per K slot int64 zero point                   [export]
#pragma once

#include <stdint.h>

#ifdef __CUDACC__
#define RDKV_HD __host__ __device__ __forceinline__
#else
#define RDKV_HD inline
#endif

namespace rdkv_b200 {

constexpr int32_t kTileMagic = 0x31544452;  // "RDT1"
constexpr int kTileAlign = 128;
constexpr int kHeaderBytes = 128;

struct TileHeader {
    int32_t magic;
    int32_t n;           // kept tokens
    int32_t r[4];        // V rows per class (2,4,8,16)
    int32_t c[4];        // K channels per class (2,4,8,16)
    int32_t kslots;      // K slots (padded channel count)
    int32_t krow_bytes;  // bytes per K row
    int32_t nslot;       // token slots
    int32_t off_k;
    uint32_t scale_bounds;  // bf16 upper bounds: lo = max K scale (2-bit channels), hi = max V scale (2-bit rows)
    int32_t off_vp;
    int32_t off_vseg[4];
    int32_t off_ids;
    int32_t off_vz;
    int32_t off_kz;
    int32_t total_bytes;
    int32_t kslot_base[4];  // first K slot of each class
    int32_t kbyte_base[4];  // byte offset of each class inside a K row
};
static_assert(sizeof(TileHeader) == kHeaderBytes, "header is 128 bytes");

// bit-width of class i (2,4,8,16) and the K-slot padding of each class
RDKV_HD int kBits(int cls) { return 2 << cls; }
RDKV_HD int kKPad(int cls) { return cls < 3 ? 32 : 8; }

RDKV_HD int32_t align_up(int64_t x, int64_t a) { return (int32_t)((x + a - 1) / a * a); }
RDKV_HD int32_t pad4(int32_t x) { return (x + 3) & ~3; }
// reference packed_row_bytes (trizone.cpp:48-57)
RDKV_HD int32_t ref_padded_len(int32_t len, int32_t bits) {
    return bits == 2 ? (len + 3) / 4 * 4 : bits == 4 ? (len + 1) / 2 * 2 : len;
}
RDKV_HD int32_t ref_row_bytes(int32_t len, int32_t bits) {
    return ref_padded_len(len, bits) * bits / 8;
}
RDKV_HD int class_of_bits(int bits) {
    return bits == 2 ? 0 : bits == 4 ? 1 : bits == 8 ? 2 : bits == 16 ? 3 : -1;
}

// Fills every derived field of the header from n, r[], c[] and d.
RDKV_HD void tile_layout(TileHeader& h, int32_t d) {
    h.magic = kTileMagic;
    h.n = h.r[0] + h.r[1] + h.r[2] + h.r[3];
    int32_t slot = 0, kbyte = 0;
    for (int i = 0; i < 4; ++i) {
        int32_t p = h.c[i] == 0 ? 0 : (h.c[i] + kKPad(i) - 1) / kKPad(i) * kKPad(i);
        h.kslot_base[i] = slot;
        h.kbyte_base[i] = kbyte;
        slot += p;
        kbyte += p * kBits(i) / 8;
    }
    if (h.n == 0) {  // build_trizone: every token evicted -> no K storage (trizone.cpp:113-118)
        for (int i = 0; i < 4; ++i) {
            h.c[i] = 0;
            h.kslot_base[i] = 0;
            h.kbyte_base[i] = 0;
        }
        slot = 0;
        kbyte = 0;
    }
    h.kslots = slot;
    h.krow_bytes = align_up(kbyte, 16);
    h.nslot = pad4(h.r[0]) + pad4(h.r[1]) + pad4(h.r[2]) + pad4(h.r[3]);
    int64_t off = kHeaderBytes;
    off += (int64_t)8 * h.kslots;
    off = align_up(off + (int64_t)2 * h.kslots, 16);
    h.off_k = (int32_t)off;
    off = align_up(off + (int64_t)h.nslot * h.krow_bytes, 16);
    for (int i = 0; i < 3; ++i) {
        h.off_vseg[i] = (int32_t)off;
        off = align_up(off + (int64_t)pad4(h.r[i]) * ref_row_bytes(d, kBits(i)), 16);
    }
    h.off_vseg[3] = (int32_t)off;
    off = align_up(off + (int64_t)pad4(h.r[3]) * d * 2, 16);
    h.scale_bounds = 0;  // filled by the packer once the scales are known
    h.off_vp = (int32_t)off;
    off = align_up(off + (int64_t)8 * h.nslot, 16);
    h.off_ids = (int32_t)off;
    off = align_up(off + (int64_t)4 * h.nslot, 16);
    h.off_vz = (int32_t)off;
    off = align_up(off + (int64_t)8 * h.nslot, 16);
    h.off_kz = (int32_t)off;
    off = align_up(off + (int64_t)8 * h.kslots, kTileAlign);
    h.total_bytes = (int32_t)off;
}

RDKV_HD int32_t chan_table_off() { return kHeaderBytes; }

// K rows are stored slot-transposed: the row of token slot s sits at position
// (s & 3) * (nslot / 4) + (s >> 2). A tensor-core lane that owns the four
// consecutive slots 4j..4j+3 (so its softmax weights pack into one 32-bit
// word per digit) then reads K rows that are 32 B apart across the lanes of a
// quarter-warp instead of 128 B apart (bank-conflict-free LDS.128).
RDKV_HD int32_t krow_pos(const TileHeader& h, int32_t s) { return (s & 3) * (h.nslot >> 2) + (s >> 2); }
RDKV_HD int64_t krow_offset(const TileHeader& h, int32_t s) {
    return (int64_t)h.off_k + (int64_t)krow_pos(h, s) * h.krow_bytes;
}

// bf16 bit pattern of a non-negative float, rounded up (an upper bound).
RDKV_HD uint32_t bf16_bound_bits(float x) {
    union { float f; uint32_t u; } v;
    v.f = x;
    return (v.u & 0xFFFFu) ? (v.u >> 16) + 1u : (v.u >> 16);
}
RDKV_HD float bf16_bits_to_float(uint32_t b) {
    union { float f; uint32_t u; } v;
    v.u = b << 16;
    return v.f;
}
RDKV_HD int32_t perm_off(const TileHeader& h) { return kHeaderBytes + 8 * h.kslots; }

// First slot of V class i.
RDKV_HD int32_t slot_base(const TileHeader& h, int i) {
    int32_t s = 0;
    for (int j = 0; j < i; ++j) s += pad4(h.r[j]);
    return s;
}

// Bytes the decode kernel reads from a tile (the roofline numerator): header,
// channel table + ids, K rows, V rows and V params. The export trailer
// (token ids, int64 zero points) is never read on device.
RDKV_HD int64_t tile_decode_bytes(const TileHeader& h) {
    return (int64_t)h.off_ids - 0;  // everything before the export trailer
}

// Byte column swizzle of the interleaved V layout: inside token group G the
// 32-bit word of byte column m is stored at column m ^ (8 * (G & 3)) whenever
// a row spans a multiple of 32 bytes, so the four token groups a tensor-core
// fragment reads at once fall into distinct shared-memory banks.
RDKV_HD int32_t vswz(int32_t m, int32_t grp, int32_t rb) {
    return (rb & 31) == 0 ? (m ^ ((grp & 3) << 3)) : m;
}

// Location of the packed byte `byte_in_row` of slot li (local index in class
// cls) in the 4-token interleaved V layout.
RDKV_HD int64_t vbyte_offset(const TileHeader& h, int cls, int32_t li, int32_t byte_in_row,
                             int32_t d) {
    const int32_t rb = ref_row_bytes(d, kBits(cls));
    const int32_t grp = li >> 2;
    return (int64_t)h.off_vseg[cls] + (int64_t)grp * 4 * rb + (int64_t)vswz(byte_in_row, grp, rb) * 4 +
           (li & 3);
}

}  // namespace rdkv_b200
