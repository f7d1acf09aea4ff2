"""numpy restatement of the device tile layout (paper_2605_08317_b200/csrc/tile_layout.h).

Builds the exact bytes the GPU packer must produce from a canonical
(reference-shaped) TriZone export — used to check the layout spec, the host
exporter (CPU tests) and the device packer byte-for-byte (GPU tests).
"""
from __future__ import annotations

import numpy as np

MAGIC = 0x31544452
HEADER = 128


def kbits(cls):
    return 2 << cls


def kpad(cls):
    return 32 if cls < 3 else 8


def pad4(x):
    return (x + 3) & ~3


def align(x, a):
    return (x + a - 1) // a * a


def ref_padded_len(n, bits):
    return (n + 3) // 4 * 4 if bits == 2 else (n + 1) // 2 * 2 if bits == 4 else n


def ref_row_bytes(n, bits):
    return ref_padded_len(n, bits) * bits // 8


def layout(r, c, d):
    h = {"r": list(r), "c": list(c)}
    n = sum(r)
    h["n"] = n
    slot = kbyte = 0
    kslot_base, kbyte_base = [], []
    for i in range(4):
        p = 0 if c[i] == 0 else (c[i] + kpad(i) - 1) // kpad(i) * kpad(i)
        kslot_base.append(slot)
        kbyte_base.append(kbyte)
        slot += p
        kbyte += p * kbits(i) // 8
    if n == 0:
        h["c"] = [0, 0, 0, 0]
        kslot_base = [0] * 4
        kbyte_base = [0] * 4
        slot = kbyte = 0
    h["kslots"] = slot
    h["krow_bytes"] = align(kbyte, 16)
    h["nslot"] = sum(pad4(x) for x in r)
    off = HEADER + 8 * slot
    off = align(off + 2 * slot, 16)
    h["off_k"] = off
    off = align(off + h["nslot"] * h["krow_bytes"], 16)
    h["off_vseg"] = []
    for i in range(3):
        h["off_vseg"].append(off)
        off = align(off + pad4(r[i]) * ref_row_bytes(d, kbits(i)), 16)
    h["off_vseg"].append(off)
    off = align(off + pad4(r[3]) * d * 2, 16)
    h["scale_bounds"] = 0
    h["off_vp"] = off
    off = align(off + 8 * h["nslot"], 16)
    h["off_ids"] = off
    off = align(off + 4 * h["nslot"], 16)
    h["off_vz"] = off
    off = align(off + 8 * h["nslot"], 16)
    h["off_kz"] = off
    off = align(off + 8 * slot, 128)
    h["total_bytes"] = off
    h["kslot_base"] = kslot_base
    h["kbyte_base"] = kbyte_base
    return h


def krow_pos(h, s):
    """Slot-transposed K row position (tile_layout.h krow_pos)."""
    return (s & 3) * (h["nslot"] >> 2) + (s >> 2)


def bf16_bound_bits(x):
    u = int(np.array([abs(x)], np.float32).view(np.uint32)[0])
    return (u >> 16) + (1 if u & 0xFFFF else 0)


def header_bytes(h):
    vals = [MAGIC, h["n"], *h["r"], *h["c"], h["kslots"], h["krow_bytes"], h["nslot"], h["off_k"],
            h["scale_bounds"], h["off_vp"], *h["off_vseg"], h["off_ids"], h["off_vz"], h["off_kz"],
            h["total_bytes"], *h["kslot_base"], *h["kbyte_base"]]
    return np.array(vals, dtype="<i8").astype("<u4").view(np.uint8)


def pack_codes(codes, bits):
    per = 8 // bits
    n = len(codes)
    out = np.zeros((n + per - 1) // per, np.uint8)
    for i, c in enumerate(codes):
        out[i // per] |= np.uint8(int(c) << ((i % per) * bits))
    return out


def offset_of(scale, zero):
    return np.float32(-np.float64(np.float32(scale)) * np.float64(zero))


def build_tile(canon, v_bits, k_bits, v_src, d):
    """canon: reference canonical export; v_bits [T], k_bits [d] (full allocation);
    v_src [T, d] float source values (for Zone B fp16 rows)."""
    kept = np.asarray(canon["kept"])
    n = len(kept)
    classes = {2: 0, 4: 1, 8: 2, 16: 3}
    r = [0, 0, 0, 0]
    for t in kept:
        r[classes[int(v_bits[t])]] += 1
    c = [0, 0, 0, 0]
    if n:
        for ch in range(d):
            b = int(k_bits[ch])
            if b in classes:
                c[classes[b]] += 1
    h = layout(r, c, d)
    tile = np.zeros(h["total_bytes"], np.uint8)
    tile[:HEADER] = header_bytes(h)
    kept_index = {int(t): i for i, t in enumerate(kept)}
    # slots
    slots = []  # token id per slot (-1 pad)
    for cls in range(4):
        members = [int(t) for t in kept if classes[int(v_bits[t])] == cls]
        slots += members + [-1] * (pad4(len(members)) - len(members))
    ids = np.array(slots, dtype="<i4")
    tile[h["off_ids"]:h["off_ids"] + 4 * len(ids)] = ids.view(np.uint8)
    # K slots
    kslots = h["kslots"]
    perm = np.zeros(kslots, "<u2")
    chan = np.zeros((kslots, 2), "<f4")
    kz = np.zeros(kslots, "<i8")
    if n:
        for cls in range(4):
            members = [ch for ch in range(d) if classes.get(int(k_bits[ch]), -1) == cls]
            for j, ch in enumerate(members):
                ks = h["kslot_base"][cls] + j
                perm[ks] = ch
                if cls == 3:
                    chan[ks] = (1.0, 0.0)
                else:
                    chan[ks] = (canon["kscale"][ch], offset_of(canon["kscale"][ch], canon["kzero"][ch]))
                    kz[ks] = canon["kzero"][ch]
    tile[HEADER:HEADER + 8 * kslots] = chan.reshape(-1).view(np.uint8)
    po = HEADER + 8 * kslots
    tile[po:po + 2 * kslots] = perm.view(np.uint8)
    tile[h["off_kz"]:h["off_kz"] + 8 * kslots] = kz.view(np.uint8)
    # K rows
    for sl, t in enumerate(slots):
        if t < 0:
            continue
        ki = kept_index[t]
        row = np.zeros(h["krow_bytes"], np.uint8)
        for cls in range(3):
            if h["c"][cls] == 0:
                continue
            pslots = (h["c"][cls] + 31) // 32 * 32
            codes = np.zeros(pslots, np.uint8)
            for j in range(h["c"][cls]):
                ch = perm[h["kslot_base"][cls] + j]
                codes[j] = canon["kcodes"][ch][ki]
            packed = pack_codes(codes, kbits(cls))
            row[h["kbyte_base"][cls]:h["kbyte_base"][cls] + len(packed)] = packed
        if h["c"][3]:
            vals = np.zeros(h["c"][3], np.float16)
            for j in range(h["c"][3]):
                ch = perm[h["kslot_base"][3] + j]
                vals[j] = np.float16(canon["kfp"][ki][ch])
            b0 = h["kbyte_base"][3]
            row[b0:b0 + 2 * len(vals)] = vals.view(np.uint8)
        o = h["off_k"] + krow_pos(h, sl) * h["krow_bytes"]
        tile[o:o + h["krow_bytes"]] = row
    # V rows + params
    vp = np.zeros((h["nslot"], 2), "<f4")
    vz = np.zeros(h["nslot"], "<i8")
    base = 0
    for cls in range(4):
        cnt = pad4(r[cls])
        for li in range(r[cls]):
            sl = base + li
            t = slots[sl]
            ki = kept_index[t]
            if cls == 3:
                o = h["off_vseg"][3] + li * d * 2
                tile[o:o + 2 * d] = v_src[t].astype(np.float16).view(np.uint8)
                continue
            bits = kbits(cls)
            packed = pack_codes(np.concatenate([canon["vcodes"][ki], np.zeros(ref_padded_len(d, bits) - d, np.uint8)]), bits)
            rb = ref_row_bytes(d, bits)
            grp = li >> 2
            for m in range(rb):
                col = (m ^ ((grp & 3) << 3)) if rb % 32 == 0 else m
                tile[h["off_vseg"][cls] + grp * 4 * rb + col * 4 + (li & 3)] = packed[m]
            vp[sl] = (canon["vscale"][ki], offset_of(canon["vscale"][ki], canon["vzero"][ki]))
            vz[sl] = canon["vzero"][ki]
        base += cnt
    tile[h["off_vp"]:h["off_vp"] + 8 * h["nslot"]] = vp.reshape(-1).view(np.uint8)
    tile[h["off_vz"]:h["off_vz"] + 8 * h["nslot"]] = vz.view(np.uint8)
    # scale bounds of the 2-bit class (bf16, rounded up): K channels low, V rows high
    km = max([abs(float(chan[h["kslot_base"][0] + j][0])) for j in range(h["c"][0])] or [0.0])
    vm = max([abs(float(vp[j][0])) for j in range(r[0])] or [0.0])
    h["scale_bounds"] = bf16_bound_bits(km) | (bf16_bound_bits(vm) << 16)
    tile[:HEADER] = header_bytes(h)
    return tile
