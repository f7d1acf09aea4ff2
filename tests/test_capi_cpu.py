"""CPU-side checks of the native library (no GPU needed):
- the .so loads and exports every RDKV_API symbol declared in include/rdkv_cuda.h;
- the device tile layout spec (tests/tilepack.py, a numpy restatement of
  csrc/tile_layout.h) round-trips through the host exporter back to the
  reference's canonical TriZone view for every golden case.
"""
import ctypes as C

import numpy as np
import pytest

import tilepack
from paper_2605_08317_b200 import capi
from paper_2605_08317_b200.pipeline import export_tile


def test_library_exports_every_declared_symbol():
    L = capi.lib()
    names = capi.declared_symbols()
    assert len(names) >= 15
    missing = [n for n in names if not hasattr(L, n)]
    assert not missing, missing
    assert L.rdkv_version() == 1
    assert L.rdkv_status_string(2) == b"numeric error"


def test_struct_layouts_match_oracle():
    import oracle

    assert C.sizeof(capi.Config) == C.sizeof(oracle.Config)
    for (a, _), (b, _) in zip(capi.Config._fields_, oracle.Config._fields_):
        assert a == b and getattr(capi.Config, a).offset == getattr(oracle.Config, b).offset
    assert C.sizeof(capi.HeadStats) == 80  # 7 doubles + 6 int32


def test_layout_kat():
    # 128 kept tokens at 2 bits, 128 channels at 2 bits, d=128 (C1/C3 observed allocation)
    h = tilepack.layout([128, 0, 0, 0], [128, 0, 0, 0], 128)
    assert h["kslots"] == 128 and h["krow_bytes"] == 32 and h["nslot"] == 128
    # decode region = header + chan table + perm + K rows + V rows + V params
    assert h["off_ids"] == 128 + 1024 + 256 + 128 * 32 + 128 * 32 + 128 * 8


def _golden_cases(golden):
    g = golden("trizone.npz")
    for i in range(int(g["n"])):
        canon = {k[len(f"t{i}_tz_"):]: g[k] for k in g if k.startswith(f"t{i}_tz_")}
        yield f"t{i}", g[f"t{i}_k"], g[f"t{i}_v"], g[f"t{i}_v_bits"], g[f"t{i}_k_bits"], canon
    a = golden("alloc.npz")
    for i in range(int(a["n"])):
        canon = {k[len(f"c{i}_tz_"):]: a[k] for k in a if k.startswith(f"c{i}_tz_")}
        kb = a[f"c{i}_k_bits"]
        d = a[f"c{i}_k"].shape[1]
        if kb.size == 0:
            kb = np.zeros(d, np.int32)
        yield f"c{i}", a[f"c{i}_k"], a[f"c{i}_v"], a[f"c{i}_v_bits"], kb, canon


def test_tile_spec_roundtrips_through_exporter(golden):
    for name, k, v, vb, kb, canon in _golden_cases(golden):
        d = k.shape[1]
        tile = tilepack.build_tile(canon, vb, kb, v, d)
        got = export_tile(tile, d)
        for key in ("kept", "vcodes", "vscale", "vzero", "kcodes", "kscale", "kzero", "payload",
                    "segtab", "perm"):
            want = np.asarray(canon[key])
            assert np.array_equal(np.asarray(got[key]).reshape(want.shape), want), (name, key)
        # fp zones: the device stores fp16; golden cases are f32 -> compare at fp16
        vfp = np.asarray(canon["vfp"]).astype(np.float16).astype(np.float32)
        kfp = np.asarray(canon["kfp"]).astype(np.float16).astype(np.float32)
        assert np.array_equal(got["vfp"].reshape(vfp.shape), vfp), name
        assert np.array_equal(got["kfp"].reshape(kfp.shape), kfp), name
        assert int(got["info"].total_bytes) == len(tile)


def test_import_is_inverse_of_export(golden):
    """rdkv_tile_import(canonical view) rebuilds the tile byte-for-byte."""
    from paper_2605_08317_b200.pipeline import import_tile

    for name, k, v, vb, kb, canon in _golden_cases(golden):
        d = k.shape[1]
        tile = tilepack.build_tile(canon, vb, kb, v, d)
        got = export_tile(tile, d)
        kept = np.asarray(got["kept"])
        back = import_tile(d, kept, np.asarray(vb)[kept], got["vcodes"], got["vscale"], got["vzero"], got["vfp"],
                           np.asarray(kb) if len(kept) else np.zeros(d), got["kcodes"], got["kscale"],
                           got["kzero"], got["kfp"])
        assert np.array_equal(back, tile), name


def test_import_rejects_bad_input():
    from paper_2605_08317_b200.pipeline import import_tile

    d = 4
    with pytest.raises(capi.InvalidArgument):  # kept not ascending
        import_tile(d, [3, 1], [2, 2], np.zeros((2, d)), [1, 1], [0, 0], np.zeros((2, d)), [2] * d,
                    np.zeros((d, 2)), [1] * d, [0] * d, np.zeros((2, d)))
    with pytest.raises(capi.InvalidArgument):  # 3-bit width
        import_tile(d, [1], [3], np.zeros((1, d)), [1], [0], np.zeros((1, d)), [2] * d,
                    np.zeros((d, 1)), [1] * d, [0] * d, np.zeros((1, d)))


def test_exporter_rejects_bad_magic():
    tile = np.zeros(256, np.uint8)
    info = capi.TileInfo()
    assert capi.lib().rdkv_tile_info_get(tile.ctypes.data, C.byref(info)) == capi.RDKV_EFORMAT
    with pytest.raises(capi.RdkvError):
        export_tile(tile, 8)


def test_cpp_dropin_library_is_self_contained():
    """librdkv_cuda_dropin.so defines the rdkv::cuda API and needs no reference
    symbol (it only uses the reference's header types)."""
    import os
    import subprocess

    so = os.path.join(os.path.dirname(capi.LIB_PATH), "librdkv_cuda_dropin.so")
    if not os.path.exists(so):
        pytest.skip("drop-in not built (needs the reference headers at build time)")
    out = subprocess.run(["nm", "-DC", so], capture_output=True, text=True, check=True).stdout
    undefined = [l for l in out.splitlines() if " U " in l and "rdkv::" in l]
    assert not undefined, undefined
    for fn in ("rdkv::cuda::allocate_model(", "rdkv::cuda::build_packed_model(", "rdkv::cuda::packed_decode_step(",
               "rdkv::cuda::mckp_bisect(", "rdkv::cuda::attention_probe(", "rdkv::cuda::build_trizone(",
               "rdkv::cuda::fused_k_logits(", "rdkv::cuda::DevicePackedModel::decode("):
        assert any(fn in l and " T " in l for l in out.splitlines()), fn
