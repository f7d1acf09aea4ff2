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


def test_exporter_rejects_bad_magic():
    tile = np.zeros(256, np.uint8)
    info = capi.TileInfo()
    assert capi.lib().rdkv_tile_info_get(tile.ctypes.data, C.byref(info)) == capi.RDKV_EFORMAT
    with pytest.raises(capi.RdkvError):
        export_tile(tile, 8)
