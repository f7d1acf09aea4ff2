"""RDKVC001 cache containers straight to device (load_cache, cache.cpp:228-287).

tests/golden/cache_io.npz holds a container written by the reference's save_cache_file and
byte-level variants of it, each with the status and dims the reference's load_cache_file
returned for it (tests/golden/make_golden.py::make_cache_io). The header check runs on the
host (no GPU); the payload load runs on the device (gpu-marked).
"""
import os
import struct

import numpy as np
import pytest
import torch

from paper_2605_08317_b200 import capi
from paper_2605_08317_b200 import pipeline as P

GOLD = np.load(os.path.join(os.path.dirname(__file__), "golden", "cache_io.npz"))
NAMES = [str(n) for n in GOLD["names"]]


def write(tmp_path, name):
    p = tmp_path / f"{name}.rdkvc"
    p.write_bytes(GOLD[f"bytes_{name}"].tobytes())
    return str(p)


def payload(name):
    data = GOLD[f"bytes_{name}"].tobytes()
    hlen = struct.unpack("<I", data[8:12])[0]
    return np.frombuffer(data[12 + hlen:], np.float32)


@pytest.mark.parametrize("name", NAMES)
def test_header_status_matches_reference(tmp_path, name):
    path = write(tmp_path, name)
    ref_status = int(GOLD[f"status_{name}"])
    expect = 0 if ref_status == capi.RDKV_ENUMERIC else ref_status  # finiteness is a payload check
    h = capi.CacheHeader()
    assert capi.lib().rdkv_cache_read_header(path.encode(), h) == expect
    if expect == 0:
        dims = [h.layers, h.q_heads, h.kv_heads, h.head_dim, h.seq_len, h.probe_window]
        if ref_status == 0:
            assert dims == list(GOLD[f"dims_{name}"])
        data = GOLD[f"bytes_{name}"]
        assert h.payload_offset + h.payload_bytes == data.size


def test_header_errors_raise_reference_exception_types(tmp_path):
    with pytest.raises(capi.FormatError):
        P.read_cache_header(write(tmp_path, "bad_magic"))
    with pytest.raises(capi.InvalidArgument):
        P.read_cache_header(write(tmp_path, "q_not_multiple"))
    with pytest.raises(capi.FormatError):
        P.read_cache_header(str(tmp_path / "does_not_exist.rdkvc"))


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["ok", "pretty_extra_keys", "float_dim", "fp16_overflow"])
def test_load_to_device_f32_bit_exact(tmp_path, name):
    c = P.load_cache_file(write(tmp_path, name), dtype=torch.float32)
    L, Hq, Hkv, d, T, Sw = (int(x) for x in GOLD[f"dims_{name}"])
    U, g = L * Hkv, Hq // Hkv
    got = np.concatenate([c.k.cpu().numpy().ravel(), c.v.cpu().numpy().ravel(), c.probe_q.cpu().numpy().ravel()])
    want = payload(name)
    assert got.view(np.uint32).tolist() == want.view(np.uint32).tolist()
    assert c.k.shape == (U, T, d) and c.probe_q.shape == (U, g, Sw, d) and c.group == g


@pytest.mark.gpu
def test_load_to_device_f16_rounds_like_numpy(tmp_path):
    c = P.load_cache_file(write(tmp_path, "ok"), dtype=torch.float16)
    got = np.concatenate([c.k.cpu().numpy().ravel(), c.v.cpu().numpy().ravel(), c.probe_q.cpu().numpy().ravel()])
    want = payload("ok").astype(np.float16)
    assert got.view(np.uint16).tolist() == want.view(np.uint16).tolist()


@pytest.mark.gpu
@pytest.mark.parametrize("name,dtype", [("nan_in_v", torch.float32), ("inf_in_q", torch.float16),
                                        ("fp16_overflow", torch.float16)])
def test_load_rejects_non_finite(tmp_path, name, dtype):
    with pytest.raises(capi.NumericError):
        P.load_cache_file(write(tmp_path, name), dtype=dtype)


@pytest.mark.gpu
def test_loaded_cache_feeds_the_pipeline(tmp_path):
    """A loaded container runs allocate -> pack like a generated one (shape plumbing)."""
    c = P.load_cache_file(write(tmp_path, "ok"), dtype=torch.float32)
    cfg = P.default_config(n_tokens=8, window=4)
    alloc = P.allocate_model(c.k, c.probe_q, cfg, kv_heads=c.kv_heads)
    alloc.check()
    m = P.build_packed_model(c.k, c.v, alloc, group=c.group)
    m.check()
    q = torch.randn((c.k.shape[0], c.group, c.k.shape[2]), dtype=torch.float32, device="cuda")
    out = P.packed_decode_step(m, q)
    assert torch.isfinite(out).all()
