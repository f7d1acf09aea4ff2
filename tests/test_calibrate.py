"""ε calibration on the device (calibrate_epsilon, quantizer.cpp:200-284) against the
reference's own tables (tests/golden/calib.npz, tests/golden/make_golden.py::make_calib):
eps values and unit counts bit-identical, error statuses as the reference's exceptions."""
import os

import numpy as np
import pytest
import torch

from paper_2605_08317_b200 import capi
from paper_2605_08317_b200 import pipeline as P

GOLD = np.load(os.path.join(os.path.dirname(__file__), "golden", "calib.npz"))
NAMES = [str(n) for n in GOLD["names"]]


def test_finalize_host_rules():
    """The host merge: eps(0)=1, eps(16)=0, job-order sums, DistortionTable::validate."""
    L = capi.lib()
    w = np.array([0, 2, 4, 16], np.int32)
    err = np.array([[0.5, 0.02], [0.25, 0.01]], np.float64)
    cnt = np.array([3, 2], np.int64)
    eps = np.zeros(4)
    units = np.zeros(1, np.int64)
    assert L.rdkv_calibrate_finalize(err.ctypes.data, cnt.ctypes.data, 2, w.ctypes.data, 4, eps.ctypes.data,
                                     units.ctypes.data) == 0
    assert eps.tolist() == [1.0, (0.5 + 0.25) / 5, (0.02 + 0.01) / 5, 0.0] and units[0] == 5
    cnt0 = np.zeros(2, np.int64)
    assert L.rdkv_calibrate_finalize(err.ctypes.data, cnt0.ctypes.data, 2, w.ctypes.data, 4, eps.ctypes.data,
                                     None) == capi.RDKV_ENUMERIC
    flat = np.array([[0.5, 0.5], [0.5, 0.5]], np.float64)  # eps(2) == eps(4): not strictly decreasing
    assert L.rdkv_calibrate_finalize(flat.ctypes.data, cnt.ctypes.data, 2, w.ctypes.data, 4, eps.ctypes.data,
                                     None) == capi.RDKV_EINVAL
    bad = np.array([0, 3, 16], np.int32)
    assert L.rdkv_calibrate_finalize(err.ctypes.data, cnt.ctypes.data, 2, bad.ctypes.data, 3, eps.ctypes.data,
                                     None) == capi.RDKV_EINVAL


@pytest.mark.gpu
@pytest.mark.parametrize("gran", [0, 1], ids=["token", "channel"])
@pytest.mark.parametrize("name", NAMES)
def test_calibrate_matches_reference(name, gran):
    k, v = GOLD[f"k_{name}"], GOLD[f"v_{name}"]  # [n][L][H_kv][T][d]
    widths = GOLD[f"widths_{name}"].tolist()
    n, L, Hkv, T, d = k.shape
    caches = [(torch.from_numpy(k[i].reshape(L * Hkv, T, d)).cuda(),
               torch.from_numpy(v[i].reshape(L * Hkv, T, d)).cuda()) for i in range(n)]
    status = int(GOLD[f"status_{name}_{gran}"])
    if status:
        with pytest.raises(capi.RdkvError) as e:
            P.calibrate_epsilon(caches, gran, widths)
        assert e.value.code == status
        return
    eps, units = P.calibrate_epsilon(caches, gran, widths)
    want = GOLD[f"eps_{name}_{gran}"]
    assert units == int(GOLD[f"units_{name}_{gran}"])
    got = np.array([eps[b] for b in widths], np.float64)
    assert got.view(np.uint64).tolist() == want.view(np.uint64).tolist(), (got, want)


@pytest.mark.gpu
def test_calibrate_fp16_storage_matches_f32():
    """fp16 device caches of FP16-representable values calibrate to the same table."""
    k, v = GOLD["k_fp16_values"], GOLD["v_fp16_values"]
    n, L, Hkv, T, d = k.shape
    f32 = [(torch.from_numpy(k[0].reshape(L * Hkv, T, d)).cuda(), torch.from_numpy(v[0].reshape(L * Hkv, T, d)).cuda())]
    f16 = [(a.half(), b.half()) for a, b in f32]
    for gran in (0, 1):
        assert P.calibrate_epsilon(f16, gran) == P.calibrate_epsilon(f32, gran)


@pytest.mark.gpu
def test_calibrate_generated_cache_runs_at_scale():
    """A C1-shaped generated cache (1 layer x 8 KV heads x 4096 x 128): the table is valid
    (eps strictly decreasing) and the counts cover every unit."""
    k = P.generate((8, 4096, 128), torch.float16, seed=3, tensor=0)
    v = P.generate((8, 4096, 128), torch.float16, seed=3, tensor=1)
    eps_t, n_t = P.calibrate_epsilon([(k, v)], "token")
    eps_c, n_c = P.calibrate_epsilon([(k, v)], "channel")
    assert n_t == 8 * 4096 and n_c == 8 * 128
    assert eps_t[0] == 1.0 and eps_t[16] == 0.0 and 1 > eps_t[2] > eps_t[4] > eps_t[8] > 0
