"""Rate sweep with duality bounds on the device (run_sweep, sweep.cpp:40-114; dual_bound,
allocator.cpp:218-246) against the reference's own rows (tests/golden/sweep.npz,
tests/golden/make_golden.py::make_sweep): primal, dual and feasibility bit-identical."""
import os

import numpy as np
import pytest
import torch

from paper_2605_08317_b200 import capi
from paper_2605_08317_b200 import pipeline as P

GOLD = np.load(os.path.join(os.path.dirname(__file__), "golden", "sweep.npz"))
NAMES = [str(n) for n in GOLD["names"]]


def device_caches(name):
    k, v, q = GOLD[f"k_{name}"], GOLD[f"v_{name}"], GOLD[f"q_{name}"]
    n, L, Hkv, T, d = k.shape
    Hq, Sw = q.shape[2], q.shape[3]
    g = Hq // Hkv
    return [P.DeviceCache(torch.from_numpy(k[i].reshape(L * Hkv, T, d)).cuda(),
                          torch.from_numpy(v[i].reshape(L * Hkv, T, d)).cuda(),
                          torch.from_numpy(q[i].reshape(L * Hkv, g, Sw, d)).cuda(), L, Hq, Hkv, Sw)
            for i in range(n)]


def test_sweep_validates_grid_on_host():
    cfg = P.default_config()
    with pytest.raises(capi.InvalidArgument):
        P.run_sweep([], [], cfg)
    with pytest.raises(capi.InvalidArgument):
        P.run_sweep([], [0.0], cfg)
    with pytest.raises(capi.InvalidArgument):
        P.run_sweep([], [16.5], cfg)


@pytest.mark.gpu
@pytest.mark.parametrize("name", NAMES)
def test_sweep_matches_reference(name):
    cfg = capi.Config.from_buffer_copy(GOLD[f"cfg_{name}"].tobytes())
    grid = GOLD[f"grid_{name}"].tolist()
    status = int(GOLD[f"status_{name}"])
    if status:
        with pytest.raises(capi.RdkvError) as e:
            P.run_sweep(device_caches(name), grid, cfg)
        assert e.value.code == status
        return
    rows = np.array([[s, b, p, du, float(f)] for s, b, p, du, f in P.run_sweep(device_caches(name), grid, cfg)])
    want = GOLD[f"rows_{name}"]
    assert rows.shape == want.shape
    assert rows.view(np.uint64).tolist() == want.view(np.uint64).tolist(), (rows, want)
    assert (rows[:, 3] <= rows[:, 2] + 1e-9).all()  # weak duality: g(lambda) <= primal
