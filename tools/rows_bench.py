"""Timing of the §8(f) rows on one B200 vs the reference CPU (oracle/_ref) on the same inputs:
RDKVC001 load, epsilon calibration, rate sweep. Writes gpurun_out/rows_bench.json.
(scratch tool; the reference CPU side is the test-infrastructure build of the unmodified
reference, used here only as the timing baseline.)"""
import json
import os
import sys
import tempfile
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
from paper_2605_08317_b200 import pipeline as P  # noqa: E402

ref = oracle.load_ref()
out = {"cpu_threads": ref.lib.ref_worker_count(), "cpu": os.cpu_count()}


def gpu_time(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    return float(np.median(ts))


# C1 shape: 1 layer, 32 q heads, 8 KV heads, d 128, T 4096, S_w 32
L, Hq, Hkv, d, T, Sw = 1, 32, 8, 128, 4096, 32
k, v, q = ref.gen_synthetic(1, L, Hq, Hkv, d, T, Sw)
cache = P.DeviceCache(torch.from_numpy(k.reshape(L * Hkv, T, d)).cuda(), torch.from_numpy(v.reshape(L * Hkv, T, d)).cuda(),
                      torch.from_numpy(q.reshape(L * Hkv, Hq // Hkv, Sw, d)).cuda(), L, Hq, Hkv, Sw)

# calibration
for gran, name in ((0, "token"), (1, "channel")):
    t0 = time.perf_counter()
    eps_r, units_r = ref.calibrate(k[None], v[None], q[None], gran, [0, 2, 4, 8, 16])
    t_ref = time.perf_counter() - t0
    eps_d, units_d = P.calibrate_epsilon([cache], gran)
    same = [eps_d[b] for b in (0, 2, 4, 8, 16)] == eps_r.tolist() and units_d == units_r
    t_dev = gpu_time(lambda: P.calibrate_epsilon([cache], gran))
    out[f"calibrate_{name}_c1"] = {"ref_s": t_ref, "b200_s": t_dev, "speedup": t_ref / t_dev, "bit_identical": same,
                                   "units": units_d}

# rate sweep
grid = [0.25, 0.5, 1.0, 2.0, 4.0, 8.0]
cfg = P.default_config()
t0 = time.perf_counter()
rows_r = ref.run_sweep(k[None], v[None], q[None], grid, cfg)
t_ref = time.perf_counter() - t0
rows_d = np.array([[s, b, p, du, float(f)] for s, b, p, du, f in P.run_sweep([cache], grid, cfg)])
t_dev = gpu_time(lambda: P.run_sweep([cache], grid, cfg), reps=3)
out["run_sweep_c1_6pts"] = {"ref_s": t_ref, "b200_s": t_dev, "speedup": t_ref / t_dev,
                            "bit_identical": rows_d.view(np.uint64).tolist() == rows_r.view(np.uint64).tolist()}

# RDKVC001 load
tmp = tempfile.mkdtemp()
path = os.path.join(tmp, "c1.rdkvc")
ref.save_cache(1, L, Hq, Hkv, d, T, Sw, path)
size = os.path.getsize(path)
t0 = time.perf_counter()
st, _ = ref.load_cache_status(path)
t_ref = time.perf_counter() - t0
t_dev = gpu_time(lambda: P.load_cache_file(path, dtype=torch.float16))
out["cache_load_c1"] = {"bytes": size, "ref_s": t_ref, "b200_s": t_dev, "b200_GBps": size / t_dev / 1e9,
                        "ref_GBps": size / t_ref / 1e9, "note": "page-cache warm file; device side includes fp16 conversion + finiteness"}

# device-only at C2 scale (32 layers x 8 KV heads x 32K x 128, fp16 generated)
U2, T2 = 256, 32768
k2 = P.generate((U2, T2, d), torch.float16, seed=2, tensor=0)
v2 = P.generate((U2, T2, d), torch.float16, seed=2, tensor=1)
for gran, name in ((0, "token"), (1, "channel")):
    t = gpu_time(lambda: P.calibrate_epsilon([(k2, v2)], gran), reps=3)
    out[f"calibrate_{name}_c2_b200_s"] = t
print(json.dumps(out, indent=1))
os.makedirs("gpurun_out", exist_ok=True)
json.dump(out, open("gpurun_out/rows_bench.json", "w"), indent=1)
