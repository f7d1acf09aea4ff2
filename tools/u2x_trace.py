"""tools: timeline of one headline decode launch (EXPERIMENTS build): per warp
pair the globaltimer at entry, after griddepcontrol.wait, and per tile the
buffer wait and the tile end, for the last of K back-to-back graph launches.
usage: python tools/u2x_trace.py [K] [--host]   (--host: one end-to-end step through
rdkv_cuda_decode_host with pinned host q / out instead of the device graph)"""
import ctypes as C
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2605_08317_b200 import capi

capi.LIB_PATH = os.path.join(ROOT, "paper_2605_08317_b200", "_lib_exp", "librdkv_b200.so")
import numpy as np
import torch

from paper_2605_08317_b200 import pipeline as P
from paper_2605_08317_b200.workload import WorkloadSpec, build

import bench

HOST = "--host" in sys.argv
if HOST:
    sys.argv.remove("--host")
K = int(sys.argv[1]) if len(sys.argv) > 1 else 50
spec = WorkloadSpec(batch=16, layers=32, ctx=131072, n_tokens=128)
model, _, _, _ = build(spec)
q = P.generate((model.units, spec.group, spec.head_dim), torch.float16, seed=bench.QSEED, tensor=2)
S = 20
buf = torch.zeros(1024 * 16 * S, dtype=torch.int64, device="cuda")
lib = capi.lib()
lib.rdkv_exp_set_u2x_trace.argtypes = [C.c_void_p]
assert lib.rdkv_exp_set_u2x_trace(buf.data_ptr()) == 0
if HOST:
    qh = q.cpu().pin_memory()
    oh = torch.empty_like(qh).pin_memory()
    out = torch.empty_like(q)
    args_c = P.decode_args(model, q, out)
    st = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for _ in range(K):
        e0.record(st)
        assert lib.rdkv_cuda_decode_host(C.byref(args_c), qh.data_ptr(), oh.data_ptr(), st.cuda_stream) == 0
        e1.record(st)
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1e3
else:
    us, _ = bench.graph_step_us(P, model, q, K)
torch.cuda.synchronize()
t = buf.cpu().numpy().reshape(-1, S)
t = t[t[:, 0] > 0]
sm = t[:, 19]
t0 = t[:, 0].min()
ev = (t[:, :19] - t0).astype(np.float64) / 1e3  # us
ev[t[:, :19] == 0] = np.nan
entry, waited = ev[:, 0], ev[:, 1]
tw, te = ev[:, 2:18:2], ev[:, 3:19:2]
ntiles = np.sum(~np.isnan(te), axis=1)
end = np.nanmax(te, axis=1)
out = {"us_per_step_graph": us, "pairs": int(len(t)),
       "entry_us": [float(np.nanmin(entry)), float(np.nanpercentile(entry, 50)), float(np.nanmax(entry))],
       "after_wait_us": [float(np.nanmin(waited)), float(np.nanpercentile(waited, 50)), float(np.nanmax(waited))],
       "first_tile_ready_us": [float(np.nanmin(tw[:, 0])), float(np.nanpercentile(tw[:, 0], 50)), float(np.nanmax(tw[:, 0]))],
       "tiles_per_pair": {str(int(k)): int(v) for k, v in zip(*np.unique(ntiles, return_counts=True))},
       "end_us": [float(np.nanmin(end)), float(np.nanpercentile(end, 50)), float(np.nanmax(end))]}
rounds = []
for k in range(8):
    d = te[:, k] - tw[:, k]
    w = tw[:, k] - (te[:, k - 1] if k else waited)
    if np.all(np.isnan(d)):
        break
    rounds.append({"round": k, "pairs": int(np.sum(~np.isnan(d))), "tile_us_median": float(np.nanmedian(d)),
                   "tile_us_p90": float(np.nanpercentile(d, 90)), "wait_before_us_median": float(np.nanmedian(w)),
                   "end_us_median": float(np.nanmedian(te[:, k])), "end_us_max": float(np.nanmax(te[:, k]))})
out["rounds"] = rounds
# active pairs over time
grid = np.arange(0, float(np.nanmax(end)) + 0.25, 0.25)
act = [int(np.sum((waited <= x) & (end > x))) for x in grid]
out["active_pairs_every_0.25us"] = act
print(json.dumps(out), flush=True)
