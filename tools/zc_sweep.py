"""tools: decode step time vs Zone C rows per tile (configs[2] headline shape), and the append
kernel alone — where the generation loop's time goes."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
if "--exp" in sys.argv:  # the EXPERIMENTS build (timing knobs), tools only
    sys.argv.remove("--exp")
    from paper_2605_08317_b200 import capi

    capi.LIB_PATH = os.path.join(ROOT, "paper_2605_08317_b200", "_lib_exp", "librdkv_b200.so")
import torch

import bench
from paper_2605_08317_b200 import pipeline as P
from paper_2605_08317_b200.workload import WorkloadSpec, build

spec = WorkloadSpec(batch=16, layers=32, ctx=131072, n_tokens=128)
model, _, _, _ = build(spec)
U, g, d = model.units, spec.group, spec.head_dim
q = P.generate((U, g, d), torch.float16, seed=bench.QSEED, tensor=2)
cap = 16
model.zc_cap, model.zc_count = cap, 0
model.zc_k = torch.zeros((U, cap, d), dtype=torch.float16, device="cuda")
model.zc_v = torch.zeros_like(model.zc_k)
model.zc_len = torch.zeros(U, dtype=torch.int32, device="cuda")
kn = P.generate((U, d), torch.float16, seed=77, tensor=1)
res = {"no_zone_c_us": None, "decode_us_by_rows": {}}
zl, zk = model.zc_len, model.zc_k
model.zc_len = None
res["no_zone_c_us"], _ = bench.graph_step_us(P, model, q, 100)
model.zc_len = zl
for rows in range(1, cap + 1):
    P.append_new_token(model, kn, kn)
    if rows in (1, 2, 4, 5, 8, 12, 16):
        us, _ = bench.graph_step_us(P, model, q, 100)
        res["decode_us_by_rows"][rows] = us
# the append kernel alone
model.zc_len.zero_()
model.zc_count = 0
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for i in range(cap):
    P.append_new_token(model, kn, kn)
e1.record()
torch.cuda.synchronize()
res["append_us"] = e0.elapsed_time(e1) / cap * 1e3
print(json.dumps(res), flush=True)
