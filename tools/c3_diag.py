"""tools: why a configs[3] arena is (not) on the mixed 2/4-bit chunked kernel: per-tile class
maxima; then a few decode steps (for ncu -k regex:u24)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2605_08317_b200 import pipeline as P
from paper_2605_08317_b200.workload import WorkloadSpec, build

name = sys.argv[1] if len(sys.argv) > 1 else "qwen"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 256
L, Hq, Hkv = {"qwen": (28, 28, 4), "mistral": (32, 32, 8)}[name]
spec = WorkloadSpec(batch=4, layers=L, q_heads=Hq, kv_heads=Hkv, ctx=65536, n_tokens=n, seed=11,
                    hh_stride=64, hh_boost=1.0, outlier_channels=4, outlier_scale=8.0)
m, _, _, _ = build(spec)
infos = m.infos()
rows = np.array([[int(x) for x in i.rows] for i in infos])
chans = np.array([[int(x) for x in i.chans] for i in infos])
print("rows max", rows.max(0), "chans max", chans.max(0), "tiles with 8/16-bit rows", int((rows[:, 2:] > 0).any(1).sum()),
      "with 8/16-bit chans", int((chans[:, 2:] > 0).any(1).sum()), "plan mix24", m.plan.mix24, "min_chunks",
      m.plan.min_chunks24, "krb", m.plan.max_krow_bytes24, flush=True)
q = P.generate((m.units, spec.group, spec.head_dim), torch.float16, seed=5, tensor=2)
for _ in range(4):
    P.packed_decode_step(m, q)
torch.cuda.synchronize()
print("done", flush=True)
