"""tools: V-row / K-channel class histograms of the configs[3] budget points (bench inputs)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

from paper_2605_08317_b200.workload import WorkloadSpec, build

for model, (L, Hq, Hkv), n in (("qwen", (28, 28, 4), 256), ("qwen", (28, 28, 4), 1024), ("qwen", (28, 28, 4), 2048),
                               ("mistral", (32, 32, 8), 64), ("mistral", (32, 32, 8), 2048)):
    spec = WorkloadSpec(batch=1, layers=min(L, 4), q_heads=Hq, kv_heads=Hkv, ctx=65536, n_tokens=n, seed=11,
                        hh_stride=64, hh_boost=1.0, outlier_channels=4, outlier_scale=8.0)
    m, _, _, _ = build(spec)
    rows = np.array([[int(x) for x in i.rows] for i in m.infos()])
    chans = np.array([[int(x) for x in i.chans] for i in m.infos()])
    print(model, n, "rows(2,4,8,16) mean", rows.mean(0).round(1), "max", rows.max(0), "chans mean",
          chans.mean(0).round(1), "max", chans.max(0), "plan", m.plan.uniform2, m.plan.max_slots, flush=True)
