"""scratch: run one configs[3] point (model, n) in isolation: build, plan, one decode + parity vs the
generic kernel. usage: c4_probe.py MODEL N [kernel]"""
import sys
import torch
sys.path.insert(0, ".")
from paper_2605_08317_b200 import pipeline as P
from paper_2605_08317_b200.workload import WorkloadSpec, build

model, n = sys.argv[1], int(sys.argv[2])
L, Hq, Hkv = {"qwen": (28, 28, 4), "mistral": (32, 32, 8)}[model]
batch = int(sys.argv[3]) if len(sys.argv) > 3 else 4
spec = WorkloadSpec(batch=batch, layers=L, q_heads=Hq, kv_heads=Hkv, ctx=65536, n_tokens=n, seed=11,
                    hh_stride=64, hh_boost=1.0, outlier_channels=4, outlier_scale=8.0)
m, _, st, _ = build(spec)
pl = m.plan
print(model, n, "units", m.units, "uniform2", pl.uniform2, "split", pl.uniform2_split, "n_uniform", pl.n_uniform,
      "max_slots", pl.max_slots, "max_zb", pl.max_zone_b_rows, "max_kq", pl.max_kq_slots, "max_bytes", pl.max_decode_bytes,
      flush=True)
q = P.generate((m.units, spec.group, spec.head_dim), torch.float16, seed=7, tensor=2)
o1 = P.packed_decode_step(m, q)
torch.cuda.synchronize()
print("default ok", flush=True)
o2 = P.packed_decode_step(m, q, kernel=1)
torch.cuda.synchronize()
rel = ((o1.float() - o2.float()).norm() / o2.float().norm()).item()
print("generic ok rel", rel, flush=True)
import bench  # noqa: E402
us, nrot = bench.graph_step_us(P, m, q, 20)
print("graph us", us, "rot", nrot, flush=True)
