"""tools: generic-kernel split sweep on configs[3] points (model, n)."""
import sys
import torch
sys.path.insert(0, ".")
from paper_2605_08317_b200 import pipeline as P
from paper_2605_08317_b200.workload import WorkloadSpec, build

for model, n in (("qwen", 1024), ("qwen", 2048), ("mistral", 2048)):
    L, Hq, Hkv = {"qwen": (28, 28, 4), "mistral": (32, 32, 8)}[model]
    spec = WorkloadSpec(batch=4, layers=L, q_heads=Hq, kv_heads=Hkv, ctx=65536, n_tokens=n, seed=11,
                        hh_stride=64, hh_boost=1.0, outlier_channels=4, outlier_scale=8.0)
    m, _, st, _ = build(spec)
    q = P.generate((m.units, spec.group, spec.head_dim), torch.float16, seed=7, tensor=2)
    ref = P.packed_decode_step(m, q, kernel=1).float()
    res = []
    for split in (1, 2, 3, 4, 8):
        ws = P.decode_workspace(m, split) if split > 1 else None
        out = torch.empty_like(q)
        for _ in range(3):
            P.packed_decode_step(m, q, out, split=split, kernel=1, workspace=ws)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            P.packed_decode_step(m, q, out, split=split, kernel=1, workspace=ws)
        e1.record()
        torch.cuda.synchronize()
        rel = ((out.float() - ref).norm() / ref.norm()).item()
        res.append(f"s{split}={e0.elapsed_time(e1) / 10 * 1e3:.0f}us(rel {rel:.1e})")
    print(model, n, "units", m.units, "max_slots", m.plan.max_slots, " ".join(res), flush=True)
