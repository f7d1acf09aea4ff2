"""tools: configs[3] budget-sweep points (bench.py secondary line) timed alone, with the
kernel choice printed (RDKV_DECODE_VERBOSE needs the experiments build; here we print the plan)."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
if "--exp" in sys.argv:  # the EXPERIMENTS build (timing knobs), tools only
    sys.argv.remove("--exp")
    from paper_2605_08317_b200 import capi

    capi.LIB_PATH = os.path.join(ROOT, "paper_2605_08317_b200", "_lib_exp", "librdkv_b200.so")
import numpy as np
import torch

import bench
from paper_2605_08317_b200 import pipeline as P
from paper_2605_08317_b200.workload import WorkloadSpec, build

peak, _ = bench.load_peaks()
pts = [("qwen2.5-7b", (28, 28, 4), n) for n in (64, 256, 1024, 2048)] + [("mistral-7b", (32, 32, 8), n) for n in (64, 2048)]
sweep = "--sweep" in sys.argv
sel = [a for a in sys.argv[1:] if a != "--sweep"] or None
for model, (L, Hq, Hkv), n in pts:
    if sel and f"{model}_n{n}" not in sel:
        continue
    spec = WorkloadSpec(batch=4, layers=L, q_heads=Hq, kv_heads=Hkv, ctx=65536, n_tokens=n, seed=11,
                        hh_stride=64, hh_boost=1.0, outlier_channels=4, outlier_scale=8.0)
    m, _, st, _ = build(spec)
    q = P.generate((m.units, spec.group, spec.head_dim), torch.float16, seed=bench.QSEED, tensor=2)
    us, _ = bench.graph_step_us(P, m, q, 50)
    if sweep:  # the chunked split-K kernel at forced parts per tile
        for S in (1, 2, 3, 4, 5, 6, 7, 8, 10, 14):
            if S <= int(m.plan.min_chunks24) and (S == 1 or m.split_ws is not None):
                su, _ = bench.graph_step_us(P, m, q, 50, kernel=2, split=S)
                print(json.dumps({"point": f"{model}_n{n}", "parts": S, "us_per_step": round(su, 2)}), flush=True)
    byts = m.survey_bytes(io_bytes=2)
    ref = P.packed_decode_step(m, q, kernel=1).float()
    out = P.packed_decode_step(m, q).float()
    err = ((out - ref).norm() / ref.norm()).item()
    print(json.dumps({"point": f"{model}_n{n}", "us_per_step": round(us, 2), "roofline_frac": byts / (us / 1e6) / 1e9 / peak,
                      "bytes": byts, "units": m.units, "mix24": int(m.plan.mix24), "min_chunks": int(m.plan.min_chunks24),
                      "uniform2": int(m.plan.uniform2), "max_slots": int(m.plan.max_slots),
                      "rel_vs_generic": err}), flush=True)
    del m, q
