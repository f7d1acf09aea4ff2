"""tools: u2x launch experiments on the headline step with the EXPERIMENTS build
(paper_2605_08317_b200/_lib_exp, make -C paper_2605_08317_b200/csrc EXPERIMENTS=1
OUT=../_lib_exp): one configuration per process (the knobs are read once).
usage: RDKV_DECODE_CTAS=2 python tools/u2x_exp.py [steps]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2605_08317_b200 import capi

capi.LIB_PATH = os.path.join(ROOT, "paper_2605_08317_b200", "_lib_exp", "librdkv_b200.so")
import torch

from paper_2605_08317_b200 import pipeline as P
from paper_2605_08317_b200.workload import WorkloadSpec, build

import bench

K = int(sys.argv[1]) if len(sys.argv) > 1 else 200
spec = WorkloadSpec(batch=16, layers=32, ctx=131072, n_tokens=128)
model, _, _, _ = build(spec)
q = P.generate((model.units, spec.group, spec.head_dim), torch.float16, seed=bench.QSEED, tensor=2)
ref = P.packed_decode_step(model, q).float()
us, _ = bench.graph_step_us(P, model, q, K)
us2, _ = bench.graph_step_us(P, model, q, K)
knobs = {k: v for k, v in os.environ.items() if k.startswith("RDKV_DECODE_")}
print(f"{knobs}: {us:.2f} / {us2:.2f} us/step", flush=True)
