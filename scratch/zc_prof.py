"""scratch: the zc=1 fused decode on the bench workload (for ncu)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2605_08317_b200 import pipeline as P
from paper_2605_08317_b200.workload import WorkloadSpec, build
spec = WorkloadSpec(batch=16, layers=32, ctx=131072)
model, _, _, _ = build(spec)
U, d = model.units, 128
model.zc_cap, model.zc_count = 16, 0
model.zc_k = torch.zeros((U, 16, d), dtype=torch.float16, device="cuda")
model.zc_v = torch.zeros_like(model.zc_k)
model.zc_len = torch.zeros(U, dtype=torch.int32, device="cuda")
kn = P.generate((U, d), torch.float16, seed=77, tensor=1)
P.append_new_token(model, kn, kn)
q = P.generate((U, 4, d), torch.float16, seed=5, tensor=2)
out = torch.empty_like(q)
for _ in range(3): P.packed_decode_step(model, q, out)
torch.cuda.synchronize()
