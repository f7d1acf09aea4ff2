"""tools: the bench's headline step (configs[2], 4096 tiles) as one CUDA graph of
K back-to-back decode launches over rotation copies of the arena (>= 3x L2),
replayed twice — the exact method of bench.py's timed region, for

    ncu --graph-profiling graph --metrics gpu__time_duration.sum,... python tools/graph_step.py K

so that the profiled graph duration / K is directly comparable with the bench's
ms_per_step (ncu's per-kernel mode serialises launches and drops the PDL overlap).
Also prints the event-timed step of the same graph (unprofiled runs only)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2605_08317_b200 import pipeline as P
from paper_2605_08317_b200.workload import WorkloadSpec, build

K = int(sys.argv[1]) if len(sys.argv) > 1 else 200
spec = WorkloadSpec(batch=16, layers=32, ctx=int(os.environ.get("CTX", "131072")), n_tokens=128)
model, _, _, _ = build(spec)
U, g, d = model.units, spec.group, spec.head_dim
q = P.generate((U, g, d), torch.float16, seed=0xD15C0, tensor=2)
l2 = torch.cuda.get_device_properties(0).L2_cache_size
per_copy = model.arena_bytes + 2 * q.numel() * q.element_size()
n_rot = max(2, -(-3 * l2 // per_copy))
rot = [(model, q, torch.empty_like(q))]
for r in range(1, n_rot):
    m = P.PackedModel(model.arena.clone(), model.offsets, model.offsets_host, U, g, d)
    m.share_plan(model)
    rot.append((m, q.clone(), torch.empty_like(q)))
for i in range(3):
    m, qq, oo = rot[i % n_rot]
    P.packed_decode_step(m, qq, oo)
torch.cuda.synchronize()
graph = torch.cuda.CUDAGraph()
side = torch.cuda.Stream()
side.wait_stream(torch.cuda.current_stream())
with torch.cuda.graph(graph, stream=side):
    for i in range(K):
        m, qq, oo = rot[i % n_rot]
        P.packed_decode_step(m, qq, oo)
torch.cuda.synchronize()
for rep in range(2):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(side):
        e0.record(side)
        graph.replay()
        e1.record(side)
    torch.cuda.synchronize()
    print(f"graph replay {rep}: {K} steps, {e0.elapsed_time(e1) / K * 1e3:.2f} us/step "
          f"(survey bytes {model.survey_bytes(io_bytes=2) / 1e6:.2f} MB/step)", flush=True)
