"""scratch: u2x step time for 4096 uniform-2-bit tiles with kept counts drawn from a given set."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2605_08317_b200 import capi, pipeline as P
U, T, D = 4096, 256, 128
g = torch.Generator(device="cuda").manual_seed(0)
K = (torch.randn((U, T, D), device="cuda", generator=g)).half().float()
V = (torch.randn((U, T, D), device="cuda", generator=g)).half().float()
q = torch.randn((U, 4, D), device="cuda", generator=g).half()
def ev(): return torch.cuda.Event(enable_timing=True)
for counts in [[int(x) for x in c.split("+")] for c in os.environ.get("COUNTS", "128,127+128+129,129,160,96").split(",")]:
    rng = np.random.default_rng(1)
    vb = np.zeros((U, T), np.uint8)
    for u in range(U):
        n = counts[u % len(counts)]
        vb[u, np.sort(rng.choice(T, n, replace=False))] = 2
    kb = np.full((U, D), 2, np.uint8)
    stats = torch.zeros(U * capi.HEAD_STATS_BYTES, dtype=torch.uint8, device="cuda")
    model = P.build_packed_model(K, V, P.Allocation(torch.from_numpy(vb).cuda(), torch.from_numpy(kb).cuda(), stats), group=4)
    NR = 6
    rot = [(model.arena.clone(), q.clone(), torch.empty_like(q)) for _ in range(NR)]
    ms = []
    for a, qq, oo in rot:
        m = P.PackedModel(a, model.offsets, model.offsets_host, U, 4, D); m.share_plan(model)
        ms.append((m, qq, oo))
    s = torch.cuda.Stream(); s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        for m, qq, oo in ms: P.packed_decode_step(m, qq, oo)
    torch.cuda.current_stream().wait_stream(s); torch.cuda.synchronize()
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr):
        for m, qq, oo in ms: P.packed_decode_step(m, qq, oo)
    for _ in range(3): gr.replay()
    torch.cuda.synchronize(); e0, e1 = ev(), ev(); e0.record()
    for _ in range(20): gr.replay()
    e1.record(); torch.cuda.synchronize()
    print(counts, f"{e0.elapsed_time(e1) * 1e3 / (20 * NR):.2f} us/step, arena {model.arena_bytes/1e6:.1f} MB", flush=True)
