"""scratch: decode step timed back-to-back in a CUDA graph over NR arena copies
(> L2), vs a plain streaming read of the same bytes (not part of the product)."""
import ctypes as C, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2605_08317_b200 import pipeline as P
from paper_2605_08317_b200.workload import WorkloadSpec, build

NR = int(os.environ.get("NR", "6"))
spec = WorkloadSpec(batch=int(os.environ.get("B", "16")), layers=32, ctx=int(os.environ.get("CTX", "131072")))
model, _, _, _ = build(spec)
U, g, d = spec.units, spec.group, spec.head_dim
models, qs, outs = [], [], []
for r in range(NR):
    a = model.arena.clone()
    m = P.PackedModel(a, model.offsets, model.offsets_host, U, g, d)
    m.share_plan(model)
    models.append(m)
    qs.append(P.generate((U, g, d), torch.float16, seed=0xD15C0 + r, tensor=2))
    outs.append(torch.empty_like(qs[-1]))
ab = model.arena_bytes
print(f"arena {ab/1e6:.1f} MB x {NR} copies", flush=True)
kern = int(os.environ.get("KERNEL", "0"))
def ev(): return torch.cuda.Event(enable_timing=True)
def graph_time(fn_list, reps=20):
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        for f in fn_list: f()
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr):
        for f in fn_list: f()
    for _ in range(3): gr.replay()
    torch.cuda.synchronize()
    torch.cuda._sleep(1000000)
    e0, e1 = ev(), ev()
    e0.record()
    for _ in range(reps): gr.replay()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / (reps * len(fn_list))
knobs = " ".join(f"{k}={os.environ[k]}" for k in ("RDKV_DECODE_NULL", "RDKV_DECODE_PAIRS", "RDKV_DECODE_SMSP") if k in os.environ)
t = graph_time([lambda r=r: P.packed_decode_step(models[r], qs[r], outs[r], kernel=kern) for r in range(NR)])
print(f"decode b2b graph [{knobs}]: {t:.2f} us/step  {ab/t/1e3:.0f} GB/s (arena only)", flush=True)
if os.environ.get("DECODE_ONLY"):
    sys.exit(0)
L = C.CDLL(os.path.join(os.path.dirname(os.path.abspath(__file__)), "bw", "libbw.so"))
o = torch.zeros(4, dtype=torch.int32, device="cuda")
for blocks, thr in ((148 * 4, 512), (148 * 16, 256)):
    t = graph_time([lambda r=r: L.run_read(C.c_void_p(models[r].arena.data_ptr()), C.c_size_t(ab // 16 * 16), blocks, thr,
                                            C.c_void_p(o.data_ptr()), C.c_void_p(torch.cuda.current_stream().cuda_stream)) for r in range(NR)])
    print(f"plain read b2b graph {blocks}x{thr}: {t:.2f} us/launch  {ab/t/1e3:.0f} GB/s", flush=True)
t = graph_time([lambda r=r: models[r].arena.view(torch.int64)[: ab // 8].sum() for r in range(NR)])
print(f"torch sum b2b graph: {t:.2f} us  {ab/t/1e3:.0f} GB/s", flush=True)
