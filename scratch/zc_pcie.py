"""scratch: zero-copy decode with q and/or out in pinned host memory (PCIe directions)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import ctypes as C, torch
from paper_2605_08317_b200 import capi, pipeline as P
from paper_2605_08317_b200.workload import WorkloadSpec, build
spec = WorkloadSpec(batch=16, layers=32, ctx=131072)
model, _, _, _ = build(spec)
U, g, d = spec.units, spec.group, spec.head_dim
q = P.generate((U, g, d), torch.float16, seed=5, tensor=2)
out = torch.empty_like(q)
qh = q.cpu().pin_memory(); oh = torch.empty_like(qh).pin_memory()
L = capi.lib()
st = torch.cuda.current_stream().cuda_stream
def ev(): return torch.cuda.Event(enable_timing=True)
def t(a, reps=20):
    L.rdkv_cuda_decode(C.byref(a), st); torch.cuda.synchronize()
    x, y = ev(), ev(); x.record()
    for _ in range(reps): L.rdkv_cuda_decode(C.byref(a), st)
    y.record(); torch.cuda.synchronize(); return x.elapsed_time(y) * 1e3 / reps
for qhost, ohost in ((False, False), (True, False), (False, True), (True, True)):
    a = P.decode_args(model, q, out)
    if qhost: a.q = qh.data_ptr()
    if ohost:
        a.out = oh.data_ptr(); a.flags |= capi.RDKV_DECODE_OUT_HOST
    print(f"q {'host' if qhost else 'dev '} out {'host' if ohost else 'dev '}: {t(a):.1f} us", flush=True)
