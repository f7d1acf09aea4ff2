"""scratch: decode reading q straight from pinned host memory (UVA zero-copy)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import ctypes as C, torch
from paper_2605_08317_b200 import capi, pipeline as P
from paper_2605_08317_b200.workload import WorkloadSpec, build
spec = WorkloadSpec(batch=16, layers=32, ctx=int(os.environ.get("CTX", "131072")))
model, _, _, _ = build(spec)
U, g, d = spec.units, spec.group, spec.head_dim
q = P.generate((U, g, d), torch.float16, seed=5, tensor=2)
out = torch.empty_like(q)
P.packed_decode_step(model, q, out)
qh = q.cpu().pin_memory(); oh = torch.empty_like(qh).pin_memory()
o2 = torch.empty_like(q)
L = capi.lib()
a = P.decode_args(model, q, o2)
a.q = qh.data_ptr()          # q read by the kernel over PCIe (UVA-mapped pinned memory)
st = torch.cuda.current_stream().cuda_stream
rc = L.rdkv_cuda_decode(C.byref(a), st); torch.cuda.synchronize()
print("rc", rc, "equal", torch.equal(o2, out))
def ev(): return torch.cuda.Event(enable_timing=True)
def t(fn, reps=20):
    fn(); torch.cuda.synchronize(); x, y = ev(), ev(); x.record()
    for _ in range(reps): fn()
    y.record(); torch.cuda.synchronize(); return x.elapsed_time(y) * 1e3 / reps
print("decode, q from host:", t(lambda: L.rdkv_cuda_decode(C.byref(a), st)))
print("decode, q from host + D2H out:", t(lambda: (L.rdkv_cuda_decode(C.byref(a), st), oh.copy_(o2, non_blocking=True))))
a.out = oh.data_ptr()
rc = L.rdkv_cuda_decode(C.byref(a), st); torch.cuda.synchronize()
print("out to host: equal", torch.equal(oh.cuda(), out))
print("decode, q from host, out to host:", t(lambda: L.rdkv_cuda_decode(C.byref(a), st)))
