"""Decode kernel sweep on the bench workload (scratch tool): builds the 128K x16 x32
packed model once, then times the decode launch for several kernel / pair settings."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2605_08317_b200 import pipeline as P
from paper_2605_08317_b200.workload import WorkloadSpec, build

ctx = int(os.environ.get("CTX", "131072"))
spec = WorkloadSpec(batch=16, layers=32, ctx=ctx)
model, _, _, _ = build(spec)
U, g, d = spec.units, spec.group, spec.head_dim
q = P.generate((U, g, d), torch.float16, seed=0xD15C0, tensor=2)
flush_w = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
flush_r = torch.ones(256 << 20, dtype=torch.uint8, device="cuda").view(torch.int64)
MODE = os.environ.get("FLUSH", "w")


class _Flush:
    def zero_(self):
        flush_w.zero_()
        if MODE == "wr":
            flush_r.sum()


flush = _Flush()
ref = torch.empty_like(q)
P.packed_decode_step(model, q, ref, kernel=1)  # generic CUDA-core result for a sanity check
configs = [c.split(":") for c in sys.argv[1:]] or [["0", "0"]]
arena64 = model.arena[: (model.arena_bytes // 8) * 8].view(torch.int64)
for it in range(3):
    flush.zero_()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    x = arena64.sum()
    e.record()
    torch.cuda.synchronize()
    print(f"torch sum over the arena ({model.arena_bytes / 1e6:.1f} MB): {s.elapsed_time(e) * 1e3:.1f} us", flush=True)
for cfg in configs:
    kern, pairs = cfg[0], cfg[1]
    os.environ["RDKV_DECODE_NULL"] = cfg[2] if len(cfg) > 2 else "0"
    os.environ["RDKV_DECODE_PAIRS"] = pairs
    out = torch.empty_like(q)
    for _ in range(5):
        flush.zero_()
        P.packed_decode_step(model, q, out, kernel=int(kern))
    ts = []
    for _ in range(50):
        flush.zero_()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        P.packed_decode_step(model, q, out, kernel=int(kern))
        e.record()
        torch.cuda.synchronize()
        ts.append(s.elapsed_time(e) * 1e3)
    ts.sort()
    err = ((out.float() - ref.float()).norm() / ref.float().norm()).item()
    bad = torch.isnan(out.float()).reshape(U, -1).any(1).nonzero().flatten()
    if bad.numel():
        info = model.infos() if hasattr(model, "infos") else None
        print("NaN tiles:", bad[:10].tolist(), "count", bad.numel(),
              "n_kept of first:", [int(info[i].n_kept) for i in bad[:5].tolist()] if info else None, flush=True)
        print("ref NaN:", torch.isnan(ref.float()).any().item(), flush=True)
    print(f"kernel {kern} pairs {pairs} null {os.environ['RDKV_DECODE_NULL']}: median {ts[len(ts)//2]:.1f} us  min {ts[0]:.1f}  rel err vs generic {err:.2e}",
          flush=True)
