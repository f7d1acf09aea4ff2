"""tools: prefill (K1 weights, K2 allocate, K3 pack) timing on one (sequence, layer)
chunk of the configs[2] workload (8 KV heads x 131072 tokens, n=128), CUDA events
around each stage after a warm-up; and configs[1] (32 layers x 32K, B=1) end to end.
Run under ncu for the per-kernel launch list."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import json

if "--exp" in sys.argv:  # the EXPERIMENTS build (timing variants), tools only
    from paper_2605_08317_b200 import capi

    capi.LIB_PATH = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_2605_08317_b200",
                                 "_lib_exp", "librdkv_b200.so")
    sys.argv.remove("--exp")

import torch

from paper_2605_08317_b200 import pipeline as P
from paper_2605_08317_b200.workload import WorkloadSpec, gen_chunk

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
spec = WorkloadSpec(batch=1, layers=1, ctx=int(os.environ.get("CTX", "131072")), n_tokens=128)
k, v, q = gen_chunk(spec, 0, 0)
cfg = P.default_config(n_tokens=128, window=spec.probe_rows)
res = {}
for r in range(reps + 1):
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    ev[0].record()
    w_t, w_c = P.compute_weights(k, q, window=cfg.window, pool_kernel=cfg.pool_kernel, kv_heads=spec.kv_heads)
    ev[1].record()
    al = P.allocate(w_t, w_c, cfg, group=spec.group, probe_rows=spec.probe_rows, kv_heads=spec.kv_heads)
    ev[2].record()
    m = P.build_packed_model(k, v, al, group=spec.group)
    ev[3].record()
    torch.cuda.synchronize()
    if r:
        for name, a, b in (("weights_ms", 0, 1), ("allocate_ms", 1, 2), ("pack_ms", 2, 3)):
            res.setdefault(name, []).append(ev[a].elapsed_time(ev[b]))
al.check()
out = {k2: min(v2) for k2, v2 in res.items()}
out["config"] = f"one (sequence, layer): {spec.kv_heads} KV heads x T={spec.ctx}, g={spec.group}, n=128"
out["kept_mean"] = float(al.stats_host()["n_kept"].mean())
import hashlib

out["w_t_sha1"] = hashlib.sha1(w_t.cpu().numpy().tobytes()).hexdigest()[:16]
out["v_bits_sha1"] = hashlib.sha1(al.v_bits.cpu().numpy().tobytes()).hexdigest()[:16]
print(json.dumps(out), flush=True)
if os.environ.get("C1", "1") == "1":
    spec1 = WorkloadSpec(batch=1, layers=32, ctx=32768, n_tokens=128)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for layer in range(spec1.layers):
        k1, v1, q1 = gen_chunk(spec1, 0, layer)
        a1 = P.allocate_model(k1, q1, cfg, kv_heads=spec1.kv_heads)
        P.build_packed_model(k1, v1, a1, group=spec1.group)
    torch.cuda.synchronize()
    print(json.dumps({"configs1_gen_allocate_pack_s": time.perf_counter() - t0}), flush=True)
