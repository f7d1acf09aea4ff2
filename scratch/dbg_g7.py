import sys, numpy as np, torch
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
from paper_2605_08317_b200 import capi, pipeline as P
import test_gpu_mma as T
rng = np.random.default_rng(107)
for g in (5, 7, 8):
    cases = [T._random_case(rng, 280, g) for _ in range(12)]
    K = torch.from_numpy(np.stack([c[0] for c in cases])).cuda(); V = torch.from_numpy(np.stack([c[1] for c in cases])).cuda()
    vb = torch.from_numpy(np.stack([c[2] for c in cases]).astype(np.uint8)).cuda(); kb = torch.from_numpy(np.stack([c[3] for c in cases]).astype(np.uint8)).cuda()
    st = torch.zeros(len(cases)*capi.HEAD_STATS_BYTES, dtype=torch.uint8, device='cuda')
    m = P.build_packed_model(K, V, P.Allocation(vb, kb, st), group=g)
    print(g, 'plan', m.plan.max_decode_bytes, m.plan.max_slots, m.plan.max_zone_b_rows, m.plan.max_kq_slots)
    q = torch.from_numpy(np.stack([c[4] for c in cases])).cuda()
    a = P.decode_args(m, q, torch.empty_like(q), 1, 2)
    import ctypes as C
    rc = capi.lib().rdkv_cuda_decode(C.byref(a), P._stream()); torch.cuda.synchronize()
    print(g, 'rc', rc, torch.cuda.current_stream())
