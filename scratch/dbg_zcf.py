"""scratch: fused (zc bound <= 4) vs chunked Zone C path vs the oracle on the failing test case."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np, torch
import oracle
from paper_2605_08317_b200 import capi, pipeline as P
import test_gpu_mma as T
orc = oracle.load()
for n_max, appends in ((128, 3), (150, 1), (160, 4)):
    rng = np.random.default_rng(80 + appends)
    cases = []
    for n in (3, 64, 100, n_max):
        k, v, vb, kb, q = T._random_case(rng, 700, 4)
        vb[:] = 0
        vb[np.sort(rng.choice(700, n, replace=False))] = 2
        kb[:] = 2
        cases.append((k, v, vb, kb, q))
    K = torch.from_numpy(np.stack([c[0] for c in cases])).cuda(); V = torch.from_numpy(np.stack([c[1] for c in cases])).cuda()
    vb = torch.from_numpy(np.stack([c[2] for c in cases]).astype(np.uint8)).cuda(); kb = torch.from_numpy(np.stack([c[3] for c in cases]).astype(np.uint8)).cuda()
    stats = torch.zeros(len(cases) * capi.HEAD_STATS_BYTES, dtype=torch.uint8, device="cuda")
    model = P.build_packed_model(K, V, P.Allocation(vb, kb, stats), group=4, zc_cap=appends)
    zk = T.f16r(rng.standard_normal((appends, len(cases), 128))); zv = T.f16r(rng.standard_normal((appends, len(cases), 128)))
    for a in range(appends):
        P.append_new_token(model, torch.from_numpy(zk[a]).cuda(), torch.from_numpy(zv[a]).cuda())
    q = torch.from_numpy(np.stack([c[4] for c in cases])).cuda()
    of = P.packed_decode_step(model, q).cpu().numpy()
    model.zc_count = None
    oc = P.packed_decode_step(model, q).cpu().numpy()
    og = P.packed_decode_step(model, q, kernel=1).cpu().numpy()
    for u, (k, v, vbs, kbs, qq) in enumerate(cases):
        tz = orc.tz_build(k, v, vbs, kbs)
        for a in range(appends): tz.append(zk[a, u], zv[a, u])
        e = []
        for j in range(4):
            want = tz.decode(qq[j])
            e.append((T.rel(of[u, j], want), T.rel(oc[u, j], want), T.rel(og[u, j], want)))
        print(n_max, appends, u, " ".join(f"f{a:.1e}/c{b:.1e}/g{c:.1e}" for a, b, c in e))
