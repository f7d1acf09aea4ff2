"""scratch: u2c Zone C path vs the generic kernel, per unit/head."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2605_08317_b200 import capi, pipeline as P
D = 128
rng = np.random.default_rng(81)
def f16r(x): return np.asarray(x, np.float32).astype(np.float16).astype(np.float32)
for appends in (0, 1, 16, 17):
    for ns in ((3, 64, 100, 150), (150,)):
        cases = []
        for n in ns:
            k = f16r(rng.standard_normal((700, D))); v = f16r(rng.standard_normal((700, D)))
            vb = np.zeros(700, np.int32); vb[np.sort(rng.choice(700, n, replace=False))] = 2
            kb = np.full(D, 2, np.int32); q = f16r(rng.standard_normal((4, D)))
            cases.append((k, v, vb, kb, q))
        K = torch.from_numpy(np.stack([c[0] for c in cases])).cuda(); V = torch.from_numpy(np.stack([c[1] for c in cases])).cuda()
        vb = torch.from_numpy(np.stack([c[2] for c in cases]).astype(np.uint8)).cuda(); kb = torch.from_numpy(np.stack([c[3] for c in cases]).astype(np.uint8)).cuda()
        stats = torch.zeros(len(cases) * capi.HEAD_STATS_BYTES, dtype=torch.uint8, device="cuda")
        model = P.build_packed_model(K, V, P.Allocation(vb, kb, stats), group=4, zc_cap=max(appends, 1))
        for a in range(appends):
            zk = torch.from_numpy(f16r(rng.standard_normal((len(cases), D)))).cuda()
            P.append_new_token(model, zk, zk * 0.5)
        q = torch.from_numpy(np.stack([c[4] for c in cases])).cuda().half()
        o2 = P.packed_decode_step(model, q, kernel=2).float().cpu().numpy()
        o1 = P.packed_decode_step(model, q, kernel=1).float().cpu().numpy()
        err = [[float(np.linalg.norm(o2[u, j] - o1[u, j]) / np.linalg.norm(o1[u, j])) for j in range(4)] for u in range(len(cases))]
        print("appends", appends, "n", ns, " ".join("[" + ",".join(f"{e:.0e}" for e in r) + "]" for r in err), flush=True)
