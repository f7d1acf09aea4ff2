"""scratch: per-unit decode errors of the kernel variants on the C1 golden case."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import oracle
from paper_2605_08317_b200 import pipeline as P
orc = oracle.load()
g = np.load(os.path.join(os.path.dirname(__file__), "..", "tests", "golden", "c1.npz"))
L, Hq, Hkv, d, T, Sw = 1, 32, 8, 128, 4096, 32
k, v, pq = orc.gen_synthetic(1, L, Hq, Hkv, d, T, Sw)
gq = Hq // Hkv
kd = torch.from_numpy(k[0]).cuda(); vd = torch.from_numpy(v[0]).cuda()
qd = torch.from_numpy(pq[0].reshape(Hkv, gq, Sw, d)).cuda()
al = P.allocate_model(kd, qd, P.default_config(), kv_heads=Hkv)
model = P.build_packed_model(kd, vd, al, group=gq)
print("plan", model.plan.max_slots, model.plan.uniform2, [model.info(u).n_kept for u in range(8)])
q = torch.from_numpy(g["q"][0].reshape(Hkv, gq, d)).cuda()
ref = g["out"][0].reshape(Hkv, gq, d)
for kern in (1, 3, 2):
    out = P.packed_decode_step(model, q, kernel=kern).cpu().numpy()
    err = [max(np.linalg.norm(out[u, j] - ref[u, j]) / np.linalg.norm(ref[u, j]) for j in range(gq)) for u in range(Hkv)]
    print("kernel", kern, " ".join(f"{e:.1e}" for e in err), flush=True)
out2 = P.packed_decode_step(model, q, kernel=2).cpu().numpy()
print("u2x head 0 first 8:", out2[0, 0, :8]); print("ref            :", ref[0, 0, :8])
print("u2x per head err unit0:", [float(np.linalg.norm(out2[0, j] - ref[0, j]) / np.linalg.norm(ref[0, j])) for j in range(4)])
