import sys, numpy as np, torch
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import oracle
from paper_2605_08317_b200 import capi, pipeline as P
orc = oracle.load()
D = 128
def f16r(x): return np.asarray(x, np.float32).astype(np.float16).astype(np.float32)
rng = np.random.default_rng(1)
def run(name, T, vbits, kbits, qzero=False, kscale=1.0, n=4):
    cases = []
    for _ in range(n):
        k = f16r(rng.standard_normal((T, D)) * kscale); v = f16r(rng.standard_normal((T, D)))
        vb = np.zeros(T, np.int32); idx = np.sort(rng.choice(T, min(T, 64), replace=False)); vb[idx] = vbits
        kb = np.full(D, kbits, np.int32)
        q = np.zeros((4, D), np.float32) if qzero else f16r(rng.standard_normal((4, D)))
        cases.append((k, v, vb, kb, q))
    K = torch.from_numpy(np.stack([c[0] for c in cases])).cuda(); V = torch.from_numpy(np.stack([c[1] for c in cases])).cuda()
    vb = torch.from_numpy(np.stack([c[2] for c in cases]).astype(np.uint8)).cuda(); kb = torch.from_numpy(np.stack([c[3] for c in cases]).astype(np.uint8)).cuda()
    st = torch.zeros(len(cases)*capi.HEAD_STATS_BYTES, dtype=torch.uint8, device='cuda')
    m = P.build_packed_model(K, V, P.Allocation(vb, kb, st), group=4)
    q = torch.from_numpy(np.stack([c[4] for c in cases])).cuda()
    a = P.packed_decode_step(m, q, kernel=2).cpu().numpy(); b = P.packed_decode_step(m, q, kernel=1).cpu().numpy()
    errs = []
    for u, c in enumerate(cases):
        tz = orc.tz_build(c[0], c[1], c[2], c[3])
        for j in range(4):
            w = tz.decode(c[4][j]); errs.append((np.linalg.norm(a[u,j]-w)/np.linalg.norm(w), np.linalg.norm(b[u,j]-w)/np.linalg.norm(w)))
    e = np.array(errs); print(f"{name:40s} mma {e[:,0].max():.2e}  gen {e[:,1].max():.2e}")
    return a, b, cases
run("V2 K2", 256, 2, 2)
run("V2 K2 q=0", 256, 2, 2, qzero=True)
run("V8 K2", 256, 8, 2)
run("V4 K2", 256, 4, 2)
run("V2 K8", 256, 2, 8)
run("V2 K4", 256, 2, 4)
run("V2 K16", 256, 2, 16)
run("V16 K2", 256, 16, 2)
run("V2 K0", 256, 2, 0)
run("V2 K2 kscale 0.1", 256, 2, 2, kscale=0.1)
run("V2 K2 kscale 3", 256, 2, 2, kscale=3.0)
a, b, cases = run("V2 K2 detail", 64, 2, 2, n=1)
print("mma", a[0,0,:8]); print("gen", b[0,0,:8])
d = a[0,0]-b[0,0]; print("diff by channel mod 4:", [float(np.abs(d[i::4]).mean()) for i in range(4)], "mod16", [float(np.abs(d[i::16]).mean()) for i in range(16)])
