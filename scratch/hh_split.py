"""scratch: heavy-hitter workload — general kernel on all tiles vs split (u2x on uniform tiles + general on mixed)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2605_08317_b200 import pipeline as P
from paper_2605_08317_b200.workload import WorkloadSpec, build
spec = WorkloadSpec(batch=16, layers=32, ctx=131072, hh_stride=64, hh_boost=1.0)
model, _, _, _ = build(spec)
infos = model.infos()
uni = np.array([i.rows[1] == 0 and i.rows[2] == 0 and i.rows[3] == 0 and i.chans[1] == 0 and i.chans[2] == 0 and i.chans[3] == 0 for i in infos])
U = model.units
q = P.generate((U, 4, 128), torch.float16, seed=5, tensor=2)
def sub(ids):
    offs = np.concatenate([model.offsets_host[ids], [0]])
    m = P.PackedModel(model.arena, torch.from_numpy(offs).cuda(), offs, len(ids), 4, 128)
    m.prepare()
    return m, q[torch.from_numpy(ids).cuda()].contiguous()
def ev(): return torch.cuda.Event(enable_timing=True)
def t(fn, reps=20):
    for _ in range(3): fn()
    torch.cuda.synchronize(); a, b = ev(), ev(); a.record()
    for _ in range(reps): fn()
    b.record(); torch.cuda.synchronize(); return a.elapsed_time(b) * 1e3 / reps
o = torch.empty_like(q)
print("all tiles (general):", t(lambda: P.packed_decode_step(model, q, o)))
iu, im = np.nonzero(uni)[0], np.nonzero(~uni)[0]
mu, qu = sub(iu); mm, qm = sub(im)
ou, om = torch.empty_like(qu), torch.empty_like(qm)
print("uniform subset", len(iu), "(u2x):", t(lambda: P.packed_decode_step(mu, qu, ou)))
print("mixed subset", len(im), "(general):", t(lambda: P.packed_decode_step(mm, qm, om)))
print("both back to back:", t(lambda: (P.packed_decode_step(mm, qm, om), P.packed_decode_step(mu, qu, ou))))
if os.environ.get("PROF_MIXED"):
    torch.cuda.synchronize()
    P.packed_decode_step(mm, qm, om)
    torch.cuda.synchronize()
print("plan uniform2", model.plan.uniform2, "n_uniform", model.plan.n_uniform, "split", model.plan.uniform2_split)
r1 = np.array([i.rows[1] for i in infos]); c1 = np.array([i.chans[1] for i in infos]); c0 = np.array([i.chans[0] for i in infos])
print("r1 max", r1.max(), "tiles r1>8", (r1 > 8).sum(), "c0 min", c0.min(), "c1 max", c1.max())
