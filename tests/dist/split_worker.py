"""torchrun worker for tests/test_dist_cpu.py: the optional sequence-split
merge on gloo (CPU). Every rank builds the same heads, takes the token chunks
c % world == rank (pipeline.chunk_ranges, the device rule), computes its
partial (unnormalised o, max in log2 units, weight sum), all-gathers the
partials (dist.gather_partials) and merges them (pipeline.merge_partials_reference,
the formula of the CUDA merge kernel)."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2605_08317_b200 import dist as D  # noqa: E402
from paper_2605_08317_b200 import pipeline as P  # noqa: E402


def heads(n_heads=3, g=2, d=16):
    rng = np.random.default_rng(5)
    out = []
    for h in range(n_heads):
        n = [100, 400, 1000][h]
        out.append((rng.standard_normal((n, d)), rng.standard_normal((n, d)), rng.standard_normal((g, d))))
    return out


def partial_of(k, v, q, rank, world):
    """[g, d + 2] partial of this rank's chunks (slots = tokens here)."""
    d = k.shape[1]
    logits = (q @ k.T) / np.sqrt(d) * np.log2(np.e)  # log2 units, like the kernels
    mine = np.zeros(k.shape[0], bool)
    for c, (s0, ns) in enumerate(P.chunk_ranges(k.shape[0])):
        if c % world == rank:
            mine[s0:s0 + ns] = True
    res = np.zeros((q.shape[0], d + 2))
    for j in range(q.shape[0]):
        if not mine.any():
            res[j, d], res[j, d + 1] = -np.inf, 0.0
            continue
        m = logits[j, mine].max()
        p = np.exp2(logits[j, mine] - m)
        res[j, :d] = p @ v[mine]
        res[j, d], res[j, d + 1] = m, p.sum()
    return res


def main():
    out_dir = sys.argv[1]
    world, rank, _ = D.init("gloo")
    hs = heads()
    part = torch.from_numpy(np.stack([partial_of(k, v, q, rank, world) for k, v, q in hs])).float()
    parts = D.gather_partials(part, world)
    merged = P.merge_partials_reference(parts).numpy()
    errs = []
    for i, (k, v, q) in enumerate(hs):
        lg = (q @ k.T) / np.sqrt(k.shape[1])
        w = np.exp(lg - lg.max(1, keepdims=True))
        want = (w @ v) / w.sum(1, keepdims=True)
        errs.append(float(np.abs(merged[i] - want).max()))
    with open(os.path.join(out_dir, f"split{rank}.json"), "w") as f:
        json.dump({"rank": rank, "world": world, "max_err": max(errs),
                   "nonempty": [bool(np.isfinite(part[i, 0, -2])) for i in range(len(hs))]}, f)
    D.finalize(world)


if __name__ == "__main__":
    main()
