"""torchrun worker for tests/test_dist_cpu.py (gloo, CPU, world_size 2).

Each rank takes its weak-scaling shard of sequences, runs the CPU checker
(oracle) on them — allocation + packing + decode of every (sequence, layer,
KV head) — and writes its results; rank 0 also exercises the timing
collectives. The test compares the union with a single-process run.
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import oracle  # noqa: E402
from paper_2605_08317_b200 import dist as D  # noqa: E402
from paper_2605_08317_b200.workload import chunk_seed  # noqa: E402


def run_sequence(orc, seq, layers, H, g, T, d, Sw, cfg):
    """Allocation + decode of every (layer, KV head) of one sequence on the CPU checker."""
    res = []
    for layer in range(layers):
        s = chunk_seed(7, seq, layer)
        k = orc.gen_counter(s, 0, 0, H * T * d, d, T).reshape(H, T, d)
        v = orc.gen_counter(s, 1, 0, H * T * d, d, T).reshape(H, T, d)
        pq = orc.gen_counter(s, 2, 0, H * g * Sw * d, d, T).reshape(H * g, Sw, d)
        q = orc.gen_counter(s ^ 0x55, 2, 0, H * g * d, d, T).reshape(H * g, d)
        for h in range(H):
            r = orc.allocate_head(k[h], pq[h * g:(h + 1) * g], H, cfg)
            tz = orc.tz_build(k[h], v[h], r["v_bits"], r["k_bits"])
            out = np.stack([tz.decode(q[h * g + j]) for j in range(g)])
            res.append({"seq": seq, "layer": layer, "head": h, "v_bits": int(np.sum(r["v_bits"])),
                        "kept": int(np.count_nonzero(r["v_bits"])), "out": float(np.sum(out))})
    return res


def main():
    out_dir = sys.argv[1]
    per_rank = int(sys.argv[2])
    world, rank, _ = D.init("gloo")
    shard = D.weak_shard(per_rank, rank, world)
    orc = oracle.load()
    cfg = oracle.default_config(n_tokens=16, window=8)
    results = []
    for seq in shard.items:
        results.extend(run_sequence(orc, seq, layers=2, H=2, g=2, T=64, d=16, Sw=8, cfg=cfg))
    t_local = 1.0 + rank  # a stand-in step time per rank
    D.barrier_sync(world)
    t_max = D.max_over_ranks(t_local, world)
    n_total = D.sum_over_ranks(float(shard.count), world)
    with open(os.path.join(out_dir, f"rank{rank}.json"), "w") as f:
        json.dump({"rank": rank, "world": world, "first": shard.first, "count": shard.count,
                   "t_max": t_max, "n_total": n_total, "results": results}, f)
    D.finalize(world)


if __name__ == "__main__":
    main()
