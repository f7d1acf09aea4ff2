"""torchrun worker for tests/test_dist_gpu.py: one rank of a 2-rank job on ONE
GPU (gloo process group, both ranks on cuda:0), each building and decoding its
own shard through librdkv_b200.so exactly as bench.py does under torchrun:
K0 generation of its (sequence, KV head) slice -> weights -> allocate -> pack
-> one decode launch. Writes its outputs keyed by global unit id."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2605_08317_b200 import dist as D  # noqa: E402
from paper_2605_08317_b200 import pipeline as P  # noqa: E402
from paper_2605_08317_b200.workload import WorkloadSpec, build  # noqa: E402

QSEED = 0x5EED


def job_spec(shard, rank, world, per_rank_batch):
    return WorkloadSpec(batch=per_rank_batch, layers=2, ctx=2048, n_tokens=128, rank=rank, shard=shard, world=world,
                        hh_stride=64, hh_boost=1.0)


def run(spec, total_units):
    """Build this rank's shard and decode it with q rows of the whole job (by global unit)."""
    model, _, stats, _ = build(spec)
    gid = np.array([spec.global_unit(b, l, h) for b in range(spec.batch) for l in range(spec.layers)
                    for h in range(spec.local_heads)], np.int64)
    qall = P.generate((total_units, spec.group, spec.head_dim), torch.float16, seed=QSEED, tensor=2)
    q = qall[torch.from_numpy(gid).cuda()].contiguous()
    out = P.packed_decode_step(model, q)
    torch.cuda.synchronize()
    return gid, out.float().cpu().numpy(), model.plan.uniform2


def main():
    out_dir, shard, per_rank_batch, total_units = sys.argv[1], sys.argv[2], int(sys.argv[3]), int(sys.argv[4])
    world, rank, _ = D.init("gloo")
    spec = job_spec(shard, rank, world, per_rank_batch)
    gid, out, u2 = run(spec, total_units)
    D.barrier_sync(world)
    t = D.max_over_ranks(float(rank + 1), world)
    np.savez(os.path.join(out_dir, f"rank{rank}.npz"), gid=gid, out=out, t=t, uniform2=u2,
             device=torch.cuda.current_device())
    D.finalize(world)


if __name__ == "__main__":
    main()
