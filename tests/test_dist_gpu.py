"""Multi-process product path on one GPU: two torchrun ranks
(gloo process group, both on cuda:0) each build and decode their shard with
librdkv_b200.so — sequence shards (weak scaling) and KV-head shards (strong
scaling, north_star "by batch and KV head") — and the union of their outputs
equals the single-process job bit for bit (tiles are independent units:
allocate_model index l * H_kv + h, pipeline.cpp:199-205)."""
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


@pytest.mark.parametrize("shard", ["seqs", "heads"])
def test_two_ranks_one_gpu_union_equals_single_process(cuda, tmp_path, shard):
    sys.path.insert(0, os.path.join(HERE, "dist"))
    import gpu_shard_worker as W

    world, per_rank = 2, 2
    job_batch = per_rank * world if shard == "seqs" else per_rank
    single = W.job_spec(shard, 0, 1, job_batch)
    total = single.units
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr=127.0.0.1", f"--master-port={_free_port()}",
           os.path.join(HERE, "dist", "gpu_shard_worker.py"), str(tmp_path), shard, str(per_rank), str(total)]
    env = dict(os.environ, MASTER_ADDR="127.0.0.1", OMP_NUM_THREADS="1")
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, env=env)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    ranks = [np.load(tmp_path / f"rank{i}.npz") for i in range(world)]
    assert all(float(x["t"]) == 2.0 for x in ranks)  # max over ranks
    gids = np.concatenate([x["gid"] for x in ranks])
    assert sorted(gids.tolist()) == list(range(total))  # a partition of the job's units
    got = np.concatenate([x["out"] for x in ranks])[np.argsort(gids)]
    gid1, want, _ = W.run(single, total)
    assert np.array_equal(gid1, np.arange(total))
    assert np.array_equal(got, want)
