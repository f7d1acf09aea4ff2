"""Multi-process (gloo, world_size 2, CPU) checks of the sharded path
(SURVEY.md §8(e)): the shards partition the job with no overlap, the job is
the same whatever the world size (per-sequence seeds), and the timing
collectives (barrier, max / sum over ranks) behave as bench.py needs."""
import json
import os
import socket
import subprocess
import sys

import pytest

from paper_2605_08317_b200 import dist as D

HERE = os.path.dirname(os.path.abspath(__file__))


def test_weak_and_strong_shards_partition():
    for world in (1, 2, 3, 8):
        seen = [i for r in range(world) for i in D.weak_shard(4, r, world).items]
        assert seen == list(range(4 * world))
        for total in (0, 1, 7, 64, 65):
            parts = [D.strong_shard(total, r, world) for r in range(world)]
            assert [i for p in parts for i in p.items] == list(range(total))
            assert max(p.count for p in parts) - min(p.count for p in parts) <= 1
    with pytest.raises(ValueError):
        D.weak_shard(4, 2, 2)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def test_two_rank_gloo_job_equals_single_process(tmp_path):
    per_rank = 2
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr=127.0.0.1", f"--master-port={_free_port()}",
           os.path.join(HERE, "dist", "shard_worker.py"), str(tmp_path), str(per_rank)]
    env = dict(os.environ, MASTER_ADDR="127.0.0.1", OMP_NUM_THREADS="1")
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=300, env=env)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    ranks = [json.load(open(tmp_path / f"rank{i}.json")) for i in range(2)]
    assert [x["first"] for x in ranks] == [0, per_rank]
    assert all(x["t_max"] == 2.0 for x in ranks)          # max over ranks of 1.0, 2.0
    assert all(x["n_total"] == 2 * per_rank for x in ranks)
    got = sorted((q["seq"], q["layer"], q["head"], q["v_bits"], q["kept"], q["out"])
                 for x in ranks for q in x["results"])
    # the same job in one process
    sys.path.insert(0, os.path.join(HERE, "dist"))
    import oracle
    import shard_worker

    orc = oracle.load()
    cfg = oracle.default_config(n_tokens=16, window=8)
    want = []
    for seq in range(2 * per_rank):
        want += [(q["seq"], q["layer"], q["head"], q["v_bits"], q["kept"], q["out"])
                 for q in shard_worker.run_sequence(orc, seq, layers=2, H=2, g=2, T=64, d=16, Sw=8, cfg=cfg)]
    assert got == sorted(want)


def test_sequence_split_merge_two_ranks(tmp_path):
    """The optional cross-GPU merge on gloo: two ranks take
    alternate token chunks of each head, all-gather the partials and merge them
    with the log-sum-exp combine the CUDA merge kernel implements."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr=127.0.0.1", f"--master-port={_free_port()}",
           os.path.join(HERE, "dist", "split_worker.py"), str(tmp_path)]
    env = dict(os.environ, MASTER_ADDR="127.0.0.1", OMP_NUM_THREADS="1")
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=300, env=env)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    ranks = [json.load(open(tmp_path / f"split{i}.json")) for i in range(2)]
    assert all(x["max_err"] < 1e-5 for x in ranks), ranks
    # the 100-token head is one chunk (rank 0 only); longer heads split across both
    assert ranks[0]["nonempty"] == [True, True, True] and ranks[1]["nonempty"] == [False, True, True]


def test_chunk_ranges_cover_slots():
    from paper_2605_08317_b200 import pipeline as P

    for nslot in (4, 128, 160, 164, 516, 804, 2048, 4100):
        r = P.chunk_ranges(nslot)
        assert r[0][0] == 0 and sum(n for _, n in r) == nslot
        assert all(0 < n <= 160 and s % 32 == 0 for s, n in r)
        assert all(r[i][0] + r[i][1] == r[i + 1][0] for i in range(len(r) - 1))
