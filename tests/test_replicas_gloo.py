"""Multi-process (gloo, world_size 2) coverage of the replica host logic used by
bench.py --gpus N: batch sharding, per-replica seeds, max-over-ranks timing -- and
bench.py's own multi-rank branch, launched by torchrun with a CPU stand-in for the
device step (`--stub-device`)."""
import json
import os
import socket
import subprocess
import sys

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2603_28708_b200 import replicas

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_shard_batch_covers_exactly():
    for gb in [1, 7, 32, 33]:
        for world in [1, 2, 3, 8]:
            spans = [replicas.shard_batch(gb, world, r) for r in range(world)]
            assert sum(c for _, c in spans) == gb
            pos = 0
            for s, c in spans:
                assert s == pos
                pos += c
    with pytest.raises(ValueError):
        replicas.shard_batch(4, 2, 2)


def test_rank_batch_weak_and_strong():
    assert [replicas.rank_batch(32, 4, r, False) for r in range(4)] == [(0, 32), (32, 32), (64, 32), (96, 32)]
    assert [replicas.rank_batch(32, 4, r, True) for r in range(4)] == [(0, 8), (8, 8), (16, 8), (24, 8)]
    assert replicas.rank_batch(32, 1, 0, True) == (0, 32)


def test_timed_steps_counts_exactly():
    calls = []
    per, mine, total = replicas.timed_steps(lambda: calls.append(1), 5, 3, replicas.WallTimer())
    assert len(calls) == 8 and len(per) == 5 and total == mine


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        start, count = replicas.shard_batch(33, world, rank)
        t = replicas.max_over_ranks(1.0 + rank, dist)  # rank 1 is the slow one
        seed = replicas.replica_token_seed(1234, rank)
        gb = replicas.sum_over_ranks(count, dist)
        q.put((rank, start, count, t, seed, int(gb), replicas.aggregate_throughput(32, world, t)))
    finally:
        dist.destroy_process_group()


def test_two_rank_replicas_gloo():
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert [r[1:3] for r in res] == [(0, 17), (17, 16)]
    assert all(r[3] == 2.0 for r in res)            # max over ranks
    assert [r[4] for r in res] == [1234, 1235]      # independent replica inputs
    assert all(r[5] == 33 for r in res)             # shards cover the global batch
    assert all(r[6] == 32.0 for r in res)           # 2 ranks x 32 seq / 2 s


def _torchrun_bench(extra):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()),
           os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "4", "--warmup", "3",
           "--stub-device"] + extra
    env = dict(os.environ, OMP_NUM_THREADS="1")
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=300, env=env, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout  # rank 0 alone prints
    return json.loads(lines[0])


def test_bench_multirank_branch_weak():
    line = _torchrun_bench([])
    assert line["n_gpus"] == 2 and line["scaling"] == "weak"
    assert line["config"]["workload"].startswith("C4")          # WORLD_SIZE > 1 -> configs[3]
    assert line["config"]["global_batch"] == 64 and line["config"]["per_replica_batch"] == 32
    # value = all ranks' sequences / the SLOWEST rank's time (rank 1 sleeps 8 ms a step, rank 0 2 ms)
    assert line["ms_per_step"] >= 8.0 and line["ms_per_step"] >= line["rank_ms"] / 4 * 1.5
    assert abs(line["value"] - 64 * 4 / (line["ms_per_step"] * 4 / 1000.0)) < 1e-6 * line["value"]


def test_bench_multirank_branch_strong():
    line = _torchrun_bench(["--strong"])
    assert line["scaling"] == "strong"
    assert line["config"]["global_batch"] == 32 and line["config"]["per_replica_batch"] == 16
