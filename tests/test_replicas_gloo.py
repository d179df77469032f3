"""Multi-process (gloo, world_size 2) coverage of the replica host logic used by
bench.py --gpus N: batch sharding, per-replica seeds and max-over-ranks timing."""
import os
import socket

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2603_28708_b200 import replicas


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
        import torch
        c = torch.tensor([count])
        dist.all_reduce(c)
        q.put((rank, start, count, t, seed, int(c.item()),
               replicas.aggregate_throughput(32, world, t)))
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
