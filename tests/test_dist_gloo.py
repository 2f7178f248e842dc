"""Multi-rank host logic of the data-parallel decode (world_size 2, gloo, CPU).

The decode path has no collective; these tests cover what bench.py does around
it: disjoint shards that cover the dataset exactly once, max-over-ranks timing,
all-ranks status reduction and the aggregate throughput formula."""
import os
import socket

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2208_08711_b200.parallel import (aggregate_throughput, all_ranks_true, max_over_ranks, shard_by_bytes,
                                            shard_range)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        shard = list(shard_range(2975, rank, world))            # Cityscapes train count
        got = [None] * world
        dist.all_gather_object(got, shard)
        elapsed = 10.0 + rank * 2.5                              # per-rank device time (ms)
        mx = max_over_ranks(elapsed)
        ok = all_ranks_true(rank != 1)
        q.put((rank, got, mx, ok))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_two_ranks_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, shards, mx, ok in res:
        flat = sorted(i for s in shards for i in s)
        assert flat == list(range(2975))                         # exactly-once coverage
        assert all(set(a).isdisjoint(b) for k, a in enumerate(shards) for b in shards[k + 1:])
        assert mx == 12.5                                        # max over ranks
        assert ok is False                                       # one rank reported failure


def test_shard_helpers():
    for n in (0, 1, 7, 32, 2975):
        for world in (1, 2, 3, 8):
            parts = [list(shard_range(n, r, world)) for r in range(world)]
            assert sum(parts, []) == list(range(n))
            assert max(map(len, parts)) - min(map(len, parts)) <= 1
    sizes = [5, 9, 1, 1, 7, 3, 8, 2]
    parts = shard_by_bytes(sizes, 3)
    assert sorted(sum(parts, [])) == list(range(len(sizes)))
    loads = [sum(sizes[i] for i in p) for p in parts]
    assert max(loads) - min(loads) <= max(sizes)
    assert aggregate_throughput(32, 4, 10, 2.0) == pytest.approx(32 * 4 * 10 / 0.002)
    assert max_over_ranks(3.0) == 3.0                            # no process group: identity
