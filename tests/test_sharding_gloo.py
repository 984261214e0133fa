"""P1 batch sharding host logic (paper_2312_17396_b200/sharding.py) on CPU:
the strong split covers the batch exactly once, weak-scaling ranks read
distinct batches, and the max-over-ranks step time over a world-size-2 gloo
group is the slowest rank's."""
import os
import socket

import pytest
import torch.multiprocessing as mp

from paper_2312_17396_b200.sharding import batch_id, shard_bounds


def test_shard_bounds_cover_the_batch():
    for batch in (1, 16, 64, 65):
        for world in (1, 2, 3, 4, 8):
            got = []
            for r in range(world):
                lo, hi = shard_bounds(batch, world, r)
                assert 0 <= hi - lo <= -(-batch // world)
                got += list(range(lo, hi))
            assert got == list(range(batch))
    with pytest.raises(ValueError):
        shard_bounds(4, 2, 2)


def test_batch_ids():
    seen = {batch_id(t, 4, r, False) for t in range(10) for r in range(4)}
    assert len(seen) == 40
    assert {batch_id(3, 4, r, True) for r in range(4)} == {12}
    assert batch_id(0, 1, 0, False) == 0


def _worker(rank, world, port, q):
    import torch.distributed as dist
    from paper_2312_17396_b200.sharding import max_over_ranks
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        q.put((rank, max_over_ranks(0.5 + rank)))
    finally:
        dist.destroy_process_group()


def test_max_over_ranks_gloo():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    out = dict(q.get(timeout=120) for _ in range(2))
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert out == {0: 1.5, 1: 1.5}
