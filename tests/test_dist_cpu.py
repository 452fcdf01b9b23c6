"""Multi-process host logic of the multi-GPU path on CPU (gloo, world_size 2):
frame sharding, the timer max-reduction and the per-frame stats gather."""
import os
import socket

import pytest
import torch
import torch.multiprocessing as mp

from paper_2201_11924_b200.dist import gather_frame_stats, max_over_ranks, shard_range


@pytest.mark.parametrize("n", [0, 1, 7, 4096])
def test_shard_range_partition(n):
    for world in range(1, 9):
        rs = [shard_range(n, r, world) for r in range(world)]
        assert rs[0][0] == 0 and rs[-1][1] == n
        assert all(a[1] == b[0] for a, b in zip(rs, rs[1:]))
        sizes = [b - a for a, b in rs]
        assert max(sizes) - min(sizes) <= 1


def test_shard_range_rejects():
    with pytest.raises(ValueError):
        shard_range(10, 2, 2)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        lo, hi = shard_range(10, rank, world)
        stats = torch.zeros(5, 4, dtype=torch.int32)
        for i, f in enumerate(range(lo, hi)):
            stats[i, 0] = 1000 + f          # stand-in checksum of frame f
            stats[i, 1] = f
        allst = gather_frame_stats(stats)
        tmax = max_over_ranks(1.5 + rank)
        if rank == 0:
            q.put((allst.tolist(), tmax))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_gather_and_max():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    allst, tmax = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert tmax == 2.5
    assert [row[1] for row in allst] == list(range(10))
    assert [row[0] for row in allst] == [1000 + f for f in range(10)]
