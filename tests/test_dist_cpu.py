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


# ---- bench.py's multi-rank report path (shard -> timed stats -> gather ->
# per-frame oracle check on rank 0), driven with a stubbed step over gloo
def _bench_worker(rank, world, port, q, corrupt):
    import torch.distributed as dist
    import bench
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        B = 6
        f0, f1 = shard_range(world * B, rank, world)
        sigs = {i: (0xA0000000 + 17 * i, 1000 + i) for i in range(bench.POOL)}   # stand-in oracle
        stats = torch.zeros(B, 4, dtype=torch.int32)
        for k, f in enumerate(range(f0, f1)):          # the stubbed step: frame f = pool[f % POOL]
            cs, valid = sigs[f % bench.POOL]
            stats[k, 0] = torch.tensor(cs, dtype=torch.int64).to(torch.int32)
            stats[k, 1] = valid
            if f == corrupt:
                stats[k, 1] += 1
        calls = []

        def sigs_fn():
            calls.append(rank)
            return sigs

        ms_max, allst, parity = bench.gather_and_check(stats, 10.0 + rank, sigs_fn)
        q.put((rank, ms_max, allst.shape[0], parity, calls))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("corrupt", [-1, 9])
def test_gloo_world2_bench_report_path(corrupt):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_bench_worker, args=(r, 2, port, q, corrupt)) for r in range(2)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(2):
        r, ms_max, nrows, parity, calls = q.get(timeout=120)
        res[r] = (ms_max, nrows, parity, calls)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert res[0][0] == res[1][0] == 11.0            # max over ranks
    assert res[0][1] == res[1][1] == 12              # every frame of the job gathered
    assert res[1][2] is None and res[1][3] == []     # only rank 0 consults the oracle
    par = res[0][2]
    assert res[0][3] == [0] and par["frames"] == 12
    if corrupt < 0:
        assert par["mismatches"] == 0
    else:
        assert par["mismatches"] == 1 and par["first_bad"] == [corrupt]
