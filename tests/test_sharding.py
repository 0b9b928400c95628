"""Sequence sharding across ranks and the final stats gather, run as a real
world_size-2 process group on the gloo backend (CPU)."""
import os
import socket

import pytest
import torch.multiprocessing as mp

from paper_1809_07986_b200.sharding import RankStats, gather_stats, job_throughput, shard


@pytest.mark.parametrize("n,world", [(64, 1), (64, 2), (64, 8), (7, 3), (3, 4), (0, 2)])
def test_shards_partition_the_batch(n, world):
    got = [list(shard(n, world, r)) for r in range(world)]
    flat = [i for g in got for i in g]
    assert flat == list(range(n))  # contiguous, ordered, disjoint, complete
    sizes = [len(g) for g in got]
    assert max(sizes) - min(sizes) <= 1


def test_bad_rank_rejected():
    with pytest.raises(ValueError):
        shard(4, 2, 2)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    mine = shard(64, world, rank)
    st = RankStats(rank, len(mine), 30 * len(mine), 1e9 * (rank + 1), 100.0 + 10 * rank)
    all_st = gather_stats(st)
    if rank == 0:
        q.put((sorted(s.rank for s in all_st), job_throughput(all_st),
               [s.sequences for s in all_st]))
    dist.barrier()
    dist.destroy_process_group()


def test_gather_over_two_gloo_ranks():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    ranks, thr, seqs = q.get(timeout=120)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert ranks == [0, 1]
    assert seqs == [32, 32]
    assert thr["max_device_ms"] == 110.0  # max over ranks
    assert thr["frames"] == 64 * 30
    assert abs(thr["frames_per_s"] - 64 * 30 / 0.110) < 1e-6
