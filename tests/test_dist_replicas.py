"""The N>1 bench path is "replicas only": every rank runs an
independent product; the job time is the max over ranks and the throughput is
world * per-rank work / that time.  Checked here with world_size 2 over gloo."""
import os

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench
    local_ms = [120.0, 150.0][rank]
    ms = bench.max_over_ranks(local_ms, dist, "cpu")
    value = bench.job_throughput(2.0e12, world, ms * 1e-3)
    q.put((rank, ms, value))
    dist.barrier()
    dist.destroy_process_group()


def test_replicas_max_over_ranks_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + os.getpid() % 1000
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert all(p.exitcode == 0 for p in procs)
    for rank, ms, value in out:
        assert ms == 150.0  # slowest rank
        assert value == pytest.approx(2 * 2.0e12 / 0.150 / 1e9)


def test_single_process_path():
    import bench
    assert bench.max_over_ranks(3.5, None, "cpu") == 3.5
    assert bench.job_throughput(1e12, 1, 2.0) == pytest.approx(500.0)
