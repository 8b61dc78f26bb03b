"""Host logic of bench.py's N > 1 path (replicas only):
max-over-ranks timing and whole-job throughput, on 2 gloo ranks (CPU)."""
import os
import socket

import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench
    local_s = [1.5, 2.25][rank]           # rank 1 is the slowest
    s_max = bench.reduce_max(local_s, dist, "cpu")
    rate = bench.whole_job_rate(1000.0, s_max, world)
    out[rank] = (s_max, rate)
    dist.barrier()
    dist.destroy_process_group()


def test_reduce_max_and_rate_two_gloo_ranks():
    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    for r in range(world):
        s_max, rate = out[r]
        assert s_max == 2.25                       # every rank sees the slowest rank's time
        assert rate == pytest.approx(2 * 1000.0 / 2.25)


def test_single_rank_identity():
    import bench
    assert bench.reduce_max(3.0, None) == 3.0
    assert bench.whole_job_rate(10.0, 2.0, 1) == 5.0
