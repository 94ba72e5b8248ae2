"""Multi-rank host logic of bench.py on CPU (gloo, world_size 2): replicas-only
aggregation (sum of units over the slowest rank's time) and the max-over-ranks timing."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench
    ms = 100.0 + 50.0 * rank  # rank 1 is slower
    units = 1e9 * (rank + 1)
    t = torch.tensor([ms, units], dtype=torch.float64)
    allt = [torch.zeros_like(t) for _ in range(world)]
    dist.all_gather(allt, t)
    value, tmax = bench.aggregate([float(x[0]) for x in allt], [float(x[1]) for x in allt])
    m = torch.tensor([ms], dtype=torch.float64)
    dist.all_reduce(m, op=dist.ReduceOp.MAX)
    q.put((rank, value, tmax, float(m)))
    dist.destroy_process_group()


def test_two_rank_aggregation():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    for rank, value, tmax, mx in res:
        assert tmax == 150.0 and mx == 150.0
        assert value == pytest.approx(3e9 / 0.150)


def test_aggregate_single():
    import bench
    v, t = bench.aggregate([10.0], [5e8])
    assert t == 10.0 and v == pytest.approx(5e10)
