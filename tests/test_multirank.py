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


def test_bench_gpus_flag_relaunches_ranks_cpu():
    """`python bench.py --gpus 2` outside torchrun re-launches itself as 2 ranks (one process per
    GPU); the CPU self-test runs the GPU arm's multi-rank skeleton (init, barrier, per-rank timing
    all_gather, max-over-ranks aggregation) on gloo and reports n_gpus = 2."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    r = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", "2", "--selftest-cpu",
                        "--config", "tiny", "--steps", "1", "--warmup", "3"], capture_output=True, text=True,
                       env=env, timeout=300, cwd=root)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1  # rank 0 alone prints
    line = json.loads(lines[0])
    assert line["n_gpus"] == 2 and len(line["per_rank_ms"]) == 2
    assert line["ms_per_step"] == pytest.approx(max(line["per_rank_ms"]))
    assert line["value"] == pytest.approx(3e6 / (max(line["per_rank_ms"]) / 1e3) / 1e9)
