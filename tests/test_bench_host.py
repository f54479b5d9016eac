"""bench.py's multi-rank host logic (replicas only) with two
gloo ranks on CPU: per-rank seeds differ, the job time is the max over ranks,
the value aggregates every rank's elements, and the reference arm prints only
on rank 0."""
import os
import socket
import sys

import pytest
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    import torch.distributed as dist

    import bench
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    ms = 10.0 + 5.0 * rank  # rank 1 is the slowest
    t = bench.max_over_ranks(ms, world, "cpu")
    seeds = [None] * world
    dist.all_gather_object(seeds, bench.rank_seed(1, rank))
    out.put((rank, t, bench.job_value(1 << 30, world, t), seeds))
    dist.destroy_process_group()


def test_two_gloo_ranks_max_time_and_job_value():
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
    for rank, t, v, seeds in res:
        assert t == 15.0                      # max over ranks, on every rank
        assert v == pytest.approx(2 * (1 << 30) / 0.015)
        assert len(set(seeds)) == world       # independent problems


def test_reference_arm_prints_on_rank0_only(capsys):
    import argparse

    import bench
    args = argparse.Namespace(workload="c1", ref_sample=1 << 12, warmup=0, steps=1, gpus=2)
    bench.run_reference(args, rank=1)
    assert capsys.readouterr().out == ""
    bench.run_reference(args, rank=0)
    line = capsys.readouterr().out
    assert '"impl": "reference"' in line and '"cpu_baseline"' in line
