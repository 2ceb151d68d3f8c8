"""N>1 path of bench.py on CPU: world_size-2 gloo ranks (replicas only, no
data-path collective; the timed duration is the max over ranks)."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import bench


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK=str(rank))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    r, w, l = bench.dist_env()
    ms = 10.0 + 5.0 * rank            # rank 1 is the slow one
    tot = bench.max_over_ranks(ms, w, torch.device("cpu"))
    val = bench.job_throughput(2.0e9, 4, w, tot)
    q.put((r, w, l, tot, val))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_gloo_replicas():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, (r, w, l, tot, val) in enumerate(res):
        assert (r, w, l) == (rank, 2, rank)
        assert tot == pytest.approx(15.0)                 # max over ranks
        assert val == pytest.approx(2.0e9 * 4 * 2 / 0.015)  # all ranks' units / max time


def test_single_rank_passthrough():
    assert bench.max_over_ranks(12.5, 1) == 12.5
    assert bench.job_throughput(1e9, 10, 1, 1000.0) == pytest.approx(1e10)
