"""CPU: the multi-GPU story is replicas only.  This exercises
the N>1 host logic bench.py relies on -- rank/world from the environment,
barrier, MAX-over-ranks timing and SUM-over-ranks work -- with the gloo
backend, world_size 2, each rank running its own (oracle) sequence replica."""

import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _replica(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port),
                      RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import sys
    repo = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, repo)
    import time
    from oracle.api import oracle_api
    from paper_1406_2831_b200.sequence import run_sequence
    from paper_1406_2831_b200.workloads import make_sequence
    dist.barrier()
    t0 = time.perf_counter()
    res = run_sequence(make_sequence("c1", small=True), baseline=False,
                       api=oracle_api(), systems=2)
    dt = time.perf_counter() - t0
    t = torch.tensor([dt, float(res.recycling.total_iterations)], dtype=torch.float64)
    mx, sm = t.clone(), t.clone()
    dist.all_reduce(mx, op=dist.ReduceOp.MAX)
    dist.all_reduce(sm, op=dist.ReduceOp.SUM)
    out[rank] = (float(mx[0]), float(sm[1]), res.recycling.total_iterations,
                 [h.resid for h in res.recycling.histories])
    dist.barrier()
    dist.destroy_process_group()


def test_two_replicas_gloo():
    world = 2
    port = _free_port()
    with mp.Manager() as m:
        out = m.dict()
        mp.spawn(_replica, args=(world, port, out), nprocs=world, join=True)
        r0, r1 = out[0], out[1]
    # max-over-ranks time and sum-over-ranks iterations agree on every rank
    assert r0[0] == r1[0] and r0[1] == r1[1]
    assert r0[1] == r0[2] + r1[2]
    # replicas are independent copies of the same deterministic sequence
    assert r0[3] == r1[3]
