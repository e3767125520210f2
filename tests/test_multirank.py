"""World-size-2 checks of the replica path on CPU (gloo): bench.py's max-over-ranks
timing reduction and per-rank scene replicas (replicas only)."""

import os
import socket

import pytest
import torch.multiprocessing as mp

from conftest import ROOT


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, out):
    import sys

    import torch.distributed as dist

    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench
    from paper_2007_01941_b200 import scenes

    # each replica solves its own problem; the job time is the slowest rank
    t = bench.max_over_ranks(10.0 + rank, world)
    sc = scenes.random_problem(2000 + rank, n_cameras=6, n_points=20)
    out[rank] = (t, sc.digest())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.timeout(120)
def test_replicas_max_over_ranks_gloo():
    world = 2
    with mp.Manager() as m:
        out = m.dict()
        mp.spawn(_worker, args=(world, _free_port(), out), nprocs=world, join=True)
        res = dict(out)
    assert res[0][0] == res[1][0] == 11.0
    assert res[0][1] != res[1][1]  # independent replicas
