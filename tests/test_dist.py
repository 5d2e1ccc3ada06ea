"""bench.py's multi-process plumbing (replicas only: barrier + max-over-ranks
time + whole-job value), world_size 2 over gloo on CPU."""
import os
import socket

import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
    import bench
    w, r, _ = bench.dist_setup("gloo")
    assert (w, r) == (world, rank)
    bench.barrier(w)
    # rank r "took" 100 + 50 r ms for 10 units: value = world * 10 / max time
    v = bench.replica_value(10.0, 100.0 + 50.0 * rank, w)
    out[rank] = v
    import torch.distributed as dist
    dist.destroy_process_group()


def test_replicas_gloo_world2():
    world = 2
    port = _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, port, out), nprocs=world, join=True)
    expect = world * 10.0 / 0.150
    assert out[0] == pytest.approx(expect) and out[1] == pytest.approx(expect)
