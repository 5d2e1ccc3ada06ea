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


def test_self_launch_gloo_world2():
    """`bench.py --gpus 2` without a torchrun environment launches the two rank
    processes itself (RANK / WORLD_SIZE / MASTER_* set per rank) and reports
    n_gpus == 2 with the whole-job value over the max-over-ranks time."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    r = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", "2", "--impl", "plumbing"],
                       capture_output=True, text=True, timeout=300, env=env)
    assert r.returncode == 0, r.stderr
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["n_gpus"] == 2
    assert line["value"] == pytest.approx(2 * 10.0 / 0.150)


def test_world_size_must_match_gpus():
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, WORLD_SIZE="1", RANK="0", LOCAL_RANK="0")
    r = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", "2", "--impl", "plumbing"],
                       capture_output=True, text=True, timeout=120, env=env)
    assert r.returncode != 0 and "WORLD_SIZE" in r.stderr
