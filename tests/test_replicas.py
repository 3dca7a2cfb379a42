"""Replica host logic: dispatch invariants, and the max-over-ranks /
sum-of-images aggregation bench.py uses, run with world_size 2 over gloo on CPU."""

import os
import socket

import pytest
import torch.multiprocessing as mp

from paper_2401_05031_b200 import replicas


def test_round_robin():
    a = replicas.round_robin(10, 4)
    assert a == [[0, 4, 8], [1, 5, 9], [2, 6], [3, 7]]
    assert sorted(sum(a, [])) == list(range(10))
    with pytest.raises(ValueError):
        replicas.round_robin(3, 0)


def test_next_free():
    from paper_2401_05031_b200.replicas import next_free

    assert next_free([5, 3, 3, 9]) == 1
    assert next_free([0]) == 0
    with pytest.raises(ValueError):
        next_free([])


def test_earliest_free():
    assign, finish = replicas.earliest_free([100, 50, 50, 10, 200], 2)
    assert assign == [[0, 3], [1, 2, 4]]
    assert finish == [100, 50, 100, 110, 300]
    # with arrival times: idle replicas wait for the batch
    assign, finish = replicas.earliest_free([10, 10], 2, ready_us=[0, 100])
    assert finish == [10, 110]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    items, ms = replicas.aggregate_throughput(256 * (rank + 1), 10.0 + rank)
    q.put((rank, items, ms))
    dist.barrier()
    dist.destroy_process_group()


def test_aggregate_gloo_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    res = sorted(q.get(timeout=10) for _ in range(2))
    for rank, items, ms in res:
        assert items == 256 + 512 and ms == 11.0


def test_aggregate_single_process():
    assert replicas.aggregate_throughput(5, 2.5) == (5.0, 2.5)


def test_launch_replicas_world2():
    """The spawn path of `bench.py --gpus N` (no launcher in the environment): N ranks over
    torch.distributed.run on 127.0.0.1, rank 0 prints the aggregated line."""
    import json

    probe = os.path.join(os.path.dirname(os.path.abspath(__file__)), "replica_probe.py")
    env_keep = os.environ.pop("WORLD_SIZE", None)
    try:
        res = replicas.launch_replicas(2, probe, [], capture=True, timeout=300)
    finally:
        if env_keep is not None:
            os.environ["WORLD_SIZE"] = env_keep
    assert res.returncode == 0, res.stderr[-2000:]
    lines = [l for l in res.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    out = json.loads(lines[0])
    assert out["world"] == 2 and out["items"] == 300.0 and out["ms"] == 6.0
    assert sorted(r["local_rank"] for r in out["ranks"]) == [0, 1]
