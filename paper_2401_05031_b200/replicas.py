"""Multi-GPU serving is replicas only (north_star): every GPU holds a full
model, batches are dispatched host-side, and nothing crosses NVLink on the data path.

This module holds the host logic around that: deterministic batch -> replica assignment
(round robin for throughput sweeps, earliest-free for a serving trace), and the
barrier-aligned throughput aggregation used by bench.py (images summed over ranks, device
time = max over ranks).  The reduction is plumbing over torch.distributed (gloo on the
host side), never a collective on the forward path.
"""

from __future__ import annotations

import heapq
import os
import socket
import subprocess
import sys
from typing import List, Optional, Sequence, Tuple

__all__ = ["round_robin", "earliest_free", "next_free", "aggregate_throughput", "launch_replicas", "free_port"]


def round_robin(n_batches: int, world: int) -> List[List[int]]:
    """Batch ids per replica: batch i -> replica i mod world."""
    if world < 1:
        raise ValueError("world must be >= 1")
    out: List[List[int]] = [[] for _ in range(world)]
    for i in range(n_batches):
        out[i % world].append(i)
    return out


def next_free(free_at_us: Sequence[int]) -> int:
    """The replica that frees up first (ties -> lowest replica id): the dispatch rule of
    ``earliest_free`` for one batch, used by the serving engine (engine.py)."""
    if not free_at_us:
        raise ValueError("no replicas")
    return min(range(len(free_at_us)), key=lambda i: (free_at_us[i], i))


def earliest_free(costs_us: Sequence[int], world: int,
                  ready_us: Optional[Sequence[int]] = None) -> Tuple[List[List[int]], List[int]]:
    """List scheduling in batch order: each batch goes to the replica that frees up first
    (ties -> lowest replica id).  Returns (batch ids per replica, finish time per batch)."""
    if world < 1:
        raise ValueError("world must be >= 1")
    heap = [(0, r) for r in range(world)]
    heapq.heapify(heap)
    assign: List[List[int]] = [[] for _ in range(world)]
    finish = [0] * len(costs_us)
    for i, c in enumerate(costs_us):
        free_at, r = heapq.heappop(heap)
        start = max(free_at, ready_us[i] if ready_us is not None else 0)
        finish[i] = start + int(c)
        assign[r].append(i)
        heapq.heappush(heap, (finish[i], r))
    return assign, finish


def aggregate_throughput(local_items: float, local_ms: float, group=None) -> Tuple[float, float]:
    """(total items over ranks, max device ms over ranks) -> the job's items/s is
    total / (max_ms / 1e3).  Single-process when torch.distributed is not initialised."""
    import torch
    import torch.distributed as dist

    if not (dist.is_available() and dist.is_initialized()):
        return float(local_items), float(local_ms)
    items = torch.tensor([float(local_items)], dtype=torch.float64)
    ms = torch.tensor([float(local_ms)], dtype=torch.float64)
    dist.all_reduce(items, op=dist.ReduceOp.SUM, group=group)
    dist.all_reduce(ms, op=dist.ReduceOp.MAX, group=group)
    return float(items.item()), float(ms.item())


def free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def launch_replicas(n: int, script: str, argv: Sequence[str], capture: bool = False,
                    timeout: Optional[float] = None) -> subprocess.CompletedProcess:
    """Run `script argv` as n ranks, one process (and replica) per GPU, through
    torch.distributed.run on 127.0.0.1 (what `bench.py --gpus N` does when it is started
    without a launcher).  Each rank reads RANK / LOCAL_RANK / WORLD_SIZE from the env; the
    ranks only share a host-side (gloo) barrier and the throughput reduction."""
    if n < 1:
        raise ValueError("n must be >= 1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(free_port()), script, *argv]
    env = dict(os.environ)
    env.setdefault("OMP_NUM_THREADS", "1")
    return subprocess.run(cmd, env=env, capture_output=capture, text=True, timeout=timeout)
