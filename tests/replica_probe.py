"""Rank body for tests/test_replicas.py::test_launch_replicas_world2 (gloo, CPU): what each
bench.py rank does around its replica — barrier, local work, max-over-ranks aggregation."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch.distributed as dist  # noqa: E402

from paper_2401_05031_b200 import replicas  # noqa: E402

rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
dist.init_process_group("gloo")
dist.barrier()
items, ms = replicas.aggregate_throughput(100 * (rank + 1), 5.0 + rank)
per_rank = [None] * world
dist.all_gather_object(per_rank, {"rank": rank, "local_rank": int(os.environ["LOCAL_RANK"])})
if rank == 0:
    print(json.dumps({"world": world, "items": items, "ms": ms, "ranks": per_rank}), flush=True)
dist.barrier()
dist.destroy_process_group()
