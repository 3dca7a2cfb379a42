"""Selective batcher: Algorithm 1 of the paper ("Batching Algorithm: Adding a Query into a
Batch"; SPEC.md:183-234 module ``batcher``).

A query joins the newest compatible batch: the scan runs newest -> oldest, stops at the first
batch that has waited longer than delta (``s_b + delta < s_r``, Alg. 1 line 2), and skips
batches that are full (``|B_b| >= epsilon``), whose deadline differs by more than eta, or whose
anchor utility differs by more than mu.  Otherwise a new singleton batch is opened.  All
times are integer microseconds (core.py:3-5).  Host-side Python, as in the reference.
"""

from __future__ import annotations

from dataclasses import dataclass, field
from typing import Iterator, List, Optional

from .core import Batch, Query, us_from_s
from .errors import ConfigError

__all__ = ["BatchingThresholds", "BatchQueue", "add_query"]


@dataclass(frozen=True)
class BatchingThresholds:
    """delta (max wait), epsilon (max batch), eta (deadline spread), mu (utility spread)."""

    max_wait_us: int
    max_batch: int
    deadline_spread_us: int
    utility_spread: float

    def __post_init__(self) -> None:
        if self.max_wait_us < 0 or self.deadline_spread_us < 0:
            raise ConfigError("batching delta / eta must be nonnegative")
        if self.max_batch < 1:
            raise ConfigError("batching epsilon must be at least 1")
        if self.utility_spread < 0:
            raise ConfigError("batching mu must be nonnegative")

    @classmethod
    def paper(cls) -> "BatchingThresholds":
        """PAPER.md §V: delta, epsilon, eta, mu = 0.5 s, 64, 0.5 s, 0.8."""
        return cls(us_from_s(0.5), 64, us_from_s(0.5), 0.8)


@dataclass
class BatchQueue:
    """Admission-ordered batches not yet handed to the engine."""

    batches: List[Batch] = field(default_factory=list)
    next_batch_id: int = 0
    last_arrival_us: Optional[int] = None

    def __len__(self) -> int:
        return len(self.batches)

    def __iter__(self) -> Iterator[Batch]:
        return iter(self.batches)

    def add_query(self, r: Query, th: BatchingThresholds) -> Batch:
        """Alg. 1; returns the batch that received ``r``."""
        if self.last_arrival_us is not None and r.arrival_us < self.last_arrival_us:
            raise ValueError(f"query {r.id} arrives before an already admitted query")
        self.last_arrival_us = r.arrival_us
        for b in reversed(self.batches):  # for b in [N_B, 1]
            if b.arrival_us + th.max_wait_us < r.arrival_us:
                break  # this and every older batch waited too long
            if b.size >= th.max_batch:
                continue
            if abs(b.deadline_us - r.deadline_us) > th.deadline_spread_us:
                continue
            if abs(b.anchor_utility - r.utility) > th.utility_spread:
                continue
            b.add(r)
            return b
        nb = Batch(self.next_batch_id, [r])
        self.next_batch_id += 1
        self.batches.append(nb)
        return nb

    def remove(self, batch: Batch) -> None:
        """The engine takes ownership of ``batch`` (executing or evicted); admission never
        reopens it."""
        self.batches.remove(batch)


def add_query(queue: BatchQueue, r: Query, th: BatchingThresholds) -> BatchQueue:
    """Functional form of SPEC.md:205 (mutates and returns ``queue``)."""
    queue.add_query(r, th)
    return queue
