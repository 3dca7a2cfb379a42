"""Query streams for the serving trace (SPEC.md:388-442 module ``workload``).

* ``PAPER_QUERY_TYPES``: the paper's query-type table: CIFAR10 /
  CIFAR100 / EuroSAT, latency budget 0.6 s or 1 s, utility 0.01..1.
* ``gen_poisson``: Poisson arrivals over a piecewise-constant rate profile (PAPER.md:617-621,
  "arrival time ... according to the Poisson distribution"), each query's type drawn from the
  weighted table, deadlines d_r = s_r + l_r.
* ``load_trace``: per-second counts (MAF-style) expanded into arrivals at
  (j + 1) / (k + 1) of each second (uniform) or jittered.
Streams are sorted by arrival and deterministic per seed; times are integer microseconds.
"""

from __future__ import annotations

import random
from dataclasses import dataclass
from typing import List, Sequence, Tuple

from .core import Query, us_from_s
from .errors import ConfigError

__all__ = ["QueryType", "PAPER_QUERY_TYPES", "gen_poisson", "load_trace", "expand_counts"]


@dataclass(frozen=True)
class QueryType:
    type_id: int
    task: str
    budget_us: int
    utility: float
    weight: float = 1.0


PAPER_QUERY_TYPES: Tuple[QueryType, ...] = (
    QueryType(1, "CIFAR10", us_from_s(0.6), 0.3),
    QueryType(2, "CIFAR10", us_from_s(1.0), 0.01),
    QueryType(3, "CIFAR100", us_from_s(0.6), 1.0),
    QueryType(4, "CIFAR100", us_from_s(1.0), 0.2),
    QueryType(5, "EuroSAT", us_from_s(0.6), 0.3),
    QueryType(6, "EuroSAT", us_from_s(1.0), 0.01),
)


def _check_types(types: Sequence[QueryType]) -> None:
    if not types:
        raise ConfigError("query type table must not be empty")
    if any(t.weight <= 0 for t in types):
        raise ConfigError("query type weights must be positive")


def _pick(rng: random.Random, types: Sequence[QueryType]) -> QueryType:
    return rng.choices(types, weights=[t.weight for t in types], k=1)[0]


def gen_poisson(rate_profile: Sequence[Tuple[float, float]], duration_s: float,
                types: Sequence[QueryType] = PAPER_QUERY_TYPES, seed: int = 0,
                first_id: int = 0) -> List[Query]:
    """``rate_profile``: [(start second, requests/s), ...] sorted by start; the last rate holds
    until ``duration_s``.  Exponential gaps within each segment (memoryless, so restarting the
    draw at a segment boundary keeps the process Poisson)."""
    _check_types(types)
    if any(r < 0 for _, r in rate_profile):
        raise ConfigError("rates must be nonnegative")
    rng = random.Random(seed)
    out: List[Query] = []
    qid = first_id
    segs = list(rate_profile) + [(duration_s, 0.0)]
    for (start, rate), (end, _) in zip(segs, segs[1:]):
        end = min(end, duration_s)
        if rate <= 0 or end <= start:
            continue
        t = start
        while True:
            t += rng.expovariate(rate)
            if t >= end:
                break
            qt = _pick(rng, types)
            out.append(Query(qid, qt.task, us_from_s(t), qt.budget_us, qt.utility))
            qid += 1
    return out


def expand_counts(counts: Sequence[int], types: Sequence[QueryType] = PAPER_QUERY_TYPES,
                  seed: int = 0, spreading: str = "uniform") -> List[Query]:
    """Second i with k requests -> k arrivals in [i, i + 1): at (j + 1) / (k + 1) (uniform) or
    uniform-random offsets (jittered), sorted."""
    _check_types(types)
    if spreading not in ("uniform", "jittered"):
        raise ConfigError("spreading must be 'uniform' or 'jittered'")
    rng = random.Random(seed)
    out: List[Query] = []
    qid = 0
    for sec, k in enumerate(counts):
        if k < 0:
            raise ConfigError(f"negative count in second {sec}")
        offs = [(j + 1) / (k + 1) for j in range(k)] if spreading == "uniform" else sorted(rng.random() for _ in range(k))
        for off in offs:
            qt = _pick(rng, types)
            out.append(Query(qid, qt.task, us_from_s(sec + off), qt.budget_us, qt.utility))
            qid += 1
    return out


def load_trace(path: str, types: Sequence[QueryType] = PAPER_QUERY_TYPES, seed: int = 0,
               spreading: str = "uniform") -> List[Query]:
    """One nonnegative integer per line = requests in that second."""
    counts: List[int] = []
    with open(path, encoding="utf-8") as fh:
        for n, line in enumerate(fh, 1):
            s = line.strip()
            if not s:
                continue
            try:
                v = int(s)
            except ValueError:
                raise ConfigError(f"{path}:{n}: not an integer: {s!r}") from None
            if v < 0:
                raise ConfigError(f"{path}:{n}: negative count")
            counts.append(v)
    return expand_counts(counts, types, seed, spreading)
