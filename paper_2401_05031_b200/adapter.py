"""Token adapter (utility optimiser): Algorithm 2 "Autonomous Token Adaptation Algorithm"
(PAPER.md:388-443), Algorithm 3 "Manually_Allocate" and an exhaustive
oracle for testing (SPEC.md:236-315 module ``adapter``).

The plan maps every queued batch to a gamma or to ``None`` (= skip: the engine evicts its
queries).  Planned utility is the expectation sum_r accuracy(task_r, gamma) * u_r and the time
model is the profiled one (``profiles.estimate_batch``), both in integer microseconds.  The
DP follows Alg. 2 literally: one (utility, clock) per (batch, column) cell, strict
improvement (earlier predecessor columns win ties), column 0 = skip carrying the best
predecessor forward, infeasible columns poisoned to -inf / +inf (one deviation: rows b >= 1
start at -inf instead of 0, see ``allocate``).  Host-side Python, as in the
reference; the gamma it picks is what ``ServeModel.forward`` executes on the GPU.
"""

from __future__ import annotations

import itertools
from dataclasses import dataclass
from typing import Dict, List, Optional, Sequence, Tuple

from .core import Batch, GammaList, TokenPlan, us_from_s
from .errors import ConfigError
from .profiles import MemoryModel, ProfileTable, RateToGammaMap, batch_memory, estimate_batch, project_rate

__all__ = ["AdapterConfig", "PAPER_GAMMAS", "PAPER_RATE_MAP", "allocate", "manual_allocate",
           "brute_force_oracle", "plan_utility"]

NEG_INF = float("-inf")

# PAPER.md:546 and the rate -> gamma table
PAPER_GAMMAS = GammaList((-20, -15, -10, -5, 0, 2, 4, 8))
PAPER_RATE_MAP = RateToGammaMap(((1, 8), (280, 4), (320, 2), (350, 0), (380, -5), (450, -10),
                                 (520, -15), (1000, -20)))


@dataclass(frozen=True)
class AdapterConfig:
    """beta, initial stage, kappa, the gamma list and the rate map f."""

    gammas: GammaList = PAPER_GAMMAS
    rate_map: RateToGammaMap = PAPER_RATE_MAP
    min_queue: int = 5                       # beta
    initial_stage_us: int = us_from_s(2.0)   # "the first 2 seconds of the service"
    utility_threshold: float = 0.8           # kappa
    rate_window_us: int = us_from_s(1.0)     # "the previous inference window"

    def __post_init__(self) -> None:
        if self.min_queue < 1:
            raise ConfigError("beta must be at least 1")
        if self.utility_threshold < 0:
            raise ConfigError("kappa must be nonnegative")
        if self.rate_window_us <= 0:
            raise ConfigError("rate window must be positive")
        self.rate_map.validate_against(self.gammas)


def _edf(batches: Sequence[Batch]) -> List[Batch]:
    return sorted(batches, key=lambda b: (b.deadline_us, b.id))


def _mem_ok(batch: Batch, gamma: int, mem: Optional[MemoryModel], table: ProfileTable) -> bool:
    return mem is None or batch_memory(batch, gamma, mem, table) < mem.gpu_capacity_bytes


def manual_allocate(batches: Sequence[Batch], now_us: int, cfg: AdapterConfig, table: ProfileTable,
                    rate_per_s: float) -> TokenPlan:
    """Alg. 3: base gamma = f(q); a batch that would miss its deadline at the base gamma gets
    min(L); a batch whose mean utility exceeds kappa gets max(L); the clock advances by the
    estimated time of the assigned gamma."""
    base = project_rate(rate_per_s, cfg.rate_map)
    clock = now_us
    plan: Dict[int, Optional[int]] = {}
    expected = 0.0
    for b in _edf(batches):
        t_base, _ = estimate_batch(b, base, table)
        mean_u = sum(q.utility for q in b.queries) / b.size
        if clock + t_base >= b.deadline_us:
            gamma = cfg.gammas.minimum
        elif mean_u > cfg.utility_threshold:
            gamma = cfg.gammas.maximum
        else:
            gamma = base
        t, u = estimate_batch(b, gamma, table)
        plan[b.id] = gamma
        expected += u
        clock += t
    return TokenPlan(plan, expected)


def allocate(batches: Sequence[Batch], now_us: int, cfg: AdapterConfig, table: ProfileTable,
             mem: Optional[MemoryModel], rate_per_s: float, initial_stage: bool = False) -> TokenPlan:
    """Alg. 2 over the EDF-sorted queue snapshot at clock ``now_us``."""
    order = _edf(batches)
    if not order:
        return TokenPlan({}, 0.0)
    if len(order) <= cfg.min_queue or initial_stage:
        return manual_allocate(order, now_us, cfg, table, rate_per_s)
    nb, ng = len(order), cfg.gammas.size
    # Alg. 2 initialises every cell of dp to 0 and S to 1; with the strict-improvement updates
    # that leaves a skip cell whose predecessors all have utility 0 pointing at column 1, and
    # backtracking then assigns L[1] to a batch that was never feasible.  Rows b >= 1 start
    # at -inf here (row 0 = 0 as in Alg. 2), so every reachable cell records its predecessor.
    dp = [[0.0] * (ng + 1)] + [[NEG_INF] * (ng + 1) for _ in range(nb)]
    S = [[0] * (ng + 1) for _ in range(nb + 1)]
    C = [[now_us] * (ng + 1) for _ in range(nb + 1)]
    for bi in range(1, nb + 1):
        b = order[bi - 1]
        est = [None] + [estimate_batch(b, cfg.gammas.at_column(l), table) for l in range(1, ng + 1)]
        mem_ok = [True] + [_mem_ok(b, cfg.gammas.at_column(l), mem, table) for l in range(1, ng + 1)]
        for l in range(ng + 1):
            J = False
            for lp in range(ng + 1):
                prev = dp[bi - 1][lp]
                if prev == NEG_INF:
                    continue
                if l == 0:
                    if prev > dp[bi][l]:
                        dp[bi][l], S[bi][l], C[bi][l] = prev, lp, C[bi - 1][lp]
                    J = True
                else:
                    t_hat, u_hat = est[l]
                    if C[bi - 1][lp] + t_hat < b.deadline_us and mem_ok[l]:
                        u = prev + u_hat
                        J = True
                        if u > dp[bi][l]:
                            dp[bi][l], S[bi][l], C[bi][l] = u, lp, C[bi - 1][lp] + t_hat
            if l > 0 and not J:
                dp[bi][l], C[bi][l] = NEG_INF, float("inf")
    last = dp[nb]
    col = max(range(ng + 1), key=lambda l: (last[l], -l))  # argmax, first on ties
    cols = [0] * (nb + 1)
    cols[nb] = col
    for bi in range(nb - 1, 0, -1):
        cols[bi] = S[bi + 1][cols[bi + 1]]
    plan = {order[bi - 1].id: (None if cols[bi] == 0 else cfg.gammas.at_column(cols[bi]))
            for bi in range(1, nb + 1)}
    return TokenPlan(plan, plan_utility(order, plan, now_us, table, mem))


def plan_utility(batches: Sequence[Batch], plan: Dict[int, Optional[int]], now_us: int,
                 table: ProfileTable, mem: Optional[MemoryModel]) -> float:
    """Replays ``plan`` in EDF order from ``now_us``: expected utility, or -inf when an executed
    batch misses ``C + t < d_b`` or the memory bound (the feasibility rule of Alg. 2)."""
    clock, total = now_us, 0.0
    for b in _edf(batches):
        gamma = plan[b.id]
        if gamma is None:
            continue
        t, u = estimate_batch(b, gamma, table)
        if not (clock + t < b.deadline_us and _mem_ok(b, gamma, mem, table)):
            return NEG_INF
        clock += t
        total += u
    return total


def brute_force_oracle(batches: Sequence[Batch], now_us: int, gammas: GammaList, table: ProfileTable,
                       mem: Optional[MemoryModel]) -> Tuple[float, TokenPlan]:
    """Every column assignment (0 = skip) in lexicographic order under the same timeline and
    feasibility rules; the first strict maximum wins."""
    order = _edf(batches)
    n = len(order)
    if (gammas.size + 1) ** n > 10 ** 7:
        raise ConfigError("brute-force search space exceeds 1e7 assignments")
    best, best_plan = NEG_INF, None
    for cols in itertools.product(range(gammas.size + 1), repeat=n):
        plan = {b.id: (None if c == 0 else gammas.at_column(c)) for b, c in zip(order, cols)}
        u = plan_utility(order, plan, now_us, table, mem)
        if u > best:
            best, best_plan = u, plan
    return best, TokenPlan(best_plan or {}, best)
