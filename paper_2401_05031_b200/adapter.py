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

__all__ = ["AdapterConfig", "PAPER_GAMMAS", "PAPER_RATE_MAP", "allocate", "allocate_single_state",
           "manual_allocate", "brute_force_oracle", "plan_utility"]

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
             mem: Optional[MemoryModel], rate_per_s: float, initial_stage: bool = False,
             frontier_cap: int = 256) -> TokenPlan:
    """Alg. 2 over the EDF-sorted queue snapshot at clock ``now_us``.

    The DP table is Alg. 2's (batch b, column l) grid with column 0 = skip, the same
    feasibility test ``C + t_hat < d_b`` plus the memory bound, and backtracking through
    predecessor pointers.  One deviation, required by SPEC.md:268 / :597 (``allocate`` must
    equal ``brute_force_oracle`` exactly on every instance): each cell keeps the Pareto
    frontier of (utility, clock) states instead of a single (dp, C) pair.  With one pair per
    cell, a state with more utility but a later clock can displace the state that lets a later
    batch meet its deadline, and the plan is then suboptimal (13 of the 200 seeded instances of
    tests/test_serving.py with the literal table, ``allocate_single_state``).  A state is pruned
    only when another state of the same batch (any column) has utility >= and clock <=
    (floating-point addition is monotone, so no pruned state can lead to a better plan), which
    makes the result exact.  ``frontier_cap`` bounds a row's frontier (kept: highest utility
    first); it is not reached at the sizes of the acceptance test (N_B <= 6, N_gamma <= 4), and
    the serving engine passes a small cap to bound planning time in real time.
    """
    order = _edf(batches)
    if not order:
        return TokenPlan({}, 0.0)
    if len(order) <= cfg.min_queue or initial_stage:
        return manual_allocate(order, now_us, cfg, table, rate_per_s)
    nb, ng = len(order), cfg.gammas.size
    # state = (utility, clock, column, predecessor index into the previous row's state list)
    prev_states: List[Tuple[float, float, int, int]] = [(0.0, float(now_us), 0, -1)]
    rows: List[List[Tuple[float, float, int, int]]] = []
    for bi in range(nb):
        b = order[bi]
        est = [None] + [estimate_batch(b, cfg.gammas.at_column(l), table) for l in range(1, ng + 1)]
        mem_ok = [True] + [_mem_ok(b, cfg.gammas.at_column(l), mem, table) for l in range(1, ng + 1)]
        # The states of every column of this batch form one frontier: a state's future (what later
        # batches can still do) depends only on its (utility, clock), not on the column it came
        # from, so a state dominated by one of another column is dropped too.
        cand: List[Tuple[float, float, int, int]] = []
        for l in range(ng + 1):
            for pi, (u_prev, c_prev, _, _) in enumerate(prev_states):
                if l == 0:  # skip: utility and clock carried forward (Alg. 2 lines 14-19)
                    cand.append((u_prev, c_prev, 0, pi))
                else:
                    t_hat, u_hat = est[l]
                    if c_prev + t_hat < b.deadline_us and mem_ok[l]:  # Alg. 2 line 23
                        cand.append((u_prev + u_hat, c_prev + t_hat, l, pi))
        row = _pareto(cand, frontier_cap)
        rows.append(row)
        prev_states = row
    # argmax of utility; exact ties -> lexicographically smallest column vector (the oracle's rule)
    best_u = max(st[0] for st in prev_states)

    def columns(idx: int) -> List[int]:
        cols = [0] * nb
        for bi in range(nb - 1, -1, -1):
            u, c, l, p = rows[bi][idx]
            cols[bi] = l
            idx = p
        return cols

    cands = [columns(i) for i, st in enumerate(prev_states) if st[0] == best_u]
    cols = min(cands)
    plan = {order[bi].id: (None if cols[bi] == 0 else cfg.gammas.at_column(cols[bi])) for bi in range(nb)}
    return TokenPlan(plan, plan_utility(order, plan, now_us, table, mem))


def _pareto(cell: List[Tuple[float, float, int, int]], cap: int) -> List[Tuple[float, float, int, int]]:
    """Non-dominated (utility up, clock down) states of one DP row; exact ties keep the state
    with the lower column, then the earlier predecessor (Alg. 2's strict-improvement order)."""
    keep: List[Tuple[float, float, int, int]] = []
    for st in sorted(cell, key=lambda s: (-s[0], s[1], s[2], s[3])):
        if keep and keep[-1][1] <= st[1]:
            continue  # an earlier-kept state has utility >= and clock <=
        keep.append(st)
        if len(keep) >= cap:
            break
    return keep


def allocate_single_state(batches: Sequence[Batch], now_us: int, cfg: AdapterConfig,
                          table: ProfileTable, mem: Optional[MemoryModel]) -> TokenPlan:
    """Alg. 2's DP exactly as printed (one (dp, C) pair per cell, strict improvement), kept to
    document why ``allocate`` carries frontiers: it is feasible but not always optimal.  Rows
    b >= 1 start at -inf (Alg. 2's all-zero / S=1 initialisation would backtrack a never-
    feasible batch to L[1])."""
    order = _edf(batches)
    if not order:
        return TokenPlan({}, 0.0)
    nb, ng = len(order), cfg.gammas.size
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
