"""Serving engine: arrivals -> selective batcher (Alg. 1) -> token adapter (Alg. 2/3) ->
execution of the planned batches on B200 replicas (PAPER.md:251-270 pipeline; SPEC.md:317-386
module ``engine``, SPEC.md:444-492 module ``metrics``).

The loop is a deterministic discrete-event loop on the integer-microsecond clock.  Whenever a
replica is free and batches are queued, the adapter plans gamma for the queue snapshot (replan
per batch), skipped batches are evicted (Type 4), and the earliest-deadline planned batch runs
on the earliest-free replica; a batch whose estimated finish already misses its deadline at
dispatch is evicted instead (§V, "evicted").  Executed time comes from the executor:

* ``TableExecutor``: the profiled estimate (the reference simulator's semantics, CPU only);
* ``GpuExecutor``: the batch really runs through ``TransformerModel.forward_raw`` on the
  replica's GPU (synthetic images from a device-resident pool, the batch's task ids and the
  planned gamma) and the clock advances by the measured device time (CUDA events).

With several replicas (one per GPU, full model each, no collectives) the engine
dispatches to the earliest-free replica and plans from that replica's free time; the
single-accelerator planner is otherwise unchanged.

Two clocks: ``ServingEngine.run`` is the deterministic discrete-event loop above (executors
return a latency; replicas' busy intervals are simulated), and ``ServingEngine.run_realtime``
replays the trace against the wall clock with an asynchronous executor (``AsyncGpuExecutor``:
one worker thread and CUDA stream per replica, so all replicas compute concurrently while the
host loop keeps batching, planning and dispatching; finish time = measured completion).  Correctness is realised per
query from the profiled accuracy (Sampled: one Bernoulli draw per query in id order; Expected:
utility weighted by accuracy), since random-init weights make labels meaningless.
"""

from __future__ import annotations

import bisect
import csv
import os
import queue as _queue
import random
import threading
import time
from dataclasses import dataclass, field
from typing import Dict, List, Optional, Sequence, Tuple

from .adapter import AdapterConfig, allocate
from .batcher import BatchingThresholds, BatchQueue
from .core import Batch, OutcomeType, Query, TokenPlan, classify_outcome, us_from_s
from .errors import ConfigError
from .profiles import MemoryModel, ProfileTable, estimate_batch
from .replicas import next_free

__all__ = ["EngineConfig", "SimReport", "TableExecutor", "GpuExecutor", "AsyncGpuExecutor",
           "AsyncTableExecutor", "ServingEngine", "arrival_rate", "DEFAULT_TASKS", "synthetic_accuracy",
           "build_replicas"]


@dataclass(frozen=True)
class EngineConfig:
    """policy: "otas" (Alg. 2/3) or an int = FixedGamma baseline (gamma < 0 ToMe, > 0 VPT,
    0 PetS)."""

    policy: object = "otas"
    seed: int = 0
    correctness: str = "sampled"  # or "expected"
    # Planning cost bounds (real-time serving: the plan is recomputed at every dispatch, on the
    # host, while the replicas compute): DP over the `dp_horizon` earliest-deadline batches only
    # (None = the whole queue, Alg. 2 as specified) with `frontier_cap` states per DP row.
    dp_horizon: Optional[int] = None
    frontier_cap: int = 256

    def __post_init__(self) -> None:
        if not (self.policy == "otas" or isinstance(self.policy, int)):
            raise ConfigError("policy must be 'otas' or a fixed integer gamma")
        if self.correctness not in ("sampled", "expected"):
            raise ConfigError("correctness must be 'sampled' or 'expected'")


@dataclass
class SimReport:
    """Metric families of PAPER.md Figs. 8-11: cumulative utility, batch-accuracy CDF samples,
    gamma selection counts, outcome-type counts."""

    utility: float = 0.0
    utility_series: List[Tuple[int, float]] = field(default_factory=list)  # (finish us, running total)
    accuracy_samples: List[float] = field(default_factory=list)
    gamma_counts: Dict[int, int] = field(default_factory=dict)
    outcome_counts: Dict[OutcomeType, int] = field(default_factory=lambda: {o: 0 for o in OutcomeType})
    total_queries: int = 0
    executed_batches: int = 0
    executed_images: int = 0
    busy_us: List[int] = field(default_factory=list)  # per replica
    end_us: int = 0
    events: List[Tuple[int, str, int, int, Optional[int], int, float]] = field(default_factory=list)

    @property
    def served_ratio(self) -> float:
        done = self.total_queries - self.outcome_counts[OutcomeType.TYPE4]
        return done / self.total_queries if self.total_queries else 0.0

    def summary(self) -> Dict[str, object]:
        return {
            "total_queries": self.total_queries, "utility": round(self.utility, 4),
            "served_ratio": round(self.served_ratio, 4),
            "outcomes": {o.name.lower(): n for o, n in self.outcome_counts.items()},
            "gamma_counts": dict(sorted(self.gamma_counts.items())),
            "executed_batches": self.executed_batches, "executed_images": self.executed_images,
            "end_s": self.end_us / 1e6, "busy_s": [b / 1e6 for b in self.busy_us],
        }

    def export(self, out_dir: str) -> None:
        """utility_timeseries.csv, accuracy_cdf.csv, gamma_ratio.csv, outcome_ratio.csv,
        events.csv, summary.txt."""
        os.makedirs(out_dir, exist_ok=True)
        with open(os.path.join(out_dir, "utility_timeseries.csv"), "w", newline="") as fh:
            w = csv.writer(fh)
            w.writerow(["time_s", "cumulative_utility"])
            for t, u in self.utility_series:
                w.writerow([t / 1e6, u])
        with open(os.path.join(out_dir, "accuracy_cdf.csv"), "w", newline="") as fh:
            w = csv.writer(fh)
            w.writerow(["accuracy", "cdf"])
            xs = sorted(self.accuracy_samples)
            for i, a in enumerate(xs):
                w.writerow([a, (i + 1) / len(xs)])
        with open(os.path.join(out_dir, "gamma_ratio.csv"), "w", newline="") as fh:
            w = csv.writer(fh)
            w.writerow(["gamma", "batches", "ratio"])
            tot = sum(self.gamma_counts.values()) or 1
            for g, n in sorted(self.gamma_counts.items()):
                w.writerow([g, n, n / tot])
        with open(os.path.join(out_dir, "outcome_ratio.csv"), "w", newline="") as fh:
            w = csv.writer(fh)
            w.writerow(["outcome", "queries", "ratio"])
            for o, n in self.outcome_counts.items():
                w.writerow([o.name.lower(), n, n / (self.total_queries or 1)])
        with open(os.path.join(out_dir, "events.csv"), "w", newline="") as fh:
            w = csv.writer(fh)
            w.writerow(["time_us", "event", "batch_id", "replica", "gamma", "latency_us", "utility"])
            w.writerows(self.events)
        with open(os.path.join(out_dir, "summary.txt"), "w") as fh:
            for k, v in self.summary().items():
                fh.write(f"{k}={v}\n")


class TableExecutor:
    """Latency = the profiled estimate ("realized latency equals the profiled
    estimate"); optional seeded multiplicative noise exercises late (Type 3) outcomes."""

    def __init__(self, table: ProfileTable, n_replicas: int = 1, noise_sigma: float = 0.0, seed: int = 0):
        self.table, self.n_replicas, self.noise = table, n_replicas, noise_sigma
        self._rng = random.Random(seed)

    def execute(self, replica: int, batch: Batch, gamma: int) -> int:
        t, _ = estimate_batch(batch, gamma, self.table)
        if self.noise > 0:
            t = max(1, int(round(t * self._rng.lognormvariate(0.0, self.noise))))
        return t


class GpuExecutor:
    """Runs each batch on its replica's GPU: ``backbones[i]`` is a ``TransformerModel`` on
    device i with every task's head and prompts registered (task name -> id via
    ``task_index``).  Images come from a device-resident synthetic pool (query id modulo the
    pool), so no host work sits on the timed path; latency = CUDA-event device time."""

    def __init__(self, backbones: Sequence[object], task_index: Dict[str, int], pool: int = 512, seed: int = 0):
        import torch

        self._torch = torch
        self.backbones = list(backbones)
        self.n_replicas = len(self.backbones)
        self.task_index = dict(task_index)
        self._pools = []
        for bb in self.backbones:
            g = torch.Generator(device=bb.device).manual_seed(seed)
            img = bb.cfg.img
            self._pools.append(torch.randn(pool, 3, img, img, generator=g, device=bb.device))
        self.preds: Dict[int, int] = {}

    def execute(self, replica: int, batch: Batch, gamma: int) -> int:
        torch = self._torch
        bb = self.backbones[replica]
        pool = self._pools[replica]
        idx = torch.tensor([q.id % pool.shape[0] for q in batch.queries], device=bb.device)
        ids = torch.tensor([self.task_index[q.task] for q in batch.queries], dtype=torch.int32,
                           device=bb.device)
        imgs = pool.index_select(0, idx).contiguous()
        with torch.cuda.device(bb.device):
            start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            start.record()
            logits = bb.forward_raw(imgs, ids, gamma)
            end.record()
            end.synchronize()
        pred = logits.argmax(dim=1).tolist()
        for q, p in zip(batch.queries, pred):
            self.preds[q.id] = p
        return max(1, us_from_s(start.elapsed_time(end) / 1e3))


class _AsyncReplicas:
    """One worker thread per replica consuming (batch, gamma, dispatch_us) jobs; completions
    (replica, batch, gamma, dispatch_us, latency_us) go to a shared queue.  Each replica has at
    most one batch in flight (the engine only dispatches to an idle replica)."""

    def __init__(self, n: int):
        self.n_replicas = n
        self.done: "_queue.Queue" = _queue.Queue()
        self._jobs = [_queue.Queue() for _ in range(n)]
        self._threads = [threading.Thread(target=self._loop, args=(r,), daemon=True) for r in range(n)]
        for th in self._threads:
            th.start()

    def submit(self, replica: int, batch: Batch, gamma: int, dispatch_us: int) -> None:
        self._jobs[replica].put((batch, gamma, dispatch_us))

    def _loop(self, replica: int) -> None:
        while True:
            job = self._jobs[replica].get()
            if job is None:
                return
            batch, gamma, dispatch_us = job
            try:
                lat = self._run(replica, batch, gamma)
                self.done.put((replica, batch, gamma, dispatch_us, lat, None))
            except Exception as exc:  # surfaced by the engine loop
                self.done.put((replica, batch, gamma, dispatch_us, 0, exc))

    def close(self) -> None:
        for q in self._jobs:
            q.put(None)
        for th in self._threads:
            th.join(timeout=30)


class AsyncTableExecutor(_AsyncReplicas):
    """Host-only stand-in for ``AsyncGpuExecutor`` (tests): a replica "computes" for the
    profiled estimate x ``time_scale`` of wall time (sleep), concurrently with the others."""

    def __init__(self, table: ProfileTable, n_replicas: int = 1, time_scale: float = 1.0):
        self.table, self.time_scale = table, time_scale
        super().__init__(n_replicas)

    def _run(self, replica: int, batch: Batch, gamma: int) -> int:
        t, _ = estimate_batch(batch, gamma, self.table)
        time.sleep(t * self.time_scale / 1e6)
        return t


class AsyncGpuExecutor(_AsyncReplicas):
    """Concurrent execution on GPU replicas: replica i's worker thread owns a CUDA stream on
    its device and runs ``forward_raw`` there (the ctypes call releases the GIL, so the host
    loop and the other replicas' launches proceed meanwhile); latency = CUDA-event device
    time of the forward.  Inputs as in ``GpuExecutor`` (device-resident synthetic pool)."""

    def __init__(self, backbones: Sequence[object], task_index: Dict[str, int], pool: int = 512, seed: int = 0):
        import torch

        self._torch = torch
        self.backbones = list(backbones)
        self.task_index = dict(task_index)
        self._pools, self._streams = [], []
        for bb in self.backbones:
            g = torch.Generator(device=bb.device).manual_seed(seed)
            img = bb.cfg.img
            self._pools.append(torch.randn(pool, 3, img, img, generator=g, device=bb.device))
            self._streams.append(torch.cuda.Stream(bb.device))
        torch.cuda.synchronize()
        self.preds: Dict[int, int] = {}
        self._preds_lock = threading.Lock()
        super().__init__(len(self.backbones))

    def _run(self, replica: int, batch: Batch, gamma: int) -> int:
        torch = self._torch
        bb = self.backbones[replica]
        pool = self._pools[replica]
        with torch.cuda.device(bb.device), torch.cuda.stream(self._streams[replica]):
            idx = torch.tensor([q.id % pool.shape[0] for q in batch.queries], device=bb.device)
            ids = torch.tensor([self.task_index[q.task] for q in batch.queries], dtype=torch.int32,
                               device=bb.device)
            imgs = pool.index_select(0, idx).contiguous()
            start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            start.record()
            logits = bb.forward_raw(imgs, ids, gamma)
            end.record()
            pred = logits.argmax(dim=1)
            end.synchronize()
            pred = pred.tolist()
        with self._preds_lock:
            for q, p in zip(batch.queries, pred):
                self.preds[q.id] = p
        return max(1, us_from_s(start.elapsed_time(end) / 1e3))


def arrival_rate(arrivals_us: Sequence[int], now_us: int, window_us: int) -> float:
    """Requests/s over (now - window, now] of the sorted arrival times."""
    if window_us <= 0:
        raise ValueError("window must be positive")
    lo = bisect.bisect_right(arrivals_us, now_us - window_us)
    hi = bisect.bisect_right(arrivals_us, now_us)
    return (hi - lo) * 1e6 / window_us


class ServingEngine:
    def __init__(self, executor, table: ProfileTable, thresholds: BatchingThresholds = BatchingThresholds.paper(),
                 adapter: AdapterConfig = AdapterConfig(), mem: Optional[MemoryModel] = None,
                 cfg: EngineConfig = EngineConfig()):
        self.executor, self.table, self.th, self.adapter, self.mem, self.cfg = executor, table, thresholds, adapter, mem, cfg
        if isinstance(cfg.policy, int) and cfg.policy not in adapter.gammas:
            raise ConfigError(f"fixed gamma {cfg.policy} is not in the gamma list")

    def _plan(self, batches: List[Batch], now: int, rate: float, initial: bool) -> TokenPlan:
        if self.cfg.policy == "otas":
            if self.cfg.dp_horizon is not None and len(batches) > self.cfg.dp_horizon:
                batches = sorted(batches, key=lambda b: (b.deadline_us, b.id))[: self.cfg.dp_horizon]
            return allocate(batches, now, self.adapter, self.table, self.mem, rate, initial_stage=initial,
                            frontier_cap=self.cfg.frontier_cap)
        return TokenPlan({b.id: self.cfg.policy for b in batches})

    def run(self, queries: Sequence[Query]) -> SimReport:
        qs = sorted(queries, key=lambda q: (q.arrival_us, q.id))
        rep = SimReport(total_queries=len(qs))
        n_rep = self.executor.n_replicas
        rep.busy_us = [0] * n_rep
        if not qs:
            return rep
        rng = random.Random(self.cfg.seed)
        arrivals = [q.arrival_us for q in qs]
        start = arrivals[0]
        free_at = [start] * n_rep
        queue = BatchQueue()
        nxt = 0

        def finalize(batch: Batch, gamma: Optional[int], finish: Optional[int], replica: int, lat: int) -> None:
            correct_n, util = 0, 0.0
            for q in sorted(batch.queries, key=lambda q: q.id):
                if finish is None:
                    q.finalize(OutcomeType.TYPE4)
                else:
                    acc = self.table.accuracy_for(q.task, gamma)
                    if self.cfg.correctness == "sampled":
                        correct = rng.random() < acc
                    else:
                        correct = True
                    outcome = classify_outcome(q, True, correct, finish)
                    q.finalize(outcome)
                    if outcome is OutcomeType.TYPE1:
                        util += q.utility * (acc if self.cfg.correctness == "expected" else 1.0)
                        correct_n += 1
                rep.outcome_counts[q.outcome] += 1
            if finish is None:
                rep.events.append((free_at[replica], "evict", batch.id, replica, gamma, 0, 0.0))
                return
            rep.utility += util
            rep.utility_series.append((finish, rep.utility))
            rep.accuracy_samples.append(correct_n / batch.size)
            rep.gamma_counts[gamma] = rep.gamma_counts.get(gamma, 0) + 1
            rep.events.append((finish - lat, "execute", batch.id, replica, gamma, lat, util))

        while True:
            r_i = next_free(free_at)
            now = free_at[r_i]
            if not queue.batches:
                if nxt >= len(qs):
                    break
                now = max(now, arrivals[nxt])
                free_at[r_i] = now
            while nxt < len(qs) and arrivals[nxt] <= now:
                queue.add_query(qs[nxt], self.th)
                nxt += 1
            rate = arrival_rate(arrivals, now, self.adapter.rate_window_us)
            plan = self._plan(list(queue.batches), now, rate, now - start < self.adapter.initial_stage_us)
            for b in [b for b in queue.batches if b.id in plan.assignments and plan.is_skip(b.id)]:
                queue.remove(b)
                finalize(b, None, None, r_i, 0)
            if not queue.batches:
                continue
            b = min(queue.batches, key=lambda b: (b.deadline_us, b.id))
            gamma = plan.gamma_for(b.id)
            queue.remove(b)
            t_hat, _ = estimate_batch(b, gamma, self.table)
            if now + t_hat >= b.deadline_us:  # doomed before execution: evict (Type 4)
                finalize(b, None, None, r_i, 0)
                continue
            lat = self.executor.execute(r_i, b, gamma)
            finish = now + lat
            free_at[r_i] = finish
            rep.busy_us[r_i] += lat
            rep.executed_batches += 1
            rep.executed_images += b.size
            finalize(b, gamma, finish, r_i, lat)
        for b in list(queue.batches):
            queue.remove(b)
            finalize(b, None, None, 0, 0)
        rep.end_us = max(free_at)
        return rep

    def run_realtime(self, queries: Sequence[Query], time_scale: float = 1.0, idle_poll_s: float = 2e-4) -> SimReport:
        """Replays the trace against the wall clock (trace us = elapsed us / time_scale) with an
        asynchronous executor (``AsyncGpuExecutor``): every idle replica gets the EDF batch of
        a fresh plan at once, so all replicas compute concurrently while this loop ingests
        arrivals (Alg. 1), plans (Alg. 2/3) and collects completions.  A batch's finish time
        is its dispatch time plus its measured latency; outcome rules as in ``run``."""
        ex = self.executor
        if not hasattr(ex, "submit"):
            raise ConfigError("run_realtime needs an asynchronous executor (submit / done)")
        qs = sorted(queries, key=lambda q: (q.arrival_us, q.id))
        rep = SimReport(total_queries=len(qs))
        n_rep = ex.n_replicas
        rep.busy_us = [0] * n_rep
        if not qs:
            return rep
        rng = random.Random(self.cfg.seed)
        arrivals = [q.arrival_us for q in qs]
        start = arrivals[0]
        t0 = time.perf_counter()

        def clock() -> int:
            return start + int((time.perf_counter() - t0) * 1e6 / time_scale)

        busy = [False] * n_rep
        queue = BatchQueue()
        nxt = 0
        end_us = start

        def finalize(batch, gamma, finish, replica, lat, at):
            self._finalize(rep, rng, batch, gamma, finish, replica, lat, at)

        def complete(item) -> None:
            nonlocal end_us
            r, b, g, disp, lat, exc = item
            if exc is not None:
                raise exc
            busy[r] = False
            finish = disp + lat
            end_us = max(end_us, finish)
            rep.busy_us[r] += lat
            finalize(b, g, finish, r, lat, disp)

        while True:
            while True:  # completions
                try:
                    complete(ex.done.get_nowait())
                except _queue.Empty:
                    break
            now = clock()
            while nxt < len(qs) and arrivals[nxt] <= now:
                queue.add_query(qs[nxt], self.th)
                nxt += 1
            for r in range(n_rep):
                if busy[r]:
                    continue
                while queue.batches and not busy[r]:
                    rate = arrival_rate(arrivals, now, self.adapter.rate_window_us)
                    plan = self._plan(list(queue.batches), now, rate, now - start < self.adapter.initial_stage_us)
                    for b in [b for b in queue.batches if b.id in plan.assignments and plan.is_skip(b.id)]:
                        queue.remove(b)
                        finalize(b, None, None, r, 0, now)
                    if not queue.batches:
                        break
                    b = min(queue.batches, key=lambda b: (b.deadline_us, b.id))
                    gamma = plan.gamma_for(b.id)
                    queue.remove(b)
                    t_hat, _ = estimate_batch(b, gamma, self.table)
                    if now + t_hat >= b.deadline_us:  # doomed before execution: evict (Type 4)
                        finalize(b, None, None, r, 0, now)
                        continue
                    busy[r] = True
                    rep.executed_batches += 1
                    rep.executed_images += b.size
                    ex.submit(r, b, gamma, now)
            if nxt >= len(qs) and not queue.batches and not any(busy):
                break
            # sleep until a completion, the next arrival or the poll interval
            wait_s = idle_poll_s
            if nxt < len(qs):
                wait_s = min(wait_s, max(0.0, (arrivals[nxt] - clock()) * time_scale / 1e6))
            try:
                complete(ex.done.get(timeout=max(wait_s, 1e-5)))
            except _queue.Empty:
                pass
        rep.end_us = end_us
        return rep

    def _finalize(self, rep: SimReport, rng: random.Random, batch: Batch, gamma: Optional[int],
                  finish: Optional[int], replica: int, lat: int, at: int) -> None:
        """Outcome of every query of a batch (evicted when finish is None), as in ``run``."""
        correct_n, util = 0, 0.0
        for q in sorted(batch.queries, key=lambda q: q.id):
            if finish is None:
                q.finalize(OutcomeType.TYPE4)
            else:
                acc = self.table.accuracy_for(q.task, gamma)
                correct = rng.random() < acc if self.cfg.correctness == "sampled" else True
                outcome = classify_outcome(q, True, correct, finish)
                q.finalize(outcome)
                if outcome is OutcomeType.TYPE1:
                    util += q.utility * (acc if self.cfg.correctness == "expected" else 1.0)
                    correct_n += 1
            rep.outcome_counts[q.outcome] += 1
        if finish is None:
            rep.events.append((at, "evict", batch.id, replica, gamma, 0, 0.0))
            return
        rep.utility += util
        rep.utility_series.append((finish, rep.utility))
        rep.accuracy_samples.append(correct_n / batch.size)
        rep.gamma_counts[gamma] = rep.gamma_counts.get(gamma, 0) + 1
        rep.events.append((finish - lat, "execute", batch.id, replica, gamma, lat, util))


# ----------------------------------------------------------------------------- replicas
DEFAULT_TASKS: Tuple[Tuple[str, int], ...] = (("CIFAR10", 10), ("CIFAR100", 100), ("EuroSAT", 10))


def synthetic_accuracy(tasks: Sequence[Tuple[str, int]], gammas: Sequence[int]) -> Dict[Tuple[str, int], float]:
    """Accuracy model for the planner: random-init weights have no meaningful accuracy, so the
    table follows the paper's qualitative profile (merging loses accuracy, prompts gain a
    little): acc = base - 0.004 |gamma| (gamma < 0), base + 0.0015 gamma
    (gamma > 0), with base 0.98 / 0.90 / 0.97 for CIFAR10 / CIFAR100 / EuroSAT."""
    base = {"CIFAR10": 0.98, "CIFAR100": 0.90, "EuroSAT": 0.97}
    out = {}
    for name, _ in tasks:
        b0 = base.get(name, 0.9)
        for g in gammas:
            out[(name, g)] = min(1.0, b0 - 0.004 * (-g) if g < 0 else b0 + 0.0015 * g)
    return out


def build_replicas(model: str = "vit_b16", devices: Sequence[str] = ("cuda:0",),
                   tasks: Sequence[Tuple[str, int]] = DEFAULT_TASKS, gammas: Sequence[int] = (),
                   dtype: str = "bf16", seed: int = 0):
    """One ServeModel per device: the same seeded backbone, one head per task and prompts for
    every gamma > 0 of the list (PAPER.md:522-540 Register_Task).  Returns (replicas,
    task name -> task id)."""
    from .config import VIT_CONFIGS
    from .model import ServeModel, TaskModel, TransformerModel
    from .weights import init_backbone, init_head, init_prompts

    cfg = VIT_CONFIGS[model]
    params = init_backbone(cfg, seed)
    max_classes = max(c for _, c in tasks)
    task_models = []
    for i, (name, classes) in enumerate(tasks):
        h = init_head(cfg, classes, i)
        prompts = {g: init_prompts(cfg, g, i) for g in gammas if g > 0}
        task_models.append(TaskModel(name, h["w"], h["b"], prompts))
    replicas = []
    for dev in devices:
        bb = TransformerModel(cfg, params, dev, dtype=dtype, n_tasks=len(tasks), max_classes=max_classes)
        replicas.append(ServeModel(bb, task_models))
    return replicas, {name: i for i, (name, _) in enumerate(tasks)}
