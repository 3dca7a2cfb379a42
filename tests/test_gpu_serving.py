"""Serving engine on the GPU: the adapter's planned gamma really executes through
ta_forward on a replica, latencies are measured device time, and the run keeps the engine's
invariants (SPEC.md engine module) on a short Poisson trace."""

import pytest

from paper_2401_05031_b200.adapter import AdapterConfig
from paper_2401_05031_b200.core import GammaList, OutcomeType
from paper_2401_05031_b200.engine import (DEFAULT_TASKS, EngineConfig, GpuExecutor, ServingEngine,
                                          build_replicas, synthetic_accuracy)
from paper_2401_05031_b200.profiles import derive_f
from paper_2401_05031_b200.workload import gen_poisson

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("policy", ["otas", 0])
def test_gpu_serving_trace(policy):
    gammas = GammaList((-8, -4, 0, 4))
    replicas, index = build_replicas("vit_tiny", ["cuda:0"], DEFAULT_TASKS, gammas.values)
    table = replicas[0].profile(gammas.values, 32, synthetic_accuracy(DEFAULT_TASKS, gammas.values), iters=2, warmup=1)
    for (task, g), us in table.sample_latency_us.items():
        assert us > 0
    cfg = AdapterConfig(gammas=gammas, rate_map=derive_f(table, gammas, 32), initial_stage_us=200_000)
    ex = GpuExecutor([r.backbone for r in replicas], index, pool=64)
    qs = gen_poisson([(0, 3000), (0.5, 9000)], 1.0, seed=3)
    rep = ServingEngine(ex, table, adapter=cfg, cfg=EngineConfig(policy=policy, seed=1)).run(qs)
    assert sum(rep.outcome_counts.values()) == len(qs)
    assert rep.executed_batches > 0 and len(ex.preds) == rep.executed_images
    assert rep.outcome_counts[OutcomeType.TYPE1] > 0
    if policy != "otas":
        assert set(rep.gamma_counts) == {policy}
    for r in replicas:
        r.backbone.close()


def test_forward_async_matches_sync():
    """ServeModel.forward_async (pipelined H2D / forward / D2H over two staging slots) gives
    the same logits as the synchronous host path, across gammas and in-flight reuse."""
    import torch

    gammas = (-4, 0, 4)
    replicas, index = build_replicas("vit_tiny", ["cuda:0"], DEFAULT_TASKS, gammas)
    sm = replicas[0]
    B = 12
    imgs = [torch.randn(B, 3, 64, 64, generator=torch.Generator().manual_seed(i)).pin_memory() for i in range(6)]
    tasks = [["CIFAR10", "CIFAR100", "EuroSAT"][i % 3] for i in range(B)]
    ref = [sm.forward(imgs[i], tasks, gamma=gammas[i % 3]).clone() for i in range(6)]
    pend = [sm.forward_async(imgs[i], tasks, gamma=gammas[i % 3]) for i in range(6)]
    for r, p in zip(ref, pend):
        out = p.wait()
        fin = torch.isfinite(r)
        assert torch.equal(fin, torch.isfinite(out))
        assert torch.equal(r[fin], out[fin])
    sm.backbone.close()


def test_gpu_serving_realtime_concurrent_replicas():
    """run_realtime + AsyncGpuExecutor: two replicas (both on cuda:0 here; one per GPU in
    serving) run batches concurrently on their own streams; every query gets one outcome and
    the replicas' device-timed executions overlap in wall time."""
    from paper_2401_05031_b200.engine import AsyncGpuExecutor

    gammas = GammaList((-8, -4, 0, 4))
    replicas, index = build_replicas("vit_tiny", ["cuda:0", "cuda:0"], DEFAULT_TASKS, gammas.values)
    table = replicas[0].profile(gammas.values, 32, synthetic_accuracy(DEFAULT_TASKS, gammas.values), iters=2, warmup=1)
    cfg = AdapterConfig(gammas=gammas, rate_map=derive_f(table, gammas, 32), initial_stage_us=100_000)
    ex = AsyncGpuExecutor([r.backbone for r in replicas], index, pool=64)
    try:
        qs = gen_poisson([(0, 6000)], 0.5, seed=4)
        rep = ServingEngine(ex, table, adapter=cfg, cfg=EngineConfig(policy="otas", seed=1)).run_realtime(qs)
    finally:
        ex.close()
    assert sum(rep.outcome_counts.values()) == len(qs)
    assert rep.executed_batches > 0 and len(ex.preds) == rep.executed_images
    assert rep.outcome_counts[OutcomeType.TYPE1] > 0
    runs = [(e[0], e[0] + e[5], e[3]) for e in rep.events if e[1] == "execute"]
    assert {r for _, _, r in runs} == {0, 1}
    for r in replicas:
        r.backbone.close()
