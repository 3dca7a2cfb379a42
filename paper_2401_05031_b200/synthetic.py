"""Synthetic serving setup for benchmarks and the profiler: seeded random-init backbone,
per-task heads and prompts (weights.py; the scheme of SURVEY.md §8d), registered on a GPU
replica.  No pretrained checkpoints exist offline, so this is the benchmark model; the parity
tests build the identical weights through tests/helpers.py for the CPU oracle."""

from __future__ import annotations

from typing import Sequence

import torch

from .config import VIT_CONFIGS
from .weights import init_backbone, init_head, init_prompts

__all__ = ["build_serve_model", "synthetic_task_params"]


def synthetic_task_params(cfg, classes: Sequence[int], gammas: Sequence[int]):
    """Per task: {"name", "head": {"w", "b"}, "prompts": {gamma: [L, gamma, D]}} (gamma > 0)."""
    out = []
    for i, c in enumerate(classes):
        out.append({"name": f"task{i}", "head": init_head(cfg, c, i),
                    "prompts": {g: init_prompts(cfg, g, i) for g in gammas if g > 0}})
    return out


def build_serve_model(name: str, classes: Sequence[int] = (100,), gammas: Sequence[int] = (),
                      dtype: str = "bf16", device="cuda:0", prompt_mode: str = "accumulate",
                      fold_ln=None, seed: int = 0):
    """ServeModel over one replica of VIT_CONFIGS[name] on `device` with len(classes) tasks."""
    from .model import ServeModel, TaskModel, TransformerModel

    cfg = VIT_CONFIGS[name]
    params = init_backbone(cfg, seed)
    tasks = synthetic_task_params(cfg, classes, gammas)
    bb = TransformerModel(cfg, params, device, dtype=dtype, prompt_mode=prompt_mode,
                          n_tasks=len(tasks), max_classes=max(classes), fold_ln=fold_ln)
    sm = ServeModel(bb)
    for t in tasks:
        sm.register_task(TaskModel(t["name"], t["head"]["w"], t["head"]["b"], dict(t["prompts"])))
    return sm
