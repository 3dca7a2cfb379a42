"""Shared builders for the parity tests: the same seeded weights feed the oracle (CPU) and
the CUDA path (GPU)."""

from __future__ import annotations

from typing import Dict, List, Sequence, Tuple

import torch

from oracle import vit_oracle
from paper_2401_05031_b200.config import VIT_CONFIGS, ViTConfig
from paper_2401_05031_b200.weights import init_backbone, init_head, init_prompts, synthetic_images

_CACHE: Dict[Tuple[str, int], Dict[str, object]] = {}


def backbone(name: str, seed: int = 0) -> Tuple[ViTConfig, Dict[str, object]]:
    cfg = VIT_CONFIGS[name]
    key = (name, seed)
    if key not in _CACHE:
        _CACHE[key] = init_backbone(cfg, seed)
    return cfg, _CACHE[key]


def task_params(cfg: ViTConfig, classes: Sequence[int], gammas: Sequence[int]) -> List[Dict[str, object]]:
    out = []
    for i, c in enumerate(classes):
        h = init_head(cfg, c, i)
        pr = {g: init_prompts(cfg, g, i) for g in gammas if g > 0}
        out.append({"name": f"task{i}", "head": h, "prompts": pr})
    return out


def oracle_forward(cfg, params, tasks, images, task_ids, gamma, prompt_mode="accumulate",
                   dtype=torch.float32, forced=None, max_classes=None):
    heads = [t["head"] for t in tasks]
    prompts = [t["prompts"].get(gamma) for t in tasks] if gamma > 0 else None
    return vit_oracle.forward(params, heads, images, task_ids, gamma, n_heads=cfg.heads,
                              patch=cfg.patch, prompts=prompts, prompt_mode=prompt_mode,
                              dtype=dtype, forced=forced, max_classes=max_classes)


def serve_model(cfg, params, tasks, dtype="bf16", prompt_mode="accumulate", max_classes=None,
                fold_ln=None):
    from paper_2401_05031_b200.model import ServeModel, TaskModel, TransformerModel

    mc = max_classes or max(t["head"]["w"].shape[0] for t in tasks)
    bb = TransformerModel(cfg, params, "cuda:0", dtype=dtype, prompt_mode=prompt_mode,
                          n_tasks=len(tasks), max_classes=mc, fold_ln=fold_ln)
    sm = ServeModel(bb)
    for t in tasks:
        sm.register_task(TaskModel(t["name"], t["head"]["w"], t["head"]["b"], dict(t["prompts"])))
    return sm


def split_trace(flat: torch.Tensor, schedule: Tuple[List[int], List[int]], batch: int):
    """Decode the flat int32 merge trace into per-layer (src, dst, unm) [B, *] tensors."""
    ts, rs = schedule
    out, off = [], 0
    for t, r in zip(ts, rs):
        if r <= 0:
            continue
        na = (t + 1) // 2
        src = flat[off: off + batch * r].reshape(batch, r)
        off += batch * r
        dst = flat[off: off + batch * r].reshape(batch, r)
        off += batch * r
        unm = flat[off: off + batch * (na - r)].reshape(batch, na - r)
        off += batch * (na - r)
        out.append((src.long(), dst.long(), unm.long()))
    return out


__all__ = ["backbone", "task_params", "oracle_forward", "serve_model", "split_trace",
           "synthetic_images", "init_head", "init_prompts"]
