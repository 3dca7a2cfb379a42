"""Prompt repository and task registry ("Register_Task"): the per-task
parameters of the shared backbone, persisted on disk and keyed by (task, gamma).

Layout under ``root``::

    <task>/head.pt            {"w": [C, D] fp32, "b": [C] fp32}
    <task>/prompts_g<gamma>.pt  [L, gamma, D] fp32 (VPT-deep prompt tokens for one gamma > 0)
    index.json                {task: {"classes": C, "gammas": [...], "dim": D, "depth": L}}

``register_task`` writes a task (new gammas can be added later, as the paper trains prompts per
gamma); ``task_model`` loads one back as a ``TaskModel``; ``ServeModel.register_from`` puts
tasks of a repository on a replica.  Host-side bookkeeping: only tensors registered with a
replica reach the GPU (ta_model_set_head / ta_model_set_prompts).
"""

from __future__ import annotations

import json
import os
from typing import Dict, List, Optional

import torch

from .errors import ConfigError, ProfileGapError

__all__ = ["PromptRepository"]


class PromptRepository:
    def __init__(self, root: str):
        self.root = root
        os.makedirs(root, exist_ok=True)
        self._index_path = os.path.join(root, "index.json")
        self._index: Dict[str, Dict[str, object]] = {}
        if os.path.exists(self._index_path):
            with open(self._index_path) as fh:
                self._index = json.load(fh)

    # -- registry ------------------------------------------------------------------------
    def tasks(self) -> List[str]:
        return sorted(self._index)

    def gammas(self, task: str) -> List[int]:
        return list(self._entry(task)["gammas"])

    def _entry(self, task: str) -> Dict[str, object]:
        if task not in self._index:
            raise KeyError(f"task {task!r} is not in the repository")
        return self._index[task]

    def _save_index(self) -> None:
        tmp = self._index_path + ".tmp"
        with open(tmp, "w") as fh:
            json.dump(self._index, fh, indent=1, sort_keys=True)
        os.replace(tmp, self._index_path)

    def register_task(self, task: str, head_w: torch.Tensor, head_b: torch.Tensor,
                      prompts: Optional[Dict[int, torch.Tensor]] = None, depth: Optional[int] = None) -> None:
        """Register_Task: store the head and any prompts; re-registering a task keeps its
        existing prompt gammas and requires the same head shape."""
        if not task or "/" in task or task.startswith("."):
            raise ConfigError(f"invalid task name {task!r}")
        w = head_w.detach().to("cpu", torch.float32).contiguous()
        b = head_b.detach().to("cpu", torch.float32).contiguous()
        if w.dim() != 2 or tuple(b.shape) != (w.shape[0],):
            raise ConfigError("head must be w [C, D] and b [C]")
        old = self._index.get(task)
        if old is not None and (old["classes"] != w.shape[0] or old["dim"] != w.shape[1]):
            raise ConfigError(f"task {task!r} already registered with a different head shape")
        d = os.path.join(self.root, task)
        os.makedirs(d, exist_ok=True)
        torch.save({"w": w, "b": b}, os.path.join(d, "head.pt"))
        entry = {"classes": int(w.shape[0]), "dim": int(w.shape[1]),
                 "depth": (old or {}).get("depth", depth), "gammas": list((old or {}).get("gammas", []))}
        self._index[task] = entry
        for gamma, p in (prompts or {}).items():
            self._put_prompts(task, int(gamma), p)
        self._save_index()

    def add_prompts(self, task: str, gamma: int, prompts: torch.Tensor) -> None:
        """Prompt tokens for one more gamma of an existing task (trained offline per gamma)."""
        self._entry(task)
        self._put_prompts(task, gamma, prompts)
        self._save_index()

    def _put_prompts(self, task: str, gamma: int, prompts: torch.Tensor) -> None:
        entry = self._index[task]
        if gamma <= 0:
            raise ConfigError("prompts exist only for gamma > 0")
        p = prompts.detach().to("cpu", torch.float32).contiguous()
        if p.dim() != 3 or p.shape[1] != gamma or p.shape[2] != entry["dim"]:
            raise ConfigError(f"prompts must be [L, gamma={gamma}, D={entry['dim']}], got {tuple(p.shape)}")
        if entry["depth"] is None:
            entry["depth"] = int(p.shape[0])
        elif entry["depth"] != p.shape[0]:
            raise ConfigError(f"prompts have {p.shape[0]} layers, the task has {entry['depth']}")
        torch.save(p, os.path.join(self.root, task, f"prompts_g{gamma}.pt"))
        if gamma not in entry["gammas"]:
            entry["gammas"] = sorted(entry["gammas"] + [gamma])

    # -- lookup --------------------------------------------------------------------------
    def head(self, task: str) -> Dict[str, torch.Tensor]:
        self._entry(task)
        return torch.load(os.path.join(self.root, task, "head.pt"), map_location="cpu", weights_only=True)

    def prompts(self, task: str, gamma: int) -> torch.Tensor:
        """The (task, gamma) prompt lookup; ProfileGapError(task, gamma, "prompt") when absent
        (the reference's missing-entry convention, errors.py:8-18)."""
        if gamma not in self.gammas(task):
            raise ProfileGapError(task, gamma, "prompt")
        return torch.load(os.path.join(self.root, task, f"prompts_g{gamma}.pt"), map_location="cpu",
                          weights_only=True)

    def task_model(self, task: str, gammas: Optional[List[int]] = None):
        """A ``TaskModel`` with the head and the prompts for ``gammas`` (default: all stored)."""
        from .model import TaskModel

        h = self.head(task)
        gs = self.gammas(task) if gammas is None else [g for g in gammas if g > 0]
        return TaskModel(task, h["w"], h["b"], {g: self.prompts(task, g) for g in gs})
