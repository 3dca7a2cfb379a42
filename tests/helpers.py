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
                   dtype=torch.float32, forced=None, max_classes=None, shadow=False):
    heads = [t["head"] for t in tasks]
    prompts = [t["prompts"].get(gamma) for t in tasks] if gamma > 0 else None
    return vit_oracle.forward(params, heads, images, task_ids, gamma, n_heads=cfg.heads,
                              patch=cfg.patch, prompts=prompts, prompt_mode=prompt_mode,
                              dtype=dtype, forced=forced, max_classes=max_classes, shadow=shadow)


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


# ---------------------------------------------------------------- near-tie accounting
# A merge decision set is "valid within tau" when it is what the exact matching would give
# if every score were perturbed by at most tau/2: every dst is within tau of its row's best
# score, the src rows come in non-increasing order of their best score (within tau), and no
# unmerged A row beats a merged one by more than tau.  Exactly-equal scores follow the tie
# rules (argmax -> lowest column, stable descending order), which only an exact comparison
# checks; those cases are never excluded.
def decision_slack(scores, src, dst, unm):
    """scores [na, nb] (float64, row 0 = -inf), src/dst [r], unm [na - r] (one image) ->
    (structurally_valid, slack): slack = largest tau-violation (0 when exactly consistent)."""
    na = scores.shape[0]
    allrows = torch.cat([src, unm]).sort().values
    if not torch.equal(allrows, torch.arange(na)) or not torch.equal(unm, unm.sort().values):
        return False, float("inf")
    if (src == 0).any():  # the class token is never merged
        return False, float("inf")
    node_max = scores.max(-1).values
    slack = 0.0
    slack = max(slack, float((node_max[src] - scores[src, dst]).max()))
    nm_src = node_max[src]
    if nm_src.numel() > 1:
        slack = max(slack, float((nm_src[1:] - nm_src[:-1]).max()))
    nm_unm = node_max[unm[unm != 0]]
    if nm_unm.numel():
        slack = max(slack, float(nm_unm.max() - nm_src.min()))
    return True, max(0.0, slack)


def compare_traces(steps, gpu_trace):
    """steps: oracle MergeSteps from a forced + shadow run (history = the GPU's trace);
    gpu_trace: [(src, dst, unm)] per merge layer.  Returns per-layer stats: image-layers
    identical to the oracle's own decisions, those that differ (excluded as near-ties), and
    the largest slack among the differing ones."""
    out = []
    for st, (s, d, u) in zip(steps, gpu_trace):
        o_src, o_dst, o_unm = st.own
        same = (o_src == s).all(1) & (o_dst == d).all(1) & (o_unm == u).all(1)
        worst, valid = 0.0, True
        for b in torch.nonzero(~same).flatten().tolist():
            ok, slack = decision_slack(st.scores[b], s[b], d[b], u[b])
            valid &= ok
            worst = max(worst, slack)
        out.append({"layer": st.layer, "t": st.t, "r": st.r, "images": int(same.numel()),
                    "identical": int(same.sum()), "differing": int((~same).sum()),
                    "max_slack": worst, "valid": bool(valid)})
    return out


def record(name, payload):
    """Append one JSON line to $TA_PARITY_LOG (the committed parity tables are made from it)."""
    import json
    import os

    path = os.environ.get("TA_PARITY_LOG")
    if path:
        with open(path, "a") as fh:
            fh.write(json.dumps({"test": name, **payload}) + "\n")


__all__ += ["decision_slack", "compare_traces", "record"]
