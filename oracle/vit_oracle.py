"""CPU ORACLE for the token-adapted ViT forward (OTAS, arXiv 2401.05031).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
CPU-baseline / ``--impl reference`` legs may import this module, and only as the checker or
the timed CPU reference.  The product path (``paper_2401_05031_b200``) never imports it
and has no CPU fallback.

PARITY: PINNED TO A THIRD-PARTY ViT (transformers), NOT TO THE REFERENCE.  The reference
ships no code for this path: SPEC.md:9 declares ToMe's merge and the attention math out of scope and ``estimate_batch`` (profiles.py:124-141)
replaces execution with a table lookup.  This module is our restatement of the algorithm
the paper describes and delegates to third-party code, none of which is
vendored here, and of which only a timm-equivalent ViT (transformers) is installed:
  * timm ``vision_transformer.VisionTransformer`` (unpinned) — pre-norm ViT:
    patch conv, cls + pos, L x (LN -> MHA -> residual -> LN -> MLP(GELU erf) -> residual),
    final LN, cls readout;
  * ToMe ``tome/merge.py::bipartite_soft_matching`` + ``merge_wavg``, ``tome/patch/timm.py``
    ``ToMeBlock`` / ``ToMeAttention`` with ``prop_attn=True`` (unpinned; PAPER.md:534,
    219-220, 281): merge after attention, before the MLP; metric = k.mean over heads;
    proportional attention adds log(size);
  * VPT prompted ViT (unpinned): gamma prompt tokens per
    layer before the norm, keyed by (task, gamma).
The restatement follows SURVEY.md Appendix A line by line, with the tie rules made
explicit (argmax -> lowest column, descending order -> stable), since upstream leaves them
unspecified.  What pins it:
  (1) THIRD-PARTY PIN: tests/golden/make_hf_golden.py runs the same seeded ViT through
      HuggingFace transformers 5.5.0 (installed in this image; models/vit/modeling_vit.py
      ViTForImageClassification, timm's architecture) with ToMe's block patch and
      bipartite_soft_matching / merge_wavg restated in upstream's own code structure and VPT
      prompt insertion over transformers' layer modules; tests/test_oracle.py requires identical
      merge traces and fp64 logits to 1e-10 on ViT-tiny and ViT-B/16 for gamma in
      {-16, -8, -3, 0, 4, 8} (committed fixture + a live regeneration when transformers is
      importable).  The backbone arithmetic (patch embed, attention, LayerNorm, GELU, MLP,
      head) is thereby pinned to an independent implementation; the ToMe / VPT glue remains a
      restatement of the published algorithms (their packages are not installed);
  (2) an independent pure-Python loop restatement of Appendix A `match` / `merge` with
      injected exact ties; (3) fp32 vs fp64 index-set agreement; (4) frozen goldens
      (tests/golden/make_golden.py) so later edits cannot drift silently.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import Dict, List, Optional, Sequence, Tuple

import torch
import torch.nn.functional as F

__all__ = ["MergeStep", "OracleTrace", "bipartite_soft_matching", "merge_wavg", "forward",
           "token_schedule"]


@dataclass
class MergeStep:
    layer: int
    t: int
    r: int
    src: torch.Tensor      # int64 [B, r]   A-row indices merged away (order = rank)
    dst: torch.Tensor      # int64 [B, r]   B-row index each src merges into
    unm: torch.Tensor      # int64 [B, ceil(t/2) - r] A rows kept, ascending (cls first)
    node_max: torch.Tensor  # [B, ceil(t/2)] best score per A row (-inf for cls)
    second: torch.Tensor    # [B, ceil(t/2)] second-best score per A row (argmax margin)
    # shadow mode (forced + shadow=True): the oracle's OWN decisions at this layer given the
    # forced history, and its score matrix, for near-tie accounting in the parity tests
    own: Optional[Tuple[torch.Tensor, torch.Tensor, torch.Tensor]] = None
    scores: Optional[torch.Tensor] = None   # [B, ceil(t/2), floor(t/2)], row 0 = -inf


@dataclass
class OracleTrace:
    merges: List[MergeStep] = field(default_factory=list)

    def flat_int32(self) -> torch.Tensor:
        """Layout of include/tokadapt_cuda.h ta_merge_trace_len: per merge layer
        src [B, r], dst [B, r], unm [B, na - r]."""
        parts = []
        for m in self.merges:
            parts += [m.src.reshape(-1), m.dst.reshape(-1), m.unm.reshape(-1)]
        if not parts:
            return torch.zeros(0, dtype=torch.int32)
        return torch.cat(parts).to(torch.int32)


def token_schedule(n_tokens: int, depth: int, gamma: int, prompt_mode: str = "accumulate"
                   ) -> Tuple[List[int], List[int]]:
    """r_l = min(|gamma|, (t_l - 1) // 2) (ToMe parse_r, constant r,
    class token protected); prompts add gamma rows per layer (accumulate) or once (replace)."""
    ts, rs, t = [], [], n_tokens
    for layer in range(depth):
        if gamma > 0:
            tl = n_tokens + gamma * (layer + 1) if prompt_mode == "accumulate" else n_tokens + gamma
            rl = 0
        else:
            tl = t
            rl = max(0, min(-gamma, (tl - 1) // 2)) if gamma < 0 else 0
        ts.append(tl)
        rs.append(rl)
        t = tl - rl
    return ts, rs


def bipartite_soft_matching(metric: torch.Tensor, r: int, return_scores: bool = False):
    """ToMe bipartite soft matching with class-token protection (Appendix A `match`).

    metric [B, t, c] -> (src, dst, unm, node_max, second), all per image (+ scores).
    """
    metric = metric / metric.norm(dim=-1, keepdim=True)
    a, b = metric[:, 0::2, :], metric[:, 1::2, :]
    scores = a @ b.transpose(-1, -2)
    scores[:, 0, :] = -math.inf
    node_idx = scores.argmax(dim=-1)                      # first (lowest) index on ties
    node_max = scores.gather(-1, node_idx[..., None])[..., 0]
    if scores.shape[-1] > 1:
        second = scores.topk(2, dim=-1).values[..., 1]
    else:
        second = torch.full_like(node_max, -math.inf)
    order = node_max.argsort(dim=-1, descending=True, stable=True)
    src = order[:, :r]
    dst = node_idx.gather(-1, src)
    unm = order[:, r:].sort(dim=-1).values               # class token first
    if return_scores:
        return src, dst, unm, node_max, second, scores
    return src, dst, unm, node_max, second


def _merge_sum(y: torch.Tensor, src: torch.Tensor, dst: torch.Tensor, unm: torch.Tensor) -> torch.Tensor:
    a, b = y[:, 0::2, :], y[:, 1::2, :]
    c = y.shape[-1]
    kept = a.gather(1, unm[..., None].expand(-1, -1, c))
    moved = a.gather(1, src[..., None].expand(-1, -1, c))
    b = b.scatter_reduce(1, dst[..., None].expand(-1, -1, c), moved, reduce="sum")
    return torch.cat([kept, b], dim=1)


def merge_wavg(x: torch.Tensor, size: Optional[torch.Tensor], src, dst, unm):
    """ToMe merge_wavg: x <- merge(x * size, sum) / merge(size, sum)."""
    if size is None:
        size = torch.ones_like(x[..., :1])
    xs = _merge_sum(x * size, src, dst, unm)
    s = _merge_sum(size, src, dst, unm)
    return xs / s, s


def _attention(h: torch.Tensor, layer: Dict[str, torch.Tensor], heads: int,
               size: Optional[torch.Tensor]):
    bsz, t, d = h.shape
    hd = d // heads
    qkv = F.linear(h, layer["qkv_w"], layer["qkv_b"]).reshape(bsz, t, 3, heads, hd)
    q, k, v = qkv.permute(2, 0, 3, 1, 4)                  # [B, H, t, hd]
    attn = (q @ k.transpose(-2, -1)) * (hd ** -0.5)
    if size is not None:
        attn = attn + size.log()[:, None, None, :, 0]       # proportional attention
    attn = attn.softmax(dim=-1)
    o = (attn @ v).transpose(1, 2).reshape(bsz, t, d)
    return F.linear(o, layer["proj_w"], layer["proj_b"]), k.mean(dim=1)


def forward(params: Dict[str, object], heads_by_task: Sequence[Dict[str, torch.Tensor]],
            images: torch.Tensor, task_ids: torch.Tensor, gamma: int, *, n_heads: int,
            patch: int, prompts: Optional[Sequence[torch.Tensor]] = None,
            prompt_mode: str = "accumulate", dtype: torch.dtype = torch.float32,
            forced: Optional[Sequence[Tuple[torch.Tensor, torch.Tensor, torch.Tensor]]] = None,
            max_classes: Optional[int] = None, shadow: bool = False) -> Tuple[torch.Tensor, OracleTrace]:
    """Token-adapted forward for one batch at one gamma.

    params     fp32 backbone weights (paper_2401_05031_b200.weights.init_backbone layout)
    heads_by_task  per task {"w": [C, D], "b": [C]}
    prompts    per task [L, gamma, D] (required when gamma > 0)
    forced     per merge layer (src, dst, unm) to replay instead of matching (teacher forcing)
    shadow     with forced: also run the matching on the oracle's own metric at every merge
               layer and keep its decisions and scores (MergeStep.own / .scores)
    returns    logits [B, C_max] (-inf beyond each task's C) and the merge trace
    """
    cv = lambda t: t.to(dtype)  # noqa: E731
    x = F.conv2d(cv(images), cv(params["patch_w"]), cv(params["patch_b"]), stride=patch)
    x = x.flatten(2).transpose(1, 2)
    bsz, _, d = x.shape
    cls = cv(params["cls"]).reshape(1, 1, d).expand(bsz, 1, d)
    x = torch.cat([cls, x], dim=1) + cv(params["pos"])[None]
    n_tokens = x.shape[1]
    layers = params["layers"]
    trace = OracleTrace()
    size: Optional[torch.Tensor] = None
    if gamma > 0 and prompts is None:
        raise ValueError("gamma > 0 needs prompts")
    merge_no = 0
    for li, lw_fp32 in enumerate(layers):
        lw = {k: cv(v) for k, v in lw_fp32.items()}
        if gamma > 0:
            block = torch.stack([cv(prompts[int(tk)][li]) for tk in task_ids])  # [B, gamma, D]
            if prompt_mode == "accumulate" or li == 0:
                x = torch.cat([x, block], dim=1)
            else:
                x = x.clone()
                x[:, n_tokens:n_tokens + gamma] = block
        t = x.shape[1]
        h = F.layer_norm(x, (d,), lw["ln1_w"], lw["ln1_b"], eps=1e-6)
        a, metric = _attention(h, lw, n_heads, size)
        x = x + a
        r = max(0, min(-gamma, (t - 1) // 2)) if gamma < 0 else 0
        if r > 0:
            own = scores = None
            if forced is not None:
                src, dst, unm = (v.to(torch.int64) for v in forced[merge_no])
                if shadow:
                    o_src, o_dst, o_unm, node_max, second, scores = bipartite_soft_matching(
                        metric, r, return_scores=True)
                    own = (o_src, o_dst, o_unm)
                else:
                    node_max = torch.full((bsz, (t + 1) // 2), float("nan"), dtype=dtype)
                    second = node_max.clone()
            else:
                src, dst, unm, node_max, second = bipartite_soft_matching(metric, r)
            trace.merges.append(MergeStep(li, t, r, src, dst, unm, node_max, second, own, scores))
            merge_no += 1
            x, size = merge_wavg(x, size, src, dst, unm)
        h = F.layer_norm(x, (d,), lw["ln2_w"], lw["ln2_b"], eps=1e-6)
        h = F.gelu(F.linear(h, lw["fc1_w"], lw["fc1_b"]))
        x = x + F.linear(h, lw["fc2_w"], lw["fc2_b"])
    cls_out = F.layer_norm(x[:, 0], (d,), cv(params["norm_w"]), cv(params["norm_b"]), eps=1e-6)
    c_max = max_classes or max(hd["w"].shape[0] for hd in heads_by_task)
    logits = torch.full((bsz, c_max), -math.inf, dtype=dtype)
    for i, tk in enumerate(task_ids.tolist()):
        hw = heads_by_task[tk]
        logits[i, : hw["w"].shape[0]] = F.linear(cls_out[i], cv(hw["w"]), cv(hw["b"]))
    return logits, trace
