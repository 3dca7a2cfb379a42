"""ViT configurations and the per-layer token schedule of the token-adapted forward.

Sizes follow PAPER.md:545 (ViT-B/16) and SURVEY.md §8a; the schedule is ToMe's
``parse_r`` with a constant r and the per-layer cap r_l = min(|gamma|, (t_l - 1) // 2)
(class token protected), or gamma prompt rows per layer.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import List, Tuple

__all__ = ["ViTConfig", "VIT_CONFIGS", "token_schedule", "flops_per_image", "PROMPT_MODES"]

PROMPT_MODES = ("accumulate", "replace")


@dataclass(frozen=True)
class ViTConfig:
    name: str
    dim: int
    depth: int
    heads: int
    mlp_dim: int
    patch: int
    img: int = 224

    @property
    def head_dim(self) -> int:
        return self.dim // self.heads

    @property
    def grid(self) -> int:
        return self.img // self.patch

    @property
    def n_patches(self) -> int:
        return self.grid * self.grid

    @property
    def n_tokens(self) -> int:
        return self.n_patches + 1

    @property
    def patch_k(self) -> int:
        return 3 * self.patch * self.patch

    @property
    def patch_k_padded(self) -> int:
        return (self.patch_k + 63) // 64 * 64


VIT_CONFIGS = {
    "vit_b16": ViTConfig("vit_b16", 768, 12, 12, 3072, 16),
    "vit_l16": ViTConfig("vit_l16", 1024, 24, 16, 4096, 16),
    "vit_h14": ViTConfig("vit_h14", 1280, 32, 16, 5120, 14),
    # small configurations for fast parity tests (same code paths, shapes the kernels accept)
    "vit_tiny": ViTConfig("vit_tiny", 256, 4, 4, 1024, 16, img=64),
    "vit_small_b": ViTConfig("vit_small_b", 768, 4, 12, 3072, 16),
}


def token_schedule(cfg: ViTConfig, gamma: int, prompt_mode: str = "accumulate") -> Tuple[List[int], List[int]]:
    """(t_l, r_l) per layer: tokens entering layer l (after its prompt rows) and tokens
    merged in layer l."""
    if prompt_mode not in PROMPT_MODES:
        raise ValueError(f"prompt_mode must be one of {PROMPT_MODES}")
    n = cfg.n_tokens
    ts: List[int] = []
    rs: List[int] = []
    t = n
    for layer in range(cfg.depth):
        if gamma > 0:
            tl = n + gamma * (layer + 1) if prompt_mode == "accumulate" else n + gamma
            rl = 0
        else:
            tl = t
            rl = max(0, min(-gamma, (tl - 1) // 2)) if gamma < 0 else 0
        ts.append(tl)
        rs.append(rl)
        t = tl - rl
    return ts, rs


def flops_per_image(cfg: ViTConfig, gamma: int, prompt_mode: str = "accumulate") -> float:
    """Algorithmic FLOPs per image: patch GEMM + per layer
    8 t D^2 (QKV + proj) + 4 t^2 D (attention) + 4 t' D MLP (fc1 + fc2)
    + 2 ceil(t/2) floor(t/2) hd (match, merge layers only).  Head excluded."""
    d = cfg.dim
    f = 2.0 * cfg.n_patches * cfg.patch_k * d
    ts, rs = token_schedule(cfg, gamma, prompt_mode)
    for t, r in zip(ts, rs):
        tp = t - r
        f += 8.0 * t * d * d + 4.0 * t * t * d + 4.0 * tp * d * cfg.mlp_dim
        if r > 0:
            f += 2.0 * ((t + 1) // 2) * (t // 2) * cfg.head_dim
    return f
