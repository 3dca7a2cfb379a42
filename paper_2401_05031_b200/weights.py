"""Seeded random-init weights shared by the oracle and the CUDA path.

There is no network for pretrained checkpoints, so both sides build
the same fp32 master weights from a CPU ``torch.Generator``: timm's ViT scheme (Linear
trunc_normal std .02; pos trunc_normal .02; cls N(0, 1e-6); conv default uniform), task
heads trunc_normal .02 (non-zero, so top-1 is meaningful), VPT prompts uniform
+-sqrt(6 / (3P^2 + D)) shaped [L, gamma, D].  Biases and LayerNorm affine parameters get
small random values instead of timm's zeros/ones so that every fused epilogue term is
exercised by the parity tests.
"""

from __future__ import annotations

import math
from typing import Dict, List, Optional

import torch

from .config import ViTConfig

__all__ = ["init_backbone", "init_head", "init_prompts", "synthetic_images"]


def _trunc_normal(shape, std: float, g: torch.Generator) -> torch.Tensor:
    # timm trunc_normal_(std, a=-2, b=2) in absolute units: sample N(0, std) truncated at +-2
    t = torch.empty(shape)
    lo, hi = -2.0, 2.0
    # inverse-CDF sampling (same construction as torch.nn.init.trunc_normal_)
    cdf = lambda x: (1.0 + math.erf(x / math.sqrt(2.0))) / 2.0  # noqa: E731
    a, b = cdf(lo / std), cdf(hi / std)
    t.uniform_(2 * a - 1, 2 * b - 1, generator=g)
    t.erfinv_().mul_(std * math.sqrt(2.0)).clamp_(min=lo, max=hi)
    return t


def _perturb(shape, scale: float, g: torch.Generator) -> torch.Tensor:
    return torch.randn(shape, generator=g) * scale


def init_backbone(cfg: ViTConfig, seed: int = 0) -> Dict[str, object]:
    """fp32 CPU master weights; layout matches timm's VisionTransformer state dict."""
    g = torch.Generator().manual_seed(seed)
    d, p = cfg.dim, cfg.patch
    fan_in = 3 * p * p
    bound = 1.0 / math.sqrt(fan_in)
    params: Dict[str, object] = {
        "patch_w": torch.empty(d, 3, p, p).uniform_(-bound, bound, generator=g),
        "patch_b": torch.empty(d).uniform_(-bound, bound, generator=g),
        "cls": torch.randn(d, generator=g) * 1e-6,
        "pos": _trunc_normal((cfg.n_tokens, d), 0.02, g),
        "norm_w": 1.0 + _perturb(d, 0.05, g),
        "norm_b": _perturb(d, 0.02, g),
    }
    layers: List[Dict[str, torch.Tensor]] = []
    for _ in range(cfg.depth):
        layers.append({
            "ln1_w": 1.0 + _perturb(d, 0.05, g),
            "ln1_b": _perturb(d, 0.02, g),
            "qkv_w": _trunc_normal((3 * d, d), 0.02, g),
            "qkv_b": _perturb(3 * d, 0.02, g),
            "proj_w": _trunc_normal((d, d), 0.02, g),
            "proj_b": _perturb(d, 0.02, g),
            "ln2_w": 1.0 + _perturb(d, 0.05, g),
            "ln2_b": _perturb(d, 0.02, g),
            "fc1_w": _trunc_normal((cfg.mlp_dim, d), 0.02, g),
            "fc1_b": _perturb(cfg.mlp_dim, 0.02, g),
            "fc2_w": _trunc_normal((d, cfg.mlp_dim), 0.02, g),
            "fc2_b": _perturb(d, 0.02, g),
        })
    params["layers"] = layers
    return params


def init_head(cfg: ViTConfig, classes: int, seed: int) -> Dict[str, torch.Tensor]:
    g = torch.Generator().manual_seed(10_000 + seed)
    return {"w": _trunc_normal((classes, cfg.dim), 0.02, g), "b": _perturb(classes, 0.02, g)}


def init_prompts(cfg: ViTConfig, gamma: int, seed: int) -> torch.Tensor:
    """VPT init: uniform(-v, v), v = sqrt(6 / (3 P^2 + D)); shape [L, gamma, D]."""
    if gamma <= 0:
        raise ValueError("prompts exist only for gamma > 0")
    g = torch.Generator().manual_seed(20_000 + 97 * seed + gamma)
    v = math.sqrt(6.0 / float(3 * cfg.patch * cfg.patch + cfg.dim))
    return torch.empty(cfg.depth, gamma, cfg.dim).uniform_(-v, v, generator=g)


def synthetic_images(batch: int, img: int, seed: int = 0,
                     device: Optional[torch.device] = None) -> torch.Tensor:
    """Normalised-image-like N(0, 1) inputs [B, 3, img, img] fp32."""
    g = torch.Generator(device=device or "cpu").manual_seed(seed)
    return torch.randn(batch, 3, img, img, generator=g, device=device)
