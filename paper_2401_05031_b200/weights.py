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

__all__ = ["init_backbone", "init_head", "init_prompts", "synthetic_images", "from_timm_state_dict",
           "to_timm_state_dict", "load_checkpoint", "head_from_timm_state_dict", "from_hf_vit_state_dict",
           "head_from_hf_vit_state_dict"]


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


# ----------------------------------------------------------------------------- checkpoints
# timm VisionTransformer state-dict names (the paper's backbone) <-> the layout
# above.  Heads: timm's `head.weight` / `head.bias` become one TaskModel head; VPT-deep prompt
# tensors ([L, gamma, D]) are used as they are.
_TIMM_LAYER = {
    "ln1_w": "norm1.weight", "ln1_b": "norm1.bias", "qkv_w": "attn.qkv.weight", "qkv_b": "attn.qkv.bias",
    "proj_w": "attn.proj.weight", "proj_b": "attn.proj.bias", "ln2_w": "norm2.weight", "ln2_b": "norm2.bias",
    "fc1_w": "mlp.fc1.weight", "fc1_b": "mlp.fc1.bias", "fc2_w": "mlp.fc2.weight", "fc2_b": "mlp.fc2.bias",
}


def from_timm_state_dict(sd: Dict[str, torch.Tensor], cfg: ViTConfig) -> Dict[str, object]:
    """timm ``vit_*_patch*_224`` state dict -> fp32 master weights for TransformerModel.
    Raises KeyError naming the first missing tensor and ValueError on a shape mismatch."""
    def get(name, shape):
        t = sd[name].detach().to("cpu", torch.float32)
        if tuple(t.shape) != tuple(shape):
            raise ValueError(f"{name}: expected shape {tuple(shape)}, got {tuple(t.shape)}")
        return t.contiguous()

    d, p, n = cfg.dim, cfg.patch, cfg.n_tokens
    params: Dict[str, object] = {
        "patch_w": get("patch_embed.proj.weight", (d, 3, p, p)),
        "patch_b": get("patch_embed.proj.bias", (d,)),
        "cls": get("cls_token", (1, 1, d)).reshape(d),
        "pos": get("pos_embed", (1, n, d)).reshape(n, d),
        "norm_w": get("norm.weight", (d,)),
        "norm_b": get("norm.bias", (d,)),
    }
    shapes = {"ln1_w": (d,), "ln1_b": (d,), "qkv_w": (3 * d, d), "qkv_b": (3 * d,), "proj_w": (d, d),
              "proj_b": (d,), "ln2_w": (d,), "ln2_b": (d,), "fc1_w": (cfg.mlp_dim, d), "fc1_b": (cfg.mlp_dim,),
              "fc2_w": (d, cfg.mlp_dim), "fc2_b": (d,)}
    params["layers"] = [{k: get(f"blocks.{i}.{v}", shapes[k]) for k, v in _TIMM_LAYER.items()}
                        for i in range(cfg.depth)]
    return params


def to_timm_state_dict(params: Dict[str, object], cfg: ViTConfig) -> Dict[str, torch.Tensor]:
    """Inverse of ``from_timm_state_dict`` (backbone tensors only)."""
    d, n = cfg.dim, cfg.n_tokens
    sd = {"patch_embed.proj.weight": params["patch_w"], "patch_embed.proj.bias": params["patch_b"],
          "cls_token": params["cls"].reshape(1, 1, d), "pos_embed": params["pos"].reshape(1, n, d),
          "norm.weight": params["norm_w"], "norm.bias": params["norm_b"]}
    for i, lw in enumerate(params["layers"]):
        for k, v in _TIMM_LAYER.items():
            sd[f"blocks.{i}.{v}"] = lw[k]
    return sd


def load_checkpoint(path: str, cfg: ViTConfig) -> Dict[str, object]:
    """A timm checkpoint file (torch.save state dict, optionally under "model" / "state_dict";
    .safetensors if the package is importable) -> master weights."""
    if path.endswith(".safetensors"):
        from safetensors.torch import load_file  # optional dependency

        sd = load_file(path)
    else:
        sd = torch.load(path, map_location="cpu", weights_only=True)
        for key in ("model", "state_dict"):
            if isinstance(sd, dict) and key in sd and isinstance(sd[key], dict):
                sd = sd[key]
    return from_timm_state_dict(sd, cfg)


def head_from_timm_state_dict(sd: Dict[str, torch.Tensor], cfg: ViTConfig) -> Dict[str, torch.Tensor]:
    """timm ``head.weight`` [C, D] / ``head.bias`` [C] -> a task head {"w", "b"} (fp32), the
    classifier of one TaskModel."""
    w = sd["head.weight"].detach().to("cpu", torch.float32).contiguous()
    b = sd["head.bias"].detach().to("cpu", torch.float32).contiguous()
    if w.dim() != 2 or w.shape[1] != cfg.dim or tuple(b.shape) != (w.shape[0],):
        raise ValueError(f"head: expected [C, {cfg.dim}] / [C], got {tuple(w.shape)} / {tuple(b.shape)}")
    return {"w": w, "b": b}


# HuggingFace transformers ViT (models/vit/modeling_vit.py; the same architecture as timm's, with
# q / k / v as three Linear layers): a second checkpoint format that is installed offline here.
_HF_LAYER = {"ln1_w": "layernorm_before.weight", "ln1_b": "layernorm_before.bias",
             "proj_w": "attention.output.dense.weight", "proj_b": "attention.output.dense.bias",
             "ln2_w": "layernorm_after.weight", "ln2_b": "layernorm_after.bias",
             "fc1_w": "intermediate.dense.weight", "fc1_b": "intermediate.dense.bias",
             "fc2_w": "output.dense.weight", "fc2_b": "output.dense.bias"}


def from_hf_vit_state_dict(sd: Dict[str, torch.Tensor], cfg: ViTConfig) -> Dict[str, object]:
    """``ViTModel`` / ``ViTForImageClassification`` state dict (keys with or without the
    ``vit.`` prefix) -> fp32 master weights; q / k / v are concatenated in that order (the
    qkv row order s*D + h*hd + j of include/tokadapt_cuda.h)."""
    pre = "vit." if any(k.startswith("vit.") for k in sd) else ""

    def get(name, shape):
        t = sd[pre + name].detach().to("cpu", torch.float32)
        if tuple(t.shape) != tuple(shape):
            raise ValueError(f"{name}: expected shape {tuple(shape)}, got {tuple(t.shape)}")
        return t.contiguous()

    d, p, n, m = cfg.dim, cfg.patch, cfg.n_tokens, cfg.mlp_dim
    params: Dict[str, object] = {
        "patch_w": get("embeddings.patch_embeddings.projection.weight", (d, 3, p, p)),
        "patch_b": get("embeddings.patch_embeddings.projection.bias", (d,)),
        "cls": get("embeddings.cls_token", (1, 1, d)).reshape(d),
        "pos": get("embeddings.position_embeddings", (1, n, d)).reshape(n, d),
        "norm_w": get("layernorm.weight", (d,)),
        "norm_b": get("layernorm.bias", (d,)),
    }
    shapes = {"ln1_w": (d,), "ln1_b": (d,), "proj_w": (d, d), "proj_b": (d,), "ln2_w": (d,), "ln2_b": (d,),
              "fc1_w": (m, d), "fc1_b": (m,), "fc2_w": (d, m), "fc2_b": (d,)}
    layers = []
    for i in range(cfg.depth):
        base = f"encoder.layer.{i}."
        lw = {k: get(base + v, shapes[k]) for k, v in _HF_LAYER.items()}
        att = base + "attention.attention."
        lw["qkv_w"] = torch.cat([get(att + f"{s}.weight", (d, d)) for s in ("query", "key", "value")], 0)
        lw["qkv_b"] = torch.cat([get(att + f"{s}.bias", (d,)) for s in ("query", "key", "value")], 0)
        layers.append(lw)
    params["layers"] = layers
    return params


def head_from_hf_vit_state_dict(sd: Dict[str, torch.Tensor], cfg: ViTConfig) -> Dict[str, torch.Tensor]:
    """``ViTForImageClassification`` ``classifier.weight`` / ``classifier.bias`` -> task head."""
    return head_from_timm_state_dict({"head.weight": sd["classifier.weight"], "head.bias": sd["classifier.bias"]}, cfg)
