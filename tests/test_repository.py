"""Task registry / prompt repository and checkpoint import
(timm head tensors, HuggingFace transformers ViT state dicts) -- host side, no GPU."""

import pytest
import torch

from paper_2401_05031_b200.config import VIT_CONFIGS
from paper_2401_05031_b200.errors import ConfigError, ProfileGapError
from paper_2401_05031_b200.repository import PromptRepository
from paper_2401_05031_b200.weights import (from_hf_vit_state_dict, from_timm_state_dict, head_from_hf_vit_state_dict,
                                           head_from_timm_state_dict, init_backbone, init_head, init_prompts,
                                           to_timm_state_dict)


def test_repository_round_trip(tmp_path):
    cfg = VIT_CONFIGS["vit_tiny"]
    repo = PromptRepository(str(tmp_path))
    h = init_head(cfg, 10, 0)
    repo.register_task("cifar10", h["w"], h["b"], {8: init_prompts(cfg, 8, 0)})
    repo.add_prompts("cifar10", 2, init_prompts(cfg, 2, 0))
    h2 = init_head(cfg, 100, 1)
    repo.register_task("cifar100", h2["w"], h2["b"])
    again = PromptRepository(str(tmp_path))  # reloaded from disk
    assert again.tasks() == ["cifar10", "cifar100"]
    assert again.gammas("cifar10") == [2, 8] and again.gammas("cifar100") == []
    assert torch.equal(again.prompts("cifar10", 8), init_prompts(cfg, 8, 0))
    tm = again.task_model("cifar10")
    assert tm.classes == 10 and sorted(tm.prompts) == [2, 8] and torch.equal(tm.head_w, h["w"])
    with pytest.raises(ProfileGapError) as ei:
        again.prompts("cifar100", 8)
    assert ei.value.task == "cifar100" and ei.value.gamma == 8 and ei.value.kind == "prompt"
    with pytest.raises(ConfigError):
        again.add_prompts("cifar10", 4, torch.zeros(cfg.depth, 3, cfg.dim))  # gamma mismatch
    with pytest.raises(ConfigError):
        again.register_task("cifar10", h2["w"], h2["b"])  # head shape changed
    with pytest.raises(KeyError):
        again.head("imagenet")


def test_timm_state_dict_with_head():
    cfg = VIT_CONFIGS["vit_tiny"]
    params = init_backbone(cfg, 3)
    sd = to_timm_state_dict(params, cfg)
    h = init_head(cfg, 10, 2)
    sd["head.weight"], sd["head.bias"] = h["w"], h["b"]
    back = from_timm_state_dict(sd, cfg)
    head = head_from_timm_state_dict(sd, cfg)
    assert torch.equal(head["w"], h["w"]) and torch.equal(head["b"], h["b"])
    assert torch.equal(back["layers"][2]["qkv_w"], params["layers"][2]["qkv_w"])
    with pytest.raises(ValueError):
        head_from_timm_state_dict({"head.weight": torch.zeros(10, 7), "head.bias": torch.zeros(10)}, cfg)


def test_hf_vit_checkpoint_import():
    """A real third-party checkpoint format: transformers' ViTForImageClassification state dict
    maps onto the backbone + head layout exactly (q/k/v concatenated in qkv row order)."""
    pytest.importorskip("transformers")
    from tests.golden.make_hf_golden import hf_model

    cfg = VIT_CONFIGS["vit_tiny"]
    params = init_backbone(cfg, 5)
    head = init_head(cfg, 10, 5)
    m = hf_model(cfg, params, head)  # our weights placed into transformers' modules
    sd = m.state_dict()
    back = from_hf_vit_state_dict(sd, cfg)
    hb = head_from_hf_vit_state_dict(sd, cfg)
    for k in ("patch_w", "patch_b", "cls", "pos", "norm_w", "norm_b"):
        assert torch.equal(back[k], params[k].float()), k
    for a, b in zip(back["layers"], params["layers"]):
        for k in b:
            assert torch.equal(a[k], b[k].float()), k
    assert torch.equal(hb["w"], head["w"]) and torch.equal(hb["b"], head["b"])
