"""Independent third-party pin of the oracle: the same seeded ViT run through HuggingFace
`transformers` (installed in this image: transformers 5.5.0, `models/vit/modeling_vit.py`
ViTForImageClassification = timm's pre-norm ViT: conv patch embed, cls + pos, layernorm_before
-> self-attention -> residual -> layernorm_after -> GELU(erf) MLP -> residual, final LayerNorm,
classifier on the cls row), with the paper's two token adaptations applied the way their
upstream projects patch a ViT:

  * ToMe (facebookresearch/ToMe, unpinned; not installed): the ToMeBlock / ToMeAttention patch
    of tome/patch/timm.py (prop_attn=True: softmax(qk^T s + log size), metric = k.mean(heads),
    merge after attention and before the MLP) and tome/merge.py bipartite_soft_matching /
    merge_wavg, restated below in upstream's own structure (max / argsort / gather /
    scatter_reduce over the alternating split), applied over HF's own layer modules; the
    log-size bias enters through HF's eager_attention_forward attention_mask argument;
  * VPT-deep prompts (accumulate): gamma prompt rows appended before each HF layer.

Everything below the ToMe/VPT glue is transformers' code.  Run in fp64 on CPU; the oracle
(oracle/vit_oracle.py, written independently from SURVEY.md Appendix A) must reproduce the
logits and merge traces saved here (tests/test_oracle.py::test_oracle_matches_hf_golden), and
when transformers is importable the comparison also runs live.

  python tests/golden/make_hf_golden.py      (writes tests/golden/hf_vit_golden.npz)
"""

from __future__ import annotations

import math
import os
import sys

import numpy as np
import torch

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

# (config, batch, gammas): ViT-tiny covers every gamma kind cheaply; ViT-B/16 is the bench model
CASES = [("vit_tiny", 4, (-8, -3, 0, 4)), ("vit_b16", 2, (-16, -8, 0, 8))]


def hf_model(cfg, params, head):
    from transformers import ViTConfig, ViTForImageClassification

    hc = ViTConfig(hidden_size=cfg.dim, num_hidden_layers=cfg.depth, num_attention_heads=cfg.heads,
                   intermediate_size=cfg.mlp_dim, hidden_act="gelu", hidden_dropout_prob=0.0,
                   attention_probs_dropout_prob=0.0, layer_norm_eps=1e-6, image_size=cfg.img,
                   patch_size=cfg.patch, num_channels=3, qkv_bias=True, num_labels=head["w"].shape[0])
    hc._attn_implementation = "eager"
    m = ViTForImageClassification(hc).double().eval()
    D = cfg.dim
    with torch.no_grad():
        emb = m.vit.embeddings
        emb.cls_token.copy_(params["cls"].reshape(1, 1, D))
        emb.position_embeddings.copy_(params["pos"].reshape(1, -1, D))
        emb.patch_embeddings.projection.weight.copy_(params["patch_w"])
        emb.patch_embeddings.projection.bias.copy_(params["patch_b"])
        for layer, lw in zip(m.vit.encoder.layer, params["layers"]):
            layer.layernorm_before.weight.copy_(lw["ln1_w"]); layer.layernorm_before.bias.copy_(lw["ln1_b"])
            att = layer.attention.attention
            for i, lin in enumerate((att.query, att.key, att.value)):
                lin.weight.copy_(lw["qkv_w"][i * D:(i + 1) * D]); lin.bias.copy_(lw["qkv_b"][i * D:(i + 1) * D])
            layer.attention.output.dense.weight.copy_(lw["proj_w"]); layer.attention.output.dense.bias.copy_(lw["proj_b"])
            layer.layernorm_after.weight.copy_(lw["ln2_w"]); layer.layernorm_after.bias.copy_(lw["ln2_b"])
            layer.intermediate.dense.weight.copy_(lw["fc1_w"]); layer.intermediate.dense.bias.copy_(lw["fc1_b"])
            layer.output.dense.weight.copy_(lw["fc2_w"]); layer.output.dense.bias.copy_(lw["fc2_b"])
        m.vit.layernorm.weight.copy_(params["norm_w"]); m.vit.layernorm.bias.copy_(params["norm_b"])
        m.classifier.weight.copy_(head["w"]); m.classifier.bias.copy_(head["b"])
    return m


# ---- ToMe, upstream structure (tome/merge.py), class token protected
def tome_bipartite_soft_matching(metric, r):
    t = metric.shape[1]
    r = min(r, (t - 1) // 2)
    metric = metric / metric.norm(dim=-1, keepdim=True)
    a, b = metric[..., ::2, :], metric[..., 1::2, :]
    scores = a @ b.transpose(-1, -2)
    scores[..., 0, :] = -math.inf
    node_max, node_idx = scores.max(dim=-1)
    edge_idx = node_max.argsort(dim=-1, descending=True)[..., None]
    unm_idx = edge_idx[..., r:, :]
    src_idx = edge_idx[..., :r, :]
    dst_idx = node_idx[..., None].gather(dim=-2, index=src_idx)
    unm_idx = unm_idx.sort(dim=1)[0]

    def merge(x, mode="mean"):
        src, dst = x[..., ::2, :], x[..., 1::2, :]
        n, t1, c = src.shape
        unm = src.gather(dim=-2, index=unm_idx.expand(n, t1 - r, c))
        src = src.gather(dim=-2, index=src_idx.expand(n, r, c))
        dst = dst.scatter_reduce(-2, dst_idx.expand(n, r, c), src, reduce=mode)
        return torch.cat([unm, dst], dim=1)

    return merge, (src_idx[..., 0], dst_idx[..., 0], unm_idx[..., 0])


def tome_merge_wavg(merge, x, size=None):
    if size is None:
        size = torch.ones_like(x[..., 0, None])
    x = merge(x * size, mode="sum")
    size = merge(size, mode="sum")
    return x / size, size


def hf_tokenadapt_forward(m, cfg, images, gamma, prompts=None):
    """HF modules + ToMe block patch (gamma < 0) / VPT-deep accumulate prompts (gamma > 0)."""
    from transformers.models.vit.modeling_vit import eager_attention_forward

    if gamma == 0:  # stock transformers forward
        with torch.no_grad():
            return m(pixel_values=images).logits, []
    with torch.no_grad():
        x = m.vit.embeddings(images)
        size, trace = None, []
        bsz, H = x.shape[0], cfg.heads
        for li, layer in enumerate(m.vit.encoder.layer):
            if gamma > 0:
                x = torch.cat([x, prompts[li][None].expand(bsz, -1, -1)], dim=1)
            t = x.shape[1]
            h = layer.layernorm_before(x)
            att = layer.attention.attention
            shp = (bsz, t, H, cfg.head_dim)
            q = att.query(h).view(shp).transpose(1, 2)
            k = att.key(h).view(shp).transpose(1, 2)
            v = att.value(h).view(shp).transpose(1, 2)
            mask = None if size is None else size.log()[:, None, None, :, 0]
            ctx, _ = eager_attention_forward(att, q, k, v, mask, scaling=att.scaling)
            x = x + layer.attention.output.dense(ctx.reshape(bsz, t, -1))
            r = min(-gamma, (t - 1) // 2) if gamma < 0 else 0
            if r > 0:
                merge, idx = tome_bipartite_soft_matching(k.mean(1), r)
                trace.append(idx)
                x, size = tome_merge_wavg(merge, x, size)
            x = layer.output(layer.intermediate(layer.layernorm_after(x)), x)
        x = m.vit.layernorm(x)
        return m.classifier(x[:, 0]), trace


def main():
    from paper_2401_05031_b200.config import VIT_CONFIGS
    from paper_2401_05031_b200.weights import init_backbone, init_head, init_prompts, synthetic_images

    torch.manual_seed(0)
    out = {}
    for name, batch, gammas in CASES:
        cfg = VIT_CONFIGS[name]
        params = init_backbone(cfg, 0)
        head = init_head(cfg, 10, 0)
        params64 = {k: (v.double() if torch.is_tensor(v) else [{kk: vv.double() for kk, vv in l.items()} for l in v])
                    for k, v in params.items()}
        m = hf_model(cfg, params64, {k: v.double() for k, v in head.items()})
        imgs = synthetic_images(batch, cfg.img, seed=21).double()
        for g in gammas:
            pr = init_prompts(cfg, g, 0).double() if g > 0 else None
            logits, trace = hf_tokenadapt_forward(m, cfg, imgs, g, pr)
            key = f"{name}_g{g}"
            out[f"{key}_logits"] = logits.numpy()
            for i, (s, d, u) in enumerate(trace):
                out[f"{key}_l{i}_src"] = s.numpy().astype(np.int32)
                out[f"{key}_l{i}_dst"] = d.numpy().astype(np.int32)
                out[f"{key}_l{i}_unm"] = u.numpy().astype(np.int32)
            out[f"{key}_nmerge"] = np.array(len(trace))
    import transformers

    out["transformers_version"] = np.array(transformers.__version__)
    np.savez_compressed(os.path.join(HERE, "hf_vit_golden.npz"), **out)
    print("wrote", os.path.join(HERE, "hf_vit_golden.npz"), len(out), "arrays")


if __name__ == "__main__":
    main()
