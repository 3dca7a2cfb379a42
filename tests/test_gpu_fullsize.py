"""Full-size properties of the CUDA forward at BASELINE configs[1] (ViT-B/16, b = 256, the bench
workload) that do not need the CPU oracle at that size (north_star):

* determinism: two forwards of the same batch give bit-identical logits and merge traces;
* permutation equivariance, bit for bit: an image's logits and merge decisions do not depend on
  where it sits in the batch (rows never mix: GEMM tiles accumulate K in a fixed order,
  attention / match / merge work per image);
* batch invariance across kernel shapes: a b = 8 sample agrees with its rows of the b = 256
  forward within the bf16 bound wherever the merge decisions agree;
* oracle parity of the sample: the 8 sampled images against the CPU oracle with the oracle's
  merge indices forced (the bf16 bound of test_gpu_forward.py), which batch invariance then
  carries to the full batch."""

import pytest
import torch

from tests import helpers

pytestmark = pytest.mark.gpu

B = 256
SAMPLE = [0, 37, 74, 111, 148, 185, 222, 255]
from tests.test_gpu_forward import BF16_TOL  # noqa: E402
_MODELS = {}


def _model(gamma):
    key = gamma > 0
    if key not in _MODELS:
        cfg, params = helpers.backbone("vit_b16")
        tasks = helpers.task_params(cfg, (10, 100), [8, 16])
        _MODELS[key] = (cfg, params, tasks, helpers.serve_model(cfg, params, tasks, dtype="bf16"))
    return _MODELS[key]


def _forward(sm, imgs, ids, gamma, forced=None):
    bb = sm.backbone
    n = imgs.shape[0]
    n_tr = bb.trace_len(n, gamma)
    trace = torch.full((max(n_tr, 1),), -1, dtype=torch.int32, device="cuda")
    out = bb.forward_raw(imgs, ids, gamma, trace=trace if n_tr and forced is None else None,
                         forced_trace=forced if n_tr else None)
    torch.cuda.synchronize()
    tr = helpers.split_trace(trace.cpu(), bb.schedule(gamma), n) if n_tr and forced is None else []
    return out.float().cpu(), tr


def _inputs(cfg):
    imgs = helpers.synthetic_images(B, cfg.img, seed=3).cuda()
    ids = (torch.arange(B, dtype=torch.int32) % 2).cuda()
    return imgs, ids


@pytest.mark.parametrize("gamma", [-16, -8, 0, 8, 16])
def test_fullsize_deterministic(gamma):
    cfg, _, _, sm = _model(gamma)
    imgs, ids = _inputs(cfg)
    a, ta = _forward(sm, imgs, ids, gamma)
    b, tb = _forward(sm, imgs, ids, gamma)
    assert torch.equal(a, b)
    for (s1, d1, u1), (s2, d2, u2) in zip(ta, tb):
        assert torch.equal(s1, s2) and torch.equal(d1, d2) and torch.equal(u1, u2)


@pytest.mark.parametrize("gamma", [-16, -8, 0, 8, 16])
def test_fullsize_batch_invariance(gamma):
    """The sample as its own b = 8 batch runs other kernel shapes (the small-M GEMM tiles, their
    row statistics), so bitwise equality is not expected: where an image's merge decisions agree
    the logits agree within the bf16 bound; decisions may flip on near-ties (reported)."""
    cfg, _, _, sm = _model(gamma)
    imgs, ids = _inputs(cfg)
    full, tfull = _forward(sm, imgs, ids, gamma)
    idx = torch.tensor(SAMPLE)
    part, tpart = _forward(sm, imgs[idx.cuda()].contiguous(), ids[idx.cuda()].contiguous(), gamma)
    same = torch.ones(len(SAMPLE), dtype=torch.bool)
    for (s1, d1, u1), (s2, d2, u2) in zip(tfull, tpart):
        same &= (s1[idx] == s2).all(1) & (d1[idx] == d2).all(1) & (u1[idx] == u2).all(1)
    fin = torch.isfinite(part)
    scale = part[fin].abs().max().item()
    diff = torch.where(fin, (full[idx] - part).abs(), torch.zeros_like(part)).amax(1)
    print(f"gamma {gamma}: {int(same.sum())}/{len(SAMPLE)} images with identical merge traces, "
          f"max |dlogit| there {diff[same].max().item() if same.any() else 0:.3e}")
    assert torch.equal(torch.isfinite(full[idx]), fin)
    assert (diff[same] <= BF16_TOL * scale).all()


@pytest.mark.parametrize("gamma", [-16, -8, 0, 8, 16])
def test_fullsize_permutation(gamma):
    cfg, _, _, sm = _model(gamma)
    imgs, ids = _inputs(cfg)
    full, tfull = _forward(sm, imgs, ids, gamma)
    perm = torch.randperm(B, generator=torch.Generator().manual_seed(gamma + 100))
    pf, tp = _forward(sm, imgs[perm.cuda()].contiguous(), ids[perm.cuda()].contiguous(), gamma)
    assert torch.equal(full[perm], pf)
    for (s1, d1, u1), (s2, d2, u2) in zip(tfull, tp):
        assert torch.equal(s1[perm], s2) and torch.equal(d1[perm], d2) and torch.equal(u1[perm], u2)


@pytest.mark.parametrize("gamma", [-16, -8, 0, 8, 16])
def test_fullsize_sample_vs_oracle(gamma):
    cfg, params, tasks, sm = _model(gamma)
    imgs, ids = _inputs(cfg)
    idx = torch.tensor(SAMPLE)
    full, _ = _forward(sm, imgs, ids, gamma)
    s_imgs = imgs[idx.cuda()].cpu()
    s_ids = ids[idx.cuda()].cpu().long()
    ref, tr = helpers.oracle_forward(cfg, params, tasks, s_imgs, s_ids, gamma)
    n_tr = sm.backbone.trace_len(len(SAMPLE), gamma)
    forced = tr.flat_int32().cuda() if n_tr else None
    part, _ = _forward(sm, s_imgs.cuda(), s_ids.to(torch.int32).cuda(), gamma, forced=forced)
    ref = ref.float()
    scale = ref[torch.isfinite(ref)].abs().max().item()
    fin = torch.isfinite(ref)
    err = (part[fin] - ref[fin]).abs().max().item()
    assert err <= BF16_TOL * scale, f"index-forced |dlogit| {err:.3e} > {BF16_TOL} * {scale:.3e}"
    # the sample inside the full batch, free-running, agrees with the forced run on top-1
    # wherever the oracle's top-2 margin is well above the bound
    top2 = torch.where(fin, ref, torch.full_like(ref, -float("inf"))).topk(2, dim=1).values
    sure = (top2[:, 0] - top2[:, 1]) > 2 * BF16_TOL * scale
    assert torch.equal(full[idx].argmax(1)[sure], ref.argmax(1)[sure])
