"""Pins the CPU oracle (oracle/vit_oracle.py), which is our restatement of the path (the
reference ships none; parity unpinned):

  1. an independent pure-Python loop restatement of SURVEY.md Appendix A `match` / `merge`
     (upstream ToMe bipartite_soft_matching + merge_wavg semantics with the explicit tie
     rules) agrees with the vectorised oracle, including injected exact ties;
  2. structural invariants: sizes sum to N, cls stays at row 0, t' = t - r_l, schedule;
  3. fp32 and fp64 oracles choose identical merge index sets (config 1);
  4. the oracle reproduces the frozen goldens in tests/golden/."""

import math
import os

import numpy as np
import pytest
import torch

from oracle import vit_oracle
from tests import helpers

HERE = os.path.dirname(os.path.abspath(__file__))


# ---------------------------------------------------------------- loop restatement
def match_loops(metric, r):
    """Appendix A `match`, one image, plain Python floats (fp64)."""
    t, c = len(metric), len(metric[0])
    m = []
    for row in metric:
        n = math.sqrt(sum(v * v for v in row))
        m.append([v / n for v in row])
    A, B = m[0::2], m[1::2]
    node_max, node_idx = [], []
    for i, a in enumerate(A):
        if i == 0:
            node_max.append(-math.inf)
            node_idx.append(0)
            continue
        best, bj = -math.inf, 0
        for j, b in enumerate(B):
            s = sum(x * y for x, y in zip(a, b))
            if s > best:  # strict: lowest column on ties
                best, bj = s, j
        node_max.append(best)
        node_idx.append(bj)
    order = sorted(range(len(A)), key=lambda i: (-node_max[i], i))  # stable descending
    src = order[:r]
    dst = [node_idx[i] for i in src]
    unm = sorted(order[r:])
    return src, dst, unm


def merge_loops(x, size, src, dst, unm):
    """Appendix A `merge` of x * size and size (sum), then divide; one image."""
    A = list(range(0, len(x), 2))
    Bt = list(range(1, len(x), 2))
    out_x, out_s = [], []
    for u in unm:
        tok = A[u]
        out_x.append([v * size[tok] / size[tok] for v in x[tok]])
        out_s.append(size[tok])
    for j, tok in enumerate(Bt):
        acc = [v * size[tok] for v in x[tok]]
        s = size[tok]
        for q, d in enumerate(dst):
            if d == j:
                st = A[src[q]]
                acc = [a + v * size[st] for a, v in zip(acc, x[st])]
                s += size[st]
        out_x.append([a / s for a in acc])
        out_s.append(s)
    return out_x, out_s


@pytest.mark.parametrize("t,r,c,seed", [(9, 3, 8, 0), (17, 8, 16, 1), (21, 10, 8, 2), (4, 1, 4, 3),
                                        (33, 5, 12, 4), (3, 1, 5, 5)])
def test_match_matches_loop_restatement(t, r, c, seed):
    g = torch.Generator().manual_seed(seed)
    metric = torch.randn(2, t, c, generator=g, dtype=torch.float64)
    metric[:, min(5, t - 1)] = metric[:, min(3, t - 1)]  # exact argmax / rank ties
    if t > 9:
        metric[:, 8] = metric[:, 2]
    src, dst, unm, _, _ = vit_oracle.bipartite_soft_matching(metric.clone(), r)
    for b in range(2):
        s2, d2, u2 = match_loops(metric[b].tolist(), r)
        assert src[b].tolist() == s2 and dst[b].tolist() == d2 and unm[b].tolist() == u2


@pytest.mark.parametrize("t,r,seed", [(9, 3, 0), (17, 8, 1), (21, 10, 2)])
def test_merge_matches_loop_restatement(t, r, seed):
    g = torch.Generator().manual_seed(seed)
    x = torch.randn(1, t, 6, generator=g, dtype=torch.float64)
    size = torch.randint(1, 5, (1, t, 1), generator=g).double()
    metric = torch.randn(1, t, 8, generator=g, dtype=torch.float64)
    src, dst, unm, _, _ = vit_oracle.bipartite_soft_matching(metric, r)
    xm, sm = vit_oracle.merge_wavg(x, size, src, dst, unm)
    lx, ls = merge_loops(x[0].tolist(), size[0, :, 0].tolist(), src[0].tolist(), dst[0].tolist(),
                         unm[0].tolist())
    np.testing.assert_allclose(xm[0].numpy(), np.array(lx), rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(sm[0, :, 0].numpy(), np.array(ls), rtol=0, atol=0)


# ---------------------------------------------------------------- invariants
@pytest.mark.parametrize("gamma", [-8, -3, -1])
def test_merge_invariants(gamma):
    cfg, params = helpers.backbone("vit_tiny")
    tasks = helpers.task_params(cfg, (10,), [])
    imgs = helpers.synthetic_images(3, cfg.img, seed=4)
    ids = torch.zeros(3, dtype=torch.int64)
    _, tr = helpers.oracle_forward(cfg, params, tasks, imgs, ids, gamma)
    ts, rs = vit_oracle.token_schedule(cfg.n_tokens, cfg.depth, gamma)
    steps = [(t, r) for t, r in zip(ts, rs) if r > 0]
    assert [(m.t, m.r) for m in tr.merges] == steps
    for m in tr.merges:
        na = (m.t + 1) // 2
        for b in range(3):
            # src/unm partition the A set; cls (0) never merged; unm ascending
            assert sorted(m.src[b].tolist() + m.unm[b].tolist()) == list(range(na))
            assert 0 in m.unm[b].tolist() and m.unm[b].tolist() == sorted(m.unm[b].tolist())
            assert all(0 <= d < m.t // 2 for d in m.dst[b].tolist())


def test_size_conservation_and_cls_row():
    cfg, params = helpers.backbone("vit_tiny")
    g = torch.Generator().manual_seed(3)
    x = torch.randn(2, cfg.n_tokens, 4, generator=g)
    size = None
    t = cfg.n_tokens
    for r in (8, 4, 2):
        metric = torch.randn(2, t, 8, generator=g)
        src, dst, unm, _, _ = vit_oracle.bipartite_soft_matching(metric, r)
        cls_before = x[:, 0].clone()
        x, size = vit_oracle.merge_wavg(x, size, src, dst, unm)
        t -= r
        assert x.shape[1] == t
        assert torch.allclose(size.sum(dim=1)[:, 0], torch.full((2,), float(cfg.n_tokens)))
        assert torch.allclose(x[:, 0], cls_before)  # cls is never merged and stays first


def test_schedule_appendix_b():
    from paper_2401_05031_b200.config import VIT_CONFIGS, flops_per_image, token_schedule

    b16, l16, h14 = VIT_CONFIGS["vit_b16"], VIT_CONFIGS["vit_l16"], VIT_CONFIGS["vit_h14"]
    assert token_schedule(b16, -16)[0] == [197, 181, 165, 149, 133, 117, 101, 85, 69, 53, 37, 21]
    assert token_schedule(b16, -16)[1][-1] == 10
    assert token_schedule(b16, -8)[0] == list(range(197, 108, -8))
    assert token_schedule(b16, 16)[0] == [197 + 16 * (l + 1) for l in range(12)]
    assert token_schedule(b16, 16, "replace")[0] == [213] * 12
    ts, rs = token_schedule(l16, -16)
    assert ts[11:18] == [21, 11, 6, 4, 3, 2, 2] and rs[16:] == [0] * 8
    ts, rs = token_schedule(h14, -24)
    assert ts[:3] == [257, 233, 209] and ts[15:] == [2] * 17
    # SURVEY.md §6 / §8a GFLOP per image
    for cfg, g, v in [(b16, -16, 17.548), (b16, -8, 26.216), (b16, 0, 35.126), (b16, 8, 44.842),
                      (b16, 16, 54.814), (l16, -16, 31.701), (l16, 0, 123.107), (l16, 16, 256.788),
                      (h14, -24, 56.791)]:
        assert flops_per_image(cfg, g) / 1e9 == pytest.approx(v, abs=2e-3)
    assert flops_per_image(b16, 16, "replace") / 1e9 == pytest.approx(38.086, abs=2e-3)


# ---------------------------------------------------------------- fp32 vs fp64, goldens
def test_fp32_fp64_index_sets_config1():
    d = np.load(os.path.join(HERE, "golden", "oracle_b16_cfg1.npz"))
    assert np.array_equal(d["trace32"], d["trace64"])  # 0 differing pairs
    assert d["topr_gap_fp64"].min() > 0  # no exact ties at the top-r boundary
    fin = lambda a: np.where(np.isinf(a), 0, a)  # noqa: E731
    np.testing.assert_allclose(fin(d["logits32"]), fin(d["logits64"]), rtol=1e-4, atol=1e-5)


@pytest.mark.parametrize("gamma,mode", [(-8, "accumulate"), (-4, "accumulate"), (-1, "accumulate"),
                                        (0, "accumulate"), (2, "accumulate"), (2, "replace"),
                                        (8, "accumulate"), (8, "replace")])
def test_oracle_reproduces_goldens(gamma, mode):
    d = np.load(os.path.join(HERE, "golden", "oracle_tiny.npz"))
    cfg, params = helpers.backbone("vit_tiny")
    tasks = helpers.task_params(cfg, (10, 100), [gamma] if gamma > 0 else [])
    imgs = helpers.synthetic_images(6, cfg.img, seed=0)
    ids = torch.arange(6) % 2
    logits, tr = helpers.oracle_forward(cfg, params, tasks, imgs, ids, gamma, mode)
    key = f"g{gamma}_{mode}"
    assert np.array_equal(tr.flat_int32().numpy(), d[key + "_trace"])
    fin = lambda a: np.where(np.isinf(a), 0, a)  # noqa: E731
    np.testing.assert_allclose(fin(logits.numpy()), fin(d[key + "_logits"]), rtol=1e-5, atol=1e-6)


@pytest.mark.slow
def test_oracle_reproduces_config1_golden():
    d = np.load(os.path.join(HERE, "golden", "oracle_b16_cfg1.npz"))
    cfg, params = helpers.backbone("vit_b16")
    tasks = helpers.task_params(cfg, (10, 100), [])
    imgs = helpers.synthetic_images(8, cfg.img, seed=0)
    logits, tr = helpers.oracle_forward(cfg, params, tasks, imgs, torch.arange(8) % 2, -8)
    assert np.array_equal(tr.flat_int32().numpy(), d["trace32"])


def test_weights_deterministic():
    from paper_2401_05031_b200.config import VIT_CONFIGS
    from paper_2401_05031_b200.weights import init_backbone, init_prompts

    cfg = VIT_CONFIGS["vit_tiny"]
    a, b = init_backbone(cfg, 0), init_backbone(cfg, 0)
    assert torch.equal(a["layers"][1]["fc1_w"], b["layers"][1]["fc1_w"])
    p = init_prompts(cfg, 4, 0)
    v = math.sqrt(6.0 / (3 * 16 * 16 + cfg.dim))
    assert p.shape == (cfg.depth, 4, cfg.dim) and p.abs().max() <= v


# ---------------------------------------------------------------- third-party pin (transformers)
def _hf_golden_cases():
    from tests.golden.make_hf_golden import CASES

    return [(n, b, g) for n, b, gs in CASES for g in gs]


@pytest.mark.parametrize("name,batch,gamma", _hf_golden_cases())
def test_oracle_matches_hf_golden(name, batch, gamma):
    """The oracle (fp64) reproduces the same seeded ViT run through HuggingFace transformers'
    ViTForImageClassification modules with upstream-structured ToMe / VPT glue
    (tests/golden/make_hf_golden.py): identical merge traces, logits to fp64 rounding."""
    gold = np.load(os.path.join(HERE, "golden", "hf_vit_golden.npz"))
    from paper_2401_05031_b200.config import VIT_CONFIGS
    from paper_2401_05031_b200.weights import init_head, init_prompts, synthetic_images

    cfg, params = helpers.backbone(name)
    head = init_head(cfg, 10, 0)
    tasks = [{"name": "t0", "head": head, "prompts": {gamma: init_prompts(cfg, gamma, 0)} if gamma > 0 else {}}]
    imgs = synthetic_images(batch, cfg.img, seed=21)
    key = f"{name}_g{gamma}"
    logits, tr = helpers.oracle_forward(cfg, params, tasks, imgs, torch.zeros(batch, dtype=torch.int64), gamma,
                                        dtype=torch.float64)
    ref = torch.from_numpy(gold[f"{key}_logits"])
    assert int(gold[f"{key}_nmerge"]) == len(tr.merges)
    for i, st in enumerate(tr.merges):
        assert np.array_equal(st.src.numpy(), gold[f"{key}_l{i}_src"]), f"layer {st.layer} src"
        assert np.array_equal(st.dst.numpy(), gold[f"{key}_l{i}_dst"]), f"layer {st.layer} dst"
        assert np.array_equal(st.unm.numpy(), gold[f"{key}_l{i}_unm"]), f"layer {st.layer} unm"
    torch.testing.assert_close(logits, ref, rtol=1e-10, atol=1e-10 * ref.abs().max().item())


def test_hf_golden_live():
    """When transformers is importable (this image, and the GPU box), regenerate one case live
    from transformers' modules and compare with the oracle: the committed fixture is not stale."""
    pytest.importorskip("transformers")
    from tests.golden.make_hf_golden import hf_model, hf_tokenadapt_forward
    from paper_2401_05031_b200.weights import init_head, synthetic_images

    cfg, params = helpers.backbone("vit_tiny")
    head = init_head(cfg, 10, 0)
    p64 = {k: (v.double() if torch.is_tensor(v) else [{kk: vv.double() for kk, vv in l.items()} for l in v])
           for k, v in params.items()}
    m = hf_model(cfg, p64, {k: v.double() for k, v in head.items()})
    imgs = synthetic_images(3, cfg.img, seed=4)
    hf_logits, hf_trace = hf_tokenadapt_forward(m, cfg, imgs.double(), -5)
    tasks = [{"name": "t0", "head": head, "prompts": {}}]
    logits, tr = helpers.oracle_forward(cfg, params, tasks, imgs, torch.zeros(3, dtype=torch.int64), -5,
                                        dtype=torch.float64)
    for st, (s, d, u) in zip(tr.merges, hf_trace):
        assert torch.equal(st.src, s) and torch.equal(st.dst, d) and torch.equal(st.unm, u)
    torch.testing.assert_close(logits, hf_logits, rtol=1e-10, atol=1e-12)
