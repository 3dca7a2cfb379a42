"""Parity of the exact path the bench runs, at the bench size, with near-tie accounting
(north_star parity bars; VERDICT r01 "pin parity on the exact path").

* a8+a9, bf16 instance: ``ta_match_qkv`` on bf16 qkv reaches the same
  ``match_fused_kernel<bf16, *, 1, 256>`` (metric = head mean of k, 1xTF32 tcgen05 scores) the
  bf16 forward launches.  Compared with ToMe matching on the fp64 head mean of the same bf16 k:
  decisions must be identical except near-ties, where the kernel's answer must still be valid
  within TAU_TF32 (helpers.decision_slack).  TAU_TF32 = 2^-9: the metric rows are unit vectors
  rounded to TF32 (2^-11 relative per element), so each score is off by at most
  sum_i |a_i b_i| 2^-10 <= 2^-10, and a difference of two scores by at most 2^-9.  Exact ties
  (duplicated rows, injected) are never excluded: they follow the tie rules bit for bit.
* fp32 mode, ViT-B/16 b=256, every gamma of the sweep, free-running: the GPU trace is replayed
  in the fp64 oracle with the oracle's own matching run beside it (shadow); every image-layer
  must be identical except near-ties valid within TAU_F32 = 2^-16 (the fp32 forward differs
  from fp64 by ~1e-6 relative), and logits match the fp64 oracle within rtol 1e-4
  (atol 1e-4 max|logit|).  The fp32 oracle's free-running trace is compared too (reported).
* bf16 mode at b=256, every gamma: logits vs the fp64 oracle forced with the GPU's own trace
  within the bf16 bound of test_gpu_forward.py; the fraction of image-layers whose bf16
  decisions differ from the oracle's own given the same history is reported (free-running bf16
  divergence).
Counts go to $TA_PARITY_LOG (profiles/r02_parity.md is made from it)."""

import ctypes

import pytest
import torch

from paper_2401_05031_b200 import _cuda
from tests import helpers
from tests.test_gpu_forward import BF16_TOL

pytestmark = pytest.mark.gpu

TAU_TF32 = 2.0 ** -9
TAU_F32 = 2.0 ** -16
B = 256
GAMMAS = (-16, -8, 0, 8, 16)


def _fin(x):
    return torch.where(torch.isinf(x), torch.zeros_like(x), x)


# ------------------------------------------------------------------ a8 + a9, bf16 kernel
@pytest.mark.parametrize("t,hd", [(197, 64), (189, 64), (21, 64), (257, 64), (257, 80), (197, 80), (65, 80)])
def test_match_qkv_bf16_vs_oracle(t, hd):
    heads = 12 if hd == 64 else 16
    D = heads * hd
    nimg = 64
    g = torch.Generator().manual_seed(t * 131 + hd)
    qkv = torch.randn(nimg, t, 3 * D, generator=g)
    k = qkv[:, :, D:2 * D]
    # exact ties: duplicate some B rows (dst ties) and A rows (order ties) in half the images
    for b in range(0, nimg, 2):
        k[b, 3] = k[b, 7]          # B rows 1 and 3 identical -> every A row ties between them
        k[b, 4] = k[b, 10]         # A rows 2 and 5 identical -> same node_max, rank tie
    qkv_bf = qkv.to(torch.bfloat16)
    na = (t + 1) // 2
    for r in sorted({min(8, (t - 1) // 2), (t - 1) // 2}):
        src = torch.empty(nimg, r, dtype=torch.int32, device="cuda")
        dst = torch.empty_like(src)
        unm = torch.empty(nimg, na - r, dtype=torch.int32, device="cuda")
        dev = qkv_bf.cuda()
        st = torch.cuda.current_stream().cuda_stream
        _cuda.check(_cuda.lib().ta_match_qkv(dev.data_ptr(), _cuda.DTYPE_BF16, nimg, t, heads, hd, r,
                                             src.data_ptr(), dst.data_ptr(), unm.data_ptr(), st))
        torch.cuda.synchronize()
        s, d, u = src.cpu().long(), dst.cpu().long(), unm.cpu().long()
        metric = qkv_bf[:, :, D:2 * D].double().reshape(nimg, t, heads, hd).mean(2)
        from oracle import vit_oracle

        o_src, o_dst, o_unm, _, _, scores = vit_oracle.bipartite_soft_matching(metric, r, return_scores=True)
        same = (o_src == s).all(1) & (o_dst == d).all(1) & (o_unm == u).all(1)
        worst = 0.0
        for b in torch.nonzero(~same).flatten().tolist():
            ok, slack = helpers.decision_slack(scores[b], s[b], d[b], u[b])
            assert ok, f"image {b}: structurally invalid decisions"
            worst = max(worst, slack)
            assert slack <= TAU_TF32, f"image {b}: differs beyond the TF32 bound ({slack:.3e})"
        # injected exact ties (bit-identical scores in the kernel too) follow the tie rules
        # exactly: B column 3 duplicates column 1, so the lowest-column argmax never picks 3;
        # A row 5 duplicates row 2, so the stable order merges 2 before (or instead of) 5
        for b in range(0, nimg, 2):
            assert not (d[b] == 3).any(), f"image {b}: argmax tie resolved to the higher column"
            pos = {int(v): i for i, v in enumerate(s[b].tolist())}
            if 5 in pos:
                assert 2 in pos and pos[2] < pos[5], f"image {b}: stable-order tie broken"
        helpers.record("match_qkv_bf16", {"t": t, "hd": hd, "r": r, "images": nimg,
                                          "identical": int(same.sum()), "excluded_near_tie": int((~same).sum()),
                                          "max_slack": worst, "tau": TAU_TF32})


# ------------------------------------------------------------------ full-size, fp32 + bf16
_CACHE = {}


def _setup():
    if "cfg" not in _CACHE:
        cfg, params = helpers.backbone("vit_b16")
        tasks = helpers.task_params(cfg, (10, 100), [8, 16])
        imgs = helpers.synthetic_images(B, cfg.img, seed=11)
        ids = torch.arange(B, dtype=torch.int64) % 2
        _CACHE.update(cfg=cfg, params=params, tasks=tasks, imgs=imgs, ids=ids)
    return _CACHE["cfg"], _CACHE["params"], _CACHE["tasks"], _CACHE["imgs"], _CACHE["ids"]


def _gpu(dtype, gamma):
    key = ("gpu", dtype, gamma)
    if key not in _CACHE:
        cfg, params, tasks, imgs, ids = _setup()
        sm = _CACHE.get(("sm", dtype))
        if sm is None:
            sm = _CACHE[("sm", dtype)] = helpers.serve_model(cfg, params, tasks, dtype=dtype)
        bb = sm.backbone
        n_tr = bb.trace_len(B, gamma)
        trace = torch.full((max(n_tr, 1),), -1, dtype=torch.int32, device="cuda")
        out = bb.forward_raw(imgs.cuda(), ids.to(torch.int32).cuda(), gamma, trace=trace if n_tr else None)
        torch.cuda.synchronize()
        tr = helpers.split_trace(trace.cpu(), bb.schedule(gamma), B) if n_tr else []
        _CACHE[key] = (out.cpu(), tr)
    return _CACHE[key]


def _oracle64(gamma, forced):
    key = ("o64", gamma, id(forced) if forced else None)
    if key not in _CACHE:
        cfg, params, tasks, imgs, ids = _setup()
        torch.set_num_threads(max(1, len(__import__("os").sched_getaffinity(0))))
        with torch.inference_mode():
            _CACHE[key] = helpers.oracle_forward(cfg, params, tasks, imgs, ids, gamma, dtype=torch.float64,
                                                 forced=forced or None, shadow=bool(forced))
    return _CACHE[key]


@pytest.mark.parametrize("gamma", GAMMAS)
def test_fullsize_fp32_free_running(gamma):
    out, tr = _gpu("fp32", gamma)
    ref, otr = _oracle64(gamma, tr)
    stats = helpers.compare_traces(otr.merges, tr)
    for s in stats:
        assert s["valid"] and s["max_slack"] <= TAU_F32, s
    rf = _fin(ref.float())
    scale = rf.abs().max().item()
    err = (_fin(out) - rf).abs().max().item()
    torch.testing.assert_close(_fin(out), rf, rtol=1e-4, atol=1e-4 * scale)
    n_il = sum(s["images"] for s in stats)
    n_diff = sum(s["differing"] for s in stats)
    payload = {"gamma": gamma, "batch": B, "image_layers": n_il, "excluded_near_tie": n_diff,
               "max_slack": max([s["max_slack"] for s in stats], default=0.0), "tau": TAU_F32,
               "max_abs_dlogit": err, "max_logit": scale, "rel": err / scale}
    if gamma < 0:  # the fp32 oracle's own free-running trace, image by image
        cfg, params, tasks, imgs, ids = _setup()
        with torch.inference_mode():
            _, tr32 = helpers.oracle_forward(cfg, params, tasks, imgs, ids, gamma)
        same = torch.ones(B, dtype=torch.bool)
        for st, (s_, d_, u_) in zip(tr32.merges, tr):
            same &= (st.src == s_).all(1) & (st.dst == d_).all(1) & (st.unm == u_).all(1)
        payload["images_identical_to_fp32_oracle_free_running"] = int(same.sum())
    helpers.record("fullsize_fp32", payload)


@pytest.mark.parametrize("gamma", GAMMAS)
def test_fullsize_bf16_index_forced_and_divergence(gamma):
    out, tr = _gpu("bf16", gamma)
    ref, otr = _oracle64(gamma, tr)
    rf = _fin(ref.float())
    fr = _fin(out)
    scale = rf.abs().max().item()
    err = (fr - rf).abs().max().item()
    assert err <= BF16_TOL * scale, (err, scale)
    top2 = rf.topk(2, dim=-1).values
    decisive = (top2[:, 0] - top2[:, 1]) > 2 * BF16_TOL * scale
    assert torch.equal(fr.argmax(-1)[decisive], rf.argmax(-1)[decisive])
    stats = helpers.compare_traces(otr.merges, tr)
    for s in stats:
        assert s["valid"], s
    n_il = sum(s["images"] for s in stats)
    n_diff = sum(s["differing"] for s in stats)
    helpers.record("fullsize_bf16", {"gamma": gamma, "batch": B, "max_abs_dlogit": err, "max_logit": scale,
                                     "rel": err / scale, "top1_checked": int(decisive.sum()),
                                     "top1_agree_all": int((fr.argmax(-1) == rf.argmax(-1)).sum()),
                                     "image_layers": n_il, "differing_from_oracle_own": n_diff,
                                     "divergence_fraction": (n_diff / n_il) if n_il else 0.0,
                                     "max_slack": max([s["max_slack"] for s in stats], default=0.0)})
