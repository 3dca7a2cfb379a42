"""Subprocess body of tests/test_gpu_forward.py::test_merge_fusion_matches_merge_kernel: the
fused proj + merge path (TA_MERGE_FUSION, read once per process) against the default path on
the same batch with the same forced merge trace."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from tests import helpers  # noqa: E402

cfg, params = helpers.backbone("vit_b16")
tasks = helpers.task_params(cfg, (10, 100), [])
B = 24  # M = B t > 3072: the CTA-pair GEMM, which carries the fused epilogue
imgs = helpers.synthetic_images(B, cfg.img, seed=3).cuda()
ids = (torch.arange(B, dtype=torch.int32) % 2).cuda()
sm = helpers.serve_model(cfg, params, tasks, dtype="bf16")
bb = sm.backbone
for gamma in (-16, -8):
    n = bb.trace_len(B, gamma)
    trace = torch.full((n,), -1, dtype=torch.int32, device="cuda")
    out = bb.forward_raw(imgs, ids, gamma, trace=trace)
    ref_path = os.path.join(sys.argv[1], f"fusion0_g{gamma}.pt")  # the default path's trace, if run
    shared = torch.load(ref_path)["trace"].cuda() if os.path.exists(ref_path) else trace.clone()
    forced = bb.forward_raw(imgs, ids, gamma, forced_trace=shared)
    # own trace replayed: with fusion the free-running row map comes from the match kernel and
    # the forced one from merge_map, so equal logits pin the two maps to each other
    replay = bb.forward_raw(imgs, ids, gamma, forced_trace=trace.clone())
    torch.cuda.synchronize()
    torch.save({"out": out.cpu(), "forced": forced.cpu(), "trace": trace.cpu(), "replay": replay.cpu()},
               os.path.join(sys.argv[1], f"fusion{os.environ.get('TA_MERGE_FUSION', '0')}"
                                         f"{'c' if os.environ.get('TA_FIXUP') == 'chain' else ''}_g{gamma}.pt"))
print("ok")
