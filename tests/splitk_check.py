"""Subprocess body of tests/test_gpu_forward.py::test_splitk_forward: the forward with split-K
tail tiles in its GEMMs (TA_GEMM_SPLITK_FWD, read once per process) against the default on the
same batch and forced merge trace.  B = 64: fc2's 150 tiles at t = 197 leave a 2-tile last wave
(4 parts each), and the merged layers' tails split too."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from tests import helpers  # noqa: E402

cfg, params = helpers.backbone("vit_b16")
tasks = helpers.task_params(cfg, (10, 100), [8])
B = 64
imgs = helpers.synthetic_images(B, cfg.img, seed=5).cuda()
ids = (torch.arange(B, dtype=torch.int32) % 2).cuda()
sm = helpers.serve_model(cfg, params, tasks, dtype="bf16")
bb = sm.backbone
tag = os.environ.get("TA_GEMM_SPLITK_FWD", "0")
for gamma in (-16, 0, 8):
    n = bb.trace_len(B, gamma)
    ref_path = os.path.join(sys.argv[1], f"sk0_g{gamma}.pt")  # the default path's trace, if run
    if n:
        trace = torch.full((n,), -1, dtype=torch.int32, device="cuda")
        out = bb.forward_raw(imgs, ids, gamma, trace=trace)
        shared = torch.load(ref_path)["trace"].cuda() if os.path.exists(ref_path) else trace.clone()
        forced = bb.forward_raw(imgs, ids, gamma, forced_trace=shared)
        again = bb.forward_raw(imgs, ids, gamma, forced_trace=shared)
    else:
        trace = torch.zeros(0, dtype=torch.int32)
        out = forced = bb.forward_raw(imgs, ids, gamma)
        again = bb.forward_raw(imgs, ids, gamma)
    torch.cuda.synchronize()
    torch.save({"out": out.cpu(), "forced": forced.cpu(), "again": again.cpu(), "trace": trace.cpu()},
               os.path.join(sys.argv[1], f"sk{tag}_g{gamma}.pt"))
print("ok")
