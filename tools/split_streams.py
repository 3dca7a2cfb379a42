"""Experiment: one batch of 256 as one forward vs K concurrent sub-batch forwards on K streams
(one CUDA graph each way), to see how much kernel-boundary / tail time concurrency recovers.
Interleaved replays (A B A B ...) so both see the same clocks.  GAMMAS, K env vars."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from tests import helpers
gammas = [int(g) for g in os.environ.get("GAMMAS", "-16,-8,0,16").split(",")]
K = int(os.environ.get("K", "2"))
B = 256
cfg, params = helpers.backbone("vit_b16")
tasks = helpers.task_params(cfg, (100,), [g for g in gammas if g > 0])
bb = helpers.serve_model(cfg, params, tasks, dtype="bf16").backbone
imgs = torch.randn(B, 3, 224, 224, device="cuda")
ids = torch.zeros(B, dtype=torch.int32, device="cuda")
sub = B // K
streams = [torch.cuda.Stream() for _ in range(K)]
base = torch.cuda.Stream()

def ws(b, g):
    import ctypes
    n = ctypes.c_size_t()
    bb._lib.ta_workspace_size(bb._h, b, g, ctypes.byref(n))
    return torch.empty(n.value, dtype=torch.uint8, device="cuda")

graphs = {}
for g in gammas:
    w1 = ws(B, g)
    wk = [ws(sub, g) for _ in range(K)]
    out1 = torch.empty(B, bb.max_classes, device="cuda")
    outk = [torch.empty(sub, bb.max_classes, device="cuda") for _ in range(K)]
    def one():
        bb.forward_raw(imgs, ids, g, logits=out1, workspace=w1)
    def split():
        cur = torch.cuda.current_stream()
        for k, s in enumerate(streams):
            s.wait_stream(cur)
            with torch.cuda.stream(s):
                bb.forward_raw(imgs[k * sub:(k + 1) * sub], ids[k * sub:(k + 1) * sub], g, logits=outk[k], workspace=wk[k])
        for s in streams:
            cur.wait_stream(s)
    with torch.cuda.stream(base):
        one(); split()
    torch.cuda.synchronize()
    ga, gb = torch.cuda.CUDAGraph(), torch.cuda.CUDAGraph()
    with torch.cuda.graph(ga):
        one()
    with torch.cuda.graph(gb):
        split()
    graphs[g] = (ga, gb, out1, outk, w1, wk)
for g in gammas:
    ga, gb, out1, outk = graphs[g][:4]
    ga.replay(); gb.replay(); torch.cuda.synchronize()
    d = (out1 - torch.cat(outk)).abs().max().item()
    ta = tb = 0.0
    for rep in range(10):
        for which in (0, 1):
            gr = ga if which == 0 else gb
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(3):
                gr.replay()
            e1.record(); e1.synchronize()
            if which == 0: ta += e0.elapsed_time(e1) / 3
            else: tb += e0.elapsed_time(e1) / 3
    print(f"TA_PDL={os.environ.get('TA_PDL', '1')} K={K} gamma {g:4d}: one {ta / 10:.3f} ms  split {tb / 10:.3f} ms  "
          f"({(ta - tb) / ta * 100:+.1f}%)  max|dlogit| {d:.2e}", flush=True)
