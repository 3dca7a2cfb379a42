"""A/B of the LayerNorm fold (LN folded into the QKV / fc1 GEMMs) vs explicit LayerNorm
kernels: both models' CUDA graphs replayed alternately in one process (same clocks / power
state), per gamma, ViT-B/16 b=256.  Prints mean ms per forward for each."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from tests import helpers

gammas = [int(g) for g in os.environ.get("GAMMAS", "-16,-8,0,8,16").split(",")]
cfg, params = helpers.backbone("vit_b16")
tasks = helpers.task_params(cfg, (100,), [g for g in gammas if g > 0])
models = {f: helpers.serve_model(cfg, params, tasks, dtype="bf16", fold_ln=bool(f)).backbone for f in (0, 1)}
B = 256
imgs = torch.randn(B, 3, 224, 224, device="cuda")
ids = torch.zeros(B, dtype=torch.int32, device="cuda")
graphs = {}
s = torch.cuda.Stream(); s.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(s):
    for f, bb in models.items():
        for g in gammas:
            bb.forward_raw(imgs, ids, g)
torch.cuda.current_stream().wait_stream(s)
torch.cuda.synchronize()
for f, bb in models.items():
    for g in gammas:
        gr = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gr):
            bb.forward_raw(imgs, ids, g)
        graphs[(f, g)] = gr
tot = {k: 0.0 for k in graphs}
rounds, reps = 6, 5
for _ in range(rounds):
    for g in gammas:
        for f in (0, 1):
            gr = graphs[(f, g)]
            gr.replay()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(reps):
                gr.replay()
            e1.record(); e1.synchronize()
            tot[(f, g)] += e0.elapsed_time(e1) / reps
for g in gammas:
    a, b = tot[(0, g)] / rounds, tot[(1, g)] / rounds
    print(f"gamma {g:4d}: explicit LN {a:7.3f} ms   folded {b:7.3f} ms   ({100 * (b - a) / a:+.1f}%)")
