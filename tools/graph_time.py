"""Graph replay time per gamma (ViT-B/16 b=256, default bf16 model), mean of 20 replays."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from tests import helpers
gammas = [int(g) for g in os.environ.get("GAMMAS", "-16,-8,0,8,16").split(",")]
cfg, params = helpers.backbone("vit_b16")
tasks = helpers.task_params(cfg, (100,), [g for g in gammas if g > 0])
bb = helpers.serve_model(cfg, params, tasks, dtype="bf16").backbone
imgs = torch.randn(256, 3, 224, 224, device="cuda")
ids = torch.zeros(256, dtype=torch.int32, device="cuda")
s = torch.cuda.Stream(); s.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(s):
    for g in gammas:
        bb.forward_raw(imgs, ids, g)
torch.cuda.current_stream().wait_stream(s); torch.cuda.synchronize()
graphs = {}
for g in gammas:
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr):
        bb.forward_raw(imgs, ids, g)
    graphs[g] = gr
for g in gammas:
    for _ in range(3): graphs[g].replay()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20): graphs[g].replay()
    e1.record(); e1.synchronize()
    print(f"TA_PDL={os.environ.get('TA_PDL', '1')} gamma {g:4d}: {e0.elapsed_time(e1) / 20:.3f} ms")
# eager launches of the same forwards for comparison
for g in gammas:
    for _ in range(3): bb.forward_raw(imgs, ids, g)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20): bb.forward_raw(imgs, ids, g)
    e1.record(); e1.synchronize()
    print(f"eager gamma {g:4d}: {e0.elapsed_time(e1) / 20:.3f} ms")
