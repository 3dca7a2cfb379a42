"""Per-stage warm timings of one eager ta_forward (TA_PROFILE_STAGES=1) vs the CUDA-graph time."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from tests import helpers
g = int(sys.argv[1]) if len(sys.argv) > 1 else 0
fold = bool(int(sys.argv[2])) if len(sys.argv) > 2 else False
MODEL = os.environ.get("MODEL", "vit_b16"); BATCH = int(os.environ.get("BATCH", "256"))
cfg, params = helpers.backbone(MODEL)
tasks = helpers.task_params(cfg, (100,), [g] if g > 0 else [])
sm = helpers.serve_model(cfg, params, tasks, dtype="bf16", fold_ln=fold)
bb = sm.backbone
imgs = torch.randn(BATCH, 3, cfg.img, cfg.img, device="cuda")
ids = torch.zeros(BATCH, dtype=torch.int32, device="cuda")
for _ in range(3): bb.forward_raw(imgs, ids, g)
torch.cuda.synchronize()
os.environ["TA_PROFILE_STAGES"] = "1"
bb.forward_raw(imgs, ids, g)
torch.cuda.synchronize()
del os.environ["TA_PROFILE_STAGES"]
# graph time for comparison
gr = torch.cuda.CUDAGraph()
s = torch.cuda.Stream(); s.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(s):
    bb.forward_raw(imgs, ids, g)
torch.cuda.current_stream().wait_stream(s)
with torch.cuda.graph(gr):
    bb.forward_raw(imgs, ids, g)
for _ in range(3): gr.replay()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10): gr.replay()
e1.record(); e1.synchronize()
print(f"graph: {e0.elapsed_time(e1) / 10 * 1e3:.1f} us per forward (gamma={g})", file=sys.stderr)
