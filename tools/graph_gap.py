"""Graph-replayed forward time vs the sum of its kernels' durations (one eager forward under
the same conditions, ta_profile_stages): the difference is launch gaps / ramps / tails.
  python tools/graph_gap.py -16 0 16"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2401_05031_b200.synthetic import build_serve_model
gammas = [int(a) for a in sys.argv[1:]] or [-16, 0, 16]
sm = build_serve_model("vit_b16", (100,), [g for g in gammas if g > 0])
bb = sm.backbone
B = 256
imgs = torch.randn(B, 3, 224, 224, device="cuda")
ids = torch.zeros(B, dtype=torch.int32, device="cuda")
for g in gammas:
    s = torch.cuda.Stream(); s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        for _ in range(2): bb.forward_raw(imgs, ids, g)
    torch.cuda.current_stream().wait_stream(s)
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr):
        bb.forward_raw(imgs, ids, g)
    for _ in range(3): gr.replay()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10): gr.replay()
    e1.record(); e1.synchronize()
    graph_us = e0.elapsed_time(e1) / 10 * 1e3
    recs = bb.stage_times(imgs, ids, g)
    eager_us = sum(u for _, _, u in recs)
    print(f"gamma={g}: graph {graph_us:.0f} us, eager stage-event sum {eager_us:.0f} us, launches {len(recs)}, PDL={os.environ.get('TA_PDL', '1')}")
