"""One eager ta_forward per gamma between cudaProfilerStart/Stop, for
`ncu --profile-from-start off --metrics gpu__time_duration.sum` launch lists of the REAL
forward (kernel order = layer order).  python tools/launch_list.py -16 0 16"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from tests import helpers
gammas = [int(a) for a in sys.argv[1:]] or [-16, -8, 0, 8, 16]
MODEL = os.environ.get("MODEL", "vit_b16"); BATCH = int(os.environ.get("BATCH", "256"))
cfg, params = helpers.backbone(MODEL)
tasks = helpers.task_params(cfg, (100,), [g for g in gammas if g > 0])
sm = helpers.serve_model(cfg, params, tasks, dtype=os.environ.get("DTYPE", "bf16"),
                         fold_ln=None if os.environ.get("FOLD_LN") is None else os.environ["FOLD_LN"] == "1")
bb = sm.backbone
imgs = torch.randn(BATCH, 3, cfg.img, cfg.img, device="cuda")
ids = torch.zeros(BATCH, dtype=torch.int32, device="cuda")
for g in gammas:
    for _ in range(2):
        bb.forward_raw(imgs, ids, g)
torch.cuda.synchronize()
for g in gammas:
    torch.cuda.profiler.start()
    bb.forward_raw(imgs, ids, g)
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
