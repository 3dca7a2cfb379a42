"""Phase timeline of the fused match kernel from a -DTA_MATCH_TRACE build (last match launch of
one bf16 ViT-B/16 forward).  TA_LIB=var/lib_mtrace.so GAMMA=-8 python tools/match_trace.py
Phases: 0 start, 1 after grid_dep_wait, 2 tiles written (metric/normalise/split), 3 S max /
argmax done, 4 ranks and outputs written."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from tests import helpers
from paper_2401_05031_b200 import _cuda

g = int(os.environ.get("GAMMA", "-8"))
B = int(os.environ.get("BATCH", "256"))
cfg, params = helpers.backbone(os.environ.get("MODEL", "vit_b16"))
sm = helpers.serve_model(cfg, params, helpers.task_params(cfg, (100,), []), dtype="bf16")
imgs = torch.randn(B, 3, cfg.img, cfg.img, device="cuda")
ids = torch.zeros(B, dtype=torch.int32, device="cuda")
for _ in range(2):
    sm.backbone.forward_raw(imgs, ids, g)
torch.cuda.synchronize()
lib = _cuda.lib()
fn = lib.ta_debug_match_trace
fn.argtypes = [ctypes.c_void_p, ctypes.c_int]
buf = (ctypes.c_ulonglong * (B * 6))()
fn(buf, B)
tr = torch.tensor(list(buf), dtype=torch.float64).reshape(B, 6)[:, :5]
t0 = tr[:, 0].min()
tr = (tr - t0) / 1e3  # us
d = tr[:, 1:] - tr[:, :-1]
print(f"launch span {tr[:, 4].max():.1f} us; CTA start times: first {tr[:, 0].min():.1f}, last {tr[:, 0].max():.1f}")
for k, name in enumerate(["dep wait", "phase 1 (metric, tiles)", "phase 2+3a (MMA, max)", "phase 3b (rank, out)"]):
    print(f"  {name:26s} mean {d[:, k].mean():6.2f} us  max {d[:, k].max():6.2f}")
print(f"  CTA total mean {(tr[:, 4] - tr[:, 0]).mean():.2f} us")
