"""fp32 parity-mode forward time, ViT-B/16 b=256 per gamma (TA_F32_GEMM=simt for the SIMT GEMMs)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2401_05031_b200.config import VIT_CONFIGS, flops_per_image
from paper_2401_05031_b200.synthetic import build_serve_model
cfg = VIT_CONFIGS["vit_b16"]
gammas = [int(g) for g in os.environ.get("GAMMAS", "-16,-8,0,8,16").split(",")]
sm = build_serve_model("vit_b16", (100,), [g for g in gammas if g > 0], dtype="fp32")
bb = sm.backbone
B = 256
imgs = torch.randn(B, 3, 224, 224, device="cuda")
ids = torch.zeros(B, dtype=torch.int32, device="cuda")
for g in gammas:
    for _ in range(2):
        bb.forward_raw(imgs, ids, g)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3):
        bb.forward_raw(imgs, ids, g)
    e1.record(); e1.synchronize()
    ms = e0.elapsed_time(e1) / 3
    print(f"fp32 mode ({os.environ.get('TA_F32_GEMM', 'tc')}) gamma={g}: {ms:.2f} ms/batch, {B / ms * 1e3:.0f} img/s, "
          f"{flops_per_image(cfg, g) * B / ms / 1e9:.0f} TFLOP/s")
