"""Small-shape driver for compute-sanitizer (memcheck / racecheck / synccheck): launches every
hand-written kernel once -- tcgen05 GEMM pair and single-CTA (ta_gemm, incl. an M that fills no
tile), attention (backend from TA_ATTENTION_BACKEND), bipartite match bf16 + fp32
(ta_match_qkv), merge, LayerNorm, and a ViT-tiny forward in bf16 (LN folded) and fp32 at
gamma -4 / 0 / +4 (patchify, insert_rows, epilogue kinds, head).
  compute-sanitizer --tool memcheck python tools/sanitize_kernels.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2401_05031_b200 import _cuda  # noqa: E402
from tests import helpers  # noqa: E402

lib = _cuda.lib()
st = torch.cuda.current_stream().cuda_stream
dev = "cuda"
chk = _cuda.check

# GEMMs: single-CTA kernel (M <= 3072 and N <= 1024) and the CTA-pair kernel (M = 4000 and
# N = 2048; the residual kind reads its residual boxes by TMA), epilogues 0 / 1 / 2
# (1280 x 1536 x 3072: 30 tiles in 2 split-K parts; 6912 x 768 x 3072: 81 tiles, the last 7 in 4 parts)
for M, N, K in ((300, 512, 128), (97, 256, 192), (1000, 768, 256), (4000, 768, 256), (3300, 2048, 128),
                (1280, 1536, 3072), (6912, 768, 3072)):
    a = torch.randn(M, K, device=dev).bfloat16()
    w = (torch.randn(N, K, device=dev) * 0.05).bfloat16()
    bias = torch.randn(N, device=dev)
    resid = torch.randn(M, N, device=dev)
    for epi in (0, 1):
        out = torch.empty(M, N, device=dev, dtype=torch.bfloat16)
        chk(lib.ta_gemm(a.data_ptr(), w.data_ptr(), bias.data_ptr(), None, out.data_ptr(), M, N, K, epi, 0, 0, st))
    out = torch.empty(M, N, device=dev)
    chk(lib.ta_gemm(a.data_ptr(), w.data_ptr(), bias.data_ptr(), resid.data_ptr(), out.data_ptr(), M, N, K, 2, 0, 1, st))
# attention at a few token counts, with and without the size vector
# (64 x 117: one-tile items on the four-slot K/V ring, > 4 items per CTA so the ring wraps)
for b, t, H, hd in ((2, 53, 12, 64), (2, 197, 12, 64), (64, 117, 12, 64), (1, 300, 12, 64), (1, 257, 16, 80)):
    qkv = torch.randn(b * t, 3 * H * hd, device=dev).bfloat16()
    size = torch.randint(1, 4, (b, t), device=dev).float()
    out = torch.empty(b * t, H * hd, device=dev, dtype=torch.bfloat16)
    for sz in (None, size):
        chk(lib.ta_attention(qkv.data_ptr(), sz.data_ptr() if sz is not None else None, b, t, H, hd,
                             out.data_ptr(), 0, st))
# bipartite matching (bf16 and fp32 instances) and merge
for dt, tt in ((_cuda.DTYPE_BF16, torch.bfloat16), (_cuda.DTYPE_F32, torch.float32)):
    for t, H, hd, r in ((197, 12, 64, 8), (21, 12, 64, 10), (257, 16, 80, 24)):
        B = 3
        qkv = torch.randn(B, t, 3 * H * hd, device=dev).to(tt)
        na = (t + 1) // 2
        src = torch.empty(B, r, dtype=torch.int32, device=dev)
        dst = torch.empty_like(src)
        unm = torch.empty(B, na - r, dtype=torch.int32, device=dev)
        chk(lib.ta_match_qkv(qkv.data_ptr(), dt, B, t, H, hd, r, src.data_ptr(), dst.data_ptr(), unm.data_ptr(), st))
        D = H * hd
        x = torch.randn(B, t, D, device=dev)
        xo = torch.empty(B, t - r, D, device=dev)
        so = torch.empty(B, t - r, device=dev)
        ho = torch.empty(B, t - r, D, device=dev, dtype=torch.bfloat16)
        lw, lb = torch.ones(D, device=dev), torch.zeros(D, device=dev)
        chk(lib.ta_merge(x.data_ptr(), None, B, t, D, r, src.data_ptr(), dst.data_ptr(), unm.data_ptr(),
                         lw.data_ptr(), lb.data_ptr(), xo.data_ptr(), so.data_ptr(), ho.data_ptr(), 0, st))
# LayerNorm
x = torch.randn(37, 768, device=dev)
o = torch.empty(37, 768, device=dev, dtype=torch.bfloat16)
chk(lib.ta_layernorm(x.data_ptr(), torch.ones(768, device=dev).data_ptr(), torch.zeros(768, device=dev).data_ptr(),
                     o.data_ptr(), 37, 768, 0, st))
# whole forward, both modes, merge / vanilla / prompts
cfg, params = helpers.backbone("vit_tiny")
tasks = helpers.task_params(cfg, (10, 100), [4])
imgs = helpers.synthetic_images(3, cfg.img, seed=1).cuda()
for dtype in ("bf16", "fp32"):
    sm = helpers.serve_model(cfg, params, tasks, dtype=dtype)
    for g in (-4, 0, 4):
        sm.forward(imgs, [0, 1, 0], gamma=g)
    torch.cuda.synchronize()
    sm.backbone.close()
# ViT-B/16 at M = B t > 3072: the CTA-pair GEMMs in the forward, incl. the fused proj + merge
# (tile::scatter4 stores, merge_fixup) and the row-remapped prompt epilogues
cfg, params = helpers.backbone("vit_b16")
tasks = helpers.task_params(cfg, (10,), [4])
imgs = helpers.synthetic_images(17, cfg.img, seed=2).cuda()
sm = helpers.serve_model(cfg, params, tasks, dtype="bf16")
for g in (-8, 0, 4):
    sm.forward(imgs, [0] * 17, gamma=g)
torch.cuda.synchronize()
sm.backbone.close()
torch.cuda.synchronize()
print("sanitize_kernels: all launches done")
