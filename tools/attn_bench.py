"""Times ta_attention (bf16) at the ViT token counts; set TA_ATTENTION_BACKEND=mma for the mma.sync kernel."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2401_05031_b200 import _cuda

lib = _cuda.lib()
st = torch.cuda.current_stream().cuda_stream
SHAPES = [tuple(int(v) for v in s.split(",")) for s in os.environ["SHAPES"].split(";")] if os.environ.get("SHAPES") else [(256, 197, 12, 64), (256, 101, 12, 64), (256, 389, 12, 64), (256, 21, 12, 64), (256, 197, 16, 64), (256, 581, 16, 64), (512, 257, 16, 80)]
for B, t, H, hd in SHAPES:
    qkv = torch.randn(B * t, 3 * H * hd, device="cuda").bfloat16()
    size = torch.ones(B, t, device="cuda")
    out = torch.empty(B * t, H * hd, device="cuda", dtype=torch.bfloat16)
    run = lambda: _cuda.check(lib.ta_attention(qkv.data_ptr(), size.data_ptr(), B, t, H, hd, out.data_ptr(), 0, st))
    for _ in range(3): run()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n = 20
    e0.record()
    for _ in range(n): run()
    e1.record(); e1.synchronize()
    ms = e0.elapsed_time(e1) / n
    fl = 4.0 * B * H * t * t * hd
    by = B * t * H * hd * 2 * 4
    print(f"B={B} t={t:4d} H={H} hd={hd}: {ms*1e3:8.1f} us  {fl/ms/1e9:7.1f} TFLOP/s  {by/ms/1e6:7.1f} GB/s")
