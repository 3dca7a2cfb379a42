import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2401_05031_b200 import _cuda
lib = _cuda.lib(); st = torch.cuda.current_stream().cuda_stream
B, t, H, hd = 256, int(os.environ.get("T", "197")), 12, 64
qkv = torch.randn(B * t, 3 * H * hd, device="cuda").bfloat16()
size = torch.ones(B, t, device="cuda")
out = torch.empty(B * t, H * hd, device="cuda", dtype=torch.bfloat16)
for _ in range(3):
    _cuda.check(lib.ta_attention(qkv.data_ptr(), size.data_ptr(), B, t, H, hd, out.data_ptr(), 0, st))
torch.cuda.synchronize()
