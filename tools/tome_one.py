"""One token-merge layer's bandwidth kernels at the ViT-B/16 b=256 gamma=-8 layer-0 shape
(metric split + tcgen05 match, merge + LN2, LayerNorm) for ncu captures."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2401_05031_b200 import _cuda  # noqa: E402

lib = _cuda.lib()
st = torch.cuda.current_stream().cuda_stream
B, t, D, r, H = 256, 197, 768, 8, 12
x = torch.randn(B, t, D, device="cuda")
size = torch.ones(B, t, device="cuda")
metric = torch.randn(B, t, 64, device="cuda")
na = (t + 1) // 2
src = torch.empty(B, r, dtype=torch.int32, device="cuda")
dst = torch.empty(B, r, dtype=torch.int32, device="cuda")
unm = torch.empty(B, na - r, dtype=torch.int32, device="cuda")
lw, lb = torch.ones(D, device="cuda"), torch.zeros(D, device="cuda")
xo = torch.empty(B, t - r, D, device="cuda")
so = torch.empty(B, t - r, device="cuda")
ho = torch.empty(B, t - r, D, device="cuda", dtype=torch.bfloat16)
hl = torch.empty(B * t, D, device="cuda", dtype=torch.bfloat16)
for _ in range(3):
    _cuda.check(lib.ta_match(metric.data_ptr(), B, t, 64, r, src.data_ptr(), dst.data_ptr(), unm.data_ptr(), st))
    _cuda.check(lib.ta_merge(x.data_ptr(), size.data_ptr(), B, t, D, r, src.data_ptr(), dst.data_ptr(),
                             unm.data_ptr(), lw.data_ptr(), lb.data_ptr(), xo.data_ptr(), so.data_ptr(),
                             ho.data_ptr(), 0, st))
    _cuda.check(lib.ta_layernorm(x.data_ptr(), lw.data_ptr(), lb.data_ptr(), hl.data_ptr(), B * t, D, 0, st))
torch.cuda.synchronize()
