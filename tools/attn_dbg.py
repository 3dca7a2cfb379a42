import sys, os
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import torch
from paper_2401_05031_b200 import _cuda
from test_gpu_kernels import _attn_ref
L = _cuda.lib()
for (b, t, with_size) in [(3, 197, True), (3, 197, False), (64, 197, True), (3, 389, True), (3, 150, True)]:
    heads, hd = 12, 64
    g = torch.Generator(device="cuda").manual_seed(t * 7 + hd)
    qkv = torch.randn(b, t, 3 * heads * hd, device="cuda", generator=g)
    size = torch.randint(1, 6, (b, t), device="cuda", generator=g).float() if with_size else None
    q = qkv.bfloat16()
    out = torch.full((b, t, heads * hd), float("nan"), device="cuda", dtype=torch.bfloat16)
    _cuda.check(L.ta_attention(q.data_ptr(), size.data_ptr() if size is not None else None, b, t, heads, hd, out.data_ptr(), 0, torch.cuda.current_stream().cuda_stream))
    torch.cuda.synchronize()
    ref = _attn_ref(q.float(), size, b, t, heads, hd)
    err = (out.double() - ref).abs()
    bad = (err > 2e-2 + 2e-2 * ref.abs()) | torch.isnan(err)
    print(b, t, with_size, "bad", int(bad.sum()), "of", bad.numel())
    if bad.any():
        idx = bad.nonzero()
        rows = idx[:, 1].unique(); cols = idx[:, 2].unique()
        print("  rows", rows[:20].tolist(), "...", len(rows), " cols", cols[:40].tolist(), len(cols))
        print("  images", idx[:, 0].unique().tolist())
