"""Times ta_gemm at the small-M shapes of the gamma < 0 tail layers (ViT-B/16, B=256)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2401_05031_b200 import _cuda
lib = _cuda.lib(); st = torch.cuda.current_stream().cuda_stream
for t in (11, 21, 37, 53, 85):
    M = 256 * t
    for name, N, K, epi in (("qkv", 2304, 768, 0), ("proj", 768, 768, 2), ("fc1", 3072, 768, 1), ("fc2", 768, 3072, 2)):
        a = torch.randn(M, K, device="cuda").bfloat16(); w = (torch.randn(N, K, device="cuda") * .02).bfloat16()
        bias = torch.zeros(N, device="cuda"); res = torch.zeros(M, N, device="cuda")
        out = torch.empty(M, N, device="cuda", dtype=torch.float32 if epi == 2 else torch.bfloat16)
        run = lambda: _cuda.check(lib.ta_gemm(a.data_ptr(), w.data_ptr(), bias.data_ptr(), res.data_ptr() if epi == 2 else None, out.data_ptr(), M, N, K, epi, 0, 1 if epi == 2 else 0, st))
        for _ in range(3): run()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(20): run()
        e1.record(); e1.synchronize()
        ms = e0.elapsed_time(e1) / 20
        print(f"t={t:3d} {name:5s} M={M:6d} N={N:5d} K={K:5d} {ms*1e3:7.1f} us {2*M*N*K/ms/1e9:7.1f} TF/s")
