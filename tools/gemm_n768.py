"""proj / fc2 (N = 768) over the gamma < 0 token schedules: pair 256x256 vs single 128x128 tiles
(TA_GEMM_TINY_M=1000000 forces the single-CTA kernel for N <= 1024)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2401_05031_b200 import _cuda
lib = _cuda.lib(); st = torch.cuda.current_stream().cuda_stream
ts = sorted({197 - 16 * l for l in range(12)} | {197 - 8 * l for l in range(12)}, reverse=True)
for t in ts:
    M = 256 * t
    row = []
    for name, N, K in (("proj", 768, 768), ("fc2", 768, 3072)):
        a = torch.randn(M, K, device="cuda").bfloat16(); w = (torch.randn(N, K, device="cuda") * .02).bfloat16()
        bias = torch.zeros(N, device="cuda"); res = torch.zeros(M, N, device="cuda")
        out = torch.empty(M, N, device="cuda")
        run = lambda: _cuda.check(lib.ta_gemm(a.data_ptr(), w.data_ptr(), bias.data_ptr(), res.data_ptr(), out.data_ptr(), M, N, K, 2, 0, 1, st))
        for _ in range(3): run()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(20): run()
        e1.record(); e1.synchronize()
        row.append(f"{name} {e0.elapsed_time(e1) / 20 * 1e3:7.1f} us")
    print(f"t={t:3d} M={M:6d}  " + "  ".join(row), flush=True)
