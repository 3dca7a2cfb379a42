"""Times the fused bipartite match (ta_match: fp32 metric input) and, through a bf16 forward
stage, the qkv-input path.  Usage: python tools/match_bench.py"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2401_05031_b200 import _cuda
lib = _cuda.lib(); st = torch.cuda.current_stream().cuda_stream
for B, t, r, c in [(512, 257, 24, 80), (512, 233, 24, 80), (256, 197, 8, 64)]:
    metric = torch.randn(B, t, c, device="cuda")
    na = (t + 1) // 2
    src = torch.empty(B, r, dtype=torch.int32, device="cuda"); dst = torch.empty_like(src)
    unm = torch.empty(B, na - r, dtype=torch.int32, device="cuda")
    run = lambda: _cuda.check(lib.ta_match(metric.data_ptr(), B, t, c, r, src.data_ptr(), dst.data_ptr(), unm.data_ptr(), st))
    for _ in range(3): run()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10): run()
    e1.record(); e1.synchronize()
    print(B, t, r, c, f"{e0.elapsed_time(e1) / 10 * 1e3:.1f} us")
