"""Times the bf16 tcgen05 GEMM (through ta_gemm) at the ViT-B/16 layer shapes."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2401_05031_b200 import _cuda

lib = _cuda.lib()
B = int(sys.argv[1]) if len(sys.argv) > 1 else 256
t = 197
D = 768
shapes = [("qkv", B * t, 3 * D, D, 0), ("proj", B * t, D, D, 2), ("fc1", B * t, 4 * D, D, 1),
          ("fc2", B * t, D, 4 * D, 2), ("patch", B * 196, D, 768, 0)]
st = torch.cuda.current_stream().cuda_stream
only = os.environ.get("ONLY")
for name, M, N, K, epi in shapes:
    if only and name != only:
        continue
    a = torch.randn(M, K, device="cuda").bfloat16()
    w = (torch.randn(N, K, device="cuda") * 0.02).bfloat16()
    bias = torch.zeros(N, device="cuda")
    res = torch.zeros(M, N, device="cuda")
    out = torch.empty(M, N, device="cuda", dtype=torch.float32 if epi == 2 else torch.bfloat16)
    od = 1 if epi == 2 else 0
    def run():
        _cuda.check(lib.ta_gemm(a.data_ptr(), w.data_ptr(), bias.data_ptr(), res.data_ptr() if epi == 2 else None,
                                out.data_ptr(), M, N, K, epi, 0, od, st))
    for _ in range(5):
        run()
    n = 30
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        run()
    e1.record(); e1.synchronize()
    ms = e0.elapsed_time(e1) / n
    tf = 2 * M * N * K / ms / 1e9
    gb = (M * K * 2 + N * K * 2 + M * N * (8 if epi == 2 else 2)) / ms / 1e6
    print(f"{name:6s} M={M:6d} N={N:5d} K={K:5d} {ms*1e3:8.1f} us  {tf:7.1f} TFLOP/s  {gb:7.1f} GB/s")
