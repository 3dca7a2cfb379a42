"""Timeline of CTA 0 of the chunk-pipelined attention kernel (attention_fa.cu) from a
-DTA_ATTN_TRACE build:  TA_LIB=var/lib_trace.so T=197 python tools/fa_trace.py
Events: producer 1 Q, 2 K, 3 V issued; MMA 20+g PV issued, 30+g S issued; softmax 10 S wait,
11 S full, 12 P-stage wait, 13 P stage free, 14 P arrived, 15 epilogue O wait, 16 O full,
17 epilogue done."""
import collections, ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2401_05031_b200 import _cuda

lib = _cuda.lib()
B, t, H, hd = 256, int(os.environ.get("T", "197")), 12, 64
qkv = torch.randn(B * t, 3 * H * hd, device="cuda").bfloat16()
size = torch.ones(B, t, device="cuda")
out = torch.empty(B * t, H * hd, device="cuda", dtype=torch.bfloat16)
st = torch.cuda.current_stream().cuda_stream
fn = lib.ta_debug_fa_trace
fn.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int, ctypes.c_int]
run = lambda: _cuda.check(lib.ta_attention(qkv.data_ptr(), size.data_ptr(), B, t, H, hd, out.data_ptr(), 0, st))
for _ in range(3):
    run()
torch.cuda.synchronize()
fn(None, None, 0, 1)
run()
torch.cuda.synchronize()
N = 16384
ts = (ctypes.c_ulonglong * N)()
tg = (ctypes.c_uint * N)()
n = fn(ts, tg, N, 0)
ev = sorted((ts[i], tg[i] >> 8, tg[i] & 255) for i in range(n) if tg[i] & 255)
t0 = ev[0][0]
name = {1: "Q", 2: "K", 3: "V", 20: "PV0", 21: "PV1", 30: "S0", 31: "S1", 10: "s-wait", 11: "S full",
        12: "p-wait", 13: "P free", 14: "P arr", 15: "o-wait", 16: "O full", 17: "epi done"}
print(f"{n} events, span {(ev[-1][0] - t0)} clk")
lim = int(os.environ.get("LINES", "300"))
for c, w, e in ev[:lim]:
    col = {8: 0, 9: 1, 10: 2}.get(w, 3 + (w // 4))
    print(f"{c - t0:8d}  " + " " * (12 * col) + f"w{w}:{name.get(e, e)}")
for wsel in range(8):
    seq = [(c, e) for c, w, e in ev if w == wsel]
    d = [c1 - c0 for (c0, e0), (c1, e1) in zip(seq, seq[1:]) if (e0, e1) == (13, 14)]
    m = [c1 - c0 for (c0, e0), (c1, e1) in zip(seq, seq[1:]) if (e0, e1) == (11, 12)]
    print(f"warp {wsel}: P free->P arr avg {sum(d) / max(1, len(d)):.0f} (n={len(d)}), S full->p-wait avg {sum(m) / max(1, len(m)):.0f}")
mma = [c for c, w, e in ev if w == 10]
print(f"MMA warp events: {len(mma)}")
for wsel in (0, 4):
    seq = [(c, e) for c, w, e in ev if w == wsel]
    gaps = collections.defaultdict(list)
    for (c0, e0), (c1, e1) in zip(seq, seq[1:]):
        gaps[(e0, e1)].append(c1 - c0)
    print(f"warp {wsel} transitions (avg clk, count, total):")
    for k, v in sorted(gaps.items(), key=lambda kv: -sum(kv[1])):
        print(f"  {name.get(k[0])} -> {name.get(k[1])}: {sum(v) / len(v):8.0f}  x{len(v)}  total {sum(v)}")
