"""Timeline of CTA 0 of the P-in-TMEM attention kernel (attention_tp.cu) from a -DTA_TP_TRACE build.

  TA_LIB=var/lib_tptrace.so TA_ATTENTION_BACKEND=tp T=197 python tools/tp_trace.py
Events: producer 1 KV issue, 2 Q issue; MMA 3 S inputs ready, 4 S committed, 5 P block ready,
6 O committed; softmax 10 S full, 11 pass-1 local, 12 max exchanged, 13 P stage free,
14 P block arrived, 15 pass-2 local, 16 sum exchanged, 17 O full, 18 O stored.
"""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2401_05031_b200 import _cuda

lib = _cuda.lib()
B, t, H, hd = 256, int(os.environ.get("T", "197")), 12, 64
qkv = torch.randn(B * t, 3 * H * hd, device="cuda").bfloat16()
size = torch.ones(B, t, device="cuda")
out = torch.empty(B * t, H * hd, device="cuda", dtype=torch.bfloat16)
st = torch.cuda.current_stream().cuda_stream
fn = lib.ta_debug_tp_trace
fn.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int, ctypes.c_int]
for _ in range(3):
    _cuda.check(lib.ta_attention(qkv.data_ptr(), size.data_ptr(), B, t, H, hd, out.data_ptr(), 0, st))
torch.cuda.synchronize()
fn(None, None, 0, 1)
_cuda.check(lib.ta_attention(qkv.data_ptr(), size.data_ptr(), B, t, H, hd, out.data_ptr(), 0, st))
torch.cuda.synchronize()
N = 16384
ts = (ctypes.c_ulonglong * N)()
tg = (ctypes.c_uint * N)()
n = fn(ts, tg, N, 0)
ev = sorted((ts[i], tg[i] >> 8, tg[i] & 255) for i in range(n) if tg[i] & 255)
t0 = ev[0][0]
name = {7: "P0 seen", 23: "P1 seen", 8: "P0 fenced", 24: "P1 fenced", 12: "mma0", 28: "mma1", 4: "S issued", 5: "PV0 issued", 21: "PV1 issued", 6: "O0 commit", 22: "O1 commit", 9: "bias",
        10: "S full", 11: "pass1 done", 14: "P arrive", 17: "O full", 18: "O stored"}
print(f"{n} events, span {(ev[-1][0] - t0)} clk")
lim = int(os.environ.get("LINES", "220"))
for c, w, e in ev[:lim]:
    col = {8: 0, 9: 1}.get(w, 2 + (w // 4))
    print(f"{c - t0:8d}  " + " " * (18 * col) + f"w{w}:{name.get(e, e)}")
# per-event average gaps for softmax warp 0
import collections
seq = [(c, e) for c, w, e in ev if w == 0]
gaps = collections.defaultdict(list)
for (c0, e0), (c1, e1) in zip(seq, seq[1:]):
    gaps[(e0, e1)].append(c1 - c0)
print("warp 0 transitions (avg clk, count):")
for k, v in sorted(gaps.items(), key=lambda kv: -sum(kv[1])):
    print(f"  {name.get(k[0])} -> {name.get(k[1])}: {sum(v) / len(v):8.0f}  x{len(v)}  total {sum(v)}")
