"""Subprocess body of tests/test_gpu_attention_backends.py: the attention backend is chosen
once per process from TA_ATTENTION_BACKEND, so each backend is checked in its own process.
Prints one line per shape and exits non-zero on the first mismatch."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2401_05031_b200 import _cuda  # noqa: E402


def ref(qkv, size, b, t, heads, hd):
    x = qkv.double().reshape(b, t, 3, heads, hd).permute(2, 0, 3, 1, 4)
    s = (x[0] @ x[1].transpose(-2, -1)) * hd ** -0.5
    if size is not None:
        s = s + size.double().log()[:, None, None, :]
    return (s.softmax(-1) @ x[2]).transpose(1, 2).reshape(b, t, heads * hd)


def main():
    lib = _cuda.lib()
    st = torch.cuda.current_stream().cuda_stream
    shapes = [(7, 1, 64), (5, 33, 64), (6, 64, 64), (4, 65, 64), (3, 197, 64), (2, 261, 64), (2, 300, 64), (2, 389, 64), (2, 449, 64), (2, 513, 64),
              (2, 581, 64), (5, 65, 80), (4, 185, 80), (3, 233, 80), (3, 257, 80), (2, 300, 80),
              # the P-in-TMEM kernel's envelope (64 < t <= 256, hd 64) with several items per CTA:
              # O at columns 192 (t <= 192) / 128 (gated first PV), one or two query tiles
              (32, 197, 64), (32, 129, 64), (24, 101, 64), (16, 256, 64), (20, 192, 64), (20, 193, 64),
              (28, 176, 64), (26, 128, 64), (30, 213, 64), (13, 245, 64)]
    for b, t, hd in shapes:
        for with_size in (False, True):
            heads = 12 if hd == 64 else 16
            g = torch.Generator(device="cuda").manual_seed(t * 31 + b)
            qkv = (torch.randn(b, t, 3 * heads * hd, device="cuda", generator=g) * 1.5).bfloat16()
            size = torch.randint(1, 7, (b, t), device="cuda", generator=g).float() if with_size else None
            out = torch.empty(b, t, heads * hd, device="cuda", dtype=torch.bfloat16)
            _cuda.check(lib.ta_attention(qkv.data_ptr(), size.data_ptr() if size is not None else None,
                                         b, t, heads, hd, out.data_ptr(), 0, st))
            torch.cuda.synchronize()
            r = ref(qkv.float(), size, b, t, heads, hd)
            # bf16 output: |err| <= 2e-2 + 2e-2 |ref| (torch.testing.assert_close form)
            excess = ((out.double() - r).abs() - (2e-2 + 2e-2 * r.abs())).max().item()
            err = (out.double() - r).abs().max().item()
            print(f"{os.environ.get('TA_ATTENTION_BACKEND', 'default')} b={b} t={t} hd={hd} size={with_size} "
                  f"max|err|={err:.3e} excess={excess:.3e}")
            if not excess <= 0:
                sys.exit(1)


if __name__ == "__main__":
    main()
