"""Per-stage parity of the CUDA kernels through the C ABI.

Each kernel is compared against a plain PyTorch fp32/fp64 statement of the same op, or
against the oracle's ToMe functions (integer outputs bit-exact)."""

import math

import pytest
import torch
import torch.nn.functional as F

from oracle import vit_oracle

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def L():
    from paper_2401_05031_b200 import _cuda

    return _cuda.lib()


def _s():
    return torch.cuda.current_stream().cuda_stream


def _chk(rc):
    from paper_2401_05031_b200 import _cuda

    _cuda.check(rc)


@pytest.mark.parametrize("m,n,k", [(1, 768, 768), (127, 384, 768), (300, 2304, 768),
                                   (1000, 768, 3072), (50432 // 8, 3072, 768),
                                   # split-K tails (gemm.cu splitk_parts): 240 tiles -> 18 x 4 parts,
                                   # 159 -> 11 x 4, ragged M 237 -> 15 x 4, 30 tiles -> 2 parts
                                   (20480, 768, 3072), (13568, 768, 3072), (20000, 768, 2048),
                                   (1280, 1536, 3072)])
@pytest.mark.parametrize("epi", [0, 1, 2])
def test_gemm_bf16_tcgen05(L, m, n, k, epi):
    g = torch.Generator(device="cuda").manual_seed(m + n + k + epi)
    a = torch.randn(m, k, device="cuda", generator=g).bfloat16()
    w = (torch.randn(n, k, device="cuda", generator=g) * 0.05).bfloat16()
    bias = torch.randn(n, device="cuda", generator=g)
    resid = torch.randn(m, n, device="cuda", generator=g)
    ref = a.float() @ w.float().t() + bias
    if epi == 1:
        ref = F.gelu(ref)
    if epi == 2:
        ref = ref + resid
        out = resid.clone()
        _chk(L.ta_gemm(a.data_ptr(), w.data_ptr(), bias.data_ptr(), out.data_ptr(), out.data_ptr(),
                       m, n, k, epi, 0, 1, _s()))
        torch.cuda.synchronize()
        torch.testing.assert_close(out, ref, rtol=1e-4, atol=2e-4)
    else:
        out = torch.empty(m, n, device="cuda", dtype=torch.bfloat16)
        _chk(L.ta_gemm(a.data_ptr(), w.data_ptr(), bias.data_ptr(), None, out.data_ptr(),
                       m, n, k, epi, 0, 0, _s()))
        torch.cuda.synchronize()
        torch.testing.assert_close(out.float(), ref, rtol=1.6e-2, atol=1e-2)


@pytest.mark.parametrize("m,n,k", [(5, 256, 768), (300, 768, 768), (129, 1024, 256)])
@pytest.mark.parametrize("epi", [0, 1, 2])
def test_gemm_f32_simt(L, m, n, k, epi):
    g = torch.Generator(device="cuda").manual_seed(7 + m)
    a = torch.randn(m, k, device="cuda", generator=g)
    w = torch.randn(n, k, device="cuda", generator=g) * 0.05
    bias = torch.randn(n, device="cuda", generator=g)
    resid = torch.randn(m, n, device="cuda", generator=g)
    ref = a.double() @ w.double().t() + bias.double()
    if epi == 1:
        ref = F.gelu(ref)
    out = resid.clone() if epi == 2 else torch.empty(m, n, device="cuda")
    if epi == 2:
        ref = ref + resid.double()
    _chk(L.ta_gemm(a.data_ptr(), w.data_ptr(), bias.data_ptr(), resid.data_ptr() if epi == 2 else None,
                   out.data_ptr(), m, n, k, epi, 1, 1, _s()))
    torch.cuda.synchronize()
    torch.testing.assert_close(out.double(), ref, rtol=1e-5, atol=1e-5)


@pytest.mark.parametrize("rows,dim", [(1, 768), (1000, 768), (77, 1024), (33, 1280), (5, 256)])
@pytest.mark.parametrize("out_dtype", [0, 1])
def test_layernorm(L, rows, dim, out_dtype):
    x = torch.randn(rows, dim, device="cuda") * 3 + 1
    w = torch.randn(dim, device="cuda")
    b = torch.randn(dim, device="cuda")
    out = torch.empty(rows, dim, device="cuda", dtype=torch.bfloat16 if out_dtype == 0 else torch.float32)
    _chk(L.ta_layernorm(x.data_ptr(), w.data_ptr(), b.data_ptr(), out.data_ptr(), rows, dim, out_dtype, _s()))
    torch.cuda.synchronize()
    ref = F.layer_norm(x.double(), (dim,), w.double(), b.double(), eps=1e-6)
    if out_dtype == 0:
        torch.testing.assert_close(out.double(), ref, rtol=1e-2, atol=2e-2)
    else:
        torch.testing.assert_close(out.double(), ref, rtol=1e-5, atol=1e-5)


def _attn_ref(qkv, size, b, t, heads, hd):
    x = qkv.double().reshape(b, t, 3, heads, hd).permute(2, 0, 3, 1, 4)
    q, k, v = x[0], x[1], x[2]
    s = (q @ k.transpose(-2, -1)) * hd ** -0.5
    if size is not None:
        s = s + size.double().log()[:, None, None, :]
    return (s.softmax(-1) @ v).transpose(1, 2).reshape(b, t, heads * hd)


@pytest.mark.parametrize("t", [1, 17, 64, 101, 128, 129, 197, 256, 257, 300, 384, 389, 512, 581])
@pytest.mark.parametrize("hd,heads", [(64, 12), (80, 16)])
@pytest.mark.parametrize("with_size", [False, True])
@pytest.mark.parametrize("dtype", [0, 1])
def test_attention(L, t, hd, heads, with_size, dtype):
    b = 3
    g = torch.Generator(device="cuda").manual_seed(t * 7 + hd)
    qkv = torch.randn(b, t, 3 * heads * hd, device="cuda", generator=g)
    size = (torch.randint(1, 6, (b, t), device="cuda", generator=g).float() if with_size else None)
    tdt = torch.bfloat16 if dtype == 0 else torch.float32
    qkv_d = qkv.to(tdt)
    out = torch.empty(b, t, heads * hd, device="cuda", dtype=tdt)
    _chk(L.ta_attention(qkv_d.data_ptr(), size.data_ptr() if size is not None else None, b, t, heads, hd,
                        out.data_ptr(), dtype, _s()))
    torch.cuda.synchronize()
    ref = _attn_ref(qkv_d.float(), size, b, t, heads, hd)
    if dtype == 0:
        torch.testing.assert_close(out.double(), ref, rtol=2e-2, atol=2e-2)
    else:
        torch.testing.assert_close(out.double(), ref, rtol=1e-5, atol=1e-5)


@pytest.mark.parametrize("t", [5, 21, 101, 133, 197, 213, 261, 341, 389])
@pytest.mark.parametrize("with_size", [False, True])
@pytest.mark.parametrize("ramp", [False, True])
def test_attention_batched_tails(L, t, with_size, ramp):
    """bf16 tcgen05 path with many images: padded keys of a tile are the next image's rows
    (or TMA zero fill), idle row warps and the trimmed last key block must not leak.  ramp:
    key norms grow with the key index, so later key chunks raise the row max far above the
    first chunk's (the lazy-rescale path of attention_fa.cu)."""
    b, heads, hd = 24, 12, 64
    g = torch.Generator(device="cuda").manual_seed(1000 + t)
    qkv = torch.randn(b, t, 3 * heads * hd, device="cuda", generator=g) * 2
    if ramp:
        D = heads * hd
        qkv[:, :, D:2 * D] *= torch.linspace(0.1, 3.0, t, device="cuda")[None, :, None]
    qkv = qkv.bfloat16()
    size = (torch.randint(1, 9, (b, t), device="cuda", generator=g).float() if with_size else None)
    out = torch.empty(b, t, heads * hd, device="cuda", dtype=torch.bfloat16)
    _chk(L.ta_attention(qkv.data_ptr(), size.data_ptr() if size is not None else None, b, t, heads, hd,
                        out.data_ptr(), 0, _s()))
    torch.cuda.synchronize()
    ref = _attn_ref(qkv.float(), size, b, t, heads, hd)
    assert torch.isfinite(out.float()).all()
    torch.testing.assert_close(out.double(), ref, rtol=2e-2, atol=2e-2)


@pytest.mark.parametrize("t", [69, 117, 128])
@pytest.mark.parametrize("with_size", [False, True])
def test_attention_kv_ring_wraps(L, t, with_size):
    """One-tile items (t <= 128) on the four-slot K/V ring with > 4 items per CTA (B = 80, H = 12:
    960 items over at most 148 CTAs), so every slot is reused several times."""
    b, heads, hd = 80, 12, 64
    g = torch.Generator(device="cuda").manual_seed(2000 + t)
    qkv = (torch.randn(b, t, 3 * heads * hd, device="cuda", generator=g) * 2).bfloat16()
    size = (torch.randint(1, 9, (b, t), device="cuda", generator=g).float() if with_size else None)
    out = torch.empty(b, t, heads * hd, device="cuda", dtype=torch.bfloat16)
    _chk(L.ta_attention(qkv.data_ptr(), size.data_ptr() if size is not None else None, b, t, heads, hd,
                        out.data_ptr(), 0, _s()))
    torch.cuda.synchronize()
    ref = _attn_ref(qkv.float(), size, b, t, heads, hd)
    torch.testing.assert_close(out.double(), ref, rtol=2e-2, atol=2e-2)


@pytest.mark.parametrize("t,r", [(197, 8), (197, 16), (189, 8), (21, 10), (3, 1), (257, 24), (4, 1)])
@pytest.mark.parametrize("c", [64, 80])
def test_match_bit_exact(L, t, r, c):
    b = 16
    g = torch.Generator().manual_seed(t * 31 + r + c)
    metric = torch.randn(b, t, c, generator=g)
    # inject exact ties: duplicated B rows (argmax ties) and duplicated A rows (rank ties)
    metric[:, 5 % t] = metric[:, 3 % t]
    if t > 9:
        metric[:, 8] = metric[:, 2]
    src, dst, unm, _, _ = vit_oracle.bipartite_soft_matching(metric.clone(), r)
    m = metric.cuda()
    na = (t + 1) // 2
    s_g = torch.empty(b, r, dtype=torch.int32, device="cuda")
    d_g = torch.empty(b, r, dtype=torch.int32, device="cuda")
    u_g = torch.empty(b, na - r, dtype=torch.int32, device="cuda")
    _chk(L.ta_match(m.data_ptr(), b, t, c, r, s_g.data_ptr(), d_g.data_ptr(), u_g.data_ptr(), _s()))
    torch.cuda.synchronize()
    assert torch.equal(s_g.cpu().long(), src)
    assert torch.equal(d_g.cpu().long(), dst)
    assert torch.equal(u_g.cpu().long(), unm)


@pytest.mark.parametrize("t,r,dim", [(197, 8, 768), (189, 16, 768), (21, 10, 1024), (257, 24, 1280), (17, 8, 256)])
@pytest.mark.parametrize("with_size", [False, True])
@pytest.mark.parametrize("h_dtype", [0, 1])
def test_merge(L, t, r, dim, with_size, h_dtype):
    b = 4
    g = torch.Generator().manual_seed(t + r + dim)
    x = torch.randn(b, t, dim, generator=g)
    size = torch.randint(1, 5, (b, t, 1), generator=g).float() if with_size else None
    metric = torch.randn(b, t, 64, generator=g)
    src, dst, unm, _, _ = vit_oracle.bipartite_soft_matching(metric, r)
    xr, sr = vit_oracle.merge_wavg(x, size, src, dst, unm)
    lw = torch.randn(dim, generator=g)
    lb = torch.randn(dim, generator=g)
    hr = F.layer_norm(xr, (dim,), lw, lb, eps=1e-6)
    tp = t - r
    xo = torch.empty(b, tp, dim, device="cuda")
    so = torch.empty(b, tp, device="cuda")
    ho = torch.empty(b, tp, dim, device="cuda", dtype=torch.bfloat16 if h_dtype == 0 else torch.float32)
    i32 = lambda v: v.to(torch.int32).cuda().contiguous()  # noqa: E731
    sg, dg, ug = i32(src), i32(dst), i32(unm)
    xd = x.cuda()
    sd = size[..., 0].cuda().contiguous() if size is not None else None
    lwd, lbd = lw.cuda(), lb.cuda()
    _chk(L.ta_merge(xd.data_ptr(), sd.data_ptr() if sd is not None else None, b, t, dim, r,
                    sg.data_ptr(), dg.data_ptr(), ug.data_ptr(), lwd.data_ptr(), lbd.data_ptr(),
                    xo.data_ptr(), so.data_ptr(), ho.data_ptr(), h_dtype, _s()))
    torch.cuda.synchronize()
    # same operation order as scatter_reduce(sum): the merged rows agree to fp32 rounding
    torch.testing.assert_close(xo.cpu(), xr, rtol=1e-6, atol=1e-6)
    torch.testing.assert_close(so.cpu(), sr[..., 0], rtol=0, atol=0)
    if h_dtype == 0:
        torch.testing.assert_close(ho.float().cpu(), hr, rtol=1e-2, atol=3e-2)
    else:
        torch.testing.assert_close(ho.cpu(), hr, rtol=1e-5, atol=1e-5)
