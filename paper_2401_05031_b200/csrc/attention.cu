// Proportional attention (ToMe prop_attn):
//   o = softmax(q k^T / sqrt(hd) + log(size_j)) v     per (image, head)
// qkv is the QKV GEMM output [B*t, 3D] (columns s*D + h*hd + j), out is [B*t, D].
// size == null means all-ones (no bias) — layer 0 and gamma >= 0.
//
// bf16: flash-style, one CTA per (64-query tile, head, image), 4 warps x 16 query rows,
// keys streamed in blocks of 64 through smem (double-buffered cp.async), online softmax
// in fp32 registers, m16n8k16 bf16 MMAs.
// fp32: SIMT reference-precision kernel for the fp32 parity mode.
#include <cfloat>
#include <cstdlib>

#include "common.h"
#include "ptx.cuh"

namespace ta {

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool pred) {
  const uint32_t s = smem_u32(smem);
  const int sz = pred ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(s), "l"(gmem), "r"(sz)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void ldsm_x4(uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3,
                                        const void* p) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(smem_u32(p)));
}
__device__ __forceinline__ void ldsm_x2(uint32_t& r0, uint32_t& r1, const void* p) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x2.shared.b16 {%0,%1}, [%2];"
               : "=r"(r0), "=r"(r1)
               : "r"(smem_u32(p)));
}
__device__ __forceinline__ void ldsm_x2_t(uint32_t& r0, uint32_t& r1, const void* p) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x2.trans.shared.b16 {%0,%1}, [%2];"
               : "=r"(r0), "=r"(r1)
               : "r"(smem_u32(p)));
}
__device__ __forceinline__ void mma_bf16_16816(float (&d)[4], const uint32_t (&a)[4],
                                               uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

template <int HD>
struct AttnCfg {
  static constexpr int kBQ = 64;        // query rows per CTA
  static constexpr int kBK = 64;        // keys per block
  static constexpr int kLd = HD + 8;    // smem row stride (bf16), breaks ldmatrix conflicts
  static constexpr int kChunks = HD / 8;  // 16-byte chunks per row
  static constexpr int kSmem = (kBQ + 4 * kBK) * kLd * 2 + 2 * kBK * 4;
};

// hd 64: capped at 128 registers (no spills) for four CTAs per SM instead of three -- the kernel
// runs the t <= 64 tail layers of the merge schedules and is latency-bound: t = 21 / 37 / 53 / 64
// 23.3 / 24.0 / 26.3 / 30.5 -> 20.6 / 21.6 / 24.0 / 27.0 us (B = 256, H = 12).  hd 80 would spill.
template <int HD>
__global__ void __launch_bounds__(128, HD == 64 ? 4 : 1)
    attn_bf16_kernel(const __nv_bfloat16* __restrict__ qkv, const float* __restrict__ size,
                     int t, int H, __nv_bfloat16* __restrict__ out, float scale_log2) {
  using C = AttnCfg<HD>;
  extern __shared__ __align__(128) uint8_t attn_smem[];
  auto* Qs = reinterpret_cast<__nv_bfloat16*>(attn_smem);
  auto (*Ks)[C::kBK * C::kLd] =
      reinterpret_cast<__nv_bfloat16(*)[C::kBK * C::kLd]>(Qs + C::kBQ * C::kLd);
  auto (*Vs)[C::kBK * C::kLd] = Ks + 2;
  auto (*Ls)[C::kBK] = reinterpret_cast<float(*)[C::kBK]>(Vs + 2);  // log2(size), -inf past t

  const int qt = blockIdx.x, h = blockIdx.y, b = blockIdx.z;
  const int D = H * HD;
  const long long rs = 3LL * D;  // qkv row stride
  const __nv_bfloat16* base = qkv + static_cast<long long>(b) * t * rs;
  const int warp = warp_id(), lane = lane_id();
  const int q0 = qt * C::kBQ;

  grid_dep_wait();

  grid_dep_launch();  // early trigger: the next kernel's prologue overlaps our tail

  auto load_kv = [&](int buf, int k0) {
    for (int i = threadIdx.x; i < C::kBK * C::kChunks; i += blockDim.x) {
      const int row = i / C::kChunks, ch = i % C::kChunks;
      const int key = k0 + row;
      const bool ok = key < t;
      const __nv_bfloat16* g = base + static_cast<long long>(ok ? key : 0) * rs + h * HD + ch * 8;
      cp_async16(&Ks[buf][row * C::kLd + ch * 8], g + D, ok);
      cp_async16(&Vs[buf][row * C::kLd + ch * 8], g + 2 * D, ok);
    }
    for (int i = threadIdx.x; i < C::kBK; i += blockDim.x) {
      const int key = k0 + i;
      float l = -INFINITY;
      if (key < t) l = size != nullptr ? __log2f(size[static_cast<long long>(b) * t + key]) : 0.f;
      Ls[buf][i] = l;
    }
  };

  // Q tile
  for (int i = threadIdx.x; i < C::kBQ * C::kChunks; i += blockDim.x) {
    const int row = i / C::kChunks, ch = i % C::kChunks;
    const int q = q0 + row;
    const bool ok = q < t;
    cp_async16(&Qs[row * C::kLd + ch * 8], base + static_cast<long long>(ok ? q : 0) * rs + h * HD + ch * 8, ok);
  }
  load_kv(0, 0);
  cp_async_commit();

  const int nkb = (t + C::kBK - 1) / C::kBK;
  constexpr int KC = HD / 16;  // k-chunks of the QK^T contraction
  uint32_t qa[KC][4];
  float o[HD / 8][4];
#pragma unroll
  for (int i = 0; i < HD / 8; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;
  float m_r[2] = {-INFINITY, -INFINITY};
  float l_r[2] = {0.f, 0.f};

  for (int kb = 0; kb < nkb; ++kb) {
    const int buf = kb & 1;
    if (kb + 1 < nkb) {
      load_kv(buf ^ 1, (kb + 1) * C::kBK);
      cp_async_commit();
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    if (kb == 0) {
      // Q fragments (rows warp*16 .. +16): A operand via ldmatrix x4.
#pragma unroll
      for (int kc = 0; kc < KC; ++kc) {
        const int row = warp * 16 + (lane % 16);
        const int col = kc * 16 + (lane / 16) * 8;
        ldsm_x4(qa[kc][0], qa[kc][1], qa[kc][2], qa[kc][3], &Qs[row * C::kLd + col]);
      }
    }
    // S = Q K^T for this warp's 16 rows x 64 keys: 8 n-chunks of 8 keys.
    float s[8][4];
#pragma unroll
    for (int nc = 0; nc < 8; ++nc) {
      s[nc][0] = s[nc][1] = s[nc][2] = s[nc][3] = 0.f;
#pragma unroll
      for (int kc = 0; kc < KC; ++kc) {
        uint32_t b0, b1;
        // B[k][n] = K[n][k]: 8x8 matrices with rows = keys, ldmatrix non-trans.
        const int krow = nc * 8 + (lane % 8);
        const int kcol = kc * 16 + ((lane / 8) % 2) * 8;
        ldsm_x2(b0, b1, &Ks[buf][krow * C::kLd + kcol]);
        mma_bf16_16816(s[nc], qa[kc], b0, b1);
      }
    }
    // scale + log-size bias (log2 domain), online softmax.
    float mx[2] = {m_r[0], m_r[1]};
#pragma unroll
    for (int nc = 0; nc < 8; ++nc) {
      const int kcol = nc * 8 + (lane % 4) * 2;
      const float l0 = Ls[buf][kcol], l1 = Ls[buf][kcol + 1];
      s[nc][0] = s[nc][0] * scale_log2 + l0;
      s[nc][1] = s[nc][1] * scale_log2 + l1;
      s[nc][2] = s[nc][2] * scale_log2 + l0;
      s[nc][3] = s[nc][3] * scale_log2 + l1;
      mx[0] = fmaxf(mx[0], fmaxf(s[nc][0], s[nc][1]));
      mx[1] = fmaxf(mx[1], fmaxf(s[nc][2], s[nc][3]));
    }
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      mx[i] = fmaxf(mx[i], __shfl_xor_sync(0xffffffffu, mx[i], 1));
      mx[i] = fmaxf(mx[i], __shfl_xor_sync(0xffffffffu, mx[i], 2));
    }
    float corr[2], rsum[2] = {0.f, 0.f};
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      corr[i] = exp2f(m_r[i] - mx[i]);  // m_r = -inf on the first block -> 0
      m_r[i] = mx[i];
    }
    uint32_t pa[4][4];  // P as A fragments: 4 k-chunks of 16 keys
#pragma unroll
    for (int nc = 0; nc < 8; ++nc) {
      const float p0 = exp2f(s[nc][0] - mx[0]);
      const float p1 = exp2f(s[nc][1] - mx[0]);
      const float p2 = exp2f(s[nc][2] - mx[1]);
      const float p3 = exp2f(s[nc][3] - mx[1]);
      rsum[0] += p0 + p1;
      rsum[1] += p2 + p3;
      const int kc = nc / 2;
      if ((nc & 1) == 0) {
        pa[kc][0] = pack_bf16(p0, p1);
        pa[kc][1] = pack_bf16(p2, p3);
      } else {
        pa[kc][2] = pack_bf16(p0, p1);
        pa[kc][3] = pack_bf16(p2, p3);
      }
    }
#pragma unroll
    for (int i = 0; i < 2; ++i) l_r[i] = l_r[i] * corr[i] + rsum[i];
#pragma unroll
    for (int dc = 0; dc < HD / 8; ++dc) {
      o[dc][0] *= corr[0];
      o[dc][1] *= corr[0];
      o[dc][2] *= corr[1];
      o[dc][3] *= corr[1];
    }
    // O += P V: B[k = key][n = d] from V rows via ldmatrix.trans.
#pragma unroll
    for (int kc = 0; kc < 4; ++kc) {
#pragma unroll
      for (int dc = 0; dc < HD / 8; ++dc) {
        uint32_t b0, b1;
        const int vrow = kc * 16 + (lane % 16);
        ldsm_x2_t(b0, b1, &Vs[buf][vrow * C::kLd + dc * 8]);
        mma_bf16_16816(o[dc], pa[kc], b0, b1);
      }
    }
    __syncthreads();
  }
  // finalize: quad-reduce the row sums, normalise, store bf16.
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    l_r[i] += __shfl_xor_sync(0xffffffffu, l_r[i], 1);
    l_r[i] += __shfl_xor_sync(0xffffffffu, l_r[i], 2);
  }
  const int r0 = q0 + warp * 16 + lane / 4;
#pragma unroll
  for (int half = 0; half < 2; ++half) {
    const int q = r0 + half * 8;
    if (q >= t) continue;
    const float inv = 1.0f / l_r[half];
    __nv_bfloat16* orow = out + (static_cast<long long>(b) * t + q) * D + h * HD;
#pragma unroll
    for (int dc = 0; dc < HD / 8; ++dc) {
      const int col = dc * 8 + (lane % 4) * 2;
      *reinterpret_cast<uint32_t*>(orow + col) =
          pack_bf16(o[dc][2 * half] * inv, o[dc][2 * half + 1] * inv);
    }
  }
}

// fp32 SIMT: one thread per query row, keys/values through smem in blocks of 32.
template <int HD>
__global__ void __launch_bounds__(128)
    attn_f32_kernel(const float* __restrict__ qkv, const float* __restrict__ size, int t, int H,
                    float* __restrict__ out, float scale) {
  __shared__ float Ks[32][HD + 1];
  __shared__ float Vs[32][HD + 1];
  __shared__ float Lb[32];
  const int h = blockIdx.y, b = blockIdx.z;
  const int D = H * HD;
  const long long rs = 3LL * D;
  const float* base = qkv + static_cast<long long>(b) * t * rs;
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  float qv[HD], o[HD];
#pragma unroll
  for (int j = 0; j < HD; ++j) {
    qv[j] = q < t ? base[q * rs + h * HD + j] : 0.f;
    o[j] = 0.f;
  }
  float m = -INFINITY, l = 0.f;
  for (int k0 = 0; k0 < t; k0 += 32) {
    __syncthreads();
    for (int i = threadIdx.x; i < 32 * HD; i += blockDim.x) {
      const int row = i / HD, j = i % HD;
      const int key = k0 + row;
      Ks[row][j] = key < t ? base[key * rs + D + h * HD + j] : 0.f;
      Vs[row][j] = key < t ? base[key * rs + 2 * D + h * HD + j] : 0.f;
    }
    if (threadIdx.x < 32) {
      const int key = k0 + threadIdx.x;
      Lb[threadIdx.x] = key < t ? (size ? logf(size[static_cast<long long>(b) * t + key]) : 0.f) : -INFINITY;
    }
    __syncthreads();
    const int kn = min(32, t - k0);
    for (int kk = 0; kk < kn; ++kk) {
      float s = 0.f;
#pragma unroll
      for (int j = 0; j < HD; ++j) s = fmaf(qv[j], Ks[kk][j], s);
      s = s * scale + Lb[kk];
      const float mn = fmaxf(m, s);
      const float corr = expf(m - mn);
      const float p = expf(s - mn);
      l = l * corr + p;
#pragma unroll
      for (int j = 0; j < HD; ++j) o[j] = o[j] * corr + p * Vs[kk][j];
      m = mn;
    }
  }
  if (q < t) {
    float* orow = out + (static_cast<long long>(b) * t + q) * D + h * HD;
#pragma unroll
    for (int j = 0; j < HD; ++j) orow[j] = o[j] / l;
  }
}

// 0 = default, by measured speed (tools/attn_bench.py, B = 256, H = 12, hd = 64): the mma.sync
// kernel for t <= 64 (one 64-row query tile: 24.7 vs 37.4 us at t = 53), the whole-row tcgen05
// kernel (attention_tc.cu) for 64 < t <= 512 (117 vs 213 / 239 us at t = 197), the chunk-
// pipelined tcgen05 kernel (attention_fa.cu) beyond (1420 vs 1771 us at t = 581, H = 16).
// head_dim 80 (ViT-H/14): the whole-row tcgen05 kernel with a 16-column SW32 tail for
// 64 < t <= 512 (1066 vs 1391 us at t = 257, B = 512, H = 16), mma.sync otherwise.
// TA_ATTENTION_BACKEND=tc / fa / mma / tp forces one kernel (the parity tests cover all four).
// The P-in-TMEM kernel (attention_tp.cu, hd 64, 64 < t <= 256) is correct but measured slower
// (141 vs 117 us at t = 197, 103 vs 90 us at t = 149; profiles/r02_attn.md), so it is not a default.
static int attention_backend() {
  static int mode = -1;
  if (mode < 0) {
    const char* v = getenv("TA_ATTENTION_BACKEND");
    mode = !v ? 0 : v[0] == 'm' ? 1 : (v[0] == 't' && v[1] == 'c') ? 2 : v[0] == 'f' ? 3 : v[0] == 't' ? 4 : 0;
  }
  return mode;
}

int attention(const void* qkv, const float* size, int B, int t, int H, int hd, void* out,
              int dtype, cudaStream_t s) {
  if (t <= 0) return TA_OK;
  cudaError_t e;
  const int backend = attention_backend();
  if (dtype == TA_DTYPE_BF16 && backend != 1 && !(backend == 0 && t <= 64)) {
    int rc = TA_ERR_SHAPE;
    if (backend == 4) rc = attention_tp(qkv, size, B, t, H, hd, out, s);
    if (rc == TA_ERR_SHAPE && (backend == 2 || ((backend == 0 || backend == 4) && t <= 512)))
      rc = attention_tc(qkv, size, B, t, H, hd, out, s);
    if (rc == TA_ERR_SHAPE && backend != 2) rc = attention_fa(qkv, size, B, t, H, hd, out, s);
    if (rc != TA_ERR_SHAPE) return rc;  // outside the tcgen05 envelopes -> mma.sync below
  }
  if (dtype == TA_DTYPE_BF16) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((t + 63) / 64, H, B);
    cfg.blockDim = dim3(128);
    cfg.dynamicSmemBytes = hd == 64 ? AttnCfg<64>::kSmem : AttnCfg<80>::kSmem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled();
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    const float scale_log2 = 1.4426950408889634f / sqrtf(static_cast<float>(hd));
    const auto* q = static_cast<const __nv_bfloat16*>(qkv);
    auto* o = static_cast<__nv_bfloat16*>(out);
    if (hd == 64) {
      cudaFuncSetAttribute(attn_bf16_kernel<64>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           AttnCfg<64>::kSmem);
      e = cudaLaunchKernelEx(&cfg, attn_bf16_kernel<64>, q, size, t, H, o, scale_log2);
    } else if (hd == 80) {
      cudaFuncSetAttribute(attn_bf16_kernel<80>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           AttnCfg<80>::kSmem);
      e = cudaLaunchKernelEx(&cfg, attn_bf16_kernel<80>, q, size, t, H, o, scale_log2);
    }
    else
      return TA_ERR_SHAPE;
  } else {
    dim3 grid((t + 127) / 128, H, B);
    const float scale = 1.0f / sqrtf(static_cast<float>(hd));
    const auto* q = static_cast<const float*>(qkv);
    auto* o = static_cast<float*>(out);
    if (hd == 64)
      attn_f32_kernel<64><<<grid, 128, 0, s>>>(q, size, t, H, o, scale);
    else if (hd == 80)
      attn_f32_kernel<80><<<grid, 128, 0, s>>>(q, size, t, H, o, scale);
    else
      return TA_ERR_SHAPE;
    e = cudaGetLastError();
  }
  return e == cudaSuccess ? TA_OK : set_last_cuda_error(e);
}

}  // namespace ta
