// Row-wise bandwidth kernels of the forward:
//   patchify     images fp32 NCHW -> patch matrix [B*Np, Kp] (im2col for the P x P / stride P conv)
//   insert_rows  cls row (layer 0) and per-task prompt rows P[task][gamma][l] (VPT prompt module)
//   layernorm    fp32 rows -> act dtype (timm eps 1e-6)
//   head         final LayerNorm on the cls row + per-task linear head (TaskModel head)
// All are HBM-bound: one warp per row, 16-byte vector accesses, fp32 statistics.
#include "common.h"
#include "ptx.cuh"

namespace ta {

// ------------------------------------------------------------------ patchify
// out[b*Np + py*G + px, c*P*P + ky*P + kx] = img[b, c, py*P + ky, px*P + kx]; cols >= 3P^2 zero.
// One CTA per (patch row py, image b): the 3 x P x S input strip is read once, coalesced,
// into smem; the G x Kp output block is written with consecutive threads on consecutive
// columns (two elements per thread).
template <typename T>
__global__ void __launch_bounds__(256) patchify_kernel(const float* __restrict__ img,
                                                       T* __restrict__ out, int S, int P, int Kp) {
  extern __shared__ float strip[];  // [3][P][S]
  const int py = blockIdx.x, b = blockIdx.y;
  const int G = S / P;
  const int K = 3 * P * P;
  const int n4 = 3 * P * S / 4;
  for (int i = threadIdx.x; i < n4; i += blockDim.x) {
    const int e = 4 * i;
    const int c = e / (P * S), rem = e % (P * S);
    const int ky = rem / S, x = rem % S;
    reinterpret_cast<float4*>(strip)[i] = *reinterpret_cast<const float4*>(
        img + ((static_cast<long long>(b) * 3 + c) * S + py * P + ky) * S + x);
  }
  __syncthreads();
  T* ob = out + (static_cast<long long>(b) * G * G + static_cast<long long>(py) * G) * Kp;
  const int total2 = G * Kp / 2;
  for (int i = threadIdx.x; i < total2; i += blockDim.x) {
    float v[2];
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int idx = 2 * i + u;
      const int px = idx / Kp, col = idx % Kp;
      float val = 0.f;
      if (col < K) {
        const int c = col / (P * P), rem = col % (P * P);
        const int ky = rem / P, kx = rem % P;
        val = strip[(c * P + ky) * S + px * P + kx];
      }
      v[u] = val;
    }
    if constexpr (sizeof(T) == 2)
      reinterpret_cast<uint32_t*>(ob)[i] = pack_bf16(v[0], v[1]);
    else
      reinterpret_cast<float2*>(ob)[i] = make_float2(v[0], v[1]);
  }
}

int patchify(const float* img, void* out, int B, int S, int P, int Kp, int dtype,
             cudaStream_t s) {
  if (S % 4 != 0 || Kp % 2 != 0) return TA_ERR_SHAPE;
  const size_t smem = static_cast<size_t>(3) * P * S * sizeof(float);
  dim3 grid(S / P, B);
  if (dtype == TA_DTYPE_BF16)
    patchify_kernel<__nv_bfloat16><<<grid, 256, smem, s>>>(img, static_cast<__nv_bfloat16*>(out), S, P, Kp);
  else
    patchify_kernel<float><<<grid, 256, smem, s>>>(img, static_cast<float*>(out), S, P, Kp);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? TA_OK : set_last_cuda_error(e);
}

// ------------------------------------------------------------------ insert rows
// x is [B, t_total, D] fp32.  If cls != null: row 0 = cls + pos[0].  If gamma > 0: rows
// [prompt_row, prompt_row + gamma) = prompts[task_b][layer] (a [gamma, D] block found via
// the per-task pointer table; prompts are fp32 [depth, gamma, D]).
__global__ void insert_rows_kernel(float* __restrict__ x, int t_total, int D,
                                   const float* __restrict__ cls, const float* __restrict__ pos,
                                   const float* const* __restrict__ prompt_tab,
                                   const int32_t* __restrict__ task_ids, int layer, int gamma,
                                   int prompt_row, __nv_bfloat16* __restrict__ xh,
                                   float* __restrict__ stats) {
  // One warp per inserted row; with xh / stats (LayerNorm folded into the QKV GEMM) the
  // row is also written as bf16 and its exact (sum, sumsq) stored.
  const int b = blockIdx.x;
  const int n_cls = cls != nullptr ? 1 : 0;
  const int n_rows = n_cls + (gamma > 0 ? gamma : 0);
  const float* P = gamma > 0 ? prompt_tab[task_ids[b]] + static_cast<long long>(layer) * gamma * D
                             : nullptr;
  const int lane = lane_id();
  for (int rr = warp_id(); rr < n_rows; rr += blockDim.x / 32) {
    const bool is_cls = rr < n_cls;
    const long long row = static_cast<long long>(b) * t_total + (is_cls ? 0 : prompt_row + rr - n_cls);
    const float* srow = is_cls ? nullptr : P + static_cast<long long>(rr - n_cls) * D;
    float s = 0.f, q = 0.f;
    for (int c = 4 * lane; c < D; c += 128) {
      float4 v;
      if (is_cls) {
        const float4 a = *reinterpret_cast<const float4*>(cls + c);
        const float4 p = *reinterpret_cast<const float4*>(pos + c);
        v = make_float4(a.x + p.x, a.y + p.y, a.z + p.z, a.w + p.w);
      } else {
        v = *reinterpret_cast<const float4*>(srow + c);
      }
      *reinterpret_cast<float4*>(x + row * D + c) = v;
      if (xh != nullptr) {
        uint2 pk;
        pk.x = pack_bf16(v.x, v.y);
        pk.y = pack_bf16(v.z, v.w);
        *reinterpret_cast<uint2*>(xh + row * D + c) = pk;
        s += (v.x + v.y) + (v.z + v.w);
        q += (v.x * v.x + v.y * v.y) + (v.z * v.z + v.w * v.w);
      }
    }
    if (stats != nullptr) {
      s = warp_sum(s);
      q = warp_sum(q);
      if (lane == 0) *reinterpret_cast<float2*>(stats + 2 * row) = make_float2(s, q);
    }
  }
}

int insert_rows(float* x, int B, int t_total, int D, const float* cls, const float* pos,
                const float* const* prompt_tab, const int32_t* task_ids, int layer, int gamma,
                int prompt_row, cudaStream_t s, void* xh, float* stats) {
  if (D % 128 != 0) return TA_ERR_SHAPE;
  insert_rows_kernel<<<B, 256, 0, s>>>(x, t_total, D, cls, pos, prompt_tab, task_ids, layer,
                                       gamma, prompt_row, static_cast<__nv_bfloat16*>(xh), stats);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? TA_OK : set_last_cuda_error(e);
}

// ------------------------------------------------------------------ layernorm
// One warp per row; VEC float4 per lane (D = 128 * VEC).  Two-pass mean / variance in
// registers (biased variance, as torch.nn.LayerNorm).
template <int VEC, typename T>
__global__ void layernorm_kernel(const float* __restrict__ x, const float* __restrict__ w,
                                 const float* __restrict__ bvec, T* __restrict__ out, int rows) {
  constexpr int D = 128 * VEC;
  grid_dep_wait();
  grid_dep_launch();  // early trigger: the next kernel's prologue overlaps our tail
  const int row = blockIdx.x * (blockDim.x / 32) + warp_id();
  if (row < rows) {
    const int lane = lane_id();
    const float4* xr = reinterpret_cast<const float4*>(x + static_cast<long long>(row) * D);
    float4 v[VEC];
    float s = 0.f;
#pragma unroll
    for (int i = 0; i < VEC; ++i) {
      v[i] = xr[lane + 32 * i];
      s += (v[i].x + v[i].y) + (v[i].z + v[i].w);
    }
    const float mean = warp_sum(s) / D;
    float q = 0.f;
#pragma unroll
    for (int i = 0; i < VEC; ++i) {
      const float a = v[i].x - mean, b = v[i].y - mean, c = v[i].z - mean, d = v[i].w - mean;
      q += (a * a + b * b) + (c * c + d * d);
    }
    const float rstd = 1.0f / sqrtf(warp_sum(q) / D + 1e-6f);
#pragma unroll
    for (int i = 0; i < VEC; ++i) {
      const int c = 4 * (lane + 32 * i);
      const float4 g = __ldg(reinterpret_cast<const float4*>(w) + lane + 32 * i);
      const float4 bb = __ldg(reinterpret_cast<const float4*>(bvec) + lane + 32 * i);
      const float y0 = (v[i].x - mean) * rstd * g.x + bb.x;
      const float y1 = (v[i].y - mean) * rstd * g.y + bb.y;
      const float y2 = (v[i].z - mean) * rstd * g.z + bb.z;
      const float y3 = (v[i].w - mean) * rstd * g.w + bb.w;
      if constexpr (sizeof(T) == 2) {
        uint2 p;
        p.x = pack_bf16(y0, y1);
        p.y = pack_bf16(y2, y3);
        *reinterpret_cast<uint2*>(out + static_cast<long long>(row) * D + c) = p;
      } else {
        *reinterpret_cast<float4*>(out + static_cast<long long>(row) * D + c) =
            make_float4(y0, y1, y2, y3);
      }
    }
  }
}

template <typename T>
static int ln_dispatch(const float* x, const float* w, const float* b, T* out, int rows, int D,
                       cudaStream_t s) {
  const int grid = (rows + 7) / 8;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(256);
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaError_t e;
  switch (D) {
    case 256: e = cudaLaunchKernelEx(&cfg, layernorm_kernel<2, T>, x, w, b, out, rows); break;
    case 768: e = cudaLaunchKernelEx(&cfg, layernorm_kernel<6, T>, x, w, b, out, rows); break;
    case 1024: e = cudaLaunchKernelEx(&cfg, layernorm_kernel<8, T>, x, w, b, out, rows); break;
    case 1280: e = cudaLaunchKernelEx(&cfg, layernorm_kernel<10, T>, x, w, b, out, rows); break;
    default: return TA_ERR_SHAPE;
  }
  return e == cudaSuccess ? TA_OK : set_last_cuda_error(e);
}

int layernorm(const float* x, const float* w, const float* b, void* out, int rows, int D,
              int out_dtype, cudaStream_t s) {
  if (rows <= 0) return TA_OK;
  if (out_dtype == TA_DTYPE_BF16)
    return ln_dispatch(x, w, b, static_cast<__nv_bfloat16*>(out), rows, D, s);
  return ln_dispatch(x, w, b, static_cast<float*>(out), rows, D, s);
}

// ------------------------------------------------------------------ head
// logits[b, c] = LN(x[b, 0, :]) . W_task[c] + b_task[c] for c < C_task, -inf beyond.
__global__ void head_kernel(const float* __restrict__ x, int t_total, int D,
                            const float* __restrict__ nw, const float* __restrict__ nb,
                            const HeadDesc* __restrict__ heads, const int32_t* __restrict__ task,
                            float* __restrict__ logits, int c_max) {
  extern __shared__ float hrow[];
  __shared__ float red[32];
  const int b = blockIdx.x;
  const float* xr = x + static_cast<long long>(b) * t_total * D;
  const int nwarps = blockDim.x / 32;
  float s = 0.f;
  for (int c = threadIdx.x; c < D; c += blockDim.x) {
    hrow[c] = xr[c];
    s += hrow[c];
  }
  s = warp_sum(s);
  if (lane_id() == 0) red[warp_id()] = s;
  __syncthreads();
  float tot = 0.f;
  for (int i = 0; i < nwarps; ++i) tot += red[i];
  const float mean = tot / D;
  __syncthreads();
  float q = 0.f;
  for (int c = threadIdx.x; c < D; c += blockDim.x) {
    const float d = hrow[c] - mean;
    q += d * d;
  }
  q = warp_sum(q);
  if (lane_id() == 0) red[warp_id()] = q;
  __syncthreads();
  float qt = 0.f;
  for (int i = 0; i < nwarps; ++i) qt += red[i];
  const float rstd = 1.0f / sqrtf(qt / D + 1e-6f);
  for (int c = threadIdx.x; c < D; c += blockDim.x) hrow[c] = (hrow[c] - mean) * rstd * nw[c] + nb[c];
  __syncthreads();
  const HeadDesc h = heads[task[b]];
  for (int c = warp_id(); c < c_max; c += nwarps) {
    float acc = 0.f;
    if (c < h.classes) {
      const float* wr = h.w + static_cast<long long>(c) * D;
      for (int k = lane_id(); k < D; k += 32) acc += hrow[k] * wr[k];
      acc = warp_sum(acc);
      acc += h.b[c];
    } else {
      acc = -INFINITY;
    }
    if (lane_id() == 0) logits[static_cast<long long>(b) * c_max + c] = acc;
  }
}

int head(const float* x, int B, int t_total, int D, const float* nw, const float* nb,
         const HeadDesc* heads, const int32_t* task, float* logits, int c_max, cudaStream_t s) {
  head_kernel<<<B, 256, D * sizeof(float), s>>>(x, t_total, D, nw, nb, heads, task, logits, c_max);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? TA_OK : set_last_cuda_error(e);
}

}  // namespace ta
