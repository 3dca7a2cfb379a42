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
// One thread per (patch, c, ky) segment: P consecutive input floats (64 B at P = 16) straight
// from HBM in registers, P consecutive output elements written back.  Consecutive threads own
// consecutive (c, ky) of one patch, so a warp's stores are one contiguous run of the output row
// and every input byte is read once; one integer division per P elements (the previous
// element-wise im2col spent most of its time in runtime divisions).
template <int kP, typename T>
__device__ __forceinline__ void patch_segment(const float* __restrict__ src, T* __restrict__ dst) {
  float v[kP];
  if constexpr (kP % 4 == 0) {
#pragma unroll
    for (int i = 0; i < kP / 4; ++i) {
      const float4 q = __ldg(reinterpret_cast<const float4*>(src) + i);
      v[4 * i] = q.x; v[4 * i + 1] = q.y; v[4 * i + 2] = q.z; v[4 * i + 3] = q.w;
    }
  } else {
#pragma unroll
    for (int i = 0; i < kP / 2; ++i) {
      const float2 q = __ldg(reinterpret_cast<const float2*>(src) + i);
      v[2 * i] = q.x; v[2 * i + 1] = q.y;
    }
  }
  if constexpr (sizeof(T) == 2) {
    uint32_t w[kP / 2];
#pragma unroll
    for (int i = 0; i < kP / 2; ++i) w[i] = pack_bf16(v[2 * i], v[2 * i + 1]);
    if constexpr (kP % 8 == 0) {
#pragma unroll
      for (int i = 0; i < kP / 8; ++i)
        reinterpret_cast<uint4*>(dst)[i] = make_uint4(w[4 * i], w[4 * i + 1], w[4 * i + 2], w[4 * i + 3]);
    } else {
#pragma unroll
      for (int i = 0; i < kP / 2; ++i) reinterpret_cast<uint32_t*>(dst)[i] = w[i];
    }
  } else {
#pragma unroll
    for (int i = 0; i < kP / 2; ++i)
      reinterpret_cast<float2*>(dst)[i] = make_float2(v[2 * i], v[2 * i + 1]);
  }
}

// kP = 0: runtime patch size (scalar copies); kP = 14 / 16: the ViT-H/14 and ViT-B,L/16 cases.
template <int kP, typename T>
__global__ void __launch_bounds__(256) patchify_kernel(const float* __restrict__ img,
                                                       T* __restrict__ out, int B, int S, int P_rt,
                                                       int Kp) {
  const int P = kP ? kP : P_rt;
  const int G = S / P;
  const int n = B * G * G * 3 * P;  // < 2^31 (checked by the launcher)
  grid_dep_wait();
  grid_dep_launch();
  // idx walks the image in memory order (b, c, py, ky, px): a warp reads whole image rows.
  for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < n; idx += gridDim.x * blockDim.x) {
    int r = idx / G;
    const int px = idx - r * G;
    int r2 = r / P;
    const int ky = r - r2 * P;
    r = r2 / G;
    const int py = r2 - r * G;
    const int b = r / 3;
    const int c = r - b * 3;
    const int patch = (b * G + py) * G + px;
    const int seg = c * P + ky;
    const float* src = img + ((static_cast<long long>(b) * 3 + c) * S + py * P + ky) * S + px * P;
    T* row = out + static_cast<long long>(patch) * Kp;
    T* dst = row + seg * P;
    if constexpr (kP != 0) {
      patch_segment<kP, T>(src, dst);
    } else {
      for (int kx = 0; kx < P; ++kx) dst[kx] = static_cast<T>(__ldg(src + kx));
    }
    if (seg == 0)  // zero padding columns [3P^2, Kp)
      for (int col = 3 * P * P; col < Kp; ++col) row[col] = static_cast<T>(0.f);
  }
}

// bf16, P = 14 (ViT-H/14): one CTA per (image, patch row py) band.  The band's 3 x P image rows are read
// with coalesced 16-byte loads into shared memory, then the G patch rows of the output are
// written as coalesced 16-byte chunks (8 bf16), the padding columns [3P^2, Kp) as zeros.
// Neither side depends on P dividing 16 bytes (P = 14: 56-byte segments): 313 -> 170 us at b=512.
template <int kP>
__global__ void __launch_bounds__(256) patchify_band_kernel(const float* __restrict__ img,
                                                            __nv_bfloat16* __restrict__ out, int S,
                                                            int Kp) {
  extern __shared__ float band[];  // [3 * kP][S]
  const int G = S / kP;
  const int b = blockIdx.x / G, py = blockIdx.x - (blockIdx.x / G) * G;
  grid_dep_wait();
  grid_dep_launch();
  const int s4 = S / 4;
  for (int i = threadIdx.x; i < 3 * kP * s4; i += blockDim.x) {
    const int row = i / s4, x4 = i - row * s4;  // row = c * kP + ky
    const int c = row / kP, ky = row - c * kP;
    const float4 v = __ldg(reinterpret_cast<const float4*>(
                               img + ((static_cast<long long>(b) * 3 + c) * S + py * kP + ky) * S) +
                           x4);
    reinterpret_cast<float4*>(band)[i] = v;
  }
  __syncthreads();
  const int kc = Kp / 8;  // 8-element output chunks per patch row
  __nv_bfloat16* orow0 = out + (static_cast<long long>(b) * G + py) * G * Kp;
  for (int q = threadIdx.x; q < G * kc; q += blockDim.x) {
    const int px = q / kc, e0 = (q - px * kc) * 8;
    uint32_t w[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      float f[2];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int e = e0 + 2 * k + h;
        float v = 0.f;
        if (e < 3 * kP * kP) {
          const int c = e / (kP * kP), rem = e - c * kP * kP;
          const int ky = rem / kP, kx = rem - ky * kP;
          v = band[(c * kP + ky) * S + px * kP + kx];
        }
        f[h] = v;
      }
      w[k] = pack_bf16(f[0], f[1]);
    }
    *reinterpret_cast<uint4*>(orow0 + static_cast<long long>(px) * Kp + e0) = make_uint4(w[0], w[1], w[2], w[3]);
  }
}

template <int kP>
static cudaError_t launch_patchify_band(const float* img, void* out, int B, int S, int Kp, cudaStream_t s) {
  const size_t smem = static_cast<size_t>(3) * kP * S * sizeof(float);
  if (smem > 48 * 1024) {
    const cudaError_t e = cudaFuncSetAttribute(patchify_band_kernel<kP>,
                                               cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    if (e != cudaSuccess) return e;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(B * (S / kP));
  cfg.blockDim = dim3(256);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled();
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, patchify_band_kernel<kP>, img, static_cast<__nv_bfloat16*>(out), S, Kp);
}

template <int kP>
static cudaError_t launch_patchify(const float* img, void* out, int B, int S, int P, int Kp,
                                   int dtype, cudaStream_t s) {
  const long long n = static_cast<long long>(B) * (S / P) * (S / P) * 3 * P;
  const long long want = (n + 255) / 256;
  const int grid = static_cast<int>(want < 148LL * 16 ? want : 148LL * 16);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(256);
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled();
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  if (dtype == TA_DTYPE_BF16)
    return cudaLaunchKernelEx(&cfg, patchify_kernel<kP, __nv_bfloat16>, img,
                              static_cast<__nv_bfloat16*>(out), B, S, P, Kp);
  return cudaLaunchKernelEx(&cfg, patchify_kernel<kP, float>, img, static_cast<float*>(out), B, S,
                            P, Kp);
}

int patchify(const float* img, void* out, int B, int S, int P, int Kp, int dtype,
             cudaStream_t s) {
  if (S % P != 0 || Kp < 3 * P * P ||
      static_cast<long long>(B) * (S / P) * (S / P) * 3 * P >= (1LL << 31))
    return TA_ERR_SHAPE;
  cudaError_t e;
  const bool band = dtype == TA_DTYPE_BF16 && S % 4 == 0 && Kp % 8 == 0 && 3LL * P * S * 4 <= 200 * 1024 &&
                    static_cast<long long>(B) * (S / P) < (1LL << 31);
  // (the band kernel measured slower at P = 16 -- 71 vs 49 us at ViT-B/16 b=256 -- where the
  // per-thread kernel's 64-byte segments are already aligned and coalesced)
  if (band && P == 14)
    e = launch_patchify_band<14>(img, out, B, S, Kp, s);
  else if (P == 16 && S % 4 == 0)
    e = launch_patchify<16>(img, out, B, S, P, Kp, dtype, s);
  else if (P == 14 && S % 2 == 0)
    e = launch_patchify<14>(img, out, B, S, P, Kp, dtype, s);
  else
    e = launch_patchify<0>(img, out, B, S, P, Kp, dtype, s);
  return e == cudaSuccess ? TA_OK : set_last_cuda_error(e);
}

// ------------------------------------------------------------------ insert rows
// x is [B, t_total, D] fp32.  If cls != null: row 0 = cls + pos[0].  If gamma > 0: rows
// [prompt_row, prompt_row + gamma) = prompts[task_b][layer] (a [gamma, D] block found via
// the per-task pointer table; prompts are fp32 [depth, gamma, D]).  A task id outside
// [0, n_tasks) or a task without prompts at this gamma (null table entry) is never
// dereferenced: its prompt rows are written as NaN, so the image's logits come out NaN
// (ta_forward takes device-side ids and cannot validate them on the host).
template <int VEC>
__global__ void insert_rows_kernel(float* __restrict__ x, int t_total,
                                   const float* __restrict__ cls, const float* __restrict__ pos,
                                   const float* const* __restrict__ prompt_tab,
                                   const int32_t* __restrict__ task_ids, int n_tasks, int layer,
                                   int gamma, int prompt_row, __nv_bfloat16* __restrict__ xh,
                                   float* __restrict__ stats) {
  // One warp per inserted row, VEC float4 per lane (D = 128 VEC), all loads before the stores;
  // with xh / stats (LayerNorm folded into the QKV GEMM) the row is also written as bf16 and
  // its exact (sum, sumsq) stored.  The previous kernel may have written the prompt slots
  // (row-remapped TMA boxes), so nothing is stored before grid_dep_wait.
  constexpr int D = 128 * VEC;
  const int b = blockIdx.x;
  const int n_cls = cls != nullptr ? 1 : 0;
  const int n_rows = n_cls + (gamma > 0 ? gamma : 0);
  const float* P = nullptr;
  if (gamma > 0) {
    const int tk = task_ids[b];
    P = (tk >= 0 && tk < n_tasks) ? prompt_tab[tk] : nullptr;
    if (P != nullptr) P += static_cast<long long>(layer) * gamma * D;
  }
  const int lane = lane_id();
  grid_dep_wait();
  grid_dep_launch();
  for (int rr = warp_id(); rr < n_rows; rr += blockDim.x / 32) {
    const bool is_cls = rr < n_cls;
    const long long row = static_cast<long long>(b) * t_total + (is_cls ? 0 : prompt_row + rr - n_cls);
    float4 v[VEC];
    if (is_cls) {
#pragma unroll
      for (int i = 0; i < VEC; ++i) {
        const float4 a = reinterpret_cast<const float4*>(cls)[lane + 32 * i];
        const float4 p = reinterpret_cast<const float4*>(pos)[lane + 32 * i];
        v[i] = make_float4(a.x + p.x, a.y + p.y, a.z + p.z, a.w + p.w);
      }
    } else if (P != nullptr) {
      const float4* srow = reinterpret_cast<const float4*>(P + static_cast<long long>(rr - n_cls) * D);
#pragma unroll
      for (int i = 0; i < VEC; ++i) v[i] = srow[lane + 32 * i];
    } else {
#pragma unroll
      for (int i = 0; i < VEC; ++i) v[i] = make_float4(NAN, NAN, NAN, NAN);
    }
    float s = 0.f, q = 0.f;
#pragma unroll
    for (int i = 0; i < VEC; ++i) {
      reinterpret_cast<float4*>(x + row * D)[lane + 32 * i] = v[i];
      if (xh != nullptr) {
        uint2 pk;
        pk.x = pack_bf16(v[i].x, v[i].y);
        pk.y = pack_bf16(v[i].z, v[i].w);
        reinterpret_cast<uint2*>(xh + row * D)[lane + 32 * i] = pk;
        s += (v[i].x + v[i].y) + (v[i].z + v[i].w);
        q += (v[i].x * v[i].x + v[i].y * v[i].y) + (v[i].z * v[i].z + v[i].w * v[i].w);
      }
    }
    if (stats != nullptr) {
      s = warp_sum(s);
      q = warp_sum(q);
      // whole-row sums in slot 0, the other 128-column slots zero (common.h GemmEpi::stats)
      if (lane < VEC)
        *reinterpret_cast<float2*>(stats + 2 * (row * VEC + lane)) =
            lane == 0 ? make_float2(s, q) : make_float2(0.f, 0.f);
    }
  }
}

int insert_rows(float* x, int B, int t_total, int D, const float* cls, const float* pos,
                const float* const* prompt_tab, const int32_t* task_ids, int n_tasks, int layer,
                int gamma, int prompt_row, cudaStream_t s, void* xh, float* stats) {
  if (D % 128 != 0) return TA_ERR_SHAPE;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(B);
  cfg.blockDim = dim3(256);
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled();
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  auto* h = static_cast<__nv_bfloat16*>(xh);
  cudaError_t e;
  switch (D / 128) {
#define TA_INSERT_CASE(V) \
  case V:                 \
    e = cudaLaunchKernelEx(&cfg, insert_rows_kernel<V>, x, t_total, cls, pos, prompt_tab, task_ids, n_tasks, layer, gamma, prompt_row, h, stats); \
    break;
    TA_INSERT_CASE(2)
    TA_INSERT_CASE(6)
    TA_INSERT_CASE(8)
    TA_INSERT_CASE(10)
#undef TA_INSERT_CASE
    default:
      return TA_ERR_SHAPE;
  }
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
  attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled();
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
// Final LayerNorm of each image's class-token row + its task's linear head.  A CTA takes
// kHeadImgs images x kHeadCls classes: one warp per image normalises its row into smem
// (two-pass statistics), then for every task present among the images each warp owns classes
// of the CTA's class chunk and dots each weight row with every image of that task, so a
// head's weights are read once per kHeadImgs images instead of once per image.
constexpr int kHeadImgs = 8;
constexpr int kHeadCls = 16;
__global__ void __launch_bounds__(256) head_kernel(const float* __restrict__ x, int B, int t_total, int D,
                                                   const float* __restrict__ nw, const float* __restrict__ nb,
                                                   const HeadDesc* __restrict__ heads,
                                                   const int32_t* __restrict__ task, int n_tasks,
                                                   float* __restrict__ logits, int c_max) {
  extern __shared__ float hrow[];  // [kHeadImgs][D]
  __shared__ int s_task[kHeadImgs];
  grid_dep_wait();
  grid_dep_launch();
  const int b0 = blockIdx.x * kHeadImgs;
  const int n_img = min(kHeadImgs, B - b0);
  const int warp = static_cast<int>(warp_id()), lane = static_cast<int>(lane_id());
  const int nwarps = blockDim.x / 32;
  // D = 128 VEC with VEC <= 10 (ViT-B / L / H: 6 / 8 / 10): each lane's class-token values are
  // loaded as up to 10 float4 at once (a loop of dependent global loads through shared
  // memory cost ~30 us per forward).
  constexpr int kMaxVec = 10;
  const int vec = D / 128;
  if (warp < n_img) {
    const int b = b0 + warp;
    const float4* xr = reinterpret_cast<const float4*>(x + static_cast<long long>(b) * t_total * D);
    float4* hr = reinterpret_cast<float4*>(hrow + warp * D);
    float4 v[kMaxVec];
#pragma unroll
    for (int i = 0; i < kMaxVec; ++i)
      if (i < vec) v[i] = xr[lane + 32 * i];
    float sm = 0.f;
#pragma unroll
    for (int i = 0; i < kMaxVec; ++i)
      if (i < vec) sm += (v[i].x + v[i].y) + (v[i].z + v[i].w);
    const float mean = warp_sum(sm) / D;
    float q = 0.f;
#pragma unroll
    for (int i = 0; i < kMaxVec; ++i)
      if (i < vec) {
        const float a = v[i].x - mean, bb = v[i].y - mean, c = v[i].z - mean, d = v[i].w - mean;
        q += (a * a + bb * bb) + (c * c + d * d);
      }
    const float rstd = 1.0f / sqrtf(warp_sum(q) / D + 1e-6f);
#pragma unroll
    for (int i = 0; i < kMaxVec; ++i)
      if (i < vec) {
        const float4 g = __ldg(reinterpret_cast<const float4*>(nw) + lane + 32 * i);
        const float4 o = __ldg(reinterpret_cast<const float4*>(nb) + lane + 32 * i);
        hr[lane + 32 * i] = make_float4((v[i].x - mean) * rstd * g.x + o.x, (v[i].y - mean) * rstd * g.y + o.y,
                                        (v[i].z - mean) * rstd * g.z + o.z, (v[i].w - mean) * rstd * g.w + o.w);
      }
    // a task id outside [0, n_tasks) is mapped to -1 and its logits written as NaN
    if (lane == 0) s_task[warp] = (task[b] >= 0 && task[b] < n_tasks) ? task[b] : -1;
  }
  __syncthreads();
  for (int j = 0; j < n_img; ++j) {
    const int tk = s_task[j];
    bool first = true;  // handle each distinct task once, at its first image
    for (int jj = 0; jj < j; ++jj) first = first && s_task[jj] != tk;
    if (!first) continue;
    const HeadDesc h = tk >= 0 ? heads[tk] : HeadDesc{nullptr, nullptr, 0};
    const int c_end = min(c_max, static_cast<int>(blockIdx.y + 1) * kHeadCls);
    for (int c = static_cast<int>(blockIdx.y) * kHeadCls + warp; c < c_end; c += nwarps) {
      if (c >= h.classes) {
        // beyond the task's classes: -inf; invalid id or no head registered: NaN (loud)
        const float fill = h.classes > 0 ? -INFINITY : NAN;
        for (int im = 0; im < n_img; ++im)
          if (s_task[im] == tk && lane == 0) logits[static_cast<long long>(b0 + im) * c_max + c] = fill;
        continue;
      }
      const float4* wr = reinterpret_cast<const float4*>(h.w + static_cast<long long>(c) * D);
      float4 wv[kMaxVec];
#pragma unroll
      for (int i = 0; i < kMaxVec; ++i)
        if (i < vec) wv[i] = __ldg(wr + lane + 32 * i);
      for (int im = 0; im < n_img; ++im) {
        if (s_task[im] != tk) continue;
        const float4* hr = reinterpret_cast<const float4*>(hrow + im * D);
        float acc = 0.f;
#pragma unroll
        for (int i = 0; i < kMaxVec; ++i)
          if (i < vec) {
            const float4 hv = hr[lane + 32 * i];
            acc += (hv.x * wv[i].x + hv.y * wv[i].y) + (hv.z * wv[i].z + hv.w * wv[i].w);
          }
        acc = warp_sum(acc);
        if (lane == 0) logits[static_cast<long long>(b0 + im) * c_max + c] = acc + h.b[c];
      }
    }
  }
}

int head(const float* x, int B, int t_total, int D, const float* nw, const float* nb,
         const HeadDesc* heads, const int32_t* task, int n_tasks, float* logits, int c_max,
         cudaStream_t s) {
  if (D % 128 != 0 || D > 1280) return TA_ERR_SHAPE;
  const size_t smem = static_cast<size_t>(kHeadImgs) * D * sizeof(float);
  if (smem > 48 * 1024) {
    const cudaError_t e = cudaFuncSetAttribute(head_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                               static_cast<int>(smem));
    if (e != cudaSuccess) return set_last_cuda_error(e);
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((B + kHeadImgs - 1) / kHeadImgs, (c_max + kHeadCls - 1) / kHeadCls);
  cfg.blockDim = dim3(256);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled();
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  const cudaError_t e = cudaLaunchKernelEx(&cfg, head_kernel, x, B, t_total, D, nw, nb, heads, task, n_tasks, logits, c_max);
  return e == cudaSuccess ? TA_OK : set_last_cuda_error(e);
}

}  // namespace ta
