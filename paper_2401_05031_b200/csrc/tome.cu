// Token merging (Appendix A `match` / `merge`):
//   match  ToMe bipartite soft matching: metric = mean_h k (optional), L2 normalise,
//          S = A B^T over alternating token sets (A = even rows incl. cls, B = odd rows),
//          S[cls, :] = -inf, row max/argmax (ties -> lowest column), top-r rows by a
//          stable descending order (rank counting: exact and deterministic),
//          unm = the remaining A rows ascending.
//   merge  size-weighted average: B_j <- (s_j x_j + sum_{i: dst_i = j} s_i x_i) / (s_j + sum s_i),
//          output order [A unmerged (cls first); B all], fused LayerNorm (LN2) of the
//          merged rows in the activation dtype.
// The per-image problem is small (A 99 x B 98 x 64 at t = 197) and latency-bound, so one
// CTA owns one image; the merge is HBM-bound (read t x D, write t' x D fp32 + t' x D act).
#include <cfloat>
#include <cstdlib>

#include "common.h"
#include "ptx.cuh"

namespace ta {

constexpr int kMatchThreads = 256;

// Dynamic smem: A rows [na][c+1], B rows [nb][c+1] (fp32, padded), node_max [na],
// node_idx [na], rank [na].
template <typename QT>
__global__ void __launch_bounds__(kMatchThreads)
    match_kernel(const float* __restrict__ metric, const QT* __restrict__ qkv, int t, int heads,
                 int c, int r, int32_t* __restrict__ src_out, int32_t* __restrict__ dst_out,
                 int32_t* __restrict__ unm_out) {
  extern __shared__ float sm[];
  const int b = blockIdx.x;
  const int na = (t + 1) / 2;
  const int nb = t / 2;
  const int cs = c + 1;
  float* As = sm;
  float* Bs = As + na * cs;
  float* node_max = Bs + nb * cs;
  int* node_idx = reinterpret_cast<int*>(node_max + na);
  int* rank = node_idx + na;
  const int warp = warp_id(), lane = lane_id(), nwarps = blockDim.x / 32;

  grid_dep_wait();

  grid_dep_launch();  // early trigger: the next kernel's prologue overlaps our tail
  // 1) metric rows (mean over heads, fixed head order), then L2-normalise (x / ||x||).
  for (int row = warp; row < t; row += nwarps) {
    float* dstrow = (row & 1) ? Bs + (row >> 1) * cs : As + (row >> 1) * cs;
    float ss = 0.f;
    for (int j = lane; j < c; j += 32) {
      float v;
      if (metric != nullptr) {
        v = metric[(static_cast<long long>(b) * t + row) * c + j];
      } else {
        const long long D = static_cast<long long>(heads) * c;
        const QT* kr = qkv + (static_cast<long long>(b) * t + row) * 3 * D + D + j;
        float acc = 0.f;
        for (int h = 0; h < heads; ++h) acc += static_cast<float>(kr[h * c]);
        v = acc / heads;
      }
      dstrow[j] = v;
      ss += v * v;
    }
    const float nrm = sqrtf(warp_sum(ss));
    for (int j = lane; j < c; j += 32) dstrow[j] = dstrow[j] / nrm;
  }
  __syncthreads();

  // 2) scores and row max / argmax (lowest column on ties); row 0 (cls) is -inf.
  for (int i = warp; i < na; i += nwarps) {
    float best = -INFINITY;
    int best_j = 0;
    if (i > 0) {
      const float* ar = As + i * cs;
      for (int j = lane; j < nb; j += 32) {
        const float* br = Bs + j * cs;
        float acc = 0.f;
        for (int k = 0; k < c; ++k) acc = fmaf(ar[k], br[k], acc);
        if (acc > best) {  // j increases per lane: strict > keeps the lowest j
          best = acc;
          best_j = j;
        }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const float ov = __shfl_xor_sync(0xffffffffu, best, o);
        const int oj = __shfl_xor_sync(0xffffffffu, best_j, o);
        if (ov > best || (ov == best && oj < best_j)) {
          best = ov;
          best_j = oj;
        }
      }
    }
    if (lane == 0) {
      node_max[i] = best;
      node_idx[i] = best_j;
    }
  }
  __syncthreads();

  // 3) rank in the stable descending order: rank_i = #{j : v_j > v_i or (v_j == v_i and j < i)}.
  for (int i = threadIdx.x; i < na; i += blockDim.x) {
    const float vi = node_max[i];
    int rk = 0;
    for (int j = 0; j < na; ++j) {
      const float vj = node_max[j];
      rk += (vj > vi) || (vj == vi && j < i);
    }
    rank[i] = rk;
  }
  __syncthreads();

  // 4) src/dst by rank; unm = rows with rank >= r in ascending index order.
  int32_t* srcb = src_out + static_cast<long long>(b) * r;
  int32_t* dstb = dst_out + static_cast<long long>(b) * r;
  int32_t* unmb = unm_out + static_cast<long long>(b) * (na - r);
  for (int i = threadIdx.x; i < na; i += blockDim.x) {
    const int rk = rank[i];
    if (rk < r) {
      srcb[rk] = i;
      dstb[rk] = node_idx[i];
    } else {
      int pos = 0;
      for (int j = 0; j < i; ++j) pos += rank[j] >= r;
      unmb[pos] = i;
    }
  }
}

static int match_backend() {
  static int mode = -1;
  if (mode < 0) {
    const char* v = getenv("TA_MATCH_BACKEND");
    mode = (v && v[0] == 's') ? 1 : 0;
  }
  return mode;
}

int match(const float* metric, const void* qkv, int qkv_dtype, int B, int t, int heads, int c,
          int r, int32_t* src, int32_t* dst, int32_t* unm, float* scratch, cudaStream_t s,
          int32_t* row_map) {
  const int na = (t + 1) / 2, nb = t / 2;
  if (r <= 0 || r > na - 1 || t < 3) return TA_ERR_INVALID;
  if (scratch != nullptr && match_backend() == 0) {
    const int rc = match_tc(metric, qkv, qkv_dtype, B, t, heads, c, r, src, dst, unm, scratch, s, row_map);
    if (rc != TA_ERR_SHAPE) return rc;
  }
  const size_t smem = (static_cast<size_t>(na + nb) * (c + 1) + 3 * na) * sizeof(float);
  if (smem > 220 * 1024) return TA_ERR_SHAPE;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(B);
  cfg.blockDim = dim3(kMatchThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled();
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaError_t e;
  if (metric != nullptr || qkv_dtype == TA_DTYPE_F32) {
    auto k = match_kernel<float>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
    e = cudaLaunchKernelEx(&cfg, k, metric, static_cast<const float*>(qkv), t, heads, c, r, src,
                           dst, unm);
  } else {
    auto k = match_kernel<__nv_bfloat16>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
    e = cudaLaunchKernelEx(&cfg, k, metric, static_cast<const __nv_bfloat16*>(qkv), t, heads, c,
                           r, src, dst, unm);
  }
  if (e != cudaSuccess) return set_last_cuda_error(e);
  return row_map != nullptr ? merge_map(src, unm, B, t, r, row_map, s) : TA_OK;
}

// ------------------------------------------------------------------ merge + LN2
// grid (B, ceil(t'/ROWS)); one warp per output row; VEC float4 per lane (D = 128 VEC).
// 3 CTAs per SM (register cap 85): more rows' loads in flight, merge 592 -> 524 us per ViT-B/16
// forward at gamma = -16 and 772 -> 676 us at -8 (1 or 4 CTAs per SM, or two rows per warp
// iteration, measured slower).
template <int VEC, typename T>
__global__ void __launch_bounds__(256, 3)
    merge_kernel(const float* __restrict__ x, const float* __restrict__ size, int t, int r,
                 const int32_t* __restrict__ src, const int32_t* __restrict__ dst,
                 const int32_t* __restrict__ unm, const float* __restrict__ ln_w,
                 const float* __restrict__ ln_b, float* __restrict__ x_out,
                 float* __restrict__ size_out, T* __restrict__ h_out, float* __restrict__ stats_out) {
  constexpr int D = 128 * VEC;
  __shared__ int s_src[256];
  __shared__ int s_dst[256];
  const int b = blockIdx.x;
  const int na = (t + 1) / 2;
  const int n_unm = na - r;
  const int tp = t - r;
  grid_dep_wait();
  grid_dep_launch();  // early trigger: the next kernel's prologue overlaps our tail
  for (int i = threadIdx.x; i < r; i += blockDim.x) {
    s_src[i] = src[static_cast<long long>(b) * r + i];
    s_dst[i] = dst[static_cast<long long>(b) * r + i];
  }
  __syncthreads();
  const int lane = lane_id();
  const float* xb = x + static_cast<long long>(b) * t * D;
  const float* sb = size != nullptr ? size + static_cast<long long>(b) * t : nullptr;
  const int rows_per_cta = (blockDim.x / 32) * 4;
  const int o_begin = blockIdx.y * rows_per_cta;
  const int o_end = min(tp, o_begin + rows_per_cta);
  for (int o = o_begin + warp_id(); o < o_end; o += blockDim.x / 32) {
    float4 acc[VEC];
    float stot;
    if (o < n_unm) {
      const int tok = 2 * unm[static_cast<long long>(b) * n_unm + o];
      const float s = sb ? sb[tok] : 1.0f;
      const float4* xr = reinterpret_cast<const float4*>(xb + static_cast<long long>(tok) * D);
#pragma unroll
      for (int i = 0; i < VEC; ++i) {
        const float4 v = xr[lane + 32 * i];
        acc[i] = make_float4(v.x * s, v.y * s, v.z * s, v.w * s);
      }
      stot = s;
    } else {
      const int j = o - n_unm;
      const int tok = 2 * j + 1;
      const float s = sb ? sb[tok] : 1.0f;
      const float4* xr = reinterpret_cast<const float4*>(xb + static_cast<long long>(tok) * D);
#pragma unroll
      for (int i = 0; i < VEC; ++i) {
        const float4 v = xr[lane + 32 * i];
        acc[i] = make_float4(v.x * s, v.y * s, v.z * s, v.w * s);
      }
      stot = s;
      // scatter_reduce(sum, include_self) order: self, then sources in src order.
      for (int q = 0; q < r; ++q) {
        if (s_dst[q] != j) continue;
        const int stok = 2 * s_src[q];
        const float ss = sb ? sb[stok] : 1.0f;
        const float4* sr = reinterpret_cast<const float4*>(xb + static_cast<long long>(stok) * D);
#pragma unroll
        for (int i = 0; i < VEC; ++i) {
          const float4 v = sr[lane + 32 * i];
          acc[i].x += v.x * ss;
          acc[i].y += v.y * ss;
          acc[i].z += v.z * ss;
          acc[i].w += v.w * ss;
        }
        stot += ss;
      }
    }
    // x = (sum s x) / (sum s)
    float sum = 0.f;
#pragma unroll
    for (int i = 0; i < VEC; ++i) {
      acc[i].x /= stot;
      acc[i].y /= stot;
      acc[i].z /= stot;
      acc[i].w /= stot;
      sum += (acc[i].x + acc[i].y) + (acc[i].z + acc[i].w);
    }
    const long long orow = static_cast<long long>(b) * tp + o;
    float4* xo = reinterpret_cast<float4*>(x_out + orow * D);
#pragma unroll
    for (int i = 0; i < VEC; ++i) xo[lane + 32 * i] = acc[i];
    if (lane == 0) size_out[orow] = stot;
    if (stats_out != nullptr) {
      // LayerNorm folded into fc1 (bf16 path): xh = bf16(x') and exact row (sum, sumsq)
      float q2 = 0.f;
#pragma unroll
      for (int i = 0; i < VEC; ++i) {
        const int cidx = 4 * (lane + 32 * i);
        q2 += (acc[i].x * acc[i].x + acc[i].y * acc[i].y) + (acc[i].z * acc[i].z + acc[i].w * acc[i].w);
        uint2 p;
        p.x = pack_bf16(acc[i].x, acc[i].y);
        p.y = pack_bf16(acc[i].z, acc[i].w);
        *reinterpret_cast<uint2*>(reinterpret_cast<__nv_bfloat16*>(h_out) + orow * D + cidx) = p;
      }
      const float s_all = warp_sum(sum), q_all = warp_sum(q2);
      // whole-row sums in slot 0, the other 128-column slots zero (common.h GemmEpi::stats)
      if (lane < D / 128)
        *reinterpret_cast<float2*>(stats_out + 2 * (orow * (D / 128) + lane)) =
            lane == 0 ? make_float2(s_all, q_all) : make_float2(0.f, 0.f);
      continue;
    }
    // fused LN2
    const float mean = warp_sum(sum) / D;
    float q = 0.f;
#pragma unroll
    for (int i = 0; i < VEC; ++i) {
      const float a0 = acc[i].x - mean, a1 = acc[i].y - mean, a2 = acc[i].z - mean,
                  a3 = acc[i].w - mean;
      q += (a0 * a0 + a1 * a1) + (a2 * a2 + a3 * a3);
    }
    const float rstd = 1.0f / sqrtf(warp_sum(q) / D + 1e-6f);
#pragma unroll
    for (int i = 0; i < VEC; ++i) {
      const int cidx = 4 * (lane + 32 * i);
      const float4 g = __ldg(reinterpret_cast<const float4*>(ln_w) + lane + 32 * i);
      const float4 bb = __ldg(reinterpret_cast<const float4*>(ln_b) + lane + 32 * i);
      const float y0 = (acc[i].x - mean) * rstd * g.x + bb.x;
      const float y1 = (acc[i].y - mean) * rstd * g.y + bb.y;
      const float y2 = (acc[i].z - mean) * rstd * g.z + bb.z;
      const float y3 = (acc[i].w - mean) * rstd * g.w + bb.w;
      if constexpr (sizeof(T) == 2) {
        uint2 p;
        p.x = pack_bf16(y0, y1);
        p.y = pack_bf16(y2, y3);
        *reinterpret_cast<uint2*>(h_out + orow * D + cidx) = p;
      } else {
        *reinterpret_cast<float4*>(h_out + orow * D + cidx) = make_float4(y0, y1, y2, y3);
      }
    }
  }
}

template <typename T>
static int merge_dispatch(const float* x, const float* size, int B, int t, int D, int r,
                          const int32_t* src, const int32_t* dst, const int32_t* unm,
                          const float* ln_w, const float* ln_b, float* x_out, float* size_out,
                          T* h_out, float* stats_out, cudaStream_t s) {
  const int tp = t - r;
  const int rows_per_cta = 8 * 4;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(B, (tp + rows_per_cta - 1) / rows_per_cta);
  cfg.blockDim = dim3(256);
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled();
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaError_t e;
#define TA_MERGE_CASE(DIM, V)                                                                  \
  case DIM:                                                                                    \
    e = cudaLaunchKernelEx(&cfg, merge_kernel<V, T>, x, size, t, r, src, dst, unm, ln_w, ln_b, \
                           x_out, size_out, h_out, stats_out);                                 \
    break;
  switch (D) {
    TA_MERGE_CASE(256, 2)
    TA_MERGE_CASE(768, 6)
    TA_MERGE_CASE(1024, 8)
    TA_MERGE_CASE(1280, 10)
    default: return TA_ERR_SHAPE;
  }
#undef TA_MERGE_CASE
  return e == cudaSuccess ? TA_OK : set_last_cuda_error(e);
}

// ------------------------------------------------------------------ fused merge (bf16 path)
// merge_map: per input row of a layer, where the proj GEMM (EPI_BIAS_RESID_MERGE) writes it:
// unmerged A token -> its position in x' (ToMe output order [A_unm ; B]), B token -> its
// position after the unmerged A tokens, merged-away A token (src rank k) -> row B tp + b r + k
// (the source rows follow the B tp merged rows in the same buffer).
__global__ void __launch_bounds__(256) merge_map_kernel(const int32_t* __restrict__ src,
                                                        const int32_t* __restrict__ unm, int t, int r,
                                                        int32_t* __restrict__ row_map) {
  const int b = blockIdx.x;
  const int na = (t + 1) / 2, nb = t / 2, n_unm = na - r, tp = t - r;
  const long long in0 = static_cast<long long>(b) * t;
  const int out0 = b * tp;
  grid_dep_wait();
  grid_dep_launch();
  for (int p = threadIdx.x; p < n_unm; p += blockDim.x)
    row_map[in0 + 2 * unm[static_cast<long long>(b) * n_unm + p]] = out0 + p;
  for (int k = threadIdx.x; k < r; k += blockDim.x)
    row_map[in0 + 2 * src[static_cast<long long>(b) * r + k]] = static_cast<int>(gridDim.x) * tp + b * r + k;
  for (int j = threadIdx.x; j < nb; j += blockDim.x) row_map[in0 + 2 * j + 1] = out0 + n_unm + j;
}

// merge_fixup: x' already holds every kept token's row (written by the proj GEMM) and `side`
// (= x' + B tp rows) the merged-away sources.  Each destination B token that received sources becomes
// (s_d x_d + sum_k s_k x_k) / (s_d + sum_k s_k) in merge_kernel's order (self, then sources by
// rank), with its bf16 copy and whole-row statistics (slot 0); block y == 0 also writes the new
// size vector (ToMe merge_wavg's size sum).  One warp per destination (at its first source).
template <int VEC>
__global__ void __launch_bounds__(256)
    merge_fixup_kernel(float* __restrict__ x_out, const float* __restrict__ side,
                       const float* __restrict__ size, float* __restrict__ size_out, int t, int r,
                       const int32_t* __restrict__ src, const int32_t* __restrict__ dst,
                       const int32_t* __restrict__ unm, __nv_bfloat16* __restrict__ xh,
                       float* __restrict__ stats) {
  constexpr int D = 128 * VEC;
  constexpr int kMaxT = 1024;
  __shared__ int s_src[256];
  __shared__ int s_dst[256];
  __shared__ float s_size[kMaxT];  // this image's token sizes (ones at the first merge layer)
  const int b = blockIdx.x;
  const int na = (t + 1) / 2, n_unm = na - r, tp = t - r;
  grid_dep_wait();
  grid_dep_launch();
  // every global read up front and coalesced: the size loop below is then shared-memory only
  for (int i = threadIdx.x; i < r; i += blockDim.x) {
    s_src[i] = src[static_cast<long long>(b) * r + i];
    s_dst[i] = dst[static_cast<long long>(b) * r + i];
  }
  for (int i = threadIdx.x; i < t; i += blockDim.x)
    s_size[i] = size != nullptr ? size[static_cast<long long>(b) * t + i] : 1.0f;
  __syncthreads();
  if (blockIdx.y == 0) {
    for (int o = threadIdx.x; o < tp; o += blockDim.x) {
      float stot;
      if (o < n_unm) {
        stot = s_size[2 * unm[static_cast<long long>(b) * n_unm + o]];
      } else {
        const int j = o - n_unm;
        stot = s_size[2 * j + 1];
        for (int q = 0; q < r; ++q)
          if (s_dst[q] == j) stot += s_size[2 * s_src[q]];
      }
      size_out[static_cast<long long>(b) * tp + o] = stot;
    }
  }
  const int k = blockIdx.y * (blockDim.x / 32) + warp_id();
  if (k >= r) return;
  const int j = s_dst[k];
  for (int q = 0; q < k; ++q)
    if (s_dst[q] == j) return;  // handled by the warp of its first source
  const int lane = lane_id();
  const long long orow = static_cast<long long>(b) * tp + n_unm + j;
  const float s = s_size[2 * j + 1];
  float4* xr = reinterpret_cast<float4*>(x_out + orow * D);
  float4 acc[VEC];
#pragma unroll
  for (int i = 0; i < VEC; ++i) {
    const float4 v = xr[lane + 32 * i];
    acc[i] = make_float4(v.x * s, v.y * s, v.z * s, v.w * s);
  }
  float stot = s;
  for (int q = k; q < r; ++q) {
    if (s_dst[q] != j) continue;
    const float ss = s_size[2 * s_src[q]];
    const float4* sr = reinterpret_cast<const float4*>(side + (static_cast<long long>(b) * r + q) * D);
#pragma unroll
    for (int i = 0; i < VEC; ++i) {
      const float4 v = sr[lane + 32 * i];
      acc[i].x += v.x * ss;
      acc[i].y += v.y * ss;
      acc[i].z += v.z * ss;
      acc[i].w += v.w * ss;
    }
    stot += ss;
  }
  float sum = 0.f, q2 = 0.f;
#pragma unroll
  for (int i = 0; i < VEC; ++i) {
    acc[i].x /= stot;
    acc[i].y /= stot;
    acc[i].z /= stot;
    acc[i].w /= stot;
    sum += (acc[i].x + acc[i].y) + (acc[i].z + acc[i].w);
    q2 += (acc[i].x * acc[i].x + acc[i].y * acc[i].y) + (acc[i].z * acc[i].z + acc[i].w * acc[i].w);
    xr[lane + 32 * i] = acc[i];
    uint2 p;
    p.x = pack_bf16(acc[i].x, acc[i].y);
    p.y = pack_bf16(acc[i].z, acc[i].w);
    *reinterpret_cast<uint2*>(xh + orow * D + 4 * (lane + 32 * i)) = p;
  }
  const float s_all = warp_sum(sum), q_all = warp_sum(q2);
  if (lane < VEC)  // whole-row sums in slot 0, the other 128-column slots zero
    *reinterpret_cast<float2*>(stats + 2 * (orow * VEC + lane)) =
        lane == 0 ? make_float2(s_all, q_all) : make_float2(0.f, 0.f);
}

// merge_fixup, one CTA per image with one warp per source (r <= 32): every warp loads its
// source row (scaled by its size) into shared memory and, if it is its destination's first
// source, the destination row, all at once; after one barrier the first-source warp adds
// self, then the sources by rank (merge_kernel's order) -- one dependent global round trip
// instead of a chain of them.  Block-wide: the new size vector.
template <int VEC>
__global__ void __launch_bounds__(1024)
    merge_fixup_par_kernel(float* __restrict__ x_out, const float* __restrict__ side,
                           const float* __restrict__ size, float* __restrict__ size_out, int t, int r,
                           const int32_t* __restrict__ src, const int32_t* __restrict__ dst,
                           const int32_t* __restrict__ unm, __nv_bfloat16* __restrict__ xh,
                           float* __restrict__ stats) {
  constexpr int D = 128 * VEC;
  extern __shared__ float4 s_rows[];  // [r][D / 4]: s_k x_k of source k
  __shared__ int s_src[32];
  __shared__ int s_dst[32];
  __shared__ float s_ssz[32];  // size of source k
  const int b = blockIdx.x;
  const int na = (t + 1) / 2, n_unm = na - r, tp = t - r;
  const int k = warp_id(), lane = lane_id();
  grid_dep_wait();
  grid_dep_launch();
  // this warp's source and destination (every lane reads the same words: one broadcast)
  const int sk = src[static_cast<long long>(b) * r + k];
  const int j = dst[static_cast<long long>(b) * r + k];
  const float ss = size != nullptr ? size[static_cast<long long>(b) * t + 2 * sk] : 1.0f;
  if (lane == 0) {
    s_src[k] = sk;
    s_dst[k] = j;
    s_ssz[k] = ss;
  }
  const float4* sr = reinterpret_cast<const float4*>(side + (static_cast<long long>(b) * r + k) * D);
  float4 v[VEC];
#pragma unroll
  for (int i = 0; i < VEC; ++i) v[i] = sr[lane + 32 * i];
  __syncthreads();  // s_dst complete
  bool first = true;
  for (int q = 0; q < k; ++q) first = first && s_dst[q] != j;
  const long long orow = static_cast<long long>(b) * tp + n_unm + j;
  float4 acc[VEC];
  float s_d = 0.f;
  if (first) {  // the destination row, loaded beside the source row
    s_d = size != nullptr ? size[static_cast<long long>(b) * t + 2 * j + 1] : 1.0f;
    const float4* xr = reinterpret_cast<const float4*>(x_out + orow * D);
#pragma unroll
    for (int i = 0; i < VEC; ++i) acc[i] = xr[lane + 32 * i];
  }
#pragma unroll
  for (int i = 0; i < VEC; ++i)
    s_rows[k * (D / 4) + lane + 32 * i] = make_float4(v[i].x * ss, v[i].y * ss, v[i].z * ss, v[i].w * ss);
  // new sizes: unmerged A tokens keep theirs, B tokens add their sources' (rank order)
  for (int o = threadIdx.x; o < tp; o += blockDim.x) {
    float stot;
    if (o < n_unm) {
      const int tok = 2 * unm[static_cast<long long>(b) * n_unm + o];
      stot = size != nullptr ? size[static_cast<long long>(b) * t + tok] : 1.0f;
    } else {
      const int jj = o - n_unm;
      stot = size != nullptr ? size[static_cast<long long>(b) * t + 2 * jj + 1] : 1.0f;
      for (int q = 0; q < r; ++q)
        if (s_dst[q] == jj) stot += s_ssz[q];
    }
    size_out[static_cast<long long>(b) * tp + o] = stot;
  }
  __syncthreads();  // every source row staged
  if (!first) return;
  float stot = s_d;
#pragma unroll
  for (int i = 0; i < VEC; ++i) acc[i] = make_float4(acc[i].x * s_d, acc[i].y * s_d, acc[i].z * s_d, acc[i].w * s_d);
  for (int q = k; q < r; ++q) {
    if (s_dst[q] != j) continue;
#pragma unroll
    for (int i = 0; i < VEC; ++i) {
      const float4 w = s_rows[q * (D / 4) + lane + 32 * i];
      acc[i].x += w.x;
      acc[i].y += w.y;
      acc[i].z += w.z;
      acc[i].w += w.w;
    }
    stot += s_ssz[q];
  }
  float sum = 0.f, q2 = 0.f;
  float4* xr = reinterpret_cast<float4*>(x_out + orow * D);
#pragma unroll
  for (int i = 0; i < VEC; ++i) {
    acc[i].x /= stot;
    acc[i].y /= stot;
    acc[i].z /= stot;
    acc[i].w /= stot;
    sum += (acc[i].x + acc[i].y) + (acc[i].z + acc[i].w);
    q2 += (acc[i].x * acc[i].x + acc[i].y * acc[i].y) + (acc[i].z * acc[i].z + acc[i].w * acc[i].w);
    xr[lane + 32 * i] = acc[i];
    uint2 p;
    p.x = pack_bf16(acc[i].x, acc[i].y);
    p.y = pack_bf16(acc[i].z, acc[i].w);
    *reinterpret_cast<uint2*>(xh + orow * D + 4 * (lane + 32 * i)) = p;
  }
  const float s_all = warp_sum(sum), q_all = warp_sum(q2);
  if (lane < VEC)  // whole-row sums in slot 0, the other 128-column slots zero
    *reinterpret_cast<float2*>(stats + 2 * (orow * VEC + lane)) =
        lane == 0 ? make_float2(s_all, q_all) : make_float2(0.f, 0.f);
}

static cudaLaunchConfig_t pdl_cfg(dim3 grid, cudaStream_t s, cudaLaunchAttribute* attr) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = dim3(256);
  cfg.stream = s;
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled();
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cfg;
}

int merge_map(const int32_t* src, const int32_t* unm, int B, int t, int r, int32_t* row_map,
              cudaStream_t s) {
  if (r <= 0 || r > (t + 1) / 2 - 1) return TA_ERR_INVALID;
  cudaLaunchAttribute attr[1];
  const cudaLaunchConfig_t cfg = pdl_cfg(dim3(B), s, attr);
  const cudaError_t e = cudaLaunchKernelEx(&cfg, merge_map_kernel, src, unm, t, r, row_map);
  return e == cudaSuccess ? TA_OK : set_last_cuda_error(e);
}

static int fixup_backend() {  // profiling: TA_FIXUP=chain keeps the per-source-chain kernel
  static int mode = -1;
  if (mode < 0) {
    const char* v = getenv("TA_FIXUP");
    mode = (v && v[0] == 'c') ? 1 : 0;
  }
  return mode;
}

int merge_fixup(float* x_out, const float* side, const float* size, float* size_out, int B, int t,
                int D, int r, const int32_t* src, const int32_t* dst, const int32_t* unm, void* xh,
                float* stats, cudaStream_t s) {
  if (r <= 0 || r > (t + 1) / 2 - 1 || r > 256 || t > 1024) return TA_ERR_INVALID;
  if (r <= 32 && fixup_backend() == 0) {
    cudaLaunchAttribute attr[1];
    cudaLaunchConfig_t cfg = pdl_cfg(dim3(B), s, attr);
    cfg.blockDim = dim3(32 * r);
    cfg.dynamicSmemBytes = static_cast<size_t>(r) * D * sizeof(float);
    auto* h = static_cast<__nv_bfloat16*>(xh);
    cudaError_t e;
    switch (D) {
#define TA_FIXUP_PAR_CASE(DIM, V)                                                                       \
  case DIM: {                                                                                           \
    static unsigned long long attr_mask = 0;                                                            \
    if (attr_needed(attr_mask)) {                                                                       \
      e = cudaFuncSetAttribute(merge_fixup_par_kernel<V>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                               32 * DIM * 4);                                                           \
      if (e != cudaSuccess) return set_last_cuda_error(e);                                              \
      attr_done(attr_mask);                                                                             \
    }                                                                                                   \
    e = cudaLaunchKernelEx(&cfg, merge_fixup_par_kernel<V>, x_out, side, size, size_out, t, r, src, dst, \
                           unm, h, stats);                                                              \
    break;                                                                                              \
  }
      TA_FIXUP_PAR_CASE(256, 2)
      TA_FIXUP_PAR_CASE(768, 6)
      TA_FIXUP_PAR_CASE(1024, 8)
      TA_FIXUP_PAR_CASE(1280, 10)
#undef TA_FIXUP_PAR_CASE
      default:
        return TA_ERR_SHAPE;
    }
    return e == cudaSuccess ? TA_OK : set_last_cuda_error(e);
  }
  cudaLaunchAttribute attr[1];
  const cudaLaunchConfig_t cfg = pdl_cfg(dim3(B, (r + 7) / 8), s, attr);
  auto* h = static_cast<__nv_bfloat16*>(xh);
  cudaError_t e;
  switch (D) {
#define TA_FIXUP_CASE(DIM, V)                                                                   \
  case DIM:                                                                                     \
    e = cudaLaunchKernelEx(&cfg, merge_fixup_kernel<V>, x_out, side, size, size_out, t, r, src, \
                           dst, unm, h, stats);                                                 \
    break;
    TA_FIXUP_CASE(256, 2)
    TA_FIXUP_CASE(768, 6)
    TA_FIXUP_CASE(1024, 8)
    TA_FIXUP_CASE(1280, 10)
#undef TA_FIXUP_CASE
    default:
      return TA_ERR_SHAPE;
  }
  return e == cudaSuccess ? TA_OK : set_last_cuda_error(e);
}

int merge(const float* x, const float* size, int B, int t, int D, int r, const int32_t* src,
          const int32_t* dst, const int32_t* unm, const float* ln_w, const float* ln_b,
          float* x_out, float* size_out, void* h_out, int h_dtype, cudaStream_t s,
          float* stats_out) {
  if (stats_out != nullptr && h_dtype != TA_DTYPE_BF16) return TA_ERR_INVALID;
  if (r <= 0 || r > (t + 1) / 2 - 1 || r > 256) return TA_ERR_INVALID;
  if (h_dtype == TA_DTYPE_BF16)
    return merge_dispatch(x, size, B, t, D, r, src, dst, unm, ln_w, ln_b, x_out, size_out,
                          static_cast<__nv_bfloat16*>(h_out), stats_out, s);
  return merge_dispatch(x, size, B, t, D, r, src, dst, unm, ln_w, ln_b, x_out, size_out,
                        static_cast<float*>(h_out), stats_out, s);
}

}  // namespace ta
