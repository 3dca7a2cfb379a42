// Bipartite soft matching on the tensor cores (north_star 1).
//
//   metric_split_kernel  metric = mean over heads of k (fixed head order), x / ||x||_2, then a
//                        3xTF32 split x = hi + lo (hi = x truncated to tf32, lo = x - hi) for the
//                        alternating sets A = even tokens (cls first) and B = odd tokens.
//                        Layout: scratch[b][part][128][cp] fp32, part = A_hi, A_lo, B_hi, B_lo,
//                        rows past the set size and columns past c are zero.
//   match_tc_kernel      TMA loads the four 128 x cp tiles (SW128, K-major, 32-float boxes),
//                        one thread issues S = A_hi B_hi^T + A_hi B_lo^T + A_lo B_hi^T as
//                        tcgen05.mma kind::tf32 (M = N = 128, K = 8) into TMEM; thread i owns
//                        A row i (TMEM lane i) and takes its max / argmax over the B columns
//                        straight from tcgen05.ld registers (ties -> lowest column; row 0 is
//                        the class token -> -inf); top-r by rank counting
//                        rank_i = #{j : v_j > v_i or (v_j == v_i and j < i)} (stable descending
//                        order), unm = remaining rows ascending.
// The 3xTF32 contraction is accurate to ~1e-6 relative, the level of an fp32 dot product.
#include <cfloat>

#include <cudaTypedefs.h>

#include "common.h"
#include "ptx.cuh"

namespace ta {

namespace {

constexpr int kRows = 128;

__device__ __forceinline__ float tf32_trunc(float x) {
  return __uint_as_float(__float_as_uint(x) & 0xFFFFE000u);
}

// grid (B, 8), block 256: one warp per token row, 32 rows per CTA.  Each lane owns column
// pairs (2 lane, 2 lane + 1) (+64): all heads' k values are loaded before the sum, in head
// order, so the fixed summation order of the SIMT kernel is kept.
template <typename QT>
__global__ void __launch_bounds__(256)
    metric_split_kernel(const float* __restrict__ metric, const QT* __restrict__ qkv, int t,
                        int heads, int c, int cp, float* __restrict__ scratch) {
  const int b = blockIdx.x;
  const int na = (t + 1) / 2, nb = t / 2;
  float* base = scratch + static_cast<long long>(b) * 4 * kRows * cp;
  grid_dep_wait();
  grid_dep_launch();  // early trigger: the next kernel's prologue overlaps our tail
  const int lane = lane_id();
  const int row = blockIdx.y * 32 + warp_id() * 4;
  for (int rr = row; rr < row + 4; ++rr) {
    const int set = rr / kRows;  // 0 = A (even tokens), 1 = B (odd tokens)
    const int ri = rr % kRows;
    const int tok = 2 * ri + set;
    const bool valid = ri < (set ? nb : na);
    float* hi = base + (static_cast<long long>(set * 2) * kRows + ri) * cp;
    float* lo = hi + static_cast<long long>(kRows) * cp;
    float v[2][2] = {{0.f, 0.f}, {0.f, 0.f}};
    float ss = 0.f;
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int j = 2 * lane + 64 * u;  // columns j, j + 1 (c is even)
      if (valid && j < c) {
        if (metric != nullptr) {
          const float2 m2 = *reinterpret_cast<const float2*>(
              metric + (static_cast<long long>(b) * t + tok) * c + j);
          v[u][0] = m2.x;
          v[u][1] = m2.y;
        } else {
          const long long D = static_cast<long long>(heads) * c;
          const QT* kr = qkv + (static_cast<long long>(b) * t + tok) * 3 * D + D + j;
          float2 kv[16];
#pragma unroll
          for (int h = 0; h < 16; ++h) {
            if (h < heads) {
              if constexpr (sizeof(QT) == 2)
                kv[h] = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(kr + h * c));
              else
                kv[h] = *reinterpret_cast<const float2*>(kr + h * c);
            }
          }
          float a0 = 0.f, a1 = 0.f;
#pragma unroll
          for (int h = 0; h < 16; ++h) {
            if (h < heads) {
              a0 += kv[h].x;
              a1 += kv[h].y;
            }
          }
          v[u][0] = a0 / heads;
          v[u][1] = a1 / heads;
        }
      }
      ss += v[u][0] * v[u][0] + v[u][1] * v[u][1];
    }
    const float nrm = sqrtf(warp_sum(ss));
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int j = 2 * lane + 64 * u;
      if (j < cp) {
        float2 h2, l2;
        const float x0 = valid ? v[u][0] / nrm : 0.f;
        const float x1 = valid ? v[u][1] / nrm : 0.f;
        h2.x = tf32_trunc(x0);
        h2.y = tf32_trunc(x1);
        l2.x = tf32_trunc(x0 - h2.x);
        l2.y = tf32_trunc(x1 - h2.y);
        *reinterpret_cast<float2*>(hi + j) = h2;
        *reinterpret_cast<float2*>(lo + j) = l2;
      }
    }
  }
}

__global__ void __launch_bounds__(128, 1)
    match_tc_kernel(const __grid_constant__ CUtensorMap tm, int t, int cp, int r,
                    int32_t* __restrict__ src_out, int32_t* __restrict__ dst_out,
                    int32_t* __restrict__ unm_out) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  const int b = blockIdx.x;
  const int na = (t + 1) / 2, nb = t / 2;
  const int nkc = cp / 32;                  // 32-float K chunks (128-byte swizzle rows)
  const int tile_bytes = nkc * kRows * 128;  // one part
  float* node_max = reinterpret_cast<float*>(smem + 4 * tile_bytes);
  int* node_idx = reinterpret_cast<int*>(node_max + kRows);
  int* rank = node_idx + kRows;
  uint64_t* bar_ld = reinterpret_cast<uint64_t*>(rank + kRows);
  uint64_t* bar_mma = bar_ld + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar_mma + 1);
  const int i = threadIdx.x;
  const uint32_t warp = warp_id();

  if (i == 0) {
    tma_prefetch(&tm);
    mbar_init(bar_ld, 1);
    mbar_init(bar_mma, 1);
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc<128>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  grid_dep_wait();  // scratch comes from metric_split_kernel
  grid_dep_launch();  // early trigger: the next kernel's prologue overlaps our tail

  if (i == 0) {
    mbar_arrive_expect_tx(bar_ld, 4 * tile_bytes);
    for (int part = 0; part < 4; ++part)
      for (int kc = 0; kc < nkc; ++kc)
        tma_load_2d(&tm, bar_ld, smem + part * tile_bytes + kc * kRows * 128, kc * 32,
                    (b * 4 + part) * kRows);
    mbar_wait(bar_ld, 0);
    tc_fence_after();
    constexpr uint32_t idesc = idesc_tf32(kRows, kRows);
    const uint32_t s0 = smem_u32(smem);
    // (A part, B part): hi*hi, hi*lo, lo*hi
    const int terms[3][2] = {{0, 2}, {0, 3}, {1, 2}};
    int n = 0;
    for (int tt = 0; tt < 3; ++tt) {
      for (int kc = 0; kc < nkc; ++kc) {
        const uint64_t ad = umma_desc_sw128(s0 + terms[tt][0] * tile_bytes + kc * kRows * 128);
        const uint64_t bd = umma_desc_sw128(s0 + terms[tt][1] * tile_bytes + kc * kRows * 128);
#pragma unroll
        for (int k = 0; k < 4; ++k, ++n)  // K = 8 tf32 = 32 bytes per instruction
          umma_tf32(tmem, ad + 2 * k, bd + 2 * k, idesc, n > 0);
      }
    }
    umma_commit(bar_mma);
  }
  __syncwarp();
  mbar_wait(bar_mma, 0);
  tc_fence_after();

  // row max / argmax of S[i, 0..nb) from TMEM (thread i = lane i)
  float best = -INFINITY;
  int best_j = 0;
  const uint32_t la = tmem + ((warp * 32u) << 16);
  for (int c0 = 0; c0 < kRows; c0 += 32) {
    uint32_t v[32];
    tmem_ld_32x32b_x32(la + c0, v);
    tmem_ld_wait();
    if (i > 0) {
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        const float s = __uint_as_float(v[j]);
        if (c0 + j < nb && s > best) {  // ascending j, strict >: lowest column on ties
          best = s;
          best_j = c0 + j;
        }
      }
    }
  }
  node_max[i] = i < na ? best : -INFINITY;
  node_idx[i] = best_j;
  tc_fence_before();
  __syncthreads();
  if (i < na) {
    const float vi = node_max[i];
    int rk = 0;
    for (int j = 0; j < na; ++j) {
      const float vj = node_max[j];
      rk += (vj > vi) || (vj == vi && j < i);
    }
    rank[i] = rk;
  }
  __syncthreads();
  if (i < na) {
    const int rk = rank[i];
    if (rk < r) {
      src_out[static_cast<long long>(b) * r + rk] = i;
      dst_out[static_cast<long long>(b) * r + rk] = node_idx[i];
    } else {
      int pos = 0;
      for (int j = 0; j < i; ++j) pos += rank[j] >= r;
      unm_out[static_cast<long long>(b) * (na - r) + pos] = i;
    }
  }
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc<128>(tmem);
  }
}

int make_tmap_f32_2d(CUtensorMap* map, const void* base, uint64_t rows, uint64_t cols,
                     uint32_t box_cols, uint32_t box_rows) {
  static PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
  if (!enc) {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) !=
            cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return TA_ERR_CUDA;
    enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {cols * 4};
  cuuint32_t box[2] = {box_cols, box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult res = enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void*>(base), dims, strides,
                     box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return res == CUDA_SUCCESS ? TA_OK : TA_ERR_SHAPE;
}

template <typename... Args>
cudaError_t launch_pdl(void (*kern)(Args...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                       Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, args...);
}

}  // namespace

size_t match_tc_scratch_bytes(int B, int c) {
  const int cp = (c + 31) / 32 * 32;
  return static_cast<size_t>(B) * 4 * kRows * cp * sizeof(float);
}

// Returns TA_ERR_SHAPE outside the kernel's envelope (t > 256 or c > 96).
int match_tc(const float* metric, const void* qkv, int qkv_dtype, int B, int t, int heads, int c,
             int r, int32_t* src, int32_t* dst, int32_t* unm, float* scratch, cudaStream_t s) {
  const int na = (t + 1) / 2;
  if (r <= 0 || r > na - 1 || t < 3) return TA_ERR_INVALID;
  if (t > 2 * kRows || c > 96 || (c & 1) || heads > 16 || scratch == nullptr) return TA_ERR_SHAPE;
  const int cp = (c + 31) / 32 * 32;
  cudaError_t e;
  if (metric != nullptr || qkv_dtype == TA_DTYPE_F32)
    e = launch_pdl(metric_split_kernel<float>, dim3(B, 2 * kRows / 32), dim3(256), 0, s, metric,
                   static_cast<const float*>(qkv), t, heads, c, cp, scratch);
  else
    e = launch_pdl(metric_split_kernel<__nv_bfloat16>, dim3(B, 2 * kRows / 32), dim3(256), 0, s, metric,
                   static_cast<const __nv_bfloat16*>(qkv), t, heads, c, cp, scratch);
  if (e != cudaSuccess) return set_last_cuda_error(e);
  CUtensorMap tm;
  int rc = make_tmap_f32_2d(&tm, scratch, static_cast<uint64_t>(B) * 4 * kRows, cp, 32, kRows);
  if (rc) return rc;
  const size_t smem = 4 * (cp / 32) * kRows * 128 + 3 * kRows * 4 + 64 + 1024;
  static bool attr_set = false;
  if (!attr_set) {
    e = cudaFuncSetAttribute(match_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    if (e != cudaSuccess) return set_last_cuda_error(e);
    attr_set = true;
  }
  e = launch_pdl(match_tc_kernel, dim3(B), dim3(128), smem, s, tm, t, cp, r, src, dst, unm);
  return e == cudaSuccess ? TA_OK : set_last_cuda_error(e);
}

}  // namespace ta
