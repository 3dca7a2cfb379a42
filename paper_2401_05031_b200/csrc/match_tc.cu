// Bipartite soft matching on the tensor cores (north_star 1).
//
//   match_fused_kernel   one CTA per image: metric = mean over heads of k (fixed head order),
//                        x / ||x||_2, 3xTF32 split x = hi + lo (hi = x truncated to tf32, lo =
//                        x - hi) for the alternating sets A = even tokens (cls first) and B =
//                        odd tokens, written straight into SW128 K-major smem tiles; one thread
//                        issues S = A_hi B_hi^T + A_hi B_lo^T + A_lo B_hi^T as tcgen05.mma
//                        kind::tf32 (M = N = 128, K = 8) into TMEM; thread i owns A row i (TMEM
//                        lane i) and takes its max / argmax over the B columns straight from
//                        tcgen05.ld registers (ties -> lowest column; row 0 is the class token
//                        -> -inf); top-r by rank counting rank_i = #{j : v_j > v_i or (v_j ==
//                        v_i and j < i)} (stable descending order), unm = remaining rows
//                        ascending.  (k is read once; no global scratch round trip.)
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

constexpr int kFusedThreads = 512;

#ifdef TA_MATCH_TRACE  // profiling build only: phase timestamps (globaltimer) of every CTA
__device__ unsigned long long g_match_trace[4096][6];
#define MTRACE(k)                                                                    \
  do {                                                                               \
    if (threadIdx.x == 0 && blockIdx.x < 4096) {                                     \
      unsigned long long t_;                                                         \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                         \
      g_match_trace[blockIdx.x][k] = t_;                                             \
    }                                                                                \
  } while (0)
#else
#define MTRACE(k) do {} while (0)
#endif

// One CTA per image, 16 warps.  Phase 1 (all warps): metric row of every token (mean over
// heads of k in fixed head order, or the given fp32 metric), x / ||x||_2, 3xTF32 split
// x = hi + lo, written straight into the four SW128 K-major smem tiles the MMA reads (A_hi,
// A_lo, B_hi, B_lo: 128 rows x cp floats, 32-float chunks of 128-byte rows, 16-byte chunk c of
// row i at slot c ^ (i & 7)); pad columns c..cp are zero.  Rows past a set's size are never
// read by the selection (their S rows / columns are masked), so they are not cleared.
// Phase 2 (thread 0): S = A_hi B_hi^T + A_hi B_lo^T + A_lo B_hi^T, kind::tf32 into TMEM.
// Phase 3 (warps 0..3, thread i = A row i = TMEM lane i): max / argmax over the B columns
// (ties -> lowest column; the class token row is -inf), top-r by rank counting, unm ascending.
// kTerms = 3: S in 3xTF32 (fp32 mode: the oracle's decisions bit for bit); kTerms = 1: one
// TF32 product (bf16 mode, where k itself is bf16: TF32's 2^-11 on the scores is below the
// input's rounding), two smem tiles instead of four, 256 threads, two CTAs per SM so one
// image's metric loads overlap another's MMA and selection.
template <typename QT, int kU, int kTerms, int kThreads>  // kU: 64-column passes per row (1: c <= 64, 2: c <= 128)
__global__ void __launch_bounds__(kThreads, kThreads == 256 ? 2 : 1)
    match_fused_kernel(const float* __restrict__ metric, const QT* __restrict__ qkv, int t,
                       int heads, int c, int cp, int r, int32_t* __restrict__ src_out,
                       int32_t* __restrict__ dst_out, int32_t* __restrict__ unm_out,
                       int32_t* __restrict__ row_map) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  const int b = blockIdx.x;
  const int na = (t + 1) / 2, nb = t / 2;
  const int nkc = cp / 32;                   // 32-float K chunks (128-byte swizzle rows)
  const int tile_bytes = nkc * kRows * 128;  // one part
  constexpr int kParts = kTerms == 3 ? 4 : 2;  // A_hi (A_lo) B_hi (B_lo)
  constexpr int kBPart = kTerms == 3 ? 2 : 1;
  float* node_max = reinterpret_cast<float*>(smem + kParts * tile_bytes);
  int* node_idx = reinterpret_cast<int*>(node_max + 2 * kRows);
  int* rank = node_idx + 2 * kRows;
  uint64_t* bar_mma = reinterpret_cast<uint64_t*>(rank + 2 * kRows);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar_mma + 1);
  const int tid = threadIdx.x;
  const uint32_t warp = warp_id(), lane = lane_id();
  const uint32_t s0 = smem_u32(smem);

  MTRACE(0);
  if (tid == 0) {
    mbar_init(bar_mma, 1);
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc<128>(tmem_slot);
  grid_dep_wait();    // qkv comes from the previous kernels
  grid_dep_launch();  // early trigger: the next kernel's prologue overlaps our tail
  MTRACE(1);

  // ---- phase 1: metric rows -> normalised, split, swizzled smem tiles
  const long long D = static_cast<long long>(heads) * c;
  // Smem row of token tok: B = odd tokens at row tok / 2; A = even tokens without the class
  // token (its S row is -inf by definition) at row tok / 2 - 1, so na <= 129 (t <= 257) fits
  // the M = 128 MMA.
  auto smem_row = [](int tok) { return (tok & 1) ? (tok >> 1) : (tok >> 1) - 1; };
  if constexpr (sizeof(QT) == 2) {
    if (metric == nullptr) {
      // bf16 k: rows in lane segments of kSeg lanes, 8 columns (16 bytes) per lane and head
      // (c = 64: 8 lanes, 4 rows per warp; c = 80: 10 of 16 lanes, 2 rows per warp); kPP row
      // groups per iteration with every head's load issued before the head-order sums.
      constexpr int kSeg = kU == 1 ? 8 : 16;
      constexpr int kRowsPerWarp = 32 / kSeg;
      constexpr int kPP = 1;  // (2 row groups in flight spill at 16 heads x 16 bytes)
      const int seg = static_cast<int>(lane) / kSeg, sl = static_cast<int>(lane) % kSeg;
      const int j = 8 * sl;  // first column of this lane
      // bf16 path: reciprocal multiplies instead of IEEE divisions (the fp32 path below keeps
      // the oracle's exact mean / norm divisions)
      const float inv_heads = 1.f / static_cast<float>(heads);
      constexpr int kStep = kRowsPerWarp * (kThreads / 32);
      for (int t0 = static_cast<int>(warp) * kRowsPerWarp; t0 < t; t0 += kPP * kStep) {
        uint4 raw[kPP][16];
#pragma unroll
        for (int pp = 0; pp < kPP; ++pp) {
          const int tok = t0 + pp * kStep + seg;
          if (tok < t && j < c) {
            const QT* kr = qkv + (static_cast<long long>(b) * t + tok) * 3 * D + D + j;
#pragma unroll
            for (int hh = 0; hh < 16; ++hh)
              if (hh < heads) raw[pp][hh] = __ldg(reinterpret_cast<const uint4*>(kr + hh * c));
          }
        }
#pragma unroll
        for (int pp = 0; pp < kPP; ++pp) {
          const int tok = t0 + pp * kStep + seg;
          float a[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
          if (tok < t && j < c) {
#pragma unroll
            for (int hh = 0; hh < 16; ++hh) {
              if (hh < heads) {
                const uint32_t w4[4] = {raw[pp][hh].x, raw[pp][hh].y, raw[pp][hh].z, raw[pp][hh].w};
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                  const float2 f = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&w4[e]));
                  a[2 * e] += f.x;
                  a[2 * e + 1] += f.y;
                }
              }
            }
          }
          float ss = 0.f;
#pragma unroll
          for (int e = 0; e < 8; ++e) {
            a[e] *= inv_heads;
            ss += a[e] * a[e];
          }
#pragma unroll
          for (int o = kSeg / 2; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
          const float inv_nrm = rsqrtf(ss);
          if (tok < t && tok > 0 && j < cp) {
            const int ri = smem_row(tok);
            const uint32_t row_hi = s0 + ((tok & 1) * kBPart) * tile_bytes + ri * 128;
            float hv[8], lv[8];
#pragma unroll
            for (int e = 0; e < 8; ++e) {
              const float x = j + e < c ? a[e] * inv_nrm : 0.f;
              hv[e] = tf32_trunc(x);
              lv[e] = tf32_trunc(x - hv[e]);
            }
            const int kc = j >> 5, jj = j & 31;
#pragma unroll
            for (int h2 = 0; h2 < 2; ++h2) {
              const uint32_t off = kc * kRows * 128 + ((((jj >> 2) + h2) ^ (ri & 7)) << 4);
              sts_f4(row_hi + off, make_float4(hv[4 * h2], hv[4 * h2 + 1], hv[4 * h2 + 2], hv[4 * h2 + 3]));
              if constexpr (kTerms == 3)
                sts_f4(row_hi + tile_bytes + off, make_float4(lv[4 * h2], lv[4 * h2 + 1], lv[4 * h2 + 2], lv[4 * h2 + 3]));
            }
          }
        }
      }
    }
  }
  if (sizeof(QT) == 4 || metric != nullptr) {
    for (int tok = static_cast<int>(warp); tok < t; tok += kThreads / 32) {
      float v[2][2] = {{0.f, 0.f}, {0.f, 0.f}};
      float ss = 0.f;
  #pragma unroll
      for (int u = 0; u < 2; ++u) {
        const int j = 2 * static_cast<int>(lane) + 64 * u;  // columns j, j + 1 (c is even)
        if (j < c) {
          if (metric != nullptr) {
            const float2 m2 = *reinterpret_cast<const float2*>(metric + (static_cast<long long>(b) * t + tok) * c + j);
            v[u][0] = m2.x;
            v[u][1] = m2.y;
          } else {
            const QT* kr = qkv + (static_cast<long long>(b) * t + tok) * 3 * D + D + j;
            float2 kv[16];
  #pragma unroll
            for (int hh = 0; hh < 16; ++hh) {
              if (hh < heads) {
                if constexpr (sizeof(QT) == 2)
                  kv[hh] = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(kr + hh * c));
                else
                  kv[hh] = *reinterpret_cast<const float2*>(kr + hh * c);
              }
            }
            float a0 = 0.f, a1 = 0.f;
  #pragma unroll
            for (int hh = 0; hh < 16; ++hh) {
              if (hh < heads) {
                a0 += kv[hh].x;
                a1 += kv[hh].y;
              }
            }
            v[u][0] = a0 / heads;
            v[u][1] = a1 / heads;
          }
        }
        ss += v[u][0] * v[u][0] + v[u][1] * v[u][1];
      }
      const float nrm = sqrtf(warp_sum(ss));
      if (tok == 0) continue;  // the class token never enters the MMA (its S row is -inf)
      const int set = tok & 1, ri = smem_row(tok);
      const uint32_t row_hi = s0 + (set * kBPart) * tile_bytes + ri * 128;
  #pragma unroll
      for (int u = 0; u < 2; ++u) {
        const int j = 2 * static_cast<int>(lane) + 64 * u;
        if (j < cp) {
          const float x0 = j < c ? v[u][0] / nrm : 0.f;
          const float x1 = j < c ? v[u][1] / nrm : 0.f;
          const float h0 = tf32_trunc(x0), h1 = tf32_trunc(x1);
          const float l0 = tf32_trunc(x0 - h0), l1 = tf32_trunc(x1 - h1);
          const int kc = j >> 5, jj = j & 31;
          const uint32_t off = kc * kRows * 128 + ((((jj >> 2) ^ (ri & 7))) << 4) + (jj & 3) * 4;
          asm volatile("st.shared.v2.f32 [%0], {%1, %2};" ::"r"(row_hi + off), "f"(h0), "f"(h1) : "memory");
          if constexpr (kTerms == 3)
            asm volatile("st.shared.v2.f32 [%0], {%1, %2};" ::"r"(row_hi + tile_bytes + off), "f"(l0), "f"(l1) : "memory");
        }
      }
    }
  }
  fence_proxy_async_shared();  // generic-proxy tile writes -> visible to the MMA (async proxy)
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  MTRACE(2);
  const uint32_t tmem = *tmem_slot;

  // ---- phase 2: S = A B^T in 3xTF32
  if (tid == 0) {
    constexpr uint32_t idesc = idesc_tf32(kRows, kRows);
    // (A part, B part): hi*hi, hi*lo, lo*hi
    const int terms[3][2] = {{0, kBPart}, {0, 3}, {1, 2}};
    int n = 0;
    for (int tt = 0; tt < kTerms; ++tt) {
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
  if (warp < 4) {
    const int i = tid;
    __syncwarp();
    mbar_wait(bar_mma, 0);
    tc_fence_after();
    // ---- phase 3: row max / argmax of S[i, 0..nb) from TMEM: thread i = TMEM lane i = A
    // row i + 1 (the class token, A row 0, is not in the MMA and gets -inf below)
    float best = -INFINITY;
    int best_j = 0;
    const uint32_t la = tmem + ((warp * 32u) << 16);
    for (int c0 = 0; c0 < kRows; c0 += 32) {
      uint32_t v[32];
      tmem_ld_32x32b_x32(la + c0, v);
      tmem_ld_wait();
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        const float sv = __uint_as_float(v[j]);
        if (c0 + j < nb && sv > best) {  // ascending j, strict >: lowest column on ties
          best = sv;
          best_j = c0 + j;
        }
      }
    }
    if (i + 1 < na) {
      node_max[i + 1] = best;
      node_idx[i + 1] = best_j;
    }
    if (i == 0) {
      node_max[0] = -INFINITY;
      node_idx[0] = 0;
    }
  }
  tc_fence_before();
  __syncthreads();
  MTRACE(3);
  if (tid < na) {
    const int i = tid;
    const float vi = node_max[i];
    int rk = 0;
    for (int j = 0; j < na; ++j) {
      const float vj = node_max[j];
      rk += (vj > vi) || (vj == vi && j < i);
    }
    rank[i] = rk;
  }
  __syncthreads();
  if (tid < na) {
    const int i = tid;
    const int rk = rank[i];
    if (rk < r) {
      src_out[static_cast<long long>(b) * r + rk] = i;
      dst_out[static_cast<long long>(b) * r + rk] = node_idx[i];
    } else {
      int pos = 0;
      for (int j = 0; j < i; ++j) pos += rank[j] >= r;
      unm_out[static_cast<long long>(b) * (na - r) + pos] = i;
      if (row_map != nullptr) row_map[static_cast<long long>(b) * t + 2 * i] = b * (t - r) + pos;
    }
    // fused merge (merge_map semantics, tome.cu): merged-away A token -> source row
    // B (t - r) + b r + rank, after the layer's merged rows
    if (row_map != nullptr && rk < r)
      row_map[static_cast<long long>(b) * t + 2 * i] = static_cast<int>(gridDim.x) * (t - r) + b * r + rk;
  }
  if (row_map != nullptr)  // B token j -> after the unmerged A tokens
    for (int j = tid; j < nb; j += kThreads)
      row_map[static_cast<long long>(b) * t + 2 * j + 1] = b * (t - r) + (na - r) + j;
  __syncthreads();
  MTRACE(4);
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc<128>(tmem);
  }
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
  attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled();
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, args...);
}

}  // namespace

// The fused kernel needs no global scratch; a non-null scratch pointer only selects the
// tensor-core path in match() (tome.cu), so a token allocation is kept in the workspace.
size_t match_tc_scratch_bytes(int, int) { return 256; }

// Returns TA_ERR_SHAPE outside the kernel's envelope (t > 257, c > 96 or > 16 heads).
int match_tc(const float* metric, const void* qkv, int qkv_dtype, int B, int t, int heads, int c,
             int r, int32_t* src, int32_t* dst, int32_t* unm, float* scratch, cudaStream_t s,
             int32_t* row_map) {
  (void)scratch;
  const int na = (t + 1) / 2;
  if (r <= 0 || r > na - 1 || t < 3) return TA_ERR_INVALID;
  if (t > 2 * kRows + 1 || c > 96 || c % 8 || heads > 16) return TA_ERR_SHAPE;
  const int cp = (c + 31) / 32 * 32;
  const size_t tiles = static_cast<size_t>(cp / 32) * kRows * 128;
  const size_t tail = 3 * 2 * kRows * 4 + 64 + 1024;
  const size_t smem3 = 4 * tiles + tail, smem1 = 2 * tiles + tail;
  static unsigned long long attr_mask = 0;  // per device
  cudaError_t e;
  if (attr_needed(attr_mask)) {
    e = cudaFuncSetAttribute(match_fused_kernel<float, 2, 3, kFusedThreads>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(match_fused_kernel<__nv_bfloat16, 1, 1, 256>,
                               cudaFuncAttributeMaxDynamicSharedMemorySize, 113 * 1024);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(match_fused_kernel<__nv_bfloat16, 2, 1, 256>,
                               cudaFuncAttributeMaxDynamicSharedMemorySize, 113 * 1024);
    if (e != cudaSuccess) return set_last_cuda_error(e);
    attr_done(attr_mask);
  }
  if (metric != nullptr || qkv_dtype == TA_DTYPE_F32)
    e = launch_pdl(match_fused_kernel<float, 2, 3, kFusedThreads>, dim3(B), dim3(kFusedThreads), smem3, s,
                   metric, static_cast<const float*>(qkv), t, heads, c, cp, r, src, dst, unm, row_map);
  else if (c <= 64)
    e = launch_pdl(match_fused_kernel<__nv_bfloat16, 1, 1, 256>, dim3(B), dim3(256), smem1, s, metric,
                   static_cast<const __nv_bfloat16*>(qkv), t, heads, c, cp, r, src, dst, unm, row_map);
  else
    e = launch_pdl(match_fused_kernel<__nv_bfloat16, 2, 1, 256>, dim3(B), dim3(256), smem1, s, metric,
                   static_cast<const __nv_bfloat16*>(qkv), t, heads, c, cp, r, src, dst, unm, row_map);
  return e == cudaSuccess ? TA_OK : set_last_cuda_error(e);
}

#ifdef TA_MATCH_TRACE
extern "C" __attribute__((visibility("default"))) int ta_debug_match_trace(unsigned long long* out, int n) {
  cudaDeviceSynchronize();
  return cudaMemcpyFromSymbol(out, g_match_trace, static_cast<size_t>(n) * 6 * sizeof(unsigned long long)) == cudaSuccess ? 0 : -1;
}
#endif
}  // namespace ta
