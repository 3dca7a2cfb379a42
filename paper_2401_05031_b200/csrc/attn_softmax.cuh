// Softmax building blocks shared by the tcgen05 attention kernels (attention_tc.cu,
// attention_fa.cu): packed-fp32x2 exponentials split between the SFU and the FMA pipe, bf16 P
// rows in the SW128 K-major layout the PV MMA reads, and the O slab TMA store.
#pragma once
#include <cstdint>

#include <cuda.h>

#include "ptx.cuh"

namespace ta {
namespace {

__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void named_bar_sync(int id, int threads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(threads) : "memory");
}

// Exponentials per 8-key chunk evaluated by exp2_poly2 on the FMA pipe (in pairs) for even /
// odd chunks; the rest go to the SFU.  The SFU issues 16 ex2/clk/SM against 128 FMA lanes,
// so with ~4.5 other instructions per key an all-SFU softmax is SFU-bound; 3 of 8 on the
// FMA pipe balances the two (measured in tools/attn_bench.py).
#ifndef TA_ATTN_POLY_EVEN
#define TA_ATTN_POLY_EVEN 1
#endif
#ifndef TA_ATTN_POLY_ODD
#define TA_ATTN_POLY_ODD 2
#endif

// p = w * 2^(s * scale_log2 - m) for 8 keys of one query row; accumulates the fp32 row sum
// into acc (two packed pairs) and returns the bf16 P chunk.
template <int kPolyPairs>
__device__ __forceinline__ uint4 softmax_chunk8(const uint32_t* rr, uint64_t sc2, uint64_t nm2,
                                                bool weighted, uint32_t s_w, uint64_t (&acc)[2]) {
  uint64_t p[4];
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    const uint64_t x = ffma2(f2_pack(__uint_as_float(rr[2 * e]), __uint_as_float(rr[2 * e + 1])), sc2, nm2);
#ifdef TA_ATTN_EXP_NONE  // profiling only: wrong results
    if (true) {
      p[e] = x;
#else
    if (e >= 4 - kPolyPairs) {
      p[e] = exp2_poly2(x);
#endif
    } else {
      const float2 v = f2_unpack(x);
      p[e] = f2_pack(ex2_approx(v.x), ex2_approx(v.y));
    }
  }
  if (weighted) {
    const float4 w0 = lds_f4(s_w);
    const float4 w1 = lds_f4(s_w + 16);
    p[0] = fmul2(p[0], f2_pack(w0.x, w0.y));
    p[1] = fmul2(p[1], f2_pack(w0.z, w0.w));
    p[2] = fmul2(p[2], f2_pack(w1.x, w1.y));
    p[3] = fmul2(p[3], f2_pack(w1.z, w1.w));
  }
  acc[0] = fadd2(acc[0], p[0]);
  acc[1] = fadd2(acc[1], p[1]);
  acc[0] = fadd2(acc[0], p[2]);
  acc[1] = fadd2(acc[1], p[3]);
  const float2 a = f2_unpack(p[0]), b = f2_unpack(p[1]), c = f2_unpack(p[2]), d = f2_unpack(p[3]);
  return make_uint4(pack_bf16(a.x, a.y), pack_bf16(b.x, b.y), pack_bf16(c.x, c.y), pack_bf16(d.x, d.y));
}

// 64 keys (one P block row): chunk c -> 16-byte swizzled slot (c ^ (row & 7)) of the row.
__device__ __forceinline__ void softmax_block64(const uint32_t (&r)[64], uint64_t sc2, uint64_t nm2,
                                                bool weighted, uint32_t s_w, uint32_t s_prow,
                                                int row, uint64_t (&acc)[2]) {
#pragma unroll
  for (int chunk = 0; chunk < 8; ++chunk) {
    const uint4 v = (chunk & 1)
                        ? softmax_chunk8<TA_ATTN_POLY_ODD>(&r[chunk * 8], sc2, nm2, weighted, s_w + chunk * 32, acc)
                        : softmax_chunk8<TA_ATTN_POLY_EVEN>(&r[chunk * 8], sc2, nm2, weighted, s_w + chunk * 32, acc);
    sts_u4(s_prow + ((chunk ^ (row & 7)) << 4), v);
  }
}

// Last 64-key block: only its first nch chunks hold keys < t (8 nch <= t_mma - 64 kb); the
// chunks up to the PV MMA's K extent (2 nkc) are written as zeros, the rest are never read.
__device__ __forceinline__ void softmax_block_tail(const uint32_t (&r)[64], uint64_t sc2, uint64_t nm2,
                                                   uint32_t s_w, uint32_t s_prow, int row, int nch,
                                                   int nzero, uint64_t (&acc)[2]) {
#pragma unroll
  for (int chunk = 0; chunk < 8; ++chunk) {
    if (chunk >= nzero) break;
    uint4 v = make_uint4(0u, 0u, 0u, 0u);
    if (chunk < nch)
      v = (chunk & 1) ? softmax_chunk8<TA_ATTN_POLY_ODD>(&r[chunk * 8], sc2, nm2, true, s_w + chunk * 32, acc)
                      : softmax_chunk8<TA_ATTN_POLY_EVEN>(&r[chunk * 8], sc2, nm2, true, s_w + chunk * 32, acc);
    sts_u4(s_prow + ((chunk ^ (row & 7)) << 4), v);
  }
}

// Row max of the raw scores of one 64-key block over its first `valid` keys (the second
// 32-column half is not loaded when it holds no valid key).
__device__ __forceinline__ void block_max(uint32_t ta, int valid, float (&m4)[4]) {
  uint32_t r[64];
  tmem_ld_32x32b_x32(ta, *reinterpret_cast<uint32_t(*)[32]>(&r[0]));
  tmem_ld_32x32b_x32(ta + 32, *reinterpret_cast<uint32_t(*)[32]>(&r[32]));
  tmem_ld_wait();
  if (valid == 64) {
#pragma unroll
    for (int j = 0; j < 64; j += 4) {
      m4[0] = fmaxf(m4[0], __uint_as_float(r[j]));
      m4[1] = fmaxf(m4[1], __uint_as_float(r[j + 1]));
      m4[2] = fmaxf(m4[2], __uint_as_float(r[j + 2]));
      m4[3] = fmaxf(m4[3], __uint_as_float(r[j + 3]));
    }
  } else {
#pragma unroll
    for (int j = 0; j < 64; ++j)
      if (j < valid) m4[j & 3] = fmaxf(m4[j & 3], __uint_as_float(r[j]));
  }
}

__device__ __forceinline__ float f2_total(const uint64_t (&acc)[2]) {
  const float2 a = f2_unpack(acc[0]), b = f2_unpack(acc[1]);
  return (a.x + a.y) + (b.x + b.y);
}

// One warp's 32 query rows x 32 head columns of O / rowsum -> bf16 into a 2 KB smem slab
// (64-byte rows, SW64 chunk swizzle: conflict-free 16-byte stores), then one TMA store of the
// slab.  The [B][t][D] output map clips rows >= t, so tail rows need no predication.
__device__ __forceinline__ void store_o_slab(const CUtensorMap* tmo, const uint32_t* o, float inv,
                                             uint32_t slab, int lane, int col, int row, int b) {
#pragma unroll
  for (int c = 0; c < 4; ++c)
    sts_u4(slab + lane * 64 + ((c ^ ((lane >> 1) & 3)) << 4),
           make_uint4(pack_bf16(__uint_as_float(o[8 * c]) * inv, __uint_as_float(o[8 * c + 1]) * inv),
                      pack_bf16(__uint_as_float(o[8 * c + 2]) * inv, __uint_as_float(o[8 * c + 3]) * inv),
                      pack_bf16(__uint_as_float(o[8 * c + 4]) * inv, __uint_as_float(o[8 * c + 5]) * inv),
                      pack_bf16(__uint_as_float(o[8 * c + 6]) * inv, __uint_as_float(o[8 * c + 7]) * inv)));
  fence_proxy_async_shared();
  __syncwarp();
  if (lane == 0) {
    tma_store_3d_s(tmo, slab, col, row, b);
    bulk_commit_group();
  }
}


}  // namespace
}  // namespace ta
