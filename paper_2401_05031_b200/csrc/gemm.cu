// Linear layers of the token-adapted ViT:
//   C[m, n] = sum_k A[m, k] * W[n, k]  + fused epilogue (bias / GELU / residual / pos).
//
// bf16 path: persistent, warp-specialised tcgen05 kernel.
//   warp 0      TMA producer (one elected lane): A and W tiles -> SW128 smem ring
//   warp 1      MMA issuer (one lane): tcgen05.mma kind::f16 128 x BN x 16 into TMEM
//   warp 2      TMEM allocator
//   warps 4..7  epilogue: tcgen05.ld -> registers -> bias/GELU/residual -> HBM
// Two TMEM accumulator stages let the epilogue of tile i overlap the MMAs of tile i+1.
// The token count per layer varies with gamma, so M is a runtime value; rows past M are
// zero-filled by TMA and masked in the epilogue.
//
// fp32 path: SIMT FFMA tile kernel with the same epilogues, used by the fp32 parity
// mode (north_star: merge index sets bit-exact in fp32 mode).
#include <cstdio>
#include <cstdlib>
#include <mutex>

#include <cudaTypedefs.h>

#include "common.h"
#include "ptx.cuh"

namespace ta {

#define TA_TRY_GEMM(expr)     \
  do {                        \
    const int rc_ = (expr);   \
    if (rc_ != TA_OK) return rc_; \
  } while (0)

// ------------------------------------------------------------------ epilogue
// One epilogue warp owns TMEM lanes [32*q, 32*q + 32) (q = warp % 4) and a 128-column
// half of the 256-wide accumulator.  Per 32-column chunk: tcgen05.ld (thread = row) ->
// swizzled smem transpose -> each lane handles 4 consecutive columns of 8 rows, so bias,
// residual loads and output stores are coalesced 16-byte accesses along the row.
// The chunk loop is software-pipelined: chunk c+1's transpose and residual loads are
// issued before chunk c's stores (out may alias resid, but only element-for-element).
struct EpiChunk {
  float4 v[8];
  float4 x[8];  // residual / positional rows, added at store time so loads stay in flight
};

template <int EPI>
__device__ __forceinline__ void epi_load(const GemmEpi& e, int M, int N, long long m_base, int n0,
                                         const uint32_t (&r)[32], float4* stage, EpiChunk& c) {
  const uint32_t lane = lane_id();
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    float4 v = make_float4(__uint_as_float(r[4 * q]), __uint_as_float(r[4 * q + 1]),
                           __uint_as_float(r[4 * q + 2]), __uint_as_float(r[4 * q + 3]));
    sts_f4(smem_u32(stage) + 16u * (lane * 8 + (q ^ (lane & 7))), v);
  }
  __syncwarp();
  const int g = lane & 7;
  const int n = n0 + 4 * g;
  const int row0 = lane >> 3;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const int row = row0 + 4 * k;
    c.v[k] = lds_f4(smem_u32(stage) + 16u * (row * 8 + (g ^ (row & 7))));
  }
  __syncwarp();
  const bool full = m_base + 32 <= M;
  if constexpr (epi_is_resid(EPI)) {
    const float* rp = e.resid + (m_base + row0) * N + n;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      if (full || m_base + row0 + 4 * k < M) {
        c.x[k] = *reinterpret_cast<const float4*>(rp + static_cast<long long>(4 * k) * N);
      }
    }
  }
  if constexpr (epi_is_patch(EPI)) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const long long m = m_base + row0 + 4 * k;
      if (m < M) {
        c.x[k] =
            __ldg(reinterpret_cast<const float4*>(e.pos + (e.row_off + (m % e.rows_in)) * N + n));
      }
    }
  }
  if constexpr (epi_is_ln(EPI)) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const long long m = m_base + row0 + 4 * k;
      if (full || m < M) {
        const float2* sp = reinterpret_cast<const float2*>(e.ln_stats) + m * e.stat_slots;
        float2 st = __ldg(sp);
        for (int j = 1; j < e.stat_slots; ++j) {
          const float2 p = __ldg(sp + j);
          st.x += p.x;
          st.y += p.y;
        }
        c.x[k].x = st.x;
        c.x[k].y = st.y;
      }
    }
  }
}

// Per-row (sum, sumsq) partials of the values a warp stores, carried across the chunks of one
// 128-column block and stored into that block's slot (EPI_*_STATS).
struct RowStats {
  float s[8];
  float q[8];
};
__device__ __forceinline__ void rowstats_clear(RowStats& r) {
#pragma unroll
  for (int k = 0; k < 8; ++k) r.s[k] = r.q[k] = 0.f;
}
template <bool kRemap>
__device__ __forceinline__ void rowstats_flush(const GemmEpi& e, int M, long long m_base, RowStats& r,
                                               int slot) {
  const uint32_t lane = lane_id();
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    float s = r.s[k], q = r.q[k];
#pragma unroll
    for (int o = 1; o < 8; o <<= 1) {  // the 8 lanes holding one row
      s += __shfl_xor_sync(0xffffffffu, s, o);
      q += __shfl_xor_sync(0xffffffffu, q, o);
    }
    const long long m = m_base + (lane >> 3) + 4 * k;
    if ((lane & 7) == 0 && m < M) {
      const long long orow = kRemap ? epi_out_row(e, m) : m;
      *reinterpret_cast<float2*>(e.stats + 2 * (orow * e.stat_slots + slot)) = make_float2(s, q);
    }
  }
  rowstats_clear(r);
}

template <int EPI, typename OutT, bool kRemap>
__device__ __forceinline__ void epi_store(const GemmEpi& e, int M, int N, long long m_base, int n0,
                                          const EpiChunk& c, RowStats& rs) {
  const uint32_t lane = lane_id();
  const int n = n0 + 4 * (lane & 7);
  const int row0 = lane >> 3;
  float4 b, c1v;
  if constexpr (epi_is_ln(EPI)) {
    b = __ldg(reinterpret_cast<const float4*>(e.c2 + n));
    c1v = __ldg(reinterpret_cast<const float4*>(e.c1 + n));
  } else {
    b = __ldg(reinterpret_cast<const float4*>(e.bias + n));
  }
  const bool full = m_base + 32 <= M;
  OutT* obase = static_cast<OutT*>(e.out);
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const long long m = m_base + row0 + 4 * k;
    if (!full && m >= M) continue;
    float4 w = c.v[k];
    if constexpr (epi_is_ln(EPI)) {
      const float mu = c.x[k].x * e.inv_dim;
      const float var = fmaxf(c.x[k].y * e.inv_dim - mu * mu, 0.f);
      const float rstd = rsqrtf(var + 1e-6f);
      w.x = fmaf(rstd, fmaf(-mu, c1v.x, w.x), b.x);
      w.y = fmaf(rstd, fmaf(-mu, c1v.y, w.y), b.y);
      w.z = fmaf(rstd, fmaf(-mu, c1v.z, w.z), b.z);
      w.w = fmaf(rstd, fmaf(-mu, c1v.w, w.w), b.w);
    } else {
      w.x += b.x;
      w.y += b.y;
      w.z += b.z;
      w.w += b.w;
    }
    if constexpr (epi_is_resid(EPI) || epi_is_patch(EPI)) {
      w.x += c.x[k].x;
      w.y += c.x[k].y;
      w.z += c.x[k].z;
      w.w += c.x[k].w;
    }
    if constexpr (epi_is_gelu(EPI)) {
      w.x = gelu_erf_fast(w.x);
      w.y = gelu_erf_fast(w.y);
      w.z = gelu_erf_fast(w.z);
      w.w = gelu_erf_fast(w.w);
    }
    const long long orow = kRemap ? epi_out_row(e, m) : m;
    if constexpr (sizeof(OutT) == 2) {
      uint2 pk;
      pk.x = pack_bf16(w.x, w.y);
      pk.y = pack_bf16(w.z, w.w);
      *reinterpret_cast<uint2*>(obase + orow * N + n) = pk;
    } else {
      *reinterpret_cast<float4*>(obase + orow * N + n) = w;
    }
    if constexpr (epi_is_stats(EPI)) {
      uint2 pk;
      pk.x = pack_bf16(w.x, w.y);
      pk.y = pack_bf16(w.z, w.w);
      *reinterpret_cast<uint2*>(static_cast<__nv_bfloat16*>(e.xh) + orow * N + n) = pk;
      rs.s[k] += (w.x + w.y) + (w.z + w.w);
      rs.q[k] += (w.x * w.x + w.y * w.y) + (w.z * w.z + w.w * w.w);
    }
  }
}

// ------------------------------------------------------------------ tcgen05 kernel
constexpr int kBM = 128;
constexpr int kBK = 64;  // 64 bf16 = 128 B rows -> SWIZZLE_128B
constexpr int kEpiWarps = 8;  // max epilogue warps (transpose staging is sized for this)
// Epilogue warps per kind on the transposed-store path: the residual / patch / stats
// epilogues keep two 32x32 chunks plus residual rows in flight and need the registers of a
// 4-warp epilogue; the arithmetic-heavy ones (GELU, LN finish) use 8 warps.
__host__ __device__ constexpr int epi_warps(int e) {
  return (epi_is_resid(e) || epi_is_patch(e) || epi_is_stats(e)) ? 4 : 8;
}
__host__ __device__ constexpr int gemm_threads(int e) { return 128 + 32 * epi_warps(e); }
// The CTA-pair kernel's TMA-store epilogue (no remap / stats / LN) is register-light: 8 warps.
__host__ __device__ constexpr bool pair_tma(int e, bool remap) { return true; }
__host__ __device__ constexpr int pair_epi_warps(int e, bool remap) {
  return pair_tma(e, remap) ? 8 : epi_warps(e);
}

// kOp 0: bf16 operands (64 K per 128-byte row).  kOp 1: fp32 parity mode on the tensor cores,
// 3xTF32: every stage holds A_hi, A_lo, W_hi, W_lo (32 fp32 K per 128-byte row; x = hi + lo
// with hi = x truncated to tf32, split by split_tf32_kernel) and C = A_hi W_hi^T + A_hi W_lo^T
// + A_lo W_hi^T accumulates in fp32 in TMEM (kind::tf32; the dropped lo*lo term is ~2^-22
// relative, the same scheme as the fp32 bipartite match in match_tc.cu).
template <int BN, int kOp = 0>
struct GemmCfg {
  static constexpr int kParts = kOp ? 2 : 1;  // hi (+ lo) per operand
  static constexpr int kStages = kOp ? 3 : (BN == 256 ? 4 : 6);
  static constexpr int kABytes = kBM * kBK * 2;  // one 128 x 128-byte tile
  static constexpr int kBBytes = BN * kBK * 2;
  static constexpr int kStageBytes = kParts * (kABytes + kBBytes);
  static constexpr int kKPerStage = kOp ? kBK / 2 : kBK;  // 32 fp32 or 64 bf16 per 128-byte row
  // kOp 0: two accumulator stages.  kOp 1: two K-chunk buffers + the running total (below).
  static constexpr int kTmemCols = kOp ? 512 : 2 * BN;
  // kOp 1: the tensor core's fp32 accumulation truncates, so its error grows with the number of
  // MMAs summed into one accumulator (measured ~2e-5 relative at K = 768 in one accumulator).  The
  // MMAs of every 64-K chunk go into a fresh chunk buffer, and the epilogue warps add the chunks
  // into a running total in TMEM with round-to-nearest FADDs (error ~24 MMAs' worth per chunk).
  static constexpr int kChunkKb = 2;  // k-blocks (of 32 fp32) per chunk
  static constexpr int kEpiBytes = kEpiWarps * 32 * 32 * 4;  // per-warp 32x32 fp32 transpose
  static constexpr int kSmemBytes = kStages * kStageBytes + kEpiBytes + 1024 + 256;
};

template <int BN, int EPI, typename OutT, bool kRemap, int kOp = 0>
__global__ void __launch_bounds__(gemm_threads(EPI), 1)
    gemm_bf16_sm100_kernel(const __grid_constant__ CUtensorMap tmA,
                           const __grid_constant__ CUtensorMap tmB,
                           const __grid_constant__ CUtensorMap tmA2,
                           const __grid_constant__ CUtensorMap tmB2, int M, int N, int K,
                           GemmEpi epi) {
  using Cfg = GemmCfg<BN, kOp>;
  constexpr int S = Cfg::kStages;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  float4* epi_stage = reinterpret_cast<float4*>(smem + S * Cfg::kStageBytes);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + S * Cfg::kStageBytes + Cfg::kEpiBytes);
  uint64_t* empty = full + S;
  uint64_t* tfull = empty + S;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const uint32_t warp = warp_id();
  const uint32_t lane = lane_id();

  if (warp == 0 && lane == 0) {
    tma_prefetch(&tmA);
    tma_prefetch(&tmB);
    if constexpr (kOp) {
      tma_prefetch(&tmA2);
      tma_prefetch(&tmB2);
    }
  }
  if (warp == 1 && lane == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], epi_warps(EPI));  // one arrive per epilogue warp
    }
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc<Cfg::kTmemCols>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  // Inputs (A) may be produced by the previous kernel in the stream (PDL).
  grid_dep_wait();
  grid_dep_launch();  // early trigger: the next kernel's prologue overlaps our tail

  const int num_m = (M + kBM - 1) / kBM;
  const int num_n = N / BN;
  const int num_tiles = num_m * num_n;
  const int num_kb = K / Cfg::kKPerStage;

  if (warp == 0) {
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
        const int m_blk = tile / num_n;
        const int n_blk = tile - m_blk * num_n;
        for (int kb = 0; kb < num_kb; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          uint8_t* sa = smem + stage * Cfg::kStageBytes;
          uint8_t* sb = sa + Cfg::kABytes;
          mbar_arrive_expect_tx(&full[stage], Cfg::kStageBytes);
          const int kc = kb * Cfg::kKPerStage;
          tma_load_2d(&tmA, &full[stage], sa, kc, m_blk * kBM);
          tma_load_2d(&tmB, &full[stage], sb, kc, n_blk * BN);
          if constexpr (kOp) {  // stage = [A_hi][W_hi][A_lo][W_lo]
            tma_load_2d(&tmA2, &full[stage], sb + Cfg::kBBytes, kc, m_blk * kBM);
            tma_load_2d(&tmB2, &full[stage], sb + Cfg::kBBytes + Cfg::kABytes, kc, n_blk * BN);
          }
          if (++stage == S) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc = idesc_bf16(kBM, BN);
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
        if constexpr (!kOp) {
          mbar_wait(&tempty[acc], acc_phase ^ 1);
          tc_fence_after();
        }
        uint32_t d_tmem = tmem_base + acc * BN;
        for (int kb = 0; kb < num_kb; ++kb) {
          if constexpr (kOp) {
            if (kb % Cfg::kChunkKb == 0) {  // a new chunk: wait for its buffer to be drained
              mbar_wait(&tempty[acc], acc_phase ^ 1);
              tc_fence_after();
              d_tmem = tmem_base + acc * BN;
            }
          }
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint32_t sa = smem_u32(smem + stage * Cfg::kStageBytes);
          const uint32_t sb = sa + Cfg::kABytes;
          const uint64_t adesc = umma_desc_sw128(sa);
          const uint64_t bdesc = umma_desc_sw128(sb);
          if constexpr (kOp) {
            constexpr uint32_t idesc32 = idesc_tf32(kBM, BN);
            const uint64_t alo = umma_desc_sw128(sb + Cfg::kBBytes);
            const uint64_t blo = umma_desc_sw128(sb + Cfg::kBBytes + Cfg::kABytes);
#pragma unroll
            for (int k = 0; k < 4; ++k) {  // K = 8 tf32 = 32 bytes per instruction
              umma_tf32(d_tmem, adesc + 2 * k, bdesc + 2 * k, idesc32, ((kb % Cfg::kChunkKb) | k) != 0);
              umma_tf32(d_tmem, adesc + 2 * k, blo + 2 * k, idesc32, 1);
              umma_tf32(d_tmem, alo + 2 * k, bdesc + 2 * k, idesc32, 1);
            }
          } else {
#pragma unroll
            for (int k = 0; k < kBK / 16; ++k) {
              // +32 bytes per K=16 step inside the 128-byte swizzle row (encoded >> 4).
              umma_f16(d_tmem, adesc + 2 * k, bdesc + 2 * k, idesc, (kb | k) != 0);
            }
          }
          umma_commit(&empty[stage]);
          if (++stage == S) {
            stage = 0;
            phase ^= 1;
          }
          if constexpr (kOp) {
            if (kb % Cfg::kChunkKb == Cfg::kChunkKb - 1 || kb == num_kb - 1) {
              umma_commit(&tfull[acc]);  // chunk complete
              if (++acc == 2) {
                acc = 0;
                acc_phase ^= 1;
              }
            }
          }
        }
        if constexpr (!kOp) {
          umma_commit(&tfull[acc]);
          if (++acc == 2) {
            acc = 0;
            acc_phase ^= 1;
          }
        }
      }
    }
  } else if (warp >= 4) {
    const uint32_t ew = warp - 4;
    const uint32_t q = ew & 3;               // TMEM lane quarter (== warp % 4)
    constexpr int kSplit = epi_warps(EPI) / 4;  // warps sharing one TMEM lane quarter
    const int col0 = (ew >> 2) * (BN / kSplit);  // column range owned by this warp
    constexpr int kChunks = BN / kSplit / 32;
    float4* stage = epi_stage + ew * 256;
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
      const int m_blk = tile / num_n;
      const int n_blk = tile - m_blk * num_n;
      const long long m_base = static_cast<long long>(m_blk) * kBM + q * 32;
      if constexpr (epi_is_resid(EPI)) {
        // Pull this warp's residual rows (32 x BN/2 fp32) into L2 while the MMAs run.
        const long long m = m_base + lane;
        if (m < M)
          prefetch_l2_bulk(epi.resid + m * N + n_blk * BN + col0, BN / 2 * sizeof(float));
      }
      uint32_t t_row = tmem_base + ((q * 32u) << 16) + acc * BN + col0;
      if constexpr (kOp) {
        // drain the tile's K-chunks into the running total (TMEM columns [2 BN, 3 BN))
        const uint32_t t_tot = tmem_base + ((q * 32u) << 16) + 2 * BN + col0;
        const int n_chunks = (num_kb + Cfg::kChunkKb - 1) / Cfg::kChunkKb;
        for (int ch = 0; ch < n_chunks; ++ch) {
          mbar_wait(&tfull[acc], acc_phase);
          tc_fence_after();
          const uint32_t t_ch = tmem_base + ((q * 32u) << 16) + acc * BN + col0;
#pragma unroll 1
          for (int c = 0; c < BN / kSplit; c += 32) {
            uint32_t a[32], b[32];
            tmem_ld_32x32b_x32(t_ch + c, a);
            if (ch > 0) tmem_ld_32x32b_x32(t_tot + c, b);
            tmem_ld_wait();
            if (ch > 0) {
#pragma unroll
              for (int j = 0; j < 32; ++j) a[j] = __float_as_uint(__uint_as_float(b[j]) + __uint_as_float(a[j]));
            }
            tmem_st_32x32b_x32(t_tot + c, a);
          }
          tmem_st_wait();
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&tempty[acc]);  // chunk buffer free for the next MMAs
          if (++acc == 2) {
            acc = 0;
            acc_phase ^= 1;
          }
        }
        t_row = t_tot;
      } else {
        mbar_wait(&tfull[acc], acc_phase);
        tc_fence_after();
      }
      uint32_t r0[32], r1[32];
      EpiChunk ca, cb;
      RowStats rs;
      if constexpr (epi_is_stats(EPI)) rowstats_clear(rs);
      const bool live = m_base < M && !epi.skip;
      const int nb = n_blk * BN + col0;
      static_assert(kChunks % 2 == 0, "chunk pairs");
      tmem_ld_32x32b_x32(t_row, r0);
      tmem_ld_wait();
      if (live) epi_load<EPI>(epi, M, N, m_base, nb, r0, stage, ca);
#pragma unroll 1
      for (int c = 0; c < kChunks; c += 2) {
        tmem_ld_32x32b_x32(t_row + (c + 1) * 32, r1);
        tmem_ld_wait();
        if (!kOp && c + 2 == kChunks) {
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&tempty[acc]);
        }
        if (live) {
          epi_load<EPI>(epi, M, N, m_base, nb + (c + 1) * 32, r1, stage, cb);
          epi_store<EPI, OutT, kRemap>(epi, M, N, m_base, nb + c * 32, ca, rs);
        }
        if (c + 2 < kChunks) {
          tmem_ld_32x32b_x32(t_row + (c + 2) * 32, r0);
          tmem_ld_wait();
          if (live) epi_load<EPI>(epi, M, N, m_base, nb + (c + 2) * 32, r0, stage, ca);
        }
        if (live) epi_store<EPI, OutT, kRemap>(epi, M, N, m_base, nb + (c + 1) * 32, cb, rs);
        if constexpr (epi_is_stats(EPI)) {
          static_assert((BN / kSplit) % 128 == 0, "stats slots are 128-column blocks");
          if ((c + 2) % 4 == 0 && live) rowstats_flush<kRemap>(epi, M, m_base, rs, (nb + (c - 2) * 32) / 128);
        }
      }
      if constexpr (!kOp) {
        if (++acc == 2) {
          acc = 0;
          acc_phase ^= 1;
        }
      } else {
        tc_fence_before();  // total read before the next tile's first chunk overwrites it
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc<Cfg::kTmemCols>(tmem_base);
  }
}

// ------------------------------------------------------------------ tcgen05 CTA-pair kernel
// Cluster of 2 CTAs on one TPC computes a 256 x 256 tile with tcgen05.mma.cta_group::2:
// each CTA stages its 128 rows of A and its 128-row half of W per K block (32 KB), so L2 ->
// SM operand traffic per FLOP is 2/3 of the single-CTA 128 x 256 kernel and each SM's tensor
// core reads half of B from the peer's smem.  The leader (rank 0) issues all MMAs; its
// commits multicast to both CTAs' barriers; each CTA's epilogue drains its own 128 TMEM
// lanes and releases the accumulator to the leader with a cluster-scope arrive (one per warp).
//
// Epilogue store path: kinds without a row remap / stats / LN finish write each 32-row x
// 128-byte box of the output through a per-warp double-buffered smem staging box and a TMA
// store (thread = row straight from tcgen05.ld: no transpose, no per-thread global stores,
// rows >= M clipped by TMA); the others keep the transposed coalesced-store path.
// One staging box per epilogue warp leaves room for a sixth 32 KB mainloop stage (measured,
// 3 interleaved runs: qkv 131.8 -> 129.0 us, fc2 192.8 -> 190.7 us, proj 83.5 -> 84.1 us).
#ifndef TA_GEMM_BUFS
#define TA_GEMM_BUFS 1
#endif
constexpr int kMaxStatSlots = 10;  // D / 128 for D <= 1280 (ViT-H)

template <int EPI, typename OutT, bool kRemap, int kVar = 0>
struct PairCfg {
  static constexpr bool kTma = pair_tma(EPI, kRemap);
  // (16 epilogue warps with one box each measured slower than 8 with two: register spills)
  static constexpr int kWarps = pair_epi_warps(EPI, kRemap);
  // Residual kinds read the residual through the same staging boxes: TMA loads box c + 1 into
  // the warp's other box while box c is finished (TA_GEMM_RESID=ldg: per-thread row loads).
  static constexpr bool kResidTma = kTma && epi_is_resid(EPI) && sizeof(OutT) == 4;
  // kVar 2 (long K: fc2, K >= 2048): one staging box per warp, the next residual box loaded once
  // this box's store has read it, so the mainloop keeps its sixth stage (a 16 us tile leaves the
  // epilogue room for the unhidden box loads)
  static constexpr bool kOneBox = kVar == 2 && kResidTma;
  static constexpr int kBufs = kOneBox ? 1 : kResidTma ? 2 : TA_GEMM_BUFS;  // staging boxes per epilogue warp
  static constexpr int kThreads = 128 + 32 * kWarps;
  static constexpr int kABytes = 128 * kBK * 2;
  static constexpr int kBBytes = 128 * kBK * 2;  // this CTA's half of the 256-row W tile
  static constexpr int kStageBytes = kABytes + kBBytes;
  static constexpr int kEpiBytes = kTma ? kWarps * kBufs * 4096 : kEpiWarps * 32 * 32 * 4;
  // fc1 (EPI_LN_GELU): the LN-fold column constants c1 / c2 of a warp's 128 columns staged in
  // shared memory once per tile (1 KB per warp, loaded before the accumulator wait) instead of
  // 32 LDG.128 per 64-column box: those loads left the tensor pipe idle ~30 % of fc1 (ncu: 186
  // -> 164 us with them removed); costs the sixth mainloop stage.  Build with
  // -DTA_GEMM_LN_SMEM=0 to keep the loads, =2 to stage them for the QKV GEMM too.
#ifndef TA_GEMM_LN_SMEM
#define TA_GEMM_LN_SMEM 1
#endif
  static constexpr bool kLnSmem =
      kTma && TA_GEMM_LN_SMEM && (EPI == EPI_LN_GELU || (TA_GEMM_LN_SMEM == 2 && EPI == EPI_LN_BIAS));
  static constexpr int kLnBytes = kLnSmem ? kWarps * 1024 : 0;
  // Short-K residual + statistics GEMM (proj; gemm_bf16 picks K <= 1024): the bf16 copy of the
  // output rows leaves by TMA too, from two 2 KB staging boxes per warp (32 rows x 64 bytes,
  // SW64) instead of two thread-per-row STG.256 per box (ncu: those stores and the statistics
  // were 19 % of proj; 86.5 -> 83.0 us); its mainloop (12 k-blocks) runs on 4 stages.
  static constexpr bool kXh = kVar == 1 && kResidTma && epi_is_stats(EPI) && !kRemap;
  static constexpr int kXhBytes = kXh ? kWarps * 2 * 2048 : 0;
  static constexpr int kStages = kXh ? 4 : (kEpiBytes > 32768 || kLnSmem) ? 5 : 6;
  static constexpr int kSmemBytes = kStages * kStageBytes + kEpiBytes + kLnBytes + kXhBytes + 1024 + 512;
  // split-K tail code compiled in for the ta_gemm kinds and the long-K residual GEMM (fc2) only
  static constexpr bool kSplitK = kVar == 2 || EPI == EPI_BIAS || EPI == EPI_BIAS_GELU || EPI == EPI_BIAS_RESID;
};

// Split-K tail.  When the last wave of 256 x 256 tiles would leave most clusters idle, the
// launcher cuts each of its R tiles along K into s parts (s <= clusters / R): unit u < full is
// tile u (full = tiles before the tail), tail unit full + i s + p is part p of tile full + i,
// k-blocks [p num_kb / s, (p + 1) num_kb / s).  Parts p > 0 store their raw fp32 accumulator to
// epi.sk_ws (L2) and count one arrival per epilogue warp on a (tile, CTA, warp) counter; part 0,
// the owner, waits for its counter to reach s - 1, adds the partials in part order (results do
// not depend on timing), zeroes the counter and runs the tile's epilogue.  Every cluster holds
// at most one tail unit and it is its last, and the grid is co-resident (one CTA per SM, at
// most SMs / 2 clusters), so an owner only ever waits on units that are already running.
struct SkUnit {
  int tile, kb0, kb1, part, tail;  // tail: index among the split tiles, -1 for full tiles
};
__device__ __forceinline__ SkUnit sk_unit(int u, int full, int s, int num_kb) {
  if (u < full) return {u, 0, num_kb, 0, -1};
  const int i = u - full, t = i / s, p = i - t * s;
  return {full + t, p * num_kb / s, (p + 1) * num_kb / s, p, t};
}
struct SplitK {
  float* ws;  // counters (kSkFlagBytes), then partials
  int split;  // parts per tail tile (1: no split)
  int full;   // tiles before the tail
};
constexpr int kSkWarpFloats = 32 * 128;  // one epilogue warp's partial: 32 rows x 128 columns
// scratch layout: counters first (room for 256 tail tiles x 2 CTAs x 8 warps), then partials
constexpr size_t kSkFlagBytes = 256 * 2 * 8 * 4;

template <int EPI, typename OutT, bool kRemap, int kVar>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(PairCfg<EPI, OutT, kRemap, kVar>::kThreads, 1)
    gemm_bf16_sm100_pair_kernel(const __grid_constant__ CUtensorMap tmA,
                                const __grid_constant__ CUtensorMap tmB,
                                const __grid_constant__ CUtensorMap tmC,
                                const __grid_constant__ CUtensorMap tmR,
                                const __grid_constant__ CUtensorMap tmX, int M, int N, int K,
                                GemmEpi epi, SplitK sk) {
  using Cfg = PairCfg<EPI, OutT, kRemap, kVar>;
  constexpr int BN = 256;
  constexpr int S = Cfg::kStages;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  uint8_t* epi_smem = smem + S * Cfg::kStageBytes;
  float4* epi_stage = reinterpret_cast<float4*>(epi_smem);
  uint8_t* ln_smem = epi_smem + Cfg::kEpiBytes;  // kLnSmem: [kWarps][c1 128 | c2 128] fp32
  uint8_t* xh_smem = ln_smem + Cfg::kLnBytes;     // kXh: [kWarps][2] 32 x 64-byte bf16 boxes
  uint64_t* full = reinterpret_cast<uint64_t*>(xh_smem + Cfg::kXhBytes);
  uint64_t* empty = full + S;
  uint64_t* tfull = empty + S;
  uint64_t* tempty = tfull + 2;
  uint64_t* rfull = tempty + 2;  // [kWarps][kBufs]: residual box landed (kResidTma)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(rfull + Cfg::kWarps * Cfg::kBufs);

  const uint32_t warp = warp_id();
  const uint32_t lane = lane_id();
  const uint32_t rank = cluster_ctarank();
  const bool leader = rank == 0;

  if (warp == 0 && lane == 0) {
    tma_prefetch(&tmA);
    tma_prefetch(&tmB);
    if constexpr (Cfg::kTma) tma_prefetch(&tmC);
    if constexpr (Cfg::kResidTma) tma_prefetch(&tmR);
    if constexpr (Cfg::kXh) tma_prefetch(&tmX);
  }
  if (warp == 1 && lane == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 2 * Cfg::kWarps);  // one arrive per epilogue warp of both CTAs
    }
    if constexpr (Cfg::kResidTma)
      for (int i = 0; i < Cfg::kWarps * Cfg::kBufs; ++i) mbar_init(&rfull[i], 1);
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc_pair<512>(tmem_slot);
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  grid_dep_wait();

  grid_dep_launch();  // early trigger: the next kernel's prologue overlaps our tail

  const int num_m = (M + 255) / 256;
  const int num_n = N / BN;
  const int num_tiles = num_m * num_n;
  const int num_kb = K / kBK;
  const int cid = static_cast<int>(cluster_id_x());
  const int ncl = static_cast<int>(nclusters_x());
  const int sk_s = Cfg::kSplitK ? sk.split : 1;
  const int sk_full = Cfg::kSplitK ? sk.full : num_tiles;
  const int num_units = Cfg::kSplitK ? sk_full + (num_tiles - sk_full) * sk_s : num_tiles;
  auto unit_of = [&](int u) { return Cfg::kSplitK ? sk_unit(u, sk_full, sk_s, num_kb) : SkUnit{u, 0, num_kb, 0, -1}; };

  if (warp == 0) {
    if (lane == 0) {
      const uint32_t full_leader0 = mapa_shared(&full[0], 0);
      int stage = 0;
      uint32_t phase = 0;
      for (int unit = cid; unit < num_units; unit += ncl) {
        const SkUnit U = unit_of(unit);
        const int m_blk = U.tile / num_n;
        const int n_blk = U.tile - m_blk * num_n;
        for (int kb = U.kb0; kb < U.kb1; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          uint8_t* sa = smem + stage * Cfg::kStageBytes;
          uint8_t* sb = sa + Cfg::kABytes;
          if (leader) mbar_arrive_expect_tx(&full[stage], 2 * Cfg::kStageBytes);
          const uint32_t fb = full_leader0 + stage * 8;
          tma_load_2d_pair(&tmA, fb, sa, kb * kBK, m_blk * 256 + rank * 128);
          tma_load_2d_pair(&tmB, fb, sb, kb * kBK, n_blk * BN + rank * 128);
          if (++stage == S) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    // the whole warp runs the issue loop, one elected lane issues (ptx.cuh umma_f16_pair_w):
    // descriptors stay in uniform registers instead of an R2UR + elect loop per MMA
    if (leader) {
      const uint32_t tmem_base_u = __shfl_sync(0xffffffffu, tmem_base, 0);
      constexpr uint32_t idesc = idesc_bf16(256, BN);
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      for (int unit = cid; unit < num_units; unit += ncl) {
        const SkUnit U = unit_of(unit);
        mbar_wait_cluster(&tempty[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base_u + acc * BN;
        for (int kb = U.kb0; kb < U.kb1; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint32_t sa = smem_u32(smem + stage * Cfg::kStageBytes);
          const uint32_t sb = sa + Cfg::kABytes;
          const uint64_t adesc = umma_desc_sw128(sa);
          const uint64_t bdesc = umma_desc_sw128(sb);
#pragma unroll
          for (int k = 0; k < kBK / 16; ++k)
            umma_f16_pair_w(d_tmem, adesc + 2 * k, bdesc + 2 * k, idesc,
                            ((Cfg::kSplitK ? kb - U.kb0 : kb) | k) != 0);
          umma_commit_pair_w(&empty[stage]);
          if (++stage == S) {
            stage = 0;
            phase ^= 1;
          }
        }
        umma_commit_pair_w(&tfull[acc]);
        if (++acc == 2) {
          acc = 0;
          acc_phase ^= 1;
        }
      }
    }
  } else if (warp >= 4) {
    const uint32_t ew = warp - 4;
    const uint32_t q = ew & 3;
    constexpr int kSplit = Cfg::kWarps / 4;          // warps sharing one TMEM lane quarter
    const int col0 = (ew >> 2) * (BN / kSplit);      // column range owned by this warp
    constexpr int kChunks = BN / kSplit / 32;
    float4* stage = epi_stage + ew * 256;
    const uint32_t tempty_leader0 = mapa_shared(&tempty[0], 0);
    int acc = 0;
    uint32_t acc_phase = 0;
    int tma_buf = 0;
    uint32_t r_par = 0u;  // kResidTma: bit b = mbarrier parity of staging box b's next load
    const bool resid_tma = Cfg::kResidTma && !epi.resid_ldg;
    for (int unit = cid; unit < num_units; unit += ncl) {
      const SkUnit U = unit_of(unit);
      const int m_blk = U.tile / num_n;
      const int n_blk = U.tile - m_blk * num_n;
      const long long m_base = static_cast<long long>(m_blk) * 256 + rank * 128 + q * 32;
      if (Cfg::kSplitK && U.part > 0) {
        // split-K part: this warp's raw accumulator (32 rows x 128 columns) to the scratch as
        // [column quad][lane] float4, then one release arrival on the owner warp's counter
        mbar_wait(&tfull[acc], acc_phase);
        tc_fence_after();
        const uint32_t t_part = tmem_base + ((q * 32u) << 16) + acc * BN + col0;
        float4* dst = reinterpret_cast<float4*>(reinterpret_cast<char*>(sk.ws) + kSkFlagBytes) +
                      static_cast<size_t>(((U.tail * (sk_s - 1) + U.part - 1) * 2 + rank) * Cfg::kWarps + ew) *
                          (kSkWarpFloats / 4) +
                      lane;
#pragma unroll 1
        for (int g = 0; g < BN / kSplit / 32; ++g) {
          uint32_t r[32];
          tmem_ld_32x32b_x32(t_part + 32 * g, r);
          tmem_ld_wait();
#pragma unroll
          for (int j = 0; j < 8; ++j)
            stcg_f4(dst + (g * 8 + j) * 32, make_float4(__uint_as_float(r[4 * j]), __uint_as_float(r[4 * j + 1]),
                                                        __uint_as_float(r[4 * j + 2]), __uint_as_float(r[4 * j + 3])));
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          mbar_arrive_remote(tempty_leader0 + acc * 8);
          __threadfence();
          int* flags = reinterpret_cast<int*>(sk.ws);
          red_release_gpu_add(flags + (U.tail * 2 + rank) * Cfg::kWarps + ew, 1);
        }
        if (++acc == 2) {
          acc = 0;
          acc_phase ^= 1;
        }
        continue;
      }
      // kResidTma: the residual box c (32 rows x 32 fp32 of this warp's columns) goes by TMA
      // into staging box c & 1, once that box's previous store has read it; box 0 before the
      // accumulator wait, box c + 1 while box c is finished.
      auto resid_load = [&](int c) {
        if constexpr (Cfg::kResidTma) {
          if (lane == 0) {
            const int b = Cfg::kOneBox ? 0 : (c & 1);
            bulk_wait_group_read<0>();
            uint64_t* bar = &rfull[ew * Cfg::kBufs + b];
            mbar_arrive_expect_tx(bar, 4096);
            tma_load_2d(&tmR, bar, epi_smem + (ew * Cfg::kBufs + b) * 4096,
                        n_blk * BN + col0 + c * 32, static_cast<int>(m_base));
          }
          __syncwarp();
        }
      };
      if (resid_tma && epi.skip != 1) resid_load(0);  // (skip 2 still finishes the boxes)
      if constexpr (epi_is_resid(EPI)) {
        // Pull this warp's residual rows into L2 while the MMAs run.
        const long long m = m_base + lane;
        if (m < M)
          prefetch_l2_bulk(epi.resid + m * N + n_blk * BN + col0, BN / kSplit * sizeof(float));
      }
      // LN finish (EPI_LN_*): this thread's row statistics, once per tile -- loaded before the
      // accumulator wait, so their L2 latency hides under this tile's mainloop
      float ln_mu = 0.f, ln_rstd = 0.f;
      if constexpr (epi_is_ln(EPI) && Cfg::kTma) {
        const long long m = m_base + lane;
        if (m < M) {
          const float2* sp = reinterpret_cast<const float2*>(epi.ln_stats) + m * epi.stat_slots;
          float2 p[kMaxStatSlots];
#pragma unroll
          for (int j = 0; j < kMaxStatSlots; ++j)
            if (j < epi.stat_slots) p[j] = __ldg(sp + j);
          float2 st = p[0];
#pragma unroll
          for (int j = 1; j < kMaxStatSlots; ++j) {
            if (j < epi.stat_slots) {
              st.x += p[j].x;
              st.y += p[j].y;
            }
          }
          ln_mu = st.x * epi.inv_dim;
          ln_rstd = rsqrtf(fmaxf(st.y * epi.inv_dim - ln_mu * ln_mu, 0.f) + 1e-6f);
        }
      }
      const uint32_t ln_s = smem_u32(ln_smem) + ew * 1024u;  // this warp's c1 | c2 (kLnSmem)
      if constexpr (Cfg::kLnSmem) {
        // lane l: columns 4 l .. 4 l + 3 of the warp's 128 (the previous tile's reads of this
        // warp-private area are done: same warp, program order)
        const int nc = n_blk * BN + col0 + 4 * static_cast<int>(lane);
        const float4 a1 = __ldg(reinterpret_cast<const float4*>(epi.c1 + nc));
        const float4 a2 = __ldg(reinterpret_cast<const float4*>(epi.c2 + nc));
        __syncwarp();
        sts_f4(ln_s + lane * 16u, a1);
        sts_f4(ln_s + 512u + lane * 16u, a2);
        __syncwarp();
      }
      mbar_wait(&tfull[acc], acc_phase);
      tc_fence_after();
      const uint32_t t_row = tmem_base + ((q * 32u) << 16) + acc * BN + col0;
      if constexpr (Cfg::kTma) {
        // ---- thread = row; bias / GELU / residual in registers; TMA store per 128-byte box
        constexpr int CW = 128 / static_cast<int>(sizeof(OutT));  // columns per box
        constexpr int NCH = (BN / kSplit) / CW;
        const long long m = m_base + lane;
        const bool row_ok = m < M;
        // row statistics of the stored values (EPI_*_STATS) and this row's output row index
        float st_s = 0.f, st_q = 0.f;
        long long orow = m;
        if constexpr (kRemap) {
          const long long bm = m / epi.rows_in;
          orow = bm * epi.rows_out + epi.row_off + (m - bm * epi.rows_in);
        }
        constexpr bool kMerge = EPI == EPI_BIAS_RESID_MERGE;
        if constexpr (kMerge) orow = row_ok ? __ldg(epi.row_map + m) : M;  // M: past the tensor
        // rows that get a bf16 copy and statistics: every valid row, except merged-away sources
        const bool keep_row = row_ok && (!kMerge || orow < epi.rows_out);
        // compute(c): TMEM columns of box c -> bias / LN / GELU / residual -> 8 packed 16-byte
        // words of this thread's row (w); stage_store(c, w): swizzled staging box + TMA store.
        auto compute = [&](int c, uint4 (&w)[8], uint4 (&xw)[4]) -> bool {
          const int n0 = n_blk * BN + col0 + c * CW;
          float v[CW];
          {
            uint32_t r[CW];
#pragma unroll
            for (int g = 0; g < CW / 32; ++g)
              tmem_ld_32x32b_x32(t_row + c * CW + 32 * g, *reinterpret_cast<uint32_t(*)[32]>(&r[32 * g]));
            tmem_ld_wait();
#pragma unroll
            for (int j = 0; j < CW; ++j) v[j] = __uint_as_float(r[j]);
          }
          if (c + 1 == NCH) {  // accumulator fully read: hand it back to the MMA warp
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive_remote(tempty_leader0 + acc * 8);
          }
          if (Cfg::kSplitK && U.tail >= 0) {  // split-K owner: add parts 1 .. s - 1 of these columns, in order
            if (c == 0) {
              if (lane == 0) {
                int* f = reinterpret_cast<int*>(sk.ws) +
                         (U.tail * 2 + rank) * Cfg::kWarps + ew;
                while (ld_acquire_gpu(f) < sk_s - 1) __nanosleep(32);
                *f = 0;  // (every part has arrived: the next launch starts from zero)
              }
              __syncwarp();
            }
            const float4* src = reinterpret_cast<const float4*>(reinterpret_cast<const char*>(sk.ws) + kSkFlagBytes) +
                                static_cast<size_t>((U.tail * (sk_s - 1) * 2 + rank) * Cfg::kWarps + ew) *
                                    (kSkWarpFloats / 4) +
                                (c * CW / 4) * 32 + lane;
#pragma unroll 1
            for (int p = 1; p < sk_s; ++p) {
              const float4* sp = src + static_cast<size_t>(p - 1) * 2 * Cfg::kWarps * (kSkWarpFloats / 4);
#pragma unroll
              for (int j = 0; j < CW / 4; ++j) {
                const float4 a = ldcg_f4(sp + j * 32);
                v[4 * j] += a.x;
                v[4 * j + 1] += a.y;
                v[4 * j + 2] += a.z;
                v[4 * j + 3] += a.w;
              }
            }
          }
          if (epi.skip == 1) return false;
          if (epi.skip >= 4 && static_cast<int>(q) == epi.skip - 4) return false;  // profiling: one lane quarter's warps idle
          if constexpr (Cfg::kResidTma) {
            if (resid_tma) {
              if (!Cfg::kOneBox && c + 1 < NCH) resid_load(c + 1);
              const int b = Cfg::kOneBox ? 0 : (c & 1);
              mbar_wait(&rfull[ew * Cfg::kBufs + b], (r_par >> b) & 1u);
              r_par ^= 1u << b;
              // this row's 32 residual values: SW128 chunk j at (j ^ (row & 7))
              const uint32_t srow = smem_u32(epi_smem + (ew * Cfg::kBufs + b) * 4096) + lane * 128;
#pragma unroll
              for (int j = 0; j < CW / 4; ++j) {
                const float4 rr = lds_f4(srow + ((j ^ (lane & 7)) << 4));
                const float2 lo = f2_unpack(fadd2(f2_pack(v[4 * j], v[4 * j + 1]), f2_pack(rr.x, rr.y)));
                const float2 hi = f2_unpack(fadd2(f2_pack(v[4 * j + 2], v[4 * j + 3]), f2_pack(rr.z, rr.w)));
                v[4 * j] = lo.x;
                v[4 * j + 1] = lo.y;
                v[4 * j + 2] = hi.x;
                v[4 * j + 3] = hi.y;
              }
            }
          }
          if constexpr (epi_is_resid(EPI) || epi_is_patch(EPI)) {
            if (row_ok && !(Cfg::kResidTma && resid_tma)) {
              const float4* rp =
                  epi_is_resid(EPI)
                      ? reinterpret_cast<const float4*>(epi.resid + m * N + n0)
                      : reinterpret_cast<const float4*>(epi.pos + (epi.row_off + m % epi.rows_in) * N + n0);
              float4 rr[CW / 4];
#pragma unroll
              for (int j = 0; j < CW / 4; ++j) rr[j] = rp[j];
#pragma unroll
              for (int j = 0; j < CW / 4; ++j) {
                const float2 lo = f2_unpack(fadd2(f2_pack(v[4 * j], v[4 * j + 1]), f2_pack(rr[j].x, rr[j].y)));
                const float2 hi = f2_unpack(fadd2(f2_pack(v[4 * j + 2], v[4 * j + 3]), f2_pack(rr[j].z, rr[j].w)));
                v[4 * j] = lo.x;
                v[4 * j + 1] = lo.y;
                v[4 * j + 2] = hi.x;
                v[4 * j + 3] = hi.y;
              }
            }
          }
          if constexpr (epi_is_ln(EPI)) {
            const float4* c1p = reinterpret_cast<const float4*>(epi.c1 + n0);
            const float4* c2p = reinterpret_cast<const float4*>(epi.c2 + n0);
            const uint64_t nmu2 = f2_pack(-ln_mu, -ln_mu), rstd2 = f2_pack(ln_rstd, ln_rstd);
#pragma unroll
            for (int j = 0; j < CW / 4; ++j) {
#ifdef TA_EXP_LN_NOLOAD  // profiling only: wrong results (LN-fold column constants not loaded)
              const float4 a1 = make_float4(v[0], v[1], v[2], v[3]), a2 = a1;
#else
              float4 a1, a2;
              if constexpr (Cfg::kLnSmem) {  // broadcast LDS of the staged constants
                a1 = lds_f4(ln_s + static_cast<uint32_t>(c * CW + 4 * j) * 4u);
                a2 = lds_f4(ln_s + 512u + static_cast<uint32_t>(c * CW + 4 * j) * 4u);
              } else {
                a1 = __ldg(c1p + j);
                a2 = __ldg(c2p + j);
              }
#endif
              const float2 lo = f2_unpack(ffma2(rstd2, ffma2(nmu2, f2_pack(a1.x, a1.y), f2_pack(v[4 * j], v[4 * j + 1])),
                                                f2_pack(a2.x, a2.y)));
              const float2 hi = f2_unpack(ffma2(rstd2, ffma2(nmu2, f2_pack(a1.z, a1.w), f2_pack(v[4 * j + 2], v[4 * j + 3])),
                                                f2_pack(a2.z, a2.w)));
              v[4 * j] = lo.x;
              v[4 * j + 1] = lo.y;
              v[4 * j + 2] = hi.x;
              v[4 * j + 3] = hi.y;
            }
          } else {
            const float4* bp = reinterpret_cast<const float4*>(epi.bias + n0);
#pragma unroll
            for (int j = 0; j < CW / 4; ++j) {
              const float4 b = __ldg(bp + j);
              const float2 lo = f2_unpack(fadd2(f2_pack(v[4 * j], v[4 * j + 1]), f2_pack(b.x, b.y)));
              const float2 hi = f2_unpack(fadd2(f2_pack(v[4 * j + 2], v[4 * j + 3]), f2_pack(b.z, b.w)));
              v[4 * j] = lo.x;
              v[4 * j + 1] = lo.y;
              v[4 * j + 2] = hi.x;
              v[4 * j + 3] = hi.y;
            }
          }
          if constexpr (epi_is_gelu(EPI)) {
#pragma unroll
            for (int j = 0; j < CW; j += 2) {
              const float2 gv = f2_unpack(gelu_poly2(f2_pack(v[j], v[j + 1])));
              v[j] = gv.x;
              v[j + 1] = gv.y;
            }
          }
          if constexpr (epi_is_stats(EPI)) {
            // bf16 copy of the stored row chunk (next GEMM's A operand) + row statistics
            if constexpr (Cfg::kXh) {  // packed here, staged and stored by TMA in stage_store
              static_assert(CW == 32, "fp32 boxes: 32 columns of bf16 copy");
#pragma unroll
              for (int j = 0; j < 4; ++j)
                xw[j] = make_uint4(pack_bf16(v[8 * j], v[8 * j + 1]), pack_bf16(v[8 * j + 2], v[8 * j + 3]),
                                   pack_bf16(v[8 * j + 4], v[8 * j + 5]), pack_bf16(v[8 * j + 6], v[8 * j + 7]));
            }
            if (keep_row) {
              uint4* xr = reinterpret_cast<uint4*>(static_cast<__nv_bfloat16*>(epi.xh) + orow * N + n0);
              static_assert(CW % 16 == 0, "32-byte xh stores");
#pragma unroll
              for (int j = 0; j < CW / 16; ++j)  // full 32-byte sectors (STG.256)
                if (!Cfg::kXh || (!kRemap && epi.direct_store))
                  stg256(xr + 2 * j,
                         make_uint4(pack_bf16(v[16 * j], v[16 * j + 1]), pack_bf16(v[16 * j + 2], v[16 * j + 3]),
                                    pack_bf16(v[16 * j + 4], v[16 * j + 5]), pack_bf16(v[16 * j + 6], v[16 * j + 7])),
                         make_uint4(pack_bf16(v[16 * j + 8], v[16 * j + 9]), pack_bf16(v[16 * j + 10], v[16 * j + 11]),
                                    pack_bf16(v[16 * j + 12], v[16 * j + 13]), pack_bf16(v[16 * j + 14], v[16 * j + 15])));
              uint64_t s2 = 0ull, q2 = 0ull;  // packed partial sums (two chains)
#pragma unroll
              for (int j = 0; j < CW; j += 2) {
                const uint64_t p = f2_pack(v[j], v[j + 1]);
                s2 = fadd2(s2, p);
                q2 = ffma2(p, p, q2);
              }
              const float2 sv = f2_unpack(s2), qv = f2_unpack(q2);
              st_s += sv.x + sv.y;
              st_q += qv.x + qv.y;
            }
          }
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            if constexpr (sizeof(OutT) == 2) {
              w[j] = make_uint4(pack_bf16(v[8 * j], v[8 * j + 1]), pack_bf16(v[8 * j + 2], v[8 * j + 3]),
                                pack_bf16(v[8 * j + 4], v[8 * j + 5]), pack_bf16(v[8 * j + 6], v[8 * j + 7]));
            } else {
              w[j] = make_uint4(__float_as_uint(v[4 * j]), __float_as_uint(v[4 * j + 1]),
                                __float_as_uint(v[4 * j + 2]), __float_as_uint(v[4 * j + 3]));
            }
          }
          return true;
        };
        auto stage_store = [&](int c, const uint4 (&w)[8], const uint4 (&xw)[4]) {
          const int n0 = n_blk * BN + col0 + c * CW;
          if (Cfg::kResidTma && resid_tma) tma_buf = Cfg::kOneBox ? 0 : (c & 1);  // the residual's box (already free)
          uint8_t* sbuf = epi_smem + (ew * Cfg::kBufs + tma_buf) * 4096;
          if (!(Cfg::kResidTma && resid_tma) && lane == 0)
            bulk_wait_group_read<Cfg::kBufs - 1>();  // last store from sbuf has read it
          __syncwarp();
          const uint32_t srow = smem_u32(sbuf) + lane * 128;
          // Row remap: a row of this box that belongs to a later image is also stored directly
          // (the box's TMA store lands it in this image's prompt / padding slots, which
          // insert_rows rewrites, or clips it past rows_out).
          uint4* spill_row = nullptr;
          if constexpr (kRemap) {
            const int b = static_cast<int>(m_base / epi.rows_in);
            const int i = static_cast<int>(m_base - static_cast<long long>(b) * epi.rows_in) + lane;
            if (i >= epi.rows_in && row_ok) {  // image b + i / rows_in (short images: >1 boundary)
              const int bi = i / epi.rows_in;
              spill_row = reinterpret_cast<uint4*>(
                  static_cast<OutT*>(epi.out) +
                  (static_cast<long long>(b + bi) * epi.rows_out + epi.row_off + i - bi * epi.rows_in) * N +
                  n0);
            }
          }
#pragma unroll
          for (int j = 0; j < 8; ++j) {  // 16-byte chunk j of this row, SW128 position j ^ (row & 7)
            sts_u4(srow + ((j ^ (lane & 7)) << 4), w[j]);
            if (kRemap && spill_row != nullptr) spill_row[j] = w[j];
          }
          // bf16 copy box c & 1 (its previous store, box c - 2, was waited for by resid_load)
          const uint32_t xbox = smem_u32(xh_smem) + (ew * 2u + static_cast<uint32_t>(c & 1)) * 2048u;
          if constexpr (Cfg::kXh) {
            if (!resid_tma) {  // (the per-thread residual path does not wait in resid_load)
              if (lane == 0) bulk_wait_group_read<0>();
              __syncwarp();
            }
#pragma unroll
            for (int j = 0; j < 4; ++j)  // SW64: 16-byte chunk j of row r at j ^ ((r >> 1) & 3)
              sts_u4(xbox + lane * 64u + ((j ^ ((lane >> 1) & 3)) << 4), xw[j]);
          }
          fence_proxy_async_shared();
          __syncwarp();
          if constexpr (kMerge) {
            // merged positions: eight 4-row scatters of the box (rows >= M are dropped by TMA)
            const int dst = static_cast<int>(orow);
#pragma unroll
            for (int g = 0; g < 8; ++g) {
              const int r0 = __shfl_sync(0xffffffffu, dst, 4 * g), r1 = __shfl_sync(0xffffffffu, dst, 4 * g + 1);
              const int r2 = __shfl_sync(0xffffffffu, dst, 4 * g + 2), r3 = __shfl_sync(0xffffffffu, dst, 4 * g + 3);
              if (lane == 0 && epi.skip != 2) {
                tma_scatter4(&tmC, smem_u32(sbuf) + g * 512, n0, r0, r1, r2, r3);
                if constexpr (Cfg::kXh) tma_scatter4(&tmX, xbox + g * 256, n0, r0, r1, r2, r3);
              }
            }
            if (lane == 0 && epi.skip != 2) bulk_commit_group();
          } else if (lane == 0 && epi.skip != 2) {
            if constexpr (kRemap) {
              // 3D view [B][rows_out][N]: the box goes to image b at its in-image row.
              const int b = static_cast<int>(m_base / epi.rows_in);
              const int i0 = static_cast<int>(m_base - static_cast<long long>(b) * epi.rows_in);
              tma_store_3d(&tmC, sbuf, n0, epi.row_off + i0, b);
            } else {
              tma_store_2d(&tmC, sbuf, n0, static_cast<int32_t>(m_base));
              if constexpr (Cfg::kXh) tma_store_2d_s(&tmX, xbox, n0, static_cast<int32_t>(m_base));
            }
            bulk_commit_group();
          }
          tma_buf = (tma_buf + 1) % Cfg::kBufs;
          // one box: the next residual box goes into it once this store has read it
          if constexpr (Cfg::kOneBox)
            if (resid_tma && c + 1 < NCH) resid_load(c + 1);
        };
        // (Interleaved per box.  Reading every box and releasing the accumulator before any
        // staging wait measured slower: the extra live registers cost more than the wait.)
        // Direct path (TA_GEMM_STORE=direct, profiling A/B): each thread writes its row's
        // 128-byte box as four 32-byte STG.256 stores instead of the smem box + TMA store.
        auto direct_store = [&](int c, const uint4 (&w)[8]) {
          if (!row_ok || epi.skip == 2) return;
          const int n0 = n_blk * BN + col0 + c * CW;
          OutT* row_ptr = static_cast<OutT*>(epi.out) + (kMerge ? orow : m) * N;
          uint4* dst = reinterpret_cast<uint4*>(row_ptr + n0);
#pragma unroll
          for (int j = 0; j < 4; ++j) stg256(dst + 2 * j, w[2 * j], w[2 * j + 1]);
        };
#pragma unroll 1
        for (int c = 0; c < NCH; ++c) {
          uint4 w[8], xw[4];
          if (compute(c, w, xw)) {
            if (!kRemap && epi.direct_store)
              direct_store(c, w);
            else
              stage_store(c, w, xw);
          }
        }
        if constexpr (epi_is_stats(EPI)) {
          static_assert(BN / kSplit == 128, "one stats slot per warp and tile");
          if (keep_row && !epi.skip)
            *reinterpret_cast<float2*>(epi.stats + 2 * (orow * epi.stat_slots + (n_blk * BN + col0) / 128)) =
                make_float2(st_s, st_q);
        }
      } else {
        uint32_t r0[32], r1[32];
        EpiChunk ca, cb;
        RowStats rs;
        if constexpr (epi_is_stats(EPI)) rowstats_clear(rs);
        const bool live = m_base < M && !epi.skip;
        const int nb = n_blk * BN + col0;
        tmem_ld_32x32b_x32(t_row, r0);
        tmem_ld_wait();
        if (live) epi_load<EPI>(epi, M, N, m_base, nb, r0, stage, ca);
#pragma unroll 1
        for (int c = 0; c < kChunks; c += 2) {
          tmem_ld_32x32b_x32(t_row + (c + 1) * 32, r1);
          tmem_ld_wait();
          if (c + 2 == kChunks) {
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive_remote(tempty_leader0 + acc * 8);
          }
          if (live) {
            epi_load<EPI>(epi, M, N, m_base, nb + (c + 1) * 32, r1, stage, cb);
            epi_store<EPI, OutT, kRemap>(epi, M, N, m_base, nb + c * 32, ca, rs);
          }
          if (c + 2 < kChunks) {
            tmem_ld_32x32b_x32(t_row + (c + 2) * 32, r0);
            tmem_ld_wait();
            if (live) epi_load<EPI>(epi, M, N, m_base, nb + (c + 2) * 32, r0, stage, ca);
          }
          if (live) epi_store<EPI, OutT, kRemap>(epi, M, N, m_base, nb + (c + 1) * 32, cb, rs);
        }
        if constexpr (epi_is_stats(EPI)) {
          if (live) rowstats_flush<kRemap>(epi, M, m_base, rs, nb / 128);
        }
      }
      if (++acc == 2) {
        acc = 0;
        acc_phase ^= 1;
      }
    }
  }
  if constexpr (Cfg::kTma) {
    if (warp >= 4 && lane == 0) bulk_wait_group<0>();  // staged boxes fully stored
  }
  tc_fence_before();
  cluster_sync();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc_pair<512>(tmem_base);
  }
}

// ------------------------------------------------------------------ SIMT fp32 kernel
// 128 x 128 tile, BK = 8, 256 threads, 8 x 8 outputs per thread.  fp32 FFMA only:
// products are exact fp32 so results differ from a CPU fp32 GEMM by summation order.
template <int EPI>
__global__ void __launch_bounds__(256) gemm_f32_simt_kernel(const float* __restrict__ A,
                                                            const float* __restrict__ W, int M,
                                                            int N, int K, GemmEpi epi) {
  __shared__ float As[2][8][128 + 4];
  __shared__ float Bs[2][8][128 + 4];
  const int tid = threadIdx.x;
  const int m0 = blockIdx.y * 128;
  const int n0 = blockIdx.x * 128;
  const int tr = tid / 16;  // 16 x 16 thread grid
  const int tc = tid % 16;
  float acc[8][8] = {};
  // Loader: 128 rows x 8 k per operand = 1024 floats = 256 threads x 4 (one float4).
  const int lrow = tid / 2;
  const int lk = (tid % 2) * 4;
  auto load = [&](int buf, int k0) {
    float4 a = make_float4(0.f, 0.f, 0.f, 0.f);
    if (m0 + lrow < M) a = *reinterpret_cast<const float4*>(A + (long long)(m0 + lrow) * K + k0 + lk);
    const float4 b = *reinterpret_cast<const float4*>(W + (long long)(n0 + lrow) * K + k0 + lk);
    As[buf][lk + 0][lrow] = a.x;
    As[buf][lk + 1][lrow] = a.y;
    As[buf][lk + 2][lrow] = a.z;
    As[buf][lk + 3][lrow] = a.w;
    Bs[buf][lk + 0][lrow] = b.x;
    Bs[buf][lk + 1][lrow] = b.y;
    Bs[buf][lk + 2][lrow] = b.z;
    Bs[buf][lk + 3][lrow] = b.w;
  };
  load(0, 0);
  __syncthreads();
  int buf = 0;
  for (int k0 = 0; k0 < K; k0 += 8) {
    if (k0 + 8 < K) load(buf ^ 1, k0 + 8);
#pragma unroll
    for (int kk = 0; kk < 8; ++kk) {
      float a[8], b[8];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        a[i] = As[buf][kk][tr * 4 + i];
        a[4 + i] = As[buf][kk][64 + tr * 4 + i];
        b[i] = Bs[buf][kk][tc * 4 + i];
        b[4 + i] = Bs[buf][kk][64 + tc * 4 + i];
      }
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
    }
    __syncthreads();
    buf ^= 1;
  }
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const long long m = m0 + (i < 4 ? tr * 4 + i : 64 + tr * 4 + (i - 4));
    if (m >= M) continue;
    const long long orow = epi_out_row(epi, m);
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int n = n0 + (j < 4 ? tc * 4 + j : 64 + tc * 4 + (j - 4));
      float v = acc[i][j] + epi.bias[n];
      if (EPI == EPI_BIAS_GELU) v = gelu_erf(v);
      if (EPI == EPI_BIAS_RESID) v = epi.resid[m * N + n] + v;
      if (EPI == EPI_PATCH) v += epi.pos[(epi.row_off + m % epi.rows_in) * (long long)N + n];
      static_cast<float*>(epi.out)[orow * N + n] = v;
    }
  }
}

// ------------------------------------------------------------------ host side
static PFN_cuTensorMapEncodeTiled_v12000 get_encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

// Row-major bf16 matrix [rows, cols] as a 2D tensor map with a (64 x box_rows) SW128 box.
// bf16 [rows, cols] map with a {box_cols, box_rows} box and 32 / 64 / 128-byte swizzle.
int make_tmap_bf16_2d_sw(CUtensorMap* map, const void* base, uint64_t rows, uint64_t cols,
                         uint32_t box_cols, uint32_t box_rows, int swizzle_bytes) {
  auto enc = get_encode_fn();
  if (!enc) return TA_ERR_CUDA;
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {cols * 2};
  cuuint32_t box[2] = {box_cols, box_rows};
  cuuint32_t estr[2] = {1, 1};
  const CUtensorMapSwizzle sw = swizzle_bytes == 32   ? CU_TENSOR_MAP_SWIZZLE_32B
                                : swizzle_bytes == 64 ? CU_TENSOR_MAP_SWIZZLE_64B
                                                      : CU_TENSOR_MAP_SWIZZLE_128B;
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims,
                   strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, sw,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? TA_OK : TA_ERR_SHAPE;
}

int make_tmap_bf16_2d(CUtensorMap* map, const void* base, uint64_t rows, uint64_t cols,
                      uint32_t box_rows) {
  auto enc = get_encode_fn();
  if (!enc) return TA_ERR_CUDA;
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {cols * 2};
  cuuint32_t box[2] = {64, box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims,
                   strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? TA_OK : TA_ERR_SHAPE;
}

template <int BN, int EPI, typename OutT, bool kRemap = false, int kOp = 0>
static int launch_bf16(const CUtensorMap& ta_, const CUtensorMap& tb_, int M, int N, int K,
                       const GemmEpi& epi, cudaStream_t stream, const CUtensorMap* ta2 = nullptr,
                       const CUtensorMap* tb2 = nullptr) {
  using Cfg = GemmCfg<BN, kOp>;
  auto kern = gemm_bf16_sm100_kernel<BN, EPI, OutT, kRemap, kOp>;
  static unsigned long long attr_mask = 0;  // per instantiation and device
  if (attr_needed(attr_mask)) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         Cfg::kSmemBytes);
    if (e != cudaSuccess) return set_last_cuda_error(e);
    attr_done(attr_mask);
  }
  const int tiles = ((M + kBM - 1) / kBM) * (N / BN);
  const int grid = tiles < device_sm_count() ? tiles : device_sm_count();
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(gemm_threads(EPI));
  cfg.dynamicSmemBytes = Cfg::kSmemBytes;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled();
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaError_t e = cudaLaunchKernelEx(&cfg, kern, ta_, tb_, ta2 ? *ta2 : ta_, tb2 ? *tb2 : tb_, M, N, K, epi);
  return e == cudaSuccess ? TA_OK : set_last_cuda_error(e);
}

// Output tensor map for the TMA-store epilogue: [M, N] row-major, 32-row x 128-byte boxes, SW128.
static int make_tmap_out(CUtensorMap* map, const void* base, uint64_t rows, uint64_t cols,
                         bool bf16, uint32_t box_rows = 32) {
  auto enc = get_encode_fn();
  if (!enc) return TA_ERR_CUDA;
  const uint64_t es = bf16 ? 2 : 4;
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {cols * es};
  cuuint32_t box[2] = {static_cast<cuuint32_t>(128 / es), box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(map, bf16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2,
                   const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? TA_OK : TA_ERR_SHAPE;
}

// bf16 copy of a residual kind's output: 32-column (64-byte) boxes, SW64.
static int make_tmap_xh(CUtensorMap* map, const void* base, uint64_t rows, uint64_t cols, uint32_t box_rows) {
  auto enc = get_encode_fn();
  if (!enc) return TA_ERR_CUDA;
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {cols * 2};
  cuuint32_t box[2] = {32, box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? TA_OK : TA_ERR_SHAPE;
}

// 3D view [B][rows_out][N] of a row-remapped output, same 32-row x 128-byte boxes.
static int make_tmap_out3(CUtensorMap* map, const void* base, uint64_t images, uint64_t rows_out,
                          uint64_t cols, bool bf16) {
  auto enc = get_encode_fn();
  if (!enc) return TA_ERR_CUDA;
  const uint64_t es = bf16 ? 2 : 4;
  cuuint64_t dims[3] = {cols, rows_out, images};
  cuuint64_t strides[2] = {cols * es, rows_out * cols * es};
  cuuint32_t box[3] = {static_cast<cuuint32_t>(128 / es), 32, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = enc(map, bf16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3,
                   const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? TA_OK : TA_ERR_SHAPE;
}

// Attention output [B][t][D] bf16 as a 3D map with 32-column (64-byte) x 32-row boxes, SW64:
// one box per softmax warp's O slab (attention_tc.cu store_o_slab); rows >= t are clipped.
int make_tmap_attn_out(CUtensorMap* map, const void* base, uint64_t images, uint64_t t,
                       uint64_t cols) {
  auto enc = get_encode_fn();
  if (!enc) return TA_ERR_CUDA;
  cuuint64_t dims[3] = {cols, t, images};
  cuuint64_t strides[2] = {cols * 2, t * cols * 2};
  cuuint32_t box[3] = {32, 32, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, strides,
                   box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? TA_OK : TA_ERR_SHAPE;
}

// Split-K tail parts for a launch of `tiles` pair tiles over `pairs` clusters (1 = no split):
// the R = tiles % pairs tiles of the last wave are cut into s = min(pairs / R, TA_GEMM_SPLITK
// (default 4)) parts of at least 4 k-blocks each, for K >= TA_GEMM_SK_MINKB k-blocks (default
// 24: fc2; a 12-k-block tile's tail costs less than the partial round trip would save).
static int splitk_parts(int tiles, int pairs, int num_kb, bool have_ws) {
  static const int max_parts = [] {
    const char* v = getenv("TA_GEMM_SPLITK");
    return v ? atoi(v) : 4;
  }();
  static const int min_kb = [] {
    const char* v = getenv("TA_GEMM_SK_MINKB");
    return v ? atoi(v) : 24;
  }();
  const int R = tiles % pairs;
  if (!have_ws || max_parts < 2 || num_kb < min_kb || R == 0) return 1;
  int p = std::min(std::min(pairs / R, max_parts), num_kb / 4);
  if (static_cast<size_t>(R) * 2 * 8 * 4 > kSkFlagBytes) p = 1;
  return p >= 2 ? p : 1;
}

size_t gemm_splitk_flag_bytes() { return kSkFlagBytes; }
// partials: R (s - 1) < pairs tiles' worth, 256 x 256 fp32 each
size_t gemm_splitk_ws_bytes() { return kSkFlagBytes + static_cast<size_t>(device_sm_count() / 2) * 256 * 256 * 4; }

template <int EPI, typename OutT, bool kRemap = false, int kVar = 0>
static int launch_pair(const CUtensorMap& ta_, const CUtensorMap& tb_, int M, int N, int K,
                       const GemmEpi& epi, cudaStream_t stream, float* sk_ws) {
  using Cfg = PairCfg<EPI, OutT, kRemap, kVar>;
  auto kern = gemm_bf16_sm100_pair_kernel<EPI, OutT, kRemap, kVar>;
  static unsigned long long attr_mask = 0;  // per instantiation and device
  if (attr_needed(attr_mask)) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         Cfg::kSmemBytes);
    if (e != cudaSuccess) return set_last_cuda_error(e);
    attr_done(attr_mask);
  }
  CUtensorMap tc_{}, tr_{};
  if (Cfg::kTma) {  // the merge kind: one-row boxes for tile::scatter4 over the M rows of out
    const int rc = kRemap ? make_tmap_out3(&tc_, epi.out, M / epi.rows_in, epi.rows_out, N, sizeof(OutT) == 2)
                          : make_tmap_out(&tc_, epi.out, M, N, sizeof(OutT) == 2,
                                          EPI == EPI_BIAS_RESID_MERGE ? 1 : 32);
    if (rc) return rc;
  }
  if (Cfg::kResidTma) {  // the residual in the input row numbering, 32-row boxes
    const int rc = make_tmap_out(&tr_, epi.resid, M, N, false);
    if (rc) return rc;
  }
  CUtensorMap tx_{};
  if (Cfg::kXh) {  // bf16 copy: 32-column (64-byte, SW64) boxes of 32 rows, or single rows to scatter
    const int rc = make_tmap_xh(&tx_, epi.xh, M, N, EPI == EPI_BIAS_RESID_MERGE ? 1 : 32);
    if (rc) return rc;
  }
  const int tiles = ((M + 255) / 256) * (N / 256);
  const int pairs = device_sm_count() / 2;
  SplitK sk{sk_ws, 1, tiles};
  sk.split = Cfg::kSplitK ? splitk_parts(tiles, pairs, K / kBK, sk_ws != nullptr) : 1;
  sk.full = sk.split > 1 ? tiles - tiles % pairs : tiles;
  const int units = sk.full + (tiles - sk.full) * sk.split;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(2 * (units < pairs ? units : pairs));
  cfg.blockDim = dim3(Cfg::kThreads);
  cfg.dynamicSmemBytes = Cfg::kSmemBytes;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled();
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaError_t e = cudaLaunchKernelEx(&cfg, kern, ta_, tb_, tc_, tr_, tx_, M, N, K, epi, sk);
  return e == cudaSuccess ? TA_OK : set_last_cuda_error(e);
}

// Residual + statistics GEMMs with K <= kShortK (proj, fused proj + merge) store the bf16 copy
// by TMA (PairCfg::kXh); TA_GEMM_XH=stg keeps the per-thread stores (A/B).
constexpr int kShortK = 1024;
// Residual GEMMs with K >= kLongK (fc2) use one staging box and keep six stages (PairCfg::kOneBox);
// TA_GEMM_ONEBOX=0 keeps two boxes (A/B).
constexpr int kLongK = 2048;
static bool one_box_enabled() {
  static const int on = [] {
    const char* v = getenv("TA_GEMM_ONEBOX");
    return (v && v[0] == '0') ? 0 : 1;
  }();
  return on != 0;
}
static bool xh_tma_enabled() {
  static const int on = [] {
    const char* v = getenv("TA_GEMM_XH");
    return (v && v[0] == 's') ? 0 : 1;
  }();
  return on != 0;
}

static int dispatch_pair(const CUtensorMap& a, const CUtensorMap& b, int M, int N, int K,
                         int epi_kind, bool out_bf16, const GemmEpi& epi, cudaStream_t s, float* sk_ws) {
  switch (epi_kind) {
    case EPI_BIAS:
      return out_bf16 ? launch_pair<EPI_BIAS, __nv_bfloat16>(a, b, M, N, K, epi, s, sk_ws)
                      : launch_pair<EPI_BIAS, float>(a, b, M, N, K, epi, s, sk_ws);
    case EPI_BIAS_GELU:
      return out_bf16 ? launch_pair<EPI_BIAS_GELU, __nv_bfloat16>(a, b, M, N, K, epi, s, sk_ws)
                      : launch_pair<EPI_BIAS_GELU, float>(a, b, M, N, K, epi, s, sk_ws);
    case EPI_BIAS_RESID:
      if (K >= kLongK && one_box_enabled())
        return epi.rows_in ? launch_pair<EPI_BIAS_RESID, float, true, 2>(a, b, M, N, K, epi, s, sk_ws)
                           : launch_pair<EPI_BIAS_RESID, float, false, 2>(a, b, M, N, K, epi, s, sk_ws);
      return epi.rows_in ? launch_pair<EPI_BIAS_RESID, float, true>(a, b, M, N, K, epi, s, sk_ws)
                         : launch_pair<EPI_BIAS_RESID, float, false>(a, b, M, N, K, epi, s, sk_ws);
    case EPI_PATCH:
      return launch_pair<EPI_PATCH, float, true>(a, b, M, N, K, epi, s, sk_ws);
    case EPI_BIAS_RESID_STATS:
      if (K >= kLongK && one_box_enabled())
        return epi.rows_in ? launch_pair<EPI_BIAS_RESID_STATS, float, true, 2>(a, b, M, N, K, epi, s, sk_ws)
                           : launch_pair<EPI_BIAS_RESID_STATS, float, false, 2>(a, b, M, N, K, epi, s, sk_ws);
      if (epi.rows_in) return launch_pair<EPI_BIAS_RESID_STATS, float, true>(a, b, M, N, K, epi, s, sk_ws);
      return K <= kShortK && xh_tma_enabled()
                 ? launch_pair<EPI_BIAS_RESID_STATS, float, false, 1>(a, b, M, N, K, epi, s, sk_ws)
                 : launch_pair<EPI_BIAS_RESID_STATS, float, false>(a, b, M, N, K, epi, s, sk_ws);
    case EPI_PATCH_STATS:
      return launch_pair<EPI_PATCH_STATS, float, true>(a, b, M, N, K, epi, s, sk_ws);
    case EPI_LN_BIAS:
      return launch_pair<EPI_LN_BIAS, __nv_bfloat16>(a, b, M, N, K, epi, s, sk_ws);
    case EPI_LN_GELU:
      return launch_pair<EPI_LN_GELU, __nv_bfloat16>(a, b, M, N, K, epi, s, sk_ws);
    case EPI_BIAS_RESID_MERGE:
      // (the merge kind keeps the per-thread bf16 stores: 16 scatter4 per box on a 4-stage ring
      // measured 81.5 -> 87.5 us per fused proj)
      return launch_pair<EPI_BIAS_RESID_MERGE, float, false>(a, b, M, N, K, epi, s, sk_ws);
  }
  return TA_ERR_INVALID;
}

// 0 = CTA-pair kernel where it applies (default), 1 = single-CTA kernel (TA_GEMM_BACKEND=single).
static int gemm_backend() {
  static int mode = -1;
  if (mode < 0) {
    const char* v = getenv("TA_GEMM_BACKEND");
    mode = (v && v[0] == 's') ? 1 : 0;
  }
  return mode;
}

template <int BN>
static int dispatch_bf16(const CUtensorMap& a, const CUtensorMap& b, int M, int N, int K,
                         int epi_kind, bool out_bf16, const GemmEpi& epi, cudaStream_t s) {
  switch (epi_kind) {
    case EPI_BIAS:
      return out_bf16 ? launch_bf16<BN, EPI_BIAS, __nv_bfloat16>(a, b, M, N, K, epi, s)
                      : launch_bf16<BN, EPI_BIAS, float>(a, b, M, N, K, epi, s);
    case EPI_BIAS_GELU:
      return out_bf16 ? launch_bf16<BN, EPI_BIAS_GELU, __nv_bfloat16>(a, b, M, N, K, epi, s)
                      : launch_bf16<BN, EPI_BIAS_GELU, float>(a, b, M, N, K, epi, s);
    case EPI_BIAS_RESID:
      return epi.rows_in ? launch_bf16<BN, EPI_BIAS_RESID, float, true>(a, b, M, N, K, epi, s)
                         : launch_bf16<BN, EPI_BIAS_RESID, float, false>(a, b, M, N, K, epi, s);
    case EPI_PATCH:
      return launch_bf16<BN, EPI_PATCH, float, true>(a, b, M, N, K, epi, s);
    case EPI_BIAS_RESID_STATS:
      return epi.rows_in ? launch_bf16<BN, EPI_BIAS_RESID_STATS, float, true>(a, b, M, N, K, epi, s)
                         : launch_bf16<BN, EPI_BIAS_RESID_STATS, float, false>(a, b, M, N, K, epi, s);
    case EPI_PATCH_STATS:
      return launch_bf16<BN, EPI_PATCH_STATS, float, true>(a, b, M, N, K, epi, s);
    case EPI_LN_BIAS:
      return launch_bf16<BN, EPI_LN_BIAS, __nv_bfloat16>(a, b, M, N, K, epi, s);
    case EPI_LN_GELU:
      return launch_bf16<BN, EPI_LN_GELU, __nv_bfloat16>(a, b, M, N, K, epi, s);
  }
  return TA_ERR_INVALID;
}

int gemm_bf16(const void* A, const void* W, int M, int N, int K, int epi_kind, bool out_bf16,
              const GemmEpi& epi_in, cudaStream_t stream, float* sk_ws) {
  static const int skip_epi = [] {
    // profiling only: 1 = mainloop + TMEM drain only, 2 = no TMA store
    const char* v = getenv("TA_GEMM_SKIP_EPILOGUE");
    return v ? atoi(v) : 0;
  }();
  static const int direct = [] {
    const char* v = getenv("TA_GEMM_STORE");
    return (v && v[0] == 'd') ? 1 : 0;
  }();
  static const int resid_ldg = [] {  // profiling: TA_GEMM_RESID=ldg reads the residual per thread
    const char* v = getenv("TA_GEMM_RESID");
    return (v && v[0] == 'l') ? 1 : 0;
  }();
  GemmEpi epi = epi_in;
  epi.skip = skip_epi;
  epi.direct_store = direct;
  epi.resid_ldg = resid_ldg;
  if (M <= 0) return TA_OK;
  if (K % kBK != 0 || N % 128 != 0) return TA_ERR_SHAPE;
  if ((epi_is_resid(epi_kind) || epi_is_patch(epi_kind)) && out_bf16) return TA_ERR_INVALID;
  if (epi_is_ln(epi_kind) && !out_bf16) return TA_ERR_INVALID;
  if (epi_is_ln(epi_kind) && epi_in.stat_slots > kMaxStatSlots) return TA_ERR_SHAPE;
  static const int force_bn = [] {  // profiling: TA_GEMM_BN=128 forces the 128 x 128 kernel
    const char* v = getenv("TA_GEMM_BN");
    return v ? atoi(v) : 0;
  }();
  // Tiny M x narrow N (ViT tail layers after merging, e.g. M = 256 x 11, N = 768): the 128 x 128
  // single-CTA kernel fills more SMs than 256 x 256 pair tiles (tools/gemm_small.py: proj 9.5 vs
  // 14.8 us, fc2 18.1 vs 25.4 us at M = 2816); everywhere else the pair kernel wins.
  static const int tiny_m = [] {  // profiling: TA_GEMM_TINY_M overrides the small-M threshold
    const char* v = getenv("TA_GEMM_TINY_M");
    return v ? atoi(v) : 3072;
  }();
  const bool tiny = M <= tiny_m && N <= 1024;
  const int BN = (force_bn == 128 || tiny) ? 128 : (N % 256 == 0) ? 256 : 128;
  if (epi_kind == EPI_BIAS_RESID_MERGE && !(BN == 256 && gemm_backend() == 0)) return TA_ERR_SHAPE;
  CUtensorMap ta_, tb_;
  int rc = make_tmap_bf16_2d(&ta_, A, M, K, kBM);
  if (rc) return rc;
  if (BN == 256 && gemm_backend() == 0) {
    rc = make_tmap_bf16_2d(&tb_, W, N, K, 128);  // each CTA of the pair loads 128 W rows
    if (rc) return rc;
    return dispatch_pair(ta_, tb_, M, N, K, epi_kind, out_bf16, epi, stream, sk_ws);
  }
  rc = make_tmap_bf16_2d(&tb_, W, N, K, BN);
  if (rc) return rc;
  return BN == 256 ? dispatch_bf16<256>(ta_, tb_, M, N, K, epi_kind, out_bf16, epi, stream)
                   : dispatch_bf16<128>(ta_, tb_, M, N, K, epi_kind, out_bf16, epi, stream);
}

// ------------------------------------------------------------------ fp32 mode on the tensor cores
// x = hi + lo with hi = tf32(x) and lo = tf32(x - hi), both rounded to nearest (cvt.rna), so
// the tensor core's tf32 read of either is exact and x - hi - lo = O(2^-22 |x|): the operand
// split of the 3xTF32 GEMM (kOp = 1), one pass over each operand.  (Truncating hi and lo, as
// the match kernel's normalised metric tolerates, leaves O(2^-20 |x|) and flipped a
// config-1 merge decision against the fp64 oracle.)
__device__ __forceinline__ float tf32_rna(float v) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(v));
  return __uint_as_float(r);
}
__global__ void __launch_bounds__(256) split_tf32_kernel(const float4* __restrict__ x, float4* __restrict__ hi,
                                                         float4* __restrict__ lo, long long n4) {
  grid_dep_wait();
  grid_dep_launch();
  auto tr = [](float v) { return tf32_rna(v); };
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n4;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const float4 v = x[i];
    const float4 h = make_float4(tr(v.x), tr(v.y), tr(v.z), tr(v.w));
    hi[i] = h;
    lo[i] = make_float4(tr(v.x - h.x), tr(v.y - h.y), tr(v.z - h.z), tr(v.w - h.w));
  }
}

static int split_tf32(const float* x, float* hi, float* lo, long long n, cudaStream_t s) {
  if (n % 4) return TA_ERR_SHAPE;
  const long long n4 = n / 4;
  cudaLaunchConfig_t cfg = {};
  const long long blocks = (n4 + 255) / 256;
  cfg.gridDim = dim3(static_cast<unsigned>(blocks < 4 * 148 ? blocks : 4 * 148));
  cfg.blockDim = dim3(256);
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled();
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  const cudaError_t e = cudaLaunchKernelEx(&cfg, split_tf32_kernel, reinterpret_cast<const float4*>(x),
                                           reinterpret_cast<float4*>(hi), reinterpret_cast<float4*>(lo), n4);
  return e == cudaSuccess ? TA_OK : set_last_cuda_error(e);
}

static int make_tmap_f32_2d(CUtensorMap* map, const void* base, uint64_t rows, uint64_t cols,
                            uint32_t box_rows) {
  auto enc = get_encode_fn();
  if (!enc) return TA_ERR_CUDA;
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {cols * 4};
  cuuint32_t box[2] = {32, box_rows};  // 32 fp32 = one 128-byte swizzle row
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void*>(base), dims, strides, box,
                   estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? TA_OK : TA_ERR_SHAPE;
}

size_t gemm_f32_tc_scratch_bytes(int M, int N, int K) {
  return (2ull * M * K + 2ull * N * K) * sizeof(float);
}

// fp32 mode: 3xTF32 tcgen05 GEMM (TA_F32_GEMM=simt selects the SIMT FFMA kernel instead).
int f32_gemm_backend() {
  static int mode = -1;
  if (mode < 0) {
    const char* v = getenv("TA_F32_GEMM");
    mode = (v && v[0] == 's') ? 1 : 0;
  }
  return mode;
}

int gemm_f32_tc(const float* A, const float* W, int M, int N, int K, int epi_kind, const GemmEpi& epi,
                void* scratch, cudaStream_t stream) {
  if (M <= 0) return TA_OK;
  if (K % 32 != 0 || N % 128 != 0 || !scratch) return TA_ERR_SHAPE;
  float* a_hi = static_cast<float*>(scratch);
  float* a_lo = a_hi + static_cast<size_t>(M) * K;
  float* w_hi = a_lo + static_cast<size_t>(M) * K;
  float* w_lo = w_hi + static_cast<size_t>(N) * K;
  TA_TRY_GEMM(split_tf32(A, a_hi, a_lo, static_cast<long long>(M) * K, stream));
  TA_TRY_GEMM(split_tf32(W, w_hi, w_lo, static_cast<long long>(N) * K, stream));
  CUtensorMap ta, tb, ta2, tb2;
  TA_TRY_GEMM(make_tmap_f32_2d(&ta, a_hi, M, K, kBM));
  TA_TRY_GEMM(make_tmap_f32_2d(&ta2, a_lo, M, K, kBM));
  TA_TRY_GEMM(make_tmap_f32_2d(&tb, w_hi, N, K, 128));
  TA_TRY_GEMM(make_tmap_f32_2d(&tb2, w_lo, N, K, 128));
  switch (epi_kind) {
    case EPI_BIAS:
      return launch_bf16<128, EPI_BIAS, float, false, 1>(ta, tb, M, N, K, epi, stream, &ta2, &tb2);
    case EPI_BIAS_GELU:
      return launch_bf16<128, EPI_BIAS_GELU, float, false, 1>(ta, tb, M, N, K, epi, stream, &ta2, &tb2);
    case EPI_BIAS_RESID:
      return epi.rows_in ? launch_bf16<128, EPI_BIAS_RESID, float, true, 1>(ta, tb, M, N, K, epi, stream, &ta2, &tb2)
                         : launch_bf16<128, EPI_BIAS_RESID, float, false, 1>(ta, tb, M, N, K, epi, stream, &ta2, &tb2);
    case EPI_PATCH:
      return launch_bf16<128, EPI_PATCH, float, true, 1>(ta, tb, M, N, K, epi, stream, &ta2, &tb2);
  }
  return TA_ERR_INVALID;
}

bool gemm_pair_path(int M, int N) {
  const char* v = getenv("TA_GEMM_BN");
  const bool force128 = v && atoi(v) == 128;
  const char* tv = getenv("TA_GEMM_TINY_M");
  const bool tiny = M <= (tv ? atoi(tv) : 3072) && N <= 1024;
  return !force128 && !tiny && N % 256 == 0 && gemm_backend() == 0;
}

int gemm_f32(const float* A, const float* W, int M, int N, int K, int epi_kind,
             const GemmEpi& epi, cudaStream_t stream) {
  if (M <= 0) return TA_OK;
  if (K % 8 != 0 || N % 128 != 0) return TA_ERR_SHAPE;
  dim3 grid(N / 128, (M + 127) / 128);
  switch (epi_kind) {
    case EPI_BIAS: gemm_f32_simt_kernel<EPI_BIAS><<<grid, 256, 0, stream>>>(A, W, M, N, K, epi); break;
    case EPI_BIAS_GELU: gemm_f32_simt_kernel<EPI_BIAS_GELU><<<grid, 256, 0, stream>>>(A, W, M, N, K, epi); break;
    case EPI_BIAS_RESID: gemm_f32_simt_kernel<EPI_BIAS_RESID><<<grid, 256, 0, stream>>>(A, W, M, N, K, epi); break;
    case EPI_PATCH: gemm_f32_simt_kernel<EPI_PATCH><<<grid, 256, 0, stream>>>(A, W, M, N, K, epi); break;
    default: return TA_ERR_INVALID;
  }
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? TA_OK : set_last_cuda_error(e);
}

}  // namespace ta
