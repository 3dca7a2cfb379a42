// Proportional attention, P kept in tensor memory (ToMe prop_attn,
// PAPER.md:534):  o = softmax(q k^T / sqrt(hd) + log size_j) v  per (image, head),
// head_dim 64, 64 < t <= 256 (ViT-B/16 and ViT-L/16 at gamma <= 0 and the early prompt layers).
//
// Why a second whole-row kernel: the trace of attention_tc.cu at t = 197 (profiles/r02_attn.md)
// shows each softmax group spending ~45 % of a tile on the exponentials and the rest waiting on
// the tensor pipe: for a P stage of the shared-memory P ring to be consumed (1.5k clk per tile),
// for the PV tail (1.9k) and for the next S (1.7k).  Here P never leaves TMEM:
//   * the softmax writes P (bf16 pairs) over the S columns it has already read (tcgen05.st), and
//     PV runs as tcgen05.mma with A = P from TMEM and B = V (MN-major SW128) from shared memory,
//     so there is no P ring to wait for and PV MMAs read 2 KB of shared memory per 16 keys
//     instead of 6 KB;
//   * O has its own columns of the tile's slot ([192, 256) when S fits in 192 columns, else
//     [128, 192), which the first PV MMA may only write once S block 2 has been read), so a tile
//     finishes when its last PV lands and its O is read, and the slot's next S follows at once.
//
// Persistent, warp-specialised, one CTA per SM, work item = (image, head), 1-2 query tiles of
// 128 rows per item; tile n of the CTA uses TMEM slot n % 2 (columns [256 s, 256 s + 256)) and
// softmax group n % 2 (warps 4g .. 4g+3; query row i = TMEM lane i).
//   warp 8 lane 0   TMA: K and V of an item (64-row SW128 boxes, 2-slot ring), Q per tile (2 slots)
//   warp 9 lane 0   MMA: S = Q K^T (N = round16(t)) into the tile's slot; PV per 64-key block as
//                   soon as its P is in TMEM, A = P [tmem], B = V
//   warps 0..7      pass 1 row max (raw scores), pass 2 p = size_j 2^(s scale - max) -> bf16 P
//                   into TMEM + row sum, epilogue O / sum -> bf16 via a per-warp smem slab + TMA.
#include <cfloat>

#include <cudaTypedefs.h>

#include "attn_softmax.cuh"
#include "common.h"
#include "ptx.cuh"

namespace ta {

int make_tmap_bf16_2d(CUtensorMap* map, const void* base, uint64_t rows, uint64_t cols,
                      uint32_t box_rows);
int make_tmap_attn_out(CUtensorMap* map, const void* base, uint64_t images, uint64_t t,
                       uint64_t cols);

namespace {

constexpr int kHd = 64;
constexpr int kQTile = 128;
constexpr int kKeyBlk = 64;
constexpr int kBlkBytes = kKeyBlk * kHd * 2;  // 8 KB: one 64-row SW128 box
constexpr int kQBytes = kQTile * kHd * 2;     // 16 KB
constexpr int kMaxT = 256;
constexpr int kThreads = 320;
constexpr int kSlabBytes = 4096;              // per softmax warp: two 2 KB O slabs

struct AttnTpLayout {
  int t_pad;     // round_up(t, 64)
  int t_mma;     // round_up(t, 16): S MMA N
  int n_kb;      // t_pad / 64
  int n_qt;      // ceil(t / 128)
  int nkc_last;  // 16-key PV steps of the last block
  int o_off;     // O columns inside a slot: 192 (t_mma <= 192) or 128
  int pv_gate;   // P block that must be in TMEM before the first PV MMA (O overwrites S block 2)
  uint32_t kv_off, slab_off, bias_off, bar_off, smem_bytes;
};

AttnTpLayout tp_layout(int t) {
  AttnTpLayout L{};
  L.t_pad = (t + kKeyBlk - 1) / kKeyBlk * kKeyBlk;
  L.t_mma = (t + 15) / 16 * 16;
  L.n_kb = L.t_pad / kKeyBlk;
  L.n_qt = (t + kQTile - 1) / kQTile;
  L.nkc_last = (t - (L.n_kb - 1) * kKeyBlk + 15) / 16;
  L.o_off = L.t_mma <= 192 ? 192 : 128;
  L.pv_gate = L.o_off == 128 ? 2 : 0;
  uint32_t off = 2 * kQBytes;  // Q: two slots
  L.kv_off = off;
  off += 2 * 2 * 4 * kBlkBytes;  // K/V ring: 2 slots x (K, V) x 4 blocks
  L.slab_off = off;
  off += 8 * kSlabBytes;
  L.bias_off = off;
  off += 2 * kMaxT * 4;
  L.bar_off = off;
  off += 32 * 8;
  L.smem_bytes = off + 1024;
  return L;
}

#ifdef TA_TP_TRACE  // profiling build only: per-event clock64 timeline of CTA 0 (tools/tp_trace.py)
__device__ unsigned long long g_tp_trace_t[16384];
__device__ unsigned int g_tp_trace_tag[16384];
#define TRACE(ev)                                                                      \
  do {                                                                                 \
    if (blockIdx.x == 0 && (threadIdx.x & 31) == 0 && tr_n < 1024u) {                  \
      const unsigned int k_ = (threadIdx.x >> 5) * 1024u + tr_n++;                     \
      g_tp_trace_t[k_] = clock64();                                                    \
      g_tp_trace_tag[k_] = (threadIdx.x >> 5) * 256u + (ev);                           \
    }                                                                                  \
  } while (0)
#define TRACE_DECL unsigned int tr_n = 0
#else
#define TRACE(ev) do {} while (0)
#define TRACE_DECL do {} while (0)
#endif

// D[tmem] (+)= A[tmem] * B[smem], kind::f16 (A = P, bf16 pairs per 32-bit column, K-major).
__device__ __forceinline__ void umma_f16_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t bdesc,
                                            uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(tmem_d),
      "r"(tmem_a), "l"(bdesc), "r"(idesc), "r"(accumulate));
}


// 64 keys of one query row -> 32 words of bf16 pairs (key 2c in the low half of word c, the
// K-major TMEM A layout).  `valid` < 64 (last block): keys >= valid get p = 0 (their scores are
// another image's keys or stale columns; masked before the exponential so no inf * 0).
template <bool kWeighted>
__device__ __forceinline__ void softmax_p64(uint32_t (&r)[64], uint64_t sc2, uint64_t nm2,
                                            uint32_t s_w, int valid, uint32_t (&p)[32],
                                            uint64_t (&acc)[2]) {
  if (valid < 64) {
#pragma unroll
    for (int j = 0; j < 64; ++j)
      if (j >= valid) r[j] = __float_as_uint(-INFINITY);
  }
#pragma unroll
  for (int chunk = 0; chunk < 8; ++chunk) {
    uint4 v;
    if (chunk * 8 >= valid) {
      v = make_uint4(0u, 0u, 0u, 0u);
    } else if (chunk & 1) {
      v = softmax_chunk8<TA_ATTN_POLY_ODD>(&r[chunk * 8], sc2, nm2, kWeighted || valid < 64, s_w + chunk * 32, acc);
    } else {
      v = softmax_chunk8<TA_ATTN_POLY_EVEN>(&r[chunk * 8], sc2, nm2, kWeighted || valid < 64, s_w + chunk * 32, acc);
    }
    p[4 * chunk] = v.x;
    p[4 * chunk + 1] = v.y;
    p[4 * chunk + 2] = v.z;
    p[4 * chunk + 3] = v.w;
  }
}

template <bool kHasSize>
__global__ void __launch_bounds__(kThreads, 1)
    attn_tp_kernel(const __grid_constant__ CUtensorMap tm, const __grid_constant__ CUtensorMap tmo,
                   const float* __restrict__ size, int t, int H, int n_items, float scale_log2,
                   AttnTpLayout L) {
  TRACE_DECL;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  const int D = H * kHd;
  uint8_t* sQ = smem;
  uint8_t* sKV = smem + L.kv_off;
  constexpr uint32_t kKvSlot = 2 * 4 * kBlkBytes;  // K blocks then V blocks
  float* bias = reinterpret_cast<float*>(smem + L.bias_off);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L.bar_off);
  uint64_t* kv_full = bars + 0;   // [2]
  uint64_t* kv_free = bars + 2;   // [2]
  uint64_t* q_full = bars + 4;    // [2]
  uint64_t* q_free = bars + 6;    // [2]
  uint64_t* s_full = bars + 8;    // [2] per slot
  uint64_t* s_free = bars + 10;   // [2] per slot: O read (and every PV done)
  uint64_t* o_full = bars + 12;   // [2] per slot
  uint64_t* p_full = bars + 14;   // [2][4] per slot and key block
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 24);

  const uint32_t warp = warp_id(), lane = lane_id();
  // items advance by gridDim.x as (b, h) pairs (no integer division in the loops)
  const int step_b = static_cast<int>(gridDim.x) / H;
  const int step_h = static_cast<int>(gridDim.x) - step_b * H;
  const int b_first = static_cast<int>(blockIdx.x) / H;
  const int h_first = static_cast<int>(blockIdx.x) - b_first * H;
  auto next_bh = [&](int& b, int& h) {
    b += step_b;
    h += step_h;
    if (h >= H) {
      h -= H;
      ++b;
    }
  };
  if (warp == 8 && lane == 0) {
    tma_prefetch(&tm);
    for (int s = 0; s < 2; ++s) {
      mbar_init(&kv_full[s], 1);
      mbar_init(&kv_free[s], 1);
      mbar_init(&q_full[s], 1);
      mbar_init(&q_free[s], 1);
      mbar_init(&s_full[s], 1);
      mbar_init(&s_free[s], 128);
      mbar_init(&o_full[s], 1);
      for (int k = 0; k < 4; ++k) mbar_init(&p_full[4 * s + k], 128);
    }
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  grid_dep_wait();    // qkv is the previous kernel's output
  grid_dep_launch();  // the next kernel's prologue may overlap our tail

  const int n_my = n_items > static_cast<int>(blockIdx.x)
                       ? (n_items - 1 - static_cast<int>(blockIdx.x)) / static_cast<int>(gridDim.x) + 1
                       : 0;
  const int T = n_my * L.n_qt;  // tiles of this CTA

  if (warp == 8) {
    // ------------------------------------------------------------ TMA producer
    if (lane == 0) {
      uint32_t it = 0, tile = 0;
      int b = b_first, h = h_first;
      for (int item = blockIdx.x; item < n_items; item += gridDim.x, ++it, next_bh(b, h)) {
        const int row_base = b * t;
        const int kvs = it & 1;
        mbar_wait(&kv_free[kvs], ((it >> 1) & 1) ^ 1);
        uint8_t* sK = sKV + kvs * kKvSlot;
        uint8_t* sV = sK + 4 * kBlkBytes;
        mbar_arrive_expect_tx(&kv_full[kvs], 2 * L.n_kb * kBlkBytes);
        for (int kb = 0; kb < L.n_kb; ++kb)
          tma_load_2d(&tm, &kv_full[kvs], sK + kb * kBlkBytes, D + h * kHd, row_base + kb * kKeyBlk);
        for (int kb = 0; kb < L.n_kb; ++kb)
          tma_load_2d(&tm, &kv_full[kvs], sV + kb * kBlkBytes, 2 * D + h * kHd, row_base + kb * kKeyBlk);
        for (int qt = 0; qt < L.n_qt; ++qt, ++tile) {
          const int qs = tile & 1;
          mbar_wait(&q_free[qs], ((tile >> 1) & 1) ^ 1);
          mbar_arrive_expect_tx(&q_full[qs], kQBytes);
          tma_load_2d(&tm, &q_full[qs], sQ + qs * kQBytes, h * kHd, row_base + qt * kQTile);
          tma_load_2d(&tm, &q_full[qs], sQ + qs * kQBytes + kBlkBytes, h * kHd, row_base + qt * kQTile + 64);
        }
      }
    }
  } else if (warp == 9) {
    // ------------------------------------------------------------ MMA issuer
    if (lane == 0) {
      const uint32_t idesc_s = idesc_bf16(kQTile, L.t_mma);
      constexpr uint32_t idesc_pv = idesc_bf16(kQTile, kHd, /*b_mn_major=*/true);
      int sN = 0, s_it = 0, s_qt = 0;      // next tile to get its S
      int pt[2] = {0, 1}, pkb[2] = {0, 0};  // per slot: current PV tile, next key block
      int p_it[2] = {0, L.n_qt == 1 ? 1 : 0};
      int p_qt[2] = {0, L.n_qt == 1 ? 0 : 1};
      int kv_tiles[2] = {0, 0};  // per K/V slot: tiles of its item whose PV is complete
      int pdone = 0;
      while (pdone < T) {
        if (sN < T) {
          const int slot = sN & 1;
          const int kvs = s_it & 1;
          if (mbar_test(&s_free[slot], ((sN >> 1) & 1) ^ 1) && mbar_test(&q_full[slot], (sN >> 1) & 1) &&
              (s_qt != 0 || mbar_test(&kv_full[kvs], (s_it >> 1) & 1))) {
            tc_fence_after();
            const uint64_t qdesc = umma_desc_sw128(smem_u32(sQ + slot * kQBytes));
            const uint64_t kdesc = umma_desc_sw128(smem_u32(sKV + kvs * kKvSlot));
#pragma unroll
            for (int k = 0; k < kHd / 16; ++k)
              umma_f16(tmem + slot * 256, qdesc + 2 * k, kdesc + 2 * k, idesc_s, k > 0);
            umma_commit(&s_full[slot]);
            umma_commit(&q_free[slot]);
            TRACE(4);
            ++sN;
            if (++s_qt == L.n_qt) {
              s_qt = 0;
              ++s_it;
            }
          }
        }
#pragma unroll
        for (int slot = 0; slot < 2; ++slot) {
          if (pt[slot] >= sN) continue;  // its S is not issued yet
          const int kb = pkb[slot];
          const uint32_t par = (pt[slot] >> 1) & 1;
          const int gate = kb == 0 ? L.pv_gate : kb;
          if (!mbar_test(&p_full[4 * slot + gate], par)) continue;
          TRACE(7 + 16 * slot);
          tc_fence_after();
          TRACE(8 + 16 * slot);
          const int kvs = p_it[slot] & 1;
          const uint32_t vbase = smem_u32(sKV + kvs * kKvSlot + 4 * kBlkBytes);
          const uint32_t o_tmem = tmem + slot * 256 + L.o_off;
          const int last = kb == 0 ? L.pv_gate : kb;  // blocks [kb, last] have their P now
          for (int k = kb; k <= last; ++k) {
            const int nkc = k == L.n_kb - 1 ? L.nkc_last : kKeyBlk / 16;
            for (int kc = 0; kc < nkc; ++kc) {
              // V rows (keys) are the K dimension: 16 keys = two 8-row groups = 2048 B
              const uint64_t vdesc = umma_desc_sw128_mn(vbase + k * kBlkBytes + kc * 2048, 8192, 1024);
#ifndef TA_TP_EXP_NOPV  // profiling only: TA_TP_EXP_NOPV drops the PV MMAs (wrong results)
              umma_f16_ts(o_tmem, tmem + slot * 256 + 32 * k + 8 * kc, vdesc, idesc_pv, (k | kc) != 0);
#endif
              TRACE(12 + 16 * slot);
            }
          }
          pkb[slot] = last + 1;
          TRACE(5 + 16 * slot);
          if (pkb[slot] == L.n_kb) {
            umma_commit(&o_full[slot]);
            TRACE(6 + 16 * slot);
            if (++kv_tiles[kvs] == L.n_qt) {  // every tile of the item has its PV issued
              umma_commit(&kv_free[kvs]);
              kv_tiles[kvs] = 0;
            }
            pt[slot] += 2;
            p_qt[slot] += 2;
            while (p_qt[slot] >= L.n_qt) {
              p_qt[slot] -= L.n_qt;
              ++p_it[slot];
            }
            pkb[slot] = 0;
            ++pdone;
          }
        }
      }
    }
  } else {
    // ------------------------------------------------------------ softmax / epilogue
    const int g = warp >> 2;
    const int i = (warp & 3) * 32 + lane;  // query row within the tile = TMEM lane
    const uint32_t la = tmem + (((warp & 3) * 32u) << 16) + g * 256;
    const uint32_t s_bias_g = smem_u32(bias) + g * kMaxT * 4;
    const uint32_t slab = smem_u32(smem + L.slab_off) + warp * kSlabBytes;
    const uint64_t sc2 = f2_pack(scale_log2, scale_log2);
    uint32_t k = 0;  // tiles processed by this group
    uint32_t tile = 0;
    int b = b_first, h = h_first;
    for (int item = blockIdx.x; item < n_items; item += gridDim.x, next_bh(b, h)) {
      const int row_base = b * t;
      bool have_bias = false;
      for (int qt = 0; qt < L.n_qt; ++qt, ++tile) {
        if (static_cast<int>(tile & 1) != g) continue;
        if (!have_bias) {
          TRACE(9);
          named_bar_sync(2 + g, 128);  // the group is done with the previous item's weights
          for (int j = i; j < L.t_pad; j += 128)
            sts_f32(s_bias_g + j * 4,
                    j < t ? (kHasSize ? size[static_cast<long long>(row_base) + j] : 1.f) : 0.f);
          named_bar_sync(2 + g, 128);
          have_bias = true;
        }
        const bool idle = qt * kQTile + static_cast<int>(warp & 3) * 32 >= t;  // no valid row
        mbar_wait(&s_full[g], k & 1);
        TRACE(10);
        tc_fence_after();
        // pass 1: row max of the raw scores over the valid keys
        float m4[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
        if (!idle)
          for (int kb = 0; kb < L.n_kb; ++kb) block_max(la + kb * 64, min(kKeyBlk, t - kb * kKeyBlk), m4);
        const float nmx = -fmaxf(fmaxf(m4[0], m4[1]), fmaxf(m4[2], m4[3])) * scale_log2;
        const uint64_t nm2 = f2_pack(nmx, nmx);
        TRACE(11);
        // pass 2: P blocks into TMEM over the S columns already read
        uint64_t acc[2] = {0ull, 0ull};
        for (int kb = 0; kb < L.n_kb; ++kb) {
          if (!idle) {
            uint32_t r[64];
            tmem_ld_32x32b_x32(la + kb * 64, *reinterpret_cast<uint32_t(*)[32]>(&r[0]));
            tmem_ld_32x32b_x32(la + kb * 64 + 32, *reinterpret_cast<uint32_t(*)[32]>(&r[32]));
            tmem_ld_wait();
            uint32_t p[32];
            const int valid = min(kKeyBlk, t - kb * kKeyBlk);
            softmax_p64<kHasSize>(r, sc2, nm2, s_bias_g + kb * 64 * 4, valid, p, acc);
#ifndef TA_TP_EXP_NOST  // profiling only: TA_TP_EXP_NOST drops the P stores (wrong results)
            tmem_st_32x32b_x32(la + 32 * kb, p);
            tmem_st_wait();
#else
            if (p[0] == 0x12345678u) acc[0] = 0;
#endif
          }
          tc_fence_before();
          mbar_arrive(&p_full[4 * g + kb]);
          TRACE(14);
        }
        const float inv = rcp_approx(f2_total(acc));
        // epilogue: O / sum -> bf16 rows
        mbar_wait(&o_full[g], k & 1);
        TRACE(17);
        tc_fence_after();
        uint32_t o0[32], o1[32];
        tmem_ld_32x32b_x32(la + L.o_off, o0);
        tmem_ld_32x32b_x32(la + L.o_off + 32, o1);
        tmem_ld_wait();
        tc_fence_before();
        mbar_arrive(&s_free[g]);  // the slot may take the next S
        const int q0 = qt * kQTile + static_cast<int>(warp & 3) * 32;
        if (q0 < t) {
          if (lane == 0) bulk_wait_group_read<0>();  // this warp's previous O slabs are read
          __syncwarp();
          store_o_slab(&tmo, o0, inv, slab, lane, h * kHd, q0, b);
          store_o_slab(&tmo, o1, inv, slab + 2048, lane, h * kHd + 32, q0, b);
        }
        TRACE(18);
        ++k;
      }
    }
    if (lane == 0) bulk_wait_group<0>();  // O stores complete before the CTA exits
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

template <bool kHasSize>
cudaError_t launch_tp(const cudaLaunchConfig_t& cfg, const CUtensorMap& tm, const CUtensorMap& tmo,
                      const float* size, int t, int H, int n_items, float scale_log2, const AttnTpLayout& L) {
  static unsigned long long attr_mask = 0;  // per instantiation and device
  if (attr_needed(attr_mask)) {
    const cudaError_t e = cudaFuncSetAttribute(attn_tp_kernel<kHasSize>,
                                               cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    if (e != cudaSuccess) return e;
    attr_done(attr_mask);
  }
  return cudaLaunchKernelEx(&cfg, attn_tp_kernel<kHasSize>, tm, tmo, size, t, H, n_items, scale_log2, L);
}

}  // namespace

// TA_ERR_SHAPE outside the kernel's envelope (hd != 64, t <= 64 or t > 256): the caller then
// uses another kernel.
int attention_tp(const void* qkv, const float* size, int B, int t, int H, int hd, void* out,
                 cudaStream_t s) {
  if (hd != kHd || t <= 64 || t > kMaxT) return TA_ERR_SHAPE;
  const AttnTpLayout L = tp_layout(t);
  if (L.smem_bytes > 227u * 1024) return TA_ERR_SHAPE;
  CUtensorMap tm, tmo;
  int rc = make_tmap_bf16_2d(&tm, qkv, static_cast<uint64_t>(B) * t, 3ull * H * hd, 64);
  if (rc) return rc;
  rc = make_tmap_attn_out(&tmo, out, B, t, static_cast<uint64_t>(H) * hd);
  if (rc) return rc;
  const int n_items = B * H;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(n_items < device_sm_count() ? n_items : device_sm_count());
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = L.smem_bytes;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled();
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  const float scale_log2 = 1.4426950408889634f / sqrtf(static_cast<float>(hd));
  const cudaError_t e = size != nullptr ? launch_tp<true>(cfg, tm, tmo, size, t, H, n_items, scale_log2, L)
                                        : launch_tp<false>(cfg, tm, tmo, size, t, H, n_items, scale_log2, L);
  return e == cudaSuccess ? TA_OK : set_last_cuda_error(e);
}

#ifdef TA_TP_TRACE
extern "C" __attribute__((visibility("default"))) int ta_debug_tp_trace(unsigned long long* t,
                                                                      unsigned int* tag, int max,
                                                                      int reset) {
  static unsigned int zeros[16384];
  if (reset) return cudaMemcpyToSymbol(g_tp_trace_tag, zeros, sizeof(zeros)) == cudaSuccess ? 0 : -1;
  cudaDeviceSynchronize();
  const int n = max < 16384 ? max : 16384;
  cudaMemcpyFromSymbol(t, g_tp_trace_t, n * sizeof(unsigned long long));
  cudaMemcpyFromSymbol(tag, g_tp_trace_tag, n * sizeof(unsigned int));
  return n;
}
#endif
}  // namespace ta
