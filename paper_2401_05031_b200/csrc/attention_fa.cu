// Proportional attention, chunk-pipelined on the 5th-gen tensor cores (SURVEY.md §8a row a6,
// north_star 3):  o = softmax(q k^T / sqrt(hd) + log size_j) v   per (image, head), hd = 64.
//
// Persistent, warp-specialised, one CTA per SM, 20 warps.  The CTA walks its (image, head)
// items; their 128-row query tiles alternate between two groups, so two tiles are in flight,
// and every tile streams its keys in 64-key chunks:
//   warps 16, 17 (TMA)   producer of group 0 / 1: with a size vector the warp stages the tile's
//                        key weights w_j = size_j (0 past t) in a double-buffered array; lane 0
//                        loads Q (128 x 64) and per chunk K_j, V_j (64 x 64 SW128 boxes) into
//                        2-stage rings.
//   warps 18, 19 (MMA)   issuer of group 0 / 1, program order S(c), PV(c - 1) over the group's
//                        chunk stream: S_c = Q K_c^T (M = 128, N <= 64) into one of two 64-column
//                        TMEM S stages; O_a += P_c[:, 0:32] V_c[0:32], O_b += P_c[:, 32:64]
//                        V_c[32:64] (V as MN-major B) into two 64-column TMEM accumulators.
//   warps 0..15          softmax, 4 per SM sub-partition: warp w owns TMEM lanes 32 (w % 4)..
//                        (query rows), half h = (w / 4) % 2 of every chunk's keys, group w / 8.
//                        Each half keeps its own lazily updated reference max m_h (raised only
//                        when a chunk's max exceeds it by more than 2^8, then O_h and the half's
//                        row sum are rescaled in place) and row sum s_h, so the two halves of a
//                        row never synchronise inside a tile; the epilogue combines them:
//                        o = (O_a 2^(m_a - M) + O_b 2^(m_b - M)) / (s_a 2^(m_a - M) + s_b 2^(m_b - M)),
//                        each half writing 32 of the 64 output columns straight from registers.
// TMEM (512 columns): group g owns [256 g, 256 g + 256): S stages at +0 / +64, O_a at +128,
// O_b at +192.  Keys past t inside the last chunk are masked to -inf (their scores come from
// the next image's rows or TMA zero fill), so p = 0 there.
#include <cfloat>
#include <cstdlib>

#include <cudaTypedefs.h>

#include "attn_softmax.cuh"
#include "common.h"
#include "ptx.cuh"

namespace ta {

int make_tmap_bf16_2d(CUtensorMap* map, const void* base, uint64_t rows, uint64_t cols,
                      uint32_t box_rows);

namespace {

#ifdef TA_ATTN_TRACE  // profiling build only: per-event clock64 timeline of CTA 0
__device__ unsigned long long g_fa_trace_t[16384];
__device__ unsigned int g_fa_trace_tag[16384];
#define TRACE(ev)                                                                      \
  do {                                                                                 \
    if (blockIdx.x == 0 && (threadIdx.x & 31) == 0 && tr_n < 1024u) {                  \
      const unsigned int k_ = (threadIdx.x >> 5) * 1024u + tr_n++;                     \
      g_fa_trace_t[k_] = clock64();                                                    \
      g_fa_trace_tag[k_] = (threadIdx.x >> 5) * 256u + (ev);                           \
    }                                                                                  \
  } while (0)
#define TRACE_DECL unsigned int tr_n = 0
#else
#define TRACE(ev) do {} while (0)
#define TRACE_DECL do {} while (0)
#endif

constexpr int kHd = 64;
constexpr int kQTile = 128;
constexpr int kChunk = 64;
constexpr uint32_t kChunkBytes = kChunk * kHd * 2;  // 8 KB: one 64-row SW128 box
constexpr uint32_t kQBytes = kQTile * kHd * 2;      // 16 KB
constexpr uint32_t kPBytes = kQTile * kChunk * 2;   // 16 KB
constexpr int kKv = 2;                              // K and V ring stages per group
constexpr int kS = 2;                               // TMEM S stages per group
constexpr int kSoftmaxWarps = 16;
constexpr int kThreads = (kSoftmaxWarps + 4) * 32;  // + 2 producers + 2 MMA issuers
constexpr int kMaxT = 4096;

struct FaLayout {
  int n_ch;      // ceil(t / 64) key chunks
  int rem;       // keys in the last chunk (1..64)
  int n_last;    // S MMA N of the last chunk: round_up(rem, 16)
  int nkc_a;     // 16-key PV steps of the last chunk for half a (keys 0..31): 1..2
  int nkc_b;     // ... for half b (keys 32..63): 1..2 (>= 1 so O_b is always initialised)
  int n_qt;      // ceil(t / 128)
  int t_pad;     // 64 n_ch
  uint32_t q_off, k_off, v_off, p_off, w_off, x_off, bar_off, smem_bytes;
};

FaLayout fa_layout(int t) {
  FaLayout L{};
  L.n_ch = (t + kChunk - 1) / kChunk;
  L.rem = t - (L.n_ch - 1) * kChunk;
  L.n_last = (L.rem + 15) / 16 * 16;
  const int nkc = L.n_last / 16;
  L.nkc_a = nkc < 2 ? nkc : 2;
  L.nkc_b = nkc > 3 ? 2 : (nkc > 2 ? 1 : 1);
  L.n_qt = (t + kQTile - 1) / kQTile;
  L.t_pad = L.n_ch * kChunk;
  uint32_t off = 0;
  L.q_off = off;
  off += 2 * kQBytes;
  L.k_off = off;
  off += 2 * kKv * kChunkBytes;
  L.v_off = off;
  off += 2 * kKv * kChunkBytes;
  L.p_off = off;
  off += 4 * kPBytes;
  L.w_off = off;
  off += 4 * L.t_pad * 4;  // key weights: 2 buffers per group
  L.x_off = off;
  off += 2 * 2 * 2 * 128 * 8;  // epilogue exchange: [tile parity][group][half][row] (m, s)
  L.bar_off = (off + 7) / 8 * 8;
  off = L.bar_off + 80 * 8;
  L.smem_bytes = off + 1024;
  return L;
}

// Barrier block (uint64 each), per group g.
struct Bars {
  uint64_t* base;
  __device__ uint64_t* q_full(int g) { return base + g; }
  __device__ uint64_t* q_free(int g) { return base + 2 + g; }
  __device__ uint64_t* k_full(int g, int s) { return base + 4 + g * kKv + s; }
  __device__ uint64_t* k_free(int g, int s) { return base + 8 + g * kKv + s; }
  __device__ uint64_t* v_full(int g, int s) { return base + 12 + g * kKv + s; }
  __device__ uint64_t* v_free(int g, int s) { return base + 16 + g * kKv + s; }
  __device__ uint64_t* s_full(int g, int s) { return base + 20 + g * kS + s; }
  __device__ uint64_t* s_free(int g, int s) { return base + 24 + g * kS + s; }
  __device__ uint64_t* p_full(int g, int s, int h) { return base + 28 + g * 4 + s * 2 + h; }
  __device__ uint64_t* p_free(int g, int s, int h) { return base + 36 + g * 4 + s * 2 + h; }
  __device__ uint64_t* o_full(int g) { return base + 44 + g; }
  __device__ uint64_t* o_free(int g) { return base + 46 + g; }
  __device__ uint64_t* w_full(int g, int s) { return base + 48 + g * 2 + s; }
  __device__ uint64_t* w_free(int g, int s) { return base + 52 + g * 2 + s; }
  __device__ uint32_t* tmem_slot() { return reinterpret_cast<uint32_t*>(base + 56); }
};

struct Ring {
  uint32_t stage = 0, phase = 0;
  __device__ void next(uint32_t n) {
    if (++stage == n) {
      stage = 0;
      phase ^= 1u;
    }
  }
};

struct TileIter {
  int k, qt, b, h;
  int step_b, step_h, H, n_qt;
  __device__ void init(int g, int H_, int n_qt_) {
    H = H_;
    n_qt = n_qt_;
    step_b = static_cast<int>(gridDim.x) / H;
    step_h = static_cast<int>(gridDim.x) - step_b * H;
    b = static_cast<int>(blockIdx.x) / H;
    h = static_cast<int>(blockIdx.x) - b * H;
    k = 0;
    qt = 0;
    advance(g);
  }
  __device__ void advance(int n) {  // n tiles forward
    qt += n;
    while (qt >= n_qt) {
      qt -= n_qt;
      ++k;
      b += step_b;
      h += step_h;
      if (h >= H) {
        h -= H;
        ++b;
      }
    }
  }
};


// One half-chunk (32 keys) of a query row: p = w 2^(s scale - m) for its first nz 8-key groups,
// bf16 P into the SW128 row (16-byte group c at slot c ^ (row & 7), c = 4 h + cc); kTrackMax
// also folds the raw scores' max into m4 (the lazy-rescale check).
template <bool kTrackMax>
__device__ __forceinline__ void fa_half(const uint32_t (&r)[32], int nz, int h, uint64_t sc2,
                                        uint64_t nm2, bool weighted, uint32_t s_w, uint32_t s_prow,
                                        int row, uint64_t (&acc)[2], float (&m4)[4]) {
#pragma unroll
  for (int cc = 0; cc < 4; ++cc) {
    if (cc < nz) {
      if (kTrackMax) {
#pragma unroll
        for (int e = 0; e < 8; ++e) m4[e & 3] = fmaxf(m4[e & 3], __uint_as_float(r[cc * 8 + e]));
      }
      const uint4 v = (cc & 1) ? softmax_chunk8<TA_ATTN_POLY_ODD>(&r[cc * 8], sc2, nm2, weighted, s_w + cc * 32, acc)
                               : softmax_chunk8<TA_ATTN_POLY_EVEN>(&r[cc * 8], sc2, nm2, weighted, s_w + cc * 32, acc);
      sts_u4(s_prow + (((4 * h + cc) ^ (row & 7)) << 4), v);
    }
  }
}

template <bool kHasSize>
__global__ void __launch_bounds__(kThreads, 1)
    attn_fa_kernel(const __grid_constant__ CUtensorMap tm, __nv_bfloat16* __restrict__ out,
                   const float* __restrict__ size, int t, int H, int n_items, float scale_log2,
                   FaLayout L) {
  TRACE_DECL;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  const int D = H * kHd;
  Bars bars{reinterpret_cast<uint64_t*>(smem + L.bar_off)};
  const uint32_t warp = warp_id(), lane = lane_id();

  // tiles of this CTA: items blockIdx.x + k gridDim.x < n_items, n_qt tiles each
  const int n_my = n_items > static_cast<int>(blockIdx.x)
                       ? (n_items - 1 - static_cast<int>(blockIdx.x)) / static_cast<int>(gridDim.x) + 1
                       : 0;
  const int T = n_my * L.n_qt;

  if (warp == kSoftmaxWarps && lane == 0) {
    tma_prefetch(&tm);
    for (int g = 0; g < 2; ++g) {
      mbar_init(bars.q_full(g), 1);
      mbar_init(bars.q_free(g), 1);
      for (int s = 0; s < kKv; ++s) {
        mbar_init(bars.k_full(g, s), 1);
        mbar_init(bars.k_free(g, s), 1);
        mbar_init(bars.v_full(g, s), 1);
        mbar_init(bars.v_free(g, s), 1);
      }
      for (int s = 0; s < kS; ++s) {
        mbar_init(bars.s_full(g, s), 1);
        mbar_init(bars.s_free(g, s), 256);
      }
      for (int s = 0; s < 2; ++s)
        for (int h = 0; h < 2; ++h) {
          mbar_init(bars.p_full(g, s, h), 128);
          mbar_init(bars.p_free(g, s, h), 1);
        }
      mbar_init(bars.o_full(g), 1);
      mbar_init(bars.o_free(g), 256);
      for (int s = 0; s < 2; ++s) {
        mbar_init(bars.w_full(g, s), 32);
        mbar_init(bars.w_free(g, s), 256);
      }
    }
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc<512>(bars.tmem_slot());
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *bars.tmem_slot();

  grid_dep_wait();    // qkv is the previous kernel's output
  grid_dep_launch();  // the next kernel's prologue overlaps our tail

  if (warp == kSoftmaxWarps || warp == kSoftmaxWarps + 1) {
    // ------------------------------------------------------------ TMA producer of group g
    const int g = static_cast<int>(warp) - kSoftmaxWarps;
    uint8_t* sQ = smem + L.q_off + g * kQBytes;
    TileIter it;
    it.init(g, H, L.n_qt);
    Ring kv;
    uint32_t n = 0;
    for (int c = g; c < T; c += 2, ++n, it.advance(2)) {
      const int row_base = it.b * t;
      if (kHasSize) {
        const uint32_t wb = n & 1;
        mbar_wait(bars.w_free(g, wb), ((n >> 1) & 1) ^ 1);
        const uint32_t s_w = smem_u32(smem + L.w_off) + (2 * g + wb) * L.t_pad * 4;
        for (int j = static_cast<int>(lane); j < L.t_pad; j += 32)
          sts_f32(s_w + j * 4, j < t ? __ldg(size + row_base + j) : 0.f);
        mbar_arrive(bars.w_full(g, wb));  // every writer lane releases its own stores
      }
      if (lane == 0) {
        mbar_wait(bars.q_free(g), (n & 1) ^ 1);
        mbar_arrive_expect_tx(bars.q_full(g), kQBytes);
        tma_load_2d(&tm, bars.q_full(g), sQ, it.h * kHd, row_base + it.qt * kQTile);
        tma_load_2d(&tm, bars.q_full(g), sQ + kChunkBytes, it.h * kHd, row_base + it.qt * kQTile + 64);
        TRACE(1);
        for (int j = 0; j < L.n_ch; ++j, kv.next(kKv)) {
          uint8_t* sK = smem + L.k_off + (g * kKv + kv.stage) * kChunkBytes;
          uint8_t* sV = smem + L.v_off + (g * kKv + kv.stage) * kChunkBytes;
          mbar_wait(bars.k_free(g, kv.stage), kv.phase ^ 1);
          mbar_arrive_expect_tx(bars.k_full(g, kv.stage), kChunkBytes);
          tma_load_2d(&tm, bars.k_full(g, kv.stage), sK, D + it.h * kHd, row_base + j * kChunk);
          TRACE(2);
          mbar_wait(bars.v_free(g, kv.stage), kv.phase ^ 1);
          mbar_arrive_expect_tx(bars.v_full(g, kv.stage), kChunkBytes);
          tma_load_2d(&tm, bars.v_full(g, kv.stage), sV, 2 * D + it.h * kHd, row_base + j * kChunk);
          TRACE(3);
        }
      }
      __syncwarp();
    }
  } else if (warp == kSoftmaxWarps + 2 || warp == kSoftmaxWarps + 3) {
    // ------------------------------------------------------------ MMA issuer of group g
    // Program order over the group's chunk stream c (all its tiles back to back): S(c), then
    // PV(c - 1).  No wait can deadlock: S(c) needs the softmax to have loaded S(c - 2) (before
    // it writes P(c - 2)), PV(c - 1) needs P(c - 1), whose S was issued before.
    const int g = static_cast<int>(warp) - kSoftmaxWarps - 2;
    if (lane == 0) {
      constexpr uint32_t idesc_pv = idesc_bf16(kQTile, kHd, /*b_mn_major=*/true);
      const uint32_t idesc_s = idesc_bf16(kQTile, kChunk);
      const uint32_t idesc_s_last = idesc_bf16(kQTile, L.n_last);
      const int n_tiles = (T - g + 1) / 2;
      const int C = n_tiles * L.n_ch;
      const uint64_t qdesc = umma_desc_sw128(smem_u32(smem + L.q_off + g * kQBytes));
      const uint32_t s_tmem0 = tmem + g * 256;
      Ring ss, ks, ps, vs;
      int s_j = 0, s_tile = 0;  // chunk / tile of the next S
      int p_j = 0, p_tile = 0;  // chunk / tile of the next PV
      for (int c = 0; c < C + 1; ++c) {
        if (c < C) {
          if (s_j == 0) mbar_wait(bars.q_full(g), s_tile & 1);
          mbar_wait(bars.k_full(g, ks.stage), ks.phase);
          mbar_wait(bars.s_free(g, ss.stage), ss.phase ^ 1);
          tc_fence_after();
          const uint64_t kdesc = umma_desc_sw128(smem_u32(smem + L.k_off + (g * kKv + ks.stage) * kChunkBytes));
          const uint32_t id = s_j == L.n_ch - 1 ? idesc_s_last : idesc_s;
#pragma unroll
          for (int k = 0; k < kHd / 16; ++k)
            umma_f16(s_tmem0 + ss.stage * 64, qdesc + 2 * k, kdesc + 2 * k, id, k > 0);
          TRACE(30 + g);
          umma_commit(bars.s_full(g, ss.stage));
          umma_commit(bars.k_free(g, ks.stage));
          ss.next(kS);
          ks.next(kKv);
          if (++s_j == L.n_ch) {
            umma_commit(bars.q_free(g));
            s_j = 0;
            ++s_tile;
          }
        }
        if (c >= 1) {
          if (p_j == 0) mbar_wait(bars.o_free(g), (p_tile & 1) ^ 1);
          mbar_wait(bars.v_full(g, vs.stage), vs.phase);
          const uint64_t pdesc = umma_desc_sw128(smem_u32(smem + L.p_off + (2 * g + ps.stage) * kPBytes));
          const uint32_t vbase = smem_u32(smem + L.v_off + (g * kKv + vs.stage) * kChunkBytes);
          const bool last = p_j == L.n_ch - 1;
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            mbar_wait(bars.p_full(g, ps.stage, h), ps.phase);
            tc_fence_after();
            const int nk = last ? (h ? L.nkc_b : L.nkc_a) : 2;
            const uint32_t o_tmem = tmem + g * 256 + 128 + 64 * h;
#pragma unroll
            for (int kc = 0; kc < 2; ++kc) {
              if (kc >= nk) break;
              const int ks16 = 2 * h + kc;  // 16-key step within the chunk
              // V rows (keys) are the K dimension: 16 keys = two 8-row groups = 2048 B.
              const uint64_t vdesc = umma_desc_sw128_mn(vbase + ks16 * 2048, 8192, 1024);
              umma_f16(o_tmem, pdesc + 2 * ks16, vdesc, idesc_pv, (p_j | kc) != 0);
            }
            umma_commit(bars.p_free(g, ps.stage, h));
          }
          TRACE(20 + g);
          umma_commit(bars.v_free(g, vs.stage));
          ps.next(2);
          vs.next(kKv);
          if (++p_j == L.n_ch) {
            umma_commit(bars.o_full(g));
            p_j = 0;
            ++p_tile;
          }
        }
      }
    }
  } else {
    // ------------------------------------------------------------ softmax / epilogue
    const int quarter = static_cast<int>(warp) & 3;
    const int h = (static_cast<int>(warp) >> 2) & 1;  // key half of every chunk
    const int g = static_cast<int>(warp) >> 3;
    const int i = quarter * 32 + static_cast<int>(lane);  // query row within the tile
    const uint32_t la = tmem + ((static_cast<uint32_t>(quarter) * 32u) << 16) + g * 256;
    const uint32_t o_own = la + 128 + 64 * h, o_oth = la + 128 + 64 * (h ^ 1);
    const uint32_t s_w0 = smem_u32(smem + L.w_off) + 2 * g * L.t_pad * 4;
    const uint32_t s_p0 = smem_u32(smem + L.p_off) + 2 * g * kPBytes;
    const uint32_t s_x0 = smem_u32(smem + L.x_off) + (g * 2 * 128 + i) * 8;  // + parity, half
    const uint64_t sc2 = f2_pack(scale_log2, scale_log2);
    const int nz_last = 2 * (h ? L.nkc_b : L.nkc_a);
    Ring ss, ps;
    // deferred epilogue of the previous tile
    bool pend = false;
    int pend_b = 0, pend_h = 0, pend_qt = 0;
    uint32_t pend_n = 0;
    float pend_m = 0.f, pend_s = 0.f;

    auto epilogue = [&]() {
      TRACE(15);
      mbar_wait(bars.o_full(g), pend_n & 1);
      TRACE(16);
      tc_fence_after();
      // exchange (m, s) with the other half of the row
      const uint32_t xs = s_x0 + (pend_n & 1) * (2 * 2 * 128 * 8);
      sts_f32(xs + h * 128 * 8, pend_m);
      sts_f32(xs + h * 128 * 8 + 4, pend_s);
      named_bar_sync(1 + g * 4 + quarter, 64);
      const float m_o = lds_f32(xs + (h ^ 1) * 128 * 8), s_o = lds_f32(xs + (h ^ 1) * 128 * 8 + 4);
      const int q0 = pend_qt * kQTile + quarter * 32;
      const int q = q0 + static_cast<int>(lane);
      const float M = fmaxf(pend_m, m_o);
      const float fo = ex2_approx(pend_m - M), fx = ex2_approx(m_o - M);
      const float inv = rcp_approx(pend_s * fo + s_o * fx);
      const float a = fo * inv, bsc = fx * inv;
      __nv_bfloat16* dst = out + (static_cast<long long>(pend_b) * t + q) * D + pend_h * kHd + 32 * h;
#pragma unroll 1
      for (int half16 = 0; half16 < 2; ++half16) {
        uint32_t oa[16], ob[16];
        if (q0 < t) {
          tmem_ld_32x32b_x16(o_own + 32 * h + 16 * half16, oa);
          tmem_ld_32x32b_x16(o_oth + 32 * h + 16 * half16, ob);
          tmem_ld_wait();
        }
        if (half16 == 1) {
          tc_fence_before();
          mbar_arrive(bars.o_free(g));
        }
        if (q < t) {
#pragma unroll
          for (int c4 = 0; c4 < 2; ++c4) {
            uint32_t w[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const int k = 8 * c4 + 2 * e;
              w[e] = pack_bf16(__uint_as_float(oa[k]) * a + __uint_as_float(ob[k]) * bsc,
                               __uint_as_float(oa[k + 1]) * a + __uint_as_float(ob[k + 1]) * bsc);
            }
            reinterpret_cast<uint4*>(dst)[2 * half16 + c4] = make_uint4(w[0], w[1], w[2], w[3]);
          }
        }
      }
      TRACE(17);
      pend = false;
    };

    TileIter it;
    it.init(g, H, L.n_qt);
    uint32_t n = 0;
    for (int c = g; c < T; c += 2, ++n, it.advance(2)) {
      const uint32_t s_bias = s_w0 + (n & 1) * L.t_pad * 4 + 32 * h * 4;
      if (kHasSize) mbar_wait(bars.w_full(g, n & 1), (n >> 1) & 1);
      const bool idle = it.qt * kQTile + quarter * 32 >= t;
      float m = 0.f;  // reference max of this half (log2 domain)
      uint64_t acc[2] = {0ull, 0ull};
      for (int j = 0; j < L.n_ch; ++j) {
        const bool last = j == L.n_ch - 1;
        const int valid = (last ? L.rem : kChunk) - 32 * h;  // valid keys of this half (may be <= 0)
        uint32_t r[32];
        TRACE(10);
        mbar_wait(bars.s_full(g, ss.stage), ss.phase);
        TRACE(11);
        tc_fence_after();
        if (!idle && valid > 0) {
          tmem_ld_32x32b_x32(la + ss.stage * 64 + 32 * h, r);
          tmem_ld_wait();
        }
        tc_fence_before();
        mbar_arrive(bars.s_free(g, ss.stage));
        ss.next(kS);
        const int nz = last ? nz_last : 4;
        if (!idle) {
          if (valid < 32) {
#pragma unroll
            for (int e = 0; e < 32; ++e)
              if (e >= valid) r[e] = 0xff800000u;  // -inf: p = 0
          }
          if (j == 0) {  // first chunk of the tile: its max is the reference
            float m4[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
            for (int e = 0; e < 32; e += 4) {
              m4[0] = fmaxf(m4[0], __uint_as_float(r[e]));
              m4[1] = fmaxf(m4[1], __uint_as_float(r[e + 1]));
              m4[2] = fmaxf(m4[2], __uint_as_float(r[e + 2]));
              m4[3] = fmaxf(m4[3], __uint_as_float(r[e + 3]));
            }
            const float cm = fmaxf(fmaxf(m4[0], m4[1]), fmaxf(m4[2], m4[3]));
            m = cm == -INFINITY ? 0.f : cm * scale_log2;  // a half with no key yet: any finite m
          }
        }
        TRACE(12);
        mbar_wait(bars.p_free(g, ps.stage, h), ps.phase ^ 1);
        TRACE(13);
        if (!idle) {
          const uint32_t s_prow = s_p0 + ps.stage * kPBytes + i * 128;
          const uint32_t s_w = s_bias + j * kChunk * 4;
          const uint64_t acc_in[2] = {acc[0], acc[1]};
          float m4[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
          fa_half<true>(r, nz, h, sc2, f2_pack(-m, -m), kHasSize, s_w, s_prow, i, acc, m4);
          const float cm = fmaxf(fmaxf(m4[0], m4[1]), fmaxf(m4[2], m4[3])) * scale_log2;
          if (j > 0 && __any_sync(0xffffffffu, cm > m + 8.f)) {
            // rare: a key exceeds the reference max by more than 2^8: raise the reference,
            // rescale O_h and the half's row sum, redo this chunk's P.  The tile's previous
            // PVs into O_h must have completed (PV of the previous use of this half).
            const bool up = cm > m + 8.f;
            const float f = up ? ex2_approx(m - cm) : 1.f;
            if (up) m = cm;
            mbar_wait(bars.p_free(g, ps.stage ^ 1, h), ps.stage == 1 ? ps.phase : ps.phase ^ 1);
            tc_fence_after();
#pragma unroll 1
            for (int q4 = 0; q4 < 4; ++q4) {
              uint32_t o[16];
              tmem_ld_32x32b_x16(o_own + 16 * q4, o);
              tmem_ld_wait();
#pragma unroll
              for (int e = 0; e < 16; ++e) o[e] = __float_as_uint(__uint_as_float(o[e]) * f);
              tmem_st_32x32b_x16(o_own + 16 * q4, o);
            }
            tmem_st_wait();
            const uint64_t f2 = f2_pack(f, f);
            acc[0] = fmul2(acc_in[0], f2);
            acc[1] = fmul2(acc_in[1], f2);
            fa_half<false>(r, nz, h, sc2, f2_pack(-m, -m), kHasSize, s_w, s_prow, i, acc, m4);
          }
          fence_proxy_async_smem();
        }
        tc_fence_before();
        mbar_arrive(bars.p_full(g, ps.stage, h));
        TRACE(14);
        ps.next(2);
        if (j == 0 && pend) epilogue();
      }
      if (kHasSize) mbar_arrive(bars.w_free(g, n & 1));
      pend = true;
      pend_b = it.b;
      pend_h = it.h;
      pend_qt = it.qt;
      pend_n = n;
      pend_m = m;
      pend_s = f2_total(acc);
    }
    if (pend) epilogue();
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

}  // namespace

#ifdef TA_ATTN_TRACE
extern "C" __attribute__((visibility("default"))) int ta_debug_fa_trace(unsigned long long* t,
                                                                      unsigned int* tag, int max,
                                                                      int reset) {
  static unsigned int zeros[16384];
  if (reset) return cudaMemcpyToSymbol(g_fa_trace_tag, zeros, sizeof(zeros)) == cudaSuccess ? 0 : -1;
  cudaDeviceSynchronize();
  const int n = max < 16384 ? max : 16384;
  cudaMemcpyFromSymbol(t, g_fa_trace_t, n * sizeof(unsigned long long));
  cudaMemcpyFromSymbol(tag, g_fa_trace_tag, n * sizeof(unsigned int));
  return n;
}
#endif

// Returns TA_ERR_SHAPE outside the kernel's envelope (hd != 64, t > 4096).
int attention_fa(const void* qkv, const float* size, int B, int t, int H, int hd, void* out,
                 cudaStream_t s) {
  if (hd != kHd || t <= 0 || t > kMaxT) return TA_ERR_SHAPE;
  const FaLayout L = fa_layout(t);
  if (L.smem_bytes > 227 * 1024) return TA_ERR_SHAPE;
  CUtensorMap tm;
  int rc = make_tmap_bf16_2d(&tm, qkv, static_cast<uint64_t>(B) * t, 3ull * H * hd, 64);
  if (rc) return rc;
  static unsigned long long attr_mask = 0;  // per device
  if (attr_needed(attr_mask)) {
    cudaError_t e = cudaFuncSetAttribute(attn_fa_kernel<true>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(attn_fa_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               227 * 1024);
    if (e != cudaSuccess) return set_last_cuda_error(e);
    attr_done(attr_mask);
  }
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
  const float scale_log2 = 1.4426950408889634f / 8.0f;
  auto* o = static_cast<__nv_bfloat16*>(out);
  cudaError_t e = size != nullptr
                      ? cudaLaunchKernelEx(&cfg, attn_fa_kernel<true>, tm, o, size, t, H, n_items, scale_log2, L)
                      : cudaLaunchKernelEx(&cfg, attn_fa_kernel<false>, tm, o, size, t, H, n_items, scale_log2, L);
  return e == cudaSuccess ? TA_OK : set_last_cuda_error(e);
}

}  // namespace ta
