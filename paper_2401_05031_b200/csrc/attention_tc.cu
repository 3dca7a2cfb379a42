// Proportional attention on the 5th-gen tensor cores (north_star 3):
//   o = softmax(q k^T / sqrt(hd) + log size_j) v        per (image, head), hd = 64 / 80, t <= 512
//
// head_dim 80 (ViT-H/14): every Q / K / V row is a 64-column SW128 part plus a 16-column SW32
// tail (its own TMA map); S = Q K^T takes the tail as a fifth K = 16 step, O += P V a second
// N = 16 MMA into O[64, 80); O[0, 80) then overlaps S block 1 as well, so a tile's first PV
// waits until block 1's P is written; the tail columns of O leave by one STG.256 per row.
//
// Persistent, warp-specialised, one CTA per SM looping over work items (image, head); each
// item walks its 128-query tiles with K / V fetched from HBM once per item.
//   warp 8 (lane 0)  TMA producer: K, V of the item (64-row SW128 boxes) into a 2-slot
//                    ring (1 slot when t > 256: then K and V have their own barriers, K is
//                    refilled after the item's last S and V after its last PV), Q tiles into
//                    one slot.
//   warp 9 (lane 0)  MMA issuer: S = Q K^T (M = 128, N <= 256 per instruction) into one of
//                    two TMEM S slots; S of tile n+1 is issued before PV of tile n so the
//                    softmax warps never wait for it; O += P_blk V_blk per 64-key block with
//                    V as an MN-major B operand.
//   warps 0..7       t_pad <= 256 (row split): group g owns every other tile and its S slot,
//                    whole rows per thread.  Otherwise softmax in two groups over even / odd
//                    64-key blocks of one S slot; query row i is
//                    TMEM lane i (warps w and w+4 share lanes 32(w%4)..); pass 1 row max m
//                    of the raw scores, pass 2 p = size_j * 2^((s - m) log2(e)/sqrt(hd))
//                    (= the log-size bias as a weight; size 0 masks keys >= t) -> bf16 P
//                    block into ring stage g (SW128, K-major) -> PV MMA; row max / sum
//                    combined through smem; epilogue O / sum -> bf16 rows.
// TMEM: slot s at columns [256 s, 256 s + t_pad); O aliases the slot's S block 0, which
// softmax has consumed before the first PV MMA is issued -- except with one S slot and room
// beside it (t_pad <= 512 - hd), where O has its own columns and the slot is released after
// pass 2, so the next tile's S overlaps the PV tail and the epilogue.  Keys past t are masked with a
// -inf bias (their K / V rows are the next image's rows or TMA zero fill: finite, p = 0).
#include <cfloat>
#include <cstdlib>
#include <type_traits>

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

// Barrier waits of the TMA producer carry a suspend-time hint (mbar_wait_sleep), so its polling
// takes fewer issue slots from the softmax warps of its sub-partition: t = 197 104.0 -> 102.6 us,
// t = 117 45.4 -> 44.9 us (B = 256, two interleaved runs).  Build flag for A/B: -DTA_ATTN_WAIT_SLEEP=0
// plain try_wait loops, =2 the MMA warps' waits too (no better than 1).
#ifndef TA_ATTN_WAIT_SLEEP
#define TA_ATTN_WAIT_SLEEP 1
#endif
#define PWAIT(b, p) (TA_ATTN_WAIT_SLEEP >= 1 ? mbar_wait_sleep((b), (p), 1000) : mbar_wait((b), (p)))
#define MWAIT(b, p) (TA_ATTN_WAIT_SLEEP >= 2 ? mbar_wait_sleep((b), (p), 1000) : mbar_wait((b), (p)))

constexpr int kHd = 64;
constexpr int kQTile = 128;
constexpr int kKeyBlk = 64;
constexpr int kBlkBytes = kKeyBlk * kHd * 2;  // 8 KB: one 64-row SW128 box
constexpr int kQBytes = kQTile * kHd * 2;     // 16 KB
constexpr int kPBytes = kQTile * kKeyBlk * 2;  // 16 KB: one P block
constexpr int kMaxTPad = 512;
constexpr int kThreads = 352;  // 8 softmax warps, TMA warp 8, MMA warps 9 and 10

struct AttnTcLayout {
  int hd;       // 64, or 80 = a 64-column SW128 part + a 16-column SW32 tail
  int tail;     // hd - 64
  uint32_t q_bytes;   // Q tile: 128 x 64 main (16 KB) + 128 x tail (SW32)
  uint32_t tail_blk;  // bytes of one 64-key block's tail columns (64 x tail x 2)
  uint32_t kt_off, vt_off;  // K / V tail regions inside a K/V slot
  int t_pad;    // round_up(t, 64)
  int t_mma;    // round_up(t, 16): S MMA N (keys past it are never read)
  int nch_last; // 8-key chunks of the last 64-key block holding keys < t
  int nkc_last; // 16-key PV steps of the last block (chunks [nch_last, 2 nkc_last) are zeros)
  int mtail;    // row split, hd 64: the last block's <= 16 keys ride with the previous P block
  int n_pb;     // P blocks per tile (n_kb - mtail)
  int n_kb;     // t_pad / 64
  int n_qt;     // ceil(t / 128)
  int n_kv;     // K/V ring slots (4 when t_pad <= 128 and they fit, 2 when t_pad <= 256)
  int n_s;      // TMEM S slots (2 when t_pad <= 256)
  int rowsplit; // 1: softmax group g owns every other tile (t_pad <= 128); 0: groups split keys
  int o_col;    // single S slot with O in its own TMEM columns [o_col, o_col + hd) (0: O aliases S)
  int qswap;    // row split, two query tiles: odd items take their tiles in reverse order
  int o_sep;    // row split: O in its own columns [256 g + o_sep, 256 g + 256) of slot g (0: aliases S)
  uint32_t kv_bytes;  // per slot: K then V
  uint32_t kv_off, p_off, mt_off, bias_off, red_off, bar_off, smem_bytes;
};

AttnTcLayout attn_layout(int t, int hd) {
  AttnTcLayout L{};
  L.hd = hd;
  L.tail = hd - kHd;
  L.q_bytes = kQBytes + kQTile * L.tail * 2;
  L.tail_blk = kKeyBlk * L.tail * 2;
  L.t_pad = (t + kKeyBlk - 1) / kKeyBlk * kKeyBlk;
  L.n_kb = L.t_pad / kKeyBlk;
  L.t_mma = (t + 15) / 16 * 16;
  {
    const int rem = t - (L.n_kb - 1) * kKeyBlk;  // 1..64 keys in the last block
    L.nch_last = (rem + 7) / 8;
    L.nkc_last = (rem + 15) / 16;
  }
  L.n_qt = (t + kQTile - 1) / kQTile;
  L.n_kv = L.t_pad <= 256 ? 2 : 1;
  L.n_s = L.t_pad <= 256 ? 2 : 1;
  // Row split (each softmax group owns whole tiles of its own S slot) for every t that fits two
  // slots: measured 121 vs 133 us at t = 197, 51 vs 64 us at t = 101 (B = 256, H = 12).
  L.rowsplit = L.t_pad <= 256;
  if (const char* e = getenv("TA_ATTN_SPLIT"))  // profiling override: "row" / "key"
    L.rowsplit = L.t_pad <= 256 && e[0] != 'k';
  L.qswap = L.rowsplit && L.n_qt == 2;
  // Row split with room beside S in the slot (t_mma + hd <= 256): O gets its own columns, the
  // slot is released as soon as pass 2 has read S, and the MMA warp computes the group's next S
  // during this tile's PV tail and epilogue (o_free hands O back before the next tile's PV).
  {
    const int hd_cols = (hd + 15) / 16 * 16;
    L.o_sep = (L.rowsplit && L.t_mma + hd_cols <= 256) ? 256 - hd_cols : 0;
    if (const char* e = getenv("TA_ATTN_OSEP"))  // profiling override: "0" keeps O in the slot
      if (e[0] == '0') L.o_sep = 0;
  }
  if (const char* e = getenv("TA_ATTN_QSWAP"))  // profiling override: "0" keeps the tile order
    if (e[0] == '0') L.qswap = 0;
  // One S slot (t_pad > 256): when S and O fit side by side, O gets its own columns, the slot
  // is released as soon as pass 2 has read it, and S of the next tile overlaps the PV tail and
  // the (deferred) epilogue, as in two-slot mode.
  L.o_col = 0;
  if (L.n_s == 1 && L.t_pad <= 512 - ((hd + 15) / 16) * 16) L.o_col = 512 - ((hd + 15) / 16) * 16;
  if (const char* e = getenv("TA_ATTN_OAPART"))  // profiling override: "0" keeps O aliased
    if (e[0] == '0') L.o_col = 0;
  // K/V slot: [K main blocks][V main blocks][K tails][V tails]
  L.kt_off = 2u * L.n_kb * kBlkBytes;
  L.vt_off = L.kt_off + L.n_kb * L.tail_blk;
  L.kv_bytes = L.vt_off + L.n_kb * L.tail_blk;
  // hd = 80 at t_pad = 256: two K/V slots would not fit beside Q and the P ring
  if (L.n_kv == 2 && L.q_bytes + 2 * L.kv_bytes + 4 * kPBytes + 8192 > 227u * 1024) L.n_kv = 1;
  // One-tile items (t_pad <= 128): a tile's softmax is short next to a K / V load, so with two
  // slots the next item's load (issued when a PV releases a slot) sat on the critical path
  // (trace at t = 69: 3100 clk from O committed to the group's next S); four slots load two
  // items ahead.  TA_ATTN_KV=2 keeps two (profiling A/B).
  if (L.t_pad <= 128 && L.q_bytes + 4 * L.kv_bytes + 4 * kPBytes + 8192 <= 227u * 1024) L.n_kv = 4;
  if (const char* e = getenv("TA_ATTN_KV"))
    if (e[0] == '2' && L.n_kv == 4) L.n_kv = 2;
  uint32_t off = (L.q_bytes + 1023) / 1024 * 1024;  // Q: one slot (Q(n+1) is only needed after S(n))
  L.kv_off = off;
  off += L.n_kv * L.kv_bytes;
  L.p_off = off;
  off += 4 * kPBytes;  // P ring: two stages per softmax group
  // Merged tail (row split, hd 64, last key block holding <= 16 keys, e.g. t = 197 / 205 / 133 / 69):
  // those keys' P goes to a 128 x 16 SW32 tile of the group (4 KB) written with the previous
  // 64-key block and taken by the same PV step as one more K = 16 MMA, so a tile walks n_kb - 1
  // P-ring stages instead of n_kb (TA_ATTN_MTAIL=0 keeps the separate last block).
  L.mtail = 0;
  {
    const int rem = t - (L.n_kb - 1) * kKeyBlk;
    const char* e = getenv("TA_ATTN_MTAIL");
    if (L.rowsplit && L.tail == 0 && L.n_kb >= 2 && rem <= 16 && !(e && e[0] == '0')) L.mtail = 1;
  }
  L.n_pb = L.n_kb - L.mtail;
  L.mt_off = off;
  if (L.mtail) off += 2 * 4096;
  L.bias_off = off;
  off += kMaxTPad * 4;
  L.red_off = off;
  off += 4 * 128 * 4;
  L.bar_off = off;
  off += 40 * 8;
  L.smem_bytes = off + 1024;  // + alignment slack
  return L;
}

#ifdef TA_ATTN_TRACE  // profiling build only: per-event clock64 timeline of CTA 0
__device__ unsigned long long g_trace_t[16384];
__device__ unsigned int g_trace_tag[16384];
// per-warp slices of 1024 events, register counter: no atomics on the traced path
#define TRACE(ev)                                                                      \
  do {                                                                                 \
    if (blockIdx.x == 0 && (threadIdx.x & 31) == 0 && tr_n < 1024u) {                  \
      const unsigned int k_ = (threadIdx.x >> 5) * 1024u + tr_n++;                     \
      g_trace_t[k_] = clock64();                                                       \
      g_trace_tag[k_] = (threadIdx.x >> 5) * 256u + (ev);                              \
    }                                                                                  \
  } while (0)
#define TRACE_DECL unsigned int tr_n = 0
#else
#define TRACE(ev) do {} while (0)
#define TRACE_DECL do {} while (0)
#endif

// Row split with two query tiles per item (128 < t <= 256): group g always owns the item's g-th
// tile in processing order, and the second tile holds only t - 128 rows, so the two groups are
// balanced by processing every odd item's tiles in reverse order (t = 133: the second tile has 5
// rows, and group 1 would otherwise idle while group 0 softmaxes every full tile).
__device__ __forceinline__ int q_order(int qt, uint32_t item_local, const AttnTcLayout& L) {
  return (L.qswap && (item_local & 1u)) ? 1 - qt : qt;
}

// kOne (kKv == 1): one K/V slot, where K and V have separate barriers and lifetimes and a
// single S slot may keep O in its own TMEM columns (L.o_col); a template parameter so that the
// two-slot instance carries none of that state (its register budget is tight).
// kKv: K/V ring slots (L.n_kv), a template parameter so that the one- and two-slot instances
// compile as before the four-slot ring (a runtime slot count cost them ~2 %).
template <bool kHasSize, int kHD, int kKv>
__global__ void __launch_bounds__(kThreads, 1)
    attn_tc_kernel(const __grid_constant__ CUtensorMap tm, const __grid_constant__ CUtensorMap tmt,
                   const __grid_constant__ CUtensorMap tmo,
                   const float* __restrict__ size, int t,
                   int H, int n_items, __nv_bfloat16* __restrict__ out, float scale_log2,
                   AttnTcLayout L) {
  TRACE_DECL;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  constexpr bool kOne = kKv == 1;
  constexpr int kTail = kHD - kHd;  // 16-column SW32 tail of a head_dim = 80 row (0 for 64)
  const uint32_t o_col = kOne ? static_cast<uint32_t>(L.o_col) : 0u;
  const int D = H * kHD;
  uint8_t* sQ = smem;
  uint8_t* sKV = smem + L.kv_off;
  uint8_t* sP = smem + L.p_off;
  float* bias = reinterpret_cast<float*>(smem + L.bias_off);
  float* red = reinterpret_cast<float*>(smem + L.red_off);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L.bar_off);
  // K and V of an item have separate lifetimes: K is free once the item's last S MMA is done,
  // V after its last PV, so with one K/V slot the next item's K (and first S) need not wait
  // for the PV tail of the previous item.
  uint64_t* kv_full = bars + (kKv == 4 ? 32 : 0);  // [kKv] K of the slot landed
  uint64_t* kv_free = bars + (kKv == 4 ? 36 : 2);  // [kKv] K of the slot consumed
  uint64_t* v_full = bars + 22;   // [2]
  uint64_t* v_free = bars + 24;   // [2]
  uint64_t* q_full = bars + 4;    // [2]
  uint64_t* q_free = bars + 6;    // [2]
  uint64_t* s_full = bars + 8;    // [2]
  uint64_t* s_free = bars + 10;   // [2]
  uint64_t* o_full = bars + 12;   // [2]
  uint64_t* p_full = bars + 14;   // [4]
  uint64_t* p_free = bars + 18;   // [4]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 26);
  uint64_t* o_free = bars + 27;  // [2] row split with L.o_sep: group g has read its O

  const uint32_t warp = warp_id(), lane = lane_id();
  // No runtime integer division in the loops below: it compiles to I2F / MUFU.RCP / F2I on
  // the SFU, which the softmax exponentials saturate on every sub-partition, and the MMA
  // issuer then waited ~700 cycles per P block.  Items advance by gridDim.x as (b, h) pairs;
  // ring indices use n_kv in {1, 2, 4}, n_s in {1, 2}.
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
  auto ring_slot = [](uint32_t x, int n) -> uint32_t { return n == 2 ? (x & 1u) : 0u; };
  auto ring_use = [](uint32_t x, int n) -> uint32_t { return n == 2 ? (x >> 1) : x; };
  // K/V ring of kKv slots
  auto kv_slot = [](uint32_t x) -> int { return static_cast<int>(x & static_cast<uint32_t>(kKv - 1)); };
  auto kv_round = [](uint32_t x) -> uint32_t { return kKv == 4 ? (x >> 2) : kKv == 2 ? (x >> 1) : x; };
  if (warp == 8 && lane == 0) {
    tma_prefetch(&tm);
    for (int s = 0; s < kKv; ++s) {
      // row split: every tile of an item releases its K / V (MMA warp 9 or 10, one per tile)
      mbar_init(&kv_full[s], 1);
      mbar_init(&kv_free[s], L.rowsplit ? L.n_qt : 1);
    }
    for (int s = 0; s < 2; ++s) {
      const int rel = L.rowsplit ? L.n_qt : 1;
      mbar_init(&v_full[s], 1);
      mbar_init(&v_free[s], rel);
      mbar_init(&q_full[s], 1);
      mbar_init(&q_free[s], 1);
      mbar_init(&s_full[s], 1);
      mbar_init(&s_free[s], L.rowsplit ? 128 : 256);  // row-split: one group reads a slot
      mbar_init(&o_full[s], 1);
      mbar_init(&o_free[s], 128);
    }
    for (int s = 0; s < 4; ++s) {
      mbar_init(&p_full[s], 128);
      mbar_init(&p_free[s], 1);
    }
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_all = *tmem_slot;
  const uint32_t tmem = tmem_all;

  grid_dep_wait();  // qkv is the previous kernel's output

  grid_dep_launch();  // early trigger: the next kernel's prologue overlaps our tail

  if (warp == 8) {
    // ------------------------------------------------------------ TMA producer
    if (lane == 0) {
      uint32_t it = 0, qcnt = 0;
      int b = b_first, h = h_first;
      for (int item = blockIdx.x; item < n_items; item += gridDim.x, ++it, next_bh(b, h)) {
        const int row_base = b * t;
        const int kvs = kv_slot(it);
        const uint32_t kv_use = kv_round(it);
        PWAIT(&kv_free[kvs], (kv_use & 1) ^ 1);
        uint8_t* sK = sKV + kvs * L.kv_bytes;
        uint8_t* sV = sK + L.n_kb * kBlkBytes;
        TRACE(1);
        // Two slots: K and V share kv_full / kv_free (the ring runs an item ahead anyway).  One
        // slot: V has its own barriers and is loaded after the item's first Q.
        constexpr bool split_v = kOne;
        const uint32_t half_bytes = L.n_kb * (kBlkBytes + L.tail_blk);
        auto load_v = [&](uint64_t* bar) {
          for (int kb = 0; kb < L.n_kb; ++kb) {
            tma_load_2d(&tm, bar, sV + kb * kBlkBytes, 2 * D + h * kHD, row_base + kb * kKeyBlk);
            if constexpr (kTail > 0)
              tma_load_2d(&tmt, bar, sK + L.vt_off + kb * L.tail_blk, 2 * D + h * kHD + kHd,
                          row_base + kb * kKeyBlk);
          }
        };
#ifdef TA_ATTN_EXP_KVONCE  // profiling only: wrong results (K / V of the first items reused)
        if (it >= static_cast<uint32_t>(kKv) && !split_v) {
          mbar_arrive(&kv_full[kvs]);
        } else
#endif
        {
        mbar_arrive_expect_tx(&kv_full[kvs], split_v ? half_bytes : 2 * half_bytes);
        for (int kb = 0; kb < L.n_kb; ++kb) {
          tma_load_2d(&tm, &kv_full[kvs], sK + kb * kBlkBytes, D + h * kHD, row_base + kb * kKeyBlk);
          if constexpr (kTail > 0)
            tma_load_2d(&tmt, &kv_full[kvs], sK + L.kt_off + kb * L.tail_blk, D + h * kHD + kHd,
                        row_base + kb * kKeyBlk);
        }
        if (!split_v) load_v(&kv_full[kvs]);
        }
        for (int qt = 0; qt < L.n_qt; ++qt, ++qcnt) {
          // One Q buffer.  Row split: tile n belongs to MMA warp 9 + (n & 1), whose own barrier
          // pair (q_full / q_free[n & 1]) completes once per tile of that warp; the buffer is
          // reloaded once S of tile n - 1 (the other warp's) is done.  Key split: one pair.
          uint64_t* qf = &q_full[L.rowsplit ? (qcnt & 1) : 0];
          if (L.rowsplit) {
            if (qcnt > 0) PWAIT(&q_free[(qcnt - 1) & 1], ((qcnt - 1) >> 1) & 1);
          } else {
            PWAIT(&q_free[0], (qcnt & 1) ^ 1);
          }
#ifdef TA_ATTN_EXP_QONCE  // profiling only: wrong results (Q of the first tile reused)
          if (qcnt > 0) { mbar_arrive(qf); continue; }
#endif
          mbar_arrive_expect_tx(qf, L.q_bytes);
          const int qe = q_order(qt, it, L);  // this tile's query rows
          tma_load_2d(&tm, qf, sQ, h * kHD, row_base + qe * kQTile);
          tma_load_2d(&tm, qf, sQ + kBlkBytes, h * kHD, row_base + qe * kQTile + 64);
          if constexpr (kTail > 0) {
            tma_load_2d(&tmt, qf, sQ + kQBytes, h * kHD + kHd, row_base + qe * kQTile);
            tma_load_2d(&tmt, qf, sQ + kQBytes + 64 * kTail * 2, h * kHD + kHd,
                        row_base + qe * kQTile + 64);
          }
          TRACE(2);
          if (qt == 0 && split_v) {
            PWAIT(&v_free[kvs], (kv_use & 1) ^ 1);
            mbar_arrive_expect_tx(&v_full[kvs], half_bytes);
            load_v(&v_full[kvs]);
          }
        }
      }
    }
  } else if (warp == 9 || warp == 10) {
    // ------------------------------------------------------------ MMA issuer(s)
    // The whole warp runs the issuer with warp-uniform state; one elected lane issues each
    // tcgen05.mma / commit (ptx.cuh umma_f16_w): the descriptor arithmetic stays in uniform
    // registers, so an MMA costs a few uniform instructions instead of an R2UR + elect loop,
    // which matters on a sub-partition shared with two softmax warps.
    {
      const uint32_t tmem = __shfl_sync(0xffffffffu, tmem_all, 0);  // warp-uniform TMEM base
      constexpr uint32_t idesc_pv = idesc_bf16(kQTile, kHd, /*b_mn_major=*/true);
      constexpr uint32_t idesc_pv_t = idesc_bf16(kQTile, kTail > 0 ? kTail : 16, /*b_mn_major=*/true);
      // O += P_blk V_blk for one 64-key block: N = 64 from the SW128 V part into O[0, 64) and,
      // for head_dim 80, N = 16 from the SW32 tail into O[64, 80).
      // kW: warp-uniform issue (the whole warp runs the caller) or lane-0 issue
      auto mma = [](auto kW, uint32_t d, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
        if constexpr (decltype(kW)::value) umma_f16_w(d, a, b, id, acc);
        else umma_f16(d, a, b, id, acc);
      };
      auto pv_block = [&](auto kW, uint32_t o_tmem, uint64_t pdesc, const uint8_t* sKVslot, int kb, int nkc) {
        const uint32_t vbase = smem_u32(sKVslot + L.n_kb * kBlkBytes + kb * kBlkBytes);
        const uint32_t vtbase = smem_u32(sKVslot + L.vt_off + kb * L.tail_blk);
#pragma unroll
        for (int kc = 0; kc < kKeyBlk / 16; ++kc) {
          if (kc >= nkc) break;
          // V rows (keys) are the K dimension: 16 keys = two 8-row groups = 2048 B.
          const uint64_t vdesc = umma_desc_sw128_mn(vbase + kc * 2048, 8192, 1024);
          mma(kW, o_tmem, pdesc + 2 * kc, vdesc, idesc_pv, (kb | kc) != 0);
          if constexpr (kTail > 0) {
            const uint64_t vtdesc = umma_desc_sw32_mn(vtbase + kc * 512, 512, 256);
            mma(kW, o_tmem + kHd, pdesc + 2 * kc, vtdesc, idesc_pv_t, (kb | kc) != 0);
          }
        }
      };
      uint32_t p_use[2] = {0, 0};  // per softmax group; stage = 2 g + (use & 1)
      // pending PV tile (issued after the next tile's S so softmax never waits)
      int pend_slot = -1, pend_kvs = 0;
      bool pend_last = false, pend_first = false;
      uint32_t pend_vpar = 0;
      auto issue_pv = [&](int sslot, int kvs, bool last_of_item, bool first_of_item, uint32_t v_par) {
        const uint8_t* sKVslot = sKV + kvs * L.kv_bytes;
        const uint32_t o_tmem = o_col ? tmem + o_col : tmem + sslot * 256;
        if (first_of_item && kOne) MWAIT(&v_full[kvs], v_par);
        for (int kb = 0; kb < L.n_kb; ++kb) {
          const int grp = kb & 1;
          const uint32_t u = p_use[grp]++;
          const int ps = 2 * grp + (u & 1);
          MWAIT(&p_full[ps], (u >> 1) & 1);
          if (kTail > 0 && kb == 0 && L.n_kb > 1 && !o_col)  // O[0, 80) overlaps S block 1: wait for its P
            MWAIT(&p_full[2 + (p_use[1] & 1)], (p_use[1] >> 1) & 1);
          TRACE(5);
          tc_fence_after();
          const uint64_t pdesc = umma_desc_sw128(smem_u32(sP + ps * kPBytes));
          const int nkc = kb == L.n_kb - 1 ? L.nkc_last : kKeyBlk / 16;
#ifndef TA_ATTN_EXP_NOPV  // profiling only: wrong results (key-split PV MMAs skipped)
          pv_block(std::true_type{}, o_tmem, pdesc, sKVslot, kb, nkc);
#endif
          umma_commit_w(&p_free[ps]);
        }
        umma_commit_w(&o_full[sslot]);
        TRACE(6);
        if (last_of_item) umma_commit_w(kOne ? &v_free[kvs] : &kv_free[kvs]);
      };
      if (L.rowsplit) {
        // Row-split mode (t_pad <= 256): tile n (this CTA's n-th tile) lives in S slot n & 1, is
        // softmaxed by group n & 1 and issued by MMA warp 9 + (n & 1) with blocking waits: S,
        // then its PV blocks as its group's P stages fill, so neither group's MMAs wait behind
        // the other group's (a single issuer polling both measured 1.3-1.6x longer per tile
        // from the last P block to O).
        const uint32_t g = warp - 9;
        const uint32_t slot_tmem = tmem + g * 256;
        const uint32_t o_tmem = slot_tmem + static_cast<uint32_t>(L.o_sep);
        uint32_t j = 0, pu = 0, n = 0, it = 0;
        for (int item = blockIdx.x; item < n_items; item += gridDim.x, ++it) {
          const int kvs = kv_slot(it);
          const uint32_t kv_par = kv_round(it) & 1;
          const uint8_t* sKVslot = sKV + kvs * L.kv_bytes;
          for (int qt = 0; qt < L.n_qt; ++qt, ++n) {
            if ((n & 1u) != g) continue;
            MWAIT(&s_free[g], (j & 1) ^ 1);  // group g has read O of its previous tile
            MWAIT(&q_full[g], j & 1);
            MWAIT(&kv_full[kvs], kv_par);
            TRACE(7);
            tc_fence_after();
            {
              const uint64_t qdesc = umma_desc_sw128(smem_u32(sQ));
              const uint32_t idesc_s = idesc_bf16(kQTile, L.t_mma);
              const uint64_t kdesc = umma_desc_sw128(smem_u32(sKVslot));
#pragma unroll
              for (int k = 0; k < kHd / 16; ++k)
                umma_f16_w(slot_tmem, qdesc + 2 * k, kdesc + 2 * k, idesc_s, k > 0);
              if constexpr (kTail > 0)  // head_dim 80: the 16-column tail as a fifth K step
                umma_f16_w(slot_tmem, umma_desc_sw32(smem_u32(sQ + kQBytes)),
                           umma_desc_sw32(smem_u32(sKVslot + L.kt_off)), idesc_s, 1);
            }
            umma_commit_w(&s_full[g]);
            umma_commit_w(&q_free[g]);
            if (kOne) umma_commit_w(&kv_free[kvs]);  // this tile's use of K is done
            TRACE(4);
            if (kOne) MWAIT(&v_full[kvs], kv_par);
            if (L.o_sep && j > 0) MWAIT(&o_free[g], (j - 1) & 1);  // O of the previous tile read
            for (int kb = 0; kb < L.n_pb; ++kb) {
              const int ps = 2 * g + (pu & 1);
              MWAIT(&p_full[ps], (pu >> 1) & 1);
              ++pu;
              // head_dim 80 with O in the slot: O[0, 80) overlaps S block 1, so block 0's PV waits
              // for block 1's P
              if (kTail > 0 && kb == 0 && L.n_kb > 1 && !L.o_sep)
                MWAIT(&p_full[2 * g + (pu & 1)], (pu >> 1) & 1);
              TRACE(8 + 16 * g);
              tc_fence_after();
              const uint64_t pdesc = umma_desc_sw128(smem_u32(sP + ps * kPBytes));
              const int nkc = kb == L.n_kb - 1 ? L.nkc_last : kKeyBlk / 16;
              pv_block(std::true_type{}, o_tmem, pdesc, sKVslot, kb, nkc);
              if (kTail == 0 && L.mtail && kb == L.n_pb - 1)  // the merged tail: keys 64 (n_kb - 1) + [0, 16)
                pv_block(std::true_type{}, o_tmem, umma_desc_sw32(smem_u32(smem + L.mt_off + g * 4096)), sKVslot,
                         L.n_kb - 1, 1);
              umma_commit_w(&p_free[ps]);
              TRACE(5 + 16 * g);
            }
            umma_commit_w(&o_full[g]);
            umma_commit_w(kOne ? &v_free[kvs] : &kv_free[kvs]);  // this tile's use of K / V is done
            TRACE(6);
            ++j;
          }
        }
      } else if (warp == 9) {
      uint32_t it = 0, qcnt = 0, tcnt = 0;
      for (int item = blockIdx.x; item < n_items; item += gridDim.x, ++it) {
        const int kvs = kv_slot(it);
        const uint32_t kv_use = kv_round(it);
        const uint8_t* sK = sKV + kvs * L.kv_bytes;
        for (int qt = 0; qt < L.n_qt; ++qt, ++qcnt, ++tcnt) {
          const int ss = ring_slot(tcnt, L.n_s);
          if (L.n_s == 1 && pend_slot >= 0) {  // single S slot: finish the previous tile first
            issue_pv(pend_slot, pend_kvs, pend_last, pend_first, pend_vpar);
            pend_slot = -1;
          }
          MWAIT(&s_free[ss], (ring_use(tcnt, L.n_s) & 1) ^ 1);
          MWAIT(&q_full[0], qcnt & 1);
          if (qt == 0) MWAIT(&kv_full[kvs], kv_use & 1);
          TRACE(3);
          tc_fence_after();
          const uint64_t qdesc = umma_desc_sw128(smem_u32(sQ));
          for (int n0 = 0; n0 < L.t_mma; n0 += 256) {
            const int n = L.t_mma - n0 < 256 ? L.t_mma - n0 : 256;
            const uint32_t idesc_s = idesc_bf16(kQTile, n);
            const uint64_t kdesc = umma_desc_sw128(smem_u32(sK + n0 * 128));
#pragma unroll
            for (int k = 0; k < kHd / 16; ++k)
              umma_f16_w(tmem + ss * 256 + n0, qdesc + 2 * k, kdesc + 2 * k, idesc_s, k > 0);
            if constexpr (kTail > 0)
              umma_f16_w(tmem + ss * 256 + n0, umma_desc_sw32(smem_u32(sQ + kQBytes)),
                       umma_desc_sw32(smem_u32(sK + L.kt_off + n0 * kTail * 2)), idesc_s, 1);
          }
          umma_commit_w(&s_full[ss]);
          TRACE(4);
          umma_commit_w(&q_free[0]);
          if (kOne && qt + 1 == L.n_qt) umma_commit_w(&kv_free[kvs]);  // the item's K is consumed
          if (pend_slot >= 0) issue_pv(pend_slot, pend_kvs, pend_last, pend_first, pend_vpar);
          pend_slot = ss;
          pend_kvs = kvs;
          pend_last = qt + 1 == L.n_qt;
          pend_first = qt == 0;
          pend_vpar = kv_use & 1;
        }
      }
      if (pend_slot >= 0) issue_pv(pend_slot, pend_kvs, pend_last, pend_first, pend_vpar);
      }
    }
  } else {
    // ------------------------------------------------------------ softmax / epilogue
    // Per tile: pass 1 (row max), pass 2 (P blocks), epilogue (O / sum).  With two S slots
    // the epilogue of tile n runs after pass 1 of tile n+1, hiding the PV completion latency.
    const int g = warp >> 2;
    const int i = (warp & 3) * 32 + lane;  // query row within the tile
    const uint32_t lane_base = tmem + (((warp & 3) * 32u) << 16);
    uint32_t use = 0;

    // shared-space addresses (explicit ld/st.shared; see lds_f4)
    const uint32_t s_bias = smem_u32(bias);
    const uint32_t s_red = smem_u32(red);
    const uint32_t s_prow0 = smem_u32(sP) + 2 * g * kPBytes + i * 128;  // + (use & 1) stage
    // O staging: this warp's 2 KB slab(s) inside its own 32 P rows (4 KB) of the group's first
    // P stage, which is idle between the tile's last PV MMA (o_full) and the next tile's first
    // P block; before the warp writes P again the slab's TMA store must have read it
    // (drain_o_store).  Only the owning warp ever writes these bytes.
    const uint32_t s_slab = smem_u32(sP) + 2 * g * kPBytes + (warp & 3) * 4096;
    auto drain_o_store = [&]() {
      if (lane == 0) bulk_wait_group_read<0>();
      __syncwarp();
    };

    // a warp whose 32 query rows of tile qt all lie past t only keeps the barrier protocol
    auto row_idle = [&](int qt) { return qt * kQTile + static_cast<int>(warp & 3) * 32 >= t; };
    auto pass1 = [&](uint32_t tcnt, int qt) -> float {
      const int ss = ring_slot(tcnt, L.n_s);
      const uint32_t la = lane_base + ss * 256;
      mbar_wait(&s_full[ss], ring_use(tcnt, L.n_s) & 1);
      TRACE(10);
      tc_fence_after();
      float m4[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
      if (!row_idle(qt))
        for (int kb = g; kb < L.n_kb; kb += 2) block_max(la + kb * 64, min(kKeyBlk, t - kb * kKeyBlk), m4);
      sts_f32(s_red + (g * 128 + i) * 4, fmaxf(fmaxf(m4[0], m4[1]), fmaxf(m4[2], m4[3])));
      TRACE(11);
      named_bar_sync(1, 256);
      TRACE(12);
      // row max of the raw scores, in the scaled log2 domain
      return fmaxf(lds_f32(s_red + i * 4), lds_f32(s_red + (128 + i) * 4)) * scale_log2;
    };

    auto pass2 = [&](uint32_t tcnt, float mx, int qt) -> float {
      const uint32_t la = lane_base + ring_slot(tcnt, L.n_s) * 256;
      const bool idle = row_idle(qt);
      drain_o_store();
      uint64_t acc[2] = {0ull, 0ull};
      const uint64_t sc2 = f2_pack(scale_log2, scale_log2), nm2 = f2_pack(-mx, -mx);
      for (int kb = g; kb < L.n_kb; kb += 2, ++use) {
        const bool last = kb == L.n_kb - 1;
        uint32_t r[64];
        if (!idle) {
          tmem_ld_32x32b_x32(la + kb * 64, *reinterpret_cast<uint32_t(*)[32]>(&r[0]));
          tmem_ld_32x32b_x32(la + kb * 64 + 32, *reinterpret_cast<uint32_t(*)[32]>(&r[32]));
        }
        const int pst = 2 * g + (use & 1);
        const uint32_t s_prow = s_prow0 + (use & 1) * kPBytes;
        mbar_wait(&p_free[pst], ((use >> 1) & 1) ^ 1);
        TRACE(13);
        if (!idle) {
          tmem_ld_wait();
          // p_j = size_j * 2^(s_j * scale - max): the log-size bias as a weight (size 0 masks
          // keys >= t); without a size vector only the last block needs the mask.
          if (!last)
            softmax_block64(r, sc2, nm2, kHasSize, s_bias + kb * 64 * 4, s_prow, i, acc);
          else
            softmax_block_tail(r, sc2, nm2, s_bias + kb * 64 * 4, s_prow, i, L.nch_last,
                               2 * L.nkc_last, acc);
          fence_proxy_async_smem();
        }
        tc_fence_before();  // S reads done before the PV MMA may overwrite block 0
        mbar_arrive(&p_full[pst]);
        TRACE(14);
      }
      if (o_col) mbar_arrive(&s_free[0]);  // S fully read (tc_fence_before above): next S may go
      TRACE(15);
      sts_f32(s_red + (256 + g * 128 + i) * 4, f2_total(acc));
      named_bar_sync(1, 256);
      TRACE(16);
      return rcp_approx(lds_f32(s_red + (256 + i) * 4) + lds_f32(s_red + (384 + i) * 4));
    };

    // head_dim 80: this thread's row's last 16 columns (32 bytes, one STG.256) of O / sum
    auto store_o_tail = [&](const uint32_t (&ot)[16], float inv, int b, int q, int h) {
      if (q >= t) return;
      uint32_t w[8];
#pragma unroll
      for (int e = 0; e < 8; ++e)
        w[e] = pack_bf16(__uint_as_float(ot[2 * e]) * inv, __uint_as_float(ot[2 * e + 1]) * inv);
      stg256(out + (static_cast<long long>(b) * t + q) * D + h * kHD + kHd, make_uint4(w[0], w[1], w[2], w[3]),
             make_uint4(w[4], w[5], w[6], w[7]));
    };
    auto epilogue = [&](uint32_t tcnt, int b, int h, int qt, float inv) {
      const int ss = ring_slot(tcnt, L.n_s);
      mbar_wait(&o_full[ss], ring_use(tcnt, L.n_s) & 1);
      TRACE(17);
      tc_fence_after();
      uint32_t o[32], ot[16];
      const uint32_t o_base = lane_base + (o_col ? o_col : ss * 256);
      tmem_ld_32x32b_x32(o_base + g * 32, o);
      if (kTail > 0 && g == 1) tmem_ld_32x32b_x16(o_base + kHd, ot);
      tmem_ld_wait();
      tc_fence_before();
      if (!o_col) mbar_arrive(&s_free[ss]);
      const int q0 = qt * kQTile + (warp & 3) * 32;
      if (q0 < t) store_o_slab(&tmo, o, inv, s_slab, lane, h * kHD + g * 32, q0, b);
      if (kTail > 0 && g == 1) store_o_tail(ot, inv, b, q0 + static_cast<int>(lane), h);
      TRACE(18);
    };

    if (L.rowsplit) {
      // ---- row-split: group g owns the tiles of S slot g (every other tile); no cross-group
      // exchange, bias kept per group.
      const uint32_t s_bias_g = s_bias + g * 256 * 4;
      const uint32_t la = lane_base + g * 256;
      uint32_t k = 0;  // tiles processed by this group
      uint32_t tile = 0, it = 0;
      int b = b_first, h = h_first;
      for (int item = blockIdx.x; item < n_items; item += gridDim.x, next_bh(b, h), ++it) {
        const int row_base = b * t;
        bool have_bias = false;
        for (int qn = 0; qn < L.n_qt; ++qn, ++tile) {
          if (static_cast<int>(tile & 1) != g) continue;
          const int qt = q_order(qn, it, L);
          if (!have_bias) {
            named_bar_sync(2 + g, 128);  // group done with the previous item's bias
            for (int j = i; j < L.t_pad; j += 128)
              sts_f32(s_bias_g + j * 4,
                      j < t ? (size != nullptr ? size[static_cast<long long>(row_base) + j] : 1.f) : 0.f);
            named_bar_sync(2 + g, 128);
            have_bias = true;
          }
          mbar_wait(&s_full[g], k & 1);
          TRACE(10);
          tc_fence_after();
          const bool idle = row_idle(qt);
          // pass 1: row max of the raw scores over the valid keys
          float m4[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
          if (!idle)
            for (int kb = 0; kb < L.n_kb; ++kb) block_max(la + kb * 64, min(kKeyBlk, t - kb * kKeyBlk), m4);
          TRACE(11);
          const float nmx = -fmaxf(fmaxf(m4[0], m4[1]), fmaxf(m4[2], m4[3])) * scale_log2;
          // pass 2: P blocks
          drain_o_store();
          uint64_t acc[2] = {0ull, 0ull};
          const uint64_t sc2 = f2_pack(scale_log2, scale_log2), nm2 = f2_pack(nmx, nmx);
          for (int kb = 0; kb < L.n_pb; ++kb, ++use) {
            const bool last = kb == L.n_kb - 1;
            uint32_t r[64];
            if (!idle) {
              tmem_ld_32x32b_x32(la + kb * 64, *reinterpret_cast<uint32_t(*)[32]>(&r[0]));
              tmem_ld_32x32b_x32(la + kb * 64 + 32, *reinterpret_cast<uint32_t(*)[32]>(&r[32]));
            }
            const int pst = 2 * g + (use & 1);
            const uint32_t s_prow = s_prow0 + (use & 1) * kPBytes;
            mbar_wait(&p_free[pst], ((use >> 1) & 1) ^ 1);
            TRACE(13);
            if (!idle) {
              tmem_ld_wait();
              if (!last)
                softmax_block64(r, sc2, nm2, kHasSize, s_bias_g + kb * 64 * 4, s_prow, i, acc);
              else
                softmax_block_tail(r, sc2, nm2, s_bias_g + kb * 64 * 4, s_prow, i, L.nch_last,
                                   2 * L.nkc_last, acc);
              if (kTail == 0 && L.mtail && kb == L.n_pb - 1) {
                // merged tail: this row's keys 64 (n_kb - 1) + [0, 16) into the group's SW32 tile
                // (16-byte chunk c of row i at c ^ ((i >> 2) & 1)); weights are 0 past t
                uint32_t rt[16];
                tmem_ld_32x32b_x16(la + (L.n_kb - 1) * 64, rt);
                tmem_ld_wait();
                const uint32_t s_mt = smem_u32(smem + L.mt_off) + g * 4096u + static_cast<uint32_t>(i) * 32u;
                const uint32_t s_wt = s_bias_g + (L.n_kb - 1) * 64 * 4;
                const uint32_t sw = (static_cast<uint32_t>(i) >> 2) & 1u;
                uint4 v0 = softmax_chunk8<TA_ATTN_POLY_EVEN>(&rt[0], sc2, nm2, true, s_wt, acc);
                uint4 v1 = make_uint4(0u, 0u, 0u, 0u);
                if (L.nch_last > 1) v1 = softmax_chunk8<TA_ATTN_POLY_ODD>(&rt[8], sc2, nm2, true, s_wt + 32, acc);
                sts_u4(s_mt + (sw << 4), v0);
                sts_u4(s_mt + ((1u ^ sw) << 4), v1);
              }
              fence_proxy_async_smem();
            }
            tc_fence_before();  // S reads done before the PV MMA may overwrite block 0
            mbar_arrive(&p_full[pst]);
            TRACE(14);
          }
          const float inv = rcp_approx(f2_total(acc));
          if (L.o_sep) mbar_arrive(&s_free[g]);  // S read (tc_fence_before above): the next S may go
          // epilogue: O (64 columns of this slot) / sum -> bf16 row
          mbar_wait(&o_full[g], k & 1);
          TRACE(17);
          tc_fence_after();
          uint32_t o0[32], o1[32], ot[16];
          const uint32_t lo = la + static_cast<uint32_t>(L.o_sep);
          tmem_ld_32x32b_x32(lo, o0);
          tmem_ld_32x32b_x32(lo + 32, o1);
          if constexpr (kTail > 0) tmem_ld_32x32b_x16(lo + kHd, ot);
          tmem_ld_wait();
          tc_fence_before();
          mbar_arrive(L.o_sep ? &o_free[g] : &s_free[g]);
          const int q0 = qt * kQTile + (warp & 3) * 32;
          if (q0 < t) {
            store_o_slab(&tmo, o0, inv, s_slab, lane, h * kHD, q0, b);
            store_o_slab(&tmo, o1, inv, s_slab + 2048, lane, h * kHD + 32, q0, b);
            if constexpr (kTail > 0) store_o_tail(ot, inv, b, q0 + static_cast<int>(lane), h);
          }
          TRACE(18);
          ++k;
        }
      }
    } else {
    // deferred epilogue of the previous tile (two-slot mode)
    bool pend = false;
    uint32_t pend_t = 0;
    int pend_row = 0, pend_h = 0, pend_qt = 0;
    float pend_inv = 0.f;
    uint32_t tcnt = 0;
    // log2(size) of the item's keys j = threadIdx.x + 256 k (k < 2), loaded one item ahead
    auto load_bias = [&](int b_n, float (&v)[2]) {
      const int row_base_n = b_n * t;
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        const int j = threadIdx.x + 256 * k;
        v[k] = (j < t && size != nullptr) ? size[static_cast<long long>(row_base_n) + j] : 1.f;
      }
    };
    float sz_next[2];
    if (static_cast<int>(blockIdx.x) < n_items) load_bias(b_first, sz_next);
    int b = b_first, h = h_first;
    for (int item = blockIdx.x; item < n_items; item += gridDim.x, next_bh(b, h)) {
      float sz[2] = {sz_next[0], sz_next[1]};
      if (item + static_cast<int>(gridDim.x) < n_items) {
        int bn = b, hn = h;
        next_bh(bn, hn);
        load_bias(bn, sz_next);
      }
      if (pend) {  // bias is rewritten below; the deferred epilogue does not read it
        epilogue(pend_t, pend_row, pend_h, pend_qt, pend_inv);
        pend = false;
      }
      named_bar_sync(1, 256);  // everyone is done with the previous item's bias
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        const int j = threadIdx.x + 256 * k;
        if (j < L.t_pad) sts_f32(s_bias + j * 4, j < t ? sz[k] : 0.f);  // key weight
      }
      named_bar_sync(1, 256);
      for (int qt = 0; qt < L.n_qt; ++qt, ++tcnt) {
        const float mx = pass1(tcnt, qt);
        if (pend) {
          epilogue(pend_t, pend_row, pend_h, pend_qt, pend_inv);
          pend = false;
        }
        const float inv = pass2(tcnt, mx, qt);
        if (L.n_s == 2) {
          pend = true;
          pend_t = tcnt;
          pend_row = b;
          pend_h = h;
          pend_qt = qt;
          pend_inv = inv;
        } else {
          epilogue(tcnt, b, h, qt, inv);
        }
      }
    }
    if (pend) epilogue(pend_t, pend_row, pend_h, pend_qt, pend_inv);
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

}  // namespace

int make_tmap_bf16_2d_sw(CUtensorMap* map, const void* base, uint64_t rows, uint64_t cols,
                         uint32_t box_cols, uint32_t box_rows, int swizzle_bytes);

template <bool kHasSize, int kHD, int kKv>
static cudaError_t launch_attn_tc(const cudaLaunchConfig_t& cfg, const CUtensorMap& tm,
                                  const CUtensorMap& tmt, const CUtensorMap& tmo, const float* size,
                                  int t, int H, int n_items, __nv_bfloat16* o, float scale_log2,
                                  const AttnTcLayout& L) {
  static unsigned long long attr_mask = 0;  // per instantiation and device
  if (attr_needed(attr_mask)) {
    const cudaError_t e = cudaFuncSetAttribute(attn_tc_kernel<kHasSize, kHD, kKv>,
                                               cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    if (e != cudaSuccess) return e;
    attr_done(attr_mask);
  }
  return cudaLaunchKernelEx(&cfg, attn_tc_kernel<kHasSize, kHD, kKv>, tm, tmt, tmo, size, t, H, n_items, o,
                            scale_log2, L);
}

// Returns TA_ERR_SHAPE when the shape is outside the tcgen05 kernel's envelope
// (hd not 64 / 80 or t > 512); the caller then uses another kernel.
int attention_tc(const void* qkv, const float* size, int B, int t, int H, int hd, void* out,
                 cudaStream_t s) {
  if ((hd != 64 && hd != 80) || t <= 0 || t > kMaxTPad) return TA_ERR_SHAPE;
  const AttnTcLayout L = attn_layout(t, hd);
  if (L.smem_bytes > 227u * 1024) return TA_ERR_SHAPE;
  const uint64_t rows = static_cast<uint64_t>(B) * t, cols = 3ull * H * hd;
  CUtensorMap tm, tmt, tmo;
  int rc = make_tmap_bf16_2d(&tm, qkv, rows, cols, 64);
  if (rc) return rc;
  tmt = tm;
  if (hd == 80) {  // the 16-column tail of each 80-column head: 32-byte rows, SW32
    rc = make_tmap_bf16_2d_sw(&tmt, qkv, rows, cols, 16, 64, 32);
    if (rc) return rc;
  }
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
  auto* o = static_cast<__nv_bfloat16*>(out);
  cudaError_t e;
#define TA_ATTN_LAUNCH(S, HD, KV) launch_attn_tc<S, HD, KV>(cfg, tm, tmt, tmo, size, t, H, n_items, o, scale_log2, L)
  const bool sz = size != nullptr;
  if (hd == 64 && L.n_kv == 4)
    e = sz ? TA_ATTN_LAUNCH(true, 64, 4) : TA_ATTN_LAUNCH(false, 64, 4);
  else if (hd == 64)
    e = L.n_kv == 1 ? (sz ? TA_ATTN_LAUNCH(true, 64, 1) : TA_ATTN_LAUNCH(false, 64, 1))
                    : (sz ? TA_ATTN_LAUNCH(true, 64, 2) : TA_ATTN_LAUNCH(false, 64, 2));
  else if (L.n_kv <= 2)
    e = L.n_kv == 1 ? (sz ? TA_ATTN_LAUNCH(true, 80, 1) : TA_ATTN_LAUNCH(false, 80, 1))
                    : (sz ? TA_ATTN_LAUNCH(true, 80, 2) : TA_ATTN_LAUNCH(false, 80, 2));
  else
    return TA_ERR_SHAPE;  // (hd 80 never gets four slots: they do not fit)
#undef TA_ATTN_LAUNCH
  return e == cudaSuccess ? TA_OK : set_last_cuda_error(e);
}

#ifdef TA_ATTN_TRACE
extern "C" __attribute__((visibility("default"))) int ta_debug_attn_trace(unsigned long long* t,
                                                                        unsigned int* tag, int max,
                                                                        int reset) {
  // tag 0 = empty slot (event ids start at 1)
  static unsigned int zeros[16384];
  if (reset) return cudaMemcpyToSymbol(g_trace_tag, zeros, sizeof(zeros)) == cudaSuccess ? 0 : -1;
  cudaDeviceSynchronize();
  const int n = max < 16384 ? max : 16384;
  cudaMemcpyFromSymbol(t, g_trace_t, n * sizeof(unsigned long long));
  cudaMemcpyFromSymbol(tag, g_trace_tag, n * sizeof(unsigned int));
  return n;
}
#endif
}  // namespace ta
