// Host+device shared definitions for the tokadapt CUDA library.
#pragma once
#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

#include "../../include/tokadapt_cuda.h"

namespace ta {

// Fused GEMM epilogues.  All GEMMs are C[m, n] = sum_k A[m, k] * W[n, k] (nn.Linear
// layout, both operands K-major) followed by one of these.
enum EpiKind : int {
  EPI_BIAS = 0,        // out(act dtype) = acc + bias
  EPI_BIAS_GELU = 1,   // out(act dtype) = gelu_erf(acc + bias)
  EPI_BIAS_RESID = 2,  // out(fp32)      = resid[m] + acc + bias   (residual stream update)
  EPI_PATCH = 3,       // out(fp32)      = acc + bias + pos[row]   (patch embedding)
  // LayerNorm folded into the next GEMM (bf16 path).  Producers also write xh = bf16(out)
  // and accumulate per-row (sum, sum of squares) of out into stats[out_row] (atomics):
  EPI_BIAS_RESID_STATS = 4,
  EPI_PATCH_STATS = 5,
  // Consumers take A = xh and W' = W o gamma and finish LN(x) W^T + b exactly as
  //   out = rstd * (acc - mu * c1[n]) + c2[n],  c1 = rowsum(W'), c2 = W beta + b,
  // with mu / rstd from ln_stats[m] (eps 1e-6, biased variance):
  EPI_LN_BIAS = 6,     // out(bf16) = LN(x) W^T + b        (QKV)
  EPI_LN_GELU = 7,     // out(bf16) = gelu(LN(x) W^T + b)  (fc1)
  // proj + residual with the ToMe merge's row movement fused in (bf16 path, LN folded): input
  // row m goes to row_map[m] of x' (fp32) with its bf16 copy and row statistics, or -- a merged
  // source token, row_map[m] = -1 - k -- to row k of `side`; merge_fixup then finishes the
  // destination rows (size-weighted averages) and the size vector.
  EPI_BIAS_RESID_MERGE = 8,
};

__host__ __device__ constexpr bool epi_is_stats(int e) {
  return e == EPI_BIAS_RESID_STATS || e == EPI_PATCH_STATS || e == EPI_BIAS_RESID_MERGE;
}
__host__ __device__ constexpr bool epi_is_ln(int e) { return e == EPI_LN_BIAS || e == EPI_LN_GELU; }
__host__ __device__ constexpr bool epi_is_resid(int e) {
  return e == EPI_BIAS_RESID || e == EPI_BIAS_RESID_STATS || e == EPI_BIAS_RESID_MERGE;
}
__host__ __device__ constexpr bool epi_is_patch(int e) { return e == EPI_PATCH || e == EPI_PATCH_STATS; }
__host__ __device__ constexpr bool epi_is_gelu(int e) { return e == EPI_BIAS_GELU || e == EPI_LN_GELU; }

struct GemmEpi {
  const float* bias = nullptr;   // [N]
  const float* resid = nullptr;  // fp32 [M, N], row m of the *input* numbering
  const float* pos = nullptr;    // EPI_PATCH: positional table [*, N], row = row_off + m % rows_in
  void* out = nullptr;           // row-major, row stride N
  // Output row remap: out_row(m) = (m / rows_in) * rows_out + row_off + m % rows_in.
  // rows_in == 0 means identity.  This is how prompt rows are reserved per image
  // (accumulate mode) and how patch rows land after the cls row, without copies.
  int rows_in = 0;
  int rows_out = 0;
  int row_off = 0;
  // LayerNorm folding (EPI_*_STATS producers / EPI_LN_* consumers)
  void* xh = nullptr;               // producer: bf16 copy of out, same rows
  // Row statistics as partials per 128-column block: [rows][stat_slots][2] (sum, sumsq) of
  // the block's values, plain stores (no atomics, no clearing); producers that see whole rows
  // store the full sums in slot 0 and zeros elsewhere.  Consumers add the slots in order.
  float* stats = nullptr;           // producer
  const float* ln_stats = nullptr;  // consumer: stats of the A rows
  int stat_slots = 0;               // D / 128
  const float* c1 = nullptr;        // consumer: [N]
  const float* c2 = nullptr;        // consumer: [N]
  float inv_dim = 0.f;              // consumer: 1 / D
  // EPI_BIAS_RESID_MERGE: output row of input row m in `out`, from the match kernel / merge_map:
  // rows [0, rows_out) are the layer's merged rows (they also get the bf16 copy and statistics),
  // rows [rows_out, M) the merged-away source tokens (image b's k-th source at rows_out + b r + k),
  // which merge_fixup folds into their destinations.
  const int32_t* row_map = nullptr;
  int skip = 0;                     // profiling only (TA_GEMM_SKIP_EPILOGUE=1): no epilogue work
  int direct_store = 0;             // TA_GEMM_STORE=direct: STG.256 rows instead of TMA boxes
  int resid_ldg = 0;                // TA_GEMM_RESID=ldg: residual rows by per-thread loads
};

__host__ __device__ inline long long epi_out_row(const GemmEpi& e, long long m) {
  if (e.rows_in == 0) return m;
  const long long b = m / e.rows_in;
  return b * e.rows_out + e.row_off + (m - b * e.rows_in);
}

// Library status codes (mirrored in include/tokadapt_cuda.h).
int set_last_cuda_error(cudaError_t e);

int device_sm_count();

// Kernel attributes such as the dynamic shared-memory limit are per device: a launcher sets
// them once per (instantiation, device).  `mask` is the launcher's static bit set (bit = device
// ordinal); returns true when the current device still needs the attribute call.  Benign race:
// the attribute call is idempotent.
inline bool attr_needed(const unsigned long long& mask) {
  int dev = 0;
  cudaGetDevice(&dev);
  return !((mask >> (dev & 63)) & 1ull);
}
inline void attr_done(unsigned long long& mask) {
  int dev = 0;
  cudaGetDevice(&dev);
  mask |= 1ull << (dev & 63);
}

// Programmatic dependent launch on every kernel (TA_PDL=0 disables it: profiling A/B).
int pdl_enabled();
int merge_fusion_enabled();

struct HeadDesc {
  const float* w;  // [classes, D]
  const float* b;  // [classes]
  int classes;
};

// Launchers (gemm.cu)
// sk_ws: split-K tail scratch (gemm_splitk_ws_bytes(); null: no split).  Not a GemmEpi field:
// growing that struct changed the generated code of every GEMM instance (fc1 +1.8 %).
int gemm_bf16(const void* A, const void* W, int M, int N, int K, int epi_kind, bool out_bf16,
              const GemmEpi& epi, cudaStream_t stream, float* sk_ws = nullptr);
int gemm_f32(const float* A, const float* W, int M, int N, int K, int epi_kind,
             const GemmEpi& epi, cudaStream_t stream);
// Split-K tail scratch for gemm_bf16 (sk_ws): its first gemm_splitk_flag_bytes() are
// counters the owner zeroes once (cudaMemsetAsync) before the first GEMM that uses it.
size_t gemm_splitk_ws_bytes();
size_t gemm_splitk_flag_bytes();
// Whether gemm_bf16 runs (M, N) on the CTA-pair kernel (the only one with EPI_BIAS_RESID_MERGE).
bool gemm_pair_path(int M, int N);
// fp32 parity mode on the tensor cores: 3xTF32 tcgen05 GEMM (kind::tf32, operands split into
// tf32 hi + lo in `scratch`, gemm_f32_tc_scratch_bytes(M, N, K)); f32_gemm_backend() == 1 when
// TA_F32_GEMM=simt selects the SIMT FFMA kernel instead.
size_t gemm_f32_tc_scratch_bytes(int M, int N, int K);
int gemm_f32_tc(const float* A, const float* W, int M, int N, int K, int epi_kind, const GemmEpi& epi,
                void* scratch, cudaStream_t stream);
int f32_gemm_backend();

// rowops.cu
int patchify(const float* img, void* out, int B, int S, int P, int Kp, int dtype, cudaStream_t s);
int insert_rows(float* x, int B, int t_total, int D, const float* cls, const float* pos,
                const float* const* prompt_tab, const int32_t* task_ids, int n_tasks, int layer,
                int gamma, int prompt_row, cudaStream_t s, void* xh = nullptr,
                float* stats = nullptr);
int layernorm(const float* x, const float* w, const float* b, void* out, int rows, int D,
              int out_dtype, cudaStream_t s);
int head(const float* x, int B, int t_total, int D, const float* nw, const float* nb,
         const HeadDesc* heads, const int32_t* task, int n_tasks, float* logits, int c_max,
         cudaStream_t s);

// tome.cu.  metric source: either fp32 [B, t, c] (metric != null) or the k third of a
// qkv activation [B, t, 3*H*c] in `qkv_dtype`, averaged over heads (ToMe k.mean(1)).
// scratch (nullable): match_tc_scratch_bytes(B, c) bytes; with it the tcgen05 path runs
// (TA_MATCH_BACKEND=simt forces the SIMT kernel), without it the SIMT kernel.
// row_map (nullable): also emit the fused merge's per-row destination map (merge_map's output).
int match(const float* metric, const void* qkv, int qkv_dtype, int B, int t, int heads, int c,
          int r, int32_t* src, int32_t* dst, int32_t* unm, float* scratch, cudaStream_t s,
          int32_t* row_map = nullptr);
size_t match_tc_scratch_bytes(int B, int c);
int match_tc(const float* metric, const void* qkv, int qkv_dtype, int B, int t, int heads, int c,
             int r, int32_t* src, int32_t* dst, int32_t* unm, float* scratch, cudaStream_t s,
             int32_t* row_map = nullptr);
// Fused merge (bf16 path): merge_map turns a layer's (src, unm) into the per-row destination map
// of EPI_BIAS_RESID_MERGE; merge_fixup, after that GEMM, computes the size-weighted rows of the
// destination tokens that received sources (and their bf16 copy / row statistics) and the new
// size vector.
int merge_map(const int32_t* src, const int32_t* unm, int B, int t, int r, int32_t* row_map,
              cudaStream_t s);
int merge_fixup(float* x_out, const float* side, const float* size, float* size_out, int B, int t,
                int D, int r, const int32_t* src, const int32_t* dst, const int32_t* unm, void* xh,
                float* stats, cudaStream_t s);
int merge(const float* x, const float* size, int B, int t, int D, int r, const int32_t* src,
          const int32_t* dst, const int32_t* unm, const float* ln_w, const float* ln_b,
          float* x_out, float* size_out, void* h_out, int h_dtype, cudaStream_t s,
          float* stats_out = nullptr);  // stats_out: write bf16(x') + row (sum, sumsq) instead of LN2

// attention.cu / attention_tc.cu
int attention_tc(const void* qkv, const float* size, int B, int t, int H, int hd, void* out,
                 cudaStream_t s);
int attention_fa(const void* qkv, const float* size, int B, int t, int H, int hd, void* out,
                 cudaStream_t s);
int attention_tp(const void* qkv, const float* size, int B, int t, int H, int hd, void* out,
                 cudaStream_t s);
int attention(const void* qkv, const float* size, int B, int t, int H, int hd, void* out,
              int dtype, cudaStream_t s);

}  // namespace ta
