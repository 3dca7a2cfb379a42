/*
 * tokadapt_cuda.h — C ABI of the B200-native token-adapted ViT forward
 * (OTAS, arXiv 2401.05031) implemented in libtokadapt_cuda.so.
 *
 * The reference has no native code and no FFI for this path:
 * the model execution it abstracts sits behind
 *   - ServeModel.forward(inputs, tasks, task_params, gamma)
 *   - TaskModel = prompts + head per task
 *   - TransformerModel with prompt module (before norm) and merge
 *     module (before MLP)
 *   - estimate_batch(batch, gamma, table) -> (time_us, utility)    pkg/src/tokadapt/profiles.py:124
 * Each entry point below names the reference interface it replaces.
 *
 * Conventions
 *   - plain C types only; every function returns int status (0 = ok, < 0 = error)
 *     and never throws or exits; ta_strerror() maps codes to text;
 *   - all device buffers are caller-owned; nothing here allocates device memory
 *     inside ta_forward (caller passes a workspace sized by ta_workspace_size),
 *     which keeps ta_forward CUDA-graph capturable;
 *   - every call is asynchronous on the caller's cudaStream_t (passed as void*);
 *   - one ta_model handle per device, used from one stream at a time.
 */
#ifndef TOKADAPT_CUDA_H
#define TOKADAPT_CUDA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TA_ABI_VERSION 3

/* Status codes.  Python maps them onto the reference's exception types
 * (pkg/src/tokadapt/errors.py): TA_ERR_NO_PROMPT -> ProfileGapError(task, gamma,
 * "prompt"); TA_ERR_INVALID / TA_ERR_SHAPE -> ValueError; TA_ERR_CONFIG ->
 * ConfigError; TA_ERR_CUDA / TA_ERR_ARCH -> RuntimeError. */
enum {
  TA_OK = 0,
  TA_ERR_INVALID = -1,    /* bad argument (null pointer, gamma out of range, ...) */
  TA_ERR_SHAPE = -2,      /* unsupported shape / alignment */
  TA_ERR_CONFIG = -3,     /* inconsistent model description */
  TA_ERR_NO_PROMPT = -4,  /* gamma > 0 but no prompts registered for (task, gamma) */
  TA_ERR_NO_WEIGHTS = -5, /* ta_forward before ta_model_set_weights / missing head */
  TA_ERR_WORKSPACE = -6,  /* workspace too small */
  TA_ERR_CUDA = -7,       /* CUDA runtime/driver error (see ta_last_cuda_error) */
  TA_ERR_ARCH = -8        /* device is not sm_100 */
};

enum { TA_DTYPE_BF16 = 0, TA_DTYPE_F32 = 1 };
/* Prompt semantics (SURVEY.md §7 "Prompt semantics are ambiguous"):
 * ACCUMULATE adds gamma new prompt rows before every layer (t_l = N + gamma(l+1),
 * matches profiles.py:165 tokens = n_i + gamma*L); REPLACE is VPT-deep (gamma rows
 * inserted before layer 0 and overwritten before each later layer). */
enum { TA_PROMPT_ACCUMULATE = 0, TA_PROMPT_REPLACE = 1 };

int ta_abi_version(void);
const char* ta_strerror(int code);
/* The cudaError_t value behind the last TA_ERR_CUDA on this thread. */
int ta_last_cuda_error(void);

/* ------------------------------------------------------------------ model */
/* Replaces: TransformerModel(...) construction. */
typedef struct ta_model_desc {
  int dim;          /* D: 768 (B/16), 1024 (L/16), 1280 (H/14) */
  int depth;        /* L: 12 / 24 / 32 */
  int heads;        /* H: 12 / 16 / 16 (head dim D/H must be 64 or 80) */
  int mlp_dim;      /* 4D */
  int patch;        /* P: 16 / 14 */
  int img;          /* 224 */
  int n_tasks;      /* number of TaskModels (heads + prompt sets) */
  int max_classes;  /* C_max over tasks; logits are [B, max_classes] */
  int prompt_mode;  /* TA_PROMPT_* */
  int dtype;        /* TA_DTYPE_BF16 (tcgen05) or TA_DTYPE_F32 (fp32 parity mode) */
} ta_model_desc;

typedef struct ta_model ta_model;

/* Per-layer weights.  Matrices use the nn.Linear layout [out, in] in the model
 * dtype; vectors are fp32. */
typedef struct ta_layer_weights {
  const void* ln1_w;
  const void* ln1_b;
  const void* qkv_w; /* [3D, D], rows ordered s*D + h*hd + j (s = q,k,v) */
  const void* qkv_b;
  const void* proj_w; /* [D, D] */
  const void* proj_b;
  const void* ln2_w;
  const void* ln2_b;
  const void* fc1_w; /* [MLP, D] */
  const void* fc1_b;
  const void* fc2_w; /* [D, MLP] */
  const void* fc2_b;
  /* Optional (bf16 mode; all six or none): LayerNorm folded into the QKV / fc1 GEMMs.
   *   *_w_ln = bf16(W o gamma)  [out, in]     (gamma = ln1_w for QKV, ln2_w for fc1)
   *   *_c1   = fp32 row sums of *_w_ln [out]
   *   *_c2   = fp32 W beta + b [out]          (beta = ln1_b / ln2_b)
   * With them ta_forward drops the LayerNorm passes: the residual's producers also emit a
   * bf16 copy and per-row (sum, sumsq), and the GEMM epilogue finishes
   * LN(x) W^T + b = rstd (x W_ln^T - mu c1) + c2. */
  const void* qkv_w_ln;
  const void* qkv_c1;
  const void* qkv_c2;
  const void* fc1_w_ln;
  const void* fc1_c1;
  const void* fc1_c2;
} ta_layer_weights;

typedef struct ta_weights {
  const void* patch_w; /* [D, Kp] model dtype; Kp = 3P^2 rounded up to 64, zero padded */
  const void* patch_b; /* fp32 [D] */
  const void* cls;     /* fp32 [D] */
  const void* pos;     /* fp32 [N, D], N = (img/P)^2 + 1 */
  const void* norm_w;  /* fp32 [D] final LayerNorm */
  const void* norm_b;
  const ta_layer_weights* layers; /* [depth]; copied, pointers must outlive the model */
} ta_weights;

int ta_model_create(int device, const ta_model_desc* desc, ta_model** out);
void ta_model_destroy(ta_model* model);
int ta_model_set_weights(ta_model* model, const ta_weights* w);
/* Replaces: TaskModel head.  W fp32 [C, D], b fp32 [C]. */
int ta_model_set_head(ta_model* model, int task, const float* w, const float* b, int classes);
/* Replaces: prompt repository lookup keyed by (task, gamma).
 * prompts fp32 [depth, gamma, D] (REPLACE mode reads row block 0..depth-1 the same way). */
int ta_model_set_prompts(ta_model* model, int task, int gamma, const float* prompts);

/* Token schedule t_l (tokens entering layer l) and r_l (tokens merged in layer l)
 * for a gamma: ToMe parse_r with constant r and the per-layer cap
 * r_l = min(|gamma|, (t_l - 1) / 2).  Arrays have depth entries. */
int ta_token_schedule(const ta_model* model, int gamma, int* t_out, int* r_out);
/* Int32 count of the merge trace for (batch, gamma): per merge layer l in order,
 * src [B, r_l], dst [B, r_l], unm [B, ceil(t_l/2) - r_l]. */
int ta_merge_trace_len(const ta_model* model, int batch, int gamma, size_t* n_int32);
int ta_workspace_size(const ta_model* model, int batch, int gamma, size_t* bytes);

/* Replaces: ServeModel.forward(inputs, tasks, task_params, gamma).
 *   images     fp32 [B, 3, img, img] (device)
 *   task_ids   int32 [B] (device), each < n_tasks
 *   logits     fp32 [B, max_classes] (device); columns >= C_task are -inf
 *   merge_trace  nullable int32 out (device), layout of ta_merge_trace_len
 *   forced_trace nullable int32 in: replay these merge indices instead of matching
 *                (teacher forcing for parity tests)
 *   ws / ws_bytes  device workspace (>= ta_workspace_size)
 *   stream     cudaStream_t */
int ta_forward(ta_model* model, const float* images, const int32_t* task_ids, int batch,
               int gamma, float* logits, int32_t* merge_trace, const int32_t* forced_trace,
               void* ws, size_t ws_bytes, void* stream);

/* Host-buffer convenience (the reference-facing e2e path): pinned or pageable host
 * images/task ids in, host logits out; copies and the forward run on `stream`,
 * which is synchronised before returning.  Uses an internally cached workspace. */
int ta_forward_host(ta_model* model, const float* images_host, const int32_t* task_ids_host,
                    int batch, int gamma, float* logits_host, void* stream);

/* ------------------------------------------------------------ unit kernels
 * Exposed for parity tests of each hot-path stage. */

/* a9: ToMe bipartite soft matching (upstream tome/merge.py::bipartite_soft_matching,
 * restated in SURVEY.md Appendix A).  metric fp32 [B, t, c] (un-normalised),
 * outputs int32 src/dst [B, r], unm [B, ceil(t/2) - r].  Class token protected. */
int ta_match(const float* metric, int batch, int t, int c, int r, int32_t* src, int32_t* dst,
             int32_t* unm, void* stream);
/* a8+a9 as the forward runs them: the metric is the head mean of the k third of a qkv
 * activation [B, t, 3 H hd] in `dtype` (ToMe k.mean(1)), computed inside the matching kernel
 * (bf16: the 1xTF32 tcgen05 instance the bf16 forward launches; fp32: 3xTF32). */
int ta_match_qkv(const void* qkv, int dtype, int batch, int t, int heads, int head_dim, int r,
                 int32_t* src, int32_t* dst, int32_t* unm, void* stream);
/* a10: size-weighted merge (tome merge_wavg) + fused LN2.  x fp32 [B, t, D], size fp32
 * [B, t] or NULL (= ones).  Writes x_out fp32 [B, t-r, D], size_out [B, t-r] and
 * h_out = LayerNorm(x_out) in `h_dtype` (TA_DTYPE_*). */
int ta_merge(const float* x, const float* size, int batch, int t, int dim, int r,
             const int32_t* src, const int32_t* dst, const int32_t* unm, const float* ln_w,
             const float* ln_b, float* x_out, float* size_out, void* h_out, int h_dtype,
             void* stream);
/* a6: proportional attention softmax(q k^T / sqrt(hd) + log size) v per (image, head).
 * qkv [B, t, 3D] in `dtype`, size fp32 [B, t] or NULL; out [B, t, D] in `dtype`. */
int ta_attention(const void* qkv, const float* size, int batch, int t, int heads, int head_dim,
                 void* out, int dtype, void* stream);
/* a5/a7/a11: C = A W^T with a fused epilogue (0 bias, 1 bias+GELU, 2 bias+residual fp32,
 * 3 bias+pos).  bf16 path runs on tcgen05; fp32 path is the SIMT parity kernel. */
int ta_gemm(const void* a, const void* w, const float* bias, const float* resid, void* out,
            int m, int n, int k, int epilogue, int dtype, int out_dtype, void* stream);
/* a4: row LayerNorm eps 1e-6, fp32 in, `out_dtype` out. */
int ta_layernorm(const float* x, const float* w, const float* b, void* out, int rows, int dim,
                 int out_dtype, void* stream);

/* ------------------------------------------------------------ stage timing
 * Measurement support: with ta_profile_stages(model, 1) every ta_forward
 * records CUDA events around each stage on its stream and synchronises at the end (so it is
 * not graph-capturable while on); ta_stage_records returns the (stage, layer, device us)
 * list of the last such forward in launch order (layer -1 = outside the layer loop). */
enum {
  TA_STAGE_PATCHIFY = 0, TA_STAGE_PATCH_GEMM, TA_STAGE_INSERT_ROWS, TA_STAGE_LN1, TA_STAGE_QKV,
  TA_STAGE_ATTENTION, TA_STAGE_PROJ, TA_STAGE_MATCH, TA_STAGE_MERGE, TA_STAGE_LN2, TA_STAGE_FC1,
  TA_STAGE_FC2, TA_STAGE_HEAD, TA_N_STAGES
};
typedef struct ta_stage_record {
  int stage;
  int layer;
  float us;
} ta_stage_record;
const char* ta_stage_name(int stage);
int ta_profile_stages(ta_model* model, int on);
int ta_stage_records(const ta_model* model, ta_stage_record* out, int max_records, int* n);

#ifdef __cplusplus
}
#endif
#endif /* TOKADAPT_CUDA_H */
