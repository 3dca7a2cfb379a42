// Token-adapted ViT forward and the C ABI of
// include/tokadapt_cuda.h.
//
// One call of ta_forward runs, for a batch at one gamma:
//   patchify -> patch GEMM (+bias +pos, rows placed after cls / before prompts)
//   -> cls / prompt rows -> L x [ prompts, LN1, QKV GEMM, attention(+log size),
//      proj GEMM (+residual), (match, merge+LN2) | LN2, fc1 GEMM (+GELU),
//      fc2 GEMM (+residual, rows re-strided for next-layer prompts) ]
//   -> final LN on cls + per-task head.
// The per-layer token count t_l is static per (model, gamma); all buffers live in the
// caller's workspace, so the whole call is CUDA-graph capturable.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <cstring>
#include <map>
#include <mutex>
#include <vector>

#include "common.h"

namespace ta {

static thread_local int g_last_cuda_error = 0;
int set_last_cuda_error(cudaError_t e) {
  g_last_cuda_error = static_cast<int>(e);
  return TA_ERR_CUDA;
}

int device_sm_count() {
  static int count = 0;
  if (count == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&count, cudaDevAttrMultiProcessorCount, dev);
    if (count <= 0) count = 148;
  }
  return count;
}

// Fused proj + merge on the bf16 LN-folded path (default; TA_MERGE_FUSION=0 restores the
// separate merge kernel): the match runs before attention and also emits the row map, the proj
// GEMM writes rows to their merged positions plus their bf16 copy / statistics, merge_fixup
// finishes the destination rows.  One full read + write of the fp32 residual less per merge
// layer than proj + merge_kernel.
int merge_fusion_enabled() {
  static int on = -1;
  if (on < 0) {
    const char* v = getenv("TA_MERGE_FUSION");
    on = (v && v[0] == '0') ? 0 : 1;
  }
  return on;
}

// Split-K tail tiles in the forward's GEMMs (gemm.cu splitk_parts), TA_GEMM_SPLITK_FWD=1.  Off by
// default: a row's fp32 summation order then depends on whether its tile falls in a launch's
// last wave, so an image's logits would change (in the last bits) with its batch position, and
// the measured gain is within the sweep's noise.
static int splitk_fwd_enabled() {
  static int on = -1;
  if (on < 0) {
    const char* v = getenv("TA_GEMM_SPLITK_FWD");
    on = (v && v[0] == '1') ? 1 : 0;
  }
  return on;
}

int pdl_enabled() {
  static int on = -1;
  if (on < 0) {
    const char* v = getenv("TA_PDL");
    on = (v && v[0] == '0') ? 0 : 1;
  }
  return on;
}

// Makes `device` current for the scope of an ABI call and restores the caller's device
// (torch keeps its own notion of the current device; the library must not move it).
struct DeviceGuard {
  int prev = -1;
  cudaError_t err = cudaSuccess;
  explicit DeviceGuard(int device) {
    cudaGetDevice(&prev);
    if (prev != device) err = cudaSetDevice(device);
  }
  ~DeviceGuard() {
    int cur = -1;
    cudaGetDevice(&cur);
    if (prev >= 0 && cur != prev) cudaSetDevice(prev);
  }
};

static int check_arch(int device) {
  int major = 0, minor = 0;
  cudaError_t e = cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, device);
  if (e != cudaSuccess) return set_last_cuda_error(e);
  cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, device);
  return (major == 10 && minor == 0) ? TA_OK : TA_ERR_ARCH;
}

}  // namespace ta

using namespace ta;

struct ta_model {
  int device = 0;
  ta_model_desc d{};
  int hd = 0, grid = 0, n_patches = 0, n_tokens = 0, kp = 0;
  bool has_weights = false;
  bool ln_folded = false;  // every layer has the LN-folded QKV / fc1 weights
  ta_weights w{};
  std::vector<ta_layer_weights> layers;
  std::vector<HeadDesc> heads;  // host copy
  HeadDesc* heads_dev = nullptr;
  std::map<int, std::vector<const float*>> prompts;  // gamma -> per-task pointer
  std::map<int, const float**> prompt_tab;             // gamma -> device table [n_tasks]
  // per-stage device times of the last profiled forward (ta_profile_stages)
  int profile_on = 0;
  std::vector<ta_stage_record> records;
  // ta_forward_host cache
  void* host_ws = nullptr;
  size_t host_ws_bytes = 0;
  std::mutex host_mu;
};

namespace {

struct Schedule {
  std::vector<int> t, r;
  int t_max = 0, t_final = 0;
};

Schedule make_schedule(const ta_model* m, int gamma) {
  Schedule s;
  const int L = m->d.depth, N = m->n_tokens;
  int t = N;
  for (int l = 0; l < L; ++l) {
    int tl, rl = 0;
    if (gamma > 0) {
      tl = m->d.prompt_mode == TA_PROMPT_ACCUMULATE ? N + gamma * (l + 1) : N + gamma;
    } else {
      tl = t;
      if (gamma < 0) rl = std::min(-gamma, (tl - 1) / 2);
      if (rl < 0) rl = 0;
    }
    s.t.push_back(tl);
    s.r.push_back(rl);
    s.t_max = std::max(s.t_max, tl);
    t = tl - rl;
  }
  s.t_final = t;
  return s;
}

size_t align_up(size_t v) { return (v + 255) & ~static_cast<size_t>(255); }

struct Workspace {
  void* patches;
  float* x[2];
  void* h;
  void* qkv;
  void* attn;
  void* mlp;
  float* size[2];
  int32_t* src;
  int32_t* dst;
  int32_t* unm;
  float* match_scratch;
  float* stats[2];  // LN-folded path: per-row (sum, sumsq) for LN1 / LN2
  void* tf32_scratch;  // fp32 mode: tf32 hi / lo operand split of the 3xTF32 GEMMs
  int32_t* row_map;  // fused merge: destination of every input row (merge_map); the merged-away
                     // source rows land after the merged rows in x (rows <= B t_max)
  float* sk_ws;      // bf16 + TA_GEMM_SPLITK_FWD=1: split-K partials + counters, zeroed per forward
  size_t total;
};

Workspace carve(const ta_model* m, int B, const Schedule& s, char* base) {
  const size_t A = m->d.dtype == TA_DTYPE_BF16 ? 2 : 4;
  const size_t D = m->d.dim, rows = static_cast<size_t>(B) * s.t_max;
  Workspace w{};
  size_t off = 0;
  auto take = [&](size_t bytes) {
    char* p = base ? base + off : nullptr;
    off += align_up(bytes);
    return p;
  };
  w.patches = take(static_cast<size_t>(B) * m->n_patches * m->kp * A);
  w.x[0] = reinterpret_cast<float*>(take(rows * D * 4));
  w.x[1] = reinterpret_cast<float*>(take(rows * D * 4));
  w.h = take(rows * D * A);
  w.qkv = take(rows * 3 * D * A);
  w.attn = take(rows * D * A);
  w.mlp = take(rows * m->d.mlp_dim * A);
  w.size[0] = reinterpret_cast<float*>(take(rows * 4));
  w.size[1] = reinterpret_cast<float*>(take(rows * 4));
  w.src = reinterpret_cast<int32_t*>(take(rows * 4));
  w.dst = reinterpret_cast<int32_t*>(take(rows * 4));
  w.unm = reinterpret_cast<int32_t*>(take(rows * 4));
  w.match_scratch = reinterpret_cast<float*>(take(match_tc_scratch_bytes(B, m->hd)));
  // LN-folded path: per-row partial (sum, sumsq) per 128-column block (GemmEpi::stats)
  w.stats[0] = reinterpret_cast<float*>(take(rows * 8 * (D / 128)));
  w.stats[1] = reinterpret_cast<float*>(take(rows * 8 * (D / 128)));
  int r_max = 0;
  for (int r : s.r) r_max = std::max(r_max, r);
  // fp32 mode: the largest GEMM operand pair (rows x MLP for fc2's A, MLP x D for its W)
  w.tf32_scratch = take(m->d.dtype == TA_DTYPE_F32
                            ? gemm_f32_tc_scratch_bytes(static_cast<int>(rows), m->d.mlp_dim,
                                                        std::max(m->d.mlp_dim, m->kp))
                            : 0);
  w.row_map = reinterpret_cast<int32_t*>(take(r_max > 0 ? rows * 4 : 0));
  w.sk_ws = m->d.dtype == TA_DTYPE_BF16 && splitk_fwd_enabled()
                ? reinterpret_cast<float*>(take(gemm_splitk_ws_bytes()))
                : nullptr;
  w.total = off;
  return w;
}

int linear(const ta_model* m, const void* a, const void* wt, int M, int N, int K, int epi_kind,
           const GemmEpi& epi_in, cudaStream_t st, const Workspace& w) {
  void* const tf32_scratch = w.tf32_scratch;
  const GemmEpi& epi = epi_in;
  if (m->d.dtype == TA_DTYPE_BF16)
    return gemm_bf16(a, wt, M, N, K, epi_kind, epi_kind == EPI_BIAS || epi_kind == EPI_BIAS_GELU || epi_is_ln(epi_kind),
                     epi, st, w.sk_ws);
  if (f32_gemm_backend() == 0)
    return gemm_f32_tc(static_cast<const float*>(a), static_cast<const float*>(wt), M, N, K, epi_kind, epi,
                       tf32_scratch, st);
  return gemm_f32(static_cast<const float*>(a), static_cast<const float*>(wt), M, N, K, epi_kind,
                  epi, st);
}

size_t trace_len(const Schedule& s, int B) {
  size_t n = 0;
  for (size_t l = 0; l < s.t.size(); ++l)
    if (s.r[l] > 0) n += static_cast<size_t>(B) * (2 * s.r[l] + (s.t[l] + 1) / 2 - s.r[l]);
  return n;
}

}  // namespace

#define TA_TRY(expr)          \
  do {                        \
    int _rc = (expr);         \
    if (_rc != TA_OK) return _rc; \
  } while (0)

// Stage timing (profiling only; never inside a graph): CUDA events around every stage of
// ta_forward.  ta_profile_stages(m, 1) keeps per-(stage, layer) device times in the model for
// ta_stage_records; TA_PROFILE_STAGES=1 prints per-stage sums to stderr.
namespace {
struct StageProfiler {
  bool on = false, print = false;
  ta_model* m = nullptr;
  cudaStream_t st = nullptr;
  struct Mark {
    int stage, layer;
    cudaEvent_t ev;
  };
  std::vector<Mark> marks;
  StageProfiler(cudaStream_t s, ta_model* model) : m(model), st(s) {
    const char* v = getenv("TA_PROFILE_STAGES");
    print = v && v[0] == '1';
    on = print || (m && m->profile_on);
    mark(-1, -1);
  }
  void mark(int stage, int layer) {
    if (!on) return;
    cudaEvent_t e;
    cudaEventCreate(&e);
    cudaEventRecord(e, st);
    marks.push_back({stage, layer, e});
  }
  ~StageProfiler() {
    if (!on || marks.size() < 2) return;
    cudaEventSynchronize(marks.back().ev);
    std::vector<ta_stage_record> recs;
    for (size_t i = 1; i < marks.size(); ++i) {
      float ms = 0.f;
      cudaEventElapsedTime(&ms, marks[i - 1].ev, marks[i].ev);
      recs.push_back({marks[i].stage, marks[i].layer, ms * 1e3f});
    }
    if (m && m->profile_on) m->records = recs;
    if (print) {
      float agg[TA_N_STAGES] = {};
      int cnt[TA_N_STAGES] = {};
      float total = 0.f;
      for (const auto& r : recs) {
        agg[r.stage] += r.us;
        cnt[r.stage] += 1;
        total += r.us;
      }
      for (int k = 0; k < TA_N_STAGES; ++k)
        if (cnt[k]) fprintf(stderr, "[ta stage] %-14s n=%3d %9.1f us\n", ta_stage_name(k), cnt[k], agg[k]);
      fprintf(stderr, "[ta stage] total %9.1f us\n", total);
    }
    for (auto& mk : marks) cudaEventDestroy(mk.ev);
  }
};
}  // namespace

extern "C" {
#pragma GCC visibility push(default)

int ta_abi_version(void) { return TA_ABI_VERSION; }

const char* ta_strerror(int code) {
  switch (code) {
    case TA_OK: return "ok";
    case TA_ERR_INVALID: return "invalid argument";
    case TA_ERR_SHAPE: return "unsupported shape or alignment";
    case TA_ERR_CONFIG: return "inconsistent model description";
    case TA_ERR_NO_PROMPT: return "no prompts registered for (task, gamma)";
    case TA_ERR_NO_WEIGHTS: return "weights or task head not set";
    case TA_ERR_WORKSPACE: return "workspace too small";
    case TA_ERR_CUDA: return "CUDA error";
    case TA_ERR_ARCH: return "device is not sm_100 (B200)";
  }
  return "unknown error";
}

int ta_last_cuda_error(void) { return g_last_cuda_error; }

const char* ta_stage_name(int stage) {
  static const char* const kNames[TA_N_STAGES] = {
      "patchify", "patch_gemm", "insert_rows", "ln1", "qkv", "attention", "proj",
      "match",    "merge",      "ln2",         "fc1", "fc2", "head"};
  return (stage >= 0 && stage < TA_N_STAGES) ? kNames[stage] : "?";
}

int ta_profile_stages(ta_model* m, int on) {
  if (!m) return TA_ERR_INVALID;
  m->profile_on = on ? 1 : 0;
  m->records.clear();
  return TA_OK;
}

int ta_stage_records(const ta_model* m, ta_stage_record* out, int max_records, int* n) {
  if (!m || !n || (max_records > 0 && !out)) return TA_ERR_INVALID;
  *n = static_cast<int>(m->records.size());
  for (int i = 0; i < *n && i < max_records; ++i) out[i] = m->records[i];
  return TA_OK;
}

int ta_model_create(int device, const ta_model_desc* desc, ta_model** out) {
  if (!desc || !out) return TA_ERR_INVALID;
  const ta_model_desc& d = *desc;
  if (d.dim <= 0 || d.depth <= 0 || d.depth > 64 || d.heads <= 0 || d.dim % d.heads ||
      d.patch <= 0 || d.img % d.patch || d.n_tasks <= 0 || d.max_classes <= 0 ||
      d.mlp_dim <= 0 || (d.dtype != TA_DTYPE_BF16 && d.dtype != TA_DTYPE_F32) ||
      (d.prompt_mode != TA_PROMPT_ACCUMULATE && d.prompt_mode != TA_PROMPT_REPLACE))
    return TA_ERR_CONFIG;
  const int hd = d.dim / d.heads;
  if (hd != 64 && hd != 80) return TA_ERR_CONFIG;
  if (d.dim % 256 != 0 || d.mlp_dim % 256 != 0) return TA_ERR_CONFIG;
  DeviceGuard guard(device);
  if (guard.err != cudaSuccess) return set_last_cuda_error(guard.err);
  TA_TRY(check_arch(device));
  cudaError_t e;
  auto* m = new ta_model();
  m->device = device;
  m->d = d;
  m->hd = hd;
  m->grid = d.img / d.patch;
  m->n_patches = m->grid * m->grid;
  m->n_tokens = m->n_patches + 1;
  m->kp = (3 * d.patch * d.patch + 63) / 64 * 64;
  m->heads.assign(d.n_tasks, HeadDesc{nullptr, nullptr, 0});
  e = cudaMalloc(&m->heads_dev, sizeof(HeadDesc) * d.n_tasks);
  if (e != cudaSuccess) {
    delete m;
    return set_last_cuda_error(e);
  }
  cudaMemcpy(m->heads_dev, m->heads.data(), sizeof(HeadDesc) * d.n_tasks, cudaMemcpyHostToDevice);
  *out = m;
  return TA_OK;
}

void ta_model_destroy(ta_model* m) {
  if (!m) return;
  DeviceGuard guard(m->device);
  cudaFree(m->heads_dev);
  for (auto& kv : m->prompt_tab) cudaFree(kv.second);
  if (m->host_ws) cudaFree(m->host_ws);
  delete m;
}

int ta_model_set_weights(ta_model* m, const ta_weights* w) {
  if (!m || !w || !w->layers || !w->patch_w || !w->patch_b || !w->cls || !w->pos || !w->norm_w ||
      !w->norm_b)
    return TA_ERR_INVALID;
  for (int l = 0; l < m->d.depth; ++l) {
    const ta_layer_weights& L = w->layers[l];
    if (!L.ln1_w || !L.ln1_b || !L.qkv_w || !L.qkv_b || !L.proj_w || !L.proj_b || !L.ln2_w ||
        !L.ln2_b || !L.fc1_w || !L.fc1_b || !L.fc2_w || !L.fc2_b)
      return TA_ERR_INVALID;
  }
  m->w = *w;
  m->layers.assign(w->layers, w->layers + m->d.depth);
  bool folded = true;
  for (const ta_layer_weights& L : m->layers)
    folded = folded && L.qkv_w_ln && L.qkv_c1 && L.qkv_c2 && L.fc1_w_ln && L.fc1_c1 && L.fc1_c2;
  // the folded epilogues exist on the tcgen05 kernels (N % 256 == 0) only
  m->ln_folded = folded && m->d.dtype == TA_DTYPE_BF16 && (3 * m->d.dim) % 256 == 0 &&
                 m->d.mlp_dim % 256 == 0;
  m->w.layers = m->layers.data();
  m->has_weights = true;
  return TA_OK;
}

int ta_model_set_head(ta_model* m, int task, const float* w, const float* b, int classes) {
  if (!m || !w || !b || task < 0 || task >= m->d.n_tasks || classes <= 0 ||
      classes > m->d.max_classes)
    return TA_ERR_INVALID;
  m->heads[task] = HeadDesc{w, b, classes};
  DeviceGuard guard(m->device);
  cudaError_t e = cudaMemcpy(m->heads_dev + task, &m->heads[task], sizeof(HeadDesc),
                             cudaMemcpyHostToDevice);
  return e == cudaSuccess ? TA_OK : set_last_cuda_error(e);
}

int ta_model_set_prompts(ta_model* m, int task, int gamma, const float* prompts) {
  if (!m || !prompts || task < 0 || task >= m->d.n_tasks || gamma <= 0) return TA_ERR_INVALID;
  DeviceGuard guard(m->device);
  auto& vec = m->prompts[gamma];
  if (vec.empty()) vec.assign(m->d.n_tasks, nullptr);
  vec[task] = prompts;
  const float** tab = nullptr;
  auto it = m->prompt_tab.find(gamma);
  if (it == m->prompt_tab.end()) {
    cudaError_t e = cudaMalloc(&tab, sizeof(float*) * m->d.n_tasks);
    if (e != cudaSuccess) return set_last_cuda_error(e);
    m->prompt_tab[gamma] = tab;
  } else {
    tab = it->second;
  }
  cudaError_t e = cudaMemcpy(tab, vec.data(), sizeof(float*) * m->d.n_tasks, cudaMemcpyHostToDevice);
  return e == cudaSuccess ? TA_OK : set_last_cuda_error(e);
}

int ta_token_schedule(const ta_model* m, int gamma, int* t_out, int* r_out) {
  if (!m || !t_out || !r_out) return TA_ERR_INVALID;
  Schedule s = make_schedule(m, gamma);
  std::copy(s.t.begin(), s.t.end(), t_out);
  std::copy(s.r.begin(), s.r.end(), r_out);
  return TA_OK;
}

int ta_merge_trace_len(const ta_model* m, int batch, int gamma, size_t* n) {
  if (!m || !n || batch <= 0) return TA_ERR_INVALID;
  *n = trace_len(make_schedule(m, gamma), batch);
  return TA_OK;
}

int ta_workspace_size(const ta_model* m, int batch, int gamma, size_t* bytes) {
  if (!m || !bytes || batch <= 0) return TA_ERR_INVALID;
  *bytes = carve(m, batch, make_schedule(m, gamma), nullptr).total;
  return TA_OK;
}

int ta_forward(ta_model* m, const float* images, const int32_t* task_ids, int B, int gamma,
               float* logits, int32_t* merge_trace, const int32_t* forced_trace, void* ws,
               size_t ws_bytes, void* stream) {
  if (!m || !images || !task_ids || !logits || !ws || B <= 0) return TA_ERR_INVALID;
  if (!m->has_weights) return TA_ERR_NO_WEIGHTS;
  // Task ids are device-side here, so heads / prompts are validated per task only where the
  // ids are known on the host (ta_forward_host, the Python front end).  At least one head
  // must exist; an image whose task has no head, no prompts at this gamma, or an id outside
  // [0, n_tasks) is never dereferenced and gets NaN logits (rowops.cu insert_rows / head).
  bool any_head = false;
  for (int k = 0; k < m->d.n_tasks; ++k) any_head = any_head || m->heads[k].w != nullptr;
  if (!any_head) return TA_ERR_NO_WEIGHTS;
  const float* const* ptab = nullptr;
  if (gamma > 0) {
    auto it = m->prompt_tab.find(gamma);
    if (it == m->prompt_tab.end()) return TA_ERR_NO_PROMPT;  // no task has prompts at gamma
    ptab = it->second;
  }
  if (gamma < -(m->n_tokens - 1)) return TA_ERR_INVALID;
  const Schedule s = make_schedule(m, gamma);
  Workspace w = carve(m, B, s, static_cast<char*>(ws));
  if (ws_bytes < w.total) return TA_ERR_WORKSPACE;
  DeviceGuard guard(m->device);
  if (guard.err != cudaSuccess) return set_last_cuda_error(guard.err);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  StageProfiler prof(st, m);
  if (w.sk_ws) {  // split-K counters start at zero (each GEMM leaves them zero)
    cudaError_t me = cudaMemsetAsync(w.sk_ws, 0, gemm_splitk_flag_bytes(), st);
    if (me != cudaSuccess) return set_last_cuda_error(me);
  }
  const ta_model_desc& d = m->d;
  const int D = d.dim, L = d.depth, N = m->n_tokens;
  const int act = d.dtype;
  const bool accumulate = d.prompt_mode == TA_PROMPT_ACCUMULATE;
  // LayerNorm folded into the QKV / fc1 GEMMs (bf16 + folded weights registered): the
  // producers of the residual emit xh = bf16(x) (in w.h) and row stats; no LN passes.
  const bool fused = m->ln_folded && act == TA_DTYPE_BF16;
  float* const ln1_stats = w.stats[0];
  float* const ln2_stats = w.stats[1];
  const int stat_slots = D / 128;  // partial row statistics per 128-column block

  // ---- patch embedding + cls + layer-0 prompts
  TA_TRY(patchify(images, w.patches, B, d.img, d.patch, m->kp, act, st));
  prof.mark(TA_STAGE_PATCHIFY, -1);
  {
    GemmEpi e;
    e.bias = static_cast<const float*>(m->w.patch_b);
    e.pos = static_cast<const float*>(m->w.pos);
    e.out = w.x[0];
    e.rows_in = m->n_patches;
    e.rows_out = s.t[0];
    e.row_off = 1;
    if (fused) {
      e.xh = w.h;
      e.stats = ln1_stats;
      e.stat_slots = stat_slots;
    }
    TA_TRY(linear(m, w.patches, m->w.patch_w, B * m->n_patches, D, m->kp,
                  fused ? EPI_PATCH_STATS : EPI_PATCH, e, st, w));
    prof.mark(TA_STAGE_PATCH_GEMM, -1);
  }
  TA_TRY(insert_rows(w.x[0], B, s.t[0], D, static_cast<const float*>(m->w.cls),
                     static_cast<const float*>(m->w.pos), ptab, task_ids, d.n_tasks, 0,
                     gamma > 0 ? gamma : 0, N, st, fused ? w.h : nullptr,
                     fused ? ln1_stats : nullptr));
      prof.mark(TA_STAGE_INSERT_ROWS, -1);

  int cur = 0;
  const float* size = nullptr;
  int size_buf = 0;
  size_t trace_off = 0;
  int t = s.t[0];
  for (int l = 0; l < L; ++l) {
    const ta_layer_weights& Lw = m->layers[l];
    t = s.t[l];
    if (l > 0 && gamma > 0)
      TA_TRY(insert_rows(w.x[cur], B, t, D, nullptr, nullptr, ptab, task_ids, d.n_tasks, l, gamma,
                         accumulate ? t - gamma : N, st, fused ? w.h : nullptr,
                         fused ? ln1_stats : nullptr));
      prof.mark(TA_STAGE_INSERT_ROWS, l);
    const int M = B * t;
    {  // LN1 + QKV
      GemmEpi e;
      e.out = w.qkv;
      if (fused) {
        e.ln_stats = ln1_stats;
        e.stat_slots = stat_slots;
        e.c1 = static_cast<const float*>(Lw.qkv_c1);
        e.c2 = static_cast<const float*>(Lw.qkv_c2);
        e.inv_dim = 1.0f / D;
        TA_TRY(linear(m, w.h, Lw.qkv_w_ln, M, 3 * D, D, EPI_LN_BIAS, e, st, w));
      prof.mark(TA_STAGE_QKV, l);
      } else {
        TA_TRY(layernorm(w.x[cur], static_cast<const float*>(Lw.ln1_w),
                         static_cast<const float*>(Lw.ln1_b), w.h, M, D, act, st));
      prof.mark(TA_STAGE_LN1, l);
        e.bias = static_cast<const float*>(Lw.qkv_b);
        TA_TRY(linear(m, w.h, Lw.qkv_w, M, 3 * D, D, EPI_BIAS, e, st, w));
      prof.mark(TA_STAGE_QKV, l);
      }
    }
    const int r = s.r[l];
    // Merge-layer indices (ToMe match on this layer's keys): the match needs only qkv, so with
    // the fused merge it runs before attention and the proj GEMM moves rows to their merged
    // positions itself (EPI_BIAS_RESID_MERGE); otherwise the classic order proj -> match -> merge.
    int32_t *src = w.src, *dst = w.dst, *unm = w.unm;
    const bool fuse_merge = r > 0 && fused && merge_fusion_enabled() && gemm_pair_path(M, D);
    // row_map (fused merge): the match kernel emits the destination map itself; a forced trace
    // gets it from merge_map.
    auto do_match = [&](int32_t* row_map) -> int {
      const int na = (t + 1) / 2;
      const int32_t* base = forced_trace ? forced_trace : merge_trace;
      if (base) {
        src = const_cast<int32_t*>(base) + trace_off;
        dst = src + static_cast<size_t>(B) * r;
        unm = dst + static_cast<size_t>(B) * r;
      }
      trace_off += static_cast<size_t>(B) * (2 * r + na - r);
      if (!forced_trace)
        return match(nullptr, w.qkv, act, B, t, d.heads, m->hd, r, src, dst, unm, w.match_scratch, st,
                     row_map);
      if (merge_trace)
        cudaMemcpyAsync(merge_trace + (src - forced_trace), src,
                        sizeof(int32_t) * static_cast<size_t>(B) * (2 * r + na - r),
                        cudaMemcpyDeviceToDevice, st);
      return row_map != nullptr ? merge_map(src, unm, B, t, r, row_map, st) : TA_OK;
    };
    if (fuse_merge) {
      TA_TRY(do_match(w.row_map));
      prof.mark(TA_STAGE_MATCH, l);
    }
    TA_TRY(attention(w.qkv, size, B, t, d.heads, m->hd, w.attn, act, st));
      prof.mark(TA_STAGE_ATTENTION, l);
    {  // proj + residual (+ LN2 stats when no merge follows; + the merge's row movement)
      GemmEpi e;
      e.bias = static_cast<const float*>(Lw.proj_b);
      e.resid = w.x[cur];
      e.out = w.x[cur];
      if (fuse_merge) {
        e.out = w.x[cur ^ 1];
        e.xh = w.h;
        e.stats = ln2_stats;
        e.stat_slots = stat_slots;
        e.row_map = w.row_map;
        e.rows_out = B * (t - r);  // merged rows; the r source rows per image follow them
        TA_TRY(linear(m, w.attn, Lw.proj_w, M, D, D, EPI_BIAS_RESID_MERGE, e, st, w));
      prof.mark(TA_STAGE_PROJ, l);
      } else if (fused && r == 0) {
        e.xh = w.h;
        e.stats = ln2_stats;
        e.stat_slots = stat_slots;
        TA_TRY(linear(m, w.attn, Lw.proj_w, M, D, D, EPI_BIAS_RESID_STATS, e, st, w));
      prof.mark(TA_STAGE_PROJ, l);
      } else {
        TA_TRY(linear(m, w.attn, Lw.proj_w, M, D, D, EPI_BIAS_RESID, e, st, w));
      prof.mark(TA_STAGE_PROJ, l);
      }
    }
    int tp = t;
    if (r > 0) {
      if (fuse_merge) {
        TA_TRY(merge_fixup(w.x[cur ^ 1], w.x[cur ^ 1] + static_cast<size_t>(B) * (t - r) * D, size,
                           w.size[size_buf], B, t, D, r, src, dst, unm, w.h,
                           ln2_stats, st));
      } else {
        TA_TRY(do_match(nullptr));
        prof.mark(TA_STAGE_MATCH, l);
        TA_TRY(merge(w.x[cur], size, B, t, D, r, src, dst, unm, static_cast<const float*>(Lw.ln2_w),
                     static_cast<const float*>(Lw.ln2_b), w.x[cur ^ 1], w.size[size_buf], w.h, act,
                     st, fused ? ln2_stats : nullptr));
      }
      prof.mark(TA_STAGE_MERGE, l);
      cur ^= 1;
      size = w.size[size_buf];
      size_buf ^= 1;
      tp = t - r;
    } else if (!fused) {
      TA_TRY(layernorm(w.x[cur], static_cast<const float*>(Lw.ln2_w),
                       static_cast<const float*>(Lw.ln2_b), w.h, M, D, act, st));
      prof.mark(TA_STAGE_LN2, l);
    }
    const int Mp = B * tp;
    {  // LN2 + fc1 + GELU
      GemmEpi e;
      e.out = w.mlp;
      if (fused) {
        e.ln_stats = ln2_stats;
        e.stat_slots = stat_slots;
        e.c1 = static_cast<const float*>(Lw.fc1_c1);
        e.c2 = static_cast<const float*>(Lw.fc1_c2);
        e.inv_dim = 1.0f / D;
        TA_TRY(linear(m, w.h, Lw.fc1_w_ln, Mp, d.mlp_dim, D, EPI_LN_GELU, e, st, w));
      prof.mark(TA_STAGE_FC1, l);
      } else {
        e.bias = static_cast<const float*>(Lw.fc1_b);
        TA_TRY(linear(m, w.h, Lw.fc1_w, Mp, d.mlp_dim, D, EPI_BIAS_GELU, e, st, w));
      prof.mark(TA_STAGE_FC1, l);
      }
    }
    {  // fc2 + residual (+ next layer's LN1 stats)
      GemmEpi e;
      e.bias = static_cast<const float*>(Lw.fc2_b);
      e.resid = w.x[cur];
      const bool restride = gamma > 0 && accumulate && l + 1 < L;
      const bool stats = fused && l + 1 < L;
      if (restride) {
        // re-stride rows so the next layer's gamma prompt rows follow each image
        e.out = w.x[cur ^ 1];
        e.rows_in = tp;
        e.rows_out = s.t[l + 1];
        e.row_off = 0;
      } else {
        e.out = w.x[cur];
      }
      if (stats) {
        e.xh = w.h;
        e.stats = ln1_stats;
        e.stat_slots = stat_slots;
      }
      TA_TRY(linear(m, w.mlp, Lw.fc2_w, Mp, D, d.mlp_dim,
                    stats ? EPI_BIAS_RESID_STATS : EPI_BIAS_RESID, e, st, w));
      prof.mark(TA_STAGE_FC2, l);
      if (restride) cur ^= 1;
    }
    t = tp;
  }
  TA_TRY(head(w.x[cur], B, t, D, static_cast<const float*>(m->w.norm_w),
              static_cast<const float*>(m->w.norm_b), m->heads_dev, task_ids, d.n_tasks, logits,
              d.max_classes, st));
  prof.mark(TA_STAGE_HEAD, -1);
  return TA_OK;
}

int ta_forward_host(ta_model* m, const float* images_host, const int32_t* task_ids_host, int B,
                    int gamma, float* logits_host, void* stream) {
  if (!m || !images_host || !task_ids_host || !logits_host || B <= 0) return TA_ERR_INVALID;
  for (int i = 0; i < B; ++i) {
    if (task_ids_host[i] < 0 || task_ids_host[i] >= m->d.n_tasks) return TA_ERR_INVALID;
    if (!m->heads[task_ids_host[i]].w) return TA_ERR_NO_WEIGHTS;
  }
  if (gamma > 0) {
    auto it = m->prompts.find(gamma);
    if (it == m->prompts.end()) return TA_ERR_NO_PROMPT;
    for (int i = 0; i < B; ++i)
      if (!it->second[task_ids_host[i]]) return TA_ERR_NO_PROMPT;
  }
  std::lock_guard<std::mutex> lock(m->host_mu);
  DeviceGuard guard(m->device);
  if (guard.err != cudaSuccess) return set_last_cuda_error(guard.err);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const size_t img_bytes = static_cast<size_t>(B) * 3 * m->d.img * m->d.img * sizeof(float);
  const size_t task_bytes = align_up(static_cast<size_t>(B) * sizeof(int32_t));
  const size_t logit_bytes = align_up(static_cast<size_t>(B) * m->d.max_classes * sizeof(float));
  size_t ws = 0;
  TA_TRY(ta_workspace_size(m, B, gamma, &ws));
  const size_t need = align_up(img_bytes) + task_bytes + logit_bytes + ws;
  if (m->host_ws_bytes < need) {
    if (m->host_ws) cudaFree(m->host_ws);
    m->host_ws = nullptr;
    m->host_ws_bytes = 0;
    cudaError_t e = cudaMalloc(&m->host_ws, need);
    if (e != cudaSuccess) return set_last_cuda_error(e);
    m->host_ws_bytes = need;
  }
  char* p = static_cast<char*>(m->host_ws);
  float* img = reinterpret_cast<float*>(p);
  int32_t* tasks = reinterpret_cast<int32_t*>(p + align_up(img_bytes));
  float* logits = reinterpret_cast<float*>(p + align_up(img_bytes) + task_bytes);
  char* wsp = p + align_up(img_bytes) + task_bytes + logit_bytes;
  cudaError_t e = cudaMemcpyAsync(img, images_host, img_bytes, cudaMemcpyHostToDevice, st);
  if (e != cudaSuccess) return set_last_cuda_error(e);
  e = cudaMemcpyAsync(tasks, task_ids_host, B * sizeof(int32_t), cudaMemcpyHostToDevice, st);
  if (e != cudaSuccess) return set_last_cuda_error(e);
  TA_TRY(ta_forward(m, img, tasks, B, gamma, logits, nullptr, nullptr, wsp, ws, stream));
  e = cudaMemcpyAsync(logits_host, logits, static_cast<size_t>(B) * m->d.max_classes * sizeof(float),
                      cudaMemcpyDeviceToHost, st);
  if (e != cudaSuccess) return set_last_cuda_error(e);
  e = cudaStreamSynchronize(st);
  return e == cudaSuccess ? TA_OK : set_last_cuda_error(e);
}

// ------------------------------------------------------------------ unit entry points
int ta_match(const float* metric, int batch, int t, int c, int r, int32_t* src, int32_t* dst,
             int32_t* unm, void* stream) {
  if (!metric || !src || !dst || !unm || batch <= 0) return TA_ERR_INVALID;
  // Unit entry point (parity tests): scratch for the tcgen05 path is stream-ordered.
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  void* scratch = nullptr;
  cudaError_t e = cudaMallocAsync(&scratch, match_tc_scratch_bytes(batch, c), st);
  if (e != cudaSuccess) return set_last_cuda_error(e);
  const int rc = match(metric, nullptr, TA_DTYPE_F32, batch, t, 1, c, r, src, dst, unm,
                       static_cast<float*>(scratch), st);
  cudaFreeAsync(scratch, st);
  return rc;
}

int ta_match_qkv(const void* qkv, int dtype, int batch, int t, int heads, int head_dim, int r,
                 int32_t* src, int32_t* dst, int32_t* unm, void* stream) {
  if (!qkv || !src || !dst || !unm || batch <= 0 || heads <= 0) return TA_ERR_INVALID;
  if (dtype != TA_DTYPE_BF16 && dtype != TA_DTYPE_F32) return TA_ERR_INVALID;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  void* scratch = nullptr;
  cudaError_t e = cudaMallocAsync(&scratch, match_tc_scratch_bytes(batch, head_dim), st);
  if (e != cudaSuccess) return set_last_cuda_error(e);
  const int rc = match(nullptr, qkv, dtype, batch, t, heads, head_dim, r, src, dst, unm,
                       static_cast<float*>(scratch), st);
  cudaFreeAsync(scratch, st);
  return rc;
}

int ta_merge(const float* x, const float* size, int batch, int t, int dim, int r,
             const int32_t* src, const int32_t* dst, const int32_t* unm, const float* ln_w,
             const float* ln_b, float* x_out, float* size_out, void* h_out, int h_dtype,
             void* stream) {
  if (!x || !src || !dst || !unm || !ln_w || !ln_b || !x_out || !size_out || !h_out || batch <= 0)
    return TA_ERR_INVALID;
  return merge(x, size, batch, t, dim, r, src, dst, unm, ln_w, ln_b, x_out, size_out, h_out,
               h_dtype, static_cast<cudaStream_t>(stream));
}

int ta_attention(const void* qkv, const float* size, int batch, int t, int heads, int head_dim,
                 void* out, int dtype, void* stream) {
  if (!qkv || !out || batch <= 0 || heads <= 0) return TA_ERR_INVALID;
  return attention(qkv, size, batch, t, heads, head_dim, out, dtype,
                   static_cast<cudaStream_t>(stream));
}

int ta_gemm(const void* a, const void* w, const float* bias, const float* resid, void* out, int m,
            int n, int k, int epilogue, int dtype, int out_dtype, void* stream) {
  if (!a || !w || !bias || !out || epilogue < 0 || epilogue > 2) return TA_ERR_INVALID;
  if (epilogue == EPI_BIAS_RESID && (!resid || out_dtype != TA_DTYPE_F32)) return TA_ERR_INVALID;
  GemmEpi e;
  e.bias = bias;
  e.resid = resid;
  e.out = out;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (dtype == TA_DTYPE_BF16) {
    // unit entry point: stream-ordered split-K scratch with zeroed counters
    void* sk = nullptr;
    cudaError_t ce = cudaMallocAsync(&sk, gemm_splitk_ws_bytes(), st);
    if (ce != cudaSuccess) return set_last_cuda_error(ce);
    ce = cudaMemsetAsync(sk, 0, gemm_splitk_flag_bytes(), st);
    if (ce != cudaSuccess) return set_last_cuda_error(ce);
    const int rc = gemm_bf16(a, w, m, n, k, epilogue, out_dtype == TA_DTYPE_BF16, e, st, static_cast<float*>(sk));
    cudaFreeAsync(sk, st);
    return rc;
  }
  if (out_dtype != TA_DTYPE_F32) return TA_ERR_INVALID;
  if (f32_gemm_backend() == 0 && k % 32 == 0 && n % 128 == 0) {
    // unit entry point: stream-ordered scratch for the tf32 operand split
    void* scratch = nullptr;
    cudaError_t ce = cudaMallocAsync(&scratch, gemm_f32_tc_scratch_bytes(m, n, k), st);
    if (ce != cudaSuccess) return set_last_cuda_error(ce);
    const int rc = gemm_f32_tc(static_cast<const float*>(a), static_cast<const float*>(w), m, n, k, epilogue,
                               e, scratch, st);
    cudaFreeAsync(scratch, st);
    return rc;
  }
  return gemm_f32(static_cast<const float*>(a), static_cast<const float*>(w), m, n, k, epilogue, e, st);
}

int ta_layernorm(const float* x, const float* w, const float* b, void* out, int rows, int dim,
                 int out_dtype, void* stream) {
  if (!x || !w || !b || !out) return TA_ERR_INVALID;
  return layernorm(x, w, b, out, rows, dim, out_dtype, static_cast<cudaStream_t>(stream));
}

}  // extern "C"
