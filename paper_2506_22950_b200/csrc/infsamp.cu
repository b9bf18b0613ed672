// libinfsamp: C-ABI of the B200 continuous-sampling decode step (include/infsamp.h).
//
// Host side: the Alg. 2 planner, the Alg. 1 initial fill
// and Alg. 3 static SJF refill order (l.218-241, l.280-295), the KV budget
// check (R25), weight packing, the paged KV pool, and the
// decode step orchestration, captured once into a CUDA graph with
// programmatic dependent launch between kernels.
#include <dlfcn.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/infsamp.h"
#include "common.cuh"
#include "gemm.cuh"
#include "kernels.cuh"

using namespace isk;

// ------------------------------------------------------------------ errors
static thread_local std::string g_err;
static is_status fail(is_status s, const char* fmt, ...) {
  static const char* names[] = {"IS_OK", "IS_ERR_CONFIG", "IS_ERR_BUDGET", "IS_ERR_CAPACITY",
                                "IS_ERR_DATA", "IS_ERR_STATE", "IS_ERR_CUDA"};
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = std::string(names[s]) + ": " + buf;
  return s;
}
#define CK(x)                                                                                     \
  do {                                                                                            \
    cudaError_t e_ = (x);                                                                         \
    if (e_ != cudaSuccess) return fail(IS_ERR_CUDA, "%s at %s:%d (%s)", cudaGetErrorString(e_), \
                                       __FILE__, __LINE__, #x);                                   \
  } while (0)
#define CKS(x)                     \
  do {                             \
    is_status s_ = (x);            \
    if (s_ != IS_OK) return s_;    \
  } while (0)

extern "C" const char* is_last_error(void) { return g_err.c_str(); }
extern "C" const char* is_version(void) { return "infsamp 0.1 sm_100a"; }

// ------------------------------------------------------------------ planner (host, pure)
static int64_t ceil_div64(int64_t a, int64_t b) { return (a + b - 1) / b; }

static int64_t kv_bytes_per_token(const is_shape& s) {
  return 2ll * s.layers * s.n_kv_heads * s.head_dim * 2;
}

static int n_groups(const is_config* c) { return c->max_groups > 0 ? c->max_groups : 1; }

static is_status check_config(const is_config* c) {
  const is_shape& s = c->shape;
  if (s.head_dim != 128) return fail(IS_ERR_CONFIG, "head_dim must be 128 (got %d)", s.head_dim);
  if (s.layers < 1 || s.hidden < 64 || s.hidden % 64 || s.ffn % 64 || s.vocab % 128 ||
      s.n_q_heads < 1 || s.n_kv_heads < 1 || s.n_q_heads % s.n_kv_heads || s.n_q_heads / s.n_kv_heads > 8)
    return fail(IS_ERR_CONFIG, "unsupported shape (hidden %% 64, ffn %% 64, vocab %% 128, Hq %% Hkv)");
  if (c->G < 1) return fail(IS_ERR_CONFIG, "G must be >= 1");
  const int g = c->mode == IS_MODE_FULL ? c->G : c->g;
  if (g < 1 || g > c->G || c->G % g) return fail(IS_ERR_CONFIG, "need 1 <= g <= G and G mod g == 0 (G=%d g=%d)", c->G, g);
  if (!(c->eps > 0)) return fail(IS_ERR_CONFIG, "eps must be > 0");
  if (c->max_new_tokens < 1 || c->prompt_len < 2) return fail(IS_ERR_CONFIG, "max_new_tokens >= 1 and prompt_len >= 2");
  if (c->page_tokens < 4 || 64 % c->page_tokens) return fail(IS_ERR_CONFIG, "page_tokens must divide 64 and be >= 4");
  if (c->prefix_k < 0 || (c->prefix_k > 0 && c->mode != IS_MODE_INFINITE))
    return fail(IS_ERR_CONFIG, "prefix_k > 0 requires IS_MODE_INFINITE");
  if (!(c->temperature > 0)) return fail(IS_ERR_CONFIG, "temperature must be > 0");
  if (!(c->top_p >= 0.f && c->top_p <= 1.f)) return fail(IS_ERR_CONFIG, "top_p must be in [0, 1] (0 or 1 = off)");
  if (c->mode < IS_MODE_FULL || c->mode > IS_MODE_DYNAMIC) return fail(IS_ERR_CONFIG, "unknown mode %d", (int)c->mode);
  if (c->eos_enabled && (c->eos_id < 0 || c->eos_id >= s.vocab || c->prefix_k > 0))
    return fail(IS_ERR_CONFIG, "eos_id must be a token id (0..vocab-1) and needs prefix_k == 0 (R37)");
  if (c->dynamic_target < 0 || c->dynamic_target > c->G || (c->dynamic_target > 0 && c->mode != IS_MODE_DYNAMIC))
    return fail(IS_ERR_CONFIG, "dynamic_target must be 0 or 1..G (got %d) and needs IS_MODE_DYNAMIC", c->dynamic_target);
  if (c->decode_impl != 0 && c->decode_impl != 1) return fail(IS_ERR_CONFIG, "decode_impl must be 0 or 1 (reserved)");
  if (c->bin_slots != 0 && (c->bin_slots != 1 || c->mode != IS_MODE_INFINITE))
    return fail(IS_ERR_CONFIG, "bin_slots must be 0 or 1 and needs IS_MODE_INFINITE");
  if (c->admit_slots != 0 &&
      (c->admit_slots <= g || c->admit_slots > 64 || c->mode != IS_MODE_INFINITE || c->prefix_k != 0 ||
       n_groups(c) != 1 || c->bin_slots != 0 || c->kv_budget_bytes <= 0 || c->eos_enabled))
    return fail(IS_ERR_CONFIG, "admit_slots needs g < S <= 64, IS_MODE_INFINITE, a KV budget, prefix_k == 0, "
                               "max_groups <= 1, bin_slots == 0 and no EOS (R41)");
  if (c->max_groups < 0 || n_groups(c) > 8 || n_groups(c) * g > 64)
    return fail(IS_ERR_CONFIG, "need 1 <= max_groups <= 8 and max_groups * g <= 64 (got %d x %d)", n_groups(c), g);
  return IS_OK;
}

static int eff_g(const is_config* c) { return c->mode == IS_MODE_FULL ? c->G : c->g; }
// rows per group slot: the micro-group size, or S with memory-aware admission (R41)
static int slots_of(const is_config* c) { return c->admit_slots > 0 ? c->admit_slots : eff_g(c); }
static int row_cap_of(const is_config* c) {
  int rc = c->row_capacity > 0 ? c->row_capacity : ((n_groups(c) * slots_of(c) + 15) / 16) * 16;
  return rc;
}

static int64_t reservation_bytes(const is_config* c) {
  const int g = eff_g(c);
  const int64_t pb = (int64_t)c->page_tokens * kv_bytes_per_token(c->shape);
  const int64_t pre = (int64_t)(c->prompt_len - 1) * kv_bytes_per_token(c->shape);
  const int64_t full = ceil_div64(c->max_new_tokens, c->page_tokens);
  const int64_t park = c->prefix_k > 0 ? ceil_div64(c->prefix_k, c->page_tokens) : 0;
  return pre + (int64_t)g * full * pb + (int64_t)(c->G - g) * park * pb;
}

extern "C" is_status is_plan(const is_config* cfg, const int32_t* pred, const uint8_t* finished,
                             is_plan_out* out) {
  if (!cfg || !out) return fail(IS_ERR_CONFIG, "null argument");
  CKS(check_config(cfg));
  const int G = cfg->G, g = eff_g(cfg);
  // Alg. 2's bins: N = G/g micro groups (the paper's Alg. 2), or g slot bins (bin_slots, R38)
  const bool slots = cfg->bin_slots != 0;
  const int N = slots ? g : G / g;
  out->K = 0;
  out->capacity = 0;
  out->n_overflow = 0;
  out->reserved_bytes = reservation_bytes(cfg);
  if (cfg->kv_budget_bytes > 0 && out->reserved_bytes > cfg->kv_budget_bytes)
    return fail(IS_ERR_BUDGET, "worst-case KV reservation %lld B exceeds budget %lld B",
                (long long)out->reserved_bytes, (long long)cfg->kv_budget_bytes);
  const bool planned = cfg->mode == IS_MODE_INFINITE || cfg->mode == IS_MODE_FPTAS_ONLY;
  if (cfg->mode == IS_MODE_SJF_ONLY) {
    // trace-order start, Alg. 3 SJF refill of the rest (DESIGN R23)
    if (!pred) return fail(IS_ERR_DATA, "IS_MODE_SJF_ONLY needs predicted lengths");
    for (int i = 0; i < G; ++i)
      if (pred[i] < 1) return fail(IS_ERR_DATA, "predicted length of sample %d is %d (< 1)", i, pred[i]);
    if (out->mask) std::fill(out->mask, out->mask + 2 * G, 0);
    if (out->scaled_len) std::fill(out->scaled_len, out->scaled_len + G, 0);
    if (out->loads) std::fill(out->loads, out->loads + N, 0);
    for (int i = 0; i < g; ++i) out->init_slots[i] = i;
    std::vector<int> rest;
    for (int i = g; i < G; ++i) rest.push_back(i);
    std::stable_sort(rest.begin(), rest.end(), [&](int a, int b) { return pred[a] < pred[b]; });
    out->queue_len = G - g;
    for (int i = 0; i < G - g; ++i) out->refill_queue[i] = rest[i];
    return IS_OK;
  }
  if (!planned) {
    if (out->mask) std::fill(out->mask, out->mask + 2 * G, 0);
    if (out->scaled_len) std::fill(out->scaled_len, out->scaled_len + G, 0);
    if (out->loads) std::fill(out->loads, out->loads + N, 0);
    for (int i = 0; i < g; ++i) out->init_slots[i] = i;
    out->queue_len = G - g;
    for (int i = g; i < G; ++i) out->refill_queue[i - g] = i;
    return IS_OK;
  }
  if (!pred) return fail(IS_ERR_DATA, "the FPTAS plan needs predicted lengths");
  int64_t S = 0;
  for (int i = 0; i < G; ++i) {
    if (pred[i] < 1) return fail(IS_ERR_DATA, "predicted length of sample %d is %d (< 1)", i, pred[i]);
    S += pred[i];
  }
  // Alg. 2: K = eps*S/N (IEEE double, this evaluation order, R14)
  const double K = (cfg->eps * (double)S) / (double)N;
  std::vector<int64_t> lt(G);
  int64_t sum_lt = 0;
  for (int i = 0; i < G; ++i) {
    lt[i] = (int64_t)std::ceil((double)pred[i] / K);
    sum_lt += lt[i];
  }
  const int64_t Ct = ceil_div64(sum_lt, N);
  std::vector<int> order(G);
  for (int i = 0; i < G; ++i) order[i] = i;
  std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return lt[a] > lt[b]; });  // ties -> lower id
  std::vector<int64_t> load(N, 0);
  std::vector<int> gsize(N, 0);
  std::vector<int> gn(G), gj(G);
  int nov = 0;
  for (int i : order) {  // first fit
    int target = -1;
    for (int n = 0; n < N; ++n)
      if (load[n] + lt[i] <= Ct) {
        target = n;
        break;
      }
    if (target < 0) {  // R15: least-loaded fallback, ties -> lowest index
      target = 0;
      for (int n = 1; n < N; ++n)
        if (load[n] < load[target]) target = n;
      if (out->overflow_ids) out->overflow_ids[nov] = i;
      ++nov;
    }
    gn[i] = target;
    gj[i] = gsize[target]++;
    load[target] += lt[i];
  }
  out->K = K;
  out->capacity = Ct;
  out->n_overflow = nov;
  for (int i = 0; i < G; ++i) {
    if (out->mask) {
      out->mask[2 * i] = gn[i] + 1;
      out->mask[2 * i + 1] = gj[i];
    }
    if (out->scaled_len) out->scaled_len[i] = lt[i];
  }
  if (out->loads)
    for (int n = 0; n < N; ++n) out->loads[n] = load[n];
  if (slots) {
    // SPEC.md l.175 / l.255 (bin_mode = slots, R38): slot j starts with bin j's head (its first
    // member in placement order not finished in the prefix phase); an empty bin's slot takes the
    // SJF queue head in ascending slot order; the rest is the Alg. 3 static queue.
    std::vector<int> head(g, -1);
    for (int i : order) {
      if (finished && finished[i]) continue;
      if (head[gn[i]] < 0) head[gn[i]] = i;
    }
    std::vector<char> used(G, 0);
    for (int j = 0; j < g; ++j)
      if (head[j] >= 0) used[head[j]] = 1;
    std::vector<int> rest;
    for (int i = 0; i < G; ++i)
      if (!used[i] && !(finished && finished[i])) rest.push_back(i);
    std::stable_sort(rest.begin(), rest.end(), [&](int a, int b) { return pred[a] < pred[b]; });
    size_t qh = 0;
    for (int j = 0; j < g; ++j) out->init_slots[j] = head[j] >= 0 ? head[j] : (qh < rest.size() ? rest[qh++] : -1);
    out->queue_len = (int32_t)(rest.size() - qh);
    for (size_t i = qh; i < rest.size(); ++i) out->refill_queue[i - qh] = rest[i];
    return IS_OK;
  }
  // Alg. 1 l.230: first g samples from mask in lexicographic (n, j) order,
  // skipping samples finished in the prefix phase (R13, R22).
  std::vector<int> lex(G);
  for (int i = 0; i < G; ++i) lex[i] = i;
  std::sort(lex.begin(), lex.end(), [&](int a, int b) { return gn[a] != gn[b] ? gn[a] < gn[b] : gj[a] < gj[b]; });
  std::vector<char> used(G, 0);
  int ni = 0;
  for (int i : lex) {
    if (finished && finished[i]) continue;
    if (ni < g) {
      out->init_slots[ni++] = i;
      used[i] = 1;
    }
  }
  for (int s = ni; s < g; ++s) out->init_slots[s] = -1;
  if (cfg->mode == IS_MODE_FPTAS_ONLY) {  // the plan's own order, FIFO refill (DESIGN R23)
    out->queue_len = 0;
    for (int i : lex)
      if (!used[i] && !(finished && finished[i])) out->refill_queue[out->queue_len++] = i;
    return IS_OK;
  }
  // Alg. 3 repeated: argmin pred over unstarted, unfinished, ties -> lower id (R17)
  std::vector<int> rest;
  for (int i = 0; i < G; ++i)
    if (!used[i] && !(finished && finished[i])) rest.push_back(i);
  std::stable_sort(rest.begin(), rest.end(), [&](int a, int b) { return pred[a] < pred[b]; });
  out->queue_len = (int32_t)rest.size();
  for (size_t i = 0; i < rest.size(); ++i) out->refill_queue[i] = rest[i];
  return IS_OK;
}

extern "C" is_status is_group_advantages(const float* r, int32_t G, is_adv_mode mode, float* adv) {
  if (!r || !adv || G < 1) return fail(IS_ERR_CONFIG, "bad arguments");
  double s = 0;
  for (int i = 0; i < G; ++i) s += (double)r[i];
  const double mean = s / G;
  if (mode == IS_ADV_MEAN_ONLY) {
    for (int i = 0; i < G; ++i) adv[i] = (float)((double)r[i] - mean);
    return IS_OK;
  }
  if (mode != IS_ADV_STD_NORM) return fail(IS_ERR_CONFIG, "unknown advantage mode");
  double v = 0;
  for (int i = 0; i < G; ++i) v += ((double)r[i] - mean) * ((double)r[i] - mean);
  const double sigma = std::sqrt(v / G);
  for (int i = 0; i < G; ++i) adv[i] = sigma == 0.0 ? 0.f : (float)(((double)r[i] - mean) / sigma);
  return IS_OK;
}

// ------------------------------------------------------------------ TMA descriptors
typedef CUresult (*PFN_encodeTiled_t)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                      const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                      CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static PFN_encodeTiled_t get_encode() {
  static PFN_encodeTiled_t fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_encodeTiled_t>(p);
  }
  return fn;
}
// bf16 row-major [rows][cols]; box = [box_rows][64] with 128-byte swizzle.
static is_status make_tmap(CUtensorMap* m, const void* ptr, int64_t rows, int64_t cols, int box_rows) {
  PFN_encodeTiled_t enc = get_encode();
  if (!enc) return fail(IS_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)cols * 2};
  cuuint32_t box[2] = {64, (cuuint32_t)box_rows};
  cuuint32_t es[2] = {1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(IS_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
  return IS_OK;
}

// The page pool ([pages][2 = K|V][Hkv][pt][128] bf16, all layers) as a 5-D tensor whose box is one
// page of one kv head: (64 dims, 2 halves, pt rows, K|V, page x head), 128-byte swizzle
// (attn_suffix_mma_kernel).  Coordinate 4 = (layer * num_pages + page) * 2 * Hkv + head.
static is_status make_tmap_pool(CUtensorMap* m, const void* ptr, int64_t layer_pages, int Hkv, int pt) {
  PFN_encodeTiled_t enc = get_encode();
  if (!enc) return fail(IS_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[5] = {64, 2, (cuuint64_t)pt, 2, (cuuint64_t)(layer_pages * 2 * Hkv)};
  cuuint64_t strides[4] = {128, 256, (cuuint64_t)Hkv * pt * 256, (cuuint64_t)pt * 256};
  cuuint32_t box[5] = {64, 2, (cuuint32_t)pt, 2, 1};
  cuuint32_t es[5] = {1, 1, 1, 1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 5, const_cast<void*>(ptr), dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(IS_ERR_CUDA, "cuTensorMapEncodeTiled (page pool) failed (%d)", (int)r);
  return IS_OK;
}

// ------------------------------------------------------------------ GEMM launch
static int g_num_sms = 0;
static int g_launches = 0;  // kernel launches issued since the last reset (enqueue_step counts its own)
static bool g_use_pdl = true;
static int g_skip = 0;
static float* g_splitk_ws = nullptr;  // set per context before enqueueing
static bool g_exact_prefix_max = false;  // IS_EXACT_PREFIX_MAX: the prefix softmax takes the column max (no bound)

static unsigned long long* g_tl = nullptr;  // current timeline buffer during enqueue
static int g_tl_n = 0;
static const char* g_tl_name[512];  // debug: bit k skips kernel class k in the decode step (timing experiments only)

// Ring depth: split-K GEMMs stream few k-blocks per CTA (4 stages keep two CTAs
// per SM so the next kernel can co-reside); persistent (split 1) GEMMs stream
// long K ranges from fewer CTAs and need more bytes in flight per SM.
template <int BN, bool DEEP>
struct Stages {
  static constexpr int v = !DEEP ? 4 : (BN == 16 ? 8 : (BN == 32 ? 6 : 4));
};

template <int BN, bool DEEP>
static int gemm_smem_of() { return GemmCfg<BN, Stages<BN, DEEP>::v>::kSmem; }

template <int BN, int EPI, int STAGES>
static is_status launch_gemm_s(const CUtensorMap& tA, const CUtensorMap& tB, GemmArgs a, cudaStream_t st) {
  using C = GemmCfg<BN, STAGES>;
  static int attr = 0;
  auto kern = gemm_swapab_kernel<BN, EPI, STAGES>;
  const int smem = C::kSmem;
  if (smem > attr) {
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    attr = smem;
  }
  cudaLaunchConfig_t cfg{};
  cudaLaunchAttribute at[2];
  int na = 0;
  cfg.blockDim = dim3(kGemmThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  if (a.split > 1) {
    cfg.gridDim = dim3(a.num_tiles * a.split);
    at[na].id = cudaLaunchAttributeClusterDimension;
    at[na].val.clusterDim.x = a.split;
    at[na].val.clusterDim.y = 1;
    at[na].val.clusterDim.z = 1;
    ++na;
  } else {
    cfg.gridDim = dim3(std::min(a.num_tiles, g_num_sms));
  }
  if (g_use_pdl) {
    at[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[na].val.programmaticStreamSerializationAllowed = 1;
    ++na;
  }
  cfg.attrs = at;
  cfg.numAttrs = na;
  if (!a.partials) a.partials = g_splitk_ws;
  if (a.split > 1 && (a.num_tiles * a.split > 2 * 160 || !a.partials))
    return fail(IS_ERR_CAPACITY, "split-K workspace too small");
  if (g_tl && g_tl_n < 512 && !a.dbg_ts) {
    a.dbg_ts = g_tl + (size_t)g_tl_n * 296 * 16;
    g_tl_name[g_tl_n++] = EPI == EPI_QKV ? "qkv" : EPI == EPI_RESID_ADD ? "resid" : EPI == EPI_SWIGLU ? "gu" : EPI == EPI_SAMPLE ? "lm" : "f32";
  }
  CK(cudaLaunchKernelEx(&cfg, kern, tA, tB, a));
  ++g_launches;
  return IS_OK;
}

template <int BN, int EPI, bool DEEP>
static is_status launch_gemm_t(const CUtensorMap& tA, const CUtensorMap& tB, GemmArgs a, cudaStream_t st) {
  return launch_gemm_s<BN, EPI, Stages<BN, DEEP>::v>(tA, tB, a, st);
}

template <int EPI>
static is_status launch_gemm(int BN, const CUtensorMap& tA, const CUtensorMap& tB, GemmArgs a, cudaStream_t st,
                             int stages = 0) {
  const bool deep = a.split == 1;
  // deeper weight ring for a split-K GEMM (more of its weights arrive before the PDL wait returns)
  if (!deep && BN == 16 && stages == 3) return launch_gemm_s<16, EPI, 3>(tA, tB, a, st);
  if (!deep && BN == 16 && stages == 5) return launch_gemm_s<16, EPI, 5>(tA, tB, a, st);
  if (!deep && BN == 16 && stages == 6) return launch_gemm_s<16, EPI, 6>(tA, tB, a, st);
  if (!deep && BN == 16 && stages == 8) return launch_gemm_s<16, EPI, 8>(tA, tB, a, st);
  // lm_head (persistent, one CTA per SM): more bytes in flight per SM (IS_STG_LM)
  if (EPI == EPI_SAMPLE && deep && BN == 16 && stages == 10) return launch_gemm_s<16, EPI, 10>(tA, tB, a, st);
  if (EPI == EPI_SAMPLE && deep && BN == 16 && stages == 11) return launch_gemm_s<16, EPI, 11>(tA, tB, a, st);
  switch (BN * 2 + (deep ? 1 : 0)) {
    case 32: return launch_gemm_t<16, EPI, false>(tA, tB, a, st);
    case 33: return launch_gemm_t<16, EPI, true>(tA, tB, a, st);
    case 64: return launch_gemm_t<32, EPI, false>(tA, tB, a, st);
    case 65: return launch_gemm_t<32, EPI, true>(tA, tB, a, st);
    case 128: return launch_gemm_t<64, EPI, false>(tA, tB, a, st);
    case 129: return launch_gemm_t<64, EPI, true>(tA, tB, a, st);
  }
  return fail(IS_ERR_CONFIG, "unsupported GEMM N tile %d", BN);
}

// Split-K so that tiles * split fills at most one CTA per SM: a GEMM never
// takes more than half an SM, so the next kernel's CTAs (PDL) co-reside and
// prefetch their weights while this one drains.  BN is the decode row tile; the
// prefill's 64-row chunks use the 16-row policy (the one measured for them).
static int choose_split(int num_tiles, int kb_total, int BN) {
  if (num_tiles > g_num_sms) return 1;
  int s = std::max(1, g_num_sms / num_tiles);
  // 75..148 tiles: a 2-CTA cluster per tile keeps every SM streaming (gate/up: -5%/step at 16 rows);
  // with 32 or 64 rows the cluster exchange costs more than it saves (+8% tokens/s with split 1)
  if (s == 1) s = BN <= 16 ? 2 : 1;
  s = std::min(s, BN <= 16 ? 8 : 4);  // >= 32 rows: o_proj / down at split 4 measured +8.5% tokens/s
  s = std::min(s, kb_total);
  return std::max(s, 1);
}

template <typename K, typename... Args>
static is_status launch_k_smem(K kern, dim3 grid, dim3 block, int smem, cudaStream_t st, Args... args) {
  // (one attribute per kernel: kernels of the same signature share this instantiation)
  static std::vector<std::pair<const void*, int>> attr;
  bool found = false;
  for (auto& pr : attr)
    if (pr.first == (const void*)kern) {
      found = pr.second >= smem;
      if (!found) pr.second = smem;
    }
  if (!found) {
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));

    attr.push_back({(const void*)kern, smem});
  }
  cudaLaunchConfig_t cfg{};
  cudaLaunchAttribute at[1];
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cfg.numAttrs = 0;
  if (g_use_pdl) {
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
  }
  CK(cudaLaunchKernelEx(&cfg, kern, args...));
  ++g_launches;
  return IS_OK;
}

template <typename K, typename... Args>
static is_status launch_k(K kern, dim3 grid, dim3 block, cudaStream_t st, Args... args) {
  cudaLaunchConfig_t cfg{};
  cudaLaunchAttribute at[1];
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.stream = st;
  cfg.numAttrs = 0;
  if (g_use_pdl) {
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
  }
  CK(cudaLaunchKernelEx(&cfg, kern, args...));
  ++g_launches;
  return IS_OK;
}

// ------------------------------------------------------------------ context
struct LayerW {
  __nv_bfloat16 *wqkv, *wo, *wgu, *wd;
  float *in_norm, *post_norm, *q_norm, *k_norm;
  CUtensorMap tm_qkv, tm_o, tm_gu, tm_d;
};

struct is_ctx {
  is_config cfg;
  is_shape sh;
  int G, g, gp, N, rc, BN, P, pcap, pt, maxp, max_new, num_pages, log_cap, max_rows, max_pos;
  int32_t *pred, *adm_seq, *stall;  // memory-aware admission (R41): [M][G], [M][G], [M][g]
  int qkv_w;  // (Hq + 2 Hkv) * 128
  int64_t page_bytes, prefix_bytes;
  cudaStream_t st, user;
  cudaEvent_t ev_in, ev_out;
  // weights
  __nv_bfloat16* embed;
  float* final_norm;
  std::vector<LayerW> L;
  CUtensorMap tm_embed;
  void* wblob;
  // KV
  __nv_bfloat16* prefix;  // [L][2][Hkv][pcap][128]
  __nv_bfloat16* pool;    // [L][pages][2][Hkv][pt][128]
  // activations [max_rows]
  float* resid;
  __nv_bfloat16 *xn, *attn, *act, *q;
  float *part_o, *part_ml;
  int* merge_cnt;  // [max_rows][Hkv] fused-merge counters (decode, tcgen05 prefix), then 2 unit counters
  bool static_units;  // IS_STATIC_UNITS: the suffix pass strides its units statically (round 1)
  float* kmax;         // [M][L][Hkv][prefix tiles] max key norm per 128-token prefix tile (prefix_kmax_kernel)
  float *ssqA, *ssqB;  // [Th][max_rows] per-128-column sums of squares: QKV input, gate/up input
  int sep_merge;       // decode suffix: 64-token CTA units + separate merge kernel
  int suffix_mma;      // decode suffix: 32-token units on mma.sync, merges spread over the grid (default)
  int suffix_shape;    //   its CTA shape: 1 = 8 warps x 1 stage (default), 0 = 6 warps x 2 stages
  int attn_carveout;   //   shared-memory carveout (%) of the attention kernels, -1 = driver default
  int prefix2;         // tcgen05 prefix with the query rows as M (default; up to 256 stacked rows)
  CUtensorMap tm_pool; // the page pool of all layers as rows of 128 bf16, box = one page (128-byte swizzle)
  int stg_lm;          // lm_head ring depth override (IS_STG_LM = 10 / 11; default 8)
  int topp;            // 0 < top_p < 1: nucleus sampling pass after the lm_head (R36)
  float* logits_tp;    //   its fp32 logits [max_rows][vocab]
  float* scores_tp;    //   the lm_head's Gumbel scores [max_rows][vocab]
  uint32_t* ebits_tp;  //   e_v bits [max_rows][vocab]
  unsigned long long *wpart_tp, *hist_tp;  // per-slice mass, level-1 histograms
  int2* sel_tp;        //   per row (e*, v_k)
  ToppState* state_tp; //   per row radix-select state
  int32_t* attn_items;
  float* splitk_ws;  // split-K partials workspace
  int NC, nc_pre, nc_suf;
  CUtensorMap tm_xn_dec, tm_attn_dec, tm_act_dec, tm_xn_pre, tm_attn_pre, tm_act_pre;
  float *rope_cos, *rope_sin;
  // rows
  int32_t *row_active, *row_uid, *row_lid, *row_t, *row_tok, *row_pos, *row_kvloc, *row_len;
  unsigned long long* keys;
  unsigned long long* lp_key;  // NEXT-3: lm_head per-(row, CTA) partials for log-probabilities
  float4* lp_mlz;
  float* logprobs;             // [M][G][max_new]
  int lp_grid;
  int32_t* last_tok;
  uint8_t* last_fin;
  // scheduler
  long long* st_dev;
  long long* st_host;  // pinned mirror
  int32_t *slot_uid, *slot_count, *tpos, *true_len, *queue, *main_init, *main_queue, *free_stack, *pagetab,
      *npages, *tokens, *log_slot, *log_live;
  uint8_t* done_flag;  // [M][G] sample completed
  float* logits_dump;
  int prompt_id, prompt_last;
  bool prefilled, started;
  int M;                                    // co-resident group slots (NEXT-1)
  std::vector<int> gprompt_id, gprompt_last;  // per group slot
  std::vector<char> gprefilled, gstarted;
  int32_t *prow_active, *prow_tok, *prow_pos, *prow_kvloc, *prow_len;  // prefill row tables
  cudaGraphExec_t graph;
  bool graph_ok;
  int32_t* d_prompt_copy;
  // splits
  int split_qkv, split_o, split_gu, split_d;
  int stg_qkv, stg_o, stg_gu, stg_d;  // weight-ring depth of the split-K decode GEMMs (0 = default 4)
  int l2_prefetch;
  int tc_prefix;       // decode prefix attention on tcgen05 (N = rc * Hq/Hkv in {16, 32, 64})
  int sc;              // decode suffix chunk (tokens per attention work item)
  int nc_pre_dec;      // prefix partial slots in decode
  CUtensorMap tm_prefix_kv;
  unsigned long long* timeline;  // debug: [launch][148 CTAs][16] GEMM stamps (IS_TIMELINE)
  int tl_count;
  int launches_per_step;  // kernels in one decode step (counted while capturing it)
  cudaGraphExec_t graphK;  // steps_per_graph decode steps in one graph (run loops)
  bool graphK_ok;
  int steps_per_graph;
  int launches_per_prefill;
  // L2 weight prefetcher (IS_L2PF = lookahead MB; 0 = off): a parallel branch of the step graph
  long long pf_lookahead;
  unsigned long long* pf_ptr;
  long long* pf_off;
  int pf_n;
  int* pf_progress;
  cudaStream_t pf_st;
  cudaEvent_t pf_fork, pf_join;
};

static void* dalloc(size_t bytes, is_status* s) {
  void* p = nullptr;
  if (cudaMalloc(&p, bytes) != cudaSuccess) {
    *s = fail(IS_ERR_CUDA, "cudaMalloc(%zu) failed", bytes);
    return nullptr;
  }
  cudaMemset(p, 0, bytes);
  return p;
}

static SchedArgs sched_args(is_ctx* c) {
  SchedArgs a;
  a.G = c->G;
  a.g = c->g;
  a.row_cap = c->rc;
  a.max_new = c->max_new;
  a.pt = c->pt;
  a.maxp = c->maxp;
  a.P = c->P;
  a.log_cap = c->log_cap;
  a.M = c->M;
  a.st = c->st_dev;
  a.slot_uid = c->slot_uid;
  a.slot_count = c->slot_count;
  a.t = c->tpos;
  a.true_len = c->true_len;
  a.queue = c->queue;
  a.main_init = c->main_init;
  a.main_queue = c->main_queue;
  a.free_stack = c->free_stack;
  a.pagetab = c->pagetab;
  a.npages = c->npages;
  a.tokens = c->tokens;
  a.log_slot = c->log_slot;
  a.log_live = c->log_live;
  a.done_flag = c->done_flag;
  a.keys = c->keys;
  a.lp_key = c->lp_key;
  a.lp_mlz = c->lp_mlz;
  a.logprobs = c->logprobs;
  a.lp_grid = c->lp_grid;
  a.tok_logits = c->topp ? (c->logits_dump ? c->logits_dump : c->logits_tp) : nullptr;
  a.vocab = c->sh.vocab;
  a.eos_on = c->cfg.eos_enabled ? 1 : 0;
  a.eos_id = c->cfg.eos_id;
  a.last_tok = c->last_tok;
  a.last_fin = c->last_fin;
  a.row_active = c->row_active;
  a.row_uid = c->row_uid;
  a.row_lid = c->row_lid;
  a.row_t = c->row_t;
  a.row_tok = c->row_tok;
  a.row_pos = c->row_pos;
  a.row_kvloc = c->row_kvloc;
  a.row_len = c->row_len;
  a.attn_items = c->attn_items;
  a.Hkv = c->sh.n_kv_heads;
  a.nc_pre = c->nc_pre_dec;
  a.nc_suf = c->nc_suf;
  a.chunk = c->sc;
  a.tc_prefix = c->tc_prefix;
  a.pf_progress = c->pf_lookahead > 0 ? c->pf_progress : nullptr;
  a.admit = c->cfg.admit_slots > 0 ? 1 : 0;
  a.gp = c->gp;
  a.W = (int)ceil_div64(c->max_new, c->pt);
  a.E = c->num_pages - c->gp * a.W;  // (one group: the pool beyond the guaranteed reservations)
  a.pred = c->pred;
  a.adm_seq = c->adm_seq;
  a.stall = c->stall;
  return a;
}

// Launch recorder for is_profile_step.
struct Prof {
  std::vector<cudaEvent_t>* ev;
  std::vector<int>* kind;
  bool graph;  // capturing: record as event nodes of the step graph
};
static Prof* g_prof = nullptr;
static void prof_mark(cudaStream_t st, int kind) {
  if (!g_prof) return;
  cudaEvent_t e;
  cudaEventCreate(&e);
  if (g_prof->graph) cudaEventRecordWithFlags(e, st, cudaEventRecordExternal);
  else cudaEventRecord(e, st);
  g_prof->ev->push_back(e);
  g_prof->kind->push_back(kind);
}


// Attention launches of one layer.  Decode: the shared-prefix part on tcgen05
// (attn_prefix_tc_kernel, one CTA per (group, kv head, 128-token prefix tile)) then the
// per-slot suffix units, whose last unit per (row, kv head) merges it (fused), or 64-token
// CTA units and a separate merge kernel; without the tcgen05 prefix (N > 64) the prefix
// chunks are CUDA-core work items of the same attn_kernel.  Prefill: causal CUDA-core
// prefix units + merge.
struct AttnLaunch {
  const CUtensorMap* tm_prefix;  // decode tcgen05 prefix: rows = groups x grp_kv_rows, 128 bf16 columns
  int kv_row_base;               // tensor-map row of this layer's prefix K, group 0
  int grp_kv_rows;               // tensor-map rows per group
  int groups;                    // co-resident groups M
  int grp_rows;                  // rows per group g
  const CUtensorMap* tm_pool;    // decode mma suffix pass: the page pool, rows of 128 bf16, box = page_tokens
  int suffix_mma;                // decode: suffix units on mma.sync (attn_suffix_mma_kernel)
  int suffix_shape;              //   0: 6 warps x 2 stages, 1: 8 warps x 1 stage
  int carveout;                  // shared-memory carveout (%) for the prefix / suffix kernels, -1: default
  int prefix2;                   // decode tcgen05 prefix with the query rows as M (attn_prefix_tc2_kernel)
};

// Per-kernel shared-memory carveout, set only when it changes (contexts of different row counts
// may share a kernel instantiation).  -1 = the driver's default (0 after a change).
static is_status set_carveout(const void* kern, int carveout) {
  static std::vector<std::pair<const void*, int>> cur;
  const int v = carveout < 0 ? 0 : carveout;
  for (auto& pr : cur)
    if (pr.first == kern) {
      if (pr.second == v) return IS_OK;
      pr.second = v;
      CK(cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, v));
      return IS_OK;
    }
  if (carveout < 0) return IS_OK;  // never set: leave the default
  cur.push_back({kern, v});
  CK(cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, v));
  return IS_OK;
}

template <int REP, int N>
static is_status launch_prefix_tc_n(const AttnArgs& aa, const AttnLaunch& al, cudaStream_t st) {
  using SM = PrefixTcSmem<N>;
  auto kern = attn_prefix_tc_kernel<REP, N>;
  static bool attr = false;
  if (!attr) {
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, SM::v));
    attr = true;
  }
  CKS(set_carveout((const void*)kern, al.carveout));
  const int nt = (int)ceil_div64(aa.plen, 128);
  cudaLaunchConfig_t cfg{};
  cudaLaunchAttribute at[1];
  cfg.gridDim = dim3(al.groups * aa.Hkv * nt);
  cfg.blockDim = dim3(128);
  cfg.dynamicSmemBytes = SM::v;
  cfg.stream = st;
  cfg.numAttrs = 0;
  if (g_use_pdl) {
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
  }
  AttnArgs a2 = aa;
  a2.dbg_ts = aa.dbg_ts ? aa.dbg_ts + (size_t)2 * 296 * 16 : nullptr;
  a2.grp_rows = al.grp_rows;
  a2.grp_kv_rows = al.grp_kv_rows;
  CK(cudaLaunchKernelEx(&cfg, kern, *al.tm_prefix, a2, al.kv_row_base));
  ++g_launches;
  return IS_OK;
}
// MMA N of the tcgen05 prefix part: one group's live slots x Hq/Hkv query heads, padded to 16.
static int prefix_cols(int g, int rep) { return (int)ceil_div64((int64_t)g * rep, 16) * 16; }

template <int REP, int MT>
static is_status launch_prefix_tc2(const AttnArgs& aa, const AttnLaunch& al, cudaStream_t st) {
  using SM = PrefixTc2Smem<MT>;
  auto kern = attn_prefix_tc2_kernel<REP, MT>;
  static bool attr = false;
  if (!attr) {
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, SM::v));
    attr = true;
  }
  CKS(set_carveout((const void*)kern, al.carveout));
  const int nt = (int)ceil_div64(aa.plen, 128);
  cudaLaunchConfig_t cfg{};
  cudaLaunchAttribute at[1];
  cfg.gridDim = dim3(al.groups * aa.Hkv * nt);
  cfg.blockDim = dim3(128);
  cfg.dynamicSmemBytes = SM::v;
  cfg.stream = st;
  cfg.numAttrs = 0;
  if (g_use_pdl) {
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
  }
  AttnArgs a2 = aa;
  a2.dbg_ts = aa.dbg_ts ? aa.dbg_ts + (size_t)2 * 296 * 16 : nullptr;
  a2.grp_rows = al.grp_rows;
  a2.grp_kv_rows = al.grp_kv_rows;
  CK(cudaLaunchKernelEx(&cfg, kern, *al.tm_prefix, a2, al.kv_row_base));
  ++g_launches;
  return IS_OK;
}

template <int REP>
static is_status launch_attn_rep(AttnArgs aa, const AttnLaunch& al, cudaStream_t st) {
  if (aa.tc_prefix && al.prefix2) {
    const int nrows = al.grp_rows * REP;
    if (nrows <= 128) CKS((launch_prefix_tc2<REP, 1>(aa, al, st)));
    else if (nrows <= 256) CKS((launch_prefix_tc2<REP, 2>(aa, al, st)));
    else return fail(IS_ERR_CONFIG, "tcgen05 prefix attention needs g * Hq/Hkv <= 256");
  } else if (aa.tc_prefix) {
    switch (prefix_cols(al.grp_rows, REP)) {
      case 16: CKS((launch_prefix_tc_n<REP, 16>(aa, al, st))); break;
      case 32: CKS((launch_prefix_tc_n<REP, 32>(aa, al, st))); break;
      case 64: CKS((launch_prefix_tc_n<REP, 64>(aa, al, st))); break;
      default: return fail(IS_ERR_CONFIG, "tcgen05 prefix attention needs g * Hq/Hkv <= 64");
    }
  }
  if (al.suffix_mma) {  // decode, 64-token units on mma.sync with the fused merge
    const bool wide = al.suffix_shape == 1;  // 8 warps x 1 stage (small launches) vs 6 x 2
    // A suffix CTA does not fit beside a tcgen05 prefix CTA: with few prefix CTAs, the last
    // suffix CTAs start only when the prefix kernel exits, so they get no static units and no
    // merges (those would set the kernel's tail).
    aa.early_ctas = 0;
    if (aa.tc_prefix && !getenv("IS_NO_EARLY_CTAS")) {
      const int npre = al.groups * aa.Hkv * (int)ceil_div64(aa.plen, 128);
      if (npre <= g_num_sms / 4) aa.early_ctas = g_num_sms - npre;
    }
#define IS_SUFFIX_MMA(P)                                                                                         \
  (wide ? (set_carveout((const void*)attn_suffix_mma_kernel<REP, P, 8, 1>, al.carveout) != IS_OK                     \
               ? IS_ERR_CUDA                                                                                     \
               : launch_k_smem(attn_suffix_mma_kernel<REP, P, 8, 1>, dim3(g_num_sms), dim3(256),                 \
                               SuffixMmaSmem<8, 1, REP>::v, st, *al.tm_pool, aa))                                \
        : (set_carveout((const void*)attn_suffix_mma_kernel<REP, P, 6, 2>, al.carveout) != IS_OK                     \
               ? IS_ERR_CUDA                                                                                     \
               : launch_k_smem(attn_suffix_mma_kernel<REP, P, 6, 2>, dim3(g_num_sms), dim3(192),                 \
                               SuffixMmaSmem<6, 2, REP>::v, st, *al.tm_pool, aa)))
    switch (aa.pt) {
      case 8: CKS(IS_SUFFIX_MMA(8)); break;
      case 16: CKS(IS_SUFFIX_MMA(16)); break;
      case 32: CKS(IS_SUFFIX_MMA(32)); break;
#undef IS_SUFFIX_MMA
      default: return fail(IS_ERR_CONFIG, "the mma suffix pass needs page_tokens 8, 16 or 32");
    }
    return IS_OK;
  }
  if (aa.merge_cnt) {  // decode, warp units with the fused merge
    CKS(launch_k_smem(attn_suffix_warp_kernel<REP>, dim3(3 * g_num_sms), dim3(kAttnThreads), SuffixWarpSmem<REP>::v,
                      st, aa));
    return IS_OK;
  }
  const int nblk = aa.prefill ? aa.Hkv * aa.nc_pre * (int)ceil_div64(aa.rows, kAttnWarps) : 4 * g_num_sms;
  CKS(launch_k_smem(attn_kernel<REP>, dim3(nblk), dim3(kAttnThreads), AttnSmem<REP>::v, st, aa));
  CKS(launch_k(attn_merge_kernel<REP>, dim3(aa.rows, aa.Hkv), dim3(32), st, aa));
  return IS_OK;
}

static is_status launch_attention(const AttnArgs& aa, const AttnLaunch& al, cudaStream_t st) {
  switch (aa.Hq / aa.Hkv) {
    case 1: return launch_attn_rep<1>(aa, al, st);
    case 2: return launch_attn_rep<2>(aa, al, st);
    case 4: return launch_attn_rep<4>(aa, al, st);
    case 8: return launch_attn_rep<8>(aa, al, st);
  }
  return fail(IS_ERR_CONFIG, "Hq / Hkv must be 1, 2, 4 or 8");
}

// One layer stack over `rows` rows starting at row 0 (decode: rows = rc, BN = c->BN;
// prefill: rows = pcap processed in 64-row GEMM chunks).
static is_status run_layers(is_ctx* c, int rows, bool prefill, int grp = 0) {
  g_splitk_ws = c->splitk_ws;
  cudaStream_t st = c->st;
  // prefill: the group slot's own prefix KV and separate row tables (decode rows stay intact)
  int32_t* r_active = prefill ? c->prow_active : c->row_active;
  int32_t* r_tok = prefill ? c->prow_tok : c->row_tok;
  int32_t* r_pos = prefill ? c->prow_pos : c->row_pos;
  int32_t* r_kvloc = prefill ? c->prow_kvloc : c->row_kvloc;
  int32_t* r_len = prefill ? c->prow_len : c->row_len;
  __nv_bfloat16* prefix_g = c->prefix + (size_t)grp * c->sh.layers * 2 * c->sh.n_kv_heads * c->pcap * kHD;
  const is_shape& s = c->sh;
  const int H = s.hidden, F = s.ffn, Hq = s.n_q_heads, Hkv = s.n_kv_heads;
  const int BN = prefill ? 64 : c->BN;
  const CUtensorMap& tm_xn = prefill ? c->tm_xn_pre : c->tm_xn_dec;
  const CUtensorMap& tm_attn = prefill ? c->tm_attn_pre : c->tm_attn_dec;
  const CUtensorMap& tm_act = prefill ? c->tm_act_pre : c->tm_act_dec;
  const int chunk = prefill ? 64 : rows;

  prof_mark(st, 0);
  if (prefill || !(g_skip & 128))
    CKS(launch_k(embed_kernel, dim3(rows), dim3(128), st, (const __nv_bfloat16*)c->embed,
                 (const int32_t*)r_tok, (const int32_t*)r_active, c->resid, H, (const float*)c->L[0].in_norm, c->xn,
                 c->ssqA, c->max_rows));
  for (int l = 0; l < s.layers; ++l) {
    LayerW& w = c->L[l];
    prof_mark(st, 0);
    const size_t prefix_layer = (size_t)2 * Hkv * c->pcap * kHD;
    const size_t pool_layer = (size_t)c->num_pages * 2 * Hkv * c->pt * kHD;
    for (int r0 = 0; r0 < rows; r0 += chunk) {
      GemmArgs a{};
      a.M = c->qkv_w;
      a.K = H;
      a.num_tiles = ceil_div64(a.M, kBM);
      a.split = prefill ? choose_split(a.num_tiles, H / kBK, 16) : c->split_qkv;
      a.row0 = r0;
      a.n_valid = std::min(chunk, rows - r0);
      QkvEpiArgs& e = a.qkv;
      e.q_gain = w.q_norm;
      e.k_gain = w.k_norm;
      e.rope_cos = c->rope_cos;
      e.rope_sin = c->rope_sin;
      e.row_active = r_active;
      e.row_pos = r_pos;
      e.row_kvloc = r_kvloc;
      e.q_out = c->q;
      e.kv = prefill ? prefix_g + l * prefix_layer : c->pool + l * pool_layer;
      e.Hq = Hq;
      e.Hkv = Hkv;
      e.pt = c->pt;
      e.pcap = c->pcap;
      e.prefill = prefill ? 1 : 0;
      e.eps = s.rms_eps;
      a.rs_ssq = c->ssqA;  // RMSNorm (R12b): B = bf16(x * in_norm) from embed / the previous down epilogue
      a.rs_nt = (int)ceil_div64(H, kBM);
      a.rs_ld = c->max_rows;
      a.rs_eps = s.rms_eps;
      if (!prefill && c->pf_lookahead > 0) {
        a.pf_progress = c->pf_progress;
        a.pf_seq = 4 * l;
      }
      if (prefill || !(g_skip & 2)) CKS(launch_gemm<EPI_QKV>(BN, w.tm_qkv, tm_xn, a, st, prefill ? 0 : c->stg_qkv));
    }
    prof_mark(st, 1);
    AttnArgs aa{};
    aa.q = c->q;
    aa.kpre = prefix_g + l * prefix_layer;
    aa.vpre = aa.kpre + (size_t)Hkv * c->pcap * kHD;
    aa.pool = c->pool + l * pool_layer;
    aa.row_active = r_active;
    aa.row_len = r_len;
    aa.part_o = c->part_o;
    aa.part_ml = c->part_ml;
    aa.items = c->attn_items;
    aa.items_cap = prefill ? 0 : Hkv * (c->nc_pre * ((c->rc + 3) / 4) + c->rc * c->nc_suf);
    aa.n_items = c->st_dev + (size_t)c->M * ST_COUNT + ST_ATTN_ITEMS;
    aa.dbg_ts = nullptr;
    aa.dbg_mode = getenv("IS_DBG_ATTN_MODE") ? atoi(getenv("IS_DBG_ATTN_MODE")) : 0;  // timing experiments
    if (g_tl && l < 4) aa.dbg_ts = g_tl + (size_t)(400 + 4 * l) * 296 * 16;  // attn: 2x296 CTAs, prefix_tc after
    aa.out = c->attn;
    aa.rows = rows;
    aa.Hq = Hq;
    aa.Hkv = Hkv;
    aa.pcap = c->pcap;
    aa.plen = c->pcap;
    aa.pt = c->pt;
    aa.nc_pre = prefill ? c->nc_pre : c->nc_pre_dec;
    aa.nc_suf = prefill ? 0 : c->nc_suf;
    aa.tc_prefix = prefill ? 0 : c->tc_prefix;
    aa.merge_cnt = (!prefill && c->tc_prefix && !c->sep_merge) ? c->merge_cnt : nullptr;
    aa.pool_row0 = l * c->num_pages * 2 * Hkv;
    aa.unit_ctr = (!prefill && !c->static_units) ? c->merge_cnt + (size_t)c->max_rows * Hkv : nullptr;
    aa.merge_done = c->merge_cnt + (size_t)c->max_rows * Hkv + 2;
    if (!prefill && !g_exact_prefix_max) {
      const int nt = (int)ceil_div64(c->pcap, 128);
      aa.kmax = c->kmax + (size_t)l * Hkv * nt;
      aa.kmax_grp = s.layers * Hkv * nt;
    }
    aa.sc = prefill ? kSC : c->sc;
    aa.NC = c->NC;
    aa.prefill = prefill ? 1 : 0;
    aa.scale = 1.0f / sqrtf((float)kHD);
    if (prefill || !(g_skip & 8)) {
      AttnLaunch al{};
      al.tm_prefix = &c->tm_prefix_kv;
      al.kv_row_base = l * 2 * Hkv * c->pcap;
      al.grp_kv_rows = s.layers * 2 * Hkv * c->pcap;
      al.groups = c->M;
      al.grp_rows = c->g;
      al.tm_pool = &c->tm_pool;
      al.suffix_mma = !prefill && c->suffix_mma;
      al.suffix_shape = c->suffix_shape;
      al.carveout = c->attn_carveout;
      al.prefix2 = c->prefix2;
      CKS(launch_attention(aa, al, st));
    }
    prof_mark(st, 3);
    for (int r0 = 0; r0 < rows; r0 += chunk) {
      GemmArgs a{};
      a.M = H;
      a.K = Hq * kHD;
      a.num_tiles = ceil_div64(a.M, kBM);
      a.split = prefill ? choose_split(a.num_tiles, a.K / kBK, 16) : c->split_o;
      a.row0 = r0;
      a.n_valid = std::min(chunk, rows - r0);
      a.out = c->resid;
      a.ld_out = H;
      a.xg_gain = w.post_norm;  // the post-attention norm's operand and sums of squares (R12b)
      a.xg_out = c->xn;
      a.ssq_out = c->ssqB;
      a.ssq_ld = c->max_rows;
      if (!prefill && c->pf_lookahead > 0) {
        a.pf_progress = c->pf_progress;
        a.pf_seq = 4 * l + 1;
      }
      if (prefill || !(g_skip & 16)) CKS(launch_gemm<EPI_RESID_ADD>(BN, w.tm_o, tm_attn, a, st, prefill ? 0 : c->stg_o));
    }
    prof_mark(st, 4);
    prof_mark(st, 0);
    for (int r0 = 0; r0 < rows; r0 += chunk) {
      GemmArgs a{};
      a.M = 2 * F;
      a.K = H;
      a.num_tiles = ceil_div64(a.M, kBM);
      a.split = prefill ? choose_split(a.num_tiles, H / kBK, 16) : c->split_gu;
      a.row0 = r0;
      a.n_valid = std::min(chunk, rows - r0);
      a.act = c->act;
      a.ld_act = F;
      a.rs_ssq = c->ssqB;
      a.rs_nt = (int)ceil_div64(H, kBM);
      a.rs_ld = c->max_rows;
      a.rs_eps = s.rms_eps;
      if (!prefill && c->pf_lookahead > 0) {
        a.pf_progress = c->pf_progress;
        a.pf_seq = 4 * l + 2;
      }
      if (prefill || !(g_skip & 32)) CKS(launch_gemm<EPI_SWIGLU>(BN, w.tm_gu, tm_xn, a, st, prefill ? 0 : c->stg_gu));
    }
    prof_mark(st, 5);
    for (int r0 = 0; r0 < rows; r0 += chunk) {
      GemmArgs a{};
      a.M = H;
      a.K = F;
      a.num_tiles = ceil_div64(a.M, kBM);
      a.split = prefill ? choose_split(a.num_tiles, F / kBK, 16) : c->split_d;
      a.row0 = r0;
      a.n_valid = std::min(chunk, rows - r0);
      a.out = c->resid;
      a.ld_out = H;
      // the next layer's input norm, or the final norm before the lm_head (R12b)
      a.xg_gain = l + 1 < s.layers ? (const float*)c->L[l + 1].in_norm : (const float*)c->final_norm;
      a.xg_out = c->xn;
      a.ssq_out = c->ssqA;
      a.ssq_ld = c->max_rows;
      if (!prefill && c->pf_lookahead > 0) {
        a.pf_progress = c->pf_progress;
        a.pf_seq = 4 * l + 3;
      }
      if (prefill || !(g_skip & 64)) CKS(launch_gemm<EPI_RESID_ADD>(BN, w.tm_d, tm_act, a, st, prefill ? 0 : c->stg_d));
    }
    prof_mark(st, 6);
  }
  return IS_OK;
}

static is_status enqueue_step_body(is_ctx* c);
static is_status enqueue_step(is_ctx* c) {
  const int launches0 = g_launches;
  is_status r = enqueue_step_body(c);
  c->launches_per_step = g_launches - launches0;
  return r;
}

static is_status enqueue_step_body(is_ctx* c) {
  cudaStream_t st = c->st;
  const is_shape& s = c->sh;
  if (c->pf_lookahead > 0) {
    // the L2 weight prefetcher runs beside the step (fork here, join before the scheduler)
    CK(cudaEventRecord(c->pf_fork, st));
    CK(cudaStreamWaitEvent(c->pf_st, c->pf_fork, 0));
    PrefetchArgs pa{c->pf_ptr, c->pf_off, c->pf_n, c->pf_progress, c->pf_lookahead};
    l2_prefetch_kernel<<<1, 32, 0, c->pf_st>>>(pa);
    CK(cudaGetLastError());
    ++g_launches;
    CK(cudaEventRecord(c->pf_join, c->pf_st));
  }
  CKS(run_layers(c, c->rc, false));
  prof_mark(st, 0);
  GemmArgs a{};
  a.M = s.vocab;
  a.K = s.hidden;
  a.num_tiles = ceil_div64(a.M, kBM);
  a.split = 1;
  a.row0 = 0;
  a.n_valid = c->rc;
  a.ld_out = s.vocab;
  a.row_uid = c->row_uid;
  a.row_t = c->row_t;
  a.row_active = c->row_active;
  a.keys = c->keys;
  a.lp_key = c->lp_key;
  a.lp_mlz = c->lp_mlz;
  a.logits_dump = c->topp ? (c->logits_dump ? c->logits_dump : c->logits_tp) : c->logits_dump;
  a.score_dump = c->topp ? c->scores_tp : nullptr;
  a.seed = c->cfg.seed;
  a.inv_temp = (float)(1.0 / (double)c->cfg.temperature);
  a.rs_ssq = c->ssqA;  // final norm (R12b): B = bf16(x * final_norm) from the last down epilogue
  a.rs_nt = (int)ceil_div64(s.hidden, kBM);
  a.rs_ld = c->max_rows;
  a.rs_eps = s.rms_eps;
  g_splitk_ws = c->splitk_ws;
  if (c->pf_lookahead > 0) {
    a.pf_progress = c->pf_progress;
    a.pf_seq = 4 * s.layers;
  }
  CKS(launch_gemm<EPI_SAMPLE>(c->BN, c->tm_embed, c->tm_xn_dec, a, st, c->stg_lm));
  if (c->topp) {  // top-p < 1 (R36): the nucleus and its Gumbel-max replace the full-vocabulary key
    ToppArgs t{};
    t.scores = c->scores_tp;
    t.logits = a.logits_dump;
    t.lp_mlz = c->lp_mlz;
    t.lp_grid = c->lp_grid;
    t.ebits = c->ebits_tp;
    t.wpart = c->wpart_tp;
    t.hist1 = c->hist_tp;
    t.sel = c->sel_tp;
    t.row_active = c->row_active;
    t.keys = c->keys;
    t.V = s.vocab;
    t.invT = a.inv_temp;
    t.top_p = c->cfg.top_p;
    ToppState* ts = c->state_tp;
    CKS(launch_k(topp_prep_kernel, dim3(kToppBlocks, c->rc), dim3(kToppThreads), st, t));
    for (int shift = 24; shift >= 0; shift -= 8) {
      if (shift < 24) CKS(launch_k(topp_hist_kernel, dim3(kToppBlocks, c->rc), dim3(kToppThreads), st, t,
                                   (const ToppState*)ts, shift));
      CKS(launch_k(topp_pick_kernel, dim3(c->rc), dim3(256), st, t, ts, shift));
    }
    CKS(launch_k(topp_tiecount_kernel, dim3(kToppBlocks, c->rc), dim3(kToppThreads), st, t, (const ToppState*)ts));
    CKS(launch_k(topp_tiepick_kernel, dim3(c->rc), dim3(kToppThreads), st, t, (const ToppState*)ts));
    CKS(launch_k(topp_sample_kernel, dim3(kToppBlocks, c->rc), dim3(kToppThreads), st, t));
  }
  prof_mark(st, 7);
  if (c->pf_lookahead > 0) CK(cudaStreamWaitEvent(st, c->pf_join, 0));
  CKS(launch_k(sched_kernel, dim3(1), dim3(kSchedThreads), st, sched_args(c), 1, (1 << c->M) - 1));
  prof_mark(st, 8);
  CK(cudaMemcpyAsync(c->st_host, c->st_dev, sizeof(long long) * ST_COUNT * (c->M + 1), cudaMemcpyDeviceToHost, st));
  return IS_OK;
}

static is_status build_graph(is_ctx* c) {
  if (c->graph_ok) {
    cudaGraphExecDestroy(c->graph);
    c->graph_ok = false;
  }
  cudaGraph_t g;
  if (getenv("IS_TIMELINE") && !c->timeline) {
    cudaMalloc(&c->timeline, (size_t)512 * 296 * 16 * 8);
    cudaMemset(c->timeline, 0, (size_t)512 * 296 * 16 * 8);
  }
  g_tl = c->timeline;
  g_tl_n = 0;
  CK(cudaStreamBeginCapture(c->st, cudaStreamCaptureModeThreadLocal));
  is_status s = enqueue_step(c);
  g_tl = nullptr;
  c->tl_count = g_tl_n;
  cudaError_t e = cudaStreamEndCapture(c->st, &g);
  if (s != IS_OK) return s;
  CK(e);
  CK(cudaGraphInstantiate(&c->graph, g, 0));
  cudaGraphDestroy(g);
  c->graph_ok = true;
  // the run loops replay K steps per launch: PDL then spans K-1 of the step boundaries
  if (c->graphK_ok) {
    cudaGraphExecDestroy(c->graphK);
    c->graphK_ok = false;
  }
  if (c->steps_per_graph > 1 && !getenv("IS_TIMELINE")) {
    CK(cudaStreamBeginCapture(c->st, cudaStreamCaptureModeThreadLocal));
    is_status sk = IS_OK;
    for (int k = 0; k < c->steps_per_graph && sk == IS_OK; ++k) sk = enqueue_step(c);
    cudaError_t ek = cudaStreamEndCapture(c->st, &g);
    if (sk != IS_OK) return sk;
    CK(ek);
    CK(cudaGraphInstantiate(&c->graphK, g, 0));
    cudaGraphDestroy(g);
    c->graphK_ok = true;
  }
  return IS_OK;
}

// Order the context stream after the caller's stream and vice versa.
struct StreamGuard {
  is_ctx* c;
  cudaStream_t user;
  StreamGuard(is_ctx* c_, cudaStream_t u) : c(c_), user(u) {
    cudaEventRecord(c->ev_in, user);
    cudaStreamWaitEvent(c->st, c->ev_in, 0);
  }
  ~StreamGuard() {
    cudaEventRecord(c->ev_out, c->st);
    cudaStreamWaitEvent(user, c->ev_out, 0);
  }
};

extern "C" is_status is_create(const is_config* cfg, const void* const* dw, int32_t nw, void* stream,
                               is_ctx** out) {
  if (!cfg || !dw || !out) return fail(IS_ERR_CONFIG, "null argument");
  CKS(check_config(cfg));
  const is_shape& s = cfg->shape;
  if (nw != 2 + 11 * s.layers) return fail(IS_ERR_CONFIG, "expected %d weight pointers, got %d", 2 + 11 * s.layers, nw);
  if (!get_encode()) return fail(IS_ERR_CUDA, "no CUDA driver / TMA encoder available");
  int dev = 0;
  CK(cudaGetDevice(&dev));
  cudaDeviceProp prop;
  CK(cudaGetDeviceProperties(&prop, dev));
  if (prop.major != 10) return fail(IS_ERR_CUDA, "needs an sm_100 (B200) device, found sm_%d%d", prop.major, prop.minor);
  g_num_sms = prop.multiProcessorCount;
  if (getenv("IS_NO_PDL")) g_use_pdl = false;
  g_exact_prefix_max = getenv("IS_EXACT_PREFIX_MAX") != nullptr;
  if (getenv("IS_SKIP")) g_skip = atoi(getenv("IS_SKIP"));

  is_ctx* c = new is_ctx{};
  c->user = (cudaStream_t)stream;
  c->cfg = *cfg;
  c->sh = s;
  c->G = cfg->G;
  c->g = slots_of(cfg);   // rows (slots) per group
  c->gp = eff_g(cfg);     // the plan's micro-group size (guaranteed slots with admission, R41)
  c->M = n_groups(cfg);
  c->gprompt_id.assign(c->M, 0);
  c->gprompt_last.assign(c->M, 0);
  c->gprefilled.assign(c->M, 0);
  c->gstarted.assign(c->M, 0);
  c->N = c->G / c->gp;
  c->rc = row_cap_of(cfg);
  if (c->rc < c->g || c->rc > 64) {
    delete c;
    return fail(IS_ERR_CAPACITY, "row_capacity %d must be in [g=%d, 64]", c->rc, c->g);
  }
  c->BN = c->rc <= 16 ? 16 : (c->rc <= 32 ? 32 : 64);
  c->P = cfg->prompt_len;
  c->pcap = c->P - 1;
  c->pt = cfg->page_tokens;
  c->max_new = cfg->max_new_tokens;
  c->maxp = (int)ceil_div64(c->max_new, c->pt);
  c->qkv_w = (s.n_q_heads + 2 * s.n_kv_heads) * 128;
  c->page_bytes = (int64_t)c->pt * kv_bytes_per_token(s);
  c->prefix_bytes = (int64_t)c->pcap * kv_bytes_per_token(s);
  const int64_t resv = reservation_bytes(cfg);
  if (cfg->kv_budget_bytes > 0) {
    if (resv > cfg->kv_budget_bytes) {
      delete c;
      return fail(IS_ERR_BUDGET, "worst-case KV reservation %lld B exceeds budget %lld B", (long long)resv,
                  (long long)cfg->kv_budget_bytes);
    }
    c->num_pages = (int)((cfg->kv_budget_bytes - c->prefix_bytes) / c->page_bytes);
  } else {
    c->num_pages = (int)((resv - c->prefix_bytes) / c->page_bytes);
  }
  c->num_pages *= c->M;  // the budget is per group; the pool is shared by the co-resident groups
  if (const char* e = getenv("IS_DBG_POOL_PAGES")) c->num_pages = std::max(1, atoi(e));  // negative tests only
  c->log_cap = c->G * c->max_new + c->N * cfg->prefix_k + 8;
  c->max_rows = std::max(c->rc, (int)ceil_div64(c->pcap, 64) * 64);
  c->max_pos = c->P + c->max_new + 1;
  c->nc_pre = (int)ceil_div64(c->pcap, kPC);  // prefill (CUDA-core causal prefix units)
  {
    const int N = prefix_cols(c->g, s.n_q_heads / s.n_kv_heads);
    // round 1's tokens-as-M kernel up to 64 stacked rows (its softmax spreads a tile's tokens over
    // all 128 threads: 5.9 vs 8.3 us at 16 rows), the query-rows-as-M kernel beyond (up to 256;
    // 1.7x the CUDA-core prefix at 128 rows); IS_PREFIX_IMPL=2 forces the latter
    const char* pe = getenv("IS_PREFIX_IMPL");
    c->prefix2 = (pe && atoi(pe) == 2) || N > 64;
    c->tc_prefix = (c->prefix2 ? c->g * (s.n_q_heads / s.n_kv_heads) <= 256 : (N == 16 || N == 32 || N == 64)) &&
                   !getenv("IS_NO_TC_PREFIX");
    c->nc_pre_dec = c->tc_prefix ? (int)ceil_div64(c->pcap, 128) : c->nc_pre;
  }
  // decode suffix pass behind the tcgen05 prefix: 64-token units on mma.sync with the fused
  // merge (default; needs page_tokens % 8 == 0 for the swizzled page boxes); IS_SUFFIX_IMPL=
  // warp / cta selects round 1's 32-token warp units (fused merge) or 64-token CTA units with
  // the separate merge kernel.  Without the tcgen05 prefix: 64-token CTA units + merge kernel.
  {
    const char* e = getenv("IS_SUFFIX_IMPL");
    c->suffix_mma = c->tc_prefix && c->pt % 8 == 0 && c->pt <= kSUnit && !(e && strcmp(e, "mma"));
    c->sep_merge = !c->suffix_mma && (!c->tc_prefix || c->pt > kSCW || (e && !strcmp(e, "cta")));
    if (c->sep_merge && c->tc_prefix && c->pt <= kSCW && c->nc_pre_dec + ceil_div64(c->max_new, kSC) > 32)
      c->sep_merge = 0;
  }
  c->sc = c->suffix_mma ? kSUnit : ((c->tc_prefix && !c->sep_merge) ? kSCW : kSC);
  {
    // suffix kernel shape: 8 warps x 1 stage up to 16 rows (each warp has ~1-2 units), else 6 x 2
    const char* e = getenv("IS_SUFFIX_SHAPE");
    c->suffix_shape = e ? atoi(e) : 1;
    // beyond 16 rows (co-resident groups) the tcgen05 prefix CTAs are many: with the maximum
    // carveout a suffix CTA fits beside each, so the suffix pass starts at once (K5 8 groups x 1024:
    // 78.9 -> 68.6 us, profiles/r02c); at 16 rows the co-resident prefix chain slows instead
    const char* cv = getenv("IS_ATTN_CARVEOUT");
    c->attn_carveout = cv ? atoi(cv) : (c->rc > 16 ? 100 : -1);
  }
  c->nc_suf = (int)ceil_div64(c->max_new, c->sc);
  c->NC = c->nc_pre + c->nc_suf;
  // partials one LSE merge combines: decode = prefix tiles + suffix chunks, prefill = prefix chunks
  const int ndec = c->nc_pre_dec + c->nc_suf, nmax = c->sep_merge || !c->tc_prefix ? 32 : 64;
  if (ndec > nmax || c->nc_pre > 32 || s.n_q_heads / s.n_kv_heads > kMaxRep) {
    delete c;
    return fail(IS_ERR_CAPACITY, "prompt_len + max_new_tokens too long for the attention merge (%d partials > %d)",
                ndec, nmax);
  }
  c->prompt_id = 0;

  is_status err = IS_OK;
  auto A = [&](size_t bytes) { return err == IS_OK ? dalloc(bytes, &err) : nullptr; };
  CK(cudaStreamCreateWithFlags(&c->st, cudaStreamNonBlocking));
  CK(cudaEventCreateWithFlags(&c->ev_in, cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&c->ev_out, cudaEventDisableTiming));
  const int H = s.hidden, F = s.ffn, Hq = s.n_q_heads, Hkv = s.n_kv_heads, V = s.vocab;
  // ---- weights (packed copies)
  const size_t per_layer = (size_t)c->qkv_w * H + (size_t)H * Hq * 128 + (size_t)2 * F * H + (size_t)H * F;
  c->wblob = A(((size_t)V * H + per_layer * s.layers) * 2);
  if (err != IS_OK) return err;
  __nv_bfloat16* wp = reinterpret_cast<__nv_bfloat16*>(c->wblob);
  c->embed = wp;
  wp += (size_t)V * H;
  CK(cudaMemcpy(c->embed, dw[0], (size_t)V * H * 2, cudaMemcpyDeviceToDevice));
  c->final_norm = (float*)A(H * 4);
  if (err != IS_OK) return err;
  bf16_to_f32_kernel<<<(H + 255) / 256, 256>>>((const __nv_bfloat16*)dw[1], c->final_norm, H);
  c->L.resize(s.layers);
  for (int l = 0; l < s.layers; ++l) {
    const void* const* p = dw + 2 + 11 * l;
    LayerW& w = c->L[l];
    w.wqkv = wp;
    wp += (size_t)c->qkv_w * H;
    w.wo = wp;
    wp += (size_t)H * Hq * 128;
    w.wgu = wp;
    wp += (size_t)2 * F * H;
    w.wd = wp;
    wp += (size_t)H * F;
    const size_t qn = (size_t)Hq * 128 * H, kn = (size_t)Hkv * 128 * H;
    CK(cudaMemcpy(w.wqkv, p[1], qn * 2, cudaMemcpyDeviceToDevice));
    CK(cudaMemcpy(w.wqkv + qn, p[2], kn * 2, cudaMemcpyDeviceToDevice));
    CK(cudaMemcpy(w.wqkv + qn + kn, p[3], kn * 2, cudaMemcpyDeviceToDevice));
    CK(cudaMemcpy(w.wo, p[6], (size_t)H * Hq * 128 * 2, cudaMemcpyDeviceToDevice));
    // gate|up interleaved per 64-row block: rows [128b, 128b+64) gate, [128b+64, 128b+128) up
    const size_t blk = (size_t)64 * H * 2;
    CK(cudaMemcpy2D(w.wgu, 2 * blk, p[8], blk, blk, F / 64, cudaMemcpyDeviceToDevice));
    CK(cudaMemcpy2D(reinterpret_cast<uint8_t*>(w.wgu) + blk, 2 * blk, p[9], blk, blk, F / 64,
                    cudaMemcpyDeviceToDevice));
    CK(cudaMemcpy(w.wd, p[10], (size_t)H * F * 2, cudaMemcpyDeviceToDevice));
    w.in_norm = (float*)A(H * 4);
    w.post_norm = (float*)A(H * 4);
    w.q_norm = (float*)A(128 * 4);
    w.k_norm = (float*)A(128 * 4);
    if (err != IS_OK) return err;
    bf16_to_f32_kernel<<<(H + 255) / 256, 256>>>((const __nv_bfloat16*)p[0], w.in_norm, H);
    bf16_to_f32_kernel<<<(H + 255) / 256, 256>>>((const __nv_bfloat16*)p[7], w.post_norm, H);
    bf16_to_f32_kernel<<<1, 128>>>((const __nv_bfloat16*)p[4], w.q_norm, 128);
    bf16_to_f32_kernel<<<1, 128>>>((const __nv_bfloat16*)p[5], w.k_norm, 128);
    CKS(make_tmap(&w.tm_qkv, w.wqkv, c->qkv_w, H, kBM));
    CKS(make_tmap(&w.tm_o, w.wo, H, Hq * 128, kBM));
    CKS(make_tmap(&w.tm_gu, w.wgu, 2 * F, H, kBM));
    CKS(make_tmap(&w.tm_d, w.wd, H, F, kBM));
  }
  CKS(make_tmap(&c->tm_embed, c->embed, V, H, kBM));
  CK(cudaDeviceSynchronize());
  // ---- KV
  c->prefix = (__nv_bfloat16*)A((size_t)c->M * s.layers * 2 * Hkv * c->pcap * 128 * 2);
  if (err == IS_OK) CKS(make_tmap(&c->tm_prefix_kv, c->prefix, (int64_t)c->M * s.layers * 2 * Hkv * c->pcap, 128, 128));
  c->pool = (__nv_bfloat16*)A((size_t)s.layers * c->num_pages * (size_t)c->page_bytes / s.layers);
  if (err == IS_OK && c->suffix_mma)
    CKS(make_tmap_pool(&c->tm_pool, c->pool, (int64_t)s.layers * c->num_pages, Hkv, c->pt));
  // ---- activations
  const int R = c->max_rows;
  c->resid = (float*)A((size_t)R * H * 4);
  c->xn = (__nv_bfloat16*)A((size_t)R * H * 2);
  c->attn = (__nv_bfloat16*)A((size_t)R * Hq * 128 * 2);
  c->act = (__nv_bfloat16*)A((size_t)R * F * 2);
  c->q = (__nv_bfloat16*)A((size_t)R * Hq * 128 * 2);
  c->part_o = (float*)A((size_t)R * Hq * c->NC * 128 * 4);
  c->part_ml = (float*)A((size_t)R * Hq * c->NC * 2 * 4);
  c->merge_cnt = (int*)A(((size_t)2 * R * Hkv + 2) * 4);  // + 2 unit counters + merged-head counters
  c->static_units = getenv("IS_STATIC_UNITS") != nullptr;  // timing comparison only
  c->kmax = (float*)A((size_t)c->M * s.layers * Hkv * ceil_div64(c->pcap, 128) * 4);
  c->ssqA = (float*)A((size_t)ceil_div64(H, 128) * R * 4);
  c->ssqB = (float*)A((size_t)ceil_div64(H, 128) * R * 4);
  c->splitk_ws = (float*)A((size_t)2 * 160 * kBM * 64 * 4);
  c->topp = cfg->top_p > 0.f && cfg->top_p < 1.f;
  c->logits_tp = c->topp ? (float*)A((size_t)R * s.vocab * 4) : nullptr;
  c->scores_tp = c->topp ? (float*)A((size_t)R * s.vocab * 4) : nullptr;
  c->ebits_tp = c->topp ? (uint32_t*)A((size_t)R * s.vocab * 4) : nullptr;
  c->wpart_tp = c->topp ? (unsigned long long*)A((size_t)R * kToppBlocks * 8) : nullptr;
  c->hist_tp = c->topp ? (unsigned long long*)A((size_t)R * kToppBlocks * 256 * 8) : nullptr;
  c->sel_tp = c->topp ? (int2*)A((size_t)R * 8) : nullptr;
  c->state_tp = c->topp ? (ToppState*)A((size_t)R * sizeof(ToppState)) : nullptr;
  c->attn_items = (int32_t*)A((size_t)Hkv * (c->nc_pre * ((c->rc + 3) / 4) + c->rc * c->nc_suf) * kItemStride * 4 + 64);
  c->rope_cos = (float*)A((size_t)c->max_pos * 64 * 4);
  c->rope_sin = (float*)A((size_t)c->max_pos * 64 * 4);
  for (int32_t** p : {&c->row_active, &c->row_uid, &c->row_lid, &c->row_t, &c->row_tok, &c->row_pos,
                      &c->row_kvloc, &c->row_len})
    *p = (int32_t*)A((size_t)R * 4);
  for (int32_t** p : {&c->prow_active, &c->prow_tok, &c->prow_pos, &c->prow_kvloc, &c->prow_len})
    *p = (int32_t*)A((size_t)R * 4);
  c->keys = (unsigned long long*)A((size_t)R * 8);
  c->lp_grid = std::min((int)ceil_div64(s.vocab, kBM), g_num_sms);  // the lm_head launch's grid
  c->lp_key = (unsigned long long*)A((size_t)R * c->lp_grid * 8);
  c->lp_mlz = (float4*)A((size_t)R * c->lp_grid * 16);
  c->last_tok = (int32_t*)A((size_t)R * 4);
  c->last_fin = (uint8_t*)A((size_t)R);
  const int M = c->M;
  c->st_dev = (long long*)A(sizeof(long long) * ST_COUNT * (M + 1));
  c->slot_uid = (int32_t*)A((size_t)M * c->g * 4);
  c->slot_count = (int32_t*)A((size_t)M * c->g * 4);
  c->tpos = (int32_t*)A((size_t)M * c->G * 4);
  c->true_len = (int32_t*)A((size_t)M * c->G * 4);
  c->queue = (int32_t*)A((size_t)M * c->G * 4);
  c->main_init = (int32_t*)A((size_t)M * c->g * 4);
  c->main_queue = (int32_t*)A((size_t)M * c->G * 4);
  c->free_stack = (int32_t*)A((size_t)std::max(c->num_pages, 1) * 4);
  c->pagetab = (int32_t*)A((size_t)M * c->G * c->maxp * 4);
  c->npages = (int32_t*)A((size_t)M * c->G * 4);
  c->tokens = (int32_t*)A((size_t)M * c->G * c->max_new * 4);
  c->log_slot = (int32_t*)A((size_t)M * c->log_cap * c->g * 4);
  c->log_live = (int32_t*)A((size_t)M * c->log_cap * 4);
  c->logprobs = (float*)A((size_t)M * c->G * c->max_new * 4);
  c->done_flag = (uint8_t*)A((size_t)M * c->G);
  c->pred = (int32_t*)A((size_t)M * c->G * 4);
  c->adm_seq = (int32_t*)A((size_t)M * c->G * 4);
  c->stall = (int32_t*)A((size_t)M * c->g * 4);
  c->d_prompt_copy = (int32_t*)A((size_t)c->P * 4);
  if (err != IS_OK) return err;
  CK(cudaMallocHost(&c->st_host, sizeof(long long) * ST_COUNT * (M + 1)));
  memset(c->st_host, 0, sizeof(long long) * ST_COUNT * (M + 1));
  {
    // shared page pool: LIFO free stack (pop order 0, 1, 2, ...), every slot idle
    std::vector<int32_t> fs(std::max(c->num_pages, 1));
    for (int i = 0; i < c->num_pages; ++i) fs[i] = c->num_pages - 1 - i;
    CK(cudaMemcpy(c->free_stack, fs.data(), fs.size() * 4, cudaMemcpyHostToDevice));
    std::vector<long long> st((size_t)ST_COUNT * (M + 1), 0);
    st[(size_t)M * ST_COUNT + ST_FREE_TOP] = c->num_pages;
    CK(cudaMemcpy(c->st_dev, st.data(), st.size() * 8, cudaMemcpyHostToDevice));
    CK(cudaMemset(c->slot_uid, 0xFF, (size_t)M * c->g * 4));
  }
  // RoPE table (rotate-half, theta^(-2i/d)), fp64 -> fp32
  {
    std::vector<float> cs((size_t)c->max_pos * 64), sn((size_t)c->max_pos * 64);
    for (int p = 0; p < c->max_pos; ++p)
      for (int i = 0; i < 64; ++i) {
        const double inv = std::pow((double)s.rope_theta, -2.0 * i / 128.0);
        const double ang = (double)p * inv;
        cs[(size_t)p * 64 + i] = (float)std::cos(ang);
        sn[(size_t)p * 64 + i] = (float)std::sin(ang);
      }
    CK(cudaMemcpy(c->rope_cos, cs.data(), cs.size() * 4, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(c->rope_sin, sn.data(), sn.size() * 4, cudaMemcpyHostToDevice));
  }
  CKS(make_tmap(&c->tm_xn_dec, c->xn, R, H, c->BN));
  CKS(make_tmap(&c->tm_attn_dec, c->attn, R, Hq * 128, c->BN));
  CKS(make_tmap(&c->tm_act_dec, c->act, R, F, c->BN));
  CKS(make_tmap(&c->tm_xn_pre, c->xn, R, H, 64));
  CKS(make_tmap(&c->tm_attn_pre, c->attn, R, Hq * 128, 64));
  CKS(make_tmap(&c->tm_act_pre, c->act, R, F, 64));
  c->split_qkv = choose_split((int)ceil_div64(c->qkv_w, kBM), H / kBK, c->BN);
  c->split_o = choose_split((int)ceil_div64(H, kBM), Hq * 128 / kBK, c->BN);
  c->split_gu = choose_split((int)ceil_div64(2 * F, kBM), H / kBK, c->BN);
  c->split_d = choose_split((int)ceil_div64(H, kBM), F / kBK, c->BN);
  c->l2_prefetch = getenv("IS_L2_PREFETCH") ? atoi(getenv("IS_L2_PREFETCH")) : 0;
  c->steps_per_graph = getenv("IS_STEPS_PER_GRAPH") ? std::max(1, atoi(getenv("IS_STEPS_PER_GRAPH"))) : 1;
  c->stg_qkv = getenv("IS_STG_QKV") ? atoi(getenv("IS_STG_QKV")) : 0;
  c->stg_o = getenv("IS_STG_O") ? atoi(getenv("IS_STG_O")) : 0;
  c->stg_gu = getenv("IS_STG_GU") ? atoi(getenv("IS_STG_GU")) : 0;
  c->stg_d = getenv("IS_STG_D") ? atoi(getenv("IS_STG_D")) : 0;
  c->stg_lm = getenv("IS_STG_LM") ? atoi(getenv("IS_STG_LM")) : 0;
  // per-GEMM split experiments (timing only)
  if (const char* e = getenv("IS_SPLIT_QKV")) c->split_qkv = std::max(1, std::min(8, atoi(e)));
  if (const char* e = getenv("IS_SPLIT_O")) c->split_o = std::max(1, std::min(8, atoi(e)));
  if (const char* e = getenv("IS_SPLIT_GU")) c->split_gu = std::max(1, std::min(8, atoi(e)));
  if (const char* e = getenv("IS_SPLIT_D")) c->split_d = std::max(1, std::min(8, atoi(e)));
  if (const char* e = getenv("IS_SPLIT_OVERRIDE")) {
    int v = atoi(e);
    if (v >= 1 && v <= 8) c->split_qkv = c->split_o = c->split_gu = c->split_d = v;
  }
  {
    // L2 weight prefetcher (opt-in: IS_L2PF = lookahead in MB)
    const char* e = getenv("IS_L2PF");
    c->pf_lookahead = e ? (long long)(atof(e) * (1 << 20)) : 0;
    if (c->pf_lookahead > 0) {
      std::vector<unsigned long long> ptr;
      std::vector<long long> off(1, 0);
      auto add = [&](const void* p, size_t bytes) {
        ptr.push_back((unsigned long long)(uintptr_t)p);
        off.push_back(off.back() + (long long)bytes);
      };
      for (int l = 0; l < s.layers; ++l) {
        const LayerW& w = c->L[l];
        add(w.wqkv, (size_t)c->qkv_w * H * 2);
        add(w.wo, (size_t)H * Hq * 128 * 2);
        add(w.wgu, (size_t)2 * F * H * 2);
        add(w.wd, (size_t)H * F * 2);
      }
      add(c->embed, (size_t)V * H * 2);
      c->pf_n = (int)ptr.size();
      c->pf_ptr = (unsigned long long*)A(ptr.size() * 8);
      c->pf_off = (long long*)A(off.size() * 8);
      c->pf_progress = (int*)A(sizeof(int));
      if (err != IS_OK) return err;
      CK(cudaMemcpy(c->pf_ptr, ptr.data(), ptr.size() * 8, cudaMemcpyHostToDevice));
      CK(cudaMemcpy(c->pf_off, off.data(), off.size() * 8, cudaMemcpyHostToDevice));
      CK(cudaMemset(c->pf_progress, 0xFF, sizeof(int)));
      CK(cudaStreamCreateWithFlags(&c->pf_st, cudaStreamNonBlocking));
      CK(cudaEventCreateWithFlags(&c->pf_fork, cudaEventDisableTiming));
      CK(cudaEventCreateWithFlags(&c->pf_join, cudaEventDisableTiming));
    }
  }
  CK(cudaDeviceSynchronize());
  *out = c;
  return IS_OK;
}

extern "C" void is_destroy(is_ctx* c) {
  if (!c) return;
  cudaStreamSynchronize(c->st);
  if (c->graph_ok) cudaGraphExecDestroy(c->graph);
  if (c->graphK_ok) cudaGraphExecDestroy(c->graphK);
  void* bufs[] = {c->wblob, c->final_norm, c->prefix, c->pool, c->resid, c->xn, c->attn, c->act, c->q,
                  c->part_o, c->part_ml, c->merge_cnt, c->kmax, c->ssqA, c->ssqB, c->attn_items, c->splitk_ws, c->rope_cos, c->rope_sin, c->row_active, c->row_uid, c->row_lid,
                  c->row_t, c->row_tok, c->row_pos, c->row_kvloc, c->row_len, c->keys, c->last_tok,
                  c->last_fin, c->st_dev, c->slot_uid, c->slot_count, c->tpos, c->true_len, c->queue,
                  c->main_init, c->main_queue, c->free_stack, c->pagetab, c->npages, c->tokens, c->log_slot,
                  c->log_live, c->d_prompt_copy, c->lp_key, c->lp_mlz, c->logprobs, c->done_flag, c->pred, c->adm_seq, c->stall, c->prow_active, c->prow_tok, c->prow_pos, c->prow_kvloc,
                  c->prow_len, c->logits_tp, c->scores_tp, c->ebits_tp, c->wpart_tp, c->hist_tp,
                  c->sel_tp, c->state_tp};
  for (void* p : bufs)
    if (p) cudaFree(p);
  for (auto& w : c->L) {
    cudaFree(w.in_norm);
    cudaFree(w.post_norm);
    cudaFree(w.q_norm);
    cudaFree(w.k_norm);
  }
  if (c->st_host) cudaFreeHost(c->st_host);
  if (c->pf_lookahead > 0) {
    cudaFree(c->pf_ptr);
    cudaFree(c->pf_off);
    cudaFree(c->pf_progress);
    cudaEventDestroy(c->pf_fork);
    cudaEventDestroy(c->pf_join);
    cudaStreamDestroy(c->pf_st);
  }
  cudaEventDestroy(c->ev_in);
  cudaEventDestroy(c->ev_out);
  cudaStreamDestroy(c->st);
  delete c;
}

// a group is done when all G samples completed, or (dynamic mode, R35) its target did
static bool group_done(const is_ctx* c, const long long* st) {
  return st[ST_DONE] >= (st[ST_TARGET] > 0 ? st[ST_TARGET] : (long long)c->G);
}

// The device scheduler found the page pool exhausted (the KV budget violated, R25):
// sticky for the context, every row idle from that step on.
static is_status budget_error() {
  return fail(IS_ERR_BUDGET, "KV page pool exhausted during decoding (budget violated); the context's rows are stopped");
}

extern "C" is_status is_prefill_slot(is_ctx* c, int32_t slot, const int32_t* d_prompt, int32_t prompt_id) {
  if (!c || !d_prompt) return fail(IS_ERR_CONFIG, "null argument");
  if (slot < 0 || slot >= c->M) return fail(IS_ERR_CONFIG, "group slot %d out of range [0, %d)", slot, c->M);
  if (c->gstarted[slot] && !group_done(c, c->st_host + (size_t)slot * ST_COUNT)) {
    // the slot's group is still decoding: wait for the stream, then look again
    CK(cudaStreamSynchronize(c->st));
    CK(cudaMemcpy(c->st_host, c->st_dev, sizeof(long long) * ST_COUNT * (c->M + 1), cudaMemcpyDeviceToHost));
  }
  StreamGuard guard(c, c->user);
  CK(cudaMemcpyAsync(c->d_prompt_copy, d_prompt, (size_t)c->P * 4, cudaMemcpyDeviceToDevice, c->st));
  int32_t last = 0;
  CK(cudaMemcpyAsync(&last, d_prompt + c->P - 1, 4, cudaMemcpyDeviceToHost, c->st));
  const int launches0 = g_launches;
  CKS(launch_k(prefill_rows_kernel, dim3((c->pcap + 127) / 128), dim3(128), c->st, (const int32_t*)c->d_prompt_copy,
               c->pcap, c->prow_active, c->prow_tok, c->prow_pos, c->prow_kvloc));
  CKS(run_layers(c, c->pcap, true, slot));
  {  // the prefix's key-norm bound per (layer, kv head, 128-token tile) for the decode prefix softmax
    const int nt = (int)ceil_div64(c->pcap, 128), Hkv = c->sh.n_kv_heads, L = c->sh.layers;
    CKS(launch_k(prefix_kmax_kernel, dim3(L * Hkv * nt), dim3(128), c->st,
                 (const __nv_bfloat16*)(c->prefix + (size_t)slot * L * 2 * Hkv * c->pcap * kHD), L, Hkv, c->pcap,
                 c->pcap, c->kmax + (size_t)slot * L * Hkv * nt));
  }
  c->launches_per_prefill = g_launches - launches0;
  CK(cudaStreamSynchronize(c->st));
  if (last < 0 || last >= c->sh.vocab) return fail(IS_ERR_DATA, "prompt token %d out of range", last);
  c->gprompt_id[slot] = prompt_id;
  c->gprompt_last[slot] = last;
  c->gprefilled[slot] = 1;
  c->gstarted[slot] = 0;
  if (slot == 0) {
    c->prompt_id = prompt_id;
    c->prompt_last = last;
    c->prefilled = true;
    c->started = false;
  }
  return IS_OK;
}

extern "C" is_status is_prefill(is_ctx* c, const int32_t* d_prompt, int32_t prompt_id) {
  return is_prefill_slot(c, 0, d_prompt, prompt_id);
}

extern "C" is_status is_start_group_slot(is_ctx* c, int32_t m, const int32_t* true_len, const int32_t* pred) {
  if (!c || !true_len) return fail(IS_ERR_CONFIG, "null argument");
  if (m < 0 || m >= c->M) return fail(IS_ERR_CONFIG, "group slot %d out of range [0, %d)", m, c->M);
  if (!c->gprefilled[m]) return fail(IS_ERR_STATE, "is_start_group before is_prefill (slot %d)", m);
  StreamGuard guard(c, c->user);
  const int G = c->G, g = c->g;  // (g = slots per group: S with memory-aware admission, R41)
  for (int i = 0; i < G; ++i)
    if (true_len[i] < 1 || true_len[i] > c->max_new)
      return fail(IS_ERR_DATA, "true length of sample %d is %d (need 1..%d)", i, true_len[i], c->max_new);
  const int k = c->cfg.prefix_k;
  std::vector<int32_t> pred_eff(G), mask(2 * G), ovf(G), init(g, -1), queue(G);
  std::vector<int64_t> sl(G), loads(std::max(c->N, c->gp));
  std::vector<uint8_t> fin(G, 0);
  for (int i = 0; i < G; ++i) {
    pred_eff[i] = pred ? pred[i] : true_len[i];
    if (k > 0 && true_len[i] <= k) {  // finished in the prefix phase: pred = true (R22)
      fin[i] = 1;
      pred_eff[i] = true_len[i];
    }
  }
  is_plan_out po{};
  po.mask = mask.data();
  po.scaled_len = sl.data();
  po.loads = loads.data();
  po.overflow_ids = ovf.data();
  po.init_slots = init.data();
  po.refill_queue = queue.data();
  CKS(is_plan(&c->cfg, pred_eff.data(), k > 0 ? fin.data() : nullptr, &po));
  // pages a previous (possibly abandoned) group of this slot still holds go back to the pool
  CKS(launch_k(reclaim_group_kernel, dim3(1), dim3(32), c->st, sched_args(c), (int)m));
  // per-group device state (block m of st; the global block M is left alone)
  std::vector<long long> st(ST_COUNT, 0);
  std::vector<int32_t> slots(g, -1), q0(G, 0);
  if (k > 0) {  // prefix phase: barriered rounds in trace order, stop at k (R22)
    st[ST_PHASE] = 0;
    st[ST_BARRIER] = 1;
    st[ST_QUOTA] = 0;
    st[ST_STOPK] = k;
    for (int s = 0; s < g; ++s) slots[s] = s;
    for (int i = g; i < G; ++i) q0[i - g] = i;
    st[ST_QLEN] = G - g;
    st[ST_MAIN_PENDING] = 1;
    st[ST_MAIN_QLEN] = po.queue_len;
    st[ST_MAIN_NINIT] = g;  // main_init holds -1 for slots left idle
  } else {
    st[ST_PHASE] = 1;
    st[ST_BARRIER] = (c->cfg.mode == IS_MODE_NAIVE || c->cfg.mode == IS_MODE_FULL) ? 1 : 0;
    st[ST_QUOTA] = c->cfg.mode == IS_MODE_FIFO ? c->N : 0;
    st[ST_STOPK] = 0;
    if (c->cfg.mode == IS_MODE_DYNAMIC) st[ST_TARGET] = c->cfg.dynamic_target > 0 ? c->cfg.dynamic_target : G;
    for (int s = 0; s < g; ++s) slots[s] = init[s];
    for (int i = 0; i < po.queue_len; ++i) q0[i] = queue[i];
    st[ST_QLEN] = po.queue_len;
  }
  st[ST_PROMPT_ID] = c->gprompt_id[m];
  st[ST_PROMPT_LAST] = c->gprompt_last[m];
  std::vector<int32_t> seq(G, 0);
  if (c->cfg.admit_slots > 0) {  // R41: the plan's initial fill is admitted first, in slot order
    for (int s = 0; s < c->gp; ++s)
      if (init[s] >= 0) seq[init[s]] = s;
    st[ST_ADMSEQ] = c->gp;
  }
  const size_t oG = (size_t)m * G, og = (size_t)m * g;
  CK(cudaMemcpyAsync(c->st_dev + (size_t)m * ST_COUNT, st.data(), st.size() * 8, cudaMemcpyHostToDevice, c->st));
  CK(cudaMemcpyAsync(c->slot_uid + og, slots.data(), g * 4, cudaMemcpyHostToDevice, c->st));
  CK(cudaMemsetAsync(c->slot_count + og, 0, g * 4, c->st));
  CK(cudaMemsetAsync(c->tpos + oG, 0, G * 4, c->st));
  CK(cudaMemcpyAsync(c->true_len + oG, true_len, G * 4, cudaMemcpyHostToDevice, c->st));
  CK(cudaMemcpyAsync(c->queue + oG, q0.data(), G * 4, cudaMemcpyHostToDevice, c->st));
  CK(cudaMemcpyAsync(c->main_init + og, init.data(), g * 4, cudaMemcpyHostToDevice, c->st));
  CK(cudaMemcpyAsync(c->main_queue + oG, queue.data(), G * 4, cudaMemcpyHostToDevice, c->st));
  CK(cudaMemsetAsync(c->npages + oG, 0, G * 4, c->st));
  CK(cudaMemsetAsync(c->done_flag + oG, 0, G, c->st));
  CK(cudaMemcpyAsync(c->pred + oG, pred_eff.data(), G * 4, cudaMemcpyHostToDevice, c->st));
  CK(cudaMemcpyAsync(c->adm_seq + oG, seq.data(), G * 4, cudaMemcpyHostToDevice, c->st));
  CK(cudaMemsetAsync(c->stall + og, 0, g * 4, c->st));
  CK(cudaMemsetAsync(c->tokens + oG * c->max_new, 0xFF, (size_t)G * c->max_new * 4, c->st));
  CK(cudaMemsetAsync(c->logprobs + oG * c->max_new, 0, (size_t)G * c->max_new * 4, c->st));
  CK(cudaMemsetAsync(c->log_slot + (size_t)m * c->log_cap * g, 0xFF, (size_t)c->log_cap * g * 4, c->st));
  CK(cudaMemsetAsync(c->log_live + (size_t)m * c->log_cap, 0, (size_t)c->log_cap * 4, c->st));
  // rows of the next step: allocate / log for this group only (the others are mid-step)
  CKS(launch_k(sched_kernel, dim3(1), dim3(kSchedThreads), c->st, sched_args(c), 0, 1 << m));
  CK(cudaMemcpyAsync(c->st_host, c->st_dev, sizeof(long long) * ST_COUNT * (c->M + 1), cudaMemcpyDeviceToHost, c->st));
  CK(cudaStreamSynchronize(c->st));
  if (!c->graph_ok) CKS(build_graph(c));
  c->gstarted[m] = 1;
  if (m == 0) c->started = true;
  return IS_OK;
}

extern "C" is_status is_start_group(is_ctx* c, const int32_t* true_len, const int32_t* pred) {
  return is_start_group_slot(c, 0, true_len, pred);
}

extern "C" is_status is_decode_step(is_ctx* c, int32_t* d_next, uint8_t* d_fin) {
  if (!c) return fail(IS_ERR_CONFIG, "null argument");
  if (!c->started && std::find(c->gstarted.begin(), c->gstarted.end(), 1) == c->gstarted.end())
    return fail(IS_ERR_STATE, "is_decode_step before is_start_group");
  if (c->st_host[(size_t)c->M * ST_COUNT + ST_ERROR]) return budget_error();  // (as of the last step copied back)
  StreamGuard guard(c, c->user);
  if (getenv("IS_NO_GRAPH")) CKS(enqueue_step(c));
  else CK(cudaGraphLaunch(c->graph, c->st));
  if (d_next) CK(cudaMemcpyAsync(d_next, c->last_tok, c->rc * 4, cudaMemcpyDeviceToDevice, c->st));
  if (d_fin) CK(cudaMemcpyAsync(d_fin, c->last_fin, c->rc, cudaMemcpyDeviceToDevice, c->st));
  return IS_OK;
}

extern "C" is_status is_refill(is_ctx* c, uint8_t* d_fin, int32_t* d_new_uid) {
  if (!c) return fail(IS_ERR_CONFIG, "null argument");
  if (!c->started && std::find(c->gstarted.begin(), c->gstarted.end(), 1) == c->gstarted.end())
    return fail(IS_ERR_STATE, "is_refill before is_start_group");
  StreamGuard guard(c, c->user);
  CKS(launch_k(sched_kernel, dim3(1), dim3(kSchedThreads), c->st, sched_args(c), 1, (1 << c->M) - 1));
  if (d_fin) CK(cudaMemcpyAsync(d_fin, c->last_fin, c->rc, cudaMemcpyDeviceToDevice, c->st));
  if (d_new_uid) {
    CK(cudaMemsetAsync(d_new_uid, 0xFF, c->rc * 4, c->st));
    CK(cudaMemcpyAsync(d_new_uid, c->slot_uid, (size_t)c->M * c->g * 4, cudaMemcpyDeviceToDevice, c->st));
  }
  return IS_OK;
}

// Decode steps until a started group completes (any = true) or until every
// started group has completed (any = false); bounded host run-ahead, no per-step
// synchronisation.  *h_done_mask: bit m set for every started group that is done.
static is_status run_until(is_ctx* c, int32_t max_steps, bool any, int32_t* h_done_mask) {
  constexpr int D = 3;  // bounded host run-ahead
  cudaEvent_t ev[D];
  for (int i = 0; i < D; ++i) CK(cudaEventCreateWithFlags(&ev[i], cudaEventDisableTiming));
  const bool nograph = getenv("IS_NO_GRAPH") != nullptr;
  auto done_mask = [&](const volatile long long* h) {
    int mask = 0, running = 0;
    for (int m = 0; m < c->M; ++m) {
      if (!c->gstarted[m]) continue;
      if (group_done(c, (const long long*)h + (size_t)m * ST_COUNT)) mask |= 1 << m;
      else running |= 1 << m;
    }
    return std::make_pair(mask, running);
  };
  // groups already complete when called do not end an `any` run
  const int done0 = done_mask(c->st_host).first;
  const long long* err = c->st_host + (size_t)c->M * ST_COUNT + ST_ERROR;
  is_status rs = IS_OK;
  for (int i = 0; i < max_steps; ++i) {
    if (i >= D) {
      cudaEventSynchronize(ev[i % D]);
      const auto dm = done_mask(c->st_host);
      if (dm.second == 0 || (any && (dm.first & ~done0)) || *err) break;
    }
    if (nograph) rs = enqueue_step(c);
    else if (cudaGraphLaunch(c->graphK_ok ? c->graphK : c->graph, c->st) != cudaSuccess)
      rs = fail(IS_ERR_CUDA, "graph launch failed");
    if (rs != IS_OK) break;
    cudaEventRecord(ev[i % D], c->st);
  }
  CK(cudaStreamSynchronize(c->st));
  for (int i = 0; i < D; ++i) cudaEventDestroy(ev[i]);
  if (rs != IS_OK) return rs;
  if (h_done_mask) *h_done_mask = done_mask(c->st_host).first;
  if (*err) return budget_error();
  return IS_OK;
}

extern "C" is_status is_run_group(is_ctx* c, int32_t max_steps, int32_t* h_steps) {
  if (!c) return fail(IS_ERR_CONFIG, "null argument");
  if (!c->gstarted[0]) return fail(IS_ERR_STATE, "is_run_group before is_start_group");
  StreamGuard guard(c, c->user);
  int32_t mask = 0;
  CKS(run_until(c, max_steps, false, &mask));
  if (h_steps) *h_steps = (int32_t)c->st_host[ST_STEP];
  if (!(mask & 1)) return fail(IS_ERR_CAPACITY, "group not finished after %d steps", max_steps);
  return IS_OK;
}

extern "C" is_status is_run_until_any_done(is_ctx* c, int32_t max_steps, int32_t* h_done_mask, int64_t* h_global_steps) {
  if (!c) return fail(IS_ERR_CONFIG, "null argument");
  StreamGuard guard(c, c->user);
  CKS(run_until(c, max_steps, true, h_done_mask));
  if (h_global_steps) *h_global_steps = c->st_host[(size_t)c->M * ST_COUNT + ST_GSTEP];
  return IS_OK;
}

extern "C" is_status is_query_slot(is_ctx* c, int32_t m, is_stats* o) {
  if (!c || !o) return fail(IS_ERR_CONFIG, "null argument");
  if (m < 0 || m >= c->M) return fail(IS_ERR_CONFIG, "group slot %d out of range [0, %d)", m, c->M);
  CK(cudaStreamSynchronize(c->st));
  std::vector<long long> all((size_t)ST_COUNT * (c->M + 1));
  CK(cudaMemcpy(all.data(), c->st_dev, all.size() * 8, cudaMemcpyDeviceToHost));
  const long long* st = all.data() + (size_t)m * ST_COUNT;
  const long long* g0 = all.data() + (size_t)c->M * ST_COUNT;
  o->steps = (int32_t)st[ST_STEP];
  o->prefix_steps = (int32_t)st[ST_PREFIX_STEPS];
  o->completed = (int32_t)st[ST_DONE];
  o->discarded = (int32_t)st[ST_DISCARDED];
  o->stalls = (int32_t)st[ST_STALLS];
  o->live_pages = (int32_t)st[ST_LIVE];
  o->peak_pages = (int32_t)st[ST_PEAK];
  o->error = (int32_t)g0[ST_ERROR];
  o->tokens_decoded = st[ST_TOKENS];
  o->page_bytes = c->page_bytes;
  o->prefix_bytes = c->prefix_bytes;
  o->peak_kv_bytes = c->prefix_bytes + st[ST_PEAK] * c->page_bytes;
  o->num_pages = c->num_pages;
  o->row_capacity = c->rc;
  o->suffix_tokens = st[ST_SUFFIX];
  o->groups = c->M;
  o->launches_per_step = c->launches_per_step;
  o->launches_per_prefill = c->launches_per_prefill;
  o->global_steps = g0[ST_GSTEP];
  o->global_peak_kv_bytes = (int64_t)c->M * c->prefix_bytes + g0[ST_GPEAK] * c->page_bytes;
  return IS_OK;
}

extern "C" is_status is_query(is_ctx* c, is_stats* o) { return is_query_slot(c, 0, o); }

extern "C" is_status is_copy_tokens_slot(is_ctx* c, int32_t m, int32_t* dst, int32_t dev) {
  if (!c || !dst) return fail(IS_ERR_CONFIG, "null argument");
  if (m < 0 || m >= c->M) return fail(IS_ERR_CONFIG, "group slot %d out of range [0, %d)", m, c->M);
  CK(cudaStreamSynchronize(c->st));
  CK(cudaMemcpy(dst, c->tokens + (size_t)m * c->G * c->max_new, (size_t)c->G * c->max_new * 4,
                dev ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost));
  return IS_OK;
}
extern "C" is_status is_copy_tokens(is_ctx* c, int32_t* dst, int32_t dev) { return is_copy_tokens_slot(c, 0, dst, dev); }

extern "C" is_status is_copy_schedule_slot(is_ctx* c, int32_t m, int32_t* h_slots, int32_t* h_live, int32_t max_steps,
                                           int32_t* h_n) {
  if (!c) return fail(IS_ERR_CONFIG, "null argument");
  if (m < 0 || m >= c->M) return fail(IS_ERR_CONFIG, "group slot %d out of range [0, %d)", m, c->M);
  CK(cudaStreamSynchronize(c->st));
  long long st[ST_COUNT];
  CK(cudaMemcpy(st, c->st_dev + (size_t)m * ST_COUNT, sizeof st, cudaMemcpyDeviceToHost));
  const int n = (int)std::min<long long>(std::min<long long>(st[ST_STEP], c->log_cap), max_steps);
  if (h_slots) CK(cudaMemcpy(h_slots, c->log_slot + (size_t)m * c->log_cap * c->g, (size_t)n * c->g * 4, cudaMemcpyDeviceToHost));
  if (h_live) CK(cudaMemcpy(h_live, c->log_live + (size_t)m * c->log_cap, (size_t)n * 4, cudaMemcpyDeviceToHost));
  if (h_n) *h_n = n;
  return IS_OK;
}
extern "C" is_status is_copy_schedule(is_ctx* c, int32_t* h_slots, int32_t* h_live, int32_t max_steps, int32_t* h_n) {
  return is_copy_schedule_slot(c, 0, h_slots, h_live, max_steps, h_n);
}

extern "C" is_status is_group_results_slot(is_ctx* c, int32_t m, float* d_reward, int32_t* d_len) {
  if (!c || !d_reward || !d_len) return fail(IS_ERR_CONFIG, "null argument");
  if (m < 0 || m >= c->M) return fail(IS_ERR_CONFIG, "group slot %d out of range [0, %d)", m, c->M);
  StreamGuard guard(c, c->user);
  results_kernel<<<(c->G + 127) / 128, 128, 0, c->st>>>(c->tokens + (size_t)m * c->G * c->max_new,
                                                      c->true_len + (size_t)m * c->G, c->done_flag + (size_t)m * c->G,
                                                      c->G, c->max_new, c->sh.vocab, d_reward, d_len);
  CK(cudaGetLastError());
  return IS_OK;
}
extern "C" is_status is_group_results(is_ctx* c, float* d_reward, int32_t* d_len) {
  return is_group_results_slot(c, 0, d_reward, d_len);
}

extern "C" is_status is_set_logits_dump(is_ctx* c, float* d_logits) {
  if (!c) return fail(IS_ERR_CONFIG, "null argument");
  c->logits_dump = d_logits;
  if (c->graph_ok) CKS(build_graph(c));
  return IS_OK;
}

static is_status profile_step(is_ctx* c, bool graph, float* h_ms, int32_t* h_kind, int32_t cap, int32_t* h_n) {
  if (!c) return fail(IS_ERR_CONFIG, "null argument");
  if (std::find(c->gstarted.begin(), c->gstarted.end(), 1) == c->gstarted.end())
    return fail(IS_ERR_STATE, "is_profile_step before is_start_group");
  StreamGuard guard(c, c->user);
  std::vector<cudaEvent_t> ev;
  std::vector<int> kind;
  Prof p{&ev, &kind, graph};
  cudaEvent_t e0;
  CK(cudaEventCreate(&e0));
  is_status s = IS_OK;
  if (graph) {
    // the step captured exactly as build_graph does, plus an event node after every
    // launch; one replay.  (An event node between two kernels turns their PDL edge into
    // a full dependency, so each interval is the kernel plus one graph-node hop.)
    cudaGraph_t g;
    cudaGraphExec_t ge;
    CK(cudaStreamBeginCapture(c->st, cudaStreamCaptureModeThreadLocal));
    cudaEventRecordWithFlags(e0, c->st, cudaEventRecordExternal);
    g_prof = &p;
    s = enqueue_step(c);
    g_prof = nullptr;
    cudaError_t e = cudaStreamEndCapture(c->st, &g);
    if (s != IS_OK) return s;
    CK(e);
    CK(cudaGraphInstantiate(&ge, g, 0));
    cudaGraphDestroy(g);
    CK(cudaGraphUpload(ge, c->st));
    CK(cudaStreamSynchronize(c->st));
    CK(cudaGraphLaunch(ge, c->st));
    CK(cudaStreamSynchronize(c->st));
    cudaGraphExecDestroy(ge);
  } else {
    CK(cudaEventRecord(e0, c->st));
    g_prof = &p;
    s = enqueue_step(c);
    g_prof = nullptr;
    CK(cudaStreamSynchronize(c->st));
  }
  int n = 0;
  cudaEvent_t prev = e0;
  for (size_t i = 0; i < ev.size(); ++i) {
    float ms = 0;
    cudaEventElapsedTime(&ms, prev, ev[i]);
    if (n < cap) {
      h_ms[n] = ms;
      h_kind[n] = kind[i];
      ++n;
    }
    prev = ev[i];
  }
  for (auto e : ev) cudaEventDestroy(e);
  cudaEventDestroy(e0);
  if (h_n) *h_n = n;
  return s;
}

// Average device duration of one decode-step GEMM kind as the step issues it
// (same arguments, tensor maps, split, stages, PDL), all layers' launches of that
// kind back to back in one CUDA graph, `reps` passes over the layers, CUDA events
// on the context stream around the replay.  kind: 1 QKV, 4 o_proj, 5 gate/up, 6 down.
extern "C" is_status is_profile_kernel(is_ctx* c, int32_t kind, int32_t reps, float* h_ms_per_launch,
                                       int32_t* h_launches) {
  if (!c || !h_ms_per_launch) return fail(IS_ERR_CONFIG, "null argument");
  int keep;
  switch (kind) {
    case 1: keep = 2; break;
    case 3: keep = 8; break;  // attention: the layer's prefix + suffix launches
    case 4: keep = 16; break;
    case 5: keep = 32; break;
    case 6: keep = 64; break;
    default: return fail(IS_ERR_CONFIG, "is_profile_kernel: kind %d is not a GEMM or attention kind", kind);
  }
  if (reps < 1) return fail(IS_ERR_CONFIG, "reps must be >= 1");
  StreamGuard guard(c, c->user);
  const int skip0 = g_skip;
  g_skip = (1 | 2 | 8 | 16 | 32 | 64 | 128) & ~keep;
  cudaGraph_t g;
  cudaGraphExec_t ge;
  const int launches0 = g_launches;
  cudaError_t e = cudaStreamBeginCapture(c->st, cudaStreamCaptureModeThreadLocal);
  is_status s = IS_OK;
  for (int r = 0; r < reps && s == IS_OK && e == cudaSuccess; ++r) s = run_layers(c, c->rc, false);
  if (e == cudaSuccess) e = cudaStreamEndCapture(c->st, &g);
  g_skip = skip0;
  const int n = g_launches - launches0;
  g_launches = launches0;
  if (s != IS_OK) return s;
  CK(e);
  CK(cudaGraphInstantiate(&ge, g, 0));
  cudaGraphDestroy(g);
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  CK(cudaGraphLaunch(ge, c->st));  // warm-up (instruction cache, TLB)
  CK(cudaEventRecord(e0, c->st));
  CK(cudaGraphLaunch(ge, c->st));
  CK(cudaEventRecord(e1, c->st));
  CK(cudaStreamSynchronize(c->st));
  float ms = 0;
  CK(cudaEventElapsedTime(&ms, e0, e1));
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaGraphExecDestroy(ge);
  *h_ms_per_launch = ms / (reps * c->sh.layers);  // per layer (kind 3: all of the layer's attention launches)
  if (h_launches) *h_launches = n;
  return IS_OK;
}

extern "C" is_status is_profile_step(is_ctx* c, float* h_ms, int32_t* h_kind, int32_t cap, int32_t* h_n) {
  return profile_step(c, false, h_ms, h_kind, cap, h_n);
}

extern "C" is_status is_profile_step_graph(is_ctx* c, float* h_ms, int32_t* h_kind, int32_t cap, int32_t* h_n) {
  return profile_step(c, true, h_ms, h_kind, cap, h_n);
}

extern "C" is_status is_dbg_gemm(const void* d_w, const void* d_x, float* d_y, int32_t M, int32_t K, int32_t rows,
                                 int32_t split, void* stream) {
  if (rows < 1 || rows > 64 || K % 64 || M % 4 || split < 1 || split > 8) return fail(IS_ERR_CONFIG, "bad dbg_gemm shape");
  if (!g_num_sms) {  // (cudaGetDeviceProperties costs milliseconds: once)
    int dev = 0;
    CK(cudaGetDevice(&dev));
    CK(cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev));
  }
  const int BN = rows <= 16 ? 16 : (rows <= 32 ? 32 : 64);
  CUtensorMap tA, tB;
  CKS(make_tmap(&tA, d_w, M, K, kBM));
  CKS(make_tmap(&tB, d_x, rows, K, BN));
  GemmArgs a{};
  a.M = M;
  a.K = K;
  a.num_tiles = (M + kBM - 1) / kBM;
  a.split = split;
  a.row0 = 0;
  a.n_valid = rows;
  a.out = d_y;
  a.ld_out = M;
  static float* ws = nullptr;
  if (!ws) CK(cudaMalloc(&ws, (size_t)2 * 160 * kBM * 64 * 4));
  a.partials = ws;
  a.dbg_ts = getenv("IS_GEMM_STAMPS") ? reinterpret_cast<unsigned long long*>(strtoull(getenv("IS_GEMM_STAMPS"), nullptr, 0)) : nullptr;
  CKS(launch_gemm<EPI_STORE_F32>(BN, tA, tB, a, (cudaStream_t)stream));
  CK(cudaGetLastError());
  return IS_OK;
}

// Kernel-level hook of the decode split attention (R8):
// the work list and the attention launches of one decode layer, exactly as the step issues
// them (launch_attention), on caller data.  See include/infsamp.h.
extern "C" is_status is_dbg_attn(const void* d_q, const void* d_prefix, int32_t plen, int32_t groups,
                                 int32_t grp_rows, const void* d_pool, int32_t num_pages, int32_t page_tokens,
                                 const int32_t* d_pagetab, int32_t maxp, const int32_t* d_row_len, int32_t rows,
                                 int32_t Hq, int32_t Hkv, int32_t impl, void* d_out, float* d_out_f32,
                                 int32_t reps, float* h_ms, void* stream) {
  if (!d_q || !d_prefix || !d_pool || !d_pagetab || !d_row_len || !d_out) return fail(IS_ERR_CONFIG, "null argument");
  if (rows < 1 || rows > 64 || groups < 1 || grp_rows < 1 || groups * grp_rows > rows || plen < 1 || Hkv < 1 ||
      Hq % Hkv || Hq / Hkv > kMaxRep || page_tokens < 4 || 64 % page_tokens || maxp < 1 || num_pages < 1 ||
      impl < 0 || impl > 6 || reps < 0 || (reps > 0 && !h_ms))
    return fail(IS_ERR_CONFIG, "bad is_dbg_attn arguments");
  if (!g_num_sms) {
    int dev = 0;
    CK(cudaGetDevice(&dev));
    CK(cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev));
  }
  const int rep = Hq / Hkv;
  // impl 5 / 6: as 0 / 4 with the query-rows-as-M prefix kernel forced (0 / 4 take it only beyond 64
  // stacked rows, as the decode step does)
  const bool force2 = impl == 5 || impl == 6 || (getenv("IS_PREFIX_IMPL") && atoi(getenv("IS_PREFIX_IMPL")) == 2);
  if (impl == 5) impl = 0;
  if (impl == 6) impl = 4;
  const bool old_prefix = !force2 && prefix_cols(grp_rows, rep) <= 64;
  const bool tc_ok = grp_rows * rep <= 256;
  const bool tc = impl == 0 ? tc_ok : impl != 3;
  const bool mma = impl == 0 ? tc_ok && page_tokens % 8 == 0 && page_tokens <= kSUnit : impl == 4;
  const bool sep = impl == 2 || impl == 3 || (impl == 0 && !mma && (!tc || page_tokens > kSCW));
  if (tc && !tc_ok) return fail(IS_ERR_CONFIG, "tcgen05 prefix needs grp_rows * Hq/Hkv <= 256 (64: impl 5/6)");
  if (mma && (page_tokens % 8 || page_tokens > kSUnit))
    return fail(IS_ERR_CONFIG, "the mma suffix pass needs page_tokens in {8, 16, 32}");
  if (!tc && groups != 1) return fail(IS_ERR_CONFIG, "the CUDA-core prefix serves one group");
  const int sc = mma ? kSUnit : ((tc && !sep) ? kSCW : kSC);
  const int nc_pre = tc ? (int)ceil_div64(plen, 128) : (int)ceil_div64(plen, kPC);
  const int nc_suf = (int)ceil_div64((int64_t)maxp * page_tokens, sc);
  const int nmax = sep ? 32 : 64;
  if (nc_pre + nc_suf > nmax) return fail(IS_ERR_CAPACITY, "%d partials exceed the merge (%d)", nc_pre + nc_suf, nmax);
  cudaStream_t st = (cudaStream_t)stream;
  std::vector<int32_t> len(rows), act(rows), lid(rows);
  CK(cudaMemcpy(len.data(), d_row_len, rows * 4, cudaMemcpyDeviceToHost));
  for (int r = 0; r < rows; ++r) {
    if (len[r] < 0 || len[r] > maxp * page_tokens) return fail(IS_ERR_DATA, "row %d length %d", r, len[r]);
    act[r] = len[r] > 0 && r < groups * grp_rows;
    lid[r] = r;
  }
  const int NC = nc_pre + nc_suf;
  is_status err = IS_OK;
  int32_t* d_act = (int32_t*)dalloc((size_t)rows * 4, &err);
  int32_t* d_lid = (int32_t*)dalloc((size_t)rows * 4, &err);
  int32_t* items = (int32_t*)dalloc((size_t)Hkv * (nc_pre * ((rows + 3) / 4) + rows * nc_suf) * kItemStride * 4 + 64, &err);
  long long* nit = (long long*)dalloc(2 * sizeof(long long), &err);
  float* part_o = (float*)dalloc((size_t)rows * Hq * NC * 128 * 4, &err);
  float* part_ml = (float*)dalloc((size_t)rows * Hq * NC * 2 * 4, &err);
  int* mcnt = (int*)dalloc(((size_t)2 * rows * Hkv + 2) * 4, &err);
  const int ntp = (int)ceil_div64(plen, 128);
  float* kmx = (float*)dalloc((size_t)groups * Hkv * ntp * 4, &err);
  uint8_t* flush = reps > 0 ? (uint8_t*)dalloc((size_t)256 << 20, &err) : nullptr;  // > 2x the 126 MB L2
  CUtensorMap tm, tmp;
  if (err == IS_OK) err = make_tmap(&tm, d_prefix, (int64_t)groups * 2 * Hkv * plen, 128, 128);
  if (err == IS_OK && mma) err = make_tmap_pool(&tmp, d_pool, num_pages, Hkv, page_tokens);
  if (err == IS_OK) {
    cudaMemcpy(d_act, act.data(), rows * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(d_lid, lid.data(), rows * 4, cudaMemcpyHostToDevice);
    WorkList wl;
    wl.row_cap = rows;
    wl.chunk = sc;
    wl.pt = page_tokens;
    wl.Hkv = Hkv;
    wl.nc_pre = nc_pre;
    wl.tc_prefix = tc ? 1 : 0;
    wl.maxp = maxp;
    wl.row_active = d_act;
    wl.row_len = d_row_len;
    wl.row_lid = d_lid;
    wl.pagetab = d_pagetab;
    wl.items = items;
    wl.n_items = nit;
    attn_worklist_kernel<<<1, kSchedThreads, 0, st>>>(wl);
    prefix_kmax_kernel<<<groups * Hkv * ntp, 128, 0, st>>>((const __nv_bfloat16*)d_prefix, 1, Hkv, plen, plen, kmx);
    AttnArgs aa{};
    aa.q = (const __nv_bfloat16*)d_q;
    aa.kpre = (const __nv_bfloat16*)d_prefix;
    aa.vpre = aa.kpre + (size_t)Hkv * plen * kHD;
    aa.pool = (const __nv_bfloat16*)d_pool;
    aa.row_active = d_act;
    aa.row_len = d_row_len;
    aa.part_o = part_o;
    aa.part_ml = part_ml;
    aa.items = items;
    aa.n_items = nit;
    aa.out = (__nv_bfloat16*)d_out;
    aa.out_f32 = d_out_f32;
    aa.rows = rows;
    aa.Hq = Hq;
    aa.Hkv = Hkv;
    aa.pcap = plen;
    aa.plen = plen;
    aa.pt = page_tokens;
    aa.nc_pre = nc_pre;
    aa.nc_suf = nc_suf;
    aa.NC = NC;
    aa.prefill = 0;
    aa.tc_prefix = tc ? 1 : 0;
    aa.merge_cnt = (tc && !sep) ? mcnt : nullptr;
    aa.unit_ctr = getenv("IS_STATIC_UNITS") ? nullptr : mcnt + (size_t)rows * Hkv;
    aa.merge_done = mcnt + (size_t)rows * Hkv + 2;
    aa.kmax = getenv("IS_EXACT_PREFIX_MAX") ? nullptr : kmx;
    aa.kmax_grp = Hkv * ntp;
    aa.sc = sc;
    aa.scale = 1.0f / sqrtf((float)kHD);
    AttnLaunch al{};
    al.tm_prefix = &tm;
    al.kv_row_base = 0;
    al.grp_kv_rows = 2 * Hkv * plen;
    al.groups = groups;
    al.grp_rows = grp_rows;
    al.tm_pool = &tmp;
    al.suffix_mma = mma ? 1 : 0;
    al.suffix_shape = getenv("IS_SUFFIX_SHAPE") ? atoi(getenv("IS_SUFFIX_SHAPE")) : 1;
    al.carveout = getenv("IS_ATTN_CARVEOUT") ? atoi(getenv("IS_ATTN_CARVEOUT")) : (rows > 16 ? 100 : -1);
    al.prefix2 = old_prefix ? 0 : 1;
    aa.pool_row0 = 0;
    aa.dbg_mode = getenv("IS_DBG_SUFFIX_MODE") ? atoi(getenv("IS_DBG_SUFFIX_MODE")) : 0;
    err = launch_attention(aa, al, st);
    if (err == IS_OK && reps > 0) {
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      for (int i = 0; i < reps && err == IS_OK; ++i) {
        cudaMemsetAsync(flush, i & 0xFF, (size_t)256 << 20, st);  // evict the KV from L2
        cudaEventRecord(e0, st);
        err = launch_attention(aa, al, st);
        cudaEventRecord(e1, st);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&h_ms[i], e0, e1);
      }
      cudaEventDestroy(e0);
      cudaEventDestroy(e1);
    }
    if (err == IS_OK) {
      cudaError_t e = cudaStreamSynchronize(st);
      if (e == cudaSuccess) e = cudaGetLastError();
      if (e != cudaSuccess) err = fail(IS_ERR_CUDA, "is_dbg_attn: %s", cudaGetErrorString(e));
    }
    if (err == IS_OK && getenv("IS_DBG_STAMPS")) {
      // one more run with globaltimer stamps of the suffix CTAs (timing experiments only)
      unsigned long long* ts = nullptr;
      cudaMalloc(&ts, (size_t)4 * 296 * 16 * 8);
      cudaMemset(ts, 0, (size_t)4 * 296 * 16 * 8);
      AttnArgs a3 = aa;
      a3.dbg_ts = ts;
      cudaMemsetAsync(flush, 1, (size_t)256 << 20, st);
      err = launch_attention(a3, al, st);
      cudaStreamSynchronize(st);
      std::vector<unsigned long long> h((size_t)4 * 296 * 16);
      cudaMemcpy(h.data(), ts, h.size() * 8, cudaMemcpyDeviceToHost);
      cudaFree(ts);
      unsigned long long t0 = ~0ull;
      for (int b = 0; b < g_num_sms; ++b)
        if (h[b * 16]) t0 = std::min(t0, h[b * 16]);
      for (int b = 0; b < 296; ++b)  // (and the prefix kernel's CTAs)
        if (h[(size_t)2 * 296 * 16 + b * 16]) t0 = std::min(t0, h[(size_t)2 * 296 * 16 + b * 16]);
      for (int i = 0; i < 9; ++i) {
        std::vector<double> v;
        for (int b = 0; b < g_num_sms; ++b)
          if (h[b * 16 + i]) v.push_back((double)(h[b * 16 + i] - t0) / 1e3);
        if (v.empty()) continue;
        std::sort(v.begin(), v.end());
        fprintf(stderr, "stamp %d: n=%zu min %.2f med %.2f max %.2f us\n", i, v.size(), v[0], v[v.size() / 2], v.back());
      }
      std::vector<double> u, m;
      for (int b = 0; b < g_num_sms; ++b) {
        u.push_back((double)h[b * 16 + 9]);
        m.push_back((double)h[b * 16 + 10]);
      }
      std::sort(u.begin(), u.end());
      std::sort(m.begin(), m.end());
      {  // the tcgen05 prefix kernel's CTAs (stamps 0 start, 1 waited, 2 q staged, 3 K/V landed, 4 S done,
         // 5 P stored, 6 O done, 7 end)
        const unsigned long long* pb = h.data() + (size_t)2 * 296 * 16;
        for (int i = 0; i < 8; ++i) {
          std::vector<double> v;
          for (int b = 0; b < 296; ++b)
            if (pb[b * 16] && pb[b * 16 + i]) v.push_back((double)((long long)(pb[b * 16 + i] - t0)) / 1e3);
          if (v.empty()) continue;
          std::sort(v.begin(), v.end());
          fprintf(stderr, "prefix stamp %d: n=%zu min %.2f med %.2f max %.2f us\n", i, v.size(), v[0], v[v.size() / 2],
                  v.back());
        }
      }
      fprintf(stderr, "slots per CTA min %.0f med %.0f max %.0f; merges per CTA min %.0f med %.0f max %.0f\n", u[0],
              u[u.size() / 2], u.back(), m[0], m[m.size() / 2], m.back());
    }
  }
  for (void* p : {(void*)d_act, (void*)d_lid, (void*)items, (void*)nit, (void*)part_o, (void*)part_ml, (void*)mcnt, (void*)kmx,
                  (void*)flush})
    if (p) cudaFree(p);
  return err;
}

// Debug: print the GEMM timeline of the last replayed step (IS_TIMELINE=1).
extern "C" int is_dbg_timeline(is_ctx* c) {
  if (!c || !c->timeline) return 0;
  cudaStreamSynchronize(c->st);
  std::vector<unsigned long long> h0((size_t)512 * 296 * 16);
  cudaMemcpy(h0.data(), c->timeline, h0.size() * 8, cudaMemcpyDeviceToHost);
  std::vector<unsigned long long> h(h0.begin(), h0.begin() + (size_t)c->tl_count * 296 * 16);
  unsigned long long t0 = ~0ull;
  for (size_t i = 0; i < h.size(); i += 16)
    if (h[i] && h[i] < t0) t0 = h[i];
  for (int L = 0; L < c->tl_count; ++L) {
    unsigned long long mn[16], mx[16];
    for (int k = 0; k < 16; ++k) { mn[k] = ~0ull; mx[k] = 0; }
    int n = 0;
    for (int b = 0; b < 296; ++b) {
      const unsigned long long* p = &h[((size_t)L * 296 + b) * 16];
      if (!p[0]) continue;
      ++n;
      for (int k = 0; k < 16; ++k)
        if (p[k]) { mn[k] = std::min(mn[k], p[k]); mx[k] = std::max(mx[k], p[k]); }
    }
    auto f = [&](unsigned long long v) { return v == ~0ull || v == 0 ? -1.0 : (double)(v - t0) / 1000.0; };
    // per-CTA phase durations (median / max, us)
    auto dur = [&](int k0, int k1, double* med, double* mxx) {
      std::vector<double> d;
      for (int b = 0; b < 296; ++b) {
        const unsigned long long* p = &h[((size_t)L * 296 + b) * 16];
        if (p[0] && p[k0] && p[k1]) d.push_back((double)((long long)(p[k1] - p[k0])) / 1000.0);
      }
      if (d.empty()) { *med = *mxx = -1; return; }
      std::sort(d.begin(), d.end());
      *med = d[d.size() / 2];
      *mxx = d.back();
    };
    double m56, x56, m67, x67, m78, x78, m8a, x8a;
    dur(5, 6, &m56, &x56);
    dur(6, 7, &m67, &x67);
    dur(7, 8, &m78, &x78);
    dur(8, 10, &m8a, &x8a);
    printf("      per-CTA us: tfull->cbar %.2f/%.2f  cbar->pulled %.2f/%.2f  pulled->epi0 %.2f/%.2f  epi %.2f/%.2f\n", m56,
           x56, m67, x67, m78, x78, m8a, x8a);
    printf("%3d %-5s ctas=%3d start %7.2f..%7.2f pre %7.2f data0 %7.2f..%7.2f mma_done %7.2f..%7.2f cbar %7.2f pulled %7.2f epi %7.2f..%7.2f exit %7.2f..%7.2f\n", L,
           g_tl_name[L], n, f(mn[0]), f(mx[0]), f(mx[2]), f(mn[3]), f(mx[3]), f(mn[5]), f(mx[5]), f(mx[6]), f(mx[7]),
           f(mn[10]), f(mx[10]), f(mn[11]), f(mx[11]));
  }
  for (int l = 0; l < 4; ++l) {
    // the mma suffix kernel's CTAs: 0 start, 3 units begin, 2 warp 0's units done, 6 all units
    // published, 7 prefix complete (PDL wait), 8 merges done
    const unsigned long long* base = &h0[(size_t)(400 + 4 * l) * 296 * 16];
    printf("suffix L%d", l);
    const int ks[6] = {0, 3, 2, 6, 7, 8};
    for (int q = 0; q < 6; ++q) {
      std::vector<double> v;
      for (int b = 0; b < 296; ++b)
        if (base[b * 16] && base[b * 16 + ks[q]]) v.push_back((double)(base[b * 16 + ks[q]] - t0) / 1e3);
      if (v.empty()) continue;
      std::sort(v.begin(), v.end());
      printf("  s%d n=%zu %.2f/%.2f/%.2f", ks[q], v.size(), v[0], v[v.size() / 2], v.back());
    }
    printf("\n");
  }
  for (int l = 0; l < 2; ++l) {
    const unsigned long long* base = &h0[((size_t)(400 + 4 * l) * 296 + 2 * 296) * 16];
    double mx[8] = {0}, mn0 = 1e30;
    int n = 0;
    for (int b = 0; b < 64; ++b) {
      const unsigned long long* p = base + b * 16;
      if (!p[0]) continue;
      ++n;
      mn0 = std::min(mn0, (double)(p[0] - t0) / 1e3);
      for (int k = 0; k < 8; ++k)
        if (p[k]) mx[k] = std::max(mx[k], (double)(p[k] - t0) / 1e3);
    }
    double mx8 = 0;
    for (int b = 0; b < 64; ++b)
      if (base[b * 16] && base[b * 16 + 8]) mx8 = std::max(mx8, (double)(base[b * 16 + 8] - t0) / 1e3);
    printf("prefix_tc L%d ctas=%d start %.2f waited %.2f q_staged %.2f tma %.2f S_done %.2f [softmax pass 0 done %.2f] P_done %.2f O_done %.2f end %.2f\n", l, n,
           mn0, mx[1], mx[2], mx[3], mx[4], mx8, mx[5], mx[6], mx[7]);
    printf("      fine:");
    for (int k = 9; k <= 15; ++k) {
      double v = 0;
      for (int b = 0; b < 64; ++b)
        if (base[b * 16] && base[b * 16 + k]) v = std::max(v, (double)(base[b * 16 + k] - t0) / 1e3);
      printf(" s%d %.2f", k, v);
    }
    printf("\n");
    // per-CTA phase durations (median / max, us): wait->q, q->S, S->P (softmax), P->O, O->end
    const char* nm[5] = {"q_stage", "S_mma", "softmax", "PV_mma", "epilogue"};
    const int k0[5] = {1, 2, 4, 5, 6}, k1[5] = {2, 4, 5, 6, 7};
    printf("      per-CTA:");
    for (int ph = 0; ph < 5; ++ph) {
      std::vector<double> d;
      for (int b = 0; b < 64; ++b) {
        const unsigned long long* p = base + b * 16;
        if (p[0] && p[k0[ph]] && p[k1[ph]]) d.push_back((double)((long long)(p[k1[ph]] - p[k0[ph]])) / 1e3);
      }
      if (d.empty()) continue;
      std::sort(d.begin(), d.end());
      printf(" %s %.2f/%.2f", nm[ph], d[d.size() / 2], d.back());
    }
    printf("\n");
  }
  fflush(stdout);
  return c->tl_count;
}

extern "C" is_status is_dbg_copy(is_ctx* c, int32_t which, void* h_dst, int64_t bytes) {
  if (!c || !h_dst) return fail(IS_ERR_CONFIG, "null argument");
  CK(cudaStreamSynchronize(c->st));
  const is_shape& s = c->sh;
  const void* src = nullptr;
  int64_t n = 0;
  switch (which) {
    case 0: src = c->q; n = (int64_t)c->rc * s.n_q_heads * 128 * 2; break;
    case 1: src = c->resid; n = (int64_t)c->rc * s.hidden * 4; break;
    case 3: src = c->xn; n = (int64_t)c->rc * s.hidden * 2; break;
    case 4: src = c->attn; n = (int64_t)c->rc * s.n_q_heads * 128 * 2; break;
    case 6: src = c->act; n = (int64_t)c->rc * s.ffn * 2; break;
    default: return fail(IS_ERR_CONFIG, "unknown buffer %d", which);
  }
  if (!src) return fail(IS_ERR_STATE, "buffer %d not in use", which);
  if (bytes < n) return fail(IS_ERR_CAPACITY, "need %lld bytes", (long long)n);
  CK(cudaMemcpy(h_dst, src, (size_t)n, cudaMemcpyDeviceToHost));
  return IS_OK;
}

// ------------------------------------------------------------------ NCCL (a9: the one exchange)
// NCCL is bound at run time (dlopen / dlsym of libnccl.so.2): the process's NCCL
// (torch's bundled one when torch is loaded) is used, and the library has no
// link-time NCCL dependency.  Types mirror nccl.h.
namespace {
struct NcclUid { char internal[128]; };
typedef void* NcclComm;
typedef int (*PfnGetUid)(NcclUid*);
typedef int (*PfnInitRank)(NcclComm*, int, NcclUid, int);
typedef int (*PfnAllGather)(const void*, void*, size_t, int, NcclComm, cudaStream_t);
typedef int (*PfnGroup)();
typedef int (*PfnDestroy)(NcclComm);
typedef const char* (*PfnErr)(int);
struct NcclApi {
  PfnGetUid get_uid = nullptr;
  PfnInitRank init_rank = nullptr;
  PfnAllGather all_gather = nullptr;
  PfnGroup group_start = nullptr, group_end = nullptr;
  PfnDestroy destroy = nullptr;
  PfnErr err = nullptr;
  bool ok = false;
};
NcclApi& nccl() {
  static NcclApi api;
  static bool tried = false;
  if (!tried) {
    tried = true;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (h) {
      api.get_uid = (PfnGetUid)dlsym(h, "ncclGetUniqueId");
      api.init_rank = (PfnInitRank)dlsym(h, "ncclCommInitRank");
      api.all_gather = (PfnAllGather)dlsym(h, "ncclAllGather");
      api.group_start = (PfnGroup)dlsym(h, "ncclGroupStart");
      api.group_end = (PfnGroup)dlsym(h, "ncclGroupEnd");
      api.destroy = (PfnDestroy)dlsym(h, "ncclCommDestroy");
      api.err = (PfnErr)dlsym(h, "ncclGetErrorString");
      api.ok = api.get_uid && api.init_rank && api.all_gather && api.group_start && api.group_end && api.destroy;
    }
  }
  return api;
}
constexpr int kNcclInt32 = 2, kNcclFloat32 = 7;
}  // namespace

#define NCK(x)                                                                                      \
  do {                                                                                              \
    int r_ = (x);                                                                                   \
    if (r_ != 0) return fail(IS_ERR_CUDA, "NCCL error %d (%s) in %s", r_,                            \
                             nccl().err ? nccl().err(r_) : "?", #x);                                \
  } while (0)

extern "C" is_status is_nccl_unique_id(void* h_uid) {
  if (!h_uid) return fail(IS_ERR_CONFIG, "null argument");
  if (!nccl().ok) return fail(IS_ERR_CUDA, "libnccl.so.2 not available");
  NcclUid u;
  NCK(nccl().get_uid(&u));
  memcpy(h_uid, &u, sizeof u);
  return IS_OK;
}

extern "C" is_status is_nccl_comm_init(const void* h_uid, int32_t rank, int32_t world, void** comm_out) {
  if (!h_uid || !comm_out || world < 1 || rank < 0 || rank >= world) return fail(IS_ERR_CONFIG, "bad arguments");
  if (!nccl().ok) return fail(IS_ERR_CUDA, "libnccl.so.2 not available");
  NcclUid u;
  memcpy(&u, h_uid, sizeof u);
  NcclComm comm = nullptr;
  NCK(nccl().init_rank(&comm, world, u, rank));
  *comm_out = comm;
  return IS_OK;
}

extern "C" is_status is_nccl_comm_destroy(void* comm) {
  if (!comm) return fail(IS_ERR_CONFIG, "null argument");
  if (!nccl().ok) return fail(IS_ERR_CUDA, "libnccl.so.2 not available");
  NCK(nccl().destroy(comm));
  return IS_OK;
}

extern "C" is_status is_allgather_results_n(is_ctx* c, void* comm, int32_t n, const int32_t* d_len,
                                            const float* d_reward, int32_t* d_all_len, float* d_all_reward) {
  if (!c || !comm || !d_len || !d_reward || !d_all_len || !d_all_reward || n < 1)
    return fail(IS_ERR_CONFIG, "null argument or n < 1");
  if (!nccl().ok) return fail(IS_ERR_CUDA, "libnccl.so.2 not available");
  StreamGuard guard(c, c->user);
  NCK(nccl().group_start());
  NCK(nccl().all_gather(d_len, d_all_len, (size_t)n, kNcclInt32, comm, c->st));
  NCK(nccl().all_gather(d_reward, d_all_reward, (size_t)n, kNcclFloat32, comm, c->st));
  NCK(nccl().group_end());
  return IS_OK;
}

extern "C" is_status is_allgather_results(is_ctx* c, void* comm, const int32_t* d_len, const float* d_reward,
                                          int32_t* d_all_len, float* d_all_reward) {
  if (!c) return fail(IS_ERR_CONFIG, "null argument");
  return is_allgather_results_n(c, comm, c->G, d_len, d_reward, d_all_len, d_all_reward);
}

extern "C" is_status is_copy_logprobs_slot(is_ctx* c, int32_t m, float* h_dst) {
  if (!c || !h_dst) return fail(IS_ERR_CONFIG, "null argument");
  if (m < 0 || m >= c->M) return fail(IS_ERR_CONFIG, "group slot %d out of range [0, %d)", m, c->M);
  CK(cudaStreamSynchronize(c->st));
  CK(cudaMemcpy(h_dst, c->logprobs + (size_t)m * c->G * c->max_new, (size_t)c->G * c->max_new * 4,
                cudaMemcpyDeviceToHost));
  return IS_OK;
}
extern "C" is_status is_copy_logprobs(is_ctx* c, float* h_dst) { return is_copy_logprobs_slot(c, 0, h_dst); }

// ------------------------------------------------------------------ NEXT-3: KL-penalised reward, objective value
extern "C" is_status is_kl_rewards(const float* rm, const float* logp, const float* logp_ref, const int32_t* len,
                                   int32_t G, int32_t max_new, float beta, float* out) {
  if (!rm || !logp || !logp_ref || !len || !out || G < 1 || max_new < 1) return fail(IS_ERR_CONFIG, "bad arguments");
  for (int i = 0; i < G; ++i) {
    if (len[i] < 1 || len[i] > max_new) return fail(IS_ERR_DATA, "length of sample %d is %d", i, len[i]);
    double s = 0;
    for (int t = 0; t < len[i]; ++t) s += (double)logp[(size_t)i * max_new + t] - (double)logp_ref[(size_t)i * max_new + t];
    out[i] = (float)((double)rm[i] - (double)beta * s);
  }
  return IS_OK;
}

extern "C" is_status is_grpo_objective(const float* logp, const float* logp_old, const float* logp_ref, const float* adv,
                                       const int32_t* len, int32_t G, int32_t max_new, float clip_eps, float beta,
                                       double* out) {
  if (!logp || !logp_old || !logp_ref || !adv || !len || !out || G < 1 || max_new < 1)
    return fail(IS_ERR_CONFIG, "bad arguments");
  double total = 0;
  for (int i = 0; i < G; ++i) {
    if (len[i] < 1 || len[i] > max_new) return fail(IS_ERR_DATA, "length of sample %d is %d", i, len[i]);
    double s = 0;
    for (int t = 0; t < len[i]; ++t) {
      const size_t k = (size_t)i * max_new + t;
      const double lam = std::exp((double)logp[k] - (double)logp_old[k]), a = adv[i];
      const double clipped = std::min(std::max(lam, 1.0 - clip_eps), 1.0 + (double)clip_eps);
      const double surr = std::min(lam * a, clipped * a);
      const double d = (double)logp_ref[k] - (double)logp[k];
      s += surr - (double)beta * (std::exp(d) - d - 1.0);
    }
    total += s / len[i];
  }
  *out = total / G;
  return IS_OK;
}

// ------------------------------------------------------------------ top-p test hook (R36)
extern "C" is_status is_dbg_topp(const float* d_logits, int32_t rows, int32_t V, float temperature, float top_p,
                                 uint64_t seed, const int32_t* d_uid, const int32_t* d_t, int32_t* d_tok, void* stream) {
  if (!d_logits || !d_uid || !d_t || !d_tok || rows < 1 || V < 4 || V % 4 || !(temperature > 0) ||
      !(top_p > 0.f && top_p < 1.f))
    return fail(IS_ERR_CONFIG, "bad is_dbg_topp arguments");
  cudaStream_t st = (cudaStream_t)stream;
  is_status err = IS_OK;
  float *scores = (float*)dalloc((size_t)rows * V * 4, &err);
  float4* mlz = (float4*)dalloc((size_t)rows * 16, &err);
  uint32_t* ebits = (uint32_t*)dalloc((size_t)rows * V * 4, &err);
  unsigned long long* wpart = (unsigned long long*)dalloc((size_t)rows * kToppBlocks * 8, &err);
  unsigned long long* hist = (unsigned long long*)dalloc((size_t)rows * kToppBlocks * 256 * 8, &err);
  int2* sel = (int2*)dalloc((size_t)rows * 8, &err);
  ToppState* ts = (ToppState*)dalloc((size_t)rows * sizeof(ToppState), &err);
  int32_t* active = (int32_t*)dalloc((size_t)rows * 4, &err);
  unsigned long long* keys = (unsigned long long*)dalloc((size_t)rows * 8, &err);
  if (err == IS_OK) {
    std::vector<int32_t> ones(rows, 1);
    cudaMemcpy(active, ones.data(), rows * 4, cudaMemcpyHostToDevice);
    const float invT = (float)(1.0 / (double)temperature);
    topp_dbg_scores_kernel<<<rows, kToppThreads, 0, st>>>(d_logits, V, d_uid, d_t, seed, invT, scores, mlz);
    ToppArgs t{};
    t.scores = scores;
    t.logits = d_logits;
    t.lp_mlz = mlz;
    t.lp_grid = 1;
    t.ebits = ebits;
    t.wpart = wpart;
    t.hist1 = hist;
    t.sel = sel;
    t.row_active = active;
    t.keys = keys;
    t.V = V;
    t.invT = invT;
    t.top_p = top_p;
    topp_prep_kernel<<<dim3(kToppBlocks, rows), kToppThreads, 0, st>>>(t);
    for (int shift = 24; shift >= 0; shift -= 8) {
      if (shift < 24) topp_hist_kernel<<<dim3(kToppBlocks, rows), kToppThreads, 0, st>>>(t, ts, shift);
      topp_pick_kernel<<<rows, 256, 0, st>>>(t, ts, shift);
    }
    topp_tiecount_kernel<<<dim3(kToppBlocks, rows), kToppThreads, 0, st>>>(t, ts);
    topp_tiepick_kernel<<<rows, kToppThreads, 0, st>>>(t, ts);
    topp_sample_kernel<<<dim3(kToppBlocks, rows), kToppThreads, 0, st>>>(t);
    std::vector<unsigned long long> hk(rows);
    cudaMemcpyAsync(hk.data(), keys, rows * 8, cudaMemcpyDeviceToHost, st);
    cudaStreamSynchronize(st);
    std::vector<int32_t> tok(rows);
    for (int r = 0; r < rows; ++r) tok[r] = (int32_t)(0xFFFFFFFFu - (uint32_t)(hk[r] & 0xFFFFFFFFull));
    cudaMemcpy(d_tok, tok.data(), rows * 4, cudaMemcpyHostToDevice);
    if (cudaGetLastError() != cudaSuccess) err = fail(IS_ERR_CUDA, "is_dbg_topp kernels failed");
  }
  for (void* p : {(void*)scores, (void*)mlz, (void*)ebits, (void*)wpart, (void*)hist, (void*)sel, (void*)ts,
                  (void*)active, (void*)keys})
    if (p) cudaFree(p);
  return err;
}
