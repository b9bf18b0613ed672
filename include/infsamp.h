/* infsamp.h -- C ABI of libinfsamp, the B200 (sm_100a) continuous-sampling
 * decode step of Infinite Sampling (arXiv 2506.22950).
 *
 * Conventions
 *   - Every call returns is_status; nothing aborts and no C++ exception crosses
 *     the ABI.  is_last_error() returns a one-line "IS_ERR_<CODE>: <detail>"
 *     message for the calling thread.
 *   - Pointers named d_* are DEVICE pointers (cudaMalloc / torch CUDA memory),
 *     h_* are HOST pointers.  The caller owns every buffer it passes; the
 *     library owns only what is_create allocates (packed weights, shared prefix
 *     KV, the KV page pool, slot/page tables, activations) and frees it in
 *     is_destroy.
 *   - A context is bound to one CUDA stream and one host thread; distinct
 *     contexts are independent.  Device work is asynchronous on that stream;
 *     CUDA errors surface as IS_ERR_CUDA on the next call (CUDA's convention).
 *   - Same inputs + same seed => byte-identical tokens, schedules and stats.
 *
 * Citations: P:n = PAPER.md line n; S:n = SPEC.md line n; R<k> = DESIGN.md
 * reading k.
 */
#ifndef INFSAMP_H_
#define INFSAMP_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  IS_OK = 0,
  IS_ERR_CONFIG = 1,   /* invalid shape / G mod g != 0 / eps <= 0 / N <= 0 */
  IS_ERR_BUDGET = 2,   /* worst-case KV reservation exceeds kv_budget_bytes (R25) */
  IS_ERR_CAPACITY = 3, /* a fixed capacity (rows, steps, pages) would be exceeded */
  IS_ERR_DATA = 4,     /* missing or < 1 lengths, bad token ids */
  IS_ERR_STATE = 5,    /* call order violated (e.g. decode before prefill) */
  IS_ERR_CUDA = 6      /* a CUDA runtime/driver error */
} is_status;

/* Sampling-loop policy (Alg. 1). */
typedef enum {
  IS_MODE_FULL = 0,    /* all G samples decode in parallel (g = G); unbudgeted reference */
  IS_MODE_NAIVE = 1,   /* N = G/g micro groups, barrier between groups */
  IS_MODE_FIFO = 2,    /* fixed-slot continuous sampling: quota N per slot, trace order (R19) */
  IS_MODE_INFINITE = 3, /* Alg. 1: [prefix phase] + Alg. 2 FPTAS plan + Alg. 3 SJF refill */
  /* Table 2's decomposition (definitions of SPEC.md, DESIGN R23): */
  IS_MODE_FPTAS_ONLY = 4, /* Alg. 2 plan in its lexicographic (n, j) order, FIFO refill, no quota */
  IS_MODE_SJF_ONLY = 5,   /* trace-order start (samples 0..g-1), Alg. 3 SJF refill, no quota */
  IS_MODE_DYNAMIC = 6     /* dynamic-slot sampling (NEXT-2, DESIGN R35): g slots, no quota,
                             the G samples are candidates drawn in trace order; the group stops at
                             the dynamic_target-th completion and in-flight samples are discarded */
} is_mode;

typedef enum { IS_ADV_STD_NORM = 0, IS_ADV_MEAN_ONLY = 1 } is_adv_mode;

/* Qwen3-shaped decoder (shapes R1).  head_dim must be 128. */
typedef struct {
  int32_t layers, hidden, n_q_heads, n_kv_heads, head_dim, ffn, vocab;
  float rms_eps, rope_theta;
} is_shape;

typedef struct {
  is_shape shape;
  int32_t G;               /* group size */
  int32_t g;               /* micro-group size = decoding slots; ignored (= G) in FULL mode */
  int32_t max_new_tokens;  /* generation cap (1024) */
  int32_t prompt_len;      /* P; the shared prefix holds positions 0..P-2 (R6) */
  int32_t prefix_k;        /* tokens decoded before length prediction; 0 = none */
  int32_t page_tokens;     /* tokens per KV page (16) */
  int32_t row_capacity;    /* rows of the fixed per-step batch (>= slots, <= 64); 0 = round_up(g, 16).
                              Kernel configuration depends only on this (batch invariance, R12). */
  int64_t kv_budget_bytes; /* KV budget (prefix + pages); <= 0 means unbudgeted (R25) */
  double eps;              /* FPTAS tolerance epsilon (Alg. 2) */
  float temperature;       /* sampling temperature (0.8) */
  uint64_t seed;           /* Philox key (R11) */
  is_mode mode;
  int32_t decode_impl;     /* reserved: 0 and 1 both select the decode step of one kernel per
                              operator in one CUDA graph (round 1's persistent whole-stack kernel
                              was slower, 2.74 vs 1.74 ms per step, and is retired); other
                              values are IS_ERR_CONFIG */
  int32_t max_groups;      /* co-resident prompt groups sharing each decode step (SURVEY §8f
                              NEXT-1; 0 or 1 = the paper's one group per GPU).  Group slot m owns
                              rows m*g .. m*g+g-1; kv_budget_bytes is per group, the page pool
                              (max_groups x the per-group pool) is shared.  max_groups*g <= 64 */
  int32_t dynamic_target;  /* IS_MODE_DYNAMIC: completions to stop at (0 = G); 0 in every other mode */
  int32_t eos_enabled;     /* R37 (SURVEY a8 "or token == eos if enabled"): 0 = trace-driven termination
                              only (R5, the parity setting); 1 = a sample also finishes when it samples
                              eos_id (its length is then shorter than true_len).  Needs prefix_k == 0 */
  int32_t eos_id;
  int32_t bin_slots;       /* IS_MODE_INFINITE: 0 = Alg. 2 over N = G/g micro groups (the paper), 1 = over
                              g slot bins (SPEC bin_mode = slots; NEXT-2, DESIGN R38): slot j starts
                              with bin j's head, then Alg. 3 SJF refill.  is_plan_out.loads then has g entries */
  int32_t admit_slots;     /* memory-aware admission by predicted length ("samples from future micro
                              groups may be promoted early if they fit the current memory profile"; NEXT-2,
                              DESIGN R41), IS_MODE_INFINITE with a KV budget: 0 = off; S > g = rows per step:
                              slots 0..g-1 keep the worst-case reservation of R25, slots g..S-1 are elastic
                              and share the rest of the budget's pages, admitting the SJF queue head when its
                              predicted pages fit.  Needs prefix_k == 0, max_groups <= 1, bin_slots == 0.
                              is_copy_schedule then has S columns; a stalled slot is logged as -2 - uid */
  float top_p;             /* nucleus sampling (DESIGN R36): 0 < top_p < 1 samples the
                              Gumbel-max token inside the top-p nucleus (integer-exact mass, fixed-
                              sequence exp); 0 or 1 = off (the paper's plain temperature sampling).
                              Costs a [row_capacity][vocab] fp32 logits buffer and one extra kernel */
} is_config;

/* Alg. 2 output plus the runtime plan (Alg. 1, Alg. 3).  All arrays are
 * caller-allocated with the sizes given. */
typedef struct {
  int32_t* mask;          /* [G][2]: (group n in 1..N, position j) */
  int64_t* scaled_len;    /* [G]: l~_i = ceil(l^_i / K) */
  int64_t* loads;         /* [N]: L_n; N = G/g, or g with bin_slots */
  int32_t* overflow_ids;  /* [G]: samples placed by the least-loaded fallback (R15) */
  int32_t* init_slots;    /* [g]: first g samples from mask, lexicographic (n, j) (R13) */
  int32_t* refill_queue;  /* [G]: static SJF order of the remaining samples (R17) */
  double K;               /* scale K = eps*S/N */
  int64_t capacity;       /* C~ = ceil(sum l~ / N) */
  int32_t n_overflow;
  int32_t queue_len;
  int64_t reserved_bytes; /* worst-case live KV bytes of this plan (R25) */
} is_plan_out;

typedef struct {
  int32_t steps;          /* decode steps run for the current group */
  int32_t prefix_steps;   /* of which in the prefix phase (R22) */
  int32_t completed;      /* samples finished */
  int32_t live_pages;     /* KV pages allocated now */
  int32_t peak_pages;     /* max over steps (R26) */
  int32_t error;          /* device-side error flag (page pool exhausted = budget violated) */
  int64_t tokens_decoded; /* sum of active slots over steps */
  int64_t peak_kv_bytes;  /* prefix bytes + peak_pages * page bytes (R26) */
  int64_t page_bytes;
  int64_t prefix_bytes;
  int32_t num_pages;      /* size of the page pool */
  int32_t row_capacity;
  int64_t suffix_tokens;  /* sum over decode steps of the live rows' suffix lengths (algorithmic KV bytes) */
  int32_t groups;         /* co-resident group slots of the context */
  int64_t global_steps;   /* decode steps with >= 1 active slot in any group */
  int64_t global_peak_kv_bytes;  /* all groups' prefixes + peak pages of the shared pool */
  int32_t launches_per_step;      /* kernel launches in one decode step (the captured graph) */
  int32_t launches_per_prefill;   /* kernel launches of one is_prefill */
  int32_t discarded;      /* IS_MODE_DYNAMIC: samples in flight at the stop, discarded (R35) */
  int32_t stalls;         /* admit_slots: slot-steps an elastic slot waited for a page (R41) */
} is_stats;

typedef struct is_ctx is_ctx;

/* Alg. 2 + Alg. 1 initial fill + Alg. 3 static refill order + budget check.
 * Pure host function.  h_pred_len[G] >= 1; h_finished[G] (nullable) marks
 * samples that completed in the prefix phase (R22).  mode FULL/NAIVE/FIFO
 * return the trace-order plan (mask etc. zeroed).  Errors: IS_ERR_CONFIG,
 * IS_ERR_DATA, IS_ERR_BUDGET. */
is_status is_plan(const is_config* cfg, const int32_t* h_pred_len, const uint8_t* h_finished,
                  is_plan_out* out);

/* Creates a context: packs the weights into the library's own layout, sizes
 * the KV page pool from kv_budget_bytes (or from the full-length worst case
 * when unbudgeted), captures the decode step.  d_weights: n_weights device
 * pointers to bf16 tensors in HF Qwen3 layout ([out, in]) in the order
 *   embed[V,H], final_norm[H], then per layer l = 0..L-1:
 *   in_norm[H], wq[Hq*d,H], wk[Hkv*d,H], wv[Hkv*d,H], q_norm[d], k_norm[d],
 *   wo[H,Hq*d], post_norm[H], w_gate[F,H], w_up[F,H], w_down[H,F]
 * (n_weights = 2 + 11*L).  The caller's weights are only read during this call.
 * stream: a cudaStream_t (NULL = legacy default stream). */
is_status is_create(const is_config* cfg, const void* const* d_weights, int32_t n_weights, void* stream,
                    is_ctx** out);
void is_destroy(is_ctx* ctx);

/* Prefill the prompt ("retain the prefill KV cache for the prompt
 * itself, which is shared by all groups"): a causal forward over positions
 * 0..P-2 writes the shared, read-only prefix KV.  d_prompt: [prompt_len] int32
 * token ids in [0, vocab).  prompt_id keys the RNG (uid = prompt_id*G + i, R11). */
is_status is_prefill(is_ctx* ctx, const int32_t* d_prompt, int32_t prompt_id);

/* Start the sampling loop for the prefilled prompt.  h_true_len[G]: trace
 * lengths (termination, R5); h_pred_len[G]: predicted lengths for Alg. 2
 * (INFINITE only; nullable otherwise).  Runs is_plan, checks the budget,
 * uploads the plan and fills the g slots (Alg. 1).  With prefix_k > 0
 * (INFINITE) the prefix phase runs first in ceil(G/g) barriered rounds (R22);
 * the plan is installed on the device and takes over when it ends. */
is_status is_start_group(is_ctx* ctx, const int32_t* h_true_len, const int32_t* h_pred_len);

/* One decode step: every active slot attends to the shared prefix
 * plus its own pages, samples its next token, then finished slots are refilled
 * in place (is_refill).  d_next_tokens / d_finished: [row_capacity] device
 * buffers (nullable) receiving the sampled token / finish flag per row (row
 * m*g + s = group m, slot s; -1 / 0 for rows idle in that step).  Asynchronous:
 * no host synchronisation.  IS_ERR_BUDGET once the device scheduler has found the
 * page pool exhausted (R25: cannot happen within a budget is_create accepted; the
 * flag is seen with the lag of the steps still in flight, and from then on every row
 * is idle: no page is ever handed out twice). */
is_status is_decode_step(is_ctx* ctx, int32_t* d_next_tokens, uint8_t* d_finished);

/* Finish/refill/page-recycle policy alone (Alg. 3, "cache is
 * cleared and the memory is reassigned back to the pool"): consumes the last
 * sampled keys, appends tokens, finishes/parks samples, refills freed slots in
 * ascending slot order from the static queue, allocates pages for the next
 * step.  Called inside is_decode_step; exported for tests.  d_finished
 * [row_capacity] (nullable) receives the finish flag per row; d_new_uid
 * [row_capacity] (nullable) the uid now in each row (m*g + s; -1 idle). */
is_status is_refill(is_ctx* ctx, uint8_t* d_finished, int32_t* d_new_uid);

/* Decode steps until the group completes (bounded host run-ahead, no per-step
 * sync).  h_steps (nullable) receives the number of steps.  IS_ERR_CAPACITY if
 * max_steps ran out first; IS_ERR_BUDGET if the page pool was exhausted (see
 * is_decode_step). */
is_status is_run_group(is_ctx* ctx, int32_t max_steps, int32_t* h_steps);

is_status is_query(is_ctx* ctx, is_stats* out); /* synchronises the stream */

/* Generated tokens [G][max_new_tokens] (row uid-major, -1 beyond true_len). */
is_status is_copy_tokens(is_ctx* ctx, int32_t* dst, int32_t dst_is_device);

/* Per-step schedule log: slot table [max_steps][g] (uid or -1) and live pages
 * [max_steps] (R26); returns the number of logged steps in *h_n. */
is_status is_copy_schedule(is_ctx* ctx, int32_t* h_slot_table, int32_t* h_live_pages, int32_t max_steps,
                           int32_t* h_n);

/* Co-resident groups (is_config.max_groups > 1).  The _slot
 * calls act on group slot m in [0, max_groups); the unsuffixed calls above are
 * the slot-0 calls.  Groups are independent: each has its own prompt (shared
 * prefix KV), plan, refill queue, RNG uids (prompt_id*G + i) and schedule log,
 * and every decode step serves all started groups' live rows at once.
 * is_prefill_slot / is_start_group_slot may be called while other groups are
 * mid-rollout (between decode steps); restarting a slot returns the pages its
 * previous group still held.  is_run_until_any_done decodes until a started
 * group completes; *h_done_mask gets bit m for every started group that is
 * done, *h_global_steps the decode steps run so far in this context. */
is_status is_prefill_slot(is_ctx* ctx, int32_t slot, const int32_t* d_prompt, int32_t prompt_id);
is_status is_start_group_slot(is_ctx* ctx, int32_t slot, const int32_t* h_true_len, const int32_t* h_pred_len);
is_status is_run_until_any_done(is_ctx* ctx, int32_t max_steps, int32_t* h_done_mask, int64_t* h_global_steps);
/* (is_run_until_any_done: IS_ERR_BUDGET as is_run_group.  Environment knob for negative
 * tests only: IS_DBG_POOL_PAGES=n at is_create sizes the page pool to n pages.) */
is_status is_query_slot(is_ctx* ctx, int32_t slot, is_stats* out);
is_status is_copy_tokens_slot(is_ctx* ctx, int32_t slot, int32_t* dst, int32_t dst_is_device);
is_status is_copy_schedule_slot(is_ctx* ctx, int32_t slot, int32_t* h_slot_table, int32_t* h_live_pages,
                                int32_t max_steps, int32_t* h_n);
is_status is_group_results_slot(is_ctx* ctx, int32_t slot, float* d_reward, int32_t* d_len);

/* KL-penalised reward, host arrays:
 *   out[i] = rm[i] - beta * sum_{t < len[i]} (logp[i][t] - logp_ref[i][t])
 * logp / logp_ref [G][max_new] (logp from is_copy_logprobs, logp_ref the caller's
 * reference model), sums in fp64 over ascending t.  Pure; IS_ERR_DATA on a bad length. */
is_status is_kl_rewards(const float* h_rm, const float* h_logp, const float* h_logp_ref, const int32_t* h_len,
                        int32_t G, int32_t max_new, float beta, float* h_out);

/* Value of the GRPO objective, Eq. 3 (l.133-141) = Eq. 4's micro-group average
 * (l.327-345; equal micro groups), host arrays [G][max_new]:
 *   (1/G) sum_i (1/len_i) sum_t { min(lam A_i, clip(lam, 1-eps, 1+eps) A_i) - beta KL_t },
 *   lam = exp(logp - logp_old), KL_t = exp(logp_ref - logp) - (logp_ref - logp) - 1 (DESIGN R34).
 * fp64; *h_out receives the value.  No gradients (training is out of scope). */
is_status is_grpo_objective(const float* h_logp, const float* h_logp_old, const float* h_logp_ref, const float* h_adv,
                            const int32_t* h_len, int32_t G, int32_t max_new, float clip_eps, float beta,
                            double* h_out);

/* Log-probability of every generated token: h_dst[G][max_new]
 * host fp32, log pi_theta(token) = z_tok - logsumexp_v(z_v) of the step's logits at
 * temperature 1 (R33), reduced on the device from the lm_head CTAs'
 * online (max, sum-exp) partials in a fixed order; 0 beyond each sample's length. */
is_status is_copy_logprobs(is_ctx* ctx, float* h_dst);
is_status is_copy_logprobs_slot(is_ctx* ctx, int32_t slot, float* h_dst);

/* Benchmark reward and completion length per sample (R29):
 * d_reward[G] = #{tokens < vocab/2}/len, d_len[G] = len.  Device buffers.  len is the
 * emitted length of a completed sample (true_len, or shorter when it stopped at
 * eos_id, R37); a sample that did not complete (IS_MODE_DYNAMIC, R35: discarded in
 * flight or never started) reports len = 0 and reward = 0, so callers select the
 * completed samples (len >= 1) before the advantages or is_kl_rewards. */
is_status is_group_results(is_ctx* ctx, float* d_reward, int32_t* d_len);

/* Group advantages, Eq. 2 or mean-only; fp64 sums in
 * ascending index, population sigma, sigma = 0 -> 0 (R28).  Host pointers. */
is_status is_group_advantages(const float* h_rewards, int32_t G, is_adv_mode mode, float* h_adv);

/* The one cross-GPU exchange (BASELINE north_star "NCCL over NVLink
 * used only to all-gather completion lengths and rewards"): prompts are sharded by
 * rank, and after a group completes every rank all-gathers its (length, reward)
 * per sample so each holds the global arrays the group advantages (Eq. 2,
 * P:128-131) and the policy update need.
 *   is_nccl_unique_id   rank 0 creates the 128-byte ncclUniqueId (h_uid); the caller
 *                       broadcasts it (e.g. over its torch process group);
 *   is_nccl_comm_init   every rank joins; *comm_out is an ncclComm_t owned by the caller;
 *   is_allgather_results  on the context's stream: d_len[G] int32, d_reward[G] fp32
 *                       (device; e.g. from is_group_results) -> d_all_len[world*G],
 *                       d_all_reward[world*G] in rank order;
 *   is_nccl_comm_destroy  frees the communicator.
 * NCCL is resolved at run time from the process's libnccl.so.2 (IS_ERR_CUDA if absent). */
is_status is_nccl_unique_id(void* h_uid);
is_status is_nccl_comm_init(const void* h_uid, int32_t rank, int32_t world, void** comm_out);
is_status is_allgather_results(is_ctx* ctx, void* comm, const int32_t* d_len, const float* d_reward,
                               int32_t* d_all_len, float* d_all_reward);
/* The same exchange for n samples per rank (e.g. all of a rank's groups at once, k x G, after
 * its last rollout: SURVEY §8e "one ncclAllGather ... after a rank's groups"): d_len / d_reward
 * [n], d_all_len / d_all_reward [world * n] in rank order.  IS_ERR_CONFIG if n < 1. */
is_status is_allgather_results_n(is_ctx* ctx, void* comm, int32_t n, const int32_t* d_len, const float* d_reward,
                                 int32_t* d_all_len, float* d_all_reward);
is_status is_nccl_comm_destroy(void* comm);

/* Debug: when d_logits != NULL every following lm_head launch also writes its
 * fp32 logits to d_logits[row_capacity][vocab] (sampler parity, R12 (i)). */
is_status is_set_logits_dump(is_ctx* ctx, float* d_logits);

/* Per-launch timing of the kernels of one decode step (CUDA events on the
 * context stream, step replayed eagerly, not from the graph): h_ms[n] receives
 * the milliseconds of launch i and h_kind[n] its kind (0 embed/norm, 1 QKV GEMM,
 * 2 qkv post, 3 attention, 4 o_proj, 5 gate/up, 6 down, 7 lm_head+sampler,
 * 8 refill).  Returns the number of launches in *h_n. */
is_status is_profile_step(is_ctx* ctx, float* h_ms, int32_t* h_kind, int32_t cap, int32_t* h_n);

/* Same outputs, but the step is captured into a CUDA graph (as the run loops
 * replay it) with an event node after every launch, then replayed once: each
 * interval is the launch's device duration plus one graph-node hop (the event
 * nodes turn PDL edges into full dependencies).  Advances one decode step. */
is_status is_profile_step_graph(is_ctx* ctx, float* h_ms, int32_t* h_kind, int32_t cap, int32_t* h_n);

/* Average device duration (ms) per layer of a decode kernel kind (1 QKV, 3 attention
 * (the layer's shared-prefix + suffix launches), 4 o_proj, 5 gate/up, 6 down), issued
 * exactly as the decode step issues it
 * (arguments, split, stages, PDL) for every layer, `reps` passes, back to back in
 * one CUDA graph timed with CUDA events on the context stream (one warm-up replay
 * first).  The launches write the step's scratch buffers (activations, residual),
 * so the context must be re-prefilled / restarted before decoding on.  Per-op path
 * only (IS_ERR_CONFIG otherwise).  *h_launches receives the launches timed. */
is_status is_profile_kernel(is_ctx* ctx, int32_t kind, int32_t reps, float* h_ms_per_launch, int32_t* h_launches);

/* Kernel-level test hook: one tcgen05 swap-AB GEMM Y[n][m] = sum_k X[n][k] W[m][k]
 * (X: d_x [rows][K] bf16, W: d_w [M][K] bf16, Y: d_y [rows][M] fp32),
 * rows <= 64, K % 64 == 0, on `stream`. split = K-split cluster size (1..8). */
is_status is_dbg_gemm(const void* d_w, const void* d_x, float* d_y, int32_t M, int32_t K, int32_t rows,
                      int32_t split, void* stream);

/* Kernel-level test hook of the top-p chain (R36) on caller logits: d_logits
 * [rows][V] fp32 (V % 4 == 0), per-row Philox counters d_uid[rows] / d_t[rows];
 * 0 < top_p < 1.  d_tok[rows] (device) receives the sampled tokens.  Synchronous;
 * allocates its scratch per call. */
is_status is_dbg_topp(const float* d_logits, int32_t rows, int32_t V, float temperature, float top_p, uint64_t seed,
                      const int32_t* d_uid, const int32_t* d_t, int32_t* d_tok, void* stream);

/* Kernel-level test hook of the decode split attention ("retain
 * the prefill KV cache for the prompt itself, which is shared by all groups", l.205 "a separate
 * KV buffer for its response tokens"; LSE merge = DESIGN R8): builds the step's attention work
 * list and issues exactly the launches one decode layer issues, on caller data (one layer):
 *   d_q        [rows][Hq][128] bf16 query rows (after QK-norm and RoPE)
 *   d_prefix   [groups][2][Hkv][plen][128] bf16 shared-prefix K then V of each group
 *   d_pool     [num_pages][2][Hkv][page_tokens][128] bf16 page pool (K then V per page)
 *   d_pagetab  [rows][maxp] int32 page ids of each row's suffix, in token order
 *   d_row_len  [rows] int32 suffix tokens each row attends to (t + 1); 0 = idle row
 *   grp_rows   rows per group: rows m*grp_rows .. attend to prefix m (groups*grp_rows <= rows <= 64)
 *   impl       0 = the decode step's choice, 1 = tcgen05 prefix + 32-token warp suffix units with
 *              the fused merge, 2 = tcgen05 prefix + 64-token CTA units + merge kernel, 3 = CUDA-core
 *              prefix chunks + CTA units + merge kernel (groups = 1), 4 = tcgen05 prefix + 64-token
 *              suffix units on mma.sync with the fused merge (the default when page_tokens % 8 == 0)
 *   d_out      [rows][Hq][128] bf16 output (rows that are idle are not written);
 *   d_out_f32  (nullable) the same before the bf16 rounding
 *   reps, h_ms reps > 0: then `reps` more timed runs, each after a 256 MiB write that evicts L2;
 *              h_ms[reps] receives each run's CUDA-event time of the attention launches alone.
 * Synchronous (allocates its scratch per call).  Errors: IS_ERR_CONFIG (shapes, impl),
 * IS_ERR_CAPACITY (more partials than the merge holds), IS_ERR_DATA (a length above
 * maxp*page_tokens). */
is_status is_dbg_attn(const void* d_q, const void* d_prefix, int32_t plen, int32_t groups, int32_t grp_rows,
                      const void* d_pool, int32_t num_pages, int32_t page_tokens, const int32_t* d_pagetab,
                      int32_t maxp, const int32_t* d_row_len, int32_t rows, int32_t Hq, int32_t Hkv, int32_t impl,
                      void* d_out, float* d_out_f32, int32_t reps, float* h_ms, void* stream);

/* Debug: copy an internal activation buffer to the host (0 q [rc][Hq][128] bf16,
 * 1 residual [rc][H] f32, 3 final normalised rows [rc][H] bf16, 4 attention
 * output [rc][Hq*128] bf16, 6 SwiGLU activations [rc][F] bf16).  Synchronises
 * the stream. */
is_status is_dbg_copy(is_ctx* ctx, int32_t which, void* h_dst, int64_t bytes);

const char* is_last_error(void);
const char* is_version(void);

#ifdef __cplusplus
}
#endif
#endif /* INFSAMP_H_ */
