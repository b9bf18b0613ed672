// Non-GEMM kernels of the decode step: embedding, RMSNorm, QK-norm + RoPE +
// KV append, split shared-prefix / per-slot-suffix attention with LSE merge,
// and the 1-CTA finish / refill / page-recycle scheduler.
#pragma once
#include "common.cuh"

namespace isk {

constexpr int kHD = 128;      // head_dim (all Qwen3 shapes, R1)
constexpr int kChunk = 64;    // attention KV chunk (tokens per CTA)
constexpr int kKPad = 136;    // smem row pitch (bf16) -> conflict-free 16-B row reads

// ------------------------------------------------------------------ embed
// resid[r][:] = E[tok[r]][:] (fp32 residual stream); idle rows get zeros.
__global__ void embed_kernel(const __nv_bfloat16* __restrict__ E, const int32_t* __restrict__ row_tok,
                             const int32_t* __restrict__ row_active, float* __restrict__ resid, int H) {
  pdl_wait();
  pdl_launch_dependents();
  const int r = blockIdx.x;
  const bool act = row_active[r] != 0;
  const __nv_bfloat16* e = E + (size_t)(act ? row_tok[r] : 0) * H;
  for (int k = threadIdx.x; k < H; k += blockDim.x)
    resid[(size_t)r * H + k] = act ? __bfloat162float(e[k]) : 0.f;
}

// ------------------------------------------------------------------ RMSNorm
// xn[r][k] = bf16(resid[r][k] / sqrt(mean(resid[r]^2) + eps) * gain[k])   (R12 r1)
// One CTA per row; every thread issues all its float4 loads before reducing
// (no serial load chain).  H % 4 == 0, H / 4 <= 4 * blockDim.
__global__ void rmsnorm_kernel(const float* __restrict__ resid, const float* __restrict__ gain,
                               __nv_bfloat16* __restrict__ xn, int H, float eps) {
  pdl_wait();
  pdl_launch_dependents();
  const int r = blockIdx.x;
  const float4* x4 = reinterpret_cast<const float4*>(resid + (size_t)r * H);
  const float4* g4 = reinterpret_cast<const float4*>(gain);
  const int n4 = H >> 2;
  float4 xv[4], gv[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int i = threadIdx.x + j * blockDim.x;
    xv[j] = i < n4 ? x4[i] : make_float4(0.f, 0.f, 0.f, 0.f);
    gv[j] = i < n4 ? g4[i] : make_float4(0.f, 0.f, 0.f, 0.f);
  }
  float ss = 0.f;
#pragma unroll
  for (int j = 0; j < 4; ++j) ss += xv[j].x * xv[j].x + xv[j].y * xv[j].y + xv[j].z * xv[j].z + xv[j].w * xv[j].w;
  __shared__ float red[32];
  ss = warp_sum(ss);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = ss;
  __syncthreads();
  float tot = 0.f;
  for (int w = 0; w < (int)(blockDim.x >> 5); ++w) tot += red[w];
  const float rs = 1.0f / sqrtf(tot / (float)H + eps);
  __nv_bfloat162* o2 = reinterpret_cast<__nv_bfloat162*>(xn + (size_t)r * H);
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int i = threadIdx.x + j * blockDim.x;
    if (i < n4) {
      o2[2 * i] = __floats2bfloat162_rn(xv[j].x * rs * gv[j].x, xv[j].y * rs * gv[j].y);
      o2[2 * i + 1] = __floats2bfloat162_rn(xv[j].z * rs * gv[j].z, xv[j].w * rs * gv[j].w);
    }
  }
}

// ------------------------------------------------------------------ QK-norm + RoPE + KV append
struct QkvPostArgs {
  const float* qkv;        // [rows][(Hq + 2 Hkv) * 128] fp32 GEMM output
  const float* q_gain;     // [128]
  const float* k_gain;     // [128]
  const float* rope_cos;   // [max_pos][64]
  const float* rope_sin;
  const int32_t* row_active;
  const int32_t* row_pos;
  const int32_t* row_kvloc;  // decode: page*pt + offset; prefill: prefix position
  __nv_bfloat16* q_out;      // [rows][Hq][128]
  __nv_bfloat16* kv;         // decode: layer page pool [pages][2][Hkv][pt][128]; prefill: prefix [2][Hkv][Pcap][128]
  int Hq, Hkv, pt, pcap, prefill;
  float eps;
};

// grid (rows, Hq + 2*Hkv), block 128 (one thread per head dim).
__global__ void qkv_post_kernel(QkvPostArgs a) {
  pdl_wait();
  pdl_launch_dependents();
  const int r = blockIdx.x, h = blockIdx.y, d = threadIdx.x;
  if (!a.row_active[r]) return;
  const int W = (a.Hq + 2 * a.Hkv) * kHD;
  float x = a.qkv[(size_t)r * W + h * kHD + d];
  __shared__ float sh[kHD];
  __shared__ float red[4];
  const bool is_v = h >= a.Hq + a.Hkv;
  if (!is_v) {
    const bool is_q = h < a.Hq;
    float ss = warp_sum(x * x);
    if ((d & 31) == 0) red[d >> 5] = ss;
    __syncthreads();
    ss = red[0] + red[1] + red[2] + red[3];
    const float rs = 1.0f / sqrtf(ss / (float)kHD + a.eps);
    const float y = x * rs * (is_q ? a.q_gain[d] : a.k_gain[d]);
    sh[d] = y;
    __syncthreads();
    const int pos = a.row_pos[r];
    const int i = d & 63;
    const float c = a.rope_cos[(size_t)pos * 64 + i], s = a.rope_sin[(size_t)pos * 64 + i];
    x = d < 64 ? (y * c - sh[d + 64] * s) : (y * c + sh[d - 64] * s);
    if (is_q) {
      a.q_out[((size_t)r * a.Hq + h) * kHD + d] = __float2bfloat16_rn(x);
      return;
    }
  }
  const int kvsel = is_v ? 1 : 0;
  const int hk = h - a.Hq - (is_v ? a.Hkv : 0);
  const int loc = a.row_kvloc[r];
  size_t off;
  if (a.prefill) {
    off = (((size_t)kvsel * a.Hkv + hk) * a.pcap + loc) * kHD + d;
  } else {
    const int page = loc / a.pt, o = loc % a.pt;
    off = ((((size_t)page * 2 + kvsel) * a.Hkv + hk) * a.pt + o) * kHD + d;
  }
  a.kv[off] = __float2bfloat16_rn(x);
}

// ------------------------------------------------------------------ split attention
struct AttnArgs {
  const __nv_bfloat16* q;     // [rows][Hq][128]
  const __nv_bfloat16* kpre;  // prefix K of this layer [Hkv][pcap][128]
  const __nv_bfloat16* vpre;  // prefix V               [Hkv][pcap][128]
  const __nv_bfloat16* pool;  // page pool of this layer [pages][2][Hkv][pt][128]
  const int32_t* pagetab;     // [G][maxp]
  const int32_t* row_active;
  const int32_t* row_lid;     // local sample id (page table row)
  const int32_t* row_len;     // suffix tokens visible (t + 1)
  float* part_o;              // [rows][Hq][NC][128] (normalised partial outputs)
  float* part_ml;             // [rows][Hq][NC][2]  (max score, sum exp)
  int rows, Hq, Hkv, pcap, plen, pt, maxp;
  int nc_pre, nc_suf, NC;
  int prefill;                // 1: rows are prompt positions, causal over the prefix, no suffix
  float scale;                // 1/sqrt(128)
};

// One CTA = one KV chunk of 64 tokens for one kv head, shared by every query
// row that attends to it: the group's live rows x (Hq/Hkv) heads for a prefix
// chunk (read once per group, not once per slot: P:205), or one slot's rows
// for a suffix chunk.  Scores use lanes over tokens (16-B conflict-free smem
// rows), P.V uses lanes over head dims.
__global__ void __launch_bounds__(256) attn_partial_kernel(AttnArgs a) {
  pdl_wait();
  pdl_launch_dependents();
  __shared__ __align__(16) __nv_bfloat16 Ks[kChunk][kKPad];
  __shared__ __align__(16) __nv_bfloat16 Vs[kChunk][kKPad];
  __shared__ __align__(16) float qs[8][kHD];
  const int rep = a.Hq / a.Hkv;
  int b = blockIdx.x;
  const bool is_pre = b < a.Hkv * a.nc_pre;
  int h, c, r_only = -1, tok0, ntok;
  if (is_pre) {
    h = b / a.nc_pre;
    c = b % a.nc_pre;
    tok0 = c * kChunk;
    ntok = min(kChunk, a.plen - tok0);
  } else {
    b -= a.Hkv * a.nc_pre;
    c = b % a.nc_suf;
    b /= a.nc_suf;
    h = b % a.Hkv;
    r_only = b / a.Hkv;
    if (r_only >= a.rows || !a.row_active[r_only]) return;
    tok0 = c * kChunk;
    ntok = min(kChunk, a.row_len[r_only] - tok0);
    if (ntok <= 0) return;
  }
  // ---- stage K/V chunk in smem (each thread copies 16-B pieces)
  for (int i = threadIdx.x; i < kChunk * (kHD / 8); i += blockDim.x) {
    const int tk = i / (kHD / 8), seg = i % (kHD / 8);
    uint4 kk = make_uint4(0, 0, 0, 0), vv = make_uint4(0, 0, 0, 0);
    if (tk < ntok) {
      const int tok = tok0 + tk;
      const __nv_bfloat16 *kp, *vp;
      if (is_pre) {
        kp = a.kpre + ((size_t)h * a.pcap + tok) * kHD;
        vp = a.vpre + ((size_t)h * a.pcap + tok) * kHD;
      } else {
        const int page = a.pagetab[(size_t)a.row_lid[r_only] * a.maxp + tok / a.pt];
        const size_t base = (((size_t)page * 2) * a.Hkv + h) * a.pt + (tok % a.pt);
        kp = a.pool + base * kHD;
        vp = a.pool + (base + (size_t)a.Hkv * a.pt) * kHD;
      }
      kk = *reinterpret_cast<const uint4*>(kp + seg * 8);
      vv = *reinterpret_cast<const uint4*>(vp + seg * 8);
    }
    *reinterpret_cast<uint4*>(&Ks[tk][seg * 8]) = kk;
    *reinterpret_cast<uint4*>(&Vs[tk][seg * 8]) = vv;
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  const int nrows = is_pre ? a.rows : 1;
  const int nitems = nrows * rep;
  for (int it = warp; it < nitems; it += nw) {
    const int r = is_pre ? it / rep : r_only;
    const int qh = h * rep + (it % rep);
    if (!a.row_active[r]) continue;
    int valid = ntok;
    if (is_pre && a.prefill) valid = min(ntok, r + 1 - tok0);  // causal over the prompt
    const size_t pidx = ((size_t)r * a.Hq + qh) * a.NC + (is_pre ? c : a.nc_pre + c);
    if (valid <= 0) {
      if (lane == 0) {
        a.part_ml[pidx * 2] = -INFINITY;
        a.part_ml[pidx * 2 + 1] = 0.f;
      }
      continue;
    }
    // q row -> smem (fp32), broadcast reads below
    const __nv_bfloat16* qp = a.q + ((size_t)r * a.Hq + qh) * kHD;
    for (int d = lane; d < kHD; d += 32) qs[warp][d] = __bfloat162float(qp[d]);
    __syncwarp();
    float s[2];
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const int tk = lane + 32 * j;
      float acc = 0.f;
#pragma unroll
      for (int d = 0; d < kHD; d += 8) {
        const uint4 kv4 = *reinterpret_cast<const uint4*>(&Ks[tk][d]);
        const __nv_bfloat162* k2 = reinterpret_cast<const __nv_bfloat162*>(&kv4);
        const float4 qa = *reinterpret_cast<const float4*>(&qs[warp][d]);
        const float4 qb = *reinterpret_cast<const float4*>(&qs[warp][d + 4]);
        float2 f0 = __bfloat1622float2(k2[0]), f1 = __bfloat1622float2(k2[1]);
        float2 f2 = __bfloat1622float2(k2[2]), f3 = __bfloat1622float2(k2[3]);
        acc += qa.x * f0.x + qa.y * f0.y + qa.z * f1.x + qa.w * f1.y;
        acc += qb.x * f2.x + qb.y * f2.y + qb.z * f3.x + qb.w * f3.y;
      }
      s[j] = tk < valid ? acc * a.scale : -INFINITY;
    }
    const float m = warp_max(fmaxf(s[0], s[1]));
    const float p0 = s[0] == -INFINITY ? 0.f : expf(s[0] - m);
    const float p1 = s[1] == -INFINITY ? 0.f : expf(s[1] - m);
    const float l = warp_sum(p0 + p1);
    float o[4] = {0.f, 0.f, 0.f, 0.f};
    for (int tk = 0; tk < valid; ++tk) {
      const float p = __shfl_sync(0xffffffffu, tk < 32 ? p0 : p1, tk & 31);
      const __nv_bfloat162* v2 = reinterpret_cast<const __nv_bfloat162*>(&Vs[tk][lane * 4]);
      const float2 a0 = __bfloat1622float2(v2[0]), a1 = __bfloat1622float2(v2[1]);
      o[0] += p * a0.x;
      o[1] += p * a0.y;
      o[2] += p * a1.x;
      o[3] += p * a1.y;
    }
    const float inv = 1.0f / l;
    float4 ov = make_float4(o[0] * inv, o[1] * inv, o[2] * inv, o[3] * inv);
    *reinterpret_cast<float4*>(a.part_o + pidx * kHD + lane * 4) = ov;
    if (lane == 0) {
      a.part_ml[pidx * 2] = m;
      a.part_ml[pidx * 2 + 1] = l;
    }
    __syncwarp();
  }
}

// LSE merge (R8): o = sum_i w_i o_i / sum_i w_i, w_i = exp(m_i - max m) * l_i,
// over prefix chunks then suffix chunks in fixed order.  grid (rows, Hq), block 128.
__global__ void attn_merge_kernel(AttnArgs a, __nv_bfloat16* __restrict__ out) {
  pdl_wait();
  pdl_launch_dependents();
  const int r = blockIdx.x, qh = blockIdx.y, d = threadIdx.x;
  __nv_bfloat16* o = out + ((size_t)r * a.Hq + qh) * kHD + d;
  if (!a.row_active[r]) {
    *o = __float2bfloat16_rn(0.f);
    return;
  }
  int npre = a.nc_pre, nsuf = 0;
  if (a.prefill) npre = min(a.nc_pre, r / kChunk + 1);
  else nsuf = (a.row_len[r] + kChunk - 1) / kChunk;
  const size_t base = ((size_t)r * a.Hq + qh) * a.NC;
  float M = -INFINITY;
  for (int i = 0; i < npre + nsuf; ++i) {
    const int slot = i < npre ? i : a.nc_pre + (i - npre);
    M = fmaxf(M, a.part_ml[(base + slot) * 2]);
  }
  float num = 0.f, den = 0.f;
  for (int i = 0; i < npre + nsuf; ++i) {
    const int slot = i < npre ? i : a.nc_pre + (i - npre);
    const float mi = a.part_ml[(base + slot) * 2];
    if (mi == -INFINITY) continue;
    const float w = expf(mi - M) * a.part_ml[(base + slot) * 2 + 1];
    num += w * a.part_o[(base + slot) * kHD + d];
    den += w;
  }
  *o = __float2bfloat16_rn(num / den);
}

// ------------------------------------------------------------------ scheduler (Alg. 1 loop body, Alg. 3)
enum SchedState {
  ST_PHASE = 0,      // 0 prefix phase, 1 main phase
  ST_QLEN,
  ST_QHEAD,
  ST_BARRIER,
  ST_QUOTA,
  ST_STOPK,
  ST_MAIN_PENDING,
  ST_MAIN_QLEN,
  ST_MAIN_NINIT,
  ST_STEP,
  ST_PREFIX_STEPS,
  ST_DONE,
  ST_LIVE,
  ST_PEAK,
  ST_FREE_TOP,
  ST_ERROR,
  ST_TOKENS,
  ST_COUNT
};

struct SchedArgs {
  int G, g, row_cap, max_new, pt, maxp, P, log_cap, prompt_id, prompt_last;
  long long* st;             // [ST_COUNT]
  int32_t* slot_uid;         // [g]
  int32_t* slot_count;       // [g]
  int32_t* t;                // [G]
  const int32_t* true_len;   // [G]
  int32_t* queue;            // [G]
  const int32_t* main_init;  // [g]
  const int32_t* main_queue; // [G]
  int32_t* free_stack;       // [num_pages]
  int32_t* pagetab;          // [G][maxp]
  int32_t* npages;           // [G]
  int32_t* tokens;           // [G][max_new]
  int32_t* log_slot;         // [log_cap][g]
  int32_t* log_live;         // [log_cap]
  unsigned long long* keys;  // [row_cap] lm_head argmax keys
  int32_t* last_tok;         // [row_cap]
  uint8_t* last_fin;         // [row_cap]
  int32_t* row_active;
  int32_t* row_uid;          // global uid (RNG counter)
  int32_t* row_lid;          // local uid (page table)
  int32_t* row_t;
  int32_t* row_tok;
  int32_t* row_pos;
  int32_t* row_kvloc;
  int32_t* row_len;
};

// Single thread: the work is O(g + pages) integer bookkeeping per step.
// consume = 1: take the sampled tokens of the step that just ran, finish /
// park / refill in ascending slot order (R18); then always prepare the rows of
// the next step (page allocation on boundary crossing, R26).
__global__ void sched_kernel(SchedArgs a, int consume) {
  pdl_wait();
  pdl_launch_dependents();
  if (threadIdx.x != 0) return;
  long long* st = a.st;
  if (consume) {
    for (int s = 0; s < a.row_cap; ++s) {
      a.last_tok[s] = -1;
      a.last_fin[s] = 0;
    }
    for (int s = 0; s < a.g; ++s) {
      const int uid = a.slot_uid[s];
      if (uid < 0) continue;
      const uint32_t tok = 0xFFFFFFFFu - (uint32_t)(a.keys[s] & 0xFFFFFFFFull);
      a.tokens[(size_t)uid * a.max_new + a.t[uid]] = (int32_t)tok;
      a.last_tok[s] = (int32_t)tok;
      a.t[uid] += 1;
      st[ST_TOKENS] += 1;
    }
    for (int s = 0; s < a.g; ++s) {  // ascending slot index
      const int uid = a.slot_uid[s];
      if (uid < 0) continue;
      if (a.t[uid] == a.true_len[uid]) {
        st[ST_DONE] += 1;
        a.last_fin[s] = 1;
        for (int i = 0; i < a.npages[uid]; ++i) a.free_stack[st[ST_FREE_TOP]++] = a.pagetab[(size_t)uid * a.maxp + i];
        st[ST_LIVE] -= a.npages[uid];
        a.npages[uid] = 0;
      } else if (st[ST_STOPK] > 0 && a.t[uid] == st[ST_STOPK]) {
        // park: keep pages (prefix reuse)
      } else {
        continue;
      }
      a.slot_uid[s] = -1;
      a.slot_count[s] += 1;
      if (!st[ST_BARRIER] && st[ST_QHEAD] < st[ST_QLEN] && (st[ST_QUOTA] == 0 || a.slot_count[s] < st[ST_QUOTA]))
        a.slot_uid[s] = a.queue[st[ST_QHEAD]++];
    }
    bool idle = true;
    for (int s = 0; s < a.g; ++s) idle = idle && a.slot_uid[s] < 0;
    if (st[ST_BARRIER] && idle && st[ST_QHEAD] < st[ST_QLEN]) {
      for (int s = 0; s < a.g && st[ST_QHEAD] < st[ST_QLEN]; ++s) a.slot_uid[s] = a.queue[st[ST_QHEAD]++];
      idle = false;
    }
    if (st[ST_PHASE] == 0 && idle && st[ST_QHEAD] >= st[ST_QLEN] && st[ST_MAIN_PENDING]) {
      // prefix phase over: install the Alg. 2 plan (init fill + static SJF queue)
      for (int i = 0; i < st[ST_MAIN_QLEN]; ++i) a.queue[i] = a.main_queue[i];
      st[ST_QLEN] = st[ST_MAIN_QLEN];
      st[ST_QHEAD] = 0;
      st[ST_BARRIER] = 0;
      st[ST_QUOTA] = 0;
      st[ST_STOPK] = 0;
      st[ST_PHASE] = 1;
      st[ST_MAIN_PENDING] = 0;
      for (int s = 0; s < a.g; ++s) {
        a.slot_count[s] = 0;
        a.slot_uid[s] = s < st[ST_MAIN_NINIT] ? a.main_init[s] : -1;
      }
    }
  }
  // ---- prepare rows of the next step
  bool any = false;
  for (int s = 0; s < a.row_cap; ++s) {
    a.keys[s] = 0ull;
    const int uid = s < a.g ? a.slot_uid[s] : -1;
    if (uid < 0) {
      a.row_active[s] = 0;
      a.row_uid[s] = 0;
      a.row_lid[s] = 0;
      a.row_t[s] = 0;
      a.row_tok[s] = 0;
      a.row_pos[s] = 0;
      a.row_kvloc[s] = 0;
      a.row_len[s] = 0;
      continue;
    }
    any = true;
    const int tt = a.t[uid];
    if (tt % a.pt == 0) {
      int page = 0;
      if (st[ST_FREE_TOP] > 0) page = a.free_stack[--st[ST_FREE_TOP]];
      else st[ST_ERROR] = 1;  // budget violated: pool exhausted
      a.pagetab[(size_t)uid * a.maxp + tt / a.pt] = page;
      a.npages[uid] += 1;
      st[ST_LIVE] += 1;
    }
    a.row_active[s] = 1;
    a.row_uid[s] = a.prompt_id * a.G + uid;
    a.row_lid[s] = uid;
    a.row_t[s] = tt;
    a.row_tok[s] = tt == 0 ? a.prompt_last : a.tokens[(size_t)uid * a.max_new + tt - 1];
    a.row_pos[s] = a.P - 1 + tt;
    a.row_kvloc[s] = a.pagetab[(size_t)uid * a.maxp + tt / a.pt] * a.pt + tt % a.pt;
    a.row_len[s] = tt + 1;
  }
  if (any) {
    const long long step = st[ST_STEP];
    if (step < a.log_cap) {
      for (int s = 0; s < a.g; ++s) a.log_slot[step * a.g + s] = a.slot_uid[s];
      a.log_live[step] = (int32_t)st[ST_LIVE];
    }
    st[ST_STEP] = step + 1;
    if (st[ST_PHASE] == 0) st[ST_PREFIX_STEPS] += 1;
    if (st[ST_LIVE] > st[ST_PEAK]) st[ST_PEAK] = st[ST_LIVE];
  }
}

// Prefill rows: row r = prompt position r (0..P-2), causal over the prefix.
__global__ void prefill_rows_kernel(const int32_t* __restrict__ prompt, int n, int32_t* row_active,
                                    int32_t* row_tok, int32_t* row_pos, int32_t* row_kvloc) {
  pdl_wait();
  pdl_launch_dependents();
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n) return;
  row_active[r] = 1;
  row_tok[r] = prompt[r];
  row_pos[r] = r;
  row_kvloc[r] = r;
}

// Benchmark reward (R29) and length per sample.
__global__ void results_kernel(const int32_t* __restrict__ tokens, const int32_t* __restrict__ true_len, int G,
                               int max_new, int vocab, float* reward, int32_t* len) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= G) return;
  int c = 0;
  const int L = true_len[i];
  for (int t = 0; t < L; ++t) c += tokens[(size_t)i * max_new + t] < vocab / 2;
  reward[i] = (float)c / (float)L;
  len[i] = L;
}

__global__ void bf16_to_f32_kernel(const __nv_bfloat16* __restrict__ x, float* __restrict__ y, int n) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) y[i] = __bfloat162float(x[i]);
}

}  // namespace isk
