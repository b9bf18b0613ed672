// Non-GEMM kernels of the decode step: embedding, RMSNorm, split shared-prefix / per-slot-suffix attention with LSE merge,
// and the 1-CTA finish / refill / page-recycle scheduler.
#pragma once
#include "common.cuh"

namespace isk {

constexpr int kHD = 128;      // head_dim (all Qwen3 shapes, R1)
constexpr int kKPad = 136;    // smem row pitch (bf16) -> conflict-free 16-B row reads

// ------------------------------------------------------------------ embed
// resid[r][:] = E[tok[r]][:] (fp32 residual stream); idle rows get zeros.
__global__ void embed_kernel(const __nv_bfloat16* __restrict__ E, const int32_t* __restrict__ row_tok,
                             const int32_t* __restrict__ row_active, float* __restrict__ resid, int H) {
  pdl_launch_dependents();  // let the next kernel launch and prefetch now; it waits for our completion itself
  pdl_wait();
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
  pdl_launch_dependents();  // let the next kernel launch and prefetch now; it waits for our completion itself
  pdl_wait();
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

// ------------------------------------------------------------------ split attention
// PAPER.md l.171-174 / l.205: every live slot attends to the prompt's shared
// prefix KV (written once by prefill) and to its own paged response KV.  The
// work is split at that boundary (R8):
//   * prefix item  = (kv head, 128-token prefix chunk): the chunk is staged in
//     shared memory ONCE and every live row of the group (x Hq/Hkv query heads)
//     is scored against it -- the prefix is read once per group per step;
//   * suffix item  = (row, kv head, 128-token chunk of that slot's pages): one
//     warp, K rows read straight from the page pool (each lane owns 4 tokens,
//     256-B contiguous rows), V read coalesced (lanes over head dims);
// each item writes a normalised partial (o, m, l) per query head; the item that
// completes a (row, kv head) -- a per-(row, head) arrival counter -- merges all
// of its partials by log-sum-exp in fixed chunk order (prefix chunks, then
// suffix chunks), so the result does not depend on arrival order.
constexpr int kAC = 64;           // tokens per suffix chunk (one CTA)
constexpr int kPC = 32;           // tokens per shared-prefix chunk (one CTA, all live rows)
constexpr int kMaxRep = 8;        // Hq / Hkv <= 8

struct AttnArgs {
  const __nv_bfloat16* q;     // [rows][Hq][128]
  const __nv_bfloat16* kpre;  // prefix K of this layer [Hkv][pcap][128]
  const __nv_bfloat16* vpre;  // prefix V               [Hkv][pcap][128]
  const __nv_bfloat16* pool;  // page pool of this layer [pages][2][Hkv][pt][128]
  const int32_t* pagetab;     // [G][maxp]
  const int32_t* row_active;
  const int32_t* row_lid;     // local sample id (page table row)
  const int32_t* row_len;     // suffix tokens visible (t + 1)
  float* part_o;              // [rows][Hq][NC][128] normalised partial outputs
  float* part_ml;             // [rows][Hq][NC][2]   (max score, sum exp)
  int32_t* cnt;               // [rows][Hkv] arrival counters (left at 0)
  const int32_t* items;       // decode work list (built by sched_kernel)
  const uint8_t* pf_ptr[4];   // weights to pull into L2 while attention runs (latency-bound phase)
  long long pf_bytes[4];
  int n_pf;
  unsigned long long* dbg_ts;  // optional [gridDim][16] globaltimer stamps
  const long long* n_items;   // its length
  __nv_bfloat16* out;         // [rows][Hq][128]
  int rows, Hq, Hkv, pcap, plen, pt, maxp;
  int nc_pre, nc_suf, NC;
  int prefill;                // 1: rows are prompt positions, causal over the prefix, no suffix
  float scale;                // 1/sqrt(128)
};

__device__ __forceinline__ void astamp(const AttnArgs& a, int i) {
  if (a.dbg_ts && threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    a.dbg_ts[blockIdx.x * 16 + i] = t;
  }
}

__device__ __forceinline__ int attn_expected(const AttnArgs& a, int r) {
  if (a.prefill) return min(a.nc_pre, r / kPC + 1);
  return a.nc_pre + (a.row_len[r] + kAC - 1) / kAC;
}

// Warp-level LSE merge of all partials of (row r, kv head h) -> bf16 output.
// Lane i holds partial i's (m, l) (<= 32 partials); the o loads are independent.
__device__ void attn_merge_warp(const AttnArgs& a, int r, int h, int lane) {
  const int rep = a.Hq / a.Hkv;
  const int npre = a.prefill ? min(a.nc_pre, r / kPC + 1) : a.nc_pre;
  const int nsuf = a.prefill ? 0 : (a.row_len[r] + kAC - 1) / kAC;
  const int n = npre + nsuf;
  const int my_slot = lane < npre ? lane : a.nc_pre + (lane - npre);
  for (int j = 0; j < rep; ++j) {
    const int qh = h * rep + j;
    const size_t base = ((size_t)r * a.Hq + qh) * a.NC;
    float mi = -INFINITY, li = 0.f;
    if (lane < n) {
      const float2 ml = __ldcg(reinterpret_cast<const float2*>(a.part_ml + (base + my_slot) * 2));
      mi = ml.x;
      li = ml.y;
    }
    const float M = warp_max(mi);
    const float wi = (lane < n && mi != -INFINITY) ? expf(mi - M) * li : 0.f;
    const float den = warp_sum(wi);
    float4 num = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll 4
    for (int i = 0; i < n; ++i) {
      const float w = __shfl_sync(0xffffffffu, wi, i);
      const int slot = i < npre ? i : a.nc_pre + (i - npre);
      if (w != 0.f) {
        const float4 o = __ldcg(reinterpret_cast<const float4*>(a.part_o + (base + slot) * kHD) + lane);
        num.x += w * o.x;
        num.y += w * o.y;
        num.z += w * o.z;
        num.w += w * o.w;
      }
    }
    const float inv = 1.0f / den;
    __nv_bfloat162* o2 = reinterpret_cast<__nv_bfloat162*>(a.out + ((size_t)r * a.Hq + qh) * kHD) + 2 * lane;
    o2[0] = __floats2bfloat162_rn(num.x * inv, num.y * inv);
    o2[1] = __floats2bfloat162_rn(num.z * inv, num.w * inv);
  }
}

// Signal one more partial for (r, h); the completing warp merges.  Called by one full warp.
__device__ __forceinline__ void attn_arrive(const AttnArgs& a, int r, int h, int lane) {
  __threadfence();
  int old = 0;
  if (lane == 0) old = atomicAdd(a.cnt + r * a.Hkv + h, 1);
  old = __shfl_sync(0xffffffffu, old, 0);
  if (old == attn_expected(a, r) - 1) {
    __threadfence();
    attn_merge_warp(a, r, h, lane);
    if (lane == 0) a.cnt[r * a.Hkv + h] = 0;
  }
}

// Scores + softmax + P.V of one (row, kv head) against ntok tokens.  kp(tok)
// returns a pointer to K row tok (128 bf16), vp(tok) to V row tok.  Writes the
// partial of query heads h*REP .. h*REP+REP-1 into chunk slot `slot`.
// REP = Hq/Hkv is a template parameter and loops are only lightly unrolled:
// the code must stay small (the attention kernel runs cold out of the
// instruction cache once per layer).
template <int REP, typename KP, typename VP>
__device__ __forceinline__ void attn_rows_chunk(const AttnArgs& a, int r, int h, int slot, int ntok, const float* qs,
                                                KP kp, VP vp, int lane) {
  float s[4][REP];
#pragma unroll 1
  for (int j = 0; j < 4; ++j) {
    const int tk = lane + 32 * j;
    float acc[REP];
#pragma unroll
    for (int e = 0; e < REP; ++e) acc[e] = 0.f;
    if (tk < ntok) {
      const uint4* k4 = reinterpret_cast<const uint4*>(kp(tk));
#pragma unroll 2
      for (int d8 = 0; d8 < kHD / 8; ++d8) {
        const uint4 kv = k4[d8];
        const __nv_bfloat162* k2 = reinterpret_cast<const __nv_bfloat162*>(&kv);
        const float2 f0 = __bfloat1622float2(k2[0]), f1 = __bfloat1622float2(k2[1]);
        const float2 f2 = __bfloat1622float2(k2[2]), f3 = __bfloat1622float2(k2[3]);
#pragma unroll
        for (int e = 0; e < REP; ++e) {
          const float4 qa = *reinterpret_cast<const float4*>(qs + e * kHD + d8 * 8);
          const float4 qb = *reinterpret_cast<const float4*>(qs + e * kHD + d8 * 8 + 4);
          acc[e] += qa.x * f0.x + qa.y * f0.y + qa.z * f1.x + qa.w * f1.y + qb.x * f2.x + qb.y * f2.y +
                    qb.z * f3.x + qb.w * f3.y;
        }
      }
    }
#pragma unroll
    for (int e = 0; e < REP; ++e) {
      const float v = tk < ntok ? acc[e] * a.scale : -INFINITY;
      if (j == 0) s[0][e] = v;
      else if (j == 1) s[1][e] = v;
      else if (j == 2) s[2][e] = v;
      else s[3][e] = v;
    }
  }
  float m[REP], l[REP];
#pragma unroll
  for (int e = 0; e < REP; ++e) {
    m[e] = warp_max(fmaxf(fmaxf(s[0][e], s[1][e]), fmaxf(s[2][e], s[3][e])));
    float ps = 0.f;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      s[j][e] = s[j][e] == -INFINITY ? 0.f : expf(s[j][e] - m[e]);
      ps += s[j][e];
    }
    l[e] = warp_sum(ps);
  }
  float o[REP][4];
#pragma unroll
  for (int e = 0; e < REP; ++e) o[e][0] = o[e][1] = o[e][2] = o[e][3] = 0.f;
#pragma unroll 1
  for (int j = 0; j < 4; ++j) {
    const int t0 = 32 * j;
    if (t0 >= ntok) break;
    float pj[REP];
#pragma unroll
    for (int e = 0; e < REP; ++e) pj[e] = j == 0 ? s[0][e] : j == 1 ? s[1][e] : j == 2 ? s[2][e] : s[3][e];
    const int nt = min(32, ntok - t0);
#pragma unroll 4
    for (int u = 0; u < nt; ++u) {
      const __nv_bfloat162* v2 = reinterpret_cast<const __nv_bfloat162*>(vp(t0 + u)) + 2 * lane;
      const float2 a0 = __bfloat1622float2(v2[0]), a1 = __bfloat1622float2(v2[1]);
#pragma unroll
      for (int e = 0; e < REP; ++e) {
        const float pv = __shfl_sync(0xffffffffu, pj[e], u);
        o[e][0] += pv * a0.x;
        o[e][1] += pv * a0.y;
        o[e][2] += pv * a1.x;
        o[e][3] += pv * a1.y;
      }
    }
  }
#pragma unroll
  for (int e = 0; e < REP; ++e) {
    const size_t pidx = ((size_t)r * a.Hq + h * REP + e) * a.NC + slot;
    const float inv = 1.0f / l[e];
    reinterpret_cast<float4*>(a.part_o + pidx * kHD)[lane] =
        make_float4(o[e][0] * inv, o[e][1] * inv, o[e][2] * inv, o[e][3] * inv);
    if (lane == 0) {
      a.part_ml[pidx * 2] = m[e];
      a.part_ml[pidx * 2 + 1] = l[e];
    }
  }
}

constexpr int kAttnThreads = 256;
// K, V chunk + per-warp q (prefix path) / q, p, reductions (suffix path)
template <int REP>
struct AttnSmem {
  static constexpr int v = 2 * kAC * kKPad * 2 + 8 * (REP < 2 ? 2 : REP) * kHD * 4;
};

// One work item: a shared-prefix chunk (is_pre) or one slot's suffix chunk.
template <int REP>
__device__ __forceinline__ void attn_item(const AttnArgs& a, bool is_pre, int h, int c, int r_item, uint8_t* asmem,
                                          int sb) {
  __nv_bfloat16* Ks = reinterpret_cast<__nv_bfloat16*>(asmem);
  __nv_bfloat16* Vs = Ks + kAC * kKPad;
  float* qbuf = reinterpret_cast<float*>(Vs + kAC * kKPad);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  constexpr int rep = REP;
  float* qs = qbuf + warp * (REP < 2 ? 2 : REP) * kHD;
  auto load_q = [&](int r, int h) {
    for (int e = 0; e < rep; ++e) {
      const __nv_bfloat16* qp = a.q + ((size_t)r * a.Hq + h * rep + e) * kHD;
      const float2 f = __bfloat1622float2(reinterpret_cast<const __nv_bfloat162*>(qp)[lane]);
      const float2 g2 = __bfloat1622float2(reinterpret_cast<const __nv_bfloat162*>(qp)[lane + 32]);
      qs[e * kHD + 2 * lane] = f.x;
      qs[e * kHD + 2 * lane + 1] = f.y;
      qs[e * kHD + 64 + 2 * lane] = g2.x;
      qs[e * kHD + 64 + 2 * lane + 1] = g2.y;
    }
    __syncwarp();
  };
  if (is_pre) {
    // ---------------- shared-prefix chunk: staged once, scored by every live row
    const int tok0 = c * kPC, ntok = min(kPC, a.plen - tok0);
    {
      constexpr int NJ = kPC * (kHD / 8) / kAttnThreads;
      uint4 kk[NJ], vv[NJ];
#pragma unroll
      for (int j = 0; j < NJ; ++j) {
        const int i = threadIdx.x + j * kAttnThreads;
        const int tk = i >> 4, seg = i & 15;
        kk[j] = vv[j] = make_uint4(0, 0, 0, 0);
        if (tk < ntok) {
          kk[j] = __ldg(reinterpret_cast<const uint4*>(a.kpre + ((size_t)h * a.pcap + tok0 + tk) * kHD + seg * 8));
          vv[j] = __ldg(reinterpret_cast<const uint4*>(a.vpre + ((size_t)h * a.pcap + tok0 + tk) * kHD + seg * 8));
        }
      }
#pragma unroll
      for (int j = 0; j < NJ; ++j) {
        const int i = threadIdx.x + j * kAttnThreads;
        const int tk = i >> 4, seg = i & 15;
        *reinterpret_cast<uint4*>(Ks + tk * kKPad + seg * 8) = kk[j];
        *reinterpret_cast<uint4*>(Vs + tk * kKPad + seg * 8) = vv[j];
      }
    }
    __syncthreads();
    astamp(a, sb);
    for (int r = warp; r < a.rows; r += kAttnThreads / 32) {
      if (!a.row_active[r]) continue;
      int valid = ntok;
      if (a.prefill) valid = min(ntok, r + 1 - tok0);
      if (valid <= 0) continue;
      load_q(r, h);
      attn_rows_chunk<REP>(a, r, h, c, valid, qs, [&](int tk) { return Ks + tk * kKPad; },
                      [&](int tk) { return Vs + tk * kKPad; }, lane);
      attn_arrive(a, r, h, lane);
    }
    return;
  }
  // ---------------- per-slot suffix chunk: one CTA per (row, kv head, chunk)
  const int r = r_item;
  const int len = a.row_len[r];
  const int tok0 = c * kAC;
  if (tok0 >= len) return;
  const int ntok = min(kAC, len - tok0);
  const int32_t* pt_row = a.pagetab + (size_t)a.row_lid[r] * a.maxp;
  const size_t head_stride = (size_t)a.pt * kHD;
  // stage: every thread issues all of its 16-B loads before storing (8 K + 8 V pieces)
  {
    constexpr int NJ = kAC * (kHD / 8) / kAttnThreads;
    uint4 kk[NJ], vv[NJ];
#pragma unroll
    for (int j = 0; j < NJ; ++j) {
      const int i = threadIdx.x + j * kAttnThreads;  // kAC tokens x 16 pieces
      const int tk = i >> 4, seg = i & 15;
      kk[j] = vv[j] = make_uint4(0, 0, 0, 0);
      if (tk < ntok) {
        const int tok = tok0 + tk;
        const int page = __ldg(pt_row + tok / a.pt);
        const size_t base = (((size_t)page * 2) * a.Hkv + h) * head_stride + (size_t)(tok % a.pt) * kHD + seg * 8;
        kk[j] = __ldg(reinterpret_cast<const uint4*>(a.pool + base));
        vv[j] = __ldg(reinterpret_cast<const uint4*>(a.pool + base + (size_t)a.Hkv * head_stride));
      }
    }
#pragma unroll
    for (int j = 0; j < NJ; ++j) {
      const int i = threadIdx.x + j * kAttnThreads;
      const int tk = i >> 4, seg = i & 15;
      *reinterpret_cast<uint4*>(Ks + tk * kKPad + seg * 8) = kk[j];
      *reinterpret_cast<uint4*>(Vs + tk * kKPad + seg * 8) = vv[j];
    }
  }
  float* qsm = qbuf;                      // [rep][128]
  float* psm = qbuf + REP * kHD;          // [rep][128]
  float* red = psm + REP * kHD;           // [2][4][kMaxRep]
  for (int i = threadIdx.x; i < rep * kHD; i += kAttnThreads)
    qsm[i] = __bfloat162float(a.q[((size_t)r * a.Hq + h * rep) * kHD + i]);
  __syncthreads();
  astamp(a, sb);
  // scores: thread t < 128 owns token t
  const int t = threadIdx.x;
  float sc[REP];
#pragma unroll
  for (int e = 0; e < REP; ++e) sc[e] = -INFINITY;
  if (t < kAC) {
    float acc[REP];
#pragma unroll
    for (int e = 0; e < REP; ++e) acc[e] = 0.f;
    const uint4* k4 = reinterpret_cast<const uint4*>(Ks + t * kKPad);
#pragma unroll 2
    for (int d8 = 0; d8 < kHD / 8; ++d8) {
      const uint4 kv = k4[d8];
      const __nv_bfloat162* k2 = reinterpret_cast<const __nv_bfloat162*>(&kv);
      const float2 f0 = __bfloat1622float2(k2[0]), f1 = __bfloat1622float2(k2[1]);
      const float2 f2 = __bfloat1622float2(k2[2]), f3 = __bfloat1622float2(k2[3]);
#pragma unroll
      for (int e = 0; e < REP; ++e) {
        if (e < rep) {
          const float4 qa = *reinterpret_cast<const float4*>(qsm + e * kHD + d8 * 8);
          const float4 qb = *reinterpret_cast<const float4*>(qsm + e * kHD + d8 * 8 + 4);
          acc[e] += qa.x * f0.x + qa.y * f0.y + qa.z * f1.x + qa.w * f1.y + qb.x * f2.x + qb.y * f2.y +
                    qb.z * f3.x + qb.w * f3.y;
        }
      }
    }
    if (t < ntok) {
#pragma unroll
      for (int e = 0; e < REP; ++e) sc[e] = acc[e] * a.scale;
    }
  }
  // block max / sum over the 128 token threads (warps 0..3)
#pragma unroll
  for (int e = 0; e < REP; ++e)
    if (e < rep) {
      const float mw = warp_max(sc[e]);
      if (lane == 0 && warp < 4) red[warp * kMaxRep + e] = mw;
    }
  __syncthreads();
  float mrow[REP];
#pragma unroll
  for (int e = 0; e < REP; ++e)
    mrow[e] = fmaxf(fmaxf(red[0 * kMaxRep + e], red[1 * kMaxRep + e]), fmaxf(red[2 * kMaxRep + e], red[3 * kMaxRep + e]));
  float* red2 = red + 4 * kMaxRep;
#pragma unroll
  for (int e = 0; e < REP; ++e)
    if (e < rep) {
      const float p = (t < ntok) ? expf(sc[e] - mrow[e]) : 0.f;
      if (t < kAC) psm[e * kHD + t] = p;
      const float sw = warp_sum(p);
      if (lane == 0 && warp < 4) red2[warp * kMaxRep + e] = sw;
    }
  __syncthreads();
  // P.V: outputs (e, d) spread over the CTA
  for (int idx = threadIdx.x; idx < rep * kHD; idx += kAttnThreads) {
    const int e = idx / kHD, d = idx % kHD;
    float o = 0.f;
    const float* pe = psm + e * kHD;
#pragma unroll 8
    for (int tk = 0; tk < ntok; ++tk) o += pe[tk] * __bfloat162float(Vs[tk * kKPad + d]);
    const float l = red2[0 * kMaxRep + e] + red2[1 * kMaxRep + e] + red2[2 * kMaxRep + e] + red2[3 * kMaxRep + e];
    const size_t pidx = ((size_t)r * a.Hq + h * rep + e) * a.NC + a.nc_pre + c;
    a.part_o[pidx * kHD + d] = o / l;
    if (d == 0) {
      a.part_ml[pidx * 2] = mrow[e];
      a.part_ml[pidx * 2 + 1] = l;
    }
  }
  __syncthreads();
  astamp(a, sb + 1);
  if (warp == 0) attn_arrive(a, r, h, lane);
}


// Persistent over the work list: decode items come from sched_kernel (prefix
// chunks first, then every live slot's chunks); prefill items are the prefix
// chunks (causal).  Items never span a CTA boundary, so the merge counters see
// each (row, head) partial exactly once.
template <int REP>
__global__ void __launch_bounds__(kAttnThreads) attn_kernel(AttnArgs a) {
  pdl_launch_dependents();  // let the next kernel launch and prefetch now; it waits for our completion itself
  pdl_wait();
  extern __shared__ __align__(16) uint8_t asmem[];
  astamp(a, 0);
  if (threadIdx.x == 0 && a.n_pf > 0) {
    // Attention moves ~1% of the step's bytes and is latency-bound: use it to
    // pull the next GEMMs' weights into L2 (cp.async.bulk.prefetch, no smem).
    long long tot = 0;
    for (int i = 0; i < a.n_pf; ++i) tot += a.pf_bytes[i];
    const long long per = ((tot / gridDim.x) + 4095) & ~4095ll;
    long long lo = (long long)blockIdx.x * per, hi = min(tot, lo + per);
    long long base = 0;
    for (int i = 0; i < a.n_pf && lo < hi; ++i) {
      const long long e0 = base, e1 = base + a.pf_bytes[i];
      const long long s0 = max(lo, e0), s1 = min(hi, e1);
      for (long long o = s0; o < s1; o += 32768) {
        const unsigned sz = (unsigned)min(32768ll, s1 - o);
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a.pf_ptr[i] + (o - e0)), "r"(sz) : "memory");
      }
      base = e1;
    }
  }
  const int n = a.prefill ? a.Hkv * a.nc_pre : (int)*a.n_items;
  astamp(a, 1);
  int nit = 0;
  for (int it = blockIdx.x; it < n; it += gridDim.x) {
    int code;
    if (a.prefill) code = (int)(0x80000000u | ((it / a.nc_pre) << 8) | (it % a.nc_pre));
    else code = a.items[it];
    const bool is_pre = code < 0;
    int h, c, r = -1;
    if (is_pre) {
      h = (code >> 8) & 0xFF;
      c = code & 0xFF;
    } else {
      c = (code >> 16) & 0xFF;
      r = (code >> 8) & 0xFF;
      h = code & 0xFF;
    }
    attn_item<REP>(a, is_pre, h, c, r, asmem, nit < 4 ? 2 + 3 * nit : 14);
    __syncthreads();
    if (nit < 4) astamp(a, 2 + 3 * nit + 2);
    ++nit;
  }
  astamp(a, 15);
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
  ST_ATTN_ITEMS,   // length of the attention work list for the next step
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
  int32_t* attn_items;       // [Hkv * (nc_pre + row_cap * nc_suf)]
  int Hkv, nc_pre, nc_suf, chunk;
};

// Single thread: the work is O(g + pages) integer bookkeeping per step.
// consume = 1: take the sampled tokens of the step that just ran, finish /
// park / refill in ascending slot order (R18); then always prepare the rows of
// the next step (page allocation on boundary crossing, R26).
__global__ void sched_kernel(SchedArgs a, int consume) {
  pdl_launch_dependents();  // let the next kernel launch and prefetch now; it waits for our completion itself
  pdl_wait();
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
  // attention work list of the next step: shared-prefix chunks first (heavier:
  // every live row), then each live slot's suffix chunks, chunk-major.
  {
    int n = 0;
    if (any) {
      for (int h = 0; h < a.Hkv; ++h)
        for (int c = 0; c < a.nc_pre; ++c) a.attn_items[n++] = (int)(0x80000000u | (h << 8) | c);
      for (int c = 0; c < a.nc_suf; ++c)
        for (int s = 0; s < a.row_cap; ++s)
          if (a.row_active[s] && c * a.chunk < a.row_len[s])
            for (int h = 0; h < a.Hkv; ++h) a.attn_items[n++] = (c << 16) | (s << 8) | h;
    }
    st[ST_ATTN_ITEMS] = n;
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
  pdl_launch_dependents();  // let the next kernel launch and prefetch now; it waits for our completion itself
  pdl_wait();
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
