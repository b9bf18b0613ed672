// Non-GEMM kernels of the decode step: embedding, RMSNorm, split shared-prefix / per-slot-suffix attention with LSE merge,
// and the 1-CTA finish / refill / page-recycle scheduler.
#pragma once
#include "common.cuh"

namespace isk {

constexpr int kHD = 128;      // head_dim (all Qwen3 shapes, R1)
constexpr int kKPad = 136;    // smem row pitch (bf16) -> conflict-free 16-B row reads

// ------------------------------------------------------------------ embed
// resid[r][:] = E[tok[r]][:] (fp32 residual stream); idle rows get zeros.  Also the
// first layer's RMSNorm operands (R12b): xg[r][k] = bf16(x * gain[k]) and the
// per-128-column sums of squares ssq[t][r] the QKV GEMM derives rs[r] from.
// One CTA of 128 threads per row.
__global__ void embed_kernel(const __nv_bfloat16* __restrict__ E, const int32_t* __restrict__ row_tok,
                             const int32_t* __restrict__ row_active, float* __restrict__ resid, int H,
                             const float* __restrict__ gain, __nv_bfloat16* __restrict__ xg,
                             float* __restrict__ ssq, int ld_ssq) {
  pdl_launch_dependents();  // let the next kernel launch and prefetch now; it waits for our completion itself
  pdl_wait();
  __shared__ float red[4];
  const int r = blockIdx.x;
  const bool act = row_active[r] != 0;
  const __nv_bfloat16* e = E + (size_t)(act ? row_tok[r] : 0) * H;
  for (int t0 = 0; t0 < H; t0 += 128) {
    const int k = t0 + threadIdx.x;
    const float x = (act && k < H) ? __bfloat162float(e[k]) : 0.f;
    if (k < H) {
      resid[(size_t)r * H + k] = x;
      xg[(size_t)r * H + k] = __float2bfloat16_rn(x * gain[k]);
    }
    const float s2 = warp_sum(x * x);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s2;
    __syncthreads();
    if (threadIdx.x == 0) ssq[(size_t)(t0 / 128) * ld_ssq + r] = red[0] + red[1] + red[2] + red[3];
    __syncthreads();
  }
}

// ------------------------------------------------------------------ split attention
// PAPER.md l.171-174 / l.205: every live slot attends to the prompt's shared
// prefix KV (written once by prefill) and to its own paged response KV.  The
// work is split at that boundary (R8) and every part returns a normalised
// partial (o, m, l) per query head:
//   * prefix item = (kv head, kPC-token prefix chunk), one CTA: the chunk is
//     DMA'd into shared memory ONCE and every live row of the group (x Hq/Hkv
//     query heads) is scored against it -- the shared prefix is read once per
//     group per step, not once per slot;
//   * suffix item = (row, kv head, kSC-token chunk of that slot's pages), one
//     WARP with its own smem slice; the scheduler embeds the chunk's page ids in
//     the work item, so staging is one bulk DMA per (page, K|V) block.
// attn_merge_kernel then combines each (row, query head)'s partials by
// log-sum-exp in fixed order (prefix chunks, then suffix chunks).
// K/V tiles are dense in smem (bulk copies cannot pad); K rows are read with
// an XOR swizzle of the 16-byte chunk index (lane t reads chunk d8 ^ (t & 7)),
// which makes the lane-per-token score loop bank-conflict free.
// Loops stay rolled: this code runs cold out of the instruction cache once per
// layer, so code length is latency.
constexpr int kPC = 32;           // tokens per shared-prefix chunk (one CTA, all live rows)
constexpr int kSC = 64;           // tokens per suffix chunk (one warp)
constexpr int kMaxRep = 8;        // Hq / Hkv <= 8
constexpr int kItemStride = 20;   // work item (80 B, 16-B aligned): [0] code, [1] row length, [2..17] page ids
constexpr int kAttnWarps = 4;
constexpr int kAttnThreads = kAttnWarps * 32;

struct AttnArgs {
  const __nv_bfloat16* q;     // [rows][Hq][128]
  const __nv_bfloat16* kpre;  // prefix K of this layer [Hkv][pcap][128]
  const __nv_bfloat16* vpre;  // prefix V               [Hkv][pcap][128]
  const __nv_bfloat16* pool;  // page pool of this layer [pages][2][Hkv][pt][128]
  const int32_t* row_active;
  const int32_t* row_len;     // suffix tokens visible (t + 1)
  float* part_o;              // [rows][Hq][NC][128] normalised partial outputs
  float* part_ml;             // [rows][Hq][NC][2]   (max score, sum exp)
  const int32_t* items;       // decode work list (sched_kernel): prefix items, then suffix items
  const long long* n_items;   // [2]: total items, prefix items
  unsigned long long* dbg_ts; // optional [gridDim][16] globaltimer stamps
  __nv_bfloat16* out;         // [rows][Hq][128]
  float* out_f32;             // optional (is_dbg_attn): the merged output before the bf16 rounding (r4)
  int rows, Hq, Hkv, pcap, plen, pt;
  int nc_pre, nc_suf, NC;
  int prefill;                // 1: rows are prompt positions, causal over the prefix, no suffix
  int tc_prefix;              // decode: shared prefix done by attn_prefix_tc_kernel (tcgen05)
  int* merge_cnt;             // decode: [rows][Hkv] suffix units done; the last one merges (reset by it)
  int pool_row0;              // decode (mma suffix): page-pool tensor-map coordinate of this layer (page x head)
  int dbg_mode;               // timing experiments (is_dbg_attn, IS_DBG_SUFFIX_MODE): 1 no KV loads, 2 no math
  int* merge_done;            // decode (mma suffix): [rows][Hkv] query heads merged per pair
  int* unit_ctr;              // decode: [2] dynamic work fetching (next unit, warps / CTAs done; the last
                              //   finisher resets both for the next launch); null = static striding
  int sc;                     // decode suffix chunk (tokens per work item): kSC, or kSCW for the warp kernel
  const float* kmax;          // decode, tcgen05 prefix: max_t ||k_t|| per (kv head, 128-token tile) of this
  int kmax_grp;               //   layer (prefix_kmax_kernel, at prefill); group stride.  null: exact max
  int items_cap;              // decode (mma suffix): work items the buffer holds (speculative queue loads)
  int early_ctas;             // decode (mma suffix): CTAs [0, early_ctas) take the static units and the
                              //   merges; the rest (placed behind the prefix kernel's CTAs) only claim (0: all)
  int grp_rows;               // decode, tcgen05 prefix: rows per co-resident group (g); group m = rows m*g ..
  int grp_kv_rows;            //   prefix-KV tensor-map rows per group (L * 2 * Hkv * pcap)
  float scale;                // 1/sqrt(128)
};

__device__ __forceinline__ void astamp(const AttnArgs& a, int i) {
  if (a.dbg_ts && threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    a.dbg_ts[blockIdx.x * 16 + i] = t;
  }
}

__device__ __forceinline__ void astamp_lane(const AttnArgs& a, int i) {  // caller picks the thread
  if (a.dbg_ts) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    a.dbg_ts[blockIdx.x * 16 + i] = t;
  }
}

// 1-D bulk DMA global -> shared, completion (bytes) on an mbarrier.
IS_DEVICE void bulk_g2s(void* smem, const void* gmem, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(smem)),
               "l"(gmem), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

// q row r, heads h*REP.. -> smem fp32 [REP][128] (one 8-byte load per lane per head)
template <int REP>
__device__ __forceinline__ void attn_load_q(const AttnArgs& a, int r, int h, float* qs, int lane) {
  uint2 b[REP];
#pragma unroll
  for (int e = 0; e < REP; ++e) b[e] = reinterpret_cast<const uint2*>(a.q + ((size_t)r * a.Hq + h * REP + e) * kHD)[lane];
#pragma unroll
  for (int e = 0; e < REP; ++e) {
    const float2 f0 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&b[e].x));
    const float2 f1 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&b[e].y));
    reinterpret_cast<float4*>(qs + e * kHD)[lane] = make_float4(f0.x, f0.y, f1.x, f1.y);
  }
}

// Partial (m, l, o[REP][4 dims per lane]) of REP query heads over `ntok` dense
// K / V rows in shared memory, one warp.  TPL = tokens per lane-group: with
// ntok <= 32 each lane owns one token (TPL = 1); with ntok <= 16 two lanes
// share a token, each dotting half of the head dims (TPL = 2).  K chunks are
// read XOR-swizzled (chunk d8 ^ (token & 7)) -> conflict-free.
template <int REP, int LPT>
struct WarpPartial {
  float m[REP], l[REP], o[REP][4];
  __device__ __forceinline__ void run(const float* qs, const __nv_bfloat16* Ks, const __nv_bfloat16* Vs, int ntok,
                                      float scale, int lane) {
    constexpr int TOK = 32 / LPT;             // tokens covered by the warp
    const int tk = lane / LPT, part = lane % LPT;
    float acc[REP];
#pragma unroll
    for (int e = 0; e < REP; ++e) acc[e] = 0.f;
    if (tk < ntok) {
      const uint4* k4 = reinterpret_cast<const uint4*>(Ks + tk * kHD);
#pragma unroll 2
      for (int i = 0; i < 16 / LPT; ++i) {
        const int d8 = part * (16 / LPT) + i;
        const int cc = d8 ^ (tk & 7);
        const uint4 kv = k4[cc];
        const __nv_bfloat162* k2 = reinterpret_cast<const __nv_bfloat162*>(&kv);
        const float2 f0 = __bfloat1622float2(k2[0]), f1 = __bfloat1622float2(k2[1]);
        const float2 f2 = __bfloat1622float2(k2[2]), f3 = __bfloat1622float2(k2[3]);
#pragma unroll
        for (int e = 0; e < REP; ++e) {
          const float4 qa = *reinterpret_cast<const float4*>(qs + e * kHD + cc * 8);
          const float4 qb = *reinterpret_cast<const float4*>(qs + e * kHD + cc * 8 + 4);
          acc[e] += qa.x * f0.x + qa.y * f0.y + qa.z * f1.x + qa.w * f1.y + qb.x * f2.x + qb.y * f2.y +
                    qb.z * f3.x + qb.w * f3.y;
        }
      }
    }
    float p[REP];
#pragma unroll
    for (int e = 0; e < REP; ++e) {
#pragma unroll
      for (int sh = 1; sh < LPT; sh <<= 1) acc[e] += __shfl_xor_sync(0xffffffffu, acc[e], sh);
      const float sc = tk < ntok ? acc[e] * scale : -INFINITY;
      m[e] = warp_max(sc);
      p[e] = sc == -INFINITY ? 0.f : expf(sc - m[e]);
      l[e] = warp_sum(p[e]) / (float)LPT;
      o[e][0] = o[e][1] = o[e][2] = o[e][3] = 0.f;
    }
#pragma unroll 4
    for (int u = 0; u < min(ntok, TOK); ++u) {
      const __nv_bfloat162* v2 = reinterpret_cast<const __nv_bfloat162*>(Vs + u * kHD) + 2 * lane;
      const float2 a0 = __bfloat1622float2(v2[0]), a1 = __bfloat1622float2(v2[1]);
#pragma unroll
      for (int e = 0; e < REP; ++e) {
        const float pv = __shfl_sync(0xffffffffu, p[e], u * LPT);
        o[e][0] += pv * a0.x;
        o[e][1] += pv * a0.y;
        o[e][2] += pv * a1.x;
        o[e][3] += pv * a1.y;
      }
    }
  }
};

template <int REP>
__device__ __forceinline__ void store_partial(const AttnArgs& a, int r, int h, int slot, const float (&m)[REP],
                                              const float (&l)[REP], const float (&o)[REP][4], int lane) {
#pragma unroll
  for (int e = 0; e < REP; ++e) {
    const size_t pidx = ((size_t)r * a.Hq + h * REP + e) * a.NC + slot;
    const float inv = 1.0f / l[e];
    reinterpret_cast<float4*>(a.part_o + pidx * kHD)[lane] =
        make_float4(o[e][0] * inv, o[e][1] * inv, o[e][2] * inv, o[e][3] * inv);
    if (lane == 0) *reinterpret_cast<float2*>(a.part_ml + pidx * 2) = make_float2(m[e], l[e]);
  }
}

// smem per CTA: K [64][128] + V [64][128] (bf16, dense) + q [4][REP][128] fp32
// + combine scratch [4][REP][2 + 128] fp32 + DMA barrier.
template <int REP>
struct AttnSmem {
  static constexpr int kKV = 2 * kSC * kHD * 2;
  static constexpr int kQ = kAttnWarps * REP * kHD * 4;
  static constexpr int kComb = kAttnWarps * REP * (kHD + 2) * 4;
  static constexpr int v = kKV + kQ + kComb + 64;
};

// Merged output of (row r, query head qh): dims 4*lane..4*lane+3, rounded to bf16 (r4).
__device__ __forceinline__ void attn_store_out(const AttnArgs& a, int r, int qh, float4 o, int lane) {
  __nv_bfloat162* o2 = reinterpret_cast<__nv_bfloat162*>(a.out + ((size_t)r * a.Hq + qh) * kHD) + 2 * lane;
  o2[0] = __floats2bfloat162_rn(o.x, o.y);
  o2[1] = __floats2bfloat162_rn(o.z, o.w);
  if (a.out_f32) reinterpret_cast<float4*>(a.out_f32 + ((size_t)r * a.Hq + qh) * kHD)[lane] = o;
}

// LSE merge (R8) of one (row r, query head h*REP + j): lane i holds partial i's
// (m, l) (<= 32 partials); all o loads are issued together; fixed order.
template <int REP>
__device__ __forceinline__ void attn_merge_one(const AttnArgs& a, int r, int h, int j, int lane) {
  const int npre = a.nc_pre;
  const int nsuf = (a.row_len[r] + a.sc - 1) / a.sc;
  const int n = npre + nsuf;  // <= 64
  const int qh = h * REP + j;
  const size_t base = ((size_t)r * a.Hq + qh) * a.NC;
  // partial i lives in slot i (prefix) or nc_pre + (i - npre) (suffix): the same index
  float m0 = -INFINITY, l0 = 0.f, m1 = -INFINITY, l1 = 0.f;
  if (lane < n) {
    const float2 ml = __ldcg(reinterpret_cast<const float2*>(a.part_ml + (base + lane) * 2));
    m0 = ml.x;
    l0 = ml.y;
  }
  if (lane + 32 < n) {
    const float2 ml = __ldcg(reinterpret_cast<const float2*>(a.part_ml + (base + lane + 32) * 2));
    m1 = ml.x;
    l1 = ml.y;
  }
  // the first 32 partial outputs do not depend on the weights: in flight with the (m, l) loads
  // (one L2 round trip for up to 32 partials)
  constexpr int B = 32;
  float4 o[B];
#pragma unroll
  for (int k = 0; k < B; ++k)
    o[k] = k < n ? __ldcg(reinterpret_cast<const float4*>(a.part_o + (base + k) * kHD) + lane) : make_float4(0, 0, 0, 0);
  const float M = warp_max(fmaxf(m0, m1));
  const float w0 = (lane < n && m0 != -INFINITY) ? expf(m0 - M) * l0 : 0.f;
  const float w1 = (lane + 32 < n && m1 != -INFINITY) ? expf(m1 - M) * l1 : 0.f;
  const float den = warp_sum(w0) + warp_sum(w1);
  float4 num = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll 1
  for (int i0 = 0; i0 < n; i0 += B) {
    if (i0 > 0) {
#pragma unroll
      for (int k = 0; k < B; ++k)
        o[k] = i0 + k < n ? __ldcg(reinterpret_cast<const float4*>(a.part_o + (base + i0 + k) * kHD) + lane)
                          : make_float4(0, 0, 0, 0);
    }
#pragma unroll
    for (int k = 0; k < B; ++k) {
      const int i = i0 + k;
      const float wa = __shfl_sync(0xffffffffu, w0, i & 31), wb = __shfl_sync(0xffffffffu, w1, i & 31);
      const float w = i < 32 ? wa : wb;
      if (i < n) {
        num.x += w * o[k].x;
        num.y += w * o[k].y;
        num.z += w * o[k].z;
        num.w += w * o[k].w;
      }
    }
  }
  const float inv = 1.0f / den;
  attn_store_out(a, r, qh, make_float4(num.x * inv, num.y * inv, num.z * inv, num.w * inv), lane);
}

// Decode suffix pass behind the tcgen05 prefix kernel (every work item is a suffix
// chunk of kSCW tokens): one WARP per unit, each warp with its own staging buffer
// and mbarrier, so a CTA keeps kAttnWarps independent units in flight and an SM
// ~12 (the latency of a unit is its page DMA, the q load and the partial's store +
// count, not its arithmetic).  Lane t scores token t of the chunk (all 128 dims,
// REP heads); partials, counting and the fused LSE merge as in attn_kernel.
constexpr int kSCW = 32;
template <int REP>
struct SuffixWarpSmem {
  static constexpr int kWarp = 2 * kSCW * kHD * 2 + REP * kHD * 4;  // K, V [32][128] bf16 + q [REP][128] fp32
  static constexpr int v = kAttnWarps * kWarp + kAttnWarps * 8 + 64;
};

template <int REP>
__global__ void __launch_bounds__(kAttnThreads) attn_suffix_warp_kernel(AttnArgs a) {
  pdl_launch_dependents();
  using SM = SuffixWarpSmem<REP>;
  extern __shared__ __align__(128) uint8_t wsm[];
  __shared__ int merge_list[kAttnWarps][64];
  __shared__ int merge_n[kAttnWarps];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __nv_bfloat16* Ks = reinterpret_cast<__nv_bfloat16*>(wsm + warp * SM::kWarp);
  __nv_bfloat16* Vs = Ks + kSCW * kHD;
  float* qs = reinterpret_cast<float*>(Vs + kSCW * kHD);
  uint64_t* bar = reinterpret_cast<uint64_t*>(wsm + kAttnWarps * SM::kWarp) + warp;
  if (lane == 0) {
    mbar_init(bar, 1);
    fence_barrier_init();
    merge_n[warp] = 0;
  }
  __syncwarp();
  // Launched behind attn_prefix_tc_kernel, which triggers only after its wait on the
  // QKV GEMM: q and the appended KV are complete here.
  const int n = (int)a.n_items[0];
  const size_t hs = (size_t)a.pt * kHD;
  uint32_t phase = 0;
  const int stride = gridDim.x * kAttnWarps;
  // Units are taken dynamically (one atomic per unit): a warp whose CTA became resident
  // late (behind the prefix kernel's CTAs) or whose units were short simply takes more.
  auto next_unit = [&](int cur) {
    if (!a.unit_ctr) return cur + stride;
    int v = 0;
    if (lane == 0) v = atomicAdd(a.unit_ctr, 1);
    return __shfl_sync(0xffffffffu, v, 0);
  };
  // Software-pipelined over this warp's units: the next unit's item is read during the
  // current one, and its pages are DMA'd as soon as the current chunk has been scored
  // (the buffer is free), i.e. before the current partial's store / fence / count.
  // Item: [0] code (c << 16 | r << 8 | h), [1..8] page ids, [16] the row's length.
  int u = a.unit_ctr ? next_unit(0) : blockIdx.x * kAttnWarps + warp;
  int code = 0, len = 0, page_l = 0;
  auto fetch = [&](int uu) {
    const int32_t* item = a.items + (size_t)uu * kItemStride;
    code = item[0];
    len = item[1];
    page_l = lane < 8 ? item[2 + lane] : 0;
  };
  auto issue = [&]() {
    const int c = (code >> 16) & 0xFF, h = code & 0xFF;
    const int ntok = min(kSCW, len - c * kSCW);
    const int npg = (ntok + a.pt - 1) / a.pt;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // our buffer was last read generically
    if (lane == 0) mbar_arrive_expect_tx(bar, (uint32_t)ntok * kHD * 2 * 2);
    __syncwarp();
    if (lane < npg) {
      const uint32_t bytes = (uint32_t)min(a.pt, ntok - lane * a.pt) * kHD * 2;
      const __nv_bfloat16* kb = a.pool + (((size_t)page_l * 2) * a.Hkv + h) * hs;
      bulk_g2s(Ks + lane * a.pt * kHD, kb, bytes, bar);
      bulk_g2s(Vs + lane * a.pt * kHD, kb + (size_t)a.Hkv * hs, bytes, bar);
    }
  };
  if (u < n) {
    fetch(u);
    issue();
  }
#pragma unroll 1
  while (u < n) {
    const int c = (code >> 16) & 0xFF, r = (code >> 8) & 0xFF, h = code & 0xFF;
    const int cur_len = len;
    const int ntok = min(kSCW, cur_len - c * kSCW);
    attn_load_q<REP>(a, r, h, qs, lane);
    const int nu = next_unit(u);
    if (nu < n) fetch(nu);  // independent loads, in flight during the wait + math
    __syncwarp();
    mbar_wait(bar, phase);
    phase ^= 1;
    WarpPartial<REP, 1> wp;
    wp.run(qs, Ks, Vs, ntok, a.scale, lane);
    __syncwarp();          // every lane is done reading the buffer
    if (nu < n) issue();   // next unit's pages overlap this unit's store / fence / count
    store_partial<REP>(a, r, h, a.nc_pre + c, wp.m, wp.l, wp.o, lane);
    __threadfence();
    __syncwarp();
    if (lane == 0) {
      const int nsuf = (cur_len + kSCW - 1) / kSCW;
      if (atomicAdd(a.merge_cnt + r * a.Hkv + h, 1) + 1 == nsuf) {
        __threadfence();
        a.merge_cnt[r * a.Hkv + h] = 0;  // ready for the next launch
        if (merge_n[warp] < 64) merge_list[warp][merge_n[warp]++] = (r << 8) | h;
      }
    }
    __syncwarp();
    u = nu;
  }
  if (a.unit_ctr && lane == 0 && atomicAdd(a.unit_ctr + 1, 1) == stride - 1) {
    a.unit_ctr[0] = 0;  // every warp has taken its last unit: ready for the next launch
    a.unit_ctr[1] = 0;
  }
  pdl_wait();  // the tcgen05 prefix partials are complete from here on
  const int nm = merge_n[warp];
  for (int j = 0; j < nm * REP; ++j) {
    const int rh = merge_list[warp][j / REP];
    attn_merge_one<REP>(a, rh >> 8, rh & 0xFF, j % REP, lane);
  }
}

// ------------------------------------------------------------------ suffix pass on mma.sync
// Decode suffix pass behind the tcgen05 prefix kernel ("a separate
// KV buffer for its response tokens"): unit = (row r, kv head h, 32-token chunk c of the slot's
// pages).  One CTA per SM of kSWarps independent warps; each warp runs its own kSWStages-deep
// ring: it TMA-loads a unit's pages (one 5-D box per page = K and V, both 64-dim halves, 128-byte
// swizzle) and the row's REP query heads into a stage, and while later units load it scores the
// oldest one on the tensor cores with warp-level mma.sync m16n8k16 (the REP query heads padded to
// the MMA's 16 rows: S = Q.K^T with the keys in N), takes the row softmax in registers (quad
// shuffles) and accumulates O = P.V with P as a bf16 hi/lo pair (two MMAs, ~2^-16 relative, like
// the prefix kernel).  The normalised partial (o, m, l) goes to partial slot nc_pre + c; the
// partials are released in batches (one fence per batch) and counted per (row, kv head), whose
// LSE merge runs after the prefix kernel is known complete, spread over the grid.
// Units: the first kSStaticPct% of the work list is split statically over the warps (contiguous
// ranges), the rest is claimed kSClaim units at a time (one atomic), so warps of CTAs that became
// resident late (behind the prefix kernel's CTAs) just claim less.
constexpr int kSUnit = 32;          // keys per unit
// Two shapes (template parameters NW warps x NST stages per warp): 6 x 2 (double-buffered; large
// launches) and 8 x 1 (more units in flight at once when every warp has only one or two units,
// e.g. one group of 16 rows).  The launcher picks by row capacity.
constexpr int kSQueue = 6;          // work items loaded ahead of their issue
constexpr int kSPublish = 8;        // units per release batch (one fence)
constexpr int kSStaticPct = 50;     // share of the work list split statically over the warps
// Sized so that the 8 x 1 shape (<= 16 rows) shares an SM with a tcgen05 prefix CTA
// (PrefixTcSmem<16>): every suffix CTA starts at once instead of behind the prefix kernel.
template <int NW, int NST, int REP>
struct SuffixMmaSmem {
  static constexpr int kKV = kSUnit * 2 * kHD * 2;    // K and V of one unit: 16 KB
  static constexpr int kQ = REP <= 4 ? 1024 : 2048;   // the row's REP query heads (bf16)
  static constexpr int kStage = kKV + kQ;             // 17 or 18 KB, a multiple of 1024 (swizzle atoms)
  static constexpr int v = NW * NST * kStage + 16 + NW * NST * 8 + 1024;
};

IS_DEVICE void ldsm_x4(uint32_t addr, uint32_t (&r)[4]) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(addr));
}
IS_DEVICE void ldsm_x4_t(uint32_t addr, uint32_t (&r)[4]) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(addr));
}
// D (16x8 fp32) += A (16x16 bf16, row) . B (16x8 bf16, col)
IS_DEVICE void mma16816(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
IS_DEVICE uint32_t pack_bf16(float lo, float hi) {
  const __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<const uint32_t*>(&v);
}
// 5-D tiled load (box = one page: K and V, both halves): coordinates innermost first.
IS_DEVICE void tma_load_5d(void* dst, const CUtensorMap* m, uint64_t* bar, int c0, int c1, int c2, int c3, int c4,
                           uint64_t cache_hint) {
  asm volatile(
      "cp.async.bulk.tensor.5d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%3, %4, %5, %6, %7}], [%2], %8;" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4),
      "l"(cache_hint)
      : "memory");
}

template <int REP, int PT, int NW, int NST>
__global__ void __launch_bounds__(32 * NW, 1) attn_suffix_mma_kernel(const __grid_constant__ CUtensorMap tmPool,
                                                                      AttnArgs a) {
  pdl_launch_dependents();
  using SM = SuffixMmaSmem<NW, NST, REP>;
  constexpr int kSWarps = NW, kSWStages = NST;
  extern __shared__ uint8_t sm_raw[];
  uint8_t* sm = align1024_smem(sm_raw);
  uint4* zero16 = reinterpret_cast<uint4*>(sm + kSWarps * kSWStages * SM::kStage);  // Q padding rows
  uint64_t* bars = reinterpret_cast<uint64_t*>(zero16 + 1);
  __shared__ int done_list[kSWarps * 32];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    astamp_lane(a, 0);
    for (int i = 0; i < kSWarps * kSWStages; ++i) mbar_init(&bars[i], 1);
    *zero16 = make_uint4(0, 0, 0, 0);
    tma_prefetch_desc(&tmPool);
    fence_barrier_init();
  }
  __syncthreads();
  const int n = (int)a.n_items[0];
  // speculative static-queue loads (items gw + q * GW of this warp, independent of n: one L2 round
  // trip instead of two before the first unit issues); validated against the static range below
  uint4 x0 = make_uint4(0xFFFFFFFFu, 0, 0, 0);
  uint2 x1 = make_uint2(0, 0);
  {
    const int early0 = a.early_ctas > 0 ? min(a.early_ctas, (int)gridDim.x) : (int)gridDim.x;
    const int u = (blockIdx.x * NW + (threadIdx.x >> 5)) + (threadIdx.x & 31) * early0 * NW;
    if ((int)blockIdx.x < early0 && a.items_cap > 0 && (threadIdx.x & 31) < kSQueue && u < a.items_cap) {
      const uint4* it = reinterpret_cast<const uint4*>(a.items + (size_t)u * kItemStride);
      x0 = it[0];
      const uint4 y = it[1];
      x1 = make_uint2(y.x, y.y);
    }
  }
  constexpr int pt = PT;  // page tokens (8, 16 or 32): the stage addressing is compile-time
  uint8_t* wsm = sm + warp * kSWStages * SM::kStage;
  uint64_t* full = bars + warp * kSWStages;
  // ---- unit source.  Units u < Ls are strided statically over the warps (warp gw: gw, gw + GW,
  // ...; their items are prefetched kSQueue deep), units >= Ls are claimed one at a time from a
  // counter, one unit ahead (claim + item load overlap the current unit's math; a warp never
  // hoards more than one unit, so the tail stays short).  Small work lists are all static.
  const bool loads = !(a.dbg_mode & 1), qload = !(a.dbg_mode & 4);
  const int early = a.early_ctas > 0 ? min(a.early_ctas, (int)gridDim.x) : (int)gridDim.x;
  const bool is_early = (int)blockIdx.x < early;
  const int GW = early * kSWarps, gw = blockIdx.x * kSWarps + warp;
  const int Ls = n <= 2 * GW ? n : (int)((long long)n * kSStaticPct / 100);
  int snext = is_early ? gw : Ls;  // next static unit to load into the queue
  // static queue: lane q < kSQueue holds the item (code, length, pages 0..3) of the q-th next static
  // unit (x0, x1 above); code -1 = none
  auto load_to = [&](int u, int q, uint4& y0, uint2& y1) {
    if (lane == q) {
      y0 = make_uint4(0xFFFFFFFFu, 0, 0, 0);
      y1 = make_uint2(0, 0);
      if (u < n) {
        const uint4* it = reinterpret_cast<const uint4*>(a.items + (size_t)u * kItemStride);
        y0 = it[0];
        const uint4 y = it[1];
        y1 = make_uint2(y.x, y.y);
      }
    }
  };
  if (is_early && a.items_cap > 0) {
    // the first kSQueue static items were loaded speculatively above (before the item count
    // arrived); drop those past the static range
    if (lane < kSQueue && gw + lane * GW >= Ls) x0 = make_uint4(0xFFFFFFFFu, 0, 0, 0);
    snext += kSQueue * GW;
  } else {
#pragma unroll 1
    for (int q = 0; q < kSQueue; ++q, snext += GW) load_to(snext < Ls ? snext : n, q, x0, x1);
  }
  // dynamic: lane 0 holds the item of the next claimed unit (d0.x = -1: none / not claimed yet)
  uint4 d0 = make_uint4(0xFFFFFFFFu, 0, 0, 0);
  uint2 d1 = make_uint2(0, 0);
  bool dyn_started = false, dyn_done = Ls >= n;
  auto claim_next = [&]() {  // claim one unit and load its item into lane 0's dynamic slot
    int u = n;
    if (lane == 0) u = Ls + atomicAdd(a.unit_ctr, 1);
    u = __shfl_sync(0xffffffffu, u, 0);
    if (u >= n) dyn_done = true;
    load_to(u, 0, d0, d1);
  };
  // issue the next unit into stage st: returns its code (-1 if there is none) and its row length
  auto issue = [&](int st, int& len_out) {
    int cd = __shfl_sync(0xffffffffu, (int)x0.x, 0);
    uint4 h0;
    uint2 h1;
    if (cd >= 0) {  // static queue head; shift and refill the tail
      h0 = make_uint4(x0.x, x0.y, x0.z, x0.w);
      h1 = x1;
      x0.x = __shfl_down_sync(0xffffffffu, x0.x, 1);
      x0.y = __shfl_down_sync(0xffffffffu, x0.y, 1);
      x0.z = __shfl_down_sync(0xffffffffu, x0.z, 1);
      x0.w = __shfl_down_sync(0xffffffffu, x0.w, 1);
      x1.x = __shfl_down_sync(0xffffffffu, x1.x, 1);
      x1.y = __shfl_down_sync(0xffffffffu, x1.y, 1);
      load_to(snext < Ls ? snext : n, kSQueue - 1, x0, x1);
      snext += GW;
      if (!dyn_started && !dyn_done && __shfl_sync(0xffffffffu, (int)x0.x, 0) < 0) {
        dyn_started = true;  // the static queue has run dry behind this unit: claim the first dynamic one
        claim_next();
      }
    } else {
      if (!dyn_started && !dyn_done) {
        dyn_started = true;
        claim_next();
      }
      cd = __shfl_sync(0xffffffffu, (int)d0.x, 0);
      h0 = d0;
      h1 = d1;
      if (cd >= 0 && !dyn_done) claim_next();  // one unit ahead
      else if (cd >= 0) d0.x = 0xFFFFFFFFu;
    }
    const int ln = __shfl_sync(0xffffffffu, (int)h0.y, 0);
    len_out = ln;
    if (cd < 0) return -1;
    const int p0 = __shfl_sync(0xffffffffu, (int)h0.z, 0), p1 = __shfl_sync(0xffffffffu, (int)h0.w, 0);
    const int p2 = __shfl_sync(0xffffffffu, (int)h1.x, 0), p3 = __shfl_sync(0xffffffffu, (int)h1.y, 0);
    const int c = (cd >> 16) & 0xFF, r = (cd >> 8) & 0xFF, h = cd & 0xFF;
    const int ntok = min(kSUnit, ln - c * kSUnit);
    const int npl = (((ntok + 15) & ~15) + pt - 1) / pt;  // pages covering the 16-key MMA steps (<= 4)
    uint8_t* stg = wsm + st * SM::kStage;
    if (lane == 0) {
      mbar_arrive_expect_tx(&full[st], (loads ? (uint32_t)npl * pt * 512 : 0u) + (qload ? REP * kHD * 2 : 0));
      if (qload) bulk_g2s(stg + SM::kKV, a.q + ((size_t)r * a.Hq + h * REP) * kHD, REP * kHD * 2, &full[st]);
      if (loads) {
#pragma unroll
        for (int j = 0; j < 4; ++j) {  // box (64 dims, 2 halves, pt rows, K|V, page x head)
          const int pg = j == 0 ? p0 : (j == 1 ? p1 : (j == 2 ? p2 : p3));
          if (j < npl)
            tma_load_5d(stg + j * pt * 512, &tmPool, &full[st], 0, 0, 0, 0, a.pool_row0 + pg * 2 * a.Hkv + h,
                        kEvictFirst);
        }
      }
    }
    return cd;
  };
  // Finite stale rows (see consume): a unit always loads its first page, and masked keys only
  // need finite V rows (their scores are replaced by -inf, their P is 0), so only the V rows of
  // pages 1.. of each stage are zeroed (stale later on = earlier units' V, finite); the K rows
  // and the rest of the stage are left as they are.  (dbg 64: the whole stage, as before)
  if (a.dbg_mode & 64) {
    for (int i = lane; i < kSWStages * SM::kStage / 16; i += 32) reinterpret_cast<uint4*>(wsm)[i] = make_uint4(0, 0, 0, 0);
  } else {
#pragma unroll 1
    for (int s = 0; s < kSWStages; ++s)
#pragma unroll 1
      for (int j = 1; j < kSUnit / pt; ++j) {
        uint4* vb = reinterpret_cast<uint4*>(wsm + s * SM::kStage + (2 * j * pt + pt) * 256);
        for (int i = lane; i < pt * 256 / 16; i += 32) vb[i] = make_uint4(0, 0, 0, 0);
      }
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // before the TMA writes
  __syncwarp();
  static_assert(kSWStages == 1 || kSWStages == 2, "the consume loop is unrolled over one or two stages");
  int hc0, hl0, hc1 = -1, hl1 = 0;  // per stage: the unit's code (-1: none) and row length
  hc0 = issue(0, hl0);
  if (kSWStages == 2) hc1 = issue(1, hl1);
  int nq = (hc0 >= 0) + (hc1 >= 0);  // units issued
  // ---- consume in order; refill the freed stage
  const int g = lane >> 2, t4 = lane & 3, mi = lane >> 3, mr = lane & 7;
  const float sl2 = a.scale * 1.4426950408889634f;  // exp(x * scale) = exp2(x * sl2)
  const uint32_t z16 = smem_u32(zero16);
  int* dl = done_list + warp * 32;  // this warp's finished units, published in batches (one fence each)
  int ndl = 0;
  auto publish = [&]() {
    __syncwarp();
    __threadfence();
    if (lane < ndl) atomicAdd(a.merge_cnt + dl[lane], 1);
    __syncwarp();
    ndl = 0;
  };
  // key row k of a stage (page k / pt, row k % pt) of K (kv = 0) or V (kv = 1): byte offset of its
  // 256-B row; the 128-B half h of that row sits at + 128 h, its 16-B chunk c at ^ swizzle
  auto krow = [&](int k0, int kv) { return (2 * k0 - (k0 & (pt - 1)) + kv * pt) * 256; };
  const int qrow = mr + 8 * (mi & 1);
  // Every unit computes all kSUnit keys (keys past the row's length are masked to -inf, p = 0):
  // no per-fragment branches.  The stages were zero-filled at launch and only ever hold finite KV,
  // so a key row that was not loaded for this unit still contributes 0 * finite.
  auto consume = [&](const int st, const int ph, int& hc, int& hl) -> bool {
    const int cd = hc;
    if (cd < 0) return false;
    mbar_wait(&full[st], ph);
    const int c = (cd >> 16) & 0xFF, r = (cd >> 8) & 0xFF, h = cd & 0xFF;
    const int ntok = (a.dbg_mode & 2) ? 0 : min(kSUnit, hl - c * kSUnit);
    const uint32_t sKV = smem_u32(wsm + st * SM::kStage), sQ = sKV + SM::kKV;
    constexpr int NJ = kSUnit / 8, NKK = kSUnit / 16;  // 8-key n-tiles of S, 16-key k-steps of P.V
    // S = Q . K^T: NJ n-tiles of 8 keys, 8 k-steps of 16 dims (taken in pairs)
    float sacc[NJ][4];
#pragma unroll
    for (int j = 0; j < NJ; ++j) sacc[j][0] = sacc[j][1] = sacc[j][2] = sacc[j][3] = 0.f;
    const uint32_t qbase = qrow < REP ? sQ + qrow * 256 + 16 * (mi >> 1) : z16;
    const uint32_t qstep = qrow < REP ? 32u : 0u;
#pragma unroll
    for (int kp = 0; kp < 4; ++kp) {
      uint32_t qa[2][4];
      ldsm_x4(qbase + (2 * kp) * qstep, qa[0]);
      ldsm_x4(qbase + (2 * kp + 1) * qstep, qa[1]);
      // chunk (kp & 1) * 4 + mi of half kp >> 1; the 128-B row index of key k, half h is 2k + h
      const int hh = kp >> 1;
      const uint32_t sw = ((((kp & 1) * 4 + mi) ^ ((2 * mr + hh) & 7)) << 4) + hh * 128 + mr * 256;
#pragma unroll
      for (int j = 0; j < NJ; ++j) {
        uint32_t kb[4];
        ldsm_x4(sKV + krow(8 * j, 0) + sw, kb);
        mma16816(sacc[j], qa[0], kb[0], kb[1]);
        mma16816(sacc[j], qa[1], kb[2], kb[3]);
      }
    }
    // row softmax: thread holds rows g (sacc[.][0..1]) and g + 8 (sacc[.][2..3], always a padding
    // row: REP <= 8), keys 8j + 2 t4 + {0,1}; the quad (t4) shares a row
    float mA = -INFINITY;
#pragma unroll
    for (int j = 0; j < NJ; ++j) {
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        sacc[j][e] = 8 * j + 2 * t4 + e < ntok ? sacc[j][e] : -INFINITY;
        mA = fmaxf(mA, sacc[j][e]);
      }
    }
    mA = fmaxf(mA, __shfl_xor_sync(0xffffffffu, mA, 1));
    mA = fmaxf(mA, __shfl_xor_sync(0xffffffffu, mA, 2));
    const float mb = mA * sl2;
    float lA = 0.f;
#pragma unroll
    for (int j = 0; j < NJ; ++j) {
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        sacc[j][e] = exp2f(fmaf(sacc[j][e], sl2, -mb));  // masked keys: exp2(-inf) = 0
        lA += sacc[j][e];
      }
    }
    lA += __shfl_xor_sync(0xffffffffu, lA, 1);
    lA += __shfl_xor_sync(0xffffffffu, lA, 2);
    // O = P . V, P = P_hi + P_lo (bf16 pair): NKK k-steps of 16 keys, 16 n-tiles of 8 dims; the
    // padding rows g + 8 enter as zeros
    float oacc[16][4];
#pragma unroll
    for (int j = 0; j < 16; ++j) oacc[j][0] = oacc[j][1] = oacc[j][2] = oacc[j][3] = 0.f;
#pragma unroll
    for (int kk = 0; kk < NKK; ++kk) {
      // A fragment: a0 (row g, keys 0-7 of the step) = n-tile 2kk, a2 (row g, keys 8-15) = 2kk+1;
      // a1 / a3 (row g + 8) = 0
      uint32_t ph[4], pl[4];
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        const float* sv = sacc[2 * kk + q];
        const __nv_bfloat162 hi = __floats2bfloat162_rn(sv[0], sv[1]);
        const float2 hf = __bfloat1622float2(hi);
        ph[2 * q] = *reinterpret_cast<const uint32_t*>(&hi);
        pl[2 * q] = pack_bf16(sv[0] - hf.x, sv[1] - hf.y);
        ph[2 * q + 1] = 0u;
        pl[2 * q + 1] = 0u;
      }
      // ldmatrix.trans rows: key 16kk + 8 (mi & 1) + mr; n-tiles nt, nt + 1 (mi >> 1)
      const uint32_t vb0 = sKV + krow(16 * kk + 8 * (mi & 1), 1) + mr * 256;
#pragma unroll
      for (int nt = 0; nt < 16; nt += 2) {
        const int hh = nt >> 3;
        uint32_t vb[4];
        ldsm_x4_t(vb0 + hh * 128 + ((((nt & 7) + (mi >> 1)) ^ ((2 * mr + hh) & 7)) << 4), vb);
        mma16816(oacc[nt], ph, vb[0], vb[1]);
        mma16816(oacc[nt + 1], ph, vb[2], vb[3]);
        mma16816(oacc[nt], pl, vb[0], vb[1]);
        mma16816(oacc[nt + 1], pl, vb[2], vb[3]);
      }
    }
    __syncwarp();  // every lane is done reading the stage: refill it
    hc = issue(st, hl);
    nq += hc >= 0;
    // partial of the unit for the real rows g < REP (published with the batch's fence)
    if (g < REP && !(a.dbg_mode & 8)) {
      const float inv = 1.0f / lA;
      const size_t pidx = ((size_t)r * a.Hq + h * REP + g) * a.NC + a.nc_pre + c;
      float2* po = reinterpret_cast<float2*>(a.part_o + pidx * kHD) + t4;
#pragma unroll
      for (int nt = 0; nt < 16; ++nt) po[4 * nt] = make_float2(oacc[nt][0] * inv, oacc[nt][1] * inv);
      if (t4 == 0) *reinterpret_cast<float2*>(a.part_ml + pidx * 2) = make_float2(mA * a.scale, lA);
    }
    if (lane == 0) dl[ndl] = r * a.Hkv + h;
    if (++ndl == kSPublish) publish();
    return true;
  };
  if (lane == 0) astamp_lane(a, 3);
#pragma unroll 1
  for (int ph = 0;; ph ^= 1) {
    if (!consume(0, ph, hc0, hl0)) break;
    if (kSWStages == 2 && !consume(1, ph, hc1, hl1)) break;
  }
  publish();
  if (lane == 0) {
    if (warp == 0) astamp_lane(a, 2);
    if (a.dbg_ts) atomicAdd(reinterpret_cast<int*>(a.dbg_ts + blockIdx.x * 16 + 9), nq);
  }
  // each warp moves on to its merges as soon as its own units are published (no CTA barrier)
  if (lane == 0 && atomicAdd(a.unit_ctr + 1, 1) == (int)gridDim.x * kSWarps - 1) {
    a.unit_ctr[0] = 0;  // every warp has taken its last unit: ready for the next launch
    a.unit_ctr[1] = 0;
  }
  if (threadIdx.x == 0) astamp_lane(a, 6);
  pdl_wait();  // the tcgen05 prefix partials are complete from here on
  if (threadIdx.x == 0) astamp_lane(a, 7);
  // LSE merge (R8): (row, kv head) pair i is merged by warp i / grid of CTA i % grid, spread over
  // the whole grid; it waits (acquire) until all the pair's units are counted.  No deadlock: units
  // are taken only by running CTAs, which finish them without waiting on anything.
  // (one query head of a pair per warp: the REP heads of a pair merge concurrently; the last of
  // them re-arms the pair's counters)
  const int npairs = a.rows * a.Hkv;
  int nm = 0;
  // merges packed onto the first CTAs (all their warps), so the other CTAs exit right after
  // their units and free their SMs for the o_proj GEMM's CTAs, which then stream their weights
  // during the merges
  const int nmc = min(early, (npairs * REP + kSWarps - 1) / kSWarps);
  for (int k = (is_early && (int)blockIdx.x < nmc) ? blockIdx.x * kSWarps + warp : npairs * REP; k < npairs * REP;
       k += nmc * kSWarps) {
    const int i = k / REP, e = k - i * REP;
    const int r = i / a.Hkv, h = i - r * a.Hkv;
    if (!a.row_active[r]) continue;
    const int nsuf = (a.row_len[r] + kSUnit - 1) / kSUnit;
    int cnt;
    while (true) {
      asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(cnt) : "l"(a.merge_cnt + i) : "memory");
      if (cnt >= nsuf) break;
      __nanosleep(128);
    }
    attn_merge_one<REP>(a, r, h, e, lane);
    if (lane == 0 && atomicAdd(a.merge_done + i, 1) == REP - 1) {
      a.merge_cnt[i] = 0;  // ready for the next launch
      a.merge_done[i] = 0;
    }
    ++nm;
  }
  if (a.dbg_ts) {
    __syncthreads();
    if (threadIdx.x == 0) {
      astamp_lane(a, 8);
      a.dbg_ts[blockIdx.x * 16 + 10] = nm;
    }
  }
}

// Work units (persistent grid, ~4 CTAs per SM):
//   prefix (h, c, g): DMA the kPC-token prefix chunk once; warp w scores row
//                     4g + w (all of its REP heads) -> partial slot c;
//   suffix (r, h, c): DMA the slot's kSC-token chunk (<= 4 pages); warp w takes
//                     page w (16 tokens, two lanes per token) and the 4 warp
//                     partials are combined in smem -> partial slot nc_pre + c.
template <int REP>
__global__ void __launch_bounds__(kAttnThreads) attn_kernel(AttnArgs a) {
  pdl_launch_dependents();
  extern __shared__ __align__(128) uint8_t asmem[];
  using SM = AttnSmem<REP>;
  __nv_bfloat16* Ks = reinterpret_cast<__nv_bfloat16*>(asmem);
  __nv_bfloat16* Vs = Ks + kSC * kHD;
  float* qs_all = reinterpret_cast<float*>(asmem + SM::kKV);
  float* comb = reinterpret_cast<float*>(asmem + SM::kKV + SM::kQ);
  uint64_t* bar = reinterpret_cast<uint64_t*>(asmem + SM::kKV + SM::kQ + SM::kComb);
  __shared__ int merge_list[128];
  __shared__ int merge_n;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) merge_n = 0;
  float* qs = qs_all + warp * REP * kHD;
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    fence_barrier_init();
  }
  __syncthreads();
  // Decode: launched behind attn_prefix_tc_kernel, which triggers only after the
  // QKV GEMM completed -> our inputs are ready; we wait for the prefix kernel at
  // the END so the merge kernel (which waits for us) sees both parts.
  if (a.prefill || !a.tc_prefix) pdl_wait();
  astamp(a, 0);
  const int n = a.prefill ? a.Hkv * a.nc_pre * ((a.rows + kAttnWarps - 1) / kAttnWarps) : (int)a.n_items[0];
  uint32_t phase = 0;
  int nu = 0;
  __shared__ int s_unit;
  const bool dyn = !a.prefill && a.unit_ctr;  // decode: units taken dynamically (see the warp kernel)
#pragma unroll 1
  for (int u = blockIdx.x;; ++nu) {
    if (dyn) {
      if (threadIdx.x == 0) s_unit = atomicAdd(a.unit_ctr, 1);
      __syncthreads();
      u = s_unit;
    } else if (nu > 0) {
      u += gridDim.x;
    }
    if (u >= n) break;
    if (nu < 3) astamp(a, 1 + 4 * nu);
    int code;
    if (a.prefill) {
      const int ng = (a.rows + kAttnWarps - 1) / kAttnWarps;
      code = (int)(0x80000000u | ((u / (a.nc_pre * ng)) << 16) | (((u / ng) % a.nc_pre) << 8) | (u % ng));
    } else {
      code = a.items[(size_t)u * kItemStride];
    }
    if (code < 0) {
      // ---------------- shared-prefix chunk, one row per warp
      const int h = (code >> 16) & 0xFF, c = (code >> 8) & 0xFF, g = code & 0xFF;
      const int tok0 = c * kPC, ntok = min(kPC, a.plen - tok0);
      if (threadIdx.x == 0) {
        const uint32_t bytes = (uint32_t)ntok * kHD * 2;
        mbar_arrive_expect_tx(bar, 2 * bytes);
        bulk_g2s(Ks, a.kpre + ((size_t)h * a.pcap + tok0) * kHD, bytes, bar);
        bulk_g2s(Vs, a.vpre + ((size_t)h * a.pcap + tok0) * kHD, bytes, bar);
      }
      const int r = g * kAttnWarps + warp;
      const bool act = r < a.rows && a.row_active[r];
      const int valid = act ? (a.prefill ? min(ntok, r + 1 - tok0) : ntok) : 0;
      if (valid > 0) attn_load_q<REP>(a, r, h, qs, lane);
      __syncwarp();
      mbar_wait(bar, phase);
      if (nu < 3) astamp(a, 2 + 4 * nu);
      if (valid > 0) {
        WarpPartial<REP, 1> wp;
        wp.run(qs, Ks, Vs, valid, a.scale, lane);
        store_partial<REP>(a, r, h, c, wp.m, wp.l, wp.o, lane);
      }
    } else {
      // ---------------- per-slot suffix chunk, one page per warp
      const int c = (code >> 16) & 0xFF, r = (code >> 8) & 0xFF, h = code & 0xFF;
      const int32_t* item = a.items + (size_t)u * kItemStride;
      const int page_l = lane < 16 ? item[2 + lane] : 0;
      const int tok0 = c * kSC, ntok = min(kSC, a.row_len[r] - tok0);
      const int npg = (ntok + a.pt - 1) / a.pt;
      const size_t hs = (size_t)a.pt * kHD;
      if (warp == 0) {
        if (lane == 0) mbar_arrive_expect_tx(bar, (uint32_t)ntok * kHD * 2 * 2);
        __syncwarp();
        if (lane < npg) {
          const uint32_t bytes = (uint32_t)min(a.pt, ntok - lane * a.pt) * kHD * 2;
          const __nv_bfloat16* kb = a.pool + (((size_t)page_l * 2) * a.Hkv + h) * hs;
          bulk_g2s(Ks + lane * a.pt * kHD, kb, bytes, bar);
          bulk_g2s(Vs + lane * a.pt * kHD, kb + (size_t)a.Hkv * hs, bytes, bar);
        }
      }
      attn_load_q<REP>(a, r, h, qs, lane);
      __syncwarp();
      mbar_wait(bar, phase);
      if (nu < 3) astamp(a, 2 + 4 * nu);
      const int wt0 = warp * 16;  // this warp's 16 tokens
      const int wn = max(0, min(16, ntok - wt0));
      WarpPartial<REP, 2> wp;
      if (wn > 0) wp.run(qs, Ks + wt0 * kHD, Vs + wt0 * kHD, wn, a.scale, lane);
      // combine the warps' partials (fixed warp order)
      float* cw = comb + warp * REP * (kHD + 2);
#pragma unroll
      for (int e = 0; e < REP; ++e) {
        if (lane == 0) {
          cw[e * (kHD + 2)] = wn > 0 ? wp.m[e] : -INFINITY;
          cw[e * (kHD + 2) + 1] = wn > 0 ? wp.l[e] : 0.f;
        }
        float* oo = cw + e * (kHD + 2) + 2;
        oo[4 * lane] = wn > 0 ? wp.o[e][0] : 0.f;
        oo[4 * lane + 1] = wn > 0 ? wp.o[e][1] : 0.f;
        oo[4 * lane + 2] = wn > 0 ? wp.o[e][2] : 0.f;
        oo[4 * lane + 3] = wn > 0 ? wp.o[e][3] : 0.f;
      }
      __syncthreads();
      if (warp == 0) {
        float M[REP], L[REP], O[REP][4];
#pragma unroll
        for (int e = 0; e < REP; ++e) {
          M[e] = -INFINITY;
          for (int w = 0; w < kAttnWarps; ++w) M[e] = fmaxf(M[e], comb[(w * REP + e) * (kHD + 2)]);
          L[e] = 0.f;
          O[e][0] = O[e][1] = O[e][2] = O[e][3] = 0.f;
          for (int w = 0; w < kAttnWarps; ++w) {
            const float* src = comb + (w * REP + e) * (kHD + 2);
            if (src[0] == -INFINITY) continue;
            const float f = expf(src[0] - M[e]);
            L[e] += f * src[1];
#pragma unroll
            for (int k = 0; k < 4; ++k) O[e][k] += f * src[2 + 4 * lane + k];
          }
        }
        store_partial<REP>(a, r, h, a.nc_pre + c, M, L, O, lane);
        if (a.merge_cnt) {
          // count this (row, kv head)'s suffix units; the last one merges it at the end
          __threadfence();
          __syncwarp();
          if (lane == 0) {
            const int nsuf = (a.row_len[r] + kSC - 1) / kSC;
            if (atomicAdd(a.merge_cnt + r * a.Hkv + h, 1) + 1 == nsuf) {
              __threadfence();
              a.merge_cnt[r * a.Hkv + h] = 0;  // ready for the next launch
              if (merge_n < 128) merge_list[merge_n++] = (r << 8) | h;  // single writer: warp 0 lane 0
            }
          }
        }
      }
    }
    __syncthreads();  // smem reuse by the next unit
    phase ^= 1;
    if (nu < 3) astamp(a, 3 + 4 * nu);
    if (nu < 3 && threadIdx.x == 0 && a.dbg_ts) a.dbg_ts[blockIdx.x * 16 + 4 + 4 * nu] = (code < 0) ? 1 : 2;
  }
  if (dyn && threadIdx.x == 0 && atomicAdd(a.unit_ctr + 1, 1) == (int)gridDim.x - 1) {
    a.unit_ctr[0] = 0;  // every CTA has taken its last unit: ready for the next launch
    a.unit_ctr[1] = 0;
  }
  if (!a.prefill && a.tc_prefix) pdl_wait();  // the tcgen05 prefix partials are complete from here on
  if (!a.prefill && a.merge_cnt) {
    // LSE merge (R8) fused: the unit that completed a (row, kv head) merges it after the wait above
    const int nm = merge_n;
    for (int j = warp; j < nm * REP; j += kAttnWarps) {
      const int rh = merge_list[j / REP];
      attn_merge_one<REP>(a, rh >> 8, rh & 0xFF, j % REP, lane);
    }
  }
  astamp(a, 15);
}

// LSE merge (R8) of (row r, kv head h): grid (rows, Hkv), one warp.  Lane i
// holds partial i's (m, l) (<= 32 partials); all o loads are issued together.
template <int REP>
__global__ void __launch_bounds__(32) attn_merge_kernel(AttnArgs a) {
  pdl_launch_dependents();
  pdl_wait();
  const int r = blockIdx.x, h = blockIdx.y, lane = threadIdx.x;
  if (!a.row_active[r]) return;
  const int npre = a.prefill ? min(a.nc_pre, r / kPC + 1) : a.nc_pre;
  const int nsuf = a.prefill ? 0 : (a.row_len[r] + kSC - 1) / kSC;
  const int n = npre + nsuf;
  const int my_slot = lane < npre ? lane : a.nc_pre + (lane - npre);
#pragma unroll 1
  for (int j = 0; j < REP; ++j) {
    const int qh = h * REP + j;
    const size_t base = ((size_t)r * a.Hq + qh) * a.NC;
    float mi = -INFINITY, li = 0.f;
    if (lane < n) {
      const float2 ml = *reinterpret_cast<const float2*>(a.part_ml + (base + my_slot) * 2);
      mi = ml.x;
      li = ml.y;
    }
    const float M = warp_max(mi);
    const float wi = (lane < n && mi != -INFINITY) ? expf(mi - M) * li : 0.f;
    const float den = warp_sum(wi);
    float4 num = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll 1
    for (int i0 = 0; i0 < n; i0 += 8) {
      float4 o[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const int i = i0 + k;
        const int slot = i < npre ? i : a.nc_pre + (i - npre);
        o[k] = i < n ? reinterpret_cast<const float4*>(a.part_o + (base + slot) * kHD)[lane] : make_float4(0, 0, 0, 0);
      }
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const float w = __shfl_sync(0xffffffffu, wi, (i0 + k) & 31);
        if (i0 + k < n) {
          num.x += w * o[k].x;
          num.y += w * o[k].y;
          num.z += w * o[k].z;
          num.w += w * o[k].w;
        }
      }
    }
    const float inv = 1.0f / den;
    attn_store_out(a, r, qh, make_float4(num.x * inv, num.y * inv, num.z * inv, num.w * inv), lane);
  }
}

// ------------------------------------------------------------------ prefix key norms
// kmax[((g * layers + l) * Hkv + h) * nt + tile] = max over the tile's tokens of ||k_t||_2 (fp32 over
// the bf16 keys), for prefix buffers [g][layers][2][Hkv][pcap][128].  The prefix is immutable after
// prefill, so this runs once per prompt; the decode prefix kernel bounds its scores with it.
__global__ void __launch_bounds__(128) prefix_kmax_kernel(const __nv_bfloat16* __restrict__ prefix, int layers,
                                                          int Hkv, int pcap, int plen, float* __restrict__ kmax) {
  const int nt = (plen + 127) / 128;
  const int tile = blockIdx.x % nt, h = (blockIdx.x / nt) % Hkv, gl = blockIdx.x / (nt * Hkv);
  const int tok = tile * 128 + threadIdx.x;
  float ss = 0.f;
  if (tok < plen) {
    const uint4* k4 = reinterpret_cast<const uint4*>(prefix + ((size_t)gl * 2 * Hkv * pcap + (size_t)h * pcap + tok) * kHD);
#pragma unroll 4
    for (int i = 0; i < 16; ++i) {
      const uint4 v = k4[i];
      const __nv_bfloat162* b = reinterpret_cast<const __nv_bfloat162*>(&v);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const float2 f = __bfloat1622float2(b[j]);
        ss += f.x * f.x + f.y * f.y;
      }
    }
  }
  __shared__ float red[4];
  ss = warp_max(ss);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = ss;
  __syncthreads();
  if (threadIdx.x == 0) kmax[blockIdx.x] = sqrtf(fmaxf(fmaxf(red[0], red[1]), fmaxf(red[2], red[3])));
}

// ------------------------------------------------------------------ shared-prefix attention on tcgen05
// The decode step's shared-prefix part as two dense tensor-core contractions
// (BASELINE north_star: "stacks the group's live queries into one dense
// Q.K_prefix^T / P.V_prefix contraction on tcgen05 tensor cores with
// TMA-staged K/V tiles"):
//   S^T[128 tok x N] = K_tile[128 tok x 128 d] . Q^T           (A = K, K-major; B = Q rows, K-major)
//   O^T[128 d  x N] = V_tile^T[128 d x 128 tok] . P^T          (A = V, MN-major; B = P rows, K-major)
// with N = row_capacity x Hq/Hkv stacked query rows of the group (every live
// slot's heads of one kv head).  One CTA per (kv head, 128-token prefix
// tile); K/V tiles arrive by TMA (128-byte swizzle); S and O accumulate in
// TMEM; the column softmax runs on the 128 token lanes; P enters the second
// MMA as a bf16 hi/lo pair (two accumulating MMAs), i.e. ~fp32 precision.  Each CTA writes one normalised
// partial (o, m, l) per query row and head into prefix slot `tile`.
template <int N>
struct PrefixTcSmem {
  static constexpr int kK = 2 * 128 * 128;   // two 64-d boxes of 128 token rows (bf16)
  static constexpr int kV = 2 * 128 * 128;
  static constexpr int kQ = 2 * N * 128;     // two 64-d atoms of N rows
  static constexpr int kP = 2 * N * 128;     // two 64-token atoms of N rows (P_hi; P_lo follows)
  static constexpr int kS = (8 * 64 + N) * 4; // softmax scratch: [4][32] maxima, [4][32] sums, [N] column sums
  static constexpr int v = kK + kV + kQ + 2 * kP + kS + 4 * N * 4 * 2 + N * 20 + 32 + 64 + 1024;
  static constexpr int kTmemCols = (2 * N) <= 32 ? 32 : ((2 * N) <= 64 ? 64 : ((2 * N) <= 128 ? 128 : 256));
};

IS_DEVICE uint64_t smem_desc_mn_sw128(const void* p, uint32_t lbo_bytes, uint32_t sbo_bytes) {
  uint64_t addr = smem_u32(p);
  uint64_t d = 0;
  d |= (addr >> 4) & 0x3FFFull;
  d |= (uint64_t)((lbo_bytes >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo_bytes >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}

template <int REP, int N>
__global__ void __launch_bounds__(128, 1)
    attn_prefix_tc_kernel(const __grid_constant__ CUtensorMap tmKV, AttnArgs a, int kv_row_base) {
  using SM = PrefixTcSmem<N>;
  extern __shared__ uint8_t tc_raw[];
  uint8_t* sm = align1024_smem(tc_raw);
  uint8_t* Ksm = sm;
  uint8_t* Vsm = Ksm + SM::kK;
  uint8_t* Qsm = Vsm + SM::kV;
  uint8_t* Psm = Qsm + SM::kQ;
  uint8_t* Plo = Psm + SM::kP;
  float* Ssm = reinterpret_cast<float*>(Plo + SM::kP);  // softmax scratch (SM::kS)
  float* red = Ssm + SM::kS / 4;                       // [4][N] max, [4][N] sum
  float* colM = red + 8 * N;                           // [N] column max, [N] 1/sum, [N] (int) partial index or -1
  float* colI = colM + N;
  long long* colP = reinterpret_cast<long long*>(colI + 2 * N);
  uint64_t* bars = reinterpret_cast<uint64_t*>(colP + N);
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bars + 2);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nt = (a.plen + 127) / 128;
  // CTA = (group, kv head, 128-token prefix tile); the group's live rows are the N columns
  const int grp = blockIdx.x / (a.Hkv * nt);
  const int h = (blockIdx.x / nt) % a.Hkv, tile = blockIdx.x % nt;
  const int row0 = grp * a.grp_rows;
  kv_row_base += grp * a.grp_kv_rows;
  const int tok0 = tile * 128, ntok = min(128, a.plen - tok0);
  if (threadIdx.x == 0) {
    tma_prefetch_desc(&tmKV);
    mbar_init(&bars[0], 1);  // TMA K+V
    mbar_init(&bars[1], 1);  // MMA commits (phase 0: S, phase 1: O)
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc<SM::kTmemCols>(tslot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tslot;
  astamp(a, 0);
  if (threadIdx.x == 0) {
    // The shared prefix KV is immutable after is_prefill: stage it BEFORE waiting for
    // the QKV GEMM, so its TMA latency hides under the previous kernel.
    // K rows: [(kv=0) * Hkv + h] * pcap + tok ; V rows: [(kv=1) * Hkv + h] * pcap + tok
    const int rk = kv_row_base + (0 * a.Hkv + h) * a.pcap + tok0;
    const int rv = kv_row_base + (1 * a.Hkv + h) * a.pcap + tok0;
    mbar_arrive_expect_tx(&bars[0], SM::kK + SM::kV);
    tma_load_2d(Ksm, &tmKV, &bars[0], 0, rk, kEvictNormal);
    tma_load_2d(Ksm + 128 * 128, &tmKV, &bars[0], 64, rk, kEvictNormal);
    tma_load_2d(Vsm, &tmKV, &bars[0], 0, rv, kEvictNormal);
    tma_load_2d(Vsm + 128 * 128, &tmKV, &bars[0], 64, rv, kEvictNormal);
  }
  // row tables (the previous step's scheduler) and the key-norm bound (prefill) are final
  // before the wait
  if (threadIdx.x < N) {
    const int rl = threadIdx.x / REP, r = row0 + rl;
    colI[N + threadIdx.x] = (rl < a.grp_rows && r < a.rows && a.row_active[r]) ? 1.f : 0.f;  // row live
  }
  const float kmx = a.kmax ? a.kmax[grp * a.kmax_grp + h * nt + tile] : 0.f;
  __syncthreads();
  // ---- the softmax below is latency-bound by instruction fetch when it runs cold (measured
  // ~25 ns per instruction in the decode step: this kernel's code is evicted between layers), so
  // pass 0 runs the bounded-offset softmax once on stale TMEM / smem while the QKV GEMM is still
  // running (its outputs are rewritten in pass 1), and pass 1 does the real work.
  constexpr int CW = N < 32 ? N : 32;
  const int t = warp * 32 + lane;  // token lane (TMEM lane quadrant = warp)
  float* sbuf = Ssm;               // [4][32] maxima, [4][32] sums, [64] column sums
  const uint32_t trow = tmem + ((uint32_t)(warp * 32) << 16);
  const bool valid = t < ntok;
  float* qb2 = red;  // [N] score bound per column (log2 units), [N] fast-path flag
#pragma unroll 1
  for (int pass = (a.kmax && !(a.dbg_mode & 32)) ? 0 : 1; pass < 2; ++pass) {
  bool fast = true;
  if (pass == 1) {
  pdl_wait();                 // q of this step comes from the QKV GEMM
  astamp(a, 1);
  pdl_launch_dependents();    // the suffix kernel may start now (it does not touch our outputs)
  // Q rows n = r*REP + e (K-major, 128-byte swizzle, two 64-d atoms); ||q_n||^2 on the way
  for (int i = threadIdx.x; i < N * 16; i += 128) {
    const int n = i >> 4, c = i & 15;
    const int rl = n / REP, r = row0 + rl, e = n % REP;
    uint4 v = make_uint4(0, 0, 0, 0);
    if (colI[N + n] != 0.f) v = *reinterpret_cast<const uint4*>(a.q + ((size_t)r * a.Hq + h * REP + e) * kHD + c * 8);
    *reinterpret_cast<uint4*>(Qsm + (c >> 3) * N * 128 + n * 128 + (((c & 7) ^ (n & 7)) << 4)) = v;
    const __nv_bfloat162* b = reinterpret_cast<const __nv_bfloat162*>(&v);
    float qs = 0.f;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const float2 f = __bfloat1622float2(b[j]);
      qs += f.x * f.x + f.y * f.y;
    }
#pragma unroll
    for (int o = 8; o >= 1; o >>= 1) qs += __shfl_xor_sync(0xffffffffu, qs, o);  // the 16 chunks of row n
    if (c == 0) {
      // Cauchy-Schwarz: s = q.k / sqrt(d) <= ||q|| max||k|| / sqrt(d) =: B (natural units).  With
      // B <= 40 every exp(s - B) lies in [e^-80, 1] (no overflow, no underflow to zero), so B
      // replaces the column max: softmax is shift-invariant and the LSE merge takes any offset.
      const float B = sqrtf(qs) * kmx * a.scale;
      qb2[n] = B * 1.4426950408889634f;
      qb2[N + n] = (a.kmax && B <= 40.f) ? 1.f : 0.f;
    }
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  for (int n = 0; n < N; ++n) fast = fast && qb2[N + n] != 0.f;
  astamp(a, 2);
  if (threadIdx.x == 0) {
    mbar_wait(&bars[0], 0);
    astamp(a, 3);
    tc_fence_after();
    constexpr uint32_t idesc = idesc_bf16_f32(128, N);
#pragma unroll
    for (int k = 0; k < 8; ++k) {  // 128 d in steps of 16
      const uint64_t da = smem_desc_k_sw128(Ksm + (k >> 2) * 128 * 128) + 2 * (k & 3);
      const uint64_t db = smem_desc_k_sw128(Qsm + (k >> 2) * N * 128) + 2 * (k & 3);
      tc_mma_f16(tmem, da, db, idesc, k > 0 ? 1u : 0u);
    }
    tc_commit(&bars[1]);
  }
  __syncwarp();
  mbar_wait(&bars[1], 0);
  astamp(a, 4);
  tc_fence_after();
  }  // pass 1 only
  // ---- column softmax in registers.  Thread t holds S^T row t (its token) for CW
  // query columns at a time (CW = min(N, 32)); a transpose reduction (CW - 1 shuffles,
  // plus one per remaining lane bit) leaves lane l with column (l mod CW)'s max / sum over
  // the warp's 32 tokens, the 4 warps combine through smem.
  if (fast) {
    // bounded-offset softmax: p = exp(s - B[column]); only the column sums need the other lanes
#pragma unroll 1
    for (int c32 = 0; c32 < N / CW; ++c32) {
      float sv[CW];
      tmem_ld16(trow + c32 * CW, sv);
      if (CW > 16) tmem_ld16(trow + c32 * CW + 16, sv + (CW > 16 ? 16 : 0));
      astamp(a, 9);
      const float sl2 = a.scale * 1.4426950408889634f;
      float r[CW];
#pragma unroll
      for (int j = 0; j < CW; ++j) {
        const int n = c32 * CW + j;
        const float p = valid ? exp2f(fmaf(sv[j], sl2, -qb2[n])) : 0.f;
        r[j] = p;
        const int off = (t >> 6) * N * 128 + n * 128 + ((((t & 63) >> 3) ^ (n & 7)) << 4) + (t & 7) * 2;
        const __nv_bfloat16 phi = __float2bfloat16_rn(p);
        *reinterpret_cast<__nv_bfloat16*>(Psm + off) = phi;
        *reinterpret_cast<__nv_bfloat16*>(Plo + off) = __float2bfloat16_rn(p - __bfloat162float(phi));
      }
      astamp(a, 10);
#pragma unroll
      for (int o = CW / 2; o >= 1; o >>= 1) {
        const bool up = (lane & o) != 0;
#pragma unroll
        for (int j = 0; j < o; ++j) {
          const float send = up ? r[j] : r[j + o];
          const float keep = up ? r[j + o] : r[j];
          r[j] = keep + __shfl_xor_sync(0xffffffffu, send, o);
        }
      }
#pragma unroll
      for (int o = CW; o < 32; o <<= 1) r[0] += __shfl_xor_sync(0xffffffffu, r[0], o);
      sbuf[128 + warp * 32 + lane] = r[0];
      astamp(a, 11);
      __syncthreads();
      astamp(a, 12);
      if (threadIdx.x < CW) {
        const int n = c32 * CW + threadIdx.x;
        colM[n] = qb2[n] * 0.6931471805599453f;  // the offset B, natural units
        sbuf[8 * 64 + n] = sbuf[128 + threadIdx.x] + sbuf[160 + threadIdx.x] + sbuf[192 + threadIdx.x] + sbuf[224 + threadIdx.x];
      }
      if (c32 + 1 < N / CW) __syncthreads();
    }
  } else {
#pragma unroll 1
  for (int c32 = 0; c32 < N / CW; ++c32) {
    float sv[CW], r[CW];
    tmem_ld16(trow + c32 * CW, sv);
    if (CW > 16) tmem_ld16(trow + c32 * CW + 16, sv + (CW > 16 ? 16 : 0));
    const float sl2 = a.scale * 1.4426950408889634f;  // scores in log2 units: exp2 below
#pragma unroll
    for (int j = 0; j < CW; ++j) {
      sv[j] = valid ? sv[j] * sl2 : -INFINITY;
      r[j] = sv[j];
    }
    // transpose-max: after the step with offset o, lanes with bit o hold the upper half
#pragma unroll
    for (int o = CW / 2; o >= 1; o >>= 1) {
      const bool up = (lane & o) != 0;
#pragma unroll
      for (int j = 0; j < o; ++j) {
        const float send = up ? r[j] : r[j + o];
        const float keep = up ? r[j + o] : r[j];
        r[j] = fmaxf(keep, __shfl_xor_sync(0xffffffffu, send, o));
      }
    }
#pragma unroll
    for (int o = CW; o < 32; o <<= 1) r[0] = fmaxf(r[0], __shfl_xor_sync(0xffffffffu, r[0], o));
    sbuf[warp * 32 + lane] = r[0];  // column c32*CW + (lane mod CW), this warp's 32 tokens
    __syncthreads();
    float mcol = fmaxf(fmaxf(sbuf[lane], sbuf[32 + lane]), fmaxf(sbuf[64 + lane], sbuf[96 + lane]));
    __syncthreads();
    // p = exp(s - M[column]); M of column j comes from lane j
    float p[CW];
#pragma unroll
    for (int j = 0; j < CW; ++j) {
      const float Mj = __shfl_sync(0xffffffffu, mcol, j);
      p[j] = valid ? exp2f(sv[j] - Mj) : 0.f;
      r[j] = p[j];
    }
#pragma unroll
    for (int o = CW / 2; o >= 1; o >>= 1) {
      const bool up = (lane & o) != 0;
#pragma unroll
      for (int j = 0; j < o; ++j) {
        const float send = up ? r[j] : r[j + o];
        const float keep = up ? r[j + o] : r[j];
        r[j] = keep + __shfl_xor_sync(0xffffffffu, send, o);
      }
    }
#pragma unroll
    for (int o = CW; o < 32; o <<= 1) r[0] += __shfl_xor_sync(0xffffffffu, r[0], o);
    sbuf[128 + warp * 32 + lane] = r[0];
    // P^T operand (row n, K index t, two 64-token atoms, 128-byte swizzle) as a bf16
    // hi/lo pair (two accumulating MMAs keep P to ~2^-16)
#pragma unroll
    for (int j = 0; j < CW; ++j) {
      const int n = c32 * CW + j;
      const int off = (t >> 6) * N * 128 + n * 128 + ((((t & 63) >> 3) ^ (n & 7)) << 4) + (t & 7) * 2;
      const __nv_bfloat16 phi = __float2bfloat16_rn(p[j]);
      *reinterpret_cast<__nv_bfloat16*>(Psm + off) = phi;
      *reinterpret_cast<__nv_bfloat16*>(Plo + off) = __float2bfloat16_rn(p[j] - __bfloat162float(phi));
    }
    __syncthreads();
    if (threadIdx.x < CW) {
      const int n = c32 * CW + threadIdx.x;
      colM[n] = mcol * 0.6931471805599453f;  // natural units (thread x < CW is lane x of warp 0: column x)
      sbuf[8 * 64 + n] = sbuf[128 + threadIdx.x] + sbuf[160 + threadIdx.x] + sbuf[192 + threadIdx.x] + sbuf[224 + threadIdx.x];
    }
    __syncthreads();
  }
  }
  if (pass == 0) {
    astamp(a, 8);
    __syncthreads();
  }
  }  // pass
  astamp(a, 13);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  astamp(a, 14);
  if (threadIdx.x == 0) {
    tc_fence_after();
    // A = V^T: M = d (MN-major: 64-d blocks 16 KB apart), K = tokens (8-row groups 1 KB apart)
    constexpr uint32_t idesc2 = idesc_bf16_f32(128, N) | (1u << 15);
#pragma unroll
    for (int k = 0; k < 16; ++k) {  // 128 tokens in steps of 16, for P_hi then P_lo
      const uint64_t da = smem_desc_mn_sw128(Vsm + (k & 7) * 2048, 128 * 128, 1024);
      const uint64_t db = smem_desc_k_sw128((k < 8 ? Psm : Plo) + ((k & 7) >> 2) * N * 128) + 2 * (k & 3);
      tc_mma_f16(tmem + N, da, db, idesc2, k > 0 ? 1u : 0u);
    }
    astamp(a, 15);
    tc_commit(&bars[1]);
  }
  __syncwarp();
  astamp(a, 5);
  mbar_wait(&bars[1], 1);
  astamp(a, 6);
  tc_fence_after();
  // ---- epilogue: lane = head dim d; normalise and write partial slot `tile`
  if (threadIdx.x < N) {
    const int n = threadIdx.x, r = row0 + n / REP, e = n % REP;
    const float L = Ssm[8 * 64 + n];
    colI[n] = 1.0f / L;
    const bool act = colI[N + n] != 0.f;
    colP[n] = act ? (long long)(((size_t)r * a.Hq + h * REP + e) * a.NC + tile) : -1ll;
    if (act) *reinterpret_cast<float2*>(a.part_ml + colP[n] * 2) = make_float2(colM[n], L);
  }
  __syncthreads();
  const int d = t;
#pragma unroll 1
  for (int c = 0; c < N / 16; ++c) {
    float o16[16];
    tmem_ld16(trow + N + c * 16, o16);
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const long long pidx = colP[c * 16 + j];
      if (pidx >= 0) a.part_o[pidx * kHD + d] = o16[j] * colI[c * 16 + j];
    }
  }
  astamp(a, 7);
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc<SM::kTmemCols>(tmem);
  }
}

// ------------------------------------------------------------------ L2 weight prefetcher
// A side branch of the decode-step graph: one warp walks the step's weights in the order the
// GEMMs consume them (per layer QKV, o_proj, gate/up, down; then the tied lm_head) and issues
// cp.async.bulk.prefetch.L2 for 64 KB chunks, staying at most `lookahead` bytes ahead of the
// GEMM that last announced itself (GemmArgs.pf_progress = its index in this order), so HBM keeps
// streaming weights into L2 while the dependent GEMM / attention chain of earlier layers runs.
// Nothing waits on it: it only changes where the GEMMs' weight TMA loads hit.
struct PrefetchArgs {
  const unsigned long long* ptr;  // [n] start address of each weight matrix, consumption order
  const long long* off;           // [n + 1] byte offset of each matrix in that order (prefix sums)
  int n;
  int* progress;                  // the GEMMs' announced index (-1 before the step's first GEMM)
  long long lookahead;            // bytes
};
__global__ void __launch_bounds__(32) l2_prefetch_kernel(PrefetchArgs a) {
  const int lane = threadIdx.x;
  constexpr long long kChunk = 64 << 10;
  long long limit = -1;  // prefetch bytes [0, limit] allowed so far
  int seen = -2;
  unsigned long long t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
#pragma unroll 1
  for (int e = 0; e < a.n - 1; ++e) {  // (not the last matrix: once its GEMM runs there is nothing left)
    const long long o0 = a.off[e], o1 = a.off[e + 1];
    const char* base = reinterpret_cast<const char*>(a.ptr[e]);
#pragma unroll 1
    for (long long r0 = o0; r0 < o1; r0 += 32 * kChunk) {  // rounds of 32 chunks, one per lane
      const long long o = r0 + lane * kChunk;
      const long long need = min(o1, r0 + 32 * kChunk) - 1;  // the round's last byte inside the window
      bool skip = false;
      while (need > limit) {
        int p = 0;
        if (lane == 0) asm volatile("ld.relaxed.gpu.global.s32 %0, [%1];" : "=r"(p) : "l"(a.progress) : "memory");
        p = __shfl_sync(0xffffffffu, p, 0);
        // the consumer is at the last matrix (nothing left worth fetching) or past this one
        if (p >= a.n - 1) return;
        if (p > e) {
          skip = true;
          break;
        }
        if (p != seen) {
          seen = p;
          limit = (p < 0 ? 0 : a.off[p]) + a.lookahead;
        } else {
          unsigned long long t;
          asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
          if (t - t0 > 50000000ull) return;  // never hold the step up: give up after 50 ms
          __nanosleep(500);
        }
      }
      if (skip) break;
      if (o < o1) {
        const long long sz = min(kChunk, o1 - o);
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(base + (o - o0)), "r"((uint32_t)sz)
                     : "memory");
      }
    }
  }
}

// ------------------------------------------------------------------ shared-prefix attention on tcgen05, q rows as M
// The same contraction as attn_prefix_tc_kernel with the group's stacked query rows as the MMA's M
// (128 per tile, MT tiles: up to 256 rows, e.g. the 4B shape with all 64 samples live):
//   S[q][tok] = Q[q][:] . K_tile[tok][:]^T        (A = Q, K-major; B = K tile, K-major; N = 128 tokens)
//   O[q][d]   = P[q][tok] . V_tile[tok][d]          (A = P, K-major; B = V tile, MN-major; N = 128 dims)
// Each thread owns one query row's TMEM lane, so the row softmax (max, exp, sum over the tile's
// 128 tokens) is in registers with no cross-thread reduction; P (bf16 hi/lo pair, ~2^-16) is
// written over the Q / K tiles MMA 1 no longer needs, so one 128-row tile needs 96 KB of shared
// memory.  One CTA per (group, kv head, 128-token prefix tile); the partial (o, m, l) of every
// live query row goes to prefix partial slot `tile`.
template <int MT>
struct PrefixTc2Smem {
  static constexpr int kTile = 2 * 128 * 128;  // [128 rows][128 bf16] as two 64-column halves: 32 KB
  static constexpr int v = (MT == 1 ? 3 : 5) * kTile + 64 + 1024;
  static constexpr int kTmemCols = MT == 1 ? 256 : 512;
};

template <int REP, int MT>
__global__ void __launch_bounds__(128, 1)
    attn_prefix_tc2_kernel(const __grid_constant__ CUtensorMap tmKV, AttnArgs a, int kv_row_base) {
  using SMc = PrefixTc2Smem<MT>;
  constexpr int T = SMc::kTile, HALF = T / 2;
  extern __shared__ uint8_t tc2_raw[];
  uint8_t* sm = align1024_smem(tc2_raw);
  uint8_t* Qs0 = sm;
  uint8_t* Qs1 = sm + T;                 // (MT == 2)
  uint8_t* Ks = sm + MT * T;
  uint8_t* Vs = Ks + T;
  uint8_t* Xs = Vs + T;                  // (MT == 2)
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm + (MT == 1 ? 3 : 5) * T);
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bars + 2);
  __shared__ uint8_t live_n[256];  // stacked row n is a live row of the group
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nt = (a.plen + 127) / 128;
  const int grp = blockIdx.x / (a.Hkv * nt);
  const int h = (blockIdx.x / nt) % a.Hkv, tile = blockIdx.x % nt;
  const int row0 = grp * a.grp_rows;
  kv_row_base += grp * a.grp_kv_rows;
  const int tok0 = tile * 128, ntok = min(128, a.plen - tok0);
  const int nrows = a.grp_rows * REP;  // stacked query rows n = (row - row0) * REP + e
  if (threadIdx.x == 0) {
    tma_prefetch_desc(&tmKV);
    mbar_init(&bars[0], 1);  // TMA K + V
    mbar_init(&bars[1], 1);  // MMA commits (phase 0: S, phase 1: O)
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc<SMc::kTmemCols>(tslot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tslot;
  astamp(a, 0);
  if (threadIdx.x == 0) {
    // the shared prefix KV is immutable after is_prefill: staged BEFORE the wait on the QKV GEMM
    const int rk = kv_row_base + (0 * a.Hkv + h) * a.pcap + tok0;
    const int rv = kv_row_base + (1 * a.Hkv + h) * a.pcap + tok0;
    mbar_arrive_expect_tx(&bars[0], 2 * T);
    tma_load_2d(Ks, &tmKV, &bars[0], 0, rk, kEvictNormal);
    tma_load_2d(Ks + HALF, &tmKV, &bars[0], 64, rk, kEvictNormal);
    tma_load_2d(Vs, &tmKV, &bars[0], 0, rv, kEvictNormal);
    tma_load_2d(Vs + HALF, &tmKV, &bars[0], 64, rv, kEvictNormal);
  }
  pdl_wait();  // q of this step comes from the QKV GEMM
  astamp(a, 1);
  pdl_launch_dependents();
  for (int n = threadIdx.x; n < nrows; n += 128) {
    const int r = row0 + n / REP;
    live_n[n] = r < a.rows && a.row_active[r];
  }
  // Q rows (K-major, 128-byte swizzle): row n of tile n >> 7, 16-B chunk c (dims 8c..8c+7); a
  // thread's chunks are loaded 16 at a time (all in flight), then stored
  for (int i0 = 0; i0 < nrows * 16; i0 += 16 * 128) {
    uint4 v[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const int i = i0 + j * 128 + threadIdx.x;
      const int n = i >> 4, c = i & 15;
      const int r = row0 + n / REP, e = n % REP;
      v[j] = (i < nrows * 16 && r < a.rows)
                 ? *reinterpret_cast<const uint4*>(a.q + ((size_t)r * a.Hq + h * REP + e) * kHD + c * 8)
                 : make_uint4(0, 0, 0, 0);
    }
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const int i = i0 + j * 128 + threadIdx.x;
      if (i >= nrows * 16) break;
      const int n = i >> 4, c = i & 15, nl = n & 127;
      uint8_t* dst = ((MT == 2 && n >= 128) ? Qs1 : Qs0) + (c >> 3) * HALF + nl * 128;
      *reinterpret_cast<uint4*>(dst + (((c & 7) ^ (nl & 7)) << 4)) = v[j];
    }
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  astamp(a, 2);
  if (threadIdx.x == 0) {
    mbar_wait(&bars[0], 0);
    astamp(a, 3);
    tc_fence_after();
    constexpr uint32_t idesc = idesc_bf16_f32(128, 128);
#pragma unroll
    for (int mt = 0; mt < MT; ++mt) {
      if (mt * 128 >= nrows) break;
      uint8_t* Q = mt == 0 ? Qs0 : Qs1;
#pragma unroll
      for (int k = 0; k < 8; ++k) {  // 128 dims in steps of 16
        const uint64_t da = smem_desc_k_sw128(Q + (k >> 2) * HALF) + 2 * (k & 3);
        const uint64_t db = smem_desc_k_sw128(Ks + (k >> 2) * HALF) + 2 * (k & 3);
        tc_mma_f16(tmem + mt * 128, da, db, idesc, k > 0 ? 1u : 0u);
      }
    }
    tc_commit(&bars[1]);
  }
  __syncwarp();
  mbar_wait(&bars[1], 0);
  astamp(a, 4);
  tc_fence_after();
  // ---- row softmax in registers: thread = TMEM lane = query row nl of each tile
  const int nl = warp * 32 + lane;
  float mrow[MT], lrow[MT];
#pragma unroll 1
  for (int mt = 0; mt < MT; ++mt) {
    mrow[mt] = -INFINITY;
    lrow[mt] = 0.f;
    if (mt * 128 + warp * 32 >= nrows) continue;  // (warp-uniform) no live row in this warp
    uint32_t sv[128];
    const uint32_t trow = tmem + ((uint32_t)(warp * 32) << 16) + mt * 128;
#pragma unroll
    for (int j = 0; j < 4; ++j) tmem_ld32_nowait(trow + 32 * j, sv + 32 * j);
    tmem_ld_wait();
    // scores in log2 units (scale * log2 e folded): p = exp2(x - max) = exp(score * scale - m)
    const float sl2 = a.scale * 1.4426950408889634f;
    float mx = -INFINITY;
#pragma unroll
    for (int j = 0; j < 128; ++j) {
      const float x = j < ntok ? __uint_as_float(sv[j]) * sl2 : -INFINITY;
      sv[j] = __float_as_uint(x);
      mx = fmaxf(mx, x);
    }
    float l = 0.f;
    uint8_t* Ph = mt == 0 ? Qs0 : Ks;
    uint8_t* Pl = mt == 0 ? (MT == 1 ? Ks : Qs1) : Xs;
#pragma unroll
    for (int c = 0; c < 16; ++c) {  // 8 tokens per 16-B chunk
      uint32_t hi[4], lo[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const float p0 = exp2f(__uint_as_float(sv[8 * c + 2 * q]) - mx);
        const float p1 = exp2f(__uint_as_float(sv[8 * c + 2 * q + 1]) - mx);
        l += p0 + p1;
        const __nv_bfloat162 hb = __floats2bfloat162_rn(p0, p1);
        const float2 hf = __bfloat1622float2(hb);
        hi[q] = *reinterpret_cast<const uint32_t*>(&hb);
        lo[q] = pack_bf16(p0 - hf.x, p1 - hf.y);
      }
      const int off = (c >> 3) * HALF + nl * 128 + (((c & 7) ^ (nl & 7)) << 4);
      *reinterpret_cast<uint4*>(Ph + off) = make_uint4(hi[0], hi[1], hi[2], hi[3]);
      *reinterpret_cast<uint4*>(Pl + off) = make_uint4(lo[0], lo[1], lo[2], lo[3]);
    }
    mrow[mt] = mx * 0.6931471805599453f;  // back to natural units: the partial's m (R8)
    lrow[mt] = l;
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  astamp(a, 5);
  if (threadIdx.x == 0) {
    tc_fence_after();
    constexpr uint32_t idesc2 = idesc_bf16_f32(128, 128) | (1u << 16);  // B (V) MN-major
#pragma unroll
    for (int mt = 0; mt < MT; ++mt) {
      if (mt * 128 >= nrows) break;
      uint8_t* Ph = mt == 0 ? Qs0 : Ks;
      uint8_t* Pl = mt == 0 ? (MT == 1 ? Ks : Qs1) : Xs;
#pragma unroll
      for (int k = 0; k < 8; ++k) {  // 128 tokens in steps of 16
        const uint64_t db = smem_desc_mn_sw128(Vs + k * 2048, HALF, 1024);
        const uint64_t dh = smem_desc_k_sw128(Ph + (k >> 2) * HALF) + 2 * (k & 3);
        const uint64_t dl = smem_desc_k_sw128(Pl + (k >> 2) * HALF) + 2 * (k & 3);
        tc_mma_f16(tmem + MT * 128 + mt * 128, dh, db, idesc2, k > 0 ? 1u : 0u);
        tc_mma_f16(tmem + MT * 128 + mt * 128, dl, db, idesc2, 1u);
      }
    }
    tc_commit(&bars[1]);
  }
  __syncwarp();
  mbar_wait(&bars[1], 1);
  astamp(a, 6);
  tc_fence_after();
  // ---- epilogue: row nl's normalised partial (o, m, l) into prefix slot `tile`.  The rows are
  // staged in shared memory (the spent Q / K / P tiles, 64 KB per 128 rows) so that each 512-B
  // partial row is written by a whole warp (coalesced), not by one thread.
  float* ost = reinterpret_cast<float*>(sm);  // [128][132] fp32 (padded rows)
#pragma unroll 1
  for (int mt = 0; mt < MT; ++mt) {
    if (mt * 128 >= nrows) break;
    if (mt * 128 + warp * 32 < nrows) {
      uint32_t ov[128];
      const uint32_t trow = tmem + ((uint32_t)(warp * 32) << 16) + MT * 128 + mt * 128;
#pragma unroll
      for (int j = 0; j < 4; ++j) tmem_ld32_nowait(trow + 32 * j, ov + 32 * j);
      tmem_ld_wait();
      const float inv = 1.0f / lrow[mt];
#pragma unroll
      for (int j = 0; j < 32; ++j)
        *reinterpret_cast<float4*>(ost + nl * 132 + 4 * j) =
            make_float4(__uint_as_float(ov[4 * j]) * inv, __uint_as_float(ov[4 * j + 1]) * inv,
                        __uint_as_float(ov[4 * j + 2]) * inv, __uint_as_float(ov[4 * j + 3]) * inv);
    }
    __syncthreads();
    // warp w writes rows w, w + 4, ...: lane = 16-B piece of the row
    for (int rl = warp; rl < 128 && mt * 128 + rl < nrows; rl += 4) {
      const int n = mt * 128 + rl;
      const int r = row0 + n / REP, e = n % REP;
      if (!live_n[n]) continue;
      const size_t pidx = ((size_t)r * a.Hq + h * REP + e) * a.NC + tile;
      reinterpret_cast<float4*>(a.part_o + pidx * kHD)[lane] = *reinterpret_cast<const float4*>(ost + rl * 132 + 4 * lane);
    }
    {
      const int n = mt * 128 + nl;
      const int r = row0 + n / REP, e = n % REP;
      if (n < nrows && live_n[n]) {
        const size_t pidx = ((size_t)r * a.Hq + h * REP + e) * a.NC + tile;
        *reinterpret_cast<float2*>(a.part_ml + pidx * 2) = make_float2(mrow[mt], lrow[mt]);
      }
    }
    __syncthreads();
  }
  astamp(a, 7);
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc<SMc::kTmemCols>(tmem);
  }
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
  ST_ATTN_PRE,     // of which shared-prefix items (must follow ST_ATTN_ITEMS)
  ST_SUFFIX,       // sum over steps of the live rows' suffix lengths
  ST_PROMPT_ID,    // prompt of the current group (RNG uid base), set by is_start_group: device state,
  ST_PROMPT_LAST,  //   not a kernel parameter, because the decode step is a CUDA graph reused across prompts
  ST_GLIVE,        // block 0 only: pages allocated by all groups (shared pool)
  ST_GPEAK,        // block 0 only: max over steps of ST_GLIVE
  ST_GSTEP,        // block 0 only: decode steps with >= 1 active slot in any group
  ST_TARGET,       // dynamic-slot mode: stop at this many completions (0 = all G), R35
  ST_DISCARDED,    //   samples in flight at the stop, discarded
  ST_ADMSEQ,       // memory-aware admission (R41): next admission sequence number
  ST_STALLS,       //   slot-steps stalled for a page
  ST_COUNT
};
// st[] holds one block of ST_COUNT words per co-resident group (NEXT-1) plus a
// global block M: the shared page pool (ST_FREE_TOP, ST_GLIVE, ST_GPEAK),
// ST_ERROR, the attention work list length and ST_GSTEP.

struct SchedArgs {
  int G, g, row_cap, max_new, pt, maxp, P, log_cap, M;  // M co-resident groups (rows m*g .. m*g+g-1)
  long long* st;             // [M + 1][ST_COUNT] (block M: global)
  int32_t* slot_uid;         // [M][g]
  int32_t* slot_count;       // [M][g]
  int32_t* t;                // [M][G]
  const int32_t* true_len;   // [M][G]
  int32_t* queue;            // [M][G]
  const int32_t* main_init;  // [M][g]
  const int32_t* main_queue; // [M][G]
  int32_t* free_stack;       // [num_pages] (shared)
  int32_t* pagetab;          // [M*G][maxp] (row_lid = m*G + uid)
  int32_t* npages;           // [M][G]
  int32_t* tokens;           // [M][G][max_new]
  int32_t* log_slot;         // [M][log_cap][g]
  int32_t* log_live;         // [M][log_cap] pages held by the group
  uint8_t* done_flag;        // [M][G] 1 once the sample completed (length or EOS)
  unsigned long long* keys;  // [row_cap] lm_head argmax keys
  const unsigned long long* lp_key;  // [row_cap][lp_grid] per-CTA best keys (NEXT-3 log-probabilities)
  const float4* lp_mlz;      // [row_cap][lp_grid] per-CTA (max z, sum exp, winner's z)
  float* logprobs;           // [M][G][max_new] log pi(token) at temperature 1 (R33)
  const float* tok_logits;   // top-p (R36): [rows][vocab] logits; the sampled token's logit is read there
  int vocab;
  int eos_on, eos_id;        // R37: a sample also finishes when it samples eos_id
  int lp_grid;
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
  int32_t* attn_items;       // [Hkv * (nc_pre + row_cap * nc_suf)][kItemStride]
  int Hkv, nc_pre, nc_suf, chunk, tc_prefix;
  int* pf_progress;          // L2 prefetcher pacing word: reset for the next step (nullable)
  // memory-aware admission by predicted length (R41; admit = 1): slots 0..gp-1 are the plan's
  // guaranteed slots, gp..g-1 elastic ones sharing E pages; W = worst-case pages per sample
  int admit, gp, W, E;
  const int32_t* pred;       // [M][G] predicted lengths
  int32_t* adm_seq;          // [M][G] admission order
  int32_t* stall;            // [M][g] slot stalled this step (no page for its token)
};

// Work list of one decode attention launch, built from the row tables by
// the kSchedThreads threads of one CTA: shared-prefix items first (CUDA-core prefix only:
// one per (group of 4 rows with a live row, kv head, kPC-token chunk)), then one suffix
// item per (row, chunk of `chunk` tokens, kv head) carrying the chunk's page ids and
// the row's length.  n_items[0] = items, n_items[1] = prefix items.
struct WorkList {
  int row_cap, chunk, pt, Hkv, nc_pre, tc_prefix, maxp;
  const int32_t* row_active;
  const int32_t* row_len;   // suffix tokens visible (t + 1)
  const int32_t* row_lid;   // page-table row of each row
  const int32_t* pagetab;   // [*][maxp]
  int32_t* items;           // [*][kItemStride]
  long long* n_items;       // [2]
};
constexpr int kSchedThreads = 128;
__device__ void build_attn_worklist(const WorkList& w, int* s_cnt /* [65] */, int* s_npre) {
  const int tid = threadIdx.x;
  int nch = 0;
  if (tid < w.row_cap) {
    nch = w.row_active[tid] ? (w.row_len[tid] + w.chunk - 1) / w.chunk : 0;
    s_cnt[tid] = nch;
  }
  __syncthreads();
  if (tid == 0) {
    // exclusive prefix sum of suffix chunks; shared-prefix items first (CUDA-core prefix only)
    int n = 0;
    if (!w.tc_prefix) {
      for (int g = 0; g * 4 < w.row_cap; ++g) {
        bool live = false;
        for (int s = 4 * g; s < 4 * g + 4 && s < w.row_cap; ++s) live = live || w.row_active[s];
        if (!live) continue;
        for (int h = 0; h < w.Hkv; ++h)
          for (int c = 0; c < w.nc_pre; ++c)
            w.items[(size_t)(n++) * kItemStride] = (int)(0x80000000u | (h << 16) | (c << 8) | g);
      }
    }
    *s_npre = n;
    int acc = 0;
    for (int s = 0; s < w.row_cap; ++s) {
      const int v = s_cnt[s];
      s_cnt[s] = acc;
      acc += v;
    }
    s_cnt[w.row_cap] = acc;
    w.n_items[0] = n + acc * w.Hkv;
    w.n_items[1] = n;
  }
  __syncthreads();
  // ---- suffix items of row s: (chunk c, kv head h) with the chunk's page ids embedded
  if (tid < w.row_cap && nch > 0) {
    const int s = tid;
    const int ppc = w.chunk / w.pt;  // pages per suffix chunk (<= 16)
    const int len = w.row_len[s], lid = w.row_lid[s];
    for (int c = 0; c < nch; ++c)
      for (int h = 0; h < w.Hkv; ++h) {
        int32_t* item = w.items + (size_t)(*s_npre + (s_cnt[s] + c) * w.Hkv + h) * kItemStride;
        item[0] = (c << 16) | (s << 8) | h;
        item[1] = len;
        const int np = min(ppc, (len - c * w.chunk + w.pt - 1) / w.pt);
        for (int j = 0; j < np; ++j) item[2 + j] = w.pagetab[(size_t)lid * w.maxp + c * ppc + j];
      }
  }
  __syncthreads();
}

// R41 refill pass of group m (thread 0): ascending slot order; an idle guaranteed slot adopts the
// stalled elastic sample admitted earliest (with its pages), else pops the SJF queue; an idle
// elastic slot admits the queue head iff the elastic slots' reservations
// sum(max(held, ceil(pred / pt))) plus the head's ceil(pred / pt) fit E pages.
__device__ void admit_refill(const SchedArgs& a, long long* st, int m) {
  int32_t* slot_uid = a.slot_uid + m * a.g;
  int32_t* stall = a.stall + m * a.g;
  const int32_t* queue = a.queue + (size_t)m * a.G;
  const int32_t* pred = a.pred + (size_t)m * a.G;
  int32_t* npages = a.npages + (size_t)m * a.G;
  int32_t* seq = a.adm_seq + (size_t)m * a.G;
  for (int s = 0; s < a.g; ++s) {
    if (slot_uid[s] >= 0) continue;
    if (s < a.gp) {
      int best = -1;
      for (int e = a.gp; e < a.g; ++e)
        if (slot_uid[e] >= 0 && stall[e] && (best < 0 || seq[slot_uid[e]] < seq[slot_uid[best]])) best = e;
      if (best >= 0) {
        slot_uid[s] = slot_uid[best];
        slot_uid[best] = -1;
        stall[best] = 0;
      } else if (st[ST_QHEAD] < st[ST_QLEN]) {
        const int u = queue[st[ST_QHEAD]++];
        slot_uid[s] = u;
        seq[u] = (int32_t)st[ST_ADMSEQ]++;
      }
    } else if (st[ST_QHEAD] < st[ST_QLEN]) {
      const int head = queue[st[ST_QHEAD]];
      long long res = 0;
      for (int e = a.gp; e < a.g; ++e) {
        const int u = slot_uid[e];
        if (u >= 0) res += max(npages[u], (pred[u] + a.pt - 1) / a.pt);
      }
      if (res + (pred[head] + a.pt - 1) / a.pt <= a.E) {
        ++st[ST_QHEAD];
        slot_uid[s] = head;
        seq[head] = (int32_t)st[ST_ADMSEQ]++;
      }
    }
  }
}

// One CTA of kSchedThreads.  The policy itself (finish / park / refill in
// ascending slot order, R18; LIFO page recycling, R26) is sequential and runs
// on thread 0; the per-row preparation of the next step and its attention work
// list are independent per row and run one thread per row.
__global__ void __launch_bounds__(kSchedThreads) sched_kernel(SchedArgs a, int consume, int prep_mask) {
  pdl_launch_dependents();  // let the next kernel launch and prefetch now; it waits for our completion itself
  pdl_wait();
  __shared__ int s_cnt[65];         // suffix chunk counts -> exclusive prefix sums
  __shared__ int s_any, s_npre;
  long long* st0 = a.st + (size_t)a.M * ST_COUNT;  // global block: shared pool, counters
  const int tid = threadIdx.x;
  if (consume && a.logprobs) {
    // log pi(token) = z_tok - logsumexp(z) from the lm_head CTAs' partials, one warp per row,
    // CTAs combined in a fixed order (before the policy below advances t)
    const int warp = tid >> 5, lane = tid & 31;
    for (int row = warp; row < a.M * a.g; row += kSchedThreads / 32) {
      const int uid = a.slot_uid[row];
      if (uid < 0) continue;
      const int m = row / a.g;
      const unsigned long long key = a.keys[row];
      float Mx = -INFINITY, zt = -INFINITY;
      for (int c = lane; c < a.lp_grid; c += 32) {
        const float4 v = a.lp_mlz[(size_t)row * a.lp_grid + c];
        Mx = fmaxf(Mx, v.x);
        if (a.lp_key[(size_t)row * a.lp_grid + c] == key) zt = v.z;
      }
      Mx = warp_max(Mx);
      zt = warp_max(zt);
      if (a.tok_logits) zt = a.tok_logits[(size_t)row * a.vocab + (0xFFFFFFFFu - (uint32_t)(key & 0xFFFFFFFFull))];
      float L = 0.f;
      for (int c = lane; c < a.lp_grid; c += 32) {
        const float4 v = a.lp_mlz[(size_t)row * a.lp_grid + c];
        if (v.x != -INFINITY) L += v.y * expf(v.x - Mx);
      }
      L = warp_sum(L);
      if (lane == 0) {
        const size_t lid = (size_t)m * a.G + uid;
        a.logprobs[lid * a.max_new + a.t[lid]] = zt - (Mx + logf(L));
      }
    }
    __syncthreads();
  }
  if (tid == 0) {
    if (consume)
      for (int s = 0; s < a.row_cap; ++s) {
        a.last_tok[s] = -1;
        a.last_fin[s] = 0;
      }
    // groups in ascending index; within a group the paper's order (R18)
    for (int m = 0; m < a.M; ++m) {
      long long* st = a.st + (size_t)m * ST_COUNT;
      int32_t* slot_uid = a.slot_uid + m * a.g;
      int32_t* slot_count = a.slot_count + m * a.g;
      int32_t* tt_ = a.t + (size_t)m * a.G;
      const int32_t* true_len = a.true_len + (size_t)m * a.G;
      int32_t* queue = a.queue + (size_t)m * a.G;
      int32_t* npages = a.npages + (size_t)m * a.G;
      int32_t* tokens = a.tokens + (size_t)m * a.G * a.max_new;
      const int32_t* pagetab = a.pagetab + (size_t)m * a.G * a.maxp;
      if (consume) {
        for (int s = 0; s < a.g; ++s) {
          const int uid = slot_uid[s];
          if (uid < 0 || (a.admit && a.stall[m * a.g + s])) continue;  // (a stalled slot decoded nothing)
          const int row = m * a.g + s;
          const uint32_t tok = 0xFFFFFFFFu - (uint32_t)(a.keys[row] & 0xFFFFFFFFull);
          tokens[(size_t)uid * a.max_new + tt_[uid]] = (int32_t)tok;
          a.last_tok[row] = (int32_t)tok;
          tt_[uid] += 1;
          st[ST_TOKENS] += 1;
        }
        for (int s = 0; s < a.g; ++s) {  // ascending slot index
          const int uid = slot_uid[s];
          if (uid < 0 || (a.admit && a.stall[m * a.g + s])) continue;
          if (tt_[uid] == true_len[uid] || (a.eos_on && tokens[(size_t)uid * a.max_new + tt_[uid] - 1] == a.eos_id)) {
            st[ST_DONE] += 1;
            a.done_flag[(size_t)m * a.G + uid] = 1;
            a.last_fin[m * a.g + s] = 1;
            for (int i = 0; i < npages[uid]; ++i) a.free_stack[st0[ST_FREE_TOP]++] = pagetab[(size_t)uid * a.maxp + i];
            st[ST_LIVE] -= npages[uid];
            st0[ST_GLIVE] -= npages[uid];
            npages[uid] = 0;
            if (st[ST_TARGET] > 0 && st[ST_DONE] >= st[ST_TARGET]) {
              // dynamic-slot stop (R35): every other slot's sample is discarded, ascending
              // slot order, its pages back to the pool; nothing is refilled
              slot_uid[s] = -1;
              for (int s2 = 0; s2 < a.g; ++s2) {
                const int u2 = slot_uid[s2];
                if (u2 < 0) continue;
                for (int i = 0; i < npages[u2]; ++i) a.free_stack[st0[ST_FREE_TOP]++] = pagetab[(size_t)u2 * a.maxp + i];
                st[ST_LIVE] -= npages[u2];
                st0[ST_GLIVE] -= npages[u2];
                npages[u2] = 0;
                slot_uid[s2] = -1;
                st[ST_DISCARDED] += 1;
              }
              st[ST_QHEAD] = st[ST_QLEN];
              break;
            }
          } else if (st[ST_STOPK] > 0 && tt_[uid] == st[ST_STOPK]) {
            // park: keep pages (prefix reuse)
          } else {
            continue;
          }
          slot_uid[s] = -1;
          slot_count[s] += 1;
          if (!a.admit && !st[ST_BARRIER] && st[ST_QHEAD] < st[ST_QLEN] &&
              (st[ST_QUOTA] == 0 || slot_count[s] < st[ST_QUOTA]))
            slot_uid[s] = queue[st[ST_QHEAD]++];
        }
        if (a.admit) admit_refill(a, st, m);  // (R41: finishes first, then one refill pass)
        bool idle = true;
        for (int s = 0; s < a.g; ++s) idle = idle && slot_uid[s] < 0;
        if (st[ST_BARRIER] && idle && st[ST_QHEAD] < st[ST_QLEN]) {
          for (int s = 0; s < a.g && st[ST_QHEAD] < st[ST_QLEN]; ++s) slot_uid[s] = queue[st[ST_QHEAD]++];
          idle = false;
        }
        if (st[ST_PHASE] == 0 && idle && st[ST_QHEAD] >= st[ST_QLEN] && st[ST_MAIN_PENDING]) {
          // prefix phase over: install the Alg. 2 plan (init fill + static SJF queue)
          for (int i = 0; i < st[ST_MAIN_QLEN]; ++i) queue[i] = a.main_queue[(size_t)m * a.G + i];
          st[ST_QLEN] = st[ST_MAIN_QLEN];
          st[ST_QHEAD] = 0;
          st[ST_BARRIER] = 0;
          st[ST_QUOTA] = 0;
          st[ST_STOPK] = 0;
          st[ST_PHASE] = 1;
          st[ST_MAIN_PENDING] = 0;
          for (int s = 0; s < a.g; ++s) {
            slot_count[s] = 0;
            slot_uid[s] = s < st[ST_MAIN_NINIT] ? a.main_init[m * a.g + s] : -1;
          }
        }
      }
      // pages for rows crossing a page boundary, ascending slot order (LIFO shared stack);
      // only for groups being prepared (all of them after a step; the new group at its start)
      if ((prep_mask >> m) & 1) {
        if (a.admit && !consume) admit_refill(a, st, m);  // the group's start: elastic admissions
        int held_e = 0;  // pages held by the elastic slots (R41)
        if (a.admit)
          for (int e = a.gp; e < a.g; ++e)
            if (slot_uid[e] >= 0) held_e += npages[slot_uid[e]];
        for (int s = 0; s < a.g; ++s) {
          int uid = slot_uid[s];
          if (a.admit) a.stall[m * a.g + s] = 0;
          if (uid < 0) continue;
          const int tt = tt_[uid];
          if (tt % a.pt == 0) {
            if (a.admit && s >= a.gp) {
              if (held_e >= a.E) {
                // no elastic page: the lowest idle guaranteed slot adopts the sample now (its
                // pages leave the elastic count), else it stalls this step
                int gs = -1;
                for (int q = 0; q < a.gp && gs < 0; ++q)
                  if (slot_uid[q] < 0) gs = q;
                if (gs < 0) {
                  a.stall[m * a.g + s] = 1;
                  st[ST_STALLS] += 1;
                  continue;
                }
                slot_uid[gs] = uid;
                slot_uid[s] = -1;
                held_e -= npages[uid];
              } else {
                ++held_e;
              }
            }
            if (st0[ST_FREE_TOP] == 0) {
              // budget violated: the pool is exhausted.  No page is handed out (nothing may
              // alias another sample's KV); the flag stops every row from the next step on
              // and the host calls report IS_ERR_BUDGET
              st0[ST_ERROR] = 1;
              continue;
            }
            a.pagetab[((size_t)m * a.G + uid) * a.maxp + tt / a.pt] = a.free_stack[--st0[ST_FREE_TOP]];
            npages[uid] += 1;
            st[ST_LIVE] += 1;
            st0[ST_GLIVE] += 1;
          }
        }
      }
    }
    int any = 0;
    for (int r = 0; r < a.M * a.g; ++r) any |= a.slot_uid[r] >= 0;
    s_any = st0[ST_ERROR] ? 0 : any;
  }
  __syncthreads();
  // ---- rows of the next step, one thread per row (row s = group m, slot s - m*g); after a
  // budget violation no row runs
  const bool any = s_any != 0;
  if (tid < a.row_cap) {
    const int s = tid;
    a.keys[s] = 0ull;
    const int m = s / a.g;
    const int uid = (m < a.M && any && !(a.admit && a.stall[s])) ? a.slot_uid[s] : -1;
    if (uid < 0) {
      a.row_active[s] = 0;
      a.row_uid[s] = 0;
      a.row_lid[s] = 0;
      a.row_t[s] = 0;
      a.row_tok[s] = 0;
      a.row_pos[s] = 0;
      a.row_kvloc[s] = 0;
      a.row_len[s] = 0;
    } else {
      const long long* st = a.st + (size_t)m * ST_COUNT;
      const int lid = m * a.G + uid;
      const int tt = a.t[lid];
      a.row_active[s] = 1;
      a.row_uid[s] = (int)st[ST_PROMPT_ID] * a.G + uid;
      a.row_lid[s] = lid;
      a.row_t[s] = tt;
      a.row_tok[s] = tt == 0 ? (int)st[ST_PROMPT_LAST] : a.tokens[(size_t)lid * a.max_new + tt - 1];
      a.row_pos[s] = a.P - 1 + tt;
      a.row_kvloc[s] = a.pagetab[(size_t)lid * a.maxp + tt / a.pt] * a.pt + tt % a.pt;
      a.row_len[s] = tt + 1;
    }
  }
  __syncthreads();
  {
    WorkList wl;
    wl.row_cap = a.row_cap;
    wl.chunk = a.chunk;
    wl.pt = a.pt;
    wl.Hkv = a.Hkv;
    wl.nc_pre = a.nc_pre;
    wl.tc_prefix = a.tc_prefix;
    wl.maxp = a.maxp;
    wl.row_active = a.row_active;
    wl.row_len = a.row_len;
    wl.row_lid = a.row_lid;
    wl.pagetab = a.pagetab;
    wl.items = a.attn_items;
    wl.n_items = st0 + ST_ATTN_ITEMS;
    build_attn_worklist(wl, s_cnt, &s_npre);
  }
  if (tid == 0) {
    for (int m = 0; m < a.M; ++m) {
      if (!((prep_mask >> m) & 1)) continue;
      long long* st = a.st + (size_t)m * ST_COUNT;
      bool gany = false;
      long long suf = 0;
      for (int s = m * a.g; s < m * a.g + a.g; ++s) {
        gany = gany || a.row_active[s];
        suf += a.row_len[s];
      }
      st[ST_SUFFIX] += suf;
      if (gany) {
        const long long step = st[ST_STEP];
        if (step < a.log_cap) {
          for (int s = 0; s < a.g; ++s) {
            const int u = a.slot_uid[m * a.g + s];  // (R41: a stalled slot is logged as -2 - uid)
            a.log_slot[((size_t)m * a.log_cap + step) * a.g + s] = (a.admit && u >= 0 && a.stall[m * a.g + s]) ? -2 - u : u;
          }
          a.log_live[(size_t)m * a.log_cap + step] = (int32_t)st[ST_LIVE];
        }
        st[ST_STEP] = step + 1;
        if (st[ST_PHASE] == 0) st[ST_PREFIX_STEPS] += 1;
        if (st[ST_LIVE] > st[ST_PEAK]) st[ST_PEAK] = st[ST_LIVE];
      }
    }
    if (any && consume) st0[ST_GSTEP] += 1;
    if (consume && a.pf_progress) *a.pf_progress = -1;  // the next step's prefetcher starts from its first GEMM
    if (st0[ST_GLIVE] > st0[ST_GPEAK]) st0[ST_GPEAK] = st0[ST_GLIVE];
  }
}

// Work list of one decode attention launch, alone (is_dbg_attn): one CTA of kSchedThreads.
__global__ void __launch_bounds__(kSchedThreads) attn_worklist_kernel(WorkList wl) {
  __shared__ int s_cnt[65];
  __shared__ int s_npre;
  build_attn_worklist(wl, s_cnt, &s_npre);
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

// Return every page still held by group m to the shared pool (a group slot is
// being restarted; its previous group may have been abandoned mid-way).
__global__ void reclaim_group_kernel(SchedArgs a, int m) {
  if (threadIdx.x != 0) return;
  long long* st0 = a.st + (size_t)a.M * ST_COUNT;
  long long* st = a.st + (size_t)m * ST_COUNT;
  for (int uid = 0; uid < a.G; ++uid) {
    int32_t* np = a.npages + (size_t)m * a.G + uid;
    for (int i = 0; i < *np; ++i) a.free_stack[st0[ST_FREE_TOP]++] = a.pagetab[((size_t)m * a.G + uid) * a.maxp + i];
    st0[ST_GLIVE] -= *np;
    *np = 0;
  }
  st[ST_LIVE] = 0;
  for (int s = 0; s < a.g; ++s) a.slot_uid[m * a.g + s] = -1;
}

// Benchmark reward (R29) and length per sample.  A sample that did not complete
// (dynamic mode, R35: discarded in flight or never started) reports length 0 and
// reward 0; a completed one its emitted length (true_len, or shorter at EOS, R37).
__global__ void results_kernel(const int32_t* __restrict__ tokens, const int32_t* __restrict__ true_len,
                               const uint8_t* __restrict__ done, int G, int max_new, int vocab, float* reward,
                               int32_t* len) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= G) return;
  if (!done[i]) {
    reward[i] = 0.f;
    len[i] = 0;
    return;
  }
  int c = 0, L = 0;
  const int T = true_len[i];
  while (L < T && tokens[(size_t)i * max_new + L] >= 0) {
    c += tokens[(size_t)i * max_new + L] < vocab / 2;
    ++L;
  }
  reward[i] = L ? (float)c / (float)L : 0.f;
  len[i] = L;
}

__global__ void bf16_to_f32_kernel(const __nv_bfloat16* __restrict__ x, float* __restrict__ y, int n) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) y[i] = __bfloat162float(x[i]);
}


// ------------------------------------------------------------------ top-p < 1 (NEXT-4, DESIGN R36)
// exp(d), d <= 0: the fixed fp32 op sequence of R36 (Cody-Waite split, degree-6 Taylor
// polynomial in Horner form, times 2^n; 0 below 2^-125), explicit _rn intrinsics.
__device__ __forceinline__ float expf_is(float d) {
  const float n = rintf(__fmul_rn(d, __uint_as_float(0x3FB8AA3Bu)));  // fl32(log2 e)
  float r = __fsub_rn(d, __fmul_rn(n, __uint_as_float(0x3F317200u)));
  r = __fsub_rn(r, __fmul_rn(n, __uint_as_float(0x35BFBE8Eu)));
  float p = __uint_as_float(0x3AB60B61u);                          // fl32(1/720)
  p = __fadd_rn(__fmul_rn(r, p), __uint_as_float(0x3C088889u));  // 1/120
  p = __fadd_rn(__fmul_rn(r, p), __uint_as_float(0x3D2AAAABu));  // 1/24
  p = __fadd_rn(__fmul_rn(r, p), __uint_as_float(0x3E2AAAABu));  // 1/6
  p = __fadd_rn(__fmul_rn(r, p), 0.5f);
  p = __fadd_rn(__fmul_rn(r, p), 1.0f);
  p = __fadd_rn(__fmul_rn(r, p), 1.0f);
  const int ni = (int)n;
  if (ni < -125) return 0.f;
  return __fmul_rn(p, __uint_as_float((uint32_t)(ni + 127) << 23));
}

__device__ __forceinline__ unsigned long long topp_w(float e) {
  return (unsigned long long)__fmul_rn(e, 17592186044416.0f /* 2^44 */);  // exact, then truncation = floor
}

constexpr int kToppThreads = 1024;
constexpr int kToppBlocks = 16;  // vocabulary slices per row for the parallel passes

// Exact 64-bit mass histograms from 32-bit shared atomics: w < 2^45 is kept as three
// 15-bit limbs; a slice holds < 2^14 elements, so every limb sum stays below 2^29.
struct ToppHist {
  unsigned int l[3][256];
  __device__ __forceinline__ void clear(int tid) {
    if (tid < 256) l[0][tid] = l[1][tid] = l[2][tid] = 0u;
  }
  __device__ __forceinline__ void add(uint32_t d, unsigned long long w) {
    if (!w) return;
    atomicAdd(&l[0][d], (unsigned)(w & 0x7FFFull));
    atomicAdd(&l[1][d], (unsigned)((w >> 15) & 0x7FFFull));
    atomicAdd(&l[2][d], (unsigned)(w >> 30));
  }
  __device__ __forceinline__ unsigned long long get(int d) const {
    return (unsigned long long)l[0][d] + ((unsigned long long)l[1][d] << 15) + ((unsigned long long)l[2][d] << 30);
  }
};

struct ToppArgs {
  const float* scores;       // [rows][V] fl(fl(z * invT) + G_v) from the lm_head epilogue
  const float* logits;       // [rows][V] z
  const float4* lp_mlz;      // [rows][lp_grid] lm_head per-CTA (max z, ...): the row max
  int lp_grid;
  uint32_t* ebits;           // [rows][V] bits of e_v
  unsigned long long* wpart; // [rows][kToppBlocks] integer mass per slice
  unsigned long long* hist1; // [rows][kToppBlocks][256] level-1 (top byte) mass histogram per slice
  int2* sel;                 // [rows] (boundary bits e*, last boundary member v_k)
  const int32_t* row_active;
  unsigned long long* keys;  // [rows]
  int V;
  float invT, top_p;
};

// Pass A (rows x kToppBlocks CTAs): e_v bits, the slice's integer mass and its top-byte
// histogram.  max u = fl(max z * invT) (rounding is monotonic), max z from the lm_head partials.
__global__ void __launch_bounds__(kToppThreads) topp_prep_kernel(ToppArgs a) {
  pdl_launch_dependents();
  pdl_wait();
  const int row = blockIdx.y;
  if (!a.row_active[row]) return;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  __shared__ float s_f[32];
  __shared__ unsigned long long s_u[32];
  __shared__ ToppHist hist;
  hist.clear(tid);
  float mz = -INFINITY;
  for (int c = tid; c < a.lp_grid; c += kToppThreads) mz = fmaxf(mz, a.lp_mlz[(size_t)row * a.lp_grid + c].x);
  mz = warp_max(mz);
  if (lane == 0) s_f[wid] = mz;
  __syncthreads();
  mz = s_f[0];
  for (int w = 1; w < kToppThreads / 32; ++w) mz = fmaxf(mz, s_f[w]);
  const float mx = __fmul_rn(mz, a.invT);
  const int per = (a.V + kToppBlocks - 1) / kToppBlocks;
  const int lo = blockIdx.x * per, hi = min(a.V, lo + per);
  const float* z = a.logits + (size_t)row * a.V;
  uint32_t* eb = a.ebits + (size_t)row * a.V;
  unsigned long long wsum = 0;
  for (int b0 = lo; b0 < hi; b0 += kToppThreads) {
    const int v = b0 + tid;
    float e = 0.f;
    if (v < hi) {
      e = expf_is(__fsub_rn(__fmul_rn(z[v], a.invT), mx));
      eb[v] = __float_as_uint(e);
    }
    const unsigned long long w = topp_w(e);
    wsum += w;
    if (v < hi) hist.add(__float_as_uint(e) >> 24, w);  // level-1 digit: the top byte
  }
  for (int o = 16; o > 0; o >>= 1) wsum += __shfl_xor_sync(0xffffffffu, wsum, o);
  if (lane == 0) s_u[wid] = wsum;
  __syncthreads();
  if (tid == 0) {
    unsigned long long W = 0;
    for (int w = 0; w < kToppThreads / 32; ++w) W += s_u[w];
    a.wpart[row * kToppBlocks + blockIdx.x] = W;
  }
  if (tid < 256) a.hist1[((size_t)row * kToppBlocks + blockIdx.x) * 256 + tid] = hist.get(tid);
}

// Pass B, level by level (radix select of the boundary value e*, most significant byte
// first): topp_pick_kernel sums the slices' histograms of the current byte and picks the
// byte (one CTA per row); topp_hist_kernel builds the next byte's per-slice histograms over
// the elements that match the picked prefix (rows x kToppBlocks CTAs, equal digits of a warp
// combined as in pass A).  Level 1's histograms come from pass A.
struct ToppState {
  unsigned long long thr, above;  // nucleus threshold; integer mass strictly above the prefix
  uint32_t prefix, mask;          // picked bytes of e*
};

__global__ void __launch_bounds__(256) topp_pick_kernel(ToppArgs a, ToppState* stt, int shift) {
  pdl_launch_dependents();
  pdl_wait();
  const int row = blockIdx.x;
  if (!a.row_active[row]) return;
  const int tid = threadIdx.x;
  __shared__ unsigned long long hist[256];
  unsigned long long h = 0;
  for (int b = 0; b < kToppBlocks; ++b) h += a.hist1[((size_t)row * kToppBlocks + b) * 256 + tid];
  hist[tid] = h;
  __syncthreads();
  if (tid == 0) {
    ToppState t = stt[row];
    if (shift == 24) {
      unsigned long long W = 0;
      for (int b = 0; b < kToppBlocks; ++b) W += a.wpart[row * kToppBlocks + b];
      t.thr = (unsigned long long)ceil(__dmul_rn((double)a.top_p, __ull2double_rn(W)));
      t.above = 0;
      t.prefix = 0;
      t.mask = 0;
      a.keys[row] = 0ull;  // pass C's atomicMax starts from zero
    }
    unsigned long long acc = t.above;
    int d = 255;
    for (; d > 0; --d) {
      if (acc + hist[d] >= t.thr) break;
      acc += hist[d];
    }
    t.above = acc;
    t.prefix |= (uint32_t)d << shift;
    t.mask |= 255u << shift;
    stt[row] = t;
  }
}

__global__ void __launch_bounds__(kToppThreads) topp_hist_kernel(ToppArgs a, const ToppState* stt, int shift) {
  pdl_launch_dependents();
  pdl_wait();
  const int row = blockIdx.y;
  if (!a.row_active[row]) return;
  const int tid = threadIdx.x;
  __shared__ ToppHist hist;
  hist.clear(tid);
  __syncthreads();
  const uint32_t prefix = stt[row].prefix, mask = stt[row].mask;
  const int per = (a.V + kToppBlocks - 1) / kToppBlocks;
  const int lo = blockIdx.x * per, hi = min(a.V, lo + per);
  const uint32_t* eb = a.ebits + (size_t)row * a.V;
  for (int b0 = lo; b0 < hi; b0 += kToppThreads) {
    const int v = b0 + tid;
    const uint32_t b = v < hi ? __ldcg(eb + v) : 0xFFFFFFFFu;
    if (v < hi && (b & mask) == prefix) hist.add((b >> shift) & 255u, topp_w(__uint_as_float(b)));
  }
  __syncthreads();
  if (tid < 256) a.hist1[((size_t)row * kToppBlocks + blockIdx.x) * 256 + tid] = hist.get(tid);
}

// Boundary members (e == e*) per slice, then the need-th one in ascending v: the slice that
// holds it is found from the counts, and one CTA scans that slice with contiguous ranges.
__global__ void __launch_bounds__(kToppThreads) topp_tiecount_kernel(ToppArgs a, const ToppState* stt) {
  pdl_launch_dependents();
  pdl_wait();
  const int row = blockIdx.y;
  if (!a.row_active[row]) return;
  const uint32_t bstar = stt[row].prefix;
  const int per = (a.V + kToppBlocks - 1) / kToppBlocks;
  const int lo = blockIdx.x * per, hi = min(a.V, lo + per);
  const uint32_t* eb = a.ebits + (size_t)row * a.V;
  int cnt = 0;
  for (int v = lo + threadIdx.x; v < hi; v += kToppThreads) cnt += __ldcg(eb + v) == bstar;
  __shared__ int s_c[kToppThreads / 32];
  for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
  if ((threadIdx.x & 31) == 0) s_c[threadIdx.x >> 5] = cnt;
  __syncthreads();
  if (threadIdx.x == 0) {
    int t = 0;
    for (int w = 0; w < kToppThreads / 32; ++w) t += s_c[w];
    reinterpret_cast<int*>(a.wpart)[row * kToppBlocks + blockIdx.x] = t;  // (pass A's masses are consumed)
  }
}

__global__ void __launch_bounds__(kToppThreads) topp_tiepick_kernel(ToppArgs a, const ToppState* stt) {
  pdl_launch_dependents();
  pdl_wait();
  const int row = blockIdx.x;
  if (!a.row_active[row]) return;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const ToppState t = stt[row];
  const uint32_t bstar = t.prefix;
  const unsigned long long wb = topp_w(__uint_as_float(bstar));
  const unsigned long long need = wb ? (t.thr - t.above + wb - 1) / wb : 1;  // boundary members (>= 1)
  const int* cnts = reinterpret_cast<const int*>(a.wpart) + row * kToppBlocks;
  int blk = kToppBlocks - 1;
  unsigned long long before = 0;
  for (int b = 0; b < kToppBlocks; ++b) {
    if (before + (unsigned long long)cnts[b] >= need) {
      blk = b;
      break;
    }
    before += cnts[b];
  }
  const int per = (a.V + kToppBlocks - 1) / kToppBlocks;
  const int lo = blk * per, hi = min(a.V, lo + per);
  const int pt = (hi - lo + kToppThreads - 1) / kToppThreads;
  const int r0 = min(hi, lo + tid * pt), r1 = min(hi, r0 + pt);
  const uint32_t* eb = a.ebits + (size_t)row * a.V;
  int cnt = 0;
  for (int v = r0; v < r1; ++v) cnt += __ldcg(eb + v) == bstar;
  __shared__ int s_cnt[kToppThreads / 32];
  __shared__ int s_vk;
  int incl = cnt;
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  if (lane == 31) s_cnt[wid] = incl;
  if (tid == 0) s_vk = hi - 1;
  __syncthreads();
  unsigned long long bef = before + (unsigned long long)(incl - cnt);
  for (int w = 0; w < wid; ++w) bef += s_cnt[w];
  if (bef < need && bef + (unsigned long long)cnt >= need) {
    unsigned long long k = bef;
    for (int v = r0; v < r1; ++v)
      if (__ldcg(eb + v) == bstar && ++k == need) {
        s_vk = v;
        break;
      }
  }
  __syncthreads();
  if (tid == 0) a.sel[row] = make_int2((int)bstar, s_vk);
}

// Pass C (rows x kToppBlocks CTAs): Gumbel-max over the nucleus with the lm_head's scores.
__global__ void __launch_bounds__(kToppThreads) topp_sample_kernel(ToppArgs a) {
  pdl_launch_dependents();
  pdl_wait();
  const int row = blockIdx.y;
  if (!a.row_active[row]) return;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  __shared__ unsigned long long s_u[32];
  const int2 sl = a.sel[row];
  const uint32_t bstar = (uint32_t)sl.x;
  const int per = (a.V + kToppBlocks - 1) / kToppBlocks;
  const int lo = blockIdx.x * per, hi = min(a.V, lo + per);
  const uint32_t* eb = a.ebits + (size_t)row * a.V;
  const float* sc = a.scores + (size_t)row * a.V;
  unsigned long long best = 0;
  for (int v = lo + tid; v < hi; v += kToppThreads) {
    const uint32_t b = eb[v];
    if (b > bstar || (b == bstar && v <= sl.y)) {
      const unsigned long long k = order_key(sc[v], (uint32_t)v);
      best = k > best ? k : best;
    }
  }
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long y = __shfl_xor_sync(0xffffffffu, best, o);
    best = y > best ? y : best;
  }
  if (lane == 0) s_u[wid] = best;
  __syncthreads();
  if (tid == 0) {
    for (int w = 1; w < kToppThreads / 32; ++w) best = s_u[w] > best ? s_u[w] : best;
    if (best) atomicMax(a.keys + row, best);
  }
}

// Test hook for the top-p chain on caller logits: per row, the lm_head's contribution
// (Gumbel scores, and the row max as a one-entry partial list).
__global__ void __launch_bounds__(kToppThreads) topp_dbg_scores_kernel(const float* __restrict__ z, int V,
                                                                       const int32_t* __restrict__ uid,
                                                                       const int32_t* __restrict__ t, uint64_t seed,
                                                                       float invT, float* scores, float4* mlz) {
  const int row = blockIdx.x, tid = threadIdx.x;
  __shared__ float s_f[32];
  float mz = -INFINITY;
  for (int v = tid; v < V; v += kToppThreads) {
    const float x = z[(size_t)row * V + v];
    mz = fmaxf(mz, x);
    scores[(size_t)row * V + v] = __fadd_rn(__fmul_rn(x, invT), gumbel(seed, (uint32_t)uid[row], (uint32_t)t[row], (uint32_t)v));
  }
  mz = warp_max(mz);
  if ((tid & 31) == 0) s_f[tid >> 5] = mz;
  __syncthreads();
  if (tid == 0) {
    for (int w = 1; w < kToppThreads / 32; ++w) mz = fmaxf(mz, s_f[w]);
    mz = fmaxf(mz, s_f[0]);
    mlz[row] = make_float4(mz, 0.f, 0.f, 0.f);
  }
}
}  // namespace isk
