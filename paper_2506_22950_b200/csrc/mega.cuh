// Persistent decode kernel: the whole layer stack of one decode step
// (embed, RMSNorm, QKV + QK-norm + RoPE + KV append,
// split shared-prefix / per-slot suffix attention with LSE merge, o_proj +
// residual, RMSNorm, gate/up + SwiGLU, down + residual, final RMSNorm) in ONE
// launch of one CTA per SM.
//
// Why: at decode the per-layer GEMMs move 8-50 MB each, a few microseconds of
// HBM time, so per-kernel launch/ramp/drain latency dominated the per-op step
// (profiles/r01).  Here the weight stream never stops at an operator boundary:
//
//   warp 0      TMA producer.  Walks this CTA's static task list and streams
//               every weight tile it will need into an NA-deep shared-memory
//               ring with 1-D bulk copies (cp.async.bulk, 16 KB per stage) from a
//               pre-swizzled tile-major weight copy.  Weights never depend on
//               the activations, so it runs ahead across layer boundaries and
//               only blocks on ring space.
//   warp 1      tcgen05 MMA issuer (one elected lane): D[128 x BN] (TMEM, fp32)
//               += W_tile[128 x 64] . X^T[64 x BN] per ring stage (swap-AB:
//               output features are the M = 128 operand, the R <= 64 decode
//               rows are N).
//   warps 2-9   two compute warp groups (WG0, WG1) that take alternate GEMM
//               units: wait for the unit's inputs (release/acquire counters in
//               global memory), bulk-copy its activation k-blocks into the WG's
//               B ring, read the accumulator from TMEM, exchange split-K partials
//               through L2 (the last arriving unit of a tile reduces them in
//               fixed part order -> deterministic, batch invariant) and run the
//               fused epilogue.  Both WGs also execute attention units, grabbed
//               dynamically per layer.
//
// Activations that feed a GEMM are written by their producer directly in the
// MMA's 128-byte-swizzled K-major layout ([k-block][BN rows][64]), so B
// operands are plain bulk copies.  RMSNorm is folded through the GEMM: the
// producer of the residual writes bf16(x * gain) and per-(128-column tile, row)
// partial sums of squares; the consumer's epilogue multiplies its accumulator
// by rs[row] = 1/sqrt(sum/H + eps) (RMSNorm's row scale commutes with the
// GEMM; R12a).
//
// Dependencies (all within one step, zeroed by the lm_head kernel that follows):
//   QKV(l)  <- all DN(l-1) tiles (or all EMBED rows)         dn_done / emb_done
//   ATT(l)h <- QKV(l) q tiles of kv head h, its k and v tiles qkv_flag
//   O(l)    <- merged attention of the kv heads in its K range att_done
//   GU(l)   <- all O(l) tiles                                  o_done
//   DN(l)   <- GU(l) tiles of its K range (GU tile t = DN k-block t)  gu_flag
//   FINAL   <- all DN(L-1) tiles
// Every wait targets work that precedes it in one global order that every CTA's
// list follows, and all CTAs are co-resident, so there is no cycle.  Every wait
// is bounded (4 s, then __trap) so a logic error aborts instead of hanging.
#pragma once
#include "common.cuh"
#include "gemm.cuh"
#include "kernels.cuh"

namespace isk {

enum MkKind { MK_EMBED = 0, MK_QKV = 1, MK_ATT = 2, MK_O = 3, MK_GU = 4, MK_DN = 5, MK_FINAL = 6 };
constexpr int kMkThreads = 320;
constexpr int kMkPC = 32;  // shared-prefix tokens per attention unit (all live rows of the group)
constexpr int kMkSC = 32;  // suffix tokens per attention unit (one slot)
constexpr int kMkStage = 16384;

struct MkGemm {
  int M, KB, T, S;   // output features, k-blocks, 128-row tiles, K split
  long long w_off;   // element offset inside a layer's packed block
};

struct MkSync {
  int stride;                                 // ints per layer
  int att_next, o_done, dn_done, emb_done;    // scalars
  int qkv_flag, att_row, att_done, gu_flag;    // arrays
};

struct MkArgs {
  const int4* tasks;     // per-CTA task lists, concatenated
  const int* task_off;   // [grid + 1]
  const __nv_bfloat16* wpk;  // packed weights [L][QKV | O | GU | DN], tile-major, swizzled
  long long layer_stride;
  MkGemm g[4];           // QKV, O, GU, DN
  int L, H, F, Hq, Hkv, rc, Th, na, nb, scratch;
  float eps, scale;
  const __nv_bfloat16* embed;  // [V][H]
  const float *in_norm, *post_norm, *q_norm, *k_norm, *final_norm;  // [L][H], [L][H], [L][128], [L][128], [H]
  const __nv_bfloat16 *in_norm_bf, *post_norm_bf;                     // the same gains as bf16 (exact) [L][H]
  const float *rope_cos, *rope_sin;
  const int32_t *row_active, *row_tok, *row_pos, *row_kvloc, *row_len, *row_lid;
  float *resid0, *resid1, *ssq;   // [rc][H] x2, [2L+1][Th][rc]
  __nv_bfloat16 *attn_sw, *act_sw;  // O / DN inputs [Hq*128/64][BN][64], [F/64][BN][64]
  __nv_bfloat16 *q, *xn_final;    // [rc][Hq][128], [rows][H] (lm_head input, row-major)
  const __nv_bfloat16* prefix;    // [L][2][Hkv][pcap][128]
  long long prefix_layer;
  __nv_bfloat16* pool;            // [L][pages][2][Hkv][pt][128]
  long long pool_layer;
  const int32_t* pagetab;
  int maxp, pt, pcap, nc_pre, NCm;
  float *part_o, *part_ml;        // [rc][Hq][NCm][128], [rc][Hq][NCm][2]
  int* sync;
  MkSync so;
  unsigned long long* clock;      // [2]: accumulated kernel ns, launches (CTA 0)
  int pf_units;                   // GEMM units of weights prefetched into L2 ahead of the ring
  int nodeps;                     // timing experiment only (IS_MK_NODEPS): skip every dependency wait
  unsigned long long* trace;      // debug (IS_MK_TRACE): [grid][4 roles][trace_cap][2] (globaltimer, code)
  int trace_cap;
};

// debug timeline record: role 0/1 = compute WG, 2 = producer, 3 = MMA
IS_DEVICE void mk_rec(const MkArgs& a, int role, int& n, int type, int idx) {
  if (!a.trace) return;
  if (n < a.trace_cap) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    unsigned long long* p = a.trace + (((size_t)blockIdx.x * 4 + role) * a.trace_cap + n) * 2;
    p[0] = t;
    p[1] = ((unsigned long long)type << 32) | (unsigned)idx;
  }
  ++n;
}

// ---------------------------------------------------------------- sync helpers
IS_DEVICE unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
IS_DEVICE int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
IS_DEVICE void red_release_add(int* p, int v) {
  asm volatile("red.release.gpu.global.add.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
IS_DEVICE int atom_acqrel_add(int* p, int v) {
  int old;
  asm volatile("atom.acq_rel.gpu.global.add.s32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}
IS_DEVICE void mk_trap(const char* what, int a0, int a1) {
  printf("infsamp persistent decode kernel: wait timed out (%s %d %d) block %d thread %d\n", what, a0, a1,
         (int)blockIdx.x, (int)threadIdx.x);
  __trap();
}
constexpr unsigned long long kMkTimeoutNs = 4000000000ull;
IS_DEVICE void spin_ge(const int* p, int target, int tag) {
  if (ld_acquire(p) >= target) return;
  const unsigned long long t0 = gtimer();
  while (ld_acquire(p) < target) {
    __nanosleep(64);
    if (gtimer() - t0 > kMkTimeoutNs) mk_trap("counter", tag, target);
  }
}
#define mk_spin(a, p, t, tag) \
  do {                         \
    if (!(a).nodeps) spin_ge((p), (t), (tag)); \
  } while (0)
IS_DEVICE bool mbar_try(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n.reg .pred p;\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, 1000000;\n"
      "selp.u32 %0, 1, 0, p;\n}\n"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
IS_DEVICE void mk_wait(uint64_t* bar, uint32_t parity, int tag) {
  if (mbar_try(bar, parity)) return;
  const unsigned long long t0 = gtimer();
  while (!mbar_try(bar, parity))
    if (gtimer() - t0 > kMkTimeoutNs) mk_trap("mbarrier", tag, (int)parity);
}
IS_DEVICE void bulk_g2s_hint(void* smem, const void* gmem, uint32_t bytes, uint64_t* bar, uint64_t hint) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_u32(smem)),
      "l"(gmem), "r"(bytes), "r"(smem_u32(bar)), "l"(hint)
      : "memory");
}
IS_DEVICE void prefetch_l2(const void* gmem, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(gmem), "r"(bytes) : "memory");
}
IS_DEVICE void fence_proxy_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
IS_DEVICE void fence_proxy_async_global() { asm volatile("fence.proxy.async.global;" ::: "memory"); }
// named barrier of one compute warp group (128 threads)
IS_DEVICE void wg_bar(int wg) { asm volatile("bar.sync %0, 128;" ::"r"(1 + wg) : "memory"); }

// element offset of (row n, column k) in a [k/64][BN][64] 128-byte-swizzled operand
IS_DEVICE int sw_off(int n, int k, int BN) {
  const int kb = k >> 6, c = (k >> 3) & 7;
  return (kb * BN + n) * 64 + ((c ^ (n & 7)) << 3) + (k & 7);
}

// Per-WG scratch (union of the epilogue and attention views) + control words.
template <int BN, int REP>
struct MkScratch {
  // epilogue view
  static constexpr int kStg = BN * 128 * 4;       // stg[BN][128] fp32
  static constexpr int kRed = 4 * 64 * 4;         // sred[4][64]
  // attention view
  static constexpr int kKV = 2 * 32 * kHD * 2;    // K, V [32][128] bf16
  static constexpr int kQ = 4 * REP * kHD * 4;    // qs[4 warps][REP][128]
  static constexpr int kComb = 4 * REP * (kHD + 2) * 4;
  static constexpr int kEpi = kStg + kRed;
  static constexpr int kAtt = kKV + kQ + kComb;
  static constexpr int kCtl = 1024 + 5 * 256 + 2048;  // rs, rows, cum, ctl | row tables | gains (bf16, 16 k-blocks)
  static constexpr int v = (((kEpi > kAtt ? kEpi : kAtt) + kCtl) + 1023) / 1024 * 1024;
};

template <int BN, int REP>
struct MkWG {
  float* stg;
  float* sred;
  __nv_bfloat16 *Ks, *Vs;
  float *qs, *comb;
  float* rs;
  int *rows, *cum, *ctl;
  int *ract, *rpos, *rkv, *rlen, *rlid;  // this step's row tables (static during the kernel)
  __nv_bfloat16* gsm;                    // RMSNorm gains of the current unit's K range
  IS_DEVICE void init(uint8_t* base) {
    using S = MkScratch<BN, REP>;
    stg = reinterpret_cast<float*>(base);
    sred = reinterpret_cast<float*>(base + S::kStg);
    Ks = reinterpret_cast<__nv_bfloat16*>(base);
    Vs = Ks + 32 * kHD;
    qs = reinterpret_cast<float*>(base + S::kKV);
    comb = reinterpret_cast<float*>(base + S::kKV + S::kQ);
    uint8_t* c = base + (S::kEpi > S::kAtt ? S::kEpi : S::kAtt);
    rs = reinterpret_cast<float*>(c);
    rows = reinterpret_cast<int*>(c + 256);
    cum = reinterpret_cast<int*>(c + 512);
    ctl = reinterpret_cast<int*>(c + 512 + 288);
    ract = reinterpret_cast<int*>(c + 1024);
    rpos = ract + 64;
    rkv = rpos + 64;
    rlen = rkv + 64;
    rlid = rlen + 64;
    gsm = reinterpret_cast<__nv_bfloat16*>(rlid + 64);
  }
};

// rs[n] = 1 / sqrt(sum_t ssq[ver][t][n] / H + eps) for n < rc (fixed tile order)
IS_DEVICE void mk_row_scale(const MkArgs& a, int ver, float* rs, int wt) {
  if (wt < a.rc) {
    const float* s = a.ssq + (size_t)ver * a.Th * a.rc + wt;
    float ss = 0.f;
#pragma unroll 1
    for (int t0 = 0; t0 < a.Th; t0 += 16) {
      float t16[16];
#pragma unroll
      for (int t = 0; t < 16; ++t) t16[t] = t0 + t < a.Th ? __ldcg(s + (size_t)(t0 + t) * a.rc) : 0.f;
#pragma unroll
      for (int t = 0; t < 16; ++t) ss += t16[t];
    }
    rs[wt] = 1.0f / sqrtf(ss / (float)a.H + a.eps);
  }
}

// ---------------------------------------------------------------- attention units
// q row r, heads h*REP.. -> per-warp smem fp32 [REP][128] (L2 loads: q is rewritten every layer)
template <int REP>
IS_DEVICE void mk_load_q(const MkArgs& a, int r, int h, float* qs, int lane) {
  uint2 b[REP];
#pragma unroll
  for (int e = 0; e < REP; ++e)
    b[e] = __ldcg(reinterpret_cast<const uint2*>(a.q + ((size_t)r * a.Hq + h * REP + e) * kHD) + lane);
#pragma unroll
  for (int e = 0; e < REP; ++e) {
    const float2 f0 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&b[e].x));
    const float2 f1 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&b[e].y));
    reinterpret_cast<float4*>(qs + e * kHD)[lane] = make_float4(f0.x, f0.y, f1.x, f1.y);
  }
}

template <int REP>
IS_DEVICE void mk_fetch_q(const MkArgs& a, int r, int h, uint2 (&b)[REP], int lane) {
#pragma unroll
  for (int e = 0; e < REP; ++e)
    b[e] = __ldcg(reinterpret_cast<const uint2*>(a.q + ((size_t)r * a.Hq + h * REP + e) * kHD) + lane);
}
template <int REP>
IS_DEVICE void mk_put_q(const uint2 (&b)[REP], float* qs, int lane) {
#pragma unroll
  for (int e = 0; e < REP; ++e) {
    const float2 f0 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&b[e].x));
    const float2 f1 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&b[e].y));
    reinterpret_cast<float4*>(qs + e * kHD)[lane] = make_float4(f0.x, f0.y, f1.x, f1.y);
  }
}

template <int REP>
IS_DEVICE void mk_store_partial(const MkArgs& a, int r, int h, int slot, const float (&m)[REP], const float (&l)[REP],
                                const float (&o)[REP][4], int lane) {
#pragma unroll
  for (int e = 0; e < REP; ++e) {
    const size_t pidx = ((size_t)r * a.Hq + h * REP + e) * a.NCm + slot;
    const float inv = l[e] > 0.f ? 1.0f / l[e] : 0.f;
    __stcg(reinterpret_cast<float4*>(a.part_o + pidx * kHD) + lane,
           make_float4(o[e][0] * inv, o[e][1] * inv, o[e][2] * inv, o[e][3] * inv));
    if (lane == 0) __stcg(reinterpret_cast<float2*>(a.part_ml + pidx * 2), make_float2(m[e], l[e]));
  }
}

// LSE merge (R8) of (row r, kv head h): warp e handles query head h*REP + e;
// partials in fixed order (prefix chunks, then suffix chunks).  Output goes to
// the o_proj operand in its swizzled layout.
template <int BN>
IS_DEVICE void mk_merge(const MkArgs& a, int r, int qh, int len, int lane) {
  const int nsuf = (len + kMkSC - 1) / kMkSC;
  const int n = a.nc_pre + nsuf;  // <= 64
  const size_t base = ((size_t)r * a.Hq + qh) * a.NCm;
  float m0 = -INFINITY, l0 = 0.f, m1 = -INFINITY, l1 = 0.f;
  if (lane < n) {
    const float2 v = __ldcg(reinterpret_cast<const float2*>(a.part_ml + (base + lane) * 2));
    m0 = v.x;
    l0 = v.y;
  }
  if (lane + 32 < n) {
    const float2 v = __ldcg(reinterpret_cast<const float2*>(a.part_ml + (base + lane + 32) * 2));
    m1 = v.x;
    l1 = v.y;
  }
  const float M = warp_max(fmaxf(m0, m1));
  const float w0 = (lane < n && m0 != -INFINITY) ? expf(m0 - M) * l0 : 0.f;
  const float w1 = (lane + 32 < n && m1 != -INFINITY) ? expf(m1 - M) * l1 : 0.f;
  const float den = warp_sum(w0) + warp_sum(w1);
  float4 num = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll 1
  for (int i0 = 0; i0 < n; i0 += 16) {
    float4 o[16];
#pragma unroll
    for (int k = 0; k < 16; ++k)
      o[k] = (i0 + k < n) ? __ldcg(reinterpret_cast<const float4*>(a.part_o + (base + i0 + k) * kHD) + lane)
                          : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
    for (int k = 0; k < 16; ++k) {
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
  const float inv = den > 0.f ? 1.0f / den : 0.f;
  const int k = qh * kHD + 4 * lane;
  __nv_bfloat162* dst = reinterpret_cast<__nv_bfloat162*>(a.attn_sw + sw_off(r, k, BN));
  dst[0] = __floats2bfloat162_rn(num.x * inv, num.y * inv);
  dst[1] = __floats2bfloat162_rn(num.z * inv, num.w * inv);
}

// One attention unit (prefix chunk shared by every live row, or one slot's
// suffix chunk), executed by one compute WG; the unit that completes a
// (row, kv head) merges it.
template <int BN, int REP>
IS_DEVICE void mk_att_unit(const MkArgs& a, MkWG<BN, REP>& S, int l, int u, int n_pre_units, int wg, int wt,
                           uint64_t* attbar, uint32_t& attph) {
  const int wwarp = wt >> 5, lane = wt & 31;
  int* sl = a.sync + (size_t)l * a.so.stride;
  int h, c, r = -1;
  if (u < n_pre_units) {
    h = u / a.nc_pre;
    c = u % a.nc_pre;
  } else {
    const int j = u - n_pre_units;
    h = j % a.Hkv;
    const int k = j / a.Hkv;
    r = 0;
    while (S.cum[r + 1] <= k) ++r;
    c = k - S.cum[r];
  }
  const bool prefix = r < 0;
  if (wt == 0) {
    fence_proxy_async_smem();  // generic writes to this scratch precede the bulk copies below
    // static K / V first: the shared prefix, and suffix chunks that do not hold this step's token
    const int len = prefix ? 0 : S.rlen[r];
    const bool cur = !prefix && (len - 1) / kMkSC == c;  // chunk holds the token appended this step
    if (prefix) {
      const int tok0 = c * kMkPC, ntok = min(kMkPC, a.pcap - tok0);
      const uint32_t bytes = (uint32_t)ntok * kHD * 2;
      const __nv_bfloat16* kp = a.prefix + (size_t)l * a.prefix_layer + ((size_t)h * a.pcap + tok0) * kHD;
      mbar_arrive_expect_tx(attbar, 2 * bytes);
      bulk_g2s_hint(S.Ks, kp, bytes, attbar, kEvictNormal);
      bulk_g2s_hint(S.Vs, kp + (size_t)a.Hkv * a.pcap * kHD, bytes, attbar, kEvictNormal);
    }
    // inputs: q tiles of kv head h (+ its k / v tiles when the chunk holds the appended token)
    for (int e = 0; e < REP; ++e) mk_spin(a, sl + a.so.qkv_flag + h * REP + e, 4, 100 + l);
    if (cur) {
      mk_spin(a, sl + a.so.qkv_flag + a.Hq + h, 4, 200 + l);
      mk_spin(a, sl + a.so.qkv_flag + a.Hq + a.Hkv + h, 4, 300 + l);
      fence_proxy_async_global();
    }
    if (!prefix) {
      const int tok0 = c * kMkSC, tend = min(tok0 + kMkSC, len);
      const int lid = S.rlid[r];
      const __nv_bfloat16* pl = a.pool + (size_t)l * a.pool_layer;
      mbar_arrive_expect_tx(attbar, (uint32_t)(tend - tok0) * kHD * 2 * 2);
      for (int t = tok0; t < tend;) {
        const int off = t % a.pt, seg = min(a.pt - off, tend - t);
        const int page = __ldg(a.pagetab + (size_t)lid * a.maxp + t / a.pt);
        const __nv_bfloat16* kp = pl + ((((size_t)page * 2 + 0) * a.Hkv + h) * a.pt + off) * kHD;
        const __nv_bfloat16* vp = pl + ((((size_t)page * 2 + 1) * a.Hkv + h) * a.pt + off) * kHD;
        bulk_g2s_hint(S.Ks + (t - tok0) * kHD, kp, (uint32_t)seg * kHD * 2, attbar, kEvictNormal);
        bulk_g2s_hint(S.Vs + (t - tok0) * kHD, vp, (uint32_t)seg * kHD * 2, attbar, kEvictNormal);
        t += seg;
      }
    }
  }
  wg_bar(wg);  // q of this head is visible to the whole WG
  float* qs = S.qs + wwarp * REP * kHD;
  if (prefix) {
    const int ntok = min(kMkPC, a.pcap - c * kMkPC);
    // q of this warp's first row is loaded before the K/V wait, the next row's during the math
    uint2 qb[REP];
    int rr = wwarp;
    while (rr < a.rc && !S.ract[rr]) rr += 4;
    if (rr < a.rc) mk_fetch_q<REP>(a, rr, h, qb, lane);
    mk_wait(attbar, attph, 10);
    while (rr < a.rc) {
      mk_put_q<REP>(qb, qs, lane);
      int nx = rr + 4;
      while (nx < a.rc && !S.ract[nx]) nx += 4;
      if (nx < a.rc) mk_fetch_q<REP>(a, nx, h, qb, lane);
      __syncwarp();
      WarpPartial<REP, 1> wp;
      wp.run(qs, S.Ks, S.Vs, ntok, a.scale, lane);
      mk_store_partial<REP>(a, rr, h, c, wp.m, wp.l, wp.o, lane);
      __syncwarp();
      rr = nx;
    }
  } else {
    const int len = S.rlen[r];
    const int ntok = min(kMkSC, len - c * kMkSC);
    mk_load_q<REP>(a, r, h, qs, lane);
    __syncwarp();
    mk_wait(attbar, attph, 11);
    const int wt0 = wwarp * 8, wn = max(0, min(8, ntok - wt0));
    WarpPartial<REP, 4> wp;
    if (wn > 0) wp.run(qs, S.Ks + wt0 * kHD, S.Vs + wt0 * kHD, wn, a.scale, lane);
    float* cw = S.comb + wwarp * REP * (kHD + 2);
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
    wg_bar(wg);
    if (wwarp == 0) {
      float M[REP], L[REP], O[REP][4];
#pragma unroll
      for (int e = 0; e < REP; ++e) {
        M[e] = -INFINITY;
        for (int w = 0; w < 4; ++w) M[e] = fmaxf(M[e], S.comb[(w * REP + e) * (kHD + 2)]);
        L[e] = 0.f;
        O[e][0] = O[e][1] = O[e][2] = O[e][3] = 0.f;
        for (int w = 0; w < 4; ++w) {
          const float* src = S.comb + (w * REP + e) * (kHD + 2);
          if (src[0] == -INFINITY) continue;
          const float f = expf(src[0] - M[e]);
          L[e] += f * src[1];
#pragma unroll
          for (int k = 0; k < 4; ++k) O[e][k] += f * src[2 + 4 * lane + k];
        }
      }
      mk_store_partial<REP>(a, r, h, a.nc_pre + c, M, L, O, lane);
    }
  }
  attph ^= 1;
  __threadfence();
  wg_bar(wg);
  // count this unit's contribution per (kv head, row), one thread per row; the
  // unit that completes a (row, kv head) merges it
  bool fin = false;
  if (wt < a.rc && (prefix ? S.ract[wt] != 0 : wt == r)) {
    const int expect = a.nc_pre + (S.rlen[wt] + kMkSC - 1) / kMkSC;
    fin = atom_acqrel_add(sl + a.so.att_row + h * a.rc + wt, 1) + 1 == expect;
  }
  const unsigned bal = __ballot_sync(0xffffffffu, fin);
  if (lane == 0 && wwarp < 2) S.ctl[4 + wwarp] = (int)bal;
  wg_bar(wg);
  const unsigned long long mask = (unsigned long long)(unsigned)S.ctl[4] | ((unsigned long long)(unsigned)S.ctl[5] << 32);
  const int nm = __popcll(mask);
  if (nm > 0) {
    for (int p = wwarp; p < nm * REP; p += 4) {
      unsigned long long mm = mask;
      for (int j = 0; j < p / REP; ++j) mm &= mm - 1;
      const int row = __ffsll((long long)mm) - 1;
      mk_merge<BN>(a, row, h * REP + p % REP, S.rlen[row], lane);
    }
    fence_proxy_async_global();
    __threadfence();
    wg_bar(wg);
    if (wt == 0) red_release_add(sl + a.so.att_done + h, nm);
  }
}

// ---------------------------------------------------------------- the kernel
constexpr int kCS = 4;  // thread-block cluster size == K split of every GEMM unit

IS_DEVICE void st_async_v4(uint32_t remote_addr, float4 v, uint32_t remote_bar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.f32 [%0], {%1, %2, %3, %4}, [%5];" ::"r"(
                   remote_addr),
               "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w), "r"(remote_bar)
               : "memory");
}
IS_DEVICE void mbar_arrive_remote(uint32_t remote_bar) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(remote_bar) : "memory");
}

template <int BN, int REP>
__global__ void __launch_bounds__(kMkThreads, 1) mk_decode_kernel(const __grid_constant__ MkArgs a) {
  extern __shared__ uint8_t mk_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(mk_raw) + 1023) & ~uintptr_t(1023));
  constexpr int kBStage = BN * 128;
  constexpr int kSlice = BN / kCS;                 // decode rows owned by each CTA of the cluster
  constexpr int kRecv = kCS * 128 * kSlice * 4;    // per WG: [src][128 m][kSlice] fp32
  uint8_t* ringA = sm;
  uint8_t* ringB = ringA + (size_t)a.na * kMkStage;
  float* recv = reinterpret_cast<float*>(ringB + (size_t)2 * a.nb * kBStage);
  uint8_t* scratch = reinterpret_cast<uint8_t*>(recv) + 2 * kRecv;
  uint64_t* bars = reinterpret_cast<uint64_t*>(scratch + 2 * a.scratch);
  uint64_t* afull = bars;
  uint64_t* aempty = afull + a.na;
  uint64_t* bfull = aempty + a.na;   // [2][nb]
  uint64_t* bempty = bfull + 2 * a.nb;
  uint64_t* tfull = bempty + 2 * a.nb;  // [2]
  uint64_t* tempty = tfull + 2;
  uint64_t* attbar = tempty + 2;        // [2]
  uint64_t* rfull = attbar + 2;         // [2] partial slices received (tx bytes)
  uint64_t* rfree = rfull + 2;          // [2] every receiver has consumed our previous slices
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(rfree + 2);
  constexpr uint32_t kTmemCols = (2 * BN) <= 32 ? 32 : ((2 * BN) <= 64 ? 64 : 128);
  constexpr uint32_t kRecvTx = kCS * 128 * kSlice * 4;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int rank = (int)cluster_ctarank();
  unsigned long long t_start = 0;
  if (threadIdx.x == 0) {
    t_start = gtimer();
    for (int i = 0; i < a.na; ++i) {
      mbar_init(&afull[i], 1);
      mbar_init(&aempty[i], 1);
    }
    for (int i = 0; i < 2 * a.nb; ++i) {
      mbar_init(&bfull[i], 1);
      mbar_init(&bempty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], 4);
      mbar_init(&attbar[i], 1);
      mbar_init(&rfull[i], 1);
      mbar_init(&rfree[i], kCS);
    }
    fence_barrier_init();
    // arm the first exchange of each WG (the peers' bytes may land right after the cluster barrier)
    mbar_arrive_expect_tx(&rfull[0], kRecvTx);
    mbar_arrive_expect_tx(&rfull[1], kRecvTx);
  }
  if (warp == 1) tmem_alloc<kTmemCols>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  cluster_sync();  // peers' barriers are initialised before any DSMEM traffic
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  pdl_launch_dependents();
  const int4* T = a.tasks + a.task_off[blockIdx.x];
  const int nt = a.task_off[blockIdx.x + 1] - a.task_off[blockIdx.x];

  if (warp == 0) {
    // ---------------------------------------------------------- weight producer
    // Streams this CTA's weight tiles into the smem ring and, ahead of it, issues
    // L2 prefetches of the next units' weight ranges (a.pf_units units ahead), so
    // HBM keeps streaming while the ring waits on a dependency.
    if (lane == 0) {
      int s = 0, nrec = 0, pf_next = 0, pf_done = 0;
      uint32_t ph = 0;
      auto unit_range = [&](int i, const __nv_bfloat16*& base, uint32_t& bytes) -> bool {
        const int4 tk = T[i];
        const int kind = tk.x & 0xFF;
        if (kind == MK_EMBED || kind == MK_ATT || kind == MK_FINAL) return false;
        const int gi = kind == MK_QKV ? 0 : kind - 2;  // O 1, GU 2, DN 3
        const MkGemm& g = a.g[gi];
        const int l = (tk.x >> 8) & 0xFF;
        base = a.wpk + (size_t)l * a.layer_stride + g.w_off + ((size_t)tk.y * g.KB + tk.z) * (kMkStage / 2);
        bytes = (uint32_t)(tk.w - tk.z) * kMkStage;
        return true;
      };
      for (int i = 0; i < nt; ++i) {
        const __nv_bfloat16* base;
        uint32_t bytes;
        if (!unit_range(i, base, bytes)) continue;
        // keep pf_units GEMM units prefetched beyond this one
        if (pf_next <= i) pf_next = i + 1;
        while (pf_next < nt && pf_done < a.pf_units) {
          const __nv_bfloat16* pb;
          uint32_t pbytes;
          if (unit_range(pf_next, pb, pbytes) && pbytes > 0) {
            prefetch_l2(pb, pbytes);
            ++pf_done;
          }
          ++pf_next;
        }
        if (pf_done > 0) --pf_done;  // unit i leaves the prefetch window
        mk_rec(a, 2, nrec, 7, i);
        for (uint32_t off = 0; off < bytes; off += kMkStage) {
          mk_wait(&aempty[s], ph ^ 1, 1);
          mbar_arrive_expect_tx(&afull[s], kMkStage);
          bulk_g2s_hint(ringA + (size_t)s * kMkStage, base + off / 2, kMkStage, &afull[s], kEvictFirst);
          if (++s == a.na) {
            s = 0;
            ph ^= 1;
          }
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    // ---------------------------------------------------------- MMA issuer
    constexpr uint32_t idesc = idesc_bf16_f32(128, BN);
    int s = 0, bs0 = 0, bs1 = 0, jg = 0, use0 = 0, use1 = 0, nrec = 0;
    uint32_t ph = 0, bph0 = 0, bph1 = 0;
    for (int i = 0; i < nt; ++i) {
      const int4 tk = T[i];
      const int kind = tk.x & 0xFF;
      if (kind == MK_EMBED || kind == MK_ATT || kind == MK_FINAL) continue;
      const int w = (jg++) & 1;
      int& bs = w ? bs1 : bs0;
      uint32_t& bph = w ? bph1 : bph0;
      int& use = w ? use1 : use0;
      mk_wait(&tempty[w], (use & 1) ^ 1, 2);
      tc_fence_after();
      if (lane == 0) mk_rec(a, 3, nrec, 8, i);
      const uint32_t d_tmem = tmem_base + w * BN;
      for (int kb = tk.z; kb < tk.w; ++kb) {
        mk_wait(&afull[s], ph, 3);
        if (lane == 0 && kb == tk.z) mk_rec(a, 3, nrec, 18, i);
        mk_wait(&bfull[w * a.nb + bs], bph, 4);
        if (lane == 0 && kb == tk.z) mk_rec(a, 3, nrec, 19, i);
        if (lane == 0 && kb == tk.w - 1) mk_rec(a, 3, nrec, 20, i);
        tc_fence_after();
        if (lane == 0) {
          const uint64_t da = smem_desc_k_sw128(ringA + (size_t)s * kMkStage);
          const uint64_t db = smem_desc_k_sw128(ringB + (size_t)(w * a.nb + bs) * kBStage);
#pragma unroll
          for (int k = 0; k < 4; ++k) tc_mma_f16(d_tmem, da + 2 * k, db + 2 * k, idesc, (kb > tk.z || k > 0) ? 1u : 0u);
          tc_commit(&aempty[s]);
          tc_commit(&bempty[w * a.nb + bs]);
        }
        __syncwarp();
        if (++s == a.na) {
          s = 0;
          ph ^= 1;
        }
        if (++bs == a.nb) {
          bs = 0;
          bph ^= 1;
        }
      }
      if (lane == 0) {
        tc_commit(&tfull[w]);  // (an empty K range commits immediately; the WG then uses zeros)
        mk_rec(a, 3, nrec, 9, i);
      }
      __syncwarp();
      ++use;
    }
  } else {
    // ---------------------------------------------------------- compute warp groups
    const int wg = (warp - 2) >> 2;
    const int wt = threadIdx.x - 64 - wg * 128;
    const int wwarp = wt >> 5;
    const int q = warp & 3;  // TMEM lane quadrant of this warp
    const int m = q * 32 + lane;
    MkWG<BN, REP> S;
    S.init(scratch + (size_t)wg * a.scratch);
    uint8_t* myB = ringB + (size_t)wg * a.nb * kBStage;
    uint64_t* myBfull = bfull + wg * a.nb;
    uint64_t* myBempty = bempty + wg * a.nb;
    float* myRecv = recv + (size_t)wg * (kRecv / 4);
    const uint32_t recv_local = smem_u32(myRecv);
    const uint32_t rfull_local = smem_u32(&rfull[wg]);
    const uint32_t rfree_local = smem_u32(&rfree[wg]);
    int bs = 0, use = 0, jg = 0, nrec = 0, xuse = 0;
    uint32_t bph = 0, attph = 0;
    pdl_wait();  // rows, tokens and page tables come from the scheduler kernel
    if (wt < a.rc) {
      S.ract[wt] = a.row_active[wt];
      S.rpos[wt] = a.row_pos[wt];
      S.rkv[wt] = a.row_kvloc[wt];
      S.rlen[wt] = a.row_len[wt];
      S.rlid[wt] = a.row_lid[wt];
    }
    wg_bar(wg);
    int n_active = 0;
    for (int r = 0; r < a.rc; ++r) n_active += S.ract[r] != 0;

    for (int i = 0; i < nt; ++i) {
      const int4 tk = T[i];
      const int kind = tk.x & 0xFF;
      const int l = (tk.x >> 8) & 0xFF;
      int* sl = a.sync + (size_t)l * a.so.stride;
      if (kind == MK_EMBED) {
        if (wg != 0) continue;
        // resid0[r] = E[tok] (fp32) and per-128-column sums of squares ssq[0][t][r]
        const int r = tk.y;
        const bool act = S.ract[r] != 0;
        const int tok = act ? __ldg(a.row_tok + r) : 0;
#pragma unroll 1
        for (int t0 = 0; t0 < a.Th; t0 += 8) {
          float xe[8];
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const int k = (t0 + j) * 128 + wt;
            xe[j] = (t0 + j < a.Th && k < a.H && act) ? __bfloat162float(a.embed[(size_t)tok * a.H + k]) : 0.f;
          }
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const int k = (t0 + j) * 128 + wt;
            if (t0 + j < a.Th && k < a.H) __stcg(a.resid0 + (size_t)r * a.H + k, xe[j]);
            const float ss = warp_sum(xe[j] * xe[j]);
            if (lane == 0 && t0 + j < a.Th) S.sred[wwarp * 64 + t0 + j] = ss;
          }
        }
        wg_bar(wg);
        if (wt < a.Th) __stcg(a.ssq + (size_t)wt * a.rc + r, S.sred[wt] + S.sred[64 + wt] + S.sred[128 + wt] + S.sred[192 + wt]);
        __threadfence();
        wg_bar(wg);
        if (wt == 0) red_release_add(a.sync + a.so.emb_done, 1);
        continue;
      }
      if (kind == MK_FINAL) {
        if (wg != 0) continue;
        const int r = tk.y;
        if (wt == 0) mk_spin(a, a.sync + (size_t)(a.L - 1) * a.so.stride + a.so.dn_done, a.g[3].T * kCS, 900);
        wg_bar(wg);
        if (wt == 0) {
          const float* s = a.ssq + (size_t)(2 * a.L) * a.Th * a.rc + r;
          float ss = 0.f;
          for (int t = 0; t < a.Th; ++t) ss += __ldcg(s + (size_t)t * a.rc);
          S.rs[0] = 1.0f / sqrtf(ss / (float)a.H + a.eps);
        }
        wg_bar(wg);
        const float rsv = S.rs[0];
#pragma unroll 4
        for (int k = wt; k < a.H; k += 128)
          a.xn_final[(size_t)r * a.H + k] =
              __float2bfloat16_rn(__ldcg(a.resid0 + (size_t)r * a.H + k) * rsv * __ldg(a.final_norm + k));
        wg_bar(wg);
        continue;
      }
      if (kind == MK_ATT) {
        // attention of layer l: units grabbed dynamically by every WG of every CTA
        if (wt == 0) {
          int cnt = 0;
          S.cum[0] = 0;
          for (int r = 0; r < a.rc; ++r) {
            const int ns = S.ract[r] ? (S.rlen[r] + kMkSC - 1) / kMkSC : 0;
            cnt += ns;
            S.cum[r + 1] = cnt;
          }
          S.ctl[1] = cnt;
        }
        wg_bar(wg);
        const int n_pre_units = n_active > 0 ? a.Hkv * a.nc_pre : 0;
        const int n_units = n_pre_units + a.Hkv * S.ctl[1];
        for (;;) {
          fence_proxy_async_smem();  // our generic writes to the scratch precede the next unit's bulk copies
          if (wt == 0) S.ctl[2] = atomicAdd(sl + a.so.att_next, 1);
          wg_bar(wg);
          const int u = S.ctl[2];
          wg_bar(wg);
          if (u >= n_units) break;
          if (wt == 0) mk_rec(a, wg, nrec, 5, u);
          mk_att_unit<BN, REP>(a, S, l, u, n_pre_units, wg, wt, &attbar[wg], attph);
          if (wt == 0) mk_rec(a, wg, nrec, 6, u);
        }
        continue;
      }
      // ---------------------------------------------------------- GEMM unit (part `rank` of a cluster tile)
      if (((jg++) & 1) != wg) continue;
      const int gi = kind == MK_QKV ? 0 : kind - 2;
      const int tile = tk.y, kb0 = tk.z, kb1 = tk.w;
      const int n_lo = rank * kSlice;
      const int gm = tile * 128 + m;
      if (wt == 0) mk_rec(a, wg, nrec, 1, i);
      // 0. static epilogue operands, loaded before anything waits
      float gq = 0.f, cs[kSlice], sn[kSlice];
      if (kind == MK_QKV) {
        const bool is_q = tile < a.Hq, is_v = tile >= a.Hq + a.Hkv;
        gq = is_v ? 1.f : (is_q ? __ldg(a.q_norm + l * 128 + m) : __ldg(a.k_norm + l * 128 + m));
#pragma unroll
        for (int j = 0; j < kSlice; ++j) {
          const int n = n_lo + j;
          const bool need = !is_v && n < a.rc && S.ract[n];
          const int pos = need ? S.rpos[n] : 0;
          cs[j] = need ? __ldg(a.rope_cos + (size_t)pos * 64 + (m & 63)) : 1.f;
          sn[j] = need ? __ldg(a.rope_sin + (size_t)pos * 64 + (m & 63)) : 0.f;
        }
      }
      // gains of this unit's K range -> smem (static data: issued before any wait)
      const bool norm_fill = (kind == MK_QKV || kind == MK_GU) && kb1 > kb0;
      if (norm_fill && wt == 0) {
        const __nv_bfloat16* gain = (kind == MK_QKV ? a.in_norm_bf : a.post_norm_bf) + (size_t)l * a.H;
        fence_proxy_async_smem();
        mbar_arrive_expect_tx(&attbar[wg], (uint32_t)(kb1 - kb0) * 128);
        bulk_g2s_hint(S.gsm, gain + kb0 * 64, (uint32_t)(kb1 - kb0) * 128, &attbar[wg], kEvictNormal);
      }
      // 1. inputs ready
      if (wt == 0) {
        if (kind == MK_QKV) {
          if (l == 0) mk_spin(a, a.sync + a.so.emb_done, a.rc, 400);
          else mk_spin(a, a.sync + (size_t)(l - 1) * a.so.stride + a.so.dn_done, a.g[3].T * kCS, 500 + l);
        } else if (kind == MK_O) {
          const int h0 = (kb0 * 64) / kHD / REP, h1 = (max(kb1, kb0 + 1) * 64 - 1) / kHD / REP;
          for (int h = h0; h <= h1; ++h) mk_spin(a, sl + a.so.att_done + h, n_active, 600 + l);
        } else if (kind == MK_GU) {
          mk_spin(a, sl + a.so.o_done, a.g[1].T * kCS, 700 + l);
        } else {
          for (int t = kb0; t < kb1; ++t) mk_spin(a, sl + a.so.gu_flag + t, kCS, 800 + l);
          // an empty K range still reads the post-attention residual in its epilogue
          if (kb1 == kb0) mk_spin(a, sl + a.so.o_done, a.g[1].T * kCS, 850 + l);
        }
        fence_proxy_async_global();
        mk_rec(a, wg, nrec, 2, i);
      }
      wg_bar(wg);
      // 2. activation operand -> this WG's B ring (128-byte-swizzled K-major rows)
      if (kind == MK_O || kind == MK_DN) {
        if (wt == 0) {
          const __nv_bfloat16* src = kind == MK_O ? a.attn_sw : a.act_sw;
          for (int kb = kb0; kb < kb1; ++kb) {
            mk_wait(&myBempty[bs], bph ^ 1, 5);
            mbar_arrive_expect_tx(&myBfull[bs], kBStage);
            bulk_g2s_hint(myB + (size_t)bs * kBStage, src + (size_t)kb * BN * 64, kBStage, &myBfull[bs], kEvictLast);
            if (++bs == a.nb) {
              bs = 0;
              bph ^= 1;
            }
          }
        }
      } else if (kb1 > kb0) {
        // RMSNorm at rounding point r1: bf16(x * rs[row] * gain), normalised in fp32 here.
        // One batch of loads (residual chunks, bf16 gains, the rows' sum-of-squares
        // partials) per up to 8 k-blocks, all in flight together.
        const float* rin = kind == MK_QKV ? a.resid0 : a.resid1;
        constexpr int kPer = BN / 16;   // 16-byte chunks per thread per k-block
        constexpr int kGrp = 8 / kPer;  // k-blocks per load batch
        const int ch = wt & 7;          // this thread's 8-column chunk (same for all its rows)
        bool rs_ready = false;
        for (int g0 = kb0; g0 < kb1; g0 += kGrp) {
          float4 xv[kGrp][kPer][2];
#pragma unroll
          for (int j = 0; j < kGrp; ++j) {
            const int kb = g0 + j;
#pragma unroll
            for (int c = 0; c < kPer; ++c) {
              const int row = (wt + 128 * c) >> 3;
              const bool ok = kb < kb1 && row < a.rc;
              const float4* src = reinterpret_cast<const float4*>(rin + (size_t)row * a.H + kb * 64 + ch * 8);
              xv[j][c][0] = ok ? __ldcg(src) : make_float4(0.f, 0.f, 0.f, 0.f);
              xv[j][c][1] = ok ? __ldcg(src + 1) : make_float4(0.f, 0.f, 0.f, 0.f);
            }
          }
          if (!rs_ready) {
            mk_row_scale(a, kind == MK_QKV ? 2 * l : 2 * l + 1, S.rs, wt);
            mk_wait(&attbar[wg], attph, 12);  // gains staged
            attph ^= 1;
            rs_ready = true;
          }
          if (wt == 0)
            for (int j = 0; j < kGrp && g0 + j < kb1; ++j) mk_wait(&myBempty[(bs + j) % a.nb], (bs + j >= a.nb ? bph ^ 1 : bph) ^ 1, 5);
          wg_bar(wg);  // rs[] ready, ring stages free
          if (wt == 0) mk_rec(a, wg, nrec, 16, i);
#pragma unroll
          for (int j = 0; j < kGrp; ++j) {
            const int kb = g0 + j;
            if (kb >= kb1) break;
            const int st = (bs + j) % a.nb;
            const uint4 gvj = *reinterpret_cast<const uint4*>(S.gsm + (kb - kb0) * 64 + ch * 8);
            const __nv_bfloat162* g2 = reinterpret_cast<const __nv_bfloat162*>(&gvj);
            const float2 ga = __bfloat1622float2(g2[0]), gb = __bfloat1622float2(g2[1]);
            const float2 gc = __bfloat1622float2(g2[2]), gd = __bfloat1622float2(g2[3]);
#pragma unroll
            for (int c = 0; c < kPer; ++c) {
              const int row = (wt + 128 * c) >> 3;
              const float r_ = row < a.rc ? S.rs[row] : 0.f;
              const float4 x0 = xv[j][c][0], x1 = xv[j][c][1];
              uint4 o;
              __nv_bfloat162 hh;
              hh = __floats2bfloat162_rn(x0.x * r_ * ga.x, x0.y * r_ * ga.y); o.x = *reinterpret_cast<uint32_t*>(&hh);
              hh = __floats2bfloat162_rn(x0.z * r_ * gb.x, x0.w * r_ * gb.y); o.y = *reinterpret_cast<uint32_t*>(&hh);
              hh = __floats2bfloat162_rn(x1.x * r_ * gc.x, x1.y * r_ * gc.y); o.z = *reinterpret_cast<uint32_t*>(&hh);
              hh = __floats2bfloat162_rn(x1.z * r_ * gd.x, x1.w * r_ * gd.y); o.w = *reinterpret_cast<uint32_t*>(&hh);
              *reinterpret_cast<uint4*>(myB + (size_t)st * kBStage + row * 128 + ((ch ^ (row & 7)) << 4)) = o;
            }
          }
          fence_proxy_async_smem();
          wg_bar(wg);
          const int nk = min(kGrp, kb1 - g0);
          if (wt == 0)
            for (int j = 0; j < nk; ++j) mbar_arrive(&myBfull[(bs + j) % a.nb]);
          if (wt == 0) mk_rec(a, wg, nrec, 17, i);
          for (int j = 0; j < nk; ++j)
            if (++bs == a.nb) {
              bs = 0;
              bph ^= 1;
            }
        }
      }
      // 3. epilogue operands that depend on earlier phases (loaded while the MMA runs)
      float rin_v[kSlice];
      if (kind == MK_O || kind == MK_DN) {
        const float* rin = kind == MK_O ? a.resid0 : a.resid1;
#pragma unroll
        for (int j = 0; j < kSlice; ++j) {
          const int n = n_lo + j;
          rin_v[j] = (n < a.rc && gm < a.H) ? __ldcg(rin + (size_t)n * a.H + gm) : 0.f;
        }
      }
      // 4. accumulator
      mk_wait(&tfull[wg], use & 1, 6);
      ++use;
      tc_fence_after();
      if (wt == 0) mk_rec(a, wg, nrec, 3, i);
      float v[BN];
      if (kb1 > kb0) {
#pragma unroll
        for (int c = 0; c < BN / 16; ++c)
          tmem_ld16(tmem_base + ((uint32_t)(q * 32) << 16) + wg * BN + c * 16, v + c * 16);
      } else {
#pragma unroll
        for (int n = 0; n < BN; ++n) v[n] = 0.f;
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[wg]);
      // 5. split-K exchange inside the cluster: rank j receives column slice j of every
      //    peer's partial over DSMEM (st.async, completion counted in bytes on its rfull)
      if (xuse > 0) mk_wait(&rfree[wg], (xuse - 1) & 1, 7);
#pragma unroll
      for (int j = 0; j < kCS; ++j) {
        const uint32_t dst = mapa_shared(recv_local, j) + (uint32_t)(((rank * 128) + m) * kSlice * 4);
        const uint32_t bar = mapa_shared(rfull_local, j);
#pragma unroll
        for (int c4 = 0; c4 < kSlice / 4; ++c4)
          st_async_v4(dst + c4 * 16, make_float4(v[j * kSlice + 4 * c4], v[j * kSlice + 4 * c4 + 1],
                                                 v[j * kSlice + 4 * c4 + 2], v[j * kSlice + 4 * c4 + 3]), bar);
      }
      mk_wait(&rfull[wg], xuse & 1, 8);
      if (wt == 0) mk_rec(a, wg, nrec, 11, i);
#pragma unroll
      for (int jn = 0; jn < kSlice; ++jn) {
        float acc = myRecv[(0 * 128 + m) * kSlice + jn];
#pragma unroll
        for (int src = 1; src < kCS; ++src) acc += myRecv[(src * 128 + m) * kSlice + jn];
        S.stg[jn * 128 + m] = acc;
      }
      wg_bar(wg);
      if (wt == 0) mbar_arrive_expect_tx(&rfull[wg], kRecvTx);  // arm our next exchange ...
      __syncwarp();
      if (wt < kCS) mbar_arrive_remote(mapa_shared(rfree_local, wt));  // ... then let the peers overwrite our slot
      ++xuse;
      if (wt == 0) mk_rec(a, wg, nrec, 13, i);
      // 6. fused epilogue over this CTA's rows n_lo .. n_lo + kSlice - 1
      if (kind == MK_QKV) {
        // per-head RMSNorm of q / k (128 lanes of a column), rotate-half RoPE, bf16 q / KV append
        const bool is_v = tile >= a.Hq + a.Hkv, is_q = tile < a.Hq;
        if (!is_v) {
#pragma unroll
          for (int jn = 0; jn < kSlice; ++jn) {
            const float x = S.stg[jn * 128 + m];
            const float ss = warp_sum(x * x);
            if (lane == 0) S.sred[q * 64 + jn] = ss;
          }
          wg_bar(wg);
#pragma unroll
          for (int jn = 0; jn < kSlice; ++jn) {
            const float ss = S.sred[jn] + S.sred[64 + jn] + S.sred[128 + jn] + S.sred[192 + jn];
            S.stg[jn * 128 + m] *= (1.0f / sqrtf(ss / 128.0f + a.eps)) * gq;
          }
          wg_bar(wg);
        }
        const int hk = tile - a.Hq - (is_v ? a.Hkv : 0);
        __nv_bfloat16* pl = a.pool + (size_t)l * a.pool_layer;
#pragma unroll
        for (int jn = 0; jn < kSlice; ++jn) {
          const int n = n_lo + jn;
          if (n >= a.rc || !S.ract[n]) continue;
          float y = S.stg[jn * 128 + m];
          if (!is_v)
            y = m < 64 ? (y * cs[jn] - S.stg[jn * 128 + m + 64] * sn[jn]) : (y * cs[jn] + S.stg[jn * 128 + m - 64] * sn[jn]);
          const __nv_bfloat16 b = __float2bfloat16_rn(y);
          if (is_q) {
            a.q[((size_t)n * a.Hq + tile) * 128 + m] = b;
          } else {
            const int loc = S.rkv[n];
            const size_t off = ((((size_t)(loc / a.pt) * 2 + (is_v ? 1 : 0)) * a.Hkv + hk) * a.pt + loc % a.pt) * 128 + m;
            pl[off] = b;
          }
        }
        if (wt == 0) mk_rec(a, wg, nrec, 15, i);
        fence_proxy_async_global();
        __threadfence();
        wg_bar(wg);
        if (wt == 0) { red_release_add(sl + a.so.qkv_flag + tile, 1); mk_rec(a, wg, nrec, 10, i); }
      } else if (kind == MK_GU) {
        // rows [0, 64) of the tile are gate features f, rows [64, 128) the matching up (R12 r5)
        if (m < 64 && tile * 64 + m < a.F)
#pragma unroll
          for (int jn = 0; jn < kSlice; ++jn) {
            const int n = n_lo + jn;
            if (n >= a.rc) continue;
            const float gt = S.stg[jn * 128 + m], up = S.stg[jn * 128 + m + 64];
            a.act_sw[sw_off(n, tile * 64 + m, BN)] = __float2bfloat16_rn(silu_f(gt) * up);
          }
        if (wt == 0) mk_rec(a, wg, nrec, 15, i);
        fence_proxy_async_global();
        __threadfence();
        wg_bar(wg);
        if (wt == 0) { red_release_add(sl + a.so.gu_flag + tile, 1); mk_rec(a, wg, nrec, 10, i); }
      } else {
        // o_proj / down: residual add (fp32 stream) and the next RMSNorm's sum-of-squares partial
        const bool is_o = kind == MK_O;
        float* rout = is_o ? a.resid1 : a.resid0;
        const int ver = is_o ? 2 * l + 1 : 2 * l + 2;
        const bool ok = gm < a.H;
#pragma unroll
        for (int jn = 0; jn < kSlice; ++jn) {
          const int n = n_lo + jn;
          float x = 0.f;
          if (n < a.rc && ok) {
            x = rin_v[jn] + S.stg[jn * 128 + m];
            __stcg(rout + (size_t)n * a.H + gm, x);
          }
          const float ss = warp_sum(x * x);
          if (lane == 0) S.sred[q * 64 + jn] = ss;
        }
        wg_bar(wg);
        if (wt < kSlice && n_lo + wt < a.rc)
          __stcg(a.ssq + ((size_t)ver * a.Th + tile) * a.rc + n_lo + wt,
                 S.sred[wt] + S.sred[64 + wt] + S.sred[128 + wt] + S.sred[192 + wt]);
        if (wt == 0) mk_rec(a, wg, nrec, 15, i);
        __threadfence();
        wg_bar(wg);
        if (wt == 0) { red_release_add(sl + (is_o ? a.so.o_done : a.so.dn_done), 1); mk_rec(a, wg, nrec, 10, i); }
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<kTmemCols>(tmem_base);
  }
  cluster_sync();  // no CTA leaves while a peer may still write into its shared memory
  if (threadIdx.x == 0 && blockIdx.x == 0 && a.clock) {
    // CTA 0's lifetime ~ the kernel's (it holds FINAL and EMBED work): live timing for bench.py
    atomicAdd(a.clock, gtimer() - t_start);
    atomicAdd(a.clock + 1, 1ull);
  }
}

// pack W [M][K] (row-major bf16) into [ceil(M/128)][K/64][128][64] tiles with the
// 128-byte swizzle the MMA descriptor expects (rows >= M are zero).
__global__ void pack_sw128_kernel(const __nv_bfloat16* __restrict__ W, int M, int K, __nv_bfloat16* __restrict__ out) {
  const int KB = K / 64;
  const long long T = (M + 127) / 128;
  const long long n = T * KB * 128 * 8;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const int c = (int)(i & 7);
    const int r = (int)((i >> 3) & 127);
    const long long tk = i >> 10;
    const int kb = (int)(tk % KB);
    const long long t = tk / KB;
    const long long row = t * 128 + r;
    uint4 v = make_uint4(0, 0, 0, 0);
    if (row < M) v = *reinterpret_cast<const uint4*>(W + row * K + kb * 64 + c * 8);
    *reinterpret_cast<uint4*>(out + (tk * 128 + r) * 64 + ((c ^ (r & 7)) << 3)) = v;
  }
}

}  // namespace isk
