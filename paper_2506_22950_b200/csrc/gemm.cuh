// Weight-streaming "swap-AB" GEMM on tcgen05 for the decode step.
//
//   Y[n][m] = sum_k X[n][k] * W[m][k]      (X: activation rows, W: [out, in] weights)
//
// computed as D = W_tile · X^T with the weight tile as the MMA A operand
// (M = 128 output features) and the R <= 64 activation rows as N, so the
// skinny decode GEMM keeps the 128-row tensor-core shape and its cost is the
// weight stream.  Both operands are TMA-loaded with 128-byte
// swizzle into a STAGES-deep mbarrier ring; one thread issues tcgen05.mma
// (kind::f16, bf16 in / fp32 accumulate in TMEM); four epilogue warps read
// TMEM with tcgen05.ld.
//
// Split-K: `split` CTAs of a thread-block cluster share one 128-row tile, each
// streaming a contiguous K range.  Column slice j of the tile belongs to rank
// j: every rank writes its fp32 partial tile to an L2-resident workspace
// (coalesced float4 stores), one cluster barrier (release / acquire) orders
// them, and each rank sums its column slice over ranks 0..split-1 in rank order
// (deterministic; no atomics).  With split == 1 the kernel is persistent over
// tiles and double-buffers the TMEM accumulator.  (Measured slower: the last
// rank to count in on a per-tile counter reducing and finishing the whole tile
// alone -- one CTA's L2 pull of all partials plus the whole tile's epilogue.)
//
// RMSNorm (R12b): a GEMM whose input is a normalised activation reads B =
// bf16(x * gain) (written by the producer's epilogue, or by embed_kernel for
// layer 0) and scales its fp32 accumulator by rs[row] = 1/sqrt(mean(x^2)+eps),
// from the producer's per-128-column sums of squares (rs_ssq): no RMSNorm
// kernel and no grid barrier between the residual update and its consumer.
//
// Epilogues (fused, no extra pass over HBM):
//   EPI_QKV        per-head RMSNorm of q/k + RoPE + bf16 q / KV-cache append (R12 r2)
//   EPI_RESID_ADD  out[row][m] += acc                    (o_proj, down: fp32 residual; optionally
//                  the next norm's operand bf16(x * gain) and per-(tile, row) sums of squares)
//   EPI_SWIGLU     act[row][f]  = bf16(silu(g) * u)      (gate|up interleaved per 64 rows; R12 r5)
//   EPI_SAMPLE     keys[row] = max(key(z*invT + Gumbel)) (lm_head + Philox Gumbel-max sampler)
//   EPI_STORE_F32  out[row][m]  = acc                    (test hook)
#pragma once
#include "common.cuh"
#include "sampler.cuh"

namespace isk {

enum EpiKind { EPI_STORE_F32 = 0, EPI_RESID_ADD = 1, EPI_SWIGLU = 2, EPI_SAMPLE = 3, EPI_QKV = 4 };

// QK-norm + RoPE + KV append (EPI_QKV).  One 128-row tile == one head of the
// concatenated [q heads | k heads | v heads] projection.
struct QkvEpiArgs {
  const float* q_gain;       // [128]
  const float* k_gain;       // [128]
  const float* rope_cos;     // [max_pos][64]
  const float* rope_sin;
  const int32_t* row_active;
  const int32_t* row_pos;
  const int32_t* row_kvloc;  // decode: page*pt + offset; prefill: prefix position
  __nv_bfloat16* q_out;      // [rows][Hq][128]
  __nv_bfloat16* kv;         // decode: layer page pool [pages][2][Hkv][pt][128]; prefill: prefix [2][Hkv][pcap][128]
  int Hq, Hkv, pt, pcap, prefill;
  float eps;
};

struct GemmArgs {
  int M;          // weight rows (output features, incl. interleaved gate|up)
  int K;          // reduction length
  int num_tiles;  // ceil(M / 128)
  int split;      // K split == cluster size (1 => persistent over tiles)
  int row0;       // first activation row of this launch
  int n_valid;    // rows [row0, row0 + n_valid) carry results
  float* out;     // STORE / RESID
  int ld_out;
  __nv_bfloat16* act;  // SWIGLU
  int ld_act;
  const int32_t* row_uid;     // SAMPLE: per row
  const int32_t* row_t;
  const int32_t* row_active;
  unsigned long long* keys;
  unsigned long long* lp_key;  // SAMPLE (NEXT-3): per (row, CTA) best key of the CTA's tiles  [rows][gridDim]
  float4* lp_mlz;              //   and its online (max z, sum exp(z - max), winner's z, -)   [rows][gridDim]
  float* logits_dump;  // optional [rows][M]
  float* score_dump;   // optional [rows][M] fl(fl(z * invT) + G_v) (top-p pass, R36)
  uint64_t seed;
  float inv_temp;
  QkvEpiArgs qkv;
  float* partials;             // split-K workspace [tiles][split][128][BN] fp32 (L2-resident)
  unsigned long long* dbg_ts;  // optional [gridDim][16] globaltimer stamps (probe)
  // RMSNorm consumer (R12b): acc[row] *= rs[row] = 1/sqrt(sum_t rs_ssq[t][row] / K + eps)
  const float* rs_ssq;         // [rs_nt][rs_ld] the producer's per-128-column sums of squares (null: no norm)
  int rs_nt, rs_ld;
  float rs_eps;
  // RMSNorm producer (EPI_RESID_ADD): the next norm's B operand and its sums of squares
  const float* xg_gain;        // [M] next norm's gain (null: no xg_out)
  __nv_bfloat16* xg_out;       // [rows][M] bf16(x * gain)
  float* ssq_out;              // [tiles][ssq_ld] per-(tile, row) sum of x^2 of the new residual
  int ssq_ld;
  int* pf_progress;            // optional: the L2 weight prefetcher's pacing word (l2_prefetch_kernel):
  int pf_seq;                  //   this GEMM's index in the step's weight order, written at launch
};

constexpr int kBM = 128;
constexpr int kBK = 64;
constexpr int kGemmThreads = 192;

template <int BN, int STAGES>
struct GemmCfg {
  static constexpr int kStageA = kBM * kBK * 2;  // 16 KB
  static constexpr int kStageB = BN * kBK * 2;
  static constexpr int kStage = kStageA + kStageB;
  static constexpr int kAux = 2 * BN * kBM * 4;  // epilogue: stg[BN][128] (accumulator tile) + pre[BN][128]
  static constexpr int kTmemCols = (2 * BN) <= 32 ? 32 : ((2 * BN) <= 64 ? 64 : 128);
  static constexpr int kSmem = STAGES * kStage + kAux + 1024 /*barriers*/ + 1024 /*align*/;
};

__device__ __forceinline__ void stamp(const GemmArgs& a, int i) {
  if (a.dbg_ts) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    a.dbg_ts[blockIdx.x * 16 + i] = t;
  }
}

__device__ __forceinline__ float silu_f(float x) { return x / (1.0f + expf(-x)); }

template <int BN, int EPI, int STAGES>
__global__ void __launch_bounds__(kGemmThreads, 1)
    gemm_swapab_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                       GemmArgs a) {
  using C = GemmCfg<BN, STAGES>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align1024_smem(smem_raw);
  uint8_t* stage_base = smem;
  float* aux = reinterpret_cast<float*>(smem + STAGES * C::kStage);  // epilogue staging
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + STAGES * C::kStage + C::kAux);
  uint64_t* full = bars;
  uint64_t* empty = bars + STAGES;
  uint64_t* tfull = bars + 2 * STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  __shared__ float sred[4][BN];  // QKV: per-row 1/rms of the head
  __shared__ float run_m[BN], run_l[BN], run_z[BN];  // the CTA's running log-sum-exp state per row
  __shared__ unsigned long long run_k[BN];
  __shared__ int srow_act[BN], srow_kv[BN];
  __shared__ float srs[BN];  // RMSNorm consumer: 1/rms per row (1 without a norm)

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int S = a.split;
  const int rank = S > 1 ? (int)cluster_ctarank() : 0;
  const int cl = S > 1 ? (int)cluster_id_x() : (int)blockIdx.x;
  const int ncl = S > 1 ? (int)nclusters_x() : (int)gridDim.x;
  const int kb_total = a.K / kBK;
  const int kb0 = rank * kb_total / S;
  const int kb1 = (rank + 1) * kb_total / S;
  // column slice owned by this rank (split-K); whole tile otherwise
  const int n_lo = rank * BN / S, n_hi = (rank + 1) * BN / S;

  if (threadIdx.x == 0) stamp(a, 0);
  if (a.pf_progress && blockIdx.x == 0 && threadIdx.x == 0)
    asm volatile("st.relaxed.gpu.global.s32 [%0], %1;" ::"l"(a.pf_progress), "r"(a.pf_seq) : "memory");
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    for (int i = 0; i < STAGES; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], 4);
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<C::kTmemCols>(tmem_slot);
  if (EPI == EPI_SAMPLE && threadIdx.x < BN) {
    run_m[threadIdx.x] = -INFINITY;
    run_l[threadIdx.x] = 0.f;
    run_z[threadIdx.x] = 0.f;
    run_k[threadIdx.x] = 0ull;
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  // start-up phase of the cluster barrier (every rank resident before the exchange)
  if (S > 1) asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
  const uint32_t tmem_base = *tmem_slot;
  if (threadIdx.x == 0) stamp(a, 1);
  pdl_launch_dependents();

  if (warp == 0) {
    // ------------------------------------------------ TMA producer
    if (lane == 0) {
      // Weights never depend on the previous kernel: fill every ring stage with
      // its weight tile BEFORE griddepcontrol.wait (PDL), so a GEMM launched
      // early streams its first STAGES x 16 KB while its predecessor drains.
      // Activation (B) tiles are issued after the wait.
      const int n_pre = (cl < a.num_tiles) ? min(STAGES, kb1 - kb0) : 0;
      for (int i = 0; i < n_pre; ++i) {
        uint8_t* sa = stage_base + i * C::kStage;
        mbar_arrive_expect_tx(&full[i], C::kStage);
        tma_load_2d(sa, &tmA, &full[i], (kb0 + i) * kBK, cl * kBM, kEvictFirst);
      }
      stamp(a, 2);
      pdl_wait();
      for (int i = 0; i < n_pre; ++i)
        tma_load_2d(stage_base + i * C::kStage + C::kStageA, &tmB, &full[i], (kb0 + i) * kBK, a.row0, kEvictLast);
      int stage = 0;
      uint32_t phase = 0;
      int done = n_pre;  // k-blocks of the first tile already issued
      for (int tile = cl; tile < a.num_tiles; tile += ncl) {
        for (int kb = kb0; kb < kb1; ++kb) {
          if (done > 0) {  // issued in the prologue
            --done;
          } else {
            mbar_wait(&empty[stage], phase ^ 1);
            uint8_t* sa = stage_base + stage * C::kStage;
            mbar_arrive_expect_tx(&full[stage], C::kStage);
            tma_load_2d(sa, &tmA, &full[stage], kb * kBK, tile * kBM, kEvictFirst);
            tma_load_2d(sa + C::kStageA, &tmB, &full[stage], kb * kBK, a.row0, kEvictLast);
          }
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    // ------------------------------------------------ MMA issuer (lane 0)
    constexpr uint32_t idesc = idesc_bf16_f32(kBM, BN);
    int stage = 0;
    uint32_t phase = 0;
    int it = 0;
    for (int tile = cl; tile < a.num_tiles; tile += ncl, ++it) {
      const int acc = it & 1;
      const uint32_t acc_phase = (it >> 1) & 1;
      mbar_wait(&tempty[acc], acc_phase ^ 1);
      tc_fence_after();
      const uint32_t d_tmem = tmem_base + acc * BN;
      for (int kb = kb0; kb < kb1; ++kb) {
        mbar_wait(&full[stage], phase);
        tc_fence_after();
        if (lane == 0 && kb == kb0) stamp(a, 3);
        if (lane == 0 && kb == kb1 - 1) stamp(a, 4);
        if (lane == 0) {
          uint8_t* sa = stage_base + stage * C::kStage;
          const uint64_t da = smem_desc_k_sw128(sa);
          const uint64_t db = smem_desc_k_sw128(sa + C::kStageA);
#pragma unroll
          for (int k = 0; k < kBK / 16; ++k)
            tc_mma_f16(d_tmem, da + 2 * k, db + 2 * k, idesc, (kb > kb0 || k > 0) ? 1u : 0u);
          tc_commit(&empty[stage]);
        }
        __syncwarp();
        if (++stage == STAGES) {
          stage = 0;
          phase ^= 1;
        }
      }
      if (lane == 0) tc_commit(&tfull[acc]);
      __syncwarp();
    }
  } else {
    // ------------------------------------------------ epilogue warps 2..5
    // Written as short runtime loops over columns: this code runs cold out of
    // the instruction cache once per launch, so its length -- not its
    // arithmetic -- sets the latency.
    const int q = warp & 3;  // TMEM lane quadrant this warp may access
    const int m = q * 32 + lane;
    const int et = threadIdx.x - 64;  // 0..127
    float* stg = aux;             // [BN][128] accumulator tile (column n = activation row)
    float* pre = aux + BN * kBM;  // [BN][128] operands prefetched during the mainloop
    pdl_wait();
    if (et < BN) {
      // RMSNorm consumer (R12b): rs per row from the producer's per-128-column partials,
      // summed in column order (all loads in flight together)
      float rs = 1.f;
      if (a.rs_ssq) {
        float ss = 0.f;
        if (et < a.n_valid) {
          float t16[16];
#pragma unroll 1
          for (int t0 = 0; t0 < a.rs_nt; t0 += 16) {
#pragma unroll
            for (int t = 0; t < 16; ++t)
              t16[t] = t0 + t < a.rs_nt ? __ldcg(a.rs_ssq + (size_t)(t0 + t) * a.rs_ld + a.row0 + et) : 0.f;
#pragma unroll
            for (int t = 0; t < 16; ++t) ss += t16[t];
          }
        }
        rs = 1.0f / sqrtf(ss / (float)a.K + a.rs_eps);
      }
      srs[et] = rs;
    }
    int it = 0;
    for (int tile = cl; tile < a.num_tiles; tile += ncl, ++it) {
      const int acc = it & 1;
      const uint32_t acc_phase = (it >> 1) & 1;
      const int gm = tile * kBM + m;
      // operands that do not depend on this GEMM, loaded while weights stream in
      if constexpr (EPI == EPI_RESID_ADD) {
        for (int n = n_lo; n < n_hi; ++n)
          pre[n * kBM + m] = (n < a.n_valid && gm < a.M) ? a.out[(size_t)(a.row0 + n) * a.ld_out + gm] : 0.f;
      }
      if constexpr (EPI == EPI_QKV) {
        const QkvEpiArgs& e = a.qkv;
        if (et < BN) {
          srow_act[et] = et < a.n_valid ? e.row_active[a.row0 + et] : 0;
          srow_kv[et] = et < a.n_valid ? e.row_kvloc[a.row0 + et] : 0;
        }
        if (tile < e.Hq + e.Hkv) {
          // all rows' positions first, then the table rows: independent loads in flight together
          int pos[BN];
#pragma unroll
          for (int n = 0; n < BN; ++n) pos[n] = (n >= n_lo && n < n_hi && n < a.n_valid) ? e.row_pos[a.row0 + n] : 0;
#pragma unroll
          for (int n = 0; n < BN; ++n)
            if (n >= n_lo && n < n_hi && n < a.n_valid)
              pre[n * kBM + m] = m < 64 ? e.rope_cos[(size_t)pos[n] * 64 + m] : e.rope_sin[(size_t)pos[n] * 64 + m - 64];
        }
      }
      // per-feature gains of the epilogue, loaded before the accumulator is ready
      // RESID_ADD: the next norm's gains of this lane's 4 features (4 lane .. 4 lane + 3)
      float4 gg4 = make_float4(0.f, 0.f, 0.f, 0.f);
      if constexpr (EPI == EPI_RESID_ADD)
        if (a.xg_out && tile * kBM + 4 * lane < a.M) gg4 = *reinterpret_cast<const float4*>(a.xg_gain + tile * kBM + 4 * lane);
      // QKV: the QK-norm gains of this thread's feature pairs (2i, 2i + 1) and (64 + 2i, 65 + 2i)
      float2 gq0 = make_float2(0.f, 0.f), gq1 = make_float2(0.f, 0.f);
      if constexpr (EPI == EPI_QKV) {
        if (tile < a.qkv.Hq + a.qkv.Hkv) {
          const float* gsrc = tile < a.qkv.Hq ? a.qkv.q_gain : a.qkv.k_gain;
          gq0 = *reinterpret_cast<const float2*>(gsrc + (et & 31) * 2);
          gq1 = *reinterpret_cast<const float2*>(gsrc + 64 + (et & 31) * 2);
        }
      }
      mbar_wait(&tfull[acc], acc_phase);
      tc_fence_after();
      if (threadIdx.x == 64) stamp(a, 5);
      float v[BN];
#pragma unroll
      for (int c = 0; c < BN / 16; ++c)
        tmem_ld16(tmem_base + ((uint32_t)(q * 32) << 16) + acc * BN + c * 16, v + c * 16);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[acc]);

      if (S > 1) {
        // Partials -> L2 workspace part[cluster][rank][m][BN] (coalesced float4
        // stores); the cluster barrier (release / acquire) orders them; each rank
        // sums its column slice [n_lo, n_hi) over ranks 0..S-1 in order.
        float* part = a.partials + (size_t)cl * S * kBM * BN;
#pragma unroll
        for (int c4 = 0; c4 < BN / 4; ++c4)
          reinterpret_cast<float4*>(part + ((size_t)rank * kBM + m) * BN)[c4] =
              make_float4(v[4 * c4], v[4 * c4 + 1], v[4 * c4 + 2], v[4 * c4 + 3]);
        asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");  // start-up phase
        asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
        asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
        if (threadIdx.x == 64) stamp(a, 6);
        // aligned float4 groups covering the slice; per group all ranks' loads in flight
        for (int c0 = n_lo & ~3; c0 < n_hi; c0 += 4) {
          float4 t[8];
#pragma unroll
          for (int j = 0; j < 8; ++j)
            if (j < S) t[j] = __ldcg(reinterpret_cast<const float4*>(part + ((size_t)j * kBM + m) * BN + c0));
          float4 sum = t[0];
#pragma unroll
          for (int j = 1; j < 8; ++j)
            if (j < S) {
              sum.x += t[j].x;
              sum.y += t[j].y;
              sum.z += t[j].z;
              sum.w += t[j].w;
            }
          stg[(c0 + 0) * kBM + m] = sum.x * srs[c0 + 0];
          stg[(c0 + 1) * kBM + m] = sum.y * srs[c0 + 1];
          stg[(c0 + 2) * kBM + m] = sum.z * srs[c0 + 2];
          stg[(c0 + 3) * kBM + m] = sum.w * srs[c0 + 3];
        }
        if (threadIdx.x == 64) stamp(a, 7);
      } else {
        asm volatile("bar.sync 1, 128;" ::: "memory");  // srs (first tile)
#pragma unroll
        for (int n = 0; n < BN; ++n) stg[n * kBM + m] = v[n] * srs[n];
      }
      asm volatile("bar.sync 1, 128;" ::: "memory");
      if (threadIdx.x == 64) stamp(a, 8);

      if constexpr (EPI == EPI_STORE_F32 || EPI == EPI_RESID_ADD) {
        // one row per warp and pass (4 rows per pass): lane l owns features 4l .. 4l + 3 (float4
        // residual store, 8-byte bf16 store of the next norm's operand), the warp's butterfly sum
        // is the row's sum of squares over the tile (M % 4 == 0)
        const int n_end = min(n_hi, a.n_valid);
        const int g4 = tile * kBM + 4 * lane;
        for (int n = n_lo + (et >> 5); n < n_end; n += 4) {
          float4 x = make_float4(0.f, 0.f, 0.f, 0.f);
          if (g4 < a.M) {
            x = *reinterpret_cast<const float4*>(stg + n * kBM + 4 * lane);
            if (EPI == EPI_RESID_ADD) {
              const float4 p4 = *reinterpret_cast<const float4*>(pre + n * kBM + 4 * lane);
              x.x += p4.x;
              x.y += p4.y;
              x.z += p4.z;
              x.w += p4.w;
            }
            *reinterpret_cast<float4*>(a.out + (size_t)(a.row0 + n) * a.ld_out + g4) = x;
            if (EPI == EPI_RESID_ADD && a.xg_out) {
              const __nv_bfloat162 b0 = __floats2bfloat162_rn(x.x * gg4.x, x.y * gg4.y);
              const __nv_bfloat162 b1 = __floats2bfloat162_rn(x.z * gg4.z, x.w * gg4.w);
              uint2 u;
              u.x = *reinterpret_cast<const uint32_t*>(&b0);
              u.y = *reinterpret_cast<const uint32_t*>(&b1);
              *reinterpret_cast<uint2*>(a.xg_out + (size_t)(a.row0 + n) * a.M + g4) = u;
            }
          }
          if (EPI == EPI_RESID_ADD && a.ssq_out) {
            const float ss = warp_sum(x.x * x.x + x.y * x.y + x.z * x.z + x.w * x.w);
            if (lane == 0) a.ssq_out[(size_t)tile * a.ssq_ld + a.row0 + n] = ss;
          }
        }
      } else if constexpr (EPI == EPI_SWIGLU) {
        // rows [0, 64) of the tile are gate features f, rows [64, 128) the matching up.  Every
        // epilogue thread takes two adjacent features of one row (one bf16x2 store); the 128
        // threads cover 4 rows per pass
        const int fp = (et & 31) * 2, f = tile * 64 + fp;
        const int n_end = min(n_hi, a.n_valid);
        if (f * 2 < a.M)
          for (int n = n_lo + (et >> 5); n < n_end; n += 4) {
            const float2 g2 = *reinterpret_cast<const float2*>(stg + n * kBM + fp);
            const float2 u2 = *reinterpret_cast<const float2*>(stg + n * kBM + 64 + fp);
            *reinterpret_cast<__nv_bfloat162*>(a.act + (size_t)(a.row0 + n) * a.ld_act + f) =
                __floats2bfloat162_rn(silu_f(g2.x) * u2.x, silu_f(g2.y) * u2.y);
          }
      } else if constexpr (EPI == EPI_QKV) {
        // head = tile: q (tile < Hq), k (< Hq + Hkv) or v.  Per-head RMSNorm over the 128
        // features of a row (8 threads per row, 16 rows per pass), then rotate-half RoPE: every
        // thread takes the feature pairs (2i, 2i + 1) and their partners (64 + 2i, 65 + 2i) of one
        // row (two bf16x2 stores), 4 rows per pass.
        const QkvEpiArgs& e = a.qkv;
        const bool is_v = tile >= e.Hq + e.Hkv, is_q = tile < e.Hq;
        const int n_end = min(n_hi, a.n_valid);
        float* rsn = &sred[0][0];  // [BN] 1/rms of the head per row
        if (!is_v) {
          const int part = et & 7;
          for (int n0 = n_lo; n0 < n_end; n0 += 16) {
            const int n = n0 + (et >> 3);
            float ss = 0.f;
            if (n < n_end)
#pragma unroll
              for (int j = 0; j < 16; ++j) {
                const float x = stg[n * kBM + j * 8 + part];
                ss += x * x;
              }
            ss += __shfl_xor_sync(0xffffffffu, ss, 1);
            ss += __shfl_xor_sync(0xffffffffu, ss, 2);
            ss += __shfl_xor_sync(0xffffffffu, ss, 4);
            if (part == 0 && n < n_end) rsn[n] = 1.0f / sqrtf(ss / (float)kBM + e.eps);
          }
          asm volatile("bar.sync 1, 128;" ::: "memory");
        }
        const int hk = tile - e.Hq - (is_v ? e.Hkv : 0);
        const int i2 = (et & 31) * 2;
        for (int n = n_lo + (et >> 5); n < n_end; n += 4) {
          if (!srow_act[n]) continue;
          const int row = a.row0 + n;
          float2 lo = *reinterpret_cast<const float2*>(stg + n * kBM + i2);
          float2 hi = *reinterpret_cast<const float2*>(stg + n * kBM + 64 + i2);
          if (!is_v) {
            const float r = rsn[n];
            lo.x *= r * gq0.x;
            lo.y *= r * gq0.y;
            hi.x *= r * gq1.x;
            hi.y *= r * gq1.y;
            const float2 c = *reinterpret_cast<const float2*>(pre + n * kBM + i2);
            const float2 s = *reinterpret_cast<const float2*>(pre + n * kBM + 64 + i2);
            const float2 ylo = make_float2(lo.x * c.x - hi.x * s.x, lo.y * c.y - hi.y * s.y);
            const float2 yhi = make_float2(hi.x * c.x + lo.x * s.x, hi.y * c.y + lo.y * s.y);
            lo = ylo;
            hi = yhi;
          }
          const __nv_bfloat162 blo = __floats2bfloat162_rn(lo.x, lo.y), bhi = __floats2bfloat162_rn(hi.x, hi.y);
          __nv_bfloat16* dst;
          if (is_q) {
            dst = e.q_out + ((size_t)row * e.Hq + tile) * kBM;
          } else {
            const int kvsel = is_v ? 1 : 0;
            const int loc = srow_kv[n];
            size_t off;
            if (e.prefill) off = (((size_t)kvsel * e.Hkv + hk) * e.pcap + loc) * kBM;
            else off = ((((size_t)(loc / e.pt) * 2 + kvsel) * e.Hkv + hk) * e.pt + loc % e.pt) * kBM;
            dst = e.kv + off;
          }
          *reinterpret_cast<__nv_bfloat162*>(dst + i2) = blo;
          *reinterpret_cast<__nv_bfloat162*>(dst + 64 + i2) = bhi;
        }
      } else if constexpr (EPI == EPI_SAMPLE) {
        // one row per warp and pass (rows n = warp, warp + 4, ...; a row always meets the same
        // warp, which keeps its running log-sum-exp state): lane l owns the tile's vocabulary
        // entries v = 4l .. 4l + 3, whose Gumbel words are exactly the 4 words of the Philox4x32-10
        // call with counter v >> 2 (R10/R11); in-lane argmax of the keys, one warp butterfly per row,
        // one atomicMax per (row, tile)
        const bool lp = a.lp_key != nullptr;
        const int nv = min(BN, a.n_valid);
        const int g4 = tile * kBM + 4 * lane;
        for (int n = et >> 5; n < nv; n += 4) {
          const int row = a.row0 + n;
          if (!a.row_active[row]) continue;  // (warp-uniform)
          const float4 zs = *reinterpret_cast<const float4*>(stg + n * kBM + 4 * lane);
          const float zv[4] = {zs.x, zs.y, zs.z, zs.w};
          const Philox4 o = philox4x32_10((uint32_t)g4 >> 2, (uint32_t)a.row_t[row], (uint32_t)a.row_uid[row], 0u,
                                          (uint32_t)a.seed, (uint32_t)(a.seed >> 32));
          unsigned long long key = 0ull;
          float zk = -INFINITY, zmax = -INFINITY;
          float sc4[4];
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            sc4[j] = 0.f;
            if (g4 + j < a.M) {
              const float z = zv[j];
              const float g = -logf_is(-logf_is(uniform_from_bits(o.x[j])));  // = gumbel(seed, uid, t, v)
              const float sc = __fadd_rn(__fmul_rn(z, a.inv_temp), g);
              sc4[j] = sc;
              const unsigned long long k = order_key(sc, (uint32_t)(g4 + j));
              if (k > key) {
                key = k;
                zk = z;
              }
              zmax = fmaxf(zmax, z);
            }
          }
          if (g4 + 3 < a.M) {
            if (a.logits_dump) *reinterpret_cast<float4*>(a.logits_dump + (size_t)row * a.ld_out + g4) = zs;
            if (a.score_dump)
              *reinterpret_cast<float4*>(a.score_dump + (size_t)row * a.ld_out + g4) = make_float4(sc4[0], sc4[1], sc4[2], sc4[3]);
          } else {
            for (int j = 0; j < 4; ++j)
              if (g4 + j < a.M) {
                if (a.logits_dump) a.logits_dump[(size_t)row * a.ld_out + g4 + j] = zv[j];
                if (a.score_dump) a.score_dump[(size_t)row * a.ld_out + g4 + j] = sc4[j];
              }
          }
#pragma unroll
          for (int s = 16; s > 0; s >>= 1) {
            const unsigned long long other = __shfl_xor_sync(0xffffffffu, key, s);
            const float oz = __shfl_xor_sync(0xffffffffu, zk, s);
            if (other > key) {
              key = other;
              zk = oz;
            }
          }
          if (lane == 0 && key) atomicMax(a.keys + row, key);
          if (lp) {
            // the tile's (max, sum exp) of this row's logits, folded into the warp's running state
            const float wm = warp_max(zmax);
            float se = 0.f;
#pragma unroll
            for (int j = 0; j < 4; ++j)
              if (g4 + j < a.M && zv[j] != -INFINITY) se += expf(zv[j] - wm);
            const float ws = warp_sum(se);
            if (lane == 0) {
              float M = run_m[n], L = run_l[n];
              if (wm != -INFINITY) {
                const float Mn = fmaxf(M, wm);
                L = (M == -INFINITY ? 0.f : L * expf(M - Mn)) + ws * expf(wm - Mn);
                M = Mn;
                if (key > run_k[n]) {
                  run_k[n] = key;
                  run_z[n] = zk;
                }
              }
              run_m[n] = M;
              run_l[n] = L;
              const size_t idx = (size_t)row * gridDim.x + blockIdx.x;
              a.lp_key[idx] = run_k[n];
              a.lp_mlz[idx] = make_float4(M, L, run_z[n], 0.f);
            }
          }
        }
      }
      // stg / pre are rewritten by the next tile
      asm volatile("bar.sync 1, 128;" ::: "memory");
    }
  }

  if (threadIdx.x == 64) stamp(a, 10);
  if (S > 1 && warp < 2) {
    // producer / MMA warps: complete the start-up barrier phase and arrive on the
    // partials-written phase the epilogue waits for.
    asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
    asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<C::kTmemCols>(tmem_base);
  }
  if (threadIdx.x == 32) stamp(a, 11);
}

}  // namespace isk
