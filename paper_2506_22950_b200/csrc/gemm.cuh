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
// j: every rank stages its partials of slice j in its idle stage ring and DMAs
// them into rank j's shared memory (cp.async.bulk, completion counted on rank
// j's mbarrier), then each rank sums its
// slice in rank order 0..split-1 -- deterministic, one cluster barrier (at
// start-up, hidden under the first TMA), no pull round trips.  With split == 1
// the kernel is persistent over tiles and double-buffers the TMEM accumulator.
//
// Epilogues (fused, no extra pass over HBM):
//   EPI_QKV        per-head RMSNorm of q/k + RoPE + bf16 q / KV-cache append (R12 r2)
//   EPI_RESID_ADD  out[row][m] += acc                    (o_proj, down: fp32 residual)
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
  float* logits_dump;  // optional [rows][M]
  uint64_t seed;
  float inv_temp;
  QkvEpiArgs qkv;
  unsigned long long* dbg_ts;  // optional [gridDim][16] globaltimer stamps (probe)
};

constexpr int kBM = 128;
constexpr int kBK = 64;
constexpr int kGemmThreads = 192;

template <int BN, int STAGES>
struct GemmCfg {
  static constexpr int kStageA = kBM * kBK * 2;  // 16 KB
  static constexpr int kStageB = BN * kBK * 2;
  static constexpr int kStage = kStageA + kStageB;
  static constexpr int kRed = (BN + 8) * kBM * 4;                           // >= split * ceil(BN/split) * 128 floats
  static constexpr int kXbuf = BN * kBM * 4;                                 // epilogue exchange
  static constexpr int kAux = kRed > kXbuf ? kRed : kXbuf;                   // red, then xbuf (aliased)
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
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* stage_base = smem;
  float* aux = reinterpret_cast<float*>(smem + STAGES * C::kStage);  // split-K receive buffer, then exchange
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + STAGES * C::kStage + C::kAux);
  uint64_t* full = bars;
  uint64_t* empty = bars + STAGES;
  uint64_t* tfull = bars + 2 * STAGES;
  uint64_t* tempty = tfull + 2;
  uint64_t* redbar = tempty + 2;    // (unused by the pull reduction; kept for layout)
  uint64_t* consumed = redbar + 1;  // split-K: S-1 peers finished reading our partials
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(consumed + 1);
  __shared__ unsigned long long skey[BN];
  __shared__ float sred[4][BN];

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
    mbar_init(redbar, 1);
    mbar_init(consumed, S > 1 ? S - 1 : 1);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<C::kTmemCols>(tmem_slot);
  if (EPI == EPI_SAMPLE && threadIdx.x < BN) skey[threadIdx.x] = 0ull;
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  // every rank's receive barrier must be armed before any peer pushes into it
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
    const int q = warp & 3;  // TMEM lane quadrant this warp may access
    const int m = q * 32 + lane;
    pdl_wait();
    int it = 0;
    for (int tile = cl; tile < a.num_tiles; tile += ncl, ++it) {
      const int acc = it & 1;
      const uint32_t acc_phase = (it >> 1) & 1;
      // Epilogue operands that do not depend on this GEMM are loaded while the
      // mainloop streams weights (hides their global-memory latency).
      float rv[BN], sv[BN];
      float qk_gain = 1.f;
      if constexpr (EPI == EPI_RESID_ADD) {
        const int gm = tile * kBM + m;
#pragma unroll
        for (int n = 0; n < BN; ++n)
          rv[n] = (n >= n_lo && n < n_hi && n < a.n_valid && gm < a.M) ? a.out[(size_t)(a.row0 + n) * a.ld_out + gm]
                                                                      : 0.f;
      }
      if constexpr (EPI == EPI_QKV) {
        const QkvEpiArgs& e = a.qkv;
        qk_gain = tile < e.Hq ? e.q_gain[m] : (tile < e.Hq + e.Hkv ? e.k_gain[m] : 1.f);
#pragma unroll
        for (int n = 0; n < BN; ++n) {
          const int row = a.row0 + n;
          rv[n] = sv[n] = 0.f;
          if (n >= n_lo && n < n_hi && n < a.n_valid && tile < e.Hq + e.Hkv) {
            const int pos = e.row_pos[row];
            rv[n] = e.rope_cos[(size_t)pos * 64 + (m & 63)];
            sv[n] = e.rope_sin[(size_t)pos * 64 + (m & 63)];
          }
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
        // Partials -> own smem aux[n][m]; one cluster barrier; then every rank
        // pulls its column slice from all ranks (independent DSMEM loads, issued
        // together) and sums in rank order.  A second cluster barrier (end of
        // kernel) keeps each rank's smem alive until its peers have read it.
#pragma unroll
        for (int n = 0; n < BN; ++n) aux[n * kBM + m] = v[n];
        asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");  // start-up phase
        asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
        asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
        if (threadIdx.x == 64) stamp(a, 6);
        const uint32_t laux = smem_u32(aux);
#pragma unroll
        for (int n = 0; n < BN; ++n) {
          if (n >= n_lo && n < n_hi) {
            float t[8];
#pragma unroll
            for (int j = 0; j < 8; ++j)
              t[j] = (j < S && j != rank) ? ld_dsmem_f32_nv(mapa_shared(laux + (uint32_t)(n * kBM + m) * 4u, j)) : 0.f;
            float sum = 0.f;
#pragma unroll
            for (int j = 0; j < 8; ++j)
              if (j < S) sum += (j == rank) ? v[n] : t[j];
            v[n] = sum;
          }
        }
        // every thread's remote reads are done (values consumed above): release peers
        asm volatile("bar.sync 1, 128;" ::: "memory");
        if (threadIdx.x == 64) {
          const uint32_t lc = smem_u32(consumed);
          for (int j = 0; j < S; ++j)
            if (j != rank)
              asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(mapa_shared(lc, j))
                           : "memory");
          stamp(a, 7);
        }
      }

      const int gm = tile * kBM + m;
      if (threadIdx.x == 64) stamp(a, 8);
      if constexpr (EPI == EPI_STORE_F32 || EPI == EPI_RESID_ADD) {
#pragma unroll
        for (int n = 0; n < BN; ++n) {
          if (n >= n_lo && n < n_hi && n < a.n_valid && gm < a.M) {
            float* p = a.out + (size_t)(a.row0 + n) * a.ld_out + gm;
            if (EPI == EPI_RESID_ADD) *p = rv[n] + v[n];
            else *p = v[n];
          }
        }
      } else if constexpr (EPI == EPI_SWIGLU) {
        float* xbuf = aux;
        if (m >= 64) {
#pragma unroll
          for (int n = 0; n < BN; ++n) xbuf[n * 64 + (m - 64)] = v[n];
        }
        asm volatile("bar.sync 1, 128;" ::: "memory");
        if (m < 64) {
          const int f = tile * 64 + m;
#pragma unroll
          for (int n = 0; n < BN; ++n) {
            if (n >= n_lo && n < n_hi && n < a.n_valid && f * 2 < a.M) {
              const float u = xbuf[n * 64 + m];
              a.act[(size_t)(a.row0 + n) * a.ld_act + f] = __float2bfloat16_rn(silu_f(v[n]) * u);
            }
          }
        }
        asm volatile("bar.sync 1, 128;" ::: "memory");
      } else if constexpr (EPI == EPI_QKV) {
        // head = tile: q (tile < Hq), k (< Hq + Hkv) or v.  Per-head RMSNorm over the
        // 128 lanes of a column, rotate-half RoPE pairs (m, m +- 64) through smem.
        const QkvEpiArgs& e = a.qkv;
        const bool is_v = tile >= e.Hq + e.Hkv, is_q = tile < e.Hq;
        float* xbuf = aux;
        if (!is_v) {
#pragma unroll
          for (int n = 0; n < BN; ++n) {
            if (n >= n_lo && n < n_hi) {
              const float ss = warp_sum(v[n] * v[n]);
              if (lane == 0) sred[q][n] = ss;
            }
          }
          asm volatile("bar.sync 1, 128;" ::: "memory");
          const float gn = qk_gain;
#pragma unroll
          for (int n = 0; n < BN; ++n) {
            if (n >= n_lo && n < n_hi) {
              const float ss = sred[0][n] + sred[1][n] + sred[2][n] + sred[3][n];
              v[n] = v[n] * (1.0f / sqrtf(ss / (float)kBM + e.eps)) * gn;
              xbuf[n * kBM + m] = v[n];
            }
          }
          asm volatile("bar.sync 1, 128;" ::: "memory");
#pragma unroll
          for (int n = 0; n < BN; ++n) {
            const int row = a.row0 + n;
            if (n >= n_lo && n < n_hi && n < a.n_valid && e.row_active[row]) {
              const float c = rv[n], s = sv[n];
              const float y = v[n];
              v[n] = m < 64 ? (y * c - xbuf[n * kBM + m + 64] * s) : (y * c + xbuf[n * kBM + m - 64] * s);
            }
          }
          asm volatile("bar.sync 1, 128;" ::: "memory");
        }
#pragma unroll
        for (int n = 0; n < BN; ++n) {
          const int row = a.row0 + n;
          if (n >= n_lo && n < n_hi && n < a.n_valid && e.row_active[row]) {
            const __nv_bfloat16 b = __float2bfloat16_rn(v[n]);
            if (is_q) {
              e.q_out[((size_t)row * e.Hq + tile) * kBM + m] = b;
            } else {
              const int kvsel = is_v ? 1 : 0;
              const int hk = tile - e.Hq - (is_v ? e.Hkv : 0);
              const int loc = e.row_kvloc[row];
              size_t off;
              if (e.prefill) {
                off = (((size_t)kvsel * e.Hkv + hk) * e.pcap + loc) * kBM + m;
              } else {
                const int page = loc / e.pt, o = loc % e.pt;
                off = ((((size_t)page * 2 + kvsel) * e.Hkv + hk) * e.pt + o) * kBM + m;
              }
              e.kv[off] = b;
            }
          }
        }
      } else if constexpr (EPI == EPI_SAMPLE) {
#pragma unroll
        for (int n = 0; n < BN; ++n) {
          if (n < a.n_valid && a.row_active[a.row0 + n]) {
            unsigned long long key = 0ull;
            if (gm < a.M) {
              if (a.logits_dump) a.logits_dump[(size_t)(a.row0 + n) * a.ld_out + gm] = v[n];
              const float g = gumbel(a.seed, (uint32_t)a.row_uid[a.row0 + n], (uint32_t)a.row_t[a.row0 + n],
                                     (uint32_t)gm);
              key = order_key(__fadd_rn(__fmul_rn(v[n], a.inv_temp), g), (uint32_t)gm);
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
              const unsigned long long other = __shfl_xor_sync(0xffffffffu, key, o);
              key = other > key ? other : key;
            }
            if (lane == 0) atomicMax(&skey[n], key);
          }
        }
        asm volatile("bar.sync 1, 128;" ::: "memory");
        if (threadIdx.x - 64 < BN) {
          const int n = threadIdx.x - 64;
          if (skey[n]) atomicMax(a.keys + a.row0 + n, skey[n]);
          skey[n] = 0ull;
        }
        asm volatile("bar.sync 1, 128;" ::: "memory");
      }
    }
  }

  if (threadIdx.x == 64) stamp(a, 10);
  if (S > 1) {
    // producer / MMA warps: complete the start-up barrier phase and arrive on the
    // partials-written phase the epilogue waits for.  Then keep this CTA's smem
    // alive until every peer has signalled that it finished reading it.
    if (warp < 2) {
      asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
      asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
    }
    if (threadIdx.x == 64) mbar_wait(consumed, 0);
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
