// Weight-streaming "swap-AB" GEMM on tcgen05 for the decode step.
//
//   Y[n][m] = sum_k X[n][k] * W[m][k]      (X: activation rows, W: [out, in] weights)
//
// computed as D = W_tile · X^T with the weight tile as the MMA A operand
// (M = 128 output features) and the R <= 64 activation rows as N, so the
// skinny decode GEMM keeps the 128-row tensor-core shape and its cost is the
// weight stream.  Both operands are TMA-loaded with 128-byte
// swizzle into a STAGES-deep mbarrier ring; one elected thread issues
// tcgen05.mma (kind::f16, bf16 in / fp32 accumulate in TMEM); four epilogue
// warps read TMEM with tcgen05.ld.
//
// Split-K: `split` CTAs of a thread-block cluster share one 128-row tile, each
// streaming a contiguous K range; partials meet in shared memory and every
// rank reduces a column slice over DSMEM in rank order 0..split-1, so the
// result is deterministic and independent of how many rows are live
// (DESIGN.md "batch invariance").  With split == 1 the kernel is persistent
// over tiles and double-buffers the TMEM accumulator.
//
// Epilogues (fused, no extra pass over HBM):
//   EPI_STORE_F32  out[row][m]  = acc                    (QKV pre-norm)
//   EPI_RESID_ADD  out[row][m] += acc                    (o_proj, down: fp32 residual)
//   EPI_SWIGLU     act[row][f]  = bf16(silu(g) * u)      (gate|up interleaved per 64 rows; R12 r5)
//   EPI_SAMPLE     keys[row] = max(key(z*invT + Gumbel)) (lm_head + Philox Gumbel-max sampler)
#pragma once
#include "common.cuh"
#include "sampler.cuh"

namespace isk {

enum EpiKind { EPI_STORE_F32 = 0, EPI_RESID_ADD = 1, EPI_SWIGLU = 2, EPI_SAMPLE = 3 };

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
};

constexpr int kBM = 128;
constexpr int kBK = 64;
constexpr int kGemmThreads = 192;

template <int BN>
struct GemmCfg {
  static constexpr int kStageA = kBM * kBK * 2;        // 16 KB
  static constexpr int kStageB = BN * kBK * 2;
  static constexpr int kStage = kStageA + kStageB;
  static constexpr int kStages = BN == 16 ? 5 : (BN == 32 ? 4 : 3);
  static constexpr int kXbuf = BN * 64 * 4;           // SWIGLU exchange
  static constexpr int kTmemCols = (2 * BN) <= 32 ? 32 : ((2 * BN) <= 64 ? 64 : 128);
  static constexpr int kSmem = kStages * kStage + kXbuf + 1024 /*barriers*/ + 1024 /*align*/;
  static_assert(kBM * BN * 4 <= kStages * kStage, "split-K reduction buffer must fit in the stage ring");
};

__device__ __forceinline__ float silu_f(float x) { return x / (1.0f + expf(-x)); }

template <int BN, int EPI>
__global__ void __launch_bounds__(kGemmThreads, 1)
    gemm_swapab_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                       GemmArgs a) {
  using C = GemmCfg<BN>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* stage_base = smem;
  float* xbuf = reinterpret_cast<float*>(smem + C::kStages * C::kStage);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::kStages * C::kStage + C::kXbuf);
  uint64_t* full = bars;
  uint64_t* empty = bars + C::kStages;
  uint64_t* tfull = bars + 2 * C::kStages;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  __shared__ unsigned long long skey[BN];

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int S = a.split;
  const int rank = S > 1 ? (int)cluster_ctarank() : 0;
  const int cl = S > 1 ? (int)cluster_id_x() : (int)blockIdx.x;
  const int ncl = S > 1 ? (int)nclusters_x() : (int)gridDim.x;
  const int kb_total = a.K / kBK;
  const int kb0 = rank * kb_total / S;
  const int kb1 = (rank + 1) * kb_total / S;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    for (int i = 0; i < C::kStages; ++i) {
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
  if (EPI == EPI_SAMPLE && threadIdx.x < BN) skey[threadIdx.x] = 0ull;
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  pdl_launch_dependents();

  if (warp == 0) {
    // ------------------------------------------------ TMA producer
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      bool waited = false;
      for (int tile = cl; tile < a.num_tiles; tile += ncl) {
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          uint8_t* sa = stage_base + stage * C::kStage;
          mbar_arrive_expect_tx(&full[stage], C::kStage);
          tma_load_2d(sa, &tmA, &full[stage], kb * kBK, tile * kBM, kEvictFirst);
          if (!waited) {  // weights never depend on the previous kernel; activations do
            pdl_wait();
            waited = true;
          }
          tma_load_2d(sa + C::kStageA, &tmB, &full[stage], kb * kBK, a.row0, kEvictLast);
          if (++stage == C::kStages) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
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
        if (++stage == C::kStages) {
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
      mbar_wait(&tfull[acc], acc_phase);
      tc_fence_after();
      float v[BN];
#pragma unroll
      for (int c = 0; c < BN / 16; ++c)
        tmem_ld16(tmem_base + ((uint32_t)(q * 32) << 16) + acc * BN + c * 16, v + c * 16);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[acc]);

      int n_lo = 0, n_hi = BN;
      if (S > 1) {
        // Partials -> own smem (ring is idle: all MMAs of this single tile are done).
        float* red = reinterpret_cast<float*>(stage_base);
#pragma unroll
        for (int n = 0; n < BN; ++n) red[n * kBM + m] = v[n];
        asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
        asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
        n_lo = rank * BN / S;
        n_hi = (rank + 1) * BN / S;
        const uint32_t laddr = smem_u32(red);
#pragma unroll
        for (int n = 0; n < BN; ++n) {
          if (n >= n_lo && n < n_hi) {
            float s = 0.f;
            for (int j = 0; j < S; ++j) s += ld_dsmem_f32(mapa_shared(laddr + (uint32_t)(n * kBM + m) * 4u, j));
            v[n] = s;
          }
        }
      }

      const int gm = tile * kBM + m;
      if constexpr (EPI == EPI_STORE_F32 || EPI == EPI_RESID_ADD) {
#pragma unroll
        for (int n = 0; n < BN; ++n) {
          if (n >= n_lo && n < n_hi && n < a.n_valid && gm < a.M) {
            float* p = a.out + (size_t)(a.row0 + n) * a.ld_out + gm;
            if (EPI == EPI_RESID_ADD) *p += v[n];
            else *p = v[n];
          }
        }
      } else if constexpr (EPI == EPI_SWIGLU) {
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

  if (S > 1) {
    // Non-epilogue warps match the epilogue's first cluster barrier; everyone
    // then waits until all ranks finished reading each other's partials.
    if (warp < 2) {
      __syncwarp();
      asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
      asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
    }
    asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
    asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<C::kTmemCols>(tmem_base);
  }
}

}  // namespace isk
