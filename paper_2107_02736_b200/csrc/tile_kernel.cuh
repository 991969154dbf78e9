// tile_kernel.cuh — the fused tcgen05 distance-tile kernel (K1 / K2 of DESIGN.md).
//
// One persistent CTA per SM sweeps work units (query block of 128 rows) x
// (chunk of 256-column dataset tiles).  Roles:
//   warp 0      TMA producer (one elected lane): A = query block (resident in
//               smem for the whole unit when it fits), B = 256x64 dataset
//               K-blocks through a multi-stage mbarrier ring.
//   warp 1      MMA issuer (one lane): tcgen05.mma kind::f16, M=128 N=256,
//               fp32 accumulator in TMEM, 2 accumulator buffers x 256 cols.
//   warp 2      TMEM allocator.
//   warps 4-19  epilogue: warp w reads TMEM lane quarter (w%4) and column
//               quarter (w-4)/4 (64 columns) with tcgen05.ld; each thread owns
//               ONE query row, so the per-query row sum needs no shuffles.
//               The tile's 256 column norms are TMA-staged in smem (1 KB ring).
// The S = Q X^T tile never leaves the SM: the epilogue turns it into
//   d2 = |q|^2 + |x|^2 - 2 S          (fp32, exact for the integer encoding)
// and then, by mode,
//   KDE_GAUSS  sum exp2(d2 * -log2e/(2h^2))       -> naive_kde gaussian
//   KDE_EXP    sum exp2(sqrt(d2) * -log2e/h)       -> naive_kde exponential
//   TILEMIN    min d2 over each 64-column quarter tile (k-NN threshold pass)
//   FILTER     append (d2, col) when d2 <= tau[row]  (k-NN candidate pass)
// Reference: naive_kde estimators.py:144-149 -> batch_sqdist distance.py:69-85
// -> kernel_from_distance kernels.py:65-83 -> .mean(axis=1); brute_force_knn
// ann.py:105-111.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdint>
#include "ptx.cuh"

namespace dk {

enum TileMode : int { MODE_KDE_GAUSS = 0, MODE_KDE_EXP = 1, MODE_TILEMIN = 2, MODE_FILTER = 3 };

constexpr int kBM = 128;           // query rows per tile (UMMA M)
constexpr int kBN = 256;           // dataset columns per tile (UMMA N)
constexpr int kBK = 64;            // K elements per block (128 B rows, SWIZZLE_128B)
constexpr int kABlockBytes = kBM * kBK * 2;   // 16 KB
constexpr int kBBlockBytes = kBN * kBK * 2;   // 32 KB
constexpr int kEpiWarp0 = 4;
constexpr int kNumEpiWarps = 16;
constexpr int kThreads = 32 * (kEpiWarp0 + kNumEpiWarps);  // 640
constexpr int kColGroups = 4;      // 64-column groups per tile (one per epilogue warp of a lane quarter)
constexpr int kXnSlots = 4;        // column-norm staging ring (1 KB per tile)
constexpr uint32_t kTmemCols = 512;  // 2 accumulator buffers x 256 fp32 columns

struct TileParams {
  int32_t nq;              // valid query rows
  int32_t nq_pad;          // multiple of 128
  int32_t nqb;             // nq_pad / 128
  int64_t n;               // valid dataset columns (local shard)
  int32_t ntiles;          // tiles in the sweep
  int32_t tile_stride;     // dataset tile index = t * tile_stride
  int32_t tiles_per_unit;
  int32_t ncc;             // column chunks = ceil(ntiles / tiles_per_unit)
  int32_t kblocks;         // Kp / 64
  int32_t a_resident;      // 1: query block loaded once per unit
  int32_t stages;          // B ring depth
  const float* xn;         // [n_pad] |x|^2 (encoding-consistent)
  const float* qn;         // [nq_pad] |q|^2
  const float* m2s;        // device scalar: -2 / (scale_q * scale_x)
  float negc;              // exp2 scale: gaussian -log2e/(2h^2); exponential -log2e/h
  double* part;            // KDE: [ncc*kColGroups][nq_pad] partial sums
  float* tmin;             // TILEMIN: [ntiles*kColGroups][nq_pad]
  const float* tau;        // FILTER: [nq_pad] thresholds
  uint32_t* cand_cnt;      // FILTER: [nq_pad]
  unsigned long long* cand;  // FILTER: [nq_pad][cap] keys (f32 bits << 32 | col)
  int32_t cap;
  const int32_t* row_map;  // FILTER subset rerun: query row -> output slot (nullptr = identity)
};

__host__ __device__ inline size_t tile_smem_bytes(int kblocks, int a_resident, int stages) {
  size_t a = a_resident ? size_t(kblocks) * kABlockBytes : size_t(stages) * kABlockBytes;
  size_t b = size_t(stages) * kBBlockBytes;
  return 1024 /*align slack*/ + a + b + size_t(kXnSlots) * kBN * 4 + 512 /*barriers*/;
}

template <int MODE>
__device__ __forceinline__ void epi_chunk(const uint32_t (&r)[32], const float* __restrict__ xs_smem, float qn,
                                          float m2s, float negc, float tau, bool full, int64_t cbase, int64_t n,
                                          float& s0, float& s1, float& s2, float& s3, float& mn, const TileParams& p,
                                          int row) {
  const float4* x4 = reinterpret_cast<const float4*>(xs_smem);
  if (full) {
#pragma unroll
    for (int j4 = 0; j4 < 8; ++j4) {
      const float4 xv = x4[j4];
      const float xs[4] = {xv.x, xv.y, xv.z, xv.w};
#pragma unroll
      for (int jj = 0; jj < 4; ++jj) {
        const int j = j4 * 4 + jj;
        const float d2 = fmaf(__uint_as_float(r[j]), m2s, qn + xs[jj]);
        if constexpr (MODE == MODE_KDE_GAUSS || MODE == MODE_KDE_EXP) {
          float e;
          if constexpr (MODE == MODE_KDE_GAUSS) e = ex2_approx(d2 * negc);
          else e = ex2_approx(sqrt_approx(fmaxf(d2, 0.f)) * negc);
          if (jj == 0) s0 += e; else if (jj == 1) s1 += e; else if (jj == 2) s2 += e; else s3 += e;
        } else if constexpr (MODE == MODE_TILEMIN) {
          mn = fminf(mn, d2);
        } else {
          if (d2 <= tau) {
            const int slot = p.row_map ? p.row_map[row] : row;
            const uint32_t pos = atomicAdd(&p.cand_cnt[slot], 1u);
            if (pos < uint32_t(p.cap))
              p.cand[size_t(slot) * p.cap + pos] =
                  (static_cast<unsigned long long>(__float_as_uint(fmaxf(d2, 0.f))) << 32) |
                  static_cast<unsigned long long>(cbase + j);
          }
        }
      }
    }
  } else {
    const int lim = int(min(int64_t(32), n - cbase));
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      if (j >= lim) continue;
      const float d2 = fmaf(__uint_as_float(r[j]), m2s, qn + xs_smem[j]);
      if constexpr (MODE == MODE_KDE_GAUSS) {
        s0 += ex2_approx(d2 * negc);
      } else if constexpr (MODE == MODE_KDE_EXP) {
        s0 += ex2_approx(sqrt_approx(fmaxf(d2, 0.f)) * negc);
      } else if constexpr (MODE == MODE_TILEMIN) {
        mn = fminf(mn, d2);
      } else {
        if (d2 <= tau) {
          const int slot = p.row_map ? p.row_map[row] : row;
          const uint32_t pos = atomicAdd(&p.cand_cnt[slot], 1u);
          if (pos < uint32_t(p.cap))
            p.cand[size_t(slot) * p.cap + pos] =
                (static_cast<unsigned long long>(__float_as_uint(fmaxf(d2, 0.f))) << 32) |
                static_cast<unsigned long long>(cbase + j);
        }
      }
    }
  }
}

template <int MODE>
__global__ void __launch_bounds__(kThreads, 1)
    tile_kernel(const __grid_constant__ CUtensorMap tmapA, const __grid_constant__ CUtensorMap tmapB,
                const TileParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int stages = p.stages;
  uint8_t* smemA = smem;
  uint8_t* smemB = smem + (p.a_resident ? size_t(p.kblocks) * kABlockBytes : size_t(stages) * kABlockBytes);
  float* smemX = reinterpret_cast<float*>(smemB + size_t(stages) * kBBlockBytes);  // [kXnSlots][256]
  uint64_t* bars = reinterpret_cast<uint64_t*>(smemX + kXnSlots * kBN);
  uint64_t* full_bar = bars;                 // [stages]
  uint64_t* empty_bar = bars + stages;       // [stages]
  uint64_t* tfull_bar = bars + 2 * stages;   // [2]
  uint64_t* tempty_bar = tfull_bar + 2;      // [2]
  uint64_t* afull_bar = tempty_bar + 2;      // [1]
  uint64_t* aempty_bar = afull_bar + 1;      // [1]
  uint64_t* xfull_bar = aempty_bar + 1;      // [kXnSlots]
  uint64_t* xempty_bar = xfull_bar + kXnSlots;  // [kXnSlots]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(xempty_bar + kXnSlots);

  const uint32_t warp = warp_id_sync();
  const uint32_t lane = lane_id();
  const int nunits = p.nqb * p.ncc;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmapA);
    tma_prefetch_desc(&tmapB);
    for (int s = 0; s < stages; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull_bar[a], 1);
      mbar_init(&tempty_bar[a], kNumEpiWarps);
    }
    mbar_init(afull_bar, 1);
    mbar_init(aempty_bar, 1);
    for (int x = 0; x < kXnSlots; ++x) {
      mbar_init(&xfull_bar[x], 1);
      mbar_init(&xempty_bar[x], kNumEpiWarps);
    }
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc<kTmemCols>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    // ===================== TMA producer =====================
    if (lane == 0) {
      const uint64_t pol_b = policy_evict_last();   // dataset tiles are re-read by other query blocks
      const uint64_t pol_a = policy_evict_last();
      int stage = 0;
      uint32_t phase = 0;
      int uiter = 0;
      uint32_t titer = 0;
      for (int u = blockIdx.x; u < nunits; u += gridDim.x, ++uiter) {
        const int qb = u % p.nqb, cc = u / p.nqb;
        const int t0 = cc * p.tiles_per_unit;
        const int t1 = min(p.ntiles, t0 + p.tiles_per_unit);
        if (p.a_resident) {
          mbar_wait(aempty_bar, (uiter & 1) ^ 1);
          mbar_arrive_expect_tx(afull_bar, uint32_t(p.kblocks) * kABlockBytes);
          for (int kb = 0; kb < p.kblocks; ++kb)
            tma_load_2d(smemA + size_t(kb) * kABlockBytes, &tmapA, afull_bar, kb * kBK, qb * kBM, pol_a);
        }
        for (int t = t0; t < t1; ++t, ++titer) {
          const int col0 = t * p.tile_stride * kBN;
          {  // column norms of this tile -> smem ring slot
            const uint32_t xs = titer % kXnSlots;
            mbar_wait(&xempty_bar[xs], ((titer / kXnSlots) & 1) ^ 1);
            mbar_arrive_expect_tx(&xfull_bar[xs], kBN * 4);
            bulk_load(smemX + xs * kBN, p.xn + col0, kBN * 4, &xfull_bar[xs]);
          }
          for (int kb = 0; kb < p.kblocks; ++kb) {
            mbar_wait(&empty_bar[stage], phase ^ 1);
            if (p.a_resident) {
              mbar_arrive_expect_tx(&full_bar[stage], kBBlockBytes);
            } else {
              mbar_arrive_expect_tx(&full_bar[stage], kBBlockBytes + kABlockBytes);
              tma_load_2d(smemA + size_t(stage) * kABlockBytes, &tmapA, &full_bar[stage], kb * kBK, qb * kBM,
                          pol_a);
            }
            tma_load_2d(smemB + size_t(stage) * kBBlockBytes, &tmapB, &full_bar[stage], kb * kBK, col0, pol_b);
            if (++stage == stages) { stage = 0; phase ^= 1; }
          }
        }
      }
    }
  } else if (warp == 1) {
    // ===================== MMA issuer =====================
    if (lane == 0) {
      constexpr uint32_t idesc = idesc_f16_f32(kBM, kBN);
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      int uiter = 0;
      const uint32_t a0 = smem_u32(smemA), b0 = smem_u32(smemB);
      for (int u = blockIdx.x; u < nunits; u += gridDim.x, ++uiter) {
        const int cc = u / p.nqb;
        const int t0 = cc * p.tiles_per_unit;
        const int t1 = min(p.ntiles, t0 + p.tiles_per_unit);
        if (p.a_resident) {
          mbar_wait(afull_bar, uiter & 1);
          tc_fence_after();
        }
        for (int t = t0; t < t1; ++t) {
          mbar_wait(&tempty_bar[acc], acc_phase ^ 1);
          tc_fence_after();
          const uint32_t d_tmem = tmem_base + uint32_t(acc * kBN);
          for (int kb = 0; kb < p.kblocks; ++kb) {
            mbar_wait(&full_bar[stage], phase);
            tc_fence_after();
            const uint32_t abase = p.a_resident ? a0 + uint32_t(kb) * kABlockBytes : a0 + uint32_t(stage) * kABlockBytes;
            const uint32_t bbase = b0 + uint32_t(stage) * kBBlockBytes;
            const uint64_t ad = sw128_kmajor_desc(abase), bd = sw128_kmajor_desc(bbase);
#pragma unroll
            for (int k = 0; k < kBK / 16; ++k)
              mma_f16_ss(d_tmem, ad + uint64_t(2 * k), bd + uint64_t(2 * k), idesc, (kb | k) != 0);
            mma_commit(&empty_bar[stage]);
            if (++stage == stages) { stage = 0; phase ^= 1; }
          }
          mma_commit(&tfull_bar[acc]);
          if (++acc == 2) { acc = 0; acc_phase ^= 1; }
        }
        if (p.a_resident) mma_commit(aempty_bar);
      }
    }
  } else if (warp >= kEpiWarp0) {
    // ===================== epilogue =====================
    const int ew = int(warp) - kEpiWarp0;
    const int quarter = int(warp & 3);
    const int cg = ew >> 2;  // 64-column group of the tile
    int acc = 0;
    uint32_t acc_phase = 0;
    uint32_t titer = 0;
    const float m2s = *p.m2s;
    const float negc = p.negc;
    for (int u = blockIdx.x; u < nunits; u += gridDim.x) {
      const int qb = u % p.nqb, cc = u / p.nqb;
      const int t0 = cc * p.tiles_per_unit;
      const int t1 = min(p.ntiles, t0 + p.tiles_per_unit);
      const int row = qb * kBM + quarter * 32 + int(lane);
      const float qn = p.qn[row];
      float tau = 0.f;
      if constexpr (MODE == MODE_FILTER) tau = p.tau[row];
      double usum = 0.0;
      for (int t = t0; t < t1; ++t, ++titer) {
        const uint32_t xs = titer % kXnSlots;
        mbar_wait(&tfull_bar[acc], acc_phase);
        tc_fence_after();
        const uint32_t taddr = tmem_base + (uint32_t(quarter * 32) << 16) + uint32_t(acc * kBN + cg * 64);
        uint32_t r0[32], r1[32];
        tmem_ld32(taddr, r0);
        tmem_ld32(taddr + 32u, r1);
        tmem_ld_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&tempty_bar[acc]);
        if (++acc == 2) { acc = 0; acc_phase ^= 1; }
        mbar_wait(&xfull_bar[xs], (titer / kXnSlots) & 1);
        const int64_t cbase = int64_t(t) * p.tile_stride * kBN + cg * 64;
        const float* xsm = smemX + xs * kBN + cg * 64;
        const bool full = cbase + 64 <= p.n;
        float s0 = 0.f, s1 = 0.f, s2 = 0.f, s3 = 0.f;
        float mn = __int_as_float(0x7f800000);
        epi_chunk<MODE>(r0, xsm, qn, m2s, negc, tau, full, cbase, p.n, s0, s1, s2, s3, mn, p, row);
        epi_chunk<MODE>(r1, xsm + 32, qn, m2s, negc, tau, full, cbase + 32, p.n, s0, s1, s2, s3, mn, p, row);
        __syncwarp();
        if (lane == 0) mbar_arrive(&xempty_bar[xs]);
        if constexpr (MODE == MODE_KDE_GAUSS || MODE == MODE_KDE_EXP) {
          usum += double((s0 + s1) + (s2 + s3));
        } else if constexpr (MODE == MODE_TILEMIN) {
          p.tmin[(size_t(t) * kColGroups + cg) * p.nq_pad + row] = mn;
        }
      }
      if constexpr (MODE == MODE_KDE_GAUSS || MODE == MODE_KDE_EXP) {
        p.part[(size_t(cc) * kColGroups + cg) * p.nq_pad + row] = usum;
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc<kTmemCols>(tmem_base);
  }
}

}  // namespace dk
