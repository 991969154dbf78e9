// l1.cu — exact laplacian KDE on CUDA cores (K4).
//
// Reference: naive_kde's L1 branch (estimators.py:134-143): for each query,
// sum_i exp(-sum_k |x_ik - y_k| / h) over row blocks, then / n.  L1 is not a
// contraction, so it cannot use the tensor cores; this is a register-tiled
// SIMT kernel: a 128-query x 128-row tile per block, 8x8 outputs per thread,
// 16-dimension double-buffered smem chunks, fp32 |a-b| accumulation with per-chunk partial
// sums, ex2.approx epilogue, fp32 per-tile row sums folded into fp64.
#include <cstdlib>

#include "internal.h"
#include "ptx.cuh"

namespace dk {

namespace {

#ifndef DK_L1_TQ
#define DK_L1_TQ 128
#endif
constexpr int TQ = DK_L1_TQ, TX = 128, DK = 16, XPAD = 4;
constexpr int kL1Threads = TQ * 2;  // 8 x 8 outputs per thread
constexpr int kL1Blocks = 256 / kL1Threads;  // CTAs per SM (~250 registers per thread)
constexpr int kTilesPerBlock = 8;

__global__ void __launch_bounds__(kL1Threads, kL1Blocks) l1_kde_kernel(const float* __restrict__ X, int64_t n, int32_t d,
                                                         const double* __restrict__ Q, int64_t nq, int32_t nq_pad,
                                                         float negc, double* __restrict__ part) {
  // double-buffered smem tiles, transposed to [k][row] so each thread reads its 4 queries
  // and 8 rows of one dimension with 3 LDS.128; the next chunk is fetched into registers
  // while the current one is consumed
  __shared__ __align__(16) float Qs[2][DK][TQ + XPAD];
  __shared__ __align__(16) float Xs[2][DK][TX + XPAD];
  constexpr int QL = (TQ * DK) / kL1Threads, XL = (TX * DK) / kL1Threads;  // per-thread staged loads
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  const int64_t q0 = int64_t(blockIdx.x) * TQ;
  const int64_t tile0 = int64_t(blockIdx.y) * kTilesPerBlock;
  const int nchunks = (d + DK - 1) / DK;
  double qacc[8] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
  for (int xt = 0; xt < kTilesPerBlock; ++xt) {
    const int64_t x0 = (tile0 + xt) * TX;
    if (x0 >= n) break;
    float acc[8][8];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
      for (int j = 0; j < 8; ++j) acc[i][j] = 0.f;
    float qreg[QL], xreg[XL];
    auto fetch = [&](int k0) {
#pragma unroll
      for (int r = 0; r < QL; ++r) {
        const int e = r * kL1Threads + threadIdx.x;
        const int qq = e / DK, kk = e % DK;
        const int64_t qi = q0 + qq;
        qreg[r] = (qi < nq && k0 + kk < d) ? float(Q[qi * d + k0 + kk]) : 0.f;
      }
#pragma unroll
      for (int r = 0; r < XL; ++r) {
        const int e = r * kL1Threads + threadIdx.x;
        const int xx = e / DK, kk = e % DK;
        const int64_t xi = x0 + xx;
        xreg[r] = (xi < n && k0 + kk < d) ? __ldg(X + xi * d + k0 + kk) : 0.f;
      }
    };
    auto stash = [&](int buf) {
#pragma unroll
      for (int r = 0; r < QL; ++r) {
        const int e = r * kL1Threads + threadIdx.x;
        Qs[buf][e % DK][e / DK] = qreg[r];
      }
#pragma unroll
      for (int r = 0; r < XL; ++r) {
        const int e = r * kL1Threads + threadIdx.x;
        Xs[buf][e % DK][e / DK] = xreg[r];
      }
    };
    fetch(0);
    stash(0);
    __syncthreads();
    for (int c = 0; c < nchunks; ++c) {
      const int buf = c & 1;
      if (c + 1 < nchunks) fetch((c + 1) * DK);  // in flight during the compute below
      // packed over row pairs: one FADD2 (x - q) and one FADD2 (acc + |d|, abs as an
      // operand modifier) per two (pair, dim) terms — half the FP32 instructions of the
      // scalar form, same IEEE operations and order per term
      float2 part_acc[8][4];
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) part_acc[i][j] = make_float2(0.f, 0.f);
#pragma unroll 4
      for (int kk = 0; kk < DK; ++kk) {
        const float4 qa = *reinterpret_cast<const float4*>(&Qs[buf][kk][ty * 4]);
        const float4 qb = *reinterpret_cast<const float4*>(&Qs[buf][kk][TQ / 2 + ty * 4]);
        // rows tx*4..+3 and 64+tx*4..+3: each 8-lane phase of an LDS.128 reads 128
        // contiguous bytes (conflict-free; tx*8 strides would 2-way conflict)
        const float4 xa = *reinterpret_cast<const float4*>(&Xs[buf][kk][tx * 4]);
        const float4 xb = *reinterpret_cast<const float4*>(&Xs[buf][kk][TX / 2 + tx * 4]);
        const float qs[8] = {qa.x, qa.y, qa.z, qa.w, qb.x, qb.y, qb.z, qb.w};
        const float2 xp[4] = {make_float2(xa.x, xa.y), make_float2(xa.z, xa.w), make_float2(xb.x, xb.y),
                              make_float2(xb.z, xb.w)};
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const float2 q2 = make_float2(qs[i], qs[i]);
#pragma unroll
          for (int j = 0; j < 4; ++j) part_acc[i][j] = add2(part_acc[i][j], abs2(sub2(q2, xp[j])));
        }
      }
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          acc[i][2 * j] += part_acc[i][j].x;
          acc[i][2 * j + 1] += part_acc[i][j].y;
        }
      if (c + 1 < nchunks) stash(buf ^ 1);
      __syncthreads();
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      float rs = 0.f;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const bool valid = x0 + (j < 4 ? tx * 4 + j : TX / 2 + tx * 4 + (j - 4)) < n;
        const float e = ex2_approx(acc[i][j] * negc);
        rs += valid ? e : 0.f;
      }
      qacc[i] += double(rs);
    }
  }
  // reduce over the 16 tx lanes (same ty within a warp half)
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    double v = qacc[i];
#pragma unroll
    for (int o = 8; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    qacc[i] = v;
  }
  if (tx == 0) {
#pragma unroll
    for (int i = 0; i < 8; ++i)
      part[size_t(blockIdx.y) * nq_pad + q0 + (i < 4 ? ty * 4 + i : TQ / 2 + ty * 4 + (i - 4))] = qacc[i];
  }
}

// ---- v2: the same register tile fed by a cp.async (LDGSTS) pipeline ----
// The register-staged loads above cost the FADD2 pipe ~30% (ncu, c4: long-scoreboard waits on the
// staged global loads before each shared-memory store, 2-way conflicts on those stores, one barrier
// per 16 dimensions with 2 warps per scheduler).  Here each chunk of 32 dimensions goes global ->
// shared memory with 4-byte cp.async (zero fill past n / d), three stages, issued two chunks ahead
// across tile boundaries, so nothing waits on a scoreboard and there is one barrier per 32
// dimensions.  The element -> (row, dim) map puts 8 consecutive dimensions x 4 rows in a warp: full
// 32-byte sectors from global memory and 32 distinct banks on the transposed store.  Queries are
// converted to fp32 once per call (q32) so they ride the same copies.
#ifndef DK_L1_DK2
#define DK_L1_DK2 32
#endif
constexpr int DK2 = DK_L1_DK2;  // dimensions per chunk (32 or 64)
constexpr int kL1KH = DK2 == 64 ? 3 : 2;  // thread-id bits (from bit 5) that index the chunk's 8-dimension groups
constexpr int kL1Pitch = TX + XPAD;  // floats per dimension row (TQ == TX)
#ifndef DK_L1_STAGES
#define DK_L1_STAGES 3
#endif
constexpr int kL1Stages = DK_L1_STAGES;
constexpr size_t kL1SmemV2 = size_t(kL1Stages) * 2 * DK2 * kL1Pitch * sizeof(float);

__global__ void l1_q32_kernel(const double* __restrict__ Q, int64_t nq, int32_t d, int64_t total,
                              float* __restrict__ q32) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < total) q32[i] = i < nq * d ? float(Q[i]) : 0.f;
}

__global__ void __launch_bounds__(256, 1) l1_kde_kernel_v2(const float* __restrict__ X, int64_t n, int32_t d,
                                                            const float* __restrict__ Q32, int32_t nq_pad,
                                                            float negc, double* __restrict__ part) {
  static_assert(TQ == 128 && TX == 128, "v2 index map");
  extern __shared__ __align__(16) float l1_smem[];
  // [stage][Q | X][DK2][kL1Pitch]
  auto qs = [&](int st) { return l1_smem + size_t(st) * 2 * DK2 * kL1Pitch; };
  auto xs = [&](int st) { return l1_smem + size_t(st) * 2 * DK2 * kL1Pitch + size_t(DK2) * kL1Pitch; };
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  const int64_t q0 = int64_t(blockIdx.x) * TQ;
  const int64_t tile0 = int64_t(blockIdx.y) * kTilesPerBlock;
  const int nchunks = (d + DK2 - 1) / DK2;
  const int ntl = int(min(int64_t(kTilesPerBlock), (n - tile0 * TX + TX - 1) / TX));
  const int total = ntl * nchunks;
  // this thread's 16 (row, dim) slots of a chunk: idx = r * 256 + tid, dim = idx[0:3) | idx[5:7) << 3,
  // row = idx[3:5) | idx[7:12) << 2
  static_assert(DK2 == 32 || DK2 == 64, "chunk widths of the index map");
  const int kk_t = (threadIdx.x & 7) | (((threadIdx.x >> 5) & (DK2 / 8 - 1)) << 3);
  const int row_t = ((threadIdx.x >> 3) & 3) | ((threadIdx.x >> (5 + kL1KH)) << 2);
  constexpr int kRowStep = 4 << (3 - kL1KH);
  auto load = [&](int it, int st) {
    const int xt = it / nchunks, c = it - xt * nchunks;
    const int64_t x0 = (tile0 + xt) * TX;
    const int k = c * DK2 + kk_t;
    const bool kin = k < d;
    float* qd = qs(st) + kk_t * kL1Pitch;
    float* xd = xs(st) + kk_t * kL1Pitch;
#pragma unroll
    for (int r = 0; r < TX / kRowStep; ++r) {
      const int row = row_t + kRowStep * r;
      const int64_t xi = x0 + row;
      const bool xin = kin && xi < n;
      cp_async4(qd + row, kin ? Q32 + (q0 + row) * d + k : Q32, kin ? 4u : 0u);
      cp_async4(xd + row, xin ? X + xi * d + k : X, xin ? 4u : 0u);
    }
  };
  double qacc[8] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
  float acc[8][8];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[i][j] = 0.f;
#pragma unroll
  for (int p = 0; p < kL1Stages - 1; ++p) {
    if (p < total) load(p, p);
    cp_async_commit();
  }
  int xt = 0, c = 0, st = 0;
  for (int it = 0; it < total; ++it) {
    cp_async_wait<kL1Stages - 2>();  // all but the newest kL1Stages - 2 groups: chunk `it` has landed
    __syncthreads();  // ... for every thread's copies; every warp is done reading the stage refilled next
    {
      const int nx = it + kL1Stages - 1;
      if (nx < total) load(nx, st == 0 ? kL1Stages - 1 : st - 1);
      cp_async_commit();
    }
    const float* Qb = qs(st);
    const float* Xb = xs(st);
    float2 part_acc[8][4];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) part_acc[i][j] = make_float2(0.f, 0.f);
#pragma unroll 4
    for (int kk = 0; kk < DK2; ++kk) {
      const float4 qa = *reinterpret_cast<const float4*>(Qb + kk * kL1Pitch + ty * 4);
      const float4 qb = *reinterpret_cast<const float4*>(Qb + kk * kL1Pitch + TQ / 2 + ty * 4);
      const float4 xa = *reinterpret_cast<const float4*>(Xb + kk * kL1Pitch + tx * 4);
      const float4 xb = *reinterpret_cast<const float4*>(Xb + kk * kL1Pitch + TX / 2 + tx * 4);
      const float qv[8] = {qa.x, qa.y, qa.z, qa.w, qb.x, qb.y, qb.z, qb.w};
      const float2 xp[4] = {make_float2(xa.x, xa.y), make_float2(xa.z, xa.w), make_float2(xb.x, xb.y),
                            make_float2(xb.z, xb.w)};
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const float2 q2 = make_float2(qv[i], qv[i]);
#pragma unroll
        for (int j = 0; j < 4; ++j) part_acc[i][j] = add2(part_acc[i][j], abs2(sub2(q2, xp[j])));
      }
    }
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        acc[i][2 * j] += part_acc[i][j].x;
        acc[i][2 * j + 1] += part_acc[i][j].y;
      }
    if (++c == nchunks) {  // tile done: exponentials, row sums
      const int64_t x0 = (tile0 + xt) * TX;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        float rs = 0.f;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const bool valid = x0 + (j < 4 ? tx * 4 + j : TX / 2 + tx * 4 + (j - 4)) < n;
          const float e = ex2_approx(acc[i][j] * negc);
          rs += valid ? e : 0.f;
          acc[i][j] = 0.f;
        }
        qacc[i] += double(rs);
      }
      c = 0;
      ++xt;
    }
    if (++st == kL1Stages) st = 0;
  }
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    double v = qacc[i];
#pragma unroll
    for (int o = 8; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    qacc[i] = v;
  }
  if (tx == 0) {
#pragma unroll
    for (int i = 0; i < 8; ++i)
      part[size_t(blockIdx.y) * nq_pad + q0 + (i < 4 ? ty * 4 + i : TQ / 2 + ty * 4 + (i - 4))] = qacc[i];
  }
}

}  // namespace

static int64_t l1_chunks(int64_t n) { return (n + int64_t(TX) * kTilesPerBlock - 1) / (int64_t(TX) * kTilesPerBlock); }

int32_t l1_nq_pad(int64_t nq) { return int32_t((nq + TQ - 1) / TQ * TQ); }

size_t l1_part_count(int64_t n, int32_t nq) {
  const int64_t nq_pad = (int64_t(nq) + TQ - 1) / TQ * TQ;
  return size_t(l1_chunks(n)) * size_t(nq_pad);
}

void launch_l1_kde(const float* X, int64_t n, int32_t d, const double* Q, int64_t nq, double inv_h, double* part,
                   int32_t* nparts, float* q32, cudaStream_t s) {
  const int32_t nq_pad = int32_t((nq + TQ - 1) / TQ * TQ);
  const int64_t chunks = l1_chunks(n);
  dim3 grid(unsigned(nq_pad / TQ), unsigned(chunks));
  const float negc = float(-inv_h * 1.4426950408889634);
  static const bool legacy = [] {  // A/B: DK_L1_LEGACY=1 runs the register-staged kernel
    const char* v = std::getenv("DK_L1_LEGACY");
    return v && v[0] == '1';
  }();
  if (q32 != nullptr && !legacy && TQ == 128) {
    const int64_t total = int64_t(nq_pad) * d;
    l1_q32_kernel<<<unsigned((total + 255) / 256), 256, 0, s>>>(Q, nq, d, total, q32);
    DK_CHECK_LAUNCH();
    static const bool attr = [] {
      DK_CUDA(cudaFuncSetAttribute(l1_kde_kernel_v2, cudaFuncAttributeMaxDynamicSharedMemorySize, int(kL1SmemV2)));
      return true;
    }();
    (void)attr;
    l1_kde_kernel_v2<<<grid, 256, kL1SmemV2, s>>>(X, n, d, q32, nq_pad, negc, part);
    DK_CHECK_LAUNCH();
  } else {
    l1_kde_kernel<<<grid, kL1Threads, 0, s>>>(X, n, d, Q, nq, nq_pad, negc, part);
    DK_CHECK_LAUNCH();
  }
  *nparts = int32_t(chunks);
}

}  // namespace dk
