// l1.cu — exact laplacian KDE on CUDA cores (K4).
//
// Reference: naive_kde's L1 branch (estimators.py:134-143): for each query,
// sum_i exp(-sum_k |x_ik - y_k| / h) over row blocks, then / n.  L1 is not a
// contraction, so it cannot use the tensor cores; this is a register-tiled
// SIMT kernel: a 128-query x 128-row tile per block, 8x8 outputs per thread,
// 16-dimension double-buffered smem chunks, fp32 |a-b| accumulation with per-chunk partial
// sums, ex2.approx epilogue, fp32 per-tile row sums folded into fp64.
#include "internal.h"
#include "ptx.cuh"

namespace dk {

namespace {

constexpr int TQ = 128, TX = 128, DK = 16, XPAD = 4;
constexpr int kTilesPerBlock = 8;

__global__ void __launch_bounds__(256, 1) l1_kde_kernel(const float* __restrict__ X, int64_t n, int32_t d,
                                                         const double* __restrict__ Q, int64_t nq, int32_t nq_pad,
                                                         float negc, double* __restrict__ part) {
  // double-buffered smem tiles, transposed to [k][row] so each thread reads its 4 queries
  // and 8 rows of one dimension with 3 LDS.128; the next chunk is fetched into registers
  // while the current one is consumed
  __shared__ __align__(16) float Qs[2][DK][TQ + XPAD];
  __shared__ __align__(16) float Xs[2][DK][TX + XPAD];
  constexpr int QL = (TQ * DK) / 256, XL = (TX * DK) / 256;  // per-thread staged loads
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
        const int e = r * 256 + threadIdx.x;
        const int qq = e / DK, kk = e % DK;
        const int64_t qi = q0 + qq;
        qreg[r] = (qi < nq && k0 + kk < d) ? float(Q[qi * d + k0 + kk]) : 0.f;
      }
#pragma unroll
      for (int r = 0; r < XL; ++r) {
        const int e = r * 256 + threadIdx.x;
        const int xx = e / DK, kk = e % DK;
        const int64_t xi = x0 + xx;
        xreg[r] = (xi < n && k0 + kk < d) ? __ldg(X + xi * d + k0 + kk) : 0.f;
      }
    };
    auto stash = [&](int buf) {
#pragma unroll
      for (int r = 0; r < QL; ++r) {
        const int e = r * 256 + threadIdx.x;
        Qs[buf][e % DK][e / DK] = qreg[r];
      }
#pragma unroll
      for (int r = 0; r < XL; ++r) {
        const int e = r * 256 + threadIdx.x;
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

}  // namespace

static int64_t l1_chunks(int64_t n) { return (n + int64_t(TX) * kTilesPerBlock - 1) / (int64_t(TX) * kTilesPerBlock); }

int32_t l1_nq_pad(int64_t nq) { return int32_t((nq + TQ - 1) / TQ * TQ); }

size_t l1_part_count(int64_t n, int32_t nq) {
  const int64_t nq_pad = (int64_t(nq) + TQ - 1) / TQ * TQ;
  return size_t(l1_chunks(n)) * size_t(nq_pad);
}

void launch_l1_kde(const float* X, int64_t n, int32_t d, const double* Q, int64_t nq, double inv_h, double* part,
                   int32_t* nparts, float* /*q32*/, cudaStream_t s) {
  const int32_t nq_pad = int32_t((nq + TQ - 1) / TQ * TQ);
  const int64_t chunks = l1_chunks(n);
  dim3 grid(unsigned(nq_pad / TQ), unsigned(chunks));
  const float negc = float(-inv_h * 1.4426950408889634);
  l1_kde_kernel<<<grid, 256, 0, s>>>(X, n, d, Q, nq, nq_pad, negc, part);
  DK_CHECK_LAUNCH();
  *nparts = int32_t(chunks);
}

}  // namespace dk
