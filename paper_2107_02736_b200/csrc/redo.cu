// redo.cu — fp64 re-evaluation of the queries an exact-KDE sweep cannot certify (capi.cu dk_naive).
//
// The tile sweeps take d2 = |q|^2 + |x|^2 - 2 q.x from fp16 operand pairs accumulated in fp32, so
// d2 carries an ABSOLUTE error delta_q ~ u (|q|^2 + |x|^2) (u: unit roundoff of the encoding plus the
// accumulation).  Two cases turn that into a relative error of the kernel value above the gate:
//  * exponential kernel, small d2: exp(-sqrt(d2)/h) sees delta_q / (2 sqrt(d2) h), unbounded at a
//    coincident pair (a query that is a data point carries its own term, usually the largest, with
//    an error of sqrt(delta_q)/h);
//  * gaussian kernel with 2h^2 small against the norms: every term sees delta_q / 2h^2.
// guard_tau_kernel turns the tolerance into a per-query threshold on d2 (exponential: the sweep flags a
// row whose smallest approximate d2 falls under it, tile_kernel.cuh exp_guard_flag) or flags the query
// outright (gaussian).  Flagged queries are listed and their sums recomputed here as the reference
// computes them — fp64 direct differences over every row (naive_kde estimators.py:144-149 via
// batch_sqdist distance.py:69-85 and kernel_from_distance kernels.py:65-83) — in a fixed summation
// order, and overwrite the sweep's values.  No host round trip: the list length stays on the device.

#include "internal.h"

namespace dk {

namespace {

constexpr int kRedoThreads = 256;
constexpr int kRedoWarps = kRedoThreads / 32;

// tau[row] = (delta_q / (tol h))^2 with delta_q = delta_rel (|q|^2 + xn_max) (exponential), or the flag
// itself when delta_q / 2h^2 > tol (gaussian; tau = 0).  Rows past nq never flag.
__global__ void guard_tau_kernel(const float* __restrict__ qn, int32_t nq_pad, int64_t nq, float xn_max,
                                 double delta_rel, double tol, double h, int32_t gaussian,
                                 float* __restrict__ tau, uint32_t* __restrict__ flag) {
  const int row = blockIdx.x * blockDim.x + threadIdx.x;
  if (row >= nq_pad) return;
  const double delta = delta_rel * (double(qn[row]) + double(xn_max));
  float t = 0.f;
  uint32_t f = 0u;
  if (row < nq) {
    if (gaussian) {
      f = delta > tol * 2.0 * h * h ? 1u : 0u;
    } else {
      const double r = delta / (tol * h);
      t = float(fmin(r * r, 3.0e38));
    }
  }
  tau[row] = t;
  flag[row] = f;
}

// the gaussian flag from the raw queries (the two-precision path keeps its operands in ball order): one warp
// per query, |q - mu|^2 in fp64, flag = delta_rel (|q - mu|^2 + xn_max) > lim (= tol 2h^2)
__global__ void guard_flag_raw_kernel(const double* __restrict__ Q, const double* __restrict__ mu, int32_t d,
                                      int64_t nq, float xn_max, double delta_rel, double lim,
                                      uint32_t* __restrict__ flag) {
  const int64_t q = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (q >= nq) return;
  double s = 0.0;
  for (int i = lane; i < d; i += 32) {
    const double t = Q[size_t(q) * d + i] - (mu != nullptr ? mu[i] : 0.0);
    s = fma(t, t, s);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) flag[q] = delta_rel * (s + double(xn_max)) > lim ? 1u : 0u;
}

// list the flagged rows (ascending), and the rows whose sweep value fell under `under`: the fp32
// epilogue bottoms out near 2^-126 per term (ex2.approx flushes, the polynomial clamps: a query far from
// every row comes back as ~1.5e-39 whatever its true 1e-50 is), the fp64 recomputation does not; one CTA
__global__ void __launch_bounds__(1024) redo_list_kernel(const uint32_t* __restrict__ flag,
                                                         const double* __restrict__ out, double under, int64_t nq,
                                                         int32_t* __restrict__ list, int32_t* __restrict__ count) {
  __shared__ int s_w[32];
  __shared__ int s_base;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) s_base = 0;
  __syncthreads();
  for (int64_t r0 = 0; r0 < nq; r0 += blockDim.x) {
    const int64_t r = r0 + threadIdx.x;
    const bool on = r < nq && ((flag != nullptr && flag[r] != 0u) || !(out[r] >= under));
    const uint32_t m = __ballot_sync(0xffffffffu, on);
    if (lane == 0) s_w[warp] = __popc(m);
    __syncthreads();
    int off = s_base;
    for (int w = 0; w < warp; ++w) off += s_w[w];
    if (on) list[off + __popc(m & ((1u << lane) - 1u))] = int32_t(r);
    __syncthreads();
    if (threadIdx.x == 0) {
      int tot = 0;
      for (int w = 0; w < 32; ++w) tot += s_w[w];
      s_base += tot;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) *count = s_base;
}

// work item = (listed query, row chunk).  G lanes share a row (coalesced float loads, fp64 direct
// difference, fixed shuffle tree), each group sums its rows' kernel values in fp64; the block's
// groups are added in a fixed order into part[item].
template <int G>
__global__ void __launch_bounds__(kRedoThreads) redo_eval_kernel(const float* __restrict__ X, int64_t n, int32_t d,
                                                                 const double* __restrict__ Q, int32_t family,
                                                                 double c, const int32_t* __restrict__ list,
                                                                 const int32_t* __restrict__ count, int32_t nchunks,
                                                                 int32_t q_smem, double* __restrict__ part) {
  extern __shared__ double sq[];  // the query (d doubles, when it fits) + kRedoWarps * (32 / G) group sums
  constexpr int R = 32 / G;
  double* sgrp = sq + (q_smem ? d : 0);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int grp = lane / G, gl = lane % G;
  const int64_t items = int64_t(*count) * nchunks;
  const int64_t rows_per_chunk = (n + nchunks - 1) / nchunks;
  for (int64_t item = blockIdx.x; item < items; item += gridDim.x) {
    const int32_t qi = list[item / nchunks];
    const int64_t lo = (item % nchunks) * rows_per_chunk;
    const int64_t hi = min(n, lo + rows_per_chunk);
    const double* qv = Q + size_t(qi) * d;
    __syncthreads();
    if (q_smem) {
      for (int i = threadIdx.x; i < d; i += blockDim.x) sq[i] = qv[i];
      qv = sq;
    }
    __syncthreads();
    double acc = 0.0;
    for (int64_t r0 = lo + warp * R; r0 < hi; r0 += int64_t(kRedoWarps) * R) {  // warp-uniform trip count
      const int64_t r = r0 + grp;
      const bool valid = r < hi;
      double s = 0.0;
      if (valid) {
        const float* x = X + size_t(r) * d;
        for (int i = gl; i < d; i += G) {
          const double df = qv[i] - double(x[i]);
          s = family == DK_LAPLACIAN ? s + fabs(df) : fma(df, df, s);
        }
      }
#pragma unroll
      for (int o = G / 2; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
      if (gl == 0 && valid) acc += family == DK_EXPONENTIAL ? exp(sqrt(s) * c) : exp(s * c);
    }
    if (gl == 0) sgrp[warp * R + grp] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
      double t = 0.0;
      for (int i = 0; i < kRedoWarps * R; ++i) t += sgrp[i];
      part[item] = t;
    }
  }
}

__global__ void redo_reduce_kernel(const double* __restrict__ part, const int32_t* __restrict__ list,
                                   const int32_t* __restrict__ count, int32_t nchunks, double scale,
                                   double* __restrict__ out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= *count) return;
  double t = 0.0;
  for (int c = 0; c < nchunks; ++c) t += part[size_t(i) * nchunks + c];
  out[list[i]] = t * scale;
}

}  // namespace

void launch_guard_tau(const float* qn, int32_t nq_pad, int64_t nq, float xn_max, double delta_rel, double tol,
                      double h, bool gaussian, float* tau, uint32_t* flag, cudaStream_t s) {
  guard_tau_kernel<<<(nq_pad + 255) / 256, 256, 0, s>>>(qn, nq_pad, nq, xn_max, delta_rel, tol, h, gaussian ? 1 : 0,
                                                        tau, flag);
  DK_CHECK_LAUNCH();
}

void launch_guard_flag_raw(const double* Q, const double* mu, int32_t d, int64_t nq, float xn_max, double delta_rel,
                           double lim, uint32_t* flag, cudaStream_t s) {
  guard_flag_raw_kernel<<<unsigned((nq * 32 + 255) / 256), 256, 0, s>>>(Q, mu, d, nq, xn_max, delta_rel, lim, flag);
  DK_CHECK_LAUNCH();
}

void launch_kde_redo(const float* X, int64_t n, int32_t d, const double* Q, int64_t nq, int32_t family, double h,
                     const uint32_t* flag, double under, int32_t* list, int32_t* count, double* part, double scale,
                     double* out, int num_sms, cudaStream_t s) {
  redo_list_kernel<<<1, 1024, 0, s>>>(flag, out, under, nq, list, count);
  DK_CHECK_LAUNCH();
  const double c = family == DK_GAUSSIAN ? -1.0 / (2.0 * h * h) : -1.0 / h;
  const int grid = num_sms * 4;
  const int G = d >= 32 ? 32 : (d > 8 ? 16 : (d > 2 ? 4 : 1));
  const bool q_smem = d <= 16384;  // wider queries are read through L1
  const size_t smem = (size_t(q_smem ? d : 0) + kRedoWarps * 32) * sizeof(double);
  auto run = [&](auto kern) {
    if (smem > 48 * 1024) DK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    kern<<<grid, kRedoThreads, smem, s>>>(X, n, d, Q, family, c, list, count, kRedoChunks, q_smem ? 1 : 0, part);
  };
  if (G == 32) run(redo_eval_kernel<32>);
  else if (G == 16) run(redo_eval_kernel<16>);
  else if (G == 4) run(redo_eval_kernel<4>);
  else run(redo_eval_kernel<1>);
  DK_CHECK_LAUNCH();
  redo_reduce_kernel<<<int((nq + 255) / 256), 256, 0, s>>>(part, list, count, kRedoChunks, scale, out);
  DK_CHECK_LAUNCH();
}

}  // namespace dk
