// prep.cu — operand preparation ("fit" and per-batch query encoding).
//
// Reference: Dataset.from_array (data.py:53-67) validates finiteness and
// caches fp64 squared norms; batch_sqdist (distance.py:69-85) computes query
// norms per call.  Here the same quantities feed the tensor-core tile:
//   exact  : fp16 copies of small-integer rows (bit-exact products, fp32 sums
//            exact below 2^24)  -> Kp = roundup(d, 64)
//   split3 : centred, power-of-two scaled fp16 hi/lo pairs, K-concatenated
//            A=[Qh|Ql|Qh], B=[Xl|Xh|Xh] so one MMA chain with K = 3d gives
//            Qh.Xl + Ql.Xh + Qh.Xh (~2^-22 relative)     -> Kp = roundup(3d, 64)
//   fp16   : single-pass scaled fp16 (k-NN sweeps, the two-precision KDE's
//            every-pair pass)                              -> Kp = roundup(d + 6, 64)
// The exact and fp16 operands carry kAugCols = 6 norm columns after the d data columns:
//   rows    B = [x | -b1 -b2 -b3 | w1 w2 w3],  queries A = [q | w1 w2 w3 | -b1 -b2 -b3]
// with w1 b1 + w2 b2 + w3 b3 = |v|^2 / 2 (scaled), so the MMA itself accumulates
//   q.x - (|q|^2 + |x|^2) / 2 = -d2 / 2
// and the KDE epilogue needs one multiply per pair (no norm loads, no cancellation in fp32
// outside the accumulator).  k-NN query operands leave the A norm columns zero (plain q.x).
#include "internal.h"

namespace dk {

namespace {

constexpr uint32_t FLAG_NONFINITE = 1u;
constexpr uint32_t FLAG_NONINT = 2u;      // value not an integer or |v| > 2048
constexpr uint32_t FLAG_BIGNORM = 4u;     // squared norm >= 2^23

__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ uint32_t warp_or(uint32_t v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v |= __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ uint32_t value_flags(double v) {
  uint32_t f = 0;
  if (!isfinite(v)) f |= FLAG_NONFINITE;
  if (!(fabs(v) <= 2048.0) || rint(v) != v) f |= FLAG_NONINT;
  return f;
}

// one warp per row: fp64 squared norm, finiteness and integrality flags
__global__ void row_stats_kernel(const float* __restrict__ X, int64_t n, int32_t d, double* __restrict__ xn64,
                                 uint32_t* __restrict__ flags) {
  const int64_t row = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (row >= n) return;
  const float* x = X + row * d;
  double s = 0.0;
  uint32_t f = 0;
  for (int k = lane; k < d; k += 32) {
    const double v = x[k];
    s = fma(v, v, s);
    f |= value_flags(v);
  }
  s = warp_sum_d(s);
  f = warp_or(f);
  if (lane == 0) {
    xn64[row] = s;
    if (!(s < 8388608.0)) f |= FLAG_BIGNORM;
    if (f) atomicOr(flags, f);
  }
}

// column sums over row blocks (deterministic two-level reduction)
__global__ void column_partial_kernel(const float* __restrict__ X, int64_t n, int32_t d, int32_t row_blocks,
                                      double* __restrict__ partial) {
  const int rb = blockIdx.y;
  const int64_t rows_per = (n + row_blocks - 1) / row_blocks;
  const int64_t r0 = rb * rows_per, r1 = min(n, r0 + rows_per);
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < d; k += gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int64_t r = r0; r < r1; ++r) s += X[r * d + k];
    partial[size_t(rb) * d + k] = s;
  }
}
__global__ void column_final_kernel(const double* __restrict__ partial, int32_t row_blocks, int32_t d, int64_t n,
                                    double* __restrict__ mu) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= d) return;
  double s = 0.0;
  for (int rb = 0; rb < row_blocks; ++rb) s += partial[size_t(rb) * d + k];
  mu[k] = s / double(n);
}

// max |x - mu| over all entries (float bits; values are >= 0 so uint order = float order)
template <class T>
__global__ void maxabs_kernel(const T* __restrict__ V, int64_t rows, int32_t d, const double* __restrict__ mu,
                              uint32_t* __restrict__ maxabs_bits) {
  float m = 0.f;
  const int64_t total = rows * d;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < total; i += int64_t(gridDim.x) * blockDim.x) {
    double v = double(V[i]);
    if (mu) v -= mu[i % d];
    m = fmaxf(m, float(fabs(v)));
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) atomicMax(maxabs_bits, __float_as_uint(m));
}

__device__ __forceinline__ float pow2_scale(uint32_t maxabs_bits) {
  const float m = __uint_as_float(maxabs_bits);
  if (!(m > 0.f)) return 1.f;
  int e;
  frexpf(m, &e);                       // m < 2^e
  int sh = 8 - e;                      // scaled max in [2^7, 2^8): scaled |v|^2 / 2 fits w1 b1 (aug columns)
  sh = max(-100, min(100, sh));
  return ldexpf(1.f, sh);
}

// one warp per row: writes the operand row (Kp halves) and the fp32 norm;
// aug: 0 = norm columns zero (k-NN queries), 1 = row side [-b | w], 2 = query side [w | -b]
template <class T>
__global__ void encode_kernel(const T* __restrict__ V, int64_t rows, int64_t rows_pad, int32_t d, int mode,
                              const double* __restrict__ mu, int32_t Kp, const uint32_t* __restrict__ maxabs_bits,
                              const float* __restrict__ other_scale, __half* __restrict__ out,
                              float* __restrict__ norms, float* __restrict__ scale_out,
                              float* __restrict__ m2s_out, uint32_t* __restrict__ check_flags, int aug,
                              __half* __restrict__ tail) {
  const int64_t row = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  // queries with norm columns share the dataset's scale (the norm terms must carry one scale)
  const float s = (mode == 0) ? 1.f : (aug == 2 && other_scale ? *other_scale : pow2_scale(*maxabs_bits));
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    if (scale_out) *scale_out = s;
    if (m2s_out) *m2s_out = -2.f / (s * (other_scale ? *other_scale : 1.f));
  }
  if (row >= rows_pad) return;
  __half* o = out + row * Kp;
  if (row >= rows) {
    for (int k = lane; k < Kp; k += 32) o[k] = __float2half_rn(0.f);
    if (tail && lane < kTailK) tail[row * kTailK + lane] = __float2half_rn(0.f);
    if (lane == 0) norms[row] = 0.f;
    return;
  }
  const T* v = V + row * d;
  double nrm = 0.0;
  uint32_t f = 0;  // exact-mode eligibility of this row (query_check_kernel's flags), mode 0 only
  for (int k = lane; k < Kp; k += 32) {
    if (mode == 1) {
      // K-concatenation A=[Qh|Ql|Qh], B=[Xl|Xh|Xh]: the two small cross terms are accumulated
      // first and the large hi*hi term last, so the fp32 accumulator spends the fewest MMA
      // steps at full magnitude (its rounding error grows with steps x |S|)
      const int blk = k / d;
      const int kk = k - blk * d;
      if (blk >= 3) { o[k] = __float2half_rn(0.f); continue; }
      double x = double(v[kk]);
      if (mu) x -= mu[kk];
      if (blk == 0) nrm = fma(x, x, nrm);
      const double xs = x * double(s);
      const __half h = __float2half_rn(float(xs));
      const __half l = __float2half_rn(float(xs - double(__half2float(h))));
      const bool is_query = (other_scale != nullptr);
      __half w;
      if (blk == 0) w = is_query ? h : l;
      else if (blk == 1) w = is_query ? l : h;
      else w = h;
      o[k] = w;
    } else {
      if (k >= d) {
        if (aug == 0 || tail || k >= d + kAugCols) o[k] = __float2half_rn(0.f);  // norm columns: below
        continue;
      }
      double x = double(v[k]);
      if (check_flags) f |= value_flags(x);
      if (mu) x -= mu[k];
      nrm = fma(x, x, nrm);
      o[k] = __float2half_rn(float(x * double(s)));
    }
  }
  nrm = warp_sum_d(nrm);
  if (lane == 0) norms[row] = float(nrm);
  if (tail && lane >= kAugCols && lane < kTailK) tail[row * kTailK + lane] = __float2half_rn(0.f);
  if (mode != 1 && aug != 0 && lane < kAugCols) {
    // |v|^2 / 2 (scaled) = w1 b1 + w2 b2 + w3 b3.  Exact integers: b from floor divisions (xn <
    // 2^23: b1 < 2^11, b2 < 64, b3 < 32 half-integers, all exact in fp16).  Scaled fp16: each b the
    // fp16 rounding of the remainder (residual <= 2^-33 relative); a query norm beyond the range
    // (v >= 2^31, or inf) poisons its row with NaN (the two-precision KDE then recomputes it).
    double w[3], b[3];
    bool bad = false;
    if (mode == 0) {
      w[0] = 2048.0; w[1] = 32.0; w[2] = 1.0;
      b[0] = floor(nrm / 4096.0);
      const double rem = nrm - b[0] * 4096.0;
      b[1] = floor(rem / 64.0);
      b[2] = (rem - b[1] * 64.0) * 0.5;
    } else {
      w[0] = 32768.0; w[1] = 32.0; w[2] = 1.0;
      const double v = nrm * double(s) * double(s) * 0.5;
      bad = !(v < 2147483648.0);
      b[0] = double(__half2float(__float2half_rn(float(v / 32768.0))));
      double r = v - b[0] * 32768.0;
      b[1] = double(__half2float(__float2half_rn(float(r / 32.0))));
      r -= b[1] * 32.0;
      b[2] = double(__half2float(__float2half_rn(float(r))));
    }
    float val;
    if (aug == 1) val = lane < 3 ? float(-b[lane]) : float(w[lane - 3]);
    else val = lane < 3 ? float(w[lane]) : float(-b[lane - 3]);
    if (bad && aug == 2 && lane == 3) val = __int_as_float(0x7fc00000);
    if (tail) tail[row * kTailK + lane] = __float2half_rn(val);
    else o[d + lane] = __float2half_rn(val);
  }
  if (check_flags) {
    f = warp_or(f);
    if (lane == 0) {
      if (!(nrm < 8388608.0)) f |= FLAG_BIGNORM;
      if (f) atomicOr(check_flags, f);
    }
  }
}

// queries: finiteness / integrality (exact-mode eligibility)
__global__ void query_check_kernel(const double* __restrict__ Q, int64_t nq, int32_t d, uint32_t* __restrict__ flags) {
  const int64_t row = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (row >= nq) return;
  const double* q = Q + row * d;
  double s = 0.0;
  uint32_t f = 0;
  for (int k = lane; k < d; k += 32) {
    const double v = q[k];
    s = fma(v, v, s);
    f |= value_flags(v);
  }
  s = warp_sum_d(s);
  f = warp_or(f);
  if (lane == 0) {
    if (!(s < 8388608.0)) f |= FLAG_BIGNORM;
    if (f) atomicOr(flags, f);
  }
}

// out[q] = scale * sum_j part[j][q].  Block = 32 queries x 8 warps: warp w sums parts
// j = w, w+8, ... sequentially (coalesced over q), then the 8 warp sums are added in
// warp order — a fixed summation tree, so the result is deterministic.
__global__ void __launch_bounds__(256) reduce_partials_kernel(const double* __restrict__ part, int32_t nparts,
                                                              int32_t nq_pad, int64_t nq, double scale,
                                                              double* __restrict__ out) {
  __shared__ double red[8][33];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t q = int64_t(blockIdx.x) * 32 + lane;
  double s = 0.0;
  if (q < nq) {
    int j = w;
    for (; j + 24 < nparts; j += 32) {  // 4 loads in flight per thread
      const double v0 = part[size_t(j) * nq_pad + q], v1 = part[size_t(j + 8) * nq_pad + q];
      const double v2 = part[size_t(j + 16) * nq_pad + q], v3 = part[size_t(j + 24) * nq_pad + q];
      s += v0;
      s += v1;
      s += v2;
      s += v3;
    }
    for (; j < nparts; j += 8) s += part[size_t(j) * nq_pad + q];
  }
  red[w][lane] = s;
  __syncthreads();
  if (w == 0 && q < nq) {
    double t = red[0][lane];
#pragma unroll
    for (int i = 1; i < 8; ++i) t += red[i][lane];
    out[q] = t * scale;
  }
}

}  // namespace

void launch_row_stats(const float* X, int64_t n, int32_t d, double* xn64, uint32_t* flags, cudaStream_t s) {
  const int64_t threads = n * 32;
  row_stats_kernel<<<unsigned((threads + 255) / 256), 256, 0, s>>>(X, n, d, xn64, flags);
  DK_CHECK_LAUNCH();
}


void launch_column_mean(const float* X, int64_t n, int32_t d, double* partial, int32_t row_blocks, double* mu,
                        cudaStream_t s) {
  dim3 g(unsigned((d + 127) / 128), unsigned(row_blocks));
  column_partial_kernel<<<g, 128, 0, s>>>(X, n, d, row_blocks, partial);
  DK_CHECK_LAUNCH();
  column_final_kernel<<<unsigned((d + 127) / 128), 128, 0, s>>>(partial, row_blocks, d, n, mu);
  DK_CHECK_LAUNCH();
}

void launch_encode_rows(const float* X, int64_t n, int64_t n_pad, int32_t d, int mode, const double* mu, int32_t Kp,
                        __half* B, float* xn, float* scale, uint32_t* maxabs_bits, cudaStream_t s, __half* tail) {
  DK_CUDA(cudaMemsetAsync(maxabs_bits, 0, sizeof(uint32_t), s));
  if (mode != 0) {
    maxabs_kernel<float><<<1184, 256, 0, s>>>(X, n, d, mu, maxabs_bits);
    DK_CHECK_LAUNCH();
  }
  // norm columns: in the main operand when they fit its padding, else in the tail (if given)
  const bool in_main = enc_aug_main(d, mode);
  if (in_main) tail = nullptr;
  const bool row_aug = in_main || (enc_aug_tail(d, mode) && tail != nullptr);
  const int64_t threads = n_pad * 32;
  encode_kernel<float><<<unsigned((threads + 255) / 256), 256, 0, s>>>(X, n, n_pad, d, mode, mu, Kp, maxabs_bits,
                                                                      nullptr, B, xn, scale, nullptr, nullptr,
                                                                      row_aug ? 1 : 0, tail);
  DK_CHECK_LAUNCH();
}

void launch_query_check(const double* Q, int64_t nq, int32_t d, uint32_t* flags, cudaStream_t s) {
  const int64_t threads = nq * 32;
  query_check_kernel<<<unsigned((threads + 255) / 256), 256, 0, s>>>(Q, nq, d, flags);
  DK_CHECK_LAUNCH();
}

void launch_encode_queries(const double* Q, int64_t nq, int32_t nq_pad, int32_t d, int mode, const double* mu,
                           int32_t Kp, const float* sx, __half* A, float* qn, float* m2s, uint32_t* maxabs_bits,
                           cudaStream_t s, uint32_t* check_flags, bool aug, __half* tail) {
  const bool q_aug = aug && (enc_aug_main(d, mode) || (enc_aug_tail(d, mode) && tail != nullptr));
  tail = (q_aug && !enc_aug_main(d, mode)) ? tail : nullptr;
  // fp16 queries with norm columns take the dataset's scale: no maximum to find
  if (mode != 0 && !(mode == 2 && q_aug)) {
    DK_CUDA(cudaMemsetAsync(maxabs_bits, 0, sizeof(uint32_t), s));
    const int64_t total = nq * d;
    const unsigned blocks = unsigned(std::min<int64_t>(1184, (total + 255) / 256 + 1));
    maxabs_kernel<double><<<blocks, 256, 0, s>>>(Q, nq, d, mu, maxabs_bits);
    DK_CHECK_LAUNCH();
  }
  const int64_t threads = int64_t(nq_pad) * 32;
  encode_kernel<double><<<unsigned((threads + 255) / 256), 256, 0, s>>>(
      Q, nq, nq_pad, d, mode, mu, Kp, maxabs_bits, sx, A, qn, nullptr, m2s, mode == 0 ? check_flags : nullptr,
      q_aug ? 2 : 0, tail);
  DK_CHECK_LAUNCH();
}

void launch_reduce_partials(const double* part, int32_t nparts, int32_t nq_pad, int64_t nq, double scale, double* out,
                            cudaStream_t s) {
  reduce_partials_kernel<<<unsigned((nq + 31) / 32), 256, 0, s>>>(part, nparts, nq_pad, nq, scale, out);
  DK_CHECK_LAUNCH();
}

}  // namespace dk
