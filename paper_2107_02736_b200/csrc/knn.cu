// knn.cu — exact brute-force k-NN on top of the tensor-core distance tiles (K2).
//
// Reference: brute_force_knn (ann.py:105-111) -> _query_sqdists (:78-79) ->
// _smallest_k (:82-102): the k smallest fp64 squared distances, ties broken by
// the lower row index, sorted by (d2, idx); NeighborList invariants (:49-67).
//
// Pipeline per query batch (host side in capi.cu):
//   1. TILEMIN sweep over every S-th tile: min approx d2 per 128-column segment.
//      tau_q = K'-th smallest segment minimum is an UPPER bound on the K'-th
//      smallest approx d2 of the whole set (each minimum is a distinct point).
//   2. FILTER sweep: append every (approx d2, col) with approx d2 <= tau_q.
//      Overflowing queries tighten tau to the K'-th of their first `cap`
//      candidates (still a valid bound) and are swept again.
//   3. select_rerank: K' smallest candidates by approx d2 -> exact fp64 direct
//      difference d2 -> sort by (d2, idx) -> top k.  Certificate: with
//      |approx - exact| <= eps, every non-selected point has exact d2 >
//      boundary - eps; the set is proven when D_k < boundary - eps.
//   4. queries whose certificate fails take an exact fp64 full scan.
#include <cfloat>

#include "internal.h"

namespace dk {

namespace {

struct Key128 {
  unsigned long long hi;  // fp64 bits of d2 (>= 0, so bit order == numeric order)
  unsigned long long lo;  // row index
};
__device__ __forceinline__ bool key_less(const Key128& a, const Key128& b) {
  return a.hi < b.hi || (a.hi == b.hi && a.lo < b.lo);
}

__device__ void bitonic_u64(unsigned long long* buf, int B) {
  for (int k = 2; k <= B; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      __syncthreads();
      for (int i = threadIdx.x; i < B; i += blockDim.x) {
        const int ixj = i ^ j;
        if (ixj > i) {
          const bool up = (i & k) == 0;
          const unsigned long long a = buf[i], b = buf[ixj];
          if ((a > b) == up) { buf[i] = b; buf[ixj] = a; }
        }
      }
    }
  }
  __syncthreads();
}

__device__ void bitonic_k128(Key128* buf, int B) {
  for (int k = 2; k <= B; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      __syncthreads();
      for (int i = threadIdx.x; i < B; i += blockDim.x) {
        const int ixj = i ^ j;
        if (ixj > i) {
          const bool up = (i & k) == 0;
          const Key128 a = buf[i], b = buf[ixj];
          if (key_less(b, a) == up) { buf[i] = b; buf[ixj] = a; }
        }
      }
    }
  }
  __syncthreads();
}

__host__ __device__ inline int pow2_ceil(int v) {
  int p = 1;
  while (p < v) p <<= 1;
  return p;
}

// Streaming selection of the Kp smallest u64 keys out of `cnt` keys fetched by `get(i)`.
// buf has B entries (B > Kp, both powers of two); on return buf[0..Kp) is sorted ascending.
template <class Get>
__device__ void stream_topk_u64(unsigned long long* buf, int B, int Kp, int64_t cnt, Get get) {
  for (int i = threadIdx.x; i < Kp; i += blockDim.x) buf[i] = ~0ull;
  const int chunk = B - Kp;
  for (int64_t pos = 0; pos < cnt || pos == 0; pos += chunk) {
    for (int i = threadIdx.x; i < chunk; i += blockDim.x) {
      const int64_t src = pos + i;
      buf[Kp + i] = src < cnt ? get(src) : ~0ull;
    }
    bitonic_u64(buf, B);
    if (cnt == 0) break;
  }
}

// tau_q = K'-th smallest tile-minimum (fp32 bits in the high word, segment id low)
__global__ void tau_from_tmin_kernel(const float* __restrict__ tmin, int32_t nseg, int32_t nq_pad, int64_t nq,
                                     int32_t kprime, int32_t B, float* __restrict__ tau) {
  extern __shared__ unsigned long long sbuf[];
  const int64_t q = blockIdx.x;
  if (q >= nq) return;
  const int Kp = pow2_ceil(kprime);
  stream_topk_u64(sbuf, B, Kp, nseg, [&](int64_t s) {
    float v = tmin[size_t(s) * nq_pad + q];
    v = fmaxf(v, 0.f);  // order-preserving on clamped values; tau only loosens
    return (static_cast<unsigned long long>(__float_as_uint(v)) << 32) | static_cast<unsigned long long>(s);
  });
  if (threadIdx.x == 0) {
    float t = __int_as_float(0x7f800000);
    if (nseg >= kprime) {
      const unsigned long long kk = sbuf[kprime - 1];
      t = __uint_as_float(uint32_t(kk >> 32));
      if (t == 0.f) t = 0.f;
    }
    tau[q] = t;
  }
}

// queries whose candidate list overflowed: tau' = K'-th smallest of the stored `cap` keys
__global__ void tau_from_cand_kernel(const unsigned long long* __restrict__ cand, const uint32_t* __restrict__ cnt,
                                     int32_t cap, int64_t nq, int32_t kprime, int32_t B, float* __restrict__ tau,
                                     int32_t* __restrict__ overflow_list, int32_t* __restrict__ n_overflow) {
  extern __shared__ unsigned long long sbuf[];
  const int64_t q = blockIdx.x;
  if (q >= nq) return;
  if (cnt[q] <= uint32_t(cap)) return;
  const int Kp = pow2_ceil(kprime);
  const unsigned long long* keys = cand + size_t(q) * cap;
  stream_topk_u64(sbuf, B, Kp, cap, [&](int64_t i) { return keys[i]; });
  if (threadIdx.x == 0) {
    tau[q] = __uint_as_float(uint32_t(sbuf[kprime - 1] >> 32));
    const int slot = atomicAdd(n_overflow, 1);
    overflow_list[slot] = int32_t(q);
  }
}

__device__ __forceinline__ double exact_d2_warp(const float* __restrict__ x, const double* __restrict__ q, int d,
                                                int lane) {
  double s = 0.0;
  for (int k = lane; k < d; k += 32) {
    const double t = double(x[k]) - q[k];
    s = fma(t, t, s);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  return s;
}

// K' smallest candidates by approx key -> exact fp64 re-rank -> top k + certificate
__global__ void select_rerank_kernel(const float* __restrict__ X, int64_t global_offset, int32_t d,
                                     const double* __restrict__ Q, int64_t nq, int32_t k, int32_t kprime,
                                     const unsigned long long* __restrict__ cand, const uint32_t* __restrict__ cnt,
                                     int32_t cap, const float* __restrict__ tau, const float* __restrict__ qn,
                                     float xn_max, float eps_rel, int32_t B, int64_t* __restrict__ idx_out,
                                     double* __restrict__ d2_out, int32_t* __restrict__ status) {
  extern __shared__ unsigned long long sbuf[];
  const int64_t q = blockIdx.x;
  if (q >= nq) return;
  const int Kp = pow2_ceil(kprime);
  const int64_t c = min(int64_t(cnt[q]), int64_t(cap));
  const unsigned long long* keys = cand + size_t(q) * cap;
  stream_topk_u64(sbuf, B, Kp, c, [&](int64_t i) { return keys[i]; });
  // exact re-rank of the first T entries
  const int T = int(min(c, int64_t(kprime)));
  Key128* ex = reinterpret_cast<Key128*>(sbuf + B);  // [Kp]
  const double* qv = Q + size_t(q) * d;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nwarps = blockDim.x >> 5;
  for (int i = warp; i < Kp; i += nwarps) {
    Key128 key{~0ull, ~0ull};
    if (i < T) {
      const unsigned long long col = sbuf[i] & 0xffffffffull;
      const double dd = exact_d2_warp(X + size_t(col) * d, qv, d, lane);
      key.hi = static_cast<unsigned long long>(__double_as_longlong(dd));
      key.lo = col;
    }
    if (lane == 0) ex[i] = key;
  }
  bitonic_k128(ex, Kp);
  if (threadIdx.x == 0) {
    int ok = 1;
    if (T < k) {
      ok = 0;
    } else {
      const double Dk = __longlong_as_double(static_cast<long long>(ex[k - 1].hi));
      const double eps = double(eps_rel) * (double(qn[q]) + double(xn_max)) + 1e-30;
      if (c > kprime) {
        const double a = double(__uint_as_float(uint32_t(sbuf[kprime - 1] >> 32)));
        ok = Dk < a - eps;
      } else {
        const double t = double(tau[q]);
        ok = isinf(t) ? 1 : (Dk <= t - eps);
      }
    }
    status[q] = ok ? 0 : 1;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < k; i += blockDim.x) {
    const Key128 key = ex[i];
    idx_out[size_t(q) * k + i] = key.lo == ~0ull ? -1 : int64_t(key.lo) + global_offset;
    d2_out[size_t(q) * k + i] = __longlong_as_double(static_cast<long long>(key.hi));
  }
}

// exact fp64 full scan for queries whose certificate failed (rare / degenerate inputs)
__global__ void exact_knn_kernel(const float* __restrict__ X, int64_t n, int64_t global_offset, int32_t d,
                                 const double* __restrict__ Q, const int32_t* __restrict__ qlist, int32_t k,
                                 int32_t B, int64_t* __restrict__ idx_out, double* __restrict__ d2_out) {
  extern __shared__ unsigned long long sbuf[];
  Key128* buf = reinterpret_cast<Key128*>(sbuf);
  const int q = qlist[blockIdx.x];
  const int Kp = pow2_ceil(k);
  const double* qv = Q + size_t(q) * d;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nwarps = blockDim.x >> 5;
  for (int i = threadIdx.x; i < Kp; i += blockDim.x) buf[i] = Key128{~0ull, ~0ull};
  const int chunk = B - Kp;
  for (int64_t pos = 0; pos < n; pos += chunk) {
    for (int i = warp; i < chunk; i += nwarps) {
      Key128 key{~0ull, ~0ull};
      const int64_t col = pos + i;
      if (col < n) {
        const double dd = exact_d2_warp(X + size_t(col) * d, qv, d, lane);
        key.hi = static_cast<unsigned long long>(__double_as_longlong(dd));
        key.lo = static_cast<unsigned long long>(col);
      }
      if (lane == 0) buf[Kp + i] = key;
    }
    bitonic_k128(buf, B);
  }
  for (int i = threadIdx.x; i < k; i += blockDim.x) {
    idx_out[size_t(q) * k + i] = int64_t(buf[i].lo) + global_offset;
    d2_out[size_t(q) * k + i] = __longlong_as_double(static_cast<long long>(buf[i].hi));
  }
}

// merge `parts` sorted (d2, idx) lists per query -> global top k (dataset-sharded mode)
__global__ void merge_topk_kernel(int32_t parts, int64_t nq, int32_t k, const int64_t* __restrict__ idx_in,
                                  const double* __restrict__ d2_in, int64_t* __restrict__ idx_out,
                                  double* __restrict__ d2_out) {
  const int64_t q = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (q >= nq) return;
  int head[64];
  for (int p = 0; p < parts; ++p) head[p] = 0;
  for (int i = 0; i < k; ++i) {
    int best = -1;
    double bd = 0;
    int64_t bi = 0;
    for (int p = 0; p < parts; ++p) {
      if (head[p] >= k) continue;
      const size_t off = (size_t(p) * nq + q) * k + head[p];
      const double dd = d2_in[off];
      const int64_t ii = idx_in[off];
      if (ii < 0) continue;
      if (best < 0 || dd < bd || (dd == bd && ii < bi)) { best = p; bd = dd; bi = ii; }
    }
    if (best < 0) { idx_out[q * k + i] = -1; d2_out[q * k + i] = __longlong_as_double(0x7ff0000000000000ll); continue; }
    ++head[best];
    idx_out[q * k + i] = bi;
    d2_out[q * k + i] = bd;
  }
}

__global__ void fill_float_kernel(float* p, int64_t count, float v) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < count) p[i] = v;
}

}  // namespace

static int topk_buffer(int kprime) {
  const int Kp = pow2_ceil(kprime);
  return std::max(2048, 2 * Kp);
}

void launch_fill_float(float* p, int64_t count, float v, cudaStream_t s) {
  if (count <= 0) return;
  fill_float_kernel<<<unsigned((count + 255) / 256), 256, 0, s>>>(p, count, v);
  DK_CHECK_LAUNCH();
}

void launch_tau_from_tmin(const float* tmin, int32_t nseg, int32_t nq_pad, int64_t nq, int32_t kprime, float* tau,
                          cudaStream_t s) {
  const int B = topk_buffer(kprime);
  const size_t smem = size_t(B) * 8;
  static bool attr = false;
  if (!attr) {
    DK_CUDA(cudaFuncSetAttribute(tau_from_tmin_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 232448));
    attr = true;
  }
  tau_from_tmin_kernel<<<unsigned(nq), 256, smem, s>>>(tmin, nseg, nq_pad, nq, kprime, B, tau);
  DK_CHECK_LAUNCH();
}

void launch_tau_from_cand(const unsigned long long* cand, const uint32_t* cand_cnt, int32_t cap, int64_t nq,
                          int32_t kprime, float* tau, int32_t* overflow_list, int32_t* n_overflow, cudaStream_t s) {
  const int B = topk_buffer(kprime);
  static bool attr = false;
  if (!attr) {
    DK_CUDA(cudaFuncSetAttribute(tau_from_cand_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 232448));
    attr = true;
  }
  tau_from_cand_kernel<<<unsigned(nq), 256, size_t(B) * 8, s>>>(cand, cand_cnt, cap, nq, kprime, B, tau,
                                                                overflow_list, n_overflow);
  DK_CHECK_LAUNCH();
}

void launch_select_rerank(const float* X, int64_t global_offset, int32_t d, const double* Q, int64_t nq, int32_t k,
                          int32_t kprime, const unsigned long long* cand, const uint32_t* cand_cnt, int32_t cap,
                          const float* tau, const float* qn, float xn_max, float eps_rel, int64_t* idx_out,
                          double* d2_out, int32_t* status, cudaStream_t s) {
  const int B = topk_buffer(kprime);
  const int Kp = pow2_ceil(kprime);
  const size_t smem = size_t(B) * 8 + size_t(Kp) * sizeof(Key128);
  static bool attr = false;
  if (!attr) {
    DK_CUDA(cudaFuncSetAttribute(select_rerank_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 232448));
    attr = true;
  }
  if (smem > 232448) throw Error{DK_EINVAL, "k too large for the k-NN selection buffer"};
  select_rerank_kernel<<<unsigned(nq), 256, smem, s>>>(X, global_offset, d, Q, nq, k, kprime, cand, cand_cnt, cap,
                                                       tau, qn, xn_max, eps_rel, B, idx_out, d2_out, status);
  DK_CHECK_LAUNCH();
}

void launch_exact_knn_fallback(const float* X, int64_t n_local, int64_t global_offset, int32_t d, const double* Q,
                               const int32_t* qlist, int32_t nlist, int32_t k, int64_t* idx_out, double* d2_out,
                               cudaStream_t s) {
  if (nlist <= 0) return;
  const int Kp = pow2_ceil(k);
  const int B = std::max(1024, 2 * Kp);
  const size_t smem = size_t(B) * sizeof(Key128);
  static bool attr = false;
  if (!attr) {
    DK_CUDA(cudaFuncSetAttribute(exact_knn_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 232448));
    attr = true;
  }
  if (smem > 232448) throw Error{DK_EINVAL, "k too large for the exact k-NN fallback"};
  exact_knn_kernel<<<unsigned(nlist), 256, smem, s>>>(X, n_local, global_offset, d, Q, qlist, k, B, idx_out, d2_out);
  DK_CHECK_LAUNCH();
}

void launch_merge_topk(int32_t parts, int64_t nq, int32_t k, const int64_t* idx_in, const double* d2_in,
                       int64_t* idx_out, double* d2_out, cudaStream_t s) {
  if (parts > 64) throw Error{DK_EINVAL, "dk_merge_topk supports at most 64 parts"};
  merge_topk_kernel<<<unsigned((nq + 127) / 128), 128, 0, s>>>(parts, nq, k, idx_in, d2_in, idx_out, d2_out);
  DK_CHECK_LAUNCH();
}

}  // namespace dk
