// knn.cu — exact brute-force k-NN on top of the tensor-core distance tiles (K2).
//
// Reference: brute_force_knn (ann.py:105-111) -> _query_sqdists (:78-79) ->
// _smallest_k (:82-102): the k smallest fp64 squared distances, ties broken by
// the lower row index, sorted by (d2, idx); NeighborList invariants (:49-67).
//
// Pipeline per query batch (host side in capi.cu).  Distances are computed on
// the tensor-core tile from an operand encoding whose error is bounded:
// |d2_approx - d2| <= eps_q = eps_rel * (|q|^2 + max|x|^2) (eps_rel = 0 for the
// exact integer encoding, ~1e-3 for single-pass fp16).
//   1. TILEMIN sweep: min approx d2 per segment of `seg_tiles` tiles (atomicMin).
//      The k-th smallest segment minimum t_q is >= the k-th smallest approx d2
//      (segments hold distinct points), so tau_q = t_q + 2 eps_q bounds the
//      approx d2 of every point whose EXACT d2 is <= the exact k-th distance.
//   2. FILTER sweep: keep every (approx d2, col) with approx d2 <= tau_q.  The
//      candidate set provably contains all points at or inside the exact k-th
//      distance, including every tie there.
//   3. select_fast: a histogram of the approx keys locates the k-th; the few
//      candidates within 2 eps_q of it are re-ranked exactly (fp64 direct
//      difference) and sorted by (d2, idx).  Queries with too many near-ties
//      go to select_slow (sorted rounds with early termination) through a
//      device-side list.
//   4. queries whose candidate list overflowed take an exact fp64 full scan
//      (device-side list again: the host never waits on the selection).
#include <cfloat>
#include <climits>
#include <cstdlib>

#include <cub/device/device_radix_sort.cuh>

#include "internal.h"
#include "tile_kernel.cuh"

namespace dk {

namespace {

constexpr int kSelHist = 1024;  // histogram bins of the k-NN selection (4 per thread of a 256-thread block)
// lanes per exactly re-ranked row, the same in every selection path for a given d (one summation
// order, so a query's distances are bit-identical whichever path serves it): 4 lanes (8 rows per
// warp step, 6-7 float4 loads per lane in flight) for rows up to 160 dimensions — faster than 8 on
// c3 (k-NN 1.65 -> 1.58 ms) and 16 (1.67 ms) — and 8 (the round-1 choice) for wider rows
inline int exact_group(int32_t d) { return d <= 160 ? 4 : 8; }

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

// tau_q = k-th smallest segment minimum + 2 eps_q
__global__ void tau_from_tmin_kernel(const float* __restrict__ tmin, int32_t nseg, int32_t nq_pad, int64_t nq,
                                     int32_t k, int32_t B, const float* __restrict__ qn, float xn_max,
                                     float eps_rel, float* __restrict__ tau) {
  extern __shared__ unsigned long long sbuf[];
  const int64_t q = blockIdx.x;
  if (q >= nq) return;
  for (int i = threadIdx.x; i < B; i += blockDim.x) {
    unsigned long long key = ~0ull;
    if (i < nseg) {
      const float v = fmaxf(tmin[size_t(i) * nq_pad + q], 0.f);
      key = (static_cast<unsigned long long>(__float_as_uint(v)) << 32) | static_cast<unsigned long long>(i);
    }
    sbuf[i] = key;
  }
  bitonic_u64(sbuf, B);
  if (threadIdx.x == 0) {
    float t = __int_as_float(0x7f800000);
    if (nseg >= k) {
      const float v = __uint_as_float(uint32_t(sbuf[k - 1] >> 32));
      const float eps = eps_rel * (qn[q] + xn_max);
      t = v + 2.f * eps;
      t = __fmul_ru(t, 1.0f + 2.4e-7f);  // absorb the rounding of the addition itself
    }
    tau[q] = t;
  }
}

// Same tau by a 4-pass 8-bit radix select of the k-th smallest segment minimum (the
// minima are >= 0, so their float bits order like the values): no sort of all segments.
__global__ void __launch_bounds__(256) tau_radix_kernel(const float* __restrict__ tmin, int32_t nseg, int32_t nq_pad,
                                                        int64_t nq, int32_t k, const float* __restrict__ qn,
                                                        float xn_max, float eps_rel, float* __restrict__ tau,
                                                        const int32_t* __restrict__ block_entries, int32_t segs_per,
                                                        float* __restrict__ hlo, float* __restrict__ hinv,
                                                        float* __restrict__ htop) {
  extern __shared__ uint32_t vals[];
  __shared__ uint32_t hist[256];
  __shared__ uint32_t s_digit, s_below, s_min;
  const int64_t q = blockIdx.x;
  if (q >= nq) return;
  // listed sweeps: only the segments of this query block's list were written
  if (block_entries != nullptr) nseg = min(nseg, block_entries[q / 128] * segs_per);
  if (hlo != nullptr && nseg < k) {  // no bound from these segments: no histogram refinement either
    if (threadIdx.x == 0) {
      tau[q] = __int_as_float(0x7f800000);
      hlo[q] = 0.f;
      hinv[q] = 0.f;
      htop[q] = __int_as_float(0xff800000);  // -inf: nothing is counted
    }
    return;
  }
  if (nseg < k) {
    if (threadIdx.x == 0) tau[q] = __int_as_float(0x7f800000);
    return;
  }
  if (threadIdx.x == 0) s_min = 0xffffffffu;
  __syncthreads();
  uint32_t vmin = 0xffffffffu;
  for (int i = threadIdx.x; i < nseg; i += blockDim.x) {
    vals[i] = __float_as_uint(fmaxf(tmin[size_t(i) * nq_pad + q], 0.f));
    vmin = min(vmin, vals[i]);
  }
  if (hlo != nullptr) atomicMin(&s_min, vmin);
  const int lane = threadIdx.x & 31;
  uint32_t prefix = 0u, mask = 0u, krem = uint32_t(k);
  for (int shift = 24; shift >= 0; shift -= 8) {
    hist[threadIdx.x] = 0u;
    __syncthreads();
    for (int i = threadIdx.x; i < nseg; i += blockDim.x) {
      const uint32_t v = vals[i];
      if ((v & mask) == prefix) atomicAdd(&hist[(v >> shift) & 255u], 1u);
    }
    __syncthreads();
    if (threadIdx.x < 32) {  // lane l owns bins [8l, 8l + 8)
      uint32_t own = 0;
#pragma unroll
      for (int j = 0; j < 8; ++j) own += hist[8 * lane + j];
      uint32_t incl = own;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += t;
      }
      uint32_t cum = incl - own;
      if (cum < krem && incl >= krem) {
        for (int j = 0; j < 8; ++j) {
          const uint32_t h = hist[8 * lane + j];
          if (cum + h >= krem) { s_digit = uint32_t(8 * lane + j); s_below = cum; break; }
          cum += h;
        }
      }
    }
    __syncthreads();
    prefix |= s_digit << shift;
    mask |= 255u << shift;
    krem -= s_below;
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    const float v = __uint_as_float(prefix);  // the k-th smallest segment minimum
    const float eps = eps_rel * (qn[q] + xn_max);
    float t = v + 2.f * eps;
    t = __fmul_ru(t, 1.0f + 2.4e-7f);  // as tau_from_tmin_kernel
    tau[q] = t;
    if (hlo != nullptr) {  // histogram range for the refinement sweep: [min segment minimum, k-th]
      const float lo = __uint_as_float(s_min);
      hlo[q] = lo;
      htop[q] = v;
      hinv[q] = v > lo ? 1.f / (v - lo) : 0.f;
    }
  }
}

// tau_q from the per-query histogram of approx d2 over [lo_q, top_q] (bin b holds the values
// with floor(64 sqrt((d2 - lo) / (top - lo))) == b): the upper edge of the first bin where the
// cumulative count reaches k bounds the k-th smallest approx d2 (k distinct rows lie at or below
// it); the edge carries a 1e-5 relative slack for the fp32 binning arithmetic.
__global__ void tau_hist_kernel(const uint32_t* __restrict__ hist, const float* __restrict__ hlo,
                                const float* __restrict__ hinv, const float* __restrict__ htop,
                                const float* __restrict__ tau_h, int64_t nq, int32_t k, const float* __restrict__ qn,
                                float xn_max, float eps_rel, float* __restrict__ tau) {
  const int64_t q = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (q >= nq) return;
  float t = tau_h[q];  // the listed segment-minimum bound (+inf when the list had < k segments)
  if (hinv[q] > 0.f) {
    const uint32_t* h = hist + size_t(q) * kHistBins;
    uint32_t cum = 0;
    int b = 0;
    for (; b < kHistBins; ++b) {
      cum += h[b];
      if (cum >= uint32_t(k)) break;
    }
    if (b < kHistBins) {  // (always: the k segment minima themselves are counted)
      const double lo = hlo[q], top = htop[q];
      const double f = double(b + 1) / kHistBins;
      const double edge = lo + (top - lo) * f * f * (1.0 + 1e-5) + 1e-6 * (top - lo);
      const float eps = eps_rel * (qn[q] + xn_max);
      float te = float(fmin(edge, double(top))) + 2.f * eps;
      te = __fmul_ru(te, 1.0f + 2.4e-7f);
      t = fminf(t, te);
    }
  }
  tau[q] = fminf(tau[q], t);  // every bound is valid: keep the tightest
}

// exact fp64 direct-difference d2 by a group of G lanes (float4 row loads when rows are
// whole float4s), reduced within the group
template <int G>
__device__ __forceinline__ double exact_d2_group(const float* __restrict__ x, const double* __restrict__ q, int d,
                                                 int gl) {
  double s = 0.0;
  if ((d & 3) == 0) {
    const float4* x4 = reinterpret_cast<const float4*>(x);
    for (int k4 = gl; k4 < (d >> 2); k4 += G) {
      const float4 v = __ldg(x4 + k4);
      const double t0 = double(v.x) - q[4 * k4 + 0], t1 = double(v.y) - q[4 * k4 + 1];
      const double t2 = double(v.z) - q[4 * k4 + 2], t3 = double(v.w) - q[4 * k4 + 3];
      s = fma(t0, t0, s);
      s = fma(t1, t1, s);
      s = fma(t2, t2, s);
      s = fma(t3, t3, s);
    }
  } else {
    for (int k = gl; k < d; k += G) {
      const double t = double(__ldg(x + k)) - q[k];
      s = fma(t, t, s);
    }
  }
#pragma unroll
  for (int o = G / 2; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  return s;
}

// Selection, fast path (one CTA per query, small shared memory): no sort of the whole
// candidate list.  T' = the largest approx key in the histogram bins up to the one holding
// the k-th smallest approx key (T' >= that key).  The k candidates with approx d2 <= T' have
// exact d2 <= T' + eps, so every member of the exact top k (ties included) has approx
// d2 <= T' + 2 eps: exactly those are evaluated (fp64 direct difference) and sorted by
// (d2, id).  The candidate keys stay in global memory (L2) and are read in four passes.
// Queries this path cannot finish are appended to device lists, so the host never waits:
//   slow list: more than 2 pow2(k) keys within 2 eps of T' -> select_slow_kernel;
//   ovf list : candidate list overflowed (> cap) or shorter than k -> exact fp64 scan.
template <int G>
__global__ void __launch_bounds__(256) select_fast_kernel(
    const float* __restrict__ X, int64_t global_offset, int32_t d, const double* __restrict__ Q, int64_t nq,
    int32_t k, const unsigned long long* __restrict__ cand, const uint32_t* __restrict__ cnt, int32_t cap,
    const float* __restrict__ qn, float xn_max, float eps_rel, int64_t* __restrict__ idx_out,
    double* __restrict__ d2_out, int32_t* __restrict__ slow_list, int32_t* __restrict__ slow_cnt,
    int32_t* __restrict__ ovf_list, int32_t* __restrict__ ovf_cnt, const int64_t* __restrict__ perm, int32_t scap) {
  // candidates are row positions of X; perm (optional) maps a position to the reported row id,
  // which is also the tie-break key (pruned k-NN: X holds the cluster-sorted rows)
  extern __shared__ unsigned long long sraw[];
  const int64_t q = blockIdx.x;
  if (q >= nq) return;
  const uint32_t craw = cnt[q];
  if (craw > uint32_t(cap) || craw < uint32_t(k)) {
    if (threadIdx.x == 0) ovf_list[atomicAdd(ovf_cnt, 1)] = int32_t(q);
    return;
  }
  const int c = int(craw);
  const unsigned long long* keys = cand + size_t(q) * cap;
  Key128* top = reinterpret_cast<Key128*>(sraw);         // [scap]
  double* qv = reinterpret_cast<double*>(top + scap);    // the query in shared memory
  uint32_t* hist = reinterpret_cast<uint32_t*>(qv + d);  // [kSelHist]
  for (int j = threadIdx.x; j < d; j += blockDim.x) qv[j] = Q[size_t(q) * d + j];
  const double eps = double(eps_rel) * (double(qn[q]) + double(xn_max));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nwarps = blockDim.x >> 5;
  const int grp = lane / G, gl = lane % G;
  __shared__ uint32_t s_lo, s_hi, s_bstar, s_tmax, s_ns;
  __shared__ uint32_t s_wsum[32];
  if (threadIdx.x == 0) { s_lo = 0xffffffffu; s_hi = 0u; s_bstar = kSelHist - 1; s_tmax = 0u; s_ns = 0u; }
  for (int i = threadIdx.x; i < kSelHist; i += blockDim.x) hist[i] = 0u;
  __syncthreads();
  uint32_t lo = 0xffffffffu, hi = 0u;
  for (int i = threadIdx.x; i < c; i += blockDim.x) {
    const uint32_t b = uint32_t(__ldg(keys + i) >> 32);  // bits of an approx d2 >= 0: uint order == float order
    lo = min(lo, b);
    hi = max(hi, b);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    lo = min(lo, __shfl_xor_sync(0xffffffffu, lo, o));
    hi = max(hi, __shfl_xor_sync(0xffffffffu, hi, o));
  }
  if (lane == 0) { atomicMin(&s_lo, lo); atomicMax(&s_hi, hi); }
  __syncthreads();
  const float flo = __uint_as_float(s_lo), fhi = __uint_as_float(s_hi);
  const float scale = fhi > flo ? float(kSelHist) / (fhi - flo) : 0.f;
  // monotone bin of a key (NaN from 0 * inf lands in bin 0, i.e. still monotone)
  auto bin_of = [&](uint32_t b) {
    return min(max(__float2int_rz((__uint_as_float(b) - flo) * scale), 0), kSelHist - 1);
  };
  for (int i = threadIdx.x; i < c; i += blockDim.x) atomicAdd(&hist[bin_of(uint32_t(__ldg(keys + i) >> 32))], 1u);
  __syncthreads();
  {  // block scan: thread t owns bins [4t, 4t + 4) (kSelHist = 4 * blockDim)
    const int t = threadIdx.x;
    const uint32_t h0 = hist[4 * t], h1 = hist[4 * t + 1], h2 = hist[4 * t + 2], h3 = hist[4 * t + 3];
    const uint32_t own = h0 + h1 + h2 + h3;
    uint32_t incl = own;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t v = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += v;
    }
    if (lane == 31) s_wsum[warp] = incl;
    __syncthreads();
    uint32_t cum = incl - own;
    for (int w = 0; w < warp; ++w) cum += s_wsum[w];
    const uint32_t hh[4] = {h0, h1, h2, h3};
    const uint32_t kk = uint32_t(k);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      if (cum < kk && cum + hh[j] >= kk) s_bstar = uint32_t(4 * t + j);
      cum += hh[j];
    }
  }
  __syncthreads();
  const int bstar = int(s_bstar);
  uint32_t tm = 0u;
  for (int i = threadIdx.x; i < c; i += blockDim.x) {
    const uint32_t b = uint32_t(__ldg(keys + i) >> 32);
    if (bin_of(b) <= bstar) tm = max(tm, b);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) tm = max(tm, __shfl_xor_sync(0xffffffffu, tm, o));
  if (lane == 0) atomicMax(&s_tmax, tm);
  __syncthreads();
  const double thr = double(__uint_as_float(s_tmax)) + 2.0 * eps;
  for (int i = threadIdx.x; i < c; i += blockDim.x) {
    const unsigned long long v = __ldg(keys + i);
    if (double(__uint_as_float(uint32_t(v >> 32))) <= thr) {
      const uint32_t pos = atomicAdd(&s_ns, 1u);
      if (pos < uint32_t(scap)) top[pos].lo = v & 0xffffffffull;
    }
  }
  __syncthreads();
  const int ns = int(s_ns);
  if (ns > scap) {  // too many keys within 2 eps of the k-th: the sorted-rounds kernel
    if (threadIdx.x == 0) slow_list[atomicAdd(slow_cnt, 1)] = int32_t(q);
    return;
  }
  int P = 2;
  while (P < ns) P <<= 1;
  for (int i0 = warp * (32 / G); i0 < ns; i0 += nwarps * (32 / G)) {
    const int i = i0 + grp;
    const bool ok = i < ns;
    const unsigned long long col = ok ? top[i].lo : 0ull;
    DK_DCHECK(col < (1ull << 40));
    const double dd = exact_d2_group<G>(X + size_t(col) * d, qv, d, gl);
    if (gl == 0 && ok) {
      top[i].hi = static_cast<unsigned long long>(__double_as_longlong(dd));
      if (perm != nullptr) top[i].lo = static_cast<unsigned long long>(perm[col]);
    }
  }
  __syncthreads();
  {
    // Of the ns exactly evaluated keys only the k smallest are output.  A histogram of their
    // exact d2 finds the bin holding the k-th; the keys up to that bin (k plus a few) are ordered
    // by counting ranks (ids are distinct, so ranks are) and the first k write themselves out:
    // O(ns + m^2) work and a handful of barriers instead of sorting all ns keys (round 1: a
    // bitonic network over pow2(ns) keys, ~40 barrier-separated stages; ns is a few hundred on c3).
    if (threadIdx.x == 0) { s_lo = 0xffffffffu; s_hi = 0u; s_bstar = kSelHist - 1; s_ns = 0u; }
    for (int i = threadIdx.x; i < kSelHist; i += blockDim.x) hist[i] = 0u;
    __syncthreads();
    // exact d2 >= 0: the fp32 value rounded up keeps the order of the fp64 keys (monotone binning)
    auto f32_of = [&](unsigned long long hi) { return __double2float_ru(__longlong_as_double(static_cast<long long>(hi))); };
    uint32_t lo2 = 0xffffffffu, hi2 = 0u;
    for (int i = threadIdx.x; i < ns; i += blockDim.x) {
      const uint32_t b = __float_as_uint(f32_of(top[i].hi));
      lo2 = min(lo2, b);
      hi2 = max(hi2, b);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      lo2 = min(lo2, __shfl_xor_sync(0xffffffffu, lo2, o));
      hi2 = max(hi2, __shfl_xor_sync(0xffffffffu, hi2, o));
    }
    if (lane == 0) { atomicMin(&s_lo, lo2); atomicMax(&s_hi, hi2); }
    __syncthreads();
    const float elo = __uint_as_float(s_lo), ehi = __uint_as_float(s_hi);
    const float escale = ehi > elo ? float(kSelHist) / (ehi - elo) : 0.f;
    auto ebin = [&](unsigned long long hi) {
      return min(max(__float2int_rz((f32_of(hi) - elo) * escale), 0), kSelHist - 1);
    };
    for (int i = threadIdx.x; i < ns; i += blockDim.x) atomicAdd(&hist[ebin(top[i].hi)], 1u);
    __syncthreads();
    {
      const int t = threadIdx.x;
      const uint32_t h0 = hist[4 * t], h1 = hist[4 * t + 1], h2 = hist[4 * t + 2], h3 = hist[4 * t + 3];
      const uint32_t own = h0 + h1 + h2 + h3;
      uint32_t incl = own;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t v = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += v;
      }
      if (lane == 31) s_wsum[warp] = incl;
      __syncthreads();
      uint32_t cum = incl - own;
      for (int w = 0; w < warp; ++w) cum += s_wsum[w];
      const uint32_t hh[4] = {h0, h1, h2, h3};
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        if (cum < uint32_t(k) && cum + hh[j] >= uint32_t(k)) s_bstar = uint32_t(4 * t + j);
        cum += hh[j];
      }
    }
    __syncthreads();
    const int eb = int(s_bstar);
    uint16_t* sel = reinterpret_cast<uint16_t*>(hist);  // the bins are no longer needed: [<= 2 kSelHist]
    __syncthreads();
    for (int i = threadIdx.x; i < ns; i += blockDim.x)
      if (ebin(top[i].hi) <= eb) {
        const uint32_t pos = atomicAdd(&s_ns, 1u);
        if (pos < uint32_t(2 * kSelHist)) sel[pos] = uint16_t(i);
      }
    __syncthreads();
    const int m = int(s_ns);
    if (m <= 2 * kSelHist) {
      for (int a = threadIdx.x; a < m; a += blockDim.x) {
        const Key128 ki = top[sel[a]];
        int r = 0;
        for (int b = 0; b < m; ++b) {
          const Key128 kj = top[sel[b]];
          r += (kj.hi < ki.hi) | ((kj.hi == ki.hi) & (kj.lo < ki.lo));
        }
        if (r < k) {
          idx_out[size_t(q) * k + r] = int64_t(ki.lo) + global_offset;
          d2_out[size_t(q) * k + r] = __longlong_as_double(static_cast<long long>(ki.hi));
        }
      }
      return;
    }
    __syncthreads();
  }
  for (int i = ns + threadIdx.x; i < P; i += blockDim.x) top[i] = Key128{~0ull, ~0ull};
  bitonic_k128(top, P);
  for (int i = threadIdx.x; i < k; i += blockDim.x) {
    const Key128 key = top[i];
    idx_out[size_t(q) * k + i] = int64_t(key.lo) + global_offset;
    d2_out[size_t(q) * k + i] = __longlong_as_double(static_cast<long long>(key.hi));
  }
}

// Selection, sorted-rounds path for the queries select_fast_kernel listed (persistent grid
// over the device list): all candidates bitonic-sorted by approx key in shared memory, then
// re-ranked exactly W at a time in that order until the next approx key - eps exceeds the
// current exact k-th distance.
template <int G>
__global__ void __launch_bounds__(256) select_slow_kernel(
    const float* __restrict__ X, int64_t global_offset, int32_t d, const double* __restrict__ Q, int32_t k,
    const unsigned long long* __restrict__ cand, const uint32_t* __restrict__ cnt, int32_t cap,
    const float* __restrict__ qn, float xn_max, float eps_rel, int32_t B, int64_t* __restrict__ idx_out,
    double* __restrict__ d2_out, const int32_t* __restrict__ slow_list, const int32_t* __restrict__ slow_cnt,
    const int64_t* __restrict__ perm) {
  extern __shared__ unsigned long long sbuf[];
  const int nlist = *slow_cnt;
  const int Kp = max(32, pow2_ceil(k));
  const int W = Kp;
  Key128* top = reinterpret_cast<Key128*>(sbuf + B);
  double* qv = reinterpret_cast<double*>(top + Kp + W);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nwarps = blockDim.x >> 5;
  const int grp = lane / G, gl = lane % G;
  __shared__ int s_stop;
  for (int li = blockIdx.x; li < nlist; li += gridDim.x) {
    const int64_t q = slow_list[li];
    DK_DCHECK(q >= 0 && int(cnt[q]) >= k);
    const int c = int(cnt[q]);
    const unsigned long long* keys = cand + size_t(q) * cap;
    __syncthreads();
    for (int j = threadIdx.x; j < d; j += blockDim.x) qv[j] = Q[size_t(q) * d + j];
    const double eps = double(eps_rel) * (double(qn[q]) + double(xn_max));
    int Bc = 2;
    while (Bc < c) Bc <<= 1;
    for (int i = threadIdx.x; i < Bc; i += blockDim.x) sbuf[i] = i < c ? keys[i] : ~0ull;
    bitonic_u64(sbuf, Bc);
    for (int i = threadIdx.x; i < Kp + W; i += blockDim.x) top[i] = Key128{~0ull, ~0ull};
    __syncthreads();
    for (int pos = 0; pos < c; pos += W) {
      for (int i0 = warp * (32 / G); i0 < W; i0 += nwarps * (32 / G)) {
        const int i = i0 + grp;
        const bool ok = i < W && pos + i < c;
        const unsigned long long col = ok ? (sbuf[pos + i] & 0xffffffffull) : 0ull;
        const double dd = exact_d2_group<G>(X + size_t(col) * d, qv, d, gl);
        if (gl == 0 && i < W)
          top[Kp + i] = ok ? Key128{static_cast<unsigned long long>(__double_as_longlong(dd)),
                                    perm != nullptr ? static_cast<unsigned long long>(perm[col]) : col}
                           : Key128{~0ull, ~0ull};
      }
      bitonic_k128(top, Kp + W);
      if (threadIdx.x == 0) {
        int stop = 0;
        if (pos + W < c && top[k - 1].hi != ~0ull) {
          const double Dk = __longlong_as_double(static_cast<long long>(top[k - 1].hi));
          const double next = double(__uint_as_float(uint32_t(sbuf[pos + W] >> 32)));
          stop = (next - eps > Dk) ? 1 : 0;
        }
        s_stop = stop;
      }
      __syncthreads();
      if (s_stop) break;
      __syncthreads();
    }
    for (int i = threadIdx.x; i < k; i += blockDim.x) {
      const Key128 key = top[i];
      idx_out[size_t(q) * k + i] = int64_t(key.lo) + global_offset;
      d2_out[size_t(q) * k + i] = __longlong_as_double(static_cast<long long>(key.hi));
    }
  }
}

// exact fp64 full scan for the queries on the overflow list (rare / degenerate inputs);
// persistent grid over the device list
template <int G>
__global__ void exact_knn_kernel(const float* __restrict__ X, int64_t n, int64_t global_offset, int32_t d,
                                 const double* __restrict__ Q, const int32_t* __restrict__ qlist,
                                 const int32_t* __restrict__ qcount, int32_t k, int32_t B,
                                 int64_t* __restrict__ idx_out, double* __restrict__ d2_out, int32_t nsplit,
                                 int32_t split_max, int64_t* __restrict__ tmp_idx, double* __restrict__ tmp_d2) {
  // Work items: with nsplit > 1 the first split_max listed queries are cut into nsplit row slices each
  // (item = (query, slice), top k of the slice into tmp, merged by exact_merge_kernel), so a handful
  // of overflowed queries use the whole GPU instead of one SM each (c5, 3 queries: 339 -> ~35 ms);
  // listed queries past split_max scan all rows in one item and write their result directly.
  extern __shared__ unsigned long long sbuf[];
  Key128* buf = reinterpret_cast<Key128*>(sbuf);
  const int nlist = *qcount;
  const int Kp = pow2_ceil(k);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nwarps = blockDim.x >> 5;
  const int chunk = B - Kp;
  const int nsq = nsplit > 1 ? min(nlist, split_max) : 0;  // queries served in slices
  const int items = nsq * nsplit + (nlist - nsq);
  const int64_t slice = nsplit > 1 ? (n + nsplit - 1) / nsplit : n;
  for (int item = blockIdx.x; item < items; item += gridDim.x) {
    const bool split = item < nsq * nsplit;
    const int li = split ? item / nsplit : nsq + (item - nsq * nsplit);
    const int part = split ? item % nsplit : 0;
    const int64_t row_lo = split ? part * slice : 0;
    const int64_t row_hi = split ? min(n, row_lo + slice) : n;
    const int q = qlist[li];
    const double* qv = Q + size_t(q) * d;
    __syncthreads();
    for (int i = threadIdx.x; i < Kp; i += blockDim.x) buf[i] = Key128{~0ull, ~0ull};
    __syncthreads();
    for (int64_t pos = row_lo; pos < row_hi; pos += chunk) {
      // G lanes per row (exact_group(d)) with the selection's summation order (exact_d2_group), so a query
      // gets bit-identical distances whichever path served it
      const int grp = lane / G, gl = lane % G;
      const Key128 kth = buf[k - 1];  // the k-th best so far (sorted prefix; all-ones until k rows are in)
      int beats = 0;
      for (int i0 = warp * (32 / G); i0 < chunk; i0 += nwarps * (32 / G)) {
        const int i = i0 + grp;
        const int64_t col = pos + i;
        const bool ok = i < chunk && col < row_hi;
        const double dd = exact_d2_group<G>(X + size_t(ok ? col : 0) * d, qv, d, gl);
        if (gl == 0 && i < chunk) {
          const Key128 key = ok ? Key128{static_cast<unsigned long long>(__double_as_longlong(dd)),
                                         static_cast<unsigned long long>(col)}
                                : Key128{~0ull, ~0ull};
          buf[Kp + i] = key;
          beats |= (key.hi < kth.hi || (key.hi == kth.hi && key.lo < kth.lo)) ? 1 : 0;
        }
      }
      // a chunk with no row ahead of the current k-th leaves the prefix as it is: no sort (after the
      // first few chunks that is nearly every chunk, so the scan costs its distances, not its sorts)
      if (__syncthreads_or(beats)) bitonic_k128(buf, B);
    }
    if (split) {  // the slice's best rows, (d2, local row) ascending; -1 pads a slice with fewer than k rows
      for (int i = threadIdx.x; i < k; i += blockDim.x) {
        const bool have = buf[i].lo != ~0ull;
        tmp_idx[(size_t(li) * nsplit + part) * k + i] = have ? int64_t(buf[i].lo) : -1;
        tmp_d2[(size_t(li) * nsplit + part) * k + i] = __longlong_as_double(static_cast<long long>(buf[i].hi));
      }
    } else {
      for (int i = threadIdx.x; i < k; i += blockDim.x) {
        idx_out[size_t(q) * k + i] = int64_t(buf[i].lo) + global_offset;
        d2_out[size_t(q) * k + i] = __longlong_as_double(static_cast<long long>(buf[i].hi));
      }
    }
  }
}

// merges the nsplit sorted slice lists of each sliced query (one warp per query, lane p = slice p):
// k rounds of the warp-wide smallest (d2, row) head, as merge_topk_kernel
__global__ void __launch_bounds__(256) exact_merge_kernel(const int32_t* __restrict__ qlist,
                                                          const int32_t* __restrict__ qcount, int32_t split_max,
                                                          int32_t nsplit, int32_t k, int64_t global_offset,
                                                          const int64_t* __restrict__ tmp_idx,
                                                          const double* __restrict__ tmp_d2,
                                                          int64_t* __restrict__ idx_out, double* __restrict__ d2_out) {
  const int li = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (li >= min(*qcount, split_max)) return;
  const int q = qlist[li];
  const double kInf = __longlong_as_double(0x7ff0000000000000ll);
  int head = 0;
  long long ci = LLONG_MAX;
  double cd = kInf;
  auto load = [&]() {
    ci = LLONG_MAX;
    cd = kInf;
    if (lane < nsplit && head < k) {
      const long long v = tmp_idx[(size_t(li) * nsplit + lane) * k + head];
      if (v >= 0) {
        ci = v;
        cd = tmp_d2[(size_t(li) * nsplit + lane) * k + head];
      }
    }
  };
  load();
  for (int i = 0; i < k; ++i) {
    double bd = cd;
    long long bi = ci;
    int bl = lane;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double od = __shfl_xor_sync(0xffffffffu, bd, o);
      const long long oi = __shfl_xor_sync(0xffffffffu, bi, o);
      const int ol = __shfl_xor_sync(0xffffffffu, bl, o);
      if (od < bd || (od == bd && (oi < bi || (oi == bi && ol < bl)))) { bd = od; bi = oi; bl = ol; }
    }
    if (lane == 0) {
      idx_out[size_t(q) * k + i] = bi + global_offset;
      d2_out[size_t(q) * k + i] = bd;
    }
    if (lane == bl) {
      ++head;
      load();
    }
  }
}

// merge `parts` sorted (d2, idx) lists per query -> global top k (dataset-sharded mode).
// One warp per query: lane p holds the head of part p (and p + 32), the warp picks the
// smallest (d2, idx) head by shuffles, its owner advances; no per-thread arrays.
__global__ void __launch_bounds__(256) merge_topk_kernel(int32_t parts, int64_t nq, int32_t k,
                                                         const int64_t* __restrict__ idx_in,
                                                         const double* __restrict__ d2_in,
                                                         int64_t* __restrict__ idx_out, double* __restrict__ d2_out) {
  const int64_t q = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (q >= nq) return;
  const double kInf = __longlong_as_double(0x7ff0000000000000ll);
  // two heads per lane (parts lane and lane + 32) in scalar registers
  int h0 = 0, h1 = 0;
  double d0 = kInf, d1 = kInf;
  long long i0 = LLONG_MAX, i1 = LLONG_MAX;
  auto load_i = [&](int p, int head) -> long long {
    if (p >= parts || head >= k) return LLONG_MAX;
    const long long v = idx_in[(size_t(p) * nq + q) * k + head];
    return v >= 0 ? v : LLONG_MAX;
  };
  auto load_d = [&](int p, int head, long long ii) -> double {
    return ii == LLONG_MAX ? kInf : d2_in[(size_t(p) * nq + q) * k + head];
  };
  i0 = load_i(lane, h0);
  d0 = load_d(lane, h0, i0);
  i1 = load_i(lane + 32, h1);
  d1 = load_d(lane + 32, h1, i1);
  for (int i = 0; i < k; ++i) {
    // this lane's best of its two heads, then the warp minimum of (d2, idx)
    const bool second = d1 < d0 || (d1 == d0 && i1 < i0);
    double bd = second ? d1 : d0;
    long long bi = second ? i1 : i0;
    int bl = lane;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double od = __shfl_xor_sync(0xffffffffu, bd, o);
      const long long oi = __shfl_xor_sync(0xffffffffu, bi, o);
      const int ol = __shfl_xor_sync(0xffffffffu, bl, o);
      if (od < bd || (od == bd && (oi < bi || (oi == bi && ol < bl)))) { bd = od; bi = oi; bl = ol; }
    }
    if (lane == 0) {
      idx_out[q * k + i] = bi == LLONG_MAX ? -1 : bi;
      d2_out[q * k + i] = bi == LLONG_MAX ? kInf : bd;
    }
    if (lane == bl && bi != LLONG_MAX) {
      if (second) {
        ++h1;
        i1 = load_i(lane + 32, h1);
        d1 = load_d(lane + 32, h1, i1);
      } else {
        ++h0;
        i0 = load_i(lane, h0);
        d0 = load_d(lane, h0, i0);
      }
    }
  }
}

__global__ void fill_float_kernel(float* p, int64_t count, float v) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < count) p[i] = v;
}

// ---------------------------------------------------------------- pruned k-NN helpers

// dq[j][c] = |q_j - cent_c| in fp64 (direct difference).  Block: 32 queries x 64 clusters,
// d in chunks of 32 through shared memory, 2 queries x 4 clusters per thread.
__global__ void __launch_bounds__(256) query_cluster_dist_kernel(const double* __restrict__ Q, int64_t nq, int32_t d,
                                                                 const double* __restrict__ cent, int32_t C,
                                                                 double* __restrict__ dq) {
  __shared__ double qs[32][33];
  __shared__ double cs[64][33];
  const int64_t q0 = int64_t(blockIdx.x) * 32;
  const int c0 = blockIdx.y * 64;
  const int tq = threadIdx.x >> 4, tc = threadIdx.x & 15;  // queries tq, tq+16; clusters tc + 16 i
  double acc[2][4] = {};
  for (int k0 = 0; k0 < d; k0 += 32) {
    for (int i = threadIdx.x; i < 32 * 32; i += 256) {
      const int r = i >> 5, k = i & 31;
      qs[r][k] = (q0 + r < nq && k0 + k < d) ? Q[(q0 + r) * d + k0 + k] : 0.0;
    }
    for (int i = threadIdx.x; i < 64 * 32; i += 256) {
      const int r = i >> 5, k = i & 31;
      cs[r][k] = (c0 + r < C && k0 + k < d) ? cent[size_t(c0 + r) * d + k0 + k] : 0.0;
    }
    __syncthreads();
#pragma unroll 8
    for (int k = 0; k < 32; ++k) {
      const double a0 = qs[tq][k], a1 = qs[tq + 16][k];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const double b = cs[tc + 16 * i][k];
        const double t0 = a0 - b, t1 = a1 - b;
        acc[0][i] = fma(t0, t0, acc[0][i]);
        acc[1][i] = fma(t1, t1, acc[1][i]);
      }
    }
    __syncthreads();
  }
#pragma unroll
  for (int a = 0; a < 2; ++a) {
    const int64_t q = q0 + tq + 16 * a;
    if (q >= nq) continue;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int c = c0 + tc + 16 * i;
      if (c < C) dq[q * C + c] = sqrt(acc[a][i]);
    }
  }
}

// Nearest ball in fp32 (an ordering heuristic only: the two-precision KDE sorts its batch by it;
// the k-NN's pruning bounds need the fp64 dq above).  Same 32 x 64 tiling; each query's
// (distance bits, ball) minimum over the block's 64 balls, then one 64-bit atomicMin per query
// and tile (deterministic: a minimum).
__global__ void __launch_bounds__(256) nearest_ball_f32_kernel(const double* __restrict__ Q, int64_t nq, int32_t d,
                                                               const double* __restrict__ cent, int32_t C,
                                                               unsigned long long* __restrict__ best) {
  __shared__ float qs[32][33];
  __shared__ float cs[64][33];
  const int64_t q0 = int64_t(blockIdx.x) * 32;
  const int c0 = blockIdx.y * 64;
  const int tq = threadIdx.x >> 4, tc = threadIdx.x & 15;
  float acc[2][4] = {};
  for (int k0 = 0; k0 < d; k0 += 32) {
    for (int i = threadIdx.x; i < 32 * 32; i += 256) {
      const int r = i >> 5, k = i & 31;
      qs[r][k] = (q0 + r < nq && k0 + k < d) ? float(Q[(q0 + r) * d + k0 + k]) : 0.f;
    }
    for (int i = threadIdx.x; i < 64 * 32; i += 256) {
      const int r = i >> 5, k = i & 31;
      cs[r][k] = (c0 + r < C && k0 + k < d) ? float(cent[size_t(c0 + r) * d + k0 + k]) : 0.f;
    }
    __syncthreads();
#pragma unroll 8
    for (int k = 0; k < 32; ++k) {
      const float a0 = qs[tq][k], a1 = qs[tq + 16][k];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const float b = cs[tc + 16 * i][k];
        const float t0 = a0 - b, t1 = a1 - b;
        acc[0][i] = fmaf(t0, t0, acc[0][i]);
        acc[1][i] = fmaf(t1, t1, acc[1][i]);
      }
    }
    __syncthreads();
  }
#pragma unroll
  for (int a = 0; a < 2; ++a) {
    unsigned long long key = ~0ull;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int c = c0 + tc + 16 * i;
      if (c < C) key = min(key, (static_cast<unsigned long long>(__float_as_uint(acc[a][i])) << 32) | uint32_t(c));
    }
#pragma unroll
    for (int o = 8; o > 0; o >>= 1) key = min(key, __shfl_xor_sync(0xffffffffu, key, o));
    const int64_t q = q0 + tq + 16 * a;
    if (tc == 0 && q < nq) atomicMin(best + q, key);
  }
}

__global__ void best_to_ball_kernel(const unsigned long long* __restrict__ best, int64_t nq,
                                    int32_t* __restrict__ nearest) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < nq) nearest[i] = int32_t(best[i] & 0xffffffffull);
}

__global__ void nearest_cluster_kernel(const double* __restrict__ dq, int64_t nq, int32_t C,
                                       int32_t* __restrict__ nearest) {
  const int64_t q = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (q >= nq) return;
  double best = INFINITY;
  int bi = 0;
  for (int c = lane; c < C; c += 32) {
    const double v = dq[q * C + c];
    if (v < best) { best = v; bi = c; }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double ob = __shfl_xor_sync(0xffffffffu, best, o);
    const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
    if (ob < best || (ob == best && oi < bi)) { best = ob; bi = oi; }
  }
  if (lane == 0) nearest[q] = bi;
}

// Tile list of one block of 128 (permuted) queries: cluster c is needed when some query
// of the block can see a row of its ball with approx d2 <= tau_q, i.e. (|q - cent_c| -
// rad_c)^2 <= tau_q + eps_q (approx d2 >= exact d2 - eps_q); a tile is needed when any
// cluster of its range is.  fp64 slack: dq shrunk by 1e-12 relative (rad is inflated at
// build), the threshold grown by 1e-6 relative.
constexpr int kListThreads = 1024;  // block_tile_lists: 32 warps, 4 rows each
__global__ void __launch_bounds__(kListThreads) block_tile_lists_kernel(
    const double* __restrict__ dq, int32_t C, const int32_t* __restrict__ qperm, int64_t bn,
    const float* __restrict__ tau, const float* __restrict__ qn, float xn_max, float eps_rel,
    const double* __restrict__ rad, const int32_t* __restrict__ tclo, const int32_t* __restrict__ tchi,
    int32_t ntiles, int32_t* __restrict__ tlist, int32_t* __restrict__ tcount, uint32_t* __restrict__ bits) {
  // need: one bit per cluster.  Each of the 32 warps takes every 32nd row of the block and sweeps
  // that query's distances to all clusters with coalesced reads (lanes over clusters), OR-ing a
  // ballot per 32 clusters into shared memory (round 1: one thread per cluster looping over the
  // rows, latency-bound, 149 us on c3; 8 warps: 108 us on c3, 0.63 ms per c5 batch).
  extern __shared__ uint32_t need[];
  constexpr int kW = kListThreads / 32;
  __shared__ int s_wcnt[kW];
  __shared__ int s_base;
  const int qb = blockIdx.x;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t r0 = int64_t(qb) * 128;
  const int rows = int(bn - r0 < 128 ? bn - r0 : 128);
  const int nw = (C + 31) >> 5;
  for (int w = threadIdx.x; w < nw; w += blockDim.x) need[w] = 0u;
  __syncthreads();
  for (int i = warp; i < rows; i += kW) {
    const int64_t row = r0 + i;
    const double thr = (double(tau[row]) + double(eps_rel) * (double(qn[row]) + double(xn_max))) * (1.0 + 1e-6);
    const double* dr = dq + int64_t(qperm[row]) * C;
    for (int c0 = 0; c0 < C; c0 += 32) {
      const int c = c0 + lane;
      bool nd = false;
      if (c < C) {
        const double lb = fmax(dr[c] * (1.0 - 1e-12) - rad[c], 0.0);
        nd = lb * lb <= thr;
      }
      const uint32_t m = __ballot_sync(0xffffffffu, nd);
      if (lane == 0 && m) atomicOr(&need[c0 >> 5], m);
    }
  }
  if (threadIdx.x == 0) s_base = 0;
  __syncthreads();
  for (int t0 = 0; t0 < ntiles; t0 += blockDim.x) {
    const int t = t0 + threadIdx.x;
    bool on = false;
    if (t < ntiles)
      for (int c = tclo[t]; c <= tchi[t] && !on; ++c) on = ((need[c >> 5] >> (c & 31)) & 1u) != 0u;
    const uint32_t b = __ballot_sync(0xffffffffu, on);
    if (lane == 0) s_wcnt[warp] = __popc(b);
    // tile-major schedule: bit t of row qb (32 tiles per word)
    const int nwords = (ntiles + 31) >> 5;
    if (bits != nullptr && lane == 0 && (t0 >> 5) + warp < nwords) bits[int64_t(qb) * nwords + (t0 >> 5) + warp] = b;
    __syncthreads();
    int off = s_base;
    for (int w = 0; w < warp; ++w) off += s_wcnt[w];
    if (on && tlist != nullptr) tlist[int64_t(qb) * ntiles + off + __popc(b & ((1u << lane) - 1u))] = t;
    __syncthreads();
    if (threadIdx.x == 0) {
      int tot = 0;
      for (int w = 0; w < kW; ++w) tot += s_wcnt[w];
      s_base += tot;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) tcount[qb] = s_base;
}

// number of query blocks that sweep each tile (tile-major schedule)
__global__ void tile_count_kernel(const uint32_t* __restrict__ bits, int32_t nqb, int32_t ntiles,
                                  int32_t* __restrict__ cnt) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= ntiles) return;
  const int nwords = (ntiles + 31) >> 5;
  int c = 0;
  for (int b = 0; b < nqb; ++b) c += (bits[int64_t(b) * nwords + (t >> 5)] >> (t & 31)) & 1u;
  cnt[t] = c;
}

// Work-unit plan over m groups holding cnt[g] list entries (one CTA, 1024 threads):
// total = sum cnt, U = max(umin, ceil(total / (per_slot * slots))) entries per unit,
// start[g] = exclusive scan of cnt, ustart[g] = exclusive scan of ceil(cnt / U).
// scal[0] = number of units, scal[1] = total, scal[2] = U.
__global__ void __launch_bounds__(1024) unit_plan_kernel(const int32_t* __restrict__ cnt, int32_t m, int32_t slots,
                                                         int32_t per_slot, int32_t umin,
                                                         int32_t* __restrict__ start, int32_t* __restrict__ ustart,
                                                         int32_t* __restrict__ scal) {
  __shared__ long long s_w[32];
  __shared__ int s_u;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int per = (m + 1023) / 1024;
  const int g0 = min(m, tid * per), g1 = min(m, g0 + per);
  auto block_excl_scan = [&](long long own) -> long long {  // exclusive prefix over threads, s_w[31] = total
    long long incl = own;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const long long v = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += v;
    }
    __syncthreads();
    if (lane == 31) s_w[warp] = incl;
    __syncthreads();
    if (warp == 0) {
      long long v = s_w[lane];
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const long long u = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += u;
      }
      s_w[lane] = v;
    }
    __syncthreads();
    return incl - own + (warp ? s_w[warp - 1] : 0ll);
  };
  long long own = 0;
  for (int g = g0; g < g1; ++g) own += cnt[g];
  long long pre = block_excl_scan(own);
  const long long total = s_w[31];
  if (tid == 0) {
    const long long want = (total + int64_t(per_slot) * slots - 1) / (int64_t(per_slot) * slots);
    s_u = int(want > (long long)umin ? want : (long long)umin);
  }
  for (int g = g0; g < g1; ++g) {
    start[g] = int32_t(pre);
    pre += cnt[g];
  }
  __syncthreads();
  const int U = s_u;
  long long uown = 0;
  for (int g = g0; g < g1; ++g) uown += (cnt[g] + U - 1) / U;
  long long upre = block_excl_scan(uown);
  for (int g = g0; g < g1; ++g) {
    ustart[g] = int32_t(upre);
    upre += (cnt[g] + U - 1) / U;
  }
  if (tid == 0) {
    scal[0] = int32_t(s_w[31]);
    scal[1] = int32_t(total);
    scal[2] = U;
  }
}

// tile-major units: unit = (tile t, query blocks blist[i0..i1)); the blocks of a tile in
// increasing order
__global__ void tile_units_fill_kernel(const uint32_t* __restrict__ bits, int32_t nqb, int32_t ntiles,
                                       const int32_t* __restrict__ cnt, const int32_t* __restrict__ start,
                                       const int32_t* __restrict__ ustart, const int32_t* __restrict__ scal,
                                       int32_t* __restrict__ blist, int32_t* __restrict__ ulist, int64_t ucap) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= ntiles) return;
  const int nwords = (ntiles + 31) >> 5;
  int pos = start[t];
  for (int b = 0; b < nqb; ++b)
    if ((bits[int64_t(b) * nwords + (t >> 5)] >> (t & 31)) & 1u) blist[pos++] = b;
  const int U = scal[2], c = cnt[t], s0 = start[t];
  int u = ustart[t];
  for (int i = 0; i < c; i += U, ++u) {
    if (u >= ucap) __trap();  // unit-list capacity (capi.cu KnnLayout) exceeded: an internal sizing bug
    ulist[3 * u] = t;
    ulist[3 * u + 1] = s0 + i;
    ulist[3 * u + 2] = s0 + min(c, i + U);
  }
}

// block-major units (per-block tile lists: the threshold sweep, and the FILTER when its operand is
// too wide to keep a tile resident): unit = (query block b, positions [i0, i1) of its list,
// flat index b * ntiles + i, ntiles = the list stride)
__global__ void block_units_fill_kernel(int32_t nqb, int32_t ntiles, const int32_t* __restrict__ cnt,
                                        const int32_t* __restrict__ ustart, const int32_t* __restrict__ scal,
                                        int32_t* __restrict__ ulist, int64_t ucap) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= nqb) return;
  const int U = scal[2], c = cnt[b];
  int u = ustart[b];
  for (int i = 0; i < c; i += U, ++u) {
    if (u >= ucap) __trap();  // unit-list capacity exceeded: an internal sizing bug
    ulist[3 * u] = b;
    ulist[3 * u + 1] = int32_t(int64_t(b) * ntiles + i);
    ulist[3 * u + 2] = int32_t(int64_t(b) * ntiles + min(c, i + U));
  }
}

// Threshold-sweep tile list of one block of 128 ball-sorted queries (thread 0 builds it; a
// shared bitmap dedupes tiles): every S-th tile, then for each distinct nearest ball of the
// block's queries (in sorted order) its tiles and those of its nearest neighbour balls until
// rows_need rows surround it, up to hmax such tiles.  Any set of disjoint segments bounds the
// k-th distance (the strided tiles alone give >= k of them); the near ones make it tight.
__global__ void __launch_bounds__(128) home_tile_lists_kernel(
    const int32_t* __restrict__ near_s, const int32_t* __restrict__ nbr, int64_t bn, const int64_t* __restrict__ off,
    int32_t ntiles, int32_t S, int64_t rows_need, int32_t hmax, int32_t lmax, int32_t* __restrict__ lists,
    int32_t* __restrict__ lcnt) {
  extern __shared__ uint32_t mark[];
  const int qb = blockIdx.x;
  const int nwords = (ntiles + 31) >> 5;
  for (int w = threadIdx.x; w < nwords; w += blockDim.x) mark[w] = 0u;
  __syncthreads();
  if (threadIdx.x != 0) return;
  int32_t* L = lists + int64_t(qb) * lmax;
  int c = 0, home = 0;
  for (int t = 0; t < ntiles && c < lmax; t += S) {
    L[c++] = t;
    mark[t >> 5] |= 1u << (t & 31);
  }
  auto add_ball = [&](int b) -> int64_t {
    const int64_t lo = off[b], hi = off[b + 1];
    if (hi <= lo) return 0;
    for (int t = int(lo / 256); t <= int((hi - 1) / 256) && home < hmax && c < lmax; ++t) {
      if ((mark[t >> 5] >> (t & 31)) & 1u) continue;
      mark[t >> 5] |= 1u << (t & 31);
      L[c++] = t;
      ++home;
    }
    return hi - lo;
  };
  int prev = -1;
  const int64_t r0 = int64_t(qb) * 128, r1 = min(bn, r0 + 128);
  for (int64_t r = r0; r < r1 && home < hmax; ++r) {
    const int b = near_s[r];
    if (b == prev) continue;
    prev = b;
    int64_t got = add_ball(b);
    for (int j = 0; j < kBallNbrs && got < rows_need && home < hmax; ++j) {
      const int nb = nbr[b * kBallNbrs + j];
      if (nb >= 0) got += add_ball(nb);
    }
  }
  DK_DCHECK(c <= lmax);
  lcnt[qb] = c;
}

// nearest other balls of each ball: one warp per ball, rounds of "smallest (d, id) above the last"
__global__ void ball_neighbors_kernel(const double* __restrict__ dq, int32_t C, int32_t* __restrict__ nbr) {
  const int b = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (b >= C) return;
  const double* row = dq + int64_t(b) * C;
  double last_d = -1.0;
  int last_i = -1;
  for (int j = 0; j < kBallNbrs; ++j) {
    double bd = INFINITY;
    int bi = -1;
    for (int c = lane; c < C; c += 32) {
      if (c == b) continue;
      const double v = row[c];
      const bool above = v > last_d || (v == last_d && c > last_i);
      if (above && (bi < 0 || v < bd || (v == bd && c < bi))) { bd = v; bi = c; }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double od = __shfl_xor_sync(0xffffffffu, bd, o);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (oi >= 0 && (bi < 0 || od < bd || (od == bd && oi < bi))) { bd = od; bi = oi; }
    }
    if (lane == 0) nbr[b * kBallNbrs + j] = bi;
    last_d = bd;
    last_i = bi;
  }
}

__global__ void iota_i32_kernel(int32_t* __restrict__ a, int64_t n) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) a[i] = int32_t(i);
}

__global__ void gather_rows_f64_kernel(const double* __restrict__ Q, const int32_t* __restrict__ perm, int64_t nq,
                                       int32_t d, double* __restrict__ out) {
  const int64_t i = blockIdx.x;
  if (i >= nq) return;
  const int64_t src = perm[i];
  for (int j = threadIdx.x; j < d; j += blockDim.x) out[i * d + j] = Q[src * d + j];
}

__global__ void scatter_knn_kernel(const int64_t* __restrict__ idx_p, const double* __restrict__ d2_p,
                                   const int32_t* __restrict__ perm, int64_t nq, int32_t k,
                                   int64_t* __restrict__ idx_out, double* __restrict__ d2_out) {
  const int64_t i = blockIdx.x;
  if (i >= nq) return;
  const int64_t dst = perm[i];
  for (int j = threadIdx.x; j < k; j += blockDim.x) {
    idx_out[dst * k + j] = idx_p[i * k + j];
    d2_out[dst * k + j] = d2_p[i * k + j];
  }
}

}  // namespace

void launch_query_cluster_dist(const double* Q, int64_t nq, int32_t d, const double* cent, int32_t C, double* dq,
                               int32_t* nearest, cudaStream_t s) {
  if (nq <= 0) return;
  dim3 grid(unsigned((nq + 31) / 32), unsigned((C + 63) / 64));
  query_cluster_dist_kernel<<<grid, 256, 0, s>>>(Q, nq, d, cent, C, dq);
  DK_CHECK_LAUNCH();
  nearest_cluster_kernel<<<unsigned((nq * 32 + 255) / 256), 256, 0, s>>>(dq, nq, C, nearest);
  DK_CHECK_LAUNCH();
}

void launch_nearest_ball_f32(const double* Q, int64_t nq, int32_t d, const double* cent, int32_t C,
                             unsigned long long* best, int32_t* nearest, cudaStream_t s) {
  if (nq <= 0) return;
  DK_CUDA(cudaMemsetAsync(best, 0xff, size_t(nq) * sizeof(unsigned long long), s));
  dim3 grid(unsigned((nq + 31) / 32), unsigned((C + 63) / 64));
  nearest_ball_f32_kernel<<<grid, 256, 0, s>>>(Q, nq, d, cent, C, best);
  DK_CHECK_LAUNCH();
  best_to_ball_kernel<<<unsigned((nq + 255) / 256), 256, 0, s>>>(best, nq, nearest);
  DK_CHECK_LAUNCH();
}

void launch_block_tile_lists(const double* dq, int32_t C, const int32_t* qperm, int64_t bn, int32_t nqb,
                             const float* tau, const float* qn, float xn_max, float eps_rel, const double* rad,
                             const int32_t* tclo, const int32_t* tchi, int32_t ntiles, int32_t* tlist,
                             int32_t* tcount, uint32_t* bits, cudaStream_t s) {
  const size_t smem = size_t((C + 31) / 32) * 4;
  set_dynamic_smem(block_tile_lists_kernel, smem);
  block_tile_lists_kernel<<<unsigned(nqb), kListThreads, smem, s>>>(dq, C, qperm, bn, tau, qn, xn_max, eps_rel, rad,
                                                                      tclo, tchi, ntiles, tlist, tcount, bits);
  DK_CHECK_LAUNCH();
}

size_t ball_sort_temp_bytes(int64_t nq) {
  size_t bytes = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, bytes, static_cast<const int32_t*>(nullptr), static_cast<int32_t*>(nullptr),
                                  static_cast<const int32_t*>(nullptr), static_cast<int32_t*>(nullptr), int(nq));
  return bytes + 256;
}

void launch_sort_queries_by_ball(const int32_t* nearest, int64_t nq, int32_t C, int32_t* nearest_sorted,
                                 int32_t* iota, int32_t* qperm, void* temp, size_t temp_bytes, cudaStream_t s) {
  if (nq <= 0) return;
  iota_i32_kernel<<<unsigned((nq + 255) / 256), 256, 0, s>>>(iota, nq);
  DK_CHECK_LAUNCH();
  int bits = 1;
  while ((int64_t(1) << bits) < int64_t(C)) ++bits;
  // stable LSD radix sort: queries of a ball keep their batch order (== a counting sort)
  DK_CUDA(cub::DeviceRadixSort::SortPairs(temp, temp_bytes, nearest, nearest_sorted, iota, qperm, int(nq), 0, bits,
                                          s));
  g_launches.fetch_add(1);
}

void launch_tile_units(const uint32_t* bits, int32_t nqb, int32_t ntiles, int32_t slots, int32_t* tcnt,
                       int32_t* tstart, int32_t* ustart, int32_t* scal, int32_t* blist, int32_t* ulist,
                       int64_t ucap, cudaStream_t s) {
  tile_count_kernel<<<unsigned((ntiles + 255) / 256), 256, 0, s>>>(bits, nqb, ntiles, tcnt);
  DK_CHECK_LAUNCH();
  // >= 4 units per CTA; a unit keeps its tile resident while its query blocks stream past
  unit_plan_kernel<<<1, 1024, 0, s>>>(tcnt, ntiles, slots, 4, 4, tstart, ustart, scal);
  DK_CHECK_LAUNCH();
  tile_units_fill_kernel<<<unsigned((ntiles + 255) / 256), 256, 0, s>>>(bits, nqb, ntiles, tcnt, tstart, ustart, scal,
                                                                        blist, ulist, ucap);
  DK_CHECK_LAUNCH();
}

void launch_home_tile_lists(const int32_t* near_sorted, const int32_t* ball_nbr, int64_t bn, int32_t nqb,
                            const int64_t* ball_off, int32_t ntiles, int32_t S, int64_t rows_need, int32_t hmax,
                            int32_t lmax, int32_t* lists, int32_t* lcnt, cudaStream_t s) {
  const size_t smem = size_t((ntiles + 31) / 32) * 4;
  set_dynamic_smem(home_tile_lists_kernel, smem);
  home_tile_lists_kernel<<<unsigned(nqb), 128, smem, s>>>(near_sorted, ball_nbr, bn, ball_off, ntiles, S, rows_need,
                                                          hmax, lmax, lists, lcnt);
  DK_CHECK_LAUNCH();
}

void launch_ball_neighbors(const double* dq, int32_t C, int32_t* nbr, cudaStream_t s) {
  ball_neighbors_kernel<<<unsigned((int64_t(C) * 32 + 255) / 256), 256, 0, s>>>(dq, C, nbr);
  DK_CHECK_LAUNCH();
}

void launch_block_units(const int32_t* tcount, int32_t nqb, int32_t ntiles, int32_t slots, int32_t* bstart,
                        int32_t* ustart, int32_t* scal, int32_t* ulist, int64_t ucap, cudaStream_t s) {
  // units of ~equal length (>= 8 tiles) so the persistent CTAs finish together
  unit_plan_kernel<<<1, 1024, 0, s>>>(tcount, nqb, slots, 4, 8, bstart, ustart, scal);
  DK_CHECK_LAUNCH();
  block_units_fill_kernel<<<unsigned((nqb + 127) / 128), 128, 0, s>>>(nqb, ntiles, tcount, ustart, scal, ulist,
                                                                       ucap);
  DK_CHECK_LAUNCH();
}

void launch_gather_rows_f64(const double* Q, const int32_t* perm, int64_t nq, int32_t d, double* out, cudaStream_t s) {
  if (nq <= 0) return;
  gather_rows_f64_kernel<<<unsigned(nq), 128, 0, s>>>(Q, perm, nq, d, out);
  DK_CHECK_LAUNCH();
}

void launch_scatter_knn(const int64_t* idx_p, const double* d2_p, const int32_t* perm, int64_t nq, int32_t k,
                        int64_t* idx_out, double* d2_out, cudaStream_t s) {
  if (nq <= 0) return;
  scatter_knn_kernel<<<unsigned(nq), 128, 0, s>>>(idx_p, d2_p, perm, nq, k, idx_out, d2_out);
  DK_CHECK_LAUNCH();
}

void launch_fill_float(float* p, int64_t count, float v, cudaStream_t s) {
  if (count <= 0) return;
  fill_float_kernel<<<unsigned((count + 255) / 256), 256, 0, s>>>(p, count, v);
  DK_CHECK_LAUNCH();
}

void launch_tau_from_hist(const uint32_t* hist, const float* hlo, const float* hinv, const float* htop,
                          const float* tau_h, int64_t nq, int32_t k, const float* qn, float xn_max, float eps_rel,
                          float* tau, cudaStream_t s) {
  if (nq <= 0) return;
  tau_hist_kernel<<<unsigned((nq + 255) / 256), 256, 0, s>>>(hist, hlo, hinv, htop, tau_h, nq, k, qn, xn_max, eps_rel,
                                                             tau);
  DK_CHECK_LAUNCH();
}

void launch_tau_from_tmin(const float* tmin, int32_t nseg, int32_t nq_pad, int64_t nq, int32_t k, const float* qn,
                          float xn_max, float eps_rel, float* tau, cudaStream_t s, const int32_t* block_entries,
                          int32_t segs_per, float* hlo, float* hinv, float* htop) {
  const bool sort_path = std::getenv("DK_TAU_SORT") != nullptr && block_entries == nullptr && hlo == nullptr;
  if (!sort_path) {
    const size_t smem = size_t(std::max(nseg, 1)) * 4;
    if (smem > 232448) throw Error{DK_EINVAL, "too many k-NN segments"};
    set_dynamic_smem(tau_radix_kernel, smem);
    tau_radix_kernel<<<unsigned(nq), 256, smem, s>>>(tmin, nseg, nq_pad, nq, k, qn, xn_max, eps_rel, tau,
                                                     block_entries, segs_per, hlo, hinv, htop);
    DK_CHECK_LAUNCH();
    return;
  }
  const int B = std::max(2, pow2_ceil(nseg));
  const size_t smem = size_t(B) * 8;
  if (smem > 232448) throw Error{DK_EINVAL, "too many k-NN segments"};
  set_dynamic_smem(tau_from_tmin_kernel, smem);
  tau_from_tmin_kernel<<<unsigned(nq), 256, smem, s>>>(tmin, nseg, nq_pad, nq, k, B, qn, xn_max, eps_rel, tau);
  DK_CHECK_LAUNCH();
}

void launch_select(const float* X, int64_t global_offset, int32_t d, const double* Q, int64_t nq, int32_t k,
                   const unsigned long long* cand, const uint32_t* cand_cnt, int32_t cap, const float* qn,
                   float xn_max, float eps_rel, int64_t* idx_out, double* d2_out, int32_t* lists, int32_t* counts,
                   int num_sms, cudaStream_t s, const int64_t* perm) {
  // lists: [2][nq] (slow, overflow), counts: [2] device counters, zeroed by the caller
  if (nq <= 0) return;
  int32_t* slow_list = lists;
  int32_t* ovf_list = lists + nq;
  const int Kp = std::max(32, pow2_ceil(k));
  // keys re-ranked by the fast path: every key within 2 eps of the k-th approx key, up to
  // max(2 pow2(k), 2048) (single-pass fp16 sweeps at c5 put ~1,000 keys in that window; 32 KB
  // of shared memory keeps 6 CTAs per SM)
  const int scap = std::max(2 * Kp, 2048);
  const size_t fast_smem = size_t(scap) * sizeof(Key128) + size_t(d) * sizeof(double) + kSelHist * sizeof(uint32_t);
  const bool g4 = exact_group(d) == 4;
  auto fast = g4 ? select_fast_kernel<4> : select_fast_kernel<8>;
  set_dynamic_smem(fast, fast_smem);
  if (fast_smem > 232448) throw Error{DK_EINVAL, "k too large for the k-NN selection buffer"};
  fast<<<unsigned(nq), 256, fast_smem, s>>>(X, global_offset, d, Q, nq, k, cand, cand_cnt, cap, qn, xn_max, eps_rel,
                                            idx_out, d2_out, slow_list, counts, ovf_list, counts + 1, perm, scap);
  DK_CHECK_LAUNCH();
  const int B = std::max(2, pow2_ceil(cap));
  const size_t slow_smem = size_t(B) * 8 + size_t(2 * Kp) * sizeof(Key128) + size_t(d) * sizeof(double);
  if (slow_smem > 232448) throw Error{DK_EINVAL, "k or candidate capacity too large for the k-NN selection buffer"};
  auto slow = g4 ? select_slow_kernel<4> : select_slow_kernel<8>;
  set_dynamic_smem(slow, slow_smem);
  slow<<<unsigned(std::max(1, 2 * num_sms)), 256, slow_smem, s>>>(X, global_offset, d, Q, k, cand, cand_cnt, cap, qn,
                                                                  xn_max, eps_rel, B, idx_out, d2_out, slow_list,
                                                                  counts, perm);
  DK_CHECK_LAUNCH();
}

void launch_exact_knn_fallback(const float* X, int64_t n_local, int64_t global_offset, int32_t d, const double* Q,
                               const int32_t* qlist, const int32_t* qcount, int32_t k, int64_t* idx_out,
                               double* d2_out, int num_sms, cudaStream_t s, void* tmp, size_t tmp_bytes) {
  const int Kp = pow2_ceil(k);
  const int B = std::max(1024, 2 * Kp);
  const size_t smem = size_t(B) * sizeof(Key128);
  auto fb = exact_group(d) == 4 ? exact_knn_kernel<4> : exact_knn_kernel<8>;
  set_dynamic_smem(fb, smem);
  if (smem > 232448) throw Error{DK_EINVAL, "k too large for the exact k-NN fallback"};
  // slices when the scratch (the candidate lists, free once the selection has run) holds them and
  // every slice has at least k rows' worth of work
  constexpr int kSplit = 32, kSplitMax = 128;
  const size_t need = size_t(kSplitMax) * kSplit * k * 16;
  const bool split = tmp != nullptr && tmp_bytes >= need && n_local >= int64_t(kSplit) * 4096;
  int64_t* tmp_idx = static_cast<int64_t*>(tmp);
  double* tmp_d2 = reinterpret_cast<double*>(tmp_idx + size_t(kSplitMax) * kSplit * k);
  fb<<<unsigned(std::max(1, 2 * num_sms)), 256, smem, s>>>(X, n_local, global_offset, d, Q, qlist, qcount, k, B,
                                                           idx_out, d2_out, split ? kSplit : 1, kSplitMax, tmp_idx,
                                                           tmp_d2);
  DK_CHECK_LAUNCH();
  if (split) {
    exact_merge_kernel<<<kSplitMax * 32 / 256, 256, 0, s>>>(qlist, qcount, kSplitMax, kSplit, k, global_offset,
                                                            tmp_idx, tmp_d2, idx_out, d2_out);
    DK_CHECK_LAUNCH();
  }
}

void launch_merge_topk(int32_t parts, int64_t nq, int32_t k, const int64_t* idx_in, const double* d2_in,
                       int64_t* idx_out, double* d2_out, cudaStream_t s) {
  if (parts > 64) throw Error{DK_EINVAL, "dk_merge_topk supports at most 64 parts"};
  if (nq <= 0) return;
  merge_topk_kernel<<<unsigned((nq * 32 + 255) / 256), 256, 0, s>>>(parts, nq, k, idx_in, d2_in, idx_out, d2_out);
  DK_CHECK_LAUNCH();
}

}  // namespace dk
