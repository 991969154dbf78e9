// sample.cu — Philox-indexed gather kernels (K3): RS, DEANN residual, explicit rows.
//
// Reference: rs_kde (estimators.py:152-164), _rs_excluding (:203-233),
// _kernel_rows (:106-119), deann's value formula (:372).
//
// Stream semantics.  For query j (global position j + query_base) the t-th
// draw is
//     r = philox4x32_10(ctr = {t_lo, t_hi, j_lo, j_hi}, key = {seed_lo, seed_hi})
//     row_t = mulhi64((r.y << 32) | r.x, N)                    (N = global n)
// i.e. uniform with replacement over [0, N).  The first m draws whose row is
// NOT in the query's exclusion list (its k-NN set X1) are accepted — exactly
// the effective rule of _rs_excluding ("keep the first `need` non-excluded
// draws of each batch", estimators.py:225-228), so feeding this stream to the
// reference through a replaying `rng.integers` reproduces its estimate.
//
// One warp per query; 32 consecutive draws per iteration; accepted draws are
// compacted with a ballot so acceptance order == draw order.  Accepted rows
// are evaluated by groups of G lanes (coalesced float4 row loads), fp64
// direct-difference distance, fp64 exp (parity ~1e-15 with the reference's
// fp64 arithmetic).
#include "internal.h"

namespace dk {

namespace {

__device__ __forceinline__ uint4 philox4x32_10(uint4 c, uint2 k) {
  constexpr uint32_t M0 = 0xD2511F53u, M1 = 0xCD9E8D57u, W0 = 0x9E3779B9u, W1 = 0xBB67AE85u;
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    if (r) { k.x += W0; k.y += W1; }
    const uint32_t lo0 = M0 * c.x, hi0 = __umulhi(M0, c.x);
    const uint32_t lo1 = M1 * c.z, hi1 = __umulhi(M1, c.z);
    c = make_uint4(hi1 ^ c.y ^ k.x, lo1, hi0 ^ c.w ^ k.y, lo0);
  }
  return c;
}

__device__ __forceinline__ int64_t draw_row(uint64_t seed, uint64_t t, uint64_t jg, uint64_t N) {
  const uint4 r = philox4x32_10(make_uint4(uint32_t(t), uint32_t(t >> 32), uint32_t(jg), uint32_t(jg >> 32)),
                                make_uint2(uint32_t(seed), uint32_t(seed >> 32)));
  const uint64_t v = (uint64_t(r.y) << 32) | uint64_t(r.x);
  return int64_t(__umul64hi(v, N));
}

__device__ __forceinline__ bool in_sorted(const int64_t* __restrict__ a, int cnt, int64_t v) {
  int lo = 0, hi = cnt;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    const int64_t x = a[mid];
    if (x < v) lo = mid + 1; else hi = mid;
  }
  return lo < cnt && a[lo] == v;
}

// fp64 kernel value between the query (fp64, in smem) and one fp32 dataset row
__device__ __forceinline__ double row_kernel(const float* __restrict__ x, const double* __restrict__ q, int d,
                                             int family, double c) {
  double acc = 0.0;
  if ((d & 3) == 0) {
    const float4* x4 = reinterpret_cast<const float4*>(x);
    for (int k4 = 0; k4 < (d >> 2); ++k4) {
      const float4 v = __ldg(x4 + k4);
      const double t0 = double(v.x) - q[4 * k4 + 0], t1 = double(v.y) - q[4 * k4 + 1];
      const double t2 = double(v.z) - q[4 * k4 + 2], t3 = double(v.w) - q[4 * k4 + 3];
      if (family == DK_LAPLACIAN) {
        acc += (fabs(t0) + fabs(t1)) + (fabs(t2) + fabs(t3));
      } else {
        acc = fma(t0, t0, acc); acc = fma(t1, t1, acc); acc = fma(t2, t2, acc); acc = fma(t3, t3, acc);
      }
    }
  } else {
    for (int k = 0; k < d; ++k) {
      const double t = double(__ldg(x + k)) - q[k];
      acc = family == DK_LAPLACIAN ? acc + fabs(t) : fma(t, t, acc);
    }
  }
  // c = 1/(2h^2) for gaussian (exp(-d2*c)), 1/h otherwise
  if (family == DK_EXPONENTIAL) acc = sqrt(acc);
  return exp(-acc * c);
}

__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Accepted rows are evaluated by groups of G lanes (G = 1..32 chosen from d):
// each group reads one row with G-wide coalesced float4 loads and reduces its
// fp64 partial with shuffles, so rows of any width stream at full sector use.
template <int G>
__device__ __forceinline__ double group_row_kernel(const float* __restrict__ x, const double* __restrict__ q, int d,
                                                   int family, double c, int gl) {
  double acc = 0.0;
  if ((d & 3) == 0) {
    // batches of 4 float4 per lane, all loads issued before the fp64 work (memory-level
    // parallelism for wide rows); the accumulation order stays k4 = gl, gl + G, ...
    const float4* x4 = reinterpret_cast<const float4*>(x);
    const int chunks = d >> 2;
    for (int b0 = gl; b0 < chunks; b0 += 4 * G) {
      float4 v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int k4 = b0 + u * G;
        v[u] = k4 < chunks ? __ldg(x4 + k4) : make_float4(0.f, 0.f, 0.f, 0.f);
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int k4 = b0 + u * G;
        if (k4 < chunks) {
          const double t0 = double(v[u].x) - q[4 * k4 + 0], t1 = double(v[u].y) - q[4 * k4 + 1];
          const double t2 = double(v[u].z) - q[4 * k4 + 2], t3 = double(v[u].w) - q[4 * k4 + 3];
          if (family == DK_LAPLACIAN) acc += (fabs(t0) + fabs(t1)) + (fabs(t2) + fabs(t3));
          else { acc = fma(t0, t0, acc); acc = fma(t1, t1, acc); acc = fma(t2, t2, acc); acc = fma(t3, t3, acc); }
        }
      }
    }
  } else {
    for (int k = gl; k < d; k += G) {
      const double t = double(__ldg(x + k)) - q[k];
      acc = family == DK_LAPLACIAN ? acc + fabs(t) : fma(t, t, acc);
    }
  }
#pragma unroll
  for (int o = G / 2; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  return acc;  // the family's distance sum (squared L2 or L1); kernel value by kernel_of_sum
}

// kernel value from a distance sum: exp(-d2 c) gaussian, exp(-sqrt(d2) c) exponential,
// exp(-L1 c) laplacian (c = 1/(2h^2) or 1/h)
__device__ __forceinline__ double kernel_of_sum(double acc, int family, double c) {
  if (family == DK_EXPONENTIAL) acc = sqrt(acc);
  return exp(-acc * c);
}

// Distance sum of one row from float4s already in registers (IT per lane, same
// accumulation order as group_row_kernel: lane gl takes chunks gl, gl+G, ...).
template <int G, int IT>
__device__ __forceinline__ double group_row_regs(const float4 (&xv)[IT], const double* __restrict__ q, int chunks,
                                                 int family, double c, int gl) {
  double acc = 0.0;
#pragma unroll
  for (int it = 0; it < IT; ++it) {
    const int k4 = gl + it * G;
    if (k4 < chunks) {
      const float4 v = xv[it];
      const double t0 = double(v.x) - q[4 * k4 + 0], t1 = double(v.y) - q[4 * k4 + 1];
      const double t2 = double(v.z) - q[4 * k4 + 2], t3 = double(v.w) - q[4 * k4 + 3];
      if (family == DK_LAPLACIAN) acc += (fabs(t0) + fabs(t1)) + (fabs(t2) + fabs(t3));
      else { acc = fma(t0, t0, acc); acc = fma(t1, t1, acc); acc = fma(t2, t2, acc); acc = fma(t3, t3, acc); }
    }
  }
#pragma unroll
  for (int o = G / 2; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  return acc;
}

template <int G, int IT>
__device__ __forceinline__ void load_row(const float* __restrict__ x, bool valid, int chunks, int gl,
                                         float4 (&b)[IT]) {
  const float4* x4 = reinterpret_cast<const float4*>(x);
#pragma unroll
  for (int it = 0; it < IT; ++it) {
    const int k4 = gl + it * G;
    b[it] = (valid && k4 < chunks) ? __ldg(x4 + k4) : make_float4(0.f, 0.f, 0.f, 0.f);
  }
}

template <int G, int IT>
__global__ void sample_kernel(const float* __restrict__ X, int64_t n_local, int64_t global_offset, int64_t N,
                              int32_t d, const double* __restrict__ Q, int64_t nq, int32_t family, double c,
                              int32_t m, uint64_t seed, int64_t query_base, const int64_t* __restrict__ excl,
                              const int32_t* __restrict__ excl_cnt, int32_t excl_stride, double* __restrict__ z_sum,
                              int64_t* __restrict__ acc_idx, int64_t* __restrict__ draws) {
  extern __shared__ double sq[];
  constexpr int R = 32 / G;  // rows evaluated per warp step
  const int wib = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nw = blockDim.x >> 5;
  const int64_t j = int64_t(blockIdx.x) * nw + wib;
  if (j >= nq) return;
  double* q = sq + size_t(wib) * d;
  int64_t* rows_s = reinterpret_cast<int64_t*>(sq + size_t(nw) * d) + wib * 32;
  for (int k = lane; k < d; k += 32) q[k] = Q[size_t(j) * d + k];
  __syncwarp();
  const int ecnt = excl ? (excl_cnt ? excl_cnt[j] : excl_stride) : 0;
  const int64_t* ex = excl ? excl + size_t(j) * excl_stride : nullptr;
  const uint64_t jg = uint64_t(j + query_base);
  const uint32_t lt_mask = (1u << lane) - 1u;
  const int grp = lane / G, gl = lane % G;
  double zsum = 0.0;
  int accepted = 0;
  uint64_t t_base = 0;
  int64_t last_t = -1;
  while (accepted < m) {
    const uint64_t t = t_base + lane;
    const int64_t row = draw_row(seed, t, jg, uint64_t(N));
    DK_DCHECK(row >= 0 && row < N);
    const bool ok = ecnt == 0 || !in_sorted(ex, ecnt, row);
    const uint32_t ballot = __ballot_sync(0xffffffffu, ok);
    const int rank = __popc(ballot & lt_mask);
    const bool take = ok && (accepted + rank < m);
    if (take) {
      rows_s[rank] = row;
      if (acc_idx) acc_idx[size_t(j) * m + accepted + rank] = row;
    }
    const uint32_t took = __ballot_sync(0xffffffffu, take);
    const int ntook = __popc(took);
    __syncwarp();
    // each group reduces its row's distance sum; batch row r's sum is handed to lane r, which
    // evaluates the fp64 exponential once for the batch (not once per lane of every group)
    double lane_sum = 0.0;
    auto hand_over = [&](int r0, double acc) {
      const int src = ((lane - r0) & (R - 1)) * G;  // group (lane - r0) holds row lane's sum
      const double a = __shfl_sync(0xffffffffu, acc, src);
      if (lane >= r0 && lane < r0 + R) lane_sum = a;
    };
    if constexpr (IT > 0) {
      // software-pipelined: the next row's float4s are in flight while this one is reduced
      const int chunks = d >> 2;
      float4 cur[IT], nxt[IT];
      int64_t loc = grp < ntook ? rows_s[grp] - global_offset : -1;
      bool mine = loc >= 0 && loc < n_local;
      load_row<G, IT>(X + size_t(mine ? loc : 0) * d, mine, chunks, gl, cur);
      for (int r0 = 0; r0 < ntook; r0 += R) {
        const int rn = r0 + R + grp;
        const int64_t locn = rn < ntook ? rows_s[rn] - global_offset : -1;
        const bool minen = locn >= 0 && locn < n_local;
        if (r0 + R < ntook) load_row<G, IT>(X + size_t(minen ? locn : 0) * d, minen, chunks, gl, nxt);
        hand_over(r0, group_row_regs<G, IT>(cur, q, chunks, family, c, gl));
#pragma unroll
        for (int it = 0; it < IT; ++it) cur[it] = nxt[it];
        mine = minen;
      }
    } else {
      for (int r0 = 0; r0 < ntook; r0 += R) {
        const int r = r0 + grp;
        const int64_t loc = r < ntook ? rows_s[r] - global_offset : -1;
        const bool mine = loc >= 0 && loc < n_local;
        // groups with no row still take part in the shuffles (G-lane reduction is warp-synchronous)
        hand_over(r0, group_row_kernel<G>(X + size_t(mine ? loc : 0) * d, q, d, family, c, gl));
      }
    }
    if (lane < ntook) {
      const int64_t loc = rows_s[lane] - global_offset;
      if (loc >= 0 && loc < n_local) zsum += kernel_of_sum(lane_sum, family, c);
    }
    __syncwarp();
    if (took) last_t = int64_t(t_base) + 31 - __clz(took);
    accepted += ntook;
    t_base += 32;
  }
  zsum = warp_sum_d(zsum);
  if (lane == 0) {
    z_sum[j] = zsum;
    if (draws) draws[j] = last_t + 1;
  }
}

// per-query ascending sort of the exclusion list (block per query, bitonic in smem)
__global__ void sort_excl_kernel(const int64_t* __restrict__ excl, const int32_t* __restrict__ cnt, int32_t stride,
                                 int32_t B, int64_t* __restrict__ sorted) {
  extern __shared__ long long sb[];
  const int64_t q = blockIdx.x;
  const int c = cnt ? cnt[q] : stride;
  for (int i = threadIdx.x; i < B; i += blockDim.x) sb[i] = i < c ? excl[size_t(q) * stride + i] : LLONG_MAX;
  for (int k = 2; k <= B; k <<= 1) {
    for (int jj = k >> 1; jj > 0; jj >>= 1) {
      __syncthreads();
      for (int i = threadIdx.x; i < B; i += blockDim.x) {
        const int ixj = i ^ jj;
        if (ixj > i) {
          const bool up = (i & k) == 0;
          const long long a = sb[i], b = sb[ixj];
          if ((a > b) == up) { sb[i] = b; sb[ixj] = a; }
        }
      }
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < c; i += blockDim.x) sorted[size_t(q) * stride + i] = sb[i];
}

// explicit rows: out[j] = sum_c K(q_j, x_rows[j*stride + c])   (one warp per query)
__global__ void eval_rows_kernel(const float* __restrict__ X, int64_t n_local, int64_t global_offset, int32_t d,
                                 const double* __restrict__ Q, int64_t nq, int32_t family, double c,
                                 const int64_t* __restrict__ rows, const int32_t* __restrict__ cnt, int32_t stride,
                                 double* __restrict__ out) {
  extern __shared__ double sq[];
  const int wib = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t j = int64_t(blockIdx.x) * (blockDim.x >> 5) + wib;
  if (j >= nq) return;
  double* q = sq + size_t(wib) * d;
  for (int k = lane; k < d; k += 32) q[k] = Q[size_t(j) * d + k];
  __syncwarp();
  const int r = cnt ? cnt[j] : stride;
  double s = 0.0;
  for (int i = lane; i < r; i += 32) {
    const int64_t loc = rows[size_t(j) * stride + i] - global_offset;
    if (loc >= 0 && loc < n_local) s += row_kernel(X + size_t(loc) * d, q, d, family, c);
  }
  s = warp_sum_d(s);
  if (lane == 0) out[j] = s;
}

// value = (k^/n) Z1 + ((n-k^)/n) Z2   (estimators.py:344-372), one thread per query;
// k^ = khat[j] neighbours (an index may return fewer than k, ann.py:30-31) or k
__global__ void deann_combine_kernel(int64_t nq, int32_t family, double c, int32_t k, int32_t m, int64_t n,
                                     const int32_t* __restrict__ khat, const double* __restrict__ nbr_d2,
                                     const double* __restrict__ z1_l1_sum, const double* __restrict__ z2_sum,
                                     double* __restrict__ value) {
  const int64_t j = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (j >= nq) return;
  const int kh = khat ? khat[j] : k;
  double z1 = 0.0;
  if (kh > 0) {
    if (family == DK_LAPLACIAN) {
      z1 = z1_l1_sum[j] / double(kh);
    } else {
      double s = 0.0;
      for (int i = 0; i < kh; ++i) {
        double dd = nbr_d2[size_t(j) * k + i];
        if (family == DK_EXPONENTIAL) dd = sqrt(dd);
        s += exp(-dd * c);
      }
      z1 = s / double(kh);
    }
  }
  double v = (double(kh) / double(n)) * z1;
  if (m > 0) v += (double(n - kh) / double(n)) * (z2_sum[j] / double(m));
  value[j] = v;
}

__global__ void kernel_values_kernel(int32_t family, double h, const double* __restrict__ dist, int64_t count,
                                     double* __restrict__ out, uint32_t* __restrict__ bad) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= count) return;
  const double v = dist[i];
  if (!isfinite(v)) atomicOr(bad, 1u);
  else if (v < 0.0) atomicOr(bad, 2u);
  out[i] = family == DK_GAUSSIAN ? exp(-v / (2.0 * h * h)) : exp(-v / h);
}

double family_c(int32_t family, double h) { return family == DK_GAUSSIAN ? 1.0 / (2.0 * h * h) : 1.0 / h; }

}  // namespace

void launch_sample(const float* X, int64_t n_local, int64_t global_offset, int64_t global_n, int32_t d,
                   const double* Q, int64_t nq, int32_t family, double bandwidth, int32_t m, uint64_t seed,
                   int64_t query_base, const int64_t* excl_sorted, const int32_t* excl_cnt, int32_t excl_stride,
                   double* z_sum, int64_t* acc_idx, int64_t* draws, cudaStream_t s) {
  // 8 warps (queries) per block; fewer for very wide rows so the fp64 query copies fit
  const int wpb = int(std::max<int64_t>(1, std::min<int64_t>(8, 232448 / (int64_t(d) * 8 + 256))));
  const size_t smem = size_t(wpb) * d * sizeof(double) + size_t(wpb) * 32 * sizeof(int64_t);
  if (smem > 232448) throw Error{DK_EINVAL, "dimension too large for the sampling kernel (d > 29000)"};
  const double c = family_c(family, bandwidth);
  const unsigned grid = unsigned((nq + wpb - 1) / wpb);
  // lanes per row: enough that one float4 sweep of the row covers >= ~1/2 of its 16 B chunks
  const int chunks = (d + 3) / 4;
#define DK_SAMPLE_LAUNCH(G, IT)                                                                               \
  do {                                                                                                        \
    set_dynamic_smem(sample_kernel<G, IT>, smem);                                                             \
    sample_kernel<G, IT><<<grid, wpb * 32, smem, s>>>(X, n_local, global_offset, global_n, d, Q, nq, family, c, \
                                                      m, seed, query_base, excl_sorted, excl_cnt, excl_stride,  \
                                                      z_sum, acc_idx, draws);                                   \
  } while (0)
  // pipelined row loads when rows are whole float4s and G < 32 (a row is at most 4 float4s
  // per lane).  For wide rows (G = 32) the double buffer costs more occupancy than it hides
  // latency (c4, d = 784: 8.5 -> 9.1 ms), so those keep the plain loop.
  const bool vec = (d & 3) == 0;
  if (chunks >= 64) {
    DK_SAMPLE_LAUNCH(32, 0);
  } else if (chunks >= 32) {
    if (vec) DK_SAMPLE_LAUNCH(16, 4); else DK_SAMPLE_LAUNCH(16, 0);
  } else if (chunks >= 16) {
    if (vec) DK_SAMPLE_LAUNCH(8, 4); else DK_SAMPLE_LAUNCH(8, 0);
  } else if (chunks >= 8) {
    if (vec) DK_SAMPLE_LAUNCH(4, 4); else DK_SAMPLE_LAUNCH(4, 0);
  } else if (chunks >= 4) {
    if (vec) DK_SAMPLE_LAUNCH(2, 4); else DK_SAMPLE_LAUNCH(2, 0);
  } else {
    if (vec) DK_SAMPLE_LAUNCH(1, 4); else DK_SAMPLE_LAUNCH(1, 0);
  }
#undef DK_SAMPLE_LAUNCH
  DK_CHECK_LAUNCH();
}

void launch_sort_excl(const int64_t* excl, const int32_t* excl_cnt, int32_t stride, int64_t nq, int64_t* sorted,
                      cudaStream_t s) {
  int B = 1;
  while (B < stride) B <<= 1;
  const size_t smem = size_t(B) * 8;
  if (smem > 232448) throw Error{DK_EINVAL, "exclusion list too long (k > 29000) for the sampling path"};
  set_dynamic_smem(sort_excl_kernel, smem);
  sort_excl_kernel<<<unsigned(nq), 256, smem, s>>>(excl, excl_cnt, stride, B, sorted);
  DK_CHECK_LAUNCH();
}

void launch_eval_rows(const float* X, int64_t n_local, int64_t global_offset, int32_t d, const double* Q, int64_t nq,
                      int32_t family, double bandwidth, const int64_t* rows, const int32_t* cnt, int32_t stride,
                      double* out, cudaStream_t s) {
  const int wpb = int(std::max<int64_t>(1, std::min<int64_t>(8, 232448 / (int64_t(d) * 8))));
  const size_t smem = size_t(wpb) * d * sizeof(double);
  if (smem > 232448) throw Error{DK_EINVAL, "dimension too large for the row evaluation (d > 29000)"};
  set_dynamic_smem(eval_rows_kernel, smem);
  eval_rows_kernel<<<unsigned((nq + wpb - 1) / wpb), wpb * 32, smem, s>>>(
      X, n_local, global_offset, d, Q, nq, family, family_c(family, bandwidth), rows, cnt, stride, out);
  DK_CHECK_LAUNCH();
}

void launch_kernel_values(int32_t family, double h, const double* dist, int64_t count, double* out, uint32_t* bad,
                          cudaStream_t s) {
  kernel_values_kernel<<<unsigned((count + 255) / 256), 256, 0, s>>>(family, h, dist, count, out, bad);
  DK_CHECK_LAUNCH();
}

void launch_deann_combine(int64_t nq, int32_t family, double bandwidth, int32_t k, int32_t m, int64_t n_total,
                          const double* nbr_d2, const double* z1_l1_sum, const double* z2_sum, double* value,
                          cudaStream_t s, const int32_t* khat) {
  deann_combine_kernel<<<unsigned((nq + 255) / 256), 256, 0, s>>>(nq, family, family_c(family, bandwidth), k, m,
                                                                  n_total, khat, nbr_d2, z1_l1_sum, z2_sum, value);
  DK_CHECK_LAUNCH();
}

}  // namespace dk
