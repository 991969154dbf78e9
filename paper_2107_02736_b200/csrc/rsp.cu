// rsp.cu — permuted-window sampler (RSP / DEANNP).
//
// Reference: rsp_kde (estimators.py:180-200), _rsp_excluding (:249-303),
// _window_kernel_sum / _block_kernel_values (:167-177, :236-246), the cursor
// threading of deann_batch (:394-409) and permute (data.py:214-233).
//
// The dataset handle used here holds the PERMUTED rows (row i = original row
// permutation[i]), so every window is a contiguous (wrapping) run of rows: the
// GPU streams it with coalesced loads instead of a random gather.  For query j
// the walk starts at its cursor, skips rows whose ORIGINAL id is excluded (its
// k-NN set), and stops after m accepted rows or one full pass:
//   * rows consumed L_j = the smallest L whose window holds m accepted rows
//     (L = m + #excluded in the window, solved by fixed-point iteration over the
//     query's sorted excluded positions), or n when fewer than m rows remain;
//   * shared cursor: start_{j+1} = start_j + L_j (mod n) — a sequential chain,
//     computed by one thread over all queries (O(k log k) per query) before the
//     parallel evaluation; independent cursors: start_j = floor(j n / nq).
#include "internal.h"

namespace dk {

namespace {

__device__ __forceinline__ int lower_bound_i64(const int64_t* a, int cnt, int64_t v) {
  int lo = 0, hi = cnt;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (a[mid] < v) lo = mid + 1; else hi = mid;
  }
  return lo;
}

// # of sorted positions in the circular window [s, s+L) mod n
__device__ __forceinline__ int64_t count_in(const int64_t* E, int cnt, int64_t s, int64_t L, int64_t n) {
  if (cnt == 0 || L <= 0) return 0;
  if (s + L <= n) return lower_bound_i64(E, cnt, s + L) - lower_bound_i64(E, cnt, s);
  return (cnt - lower_bound_i64(E, cnt, s)) + lower_bound_i64(E, cnt, s + L - n);
}

// rows consumed and rows accepted by one query's walk (see the file comment)
__device__ __forceinline__ void walk_len(const int64_t* E, int cnt, int64_t s, int64_t n, int64_t m, int64_t* L_out,
                                         int64_t* taken_out) {
  if (cnt == 0) {
    const int64_t L = m < n ? m : n;
    *L_out = L;
    *taken_out = L;
    return;
  }
  const int64_t avail = n - cnt;
  if (avail < m) {  // one full pass, clamped (estimators.py:279, 300-303)
    *L_out = n;
    *taken_out = avail;
    return;
  }
  int64_t L = m;
  for (;;) {
    const int64_t e = count_in(E, cnt, s, L, n);
    if (L - e >= m) break;
    L = m + e;
  }
  *L_out = L;
  *taken_out = m;
}

// per query: original ids -> permuted positions (inverse permutation), sorted ascending
__global__ void map_sort_kernel(const int64_t* __restrict__ excl, int32_t stride, const int64_t* __restrict__ inverse,
                                int32_t B, int64_t* __restrict__ pos) {
  extern __shared__ long long sb[];
  const int64_t q = blockIdx.x;
  for (int i = threadIdx.x; i < B; i += blockDim.x)
    sb[i] = i < stride ? inverse[excl[size_t(q) * stride + i]] : LLONG_MAX;
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
  for (int i = threadIdx.x; i < stride; i += blockDim.x) pos[size_t(q) * stride + i] = sb[i];
}

// shared cursor: one thread threads the cursor through the batch in query order
__global__ void chain_kernel(const int64_t* __restrict__ pos, int32_t cnt, int64_t nq, int64_t n, int64_t m,
                             int64_t cursor_in, int64_t* __restrict__ start, int64_t* __restrict__ len,
                             int32_t* __restrict__ taken, int64_t* __restrict__ cursor_out) {
  if (blockIdx.x != 0 || threadIdx.x != 0) return;
  int64_t s = cursor_in;
  for (int64_t j = 0; j < nq; ++j) {
    int64_t L, t;
    walk_len(pos ? pos + size_t(j) * cnt : nullptr, pos ? cnt : 0, s, n, m, &L, &t);
    start[j] = s;
    len[j] = L;
    taken[j] = int32_t(t);
    s = (s + L) % n;
  }
  *cursor_out = s;
}

// independent cursors: query j starts at floor(j n / nq) (estimators.py:407-408)
__global__ void independent_kernel(const int64_t* __restrict__ pos, int32_t cnt, int64_t nq, int64_t n, int64_t m,
                                   int64_t* __restrict__ start, int64_t* __restrict__ len,
                                   int32_t* __restrict__ taken) {
  const int64_t j = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (j >= nq) return;
  const int64_t s = (j * n) / nq;
  int64_t L, t;
  walk_len(pos ? pos + size_t(j) * cnt : nullptr, pos ? cnt : 0, s, n, m, &L, &t);
  start[j] = s;
  len[j] = L;
  taken[j] = int32_t(t);
}

template <int G>
__device__ __forceinline__ double group_row(const float* __restrict__ x, const double* __restrict__ q, int d,
                                            int family, double c, int gl) {
  double acc = 0.0;
  if ((d & 3) == 0) {
    const float4* x4 = reinterpret_cast<const float4*>(x);
    for (int k4 = gl; k4 < (d >> 2); k4 += G) {
      const float4 v = __ldg(x4 + k4);
      const double t0 = double(v.x) - q[4 * k4 + 0], t1 = double(v.y) - q[4 * k4 + 1];
      const double t2 = double(v.z) - q[4 * k4 + 2], t3 = double(v.w) - q[4 * k4 + 3];
      if (family == DK_LAPLACIAN) acc += (fabs(t0) + fabs(t1)) + (fabs(t2) + fabs(t3));
      else { acc = fma(t0, t0, acc); acc = fma(t1, t1, acc); acc = fma(t2, t2, acc); acc = fma(t3, t3, acc); }
    }
  } else {
    for (int k = gl; k < d; k += G) {
      const double t = double(__ldg(x + k)) - q[k];
      acc = family == DK_LAPLACIAN ? acc + fabs(t) : fma(t, t, acc);
    }
  }
#pragma unroll
  for (int o = G / 2; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if (family == DK_EXPONENTIAL) acc = sqrt(acc);
  return exp(-acc * c);
}

// one warp per query walks its window; G lanes per row, R = 32/G rows per step
template <int G>
__global__ void rsp_eval_kernel(const float* __restrict__ X, int64_t n, int32_t d, const double* __restrict__ Q,
                                int64_t nq, int32_t family, double c, const int64_t* __restrict__ pos, int32_t cnt,
                                const int64_t* __restrict__ start, const int64_t* __restrict__ len,
                                double* __restrict__ z_sum) {
  extern __shared__ double sq[];
  constexpr int R = 32 / G;
  const int wib = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t j = int64_t(blockIdx.x) * (blockDim.x >> 5) + wib;
  if (j >= nq) return;
  double* q = sq + size_t(wib) * d;
  for (int k = lane; k < d; k += 32) q[k] = Q[size_t(j) * d + k];
  __syncwarp();
  const int64_t* E = pos ? pos + size_t(j) * cnt : nullptr;
  const int ecnt = pos ? cnt : 0;
  const int64_t s = start[j], L = len[j];
  const int grp = lane / G, gl = lane % G;
  double zsum = 0.0;
  for (int64_t w0 = 0; w0 < L; w0 += R) {
    const int64_t w = w0 + grp;
    int64_t row = s + w;
    if (row >= n) row -= n;
    bool ok = w < L;
    if (ok && ecnt) {
      const int i = lower_bound_i64(E, ecnt, row);
      ok = !(i < ecnt && E[i] == row);
    }
    const double v = group_row<G>(X + size_t(ok ? row : 0) * d, q, d, family, c, gl);
    if (ok && gl == 0) zsum += v;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) zsum += __shfl_xor_sync(0xffffffffu, zsum, o);
  if (lane == 0) z_sum[j] = zsum;
}

}  // namespace

void launch_rsp_map_sort(const int64_t* excl, int32_t stride, const int64_t* inverse, int64_t nq, int64_t* pos,
                         cudaStream_t s) {
  int B = 1;
  while (B < stride) B <<= 1;
  const size_t smem = size_t(B) * 8;
  set_dynamic_smem(map_sort_kernel, smem);
  map_sort_kernel<<<unsigned(nq), 256, smem, s>>>(excl, stride, inverse, B, pos);
  DK_CHECK_LAUNCH();
}

void launch_rsp_starts(const int64_t* pos, int32_t cnt, int64_t nq, int64_t n, int64_t m, int64_t cursor_in,
                       bool independent, int64_t* start, int64_t* len, int32_t* taken, int64_t* cursor_out,
                       cudaStream_t s) {
  if (independent) {
    independent_kernel<<<unsigned((nq + 127) / 128), 128, 0, s>>>(pos, cnt, nq, n, m, start, len, taken);
    DK_CHECK_LAUNCH();  // the shared cursor is untouched (the caller reports cursor_in)
  } else {
    chain_kernel<<<1, 32, 0, s>>>(pos, cnt, nq, n, m, cursor_in, start, len, taken, cursor_out);
    DK_CHECK_LAUNCH();
  }
}

void launch_rsp_eval(const float* X, int64_t n, int32_t d, const double* Q, int64_t nq, int32_t family,
                     double bandwidth, const int64_t* pos, int32_t cnt, const int64_t* start, const int64_t* len,
                     double* z_sum, cudaStream_t s) {
  const int wpb = int(std::max<int64_t>(1, std::min<int64_t>(8, 232448 / (int64_t(d) * 8))));
  const size_t smem = size_t(wpb) * d * sizeof(double);
  if (smem > 232448) throw Error{DK_EINVAL, "dimension too large for the permuted sampler (d > 29000)"};
  const double c = family == DK_GAUSSIAN ? 1.0 / (2.0 * bandwidth * bandwidth) : 1.0 / bandwidth;
  const unsigned grid = unsigned((nq + wpb - 1) / wpb);
  const int chunks = (d + 3) / 4;
#define DK_RSP_LAUNCH(G)                                                                                      \
  do {                                                                                                        \
    set_dynamic_smem(rsp_eval_kernel<G>, smem);                                                               \
    rsp_eval_kernel<G><<<grid, wpb * 32, smem, s>>>(X, n, d, Q, nq, family, c, pos, cnt, start, len, z_sum);  \
  } while (0)
  if (chunks >= 64) DK_RSP_LAUNCH(32);
  else if (chunks >= 32) DK_RSP_LAUNCH(16);
  else if (chunks >= 16) DK_RSP_LAUNCH(8);
  else if (chunks >= 8) DK_RSP_LAUNCH(4);
  else if (chunks >= 4) DK_RSP_LAUNCH(2);
  else DK_RSP_LAUNCH(1);
#undef DK_RSP_LAUNCH
  DK_CHECK_LAUNCH();
}

}  // namespace dk
