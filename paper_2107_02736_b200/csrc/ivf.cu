// ivf.cu — GPU inverted-file index: k-means build and probed scans.
//
// Reference: ann.py:124-316 (IvfIndex, _centroid_sqdists, _kmeans_pp_init,
// ivf_build, ivf_query, IvfAnnIndex).  The build keeps the reference's numpy
// PCG64 stream on the host (ivf.py drives k-means++ one centroid at a time and
// draws exactly what rng.integers / rng.choice draw); everything that touches
// the n rows runs here:
//   * k-means++ distances   closest_i = min(closest_i, sum_j (x_ij - c_j)^2)      fp64
//   * rng.choice(n, p)      searchsorted(cumsum(p) / cumsum(p)[-1], u, 'right')   fp64 scan
//   * Lloyd assignment      d2 = ((x.c) * -2 + |x|^2) + |c|^2, argmin (lower id on ties), fp64
//                           register-tiled over (64 rows x 64 centroids) tiles
//   * centroid update       members in increasing row order summed sequentially in fp64 /
//                           count — numpy's axis-0 mean — empty clusters keep their centroid
//   * inverted lists        stable radix sort of (label, row): rows cluster-contiguous in
//                           increasing id order = np.flatnonzero(labels == c); the fp32 rows
//                           are re-stored in that order so a probed list is one contiguous block
// Query (batched): per query the n_probe nearest centroids ((d2, id) order), then an
// exact fp64 scan of the probed lists with a shared-memory top-k ((d2, row) order,
// threshold-filtered), d2 = ((x.y) * -2 + |x|^2) + |y|^2 clamped at 0 (ann.py:224-229).
#include <algorithm>
#include <cmath>
#include <climits>
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_reduce.cuh>
#include <cub/device/device_scan.cuh>
#include <cub/device/device_segmented_radix_sort.cuh>

#include <type_traits>

#include "internal.h"
#include "ptx.cuh"

struct dk_ivf {
  dk_dataset* ds = nullptr;
  int32_t C = 0, d = 0;
  int64_t n = 0;
  double* cent = nullptr;        // [C][d]
  double* cnorm = nullptr;       // [C]
  double* closest = nullptr;     // [n]  k-means++ D^2
  double* cdf = nullptr;         // [n]
  int32_t* labels = nullptr;     // [n]
  int32_t* labels_s = nullptr;   // [n] sorted
  int64_t* ids = nullptr;        // [n] 0..n-1
  int64_t* rows = nullptr;       // [n] cluster-sorted row ids
  int64_t* offsets = nullptr;    // [C + 1]
  double* d2min = nullptr;       // [n]
  float* xs = nullptr;           // [n][d] rows in list order
  double* xns = nullptr;         // [n] |x|^2 in list order
  double* scal = nullptr;        // device scalars
  void* temp = nullptr;          // CUB scratch
  size_t temp_bytes = 0;
  void* keys1 = nullptr;         // query scratch: phase-1 (d2, row) keys, grow-only
  size_t keys1_bytes = 0;
  void* ckeys = nullptr;         // query scratch: centroid distance keys [queries][C], grow-only
  size_t ckeys_bytes = 0;
  void* dws = nullptr;           // dk_deann_ivf scratch, grow-only
  size_t dws_bytes = 0;
  bool lists = false;
};

namespace dk {
namespace {

struct K128 {
  unsigned long long hi, lo;
};
__device__ __forceinline__ bool k_less(const K128& a, const K128& b) {
  return a.hi < b.hi || (a.hi == b.hi && a.lo < b.lo);
}
__device__ void bitonic(K128* buf, int B) {
  for (int k = 2; k <= B; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      __syncthreads();
      for (int i = threadIdx.x; i < B; i += blockDim.x) {
        const int ixj = i ^ j;
        if (ixj > i) {
          const bool up = (i & k) == 0;
          const K128 a = buf[i], b = buf[ixj];
          if (k_less(b, a) == up) { buf[i] = b; buf[ixj] = a; }
        }
      }
    }
  }
  __syncthreads();
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// ---------------------------------------------------------------- build

__global__ void set_row_kernel(const float* __restrict__ X, int64_t row, int32_t d, double* __restrict__ c) {
  for (int j = threadIdx.x; j < d; j += blockDim.x) c[j] = double(X[row * d + j]);
}

// k-means++ D^2 update (ann.py:157-168): warp per row, direct difference in fp64
__global__ void pp_dist_kernel(const float* __restrict__ X, int64_t n, int32_t d, const double* __restrict__ c,
                               int init, double* __restrict__ closest) {
  const int64_t row = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (row >= n) return;
  const float* x = X + row * d;
  double s = 0.0;
  for (int j = lane; j < d; j += 32) {
    const double t = double(x[j]) - c[j];
    s = fma(t, t, s);
  }
  s = warp_sum(s);
  if (lane == 0) closest[row] = init ? s : fmin(closest[row], s);
}

__global__ void div_kernel(const double* __restrict__ a, int64_t n, double total, double* __restrict__ out) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) out[i] = a[i] / total;
}

// first i with cdf[i] / cdf[n-1] > u (numpy searchsorted side='right' on the normalised cdf)
__global__ void search_kernel(const double* __restrict__ cdf, int64_t n, double u, int64_t* __restrict__ out) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double last = cdf[n - 1];
  const bool here = cdf[i] / last > u;
  const bool before = i > 0 && cdf[i - 1] / last > u;
  if (here && !before) *out = i;
}

__global__ void cnorm_kernel(const double* __restrict__ cent, int32_t C, int32_t d, double* __restrict__ cn) {
  const int c = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (c >= C) return;
  double s = 0.0;
  for (int j = lane; j < d; j += 32) s = fma(cent[size_t(c) * d + j], cent[size_t(c) * d + j], s);
  s = warp_sum(s);
  if (lane == 0) cn[c] = s;
}

// Lloyd assignment (ann.py:142-149, 187-189): 64 rows x 64 centroids per tile, 4 x 4 fp64
// accumulators per thread, K staged through shared memory in chunks of 16.
constexpr int AM = 64, AN = 64, AK = 16;
__global__ __launch_bounds__(256) void assign_kernel(const float* __restrict__ X, const double* __restrict__ xn,
                                                     int64_t n, int32_t d, const double* __restrict__ cent,
                                                     const double* __restrict__ cn, int32_t C,
                                                     int32_t* __restrict__ labels, double* __restrict__ d2min) {
  __shared__ double xsm[AK][AM + 2];
  __shared__ __align__(16) double csm[AK][AN];
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  const int64_t row0 = int64_t(blockIdx.x) * AM;
  double best[4];
  int bidx[4];
  double xnr[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    best[i] = __longlong_as_double(0x7ff0000000000000ll);
    bidx[i] = 0;
    const int64_t r = row0 + ty * 4 + i;
    xnr[i] = r < n ? xn[r] : 0.0;
  }
  for (int c0 = 0; c0 < C; c0 += AN) {
    double acc[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[i][j] = 0.0;
    for (int k0 = 0; k0 < d; k0 += AK) {
      for (int e = threadIdx.x; e < AM * AK; e += 256) {
        const int r = e / AK, kk = e % AK;
        const int64_t row = row0 + r;
        xsm[kk][r] = (row < n && k0 + kk < d) ? double(X[row * d + k0 + kk]) : 0.0;
      }
      for (int e = threadIdx.x; e < AN * AK; e += 256) {
        const int cc = e / AK, kk = e % AK;
        const int c = c0 + cc;
        csm[kk][cc] = (c < C && k0 + kk < d) ? cent[size_t(c) * d + k0 + kk] : 0.0;
      }
      __syncthreads();
#pragma unroll
      for (int kk = 0; kk < AK; ++kk) {
        double a[4], b[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) a[i] = xsm[kk][ty * 4 + i];
        const double2 b01 = *reinterpret_cast<const double2*>(&csm[kk][tx * 4]);
        const double2 b23 = *reinterpret_cast<const double2*>(&csm[kk][tx * 4 + 2]);
        b[0] = b01.x; b[1] = b01.y; b[2] = b23.x; b[3] = b23.y;
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) acc[i][j] = fma(a[i], b[j], acc[i][j]);
      }
      __syncthreads();
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int c = c0 + tx * 4 + j;
      if (c < C) {
        const double cnc = cn[c];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          double t = acc[i][j] * -2.0;
          t += xnr[i];
          t += cnc;
          t = fmax(t, 0.0);
          if (t < best[i]) { best[i] = t; bidx[i] = c; }
        }
      }
    }
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
#pragma unroll
    for (int o = 8; o > 0; o >>= 1) {
      const double ob = __shfl_xor_sync(0xffffffffu, best[i], o);
      const int oi = __shfl_xor_sync(0xffffffffu, bidx[i], o);
      if (ob < best[i] || (ob == best[i] && oi < bidx[i])) { best[i] = ob; bidx[i] = oi; }
    }
    const int64_t r = row0 + ty * 4 + i;
    if (tx == 0 && r < n) {
      labels[r] = bidx[i];
      d2min[r] = best[i];
    }
  }
}

__global__ void iota_kernel(int64_t* __restrict__ a, int64_t n) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) a[i] = i;
}

// offsets[c] = first position of label c in the sorted labels (c = 0..C)
__global__ void offsets_kernel(const int32_t* __restrict__ ls, int64_t n, int32_t C, int64_t* __restrict__ off) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c > C) return;
  int64_t lo = 0, hi = n;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (ls[mid] < c) lo = mid + 1; else hi = mid;
  }
  off[c] = lo;
}

// centroid c, dims j: sequential fp64 sum over members in increasing row order, / count
// (numpy's x64[labels == c].mean(axis=0)); empty clusters keep their centroid (ann.py:191-193)
__global__ void update_kernel(const float* __restrict__ X, int32_t d, const int64_t* __restrict__ rows,
                              const int64_t* __restrict__ off, int32_t C, double* __restrict__ cent) {
  const int c = blockIdx.x;
  const int j = blockIdx.y * blockDim.x + threadIdx.x;
  if (c >= C || j >= d) return;
  const int64_t b = off[c], e = off[c + 1];
  if (e == b) return;
  double acc = 0.0;
  int64_t m = b;
  for (; m + 4 <= e; m += 4) {
    const int64_t r0 = rows[m], r1 = rows[m + 1], r2 = rows[m + 2], r3 = rows[m + 3];
    const float v0 = X[r0 * d + j], v1 = X[r1 * d + j], v2 = X[r2 * d + j], v3 = X[r3 * d + j];
    acc += double(v0);
    acc += double(v1);
    acc += double(v2);
    acc += double(v3);
  }
  for (; m < e; ++m) acc += double(X[rows[m] * d + j]);
  cent[size_t(c) * d + j] = acc / double(e - b);
}

__global__ void gather_rows_kernel(const float* __restrict__ X, const double* __restrict__ xn, int32_t d,
                                   const int64_t* __restrict__ rows, int64_t n, float* __restrict__ xs,
                                   double* __restrict__ xns) {
  const int64_t p = blockIdx.x;
  if (p >= n) return;
  const int64_t r = rows[p];
  for (int j = threadIdx.x; j < d; j += blockDim.x) xs[p * d + j] = X[r * d + j];
  if (threadIdx.x == 0) xns[p] = xn[r];
}

// ---------------------------------------------------------------- query

// Exact scan of the probed lists with a (d2, row) top-k in shared memory.  Rounds of
// S rows: G lanes per row (float4 loads, fp64 FMA, G-lane shuffle reduction), rows
// beating the current k-th key are staged, and a bitonic merge of [top | stage]
// keeps the k smallest.  d2 = ((x.y) * -2 + |x|^2) + |y|^2 clamped at 0.
template <int G, int IT>
__global__ void __launch_bounds__(256) scan_kernel(const float* __restrict__ xs, const double* __restrict__ xns,
                                                   const int64_t* __restrict__ rows, const int64_t* __restrict__ off,
                                                   int32_t d, const int32_t* __restrict__ order,
                                                   const double* __restrict__ Q,
                                                   const int32_t* __restrict__ probe, int32_t n_probe,
                                                   const int32_t* __restrict__ np_q, int32_t k,
                                                   int32_t Kp, int32_t S, int32_t B, int64_t* __restrict__ idx_out,
                                                   double* __restrict__ d2_out, int32_t* __restrict__ cnt_out) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  K128* top = reinterpret_cast<K128*>(smem_raw);  // [B]: sorted top Kp, then the stage of S
  double* y = reinterpret_cast<double*>(top + B);
  __shared__ int s_cnt;
  __shared__ double s_yy;
  constexpr int RPW = 32 / G;  // rows per warp step
  // blocks take the queries grouped by their nearest list, so concurrently running blocks
  // stream the same lists through L2
  const int64_t q = order ? order[blockIdx.x] : blockIdx.x;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  const int grp = lane / G, gl = lane % G;
  for (int j = threadIdx.x; j < d; j += blockDim.x) y[j] = Q[q * d + j];
  for (int i = threadIdx.x; i < B; i += blockDim.x) top[i] = K128{~0ull, ~0ull};
  if (threadIdx.x == 0) s_cnt = 0;
  __syncthreads();
  if (warp == 0) {
    double sy = 0.0;
    for (int j = lane; j < d; j += 32) sy = fma(y[j], y[j], sy);
    sy = warp_sum(sy);
    if (lane == 0) s_yy = sy;
  }
  __syncthreads();
  const double yy = s_yy;
  const bool vec = (d & 3) == 0;
  // IT > 0: this lane's slice of the query in registers (no per-row shared-memory reads)
  double yv[IT > 0 ? IT : 1][4];
  if constexpr (IT > 0) {
#pragma unroll
    for (int it = 0; it < IT; ++it) {
      const int j4 = gl + it * G;
#pragma unroll
      for (int i = 0; i < 4; ++i) yv[it][i] = j4 < (d >> 2) ? y[4 * j4 + i] : 0.0;
    }
  }
  int64_t total = 0;
  const int np = np_q ? np_q[q] : n_probe;  // np_q: scan only the leading probed lists
  for (int p = 0; p < np; ++p) {
    const int c = probe[q * n_probe + p];
    const int64_t b = off[c], e = off[c + 1];
    total += e - b;
    for (int64_t r0 = b; r0 < e; r0 += S) {
      const K128 tau = top[Kp - 1];
      const int64_t r1 = min(e, r0 + S);
      for (int64_t base = r0 + int64_t(warp) * RPW; base < r1; base += int64_t(nw) * RPW) {
        const int64_t pos = base + grp;
        const bool ok = pos < r1;
        const float* x = xs + (ok ? pos : b) * d;
        double s = 0.0;
        if constexpr (IT > 0) {
          const float4* x4 = reinterpret_cast<const float4*>(x);
#pragma unroll
          for (int it = 0; it < IT; ++it) {
            const int j4 = gl + it * G;
            if (j4 < (d >> 2)) {
              const float4 v = __ldg(x4 + j4);
              s = fma(double(v.x), yv[it][0], s);
              s = fma(double(v.y), yv[it][1], s);
              s = fma(double(v.z), yv[it][2], s);
              s = fma(double(v.w), yv[it][3], s);
            }
          }
        } else if (vec) {
          const float4* x4 = reinterpret_cast<const float4*>(x);
          for (int j4 = gl; j4 < (d >> 2); j4 += G) {
            const float4 v = __ldg(x4 + j4);
            s = fma(double(v.x), y[4 * j4 + 0], s);
            s = fma(double(v.y), y[4 * j4 + 1], s);
            s = fma(double(v.z), y[4 * j4 + 2], s);
            s = fma(double(v.w), y[4 * j4 + 3], s);
          }
        } else {
          for (int j = gl; j < d; j += G) s = fma(double(__ldg(x + j)), y[j], s);
        }
#pragma unroll
        for (int o = G / 2; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if (ok && gl == 0) {
          double t = s * -2.0;
          t += xns[pos];
          t += yy;
          t = fmax(t, 0.0);
          const K128 key{static_cast<unsigned long long>(__double_as_longlong(t)),
                         static_cast<unsigned long long>(rows[pos])};
          if (k_less(key, tau)) top[Kp + atomicAdd(&s_cnt, 1)] = key;
        }
      }
      __syncthreads();
      if (s_cnt > 0) {
        bitonic(top, B);
        for (int i = Kp + threadIdx.x; i < B; i += blockDim.x) top[i] = K128{~0ull, ~0ull};
        if (threadIdx.x == 0) s_cnt = 0;
        __syncthreads();
      }
    }
  }
  const int cnt = int(total < int64_t(k) ? total : int64_t(k));
  for (int i = threadIdx.x; i < k; i += blockDim.x) {
    const bool ok = i < cnt;
    idx_out[q * k + i] = ok ? static_cast<int64_t>(top[i].lo) : -1;
    d2_out[q * k + i] = ok ? __longlong_as_double(static_cast<long long>(top[i].hi))
                           : __longlong_as_double(0x7ff0000000000000ll);
  }
  if (threadIdx.x == 0) cnt_out[q] = cnt;
}

__global__ void first_probe_kernel(const int32_t* __restrict__ probe, int64_t nq, int32_t n_probe,
                                   int32_t* __restrict__ key, int32_t* __restrict__ val) {
  const int64_t q = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (q >= nq) return;
  key[q] = probe[q * n_probe];
  val[q] = int32_t(q);
}

// ---- large k (> 4096, beyond the shared-memory top-k): every probed candidate's exact
// (d2, row) pair, then a stable two-pass segmented radix sort (row id, then d2) per query
__global__ void probe_total_kernel(const int32_t* __restrict__ probe, const int64_t* __restrict__ off, int64_t nq,
                                   int32_t n_probe, int64_t* __restrict__ tot) {
  const int64_t q = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (q >= nq) return;
  int64_t t = 0;
  for (int p = 0; p < n_probe; ++p) {
    const int c = probe[q * n_probe + p];
    t += off[c + 1] - off[c];
  }
  tot[q] = t;
}

__global__ void gather_cands_kernel(const float* __restrict__ xs, const double* __restrict__ xns,
                                    const int64_t* __restrict__ rows, const int64_t* __restrict__ off, int32_t d,
                                    const double* __restrict__ Q, const int32_t* __restrict__ probe, int32_t n_probe,
                                    int64_t q0, const int64_t* __restrict__ seg, unsigned long long* __restrict__ key,
                                    unsigned long long* __restrict__ val) {
  extern __shared__ double y[];
  __shared__ double s_yy;
  const int64_t q = q0 + blockIdx.x;
  for (int j = threadIdx.x; j < d; j += blockDim.x) y[j] = Q[q * d + j];
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int j = 0; j < d; ++j) t = fma(y[j], y[j], t);
    s_yy = t;
  }
  __syncthreads();
  const double yy = s_yy;
  int64_t o = seg[blockIdx.x];
  for (int p = 0; p < n_probe; ++p) {
    const int c = probe[q * n_probe + p];
    const int64_t b = off[c], e = off[c + 1];
    for (int64_t pos = b + threadIdx.x; pos < e; pos += blockDim.x) {
      const float* x = xs + pos * d;
      double dot = 0.0;
      for (int j = 0; j < d; ++j) dot = fma(double(x[j]), y[j], dot);
      double t = dot * -2.0;
      t += xns[pos];
      t += yy;
      t = fmax(t, 0.0);
      key[o + (pos - b)] = static_cast<unsigned long long>(rows[pos]);
      val[o + (pos - b)] = static_cast<unsigned long long>(__double_as_longlong(t));
    }
    o += e - b;
  }
}

__global__ void take_cands_kernel(const unsigned long long* __restrict__ d2bits,
                                  const unsigned long long* __restrict__ ids, const int64_t* __restrict__ seg,
                                  int64_t q0, int64_t nqc, int32_t k, int64_t* __restrict__ idx_out,
                                  double* __restrict__ d2_out, int32_t* __restrict__ cnt_out) {
  const int64_t qi = blockIdx.x;
  if (qi >= nqc) return;
  const int64_t b = seg[qi], e = seg[qi + 1];
  const int64_t cnt = min(int64_t(k), e - b);
  const int64_t q = q0 + qi;
  for (int i = threadIdx.x; i < k; i += blockDim.x) {
    const bool ok = i < cnt;
    idx_out[q * k + i] = ok ? static_cast<int64_t>(ids[b + i]) : -1;
    d2_out[q * k + i] = ok ? __longlong_as_double(static_cast<long long>(d2bits[b + i]))
                           : __longlong_as_double(0x7ff0000000000000ll);
  }
  if (threadIdx.x == 0) cnt_out[q] = int32_t(cnt);
}

struct DevBuf {
  void* p = nullptr;
  explicit DevBuf(size_t bytes) { DK_CUDA(cudaMalloc(&p, std::max<size_t>(bytes, 16))); }
  ~DevBuf() {
    if (p) cudaFree(p);
  }
  template <class T>
  T* as(size_t byte_off = 0) const {
    return reinterpret_cast<T*>(static_cast<uint8_t*>(p) + byte_off);
  }
};

// Queries in chunks of <= 2^26 candidates (the reference accepts any k >= 1, ann.py:208-209).
void ivf_query_bigk(dk_ivf* v, const double* Qd, int64_t nq, int32_t k, int32_t n_probe, const int32_t* probe,
                    int64_t* io, double* dd, int32_t* co, cudaStream_t s) {
  DevBuf totb(size_t(nq) * 8);
  probe_total_kernel<<<unsigned((nq + 255) / 256), 256, 0, s>>>(probe, v->offsets, nq, n_probe,
                                                                totb.as<int64_t>());
  DK_CHECK_LAUNCH();
  std::vector<int64_t> tot(static_cast<size_t>(nq));
  DK_CUDA(cudaMemcpyAsync(tot.data(), totb.p, size_t(nq) * 8, cudaMemcpyDeviceToHost, s));
  DK_CUDA(cudaStreamSynchronize(s));
  const int64_t cap = int64_t(1) << 26;
  const size_t smem = size_t(v->d) * sizeof(double);
  set_dynamic_smem(gather_cands_kernel, smem);
  int64_t q0 = 0;
  while (q0 < nq) {
    int64_t q1 = q0, T = 0;
    while (q1 < nq && (q1 == q0 || T + tot[size_t(q1)] <= cap)) T += tot[size_t(q1++)];
    DK_REQUIRE(T < (int64_t(1) << 31), "too many IVF candidates for one query");
    const int64_t nqc = q1 - q0;
    std::vector<int64_t> seg(static_cast<size_t>(nqc) + 1, 0);
    for (int64_t i = 0; i < nqc; ++i) seg[size_t(i) + 1] = seg[size_t(i)] + tot[size_t(q0 + i)];
    size_t sort_bytes = 0;
    cub::DeviceSegmentedRadixSort::SortPairs(nullptr, sort_bytes, static_cast<const unsigned long long*>(nullptr),
                                             static_cast<unsigned long long*>(nullptr),
                                             static_cast<const unsigned long long*>(nullptr),
                                             static_cast<unsigned long long*>(nullptr), int(T), int(nqc),
                                             static_cast<const int64_t*>(nullptr),
                                             static_cast<const int64_t*>(nullptr));
    const size_t eT = size_t(std::max<int64_t>(T, 1)) * 8;
    DevBuf buf(4 * eT + size_t(nqc + 1) * 8 + sort_bytes + 256);
    auto* k0 = buf.as<unsigned long long>(0);
    auto* v0 = buf.as<unsigned long long>(eT);
    auto* k1 = buf.as<unsigned long long>(2 * eT);
    auto* v1 = buf.as<unsigned long long>(3 * eT);
    auto* segd = buf.as<int64_t>(4 * eT);
    void* tmp = buf.as<uint8_t>((4 * eT + size_t(nqc + 1) * 8 + 255) & ~size_t(255));
    DK_CUDA(cudaMemcpyAsync(segd, seg.data(), seg.size() * 8, cudaMemcpyHostToDevice, s));
    gather_cands_kernel<<<unsigned(nqc), 128, smem, s>>>(v->xs, v->xns, v->rows, v->offsets, v->d, Qd, probe,
                                                         n_probe, q0, segd, k0, v0);
    DK_CHECK_LAUNCH();
    size_t tb = sort_bytes;  // pass 1: by row id (keys k0 = ids), pass 2 (stable): by d2
    DK_CUDA(cub::DeviceSegmentedRadixSort::SortPairs(tmp, tb, k0, k1, v0, v1, int(T), int(nqc), segd, segd + 1,
                                                     0, 64, s));
    tb = sort_bytes;
    DK_CUDA(cub::DeviceSegmentedRadixSort::SortPairs(tmp, tb, v1, v0, k1, k0, int(T), int(nqc), segd, segd + 1,
                                                     0, 64, s));
    take_cands_kernel<<<unsigned(nqc), 128, 0, s>>>(v0, k0, segd, q0, nqc, k, io, dd, co);
    DK_CHECK_LAUNCH();
    DK_CUDA(cudaStreamSynchronize(s));  // buffers are freed at the end of the chunk
    q0 = q1;
  }
}

// ---- n_clusters beyond the shared-memory probe sort (> 8192): all centroid distances of a
// query chunk, one stable segmented radix sort by the order-preserving key (ties keep the
// lower centroid id), first n_probe taken
__global__ void centroid_keys_kernel(const double* __restrict__ Q, int32_t d, const double* __restrict__ cent,
                                     const double* __restrict__ cn, int32_t C, int64_t q0, int32_t formula,
                                     unsigned long long* __restrict__ key, int32_t* __restrict__ val) {
  const int64_t qi = blockIdx.y;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int c = blockIdx.x * (blockDim.x >> 5) + warp;
  if (c >= C) return;
  const double* y = Q + (q0 + qi) * d;
  const double* cc = cent + size_t(c) * d;
  double sacc = 0.0;
  if (formula == 0) {
    for (int j = lane; j < d; j += 32) {
      const double t = cc[j] - y[j];
      sacc = fma(t, t, sacc);
    }
    sacc = warp_sum(sacc);
  } else {
    for (int j = lane; j < d; j += 32) sacc = fma(cc[j], y[j], sacc);
    sacc = warp_sum(sacc);
    sacc = sacc * -2.0 + cn[c];
  }
  if (lane == 0) {
    const unsigned long long b = static_cast<unsigned long long>(__double_as_longlong(sacc));
    key[qi * C + c] = (b >> 63) ? ~b : (b | 0x8000000000000000ull);
    val[qi * C + c] = c;
  }
}

__global__ void take_probe_kernel(const int32_t* __restrict__ sval, int32_t C, int64_t q0, int64_t nqc,
                                  int32_t n_probe, int32_t* __restrict__ probe) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= nqc * n_probe) return;
  const int64_t qi = i / n_probe, p = i % n_probe;
  probe[(q0 + qi) * n_probe + p] = sval[qi * C + p];
}

// Probe: the n_probe nearest centroids per query in (distance, id) order.  formula 0:
// sum (c - y)^2 (ivf_query, ann.py:212-214); formula 1: (C y) * -2 + |c|^2
// (IvfAnnIndex._probe_clusters, ann.py:262-275).
// Tiled: every (query, centroid) distance of a query chunk as an order-preserving key
// (32 queries x 128 centroids per block, staged 16 dimensions at a time, each distance the
// sequential fma chain over j), then the n_probe smallest (key, centroid id) per query.
constexpr int CQ = 32, CW = 8, CR = 4, CRC = 32 * CR, CDJ = 16;

__device__ __forceinline__ unsigned long long order_key(double v) {  // signed double -> ordered bits
  const unsigned long long b = static_cast<unsigned long long>(__double_as_longlong(v));
  return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}

template <int FORMULA>
__global__ void __launch_bounds__(128) centroid_tile_kernel(const double* __restrict__ Q, int64_t q0, int64_t nqc,
                                                            int32_t d, const double* __restrict__ cent,
                                                            const double* __restrict__ cn, int32_t C,
                                                            unsigned long long* __restrict__ keys) {
  __shared__ double cr[CRC * (CDJ + 1)];
  __shared__ double ys[CQ * CDJ];
  const int c0 = blockIdx.x * CRC;
  const int64_t qb = int64_t(blockIdx.y) * CQ;  // within the chunk
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double acc[CW][CR];
#pragma unroll
  for (int t = 0; t < CW; ++t)
#pragma unroll
    for (int i = 0; i < CR; ++i) acc[t][i] = 0.0;
  for (int j0 = 0; j0 < d; j0 += CDJ) {
    const int dj = min(CDJ, d - j0);
    __syncthreads();
#pragma unroll
    for (int u = 0; u < CRC * CDJ / 128; ++u) {
      const int t = threadIdx.x + 128 * u, r = t / CDJ, jj = t % CDJ;
      cr[r * (CDJ + 1) + jj] = (c0 + r < C && jj < dj) ? cent[int64_t(c0 + r) * d + j0 + jj] : 0.0;
    }
#pragma unroll
    for (int u = 0; u < CQ * CDJ / 128; ++u) {
      const int t = threadIdx.x + 128 * u, qq = t / CDJ, jj = t % CDJ;
      ys[t] = (qb + qq < nqc && jj < dj) ? Q[(q0 + qb + qq) * d + j0 + jj] : 0.0;
    }
    __syncthreads();
    for (int jj = 0; jj < dj; ++jj) {
      double y[CW], x[CR];
#pragma unroll
      for (int t = 0; t < CW; ++t) y[t] = ys[(warp * CW + t) * CDJ + jj];
#pragma unroll
      for (int i = 0; i < CR; ++i) x[i] = cr[(lane + 32 * i) * (CDJ + 1) + jj];
#pragma unroll
      for (int t = 0; t < CW; ++t)
#pragma unroll
        for (int i = 0; i < CR; ++i) {
          if (FORMULA == 0) {
            const double df = x[i] - y[t];
            acc[t][i] = fma(df, df, acc[t][i]);
          } else {
            acc[t][i] = fma(x[i], y[t], acc[t][i]);
          }
        }
    }
  }
#pragma unroll
  for (int t = 0; t < CW; ++t) {
    const int64_t qq = qb + warp * CW + t;
    if (qq >= nqc) continue;
#pragma unroll
    for (int i = 0; i < CR; ++i) {
      const int c = c0 + lane + 32 * i;
      if (c >= C) continue;
      const double v = FORMULA == 0 ? acc[t][i] : acc[t][i] * -2.0 + cn[c];
      keys[qq * C + c] = order_key(v);
    }
  }
}

// n_probe <= 64: warp per query, n_probe rounds of "smallest (key, id) above the previous one"
__global__ void probe_select_kernel(const unsigned long long* __restrict__ keys, int64_t q0, int64_t nqc,
                                    int32_t C, int32_t n_probe, int32_t* __restrict__ probe) {
  const int64_t qq = int64_t(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (qq >= nqc) return;
  const unsigned long long* kq = keys + qq * C;
  unsigned long long pk = 0ull;
  int pc = -1;
  for (int r = 0; r < n_probe; ++r) {
    unsigned long long bk = ~0ull;
    int bc = INT_MAX;
    for (int c = lane; c < C; c += 32) {
      const unsigned long long kv = kq[c];
      const bool above = kv > pk || (kv == pk && c > pc);
      if (above && (kv < bk || (kv == bk && c < bc))) {
        bk = kv;
        bc = c;
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const unsigned long long ok = __shfl_xor_sync(0xffffffffu, bk, o);
      const int oc = __shfl_xor_sync(0xffffffffu, bc, o);
      if (ok < bk || (ok == bk && oc < bc)) {
        bk = ok;
        bc = oc;
      }
    }
    if (lane == 0) probe[(q0 + qq) * n_probe + r] = bc;
    pk = bk;
    pc = bc;
  }
}

// n_probe > 64: block per query, bitonic over pow2(C) (key, id) pairs
__global__ void probe_sort_kernel(const unsigned long long* __restrict__ keys, int64_t q0, int32_t C, int32_t Bc,
                                  int32_t n_probe, int32_t* __restrict__ probe) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  K128* buf = reinterpret_cast<K128*>(smem_raw);
  const int64_t qq = blockIdx.x;
  for (int c = threadIdx.x; c < Bc; c += blockDim.x)
    buf[c] = c < C ? K128{keys[qq * C + c], static_cast<unsigned long long>(c)} : K128{~0ull, ~0ull};
  bitonic(buf, Bc);
  for (int i = threadIdx.x; i < n_probe; i += blockDim.x) probe[(q0 + qq) * n_probe + i] = int32_t(buf[i].lo);
}

__global__ void seg_starts_kernel(int64_t nqc, int32_t C, int64_t* __restrict__ seg) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i <= nqc) seg[i] = i * C;
}

// ---- two-phase probed k-NN (the default path):
//  (1) per query, its nearest probed lists until they hold >= k rows: every (d2, row) key of
//      those rows (list-major, pair_tile_kernel<0>), then their exact top-k (seg_topk_kernel)
//      -> tau_q = that k-th key, an upper bound on the query's true k-th key over all its
//      probed lists;
//  (2) the remaining (list, query) pairs, list-major: keys < tau_q are appended to the
//      query's candidate buffer (pair_tile_kernel<1>);
//  (3) per query: top-k of (phase-1 top-k + appended keys) by (d2, row) (seg_topk_kernel).
// Queries whose candidate buffer overflows are redone exactly, one block per (query, list).
__global__ void prefix_probes_kernel(const int32_t* __restrict__ probe, const int64_t* __restrict__ off,
                                     int64_t nq, int32_t n_probe, int32_t k, int32_t* __restrict__ np_q,
                                     int32_t* __restrict__ cnt_all, int64_t* __restrict__ rows1) {
  const int64_t q = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (q >= nq) return;
  int64_t all = 0, r1 = 0;
  int p1 = n_probe;
  for (int p = 0; p < n_probe; ++p) {
    const int c = probe[q * n_probe + p];
    all += off[c + 1] - off[c];
    if (p1 == n_probe && all >= k) {
      p1 = p + 1;
      r1 = all;
    }
  }
  if (p1 == n_probe) r1 = all;
  np_q[q] = p1;
  cnt_all[q] = int32_t(all < k ? all : k);
  rows1[q] = r1;
  if (q == nq - 1) rows1[nq] = 0;
}

__global__ void list_pairs_kernel(const int32_t* __restrict__ skey, int64_t npairs, int32_t C,
                                  int64_t* __restrict__ pstart) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c > C) return;
  int64_t lo = 0, hi = npairs;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (skey[mid] < c) lo = mid + 1; else hi = mid;
  }
  pstart[c] = lo;
}

// items of bucket b (list b for b < C, list b - C - 1 for b > C): query groups x row spans
// of `span` rows (long lists are split so no item trails)
__global__ void list_items_kernel(const int64_t* __restrict__ pstart, const int64_t* __restrict__ off, int32_t C,
                                  int32_t nb, int32_t per, int32_t span, int64_t* __restrict__ nitems) {
  const int bk = blockIdx.x * blockDim.x + threadIdx.x;
  if (bk > nb) return;
  const int c = bk < C ? bk : bk - C - 1;
  if (bk == nb || bk == C || c >= C) {
    nitems[bk] = 0;
    return;
  }
  const int64_t ns = (off[c + 1] - off[c] + span - 1) / span;
  nitems[bk] = (pstart[bk + 1] - pstart[bk] + per - 1) / per * ns;
}

// ---- tiled list-major pass (both phases): a work item is one list and up to PQ = 32 of the
// (query, list) pairs that probe it.  4 warps x 8 queries; lane = 4 rows of a 128-row chunk.
// Rows (as fp64) and query slices are staged DJ = 16 dimensions at a time, so every staged x
// value feeds 8 fp64 FMAs and every broadcast query value 4, and the dot product of each
// (query, row) is the same sequential fma chain over j = 0..d-1 as gather_cands_kernel.
//   MODE 0 (phase 1): every key of the pair is written to the query's key segment.
//   MODE 1 (phase 2): keys < tau_q are appended to the query's candidate buffer.
constexpr int PQ = 32, PW = 8, PR = 4, PRC = 32 * PR, PDJ = 16;

__global__ void query_norms_kernel(const double* __restrict__ Q, int64_t nq, int32_t d, double* __restrict__ yy) {
  const int64_t q = int64_t(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (q >= nq) return;
  double sy = 0.0;  // the order of scan_kernel
  for (int j = lane; j < d; j += 32) sy = fma(Q[q * d + j], Q[q * d + j], sy);
  sy = warp_sum(sy);
  if (lane == 0) yy[q] = sy;
}

// bucket b < nb: (list b, phase 1); bucket nb + 1 + c: (list c, phase 2); pairs sorted by bucket
__global__ void bucket_pairs_kernel(const int32_t* __restrict__ probe, const int32_t* __restrict__ np_q, int64_t nq,
                                    int32_t n_probe, int32_t C, int32_t* __restrict__ key,
                                    int32_t* __restrict__ val) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= nq * n_probe) return;
  const int64_t q = i / n_probe;
  const int slot = int(i % n_probe);
  key[i] = slot < np_q[q] ? probe[i] : C + 1 + probe[i];
  val[i] = int32_t(i);
}

template <int MODE>
__global__ void __launch_bounds__(128) pair_tile_kernel(
    const float* __restrict__ xs, const double* __restrict__ xns, const int64_t* __restrict__ rows,
    const int64_t* __restrict__ off, int32_t d, int32_t C, const double* __restrict__ Q,
    const double* __restrict__ yyq, const int32_t* __restrict__ probe, int32_t n_probe,
    const int32_t* __restrict__ sval, const int64_t* __restrict__ pstart, const int64_t* __restrict__ istart,
    int32_t blo, int32_t bhi, int32_t span, const int64_t* __restrict__ qoff, K128* __restrict__ keys,
    const K128* __restrict__ tau, int32_t cap, K128* __restrict__ cand, int32_t* __restrict__ ccnt) {
  __shared__ double xr[PRC * (PDJ + 1)];
  __shared__ double ys[PQ * PDJ];
  __shared__ int64_t s_q[PQ], s_pos[PQ], s_base[PQ];
  __shared__ double s_yy[PQ];
  __shared__ K128 s_tau[PQ];
  const int64_t i0 = istart[blo], item = i0 + blockIdx.x;
  if (item >= istart[bhi]) return;
  int lo = blo, hi = bhi - 1;  // bucket: istart[b] <= item < istart[b + 1]
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (istart[mid] <= item) lo = mid; else hi = mid - 1;
  }
  const int bkt = lo;
  // MODE 0 / 2: phase-1 buckets (every key written); MODE 1 / 3: phase-2 buckets (keys below tau_q
  // appended).  MODE 2 / 3 rank like IvfAnnIndex (fp32 keys), MODE 0 / 1 exactly (fp64)
  constexpr bool kF32 = MODE >= 2;
  constexpr bool kFilter = MODE == 1 || MODE == 3;
  const int c = kFilter ? bkt - C - 1 : bkt;
  // item = (query group, row span) of the bucket, spans of `span` rows
  const int64_t lb = off[c], le = off[c + 1];
  const int64_t nspan = (le - lb + span - 1) / span, local = item - istart[bkt];
  const int64_t p0 = pstart[bkt] + (local / nspan) * PQ;
  const int np = int(min(pstart[bkt + 1] - p0, int64_t(PQ)));
  const int64_t b = lb + (local % nspan) * span, e = min(le, b + span);
  if (threadIdx.x < PQ) {
    const int t = threadIdx.x;
    int64_t q = -1, pos = 0;
    if (t < np) {
      const int64_t pr = sval[p0 + t];
      q = pr / n_probe;
      if (!kFilter || kF32) {  // position: the rows of the query's earlier probed lists
        const int64_t qb = qoff != nullptr ? qoff[q] : 0;
        pos = qb;
        for (int64_t p = q * n_probe; p < pr; ++p) pos += off[probe[p] + 1] - off[probe[p]];
        s_base[t] = qb;
      }
      if (kFilter) s_tau[t] = tau[q];
      s_yy[t] = yyq[q];
    }
    s_q[t] = q;
    s_pos[t] = pos;
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // MODE 2 (IvfAnnIndex ranking, ann.py:294-312): fp32 dot of the fp32 row and fl32(y), one
  // sequential FMA chain over the dimensions; every other mode accumulates in fp64
  using Acc = typename std::conditional<kF32, float, double>::type;
  for (int64_t r0 = b; r0 < e; r0 += PRC) {
    const int rn = int(min(e - r0, int64_t(PRC)));
    Acc acc[PW][PR];
#pragma unroll
    for (int t = 0; t < PW; ++t)
#pragma unroll
      for (int i = 0; i < PR; ++i) acc[t][i] = 0.0;
    for (int j0 = 0; j0 < d; j0 += PDJ) {
      const int dj = min(PDJ, d - j0);
      __syncthreads();  // previous slice consumed (and s_q visible)
      float xv[PRC * PDJ / 128];  // all loads of the slice in flight before the stores
#pragma unroll
      for (int u = 0; u < PRC * PDJ / 128; ++u) {
        const int t = threadIdx.x + 128 * u, r = t / PDJ, jj = t % PDJ;
        xv[u] = (r < rn && jj < dj) ? __ldg(xs + (r0 + r) * d + j0 + jj) : 0.0f;
      }
#pragma unroll
      for (int u = 0; u < PQ * PDJ / 128; ++u) {
        const int t = threadIdx.x + 128 * u, qq = t / PDJ, jj = t % PDJ;
        ys[t] = (qq < np && jj < dj) ? Q[s_q[qq] * d + j0 + jj] : 0.0;
      }
#pragma unroll
      for (int u = 0; u < PRC * PDJ / 128; ++u) {
        const int t = threadIdx.x + 128 * u, r = t / PDJ, jj = t % PDJ;
        xr[r * (PDJ + 1) + jj] = double(xv[u]);
      }
      __syncthreads();
      if (warp * PW >= np) continue;  // no query on this warp (it still stages)
      for (int jj = 0; jj < dj; ++jj) {
        Acc y[PW], x[PR];
#pragma unroll
        for (int t = 0; t < PW; ++t) y[t] = Acc(ys[(warp * PW + t) * PDJ + jj]);
#pragma unroll
        for (int i = 0; i < PR; ++i) x[i] = Acc(xr[(lane + 32 * i) * (PDJ + 1) + jj]);
#pragma unroll
        for (int t = 0; t < PW; ++t)
#pragma unroll
          for (int i = 0; i < PR; ++i) acc[t][i] = fma(x[i], y[t], acc[t][i]);
      }
    }
#pragma unroll
    for (int i = 0; i < PR; ++i) {
      const int r = lane + 32 * i;
      if (r >= rn) continue;
      const double xn = xns[r0 + r];
      const unsigned long long id = static_cast<unsigned long long>(rows[r0 + r]);
#pragma unroll
      for (int t = 0; t < PW; ++t) {
        const int qq = warp * PW + t;
        if (qq >= np) continue;
        if constexpr (kF32) {
          // key32 = norms32 - 2 dot32 (one fp32 rounding), ranked with the row's position in the
          // query's probe concatenation: (order-preserving key bits << 32 | position), row id
          const float key32 = __fsub_rn(float(xn), 2.0f * float(acc[t][i]));
          uint32_t u = __float_as_uint(key32);
          u = (u & 0x80000000u) ? ~u : (u | 0x80000000u);
          const int64_t p = s_pos[qq] - s_base[qq] + (r0 - lb) + r;
          const K128 key{(static_cast<unsigned long long>(u) << 32) | static_cast<unsigned long long>(uint32_t(p)),
                         id};
          if constexpr (!kFilter) {
            keys[s_pos[qq] + (r0 - lb) + r] = key;
          } else if (k_less(key, s_tau[qq])) {
            const int64_t q = s_q[qq];
            const int slot = atomicAdd(&ccnt[q], 1);
            if (slot < cap) cand[q * cap + slot] = key;
          }
          continue;
        }
        double v = double(acc[t][i]) * -2.0;
        v += xn;
        v += s_yy[qq];
        v = fmax(v, 0.0);
        const K128 key{static_cast<unsigned long long>(__double_as_longlong(v)), id};
        if (MODE == 0) {
          keys[s_pos[qq] + (r0 - lb) + r] = key;
        } else if (k_less(key, s_tau[qq])) {
          const int64_t q = s_q[qq];
          const int slot = atomicAdd(&ccnt[q], 1);
          if (slot < cap) cand[q * cap + slot] = key;
        }
      }
    }
  }
}

// Phase 2 on packed fp32 FMAs (FFMA2) with an exact fp64 re-check.  The fp32 dot
// dot_f = sum x_j * fl32(y_j) (two interleaved chains, even and odd j, added at the end)
// satisfies |dot_f - x.y| <= (d + 1) u |x||y| (u = 2^-24: the rounding of y plus the chains),
// so with d2_f = |x|^2 + |y|^2 - 2 dot_f (fp32, each operand rounding <= u times
// |x|^2 + |y|^2 + 2|x.y| <= 2(|x|^2 + |y|^2))
//   d2 <= tau  =>  d2_f <= tau + 2.05 (d + 1) u |x||y| + 10 u (|x|^2 + |y|^2 + tau);
// rows passing that test are re-evaluated exactly (the fp64 chain of pair_tile_kernel) and
// appended when their (d2, row) key is below tau_q.
// Work item: 32 queries x up to `span` rows; per step 128 rows x 16 dimensions of x and the
// 32 query slices (fp32) arrive by cp.async into one of two buffers while the other is
// consumed; lane = 4 rows x 8 queries, 16-byte shared loads (x rows at a stride of 5
// 16-byte units: conflict-free), accumulators as {even j, odd j} pairs.
constexpr int FQ = 32, FW = 8, FR = 4, FRC = 32 * FR, FDJ = 16, FXS = FDJ + 4;
constexpr size_t kFilterSmem = size_t(2) * FRC * FXS * 4 + size_t(2) * FQ * FDJ * 4 + size_t(4) * FW * FRC * 2;
static_assert(FQ == PQ, "phase-2 items are built with PQ queries each");

__global__ void to_f32_kernel(const double* __restrict__ a, int64_t n, float* __restrict__ b) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) b[i] = __double2float_rn(a[i]);
}

template <bool VEC>
__global__ void __launch_bounds__(128, 4) pair_filter_f32_kernel(
    const float* __restrict__ xs, const double* __restrict__ xns, const int64_t* __restrict__ rows,
    const int64_t* __restrict__ off, int32_t d, int32_t C, const double* __restrict__ Q,
    const float* __restrict__ Qf, const double* __restrict__ yyq, int32_t n_probe,
    const int32_t* __restrict__ sval, const int64_t* __restrict__ pstart, const int64_t* __restrict__ istart,
    int32_t blo, int32_t bhi, int32_t span, const K128* __restrict__ tau, int32_t cap, K128* __restrict__ cand,
    int32_t* __restrict__ ccnt) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  float* xb = reinterpret_cast<float*>(smem_raw);                     // [2][FRC][FXS]
  float* yb = xb + 2 * FRC * FXS;                                      // [2][FQ][FDJ]
  uint16_t* s_queue = reinterpret_cast<uint16_t*>(yb + 2 * FQ * FDJ);  // [4][FW * FRC]
  __shared__ int64_t s_q[FQ];
  __shared__ double s_yy[FQ];
  __shared__ K128 s_tau[FQ];
  __shared__ float s_A[FQ], s_P[FQ];
  const int64_t i0 = istart[blo], item = i0 + blockIdx.x;
  if (item >= istart[bhi]) return;
  int lo = blo, hi = bhi - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (istart[mid] <= item) lo = mid; else hi = mid - 1;
  }
  const int bkt = lo, c = bkt - C - 1;
  // item = (query group, row span) of the bucket, spans of `span` rows
  const int64_t lb = off[c], le = off[c + 1];
  const int64_t nspan = (le - lb + span - 1) / span, local = item - istart[bkt];
  const int64_t p0 = pstart[bkt] + (local / nspan) * FQ;
  const int np = int(min(pstart[bkt + 1] - p0, int64_t(FQ)));
  const int64_t b = lb + (local % nspan) * span, e = min(le, b + span);
  constexpr float u = 5.9604645e-8f;  // 2^-24
  if (threadIdx.x < FQ) {
    const int t = threadIdx.x;
    int64_t q = -1;
    float A = 0.f, P = -INFINITY;  // inactive slots pass nothing
    if (t < np) {
      q = int64_t(sval[p0 + t]) / n_probe;
      const K128 tq = tau[q];
      const double yy = yyq[q];
      s_tau[t] = tq;
      s_yy[t] = yy;
      if (tq.hi == ~0ull) {  // no threshold: every row passes
        P = INFINITY;
      } else {
        const float tf = __double2float_ru(__longlong_as_double(static_cast<long long>(tq.hi)));
        const float yf = __double2float_rn(yy);
        A = 2.05f * float(d + 1) * u * sqrtf(yf) * 1.0001f;
        P = tf + 10.f * u * (yf + tf) - yf;  // test: -2 dot_f <= A |x| + P + 10 u |x|^2 - |x|^2
      }
    }
    s_q[t] = q;
    s_A[t] = A;
    s_P[t] = P;
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint16_t* queue = s_queue + warp * FW * FRC;
  const int nstage = (d + FDJ - 1) / FDJ;
  const int nst = int((e - b + FRC - 1) / FRC) * nstage;
  auto issue = [&](int st) {
    const int64_t r0 = b + int64_t(st / nstage) * FRC;
    const int j0 = (st % nstage) * FDJ;
    const int rn = int(min(e - r0, int64_t(FRC))), dj = min(FDJ, d - j0);
    float* xd = xb + (st & 1) * FRC * FXS;
    float* yd = yb + (st & 1) * FQ * FDJ;
    if constexpr (VEC) {
#pragma unroll
      for (int w = 0; w < FRC * FDJ / 4 / 128; ++w) {
        const int t = threadIdx.x + 128 * w, r = t >> 2, c4 = t & 3;
        const int nb = r < rn ? min(max(dj - 4 * c4, 0), 4) * 4 : 0;
        cp_async16(xd + r * FXS + 4 * c4, nb ? xs + (r0 + r) * d + j0 + 4 * c4 : xs, uint32_t(nb));
      }
      {
        const int t = threadIdx.x, qq = t >> 2, c4 = t & 3;
        const int nb = qq < np ? min(max(dj - 4 * c4, 0), 4) * 4 : 0;
        cp_async16(yd + qq * FDJ + 4 * c4, nb ? Qf + s_q[qq] * d + j0 + 4 * c4 : Qf, uint32_t(nb));
      }
    } else {
#pragma unroll 4
      for (int w = 0; w < FRC * FDJ / 128; ++w) {
        const int t = threadIdx.x + 128 * w, r = t / FDJ, jj = t % FDJ;
        const bool ok = r < rn && jj < dj;
        cp_async4(xd + r * FXS + jj, ok ? xs + (r0 + r) * d + j0 + jj : xs, ok ? 4u : 0u);
      }
#pragma unroll
      for (int w = 0; w < FQ * FDJ / 128; ++w) {
        const int t = threadIdx.x + 128 * w, qq = t / FDJ, jj = t % FDJ;
        const bool ok = qq < np && jj < dj;
        cp_async4(yd + qq * FDJ + jj, ok ? Qf + s_q[qq] * d + j0 + jj : Qf, ok ? 4u : 0u);
      }
    }
    cp_async_commit();
  };
  float2 acc[FW][FR];
#pragma unroll
  for (int t = 0; t < FW; ++t)
#pragma unroll
    for (int i = 0; i < FR; ++i) acc[t][i] = make_float2(0.f, 0.f);
  if (nst > 0) issue(0);
  for (int st = 0; st < nst; ++st) {
    if (st + 1 < nst) {
      issue(st + 1);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    const int js = st % nstage, dj = min(FDJ, d - js * FDJ);
    const float* xc = xb + (st & 1) * FRC * FXS;
    const float* yc = yb + (st & 1) * FQ * FDJ;
    if (warp * FW < np) {  // (a warp without queries only stages)
      for (int jj = 0; jj < dj; jj += 4) {
        float4 x[FR];
#pragma unroll
        for (int i = 0; i < FR; ++i) x[i] = *reinterpret_cast<const float4*>(xc + (lane + 32 * i) * FXS + jj);
#pragma unroll
        for (int t = 0; t < FW; ++t) {
          const float4 y = *reinterpret_cast<const float4*>(yc + (warp * FW + t) * FDJ + jj);
#pragma unroll
          for (int i = 0; i < FR; ++i) {
            acc[t][i] = fma2(make_float2(x[i].x, x[i].y), make_float2(y.x, y.y), acc[t][i]);
            acc[t][i] = fma2(make_float2(x[i].z, x[i].w), make_float2(y.z, y.w), acc[t][i]);
          }
        }
      }
    }
    if (js == nstage - 1 && warp * FW < np) {
      // chunk done: approximate test, survivors queued per warp as (query slot, row)
      const int64_t r0 = b + int64_t(st / nstage) * FRC;
      const int rn = int(min(e - r0, int64_t(FRC)));
      int qn = 0;
#pragma unroll
      for (int i = 0; i < FR; ++i) {
        const int r = lane + 32 * i;
        const bool rv = r < rn;
        const float xf = rv ? float(xns[r0 + r]) : 0.f, xnorm = sqrtf(xf);
        const float R = 10.f * u * xf - xf;
#pragma unroll
        for (int t = 0; t < FW; ++t) {
          const int qq = warp * FW + t;
          const float dot = acc[t][i].x + acc[t][i].y;
          const bool pass = rv && (-2.f * dot <= fmaf(s_A[qq], xnorm, s_P[qq] + R));
          const unsigned m = __ballot_sync(0xffffffffu, pass);
          if (pass) queue[qn + __popc(m & ((1u << lane) - 1u))] = uint16_t((t << 8) | r);
          qn += __popc(m);
          acc[t][i] = make_float2(0.f, 0.f);
        }
      }
      __syncwarp();
      // exact re-check, one queued pair per lane
      for (int k2 = lane; k2 < qn; k2 += 32) {
        const int ent = queue[k2], t = ent >> 8, r = ent & 255, qq = warp * FW + t;
        const int64_t q = s_q[qq], pos = r0 + r;
        const float* x = xs + pos * d;
        const double* y = Q + q * d;
        double dot = 0.0;
        for (int j = 0; j < d; ++j) dot = fma(double(__ldg(x + j)), y[j], dot);
        double v = dot * -2.0;
        v += xns[pos];
        v += s_yy[qq];
        v = fmax(v, 0.0);
        const K128 key{static_cast<unsigned long long>(__double_as_longlong(v)),
                       static_cast<unsigned long long>(rows[pos])};
        if (k_less(key, s_tau[qq])) {
          const int slot = atomicAdd(&ccnt[q], 1);
          if (slot < cap) cand[q * cap + slot] = key;
        }
      }
      __syncwarp();
    }
    __syncthreads();  // buffer (st & 1) is refilled by the next iteration's issue
  }
}

// per query: top-k by (d2, row) of an optional sorted head (idx/d2, c1 entries) and a key
// segment, through a shared-memory buffer of NB keys (chunks of the segment when it is larger)
__global__ void seg_topk_kernel(const int64_t* __restrict__ hidx, const double* __restrict__ hd2,
                                const int32_t* __restrict__ hcnt, const K128* __restrict__ seg,
                                const int64_t* __restrict__ seg_off, int64_t seg_stride,
                                const int32_t* __restrict__ seg_cnt, int32_t seg_cap, int32_t NB, int32_t k,
                                const int32_t* __restrict__ cnt_valid, int64_t* __restrict__ idx_out,
                                double* __restrict__ d2_out, int32_t* __restrict__ cnt_out,
                                K128* __restrict__ tau_out, int32_t* __restrict__ overflow) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  K128* buf = reinterpret_cast<K128*>(smem_raw);
  const int64_t q = blockIdx.x;
  const int64_t n = seg_off ? seg_off[q + 1] - seg_off[q] : int64_t(seg_cnt[q]);
  const K128* src = seg + (seg_off ? seg_off[q] : q * seg_stride);
  if (overflow) {
    if (n > seg_cap) {  // redone separately
      if (threadIdx.x == 0) overflow[q] = 1;
      return;
    }
    if (threadIdx.x == 0) overflow[q] = 0;
  }
  const int c1 = hcnt ? hcnt[q] : 0;
  auto head = [&](int i) {
    return K128{static_cast<unsigned long long>(__double_as_longlong(hd2[q * k + i])),
                static_cast<unsigned long long>(hidx[q * k + i])};
  };
  int filled = c1;
  int64_t pos = 0;
  if (c1 + n > 1024 && c1 + n >= k) {
    // selection: a 2048-bin histogram of the d2 bits (monotone for d2 >= 0) between the
    // smallest and largest key; every key in the bins up to the k-th key's bin is kept
    __shared__ unsigned long long s_mn, s_mx;
    __shared__ int s_hist[2048], s_m, s_bin;
    if (threadIdx.x == 0) {
      s_mn = ~0ull;
      s_mx = 0ull;
      s_m = 0;
    }
    for (int i = threadIdx.x; i < 2048; i += blockDim.x) s_hist[i] = 0;
    __syncthreads();
    unsigned long long mn = ~0ull, mx = 0ull;
    for (int i = threadIdx.x; i < c1; i += blockDim.x) {
      const unsigned long long h = head(i).hi;
      mn = h < mn ? h : mn;
      mx = h > mx ? h : mx;
    }
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
      const unsigned long long h = src[i].hi;
      mn = h < mn ? h : mn;
      mx = h > mx ? h : mx;
    }
    atomicMin(&s_mn, mn);
    atomicMax(&s_mx, mx);
    __syncthreads();
    mn = s_mn;
    const unsigned long long span = s_mx - mn;
    const int shift = span == 0 ? 0 : max(0, 64 - __clzll(static_cast<long long>(span)) - 11);
    for (int i = threadIdx.x; i < c1; i += blockDim.x) atomicAdd(&s_hist[(head(i).hi - mn) >> shift], 1);
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) atomicAdd(&s_hist[(src[i].hi - mn) >> shift], 1);
    __syncthreads();
    if (threadIdx.x < 32) {  // bin of the k-th key: warp scan over 64 bins per lane
      const int l = threadIdx.x;
      int sum = 0;
      for (int i = 0; i < 64; ++i) sum += s_hist[l * 64 + i];
      int incl = sum;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_up_sync(0xffffffffu, incl, o);
        if (l >= o) incl += t;
      }
      const unsigned hit = __ballot_sync(0xffffffffu, incl >= k);
      const int L = __ffs(hit) - 1;
      if (l == L) {
        int cum = incl - sum, b = l * 64;
        while (cum + s_hist[b] < k) cum += s_hist[b++];
        s_bin = b;
        s_m = cum + s_hist[b];
      }
    }
    __syncthreads();
    if (s_m <= NB) {
      const unsigned long long lim = static_cast<unsigned long long>(s_bin);
      if (threadIdx.x == 0) s_m = 0;
      __syncthreads();
      for (int i = threadIdx.x; i < c1; i += blockDim.x) {
        const K128 v = head(i);
        if (((v.hi - mn) >> shift) <= lim) buf[atomicAdd(&s_m, 1)] = v;
      }
      for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
        const K128 v = src[i];
        if (((v.hi - mn) >> shift) <= lim) buf[atomicAdd(&s_m, 1)] = v;
      }
      __syncthreads();
      filled = s_m;
      pos = n;  // every candidate is in buf: one sort below
    }
  }
  if (pos == 0)
    for (int i = threadIdx.x; i < c1; i += blockDim.x) buf[i] = head(i);
  do {
    const int take = int(min(n - pos, int64_t(NB - filled)));
    const int tot = filled + take;
    int B = 2;
    while (B < tot) B <<= 1;
    for (int i = threadIdx.x; i < B - filled; i += blockDim.x)
      buf[filled + i] = i < take ? src[pos + i] : K128{~0ull, ~0ull};
    bitonic(buf, B);
    pos += take;
    filled = min(tot, k);
  } while (pos < n);
  const int cnt = cnt_valid ? cnt_valid[q] : filled;
  for (int i = threadIdx.x; i < k; i += blockDim.x) {
    const bool ok = i < cnt;
    idx_out[q * k + i] = ok ? static_cast<int64_t>(buf[i].lo) : -1;
    d2_out[q * k + i] = ok ? __longlong_as_double(static_cast<long long>(buf[i].hi))
                           : __longlong_as_double(0x7ff0000000000000ll);
  }
  if (threadIdx.x == 0) {
    cnt_out[q] = cnt;
    if (tau_out) tau_out[q] = cnt == k ? buf[k - 1] : K128{~0ull, ~0ull};
  }
}

// overflowed queries: compacted (query row, probe list), every probed key through the
// list-major pass, the per-query top-k, and the answers scattered back
__global__ void redo_compact_kernel(const int32_t* __restrict__ redo, int64_t nr, const double* __restrict__ Q,
                                    int32_t d, const int32_t* __restrict__ probe, int32_t n_probe,
                                    double* __restrict__ Qr, int32_t* __restrict__ pr) {
  const int64_t i = blockIdx.x;
  if (i >= nr) return;
  const int64_t q = redo[i];
  for (int j = threadIdx.x; j < d; j += blockDim.x) Qr[i * d + j] = Q[q * d + j];
  for (int p = threadIdx.x; p < n_probe; p += blockDim.x) pr[i * n_probe + p] = probe[q * n_probe + p];
}

__global__ void redo_scatter_kernel(const int32_t* __restrict__ redo, int64_t nr, int32_t k,
                                    const int64_t* __restrict__ ir, const double* __restrict__ dr,
                                    const int32_t* __restrict__ cr, int64_t* __restrict__ io,
                                    double* __restrict__ dd, int32_t* __restrict__ co) {
  const int64_t i = blockIdx.x;
  if (i >= nr) return;
  const int64_t q = redo[i];
  for (int j = threadIdx.x; j < k; j += blockDim.x) {
    io[q * k + j] = ir[i * k + j];
    dd[q * k + j] = dr[i * k + j];
  }
  if (threadIdx.x == 0) co[q] = cr[i];
}

// IvfAnnIndex (ann.py:313-316): the fp32-ranked selection (row ids in `sel`, `cnt` per query)
// re-evaluated in fp64 — (x64 . y) * -2 + |x|^2 + |y|^2 clamped at 0, the sequential fma chain of
// pair_tile_kernel — and ordered by (d2, row) like _smallest_k.  One block per query.
__global__ void __launch_bounds__(128) ref32_finish_kernel(const float* __restrict__ X,
                                                           const double* __restrict__ xn64, int32_t d,
                                                           const double* __restrict__ Q,
                                                           const double* __restrict__ yyq, int32_t k, int32_t P,
                                                           const int64_t* __restrict__ sel,
                                                           const int32_t* __restrict__ cnt,
                                                           int64_t* __restrict__ io, double* __restrict__ dd,
                                                           int32_t* __restrict__ co) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  K128* buf = reinterpret_cast<K128*>(smem_raw);
  const int64_t q = blockIdx.x;
  const int c = cnt[q];
  const double* y = Q + size_t(q) * d;
  for (int i = threadIdx.x; i < P; i += blockDim.x) {
    K128 key{~0ull, ~0ull};
    if (i < c) {
      const int64_t row = sel[size_t(q) * k + i];
      const float* x = X + size_t(row) * d;
      double dot = 0.0;
      for (int j = 0; j < d; ++j) dot = fma(double(x[j]), y[j], dot);
      double v = dot * -2.0;
      v += xn64[row];
      v += yyq[q];
      v = fmax(v, 0.0);
      key = K128{static_cast<unsigned long long>(__double_as_longlong(v)), static_cast<unsigned long long>(row)};
    }
    buf[i] = key;
  }
  for (int kk = 2; kk <= P; kk <<= 1) {
    for (int j = kk >> 1; j > 0; j >>= 1) {
      __syncthreads();
      for (int i = threadIdx.x; i < P; i += blockDim.x) {
        const int ixj = i ^ j;
        if (ixj > i) {
          const bool up = (i & kk) == 0;
          const K128 a = buf[i], b = buf[ixj];
          if (k_less(b, a) == up) {
            buf[i] = b;
            buf[ixj] = a;
          }
        }
      }
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < k; i += blockDim.x) {
    const bool ok = i < c;
    io[size_t(q) * k + i] = ok ? int64_t(buf[i].lo) : -1;
    dd[size_t(q) * k + i] = ok ? __longlong_as_double(static_cast<long long>(buf[i].hi)) : __longlong_as_double(0x7ff0000000000000ll);
  }
  if (threadIdx.x == 0) co[q] = c;
}

size_t cub_bytes(int64_t n) {
  size_t a = 0, b = 0, c = 0;
  cub::DeviceReduce::Sum(nullptr, a, static_cast<const double*>(nullptr), static_cast<double*>(nullptr), n);
  cub::DeviceScan::InclusiveSum(nullptr, b, static_cast<const double*>(nullptr), static_cast<double*>(nullptr), n);
  cub::DeviceRadixSort::SortPairs(nullptr, c, static_cast<const int32_t*>(nullptr), static_cast<int32_t*>(nullptr),
                                  static_cast<const int64_t*>(nullptr), static_cast<int64_t*>(nullptr), n);
  return std::max(a, std::max(b, c)) + 256;
}

void free_ivf(dk_ivf* v) {
  if (!v) return;
  for (void* p : {static_cast<void*>(v->cent), static_cast<void*>(v->cnorm), static_cast<void*>(v->closest),
                  static_cast<void*>(v->cdf), static_cast<void*>(v->labels), static_cast<void*>(v->labels_s),
                  static_cast<void*>(v->ids), static_cast<void*>(v->rows), static_cast<void*>(v->offsets),
                  static_cast<void*>(v->d2min), static_cast<void*>(v->xs), static_cast<void*>(v->xns),
                  static_cast<void*>(v->scal), v->temp, v->keys1, v->ckeys, v->dws})
    if (p) cudaFree(p);
  delete v;
}

struct IvfDeleter {
  void operator()(dk_ivf* v) const { free_ivf(v); }
};

double read_scalar(const double* p) {
  double v = 0;
  DK_CUDA(cudaMemcpy(&v, p, sizeof(double), cudaMemcpyDeviceToHost));
  return v;
}

void launch_cnorm(dk_ivf* v) {
  cnorm_kernel<<<unsigned((int64_t(v->C) * 32 + 255) / 256), 256>>>(v->cent, v->C, v->d, v->cnorm);
  DK_CHECK_LAUNCH();
}

// labels for the current centroids; returns wcss = sum of the clamped minimum d2
double assign(dk_ivf* v) {
  const dk_dataset* h = v->ds;
  launch_cnorm(v);
  assign_kernel<<<unsigned((v->n + AM - 1) / AM), 256>>>(h->X, h->xn64, v->n, v->d, v->cent, v->cnorm, v->C,
                                                        v->labels, v->d2min);
  DK_CHECK_LAUNCH();
  size_t tb = v->temp_bytes;
  DK_CUDA(cub::DeviceReduce::Sum(v->temp, tb, v->d2min, v->scal, v->n));
  return read_scalar(v->scal);
}

// stable (label, row) sort -> cluster-contiguous rows in increasing id order + offsets
void build_lists(dk_ivf* v) {
  iota_kernel<<<unsigned((v->n + 255) / 256), 256>>>(v->ids, v->n);
  DK_CHECK_LAUNCH();
  int bits = 1;
  while ((int64_t(1) << bits) < int64_t(v->C)) ++bits;
  size_t tb = v->temp_bytes;
  DK_CUDA(cub::DeviceRadixSort::SortPairs(v->temp, tb, v->labels, v->labels_s, v->ids, v->rows, v->n, 0, bits));
  offsets_kernel<<<unsigned((v->C + 1 + 255) / 256), 256>>>(v->labels_s, v->n, v->C, v->offsets);
  DK_CHECK_LAUNCH();
}

void update_centroids(dk_ivf* v) {
  dim3 grid(unsigned(v->C), unsigned((v->d + 31) / 32));
  update_kernel<<<grid, 32>>>(v->ds->X, v->d, v->rows, v->offsets, v->C, v->cent);
  DK_CHECK_LAUNCH();
}

void restore_rows(dk_ivf* v) {
  const dk_dataset* h = v->ds;
  if (!v->xs) DK_CUDA(cudaMalloc(&v->xs, size_t(v->n) * v->d * sizeof(float)));
  if (!v->xns) DK_CUDA(cudaMalloc(&v->xns, size_t(v->n) * sizeof(double)));
  gather_rows_kernel<<<unsigned(v->n), 128>>>(h->X, h->xn64, v->d, v->rows, v->n, v->xs, v->xns);
  DK_CHECK_LAUNCH();
  v->lists = true;
}

// per cluster: max fp64 distance of its members (list order) to the centroid, inflated
__global__ void cluster_radius_kernel(const float* __restrict__ xs, const int64_t* __restrict__ off, int32_t d,
                                      const double* __restrict__ cent, double* __restrict__ rad) {
  const int c = blockIdx.x;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  __shared__ double smax[32];
  double mx = 0.0;
  for (int64_t r = off[c] + w; r < off[c + 1]; r += nw) {
    double acc = 0.0;
    for (int j = lane; j < d; j += 32) {
      const double t = double(xs[r * d + j]) - cent[size_t(c) * d + j];
      acc = fma(t, t, acc);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    mx = fmax(mx, acc);
  }
  if (lane == 0) smax[w] = mx;
  __syncthreads();
  if (threadIdx.x == 0) {
    double m = 0.0;
    for (int i = 0; i < nw; ++i) m = fmax(m, smax[i]);
    rad[c] = sqrt(m) * (1.0 + 1e-12) + 1e-300;
  }
}

__global__ void tile_range_kernel(const int32_t* __restrict__ ls, int64_t n, int32_t ntiles, int32_t* __restrict__ lo,
                                  int32_t* __restrict__ hi) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= ntiles) return;
  const int64_t a = int64_t(t) * 256;
  if (a >= n) { lo[t] = 1; hi[t] = 0; return; }  // padding tile: empty range
  lo[t] = ls[a];
  hi[t] = ls[min(n, a + 256) - 1];
}

}  // namespace

// Cluster-sorted rows for the pruned k-NN (internal.h KnnClusters): C centroids seeded
// with evenly spaced rows, `iters` Lloyd rounds (fp64 assignment, member means), then the
// rows in cluster order, per-cluster radii and per-tile cluster ranges.
void build_knn_clusters(dk_dataset* h, int32_t C, int32_t iters, KnnClusters& kc, cudaStream_t s) {
  DK_CUDA(cudaStreamSynchronize(s));
  std::unique_ptr<dk_ivf, IvfDeleter> v(new dk_ivf());
  v->ds = h;
  v->C = C;
  v->d = h->d;
  v->n = h->n;
  DK_CUDA(cudaMalloc(&v->cent, size_t(C) * v->d * sizeof(double)));
  DK_CUDA(cudaMalloc(&v->cnorm, size_t(C) * sizeof(double)));
  DK_CUDA(cudaMalloc(&v->labels, size_t(v->n) * sizeof(int32_t)));
  DK_CUDA(cudaMalloc(&v->labels_s, size_t(v->n) * sizeof(int32_t)));
  DK_CUDA(cudaMalloc(&v->ids, size_t(v->n) * sizeof(int64_t)));
  DK_CUDA(cudaMalloc(&v->rows, size_t(v->n) * sizeof(int64_t)));
  DK_CUDA(cudaMalloc(&v->offsets, size_t(C + 1) * sizeof(int64_t)));
  DK_CUDA(cudaMalloc(&v->d2min, size_t(v->n) * sizeof(double)));
  DK_CUDA(cudaMalloc(&v->scal, 4 * sizeof(double)));
  v->temp_bytes = cub_bytes(v->n);
  DK_CUDA(cudaMalloc(&v->temp, v->temp_bytes));
  for (int c = 0; c < C; ++c) {
    set_row_kernel<<<1, 128>>>(h->X, (int64_t(c) * v->n) / C, v->d, v->cent + size_t(c) * v->d);
    DK_CHECK_LAUNCH();
  }
  for (int it = 0; it < iters; ++it) {
    assign(v.get());
    build_lists(v.get());
    update_centroids(v.get());
  }
  restore_rows(v.get());
  const int32_t ntiles = int32_t(h->n_pad / 256);
  kc.C = C;
  DK_CUDA(cudaMalloc(&kc.rad, size_t(C) * sizeof(double)));
  DK_CUDA(cudaMalloc(&kc.tclo, size_t(ntiles) * sizeof(int32_t)));
  DK_CUDA(cudaMalloc(&kc.tchi, size_t(ntiles) * sizeof(int32_t)));
  cluster_radius_kernel<<<unsigned(C), 256>>>(v->xs, v->offsets, v->d, v->cent, kc.rad);
  DK_CHECK_LAUNCH();
  tile_range_kernel<<<unsigned((ntiles + 255) / 256), 256>>>(v->labels_s, v->n, ntiles, kc.tclo, kc.tchi);
  DK_CHECK_LAUNCH();
  DK_CUDA(cudaDeviceSynchronize());
  kc.cent = v->cent; v->cent = nullptr;   // ownership moves to kc
  kc.perm = v->rows; v->rows = nullptr;
  kc.xs = v->xs; v->xs = nullptr;
  kc.off = v->offsets; v->offsets = nullptr;
}

void free_knn_clusters(KnnClusters& kc) {
  for (void* p : {static_cast<void*>(kc.cent), static_cast<void*>(kc.rad), static_cast<void*>(kc.perm),
                  static_cast<void*>(kc.xs), static_cast<void*>(kc.tclo), static_cast<void*>(kc.tchi),
                  static_cast<void*>(kc.off), static_cast<void*>(kc.nbr)})
    if (p) cudaFree(p);
  for (void* p : {static_cast<void*>(kc.enc.B), static_cast<void*>(kc.enc.xn), static_cast<void*>(kc.enc.sx),
                  static_cast<void*>(kc.enc.T),
                  static_cast<void*>(kc.enc3.B), static_cast<void*>(kc.enc3.xn), static_cast<void*>(kc.enc3.sx)})
    if (p) cudaFree(p);
  if (kc.stat_host) cudaFreeHost(kc.stat_host);
  if (kc.stat_ev) cudaEventDestroy(kc.stat_ev);
  if (kc.hyb_stat_host) cudaFreeHost(kc.hyb_stat_host);
  if (kc.hyb_stat_ev) cudaEventDestroy(kc.hyb_stat_ev);
  kc = KnnClusters{};
}

}  // namespace dk

using namespace dk;

extern "C" {

dk_status dk_ivf_create(dk_handle h, int32_t n_clusters, dk_ivf_handle* out) {
  DK_NVTX();
  return guard([&] {
    DK_REQUIRE(h != nullptr && out != nullptr, "NULL argument");
    *out = nullptr;
    DK_REQUIRE(n_clusters >= 1 && int64_t(n_clusters) <= h->n,
               "n_clusters=" + std::to_string(n_clusters) + " out of range [1, " + std::to_string(h->n) + "]");
    DeviceGuard g(h->device);
    std::unique_ptr<dk_ivf, IvfDeleter> v(new dk_ivf());
    v->ds = h;
    v->C = n_clusters;
    v->d = h->d;
    v->n = h->n;
    DK_CUDA(cudaMalloc(&v->cent, size_t(v->C) * v->d * sizeof(double)));
    DK_CUDA(cudaMalloc(&v->cnorm, size_t(v->C) * sizeof(double)));
    DK_CUDA(cudaMalloc(&v->closest, size_t(v->n) * sizeof(double)));
    DK_CUDA(cudaMalloc(&v->cdf, size_t(v->n) * sizeof(double)));
    DK_CUDA(cudaMalloc(&v->labels, size_t(v->n) * sizeof(int32_t)));
    DK_CUDA(cudaMalloc(&v->labels_s, size_t(v->n) * sizeof(int32_t)));
    DK_CUDA(cudaMalloc(&v->ids, size_t(v->n) * sizeof(int64_t)));
    DK_CUDA(cudaMalloc(&v->rows, size_t(v->n) * sizeof(int64_t)));
    DK_CUDA(cudaMalloc(&v->offsets, size_t(v->C + 1) * sizeof(int64_t)));
    DK_CUDA(cudaMalloc(&v->d2min, size_t(v->n) * sizeof(double)));
    DK_CUDA(cudaMalloc(&v->scal, 4 * sizeof(double)));
    v->temp_bytes = cub_bytes(v->n);
    DK_CUDA(cudaMalloc(&v->temp, v->temp_bytes));
    *out = v.release();
  });
}

dk_status dk_ivf_free(dk_ivf_handle v) {
  DK_NVTX();
  return guard([&] {
    if (!v) return;
    DeviceGuard g(v->ds->device);
    cudaDeviceSynchronize();
    free_ivf(v);
  });
}

dk_status dk_kmeanspp_seed(dk_ivf_handle v, int32_t c, int64_t row, double* total_out) {
  DK_NVTX();
  return guard([&] {
    DK_REQUIRE(v != nullptr && total_out != nullptr, "NULL argument");
    DK_REQUIRE(c >= 0 && c < v->C && row >= 0 && row < v->n, "centroid or row out of range");
    DeviceGuard g(v->ds->device);
    double* cc = v->cent + size_t(c) * v->d;
    set_row_kernel<<<1, 128>>>(v->ds->X, row, v->d, cc);
    DK_CHECK_LAUNCH();
    pp_dist_kernel<<<unsigned((v->n * 32 + 255) / 256), 256>>>(v->ds->X, v->n, v->d, cc, c == 0 ? 1 : 0,
                                                               v->closest);
    DK_CHECK_LAUNCH();
    size_t tb = v->temp_bytes;
    DK_CUDA(cub::DeviceReduce::Sum(v->temp, tb, v->closest, v->scal, v->n));
    *total_out = read_scalar(v->scal);
  });
}

dk_status dk_kmeanspp_pick(dk_ivf_handle v, double u, double total, int64_t* row_out) {
  DK_NVTX();
  return guard([&] {
    DK_REQUIRE(v != nullptr && row_out != nullptr, "NULL argument");
    DK_REQUIRE(total > 0.0 && u >= 0.0 && u < 1.0, "pick needs total > 0 and u in [0, 1)");
    DeviceGuard g(v->ds->device);
    div_kernel<<<unsigned((v->n + 255) / 256), 256>>>(v->closest, v->n, total, v->cdf);
    DK_CHECK_LAUNCH();
    size_t tb = v->temp_bytes;
    DK_CUDA(cub::DeviceScan::InclusiveSum(v->temp, tb, v->cdf, v->cdf, v->n));
    int64_t* out = reinterpret_cast<int64_t*>(v->scal + 1);
    const int64_t sentinel = v->n - 1;  // cdf[-1] / cdf[-1] == 1 > u always selects something
    DK_CUDA(cudaMemcpy(out, &sentinel, sizeof(int64_t), cudaMemcpyHostToDevice));
    search_kernel<<<unsigned((v->n + 255) / 256), 256>>>(v->cdf, v->n, u, out);
    DK_CHECK_LAUNCH();
    DK_CUDA(cudaMemcpy(row_out, out, sizeof(int64_t), cudaMemcpyDeviceToHost));
  });
}

dk_status dk_kmeans_lloyd(dk_ivf_handle v, int32_t max_iter, double rel_tol, int32_t* iters_out) {
  DK_NVTX();
  return guard([&] {
    DK_REQUIRE(v != nullptr, "NULL argument");
    DK_REQUIRE(max_iter >= 0 && rel_tol >= 0.0, "bad k-means parameters");
    DeviceGuard g(v->ds->device);
    double prev = std::numeric_limits<double>::infinity();
    int32_t it = 0;
    for (; it < max_iter;) {  // ann.py:184-195
      const double wcss = assign(v);
      build_lists(v);
      update_centroids(v);
      ++it;
      if (prev - wcss <= rel_tol * std::max(prev, 1e-300)) break;
      prev = wcss;
    }
    assign(v);  // final assignment against the final centroids (ann.py:196-198)
    build_lists(v);
    launch_cnorm(v);
    restore_rows(v);
    DK_CUDA(cudaDeviceSynchronize());
    if (iters_out) *iters_out = it;
  });
}

dk_status dk_ivf_get(dk_ivf_handle v, double* centroids, int64_t* rows, int64_t* offsets) {
  DK_NVTX();
  return guard([&] {
    DK_REQUIRE(v != nullptr, "NULL argument");
    DeviceGuard g(v->ds->device);
    if (centroids)
      DK_CUDA(cudaMemcpy(centroids, v->cent, size_t(v->C) * v->d * sizeof(double), cudaMemcpyDefault));
    if (rows) DK_CUDA(cudaMemcpy(rows, v->rows, size_t(v->n) * sizeof(int64_t), cudaMemcpyDefault));
    if (offsets) DK_CUDA(cudaMemcpy(offsets, v->offsets, size_t(v->C + 1) * sizeof(int64_t), cudaMemcpyDefault));
  });
}

dk_status dk_ivf_set(dk_ivf_handle v, const double* centroids, const int64_t* rows, const int64_t* offsets) {
  DK_NVTX();
  return guard([&] {
    DK_REQUIRE(v != nullptr && centroids != nullptr && rows != nullptr && offsets != nullptr, "NULL argument");
    std::vector<int64_t> off(static_cast<size_t>(v->C) + 1);
    std::memcpy(off.data(), offsets, off.size() * sizeof(int64_t));
    DK_REQUIRE(off[0] == 0, "offsets must start at 0");
    for (int32_t c = 0; c < v->C; ++c) DK_REQUIRE(off[size_t(c) + 1] >= off[size_t(c)], "offsets must be nondecreasing");
    DK_REQUIRE(off.back() == v->n, "the lists must hold every dataset row exactly once");
    std::vector<char> seen(static_cast<size_t>(v->n), 0);
    for (int64_t i = 0; i < v->n; ++i) {
      DK_REQUIRE(rows[i] >= 0 && rows[i] < v->n && !seen[size_t(rows[i])],
                 "the lists must hold every dataset row exactly once");
      seen[size_t(rows[i])] = 1;
    }
    DeviceGuard g(v->ds->device);
    DK_CUDA(cudaMemcpy(v->cent, centroids, size_t(v->C) * v->d * sizeof(double), cudaMemcpyHostToDevice));
    DK_CUDA(cudaMemcpy(v->rows, rows, size_t(v->n) * sizeof(int64_t), cudaMemcpyHostToDevice));
    DK_CUDA(cudaMemcpy(v->offsets, off.data(), off.size() * sizeof(int64_t), cudaMemcpyHostToDevice));
    launch_cnorm(v);
    restore_rows(v);
    DK_CUDA(cudaDeviceSynchronize());
  });
}

dk_status dk_ivf_query(dk_ivf_handle v, const double* Q, int64_t nq, int32_t k, int32_t n_probe, int32_t formula,
                       int64_t* idx_out, double* d2_out, int32_t* cnt_out, void* stream) {
  DK_NVTX();
  return guard([&] {
    DK_REQUIRE(v != nullptr, "NULL handle");
    DK_REQUIRE(v->lists, "index lists are not built (dk_kmeans_lloyd or dk_ivf_set first)");
    DK_REQUIRE(k >= 1, "k=" + std::to_string(k) + " must be >= 1");
    DK_REQUIRE(n_probe >= 1 && n_probe <= v->C,
               "n_probe=" + std::to_string(n_probe) + " out of range [1, " + std::to_string(v->C) + "]");
    DK_REQUIRE(formula == 0 || formula == 1, "unknown probe formula");
    DK_REQUIRE(nq >= 0, "negative query count");
    if (nq == 0) return;
    DK_REQUIRE(Q != nullptr && idx_out != nullptr && d2_out != nullptr && cnt_out != nullptr, "NULL argument");
    dk_dataset* h = v->ds;
    DeviceGuard g(h->device);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    int Bc = 2;
    while (Bc < v->C) Bc <<= 1;
    const size_t probe_smem = size_t(Bc) * sizeof(K128) + size_t(v->d) * sizeof(double);
    const bool bigc = probe_smem > 232448;  // probe by a segmented radix sort instead
    int Kp = 32;
    while (Kp < k) Kp <<= 1;
    const int S = std::max(Kp, 256);  // rows per round (stage capacity)
    int B = 2;
    while (B < Kp + S) B <<= 1;
    const size_t scan_smem = size_t(B) * sizeof(K128) + size_t(v->d) * sizeof(double);
    const bool bigk = k > 4096 || scan_smem > 232000;  // beyond the shared-memory top-k
    // staging: queries, probe lists, outputs
    size_t off = 0;
    auto take = [&](size_t bytes) {
      const size_t a = (off + 255) & ~size_t(255);
      off = a + bytes;
      return a;
    };
    const size_t o_q = take(size_t(nq) * v->d * sizeof(double));
    const size_t o_p = take(size_t(nq) * n_probe * sizeof(int32_t));
    const size_t o_i = take(size_t(nq) * k * sizeof(int64_t));  // (host outputs only)
    const size_t o_d = take(size_t(nq) * k * sizeof(double));
    const size_t o_c = take(size_t(nq) * sizeof(int32_t));
    DK_REQUIRE(nq < (int64_t(1) << 31), "too many queries in one IVF call");
    size_t ord_bytes = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, ord_bytes, static_cast<const int32_t*>(nullptr),
                                    static_cast<int32_t*>(nullptr), static_cast<const int32_t*>(nullptr),
                                    static_cast<int32_t*>(nullptr), int(nq));
    const size_t o_k0 = take(size_t(nq) * 4), o_k1 = take(size_t(nq) * 4), o_v0 = take(size_t(nq) * 4);
    const size_t o_ord = take(size_t(nq) * 4), o_ot = take(ord_bytes + 256);
    // two-phase plan (see pair_tile_kernel)
    static const bool one_phase = std::getenv("DK_IVF_ONE_PHASE") != nullptr;  // A/B switch
    const int64_t npairs = nq * int64_t(n_probe);
    const int32_t NBK = 2 * v->C + 2;  // pair buckets: phase-1 lists, a gap, phase-2 lists
    const bool two_phase = !bigk && !one_phase && npairs < (int64_t(1) << 31);
    // IvfAnnIndex (formula 1) ranks the probed rows in fp32 like the reference (ann.py:294-312):
    // the two-phase pass over (fp32 key, probe position) keys — the k smallest per query — then
    // the fp64 re-evaluation of those (ref32_finish_kernel).  DK_IVF_EXACT_RANK=1: exact fp64
    // ranking instead (differs only at fp32 near-ties).
    static const bool exact_rank = std::getenv("DK_IVF_EXACT_RANK") != nullptr;
    const bool ref32 = formula == 1 && two_phase && !exact_rank;
    int64_t cap_rows = std::max<int64_t>(2048, 16 * int64_t(k));
    if (const char* e = std::getenv("DK_IVF_CAP")) cap_rows = std::max<int64_t>(1, std::atoll(e));  // tests
    const int32_t cap = int32_t(std::min<int64_t>(int64_t(1) << 20, cap_rows));
    int NB = 2048;  // seg_topk_kernel buffer: at least twice the top-k
    while (NB < 2 * Kp) NB <<= 1;
    size_t cub2 = 0;
    size_t o_i1 = 0, o_d1 = 0, o_c1 = 0, o_np = 0, o_ca = 0, o_tau = 0, o_kin = 0, o_kout = 0, o_vin = 0,
           o_vout = 0, o_ps = 0, o_ni = 0, o_is = 0, o_t2 = 0, o_cc = 0, o_cand = 0, o_ov = 0, o_rq = 0, o_rQ = 0,
           o_rp = 0, o_yy = 0, o_r1 = 0, o_qo = 0, o_qf = 0;
    int64_t redo_R = 0;
    if (two_phase) {
      size_t a = 0, b2 = 0;
      cub::DeviceRadixSort::SortPairs(nullptr, a, static_cast<const int32_t*>(nullptr),
                                      static_cast<int32_t*>(nullptr), static_cast<const int32_t*>(nullptr),
                                      static_cast<int32_t*>(nullptr), int(npairs));
      cub::DeviceScan::ExclusiveSum(nullptr, b2, static_cast<const int64_t*>(nullptr),
                                    static_cast<int64_t*>(nullptr), std::max<int64_t>(NBK + 1, nq + 1));
      cub2 = std::max(a, b2) + 256;
      o_i1 = take(size_t(nq) * k * 8);
      o_d1 = take(size_t(nq) * k * 8);
      o_c1 = take(size_t(nq) * 4);
      o_np = take(size_t(nq) * 4);
      o_ca = take(size_t(nq) * 4);
      o_tau = take(size_t(nq) * sizeof(K128));
      o_yy = take(size_t(nq) * 8);
      o_qf = take(size_t(nq) * v->d * 4);
      o_r1 = take(size_t(nq + 1) * 8);
      o_qo = take(size_t(nq + 1) * 8);
      o_kin = take(size_t(npairs) * 4);
      o_kout = take(size_t(npairs) * 4);
      o_vin = take(size_t(npairs) * 4);
      o_vout = take(size_t(npairs) * 4);
      o_ps = take(size_t(NBK + 1) * 8);
      o_ni = take(size_t(NBK + 1) * 8);
      o_is = take(size_t(NBK + 1) * 8);
      o_t2 = take(cub2);
      o_cc = take(size_t(nq) * 4);
      o_cand = take(size_t(nq) * cap * sizeof(K128));
      o_ov = take(size_t(nq) * 4);
      // overflow redo in chunks of R queries (compacted query rows and probe lists)
      redo_R = std::min<int64_t>(nq, 1024);
      o_rq = take(size_t(redo_R) * 4);
      o_rQ = take(size_t(redo_R) * v->d * 8);
      o_rp = take(size_t(redo_R) * n_probe * 4);
    }
    h->ws.reserve(off);
    uint8_t* base = h->ws.base;
    const double* Qd = Q;
    if (!is_device_ptr(Q)) {
      DK_CUDA(cudaMemcpyAsync(base + o_q, Q, size_t(nq) * v->d * sizeof(double), cudaMemcpyHostToDevice, s));
      Qd = reinterpret_cast<const double*>(base + o_q);
    }
    int32_t* probe = reinterpret_cast<int32_t*>(base + o_p);
    if (!bigc) {
      const int64_t chunk = std::max<int64_t>(CQ, std::min<int64_t>(nq, (int64_t(1) << 24) / v->C));
      const size_t cbytes = size_t(chunk) * v->C * 8;
      if (cbytes > v->ckeys_bytes) {
        if (v->ckeys) DK_CUDA(cudaFree(v->ckeys));
        v->ckeys = nullptr;
        v->ckeys_bytes = 0;
        DK_CUDA(cudaMalloc(&v->ckeys, cbytes));
        v->ckeys_bytes = cbytes;
      }
      auto* ck = static_cast<unsigned long long*>(v->ckeys);
      for (int64_t q0 = 0; q0 < nq; q0 += chunk) {
        const int64_t nqc = std::min(chunk, nq - q0);
        const dim3 grid(unsigned((v->C + CRC - 1) / CRC), unsigned((nqc + CQ - 1) / CQ));
        if (formula == 0)
          centroid_tile_kernel<0><<<grid, 128, 0, s>>>(Qd, q0, nqc, v->d, v->cent, v->cnorm, v->C, ck);
        else
          centroid_tile_kernel<1><<<grid, 128, 0, s>>>(Qd, q0, nqc, v->d, v->cent, v->cnorm, v->C, ck);
        DK_CHECK_LAUNCH();
        if (n_probe <= 64) {
          probe_select_kernel<<<unsigned((nqc + 7) / 8), 256, 0, s>>>(ck, q0, nqc, v->C, n_probe, probe);
        } else {
          const size_t psm = size_t(Bc) * sizeof(K128);
          set_dynamic_smem(probe_sort_kernel, psm);
          probe_sort_kernel<<<unsigned(nqc), 256, psm, s>>>(ck, q0, v->C, Bc, n_probe, probe);
        }
        DK_CHECK_LAUNCH();
      }
    } else {
      const int64_t chunk = std::max<int64_t>(1, (int64_t(1) << 26) / v->C);
      for (int64_t q0 = 0; q0 < nq; q0 += chunk) {
        const int64_t nqc = std::min(chunk, nq - q0);
        const int64_t T = nqc * v->C;
        size_t sb = 0;
        cub::DeviceSegmentedRadixSort::SortPairs(nullptr, sb, static_cast<const unsigned long long*>(nullptr),
                                                 static_cast<unsigned long long*>(nullptr),
                                                 static_cast<const int32_t*>(nullptr), static_cast<int32_t*>(nullptr),
                                                 int(T), int(nqc), static_cast<const int64_t*>(nullptr),
                                                 static_cast<const int64_t*>(nullptr));
        DevBuf buf(size_t(T) * (8 + 8 + 4 + 4) + size_t(nqc + 1) * 8 + sb + 512);
        auto* k0 = buf.as<unsigned long long>(0);
        auto* k1 = buf.as<unsigned long long>(size_t(T) * 8);
        auto* v0 = buf.as<int32_t>(size_t(T) * 16);
        auto* v1 = buf.as<int32_t>(size_t(T) * 20);
        auto* seg = buf.as<int64_t>((size_t(T) * 24 + 7) & ~size_t(7));
        void* tmp = buf.as<uint8_t>((size_t(T) * 24 + size_t(nqc + 1) * 8 + 255 + 8) & ~size_t(255));
        seg_starts_kernel<<<unsigned((nqc + 1 + 255) / 256), 256, 0, s>>>(nqc, v->C, seg);
        DK_CHECK_LAUNCH();
        dim3 grid(unsigned((v->C + 7) / 8), unsigned(nqc));
        centroid_keys_kernel<<<grid, 256, 0, s>>>(Qd, v->d, v->cent, v->cnorm, v->C, q0, formula, k0, v0);
        DK_CHECK_LAUNCH();
        size_t tb = sb;
        DK_CUDA(cub::DeviceSegmentedRadixSort::SortPairs(tmp, tb, k0, k1, v0, v1, int(T), int(nqc), seg, seg + 1,
                                                         0, 64, s));
        take_probe_kernel<<<unsigned((nqc * n_probe + 255) / 256), 256, 0, s>>>(v1, v->C, q0, nqc, n_probe, probe);
        DK_CHECK_LAUNCH();
        DK_CUDA(cudaStreamSynchronize(s));
      }
    }
    const bool idev = is_device_ptr(idx_out), ddev = is_device_ptr(d2_out), cdev = is_device_ptr(cnt_out);
    int64_t* io = idev ? idx_out : reinterpret_cast<int64_t*>(base + o_i);
    double* dd = ddev ? d2_out : reinterpret_cast<double*>(base + o_d);
    int32_t* co = cdev ? cnt_out : reinterpret_cast<int32_t*>(base + o_c);
    if (bigk) {
      ivf_query_bigk(v, Qd, nq, k, n_probe, probe, io, dd, co, s);
    } else {
    // lanes per row: enough that one float4 sweep covers about half of a row's 16-byte chunks
    const int chunks = (v->d + 3) / 4;
    // query order: sorted by nearest probed list (L2 reuse across concurrently running blocks)
    int32_t* order = reinterpret_cast<int32_t*>(base + o_ord);
    {
      auto* kin = reinterpret_cast<int32_t*>(base + o_k0);
      auto* kout = reinterpret_cast<int32_t*>(base + o_k1);
      auto* vin = reinterpret_cast<int32_t*>(base + o_v0);
      first_probe_kernel<<<unsigned((nq + 255) / 256), 256, 0, s>>>(probe, nq, n_probe, kin, vin);
      DK_CHECK_LAUNCH();
      int bits = 1;
      while ((int64_t(1) << bits) < int64_t(v->C)) ++bits;
      size_t tb = ord_bytes;
      DK_CUDA(cub::DeviceRadixSort::SortPairs(base + o_ot, tb, kin, kout, vin, order, int(nq), 0, bits, s));
    }
    const bool vec = (v->d & 3) == 0;
    // per-query scan over all probed lists (np_q == nullptr) or a per-query prefix of them, of the
    // queries Qs with probe lists ps (npr per query), taken in the order ord (nullptr: 0..count-1)
    auto scan_with = [&](const double* Qs, const int32_t* ps, int32_t npr, const int32_t* ord, int64_t count,
                         int64_t* oi, double* od2, int32_t* oc, const int32_t* np_q = nullptr) {
#define DK_SCAN(G, IT)                                                                                       \
  do {                                                                                                       \
    set_dynamic_smem(scan_kernel<G, IT>, scan_smem);                                                         \
    scan_kernel<G, IT><<<unsigned(count), 256, scan_smem, s>>>(v->xs, v->xns, v->rows, v->offsets, v->d, ord, \
                                                              Qs, ps, npr, np_q, k, Kp, S, B, oi, od2, oc); \
  } while (0)
      // register-resident query slices where a row is at most 4 float4 steps per lane (G < 32)
      if (chunks >= 64) DK_SCAN(32, 0);
      else if (chunks >= 32) { if (vec) DK_SCAN(16, 4); else DK_SCAN(16, 0); }
      else if (chunks >= 16) { if (vec) DK_SCAN(8, 4); else DK_SCAN(8, 0); }
      else if (chunks >= 8) { if (vec) DK_SCAN(4, 4); else DK_SCAN(4, 0); }
      else if (chunks >= 4) { if (vec) DK_SCAN(2, 4); else DK_SCAN(2, 0); }
      else { if (vec) DK_SCAN(1, 4); else DK_SCAN(1, 0); }
#undef DK_SCAN
      DK_CHECK_LAUNCH();
    };
    auto run_scan = [&](const int32_t* ord, int64_t count, const int32_t* np_q, int64_t* oi, double* od2,
                        int32_t* oc) { scan_with(Qd, probe, n_probe, ord, count, oi, od2, oc, np_q); };
    if (!two_phase) {
      run_scan(order, nq, nullptr, io, dd, co);
    } else {
      auto* idx1 = reinterpret_cast<int64_t*>(base + o_i1);
      auto* d21 = reinterpret_cast<double*>(base + o_d1);
      auto* cnt1 = reinterpret_cast<int32_t*>(base + o_c1);
      auto* npq = reinterpret_cast<int32_t*>(base + o_np);
      auto* call = reinterpret_cast<int32_t*>(base + o_ca);
      auto* tau = reinterpret_cast<K128*>(base + o_tau);
      auto* kin = reinterpret_cast<int32_t*>(base + o_kin);
      auto* kout = reinterpret_cast<int32_t*>(base + o_kout);
      auto* vin = reinterpret_cast<int32_t*>(base + o_vin);
      auto* vout = reinterpret_cast<int32_t*>(base + o_vout);
      auto* ps = reinterpret_cast<int64_t*>(base + o_ps);
      auto* ni = reinterpret_cast<int64_t*>(base + o_ni);
      auto* is = reinterpret_cast<int64_t*>(base + o_is);
      auto* ccnt = reinterpret_cast<int32_t*>(base + o_cc);
      auto* cand = reinterpret_cast<K128*>(base + o_cand);
      auto* ovf = reinterpret_cast<int32_t*>(base + o_ov);
      auto* yyq = reinterpret_cast<double*>(base + o_yy);
      auto* rows1 = reinterpret_cast<int64_t*>(base + o_r1);
      auto* qoff = reinterpret_cast<int64_t*>(base + o_qo);
      // (1) per query: the leading probed lists holding >= k rows, their row count
      prefix_probes_kernel<<<unsigned((nq + 255) / 256), 256, 0, s>>>(probe, v->offsets, nq, n_probe, k, npq, call,
                                                                       rows1);
      DK_CHECK_LAUNCH();
      query_norms_kernel<<<unsigned((nq + 7) / 8), 256, 0, s>>>(Qd, nq, v->d, yyq);
      DK_CHECK_LAUNCH();
      size_t tb = cub2;
      DK_CUDA(cub::DeviceScan::ExclusiveSum(base + o_t2, tb, rows1, qoff, nq + 1, s));
      static const int span = [] {  // rows per list-major work item
        const char* e = std::getenv("DK_IVF_SPAN");
        return e ? std::max(128, std::atoi(e)) : 512;
      }();
      // (list, query) pairs bucketed by phase and list
      bucket_pairs_kernel<<<unsigned((npairs + 255) / 256), 256, 0, s>>>(probe, npq, nq, n_probe, v->C, kin, vin);
      DK_CHECK_LAUNCH();
      int bits = 1;
      while ((int64_t(1) << bits) < int64_t(NBK)) ++bits;
      tb = cub2;
      DK_CUDA(cub::DeviceRadixSort::SortPairs(base + o_t2, tb, kin, kout, vin, vout, int(npairs), 0, bits, s));
      list_pairs_kernel<<<unsigned((NBK + 1 + 255) / 256), 256, 0, s>>>(kout, npairs, NBK, ps);
      DK_CHECK_LAUNCH();
      list_items_kernel<<<unsigned((NBK + 1 + 255) / 256), 256, 0, s>>>(ps, v->offsets, v->C, NBK, PQ, span,
                                                                         ni);
      DK_CHECK_LAUNCH();
      tb = cub2;
      DK_CUDA(cub::DeviceScan::ExclusiveSum(base + o_t2, tb, ni, is, NBK + 1, s));
      int64_t tot1 = 0, items1 = 0, items2 = 0;  // phase-1 keys, items of either phase
      DK_CUDA(cudaMemcpyAsync(&tot1, qoff + nq, 8, cudaMemcpyDeviceToHost, s));
      DK_CUDA(cudaMemcpyAsync(&items1, is + v->C, 8, cudaMemcpyDeviceToHost, s));
      DK_CUDA(cudaMemcpyAsync(&items2, is + (NBK - 1), 8, cudaMemcpyDeviceToHost, s));
      DK_CUDA(cudaStreamSynchronize(s));
      items2 -= items1;
      const size_t kbytes = size_t(std::max<int64_t>(tot1, 1)) * sizeof(K128);
      if (kbytes > v->keys1_bytes) {
        if (v->keys1) DK_CUDA(cudaFree(v->keys1));
        v->keys1 = nullptr;
        v->keys1_bytes = 0;
        DK_CUDA(cudaMalloc(&v->keys1, kbytes));
        v->keys1_bytes = kbytes;
      }
      auto* keys1 = static_cast<K128*>(v->keys1);
      // (2) every key of the leading lists, then the exact top-k of each query -> tau_q
      if (items1 > 0) {
        if (ref32)
          pair_tile_kernel<2><<<unsigned(items1), 128, 0, s>>>(v->xs, v->xns, v->rows, v->offsets, v->d, v->C, Qd,
                                                               yyq, probe, n_probe, vout, ps, is, 0, v->C, span, qoff,
                                                               keys1, nullptr, 0, nullptr, nullptr);
        else
          pair_tile_kernel<0><<<unsigned(items1), 128, 0, s>>>(v->xs, v->xns, v->rows, v->offsets, v->d, v->C, Qd,
                                                               yyq, probe, n_probe, vout, ps, is, 0, v->C, span, qoff,
                                                               keys1, nullptr, 0, nullptr, nullptr);
      }
      DK_CHECK_LAUNCH();
      const size_t tsm = size_t(NB) * sizeof(K128);
      set_dynamic_smem(seg_topk_kernel, tsm);
      seg_topk_kernel<<<unsigned(nq), 256, tsm, s>>>(nullptr, nullptr, nullptr, keys1, qoff, 0, nullptr, 0, NB, k,
                                                     nullptr, idx1, d21, cnt1, tau, nullptr);
      DK_CHECK_LAUNCH();
      // (3) the remaining pairs: keys below tau_q into the query's candidate buffer
      DK_CUDA(cudaMemsetAsync(ccnt, 0, size_t(nq) * 4, s));
      static const bool f64_filter = std::getenv("DK_IVF_F64_FILTER") != nullptr;  // A/B switch
      if (ref32) {
        if (items2 > 0)
          pair_tile_kernel<3><<<unsigned(items2), 128, 0, s>>>(v->xs, v->xns, v->rows, v->offsets, v->d, v->C, Qd,
                                                               yyq, probe, n_probe, vout, ps, is, v->C + 1, NBK - 1,
                                                               span, nullptr, nullptr, tau, cap, cand, ccnt);
      } else if (f64_filter) {
        if (items2 > 0)
          pair_tile_kernel<1><<<unsigned(items2), 128, 0, s>>>(v->xs, v->xns, v->rows, v->offsets, v->d, v->C, Qd, yyq, probe,
                                                 n_probe, vout, ps, is, v->C + 1, NBK - 1, span, nullptr, nullptr, tau, cap,
                                                 cand, ccnt);
      } else {
        auto* Qf = reinterpret_cast<float*>(base + o_qf);
        to_f32_kernel<<<unsigned((nq * v->d + 255) / 256), 256, 0, s>>>(Qd, nq * v->d, Qf);
        DK_CHECK_LAUNCH();
        if (items2 > 0) {
          if ((v->d & 3) == 0) {
            set_dynamic_smem(pair_filter_f32_kernel<true>, kFilterSmem);
            pair_filter_f32_kernel<true><<<unsigned(items2), 128, kFilterSmem, s>>>(
                v->xs, v->xns, v->rows, v->offsets, v->d, v->C, Qd, Qf, yyq, n_probe, vout, ps, is, v->C + 1,
                NBK - 1, span, tau, cap, cand, ccnt);
          } else {
            set_dynamic_smem(pair_filter_f32_kernel<false>, kFilterSmem);
            pair_filter_f32_kernel<false><<<unsigned(items2), 128, kFilterSmem, s>>>(
                v->xs, v->xns, v->rows, v->offsets, v->d, v->C, Qd, Qf, yyq, n_probe, vout, ps, is, v->C + 1,
                NBK - 1, span, tau, cap, cand, ccnt);
          }
        }
      }
      DK_CHECK_LAUNCH();
      // (4) top-k of the phase-1 top-k and the candidates
      seg_topk_kernel<<<unsigned(nq), 256, tsm, s>>>(idx1, d21, cnt1, cand, nullptr, cap, ccnt, cap, NB, k, call, io,
                                                     dd, co, nullptr, ovf);
      DK_CHECK_LAUNCH();
      std::vector<int32_t> ov(static_cast<size_t>(nq));
      DK_CUDA(cudaMemcpyAsync(ov.data(), ovf, size_t(nq) * 4, cudaMemcpyDeviceToHost, s));
      DK_CUDA(cudaStreamSynchronize(s));
      std::vector<int32_t> redo;
      for (int64_t q = 0; q < nq; ++q)
        if (ov[size_t(q)]) redo.push_back(int32_t(q));
      if (std::getenv("DK_IVF_DEBUG")) {
        std::vector<int32_t> cc(static_cast<size_t>(nq));
        DK_CUDA(cudaMemcpy(cc.data(), ccnt, size_t(nq) * 4, cudaMemcpyDeviceToHost));
        std::vector<int32_t> srt(cc);
        std::sort(srt.begin(), srt.end());
        fprintf(stderr, "ivf two-phase: redo %zu, cand p50 %d p90 %d p99 %d max %d\n", redo.size(),
                srt[srt.size() / 2], srt[srt.size() * 9 / 10], srt[srt.size() * 99 / 100], srt.back());
      }
      // candidate buffer overflowed (queries far from every list, whose tau_q passes most rows):
      // every probed key of those queries through the list-major pass, then the top-k
      for (size_t r0 = 0; r0 < redo.size(); r0 += size_t(redo_R)) {
        const int64_t nr = int64_t(std::min(redo.size() - r0, size_t(redo_R)));
        auto* rq = reinterpret_cast<int32_t*>(base + o_rq);
        auto* Qr = reinterpret_cast<double*>(base + o_rQ);
        auto* pr = reinterpret_cast<int32_t*>(base + o_rp);
        DK_CUDA(cudaMemcpyAsync(rq, redo.data() + r0, size_t(nr) * 4, cudaMemcpyHostToDevice, s));
        redo_compact_kernel<<<unsigned(nr), 128, 0, s>>>(rq, nr, Qd, v->d, probe, n_probe, Qr, pr);
        DK_CHECK_LAUNCH();
        const int64_t rpairs = nr * n_probe;
        prefix_probes_kernel<<<unsigned((nr + 255) / 256), 256, 0, s>>>(pr, v->offsets, nr, n_probe, INT_MAX, npq,
                                                                         call, rows1);
        DK_CHECK_LAUNCH();
        query_norms_kernel<<<unsigned((nr + 7) / 8), 256, 0, s>>>(Qr, nr, v->d, yyq);
        DK_CHECK_LAUNCH();
        size_t tb2 = cub2;
        DK_CUDA(cub::DeviceScan::ExclusiveSum(base + o_t2, tb2, rows1, qoff, nr + 1, s));
        bucket_pairs_kernel<<<unsigned((rpairs + 255) / 256), 256, 0, s>>>(pr, npq, nr, n_probe, v->C, kin, vin);
        DK_CHECK_LAUNCH();
        tb2 = cub2;
        DK_CUDA(cub::DeviceRadixSort::SortPairs(base + o_t2, tb2, kin, kout, vin, vout, int(rpairs), 0, bits, s));
        list_pairs_kernel<<<unsigned((NBK + 1 + 255) / 256), 256, 0, s>>>(kout, rpairs, NBK, ps);
        DK_CHECK_LAUNCH();
        list_items_kernel<<<unsigned((NBK + 1 + 255) / 256), 256, 0, s>>>(ps, v->offsets, v->C, NBK, PQ, 256,
                                                                           ni);
        DK_CHECK_LAUNCH();
        tb2 = cub2;
        DK_CUDA(cub::DeviceScan::ExclusiveSum(base + o_t2, tb2, ni, is, NBK + 1, s));
        int64_t totr = 0, itemsr = 0;
        DK_CUDA(cudaMemcpyAsync(&totr, qoff + nr, 8, cudaMemcpyDeviceToHost, s));
        DK_CUDA(cudaMemcpyAsync(&itemsr, is + v->C, 8, cudaMemcpyDeviceToHost, s));
        DK_CUDA(cudaStreamSynchronize(s));
        const size_t rbytes = size_t(std::max<int64_t>(totr, 1)) * sizeof(K128);
        if (rbytes > v->keys1_bytes) {
          DK_CUDA(cudaFree(v->keys1));
          v->keys1 = nullptr;
          v->keys1_bytes = 0;
          DK_CUDA(cudaMalloc(&v->keys1, rbytes));
          v->keys1_bytes = rbytes;
        }
        auto* keysr = static_cast<K128*>(v->keys1);
        if (itemsr > 0) {
          if (ref32)
            pair_tile_kernel<2><<<unsigned(itemsr), 128, 0, s>>>(v->xs, v->xns, v->rows, v->offsets, v->d, v->C, Qr,
                                                                 yyq, pr, n_probe, vout, ps, is, 0, v->C, 256, qoff,
                                                                 keysr, nullptr, 0, nullptr, nullptr);
          else
            pair_tile_kernel<0><<<unsigned(itemsr), 128, 0, s>>>(v->xs, v->xns, v->rows, v->offsets, v->d, v->C, Qr,
                                                                 yyq, pr, n_probe, vout, ps, is, 0, v->C, 256, qoff,
                                                                 keysr, nullptr, 0, nullptr, nullptr);
        }
        DK_CHECK_LAUNCH();
        seg_topk_kernel<<<unsigned(nr), 256, tsm, s>>>(nullptr, nullptr, nullptr, keysr, qoff, 0, nullptr, 0, NB, k,
                                                       nullptr, idx1, d21, cnt1, nullptr, nullptr);
        DK_CHECK_LAUNCH();
        redo_scatter_kernel<<<unsigned(nr), 128, 0, s>>>(rq, nr, k, idx1, d21, cnt1, io, dd, co);
        DK_CHECK_LAUNCH();
      }
    }
    }
    if (ref32) {  // the fp32-ranked selection re-evaluated in fp64 and ordered by (d2, row)
      int P = 2;
      while (P < k) P <<= 1;
      const size_t fsm = size_t(P) * sizeof(K128);
      set_dynamic_smem(ref32_finish_kernel, fsm);
      ref32_finish_kernel<<<unsigned(nq), 128, fsm, s>>>(h->X, h->xn64, v->d, Qd,
                                                         reinterpret_cast<double*>(base + o_yy), k, P, io, co, io, dd,
                                                         co);
      DK_CHECK_LAUNCH();
    }
    if (!idev) DK_CUDA(cudaMemcpyAsync(idx_out, io, size_t(nq) * k * sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    if (!ddev) DK_CUDA(cudaMemcpyAsync(d2_out, dd, size_t(nq) * k * sizeof(double), cudaMemcpyDeviceToHost, s));
    if (!cdev) DK_CUDA(cudaMemcpyAsync(cnt_out, co, size_t(nq) * sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    if (!idev || !ddev || !cdev) DK_CUDA(cudaStreamSynchronize(s));
  });
}

dk_status dk_deann_ivf(dk_ivf_handle v, const double* Q, int64_t nq, int32_t family, double bandwidth,
                       int32_t k, int32_t m, int32_t n_probe, uint64_t seed, int64_t query_base,
                       double* value_out, int32_t* khat_out, void* stream) {
  DK_NVTX();
  return guard([&] {
    DK_REQUIRE(v != nullptr, "NULL handle");
    DK_REQUIRE(family == DK_GAUSSIAN || family == DK_EXPONENTIAL || family == DK_LAPLACIAN,
               "unknown kernel family " + std::to_string(family));
    DK_REQUIRE(std::isfinite(bandwidth) && bandwidth > 0.0,
               "bandwidth must be positive and finite, got " + std::to_string(bandwidth));
    dk_dataset* h = v->ds;
    const int64_t n = h->n;
    DK_REQUIRE(h->global_offset == 0 && h->global_n == n, "dk_deann_ivf runs on an unsharded handle");
    DK_REQUIRE(k >= 1 && int64_t(k) <= n, "k=" + std::to_string(k) + " out of range [1, " + std::to_string(n) + "]");
    DK_REQUIRE(m >= 0, "m=" + std::to_string(m) + " must be >= 0");
    DK_REQUIRE(!(m > 0 && int64_t(k) >= n), "m > 0 requires k + 1 <= n so the remainder is nonempty");
    DK_REQUIRE(nq >= 0, "negative query count");
    if (nq == 0) return;
    DK_REQUIRE(Q != nullptr && value_out != nullptr, "NULL argument");
    DeviceGuard g(h->device);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const bool long_excl = m > 0 && k > kSmemSortMax;
    const size_t seg_bytes = long_excl ? seg_sort_temp_bytes(k, nq) : 0;
    size_t off = 0;
    auto take = [&](size_t bytes) {
      const size_t a = (off + 255) & ~size_t(255);
      off = a + bytes;
      return a;
    };
    const size_t o_q = take(size_t(nq) * h->d * 8), o_i = take(size_t(nq) * k * 8), o_d = take(size_t(nq) * k * 8);
    const size_t o_c = take(size_t(nq) * 4), o_s = take(m > 0 ? size_t(nq) * k * 8 : 8);
    const size_t o_z1 = take(size_t(nq) * 8), o_z2 = take(size_t(nq) * 8), o_v = take(size_t(nq) * 8);
    const size_t o_g = take(seg_bytes);
    if (off > v->dws_bytes) {
      if (v->dws) DK_CUDA(cudaFree(v->dws));
      v->dws = nullptr;
      v->dws_bytes = 0;
      DK_CUDA(cudaMalloc(&v->dws, off));
      v->dws_bytes = off;
    }
    uint8_t* base = static_cast<uint8_t*>(v->dws);
    const double* Qd = Q;
    if (!is_device_ptr(Q)) {
      DK_CUDA(cudaMemcpyAsync(base + o_q, Q, size_t(nq) * h->d * 8, cudaMemcpyHostToDevice, s));
      Qd = reinterpret_cast<const double*>(base + o_q);
    }
    auto* idx = reinterpret_cast<int64_t*>(base + o_i);
    auto* d2 = reinterpret_cast<double*>(base + o_d);
    auto* cnt = reinterpret_cast<int32_t*>(base + o_c);
    auto* z1 = reinterpret_cast<double*>(base + o_z1);
    auto* z2 = reinterpret_cast<double*>(base + o_z2);
    const dk_status st = dk_ivf_query(v, Qd, nq, k, n_probe, 1, idx, d2, cnt, stream);
    if (st != DK_OK) throw Error{st, dk_last_error()};
    if (family == DK_LAPLACIAN) launch_eval_rows(h->X, n, 0, h->d, Qd, nq, family, bandwidth, idx, cnt, k, z1, s);
    if (m > 0) {
      auto* srt = reinterpret_cast<int64_t*>(base + o_s);
      if (long_excl) launch_seg_sort_i64(idx, srt, cnt, k, nq, base + o_g, seg_bytes, s);
      else launch_sort_excl(idx, cnt, k, nq, srt, s);
      launch_sample(h->X, n, 0, n, h->d, Qd, nq, family, bandwidth, m, seed, query_base, srt, cnt, k, z2, nullptr,
                    nullptr, s);
    }
    const bool v_dev = is_device_ptr(value_out);
    double* vd = v_dev ? value_out : reinterpret_cast<double*>(base + o_v);
    launch_deann_combine(nq, family, bandwidth, k, m, n, d2, z1, z2, vd, s, cnt);
    bool sync = false;
    if (!v_dev) {
      DK_CUDA(cudaMemcpyAsync(value_out, vd, size_t(nq) * 8, cudaMemcpyDeviceToHost, s));
      sync = true;
    }
    if (khat_out) {
      DK_CUDA(cudaMemcpyAsync(khat_out, cnt, size_t(nq) * 4, cudaMemcpyDefault, s));
      sync = sync || !is_device_ptr(khat_out);
    }
    if (sync) DK_CUDA(cudaStreamSynchronize(s));
  });
}

}  // extern "C"
