// bigk.cu — exact k-NN for very large k (k > 4096, up to n) and long exclusion lists.
//
// The tile-based selection (knn.cu) keeps k <= 4096 candidates in shared memory.
// The reference accepts any 1 <= k <= n (ann.py:107-108; e.g. deann(k=n, m=0),
// acceptance 2), so larger k take an exact path: fp64 direct-difference squared
// distances to every row, then a stable LSD radix sort of (d2 bits, row id) —
// stability keeps equal distances in increasing row order, i.e. the reference's
// lower-index tie break (_smallest_k, ann.py:82-102).  Exclusion lists longer
// than the shared-memory bitonic sort holds are sorted the same way.
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_segmented_radix_sort.cuh>

#include "internal.h"

namespace dk {

namespace {

// one warp per row: fp64 squared distance (bits as a sortable key, d2 >= 0) and the row id
__global__ void exact_d2_all_kernel(const float* __restrict__ X, int64_t n, int32_t d, const double* __restrict__ q,
                                    unsigned long long* __restrict__ keys, int64_t* __restrict__ vals) {
  const int64_t row = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (row >= n) return;
  const float* x = X + row * d;
  double s = 0.0;
  for (int k = lane; k < d; k += 32) {
    const double t = double(x[k]) - q[k];
    s = fma(t, t, s);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) {
    keys[row] = static_cast<unsigned long long>(__double_as_longlong(s));
    vals[row] = row;
  }
}

__global__ void take_k_kernel(const unsigned long long* __restrict__ keys, const int64_t* __restrict__ vals, int32_t k,
                              int64_t offset, int64_t* __restrict__ idx_out, double* __restrict__ d2_out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= k) return;
  idx_out[i] = vals[i] + offset;
  d2_out[i] = __longlong_as_double(static_cast<long long>(keys[i]));
}

__global__ void gather_positions_kernel(const int64_t* __restrict__ ids, const int64_t* __restrict__ inverse,
                                        int64_t count, int64_t* __restrict__ out) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < count) out[i] = inverse[ids[i]];
}

__global__ void seg_offsets_kernel(const int32_t* __restrict__ cnt, int32_t stride, int64_t nq,
                                   int64_t* __restrict__ begin, int64_t* __restrict__ end) {
  const int64_t j = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (j >= nq) return;
  begin[j] = j * stride;
  end[j] = j * stride + (cnt ? cnt[j] : stride);
}

void* align256(void* p) { return reinterpret_cast<void*>((reinterpret_cast<uintptr_t>(p) + 255) & ~uintptr_t(255)); }

}  // namespace

size_t bigk_temp_bytes(int64_t n) {
  size_t pairs = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, pairs, static_cast<const unsigned long long*>(nullptr),
                                  static_cast<unsigned long long*>(nullptr), static_cast<const int64_t*>(nullptr),
                                  static_cast<int64_t*>(nullptr), n);
  return pairs + 4 * size_t(n) * 8 + 1024;
}

void launch_knn_bigk(const float* X, int64_t n, int64_t offset, int32_t d, const double* Q, int64_t nq, int32_t k,
                     int64_t* idx_out, double* d2_out, void* temp, size_t temp_bytes, cudaStream_t s) {
  uint8_t* t = static_cast<uint8_t*>(temp);
  auto* k_in = reinterpret_cast<unsigned long long*>(t);
  auto* k_out = k_in + n;
  auto* v_in = reinterpret_cast<int64_t*>(k_out + n);
  auto* v_out = v_in + n;
  void* cub_temp = align256(v_out + n);
  size_t cub_bytes = temp_bytes - 4 * size_t(n) * 8 - 256;
  for (int64_t j = 0; j < nq; ++j) {
    exact_d2_all_kernel<<<unsigned((n * 32 + 255) / 256), 256, 0, s>>>(X, n, d, Q + j * d, k_in, v_in);
    DK_CHECK_LAUNCH();
    DK_CUDA(cub::DeviceRadixSort::SortPairs(cub_temp, cub_bytes, k_in, k_out, v_in, v_out, n, 0, 64, s));
    take_k_kernel<<<unsigned((k + 255) / 256), 256, 0, s>>>(k_out, v_out, k, offset, idx_out + j * k, d2_out + j * k);
    DK_CHECK_LAUNCH();
  }
}

size_t seg_sort_temp_bytes(int32_t stride, int64_t nq) {
  const int64_t chunk = std::min(nq, std::max<int64_t>(1, (int64_t(1) << 30) / stride));
  size_t bytes = 0;
  cub::DeviceSegmentedRadixSort::SortKeys(nullptr, bytes, static_cast<const int64_t*>(nullptr),
                                          static_cast<int64_t*>(nullptr), int(chunk * stride), int(chunk),
                                          static_cast<const int64_t*>(nullptr), static_cast<const int64_t*>(nullptr));
  return bytes + 2 * size_t(nq) * sizeof(int64_t) + 1024;
}

// Each query's list (the first cnt[j] of `stride` slots, or all of them) sorted
// ascending into out — the long-list counterpart of the shared-memory bitonic
// sorts (sample.cu sort_excl_kernel, rsp.cu map_sort_kernel).  Slots past cnt[j]
// are left unwritten; every consumer reads only the first cnt[j].
void launch_seg_sort_i64(const int64_t* in, int64_t* out, const int32_t* cnt, int32_t stride, int64_t nq, void* temp,
                         size_t temp_bytes, cudaStream_t s) {
  auto* begin = static_cast<int64_t*>(temp);
  auto* end = begin + nq;
  void* cub_temp = align256(end + nq);
  const size_t cub_bytes = temp_bytes - 2 * size_t(nq) * sizeof(int64_t) - 256;
  // CUB counts items in int: sort in chunks of queries holding < 2^30 slots
  const int64_t chunk = std::max<int64_t>(1, (int64_t(1) << 30) / stride);
  for (int64_t j0 = 0; j0 < nq; j0 += chunk) {
    const int64_t cn = std::min(chunk, nq - j0);
    seg_offsets_kernel<<<unsigned((cn + 255) / 256), 256, 0, s>>>(cnt ? cnt + j0 : nullptr, stride, cn, begin, end);
    DK_CHECK_LAUNCH();
    size_t bytes = cub_bytes;
    DK_CUDA(cub::DeviceSegmentedRadixSort::SortKeys(cub_temp, bytes, in + j0 * stride, out + j0 * stride,
                                                    int(cn * stride), int(cn), begin, end, 0, 64, s));
  }
}

void launch_gather_positions(const int64_t* ids, const int64_t* inverse, int64_t count, int64_t* out, cudaStream_t s) {
  gather_positions_kernel<<<unsigned((count + 255) / 256), 256, 0, s>>>(ids, inverse, count, out);
  DK_CHECK_LAUNCH();
}

}  // namespace dk
