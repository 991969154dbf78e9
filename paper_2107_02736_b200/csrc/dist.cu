// dist.cu — materialised squared-distance matrices (batch_sqdist / window_sqdist).
//
// Reference: distance.py:58-123.  The fused KDE never writes the N x n matrix; these
// entry points exist for callers of the reference's distance API.  Same arithmetic as
// the reference: the norms identity in fp64, d2 = ((q.x) * -2 + |q|^2) + |x|^2, the most
// negative entry reported before clamping at 0 (NormConsistencyError is raised by the
// Python layer exactly as _clamp does).  The dot products are a register-tiled fp64
// "GEMM": 64 queries x 64 rows per block, 4 x 4 per thread, K staged in chunks of 16.
#include <cstring>

#include "internal.h"

namespace dk {
namespace {

constexpr int TQ = 64, TR = 64, TK = 16;

__device__ __forceinline__ unsigned long long ordered_bits(double v) {
  const unsigned long long b = static_cast<unsigned long long>(__double_as_longlong(v));
  return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}

__global__ void qnorm_kernel(const double* __restrict__ Q, int64_t nq, int32_t d, double* __restrict__ qn) {
  const int64_t q = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (q >= nq) return;
  double s = 0.0;
  for (int j = lane; j < d; j += 32) s = fma(Q[q * d + j], Q[q * d + j], s);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) qn[q] = s;
}

__global__ void __launch_bounds__(256) sqdist_kernel(const float* __restrict__ X, int64_t row0, int64_t nrows,
                                                     int32_t d, const double* __restrict__ xn,
                                                     const double* __restrict__ Q, int64_t nq,
                                                     const double* __restrict__ qn, double* __restrict__ out,
                                                     unsigned long long* __restrict__ worst) {
  __shared__ double qs[TK][TQ + 1];
  __shared__ __align__(16) double xs[TK][TR];
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;  // tx: 4 rows, ty: 4 queries
  const int64_t r0 = int64_t(blockIdx.x) * TR, q0 = int64_t(blockIdx.y) * TQ;
  double acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.0;
  for (int k0 = 0; k0 < d; k0 += TK) {
    for (int e = threadIdx.x; e < TQ * TK; e += 256) {
      const int qq = e / TK, kk = e % TK;
      qs[kk][qq] = (q0 + qq < nq && k0 + kk < d) ? Q[(q0 + qq) * d + k0 + kk] : 0.0;
    }
    for (int e = threadIdx.x; e < TR * TK; e += 256) {
      const int rr = e / TK, kk = e % TK;
      xs[kk][rr] = (r0 + rr < nrows && k0 + kk < d) ? double(X[(row0 + r0 + rr) * d + k0 + kk]) : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < TK; ++kk) {
      double a[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = qs[kk][ty * 4 + i];
      const double2 b01 = *reinterpret_cast<const double2*>(&xs[kk][tx * 4]);
      const double2 b23 = *reinterpret_cast<const double2*>(&xs[kk][tx * 4 + 2]);
      const double b[4] = {b01.x, b01.y, b23.x, b23.y};
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fma(a[i], b[j], acc[i][j]);
    }
    __syncthreads();
  }
  double lo = __longlong_as_double(0x7ff0000000000000ll);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int64_t q = q0 + ty * 4 + i;
    if (q >= nq) continue;
    const double qv = qn[q];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int64_t r = r0 + tx * 4 + j;
      if (r >= nrows) continue;
      double t = acc[i][j] * -2.0;
      t += qv;
      t += xn[row0 + r];
      lo = fmin(lo, t);
      out[q * nrows + r] = fmax(t, 0.0);
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) lo = fmin(lo, __shfl_xor_sync(0xffffffffu, lo, o));
  if ((threadIdx.x & 31) == 0) atomicMin(worst, ordered_bits(lo));
}

}  // namespace
}  // namespace dk

using namespace dk;

extern "C" dk_status dk_sqdist(dk_handle h, const double* Q, int64_t nq, const double* x_norms, int64_t row_begin,
                               int64_t row_count, double* out, double* worst_out, void* stream) {
  return guard([&] {
    DK_REQUIRE(h != nullptr, "NULL handle");
    DK_REQUIRE(nq >= 0 && row_begin >= 0 && row_count >= 0 && row_begin + row_count <= h->n,
               "query count or row range out of range");
    if (worst_out) *worst_out = 0.0;
    if (nq == 0 || row_count == 0) return;
    DK_REQUIRE(Q != nullptr && out != nullptr, "NULL argument");
    DeviceGuard g(h->device);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    size_t off = 0;
    auto take = [&](size_t bytes) {
      const size_t a = (off + 255) & ~size_t(255);
      off = a + bytes;
      return a;
    };
    const size_t o_q = take(size_t(nq) * h->d * sizeof(double));
    const size_t o_qn = take(size_t(nq) * sizeof(double));
    const size_t o_xn = take(size_t(h->n) * sizeof(double));
    const size_t o_w = take(sizeof(unsigned long long));
    const bool odev = is_device_ptr(out);
    const size_t o_o = take(odev ? 1 : size_t(nq) * row_count * sizeof(double));
    h->ws.reserve(off);
    uint8_t* base = h->ws.base;
    const double* Qd = Q;
    if (!is_device_ptr(Q)) {
      DK_CUDA(cudaMemcpyAsync(base + o_q, Q, size_t(nq) * h->d * sizeof(double), cudaMemcpyHostToDevice, s));
      Qd = reinterpret_cast<const double*>(base + o_q);
    }
    const double* xn = h->xn64;
    if (x_norms) {  // caller-supplied cached norms (a reference Dataset's sq_norms), as data.py keeps them
      if (is_device_ptr(x_norms)) {
        xn = x_norms;
      } else {
        DK_CUDA(cudaMemcpyAsync(base + o_xn, x_norms, size_t(h->n) * sizeof(double), cudaMemcpyHostToDevice, s));
        xn = reinterpret_cast<const double*>(base + o_xn);
      }
    }
    auto* qn = reinterpret_cast<double*>(base + o_qn);
    auto* w = reinterpret_cast<unsigned long long*>(base + o_w);
    DK_CUDA(cudaMemsetAsync(w, 0xff, sizeof(unsigned long long), s));
    qnorm_kernel<<<unsigned((nq * 32 + 255) / 256), 256, 0, s>>>(Qd, nq, h->d, qn);
    DK_CHECK_LAUNCH();
    double* od = odev ? out : reinterpret_cast<double*>(base + o_o);
    dim3 grid(unsigned((row_count + TR - 1) / TR), unsigned((nq + TQ - 1) / TQ));
    sqdist_kernel<<<grid, 256, 0, s>>>(h->X, row_begin, row_count, h->d, xn, Qd, nq, qn, od, w);
    DK_CHECK_LAUNCH();
    if (!odev) DK_CUDA(cudaMemcpyAsync(out, od, size_t(nq) * row_count * sizeof(double), cudaMemcpyDeviceToHost, s));
    unsigned long long wb = 0;
    DK_CUDA(cudaMemcpyAsync(&wb, w, sizeof(wb), cudaMemcpyDeviceToHost, s));
    DK_CUDA(cudaStreamSynchronize(s));
    const unsigned long long raw = (wb >> 63) ? (wb & 0x7fffffffffffffffull) : ~wb;
    double worst;
    std::memcpy(&worst, &raw, sizeof(worst));
    if (worst_out) *worst_out = worst;
  });
}
