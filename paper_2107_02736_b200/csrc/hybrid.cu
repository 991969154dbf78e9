// hybrid.cu — bookkeeping kernels of the two-precision exact gaussian KDE (capi.cu kde_hybrid).
//
// The KDE of a query is dominated by the rows near it.  A single-pass fp16 sweep (MODE_KDE_COLD,
// one MMA pass instead of split3's three) sums every 128-column tile half whose fp32 sum is at
// most hot_thr and marks the others ("hot") in a bitmap; the hot (query block, tile) pairs are
// listed here and swept again in split3 (MODE_KDE_HOT), which sums exactly the marked halves.
// Every (query, row) pair is evaluated once at its precision.  The fp16 part carries the proven
// bound |approx d2 - d2| <= eps_q of the k-NN encoding, so its sum S_cold is off by at most
// S_cold * expm1(eps_q / 2h^2); the combine kernel checks that bound per query against tol x S
// and lists the queries that fail it for an exact split3 recomputation (none on c3).
// Reference: naive_kde estimators.py:144-149 (the value computed), kernels.py:65-83 (gaussian).

#include "internal.h"
#include "tile_kernel.cuh"

namespace dk {

namespace {

// per block of 128 (ball-sorted) queries: the tiles with any hot half, in increasing order
__global__ void __launch_bounds__(256) hot_lists_kernel(const uint32_t* __restrict__ bits, int32_t ntiles,
                                                        int32_t* __restrict__ tlist, int32_t* __restrict__ tcount) {
  __shared__ int s_wcnt[8];
  __shared__ int s_base;
  const int qb = blockIdx.x;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) s_base = 0;
  __syncthreads();
  const uint4* b4 = reinterpret_cast<const uint4*>(bits + size_t(qb) * ntiles * kHotWords);
  for (int t0 = 0; t0 < ntiles; t0 += blockDim.x) {
    const int t = t0 + int(threadIdx.x);
    bool on = false;
    if (t < ntiles) {
      const uint4 a = b4[2 * size_t(t)], b = b4[2 * size_t(t) + 1];
      on = ((a.x | a.y | a.z | a.w) | (b.x | b.y | b.z | b.w)) != 0u;
    }
    const uint32_t m = __ballot_sync(0xffffffffu, on);
    if (lane == 0) s_wcnt[warp] = __popc(m);
    __syncthreads();
    int off = s_base;
    for (int w = 0; w < warp; ++w) off += s_wcnt[w];
    if (on) tlist[size_t(qb) * ntiles + off + __popc(m & ((1u << lane) - 1u))] = t;
    __syncthreads();
    if (threadIdx.x == 0) {
      int tot = 0;
      for (int w = 0; w < 8; ++w) tot += s_wcnt[w];
      s_base += tot;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) tcount[qb] = s_base;
}

// work units of the split3 sweep: block b's list is cut into at most kHotUnitsPerBlock units of
// >= 8 tiles (unit = (b, [i0, i1)) in the flat list b * ntiles + i).  One CTA; ubeg / ucnt give
// each block's units to the combine kernel, scal[0] = unit count, scal[1] = listed pairs.
__global__ void __launch_bounds__(1024) hot_units_kernel(const int32_t* __restrict__ tcount, int32_t nqb,
                                                         int32_t ntiles, int32_t* __restrict__ ubeg,
                                                         int32_t* __restrict__ ucnt, int32_t* __restrict__ scal,
                                                         int32_t* __restrict__ ulist) {
  __shared__ int s_w[32];
  __shared__ int s_pairs;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) s_pairs = 0;
  __syncthreads();
  int carry = 0;
  for (int b0 = 0; b0 < nqb; b0 += 1024) {
    const int b = b0 + tid;
    const int c = b < nqb ? tcount[b] : 0;
    const int U = max(8, (c + kHotUnitsPerBlock - 1) / kHotUnitsPerBlock);
    const int nu = (c + U - 1) / U;
    int incl = nu;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int v = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += v;
    }
    if (lane == 31) s_w[warp] = incl;
    if (c) atomicAdd(&s_pairs, c);
    __syncthreads();
    if (warp == 0) {
      int v = s_w[lane];
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int w = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += w;
      }
      s_w[lane] = v;
    }
    __syncthreads();
    const int first = carry + incl - nu + (warp ? s_w[warp - 1] : 0);
    if (b < nqb) {
      ubeg[b] = first;
      ucnt[b] = nu;
      for (int i = 0, u = first; i < c; i += U, ++u) {
        ulist[3 * u] = b;
        ulist[3 * u + 1] = int32_t(int64_t(b) * ntiles + i);
        ulist[3 * u + 2] = int32_t(int64_t(b) * ntiles + min(c, i + U));
      }
    }
    carry += s_w[31];
    __syncthreads();
  }
  if (tid == 0) {
    scal[0] = carry;
    scal[1] = s_pairs;
  }
}

// per ball-sorted query row r: S = S_cold + S_hot in a fixed order, the fp16 bound, the output
// (scattered back to the batch order) and the list of queries whose bound fails
__global__ void hyb_combine_kernel(const double* __restrict__ part_cold, int32_t nparts, int32_t nq_pad, int64_t bn,
                                   const double* __restrict__ part_hot, const int32_t* __restrict__ ubeg,
                                   const int32_t* __restrict__ ucnt, const float* __restrict__ qn, float eps_rel,
                                   float xn_max, double inv2h2, double tol, double scale,
                                   const int32_t* __restrict__ qperm, int64_t qbase, double* __restrict__ out,
                                   int32_t* __restrict__ fail, int32_t* __restrict__ nfail, double* __restrict__ bound_out) {
  const int64_t r = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (r >= bn) return;
  double cold = 0.0;
  for (int i = 0; i < nparts; ++i) cold += part_cold[size_t(i) * nq_pad + r];
  const int b = int(r / kBM), lr = int(r % kBM);
  double hot = 0.0;
  const int u0 = ubeg[b], u1 = u0 + ucnt[b];
  for (int u = u0; u < u1; ++u)
#pragma unroll
    for (int cg = 0; cg < kColGroups; ++cg) hot += part_hot[(size_t(u) * kColGroups + cg) * kBM + lr];
  const double S = cold + hot;
  // |d2~ - d2| <= eps_q on every fp16 pair: each cold term is within a factor exp(+-eps_q / 2h^2)
  const double eps_q = double(eps_rel) * (double(qn[r]) + double(xn_max));
  const double bound = cold * expm1(eps_q * inv2h2) * (1.0 + 1e-6);
  const int32_t q = qperm[r];
  out[q] = S * scale;
  if (bound_out) bound_out[q] = S > 0.0 ? bound / S : (bound > 0.0 ? INFINITY : 0.0);
  if (!(bound <= tol * S)) {
    const int32_t i = atomicAdd(nfail, 1);
    fail[i] = int32_t(qbase + q);
  }
}

__global__ void scatter_f64_kernel(const double* __restrict__ v, const int32_t* __restrict__ idx, int64_t n,
                                   double* __restrict__ out) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) out[idx[i]] = v[i];
}

}  // namespace

void launch_hot_lists(const uint32_t* bits, int32_t nqb, int32_t ntiles, int32_t* tlist, int32_t* tcount,
                      cudaStream_t s) {
  hot_lists_kernel<<<unsigned(nqb), 256, 0, s>>>(bits, ntiles, tlist, tcount);
  DK_CHECK_LAUNCH();
}

void launch_hot_units(const int32_t* tcount, int32_t nqb, int32_t ntiles, int32_t* ubeg, int32_t* ucnt,
                      int32_t* scal, int32_t* ulist, cudaStream_t s) {
  hot_units_kernel<<<1, 1024, 0, s>>>(tcount, nqb, ntiles, ubeg, ucnt, scal, ulist);
  DK_CHECK_LAUNCH();
}

void launch_hyb_combine(const double* part_cold, int32_t nparts, int32_t nq_pad, int64_t bn, const double* part_hot,
                        const int32_t* ubeg, const int32_t* ucnt, const float* qn, float eps_rel, float xn_max,
                        double inv2h2, double tol, double scale, const int32_t* qperm, int64_t qbase, double* out,
                        int32_t* fail, int32_t* nfail, double* bound_out, cudaStream_t s) {
  if (bn <= 0) return;
  hyb_combine_kernel<<<unsigned((bn + 127) / 128), 128, 0, s>>>(part_cold, nparts, nq_pad, bn, part_hot, ubeg, ucnt,
                                                                 qn, eps_rel, xn_max, inv2h2, tol, scale, qperm, qbase,
                                                                 out, fail, nfail, bound_out);
  DK_CHECK_LAUNCH();
}

void launch_scatter_f64(const double* v, const int32_t* idx, int64_t n, double* out, cudaStream_t s) {
  if (n <= 0) return;
  scatter_f64_kernel<<<unsigned((n + 255) / 256), 256, 0, s>>>(v, idx, n, out);
  DK_CHECK_LAUNCH();
}

}  // namespace dk
