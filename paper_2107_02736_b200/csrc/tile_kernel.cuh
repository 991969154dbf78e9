// tile_kernel.cuh — the fused tcgen05 distance-tile kernel (K1 / K2 of DESIGN.md).
//
// One persistent CTA per SM sweeps work units (query block of 128 rows) x
// (chunk of 256-column dataset tiles).  Roles:
//   warp 0      TMA producer (one elected lane): A = query block (resident in
//               smem for the whole unit when it fits), B = 256x64 dataset
//               K-blocks through a multi-stage mbarrier ring, plus the tile's
//               256 column norms (1 KB bulk copy into a 4-slot ring).
//   warp 1      MMA issuer (one lane): tcgen05.mma kind::f16, M=128 N=256,
//               fp32 accumulator in TMEM, 2 accumulator buffers x 256 cols.
//   warp 2      TMEM allocator.
//   warps 4-19  epilogue: warp w reads TMEM lane quarter (w%4) and 64-column
//               group (w-4)/4 with tcgen05.ld; each thread owns ONE query row,
//               so the per-query row sum needs no shuffles.
// The S = Q X^T tile never leaves the SM: the epilogue turns it into
//   d2 = |q|^2 + |x|^2 - 2 S          (fp32, exact for the integer encoding)
// and then, by mode,
//   KDE_GAUSS  sum exp2(d2 * -log2e/(2h^2))       -> naive_kde gaussian
//   KDE_EXP    sum exp2(sqrt(d2) * -log2e/h)       -> naive_kde exponential
//   TILEMIN    min d2 over segments of `seg_tiles` tiles (k-NN threshold pass)
//   FILTER     keep (d2, col) with d2 <= tau[row]    (k-NN candidate pass)
// The gaussian epilogue does the per-element arithmetic on packed f32x2
// (FADD2 / FFMA2 / FMUL2) and evaluates a fixed fraction of the exponentials
// with a polynomial on the FMA pipe instead of MUFU.EX2, balancing the two
// pipes (the SFU alone would bound the kernel).
// Reference: naive_kde estimators.py:144-149 -> batch_sqdist distance.py:69-85
// -> kernel_from_distance kernels.py:65-83 -> .mean(axis=1); brute_force_knn
// ann.py:105-111.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <type_traits>
#include "ptx.cuh"

namespace dk {

#ifdef DK_TIMING
// debug-only wait accounting (scripts/epi_timing.py): [0] epilogue tfull wait cycles,
// [1] epilogue xfull wait, [2] epilogue busy cycles, [3] MMA tempty wait, [4] MMA full wait,
// [5] producer empty wait, [6] epilogue tile count
__device__ unsigned long long g_dbg[8];
#define DK_TWAIT(slot, call)               \
  do {                                     \
    const long long t0_ = clock64();       \
    call;                                  \
    dbgw[slot] += clock64() - t0_;         \
  } while (0)
#else
#define DK_TWAIT(slot, call) call
#endif

enum TileMode : int {
  MODE_KDE_GAUSS = 0,
  MODE_KDE_EXP = 1,
  MODE_TILEMIN = 2,
  MODE_FILTER = 3,
  MODE_NULL = 4,
  MODE_KDE_GAUSS_MUFU = 5,  // gaussian with every exponential on MUFU (MMA-heavy encodings)
  MODE_HIST = 6,            // k-NN threshold refinement: per-query histogram of approx d2 (listed sweeps)
  // exact gaussian KDE in two precisions (capi.cu kde_hybrid): the single-pass fp16 sweep sums every
  // 128-column tile half whose fp32 sum is at most hot_thr and marks the others in a bitmap; the
  // split3 sweep over the listed (block, tile) pairs sums exactly the marked halves
  MODE_KDE_COLD = 7,
  MODE_KDE_HOT = 8,
  // gaussian over operands with norm columns (prep.cu: exact / fp16 with A = [q | w | -b(q)], B =
  // [x | -b(x) | w]): the accumulator already holds -d2/2, so t = S * (m2s * negc) (KDE_COLD too)
  MODE_KDE_GAUSS_AUG = 9,
  MODE_KDE_COLD_AUG = 10   // KDE_COLD over operands with norm columns
};
constexpr int kHistBins = 64;  // MODE_HIST bins per query (quadratic spacing over [lo_q, top_q])
constexpr int kHistStride = kHistBins + 1;  // shared-memory row stride of the bins (rows on distinct banks)
__host__ __device__ constexpr bool is_kde(int mode) {
  return mode == MODE_KDE_GAUSS || mode == MODE_KDE_EXP || mode == MODE_KDE_GAUSS_MUFU || mode == MODE_KDE_COLD ||
         mode == MODE_KDE_HOT || mode == MODE_KDE_GAUSS_AUG || mode == MODE_KDE_COLD_AUG;
}
__host__ __device__ constexpr bool is_aug(int mode) { return mode == MODE_KDE_GAUSS_AUG || mode == MODE_KDE_COLD_AUG; }
__host__ __device__ constexpr bool is_cold(int mode) { return mode == MODE_KDE_COLD || mode == MODE_KDE_COLD_AUG; }
// the per-element epilogue of a mode: the two-precision sweeps are gaussian (the split3 one with every
// exponential on MUFU: it is MMA-bound)
__host__ __device__ constexpr int epi_mode(int mode) {
  return mode == MODE_KDE_COLD       ? int(MODE_KDE_GAUSS)
         : mode == MODE_KDE_COLD_AUG ? int(MODE_KDE_GAUSS_AUG)
         : mode == MODE_KDE_HOT      ? int(MODE_KDE_GAUSS_MUFU)
                                     : mode;
}
constexpr int kHotWords = 8;  // hot bitmap words per (query block, tile): 4 lane quarters x 2 column halves

constexpr int kBM = 128;           // query rows per tile (UMMA M)
constexpr int kBN = 256;           // dataset columns per tile (UMMA N)
constexpr int kBK = 64;            // K elements per block (128 B rows, SWIZZLE_128B)
constexpr int kABlockBytes = kBM * kBK * 2;   // 16 KB
constexpr int kBBlockBytes = kBN * kBK * 2;   // 32 KB
constexpr int kEpiWarp0 = 4;
constexpr int kNumEpiWarps = 16;
constexpr int kThreads = 32 * (kEpiWarp0 + kNumEpiWarps);  // 640
constexpr int kColGroups = 4;      // 64-column groups per tile (one per epilogue warp of a lane quarter)
constexpr int kXnSlots = 4;        // column-norm staging ring (1 KB per tile)
constexpr uint32_t kTmemCols = 512;  // 2 accumulator buffers x 256 fp32 columns
constexpr int kStageCap = 32;      // FILTER: per-row smem candidate staging (entries)
constexpr int kUnitSlots = 4;
// tile-major FILTER: per epilogue warp, each lane's 32 d2 values of a chunk with hits staged in shared
// memory (row stride 36 floats: conflict-free 16-byte stores), so a hit's key is one shared load
constexpr int kSdStride = 36;
constexpr size_t kTmSdBytes = size_t(kNumEpiWarps) * 32 * kSdStride * 4;      // tile-major: ring of claimed unit ids (producer -> MMA / epilogue)

struct TileParams {
  int32_t nq;              // valid query rows
  int32_t nq_pad;          // multiple of 128
  int32_t nqb;             // nq_pad / 128
  int64_t n;               // valid dataset columns (local shard)
  int32_t ntiles;          // tiles in the sweep
  int32_t tile_stride;     // dataset tile index = t * tile_stride
  int32_t tiles_per_unit;
  int32_t ncc;             // column chunks = ceil(ntiles / tiles_per_unit)
  int32_t kblocks;         // Kp / 64
  int32_t klast;           // 16-wide MMA k-steps of the last K-block that touch real columns (1..4)
  int32_t a_resident;      // 1: query block loaded once per unit
  int32_t stages;          // B ring depth
  int32_t seg_tiles;       // TILEMIN: tiles per segment (0: one segment per 64-column group)
  // tile-list mode (FILTER over pruned per-block lists, capi.cu knn_device): unit u covers query
  // block ulist[3u] and positions [ulist[3u+1], ulist[3u+2]) of tlist (tile ids of the sweep operand)
  const int32_t* ulist;
  const int32_t* tlist;
  int32_t nunits_list;
  // tile-major FILTER (tmajor = 1): unit u = dataset tile ulist[3u] (resident in shared memory)
  // x query blocks blist[ulist[3u+1] .. ulist[3u+2]) streamed through the ring; the unit count
  // is read from device memory (built on the device, capi.cu knn_device)
  int32_t knn_aug;         // k-NN sweeps over operands with norm columns: the accumulator is -d2/2
                           // (scaled), d2 = S * m2s (no |q|^2 / |x|^2 terms in the epilogue)
  int32_t tmajor;          // tile-major FILTER: resident dataset-tile buffers (1, or 2: the next unit's tile
                           // loads while the current unit's query blocks stream past); 0 = block-major
  const int32_t* blist;
  const int32_t* nunits_dev;
  int32_t* unit_counter;   // tile-major: units are claimed dynamically (atomicAdd), zeroed per launch
  int32_t list_stride;     // TILEMIN over per-block tile lists: segment = (list position) x 64-column group
  // MODE_HIST: per query row, bins b = floor(64 sqrt((d2 - hlo) * hinv)) for d2 <= htop, counted into
  // hist[row][64] (shared-memory counts flushed with global atomics per work unit)
  const float* hlo;
  const float* hinv;
  const float* htop;
  uint32_t* hist;
  // MODE_KDE_COLD writes / MODE_KDE_HOT reads: [nqb][ntiles][kHotWords] lane masks, word quarter * 2 +
  // half = rows quarter*32 + lane of the block, columns [128 half, 128 half + 128) of the tile
  uint32_t* hot_bits;
  float hot_thr;           // MODE_KDE_COLD: a tile half whose fp32 sum exceeds this is hot
  // norm-column tail (prep.cu, d within 6 of a multiple of 64): the query block's 16-column tail
  // rides with the resident A, each tile's 256 x 16 tail takes the column-norm slot (8 KB), and
  // one more 16-wide MMA step closes the accumulation (KDE_GAUSS_AUG / KDE_COLD_AUG only)
  int32_t tail;
  const float* xn;         // [n_pad] |x|^2 (encoding-consistent)
  const float* qn;         // [nq_pad] |q|^2
  const float* m2s;        // device scalar: -2 / (scale_q * scale_x)
  float negc;              // exp2 scale: gaussian -log2e/(2h^2); exponential -log2e/h
  double* part;            // KDE: [ncc*kColGroups][nq_pad] partial sums
  float* tmin;             // TILEMIN: [nseg][nq_pad], pre-filled with +inf (atomicMin on int bits)
  const float* tau;        // FILTER: [nq_pad] thresholds
  uint32_t* cand_cnt;      // FILTER: [nq_pad]
  unsigned long long* cand;  // FILTER: [nq_pad][cap] keys (f32 bits << 32 | col)
  int32_t cap;
  const uint32_t* guard;     // optional: the sweep is skipped when (*guard & 6) != 0 (queries not exact-mode)
};

constexpr int kTailABytes = kBM * 16 * 2;  // 4 KB: the query block's norm-column tail
constexpr int kTailBBytes = kBN * 16 * 2;  // 8 KB: a dataset tile's norm-column tail (a column-norm slot)

__host__ __device__ inline size_t tile_smem_bytes(int kblocks, int a_resident, int stages, int mode, bool pair,
                                                  int tmajor = 0, bool tail = false) {
  size_t a = a_resident ? size_t(kblocks) * kABlockBytes : size_t(stages) * kABlockBytes;
  size_t b = size_t(stages) * (pair ? kBBlockBytes / 2 : kBBlockBytes);
  if (tmajor) {  // resident dataset tile(s) + ring of query K-blocks; candidates go straight to global lists
    a = size_t(stages) * kABlockBytes;
    b = size_t(tmajor) * size_t(kblocks) * kBBlockBytes;
  }
  size_t stage = ((mode == MODE_FILTER && !tmajor) || mode == MODE_HIST) ? size_t(kBM) * kStageCap * 8 + kBM * 4
                 : (mode == MODE_FILTER && tmajor)                      ? kTmSdBytes
                                                                        : 0;
  const size_t xslots = size_t(kXnSlots) * (tail ? kTailBBytes : kBN * 4) + (tail ? kTailABytes : 0);
  return 1024 /*align slack*/ + a + b + xslots + stage + 512 /*barriers*/;
}


// Gaussian epilogue: which of the 16 pairs of a 32-column chunk take the FMA-pipe
// polynomial instead of MUFU.EX2 (bit i = pair i), trading XU-pipe cycles (8 per
// warp MUFU) for FMA-pipe cycles (2 per packed FADD2/FFMA2).  Measured on c2 (B200,
// power-capped at ~990 W): 0 pairs 2.98 ms, 1: 2.92, 2: 2.83, 3: 2.86, 4: 2.87, 6: 2.99,
// 8: 3.19 ms — the sweet spot is small because the kernel also runs at the power cap.
#ifndef DK_POLY_PAIRS
#define DK_POLY_PAIRS 0x0808u
#endif
constexpr uint32_t kPolyPairs = DK_POLY_PAIRS;
// the norm-column epilogue spends 2 packed FMA-pipe ops per 2 pairs (t = S c, the sum) instead of 4,
// so more of the exponentials can move to the FMA pipe
#ifndef DK_POLY_PAIRS_AUG
#define DK_POLY_PAIRS_AUG 0x2222u
#endif
constexpr uint32_t kPolyPairsAug = DK_POLY_PAIRS_AUG;

// Ping-pong epilogue for the KDE sweeps (single-CTA): the two accumulator buffers are
// consumed by two different groups of 8 epilogue warps (group = accumulator), each warp
// taking 128 columns of every other tile, so on every SM sub-partition one group's
// TMEM loads and barrier waits overlap the other group's exponentials instead of all
// four warps stalling together at every tile boundary.  c2: 2.704 -> 2.633 ms (A/B,
// interleaved runs); split3 / exponential sweeps are MMA-bound and unchanged.  Issuing
// the second 32-column TMEM load only after the first chunk's wait (to overlap it with
// that chunk's math) measured slower (2.76 ms), as did 1 or 3 polynomial pairs (2.64).
#ifndef DK_PINGPONG
#define DK_PINGPONG 1
#endif
__host__ __device__ constexpr bool is_knn_sweep(int mode) {
  return mode == MODE_TILEMIN || mode == MODE_FILTER || mode == MODE_HIST;
}

template <int MODE, bool kPair>
__host__ __device__ constexpr bool use_pingpong() {
  return DK_PINGPONG != 0 && !kPair &&
         (MODE == MODE_KDE_GAUSS || MODE == MODE_KDE_GAUSS_MUFU || MODE == MODE_KDE_EXP || is_cold(MODE) ||
          MODE == MODE_KDE_GAUSS_AUG);
}

// 2^t for a pair, t <= 0, on the FMA pipe: t = j + f (j = round(t), |f| <= 1/2),
// 2^f by a degree-5 polynomial (relative error < 2.4e-7 on |f| <= 1/2, i.e. at the
// level of ex2.approx), exponent j added to the float bits.  t is clamped at -126, so a
// term below fp32's normal range contributes 2^-126 instead of ex2.approx.ftz's 0: at
// most 2/16 x 2^-126 = 1.5e-39 on a mean, far below the parity floor (1e-16).  Selecting
// 0 there costs 4 instructions per 32 columns, 3.5% of the c2 sweep (issue-bound).
__device__ __forceinline__ float2 exp2_poly2(float2 t) {
  t.x = fmaxf(t.x, -126.f);
  t.y = fmaxf(t.y, -126.f);
  const float2 tr = add2(t, make_float2(12582912.f, 12582912.f));  // 1.5 * 2^23: round to integer
  const float2 jf = add2(tr, make_float2(-12582912.f, -12582912.f));
  const float2 f = add2(t, make_float2(-jf.x, -jf.y));
  // near-minimax (relative error) fit of 2^f on [-1/2, 1/2]: max rel err 2.3e-7 in fp32 Horner
  float2 p = make_float2(1.3276207e-3f, 1.3276207e-3f);
  p = fma2(p, f, make_float2(9.6754571e-3f, 9.6754571e-3f));
  p = fma2(p, f, make_float2(5.5507135e-2f, 5.5507135e-2f));
  p = fma2(p, f, make_float2(2.4022122e-1f, 2.4022122e-1f));
  p = fma2(p, f, make_float2(6.9314694e-1f, 6.9314694e-1f));
  p = fma2(p, f, make_float2(1.0000001f, 1.0000001f));
  float2 r;
  r.x = __int_as_float(__float_as_int(p.x) + (__float_as_int(tr.x) << 23));
  r.y = __int_as_float(__float_as_int(p.y) + (__float_as_int(tr.y) << 23));
  return r;
}

// k-NN sweeps: the approximate d2 of a 32-column chunk.  Plain operands: S * m2s + (|q|^2 + |x|^2)
// (packed FFMA2, the norms of the columns from shared memory).  Operands with norm columns (aug):
// the accumulator already is -d2/2 in the operands' scale, d2 = S * m2s (an exact power-of-two
// product); both are within the encoding's eps_q of the exact d2 (capi.cu make_encoding).
__device__ __forceinline__ void knn_d2(const uint32_t (&r)[32], const float4* __restrict__ x4, float qn, float m2s,
                                       bool aug, float (&d2v)[32]) {
  const float2 m2 = make_float2(m2s, m2s);
  if (aug) {
#pragma unroll
    for (int j2 = 0; j2 < 16; ++j2) {
      const float2 v = mul2(make_float2(__uint_as_float(r[2 * j2]), __uint_as_float(r[2 * j2 + 1])), m2);
      d2v[2 * j2] = v.x; d2v[2 * j2 + 1] = v.y;
    }
    return;
  }
  const float2 q2 = make_float2(qn, qn);
#pragma unroll
  for (int j4 = 0; j4 < 8; ++j4) {
    const float4 xv = x4[j4];
    const float2 da = fma2(make_float2(__uint_as_float(r[4 * j4]), __uint_as_float(r[4 * j4 + 1])), m2,
                           add2(q2, make_float2(xv.x, xv.y)));
    const float2 db = fma2(make_float2(__uint_as_float(r[4 * j4 + 2]), __uint_as_float(r[4 * j4 + 3])), m2,
                           add2(q2, make_float2(xv.z, xv.w)));
    d2v[4 * j4] = da.x; d2v[4 * j4 + 1] = da.y; d2v[4 * j4 + 2] = db.x; d2v[4 * j4 + 3] = db.y;
  }
}

// One 32-column chunk of the epilogue.  `full` = all 32 columns valid (warp-uniform).
template <int MODE, bool kAug = false>
__device__ __forceinline__ void epi_chunk(const uint32_t (&r)[32], const float* __restrict__ xs_smem, float qn,
                                          float m2s, float negc, float tau, bool full, int64_t cbase, int64_t n,
                                          float2& acc0, float2& acc1, float& mn, const TileParams& p, int row,
                                          uint32_t* scnt, unsigned long long* sbuf, int lrow) {
  const float4* x4 = reinterpret_cast<const float4*>(xs_smem);
  if (full || MODE == MODE_TILEMIN || MODE == MODE_FILTER || MODE == MODE_HIST) {
    if constexpr (MODE == MODE_KDE_GAUSS_AUG) {
      // the accumulator is q.x - (|q|^2 + |x|^2)/2 = -d2/2 (scaled): t = S * negc (negc = m2s x the
      // exp2 scale, an exact power-of-two product), no column norms
      (void)x4;
      const float2 c2 = make_float2(negc, negc);
#pragma unroll
      for (int j4 = 0; j4 < 8; ++j4) {
        const float2 ta = mul2(make_float2(__uint_as_float(r[4 * j4]), __uint_as_float(r[4 * j4 + 1])), c2);
        const float2 tb = mul2(make_float2(__uint_as_float(r[4 * j4 + 2]), __uint_as_float(r[4 * j4 + 3])), c2);
        const float2 ea = (kPolyPairsAug >> (2 * j4)) & 1 ? exp2_poly2(ta) : make_float2(ex2_approx(ta.x), ex2_approx(ta.y));
        const float2 eb = (kPolyPairsAug >> (2 * j4 + 1)) & 1 ? exp2_poly2(tb) : make_float2(ex2_approx(tb.x), ex2_approx(tb.y));
        acc0 = add2(acc0, ea);
        acc1 = add2(acc1, eb);
      }
    } else if constexpr (MODE == MODE_KDE_GAUSS || MODE == MODE_KDE_GAUSS_MUFU) {
      constexpr uint32_t poly = MODE == MODE_KDE_GAUSS ? kPolyPairs : 0u;
      // d2 = S * m2s + (qn + xn) in the cancellation-safe order, then t = d2 * negc
      const float2 q2 = make_float2(qn, qn), m2 = make_float2(m2s, m2s), c2 = make_float2(negc, negc);
#pragma unroll
      for (int j4 = 0; j4 < 8; ++j4) {
        const float4 xv = x4[j4];
        const float2 ua = add2(q2, make_float2(xv.x, xv.y));
        const float2 ub = add2(q2, make_float2(xv.z, xv.w));
        const float2 da = fma2(make_float2(__uint_as_float(r[4 * j4]), __uint_as_float(r[4 * j4 + 1])), m2, ua);
        const float2 db = fma2(make_float2(__uint_as_float(r[4 * j4 + 2]), __uint_as_float(r[4 * j4 + 3])), m2, ub);
        const float2 ta = mul2(da, c2), tb = mul2(db, c2);
        const float2 ea = (poly >> (2 * j4)) & 1 ? exp2_poly2(ta) : make_float2(ex2_approx(ta.x), ex2_approx(ta.y));
        const float2 eb = (poly >> (2 * j4 + 1)) & 1 ? exp2_poly2(tb) : make_float2(ex2_approx(tb.x), ex2_approx(tb.y));
        acc0 = add2(acc0, ea);
        acc1 = add2(acc1, eb);
      }
    } else if constexpr (MODE == MODE_KDE_EXP) {
#pragma unroll
      for (int j4 = 0; j4 < 8; ++j4) {
        const float4 xv = x4[j4];
        const float xs[4] = {xv.x, xv.y, xv.z, xv.w};
#pragma unroll
        for (int jj = 0; jj < 4; ++jj) {
          const int j = j4 * 4 + jj;
          const float d2 = fmaf(__uint_as_float(r[j]), m2s, qn + xs[jj]);
          mn = fminf(mn, d2);  // near-pair guard: the row's smallest approximate d2 (see the unit end)
          const float e = ex2_approx(sqrt_approx(fmaxf(d2, 0.f)) * negc);
          if (jj & 1) acc0.y += e; else acc0.x += e;
        }
      }
    } else {
      // k-NN passes: packed distance arithmetic, branch-free hit mask
      float d2v[32];
      knn_d2(r, x4, qn, m2s, kAug, d2v);
      if (!full) {  // columns past n: +inf never wins a min; NaN never passes a threshold (not even +inf)
        const int lim = int(min(int64_t(32), n - cbase));
        const float pad = MODE != MODE_TILEMIN ? __int_as_float(0x7fc00000) : __int_as_float(0x7f800000);
#pragma unroll
        for (int j = 0; j < 32; ++j) d2v[j] = j < lim ? d2v[j] : pad;
      }
      if constexpr (MODE == MODE_HIST) {
        // tau holds htop; acc0 = (hlo, hinv) of this row (set by the caller); NaN pads never count
        // bin b = floor(64 sqrt((d2 - lo) / (top - lo))): the approximate square root's ~2^-22 relative
        // error sits far inside the 1e-5 slack of the bin edges (knn.cu tau_hist_kernel)
        uint32_t* hrow = reinterpret_cast<uint32_t*>(sbuf) + lrow * kHistStride;
        const float2 nlo = make_float2(-acc0.x, -acc0.x), hinv = make_float2(acc0.y, acc0.y);
#pragma unroll
        for (int j2 = 0; j2 < 16; ++j2) {
          const float2 u = mul2(add2(make_float2(d2v[2 * j2], d2v[2 * j2 + 1]), nlo), hinv);
          if (d2v[2 * j2] <= tau)
            atomicAdd(hrow + min(kHistBins - 1, __float2int_rz(sqrt_approx(fmaxf(u.x, 0.f)) * float(kHistBins))), 1u);
          if (d2v[2 * j2 + 1] <= tau)
            atomicAdd(hrow + min(kHistBins - 1, __float2int_rz(sqrt_approx(fmaxf(u.y, 0.f)) * float(kHistBins))), 1u);
        }
      } else if constexpr (MODE == MODE_TILEMIN) {
        // minima of the two 16-column halves (listed sweeps keep them as separate segments)
        float m0 = d2v[0], m1 = d2v[1], m2_ = d2v[16], m3 = d2v[17];
#pragma unroll
        for (int j = 2; j < 16; j += 2) {
          m0 = fminf(m0, d2v[j]); m1 = fminf(m1, d2v[j + 1]);
          m2_ = fminf(m2_, d2v[16 + j]); m3 = fminf(m3, d2v[17 + j]);
        }
        acc0 = make_float2(fminf(m0, m1), fminf(m2_, m3));
        mn = fminf(mn, fminf(acc0.x, acc0.y));
      } else {
        // candidates are rare (~1e-4 of the pairs): a min tree (4 independent chains)
        // rejects the whole chunk before any per-column mask is built
        float m0 = d2v[0], m1 = d2v[1], m2_ = d2v[2], m3 = d2v[3];
#pragma unroll
        for (int j = 4; j < 32; j += 4) {
          m0 = fminf(m0, d2v[j]); m1 = fminf(m1, d2v[j + 1]);
          m2_ = fminf(m2_, d2v[j + 2]); m3 = fminf(m3, d2v[j + 3]);
        }
        uint32_t hits = 0;
        if (fminf(fminf(m0, m1), fminf(m2_, m3)) <= tau) {
#pragma unroll
          for (int j = 0; j < 32; ++j) hits |= (d2v[j] <= tau ? 1u : 0u) << j;
        }
        if (hits && scnt == nullptr) {  // tile-major sweep: straight to the global list
          const uint32_t g = atomicAdd(&p.cand_cnt[row], uint32_t(__popc(hits)));
          uint32_t slot = g;
          while (hits) {
            const int j = __ffs(hits) - 1;
            hits &= hits - 1;
            float dj = d2v[0];
#pragma unroll
            for (int i = 1; i < 32; ++i) dj = (i == j) ? d2v[i] : dj;
            const unsigned long long key = (static_cast<unsigned long long>(__float_as_uint(fmaxf(dj, 0.f))) << 32) |
                                           static_cast<unsigned long long>(cbase + j);
            if (slot < uint32_t(p.cap)) p.cand[size_t(row) * p.cap + slot] = key;
            ++slot;
          }
        } else if (hits) {  // appended candidates: one shared (and at most one global) atomic per chunk
          const uint32_t nh = uint32_t(__popc(hits));
          const uint32_t pos = atomicAdd(&scnt[lrow], nh);
          const uint32_t first_spill = max(pos, uint32_t(kStageCap));
          const uint32_t nspill = pos + nh > first_spill ? pos + nh - first_spill : 0u;
          const uint32_t g = nspill ? atomicAdd(&p.cand_cnt[row], nspill) : 0u;
          uint32_t slot = pos;
          while (hits) {
            const int j = __ffs(hits) - 1;
            hits &= hits - 1;
            float dj = d2v[0];
#pragma unroll
            for (int i = 1; i < 32; ++i) dj = (i == j) ? d2v[i] : dj;
            const unsigned long long key = (static_cast<unsigned long long>(__float_as_uint(fmaxf(dj, 0.f))) << 32) |
                                           static_cast<unsigned long long>(cbase + j);
            if (slot < uint32_t(kStageCap)) {
              sbuf[lrow * kStageCap + slot] = key;
            } else {  // dense region: straight to the global list
              const uint32_t gi = g + (slot - first_spill);
              if (gi < uint32_t(p.cap)) p.cand[size_t(row) * p.cap + gi] = key;
            }
            ++slot;
          }
        }
      }
    }
  } else {
    const int lim = int(min(int64_t(32), n - cbase));
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      if (j >= lim) continue;
      if constexpr (MODE == MODE_KDE_GAUSS_AUG) {
        acc0.x += ex2_approx(__uint_as_float(r[j]) * negc);
        continue;
      }
      const float d2 = fmaf(__uint_as_float(r[j]), m2s, qn + xs_smem[j]);
      if constexpr (MODE == MODE_KDE_GAUSS || MODE == MODE_KDE_GAUSS_MUFU) {
        acc0.x += ex2_approx(d2 * negc);
      } else {
        if constexpr (MODE == MODE_KDE_EXP) mn = fminf(mn, d2);
        acc0.x += ex2_approx(sqrt_approx(fmaxf(d2, 0.f)) * negc);
      }
    }
  }
}

// Exponential kernel, near-pair guard: exp(-sqrt(d2)/h) amplifies the operand-rounding error of a small
// d2 (|sqrt(a) - sqrt(b)| ~ |a - b| / (2 sqrt(b)), unbounded at a coincident pair).  A row whose smallest
// approximate d2 falls under its threshold tau (capi.cu exp_guard: the d2 below which the error of
// sqrt(d2)/h can exceed the tolerance) is flagged and re-evaluated in fp64 (redo.cu).
template <int MODE>
__device__ __forceinline__ void exp_guard_flag(const TileParams& p, int row, float mn) {
  if constexpr (MODE == MODE_KDE_EXP) {
    if (p.tau != nullptr && mn < p.tau[row]) p.cand_cnt[row] = 1u;
  }
}

// Tile-major FILTER, one 32-column chunk: d2 exactly as epi_chunk's k-NN branch computes it (knn_d2, packed
// FFMA2 of S * m2s + (|q|^2 + |x|^2)), a min tree to reject the chunk, and for the chunks of a warp
// with hits the d2 row staged in shared memory (`sd`, this lane's row), from which each hit's key
// is one load — no per-hit select chain over the registers.  Candidates go straight to the row's
// global list (one atomic per row and chunk with hits).
template <bool kAug>
__device__ __forceinline__ void filter_chunk_tm(const uint32_t (&r)[32], const float* __restrict__ xs_smem, float qn,
                                                float m2s, float tau, bool full, int64_t cbase, const TileParams& p,
                                                int row, float* sd) {
  float d2v[32];
  knn_d2(r, reinterpret_cast<const float4*>(xs_smem), qn, m2s, kAug, d2v);
  float m0 = d2v[0], m1 = d2v[1], m2_ = d2v[2], m3 = d2v[3];
#pragma unroll
  for (int j = 4; j < 32; j += 4) {
    m0 = fminf(m0, d2v[j]); m1 = fminf(m1, d2v[j + 1]);
    m2_ = fminf(m2_, d2v[j + 2]); m3 = fminf(m3, d2v[j + 3]);
  }
  uint32_t hits = 0;
  if (fminf(fminf(m0, m1), fminf(m2_, m3)) <= tau) {
#pragma unroll
    for (int j = 0; j < 32; ++j) hits |= (d2v[j] <= tau ? 1u : 0u) << j;
  }
  if (!full) {  // columns past n never hit
    const int64_t lim = p.n - cbase;
    hits &= lim >= 32 ? 0xffffffffu : (lim <= 0 ? 0u : (1u << lim) - 1u);
  }
  if (__any_sync(0xffffffffu, hits != 0u)) {
#pragma unroll
    for (int j4 = 0; j4 < 8; ++j4)
      reinterpret_cast<float4*>(sd)[j4] = make_float4(d2v[4 * j4], d2v[4 * j4 + 1], d2v[4 * j4 + 2], d2v[4 * j4 + 3]);
    if (hits) {
      uint32_t slot = atomicAdd(&p.cand_cnt[row], uint32_t(__popc(hits)));
      unsigned long long* dst = p.cand + size_t(row) * p.cap;
      while (hits) {
        const int j = __ffs(hits) - 1;
        hits &= hits - 1;
        const unsigned long long key = (static_cast<unsigned long long>(__float_as_uint(fmaxf(sd[j], 0.f))) << 32) |
                                       static_cast<unsigned long long>(cbase + j);
        if (slot < uint32_t(p.cap)) dst[slot] = key;
        ++slot;
      }
    }
    __syncwarp();
  }
}

__device__ __forceinline__ void epi_bar() { asm volatile("bar.sync 1, %0;" ::"n"(kNumEpiWarps * 32) : "memory"); }

// kPair: a 2-CTA cluster runs tcgen05.mma.cta_group::2 with M = 256 — the two CTAs
// own two query blocks (128 rows each, A resident in each CTA) and each TMA-loads one
// half (128 rows) of every 256-row dataset K-block.  Each SM then streams half the B
// bytes and reads half the B operand per MMA from its shared memory, which is what
// keeps a single-CTA M=128 sweep below the tensor peak (smem bandwidth).  The leader
// (rank 0) issues every MMA; stage / accumulator / A releases are multicast commits to
// both CTAs; both CTAs' epilogue warps arrive on the leader's accumulator-empty barrier.
template <int MODE, bool kPair>
__global__ void __launch_bounds__(kThreads, 1)
    tile_kernel(const __grid_constant__ CUtensorMap tmapA, const __grid_constant__ CUtensorMap tmapB,
                const __grid_constant__ CUtensorMap tmapAt, const __grid_constant__ CUtensorMap tmapBt,
                const TileParams p) {
  // speculative exact-mode launch (capi.cu dk_naive): the host has not waited for the query
  // check, so a batch that turned out fractional skips this sweep and is redone in split3
  if (p.guard != nullptr && (*p.guard & 6u) != 0u) return;
  constexpr bool kPP = use_pingpong<MODE, kPair>();
  extern __shared__ uint8_t smem_raw[];
  // 1024-byte alignment (SWIZZLE_128B atoms) by offsetting the shared pointer itself, so the
  // compiler keeps the shared address space (LDS/ATOMS instead of generic LD/ATOM)
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  const int stages = p.stages;
  constexpr int kBStage = kPair ? kBBlockBytes / 2 : kBBlockBytes;  // B bytes per CTA per stage
  const bool tmajor = MODE == MODE_FILTER && !kPair && p.tmajor != 0;
  const int tbufs = tmajor ? p.tmajor : 1;  // tile-major: resident tile buffers
  uint8_t* smemA = smem;
  const bool tail = is_aug(MODE) && p.tail != 0;
  // [A: resident K-blocks or ring][A tail (tail mode)][B ring][column-norm / B-tail slots]
  uint8_t* smemAt = smem + (p.a_resident ? size_t(p.kblocks) * kABlockBytes : size_t(stages) * kABlockBytes);
  uint8_t* smemB = smemAt + (tail ? kTailABytes : 0);
  float* smemX = reinterpret_cast<float*>(smemB + size_t(stages) * kBStage);  // [kXnSlots][xslot]
  const int xslot = tail ? kTailBBytes / 4 : kBN;  // floats per slot
  if (tmajor) {  // [resident tiles: tbufs x kblocks x 32 KB][ring: stages x 16 KB query K-blocks][norms]
    smemB = smem;
    smemA = smem + size_t(tbufs) * p.kblocks * kBBlockBytes;
    smemX = reinterpret_cast<float*>(smemA + size_t(stages) * kABlockBytes);
  }
  unsigned long long* sbuf = reinterpret_cast<unsigned long long*>(smemX + kXnSlots * xslot);  // FILTER staging
  const bool kStage = (MODE == MODE_FILTER && !tmajor) || MODE == MODE_HIST;  // FILTER staging / HIST bins
  uint32_t* scnt = reinterpret_cast<uint32_t*>(sbuf + (kStage ? kBM * kStageCap : tmajor ? kTmSdBytes / 8 : 0));
  uint64_t* bars = reinterpret_cast<uint64_t*>(scnt + (kStage ? kBM : 0));
  uint64_t* full_bar = bars;                 // [stages]   (leader's counts both CTAs' bytes)
  uint64_t* empty_bar = bars + stages;       // [stages]
  uint64_t* tfull_bar = bars + 2 * stages;   // [2]
  uint64_t* tempty_bar = tfull_bar + 2;      // [2]        (leader's counts both CTAs' warps)
  uint64_t* afull_bar = tempty_bar + 2;      // [2]        (the second: tile-major's other tile buffer)
  uint64_t* aempty_bar = afull_bar + 2;      // [2]
  uint64_t* xfull_bar = aempty_bar + 2;      // [kXnSlots]
  uint64_t* xempty_bar = xfull_bar + kXnSlots;  // [kXnSlots]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(xempty_bar + kXnSlots);
  uint64_t* ufull_bar = reinterpret_cast<uint64_t*>(tmem_slot + 2);  // [kUnitSlots] (tile-major)
  uint64_t* uempty_bar = ufull_bar + kUnitSlots;                     // [kUnitSlots]
  int32_t* s_unit = reinterpret_cast<int32_t*>(uempty_bar + kUnitSlots);  // [kUnitSlots]

  const uint32_t warp = warp_id_sync();
  const uint32_t lane = lane_id();
  const uint32_t crank = kPair ? cluster_ctarank() : 0u;
  const bool leader = crank == 0;
  // work units: (query-block group, column chunk); a pair owns 2 query blocks
  const int ngroups = kPair ? p.nqb / 2 : p.nqb;
  const int nunits = p.ulist != nullptr ? (p.nunits_dev != nullptr ? *p.nunits_dev : p.nunits_list) : ngroups * p.ncc;
  const int first_unit = kPair ? int(blockIdx.x) / 2 : int(blockIdx.x);
  const int unit_step = kPair ? int(gridDim.x) / 2 : int(gridDim.x);

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmapA);
    tma_prefetch_desc(&tmapB);
    for (int s = 0; s < stages; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull_bar[a], 1);
      mbar_init(&tempty_bar[a], kPair ? 2 * kNumEpiWarps : (kPP ? kNumEpiWarps / 2 : kNumEpiWarps));
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&afull_bar[a], 1);
      mbar_init(&aempty_bar[a], 1);
    }
    for (int x = 0; x < kXnSlots; ++x) {
      mbar_init(&xfull_bar[x], 1);
      mbar_init(&xempty_bar[x], kPP ? kNumEpiWarps / 2 : kNumEpiWarps);
    }
    if (tmajor) {
      for (int x = 0; x < kUnitSlots; ++x) {
        mbar_init(&ufull_bar[x], 1);
        mbar_init(&uempty_bar[x], 1 + kNumEpiWarps);  // the MMA thread and every epilogue warp
      }
    }
    fence_mbar_init();
  }
  if constexpr (MODE == MODE_FILTER) {
    if (!tmajor)
      for (int i = threadIdx.x; i < kBM; i += blockDim.x) scnt[i] = 0;
  }
  if constexpr (MODE == MODE_HIST) {
    static_assert(kBM * kHistStride * 4 <= kBM * kStageCap * 8 + kBM * 4, "histogram bins must fit the staging area");
    uint32_t* hb = reinterpret_cast<uint32_t*>(sbuf);
    for (int i = threadIdx.x; i < kBM * kHistStride; i += blockDim.x) hb[i] = 0u;
  }
  if (warp == 2) {
    if constexpr (kPair) tmem_alloc_pair<kTmemCols>(tmem_slot);
    else tmem_alloc<kTmemCols>(tmem_slot);
  }
  tc_fence_before();
  if constexpr (kPair) cluster_sync_all();  // both CTAs' barriers live before any remote arrive / TMA
  else __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
#ifdef DK_TIMING
  long long dbgw[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#endif

  if (warp == 0) {
    // ===================== TMA producer (each CTA) =====================
    if (lane == 0 && tmajor) {
      // tile-major FILTER: the unit's dataset tile once into the resident buffer, then the
      // query blocks that list it through the ring (they stay in L2: a batch's whole query
      // operand is a few MB; the tile is read from DRAM about once per batch)
      const uint64_t pol_b = policy_evict_first();
      const uint64_t pol_a = policy_evict_last();
      int stage = 0;
      uint32_t phase = 0;
      int uiter = 0;
      uint32_t titer = 0;
      // units are claimed dynamically (they differ in length: 1..many query blocks per tile) and
      // published to the MMA / epilogue warps through a small ring; -1 ends the sweep
      int uslot = 0;
      uint32_t uph = 0;
      for (;; ++uiter) {
        int u = atomicAdd(p.unit_counter, 1);
        if (u >= nunits) u = -1;
        mbar_wait(&uempty_bar[uslot], uph ^ 1);
        s_unit[uslot] = u;
        mbar_arrive(&ufull_bar[uslot]);
        if (++uslot == kUnitSlots) { uslot = 0; uph ^= 1; }
        if (u < 0) break;
        const int col0 = __ldg(p.ulist + 3 * u) * kBN;
        const int i0 = __ldg(p.ulist + 3 * u + 1), i1 = __ldg(p.ulist + 3 * u + 2);
        DK_DCHECK(col0 >= 0 && col0 < p.n && i0 <= i1);
        // the unit's tile buffer (alternating with tbufs == 2: it fills while the previous unit computes)
        const int tb = tbufs == 2 ? (uiter & 1) : 0;
        const uint32_t tuse = tbufs == 2 ? uint32_t(uiter >> 1) : uint32_t(uiter);
        mbar_wait(&aempty_bar[tb], (tuse & 1) ^ 1);
        mbar_arrive_expect_tx(&afull_bar[tb], uint32_t(p.kblocks) * kBBlockBytes);
        uint8_t* tbuf = smemB + size_t(tb) * p.kblocks * kBBlockBytes;
        for (int kb = 0; kb < p.kblocks; ++kb)
          tma_load_2d(tbuf + size_t(kb) * kBBlockBytes, &tmapB, &afull_bar[tb], kb * kBK, col0, pol_b);
        for (int i = i0; i < i1; ++i, ++titer) {
          const int qb = __ldg(p.blist + i);
          DK_DCHECK(qb >= 0 && qb < p.nqb);
          const uint32_t xs = titer % kXnSlots;
          mbar_wait(&xempty_bar[xs], ((titer / kXnSlots) & 1) ^ 1);
          mbar_arrive_expect_tx(&xfull_bar[xs], kBN * 4);
          bulk_load(smemX + xs * kBN, p.xn + col0, kBN * 4, &xfull_bar[xs]);
          for (int kb = 0; kb < p.kblocks; ++kb) {
            mbar_wait(&empty_bar[stage], phase ^ 1);
            mbar_arrive_expect_tx(&full_bar[stage], kABlockBytes);
            tma_load_2d(smemA + size_t(stage) * kABlockBytes, &tmapA, &full_bar[stage], kb * kBK, qb * kBM, pol_a);
            if (++stage == stages) { stage = 0; phase ^= 1; }
          }
        }
      }
    } else if (lane == 0) {
      const uint64_t pol_b = policy_evict_last();   // dataset tiles are re-read by other query blocks
      const uint64_t pol_a = policy_evict_last();
      int stage = 0;
      uint32_t phase = 0;
      int uiter = 0;
      uint32_t titer = 0;
      for (int u = first_unit; u < nunits; u += unit_step, ++uiter) {
        int qb = (u % ngroups) * (kPair ? 2 : 1) + int(crank), cc = u / ngroups;
        int t0 = cc * p.tiles_per_unit;
        int t1 = min(p.ntiles, t0 + p.tiles_per_unit);
        if (p.ulist != nullptr) { qb = p.ulist[3 * u]; t0 = p.ulist[3 * u + 1]; t1 = p.ulist[3 * u + 2]; }
        if (p.a_resident) {
          mbar_wait(aempty_bar, (uiter & 1) ^ 1);
          if constexpr (kPair) {
            if (leader) mbar_arrive_expect_tx(afull_bar, 2u * uint32_t(p.kblocks) * kABlockBytes);
            for (int kb = 0; kb < p.kblocks; ++kb)
              tma_load_2d_pair(smemA + size_t(kb) * kABlockBytes, &tmapA, afull_bar, kb * kBK, qb * kBM, pol_a);
          } else {
            mbar_arrive_expect_tx(afull_bar, uint32_t(p.kblocks) * kABlockBytes + (tail ? kTailABytes : 0u));
            for (int kb = 0; kb < p.kblocks; ++kb)
              tma_load_2d(smemA + size_t(kb) * kABlockBytes, &tmapA, afull_bar, kb * kBK, qb * kBM, pol_a);
            if (tail) tma_load_2d(smemAt, &tmapAt, afull_bar, 0, qb * kBM, pol_a);
          }
        }
        // tile-list mode: the next tile id is loaded one tile ahead (off the issue path)
        int tnext = (p.tlist != nullptr && t0 < t1) ? __ldg(p.tlist + t0) : 0;
        for (int t = t0; t < t1; ++t, ++titer) {
          int col0;
          if (p.tlist != nullptr) {
            col0 = tnext * kBN;
            DK_DCHECK(tnext >= 0 && col0 < p.n && qb >= 0 && qb < p.nqb);
            if (t + 1 < t1) tnext = __ldg(p.tlist + t + 1);
          } else {
            col0 = t * p.tile_stride * kBN;
          }
          {  // column norms of this tile (tail mode: its norm-column tail) -> own smem ring slot
            const uint32_t xs = titer % kXnSlots;
            mbar_wait(&xempty_bar[xs], ((titer / kXnSlots) & 1) ^ 1);
            if (tail) {
              mbar_arrive_expect_tx(&xfull_bar[xs], kTailBBytes);
              tma_load_2d(smemX + xs * xslot, &tmapBt, &xfull_bar[xs], 0, col0, pol_b);
            } else {
              mbar_arrive_expect_tx(&xfull_bar[xs], kBN * 4);
              bulk_load(smemX + xs * xslot, p.xn + col0, kBN * 4, &xfull_bar[xs]);
            }
          }
          for (int kb = 0; kb < p.kblocks; ++kb) {
            DK_TWAIT(5, mbar_wait(&empty_bar[stage], phase ^ 1));
            if constexpr (kPair) {
              const uint32_t bytes = 2u * (kBStage + (p.a_resident ? 0u : uint32_t(kABlockBytes)));
              if (leader) mbar_arrive_expect_tx(&full_bar[stage], bytes);
              if (!p.a_resident)
                tma_load_2d_pair(smemA + size_t(stage) * kABlockBytes, &tmapA, &full_bar[stage], kb * kBK,
                                 qb * kBM, pol_a);
              tma_load_2d_pair(smemB + size_t(stage) * kBStage, &tmapB, &full_bar[stage], kb * kBK,
                               col0 + int(crank) * (kBN / 2), pol_b);
            } else {
              if (p.a_resident) {
                mbar_arrive_expect_tx(&full_bar[stage], kBBlockBytes);
              } else {
                mbar_arrive_expect_tx(&full_bar[stage], kBBlockBytes + kABlockBytes);
                tma_load_2d(smemA + size_t(stage) * kABlockBytes, &tmapA, &full_bar[stage], kb * kBK, qb * kBM,
                            pol_a);
              }
              tma_load_2d(smemB + size_t(stage) * kBBlockBytes, &tmapB, &full_bar[stage], kb * kBK, col0, pol_b);
            }
            if (++stage == stages) { stage = 0; phase ^= 1; }
          }
        }
      }
    }
  } else if (warp == 1) {
    // ===================== MMA issuer (leader CTA only) =====================
    if (lane == 0 && tmajor) {
      constexpr uint32_t idesc = idesc_f16_f32(kBM, kBN);
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      int uiter = 0;
      const uint32_t a0 = smem_u32(smemA), b0 = smem_u32(smemB);
      int uslot = 0;
      uint32_t uph = 0;
      for (;; ++uiter) {
        mbar_wait(&ufull_bar[uslot], uph);
        const int u = s_unit[uslot];
        mbar_arrive(&uempty_bar[uslot]);
        if (++uslot == kUnitSlots) { uslot = 0; uph ^= 1; }
        if (u < 0) break;
        const int i0 = __ldg(p.ulist + 3 * u + 1), i1 = __ldg(p.ulist + 3 * u + 2);
        const int tb = tbufs == 2 ? (uiter & 1) : 0;
        const uint32_t tuse = tbufs == 2 ? uint32_t(uiter >> 1) : uint32_t(uiter);
        const uint32_t bt = b0 + uint32_t(tb) * uint32_t(p.kblocks) * kBBlockBytes;
        mbar_wait(&afull_bar[tb], tuse & 1);
        tc_fence_after();
        for (int i = i0; i < i1; ++i) {
          mbar_wait(&tempty_bar[acc], acc_phase ^ 1);
          tc_fence_after();
          const uint32_t d_tmem = tmem_base + uint32_t(acc * kBN);
          for (int kb = 0; kb < p.kblocks; ++kb) {
            mbar_wait(&full_bar[stage], phase);
            tc_fence_after();
            const uint64_t ad = sw128_kmajor_desc(a0 + uint32_t(stage) * kABlockBytes);
            const uint64_t bd = sw128_kmajor_desc(bt + uint32_t(kb) * kBBlockBytes);
            const int ksteps = kb == p.kblocks - 1 ? p.klast : kBK / 16;
#pragma unroll
            for (int k = 0; k < kBK / 16; ++k)
              if (k < ksteps) mma_f16_ss(d_tmem, ad + uint64_t(2 * k), bd + uint64_t(2 * k), idesc, (kb | k) != 0);
            mma_commit(&empty_bar[stage]);
            if (++stage == stages) { stage = 0; phase ^= 1; }
          }
          mma_commit(&tfull_bar[acc]);
          if (++acc == 2) { acc = 0; acc_phase ^= 1; }
        }
        mma_commit(&aempty_bar[tb]);  // the resident tile may be replaced
      }
    } else if (lane == 0 && leader) {
      constexpr uint32_t idesc = idesc_f16_f32(kPair ? 2 * kBM : kBM, kBN);
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      int uiter = 0;
      uint32_t titer = 0;
      const uint32_t a0 = smem_u32(smemA), b0 = smem_u32(smemB);
      const uint64_t at_desc = sw32_kmajor_desc(smem_u32(smemAt));
      for (int u = first_unit; u < nunits; u += unit_step, ++uiter) {
        const int cc = u / ngroups;
        int t0 = cc * p.tiles_per_unit;
        int t1 = min(p.ntiles, t0 + p.tiles_per_unit);
        if (p.ulist != nullptr) { t0 = p.ulist[3 * u + 1]; t1 = p.ulist[3 * u + 2]; }
        if (p.a_resident) {
          mbar_wait(afull_bar, uiter & 1);
          tc_fence_after();
        }
        for (int t = t0; t < t1; ++t) {
          DK_TWAIT(3, mbar_wait(&tempty_bar[acc], acc_phase ^ 1));
          tc_fence_after();
          const uint32_t d_tmem = tmem_base + uint32_t(acc * kBN);
          for (int kb = 0; kb < p.kblocks; ++kb) {
            DK_TWAIT(4, mbar_wait(&full_bar[stage], phase));
            tc_fence_after();
            const uint32_t abase = p.a_resident ? a0 + uint32_t(kb) * kABlockBytes : a0 + uint32_t(stage) * kABlockBytes;
            const uint32_t bbase = b0 + uint32_t(stage) * kBStage;
            const uint64_t ad = sw128_kmajor_desc(abase), bd = sw128_kmajor_desc(bbase);
            // k-steps over the K padding only multiply zeros: skipped (c3 fp16 sweeps: 7 of 8)
            const int ksteps = kb == p.kblocks - 1 ? p.klast : kBK / 16;
#pragma unroll
            for (int k = 0; k < kBK / 16; ++k) {
              if (k < ksteps) {
                if constexpr (kPair) mma_f16_ss_pair(d_tmem, ad + uint64_t(2 * k), bd + uint64_t(2 * k), idesc, (kb | k) != 0);
                else mma_f16_ss(d_tmem, ad + uint64_t(2 * k), bd + uint64_t(2 * k), idesc, (kb | k) != 0);
              }
            }
            if constexpr (kPair) mma_commit_pair_mc(&empty_bar[stage], uint16_t(0x3));
            else mma_commit(&empty_bar[stage]);
            if (++stage == stages) { stage = 0; phase ^= 1; }
          }
          if (tail) {  // the 16 norm columns: A tail (resident) x this tile's B tail (column-norm slot)
            const uint32_t xs = titer % kXnSlots;
            mbar_wait(&xfull_bar[xs], (titer / kXnSlots) & 1);
            tc_fence_after();
            mma_f16_ss(d_tmem, at_desc, sw32_kmajor_desc(smem_u32(smemX + xs * xslot)), idesc, 1u);
          }
          ++titer;
          if constexpr (kPair) mma_commit_pair_mc(&tfull_bar[acc], uint16_t(0x3));
          else mma_commit(&tfull_bar[acc]);
          if (++acc == 2) { acc = 0; acc_phase ^= 1; }
        }
        if (p.a_resident) {
          if constexpr (kPair) mma_commit_pair_mc(aempty_bar, uint16_t(0x3));
          else mma_commit(aempty_bar);
        }
      }
    }
  } else if (kPP && warp >= kEpiWarp0) {
    // ===================== ping-pong KDE epilogue =====================
    // warp (quarter, cg): group = cg >> 1 owns accumulator `group` (tiles with titer % 2 ==
    // group), half = cg & 1 its columns [128 half, 128 half + 128), in two 64-column steps
    const int ew = int(warp) - kEpiWarp0;
    const int quarter = int(warp & 3);
    const int cg = ew >> 2;
    const uint32_t group = uint32_t(cg >> 1);
    const int half = cg & 1;
    const int lrow = quarter * 32 + int(lane);
    uint32_t ph = 0;  // phase of this group's accumulator barriers
    uint32_t titer = 0;
    const float m2s = *p.m2s;
    const float negc = is_aug(MODE) ? p.negc * m2s : p.negc;  // norm columns: t = S * m2s * negc
    for (int u = first_unit; u < nunits; u += unit_step) {
      float mn = __int_as_float(0x7f800000);  // MODE_KDE_EXP: smallest approximate d2 of the row in this unit
      const int qb = u % ngroups, cc = u / ngroups;
      const int t0 = cc * p.tiles_per_unit;
      const int t1 = min(p.ntiles, t0 + p.tiles_per_unit);
      const int row = qb * kBM + lrow;
      const float qn = p.qn[row];
      double usum = 0.0;
      for (int t = t0; t < t1; ++t, ++titer) {
        if ((titer & 1u) != group) continue;
        const uint32_t xs = titer % kXnSlots;
        DK_TWAIT(0, mbar_wait(&tfull_bar[group], ph));
        tc_fence_after();
        DK_TWAIT(1, mbar_wait(&xfull_bar[xs], (titer / kXnSlots) & 1));
        const uint32_t taddr = tmem_base + (uint32_t(quarter * 32) << 16) + uint32_t(group * kBN + half * 128);
        const int64_t tbase = int64_t(t) * p.tile_stride * kBN + half * 128;
        const float* xsm = smemX + xs * xslot + half * 128;
        float2 a0 = make_float2(0.f, 0.f), a1 = make_float2(0.f, 0.f);
#pragma unroll 1
        for (int sub = 0; sub < 2; ++sub) {
          uint32_t r0[32], r1[32];
          const int64_t cbase = tbase + sub * 64;
          const bool full = cbase + 64 <= p.n;
          tmem_ld32(taddr + uint32_t(sub * 64), r0);
          tmem_ld32(taddr + uint32_t(sub * 64 + 32), r1);
          tmem_ld_wait();
          if (sub == 1) {  // the whole 128-column slice is in registers: release the accumulator
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&tempty_bar[group]);
          }
          epi_chunk<epi_mode(MODE)>(r0, xsm + sub * 64, qn, m2s, negc, 0.f, full, cbase, p.n, a0, a1, mn, p,
                                    row, nullptr, nullptr, lrow);
          epi_chunk<epi_mode(MODE)>(r1, xsm + sub * 64 + 32, qn, m2s, negc, 0.f, full, cbase + 32, p.n, a0, a1,
                                    mn, p, row, nullptr, nullptr, lrow);
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&xempty_bar[xs]);
        ph ^= 1u;
        const float hs = (a0.x + a0.y) + (a1.x + a1.y);
        if constexpr (is_cold(MODE)) {
          // a half whose sum exceeds hot_thr is left to the split3 sweep (bit set); the others are summed here
          const bool hot = hs > p.hot_thr && row < p.nq;
          const uint32_t w = __ballot_sync(0xffffffffu, hot);
          if (lane == 0) p.hot_bits[(size_t(qb) * p.ntiles + t) * kHotWords + quarter * 2 + half] = w;
          if (!hot) usum += double(hs);
        } else {
          usum += double(hs);
        }
      }
      p.part[(size_t(cc) * kColGroups + cg) * p.nq_pad + row] = usum;
      exp_guard_flag<MODE>(p, row, mn);
    }
  } else if (tmajor && warp >= kEpiWarp0) {
    // ===================== tile-major FILTER epilogue =====================
    // the query block changes every iteration: its |q|^2 and thresholds are read per tile
    // pass, candidates go straight to the global lists (one atomic per 32-column chunk with hits)
    if constexpr (MODE == MODE_FILTER) {
      const int ew = int(warp) - kEpiWarp0;
      const int quarter = int(warp & 3);
      const int cg = ew >> 2;
      const int lrow = quarter * 32 + int(lane);
      int acc = 0;
      uint32_t acc_phase = 0;
      uint32_t titer = 0;
      const float m2s = *p.m2s;
      float* sd = reinterpret_cast<float*>(sbuf) + (size_t(ew) * 32 + lane) * kSdStride;  // this lane's d2 row
      int uslot = 0;
      uint32_t uph = 0;
      for (;;) {
        mbar_wait(&ufull_bar[uslot], uph);
        const int u = s_unit[uslot];
        __syncwarp();
        if (lane == 0) mbar_arrive(&uempty_bar[uslot]);
        if (++uslot == kUnitSlots) { uslot = 0; uph ^= 1; }
        if (u < 0) break;
        const int64_t cbase = int64_t(__ldg(p.ulist + 3 * u)) * kBN + cg * 64;
        const int i0 = __ldg(p.ulist + 3 * u + 1), i1 = __ldg(p.ulist + 3 * u + 2);
        const bool full = cbase + 64 <= p.n;
        for (int i = i0; i < i1; ++i, ++titer) {
          const int row = __ldg(p.blist + i) * kBM + lrow;
          const float qn = __ldg(p.qn + row);
          const float tau = __ldg(p.tau + row);
          const uint32_t xs = titer % kXnSlots;
          mbar_wait(&tfull_bar[acc], acc_phase);
          tc_fence_after();
          const uint32_t taddr = tmem_base + (uint32_t(quarter * 32) << 16) + uint32_t(acc * kBN + cg * 64);
          uint32_t r0[32], r1[32];
          tmem_ld32(taddr, r0);
          tmem_ld32(taddr + 32u, r1);
          tmem_ld_wait();
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&tempty_bar[acc]);
          if (++acc == 2) { acc = 0; acc_phase ^= 1; }
          mbar_wait(&xfull_bar[xs], (titer / kXnSlots) & 1);
          const float* xsm = smemX + xs * kBN + cg * 64;
          if (p.knn_aug) {
            filter_chunk_tm<true>(r0, xsm, qn, m2s, tau, full, cbase, p, row, sd);
            filter_chunk_tm<true>(r1, xsm + 32, qn, m2s, tau, full, cbase + 32, p, row, sd);
          } else {
            filter_chunk_tm<false>(r0, xsm, qn, m2s, tau, full, cbase, p, row, sd);
            filter_chunk_tm<false>(r1, xsm + 32, qn, m2s, tau, full, cbase + 32, p, row, sd);
          }
          __syncwarp();
          if (lane == 0) mbar_arrive(&xempty_bar[xs]);
        }
      }
    }
  } else if (warp >= kEpiWarp0) {
    // ===================== epilogue (each CTA, its own 128 rows) =====================
    const int ew = int(warp) - kEpiWarp0;
    const int quarter = int(warp & 3);
    const int cg = ew >> 2;  // 64-column group of the tile
    const int lrow = quarter * 32 + int(lane);
    int acc = 0;
    uint32_t acc_phase = 0;
    uint32_t titer = 0;
    const float m2s = *p.m2s;
    const float negc = is_aug(MODE) ? p.negc * m2s : p.negc;
#ifdef DK_TIMING
    const long long tepi0 = clock64();
#endif
    for (int u = first_unit; u < nunits; u += unit_step) {
      int qb = (u % ngroups) * (kPair ? 2 : 1) + int(crank), cc = u / ngroups;
      int t0 = cc * p.tiles_per_unit;
      int t1 = min(p.ntiles, t0 + p.tiles_per_unit);
      if (p.ulist != nullptr) { qb = p.ulist[3 * u]; t0 = p.ulist[3 * u + 1]; t1 = p.ulist[3 * u + 2]; }
      const int row = qb * kBM + lrow;
      const float qn = p.qn[row];
      float tau = 0.f;
      if constexpr (MODE == MODE_FILTER) tau = p.tau[row];
      float2 hpar = make_float2(0.f, 0.f);  // MODE_HIST: (lo, 1 / (top - lo)) of the row
      if constexpr (MODE == MODE_HIST) {
        tau = p.htop[row];
        hpar = make_float2(p.hlo[row], p.hinv[row]);
      }
      double usum = 0.0;
      float mn = __int_as_float(0x7f800000);
      // TILEMIN segments: seg_tiles > 0 -> groups of seg_tiles whole tiles; seg_tiles == 0 -> one
      // segment per (tile, 64-column group)
      const int segdiv = p.seg_tiles > 0 ? p.seg_tiles : 1;
      int seg = MODE == MODE_TILEMIN ? t0 / segdiv : 0;
      for (int t = t0; t < t1; ++t, ++titer) {
        const uint32_t xs = titer % kXnSlots;
        bool take = true;  // MODE_KDE_HOT: this row's half of the tile is hot (summed here)
        bool any = true;   // MODE_KDE_HOT: some row of this warp's quarter is (else no epilogue math)
        if constexpr (MODE == MODE_KDE_HOT) {
          const uint32_t w = p.hot_bits[(size_t(qb) * p.ntiles + p.tlist[t]) * kHotWords + quarter * 2 + (cg >> 1)];
          take = ((w >> lane) & 1u) != 0u;
          any = w != 0u;
        }
        if constexpr (MODE == MODE_TILEMIN) {
          if (p.seg_tiles > 0 && t / segdiv != seg) {
            atomicMin(reinterpret_cast<int*>(&p.tmin[size_t(seg) * p.nq_pad + row]), __float_as_int(fmaxf(mn, 0.f)));
            seg = t / segdiv;
            mn = __int_as_float(0x7f800000);
          }
        }
        DK_TWAIT(0, mbar_wait(&tfull_bar[acc], acc_phase));
        tc_fence_after();
        const uint32_t taddr = tmem_base + (uint32_t(quarter * 32) << 16) + uint32_t(acc * kBN + cg * 64);
        uint32_t r0[32], r1[32];
        tmem_ld32(taddr, r0);
        tmem_ld32(taddr + 32u, r1);
        tmem_ld_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          if constexpr (kPair) mbar_arrive_cluster(&tempty_bar[acc], 0u);
          else mbar_arrive(&tempty_bar[acc]);
        }
        if (++acc == 2) { acc = 0; acc_phase ^= 1; }
        DK_TWAIT(1, mbar_wait(&xfull_bar[xs], (titer / kXnSlots) & 1));
        if constexpr (MODE == MODE_NULL) {  // pipeline probe: consume the accumulator, no epilogue math
          uint32_t x = 0;
#pragma unroll
          for (int j = 0; j < 32; ++j) x ^= r0[j] ^ r1[j];
          if (x == 0x9e3779b9u) p.tmin[row] = 0.f;
          __syncwarp();
          if (lane == 0) mbar_arrive(&xempty_bar[xs]);
          continue;
        }
        const int64_t cbase = int64_t(p.tlist != nullptr ? p.tlist[t] : t * p.tile_stride) * kBN + cg * 64;
        const float* xsm = smemX + xs * xslot + cg * 64;
        const bool full = cbase + 64 <= p.n;
        float2 a0 = MODE == MODE_HIST ? hpar : make_float2(0.f, 0.f), a1 = make_float2(0.f, 0.f), b0 = a0;
        // k-NN sweeps over operands with norm columns take the aug arithmetic (knn_d2), chosen per pass
        auto chunks = [&](auto aug) {
          constexpr bool kA = decltype(aug)::value;
          epi_chunk<epi_mode(MODE), kA>(r0, xsm, qn, m2s, negc, tau, full, cbase, p.n, a0, a1, mn, p, row, scnt,
                                        sbuf, lrow);
          // TILEMIN returns the chunk's two 16-column minima in its first accumulator
          epi_chunk<epi_mode(MODE), kA>(r1, xsm + 32, qn, m2s, negc, tau, full, cbase + 32, p.n,
                                        MODE == MODE_TILEMIN ? b0 : a0, a1, mn, p, row, scnt, sbuf, lrow);
        };
        if (any) {  // warp-uniform
          if (is_knn_sweep(MODE) && p.knn_aug) chunks(std::true_type{});
          else chunks(std::false_type{});
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&xempty_bar[xs]);
        if constexpr (is_kde(MODE)) {
          if (take) usum += double((a0.x + a0.y) + (a1.x + a1.y));
        } else if constexpr (MODE == MODE_TILEMIN) {
          if (p.tlist != nullptr) {
            // listed threshold sweep: 8 segments of 32 columns per tile (segment = list position x 8 + 32-column
            // group), fine enough that the tiles near a query hold k segments
            DK_DCHECK(t - qb * p.list_stride >= 0 && t - qb * p.list_stride < p.list_stride);
            float* tm = p.tmin + (size_t(t - qb * p.list_stride) * 8 + cg * 2) * p.nq_pad + row;
            tm[0] = fmaxf(fminf(a0.x, a0.y), 0.f);
            tm[size_t(p.nq_pad)] = fmaxf(fminf(b0.x, b0.y), 0.f);
            mn = __int_as_float(0x7f800000);
          } else if (p.seg_tiles == 0) {
            p.tmin[(size_t(t) * kColGroups + cg) * p.nq_pad + row] = fmaxf(mn, 0.f);
            mn = __int_as_float(0x7f800000);
          }
        }
      }
      if constexpr (MODE == MODE_KDE_HOT) {
        p.part[(size_t(u) * kColGroups + cg) * kBM + lrow] = usum;  // listed: one partial per unit
      } else if constexpr (is_kde(MODE)) {
        p.part[(size_t(cc) * kColGroups + cg) * p.nq_pad + row] = usum;
        exp_guard_flag<MODE>(p, row, mn);
      } else if constexpr (MODE == MODE_TILEMIN) {
        if (t1 > t0 && p.seg_tiles > 0)
          atomicMin(reinterpret_cast<int*>(&p.tmin[size_t(seg) * p.nq_pad + row]), __float_as_int(fmaxf(mn, 0.f)));
      } else if constexpr (MODE == MODE_HIST) {
        // flush the unit's bins: one global atomic per nonzero (row, bin)
        epi_bar();
        if (cg == 0) {
          uint32_t* hrow = reinterpret_cast<uint32_t*>(sbuf) + lrow * kHistStride;
          for (int b = 0; b < kHistBins; ++b) {
            const uint32_t v = hrow[b];
            if (v) {
              atomicAdd(p.hist + size_t(row) * kHistBins + b, v);
              hrow[b] = 0u;
            }
          }
        }
        epi_bar();
      } else if constexpr (MODE == MODE_FILTER) {
        // flush the unit's staged candidates: one global atomic per row
        epi_bar();
        if (cg == 0) {
          const uint32_t c = min(scnt[lrow], uint32_t(kStageCap));
          if (c) {
            const uint32_t base = atomicAdd(&p.cand_cnt[row], c);
            for (uint32_t i = 0; i < c; ++i)
              if (base + i < uint32_t(p.cap)) p.cand[size_t(row) * p.cap + base + i] = sbuf[lrow * kStageCap + i];
          }
          scnt[lrow] = 0;
        }
        epi_bar();
      }
    }
#ifdef DK_TIMING
    dbgw[2] = clock64() - tepi0;
    dbgw[6] = titer;
#endif
  }
#ifdef DK_TIMING
  if (lane == 0)
#pragma unroll
    for (int i = 0; i < 8; ++i)
      if (dbgw[i]) atomicAdd(&g_dbg[i], (unsigned long long)dbgw[i]);
#endif

  __syncwarp();
  tc_fence_before();
  if constexpr (kPair) cluster_sync_all();  // no remote arrive / MMA write may target an exited CTA
  else __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    if constexpr (kPair) tmem_dealloc_pair<kTmemCols>(tmem_base);
    else tmem_dealloc<kTmemCols>(tmem_base);
  }
}

}  // namespace dk
