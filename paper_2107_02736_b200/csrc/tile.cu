// tile.cu — host launcher for the tcgen05 tile sweep (tile_kernel.cuh).

#include <algorithm>
#include <limits>
#include <map>
#include <mutex>
#include <tuple>
#include <vector>

#include "internal.h"
#include "tile_kernel.cuh"

namespace dk {

namespace {

typedef CUresult (*PFN_encodeTiled_t)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                      const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                      CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

PFN_encodeTiled_t get_encode_fn() {
  static PFN_encodeTiled_t fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_encodeTiled_t>(p);
  });
  if (!fn) throw Error{DK_ECUDA, "cuTensorMapEncodeTiled entry point unavailable"};
  return fn;
}

constexpr size_t kMaxSmem = 232448;  // sm_100 opt-in dynamic shared memory per block

struct Plan {
  int a_resident, stages, tiles_per_unit, ncc;
  int tbufs;  // tile-major: resident tile buffers
  size_t smem;
};

// Tiles per work unit.  Units (query block, column chunk) are dealt to the persistent CTAs
// round-robin, so the sweep ends when the most loaded CTA does: pick, among 12-48 units
// per CTA, the chunk length whose exact makespan (in tiles, the ragged last chunk
// included) is smallest — e.g. c2 (3907 tiles x 79 query blocks on 148 SMs): 130 tiles
// per unit gives 2210 tiles on the busiest CTA vs an average of 2085; the balanced
// choice is within ~1%.  Ties go to the longer chunk (fewer partial sums).  Cached.
int64_t balanced_tiles_per_unit(int ntiles, int ngroups, int nslots) {
  static std::mutex mu;
  static std::map<std::tuple<int, int, int>, int64_t> cache;
  const auto key = std::make_tuple(ntiles, ngroups, nslots);
  {
    std::lock_guard<std::mutex> lk(mu);
    auto it = cache.find(key);
    if (it != cache.end()) return it->second;
  }
  const int64_t total = int64_t(ntiles) * ngroups;
  int64_t lo = std::max<int64_t>(1, total / (int64_t(nslots) * 48));
  int64_t hi = std::max<int64_t>(1, total / (int64_t(nslots) * 12));
  hi = std::min<int64_t>(hi, ntiles);
  lo = std::min(lo, hi);
  int64_t best = hi, best_span = std::numeric_limits<int64_t>::max();
  std::vector<int64_t> load(static_cast<size_t>(nslots));
  for (int64_t tpu = hi; tpu >= lo; --tpu) {
    const int64_t ncc = (ntiles + tpu - 1) / tpu;
    const int64_t last = ntiles - (ncc - 1) * tpu;
    const int64_t units = int64_t(ngroups) * ncc;
    std::fill(load.begin(), load.end(), 0);
    for (int64_t u = 0; u < units; ++u) load[size_t(u % nslots)] += (u / ngroups == ncc - 1) ? last : tpu;
    const int64_t span = *std::max_element(load.begin(), load.end());
    if (span < best_span) {
      best_span = span;
      best = tpu;
    }
  }
  std::lock_guard<std::mutex> lk(mu);
  cache[key] = best;
  return best;
}

Plan make_plan(int kblocks, int ntiles, int ngroups, int nslots, int mode, bool pair, bool tmajor = false) {
  Plan pl{};
  if (tmajor) {
    pl.a_resident = 0;
    // two tile buffers when they leave a >= 4-stage ring: the next unit's tile (a DRAM read) loads
    // while the current one's query blocks stream past, instead of stalling the MMA once per unit
    static const int want = [] {
      const char* v = std::getenv("DK_KNN_TBUFS");  // A/B switch
      return v != nullptr && std::atoi(v) == 1 ? 1 : 2;
    }();
    const int bufs = want == 2 && tile_smem_bytes(kblocks, 0, 4, mode, false, 2) <= kMaxSmem ? 2 : 1;
    int st = 3;
    while (st < 8 && tile_smem_bytes(kblocks, 0, st + 1, mode, false, bufs) <= kMaxSmem) ++st;
    pl.stages = st;
    pl.tbufs = bufs;
    pl.tiles_per_unit = 1;
    pl.ncc = 1;
    pl.smem = tile_smem_bytes(kblocks, 0, st, mode, false, bufs);
    return pl;
  }
  // keep the query block resident when it fits next to a >=3-stage ring
  if (tile_smem_bytes(kblocks, 1, 3, mode, pair) <= kMaxSmem) {
    pl.a_resident = 1;
    int st = 3;
    while (st < 10 && tile_smem_bytes(kblocks, 1, st + 1, mode, pair) <= kMaxSmem) ++st;
    pl.stages = st;
  } else {
    pl.a_resident = 0;
    int st = 2;
    while (st < 6 && tile_smem_bytes(kblocks, 0, st + 1, mode, pair) <= kMaxSmem) ++st;
    pl.stages = st;
  }
  const int64_t tpu = balanced_tiles_per_unit(ntiles, ngroups, nslots);
  pl.tiles_per_unit = int(tpu);
  pl.ncc = int((ntiles + tpu - 1) / tpu);
  pl.smem = tile_smem_bytes(kblocks, pl.a_resident, pl.stages, mode, pair);
  return pl;
}

template <int MODE, bool kPair>
void launch_mode(const CUtensorMap& ta, const CUtensorMap& tb, const TileParams& p, int grid, size_t smem,
                 cudaStream_t s, const CUtensorMap* tat = nullptr, const CUtensorMap* tbt = nullptr) {
  static std::once_flag once;
  static cudaError_t attr_err = cudaSuccess;
  std::call_once(once, [] {
    attr_err = cudaFuncSetAttribute(tile_kernel<MODE, kPair>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    int(kMaxSmem));
  });
  DK_CUDA(attr_err);
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(unsigned(grid));
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = kPair ? 2 : 1;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  DK_CUDA(cudaLaunchKernelEx(&cfg, tile_kernel<MODE, kPair>, ta, tb, tat ? *tat : ta, tbt ? *tbt : tb, p));
  DK_CHECK_LAUNCH();
}

template <int MODE>
void launch_any(bool pair, const CUtensorMap& ta, const CUtensorMap& tb, const TileParams& p, int grid, size_t smem,
                cudaStream_t s) {
  if (pair) launch_mode<MODE, true>(ta, tb, p, grid, smem, s);
  else launch_mode<MODE, false>(ta, tb, p, grid, smem, s);
}

bool g_pair_enabled = false;  // DK_PAIR=1 enables: measured slower (CTA coupling), see DESIGN.md

}  // namespace

CUtensorMap make_tmap_2d_f16(const void* base, uint64_t rows, uint64_t kp, uint32_t box_rows) {
  CUtensorMap m;
  cuuint64_t dims[2] = {kp, rows};
  cuuint64_t strides[1] = {kp * 2};
  cuuint32_t box[2] = {uint32_t(kBK), box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = get_encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, const_cast<void*>(base), dims, strides, box,
                               estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                               CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw Error{DK_ECUDA, "cuTensorMapEncodeTiled failed: " + std::to_string(int(r))};
  return m;
}

CUtensorMap make_tmap_tail_f16(const void* base, uint64_t rows, uint32_t box_rows) {
  CUtensorMap m;
  cuuint64_t dims[2] = {uint64_t(kTailK), rows};
  cuuint64_t strides[1] = {uint64_t(kTailK) * 2};
  cuuint32_t box[2] = {uint32_t(kTailK), box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = get_encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, const_cast<void*>(base), dims, strides, box,
                               estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_32B,
                               CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw Error{DK_ECUDA, "cuTensorMapEncodeTiled (tail) failed: " + std::to_string(int(r))};
  return m;
}

bool tile_major_fits(int32_t Kp) {
  return tile_smem_bytes(enc_kblocks(Kp), 0, 3, MODE_FILTER, false, true) <= kMaxSmem;
}

static bool use_pair(int nqb) { return g_pair_enabled && nqb >= 2 && nqb % 2 == 0; }

size_t sweep_part_count(int64_t n_pad, int32_t nq_pad, int num_sms, bool allow_pair) {
  const int ntiles = int(n_pad / kBN);
  const int nqb = nq_pad / kBM;
  const bool pr = allow_pair && use_pair(nqb);
  const Plan pl = make_plan(1, ntiles, pr ? nqb / 2 : nqb, pr ? num_sms / 2 : num_sms, MODE_KDE_GAUSS, pr);
  return size_t(pl.ncc) * kColGroups * size_t(nq_pad);
}

// An upper bound of sweep_part_count over every query padding up to max_pad, from the plan's
// chunk-length range alone (balanced_tiles_per_unit picks tiles_per_unit >= lo, so a plan has at
// most ceil(ntiles / lo) column chunks) — no makespan search per padding.
size_t sweep_part_bound(int64_t n_pad, int32_t max_pad, int num_sms) {
  const int64_t ntiles = n_pad / kBN;
  size_t cap = 0;
  for (int32_t pad = kBM; pad <= max_pad; pad = pad == kBM ? 2 * kBM : pad + 2 * kBM) {
    const int nqb = pad / kBM;
    for (int pr = 0; pr < 2; ++pr) {
      const int64_t ngroups = pr ? std::max(1, nqb / 2) : nqb;
      const int64_t nslots = pr ? std::max(1, num_sms / 2) : num_sms;
      const int64_t total = ntiles * ngroups;
      const int64_t hi = std::min<int64_t>(std::max<int64_t>(1, total / (nslots * 12)), ntiles);
      const int64_t lo = std::min(std::max<int64_t>(1, total / (nslots * 48)), hi);
      cap = std::max(cap, size_t((ntiles + lo - 1) / lo) * kColGroups * size_t(pad));
    }
  }
  return cap;
}

void set_pair_enabled(bool on) { g_pair_enabled = on; }

void launch_sweep(const SweepArgs& a, int num_sms, cudaStream_t s) {
  const QueryOperand& q = *a.qop;
  const Encoding& e = *a.enc;
  const int kblocks = enc_kblocks(e.Kp);
  const int ntiles_all = int(a.n_pad / kBN);
  const int ntiles = (ntiles_all + a.tile_stride - 1) / a.tile_stride;
  const int nqb = q.nq_pad / kBM;
  const bool pr = a.ulist == nullptr && a.mode != MODE_KDE_COLD && !q.aug && use_pair(nqb);  // never with norm columns
  const int ngroups = pr ? nqb / 2 : nqb;
  const int nslots = pr ? num_sms / 2 : num_sms;  // CTAs (or CTA pairs) resident at once
  const bool tmajor = a.tmajor != 0;
  if (tmajor && (a.mode != MODE_FILTER || a.ulist == nullptr || a.blist == nullptr))
    throw Error{DK_EINVAL, "internal: tile-major sweeps are FILTER tile lists"};
  // norm columns in tail operands: only the resident-A KDE sweeps (otherwise the plain epilogue:
  // the main A of a tail-mode query operand is plain q)
  const bool want_tail = q.aug && q.T != nullptr && e.T != nullptr && a.ulist == nullptr && !pr &&
                         (a.mode == MODE_KDE_GAUSS || a.mode == MODE_KDE_COLD);
  Plan pl = make_plan(kblocks, ntiles, ngroups, nslots, a.mode, pr, tmajor);
  bool tail = false;
  if (want_tail && pl.a_resident) {
    int st = pl.stages;
    while (st > 2 && tile_smem_bytes(kblocks, 1, st, a.mode, false, false, true) > kMaxSmem) --st;
    if (tile_smem_bytes(kblocks, 1, st, a.mode, false, false, true) <= kMaxSmem) {
      tail = true;
      pl.stages = st;
      pl.smem = tile_smem_bytes(kblocks, 1, st, a.mode, false, false, true);
    }
  }
  const bool aug = q.aug && (q.T == nullptr || tail);  // norm columns usable by this sweep

  TileParams p{};
  p.nq = q.nq;
  p.nq_pad = q.nq_pad;
  p.nqb = nqb;
  p.n = a.n;
  p.ntiles = ntiles;
  p.tile_stride = a.tile_stride;
  p.tiles_per_unit = pl.tiles_per_unit;
  p.ncc = pl.ncc;
  p.kblocks = kblocks;
#ifndef DK_KSKIP
#define DK_KSKIP 1
#endif
  {
    // columns holding data (the rest is zero padding); the norm columns of the main operand only
    // when this sweep's A carries them (k-NN sweeps leave them zero: c5, d = 96, 6 MMA steps not 7)
    const bool main_aug = aug && q.T == nullptr && enc_aug_main(e.d, e.mode);
    const int kused = int(enc_kdata(e.d, e.mode)) + (main_aug ? kAugCols : 0);
    const int rem = kused - (kblocks - 1) * kBK;
    p.klast = DK_KSKIP && e.d > 0 && rem > 0 && rem <= kBK ? (rem + 15) / 16 : kBK / 16;
  }
  p.a_resident = pl.a_resident;
  p.stages = pl.stages;
  p.xn = e.xn;
  p.qn = q.qn;
  p.m2s = q.m2s;
  p.negc = a.negc;
  p.part = a.part;
  p.tmin = a.tmin;
  p.tau = a.tau;
  p.cand_cnt = a.cand_cnt;
  p.cand = a.cand;
  p.cap = a.cap;
  p.seg_tiles = a.seg_tiles;
  p.ulist = a.ulist;
  p.tlist = a.tlist;
  p.nunits_list = a.nunits_list;
  p.nunits_dev = a.nunits_dev;
  p.list_stride = a.list_stride;
  p.hlo = a.hlo;
  p.hinv = a.hinv;
  p.htop = a.htop;
  p.hist = a.hist;
  p.hot_bits = a.hot_bits;
  p.hot_thr = a.hot_thr;
  p.tail = tail ? 1 : 0;
  p.knn_aug = aug && (a.mode == MODE_TILEMIN || a.mode == MODE_FILTER || a.mode == MODE_HIST) ? 1 : 0;
  p.tmajor = tmajor ? pl.tbufs : 0;
  p.blist = a.blist;
  p.unit_counter = a.unit_counter;
  if (tmajor && a.unit_counter == nullptr) throw Error{DK_EINVAL, "internal: tile-major sweeps need a unit counter"};
  p.guard = a.guard;
  if (a.ncc_out) *a.ncc_out = pl.ncc;

  // a device-side unit count is unknown here: one CTA per SM, surplus CTAs find no unit
  const int nunits = a.ulist != nullptr ? (a.nunits_dev != nullptr ? nslots : a.nunits_list) : ngroups * pl.ncc;
  if (nunits <= 0) return;
  if (a.ulist != nullptr &&
      (pr || (a.mode != MODE_FILTER && a.mode != MODE_TILEMIN && a.mode != MODE_HIST && a.mode != MODE_KDE_HOT)))
    throw Error{DK_EINVAL, "internal: tile lists are k-NN and two-precision KDE sweeps only"};
  if ((a.mode == MODE_KDE_HOT && a.ulist == nullptr) ||
      ((a.mode == MODE_KDE_HOT || a.mode == MODE_KDE_COLD) && a.hot_bits == nullptr))
    throw Error{DK_EINVAL, "internal: two-precision KDE sweeps need a hot bitmap (and a list for the split3 pass)"};
  if (a.ulist != nullptr && a.mode == MODE_TILEMIN && a.seg_tiles != 0)
    throw Error{DK_EINVAL, "internal: listed TILEMIN sweeps use one segment per 64-column group"};
  const int grid = std::min(nunits, nslots) * (pr ? 2 : 1);
  const CUtensorMap& tb = pr ? e.tmap_half : e.tmap;
  switch (a.mode) {
    case MODE_KDE_GAUSS:
      // MMA-heavy encodings (split3: >= 4 K-blocks per tile) leave no FMA-pipe slack for the
      // exp2 polynomial and run power-capped: every exponential on MUFU is faster there
      // (c3: 6.6 vs 7.0 ms); the single-pass encodings offload 2 of 16 pairs (c2: 2.83 vs 2.98 ms),
      // 4 of 16 with the norm columns (q.aug: one multiply per pair before the exponential)
      if (aug) launch_mode<MODE_KDE_GAUSS_AUG, false>(q.tmap, tb, p, grid, pl.smem, s, &q.tmap_t, &e.tmap_t);
      else if (kblocks >= 4) launch_any<MODE_KDE_GAUSS_MUFU>(pr, q.tmap, tb, p, grid, pl.smem, s);
      else launch_any<MODE_KDE_GAUSS>(pr, q.tmap, tb, p, grid, pl.smem, s);
      break;
    case MODE_KDE_GAUSS_MUFU: launch_any<MODE_KDE_GAUSS_MUFU>(pr, q.tmap, tb, p, grid, pl.smem, s); break;
    case MODE_KDE_EXP: launch_any<MODE_KDE_EXP>(pr, q.tmap, tb, p, grid, pl.smem, s); break;
    case MODE_TILEMIN: launch_any<MODE_TILEMIN>(pr, q.tmap, tb, p, grid, pl.smem, s); break;
    case MODE_FILTER: launch_any<MODE_FILTER>(pr, q.tmap, tb, p, grid, pl.smem, s); break;
    case MODE_NULL: launch_any<MODE_NULL>(pr, q.tmap, tb, p, grid, pl.smem, s); break;
    case MODE_KDE_COLD:
      if (aug) launch_mode<MODE_KDE_COLD_AUG, false>(q.tmap, tb, p, grid, pl.smem, s, &q.tmap_t, &e.tmap_t);
      else launch_mode<MODE_KDE_COLD, false>(q.tmap, tb, p, grid, pl.smem, s);
      break;
    case MODE_KDE_HOT: launch_mode<MODE_KDE_HOT, false>(q.tmap, tb, p, grid, pl.smem, s); break;
    case MODE_HIST:
      if (pr || a.ulist == nullptr) throw Error{DK_EINVAL, "internal: histogram sweeps are listed single-CTA sweeps"};
      launch_mode<MODE_HIST, false>(q.tmap, tb, p, grid, pl.smem, s);
      break;
    default: throw Error{DK_EINVAL, "bad tile mode"};
  }
}

}  // namespace dk

#ifdef DK_TIMING
extern "C" int dk_debug_counters(unsigned long long* out, int reset) {
  if (cudaDeviceSynchronize() != cudaSuccess) return 2;
  if (cudaMemcpyFromSymbol(out, dk::g_dbg, sizeof(unsigned long long) * 8) != cudaSuccess) return 2;
  if (reset) {
    unsigned long long z[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    if (cudaMemcpyToSymbol(dk::g_dbg, z, sizeof(z)) != cudaSuccess) return 2;
  }
  return 0;
}
#endif
