// internal.h — host-side internals shared by the C-ABI translation units.
#pragma once
#include <cuda.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <atomic>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <vector>

#include "../../include/deann_b200.h"
#include <nvtx3/nvToolsExt.h>

#include "checks.cuh"

namespace dk {

void set_error(const std::string& msg);

// NVTX range around every C-ABI entry point (header-only NVTX v3: a no-op unless a profiler
// such as Nsight Systems / Compute is attached), named after the function.
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};
#define DK_NVTX() ::dk::NvtxRange dk_nvtx_range_(__func__)

struct Error {
  dk_status code;
  std::string msg;
};

#define DK_CUDA(call)                                                                           \
  do {                                                                                          \
    cudaError_t e_ = (call);                                                                    \
    if (e_ != cudaSuccess) {                                                                    \
      throw ::dk::Error{e_ == cudaErrorMemoryAllocation ? DK_ENOMEM : DK_ECUDA,                 \
                        std::string(#call) + ": " + cudaGetErrorString(e_) + " at " + __FILE__ + \
                            ":" + std::to_string(__LINE__)};                                    \
    }                                                                                           \
  } while (0)

extern std::atomic<long long> g_launches;  // kernels launched by this library
#define DK_CHECK_LAUNCH()                         \
  do {                                            \
    ::dk::g_launches.fetch_add(1);                \
    DK_CUDA(cudaGetLastError());                  \
  } while (0)

inline bool is_device_ptr(const void* p) {
  if (!p) return false;
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

// C-ABI entry wrapper: exceptions -> status + thread-local message
template <class F>
inline dk_status guard(F&& f) {
  try {
    f();
    return DK_OK;
  } catch (const Error& e) {
    set_error(e.msg);
    cudaGetLastError();  // do not leak a non-sticky error into the next call
    return e.code;
  } catch (const std::bad_alloc&) {
    set_error("host allocation failed");
    return DK_ENOMEM;
  } catch (const std::exception& e) {
    set_error(e.what());
    return DK_ECUDA;
  }
}

struct DeviceGuard {
  int prev = 0;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) DK_CUDA(cudaSetDevice(dev));
  }
  ~DeviceGuard() { cudaSetDevice(prev); }
};

// Opt a kernel into `bytes` of dynamic shared memory (only ever raises the limit).
template <class K>
inline void set_dynamic_smem(K* kernel, size_t bytes) {
  if (bytes <= 48 * 1024) return;
  cudaFuncAttributes fa;
  DK_CUDA(cudaFuncGetAttributes(&fa, kernel));
  if (size_t(fa.maxDynamicSharedSizeBytes) >= bytes) return;
  if (bytes + fa.sharedSizeBytes > 232448)
    throw Error{DK_EINVAL, "kernel needs " + std::to_string(bytes) + " B of shared memory (> 227 KB)"};
  DK_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(bytes)));
}

#define DK_REQUIRE(cond, msg)                          \
  do {                                                 \
    if (!(cond)) throw ::dk::Error{DK_EINVAL, (msg)};  \
  } while (0)

// Norm columns of the exact / fp16 operands (prep.cu): 3 for the row norm, 3 for the query norm.
// They ride in the K padding when they fit (d = 100: 106 of 128).  When d is within 6 of a
// multiple of 64 (c2, d = 128) they go to a separate 16-column "tail" operand instead — one
// 16-wide MMA step on 32-byte-swizzled tiles (8 KB per dataset tile) — because a whole extra
// 64-column K-block costs more feed than the epilogue saves (c2: 2.67 -> 2.83 ms).
constexpr int32_t kAugCols = 6;
constexpr int32_t kTailK = 16;
// K columns holding data: split3 3d (A=[Qh|Ql|Qh], B=[Xl|Xh|Xh]), exact / fp16 d
inline int64_t enc_kdata(int32_t d, int mode) { return mode == 1 ? 3 * int64_t(d) : int64_t(d); }
inline bool enc_aug_main(int32_t d, int mode) {
  return mode != 1 && (int64_t(d) + kAugCols + 63) / 64 == (int64_t(d) + 63) / 64;
}
inline bool enc_aug_tail(int32_t d, int mode) {
  static const bool off = [] {  // A/B: DK_AUG_TAIL=0 leaves such operands without norm columns
    const char* v = std::getenv("DK_AUG_TAIL");
    return v != nullptr && std::atoi(v) == 0;
  }();
  return mode != 1 && !off && !enc_aug_main(d, mode);
}
inline bool enc_has_aug(int32_t d, int mode) { return enc_aug_main(d, mode) || enc_aug_tail(d, mode); }
// padded K (row stride, a multiple of 64) of an encoding: split3 3d, exact / fp16 d (+ norm columns)
inline int32_t enc_kp(int32_t d, int mode) {
  const int64_t k = mode == 1 ? 3 * int64_t(d) : int64_t(d) + (enc_aug_main(d, mode) ? kAugCols : 0);
  return int32_t((k + 63) / 64 * 64);
}
inline int32_t enc_kblocks(int32_t Kp) { return (Kp + 63) / 64; }

// One operand encoding of the dataset for the tensor-core tile.
struct Encoding {
  int mode = -1;            // 0 exact fp16, 1 split3, 2 fp16 single (lossy)
  int32_t Kp = 0;           // padded K (multiple of 64)
  int32_t d = 0;            // data columns per part (K used = d, or 3d for split3)
  __half* B = nullptr;      // [n_pad][Kp]
  __half* T = nullptr;      // [n_pad][kTailK] norm-column tail (enc_aug_tail), else nullptr
  CUtensorMap tmap_t;       // T boxes of 256 rows x 16 columns, 32-byte swizzle
  float* xn = nullptr;      // [n_pad] |x - mu|^2 in fp32
  double* mu = nullptr;     // [d] centring (nullptr = none)
  float* sx = nullptr;      // device scalar: power-of-two scale applied to x
  float xn_max = 0.f;       // max of xn (host copy, k-NN certificate)
  float eps_rel = 0.f;      // |approx d2 - exact d2| <= eps_rel * (|q|^2 + xn_max)
  CUtensorMap tmap;         // B boxes of 256 rows (single-CTA sweep)
  CUtensorMap tmap_half;    // B boxes of 128 rows (2-CTA pair sweep: each CTA loads half)
};

// Cluster-sorted copy of the rows for the pruned k-NN FILTER pass (ivf.cu build,
// capi.cu knn_device): rows grouped by a few Lloyd iterations of k-means, the sweep
// operand re-encoded in that order (same scale and centring as the k-NN encoding, so
// the query operand is shared), and per-cluster balls (centroid, radius) that bound
// the distance from a query to every row of a tile from below.
constexpr int32_t kBallNbrs = 16;
struct KnnClusters {
  int32_t C = 0;
  double* cent = nullptr;    // [C][d] centroids (fp64)
  double* rad = nullptr;     // [C] max |x - cent| over the members, inflated by 1e-12 relative
  int64_t* perm = nullptr;   // [n] sorted position -> dataset row
  float* xs = nullptr;       // [n][d] rows in sorted order
  int64_t* off = nullptr;    // [C + 1] first sorted position of each ball
  int32_t* nbr = nullptr;    // [C][kBallNbrs] nearest other balls by centroid distance (threshold-sweep lists)
  int32_t* tclo = nullptr;   // [ntiles] first / last cluster of each 256-row tile of the sorted rows
  int32_t* tchi = nullptr;
  Encoding enc;              // sweep operand of xs (mode of the k-NN encoding)
  // pruning pays only when it skips tiles: the swept fraction of each call's last batch is
  // copied back asynchronously (stat_host, stat_ev) and read at the next call; 3 calls in a
  // row sweeping > 60% of the pairs turn pruning off, and every 32nd call re-tests it
  bool useless = false;
  int over = 0, off_calls = 0;
  int32_t* stat_host = nullptr;  // pinned: [0] swept (block, tile) pairs of the last batch
  double stat_total = 0;         // (block, tile) pairs of that batch
  bool stat_pending = false;
  cudaEvent_t stat_ev = nullptr;
  // two-precision exact KDE (capi.cu kde_hybrid): split3 operand of the sorted rows (same centring
  // as the k-NN encoding), built on the first hybrid call; the hot fraction of each call's first
  // batch is read back like the pruning statistic (at once when more batches follow), and a
  // bandwidth that makes most (block, tile) pairs hot (a wide kernel: c5) turns the hybrid off for
  // the rest of the call and the next 32 calls
  Encoding enc3;
  bool hyb_failed = false;     // the split3 copy did not fit in device memory
  bool hyb_useless = false;
  int hyb_off_calls = 0;
  int32_t* hyb_stat_host = nullptr;  // pinned: [0] hot (block, tile) pairs of the last first batch
  double hyb_stat_total = 0;
  bool hyb_stat_pending = false;
  cudaEvent_t hyb_stat_ev = nullptr;
};

// Growable device scratch, carved per call.
struct Workspace {
  uint8_t* base = nullptr;
  size_t cap = 0;
  size_t off = 0;
  void reserve(size_t bytes);
  void reset() { off = 0; }
  template <class T>
  T* take(size_t count) {
    size_t a = (off + 255) & ~size_t(255);
    T* p = reinterpret_cast<T*>(base + a);
    off = a + count * sizeof(T);
    if (off > cap) throw Error{DK_ECUDA, "workspace overflow (internal sizing bug)"};
    return p;
  }
  ~Workspace();
};

}  // namespace dk

struct dk_dataset {
  int device = 0;
  int num_sms = 148;
  int64_t n = 0, n_pad = 0;
  int32_t d = 0;
  int64_t global_offset = 0, global_n = 0;
  int precision = 0;
  bool int_exact = false;   // rows are small integers: exact fp16 encoding valid
  float* X = nullptr;       // [n][d] fp32 rows
  double* xn64 = nullptr;   // [n]
  dk::Encoding enc_exact;   // mode 0 (only if int_exact)
  dk::Encoding enc_split;   // mode 1 (built lazily when needed)
  dk::Encoding enc_fp16;    // mode 2 (opt-in)
  dk::Workspace ws;
  double* mu = nullptr;     // [d] column means (split/fp16 centring)
  int64_t* rsp_inverse = nullptr;  // [n] original id -> permuted position (dk_rsp_attach)
  uint32_t* flag_host = nullptr;   // pinned words: query-check flags of the speculative sweeps (2 chunks)
  cudaEvent_t flag_event = nullptr;
  // exact-KDE guard (redo.cu): queries of the last dk_naive call recomputed in fp64, per chunk (pinned)
  int32_t* redo_host = nullptr;
  cudaEvent_t redo_event = nullptr;
  int redo_mask = 0;
  int64_t knn_budget = 0;  // bytes of k-NN candidate storage per batch (set at fit from the free memory)
  cudaStream_t copy_stream = nullptr;  // side stream for the overlapped host->device query copy
  cudaEvent_t copy_ready = nullptr, copy_done = nullptr;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> prof_events;
  size_t prof_used = 0;
  int profiling = 0;  // 0 off, 1 tile sweeps, 2 sampling gathers (ProfScope kinds)
  double last_flops = 0, last_bytes = 0;
  int64_t launches = 0;
  // k-NN diagnostics (DK_KNN_STATS=1 in the environment): candidates per query, fallbacks
  dk::KnnClusters* kc = nullptr;  // pruned k-NN (built on the first large k-NN call)
  bool kc_failed = false;          // the cluster build did not fit in device memory: unpruned sweeps
  bool knn_stats = false;
  int64_t knn_queries = 0, knn_cand_sum = 0, knn_cand_max = 0, knn_fallbacks = 0;
  int64_t hyb_queries = 0, hyb_fallbacks = 0;  // two-precision exact KDE: queries served / recomputed in split3
};

namespace dk {

// ---- launchers (prep.cu / tile.cu / sample.cu / l1.cu / knn.cu) ----------
struct QueryOperand {
  int32_t nq = 0, nq_pad = 0;
  __half* A = nullptr;        // [nq_pad][Kp]
  float* qn = nullptr;        // [nq_pad]
  float* m2s = nullptr;       // device scalar
  bool aug = false;           // A carries the query-norm columns (KDE: the MMA yields -d2/2)
  __half* T = nullptr;        // [nq_pad][kTailK] query tail (the encoding has a tail)
  CUtensorMap tmap;
  CUtensorMap tmap_t;
};

CUtensorMap make_tmap_2d_f16(const void* base, uint64_t rows, uint64_t kp, uint32_t box_rows);
// rows x kTailK halves, boxes of box_rows x 16 with 32-byte swizzle (the norm-column tail)
CUtensorMap make_tmap_tail_f16(const void* base, uint64_t rows, uint32_t box_rows);

// dataset prep
void launch_row_stats(const float* X, int64_t n, int32_t d, double* xn64, uint32_t* flags, cudaStream_t s);
void launch_column_mean(const float* X, int64_t n, int32_t d, double* partial, int32_t row_blocks, double* mu,
                        cudaStream_t s);
void launch_encode_rows(const float* X, int64_t n, int64_t n_pad, int32_t d, int mode, const double* mu,
                        int32_t Kp, __half* B, float* xn, float* scale, uint32_t* maxabs_bits, cudaStream_t s,
                        __half* tail = nullptr);
// queries
void launch_query_check(const double* Q, int64_t nq, int32_t d, uint32_t* flags, cudaStream_t s);
// check_flags (mode 0 only, nullable): also OR query_check's exact-mode flags into *check_flags
// aug (exact / fp16 modes): write the query-norm columns (the KDE sweeps; k-NN leaves them zero)
void launch_encode_queries(const double* Q, int64_t nq, int32_t nq_pad, int32_t d, int mode, const double* mu,
                           int32_t Kp, const float* sx, __half* A, float* qn, float* m2s, uint32_t* maxabs_bits,
                           cudaStream_t s, uint32_t* check_flags = nullptr, bool aug = false,
                           __half* tail = nullptr);
void launch_reduce_partials(const double* part, int32_t nparts, int32_t nq_pad, int64_t nq, double scale,
                            double* out, cudaStream_t s);

// tcgen05 tile sweep
struct SweepArgs {
  int mode;                   // TileMode
  const QueryOperand* qop;
  const Encoding* enc;
  int64_t n, n_pad;
  int32_t tile_stride;        // 1 = all tiles
  float negc;
  double* part;               // out partials (KDE)
  int32_t* ncc_out;           // number of column chunks used (KDE)
  float* tmin;                // TILEMIN output
  const float* tau;
  uint32_t* cand_cnt;
  unsigned long long* cand;
  int32_t cap;
  int32_t seg_tiles;          // TILEMIN: tiles per segment
  const uint32_t* guard;      // optional device flags: skip the sweep if (*guard & 6) (see TileParams)
  // tile-list mode (FILTER over pruned lists): unit u = (query block ulist[3u], list positions
  // [ulist[3u+1], ulist[3u+2])) of the flat tile list tlist
  const int32_t* ulist;
  const int32_t* tlist;
  int32_t nunits_list;
  const int32_t* nunits_dev;  // unit count in device memory (built on the device); overrides nunits_list
  int32_t list_stride;        // TILEMIN over tile lists: entries per query block in tlist (segment = list position)
  // MODE_HIST (threshold refinement): per-row bin range and the [nq_pad][64] counts
  const float* hlo;
  const float* hinv;
  const float* htop;
  uint32_t* hist;
  // tile-major FILTER: unit u = (dataset tile ulist[3u], query blocks blist[ulist[3u+1] .. ulist[3u+2]))
  int32_t tmajor;
  const int32_t* blist;
  int32_t* unit_counter;  // tile-major: dynamic unit claims (zeroed by the caller)
  // two-precision exact KDE (MODE_KDE_COLD / MODE_KDE_HOT): [nqb][ntiles][8] hot lane masks
  uint32_t* hot_bits;
  float hot_thr;
};
// tile-major FILTER fits when the resident dataset tile (kblocks x 32 KB) leaves a >= 3-stage ring
bool tile_major_fits(int32_t Kp);
// doubles needed for KDE partials (allow_pair = false: sweeps that never run as 2-CTA pairs)
size_t sweep_part_count(int64_t n_pad, int32_t nq_pad, int num_sms, bool allow_pair = true);
// >= sweep_part_count for every query padding up to max_pad (no plan search)
size_t sweep_part_bound(int64_t n_pad, int32_t max_pad, int num_sms);
void launch_sweep(const SweepArgs& a, int num_sms, cudaStream_t s);
void set_pair_enabled(bool on);  // 2-CTA (cta_group::2) sweeps; off by default (DK_PAIR=1)

// exact-KDE guard (redo.cu): per-query thresholds / flags, and the fp64 recomputation of flagged queries
constexpr int32_t kRedoChunks = 64;  // row chunks per listed query (partials: [nq][kRedoChunks])
void launch_guard_tau(const float* qn, int32_t nq_pad, int64_t nq, float xn_max, double delta_rel, double tol,
                      double h, bool gaussian, float* tau, uint32_t* flag, cudaStream_t s);
void launch_guard_flag_raw(const double* Q, const double* mu, int32_t d, int64_t nq, float xn_max, double delta_rel,
                           double lim, uint32_t* flag, cudaStream_t s);
// flag may be nullptr; rows whose value in `out` is under `under` are recomputed too (fp32 underflow)
void launch_kde_redo(const float* X, int64_t n, int32_t d, const double* Q, int64_t nq, int32_t family, double h,
                     const uint32_t* flag, double under, int32_t* list, int32_t* count, double* part, double scale,
                     double* out, int num_sms, cudaStream_t s);

// two-precision exact gaussian KDE (hybrid.cu)
constexpr int32_t kHotUnitsPerBlock = 16;  // split3 work units per query block (partials: [units][4][128])
void launch_hot_lists(const uint32_t* bits, int32_t nqb, int32_t ntiles, int32_t* tlist, int32_t* tcount,
                      cudaStream_t s);
void launch_hot_units(const int32_t* tcount, int32_t nqb, int32_t ntiles, int32_t* ubeg, int32_t* ucnt,
                      int32_t* scal, int32_t* ulist, cudaStream_t s);
void launch_hyb_combine(const double* part_cold, int32_t nparts, int32_t nq_pad, int64_t bn, const double* part_hot,
                        const int32_t* ubeg, const int32_t* ucnt, const float* qn, float eps_rel, float xn_max,
                        double inv2h2, double tol, double scale, const int32_t* qperm, int64_t qbase, double* out,
                        int32_t* fail, int32_t* nfail, double* bound_out, cudaStream_t s);
void launch_scatter_f64(const double* v, const int32_t* idx, int64_t n, double* out, cudaStream_t s);

// L1 / laplacian exact KDE on CUDA cores
size_t l1_part_count(int64_t n, int32_t nq);
int32_t l1_nq_pad(int64_t nq);  // row stride of the L1 partials
void launch_l1_kde(const float* X, int64_t n, int32_t d, const double* Q, int64_t nq, double inv_h, double* part,
                   int32_t* nparts, float* q32, cudaStream_t s);

// sampling / explicit rows (fp64 direct difference)
void launch_sample(const float* X, int64_t n_local, int64_t global_offset, int64_t global_n, int32_t d,
                   const double* Q, int64_t nq, int32_t family, double bandwidth, int32_t m, uint64_t seed,
                   int64_t query_base, const int64_t* excl_sorted, const int32_t* excl_cnt, int32_t excl_stride,
                   double* z_sum, int64_t* acc_idx, int64_t* draws, cudaStream_t s);
void launch_sort_excl(const int64_t* excl, const int32_t* excl_cnt, int32_t stride, int64_t nq, int64_t* sorted,
                      cudaStream_t s);
void launch_eval_rows(const float* X, int64_t n_local, int64_t global_offset, int32_t d, const double* Q, int64_t nq,
                      int32_t family, double bandwidth, const int64_t* rows, const int32_t* cnt, int32_t stride,
                      double* out, cudaStream_t s);

// pruned k-NN (ivf.cu / knn.cu)
void build_knn_clusters(dk_dataset* h, int32_t C, int32_t iters, KnnClusters& kc, cudaStream_t s);
void free_knn_clusters(KnnClusters& kc);
// dq[j][c] = |q_j - cent_c| (fp64 direct difference), nearest[j] = argmin_c dq[j][c]
void launch_query_cluster_dist(const double* Q, int64_t nq, int32_t d, const double* cent, int32_t C, double* dq,
                               int32_t* nearest, cudaStream_t s);
// nearest[j] = argmin_c |q_j - cent_c| in fp32 (ordering heuristic; best: nq scratch keys)
void launch_nearest_ball_f32(const double* Q, int64_t nq, int32_t d, const double* cent, int32_t C,
                             unsigned long long* best, int32_t* nearest, cudaStream_t s);
// per block of 128 permuted queries: the tiles whose clusters can hold a row with approx d2 <= tau_q
void launch_block_tile_lists(const double* dq, int32_t C, const int32_t* qperm, int64_t bn, int32_t nqb,
                             const float* tau, const float* qn, float xn_max, float eps_rel, const double* rad,
                             const int32_t* tclo, const int32_t* tchi, int32_t ntiles, int32_t* tlist,
                             int32_t* tcount, uint32_t* bits, cudaStream_t s);
// stable sort of the batch by nearest ball (CUB radix sort): qperm[i] = batch position of the
// i-th query in ball order
size_t ball_sort_temp_bytes(int64_t nq);
void launch_sort_queries_by_ball(const int32_t* nearest, int64_t nq, int32_t C, int32_t* nearest_sorted,
                                 int32_t* iota, int32_t* qperm, void* temp, size_t temp_bytes, cudaStream_t s);
// FILTER work units built on the device (scal[0] = unit count, [1] = swept (block, tile) pairs)
void launch_tile_units(const uint32_t* bits, int32_t nqb, int32_t ntiles, int32_t slots, int32_t* tcnt,
                       int32_t* tstart, int32_t* ustart, int32_t* scal, int32_t* blist, int32_t* ulist,
                       int64_t ucap, cudaStream_t s);
void launch_block_units(const int32_t* tcount, int32_t nqb, int32_t list_stride, int32_t slots, int32_t* bstart,
                        int32_t* ustart, int32_t* scal, int32_t* ulist, int64_t ucap, cudaStream_t s);
// per block of 128 ball-sorted queries: the threshold sweep's tiles — every S-th tile of the
// sorted rows (>= k/4 disjoint 64-column segments for every block) plus up to hmax tiles of
// the balls nearest to the block's queries, each extended by its nearest neighbour balls until
// rows_need rows surround it (tight bound); lists [nqb][lmax], lcnt [nqb]
void launch_home_tile_lists(const int32_t* near_sorted, const int32_t* ball_nbr, int64_t bn, int32_t nqb,
                            const int64_t* ball_off, int32_t ntiles, int32_t S, int64_t rows_need, int32_t hmax,
                            int32_t lmax, int32_t* lists, int32_t* lcnt, cudaStream_t s);
// nbr[c][0..kBallNbrs) = the nearest other balls of ball c ((distance, id) order) from dq [C][C]
void launch_ball_neighbors(const double* dq, int32_t C, int32_t* nbr, cudaStream_t s);
void launch_gather_rows_f64(const double* Q, const int32_t* perm, int64_t nq, int32_t d, double* out, cudaStream_t s);
void launch_scatter_knn(const int64_t* idx_p, const double* d2_p, const int32_t* perm, int64_t nq, int32_t k,
                        int64_t* idx_out, double* d2_out, cudaStream_t s);

// k-NN selection
// block_entries (nullable): per block of 128 queries, the entries of its listed threshold sweep;
// only their segments_per x entries segments are read (the rest of tmin is never written)
void launch_tau_from_tmin(const float* tmin, int32_t nseg, int32_t nq_pad, int64_t nq, int32_t k, const float* qn,
                          float xn_max, float eps_rel, float* tau, cudaStream_t s,
                          const int32_t* block_entries = nullptr, int32_t segs_per = 0, float* hlo = nullptr,
                          float* hinv = nullptr, float* htop = nullptr);
// threshold refinement from the MODE_HIST counts: tau_q = min(tau_q, tau_h_q, upper edge of the
// first bin where the cumulative count reaches k + 2 eps_q)
void launch_tau_from_hist(const uint32_t* hist, const float* hlo, const float* hinv, const float* htop,
                          const float* tau_h, int64_t nq, int32_t k, const float* qn, float xn_max, float eps_rel,
                          float* tau, cudaStream_t s);
void launch_fill_float(float* p, int64_t count, float v, cudaStream_t s);
// selection: fast path for every query, sorted-rounds kernel over the device list of queries
// the fast path could not finish; queries with overflowing or too-short candidate lists are
// appended to the overflow list (lists + nq, counts[1]) for launch_exact_knn_fallback
void launch_select(const float* X, int64_t global_offset, int32_t d, const double* Q, int64_t nq, int32_t k,
                   const unsigned long long* cand, const uint32_t* cand_cnt, int32_t cap, const float* qn,
                   float xn_max, float eps_rel, int64_t* idx_out, double* d2_out, int32_t* lists, int32_t* counts,
                   int num_sms, cudaStream_t s, const int64_t* perm = nullptr);
void launch_exact_knn_fallback(const float* X, int64_t n_local, int64_t global_offset, int32_t d, const double* Q,
                               const int32_t* qlist, const int32_t* qcount, int32_t k, int64_t* idx_out,
                               double* d2_out, int num_sms, cudaStream_t s, void* tmp = nullptr,
                               size_t tmp_bytes = 0);  // tmp: scratch for row slices (>= 65,536 k bytes to use them)
void launch_merge_topk(int32_t parts, int64_t nq, int32_t k, const int64_t* idx_in, const double* d2_in,
                       int64_t* idx_out, double* d2_out, cudaStream_t s);
void launch_kernel_values(int32_t family, double h, const double* dist, int64_t count, double* out, uint32_t* bad,
                          cudaStream_t s);
// bigk.cu: exact k-NN for k > kSelectMaxK and CUB sorts of lists longer than kSmemSortMax
constexpr int32_t kSelectMaxK = 4096;
constexpr int32_t kSmemSortMax = 16384;
size_t bigk_temp_bytes(int64_t n);
void launch_knn_bigk(const float* X, int64_t n, int64_t offset, int32_t d, const double* Q, int64_t nq, int32_t k,
                     int64_t* idx_out, double* d2_out, void* temp, size_t temp_bytes, cudaStream_t s);
size_t seg_sort_temp_bytes(int32_t stride, int64_t nq);
void launch_seg_sort_i64(const int64_t* in, int64_t* out, const int32_t* cnt, int32_t stride, int64_t nq, void* temp,
                         size_t temp_bytes, cudaStream_t s);
void launch_gather_positions(const int64_t* ids, const int64_t* inverse, int64_t count, int64_t* out, cudaStream_t s);
void launch_rsp_map_sort(const int64_t* excl, int32_t stride, const int64_t* inverse, int64_t nq, int64_t* pos,
                         cudaStream_t s);
void launch_rsp_starts(const int64_t* pos, int32_t cnt, int64_t nq, int64_t n, int64_t m, int64_t cursor_in,
                       bool independent, int64_t* start, int64_t* len, int32_t* taken, int64_t* cursor_out,
                       cudaStream_t s);
void launch_rsp_eval(const float* X, int64_t n, int32_t d, const double* Q, int64_t nq, int32_t family,
                     double bandwidth, const int64_t* pos, int32_t cnt, const int64_t* start, const int64_t* len,
                     double* z_sum, cudaStream_t s);
void launch_deann_combine(int64_t nq, int32_t family, double bandwidth, int32_t k, int32_t m, int64_t n_total,
                          const double* nbr_d2, const double* z1_l1_sum, const double* z2_sum, double* value,
                          cudaStream_t s, const int32_t* khat = nullptr);

}  // namespace dk
