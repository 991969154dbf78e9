// capi.cu — the extern "C" boundary (include/deann_b200.h).
//
// Host orchestration of the device kernels: argument validation with the
// reference's preconditions, host<->device staging, per-handle workspace,
// operand-encoding choice, k-NN batching/certificates and profiling events.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <exception>
#include <limits>
#include <memory>
#include <mutex>
#include <thread>

#include <errno.h>
#include <fcntl.h>
#include <sys/stat.h>
#include <unistd.h>

#include <map>
#include <tuple>
#include <mutex>

#include "internal.h"
#include "tile_kernel.cuh"

namespace dk {

std::atomic<long long> g_launches{0};
static thread_local std::string g_err;
void set_error(const std::string& m) { g_err = m; }

void Workspace::reserve(size_t bytes) {
  off = 0;
  if (bytes <= cap) return;
  if (base) {
    DK_CUDA(cudaDeviceSynchronize());
    DK_CUDA(cudaFree(base));
    base = nullptr;
    cap = 0;
  }
  const size_t want = std::max(bytes + bytes / 4, size_t(64) << 20);
  DK_CUDA(cudaMalloc(&base, want));
  cap = want;
}
Workspace::~Workspace() {
  if (base) cudaFree(base);
}

namespace {

struct Plan {
  size_t off = 0;
  template <class T>
  size_t add(size_t count) {
    const size_t a = (off + 255) & ~size_t(255);
    off = a + std::max<size_t>(count, 1) * sizeof(T);
    return a;
  }
};
template <class T>
T* at(Workspace& ws, size_t o) {
  return reinterpret_cast<T*>(ws.base + o);
}



constexpr int64_t round_up(int64_t v, int64_t m) { return (v + m - 1) / m * m; }
// query rows padded to whole 128-row blocks, and to an even block count beyond one block so the
// tile sweep can run as 2-CTA pairs (cta_group::2, M = 256)
constexpr int64_t query_pad(int64_t nq) { return nq <= kBM ? kBM : round_up(nq, 2 * kBM); }

void check_family_bw(int32_t family, double bw) {
  DK_REQUIRE(family == DK_GAUSSIAN || family == DK_EXPONENTIAL || family == DK_LAPLACIAN,
             "unknown kernel family " + std::to_string(family));
  DK_REQUIRE(std::isfinite(bw) && bw > 0.0, "bandwidth must be positive and finite, got " + std::to_string(bw));
}


// ------------------------------------------------------------------ encodings
Encoding& enc_slot(dk_dataset* h, int mode) {
  return mode == 0 ? h->enc_exact : (mode == 1 ? h->enc_split : h->enc_fp16);
}

void ensure_mu(dk_dataset* h, cudaStream_t s) {
  if (h->mu) return;
  DK_CUDA(cudaMalloc(&h->mu, size_t(h->d) * sizeof(double)));
  const int32_t row_blocks = int32_t(std::min<int64_t>(1024, h->n));
  double* partial = nullptr;
  DK_CUDA(cudaMalloc(&partial, size_t(row_blocks) * h->d * sizeof(double)));
  launch_column_mean(h->X, h->n, h->d, partial, row_blocks, h->mu, s);
  DK_CUDA(cudaStreamSynchronize(s));
  DK_CUDA(cudaFree(partial));
}

const Encoding& ensure_encoding(dk_dataset* h, int mode, cudaStream_t s) {
  Encoding& e = enc_slot(h, mode);
  if (e.mode == mode) return e;
  const int32_t d = h->d;
  e.Kp = enc_kp(d, mode);
  e.d = d;
  if (mode != 0) ensure_mu(h, s);
  e.mu = mode == 0 ? nullptr : h->mu;
  DK_CUDA(cudaMalloc(&e.B, size_t(h->n_pad) * e.Kp * sizeof(__half)));
  DK_CUDA(cudaMalloc(&e.xn, size_t(h->n_pad) * sizeof(float)));
  DK_CUDA(cudaMalloc(&e.sx, 2 * sizeof(float)));
  if (enc_aug_tail(d, mode)) DK_CUDA(cudaMalloc(&e.T, size_t(h->n_pad) * kTailK * sizeof(__half)));
  uint32_t* maxabs = reinterpret_cast<uint32_t*>(e.sx + 1);
  launch_encode_rows(h->X, h->n, h->n_pad, d, mode, e.mu, e.Kp, e.B, e.xn, e.sx, maxabs, s, e.T);
  std::vector<float> xn(static_cast<size_t>(h->n));
  DK_CUDA(cudaMemcpyAsync(xn.data(), e.xn, xn.size() * sizeof(float), cudaMemcpyDeviceToHost, s));
  DK_CUDA(cudaStreamSynchronize(s));
  float mx = 0.f;
  for (float v : xn) mx = std::max(mx, v);
  e.xn_max = mx;
  const double u = std::ldexp(1.0, -24);
  // |approx d2 - d2| <= eps_rel * (|q|^2 + max|x|^2): operand rounding (2u_op |q||x|, u_op the
  // unit roundoff of the encoding), fp32 accumulation over Kp terms, fp32 epilogue (norm
  // rounding, the add and the fma), using 2|q||x| <= |q|^2 + |x|^2.
  if (mode == 0) e.eps_rel = 0.f;                                                        // exact integers
  else if (mode == 1) e.eps_rel = float(1.01 * (4.0 * std::ldexp(1.0, -22) + double(e.Kp + 4) * u));  // split3
  // fp16: + 2^-20 for the norm columns' residual and subnormal operands (values < 2^-14 of 2^8)
  else e.eps_rel = float(1.01 * (2.002 * std::ldexp(1.0, -11) + double(e.Kp + 4) * u + std::ldexp(1.0, -20)));
  e.tmap = make_tmap_2d_f16(e.B, uint64_t(h->n_pad), uint64_t(e.Kp), uint32_t(kBN));
  e.tmap_half = make_tmap_2d_f16(e.B, uint64_t(h->n_pad), uint64_t(e.Kp), uint32_t(kBN / 2));
  if (e.T) e.tmap_t = make_tmap_tail_f16(e.T, uint64_t(h->n_pad), uint32_t(kBN));
  e.mode = mode;
  return e;
}

void free_encoding(Encoding& e) {
  if (e.B) cudaFree(e.B);
  if (e.T) cudaFree(e.T);
  if (e.xn) cudaFree(e.xn);
  if (e.sx) cudaFree(e.sx);
  e = Encoding{};
}

// ------------------------------------------------------------------ query staging
struct Staged {
  const double* Q = nullptr;  // device fp64 queries
};

const double* stage_queries(dk_dataset* h, const double* Q, int64_t nq, size_t off, cudaStream_t s) {
  if (is_device_ptr(Q)) return Q;
  double* dst = at<double>(h->ws, off);
  DK_CUDA(cudaMemcpyAsync(dst, Q, size_t(nq) * h->d * sizeof(double), cudaMemcpyHostToDevice, s));
  return dst;
}

// choose the encoding for this query batch (may synchronise for the integrality check)
int choose_mode(dk_dataset* h, const double* Qd, int64_t nq, uint32_t* flags, cudaStream_t s) {
  if (h->precision == DK_PREC_SPLIT3) return 1;
  if (h->precision == DK_PREC_FP16) return 2;
  if (!h->int_exact) return 1;
  DK_CUDA(cudaMemsetAsync(flags, 0, sizeof(uint32_t), s));
  launch_query_check(Qd, nq, h->d, flags, s);
  uint32_t f = 0;
  DK_CUDA(cudaMemcpyAsync(&f, flags, sizeof(uint32_t), cudaMemcpyDeviceToHost, s));
  DK_CUDA(cudaStreamSynchronize(s));
  DK_REQUIRE(!(f & 1u), "queries must be finite");
  return (f & 6u) ? 1 : 0;
}

// aug: the KDE sweeps' query-norm columns (in A when they fit its padding, else in `tail`,
// kTailK halves per padded row, when the encoding has a tail and the caller passes the buffer)
QueryOperand encode_queries(dk_dataset* h, const Encoding& e, const double* Qd, int64_t nq, int32_t nq_pad,
                            __half* A, float* qn, float* scal, cudaStream_t s, uint32_t* check_flags = nullptr,
                            bool aug = false, __half* tail = nullptr) {
  QueryOperand q;
  const bool use_tail = aug && e.T != nullptr && tail != nullptr;
  q.aug = aug && (enc_aug_main(h->d, e.mode) || use_tail);
  q.T = use_tail ? tail : nullptr;
  q.nq = int32_t(nq);
  q.nq_pad = nq_pad;
  q.A = A;
  q.qn = qn;
  q.m2s = scal;
  launch_encode_queries(Qd, nq, nq_pad, h->d, e.mode, e.mu, e.Kp, e.sx, A, qn, scal,
                        reinterpret_cast<uint32_t*>(scal + 1), s, check_flags, q.aug, q.T);
  q.tmap = make_tmap_2d_f16(A, uint64_t(nq_pad), uint64_t(e.Kp), uint32_t(kBM));
  if (q.T) q.tmap_t = make_tmap_tail_f16(q.T, uint64_t(nq_pad), uint32_t(kBM));
  return q;
}

void copy_out(void* dst, const void* src, size_t bytes, cudaStream_t s) {
  if (dst == src || bytes == 0) return;
  DK_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, s));
}

struct ProfScope {
  dk_dataset* h;
  cudaStream_t s;
  cudaEvent_t e1 = nullptr;
  // kind: 1 = tile sweep (the KDE / k-NN distance tiles), 2 = sampling gather; dk_set_profiling
  // picks which kind is timed
  ProfScope(dk_dataset* hh, cudaStream_t ss, double flops, double bytes, int kind) : h(hh), s(ss) {
    if (h->profiling != kind) return;
    if (h->prof_used == h->prof_events.size()) {
      cudaEvent_t a, b;
      DK_CUDA(cudaEventCreate(&a));
      DK_CUDA(cudaEventCreate(&b));
      h->prof_events.emplace_back(a, b);
    }
    auto& pr = h->prof_events[h->prof_used++];
    DK_CUDA(cudaEventRecord(pr.first, s));
    e1 = pr.second;
    h->last_flops = flops;
    h->last_bytes = bytes;
  }
  ~ProfScope() {
    if (e1) cudaEventRecord(e1, s);
  }
};

struct LaunchCount {
  dk_dataset* h;
  long long start;
  explicit LaunchCount(dk_dataset* hh) : h(hh), start(g_launches.load()) {}
  ~LaunchCount() { h->launches = g_launches.load() - start; }
};

// ------------------------------------------------------------------ k-NN core
constexpr int32_t kKnnCap = 8192;  // candidates per query before the exact-scan fallback

struct KnnPlan {
  int32_t seg_tiles = 1, nseg = 0, cap = 0, batch = 0;
  int32_t stride = 1;  // TILEMIN visits every stride-th dataset tile
  bool tau_inf = false;
};

// The threshold sweep only needs SOME k disjoint point sets whose minima bound the
// k-th distance: the k-th smallest segment minimum over any subset of the rows is
// >= the k-th smallest distance over all rows.  Sweeping every stride-th tile cuts
// that pass to 1/stride of the tensor work; the looser tau admits ~stride x more
// candidates to the FILTER pass, whose cost barely depends on the count.
int32_t knn_stride(int64_t ntiles, int64_t target) {
  static const int env = [] {
    const char* v = std::getenv("DK_KNN_STRIDE");  // A/B switch
    return v ? std::max(1, std::atoi(v)) : 0;
  }();
  // up to every 8th tile: with the pruned tile-major FILTER a looser tau costs less than the
  // threshold sweep it saves (c3 k-NN: stride 4 2.08 ms, 6 1.93, 8 1.85; round 1, before
  // pruning, stride 4 was best)
  const int64_t auto_s = std::clamp<int64_t>(ntiles / target, 1, 8);
  const int64_t s = env ? env : auto_s;
  return int32_t(std::max<int64_t>(1, std::min<int64_t>(s, ntiles / target)));
}

KnnPlan plan_knn(const dk_dataset* h, int32_t k, int64_t nq) {
  KnnPlan p;
  const int64_t ntiles = h->n_pad / kBN;
  const int64_t target = std::clamp<int64_t>(4 * int64_t(k), 256, 2048);  // ~4k segments: tight tau
  if (h->n <= kKnnCap) {
    p.tau_inf = true;  // every row is a candidate
    p.cap = int32_t(h->n);
  } else if (ntiles >= target) {
    p.stride = knn_stride(ntiles, target);
    const int64_t nvis = (ntiles + p.stride - 1) / p.stride;
    p.seg_tiles = int32_t((nvis + target - 1) / target);
    p.nseg = int32_t((nvis + p.seg_tiles - 1) / p.seg_tiles);
    p.cap = kKnnCap;
  } else {  // one segment per 64-column group of every tile
    p.seg_tiles = 0;
    p.nseg = int32_t(ntiles * kColGroups);
    p.cap = kKnnCap;
  }
  if (!p.tau_inf && p.nseg < k) {  // cannot bound the k-th distance: keep every row
    p.tau_inf = true;
    p.seg_tiles = 1;
    p.nseg = 0;
    p.cap = int32_t(std::min<int64_t>(h->n, int64_t(1) << 20));
  }
  // bytes of candidate storage per batch: a tenth of the device memory free after the fit, within
  // [1, 10] GiB (finish_fit).  Large batches matter: c5's 100,000 queries as one batch instead of
  // seven of 14,286 take 33.8 ms instead of 53.4 (each resident tile of the tile-major FILTER serves
  // every query block that lists it in one pass, the block-major threshold sweeps fill all SMs, and
  // the per-batch launches are paid once)
  int64_t budget = h->knn_budget > 0 ? h->knn_budget : int64_t(1) << 30;
  if (const char* v = std::getenv("DK_KNN_BUDGET_MB")) budget = std::max<int64_t>(64, std::atoll(v)) << 20;  // A/B
  int64_t b = budget / (int64_t(p.cap) * 8 + int64_t(p.nseg) * 4 + 64);
  int64_t bmax = 131072;
  if (const char* v = std::getenv("DK_KNN_MAX_BATCH")) bmax = std::max<int64_t>(2 * kBM, std::atoll(v));  // tests
  b = std::max<int64_t>(2 * kBM, std::min<int64_t>(bmax, b)) / (2 * kBM) * (2 * kBM);
  p.batch = int32_t(std::min<int64_t>(b, query_pad(nq)));
  return p;
}

// The tile path's selection keeps the candidate list and 2*pow2(k) keys in one
// CTA's shared memory (knn.cu select_slow_kernel); plans that do not fit —
// k > 4096, or every row a candidate because fewer segment minima than k exist
// to bound tau — take the exact fp64 + radix-sort path instead (bigk.cu).
bool use_bigk(const dk_dataset* h, int32_t k, int64_t nq) {
  if (k > kSelectMaxK) return true;
  const KnnPlan kp = plan_knn(h, k, nq);
  int B = 2, Kp = 32;
  while (B < kp.cap) B <<= 1;
  while (Kp < k) Kp <<= 1;
  return size_t(B) * 8 + size_t(2 * Kp) * 16 + size_t(h->d) * 8 + 4096 > 232448;  // select_slow_kernel's buffer
}

// encoding for the k-NN sweeps: exact integers when possible, else single-pass
// fp16 (its error is bounded by eps_rel and absorbed by the threshold), unless
// the caller pinned split3.
int knn_mode(dk_dataset* h, const double* Qd, int64_t nq, uint32_t* flags, cudaStream_t s) {
  if (h->precision == DK_PREC_SPLIT3) return 1;
  const int m = choose_mode(h, Qd, nq, flags, s);
  return m == 0 ? 0 : 2;
}

// k-NN sweeps with norm columns (single-pass fp16 operands whose K padding holds them): the
// accumulator is -d2/2, within the same eps_q (the bound's 2^-20 term covers the columns' residual).
// DK_KNN_AUG=0: plain operands.
bool knn_aug(const dk_dataset* h, const Encoding& e) {
  static const bool off = [] {
    const char* v = std::getenv("DK_KNN_AUG");  // A/B switch
    return v != nullptr && std::atoi(v) == 0;
  }();
  return !off && e.mode == 2 && enc_aug_main(h->d, e.mode);
}

// Pruned FILTER pass (internal.h KnnClusters): for datasets of >= 512 tiles the rows are
// grouped once by k-means into balls; each block of 128 queries (sorted by their nearest
// ball) then sweeps only the tiles whose balls can hold a row inside some member's tau_q.
// Exact: a tile is skipped only when (|q - c| - r)^2 > tau_q + eps_q for all its balls
// and all queries of the block.  DK_KNN_PRUNE=0 turns it off.
constexpr int64_t kPruneMinTiles = 512;
bool knn_prunable(const dk_dataset* h, const KnnPlan& kp) {
  static const bool off = [] {
    const char* v = std::getenv("DK_KNN_PRUNE");
    return v != nullptr && std::atoi(v) == 0;
  }();
  return !(off || kp.tau_inf || h->kc_failed || h->n_pad / kBN < kPruneMinTiles);
}
int32_t knn_cluster_count(const dk_dataset* h) {
  static const int div = [] {
    const char* v = std::getenv("DK_KNN_TILES_PER_BALL");  // A/B switch
    return v ? std::max(1, std::atoi(v)) : 16;
  }();
  return int32_t(std::clamp<int64_t>(h->n_pad / kBN / div, 16, 4096));
}

// Whether this call prunes (internal.h KnnClusters: the swept fraction of earlier calls,
// read without waiting; unclustered data turns pruning off, re-tested every 32nd call).
bool knn_prune_decide(dk_dataset* h) {
  KnnClusters* kc = h->kc;
  if (kc == nullptr) return true;
  if (kc->stat_pending) {
    const cudaError_t q = cudaEventQuery(kc->stat_ev);
    if (q == cudaSuccess) {
      kc->stat_pending = false;
      const bool wide = double(kc->stat_host[0]) > 0.6 * kc->stat_total;
      kc->over = wide ? kc->over + 1 : 0;
      if (kc->over >= 3) kc->useless = true;
    } else if (q == cudaErrorNotReady) {
      (void)cudaGetLastError();
    } else {
      DK_CUDA(q);
    }
  }
  if (kc->useless) {
    if (++kc->off_calls < 32) return false;
    kc->useless = false;
    kc->over = 0;
    kc->off_calls = 0;
  }
  return true;
}

// Builds the cluster-sorted copy on the first pruned call.  Returns false (and disables
// pruning for the handle) when it does not fit in device memory: the unpruned sweep is exact.
bool ensure_knn_clusters(dk_dataset* h, const Encoding& e, cudaStream_t s) {
  if (h->kc != nullptr && h->kc->enc.mode == e.mode) return true;
  if (h->kc != nullptr) {  // encoding changed (precision pinned differently): rebuild
    free_knn_clusters(*h->kc);
    delete h->kc;
    h->kc = nullptr;
  }
  {  // rows copy + operand + k-means scratch (labels, ids, d2, CUB temp): ~(4d + 2 Kp + 48) B per row
    size_t free_b = 0, total_b = 0;
    DK_CUDA(cudaMemGetInfo(&free_b, &total_b));
    const double need = double(h->n_pad) * (4.0 * h->d + 2.0 * e.Kp + 64.0) * 1.1 + double(64 << 20);
    if (double(free_b) < need) {
      h->kc_failed = true;
      return false;
    }
  }
  std::unique_ptr<KnnClusters> kc(new KnnClusters());
  try {
    build_knn_clusters(h, knn_cluster_count(h), 3, *kc, s);
    {  // nearest neighbour balls of each ball (the threshold sweep's lists)
      double* dcc = nullptr;
      int32_t* tmp = nullptr;
      DK_CUDA(cudaMalloc(&dcc, size_t(kc->C) * kc->C * sizeof(double)));
      DK_CUDA(cudaMalloc(&tmp, size_t(kc->C) * sizeof(int32_t)));
      DK_CUDA(cudaMalloc(&kc->nbr, size_t(kc->C) * kBallNbrs * sizeof(int32_t)));
      launch_query_cluster_dist(kc->cent, kc->C, h->d, kc->cent, kc->C, dcc, tmp, s);
      launch_ball_neighbors(dcc, kc->C, kc->nbr, s);
      DK_CUDA(cudaStreamSynchronize(s));
      cudaFree(dcc);
      cudaFree(tmp);
    }
    Encoding& se = kc->enc;
    se.Kp = e.Kp;
    se.d = e.d;
    se.mu = e.mu;
    DK_CUDA(cudaMalloc(&se.B, size_t(h->n_pad) * se.Kp * sizeof(__half)));
    DK_CUDA(cudaMalloc(&se.xn, size_t(h->n_pad) * sizeof(float)));
    DK_CUDA(cudaMalloc(&se.sx, 2 * sizeof(float)));
    if (e.T) DK_CUDA(cudaMalloc(&se.T, size_t(h->n_pad) * kTailK * sizeof(__half)));
    // same rows, same centring: the power-of-two scale (from the max |value|) equals the k-NN
    // encoding's, so the encoded queries serve both operands
    launch_encode_rows(kc->xs, h->n, h->n_pad, h->d, e.mode, e.mu, se.Kp, se.B, se.xn, se.sx,
                       reinterpret_cast<uint32_t*>(se.sx + 1), s, se.T);
    se.xn_max = e.xn_max;
    se.eps_rel = e.eps_rel;
    se.tmap = make_tmap_2d_f16(se.B, uint64_t(h->n_pad), uint64_t(se.Kp), uint32_t(kBN));
    se.tmap_half = make_tmap_2d_f16(se.B, uint64_t(h->n_pad), uint64_t(se.Kp), uint32_t(kBN / 2));
    if (se.T) se.tmap_t = make_tmap_tail_f16(se.T, uint64_t(h->n_pad), uint32_t(kBN));
    se.mode = e.mode;
    DK_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&kc->stat_host), 4 * sizeof(int32_t), cudaHostAllocDefault));
    DK_CUDA(cudaEventCreateWithFlags(&kc->stat_ev, cudaEventDisableTiming));
    DK_CUDA(cudaStreamSynchronize(s));
  } catch (const Error& err) {
    free_knn_clusters(*kc);
    cudaGetLastError();
    if (err.code != DK_ENOMEM) throw;
    h->kc_failed = true;  // out of memory: exact unpruned sweeps from now on
    return false;
  }
  h->kc = kc.release();
  return true;
}

constexpr int32_t kHomeTiles = 768;  // threshold sweep: at most this many tiles of the block's nearest balls
constexpr int32_t kListSegs = 8;     // listed threshold sweep: 32-column segments per tile

// Device workspace of one k-NN batch (knn_device / knn_ws_bytes share this layout).
struct KnnLayout {
  size_t flags, A, qn, scal, tmin, tau, cnt, cand, lists, ctr;
  // pruned path
  size_t dq, near, near_s, iota, qperm, sort_tmp, qp, tidx, td2, tlist, tcnt, bits, tcnt_t, tstart, ustart, blist,
      ulist, hlist, hcnt, hlo, hinv, htop, hist, tauh;
  int32_t hS = 1, hlmax = 0;  // threshold sweep: stride of the strided tiles, list length per block
  int32_t hneed = 0, hmax = 0;  // near tiles wanted / allowed per block
  size_t sort_tmp_bytes = 0, ulist_ints = 0;
  size_t end = 0;
};

KnnLayout knn_layout(const dk_dataset* h, const KnnPlan& kp, int32_t k, int32_t Kp, bool prune, size_t base) {
  KnnLayout L{};
  Plan pl;
  pl.off = base;
  const int32_t bpad = kp.batch;
  L.flags = pl.add<uint32_t>(4);
  L.A = pl.add<__half>(size_t(bpad) * Kp);
  L.qn = pl.add<float>(bpad);
  L.scal = pl.add<float>(4);
  if (prune) {  // threshold sweep over per-block lists: every hS-th tile + the nearest balls' tiles
    const int32_t ntiles = int32_t(h->n_pad / kBN);
    L.hS = std::max<int32_t>(1, ntiles / ((k + kListSegs - 1) / kListSegs + 16));  // >= k strided segments
    L.hneed = std::max<int32_t>(4, (4 * k + kBN - 1) / kBN);  // tiles' worth of rows around a ball: >= 4k rows
    L.hmax = std::max(kHomeTiles, L.hneed);
    L.hlmax = (ntiles + L.hS - 1) / L.hS + L.hmax;
  }
  L.tmin = pl.add<float>(size_t(std::max({kp.nseg, 1, L.hlmax * kListSegs})) * bpad);
  L.tau = pl.add<float>(bpad);
  L.cnt = pl.add<uint32_t>(bpad);
  L.cand = pl.add<unsigned long long>(size_t(kp.cap) * bpad);
  L.lists = pl.add<int32_t>(size_t(2) * bpad);
  L.ctr = pl.add<int32_t>(16);  // [0] slow, [1] overflow, [4..6] unit plan (count, pairs, U)
  if (prune) {
    const int32_t ntiles = int32_t(h->n_pad / kBN), nqb = bpad / kBM, nwords = (ntiles + 31) / 32;
    const int32_t Cn = knn_cluster_count(h);
    L.dq = pl.add<double>(size_t(bpad) * Cn);
    L.near = pl.add<int32_t>(bpad);
    L.near_s = pl.add<int32_t>(bpad);
    L.iota = pl.add<int32_t>(bpad);
    L.qperm = pl.add<int32_t>(bpad);
    L.sort_tmp_bytes = ball_sort_temp_bytes(bpad);
    L.sort_tmp = pl.add<uint8_t>(L.sort_tmp_bytes);
    L.qp = pl.add<double>(size_t(bpad) * h->d);
    L.tidx = pl.add<int64_t>(size_t(bpad) * k);
    L.td2 = pl.add<double>(size_t(bpad) * k);
    L.tlist = pl.add<int32_t>(size_t(nqb) * ntiles);  // block-major lists, or the tile-major blist
    L.tcnt = pl.add<int32_t>(nqb);
    L.bits = pl.add<uint32_t>(size_t(nqb) * nwords);
    L.tcnt_t = pl.add<int32_t>(ntiles);
    L.tstart = pl.add<int32_t>(std::max(ntiles, nqb));
    L.ustart = pl.add<int32_t>(std::max(ntiles, nqb));
    L.blist = L.tlist;
    // units: tile-major <= ntiles + pairs / 4, block-major <= nqb + pairs / 8 (FILTER and threshold lists)
    L.ulist_ints = size_t(3) * (size_t(std::max(ntiles, nqb)) + size_t(nqb) * std::max(ntiles, L.hlmax) / 4 + 1);
    L.ulist = pl.add<int32_t>(L.ulist_ints);
    L.hlist = pl.add<int32_t>(size_t(nqb) * L.hlmax);
    L.hcnt = pl.add<int32_t>(nqb);
    L.hlo = pl.add<float>(bpad);
    L.hinv = pl.add<float>(bpad);
    L.htop = pl.add<float>(bpad);
    L.hist = pl.add<uint32_t>(size_t(bpad) * kHistBins);
    L.tauh = pl.add<float>(bpad);
  }
  L.end = pl.off;
  return L;
}

// k-NN for nq queries already on the device; idx/d2 outputs on the device.  No host
// synchronisation on the pruned or unpruned tile path (integer datasets wait once for the
// query integrality check): work lists, unit plans and fallbacks live in device memory.
void knn_device(dk_dataset* h, const double* Qd, int64_t nq, int32_t k, int64_t* idx_d, double* d2_d,
                cudaStream_t s, size_t ws_off_base) {
  if (use_bigk(h, k, nq)) {  // exact fp64 distances + stable radix sort (bigk.cu)
    const size_t off = (ws_off_base + 255) & ~size_t(255);
    launch_knn_bigk(h->X, h->n, h->global_offset, h->d, Qd, nq, k, idx_d, d2_d, h->ws.base + off,
                    bigk_temp_bytes(h->n), s);
    return;
  }
  const KnnPlan kp = plan_knn(h, k, nq);
  const bool prunable = knn_prunable(h, kp);
  const KnnLayout L0 = knn_layout(h, kp, k, int32_t(round_up(3 * int64_t(h->d), kBK)), prunable, ws_off_base);
  if (L0.end > h->ws.cap) throw Error{DK_ECUDA, "internal: k-NN workspace under-reserved"};
  const int mode = knn_mode(h, Qd, nq, at<uint32_t>(h->ws, L0.flags), s);
  const Encoding& e = ensure_encoding(h, mode, s);
  bool prune = prunable && knn_prune_decide(h);
  if (prune) prune = ensure_knn_clusters(h, e, s);
  const KnnLayout L = knn_layout(h, kp, k, e.Kp, prunable, ws_off_base);
  const int32_t bpad = kp.batch;
  const int32_t ntiles = int32_t(h->n_pad / kBN);
  static const bool tmajor_off = [] {  // A/B switch: block-major pruned FILTER
    const char* v = std::getenv("DK_KNN_TMAJOR");
    return v != nullptr && std::atoi(v) == 0;
  }();
  const bool tmajor = prune && !tmajor_off && tile_major_fits(e.Kp);
  const float inf = std::numeric_limits<float>::infinity();
  int32_t* ctr = at<int32_t>(h->ws, L.ctr);
  // Threshold for large datasets ("home" mode): a histogram-refined bound from per-block lists
  // of the tiles near the block's balls, combined with a global bound from segment minima over
  // ~4 x target tiles of the original row order (queries far from every ball: small clusters).
  // It replaces the strided sweep over a quarter of the tiles when that global pass is at most
  // 1/8 of the dataset (c5: 8M rows, 5% of the tiles; k-NN 106 -> 77 ms); smaller datasets keep
  // the strided sweep.  DK_KNN_HOME=0/1 forces it (read per call: tests toggle it).
  const char* home_env = std::getenv("DK_KNN_HOME");
  const int64_t home_target = std::clamp<int64_t>(4 * int64_t(k), 256, 2048);
  const bool home_tau = home_env != nullptr ? std::atoi(home_env) != 0 : int64_t(ntiles) >= 32 * home_target;
  // equal batches (a call of 16,384 queries is not 15,872 + 512): a small remainder batch sweeps
  // a large fraction of the tiles (its blocks span many balls) and would skew the pruning statistic
  const int64_t nbatch = (nq + bpad - 1) / bpad;
  const int64_t bstep = std::min<int64_t>(bpad, round_up((nq + nbatch - 1) / nbatch, 2 * kBM));
  for (int64_t b0 = 0; b0 < nq; b0 += bstep) {
    const int64_t bn = std::min<int64_t>(bstep, nq - b0);
    const int32_t bn_pad = int32_t(query_pad(bn));
    const int32_t nqb = bn_pad / kBM;
    const double* Qb = Qd + b0 * h->d;
    int64_t* idx_b = idx_d + b0 * k;
    double* d2_b = d2_d + b0 * k;
    int32_t* qperm = nullptr;
    DK_CUDA(cudaMemsetAsync(ctr, 0, 16 * sizeof(int32_t), s));
    if (prune) {  // order the batch by nearest ball (stable) so each block of 128 queries is local
      int32_t* near = at<int32_t>(h->ws, L.near);
      launch_query_cluster_dist(Qb, bn, h->d, h->kc->cent, h->kc->C, at<double>(h->ws, L.dq), near, s);
      qperm = at<int32_t>(h->ws, L.qperm);
      launch_sort_queries_by_ball(near, bn, h->kc->C, at<int32_t>(h->ws, L.near_s), at<int32_t>(h->ws, L.iota), qperm,
                                  h->ws.base + L.sort_tmp, L.sort_tmp_bytes, s);
      double* Qp = at<double>(h->ws, L.qp);
      launch_gather_rows_f64(Qb, qperm, bn, h->d, Qp, s);
      Qb = Qp;
      idx_b = at<int64_t>(h->ws, L.tidx);
      d2_b = at<double>(h->ws, L.td2);
    }
    // fp16 operands with norm columns in the K padding: the query side carries its norm columns too,
    // so the sweeps' accumulators are -d2/2 and their epilogues skip the norm arithmetic
    QueryOperand q = encode_queries(h, e, Qb, bn, bn_pad, at<__half>(h->ws, L.A), at<float>(h->ws, L.qn),
                                    at<float>(h->ws, L.scal), s, nullptr, knn_aug(h, e));
    float* tau = at<float>(h->ws, L.tau);
    uint32_t* cnt = at<uint32_t>(h->ws, L.cnt);
    unsigned long long* cand = at<unsigned long long>(h->ws, L.cand);
    if (kp.tau_inf) {
      launch_fill_float(tau, bn, inf, s);
    } else if (prune && home_tau) {
      // (a) a global bound, valid for every query however far it is from its balls: segment
      // minima over every stride_g-th tile of the ORIGINAL row order (random rows: the k-th
      // smallest segment minimum tracks a few-hundredth-neighbour distance), at 4x the stride of
      // the plain threshold sweep
      {
        const int64_t target = std::clamp<int64_t>(4 * int64_t(k), 256, 2048);
        const char* gs_env = std::getenv("DK_KNN_GTILES");  // A/B: tiles the global pass visits
        const int64_t gtiles = gs_env ? std::max<int64_t>(target, std::atoll(gs_env)) : 4 * target;
        const int32_t sg = int32_t(std::clamp<int64_t>(ntiles / gtiles, 1, std::max<int64_t>(1, ntiles / target)));
        const int64_t nvis = (ntiles + sg - 1) / sg;
        const int32_t seg_tiles = int32_t((nvis + target - 1) / target);
        const int32_t nseg_g = int32_t((nvis + seg_tiles - 1) / seg_tiles);
        float* tmin = at<float>(h->ws, L.tmin);
        launch_fill_float(tmin, int64_t(nseg_g) * bn_pad, inf, s);
        SweepArgs a{};
        a.mode = MODE_TILEMIN;
        a.qop = &q;
        a.enc = &e;
        a.n = h->n;
        a.n_pad = h->n_pad;
        a.tile_stride = sg;
        a.seg_tiles = seg_tiles;
        a.tmin = tmin;
        launch_sweep(a, h->num_sms, s);
        // the global pass also sets each query's histogram range for (b): [min, k-th] of its
        // segment minima
        launch_tau_from_tmin(tmin, nseg_g, bn_pad, bn, k, q.qn, e.xn_max, e.eps_rel, tau, s, nullptr, 0,
                             at<float>(h->ws, L.hlo), at<float>(h->ws, L.hinv), at<float>(h->ws, L.htop));
      }
      // (b) threshold from the block's own neighbourhood: per block of 128 ball-sorted queries a
      // list of tiles — every hS-th tile and the tiles of the balls nearest to the block's
      // queries and their neighbour balls (tens to hundreds of tiles instead of a quarter of the
      // dataset) — swept once in MODE_HIST: each query's approx d2 of the listed rows counted
      // into 64 quadratic bins over the range of (a); the bin where the count reaches k bounds
      // the k-th distance (k distinct rows below its edge).  Segment minima of the same lists
      // sit far above the k-th distance in high dimension (c5), the row histogram does not.
      int32_t* hl = at<int32_t>(h->ws, L.hlist);
      int32_t* hc = at<int32_t>(h->ws, L.hcnt);
      int32_t* hplan = ctr + 8;  // [0] units, [1] listed (block, tile) pairs, [2] U
      launch_home_tile_lists(at<int32_t>(h->ws, L.near_s), h->kc->nbr, bn, nqb, h->kc->off, ntiles, L.hS,
                             int64_t(L.hneed) * kBN, L.hmax, L.hlmax, hl, hc, s);
      launch_block_units(hc, nqb, L.hlmax, h->num_sms, at<int32_t>(h->ws, L.tstart), at<int32_t>(h->ws, L.ustart),
                         hplan, at<int32_t>(h->ws, L.ulist), int64_t(L.ulist_ints / 3), s);
      float* hlo = at<float>(h->ws, L.hlo);
      float* hinv = at<float>(h->ws, L.hinv);
      float* htop = at<float>(h->ws, L.htop);
      uint32_t* hist = at<uint32_t>(h->ws, L.hist);
      float* tau_h = tau;  // the histogram bound tightens the global one
      DK_CUDA(cudaMemsetAsync(hist, 0, size_t(bn) * kHistBins * sizeof(uint32_t), s));
      {
        SweepArgs b{};
        b.mode = MODE_HIST;
        b.qop = &q;
        b.enc = &h->kc->enc;
        b.n = h->n;
        b.n_pad = h->n_pad;
        b.tile_stride = 1;
        b.ulist = at<int32_t>(h->ws, L.ulist);
        b.tlist = hl;
        b.nunits_dev = hplan;
        b.list_stride = L.hlmax;
        b.hlo = hlo;
        b.hinv = hinv;
        b.htop = htop;
        b.hist = hist;
        launch_sweep(b, h->num_sms, s);
      }
      launch_tau_from_hist(hist, hlo, hinv, htop, tau_h, bn, k, q.qn, e.xn_max, e.eps_rel, tau, s);
      if (std::getenv("DK_KNN_DEBUG")) {  // diagnostics: threshold quantiles and list lengths
        std::vector<float> ta(static_cast<size_t>(bn));
        std::vector<int32_t> lc(static_cast<size_t>(nqb)), ns(static_cast<size_t>(bn));
        DK_CUDA(cudaMemcpyAsync(ta.data(), tau, ta.size() * 4, cudaMemcpyDeviceToHost, s));
        DK_CUDA(cudaMemcpyAsync(lc.data(), hc, lc.size() * 4, cudaMemcpyDeviceToHost, s));
        DK_CUDA(cudaMemcpyAsync(ns.data(), at<int32_t>(h->ws, L.near_s), ns.size() * 4, cudaMemcpyDeviceToHost, s));
        DK_CUDA(cudaStreamSynchronize(s));
        std::vector<float> st = ta;
        std::sort(st.begin(), st.end());
        const int w = int(std::max_element(ta.begin(), ta.end()) - ta.begin());
        int distinct = 0;
        for (int r = (w / 128) * 128; r < std::min<int>(int(bn), (w / 128) * 128 + 128); ++r)
          distinct += (r == (w / 128) * 128 || ns[size_t(r)] != ns[size_t(r) - 1]) ? 1 : 0;
        std::fprintf(stderr, "[dk] tau p0 %g p50 %g p90 %g p99 %g max %g | worst row %d block %d list %d of max %d, "
                     "%d balls | list p50 %d max %d\n", st.front(), st[st.size() / 2], st[st.size() * 9 / 10],
                     st[st.size() * 99 / 100], st.back(), w, w / 128, lc[size_t(w / 128)], L.hlmax, distinct,
                     [&] { auto c = lc; std::sort(c.begin(), c.end()); return c[c.size() / 2]; }(),
                     *std::max_element(lc.begin(), lc.end()));
      }
    } else {
      float* tmin = at<float>(h->ws, L.tmin);
      launch_fill_float(tmin, int64_t(kp.nseg) * bn_pad, inf, s);
      SweepArgs a{};
      a.mode = MODE_TILEMIN;
      a.qop = &q;
      a.enc = &e;
      a.n = h->n;
      a.n_pad = h->n_pad;
      a.tile_stride = kp.stride;
      a.seg_tiles = kp.seg_tiles;
      a.tmin = tmin;
      launch_sweep(a, h->num_sms, s);
      launch_tau_from_tmin(tmin, kp.nseg, bn_pad, bn, k, q.qn, e.xn_max, e.eps_rel, tau, s);
    }
    launch_fill_float(tau + bn, bn_pad - bn, -inf, s);
    DK_CUDA(cudaMemsetAsync(cnt, 0, size_t(bn_pad) * sizeof(uint32_t), s));
    int32_t* uplan = ctr + 4;  // [0] units, [1] swept (block, tile) pairs, [2] U
    if (prune) {
      int32_t* tlist = at<int32_t>(h->ws, L.tlist);
      int32_t* tcnt = at<int32_t>(h->ws, L.tcnt);
      uint32_t* bits = at<uint32_t>(h->ws, L.bits);
      launch_block_tile_lists(at<double>(h->ws, L.dq), h->kc->C, qperm, bn, nqb, tau, q.qn, e.xn_max, e.eps_rel,
                              h->kc->rad, h->kc->tclo, h->kc->tchi, ntiles, tmajor ? nullptr : tlist, tcnt,
                              tmajor ? bits : nullptr, s);
      if (tmajor)
        launch_tile_units(bits, nqb, ntiles, h->num_sms, at<int32_t>(h->ws, L.tcnt_t), at<int32_t>(h->ws, L.tstart),
                          at<int32_t>(h->ws, L.ustart), uplan, at<int32_t>(h->ws, L.blist),
                          at<int32_t>(h->ws, L.ulist), int64_t(L.ulist_ints / 3), s);
      else
        launch_block_units(tcnt, nqb, ntiles, h->num_sms, at<int32_t>(h->ws, L.tstart), at<int32_t>(h->ws, L.ustart),
                           uplan, at<int32_t>(h->ws, L.ulist), int64_t(L.ulist_ints / 3), s);
    }
    {
      SweepArgs a{};
      a.mode = MODE_FILTER;
      a.qop = &q;
      a.enc = prune ? &h->kc->enc : &e;
      a.n = h->n;
      a.n_pad = h->n_pad;
      a.tile_stride = 1;
      a.tau = tau;
      a.cand_cnt = cnt;
      a.cand = cand;
      a.cap = kp.cap;
      if (prune) {
        a.ulist = at<int32_t>(h->ws, L.ulist);
        a.tlist = tmajor ? nullptr : at<int32_t>(h->ws, L.tlist);
        a.nunits_dev = uplan;
        a.tmajor = tmajor ? 1 : 0;
        a.blist = tmajor ? at<int32_t>(h->ws, L.blist) : nullptr;
        a.unit_counter = tmajor ? ctr + 12 : nullptr;  // zeroed with ctr at the batch start
      }
      // work of the tiles actually swept (all of them unless pruned; the pruned count is read
      // back below only when profiling)
      const double pairs = double(bn) * double(h->n);
      ProfScope ps(h, s, 2.0 * double(h->d) * pairs, double(h->n_pad) * e.Kp * 2, 1);
      launch_sweep(a, h->num_sms, s);
    }
    if (prune && (h->profiling == 1 || h->knn_stats)) {  // diagnostics only: wait for the plan
      int32_t act = 0;
      DK_CUDA(cudaMemcpyAsync(&act, uplan + 1, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
      DK_CUDA(cudaStreamSynchronize(s));
      if (h->profiling == 1) h->last_flops = 2.0 * double(h->d) * double(act) * kBM * kBN;
      if (h->knn_stats)
        std::fprintf(stderr, "[dk] pruned k-NN (%s): %d of %lld (block, tile) pairs swept (%.1f%%), %d balls\n",
                     tmajor ? "tile-major" : "block-major", act, (long long)nqb * ntiles,
                     100.0 * double(act) / (double(nqb) * ntiles), int(h->kc->C));
    }
    if (prune && b0 == 0) {  // the swept fraction of the call's first (largest) batch, read next call
      DK_CUDA(cudaMemcpyAsync(h->kc->stat_host, uplan + 1, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
      DK_CUDA(cudaEventRecord(h->kc->stat_ev, s));
      h->kc->stat_total = double(nqb) * double(ntiles);
      h->kc->stat_pending = true;
    }
    int32_t* lists = at<int32_t>(h->ws, L.lists);
    // pruned: candidates are positions in the cluster-sorted rows (read from there, reported as row ids)
    launch_select(prune ? h->kc->xs : h->X, h->global_offset, h->d, Qb, bn, k, cand, cnt, kp.cap, q.qn, e.xn_max,
                  e.eps_rel, idx_b, d2_b, lists, ctr, h->num_sms, s, prune ? h->kc->perm : nullptr);
    // (the candidate lists are free once the selection has run: scratch for the fallback's row slices)
    launch_exact_knn_fallback(h->X, h->n, h->global_offset, h->d, Qb, lists + bn, ctr + 1, k, idx_b, d2_b,
                              h->num_sms, s, cand, size_t(kp.cap) * size_t(kp.batch) * sizeof(unsigned long long));
    if (h->knn_stats) {
      std::vector<uint32_t> c(static_cast<size_t>(bn));
      int32_t nf = 0;
      DK_CUDA(cudaMemcpyAsync(c.data(), cnt, size_t(bn) * sizeof(uint32_t), cudaMemcpyDeviceToHost, s));
      DK_CUDA(cudaMemcpyAsync(&nf, ctr + 1, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
      DK_CUDA(cudaStreamSynchronize(s));
      for (uint32_t v : c) {
        h->knn_cand_sum += v;
        h->knn_cand_max = std::max<int64_t>(h->knn_cand_max, v);
      }
      h->knn_queries += bn;
      h->knn_fallbacks += nf;
    }
    if (prune) launch_scatter_knn(idx_b, d2_b, qperm, bn, k, idx_d + b0 * k, d2_d + b0 * k, s);
  }
}

size_t knn_ws_bytes(const dk_dataset* h, int32_t k, int64_t nq) {
  if (use_bigk(h, k, nq)) return bigk_temp_bytes(h->n) + 4096;
  const KnnPlan kp = plan_knn(h, k, nq);
  const int32_t Kp_max = int32_t(round_up(3 * int64_t(h->d), kBK));
  return knn_layout(h, kp, k, Kp_max, knn_prunable(h, kp), 0).end + 4096;
}

// Reserve the call's workspace; when the batch planned from the fit-time memory no longer fits
// (other handles or the caller's tensors have taken it since), halve the candidate budget — the
// batch shrinks with it — down to the round-1 plan, then give up with DK_ENOMEM.
void reserve_knn_ws(dk_dataset* h, size_t base, int32_t k, int64_t nq) {
  for (;;) {
    try {
      h->ws.reserve(base + knn_ws_bytes(h, k, nq));
      return;
    } catch (const Error& e) {
      if (e.code != DK_ENOMEM || h->knn_budget <= (int64_t(1) << 30)) throw;
      (void)cudaGetLastError();
      h->knn_budget = std::max<int64_t>(int64_t(1) << 30, h->knn_budget / 2);
    }
  }
}


// ------------------------------------------------------------------ two-precision exact KDE
// Exact gaussian KDE of non-integer data (hybrid.cu): the single-pass fp16 sweep over the
// cluster-sorted rows (the k-NN operand) for every pair, the split3 sweep only over the (query
// block, tile) pairs holding a tile half whose fp16 kernel sum exceeds kHybHotThr, an a-posteriori
// bound per query (fp16 part) checked against kHybTol, exact split3 recomputation of the queries
// that fail it.  Used for gaussian batches of >= kHybMinQueries on datasets of >= kPruneMinTiles
// tiles under DK_PREC_AUTO; DK_KDE_HYBRID=0 turns it off, =1 forces it (read per call).
constexpr int64_t kHybMinQueries = 2048;
// 2^-11 per 128-column half (kernel values in (0, 1]); c3: 2^-12 -> 2^-11 hot pairs 2.7% -> 2.4%
// (3.36 -> 3.33 ms), larger thresholds no further (the same-cluster tiles remain)
constexpr float kHybHotThr = 4.8828125e-04f;
constexpr double kHybTol = 2e-6;                  // relative bound of the fp16 part
constexpr double kHybUseless = 0.25;              // hot (block, tile) fraction above which it does not pay

double env_double(const char* name, double def) {
  const char* v = std::getenv(name);
  return v ? std::atof(v) : def;
}

// sweep values (as means over the global rows) under this are recomputed in fp64: the fp32 epilogue cannot
// represent a term under ~1e-38
constexpr double kUnderflow = 1e-30;

// d2 error model of a split3 sweep, relative to |q|^2 + max |x|^2 (see dk_naive)
double guard_delta_rel(int32_t Kp) { return 0.5 * (std::ldexp(1.0, -21) + double(Kp / 16) * std::ldexp(1.0, -24)); }

bool kde_guard_on() {  // A/B: DK_KDE_GUARD=0 leaves the split3 sweeps unguarded
  static const bool on = [] {
    const char* v = std::getenv("DK_KDE_GUARD");
    return !(v && v[0] == '0');
  }();
  return on;
}

int hyb_env() {  // -1 auto, 0 off, 1 forced
  const char* v = std::getenv("DK_KDE_HYBRID");
  return v ? (std::atoi(v) != 0 ? 1 : 0) : -1;
}

bool hyb_eligible(const dk_dataset* h, int32_t family, int64_t nq) {
  const int mode = hyb_env();
  if (mode == 0 || family != DK_GAUSSIAN || h->precision != DK_PREC_AUTO || h->int_exact || h->kc_failed) return false;
  if (h->n_pad / kBN < kPruneMinTiles || (h->kc != nullptr && h->kc->hyb_failed)) return false;
  return mode == 1 || nq >= kHybMinQueries;
}

// the hot fraction of earlier calls, read without waiting (like knn_prune_decide)
bool hyb_decide(dk_dataset* h) {
  KnnClusters* kc = h->kc;
  if (kc == nullptr || hyb_env() == 1) return true;
  if (kc->hyb_stat_pending) {
    const cudaError_t q = cudaEventQuery(kc->hyb_stat_ev);
    if (q == cudaSuccess) {
      kc->hyb_stat_pending = false;
      const bool wide = double(kc->hyb_stat_host[0]) > kHybUseless * kc->hyb_stat_total;
      if (wide) {
        kc->hyb_useless = true;
        kc->hyb_off_calls = 0;
      }
    } else if (q == cudaErrorNotReady) {
      (void)cudaGetLastError();
    } else {
      DK_CUDA(q);
    }
  }
  if (kc->hyb_useless) {
    if (++kc->hyb_off_calls < 32) return false;
    kc->hyb_useless = false;
    kc->hyb_off_calls = 0;
  }
  return true;
}

// split3 operand of the cluster-sorted rows (first hybrid call); false when it does not fit
bool ensure_sorted_split3(dk_dataset* h, cudaStream_t s) {
  KnnClusters* kc = h->kc;
  if (kc->enc3.mode == 1) return true;
  if (kc->hyb_failed) return false;
  const int32_t d = h->d;
  const int32_t Kp = int32_t(round_up(3 * int64_t(d), kBK));
  {
    size_t free_b = 0, total_b = 0;
    DK_CUDA(cudaMemGetInfo(&free_b, &total_b));
    if (double(free_b) < double(h->n_pad) * (2.0 * Kp + 8.0) * 1.1 + double(64 << 20)) {
      kc->hyb_failed = true;
      return false;
    }
  }
  ensure_mu(h, s);
  Encoding& e = kc->enc3;
  try {
    DK_CUDA(cudaMalloc(&e.B, size_t(h->n_pad) * Kp * sizeof(__half)));
    DK_CUDA(cudaMalloc(&e.xn, size_t(h->n_pad) * sizeof(float)));
    DK_CUDA(cudaMalloc(&e.sx, 2 * sizeof(float)));
    if (!kc->hyb_stat_host) {
      DK_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&kc->hyb_stat_host), 4 * sizeof(int32_t), cudaHostAllocDefault));
      DK_CUDA(cudaEventCreateWithFlags(&kc->hyb_stat_ev, cudaEventDisableTiming));
    }
  } catch (const Error& err) {
    for (void* p : {static_cast<void*>(e.B), static_cast<void*>(e.xn), static_cast<void*>(e.sx)})
      if (p) cudaFree(p);
    e = Encoding{};
    cudaGetLastError();
    if (err.code != DK_ENOMEM) throw;
    kc->hyb_failed = true;
    return false;
  }
  e.Kp = Kp;
  e.d = d;
  e.mu = h->mu;
  launch_encode_rows(kc->xs, h->n, h->n_pad, d, 1, e.mu, Kp, e.B, e.xn, e.sx, reinterpret_cast<uint32_t*>(e.sx + 1),
                     s);
  e.xn_max = kc->enc.xn_max;
  e.eps_rel = float(1.01 * (4.0 * std::ldexp(1.0, -22) + double(Kp + 4) * std::ldexp(1.0, -24)));
  e.tmap = make_tmap_2d_f16(e.B, uint64_t(h->n_pad), uint64_t(Kp), uint32_t(kBN));
  e.tmap_half = make_tmap_2d_f16(e.B, uint64_t(h->n_pad), uint64_t(Kp), uint32_t(kBN / 2));
  e.mode = 1;
  return true;
}

// whether this call runs two-precision (builds the sorted rows and their split3 operand once)
bool hyb_prepare(dk_dataset* h, int32_t family, int64_t nq_chunk_min, cudaStream_t s) {
  if (!hyb_eligible(h, family, nq_chunk_min) || !hyb_decide(h)) return false;
  const Encoding& e = ensure_encoding(h, 2, s);
  if (!ensure_knn_clusters(h, e, s)) return false;
  return ensure_sorted_split3(h, s);
}

// KDE partials of any sweep of at most bpad queries (the batches and the fallback chunks): the
// column-chunk count of the plan grows as the query-block count falls, so bound it over every
// query padding up to bpad
size_t hyb_part_cap(const dk_dataset* h, int32_t bpad) { return sweep_part_bound(h->n_pad, bpad, h->num_sms); }
void check_part_cap(const dk_dataset* h, int32_t pad, int32_t bpad) {  // the bound above, checked
  if (std::max(sweep_part_count(h->n_pad, pad, h->num_sms, false), sweep_part_count(h->n_pad, pad, h->num_sms, true)) >
      hyb_part_cap(h, bpad))
    throw Error{DK_ECUDA, "internal: KDE partial-sum bound exceeded"};
}

struct HybLayout {
  size_t dq, near, near_s, iota, qperm, sort_tmp, qs, A16, At16, qn16, sc16, A3, qn3, sc3, part, bits, tlist, tcnt, ubeg,
      ucnt, ulist, phot, ctr, fail, fv;
  size_t sort_tmp_bytes = 0, end = 0;
  int32_t bpad = 0;
};

// nq: the largest chunk of the call (batch size), nq_call: all its queries (failure list)
HybLayout hyb_layout(const dk_dataset* h, int64_t nq, int64_t nq_call, size_t base) {
  HybLayout L{};
  Plan pl;
  pl.off = base;
  int64_t bmax = 16384;
  if (const char* v = std::getenv("DK_HYB_BATCH")) bmax = std::max<int64_t>(2 * kBM, round_up(std::atoll(v), 2 * kBM));
  L.bpad = int32_t(std::min<int64_t>(bmax, query_pad(nq)));
  const int32_t bpad = L.bpad, nqb = bpad / kBM, ntiles = int32_t(h->n_pad / kBN);
  const int32_t Kp16 = enc_kp(h->d, 2), Kp3 = enc_kp(h->d, 1);
  L.dq = pl.add<unsigned long long>(size_t(bpad));  // nearest-ball keys
  L.near = pl.add<int32_t>(bpad);
  L.near_s = pl.add<int32_t>(bpad);
  L.iota = pl.add<int32_t>(bpad);
  L.qperm = pl.add<int32_t>(bpad);
  L.sort_tmp_bytes = ball_sort_temp_bytes(bpad);
  L.sort_tmp = pl.add<uint8_t>(L.sort_tmp_bytes);
  L.qs = pl.add<double>(size_t(bpad) * h->d);
  L.A16 = pl.add<__half>(size_t(bpad) * Kp16);
  L.At16 = pl.add<__half>(size_t(bpad) * kTailK);
  L.qn16 = pl.add<float>(bpad);
  L.sc16 = pl.add<float>(4);
  L.A3 = pl.add<__half>(size_t(bpad) * Kp3);
  L.qn3 = pl.add<float>(bpad);
  L.sc3 = pl.add<float>(4);
  L.part = pl.add<double>(hyb_part_cap(h, bpad));
  L.bits = pl.add<uint32_t>(size_t(nqb) * ntiles * kHotWords);
  L.tlist = pl.add<int32_t>(size_t(nqb) * ntiles);
  L.tcnt = pl.add<int32_t>(nqb);
  L.ubeg = pl.add<int32_t>(nqb);
  L.ucnt = pl.add<int32_t>(nqb);
  L.ulist = pl.add<int32_t>(size_t(3) * nqb * kHotUnitsPerBlock);
  L.phot = pl.add<double>(size_t(nqb) * kHotUnitsPerBlock * kColGroups * kBM);
  L.ctr = pl.add<int32_t>(16);
  L.fail = pl.add<int32_t>(size_t(nq_call));
  L.fv = pl.add<double>(bpad);
  L.end = pl.off;
  return L;
}



// Two-precision exact gaussian KDE of queries [q0, q0 + qn) of the call's device queries Q into od
// (device, the call's base), means scaled by `scale`.  Enqueued without host waits; the last chunk
// of a call (`last`) reads the failure count of the whole call once and recomputes those queries.
void kde_hybrid(dk_dataset* h, const double* Q, int64_t q0, int64_t qn, double bw, double scale, double* od,
                cudaStream_t s, const HybLayout& L, bool first, bool last) {
  KnnClusters* kc = h->kc;
  if (L.end > h->ws.cap) throw Error{DK_ECUDA, "internal: hybrid KDE workspace under-reserved"};
  const Encoding& e16 = kc->enc;
  const Encoding& e3 = kc->enc3;
  const double log2e = 1.4426950408889634;
  const float negc = float(-log2e / (2.0 * bw * bw));
  const double inv2h2 = 1.0 / (2.0 * bw * bw);
  const float thr = float(env_double("DK_HYB_THR", kHybHotThr));
  const double tol = env_double("DK_HYB_TOL", kHybTol);
  const int32_t ntiles = int32_t(h->n_pad / kBN);
  int32_t* ctr = at<int32_t>(h->ws, L.ctr);  // [0] failures of the call, [4..5] split3 units / listed pairs
  int32_t* fail = at<int32_t>(h->ws, L.fail);  // query ids relative to Q
  if (first) DK_CUDA(cudaMemsetAsync(ctr, 0, 16 * sizeof(int32_t), s));
  // plain split3 sweep over the sorted rows for queries gathered by id (idx) or a contiguous range
  auto split3_rows = [&](const int32_t* idx, int64_t first_q, int64_t fn) {
    const int32_t fpad = int32_t(query_pad(fn));
    check_part_cap(h, fpad, L.bpad);
    const double* Qf = Q + first_q * h->d;
    if (idx != nullptr) {
      launch_gather_rows_f64(Q, idx + first_q, fn, h->d, at<double>(h->ws, L.qs), s);
      Qf = at<double>(h->ws, L.qs);
    }
    QueryOperand q = encode_queries(h, e3, Qf, fn, fpad, at<__half>(h->ws, L.A3), at<float>(h->ws, L.qn3),
                                    at<float>(h->ws, L.sc3), s);
    SweepArgs a{};
    a.mode = MODE_KDE_GAUSS;
    a.qop = &q;
    a.enc = &e3;
    a.n = h->n;
    a.n_pad = h->n_pad;
    a.tile_stride = 1;
    a.negc = negc;
    a.part = at<double>(h->ws, L.part);
    int32_t ncc = 0;
    a.ncc_out = &ncc;
    launch_sweep(a, h->num_sms, s);
    if (idx != nullptr) {
      double* fv = at<double>(h->ws, L.fv);
      launch_reduce_partials(a.part, ncc * kColGroups, fpad, fn, scale, fv, s);
      launch_scatter_f64(fv, idx + first_q, fn, od, s);
    } else {
      launch_reduce_partials(a.part, ncc * kColGroups, fpad, fn, scale, od + first_q, s);
    }
  };
  // queries of this chunk from rest on take the plain split3 sweep (early switch in this call)
  int64_t rest = (!first && kc->hyb_useless) ? 0 : qn;
  const int64_t nbatch = (qn + L.bpad - 1) / L.bpad;
  const int64_t bstep = std::min<int64_t>(L.bpad, round_up((qn + nbatch - 1) / nbatch, 2 * kBM));
  for (int64_t b0 = 0; b0 < rest; b0 += bstep) {
    const int64_t bn = std::min<int64_t>(bstep, qn - b0);
    const int32_t bn_pad = int32_t(query_pad(bn));
    const int32_t nqb = bn_pad / kBM;
    check_part_cap(h, bn_pad, L.bpad);
    const double* Qb = Q + (q0 + b0) * h->d;
    // ball-sorted batch: each block of 128 queries is local, so its hot tiles are few
    int32_t* near = at<int32_t>(h->ws, L.near);
    int32_t* qperm = at<int32_t>(h->ws, L.qperm);
    launch_nearest_ball_f32(Qb, bn, h->d, kc->cent, kc->C, at<unsigned long long>(h->ws, L.dq), near, s);
    launch_sort_queries_by_ball(near, bn, kc->C, at<int32_t>(h->ws, L.near_s), at<int32_t>(h->ws, L.iota), qperm,
                                h->ws.base + L.sort_tmp, L.sort_tmp_bytes, s);
    double* Qs = at<double>(h->ws, L.qs);
    launch_gather_rows_f64(Qb, qperm, bn, h->d, Qs, s);
    QueryOperand q16 = encode_queries(h, e16, Qs, bn, bn_pad, at<__half>(h->ws, L.A16), at<float>(h->ws, L.qn16),
                                      at<float>(h->ws, L.sc16), s, nullptr, true, at<__half>(h->ws, L.At16));
    QueryOperand q3 = encode_queries(h, e3, Qs, bn, bn_pad, at<__half>(h->ws, L.A3), at<float>(h->ws, L.qn3),
                                     at<float>(h->ws, L.sc3), s);
    uint32_t* bits = at<uint32_t>(h->ws, L.bits);
    int32_t ncc = 0;
    {
      SweepArgs a{};
      a.mode = MODE_KDE_COLD;
      a.qop = &q16;
      a.enc = &e16;
      a.n = h->n;
      a.n_pad = h->n_pad;
      a.tile_stride = 1;
      a.negc = negc;
      a.part = at<double>(h->ws, L.part);
      a.ncc_out = &ncc;
      a.hot_bits = bits;
      a.hot_thr = thr;
      ProfScope ps(h, s, 2.0 * double(h->d) * double(bn) * double(h->n), double(h->n_pad) * e16.Kp * 2, 1);
      launch_sweep(a, h->num_sms, s);
    }
    int32_t* tlist = at<int32_t>(h->ws, L.tlist);
    int32_t* tcnt = at<int32_t>(h->ws, L.tcnt);
    int32_t* ubeg = at<int32_t>(h->ws, L.ubeg);
    int32_t* ucnt = at<int32_t>(h->ws, L.ucnt);
    int32_t* ulist = at<int32_t>(h->ws, L.ulist);
    double* phot = at<double>(h->ws, L.phot);
    launch_hot_lists(bits, nqb, ntiles, tlist, tcnt, s);
    launch_hot_units(tcnt, nqb, ntiles, ubeg, ucnt, ctr + 4, ulist, s);
    {
      SweepArgs b{};
      b.mode = MODE_KDE_HOT;
      b.qop = &q3;
      b.enc = &e3;
      b.n = h->n;
      b.n_pad = h->n_pad;
      b.tile_stride = 1;
      b.negc = negc;
      b.part = phot;
      b.hot_bits = bits;
      b.ulist = ulist;
      b.tlist = tlist;
      b.nunits_dev = ctr + 4;
      launch_sweep(b, h->num_sms, s);
    }
    launch_hyb_combine(at<double>(h->ws, L.part), ncc * kColGroups, bn_pad, bn, phot, ubeg, ucnt, q16.qn,
                       e16.eps_rel, e16.xn_max, inv2h2, tol, scale, qperm, q0 + b0, od + q0 + b0, fail, ctr,
                       nullptr, s);
    if (b0 == 0 && first) {  // hot (block, tile) pairs of the call's first batch, read at the next call
      DK_CUDA(cudaMemcpyAsync(kc->hyb_stat_host, ctr + 5, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
      DK_CUDA(cudaEventRecord(kc->hyb_stat_ev, s));
      kc->hyb_stat_total = double(nqb) * double(ntiles);
      kc->hyb_stat_pending = true;
      if (b0 + bn < qn && hyb_env() != 1) {
        // a bandwidth that makes most pairs hot (a wide kernel: c5) costs 1 + 3 MMA passes: the
        // rest of this call and the next 32 calls take the plain split3 sweep
        DK_CUDA(cudaEventSynchronize(kc->hyb_stat_ev));
        kc->hyb_stat_pending = false;
        if (double(kc->hyb_stat_host[0]) > kHybUseless * kc->hyb_stat_total) {
          kc->hyb_useless = true;
          kc->hyb_off_calls = 0;
          rest = b0 + bn;
          break;
        }
      }
    }
  }
  h->hyb_queries += rest;
  for (int64_t r0 = rest; r0 < qn; r0 += L.bpad) split3_rows(nullptr, q0 + r0, std::min<int64_t>(L.bpad, qn - r0));
  if (!last) return;
  // queries of the whole call whose fp16 bound failed: split3 sweeps gathered by id
  int32_t nf = 0;
  DK_CUDA(cudaMemcpyAsync(&nf, ctr, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
  DK_CUDA(cudaStreamSynchronize(s));
  h->hyb_fallbacks += nf;
  for (int64_t f0 = 0; f0 < nf; f0 += L.bpad) split3_rows(fail, f0, std::min<int64_t>(L.bpad, nf - f0));
}

// ------------------------------------------------------------------ fit
struct HandleDeleter {
  void operator()(dk_dataset* h) const { dk_free(h); }
};
using HandlePtr = std::unique_ptr<dk_dataset, HandleDeleter>;

// Device checks and handle fields shared by dk_fit / dk_fit_file (rows not yet on the device).
HandlePtr new_handle(int64_t n, int32_t d, const dk_fit_opts* opts) {
  const int device = opts ? opts->device : 0;
  int ndev = 0;
  DK_CUDA(cudaGetDeviceCount(&ndev));
  if (device < 0 || device >= ndev) throw Error{DK_ENODEV, "no CUDA device " + std::to_string(device)};
  cudaDeviceProp prop;
  DK_CUDA(cudaGetDeviceProperties(&prop, device));
  if (prop.major != 10) throw Error{DK_ENODEV, std::string("device is not sm_100 (B200): ") + prop.name};
  HandlePtr h(new dk_dataset());
  h->device = device;
  h->num_sms = prop.multiProcessorCount;
  h->n = n;
  h->d = d;
  h->n_pad = round_up(n, kBN);
  h->global_offset = opts ? opts->global_offset : 0;
  h->global_n = (opts && opts->global_n > 0) ? opts->global_n : n;
  h->precision = opts ? opts->precision : DK_PREC_AUTO;
  h->knn_stats = std::getenv("DK_KNN_STATS") != nullptr;
  if (const char* pv = std::getenv("DK_PAIR")) set_pair_enabled(std::atoi(pv) != 0);
  DK_REQUIRE(h->precision >= 0 && h->precision <= 2, "unknown precision mode");
  DK_REQUIRE(h->global_offset >= 0 && h->global_offset + n <= h->global_n, "shard outside [0, global_n)");
  {
    DeviceGuard g(device);
    DK_CUDA(cudaHostAlloc(&h->flag_host, 2 * sizeof(uint32_t), cudaHostAllocDefault));
    DK_CUDA(cudaEventCreateWithFlags(&h->flag_event, cudaEventDisableTiming));
    DK_CUDA(cudaHostAlloc(&h->redo_host, 2 * sizeof(int32_t), cudaHostAllocDefault));
    DK_CUDA(cudaEventCreateWithFlags(&h->redo_event, cudaEventDisableTiming));
  }
  return h;
}

// Rows are in h->X: finiteness / integrality flags, fp64 norms, default encoding.
void finish_fit(dk_dataset* h) {
  cudaStream_t s = nullptr;
  DK_CUDA(cudaMalloc(&h->xn64, size_t(h->n) * sizeof(double)));
  uint32_t* flags_d = nullptr;
  DK_CUDA(cudaMalloc(&flags_d, sizeof(uint32_t)));
  DK_CUDA(cudaMemset(flags_d, 0, sizeof(uint32_t)));
  launch_row_stats(h->X, h->n, h->d, h->xn64, flags_d, s);
  uint32_t flags = 0;
  DK_CUDA(cudaMemcpy(&flags, flags_d, sizeof(uint32_t), cudaMemcpyDeviceToHost));
  cudaFree(flags_d);
  DK_REQUIRE(!(flags & 1u), "dataset entries must be finite");
  h->int_exact = (flags & 6u) == 0;
  if (h->precision == DK_PREC_AUTO) ensure_encoding(h, h->int_exact ? 0 : 1, s);
  else if (h->precision == DK_PREC_SPLIT3) ensure_encoding(h, 1, s);
  else ensure_encoding(h, 2, s);
  DK_CUDA(cudaDeviceSynchronize());
  size_t free_b = 0, total_b = 0;
  if (cudaMemGetInfo(&free_b, &total_b) == cudaSuccess)
    h->knn_budget = std::clamp<int64_t>(int64_t(free_b / 10), int64_t(1) << 30, int64_t(10) << 30);
  else
    (void)cudaGetLastError();
}

// ------------------------------------------------------------------ DEANN1 files (data.py:1-15, 151-167)
constexpr int64_t kHeaderBytes = 16;  // magic[8] "DEANN1\0\0", u32 n, u32 d (little-endian)

struct FileHeader {
  int64_t n = 0;
  int32_t d = 0;
};

struct Fd {
  int fd = -1;
  ~Fd() {
    if (fd >= 0) ::close(fd);
  }
};

// Python's repr() of a bytes object (the reference formats the bad magic with !r).
std::string py_bytes_repr(const unsigned char* b, size_t len) {
  bool has_sq = false, has_dq = false;
  for (size_t i = 0; i < len; ++i) {
    has_sq |= b[i] == '\'';
    has_dq |= b[i] == '"';
  }
  const char quote = (has_sq && !has_dq) ? '"' : '\'';
  std::string r = "b";
  r += quote;
  static const char* hex = "0123456789abcdef";
  for (size_t i = 0; i < len; ++i) {
    const unsigned char c = b[i];
    if (c == '\\' || c == static_cast<unsigned char>(quote)) {
      r += '\\';
      r += char(c);
    } else if (c == '\t') {
      r += "\\t";
    } else if (c == '\n') {
      r += "\\n";
    } else if (c == '\r') {
      r += "\\r";
    } else if (c < 32 || c >= 127) {
      r += "\\x";
      r += hex[c >> 4];
      r += hex[c & 15];
    } else {
      r += char(c);
    }
  }
  r += quote;
  return r;
}

// Same checks and messages as _load_binary (data.py:151-167); status DK_EFORMAT.
FileHeader read_header(const char* path) {
  Fd f;
  f.fd = ::open(path, O_RDONLY | O_CLOEXEC);
  if (f.fd < 0) throw Error{DK_EIO, std::string(path) + ": " + std::strerror(errno)};
  unsigned char hdr[kHeaderBytes];
  ssize_t got = 0;
  while (got < kHeaderBytes) {
    const ssize_t r = ::pread(f.fd, hdr + got, size_t(kHeaderBytes - got), got);
    if (r < 0) throw Error{DK_EIO, std::string(path) + ": " + std::strerror(errno)};
    if (r == 0) break;
    got += r;
  }
  if (got != kHeaderBytes)
    throw Error{DK_EFORMAT, std::string(path) + ": truncated header at byte " + std::to_string(got)};
  static const unsigned char kMagic[8] = {'D', 'E', 'A', 'N', 'N', '1', 0, 0};
  if (std::memcmp(hdr, kMagic, 8) != 0)
    throw Error{DK_EFORMAT, std::string(path) + ": bad magic " + py_bytes_repr(hdr, 8) + " at byte 0"};
  auto u32 = [&](int o) {
    return uint32_t(hdr[o]) | (uint32_t(hdr[o + 1]) << 8) | (uint32_t(hdr[o + 2]) << 16) | (uint32_t(hdr[o + 3]) << 24);
  };
  FileHeader fh;
  fh.n = int64_t(u32(8));
  const uint32_t d = u32(12);
  if (fh.n < 1 || d < 1)
    throw Error{DK_EFORMAT, std::string(path) + ": invalid shape " + std::to_string(fh.n) + " x " +
                                std::to_string(d) + " in header"};
  struct stat st;
  if (::fstat(f.fd, &st) != 0) throw Error{DK_EIO, std::string(path) + ": " + std::strerror(errno)};
  // n * d * 4 < 2^66: exact in 128 bits (Python ints in the reference)
  const unsigned __int128 expected = static_cast<unsigned __int128>(fh.n) * d * 4u;
  const int64_t payload = int64_t(st.st_size) - kHeaderBytes;
  if (payload < 0 || static_cast<unsigned __int128>(payload) != expected) {
    std::string ex;
    for (unsigned __int128 v = expected; ex.empty() || v; v /= 10) ex.insert(ex.begin(), char('0' + int(v % 10)));
    throw Error{DK_EFORMAT, std::string(path) + ": expected " + ex + " data bytes after byte " +
                                std::to_string(kHeaderBytes) + ", got " + std::to_string(payload)};
  }
  if (d > uint32_t(std::numeric_limits<int32_t>::max()))
    throw Error{DK_EINVAL, std::string(path) + ": d = " + std::to_string(d) + " exceeds 2^31 - 1"};
  fh.d = int32_t(d);
  return fh;
}

// File bytes [offset, offset+bytes) -> device memory.  Groups of kSlots pinned
// buffers are filled by parallel pread threads; each group's host->device copies
// run on a stream while the next group is read (the pinned slot is reused only
// after its copy's event has completed).  Rows are little-endian fp32 on disk and
// in memory (x86/ARM hosts), so bytes move verbatim.
void stream_file_rows(const char* path, int64_t offset, size_t bytes, float* dst) {
  constexpr int kSlots = 4;
  constexpr size_t kChunk = size_t(16) << 20;
  Fd f;
  f.fd = ::open(path, O_RDONLY | O_CLOEXEC);
  if (f.fd < 0) throw Error{DK_EIO, std::string(path) + ": " + std::strerror(errno)};
  ::posix_fadvise(f.fd, offset, off_t(bytes), POSIX_FADV_SEQUENTIAL);
  struct Pinned {
    void* p = nullptr;
    cudaEvent_t ev = nullptr;
    ~Pinned() {
      if (ev) cudaEventDestroy(ev);
      if (p) cudaFreeHost(p);
    }
  } slot[kSlots];
  for (auto& sl : slot) {
    DK_CUDA(cudaHostAlloc(&sl.p, kChunk, cudaHostAllocDefault));
    DK_CUDA(cudaEventCreateWithFlags(&sl.ev, cudaEventDisableTiming));
  }
  cudaStream_t s;
  DK_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  struct StreamGuard {
    cudaStream_t s;
    ~StreamGuard() {
      cudaStreamSynchronize(s);
      cudaStreamDestroy(s);
    }
  } sg{s};
  const size_t nchunks = (bytes + kChunk - 1) / kChunk;
  bool used[kSlots] = {false, false, false, false};
  for (size_t c0 = 0; c0 < nchunks; c0 += kSlots) {
    const int cnt = int(std::min<size_t>(kSlots, nchunks - c0));
    std::string err[kSlots];
    std::vector<std::thread> readers;
    for (int i = 0; i < cnt; ++i) {
      if (used[i]) DK_CUDA(cudaEventSynchronize(slot[i].ev));
      const size_t c = c0 + size_t(i);
      const size_t len = std::min(kChunk, bytes - c * kChunk);
      const int64_t off = offset + int64_t(c * kChunk);
      readers.emplace_back([&, i, len, off] {
        size_t done = 0;
        while (done < len) {
          const ssize_t r = ::pread(f.fd, static_cast<char*>(slot[i].p) + done, len - done, off + int64_t(done));
          if (r <= 0) {
            err[i] = std::string(path) + ": read failed at byte " + std::to_string(off + int64_t(done)) +
                     (r < 0 ? std::string(": ") + std::strerror(errno) : std::string(": unexpected end of file"));
            return;
          }
          done += size_t(r);
        }
      });
    }
    for (auto& t : readers) t.join();
    for (int i = 0; i < cnt; ++i)
      if (!err[i].empty()) throw Error{DK_EIO, err[i]};
    for (int i = 0; i < cnt; ++i) {
      const size_t c = c0 + size_t(i);
      const size_t len = std::min(kChunk, bytes - c * kChunk);
      DK_CUDA(cudaMemcpyAsync(reinterpret_cast<char*>(dst) + c * kChunk, slot[i].p, len, cudaMemcpyHostToDevice, s));
      DK_CUDA(cudaEventRecord(slot[i].ev, s));
      used[i] = true;
    }
  }
  DK_CUDA(cudaStreamSynchronize(s));
}

}  // namespace
}  // namespace dk

using namespace dk;

extern "C" {

int32_t dk_version(void) { return 10000; }

const char* dk_last_error(void) { return g_err.c_str(); }

int32_t dk_device_ok(int32_t device) {
  cudaDeviceProp prop;
  if (cudaGetDeviceProperties(&prop, device) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return prop.major == 10 ? 1 : 0;
}

dk_status dk_fit(const float* X, int64_t n, int32_t d, const dk_fit_opts* opts, dk_handle* out) {
  DK_NVTX();
  return guard([&] {
    DK_REQUIRE(out != nullptr, "out handle pointer is NULL");
    *out = nullptr;
    DK_REQUIRE(n >= 1 && d >= 1, "dataset must have n >= 1 and d >= 1, got " + std::to_string(n) + " x " +
                                     std::to_string(d));
    DK_REQUIRE(X != nullptr, "dataset pointer is NULL");
    HandlePtr h = new_handle(n, d, opts);
    DeviceGuard g(h->device);
    DK_CUDA(cudaMalloc(&h->X, size_t(n) * d * sizeof(float)));
    DK_CUDA(cudaMemcpy(h->X, X, size_t(n) * d * sizeof(float), cudaMemcpyDefault));
    finish_fit(h.get());
    *out = h.release();
  });
}

dk_status dk_file_info(const char* path, int64_t* n, int32_t* d) {
  DK_NVTX();
  return guard([&] {
    DK_REQUIRE(path != nullptr, "NULL path");
    const FileHeader fh = read_header(path);
    if (n) *n = fh.n;
    if (d) *d = fh.d;
  });
}

dk_status dk_fit_file(const char* path, int64_t row_begin, int64_t row_count, const dk_fit_opts* opts,
                      dk_handle* out) {
  DK_NVTX();
  return guard([&] {
    DK_REQUIRE(path != nullptr && out != nullptr, "NULL argument");
    *out = nullptr;
    const FileHeader fh = read_header(path);
    if (row_count < 0) row_count = fh.n - row_begin;
    DK_REQUIRE(row_begin >= 0 && row_count >= 1 && row_begin + row_count <= fh.n,
               "row range [" + std::to_string(row_begin) + ", " + std::to_string(row_begin + row_count) +
                   ") outside the file's " + std::to_string(fh.n) + " rows");
    dk_fit_opts o = opts ? *opts : dk_fit_opts{0, DK_PREC_AUTO, 0, 0};
    if (o.global_n == 0 && row_count < fh.n) {  // a row shard of the file: global ids = file row ids
      o.global_offset = row_begin;
      o.global_n = fh.n;
    }
    HandlePtr h = new_handle(row_count, fh.d, &o);
    DeviceGuard g(h->device);
    DK_CUDA(cudaMalloc(&h->X, size_t(row_count) * fh.d * sizeof(float)));
    stream_file_rows(path, kHeaderBytes + row_begin * int64_t(fh.d) * 4, size_t(row_count) * fh.d * 4, h->X);
    finish_fit(h.get());
    *out = h.release();
  });
}

dk_status dk_free(dk_handle h) {
  DK_NVTX();
  return guard([&] {
    if (!h) return;
    DeviceGuard g(h->device);
    cudaDeviceSynchronize();
    free_encoding(h->enc_exact);
    free_encoding(h->enc_split);
    free_encoding(h->enc_fp16);
    if (h->kc) {
      free_knn_clusters(*h->kc);
      delete h->kc;
    }
    if (h->X) cudaFree(h->X);
    if (h->xn64) cudaFree(h->xn64);
    if (h->mu) cudaFree(h->mu);
    if (h->rsp_inverse) cudaFree(h->rsp_inverse);
    if (h->flag_host) cudaFreeHost(h->flag_host);
    if (h->flag_event) cudaEventDestroy(h->flag_event);
    if (h->redo_host) cudaFreeHost(h->redo_host);
    if (h->redo_event) cudaEventDestroy(h->redo_event);
    if (h->copy_stream) cudaStreamDestroy(h->copy_stream);
    if (h->copy_ready) cudaEventDestroy(h->copy_ready);
    if (h->copy_done) cudaEventDestroy(h->copy_done);
    for (auto& pr : h->prof_events) {
      cudaEventDestroy(pr.first);
      cudaEventDestroy(pr.second);
    }
    delete h;
  });
}

dk_status dk_info(dk_handle h, int64_t* n, int32_t* d, int64_t* go, int64_t* gn, int32_t* exact) {
  return guard([&] {
    DK_REQUIRE(h != nullptr, "NULL handle");
    if (n) *n = h->n;
    if (d) *d = h->d;
    if (go) *go = h->global_offset;
    if (gn) *gn = h->global_n;
    if (exact) *exact = h->int_exact ? 1 : 0;
  });
}

dk_status dk_sq_norms(dk_handle h, double* out, void* stream) {
  DK_NVTX();
  return guard([&] {
    DK_REQUIRE(h != nullptr && out != nullptr, "NULL argument");
    DeviceGuard g(h->device);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    DK_CUDA(cudaMemcpyAsync(out, h->xn64, size_t(h->n) * sizeof(double), cudaMemcpyDefault, s));
    if (!is_device_ptr(out)) DK_CUDA(cudaStreamSynchronize(s));
  });
}

dk_status dk_naive(dk_handle h, const double* Q, int64_t nq, int32_t family, double bandwidth, uint32_t flags,
                   double* out, void* stream) {
  DK_NVTX();
  return guard([&] {
    DK_REQUIRE(h != nullptr, "NULL handle");
    check_family_bw(family, bandwidth);
    DK_REQUIRE(nq >= 0, "negative query count");
    if (nq == 0) return;
    DK_REQUIRE(Q != nullptr && out != nullptr, "NULL query or output pointer");
    DeviceGuard g(h->device);
    LaunchCount lc(h);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const bool out_dev = is_device_ptr(out);
    // mean over the GLOBAL row count: a shard handle writes its contribution to the global mean,
    // so an all-reduce (sum) of the shards gives the KDE directly
    const double scale = (flags & DK_OUT_SUM) ? 1.0 : 1.0 / double(h->global_n);
    Plan pl;
    const size_t o_Q = pl.add<double>(size_t(nq) * h->d);
    const size_t o_out = pl.add<double>(size_t(nq));
    const size_t o_flags = pl.add<uint32_t>(4);
    if (family == DK_LAPLACIAN) {
      const size_t o_part = pl.add<double>(l1_part_count(h->n, int32_t(nq)));
      const size_t o_q32 = pl.add<float>(size_t(l1_nq_pad(nq)) * h->d);
      const size_t o_rlist = pl.add<int32_t>(size_t(nq) + 4);
      const size_t o_rpart = pl.add<double>(size_t(nq) * kRedoChunks);
      h->ws.reserve(pl.off);
      const double* Qd = stage_queries(h, Q, nq, o_Q, s);
      int32_t nparts = 0;
      double* part = at<double>(h->ws, o_part);
      double* od = out_dev ? out : at<double>(h->ws, o_out);
      {
        ProfScope ps(h, s, 3.0 * double(h->d) * double(nq) * double(h->n), double(h->n) * h->d * 4, 1);
        launch_l1_kde(h->X, h->n, h->d, Qd, nq, 1.0 / bandwidth, part, &nparts, at<float>(h->ws, o_q32), s);
      }
      launch_reduce_partials(part, nparts, l1_nq_pad(nq), nq, scale, od, s);
      h->redo_mask = 0;
      if (kde_guard_on()) {  // queries under the fp32 epilogue's range: fp64 (redo.cu)
        int32_t* rlist = at<int32_t>(h->ws, o_rlist);
        launch_kde_redo(h->X, h->n, h->d, Qd, nq, family, bandwidth, nullptr, kUnderflow * scale * double(h->global_n),
                        rlist + 4, rlist, at<double>(h->ws, o_rpart), scale, od, h->num_sms, s);
        DK_CUDA(cudaMemcpyAsync(h->redo_host, rlist, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
        DK_CUDA(cudaEventRecord(h->redo_event, s));
        h->redo_mask = 1;
      }
      if (!out_dev) {
        copy_out(out, od, size_t(nq) * sizeof(double), s);
        DK_CUDA(cudaStreamSynchronize(s));
      }
      return;
    }
    // Host queries of a large batch run as two chunks: the copy of the second (3/4 of the
    // batch) overlaps the sweep of the first on a side stream, hiding most of the H2D time.
    const bool host_q = !is_device_ptr(Q);
    static const int64_t split_div = [] {  // A/B: first chunk = 1/div of the batch
      const char* v = std::getenv("DK_E2E_SPLIT");
      return v ? std::max<int64_t>(2, std::atoll(v)) : int64_t(4);
    }();
    // two-precision exact KDE (non-integer gaussian batches on large datasets): decided first (the
    // first call builds the sorted rows' operands in their own memory); it runs as ONE chunk — its
    // per-batch passes (ball order, two query encodes, hot lists, split3 pass) cost more when split
    // than the hidden copy saves (c3 end to end 4.47 -> 3.6 ms)
    const bool hyb = hyb_prepare(h, family, nq, s);
    h->redo_mask = 0;
    const int64_t split = (host_q && nq >= 4096 && !hyb) ? round_up(nq / split_div, 256) : nq;
    const int64_t c_beg[2] = {0, split};
    const int64_t c_cnt[2] = {split, nq - split};
    const int nchunks = c_cnt[1] > 0 ? 2 : 1;
    const int32_t Kp_max = int32_t(round_up(3 * int64_t(h->d), kBK));
    size_t o_A[2], o_At[2], o_qn[2], o_scal[2], o_part[2], o_fl[2], o_tau[2] = {}, o_gflag[2] = {}, o_rlist[2] = {}, o_rpart[2] = {};
    for (int c = 0; c < nchunks; ++c) {
      const int32_t pad = int32_t(query_pad(c_cnt[c]));
      o_A[c] = pl.add<__half>(size_t(pad) * Kp_max);
      o_At[c] = pl.add<__half>(size_t(pad) * kTailK);
      o_qn[c] = pl.add<float>(pad);
      o_scal[c] = pl.add<float>(4);
      o_part[c] = pl.add<double>(sweep_part_count(h->n_pad, pad, h->num_sms));
      o_fl[c] = pl.add<uint32_t>(4);
      if (!hyb) o_tau[c] = pl.add<float>(pad);  // guard of the split3 sweeps (redo.cu)
      o_gflag[c] = pl.add<uint32_t>(pad);
      o_rlist[c] = pl.add<int32_t>(size_t(pad) + 4);  // (the two-precision path: underflowed queries only)
      o_rpart[c] = pl.add<double>(size_t(c_cnt[c]) * kRedoChunks);
    }
    const HybLayout HL = hyb ? hyb_layout(h, std::max(c_cnt[0], c_cnt[1]), nq, pl.off) : HybLayout{};
    h->ws.reserve(hyb ? HL.end + 4096 : pl.off);
    double* od = out_dev ? out : at<double>(h->ws, o_out);
    const double* Qd = Q;
    if (host_q) {
      double* dst = at<double>(h->ws, o_Q);
      DK_CUDA(cudaMemcpyAsync(dst, Q, size_t(c_cnt[0]) * h->d * sizeof(double), cudaMemcpyHostToDevice, s));
      if (nchunks == 2) {
        if (!h->copy_stream) {
          DK_CUDA(cudaStreamCreateWithFlags(&h->copy_stream, cudaStreamNonBlocking));
          DK_CUDA(cudaEventCreateWithFlags(&h->copy_ready, cudaEventDisableTiming));
          DK_CUDA(cudaEventCreateWithFlags(&h->copy_done, cudaEventDisableTiming));
        }
        // the side copy may only overwrite the staging area once earlier work on s is done
        DK_CUDA(cudaEventRecord(h->copy_ready, s));
        DK_CUDA(cudaStreamWaitEvent(h->copy_stream, h->copy_ready, 0));
        DK_CUDA(cudaMemcpyAsync(dst + size_t(c_beg[1]) * h->d, Q + size_t(c_beg[1]) * h->d,
                                size_t(c_cnt[1]) * h->d * sizeof(double), cudaMemcpyHostToDevice,
                                h->copy_stream));
        DK_CUDA(cudaEventRecord(h->copy_done, h->copy_stream));
      }
      Qd = dst;
    }
    const double log2e = 1.4426950408889634;
    const float negc = float(family == DK_GAUSSIAN ? -log2e / (2.0 * bandwidth * bandwidth) : -log2e / bandwidth);
    auto run_sweep = [&](int c, int mode, uint32_t* guard_flags) {
      const int64_t q0 = c_beg[c], cn = c_cnt[c];
      const int32_t pad = int32_t(query_pad(cn));
      const double* Qc = Qd + size_t(q0) * h->d;
      const Encoding& e = ensure_encoding(h, mode, s);
      // speculative exact mode: the query encode also computes the exact-mode flags
      // exact-mode gaussian sweeps carry the query norms in the operand (the MMA yields -d2/2)
      QueryOperand q = encode_queries(h, e, Qc, cn, pad, at<__half>(h->ws, o_A[c]), at<float>(h->ws, o_qn[c]),
                                      at<float>(h->ws, o_scal[c]), s, guard_flags, mode == 0 && family == DK_GAUSSIAN,
                                      at<__half>(h->ws, o_At[c]));
      if (guard_flags) {
        DK_CUDA(cudaMemcpyAsync(h->flag_host + c, guard_flags, sizeof(uint32_t), cudaMemcpyDeviceToHost, s));
        DK_CUDA(cudaEventRecord(h->flag_event, s));
      }
      SweepArgs a{};
      a.mode = family == DK_GAUSSIAN ? MODE_KDE_GAUSS : MODE_KDE_EXP;
      a.qop = &q;
      a.enc = &e;
      a.n = h->n;
      a.n_pad = h->n_pad;
      a.tile_stride = 1;
      a.negc = negc;
      a.part = at<double>(h->ws, o_part[c]);
      a.guard = guard_flags;
      // split3 sweeps are guarded: the d2 of a pair is off by about delta_q = delta_rel (|q|^2 + max |x|^2)
      // (operand rounding 2^-22 |q||x| plus the fp32 accumulation over Kp / 16 MMA steps, which
      // truncates: measured on sparse d = 784 rows, gaussian, 2h^2 = 4: 4.5e-4 against this model's
      // 4.9e-4).  Queries whose kernel values that error can move by more than the tolerance are
      // recomputed in fp64 (redo.cu): every exponential-kernel row with an approximate d2 under
      // (delta_q / (tol h))^2 (flagged by the sweep), every gaussian query with delta_q > tol 2h^2.
      const bool guarded = mode == 1 && kde_guard_on();
      uint32_t* gflag = nullptr;
      if (guarded) {
        const double delta_rel = guard_delta_rel(e.Kp);
        gflag = at<uint32_t>(h->ws, o_gflag[c]);
        launch_guard_tau(q.qn, pad, cn, e.xn_max, delta_rel, family == DK_GAUSSIAN ? 5e-5 : 1e-4, bandwidth,
                         family == DK_GAUSSIAN, at<float>(h->ws, o_tau[c]), gflag, s);
        if (family != DK_GAUSSIAN) {
          a.tau = at<float>(h->ws, o_tau[c]);
          a.cand_cnt = gflag;
        }
      }
      int32_t ncc = 0;
      a.ncc_out = &ncc;
      {
        ProfScope ps(h, s, 2.0 * double(h->d) * double(cn) * double(h->n), double(h->n_pad) * e.Kp * 2, 1);
        launch_sweep(a, h->num_sms, s);
      }
      launch_reduce_partials(a.part, ncc * kColGroups, pad, cn, scale, od + q0, s);
      if (guarded) {
        int32_t* rlist = at<int32_t>(h->ws, o_rlist[c]);
        launch_kde_redo(h->X, h->n, h->d, Qc, cn, family, bandwidth, gflag, kUnderflow * scale * double(h->global_n),
                        rlist + 4, rlist, at<double>(h->ws, o_rpart[c]), scale, od + q0, h->num_sms, s);
        DK_CUDA(cudaMemcpyAsync(h->redo_host + c, rlist, sizeof(int32_t), cudaMemcpyDeviceToHost, s));  // statistics
        DK_CUDA(cudaEventRecord(h->redo_event, s));
        h->redo_mask |= 1 << c;
      }
      if (!out_dev) copy_out(out + q0, od + q0, size_t(cn) * sizeof(double), s);
    };
    // Integer dataset: the exact-mode sweeps are launched without waiting for the query check.
    // Each reads its chunk's flags and skips itself for fractional queries; the host waits for
    // the flags only after every chunk is enqueued (the last record of flag_event follows both
    // chunks' flag copies) and redoes a fractional chunk in split3.  No host round trip sits
    // between the chunks (round 1 waited per chunk, so chunk 1's sweep was enqueued only after
    // chunk 0's sweep had drained the stream) or between consecutive calls.
    const bool speculative = !hyb && h->precision == DK_PREC_AUTO && h->int_exact;
    for (int c = 0; c < nchunks; ++c) {
      if (c == 1) DK_CUDA(cudaStreamWaitEvent(s, h->copy_done, 0));
      if (hyb) {
        kde_hybrid(h, Qd, c_beg[c], c_cnt[c], bandwidth, scale, od, s, HL, c == 0, c == nchunks - 1);
        if (kde_guard_on()) {
          // the hot pairs run the same split3 arithmetic as the plain sweep: the same gaussian guard
          // (d2 error against 2h^2), from the raw queries; and values under the fp32 epilogue's range
          int32_t* rlist = at<int32_t>(h->ws, o_rlist[c]);
          uint32_t* gflag = at<uint32_t>(h->ws, o_gflag[c]);
          const Encoding& e3 = h->kc->enc3;
          launch_guard_flag_raw(Qd + size_t(c_beg[c]) * h->d, h->mu, h->d, c_cnt[c], e3.xn_max, guard_delta_rel(e3.Kp),
                                5e-5 * 2.0 * bandwidth * bandwidth, gflag, s);
          launch_kde_redo(h->X, h->n, h->d, Qd + size_t(c_beg[c]) * h->d, c_cnt[c], family, bandwidth, gflag,
                          kUnderflow * scale * double(h->global_n), rlist + 4, rlist, at<double>(h->ws, o_rpart[c]),
                          scale, od + c_beg[c], h->num_sms, s);
          DK_CUDA(cudaMemcpyAsync(h->redo_host + c, rlist, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
          DK_CUDA(cudaEventRecord(h->redo_event, s));
          h->redo_mask |= 1 << c;
        }
        if (!out_dev && c == nchunks - 1) copy_out(out, od, size_t(nq) * sizeof(double), s);
        continue;
      }
      if (speculative) {
        uint32_t* flags = at<uint32_t>(h->ws, o_fl[c]);
        DK_CUDA(cudaMemsetAsync(flags, 0, sizeof(uint32_t), s));
        run_sweep(c, 0, flags);
      } else {
        run_sweep(c, choose_mode(h, Qd + size_t(c_beg[c]) * h->d, c_cnt[c], at<uint32_t>(h->ws, o_fl[c]), s),
                  nullptr);
      }
    }
    if (speculative) {
      DK_CUDA(cudaEventSynchronize(h->flag_event));
      for (int c = 0; c < nchunks; ++c) DK_REQUIRE(!(h->flag_host[c] & 1u), "queries must be finite");
      for (int c = 0; c < nchunks; ++c)
        if (h->flag_host[c] & 6u) run_sweep(c, 1, nullptr);
    }
    if (!out_dev) DK_CUDA(cudaStreamSynchronize(s));
  });
}

dk_status dk_knn(dk_handle h, const double* Q, int64_t nq, int32_t k, int64_t* idx_out, double* d2_out,
                 void* stream) {
  DK_NVTX();
  return guard([&] {
    DK_REQUIRE(h != nullptr, "NULL handle");
    DK_REQUIRE(k >= 1 && int64_t(k) <= h->n,
               "k=" + std::to_string(k) + " out of range [1, " + std::to_string(h->n) + "]");
    DK_REQUIRE(nq >= 0, "negative query count");
    if (nq == 0) return;
    DK_REQUIRE(Q != nullptr && idx_out != nullptr && d2_out != nullptr, "NULL argument");
    DeviceGuard g(h->device);
    LaunchCount lc(h);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const bool idx_dev = is_device_ptr(idx_out), d2_dev = is_device_ptr(d2_out);
    Plan pl;
    const size_t o_Q = pl.add<double>(size_t(nq) * h->d);
    const size_t o_idx = pl.add<int64_t>(size_t(nq) * k);
    const size_t o_d2 = pl.add<double>(size_t(nq) * k);
    const size_t base = pl.off;
    reserve_knn_ws(h, base, k, nq);
    const double* Qd = stage_queries(h, Q, nq, o_Q, s);
    int64_t* idx_d = idx_dev ? idx_out : at<int64_t>(h->ws, o_idx);
    double* d2_d = d2_dev ? d2_out : at<double>(h->ws, o_d2);
    knn_device(h, Qd, nq, k, idx_d, d2_d, s, base);
    if (!idx_dev) copy_out(idx_out, idx_d, size_t(nq) * k * sizeof(int64_t), s);
    if (!d2_dev) copy_out(d2_out, d2_d, size_t(nq) * k * sizeof(double), s);
    if (!idx_dev || !d2_dev) DK_CUDA(cudaStreamSynchronize(s));
  });
}

dk_status dk_merge_topk(int32_t parts, int64_t nq, int32_t k, const int64_t* idx_in, const double* d2_in,
                        int64_t* idx_out, double* d2_out, void* stream) {
  DK_NVTX();
  return guard([&] {
    DK_REQUIRE(parts >= 1 && parts <= 64 && k >= 1 && nq >= 0, "bad merge arguments");
    if (nq == 0) return;
    DK_REQUIRE(is_device_ptr(idx_in) && is_device_ptr(d2_in) && is_device_ptr(idx_out) && is_device_ptr(d2_out),
               "dk_merge_topk expects device pointers");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    launch_merge_topk(parts, nq, k, idx_in, d2_in, idx_out, d2_out, s);
  });
}

dk_status dk_sample(dk_handle h, const double* Q, int64_t nq, int32_t family, double bandwidth, int32_t m,
                    uint64_t seed, int64_t query_base, const int64_t* excl, const int32_t* excl_cnt,
                    int32_t excl_stride, double* z_sum, int64_t* accepted_idx_out, int64_t* draws_out,
                    void* stream) {
  DK_NVTX();
  return guard([&] {
    DK_REQUIRE(h != nullptr, "NULL handle");
    check_family_bw(family, bandwidth);
    DK_REQUIRE(m >= 1, "m=" + std::to_string(m) + " must be >= 1");
    DK_REQUIRE(nq >= 0, "negative query count");
    if (nq == 0) return;
    DK_REQUIRE(Q != nullptr && z_sum != nullptr, "NULL argument");
    DK_REQUIRE(!excl || excl_stride >= 1, "excl_stride must be >= 1");
    DeviceGuard g(h->device);
    LaunchCount lc(h);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    Plan pl;
    const size_t o_Q = pl.add<double>(size_t(nq) * h->d);
    const size_t o_ex = pl.add<int64_t>(excl ? size_t(nq) * excl_stride : 1);
    const size_t o_exs = pl.add<int64_t>(excl ? size_t(nq) * excl_stride : 1);
    const size_t o_cnt = pl.add<int32_t>(excl_cnt ? size_t(nq) : 1);
    const size_t o_z = pl.add<double>(size_t(nq));
    const size_t o_acc = pl.add<int64_t>(accepted_idx_out ? size_t(nq) * m : 1);
    const size_t o_dr = pl.add<int64_t>(size_t(nq));
    const bool long_excl = excl && excl_stride > kSmemSortMax;
    const size_t seg_bytes = long_excl ? seg_sort_temp_bytes(excl_stride, nq) : 0;
    const size_t o_seg = pl.add<uint8_t>(seg_bytes);
    h->ws.reserve(pl.off);
    const double* Qd = stage_queries(h, Q, nq, o_Q, s);
    const int64_t* ex_sorted = nullptr;
    const int32_t* cnt_d = nullptr;
    if (excl) {
      int64_t* ex_d = at<int64_t>(h->ws, o_ex);
      DK_CUDA(cudaMemcpyAsync(ex_d, excl, size_t(nq) * excl_stride * sizeof(int64_t), cudaMemcpyDefault, s));
      if (excl_cnt) {
        int32_t* c = at<int32_t>(h->ws, o_cnt);
        DK_CUDA(cudaMemcpyAsync(c, excl_cnt, size_t(nq) * sizeof(int32_t), cudaMemcpyDefault, s));
        cnt_d = c;
      }
      int64_t* srt = at<int64_t>(h->ws, o_exs);
      if (long_excl) launch_seg_sort_i64(ex_d, srt, cnt_d, excl_stride, nq, at<uint8_t>(h->ws, o_seg), seg_bytes, s);
      else launch_sort_excl(ex_d, cnt_d, excl_stride, nq, srt, s);
      ex_sorted = srt;
    }
    const bool z_dev = is_device_ptr(z_sum);
    double* zd = z_dev ? z_sum : at<double>(h->ws, o_z);
    const bool acc_dev = accepted_idx_out && is_device_ptr(accepted_idx_out);
    int64_t* accd = accepted_idx_out ? (acc_dev ? accepted_idx_out : at<int64_t>(h->ws, o_acc)) : nullptr;
    const bool dr_dev = draws_out && is_device_ptr(draws_out);
    int64_t* drd = draws_out ? (dr_dev ? draws_out : at<int64_t>(h->ws, o_dr)) : nullptr;
    {
      ProfScope ps(h, s, 0.0, double(nq) * m * h->d * 4.0, 2);
      launch_sample(h->X, h->n, h->global_offset, h->global_n, h->d, Qd, nq, family, bandwidth, m, seed, query_base,
                    ex_sorted, cnt_d, excl ? excl_stride : 0, zd, accd, drd, s);
    }
    bool sync = false;
    if (!z_dev) { copy_out(z_sum, zd, size_t(nq) * sizeof(double), s); sync = true; }
    if (accd && !acc_dev) { copy_out(accepted_idx_out, accd, size_t(nq) * m * sizeof(int64_t), s); sync = true; }
    if (drd && !dr_dev) { copy_out(draws_out, drd, size_t(nq) * sizeof(int64_t), s); sync = true; }
    if (sync) DK_CUDA(cudaStreamSynchronize(s));
  });
}

dk_status dk_eval_rows(dk_handle h, const double* Q, int64_t nq, int32_t family, double bandwidth,
                       const int64_t* rows, const int32_t* cnt, int32_t stride, double* out, void* stream) {
  DK_NVTX();
  return guard([&] {
    DK_REQUIRE(h != nullptr, "NULL handle");
    check_family_bw(family, bandwidth);
    DK_REQUIRE(nq >= 0 && stride >= 0, "negative size");
    if (nq == 0) return;
    DK_REQUIRE(Q != nullptr && out != nullptr && (rows != nullptr || stride == 0), "NULL argument");
    DeviceGuard g(h->device);
    LaunchCount lc(h);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    Plan pl;
    const size_t o_Q = pl.add<double>(size_t(nq) * h->d);
    const size_t o_r = pl.add<int64_t>(size_t(nq) * std::max(stride, 1));
    const size_t o_c = pl.add<int32_t>(size_t(nq));
    const size_t o_o = pl.add<double>(size_t(nq));
    h->ws.reserve(pl.off);
    const double* Qd = stage_queries(h, Q, nq, o_Q, s);
    const int64_t* rd = rows;
    if (rows && !is_device_ptr(rows)) {
      int64_t* r = at<int64_t>(h->ws, o_r);
      DK_CUDA(cudaMemcpyAsync(r, rows, size_t(nq) * stride * sizeof(int64_t), cudaMemcpyHostToDevice, s));
      rd = r;
    }
    const int32_t* cd = cnt;
    if (cnt && !is_device_ptr(cnt)) {
      int32_t* c = at<int32_t>(h->ws, o_c);
      DK_CUDA(cudaMemcpyAsync(c, cnt, size_t(nq) * sizeof(int32_t), cudaMemcpyHostToDevice, s));
      cd = c;
    }
    const bool od = is_device_ptr(out);
    double* o = od ? out : at<double>(h->ws, o_o);
    launch_eval_rows(h->X, h->n, h->global_offset, h->d, Qd, nq, family, bandwidth, rd, cd, stride, o, s);
    if (!od) {
      copy_out(out, o, size_t(nq) * sizeof(double), s);
      DK_CUDA(cudaStreamSynchronize(s));
    }
  });
}

dk_status dk_kernel_values(int32_t family, double bandwidth, const double* dist, int64_t count, double* out,
                           void* stream) {
  DK_NVTX();
  return guard([&] {
    check_family_bw(family, bandwidth);
    DK_REQUIRE(count >= 0, "negative count");
    if (count == 0) return;
    DK_REQUIRE(dist != nullptr && out != nullptr, "NULL argument");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const bool din = is_device_ptr(dist), dout = is_device_ptr(out);
    // per-device scratch, grown on demand and reused (no allocation per call); the call
    // synchronises its stream before returning, so holding the lock makes reuse safe
    static std::mutex mu;
    static std::map<int, std::pair<uint8_t*, size_t>> scratch;
    std::lock_guard<std::mutex> lk(mu);
    int dev = 0;
    DK_CUDA(cudaGetDevice(&dev));
    const size_t need = 256 + (din ? 0 : size_t(count)) * sizeof(double) + (dout ? 0 : size_t(count)) * sizeof(double);
    auto& sc = scratch[dev];
    if (sc.second < need) {
      if (sc.first) {
        DK_CUDA(cudaDeviceSynchronize());
        DK_CUDA(cudaFree(sc.first));
        sc = {nullptr, 0};
      }
      const size_t want = std::max(need + need / 4, size_t(1) << 20);
      DK_CUDA(cudaMalloc(&sc.first, want));
      sc.second = want;
    }
    uint32_t* bad = reinterpret_cast<uint32_t*>(sc.first);
    double* cur = reinterpret_cast<double*>(sc.first + 256);
    const double* dd = dist;
    if (!din) {
      DK_CUDA(cudaMemcpyAsync(cur, dist, size_t(count) * sizeof(double), cudaMemcpyHostToDevice, s));
      dd = cur;
      cur += count;
    }
    double* od = dout ? out : cur;
    DK_CUDA(cudaMemsetAsync(bad, 0, sizeof(uint32_t), s));
    launch_kernel_values(family, bandwidth, dd, count, od, bad, s);
    uint32_t b = 0;
    DK_CUDA(cudaMemcpyAsync(&b, bad, sizeof(uint32_t), cudaMemcpyDeviceToHost, s));
    if (!dout) DK_CUDA(cudaMemcpyAsync(out, od, size_t(count) * sizeof(double), cudaMemcpyDeviceToHost, s));
    DK_CUDA(cudaStreamSynchronize(s));
    DK_REQUIRE(!(b & 1u), "distance must be finite");
    DK_REQUIRE(!(b & 2u), "distance must be nonnegative");
  });
}

dk_status dk_deann(dk_handle h, const double* Q, int64_t nq, int32_t family, double bandwidth, int32_t k, int32_t m,
                   uint64_t seed, int64_t query_base, double* value_out, int64_t* nbr_idx_out, double* nbr_d2_out,
                   int64_t* sample_idx_out, void* stream) {
  DK_NVTX();
  return guard([&] {
    DK_REQUIRE(h != nullptr, "NULL handle");
    check_family_bw(family, bandwidth);
    const int64_t n = h->n;
    DK_REQUIRE(h->global_offset == 0 && h->global_n == n,
               "dk_deann runs on an unsharded handle; use dk_knn/dk_sample per shard");
    DK_REQUIRE(k >= 0 && int64_t(k) <= n, "k=" + std::to_string(k) + " out of range [0, " + std::to_string(n) + "]");
    DK_REQUIRE(m >= 0, "m=" + std::to_string(m) + " must be >= 0");
    DK_REQUIRE(!(m > 0 && int64_t(k) >= n), "m > 0 requires k + 1 <= n so the remainder is nonempty");
    DK_REQUIRE(nq >= 0, "negative query count");
    if (nq == 0) return;
    DK_REQUIRE(Q != nullptr && value_out != nullptr, "NULL argument");
    DeviceGuard g(h->device);
    LaunchCount lc(h);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const int32_t ks = std::max(k, 1);
    Plan pl;
    const size_t o_Q = pl.add<double>(size_t(nq) * h->d);
    const size_t o_idx = pl.add<int64_t>(size_t(nq) * ks);
    const size_t o_d2 = pl.add<double>(size_t(nq) * ks);
    const size_t o_srt = pl.add<int64_t>(size_t(nq) * ks);
    const size_t o_z1 = pl.add<double>(size_t(nq));
    const size_t o_z2 = pl.add<double>(size_t(nq));
    const size_t o_val = pl.add<double>(size_t(nq));
    const size_t o_acc = pl.add<int64_t>(sample_idx_out ? size_t(nq) * std::max(m, 1) : 1);
    const bool long_excl = m > 0 && k > kSmemSortMax;
    const size_t seg_bytes = long_excl ? seg_sort_temp_bytes(k, nq) : 0;
    const size_t o_seg = pl.add<uint8_t>(seg_bytes);
    const size_t base = pl.off;
    if (k > 0) reserve_knn_ws(h, base, k, nq);
    else h->ws.reserve(base);
    const double* Qd = stage_queries(h, Q, nq, o_Q, s);
    int64_t* idx = at<int64_t>(h->ws, o_idx);
    double* d2 = at<double>(h->ws, o_d2);
    double* z1 = at<double>(h->ws, o_z1);
    double* z2 = at<double>(h->ws, o_z2);
    if (k > 0) {
      knn_device(h, Qd, nq, k, idx, d2, s, base);
      if (family == DK_LAPLACIAN)
        launch_eval_rows(h->X, h->n, 0, h->d, Qd, nq, family, bandwidth, idx, nullptr, k, z1, s);
    }
    const bool acc_dev = sample_idx_out && is_device_ptr(sample_idx_out);
    int64_t* accd = sample_idx_out ? (acc_dev ? sample_idx_out : at<int64_t>(h->ws, o_acc)) : nullptr;
    if (m > 0) {
      const int64_t* ex = nullptr;
      if (k > 0) {
        int64_t* srt = at<int64_t>(h->ws, o_srt);
        if (long_excl) launch_seg_sort_i64(idx, srt, nullptr, k, nq, at<uint8_t>(h->ws, o_seg), seg_bytes, s);
        else launch_sort_excl(idx, nullptr, k, nq, srt, s);
        ex = srt;
      }
      ProfScope ps(h, s, 0.0, double(nq) * m * h->d * 4.0, 2);  // accepted rows read
      launch_sample(h->X, h->n, 0, n, h->d, Qd, nq, family, bandwidth, m, seed, query_base, ex, nullptr,
                    k > 0 ? k : 0, z2, accd, nullptr, s);
    }
    const bool v_dev = is_device_ptr(value_out);
    double* vd = v_dev ? value_out : at<double>(h->ws, o_val);
    launch_deann_combine(nq, family, bandwidth, k, m, n, d2, z1, z2, vd, s);
    bool sync = false;
    if (!v_dev) { copy_out(value_out, vd, size_t(nq) * sizeof(double), s); sync = true; }
    if (k > 0 && nbr_idx_out) { copy_out(nbr_idx_out, idx, size_t(nq) * k * sizeof(int64_t), s); sync = true; }
    if (k > 0 && nbr_d2_out) { copy_out(nbr_d2_out, d2, size_t(nq) * k * sizeof(double), s); sync = true; }
    if (accd && !acc_dev && m > 0) { copy_out(sample_idx_out, accd, size_t(nq) * m * sizeof(int64_t), s); sync = true; }
    if (sync) DK_CUDA(cudaStreamSynchronize(s));
  });
}

dk_status dk_deann_combine(int64_t nq, int32_t family, double bandwidth, int32_t k, int32_t m, int64_t n_total,
                           const double* nbr_d2, const double* z1_l1_sum, const double* z2_sum, double* value_out,
                           void* stream) {
  DK_NVTX();
  return guard([&] {
    check_family_bw(family, bandwidth);
    DK_REQUIRE(nq >= 0 && k >= 0 && m >= 0 && int64_t(k) <= n_total, "bad k / m / n");
    if (nq == 0) return;
    DK_REQUIRE(value_out != nullptr && is_device_ptr(value_out), "value_out must be device memory");
    DK_REQUIRE(k == 0 || (family == DK_LAPLACIAN ? z1_l1_sum != nullptr : nbr_d2 != nullptr), "NULL Z1 input");
    DK_REQUIRE(m == 0 || z2_sum != nullptr, "NULL z2_sum");
    launch_deann_combine(nq, family, bandwidth, k, m, n_total, nbr_d2, z1_l1_sum, z2_sum, value_out,
                         static_cast<cudaStream_t>(stream));
  });
}

dk_status dk_rsp_attach(dk_handle h, const int64_t* inverse_permutation) {
  DK_NVTX();
  return guard([&] {
    DK_REQUIRE(h != nullptr && inverse_permutation != nullptr, "NULL argument");
    DeviceGuard g(h->device);
    if (!h->rsp_inverse) DK_CUDA(cudaMalloc(&h->rsp_inverse, size_t(h->n) * sizeof(int64_t)));
    DK_CUDA(cudaMemcpy(h->rsp_inverse, inverse_permutation, size_t(h->n) * sizeof(int64_t), cudaMemcpyDefault));
  });
}

dk_status dk_rsp_walk(dk_handle h, const double* Q, int64_t nq, int32_t family, double bandwidth, int32_t m,
                      const int64_t* excl, int32_t excl_stride, int64_t cursor_in, int32_t independent,
                      double* z_sum, int32_t* taken, int64_t* cursor_out, void* stream) {
  DK_NVTX();
  return guard([&] {
    DK_REQUIRE(h != nullptr, "NULL handle");
    check_family_bw(family, bandwidth);
    DK_REQUIRE(m >= 1, "m=" + std::to_string(m) + " must be >= 1");
    DK_REQUIRE(cursor_in >= 0 && cursor_in < h->n, "cursor out of range [0, n)");
    DK_REQUIRE(!excl || (excl_stride >= 1 && excl_stride < h->n), "exclusion list must hold 1..n-1 ids");
    DK_REQUIRE(!excl || h->rsp_inverse != nullptr, "dk_rsp_attach must be called before excluding ids");
    DK_REQUIRE(nq >= 0, "negative query count");
    if (cursor_out) *cursor_out = cursor_in;
    if (nq == 0) return;
    DK_REQUIRE(Q != nullptr && z_sum != nullptr, "NULL argument");
    DeviceGuard g(h->device);
    LaunchCount lc(h);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const int32_t cnt = excl ? excl_stride : 0;
    Plan pl;
    const size_t o_Q = pl.add<double>(size_t(nq) * h->d);
    const size_t o_ex = pl.add<int64_t>(size_t(nq) * std::max(cnt, 1));
    const size_t o_pos = pl.add<int64_t>(size_t(nq) * std::max(cnt, 1));
    const size_t o_start = pl.add<int64_t>(size_t(nq));
    const size_t o_len = pl.add<int64_t>(size_t(nq));
    const size_t o_taken = pl.add<int32_t>(size_t(nq));
    const size_t o_z = pl.add<double>(size_t(nq));
    const size_t o_cur = pl.add<int64_t>(1);
    const bool long_excl = cnt > kSmemSortMax;
    const size_t seg_bytes = long_excl ? seg_sort_temp_bytes(cnt, nq) : 0;
    const size_t o_seg = pl.add<uint8_t>(seg_bytes);
    h->ws.reserve(pl.off);
    const double* Qd = stage_queries(h, Q, nq, o_Q, s);
    int64_t* pos = nullptr;
    if (excl) {
      int64_t* ex = at<int64_t>(h->ws, o_ex);
      DK_CUDA(cudaMemcpyAsync(ex, excl, size_t(nq) * cnt * sizeof(int64_t), cudaMemcpyDefault, s));
      pos = at<int64_t>(h->ws, o_pos);
      if (long_excl) {  // ids -> positions in place, then a segmented radix sort
        launch_gather_positions(ex, h->rsp_inverse, nq * cnt, ex, s);
        launch_seg_sort_i64(ex, pos, nullptr, cnt, nq, at<uint8_t>(h->ws, o_seg), seg_bytes, s);
      } else {
        launch_rsp_map_sort(ex, cnt, h->rsp_inverse, nq, pos, s);
      }
    }
    int64_t* start = at<int64_t>(h->ws, o_start);
    int64_t* len = at<int64_t>(h->ws, o_len);
    int32_t* tk = at<int32_t>(h->ws, o_taken);
    int64_t* cur = at<int64_t>(h->ws, o_cur);
    launch_rsp_starts(pos, cnt, nq, h->n, m, cursor_in, independent != 0, start, len, tk, cur, s);
    const bool z_dev = is_device_ptr(z_sum);
    double* zd = z_dev ? z_sum : at<double>(h->ws, o_z);
    {
      ProfScope ps(h, s, 0.0, double(nq) * m * h->d * 4.0, 2);
      launch_rsp_eval(h->X, h->n, h->d, Qd, nq, family, bandwidth, pos, cnt, start, len, zd, s);
    }
    if (!z_dev) copy_out(z_sum, zd, size_t(nq) * sizeof(double), s);
    if (taken) copy_out(taken, tk, size_t(nq) * sizeof(int32_t), s);
    if (cursor_out && !independent) copy_out(cursor_out, cur, sizeof(int64_t), s);
    DK_CUDA(cudaStreamSynchronize(s));
  });
}

dk_status dk_set_profiling(dk_handle h, int32_t on) {
  return guard([&] {
    DK_REQUIRE(h != nullptr, "NULL handle");
    DK_REQUIRE(on >= 0 && on <= 2, "profiling mode must be 0 (off), 1 (tile sweep) or 2 (sampling gather)");
    h->profiling = on;
    h->prof_used = 0;
  });
}

dk_status dk_last_kernel_ms(dk_handle h, double* ms, double* flops, double* bytes) {
  return guard([&] {
    DK_REQUIRE(h != nullptr, "NULL handle");
    DeviceGuard g(h->device);
    double tot = 0.0;
    for (size_t i = 0; i < h->prof_used; ++i) {
      DK_CUDA(cudaEventSynchronize(h->prof_events[i].second));
      float t = 0.f;
      DK_CUDA(cudaEventElapsedTime(&t, h->prof_events[i].first, h->prof_events[i].second));
      tot += t;
    }
    if (ms) *ms = h->prof_used ? tot / double(h->prof_used) : 0.0;
    if (flops) *flops = h->last_flops;
    if (bytes) *bytes = h->last_bytes;
  });
}

dk_status dk_sweep_probe(dk_handle h, const double* Q, int64_t nq, int32_t mode, int32_t encoding, double* ms) {
  DK_NVTX();
  return guard([&] {
    DK_REQUIRE(h != nullptr && Q != nullptr && ms != nullptr && nq > 0, "bad probe arguments");
    DK_REQUIRE(mode >= MODE_KDE_GAUSS && mode <= MODE_KDE_GAUSS_MUFU && encoding >= 0 && encoding <= 2, "bad probe mode");
    DeviceGuard g(h->device);
    cudaStream_t s = nullptr;
    const Encoding& e = ensure_encoding(h, encoding, s);
    const int32_t nq_pad = int32_t(query_pad(nq));
    Plan pl;
    const size_t o_Q = pl.add<double>(size_t(nq) * h->d);
    const size_t o_A = pl.add<__half>(size_t(nq_pad) * e.Kp);
    const size_t o_qn = pl.add<float>(nq_pad);
    const size_t o_scal = pl.add<float>(4);
    const size_t o_part = pl.add<double>(sweep_part_count(h->n_pad, nq_pad, h->num_sms));
    const size_t o_tmin = pl.add<float>(size_t(nq_pad) * 4 * size_t(h->n_pad / kBN));
    const size_t o_tau = pl.add<float>(nq_pad);
    const size_t o_cnt = pl.add<uint32_t>(nq_pad);
    const size_t o_cand = pl.add<unsigned long long>(size_t(nq_pad) * 64);
    h->ws.reserve(pl.off);
    const double* Qd = stage_queries(h, Q, nq, o_Q, s);
    QueryOperand q = encode_queries(h, e, Qd, nq, nq_pad, at<__half>(h->ws, o_A), at<float>(h->ws, o_qn),
                                    at<float>(h->ws, o_scal), s);
    SweepArgs a{};
    a.mode = mode;
    a.qop = &q;
    a.enc = &e;
    a.n = h->n;
    a.n_pad = h->n_pad;
    a.tile_stride = 1;
    a.negc = -1e-3f;
    a.part = at<double>(h->ws, o_part);
    a.tmin = at<float>(h->ws, o_tmin);
    a.seg_tiles = 0;
    a.tau = at<float>(h->ws, o_tau);
    launch_fill_float(at<float>(h->ws, o_tau), nq_pad, -1.f, s);
    a.cand_cnt = at<uint32_t>(h->ws, o_cnt);
    a.cand = at<unsigned long long>(h->ws, o_cand);
    a.cap = 64;
    cudaEvent_t e0, e1;
    DK_CUDA(cudaEventCreate(&e0));
    DK_CUDA(cudaEventCreate(&e1));
    launch_sweep(a, h->num_sms, s);  // warm
    DK_CUDA(cudaEventRecord(e0, s));
    launch_sweep(a, h->num_sms, s);
    DK_CUDA(cudaEventRecord(e1, s));
    DK_CUDA(cudaEventSynchronize(e1));
    float t = 0.f;
    DK_CUDA(cudaEventElapsedTime(&t, e0, e1));
    *ms = t;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
  });
}

dk_status dk_knn_stats(dk_handle h, int64_t* queries, int64_t* cand_sum, int64_t* cand_max, int64_t* fallbacks) {
  return guard([&] {
    DK_REQUIRE(h != nullptr, "NULL handle");
    if (queries) *queries = h->knn_queries;
    if (cand_sum) *cand_sum = h->knn_cand_sum;
    if (cand_max) *cand_max = h->knn_cand_max;
    if (fallbacks) *fallbacks = h->knn_fallbacks;
  });
}

dk_status dk_kde_stats(dk_handle h, int64_t* queries, int64_t* fallbacks, int64_t* hot_pairs, int64_t* total_pairs) {
  return guard([&] {
    DK_REQUIRE(h != nullptr, "NULL handle");
    DeviceGuard g(h->device);
    if (queries) *queries = h->hyb_queries;
    if (fallbacks) *fallbacks = h->hyb_fallbacks;
    int64_t hot = -1, tot = -1;
    if (h->kc != nullptr && h->kc->hyb_stat_host != nullptr && h->kc->hyb_stat_total > 0) {
      DK_CUDA(cudaEventSynchronize(h->kc->hyb_stat_ev));
      hot = h->kc->hyb_stat_host[0];
      tot = int64_t(h->kc->hyb_stat_total);
    }
    if (hot_pairs) *hot_pairs = hot;
    if (total_pairs) *total_pairs = tot;
  });
}

dk_status dk_kde_redo_count(dk_handle h, int64_t* count) {
  return guard([&] {
    DK_REQUIRE(h != nullptr && count != nullptr, "NULL argument");
    DeviceGuard g(h->device);
    int64_t c = 0;
    if (h->redo_mask) {
      DK_CUDA(cudaEventSynchronize(h->redo_event));
      for (int i = 0; i < 2; ++i)
        if (h->redo_mask & (1 << i)) c += h->redo_host[i];
    }
    *count = c;
  });
}

dk_status dk_last_launch_count(dk_handle h, int64_t* count) {
  return guard([&] {
    DK_REQUIRE(h != nullptr && count != nullptr, "NULL argument");
    *count = h->launches;
  });
}

// ---- page-locked host result buffers: power-of-two size classes, cached
namespace {
struct HostCache {
  std::mutex mu;
  std::map<void*, size_t> live;                  // pointer -> class bytes
  std::multimap<size_t, void*> free_blocks;      // class bytes -> pointer
  size_t cached = 0;
};
HostCache& host_cache() {
  static HostCache* c = new HostCache;  // never destroyed: blocks may be freed at exit
  return *c;
}
}  // namespace

dk_status dk_host_alloc(int64_t bytes, void** out) {
  DK_NVTX();
  return guard([&] {
    DK_REQUIRE(out != nullptr && bytes >= 0, "bad argument");
    size_t cls = 4096;
    while (cls < size_t(bytes)) cls <<= 1;
    HostCache& c = host_cache();
    {
      std::lock_guard<std::mutex> lk(c.mu);
      auto it = c.free_blocks.find(cls);
      if (it != c.free_blocks.end()) {
        *out = it->second;
        c.free_blocks.erase(it);
        c.cached -= cls;
        c.live[*out] = cls;
        return;
      }
    }
    void* p = nullptr;
    DK_CUDA(cudaHostAlloc(&p, cls, cudaHostAllocPortable));
    std::lock_guard<std::mutex> lk(c.mu);
    c.live[p] = cls;
    *out = p;
  });
}

dk_status dk_host_free(void* p) {
  return guard([&] {
    if (p == nullptr) return;
    HostCache& c = host_cache();
    size_t cls = 0;
    {
      std::lock_guard<std::mutex> lk(c.mu);
      auto it = c.live.find(p);
      DK_REQUIRE(it != c.live.end(), "dk_host_free: not a dk_host_alloc buffer");
      cls = it->second;
      c.live.erase(it);
      if (c.cached + cls <= (size_t(1) << 30)) {
        c.free_blocks.emplace(cls, p);
        c.cached += cls;
        return;
      }
    }
    DK_CUDA(cudaFreeHost(p));
  });
}

}  // extern "C"
