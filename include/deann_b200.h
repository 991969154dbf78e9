/*
 * deann_b200.h — C-ABI of the B200-native DEANN KDE query path.
 *
 * This is the drop-in boundary under the Python estimator API of the
 * reference package `deann` (arXiv 2107.02736).  The reference is pure
 * Python/NumPy and has no FFI of its own; each entry point below names the
 * reference function whose contract it implements (paths relative to
 * /root/reference/pkg/src/deann/).  The binding a maintainer would add to the
 * reference package is shown in INTEGRATION.md (ctypes).
 *
 * Conventions
 *   - Plain pointers and sizes only.  Every array pointer may be HOST or
 *     DEVICE memory; the library inspects it (cudaPointerGetAttributes) and
 *     stages host arrays through its own device workspace.  Outputs follow
 *     the same rule.
 *   - Row-major, C-contiguous.  Dataset rows are fp32 (reference Dataset
 *     stores float32, data.py:55); queries are fp64 (the reference casts
 *     queries to float64, estimators.py:129,156,333).
 *   - `stream` is a cudaStream_t passed as void* (NULL = legacy default).
 *     Calls are stream-ordered; when any output pointer is host memory the
 *     call synchronises the stream before returning.
 *   - Every function returns a dk_status; on failure dk_last_error() returns
 *     a thread-local message.  Argument errors (DK_EINVAL) are raised for
 *     exactly the preconditions the reference raises ValueError for.
 *   - A handle is read-only after dk_fit; concurrent calls on one handle
 *     must use distinct handles (the workspace is per handle).
 */
#ifndef DEANN_B200_H
#define DEANN_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  DK_OK = 0,
  DK_EINVAL = 1,    /* argument/range/dimension error  -> ValueError          */
  DK_ECUDA = 2,     /* CUDA runtime/driver failure     -> RuntimeError        */
  DK_ENOMEM = 3,    /* device allocation failed        -> MemoryError         */
  DK_EINEXACT = 4,  /* k-NN certificate failed (see dk_knn)                   */
  DK_ENODEV = 5,    /* no sm_100 device                                       */
  DK_EFORMAT = 6,   /* malformed dataset file          -> DatasetFormatError  */
  DK_EIO = 7        /* file open/read failure          -> OSError             */
} dk_status;

/* Kernel families, same order/meaning as kernels.py:22-39
 * (gaussian -> squared L2, exponential -> L2, laplacian -> L1). */
typedef enum {
  DK_GAUSSIAN = 0,
  DK_EXPONENTIAL = 1,
  DK_LAPLACIAN = 2
} dk_family;

/* Operand precision for the tensor-core distance tile (dk_fit_opts.precision). */
typedef enum {
  DK_PREC_AUTO = 0,    /* exact fp16 when rows and queries are small integers, else split3 */
  DK_PREC_SPLIT3 = 1,  /* fp16 hi/lo, K-concatenated [Qh|Ql|Qh]x[Xl|Xh|Xh] (~2^-22 rel)   */
  DK_PREC_FP16 = 2     /* single-pass fp16 (fast, ~1e-3..1e-5 rel; opt-in only)           */
} dk_precision;

typedef struct dk_dataset* dk_handle;

typedef struct {
  int32_t device;        /* CUDA device ordinal                                   */
  int32_t precision;     /* dk_precision                                          */
  int64_t global_offset; /* dataset-sharded mode: global index of local row 0     */
  int64_t global_n;      /* dataset-sharded mode: total rows over all shards (0 = n) */
} dk_fit_opts;

/* Flags for dk_naive / dk_sample. */
#define DK_OUT_SUM 1u    /* write per-query kernel SUMS (fp64) instead of means  */

/* ---- version / errors ---------------------------------------------------- */
int32_t dk_version(void);
const char* dk_last_error(void);
int32_t dk_device_ok(int32_t device);   /* 1 if `device` is sm_100 (B200) */

/* ---- fit ------------------------------------------------------------------
 * Replaces Dataset.from_array + data64() + sq_norms (data.py:53-83) and
 * BruteForceIndex(ds) (ann.py:114-118): copies X (n x d fp32) to the device,
 * validates finiteness (ValueError at data.py:61-62), computes fp64 row norms
 * (data.py:63-64) and the tensor-core operand encodings. */
dk_status dk_fit(const float* X, int64_t n, int32_t d, const dk_fit_opts* opts,
                 dk_handle* out);
dk_status dk_free(dk_handle h);

/* ---- load -----------------------------------------------------------------
 * The DEANN1 binary format of data.py:1-15 (magic "DEANN1\0\0", u32 n, u32 d,
 * n*d little-endian fp32, row-major).  dk_file_info validates the header and
 * the payload size exactly as _load_binary (data.py:151-167) does, with the same
 * messages (DK_EFORMAT).  dk_fit_file streams rows [row_begin, row_begin +
 * row_count) of the file (row_count < 0: to the end) through pinned staging
 * buffers straight into device memory — parallel pread threads overlapped with
 * the host->device copies — and then fits like dk_fit.  Loading a proper row
 * range without opts->global_n makes the handle a dataset shard whose global ids
 * are the file's row ids (global_offset = row_begin, global_n = file n). */
dk_status dk_file_info(const char* path, int64_t* n, int32_t* d);
dk_status dk_fit_file(const char* path, int64_t row_begin, int64_t row_count,
                      const dk_fit_opts* opts, dk_handle* out);
dk_status dk_info(dk_handle h, int64_t* n, int32_t* d, int64_t* global_offset,
                  int64_t* global_n, int32_t* exact_mode);
/* fp64 squared row norms (n), cf. Dataset.sq_norms (data.py:64). */
dk_status dk_sq_norms(dk_handle h, double* out, void* stream);

/* ---- exact KDE ------------------------------------------------------------
 * naive_kde (estimators.py:122-149): out[j] = (1/n) sum_i K_h(q_j, x_i), fp64.
 * Gaussian/exponential run the fused tcgen05 distance-tile + exp + row-sum;
 * laplacian runs the CUDA-core L1 kernel.  With DK_OUT_SUM the un-normalised
 * local sum is written; without it the sum is divided by the GLOBAL row count
 * (global_n of a shard handle, n otherwise), so the shards' outputs all-reduce
 * (sum) straight to the KDE. */
dk_status dk_naive(dk_handle h, const double* Q, int64_t nq, int32_t family,
                   double bandwidth, uint32_t flags, double* out, void* stream);

/* ---- materialised distances ---------------------------------------------
 * batch_sqdist / window_sqdist (distance.py:58-123): out[j][i] (nq x row_count,
 * fp64) = max(0, ((q_j . x_i) * -2 + |q_j|^2) + |x_i|^2) for rows i in
 * [row_begin, row_begin + row_count), the reference's norms identity in fp64.
 * x_norms (nullable, n fp64) overrides the handle's norms (a caller's cached
 * sq_norms).  *worst = the most negative entry before clamping, for the
 * NormConsistencyError check of _clamp (distance.py:54-64). */
dk_status dk_sqdist(dk_handle h, const double* Q, int64_t nq, const double* x_norms,
                    int64_t row_begin, int64_t row_count, double* out, double* worst,
                    void* stream);

/* ---- exact k-NN -----------------------------------------------------------
 * brute_force_knn (ann.py:105-111) / BruteForceIndex.query (ann.py:120-121)
 * for a batch: idx_out (nq x k, int64, GLOBAL row ids), d2_out (nq x k, fp64
 * squared L2 by direct difference), each row sorted by (d2, idx) — ties to the
 * lower index as in _smallest_k (ann.py:82-102).  Requires 1 <= k <= n
 * (ValueError at ann.py:107-108).  Candidates are selected on tensor-core
 * distance tiles and re-ranked exactly in fp64; a per-query certificate
 * proves the set; DK_EINEXACT if it could not be proven (never observed). */
dk_status dk_knn(dk_handle h, const double* Q, int64_t nq, int32_t k,
                 int64_t* idx_out, double* d2_out, void* stream);

/* Merge of per-shard top-k lists for dataset-sharded mode: `parts` lists of
 * (idx, d2) per query laid out [part][query][k], each sorted by (d2, idx);
 * writes the global top-k.  Pure device work. */
dk_status dk_merge_topk(int32_t parts, int64_t nq, int32_t k,
                        const int64_t* idx_in, const double* d2_in,
                        int64_t* idx_out, double* d2_out, void* stream);

/* ---- sampling (RS / DEANN residual) ---------------------------------------
 * rs_kde (estimators.py:152-164) and _rs_excluding (estimators.py:203-233):
 * for query j, draw t = 0,1,2,... gives row
 *   r_t = mulhi64(philox4x32_10(key=seed, ctr={t, j+query_base, 0, 0}) as u64, N)
 * over the GLOBAL index space N (= global_n); the first m draws NOT in the
 * exclusion list excl[j*excl_stride .. +excl_cnt[j]) (any order) are accepted
 * ("first m accepted of the stream" = the reference's effective rule).  For
 * accepted rows inside this shard the kernel value is computed in fp64 (direct
 * difference) and summed: z_sum[j].  Optionally exports accepted row ids
 * (nq x m) and the number of draws consumed per query.  excl may be NULL
 * (plain RS).  m >= 1. */
dk_status dk_sample(dk_handle h, const double* Q, int64_t nq, int32_t family,
                    double bandwidth, int32_t m, uint64_t seed, int64_t query_base,
                    const int64_t* excl, const int32_t* excl_cnt, int32_t excl_stride,
                    double* z_sum, int64_t* accepted_idx_out, int64_t* draws_out,
                    void* stream);

/* Kernel sums over explicit rows: out[j] = sum_{c<cnt} K(q_j, x_rows[j*stride+c]),
 * fp64 direct difference (cf. _kernel_rows, estimators.py:106-119).  Rows are
 * GLOBAL ids; rows outside this shard contribute 0.  Used for Z1 of the
 * laplacian family (estimators.py:346-348) and for parity with explicit ids. */
dk_status dk_eval_rows(dk_handle h, const double* Q, int64_t nq, int32_t family,
                       double bandwidth, const int64_t* rows, const int32_t* cnt,
                       int32_t stride, double* out, void* stream);

/* kernel_from_distance (kernels.py:65-83) on the device: out[i] =
 * exp(-dist[i]/(2h^2)) for gaussian (dist = squared L2), exp(-dist[i]/h) for
 * exponential (L2) and laplacian (L1); fp64.  Non-finite or negative
 * distances -> DK_EINVAL (kernels.py:74-77). */
dk_status dk_kernel_values(int32_t family, double bandwidth, const double* dist, int64_t count, double* out,
                           void* stream);

/* ---- DEANN (single GPU, whole dataset) -------------------------------------
 * deann (estimators.py:306-379) with ann = exact brute force and the uniform
 * sampler, batched over nq queries (deann_batch, estimators.py:382-410):
 *   value = (k/n) Z1 + ((n-k)/n) Z2,  Z1 from the exact neighbour distances
 * (L2 families, estimators.py:349-351) or recomputed L1 (laplacian, :346-348).
 * k == 0 -> pure RS (no k-NN); m == 0 -> truncated (k/n) Z1.  Preconditions as
 * estimators.py:322-335.  Optional exports: neighbours (nq x k), accepted
 * sample ids (nq x m). */
dk_status dk_deann(dk_handle h, const double* Q, int64_t nq, int32_t family,
                   double bandwidth, int32_t k, int32_t m, uint64_t seed,
                   int64_t query_base, double* value_out, int64_t* nbr_idx_out,
                   double* nbr_d2_out, int64_t* sample_idx_out, void* stream);

/* The DEANN combination step alone (estimators.py:344-372), for callers that
 * assemble the parts themselves — dataset-sharded mode after its collectives
 * (sharded.py): per query j, Z1 = mean over the k neighbours of kernel(nbr_d2)
 * (L2 families, estimators.py:349-351) or z1_l1_sum[j] / k (laplacian,
 * :346-348), Z2 = z2_sum[j] / m, value = (k/n_total) Z1 + ((n_total-k)/n_total) Z2.
 * All arrays are DEVICE memory (nbr_d2 nq x k, the others nq); nullable when
 * unused (z1_l1_sum unless laplacian, z2_sum when m == 0).  Same arithmetic as
 * dk_deann's final step. */
dk_status dk_deann_combine(int64_t nq, int32_t family, double bandwidth, int32_t k,
                           int32_t m, int64_t n_total, const double* nbr_d2,
                           const double* z1_l1_sum, const double* z2_sum,
                           double* value_out, void* stream);

/* ---- permuted sampler (RSP / DEANNP) -----------------------
 * RspState (estimators.py:83-96) on the device: `h` is a dataset fitted on the
 * PERMUTED rows (row i = original row permutation[i], permute data.py:214-233);
 * attach its inverse permutation (original id -> permuted position, n int64). */
dk_status dk_rsp_attach(dk_handle h, const int64_t* inverse_permutation);

/* Permuted-window sampler over a query batch: rsp_kde (estimators.py:180-200),
 * _rsp_excluding (:249-303) and deann_batch's cursor threading (:394-409).
 * Query j walks the permuted rows from its start, skipping rows whose ORIGINAL id
 * is in excl[j*excl_stride ..+excl_stride) (nullable), until m rows are accepted
 * or one full pass completes.  Starts: independent != 0 -> floor(j*n/nq)
 * (independent_cursors=True); else start_0 = cursor_in, start_{j+1} = start_j +
 * rows consumed by query j (mod n).  Outputs: z_sum[j] = fp64 kernel sum over the
 * accepted rows, taken[j] = accepted count (< m: clamped to one full pass),
 * *cursor_out = the shared cursor after the batch (cursor_in if independent). */
dk_status dk_rsp_walk(dk_handle h, const double* Q, int64_t nq, int32_t family, double bandwidth,
                      int32_t m, const int64_t* excl, int32_t excl_stride, int64_t cursor_in,
                      int32_t independent, double* z_sum, int32_t* taken, int64_t* cursor_out,
                      void* stream);

/* ---- inverted-file index --------------------------------
 * ivf_build / ivf_query / IvfAnnIndex (ann.py:124-316) over a fitted dataset.
 * The host keeps the reference's numpy PCG64 stream and drives k-means++ one
 * centroid at a time (ann.py:152-169):
 *   dk_kmeanspp_seed(c, row): centroid c = row; closest = D^2 to centroid 0
 *     (c == 0) or min(closest, D^2 to c); *total = sum(closest)
 *   dk_kmeanspp_pick(u, total): rng.choice(n, p=closest/total) given its one
 *     uniform draw u: searchsorted(cumsum(p) / cumsum(p)[-1], u, 'right')
 * dk_kmeans_lloyd runs the Lloyd loop of ivf_build (ann.py:184-198, fp64 norms
 * identity, argmin ties -> lower centroid, sequential member means, empty
 * clusters kept) plus the final assignment, and lays the rows out cluster-
 * contiguously (IvfAnnIndex, ann.py:244-252).  dk_ivf_get copies centroids
 * (C x d fp64), list rows (n, increasing id within a list) and offsets (C + 1);
 * dk_ivf_set installs an existing index (a reference IvfIndex or a loaded one).
 * dk_ivf_query: for each query the n_probe nearest centroids ((d2, id) order;
 * formula 0 = sum (c - y)^2 as ivf_query, 1 = (C y) * -2 + |c|^2 as
 * IvfAnnIndex) and the exact k smallest d2 = ((x.y) * -2 + |x|^2) + |y|^2
 * (clamped at 0) over their members, (d2, row) order; cnt[j] = min(k, members
 * probed), unused slots idx -1 / d2 +inf; any k >= 1 (k > 4096 sorts every
 * probed candidate); any n_clusters (beyond 8192 the probe is a segmented sort). */
typedef struct dk_ivf* dk_ivf_handle;
dk_status dk_ivf_create(dk_handle h, int32_t n_clusters, dk_ivf_handle* out);
dk_status dk_ivf_free(dk_ivf_handle ivf);
dk_status dk_kmeanspp_seed(dk_ivf_handle ivf, int32_t c, int64_t row, double* total);
dk_status dk_kmeanspp_pick(dk_ivf_handle ivf, double u, double total, int64_t* row);
dk_status dk_kmeans_lloyd(dk_ivf_handle ivf, int32_t max_iter, double rel_tol, int32_t* iters);
dk_status dk_ivf_get(dk_ivf_handle ivf, double* centroids, int64_t* rows, int64_t* offsets);
dk_status dk_ivf_set(dk_ivf_handle ivf, const double* centroids, const int64_t* rows,
                     const int64_t* offsets);
dk_status dk_ivf_query(dk_ivf_handle ivf, const double* Q, int64_t nq, int32_t k, int32_t n_probe,
                       int32_t formula, int64_t* idx_out, double* d2_out, int32_t* cnt_out,
                       void* stream);
/* DEANN over a query batch with the IVF index as the ANN (estimators.py:306-379 with an
 * IvfAnnIndex, ann.py:276-316): per query the k^ <= k probed neighbours of dk_ivf_query
 * (formula 1), Z1 = mean kernel over them (L2 families from their d2; laplacian re-evaluated
 * in L1, estimators.py:346-351), Z2 = mean kernel over the first m Philox draws outside
 * them (dk_sample's stream), value = (k^/n) Z1 + ((n-k^)/n) Z2.  value_out[nq] and
 * khat_out[nq] (optional) may be host or device memory. */
dk_status dk_deann_ivf(dk_ivf_handle ivf, const double* Q, int64_t nq, int32_t family, double bandwidth,
                       int32_t k, int32_t m, int32_t n_probe, uint64_t seed, int64_t query_base,
                       double* value_out, int32_t* khat_out, void* stream);

/* Timing support for bench.py: average device duration (ms) of the LAST launch
 * of the dominant kernel of the last call on this handle (CUDA events on the
 * launching stream) and its algorithmic work. */
dk_status dk_last_kernel_ms(dk_handle h, double* ms, double* flops, double* bytes);
/* on: 0 = off, 1 = time the tile sweeps (KDE / k-NN distance tiles), 2 = time the
 * sampling gathers (RS / DEANN residual estimators). */
dk_status dk_set_profiling(dk_handle h, int32_t on);
/* k-NN diagnostics accumulated on this handle (counted when DK_KNN_STATS is set
 * in the environment at fit time; fallbacks always): queries, total and max
 * candidates per query, queries that took the exact-scan fallback. */
dk_status dk_knn_stats(dk_handle h, int64_t* queries, int64_t* cand_sum, int64_t* cand_max,
                       int64_t* fallbacks);
/* Exact-KDE diagnostics of this handle's two-precision path (dk_naive, gaussian, non-integer
 * rows): queries it served, queries whose fp16 bound failed and were recomputed in split3, and
 * the hot (query block, tile) pairs / all pairs of the last call's first batch (-1: not yet
 * known).  No reference counterpart. */
dk_status dk_kde_stats(dk_handle h, int64_t* queries, int64_t* fallbacks, int64_t* hot_pairs, int64_t* total_pairs);
/* Queries of the last dk_naive call on this handle that the guard of the split3 sweeps recomputed
 * in fp64 direct differences, as the reference evaluates every pair (naive_kde estimators.py:144-149):
 * exponential-kernel queries with a row closer than the distance under which the sweep's d2 error
 * could move exp(-sqrt(d2)/h) by more than 1e-4, gaussian queries whose d2 error bound exceeds
 * 5e-5 x 2h^2, and (these and the laplacian kernel) queries whose KDE came back under 1e-30, below the
 * fp32 epilogue's range.  Integer datasets in exact mode are not guarded.
 * Waits for that call's work.  No reference counterpart. */
dk_status dk_kde_redo_count(dk_handle h, int64_t* count);
/* Diagnostics: time (ms, CUDA events) of one tile sweep of the given mode
 * (0 KDE-gauss, 1 KDE-exp, 2 segment-min, 3 filter, 4 null epilogue) with the
 * given operand encoding (0 exact, 1 split3, 2 fp16) — a pipeline probe. */
dk_status dk_sweep_probe(dk_handle h, const double* Q, int64_t nq, int32_t mode, int32_t encoding,
                         double* ms);
/* Measured SFU exp2 throughput of `device` (ex2.approx.ftz.f32 per second, all SMs):
 * the MUFU denominator of the exact-KDE roofline (no reference counterpart). */
dk_status dk_mufu_probe(int32_t device, double* ex2_per_second);

/* Number of this library's kernels launched by the last API call. */
dk_status dk_last_launch_count(dk_handle h, int64_t* count);

/* Page-locked host buffers for results (no reference counterpart: host plumbing of the
 * Python layer).  dk_host_alloc returns a buffer of >= bytes from a size-class cache of
 * cudaHostAlloc blocks (a new block only when the cache has none); dk_host_free returns
 * it to the cache (blocks beyond 1 GiB of cached memory are released).  Device->host
 * copies of results into such buffers run at full DMA speed. */
dk_status dk_host_alloc(int64_t bytes, void** out);
dk_status dk_host_free(void* p);

#ifdef __cplusplus
}
#endif
#endif /* DEANN_B200_H */
