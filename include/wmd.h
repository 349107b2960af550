/*
 * wmd.h — C ABI of the B200-native sparse Sinkhorn Word Mover's Distance library
 * (libwmd_b200.so), implementing the hot path of arXiv 2005.06727
 * ("Parallel sparse Sinkhorn-Knopp WMD", PAPER.md in the reference tree).
 *
 * One query document r against N target documents c at once:
 *
 *   I=(r>0); r=r(I); M=M(I,:); K=exp(-lambda*M)            Algorithm 1 l.1
 *   x = ones(v_r, N)/v_r                                    Algorithm 1 l.2
 *   repeat iters times:  x = diag(1./r) K (c .* 1./(K^T (1./x)))   l.3-5
 *        evaluated sparsely as the fused SDDMM_SpMM kernel
 *   u = 1./x; v = c .* 1./(K^T u); WMD = sum_i u .* ((K.*M) v)     l.6-7
 *
 * M is the v_r x V Euclidean distance between the query words' embeddings and every
 * vocabulary embedding ("m(i,j) = sqrt(sum(pow(embedding[i]-embedding[j],2)))").
 *
 * Numerics: all device arithmetic is FP32 except the FP64 fallback. K is stored
 * column-rescaled, K~_ki = exp(-lambda (M_ik - min_i' M_i'k)), and u carries an exact per-document
 * power-of-two gauge; both leave u, the transport plan and every WMD unchanged in exact
 * arithmetic. Documents whose FP32 iterates leave the normal range are recomputed in FP64 on the
 * GPU. There is no CPU fallback: every compute step runs in CUDA kernels.
 *
 * Conventions
 *  - Every function returns a wmd_status; WMD_OK == 0. No function aborts or prints.
 *  - Pointers documented "host or device" are classified with cudaPointerGetAttributes.
 *  - Array arguments are copied into handle-owned device memory before the call returns;
 *    the caller may free them on return. Exception: out_dist (see wmd_query).
 *  - A handle is used by one host thread at a time; handles are independent; there is no
 *    global mutable state.
 *  - Indices are 0-based. c is a V x N matrix stored CSC (= document-major, one column per
 *    target document), the doc-major reading of the paper's "CSR" (reading R12).
 */
#ifndef WMD_B200_H
#define WMD_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#define WMD_API __attribute__((visibility("default")))
#else
#define WMD_API
#endif

#define WMD_MAX_VR 128          /* maximum distinct query words v_r per query */
#define WMD_MAX_V (1 << 24)     /* maximum vocabulary size (V * WMD_MAX_VR < 2^31: 32-bit row offsets) */

typedef struct wmd_handle wmd_handle; /* opaque; one per GPU / rank */

typedef enum {
  WMD_OK = 0,
  WMD_ERR_INVALID_ARGUMENT = 1,   /* bad size / NULL / lambda<=0 / iters<0 / v_r out of [1,WMD_MAX_VR] */
  WMD_ERR_INDEX_OUT_OF_RANGE = 2, /* a word id not in [0, V) */
  WMD_ERR_EMPTY_DOCUMENT = 3,     /* col_ptr[j] == col_ptr[j+1]; wmd_last_error names j */
  WMD_ERR_MALFORMED_CSC = 4,      /* col_ptr not starting at 0 / decreasing / != nnz; rows not strictly increasing */
  WMD_ERR_BAD_WEIGHTS = 5,        /* weight <= 0 or non-finite, |sum-1| > 1e-5 (FP64 sum), duplicate query id */
  WMD_ERR_NONFINITE_EMBEDDING = 6,/* NaN/Inf in vocab_emb */
  WMD_ERR_STATE = 7,              /* e.g. wmd_query before wmd_set_targets */
  WMD_ERR_NUMERICAL_BREAKDOWN = 8,/* deferred: a distance stayed non-finite even in FP64 */
  WMD_ERR_OUT_OF_MEMORY = 9,
  WMD_ERR_CUDA = 10               /* any other CUDA runtime error; wmd_last_error has the text */
} wmd_status;

/* Execution path of the Sinkhorn loop (wmd_set_option(WMD_OPT_PATH, ...)). */
typedef enum {
  WMD_PATH_AUTO = 0,       /* library choice: WMD_PATH_FUSED when it supports the shape (v_r <= 128,
                              every document <= 320 words; <= 64 words while a stopping tolerance is
                              set; lambda >= 1e-3, below which its final step's recovery of M from
                              the FP32 block loses accuracy), else WMD_PATH_PER_ITER */
  WMD_PATH_PER_ITER = 1,   /* one fused SDDMM_SpMM launch per iteration + final kernel */
  WMD_PATH_FUSED = 2       /* all iterations + final in one launch per length bucket, per-document
                              state on chip (one warp per document up to 64 words, one CTA per
                              document up to 320); WMD_ERR_INVALID_ARGUMENT if the shape is outside
                              the limits above */
} wmd_path;

typedef enum {
  WMD_OPT_PATH = 1,        /* wmd_path; default WMD_PATH_AUTO */
  WMD_OPT_TIMING = 2,      /* 1: record CUDA events per phase (read with wmd_get_stats); default 0 */
  WMD_OPT_FALLBACK = 3,    /* 1: FP64 re-run of flagged documents (default); 0: leave them flagged */
  WMD_OPT_GRAPH = 4,       /* 1: capture a query's launches (build, Sinkhorn, final, fallback) once
                              and replay them as a CUDA graph while the query width, lambda, iters,
                              tolerance, path, output pointer and buffers repeat (the query rows are
                              re-uploaded every call); per-phase timing is off in this mode.
                              Default 0 */
  WMD_OPT_BUILD = 5,       /* distance build (a2), a wmd_build value; default WMD_BUILD_EXACT where
                              available (dp <= 1280), else WMD_BUILD_DIRECT */
  WMD_OPT_BATCH = 7,       /* wmd_query_batch, queries per fused pass (NEXT-2 (ii)): 0 = automatic
                              (as many tables as fit in half the L2, at most 16; default),
                              1 = one query at a time, 2..64 = that many. Applies when every query
                              takes the one-warp kernel for every document, no tolerance is set and
                              graph mode is off; results are bitwise those of single queries */
  WMD_OPT_LAYOUT_DOC_NNZ = 6, /* >= 0: the path and table-width decision of every query assumes the
                              longest document has max(this, local longest) words. A document-
                              sharded run passes the GLOBAL longest document on every
                              rank, so all ranks pick the same path and row width (their tables
                              are then all-gatherable and their results bitwise equal to an
                              unsharded run). Default 0 (the local targets decide) */
  WMD_OPT_LAYOUT_DOCS = 8  /* >= 0: the fused kernels' choice assumes max(this, local N) target
                              documents: documents of <= 40 words run two per warp (half-warp
                              kernel) at table widths 16-40 on corpora of >= 32768 documents,
                              one per warp below. A document-sharded run passes the GLOBAL N on
                              every rank (same kernels, bitwise equal to an unsharded run).
                              Default 0 */
} wmd_option;

/* Distance build (a2) kernels, wmd_set_option(WMD_OPT_BUILD, ...). PAPER.md:259-268 (§6) compares
 * a dot-type and a GEMM-type distance kernel; both are here:
 *  WMD_BUILD_DIRECT: M_ik = sqrt(sum_t (E[sel_i,t] - E[k,t])^2) in FP32 SIMT (direct difference).
 *    Accurate for any embedding geometry (relative error of M ~1e-7); the default where
 *    WMD_BUILD_EXACT is unavailable.
 *  WMD_BUILD_TENSOR_CORE: M^2 = |e|^2 + |q|^2 - 2 e.q with e.q on the tcgen05 tensor cores in
 *    3xTF32, near pairs recomputed directly. Faster, but the expansion's absolute error
 *    ~eps (|e|^2 + |q|^2) reaches lambda*dM ~ 1e-2 on clustered embeddings of varied norm, where
 *    distances end up ~1e-4 off (R34); accurate on isotropic (N(0,1)-like) data.
 *  WMD_BUILD_EXACT: the same expansion in exact integer arithmetic on the tcgen05 tensor cores
 *    (kind::i8): at wmd_create E is rounded once to fixed point n = rint(E 2^F) with |n| <= 2^26
 *    (F from max|E|: about one FP32 ulp of the largest coordinates) and split into byte limbs;
 *    the limb products, their int64 combination and M^2 = (|n_k|^2 - n_k.n_q) + (|n_q|^2 - n_k.n_q)
 *    are exact, so M_{i,sel_i} = 0 and there is no cancellation for any geometry. Needs
 *    dp = d rounded up to 32 <= 1280 (wmd_set_option fails with WMD_ERR_INVALID_ARGUMENT
 *    otherwise); a query whose limbs do not fit in shared memory (dp * 128 B per 32 query rows,
 *    e.g. dp = 1280 with v_r > 32) is built by WMD_BUILD_DIRECT (see wmd_stats.last_build).
 *    Costs 4 * V * dp + 8 * V bytes of extra device memory per handle. The default. */
typedef enum {
  WMD_BUILD_TENSOR_CORE = 0,
  WMD_BUILD_DIRECT = 1,
  WMD_BUILD_EXACT = 2
} wmd_build;

typedef struct {
  int64_t queries;           /* wmd_query calls since create / wmd_reset_stats */
  int64_t iter_launches;     /* Sinkhorn-loop kernel launches (per-iteration path: iters per query) */
  int64_t kernel_launches;   /* all kernel launches issued by queries */
  int64_t fallback_docs;     /* documents recomputed in FP64, summed over queries (updated by wmd_sync) */
  int64_t flagged_docs;      /* documents of the last query flagged in FP32 (updated by wmd_sync) */
  int32_t last_v_r;
  int32_t last_ld;           /* row width (floats) of the K~ / M tables: v_r rounded up to 8 (per-iteration path); on the fused path 8 CW with CW in {1, 2, 3, 4, 5, 6, 8} when every document fits the one-warp kernel, else in {4, 5, 6, 8, 10, 12, 13, 16} */
  int32_t last_path;         /* wmd_path actually used by the last query */
  int32_t last_build;        /* wmd_build kernel that built the last query's distance table */
  int32_t timing_valid;      /* 1 if the *_ms fields below are populated (WMD_OPT_TIMING) */
  double build_ms;           /* distance + kernel build (step a2), summed over queries */
  double iter_ms;            /* Sinkhorn iterations (a4) */
  double final_ms;           /* final step (a5); 0 for the fused path (included in iter_ms) */
  double fallback_ms;        /* FP64 fallback (a6) */
  double query_ms;           /* whole device-side query */
} wmd_stats;

/* Create a handle on CUDA device `device` holding a copy of the embeddings.
 * vocab_emb: host or device, V x d FP32 row-major (the paper's `vecs`).
 * Errors: INVALID_ARGUMENT (NULL, V<1, d<1, V > WMD_MAX_V), NONFINITE_EMBEDDING, OUT_OF_MEMORY, CUDA.
 * On error *out is set to NULL. */
WMD_API wmd_status wmd_create(const float* vocab_emb, int64_t V, int32_t d, int32_t device, wmd_handle** out);

/* Use `cuda_stream` (a cudaStream_t, e.g. torch.cuda.current_stream().cuda_stream) for all
 * subsequent work of this handle; NULL restores the handle's own stream. The legacy default
 * stream (torch's default, handle 0) is selected with cudaStreamLegacy ((void*)1). */
WMD_API wmd_status wmd_set_stream(wmd_handle* h, void* cuda_stream);

WMD_API wmd_status wmd_set_option(wmd_handle* h, int32_t option, int64_t value);

/* "While x changes" (Algorithm 1 l.3). tol < 0 (default):
 * every query runs exactly `iters` x-updates. tol >= 0: each document stops on its own after
 * the first x-update with max_i |x_new_ij / x_ij - 1| <= tol (a relative, scale-free reading of
 * the paper's untoleranced rule, R31), at most `iters` updates; then the final step.
 * The per-document update counts of the last query are read with wmd_read_iterations.
 * Errors: INVALID_ARGUMENT (NaN). */
WMD_API wmd_status wmd_set_tolerance(wmd_handle* h, double tol);

/* Install the target documents c ("c is a sparse vocabulary_size x num_docs
 * matrix ... columns of c are normalized"). CSC: col_ptr[N+1] int64 (col_ptr[0]==0,
 * non-decreasing, col_ptr[N]==nnz), row_idx[nnz] int32 word ids strictly increasing within
 * each column, val[nnz] FP32 weights > 0 with |sum_col - 1| <= 1e-5. Host or device pointers
 * (validated synchronously). For a multi-GPU shard pass the rebased column range.
 * Errors: INVALID_ARGUMENT (N<1, nnz<1, nnz >= 2^31), MALFORMED_CSC, EMPTY_DOCUMENT,
 * INDEX_OUT_OF_RANGE, BAD_WEIGHTS, OUT_OF_MEMORY, CUDA. On error the previous targets are
 * dropped (state as if never set). */
WMD_API wmd_status wmd_set_targets(wmd_handle* h, const int64_t* col_ptr, const int32_t* row_idx,
                           const float* val, int64_t N, int64_t nnz);

/* One query (PAPER.md:88 sinkhorn_wmd(r, c, vecs, lamda, max_iter)).
 * query_ids[n] / query_weights[n]: HOST arrays, the nonzeros of r in any order (sorted
 *   ascending inside — Algorithm 1 l.1 selects them in vocabulary order); ids distinct.
 * lambda > 0 (K = exp(-lambda M); the paper passes it negated).
 * iters >= 0 = number of x-updates (Table 1 `while it < max_iter`); the final u/v/WMD step is extra.
 * out_dist: N floats, host or device. Device: written asynchronously on the handle's stream,
 *   valid after stream synchronisation. Host: the call copies back and synchronises.
 * Errors (returned synchronously): STATE, INVALID_ARGUMENT, INDEX_OUT_OF_RANGE, BAD_WEIGHTS,
 * CUDA. A numerical breakdown (non-finite even after FP64) is latched on the device and
 * returned by the next wmd_sync; the non-finite value stays in out_dist. */
WMD_API wmd_status wmd_query(wmd_handle* h, const int32_t* query_ids, const float* query_weights,
                     int32_t n, float lambda, int32_t iters, float* out_dist);

/* A batch of nq queries against the same targets in one call (many
 * queries, PAPER.md:12 "one tweet vs a day of tweets", :255 per-query runs). Query q is
 * query_ids[q_ptr[q] .. q_ptr[q+1]) with weights at the same positions (HOST arrays, each query
 * as in wmd_query); q_ptr: nq+1 int64 offsets, q_ptr[0] == 0, non-decreasing.
 * out_dist: nq x N floats row-major (row q = query q), host or device as in wmd_query.
 * Every query is validated before any work is enqueued (all-or-nothing; the message names the
 * first bad query). The rows of all queries go to the device in one copy; the queries then run
 * back to back with no host round trip between them (each: build, Sinkhorn, final, re-runs).
 * When every query takes the one-warp fused kernel (documents of at most 64 words at v_r <= 64,
 * no tolerance, no graph mode), the queries are solved B at a time (WMD_OPT_BATCH): one fused
 * pass per length bucket serves B queries, reading each document's entries once for all of them
 * (NEXT-2 (ii)). Otherwise, when every query takes the fused path, query q's table is built on a
 * second internal stream into one of two tables while query q-1 is solved on the handle's
 * stream. The call's work is complete on the handle's stream when it returns (device output) or
 * synchronised (host output). Results equal nq separate wmd_query calls bit for bit; the
 * introspection calls (wmd_read_flags, wmd_get_query_rows, wmd_sync's counts) report the last
 * query.
 * Errors: as wmd_query, plus INVALID_ARGUMENT for nq < 1 or bad q_ptr. */
WMD_API wmd_status wmd_query_batch(wmd_handle* h, const int32_t* query_ids, const float* query_weights,
                           const int64_t* q_ptr, int32_t nq, float lambda, int32_t iters,
                           float* out_dist);

/* Two-phase query, for a build sharded across ranks (SURVEY.md §8f NEXT-4, §8e Amdahl term B):
 * wmd_query_begin validates and uploads the query like wmd_query and builds rows
 * [row_begin, row_end) of the vocabulary tables only (each rank its share, PAPER.md:259-268's
 * distance kernel split over vocabulary rows); the tables are allocated with
 * max(V, table_rows) rows so equal row slices can be all-gathered in place.
 * wmd_query_tables returns the device tables (valid until the next query on the handle):
 * Mx (rows of mx_row_floats floats: M, then m_k at column mx_row_floats - 4) and, on the
 * per-iteration path only, K~ (rows of kt_row_floats floats; NULL / 0 on the fused path).
 * The caller completes every row [0, V) of both (e.g. torch.distributed.all_gather_into_tensor
 * over NCCL: the library itself never communicates), on the handle's stream order, then
 * wmd_query_finish runs the Sinkhorn iterations, final step and FP64 fallback into out_dist
 * (as in wmd_query). wmd_query(...) == begin(rows [0, V)) + finish.
 * Errors: as wmd_query; INVALID_ARGUMENT for a bad row range; STATE for finish/tables without
 * a begun query. */
WMD_API wmd_status wmd_query_begin(wmd_handle* h, const int32_t* query_ids, const float* query_weights,
                           int32_t n, float lambda, int32_t iters, int64_t row_begin, int64_t row_end,
                           int64_t table_rows);
WMD_API wmd_status wmd_query_tables(wmd_handle* h, float** mx, int32_t* mx_row_floats, float** kt,
                            int32_t* kt_row_floats);
WMD_API wmd_status wmd_query_finish(wmd_handle* h, float* out_dist);

/* Wait for the handle's stream; return a latched deferred status (then clear it). */
WMD_API wmd_status wmd_sync(wmd_handle* h);

/* nnz-balanced contiguous document partition ("divided the number of non-zeros
 * in c evenly among the threads ... starting exploration point ... using a binary search"),
 * snapped to document boundaries: bounds[0]=0, bounds[P]=N,
 * bounds[g] = first j with col_ptr[j] >= ceil(g*nnz/P). Pure host; bit-exact.
 * Errors: INVALID_ARGUMENT (NULL, N<0, P<1). */
WMD_API wmd_status wmd_partition(const int64_t* col_ptr, int64_t N, int32_t P, int64_t* bounds);

/* Pure host validation (the same checks wmd_set_targets / wmd_query run). bad_index (may be
 * NULL) receives the first offending document / query position, or -1. */
WMD_API wmd_status wmd_validate_csc(const int64_t* col_ptr, const int32_t* row_idx, const float* val,
                            int64_t N, int64_t nnz, int64_t V, int64_t* bad_index);
WMD_API wmd_status wmd_validate_query(const int32_t* ids, const float* weights, int32_t n, int64_t V,
                              int64_t* bad_index);

/* Statistics (synchronises the handle's stream when timing is enabled). */
WMD_API wmd_status wmd_get_stats(wmd_handle* h, wmd_stats* out);
WMD_API wmd_status wmd_reset_stats(wmd_handle* h);

/* Introspection of the last query (device -> host copies; synchronises). For tests.
 * wmd_get_query_rows: sel[v_r] (ascending ids), r[v_r] (weights in that order).
 * wmd_read_kernel: rows [k0, k0+count) of K~ and of M (each row ld floats, ld = last_ld;
 *   zero padded beyond v_r) and colmin[k] = min_i M_ik. Any output pointer may be NULL.
 * wmd_read_scaling: u after the last iteration, documents [j0, j0+count), ld floats each
 *   (gauge-scaled: only ratios within a document are meaningful). Per-iteration path only.
 * wmd_read_flags: flags[N] (bit0: FP32 iterate left the normal range; bit1: FP64 re-run;
 *   bit2: re-run in FP32 by the one-CTA kernel with re-anchoring, R33; bit4: the
 *   one-warp kernel's FP32 block had entries below FLT_MIN, so its range certificate was in
 *   force). */
WMD_API wmd_status wmd_get_query_rows(wmd_handle* h, int32_t* sel, float* r);
WMD_API wmd_status wmd_read_kernel(wmd_handle* h, int64_t k0, int64_t count, float* ktilde, float* m,
                           float* colmin);
WMD_API wmd_status wmd_read_scaling(wmd_handle* h, int64_t j0, int64_t count, float* u);
WMD_API wmd_status wmd_read_flags(wmd_handle* h, uint8_t* flags);
/* iters_out[N]: x-updates each document of the last query ran (== iters unless a tolerance is
 * set; for wmd_query_batch: the last query of the batch). */
WMD_API wmd_status wmd_read_iterations(wmd_handle* h, int32_t* iters_out);

WMD_API const char* wmd_status_string(wmd_status s);
WMD_API const char* wmd_last_error(const wmd_handle* h); /* detail of the last error on h ("" if none) */
WMD_API const char* wmd_version(void);
WMD_API void wmd_destroy(wmd_handle* h);

#ifdef __cplusplus
}
#endif
#endif /* WMD_B200_H */
