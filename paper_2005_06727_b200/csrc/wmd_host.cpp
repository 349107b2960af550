// wmd_host.cpp — host runtime behind the C ABI in include/wmd.h.
//
// Owns the handle (device buffers, stream, options, statistics), validates every input on the
// host (integer bookkeeping is bit-exact and never touches floating point except the FP64
// normalisation sums), sorts the query (Algorithm 1 line 1) and enqueues the
// kernels of wmd_kernels.cu on the handle's stream. No arithmetic of the method runs here.
#include <algorithm>
#include <functional>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <deque>
#include <new>
#include <numeric>
#include <string>
#include <vector>

#include <cuda_runtime.h>

#include "wmd_internal.h"

using wmd::Entry;

// Zeroed slack entries after ent / sdoc. 0: the slack (1,024 entries in rounds 1-2) contained the
// one-CTA kernel's illegal-address fault before its cause was found (a ptxas wait-count hazard on
// a CS2R-zeroed register); no kernel reads past the arrays' ends.
#ifndef WMD_GUARD_ENTRIES
#define WMD_GUARD_ENTRIES 0
#endif
namespace {
constexpr int64_t kGuard = WMD_GUARD_ENTRIES;
}  // namespace

namespace {

constexpr double kWeightTol = 1e-5;  // |sum - 1| for FP32 weights summed in FP64 (R23)

struct DeviceGuard {
  int prev = -1;
  bool ok = true;
  explicit DeviceGuard(int dev) {
    if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
    if (prev != dev) ok = cudaSetDevice(dev) == cudaSuccess;
  }
  ~DeviceGuard() {
    int cur = -1;
    if (prev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
  }
};

bool is_device_ptr(const void* p) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();  // clear: unregistered host memory on old runtimes
    return false;
  }
  return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

template <typename T>
struct DevBuf {
  T* p = nullptr;
  size_t n = 0;
  cudaError_t ensure(size_t count) {
    if (count <= n && p) return cudaSuccess;
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
    cudaError_t e = cudaMalloc(&p, sizeof(T) * std::max<size_t>(count, 1));
    if (e == cudaSuccess) n = count;
    return e;
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
  }
};

struct PhaseEvents {
  cudaEvent_t ev[5];      // start, after build, after iterations, after final, after fallback
  bool complete = false;  // ev[4] recorded: the query's whole stream work is enqueued
};

// What a captured query graph depends on (WMD_OPT_GRAPH).
struct GraphKey {
  const void* sel;
  const void* r;
  const void* dist;
  int32_t v_r, ld;
  float lambda;
  int32_t iters;
  double tol;
  bool fused;
  int64_t fallback, build, targets_gen;
  const void* bufs[5];  // Mx, Kt, ua, ub, umask: a reallocation invalidates the graph
  bool operator==(const GraphKey& o) const {
    for (int i = 0; i < 5; ++i)
      if (bufs[i] != o.bufs[i]) return false;
    return sel == o.sel && r == o.r && dist == o.dist && v_r == o.v_r && ld == o.ld && lambda == o.lambda &&
           iters == o.iters && tol == o.tol && fused == o.fused && fallback == o.fallback &&
           build == o.build && targets_gen == o.targets_gen;
  }
};

}  // namespace

struct wmd_handle {
  int device = 0;
  cudaStream_t own_stream = nullptr;
  cudaStream_t stream = nullptr;
  static constexpr int kLanes = 3;               // streams of the fused phase's length buckets
  cudaStream_t lanes[kLanes] = {};
  cudaEvent_t fork_ev = nullptr, join_ev[kLanes] = {};
  cudaStream_t bstream = nullptr;                // builds of the next queries
  cudaEvent_t built_ev = nullptr;
  // embeddings
  DevBuf<float> E;
  wmd::ExactE ex;            // E in fixed-point limbs (exact tensor-core build)
  int64_t V = 0;
  int32_t d = 0, dp = 0;     // dp: padded row stride of E (multiple of 32)
  // targets
  bool has_targets = false;
  DevBuf<int32_t> doc_ptr;
  DevBuf<int32_t> order;     // documents sorted by length (stable counting sort)
  DevBuf<int4> sdoc;         // {id, first nonzero, length, 0} in that order (fused path)
  DevBuf<Entry> ent;
  int64_t N = 0, nnz = 0, max_doc_nnz = 0;
  std::vector<int64_t> len_prefix;  // [L] = documents with fewer than L nonzeros (host)
  // per-query device state
  DevBuf<int32_t> sel;       // WMD_MAX_VR
  DevBuf<float> rpad;        // WMD_MAX_VR (zero padded to ld)
  DevBuf<float> Kt;          // V * ld: K~ (FP32, vocab-major; per-iteration path only)
  DevBuf<float> Mx;          // V * (ld + 4): M rows + m_k (FP32, vocab-major)
  // Query units: (Mx, sel, rpad, mx_free) and (Mx2, sel2, rpad2, mx2_free) swap per query in
  // the overlapped paths, so the build of query q (build stream) overlaps the solve of q-1
  DevBuf<float> Mx2;
  DevBuf<int32_t> sel2;
  DevBuf<float> rpad2;
  cudaEvent_t mx_free = nullptr, mx2_free = nullptr;  // recorded after the unit's last solve
  bool kt_valid = false;     // Kt holds the last query's K~
  DevBuf<float> ua, ub;      // N * ld
  DevBuf<uint32_t> umask;    // N * ceil(ld/32): rows with an underflowed K~ entry, per doc
  DevBuf<float> dist_tmp;    // N (host-output queries)
  DevBuf<uint8_t> flags;     // N
  DevBuf<int32_t> flagged;   // N
  DevBuf<int32_t> iters_doc; // N: x-updates per document of the last query
  DevBuf<uint8_t> conv;      // N: converged flags ("while x changes", per-iteration path)
  double tol = -1.0;         // "while x changes" relative tolerance; < 0: fixed iterations
  DevBuf<int32_t> flagged2;  // N: documents the one-CTA re-run could not certify either
  DevBuf<int32_t> counters;  // [0] flagged count, [1] breakdown, [2] fallback count, [3] scratch,
                             // [4] flagged2 count
  DevBuf<double> fb_scratch;
  // pinned staging for the query upload (double buffered)
  void* stage[2] = {nullptr, nullptr};
  cudaEvent_t stage_ev[2] = {nullptr, nullptr};
  int stage_slot = 0;
  // batched queries (wmd_query_batch): device rows, pinned staging, host-output buffer
  DevBuf<int32_t> bsel;
  DevBuf<float> brpad, batch_dist;
  // batched fused passes (NEXT-2 (ii)): widths and width-sorted order of the batch's queries,
  // B side-by-side tables, batch-local flags / flagged lists / counts
  DevBuf<int32_t> bvr, bqmap, bflagged, bcount;
  DevBuf<float> Mxb[2];                            // tables of two passes: the next pass's builds
  cudaEvent_t mxb_free[2] = {nullptr, nullptr};    // (build stream) overlap this pass's solve
  cudaEvent_t up_ev = nullptr;                     // the batch's uploads are on the device
  DevBuf<uint8_t> bflags;
  void* batch_stage = nullptr;
  size_t batch_stage_bytes = 0;
  cudaEvent_t batch_ev = nullptr;
  // last query
  int32_t v_r = 0, ld = 0, path_used = 0;
  const int32_t* last_sel = nullptr;
  const float* last_r = nullptr;
  bool u_valid = false;
  const float* u_last = nullptr;
  std::vector<int32_t> h_sel;
  std::vector<float> h_r;
  // two-phase query (wmd_query_begin / wmd_query_finish)
  struct {
    bool active = false, fused = false;
    int32_t v_r = 0, ld = 0, iters = 0;
    float lambda = 0.f;
    PhaseEvents* pe = nullptr;
  } pq;
  // captured query graph (WMD_OPT_GRAPH)
  cudaGraphExec_t graph_exec = nullptr;
  GraphKey graph_key{};
  int64_t graph_launches = 0;
  int64_t targets_gen = 0;   // bumped by every wmd_set_targets (buffers may move)
  // options
  int64_t opt_path = WMD_PATH_AUTO, opt_timing = 0, opt_fallback = 1, opt_graph = 0;
  int64_t opt_build = WMD_BUILD_DIRECT;  // WMD_OPT_BUILD (WMD_BUILD_EXACT once ex is built)
  int32_t build_used = WMD_BUILD_DIRECT; // kernel of the last build_rows
  int64_t opt_layout_nnz = 0;  // WMD_OPT_LAYOUT_DOC_NNZ
  int64_t opt_layout_docs = 0; // WMD_OPT_LAYOUT_DOCS
  int64_t opt_batch = 0;       // WMD_OPT_BATCH
  // stats
  wmd_stats st{};
  // per-phase timing (WMD_OPT_TIMING): events of queries in flight (a deque: push_back /
  // pop_front keep the other entries' addresses, which pq.pe holds across begin / finish),
  // folded into phase_ms as they complete and recycled through event_pool
  std::deque<PhaseEvents> events;
  std::vector<PhaseEvents> event_pool;
  double phase_ms[5] = {};  // build, iterations, final, fallback, whole query
  int64_t phase_n = 0;
  std::string err;
};

namespace {

wmd_status fail(wmd_handle* h, wmd_status s, const char* fmt, ...) {
  if (h) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    h->err = buf;
  }
  return s;
}

wmd_status cuda_fail(wmd_handle* h, cudaError_t e, const char* what) {
  if (e == cudaErrorMemoryAllocation) {
    cudaGetLastError();
    return fail(h, WMD_ERR_OUT_OF_MEMORY, "%s: %s", what, cudaGetErrorString(e));
  }
  return fail(h, WMD_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
}

// WMD_DEBUG_SYNC=1 (environment): synchronise and check after every phase's launches, naming the
// phase in the error (debugging aid; off by default, never inside a graph capture).
bool debug_sync() {
  static const bool on = [] { const char* e = std::getenv("WMD_DEBUG_SYNC"); return e && e[0] == '1'; }();
  return on;
}

#define CK(h, call)                                                    \
  do {                                                                 \
    cudaError_t e_ = (call);                                           \
    if (e_ != cudaSuccess) return cuda_fail((h), e_, #call);           \
  } while (0)
#define DBG_PHASE(h, st, what)                                         \
  do {                                                                 \
    if (debug_sync()) {                                                \
      cudaError_t e_ = cudaDeviceSynchronize();                        \
      if (e_ == cudaSuccess) e_ = cudaGetLastError();                  \
      if (e_ != cudaSuccess) return cuda_fail((h), e_, what);          \
    }                                                                  \
  } while (0)

int32_t round_up8(int32_t x) { return (x + 7) / 8 * 8; }

// Pure-host CSC validation; `bad` receives the first offending column (or nonzero for
// out-of-range ids) and `msg` a description.
wmd_status validate_csc(const int64_t* col_ptr, const int32_t* row_idx, const float* val,
                        int64_t N, int64_t nnz, int64_t V, int64_t* bad, std::string* msg) {
  if (bad) *bad = -1;
  if (!col_ptr || !row_idx || !val || N < 1 || nnz < 1 || V < 1) {
    if (msg) *msg = "NULL array or N/nnz/V < 1";
    return WMD_ERR_INVALID_ARGUMENT;
  }
  if (col_ptr[0] != 0 || col_ptr[N] != nnz) {
    if (msg) *msg = "col_ptr[0] must be 0 and col_ptr[N] must equal nnz";
    return WMD_ERR_MALFORMED_CSC;
  }
  for (int64_t j = 0; j < N; ++j) {
    if (col_ptr[j + 1] < col_ptr[j]) {
      if (bad) *bad = j;
      if (msg) *msg = "col_ptr decreases at column " + std::to_string(j);
      return WMD_ERR_MALFORMED_CSC;
    }
  }
  for (int64_t j = 0; j < N; ++j) {
    const int64_t b = col_ptr[j], e = col_ptr[j + 1];
    if (b == e) {
      if (bad) *bad = j;
      if (msg) *msg = "empty document " + std::to_string(j);
      return WMD_ERR_EMPTY_DOCUMENT;
    }
    double s = 0.0;
    for (int64_t q = b; q < e; ++q) {
      const int32_t k = row_idx[q];
      if (k < 0 || k >= V) {
        if (bad) *bad = j;
        if (msg) *msg = "word id " + std::to_string(k) + " out of range in document " + std::to_string(j);
        return WMD_ERR_INDEX_OUT_OF_RANGE;
      }
      if (q > b && k <= row_idx[q - 1]) {
        if (bad) *bad = j;
        if (msg) *msg = "row ids not strictly increasing in document " + std::to_string(j);
        return WMD_ERR_MALFORMED_CSC;
      }
      const float w = val[q];
      if (!(w > 0.f) || !std::isfinite(w)) {
        if (bad) *bad = j;
        if (msg) *msg = "weight not finite and > 0 in document " + std::to_string(j);
        return WMD_ERR_BAD_WEIGHTS;
      }
      s += (double)w;
    }
    if (std::fabs(s - 1.0) > kWeightTol) {
      if (bad) *bad = j;
      if (msg) *msg = "document " + std::to_string(j) + " weights do not sum to 1";
      return WMD_ERR_BAD_WEIGHTS;
    }
  }
  return WMD_OK;
}

wmd_status validate_query(const int32_t* ids, const float* w, int32_t n, int64_t V, int64_t* bad,
                          std::string* msg, std::vector<int32_t>* sel_out,
                          std::vector<float>* r_out) {
  if (bad) *bad = -1;
  if (!ids || !w || n < 1 || n > WMD_MAX_VR || V < 1) {
    if (msg) *msg = "NULL query or v_r outside [1, WMD_MAX_VR]";
    return WMD_ERR_INVALID_ARGUMENT;
  }
  double s = 0.0;
  for (int32_t q = 0; q < n; ++q) {
    if (ids[q] < 0 || ids[q] >= V) {
      if (bad) *bad = q;
      if (msg) *msg = "query id out of range at position " + std::to_string(q);
      return WMD_ERR_INDEX_OUT_OF_RANGE;
    }
    if (!(w[q] > 0.f) || !std::isfinite(w[q])) {
      if (bad) *bad = q;
      if (msg) *msg = "query weight not finite and > 0 at position " + std::to_string(q);
      return WMD_ERR_BAD_WEIGHTS;
    }
    s += (double)w[q];
  }
  if (std::fabs(s - 1.0) > kWeightTol) {
    if (msg) *msg = "query weights do not sum to 1";
    return WMD_ERR_BAD_WEIGHTS;
  }
  // Algorithm 1 line 1: the selected rows in ascending vocabulary order (stable sort by id).
  std::vector<int32_t> perm(n);
  std::iota(perm.begin(), perm.end(), 0);
  std::stable_sort(perm.begin(), perm.end(), [&](int32_t a, int32_t b) { return ids[a] < ids[b]; });
  for (int32_t q = 1; q < n; ++q) {
    if (ids[perm[q]] == ids[perm[q - 1]]) {
      if (bad) *bad = perm[q];
      if (msg) *msg = "duplicate query id " + std::to_string(ids[perm[q]]);
      return WMD_ERR_BAD_WEIGHTS;
    }
  }
  if (sel_out && r_out) {
    sel_out->resize(n);
    r_out->resize(n);
    for (int32_t q = 0; q < n; ++q) {
      (*sel_out)[q] = ids[perm[q]];
      (*r_out)[q] = w[perm[q]];
    }
  }
  return WMD_OK;
}

void drop_targets(wmd_handle* h) {
  h->has_targets = false;
  h->doc_ptr.release();
  h->order.release();
  h->sdoc.release();
  h->ent.release();
  h->N = h->nnz = h->max_doc_nnz = 0;
  h->u_valid = false;
}

}  // namespace

extern "C" {

const char* wmd_version(void) { return "wmd_b200 0.1 (sm_100a)"; }

const char* wmd_status_string(wmd_status s) {
  switch (s) {
    case WMD_OK: return "ok";
    case WMD_ERR_INVALID_ARGUMENT: return "invalid argument";
    case WMD_ERR_INDEX_OUT_OF_RANGE: return "index out of range";
    case WMD_ERR_EMPTY_DOCUMENT: return "empty document";
    case WMD_ERR_MALFORMED_CSC: return "malformed CSC matrix";
    case WMD_ERR_BAD_WEIGHTS: return "bad weights";
    case WMD_ERR_NONFINITE_EMBEDDING: return "non-finite embedding";
    case WMD_ERR_STATE: return "invalid state";
    case WMD_ERR_NUMERICAL_BREAKDOWN: return "numerical breakdown";
    case WMD_ERR_OUT_OF_MEMORY: return "out of device memory";
    case WMD_ERR_CUDA: return "CUDA error";
  }
  return "unknown status";
}

const char* wmd_last_error(const wmd_handle* h) { return h ? h->err.c_str() : ""; }

wmd_status wmd_partition(const int64_t* col_ptr, int64_t N, int32_t P, int64_t* bounds) {
  if (!col_ptr || !bounds || N < 0 || P < 1) return WMD_ERR_INVALID_ARGUMENT;
  const int64_t nnz = col_ptr[N];
  bounds[0] = 0;
  for (int32_t g = 1; g < P; ++g) {
    const int64_t target = (g * nnz + P - 1) / P;  // ceil(g * nnz / P)
    bounds[g] = std::lower_bound(col_ptr, col_ptr + N + 1, target) - col_ptr;  // binary search
    if (bounds[g] > N) bounds[g] = N;
  }
  bounds[P] = N;
  return WMD_OK;
}

wmd_status wmd_validate_csc(const int64_t* col_ptr, const int32_t* row_idx, const float* val,
                            int64_t N, int64_t nnz, int64_t V, int64_t* bad_index) {
  return validate_csc(col_ptr, row_idx, val, N, nnz, V, bad_index, nullptr);
}

wmd_status wmd_validate_query(const int32_t* ids, const float* weights, int32_t n, int64_t V,
                              int64_t* bad_index) {
  return validate_query(ids, weights, n, V, bad_index, nullptr, nullptr, nullptr);
}

wmd_status wmd_create(const float* vocab_emb, int64_t V, int32_t d, int32_t device, wmd_handle** out) {
  if (!out) return WMD_ERR_INVALID_ARGUMENT;
  *out = nullptr;
  if (!vocab_emb || V < 1 || d < 1 || V > WMD_MAX_V || device < 0) return WMD_ERR_INVALID_ARGUMENT;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || device >= ndev) {
    cudaGetLastError();
    return WMD_ERR_CUDA;
  }
  DeviceGuard g(device);
  if (!g.ok) return WMD_ERR_CUDA;
  wmd_handle* h = new (std::nothrow) wmd_handle();
  if (!h) return WMD_ERR_OUT_OF_MEMORY;
  h->device = device;
  h->V = V;
  h->d = d;
  auto bail = [&](wmd_status s) { wmd_destroy(h); return s; };
  if (cudaStreamCreateWithFlags(&h->own_stream, cudaStreamNonBlocking) != cudaSuccess) return bail(WMD_ERR_CUDA);
  h->stream = h->own_stream;
  // E is kept with rows padded to dp = d rounded up to 32 floats (zeros add nothing to a
  // distance): the build kernel streams whole 32-float chunks with 16-byte async copies.
  const int32_t dp = (d + 31) / 32 * 32;
  h->dp = dp;
  const size_t n = (size_t)V * d;
  if (h->E.ensure((size_t)V * dp) != cudaSuccess) return bail(WMD_ERR_OUT_OF_MEMORY);
  if (cudaMemsetAsync(h->E.p, 0, (size_t)V * dp * sizeof(float), h->stream) != cudaSuccess) return bail(WMD_ERR_CUDA);
  if (h->counters.ensure(6) != cudaSuccess) return bail(WMD_ERR_OUT_OF_MEMORY);
  // every counter starts at zero whichever branch below runs (cudaMalloc may recycle memory of an
  // earlier handle: a stale breakdown latch would surface as a spurious error at wmd_sync)
  if (cudaMemsetAsync(h->counters.p, 0, 6 * sizeof(int32_t), h->stream) != cudaSuccess) return bail(WMD_ERR_CUDA);
  if (is_device_ptr(vocab_emb)) {
    if (cudaMemcpy2DAsync(h->E.p, dp * sizeof(float), vocab_emb, d * sizeof(float), d * sizeof(float), V,
                          cudaMemcpyDeviceToDevice, h->stream) != cudaSuccess)
      return bail(WMD_ERR_CUDA);
    wmd::launch_check_finite(h->E.p, (int64_t)V * dp, h->counters.p + 3, h->stream);
    int32_t bad = 0;
    if (cudaMemcpyAsync(&bad, h->counters.p + 3, sizeof bad, cudaMemcpyDeviceToHost, h->stream) != cudaSuccess ||
        cudaStreamSynchronize(h->stream) != cudaSuccess)
      return bail(WMD_ERR_CUDA);
    if (bad) return bail(WMD_ERR_NONFINITE_EMBEDDING);
  } else {
    for (size_t i = 0; i < n; ++i)
      if (!std::isfinite(vocab_emb[i])) return bail(WMD_ERR_NONFINITE_EMBEDDING);
    if (cudaMemcpy2DAsync(h->E.p, dp * sizeof(float), vocab_emb, d * sizeof(float), d * sizeof(float), V,
                          cudaMemcpyHostToDevice, h->stream) != cudaSuccess ||
        cudaStreamSynchronize(h->stream) != cudaSuccess)
      return bail(WMD_ERR_CUDA);
  }
  // fixed-point limb planes for the exact tensor-core build (unsupported shapes leave ex.ok false)
  if (const int e = wmd::prepare_exact_e(h->E.p, V, dp, &h->ex, h->stream))
    return bail(e == (int)cudaErrorMemoryAllocation ? WMD_ERR_OUT_OF_MEMORY : WMD_ERR_CUDA);
  if (h->ex.ok) h->opt_build = WMD_BUILD_EXACT;
  if (h->sel.ensure(WMD_MAX_VR) != cudaSuccess || h->rpad.ensure(WMD_MAX_VR) != cudaSuccess ||
      h->counters.ensure(6) != cudaSuccess)
    return bail(WMD_ERR_OUT_OF_MEMORY);
  if (cudaEventCreateWithFlags(&h->batch_ev, cudaEventDisableTiming) != cudaSuccess) return bail(WMD_ERR_CUDA);
  if (cudaEventCreateWithFlags(&h->up_ev, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&h->mxb_free[0], cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&h->mxb_free[1], cudaEventDisableTiming) != cudaSuccess)
    return bail(WMD_ERR_CUDA);
  if (cudaEventCreateWithFlags(&h->fork_ev, cudaEventDisableTiming) != cudaSuccess) return bail(WMD_ERR_CUDA);
  if (cudaStreamCreateWithFlags(&h->bstream, cudaStreamNonBlocking) != cudaSuccess) return bail(WMD_ERR_CUDA);
  if (cudaEventCreateWithFlags(&h->built_ev, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&h->mx_free, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&h->mx2_free, cudaEventDisableTiming) != cudaSuccess ||
      h->sel2.ensure(WMD_MAX_VR) != cudaSuccess || h->rpad2.ensure(WMD_MAX_VR) != cudaSuccess)
    return bail(WMD_ERR_CUDA);
  int prio_lo = 0, prio_hi = 0;  // the bucket lanes get the highest priority: the overlapped build
  cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi);  // of the next query only fills gaps
  for (int i = 0; i < wmd_handle::kLanes; ++i)
    if (cudaStreamCreateWithPriority(&h->lanes[i], cudaStreamNonBlocking, prio_hi) != cudaSuccess ||
        cudaEventCreateWithFlags(&h->join_ev[i], cudaEventDisableTiming) != cudaSuccess)
      return bail(WMD_ERR_CUDA);
  for (int s = 0; s < 2; ++s) {
    if (cudaMallocHost(&h->stage[s], WMD_MAX_VR * 8) != cudaSuccess) return bail(WMD_ERR_OUT_OF_MEMORY);
    if (cudaEventCreateWithFlags(&h->stage_ev[s], cudaEventDisableTiming) != cudaSuccess) return bail(WMD_ERR_CUDA);
  }
  if (cudaStreamSynchronize(h->stream) != cudaSuccess) return bail(WMD_ERR_CUDA);
  *out = h;
  return WMD_OK;
}

void wmd_destroy(wmd_handle* h) {
  if (!h) return;
  DeviceGuard g(h->device);
  if (h->own_stream) cudaStreamSynchronize(h->own_stream);
  if (h->stream && h->stream != h->own_stream) cudaStreamSynchronize(h->stream);
  if (h->graph_exec) cudaGraphExecDestroy(h->graph_exec);
  for (auto& pe : h->events)
    for (auto& e : pe.ev) cudaEventDestroy(e);
  for (auto& pe : h->event_pool)
    for (auto& e : pe.ev) cudaEventDestroy(e);
  if (h->batch_stage) cudaFreeHost(h->batch_stage);
  if (h->batch_ev) cudaEventDestroy(h->batch_ev);
  h->bsel.release(); h->brpad.release(); h->batch_dist.release();
  h->bvr.release(); h->bqmap.release(); h->bflagged.release(); h->bcount.release();
  h->Mxb[0].release(); h->Mxb[1].release();
  h->bflags.release();
  for (auto& e : h->mxb_free)
    if (e) cudaEventDestroy(e);
  if (h->up_ev) cudaEventDestroy(h->up_ev);
  for (int s = 0; s < 2; ++s) {
    if (h->stage[s]) cudaFreeHost(h->stage[s]);
    if (h->stage_ev[s]) cudaEventDestroy(h->stage_ev[s]);
  }
  wmd::free_exact_e(&h->ex);
  h->E.release(); h->doc_ptr.release(); h->order.release(); h->sdoc.release(); h->ent.release(); h->sel.release(); h->rpad.release();
  h->Kt.release(); h->Mx.release(); h->Mx2.release(); h->ua.release(); h->ub.release(); h->umask.release();
  h->dist_tmp.release(); h->flags.release(); h->flagged.release(); h->flagged2.release(); h->counters.release();
  h->iters_doc.release(); h->conv.release();
  h->fb_scratch.release();
  for (int i = 0; i < wmd_handle::kLanes; ++i) {
    if (h->lanes[i]) { cudaStreamSynchronize(h->lanes[i]); cudaStreamDestroy(h->lanes[i]); }
    if (h->join_ev[i]) cudaEventDestroy(h->join_ev[i]);
  }
  if (h->fork_ev) cudaEventDestroy(h->fork_ev);
  if (h->bstream) { cudaStreamSynchronize(h->bstream); cudaStreamDestroy(h->bstream); }
  if (h->built_ev) cudaEventDestroy(h->built_ev);
  if (h->mx_free) cudaEventDestroy(h->mx_free);
  if (h->mx2_free) cudaEventDestroy(h->mx2_free);
  h->sel2.release(); h->rpad2.release();
  if (h->own_stream) cudaStreamDestroy(h->own_stream);
  delete h;
}

wmd_status wmd_set_stream(wmd_handle* h, void* cuda_stream) {
  if (!h) return WMD_ERR_INVALID_ARGUMENT;
  h->stream = cuda_stream ? (cudaStream_t)cuda_stream : h->own_stream;
  return WMD_OK;
}

wmd_status wmd_set_option(wmd_handle* h, int32_t option, int64_t value) {
  if (!h) return WMD_ERR_INVALID_ARGUMENT;
  switch (option) {
    case WMD_OPT_PATH:
      if (value < WMD_PATH_AUTO || value > WMD_PATH_FUSED) return fail(h, WMD_ERR_INVALID_ARGUMENT, "bad path");
      h->opt_path = value;
      return WMD_OK;
    case WMD_OPT_TIMING: h->opt_timing = value != 0; return WMD_OK;
    case WMD_OPT_FALLBACK: h->opt_fallback = value != 0; return WMD_OK;
    case WMD_OPT_GRAPH: h->opt_graph = value != 0; return WMD_OK;
    case WMD_OPT_BUILD:
      if (value != WMD_BUILD_TENSOR_CORE && value != WMD_BUILD_DIRECT && value != WMD_BUILD_EXACT)
        return fail(h, WMD_ERR_INVALID_ARGUMENT, "bad build kernel");
      if (value == WMD_BUILD_EXACT && !h->ex.ok)
        return fail(h, WMD_ERR_INVALID_ARGUMENT, "exact build unavailable (dp=%d outside [32, 1280] or max|E| out of range)", h->dp);
      h->opt_build = value;
      return WMD_OK;
    case WMD_OPT_BATCH:
      if (value < 0 || value > 64) return fail(h, WMD_ERR_INVALID_ARGUMENT, "batch size outside [0, 64]");
      h->opt_batch = value;
      return WMD_OK;
    case WMD_OPT_LAYOUT_DOCS:
      if (value < 0) return fail(h, WMD_ERR_INVALID_ARGUMENT, "negative layout document count");
      h->opt_layout_docs = value;
      return WMD_OK;
    case WMD_OPT_LAYOUT_DOC_NNZ:
      if (value < 0) return fail(h, WMD_ERR_INVALID_ARGUMENT, "negative layout document length");
      h->opt_layout_nnz = value;
      return WMD_OK;
  }
  return fail(h, WMD_ERR_INVALID_ARGUMENT, "unknown option %d", option);
}

wmd_status wmd_set_targets(wmd_handle* h, const int64_t* col_ptr, const int32_t* row_idx,
                           const float* val, int64_t N, int64_t nnz) {
  if (!h) return WMD_ERR_INVALID_ARGUMENT;
  h->err.clear();
  DeviceGuard g(h->device);
  if (!g.ok) return fail(h, WMD_ERR_CUDA, "cudaSetDevice failed");
  drop_targets(h);
  if (!col_ptr || !row_idx || !val || N < 1 || nnz < 1 || nnz >= (int64_t(1) << 31) || N >= (int64_t(1) << 31))
    return fail(h, WMD_ERR_INVALID_ARGUMENT, "NULL array, N/nnz < 1, or nnz >= 2^31");
  // Device inputs are brought to the host once for validation (bit-exact integer checks).
  std::vector<int64_t> hc;
  std::vector<int32_t> hr;
  std::vector<float> hv;
  if (is_device_ptr(col_ptr)) {
    hc.resize(N + 1);
    CK(h, cudaMemcpy(hc.data(), col_ptr, (N + 1) * sizeof(int64_t), cudaMemcpyDeviceToHost));
    col_ptr = hc.data();
  }
  if (col_ptr[N] != nnz) return fail(h, WMD_ERR_MALFORMED_CSC, "col_ptr[N] != nnz");
  if (is_device_ptr(row_idx)) {
    hr.resize(nnz);
    CK(h, cudaMemcpy(hr.data(), row_idx, nnz * sizeof(int32_t), cudaMemcpyDeviceToHost));
    row_idx = hr.data();
  }
  if (is_device_ptr(val)) {
    hv.resize(nnz);
    CK(h, cudaMemcpy(hv.data(), val, nnz * sizeof(float), cudaMemcpyDeviceToHost));
    val = hv.data();
  }
  int64_t bad = -1;
  std::string msg;
  wmd_status s = validate_csc(col_ptr, row_idx, val, N, nnz, h->V, &bad, &msg);
  if (s != WMD_OK) return fail(h, s, "%s", msg.c_str());
  std::vector<int32_t> dp(N + 1);
  int64_t mx = 0;
  for (int64_t j = 0; j <= N; ++j) dp[j] = (int32_t)col_ptr[j];
  for (int64_t j = 0; j < N; ++j) mx = std::max(mx, col_ptr[j + 1] - col_ptr[j]);
  // processing order: stable counting sort of the documents by length (integer bookkeeping)
  std::vector<int64_t> cnt(mx + 2, 0);
  for (int64_t j = 0; j < N; ++j) cnt[col_ptr[j + 1] - col_ptr[j] + 1]++;
  for (int64_t L = 1; L < mx + 2; ++L) cnt[L] += cnt[L - 1];
  // cnt[L] = number of documents shorter than L (kept: length buckets of the sorted order)
  std::vector<int64_t> len_prefix = cnt;
  std::vector<int32_t> ord(N);
  for (int64_t j = 0; j < N; ++j) ord[cnt[col_ptr[j + 1] - col_ptr[j]]++] = (int32_t)j;
  std::vector<Entry> en(nnz);
  for (int64_t q = 0; q < nnz; ++q) en[q] = Entry{row_idx[q], val[q]};
  CK(h, h->doc_ptr.ensure(N + 1));
  // (+ kGuard zeroed slack entries past the end, WMD_GUARD_ENTRIES, 0 by default)
  CK(h, h->ent.ensure(nnz + kGuard));
  if (kGuard) CK(h, cudaMemsetAsync(h->ent.p + nnz, 0, kGuard * sizeof(Entry), h->stream));
  CK(h, h->order.ensure(N));
  CK(h, cudaMemcpyAsync(h->order.p, ord.data(), N * sizeof(int32_t), cudaMemcpyHostToDevice, h->stream));
  std::vector<int4> sd(N);
  for (int64_t p = 0; p < N; ++p) {
    const int32_t j = ord[p];
    sd[p] = make_int4(j, dp[j], dp[j + 1] - dp[j], 0);
  }
  CK(h, h->sdoc.ensure(N + kGuard));
  if (kGuard) CK(h, cudaMemsetAsync(h->sdoc.p + N, 0, kGuard * sizeof(int4), h->stream));
  CK(h, cudaMemcpyAsync(h->sdoc.p, sd.data(), N * sizeof(int4), cudaMemcpyHostToDevice, h->stream));
  CK(h, cudaMemcpyAsync(h->doc_ptr.p, dp.data(), (N + 1) * sizeof(int32_t), cudaMemcpyHostToDevice, h->stream));
  CK(h, cudaMemcpyAsync(h->ent.p, en.data(), nnz * sizeof(Entry), cudaMemcpyHostToDevice, h->stream));
  CK(h, h->flags.ensure(N));
  CK(h, h->flagged.ensure(N));
  CK(h, h->flagged2.ensure(N));
  CK(h, h->iters_doc.ensure(N));
  CK(h, h->conv.ensure(N));
  CK(h, h->dist_tmp.ensure(N));
  CK(h, h->fb_scratch.ensure(wmd::fallback_scratch_bytes(mx) / sizeof(double)));
  CK(h, cudaStreamSynchronize(h->stream));
  h->N = N;
  h->nnz = nnz;
  h->max_doc_nnz = mx;
  h->len_prefix.swap(len_prefix);
  h->has_targets = true;
  ++h->targets_gen;
  return WMD_OK;
}

}  // extern "C"

namespace {

// Longest document the path / table-width decision assumes: the local maximum, or the larger
// WMD_OPT_LAYOUT_DOC_NNZ (every rank of a sharded run passes the global maximum, so all ranks
// choose the same path and row width and their tables can be all-gathered).
int64_t layout_doc_nnz(const wmd_handle* h) { return std::max(h->max_doc_nnz, h->opt_layout_nnz); }
int64_t layout_docs(const wmd_handle* h) { return std::max(h->N, h->opt_layout_docs); }

// Path decision and buffer allocation for one query (never inside a graph capture). The tables
// get max(V, table_rows) rows (a sharded build all-gathers equal row slices, which may pad).
wmd_status prepare_query(wmd_handle* h, int32_t v_r, float lambda, int64_t table_rows, bool* fused_out,
                         int32_t* ld_out) {
  const int64_t N = h->N;
  // fused path: ld = v_r rounded up to a power of two (the 2-D lane tiling); per-iteration
  // path: v_r rounded up to 8
  const int32_t fld = lambda >= wmd::kFusedMinLambda ? wmd::fused_ld(v_r, layout_doc_nnz(h), h->tol >= 0.0) : 0;
  const bool fused = (h->opt_path == WMD_PATH_FUSED || h->opt_path == WMD_PATH_AUTO) && fld > 0;
  if (h->opt_path == WMD_PATH_FUSED && !fused)
    return fail(h, WMD_ERR_INVALID_ARGUMENT, "fused path does not support v_r=%d, max doc nnz=%lld, lambda=%g",
                v_r, (long long)layout_doc_nnz(h), (double)lambda);
  const int32_t ld = fused ? fld : round_up8(v_r);
  const int64_t rows = std::max(h->V, table_rows);
  // +128 floats: the pass kernels gather unpredicated float4s up to 4*32 floats past a row
  if (!fused) CK(h, h->Kt.ensure((size_t)rows * ld + 128));
  CK(h, h->Mx.ensure((size_t)rows * (ld + 4) + 128));
  if (!fused) {
    CK(h, h->ua.ensure((size_t)N * ld));
    CK(h, h->ub.ensure((size_t)N * ld));
    CK(h, h->umask.ensure((size_t)N * ((ld + 31) / 32)));
  }
  *fused_out = fused;
  *ld_out = ld;
  return WMD_OK;
}

// The distance build of the handle's WMD_OPT_BUILD kernel for rows [row0, row1).
void build_rows(wmd_handle* h, const int32_t* d_sel, int32_t v_r, int32_t ld, float lambda, float* Kt, float* Mx,
                int64_t row0, int64_t row1, cudaStream_t st) {
  if (h->opt_build == WMD_BUILD_EXACT && wmd::launch_build_exact(h->ex, row0, row1, d_sel, v_r, ld, lambda, Kt, Mx, st)) {
    h->build_used = WMD_BUILD_EXACT;
    return;
  }
  h->build_used = h->opt_build == WMD_BUILD_TENSOR_CORE ? WMD_BUILD_TENSOR_CORE : WMD_BUILD_DIRECT;
  wmd::launch_build_ktilde(h->E.p, row0, row1, h->dp, d_sel, v_r, ld, lambda, Kt, Mx,
                           h->opt_build == WMD_BUILD_TENSOR_CORE, st);
}

// a2 for vocabulary rows [row0, row1) (capturable stream work).
wmd_status record_build(wmd_handle* h, const int32_t* d_sel, int32_t v_r, float lambda, int64_t row0,
                        int64_t row1, bool fused, int32_t ld, PhaseEvents* pe) {
  cudaStream_t st = h->stream;
  if (pe) CK(h, cudaEventRecord(pe->ev[0], st));
  // M (+ m), and K~ for the per-iteration path
  build_rows(h, d_sel, v_r, ld, lambda, fused ? nullptr : h->Kt.p, h->Mx.p, row0, row1, st);
  DBG_PHASE(h, st, "distance build");
  if (pe) CK(h, cudaEventRecord(pe->ev[1], st));
  CK(h, cudaGetLastError());
  return WMD_OK;
}

// a3-a6 on complete tables (capturable stream work). *launches_out: kernel launches.
wmd_status record_solve(wmd_handle* h, const float* d_r, int32_t v_r, float lambda, int32_t iters,
                        float* dist, bool fused, int32_t ld, PhaseEvents* pe, int64_t* launches_out) {
  const int64_t N = h->N;
  cudaStream_t st = h->stream;
  CK(h, cudaMemsetAsync(h->flags.p, 0, N, st));
  CK(h, cudaMemsetAsync(h->counters.p, 0, sizeof(int32_t), st));  // flagged-list length
  int64_t launches = 0;
  const float tol = h->tol >= 0.0 ? (float)h->tol : -1.f;
  if (fused) {
    // the length buckets run on the handle's lanes (forked from and joined to `st`), so one
    // bucket's tail overlaps the next one's start
    const int nb = wmd::fused_launch_count(h->len_prefix.data(), h->max_doc_nnz, N, layout_docs(h), ld, tol);
    wmd::StreamRing ring;
    if (nb > 1) {
      ring.s = h->lanes;
      ring.n = std::min(nb, (int)wmd_handle::kLanes);
      CK(h, cudaEventRecord(h->fork_ev, st));
      for (int i = 0; i < ring.n; ++i) CK(h, cudaStreamWaitEvent(h->lanes[i], h->fork_ev, 0));
    }
    wmd::QuerySet qs{};
    qs.Mx = h->Mx.p;
    qs.rpad = d_r;
    qs.v_r = v_r;
    qs.nq = 1;
    qs.N = N;
    qs.dist = dist;
    qs.flags = h->flags.p;
    qs.iters_doc = h->iters_doc.p;
    qs.flagged_list = h->flagged.p;
    qs.flagged_count = h->counters.p;
    wmd::launch_sinkhorn_fused(h->sdoc.p, h->ent.p, N, layout_docs(h), h->len_prefix.data(), h->max_doc_nnz, ld, qs, lambda,
                               iters, tol, st, &ring);
    DBG_PHASE(h, st, "fused Sinkhorn kernels");
    for (int i = 0; i < ring.n; ++i) {
      CK(h, cudaEventRecord(h->join_ev[i], h->lanes[i]));
      CK(h, cudaStreamWaitEvent(st, h->join_ev[i], 0));
    }
    launches += wmd::fused_launch_count(h->len_prefix.data(), h->max_doc_nnz, N, layout_docs(h), ld, tol);
    if (pe) { CK(h, cudaEventRecord(pe->ev[2], st)); CK(h, cudaEventRecord(pe->ev[3], st)); }
  } else {
    // a4: iters fused SDDMM_SpMM launches, u ping-pong
    const float* u_in = nullptr;
    float* bufs[2] = {h->ua.p, h->ub.p};
    wmd::launch_fill_i32(h->iters_doc.p, N, iters, st);
    ++launches;
    if (tol >= 0.f) CK(h, cudaMemsetAsync(h->conv.p, 0, N, st));
    for (int32_t t = 0; t < iters; ++t) {
      float* u_out = bufs[t & 1];
      wmd::launch_sddmm_spmm_iter(h->order.p, h->doc_ptr.p, h->ent.p, N, h->Kt.p, ld, v_r, d_r, u_in, u_out,
                                  h->umask.p, h->flags.p, wmd::ConvParams{tol, h->conv.p, h->iters_doc.p, t},
                                  st);
      u_in = u_out;
    }
    launches += iters;
    if (pe) CK(h, cudaEventRecord(pe->ev[2], st));
    // a5
    wmd::launch_final_wmd(h->order.p, h->doc_ptr.p, h->ent.p, N, h->Kt.p, h->Mx.p, ld, v_r, d_r, u_in,
                          h->umask.p, dist, h->flags.p, h->flagged.p, h->counters.p, st);
    ++launches;
    if (pe) CK(h, cudaEventRecord(pe->ev[3], st));
  }
  // a6: re-run of flagged documents (device-side lists; zero-cost when empty): on the fused path
  // first in FP32 by the one-CTA kernel with re-anchoring (R33; fixed iteration count),
  // then whatever is left in FP64
  if (h->opt_fallback) {
    const int32_t* fl = h->flagged.p;
    int32_t* fc = h->counters.p;
    if (fused && tol < 0.f && wmd::cta_rerun_supported(ld)) {
      CK(h, cudaMemsetAsync(h->counters.p + 4, 0, sizeof(int32_t), st));
      wmd::launch_cta_rerun(h->flagged.p, h->counters.p, h->doc_ptr.p, h->ent.p, h->Mx.p, ld, v_r, d_r, lambda,
                            iters, h->iters_doc.p, dist, h->flags.p, h->flagged2.p, h->counters.p + 4, st);
      ++launches;
      DBG_PHASE(h, st, "FP32 re-run of flagged documents");
      fl = h->flagged2.p;
      fc = h->counters.p + 4;
    }
    wmd::launch_fallback_fp64(h->Mx.p, ld, d_r, v_r, (double)lambda, iters, tol, h->iters_doc.p, h->doc_ptr.p,
                              h->ent.p, fl, fc, h->fb_scratch.p, h->max_doc_nnz, dist,
                              h->flags.p, h->counters.p + 1, h->counters.p + 2, st);
    ++launches;
    DBG_PHASE(h, st, "FP64 re-run");
  }
  if (pe) {
    CK(h, cudaEventRecord(pe->ev[4], st));
    pe->complete = true;
  }
  CK(h, cudaGetLastError());
  *launches_out = launches;
  return WMD_OK;
}

// Folds the completed queries at the front of h->events into h->phase_ms (wait: block on each
// one, else stop at the first still running) and recycles their events.
cudaError_t fold_events(wmd_handle* h, bool wait) {
  while (!h->events.empty() && h->events.front().complete) {
    PhaseEvents& pe = h->events.front();
    if (wait) {
      const cudaError_t e = cudaEventSynchronize(pe.ev[4]);
      if (e != cudaSuccess) return e;
    } else if (cudaEventQuery(pe.ev[4]) != cudaSuccess) {
      cudaGetLastError();  // cudaErrorNotReady is not sticky, but clear it anyway
      break;
    }
    float t[5];
    for (int q = 0; q < 4; ++q) {
      const cudaError_t e = cudaEventElapsedTime(&t[q], pe.ev[q], pe.ev[q + 1]);
      if (e != cudaSuccess) return e;
    }
    const cudaError_t e = cudaEventElapsedTime(&t[4], pe.ev[0], pe.ev[4]);
    if (e != cudaSuccess) return e;
    for (int q = 0; q < 5; ++q) h->phase_ms[q] += t[q];
    ++h->phase_n;
    pe.complete = false;
    h->event_pool.push_back(pe);
    h->events.pop_front();
  }
  return cudaSuccess;
}

PhaseEvents* new_phase_events(wmd_handle* h) {
  if (!h->opt_timing) return nullptr;
  // a query that failed after taking its events never completes them: recycle it (unless it is
  // the begun two-phase query, whose events wmd_query_finish still records)
  if (!h->events.empty() && !h->events.back().complete && !(h->pq.active && h->pq.pe == &h->events.back())) {
    h->event_pool.push_back(h->events.back());
    h->events.pop_back();
  }
  if (h->events.size() >= 16) fold_events(h, false);  // bounded: completed queries fold as we go
  PhaseEvents e{};
  if (!h->event_pool.empty()) {
    e = h->event_pool.back();
    h->event_pool.pop_back();
  } else {
    for (auto& x : e.ev)
      if (cudaEventCreate(&x) != cudaSuccess) return nullptr;
  }
  e.complete = false;
  h->events.push_back(e);
  return &h->events.back();
}

// Host bookkeeping after a query's solve was enqueued.
void note_query(wmd_handle* h, const int32_t* d_sel, const float* d_r, int32_t v_r, int32_t iters, bool fused,
                int32_t ld, int64_t launches) {
  h->kt_valid = !fused;
  h->u_valid = !fused && iters > 0;
  h->u_last = (!fused && iters > 0) ? ((iters - 1) & 1 ? h->ub.p : h->ua.p) : nullptr;
  h->path_used = fused ? WMD_PATH_FUSED : WMD_PATH_PER_ITER;
  h->st.iter_launches += fused ? wmd::fused_launch_count(h->len_prefix.data(), h->max_doc_nnz, h->N, layout_docs(h), ld,
                                                          h->tol >= 0.0 ? (float)h->tol : -1.f) : iters;
  h->v_r = v_r;
  h->ld = ld;
  h->last_sel = d_sel;
  h->last_r = d_r;
  h->st.queries += 1;
  h->st.kernel_launches += launches;
  h->st.last_v_r = v_r;
  h->st.last_ld = ld;
  h->st.last_path = h->path_used;
  h->st.last_build = h->build_used;
}

// Enqueue one validated query whose sorted rows sel (device, v_r ids) and r (device, zero padded
// to WMD_MAX_VR) are already on the device. dist: device, N floats. Asynchronous on the handle's
// stream. With WMD_OPT_GRAPH (and no timing) the stream work is captured once per distinct
// (rows, output, lambda, iters, tolerance, path, options) and replayed as a CUDA graph.
void swap_units(wmd_handle* h) {
  std::swap(h->Mx, h->Mx2);
  std::swap(h->sel, h->sel2);
  std::swap(h->rpad, h->rpad2);
  std::swap(h->mx_free, h->mx2_free);
}

// One fused-path query with its build on the build stream (after the unit's previous solve
// freed it) and its solve on the main stream: consecutive queries overlap build and solve.
// `upload` enqueues the copies of the query rows into d_sel / d_r on the given stream (or is
// empty when they are already on the device). Returns false through *ok if the query does not
// take the fused path (nothing enqueued).
wmd_status enqueue_overlapped(wmd_handle* h, const int32_t* d_sel, const float* d_r, int32_t v_r, float lambda,
                              int32_t iters, float* dist, const std::function<wmd_status(cudaStream_t)>& upload) {
  bool fused = false;
  int32_t ld = 0;
  wmd_status s = prepare_query(h, v_r, lambda, h->V, &fused, &ld);
  if (s != WMD_OK) return s;
  cudaStream_t main = h->stream;
  CK(h, cudaStreamWaitEvent(h->bstream, h->mx_free, 0));  // the unit's previous solve is done
  if (upload) {
    s = upload(h->bstream);
    if (s != WMD_OK) return s;
  }
  PhaseEvents* pe = new_phase_events(h);
  h->stream = h->bstream;
  s = record_build(h, d_sel, v_r, lambda, 0, h->V, fused, ld, pe);
  h->stream = main;
  if (s != WMD_OK) return s;
  CK(h, cudaEventRecord(h->built_ev, h->bstream));
  CK(h, cudaStreamWaitEvent(main, h->built_ev, 0));
  // phase timing: the solve starts here (build_ms then includes any wait for the previous solve)
  if (pe) CK(h, cudaEventRecord(pe->ev[1], main));
  int64_t launches = 0;
  s = record_solve(h, d_r, v_r, lambda, iters, dist, fused, ld, pe, &launches);
  if (s != WMD_OK) return s;
  CK(h, cudaEventRecord(h->mx_free, main));
  note_query(h, d_sel, d_r, v_r, iters, fused, ld, launches + 1);
  return WMD_OK;
}


wmd_status enqueue_query(wmd_handle* h, const int32_t* d_sel, const float* d_r, int32_t v_r,
                         float lambda, int32_t iters, float* dist) {
  bool fused = false;
  int32_t ld = 0;
  wmd_status s = prepare_query(h, v_r, lambda, h->V, &fused, &ld);
  if (s != WMD_OK) return s;
  int64_t launches = 0;
  if (h->opt_graph && !h->opt_timing) {
    const GraphKey key{d_sel, d_r, dist, v_r, ld, lambda, iters, h->tol, fused, h->opt_fallback, h->opt_build,
                       h->targets_gen, {h->Mx.p, h->Kt.p, h->ua.p, h->ub.p, h->umask.p}};
    if (!(h->graph_exec && h->graph_key == key)) {
      if (h->graph_exec) {  // re-capture: the old executable may still be in flight
        CK(h, cudaStreamSynchronize(h->stream));
        cudaGraphExecDestroy(h->graph_exec);
      }
      h->graph_exec = nullptr;
      // capture on the handle's own stream (the caller's may be the uncapturable legacy
      // default stream); the graph is then launched on the caller's stream
      cudaStream_t user = h->stream;
      h->stream = h->own_stream;
      CK(h, cudaStreamBeginCapture(h->own_stream, cudaStreamCaptureModeRelaxed));
      s = record_build(h, d_sel, v_r, lambda, 0, h->V, fused, ld, nullptr);
      if (s == WMD_OK) s = record_solve(h, d_r, v_r, lambda, iters, dist, fused, ld, nullptr, &launches);
      cudaGraph_t g = nullptr;
      const cudaError_t e = cudaStreamEndCapture(h->own_stream, &g);
      h->stream = user;
      if (s != WMD_OK) { if (g) cudaGraphDestroy(g); return s; }
      if (e != cudaSuccess) return cuda_fail(h, e, "cudaStreamEndCapture");
      const cudaError_t e2 = cudaGraphInstantiate(&h->graph_exec, g, 0);
      cudaGraphDestroy(g);
      if (e2 != cudaSuccess) { h->graph_exec = nullptr; return cuda_fail(h, e2, "cudaGraphInstantiate"); }
      h->graph_key = key;
      h->graph_launches = launches + 1;
    }
    CK(h, cudaGraphLaunch(h->graph_exec, h->stream));
    launches = h->graph_launches;
  } else {
    PhaseEvents* pe = new_phase_events(h);
    s = record_build(h, d_sel, v_r, lambda, 0, h->V, fused, ld, pe);
    if (s != WMD_OK) return s;
    s = record_solve(h, d_r, v_r, lambda, iters, dist, fused, ld, pe, &launches);
    if (s != WMD_OK) return s;
    ++launches;  // the build
  }
  note_query(h, d_sel, d_r, v_r, iters, fused, ld, launches);
  return WMD_OK;
}

// NEXT-2 (ii): a wmd_query_batch call is solved B queries per fused pass when every query takes
// the one-warp kernel for every document (no stopping tolerance, no graph mode). *bmax: queries
// per pass, WMD_OPT_BATCH or, by default, as many tables as fit in half the L2 (the pass is
// document-major, so the B tables are gathered concurrently), at most 16.
bool batch_eligible(wmd_handle* h, const std::vector<int32_t>& nrow, float lambda, int32_t* bmax) {
  const int32_t nq = (int32_t)nrow.size();
  if (nq < 2 || h->opt_batch == 1 || h->opt_graph || h->tol >= 0.0 || h->opt_path == WMD_PATH_PER_ITER ||
      lambda < wmd::kFusedMinLambda)
    return false;
  int32_t ldmax = 0;
  for (int32_t q = 0; q < nq; ++q) {
    const int32_t ld = wmd::fused_ld(nrow[q], layout_doc_nnz(h), false);
    if (ld <= 0 || ld > 64 || layout_doc_nnz(h) > wmd::warp_max_rows(ld)) return false;
    ldmax = std::max(ldmax, ld);
  }
  const double table = (double)h->V * (ldmax + 4) * 4;
  int32_t b = h->opt_batch >= 2 ? (int32_t)h->opt_batch : (int32_t)std::min(16.0, std::floor(64e6 / table));
  *bmax = std::max(1, std::min(b, nq));
  return *bmax >= 2;
}

// The batched passes: queries sorted (stably) by table width, then for each run of B queries of
// one width: a build per query into B side-by-side tables, one fused launch per length bucket
// for all B (each document's entries read once), then each query's re-runs of flagged
// documents (FP32 re-anchoring, FP64) as in a single query. Results equal single queries bit
// for bit (the per-(document, query) arithmetic is the same). svr / smap: pinned staging for
// the widths and the order (nq entries each).
wmd_status enqueue_batched(wmd_handle* h, const std::vector<int32_t>& nrow, int32_t* svr, int32_t* smap,
                           int32_t bmax, float lambda, int32_t iters, float* dist) {
  const int32_t nq = (int32_t)nrow.size();
  const int64_t N = h->N, V = h->V;
  cudaStream_t st = h->stream;
  std::vector<int32_t> ld(nq);
  for (int32_t q = 0; q < nq; ++q) ld[q] = wmd::fused_ld(nrow[q], layout_doc_nnz(h), false);
  std::vector<int32_t> order(nq);
  std::iota(order.begin(), order.end(), 0);
  std::stable_sort(order.begin(), order.end(), [&](int32_t x, int32_t y) { return ld[x] < ld[y]; });
  for (int32_t q = 0; q < nq; ++q) { svr[q] = nrow[q]; smap[q] = order[q]; }
  CK(h, h->bvr.ensure(nq));
  CK(h, h->bqmap.ensure(nq));
  CK(h, cudaMemcpyAsync(h->bvr.p, svr, nq * sizeof(int32_t), cudaMemcpyHostToDevice, st));
  CK(h, cudaMemcpyAsync(h->bqmap.p, smap, nq * sizeof(int32_t), cudaMemcpyHostToDevice, st));
  int32_t ldmax = 0;
  for (int32_t q = 0; q < nq; ++q) ldmax = std::max(ldmax, ld[q]);
  const int64_t stride = V * (ldmax + 4) + 128;
  CK(h, h->Mxb[0].ensure((size_t)bmax * stride));
  CK(h, h->Mxb[1].ensure((size_t)bmax * stride));
  // builds on the build stream, after the uploads; pass k's builds go to Mxb[k & 1] once pass
  // k - 2 (the last user of that buffer) is done, so they overlap the solve of pass k - 1
  CK(h, cudaEventRecord(h->up_ev, st));
  CK(h, cudaStreamWaitEvent(h->bstream, h->up_ev, 0));
  CK(h, h->bflags.ensure((size_t)bmax * N));
  CK(h, h->bflagged.ensure((size_t)bmax * N));
  CK(h, h->bcount.ensure(bmax));
  wmd::launch_fill_i32(h->iters_doc.p, N, iters, st);   // fixed iterations for every document
  int64_t launches = 1;
  const int32_t last = nq - 1;                          // flags / counts kept for the introspection calls
  int pass = 0;
  for (int32_t c0 = 0; c0 < nq; ++pass) {
    int32_t c1 = c0;
    while (c1 < nq && c1 - c0 < bmax && ld[order[c1]] == ld[order[c0]]) ++c1;
    const int32_t B = c1 - c0, w = ld[order[c0]];
    float* const mxb = h->Mxb[pass & 1].p;
    PhaseEvents* pe = new_phase_events(h);
    if (pass >= 2) CK(h, cudaStreamWaitEvent(h->bstream, h->mxb_free[pass & 1], 0));
    if (pe) CK(h, cudaEventRecord(pe->ev[0], h->bstream));
    for (int32_t q = 0; q < B; ++q) {
      const int32_t g = order[c0 + q];
      build_rows(h, h->bsel.p + (size_t)g * WMD_MAX_VR, nrow[g], w, lambda, nullptr, mxb + q * stride, 0, V,
                 h->bstream);
    }
    launches += B;
    DBG_PHASE(h, h->bstream, "batched distance builds");
    CK(h, cudaEventRecord(h->built_ev, h->bstream));
    CK(h, cudaStreamWaitEvent(st, h->built_ev, 0));
    // phase timing: the solve starts here (build_ms then includes any wait for the previous solve)
    if (pe) CK(h, cudaEventRecord(pe->ev[1], st));
    CK(h, cudaMemsetAsync(h->bflags.p, 0, (size_t)B * N, st));
    CK(h, cudaMemsetAsync(h->bcount.p, 0, B * sizeof(int32_t), st));
    wmd::QuerySet qs{};
    qs.Mx = mxb;
    qs.mx_stride = stride;
    qs.rpad = h->brpad.p;
    qs.qmap = h->bqmap.p + c0;
    qs.vr = h->bvr.p;
    qs.nq = B;
    qs.N = N;
    qs.dist = dist;
    qs.flags = h->bflags.p;
    qs.iters_doc = nullptr;
    qs.flagged_list = h->bflagged.p;
    qs.flagged_count = h->bcount.p;
    const int nb = wmd::fused_launch_count(h->len_prefix.data(), h->max_doc_nnz, N, layout_docs(h), w, -1.f);
    wmd::StreamRing ring;
    if (nb > 1) {
      ring.s = h->lanes;
      ring.n = std::min(nb, (int)wmd_handle::kLanes);
      CK(h, cudaEventRecord(h->fork_ev, st));
      for (int i = 0; i < ring.n; ++i) CK(h, cudaStreamWaitEvent(h->lanes[i], h->fork_ev, 0));
    }
    wmd::launch_sinkhorn_fused(h->sdoc.p, h->ent.p, N, layout_docs(h), h->len_prefix.data(), h->max_doc_nnz, w, qs, lambda, iters,
                               -1.f, st, &ring);
    DBG_PHASE(h, st, "batched fused Sinkhorn kernels");
    for (int i = 0; i < ring.n; ++i) {
      CK(h, cudaEventRecord(h->join_ev[i], h->lanes[i]));
      CK(h, cudaStreamWaitEvent(st, h->join_ev[i], 0));
    }
    launches += nb;
    h->st.iter_launches += nb;
    if (pe) { CK(h, cudaEventRecord(pe->ev[2], st)); CK(h, cudaEventRecord(pe->ev[3], st)); }
    for (int32_t q = 0; q < B && h->opt_fallback; ++q) {
      const int32_t g = order[c0 + q];
      const float* mxq = mxb + q * stride;
      const float* rq = h->brpad.p + (size_t)g * WMD_MAX_VR;
      float* dq = dist + (size_t)g * N;
      uint8_t* fq = h->bflags.p + (size_t)q * N;
      const int32_t* fl = h->bflagged.p + (size_t)q * N;
      int32_t* fc = h->bcount.p + q;
      if (wmd::cta_rerun_supported(w)) {
        CK(h, cudaMemsetAsync(h->counters.p + 4, 0, sizeof(int32_t), st));
        wmd::launch_cta_rerun(fl, fc, h->doc_ptr.p, h->ent.p, mxq, w, nrow[g], rq, lambda, iters, nullptr, dq, fq,
                              h->flagged2.p, h->counters.p + 4, st);
        ++launches;
        fl = h->flagged2.p;
        fc = h->counters.p + 4;
      }
      wmd::launch_fallback_fp64(mxq, w, rq, nrow[g], (double)lambda, iters, -1.f, nullptr, h->doc_ptr.p, h->ent.p,
                                fl, fc, h->fb_scratch.p, h->max_doc_nnz, dq, fq, h->counters.p + 1,
                                h->counters.p + 2, st);
      ++launches;
    }
    DBG_PHASE(h, st, "batched re-runs");
    CK(h, cudaEventRecord(h->mxb_free[pass & 1], st));
    if (pe) {
      CK(h, cudaEventRecord(pe->ev[4], st));
      pe->complete = true;
    }
    // the last query's flags and flagged count (wmd_read_flags / wmd_sync report the last query)
    for (int32_t q = 0; q < B; ++q)
      if (order[c0 + q] == last) {
        CK(h, cudaMemcpyAsync(h->flags.p, h->bflags.p + (size_t)q * N, N, cudaMemcpyDeviceToDevice, st));
        CK(h, cudaMemcpyAsync(h->counters.p, h->bcount.p + q, sizeof(int32_t), cudaMemcpyDeviceToDevice, st));
      }
    c0 = c1;
  }
  CK(h, cudaGetLastError());
  h->kt_valid = false;
  h->u_valid = false;
  h->path_used = WMD_PATH_FUSED;
  h->v_r = nrow[last];
  h->ld = ld[last];
  h->last_sel = h->bsel.p + (size_t)last * WMD_MAX_VR;
  h->last_r = h->brpad.p + (size_t)last * WMD_MAX_VR;
  h->st.queries += nq;
  h->st.kernel_launches += launches;
  h->st.last_v_r = nrow[last];
  h->st.last_ld = ld[last];
  h->st.last_path = WMD_PATH_FUSED;
  h->st.last_build = h->build_used;
  return WMD_OK;
}

wmd_status check_query_args(wmd_handle* h, const void* out_dist, float lambda, int32_t iters) {
  if (!h->has_targets) return fail(h, WMD_ERR_STATE, "query before wmd_set_targets");
  if (!out_dist || !(lambda > 0.f) || !std::isfinite(lambda) || iters < 0)
    return fail(h, WMD_ERR_INVALID_ARGUMENT, "out_dist NULL, lambda not finite > 0, or iters < 0");
  return WMD_OK;
}

}  // namespace

extern "C" {

wmd_status wmd_query(wmd_handle* h, const int32_t* query_ids, const float* query_weights,
                     int32_t n, float lambda, int32_t iters, float* out_dist) {
  if (!h) return WMD_ERR_INVALID_ARGUMENT;
  h->err.clear();
  wmd_status s = check_query_args(h, out_dist, lambda, iters);
  if (s != WMD_OK) return s;
  int64_t bad = -1;
  std::string msg;
  s = validate_query(query_ids, query_weights, n, h->V, &bad, &msg, &h->h_sel, &h->h_r);
  if (s != WMD_OK) return fail(h, s, "%s", msg.c_str());
  DeviceGuard g(h->device);
  if (!g.ok) return fail(h, WMD_ERR_CUDA, "cudaSetDevice failed");
  cudaStream_t st = h->stream;

  // Upload (sel, r padded with zeros) from pinned staging, double-buffered.
  const int slot = h->stage_slot;
  h->stage_slot ^= 1;
  CK(h, cudaEventSynchronize(h->stage_ev[slot]));
  int32_t* ssel = (int32_t*)h->stage[slot];
  float* sr = (float*)((char*)h->stage[slot] + WMD_MAX_VR * 4);
  std::memset(h->stage[slot], 0, WMD_MAX_VR * 8);
  for (int32_t i = 0; i < n; ++i) { ssel[i] = h->h_sel[i]; sr[i] = h->h_r[i]; }
  const bool dev_out = is_device_ptr(out_dist);
  float* dist = dev_out ? out_dist : h->dist_tmp.p;
  // (single queries run build and solve on one stream: overlapping the next query's build with
  // this solve, as wmd_query_batch does, measured slower at Scaling)
  CK(h, cudaMemcpyAsync(h->sel.p, ssel, WMD_MAX_VR * 4, cudaMemcpyHostToDevice, st));
  CK(h, cudaMemcpyAsync(h->rpad.p, sr, WMD_MAX_VR * 4, cudaMemcpyHostToDevice, st));
  CK(h, cudaEventRecord(h->stage_ev[slot], st));
  s = enqueue_query(h, h->sel.p, h->rpad.p, n, lambda, iters, dist);
  if (s != WMD_OK) return s;
  if (!dev_out) {
    CK(h, cudaMemcpyAsync(out_dist, dist, h->N * sizeof(float), cudaMemcpyDeviceToHost, st));
    CK(h, cudaStreamSynchronize(st));
  }
  return WMD_OK;
}

wmd_status wmd_query_batch(wmd_handle* h, const int32_t* query_ids, const float* query_weights,
                           const int64_t* q_ptr, int32_t nq, float lambda, int32_t iters,
                           float* out_dist) {
  if (!h) return WMD_ERR_INVALID_ARGUMENT;
  h->err.clear();
  wmd_status s = check_query_args(h, out_dist, lambda, iters);
  if (s != WMD_OK) return s;
  if (nq < 1 || !q_ptr || q_ptr[0] != 0) return fail(h, WMD_ERR_INVALID_ARGUMENT, "nq < 1 or q_ptr[0] != 0");
  for (int32_t q = 0; q < nq; ++q)
    if (q_ptr[q + 1] < q_ptr[q]) return fail(h, WMD_ERR_INVALID_ARGUMENT, "q_ptr decreases at query %d", q);
  DeviceGuard g(h->device);
  if (!g.ok) return fail(h, WMD_ERR_CUDA, "cudaSetDevice failed");
  cudaStream_t st = h->stream;
  // validate and sort every query before any work is enqueued (all-or-nothing)
  CK(h, cudaEventSynchronize(h->batch_ev));  // the previous batch's upload has left the staging
  const size_t need = (size_t)nq * WMD_MAX_VR * 8 + (size_t)nq * 8;  // ids, weights, widths, order
  if (h->batch_stage_bytes < need) {
    if (h->batch_stage) cudaFreeHost(h->batch_stage);
    h->batch_stage = nullptr;
    h->batch_stage_bytes = 0;
    CK(h, cudaMallocHost(&h->batch_stage, need));
    h->batch_stage_bytes = need;
  }
  int32_t* ssel = (int32_t*)h->batch_stage;
  float* sr = (float*)((char*)h->batch_stage + (size_t)nq * WMD_MAX_VR * 4);
  std::memset(h->batch_stage, 0, need);
  std::vector<int32_t> nrow(nq);
  for (int32_t q = 0; q < nq; ++q) {
    int64_t bad = -1;
    std::string msg;
    const int64_t n = q_ptr[q + 1] - q_ptr[q];
    if (n > WMD_MAX_VR) return fail(h, WMD_ERR_INVALID_ARGUMENT, "query %d: v_r > WMD_MAX_VR", q);
    s = validate_query(query_ids + q_ptr[q], query_weights + q_ptr[q], (int32_t)n, h->V, &bad, &msg,
                       &h->h_sel, &h->h_r);
    if (s != WMD_OK) return fail(h, s, "query %d: %s", q, msg.c_str());
    nrow[q] = (int32_t)n;
    for (int64_t i = 0; i < n; ++i) {
      ssel[(size_t)q * WMD_MAX_VR + i] = h->h_sel[i];
      sr[(size_t)q * WMD_MAX_VR + i] = h->h_r[i];
    }
  }
  CK(h, h->bsel.ensure((size_t)nq * WMD_MAX_VR));
  CK(h, h->brpad.ensure((size_t)nq * WMD_MAX_VR));
  CK(h, cudaMemcpyAsync(h->bsel.p, ssel, (size_t)nq * WMD_MAX_VR * 4, cudaMemcpyHostToDevice, st));
  CK(h, cudaMemcpyAsync(h->brpad.p, sr, (size_t)nq * WMD_MAX_VR * 4, cudaMemcpyHostToDevice, st));
  const bool dev_out = is_device_ptr(out_dist);
  if (!dev_out) CK(h, h->batch_dist.ensure((size_t)nq * h->N));
  float* dist = dev_out ? out_dist : h->batch_dist.p;
  // NEXT-2 (ii): B queries per fused pass when every query takes the one-warp kernel
  int32_t bmax = 0;
  if (batch_eligible(h, nrow, lambda, &bmax)) {
    int32_t* svr = (int32_t*)((char*)h->batch_stage + (size_t)nq * WMD_MAX_VR * 8);
    int32_t* smap = svr + nq;
    s = enqueue_batched(h, nrow, svr, smap, bmax, lambda, iters, dist);
    CK(h, cudaEventRecord(h->batch_ev, st));
    if (s != WMD_OK) return s;
    if (!dev_out) {
      CK(h, cudaMemcpyAsync(out_dist, dist, (size_t)nq * h->N * sizeof(float), cudaMemcpyDeviceToHost, st));
      CK(h, cudaStreamSynchronize(st));
    }
    return WMD_OK;
  }
  CK(h, cudaEventRecord(h->batch_ev, st));
  // Build/solve overlap: when every query takes the fused path, query q's
  // table is built on the handle's build stream into one of two tables while query q-1 is
  // solved on the main stream (the build is latency-bound and leaves most of the GPU idle).
  bool overlap = nq > 1 && !h->opt_graph && h->opt_path != WMD_PATH_PER_ITER;
  size_t mx_need = 0;
  for (int32_t q = 0; overlap && q < nq; ++q) {
    const int32_t ld = lambda >= wmd::kFusedMinLambda ? wmd::fused_ld(nrow[q], layout_doc_nnz(h), h->tol >= 0.0) : 0;
    if (ld <= 0) overlap = false;
    mx_need = std::max(mx_need, (size_t)h->V * (ld + 4) + 128);
  }
  if (!overlap) {
    for (int32_t q = 0; q < nq; ++q) {
      s = enqueue_query(h, h->bsel.p + (size_t)q * WMD_MAX_VR, h->brpad.p + (size_t)q * WMD_MAX_VR, nrow[q],
                        lambda, iters, dist + (size_t)q * h->N);
      if (s != WMD_OK) return s;
    }
  } else {
    CK(h, h->Mx.ensure(mx_need));
    CK(h, h->Mx2.ensure(mx_need));
    CK(h, cudaStreamWaitEvent(h->bstream, h->batch_ev, 0));  // the uploaded query rows
    for (int32_t q = 0; q < nq; ++q) {
      swap_units(h);
      s = enqueue_overlapped(h, h->bsel.p + (size_t)q * WMD_MAX_VR, h->brpad.p + (size_t)q * WMD_MAX_VR,
                             nrow[q], lambda, iters, dist + (size_t)q * h->N, nullptr);
      if (s != WMD_OK) return s;
    }
  }
  if (!dev_out) {
    CK(h, cudaMemcpyAsync(out_dist, dist, (size_t)nq * h->N * sizeof(float), cudaMemcpyDeviceToHost, st));
    CK(h, cudaStreamSynchronize(st));
  }
  return WMD_OK;
}

wmd_status wmd_query_begin(wmd_handle* h, const int32_t* query_ids, const float* query_weights, int32_t n,
                           float lambda, int32_t iters, int64_t row_begin, int64_t row_end, int64_t table_rows) {
  if (!h) return WMD_ERR_INVALID_ARGUMENT;
  h->err.clear();
  h->pq.active = false;
  wmd_status s = check_query_args(h, (const void*)1, lambda, iters);
  if (s != WMD_OK) return s;
  if (row_begin < 0 || row_end < row_begin || row_end > h->V || table_rows < 0)
    return fail(h, WMD_ERR_INVALID_ARGUMENT, "row range [%lld, %lld) outside [0, V)", (long long)row_begin,
                (long long)row_end);
  int64_t bad = -1;
  std::string msg;
  s = validate_query(query_ids, query_weights, n, h->V, &bad, &msg, &h->h_sel, &h->h_r);
  if (s != WMD_OK) return fail(h, s, "%s", msg.c_str());
  DeviceGuard g(h->device);
  if (!g.ok) return fail(h, WMD_ERR_CUDA, "cudaSetDevice failed");
  cudaStream_t st = h->stream;
  const int slot = h->stage_slot;
  h->stage_slot ^= 1;
  CK(h, cudaEventSynchronize(h->stage_ev[slot]));
  int32_t* ssel = (int32_t*)h->stage[slot];
  float* sr = (float*)((char*)h->stage[slot] + WMD_MAX_VR * 4);
  std::memset(h->stage[slot], 0, WMD_MAX_VR * 8);
  for (int32_t i = 0; i < n; ++i) { ssel[i] = h->h_sel[i]; sr[i] = h->h_r[i]; }
  CK(h, cudaMemcpyAsync(h->sel.p, ssel, WMD_MAX_VR * 4, cudaMemcpyHostToDevice, st));
  CK(h, cudaMemcpyAsync(h->rpad.p, sr, WMD_MAX_VR * 4, cudaMemcpyHostToDevice, st));
  CK(h, cudaEventRecord(h->stage_ev[slot], st));
  bool fused = false;
  int32_t ld = 0;
  s = prepare_query(h, n, lambda, table_rows, &fused, &ld);
  if (s != WMD_OK) return s;
  PhaseEvents* pe = new_phase_events(h);
  s = record_build(h, h->sel.p, n, lambda, row_begin, row_end, fused, ld, pe);
  if (s != WMD_OK) return s;
  h->pq.active = true;
  h->pq.fused = fused;
  h->pq.v_r = n;
  h->pq.ld = ld;
  h->pq.iters = iters;
  h->pq.lambda = lambda;
  h->pq.pe = pe;
  return WMD_OK;
}

wmd_status wmd_query_tables(wmd_handle* h, float** mx, int32_t* mx_row_floats, float** kt,
                            int32_t* kt_row_floats) {
  if (!h || !mx || !mx_row_floats) return WMD_ERR_INVALID_ARGUMENT;
  if (!h->pq.active) return fail(h, WMD_ERR_STATE, "no query begun");
  *mx = h->Mx.p;
  *mx_row_floats = h->pq.ld + 4;
  if (kt) *kt = h->pq.fused ? nullptr : h->Kt.p;
  if (kt_row_floats) *kt_row_floats = h->pq.fused ? 0 : h->pq.ld;
  return WMD_OK;
}

wmd_status wmd_query_finish(wmd_handle* h, float* out_dist) {
  if (!h) return WMD_ERR_INVALID_ARGUMENT;
  if (!h->pq.active) return fail(h, WMD_ERR_STATE, "wmd_query_finish without wmd_query_begin");
  if (!out_dist) return fail(h, WMD_ERR_INVALID_ARGUMENT, "out_dist NULL");
  DeviceGuard g(h->device);
  if (!g.ok) return fail(h, WMD_ERR_CUDA, "cudaSetDevice failed");
  h->pq.active = false;
  const bool dev_out = is_device_ptr(out_dist);
  float* dist = dev_out ? out_dist : h->dist_tmp.p;
  int64_t launches = 0;
  wmd_status s = record_solve(h, h->rpad.p, h->pq.v_r, h->pq.lambda, h->pq.iters, dist, h->pq.fused,
                              h->pq.ld, h->pq.pe, &launches);
  if (s != WMD_OK) return s;
  note_query(h, h->sel.p, h->rpad.p, h->pq.v_r, h->pq.iters, h->pq.fused, h->pq.ld, launches + 1);
  if (!dev_out) {
    CK(h, cudaMemcpyAsync(out_dist, dist, h->N * sizeof(float), cudaMemcpyDeviceToHost, h->stream));
    CK(h, cudaStreamSynchronize(h->stream));
  }
  return WMD_OK;
}

wmd_status wmd_sync(wmd_handle* h) {
  if (!h) return WMD_ERR_INVALID_ARGUMENT;
  DeviceGuard g(h->device);
  CK(h, cudaStreamSynchronize(h->stream));
  if (!h->has_targets || h->st.queries == 0) return WMD_OK;
  int32_t c[3] = {0, 0, 0};
  CK(h, cudaMemcpy(c, h->counters.p, sizeof c, cudaMemcpyDeviceToHost));
  // c[0]: flagged documents of the last query; c[1] breakdown latch and c[2] FP64 re-runs
  // accumulate on the device until this sync.
  h->st.flagged_docs = c[0];
  h->st.fallback_docs += c[2];
  int32_t z[2] = {0, 0};
  CK(h, cudaMemcpy(h->counters.p + 1, z, sizeof z, cudaMemcpyHostToDevice));
  if (c[1]) return fail(h, WMD_ERR_NUMERICAL_BREAKDOWN, "a distance stayed non-finite after the FP64 re-run");
  return WMD_OK;
}

wmd_status wmd_get_stats(wmd_handle* h, wmd_stats* out) {
  if (!h || !out) return WMD_ERR_INVALID_ARGUMENT;
  DeviceGuard g(h->device);
  CK(h, fold_events(h, true));
  wmd_stats s = h->st;
  s.build_ms = h->phase_ms[0];
  s.iter_ms = h->phase_ms[1];
  s.final_ms = h->phase_ms[2];
  s.fallback_ms = h->phase_ms[3];
  s.query_ms = h->phase_ms[4];
  s.timing_valid = h->phase_n > 0;
  *out = s;
  return WMD_OK;
}

wmd_status wmd_reset_stats(wmd_handle* h) {
  if (!h) return WMD_ERR_INVALID_ARGUMENT;
  DeviceGuard g(h->device);
  cudaStreamSynchronize(h->stream);
  for (auto& pe : h->events) {
    if (h->pq.active && h->pq.pe == &pe) continue;  // still owned by a begun two-phase query
    pe.complete = false;
    h->event_pool.push_back(pe);
  }
  if (h->pq.active && h->pq.pe) {
    PhaseEvents keep = *h->pq.pe;
    h->events.clear();
    h->events.push_back(keep);
    h->pq.pe = &h->events.back();
  } else {
    h->events.clear();
  }
  for (double& x : h->phase_ms) x = 0.0;
  h->phase_n = 0;
  h->st = wmd_stats{};
  return WMD_OK;
}

wmd_status wmd_get_query_rows(wmd_handle* h, int32_t* sel, float* r) {
  if (!h || !sel || !r) return WMD_ERR_INVALID_ARGUMENT;
  if (h->st.queries == 0) return fail(h, WMD_ERR_STATE, "no query yet");
  DeviceGuard g(h->device);
  CK(h, cudaStreamSynchronize(h->stream));
  CK(h, cudaMemcpy(sel, h->last_sel, h->v_r * sizeof(int32_t), cudaMemcpyDeviceToHost));
  CK(h, cudaMemcpy(r, h->last_r, h->v_r * sizeof(float), cudaMemcpyDeviceToHost));
  return WMD_OK;
}

wmd_status wmd_read_kernel(wmd_handle* h, int64_t k0, int64_t count, float* ktilde, float* m,
                           float* colmin) {
  if (!h || k0 < 0 || count < 0 || k0 + count > h->V) return WMD_ERR_INVALID_ARGUMENT;
  if (h->st.queries == 0) return fail(h, WMD_ERR_STATE, "no query yet");
  DeviceGuard g(h->device);
  CK(h, cudaStreamSynchronize(h->stream));
  const size_t row = (size_t)h->ld, rowx = row + 4;
  if (ktilde && !h->kt_valid)
    return fail(h, WMD_ERR_STATE, "K~ table not built by the last query (fused path builds M only)");
  if (ktilde) CK(h, cudaMemcpy(ktilde, h->Kt.p + k0 * row, count * row * 4, cudaMemcpyDeviceToHost));
  if (m && count > 0)
    CK(h, cudaMemcpy2D(m, row * 4, h->Mx.p + k0 * rowx, rowx * 4, row * 4, count, cudaMemcpyDeviceToHost));
  if (colmin && count > 0)  // m_k is column ld of the Mx rows
    CK(h, cudaMemcpy2D(colmin, 4, h->Mx.p + k0 * rowx + row, rowx * 4, 4, count, cudaMemcpyDeviceToHost));
  return WMD_OK;
}

wmd_status wmd_read_scaling(wmd_handle* h, int64_t j0, int64_t count, float* u) {
  if (!h || !u || j0 < 0 || count < 0 || j0 + count > h->N) return WMD_ERR_INVALID_ARGUMENT;
  if (!h->u_valid) return fail(h, WMD_ERR_STATE, "no per-iteration u available (fused path or iters == 0)");
  DeviceGuard g(h->device);
  CK(h, cudaStreamSynchronize(h->stream));
  CK(h, cudaMemcpy(u, h->u_last + j0 * h->ld, count * h->ld * 4, cudaMemcpyDeviceToHost));
  return WMD_OK;
}

wmd_status wmd_set_tolerance(wmd_handle* h, double tol) {
  if (!h) return WMD_ERR_INVALID_ARGUMENT;
  if (std::isnan(tol)) return fail(h, WMD_ERR_INVALID_ARGUMENT, "tolerance is NaN");
  h->tol = tol;
  return WMD_OK;
}

wmd_status wmd_read_iterations(wmd_handle* h, int32_t* iters_out) {
  if (!h || !iters_out) return WMD_ERR_INVALID_ARGUMENT;
  if (!h->has_targets || h->st.queries == 0) return fail(h, WMD_ERR_STATE, "no query yet");
  DeviceGuard g(h->device);
  CK(h, cudaStreamSynchronize(h->stream));
  CK(h, cudaMemcpy(iters_out, h->iters_doc.p, h->N * sizeof(int32_t), cudaMemcpyDeviceToHost));
  return WMD_OK;
}

wmd_status wmd_read_flags(wmd_handle* h, uint8_t* flags) {
  if (!h || !flags) return WMD_ERR_INVALID_ARGUMENT;
  if (!h->has_targets) return fail(h, WMD_ERR_STATE, "no targets");
  DeviceGuard g(h->device);
  CK(h, cudaStreamSynchronize(h->stream));
  CK(h, cudaMemcpy(flags, h->flags.p, h->N, cudaMemcpyDeviceToHost));
  return WMD_OK;
}

}  // extern "C"
