// Internal interface between the host runtime (wmd_host.cpp) and the CUDA kernels
// (wmd_kernels.cu). Not installed; not part of the C ABI (include/wmd.h is).
#pragma once
#include <atomic>
#include <cstdint>
#include <cuda_runtime.h>

#include "wmd.h"

#define WMD_MAX_VR_DEV WMD_MAX_VR

namespace wmd {

// Per-device cache of a launch setting (function attributes and occupancy belong to a device
// context, so a handle on a second GPU in the same process must not reuse the first GPU's).
// Slot dev holds value + 1 once computed; `compute` runs on the current device. Two threads
// racing on an empty slot both compute (cudaFuncSetAttribute is idempotent) and store the
// same value. Static instances are zero-initialised (trivial std::atomic constructor).
struct PerDevice {
  static constexpr int kMaxDevices = 64;
  std::atomic<int> slot[kMaxDevices];
  template <class F>
  int get(F&& compute) {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDevices) return compute();
    const int x = slot[dev].load(std::memory_order_acquire);
    if (x) return x - 1;
    const int v = compute();
    slot[dev].store(v + 1, std::memory_order_release);
    return v;
  }
};

// Multiprocessor count of the current device (148 on B200).
inline int device_sms() {
  static PerDevice cache;
  return cache.get([] {
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    return sms > 0 ? sms : 148;
  });
}

// One CSC nonzero of the target matrix c: vocabulary word k and weight c_kj, packed so a
// lane fetches both with one 8-byte load (D1 in SURVEY.md §2.4).
struct Entry {
  int32_t k;
  float c;
};

// Flag bits per document.
constexpr uint8_t kFlagFp32Range = 1;  // an FP32 iterate left the normal range
constexpr uint8_t kFlagFp64 = 2;       // recomputed in FP64
constexpr uint8_t kFlagRerun = 4;      // recomputed in FP32 by the one-CTA kernel (re-anchoring)
constexpr uint8_t kFlagUnderflow = 16; // the one-warp kernel's FP32 block had entries below
                                       // FLT_MIN: the range certificate was in force

// Device-side per-query scalars the kernels read (written by one H2D copy per query).
struct QueryDev {
  int32_t v_r;
  int32_t ld;          // row stride of K~ / M / u (floats), v_r rounded up to 8
  float lambda;
  int32_t iters;
};

// --- a2: distance + column-rescaled kernel build -------
// Mx: V rows of ld + 4 floats [M_k0 .. M_k,ld-1 (zero beyond v_r), m_k = min_i M_ik, 0, 0, 0].
// Kt (V x ld, K~ = exp(-lambda (M - m))) is written only when non-null (per-iteration path).
// Rows [row0, row1) only (a rank's share of a sharded build); E: rows of dp floats (d padded
// with zeros to a multiple of 32). use_tc: tensor-core 3xTF32 GEMM form, else SIMT.
void launch_build_ktilde(const float* E, int64_t row0, int64_t row1, int dp, const int32_t* sel, int v_r,
                         int ld, float lambda, float* Kt, float* Mx, bool use_tc, cudaStream_t st);

// Exact build (wmd_build_exact.cu): E in fixed point, n = rint(E 2^frac_bits), as four byte-limb
// planes limbs[limb][dp/16][V][16 B] (chunk-major: the TMA boxes of 128 rows are contiguous) and
// nn[k] = sum_t n_kt^2 (int64); tmap: the planes' 4-D TMA descriptor (a CUtensorMap).
struct ExactE {
  uint8_t* limbs = nullptr;
  long long* nn = nullptr;
  int64_t V = 0;
  int dp = 0;
  int frac_bits = 0;
  float inv_scale = 1.f;  // 2^-frac_bits
  bool ok = false;        // tables built (false: unsupported dp / range; the build is unavailable)
  alignas(64) unsigned char tmap[128] = {};
};
bool exact_build_supported(int dp);
int exact_frac_bits_limit(int dp);
// (Re)builds *x from E (V x dp, device) on st; synchronises st once (max |E|). Returns a
// cudaError_t value (0 also when the shape is unsupported: x->ok stays false).
int prepare_exact_e(const float* E, int64_t V, int dp, ExactE* x, cudaStream_t st);
void free_exact_e(ExactE* x);
// Same contract as launch_build_ktilde (x.ok required). Returns false, launching nothing, when
// the query's limbs do not fit in shared memory (dp * 128 B per 32 query rows).
bool launch_build_exact(const ExactE& x, int64_t row0, int64_t row1, const int32_t* sel, int v_r, int ld,
                        float lambda, float* Kt, float* Mx, cudaStream_t st);

// "While x changes" (NEXT-3): tol < 0 runs the fixed iteration count. Otherwise a
// document stops after the first x-update with max_i |x_new/x - 1| <= tol (R31);
// conv[j] marks it (per-iteration path), iters_doc[j] receives its number of x-updates.
struct ConvParams {
  float tol;
  uint8_t* conv;
  int32_t* iters_doc;
  int it_index;  // index of this x-update (per-iteration path)
};

// --- a4: one fused SDDMM_SpMM iteration for all documents ------------
// u_in == nullptr: first iteration with the constant u0 = 1/x0 = v_r.
// `order` lists the documents sorted by length (processing order only; results are per document).
void launch_sddmm_spmm_iter(const int32_t* order, const int32_t* doc_ptr, const Entry* ent, int64_t N,
                            const float* Kt, int ld, int v_r, const float* rpad, const float* u_in,
                            float* u_out, uint32_t* umask, uint8_t* flags, ConvParams cv,
                            cudaStream_t st);

// --- a5: final u/v/WMD step -----------------------------------
void launch_final_wmd(const int32_t* order, const int32_t* doc_ptr, const Entry* ent, int64_t N,
                      const float* Kt, const float* Mt, int ld, int v_r, const float* rpad,
                      const float* u_in, const uint32_t* umask, float* dist, uint8_t* flags,
                      int32_t* flagged_list, int32_t* flagged_count, cudaStream_t st);

// --- NEXT-1: all iterations + final step in one launch (wmd_fused.cu) ------------------------
// The fused kernels recover M from the block in the final step (D = mu - log2(Kh) / alpha), whose
// absolute error ~2^-22 / alpha grows as lambda shrinks (1.5e-3 of the distance at lambda = 1e-6,
// ~1e-6 at 1e-3): below kFusedMinLambda the per-iteration path, whose final step reads M, runs.
constexpr float kFusedMinLambda = 1e-3f;
// Returns false if the shape is not supported by the fused kernel (the caller then uses the
// per-iteration path). `len_prefix` (host, max_len + 2 entries): len_prefix[L] = number of
// documents with fewer than L nonzeros, i.e. bucket boundaries in the length-sorted `order`.
// Row width of the fused path's tables for query length v_r and longest document max_doc_nnz
// (8 CW, CW in {1, 2, 3, 4, 5, 6, 8}; cta_ld(v_r) when a document needs the one-CTA kernel),
// or 0 if the fused path does not take the shape (the caller then uses the per-iteration path).
// conv: a per-document stopping tolerance is set (one-warp kernel only).
int fused_ld(int v_r, int64_t max_doc_nnz, bool conv);
int warp_max_rows(int ld);  // longest document of the one-warp kernel at row width ld
// Streams the length buckets are launched on (round robin; the caller forks them from and joins
// them to its stream) so that one bucket's tail overlaps the next bucket; n = 0: all on `st`.
struct StreamRing {
  const cudaStream_t* s = nullptr;
  int n = 0;
  int k = 0;
  cudaStream_t next(cudaStream_t st) { return n ? s[k++ % n] : st; }
};
// The queries one fused launch solves (NEXT-2 (ii), "one tweet vs a day of tweets"):
// nq queries against the same documents, each document's entries read once for all of them.
// Query q (0 <= q < nq) has a caller index g = qmap ? qmap[q] : q and: table Mx + q * mx_stride,
// weights rpad + g * WMD_MAX_VR (zero padded), width vr ? vr[g] : v_r, distances dist + g * N;
// its flags (flags + q * N), iteration counts (iters_doc + q * N) and flagged documents
// (flagged_list + q * N, count flagged_count[q]) are batch-local. nq = 1, qmap = vr = nullptr is
// a single query (wmd_query).
struct QuerySet {
  const float* Mx;
  int64_t mx_stride;
  const float* rpad;
  const int32_t* qmap;     // device, nq entries, or nullptr
  const int32_t* vr;       // device, indexed by g, or nullptr (every query has width v_r)
  int32_t v_r;
  int32_t nq;
  int64_t N;
  float* dist;
  uint8_t* flags;
  int32_t* iters_doc;      // may be nullptr
  int32_t* flagged_list;
  int32_t* flagged_count;
};

// sdoc[p] = {document id, first nonzero, length, 0} of the p-th document in length order.
// qs.nq > 1 needs every document within the one-warp kernel's rows (warp_max_rows(ld)).
void launch_sinkhorn_fused(const int4* sdoc, const Entry* ent, int64_t N, int64_t layout_docs,
                           const int64_t* len_prefix, int64_t max_len, int ld, const QuerySet& qs,
                           float lambda, int iters, float tol, cudaStream_t st, StreamRing* ring = nullptr);
int fused_launch_count(const int64_t* len_prefix, int64_t max_len, int64_t N, int64_t layout_docs, int ld, float tol);
// Short documents, two per warp (wmd_fused_half.cu): ld in {16, 24, 32, 40}, fixed iteration count
// (tol < 0), corpora of at least kHalfMinDocs documents (layout_docs: max(local N,
// WMD_OPT_LAYOUT_DOCS)); WMD_FUSED_HALF=0 / 1 in the environment disables it / lifts the
// corpus-size condition.
constexpr int64_t kHalfMinDocs = 32768;
bool use_half(int ld, float tol, int64_t layout_docs);
int half_max_rows();
// Launches the half-warp buckets over the length-sorted documents from position 0 while they fit
// (<= half_max_rows() nonzeros); returns the first position not covered. sdoc == nullptr: only
// counts the launches (into *launches).
int64_t launch_sinkhorn_half(const int4* sdoc, const Entry* ent, int64_t N, const int64_t* len_prefix,
                             int64_t max_len, int ld, const QuerySet& qs, float lambda, int iters,
                             cudaStream_t st0, StreamRing* ring, int* launches);

// --- NEXT-1, long documents: one CTA of ceil(n/32) warps per document (wmd_fused_cta.cu) -----
int cta_max_rows();  // longest document the one-CTA kernel takes
int cta_ld(int v_r);  // its table row width for v_r query rows: 8 CW, CW in {4, 5, 6, 8, 10, 12, 13, 16}
// Documents [p0, N) of the length-sorted order, ld = cta_ld(v_r), fixed iteration count.
void launch_sinkhorn_cta(const int4* sdoc, const Entry* ent, int64_t p0, int64_t N, const int64_t* len_prefix,
                         int64_t max_len, const float* Mx, int ld, int v_r, const float* rpad, float lambda,
                         int iters, int32_t* iters_doc, float* dist, uint8_t* flags, int32_t* flagged_list,
                         int32_t* flagged_count, cudaStream_t st, StreamRing* ring = nullptr);
int cta_launch_count(int64_t p0, int64_t N, const int64_t* len_prefix, int64_t max_len);
// Re-run (FP32, re-anchoring) of the documents of a device list (ids[0 .. *count)) that the
// one-warp kernel flagged, for ld in {32, 40, 48, 64}; documents that still fail (or are longer
// than 64 words) are appended to out_list / *out_count for the FP64 re-run.
bool cta_rerun_supported(int ld);
void launch_cta_rerun(const int32_t* ids, const int32_t* count, const int32_t* doc_ptr, const Entry* ent,
                      const float* Mx, int ld, int v_r, const float* rpad, float lambda, int iters,
                      int32_t* iters_doc, float* dist, uint8_t* flags, int32_t* out_list, int32_t* out_count,
                      cudaStream_t st);

// --- a6: FP64 re-run of flagged documents (no CPU fallback) --------------------------------
constexpr int kFallbackBlocks = 296;  // 2 per SM (1 per SM for documents whose K needs > 100 KB)
size_t fallback_scratch_bytes(int64_t max_doc_nnz);
void launch_fallback_fp64(const float* Mx, int ld, const float* rpad, int v_r,
                          double lambda, int iters, float tol, int32_t* iters_doc,
                          const int32_t* doc_ptr, const Entry* ent,
                          const int32_t* flagged_list, const int32_t* flagged_count,
                          double* scratch, int64_t max_doc_nnz, float* dist, uint8_t* flags,
                          int32_t* breakdown, int32_t* fallback_count, cudaStream_t st);

// --- validation helpers (device-resident inputs) -------------------------------------------
void launch_check_finite(const float* x, int64_t n, int32_t* bad, cudaStream_t st);
void launch_fill_i32(int32_t* p, int64_t n, int32_t v, cudaStream_t st);

}  // namespace wmd
