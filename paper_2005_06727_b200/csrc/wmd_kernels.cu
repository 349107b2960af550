// wmd_kernels.cu — sm_100a kernels of the sparse Sinkhorn-WMD hot path (arXiv 2005.06727).
//
// All arithmetic is FP32 SIMT (no tensor cores in the sparse steps: they are gathers, not
// contractions), except the FP64 fallback. See DESIGN.md §5 for each kernel's roofline.
//
//   (a2, the distance build, is in wmd_build.cu; NEXT-1, the fused kernel, in wmd_fused.cu)
//   sddmm_spmm_iter   a4: one fused SDDMM_SpMM iteration over all documents
//   final_wmd         a5: u/v/WMD final step
//   fallback_fp64     a6: FP64 re-run of documents whose FP32 iterates left the normal range
#include <cfloat>
#include <cmath>
#include <algorithm>
#include <cstdint>

#include "wmd_device.cuh"
#include "wmd_internal.h"

namespace wmd {
namespace {

using dev::ldg_guarded;

constexpr unsigned kFull = 0xffffffffu;

__device__ __forceinline__ float4 ldg4(const float* p) { return __ldg(reinterpret_cast<const float4*>(p)); }
__device__ __forceinline__ float dot4(float4 a, float4 b) {
  return fmaf(a.w, b.w, fmaf(a.z, b.z, fmaf(a.y, b.y, a.x * b.x)));
}
__device__ __forceinline__ void axpy4(float4& acc, float4 x, float s) {
  acc.x = fmaf(x.x, s, acc.x); acc.y = fmaf(x.y, s, acc.y);
  acc.z = fmaf(x.z, s, acc.z); acc.w = fmaf(x.w, s, acc.w);
}
__device__ __forceinline__ bool normal_pos(float x) { return x >= FLT_MIN && x <= FLT_MAX; }

// L2 residency: the K~ / M tables (<= V*ld*4 bytes, 51 MB at Scaling) are gathered every
// iteration and must stay in the 126 MB L2 while ~1 GB of c and u streams past them. Table
// gathers carry an evict_last policy; the streamed arrays use .cs (evict-first) loads/stores.
__device__ __forceinline__ uint64_t l2_evict_last_policy() {
  uint64_t pol;
  asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ float4 ldg4_keep(const float4* p, uint64_t pol) {
#ifdef WMD_NO_L2_HINTS
  return __ldg(p);
#else
  float4 v;
  asm("ld.global.nc.L2::cache_hint.v4.f32 {%0, %1, %2, %3}, [%4], %5;"
      : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
      : "l"(p), "l"(pol));
  return v;
#endif
}
#ifdef WMD_STREAM_HINTS
#define WMD_LDS(p) __ldcs(p)
#define WMD_STS(p, v) __stcs(p, v)
#else
#define WMD_LDS(p) __ldg(p)
#define WMD_STS(p, v) (*(p) = (v))
#endif

// FP32 range certificate (R21). A K~ entry below FLT_MIN = 2^-126 is subnormal or
// flushed to 0 and carries an absolute error of up to 2^-149 (a normal entry only its relative
// rounding). A document keeps its FP32 result only if, in every sum of every iteration,
//     s_e   = sum_i K~_ki u_i :   u_i * v_r * 2^-149 <= 2^-16 * s_e   for each underflowed K~_ki
//     acc_i = sum_e K~_ki v~_e:   (sum_{e: K~_ki underflowed} v~_e) * 2^-149 <= 2^-16 * acc_i
// otherwise it is flagged for the FP64 re-run. The test is gauge-invariant (u -> a u scales s by
// a and v~, acc by 1/a) and only fires when underflowed entries could matter: the FP32 error of
// a certified sum stays ~1e-6 relative (measured: DESIGN.md §4).
constexpr float kUnderScale = 0x1p-133f;  // 2^-149 / 2^-16

// FP64 fallback scratch per block: K (documents too long for shared memory) + v + final terms.
__host__ __device__ constexpr int64_t fallback_block_doubles(int64_t max_doc_nnz) {
  return max_doc_nnz * (WMD_MAX_VR_DEV + 1) + 2 * max_doc_nnz;
}

// ============================================================================================
// a4 + a5. sinkhorn_pass<G, U, FINAL>: one pass over all target documents.
//
// FINAL = false (a4, one launch per iteration; the paper's fused SDDMM_SpMM):
//   per nonzero e = (k, c_kj):  s_e = sum_i K~_ki u_ij           (SDDMM at c's support, :146)
//                                v~_e = c_kj / s_e                (c .* 1./(K^T u))
//                                acc_i += K~_ki v~_e              (SpMM K v; v never stored)
//   then u_ij = r_i / acc_i (= 1/x, x = diag(1/r) K v; update_x_u) and the exact
//   per-document power-of-two gauge 2^-floor((e_max+e_min)/2) (R21).
// FINAL = true (a5): s_e, v~_e as above, q_e = sum_i K~_ki M_ik u_i and
//   WMD_j = sum_e v~_e q_e (= sum_i u_i ((K.*M) v)_i, summed over e instead of i).
//
// Mapping: one warp per document (warp-persistent, next document prefetched while the current
// one's K~ rows are in flight); G lanes per K~ row (float4 each, ld <= 4G); NG = 32/G groups
// per warp, each taking U consecutive nonzeros per step (STEP = NG*U <= 32 gathers in flight
// per warp). The U partial dot products of a group are combined by a transpose-reduce
// (U-1 shuffles for U = G instead of U log2 G), so each lane ends with the full s of ONE
// nonzero: one division per lane per step, then U broadcasts of v~ for the axpy.
// Documents are owned by one warp: no atomics in the arithmetic, deterministic.
// Bound: K~ row gathers from L2 (4*ld bytes per nonzero) + the HBM stream of c and u.
// ============================================================================================
template <int X>
struct Log2 { static constexpr int value = 1 + Log2<X / 2>::value; };
template <>
struct Log2<1> { static constexpr int value = 0; };

// p[0..U) per lane; returns, in lane `sub` of a G-lane group, the group sum of p[sub >> SHIFT]
// where SHIFT = log2(G) - log2(U).
template <int G, int U>
__device__ __forceinline__ float transpose_reduce(float (&p)[U], int sub) {
#pragma unroll
  for (int r = 0, o = G / 2; o >= 1; ++r, o >>= 1) {
    const int n = U >> r;  // values still held (compile-time after unrolling)
    if (n > 1) {
      const bool upper = (sub & o) != 0;
#pragma unroll
      for (int t = 0; t < n / 2; ++t) {
        const float send = upper ? p[t] : p[t + n / 2];
        const float keep = upper ? p[t + n / 2] : p[t];
        p[t] = keep + __shfl_xor_sync(kFull, send, o);
      }
    } else {
      p[0] += __shfl_xor_sync(kFull, p[0], o);
    }
  }
  return p[0];
}

__device__ __forceinline__ uint32_t under_bits(float4 k) {
  return (k.x < FLT_MIN ? 1u : 0u) | (k.y < FLT_MIN ? 2u : 0u) | (k.z < FLT_MIN ? 4u : 0u) |
         (k.w < FLT_MIN ? 8u : 0u);
}

#ifndef PASS_BLOCKS_PER_SM
#define PASS_BLOCKS_PER_SM 3
#endif
template <int G, int U, bool FINAL, bool MAKE_MASK>
__global__ void __launch_bounds__(256, FINAL ? 2 : PASS_BLOCKS_PER_SM) sinkhorn_pass_kernel(
    const int32_t* __restrict__ order, const int32_t* __restrict__ doc_ptr,
    const Entry* __restrict__ ent, int64_t N, const float* __restrict__ Kt,
    const float* __restrict__ Mt, int ld, int v_r, const float* __restrict__ rpad,
    const float* __restrict__ u_in, float* __restrict__ u_out, uint32_t* __restrict__ umask,
    int mask_words, float* __restrict__ dist, uint8_t* __restrict__ flags,
    int32_t* __restrict__ flagged_list, int32_t* __restrict__ flagged_count, ConvParams cv) {
  constexpr int NG = 32 / G;
  constexpr int SHIFT = Log2<G>::value - Log2<U>::value;
  static_assert(U <= G, "at most one nonzero per lane per step");
  const int lane = threadIdx.x & 31, grp = lane / G, sub = lane % G;
  const int qm = sub >> SHIFT;                       // this lane's nonzero slot within a step
  const bool owner = (sub & ((1 << SHIFT) - 1)) == 0;
  const int gbase = grp * G;
  const int64_t warp = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int64_t nwarps = (int64_t)gridDim.x * (blockDim.x >> 5);
  const bool act = sub * 4 < ld;
  const float u0 = (float)v_r;
  const int mword = (sub * 4) >> 5, mshift = (sub * 4) & 31;
  const float4 zero = make_float4(0.f, 0.f, 0.f, 0.f);
  const float4 r = act ? ldg4(rpad + sub * 4) : zero;
  const int2* ent2 = reinterpret_cast<const int2*>(ent);
  const uint32_t ld4 = (uint32_t)ld >> 2;           // row stride in float4s
  const float4* kb = reinterpret_cast<const float4*>(Kt) + sub;  // this lane's float4 of a K~ row
  const float4* mb = FINAL ? reinterpret_cast<const float4*>(Mt) + sub : nullptr;  // ... of an M row
  const uint32_t ldx4 = ld4 + 1;                    // Mx row stride in float4s (ld + 4 floats)
  const uint64_t keep = l2_evict_last_policy();

  // Round structure: in each round the warp's NG groups take NG consecutive documents of the
  // length-sorted order, so their step counts match; the next round is prefetched.
  // (ldg_guarded: loads that stay behind their guard)
  auto head = [&](int64_t pos, int64_t& jj, int& bb, int& nn) {
    jj = -1; bb = 0; nn = 0;
    if (pos < N) {
      jj = ldg_guarded(order + pos);
      bb = ldg_guarded(doc_ptr + jj);
      nn = ldg_guarded(doc_ptr + jj + 1) - bb;
    }
  };
  auto body = [&](int64_t jj, int bb, int nn, int2& e0, float4& uu, uint32_t& mb) {
    e0 = make_int2(0, 0); uu = zero; mb = 0u;
    if (jj < 0) return;
    if (qm < nn) e0 = ldg_guarded(ent2 + bb + qm);
    if (u_in == nullptr) {  // x0 = 1/v_r  =>  u0 = v_r on the v_r real rows
      uu = make_float4(r.x > 0.f ? u0 : 0.f, r.y > 0.f ? u0 : 0.f, r.z > 0.f ? u0 : 0.f,
                       r.w > 0.f ? u0 : 0.f);
    } else if (act) {
      uu = WMD_LDS(reinterpret_cast<const float4*>(u_in + jj * ld) + sub);
    }
    if (!MAKE_MASK && act) mb = (WMD_LDS(umask + jj * mask_words + mword) >> mshift) & 0xFu;
  };

  int64_t pos = warp * NG + grp;
  int64_t j;
  int b, n;
  head(pos, j, b, n);
  int2 my;
  float4 u;
  uint32_t mbits;
  body(j, b, n, my, u, mbits);
  for (int64_t rb = warp * NG; rb < N; rb += nwarps * NG, pos += nwarps * NG) {
    int64_t jn;
    int bn, nn_;
    head(pos + nwarps * NG, jn, bn, nn_);
    int2 myn;
    float4 unx;
    uint32_t mbn;
    bool prefetched = false;
    const int steps = __reduce_max_sync(kFull, (n + U - 1) / U);
    float4 acc = zero;
    float smin = FLT_MAX, vmax = 0.f, wsum = 0.f;
    uint32_t ubits = 0u;
    for (int s = 0; s < steps; ++s) {
      const int eb = s * U;
      float4 kr[U], mr[U];
#pragma unroll
      for (int q = 0; q < U; ++q) {
        // Unpredicated gathers: empty slots carry k = 0 (row 0) and lanes past ld read into the
        // next row (the tables are padded); both only meet u = 0 / v~ = 0 below.
        const uint32_t kk = (uint32_t)__shfl_sync(kFull, my.x, gbase + (q << SHIFT));
        kr[q] = ldg4_keep(kb + kk * ld4, keep);
        if (FINAL) mr[q] = ldg4_keep(mb + kk * ldx4, keep);
        if (MAKE_MASK && eb + q < n && act) ubits |= under_bits(kr[q]);
      }
      const bool myvalid = eb + qm < n;
      const float c = __int_as_float(my.y);
      // next step's nonzero (and, once per round, the next round's document) while K~ is in flight
      my = make_int2(0, 0);
      if (eb + U + qm < n) my = ldg_guarded(ent2 + b + eb + U + qm);
      if (!prefetched) {
        prefetched = true;
        body(jn, bn, nn_, myn, unx, mbn);
      }
      float p[U];
#pragma unroll
      for (int q = 0; q < U; ++q) p[q] = dot4(kr[q], u);
      const float sv = transpose_reduce<G, U>(p, sub);
      // empty slots divide 1 by 1 (a zero numerator would take the IEEE division slow path)
      float vt = (myvalid ? c : 1.f) / (myvalid ? sv : 1.f);
      if (myvalid) {
        smin = fminf(smin, sv);
        vmax = fmaxf(vmax, vt);
      } else {
        vt = 0.f;
      }
      if (FINAL) {
        float t[U];
#pragma unroll
        for (int q = 0; q < U; ++q) {  // (K .* M) row times u
          const float4 km = make_float4(kr[q].x * mr[q].x, kr[q].y * mr[q].y,
                                        kr[q].z * mr[q].z, kr[q].w * mr[q].w);
          t[q] = dot4(km, u);
        }
        const float tv = transpose_reduce<G, U>(t, sub);
        if (myvalid && owner) wsum = fmaf(vt, tv, wsum);
      } else {
#pragma unroll
        for (int q = 0; q < U; ++q) axpy4(acc, kr[q], __shfl_sync(kFull, vt, gbase + (q << SHIFT)));
      }
    }
    // ---- per-document epilogue (each G-lane group owns one document)
    if (MAKE_MASK) {  // rows with an underflowed K~ entry in this document (iteration-invariant)
      mbits = ubits;
      if (!FINAL) {
        for (int w = 0; w < mask_words; ++w) {
          uint32_t word = (act && mword == w) ? (ubits << mshift) : 0u;
#pragma unroll
          for (int off = G / 2; off; off >>= 1) word |= __shfl_xor_sync(kFull, word, off);
          if (sub == 0 && j >= 0) umask[j * mask_words + w] = word;
        }
      }
    }
    // FP32 range certificate (see kUnderScale)
    float umu = 0.f;
    if (mbits & 1u) umu = fmaxf(umu, u.x);
    if (mbits & 2u) umu = fmaxf(umu, u.y);
    if (mbits & 4u) umu = fmaxf(umu, u.z);
    if (mbits & 8u) umu = fmaxf(umu, u.w);
#pragma unroll
    for (int off = G / 2; off; off >>= 1) {
      smin = fminf(smin, __shfl_xor_sync(kFull, smin, off));
      vmax = fmaxf(vmax, __shfl_xor_sync(kFull, vmax, off));
      umu = fmaxf(umu, __shfl_xor_sync(kFull, umu, off));
    }
    int bad = ((umu * u0) * kUnderScale > smin || !(vmax <= FLT_MAX)) ? 1 : 0;
    if (FINAL) {
#pragma unroll
      for (int off = G / 2; off; off >>= 1) {
        wsum += __shfl_xor_sync(kFull, wsum, off);
        bad |= __shfl_xor_sync(kFull, bad, off);
      }
      if (sub == 0 && j >= 0) {
        dist[j] = wsum;
        if (bad || !(fabsf(wsum) <= FLT_MAX) || (flags[j] & kFlagFp32Range)) {
          flags[j] |= kFlagFp32Range;
          flagged_list[atomicAdd(flagged_count, 1)] = (int32_t)j;
        }
      }
    } else {
      float4 un;
      // padded rows (r = 0) compute 1/1, not 0/garbage: a zero numerator takes the IEEE slow path
#define WMD_UDIV(c) \
      un.c = (r.c > 0.f ? r.c : 1.f) / (r.c > 0.f ? acc.c : 1.f); if (!(r.c > 0.f)) un.c = 0.f;
      WMD_UDIV(x) WMD_UDIV(y) WMD_UDIV(z) WMD_UDIV(w)
#undef WMD_UDIV
      // "while x changes" (NEXT-3): a converged document keeps its u (x is frozen); otherwise
      // the relative change max_i |x_new/x - 1| = max_i |u/u_new - 1| (gauge invariant)
      const bool frozen = cv.tol >= 0.f && j >= 0 && cv.conv[j];
      float chg = 0.f;
      if (cv.tol >= 0.f) {
#define WMD_CHG(c) if (r.c > 0.f) chg = fmaxf(chg, fabsf(u.c / un.c - 1.f));
        WMD_CHG(x) WMD_CHG(y) WMD_CHG(z) WMD_CHG(w)
#undef WMD_CHG
        if (!(chg <= FLT_MAX)) chg = FLT_MAX;  // NaN: not converged
#pragma unroll
        for (int off = G / 2; off; off >>= 1) chg = fmaxf(chg, __shfl_xor_sync(kFull, chg, off));
      }
      const float vcap = (float)n * vmax * kUnderScale;  // bound on the underflowed terms
      float mx = 0.f, mn = FLT_MAX;
#define WMD_ROW(c, bit)                                                   \
      if (r.c > 0.f) {                                                    \
        bad |= (!normal_pos(un.c) || ((mbits & bit) && vcap > acc.c));    \
        mx = fmaxf(mx, un.c); mn = fminf(mn, un.c);                       \
      }
      WMD_ROW(x, 1u) WMD_ROW(y, 2u) WMD_ROW(z, 4u) WMD_ROW(w, 8u)
#undef WMD_ROW
#pragma unroll
      for (int off = G / 2; off; off >>= 1) {
        mx = fmaxf(mx, __shfl_xor_sync(kFull, mx, off));
        mn = fminf(mn, __shfl_xor_sync(kFull, mn, off));
        bad |= __shfl_xor_sync(kFull, bad, off);
      }
      if (frozen) {
        un = u;
      } else if (!bad) {
        const int g = (ilogbf(mx) + ilogbf(mn)) >> 1;  // floor((e_max + e_min) / 2)
        const float sc = ldexpf(1.0f, -g);             // |g| <= 126 when all u are normal
        un.x *= sc; un.y *= sc; un.z *= sc; un.w *= sc;
      } else if (sub == 0 && j >= 0) {
        flags[j] |= kFlagFp32Range;
      }
      if (!frozen && cv.tol >= 0.f && chg <= cv.tol && sub == 0 && j >= 0) {
        cv.conv[j] = 1;
        cv.iters_doc[j] = cv.it_index + 1;
      }
      if (act && j >= 0) WMD_STS(reinterpret_cast<float4*>(u_out + j * ld) + sub, un);
    }
    j = jn; b = bn; n = nn_; my = myn; u = unx; mbits = mbn;
  }
}

// ============================================================================================
// a6. FP64 fallback: one block per flagged document (grid-stride over the device-side list, so
// the launch needs no host read-back; an empty list costs one tiny launch). K is rebuilt in FP64
// from the FP32 distance table, K_ki = exp(-lambda (M_ik - m_k)) (same exact column rescale, now
// with FP64 range), and the iterations and the final step run in FP64 with the exact
// power-of-two gauge. FP32 M is accurate to ~3e-7 relative, so this recovers oracle parity where
// FP32 *range* failed (measured: DESIGN.md §4). Deterministic: sequential per-thread sums and a
// serial final sum.
// ============================================================================================
// One block per flagged document (grid-stride over the device-side list). K = exp(-lambda
// (M - m)) in FP64 lives in shared memory (row pitch v_r + 1 doubles: the SDDMM reads it with
// threads over rows, the SpMM with threads over columns) when the document fits
// (kFallbackSmem), else in a per-block global scratch with the same layout. The SpMM splits
// the rows over two thread halves; gauge and change test are block reductions.
constexpr int kFallbackSmem = 200 * 1024;  // per block at most; 100 KB lets two blocks share an SM

__global__ void __launch_bounds__(256) fallback_fp64_kernel(
    const float* __restrict__ Mt, int ld,
    const float* __restrict__ rpad, int v_r, double lambda, int iters, float tol,
    int32_t* __restrict__ iters_doc, const int32_t* __restrict__ doc_ptr, const Entry* __restrict__ ent,
    const int32_t* __restrict__ flagged_list, const int32_t* __restrict__ flagged_count,
    double* __restrict__ scratch, int64_t max_doc_nnz, float* __restrict__ dist,
    uint8_t* __restrict__ flags, int32_t* __restrict__ breakdown, int32_t* __restrict__ fb_count,
    int smem_bytes) {
  extern __shared__ double ksm[];
  __shared__ double u[WMD_MAX_VR_DEV], part[2][WMD_MAX_VR_DEV], red[3][8];
  const int n = *flagged_count;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int ci = tid & 127, half = tid >> 7;
  const int ldx = ld + 4, pitch = v_r + 1;
  double* gK = scratch + (int64_t)blockIdx.x * fallback_block_doubles(max_doc_nnz);
  double* vv = gK + max_doc_nnz * (WMD_MAX_VR_DEV + 1);
  double* qv = vv + max_doc_nnz;
  for (int idx = blockIdx.x; idx < n; idx += gridDim.x) {
    const int j = flagged_list[idx];
    const int b = doc_ptr[j], L = doc_ptr[j + 1] - b;
    double* K = (int64_t)L * pitch * 8 <= smem_bytes ? ksm : gK;
    for (int p = tid; p < L * v_r; p += blockDim.x) {  // K = exp(-lambda (M - m)), FP64
      const int e_ = p / v_r, i = p % v_r;
      const int k = ent[b + e_].k;
      // column minimum m_k sits at Mx row position ld
      K[(int64_t)e_ * pitch + i] = exp(-lambda * ((double)Mt[(int64_t)k * ldx + i] - (double)Mt[(int64_t)k * ldx + ld]));
    }
    for (int i = tid; i < v_r; i += blockDim.x) u[i] = (double)v_r;  // x0 = 1/v_r
    __syncthreads();
    int it = 0;
    for (; it < iters; ++it) {
      for (int e_ = tid; e_ < L; e_ += blockDim.x) {  // SDDMM (4 partial sums: pipelined loads)
        const double* Ke = K + (int64_t)e_ * pitch;
        double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
        int i = 0;
        for (; i + 4 <= v_r; i += 4) {
          s0 = fma(Ke[i], u[i], s0); s1 = fma(Ke[i + 1], u[i + 1], s1);
          s2 = fma(Ke[i + 2], u[i + 2], s2); s3 = fma(Ke[i + 3], u[i + 3], s3);
        }
        for (; i < v_r; ++i) s0 = fma(Ke[i], u[i], s0);
        vv[e_] = (double)ent[b + e_].c / ((s0 + s1) + (s2 + s3));
      }
      __syncthreads();
      for (int i0 = 0; i0 < v_r; i0 += 128) {  // SpMM, two row halves
        const int i = i0 + ci;
        if (i < v_r) {
          double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
          int e_ = half;
          for (; e_ + 6 < L; e_ += 8) {
            a0 = fma(K[(int64_t)e_ * pitch + i], vv[e_], a0);
            a1 = fma(K[(int64_t)(e_ + 2) * pitch + i], vv[e_ + 2], a1);
            a2 = fma(K[(int64_t)(e_ + 4) * pitch + i], vv[e_ + 4], a2);
            a3 = fma(K[(int64_t)(e_ + 6) * pitch + i], vv[e_ + 6], a3);
          }
          for (; e_ < L; e_ += 2) a0 = fma(K[(int64_t)e_ * pitch + i], vv[e_], a0);
          part[half][i] = (a0 + a1) + (a2 + a3);
        }
      }
      __syncthreads();
      double mx = 0.0, mn = DBL_MAX, chg = 0.0, un = 0.0;
      if (tid < v_r) {  // v_r <= WMD_MAX_VR <= blockDim
        un = (double)rpad[tid] / (part[0][tid] + part[1][tid]);
        mx = un; mn = un;
        const double c = fabs(u[tid] / un - 1.0);  // "while x changes": |x_new/x - 1|
        chg = c <= DBL_MAX ? c : DBL_MAX;
      }
#pragma unroll
      for (int off = 16; off; off >>= 1) {
        mx = fmax(mx, __shfl_xor_sync(kFull, mx, off));
        mn = fmin(mn, __shfl_xor_sync(kFull, mn, off));
        chg = fmax(chg, __shfl_xor_sync(kFull, chg, off));
      }
      if (lane == 0) { red[0][warp] = mx; red[1][warp] = mn; red[2][warp] = chg; }
      __syncthreads();
      mx = red[0][0]; mn = red[1][0]; chg = red[2][0];
#pragma unroll
      for (int w = 1; w < 8; ++w) { mx = fmax(mx, red[0][w]); mn = fmin(mn, red[1][w]); chg = fmax(chg, red[2][w]); }
      const int gexp = (mx > 0.0 && mn > 0.0 && mx <= DBL_MAX) ? ((ilogb(mx) + ilogb(mn)) >> 1) : 0;
      if (tid < v_r) u[tid] = ldexp(un, -gexp);
      __syncthreads();
      if (tol >= 0.f && chg <= (double)tol) { ++it; break; }
    }
    for (int e_ = tid; e_ < L; e_ += blockDim.x) {  // final step
      const int k = ent[b + e_].k;
      double s = 0.0, t = 0.0;
      for (int i = 0; i < v_r; ++i) {
        const double kk = K[(int64_t)e_ * pitch + i];
        s += kk * u[i];
        t += kk * (double)Mt[(int64_t)k * ldx + i] * u[i];
      }
      qv[e_] = ((double)ent[b + e_].c / s) * t;
    }
    __syncthreads();
    if (tid == 0) {
      double w = 0.0;
      for (int e_ = 0; e_ < L; ++e_) w += qv[e_];
      dist[j] = (float)w;
      flags[j] |= kFlagFp64;
      if (iters_doc) iters_doc[j] = it;
      if (!isfinite(w)) atomicExch(breakdown, 1);
      atomicAdd(fb_count, 1);
    }
    __syncthreads();
  }
}

__global__ void check_finite_kernel(const float* __restrict__ x, int64_t n, int32_t* bad) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    if (!isfinite(x[i])) { atomicExch(bad, 1); return; }
}

int lanes_per_row(int ld) {
  int g = 2;
  while (g * 4 < ld) g *= 2;
  return g;
}

}  // namespace

// ------------------------------------------------------------------------------ launchers
// U = nonzeros per group per step: U = G up to 8 so that the transpose-reduce leaves exactly one
// nonzero per lane (fewer lanes idle); (32/G) documents per warp.
#define WMD_DISPATCH_G(ld, MACRO) \
  switch (lanes_per_row(ld)) {    \
    case 2: MACRO(2, 2); break;   \
    case 4: MACRO(4, 4); break;   \
    case 8: MACRO(8, 8); break;   \
    case 16: MACRO(16, 8); break; \
    default: MACRO(32, 8); break; \
  }

// Persistent grid for the pass kernels: `per_sm` resident 256-thread blocks per SM, or fewer if
// the documents (groups_per_warp per warp) do not need them.
unsigned pass_grid(int64_t N, int ld, int per_sm) {
  const int sms = device_sms();
  const int ng = 32 / lanes_per_row(ld);
  const int64_t warps = (N + ng - 1) / ng;
  const int64_t need = (warps + 7) / 8;
  return (unsigned)std::max<int64_t>(1, std::min<int64_t>(need, (int64_t)sms * per_sm));
}

int mask_words_for(int ld) { return (ld + 31) / 32; }

void launch_sddmm_spmm_iter(const int32_t* order, const int32_t* doc_ptr, const Entry* ent, int64_t N,
                            const float* Kt, int ld, int v_r, const float* rpad, const float* u_in,
                            float* u_out, uint32_t* umask, uint8_t* flags, ConvParams cv,
                            cudaStream_t st) {
  const unsigned grid = pass_grid(N, ld, PASS_BLOCKS_PER_SM);
  const int mw = mask_words_for(ld);
  // the first iteration records the underflow row masks, later ones read them
  if (u_in == nullptr) {
#define L_(G, U) sinkhorn_pass_kernel<G, U, false, true><<<grid, 256, 0, st>>>(order, doc_ptr, ent, N, Kt, nullptr, ld, v_r, rpad, u_in, u_out, umask, mw, nullptr, flags, nullptr, nullptr, cv)
    WMD_DISPATCH_G(ld, L_)
#undef L_
  } else {
#define L_(G, U) sinkhorn_pass_kernel<G, U, false, false><<<grid, 256, 0, st>>>(order, doc_ptr, ent, N, Kt, nullptr, ld, v_r, rpad, u_in, u_out, umask, mw, nullptr, flags, nullptr, nullptr, cv)
    WMD_DISPATCH_G(ld, L_)
#undef L_
  }
}

void launch_final_wmd(const int32_t* order, const int32_t* doc_ptr, const Entry* ent, int64_t N,
                      const float* Kt, const float* Mt, int ld, int v_r, const float* rpad,
                      const float* u_in, const uint32_t* umask, float* dist, uint8_t* flags,
                      int32_t* flagged_list, int32_t* flagged_count, cudaStream_t st) {
  const unsigned grid = pass_grid(N, ld, 2);
  const int mw = mask_words_for(ld);
  uint32_t* um = const_cast<uint32_t*>(umask);
  if (u_in == nullptr) {  // iters == 0: no iteration recorded the masks
#define L_(G, U) sinkhorn_pass_kernel<G, U, true, true><<<grid, 256, 0, st>>>(order, doc_ptr, ent, N, Kt, Mt, ld, v_r, rpad, u_in, nullptr, um, mw, dist, flags, flagged_list, flagged_count, ConvParams{-1.f, nullptr, nullptr, 0})
    WMD_DISPATCH_G(ld, L_)
#undef L_
  } else {
#define L_(G, U) sinkhorn_pass_kernel<G, U, true, false><<<grid, 256, 0, st>>>(order, doc_ptr, ent, N, Kt, Mt, ld, v_r, rpad, u_in, nullptr, um, mw, dist, flags, flagged_list, flagged_count, ConvParams{-1.f, nullptr, nullptr, 0})
    WMD_DISPATCH_G(ld, L_)
#undef L_
  }
}

size_t fallback_scratch_bytes(int64_t max_doc_nnz) {
  return sizeof(double) * (size_t)kFallbackBlocks * (size_t)fallback_block_doubles(max_doc_nnz);
}

void launch_fallback_fp64(const float* Mt, int ld, const float* rpad, int v_r,
                          double lambda, int iters, float tol, int32_t* iters_doc,
                          const int32_t* doc_ptr, const Entry* ent,
                          const int32_t* flagged_list, const int32_t* flagged_count,
                          double* scratch, int64_t max_doc_nnz, float* dist, uint8_t* flags,
                          int32_t* breakdown, int32_t* fallback_count, cudaStream_t st) {
  // shared memory for the largest document's K (two blocks per SM when it fits in 100 KB)
  const int64_t need = max_doc_nnz * (v_r + 1) * 8;
  const int smem = (int)std::min<int64_t>(need, kFallbackSmem);
  const int blocks = smem <= kFallbackSmem / 2 ? kFallbackBlocks : kFallbackBlocks / 2;
  static PerDevice attr;
  attr.get([] { return (int)cudaFuncSetAttribute(fallback_fp64_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kFallbackSmem); });
  fallback_fp64_kernel<<<blocks, 256, smem, st>>>(Mt, ld, rpad, v_r, lambda, iters, tol, iters_doc, doc_ptr, ent,
                                                  flagged_list, flagged_count, scratch, max_doc_nnz, dist, flags,
                                                  breakdown, fallback_count, smem);
}

__global__ void fill_i32_kernel(int32_t* p, int64_t n, int32_t v) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    p[i] = v;
}

void launch_fill_i32(int32_t* p, int64_t n, int32_t v, cudaStream_t st) {
  fill_i32_kernel<<<(unsigned)std::min<int64_t>(1184, (n + 255) / 256 + 1), 256, 0, st>>>(p, n, v);
}

void launch_check_finite(const float* x, int64_t n, int32_t* bad, cudaStream_t st) {
  check_finite_kernel<<<device_sms() * 4, 256, 0, st>>>(x, n, bad);
}

}  // namespace wmd
