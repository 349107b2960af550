// wmd_kernels.cu — sm_100a kernels of the sparse Sinkhorn-WMD hot path (arXiv 2005.06727).
//
// All arithmetic is FP32 SIMT (no tensor cores in the sparse steps: they are gathers, not
// contractions), except the FP64 fallback. See DESIGN.md §5 for each kernel's roofline.
//
//   build_ktilde      a2: M and the column-rescaled K~ = exp(-lambda (M - min_i M)) (vocab-major tables)
//   sddmm_spmm_iter   a4: one fused SDDMM_SpMM iteration over all documents
//   final_wmd         a5: u/v/WMD final step
//   fallback_fp64     a6: FP64 re-run of documents whose FP32 iterates left the normal range
#include <cfloat>
#include <cmath>
#include <algorithm>
#include <cstdint>

#include "wmd_internal.h"

namespace wmd {
namespace {

constexpr unsigned kFull = 0xffffffffu;

__device__ __forceinline__ float4 ldg4(const float* p) { return __ldg(reinterpret_cast<const float4*>(p)); }
__device__ __forceinline__ float dot4(float4 a, float4 b) {
  return fmaf(a.w, b.w, fmaf(a.z, b.z, fmaf(a.y, b.y, a.x * b.x)));
}
__device__ __forceinline__ void axpy4(float4& acc, float4 x, float s) {
  acc.x = fmaf(x.x, s, acc.x); acc.y = fmaf(x.y, s, acc.y);
  acc.z = fmaf(x.z, s, acc.z); acc.w = fmaf(x.w, s, acc.w);
}
__device__ __forceinline__ float4 shfl_xor4(float4 v, int off) {
  v.x = __shfl_xor_sync(kFull, v.x, off); v.y = __shfl_xor_sync(kFull, v.y, off);
  v.z = __shfl_xor_sync(kFull, v.z, off); v.w = __shfl_xor_sync(kFull, v.w, off);
  return v;
}
__device__ __forceinline__ bool normal_pos(float x) { return x >= FLT_MIN && x <= FLT_MAX; }
__device__ __forceinline__ float max4(float4 v) { return fmaxf(fmaxf(v.x, v.y), fmaxf(v.z, v.w)); }

// FP32 range certificate (R21). A K~ entry below FLT_MIN = 2^-126 is subnormal or
// flushed to 0 and carries an absolute error of up to 2^-149 (a normal entry only its relative
// rounding). A document keeps its FP32 result only if, in every sum of every iteration,
//     s_e   = sum_i K~_ki u_i :   u_i * v_r * 2^-149 <= 2^-16 * s_e   for each underflowed K~_ki
//     acc_i = sum_e K~_ki v~_e:   (sum_{e: K~_ki underflowed} v~_e) * 2^-149 <= 2^-16 * acc_i
// otherwise it is flagged for the FP64 re-run. The test is gauge-invariant (u -> a u scales s by
// a and v~, acc by 1/a) and only fires when underflowed entries could matter: the FP32 error of
// a certified sum stays ~1e-6 relative (measured: DESIGN.md §4).
constexpr float kUnderScale = 0x1p-133f;  // 2^-149 / 2^-16

// ============================================================================================
// a2. build_ktilde: per vocabulary word k and query row i
//        M_ik  = sqrt(sum_t (E[sel_i,t] - E[k,t])^2)        (direct difference so
//                                                             M_{i,sel_i} == 0 exactly)
//        m_k   = min_i M_ik
//        K~_ki = expf(-lambda (M_ik - m_k)),  and M itself                (vocab-major, ld floats)
// Block: 256 threads, 64 vocabulary words x all query rows (32-row tiles), d staged through
// shared memory in chunks of 32. Thread micro-tile: 2 rows x 4 words, float4 smem reads.
// Bound: FP32 issue (2 flops per (i,k,t) triple, PAPER.md:260 counts 3) vs reading E once.
// ============================================================================================
constexpr int BK_TW = 64, BK_TI = 32, BK_DC = 32, BK_STR = BK_DC + 4, BK_LDM = 129;

__global__ void __launch_bounds__(256) build_ktilde_kernel(const float* __restrict__ E, int64_t V,
                                                           int d, const int32_t* __restrict__ sel,
                                                           int v_r, int ld, float lambda,
                                                           float* __restrict__ Kt,
                                                           float* __restrict__ Mt,
                                                           float* __restrict__ colmin) {
  extern __shared__ __align__(16) float smem[];
  float* Qs = smem;                          // [BK_TI][BK_STR]
  float* Es = Qs + BK_TI * BK_STR;           // [BK_TW][BK_STR]
  float* Ms = Es + BK_TW * BK_STR;           // [BK_TW][BK_LDM]  (word-major, row i)
  const int tid = threadIdx.x;
  const int tw = tid & 15, ti = tid >> 4;
  const int64_t k0 = (int64_t)blockIdx.x * BK_TW;

  for (int it0 = 0; it0 < v_r; it0 += BK_TI) {
    float acc[2][4];
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
      for (int s = 0; s < 4; ++s) acc[a][s] = 0.f;
    for (int d0 = 0; d0 < d; d0 += BK_DC) {
      for (int idx = tid; idx < BK_TI * BK_DC; idx += 256) {
        const int r = idx / BK_DC, c = idx % BK_DC;
        float x = 0.f;
        if (it0 + r < v_r && d0 + c < d) x = __ldg(E + (int64_t)sel[it0 + r] * d + d0 + c);
        Qs[r * BK_STR + c] = x;
      }
      for (int idx = tid; idx < BK_TW * BK_DC; idx += 256) {
        const int w = idx / BK_DC, c = idx % BK_DC;
        float x = 0.f;
        if (k0 + w < V && d0 + c < d) x = __ldg(E + (k0 + w) * d + d0 + c);
        Es[w * BK_STR + c] = x;
      }
      __syncthreads();
      const int tmax = min(BK_DC, d - d0);   // padded columns are 0-0 = 0: harmless, skip anyway
#pragma unroll 2
      for (int t4 = 0; t4 < BK_DC; t4 += 4) {
        if (t4 >= tmax) break;
        const float4 q0 = *reinterpret_cast<const float4*>(Qs + ti * BK_STR + t4);
        const float4 q1 = *reinterpret_cast<const float4*>(Qs + (ti + 16) * BK_STR + t4);
#pragma unroll
        for (int s = 0; s < 4; ++s) {
          const float4 e = *reinterpret_cast<const float4*>(Es + (tw + 16 * s) * BK_STR + t4);
          float df;
          df = q0.x - e.x; acc[0][s] = fmaf(df, df, acc[0][s]);
          df = q0.y - e.y; acc[0][s] = fmaf(df, df, acc[0][s]);
          df = q0.z - e.z; acc[0][s] = fmaf(df, df, acc[0][s]);
          df = q0.w - e.w; acc[0][s] = fmaf(df, df, acc[0][s]);
          df = q1.x - e.x; acc[1][s] = fmaf(df, df, acc[1][s]);
          df = q1.y - e.y; acc[1][s] = fmaf(df, df, acc[1][s]);
          df = q1.z - e.z; acc[1][s] = fmaf(df, df, acc[1][s]);
          df = q1.w - e.w; acc[1][s] = fmaf(df, df, acc[1][s]);
        }
      }
      __syncthreads();
    }
#pragma unroll
    for (int a = 0; a < 2; ++a) {
      const int i = it0 + ti + 16 * a;
      if (i < v_r) {
#pragma unroll
        for (int s = 0; s < 4; ++s) Ms[(tw + 16 * s) * BK_LDM + i] = sqrtf(acc[a][s]);
      }
    }
  }
  __syncthreads();

  // Epilogue: one warp per word; lanes over query rows (coalesced row writes).
  const int warp = tid >> 5, lane = tid & 31;
  for (int w = warp; w < BK_TW; w += 8) {
    const int64_t k = k0 + w;
    if (k >= V) break;
    const float* mrow = Ms + w * BK_LDM;
    float mn = FLT_MAX;
    for (int i = lane; i < v_r; i += 32) mn = fminf(mn, mrow[i]);
#pragma unroll
    for (int off = 16; off; off >>= 1) mn = fminf(mn, __shfl_xor_sync(kFull, mn, off));
    for (int i = lane; i < ld; i += 32) {
      float kt = 0.f, m = 0.f;
      if (i < v_r) {
        m = mrow[i];
        kt = expf(-lambda * (m - mn));
      }
      Kt[k * ld + i] = kt;
      Mt[k * ld + i] = m;
    }
    if (lane == 0) colmin[k] = mn;
  }
}

// ============================================================================================
// a4. sddmm_spmm_iter: one warp per target document j; G lanes per K~ row (float4 each), so a
// warp step handles NG = 32/G nonzeros. Per nonzero e = (k, c_kj):
//     s_e   = sum_i K~_ki u_ij              (SDDMM: K^T u only at c's support)
//     v~_e  = c_kj / s_e                     (c .* 1./(K^T u))
//     acc_i += K~_ki v~_e                    (SpMM: K v, v never stored)
// then u_ij = r_i / acc_i  (= 1/x with x = diag(1/r) K v; update_x_u) and an
// exact per-document power-of-two gauge 2^-round((e_max+e_min)/2) (R21).
// Documents are owned by one warp: no atomics, deterministic.
// Bound: L2->SM gather of K~ rows (4*ld bytes per nonzero) + HBM stream of c and u.
// ============================================================================================
template <int G, int U>
__global__ void __launch_bounds__(256, 3) sddmm_spmm_iter_kernel(
    const int32_t* __restrict__ doc_ptr, const Entry* __restrict__ ent, int64_t N,
    const float* __restrict__ Kt, int ld, float u0, const float* __restrict__ rpad,
    const float* __restrict__ u_in, float* __restrict__ u_out, uint8_t* __restrict__ flags) {
  constexpr int NG = 32 / G, STEP = NG * U;
  static_assert(STEP <= 32, "one step covers at most one 32-entry chunk");
  const int lane = threadIdx.x & 31, grp = lane / G, sub = lane % G;
  const int64_t nwarps = (int64_t)gridDim.x * (blockDim.x >> 5);
  const bool act = sub * 4 < ld;
  const float4 zero = make_float4(0.f, 0.f, 0.f, 0.f);
  const float4 r = act ? ldg4(rpad + sub * 4) : zero;
  auto load_u = [&](int64_t jj) -> float4 {
    if (u_in == nullptr) {  // x0 = 1/v_r  =>  u0 = v_r on the v_r real rows
      return make_float4(r.x > 0.f ? u0 : 0.f, r.y > 0.f ? u0 : 0.f, r.z > 0.f ? u0 : 0.f,
                         r.w > 0.f ? u0 : 0.f);
    }
    return act ? ldg4(u_in + jj * ld + sub * 4) : zero;
  };
  // Warp-persistent over documents j = warp, warp + nwarps, ...; the next document's pointers,
  // first 32 entries and u are prefetched while the current document's K~ rows are in flight.
  int64_t j = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  int b = 0, e = 0;
  int2 my = make_int2(0, 0);
  float4 u = zero;
  if (j < N) {
    b = __ldg(doc_ptr + j); e = __ldg(doc_ptr + j + 1);
    if (lane < e - b) my = __ldg(reinterpret_cast<const int2*>(ent) + b + lane);
    u = load_u(j);
  }
  for (; j < N; j += nwarps) {
    const int64_t jn = j + nwarps;
    int bn = 0, en = 0;
    if (jn < N) { bn = __ldg(doc_ptr + jn); en = __ldg(doc_ptr + jn + 1); }
    int2 myn = make_int2(0, 0);
    float4 unx = zero;
    bool prefetched = false;
    const float4 uscaled = make_float4(u.x * u0 * kUnderScale, u.y * u0 * kUnderScale,
                                       u.z * u0 * kUnderScale, u.w * u0 * kUnderScale);
    float4 acc = zero, under = zero;
    bool bad = false;
    for (int base = b; base < e; base += 32) {
      const int cnt = min(32, e - base);
      if (base != b) {
        my = make_int2(0, 0);
        if (lane < cnt) my = __ldg(reinterpret_cast<const int2*>(ent) + base + lane);
      }
      for (int s0 = 0; s0 < cnt; s0 += STEP) {
        float4 kr[U];
        float cv[U];
#pragma unroll
        for (int q = 0; q < U; ++q) {
          const int idx = s0 + q * NG + grp;
          const int k = __shfl_sync(kFull, my.x, idx & 31);
          const float c = __int_as_float(__shfl_sync(kFull, my.y, idx & 31));
          const bool valid = idx < cnt;
          cv[q] = valid ? c : 0.f;
          kr[q] = (valid && act) ? ldg4(Kt + (int64_t)k * ld + sub * 4) : zero;
        }
        if (!prefetched) {  // overlap the next document's metadata with these gathers
          prefetched = true;
          if (jn < N) {
            if (lane < en - bn) myn = __ldg(reinterpret_cast<const int2*>(ent) + bn + lane);
            unx = load_u(jn);
          }
        }
#pragma unroll
        for (int q = 0; q < U; ++q) {
          float s = dot4(kr[q], u);
#pragma unroll
          for (int off = G / 2; off; off >>= 1) s += __shfl_xor_sync(kFull, s, off);
          if (cv[q] != 0.f) {
            const float vt = cv[q] / s;
            // certificate: underflowed K~ entries must not matter (see kUnderScale)
            bad |= (kr[q].x < FLT_MIN && uscaled.x > s) | (kr[q].y < FLT_MIN && uscaled.y > s) |
                   (kr[q].z < FLT_MIN && uscaled.z > s) | (kr[q].w < FLT_MIN && uscaled.w > s);
            under.x += kr[q].x < FLT_MIN ? vt : 0.f; under.y += kr[q].y < FLT_MIN ? vt : 0.f;
            under.z += kr[q].z < FLT_MIN ? vt : 0.f; under.w += kr[q].w < FLT_MIN ? vt : 0.f;
            axpy4(acc, kr[q], vt);
          }
        }
      }
    }
#pragma unroll
    for (int off = G; off < 32; off <<= 1) {
      const float4 o = shfl_xor4(acc, off);
      acc.x += o.x; acc.y += o.y; acc.z += o.z; acc.w += o.w;
      const float4 p = shfl_xor4(under, off);
      under.x += p.x; under.y += p.y; under.z += p.z; under.w += p.w;
    }
    float4 un;
    un.x = r.x > 0.f ? r.x / acc.x : 0.f; un.y = r.y > 0.f ? r.y / acc.y : 0.f;
    un.z = r.z > 0.f ? r.z / acc.z : 0.f; un.w = r.w > 0.f ? r.w / acc.w : 0.f;
    // range certificate + gauge over the real rows
    float mx = 0.f, mn = FLT_MAX;
#define WMD_ROW(c)                                               \
    if (r.c > 0.f) {                                             \
      bad |= !normal_pos(un.c) || under.c * kUnderScale > acc.c; \
      mx = fmaxf(mx, un.c); mn = fminf(mn, un.c);                \
    }
    WMD_ROW(x) WMD_ROW(y) WMD_ROW(z) WMD_ROW(w)
#undef WMD_ROW
    bad = __any_sync(kFull, bad);
#pragma unroll
    for (int off = G / 2; off; off >>= 1) {
      mx = fmaxf(mx, __shfl_xor_sync(kFull, mx, off));
      mn = fminf(mn, __shfl_xor_sync(kFull, mn, off));
    }
    if (!bad) {
      const int g = (ilogbf(mx) + ilogbf(mn)) >> 1;  // floor((e_max + e_min) / 2)
      un.x = ldexpf(un.x, -g); un.y = ldexpf(un.y, -g); un.z = ldexpf(un.z, -g); un.w = ldexpf(un.w, -g);
    } else if (lane == 0) {
      flags[j] |= kFlagFp32Range;
    }
    if (grp == 0 && act) *reinterpret_cast<float4*>(u_out + j * ld + sub * 4) = un;
    b = bn; e = en; my = myn; u = unx;
  }
}

// ============================================================================================
// a5. final_wmd: u from the last iteration; per nonzero
//     s_e = sum_i K~_ki u_i,  v~_e = c_kj / s_e,  q_e = sum_i K~_ki M_ik u_i,  WMD_j = sum_e v~_e q_e
// (= sum_i u_i ((K.*M) v)_i; summed over e instead of i). Non-finite results and
// documents flagged by the iterations go to the FP64 fallback list.
// ============================================================================================
template <int G, int U>
__global__ void __launch_bounds__(256) final_wmd_kernel(
    const int32_t* __restrict__ doc_ptr, const Entry* __restrict__ ent, int64_t N,
    const float* __restrict__ Kt, const float* __restrict__ Mt, int ld, float u0,
    const float* __restrict__ rpad, const float* __restrict__ u_in, float* __restrict__ dist,
    uint8_t* __restrict__ flags, int32_t* __restrict__ flagged_list,
    int32_t* __restrict__ flagged_count) {
  constexpr int NG = 32 / G;
  const int lane = threadIdx.x & 31, grp = lane / G, sub = lane % G;
  const int64_t j = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (j >= N) return;
  const bool act = sub * 4 < ld;
  const float4 zero = make_float4(0.f, 0.f, 0.f, 0.f);
  float4 u;
  if (u_in == nullptr) {
    const float4 r = act ? ldg4(rpad + sub * 4) : zero;
    u.x = r.x > 0.f ? u0 : 0.f; u.y = r.y > 0.f ? u0 : 0.f;
    u.z = r.z > 0.f ? u0 : 0.f; u.w = r.w > 0.f ? u0 : 0.f;
  } else {
    u = act ? ldg4(u_in + j * ld + sub * 4) : zero;
  }
  const float4 uscaled = make_float4(u.x * u0 * kUnderScale, u.y * u0 * kUnderScale,
                                     u.z * u0 * kUnderScale, u.w * u0 * kUnderScale);
  const int b = doc_ptr[j], e = doc_ptr[j + 1];
  float wsum = 0.f;
  bool bad = false;
  for (int base = b; base < e; base += 32) {
    const int cnt = min(32, e - base);
    int2 my = make_int2(0, 0);
    if (lane < cnt) my = __ldg(reinterpret_cast<const int2*>(ent) + base + lane);
    for (int s0 = 0; s0 < cnt; s0 += NG * U) {
      float4 kr[U], km[U];
      float cv[U];
#pragma unroll
      for (int q = 0; q < U; ++q) {
        const int idx = s0 + q * NG + grp;
        const int k = __shfl_sync(kFull, my.x, idx & 31);
        const float c = __int_as_float(__shfl_sync(kFull, my.y, idx & 31));
        const bool valid = idx < cnt;
        cv[q] = valid ? c : 0.f;
        kr[q] = (valid && act) ? ldg4(Kt + (int64_t)k * ld + sub * 4) : zero;
        km[q] = (valid && act) ? ldg4(Mt + (int64_t)k * ld + sub * 4) : zero;
      }
#pragma unroll
      for (int q = 0; q < U; ++q) {
        const float4 kmq = make_float4(kr[q].x * km[q].x, kr[q].y * km[q].y, kr[q].z * km[q].z,
                                       kr[q].w * km[q].w);  // (K .* M)
        float s = dot4(kr[q], u), t = dot4(kmq, u);
#pragma unroll
        for (int off = G / 2; off; off >>= 1) {
          s += __shfl_xor_sync(kFull, s, off);
          t += __shfl_xor_sync(kFull, t, off);
        }
        if (cv[q] != 0.f) {
          const float vt = cv[q] / s;
          bad |= !(fabsf(vt) <= FLT_MAX);
          bad |= (kr[q].x < FLT_MIN && uscaled.x > s) | (kr[q].y < FLT_MIN && uscaled.y > s) |
                 (kr[q].z < FLT_MIN && uscaled.z > s) | (kr[q].w < FLT_MIN && uscaled.w > s);
          wsum = fmaf(vt, t, wsum);
        }
      }
    }
  }
  // sum the NG per-group partials (each replicated across its G lanes)
#pragma unroll
  for (int off = G; off < 32; off <<= 1) wsum += __shfl_xor_sync(kFull, wsum, off);
  bad = __any_sync(kFull, bad);
  if (lane == 0) {
    dist[j] = wsum;
    const bool need = bad || !(fabsf(wsum) <= FLT_MAX) || (flags[j] & kFlagFp32Range);
    if (need) {
      flags[j] |= kFlagFp32Range;
      const int32_t slot = atomicAdd(flagged_count, 1);
      flagged_list[slot] = (int32_t)j;
    }
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
__global__ void __launch_bounds__(256) fallback_fp64_kernel(
    const float* __restrict__ Mt, const float* __restrict__ colmin, int ld,
    const float* __restrict__ rpad, int v_r, double lambda, int iters,
    const int32_t* __restrict__ doc_ptr, const Entry* __restrict__ ent,
    const int32_t* __restrict__ flagged_list, const int32_t* __restrict__ flagged_count,
    double* __restrict__ scratch, int64_t max_doc_nnz, float* __restrict__ dist,
    uint8_t* __restrict__ flags, int32_t* __restrict__ breakdown, int32_t* __restrict__ fb_count) {
  __shared__ double u[WMD_MAX_VR_DEV], un[WMD_MAX_VR_DEV];
  __shared__ int gexp;
  const int n = *flagged_count;
  double* Kb = scratch + (int64_t)blockIdx.x * (max_doc_nnz * WMD_MAX_VR_DEV + 2 * max_doc_nnz);
  double* vv = Kb + max_doc_nnz * WMD_MAX_VR_DEV;
  double* qv = vv + max_doc_nnz;
  for (int idx = blockIdx.x; idx < n; idx += gridDim.x) {
    const int j = flagged_list[idx];
    const int b = doc_ptr[j], L = doc_ptr[j + 1] - b;
    for (int p = threadIdx.x; p < L * v_r; p += blockDim.x) {
      const int e_ = p / v_r, i = p % v_r;
      const int k = ent[b + e_].k;
      Kb[p] = exp(-lambda * ((double)Mt[(int64_t)k * ld + i] - (double)colmin[k]));
    }
    for (int i = threadIdx.x; i < v_r; i += blockDim.x) u[i] = (double)v_r;  // x0 = 1/v_r
    __syncthreads();
    for (int it = 0; it < iters; ++it) {
      for (int e_ = threadIdx.x; e_ < L; e_ += blockDim.x) {
        double s = 0.0;
        for (int i = 0; i < v_r; ++i) s += Kb[(int64_t)e_ * v_r + i] * u[i];
        vv[e_] = (double)ent[b + e_].c / s;
      }
      __syncthreads();
      for (int i = threadIdx.x; i < v_r; i += blockDim.x) {
        double a = 0.0;
        for (int e_ = 0; e_ < L; ++e_) a += Kb[(int64_t)e_ * v_r + i] * vv[e_];
        un[i] = (double)rpad[i] / a;
      }
      __syncthreads();
      if (threadIdx.x == 0) {
        double mx = 0.0, mn = DBL_MAX;
        for (int i = 0; i < v_r; ++i) { mx = fmax(mx, un[i]); mn = fmin(mn, un[i]); }
        gexp = (mx > 0.0 && mn > 0.0 && mx <= DBL_MAX) ? ((ilogb(mx) + ilogb(mn)) >> 1) : 0;
      }
      __syncthreads();
      for (int i = threadIdx.x; i < v_r; i += blockDim.x) u[i] = ldexp(un[i], -gexp);
      __syncthreads();
    }
    for (int e_ = threadIdx.x; e_ < L; e_ += blockDim.x) {
      const int k = ent[b + e_].k;
      double s = 0.0, t = 0.0;
      for (int i = 0; i < v_r; ++i) {
        const double kk = Kb[(int64_t)e_ * v_r + i];
        s += kk * u[i];
        t += kk * (double)Mt[(int64_t)k * ld + i] * u[i];
      }
      qv[e_] = ((double)ent[b + e_].c / s) * t;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      double w = 0.0;
      for (int e_ = 0; e_ < L; ++e_) w += qv[e_];
      dist[j] = (float)w;
      flags[j] |= kFlagFp64;
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
void launch_build_ktilde(const float* E, int64_t V, int d, const int32_t* sel, int v_r, int ld,
                         float lambda, float* Kt, float* Mt, float* colmin, cudaStream_t st) {
  const size_t smem = sizeof(float) * (BK_TI * BK_STR + BK_TW * BK_STR + BK_TW * BK_LDM);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(build_ktilde_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr = true;
  }
  const int64_t grid = (V + BK_TW - 1) / BK_TW;
  build_ktilde_kernel<<<(unsigned)grid, 256, smem, st>>>(E, V, d, sel, v_r, ld, lambda, Kt, Mt, colmin);
}

// U = gathers in flight per lane per step: NG*U covers a 32-entry chunk where registers allow.
#define WMD_DISPATCH_G(ld, MACRO) \
  switch (lanes_per_row(ld)) {    \
    case 2: MACRO(2, 2); break;   \
    case 4: MACRO(4, 4); break;   \
    case 8: MACRO(8, 8); break;   \
    case 16: MACRO(16, 8); break; \
    default: MACRO(32, 8); break; \
  }

// Persistent grid for the per-iteration kernel: 3 resident 256-thread blocks per SM.
unsigned iter_grid(int64_t N) {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
  }
  const int64_t need = (N + 7) / 8;
  return (unsigned)std::min<int64_t>(need, (int64_t)sms * 3);
}

void launch_sddmm_spmm_iter(const int32_t* doc_ptr, const Entry* ent, int64_t N, const float* Kt,
                            int ld, int v_r, const float* rpad, const float* u_in, float* u_out,
                            uint8_t* flags, cudaStream_t st) {
  const unsigned grid = iter_grid(N);
#define L_(G, U) sddmm_spmm_iter_kernel<G, U><<<grid, 256, 0, st>>>(doc_ptr, ent, N, Kt, ld, (float)v_r, rpad, u_in, u_out, flags)
  WMD_DISPATCH_G(ld, L_)
#undef L_
}

void launch_final_wmd(const int32_t* doc_ptr, const Entry* ent, int64_t N, const float* Kt,
                      const float* Mt, int ld, int v_r, const float* rpad, const float* u_in,
                      float* dist, uint8_t* flags, int32_t* flagged_list, int32_t* flagged_count,
                      cudaStream_t st) {
  const unsigned grid = (unsigned)((N + 7) / 8);
#define L_(G, U) final_wmd_kernel<G, U><<<grid, 256, 0, st>>>(doc_ptr, ent, N, Kt, Mt, ld, (float)v_r, rpad, u_in, dist, flags, flagged_list, flagged_count)
  WMD_DISPATCH_G(ld, L_)
#undef L_
}

size_t fallback_scratch_bytes(int64_t max_doc_nnz) {
  return sizeof(double) * (size_t)kFallbackBlocks * (size_t)(max_doc_nnz * WMD_MAX_VR_DEV + 2 * max_doc_nnz);
}

void launch_fallback_fp64(const float* Mt, const float* colmin, int ld, const float* rpad, int v_r,
                          double lambda, int iters, const int32_t* doc_ptr, const Entry* ent,
                          const int32_t* flagged_list, const int32_t* flagged_count,
                          double* scratch, int64_t max_doc_nnz, float* dist, uint8_t* flags,
                          int32_t* breakdown, int32_t* fallback_count, cudaStream_t st) {
  fallback_fp64_kernel<<<kFallbackBlocks, 256, 0, st>>>(Mt, colmin, ld, rpad, v_r, lambda, iters, doc_ptr,
                                                        ent, flagged_list, flagged_count, scratch,
                                                        max_doc_nnz, dist, flags, breakdown,
                                                        fallback_count);
}

void launch_check_finite(const float* x, int64_t n, int32_t* bad, cudaStream_t st) {
  check_finite_kernel<<<148 * 4, 256, 0, st>>>(x, n, bad);
}

bool fused_supported(int, int64_t) { return false; }
void launch_sinkhorn_fused(const int32_t*, const Entry*, int64_t, const float*, const float*, int,
                           int, const float*, int, float*, uint8_t*, int32_t*, int32_t*, int64_t,
                           cudaStream_t) {}

}  // namespace wmd
