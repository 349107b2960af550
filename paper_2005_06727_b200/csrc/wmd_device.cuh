// wmd_device.cuh — device helpers shared by the kernels of wmd_kernels.cu and wmd_fused.cu.
#pragma once
#include <cfloat>
#include <cstdint>

#include "wmd_internal.h"

namespace wmd {
namespace dev {

constexpr unsigned kFull = 0xffffffffu;

// FP32 range certificate (R21). A K~ entry below FLT_MIN = 2^-126 is subnormal or
// flushed to 0 and carries an absolute error of up to 2^-149 (a normal entry only its relative
// rounding). A document keeps its FP32 result only if, in every sum of every iteration,
//     s_e   = sum_i K~_ki u_i :   u_i * v_r * 2^-149 <= 2^-16 * s_e   for each underflowed K~_ki
//     acc_i = sum_e K~_ki v~_e:   (sum_{e: K~_ki underflowed} v~_e) * 2^-149 <= 2^-16 * acc_i
// otherwise it is flagged for the FP64 re-run. The test is gauge-invariant (u -> a u scales s by
// a and v~, acc by 1/a) and only fires when underflowed entries could matter: the FP32 error of
// a certified sum stays ~1e-6 relative (measured: DESIGN.md §4). Kernels apply it in the
// conservative form "max over rows with any underflowed entry in the document".
constexpr float kUnderScale = 0x1p-133f;  // 2^-149 / 2^-16

__device__ __forceinline__ bool normal_pos(float x) { return x >= FLT_MIN && x <= FLT_MAX; }

// Read-only loads that stay behind their guard: an `if (i < n) x = __ldg(p + i)` may be hoisted
// above the guard by the compiler (it treats __ldg as free of side effects), which reads past the
// end of an array; the asm volatile form is neither hoisted nor speculated.
__device__ __forceinline__ int ldg_guarded(const int* p) {
  int v;
  asm volatile("ld.global.nc.s32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ int2 ldg_guarded(const int2* p) {
  int2 v;
  asm volatile("ld.global.nc.v2.s32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "l"(p));
  return v;
}
// streaming variant (read once): L2 evict_first, so the gathered tables keep their L2 lines
__device__ __forceinline__ int2 ldg_guarded_stream(const int2* p, uint64_t pol) {
  int2 v;
  asm volatile("ld.global.nc.L2::cache_hint.v2.s32 {%0, %1}, [%2], %3;" : "=r"(v.x), "=r"(v.y) : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ float4 ldg4_hint(const float4* p, uint64_t pol) {
  float4 v;
  asm("ld.global.nc.L2::cache_hint.v4.f32 {%0, %1, %2, %3}, [%4], %5;"
      : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ int2 ldg2_hint(const int2* p, uint64_t pol) {
  int2 v;
  asm("ld.global.nc.L2::cache_hint.v2.s32 {%0, %1}, [%2], %3;" : "=r"(v.x), "=r"(v.y) : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ uint64_t l2_evict_first_policy() {
  uint64_t pol;
  asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ int4 ldg_guarded(const int4* p) {
  int4 v;
  asm volatile("ld.global.nc.v4.s32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
  return v;
}

// L2 residency: the K~ / M tables (<= V*ld*4 bytes, 51 MB at Scaling) are gathered repeatedly
// and should stay in the 126 MB L2 while c and u stream past them: table gathers carry an
// evict_last policy.
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
__device__ __forceinline__ float ldg_keep(const float* p, uint64_t pol) {
#ifdef WMD_NO_L2_HINTS
  return __ldg(p);
#else
  float v;
  asm("ld.global.nc.L2::cache_hint.f32 %0, [%1], %2;" : "=f"(v) : "l"(p), "l"(pol));
  return v;
#endif
}

// Fast reciprocal (MUFU.RCP, relative error <= 2^-23, subnormal input -> inf). Used where the
// input is either normal or the document is flagged anyway: s_e >= u_{i*} (the column-minimum
// row has K~ = 1) is normal whenever u is, and a subnormal acc_i yields u_i = inf, which the
// range check rejects.
__device__ __forceinline__ float rcp_fast(float x) {
  float y;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// Exact power-of-two gauge factor 2^-floor((e_max + e_min)/2) from the bit patterns of the
// largest and smallest (positive, normal) entries: the biased exponent is bits >> 23.
__device__ __forceinline__ float gauge_scale(uint32_t max_bits, uint32_t min_bits) {
  const int g = ((int)(max_bits >> 23) + (int)(min_bits >> 23) - 254) >> 1;  // floor
  return __uint_as_float((uint32_t)(127 - g) << 23);                         // |g| <= 126
}

}  // namespace dev
}  // namespace wmd
