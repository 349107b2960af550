// wmd_fused.cu — NEXT-1: all Sinkhorn iterations and the final step of a
// document in ONE launch, with the document's K~ block resident in registers.
//
// Algorithm 1 touches document j only through c[:,j], x[:,j] and u[:,j]
// (PAPER.md:62-66), so the t iterations of one document need nothing from any other document:
// the K~ rows of its nonzeros are gathered from L2 once, the iterations run on chip, u never
// goes to memory, and c is read once (the per-iteration path streams c and u and re-gathers
// K~ every iteration). Arithmetic is identical in kind to the per-iteration path: FP32, the
// exact column rescale, the exact power-of-two gauge and the FP32 range certificate.
//
// Mapping: one warp per document (warp-persistent over the length-sorted order). The warp
// keeps the n x v_r block twice:
//   row copy    lane e holds K~[k_e, 0:LD)        -> s_e = sum_i K~_ei u_i is lane-local
//   column copy lane i holds K~[k_0..k_{n-1}, i] -> acc_i = sum_e K~_ei v~_e is lane-local
// and exchanges only the two vectors u (v_r floats) and v~ (n floats) per iteration through
// shared memory (broadcast float4 reads). Per iteration: ~2 * 32 FMA instructions per warp
// plus two divisions per lane; the gauge and the certificate use redux.sync on the bit
// patterns of positive floats. Bound: FP32 issue.
#include <algorithm>
#include <cfloat>
#include <cstdint>

#include "wmd_device.cuh"

namespace wmd {
namespace {

using namespace dev;

// Resident 256-thread blocks per SM: 2 (<= 128 registers) when both copies of the block plus
// ~40 registers of state fit, else 1.
template <int LD, int NW>
constexpr int fused_blocks_per_sm() {
  return (NW * LD + ((LD + 31) / 32) * 32 * NW + 40 <= 128) ? 2 : 1;
}

// LD: row stride of K~ (v_r rounded up to 8), <= 64. NW: nonzeros per lane (n <= 32 * NW).
template <int LD, int NW>
__global__ void __launch_bounds__(256, fused_blocks_per_sm<LD, NW>()) sinkhorn_fused_kernel(
    const int32_t* __restrict__ order, const int32_t* __restrict__ doc_ptr,
    const Entry* __restrict__ ent, int64_t pos0, int64_t pos1, const float* __restrict__ Kt,
    const float* __restrict__ Mt, int v_r, const float* __restrict__ rpad, int iters,
    float* __restrict__ dist, uint8_t* __restrict__ flags, int32_t* __restrict__ flagged_list,
    int32_t* __restrict__ flagged_count) {
  constexpr int CPL = (LD + 31) / 32;  // query rows (columns of the block) per lane
  constexpr int NMAX = 32 * NW;
  static_assert(LD % 8 == 0 && LD <= 64, "LD");
  __shared__ __align__(16) float sh_u[8][32 * CPL];
  __shared__ __align__(16) float sh_v[8][NMAX];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  float* su = sh_u[wib];
  float* sv = sh_v[wib];
  const int64_t nwarps = (int64_t)gridDim.x * (blockDim.x >> 5);
  const uint64_t keep = l2_evict_last_policy();
  const float4* Kt4 = reinterpret_cast<const float4*>(Kt);
  const float4* Mt4 = reinterpret_cast<const float4*>(Mt);
  const int2* ent2 = reinterpret_cast<const int2*>(ent);
  const float u0 = (float)v_r;
  float r[CPL];
#pragma unroll
  for (int c = 0; c < CPL; ++c) r[c] = (lane + 32 * c < LD) ? __ldg(rpad + lane + 32 * c) : 0.f;

  for (int64_t pos = pos0 + (int64_t)blockIdx.x * (blockDim.x >> 5) + wib; pos < pos1; pos += nwarps) {
    const int j = __ldg(order + pos);
    const int b = __ldg(doc_ptr + j);
    const int n = __ldg(doc_ptr + j + 1) - b;
    // ---- load the document: its nonzeros and both copies of its K~ block
    int ke[NW];
    float ce[NW];
    bool ve[NW];
#pragma unroll
    for (int w = 0; w < NW; ++w) {
      const int e = lane + 32 * w;
      ve[w] = e < n;
      const int2 x = ve[w] ? __ldg(ent2 + b + e) : make_int2(0, 0);  // empty slots: row 0, c = 0
      ke[w] = x.x;
      ce[w] = __int_as_float(x.y);
    }
    float kr[NW][LD];
#pragma unroll
    for (int w = 0; w < NW; ++w)
#pragma unroll
      for (int q = 0; q < LD / 4; ++q) {
        const float4 t = ldg4_keep(Kt4 + (uint32_t)ke[w] * (LD / 4) + q, keep);
        kr[w][4 * q] = t.x; kr[w][4 * q + 1] = t.y; kr[w][4 * q + 2] = t.z; kr[w][4 * q + 3] = t.w;
      }
    float kc[CPL][NMAX];
    bool under[CPL];
#pragma unroll
    for (int c = 0; c < CPL; ++c) under[c] = false;
#pragma unroll
    for (int e = 0; e < NMAX; ++e) {
      const int k = __shfl_sync(kFull, ke[e / 32], e % 32);
#pragma unroll
      for (int c = 0; c < CPL; ++c) {
        const int col = lane + 32 * c;
        kc[c][e] = (col < LD) ? ldg_keep(Kt + (uint32_t)k * LD + col, keep) : 0.f;
        under[c] |= (e < n) && (r[c] > 0.f) && kc[c][e] < FLT_MIN;  // static underflow rows
      }
    }
    float u[CPL];
#pragma unroll
    for (int c = 0; c < CPL; ++c) u[c] = r[c] > 0.f ? u0 : 0.f;  // x0 = 1/v_r
    bool bad = false;
    float vt[NW];
    for (int it = 0;; ++it) {
      // ---- broadcast u, then SDDMM: s_e = K~[e,:] . u and v~_e = c_e / s_e (lane-local)
      __syncwarp();
#pragma unroll
      for (int c = 0; c < CPL; ++c) su[lane + 32 * c] = u[c];
      __syncwarp();
      // four independent FMA chains per dot product (FMA latency, few resident warps)
      float s[NW], sp[NW][4];
#pragma unroll
      for (int w = 0; w < NW; ++w) sp[w][0] = sp[w][1] = sp[w][2] = sp[w][3] = 0.f;
#pragma unroll
      for (int q = 0; q < LD / 4; ++q) {
        const float4 uu = *reinterpret_cast<const float4*>(su + 4 * q);
#pragma unroll
        for (int w = 0; w < NW; ++w) {
          sp[w][0] = fmaf(kr[w][4 * q], uu.x, sp[w][0]);
          sp[w][1] = fmaf(kr[w][4 * q + 1], uu.y, sp[w][1]);
          sp[w][2] = fmaf(kr[w][4 * q + 2], uu.z, sp[w][2]);
          sp[w][3] = fmaf(kr[w][4 * q + 3], uu.w, sp[w][3]);
        }
      }
#pragma unroll
      for (int w = 0; w < NW; ++w) s[w] = (sp[w][0] + sp[w][1]) + (sp[w][2] + sp[w][3]);
      uint32_t smin_b = 0xffffffffu, vmax_b = 0u, umu_b = 0u;
#pragma unroll
      for (int w = 0; w < NW; ++w) {
        // empty slots divide 1 by 1 (a zero numerator would take the IEEE slow path)
        vt[w] = (ve[w] ? ce[w] : 1.f) / (ve[w] ? s[w] : 1.f);
        if (!ve[w]) vt[w] = 0.f;
        if (ve[w]) smin_b = min(smin_b, __float_as_uint(s[w]));
        vmax_b = max(vmax_b, __float_as_uint(vt[w]));
      }
#pragma unroll
      for (int c = 0; c < CPL; ++c)
        if (under[c]) umu_b = max(umu_b, __float_as_uint(u[c]));
      // certificate for the sums s (positive floats order like their bit patterns)
      smin_b = __reduce_min_sync(kFull, smin_b);
      umu_b = __reduce_max_sync(kFull, umu_b);
      vmax_b = __reduce_max_sync(kFull, vmax_b);
      bad |= __uint_as_float(umu_b) * (u0 * kUnderScale) > __uint_as_float(smin_b) ||
             vmax_b > 0x7f7fffffu;
      if (it == iters || bad) break;  // after `iters` x-updates: the final step below
      // ---- broadcast v~, then SpMM: acc_i = K~[:,i] . v~ (lane-local), u_i = r_i / acc_i
#pragma unroll
      for (int w = 0; w < NW; ++w) sv[lane + 32 * w] = vt[w];
      __syncwarp();
      float acc[CPL], ap[CPL][4];
#pragma unroll
      for (int c = 0; c < CPL; ++c) ap[c][0] = ap[c][1] = ap[c][2] = ap[c][3] = 0.f;
#pragma unroll
      for (int e4 = 0; e4 < NMAX / 4; ++e4) {
        const float4 vv = *reinterpret_cast<const float4*>(sv + 4 * e4);
#pragma unroll
        for (int c = 0; c < CPL; ++c) {
          ap[c][0] = fmaf(kc[c][4 * e4], vv.x, ap[c][0]);
          ap[c][1] = fmaf(kc[c][4 * e4 + 1], vv.y, ap[c][1]);
          ap[c][2] = fmaf(kc[c][4 * e4 + 2], vv.z, ap[c][2]);
          ap[c][3] = fmaf(kc[c][4 * e4 + 3], vv.w, ap[c][3]);
        }
      }
#pragma unroll
      for (int c = 0; c < CPL; ++c) acc[c] = (ap[c][0] + ap[c][1]) + (ap[c][2] + ap[c][3]);
      const float vcap = (float)n * __uint_as_float(vmax_b) * kUnderScale;
      uint32_t umax_b = 0u, umin_b = 0xffffffffu;
      float un[CPL];
#pragma unroll
      for (int c = 0; c < CPL; ++c) {
        un[c] = (r[c] > 0.f ? r[c] : 1.f) / (r[c] > 0.f ? acc[c] : 1.f);  // padded rows: 1/1
        if (!(r[c] > 0.f)) un[c] = 0.f;
        if (r[c] > 0.f) {
          bad |= under[c] && vcap > acc[c];
          umax_b = max(umax_b, __float_as_uint(un[c]));
          umin_b = min(umin_b, __float_as_uint(un[c]));
        }
      }
      umax_b = __reduce_max_sync(kFull, umax_b);
      umin_b = __reduce_min_sync(kFull, umin_b);
      bad = __any_sync(kFull, bad) || umin_b < 0x00800000u || umax_b > 0x7f7fffffu;
      if (bad) break;
      const float sc = gauge_scale(umax_b, umin_b);  // exact power of two
#pragma unroll
      for (int c = 0; c < CPL; ++c) u[c] = un[c] * sc;
    }
    // ---- final step: WMD_j = sum_e v~_e q_e, q_e = sum_i K~_ei M_ei u_i
    float wsum = 0.f;
    if (!bad) {
#pragma unroll
      for (int w = 0; w < NW; ++w) {
        float q = 0.f;
#pragma unroll
        for (int q4 = 0; q4 < LD / 4; ++q4) {
          const float4 m = ldg4_keep(Mt4 + (uint32_t)ke[w] * (LD / 4) + q4, keep);
          const float4 uu = *reinterpret_cast<const float4*>(su + 4 * q4);
          q = fmaf(kr[w][4 * q4] * m.x, uu.x, q);
          q = fmaf(kr[w][4 * q4 + 1] * m.y, uu.y, q);
          q = fmaf(kr[w][4 * q4 + 2] * m.z, uu.z, q);
          q = fmaf(kr[w][4 * q4 + 3] * m.w, uu.w, q);
        }
        if (ve[w]) wsum = fmaf(vt[w], q, wsum);
      }
#pragma unroll
      for (int off = 16; off; off >>= 1) wsum += __shfl_xor_sync(kFull, wsum, off);
    }
    if (lane == 0) {
      dist[j] = wsum;
      if (bad || !(fabsf(wsum) <= FLT_MAX)) {
        flags[j] |= kFlagFp32Range;
        flagged_list[atomicAdd(flagged_count, 1)] = j;
      }
    }
  }
}

template <int LD, int NW>
void launch_fused_range(const int32_t* order, const int32_t* doc_ptr, const Entry* ent, int64_t p0,
                        int64_t p1, const float* Kt, const float* Mt, int v_r, const float* rpad,
                        int iters, float* dist, uint8_t* flags, int32_t* fl, int32_t* fc,
                        cudaStream_t st) {
  if (p1 <= p0) return;
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
  }
  const int per_sm = fused_blocks_per_sm<LD, NW>();
  const int64_t need = (p1 - p0 + 7) / 8;
  const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>(need, (int64_t)sms * per_sm * 4));
  sinkhorn_fused_kernel<LD, NW><<<grid, 256, 0, st>>>(order, doc_ptr, ent, p0, p1, Kt, Mt, v_r, rpad,
                                                       iters, dist, flags, fl, fc);
}

template <int NW>
void dispatch_ld(int ld, const int32_t* order, const int32_t* doc_ptr, const Entry* ent, int64_t p0,
                 int64_t p1, const float* Kt, const float* Mt, int v_r, const float* rpad, int iters,
                 float* dist, uint8_t* flags, int32_t* fl, int32_t* fc, cudaStream_t st) {
#define F_(LD) launch_fused_range<LD, NW>(order, doc_ptr, ent, p0, p1, Kt, Mt, v_r, rpad, iters, dist, flags, fl, fc, st)
  switch (ld) {
    case 8: F_(8); break;
    case 16: F_(16); break;
    case 24: F_(24); break;
    case 32: F_(32); break;
    case 40: if (NW == 1) launch_fused_range<40, 1>(order, doc_ptr, ent, p0, p1, Kt, Mt, v_r, rpad, iters, dist, flags, fl, fc, st); break;
    case 48: if (NW == 1) launch_fused_range<48, 1>(order, doc_ptr, ent, p0, p1, Kt, Mt, v_r, rpad, iters, dist, flags, fl, fc, st); break;
    case 56: if (NW == 1) launch_fused_range<56, 1>(order, doc_ptr, ent, p0, p1, Kt, Mt, v_r, rpad, iters, dist, flags, fl, fc, st); break;
    case 64: if (NW == 1) launch_fused_range<64, 1>(order, doc_ptr, ent, p0, p1, Kt, Mt, v_r, rpad, iters, dist, flags, fl, fc, st); break;
    default: break;
  }
#undef F_
}

}  // namespace

bool fused_supported(int ld, int64_t max_doc_nnz) {
  if (ld <= 32) return max_doc_nnz <= 64;
  return ld <= 64 && max_doc_nnz <= 32;
}

void launch_sinkhorn_fused(const int32_t* order, const int32_t* doc_ptr, const Entry* ent, int64_t N,
                           int64_t n_short, const float* Kt, const float* Mt, int ld, int v_r,
                           const float* rpad, int iters, float* dist, uint8_t* flags,
                           int32_t* flagged_list, int32_t* flagged_count, cudaStream_t st) {
  // documents [0, n_short) of the length-sorted order have <= 32 nonzeros, the rest <= 64
  dispatch_ld<1>(ld, order, doc_ptr, ent, 0, n_short, Kt, Mt, v_r, rpad, iters, dist, flags,
                 flagged_list, flagged_count, st);
  if (ld <= 32)
    dispatch_ld<2>(ld, order, doc_ptr, ent, n_short, N, Kt, Mt, v_r, rpad, iters, dist, flags,
                   flagged_list, flagged_count, st);
}

}  // namespace wmd
