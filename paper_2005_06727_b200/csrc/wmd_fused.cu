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
//   column copy lane i holds K~[k_0..k_{NE-1}, i] -> acc_i = sum_e K~_ei v~_e is lane-local
// and exchanges only the two vectors u (v_r floats) and v~ (n floats) per iteration through
// shared memory (broadcast float4 reads). Per iteration: LD + NE FMA instructions per warp,
// two reciprocals per lane, two redux.sync for the gauge. The range certificate is tracked
// per lane in gauge-invariant form and reduced once per document. Bound: FP32 issue
// (DESIGN.md §5).
#include <algorithm>
#include <cfloat>
#include <cstdint>

#include "wmd_device.cuh"

namespace wmd {
namespace {

using namespace dev;

constexpr int kFusedThreads = 128;  // 4 warps per block: finer register-limited occupancy steps
#ifndef FUSED_STATE_REGS
#define FUSED_STATE_REGS 40
#endif

// Registers for the two copies of the block plus ~40 of state -> resident blocks per SM.
template <int LD, int NE>
constexpr int fused_min_blocks() {
  constexpr int nw = (NE + 31) / 32, cpl = (LD + 31) / 32;
  constexpr int regs = ((nw * LD + cpl * NE + FUSED_STATE_REGS) + 7) / 8 * 8;
  constexpr int b = 65536 / (kFusedThreads * regs);
  return b < 1 ? 1 : (b > 16 ? 16 : b);
}

// LD: row stride of K~ (v_r rounded up to 8), <= 64. NE: maximum nonzeros per document (<= 64).
template <int LD, int NE>
__global__ void __launch_bounds__(kFusedThreads, fused_min_blocks<LD, NE>()) sinkhorn_fused_kernel(
    const int32_t* __restrict__ order, const int32_t* __restrict__ doc_ptr,
    const Entry* __restrict__ ent, int64_t pos0, int64_t pos1, const float* __restrict__ Kt,
    const float* __restrict__ Mt, int v_r, const float* __restrict__ rpad, int iters,
    float* __restrict__ dist, uint8_t* __restrict__ flags, int32_t* __restrict__ flagged_list,
    int32_t* __restrict__ flagged_count) {
  constexpr int CPL = (LD + 31) / 32;  // query rows (columns of the block) per lane
  constexpr int NW = (NE + 31) / 32;   // nonzero slots per lane (row copy)
  constexpr int NEP = (NE + 3) / 4 * 4;
  constexpr int WARPS = kFusedThreads / 32;
  static_assert(LD % 8 == 0 && LD <= 64 && NE <= 64, "shape");
  __shared__ __align__(16) float sh_u[WARPS][32 * CPL];
  __shared__ __align__(16) float sh_v[WARPS][32 * NW];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  float* su = sh_u[wib];
  float* sv = sh_v[wib];
  const int64_t nwarps = (int64_t)gridDim.x * WARPS;
  const uint64_t keep = l2_evict_last_policy();
  const float4* Kt4 = reinterpret_cast<const float4*>(Kt);
  const float4* Mt4 = reinterpret_cast<const float4*>(Mt);
  const int2* ent2 = reinterpret_cast<const int2*>(ent);
  const float u0 = (float)v_r;
  float r[CPL];
#pragma unroll
  for (int c = 0; c < CPL; ++c) r[c] = (lane + 32 * c < LD) ? __ldg(rpad + lane + 32 * c) : 0.f;

  for (int64_t pos = pos0 + (int64_t)blockIdx.x * WARPS + wib; pos < pos1; pos += nwarps) {
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
    for (int w = 0; w < NW; ++w) {
      const bool load = (w == 0) || (lane + 32 * w < NE);
#pragma unroll
      for (int q = 0; q < LD / 4; ++q) {
        const float4 t = load ? ldg4_keep(Kt4 + (uint32_t)ke[w] * (LD / 4) + q, keep)
                              : make_float4(0.f, 0.f, 0.f, 0.f);
        kr[w][4 * q] = t.x; kr[w][4 * q + 1] = t.y; kr[w][4 * q + 2] = t.z; kr[w][4 * q + 3] = t.w;
      }
    }
    float kc[CPL][NEP];
    bool under[CPL];
#pragma unroll
    for (int c = 0; c < CPL; ++c) under[c] = false;
#pragma unroll
    for (int e = 0; e < NEP; ++e) {
      const int k = __shfl_sync(kFull, ke[(e < NE ? e : 0) / 32], e % 32);
#pragma unroll
      for (int c = 0; c < CPL; ++c) {
        const int col = lane + 32 * c;
        kc[c][e] = (col < LD && e < NE) ? ldg_keep(Kt + (uint32_t)k * LD + col, keep) : 0.f;
        under[c] |= (e < n) && (r[c] > 0.f) && kc[c][e] < FLT_MIN;  // static underflow rows
      }
    }
    float u[CPL];
#pragma unroll
    for (int c = 0; c < CPL; ++c) u[c] = r[c] > 0.f ? u0 : 0.f;  // x0 = 1/v_r
    bool any_under = false;
#pragma unroll
    for (int c = 0; c < CPL; ++c) any_under |= under[c];
    any_under = __any_sync(kFull, any_under);
    bool bad = false;
    float vt[NW];
    for (int it = 0;; ++it) {
      // ---- broadcast u, then SDDMM: s_e = K~[e,:] . u and v~_e = c_e / s_e (lane-local)
      __syncwarp();
#pragma unroll
      for (int c = 0; c < CPL; ++c) su[lane + 32 * c] = u[c];
      __syncwarp();
      float sp[NW][4];  // four independent FMA chains per dot product
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
      // certificate of this iteration (kUnderScale): positive floats order like their bits
      uint32_t umu_b = 0u, smin_b = 0xffffffffu, vmax_b = 0u;
#pragma unroll
      for (int c = 0; c < CPL; ++c)
        if (under[c]) umu_b = max(umu_b, __float_as_uint(u[c]));
#pragma unroll
      for (int w = 0; w < NW; ++w) {
        const float s = (sp[w][0] + sp[w][1]) + (sp[w][2] + sp[w][3]);
        vt[w] = ve[w] ? ce[w] * rcp_fast(s) : 0.f;
        if (ve[w]) smin_b = min(smin_b, __float_as_uint(s));
        vmax_b = max(vmax_b, __float_as_uint(vt[w]));
      }
      if (any_under) {
        umu_b = __reduce_max_sync(kFull, umu_b);
        smin_b = __reduce_min_sync(kFull, smin_b);
        bad |= __uint_as_float(umu_b) * (u0 * kUnderScale) > __uint_as_float(smin_b);
      }
      vmax_b = __reduce_max_sync(kFull, vmax_b);
      bad |= vmax_b > 0x7f7fffffu;
      if (it == iters || bad) break;  // after `iters` x-updates: the final step below
      // ---- broadcast v~, then SpMM: acc_i = K~[:,i] . v~ (lane-local), u_i = r_i / acc_i
#pragma unroll
      for (int w = 0; w < NW; ++w) sv[lane + 32 * w] = vt[w];
      __syncwarp();
      float ap[CPL][4];
#pragma unroll
      for (int c = 0; c < CPL; ++c) ap[c][0] = ap[c][1] = ap[c][2] = ap[c][3] = 0.f;
#pragma unroll
      for (int e4 = 0; e4 < NEP / 4; ++e4) {
        const float4 vv = *reinterpret_cast<const float4*>(sv + 4 * e4);
#pragma unroll
        for (int c = 0; c < CPL; ++c) {
          ap[c][0] = fmaf(kc[c][4 * e4], vv.x, ap[c][0]);
          ap[c][1] = fmaf(kc[c][4 * e4 + 1], vv.y, ap[c][1]);
          ap[c][2] = fmaf(kc[c][4 * e4 + 2], vv.z, ap[c][2]);
          ap[c][3] = fmaf(kc[c][4 * e4 + 3], vv.w, ap[c][3]);
        }
      }
      uint32_t umax_b = 0u, umin_b = 0xffffffffu;
      const float vcap = (float)n * __uint_as_float(vmax_b) * kUnderScale;  // underflowed terms
      bool bad_l = false;
      float un[CPL];
#pragma unroll
      for (int c = 0; c < CPL; ++c) {
        const float acc = (ap[c][0] + ap[c][1]) + (ap[c][2] + ap[c][3]);
        un[c] = r[c] > 0.f ? r[c] * rcp_fast(acc) : 0.f;
        if (r[c] > 0.f) {
          bad_l |= under[c] && vcap > acc;
          umax_b = max(umax_b, __float_as_uint(un[c]));
          umin_b = min(umin_b, __float_as_uint(un[c]));
        }
      }
      // gauge: positive floats order like their bit patterns
      umax_b = __reduce_max_sync(kFull, umax_b);
      umin_b = __reduce_min_sync(kFull, umin_b);
      if (__any_sync(kFull, bad_l) || umin_b < 0x00800000u || umax_b > 0x7f7fffffu) {
        bad = true;  // an underflowed term could matter, or u left the normal range
        break;
      }
      const float sc = gauge_scale(umax_b, umin_b);  // exact power of two
#pragma unroll
      for (int c = 0; c < CPL; ++c) u[c] = un[c] * sc;
    }
    // ---- final step: WMD_j = sum_e v~_e q_e,  q_e = sum_i K~_ei M_ei u_i
    float wsum = 0.f;
    if (!bad) {
#pragma unroll
      for (int w = 0; w < NW; ++w) {
        if (w > 0 && !__any_sync(kFull, ve[w])) break;
        float q0 = 0.f, q1 = 0.f;
#pragma unroll
        for (int q4 = 0; q4 < LD / 4; ++q4) {
          const float4 m = ldg4_keep(Mt4 + (uint32_t)ke[w] * (LD / 4) + q4, keep);
          const float4 uu = *reinterpret_cast<const float4*>(su + 4 * q4);
          q0 = fmaf(kr[w][4 * q4] * m.x, uu.x, q0);
          q1 = fmaf(kr[w][4 * q4 + 1] * m.y, uu.y, q1);
          q0 = fmaf(kr[w][4 * q4 + 2] * m.z, uu.z, q0);
          q1 = fmaf(kr[w][4 * q4 + 3] * m.w, uu.w, q1);
        }
        if (ve[w]) wsum = fmaf(vt[w], q0 + q1, wsum);
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

int num_sms() {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
  }
  return sms;
}

template <int LD, int NE>
void launch_fused_range(const int32_t* order, const int32_t* doc_ptr, const Entry* ent, int64_t p0,
                        int64_t p1, const float* Kt, const float* Mt, int v_r, const float* rpad,
                        int iters, float* dist, uint8_t* flags, int32_t* fl, int32_t* fc,
                        cudaStream_t st) {
  if (p1 <= p0) return;
  constexpr int warps = kFusedThreads / 32;
  const int64_t need = (p1 - p0 + warps - 1) / warps;
  const int64_t resident = (int64_t)num_sms() * fused_min_blocks<LD, NE>();
  const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>(need, resident * 4));
  sinkhorn_fused_kernel<LD, NE><<<grid, kFusedThreads, 0, st>>>(order, doc_ptr, ent, p0, p1, Kt, Mt,
                                                                 v_r, rpad, iters, dist, flags, fl, fc);
}

// Document-length buckets of the fused kernel (the order is sorted by length).
constexpr int kBuckets[] = {32, 40, 48, 64};

template <int NE>
void dispatch_ld(int ld, const int32_t* order, const int32_t* doc_ptr, const Entry* ent, int64_t p0,
                 int64_t p1, const float* Kt, const float* Mt, int v_r, const float* rpad, int iters,
                 float* dist, uint8_t* flags, int32_t* fl, int32_t* fc, cudaStream_t st) {
#define F_(LD) launch_fused_range<LD, NE>(order, doc_ptr, ent, p0, p1, Kt, Mt, v_r, rpad, iters, dist, flags, fl, fc, st)
  switch (ld) {
    case 8: F_(8); break;
    case 16: F_(16); break;
    case 24: F_(24); break;
    case 32: F_(32); break;
    case 40: if (NE <= 32) launch_fused_range<40, 32>(order, doc_ptr, ent, p0, p1, Kt, Mt, v_r, rpad, iters, dist, flags, fl, fc, st); break;
    case 48: if (NE <= 32) launch_fused_range<48, 32>(order, doc_ptr, ent, p0, p1, Kt, Mt, v_r, rpad, iters, dist, flags, fl, fc, st); break;
    case 56: if (NE <= 32) launch_fused_range<56, 32>(order, doc_ptr, ent, p0, p1, Kt, Mt, v_r, rpad, iters, dist, flags, fl, fc, st); break;
    case 64: if (NE <= 32) launch_fused_range<64, 32>(order, doc_ptr, ent, p0, p1, Kt, Mt, v_r, rpad, iters, dist, flags, fl, fc, st); break;
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
                           const int64_t* len_prefix, int64_t max_len, const float* Kt,
                           const float* Mt, int ld, int v_r, const float* rpad, int iters,
                           float* dist, uint8_t* flags, int32_t* flagged_list,
                           int32_t* flagged_count, cudaStream_t st) {
  // len_prefix[L] = number of documents with fewer than L nonzeros: the length-sorted order
  // splits into buckets of at most 32 / 40 / 48 / 64 nonzeros, one launch each.
  int64_t p0 = 0;
  for (int bi = 0; bi < 4 && p0 < N; ++bi) {
    const int NE = kBuckets[bi];
    const int64_t p1 = NE >= max_len ? N : len_prefix[NE + 1];
    if (p1 > p0) {
      switch (NE) {
        case 32: dispatch_ld<32>(ld, order, doc_ptr, ent, p0, p1, Kt, Mt, v_r, rpad, iters, dist, flags, flagged_list, flagged_count, st); break;
        case 40: dispatch_ld<40>(ld, order, doc_ptr, ent, p0, p1, Kt, Mt, v_r, rpad, iters, dist, flags, flagged_list, flagged_count, st); break;
        case 48: dispatch_ld<48>(ld, order, doc_ptr, ent, p0, p1, Kt, Mt, v_r, rpad, iters, dist, flags, flagged_list, flagged_count, st); break;
        default: dispatch_ld<64>(ld, order, doc_ptr, ent, p0, p1, Kt, Mt, v_r, rpad, iters, dist, flags, flagged_list, flagged_count, st); break;
      }
    }
    p0 = p1;
  }
}

int fused_launch_count(const int64_t* len_prefix, int64_t max_len, int64_t N) {
  int64_t p0 = 0;
  int cnt = 0;
  for (int bi = 0; bi < 4 && p0 < N; ++bi) {
    const int64_t p1 = kBuckets[bi] >= max_len ? N : len_prefix[kBuckets[bi] + 1];
    cnt += p1 > p0;
    p0 = p1;
  }
  return cnt;
}

}  // namespace wmd
