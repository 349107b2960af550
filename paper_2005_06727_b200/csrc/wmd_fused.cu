// wmd_fused.cu — NEXT-1: all Sinkhorn iterations and the final step of a
// document in ONE launch, the document's kernel block resident in registers.
//
// Algorithm 1 touches document j only through c[:,j], x[:,j] and u[:,j]
// (PAPER.md:62-66), so the t iterations of one document need nothing from any other document:
// the M rows of its nonzeros are fetched once, the iterations run on chip, u never goes to
// memory and c is read once.
//
// Doc-local two-sided rescale (R21). With D_ei = M_ie - m_e (m_e = min_i M_ie,
// the build's vocabulary-wide column minimum) and mu_i = min_{e in doc} D_ei, the kernel uses
//     Kh_ei = exp(-lambda (D_ei - mu_i)) = K_ie e^{lambda m_e} e^{lambda mu_i}      (in (0, 1])
// which has a 1 in every row and every column of the document block. Substituting
// u = uh e^{-lambda mu}, v = vh e^{-lambda m} into Algorithm 1 gives the same iteration with Kh
// (exact in real arithmetic), started from uh0_i = v_r e^{-lambda mu_i} (x0 = 1/v_r),
// and the same distance WMD = sum_e vh_e sum_i Kh_ei M_ie uh_i. Every sum then has
// a unit-size term, so FP32 only loses range when the scalings themselves spread by >2^100.
// Each iteration applies an exact power-of-two gauge to uh (R21).
//
// FP32 range certificate (kUnder): an entry flushed to 0 (true value < 2^-126) is an absolute
// error < 2^-126 in its product. A document keeps its FP32 result only if every sum that has a
// flushed term satisfies, every iteration,
//     s_e   = sum_i Kh_ei uh_i :  v_r * max_i uh_i * 2^-126 <= 2^-16 s_e
//     acc_i = sum_e Kh_ei vh_e :  n   * max_e vh_e * 2^-126 <= 2^-16 acc_i
// and all uh stay normal; otherwise it is flagged and recomputed in FP64 (fallback_fp64).
//
// Mapping: one warp per document, warp-persistent over the length-sorted order. The warp keeps
// the n x v_r block twice:
//   row copy    lane e holds Kh[e, 0:LD)          -> s_e = Kh[e,:] . uh is lane-local
//   column copy lane i holds Kh[0:NE, i]          -> acc_i = Kh[:,i] . vh is lane-local
// and exchanges only uh (v_r floats) and vh (n floats) per iteration through shared memory
// (broadcast float4 reads). The block is built from the M rows staged in shared memory by
// cp.async (prefetched during the previous document's iterations): the column copy computes
// D, mu and Kh (one ex2 per entry) and hands Kh to the row copy through a second shared buffer.
// Per iteration: LD + NE FFMA per warp, two reciprocals per lane, three redux.sync (the v
// maximum for the certificate and the gauge's max / min); no global memory traffic.
// Bound: FP32 issue.
#include <algorithm>
#include <cfloat>
#include <cstdint>

#include "wmd_device.cuh"

namespace wmd {
namespace {

using namespace dev;

constexpr int kWarps = 4;                  // warps per block
constexpr int kThreads = 32 * kWarps;
constexpr float kUnder = 0x1p-110f;        // 2^-126 / 2^-16
constexpr float kLog2e = 1.4426950408889634f;

template <int LD, int NE>
struct Shape {
  static constexpr int CPL = (LD + 31) / 32;   // query rows (block columns) per lane
  static constexpr int NW = (NE + 31) / 32;    // nonzero slots per lane (row copy)
  static constexpr int NEP = (NE + 3) / 4 * 4;
  static constexpr int P = LD + 4;             // row pitch (floats) of Mx and of the smem buffers
  static constexpr int BUF = NE * P;           // one staging buffer
  static constexpr int SU = 32 * CPL, SV = 32 * NW, SM = 32 * NW;
  static constexpr int WARP_FLOATS = 2 * BUF + SU + SV + SM;
  static constexpr int REGS = NW * LD + CPL * NE;  // block registers per lane
};

__device__ __forceinline__ float ex2_ftz(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src, uint64_t pol) {
  asm volatile("cp.async.ca.shared.global.L2::cache_hint [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "l"(pol)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

template <int LD, int NE>
constexpr int min_blocks() {
  constexpr int regs = ((Shape<LD, NE>::REGS + 56) + 7) / 8 * 8;
  constexpr int b = 65536 / (kThreads * regs);
  return b < 1 ? 1 : (b > 8 ? 8 : b);
}

// LD: query rows rounded up to 8 (<= 64). NE: maximum nonzeros per document of this launch.
template <int LD, int NE>
__global__ void __launch_bounds__(kThreads, min_blocks<LD, NE>()) sinkhorn_fused_kernel(
    const int32_t* __restrict__ order, const int32_t* __restrict__ doc_ptr,
    const Entry* __restrict__ ent, int64_t pos0, int64_t pos1, const float* __restrict__ Mx,
    int v_r, const float* __restrict__ rpad, float lambda, int iters, float* __restrict__ dist,
    uint8_t* __restrict__ flags, int32_t* __restrict__ flagged_list,
    int32_t* __restrict__ flagged_count) {
  using S = Shape<LD, NE>;
  constexpr int CPL = S::CPL, NW = S::NW, NEP = S::NEP, P = S::P;
  static_assert(LD % 8 == 0 && LD <= 64 && NE <= 64, "shape");
  extern __shared__ __align__(16) float smem[];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  float* wbase = smem + wib * S::WARP_FLOATS;
  float* buf0 = wbase;
  float* su = wbase + 2 * S::BUF;
  float* sv = su + S::SU;
  float* sm = sv + S::SV;
  const int64_t nwarps = (int64_t)gridDim.x * kWarps;
  const uint64_t keep = l2_evict_last_policy();
  const int2* ent2 = reinterpret_cast<const int2*>(ent);
  const float a = lambda * kLog2e;            // exp(-lambda x) = 2^(-a x)
  const float kv_s = (float)v_r * kUnder;

  float r[CPL];
  bool real[CPL];
#pragma unroll
  for (int c = 0; c < CPL; ++c) {
    const int col = lane + 32 * c;
    real[c] = col < v_r;
    r[c] = (col < LD) ? __ldg(rpad + col) : 0.f;  // zero beyond v_r
  }

  // ---- prefetch machinery: stage 1 (order, doc_ptr), stage 2 (entries), stage 3 (cp.async rows)
  int64_t pos = pos0 + (int64_t)blockIdx.x * kWarps + wib;
  int pj = -1, pb = 0, pn = 0;    // next document: id, first nonzero, length
  int pk[NW];
  float pc[NW];
  int cur = 0;                    // staging buffer of the current document
  auto stage1 = [&](int64_t p) {
    pj = -1; pn = 0;
    if (p < pos1) {
      pj = __ldg(order + p);
      pb = __ldg(doc_ptr + pj);
      pn = __ldg(doc_ptr + pj + 1) - pb;
    }
  };
  auto stage2 = [&]() {
#pragma unroll
    for (int w = 0; w < NW; ++w) {
      const int e = lane + 32 * w;
      int2 x = make_int2(0, 0);
      if (e < pn) x = __ldg(ent2 + pb + e);
      pk[w] = x.x;
      pc[w] = __int_as_float(x.y);
    }
  };
  auto stage3 = [&](float* dst) {
#pragma unroll
    for (int w = 0; w < NW; ++w) {
      const int e = lane + 32 * w;
      if (e < pn) {
        const float* src = Mx + (size_t)(uint32_t)pk[w] * P;
        const uint32_t d = smem_u32(dst + e * P);
#pragma unroll
        for (int q = 0; q < P / 4; ++q) cp_async16(d + 16 * q, src + 4 * q, keep);
      }
    }
    cp_async_commit();
  };

  // prologue: the first document goes to buffer 0
  stage1(pos);
  stage2();
  stage3(buf0);

  for (; pos < pos1; pos += nwarps) {
    // current document (prefetched)
    const int j = pj, n = pn;
    int ke[NW];
    float ce[NW];
    bool ve[NW];
#pragma unroll
    for (int w = 0; w < NW; ++w) {
      ke[w] = pk[w];
      ce[w] = pc[w];
      ve[w] = lane + 32 * w < n;
    }
    float* Sb = buf0 + cur * S::BUF;          // M rows of this document (row e at Sb + e*P)
    float* Tb = buf0 + (cur ^ 1) * S::BUF;    // transpose scratch, then the next document's rows
    stage1(pos + nwarps);                     // next document's header loads are in flight
    cp_async_wait_all();
    __syncwarp();

    // ---- m_e (stored at M row position LD) to a contiguous vector
    float me[NW];
#pragma unroll
    for (int w = 0; w < NW; ++w) {
      const int e = lane + 32 * w;
      me[w] = ve[w] ? Sb[e * P + LD] : 0.f;
      sm[e] = me[w];
    }
    __syncwarp();

    // ---- column copy: D, mu, Kh (lane i owns column i)
    float kc[CPL][NE];
    bool und[CPL];
    float uh[CPL];
#pragma unroll
    for (int c = 0; c < CPL; ++c) {
      const int col = lane + 32 * c;
      const bool colok = col < LD;  // lanes past LD (CPL*32 > LD) hold a phantom column of 1s
      float mu = FLT_MAX;
#pragma unroll
      for (int e4 = 0; e4 < NEP / 4; ++e4) {
        const float4 m4 = *reinterpret_cast<const float4*>(sm + 4 * e4);
        const float mm[4] = {m4.x, m4.y, m4.z, m4.w};
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          const int e = 4 * e4 + t;
          if (e < NE) {
            float dv = 0.f;
            if (e < n && colok) {
              dv = Sb[e * P + col] - mm[t];
              mu = fminf(mu, dv);
            }
            kc[c][e] = dv;
          }
        }
      }
      const float amu = a * mu;
      uh[c] = real[c] ? (float)v_r * ex2_ftz(-amu) : 0.f;   // uh0 = v_r e^{-lambda mu_i}
      bool u_ = false;
#pragma unroll
      for (int e = 0; e < NE; ++e) {
        float kv = 0.f;
        if (e < n) {
          kv = real[c] ? ex2_ftz(fmaf(-a, kc[c][e], amu)) : 1.f;  // padded columns: 1 (uh = 0)
          u_ |= kv < FLT_MIN;
          if (colok) Tb[e * P + col] = kv;
        }
        kc[c][e] = kv;
      }
      und[c] = u_ && real[c];
    }
    __syncwarp();

    // ---- row copy (lane e owns row e) from the transpose buffer
    float kr[NW][LD];
    bool unde[NW];
#pragma unroll
    for (int w = 0; w < NW; ++w) {
      const int e = lane + 32 * w;
      float mn = 1.f;
#pragma unroll
      for (int q = 0; q < LD / 4; ++q) {
        float4 t = make_float4(1.f, 1.f, 1.f, 1.f);
        if (e < NE) t = *reinterpret_cast<const float4*>(Tb + e * P + 4 * q);
        kr[w][4 * q] = t.x; kr[w][4 * q + 1] = t.y; kr[w][4 * q + 2] = t.z; kr[w][4 * q + 3] = t.w;
        mn = fminf(mn, fminf(fminf(t.x, t.y), fminf(t.z, t.w)));
      }
      unde[w] = ve[w] && mn < FLT_MIN;
    }
    __syncwarp();
    // the transpose buffer is free: the next document's rows go there while this one iterates
    stage2();
    bool staged = false;

    // ---- iterations, then the final step
    float umax_k = (float)v_r * kv_s;   // v_r * max(uh) * 2^-110 (max uh0 <= v_r)
    bool bad = false;
    uint32_t badu = 0u;
    float vt[NW];
    for (int it = 0;; ++it) {
      __syncwarp();
#pragma unroll
      for (int c = 0; c < CPL; ++c) su[lane + 32 * c] = uh[c];
      __syncwarp();
      // SDDMM: s_e = Kh[e,:] . uh,  vh_e = c_e / s_e
      float sp[NW][4];
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
      uint32_t vmax_b = 0u;
#pragma unroll
      for (int w = 0; w < NW; ++w) {
        const float s = (sp[w][0] + sp[w][1]) + (sp[w][2] + sp[w][3]);
        vt[w] = ve[w] ? ce[w] * rcp_fast(s) : 0.f;
        bad |= unde[w] && umax_k > s;
        vmax_b = max(vmax_b, __float_as_uint(vt[w]));
      }
      if (it == iters) break;
      if (it == 1) {  // the next document's entries have landed: start its row copies
        staged = true;
        stage3(Tb);
      }
      // SpMM: acc_i = Kh[:,i] . vh,  uh_i = r_i / acc_i
#pragma unroll
      for (int w = 0; w < NW; ++w) sv[lane + 32 * w] = vt[w];
      vmax_b = __reduce_max_sync(kFull, vmax_b);
      __syncwarp();
      float ap[CPL][4];
#pragma unroll
      for (int c = 0; c < CPL; ++c) ap[c][0] = ap[c][1] = ap[c][2] = ap[c][3] = 0.f;
#pragma unroll
      for (int e4 = 0; e4 < NEP / 4; ++e4) {
        const float4 vv = *reinterpret_cast<const float4*>(sv + 4 * e4);
        const float vq[4] = {vv.x, vv.y, vv.z, vv.w};
#pragma unroll
        for (int c = 0; c < CPL; ++c)
#pragma unroll
          for (int t = 0; t < 4; ++t)
            if (4 * e4 + t < NE) ap[c][t] = fmaf(kc[c][4 * e4 + t], vq[t], ap[c][t]);
      }
      const float vcap = (float)n * __uint_as_float(vmax_b) * kUnder;
      uint32_t umax_b = 0u, umin_b = 0xffffffffu;
      float un[CPL];
#pragma unroll
      for (int c = 0; c < CPL; ++c) {
        const float acc = (ap[c][0] + ap[c][1]) + (ap[c][2] + ap[c][3]);
        un[c] = r[c] * rcp_fast(acc);
        bad |= und[c] && vcap > acc;
        umax_b = max(umax_b, __float_as_uint(un[c]));
        if (real[c]) umin_b = min(umin_b, __float_as_uint(un[c]));
      }
      // gauge: positive floats order like their bit patterns
      umax_b = __reduce_max_sync(kFull, umax_b);
      umin_b = __reduce_min_sync(kFull, umin_b);
      badu |= (umin_b < 0x00800000u) | (umax_b > 0x7f7fffffu);
      const float sc = gauge_scale(umax_b, umin_b);  // exact power of two
#pragma unroll
      for (int c = 0; c < CPL; ++c) uh[c] = un[c] * sc;
      umax_k = __uint_as_float(umax_b) * sc * kv_s;
    }
    if (!staged) stage3(Tb);
    // ---- final step: WMD_j = sum_e vh_e q_e,  q_e = sum_i Kh_ei M_ie uh_i  (su holds uh)
    float wsum = 0.f;
#pragma unroll
    for (int w = 0; w < NW; ++w) {
      const int e = lane + 32 * w;
      if (w > 0 && !__any_sync(kFull, ve[w])) break;
      float q0 = 0.f, q1 = 0.f;
#pragma unroll
      for (int q4 = 0; q4 < LD / 4; ++q4) {
        float4 m4 = make_float4(0.f, 0.f, 0.f, 0.f);
        if (e < NE) m4 = *reinterpret_cast<const float4*>(Sb + e * P + 4 * q4);
        const float4 uu = *reinterpret_cast<const float4*>(su + 4 * q4);
        q0 = fmaf(kr[w][4 * q4] * m4.x, uu.x, q0);
        q1 = fmaf(kr[w][4 * q4 + 1] * m4.y, uu.y, q1);
        q0 = fmaf(kr[w][4 * q4 + 2] * m4.z, uu.z, q0);
        q1 = fmaf(kr[w][4 * q4 + 3] * m4.w, uu.w, q1);
      }
      if (ve[w]) wsum = fmaf(vt[w], q0 + q1, wsum);
    }
#pragma unroll
    for (int off = 16; off; off >>= 1) wsum += __shfl_xor_sync(kFull, wsum, off);
    const bool flag = __any_sync(kFull, bad) || badu || !(fabsf(wsum) <= FLT_MAX);
    if (lane == 0) {
      dist[j] = wsum;
      if (flag) {
        flags[j] |= kFlagFp32Range;
        flagged_list[atomicAdd(flagged_count, 1)] = j;
      }
    }
    cur ^= 1;
  }
  cp_async_wait_all();  // nothing may be in flight when the warp exits
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
                        int64_t p1, const float* Mx, int v_r, const float* rpad, float lambda,
                        int iters, float* dist, uint8_t* flags, int32_t* fl, int32_t* fc,
                        cudaStream_t st) {
  if (p1 <= p0) return;
  constexpr size_t smem = sizeof(float) * Shape<LD, NE>::WARP_FLOATS * kWarps;
  static int resident = 0;
  if (!resident) {
    cudaFuncSetAttribute(sinkhorn_fused_kernel<LD, NE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(sinkhorn_fused_kernel<LD, NE>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, sinkhorn_fused_kernel<LD, NE>, kThreads, smem);
    resident = std::max(1, per_sm) * num_sms();
  }
  const int64_t need = (p1 - p0 + kWarps - 1) / kWarps;
  // persistent warps: a few waves of documents per warp keep the staging pipeline busy
  const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>(need, resident));
  sinkhorn_fused_kernel<LD, NE><<<grid, kThreads, smem, st>>>(order, doc_ptr, ent, p0, p1, Mx, v_r, rpad,
                                                               lambda, iters, dist, flags, fl, fc);
}

// Length buckets of the fused kernel over the length-sorted order. A bucket with NE > 32 keeps
// two row slots per lane; supported pairs keep the block within ~136 registers per lane.
constexpr int kBuckets[] = {16, 24, 32, 40, 48, 64};
constexpr int kNumBuckets = 6;

constexpr bool fits(int ld, int ne) {
  return ((ne + 31) / 32) * ld + ((ld + 31) / 32) * ne <= 136;
}

template <int LD>
void dispatch_ne(int ne, const int32_t* order, const int32_t* doc_ptr, const Entry* ent, int64_t p0,
                 int64_t p1, const float* Mx, int v_r, const float* rpad, float lambda, int iters,
                 float* dist, uint8_t* flags, int32_t* fl, int32_t* fc, cudaStream_t st) {
#define F_(NE) \
  if constexpr (fits(LD, NE)) launch_fused_range<LD, NE>(order, doc_ptr, ent, p0, p1, Mx, v_r, rpad, lambda, iters, dist, flags, fl, fc, st)
  switch (ne) {
    case 16: F_(16); break;
    case 24: F_(24); break;
    case 32: F_(32); break;
    case 40: F_(40); break;
    case 48: F_(48); break;
    default: F_(64); break;
  }
#undef F_
}

}  // namespace

bool fused_supported(int ld, int64_t max_doc_nnz) {
  if (ld > 64 || max_doc_nnz > 64) return false;
  for (int b = 0; b < kNumBuckets; ++b)
    if (kBuckets[b] >= max_doc_nnz) return fits(ld, kBuckets[b]);
  return false;
}

void launch_sinkhorn_fused(const int32_t* order, const int32_t* doc_ptr, const Entry* ent, int64_t N,
                           const int64_t* len_prefix, int64_t max_len, const float* Mx, int ld,
                           int v_r, const float* rpad, float lambda, int iters, float* dist,
                           uint8_t* flags, int32_t* flagged_list, int32_t* flagged_count,
                           cudaStream_t st) {
  // len_prefix[L] = number of documents with fewer than L nonzeros: the length-sorted order
  // splits into buckets of at most 16 / 24 / 32 / 40 / 48 / 64 nonzeros, one launch each.
  int64_t p0 = 0;
  for (int bi = 0; bi < kNumBuckets && p0 < N; ++bi) {
    const int NE = kBuckets[bi];
    const int64_t p1 = NE >= max_len ? N : len_prefix[NE + 1];
    if (p1 > p0) {
      switch (ld) {
#define L_(LD) case LD: dispatch_ne<LD>(NE, order, doc_ptr, ent, p0, p1, Mx, v_r, rpad, lambda, iters, dist, flags, flagged_list, flagged_count, st); break;
        L_(8) L_(16) L_(24) L_(32) L_(40) L_(48) L_(56) L_(64)
#undef L_
        default: break;
      }
    }
    p0 = p1;
  }
}

int fused_launch_count(const int64_t* len_prefix, int64_t max_len, int64_t N) {
  int64_t p0 = 0;
  int cnt = 0;
  for (int bi = 0; bi < kNumBuckets && p0 < N; ++bi) {
    const int64_t p1 = kBuckets[bi] >= max_len ? N : len_prefix[kBuckets[bi] + 1];
    cnt += p1 > p0;
    p0 = p1;
  }
  return cnt;
}

}  // namespace wmd
