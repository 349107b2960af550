// EXPERIMENT, NOT BUILT (kept for the record, DESIGN.md §6 "What did not help"): measured
// slower than the one-warp kernel's 16-row bucket (Scaling fused phase 8.82 -> 9.04 ms).
// wmd_fused_pair.cu — NEXT-1 for short documents: all Sinkhorn iterations and the final step of
// TWO documents of up to 16 words per warp, one per half-warp, the blocks in registers.
//
// Same method and numerics as the one-warp kernel (wmd_fused.cu: doc-local two-sided rescale
// Kh = 2^(-alpha (D - mu)), power-of-two gauge per document, FP32 range certificate, final step
// with D recovered from Kh). The one-warp kernel spends a fixed per-iteration overhead (the
// transpose-reduces, reciprocals, gauge and checks) on a 16-row block as on a 32-row one; here
// a half-warp holds a 16-row document as a 4 x 4 lane tile, lane = 16 d + 4 a + b:
//   rows    4a + (s ^ b), s < 4            (transpose-reduce over the b-lanes: lane xor 1, 2)
//   columns CW2 = LD / 4 per lane: Q quads 16g + 4b + (t ^ a) and R plain columns 16Q + Rb + r
//                                          (transpose-reduce over the a-lanes: lane xor 4, 8)
// so the two documents of a warp share every instruction and no shuffle crosses the halves
// (xor 16 is never used). Per iteration and lane: 4 x CW2 FFMA twice for two documents.
// Bound: FP32 issue.
#include <algorithm>
#include <cfloat>
#include <cstdint>

#include "wmd_tile.cuh"

namespace wmd {
namespace {

using namespace dev;
using namespace tile;

constexpr int kPairWarps = 4;              // warps per block
constexpr float kUnderP = 0x1p-110f;       // 2^-126 / 2^-16
constexpr float kLog2eP = 1.4426950408889634f;
constexpr int kPairRows = 16;              // rows (words) per document
#ifndef WMD_PAIR_MINB
#define WMD_PAIR_MINB 4
#endif

template <int CW2>
struct PCols {
  static constexpr int Q = CW2 / 4, R = CW2 % 4;
  static constexpr int LD = 4 * CW2;
};

// natural-order column of slot c of lane (., b) / column of register slot c of lane (a, b)
template <int CW2>
__device__ __forceinline__ int pnat_col(int c, int b) {
  constexpr int Q = PCols<CW2>::Q, R = PCols<CW2>::R;
  return c < 4 * Q ? 16 * (c >> 2) + 4 * b + (c & 3) : 16 * Q + R * b + (c - 4 * Q);
}
template <int CW2>
__device__ __forceinline__ int pcol_of(int c, int a, int b) {
  constexpr int Q = PCols<CW2>::Q, R = PCols<CW2>::R;
  return c < 4 * Q ? 16 * (c >> 2) + 4 * b + ((c & 3) ^ a) : 16 * Q + R * b + (c - 4 * Q);
}
template <int CW2>
__device__ __forceinline__ void pload_cols(const float* row, int b, float (&x)[CW2]) {
  constexpr int Q = PCols<CW2>::Q, R = PCols<CW2>::R;
#pragma unroll
  for (int q = 0; q < Q; ++q) {
    const float4 t = *reinterpret_cast<const float4*>(row + 16 * q + 4 * b);
    x[4 * q] = t.x; x[4 * q + 1] = t.y; x[4 * q + 2] = t.z; x[4 * q + 3] = t.w;
  }
#pragma unroll
  for (int r = 0; r < R; ++r) x[4 * Q + r] = row[16 * Q + R * b + r];
}
// row partials of the 4 slots -> p[0] = sum of row 4a + b
__device__ __forceinline__ void preduce_rows(float (&q)[4]) {
  q[0] += shx(q[2], 2); q[1] += shx(q[3], 2);
  q[0] += shx(q[1], 1);
}
// column partials -> q[4g] = sum of column 16g + 4b + a, q[4Q + r] = sum of plain column r
template <int CW2>
__device__ __forceinline__ void preduce_cols(float (&q)[CW2]) {
  constexpr int Q = PCols<CW2>::Q, R = PCols<CW2>::R;
#pragma unroll
  for (int g = 0; g < Q; ++g) {
    float* y = q + 4 * g;
    y[0] += shx(y[2], 8); y[1] += shx(y[3], 8);
    y[0] += shx(y[1], 4);
  }
#pragma unroll
  for (int r = 0; r < R; ++r) {
    q[4 * Q + r] += shx(q[4 * Q + r], 8);
    q[4 * Q + r] += shx(q[4 * Q + r], 4);
  }
}

template <int CW2>
__global__ void __launch_bounds__(32 * kPairWarps, WMD_PAIR_MINB) sinkhorn_pair_kernel(
    const int4* __restrict__ sdoc, const Entry* __restrict__ ent, int64_t pos0, int64_t pos1,
    const float* __restrict__ Mx, int v_r, const float* __restrict__ rpad, float lambda, int iters,
    int32_t* __restrict__ iters_doc, float* __restrict__ dist, uint8_t* __restrict__ flags,
    int32_t* __restrict__ flagged_list, int32_t* __restrict__ flagged_count) {
  constexpr int Q = PCols<CW2>::Q, R = PCols<CW2>::R, LD = PCols<CW2>::LD, P = LD + 4, RW = 4;
  constexpr int NCO = Q + R;  // own columns after the column reduce
  constexpr int BUF = kPairRows * P;
  static_assert(Q >= 1, "at least one column quad per lane");
  extern __shared__ __align__(16) float psm[];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int d = lane >> 4, a = (lane >> 2) & 3, b = lane & 3, e_own = lane & 15;
  const unsigned hm = 0xFFFFu << (16 * d);  // this document's half of the warp
  float* buf = psm + (wib * 2 + d) * BUF;    // the staged M rows of this half's document
  const int64_t stride = (int64_t)gridDim.x * kPairWarps * 2;
  const uint64_t keep = l2_evict_last_policy();
  const int2* ent2 = reinterpret_cast<const int2*>(ent);
  const float alpha = lambda * kLog2eP;
  const float kv_s = (float)v_r * kUnderP;
  float r_own[NCO];
  bool oreal[NCO];
#pragma unroll
  for (int g = 0; g < NCO; ++g) {
    const int oc = g < Q ? 16 * g + 4 * b + a : 16 * Q + R * b + (g - Q);
    r_own[g] = __ldg(rpad + oc);
    oreal[g] = oc < v_r;
  }
  bool nreal[CW2];
#pragma unroll
  for (int c = 0; c < CW2; ++c) nreal[c] = pnat_col<CW2>(c, b) < v_r;

  // ---- prefetch (per half): header, this lane's entry (row e_own), cp.async of that row
  int64_t pos = pos0 + ((int64_t)blockIdx.x * kPairWarps + wib) * 2;
  int pj = -1, pb = 0, pn = 0, pk = 0;
  float pc = 0.f;
  auto stage1 = [&](int64_t p) {
    pj = -1; pn = 0; pb = 0;
    if (p + d < pos1) {
      const int4 x = ldg_guarded(sdoc + p + d);
      pj = x.x; pb = x.y; pn = x.z;
    }
  };
  auto stage2 = [&]() {
    int2 x = make_int2(0, 0);
    if (e_own < pn) x = ldg_guarded(ent2 + pb + e_own);
    pk = x.x;
    pc = __int_as_float(x.y);
  };
  auto stage3 = [&]() {
    if (e_own < pn) {
      uint32_t k;
      asm volatile("mov.b32 %0, %1;" : "=r"(k) : "r"(pk));
      const float* src = Mx + (size_t)k * P;
      const uint32_t dst = smem_u32(buf + e_own * P);
#pragma unroll
      for (int q = 0; q < P / 4; ++q) cp_async16(dst + 16 * q, src + 4 * q, keep);
    }
    cp_async_commit();
  };
  stage1(pos);
  stage2();
  stage3();

  for (; pos < pos1; pos += stride) {
    const int j = pj, n = pn;
    const float c_own = pc;
    const bool v_ok = e_own < n;  // the lane's own row after the row reduce is 4a + b = e_own
    stage1(pos + stride);
    cp_async_wait_all();
    __syncwarp();

    // ---- block tile: D = M - m, mu = column minima over the document, Kh = 2^(-alpha (D - mu))
    float K[RW][CW2], u[CW2], mu_s[CW2];
    bool flushed = false;
    {
      float mu[CW2];
#pragma unroll
      for (int c = 0; c < CW2; ++c) mu[c] = FLT_MAX;
#pragma unroll
      for (int s = 0; s < RW; ++s) {
        const int e = 4 * a + (s ^ b);
        const bool ok = e < n;
        const float* row = buf + (ok ? e : 0) * P;
        float x[CW2];
        pload_cols<CW2>(row, b, x);
        const float me = row[LD];
#pragma unroll
        for (int c = 0; c < CW2; ++c) {
          K[s][c] = ok ? x[c] - me : FLT_MAX;
          mu[c] = fminf(mu[c], K[s][c]);
        }
      }
#pragma unroll
      for (int c = 0; c < CW2; ++c) {  // over the 4 a-lanes of this half
        mu[c] = fminf(mu[c], shx(mu[c], 4));
        mu[c] = fminf(mu[c], shx(mu[c], 8));
      }
#pragma unroll
      for (int s = 0; s < RW; ++s) {
#pragma unroll
        for (int c = 0; c < CW2; ++c) {
          const float dd = K[s][c];
          const float kx = ex2_ftz(fmaf(-alpha, dd, alpha * mu[c]));
          flushed |= nreal[c] && kx < FLT_MIN && dd != FLT_MAX;
          K[s][c] = nreal[c] ? kx : (dd != FLT_MAX ? 1.f : 0.f);  // padded columns: 1 on real rows
        }
        to_slots<CW2>(K[s], a);
      }
#pragma unroll
      for (int c = 0; c < CW2; ++c) {
        mu_s[c] = mu[c];
        u[c] = nreal[c] ? (float)v_r * ex2_ftz(-alpha * mu[c]) : 0.f;  // uh0 (x0 = 1/v_r)
      }
      to_slots<CW2>(mu_s, a);
      to_slots<CW2>(u, a);
    }
    const bool und = (__ballot_sync(kFull, flushed) & hm) != 0u;
    const float m_own = v_ok ? buf[e_own * P + LD] : 0.f;
    __syncwarp();  // the staged rows are consumed: the buffers take the next documents
    stage2();
    bool staged = false;

    float umax_k = (float)v_r * kv_s;  // v_r * max(uh) * 2^-110 (max uh0 <= v_r)
    bool bad = false, badu = false;
    float v_own = 0.f, s_own = 0.f;
    int it = 0;
    for (;; ++it) {
      // SDDMM
      float p[RW];
#pragma unroll
      for (int s = 0; s < RW; ++s) {
        float acc = K[s][0] * u[0];
#pragma unroll
        for (int c = 1; c < CW2; ++c) acc = fmaf(K[s][c], u[c], acc);
        p[s] = acc;
      }
      preduce_rows(p);
      s_own = p[0];
      v_own = v_ok ? c_own * rcp_fast(s_own) : 0.f;
      bad |= v_ok && und && umax_k > s_own;
      if (it == iters) break;
      if (it == 1) {
        staged = true;
        stage3();
      }
      // (the max over both documents of the warp: a conservative bound for each)
      const uint32_t vmax_b = __reduce_max_sync(kFull, __float_as_uint(v_own));
      float vs[RW];
      vs[0] = v_own;
#pragma unroll
      for (int t = 1; t < RW; ++t) vs[t] = shx(v_own, t);
      // SpMM
      float q[CW2];
#pragma unroll
      for (int c = 0; c < CW2; ++c) {
        float q0 = K[0][c] * vs[0];
#pragma unroll
        for (int s = 1; s < RW; ++s) q0 = fmaf(K[s][c], vs[s], q0);
        q[c] = q0;
      }
      preduce_cols<CW2>(q);
      const float vcap = (float)n * __uint_as_float(vmax_b) * kUnderP;
      uint32_t umax_b = 0u;
      float uo[NCO];
#pragma unroll
      for (int g = 0; g < NCO; ++g) {
        const float acc = q[g < Q ? 4 * g : 4 * Q + (g - Q)];
        uo[g] = r_own[g] * rcp_fast(acc);
        bad |= und && vcap > acc;
        umax_b = max(umax_b, __float_as_uint(uo[g]));
      }
      // gauge of this document: max uh -> [1, 2) by an exact power of two
      umax_b = __reduce_max_sync(hm, umax_b);
      badu |= umax_b > 0x7f7fffffu;
      const float sc = __uint_as_float((254u - min(umax_b >> 23, 253u)) << 23);
      umax_k = 2.f * kv_s;
#pragma unroll
      for (int g = 0; g < NCO; ++g) {
        uo[g] *= sc;
        bad |= oreal[g] && !(uo[g] >= FLT_MIN);
      }
      // slot 4g + t holds column 16g + 4b + (t ^ a), owned by lane ^ 4t
#pragma unroll
      for (int g = 0; g < Q; ++g) {
        u[4 * g] = uo[g];
#pragma unroll
        for (int t = 1; t < 4; ++t) u[4 * g + t] = shx(uo[g], 4 * t);
      }
#pragma unroll
      for (int r = 0; r < R; ++r) u[4 * Q + r] = uo[Q + r];
    }
    if (!staged) stage3();
    // ---- final step, M recovered from Kh as in wmd_fused.cu
    const float ia = -rcp_fast(alpha);
    float p[RW];
#pragma unroll
    for (int s = 0; s < RW; ++s) {
      float acc = 0.f;
#pragma unroll
      for (int c = 0; c < CW2; ++c) {
        const float k = K[s][c];
        const float kl = k > 0.f ? k * lg2_approx(k) : 0.f;
        acc = fmaf(fmaf(kl, ia, k * mu_s[c]), u[c], acc);
      }
      p[s] = acc;
    }
    preduce_rows(p);
    float wsum = v_ok ? v_own * fmaf(m_own, s_own, p[0]) : 0.f;
#pragma unroll
    for (int off = 8; off; off >>= 1) wsum += shx(wsum, off);  // within the half
    const bool flag = (__ballot_sync(kFull, bad) & hm) != 0u || badu || !(fabsf(wsum) <= FLT_MAX);
    if (e_own == 0 && j >= 0) {
      dist[j] = wsum;
      if (iters_doc) iters_doc[j] = it;
      if (flag) {
        flags[j] |= kFlagFp32Range;
        flagged_list[atomicAdd(flagged_count, 1)] = j;
      }
    }
  }
  cp_async_wait_all();
}

int num_sms_pair() {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
  }
  return sms;
}

template <int CW2>
void launch_pair_range(const int4* sdoc, const Entry* ent, int64_t p0, int64_t p1, const float* Mx, int v_r,
                       const float* rpad, float lambda, int iters, int32_t* itd, float* dist, uint8_t* flags,
                       int32_t* fl, int32_t* fc, cudaStream_t st) {
  if (p1 <= p0) return;
  constexpr size_t smem = sizeof(float) * kPairRows * (PCols<CW2>::LD + 4) * 2 * kPairWarps;
  static int resident = 0;
  if (!resident) {
    cudaFuncSetAttribute(sinkhorn_pair_kernel<CW2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, sinkhorn_pair_kernel<CW2>, 32 * kPairWarps, smem);
    resident = std::max(1, per_sm) * num_sms_pair();
  }
  const int64_t need = (p1 - p0 + 2 * kPairWarps - 1) / (2 * kPairWarps);
  const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>(need, resident));
  sinkhorn_pair_kernel<CW2><<<grid, 32 * kPairWarps, smem, st>>>(sdoc, ent, p0, p1, Mx, v_r, rpad, lambda, iters,
                                                                 itd, dist, flags, fl, fc);
}

}  // namespace

#ifndef WMD_PAIR_KERNEL
#define WMD_PAIR_KERNEL 1
#endif

bool pair_supported(int ld) { return WMD_PAIR_KERNEL && (ld == 24 || ld == 32 || ld == 40 || ld == 48); }

void launch_sinkhorn_pair(const int4* sdoc, const Entry* ent, int64_t p0, int64_t p1, const float* Mx, int ld,
                          int v_r, const float* rpad, float lambda, int iters, int32_t* iters_doc, float* dist,
                          uint8_t* flags, int32_t* flagged_list, int32_t* flagged_count, cudaStream_t st) {
  switch (ld) {
#define P_(LDV) case LDV: launch_pair_range<LDV / 4>(sdoc, ent, p0, p1, Mx, v_r, rpad, lambda, iters, iters_doc, dist, flags, flagged_list, flagged_count, st); break;
    P_(24) P_(32) P_(40) P_(48)
#undef P_
    default: break;
  }
}

}  // namespace wmd
