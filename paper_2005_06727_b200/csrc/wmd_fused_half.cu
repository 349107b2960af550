// wmd_fused_half.cu — NEXT-1 for short documents: the one-warp fused kernel's
// algorithm (wmd_fused.cu: all Sinkhorn iterations and the final step of a document in one
// launch, doc-local two-sided rescale, FP32 range certificate) with HALF a warp per
// document (each 16-lane half-warp solves its own (document, query) item) and, unlike it, no
// per-iteration gauge of uh (R39).
//
// Why: the one-warp kernel is bound by its warp shuffles (one SHFL per SM-cycle against ~3.5
// FFMA, profiles/r01_issue_bench.jsonl; L1/TEX pipe 60-71 % busy, r02_full_scaling_fused_
// summary.txt). A reduce-scatter + all-gather of S register slots over P lanes costs
// 2 S (P - 1) / P shuffles, so per iteration a lane of the one-warp layout (8 b-lanes x 4 a-lanes,
// RW x CW = 8 x 4 tile) issues 20 shuffles for 64 FFMA; here (4 b-lanes x 4 a-lanes per
// document, RW x CW = 8 x 8 tile) a lane issues 24 shuffles for 128 FFMA, and every shuffle
// instruction serves two documents: 12 shuffle issues per document-iteration instead of 20.
//
// Mapping: lane = 16 h + 4 a + b (h: the half-warp's item, a: row group, b: column group).
// Row slots: full 16-row tiles T, slot 4T + t holds row 16T + 4a + (t ^ b); a tail tile (TW = 2)
// slot 4NT + t holds row 16NT + 2a + (t ^ (b >> 1)); (TW = 1) slot 4NT holds row 16NT + a. Column slots: CW = 4Q + R per lane,
// LD = 4 CW in {16, 24, 32, 40}: quads g, slot 4g + t holds column 16g + 4b + (t ^ a), then R = 0
// or 2 plain columns 16Q + Rb + r (the same in the four a-lanes, reduced by a butterfly).
//
// Final step without M: the staging buffer is reused for the next item as soon as the block is
// built (one buffer per half-warp, so four blocks fit per SM), so the final step recovers the
// distance from the block: with Kh_ei = 2^(-alpha (D_ei - mu_i)) and M_ie = D_ei + m_e,
//     sum_i Kh_ei uh_i M_ie = sum_i Kh_ei uh_i (mu_i - log2(Kh_ei) / alpha) + m_e s_e
// (s_e = sum_i Kh_ei uh_i), and vh_e s_e = c_e after the last row step, so
//     WMD_j = sum_e vh_e sum_i Kh_ei uh_i (mu_i - log2(Kh_ei) / alpha) + sum_e c_e m_e.
// Every term is non-negative (no cancellation); log2 of an ex2 result returns its argument to
// ~2^-22 relative, so M is recovered to ~3e-7 relative for lambda >= kFusedMinLambda (R35, R37).
// Flushed entries (Kh = 0) contribute 0.
#include <algorithm>
#include <cfloat>
#include <cstdint>
#include <type_traits>

#include "wmd_tile.cuh"

namespace wmd {
namespace {

using namespace dev;
using namespace tile;

constexpr int kWarps = 4;
constexpr int kThreads = 32 * kWarps;
#ifndef WMD_HALF_TWO_BUF   // 1: two staging buffers per half-warp, the final step reads M back
#define WMD_HALF_TWO_BUF 0
#endif
constexpr int kBufs = WMD_HALF_TWO_BUF ? 2 : 1;
constexpr float kUnder = 0x1p-110f;        // 2^-126 / 2^-16
constexpr float kLog2e = 1.4426950408889634f;

template <int CW, int NT, int TW>
struct HShape {
  static_assert((CW % 4 == 0 || CW % 4 == 2) && TW >= 0 && TW <= 2, "quads + 0 or 2 plain columns; 0-2-row tail");
  static constexpr int LD = 4 * CW;
  static constexpr int Q = CW / 4;               // column quads per lane
  static constexpr int R = CW % 4;               // plain columns per lane
  static constexpr int NCO = Q + R;              // own columns per lane after the column reduce
  static constexpr int RW = 4 * NT + TW;         // row slots per lane
  static constexpr int NE = 16 * NT + 4 * TW;    // document rows covered
  static constexpr int NW = (NE + 15) / 16;      // entry slots per lane
  static constexpr int NOWN = NT + (TW ? 1 : 0); // own rows per lane after the row reduce
  static constexpr int P = LD + 4;               // row pitch (floats) of Mx and the staging buffer
  static constexpr int BUF = NE * P;
  static constexpr int REGS = RW * CW;
};

template <int CW, int NT, int TW>
constexpr int hmin_blocks() {
  using S = HShape<CW, NT, TW>;
#ifndef WMD_HALF_REGS
#define WMD_HALF_REGS 24
#endif
  constexpr int regs = ((S::REGS + 3 * S::RW + 3 * CW + WMD_HALF_REGS) + 7) / 8 * 8;
  constexpr int b = 65536 / (kThreads * regs);
  return b < 1 ? 1 : (b > 8 ? 8 : b);
}

template <int NT, int TW>
__device__ __forceinline__ int hrow_of(int s, int a, int b) {
  if (s < 4 * NT) return 16 * (s >> 2) + 4 * a + ((s & 3) ^ b);
  if constexpr (TW == 1) return 16 * NT + a;   // one tail row per row group, in all four b-lanes
  return 16 * NT + 2 * a + ((s - 4 * NT) ^ (b >> 1));
}
// natural-order column of slot c (the order hload_cols delivers)
template <int CW>
__device__ __forceinline__ int hnat_col(int c, int b) {
  constexpr int Q = CW / 4, R = CW % 4;
  return c < 4 * Q ? 16 * (c >> 2) + 4 * b + (c & 3) : 16 * Q + R * b + (c - 4 * Q);
}

template <int CW>
__device__ __forceinline__ void hload_cols(const float* row, int b, float (&x)[CW]) {
  constexpr int Q = CW / 4, R = CW % 4;
#pragma unroll
  for (int g = 0; g < Q; ++g) {
    const float4 t = *reinterpret_cast<const float4*>(row + 16 * g + 4 * b);
    x[4 * g] = t.x; x[4 * g + 1] = t.y; x[4 * g + 2] = t.z; x[4 * g + 3] = t.w;
  }
  if constexpr (R == 2) {
    const float2 t = *reinterpret_cast<const float2*>(row + 16 * Q + 2 * b);
    x[4 * Q] = t.x; x[4 * Q + 1] = t.y;
  }
}

// reduce-scatter of the row partials over the 4 b-lanes (xor 2, 1): p[4T] = row 16T + 4a + b,
// p[4NT] = tail row 16NT + 2a + (b >> 1)
template <int NT, int TW>
__device__ __forceinline__ void hreduce_rows(float* p) {
#pragma unroll
  for (int T = 0; T < NT; ++T) {
    float* q = p + 4 * T;
    q[0] += shx(q[2], 2); q[1] += shx(q[3], 2);
    q[0] += shx(q[1], 1);
  }
  if constexpr (TW == 2) {
    float* q = p + 4 * NT;
    q[0] += shx(q[1], 2);
    q[0] += shx(q[0], 1);
  } else if constexpr (TW == 1) {   // butterfly: every b-lane gets row 16NT + a
    float* q = p + 4 * NT;
    q[0] += shx(q[0], 2);
    q[0] += shx(q[0], 1);
  }
}

// reduce-scatter of the column partials over the 4 a-lanes (xor 8, 4): q[4g] = column 16g + 4b + a;
// plain columns by a butterfly (every a-lane gets the sum)
template <int CW>
__device__ __forceinline__ void hreduce_cols(float* q) {
  constexpr int Q = CW / 4, R = CW % 4;
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

// max over the lanes of each half-warp (two warp reductions, one per half)
__device__ __forceinline__ uint32_t half_max(uint32_t x, int h) {
  const uint32_t m0 = __reduce_max_sync(kFull, h ? 0u : x);
  const uint32_t m1 = __reduce_max_sync(kFull, h ? x : 0u);
  return h ? m1 : m0;
}
__device__ __forceinline__ bool half_any(bool x, int h) {
  return ((__ballot_sync(kFull, x) >> (16 * h)) & 0xffffu) != 0u;
}

template <int CW, int NT, int TW>
__global__ void __launch_bounds__(kThreads, hmin_blocks<CW, NT, TW>()) sinkhorn_half_kernel(
    const int4* __restrict__ sdoc, const Entry* __restrict__ ent, int64_t pos0, int64_t pos1,
    QuerySet qs, float lambda, int iters) {
  using S = HShape<CW, NT, TW>;
  constexpr int LD = S::LD, RW = S::RW, NW = S::NW, P = S::P, Q = S::Q, R = S::R, NCO = S::NCO, NOWN = S::NOWN;
  extern __shared__ __align__(16) float smem[];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int h = lane >> 4, l16 = lane & 15;
  const int a = l16 >> 2, b = l16 & 3;
  float* const buf0 = smem + (2 * wib + h) * kBufs * S::BUF;   // this half-warp's staging buffer(s)
  int cur = 0;                                                  // the current item's buffer
  const int64_t stride = (int64_t)gridDim.x * kWarps * 2;
  const uint64_t keep = l2_evict_last_policy();
  const uint64_t stream_pol = l2_evict_first_policy();
  const int2* ent2 = reinterpret_cast<const int2*>(ent);
  const float alpha = lambda * kLog2e;
  const float inv_alpha = 1.f / alpha;
  const int nq = qs.nq;

  int v_r = 0;
  float kv_s = 0.f;
  float r_own[NCO];
  bool oreal[NCO], nreal[CW];
  int64_t out0 = 0;
  auto set_query = [&](int q) {
    const int g = qs.qmap ? __ldg(qs.qmap + q) : q;
    out0 = (int64_t)g * qs.N;
    v_r = qs.vr ? __ldg(qs.vr + g) : qs.v_r;
    kv_s = (float)v_r * kUnder;
    const float* rp = qs.rpad + (size_t)g * WMD_MAX_VR_DEV;
#pragma unroll
    for (int gq = 0; gq < NCO; ++gq) {
      const int oc = gq < Q ? 16 * gq + 4 * b + a : 16 * Q + R * b + (gq - Q);
      r_own[gq] = __ldg(rp + oc);
      oreal[gq] = oc < v_r;
    }
#pragma unroll
    for (int c = 0; c < CW; ++c) nreal[c] = hnat_col<CW>(c, b) < v_r;
  };

  int64_t pos = pos0 + ((int64_t)blockIdx.x * kWarps + wib) * 2 + h;
  int pj = -1, pb = 0, pn = 0;
  int pk[NW];
  float pc[NW];
  int cj, cn;
  int ck[NW];
  float cc[NW];
  auto stage1 = [&](int64_t p) {
    pj = -1; pn = 0; pb = 0;
    if (p < pos1) {
      const int4 x = ldg_guarded(sdoc + p);
      pj = x.x; pb = x.y; pn = x.z;
    }
  };
  auto stage2 = [&]() {
#pragma unroll
    for (int w = 0; w < NW; ++w) {
      const int e = l16 + 16 * w;
      int2 x = make_int2(0, 0);
      if (e < pn) x = ldg_guarded_stream(ent2 + pb + e, stream_pol);
      pk[w] = x.x;
      pc[w] = __int_as_float(x.y);
    }
  };
  auto stage3 = [&](const int (&ids)[NW], int nrows, int q) {
    const float* tab = qs.Mx + (size_t)q * qs.mx_stride;
#pragma unroll
    for (int w = 0; w < NW; ++w) {
      const int e = l16 + 16 * w;
      if (e < nrows) {
        uint32_t k;
        asm volatile("mov.b32 %0, %1;" : "=r"(k) : "r"(ids[w]));
        const float* src = tab + (size_t)k * P;
        const uint32_t dst = smem_u32(buf0 + (kBufs == 2 ? (cur ^ 1) : 0) * S::BUF + e * P);
#pragma unroll
        for (int x = 0; x < P / 4; ++x) cp_async16(dst + 16 * x, src + 4 * x, keep);
      }
    }
    cp_async_commit();
  };
  auto take_next_doc = [&]() {
    cj = pj; cn = pn;
#pragma unroll
    for (int w = 0; w < NW; ++w) { ck[w] = pk[w]; cc[w] = pc[w]; }
  };

  cur = kBufs == 2 ? 1 : 0;   // the first item's rows go to buffer cur ^ 1, flipped below
  stage1(pos);
  stage2();
  stage3(pk, pn, 0);
  take_next_doc();
  int q = 0;

  while (__any_sync(kFull, pos < pos1)) {   // a half-warp past the end runs an empty item
    const int j = cj, n = cn;
    if constexpr (kBufs == 2) cur ^= 1;
    const float* const buf = buf0 + cur * S::BUF;
    set_query(q);
    // c and m of the lane's own rows: row 16T + l16 (full tiles), tail row 16NT + 2a + (b >> 1)
    float c_own[NOWN], m_own[NOWN];
    bool v_ok[NOWN];
#pragma unroll
    for (int T = 0; T < NT; ++T) {
      c_own[T] = cc[T];
      v_ok[T] = 16 * T + l16 < n;
    }
    if constexpr (TW > 0) {
      const int tr = TW == 1 ? a : 2 * a + (b >> 1);
      c_own[NT] = __shfl_sync(kFull, cc[NT], 16 * h + tr);
      v_ok[NT] = 16 * NT + tr < n;
    }
    if (q == 0) stage1(pos + stride);
    cp_async_wait_all();
    __syncwarp();

    // ---- block tile: D = M - m, mu = column minima over the document, Kh = 2^(-alpha (D - mu))
    float K[RW][CW];
    float u[CW], mu_s[CW];
    bool und_mine;
    {
#pragma unroll
      for (int T = 0; T < NOWN; ++T) {
        const int e = T < NT ? 16 * T + l16 : 16 * NT + (TW == 1 ? a : 2 * a + (b >> 1));
        m_own[T] = v_ok[T] ? buf[e * P + LD] : 0.f;
      }
      float mu[CW];
#pragma unroll
      for (int c = 0; c < CW; ++c) mu[c] = INFINITY;
      bool rok[RW];
#pragma unroll
      for (int s = 0; s < RW; ++s) {
        const int e = hrow_of<NT, TW>(s, a, b);
        rok[s] = e < n;
        const float* row = buf + (rok[s] ? e : 0) * P;
        float x[CW];
        hload_cols<CW>(row, b, x);
        const float bias = rok[s] ? -row[LD] : INFINITY;
#pragma unroll
        for (int c = 0; c < CW; ++c) {
          K[s][c] = x[c] + bias;
          mu[c] = fminf(mu[c], K[s][c]);
        }
      }
#pragma unroll
      for (int c = 0; c < CW; ++c) {  // column minima over the 4 a-lanes
        mu[c] = fminf(mu[c], shx(mu[c], 4));
        mu[c] = fminf(mu[c], shx(mu[c], 8));
      }
      float amu[CW], kmin[CW];
#pragma unroll
      for (int c = 0; c < CW; ++c) {
        amu[c] = alpha * mu[c];
        kmin[c] = 1.f;
      }
#pragma unroll
      for (int s = 0; s < RW; ++s) {
#pragma unroll
        for (int c = 0; c < CW; ++c) {
          K[s][c] = rok[s] ? ex2_ftz(fmaf(-alpha, K[s][c], amu[c])) : 1.f;
          kmin[c] = fminf(kmin[c], K[s][c]);
        }
        to_slots<CW>(K[s], a);
      }
      bool flushed = false;
#pragma unroll
      for (int c = 0; c < CW; ++c) flushed |= nreal[c] && kmin[c] < FLT_MIN;
      und_mine = half_any(flushed, h);
#pragma unroll
      for (int c = 0; c < CW; ++c) {
        u[c] = nreal[c] ? (float)v_r * ex2_ftz(-alpha * mu[c]) : 0.f;
        mu_s[c] = nreal[c] ? mu[c] : 0.f;   // padded columns: uh = 0 there
      }
      to_slots<CW>(u, a);
      to_slots<CW>(mu_s, a);
    }
    __syncwarp();   // every lane of the half is done with the staged rows: the buffer is free
    const bool und = __any_sync(kFull, und_mine);
    if (q == nq - 1) stage2();
    auto stage3_next = [&]() {
      if (q + 1 < nq) stage3(ck, n, q + 1);
      else stage3(pk, pn, 0);
    };

    // ---- iterations
    float v_own[NOWN];
    bool bad = false;
    float umin = FLT_MAX;
    uint32_t umax_all = 0u;
    float vlo = FLT_MAX, vhi = 0.f;   // range of the real v over all row steps (UND blocks)
    int it = 0;
    auto iterate = [&](auto und_tag) {
      constexpr bool UND = decltype(und_tag)::value;
      // FIRST: the first row step, the only one that checks s_e directly (uh0 is outside the
      // running range of the column steps' uh)
      auto row_step = [&](auto first_tag) {
        constexpr bool FIRST = decltype(first_tag)::value;
        // rows in pairs (s, s + 1), one FFMA2 per column with uh broadcast
        float p[RW];
#pragma unroll
        for (int s = 0; s + 1 < RW; s += 2) {
          float a0, a1;
          fmul2(a0, a1, K[s][0], K[s + 1][0], u[0], u[0]);
#pragma unroll
          for (int c = 1; c < CW; ++c) ffma2(a0, a1, K[s][c], K[s + 1][c], u[c], u[c], a0, a1);
          p[s] = a0;
          p[s + 1] = a1;
        }
        if constexpr (RW & 1) {
          float acc = K[RW - 1][0] * u[0];
#pragma unroll
          for (int c = 1; c < CW; ++c) acc = fmaf(K[RW - 1][c], u[c], acc);
          p[RW - 1] = acc;
        }
        hreduce_rows<NT, TW>(p);
#pragma unroll
        for (int o = 0; o < NOWN; ++o) {
          const float sv = p[4 * o];
          v_own[o] = c_own[o] * rcp_fast(sv);
          if constexpr (UND) {
            if constexpr (FIRST) bad |= und_mine && v_ok[o] && (float)v_r * kv_s > sv;
            vlo = fminf(vlo, v_ok[o] ? v_own[o] : FLT_MAX);
            vhi = fmaxf(vhi, v_own[o]);
          }
        }
      };
      auto col_step = [&]() {
        float vs[RW];
#pragma unroll
        for (int T = 0; T < NT; ++T) {
          vs[4 * T] = v_own[T];
#pragma unroll
          for (int t = 1; t < 4; ++t) vs[4 * T + t] = shx(v_own[T], t);
        }
        if constexpr (TW > 0) {
          vs[4 * NT] = v_own[NT];
          if constexpr (TW == 2) vs[4 * NT + 1] = shx(v_own[NT], 2);
        }
        // the same row pairs: even- and odd-row partial sums of each column in one FFMA2, added
        uint64_t vp[RW / 2];
#pragma unroll
        for (int s = 0; s + 1 < RW; s += 2) vp[s / 2] = pack2(vs[s], vs[s + 1]);
        float qv[CW];
#pragma unroll
        for (int c = 0; c < CW; ++c) {
          // (the chain starts at a pair of shuffled v values: one that holds v_own is copied
          // first by ptxas)
          constexpr int NP = RW / 2, P0 = NP > 1 ? 1 : 0;
          float e0, e1;
          fmul2p(e0, e1, K[2 * P0][c], K[2 * P0 + 1][c], vp[P0]);
#pragma unroll
          for (int pp = 0; pp < NP; ++pp)
            if (pp != P0) ffma2p(e0, e1, K[2 * pp][c], K[2 * pp + 1][c], vp[pp], e0, e1);
          float q0 = e0 + e1;
          if constexpr (RW & 1) q0 = fmaf(K[RW - 1][c], vs[RW - 1], q0);
          qv[c] = q0;
        }
        hreduce_cols<CW>(qv);
        uint32_t umax_b = 0u;
        float uo[NCO];
#pragma unroll
        for (int g = 0; g < NCO; ++g) {
          const float acc = qv[g < Q ? 4 * g : 4 * Q + (g - Q)];
          uo[g] = r_own[g] * rcp_fast(acc);
          umax_b = max(umax_b, __float_as_uint(uo[g]));
        }
        // no per-iteration gauge (R39): the lane's running max / min of the real uh,
        // reduced over the half once per document
        umax_all = max(umax_all, umax_b);
#pragma unroll
        for (int g = 0; g < NCO; ++g) umin = fminf(umin, oreal[g] ? uo[g] : FLT_MAX);
#pragma unroll
        for (int g = 0; g < Q; ++g) {
          u[4 * g] = uo[g];
#pragma unroll
          for (int c = 1; c < 4; ++c) u[4 * g + c] = shx(uo[g], 4 * c);
        }
#pragma unroll
        for (int r = 0; r < R; ++r) u[4 * Q + r] = uo[Q + r];
      };
      row_step(std::true_type{});
      if (iters > 0) {
        col_step();
        it = 1;
        row_step(std::false_type{});
        stage3_next();   // the next item's entries have landed: start its row copies
        while (it != iters) {
          col_step();
          ++it;
          row_step(std::false_type{});
        }
      } else {
        stage3_next();
      }
    };
    if (und) iterate(std::true_type{});
    else iterate(std::false_type{});

    // ---- final step, M recovered from the block (header comment)
    float p[RW];
    if constexpr (kBufs == 2) {   // M read back from the item's staged rows (exact)
#pragma unroll
      for (int s = 0; s < RW; ++s) {
        const int e = hrow_of<NT, TW>(s, a, b);
        float x[CW];
        hload_cols<CW>(buf + (e < n ? e : 0) * P, b, x);
        to_slots<CW>(x, a);
        float acc = 0.f;
#pragma unroll
        for (int c = 0; c < CW; ++c) acc = fmaf(K[s][c] * u[c], x[c], acc);
        p[s] = acc;
      }
    } else {                      // M recovered from the block (R37)
      // Kh is 0 or normal (ex2.approx.ftz); a flushed entry gets a finite dm and k u = 0
#pragma unroll
      for (int s = 0; s + 1 < RW; s += 2) {
        float a0 = 0.f, a1 = 0.f;
#pragma unroll
        for (int c = 0; c < CW; ++c) {
          const float k0 = K[s][c], k1 = K[s + 1][c];
          float d0, d1, w0, w1;
          ffma2(d0, d1, lg2_ftz(fmaxf(k0, FLT_MIN)), lg2_ftz(fmaxf(k1, FLT_MIN)), -inv_alpha, -inv_alpha,
                mu_s[c], mu_s[c]);
          fmul2(w0, w1, k0, k1, u[c], u[c]);
          ffma2(a0, a1, w0, w1, d0, d1, a0, a1);
        }
        p[s] = a0;
        p[s + 1] = a1;
      }
      if constexpr (RW & 1) {
        float acc = 0.f;
#pragma unroll
        for (int c = 0; c < CW; ++c) {
          const float k = K[RW - 1][c];
          const float dm = fmaf(-inv_alpha, lg2_ftz(fmaxf(k, FLT_MIN)), mu_s[c]);
          acc = fmaf(k * u[c], dm, acc);
        }
        p[RW - 1] = acc;
      }
    }
    hreduce_rows<NT, TW>(p);
    float wsum = 0.f;
    const float cm_w = kBufs == 2 ? 0.f : 1.f;   // the sum_e c_e m_e term of the recovered form
#pragma unroll
    for (int T = 0; T < NT; ++T)
      if (v_ok[T]) wsum += fmaf(v_own[T], p[4 * T], cm_w * c_own[T] * m_own[T]);
    if constexpr (TW > 0) {  // each tail row is held by 2 (TW = 2) or 4 (TW = 1) lanes: count it once
      if (v_ok[NT] && (b & (TW == 1 ? 3 : 1)) == 0) wsum += fmaf(v_own[NT], p[4 * NT], cm_w * c_own[NT] * m_own[NT]);
    }
#pragma unroll
    for (int off = 8; off; off >>= 1) wsum += shx(wsum, off);
    // range form of the certificate (blocks with flushed entries; R38, R39): every real
    // row and column of Kh holds a 1, so s_e >= min_i uh_i and acc_i >= min_e vh_e. Sufficient
    // for every iteration t >= 1: min uh >= v_r 2^-110 max uh, and for every t: min vh >=
    // n 2^-110 max vh, with min / max taken over all t (t = 0 checked directly above)
    const uint32_t umax_h = half_max(umax_all, h);
    if (__any_sync(kFull, und_mine)) {
      const float vcap = (float)n * kUnder * __uint_as_float(half_max(__float_as_uint(vhi), h));
      bad |= und_mine && (umin < kv_s * __uint_as_float(umax_h) || vlo < vcap);
    }
    const bool flag = half_any(bad || !(umin >= FLT_MIN), h) || umax_h > 0x7f7fffffu || !(fabsf(wsum) <= FLT_MAX);
    if (l16 == 0 && j >= 0) {
      const int64_t o = (int64_t)q * qs.N + j;
      qs.dist[out0 + j] = wsum;
      if (qs.iters_doc) qs.iters_doc[o] = it;
      uint8_t f = und_mine ? kFlagUnderflow : 0;
      if (flag) {
        f |= kFlagFp32Range;
        qs.flagged_list[(int64_t)q * qs.N + atomicAdd(qs.flagged_count + q, 1)] = j;
      }
      // a plain store, not |=: the flags are zeroed at the query's start and this kernel is the
      // first writer of its documents' bytes (the read of the RMW exposed a global-load latency
      // per item, 2.5 % of the Scaling fused phase)
      if (f) qs.flags[o] = f;
    }
    if (q + 1 < nq) {
      ++q;
    } else {
      q = 0;
      pos += stride;
      take_next_doc();
    }
  }
  cp_async_wait_all();
}

template <int CW, int NT, int TW>
void launch_half_range(const int4* sdoc, const Entry* ent, int64_t p0, int64_t p1, const QuerySet& qs,
                       float lambda, int iters, cudaStream_t st) {
  if (p1 <= p0) return;
  constexpr size_t smem = sizeof(float) * HShape<CW, NT, TW>::BUF * kWarps * 2 * kBufs;  // per half-warp
  static PerDevice cache;
  const int resident = cache.get([&] {
    cudaFuncSetAttribute(sinkhorn_half_kernel<CW, NT, TW>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(sinkhorn_half_kernel<CW, NT, TW>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, sinkhorn_half_kernel<CW, NT, TW>, kThreads, smem);
    return std::max(1, per_sm) * device_sms();
  });
  const int64_t need = (p1 - p0 + 2 * kWarps - 1) / (2 * kWarps);
  const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>(need, resident));
  sinkhorn_half_kernel<CW, NT, TW><<<grid, kThreads, smem, st>>>(sdoc, ent, p0, p1, qs, lambda, iters);
}

// Length buckets (rows covered: 8, 16, 20, 24, 32, 36, 40)
struct HBucket { int ne, nt, tw; };
constexpr HBucket kHBuckets[] = {{8, 0, 2}, {16, 1, 0}, {20, 1, 1}, {24, 1, 2}, {32, 2, 0}, {36, 2, 1}, {40, 2, 2}};
constexpr int kNumHBuckets = 7;

template <int CW>
void dispatch_half(int bi, const int4* sdoc, const Entry* ent, int64_t p0, int64_t p1, const QuerySet& qs,
                   float lambda, int iters, cudaStream_t st) {
  switch (bi) {
    case 0: launch_half_range<CW, 0, 2>(sdoc, ent, p0, p1, qs, lambda, iters, st); break;
    case 1: launch_half_range<CW, 1, 0>(sdoc, ent, p0, p1, qs, lambda, iters, st); break;
    case 2: launch_half_range<CW, 1, 1>(sdoc, ent, p0, p1, qs, lambda, iters, st); break;
    case 3: launch_half_range<CW, 1, 2>(sdoc, ent, p0, p1, qs, lambda, iters, st); break;
    case 4: launch_half_range<CW, 2, 0>(sdoc, ent, p0, p1, qs, lambda, iters, st); break;
    case 5: launch_half_range<CW, 2, 1>(sdoc, ent, p0, p1, qs, lambda, iters, st); break;
    default: launch_half_range<CW, 2, 2>(sdoc, ent, p0, p1, qs, lambda, iters, st); break;
  }
}

}  // namespace

int half_max_rows() { return kHBuckets[kNumHBuckets - 1].ne; }

int64_t launch_sinkhorn_half(const int4* sdoc, const Entry* ent, int64_t N, const int64_t* len_prefix,
                             int64_t max_len, int ld, const QuerySet& qs, float lambda, int iters,
                             cudaStream_t st0, StreamRing* ring, int* launches) {
  // bucket ranges of the length-sorted order
  int64_t r0[kNumHBuckets], r1[kNumHBuckets];
  int64_t p0 = 0;
  for (int bi = 0; bi < kNumHBuckets; ++bi) {
    const int NE = kHBuckets[bi].ne;
    const int64_t p1 = p0 >= N ? p0 : (NE >= max_len ? N : len_prefix[NE + 1]);
    r0[bi] = p0;
    r1[bi] = std::max(p0, p1);
    p0 = r1[bi];
  }
  // longest bucket first: the shorter ones fill the SMs its tail leaves idle (Scaling 6.57 ->
  // 6.55 ms)
  for (int k = 0; k < kNumHBuckets; ++k) {
    const int bi = kNumHBuckets - 1 - k;
    if (r1[bi] <= r0[bi]) continue;
    if (launches) ++*launches;
    if (!sdoc) continue;
    const cudaStream_t st = ring ? ring->next(st0) : st0;
    switch (ld) {
      case 16: dispatch_half<4>(bi, sdoc, ent, r0[bi], r1[bi], qs, lambda, iters, st); break;
      case 24: dispatch_half<6>(bi, sdoc, ent, r0[bi], r1[bi], qs, lambda, iters, st); break;
      case 32: dispatch_half<8>(bi, sdoc, ent, r0[bi], r1[bi], qs, lambda, iters, st); break;
      default: dispatch_half<10>(bi, sdoc, ent, r0[bi], r1[bi], qs, lambda, iters, st); break;
    }
  }
  return p0;
}

}  // namespace wmd
