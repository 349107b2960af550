// EXPERIMENT, not built: a second one-CTA design with 16-row slabs and a two-level
// column sum (two barriers per pass). Correct on the whole shape sweep of
// test_fused_cta_long_documents, but slower at Long (23.0 vs 17.3 ms per query: the second
// barrier and the column-sum phase idle the SM, which holds one CTA), so the library keeps
// wmd_fused_cta.cu. Kept as the record of the attempt; it was wired in as launch_cta2_range.
// wmd_fused_cta2.cu — NEXT-1 for long documents, second design: all Sinkhorn iterations and the
// final step of a document of up to 320 words in ONE CTA of W warps, each warp holding a
// 16-row slab of the document block (the one-CTA kernel of wmd_fused_cta.cu holds 32-48-row
// slabs at up to 255 registers per thread, 8 warps per SM; here ~100-120, 12-20 warps per SM).
//
// Same method (R21, R33): the doc-local two-sided rescale Kh = 2^(-alpha D + beta_i +
// gamma_e) of Algorithm 1, u the power-of-two-gauged iterate, the FP32 range
// certificate, re-anchoring (beta_i += log2 uh_i of the pass input, the block recomputed from D
// in the log domain) instead of flagging, the final step with D recovered from Kh.
//
// Mapping. Warp w owns rows [16 w, 16 w + 16); lane = 8a + b holds 4 row slots (row
// 16w + 4a + (t ^ (b >> 1)), the one-warp kernel's 16-row tail layout) x CW = 4Q + R columns
// (wmd_tile.cuh: Q XOR-permuted quads + R plain columns), LD = 8 CW <= 128.
//   SDDMM  s = Kh uh    : warp-local (4 + CW-column FMA chains, reduce over the b-lanes)
//   SpMM   acc = Kh^T vh: per-warp column partials (reduce over the a-lanes) to shared memory;
//                         barrier 1; thread c < LD sums column c over the W warps (fixed order),
//                         uh_c = r_c / acc_c, and the warp max / min of uh feed shared atomics;
//                         barrier 2; every lane reads its CW columns of uh, scaled by the gauge
//                         (an exact power of two from the max) — two barriers per pass instead of
//                         every warp summing every column (W loads + 4W adds per lane per pass).
// Per-pass shared state (column partials, uh, the max / min / vmax words) is double-buffered by
// pass parity: each buffer is written between the barriers of one pass and read before the
// barriers of the next, so two barriers per pass order everything.
#include <algorithm>
#include <cfloat>
#include <cstdint>

#include "wmd_tile.cuh"

namespace wmd {
namespace {

using namespace dev;
using namespace tile;

constexpr float kUnder2 = 0x1p-110f;        // 2^-126 / 2^-16
constexpr float kLog2e2 = 1.4426950408889634f;
constexpr int kMaxAnchors2 = 4;

template <int CW, int W>
struct Cta2Shape {
  static constexpr int Q = CW / 4;             // XOR-permuted column quads per lane
  static constexpr int R = CW % 4;             // plain columns per lane
  static constexpr int LD = 8 * CW;            // = 32 Q + 8 R
  static constexpr int P = LD + 4;             // row pitch of Mx
  static constexpr int ROWS = 16 * W;
  static constexpr int NT = 32 * W;
  // one warp's column partials: quads lane-major (4 floats per lane), then the 8R plain columns
  static constexpr int CREM = 128, CP = 128 + 8 * R;
  static constexpr int SMEM_FLOATS = 2 * W * CP + 2 * LD + LD + 2 * ROWS + W + 8;
  static constexpr int SPL = NT >= 4 * LD ? 4 : (NT >= 2 * LD ? 2 : 1);  // threads per column sum
};

// 64K registers per SM: at most ~65536 / (32 W) registers per thread for one CTA per SM
template <int CW, int W>
constexpr int cta2_min_blocks() {
  constexpr int regs = 4 * CW + CW + 56;                       // block + uh + working set
  constexpr int b = 65536 / (32 * W * ((regs + 7) / 8 * 8));
  return b < 1 ? 1 : b;
}

template <int CW, int W>
__global__ void __launch_bounds__(32 * W, cta2_min_blocks<CW, W>()) sinkhorn_cta2_kernel(
    const int4* __restrict__ sdoc, const Entry* __restrict__ ent, int64_t pos0, int64_t pos1,
    const float* __restrict__ Mx, int v_r, const float* __restrict__ rpad, float lambda, int iters,
    int32_t* __restrict__ iters_doc, float* __restrict__ dist, uint8_t* __restrict__ flags,
    int32_t* __restrict__ flagged_list, int32_t* __restrict__ flagged_count) {
  using S = Cta2Shape<CW, W>;
  constexpr int LD = S::LD, Q = S::Q, R = S::R, P = S::P, CP = S::CP, ROWS = S::ROWS, NT = S::NT;
  constexpr int EPT = (ROWS + NT - 1) / NT;    // entries each thread prefetches
  static_assert(Q >= 1 && Q <= 4, "1 to 4 column quads per lane (LD <= 128)");
  static_assert(NT >= LD, "one column thread per column");
  extern __shared__ __align__(16) float csm[];
  float* const colpart = csm;                                 // [2][W][CP]
  float* const ucol = colpart + 2 * W * CP;                   // [2][LD] uh of the pass, by column
  float* const betal = ucol + 2 * LD;                         // [LD] column shifts beta (log2 units)
  int* const ents = reinterpret_cast<int*>(betal + LD);       // [ROWS] vocabulary row of each word
  float* const cents = reinterpret_cast<float*>(ents + ROWS); // [ROWS] its c
  float* const wred = cents + ROWS;                           // [W] per-warp distance partials
  uint32_t* const stat = reinterpret_cast<uint32_t*>(wred + W);  // [2][4]: max uh, min uh, max vh (bits)
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int a = lane >> 3, b = lane & 7;
  const int row0 = 16 * warp;
  const int2* ent2 = reinterpret_cast<const int2*>(ent);
  const uint64_t keep = l2_evict_last_policy();          // the gathered M rows stay in L2
  const uint64_t stream_pol = l2_evict_first_policy();   // the entries are read once
  const float alpha = lambda * kLog2e2;
  const float ia = -rcp_fast(alpha);
  const float kv_s = (float)v_r * kUnder2;
  // the column this thread sums: SPL consecutive threads per column (each over every SPL-th
  // warp, then a butterfly within the group), its r and whether it is a real query row
  constexpr int SPL = S::SPL;
  const int col = tid / SPL, kspl = tid % SPL;
  const bool colt = col < LD;
  const float rcol = colt ? __ldg(rpad + col) : 0.f;     // zero beyond v_r
  const bool creal = colt && col < v_r;
  int cidx = 0;                                          // its slot in a warp's partials
  if (colt) {
    if (col < 32 * Q) {                                  // quad column 32g + 4b' + a'
      const int g = col >> 5, bb = (col >> 2) & 7, aa = col & 3;
      cidx = 4 * (8 * aa + bb) + g;
    } else {                                             // plain column 32Q + R b' + r
      cidx = S::CREM + (col - 32 * Q);
    }
  }
  bool sreal[CW];  // the lane's column slots that are real query rows
#pragma unroll
  for (int c = 0; c < CW; ++c) sreal[c] = col_of<CW>(c, a, b) < v_r;
  const int orow = row0 + 4 * a + (b >> 1);             // own row after the row reduce

  // ---- prefetch: header and this thread's entries (rows tid, tid + NT, ...) of the next document
  // (unconditional loads of clamped, always valid indices, then selects: DESIGN.md §5)
  int64_t pos = pos0 + blockIdx.x;
  int pj = -1, pb = 0, pn = 0;
  int2 pe[EPT];
  auto stage1 = [&](int64_t p) {
    const bool ok = p < pos1;
    const int4 x = __ldg(sdoc + (ok ? p : pos1 - 1));
    pj = ok ? x.x : -1; pb = ok ? x.y : 0; pn = ok ? x.z : 0;
  };
  auto stage2 = [&]() {
#pragma unroll
    for (int x = 0; x < EPT; ++x) {
      const int e = tid + NT * x;
      const int2 v = ldg2_hint(ent2 + pb + (e < pn ? e : 0), stream_pol);
      pe[x] = e < pn ? v : make_int2(0, 0);
    }
  };
  stage1(pos);
  stage2();

  float K[4][CW];
  bool rok[4];
  // D = M - m of this lane's row slots, natural column order; +inf on rows past n
  auto load_D = [&](int n) {
#pragma unroll
    for (int s = 0; s < 4; ++s) {
      const int e = row0 + row_of<0, 4>(s, a, b);
      rok[s] = e < n;
      const float* row = Mx + (size_t)(rok[s] ? ents[e] : 0) * P;
      float x[CW];
#pragma unroll
      for (int q = 0; q < Q; ++q) {
        const float4 t = ldg4_hint(reinterpret_cast<const float4*>(row + 32 * q + 4 * b), keep);
        x[4 * q] = t.x; x[4 * q + 1] = t.y; x[4 * q + 2] = t.z; x[4 * q + 3] = t.w;
      }
#pragma unroll
      for (int r = 0; r < R; ++r) x[4 * Q + r] = __ldg(row + 32 * Q + R * b + r);
      const float bias = rok[s] ? -__ldg(row + LD) : INFINITY;
#pragma unroll
      for (int c = 0; c < CW; ++c) K[s][c] = x[c] + bias;
    }
  };

  for (; pos < pos1; pos += gridDim.x) {
    const int j = pj, n = pn;
#pragma unroll
    for (int x = 0; x < EPT; ++x) {
      const int e = tid + NT * x;
      if (e < ROWS) {
        ents[e] = pe[x].x;
        cents[e] = __int_as_float(pe[x].y);
      }
    }
    if (tid < 8) stat[tid] = (tid & 3) == 1 ? 0x7f800000u : 0u;   // max 0, min +inf, vmax 0
    stage1(pos + gridDim.x);
    __syncthreads();  // entries published; the previous document is done with shared memory

    const bool v_ok = orow < n;
    const float c_own = v_ok ? cents[orow] : 0.f;
    const float m_own = v_ok ? __ldg(Mx + (size_t)ents[v_ok ? orow : 0] * P + LD) : 0.f;
    // ---- block: D, column minima mu over the document, beta = alpha mu, Kh = 2^(-alpha D + beta)
    load_D(n);
    bool und;
    {
#pragma unroll
      for (int c = 0; c < CW; ++c) {  // per-warp column minima (natural order)
        float m = fminf(fminf(K[0][c], K[1][c]), fminf(K[2][c], K[3][c]));
        m = fminf(m, shx(m, 8));
        m = fminf(m, shx(m, 16));
        if (a == 0) colpart[warp * CP + nat_col<CW>(c, b)] = m;
      }
      __syncthreads();
      if (colt && kspl == 0) {  // CTA minima of the column (partials laid out by natural column here)
        float m = colpart[col];
#pragma unroll 4
        for (int w = 1; w < W; ++w) m = fminf(m, colpart[w * CP + col]);
        betal[col] = alpha * m;
      }
      __syncthreads();
      bool flushed = false;
#pragma unroll
      for (int c = 0; c < CW; ++c) {
        const float bc = betal[nat_col<CW>(c, b)];
        const bool real = nat_col<CW>(c, b) < v_r;
        float kmin = 1.f;
#pragma unroll
        for (int s = 0; s < 4; ++s) {
          K[s][c] = rok[s] ? ex2_ftz(fmaf(-alpha, K[s][c], bc)) : 1.f;  // rows past n: 1
          kmin = fminf(kmin, K[s][c]);
        }
        flushed |= real && kmin < FLT_MIN;
      }
#pragma unroll
      for (int s = 0; s < 4; ++s) to_slots<CW>(K[s], a);
      und = __syncthreads_or(flushed);
    }
    // the column threads' current input uh (for re-anchoring), and the lanes' uh (slot order)
    float uin = creal ? (float)v_r * ex2_ftz(-betal[col]) : 0.f;
    float u[CW];
#pragma unroll
    for (int c = 0; c < CW; ++c) u[c] = sreal[c] ? (float)v_r * ex2_ftz(-betal[col_of<CW>(c, a, b)]) : 0.f;
    stage2();  // the next document's entries

    float umax_k = (float)v_r * kv_s;   // v_r max(uh) 2^-110 (max uh0 <= v_r)
    float gamma_own = 0.f;              // row shift of the own row
    bool bad = false;
    int anchors = 0, it = 0;
    float v_own = 0.f, s_own = 0.f;
    for (int pass = 0;; ++pass) {
      const int par = pass & 1;
      float* const cp = colpart + par * W * CP;
      uint32_t* const st = stat + 4 * par;
      // SDDMM (warp-local)
      {
        float p[4];
#pragma unroll
        for (int s = 0; s < 4; ++s) {
          float acc = K[s][0] * u[0];
#pragma unroll
          for (int c = 1; c < CW; ++c) acc = fmaf(K[s][c], u[c], acc);
          p[s] = acc;
        }
        reduce_rows<0, 4>(p);
        s_own = p[0];
        v_own = c_own * rcp_fast(s_own);   // rows past n: Kh = 1 makes s > 0, c = 0 makes v = 0
      }
      const bool sfail = und && umax_k > s_own;
      const bool last = it == iters;
      if (!last) {
        // SpMM: this warp's column partials, transpose-reduced over the a-lanes
        float vs[4];
        vs[0] = v_own;
#pragma unroll
        for (int t = 1; t < 4; ++t) vs[t] = shx(v_own, t << 1);
        float q[CW];
#pragma unroll
        for (int c = 0; c < CW; ++c) {
          float q0 = K[0][c] * vs[0];
#pragma unroll
          for (int s = 1; s < 4; ++s) q0 = fmaf(K[s][c], vs[s], q0);
          q[c] = q0;
        }
        reduce_cols<CW>(q);
        float qo[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
        for (int g = 0; g < Q; ++g) qo[g] = q[4 * g];
        *reinterpret_cast<float4*>(cp + warp * CP + 4 * lane) = make_float4(qo[0], qo[1], qo[2], qo[3]);
        if (a == 0) {
#pragma unroll
          for (int r = 0; r < R; ++r) cp[warp * CP + S::CREM + R * b + r] = q[4 * Q + r];
        }
        if (und) {
          const uint32_t vm = __reduce_max_sync(kFull, __float_as_uint(v_own));
          if (lane == 0) atomicMax(st + 2, vm);
        }
      }
      bool fail = __syncthreads_or(sfail);
      // the other parity's statistics are free (read before this pass's barrier): reset them
      if (tid == 0) {
        stat[4 * (par ^ 1)] = 0u;
        stat[4 * (par ^ 1) + 1] = 0x7f800000u;
        stat[4 * (par ^ 1) + 2] = 0u;
      }
      float sc = 1.f, un = 0.f;
      if (!fail && !last) {
        // column step: thread c sums column c over the warps (fixed order), uh_c = r_c / acc_c
        bool cfail = false;
        uint32_t mx = 0u, mn = 0x7f800000u;
        if (warp * 32 < SPL * LD) {  // warps holding column threads (groups never straddle warps)
          float acc = 0.f;
          if (colt) {
#pragma unroll 4
            for (int w = kspl; w < W; w += SPL) acc += colpart[par * W * CP + w * CP + cidx];
          }
#pragma unroll
          for (int o = 1; o < SPL; o <<= 1) acc += shx(acc, o);   // same bits in every thread of the group
          if (colt) {
            un = rcol * rcp_fast(acc);
            if (und) cfail = (float)n * __uint_as_float(st[2]) * kUnder2 > acc;
            if (kspl == 0) ucol[par * LD + col] = un;
            if (creal) {
              mx = __float_as_uint(un);
              mn = __float_as_uint(un);
            }
          }
          mx = __reduce_max_sync(kFull, mx);
          mn = __reduce_min_sync(kFull, mn);
          if (lane == 0) {
            atomicMax(st, mx);
            atomicMin(st + 1, mn);
          }
        }
        const bool cf = __syncthreads_or(cfail);
        const uint32_t umax_b = st[0], umin_b = st[1];
        // gauge: max uh -> [1, 2) by an exact power of two (positive floats order like their bits)
        sc = __uint_as_float((254u - min(umax_b >> 23, 253u)) << 23);
        fail = cf || umax_b > 0x7f7fffffu || !(__uint_as_float(umin_b) * sc >= FLT_MIN);
      }
      if (fail && anchors == kMaxAnchors2) {
        bad = true;  // give up: the FP64 re-run recomputes this document
        fail = false;
      }
      if (fail) {
        // ---- re-anchor (CTA-uniform): beta += log2 uh of the pass input, Kh recomputed from D
        ++anchors;
        if (colt && kspl == 0 && uin > 0.f) betal[col] += lg2_approx(uin);
        __syncthreads();  // the new betal is published
        load_D(n);
        // L = -alpha D + beta (natural order); gamma_e = -(max of L over the real columns of row e)
        float rmax[4] = {-FLT_MAX, -FLT_MAX, -FLT_MAX, -FLT_MAX};
#pragma unroll
        for (int c = 0; c < CW; ++c) {
          const float bc = betal[nat_col<CW>(c, b)];
          const bool real = nat_col<CW>(c, b) < v_r;
#pragma unroll
          for (int s = 0; s < 4; ++s) {
            const float L = fmaf(-alpha, K[s][c], bc);
            K[s][c] = L;
            rmax[s] = (real && rok[s]) ? fmaxf(rmax[s], L) : rmax[s];
          }
        }
        reduce_rows_max<0, 4>(rmax);
        gamma_own = v_ok ? -rmax[0] : 0.f;
        float gs[4];
        gs[0] = gamma_own;
#pragma unroll
        for (int t = 1; t < 4; ++t) gs[t] = shx(gamma_own, t << 1);
        bool flushed = false;
#pragma unroll
        for (int c = 0; c < CW; ++c) {
          const bool real = nat_col<CW>(c, b) < v_r;
#pragma unroll
          for (int s = 0; s < 4; ++s) {
            const float kx = ex2_ftz(K[s][c] + gs[s]);
            flushed |= real && rok[s] && kx < FLT_MIN;
            K[s][c] = (rok[s] && real) ? kx : 1.f;   // padded columns (uh = 0) and rows past n: 1
          }
        }
#pragma unroll
        for (int s = 0; s < 4; ++s) to_slots<CW>(K[s], a);
#pragma unroll
        for (int c = 0; c < CW; ++c) u[c] = sreal[c] ? 1.f : 0.f;
        uin = creal ? 1.f : 0.f;
        umax_k = kv_s;
        und = __syncthreads_or(flushed);  // also: every warp is done with this pass's betal
        continue;                         // redo this pass in the new scale
      }
      if (last) break;
      ++it;
      umax_k = 2.f * kv_s;
      uin = un * sc;
#pragma unroll
      for (int c = 0; c < CW; ++c) u[c] = ucol[par * LD + col_of<CW>(c, a, b)] * sc;
    }
    // ---- final step: D = (beta + gamma - log2 Kh) / alpha (PAPER.md:64-66 with M = m + D)
    {
      float p[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
      for (int c = 0; c < CW; ++c) {
        const float uc = u[c];
        const float ub = uc * (-ia * betal[col_of<CW>(c, a, b)]);
#pragma unroll
        for (int s = 0; s < 4; ++s) {
          const float k = K[s][c];
          const float kl = k * lg2_approx(k + FLT_MIN);   // 0 at Kh = 0 (ex2.ftz: no subnormals)
          p[s] = fmaf(k, ub, fmaf(kl * ia, uc, p[s]));
        }
      }
      reduce_rows<0, 4>(p);
      float wsum = 0.f;
      // the own row is held by 2 lanes (b bit 0): count it once
      if (v_ok && (b & 1) == 0) wsum = v_own * fmaf(fmaf(-ia, gamma_own, m_own), s_own, p[0]);
#pragma unroll
      for (int off = 16; off; off >>= 1) wsum += shx(wsum, off);
      if (lane == 0) wred[warp] = wsum;
    }
    const bool anybad = __syncthreads_or(bad);
    if (tid == 0) {
      float total = 0.f;
#pragma unroll 4
      for (int w = 0; w < W; ++w) total += wred[w];
      dist[j] = total;
      if (iters_doc) iters_doc[j] = it;
      if (anybad || !(fabsf(total) <= FLT_MAX)) {
        flags[j] |= kFlagFp32Range;
        flagged_list[atomicAdd(flagged_count, 1)] = j;
      }
    }
  }
}

}  // namespace

// Documents [p0, p1) of the length-sorted order in CTAs of W = rows / 16 warps (rows in {64,
// 128, 192, 256, 320}); false if the (width, rows) pair is not instantiated.
bool launch_cta2_range(int ld, int rows, const int4* sdoc, const Entry* ent, int64_t p0, int64_t p1, const float* Mx,
                       int v_r, const float* rpad, float lambda, int iters, int32_t* itd, float* dist, uint8_t* flags,
                       int32_t* fl, int32_t* fc, cudaStream_t st) {
  auto go = [&](auto kern, int W, size_t smem_floats) {
    if (p1 <= p0) return;
    const size_t smem = sizeof(float) * smem_floats;
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 32 * W, smem);
    const int64_t resident = (int64_t)std::max(1, per_sm) * device_sms();
    const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>(p1 - p0, resident));
    kern<<<grid, 32 * W, smem, st>>>(sdoc, ent, p0, p1, Mx, v_r, rpad, lambda, iters, itd, dist, flags, fl, fc);
  };
#define K2_(CWV, WV)                                                                                     \
  if (ld == 8 * CWV && rows == 16 * WV) {                                                                \
    go(sinkhorn_cta2_kernel<CWV, WV>, WV, Cta2Shape<CWV, WV>::SMEM_FLOATS);                              \
    return true;                                                                                         \
  }
#define KW_(CWV) K2_(CWV, 4) K2_(CWV, 8) K2_(CWV, 12) K2_(CWV, 16) K2_(CWV, 20)
  KW_(4) KW_(5) KW_(6) KW_(8) KW_(10) KW_(12) KW_(13)
  K2_(16, 4) K2_(16, 8) K2_(16, 12) K2_(16, 16)
#undef KW_
#undef K2_
  return false;
}

}  // namespace wmd
