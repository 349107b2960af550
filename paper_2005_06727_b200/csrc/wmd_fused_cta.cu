// wmd_fused_cta.cu — NEXT-1 for long documents: all Sinkhorn iterations and the final step of a
// document of up to 320 words in ONE CTA of W warps, the document's Kh block in registers.
//
// Same method as the one-warp-per-document kernel (wmd_fused.cu: doc-local two-sided rescale
// Kh = 2^(-alpha D + beta_i + gamma_e), power-of-two gauge, FP32 range certificate, final step
// with D recovered from Kh), for the shapes that do not fit one warp's registers (the Long
// config: 50-300-word documents against 100 query words). Warp w holds rows [RPW w, RPW (w+1))
// of the block (RPW = 32, or 32 + 4 TW with a tail) as a 2-D lane tile, lane = 8a + b: row slots
// as in wmd_tile.cuh, and CW = 4Q + R columns per lane, LD = 8 CW: Q XOR-permuted quads (quad g
// of lane b: columns 32g + 4b + j, slot 4g + t holding j = t ^ a) and R plain columns
// (32Q + Rb + r), so LD need not be a power of two (v_r = 100: LD = 104, not 128).
//   SDDMM  s = Kh uh    : warp-local (row partials, transpose-reduce over the b-lanes)
//   SpMM   acc = Kh^T vh: per-warp column partials (transpose-reduce over the a-lanes) to shared
//                         memory; ONE barrier; then every warp sums the W partials of all LD
//                         columns itself (Q + R per lane), so uh = r / acc, its gauge and the
//                         range checks are computed redundantly and bit-identically by every
//                         warp (no second barrier); each lane gets its quad slots by three
//                         xor-shuffles per quad.
// The column partials are double-buffered by pass parity, so one barrier per iteration orders
// everything. No global memory traffic inside the loop.
//
// Re-anchoring (R33) instead of flagging: when a range check fails (a uh spread too
// wide for the FP32 exponent; PAPER.md:62-66 iterates K = exp(-lambda M) in FP64), the CTA
// recomputes the block from D in the log domain with the pass's input uh absorbed into the
// column shifts, beta_i += log2 uh_i, and row shifts gamma_e = -max_i(-alpha D_ei + beta_i) (each
// row's largest entry becomes 1), sets uh = 1 and redoes the pass. Kh -> diag(a) Kh diag(b) is a
// diagonal rescaling under which Algorithm 1's iterates are equivariant (u -> u / b, v -> v / a,
// transport plan and distance unchanged), so only rounding changes; entries are recomputed from
// D, never from flushed products, so the certificate's invariant (a zero entry stands for a true
// value < 2^-126 in the current scale) holds after the rescale. Only a document that still fails
// after kMaxAnchors re-anchors is flagged for the FP64 re-run. Bound: FP32 issue.
#include <algorithm>
#include <cfloat>
#include <cstdint>

#include "wmd_tile.cuh"

namespace wmd {
namespace {

using namespace dev;
using namespace tile;

constexpr float kUnderC = 0x1p-110f;        // 2^-126 / 2^-16
constexpr float kLog2eC = 1.4426950408889634f;
#ifndef WMD_CTA_MAX_ANCHORS
#define WMD_CTA_MAX_ANCHORS 4
#endif
constexpr int kMaxAnchors = WMD_CTA_MAX_ANCHORS;
#ifndef WMD_CTA_GUARDED_LOADS
#define WMD_CTA_GUARDED_LOADS 0
#endif

template <int CW, int W, int TW>
struct CtaShape {
  static constexpr int Q = CW / 4;             // XOR-permuted column quads per lane
  static constexpr int R = CW % 4;             // plain columns per lane
  static constexpr int LD = 8 * CW;            // = 32 Q + 8 R
  static constexpr int RPW = 32 + 4 * TW;      // rows per warp: a 32-row tile + 4 TW tail rows
  static constexpr int RW = 8 + TW;            // row slots per lane
  static constexpr int NOWN = TW ? 2 : 1;      // own rows per lane after the row reduce
  static constexpr int TSH = TW == 4 ? 1 : 2;  // tail row slot t of lane b: 32 + TW a + (t ^ (b >> TSH))
  static constexpr int ROWS = W * RPW;
  static constexpr int P = LD + 4;             // row pitch of Mx
  // one warp's column partials: quads lane-major (4 floats per lane), then the 8R plain
  // columns, then the warp's vmax
  static constexpr int CREM = 128, CVMAX = 128 + 8 * R, CP = CVMAX + 4;
  static constexpr int SMEM_FLOATS = 2 * W * CP + LD + 2 * ROWS + W + 4;
};

// Column layout (quads + plain columns, nat_col / col_of / to_slots / reduce_cols): wmd_tile.cuh.

// Resident warps per SM the register budget is written for: 12 (168 registers per thread) when
// the block takes at most 96 registers per thread, else 8 (255; at 168 those instances spill).
#ifndef WMD_CTA_WPS_BIG
#define WMD_CTA_WPS_BIG 8
#endif
template <int CW, int W, int TW>
constexpr int cta_min_blocks() {
  constexpr int wps = (8 + TW) * CW > 96 ? WMD_CTA_WPS_BIG : 12;
  return W < wps ? wps / W : 1;
}

// LIST: the documents are the ids of a device list (of *count entries) instead of a range of the
// length-sorted order: the re-run of documents the one-warp kernel could not certify (DESIGN.md
// R33); documents longer than the bucket go straight to the output list (the FP64 re-run).
struct DocList {
  const int32_t* ids;
  const int32_t* count;
  const int32_t* doc_ptr;
};

template <int CW, int W, int TW, bool LIST>
__global__ void __launch_bounds__(32 * W, cta_min_blocks<CW, W, TW>()) sinkhorn_cta_kernel(
    const int4* __restrict__ sdoc, const Entry* __restrict__ ent, int64_t pos0, int64_t pos1,
    const float* __restrict__ Mx, int v_r, const float* __restrict__ rpad, float lambda, int iters,
    int32_t* __restrict__ iters_doc, float* __restrict__ dist, uint8_t* __restrict__ flags,
    int32_t* __restrict__ flagged_list, int32_t* __restrict__ flagged_count, DocList dl) {
  using S = CtaShape<CW, W, TW>;
  constexpr int LD = S::LD, Q = S::Q, R = S::R, P = S::P, CP = S::CP, RW = S::RW, RPW = S::RPW;
  constexpr int NOWN = S::NOWN, TSH = S::TSH, ROWS = S::ROWS, NT = 32 * W;
  constexpr int EPT = (ROWS + NT - 1) / NT;    // entries each thread prefetches
  static_assert(Q >= 1 && Q <= 4, "1 to 4 column quads per lane (LD <= 128)");
  static_assert(TW == 0 || TW == 2 || TW == 4, "tail width");
  static_assert(RW % 2 == 0 && RW >= 4, "row slots in pairs (FFMA2)");
  extern __shared__ __align__(16) float csm[];
  float* colpart = csm;                                    // [2][W][CP]
  float* betal = colpart + 2 * W * CP;                     // [LD] column shifts beta (log2 units)
  int* ents = reinterpret_cast<int*>(betal + LD);          // [ROWS] vocabulary row of each word
  float* cents = reinterpret_cast<float*>(ents + ROWS);    // [ROWS] its c
  float* wred = cents + ROWS;                              // [W] per-warp distance partials
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int a = lane >> 3, b = lane & 7;
  const int row0 = RPW * warp;                             // first row of this warp's block
  const int2* ent2 = reinterpret_cast<const int2*>(ent);
  const uint64_t keep = l2_evict_last_policy();         // the gathered M rows stay in L2
  const uint64_t stream_pol = l2_evict_first_policy();  // the entries are read once
  const float alpha = lambda * kLog2eC;
  const float ia = -rcp_fast(alpha);  // (approximate: no IEEE-division slow-path call)
  const float kv_s = (float)v_r * kUnderC;
  // column step: this lane owns quad columns 32g + 4b + a (the ones reduce_cols leaves it) and,
  // with its three a-partners, the plain columns 32Q + Rb + r
  float r_own[Q], r_rem[R > 0 ? R : 1];
#pragma unroll
  for (int g = 0; g < Q; ++g) r_own[g] = __ldg(rpad + 32 * g + 4 * b + a);  // zero beyond v_r
#pragma unroll
  for (int r = 0; r < R; ++r) r_rem[r] = __ldg(rpad + 32 * Q + R * b + r);
  // own rows after the row reduce: row0 + lane, and the tail row row0 + 32 + TW a + (b >> TSH)
  int orow[NOWN];
  orow[0] = row0 + lane;
  if constexpr (TW > 0) orow[NOWN - 1] = row0 + 32 + TW * a + (b >> TSH);

  if constexpr (LIST) {
    pos1 = *dl.count;
    if (pos1 <= 0) return;
  }
  // ---- prefetch: header and this thread's entries (rows tid, tid + 32 W, ...) of the next document
  int64_t pos = pos0 + blockIdx.x;
  int pj = -1, pb = 0, pn = 0;
  int2 pe[EPT];
  // (unconditional loads of clamped, always valid indices, then selects. The round-1 guarded
  // form is kept under WMD_CTA_GUARDED_LOADS; the faults once blamed on it came from load_D's
  // select, see there and DESIGN.md §5)
  auto stage1 = [&](int64_t p) {
    const bool ok = p < pos1;
#if WMD_CTA_GUARDED_LOADS  // the round-1 form (sanitizer study only, tools/cta_fault_study.py)
    if constexpr (!LIST) {
      pj = -1; pn = 0; pb = 0;
      if (ok) {
        const int4 x = __ldg(sdoc + p);
        pj = x.x; pb = x.y; pn = x.z;
      }
      return;
    }
#endif
    if constexpr (LIST) {
      const int jj = __ldg(dl.ids + (ok ? p : pos1 - 1));
      const int b0 = __ldg(dl.doc_ptr + jj), n0 = __ldg(dl.doc_ptr + jj + 1) - b0;
      // a document longer than this bucket: id encoded as -2 - j, nothing to prefetch
      pj = ok ? (n0 <= ROWS ? jj : -2 - jj) : -1;
      pb = ok ? b0 : 0;
      pn = ok && n0 <= ROWS ? n0 : 0;
    } else {
      const int4 x = __ldg(sdoc + (ok ? p : pos1 - 1));
      pj = ok ? x.x : -1; pb = ok ? x.y : 0; pn = ok ? x.z : 0;
    }
  };
  auto stage2 = [&]() {
#pragma unroll
    for (int x = 0; x < EPT; ++x) {
      const int e = tid + NT * x;
#if WMD_CTA_GUARDED_LOADS
      pe[x] = e < pn ? __ldg(ent2 + pb + e) : make_int2(0, 0);
#else
      const int2 v = ldg2_hint(ent2 + pb + (e < pn ? e : 0), stream_pol);  // read once
      pe[x] = e < pn ? v : make_int2(0, 0);
#endif
    }
  };
  stage1(pos);
  stage2();

  float K[RW][CW];
  // a per-own-row value broadcast to the row slots (slot s < 8: row 8a + (s ^ b), lane ^ s;
  // tail slot 8 + t: row 32 + TW a + (t ^ (b >> TSH)), lane ^ (t << TSH))
  auto rows_to_slots = [&](const float (&o)[NOWN], float (&x)[RW]) {
    x[0] = o[0];
#pragma unroll
    for (int t = 1; t < 8; ++t) x[t] = shx(o[0], t);
    if constexpr (TW > 0) {
      x[8] = o[NOWN - 1];
#pragma unroll
      for (int t = 1; t < TW; ++t) x[8 + t] = shx(o[NOWN - 1], t << TSH);
    }
  };
  // D = M - m of this lane's row slots, natural column order; FLT_MAX on rows past n
  auto load_D = [&](int n) {
#pragma unroll
    for (int s = 0; s < RW; ++s) {
      const int e = row0 + row_of<1, TW>(s, a, b);
      const bool ok = e < n;
      // ents[e] is 0 for the rows past n (the prefetch zero-fills them), so no select: the form
      // (ok ? ents[e] : 0) compiled to CS2R Rx, SRZ + a predicated IMAD.WIDE Rx + a read of Rx
      // 5 cycles after the CS2R, which on rows past n read Rx's previous contents (a float) as
      // the row offset — the illegal-address / misaligned / invalid-address-space fault of
      // DESIGN.md §5, located with cuda-gdb (tools/sass_hazard_scan.py lists such sites)
      const float* row = Mx + (size_t)ents[e] * P;
      float x[CW];
#pragma unroll
      for (int q = 0; q < Q; ++q) {
        const float4 t = ldg4_hint(reinterpret_cast<const float4*>(row + 32 * q + 4 * b), keep);
        x[4 * q] = t.x; x[4 * q + 1] = t.y; x[4 * q + 2] = t.z; x[4 * q + 3] = t.w;
      }
#pragma unroll
      for (int r = 0; r < R; ++r) x[4 * Q + r] = __ldg(row + 32 * Q + R * b + r);
      const float me = __ldg(row + LD);
#pragma unroll
      for (int c = 0; c < CW; ++c) K[s][c] = ok ? x[c] - me : FLT_MAX;
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
    stage1(pos + gridDim.x);
    __syncthreads();  // entries published; the previous document is done with shared memory
    if constexpr (LIST) {
      if (j <= -2) {  // too long for this bucket: on to the FP64 re-run (CTA-uniform branch)
        if (tid == 0) flagged_list[atomicAdd(flagged_count, 1)] = -2 - j;
        stage2();
        continue;
      }
    }

    bool v_ok[NOWN];
    float c_own[NOWN], m_own[NOWN];
#pragma unroll
    for (int o = 0; o < NOWN; ++o) {
      v_ok[o] = orow[o] < n;
      c_own[o] = v_ok[o] ? cents[orow[o]] : 0.f;
      m_own[o] = v_ok[o] ? __ldg(Mx + (size_t)ents[orow[o]] * P + LD) : 0.f;
    }
    // ---- block tile: D, column minima mu (per warp, then over the CTA), beta = alpha mu, Kh
    load_D(n);
    float uo[Q], ur[R > 0 ? R : 1];  // uh of the owned quad columns and of the plain columns
    bool und;
    {
      // per-warp column minima (one column at a time: the block alone fills the registers)
#pragma unroll
      for (int c = 0; c < CW; ++c) {
        float m = K[0][c];
#pragma unroll
        for (int s = 1; s < RW; ++s) m = fminf(m, K[s][c]);
        m = fminf(m, shx(m, 8));
        m = fminf(m, shx(m, 16));
        if (a == 0) colpart[warp * CP + nat_col<CW>(c, b)] = m;
      }
      __syncthreads();
      if (warp == 0) {  // CTA minima: beta = alpha mu (gamma = 0)
        for (int col = lane; col < LD; col += 32) {
          float m = colpart[col];
#pragma unroll
          for (int w = 1; w < W; ++w) m = fminf(m, colpart[w * CP + col]);
          betal[col] = alpha * m;
        }
      }
      __syncthreads();
      bool flushed = false;
#pragma unroll
      for (int c = 0; c < CW; ++c) {
        const int col = nat_col<CW>(c, b);
        const bool real = col < v_r;
        const float bc = betal[col];
#pragma unroll
        for (int s = 0; s < RW; ++s) {
          const float dd = K[s][c];
          const float kx = ex2_ftz(fmaf(-alpha, dd, bc));
          flushed |= real && kx < FLT_MIN && dd != FLT_MAX;
          K[s][c] = real ? kx : (dd != FLT_MAX ? 1.f : 0.f);  // padded columns: 1 on real rows
        }
      }
#pragma unroll
      for (int s = 0; s < RW; ++s) to_slots<CW>(K[s], a);
      und = __syncthreads_or(flushed);  // also: the minima are read
    }
    // uh0 = v_r 2^-beta (x0 = 1 / v_r, in the rescaled variables)
#pragma unroll
    for (int g = 0; g < Q; ++g) {
      const int col = 32 * g + 4 * b + a;
      uo[g] = col < v_r ? (float)v_r * ex2_ftz(-betal[col]) : 0.f;
    }
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int col = 32 * Q + R * b + r;
      ur[r] = col < v_r ? (float)v_r * ex2_ftz(-betal[col]) : 0.f;
    }
    stage2();  // the next document's entries

    float umax_k = (float)v_r * kv_s;  // v_r max(uh) 2^-110 (max uh0 <= v_r)
    float gamma_own[NOWN];             // row shifts of this lane's own rows
#pragma unroll
    for (int o = 0; o < NOWN; ++o) gamma_own[o] = 0.f;
    bool bad = false;
    int anchors = 0;
    float v_own[NOWN], s_own[NOWN];
    int it = 0;
    for (int pass = 0;; ++pass) {
      // SDDMM (warp-local; one quad of uh live at a time: its slots come from lanes ^ 0, 8, 16, 24)
      float p[RW];
#pragma unroll
      for (int g = 0; g < Q; ++g) {
        float u4[4];
        u4[0] = uo[g];
#pragma unroll
        for (int t = 1; t < 4; ++t) u4[t] = shx(uo[g], 8 * t);
        // rows in pairs (s, s + 1) (RW is even), one FFMA2 per column with uh broadcast
#pragma unroll
        for (int s = 0; s < RW; s += 2) {
          float a0, a1;
          if (g == 0) fmul2(a0, a1, K[s][0], K[s + 1][0], u4[0], u4[0]);
          else ffma2(a0, a1, K[s][4 * g], K[s + 1][4 * g], u4[0], u4[0], p[s], p[s + 1]);
#pragma unroll
          for (int t = 1; t < 4; ++t) ffma2(a0, a1, K[s][4 * g + t], K[s + 1][4 * g + t], u4[t], u4[t], a0, a1);
          p[s] = a0;
          p[s + 1] = a1;
        }
      }
#pragma unroll
      for (int r = 0; r < R; ++r) {
#pragma unroll
        for (int s = 0; s < RW; s += 2)
          ffma2(p[s], p[s + 1], K[s][4 * Q + r], K[s + 1][4 * Q + r], ur[r], ur[r], p[s], p[s + 1]);
      }
      reduce_rows<1, TW>(p);
      bool sfail = false;
      uint32_t vmax_l = 0u;
#pragma unroll
      for (int o = 0; o < NOWN; ++o) {
        s_own[o] = p[8 * o];
        v_own[o] = v_ok[o] ? c_own[o] * rcp_fast(s_own[o]) : 0.f;
        sfail |= v_ok[o] && und && umax_k > s_own[o];
        vmax_l = max(vmax_l, __float_as_uint(v_own[o]));
      }
      const bool last = it == iters;
      float* cp = colpart + (pass & 1) * W * CP;
      if (!last) {
        const uint32_t vmax_w = __reduce_max_sync(kFull, vmax_l);
        // SpMM: this warp's column partials, one quad at a time, then its transpose-reduce
        float vs[RW];
        rows_to_slots(v_own, vs);
        uint64_t vp[RW / 2];  // the row pairs' v, packed once
#pragma unroll
        for (int s = 0; s < RW; s += 2) vp[s / 2] = pack2(vs[s], vs[s + 1]);
        float qo[4];
#pragma unroll
        for (int g = 0; g < 4; ++g) qo[g] = 0.f;
#pragma unroll
        for (int g = 0; g < Q; ++g) {
          float q[4];
#pragma unroll
          for (int t = 0; t < 4; ++t) {  // even- and odd-row partial sums in one FFMA2, added
            float e0, e1;
            fmul2p(e0, e1, K[2][4 * g + t], K[3][4 * g + t], vp[1]);
#pragma unroll
            for (int pp = 0; pp < RW / 2; ++pp)
              if (pp != 1) ffma2p(e0, e1, K[2 * pp][4 * g + t], K[2 * pp + 1][4 * g + t], vp[pp], e0, e1);
            q[t] = e0 + e1;
          }
          reduce_cols<4>(q);
          qo[g] = q[0];
        }
        // lane-major quads: this lane's columns are contiguous (read back by the same lane)
        *reinterpret_cast<float4*>(cp + warp * CP + 4 * lane) = make_float4(qo[0], qo[1], qo[2], qo[3]);
#pragma unroll
        for (int r = 0; r < R; ++r) {
          float e0, e1;
          fmul2p(e0, e1, K[2][4 * Q + r], K[3][4 * Q + r], vp[1]);
#pragma unroll
          for (int pp = 0; pp < RW / 2; ++pp)
            if (pp != 1) ffma2p(e0, e1, K[2 * pp][4 * Q + r], K[2 * pp + 1][4 * Q + r], vp[pp], e0, e1);
          float q0 = e0 + e1;
          q0 += shx(q0, 16);
          q0 += shx(q0, 8);
          if (a == 0) cp[warp * CP + S::CREM + R * b + r] = q0;
        }
        if (lane == 0) cp[warp * CP + S::CVMAX] = __uint_as_float(vmax_w);
      }
      bool fail = __syncthreads_or(sfail);
      float un[Q], unr[R > 0 ? R : 1];
#pragma unroll
      for (int g = 0; g < Q; ++g) un[g] = 0.f;
#pragma unroll
      for (int r = 0; r < R; ++r) unr[r] = 0.f;
      if (!fail && !last) {
        // column step, redundantly in every warp: acc = sum of the W warps' partials
        float acc[4], accr[R > 0 ? R : 1];
#pragma unroll
        for (int g = 0; g < 4; ++g) acc[g] = 0.f;
#pragma unroll
        for (int r = 0; r < R; ++r) accr[r] = 0.f;
        // fully unrolled: Long 16.55 -> 16.31 ms, although the W float4 loads in flight make the
        // 4-warp x 48-row instance at CW = 13 reload 4 spilled scalars per pass (L1 hits; the
        // spill-free 2-unrolled form measured 16.47 ms)
#pragma unroll
        for (int w = 0; w < W; ++w) {
          const float4 t = *reinterpret_cast<const float4*>(cp + w * CP + 4 * lane);
          acc[0] += t.x; acc[1] += t.y; acc[2] += t.z; acc[3] += t.w;
#pragma unroll
          for (int r = 0; r < R; ++r) accr[r] += cp[w * CP + S::CREM + R * b + r];
        }
        bool cfail = false;
        if (und) {  // acc-side certificate: flushed entries move acc_i by < n vmax 2^-126
          float vmax = 0.f;
#pragma unroll
          for (int w = 0; w < W; ++w) vmax = fmaxf(vmax, cp[w * CP + S::CVMAX]);
          const float vcap = (float)n * vmax * kUnderC;
#pragma unroll
          for (int g = 0; g < Q; ++g) cfail |= vcap > acc[g];
#pragma unroll
          for (int r = 0; r < R; ++r) cfail |= vcap > accr[r];
        }
        uint32_t um = 0u;
#pragma unroll
        for (int g = 0; g < Q; ++g) {
          un[g] = r_own[g] * rcp_fast(acc[g]);
          um = max(um, __float_as_uint(un[g]));
        }
#pragma unroll
        for (int r = 0; r < R; ++r) {
          unr[r] = r_rem[r] * rcp_fast(accr[r]);
          um = max(um, __float_as_uint(unr[r]));
        }
        // gauge: max uh -> [1, 2) by an exact power of two (identical in every warp)
        const uint32_t umax_b = __reduce_max_sync(kFull, um);
        const float sc = __uint_as_float((254u - min(umax_b >> 23, 253u)) << 23);
        cfail |= umax_b > 0x7f7fffffu;
#pragma unroll
        for (int g = 0; g < Q; ++g) {
          un[g] *= sc;
          cfail |= 32 * g + 4 * b + a < v_r && !(un[g] >= FLT_MIN);
        }
#pragma unroll
        for (int r = 0; r < R; ++r) {
          unr[r] *= sc;
          cfail |= 32 * Q + R * b + r < v_r && !(unr[r] >= FLT_MIN);
        }
        fail = __any_sync(kFull, cfail);  // warp-uniform, and the same in every warp
      }
      if (fail && anchors == kMaxAnchors) {
        bad = true;  // give up: the FP64 re-run recomputes this document
        fail = false;
      }
      if (fail) {
        // ---- re-anchor (CTA-uniform branch): beta += log2 uh, Kh recomputed from D
        ++anchors;
        float bown[Q], brem[R > 0 ? R : 1];  // new beta of this lane's columns (same in every warp)
#pragma unroll
        for (int g = 0; g < Q; ++g) {
          const float bo = betal[32 * g + 4 * b + a];
          bown[g] = uo[g] > 0.f ? bo + lg2_approx(uo[g]) : bo;
        }
#pragma unroll
        for (int r = 0; r < R; ++r) {
          const float bo = betal[32 * Q + R * b + r];
          brem[r] = ur[r] > 0.f ? bo + lg2_approx(ur[r]) : bo;
        }
        __syncthreads();  // every warp has read betal
        if (warp == 0) {
#pragma unroll
          for (int g = 0; g < Q; ++g) betal[32 * g + 4 * b + a] = bown[g];
          if (a == 0) {
#pragma unroll
            for (int r = 0; r < R; ++r) betal[32 * Q + R * b + r] = brem[r];
          }
        }
        load_D(n);
#pragma unroll
        for (int s = 0; s < RW; ++s) to_slots<CW>(K[s], a);
        __syncthreads();  // the new betal is published
        // L = -alpha D + beta; gamma_e = -(max of L over the real columns of row e)
        float rmax[RW];
#pragma unroll
        for (int s = 0; s < RW; ++s) rmax[s] = -FLT_MAX;
#pragma unroll
        for (int c = 0; c < CW; ++c) {
          const int col = col_of<CW>(c, a, b);
          const float bc = betal[col];
#pragma unroll
          for (int s = 0; s < RW; ++s) {
            const float dd = K[s][c];
            const float L = fmaf(-alpha, dd, bc);
            K[s][c] = L;
            rmax[s] = (col < v_r && dd != FLT_MAX) ? fmaxf(rmax[s], L) : rmax[s];
          }
        }
        reduce_rows_max<1, TW>(rmax);
#pragma unroll
        for (int o = 0; o < NOWN; ++o) gamma_own[o] = v_ok[o] ? -rmax[8 * o] : 0.f;
        float gs[RW];
        rows_to_slots(gamma_own, gs);
        bool flushed = false;
#pragma unroll
        for (int s = 0; s < RW; ++s) {
          const bool rowok = row0 + row_of<1, TW>(s, a, b) < n;
#pragma unroll
          for (int c = 0; c < CW; ++c) {
            const bool real = col_of<CW>(c, a, b) < v_r;
            const float kx = ex2_ftz(K[s][c] + gs[s]);
            flushed |= real && rowok && kx < FLT_MIN;
            K[s][c] = rowok ? (real ? kx : 1.f) : 0.f;
          }
        }
#pragma unroll
        for (int g = 0; g < Q; ++g) uo[g] = 32 * g + 4 * b + a < v_r ? 1.f : 0.f;
#pragma unroll
        for (int r = 0; r < R; ++r) ur[r] = 32 * Q + R * b + r < v_r ? 1.f : 0.f;
        umax_k = kv_s;
        und = __syncthreads_or(flushed);  // also: betal published
        continue;                         // redo this pass in the new scale
      }
      if (last) break;
      ++it;
      umax_k = 2.f * kv_s;
#pragma unroll
      for (int g = 0; g < Q; ++g) uo[g] = un[g];
#pragma unroll
      for (int r = 0; r < R; ++r) ur[r] = unr[r];
    }
    // ---- final step: D = (beta + gamma - log2 Kh) / alpha (PAPER.md:64-66 with M = m + D); the
    // recovery's absolute error ~2^-22 / alpha sets kFusedMinLambda (wmd_internal.h)
    {
      float p[RW];
#pragma unroll
      for (int s = 0; s < RW; ++s) p[s] = 0.f;
#pragma unroll
      for (int c = 0; c < CW; ++c) {
        // uh of slot c, and uh beta / alpha
        const float uc = c < 4 * Q ? ((c & 3) == 0 ? uo[c >> 2] : shx(uo[c >> 2], 8 * (c & 3))) : ur[c - 4 * Q];
        const float ub = uc * (-ia * betal[col_of<CW>(c, a, b)]);
#pragma unroll
        for (int s = 0; s < RW; s += 2) {  // row pairs; k = 0 or normal (ex2.approx.ftz): k log2 k = 0 for k = 0
          const float k0 = K[s][c], k1 = K[s + 1][c];
          float l0, l1, t0, t1;
          fmul2(l0, l1, k0, k1, lg2_ftz(fmaxf(k0, FLT_MIN)), lg2_ftz(fmaxf(k1, FLT_MIN)));
          ffma2(t0, t1, l0, l1, ia * uc, ia * uc, p[s], p[s + 1]);
          ffma2(p[s], p[s + 1], k0, k1, ub, ub, t0, t1);
        }
      }
      reduce_rows<1, TW>(p);
      float wsum = 0.f;
#pragma unroll
      for (int o = 0; o < NOWN; ++o) {
        const float m = fmaf(-ia, gamma_own[o], m_own[o]);
        // each tail row is held by 2^TSH lanes: count it once
        const bool once = o == 0 || (b & ((1 << TSH) - 1)) == 0;
        if (v_ok[o] && once) wsum = fmaf(v_own[o], fmaf(m, s_own[o], p[8 * o]), wsum);
      }
#pragma unroll
      for (int off = 16; off; off >>= 1) wsum += shx(wsum, off);
      if (lane == 0) wred[warp] = wsum;
    }
    const bool anybad = __syncthreads_or(bad);
    if (tid == 0) {
      float total = 0.f;
#pragma unroll
      for (int w = 0; w < W; ++w) total += wred[w];
      dist[j] = total;
      if (iters_doc) iters_doc[j] = it;
      if (anybad || !(fabsf(total) <= FLT_MAX)) {
        flags[j] |= kFlagFp32Range;
        flagged_list[atomicAdd(flagged_count, 1)] = j;
      } else if (LIST) {
        flags[j] |= kFlagRerun;
      }
    }
  }
}

template <int CW, int W, int TW, bool LIST>
int cta_resident() {
  constexpr size_t smem = sizeof(float) * CtaShape<CW, W, TW>::SMEM_FLOATS;
  static PerDevice cache;
  return cache.get([&] {
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, sinkhorn_cta_kernel<CW, W, TW, LIST>, 32 * W, smem);
    return std::max(1, per_sm) * device_sms();
  });
}

template <int CW, int W, int TW>
void launch_cta_range(const int4* sdoc, const Entry* ent, int64_t p0, int64_t p1, const float* Mx, int v_r,
                      const float* rpad, float lambda, int iters, int32_t* itd, float* dist, uint8_t* flags,
                      int32_t* fl, int32_t* fc, cudaStream_t st) {
  if (p1 <= p0) return;
  constexpr size_t smem = sizeof(float) * CtaShape<CW, W, TW>::SMEM_FLOATS;
  const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>(p1 - p0, cta_resident<CW, W, TW, false>()));
  sinkhorn_cta_kernel<CW, W, TW, false><<<grid, 32 * W, smem, st>>>(sdoc, ent, p0, p1, Mx, v_r, rpad, lambda,
                                                                    iters, itd, dist, flags, fl, fc, DocList{});
}

// The re-run of a device list of documents (at most 64 words each are re-run; longer ones are
// passed on) in 2-warp CTAs, one resident wave that loops over the list.
template <int CW>
void launch_cta_list(const int32_t* ids, const int32_t* count, const int32_t* doc_ptr, const Entry* ent,
                     const float* Mx, int v_r, const float* rpad, float lambda, int iters, int32_t* itd,
                     float* dist, uint8_t* flags, int32_t* out_list, int32_t* out_count, cudaStream_t st) {
  constexpr size_t smem = sizeof(float) * CtaShape<CW, 2, 0>::SMEM_FLOATS;
  const unsigned grid = (unsigned)cta_resident<CW, 2, 0, true>();
  sinkhorn_cta_kernel<CW, 2, 0, true><<<grid, 64, smem, st>>>(nullptr, ent, 0, 0, Mx, v_r, rpad, lambda, iters,
                                                             itd, dist, flags, out_list, out_count,
                                                             DocList{ids, count, doc_ptr});
}

// Row buckets (rows = W x (32 + 4 TW)), W dividing the 8 resident warps per SM: 2 warps of 32 /
// 40 / 48 rows (64, 80, 96), 4 warps of 32 / 40 / 48 rows (128, 160, 192: two CTAs per SM, where
// 6 warps of 32 rows would leave one 6-warp CTA per SM), 8 warps of 32 rows (256) and of 40
// rows (320). The 80-, 96- and 160-row buckets cut Long's padded rows by 4.4 % (16.30 -> 15.74
// ms per query).
struct CtaBucket { int rows, w, tw; };
constexpr CtaBucket kCta[] = {{64, 2, 0}, {80, 2, 2}, {96, 2, 4}, {128, 4, 0}, {160, 4, 2}, {192, 4, 4}, {256, 8, 0}, {320, 8, 2}};
constexpr int kNumCta = 8;

template <int CW>
void dispatch_cta(int wi, const int4* sdoc, const Entry* ent, int64_t p0, int64_t p1, const float* Mx, int v_r,
                  const float* rpad, float lambda, int iters, int32_t* itd, float* dist, uint8_t* flags,
                  int32_t* fl, int32_t* fc, cudaStream_t st) {
  switch (wi) {
#define C_(I, W, TW) case I: launch_cta_range<CW, W, TW>(sdoc, ent, p0, p1, Mx, v_r, rpad, lambda, iters, itd, dist, flags, fl, fc, st); break;
    C_(0, 2, 0) C_(1, 2, 2) C_(2, 2, 4) C_(3, 4, 0) C_(4, 4, 2) C_(5, 4, 4) C_(6, 8, 0) C_(7, 8, 2)
#undef C_
    default: break;
  }
}

}  // namespace

int cta_max_rows() { return kCta[kNumCta - 1].rows; }

// Row width of the one-CTA kernel's tables for a query of v_r rows: 8 CW with CW in {4, 5, 6,
// 8, 10, 12, 13, 16} (at v_r = 100: 104 columns, 4 padded, instead of 128); the one-warp kernel
// shares it for the shorter documents of the same query.
int cta_ld(int v_r) {
  for (int cw : {4, 5, 6, 8, 10, 12, 13, 16})
    if (8 * cw >= v_r) return 8 * cw;
  return 0;
}

// Documents of the length-sorted range [p0, N) by row buckets (kCta); len_prefix[L] = number of
// documents with fewer than L nonzeros.
void launch_sinkhorn_cta(const int4* sdoc, const Entry* ent, int64_t p0, int64_t N, const int64_t* len_prefix,
                         int64_t max_len, const float* Mx, int ld, int v_r, const float* rpad, float lambda,
                         int iters, int32_t* iters_doc, float* dist, uint8_t* flags, int32_t* flagged_list,
                         int32_t* flagged_count, cudaStream_t st0, StreamRing* ring) {
  for (int wi = 0; wi < kNumCta && p0 < N; ++wi) {
    const int rows = kCta[wi].rows;
    const int64_t p1 = rows >= max_len ? N : len_prefix[rows + 1];
    if (p1 > p0) {
      const cudaStream_t st = ring ? ring->next(st0) : st0;
      switch (ld) {
#define D_(LDV) case LDV: dispatch_cta<LDV / 8>(wi, sdoc, ent, p0, p1, Mx, v_r, rpad, lambda, iters, iters_doc, dist, flags, flagged_list, flagged_count, st); break;
        D_(32) D_(40) D_(48) D_(64) D_(80) D_(96) D_(104) D_(128)
#undef D_
        default: break;
      }
    }
    p0 = std::max(p0, p1);
  }
}

bool cta_rerun_supported(int ld) { return ld == 32 || ld == 40 || ld == 48 || ld == 64; }

void launch_cta_rerun(const int32_t* ids, const int32_t* count, const int32_t* doc_ptr, const Entry* ent,
                      const float* Mx, int ld, int v_r, const float* rpad, float lambda, int iters,
                      int32_t* iters_doc, float* dist, uint8_t* flags, int32_t* out_list, int32_t* out_count,
                      cudaStream_t st) {
  switch (ld) {
#define R_(LDV) case LDV: launch_cta_list<LDV / 8>(ids, count, doc_ptr, ent, Mx, v_r, rpad, lambda, iters, iters_doc, dist, flags, out_list, out_count, st); break;
    R_(32) R_(40) R_(48) R_(64)
#undef R_
    default: break;
  }
}

int cta_launch_count(int64_t p0, int64_t N, const int64_t* len_prefix, int64_t max_len) {
  int cnt = 0;
  for (int wi = 0; wi < kNumCta && p0 < N; ++wi) {
    const int rows = kCta[wi].rows;
    const int64_t p1 = rows >= max_len ? N : len_prefix[rows + 1];
    cnt += p1 > p0;
    p0 = std::max(p0, p1);
  }
  return cnt;
}

}  // namespace wmd
