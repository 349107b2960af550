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
// and the same distance WMD = sum_e vh_e sum_i Kh_ei M_ie uh_i. Every sum has a
// unit-size term. Each iteration applies an exact power-of-two gauge to uh (R21).
//
// FP32 range certificate: an entry flushed to 0 (true value < 2^-126) is an absolute error
// < 2^-126 in its product. If the document has any flushed entry, it keeps its FP32 result only
// if every iteration satisfies, for every e and i,
//     s_e   = sum_i Kh_ei uh_i :  v_r * max_i uh_i * 2^-126 <= 2^-16 s_e
//     acc_i = sum_e Kh_ei vh_e :  n   * max_e vh_e * 2^-126 <= 2^-16 acc_i
// and all uh stay normal; otherwise it is flagged and recomputed in FP64 (fallback_fp64).
//
// Mapping (2-D tiling of the document block over a warp). Lane = 8a + b: a in [0,4) picks a
// group of document rows (words), b in [0,8) a group of CW = LD/8 block columns (query rows).
// Each lane holds an RW x CW tile of Kh in registers (one copy of the block per warp), so
//   SDDMM  s = Kh uh     : RW*CW FFMA per lane, then a transpose-reduce over the 8 b-lanes
//   SpMM   acc = Kh^T vh : the same FFMA count, then a transpose-reduce over the 4 a-lanes
// and the reduced values (one row / one column per lane) are redistributed with xor-shuffles.
// The register slots are XOR-permuted by the lane bits (row slot t holds row 8a + (t ^ b),
// column slot c holds column 4b + (c ^ a)) so that every transpose stage sends the upper half
// of the slots and keeps the lower half with no selects. Per iteration and 32x32 block: 64 FFMA
// and 20 SHFL per lane, two reciprocals, three redux.sync; no shared or global memory traffic
// (measured on this B200: a warp shuffle costs one SM-cycle, a broadcast LDS.128 2.5,
// profiles/r01_issue_bench.jsonl). The M rows of the next document are staged in shared memory
// by cp.async while the current one iterates. Bound: FP32 issue / shuffle throughput.
#include <algorithm>
#include <cfloat>
#include <cstdint>
#include <cstdlib>
#include <type_traits>

#include "wmd_tile.cuh"

namespace wmd {
namespace {

using namespace dev;
using namespace tile;

constexpr int kWarps = 4;                  // warps per block
constexpr int kThreads = 32 * kWarps;
constexpr float kUnder = 0x1p-110f;        // 2^-126 / 2^-16
constexpr float kLog2e = 1.4426950408889634f;

// CW: block columns per lane (LD = 8 CW query rows, CW in {1, 2, 4, 8}).
// NT: full 32-row tiles; TW: rows per lane of a trailing 4*TW-row tile (0, 2 or 4).
template <int CW, int NT, int TW>
struct Shape {
  static constexpr int LD = 8 * CW;
  static constexpr int RW = 8 * NT + TW;        // row slots per lane
  static constexpr int NE = 32 * NT + 4 * TW;   // document rows covered
  static constexpr int NW = (NE + 31) / 32;     // entry slots per lane (staging)
  static constexpr int P = LD + 4;              // row pitch (floats) of Mx and the staging buffers
  static constexpr int BUF = NE * P;
  static constexpr int TSH = TW == 4 ? 1 : 2;   // tail row slot t of lane b: TW a + (t ^ (b >> TSH))
  static constexpr int REGS = RW * CW;
};

#ifndef WMD_FUSED_REG_SLACK
#define WMD_FUSED_REG_SLACK 8
#endif
template <int CW, int NT, int TW>
constexpr int min_blocks() {
  using S = Shape<CW, NT, TW>;
  constexpr int regs = ((S::REGS + 3 * S::RW + 2 * CW + 16 + WMD_FUSED_REG_SLACK) + 7) / 8 * 8;
  constexpr int b = 65536 / (kThreads * regs);
  return b < 1 ? 1 : (b > 8 ? 8 : b);
}

// Items: (document, query) pairs, document-major: a warp takes a document (grid stride over the
// length-sorted positions) and solves it for the qs.nq queries in turn, so the document's
// header and entries (c) are read once per batch; only its M rows differ per query (each query
// has its own table). The per-query lane constants are reloaded when the query changes.
template <int CW, int NT, int TW, bool CONV>
__global__ void __launch_bounds__(kThreads, min_blocks<CW, NT, TW>()) sinkhorn_fused_kernel(
    const int4* __restrict__ sdoc, const Entry* __restrict__ ent, int64_t pos0, int64_t pos1,
    QuerySet qs, float lambda, int iters, float tol) {
  using S = Shape<CW, NT, TW>;
  constexpr int LD = S::LD, RW = S::RW, NW = S::NW, P = S::P;
  constexpr int NOWN = NT + (TW ? 1 : 0);        // own rows per lane after the row reduce
  // own columns per lane after the column reduce: the quad columns 32g + 4b + a and the plain
  // columns 32Q + Rb + r (CW >= 3), else column 2b + (a >> 1) (CW = 2) or b (CW = 1)
  constexpr int CQ = Cols<CW>::Q, CR = Cols<CW>::R;
  constexpr int NCO = CW >= 3 ? CQ + CR : 1;
  extern __shared__ __align__(16) float smem[];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int a = lane >> 3, b = lane & 7;
  // the staged M rows: two buffers per warp, the current item's (read again by the final step)
  // and the next item's (filled by cp.async while the current one iterates)
  float* const buf0 = smem + 2 * wib * S::BUF;
  int cur = 1;                                   // buffer of the current item (flipped per item)
  const int64_t stride = (int64_t)gridDim.x * kWarps;
  const uint64_t keep = l2_evict_last_policy();         // the gathered M rows stay in L2
  const uint64_t stream_pol = l2_evict_first_policy();  // c is read once
  const int2* ent2 = reinterpret_cast<const int2*>(ent);
  const float alpha = lambda * kLog2e;          // exp(-lambda x) = 2^(-alpha x)
  const int nq = qs.nq;

  // per-query constants of the current item: width, own columns (after the column reduce) and
  // their marginals r_i (zero beyond v_r), real natural-order columns of the lane's group
  int v_r = 0;
  float kv_s = 0.f;
  float r_own[NCO];
  bool oreal[NCO], nreal[CW];
  int64_t out0 = 0;               // the current query's distance row
  auto set_query = [&](int q) {
    const int g = qs.qmap ? __ldg(qs.qmap + q) : q;
    out0 = (int64_t)g * qs.N;
    v_r = qs.vr ? __ldg(qs.vr + g) : qs.v_r;
    kv_s = (float)v_r * kUnder;
    const float* rp = qs.rpad + (size_t)g * WMD_MAX_VR_DEV;
#pragma unroll
    for (int g = 0; g < NCO; ++g) {
      const int oc = CW >= 3 ? (g < CQ ? 32 * g + 4 * b + a : 32 * CQ + CR * b + (g - CQ))
                             : (CW == 2 ? 2 * b + (a >> 1) : b);
      r_own[g] = __ldg(rp + oc);
      oreal[g] = oc < v_r;
    }
#pragma unroll
    for (int c = 0; c < CW; ++c) nreal[c] = nat_col<CW>(c, b) < v_r;
  };

  // ---- prefetch: stage 1 (next document's header), stage 2 (its entries), stage 3 (cp.async of
  // the next item's M rows)
  int64_t pos = pos0 + (int64_t)blockIdx.x * kWarps + wib;
  int pj = -1, pb = 0, pn = 0;     // next document
  int pk[NW];
  float pc[NW];
  int cj, cn;                      // current document
  int ck[NW];
  float cc[NW];
  auto stage1 = [&](int64_t p) {
    pj = -1; pn = 0; pb = 0;
    if (p < pos1) {  // {document id, first nonzero, length, -} (a load that stays guarded)
      const int4 x = ldg_guarded(sdoc + p);
      pj = x.x; pb = x.y; pn = x.z;
    }
  };
  auto stage2 = [&]() {
#pragma unroll
    for (int w = 0; w < NW; ++w) {
      const int e = lane + 32 * w;
      int2 x = make_int2(0, 0);
      if (e < pn) x = ldg_guarded_stream(ent2 + pb + e, stream_pol);
      pk[w] = x.x;
      pc[w] = __int_as_float(x.y);   // 0 on rows past the document: v = 0 there
    }
  };
  auto stage3 = [&](const int (&ids)[NW], int nrows, int q) {
    const float* tab = qs.Mx + (size_t)q * qs.mx_stride;
#pragma unroll
    for (int w = 0; w < NW; ++w) {
      const int e = lane + 32 * w;
      if (e < nrows) {
        uint32_t k;  // opaque copy: keeps the address arithmetic (and its wait on the entry
        asm volatile("mov.b32 %0, %1;" : "=r"(k) : "r"(ids[w]));  // load) at this point
        const float* src = tab + (size_t)k * P;
        const uint32_t dst = smem_u32(buf0 + (cur ^ 1) * S::BUF + e * P);
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

  stage1(pos);
  stage2();
  stage3(pk, pn, 0);
  take_next_doc();
  int q = 0;

  while (pos < pos1) {
    cur ^= 1;      // this item's rows are in buffer cur; the next item's go to cur ^ 1
    const float* const buf = buf0 + cur * S::BUF;
    const int j = cj, n = cn;
    set_query(q);
    // c of the lane's own rows: row 32T + lane (full tiles), tail row 32NT + TW a + (b >> TSH)
    float c_own[NOWN];
    bool v_ok[NOWN];
#pragma unroll
    for (int T = 0; T < NT; ++T) {
      c_own[T] = cc[T];
      v_ok[T] = 32 * T + lane < n;
    }
    if constexpr (TW > 0) {
      const int tr = TW * a + (b >> S::TSH);
      c_own[NT] = __shfl_sync(kFull, cc[NT], tr);
      v_ok[NT] = 32 * NT + tr < n;
    }
    if (q == 0) stage1(pos + stride);   // the next document's header
    cp_async_wait_all();
    __syncwarp();

    // ---- block tile: D = M - m, mu = column minima over the document, Kh = 2^(-alpha (D - mu))
    float K[RW][CW];
    float u[CW];
    bool und;
    {
      float mu[CW];
#pragma unroll
      for (int c = 0; c < CW; ++c) mu[c] = INFINITY;
      // branch-free: rows past n read a staged row (stale contents); their D is +inf through the
      // per-row bias (so they drop out of the minima) and their Kh is set to 1 below
      bool rok[RW];
#pragma unroll
      for (int s = 0; s < RW; ++s) {
        const int e = row_of<NT, TW>(s, a, b);
        rok[s] = e < n;
        const float* row = buf + (rok[s] ? e : 0) * P;
        float x[CW];
        load_cols<CW>(row, b, x);
        const float bias = rok[s] ? -row[LD] : INFINITY;
#pragma unroll
        for (int c = 0; c < CW; ++c) {
          K[s][c] = x[c] + bias;   // D = M - m
          mu[c] = fminf(mu[c], K[s][c]);
        }
      }
#pragma unroll
      for (int c = 0; c < CW; ++c) {  // column minima over the 4 a-lanes (natural column order)
        mu[c] = fminf(mu[c], shx(mu[c], 8));
        mu[c] = fminf(mu[c], shx(mu[c], 16));
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
          // rows past n hold 1 (their c = 0 makes v = 0, and every row sum s stays positive);
          // padded columns keep their finite value (their uh = 0 cancels it everywhere)
          K[s][c] = rok[s] ? ex2_ftz(fmaf(-alpha, K[s][c], amu[c])) : 1.f;
          kmin[c] = fminf(kmin[c], K[s][c]);
        }
        to_slots<CW>(K[s], a);
      }
      bool flushed = false;   // a real entry flushed to 0 (true value < 2^-126)
#pragma unroll
      for (int c = 0; c < CW; ++c) flushed |= nreal[c] && kmin[c] < FLT_MIN;
      und = __any_sync(kFull, flushed);
      // uh0 = v_r 2^(-alpha mu) on real columns (slot order)
#pragma unroll
      for (int c = 0; c < CW; ++c) u[c] = nreal[c] ? (float)v_r * ex2_ftz(-alpha * mu[c]) : 0.f;
      to_slots<CW>(u, a);
    }
    if (q == nq - 1) stage2();   // the next document's entries (its header load was issued above)
    // the next item's rows: the same document for the next query, else the next document
    auto stage3_next = [&]() {
      if (q + 1 < nq) stage3(ck, n, q + 1);
      else stage3(pk, pn, 0);
    };

    // ---- iterations, then the final step
    float v_own[NOWN];
    bool bad = false;          // range certificate failed (blocks with flushed entries only)
    float umin = FLT_MAX;      // smallest real uh after a gauge: must stay normal
    uint32_t umax_all = 0u;    // largest uh before a gauge (bits): must stay finite
    bool done = false;         // "while x changes" (CONV)
    int it = 0;
    // The loop is instantiated twice: blocks without a flushed entry (the common case) carry no
    // certificate arithmetic; the stage-3 prefetch of the next document is peeled out of the
    // loop, so the loop body has no divergent branch.
    auto iterate = [&](auto und_tag) {
      constexpr bool UND = decltype(und_tag)::value;
      float umax_k = (float)v_r * kv_s;   // v_r * max(uh) * 2^-110 (max uh0 <= v_r)
      uint32_t vmax_b = 0u;
      // SDDMM: row partials over this lane's columns, the reduce over the b-lanes, v = c / s
      auto row_step = [&]() {
        float p[RW];
#pragma unroll
        for (int s = 0; s < RW; ++s) {
          float acc = K[s][0] * u[0];
#pragma unroll
          for (int c = 1; c < CW; ++c) acc = fmaf(K[s][c], u[c], acc);
          p[s] = acc;
        }
        reduce_rows<NT, TW>(p);
        vmax_b = 0u;
#pragma unroll
        for (int o = 0; o < NOWN; ++o) {
          const float sv = p[8 * o];
          v_own[o] = c_own[o] * rcp_fast(sv);
          if constexpr (UND) {
            bad |= v_ok[o] && umax_k > sv;
            vmax_b = max(vmax_b, __float_as_uint(v_own[o]));
          }
        }
      };
      // SpMM: column partials over this lane's rows, the reduce over the a-lanes, u = r / acc,
      // the exact power-of-two gauge, redistribution of u to the column slots
      auto col_step = [&]() {
        float vcap = 0.f;
        if constexpr (UND) vcap = (float)n * __uint_as_float(__reduce_max_sync(kFull, vmax_b)) * kUnder;
        float vs[RW];
#pragma unroll
        for (int T = 0; T < NT; ++T) {
          vs[8 * T] = v_own[T];
#pragma unroll
          for (int t = 1; t < 8; ++t) vs[8 * T + t] = shx(v_own[T], t);
        }
        if constexpr (TW > 0) {
          vs[8 * NT] = v_own[NT];
#pragma unroll
          for (int t = 1; t < TW; ++t) vs[8 * NT + t] = shx(v_own[NT], t << S::TSH);
        }
        float q[CW];
#pragma unroll
        for (int c = 0; c < CW; ++c) {
          float q0 = K[0][c] * vs[0];
#pragma unroll
          for (int s = 1; s < RW; ++s) q0 = fmaf(K[s][c], vs[s], q0);
          q[c] = q0;
        }
        reduce_cols<CW>(q);
        uint32_t umax_b = 0u, chg_b = 0u;
        float uo[NCO];
#pragma unroll
        for (int g = 0; g < NCO; ++g) {
          const int qs = CW >= 3 && g >= CQ ? 4 * CQ + (g - CQ) : 4 * g;  // slot of own column g
          const float acc = q[qs];
          uo[g] = r_own[g] * rcp_fast(acc);
          // "while x changes" (NEXT-3): |x_new/x - 1| = |uh/uh_new - 1| (gauge invariant; the
          // own column's current uh sits in column slot qs); NaN compares above every float
          if (CONV && oreal[g]) chg_b = max(chg_b, __float_as_uint(fabsf(u[qs] / uo[g] - 1.f)));
          if constexpr (UND) bad |= vcap > acc;
          umax_b = max(umax_b, __float_as_uint(uo[g]));
        }
        // gauge: max uh -> [1, 2) by an exact power of two (positive floats order like their bits)
        umax_b = __reduce_max_sync(kFull, umax_b);
        umax_all = max(umax_all, umax_b);
        if (CONV) done = __uint_as_float(__reduce_max_sync(kFull, chg_b)) <= tol;
        const float sc = __uint_as_float((254u - min(umax_b >> 23, 253u)) << 23);
        if constexpr (UND) umax_k = 2.f * kv_s;
#pragma unroll
        for (int g = 0; g < NCO; ++g) {
          uo[g] *= sc;
          umin = fminf(umin, oreal[g] ? uo[g] : 1.f);
        }
        if constexpr (CW >= 3) {
#pragma unroll
          for (int g = 0; g < CQ; ++g) {
            u[4 * g] = uo[g];
#pragma unroll
            for (int c = 1; c < 4; ++c) u[4 * g + c] = shx(uo[g], 8 * c);
          }
#pragma unroll
          for (int r = 0; r < CR; ++r) u[4 * CQ + r] = uo[CQ + r];
        } else if constexpr (CW == 2) {
          u[0] = uo[0];
          u[1] = shx(uo[0], 16);
        } else {
          u[0] = uo[0];
        }
      };
      row_step();
      if (iters > 0) {
        col_step();
        it = 1;
        row_step();
        stage3_next();  // the next document's entries have landed: start its row copies
        while (it != iters && !(CONV && done)) {
          col_step();
          ++it;
          row_step();
        }
      } else {
        stage3_next();
      }
    };
    if (und) iterate(std::true_type{});
    else iterate(std::false_type{});

    // ---- final step: WMD_j = sum_e vh_e q_e,  q_e = sum_i Kh_ei M_ie uh_i, with
    // M read back from the document's staged rows (still in buffer cur): each slot's column is
    // read directly at its XOR-permuted position (col_of), matching Kh and uh slot by slot.
    // (rows past n read a staged row and are left out of the sum below)
    float p[RW];
#pragma unroll
    for (int s = 0; s < RW; ++s) {
      const float* row = buf + row_of<NT, TW>(s, a, b) * P;
      float acc = 0.f;
#pragma unroll
      for (int c = 0; c < CW; ++c) acc = fmaf(K[s][c] * u[c], row[col_of<CW>(c, a, b)], acc);
      p[s] = acc;
    }
    reduce_rows<NT, TW>(p);
    float wsum = 0.f;
#pragma unroll
    for (int T = 0; T < NT; ++T)
      if (v_ok[T]) wsum = fmaf(v_own[T], p[8 * T], wsum);
    if constexpr (TW > 0) {  // each tail row is held by 2^TSH lanes: count it once
      if (v_ok[NT] && (b & ((1 << S::TSH) - 1)) == 0) wsum = fmaf(v_own[NT], p[8 * NT], wsum);
    }
#pragma unroll
    for (int off = 16; off; off >>= 1) wsum += shx(wsum, off);
    const bool flag = __any_sync(kFull, bad || !(umin >= FLT_MIN)) || umax_all > 0x7f7fffffu ||
                      !(fabsf(wsum) <= FLT_MAX);
    if (lane == 0) {
      const int64_t o = (int64_t)q * qs.N + j;
      qs.dist[out0 + j] = wsum;
      if (qs.iters_doc) qs.iters_doc[o] = it;
      uint8_t f = und ? kFlagUnderflow : 0;
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
  cp_async_wait_all();  // nothing may be in flight when the warp exits
}

template <int CW, int NT, int TW, bool CONV>
void launch_fused_range_t(const int4* sdoc, const Entry* ent, int64_t p0, int64_t p1, const QuerySet& qs,
                          float lambda, int iters, float tol, cudaStream_t st) {
  if (p1 <= p0) return;
  constexpr size_t smem = sizeof(float) * Shape<CW, NT, TW>::BUF * kWarps * 2;  // two row buffers per warp
  static PerDevice cache;
  const int resident = cache.get([&] {
    cudaFuncSetAttribute(sinkhorn_fused_kernel<CW, NT, TW, CONV>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(sinkhorn_fused_kernel<CW, NT, TW, CONV>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, sinkhorn_fused_kernel<CW, NT, TW, CONV>, kThreads, smem);
    return std::max(1, per_sm) * device_sms();
  });
  const int64_t need = (p1 - p0 + kWarps - 1) / kWarps;
  const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>(need, resident));
  sinkhorn_fused_kernel<CW, NT, TW, CONV><<<grid, kThreads, smem, st>>>(sdoc, ent, p0, p1, qs, lambda, iters, tol);
}

template <int CW, int NT, int TW>
void launch_fused_range(const int4* sdoc, const Entry* ent, int64_t p0, int64_t p1, const QuerySet& qs,
                        float lambda, int iters, float tol, cudaStream_t st) {
  if (tol >= 0.f)
    launch_fused_range_t<CW, NT, TW, true>(sdoc, ent, p0, p1, qs, lambda, iters, tol, st);
  else
    launch_fused_range_t<CW, NT, TW, false>(sdoc, ent, p0, p1, qs, lambda, iters, tol, st);
}

// Length buckets (rows covered: 8, 16, 32, 40, 48, 64) over the length-sorted order.
struct Bucket { int ne, nt, tw; };
constexpr Bucket kBuckets[] = {{8, 0, 2}, {16, 0, 4}, {32, 1, 0}, {40, 1, 2}, {48, 1, 4}, {64, 2, 0}};
constexpr int kNumBuckets = 6;

constexpr bool fits(int cw, int ne) { return (ne / 4) * cw <= 96; }  // block registers per lane

template <int CW>
void dispatch_bucket(int bi, const int4* sdoc, const Entry* ent, int64_t p0, int64_t p1, const QuerySet& qs,
                     float lambda, int iters, float tol, cudaStream_t st) {
#define F_(NT, TW) \
  if constexpr (fits(CW, 32 * NT + 4 * TW)) launch_fused_range<CW, NT, TW>(sdoc, ent, p0, p1, qs, lambda, iters, tol, st)
  switch (bi) {
    case 0: F_(0, 2); break;
    case 1: F_(0, 4); break;
    case 2: F_(1, 0); break;
    case 3: F_(1, 2); break;
    case 4: F_(1, 4); break;
    default: F_(2, 0); break;
  }
#undef F_
}

}  // namespace

// Longest document the one-warp kernel takes at row width ld (0: none).
int warp_max_rows(int ld) {
  int best = 0;
  for (int b = 0; b < kNumBuckets; ++b)
    if (fits(ld / 8, kBuckets[b].ne)) best = kBuckets[b].ne;
  return ld <= 64 ? best : 0;
}

int fused_ld(int v_r, int64_t max_doc_nnz, bool conv) {
  // one-warp kernel: 8 CW columns, CW in {1, 2, 3, 4, 5, 6, 8}
  int ld = 0;
  for (int cw : {1, 2, 3, 4, 5, 6, 8})
    if (8 * cw >= v_r) { ld = 8 * cw; break; }
  if (const char* e = std::getenv("WMD_LD_OVERRIDE")) {   // measurement knob: a wider table
    const int w = std::atoi(e);
    if (w >= ld && w <= 64 && w % 8 == 0 && !conv) ld = w;
  }
  if (ld && max_doc_nnz <= warp_max_rows(ld)) return ld;
  // longer documents (or v_r > 64): one CTA per document (wmd_fused_cta.cu; fixed iteration
  // count), whose table width the one-warp kernel then shares for the shorter documents
  if (v_r > 128 || conv || max_doc_nnz > cta_max_rows()) return 0;
  return cta_ld(v_r);
}

bool use_half(int ld, float tol, int64_t layout_docs) {
  // WMD_FUSED_HALF: "0" never, "1" always (where the shape allows), unset: large corpora only
  // (a few thousand documents leave most of the GPU idle at two documents per warp: Tweet's
  // fused phase 0.036 ms one-warp vs 0.043 half-warp; Scaling 8.08 vs 7.36 ms)
  const char* e = std::getenv("WMD_FUSED_HALF");
  const bool shape = (ld == 16 || ld == 24 || ld == 32 || ld == 40) && tol < 0.f;
  if (e && e[0] == '0') return false;
  if (e && e[0] == '1') return shape;
  return shape && layout_docs >= kHalfMinDocs;
}

void launch_sinkhorn_fused(const int4* sdoc, const Entry* ent, int64_t N, int64_t layout_docs,
                           const int64_t* len_prefix, int64_t max_len, int ld, const QuerySet& qs,
                           float lambda, int iters, float tol, cudaStream_t st0, StreamRing* ring) {
  // len_prefix[L] = number of documents with fewer than L nonzeros: the length-sorted order
  // splits into buckets of at most 8 / 16 / 32 / 40 / 48 / 64 nonzeros (one-warp kernel, one
  // launch each) and, past warp_max_rows(ld), 64 / 128 / ... / 320 (one-CTA kernel, one query).
  const int wmax = warp_max_rows(ld);
  // documents of at most half_max_rows() nonzeros: two per warp (wmd_fused_half.cu)
  int64_t p0 = use_half(ld, tol, layout_docs) ? launch_sinkhorn_half(sdoc, ent, N, len_prefix, max_len, ld, qs, lambda, iters,
                                                        st0, ring, nullptr)
                                 : 0;
  for (int bi = 0; bi < kNumBuckets && p0 < N && kBuckets[bi].ne <= wmax; ++bi) {
    const int NE = kBuckets[bi].ne;
    const int64_t p1 = NE >= max_len ? N : len_prefix[NE + 1];
    if (p1 > p0) {
      const cudaStream_t st = ring ? ring->next(st0) : st0;
      switch (ld) {
        case 8: dispatch_bucket<1>(bi, sdoc, ent, p0, p1, qs, lambda, iters, tol, st); break;
        case 16: dispatch_bucket<2>(bi, sdoc, ent, p0, p1, qs, lambda, iters, tol, st); break;
        case 24: dispatch_bucket<3>(bi, sdoc, ent, p0, p1, qs, lambda, iters, tol, st); break;
        case 32: dispatch_bucket<4>(bi, sdoc, ent, p0, p1, qs, lambda, iters, tol, st); break;
        case 40: dispatch_bucket<5>(bi, sdoc, ent, p0, p1, qs, lambda, iters, tol, st); break;
        case 48: dispatch_bucket<6>(bi, sdoc, ent, p0, p1, qs, lambda, iters, tol, st); break;
        case 64: dispatch_bucket<8>(bi, sdoc, ent, p0, p1, qs, lambda, iters, tol, st); break;
        default: break;
      }
    }
    p0 = std::max(p0, p1);
  }
  if (p0 < N && qs.nq == 1)
    launch_sinkhorn_cta(sdoc, ent, p0, N, len_prefix, max_len, qs.Mx, ld, qs.v_r, qs.rpad, lambda, iters,
                        qs.iters_doc, qs.dist, qs.flags, qs.flagged_list, qs.flagged_count, st0, ring);
}

int fused_launch_count(const int64_t* len_prefix, int64_t max_len, int64_t N, int64_t layout_docs, int ld,
                       float tol) {
  const int wmax = warp_max_rows(ld);
  int cnt = 0;
  const int64_t p0h = use_half(ld, tol, layout_docs) ? launch_sinkhorn_half(nullptr, nullptr, N, len_prefix, max_len, ld,
                                                               QuerySet{}, 0.f, 0, nullptr, nullptr, &cnt)
                                        : 0;
  int64_t p0 = p0h;
  for (int bi = 0; bi < kNumBuckets && p0 < N && kBuckets[bi].ne <= wmax; ++bi) {
    const int64_t p1 = kBuckets[bi].ne >= max_len ? N : len_prefix[kBuckets[bi].ne + 1];
    cnt += p1 > p0;
    p0 = std::max(p0, p1);
  }
  return cnt + (p0 < N ? cta_launch_count(p0, N, len_prefix, max_len) : 0);
}

}  // namespace wmd
