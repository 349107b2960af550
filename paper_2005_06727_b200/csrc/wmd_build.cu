// wmd_build.cu — a2: query x vocabulary distances (§6 :259-268).
//
// Per vocabulary word k and query row i (sel = the query's word ids, ascending):
//     M_ik  = sqrt(sum_t (E[sel_i,t] - E[k,t])^2)   direct difference in FP32, so M_{i,sel_i} == 0
//                                                   exactly (no |a|^2 + |b|^2 - 2ab cancellation:
//                                                   exp(-lambda M) amplifies absolute errors)
//     m_k   = min_i M_ik
//     Mx_k  = [M_k0 .. M_k,ld-1 (zero beyond v_r), m_k, 0, 0, 0]        (ld + 4 floats)
//     K~_ki = expf(-lambda (M_ik - m_k))            (ld floats; only when the per-iteration path
//                                                   runs)
// E is stored with rows padded to dp (a multiple of 32) floats of zeros, which add nothing.
//
// Mapping: a block owns 256 vocabulary words x 8 RB query rows per pass (RB <= 6 chosen per
// query so that the passes cover v_r with at most 7 padded rows each) and streams d in chunks of
// 32 through shared memory with cp.async, double buffered. Thread micro-tile: RB query rows x 8
// words = 8 RB independent accumulators; per d-quad a thread issues RB + 8 LDS.128 (RB
// warp-broadcast query quads, 8 conflict-free word quads) for 64 RB FP32 instructions (FADD +
// FFMA per (i, k, t) triple). Bound: FP32 issue, 2 instructions per triple (PAPER.md:260 counts
// 3 flops), E read once per pass from HBM.
#include <algorithm>
#include <cfloat>
#include <cmath>
#include <cstdint>

#include "wmd_internal.h"
#include "wmd_umma.cuh"

namespace wmd {
namespace {

using umma::su32;
using umma::mbar_wait;
using umma::tmem_ld32;

constexpr int BW = 256;        // vocabulary words per block (tensor-core variant, SIMT default)
constexpr int BD = 32;         // d chunk
constexpr int BP = BD + 4;     // smem pitch of a staged row (floats)
constexpr int kThreads = 256;
constexpr int kMaxRB = 6;      // query rows per thread and pass (8 RB rows per pass)

// query rows + words of one pipeline stage (NWT words per thread: 32 NWT words per block)
template <int RB, int NWT> constexpr int stage_floats() { return 8 * RB * BP + 32 * NWT * BP; }

__device__ __forceinline__ void cp16(float* dst, const float* src, bool valid) {
  const uint32_t d = static_cast<uint32_t>(__cvta_generic_to_shared(dst));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(d), "l"(src), "r"(valid ? 16 : 0)
               : "memory");
}

// RB: query rows per thread and pass; a pass covers BI = 8 RB query rows (the host picks the
// smallest RB whose passes cover v_r: v_r = 15 -> one pass of 16, 30 -> 32, 40 -> 40,
// 100 -> three of 40), so a pass wastes at most 7 padded rows.
// NWT: words per thread (8: 256 words per block; 4: 128, for small vocabularies, where 256-word
// blocks leave the last wave mostly empty).
template <int RB, int NWT>
__global__ void __launch_bounds__(kThreads, NWT == 4 ? 3 : 2) build_mx_kernel(
    const float* __restrict__ E, int64_t row0, int64_t V, int dp, const int32_t* __restrict__ sel,
    int v_r, int ld, float lambda, float* __restrict__ Kt, float* __restrict__ Mx) {
  constexpr int BI = 8 * RB;
  constexpr int BWW = 32 * NWT;            // words per block
  constexpr int STAGE = stage_floats<RB, NWT>();
  constexpr int MSP = BI + 1;              // pitch of the M tile of a pass in shared memory
  extern __shared__ __align__(16) float smem[];  // two pipeline stages of STAGE floats
  __shared__ float cmin[BWW];
  const int tid = threadIdx.x, tw = tid & 31, ti = tid >> 5;
  const int64_t k0 = row0 + (int64_t)blockIdx.x * BWW;  // rows [row0, V) of this launch
  const int nchunk = dp / BD;
  const int ldx = ld + 4;
  for (int w = tid; w < BWW; w += kThreads) cmin[w] = FLT_MAX;

  for (int i0 = 0; i0 < v_r; i0 += BI) {
    // stage one d chunk: BI query rows + BWW words, one 16 B copy per (row, 4 floats)
    auto issue = [&](int c, float* buf) {
      for (int x = tid; x < BI * 8; x += kThreads) {
        const int r = x >> 3, t4 = x & 7;
        const bool ok = i0 + r < v_r;
        const int64_t row = ok ? sel[i0 + r] : 0;
        cp16(buf + r * BP + 4 * t4, E + row * dp + c * BD + 4 * t4, ok);
      }
      const int t4 = tid & 7;
#pragma unroll
      for (int q = 0; q < BWW / 32; ++q) {
        const int w = (tid >> 3) + 32 * q;            // 0..BWW-1
        const bool ok = k0 + w < V;
        cp16(buf + BI * BP + w * BP + 4 * t4, E + (ok ? k0 + w : 0) * dp + c * BD + 4 * t4, ok);
      }
      asm volatile("cp.async.commit_group;" ::: "memory");
    };
    float acc[RB][NWT];
#pragma unroll
    for (int r = 0; r < RB; ++r)
#pragma unroll
      for (int s = 0; s < NWT; ++s) acc[r][s] = 0.f;
    issue(0, smem);
    for (int c = 0; c < nchunk; ++c) {
      if (c + 1 < nchunk) {
        issue(c + 1, smem + ((c + 1) & 1) * STAGE);
        asm volatile("cp.async.wait_group 1;" ::: "memory");
      } else {
        asm volatile("cp.async.wait_group 0;" ::: "memory");
      }
      __syncthreads();
      const float* Qs = smem + (c & 1) * STAGE;
      const float* Es = Qs + BI * BP;
#pragma unroll 2
      for (int t = 0; t < BD; t += 4) {
        float4 q[RB], e[NWT];
#pragma unroll
        for (int r = 0; r < RB; ++r) q[r] = *reinterpret_cast<const float4*>(Qs + (ti + 8 * r) * BP + t);
#pragma unroll
        for (int s = 0; s < NWT; ++s) e[s] = *reinterpret_cast<const float4*>(Es + (tw + 32 * s) * BP + t);
#pragma unroll
        for (int r = 0; r < RB; ++r)
#pragma unroll
          for (int s = 0; s < NWT; ++s) {
            float df;
            df = q[r].x - e[s].x; acc[r][s] = fmaf(df, df, acc[r][s]);
            df = q[r].y - e[s].y; acc[r][s] = fmaf(df, df, acc[r][s]);
            df = q[r].z - e[s].z; acc[r][s] = fmaf(df, df, acc[r][s]);
            df = q[r].w - e[s].w; acc[r][s] = fmaf(df, df, acc[r][s]);
          }
      }
      __syncthreads();  // the stage is refilled by the next iteration's issue
    }
    // epilogue of this pass: M tile through shared memory (the staging buffers are idle)
    float* Ms = smem;  // [BWW][MSP]
#pragma unroll
    for (int r = 0; r < RB; ++r)
#pragma unroll
      for (int s = 0; s < NWT; ++s) Ms[(tw + 32 * s) * MSP + ti + 8 * r] = sqrtf(acc[r][s]);
    __syncthreads();
    // warp per word: lane l owns query rows i0 + l and i0 + 32 + l (coalesced row writes)
    const int warp = tid >> 5, lane = tid & 31;
    const bool last = i0 + BI >= v_r;
    for (int w = warp; w < BWW; w += kThreads / 32) {
      const int64_t k = k0 + w;
      if (k >= V) break;
      float mn = FLT_MAX;
#pragma unroll
      for (int h = 0; h < (BI + 31) / 32; ++h) {
        const int x = 32 * h + lane;
        if (x < BI && i0 + x < v_r) {
          const float m = Ms[w * MSP + x];
          mn = fminf(mn, m);
          Mx[k * ldx + i0 + x] = m;
        }
      }
#pragma unroll
      for (int off = 16; off; off >>= 1) mn = fminf(mn, __shfl_xor_sync(0xffffffffu, mn, off));
      mn = fminf(mn, cmin[w]);
      __syncwarp();
      if (!last) {
        if (lane == 0) cmin[w] = mn;
        continue;
      }
      // row complete: zero padding, m_k, and K~ (reading back earlier passes' M from Mx)
      for (int x = v_r + lane; x < ldx; x += 32) Mx[k * ldx + x] = x == ld ? mn : 0.f;
      if (Kt) {
        for (int x = lane; x < ld; x += 32) {
          float kt = 0.f;
          if (x < v_r) kt = expf(-lambda * ((x >= i0 ? Ms[w * MSP + x - i0] : Mx[k * ldx + x]) - mn));
          Kt[k * ld + x] = kt;
        }
      }
    }
    __syncthreads();  // Ms aliases the staging buffers of the next pass
  }
}

// ============================================================================================
// Tensor-core variant (NEXT-4, "GEMM-like" distance): the cross term of
//     M_ik^2 = |E_k|^2 + |q_i|^2 - 2 E_k . q_i
// on the 5th-generation tensor cores in 3xTF32 (exact-FP32 emulation: x = hi + lo with hi the
// TF32 truncation; E.q ~ hi.hi + hi.lo + lo.hi, the lo.lo term below FP32 rounding), FP32
// accumulation in TMEM. The norms are FP32 sums of the same staged values. Cancellation: where
// M^2 < kNearFrac (|E_k|^2 + |q_i|^2) the distance is recomputed by direct difference (and
// M_{i,sel_i} = 0 exactly), so near-duplicate words keep the direct-difference accuracy that
// exp(-lambda M) needs.
//
// Block: 128 threads, 128 vocabulary rows (TMEM lanes) x NP query rows (TMEM columns, NP = v_r
// rounded up to 32, <= 128). d streams in 32-float chunks, double buffered with cp.async
// straight into the K-major no-swizzle core-matrix layout the MMA descriptors read (8 rows x
// 16 B per core matrix); the threads add the lo parts and the squared norms; one elected thread
// issues 12 tcgen05.mma (M=128, N=NP, K=8) per chunk and commits them to the stage's mbarrier.
// Epilogue: tcgen05.ld of each thread's accumulator row (row = TMEM lane), sqrt, column minimum,
// Mx / K~ rows. Bound: reading E once from HBM (the MMAs need ~2 % of the tensor peak).
// ============================================================================================
constexpr int TC_M = 128;             // vocabulary rows per block (MMA M, TMEM lanes)
// d chunk (floats) and layout per query-tile width: swizzled 32-float chunks up to
// WMD_TC_SWZ_MAX query rows, no-swizzle 16-float chunks beyond (shared memory per stage)
#ifndef WMD_TC_SWZ_MAX
#define WMD_TC_SWZ_MAX 128
#endif
#ifndef WMD_TC_SWZ_BYTES  // swizzle span of the swizzled layout: 128 (32-float chunks) or 64 (16)
#define WMD_TC_SWZ_BYTES 64
#endif
template <int NP> constexpr int tc_swz() { return NP <= WMD_TC_SWZ_MAX ? WMD_TC_SWZ_BYTES : 0; }
template <int NP> constexpr int tc_k() { return tc_swz<NP>() ? tc_swz<NP>() / 4 : 16; }
#ifndef WMD_TC_STAGES
#define WMD_TC_STAGES 3
#endif
#ifndef WMD_TC_LO
#define WMD_TC_LO 2
#endif
constexpr int TC_NS = WMD_TC_STAGES;  // raw-chunk ring stages
constexpr int TC_LO = WMD_TC_LO;      // lo-part buffers = how many chunks back the MMA wait is
constexpr float kNearFrac = 1.0f / 64.f;

// byte offset of element (r, k) (k < 32) in a K-major no-swizzle tile of R rows: core matrices
// of 8 rows x 4 floats; SBO = 128 B between 8-row groups, LBO = R/8 * 128 B between K quads
// Operand layouts (K-major). SWZ = 64 (default): SWIZZLE_64B with 16-float chunks (one 64-byte
// row): 8-row atoms of 512 B, piece j of row r stored at piece j ^ ((r >> 1) % 4); SWZ = 128:
// SWIZZLE_128B with 32-float chunks, 1024-B atoms, piece j at j ^ (r % 8) (the tensor core undoes
// the XOR; conflict-free either way); SWZ = 0: the no-swizzle core-matrix layout (8 rows x 16 B,
// SBO = 128 B, LBO = R / 8 * 128 B), which measured slowest. The 64-byte chunks halve the shared
// memory per stage: four 32-query-row blocks per SM (latency-bound on the MMA-completion wait,
// so occupancy is what counts: Scaling 0.30 (no swizzle) -> 0.26 (128 B) -> 0.19 ms (64 B)).
template <int SWZ>
__device__ __forceinline__ uint32_t km_off(int r, int k, int R) {
  if constexpr (SWZ == 128) return (uint32_t)((r >> 3) * 1024 + (r & 7) * 128 + ((((k >> 2) ^ r) & 7) << 4) + (k & 3) * 4);
  // SWIZZLE_64B: 64-byte rows, 8-row atoms of 512 B, piece j of row r at j ^ ((r >> 1) & 3)
  else if constexpr (SWZ == 64) return (uint32_t)((r >> 3) * 512 + (r & 7) * 64 + ((((k >> 2) ^ (r >> 1)) & 3) << 4) + (k & 3) * 4);
  else return (uint32_t)((k >> 2) * (R / 8 * 128) + (r >> 3) * 128 + (r & 7) * 16 + (k & 3) * 4);
}
__device__ __forceinline__ void mma_tf32(uint32_t tmem, uint64_t da, uint64_t db, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n"
      ::"r"(tmem), "l"(da), "l"(db), "r"(idesc), "r"(acc));
}
template <int NP>
__global__ void __launch_bounds__(128, NP <= 32 ? (WMD_TC_SWZ_BYTES == 64 ? 4 : 2) : (NP <= 64 && WMD_TC_SWZ_MAX >= 64 ? 2 : 1)) build_mx_tc_kernel(
    const float* __restrict__ E, int64_t row0, int64_t V, int dp, const int32_t* __restrict__ sel,
    int v_r, int ld, float lambda, float* __restrict__ Kt, float* __restrict__ Mx) {
  constexpr int SWZ = tc_swz<NP>();
  constexpr int TC_K = tc_k<NP>();
  constexpr int A_BYTES = TC_M * TC_K * 4, B_BYTES = NP * TC_K * 4;
  constexpr int STAGE = A_BYTES + B_BYTES;                  // one chunk: A rows, then B rows
  constexpr uint32_t TMEM_COLS = NP <= 32 ? 32 : (NP <= 64 ? 64 : 128);
  constexpr uint32_t IDESC = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(NP >> 3) << 17) |
                             ((uint32_t)(TC_M >> 4) << 24);   // F32 += TF32 x TF32, K-major both
  extern __shared__ __align__(1024) uint8_t tc_smem[];
  // operand tiles at a 1024-byte aligned base (the swizzle atoms); 1 KB of slack is allocated
  uint8_t* smem = tc_smem + ((1024u - (su32(tc_smem) & 1023u)) & 1023u);  // [TC_NS][STAGE]: raw (= hi)
  uint8_t* lo_buf = smem + TC_NS * STAGE;                   // [TC_LO][STAGE]: their lo parts
  __shared__ uint32_t tmem_base;
  __shared__ __align__(8) uint64_t mbar[TC_NS];
  __shared__ float qn[NP];
  __shared__ int32_t qsel[NP];
  const int tid = threadIdx.x, warp = tid >> 5;
  const int64_t k0 = row0 + (int64_t)blockIdx.x * TC_M;  // rows [row0, V) of this launch
  const int nchunk = dp / TC_K;
  const int ldx = ld + 4;
  if (tid < NP) qsel[tid] = tid < v_r ? sel[tid] : -1;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(&tmem_base)), "n"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    for (int i = 0; i < TC_NS; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&mbar[i])), "r"(1));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tm = tmem_base;

  // raw chunk copies: A rows k0 + r (zero past V), B rows = the query rows (zero past v_r)
  auto issue = [&](int c, int st) {
    uint8_t* base = smem + st * STAGE;
    for (int p = tid; p < TC_M * (TC_K / 4); p += 128) {
      const int r = p / (TC_K / 4), q = p % (TC_K / 4);
      const bool ok = k0 + r < V;
      const float* src = E + (ok ? k0 + r : 0) * (int64_t)dp + c * TC_K + 4 * q;
      const uint32_t dst = su32(base + km_off<SWZ>(r, 4 * q, TC_M));
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(ok ? 16 : 0) : "memory");
    }
    for (int p = tid; p < NP * (TC_K / 4); p += 128) {
      const int r = p / (TC_K / 4), q = p % (TC_K / 4);
      const int row = qsel[r];
      const float* src = E + (row >= 0 ? row : 0) * (int64_t)dp + c * TC_K + 4 * q;
      const uint32_t dst = su32(base + A_BYTES + km_off<SWZ>(r, 4 * q, NP));
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(row >= 0 ? 16 : 0) : "memory");
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  __syncthreads();  // qsel
  float en = 0.f, qq = 0.f;   // |E_row|^2 of this thread's vocabulary row; |q|^2 (tid < NP)
  // Raw chunks land AHEAD = TC_NS - TC_LO chunks ahead in a TC_NS-stage ring (the raw copy is
  // also the hi operand: the tensor core reads TF32 from the FP32 bits); the lo parts go to a
  // TC_LO-deep buffer. Ring stage (c + AHEAD) % TC_NS and lo buffer c % TC_LO are free once the
  // MMAs of chunk c - TC_LO retired: waiting TC_LO chunks back hides the MMA completion latency.
  constexpr int AHEAD = TC_NS - TC_LO;
  static_assert(AHEAD >= 1, "ring deeper than the lo buffer");
  for (int c = 0; c < AHEAD; ++c) {
    if (c < nchunk) issue(c, c);
    else asm volatile("cp.async.commit_group;" ::: "memory");
  }
  for (int c = 0; c < nchunk; ++c) {
    const int st = c % TC_NS;
    if (c >= TC_LO) mbar_wait(su32(&mbar[(c - TC_LO) % TC_NS]), ((c - TC_LO) / TC_NS) & 1);
    const int cn = c + AHEAD;
    if (cn < nchunk) issue(cn, cn % TC_NS);
    else asm volatile("cp.async.commit_group;" ::: "memory");
    asm volatile("cp.async.wait_group %0;" ::"n"(AHEAD) : "memory");  // chunk c has landed
    __syncthreads();
    uint8_t* base = smem + st * STAGE;
    uint8_t* lob = lo_buf + (c % TC_LO) * STAGE;
    // lo parts and norms: thread tid owns vocabulary row tid (and query row tid < NP)
#pragma unroll
    for (int q = 0; q < TC_K / 4; ++q) {
      const uint32_t off = km_off<SWZ>(tid, 4 * q, TC_M);
      const float4 x = *reinterpret_cast<const float4*>(base + off);
      en = fmaf(x.x, x.x, en); en = fmaf(x.y, x.y, en); en = fmaf(x.z, x.z, en); en = fmaf(x.w, x.w, en);
      float4 lo;
      lo.x = x.x - __uint_as_float(__float_as_uint(x.x) & 0xffffe000u);
      lo.y = x.y - __uint_as_float(__float_as_uint(x.y) & 0xffffe000u);
      lo.z = x.z - __uint_as_float(__float_as_uint(x.z) & 0xffffe000u);
      lo.w = x.w - __uint_as_float(__float_as_uint(x.w) & 0xffffe000u);
      *reinterpret_cast<float4*>(lob + off) = lo;
    }
    if (tid < NP) {
#pragma unroll
      for (int q = 0; q < TC_K / 4; ++q) {
        const uint32_t off = A_BYTES + km_off<SWZ>(tid, 4 * q, NP);
        const float4 x = *reinterpret_cast<const float4*>(base + off);
        qq = fmaf(x.x, x.x, qq); qq = fmaf(x.y, x.y, qq); qq = fmaf(x.z, x.z, qq); qq = fmaf(x.w, x.w, qq);
        float4 lo;
        lo.x = x.x - __uint_as_float(__float_as_uint(x.x) & 0xffffe000u);
        lo.y = x.y - __uint_as_float(__float_as_uint(x.y) & 0xffffe000u);
        lo.z = x.z - __uint_as_float(__float_as_uint(x.z) & 0xffffe000u);
        lo.w = x.w - __uint_as_float(__float_as_uint(x.w) & 0xffffe000u);
        *reinterpret_cast<float4*>(lob + off) = lo;
      }
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic writes -> tensor core
    __syncthreads();
    if (tid == 0) {
      asm volatile("tcgen05.fence::after_thread_sync;");
      const uint32_t a_hi = su32(base), a_lo = su32(lob);
      const uint32_t b_hi = a_hi + A_BYTES, b_lo = a_lo + A_BYTES;
#pragma unroll
      for (int pass = 0; pass < 3; ++pass) {          // hi.hi + hi.lo + lo.hi
        const uint32_t a = pass == 2 ? a_lo : a_hi, b = pass == 1 ? b_lo : b_hi;
#pragma unroll
        for (int kk = 0; kk < TC_K; kk += 8) {
          uint64_t da, db;
          if constexpr (SWZ == 128) {
            da = umma::desc_sw128(a + 4 * kk);
            db = umma::desc_sw128(b + 4 * kk);
          } else if constexpr (SWZ == 64) {
            da = umma::desc_sw64(a + 4 * kk);
            db = umma::desc_sw64(b + 4 * kk);
          } else {
            da = umma::desc(a + (kk >> 2) * (TC_M / 8 * 128), TC_M / 8 * 128, 128);
            db = umma::desc(b + (kk >> 2) * (NP / 8 * 128), NP / 8 * 128, 128);
          }
          mma_tf32(tm, da, db, IDESC, (c | pass | kk) ? 1u : 0u);
        }
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&mbar[st])));
    }
  }
  if (tid < NP) qn[tid] = qq;
  // the last chunk's commit also covers every earlier MMA
  mbar_wait(su32(&mbar[(nchunk - 1) % TC_NS]), ((nchunk - 1) / TC_NS) & 1);
  asm volatile("tcgen05.fence::after_thread_sync;");
  __syncthreads();  // qn

  // ---- epilogue: thread tid = vocabulary row k0 + tid = TMEM lane tid
  const int64_t k = k0 + tid;
  const bool kok = k < V;
  float Mrow[NP];
  uint32_t near[(NP + 31) / 32];
#pragma unroll
  for (int c0 = 0; c0 < NP; c0 += 32) {
    float dot[32];
    tmem_ld32(tm + ((uint32_t)(warp * 32) << 16) + (uint32_t)c0, dot);
    uint32_t nb = 0u;
#pragma unroll
    for (int c = 0; c < 32; ++c) {
      const float m2 = fmaxf(en + qn[c0 + c] - 2.f * dot[c], 0.f);
      Mrow[c0 + c] = sqrtf(m2);
      if (c0 + c < v_r && m2 < kNearFrac * (en + qn[c0 + c])) nb |= 1u << c;
    }
    near[c0 / 32] = nb;
  }
  if (kok) {
    // cancellation-prone pairs (rare; M_{i,sel_i} among them): direct difference
#pragma unroll
    for (int w = 0; w < (NP + 31) / 32; ++w) {
      for (uint32_t nb = near[w]; nb; nb &= nb - 1) {
        const int i = 32 * w + __ffs(nb) - 1;
        const float* er = E + k * (int64_t)dp;
        const float* qr = E + (int64_t)qsel[i] * dp;
        float s2 = 0.f;
        for (int t = 0; t < dp; ++t) { const float df = qr[t] - er[t]; s2 = fmaf(df, df, s2); }
        const float m = sqrtf(s2);  // == 0 exactly for k == sel_i
#pragma unroll
        for (int ii = 0; ii < NP; ++ii) if (ii == i) Mrow[ii] = m;
      }
    }
    float mn = FLT_MAX;
#pragma unroll
    for (int i = 0; i < NP; ++i) if (i < v_r) mn = fminf(mn, Mrow[i]);
    float* row = reinterpret_cast<float*>(smem) + tid * (ldx + 1);  // staging buffers are idle
#pragma unroll
    for (int i = 0; i < NP; ++i)
      if (i < ldx) row[i] = i < v_r ? Mrow[i] : (i == ld ? mn : 0.f);
    for (int x = NP; x < ldx; ++x) row[x] = x == ld ? mn : 0.f;
  }
  __syncthreads();
  // the block's rows are contiguous in Mx (and K~): coalesced copies out of shared memory
  const int rows = (int)(V - k0 < TC_M ? V - k0 : TC_M);
  {
    const float* tile = reinterpret_cast<const float*>(smem);
    float* dst = Mx + k0 * ldx;
    for (int g = tid; g < rows * ldx; g += 128) dst[g] = tile[(g / ldx) * (ldx + 1) + g % ldx];
    if (Kt) {
      float* kd = Kt + k0 * ld;
      for (int g = tid; g < rows * ld; g += 128) {
        const int r = g / ld, x = g % ld;
        const float mv = tile[r * (ldx + 1) + x], mn = tile[r * (ldx + 1) + ld];
        kd[g] = x < v_r ? expf(-lambda * (mv - mn)) : 0.f;
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tm), "n"(TMEM_COLS));
}

}  // namespace

void launch_build_ktilde(const float* E, int64_t row0, int64_t row1, int dp, const int32_t* sel, int v_r,
                         int ld, float lambda, float* Kt, float* Mx, bool use_tc, cudaStream_t st) {
  if (row1 <= row0) return;
  if (!use_tc) {
    // fewest passes of at most 8 kMaxRB query rows, then the smallest rows-per-thread covering them
    const int passes = (v_r + 8 * kMaxRB - 1) / (8 * kMaxRB);
    const int rb = ((v_r + passes - 1) / passes + 7) / 8;
    // 128-word blocks when 256-word blocks would fill fewer than ~4 waves of 2 blocks per SM
    const bool small = (row1 - row0) < (int64_t)BW * device_sms() * 8;
#define SIMT2_(RB, NWT)                                                                                  \
  {                                                                                                      \
    constexpr size_t smem = sizeof(float) * 2 * stage_floats<RB, NWT>();                                  \
    static_assert(32 * NWT * (8 * RB + 1) <= 2 * stage_floats<RB, NWT>(), "M tile must fit in the staging buffers"); \
    static PerDevice attr;                                                                               \
    attr.get([&] { return (int)cudaFuncSetAttribute(build_mx_kernel<RB, NWT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); }); \
    const int64_t grid = (row1 - row0 + 32 * NWT - 1) / (32 * NWT);                                     \
    build_mx_kernel<RB, NWT><<<(unsigned)grid, kThreads, smem, st>>>(E, row0, row1, dp, sel, v_r, ld, lambda, Kt, Mx); \
  }
#define SIMT_(RB) if (small) SIMT2_(RB, 4) else SIMT2_(RB, 8)
    switch (rb) {
      case 1: SIMT_(1) break;
      case 2: SIMT_(2) break;
      case 3: SIMT_(3) break;
      case 4: SIMT_(4) break;
      case 5: SIMT_(5) break;
      default: SIMT_(6) break;
    }
#undef SIMT_
#undef SIMT2_
    return;
  }
  const unsigned grid = (unsigned)((row1 - row0 + TC_M - 1) / TC_M);
#define TC_(NP)                                                                                       \
  {                                                                                                   \
    constexpr size_t sm = (TC_NS + TC_LO) * (TC_M + NP) * tc_k<NP>() * 4 + 1024;                    \
    static PerDevice a;                                                                               \
    a.get([&] { return (int)cudaFuncSetAttribute(build_mx_tc_kernel<NP>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm); }); \
    build_mx_tc_kernel<NP><<<grid, 128, sm, st>>>(E, row0, row1, dp, sel, v_r, ld, lambda, Kt, Mx);  \
  }
  if (v_r <= 32) TC_(32)
  else if (v_r <= 64) TC_(64)
  else if (v_r <= 96) TC_(96)
  else TC_(128)
#undef TC_
}

}  // namespace wmd
