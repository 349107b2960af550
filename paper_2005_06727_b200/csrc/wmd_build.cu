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
// Mapping: a block owns 256 vocabulary words x 32 query rows (more rows: further passes) and
// streams d in chunks of 32 through shared memory with cp.async, double buffered. Thread
// micro-tile: 4 query rows x 8 words = 32 independent accumulators; per d-quad a thread issues
// 12 LDS.128 (4 warp-broadcast query quads, 8 conflict-free word quads) for 256 FP32
// instructions (FADD + FFMA per (i, k, t) triple). Bound: FP32 issue, 2 instructions per
// triple (PAPER.md:260 counts 3 flops), E read once from HBM.
#include <algorithm>
#include <cfloat>
#include <cmath>
#include <cstdint>

#include "wmd_internal.h"

namespace wmd {
namespace {

constexpr int BW = 256;        // vocabulary words per block
constexpr int BI = 32;         // query rows per pass
constexpr int BD = 32;         // d chunk
constexpr int BP = BD + 4;     // smem pitch of a staged row (floats)
constexpr int kThreads = 256;
constexpr int kStageFloats = BI * BP + BW * BP;  // one pipeline stage: query rows + words
constexpr int kMsPitch = BI + 1;

__device__ __forceinline__ void cp16(float* dst, const float* src, bool valid) {
  const uint32_t d = static_cast<uint32_t>(__cvta_generic_to_shared(dst));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(d), "l"(src), "r"(valid ? 16 : 0)
               : "memory");
}

__global__ void __launch_bounds__(kThreads, 2) build_mx_kernel(
    const float* __restrict__ E, int64_t V, int dp, const int32_t* __restrict__ sel, int v_r,
    int ld, float lambda, float* __restrict__ Kt, float* __restrict__ Mx,
    float* __restrict__ colmin) {
  extern __shared__ __align__(16) float smem[];
  float* stage[2] = {smem, smem + kStageFloats};
  __shared__ float cmin[BW];
  const int tid = threadIdx.x, tw = tid & 31, ti = tid >> 5;
  const int64_t k0 = (int64_t)blockIdx.x * BW;
  const int nchunk = dp / BD;
  const int ldx = ld + 4;
  for (int w = tid; w < BW; w += kThreads) cmin[w] = FLT_MAX;

  for (int i0 = 0; i0 < v_r; i0 += BI) {
    // stage one d chunk: 32 query rows (one 16 B copy per thread) + 256 words (eight per thread)
    auto issue = [&](int c, float* buf) {
      const int t4 = tid & 7;
      {
        const int r = tid >> 3;                       // 0..31
        const bool ok = i0 + r < v_r;
        const int64_t row = ok ? sel[i0 + r] : 0;
        cp16(buf + r * BP + 4 * t4, E + row * dp + c * BD + 4 * t4, ok);
      }
#pragma unroll
      for (int q = 0; q < BW / 32; ++q) {
        const int w = (tid >> 3) + 32 * q;            // 0..255
        const bool ok = k0 + w < V;
        cp16(buf + BI * BP + w * BP + 4 * t4, E + (ok ? k0 + w : 0) * dp + c * BD + 4 * t4, ok);
      }
      asm volatile("cp.async.commit_group;" ::: "memory");
    };
    float acc[4][8];
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
      for (int s = 0; s < 8; ++s) acc[r][s] = 0.f;
    issue(0, stage[0]);
    for (int c = 0; c < nchunk; ++c) {
      if (c + 1 < nchunk) {
        issue(c + 1, stage[(c + 1) & 1]);
        asm volatile("cp.async.wait_group 1;" ::: "memory");
      } else {
        asm volatile("cp.async.wait_group 0;" ::: "memory");
      }
      __syncthreads();
      const float* Qs = stage[c & 1];
      const float* Es = Qs + BI * BP;
#pragma unroll 2
      for (int t = 0; t < BD; t += 4) {
        float4 q[4], e[8];
#pragma unroll
        for (int r = 0; r < 4; ++r) q[r] = *reinterpret_cast<const float4*>(Qs + (ti + 8 * r) * BP + t);
#pragma unroll
        for (int s = 0; s < 8; ++s) e[s] = *reinterpret_cast<const float4*>(Es + (tw + 32 * s) * BP + t);
#pragma unroll
        for (int r = 0; r < 4; ++r)
#pragma unroll
          for (int s = 0; s < 8; ++s) {
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
    float* Ms = smem;  // [BW][kMsPitch]
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
      for (int s = 0; s < 8; ++s) Ms[(tw + 32 * s) * kMsPitch + ti + 8 * r] = sqrtf(acc[r][s]);
    __syncthreads();
    // warp per word: lane i owns query row i0 + i (coalesced row writes)
    const int warp = tid >> 5, lane = tid & 31;
    const bool last = i0 + BI >= v_r;
    for (int w = warp; w < BW; w += kThreads / 32) {
      const int64_t k = k0 + w;
      if (k >= V) break;
      const int i = i0 + lane;
      const float m = Ms[w * kMsPitch + lane];
      float mn = i < v_r ? m : FLT_MAX;
#pragma unroll
      for (int off = 16; off; off >>= 1) mn = fminf(mn, __shfl_xor_sync(0xffffffffu, mn, off));
      mn = fminf(mn, cmin[w]);
      __syncwarp();
      if (i < v_r) Mx[k * ldx + i] = m;
      if (!last) {
        if (lane == 0) cmin[w] = mn;
        continue;
      }
      // row complete: zero padding, m_k, and K~ (reading back earlier passes' M from Mx)
      for (int x = v_r + lane; x < ldx; x += 32) Mx[k * ldx + x] = x == ld ? mn : 0.f;
      if (lane == 0) colmin[k] = mn;
      if (Kt) {
        for (int x = lane; x < ld; x += 32) {
          float kt = 0.f;
          if (x < v_r) kt = expf(-lambda * ((x >= i0 ? Ms[w * kMsPitch + x - i0] : Mx[k * ldx + x]) - mn));
          Kt[k * ld + x] = kt;
        }
      }
    }
    __syncthreads();  // Ms aliases the staging buffers of the next pass
  }
}

}  // namespace

void launch_build_ktilde(const float* E, int64_t V, int dp, const int32_t* sel, int v_r, int ld,
                         float lambda, float* Kt, float* Mx, float* colmin, cudaStream_t st) {
  constexpr size_t smem = sizeof(float) * 2 * kStageFloats;
  static_assert(BW * kMsPitch <= 2 * kStageFloats, "M tile must fit in the staging buffers");
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(build_mx_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr = true;
  }
  const int64_t grid = (V + BW - 1) / BW;
  build_mx_kernel<<<(unsigned)grid, kThreads, smem, st>>>(E, V, dp, sel, v_r, ld, lambda, Kt, Mx, colmin);
}

}  // namespace wmd
