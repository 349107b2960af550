// wmd_tile.cuh — register-tile helpers shared by the fused Sinkhorn kernels (wmd_fused.cu: one
// warp per document; wmd_fused_cta.cu: one CTA per long document). A warp holds a document-row
// x query-row tile of Kh with lane = 8a + b: a in [0,4) selects 8-row groups of a 32-row tile,
// b in [0,8) selects CW-column groups; register slots are XOR-permuted by the lane bits so the
// transpose-reduces below send the upper half of the slots and keep the lower half (no selects).
#pragma once
#include <cstdint>

#include "wmd_device.cuh"

namespace wmd {
namespace tile {

using dev::kFull;

__device__ __forceinline__ float lg2_approx(float x) {
  float y;
  asm("lg2.approx.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
// log2 with subnormal inputs flushed (one MUFU.LG2; the non-ftz form adds a rescale of
// subnormal inputs, ~6 more instructions per call). lg2_ftz(0) = -inf.
__device__ __forceinline__ float lg2_ftz(float x) {
  float y;
  asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
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
__device__ __forceinline__ float shx(float v, int m) { return __shfl_xor_sync(kFull, v, m); }

// Packed FP32 FMA on two lanes: (d0, d1) = (a0 b0 + c0, a1 b1 + c1), one fma.rn.f32x2 (SASS
// FFMA2, sm_100a): the same 128 FMA/clk/SM as scalar FFMA in half the issue slots, IEEE
// round-to-nearest per lane (profiles/r02_ffma2.jsonl). With b0 == b1 ptxas uses the scalar
// (broadcast) operand form; the pair (a0, a1) is one 64-bit register pair, so the fused kernels
// use each block entry in the same pairing (two adjacent document rows) in every step.
__device__ __forceinline__ void ffma2(float& d0, float& d1, float a0, float a1, float b0, float b1, float c0,
                                      float c1) {
  asm("{.reg .b64 A, B, C, D;\n\t"
      "mov.b64 A, {%2, %3};\n\t"
      "mov.b64 B, {%4, %5};\n\t"
      "mov.b64 C, {%6, %7};\n\t"
      "fma.rn.f32x2 D, A, B, C;\n\t"
      "mov.b64 {%0, %1}, D;}"
      : "=f"(d0), "=f"(d1)
      : "f"(a0), "f"(a1), "f"(b0), "f"(b1), "f"(c0), "f"(c1));
}
// A (b0, b1) operand packed once and reused by several ffma2p / fmul2p (ptxas otherwise copies
// the pair before each use)
__device__ __forceinline__ uint64_t pack2(float x, float y) {
  uint64_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(x), "f"(y));
  return r;
}
__device__ __forceinline__ void ffma2p(float& d0, float& d1, float a0, float a1, uint64_t b, float c0, float c1) {
  asm("{.reg .b64 A, C, D;\n\t"
      "mov.b64 A, {%2, %3};\n\t"
      "mov.b64 C, {%5, %6};\n\t"
      "fma.rn.f32x2 D, A, %4, C;\n\t"
      "mov.b64 {%0, %1}, D;}"
      : "=f"(d0), "=f"(d1)
      : "f"(a0), "f"(a1), "l"(b), "f"(c0), "f"(c1));
}
__device__ __forceinline__ void fmul2p(float& d0, float& d1, float a0, float a1, uint64_t b) {
  asm("{.reg .b64 A, D;\n\t"
      "mov.b64 A, {%2, %3};\n\t"
      "mul.rn.f32x2 D, A, %4;\n\t"
      "mov.b64 {%0, %1}, D;}"
      : "=f"(d0), "=f"(d1)
      : "f"(a0), "f"(a1), "l"(b));
}
// (d0, d1) = (a0 b0, a1 b1): one mul.rn.f32x2 (FMUL2)
__device__ __forceinline__ void fmul2(float& d0, float& d1, float a0, float a1, float b0, float b1) {
  asm("{.reg .b64 A, B, D;\n\t"
      "mov.b64 A, {%2, %3};\n\t"
      "mov.b64 B, {%4, %5};\n\t"
      "mul.rn.f32x2 D, A, B;\n\t"
      "mov.b64 {%0, %1}, D;}"
      : "=f"(d0), "=f"(d1)
      : "f"(a0), "f"(a1), "f"(b0), "f"(b1));
}

// Row index (within the document) of row slot s of lane (a, b).
template <int NT, int TW>
__device__ __forceinline__ int row_of(int s, int a, int b) {
  constexpr int TSH = TW == 4 ? 1 : 2;
  if (s < 8 * NT) return 32 * (s >> 3) + 8 * a + ((s & 7) ^ b);
  return 32 * NT + TW * a + ((s - 8 * NT) ^ (b >> TSH));
}

// Column layout of a lane's CW = 4Q + R block columns (CW = 3 or CW >= 4; CW = 1, 2 below):
// Q quads, quad g of lane b covering columns 32g + 4b + j (j < 4), then R plain columns
// 32Q + Rb + r. In register-slot order the quads are XOR-permuted by a (slot 4g + t holds
// j = t ^ a) so that the column transpose-reduce over the a-lanes needs no selects; the plain
// columns are the same in all four a-lanes and are reduced by a full butterfly.
template <int CW>
struct Cols {
  static constexpr int Q = CW >= 3 ? CW / 4 : 0;
  static constexpr int R = CW >= 3 ? CW % 4 : 0;
};

// Natural-order column of slot c (the order load_cols delivers).
template <int CW>
__device__ __forceinline__ int nat_col(int c, int b) {
  constexpr int Q = Cols<CW>::Q, R = Cols<CW>::R;
  if constexpr (CW >= 3) return c < 4 * Q ? 32 * (c >> 2) + 4 * b + (c & 3) : 32 * Q + R * b + (c - 4 * Q);
  else return CW * b + c;
}

// Column (query row) of column slot c of lane (a, b).
template <int CW>
__device__ __forceinline__ int col_of(int c, int a, int b) {
  constexpr int Q = Cols<CW>::Q, R = Cols<CW>::R;
  if constexpr (CW >= 3) return c < 4 * Q ? 32 * (c >> 2) + 4 * b + ((c & 3) ^ a) : 32 * Q + R * b + (c - 4 * Q);
  else if constexpr (CW == 2) return 2 * b + (c ^ (a >> 1));
  else return b;
}

// Permute x[0..CW) (natural column order of this lane's column group) into slot order:
// x'[c] = x[c ^ key], key = a (per quad) or a >> 1 (CW = 2); plain columns stay.
template <int CW>
__device__ __forceinline__ void to_slots(float (&x)[CW], int a) {
  if constexpr (CW >= 3) {
#pragma unroll
    for (int q = 0; q < Cols<CW>::Q; ++q) {
      float* y = x + 4 * q;
      const bool s1 = a & 1, s2 = a & 2;
      float t0 = s1 ? y[1] : y[0], t1 = s1 ? y[0] : y[1];
      float t2 = s1 ? y[3] : y[2], t3 = s1 ? y[2] : y[3];
      y[0] = s2 ? t2 : t0; y[2] = s2 ? t0 : t2;
      y[1] = s2 ? t3 : t1; y[3] = s2 ? t1 : t3;
    }
  } else if constexpr (CW == 2) {
    const bool s2 = a & 2;
    const float t0 = s2 ? x[1] : x[0], t1 = s2 ? x[0] : x[1];
    x[0] = t0; x[1] = t1;
  }
}

// Loads this lane's CW natural-order columns of one staged row.
template <int CW>
__device__ __forceinline__ void load_cols(const float* row, int b, float (&x)[CW]) {
  if constexpr (CW >= 3) {
    constexpr int Q = Cols<CW>::Q, R = Cols<CW>::R;
#pragma unroll
    for (int q = 0; q < Q; ++q) {
      const float4 t = *reinterpret_cast<const float4*>(row + 32 * q + 4 * b);
      x[4 * q] = t.x; x[4 * q + 1] = t.y; x[4 * q + 2] = t.z; x[4 * q + 3] = t.w;
    }
#pragma unroll
    for (int r = 0; r < R; ++r) x[4 * Q + r] = row[32 * Q + R * b + r];
  } else if constexpr (CW == 2) {
    const float2 t = *reinterpret_cast<const float2*>(row + 2 * b);
    x[0] = t.x; x[1] = t.y;
  } else {
    x[0] = row[b];
  }
}

// Transpose-reduce of the row partials p[0..RW) over the 8 b-lanes: afterwards p[8T] holds the
// full sum of row 32T + 8a + b (full tiles) and p[8NT] that of tail row 32NT + TW a + (b >> TSH).
template <int NT, int TW>
__device__ __forceinline__ void reduce_rows(float* p) {
#pragma unroll
  for (int T = 0; T < NT; ++T) {
    float* q = p + 8 * T;
#pragma unroll
    for (int t = 0; t < 4; ++t) q[t] += shx(q[t + 4], 4);
#pragma unroll
    for (int t = 0; t < 2; ++t) q[t] += shx(q[t + 2], 2);
    q[0] += shx(q[1], 1);
  }
  if constexpr (TW == 4) {
    float* q = p + 8 * NT;
    q[0] += shx(q[2], 4); q[1] += shx(q[3], 4);
    q[0] += shx(q[1], 2);
    q[0] += shx(q[0], 1);
  } else if constexpr (TW == 2) {
    float* q = p + 8 * NT;
    q[0] += shx(q[1], 4);
    q[0] += shx(q[0], 2);
    q[0] += shx(q[0], 1);
  }
}

// As reduce_rows with max instead of sum.
template <int NT, int TW>
__device__ __forceinline__ void reduce_rows_max(float* p) {
#pragma unroll
  for (int T = 0; T < NT; ++T) {
    float* q = p + 8 * T;
#pragma unroll
    for (int t = 0; t < 4; ++t) q[t] = fmaxf(q[t], shx(q[t + 4], 4));
#pragma unroll
    for (int t = 0; t < 2; ++t) q[t] = fmaxf(q[t], shx(q[t + 2], 2));
    q[0] = fmaxf(q[0], shx(q[1], 1));
  }
  if constexpr (TW == 4) {
    float* q = p + 8 * NT;
    q[0] = fmaxf(q[0], shx(q[2], 4)); q[1] = fmaxf(q[1], shx(q[3], 4));
    q[0] = fmaxf(q[0], shx(q[1], 2));
    q[0] = fmaxf(q[0], shx(q[0], 1));
  } else if constexpr (TW == 2) {
    float* q = p + 8 * NT;
    q[0] = fmaxf(q[0], shx(q[1], 4));
    q[0] = fmaxf(q[0], shx(q[0], 2));
    q[0] = fmaxf(q[0], shx(q[0], 1));
  }
}

// Transpose-reduce of the column partials q[0..CW) over the 4 a-lanes (lane xor 16, 8):
// afterwards q[4g] holds the full sum of quad column 32g + 4b + a, q[4Q + r] that of plain
// column 32Q + Rb + r (CW >= 3); q[0] that of column 2b + (a >> 1) (CW = 2) or b (CW = 1).
template <int CW>
__device__ __forceinline__ void reduce_cols(float* q) {
  if constexpr (CW >= 3) {
    constexpr int Q = Cols<CW>::Q, R = Cols<CW>::R;
#pragma unroll
    for (int g = 0; g < Q; ++g) {
      float* y = q + 4 * g;
      y[0] += shx(y[2], 16); y[1] += shx(y[3], 16);
      y[0] += shx(y[1], 8);
    }
#pragma unroll
    for (int r = 0; r < R; ++r) {
      q[4 * Q + r] += shx(q[4 * Q + r], 16);
      q[4 * Q + r] += shx(q[4 * Q + r], 8);
    }
  } else if constexpr (CW == 2) {
    q[0] += shx(q[1], 16);
    q[0] += shx(q[0], 8);
  } else {
    q[0] += shx(q[0], 16);
    q[0] += shx(q[0], 8);
  }
}

}  // namespace tile
}  // namespace wmd
