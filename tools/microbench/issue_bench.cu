// Throughput microbenchmarks for the fused-kernel design (not product code):
//   ffma      : independent FFMA chains (8 per thread)
//   shfl      : independent __shfl_xor_sync (8 per thread)
//   lds128b   : broadcast LDS.128 (all lanes same address)
//   lds128    : conflict-free LDS.128 (lane-distinct rows, pitch 36 floats)
//   lds32     : conflict-free LDS.32
//   redux     : __reduce_max_sync on unsigned
//   mufu      : rcp.approx
// Each kernel runs `iters` rounds of 8 independent ops per thread; grid = 148 * blocks.
// Output: warp-instructions per SM-cycle (sm clock read via clock64 on one SM).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define K_BEGIN(name) __global__ void name(float* out, int iters, long long* clk) { \
  long long t0 = clock64(); \
  const int lane = threadIdx.x & 31;
#define K_END(expr) \
  long long t1 = clock64(); \
  if (threadIdx.x == 0 && blockIdx.x == 0) *clk = t1 - t0; \
  if (expr == 12345.f) out[threadIdx.x] = expr; }

K_BEGIN(k_ffma)
  float a[8];
  for (int i = 0; i < 8; ++i) a[i] = lane * 0.1f + i;
  const float b = 1.0001f, c = 0.0001f;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = fmaf(a[i], b, c);
  }
  float s = 0; for (int i = 0; i < 8; ++i) s += a[i];
K_END(s)

K_BEGIN(k_ffma3)
  // 3-register FFMA: both multiplicands from registers that change
  float a[8], bb[8];
  for (int i = 0; i < 8; ++i) { a[i] = lane * 0.1f + i; bb[i] = 1.0f + i * 1e-6f; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = fmaf(a[i], bb[i], bb[(i + 1) & 7]);
  }
  float s = 0; for (int i = 0; i < 8; ++i) s += a[i];
K_END(s)

K_BEGIN(k_ffma2)
  // packed FFMA2: 8 independent float2 chains, register operands
  float2 a[8], bb[8];
  for (int i = 0; i < 8; ++i) { a[i] = make_float2(lane * 0.1f + i, i); bb[i] = make_float2(1.0f + i * 1e-6f, 1.0f - i * 1e-6f); }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = __ffma2_rn(a[i], bb[i], bb[(i + 1) & 7]);
  }
  float s = 0; for (int i = 0; i < 8; ++i) s += a[i].x + a[i].y;
K_END(s)

K_BEGIN(k_dfma)
  double a[8], bb[8];
  for (int i = 0; i < 8; ++i) { a[i] = lane * 0.1 + i; bb[i] = 1.0 + i * 1e-9; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = fma(a[i], bb[i], bb[(i + 1) & 7]);
  }
  double s = 0; for (int i = 0; i < 8; ++i) s += a[i];
K_END((float)s)

K_BEGIN(k_shfl)
  float a[8];
  for (int i = 0; i < 8; ++i) a[i] = lane * 0.1f + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = __shfl_xor_sync(0xffffffffu, a[i], 1 + (i & 3));
  }
  float s = 0; for (int i = 0; i < 8; ++i) s += a[i];
K_END(s)

K_BEGIN(k_lds128b)
  __shared__ __align__(16) float sh[32 * 36];
  for (int i = threadIdx.x; i < 32 * 36; i += blockDim.x) sh[i] = i;
  __syncthreads();
  float4 acc = make_float4(0, 0, 0, 0);
  int off = 0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      float4 v = *reinterpret_cast<const float4*>(sh + ((off + 4 * i) & 1023));
      acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
    }
    off += 4 * (int)(acc.x > 1e30f);
  }
K_END(acc.x + acc.y + acc.z + acc.w)

K_BEGIN(k_lds128)
  __shared__ __align__(16) float sh[32 * 36 * 4];
  for (int i = threadIdx.x; i < 32 * 36 * 4; i += blockDim.x) sh[i] = i;
  __syncthreads();
  float4 acc = make_float4(0, 0, 0, 0);
  const int w = (threadIdx.x >> 5) & 3;
  int off = 0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      float4 v = *reinterpret_cast<const float4*>(sh + w * 1152 + lane * 36 + ((off + 4 * i) & 31));
      acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
    }
    off += 4 * (int)(acc.x > 1e30f);
  }
K_END(acc.x + acc.y + acc.z + acc.w)

K_BEGIN(k_lds32)
  __shared__ float sh[32 * 36];
  for (int i = threadIdx.x; i < 32 * 36; i += blockDim.x) sh[i] = i;
  __syncthreads();
  float acc = 0;
  int off = 0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) acc += sh[((off + i) & 31) * 36 + lane];
    off += (int)(acc > 1e30f);
  }
K_END(acc)

K_BEGIN(k_redux)
  unsigned a[8];
  for (int i = 0; i < 8; ++i) a[i] = lane * 7 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = __reduce_max_sync(0xffffffffu, a[i] + lane) ;
  }
  unsigned s = 0; for (int i = 0; i < 8; ++i) s += a[i];
K_END((float)s)

K_BEGIN(k_mufu)
  float a[8];
  for (int i = 0; i < 8; ++i) a[i] = lane * 0.1f + i + 1.f;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    // volatile, and not an involution (rcp(rcp(x)) = x was folded away: the round-1 numbers of
    // this entry were impossible); the FADD runs on the FMA pipe, not the MUFU unit
    for (int i = 0; i < 8; ++i) { float y; asm volatile("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(a[i])); a[i] = y + 1.f; }
  }
  float s = 0; for (int i = 0; i < 8; ++i) s += a[i];
K_END(s)

typedef void (*KF)(float*, int, long long*);

int main() {
  float* out; long long* clk;
  cudaMalloc(&out, 1 << 20); cudaMalloc(&clk, 8);
  struct { const char* name; KF f; } ks[] = {
    {"ffma_imm", k_ffma}, {"ffma3", k_ffma3}, {"ffma2", k_ffma2}, {"dfma", k_dfma}, {"shfl", k_shfl}, {"lds128_bcast", k_lds128b},
    {"lds128", k_lds128}, {"lds32", k_lds32}, {"redux", k_redux}, {"mufu_rcp", k_mufu}};
  int sms = 0; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (auto& k : ks) {
    for (int wpb : {4, 8, 16}) {
      const int threads = 32 * wpb, blocks = sms * 2, iters = 4096;
      k.f<<<blocks, threads>>>(out, 16, clk);
      cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
      cudaEventRecord(a);
      k.f<<<blocks, threads>>>(out, iters, clk);
      cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      long long c; cudaMemcpy(&c, clk, 8, cudaMemcpyDeviceToHost);
      // warp-instructions per SM per cycle, using the measured kernel time and the SM clock from clk
      const double warp_ops = (double)blocks * wpb * iters * 8;
      const double sm_cycles = ms * 1e-3 * 1.965e9;  // nominal max clock
      printf("{\"op\":\"%s\",\"warps_per_sm\":%d,\"ms\":%.4f,\"warp_ops_per_sm_cycle\":%.3f,\"block0_cycles\":%lld}\n",
             k.name, 2 * wpb, ms, warp_ops / sms / sm_cycles, c);
    }
  }
  return 0;
}
