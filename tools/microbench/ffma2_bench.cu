// Microbenchmark: packed FP32 FMA (fma.rn.f32x2 -> SASS FFMA2, sm_100a) against scalar FFMA on
// B200 — throughput (many independent chains, full occupancy) and dependent-chain latency (one
// warp). Decides whether the fused Sinkhorn kernels' FMA work can be issued two FMAs per
// instruction.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ffma2_bench ffma2_bench.cu
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); exit(1);} } while (0)

__device__ __forceinline__ float2 fma2(float2 a, float2 b, float2 c) {
  float2 d;
  asm volatile("{.reg .b64 A,B,C,D; mov.b64 A,{%2,%3}; mov.b64 B,{%4,%5}; mov.b64 C,{%6,%7};"
               " fma.rn.f32x2 D, A, B, C; mov.b64 {%0,%1}, D;}"
               : "=f"(d.x), "=f"(d.y) : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y), "f"(c.x), "f"(c.y));
  return d;
}
__device__ __forceinline__ float fma1(float a, float b, float c) {
  float d;
  asm volatile("fma.rn.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
  return d;
}

// CH independent chains per thread; each step one FMA (scalar) or one FFMA2 (2 FMAs)
template <int CH>
__global__ void thr_ffma(float* out, int iters, float b) {
  float c[CH];
#pragma unroll
  for (int i = 0; i < CH; ++i) c[i] = threadIdx.x + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CH; ++i) c[i] = fma1(c[i], b, 1.0f);
  }
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < CH; ++i) s += c[i];
  if (s == 1234.5f) out[0] = s;
}
template <int CH>
__global__ void thr_ffma2(float* out, int iters, float b) {
  float2 c[CH];
  const float2 bb = make_float2(b, b), one = make_float2(1.f, 1.f);
#pragma unroll
  for (int i = 0; i < CH; ++i) c[i] = make_float2(threadIdx.x + i, threadIdx.x - i);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CH; ++i) c[i] = fma2(c[i], bb, one);
  }
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < CH; ++i) s += c[i].x + c[i].y;
  if (s == 1234.5f) out[0] = s;
}
// FFMA2 with a scalar (broadcast) second operand, the SDDMM form
template <int CH>
__global__ void thr_ffma2_bc(float* out, int iters, float b) {
  float2 c[CH];
  const float2 one = make_float2(1.f, 1.f);
#pragma unroll
  for (int i = 0; i < CH; ++i) c[i] = make_float2(threadIdx.x + i, threadIdx.x - i);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CH; ++i) c[i] = fma2(c[i], make_float2(b, b), one);
  }
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < CH; ++i) s += c[i].x + c[i].y;
  if (s == 1234.5f) out[0] = s;
}

int main() {
  int sms = 0, clk = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  CK(cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0));
  float* out;
  CK(cudaMalloc(&out, 16));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  auto run = [&](const char* name, void (*k)(float*, int, float), int grid, int block, int iters, double fma_per_step) {
    k<<<grid, block>>>(out, 16, 1.0001f);
    CK(cudaDeviceSynchronize());
    CK(cudaEventRecord(e0));
    k<<<grid, block>>>(out, iters, 1.0001f);
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    const double threads = (double)grid * block;
    const double fmas = threads * iters * fma_per_step;
    const double tflops = 2.0 * fmas / (ms * 1e-3) / 1e12;
    const double warp_instr = threads / 32.0 * iters * (fma_per_step / (strstr(name, "ffma2") ? 2.0 : 1.0));
    const double cyc = ms * 1e-3 * clk * 1e3;  // at the nominal clock
    printf("{\"bench\": \"%s\", \"grid\": %d, \"block\": %d, \"ms\": %.4f, \"tflops\": %.2f, "
           "\"fma_per_sm_per_clk\": %.1f, \"warp_instr_per_smsp_per_clk\": %.3f, \"cyc_per_step\": %.2f}\n",
           name, grid, block, ms, tflops, fmas / sms / cyc, warp_instr / (4.0 * sms) / cyc, cyc / iters);
  };
  const int G = sms * 8;
  run("ffma_thr_ch8", thr_ffma<8>, G, 256, 20000, 8);
  run("ffma2_thr_ch8", thr_ffma2<8>, G, 256, 20000, 16);
  run("ffma2_bc_thr_ch8", thr_ffma2_bc<8>, G, 256, 20000, 16);
  run("ffma2_thr_ch4", thr_ffma2<4>, G, 256, 20000, 8);
  // latency: one warp, one chain
  run("ffma_lat_ch1", thr_ffma<1>, 1, 32, 200000, 1);
  run("ffma2_lat_ch1", thr_ffma2<1>, 1, 32, 200000, 2);
  // one warp per scheduler with 4 / 8 chains (issue-limited regime of the fused kernels)
  run("ffma_1wps_ch8", thr_ffma<8>, sms, 128, 200000, 8);
  run("ffma2_1wps_ch8", thr_ffma2<8>, sms, 128, 200000, 16);
  run("ffma2_1wps_ch4", thr_ffma2<4>, sms, 128, 200000, 8);
  return 0;
}
