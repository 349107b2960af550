// Microbenchmark: L2/L1 row-gather bandwidth on B200 (the binding roof of the
// per-iteration SDDMM_SpMM kernel), plus a plain HBM stream read.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gather_bw gather_bw.cu
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <vector>
#include <random>
#include <cmath>
#include <algorithm>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); exit(1);} } while (0)

// G lanes per row, each lane loads one float4 (row = 4*G floats). U rows in flight per group.
template <int G, int U, bool NC>
__global__ void gather(const float4* __restrict__ tab, const int* __restrict__ idx, long n, float* out) {
  const int lane = threadIdx.x & 31;
  const int grp = lane / G, sub = lane % G;
  constexpr int RPW = 32 / G;  // rows per warp step
  long warp = (blockIdx.x * (long)blockDim.x + threadIdx.x) >> 5;
  long nwarps = ((long)gridDim.x * blockDim.x) >> 5;
  float acc = 0.f;
  for (long base = warp * RPW * U; base < n; base += nwarps * RPW * U) {
    float4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      long e = base + u * RPW + grp;
      if (e < n) {
        int k = __ldg(idx + e);
        const float4* p = tab + (long)k * G + sub;
        v[u] = NC ? __ldg(p) : *p;
      } else v[u] = make_float4(0, 0, 0, 0);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) acc += v[u].x + v[u].y + v[u].z + v[u].w;
  }
  if (acc == 1234.5f) out[0] = acc;
}

__global__ void stream_read(const float4* __restrict__ a, long n4, float* out) {
  float acc = 0.f;
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n4; i += (long)gridDim.x * blockDim.x) {
    float4 v = __ldcs(a + i);
    acc += v.x + v.y + v.z + v.w;
  }
  if (acc == 1234.5f) out[0] = acc;
}

__global__ void shfl_fma(float* out, int iters) {
  float a = threadIdx.x, b = 1.0001f, c = 0.f, d = 1.f;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      c += __shfl_xor_sync(0xffffffffu, a, 1 << (j & 3));
      a = fmaf(a, b, d);
    }
  }
  if (c == 1234.5f) out[0] = c + a;
}
__global__ void fma_only(float* out, int iters) {
  float a0 = threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, b = 1.0001f, d = 0.5f;
  float a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      a0 = fmaf(a0, b, d); a1 = fmaf(a1, b, d); a2 = fmaf(a2, b, d); a3 = fmaf(a3, b, d);
      a4 = fmaf(a4, b, d); a5 = fmaf(a5, b, d); a6 = fmaf(a6, b, d); a7 = fmaf(a7, b, d);
    }
  }
  if (a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7 == 1234.5f) out[0] = a0;
}
__global__ void shfl_only(float* out, int iters) {
  float a0 = threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      a0 = __shfl_xor_sync(0xffffffffu, a0, 1); a1 = __shfl_xor_sync(0xffffffffu, a1, 2);
      a2 = __shfl_xor_sync(0xffffffffu, a2, 4); a3 = __shfl_xor_sync(0xffffffffu, a3, 8);
    }
  }
  if (a0 + a1 + a2 + a3 == 1234.5f) out[0] = a0;
}

template <typename F>
float time_ms(F f, int reps = 10) {
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  f(); CK(cudaDeviceSynchronize());
  float best = 1e30f;
  for (int r = 0; r < reps; ++r) {
    cudaEventRecord(a); f(); cudaEventRecord(b); CK(cudaEventSynchronize(b));
    float ms; cudaEventElapsedTime(&ms, a, b); best = std::min(best, ms);
  }
  return best;
}

int main() {
  cudaDeviceProp prop; CK(cudaGetDeviceProperties(&prop, 0));
  int nsm = prop.multiProcessorCount;
  printf("{\"gpu\":\"%s\",\"sms\":%d,\"l2_bytes\":%d,\"smem_per_sm\":%zu}\n", prop.name, nsm, prop.l2CacheSize, prop.sharedMemPerMultiprocessor);
  float* out; CK(cudaMalloc(&out, 4));
  // HBM stream read, 2 GiB
  {
    long n4 = (2L << 30) / 16;
    float4* a; CK(cudaMalloc(&a, n4 * 16)); CK(cudaMemset(a, 0, n4 * 16));
    float ms = time_ms([&] { stream_read<<<nsm * 8, 512>>>(a, n4, out); });
    printf("{\"test\":\"hbm_stream_read\",\"bytes\":%ld,\"ms\":%.4f,\"GBps\":%.1f}\n", n4 * 16, ms, n4 * 16 / ms / 1e6);
    CK(cudaFree(a));
  }
  // gathers
  std::mt19937_64 rng(7);
  long n = 64L << 20;  // 64M gathers
  std::vector<int> h(n);
  int* didx; CK(cudaMalloc(&didx, n * 4));
  struct Cfg { long rows; const char* dist; };
  for (long rows : {100000L, 400000L}) {
    for (int zipf = 0; zipf < 2; ++zipf) {
      if (!zipf) { std::uniform_int_distribution<long> U(0, rows - 1); for (long i = 0; i < n; ++i) h[i] = (int)U(rng); }
      else {
        std::vector<double> cdf(rows); double s = 0; for (long k = 0; k < rows; ++k) { s += std::pow((double)(k + 1), -1.07); cdf[k] = s; }
        std::uniform_real_distribution<double> U(0, s);
        for (long i = 0; i < n; ++i) h[i] = (int)(std::lower_bound(cdf.begin(), cdf.end(), U(rng)) - cdf.begin());
        for (long i = 0; i < n; ++i) if (h[i] >= rows) h[i] = rows - 1;
      }
      CK(cudaMemcpy(didx, h.data(), n * 4, cudaMemcpyHostToDevice));
      for (int G : {8, 32}) {
        long tabbytes = rows * G * 16;
        float4* tab; CK(cudaMalloc(&tab, tabbytes)); CK(cudaMemset(tab, 0, tabbytes));
        for (int nc = 0; nc < 2; ++nc) {
          float ms;
          int grid = nsm * 8, blk = 256;
          if (G == 8) ms = nc ? time_ms([&] { gather<8, 4, true><<<grid, blk>>>(tab, didx, n, out); }) : time_ms([&] { gather<8, 4, false><<<grid, blk>>>(tab, didx, n, out); });
          else ms = nc ? time_ms([&] { gather<32, 4, true><<<grid, blk>>>(tab, didx, n, out); }) : time_ms([&] { gather<32, 4, false><<<grid, blk>>>(tab, didx, n, out); });
          double bytes = (double)n * G * 16 + n * 4.0;
          printf("{\"test\":\"gather\",\"rows\":%ld,\"row_bytes\":%d,\"table_MB\":%.1f,\"dist\":\"%s\",\"nc\":%d,\"ms\":%.4f,\"GBps\":%.1f,\"Grows_per_s\":%.2f}\n",
                 rows, G * 16, tabbytes / 1e6, zipf ? "zipf1.07" : "uniform", nc, ms, bytes / ms / 1e6, n / ms / 1e6);
        }
        CK(cudaFree(tab));
      }
    }
  }
  // SHFL vs FMA issue throughput
  {
    int iters = 4096, grid = nsm * 16, blk = 256;
    float ms = time_ms([&] { fma_only<<<grid, blk>>>(out, iters); });
    double ops = (double)grid * blk * iters * 64;
    printf("{\"test\":\"fma\",\"Gfma_per_s\":%.1f,\"per_sm_per_clk_at_1965\":%.1f}\n", ops / ms / 1e6, ops / ms * 1e3 / nsm / 1.965e9);
    ms = time_ms([&] { shfl_only<<<grid, blk>>>(out, iters); });
    ops = (double)grid * blk * iters * 32;
    printf("{\"test\":\"shfl\",\"Gshfl_lanes_per_s\":%.1f,\"lanes_per_sm_per_clk_at_1965\":%.1f}\n", ops / ms / 1e6, ops / ms * 1e3 / nsm / 1.965e9);
  }
  return 0;
}
