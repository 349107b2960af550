// roofbench.cu — in-run roofline denominators for bench.py (measurement tool, not product code;
// built by paper_2005_06727_b200/build.py into tools/microbench/libroofbench.so).
//
// The sparse Sinkhorn path is bounded by row gathers from an L2-resident table (per-iteration
// kernel), by HBM streaming (c, u), or by FP32 issue (fused kernels).
// MEASURED_PEAKS.json holds only HBM copy bandwidth and bf16 tensor throughput, so bench.py
// measures the other two on the box, in the same run, with these plain C entry points (device
// pointers from torch, sizes; CUDA events on the given stream; best of `reps`):
//   rb_gather_ms  : gather of n rows of row_floats floats from tab[rows][row_floats], row ids
//                   idx[n] (bench passes the config's own word-id stream), one warp-slice per row
//   rb_stream_ms  : plain read of n float4 (HBM when the buffer is larger than L2)
//   rb_ffma_ms    : independent FFMA chains, grid of `blocks` x 256 threads, `iters` x 64 FMA/thread
#include <cstdint>
#include <cuda_runtime.h>

namespace {

// rows of row_floats floats, row_floats % 4 == 0; g = row_floats / 4 lanes per row (<= 32)
__global__ void gather_kernel(const float4* __restrict__ tab, int row4, const int* __restrict__ idx,
                              int64_t n, float* __restrict__ sink) {
  const int lane = threadIdx.x & 31;
  const int rpw = 32 / row4;                  // rows per warp step
  const int grp = lane / row4, sub = lane % row4;
  const bool active = grp < rpw;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  constexpr int U = 4;
  float acc = 0.f;
  for (int64_t base = warp * rpw * U; base < n; base += nwarps * rpw * U) {
    float4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t e = base + (int64_t)u * rpw + grp;
      v[u] = make_float4(0.f, 0.f, 0.f, 0.f);
      if (active && e < n) {
        const int k = __ldg(idx + e);
        v[u] = __ldg(tab + (int64_t)k * row4 + sub);
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) acc += v[u].x + v[u].y + v[u].z + v[u].w;
  }
  if (acc == 1234.5f) sink[0] = acc;
}

__global__ void stream_kernel(const float4* __restrict__ a, int64_t n4, float* __restrict__ sink) {
  float acc = 0.f;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += (int64_t)gridDim.x * blockDim.x) {
    const float4 v = __ldcs(a + i);
    acc += v.x + v.y + v.z + v.w;
  }
  if (acc == 1234.5f) sink[0] = acc;
}

__global__ void ffma_kernel(float* __restrict__ sink, int iters, float b) {
  float a[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) a[j] = threadIdx.x + j;
  const float d = 0.5f;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
#pragma unroll
      for (int t = 0; t < 8; ++t) a[t] = fmaf(a[t], b, d);
    }
  }
  float s = 0.f;
#pragma unroll
  for (int j = 0; j < 8; ++j) s += a[j];
  if (s == 1234.5f) sink[0] = s;  // b is a runtime value: the chains cannot be folded
}

template <class F>
int best_ms(cudaStream_t st, int reps, F launch, float* ms_out) {
  cudaEvent_t a, b;
  if (cudaEventCreate(&a) != cudaSuccess || cudaEventCreate(&b) != cudaSuccess) return 1;
  launch();  // warm-up
  float best = 1e30f;
  for (int r = 0; r < reps; ++r) {
    cudaEventRecord(a, st);
    launch();
    cudaEventRecord(b, st);
    if (cudaEventSynchronize(b) != cudaSuccess) return 2;
    float ms = 0.f;
    cudaEventElapsedTime(&ms, a, b);
    best = ms < best ? ms : best;
  }
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  *ms_out = best;
  return cudaGetLastError() != cudaSuccess ? 3 : 0;
}

int grid_for(int per_sm) {
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return (sms > 0 ? sms : 148) * per_sm;
}

}  // namespace

extern "C" {

int rb_gather_ms(const float* tab, int row_floats, const int32_t* idx, int64_t n, float* sink, void* stream,
                 int reps, float* ms_out) {
  if (!tab || !idx || !sink || !ms_out || row_floats % 4 || row_floats < 4 || row_floats > 128) return -1;
  cudaStream_t st = (cudaStream_t)stream;
  const int grid = grid_for(8);
  return best_ms(st, reps, [&] {
    gather_kernel<<<grid, 256, 0, st>>>(reinterpret_cast<const float4*>(tab), row_floats / 4, idx, n, sink);
  }, ms_out);
}

int rb_stream_ms(const float* a, int64_t n4, float* sink, void* stream, int reps, float* ms_out) {
  if (!a || !sink || !ms_out) return -1;
  cudaStream_t st = (cudaStream_t)stream;
  const int grid = grid_for(8);
  return best_ms(st, reps, [&] { stream_kernel<<<grid, 512, 0, st>>>(reinterpret_cast<const float4*>(a), n4, sink); },
                 ms_out);
}

// FMA count of one rb_ffma_ms launch: blocks * 256 * iters * 64
int rb_ffma_ms(int blocks_per_sm, int iters, float* sink, void* stream, int reps, float* ms_out, int64_t* fmas) {
  if (!sink || !ms_out || !fmas) return -1;
  cudaStream_t st = (cudaStream_t)stream;
  const int grid = grid_for(blocks_per_sm);
  *fmas = (int64_t)grid * 256 * iters * 64;
  return best_ms(st, reps, [&] { ffma_kernel<<<grid, 256, 0, st>>>(sink, iters, 1.0001f); }, ms_out);
}

}  // extern "C"
