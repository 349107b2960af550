// Standalone check of a hand-written tcgen05 TF32 MMA (not product code): one CTA computes
// D[128 x 32] = A[128 x K] * B[32 x K]^T with K-major SWIZZLE_NONE operands staged in shared
// memory, the accumulator in TMEM, and a tcgen05.ld epilogue; 1xTF32 and 3xTF32 (split
// hi/lo) against an FP64 CPU reference.
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cmath>
#include <vector>
#include <cuda_runtime.h>

constexpr int M = 128, N = 32, K = 64;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// K-major, no swizzle: core matrix = 8 rows x 16 bytes (4 fp32); element (r, k) of an R x K
// tile at byte offset (k/4)*LBO + (r/8)*SBO + (r%8)*16 + (k%4)*4 with SBO = 128, LBO = R/8*128.
__device__ __forceinline__ int kmaj_off(int r, int k, int R) {
  return (k >> 2) * (R / 8 * 128) + (r >> 3) * 128 + (r & 7) * 16 + (k & 3) * 4;
}

__device__ __forceinline__ uint64_t make_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;  // version = 1 (sm100)
  // base_offset 0, lbo_mode 0, layout_type 0 (SWIZZLE_NONE)
  return d;
}

__device__ __forceinline__ uint32_t idesc_tf32(int m, int n) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(m >> 4) << 24);
}

__global__ void umma_kernel(const float* A, const float* B, float* D, int split) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* sAh = sm;                       // M x K
  uint8_t* sAl = sAh + M * K * 4;
  uint8_t* sBh = sAl + M * K * 4;          // N x K
  uint8_t* sBl = sBh + N * K * 4;
  __shared__ uint32_t tmem_base;
  __shared__ __align__(8) uint64_t mbar;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < M * K; i += blockDim.x) {
    const int r = i / K, k = i % K;
    const float x = A[i];
    const float hi = __uint_as_float(__float_as_uint(x) & 0xffffe000u);
    *reinterpret_cast<float*>(sAh + kmaj_off(r, k, M)) = x;
    *reinterpret_cast<float*>(sAl + kmaj_off(r, k, M)) = x - hi;
  }
  for (int i = tid; i < N * K; i += blockDim.x) {
    const int r = i / K, k = i % K;
    const float x = B[i];
    const float hi = __uint_as_float(__float_as_uint(x) & 0xffffe000u);
    *reinterpret_cast<float*>(sBh + kmaj_off(r, k, N)) = x;
    *reinterpret_cast<float*>(sBl + kmaj_off(r, k, N)) = x - hi;
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base)), "n"(32));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&mbar)), "r"(1));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  // make the generic-proxy smem writes visible to the tensor core (async proxy)
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tm = tmem_base;
  if (tid == 0) {
    const uint32_t idesc = idesc_tf32(M, N);
    const int npass = split ? 3 : 1;
    int first = 1;
    for (int pass = 0; pass < npass; ++pass) {
      const uint8_t* a = (pass == 2) ? sAl : sAh;   // hi*hi, hi*lo, lo*hi
      const uint8_t* b = (pass == 1) ? sBl : sBh;
      for (int kk = 0; kk < K; kk += 8) {
        // K step of 8 fp32 = two core matrices along K: start at k = kk
        const uint64_t da = make_desc(smem_u32(a) + (kk >> 2) * (M / 8 * 128), M / 8 * 128, 128);
        const uint64_t db = make_desc(smem_u32(b) + (kk >> 2) * (N / 8 * 128), N / 8 * 128, 128);
        const uint32_t acc = first ? 0u : 1u;
        first = 0;
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n"
            ::"r"(tm), "l"(da), "l"(db), "r"(idesc), "r"(acc));
      }
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&mbar)));
  }
  // wait for the MMAs (phase 0)
  {
    uint32_t done = 0;
    while (!done) {
      asm volatile("{\n\t.reg .pred P1;\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n\tselp.b32 %0, 1, 0, P1;\n\t}\n"
                   : "=r"(done) : "r"(smem_u32(&mbar)), "r"(0));
    }
  }
  asm volatile("tcgen05.fence::after_thread_sync;");
  // epilogue: warp w reads TMEM lanes 32w..32w+31, 32 columns each
  uint32_t v[32];
  const uint32_t taddr = tm + ((uint32_t)(warp * 32) << 16);
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
        "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
        "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
        "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;");
  const int row = tid;  // 128 threads: one accumulator row each
  for (int c = 0; c < N; ++c) D[row * N + c] = __uint_as_float(v[c]);
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tm), "n"(32));
}

int main() {
  std::vector<float> A(M * K), B(N * K), D(M * N);
  srand(1);
  for (auto& x : A) x = (float)((rand() / (double)RAND_MAX) * 2 - 1);
  for (auto& x : B) x = (float)((rand() / (double)RAND_MAX) * 2 - 1);
  float *dA, *dB, *dD;
  cudaMalloc(&dA, A.size() * 4); cudaMalloc(&dB, B.size() * 4); cudaMalloc(&dD, D.size() * 4);
  cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
  const size_t smem = 2 * (M + N) * K * 4;
  cudaFuncSetAttribute(umma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  for (int split = 0; split < 2; ++split) {
    cudaMemset(dD, 0, D.size() * 4);
    umma_kernel<<<1, 128, smem>>>(dA, dB, dD, split);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("{\"error\": \"%s\"}\n", cudaGetErrorString(e)); return 1; }
    cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
    double maxrel = 0, maxabs = 0;
    for (int i = 0; i < M; ++i)
      for (int j = 0; j < N; ++j) {
        double ref = 0;
        for (int k = 0; k < K; ++k) ref += (double)A[i * K + k] * (double)B[j * K + k];
        const double err = fabs(D[i * N + j] - ref);
        maxabs = fmax(maxabs, err);
        maxrel = fmax(maxrel, err / (fabs(ref) + 1e-3));
      }
    printf("{\"split\": %d, \"max_abs_err\": %.3e, \"max_rel_err\": %.3e, \"D00\": %f}\n", split, maxabs, maxrel, D[0]);
  }
  return 0;
}
