// wmd_build_exact.cu — a2 on the 5th-generation tensor cores, exact: the query x vocabulary
// distance table (PAPER.md:98, :118-123; the "GEMM-like" distance of §6, :259-268) from integer
// products, so the |a|^2 + |b|^2 - 2 a.b form has no cancellation error at all.
//
// Fixed point (once per handle, at wmd_create): with e = the exponent of max|E| (max|E| < 2^e),
//     n_kt = rint(E_kt * 2^F),   F = B - e,   |n_kt| <= 2^B,   B = 26 for dp <= 320
// (B is the largest value for which every intermediate below fits in int64, given dp). The
// rounding is the only approximation: |E_kt - n_kt 2^-F| <= 2^-(F+1), about one FP32 ulp of the
// largest coordinates. Each n is split into four byte limbs, n = L0 + 2^8 L1 + 2^16 L2 + 2^24 L3
// (balanced base-256 digits L_a in [-128, 127], |L3| <= 4), stored as four planes;
// nn_k = sum_t n_kt^2 exactly in int64.
//
// Per query row i (word sel_i) and vocabulary word k, the tensor cores compute the 16 limb
// products  P_ab = sum_t L_a(n_k,t) L_b(n_sel_i,t)  (tcgen05.mma kind::i8, s8 x s8 -> s32)
// accumulated by g = a + b into seven int32 TMEM accumulators A_g (|A_g| <= 4 dp 128^2 < 2^31):
// the B operand holds the four limbs of the 32 query rows side by side (N = 128, column
// 32 b + i), and the MMA of vocabulary limb a writes TMEM columns from 32 a, so its column block
// b lands on accumulator a + b: four N = 128 MMAs per K-step (the accumulators are zeroed by the
// epilogue after it reads them),
// and the epilogue forms, in int64,
//     dot = sum_g A_g 2^(8g),   M_ik^2 2^(2F) = (nn_k - dot) + (nn_sel_i - dot)    (exact)
//     M_ik = sqrt(float(M^2 2^(2F))) * 2^-F          (two roundings: M within ~1 ulp of the
//                                                      distance between the quantised rows)
// so M_{i,sel_i} = 0 exactly and near-duplicate words lose nothing to cancellation.
//
// Block: 128 threads, 128 vocabulary rows (TMEM lanes, MMA M) x 32 query rows per pass (MMA N);
// v_r > 32 runs ceil(v_r/32) passes over the same rows (the A tile is re-read, mostly from L2).
// (16 MMAs of N = 32 per K-step measured tensor-pipe bound: 68 % busy at 2.9 TB/s.)
// Operands (K-major, no swizzle, core matrices of 8 rows x 16 B): A = the vocabulary limbs,
// one 3-D TMA box per 32-coordinate K-step (128 rows x 16 B x 2 chunks x 4 planes = 16 KB) into
// a 4-stage mbarrier ring (expect-tx); B = the pass's 32 query rows, all K-steps resident in
// shared memory (cp.async gather of the selected rows). One thread issues the TMA loads and the
// 16 MMAs per K-step, committing each step to the stage's "empty" barrier; the refill of a stage
// waits for the step before the one just issued, so the tensor pipe always has a step queued.
// Epilogue: 7 tcgen05.ld (32x32b.x32) per pass, int64 combine, sqrt, column minimum, Mx (and
// K~ for the per-iteration path). Bound: reading the limb planes (4 B per coordinate) from HBM.
#include <algorithm>
#include <cfloat>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <cuda.h>
#include <cudaTypedefs.h>

#include "wmd_internal.h"
#include "wmd_umma.cuh"

namespace wmd {
namespace {

using umma::su32;

constexpr int XM = 128;                 // vocabulary rows per block (MMA M, TMEM lanes)
constexpr int XN = 32;                  // query rows per pass (MMA N)
constexpr int XK = 32;                  // coordinates (= bytes per limb) per K-step (MMA K)
constexpr int XL = 4;                   // limbs
constexpr int kMaxStages = 8;           // TMA ring stages (as many as shared memory allows)
constexpr int XT = 192;                 // warps: TMA, MMA, 4 x epilogue
constexpr int XA = XM * XK * XL;        // A bytes per stage (16 KB)
constexpr int XB = XN * XK * XL;        // B bytes per K-step (4 KB)
constexpr uint32_t XCOLS = 512;         // TMEM: two sets of 7 accumulators x 32 columns
constexpr int kMaxExactDp = 1280;       // query limbs resident in shared memory: 128 B per coordinate

// kind::i8 instruction descriptor: S32 accumulate, signed A and B, N = 4 limbs x 32 query rows,
// M = 128, both K-major
constexpr uint32_t kIdescI8 = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)((XL * XN) >> 3) << 17) |
                              ((uint32_t)(XM >> 4) << 24);

__device__ __forceinline__ void mma_i8(uint32_t tmem, uint64_t da, uint64_t db, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}\n"
      ::"r"(tmem), "l"(da), "l"(db), "r"(idesc), "r"(acc));
}

__device__ __forceinline__ void cp16z(void* dst, const void* src, bool valid) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(su32(dst)), "l"(src), "r"(valid ? 16 : 0)
               : "memory");
}

// Persistent, warp-specialised: one block per SM, tiles blockIdx.x, + gridDim.x, ...
//   warp 0 (one lane): TMA producer, K-step G of the block's job into ring stage G % stages
//   warp 1 (one lane): MMA issuer, 16 MMAs per K-step into accumulator set U & 1 (of two)
//   warps 2-5: epilogue of accumulator set U & 1 (TMEM lane quarter warp % 4), released to the
//              MMA warp as soon as its tcgen05.ld are done
// so the loads of the next tile stream while this tile's products finish and its epilogue runs.
// The query limbs of every pass stay resident in shared memory for the whole kernel.
__global__ void __launch_bounds__(XT, 1) build_mx_exact_kernel(
    const __grid_constant__ CUtensorMap tmap, const uint8_t* __restrict__ limbs,
    const long long* __restrict__ nn, int64_t V, int64_t row0, int64_t row1, int dp,
    const int32_t* __restrict__ sel, int v_r, int ld, float inv_scale, float lambda,
    float* __restrict__ Kt, float* __restrict__ Mx, int stages) {
  extern __shared__ __align__(1024) uint8_t xs_raw[];
  uint8_t* const ring = xs_raw + ((1024u - (su32(xs_raw) & 1023u)) & 1023u);  // [stages][XA]
  uint8_t* const bq = ring + stages * XA;                                      // [npass][nsteps][XB]
  __shared__ uint32_t tmem_base;
  __shared__ __align__(8) uint64_t full[kMaxStages], empty[kMaxStages], accf[2], acce[2];
  __shared__ long long qn[4 * XN];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int nsteps = dp / XK, nch = dp / 16;
  const int npass = (v_r + XN - 1) / XN;
  const int64_t ntiles = (row1 - row0 + XM - 1) / XM;
  const int ldx = ld + 4;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(&tmem_base)), "n"(XCOLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 32) {
    for (int i = 0; i < stages; ++i) {
      umma::mbar_init(&full[i], 1);
      umma::mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      umma::mbar_init(&accf[i], 1);
      umma::mbar_init(&acce[i], 4);   // one arrival per epilogue warp
    }
    asm volatile("fence.mbarrier_init.release.cluster;");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmap)) : "memory");
  }
  // the query limbs of every pass: rows p*32 .. p*32 + 31 of sel (zeros past v_r), every K-step
  const int nb = npass * nsteps * XL * 2 * XN;
  for (int x = tid; x < nb; x += XT) {
    const int r = x % XN;
    int t = x / XN;
    const int h = t & 1;
    t >>= 1;
    const int a = t % XL;
    t /= XL;
    const int s = t % nsteps, p = t / nsteps;
    const int i = p * XN + r;
    const bool ok = i < v_r;
    const int64_t row = ok ? sel[i] : 0;
    cp16z(bq + (p * nsteps + s) * XB + ((h * XL + a) * XN + r) * 16,   // N row 32 a + r
          limbs + (((int64_t)a * nch + 2 * s + h) * V + row) * 16, ok);
  }
  asm volatile("cp.async.commit_group;" ::: "memory");
  for (int x = tid; x < npass * XN; x += XT) qn[x] = x < v_r ? nn[sel[x]] : 0;
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();  // tmem_base
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (warp >= 2) {  // both accumulator sets start at zero (the MMAs always accumulate)
    for (int c = 0; c < 512; c += 32) umma::tmem_zero32(tmem_base + ((uint32_t)(32 * (warp & 3)) << 16) + (uint32_t)c);
    umma::tmem_wait_st();
  }
  asm volatile("cp.async.wait_group 0;" ::: "memory");
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic-proxy writes -> tensor core
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tm = tmem_base;

  if (warp == 0) {
    if (lane == 0) {  // TMA producer
      int G = 0;
      for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
        const int c0 = (int)(2 * (row0 + t * XM));
        for (int p = 0; p < npass; ++p) {
          for (int s = 0; s < nsteps; ++s, ++G) {
            const int st = G % stages;
            if (G >= stages) umma::mbar_wait(su32(&empty[st]), ((G / stages) - 1) & 1);
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&full[st])), "r"(XA) : "memory");
            asm volatile(
                "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
                ::"r"(su32(ring + st * XA)), "l"(reinterpret_cast<uint64_t>(&tmap)), "r"(c0), "r"(2 * s), "r"(0),
                "r"(su32(&full[st]))
                : "memory");
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // MMA issuer
      int G = 0, U = 0;
      for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
        for (int p = 0; p < npass; ++p, ++U) {
          const int buf = U & 1;
          if (U >= 2) umma::mbar_wait(su32(&acce[buf]), ((U >> 1) - 1) & 1);
          asm volatile("tcgen05.fence::after_thread_sync;");
          const uint32_t acc = tm + 256u * (uint32_t)buf;
          for (int s = 0; s < nsteps; ++s, ++G) {
            const int st = G % stages;
            umma::mbar_wait(su32(&full[st]), (G / stages) & 1);
            asm volatile("tcgen05.fence::after_thread_sync;");
            const uint32_t a0 = su32(ring + st * XA), b0 = su32(bq + (p * nsteps + s) * XB);
            const uint64_t db = umma::desc(b0, XL * XN * 16, 128);
#pragma unroll
            for (int a = 0; a < XL; ++a)  // vocabulary limb a x query limbs 0..3 -> accumulators a .. a + 3
              mma_i8(acc + 32u * (uint32_t)a, umma::desc(a0 + a * 2 * XM * 16, XM * 16, 128), db, kIdescI8, 1u);
            umma::commit(&empty[st]);   // the stage is free once these MMAs have read it
          }
          umma::commit(&accf[buf]);     // the pass's products are complete
        }
      }
    }
  } else {  // epilogue: row r of the tile = TMEM lane r, lane quarter warp % 4
    const int r = 32 * (warp & 3) + lane;
    const uint32_t lanes = (uint32_t)(32 * (warp & 3)) << 16;
    int U = 0;
    for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
      const int64_t k = row0 + t * XM + r;
      const bool kok = k < row1;
      const long long nnk = kok ? nn[k] : 0;
      float* const out = Mx + k * ldx;
      float mn = FLT_MAX;
      for (int p = 0; p < npass; ++p, ++U) {
        const int buf = U & 1, i0 = p * XN;
        umma::mbar_wait(su32(&accf[buf]), (U >> 1) & 1);
        __syncwarp();  // tcgen05.ld is warp-collective
        asm volatile("tcgen05.fence::after_thread_sync;");
        long long dot[XN];
#pragma unroll
        for (int c = 0; c < XN; ++c) dot[c] = 0;
#pragma unroll
        for (int g = 0; g < 2 * XL - 1; ++g) {
          uint32_t v[32];
          umma::tmem_ld32(tm + lanes + 256u * (uint32_t)buf + 32u * (uint32_t)g, v);
#pragma unroll
          for (int c = 0; c < XN; ++c) dot[c] += (long long)(int32_t)v[c] * (1LL << (8 * g));
          umma::tmem_zero32(tm + lanes + 256u * (uint32_t)buf + 32u * (uint32_t)g);
        }
        umma::tmem_wait_st();
        asm volatile("tcgen05.fence::before_thread_sync;");
        __syncwarp();
        if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(&acce[buf])) : "memory");
        if (kok) {
#pragma unroll
          for (int c4 = 0; c4 < XN; c4 += 4) {
            float m4[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              const int c = c4 + u;
              const long long m2 = (nnk - dot[c]) + (qn[i0 + c] - dot[c]);
              const float m = __fsqrt_rn(__ll2float_rn(m2)) * inv_scale;
              const bool real = i0 + c < v_r;
              m4[u] = real ? m : 0.f;
              if (real) mn = fminf(mn, m);
            }
            if (i0 + c4 < ld) *reinterpret_cast<float4*>(out + i0 + c4) = make_float4(m4[0], m4[1], m4[2], m4[3]);
          }
        }
      }
      if (kok) {
        for (int x = std::min(npass * XN, ld); x < ldx; ++x) out[x] = x == ld ? mn : 0.f;
        if (Kt) {
          for (int x = 0; x < ld; ++x) Kt[k * ld + x] = x < v_r ? expf(-lambda * (out[x] - mn)) : 0.f;
        }
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tm), "n"(XCOLS));
}

__global__ void abs_max_kernel(const float* __restrict__ E, int64_t n, unsigned* __restrict__ out) {
  float m = 0.f;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    m = fmaxf(m, fabsf(E[i]));
#pragma unroll
  for (int off = 16; off; off >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, off));
  if ((threadIdx.x & 31) == 0) atomicMax(out, __float_as_uint(m));  // |x| >= 0: bits order as values
}

// one thread per vocabulary row: limbs of n = rint(E * 2^F) into the chunk-major planes
// limbs[a][chunk][row][16 B], and nn = sum n^2
__global__ void limbs_kernel(const float* __restrict__ E, int64_t V, int dp, int F, uint8_t* __restrict__ limbs,
                             long long* __restrict__ nn) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= V) return;
  const int nch = dp / 16;
  long long acc = 0;
  for (int c = 0; c < nch; ++c) {
    uint32_t w[XL][4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const float4 x = *reinterpret_cast<const float4*>(E + k * dp + 16 * c + 4 * q);
      const float xs[4] = {x.x, x.y, x.z, x.w};
      uint32_t b[XL] = {0u, 0u, 0u, 0u};
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int n = __float2int_rn(ldexpf(xs[u], F));
        acc += (long long)n * n;
        int rest = n;
#pragma unroll
        for (int a = 0; a < XL; ++a) {  // balanced digits: rest = L + 256 rest', L in [-128, 127]
          const int L = ((rest + 128) & 255) - 128;
          rest = (rest - L) >> 8;
          b[a] |= ((uint32_t)L & 0xffu) << (8 * u);
        }
      }
#pragma unroll
      for (int a = 0; a < XL; ++a) w[a][q] = b[a];
    }
#pragma unroll
    for (int a = 0; a < XL; ++a)
      *reinterpret_cast<uint4*>(limbs + (((int64_t)a * nch + c) * V + k) * 16) = make_uint4(w[a][0], w[a][1], w[a][2], w[a][3]);
  }
  nn[k] = acc;
}

}  // namespace

int exact_frac_bits_limit(int dp) {
  // M^2 2^(2F) <= dp (2^(B+1))^2 < 2^63  and  |n| <= 2^B with the top limb within s8
  int b = 0;
  while (b < 26 && std::ldexp((double)dp, 2 * (b + 1) + 2) < std::ldexp(1.0, 63)) ++b;
  return b;
}

bool exact_build_supported(int dp) { return dp % XK == 0 && dp <= kMaxExactDp; }

void free_exact_e(ExactE* x) {
  if (x->limbs) cudaFree(x->limbs);
  if (x->nn) cudaFree(x->nn);
  x->limbs = nullptr;
  x->nn = nullptr;
  x->ok = false;
}

int prepare_exact_e(const float* E, int64_t V, int dp, ExactE* x, cudaStream_t st) {
  free_exact_e(x);
  x->V = V;
  x->dp = dp;
  if (!exact_build_supported(dp) || V <= 0 || 2 * V > INT32_MAX) return 0;  // unsupported shape: not an error
  unsigned* d_max = nullptr;
  cudaError_t e = cudaMallocAsync(&d_max, sizeof(unsigned), st);
  if (e != cudaSuccess) return (int)e;
  unsigned bits = 0u;
  cudaMemsetAsync(d_max, 0, sizeof(unsigned), st);
  abs_max_kernel<<<device_sms() * 4, 256, 0, st>>>(E, V * dp, d_max);
  cudaMemcpyAsync(&bits, d_max, sizeof bits, cudaMemcpyDeviceToHost, st);
  cudaFreeAsync(d_max, st);
  if ((e = cudaStreamSynchronize(st)) != cudaSuccess) return (int)e;
  float amax;
  std::memcpy(&amax, &bits, sizeof amax);
  int ex = 0;
  if (amax > 0.f) std::frexp(amax, &ex);  // amax < 2^ex
  const int B = exact_frac_bits_limit(dp);
  const int F = B - ex;
  if (F < -120 || F > 120) return 0;     // no representable 2^-F: the exact build is unavailable
  x->frac_bits = F;
  x->inv_scale = std::ldexp(1.0f, -F);
  if ((e = cudaMalloc(&x->limbs, (size_t)XL * V * dp)) != cudaSuccess) return (int)e;
  if ((e = cudaMalloc(&x->nn, (size_t)V * sizeof(long long))) != cudaSuccess) return (int)e;
  limbs_kernel<<<(unsigned)((V + 127) / 128), 128, 0, st>>>(E, V, dp, F, x->limbs, x->nn);
  if ((e = cudaGetLastError()) != cudaSuccess) return (int)e;
  // TMA map of the planes in 8-byte elements: dims (innermost first) 2 V (the 16-byte row
  // pieces of one chunk, contiguous), dp/16 chunks, 4 planes; a box of 256 x 2 x 4 elements is
  // 128 rows x 2 chunks x 4 planes, each (plane, chunk) a contiguous 2 KB run
  static const PFN_cuTensorMapEncodeTiled_v12000 encode = [] {   // thread-safe one-time lookup
    cudaDriverEntryPointQueryResult q;
    void* fn = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      fn = nullptr;
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  }();
  if (!encode) {   // no tensor-map encoder in this driver: the exact build is unavailable
    free_exact_e(x);
    return 0;
  }
  static_assert(sizeof(CUtensorMap) <= sizeof(x->tmap), "tensor map storage");
  const cuuint64_t dims[3] = {(cuuint64_t)V * 2, (cuuint64_t)(dp / 16), (cuuint64_t)XL};
  const cuuint64_t strides[2] = {(cuuint64_t)V * 16, (cuuint64_t)V * dp};
  const cuuint32_t box[3] = {2 * XM, 2, XL};
  const cuuint32_t estr[3] = {1, 1, 1};
  const CUresult r = encode(reinterpret_cast<CUtensorMap*>(x->tmap), CU_TENSOR_MAP_DATA_TYPE_UINT64, 3, x->limbs, dims,
                            strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {   // shape the TMA unit does not take: unavailable, not an error
    free_exact_e(x);
    return 0;
  }
  x->ok = true;
  return 0;
}

bool launch_build_exact(const ExactE& x, int64_t row0, int64_t row1, const int32_t* sel, int v_r, int ld,
                        float lambda, float* Kt, float* Mx, cudaStream_t st) {
  static PerDevice attr, optin;
  const int budget = optin.get([&] {
    int dev = 0, v = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    return v;
  }) - 2048;  // static shared memory (barriers, norms) and slack
  const int npass = (v_r + XN - 1) / XN;
  const int bbytes = npass * (x.dp / XK) * XB;
  const int stages = std::min(kMaxStages, (budget - 1024 - bbytes) / XA);
  if (stages < 2) return false;  // the query limbs do not fit: the caller runs another build
  if (row1 <= row0) return true;
  attr.get([&] {
    return (int)cudaFuncSetAttribute(build_mx_exact_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, budget);
  });
  const size_t smem = (size_t)stages * XA + bbytes + 1024;
  const int64_t ntiles = (row1 - row0 + XM - 1) / XM;
  const unsigned grid = (unsigned)std::min<int64_t>(ntiles, device_sms());
  build_mx_exact_kernel<<<grid, XT, smem, st>>>(*reinterpret_cast<const CUtensorMap*>(x.tmap), x.limbs, x.nn, x.V,
                                                row0, row1, x.dp, sel, v_r, ld, x.inv_scale, lambda, Kt, Mx, stages);
  return true;
}

}  // namespace wmd
