// tcgen05.mma kind::i8 issue-rate microbenchmark for sm_100a (the INT8
// tensor-core peak the residue GEMM is measured against).  No global-memory
// traffic: every CTA issues back-to-back MMAs from (pseudo-random) shared-memory
// operands into two alternating TMEM accumulators, one elected thread per
// CTA (cta_group::1, M = 128, N = 256, K = 32) or per CTA pair
// (cta_group::2, M = 256, N = 256, K = 32, the residue GEMM's shape).
// One JSON line per variant and duration: int8 TOPS (2 ops per MAC) from
// CUDA events, plus MACs/clk/SM from clock64.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/i8_peaks tools/i8_peaks.cu
//   tools/i8_peaks [burst_ms=20] [sustained_ms=4000]
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>

#define CK(x)                                                          \
  do {                                                                 \
    cudaError_t e = (x);                                               \
    if (e != cudaSuccess) {                                            \
      printf("CUDA %s @%d\n", cudaGetErrorString(e), __LINE__);        \
      return 1;                                                        \
    }                                                                  \
  } while (0)

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr) {  // K-major, 64 B swizzle
  return (uint64_t)((saddr & 0x3FFFF) >> 4) | ((uint64_t)1 << 16) | ((uint64_t)(512 >> 4) << 32) |
         ((uint64_t)1 << 46) | ((uint64_t)4 << 61);
}
template <int M>
__host__ __device__ constexpr uint32_t idesc() {
  return (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(256 >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

template <int CG>
__global__ void __launch_bounds__(128, 1) k_mma(long long iters, long long* clk) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  __shared__ uint32_t tmem_slot;
  __shared__ __align__(8) uint64_t bar;
  // pseudo-random operand bytes (zeros would under-state the power draw)
  for (int i = threadIdx.x; i < 64 * 1024 / 4; i += blockDim.x) {
    uint32_t x = (uint32_t)i * 2654435761u + blockIdx.x * 40503u + 12345u;
    x ^= x >> 13;
    x *= 0x5bd1e995u;
    x ^= x >> 15;
    reinterpret_cast<uint32_t*>(smem)[i] = x;
  }
  uint32_t rank = 0;
  if (CG == 2) asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (threadIdx.x < 32) {
    if (CG == 1) {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tmem_slot)));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    } else {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tmem_slot)));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    }
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;");
  if (CG == 2)
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  else
    __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tmem_slot;
  long long t0 = clock64();
  if (threadIdx.x == 0 && rank == 0) {
    const uint32_t a = smem_u32(smem), b = a + 16384;
    for (long long i = 0; i < iters; ++i) {
      const uint32_t d = tmem + (uint32_t)(i & 1) * 256;
      const uint64_t ad = sdesc(a + (uint32_t)(i & 1) * 32), bd = sdesc(b + (uint32_t)(i & 1) * 32);
      if (CG == 1)
        asm volatile("tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, 1;" ::"r"(d), "l"(ad), "l"(bd),
                     "r"(idesc<128>()));
      else
        asm volatile("tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, 1;" ::"r"(d), "l"(ad), "l"(bd),
                     "r"(idesc<256>()));
    }
    if (CG == 1)
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                       smem_u32(&bar))
                   : "memory");
    else
      asm volatile(
          "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
              smem_u32(&bar)),
          "h"((unsigned short)3)
          : "memory");
  }
  if (threadIdx.x == 0) {
    asm volatile(
        "{\n\t.reg .pred p;\nW:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W;\n\t}" ::"r"(
            smem_u32(&bar))
        : "memory");
  }
  long long t1 = clock64();
  asm volatile("tcgen05.fence::before_thread_sync;");
  if (CG == 2)
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  else
    __syncthreads();
  if (threadIdx.x < 32) {
    if (CG == 1)
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
    else
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  }
  if (threadIdx.x == 0) clk[blockIdx.x] = t1 - t0;
}

template <int CG>
static int run(const char* name, int sms, double target_ms) {
  const int smem = 64 * 1024 + 1024;
  CK(cudaFuncSetAttribute(k_mma<CG>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  long long* clk;
  CK(cudaMalloc(&clk, sizeof(long long) * sms));
  const int grid = CG == 2 ? sms / 2 * 2 : sms;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(128);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = CG;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  // MACs per MMA per SM: 128 x 256 x 32 in both variants (a pair does 256 x 256 x 32)
  const double macs_per_sm_mma = 128.0 * 256 * 32;
  long long iters = 1000;
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  float ms = 0;
  for (int rep = 0; rep < 8; ++rep) {  // calibrate the iteration count to the target duration
    CK(cudaEventRecord(e0));
    CK(cudaLaunchKernelEx(&cfg, k_mma<CG>, iters, clk));
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    CK(cudaGetLastError());
    CK(cudaEventElapsedTime(&ms, e0, e1));
    if (ms > 0.8 * target_ms) break;
    iters = (long long)(iters * (target_ms / (ms > 0.01 ? ms : 0.01)));
  }
  long long* h = (long long*)malloc(sizeof(long long) * grid);
  CK(cudaMemcpy(h, clk, sizeof(long long) * grid, cudaMemcpyDeviceToHost));
  double cyc = 0;
  for (int i = 0; i < grid; ++i) cyc = cyc > h[i] ? cyc : (double)h[i];
  const double ops = 2.0 * macs_per_sm_mma * iters * grid;
  printf("{\"bench\": \"%s\", \"target_ms\": %.0f, \"ms\": %.3f, \"iters\": %lld, \"sms\": %d, \"tops\": %.1f, "
         "\"macs_per_clk_sm\": %.1f, \"clk_mhz_effective\": %.0f}\n",
         name, target_ms, ms, iters, grid, ops / (ms * 1e-3) / 1e12, macs_per_sm_mma * iters / cyc,
         cyc / (ms * 1e-3) / 1e6);
  fflush(stdout);
  free(h);
  cudaFree(clk);
  return 0;
}

int main(int argc, char** argv) {
  const double burst = argc > 1 ? atof(argv[1]) : 20.0, sustained = argc > 2 ? atof(argv[2]) : 4000.0;
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  if (run<1>("tcgen05.mma.cta_group::1.kind::i8 128x256x32 burst", sms, burst)) return 1;
  if (run<2>("tcgen05.mma.cta_group::2.kind::i8 256x256x32 burst", sms, burst)) return 1;
  if (run<2>("tcgen05.mma.cta_group::2.kind::i8 256x256x32 sustained", sms, sustained)) return 1;
  if (run<1>("tcgen05.mma.cta_group::1.kind::i8 128x256x32 sustained", sms, sustained)) return 1;
  return 0;
}
