// FP64 issue-rate microbenchmark for sm_100a: DMMA (mma.sync f64 shapes) vs DFMA.
// Prints one JSON line per variant: flop/s, flop/clk/SM (from clock64 deltas).
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

template <int ILP>
__global__ void k_dmma884(double* out, int iters, long long* clk) {
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
  double c[ILP][2];
#pragma unroll
  for (int i = 0; i < ILP; ++i) { c[i][0] = i; c[i][1] = -i; }
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < ILP; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
  }
  long long t1 = clock64();
  double s = 0;
#pragma unroll
  for (int i = 0; i < ILP; ++i) s += c[i][0] + c[i][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) clk[blockIdx.x] = t1 - t0;
}

template <int ILP>
__global__ void k_dmma1684(double* out, int iters, long long* clk) {
  double a0 = threadIdx.x * 1e-3, a1 = a0 + 1, b = 1.0 + threadIdx.x * 1e-4;
  double c[ILP][4];
#pragma unroll
  for (int i = 0; i < ILP; ++i) { c[i][0] = i; c[i][1] = -i; c[i][2] = 1; c[i][3] = 2; }
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < ILP; ++i)
      asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3]) : "d"(a0), "d"(a1), "d"(b));
  }
  long long t1 = clock64();
  double s = 0;
#pragma unroll
  for (int i = 0; i < ILP; ++i) s += c[i][0] + c[i][1] + c[i][2] + c[i][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) clk[blockIdx.x] = t1 - t0;
}

template <int ILP>
__global__ void k_dmma16816(double* out, int iters, long long* clk) {
  double a[8], b[4];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3 + i;
#pragma unroll
  for (int i = 0; i < 4; ++i) b[i] = 1.0 + threadIdx.x * 1e-4 + i;
  double c[ILP][4];
#pragma unroll
  for (int i = 0; i < ILP; ++i) { c[i][0] = i; c[i][1] = -i; c[i][2] = 1; c[i][3] = 2; }
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < ILP; ++i)
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3])
                   : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                     "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
  }
  long long t1 = clock64();
  double s = 0;
#pragma unroll
  for (int i = 0; i < ILP; ++i) s += c[i][0] + c[i][1] + c[i][2] + c[i][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) clk[blockIdx.x] = t1 - t0;
}

template <int ILP>
__global__ void k_dfma(double* out, int iters, long long* clk) {
  double x[ILP];
  double a = 1.0 + threadIdx.x * 1e-9, b = 1e-9;
#pragma unroll
  for (int i = 0; i < ILP; ++i) x[i] = i;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < ILP; ++i) asm volatile("fma.rn.f64 %0, %0, %1, %2;" : "+d"(x[i]) : "d"(a), "d"(b));
  }
  long long t1 = clock64();
  double s = 0;
#pragma unroll
  for (int i = 0; i < ILP; ++i) s += x[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) clk[blockIdx.x] = t1 - t0;
}

typedef void (*kfn)(double*, int, long long*);

static int run(const char* name, kfn k, double flop_per_warp_iter, int blocks, int threads, int iters) {
  double* out; long long* clk;
  CK(cudaMalloc(&out, sizeof(double) * blocks * threads));
  CK(cudaMalloc(&clk, sizeof(long long) * blocks));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int w = 0; w < 2; ++w) k<<<blocks, threads>>>(out, iters, clk);
  CK(cudaDeviceSynchronize());
  cudaEventRecord(e0);
  k<<<blocks, threads>>>(out, iters, clk);
  cudaEventRecord(e1);
  CK(cudaEventSynchronize(e1));
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  long long* hclk = new long long[blocks];
  cudaMemcpy(hclk, clk, sizeof(long long) * blocks, cudaMemcpyDeviceToHost);
  long long mx = 0; for (int i = 0; i < blocks; ++i) if (hclk[i] > mx) mx = hclk[i];
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double warps = double(blocks) * threads / 32;
  double flop = warps * iters * flop_per_warp_iter;
  // per-SM clk rate: blocks per SM resident simultaneously assumed (blocks <= sms * occ)
  double flop_per_clk_sm = flop / sms / double(mx);
  printf("{\"bench\":\"%s\",\"blocks\":%d,\"threads\":%d,\"ms\":%.4f,\"tflops\":%.3f,\"flop_per_clk_per_sm\":%.2f,\"max_clk\":%lld,\"implied_mhz\":%.1f}\n",
         name, blocks, threads, ms, flop / ms / 1e9, flop_per_clk_sm, mx, mx / (ms * 1e3));
  delete[] hclk; cudaFree(out); cudaFree(clk);
  return 0;
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceProp p; cudaGetDeviceProperties(&p, 0);
  printf("{\"device\":\"%s\",\"sms\":%d,\"cc\":\"%d.%d\",\"l2_mb\":%.1f,\"smem_optin\":%zu}\n", p.name, sms, p.major, p.minor,
         p.l2CacheSize / 1048576.0, p.sharedMemPerBlockOptin);
  const int it = 4096;
  for (int thr : {128, 256, 512}) {
    run("dmma_m8n8k4_ilp4", k_dmma884<4>, 4 * 512.0, sms, thr, it);
    run("dmma_m8n8k4_ilp8", k_dmma884<8>, 8 * 512.0, sms, thr, it);
    run("dmma_m16n8k4_ilp4", k_dmma1684<4>, 4 * 1024.0, sms, thr, it);
    run("dmma_m16n8k16_ilp2", k_dmma16816<2>, 2 * 4096.0, sms, thr, it / 4);
    run("dfma_ilp8", k_dfma<8>, 8 * 32 * 2.0, sms, thr, it);
  }
  run("dmma_m8n8k4_ilp8_2x", k_dmma884<8>, 8 * 512.0, 2 * sms, 256, it);
  run("dfma_ilp8_4x", k_dfma<8>, 8 * 32 * 2.0, 4 * sms, 256, it);
  return 0;
}
