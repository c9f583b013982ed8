// Shared helpers for the sm_100a isospectral hot path.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <string>
#include <utility>

#include "../../include/zt.h"

// Per-N operator (opaque to C callers): closed-form sqrt table, deflated
// m = 0 factors, and per-(chunk, diagonal) pivots / carry gains.
struct zt_operator {
  int n = 0, device = 0, C = 0;
  double* sqB = nullptr;
  double* Bq = nullptr;  // (j+1)(N-1-j) as exact doubles
  double* L0 = nullptr;
  double* dinv0 = nullptr;
  double* d0 = nullptr;
  double* lins = nullptr;  // L of the row before every 16-row sub-chunk start
  double* lin = nullptr;
  double* G = nullptr;
  double* H = nullptr;
  double* K = nullptr;
  double* m0x = nullptr;  // m = 0 per-chunk constant-RHS responses
  int2* gen_tiles = nullptr;  // (chunk, group) of the boundary tiles
  int ngen = 0;
  void* block = nullptr;  // single allocation holding every table
};

namespace zt {

extern std::atomic<int64_t> g_launches;

void set_error(const std::string& msg);
int fail(int status, const std::string& msg);
int cuda_fail(cudaError_t e, const char* where);

#define ZT_CUDA_CHECK(expr)                                   \
  do {                                                        \
    cudaError_t _e = (expr);                                  \
    if (_e != cudaSuccess) return ::zt::cuda_fail(_e, #expr); \
  } while (0)

#define ZT_LAUNCHED() ::zt::g_launches.fetch_add(1, std::memory_order_relaxed)

// Programmatic dependent launch along the step's main chain (conversion ->
// residue GEMM -> reconstruction -> update): a kernel launched by launch_pdl
// may start while its stream predecessor drains (its blocks are scheduled,
// set up TMEM / barriers / tensor-map prefetches) and MUST execute
// pdl_wait() before touching memory the predecessor writes or reads (the
// wait returns once every predecessor grid completed and flushed; completion
// is transitive along the chain).  pdl_trigger() lets the dependent launch
// early.  ZT_PDL=0 turns the attribute off (plain stream order).
extern bool g_pdl;
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
#ifndef ZT_PDL_TRIGGER
#define ZT_PDL_TRIGGER 0
#endif
__device__ __forceinline__ void pdl_trigger() {
#if ZT_PDL_TRIGGER
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
#endif
}
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*k)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                              Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = g_pdl ? 1 : 0;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, k, std::forward<Args>(args)...);
}

// progressive final update (zt_gemm.cu, FusedArgs::prog): W_{n+1} rows are
// published block by block for an overlapped device-to-host copy
struct ProgParams {
  const double* wn;
  double* wout;
  double h;
  unsigned int* words;  // zupdate_prog_words(n): pair / row counters, row flags
};

// complex128 as double2 (re, im) — matches numpy/torch interleaved layout
struct cplx {
  double re, im;
};

__device__ __forceinline__ double2 ld2(const double* p) {
  return __ldg(reinterpret_cast<const double2*>(p));
}
__device__ __forceinline__ double2 ld2_plain(const double* p) {
  return *reinterpret_cast<const double2*>(p);
}
__device__ __forceinline__ void st2(double* p, double2 v) { *reinterpret_cast<double2*>(p) = v; }

// Separately rounded real*complex and complex ops (no FMA contraction) so
// sweeps and stencils follow the reference's numpy/numba rounding exactly.
__device__ __forceinline__ double2 rmul(double a, double2 z) {
  return make_double2(__dmul_rn(a, z.x), __dmul_rn(a, z.y));
}
__device__ __forceinline__ double2 csub(double2 a, double2 b) {
  return make_double2(__dsub_rn(a.x, b.x), __dsub_rn(a.y, b.y));
}
__device__ __forceinline__ double2 cadd(double2 a, double2 b) {
  return make_double2(__dadd_rn(a.x, b.x), __dadd_rn(a.y, b.y));
}

// Closed-form block entries (laplacian.py:129-137).  All quantities are
// exact in binary64 for n < 2^26: diag is a half-integer combination.
__device__ __forceinline__ double block_diag(int n, int m, int k) {
  const double s = (n - 1) * 0.5;
  const double kd = (double)k;
  return 2.0 * (s * (2.0 * kd + 1.0 + (double)m) - kd * (kd + (double)m));
}

// Max of a non-negative double via integer atomics on the bit pattern.
// fabs() clears the sign so NaN (0x7ff8...) orders above +inf: a NaN
// residual propagates to "not converged" as in the reference.
__device__ __forceinline__ void atomic_max_nonneg(unsigned long long* addr, double v) {
  atomicMax(addr, (unsigned long long)__double_as_longlong(fabs(v)));
}

}  // namespace zt
