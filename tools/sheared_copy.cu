// Access-pattern ceiling for the stream solve: the same sheared tile walk
// (warp = 8 diagonals x 64 rows, lane = 16 rows of one diagonal) without
// the recurrences.  read: sum the tile (pass-1 traffic); copy: read + write
// lower + transposed upper through smem (pass-3 traffic).
#include <cstdio>
#include <cuda_runtime.h>
constexpr int SUB = 16, DPW = 8, SR = 64;
__device__ __forceinline__ void tc(int t, int& c, int& g) {
  int q = (int)((sqrt(1.0 + (double)t) - 1.0) * 0.5);
  while (4 * (q + 1) * (q + 2) <= t) ++q;
  while (4 * q * (q + 1) > t) --q;
  c = q; g = t - 4 * q * (q + 1);
}
template <bool COPY>
__global__ void __launch_bounds__(128, 4) k(int n, const double2* __restrict__ w, double2* __restrict__ p, int nt, double2* sink) {
  __shared__ double2 sm[4][SR * DPW];
  int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int t = blockIdx.x * 4 + warp;
  if (t >= nt) return;
  int c, g; tc(t, c, g);
  int i0 = c * SR, m0 = g * DPW;
  if (m0 + DPW - 1 >= i0) return;  // interior only
  int dl = lane % DPW, s = lane / DPW, m = m0 + dl, ib = i0 + s * SUB;
  if (ib + SUB > n) return;
  const double2* wp = w + (size_t)ib * n + (ib - m);
  double2 v[SUB];
#pragma unroll
  for (int r = 0; r < SUB; ++r) v[r] = __ldg(wp + (size_t)r * (n + 1));
  if (!COPY) {
    double2 a = make_double2(0, 0);
#pragma unroll
    for (int r = 0; r < SUB; ++r) { a.x += v[r].x; a.y += v[r].y; }
    if (a.x == 12345.0) sink[0] = a;
    return;
  }
  double2* pp = p + (size_t)ib * n + (ib - m);
#pragma unroll
  for (int r = 0; r < SUB; ++r) { pp[(size_t)r * (n + 1)] = v[r]; sm[warp][(s * SUB + r) * DPW + dl] = v[r]; }
  __syncwarp();
  int u = lane % DPW, mm = m0 + u;
  for (int t0 = -(DPW - 1); t0 < SR; t0 += 4) {
    int tt = t0 + lane / DPW, r = tt + u, i = i0 + r;
    if (tt < SR && r >= 0 && r < SR && i >= mm && i < n) {
      double2 xv = sm[warp][r * DPW + u];
      p[(size_t)(i - mm) * n + i] = make_double2(xv.x, -xv.y);
    }
  }
}
int main() {
  for (int n : {2048, 4096}) {
    size_t bytes = (size_t)n * n * 16;
    double2 *w, *p, *sink;
    cudaMalloc(&w, bytes); cudaMalloc(&p, bytes); cudaMalloc(&sink, 64);
    cudaMemset(w, 0, bytes);
    int C = n / SR, nt = 4 * C * (C + 1);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int copy = 0; copy < 2; ++copy) {
      for (int rep = 0; rep < 3; ++rep) {
        if (copy) k<true><<<(nt + 3) / 4, 128>>>(n, w, p, nt, sink); else k<false><<<(nt + 3) / 4, 128>>>(n, w, p, nt, sink);
      }
      cudaEventRecord(e0);
      for (int rep = 0; rep < 10; ++rep) {
        if (copy) k<true><<<(nt + 3) / 4, 128>>>(n, w, p, nt, sink); else k<false><<<(nt + 3) / 4, 128>>>(n, w, p, nt, sink);
      }
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1); ms /= 10;
      double lower = (double)n * n / 2 * 16;
      double traffic = copy ? 3 * lower : lower;
      printf("{\"n\":%d,\"mode\":\"%s\",\"us\":%.1f,\"GBps\":%.0f}\n", n, copy ? "read+write_lower+upper" : "read", ms * 1e3, traffic / ms / 1e6);
    }
    cudaFree(w); cudaFree(p); cudaFree(sink);
  }
  return 0;
}
