/* A plain C99 consumer of include/zt.h: the drop-in boundary used the way a
 * non-Python host (cgo / JNI / FFI stub) would use it — device pointers from
 * cudaMalloc, sizes, a stream, status codes; no torch, no C++.
 *
 *   gcc -std=c99 -I include -I /usr/local/cuda/include tests/abi_c/zt_c_consumer.c \
 *       -L paper_2206_05466_b200 -lzt -L /usr/local/cuda/lib64 -lcudart -lm -o zt_c_consumer
 *
 * Checks (size-independent properties, the oracle is Python): the round trip
 * lap(lap^-1 W) = W (laplacian.py:341-431), the input gate's status codes, and
 * one midpoint step (integrator.py:141-171) whose result is finite, exactly
 * skew-Hermitian off the diagonal, and whose fixed point W~ reproduces the
 * step: the reported consistency error max|W~ - (h/2)(a - a^H) - (h^2/4) a P~ - W_n|
 * (integrator.py:160-163) is at round-off.  Prints "zt_c_consumer ok". */
#include <math.h>
#include <stdio.h>
#include <stdlib.h>

#include <cuda_runtime_api.h>

#include "zt.h"

#define CHECK_ZT(x)                                                                        \
  do {                                                                                     \
    int rc_ = (x);                                                                         \
    if (rc_ != ZT_OK) {                                                                    \
      fprintf(stderr, "%s -> %s: %s\n", #x, zt_strerror(rc_), zt_last_error());            \
      return 1;                                                                            \
    }                                                                                      \
  } while (0)
#define CHECK_CU(x)                                                                        \
  do {                                                                                     \
    cudaError_t e_ = (x);                                                                  \
    if (e_ != cudaSuccess) {                                                               \
      fprintf(stderr, "%s -> %s\n", #x, cudaGetErrorString(e_));                           \
      return 1;                                                                            \
    }                                                                                      \
  } while (0)

static unsigned long long lcg_state = 0x2206054660ULL;
static double uniform(void) { /* in (-1, 1) */
  lcg_state = lcg_state * 6364136223846793005ULL + 1442695040888963407ULL;
  return ((double)(lcg_state >> 11) / 9007199254740992.0) * 2.0 - 1.0;
}

int main(int argc, char** argv) {
  const int n = argc > 1 ? atoi(argv[1]) : 97;
  const size_t elems = (size_t)n * n, bytes = elems * 2 * sizeof(double);
  double* w = (double*)malloc(bytes);
  double* out = (double*)malloc(bytes);
  if (!w || !out || n < 2) return 1;
  /* W = (A - A^H) / 2 with the trace removed, entries O(1 / n) */
  for (int i = 0; i < n; ++i)
    for (int j = 0; j <= i; ++j) {
      const double re = uniform() / n, im = uniform() / n;
      if (i == j) {
        w[((size_t)i * n + i) * 2] = 0.0;
        w[((size_t)i * n + i) * 2 + 1] = im;
      } else {
        w[((size_t)i * n + j) * 2] = re;
        w[((size_t)i * n + j) * 2 + 1] = im;
        w[((size_t)j * n + i) * 2] = -re;
        w[((size_t)j * n + i) * 2 + 1] = im;
      }
    }
  double tr = 0.0;
  for (int i = 0; i < n; ++i) tr += w[((size_t)i * n + i) * 2 + 1];
  for (int i = 0; i < n; ++i) w[((size_t)i * n + i) * 2 + 1] -= tr / n;

  CHECK_CU(cudaSetDevice(0));
  cudaStream_t st;
  CHECK_CU(cudaStreamCreate(&st));
  double *dw, *dp, *dy, *dnext, *dres;
  void* ws;
  CHECK_CU(cudaMalloc((void**)&dw, bytes));
  CHECK_CU(cudaMalloc((void**)&dp, bytes));
  CHECK_CU(cudaMalloc((void**)&dy, bytes));
  CHECK_CU(cudaMalloc((void**)&dnext, bytes));
  CHECK_CU(cudaMalloc((void**)&dres, 3 * sizeof(double)));
  const size_t ws_bytes = zt_step_workspace_bytes(n);
  CHECK_CU(cudaMalloc(&ws, ws_bytes));
  CHECK_CU(cudaMemcpyAsync(dw, w, bytes, cudaMemcpyHostToDevice, st));

  zt_op_t op;
  CHECK_ZT(zt_op_create(n, 0, &op));
  if (zt_op_n(op) != n) return 1;

  /* gate values, then the round trip lap(lap^-1 W) = W */
  double res[3];
  CHECK_ZT(zt_residuals(n, dw, n, dres, st));
  CHECK_CU(cudaMemcpyAsync(res, dres, sizeof(res), cudaMemcpyDeviceToHost, st));
  CHECK_ZT(zt_stream_solve(op, dw, n, 0, dp, n, 0, 1, st));
  CHECK_ZT(zt_apply_laplacian(op, dp, n, 0, dy, n, 0, -1, 1, st));
  CHECK_CU(cudaMemcpyAsync(out, dy, bytes, cudaMemcpyDeviceToHost, st));
  CHECK_CU(cudaStreamSynchronize(st));
  if (!(res[0] <= 1e-14 && res[1] <= 1e-14 && res[2] > 0.0)) {
    fprintf(stderr, "residuals %g %g %g\n", res[0], res[1], res[2]);
    return 1;
  }
  double num = 0.0, den = 0.0;
  for (size_t k = 0; k < 2 * elems; ++k) {
    num += (out[k] - w[k]) * (out[k] - w[k]);
    den += w[k] * w[k];
  }
  const double rt = sqrt(num / den);
  if (!(rt <= 1e-10)) {
    fprintf(stderr, "round trip relF %g\n", rt);
    return 1;
  }

  /* one midpoint step with the consistency output */
  int iters = 0;
  double residual = -1.0, cons = -1.0;
  CHECK_ZT(zt_midpoint_step(op, dw, dnext, 0.01, 1e-12, 10, ws, ws_bytes, &iters, &residual, &cons, st));
  CHECK_CU(cudaMemcpyAsync(out, dnext, bytes, cudaMemcpyDeviceToHost, st));
  CHECK_CU(cudaStreamSynchronize(st));
  if (iters < 1 || iters > 10 || !(residual <= 1e-12) || !(cons >= 0.0 && cons <= 1e-12)) {
    fprintf(stderr, "step: iterations %d residual %g consistency %g\n", iters, residual, cons);
    return 1;
  }
  double skew = 0.0, moved = 0.0;
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) {
      const double a = out[((size_t)i * n + j) * 2], b = out[((size_t)i * n + j) * 2 + 1];
      const double c = out[((size_t)j * n + i) * 2], d = out[((size_t)j * n + i) * 2 + 1];
      if (!isfinite(a) || !isfinite(b)) return 1;
      if (i != j) skew = fmax(skew, fmax(fabs(a + c), fabs(b - d)));
      moved = fmax(moved, fabs(a - w[((size_t)i * n + j) * 2]));
    }
  /* n = 2 carries only l = 1 (lap^-1 W is a multiple of W): every state is steady */
  if (skew != 0.0 || (n > 2 && moved == 0.0)) {
    fprintf(stderr, "step: max|W + W^H| off the diagonal %g, max change %g\n", skew, moved);
    return 1;
  }

  /* status codes: a matrix that is not skew-Hermitian is rejected by the gate; bad arguments */
  w[2] += 0.5; /* W[0][1].re */
  CHECK_CU(cudaMemcpyAsync(dw, w, bytes, cudaMemcpyHostToDevice, st));
  int rc = zt_midpoint_step(op, dw, dnext, 0.01, 1e-12, 10, ws, ws_bytes, &iters, &residual, NULL, st);
  if (rc != ZT_ESTRUCTURE) {
    fprintf(stderr, "gate: expected ZT_ESTRUCTURE, got %s\n", zt_strerror(rc));
    return 1;
  }
  rc = zt_midpoint_step(op, dw, dnext, -1.0, 1e-12, 10, ws, ws_bytes, &iters, &residual, NULL, st);
  if (rc != ZT_EINVAL) {
    fprintf(stderr, "h < 0: expected ZT_EINVAL, got %s\n", zt_strerror(rc));
    return 1;
  }
  rc = zt_midpoint_step(op, dw, dnext, 0.01, 1e-12, 10, ws, ws_bytes / 2, &iters, &residual, NULL, st);
  if (rc == ZT_OK) {
    fprintf(stderr, "short workspace accepted\n");
    return 1;
  }
  CHECK_ZT(zt_op_destroy(op));
  cudaFree(dw), cudaFree(dp), cudaFree(dy), cudaFree(dnext), cudaFree(dres), cudaFree(ws);
  cudaStreamDestroy(st);
  free(w), free(out);
  printf("zt_c_consumer ok: n=%d round trip %.2e iterations %d residual %.2e consistency %.2e (zt_version %d)\n", n,
         rt, iters, residual, cons, zt_version());
  return 0;
}
