// C ABI (include/zt.h) and the device-resident fixed-point / midpoint step
// driver (integrator.py:96-171) for sm_100a.
#include <cuda_runtime.h>
#include <math.h>
#include <stdio.h>

#include <algorithm>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "zt_tma.cuh"



namespace zt {

std::atomic<int64_t> g_launches{0};
bool g_pdl = [] {
  const char* e = getenv("ZT_PDL");
  return !(e && e[0] == '0');
}();
static thread_local std::string t_err;

static PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;
int encode_tiled_f64(CUtensorMap* map, int rank, const void* base, const cuuint64_t* dims,
                     const cuuint64_t* strides, const cuuint32_t* box, CUtensorMapSwizzle swz) {
  if (!g_encode) {
    cudaDriverEntryPointQueryResult q;
    void* fn = nullptr;
    ZT_CUDA_CHECK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
    if (!fn || q != cudaDriverEntryPointSuccess) return fail(ZT_ECUDA, "cuTensorMapEncodeTiled unavailable");
    g_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  }
  cuuint32_t es[3] = {1, 1, 1};
  CUresult r = g_encode(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, rank, const_cast<void*>(base), dims, strides,
                        box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, swz, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(ZT_ECUDA, "cuTensorMapEncodeTiled failed: " + std::to_string((int)r));
  return ZT_OK;
}

void set_error(const std::string& msg) { t_err = msg; }
int fail(int status, const std::string& msg) {
  t_err = msg;
  return status;
}
int cuda_fail(cudaError_t e, const char* where) {
  t_err = std::string(where) + ": " + cudaGetErrorString(e);
  return ZT_ECUDA;
}

// implemented in zt_solve.cu / zt_gemm.cu
int op_create(int n, int device, zt_operator** out);
int op_destroy(zt_operator* op);
int op_factors(zt_operator* op, double* linv_h, double* dinv_h);
size_t solve_workspace_bytes(int n, int batch);
int stream_solve(zt_operator* op, const double* w, int64_t ldw, int64_t sw, double* p, int64_t ldp,
                 int64_t sp, int batch, void* ws, size_t ws_bytes, cudaStream_t st);
int apply_laplacian(zt_operator* op, const double* w, int64_t ldw, int64_t sw, double* y,
                    int64_t ldy, int64_t sy, int sign, int batch, cudaStream_t st);
size_t resid_workspace_bytes(int n);
int residuals(int n, const double* w, int64_t ldw, double* out, void* ws, cudaStream_t st);
int zgemm(int n, const double* a, int64_t lda, const double* b, int64_t ldb, double* c, int64_t ldc,
          int algo, cudaStream_t st);
int zgemm_update(int n, const double* amat, const double* p, const double* base, const double* xprev,
                 const double* wn, double* out, int64_t ld, double hh, double qq,
                 unsigned long long* resid, unsigned long long* cons, int algo, cudaStream_t st);
int skew_diff(int n, const double* a, double* c, cudaStream_t st);
int zupdate_fused(int n, const double* p, const double* x, double* a, const double* base, const double* xprev,
                  const double* wn, double* out, double hh, double qq, unsigned long long* resid,
                  unsigned long long* cons, unsigned int* sync, int algo, double* planes, double* split,
                  cudaStream_t st, int gemm1_only = 0, double* bbuf = nullptr, const ProgParams* prog = nullptr);
size_t zupdate_prog_words(int n);
size_t oz_update_workspace_bytes(int n);
void oz_profile_enable(bool on);
int oz_update(int n, const double* p, const double* x, double* a, double* bbuf, const double* base,
              const double* xprev, const double* wn, double* out, double hh, double qq, unsigned long long* resid,
              unsigned long long* cons, void* ws, cudaStream_t st, int gemm1_only, cudaEvent_t x_join);
int oz_convert_x(int n, const double* x, void* ws, cudaStream_t st);
int final_commutator(int n, const double* a, const double* wn, double h, double* out, cudaStream_t st);
size_t oz_workspace_bytes(int n);
int oz_zgemm(int n, const double* a, int64_t lda, const double* b, int64_t ldb, int bmode, double* c, int64_t ldc,
             int lower, void* ws, size_t ws_bytes, cudaStream_t st);
int update_pairs(int n, const double* a, const double* bm, double* out, const double* base, const double* xprev,
                 const double* wn, double hh, double qq, unsigned long long* resid, unsigned long long* cons,
                 cudaStream_t st);
size_t zupdate_split_bytes(int n);
int zgemm_rect_scatter(int m, int n, int k, const double* a, int64_t lda, const double* b, int64_t ldb, double* c,
                       int64_t ldc, const unsigned long long* peers, int npeer, int r0, int mloc, int algo,
                       cudaStream_t st);
int zgemm_update_rows_peer(int m, int n, const double* a_rows, const double* p, const double* acol, int mloc,
                           const double* base, const double* xprev, double* out, int64_t ld, double hh, double qq,
                           unsigned long long* resid, const unsigned long long* peers, int npeer, int r0, int algo,
                           cudaStream_t st);
int rows_broadcast(int m, int n, const double* rows, int64_t ld, const unsigned long long* peers, int npeer, int r0,
                   cudaStream_t st);
int zgemm_rect_mirror(int m, int n, int k, const double* a, int64_t lda, const double* b, int64_t ldb, double* c,
                      int64_t ldc, double* mirror, int64_t ld_mirror, int algo, cudaStream_t st);
int update_rows_ew(int m, int n, const double* a_rows, const double* acol, int mloc, const double* b_rows,
                   const double* base, const double* xprev, double* out, int64_t ld, double hh, double qq,
                   unsigned long long* resid, const unsigned long long* peers, int npeer, int r0, cudaStream_t st);
int basis_vectors(int n, int m0, int m1, const long long* off, double* vec, cudaStream_t st);
int grid_eval(int n, int lmax, int nlat, int nlon, const long long* coff, const double* pos, double* work,
              double* field, cudaStream_t st);
int basis_extract(int n, int m0, int m1, const long long* off, const long long* coff, const double* vec,
                  const double* w, int64_t ldw, double* pos, double* neg, cudaStream_t st);
int basis_project(int n, int m0, int m1, const long long* off, const long long* coff, const double* vec,
                  const double* pos, const double* neg, double* w, int64_t ldw, cudaStream_t st);
int zupdate_sync_words(int n);
size_t sum_plane_bytes(int n);
int zgemm_rect(int m, int n, int k, const double* a, int64_t lda, const double* b, int64_t ldb, double* c,
               int64_t ldc, int algo, cudaStream_t st);
int zgemm_update_rows(int m, int n, const double* a_rows, const double* p, const double* ah_rows,
                      const double* base, const double* xprev, double* out, int64_t ld, double hh,
                      double qq, unsigned long long* resid, int algo, cudaStream_t st);

// Library configuration, read ONCE from the environment when the library is
// loaded (so a workspace sized by zt_step_workspace_bytes stays valid for
// every later call in the process):
// step products: 2 = FP64-accurate Ozaki-II on the INT8 tensor cores (default),
// 0 = 3M DMMA (ZT_GEMM_ALGO=3m or dmma), 1 = 4M DMMA (ZT_GEMM_ALGO=4m)
static bool env_on(const char* name, bool dflt) {
  const char* e = getenv(name);
  return e ? std::string(e) != "0" : dflt;
}
static const int g_algo = [] {
  const char* e = getenv("ZT_GEMM_ALGO");
  if (!e) return 2;
  const std::string v(e);
  return v == "4m" ? 1 : ((v == "3m" || v == "dmma") ? 0 : 2);
}();
// DMMA kernel variant for the products that stay on the FP64 pipe
static inline int dmma_algo() { return g_algo == 1 ? 1 : 0; }
static const bool g_fused = env_on("ZT_FUSED", true);   // persistent fused GEMM-1 + GEMM-2 per update (DMMA path)
static const bool g_planes = env_on("ZT_SUM_PLANES", true);  // fused 3M reads precomputed sum planes
static const bool g_split = env_on("ZT_SPLIT", true);   // split-K tail in the fused update
static const bool g_sep_update = env_on("ZT_SEP_UPDATE", true);  // update as a streaming pass after the GEMMs

// ---- step workspace layout -------------------------------------------------
struct StepWS {
  double* p;     // n x n complex: stream matrix
  double* a;     // n x n complex: a = P X
  void* solve;   // solve carries
  size_t solve_bytes;
  void* resid;   // residual partials
  unsigned long long* flags;  // [0] residual bits, [1] consistency bits
  double* val;   // [0..2] validation residuals
  unsigned int* sync;  // fused update: tile counter + per-panel completion counts
  double* planes;      // 3M sum planes (P A/B layout, X B layout, a A layout)
  double* split;       // split-K tail partial accumulators
  double* b;           // n x n complex: b = a P (lower / diagonal tiles) for the update pass;
                       // W_{n+1} staging of the progressive final update
  unsigned int* prog;  // zupdate_prog_words(n): progressive final update counters / flags / epoch
  void* oz;            // INT8 Ozaki-II residue planes (ZT_GEMM_ALGO=oz only)
};

static size_t align_up(size_t x) { return (x + 255) & ~(size_t)255; }

static size_t ws_layout(int n, char* base, StepWS* w) {
  const size_t mat = align_up((size_t)n * n * 16);
  const size_t sb = align_up(solve_workspace_bytes(n, 1));
  const size_t rb = align_up(resid_workspace_bytes(n));
  const size_t yb = align_up(sizeof(unsigned int) * zupdate_sync_words(n));
  const size_t pl = align_up(4 * sum_plane_bytes(n));
  const size_t spl = align_up(zupdate_split_bytes(n));
  size_t off = 0;
  if (w) {
    w->p = reinterpret_cast<double*>(base + off);
    w->a = reinterpret_cast<double*>(base + off + mat);
    w->solve = base + off + 2 * mat;
    w->solve_bytes = sb;
    w->resid = base + off + 2 * mat + sb;
    w->flags = reinterpret_cast<unsigned long long*>(base + off + 2 * mat + sb + rb);
    w->val = reinterpret_cast<double*>(base + off + 2 * mat + sb + rb + 64);
    w->sync = reinterpret_cast<unsigned int*>(base + off + 2 * mat + sb + rb + 256);
    w->planes = reinterpret_cast<double*>(base + off + 2 * mat + sb + rb + 256 + yb);
    w->split = reinterpret_cast<double*>(base + off + 2 * mat + sb + rb + 256 + yb + pl);
    w->b = reinterpret_cast<double*>(base + off + 2 * mat + sb + rb + 256 + yb + pl + spl);
    w->prog = reinterpret_cast<unsigned int*>(base + off + 3 * mat + sb + rb + 256 + yb + pl + spl);
    w->oz = base + off + 3 * mat + sb + rb + 256 + yb + pl + spl + align_up(sizeof(unsigned int) * zupdate_prog_words(n));
  }
  return 3 * mat + sb + rb + 256 + yb + pl + spl + align_up(sizeof(unsigned int) * zupdate_prog_words(n)) +
         (g_algo == 2 ? align_up(oz_update_workspace_bytes(n)) : 0);
}

// small pinned host mailbox for the per-iteration read-back
struct Mailbox {
  unsigned long long* h = nullptr;
  Mailbox() {
    if (cudaHostAlloc(&h, 64 * sizeof(unsigned long long), cudaHostAllocDefault) != cudaSuccess) h = nullptr;
  }
};
static thread_local Mailbox t_mail;

static double bits_to_double(unsigned long long b) {
  double d;
  std::memcpy(&d, &b, sizeof d);
  return d;
}

// ---- optional per-kernel device timing (bench.py roofline) -----------------
// When enabled, events bracket the solve / GEMM-1 / GEMM-2 of every update on
// the launching stream; durations are accumulated after the call's syncs.
static bool g_prof = false;
struct ProfSlot {
  cudaEvent_t ev[4];
  int final_update = 0;  // 1: [solve, a = P W~ (GEMM-1 only), W_n + h (a - a^H)]
};
static std::vector<ProfSlot> g_slots;
static size_t g_used = 0;
static double g_prof_ms[3] = {0, 0, 0};
static int64_t g_prof_cnt[3] = {0, 0, 0};

static thread_local bool t_capturing = false;

static void prof_mark(int which, cudaStream_t st, int final_update = 0) {
  if (!g_prof || t_capturing) return;
  if (which == 0) {
    if (g_used == g_slots.size()) {
      ProfSlot s;
      for (auto& e : s.ev) cudaEventCreate(&e);
      g_slots.push_back(s);
    }
    ++g_used;
    g_slots[g_used - 1].final_update = final_update;
  }
  cudaEventRecord(g_slots[g_used - 1].ev[which], st);
}

static void prof_collect() {
  if (!g_prof) return;
  // slots: [0] stream solve, [1] full update (GEMM-1 + GEMM-2 + epilogue, or
  // GEMM-1 alone when unfused), [2] GEMM-2 (unfused) or the step's final
  // update (GEMM-1 only + the commutator pass)
  for (size_t i = 0; i < g_used; ++i) {
    cudaEventSynchronize(g_slots[i].ev[3]);
    const bool fin = g_slots[i].final_update;
    for (int k = 0; k < 3; ++k) {
      if (fin && k == 1) continue;
      float ms = 0.f;
      const cudaEvent_t e0 = g_slots[i].ev[k], e1 = (fin && k == 2) ? g_slots[i].ev[3] : g_slots[i].ev[k + 1];
      const cudaEvent_t s0 = (fin && k == 2) ? g_slots[i].ev[1] : e0;
      if (cudaEventElapsedTime(&ms, s0, e1) == cudaSuccess) {
        g_prof_ms[k] += ms;
        g_prof_cnt[k] += 1;
      }
    }
  }
  g_used = 0;
}

// INT8 path: X's column conversion is independent of the solve, so it runs
// on a side stream forked from `st` (event fork / join: captured into the
// step graph as parallel branches) while the latency-bound solve runs.
// Streams and events this library creates lazily, per calling thread AND per
// device (a stream belongs to the device current when it was created)
struct DevStreams {
  cudaStream_t side = nullptr, cap[2] = {nullptr, nullptr}, copy = nullptr, copy2 = nullptr;
  cudaEvent_t fork = nullptr, join = nullptr, copy_ev = nullptr, copy_ev2 = nullptr, reset_ev = nullptr;
};
static thread_local DevStreams t_ds[64];
static DevStreams& ds() {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) dev = 0;
  return t_ds[dev];
}
static int oz_fork_x(int n, const double* x, StepWS& w, cudaStream_t st) {
  DevStreams& d = ds();
  if (!d.side) {
    ZT_CUDA_CHECK(cudaStreamCreateWithFlags(&d.side, cudaStreamNonBlocking));
    ZT_CUDA_CHECK(cudaEventCreateWithFlags(&d.fork, cudaEventDisableTiming));
    ZT_CUDA_CHECK(cudaEventCreateWithFlags(&d.join, cudaEventDisableTiming));
  }
  ZT_CUDA_CHECK(cudaEventRecord(d.fork, st));
  ZT_CUDA_CHECK(cudaStreamWaitEvent(d.side, d.fork, 0));
  const int rc = oz_convert_x(n, x, w.oz, d.side);
  if (rc) return rc;
  ZT_CUDA_CHECK(cudaEventRecord(d.join, d.side));
  return ZT_OK;
}

// One update: P = lap^-1 X; a = P X; out = base + hh (a - a^H) + qq a P.
static int update(zt_operator* op, const double* x, const double* base, const double* xprev,
                  const double* wn, double* out, double hh, double qq, StepWS& w,
                  unsigned long long* resid, unsigned long long* cons, cudaStream_t st) {
  const int n = op->n;
  prof_mark(0, st);
  if (g_algo == 2) {
    const int rc0 = oz_fork_x(n, x, w, st);
    if (rc0) return rc0;
  }
  int rc = stream_solve(op, x, n, 0, w.p, n, 0, 1, w.solve, w.solve_bytes, st);
  if (rc) return rc;
  prof_mark(1, st);
  if (g_algo == 2) {
    rc = oz_update(n, w.p, x, w.a, w.b, base, xprev, wn, out, hh, qq, resid, cons, w.oz, st, 0, ds().join);
    prof_mark(2, st);
    prof_mark(3, st);
    return rc;
  }
  if (g_fused) {
    // GEMM-1 and GEMM-2 in one persistent launch (profiled as "gemm1")
    rc = zupdate_fused(n, w.p, x, w.a, base, xprev, wn, out, hh, qq, resid, cons, w.sync,
                       g_algo == 0 && g_planes ? 3 : g_algo, w.planes, g_split ? w.split : nullptr, st, 0,
                       g_sep_update ? w.b : nullptr);
    prof_mark(2, st);
    prof_mark(3, st);
    return rc;
  }
  rc = zgemm(n, w.p, n, x, n, w.a, n, dmma_algo(), st);
  if (rc) return rc;
  prof_mark(2, st);
  rc = zgemm_update(n, w.a, w.p, base, xprev, wn, out, n, hh, qq, resid, cons, dmma_algo(), st);
  prof_mark(3, st);
  return rc;
}

// The step's last update without GEMM-2 (see k_final_commutator): solve,
// a = P W~, W_{n+1} = W_n + h (a - a^H), in place over W~.  ZT_FINAL_SANDWICH=1
// (or a consistency request) keeps the reference's sandwich form.
static const bool g_final_comm = !env_on("ZT_FINAL_SANDWICH", false);
// prog: the GEMM-1 kernel itself writes W_{n+1} into w.b pair by pair and
// publishes each 64-row block (FusedArgs::prog) for an overlapped D2H copy;
// x receives it by one device copy at the end.
static int final_update(zt_operator* op, double* x, const double* wn, double h, StepWS& w, cudaStream_t st,
                        bool prog = false) {
  const int n = op->n;
  prof_mark(0, st, 1);
  if (g_algo == 2) {
    const int rc0 = oz_fork_x(n, x, w, st);
    if (rc0) return rc0;
  }
  int rc = stream_solve(op, x, n, 0, w.p, n, 0, 1, w.solve, w.solve_bytes, st);
  if (rc) return rc;
  prof_mark(1, st);
  if (g_algo == 2) {
    rc = oz_update(n, w.p, x, w.a, nullptr, nullptr, nullptr, wn, x, h, 0.0, nullptr, nullptr, w.oz, st, 1, ds().join);
    prof_mark(2, st);
    prof_mark(3, st);
    return rc;
  }
  prog = prog && g_fused;
  if (g_fused) {
    ProgParams pp{wn, w.b, h, w.prog};
    rc = zupdate_fused(n, w.p, x, w.a, nullptr, nullptr, nullptr, nullptr, 0.0, 0.0, nullptr, nullptr, w.sync,
                       g_algo == 0 && g_planes ? 3 : g_algo, w.planes, nullptr, st, 1, nullptr, prog ? &pp : nullptr);
  } else {
    rc = zgemm(n, w.p, n, x, n, w.a, n, dmma_algo(), st);
  }
  if (rc) return rc;
  prof_mark(2, st);
  if (prog)
    rc = cudaMemcpyAsync(x, w.b, (size_t)n * n * 16, cudaMemcpyDeviceToDevice, st) ? ZT_ECUDA : ZT_OK;
  else
    rc = final_commutator(n, w.a, wn, h, x, st);
  prof_mark(3, st);
  return rc;
}

static int fixed_point_impl(zt_operator* op, const double* wn, double* x, double h, double tol,
                            int max_iter, StepWS& w, int* iterations, double* residual,
                            cudaStream_t st) {
  const int n = op->n;
  if (!(h >= 0.0)) return fail(ZT_EINVAL, "time-step must be nonnegative, got " + std::to_string(h));
  if (!(tol > 0.0)) return fail(ZT_EINVAL, "tolerance must be positive, got " + std::to_string(tol));
  if (max_iter < 1) return fail(ZT_EINVAL, "max_iter must be at least 1, got " + std::to_string(max_iter));
  if (!t_mail.h) return fail(ZT_ENOMEM, "pinned mailbox allocation failed");
  // input gate (integrator.py:121 -> laplacian.py:107-116), checked at the
  // first read-back; the loop is enqueued behind it without a sync.
  int rc = residuals(n, wn, n, w.val, w.resid, st);
  if (rc) return rc;
  ZT_CUDA_CHECK(cudaMemcpyAsync(x, wn, (size_t)n * n * 16, cudaMemcpyDeviceToDevice, st));
  const double hh = 0.5 * h, qq = 0.25 * h * h;
  double r = INFINITY;
  for (int k = 1; k <= max_iter; ++k) {
    ZT_CUDA_CHECK(cudaMemsetAsync(w.flags, 0, sizeof(unsigned long long), st));
    // in place: X <- W_n + (h/2)(a - a^H) + (h^2/4) a P, residual vs old X
    rc = update(op, x, wn, x, nullptr, x, hh, qq, w, w.flags, nullptr, st);
    if (rc) return rc;
    ZT_CUDA_CHECK(cudaMemcpyAsync(t_mail.h, w.flags, sizeof(unsigned long long), cudaMemcpyDeviceToHost, st));
    if (k == 1) ZT_CUDA_CHECK(cudaMemcpyAsync(t_mail.h + 1, w.val, 3 * sizeof(double), cudaMemcpyDeviceToHost, st));
    ZT_CUDA_CHECK(cudaStreamSynchronize(st));
    if (k == 1) {
      const double sk = bits_to_double(t_mail.h[1]), tr = bits_to_double(t_mail.h[2]);
      char buf[160];
      if (sk > 1e-10) {  // NaN passes, as `r > tol` in the reference
        snprintf(buf, sizeof buf, "matrix is not skew-Hermitian: residual %.3e > 1.0e-10", sk);
        return fail(ZT_ESTRUCTURE, buf);
      }
      if (tr > 1e-10) {
        snprintf(buf, sizeof buf, "matrix is not traceless: residual %.3e > 1.0e-10", tr);
        return fail(ZT_ESTRUCTURE, buf);
      }
    }
    r = bits_to_double(t_mail.h[0]);
    *iterations = k;
    *residual = r;
    if (r <= tol) return ZT_OK;
  }
  char buf[200];
  snprintf(buf, sizeof buf,
           "fixed-point iteration did not reach tol=%.1e in %d iterations (last residual %.3e)", tol,
           max_iter, r);
  return fail(ZT_ENOCONV, buf);
}

// ---- CUDA-graph step: the fixed point as a conditional WHILE node ------------
// Prologue (input gate, X <- W_n, counter reset) -> while(cond) { update;
// decide } -> final update.  One graph launch and one 40-byte read-back per
// step instead of a host round trip per fixed-point iteration.
__global__ void k_fp_decide(unsigned long long* flags, double tol, int max_iter, cudaGraphConditionalHandle h) {
  const unsigned long long bits = flags[0];
  double r;
  memcpy(&r, &bits, sizeof r);
  const unsigned long long k = ++flags[2];
  flags[3] = bits;  // last residual
  // continue while not converged (NaN never converges, integrator.py:131)
  cudaGraphSetConditional(h, (!(r <= tol) && (int)k < max_iter) ? 1u : 0u);
}

// laplacian.py:107-116 on the gate's residuals (NaN passes, as `r > tol`
// is false in the reference); the WHILE condition starts at 1 otherwise
__global__ void k_gate(const double* val, cudaGraphConditionalHandle h) {
  cudaGraphSetConditional(h, (val[0] > 1e-10 || val[1] > 1e-10) ? 0u : 1u);
}

struct GraphEntry {
  zt_operator* op;
  int n;
  const double* wn;
  double* wnext;
  void* ws;
  double h, tol;
  int max_iter;
  bool cons;
  bool prog = false;  // progressive final update (host-copy variant)
  cudaGraphExec_t exec = nullptr;
  int64_t kp = 0, kb = 0, ke = 0;  // kernels in prologue / per iteration / epilogue
};
static thread_local std::vector<GraphEntry> t_graphs;

// ZT_GRAPH=0 or zt_set_graph(0): eager step with per-iteration host sync
static std::atomic<bool> g_graph{env_on("ZT_GRAPH", true)};

static int build_step_graph(GraphEntry& e, StepWS& w) {
  zt_operator* op = e.op;
  const int n = op->n;
  DevStreams& d = ds();
  for (auto& s : d.cap)
    if (!s) ZT_CUDA_CHECK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  cudaStream_t cs = d.cap[0], cb = d.cap[1];
  const double hh = 0.5 * e.h, qq = 0.25 * e.h * e.h;
  double* x = e.wnext;
  t_capturing = true;
  int rc = ZT_OK;
  cudaGraph_t graph = nullptr;
  ZT_CUDA_CHECK(cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal));
  int64_t c0 = g_launches.load();
  cudaGraphConditionalHandle hc;
  {
    cudaStreamCaptureStatus stt;
    cudaGraph_t cg;
    cudaError_t ce = cudaStreamGetCaptureInfo(cs, &stt, nullptr, &cg, nullptr, nullptr);
    if (!ce) ce = cudaGraphConditionalHandleCreate(&hc, cg, 1, cudaGraphCondAssignDefault);
    if (ce) rc = cuda_fail(ce, "graph: conditional handle");
  }
  if (!rc) rc = residuals(n, e.wn, n, w.val, w.resid, cs);
  if (!rc) rc = cudaMemcpyAsync(x, e.wn, (size_t)n * n * 16, cudaMemcpyDeviceToDevice, cs) ? ZT_ECUDA : ZT_OK;
  if (!rc) rc = cudaMemsetAsync(w.flags + 2, 0, sizeof(unsigned long long), cs) ? ZT_ECUDA : ZT_OK;
  if (!rc) {
    // the input gate decides before the first update: a rejected W_n skips
    // the fixed point entirely (0 iterations; the host raises StructureError)
    k_gate<<<1, 1, 0, cs>>>(w.val, hc);
    ZT_LAUNCHED();
  }
  int64_t c1 = g_launches.load();
  if (!rc) {
    cudaStreamCaptureStatus stt;
    cudaGraph_t cg;
    const cudaGraphNode_t* deps;
    size_t nd;
    cudaError_t ce = cudaStreamGetCaptureInfo(cs, &stt, nullptr, &cg, &deps, &nd);
    cudaGraphNodeParams cp = {};
    cp.type = cudaGraphNodeTypeConditional;
    cp.conditional.handle = hc;
    cp.conditional.type = cudaGraphCondTypeWhile;
    cp.conditional.size = 1;
    cudaGraphNode_t cnode;
    if (!ce) ce = cudaGraphAddNode(&cnode, cg, deps, nd, &cp);
    if (!ce) ce = cudaStreamUpdateCaptureDependencies(cs, &cnode, 1, cudaStreamSetCaptureDependencies);
    cudaGraph_t body = cp.conditional.phGraph_out ? cp.conditional.phGraph_out[0] : nullptr;
    if (!ce) ce = cudaStreamBeginCaptureToGraph(cb, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal);
    if (ce) rc = cuda_fail(ce, "graph: conditional node");
    if (!rc) {
      rc = cudaMemsetAsync(w.flags, 0, sizeof(unsigned long long), cb) ? ZT_ECUDA : ZT_OK;
      if (!rc) rc = update(op, x, e.wn, x, nullptr, x, hh, qq, w, w.flags, nullptr, cb);
      if (!rc) {
        k_fp_decide<<<1, 1, 0, cb>>>(w.flags, e.tol, e.max_iter, hc);
        ZT_LAUNCHED();
      }
      cudaGraph_t bg;
      cudaError_t ce2 = cudaStreamEndCapture(cb, &bg);
      if (!rc && ce2) rc = cuda_fail(ce2, "graph: body capture");
    }
  }
  int64_t c2 = g_launches.load();
  if (!rc && e.cons) rc = cudaMemsetAsync(w.flags + 1, 0, sizeof(unsigned long long), cs) ? ZT_ECUDA : ZT_OK;
  if (!rc) {
    if (!e.cons && g_final_comm)
      rc = final_update(op, x, e.wn, e.h, w, cs, e.prog);
    else
      rc = update(op, x, x, nullptr, e.cons ? e.wn : nullptr, x, hh, -qq, w, nullptr, e.cons ? w.flags + 1 : nullptr,
                  cs);
  }
  int64_t c3 = g_launches.load();
  cudaError_t ce = cudaStreamEndCapture(cs, &graph);
  t_capturing = false;
  g_launches.fetch_sub(c3 - c0);  // captured, not executed
  if (rc) {
    if (graph) cudaGraphDestroy(graph);
    return rc;
  }
  if (ce) return cuda_fail(ce, "graph: capture");
  ce = cudaGraphInstantiate(&e.exec, graph, 0);
  cudaGraphDestroy(graph);
  if (ce) return cuda_fail(ce, "graph: instantiate");
  e.kp = c1 - c0;
  e.kb = c2 - c1;
  e.ke = c3 - c2;
  return ZT_OK;
}

using wait_value_fn = CUresult (*)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
static wait_value_fn wait_value32() {
  static wait_value_fn fn = nullptr;
  static bool tried = false;
  if (!tried) {
    tried = true;
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuStreamWaitValue32", &f, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<wait_value_fn>(f);
  }
  return fn;
}

// Enqueue the row-block device-to-host copies of W_{n+1} behind the progressive
// final update's flags: clear the flags on `st`, then (after that clear, via an
// event) wait for each block's flag on the copy stream and copy the block.
// Call right before the step graph launch on `st`; `join` makes `st` wait for
// the copies (call after the launch).
static int host_copy_prologue(int n, StepWS& w, cudaStream_t st) {
  DevStreams& d = ds();
  if (!d.copy) {
    ZT_CUDA_CHECK(cudaStreamCreateWithFlags(&d.copy, cudaStreamNonBlocking));
    ZT_CUDA_CHECK(cudaStreamCreateWithFlags(&d.copy2, cudaStreamNonBlocking));
    ZT_CUDA_CHECK(cudaEventCreateWithFlags(&d.copy_ev, cudaEventDisableTiming));
    ZT_CUDA_CHECK(cudaEventCreateWithFlags(&d.copy_ev2, cudaEventDisableTiming));
    ZT_CUDA_CHECK(cudaEventCreateWithFlags(&d.reset_ev, cudaEventDisableTiming));
  }
  const int T = (n + 63) / 64;
  unsigned* flags = w.prog + (size_t)T * (T + 1) / 2 + T;
  ZT_CUDA_CHECK(cudaMemsetAsync(flags, 0, sizeof(unsigned) * T, st));
  ZT_CUDA_CHECK(cudaEventRecord(d.reset_ev, st));
  ZT_CUDA_CHECK(cudaStreamWaitEvent(d.copy, d.reset_ev, 0));
  ZT_CUDA_CHECK(cudaStreamWaitEvent(d.copy2, d.reset_ev, 0));
  return ZT_OK;
}
static int host_copy_enqueue(int n, StepWS& w, double* host_out, cudaStream_t st) {
  DevStreams& d = ds();
  const int T = (n + 63) / 64;
  const unsigned* flags = w.prog + (size_t)T * (T + 1) / 2 + T;
  // two copy streams (alternating blocks) so one block's flag wait and copy
  // setup overlap the other's transfer
  for (int s = 0; s < T; ++s) {
    cudaStream_t cs = (s & 1) ? d.copy2 : d.copy;
    const CUresult r = wait_value32()(reinterpret_cast<CUstream>(cs), reinterpret_cast<CUdeviceptr>(flags + s),
                                      1u, CU_STREAM_WAIT_VALUE_GEQ);
    if (r != CUDA_SUCCESS) return fail(ZT_ECUDA, "cuStreamWaitValue32 failed");
    const size_t rows = std::min(64, n - s * 64);
    ZT_CUDA_CHECK(cudaMemcpyAsync(host_out + (size_t)s * 64 * n * 2, w.b + (size_t)s * 64 * n * 2, rows * n * 16,
                                  cudaMemcpyDeviceToHost, cs));
  }
  ZT_CUDA_CHECK(cudaEventRecord(d.copy_ev, d.copy));
  ZT_CUDA_CHECK(cudaEventRecord(d.copy_ev2, d.copy2));
  ZT_CUDA_CHECK(cudaStreamWaitEvent(st, d.copy_ev, 0));
  ZT_CUDA_CHECK(cudaStreamWaitEvent(st, d.copy_ev2, 0));
  return ZT_OK;
}

static int midpoint_step_graph(zt_operator* op, const double* wn, double* w_next, double h, double tol,
                               int max_iter, StepWS& w, void* ws, int* iterations, double* residual,
                               double* consistency, cudaStream_t st, double* host_out = nullptr) {
  if (!(h >= 0.0)) return fail(ZT_EINVAL, "time-step must be nonnegative, got " + std::to_string(h));
  if (!(tol > 0.0)) return fail(ZT_EINVAL, "tolerance must be positive, got " + std::to_string(tol));
  if (max_iter < 1) return fail(ZT_EINVAL, "max_iter must be at least 1, got " + std::to_string(max_iter));
  if (!t_mail.h) return fail(ZT_ENOMEM, "pinned mailbox allocation failed");
  const bool cons = consistency != nullptr;
  const bool prog = host_out != nullptr && !cons && g_fused && g_algo != 2 && g_final_comm && wait_value32() != nullptr;
  GraphEntry* hit = nullptr;
  for (auto& e : t_graphs)
    if (e.op == op && e.n == op->n && e.wn == wn && e.wnext == w_next && e.ws == ws && e.h == h && e.tol == tol &&
        e.max_iter == max_iter && e.cons == cons && e.prog == prog)
      hit = &e;
  if (!hit) {
    if (t_graphs.size() >= 8) {
      cudaGraphExecDestroy(t_graphs.front().exec);
      t_graphs.erase(t_graphs.begin());
    }
    GraphEntry e;
    e.op = op;
    e.n = op->n;
    e.wn = wn;
    e.wnext = w_next;
    e.ws = ws;
    e.h = h;
    e.tol = tol;
    e.max_iter = max_iter;
    e.cons = cons;
    e.prog = prog;
    int rc = build_step_graph(e, w);
    if (rc) return rc;
    t_graphs.push_back(e);
    hit = &t_graphs.back();
  }
  if (prog) {
    int rc = host_copy_prologue(op->n, w, st);
    if (rc) return rc;
    ZT_CUDA_CHECK(cudaGraphLaunch(hit->exec, st));
    rc = host_copy_enqueue(op->n, w, host_out, st);
    if (rc) return rc;
  } else {
    ZT_CUDA_CHECK(cudaGraphLaunch(hit->exec, st));
  }
  ZT_CUDA_CHECK(cudaMemcpyAsync(t_mail.h, w.flags, 4 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, st));
  ZT_CUDA_CHECK(cudaMemcpyAsync(t_mail.h + 8, w.val, 3 * sizeof(double), cudaMemcpyDeviceToHost, st));
  ZT_CUDA_CHECK(cudaStreamSynchronize(st));
  const int k = (int)t_mail.h[2];
  g_launches.fetch_add(hit->kp + (int64_t)k * hit->kb + hit->ke);
  const double sk = bits_to_double(t_mail.h[8]), tr = bits_to_double(t_mail.h[9]);
  char buf[200];
  if (sk > 1e-10) {
    snprintf(buf, sizeof buf, "matrix is not skew-Hermitian: residual %.3e > 1.0e-10", sk);
    return fail(ZT_ESTRUCTURE, buf);
  }
  if (tr > 1e-10) {
    snprintf(buf, sizeof buf, "matrix is not traceless: residual %.3e > 1.0e-10", tr);
    return fail(ZT_ESTRUCTURE, buf);
  }
  const double r = bits_to_double(t_mail.h[3]);
  *iterations = k;
  *residual = r;
  if (!(r <= tol)) {
    snprintf(buf, sizeof buf,
             "fixed-point iteration did not reach tol=%.1e in %d iterations (last residual %.3e)", tol,
             max_iter, r);
    return fail(ZT_ENOCONV, buf);
  }
  if (cons) *consistency = bits_to_double(t_mail.h[1]);
  if (host_out && !prog) {
    ZT_CUDA_CHECK(cudaMemcpyAsync(host_out, w_next, (size_t)op->n * op->n * 16, cudaMemcpyDeviceToHost, st));
    ZT_CUDA_CHECK(cudaStreamSynchronize(st));
  }
  return ZT_OK;
}

}  // namespace zt

using namespace zt;

extern "C" {

int zt_version(void) { return 1; }

const char* zt_strerror(int s) {
  switch (s) {
    case ZT_OK: return "ok";
    case ZT_EINVAL: return "invalid argument";
    case ZT_ESTRUCTURE: return "structure violation";
    case ZT_ENOCONV: return "fixed point did not converge";
    case ZT_ELINALG: return "factorisation failed";
    case ZT_ECUDA: return "CUDA error";
    case ZT_ENCCL: return "collective error";
    case ZT_ENOMEM: return "out of memory / workspace too small";
    default: return "unknown status";
  }
}

const char* zt_last_error(void) { return t_err.c_str(); }

int64_t zt_launch_count(void) { return g_launches.load(); }

int zt_set_graph(int on) { return g_graph.exchange(on != 0) ? 1 : 0; }

// ---- device-driven fixed point for caller-enqueued updates (sharded step) ---
}  // extern "C"
struct zt_loop_graph {
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
  cudaGraphConditionalHandle cond = 0;
};
namespace zt {
__global__ void k_loop_decide(const unsigned long long* slots, int nslots, unsigned long long* mail, double tol,
                              int max_iter, cudaGraphConditionalHandle h) {
  unsigned long long bits = 0;
  for (int g = 0; g < nslots; ++g) bits = max(bits, ((const volatile unsigned long long*)slots)[g]);
  double r;
  memcpy(&r, &bits, sizeof r);
  const unsigned long long k = ++mail[2];
  mail[3] = bits;
  cudaGraphSetConditional(h, (!(r <= tol) && (long long)k < (long long)max_iter) ? 1u : 0u);
}
__global__ void k_peer_put_u64(const unsigned long long* src, const unsigned long long* dst, int index, int npeer) {
  const int h = threadIdx.x;
  if (h < npeer) reinterpret_cast<volatile unsigned long long*>(dst[h])[index] = *src;
  __threadfence_system();
}
}  // namespace zt
extern "C" {

int zt_loop_graph_begin(void* stream, zt_loop_graph_t* out) {
  if (!out) return fail(ZT_EINVAL, "zt_loop_graph_begin: null output");
  cudaStream_t st = (cudaStream_t)stream;
  zt_loop_graph* g = new zt_loop_graph;
  cudaError_t e = cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal);
  cudaStreamCaptureStatus stt;
  cudaGraph_t cg = nullptr;
  if (!e) e = cudaStreamGetCaptureInfo(st, &stt, nullptr, &cg, nullptr, nullptr);
  if (!e) e = cudaGraphConditionalHandleCreate(&g->cond, cg, 1, cudaGraphCondAssignDefault);
  if (e) {
    delete g;
    return cuda_fail(e, "zt_loop_graph_begin");
  }
  *out = g;
  return ZT_OK;
}

int zt_loop_graph_gate(zt_loop_graph_t g, const double* val, void* stream) {
  if (!g || !val) return fail(ZT_EINVAL, "zt_loop_graph_gate: bad argument");
  k_gate<<<1, 1, 0, (cudaStream_t)stream>>>(val, g->cond);
  ZT_LAUNCHED();
  ZT_CUDA_CHECK(cudaGetLastError());
  return ZT_OK;
}

int zt_loop_graph_body_begin(zt_loop_graph_t g, void* stream, void* body) {
  if (!g) return fail(ZT_EINVAL, "zt_loop_graph_body_begin: null graph");
  cudaStream_t st = (cudaStream_t)stream;
  cudaStreamCaptureStatus stt;
  cudaGraph_t cg;
  const cudaGraphNode_t* deps;
  size_t nd;
  cudaError_t e = cudaStreamGetCaptureInfo(st, &stt, nullptr, &cg, &deps, &nd);
  cudaGraphNodeParams cp = {};
  cp.type = cudaGraphNodeTypeConditional;
  cp.conditional.handle = g->cond;
  cp.conditional.type = cudaGraphCondTypeWhile;
  cp.conditional.size = 1;
  cudaGraphNode_t node;
  if (!e) e = cudaGraphAddNode(&node, cg, deps, nd, &cp);
  if (!e) e = cudaStreamUpdateCaptureDependencies(st, &node, 1, cudaStreamSetCaptureDependencies);
  if (!e)
    e = cudaStreamBeginCaptureToGraph((cudaStream_t)body, cp.conditional.phGraph_out[0], nullptr, nullptr, 0,
                                      cudaStreamCaptureModeThreadLocal);
  if (e) return cuda_fail(e, "zt_loop_graph_body_begin");
  return ZT_OK;
}

int zt_loop_graph_decide(zt_loop_graph_t g, const unsigned long long* slots, int nslots, unsigned long long* mail,
                         double tol, int max_iter, void* body) {
  if (!g || !slots || !mail || nslots < 1) return fail(ZT_EINVAL, "zt_loop_graph_decide: bad argument");
  k_loop_decide<<<1, 1, 0, (cudaStream_t)body>>>(slots, nslots, mail, tol, max_iter, g->cond);
  ZT_LAUNCHED();
  ZT_CUDA_CHECK(cudaGetLastError());
  return ZT_OK;
}

int zt_loop_graph_body_end(zt_loop_graph_t g, void* body) {
  if (!g) return fail(ZT_EINVAL, "zt_loop_graph_body_end: null graph");
  cudaGraph_t bg;
  ZT_CUDA_CHECK(cudaStreamEndCapture((cudaStream_t)body, &bg));
  return ZT_OK;
}

int zt_loop_graph_end(zt_loop_graph_t g, void* stream) {
  if (!g) return fail(ZT_EINVAL, "zt_loop_graph_end: null graph");
  ZT_CUDA_CHECK(cudaStreamEndCapture((cudaStream_t)stream, &g->graph));
  ZT_CUDA_CHECK(cudaGraphInstantiate(&g->exec, g->graph, 0));
  return ZT_OK;
}

int zt_loop_graph_launch(zt_loop_graph_t g, void* stream) {
  if (!g || !g->exec) return fail(ZT_EINVAL, "zt_loop_graph_launch: graph not built");
  ZT_CUDA_CHECK(cudaGraphLaunch(g->exec, (cudaStream_t)stream));
  return ZT_OK;
}

int zt_loop_graph_destroy(zt_loop_graph_t g) {
  if (!g) return ZT_OK;
  if (g->exec) cudaGraphExecDestroy(g->exec);
  if (g->graph) cudaGraphDestroy(g->graph);
  delete g;
  return ZT_OK;
}

int zt_peer_put_u64(const unsigned long long* src, const unsigned long long* dst_ptrs, int index, int npeer,
                    void* stream) {
  if (!src || !dst_ptrs || npeer < 1 || npeer > 1024 || index < 0) return fail(ZT_EINVAL, "zt_peer_put_u64: bad argument");
  k_peer_put_u64<<<1, npeer, 0, (cudaStream_t)stream>>>(src, dst_ptrs, index, npeer);
  ZT_LAUNCHED();
  ZT_CUDA_CHECK(cudaGetLastError());
  return ZT_OK;
}

int zt_step_algo(void) { return g_algo; }

int zt_profile_enable(int on) {
  g_prof = on != 0;
  oz_profile_enable(g_prof);
  g_used = 0;
  return ZT_OK;
}

int zt_profile_read(double* ms, int64_t* counts, int reset) {
  for (int k = 0; k < 3; ++k) {
    if (ms) ms[k] = g_prof_ms[k];
    if (counts) counts[k] = g_prof_cnt[k];
    if (reset) {
      g_prof_ms[k] = 0;
      g_prof_cnt[k] = 0;
    }
  }
  return ZT_OK;
}

int zt_op_create(int n, int device, zt_op_t* op) {
  if (!op) return fail(ZT_EINVAL, "null output");
  return op_create(n, device, op);
}
int zt_op_destroy(zt_op_t op) { return op_destroy(op); }
int zt_op_n(zt_op_t op) { return op ? op->n : -1; }
int zt_op_factors(zt_op_t op, double* linv, double* dinv) { return op_factors(op, linv, dinv); }

size_t zt_solve_workspace_bytes(int n, int batch) { return solve_workspace_bytes(n, batch); }

int zt_stream_solve_ws(zt_op_t op, const double* w, int64_t ldw, int64_t sw, double* p, int64_t ldp,
                       int64_t sp, int batch, void* ws, size_t ws_bytes, void* stream) {
  if (!op || !w || !p || batch < 1) return fail(ZT_EINVAL, "zt_stream_solve: bad argument");
  return stream_solve(op, w, ldw, sw, p, ldp, sp, batch, ws, ws_bytes, (cudaStream_t)stream);
}

// Stream-ordered temporaries of the convenience entry points (solve / residual
// workspaces, the cfg-3 ops' residue planes) come from a library-owned pool
// per device that keeps its memory between calls: the default pool's zero
// release threshold returned it at every synchronisation, and re-mapping a
// few hundred MB per call cost milliseconds (cfg 3 at N = 2048 measured
// 11 ms per commutator instead of ~0.5 ms).
static cudaError_t lib_malloc(void** ptr, size_t bytes, cudaStream_t st) {
  static std::mutex mu;
  static cudaMemPool_t pools[64] = {};
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e) return e;
  if (dev < 0 || dev >= 64) return cudaErrorInvalidDevice;
  {
    std::lock_guard<std::mutex> lk(mu);
    if (!pools[dev]) {
      cudaMemPoolProps props = {};
      props.allocType = cudaMemAllocationTypePinned;
      props.location.type = cudaMemLocationTypeDevice;
      props.location.id = dev;
      if ((e = cudaMemPoolCreate(&pools[dev], &props))) return e;
      uint64_t thr = UINT64_MAX;
      if ((e = cudaMemPoolSetAttribute(pools[dev], cudaMemPoolAttrReleaseThreshold, &thr))) return e;
    }
  }
  return cudaMallocFromPoolAsync(ptr, bytes, pools[dev], st);
}

int zt_stream_solve(zt_op_t op, const double* w, int64_t ldw, int64_t sw, double* p, int64_t ldp,
                    int64_t sp, int batch, void* stream) {
  // convenience form: allocates its carry workspace with stream-ordered
  // stream-ordered allocation from the library pool (lib_malloc, no device sync)
  if (!op || !w || !p || batch < 1) return fail(ZT_EINVAL, "zt_stream_solve: bad argument");
  const size_t b = solve_workspace_bytes(op->n, batch);
  void* ws = nullptr;
  ZT_CUDA_CHECK(lib_malloc(&ws, b, (cudaStream_t)stream));
  int rc = stream_solve(op, w, ldw, sw, p, ldp, sp, batch, ws, b, (cudaStream_t)stream);
  cudaFreeAsync(ws, (cudaStream_t)stream);
  return rc;
}

int zt_apply_laplacian(zt_op_t op, const double* w, int64_t ldw, int64_t sw, double* y, int64_t ldy,
                       int64_t sy, int sign, int batch, void* stream) {
  if (!op || !w || !y || batch < 1) return fail(ZT_EINVAL, "zt_apply_laplacian: bad argument");
  return apply_laplacian(op, w, ldw, sw, y, ldy, sy, sign, batch, (cudaStream_t)stream);
}

size_t zt_resid_workspace_bytes(int n) { return resid_workspace_bytes(n); }

int zt_residuals_ws(int n, const double* w, int64_t ldw, double* out, void* ws, void* stream) {
  if (n < 1 || !w || !out) return fail(ZT_EINVAL, "zt_residuals: bad argument");
  return residuals(n, w, ldw, out, ws, (cudaStream_t)stream);
}

int zt_residuals(int n, const double* w, int64_t ldw, double* out, void* stream) {
  if (n < 1 || !w || !out) return fail(ZT_EINVAL, "zt_residuals: bad argument");
  const size_t b = resid_workspace_bytes(n);
  void* ws = nullptr;
  ZT_CUDA_CHECK(lib_malloc(&ws, b, (cudaStream_t)stream));
  int rc = residuals(n, w, ldw, out, ws, (cudaStream_t)stream);
  cudaFreeAsync(ws, (cudaStream_t)stream);
  return rc;
}

int zt_zgemm(int n, const double* a, int64_t lda, const double* b, int64_t ldb, double* c, int64_t ldc,
             int algo, void* stream) {
  if (n < 1 || !a || !b || !c) return fail(ZT_EINVAL, "zt_zgemm: bad argument");
  return zgemm(n, a, lda, b, ldb, c, ldc, algo, (cudaStream_t)stream);
}

int zt_zgemm_rect(int m, int n, int k, const double* a, int64_t lda, const double* b, int64_t ldb, double* c,
                  int64_t ldc, int algo, void* stream) {
  if (!a || !b || !c) return fail(ZT_EINVAL, "zt_zgemm_rect: bad argument");
  return zgemm_rect(m, n, k, a, lda, b, ldb, c, ldc, algo, (cudaStream_t)stream);
}

int zt_zgemm_update_rows(int m, int n, const double* a_rows, const double* p, const double* ah_rows,
                         const double* base, const double* xprev, double* out, int64_t ld, double hh,
                         double qq, unsigned long long* resid_dev, void* stream) {
  if (m < 1 || n < 1 || !a_rows || !p || !ah_rows || !base || !out)
    return fail(ZT_EINVAL, "zt_zgemm_update_rows: bad argument");
  return zgemm_update_rows(m, n, a_rows, p, ah_rows, base, xprev, out, ld, hh, qq, resid_dev, dmma_algo(),
                           (cudaStream_t)stream);
}

size_t zt_step_workspace_bytes(int n) { return ws_layout(n, nullptr, nullptr); }

int zt_fixed_point(zt_op_t op, const double* wn, double* wt, double h, double tol, int max_iter,
                   void* workspace, size_t workspace_bytes, int* iterations, double* residual,
                   void* stream) {
  if (!op || !wn || !wt || !workspace || !iterations || !residual)
    return fail(ZT_EINVAL, "zt_fixed_point: bad argument");
  if (workspace_bytes < zt_step_workspace_bytes(op->n)) return fail(ZT_ENOMEM, "step workspace too small");
  StepWS w;
  ws_layout(op->n, reinterpret_cast<char*>(workspace), &w);
  return fixed_point_impl(op, wn, wt, h, tol, max_iter, w, iterations, residual, (cudaStream_t)stream);
}

int zt_midpoint_step(zt_op_t op, const double* wn, double* w_next, double h_eff, double tol,
                     int max_iter, void* workspace, size_t workspace_bytes, int* iterations,
                     double* residual, double* consistency, void* stream) {
  if (!op || !wn || !w_next || !workspace || !iterations || !residual)
    return fail(ZT_EINVAL, "zt_midpoint_step: bad argument");
  if (wn == w_next) return fail(ZT_EINVAL, "zt_midpoint_step: w_next must not alias w_n");
  if (workspace_bytes < zt_step_workspace_bytes(op->n)) return fail(ZT_ENOMEM, "step workspace too small");
  cudaStream_t st = (cudaStream_t)stream;
  StepWS w;
  ws_layout(op->n, reinterpret_cast<char*>(workspace), &w);
  if (g_graph && !g_prof)
    return midpoint_step_graph(op, wn, w_next, h_eff, tol, max_iter, w, workspace, iterations, residual,
                               consistency, st);
  int rc = fixed_point_impl(op, wn, w_next, h_eff, tol, max_iter, w, iterations, residual, st);
  if (rc) return rc;
  // final update (integrator.py:154-158): W_{n+1} = W~ + (h/2)(a - a^H) - (h^2/4) a P~
  const double hh = 0.5 * h_eff, q = 0.25 * h_eff * h_eff;
  if (consistency) ZT_CUDA_CHECK(cudaMemsetAsync(w.flags + 1, 0, sizeof(unsigned long long), st));
  if (!consistency && g_final_comm)
    rc = final_update(op, w_next, wn, h_eff, w, st);
  else
    rc = update(op, w_next, w_next, nullptr, consistency ? wn : nullptr, w_next, hh, -q, w, nullptr,
                consistency ? w.flags + 1 : nullptr, st);
  if (rc) return rc;
  prof_collect();
  if (consistency) {
    ZT_CUDA_CHECK(cudaMemcpyAsync(t_mail.h + 4, w.flags + 1, sizeof(unsigned long long), cudaMemcpyDeviceToHost, st));
    ZT_CUDA_CHECK(cudaStreamSynchronize(st));
    *consistency = bits_to_double(t_mail.h[4]);
  }
  return ZT_OK;
}

int zt_midpoint_step_host(zt_op_t op, const double* wn, double* w_next, double* host_out, double h_eff, double tol,
                          int max_iter, void* workspace, size_t workspace_bytes, int* iterations, double* residual,
                          void* stream) {
  if (!op || !wn || !w_next || !host_out || !workspace || !iterations || !residual)
    return fail(ZT_EINVAL, "zt_midpoint_step_host: bad argument");
  if (wn == w_next) return fail(ZT_EINVAL, "zt_midpoint_step_host: w_next must not alias w_n");
  if (workspace_bytes < zt_step_workspace_bytes(op->n)) return fail(ZT_ENOMEM, "step workspace too small");
  cudaStream_t st = (cudaStream_t)stream;
  if (g_graph && !g_prof) {
    StepWS w;
    ws_layout(op->n, reinterpret_cast<char*>(workspace), &w);
    return midpoint_step_graph(op, wn, w_next, h_eff, tol, max_iter, w, workspace, iterations, residual, nullptr,
                               st, host_out);
  }
  int rc = zt_midpoint_step(op, wn, w_next, h_eff, tol, max_iter, workspace, workspace_bytes, iterations, residual,
                            nullptr, stream);
  if (rc) return rc;
  ZT_CUDA_CHECK(cudaMemcpyAsync(host_out, w_next, (size_t)op->n * op->n * 16, cudaMemcpyDeviceToHost, st));
  ZT_CUDA_CHECK(cudaStreamSynchronize(st));
  return ZT_OK;
}

// cfg 3 ops on the step's product: the INT8 Ozaki-II GEMM by default (its
// residue planes in a stream-ordered temporary), the DMMA GEMM under
// ZT_GEMM_ALGO=3m/4m
static int product_for_op(int n, const double* a, const double* b, int bmode, int lower, double* c, void* oz_ws,
                          cudaStream_t st) {
  if (g_algo == 2) return oz_zgemm(n, a, n, b, n, bmode, c, n, lower, oz_ws, oz_workspace_bytes(n), st);
  return zgemm(n, a, n, b, n, c, n, dmma_algo(), st);
}

int zt_commutator(int n, const double* p, const double* w, double* c, double* work, void* stream) {
  if (n < 1 || !p || !w || !c || !work) return fail(ZT_EINVAL, "zt_commutator: bad argument");
  cudaStream_t st = (cudaStream_t)stream;
  void* oz = nullptr;
  if (g_algo == 2) ZT_CUDA_CHECK(lib_malloc(&oz, oz_workspace_bytes(n), st));
  int rc = product_for_op(n, p, w, 0, 0, work, oz, st);
  if (oz) cudaFreeAsync(oz, st);
  if (rc) return rc;
  return skew_diff(n, work, c, st);
}

int zt_grid_eval(int n, int lmax, int nlat, int nlon, const long long* coff, const double* pos, double* work,
                 double* field, void* stream) {
  if (!coff || !pos || !work || !field) return fail(ZT_EINVAL, "zt_grid_eval: bad argument");
  return grid_eval(n, lmax, nlat, nlon, coff, pos, work, field, (cudaStream_t)stream);
}

int zt_zgemm_rect_scatter(int m, int n, int k, const double* a, int64_t lda, const double* b, int64_t ldb,
                          double* c, int64_t ldc, const unsigned long long* peers, int npeer, int r0, int mloc,
                          void* stream) {
  if (!a || !b || !c || !peers) return fail(ZT_EINVAL, "zt_zgemm_rect_scatter: bad argument");
  return zgemm_rect_scatter(m, n, k, a, lda, b, ldb, c, ldc, peers, npeer, r0, mloc, dmma_algo(), (cudaStream_t)stream);
}

int zt_zgemm_update_rows_peer(int m, int n, const double* a_rows, const double* p, const double* acol, int mloc,
                              const double* base, const double* xprev, double* out, int64_t ld, double hh,
                              double qq, unsigned long long* resid, const unsigned long long* peers, int npeer,
                              int r0, void* stream) {
  if (!a_rows || !p || !acol || !base || !out || (npeer && !peers))
    return fail(ZT_EINVAL, "zt_zgemm_update_rows_peer: bad argument");
  return zgemm_update_rows_peer(m, n, a_rows, p, acol, mloc, base, xprev, out, ld, hh, qq, resid, peers, npeer, r0,
                                dmma_algo(), (cudaStream_t)stream);
}

int zt_zgemm_rect_mirror(int m, int n, int k, const double* a, int64_t lda, const double* b, int64_t ldb,
                         double* c, int64_t ldc, double* mirror, int64_t ld_mirror, void* stream) {
  if (!a || !b || !c) return fail(ZT_EINVAL, "zt_zgemm_rect_mirror: bad argument");
  return zgemm_rect_mirror(m, n, k, a, lda, b, ldb, c, ldc, mirror, ld_mirror, dmma_algo(), (cudaStream_t)stream);
}

int zt_update_rows_ew(int m, int n, const double* a_rows, const double* acol, int mloc, const double* b_rows,
                      const double* base, const double* xprev, double* out, int64_t ld, double hh, double qq,
                      unsigned long long* resid, const unsigned long long* peers, int npeer, int r0, void* stream) {
  if (!a_rows || !acol || !base || !out || (npeer && !peers))
    return fail(ZT_EINVAL, "zt_update_rows_ew: bad argument");
  return update_rows_ew(m, n, a_rows, acol, mloc, b_rows, base, xprev, out, ld, hh, qq, resid, peers, npeer, r0,
                        (cudaStream_t)stream);
}

int zt_rows_broadcast(int m, int n, const double* rows, int64_t ld, const unsigned long long* peers, int npeer,
                      int r0, void* stream) {
  if (!rows || !peers) return fail(ZT_EINVAL, "zt_rows_broadcast: bad argument");
  return rows_broadcast(m, n, rows, ld, peers, npeer, r0, (cudaStream_t)stream);
}

int zt_basis_vectors(int n, int m0, int m1, const long long* off, double* vec, void* stream) {
  if (!off || !vec) return fail(ZT_EINVAL, "zt_basis_vectors: bad argument");
  return basis_vectors(n, m0, m1, off, vec, (cudaStream_t)stream);
}

int zt_basis_extract(int n, int m0, int m1, const long long* off, const long long* coff, const double* vec,
                     const double* w, int64_t ldw, double* pos, double* neg, void* stream) {
  if (!off || !coff || !vec || !w || !pos || !neg || ldw < n) return fail(ZT_EINVAL, "zt_basis_extract: bad argument");
  return basis_extract(n, m0, m1, off, coff, vec, w, ldw, pos, neg, (cudaStream_t)stream);
}

int zt_basis_project(int n, int m0, int m1, const long long* off, const long long* coff, const double* vec,
                     const double* pos, const double* neg, double* w, int64_t ldw, void* stream) {
  if (!off || !coff || !vec || !pos || !w || ldw < n) return fail(ZT_EINVAL, "zt_basis_project: bad argument");
  return basis_project(n, m0, m1, off, coff, vec, pos, neg, w, ldw, (cudaStream_t)stream);
}

int zt_sandwich(int n, const double* p, const double* w, double h, double* s, double* work, void* stream) {
  // S = W - (h/2)(a - a^H) - (h^2/4) a P  with a = P W; a P = P W P is
  // skew-Hermitian for skew P, W, so (as in the step) only its lower tiles
  // are computed and the update pass mirrors them
  if (n < 1 || !p || !w || !s || !work) return fail(ZT_EINVAL, "zt_sandwich: bad argument");
  cudaStream_t st = (cudaStream_t)stream;
  if (g_algo != 2) {
    int rc = zgemm(n, p, n, w, n, work, n, dmma_algo(), st);
    if (rc) return rc;
    return zgemm_update(n, work, p, w, nullptr, nullptr, s, n, -0.5 * h, -0.25 * h * h, nullptr, nullptr,
                        dmma_algo(), st);
  }
  void* oz = nullptr;
  double* b = nullptr;
  ZT_CUDA_CHECK(lib_malloc(&oz, oz_workspace_bytes(n), st));
  ZT_CUDA_CHECK(lib_malloc(reinterpret_cast<void**>(&b), (size_t)n * n * 16, st));
  int rc = product_for_op(n, p, w, 0, 0, work, oz, st);
  if (!rc) rc = product_for_op(n, work, p, 0, 1, b, oz, st);
  if (!rc) rc = update_pairs(n, work, b, s, w, nullptr, nullptr, -0.5 * h, -0.25 * h * h, nullptr, nullptr, st);
  cudaFreeAsync(b, st);
  cudaFreeAsync(oz, st);
  return rc;
}

}  // extern "C"
