// Complex128 GEMM on the sm_100a FP64 tensor pipe (DMMA.8x8x4), with the
// fused epilogues of the isospectral midpoint update.
//
// Replaces the numpy `@` products of integrator.py:127-128 / 155-158
// (OpenBLAS zgemm) and the elementwise update around them.
//
// Design:
//  * sm_100a has no tcgen05 kind::f64, so FP64 MMA is the warp-level
//    mma.sync m8n8k4 (SASS DMMA.8x8x4, 64 FMA/clk/SM measured = 37 TF at
//    1.965 GHz).  The kernel is warp-specialised Blackwell style anyway:
//    one producer thread streams operand tiles with 2D TMA
//    (cp.async.bulk.tensor, 128B swizzle, OOB zero fill) into a ring of
//    shared-memory stages guarded by mbarriers (full/empty); 8 consumer
//    warps issue DMMA.  Fragment k-indices are permuted (DMMA k-slot kk of
//    k4-step s reads 16B chunk 2kk+(s&1) of the 128B swizzle row) so every
//    LDS.128 fragment load is bank-conflict free under the swizzle.
//  * complex products use the 3M (Gauss) form by default:
//      T1 = Ar Br, T2 = Ai Bi, T3 = (Ar+Ai)(Br+Bi); Cr = T1-T2, Ci = T3-T1-T2
//    — 3 real MMAs per complex MMA instead of 4 (25% fewer DMMA), operand
//    sums formed in registers from the (re,im) pair one LDS.128 returns.
//    ALGO_4M keeps the classical 4-product form for comparison.
//  * EPI_STORE writes C.  EPI_UPDATE runs only on lower-triangle tiles of
//    b = a P (skew-Hermitian: P X P), forms
//        new = base + (h/2)(a - a^H) + qq * b
//    for the tile and its mirror (b_ji = -conj(b_ij)), writes it, and
//    reduces max|new - X| (fixed-point residual, integrator.py:129) and
//    optionally max|recon - W_n| (consistency, integrator.py:160-163) with
//    one atomic per CTA.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <stdio.h>

#include <algorithm>
#include <cstring>
#include <string>

#include "zt_tma.cuh"

namespace zt {

constexpr int BM = 64, BN = 64, BK = 16;
constexpr int STAGES = 4;
// TMA boxes: 128B-wide (8 complex) swizzled rows
constexpr int A_BOXES = BK / 8;            // A stage = A_BOXES boxes of [BM rows][8 complex]
constexpr int B_BOXES = BN / 8;            // B stage = B_BOXES boxes of [BK rows][8 complex]
constexpr int A_BOX_BYTES = BM * 128;
constexpr int B_BOX_BYTES = BK * 128;
constexpr int A_STAGE_BYTES = A_BOXES * A_BOX_BYTES;
constexpr int B_STAGE_BYTES = B_BOXES * B_BOX_BYTES;
constexpr int STAGE_BYTES = A_STAGE_BYTES + B_STAGE_BYTES;
// Warp layout: WNB n8-blocks per consumer warp (warp tile 32 x 8*WNB complex);
// WNB = 2: 8 consumer warps (2 x 4), WNB = 4: 4 consumer warps (2 x 2) with
// fewer 3M operand-sum DADDs per DMMA (8 per 48 instead of 6 per 24).
#ifndef ZT_WNB
#define ZT_WNB 2
#endif
constexpr int WNB = ZT_WNB;
constexpr int WN_WARPS = 64 / (8 * WNB);
// 3M sum planes (ALGO_3MS): per 64-row x 16-k A tile and 16-k x 64-col B tile,
// 1024 doubles each in DMMA-fragment order, so one 8 KB bulk copy per tile
// lands them in shared memory ready for conflict-free LDS.64.
constexpr int PLANE_TILE = 1024;                   // doubles per plane tile
constexpr int SUM_STAGE_BYTES = 2 * PLANE_TILE * 8;  // A + B plane tiles per stage
constexpr int CONSUMER_WARPS = 2 * WN_WARPS;
constexpr int GEMM_THREADS = (CONSUMER_WARPS + 1) * 32;
constexpr int GEMM_SMEM = STAGES * STAGE_BYTES + (2 * STAGES + 4) * 8 + 1024 + 64;
constexpr int GEMM_SMEM_S = STAGES * (STAGE_BYTES + 2 * 1024 * 8) + (2 * STAGES + 4) * 8 + 1024 + 64;

enum {
  ALGO_3M = 0,        // Gauss 3M, operand sums (re + im) formed per warp in registers
  ALGO_4M = 1,        // classical 4 real products
  ALGO_3MS = 3        // Gauss 3M, sums read from precomputed fragment-order sum planes
};
enum {
  EPI_STORE = 0,   // C = A B
  EPI_UPDATE = 1,  // square, lower tiles + mirror: new = base + hh (a - a^H) + qq b
  EPI_ROWS = 2     // row block (sharded step): new = base + hh (a - ah) + qq b, ah given
};

struct GemmArgs {
  int n;        // square size (EPI_UPDATE) / output columns
  int m, k;     // rows of A / C, inner dimension (rectangular EPI_STORE / EPI_ROWS)
  CUtensorMap tma_a;  // 2D map of A (and "a" operand) as doubles, box 16 x BM
  CUtensorMap tma_b;  // 2D map of B, box 16 x BK
  const double* a;  // row-major n x n complex, lda
  int64_t lda;
  const double* b;
  int64_t ldb;
  double* c;  // EPI_STORE output
  int64_t ldc;
  // EPI_UPDATE
  const double* amat;  // the left operand "a" again (for a^H in the epilogue)
  const double* ah;    // EPI_ROWS: rows of a^H matching the output rows
  const double* base;  // W_n (iterate) or W~ (final)
  const double* xprev; // previous iterate for the residual (may alias out), or null
  const double* wn;    // for consistency (final step), or null
  double* out;
  int64_t ld;          // shared leading dimension for amat/base/xprev/wn/out
  double hh, qq;       // new = base + hh (a - a^H) + qq b
  unsigned long long* resid;  // max |new - xprev| bits
  unsigned long long* cons;   // max |base - hh(a-a^H) + qq b - wn| bits
  // peer-memory collectives fused into the epilogue (sharded step): `peers`
  // holds npeer device pointers (one per rank, NVLink peer-mapped).
  //   EPI_STORE: element (i, j) of this rank's row block (global row r0 + i)
  //     also goes to rank h = j / mloc's N x mloc buffer a[:, R_h] at
  //     (r0 + i, j - h mloc) -- the all-to-all behind (a^H)_R;
  //   EPI_ROWS: every output element also goes to each rank's N x N iterate
  //     at (r0 + i, j) -- the all-gather of the next iterate;
  //     with `acol` set, (a^H)_R[i][j] = conj(acol[j][i]) (acol: N x mloc).
  const unsigned long long* peers;
  int npeer, r0, mloc;
  const double* acol;
  // EPI_STORE: also -conj(C^T) into `mirror` (ld_mirror), e.g. the partner
  // rank's rows of a skew-Hermitian product
  double* mirror;
  int64_t ld_mirror;
  // EPI_STORE on a square skew-Hermitian block: lower tiles only, the strict
  // upper tiles stored as -conj of the lower ones
  int lower;
};

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

// max that keeps a NaN once seen (fmax would drop it): a NaN residual must
// read as "not converged" exactly like numpy's max in integrator.py:129
__device__ __forceinline__ double nanmax(double acc, double v) {
  return (acc != acc) ? acc : ((v != v || v > acc) ? v : acc);
}

__device__ __forceinline__ void tile_of(int t, bool lower, int T, int& I, int& J) {
  if (lower) {
    int c = (int)((sqrt(8.0 * t + 1.0) - 1.0) * 0.5);
    while ((c + 1) * (c + 2) / 2 <= t) ++c;
    while (c * (c + 1) / 2 > t) --c;
    I = c;
    J = t - c * (c + 1) / 2;
  } else {
    // grouped rasterisation: 8 tile-rows per group for L2 reuse
    const int G = 8;
    const int per = G * T;
    const int grp = t / per;
    const int first = grp * G;
    const int rows = min(G, T - first);
    const int r = t - grp * per;
    I = first + r % rows;
    J = r / rows;
  }
}

// Row-block shell order: shell s = tiles (s, s..T-1) then (s+1..T-1, s);
// prefix(s) = s (2T - s).  Row block s of W_{n+1} needs shells 0..s only.
__device__ __forceinline__ void shell_tile(int t, int T, int& I, int& J) {
  int s = (int)((double)T - sqrt((double)T * T - (double)t));
  s = max(0, min(s, T - 1));
  while (s > 0 && s * (2 * T - s) > t) --s;
  while (s + 1 < T && (s + 1) * (2 * T - s - 1) <= t) ++s;
  const int r = t - s * (2 * T - s);
  if (r < T - s) {
    I = s;
    J = s + r;
  } else {
    I = s + 1 + (r - (T - s));
    J = s;
  }
}

// ---- shared pieces --------------------------------------------------------
template <int ALGO>
struct Acc {
  static constexpr int NACC = (ALGO != ALGO_4M) ? 3 : 2;
  double v[NACC][4][WNB][2];
  __device__ __forceinline__ void zero() {
#pragma unroll
    for (int q = 0; q < NACC; ++q)
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < WNB; ++j) v[q][i][j][0] = v[q][i][j][1] = 0.0;
  }
};

// One BK-deep stage of DMMA for warp (wm, wn) from the swizzled stage `st`.
template <int ALGO>
__device__ __forceinline__ void consume_stage(const unsigned char* st, Acc<ALGO>& A, int wm, int wn, int lane) {
  const double* sa = reinterpret_cast<const double*>(st + STAGE_BYTES);  // ALGO_3MS planes
  const double* sb = sa + PLANE_TILE;
  const int fr = lane >> 2, fk = lane & 3;
  // A fragment row r = wm*32 + i*8 + fr (r & 7 == fr); B fragment column
  // n = wn*16 + j*8 + fr lives in box (wn*2 + j), in-box column fr.
#pragma unroll
  for (int ks = 0; ks < BK / 4; ++ks) {
    const int jb = ks >> 1, par = ks & 1;
    const int c = 2 * fk + par;  // 16B chunk inside the 128B row
    const int kr = 8 * jb + c;   // k row of the B stage
    double2 af[4], bf[WNB];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int r = wm * 32 + i * 8 + fr;
      af[i] = *reinterpret_cast<const double2*>(st + jb * A_BOX_BYTES + r * 128 + ((c ^ fr) << 4));
    }
#pragma unroll
    for (int j = 0; j < WNB; ++j)
      bf[j] = *reinterpret_cast<const double2*>(st + A_STAGE_BYTES + (wn * WNB + j) * B_BOX_BYTES + kr * 128 +
                                                 ((fr ^ (kr & 7)) << 4));
    if (ALGO != ALGO_4M) {
      double bsum[WNB];
#pragma unroll
      for (int j = 0; j < WNB; ++j)
        bsum[j] = (ALGO == ALGO_3MS) ? sb[((ks * WN_WARPS + wn) * WNB + j) * 32 + lane] : bf[j].x + bf[j].y;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const double asum = (ALGO == ALGO_3MS) ? sa[((ks * 2 + wm) * 4 + i) * 32 + lane] : af[i].x + af[i].y;
#pragma unroll
        for (int j = 0; j < WNB; ++j) {
          dmma(A.v[0][i][j][0], A.v[0][i][j][1], af[i].x, bf[j].x);
          dmma(A.v[1][i][j][0], A.v[1][i][j][1], af[i].y, bf[j].y);
          dmma(A.v[2][i][j][0], A.v[2][i][j][1], asum, bsum[j]);
        }
      }
    } else {
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const double ain = -af[i].y;
#pragma unroll
        for (int j = 0; j < WNB; ++j) {
          dmma(A.v[0][i][j][0], A.v[0][i][j][1], af[i].x, bf[j].x);
          dmma(A.v[0][i][j][0], A.v[0][i][j][1], ain, bf[j].y);
          dmma(A.v[1][i][j][0], A.v[1][i][j][1], af[i].x, bf[j].y);
          dmma(A.v[1][i][j][0], A.v[1][i][j][1], af[i].y, bf[j].x);
        }
      }
    }
  }
}

// Epilogue of one 64 x 64 tile (I, J) for warp (wm, wn).
template <int ALGO, int EPI>
__device__ __forceinline__ void epilogue_tile(const GemmArgs& g, const Acc<ALGO>& A, int I, int J, int wm, int wn,
                                              int lane, double& rmax, double& cmax) {
  const int fr = lane >> 2, fk = lane & 3;
  const int n = g.n, mrows = g.m;
  const int row0 = I * BM, col0 = J * BN;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
#pragma unroll
    for (int j = 0; j < WNB; ++j) {
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        double cr, ci;
        if (ALGO != ALGO_4M) {
          cr = A.v[0][i][j][e] - A.v[1][i][j][e];
          ci = A.v[2][i][j][e] - A.v[0][i][j][e] - A.v[1][i][j][e];
        } else {
          cr = A.v[0][i][j][e];
          ci = A.v[1][i][j][e];
        }
        const int gi = row0 + wm * 32 + i * 8 + fr;
        const int gj = col0 + wn * 8 * WNB + j * 8 + fk * 2 + e;
        if (gi >= mrows || gj >= n) continue;
        if (EPI == EPI_STORE) {
          st2(g.c + ((size_t)gi * g.ldc + gj) * 2, make_double2(cr, ci));
          if (g.npeer) {
            const int h = gj / g.mloc;
            double* dst = reinterpret_cast<double*>(g.peers[h]);
            st2(dst + ((size_t)(g.r0 + gi) * g.mloc + (gj - h * g.mloc)) * 2, make_double2(cr, ci));
          }
          if (g.mirror) st2(g.mirror + ((size_t)gj * g.ld_mirror + gi) * 2, make_double2(-cr, ci));
          if (g.lower && I != J) st2(g.c + ((size_t)gj * g.ldc + gi) * 2, make_double2(-cr, ci));
        } else if (EPI == EPI_ROWS) {
          const size_t o = ((size_t)gi * g.ld + gj) * 2;
          const double2 aij = ld2_plain(g.amat + o);
          double2 ahij;
          if (g.acol) {
            const double2 t = ld2_plain(g.acol + ((size_t)gj * g.mloc + gi) * 2);
            ahij = make_double2(t.x, -t.y);
          } else {
            ahij = ld2_plain(g.ah + o);
          }
          const double2 dij = csub(aij, ahij);  // (a - a^H) on this row block
          const double2 base = ld2_plain(g.base + o);
          const double2 nw = cadd(cadd(base, rmul(g.hh, dij)), rmul(g.qq, make_double2(cr, ci)));
          if (g.xprev) {
            const double2 xp = ld2_plain(g.xprev + o);
            rmax = nanmax(rmax, hypot(nw.x - xp.x, nw.y - xp.y));
          }
          st2(g.out + o, nw);
          for (int h = 0; h < g.npeer; ++h)
            st2(reinterpret_cast<double*>(g.peers[h]) + ((size_t)(g.r0 + gi) * g.n + gj) * 2, nw);
        } else {
          const size_t oij = ((size_t)gi * g.ld + gj) * 2, oji = ((size_t)gj * g.ld + gi) * 2;
          const double2 aij = ld2_plain(g.amat + oij), aji = ld2_plain(g.amat + oji);
          // (a - a^H)_ij = a_ij - conj(a_ji)
          const double2 dij = make_double2(__dsub_rn(aij.x, aji.x), __dadd_rn(aij.y, aji.y));
          {
            const double2 bij = make_double2(cr, ci);
            const double2 base = ld2_plain(g.base + oij);
            const double2 s1 = cadd(base, rmul(g.hh, dij));
            const double2 nw = cadd(s1, rmul(g.qq, bij));
            if (g.xprev) {
              const double2 xp = ld2_plain(g.xprev + oij);
              rmax = nanmax(rmax, hypot(nw.x - xp.x, nw.y - xp.y));
            }
            if (g.wn) {
              const double2 s2 = csub(base, rmul(g.hh, dij));
              const double2 rc = cadd(s2, rmul(g.qq, bij));
              const double2 w0 = ld2_plain(g.wn + oij);
              cmax = nanmax(cmax, hypot(rc.x - w0.x, rc.y - w0.y));
            }
            st2(g.out + oij, nw);
          }
          if (I != J) {
            // mirror: b_ji = -conj(b_ij); (a - a^H)_ji = -conj(dij)
            const double2 bji = make_double2(-cr, ci);
            const double2 dji = make_double2(-dij.x, dij.y);
            const double2 base = ld2_plain(g.base + oji);
            const double2 s1 = cadd(base, rmul(g.hh, dji));
            const double2 nw = cadd(s1, rmul(g.qq, bji));
            if (g.xprev) {
              const double2 xp = ld2_plain(g.xprev + oji);
              rmax = nanmax(rmax, hypot(nw.x - xp.x, nw.y - xp.y));
            }
            if (g.wn) {
              const double2 s2 = csub(base, rmul(g.hh, dji));
              const double2 rc = cadd(s2, rmul(g.qq, bji));
              const double2 w0 = ld2_plain(g.wn + oji);
              cmax = nanmax(cmax, hypot(rc.x - w0.x, rc.y - w0.y));
            }
            st2(g.out + oji, nw);
          }
        }
      }
    }
  }
}

// CTA-wide NaN-propagating max of the consumer warps, one atomic per CTA.
__device__ __forceinline__ void reduce_max_atomic(double rmax, double cmax, unsigned long long* resid,
                                                  unsigned long long* cons, unsigned long long* red_res,
                                                  unsigned long long* red_cons) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  unsigned long long rb = (unsigned long long)__double_as_longlong(fabs(rmax));
  unsigned long long cb = (unsigned long long)__double_as_longlong(fabs(cmax));
  if (rmax != rmax) rb = 0x7ff8000000000000ull;
  if (cmax != cmax) cb = 0x7ff8000000000000ull;
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    rb = max(rb, __shfl_xor_sync(0xffffffff, rb, off));
    cb = max(cb, __shfl_xor_sync(0xffffffff, cb, off));
  }
  if (lane == 0) {
    red_res[warp] = rb;
    red_cons[warp] = cb;
  }
  asm volatile("bar.sync 1, %0;" ::"r"(CONSUMER_WARPS * 32));
  if (threadIdx.x == 0) {
    unsigned long long r = 0, c = 0;
    for (int q = 0; q < CONSUMER_WARPS; ++q) {
      r = max(r, red_res[q]);
      c = max(c, red_cons[q]);
    }
    if (resid) atomicMax(resid, r);
    if (cons) atomicMax(cons, c);
  }
}

__device__ __forceinline__ void producer_load_stage(unsigned char* st, const CUtensorMap* ma, const CUtensorMap* mb,
                                                    int k0, int row0, int col0, uint64_t* bar,
                                                    const double* pa = nullptr, const double* pb = nullptr) {
  // pa / pb: the sum-plane tiles (A: rows row0.., k k0..; B: k k0.., cols col0..)
  mbar_arrive_expect_tx(bar, STAGE_BYTES + (pa ? SUM_STAGE_BYTES : 0));
  if (pa) {
    bulk_g2s(st + STAGE_BYTES, pa, PLANE_TILE * 8, bar);
    bulk_g2s(st + STAGE_BYTES + PLANE_TILE * 8, pb, PLANE_TILE * 8, bar);
  }
#pragma unroll
  for (int j = 0; j < A_BOXES; ++j) tma_2d(st + j * A_BOX_BYTES, ma, 2 * (k0 + 8 * j), row0, bar);
#pragma unroll
  for (int q = 0; q < B_BOXES; ++q) tma_2d(st + A_STAGE_BYTES + q * B_BOX_BYTES, mb, 2 * (col0 + 8 * q), k0, bar);
}

// ---- one-tile-per-CTA kernel (generic products, config-3 ops, sharded) ----
template <int ALGO, int EPI>
__global__ void __launch_bounds__(GEMM_THREADS, 1) k_zgemm(const __grid_constant__ GemmArgs g) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  // 128B swizzle needs 1024B-aligned boxes
  // offset (not an integer cast) keeps the shared address space visible to
  // the compiler: fragment loads become LDS, not generic LD
  unsigned char* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES);
  uint64_t* empty = full + STAGES;
  __shared__ unsigned long long red_res[CONSUMER_WARPS], red_cons[CONSUMER_WARPS];

  const int n = g.n;
  const int mrows = g.m;
  const int T = (n + BM - 1) / BM;
  int I, J;
  if (EPI == EPI_UPDATE || (EPI == EPI_STORE && g.lower)) {
    tile_of(blockIdx.x, true, T, I, J);
  } else {
    // grouped rasterisation over a (ceil(m/64) x ceil(n/64)) tile grid
    const int Tm = (mrows + BM - 1) / BM;
    const int G = 8, per = G * T, t = blockIdx.x;
    const int grp = t / per, first = grp * G, rows = min(G, Tm - first), r = t - grp * per;
    I = first + r % rows;
    J = r / rows;
  }
  const int row0 = I * BM, col0 = J * BN;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int KT = (g.k + BK - 1) / BK;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], CONSUMER_WARPS);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  if (warp == CONSUMER_WARPS) {
    // ===== producer: one thread issues 2D TMA boxes into the ring =====
    if (lane == 0) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(&g.tma_a) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(&g.tma_b) : "memory");
      for (int kt = 0; kt < KT; ++kt) {
        const int s = kt % STAGES;
        mbar_wait(&empty[s], ((kt / STAGES) & 1) ^ 1);
        producer_load_stage(smem + s * STAGE_BYTES, &g.tma_a, &g.tma_b, kt * BK, row0, col0, &full[s]);
      }
    }
    return;
  }

  // ===== consumer warps: 2 (M) x 4 (N), warp tile 32 x 16 complex =====
  const int wm = warp / WN_WARPS, wn = warp % WN_WARPS;
  Acc<ALGO> acc;
  acc.zero();
  for (int kt = 0; kt < KT; ++kt) {
    const int s = kt % STAGES;
    mbar_wait(&full[s], (kt / STAGES) & 1);
    consume_stage<ALGO>(smem + s * STAGE_BYTES, acc, wm, wn, lane);
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
  }
  double rmax = 0.0, cmax = 0.0;
  epilogue_tile<ALGO, EPI>(g, acc, I, J, wm, wn, lane, rmax, cmax);
  if (g.npeer || g.mirror) __threadfence_system();  // peer stores visible before the rank barrier
  if (EPI != EPI_STORE) reduce_max_atomic(rmax, cmax, g.resid, g.cons, red_res, red_cons);
}

// ---- 3M sum planes --------------------------------------------------------
// A layout (operand rows r, inner index k): tile (r/64, k/16), slot
// ((ks*2 + wm)*4 + i)*32 + fr*4 + fk with r%64 = wm*32 + i*8 + fr and
// k%16 = 8*(ks>>1) + 2*fk + (ks&1) — exactly the DMMA A-fragment order of
// consume_stage.  B layout (inner k, columns c): tile (k/16, c/64), slot
// ((ks*WN_WARPS + wn)*WNB + j)*32 + fr*4 + fk with c%64 = wn*8*WNB + j*8 + fr.
__device__ __forceinline__ size_t a_plane_index(int r, int k, int kbt) {
  const int ri = r & 63, ki = k & 15;
  const int wm = ri >> 5, i = (ri >> 3) & 3, fr = ri & 7;
  const int ks = 2 * (ki >> 3) + (ki & 1), fk = (ki & 7) >> 1;
  return ((size_t)(r >> 6) * kbt + (k >> 4)) * PLANE_TILE + (((ks * 2 + wm) * 4 + i) * 32 + fr * 4 + fk);
}

__global__ void __launch_bounds__(256) k_sum_planes(int n, const double* __restrict__ p, const double* __restrict__ x,
                                                    int64_t ld, double* pa, double* pb, double* xb, int skip_pb) {
  // blockIdx.y: 0 -> P in A layout, 1 -> P in B layout, 2 -> X in B layout
  // (skip_pb: GEMM-1 only, grid.y = 2 maps 1 -> X)
  const int which = (skip_pb && blockIdx.y == 1) ? 2 : blockIdx.y;
  const int kbt = (n + 15) / 16, cbt = (n + 63) / 64;
  const int ntiles = (which == 0) ? cbt * kbt : kbt * cbt;
  const int tile = blockIdx.x;
  if (tile >= ntiles) return;
  const double* src = (which == 2) ? x : p;
  double* out = (which == 0) ? pa : (which == 1 ? pb : xb);
  for (int slot = threadIdx.x; slot < PLANE_TILE; slot += blockDim.x) {
    const int qq = slot >> 5, ln = slot & 31, fr = ln >> 2, fk = ln & 3;
    int r, c;
    if (which == 0) {
      const int rb = tile / kbt, kb = tile % kbt;
      const int ks = qq >> 3, wm = (qq >> 2) & 1, i = qq & 3;
      r = rb * 64 + wm * 32 + i * 8 + fr;
      c = kb * 16 + 8 * (ks >> 1) + 2 * fk + (ks & 1);
    } else {
      const int kb = tile / cbt, cb = tile % cbt;
      const int ks = qq / (WN_WARPS * WNB), wn = (qq / WNB) % WN_WARPS, j = qq % WNB;
      r = kb * 16 + 8 * (ks >> 1) + 2 * fk + (ks & 1);
      c = cb * 64 + wn * 8 * WNB + j * 8 + fr;
    }
    double v = 0.0;
    if (r < n && c < n) {
      const double2 z = ld2(src + ((size_t)r * ld + c) * 2);
      v = z.x + z.y;
    }
    out[(size_t)tile * PLANE_TILE + slot] = v;
  }
}

// ---- persistent fused update: GEMM-1 tiles then GEMM-2 lower tiles --------
// Work ids [0, T^2) are GEMM-1 tiles a = P X (grouped rasterisation, store a
// and count the finished tiles of each row panel); ids [T^2, T^2 + T(T+1)/2)
// are GEMM-2 lower tiles b = a P with the fused update epilogue, which need
// a's row panels I (operand) and J (a^H in the epilogue) complete.  Ids are
// handed out in order by one global atomic, so every dependency of a running
// tile belongs to a tile already held by a co-resident CTA: no deadlock.
struct FusedArgs {
  GemmArgs g2;           // GEMM-2 + update (EPI_UPDATE fields; tma_a = a, tma_b = P)
  CUtensorMap tma_p;     // GEMM-1 A operand (P)
  CUtensorMap tma_x;     // GEMM-1 B operand (X)
  double* a_out;         // GEMM-1 output a
  unsigned int* next;    // global tile counter (zeroed per launch)
  unsigned int* done;    // [T] finished GEMM-1 tiles per row panel (zeroed per launch)
  // ALGO_3MS sum planes: GEMM-1 A (P, A layout) / B (X, B layout); GEMM-2
  // A (a, A layout, written by the GEMM-1 epilogue) / B (P, B layout)
  const double* pa1;
  const double* pb1;
  double* pa2;
  const double* pb2;
  // split-K tail: the last `split_s` GEMM-2 tiles run as `split_f` K-slices
  // each (one work id per slice), so the last round of the persistent grid is
  // a fraction of a tile instead of a partial wave of whole tiles; slices
  // store their 3M accumulators to `split_acc` and the last slice to finish
  // (per-tile counter `split_sem`) sums them and runs the update epilogue
  int split_s, split_f;
  unsigned int* split_sem;  // [split_s] (zeroed per launch)
  // b_out != nullptr: GEMM-2 tiles store b = a P (lower and diagonal tiles)
  // there and the update runs as a separate streaming pass (k_update_pairs)
  double* b_out;
  double* split_acc;        // [split_s * split_f][NACC*4*WNB*2][consumer threads]
  int gemm1_only;           // final update: only a = P X (no GEMM-2, no a plane)
  // progressive final update (gemm1_only): tiles in row-block shell order;
  // the second CTA to finish a tile pair {(I,J), (J,I)} writes W_{n+1} on
  // both tiles (W_n + h (a - a^H), k_final_commutator's arithmetic) into
  // `wout`, and the last pair of a 64-row block publishes it by storing the
  // step's epoch into row_flag[block] (a copy stream waits on it and moves
  // the block to the host while the GEMM continues)
  int prog;
  const double* wn;
  double* wout;
  double h;
  unsigned int* pair_cnt;   // [T (T + 1) / 2] (zeroed per launch)
  unsigned int* rows_done;  // [T] (zeroed per launch)
  unsigned int* row_flag;   // [T] block-ready flags (cleared by the host per step)
};

constexpr int SPLIT_MAX_PARTS = 320;
constexpr int SPLIT_PART_DOUBLES = 3 * 4 * WNB * 2 * CONSUMER_WARPS * 32;

__device__ __forceinline__ unsigned int ld_acquire(const unsigned int* p) {
  unsigned int v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// Progressive final update, called by every consumer thread right after its
// CTA published GEMM-1 tile (I, J) of a (stores fenced, consumer barrier
// passed).  The second tile of the pair to finish writes W_{n+1} on both
// tiles from its own accumulators and the partner tile of a.
template <int ALGO>
__device__ __forceinline__ void progressive_pair(const FusedArgs& f, const Acc<ALGO>& A, int I, int J, int T,
                                                 int wm, int wn, int lane, int& flag_smem) {
  const int lo = min(I, J), hi = max(I, J);
  if (threadIdx.x == 0) {
    const unsigned old = (I == J) ? 1u : atomicAdd(f.pair_cnt + hi * (hi + 1) / 2 + lo, 1u);
    flag_smem = (old == 1u);
  }
  asm volatile("bar.sync 2, %0;" ::"r"(CONSUMER_WARPS * 32));
  const bool fin = flag_smem;
  asm volatile("bar.sync 2, %0;" ::"r"(CONSUMER_WARPS * 32));
  if (!fin) return;
  __threadfence();  // acquire: the partner CTA fenced its a tile before counting
  const int n = f.g2.n;
  const double h = f.h;
  const double* a = f.a_out;
  const int fr = lane >> 2, fk = lane & 3;
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < WNB; ++j)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int gi = I * BM + wm * 32 + i * 8 + fr;
        const int gj = J * BN + wn * 8 * WNB + j * 8 + fk * 2 + e;
        if (gi >= n || gj >= n) continue;
        double cr, ci;
        if (ALGO != ALGO_4M) {
          cr = A.v[0][i][j][e] - A.v[1][i][j][e];
          ci = A.v[2][i][j][e] - A.v[0][i][j][e] - A.v[1][i][j][e];
        } else {
          cr = A.v[0][i][j][e];
          ci = A.v[1][i][j][e];
        }
        const size_t oij = ((size_t)gi * n + gj) * 2, oji = ((size_t)gj * n + gi) * 2;
        const double2 aji = __ldcg(reinterpret_cast<const double2*>(a + oji));
        // k_final_commutator's arithmetic: d = a - a^H, W_n + h d
        const double2 d = make_double2(__dsub_rn(cr, aji.x), __dadd_rn(ci, aji.y));
        const double2 w0 = ld2(f.wn + oij);
        st2(f.wout + oij, make_double2(__dadd_rn(w0.x, __dmul_rn(h, d.x)), __dadd_rn(w0.y, __dmul_rn(h, d.y))));
        if (I != J) {  // (a - a^H)_ji = -conj(d)
          const double2 w1 = ld2(f.wn + oji);
          st2(f.wout + oji, make_double2(__dadd_rn(w1.x, __dmul_rn(h, -d.x)), __dadd_rn(w1.y, __dmul_rn(h, d.y))));
        }
      }
  __threadfence_system();
  asm volatile("bar.sync 2, %0;" ::"r"(CONSUMER_WARPS * 32));
  if (threadIdx.x == 0) {
    for (int q = 0; q < (I == J ? 1 : 2); ++q) {
      const int rb = q ? J : I;
      if (atomicAdd(f.rows_done + rb, 1u) + 1u == (unsigned)T) {
        __threadfence_system();
        asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(f.row_flag + rb), "r"(1u) : "memory");
      }
    }
  }
}

template <int ALGO>
__global__ void __launch_bounds__(GEMM_THREADS, 1) k_zupdate(const __grid_constant__ FusedArgs f) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  constexpr bool PL = (ALGO == ALGO_3MS);
  constexpr int SB = STAGE_BYTES + (PL ? SUM_STAGE_BYTES : 0);
  // offset (not an integer cast) keeps the shared address space visible to
  // the compiler: fragment loads become LDS, not generic LD
  unsigned char* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * SB);
  uint64_t* empty = full + STAGES;
  uint64_t* tq_full = empty + STAGES;  // [2]
  uint64_t* tq_empty = tq_full + 2;    // [2]
  __shared__ int tq[2];
  __shared__ unsigned long long red_res[CONSUMER_WARPS], red_cons[CONSUMER_WARPS];
  __shared__ int split_last;

  const GemmArgs& g = f.g2;
  const int n = g.n;
  const int T = (n + BM - 1) / BM;
  const int L2 = T * (T + 1) / 2;
  const int T1 = T * T, total = f.gemm1_only ? T1 : T1 + L2 + f.split_s * (f.split_f - 1);
  const int KT = (n + BK - 1) / BK;
  // work id -> (GEMM-2 lower-tile index, K slice): ids past the unsplit
  // GEMM-2 tiles are slices of the tail tiles
  auto g2_unit = [&](int u, int& tile, int& part, int& sidx) {
    const int full = L2 - f.split_s;
    if (u < full) {
      tile = u;
      part = -1;
      sidx = -1;
    } else {
      sidx = (u - full) / f.split_f;
      part = (u - full) - sidx * f.split_f;
      tile = full + sidx;
    }
  };
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], CONSUMER_WARPS);
    }
    for (int q = 0; q < 2; ++q) {
      mbar_init(&tq_full[q], 1);
      mbar_init(&tq_empty[q], CONSUMER_WARPS);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  if (warp == CONSUMER_WARPS) {
    if (lane != 0) return;
    // ===== producer thread: fetch tile ids, resolve dependencies, stream stages =====
    asm volatile("prefetch.tensormap [%0];" ::"l"(&f.tma_p) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&f.tma_x) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&g.tma_a) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&g.tma_b) : "memory");
    unsigned int gs = 0;  // running stage count (ring position)
    for (int j = 0;; ++j) {
      const int id = (int)atomicAdd(f.next, 1u);
      const int slot = j & 1;
      mbar_wait(&tq_empty[slot], ((j >> 1) & 1) ^ 1);
      tq[slot] = id < total ? id : -1;
      mbar_arrive(&tq_full[slot]);
      if (id >= total) break;
      int I, J, tl, part = -1, sidx = -1;
      const CUtensorMap *ma, *mb;
      const double *pla, *plb;
      if (id < T1) {
        if (f.prog)
          shell_tile(id, T, I, J);
        else
          tile_of(id, false, T, I, J);
        ma = &f.tma_p;
        mb = &f.tma_x;
        pla = f.pa1;
        plb = f.pb1;
      } else {
        g2_unit(id - T1, tl, part, sidx);
        tile_of(tl, true, T, I, J);
        ma = &g.tma_a;
        mb = &g.tma_b;
        pla = f.pa2;
        plb = f.pb2;
        // a's row panels I and J must be complete (stored by other CTAs)
        while (ld_acquire(f.done + I) < (unsigned)T) __nanosleep(64);
        if (!f.b_out)
          while (ld_acquire(f.done + J) < (unsigned)T) __nanosleep(64);
        asm volatile("fence.proxy.async.global;" ::: "memory");
      }
      const int kbt = KT;  // k blocks of 16
      const int k0 = part < 0 ? 0 : part * KT / f.split_f;
      const int k1 = part < 0 ? KT : (part + 1) * KT / f.split_f;
      for (int kt = k0; kt < k1; ++kt, ++gs) {
        const int s = gs % STAGES;
        mbar_wait(&empty[s], ((gs / STAGES) & 1) ^ 1);
        if (PL)
          producer_load_stage(smem + s * SB, ma, mb, kt * BK, I * BM, J * BN, &full[s],
                              pla + ((size_t)I * kbt + kt) * PLANE_TILE, plb + ((size_t)kt * T + J) * PLANE_TILE);
        else
          producer_load_stage(smem + s * SB, ma, mb, kt * BK, I * BM, J * BN, &full[s]);
      }
    }
    return;
  }

  // ===== consumers =====
  const int wm = warp / WN_WARPS, wn = warp % WN_WARPS;
  double rmax = 0.0, cmax = 0.0;
  unsigned int gs = 0;
  GemmArgs g1 = g;  // GEMM-1 epilogue: plain store of a
  g1.c = f.a_out;
  g1.ldc = g.ld;
  g1.m = n;
  for (int j = 0;; ++j) {
    const int slot = j & 1;
    mbar_wait(&tq_full[slot], (j >> 1) & 1);
    const int id = tq[slot];
    __syncwarp();
    if (lane == 0) mbar_arrive(&tq_empty[slot]);
    if (id < 0) break;
    int I, J, tl = 0, part = -1, sidx = -1;
    const bool phase1 = id < T1;
    if (phase1) {
      if (f.prog)
        shell_tile(id, T, I, J);
      else
        tile_of(id, false, T, I, J);
    } else {
      g2_unit(id - T1, tl, part, sidx);
      tile_of(tl, true, T, I, J);
    }
    Acc<ALGO> acc;
    acc.zero();
    const int k0 = part < 0 ? 0 : part * KT / f.split_f;
    const int k1 = part < 0 ? KT : (part + 1) * KT / f.split_f;
    for (int kt = k0; kt < k1; ++kt, ++gs) {
      const int s = gs % STAGES;
      mbar_wait(&full[s], (gs / STAGES) & 1);
      consume_stage<ALGO>(smem + s * SB, acc, wm, wn, lane);
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
    }
    if (phase1) {
      epilogue_tile<ALGO, EPI_STORE>(g1, acc, I, J, wm, wn, lane, rmax, cmax);
      if (PL && !f.gemm1_only) {
        // a's 3M sum plane (A layout) for the GEMM-2 tiles of this row panel
        const int fr = lane >> 2, fk = lane & 3;
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < WNB; ++j)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
              const int gi = I * BM + wm * 32 + i * 8 + fr;
              const int gj = J * BN + wn * 8 * WNB + j * 8 + fk * 2 + e;
              const double cr = acc.v[0][i][j][e] - acc.v[1][i][j][e];
              const double ci = acc.v[2][i][j][e] - acc.v[0][i][j][e] - acc.v[1][i][j][e];
              // padding rows/cols (>= n) must hold zeros, as the zero-filled TMA
              // tiles; columns past the plane's 16*KT width do not exist in it
              if (gj < KT * BK) f.pa2[a_plane_index(gi, gj, KT)] = (gi < n && gj < n) ? cr + ci : 0.0;
            }
      }
      // publish the tile: every thread fences its stores (generic and async
      // proxy), the consumer group syncs, one thread counts the tile
      __threadfence();
      asm volatile("fence.proxy.async.global;" ::: "memory");
      asm volatile("bar.sync 2, %0;" ::"r"(CONSUMER_WARPS * 32));
      if (threadIdx.x == 0) atomicAdd(f.done + I, 1u);
      if (f.prog) progressive_pair(f, acc, I, J, T, wm, wn, lane, split_last);
    } else {
      if (part >= 0) {
        // K slice of a tail tile: publish the partial accumulators; the last
        // slice to arrive adds the others and runs the epilogue
        constexpr int NV = Acc<ALGO>::NACC * 4 * WNB * 2;
        const int tid = threadIdx.x;
        double* mine = f.split_acc + (size_t)(sidx * f.split_f + part) * SPLIT_PART_DOUBLES;
        const double* av = &acc.v[0][0][0][0];
#pragma unroll
        for (int q = 0; q < NV; ++q) __stcg(mine + (size_t)q * (CONSUMER_WARPS * 32) + tid, av[q]);
        __threadfence();
        asm volatile("bar.sync 2, %0;" ::"r"(CONSUMER_WARPS * 32));
        if (tid == 0) split_last = (atomicAdd(f.split_sem + sidx, 1u) == (unsigned)f.split_f - 1u);
        asm volatile("bar.sync 2, %0;" ::"r"(CONSUMER_WARPS * 32));
        const bool last = split_last;
        asm volatile("bar.sync 2, %0;" ::"r"(CONSUMER_WARPS * 32));
        if (!last) continue;
        __threadfence();
        double* aw = &acc.v[0][0][0][0];
        for (int o = 0; o < f.split_f; ++o) {
          if (o == part) continue;
          const double* other = f.split_acc + (size_t)(sidx * f.split_f + o) * SPLIT_PART_DOUBLES;
#pragma unroll
          for (int q = 0; q < NV; ++q) aw[q] += __ldcg(other + (size_t)q * (CONSUMER_WARPS * 32) + tid);
        }
      }
      if (f.b_out) {
        GemmArgs gb = g1;
        gb.c = f.b_out;
        epilogue_tile<ALGO, EPI_STORE>(gb, acc, I, J, wm, wn, lane, rmax, cmax);
        continue;
      }
      if (lane == 0) {
        // order this warp's epilogue reads of a after the producer's acquire
        while (ld_acquire(f.done + I) < (unsigned)T) __nanosleep(32);
        while (ld_acquire(f.done + J) < (unsigned)T) __nanosleep(32);
      }
      __syncwarp();
      epilogue_tile<ALGO, EPI_UPDATE>(g, acc, I, J, wm, wn, lane, rmax, cmax);
    }
  }
  reduce_max_atomic(rmax, cmax, g.resid, g.cons, red_res, red_cons);
}

// elementwise c = a - a^H (commutator op, integrator.py:127-128 form)
__global__ void k_skew_diff(int n, const double* __restrict__ a, double* __restrict__ c) {
  __shared__ double2 tile[32][33];
  const int bx = blockIdx.x * 32, by = blockIdx.y * 32;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  for (int r = ty; r < 32; r += 8) {
    const int i = bx + r, j = by + tx;  // a[bx.., by..] transposed source tile
    tile[r][tx] = (i < n && j < n) ? ld2(a + ((size_t)i * n + j) * 2) : make_double2(0, 0);
  }
  __syncthreads();
  for (int r = ty; r < 32; r += 8) {
    const int i = by + r, j = bx + tx;
    if (i < n && j < n) {
      const double2 aij = ld2(a + ((size_t)i * n + j) * 2);
      const double2 aji = tile[tx][r];
      st2(c + ((size_t)i * n + j) * 2, make_double2(aij.x - aji.x, aij.y + aji.y));
    }
  }
}

static int make_map(CUtensorMap* map, const double* base, int rows, int cols, int64_t ld, int box_rows) {
  if ((reinterpret_cast<uintptr_t>(base) & 15) || ld < cols) return fail(ZT_EINVAL, "zgemm: operand must be 16B aligned with ld >= cols");
  cuuint64_t dims[2] = {(cuuint64_t)2 * cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)ld * 16};
  cuuint32_t box[2] = {16, (cuuint32_t)box_rows};
  return encode_tiled_f64(map, 2, base, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_128B);
}

static bool g_attr[16][16];

template <int ALGO, int EPI>
static int launch(GemmArgs& g, int ntiles, cudaStream_t st) {
  int rc = make_map(&g.tma_a, g.a, g.m, g.k, g.lda, BM);
  if (rc) return rc;
  rc = make_map(&g.tma_b, g.b, g.k, g.n, g.ldb, BK);
  if (rc) return rc;
  int dev;
  cudaGetDevice(&dev);
  const int slot = ALGO * 3 + EPI;
  if (dev < 16 && !g_attr[dev][slot]) {
    ZT_CUDA_CHECK(cudaFuncSetAttribute(k_zgemm<ALGO, EPI>, cudaFuncAttributeMaxDynamicSharedMemorySize, GEMM_SMEM));
    g_attr[dev][slot] = true;
  }
  k_zgemm<ALGO, EPI><<<ntiles, GEMM_THREADS, GEMM_SMEM, st>>>(g);
  ZT_LAUNCHED();
  ZT_CUDA_CHECK(cudaGetLastError());
  return ZT_OK;
}

int zgemm(int n, const double* a, int64_t lda, const double* b, int64_t ldb, double* c, int64_t ldc,
          int algo, cudaStream_t st) {
  if (n < 1) return fail(ZT_EINVAL, "zgemm: n must be positive");
  GemmArgs g{};
  g.n = n;
  g.m = n;
  g.k = n;
  g.a = a;
  g.lda = lda;
  g.b = b;
  g.ldb = ldb;
  g.c = c;
  g.ldc = ldc;
  const int T = (n + BM - 1) / BM;
  if (algo == ALGO_4M) return launch<ALGO_4M, EPI_STORE>(g, T * T, st);
  return launch<ALGO_3M, EPI_STORE>(g, T * T, st);
}

// b = amat @ p on lower tiles; out = base + hh (a - a^H) + qq b (+ mirror)
int zgemm_update(int n, const double* amat, const double* p, const double* base, const double* xprev,
                 const double* wn, double* out, int64_t ld, double hh, double qq,
                 unsigned long long* resid, unsigned long long* cons, int algo, cudaStream_t st) {
  GemmArgs g{};
  g.n = n;
  g.m = n;
  g.k = n;
  g.a = amat;
  g.lda = ld;
  g.b = p;
  g.ldb = ld;
  g.amat = amat;
  g.base = base;
  g.xprev = xprev;
  g.wn = wn;
  g.out = out;
  g.ld = ld;
  g.hh = hh;
  g.qq = qq;
  g.resid = resid;
  g.cons = cons;
  const int T = (n + BM - 1) / BM;
  const int nt = T * (T + 1) / 2;
  if (algo == ALGO_4M) return launch<ALGO_4M, EPI_UPDATE>(g, nt, st);
  return launch<ALGO_3M, EPI_UPDATE>(g, nt, st);
}

// Rectangular C (m x n) = A (m x k) B (k x n)
int zgemm_rect(int m, int n, int k, const double* a, int64_t lda, const double* b, int64_t ldb, double* c,
               int64_t ldc, int algo, cudaStream_t st) {
  if (m < 1 || n < 1 || k < 1) return fail(ZT_EINVAL, "zgemm: sizes must be positive");
  GemmArgs g{};
  g.n = n;
  g.m = m;
  g.k = k;
  g.a = a;
  g.lda = lda;
  g.b = b;
  g.ldb = ldb;
  g.c = c;
  g.ldc = ldc;
  const int nt = ((m + BM - 1) / BM) * ((n + BN - 1) / BN);
  if (algo == ALGO_4M) return launch<ALGO_4M, EPI_STORE>(g, nt, st);
  return launch<ALGO_3M, EPI_STORE>(g, nt, st);
}

// Rectangular product whose epilogue also scatters the result's column
// blocks into the ranks' a[:, R_h] buffers (fused all-to-all).
int zgemm_rect_scatter(int m, int n, int k, const double* a, int64_t lda, const double* b, int64_t ldb, double* c,
                       int64_t ldc, const unsigned long long* peers, int npeer, int r0, int mloc, int algo,
                       cudaStream_t st) {
  if (m < 1 || n < 1 || k < 1 || npeer < 1 || mloc < 1 || n != npeer * mloc)
    return fail(ZT_EINVAL, "zgemm_rect_scatter: bad sizes");
  GemmArgs g{};
  g.n = n;
  g.m = m;
  g.k = k;
  g.a = a;
  g.lda = lda;
  g.b = b;
  g.ldb = ldb;
  g.c = c;
  g.ldc = ldc;
  g.peers = peers;
  g.npeer = npeer;
  g.r0 = r0;
  g.mloc = mloc;
  const int nt = ((m + BM - 1) / BM) * ((n + BN - 1) / BN);
  if (algo == ALGO_4M) return launch<ALGO_4M, EPI_STORE>(g, nt, st);
  return launch<ALGO_3M, EPI_STORE>(g, nt, st);
}

// Row-block update reading (a^H)_R from this rank's a[:, R] buffer and
// broadcasting the new rows into every rank's N x N iterate (fused all-gather).
int zgemm_update_rows_peer(int m, int n, const double* a_rows, const double* p, const double* acol, int mloc,
                           const double* base, const double* xprev, double* out, int64_t ld, double hh, double qq,
                           unsigned long long* resid, const unsigned long long* peers, int npeer, int r0, int algo,
                           cudaStream_t st) {
  if (m < 1 || n < 1 || npeer < 0 || !acol) return fail(ZT_EINVAL, "zgemm_update_rows_peer: bad arguments");
  GemmArgs g{};
  g.n = n;
  g.m = m;
  g.k = n;
  g.a = a_rows;
  g.lda = ld;
  g.b = p;
  g.ldb = n;
  g.amat = a_rows;
  g.acol = acol;
  g.mloc = mloc;
  g.base = base;
  g.xprev = xprev;
  g.out = out;
  g.ld = ld;
  g.hh = hh;
  g.qq = qq;
  g.resid = resid;
  g.peers = peers;
  g.npeer = npeer;
  g.r0 = r0;
  const int nt = ((m + BM - 1) / BM) * ((n + BN - 1) / BN);
  if (algo == ALGO_4M) return launch<ALGO_4M, EPI_ROWS>(g, nt, st);
  return launch<ALGO_3M, EPI_ROWS>(g, nt, st);
}

// C = A B (m x n, inner k) and -conj(C^T) into `mirror` (n x m, ld_mirror):
// one skew-Hermitian block product for this rank and its partner.
int zgemm_rect_mirror(int m, int n, int k, const double* a, int64_t lda, const double* b, int64_t ldb, double* c,
                      int64_t ldc, double* mirror, int64_t ld_mirror, int algo, cudaStream_t st) {
  if (m < 1 || n < 1 || k < 1) return fail(ZT_EINVAL, "zgemm_rect_mirror: sizes must be positive");
  if (!mirror && m == n) {
    // a diagonal block of the skew-Hermitian product: lower tiles + mirror in place
    GemmArgs g{};
    g.n = n;
    g.m = m;
    g.k = k;
    g.a = a;
    g.lda = lda;
    g.b = b;
    g.ldb = ldb;
    g.c = c;
    g.ldc = ldc;
    g.lower = 1;
    const int T = (n + BM - 1) / BM;
    if (algo == ALGO_4M) return launch<ALGO_4M, EPI_STORE>(g, T * (T + 1) / 2, st);
    return launch<ALGO_3M, EPI_STORE>(g, T * (T + 1) / 2, st);
  }
  GemmArgs g{};
  g.n = n;
  g.m = m;
  g.k = k;
  g.a = a;
  g.lda = lda;
  g.b = b;
  g.ldb = ldb;
  g.c = c;
  g.ldc = ldc;
  g.mirror = mirror;
  g.ld_mirror = ld_mirror;
  const int nt = ((m + BM - 1) / BM) * ((n + BN - 1) / BN);
  if (algo == ALGO_4M) return launch<ALGO_4M, EPI_STORE>(g, nt, st);
  return launch<ALGO_3M, EPI_STORE>(g, nt, st);
}

// Elementwise row-block update from a precomputed b_R (the skew-balanced
// sharded GEMM-2): new = base + hh (a_R - conj(acol)^T) + qq b_R, residual
// max |new - xprev|, new rows also into every rank's N x N iterate.
__global__ void __launch_bounds__(256) k_update_rows_ew(int m, int n, const double* __restrict__ a_rows,
                                                        const double* __restrict__ acol, int mloc,
                                                        const double* __restrict__ b_rows,
                                                        const double* __restrict__ base, const double* xprev,
                                                        double* out, int64_t ld, double hh, double qq,
                                                        unsigned long long* resid,
                                                        const unsigned long long* __restrict__ peers, int npeer,
                                                        int r0) {
  __shared__ double2 tile[32][33];
  const int bj = blockIdx.x * 32, bi = blockIdx.y * 32;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  // (a^H)_R[i][j] = conj(acol[j][i]): stage the transposed 32 x 32 block
  for (int r = ty; r < 32; r += 8) {
    const int j = bj + r, i = bi + tx;
    tile[r][tx] = (j < n && i < m) ? ld2(acol + ((size_t)j * mloc + i) * 2) : make_double2(0.0, 0.0);
  }
  __syncthreads();
  double rmax = 0.0;
  for (int r = ty; r < 32; r += 8) {
    const int i = bi + r, j = bj + tx;
    if (i >= m || j >= n) continue;
    const size_t o = ((size_t)i * ld + j) * 2;
    const double2 aij = ld2(a_rows + o), t = tile[tx][r];
    const double2 d = make_double2(__dsub_rn(aij.x, t.x), __dadd_rn(aij.y, t.y));  // a - conj(acol^T)
    const double2 bb = b_rows ? ld2(b_rows + o) : make_double2(0.0, 0.0);  // null: no b term
    const double2 nw = cadd(cadd(ld2(base + o), rmul(hh, d)), rmul(qq, bb));
    if (xprev) {
      const double2 xp = *reinterpret_cast<const double2*>(xprev + o);
      rmax = nanmax(rmax, hypot(nw.x - xp.x, nw.y - xp.y));
    }
    st2(out + o, nw);
    for (int h = 0; h < npeer; ++h) {
      // (out may be this rank's own rows of the gathered iterate: no second store)
      double* dst = reinterpret_cast<double*>(peers[h]) + ((size_t)(r0 + i) * n + j) * 2;
      if (dst != out + o) st2(dst, nw);
    }
  }
  if (npeer) {  // one system-scope fence per block (cumulative over the block's stores)
    __syncthreads();
    if (threadIdx.x == 0) __threadfence_system();
  }
  if (resid) {
    unsigned long long bits = (unsigned long long)__double_as_longlong(fabs(rmax));
    if (rmax != rmax) bits = 0x7ff8000000000000ull;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) bits = max(bits, __shfl_xor_sync(0xffffffff, bits, off));
    if (tx == 0) atomicMax(resid, bits);
  }
}

int update_rows_ew(int m, int n, const double* a_rows, const double* acol, int mloc, const double* b_rows,
                   const double* base, const double* xprev, double* out, int64_t ld, double hh, double qq,
                   unsigned long long* resid, const unsigned long long* peers, int npeer, int r0, cudaStream_t st) {
  if (m < 1 || n < 1) return fail(ZT_EINVAL, "update_rows_ew: bad sizes");
  dim3 grid((n + 31) / 32, (m + 31) / 32);
  k_update_rows_ew<<<grid, 256, 0, st>>>(m, n, a_rows, acol, mloc, b_rows, base, xprev, out, ld, hh, qq, resid,
                                         peers, npeer, r0);
  ZT_LAUNCHED();
  ZT_CUDA_CHECK(cudaGetLastError());
  return ZT_OK;
}

// Copy a row block into every rank's N x N buffer at rows r0.. (seeds the
// gathered iterate with W_n at the start of a sharded step).
__global__ void k_rows_broadcast(int m, int n, const double* __restrict__ rows, int64_t ld,
                                 const unsigned long long* __restrict__ peers, int npeer, int r0) {
  const size_t total = (size_t)m * n;
  for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < total; e += (size_t)gridDim.x * blockDim.x) {
    const size_t i = e / n, j = e % n;
    const double2 v = ld2(rows + (i * ld + j) * 2);
    for (int h = 0; h < npeer; ++h) st2(reinterpret_cast<double*>(peers[h]) + ((r0 + i) * (size_t)n + j) * 2, v);
  }
  __syncthreads();
  if (threadIdx.x == 0) __threadfence_system();
}

int rows_broadcast(int m, int n, const double* rows, int64_t ld, const unsigned long long* peers, int npeer, int r0,
                   cudaStream_t st) {
  if (m < 1 || n < 1 || npeer < 1) return fail(ZT_EINVAL, "rows_broadcast: bad sizes");
  k_rows_broadcast<<<592, 256, 0, st>>>(m, n, rows, ld, peers, npeer, r0);
  ZT_LAUNCHED();
  ZT_CUDA_CHECK(cudaGetLastError());
  return ZT_OK;
}

// Row-block update of the sharded step: b = a_R P (m x n, inner n);
// out = base + hh (a_R - ah_R) + qq b, residual max|out - xprev|.
int zgemm_update_rows(int m, int n, const double* a_rows, const double* p, const double* ah_rows,
                      const double* base, const double* xprev, double* out, int64_t ld, double hh,
                      double qq, unsigned long long* resid, int algo, cudaStream_t st) {
  GemmArgs g{};
  g.n = n;
  g.m = m;
  g.k = n;
  g.a = a_rows;
  g.lda = ld;
  g.b = p;
  g.ldb = n;
  g.amat = a_rows;
  g.ah = ah_rows;
  g.base = base;
  g.xprev = xprev;
  g.out = out;
  g.ld = ld;
  g.hh = hh;
  g.qq = qq;
  g.resid = resid;
  const int nt = ((m + BM - 1) / BM) * ((n + BN - 1) / BN);
  if (algo == ALGO_4M) return launch<ALGO_4M, EPI_ROWS>(g, nt, st);
  return launch<ALGO_3M, EPI_ROWS>(g, nt, st);
}

// One fixed-point update after the solve: a = P X and the GEMM-2 update in
// one persistent launch (grid = SMs).  `sync` must hold (T + 1) u32 zeros.
static bool g_fattr[16][3];
static int g_sms[16];

size_t sum_plane_bytes(int n) {
  return (size_t)((n + 63) / 64) * 64 * ((n + 15) / 16) * 16 * sizeof(double);
}

// progressive final update words: pair counters, row counters, row flags
size_t zupdate_prog_words(int n) {
  const size_t T = (n + BM - 1) / BM;
  return T * (T + 1) / 2 + 2 * T;
}

size_t zupdate_split_bytes(int n) {
  const int T = (n + BM - 1) / BM;
  const int parts = std::min(SPLIT_MAX_PARTS, 4 * (T * (T + 1) / 2));
  return sizeof(double) * (size_t)parts * SPLIT_PART_DOUBLES;
}
int zupdate_sync_words(int n) { return (n + BM - 1) / BM + 1 + SPLIT_MAX_PARTS; }

// Split-K tail: with U work units on G resident CTAs the last round holds
// r = U mod G whole tiles; splitting them into f K-slices makes it
// ceil(f r / G) / f tiles long.  Pick the f in {2, 3, 4} that shortens it most.
static void pick_split(int U, int G, int L2, int n, int& S, int& F) {
  S = 0;
  F = 1;
  const int r = U % G;
  if (r == 0 || G <= 1 || n < 256) return;
  double best = 1.0;
  const int cap = (int)(zupdate_split_bytes(n) / (sizeof(double) * SPLIT_PART_DOUBLES));
  for (int fs = 2; fs <= 4; ++fs) {
    if (r > L2 || r * fs > cap) continue;
    const double len = (double)((fs * r + G - 1) / G) / fs;
    if (len < best - 1e-9) {
      best = len;
      S = r;
      F = fs;
    }
  }
}

// Final update of a step without GEMM-2: W_{n+1} = W_n + h (a - a^H).
// With W~ = W_n + (h/2)(a - a^H) + (h^2/4) a P at the fixed point, the
// reference's W~ + (h/2)(a - a^H) - (h^2/4) a P (integrator.py:154-158) is
// W_n + h (a - a^H): the (h^2/4) a P terms cancel.  The two differ only by
// O(h |P| |X_k - X_{k-1}|) from the fixed point's last correction (~1e-19
// at the configs' contraction); tests hold it to the reference.
__global__ void __launch_bounds__(256) k_final_commutator(int n, const double* __restrict__ a,
                                                          const double* __restrict__ wn, double h,
                                                          double* __restrict__ out) {
  __shared__ double2 tile[32][33];
  const int bx = blockIdx.x * 32, by = blockIdx.y * 32;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  pdl_wait();
  for (int r = ty; r < 32; r += 8) {
    const int i = bx + r, j = by + tx;  // a[bx.., by..], read transposed below
    tile[r][tx] = (i < n && j < n) ? ld2(a + ((size_t)i * n + j) * 2) : make_double2(0, 0);
  }
  __syncthreads();
  for (int r = ty; r < 32; r += 8) {
    const int i = by + r, j = bx + tx;
    if (i < n && j < n) {
      const size_t o = ((size_t)i * n + j) * 2;
      const double2 aij = ld2(a + o), aji = tile[tx][r];
      const double2 d = make_double2(__dsub_rn(aij.x, aji.x), __dadd_rn(aij.y, aji.y));  // a - a^H
      const double2 w0 = ld2(wn + o);
      st2(out + o, make_double2(__dadd_rn(w0.x, __dmul_rn(h, d.x)), __dadd_rn(w0.y, __dmul_rn(h, d.y))));
    }
  }
}

int final_commutator(int n, const double* a, const double* wn, double h, double* out, cudaStream_t st) {
  dim3 grid((n + 31) / 32, (n + 31) / 32);
  ZT_CUDA_CHECK(launch_pdl(k_final_commutator, grid, dim3(256), 0, st, n, a, wn, h, out));
  ZT_LAUNCHED();
  ZT_CUDA_CHECK(cudaGetLastError());
  return ZT_OK;
}

// The update as a streaming pass over 32 x 32 tile pairs (R, C), R >= C:
// new = base + hh (a - a^H) + qq b with b read on and below the diagonal
// and mirrored (b_ji = -conj(b_ij)) above it; every mirror pair is computed
// from negated conjugate operands in the same operation order, so the new
// iterate is exactly skew-Hermitian off the diagonal whenever the base is;
// plus the NaN-propagating residual / consistency maxima.  `out` may alias `xprev`
// (in-place iteration): every element is read and written by one thread.
template <bool XP, bool WN>
__global__ void __launch_bounds__(256, 2) k_update_pairs(int n, const double* __restrict__ a,
                                                      const double* __restrict__ bm, double* out,
                                                      const double* __restrict__ base, const double* xprev,
                                                      const double* __restrict__ wn, double hh, double qq,
                                                      unsigned long long* resid, unsigned long long* cons) {
  // tb[c][r]: a_ji of tile element (r, c) for phase 1, then (the same slot,
  // read once) b_ij for the mirror in phase 2
  __shared__ double2 tb[32][33];
  __shared__ double2 dd[32][33];  // (a - a^H)_ij of tile (R, C)
  __shared__ unsigned long long red[2][8];
  int I = (int)((sqrt(8.0 * blockIdx.x + 1.0) - 1.0) * 0.5);
  while ((I + 1) * (I + 2) / 2 <= (int)blockIdx.x) ++I;
  while (I * (I + 1) / 2 > (int)blockIdx.x) --I;
  const int J = blockIdx.x - I * (I + 1) / 2;
  const int R = I * 32, C = J * 32;
  pdl_wait();
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  double rmax = 0.0, cmax = 0.0;
  // all loads of both phases first (the in-place `out` == `xprev` stores
  // would otherwise pin every load behind the previous row's store)
  const bool two = I != J;
  double2 aij[4], bij[4], b0[4], xp[4], w0[4], b0m[4], xpm[4], w0m[4];  // unused ones fold away
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int r = ty + 8 * q;
    {
      const int i = C + r, j = R + tx;
      tb[r][tx] = (i < n && j < n) ? ld2(a + ((size_t)i * n + j) * 2) : make_double2(0, 0);
    }
    const int i = R + r, j = C + tx;
    const bool ok = i < n && j < n;
    const size_t o = ((size_t)i * n + j) * 2;
    const double2 z = make_double2(0, 0);
    aij[q] = ok ? ld2(a + o) : z;
    bij[q] = ok ? ld2(bm + o) : z;
    b0[q] = ok ? ld2(base + o) : z;
    xp[q] = (XP && ok) ? ld2_plain(xprev + o) : z;
    w0[q] = (WN && ok) ? ld2(wn + o) : z;
    // mirror side: (C + r, R + tx)
    const int im = C + r, jm = R + tx;
    const bool okm = two && im < n && jm < n;
    const size_t om = ((size_t)im * n + jm) * 2;
    b0m[q] = okm ? ld2(base + om) : z;
    xpm[q] = (XP && okm) ? ld2_plain(xprev + om) : z;
    w0m[q] = (WN && okm) ? ld2(wn + om) : z;
  }
  if (!two) {
    // b is used from the lower half only: the upper half of a diagonal tile
    // takes -conj of its mirror, like every other upper entry, so the new
    // iterate is exactly skew-Hermitian off the diagonal whenever the base
    // is (dd, unused by diagonal tiles until the loop below, holds b)
#pragma unroll
    for (int q = 0; q < 4; ++q) dd[ty + 8 * q][tx] = bij[q];
  }
  __syncthreads();
  if (!two) {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int r = ty + 8 * q;
      if (r < tx) {
        const double2 t = dd[tx][r];
        bij[q] = make_double2(-t.x, t.y);
      }
    }
    __syncthreads();  // every read of dd before the loop below rewrites it
  }
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int r = ty + 8 * q;
    const int i = R + r, j = C + tx;
    const double2 aji = tb[tx][r];
    const double2 dij = make_double2(__dsub_rn(aij[q].x, aji.x), __dadd_rn(aij[q].y, aji.y));
    const double2 nw = cadd(cadd(b0[q], rmul(hh, dij)), rmul(qq, bij[q]));
    dd[r][tx] = dij;
    if (i < n && j < n) {
      if (XP) rmax = nanmax(rmax, hypot(nw.x - xp[q].x, nw.y - xp[q].y));
      if (WN) {
        const double2 rc = cadd(csub(b0[q], rmul(hh, dij)), rmul(qq, bij[q]));
        cmax = nanmax(cmax, hypot(rc.x - w0[q].x, rc.y - w0[q].y));
      }
      st2(out + ((size_t)i * n + j) * 2, nw);
    }
  }
  if (two) {
    __syncthreads();  // every a_ji of tb is read; reuse it for b_ij
#pragma unroll
    for (int q = 0; q < 4; ++q) tb[tx][ty + 8 * q] = bij[q];
    __syncthreads();
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int r = ty + 8 * q;
      const int i = C + r, j = R + tx;  // (i, j) = mirror of tile element (tx, r)
      if (i < n && j < n) {
        const double2 d = dd[tx][r];
        const double2 dji = make_double2(-d.x, d.y);
        const double2 t = tb[r][tx];
        const double2 bji = make_double2(-t.x, t.y);
        const double2 nw = cadd(cadd(b0m[q], rmul(hh, dji)), rmul(qq, bji));
        if (XP) rmax = nanmax(rmax, hypot(nw.x - xpm[q].x, nw.y - xpm[q].y));
        if (WN) {
          const double2 rc = cadd(csub(b0m[q], rmul(hh, dji)), rmul(qq, bji));
          cmax = nanmax(cmax, hypot(rc.x - w0m[q].x, rc.y - w0m[q].y));
        }
        st2(out + ((size_t)i * n + j) * 2, nw);
      }
    }
  }
  unsigned long long rb = (unsigned long long)__double_as_longlong(fabs(rmax));
  unsigned long long cb = (unsigned long long)__double_as_longlong(fabs(cmax));
  if (rmax != rmax) rb = 0x7ff8000000000000ull;
  if (cmax != cmax) cb = 0x7ff8000000000000ull;
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    rb = max(rb, __shfl_xor_sync(0xffffffff, rb, off));
    cb = max(cb, __shfl_xor_sync(0xffffffff, cb, off));
  }
  if (tx == 0) {
    red[0][ty] = rb;
    red[1][ty] = cb;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long r = 0, c = 0;
    for (int q = 0; q < 8; ++q) {
      r = max(r, red[0][q]);
      c = max(c, red[1][q]);
    }
    if (resid && xprev) atomicMax(resid, r);
    if (cons && wn) atomicMax(cons, c);
  }
}

// the streaming update pass on its own (b from any GEMM that computed the
// lower and diagonal BM x BN tiles)
int update_pairs(int n, const double* a, const double* bm, double* out, const double* base, const double* xprev,
                 const double* wn, double hh, double qq, unsigned long long* resid, unsigned long long* cons,
                 cudaStream_t st) {
  const int t32 = (n + 31) / 32;
  const int nb = t32 * (t32 + 1) / 2;
  auto k = xprev ? (wn ? k_update_pairs<true, true> : k_update_pairs<true, false>)
                 : (wn ? k_update_pairs<false, true> : k_update_pairs<false, false>);
  ZT_CUDA_CHECK(launch_pdl(k, dim3(nb), dim3(256), 0, st, n, a, bm, out, base, xprev, wn, hh, qq, resid, cons));
  ZT_LAUNCHED();
  return ZT_OK;
}

int zupdate_fused(int n, const double* p, const double* x, double* a, const double* base, const double* xprev,
                  const double* wn, double* out, double hh, double qq, unsigned long long* resid,
                  unsigned long long* cons, unsigned int* sync, int algo, double* planes, double* split,
                  cudaStream_t st, int gemm1_only, double* bbuf, const ProgParams* prog) {
  FusedArgs f;
  memset(&f, 0, sizeof f);
  GemmArgs& g = f.g2;
  g.n = n;
  g.m = n;
  g.k = n;
  g.a = a;
  g.lda = n;
  g.b = p;
  g.ldb = n;
  g.amat = a;
  g.base = base;
  g.xprev = xprev;
  g.wn = wn;
  g.out = out;
  g.ld = n;
  g.hh = hh;
  g.qq = qq;
  g.resid = resid;
  g.cons = cons;
  int rc = make_map(&g.tma_a, a, n, n, n, BM);
  if (!rc) rc = make_map(&g.tma_b, p, n, n, n, BK);
  if (!rc) rc = make_map(&f.tma_p, p, n, n, n, BM);
  if (!rc) rc = make_map(&f.tma_x, x, n, n, n, BK);
  if (rc) return rc;
  f.a_out = a;
  f.next = sync;
  f.done = sync + 1;
  if (algo == ALGO_3MS) {
    if (!planes) return fail(ZT_EINVAL, "3M sum planes need workspace");
    const size_t pe = sum_plane_bytes(n) / sizeof(double);
    double *pa = planes, *pb = planes + pe, *xb = planes + 2 * pe, *aa = planes + 3 * pe;
    f.pa1 = pa;
    f.pb1 = xb;
    f.pa2 = aa;
    f.pb2 = pb;
    const int kbt = (n + 15) / 16, cbt = (n + 63) / 64;
    k_sum_planes<<<dim3(kbt * cbt, gemm1_only ? 2 : 3), 256, 0, st>>>(n, p, x, n, pa, pb, xb, gemm1_only);
    ZT_LAUNCHED();
  }
  int dev;
  cudaGetDevice(&dev);
  const int slot = algo == ALGO_4M ? 1 : (algo == ALGO_3MS ? 2 : 0);
  if (dev < 16 && !g_fattr[dev][slot]) {
    if (algo == ALGO_4M)
      ZT_CUDA_CHECK(cudaFuncSetAttribute(k_zupdate<ALGO_4M>, cudaFuncAttributeMaxDynamicSharedMemorySize, GEMM_SMEM));
    else if (algo == ALGO_3MS)
      ZT_CUDA_CHECK(cudaFuncSetAttribute(k_zupdate<ALGO_3MS>, cudaFuncAttributeMaxDynamicSharedMemorySize, GEMM_SMEM_S));
    else
      ZT_CUDA_CHECK(cudaFuncSetAttribute(k_zupdate<ALGO_3M>, cudaFuncAttributeMaxDynamicSharedMemorySize, GEMM_SMEM));
    cudaDeviceGetAttribute(&g_sms[dev], cudaDevAttrMultiProcessorCount, dev);
    g_fattr[dev][slot] = true;
  }
  const int T = (n + BM - 1) / BM;
  const int total = T * T + T * (T + 1) / 2;
  const int grid = std::min(total, dev < 16 ? g_sms[dev] : 148);
  int S = 0, F = 1;
  f.gemm1_only = gemm1_only;
  // bbuf: GEMM-2 stores b there and the update runs as k_update_pairs after
  // the persistent kernel (X is then rewritten only once no tile reads it)
  const bool sep = bbuf && !gemm1_only;
  f.b_out = sep ? bbuf : nullptr;
  if (split && !gemm1_only) pick_split(total, grid, T * (T + 1) / 2, n, S, F);
  f.split_s = S;
  f.split_f = F;
  f.split_sem = sync + 1 + T;
  f.split_acc = split;
  ZT_CUDA_CHECK(cudaMemsetAsync(sync, 0, sizeof(unsigned int) * (T + 1 + S), st));
  if (prog && gemm1_only) {
    f.prog = 1;
    f.wn = prog->wn;
    f.wout = prog->wout;
    f.h = prog->h;
    f.pair_cnt = prog->words;
    f.rows_done = prog->words + T * (T + 1) / 2;
    f.row_flag = f.rows_done + T;
    ZT_CUDA_CHECK(cudaMemsetAsync(prog->words, 0, sizeof(unsigned int) * (T * (T + 1) / 2 + T), st));
  }
  if (algo == ALGO_4M)
    k_zupdate<ALGO_4M><<<grid, GEMM_THREADS, GEMM_SMEM, st>>>(f);
  else if (algo == ALGO_3MS)
    k_zupdate<ALGO_3MS><<<grid, GEMM_THREADS, GEMM_SMEM_S, st>>>(f);
  else
    k_zupdate<ALGO_3M><<<grid, GEMM_THREADS, GEMM_SMEM, st>>>(f);
  ZT_LAUNCHED();
  ZT_CUDA_CHECK(cudaGetLastError());
  if (sep) {
    const int t32 = (n + 31) / 32;
    const int nb = t32 * (t32 + 1) / 2;
    if (xprev && wn)
      k_update_pairs<true, true><<<nb, 256, 0, st>>>(n, a, bbuf, out, base, xprev, wn, hh, qq, resid, cons);
    else if (xprev)
      k_update_pairs<true, false><<<nb, 256, 0, st>>>(n, a, bbuf, out, base, xprev, wn, hh, qq, resid, cons);
    else if (wn)
      k_update_pairs<false, true><<<nb, 256, 0, st>>>(n, a, bbuf, out, base, xprev, wn, hh, qq, resid, cons);
    else
      k_update_pairs<false, false><<<nb, 256, 0, st>>>(n, a, bbuf, out, base, xprev, wn, hh, qq, resid, cons);
    ZT_LAUNCHED();
    ZT_CUDA_CHECK(cudaGetLastError());
  }
  return ZT_OK;
}

int skew_diff(int n, const double* a, double* c, cudaStream_t st) {
  dim3 grid((n + 31) / 32, (n + 31) / 32);
  k_skew_diff<<<grid, 256, 0, st>>>(n, a, c);
  ZT_LAUNCHED();
  ZT_CUDA_CHECK(cudaGetLastError());
  return ZT_OK;
}

}  // namespace zt
