// Stream solve P = lap^{-1} W, apply_laplacian and structure residuals for
// sm_100a.  Restates the per-diagonal LDL^T sweeps of the reference
// (laplacian.py:189-219 factor build, 272-300 sweeps, 306-316 reflection,
// 341-367 stencil) as HBM-bound, chunk-parallel kernels:
//
//  * sheared tiles: warp = 32 consecutive diagonals m x SR consecutive rows
//    i ("chunk"); lane m reads W[i][i-m], so each tile row is one contiguous
//    512 B segment (the reference's sheared layout, laplacian.py:16-21,
//    applied on the fly instead of materialised);
//  * LDL^T factors are regenerated in registers from the closed-form block
//    entries (a fast reciprocal + 2 Newton steps per row, within an ulp of
//    dpttrf) starting from the exact dpttrf pivot at each chunk start, so no
//    factor bytes are streamed from HBM;
//  * chunks couple affinely: pass 1 computes each chunk's zero-carry forward
//    end value and backward start value; pass 2 (one warp per diagonal,
//    warp-level affine scans) chains the carries with precomputed gains
//    G/H/K; pass 3 re-sweeps every chunk with its true carries and writes the
//    lower triangle coalesced and the skew reflection through a shared-memory
//    transpose;
//  * the singular m = 0 diagonal (deflated block, null-mode projection of the
//    RHS and zero-mean gauge, laplacian.py:201-215, 276-298) runs in the same
//    tiles: by linearity pass 1 records per-chunk trace partials and x-sums,
//    and pass 2 resolves mu = tr/N and the gauge from precomputed responses
//    to a constant right-hand side.
#include <math.h>
#include <stdio.h>

#include <algorithm>
#include <string>
#include <vector>

#include "zt_tma.cuh"

namespace zt {

#ifndef SOLVE_SUB
#define SOLVE_SUB 16
#endif
constexpr int SUB = SOLVE_SUB;  // rows per lane (sub-chunk)
constexpr int LPD = 64 / SUB;   // lanes per diagonal
constexpr int DPW = 32 / LPD;  // diagonals per warp tile
constexpr int SR = SUB * LPD;  // rows per chunk (carry granularity)
constexpr int SOLVE_WARPS = 4;
// pass 3's interior tiles regenerate the block entries from integer
// recurrences (as pass 1 does) instead of loading them per row
#ifndef SOLVE_P3REC
#define SOLVE_P3REC 1
#endif

// L2 residency between the passes: pass 1 reads W with evict_last so pass 3's
// re-read hits L2 when the batch runs one matrix (or diagonal group) at a time;
// pass 3 reads W for the last time (evict_first) and streams P out.
#ifndef SOLVE_L2HINT
#define SOLVE_L2HINT 1
#endif
__device__ __forceinline__ uint64_t pol_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t pol_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ double2 ld2_pol(const double* p, uint64_t pol) {
  double2 v;
  asm volatile("ld.global.nc.L2::cache_hint.v2.f64 {%0, %1}, [%2], %3;"
               : "=d"(v.x), "=d"(v.y) : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ void st2_pol(double* p, double2 v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.v2.f64 [%0], {%1, %2}, %3;" ::"l"(p), "d"(v.x), "d"(v.y), "l"(pol)
               : "memory");
}
constexpr int TR = 32;  // rows per apply tile / diagonals per apply tile
constexpr int M0X = 5;  // m = 0 per-chunk responses: Y1, X1, S1, SH, SK

// ---------------------------------------------------------------------------
// operator build (laplacian.py:197-215): one thread per diagonal walks the
// exact dpttrf recurrence once and records the pivot at every 16-row
// sub-chunk start, and per 64-row chunk the coupling into the chunk and the
// carry gains G (forward), H (backward), K (forward carry -> backward start).
// ---------------------------------------------------------------------------
__global__ void k_op_sqrt_table(int n, double* sqB, double* Bq) {
  int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j < n) {
    Bq[j] = (j + 1.0) * (n - 1.0 - j);
    sqB[j] = sqrt(Bq[j]);  // sqrt((i+1)(N-1-i)), laplacian.py:134-136
  }
}

__global__ void k_op_build(int n, int C, const double* __restrict__ sqB, double* d0s, double* lins,
                           double* lin, double* G, double* H, double* K, double* L0, double* dinv0,
                           double* m0x) {
  const int m = blockIdx.x * blockDim.x + threadIdx.x;
  if (m >= n) return;
  const int len = n - m;
  double d = block_diag(n, m, 0);
  double Lprev = 0.0;
  double Lc[SR], Dc[SR], g[SR], z[SR], hh[SR];
  double Lrow = 0.0;  // L of the previous row
  int k = 0;
  // m = 0 is deflated to its leading (N-1) block; row N-1 is the gauge row
  const int last = (m == 0) ? n - 2 : len - 1;  // last factored row
  while (k < len) {
    const int i = m + k;
    const int c = i / SR;
    const int k0 = k;
    const int cnt = min((c + 1) * SR, n) - i;
    const double lin_c = (k0 == 0) ? 0.0 : Lprev;
    lin[(size_t)c * n + m] = lin_c;
    for (int r = 0; r < cnt; ++r, ++k) {
      if ((m + k) % SUB == 0 || r == 0) {
        d0s[(size_t)((m + k) / SUB) * n + m] = d;
        lins[(size_t)((m + k) / SUB) * n + m] = Lrow;
      }
      if (k <= last) {
        Dc[r] = __drcp_rn(d);
        if (k < last) {
          const double e = __dmul_rn(-sqB[m + k], sqB[k]);
          const double L = __ddiv_rn(e, d);
          Lc[r] = L;
          d = __dsub_rn(block_diag(n, m, k + 1), __dmul_rn(L, e));
        } else {
          Lc[r] = 0.0;
        }
      } else {
        Dc[r] = 0.0;
        Lc[r] = 0.0;
      }
      Lrow = Lc[r];
      if (m == 0) {
        L0[k] = Lc[r];
        dinv0[k] = Dc[r];
      }
    }
    double gg = -lin_c;
    for (int r = 0; r < cnt; ++r) {
      if (r > 0) gg = -Lc[r - 1] * gg;
      g[r] = gg;
    }
    double zz = 0.0, hv = 1.0;
    for (int r = cnt - 1; r >= 0; --r) {
      zz = g[r] * Dc[r] - Lc[r] * zz;
      hv = -Lc[r] * hv;
      z[r] = zz;
      hh[r] = hv;
    }
    G[(size_t)c * n + m] = g[cnt - 1];
    H[(size_t)c * n + m] = hh[0];
    K[(size_t)c * n + m] = z[0];
    if (m == 0) {
      // responses to a constant right-hand side 1 with zero carries, and the
      // chunk sums of the x responses (for the zero-mean gauge)
      double yy = 0.0;
      for (int r = 0; r < cnt; ++r) {
        yy = (r == 0) ? 1.0 : 1.0 - Lc[r - 1] * yy;
        g[r] = yy;  // reuse as y1
      }
      double x1 = 0.0, s1 = 0.0, sh = 0.0, sk = 0.0;
      for (int r = cnt - 1; r >= 0; --r) {
        x1 = g[r] * Dc[r] - Lc[r] * x1;
        s1 += x1;
        sh += hh[r];
        sk += z[r];
      }
      double* q = m0x + (size_t)c * M0X;
      q[0] = g[cnt - 1];
      q[1] = x1;
      q[2] = s1;
      q[3] = sh;
      q[4] = sk;
    }
    Lprev = Lc[cnt - 1];
  }
}

// Fast pivot reciprocal: approximate rcp + 2 Newton steps (d > 0, well
// scaled: 1 <= d <= 2e8 for N <= 16384), within ~1 ulp of 1/d.
__device__ __forceinline__ double fast_rcp(double d) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(d));
  double e = fma(-d, r, 1.0);
  r = fma(r, e, r);
  e = fma(-d, r, 1.0);
  return fma(r, e, r);
}

// sqrt of an exact integer-valued double (< 2^53): rsqrt seed, one Goldschmidt
// step and a residual correction (~1 ulp).  Used for the block off-diagonal
// e = -sqrt(B(i) B(k)) so the interior tiles read no factor tables per row.
__device__ __forceinline__ double fast_sqrt(double x) {
  double r;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  double y = x * r, h = 0.5 * r;
  const double t = fma(-y, h, 0.5);
  y = fma(y, t, y);
  h = fma(h, t, h);
  return fma(fma(-y, y, x), h, y);
}

// ---------------------------------------------------------------------------
// chunk tiles: warp = 8 diagonals x 64 rows; lane (d = lane & 7,
// s = lane >> 3) owns rows [16 s, 16 s + 16) of diagonal m0 + d.
// FINAL=false: pass 1 (chunk aggregates).  FINAL=true: pass 3 (writes P).
// ---------------------------------------------------------------------------
struct SolveArgs {
  int n, C, ntiles;
  const double* sqB;
  const double* Bq;  // (j+1)(N-1-j), exact
  const double* d0s;
  const double* lins;
  const double* lin;
  const double* L0;
  const double* dinv0;
  const double* w;
  int64_t ldw, sw;
  double* p;
  int64_t ldp, sp;
  double2* yend;   // [batch][C][n]: pass1 y_end -> pass2 y_in
  double2* xst;    // [batch][C][n]: pass1 x_start -> pass2 x_in
  double2* m0acc;  // [batch][C][2]: (trace partial, x-sum) of the m = 0 chunk
  double2* m0mg;   // [batch][2]: (mu, gauge)
};

struct AffW {  // y_out = a + g * y_in
  double2 a;
  double g;
};
__device__ __forceinline__ AffW aff_compose(AffW first, AffW second) {
  // apply `first`, then `second`
  AffW r;
  r.a = make_double2(fma(second.g, first.a.x, second.a.x), fma(second.g, first.a.y, second.a.y));
  r.g = second.g * first.g;
  return r;
}
__device__ __forceinline__ AffW aff_shfl(AffW v, int src) {
  AffW o;
  o.a.x = __shfl_sync(0xffffffff, v.a.x, src);
  o.a.y = __shfl_sync(0xffffffff, v.a.y, src);
  o.g = __shfl_sync(0xffffffff, v.g, src);
  return o;
}

// tile t -> (chunk c, group g of 8 diagonals): chunk c holds 8(c+1) groups
__device__ __forceinline__ void solve_tile_coords(int t, int& c, int& g) {
  int q = (int)((sqrt(1.0 + (double)t) - 1.0) * 0.5);
  while (4 * (q + 1) * (q + 2) <= t) ++q;
  while (4 * q * (q + 1) > t) --q;
  c = q;
  g = t - 4 * q * (q + 1);
}

static int solve_ntiles(int C) { return 4 * C * (C + 1); }

// Per-lane body.  FAST: every lane owns 16 interior rows of its diagonal
// (k >= 1 at the first row, the diagonal's last row not inside, m != 0), so
// all boundary predicates vanish and addresses advance by a constant stride.
template <bool FINAL, bool FAST, bool LAST = false>
__device__ __forceinline__ void tile_body(const SolveArgs& A, const double* __restrict__ w,
                                          double* __restrict__ p, int b, int c, int m0, int lane,
                                          double2* sm) {
  const int n = A.n;
  const int i0 = c * SR;
  const int dl = lane % DPW, s = lane / DPW;
  const int m = m0 + dl;
  const int ib = i0 + s * SUB;
  const bool mok = m < n;
  const int len = n - m;
  const int rs = FAST ? 0 : max(0, m - ib);
  const int re = FAST ? SUB - 1 : min(SUB - 1, n - 1 - ib);
  const bool has = FAST || (mok && rs <= re);
  // FAST tiles may end exactly at row N-1 (N % 64 == 0): that row is every
  // diagonal's last element (no coupling below it)
  const bool lastrow = FAST && LAST && (ib + SUB - 1 == n - 1);
  const size_t cm = (size_t)b * A.C * n + (size_t)c * n + m;
  const int64_t wstride = (A.ldw + 1) * 2;  // doubles between W[i][i-m] and W[i+1][i+1-m]
  const double* wp = w + ((int64_t)ib * A.ldw + (ib - m)) * 2;
#define ROW_OK(r) (FAST || ((r) >= rs && (r) <= re))

  // 1. loads (16 rows; each instruction covers 4 rows x 128 B)
  double2 v[SUB];
#pragma unroll
#if SOLVE_L2HINT
  const uint64_t wpol = FINAL ? pol_first() : pol_last();
  const uint64_t ppol = pol_first();
  for (int r = 0; r < SUB; ++r) v[r] = (has && ROW_OK(r)) ? ld2_pol(wp + r * wstride, wpol) : make_double2(0.0, 0.0);
#define PST(ptr, val) st2_pol(ptr, val, ppol)
#else
  for (int r = 0; r < SUB; ++r) v[r] = (has && ROW_OK(r)) ? ld2(wp + r * wstride) : make_double2(0.0, 0.0);
#define PST(ptr, val) st2(ptr, val)
#endif
  const double2 ych = (FINAL && mok) ? __ldcg(A.yend + cm) : make_double2(0.0, 0.0);
  const double2 xch = (FINAL && mok) ? __ldcg(A.xst + cm) : make_double2(0.0, 0.0);

  // 2. factor chain from the exact sub-chunk pivot (dpttrf order, fast rcp)
  if (has) {
    if (!FAST && m == 0) {
#pragma unroll
      for (int r = 0; r < SUB; ++r)
        if (r <= re) sm[(s * SUB + r) * DPW + dl] = make_double2(A.L0[ib + r], A.dinv0[ib + r]);
    } else if (FAST && SOLVE_P3REC) {
      // interior tiles: pass 1's register form of the chain (agg_body) --
      // e^2 = B(i) B(k) from exact integer recurrences and e = -sqrt(e^2),
      // no per-row table loads (pass 3 was L1-bound on 4 loads per row)
      const int k = ib - m;
      double qm1 = 1.0, q0 = __ldg(A.d0s + (size_t)(ib / SUB) * n + m);
      double dg = block_diag(n, m, k);
      double inc = 2.0 * (double)(n - 2 - 2 * k - m);
      double bi = (ib + 1.0) * (double)(n - 1 - ib), dbi = (double)(n - 3 - 2 * ib);
      double bk = (k + 1.0) * (double)(n - 1 - k), dbk = (double)(n - 3 - 2 * k);
#pragma unroll
      for (int r = 0; r < SUB; ++r) {
        const double di = qm1 * fast_rcp(q0);
        double L = 0.0;
        if (!(lastrow && r == SUB - 1)) {
          const double e2 = bi * bk;
          L = -fast_sqrt(e2) * di;
          dg += inc;
          inc -= 4.0;
          const double q1 = fma(dg, q0, -e2 * qm1);
          qm1 = q0;
          q0 = q1;
          bi += dbi;
          dbi -= 2.0;
          bk += dbk;
          dbk -= 2.0;
        }
        sm[(s * SUB + r) * DPW + dl] = make_double2(L, di);
      }
    } else {
      // Leading-minor form of the pivot recurrence: with q_{-1} = 1 and
      // q_0 = d(k0) (exact dpttrf pivot), q_j = diag q_{j-1} - e^2 q_{j-2}
      // gives d(k0+j) = q_j / q_{j-1}; e^2 = B(i) B(k) is exact
      // (B(j) = (j+1)(N-1-j)), so the loop-carried chain is one FMA per row
      // and the reciprocals are off the chain.  |q| <= d_max^16 < 1e150.
      int k = ib + rs - m;
      double qm1 = 1.0, q0 = __ldg(A.d0s + (size_t)(ib / SUB) * n + m);
      double dg = block_diag(n, m, k);
      double inc = 2.0 * (double)(n - 2 - 2 * k - m);  // diag(k+1) - diag(k), exact
      const double* sqi = A.sqB + ib + rs;
      const double* sqk = A.sqB + k;
      const double* bqi = A.Bq + ib + rs;
      const double* bqk = A.Bq + k;
#pragma unroll
      for (int r = 0; r < SUB; ++r) {
        if (ROW_OK(r)) {
          const int rr = r - rs;
          const double rq = fast_rcp(q0);
          const double di = qm1 * rq;  // 1 / d_k
          double L = 0.0;
          if (FAST ? !(lastrow && r == SUB - 1) : (k + rr < len - 1)) {
            const double e = -__ldg(sqi + rr) * __ldg(sqk + rr);
            L = e * di;
            const double e2 = __ldg(bqi + rr) * __ldg(bqk + rr);
            dg += inc;
            inc -= 4.0;
            const double q1 = fma(dg, q0, -e2 * qm1);
            qm1 = q0;
            q0 = q1;
          }
          sm[(s * SUB + r) * DPW + dl] = make_double2(L, di);
        }
      }
    }
  }
  __syncwarp();
  // coupling into my first row: previous chunk (table) or my s-1 neighbour
  double Lin = 0.0;
  if (has) Lin = (s == 0) ? __ldg(A.lin + (size_t)c * n + m) : sm[(s * SUB - 1) * DPW + dl].x;

  double2 mu = make_double2(0.0, 0.0), gauge = make_double2(0.0, 0.0);
  if (!FAST && FINAL && m == 0) {
    mu = __ldcg(A.m0mg + 2 * b);
    gauge = __ldcg(A.m0mg + 2 * b + 1);
  }
  // 3. forward sweep with zero carry (laplacian.py:280-287) -> affine map
  double2 tb = make_double2(0.0, 0.0);
  AffW fm;
  fm.a = make_double2(0.0, 0.0);
  fm.g = 1.0;
  if (has) {
    double Lp = Lin;
#pragma unroll
    for (int r = 0; r < SUB; ++r) {
      if (ROW_OK(r)) {
        double2 bb = v[r];
        if (!FAST && !FINAL && m == 0) tb = make_double2(tb.x + bb.x, tb.y + bb.y);
        if (!FAST && FINAL && m == 0) bb = csub(bb, mu);
        if (!FAST && ib + r - m == 0) {
          fm.a = bb;
          fm.g = 0.0;
        } else {
          fm.a = make_double2(fma(-Lp, fm.a.x, bb.x), fma(-Lp, fm.a.y, bb.y));
          fm.g = -Lp * fm.g;
        }
        Lp = sm[(s * SUB + r) * DPW + dl].x;
        v[r] = fm.a;
      }
    }
  }
  // 4. compose the 4 segment maps of each diagonal (lanes dl, dl+8, dl+16, dl+24)
  AffW inc = fm;
#pragma unroll
  for (int step = 1; step < LPD; step <<= 1) {
    AffW o = aff_shfl(inc, max(lane - step * DPW, 0));
    if (s >= step) inc = aff_compose(o, inc);
  }
  AffW exm = aff_shfl(inc, max(lane - DPW, 0));
  if (s == 0) {
    exm.a = make_double2(0.0, 0.0);
    exm.g = 1.0;
  }
  const double2 yin = make_double2(fma(exm.g, ych.x, exm.a.x), fma(exm.g, ych.y, exm.a.y));
  if (!FINAL && s == LPD - 1 && mok) A.yend[cm] = inc.a;  // chunk forward aggregate (zero carry)
  // 5. forward fix-up: y(r) += g(r) y_in, g(r) = prod(-L) from the segment start
  if (has) {
    double gg = 1.0, Lp = Lin;
#pragma unroll
    for (int r = 0; r < SUB; ++r) {
      if (ROW_OK(r)) {
        gg = (!FAST && ib + r - m == 0) ? 0.0 : -Lp * gg;
        v[r] = make_double2(fma(gg, yin.x, v[r].x), fma(gg, yin.y, v[r].y));
        Lp = sm[(s * SUB + r) * DPW + dl].x;
      }
    }
  }
  // 6. backward sweep with zero carry (laplacian.py:288-292)
  AffW bm;
  bm.a = make_double2(0.0, 0.0);
  bm.g = 1.0;
  if (has) {
#pragma unroll
    for (int r = SUB - 1; r >= 0; --r) {
      if (ROW_OK(r)) {
        const double2 f = sm[(s * SUB + r) * DPW + dl];
        if (FAST ? (lastrow && r == SUB - 1) : (ib + r - m == len - 1)) {
          bm.a = make_double2(f.y * v[r].x, f.y * v[r].y);
          bm.g = 0.0;
        } else {
          bm.a = make_double2(fma(-f.x, bm.a.x, f.y * v[r].x), fma(-f.x, bm.a.y, f.y * v[r].y));
          bm.g = -f.x * bm.g;
        }
        v[r] = bm.a;
      }
    }
  }
  // 7. reverse composition over segments: x_in(s) = x_start(s+1)
  AffW rinc = bm;
#pragma unroll
  for (int step = 1; step < LPD; step <<= 1) {
    AffW o = aff_shfl(rinc, min(lane + step * DPW, 31));
    if (s + step <= LPD - 1) rinc = aff_compose(o, rinc);
  }
  AffW rex = aff_shfl(rinc, min(lane + DPW, 31));
  if (s == LPD - 1) {
    rex.a = make_double2(0.0, 0.0);
    rex.g = 1.0;
  }
  const double2 xin = make_double2(fma(rex.g, xch.x, rex.a.x), fma(rex.g, xch.y, rex.a.y));
  if (!FINAL) {
    if (s == 0 && mok) A.xst[cm] = rinc.a;  // chunk backward aggregate (zero carries)
    if (!FAST && m0 == 0) {
      // chunk sums for the m = 0 null-mode projection and gauge (lanes dl == 0)
      double2 xs = make_double2(0.0, 0.0);
      if (has && m == 0) {
        double hh = 1.0;
#pragma unroll
        for (int r = SUB - 1; r >= 0; --r) {
          if (r >= rs && r <= re) {
            hh = (ib + r - m == len - 1) ? 0.0 : -sm[(s * SUB + r) * DPW + dl].x * hh;
            xs = make_double2(xs.x + fma(hh, xin.x, v[r].x), xs.y + fma(hh, xin.y, v[r].y));
          }
        }
      }
#pragma unroll
      for (int off = DPW; off < 32; off <<= 1) {
        tb.x += __shfl_xor_sync(0xffffffff, tb.x, off);
        tb.y += __shfl_xor_sync(0xffffffff, tb.y, off);
        xs.x += __shfl_xor_sync(0xffffffff, xs.x, off);
        xs.y += __shfl_xor_sync(0xffffffff, xs.y, off);
      }
      if (lane == 0) {
        A.m0acc[((size_t)b * A.C + c) * 2] = tb;
        A.m0acc[((size_t)b * A.C + c) * 2 + 1] = xs;
      }
    }
    return;
  }
  // 8. backward fix-up and output
  const int64_t pstride = (A.ldp + 1) * 2;
  double* pp = p + ((int64_t)ib * A.ldp + (ib - m)) * 2;
  if (has) {
    double hh = 1.0;
#pragma unroll
    for (int r = SUB - 1; r >= 0; --r) {
      if (ROW_OK(r)) {
        hh = (FAST ? (lastrow && r == SUB - 1) : (ib + r - m == len - 1)) ? 0.0
                                                                             : -sm[(s * SUB + r) * DPW + dl].x * hh;
        const double2 x = make_double2(fma(hh, xin.x, v[r].x), fma(hh, xin.y, v[r].y));
        if (!FAST && m == 0) {
          // zero-mean gauge (laplacian.py:293-298): P[i][i] = -(x - g)
          PST(pp + r * pstride, make_double2(-(x.x - gauge.x), -(x.y - gauge.y)));
        } else {
          // lower triangle: P[i][i-m] = -x (laplacian.py:299-300)
          PST(pp + r * pstride, make_double2(-x.x, -x.y));
        }
        v[r] = x;
      }
    }
  }
#undef ROW_OK
  __syncwarp();
  // stage x for the transposed store (reuse the factor tile)
  double2* xs_buf = sm;
#pragma unroll
  for (int r = 0; r < SUB; ++r) xs_buf[(s * SUB + r) * DPW + dl] = v[r];
  __syncwarp();
  // strict upper by skew reflection: P[i-m][i] = conj(x) (laplacian.py:306-316).
  // Output row j = i0 - m0 + t holds columns i0 + t + u, u = 0..7 (one 128 B
  // run); each instruction writes 4 such rows.
  const int u = lane % DPW;
  const int mm = m0 + u;
  const bool uok = mm >= 1 && mm < n;
  for (int t0 = -(DPW - 1); t0 < SR; t0 += 32 / DPW) {
    const int tt = t0 + lane / DPW;
    const int r = tt + u;  // row in chunk of diagonal m0 + u
    const int i = i0 + r;
    if (uok && tt < SR && r >= 0 && r < SR && i >= mm && i < n) {
      const double2 xv = xs_buf[r * DPW + u];
      PST(p + ((size_t)(i - mm) * A.ldp + i) * 2, make_double2(xv.x, -xv.y));
    }
  }
#undef PST
}



// Pass-1 body of the interior tiles: one ascending loop runs the factor
// chain, the zero-carry forward sweep and (by linearity) the zero-carry
// backward start, so nothing is stored per row; the block entries come from
// exact integer recurrences (B(j+1) = B(j) + N - 3 - 2j) and fast_sqrt
// instead of table loads.  The shared-memory form was L1-bound here (ncu:
// L1/TEX 93% busy at 47% of DRAM on per-row table loads and factor round
// trips).
__device__ __forceinline__ void agg_body(const SolveArgs& A, const double* __restrict__ w, int b, int c,
                                         int m0, int lane) {
  const int n = A.n;
  const int i0 = c * SR;
  const int dl = lane % DPW, s = lane / DPW;
  const int m = m0 + dl;
  const int ib = i0 + s * SUB;
  const int k0 = ib - m;  // >= 1 on interior tiles
  const size_t cm = (size_t)b * A.C * n + (size_t)c * n + m;
  const int64_t wstride = (A.ldw + 1) * 2;
  const double* wp = w + ((int64_t)ib * A.ldw + k0) * 2;

  double2 v[SUB];
#pragma unroll
#if SOLVE_L2HINT
  const uint64_t wpol = pol_last();
  for (int r = 0; r < SUB; ++r) v[r] = ld2_pol(wp + r * wstride, wpol);
#else
  for (int r = 0; r < SUB; ++r) v[r] = ld2(wp + r * wstride);
#endif

  const size_t sub = (size_t)(ib / SUB) * n + m;
  double qm1 = 1.0, q0 = __ldg(A.d0s + sub);
  const double Lin = __ldg(A.lins + sub);
  double dg = block_diag(n, m, k0);
  double inc = 2.0 * (double)(n - 2 - 2 * k0 - m);
  double bi = (ib + 1.0) * (double)(n - 1 - ib), dbi = (double)(n - 3 - 2 * ib);
  double bk = (k0 + 1.0) * (double)(n - 1 - k0), dbk = (double)(n - 3 - 2 * k0);
  // factor chain fused with the zero-carry forward sweep (laplacian.py:280-287);
  // the segment's zero-carry backward start is accumulated on the way up:
  // x(0) = sum_r P_r D_r y(r) + P_SUB x_in with P_r = prod_{j<r} (-L_j), and
  // its response to the segment's incoming y is ks = sum_r P_r D_r g(r)
  AffW fm;
  fm.a = make_double2(0.0, 0.0);
  fm.g = 1.0;
  double2 bl = make_double2(0.0, 0.0);
  double ks = 0.0, P = 1.0;
  double Lp = Lin;
#pragma unroll
  for (int r = 0; r < SUB; ++r) {
    const double di = qm1 * fast_rcp(q0);
    const double e2 = bi * bk;
    const double L = -fast_sqrt(e2) * di;
    dg += inc;
    inc -= 4.0;
    const double q1 = fma(dg, q0, -e2 * qm1);
    qm1 = q0;
    q0 = q1;
    bi += dbi;
    dbi -= 2.0;
    bk += dbk;
    dbk -= 2.0;
    fm.a = make_double2(fma(-Lp, fm.a.x, v[r].x), fma(-Lp, fm.a.y, v[r].y));
    fm.g = -Lp * fm.g;
    const double cf = P * di;
    bl = make_double2(fma(cf, fm.a.x, bl.x), fma(cf, fm.a.y, bl.y));
    ks = fma(cf, fm.g, ks);
    P = -L * P;
    Lp = L;
  }
  AffW incf = fm;
#pragma unroll
  for (int step = 1; step < LPD; step <<= 1) {
    AffW o = aff_shfl(incf, max(lane - step * DPW, 0));
    if (s >= step) incf = aff_compose(o, incf);
  }
  AffW exm = aff_shfl(incf, max(lane - DPW, 0));
  if (s == 0) {
    exm.a = make_double2(0.0, 0.0);
    exm.g = 1.0;
  }
  // segment backward map with zero chunk carries: a = Back(y_loc + g exm.a)(0)
  AffW bm;
  bm.a = make_double2(fma(ks, exm.a.x, bl.x), fma(ks, exm.a.y, bl.y));
  bm.g = P;
#pragma unroll
  for (int step = 1; step < LPD; step <<= 1) {
    AffW o = aff_shfl(bm, min(lane + step * DPW, 31));
    if (s + step <= LPD - 1) bm = aff_compose(o, bm);
  }
  if (s == LPD - 1) A.yend[cm] = incf.a;  // chunk forward aggregate (zero carry)
  if (s == 0) A.xst[cm] = bm.a;           // chunk backward aggregate (zero carries)
}

// Interior tiles: chunks c < Cf (the chunk ends before row n-2), groups
// g = 1 .. GPC*c-1 with GPC = SR/DPW groups per chunk height (all DPW
// diagonals start before the chunk).  Count per chunk GPC*c-1, prefix
// P(c) = GPC*c(c-1)/2 - (c-1) for c >= 1.
constexpr int GPC = SR / DPW;
__host__ __device__ __forceinline__ long long fast_prefix(long long c) {
  return c >= 1 ? (long long)GPC * c * (c - 1) / 2 - (c - 1) : 0;
}
__device__ __forceinline__ void fast_tile_coords(int t, int& c, int& g) {
  int q = (int)(sqrt(2.0 * (double)t / GPC)) + 1;
  while (q > 1 && fast_prefix(q) > t) --q;
  while (fast_prefix(q + 1) <= t) ++q;
  c = q;
  g = 1 + (int)(t - fast_prefix(q));
}

static int fast_chunks(int n) {

  int cf = 0;
  while ((cf + 1) * SR < n - 1) ++cf;
  return cf;
}
static int fast_ntiles(int cf) { return (int)fast_prefix(cf); }

// One launch for a whole tile pass: blocks [0, gblocks) take the boundary
// tiles (dispatched first, so their latency hides under the interior tiles
// that follow), the rest the interior tiles.
#ifndef SOLVE_MINB_AGG
#define SOLVE_MINB_AGG 4
#endif
#ifndef SOLVE_MINB_FIN
#define SOLVE_MINB_FIN 3
#endif
template <bool FINAL>
__global__ void __launch_bounds__(SOLVE_WARPS * 32, FINAL ? SOLVE_MINB_FIN : SOLVE_MINB_AGG)
    k_solve_merged(SolveArgs A, const int2* __restrict__ tiles, int count, int gblocks) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int b = blockIdx.y;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double2* sm = reinterpret_cast<double2*>(smem_raw) + warp * SR * DPW;
  pdl_wait();  // W from the previous kernel (update pass) / the carries
  const double* w = A.w + (size_t)b * A.sw * 2;
  double* p = A.p + (size_t)b * A.sp * 2;
  if ((int)blockIdx.x < gblocks) {
    const int t = blockIdx.x * SOLVE_WARPS + warp;
    if (t >= count) return;
    const int2 cg = tiles[t];
    const int c = cg.x & ~(1 << 30);
    if (cg.x & (1 << 30))
      tile_body<FINAL, true, true>(A, w, p, b, c, cg.y * DPW, lane, sm);
    else
      tile_body<FINAL, false>(A, w, p, b, c, cg.y * DPW, lane, sm);
  } else {
    const int t = (blockIdx.x - gblocks) * SOLVE_WARPS + warp;
    if (t >= A.ntiles) return;
    int c, g;
    fast_tile_coords(t, c, g);
    // pass 1: register body (no factor tables, no shared memory); pass 3:
    // shared-memory factors (the register form needs > 168 registers there)
    if (!FINAL)
      agg_body(A, w, b, c, g * DPW, lane);
    else
      tile_body<true, true>(A, w, p, b, c, g * DPW, lane, sm);
  }
}

// ---------------------------------------------------------------------------
// pass 2: chain the chunk carries.  Block = 32 diagonals (lanes) x 8 chunk
// segments (warps); loads are coalesced across diagonals; the segment maps
// are composed through shared memory.
// ---------------------------------------------------------------------------
// Block = 32 diagonals (lanes) x SEG chunk segments (warps, SEG = 8..32);
// each thread caches its <= CE chunks' values in registers so every phase
// costs one memory round trip.
constexpr int CE = 8;

template <int MAXT>
__global__ void __launch_bounds__(MAXT) k_solve_carry(int n, int C, const double* __restrict__ G,
                                                      const double* __restrict__ H,
                                                      const double* __restrict__ K,
                                                      const double* __restrict__ m0x, double2* yend,
                                                      double2* xst, const double2* __restrict__ m0acc,
                                                      double2* m0mg) {
  __shared__ AffW agg[32][32];
  __shared__ double2 red[32];
  pdl_wait();  // the pass-1 aggregates
  const int SEG = blockDim.x >> 5;
  const int lane = threadIdx.x & 31, wseg = threadIdx.x >> 5;
  const int m = blockIdx.x * 32 + lane;
  const int b = blockIdx.y;
  const size_t base = (size_t)b * C * n;
  const bool ok = m < n;
  const int cs = (blockIdx.x * 32) / SR;  // first chunk holding any of the 32 diagonals
  const int nc = C - cs;
  const int E = (nc + SEG - 1) / SEG;  // <= CE (host picks SEG)
  const int cb = cs + wseg * E, ce = min(cb + E, C);
  const bool is0 = (m == 0);
  // m = 0: mu = tr W / N from the chunk trace partials (laplacian.py:276-279)
  double2 mu = make_double2(0.0, 0.0);
  if (blockIdx.x == 0) {
    double2 tr = make_double2(0.0, 0.0);
    if (lane == 0)
      for (int c = cb; c < ce; ++c) {
        const double2 q = m0acc[((size_t)b * C + c) * 2];
        tr = make_double2(tr.x + q.x, tr.y + q.y);
      }
    if (lane == 0) red[wseg] = tr;
    __syncthreads();
    double2 t = make_double2(0.0, 0.0);
    for (int q = 0; q < SEG; ++q) t = make_double2(t.x + red[q].x, t.y + red[q].y);
    mu = make_double2(t.x / n, t.y / n);
    __syncthreads();
  }
  // ---- forward: y_end(c) = a(c) + G(c) y_end(c-1) ----
  double2 av[CE];
  double gv[CE];
#pragma unroll
  for (int q = 0; q < CE; ++q) {
    const int c = cb + q;
    if (ok && c < ce) {
      const size_t o = (size_t)c * n + m;
      av[q] = yend[base + o];
      gv[q] = G[o];
      if (is0) av[q] = make_double2(av[q].x - mu.x * m0x[c * M0X + 0], av[q].y - mu.y * m0x[c * M0X + 0]);
    } else {
      av[q] = make_double2(0.0, 0.0);
      gv[q] = 1.0;
    }
  }
  AffW f;
  f.a = make_double2(0.0, 0.0);
  f.g = 1.0;
#pragma unroll
  for (int q = 0; q < CE; ++q) {
    f.a = make_double2(fma(gv[q], f.a.x, av[q].x), fma(gv[q], f.a.y, av[q].y));
    f.g *= gv[q];
  }
  agg[wseg][lane] = f;
  __syncthreads();
  AffW pre;
  pre.a = make_double2(0.0, 0.0);
  pre.g = 1.0;
  for (int q = 0; q < wseg; ++q) pre = aff_compose(pre, agg[q][lane]);
  double2 yin[CE];
  {
    double2 y = pre.a;
#pragma unroll
    for (int q = 0; q < CE; ++q) {
      yin[q] = y;
      y = make_double2(fma(gv[q], y.x, av[q].x), fma(gv[q], y.y, av[q].y));
      const int c = cb + q;
      if (ok && c < ce) yend[base + (size_t)c * n + m] = yin[q];  // y_in(c)
    }
  }
  __syncthreads();
  // ---- backward: x_start(c) = (xst(c) + K y_in(c)) + H x_start(c+1) ----
  double hv[CE];
#pragma unroll
  for (int q = 0; q < CE; ++q) {
    const int c = cb + q;
    if (ok && c < ce) {
      const size_t o = (size_t)c * n + m;
      av[q] = xst[base + o];
      if (is0) av[q] = make_double2(av[q].x - mu.x * m0x[c * M0X + 1], av[q].y - mu.y * m0x[c * M0X + 1]);
      const double kk = K[o];
      hv[q] = H[o];
      av[q] = make_double2(fma(kk, yin[q].x, av[q].x), fma(kk, yin[q].y, av[q].y));
    } else {
      av[q] = make_double2(0.0, 0.0);
      hv[q] = 1.0;
    }
  }
  AffW bk;
  bk.a = make_double2(0.0, 0.0);
  bk.g = 1.0;
#pragma unroll
  for (int q = CE - 1; q >= 0; --q) {
    bk.a = make_double2(fma(hv[q], bk.a.x, av[q].x), fma(hv[q], bk.a.y, av[q].y));
    bk.g *= hv[q];
  }
  agg[wseg][lane] = bk;
  __syncthreads();
  AffW suf;
  suf.a = make_double2(0.0, 0.0);
  suf.g = 1.0;
  for (int q = SEG - 1; q > wseg; --q) suf = aff_compose(suf, agg[q][lane]);
  double2 x = suf.a;
  double2 gs = make_double2(0.0, 0.0);
#pragma unroll
  for (int q = CE - 1; q >= 0; --q) {
    const int c = cb + q;
    if (ok && c < ce) {
      xst[base + (size_t)c * n + m] = x;  // x_in(c)
      if (is0) {
        // chunk x-sum = (sum x^ - mu S1) + SH x_in + SK y_in  (zero-mean gauge)
        const double2 sx = m0acc[((size_t)b * C + c) * 2 + 1];
        const double* qq = m0x + (size_t)c * M0X;
        gs.x += (sx.x - mu.x * qq[2]) + qq[3] * x.x + qq[4] * yin[q].x;
        gs.y += (sx.y - mu.y * qq[2]) + qq[3] * x.y + qq[4] * yin[q].y;
      }
    }
    x = make_double2(fma(hv[q], x.x, av[q].x), fma(hv[q], x.y, av[q].y));
  }
  if (blockIdx.x == 0) {
    __syncthreads();
    if (lane == 0) red[wseg] = gs;
    __syncthreads();
    if (threadIdx.x == 0) {
      double2 t = make_double2(0.0, 0.0);
      for (int q = 0; q < SEG; ++q) t = make_double2(t.x + red[q].x, t.y + red[q].y);
      m0mg[2 * b] = mu;
      m0mg[2 * b + 1] = make_double2(t.x / n, t.y / n);  // laplacian.py:293-296
    }
  }
}

__device__ __forceinline__ void tile_coords(int t, int& c, int& g) {
  c = (int)((sqrt(8.0 * t + 1.0) - 1.0) * 0.5);
  while ((c + 1) * (c + 2) / 2 <= t) ++c;
  while (c * (c + 1) / 2 > t) --c;
  g = t - c * (c + 1) / 2;
}

// ---------------------------------------------------------------------------
// apply_laplacian: y_i = (diag*s_i + off_{k-1}*s_{i-1}) + off_k*s_{i+1}
// in the reference's exact order (laplacian.py:358-367).
// ---------------------------------------------------------------------------
struct ApplyArgs {
  int n, C, ntiles, sign;
  const double* sqB;
  const double* w;
  int64_t ldw, sw;
  double* y;
  int64_t ldy, sy;
};

__global__ void __launch_bounds__(SOLVE_WARPS * 32) k_apply_tiles(ApplyArgs A) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int b = blockIdx.y;
  const double* w = A.w + (size_t)b * A.sw * 2;
  double* out = A.y + (size_t)b * A.sy * 2;
  const int n = A.n;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int t = blockIdx.x * SOLVE_WARPS + warp;
  if (t >= A.ntiles) return;
  int c, g;
  tile_coords(t, c, g);
  const int i0 = c * TR, m0 = g * TR, m = m0 + lane;
  double2* sm = reinterpret_cast<double2*>(smem_raw) + warp * TR * 32;
  const bool lane_ok = (m < n) && (m <= i0 + TR - 1);
  const int r0 = max(0, m - i0);
  const int rl = min(TR - 1, n - 1 - i0);
  const double sgn = (double)A.sign;
  double2 s[TR + 2];  // rows i0-1 .. i0+TR
#pragma unroll
  for (int q = 0; q < TR + 2; ++q) {
    const int i = i0 - 1 + q;
    s[q] = (lane_ok && i >= m && i < n) ? ld2(w + ((size_t)i * A.ldw + (i - m)) * 2)
                                        : make_double2(0.0, 0.0);
  }
#pragma unroll
  for (int r = 0; r < TR; ++r) {
    double2 res = make_double2(0.0, 0.0);
    if (lane_ok && r >= r0 && r <= rl) {
      const int i = i0 + r;
      const int k = i - m;
      double2 yy = rmul(block_diag(n, m, k), s[r + 1]);
      if (i >= 1) {  // y[1:] += off[:-1] * S[:-1]   (zero padding above the diagonal start)
        const double offp = (k >= 1) ? __dmul_rn(-A.sqB[i - 1], A.sqB[k - 1]) : 0.0;
        yy = cadd(yy, rmul(offp, s[r]));
      }
      if (i <= n - 2) {  // y[:-1] += off[:-1] * S[1:]
        const double off = __dmul_rn(-A.sqB[i], A.sqB[k]);
        yy = cadd(yy, rmul(off, s[r + 2]));
      }
      res = make_double2(yy.x * sgn, yy.y * sgn);
      st2(out + ((size_t)i * A.ldy + (i - m)) * 2, res);
    }
    sm[r * 32 + lane] = res;
  }
  // reflection of the strict upper triangle: out[i-m][i] = -conj(out[i][i-m])
#pragma unroll 4
  for (int tt = -(TR - 1); tt <= TR - 1; ++tt) {
    const int r = tt + lane;
    if (lane_ok && m >= 1 && r >= r0 && r <= rl && r >= 0 && r < TR) {
      const double2 xv = sm[r * 32 + lane];
      const int j = i0 - m0 + tt;
      st2(out + ((size_t)j * A.ldy + (i0 + r)) * 2, make_double2(-xv.x, xv.y));
    }
  }
}

// ---------------------------------------------------------------------------
// skewness / trace residuals (laplacian.py:75-104): lower tile pairs
// ---------------------------------------------------------------------------
constexpr int RT = 32;
__global__ void __launch_bounds__(256) k_resid_partial(int n, const double* __restrict__ w,
                                                        int64_t ldw, int nt, double* partial) {
  __shared__ double2 ta[RT][RT + 1];
  __shared__ double2 tb[RT][RT + 1];
  __shared__ double red[8][4];
  int I, J;
  tile_coords(blockIdx.x, I, J);
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  for (int r = ty; r < RT; r += 8) {
    const int i = I * RT + r, j = J * RT + tx;
    ta[r][tx] = (i < n && j < n) ? ld2(w + ((size_t)i * ldw + j) * 2) : make_double2(0.0, 0.0);
    const int i2 = J * RT + r, j2 = I * RT + tx;
    tb[r][tx] = (i2 < n && j2 < n) ? ld2(w + ((size_t)i2 * ldw + j2) * 2) : make_double2(0.0, 0.0);
  }
  __syncthreads();
  double sk = 0.0, nr = 0.0, trr = 0.0, tri = 0.0;
  const double f = (I == J) ? 1.0 : 2.0;
  for (int r = ty; r < RT; r += 8) {
    const double2 a = ta[r][tx];   // W[i][j]
    const double2 bt = tb[tx][r];  // W[j][i]
    const double hx = a.x + bt.x, hy = a.y - bt.y;
    sk += f * (hx * hx + hy * hy);
    nr += a.x * a.x + a.y * a.y;
    if (I != J) nr += bt.x * bt.x + bt.y * bt.y;
    if (I == J && r == tx) {
      trr += a.x;
      tri += a.y;
    }
  }
  double vals[4] = {sk, nr, trr, tri};
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    double v = vals[q];
    for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffff, v, off);
    if (tx == 0) red[ty][q] = v;
  }
  __syncthreads();
  if (threadIdx.x < 4) {
    double v = 0.0;
    for (int q = 0; q < 8; ++q) v += red[q][threadIdx.x];
    partial[(size_t)blockIdx.x * 4 + threadIdx.x] = v;
  }
}

__global__ void k_resid_final(int nt, const double* __restrict__ partial, double* out) {
  __shared__ double red[32][4];
  double v[4] = {0, 0, 0, 0};
  for (int t = threadIdx.x; t < nt; t += blockDim.x)
    for (int q = 0; q < 4; ++q) v[q] += partial[(size_t)t * 4 + q];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int q = 0; q < 4; ++q) {
    for (int off = 16; off > 0; off >>= 1) v[q] += __shfl_xor_sync(0xffffffff, v[q], off);
    if (lane == 0) red[w][q] = v[q];
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double s[4] = {0, 0, 0, 0};
    for (int j = 0; j < (int)(blockDim.x >> 5); ++j)
      for (int q = 0; q < 4; ++q) s[q] += red[j][q];
    const double nrm = sqrt(s[1]);
    if (nrm == 0.0) {
      out[0] = 0.0;
      out[1] = 0.0;
      out[2] = 0.0;
    } else {
      out[0] = sqrt(s[0]) / nrm;
      out[1] = hypot(s[2], s[3]) / nrm;
      out[2] = nrm;
    }
  }
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------

static std::vector<int2> generic_tiles(int n) {
  const int C = (n + SR - 1) / SR, Gt = (n + DPW - 1) / DPW, cf = fast_chunks(n);
  std::vector<int2> v;
  for (int c = 0; c < C; ++c) {
    const int gmax = std::min(Gt - 1, (c * SR + SR - 1) / DPW);
    for (int g = 0; g <= gmax; ++g) {
      const bool interior = g >= 1 && g <= GPC * c - 1;
      const bool fast = (c < cf) && interior;
      // the chunk ending exactly at row N-1 runs the fast body with the
      // last-row special case (flag bit 30 of .x)
      const bool fast_last = !fast && interior && (c + 1) * SR == n;
      if (!fast) v.push_back(make_int2(c | (fast_last ? (1 << 30) : 0), g));
    }
  }
  return v;
}

static size_t op_bytes(int n, int C) {
  const size_t nsub = (size_t)(n + SUB - 1) / SUB;
  const size_t ngen = generic_tiles(n).size();
  return sizeof(double) * ((size_t)4 * n + 2 * nsub * n + (size_t)4 * C * n + (size_t)M0X * C) +
         sizeof(int2) * ngen + 512;
}

int op_create(int n, int device, zt_operator** out) {
  if (n < 2) return fail(ZT_EINVAL, "matrix truncation must be at least 2, got " + std::to_string(n));
  if (n > 16384) return fail(ZT_EINVAL, "matrix truncation above 16384 is not supported");
  int prev;
  ZT_CUDA_CHECK(cudaGetDevice(&prev));
  ZT_CUDA_CHECK(cudaSetDevice(device));
  zt_operator* op = new zt_operator;
  op->n = n;
  op->device = device;
  op->C = (n + SR - 1) / SR;
  const int C = op->C;
  cudaError_t e = cudaMalloc(&op->block, op_bytes(n, C));
  if (e != cudaSuccess) {
    delete op;
    cudaSetDevice(prev);
    return cuda_fail(e, "cudaMalloc(operator)");
  }
  double* q = reinterpret_cast<double*>(op->block);
  op->sqB = q;
  q += n;
  op->Bq = q;
  q += n;
  op->L0 = q;
  q += n;
  op->dinv0 = q;
  q += n;
  op->d0 = q;
  q += (size_t)((n + SUB - 1) / SUB) * n;
  op->lins = q;
  q += (size_t)((n + SUB - 1) / SUB) * n;
  op->lin = q;
  q += (size_t)C * n;
  op->G = q;
  q += (size_t)C * n;
  op->H = q;
  q += (size_t)C * n;
  op->K = q;
  q += (size_t)C * n;
  op->m0x = q;
  q += (size_t)M0X * C;
  cudaMemset(op->block, 0, op_bytes(n, C));
  {
    std::vector<int2> gt = generic_tiles(n);
    op->gen_tiles = reinterpret_cast<int2*>(reinterpret_cast<uintptr_t>(q + 1) & ~(uintptr_t)7);
    op->ngen = (int)gt.size();
    cudaMemcpy(op->gen_tiles, gt.data(), sizeof(int2) * gt.size(), cudaMemcpyHostToDevice);
  }
  k_op_sqrt_table<<<(n + 255) / 256, 256>>>(n, op->sqB, op->Bq);
  ZT_LAUNCHED();
  k_op_build<<<(n + 127) / 128, 128>>>(n, C, op->sqB, op->d0, op->lins, op->lin, op->G, op->H, op->K, op->L0,
                                        op->dinv0, op->m0x);
  ZT_LAUNCHED();
  int smem = SOLVE_WARPS * SR * DPW * (int)sizeof(double2);
  int asmem = SOLVE_WARPS * TR * 32 * (int)sizeof(double2);
  cudaFuncSetAttribute(k_solve_merged<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k_solve_merged<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k_apply_tiles, cudaFuncAttributeMaxDynamicSharedMemorySize, asmem);
  e = cudaDeviceSynchronize();
  cudaSetDevice(prev);
  if (e != cudaSuccess) {
    cudaFree(op->block);
    delete op;
    return cuda_fail(e, "operator build");
  }
  *out = op;
  return ZT_OK;
}

int op_destroy(zt_operator* op) {
  if (!op) return ZT_OK;
  cudaFree(op->block);
  delete op;
  return ZT_OK;
}

size_t solve_workspace_bytes(int n, int batch) {
  const int C = (n + SR - 1) / SR;
  const size_t one = ((2 * (size_t)C * n + 2 * (size_t)C + 2) * sizeof(double2) + 511) & ~(size_t)255;
  return one * batch;
}


static int stream_solve_one(zt_operator* op, const double* w, int64_t ldw, int64_t sw, double* p,
                            int64_t ldp, int64_t sp, int batch, void* ws, size_t ws_bytes,
                            cudaStream_t st) {
  const int n = op->n, C = op->C;
  if (ws_bytes < solve_workspace_bytes(n, batch)) return fail(ZT_ENOMEM, "solve workspace too small");
  SolveArgs A;
  A.n = n;
  A.C = C;
  A.ntiles = solve_ntiles(C);
  A.sqB = op->sqB;
  A.Bq = op->Bq;
  A.d0s = op->d0;
  A.lins = op->lins;
  A.lin = op->lin;
  A.L0 = op->L0;
  A.dinv0 = op->dinv0;
  A.w = w;
  A.ldw = ldw;
  A.sw = sw;
  A.p = p;
  A.ldp = ldp;
  A.sp = sp;
  A.yend = reinterpret_cast<double2*>(ws);
  A.xst = A.yend + (size_t)batch * C * n;
  A.m0acc = A.xst + (size_t)batch * C * n;
  A.m0mg = A.m0acc + (size_t)batch * C * 2;
  const int smem = SOLVE_WARPS * SR * DPW * (int)sizeof(double2);
  A.ntiles = fast_ntiles(fast_chunks(n));
  const int tg = (op->ngen + SOLVE_WARPS - 1) / SOLVE_WARPS;
  const int td = (A.ntiles + SOLVE_WARPS - 1) / SOLVE_WARPS;
  // one launch per tile pass: boundary tiles first (dispatched first, their
  // latency hides under the interior tiles), then the interior tiles
  // programmatic dependent launches: each pass's blocks are scheduled under
  // its predecessor's tail and wait (griddepcontrol.wait) before reading
  auto pass = [&](bool fin) -> int {
    const dim3 grid(tg + td, batch);
    ZT_CUDA_CHECK(launch_pdl(fin ? k_solve_merged<true> : k_solve_merged<false>, grid, dim3(SOLVE_WARPS * 32),
                             smem, st, A, (const int2*)op->gen_tiles, op->ngen, tg));
    ZT_LAUNCHED();
    return ZT_OK;
  };
  int rc = pass(false);
  if (rc) return rc;
  const int seg = std::max(8, (C + CE - 1) / CE);  // chunk segments per carry block
  ZT_CUDA_CHECK(launch_pdl(seg <= 16 ? k_solve_carry<512> : k_solve_carry<1024>,  // N > 8192: 32 segments
                           dim3((n + 31) / 32, batch), dim3(32 * seg), 0, st, n, C, (const double*)op->G,
                           (const double*)op->H, (const double*)op->K, (const double*)op->m0x, A.yend, A.xst,
                           (const double2*)A.m0acc, A.m0mg));
  ZT_LAUNCHED();
  rc = pass(true);
  if (rc) return rc;
  ZT_CUDA_CHECK(cudaGetLastError());
  return ZT_OK;
}

int stream_solve(zt_operator* op, const double* w, int64_t ldw, int64_t sw, double* p, int64_t ldp,
                 int64_t sp, int batch, void* ws, size_t ws_bytes, cudaStream_t st) {
  return stream_solve_one(op, w, ldw, sw, p, ldp, sp, batch, ws, ws_bytes, st);
}

int apply_laplacian(zt_operator* op, const double* w, int64_t ldw, int64_t sw, double* y,
                    int64_t ldy, int64_t sy, int sign, int batch, cudaStream_t st) {
  if (sign != 1 && sign != -1) return fail(ZT_EINVAL, "sign must be -1 or +1");
  const int n = op->n, Ca = (n + TR - 1) / TR;
  ApplyArgs A;
  A.n = n;
  A.C = Ca;
  A.ntiles = Ca * (Ca + 1) / 2;
  A.sign = sign;
  A.sqB = op->sqB;
  A.w = w;
  A.ldw = ldw;
  A.sw = sw;
  A.y = y;
  A.ldy = ldy;
  A.sy = sy;
  const int tb = (A.ntiles + SOLVE_WARPS - 1) / SOLVE_WARPS;
  k_apply_tiles<<<dim3(tb, batch), SOLVE_WARPS * 32, SOLVE_WARPS * TR * 32 * (int)sizeof(double2), st>>>(A);
  ZT_LAUNCHED();
  ZT_CUDA_CHECK(cudaGetLastError());
  return ZT_OK;
}

size_t resid_workspace_bytes(int n) {
  const int T = (n + RT - 1) / RT;
  return (size_t)(T * (T + 1) / 2) * 4 * sizeof(double) + 256;
}

int residuals(int n, const double* w, int64_t ldw, double* out, void* ws, cudaStream_t st) {
  const int T = (n + RT - 1) / RT;
  const int nt = T * (T + 1) / 2;
  double* partial = reinterpret_cast<double*>(ws);
  k_resid_partial<<<nt, 256, 0, st>>>(n, w, ldw, nt, partial);
  ZT_LAUNCHED();
  k_resid_final<<<1, 1024, 0, st>>>(nt, partial, out);
  ZT_LAUNCHED();
  ZT_CUDA_CHECK(cudaGetLastError());
  return ZT_OK;
}

int op_factors(zt_operator* op, double* linv_h, double* dinv_h) {
  // reconstruct the reference's sheared N x N tables (laplacian.py:213-215)
  // by replaying the recurrence on the host from the device chunk pivots —
  // used by tests to prove bit-identity with dpttrf.
  const int n = op->n, C = op->C;
  const size_t nsub = (size_t)(n + SUB - 1) / SUB;
  std::vector<double> sq(n), d0(nsub * n), L0(n), di0(n);
  ZT_CUDA_CHECK(cudaMemcpy(sq.data(), op->sqB, sizeof(double) * n, cudaMemcpyDeviceToHost));
  ZT_CUDA_CHECK(cudaMemcpy(d0.data(), op->d0, sizeof(double) * nsub * n, cudaMemcpyDeviceToHost));
  ZT_CUDA_CHECK(cudaMemcpy(L0.data(), op->L0, sizeof(double) * n, cudaMemcpyDeviceToHost));
  ZT_CUDA_CHECK(cudaMemcpy(di0.data(), op->dinv0, sizeof(double) * n, cudaMemcpyDeviceToHost));
  if (linv_h) std::fill(linv_h, linv_h + (size_t)n * n, 0.0);
  if (dinv_h) std::fill(dinv_h, dinv_h + (size_t)n * n, 0.0);
  for (int k = 0; k < n; ++k) {
    if (linv_h) linv_h[(size_t)k * n] = L0[k];
    if (dinv_h) dinv_h[(size_t)k * n] = di0[k];
  }
  for (int m = 1; m < n; ++m) {
    const int len = n - m;
    for (int k = 0; k < len; ++k) {
      const int i = m + k;
      // pivots at each row are recomputed exactly as the device does
      double d = d0[(size_t)(i / SUB) * n + m];
      const int kstart = std::max(i / SUB * SUB, m) - m;
      for (int kk = kstart; kk < k; ++kk) {
        const double e = (-sq[m + kk]) * sq[kk];
        const double L = e / d;
        const double s = (n - 1) * 0.5;
        const double kd = kk + 1.0;
        const double dg = 2.0 * (s * (2.0 * kd + 1.0 + m) - kd * (kd + m));
        volatile double prod = L * e;
        d = dg - prod;
      }
      if (dinv_h) dinv_h[(size_t)i * n + m] = 1.0 / d;
      if (linv_h && k < len - 1) {
        const double e = (-sq[m + k]) * sq[k];
        linv_h[(size_t)i * n + m] = e / d;
      }
    }
  }
  return ZT_OK;
}

}  // namespace zt
