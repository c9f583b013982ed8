// Quantized spherical-harmonic basis on the device:
// the eigenvectors of every tridiagonal Laplacian block (basis.py:119-165)
// and the per-diagonal transforms extract / project (basis.py:276-331).
//
// Block m (size L = N - m) has the exact spectrum {l(l+1) : l = m..N-1}
// (laplacian.py:156-159), so no eigenvalue solve is needed: each vector
// (l, m) is one O(L) twisted factorisation of T_m - l(l+1) I, one thread per
// vector, all (l, m) pairs in parallel.  Vectors are stored exactly as the
// reference's `QuantizedBasis.vectors[m]`: row-major (N - m) x n_l(m),
// n_l(m) = N - max(m, 1), columns l = max(m, 1) .. N-1, so a warp of
// consecutive l touches consecutive doubles at every row k.
#include <math.h>

#include "zt_tma.cuh"

namespace zt {

// block entries exactly as laplacian.py:129-137 computes them in float64
__device__ __forceinline__ double blk_diag(int n, int m, int k) {
  const double s = (n - 1) / 2.0;
  const double i = (double)k;
  return 2.0 * (s * (2.0 * i + 1.0 + m) - i * (i + m));
}
__device__ __forceinline__ double blk_off(int n, int m, int k) {
  const double i = (double)k;
  return -sqrt((i + m + 1.0) * (n - 1.0 - i - m)) * sqrt((i + 1.0) * (n - 1.0 - i));
}
__device__ __forceinline__ double guard(double d) {
  return fabs(d) < 1e-290 ? (d < 0.0 ? -1e-290 : 1e-290) : d;
}
// e / d without the IEEE division sequence: rcp seed + 2 Newton steps (~1 ulp)
__device__ __forceinline__ double qdiv(double e, double d) {
  d = guard(d);
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(d));
  double t = fma(-d, r, 1.0);
  r = fma(r, t, r);
  t = fma(-d, r, 1.0);
  r = fma(r, t, r);
  return e * r;
}

// One eigenvector per thread.  Twisted factorisation of A = T_m - lambda I:
// backward U D U^T (U_k = e_k / D-_{k+1}) stored in the output column, then
// forward L D L^T with twist values gamma_k = D+_k - e_k U_k; the vector is
// v_r = 1 at r = argmin |gamma_k| and v_k = -L_k v_{k+1} above, v_{k+1} =
// -U_k v_k below.  Normalised to unit 2-norm and signed so the
// largest-magnitude entry (lowest index on ties) is positive
// (basis.py:110-114).
__global__ void __launch_bounds__(128) k_basis_vectors(int n, int m0, const long long* __restrict__ off,
                                                       double* __restrict__ vec) {
  const int m = m0 + blockIdx.y;
  const int nl = n - max(m, 1);
  const int lp = blockIdx.x * blockDim.x + threadIdx.x;
  if (lp >= nl) return;
  const int L = n - m;
  const int l = lp + max(m, 1);
  double* v = vec + off[m] + lp;  // v[k * nl]
  const size_t st = (size_t)nl;
  if (L == 1) {
    v[0] = 1.0;
    return;
  }
  const double lam = (double)l * (l + 1.0);
  // pass A: backward factorisation, U_k -> v[k]
  double dm = blk_diag(n, m, L - 1) - lam;
  for (int k = L - 2; k >= 0; --k) {
    const double e = blk_off(n, m, k);
    const double u = qdiv(e, dm);
    v[k * st] = u;
    dm = (blk_diag(n, m, k) - lam) - e * u;
  }
  // pass B: forward factorisation and twist index.  The loops that read the
  // column back fetch 8 rows ahead (one thread streams its own column, so
  // the loads would otherwise be serialised DRAM round trips).
  constexpr int PB = 8;
  double dp = blk_diag(n, m, 0) - lam;
  int r = 0;
  double gbest = INFINITY;
  for (int k0 = 0; k0 < L; k0 += PB) {
    double uu[PB];
#pragma unroll
    for (int q = 0; q < PB; ++q) uu[q] = (k0 + q < L - 1) ? v[(size_t)(k0 + q) * st] : 0.0;
#pragma unroll
    for (int q = 0; q < PB; ++q) {
      const int k = k0 + q;
      if (k < L) {
        const double e = (k < L - 1) ? blk_off(n, m, k) : 0.0;
        const double g = dp - e * uu[q];
        if (fabs(g) < gbest) {
          gbest = fabs(g);
          r = k;
        }
        if (k < L - 1) dp = (blk_diag(n, m, k + 1) - lam) - e * qdiv(e, dp);
      }
    }
  }
  // pass C: L_k for k < r over the stored U_k
  dp = blk_diag(n, m, 0) - lam;
  for (int k = 0; k < r; ++k) {
    const double e = blk_off(n, m, k);
    const double lk = qdiv(e, dp);
    v[k * st] = lk;
    dp = (blk_diag(n, m, k + 1) - lam) - e * lk;
  }
  // pass D: back-substitution from the twist
  double u = (r < L - 1) ? v[r * st] : 0.0;
  v[r * st] = 1.0;
  double x = 1.0;
  for (int k1 = r; k1 > 0; k1 -= PB) {  // rows k1-1 .. k1-PB, descending
    double lk[PB];
#pragma unroll
    for (int q = 0; q < PB; ++q) lk[q] = (k1 - 1 - q >= 0) ? v[(size_t)(k1 - 1 - q) * st] : 0.0;
#pragma unroll
    for (int q = 0; q < PB; ++q) {
      const int k = k1 - 1 - q;
      if (k >= 0) {
        x = -lk[q] * x;
        v[(size_t)k * st] = x;
      }
    }
  }
  x = 1.0;
  for (int k0 = r; k0 < L - 1; k0 += PB) {  // writes rows k0+1 .. k0+PB
    double un[PB];
#pragma unroll
    for (int q = 0; q < PB; ++q) un[q] = (k0 + 1 + q < L - 1) ? v[(size_t)(k0 + 1 + q) * st] : 0.0;
#pragma unroll
    for (int q = 0; q < PB; ++q) {
      const int k = k0 + q;
      if (k < L - 1) {
        x = -u * x;
        v[(size_t)(k + 1) * st] = x;
        u = un[q];
      }
    }
  }
  // pass E: norm and the sign of the largest-magnitude entry
  double ss = 0.0, big = -1.0, sgn = 1.0;
  for (int k0 = 0; k0 < L; k0 += PB) {
    double t[PB];
#pragma unroll
    for (int q = 0; q < PB; ++q) t[q] = (k0 + q < L) ? v[(size_t)(k0 + q) * st] : 0.0;
#pragma unroll
    for (int q = 0; q < PB; ++q) {
      ss = fma(t[q], t[q], ss);
      if (fabs(t[q]) > big) {
        big = fabs(t[q]);
        sgn = t[q] < 0.0 ? -1.0 : 1.0;
      }
    }
  }
  const double sc = sgn / sqrt(ss);
  for (int k0 = 0; k0 < L; k0 += PB) {
    double t[PB];
#pragma unroll
    for (int q = 0; q < PB; ++q) t[q] = (k0 + q < L) ? v[(size_t)(k0 + q) * st] : 0.0;
#pragma unroll
    for (int q = 0; q < PB; ++q)
      if (k0 + q < L) v[(size_t)(k0 + q) * st] = t[q] * sc;
  }
}

// extract (basis.py:319-331): pos[m][l'] = -i sum_k V[k][l'] W[k+m][k],
// neg[m][l'] = -i (-1)^m sum_k V[k][l'] W[k][k+m]  (m >= 1).
__global__ void __launch_bounds__(128) k_basis_extract(int n, int m0, const long long* __restrict__ off,
                                                       const long long* __restrict__ coff,
                                                       const double* __restrict__ vec,
                                                       const double* __restrict__ w, int64_t ldw,
                                                       double* __restrict__ pos, double* __restrict__ neg) {
  const int m = m0 + blockIdx.y;
  const int nl = n - max(m, 1);
  const int lp = blockIdx.x * blockDim.x + threadIdx.x;
  if (lp >= nl) return;
  const int L = n - m;
  const double* v = vec + off[m] + lp;
  double2 a = make_double2(0.0, 0.0), b = make_double2(0.0, 0.0);
  for (int k = 0; k < L; ++k) {
    const double t = __ldg(v + (size_t)k * nl);
    const double2 lo = ld2(w + ((size_t)(k + m) * ldw + k) * 2);  // broadcast across the warp
    a.x = fma(t, lo.x, a.x);
    a.y = fma(t, lo.y, a.y);
    if (m >= 1) {
      const double2 up = ld2(w + ((size_t)k * ldw + k + m) * 2);
      b.x = fma(t, up.x, b.x);
      b.y = fma(t, up.y, b.y);
    }
  }
  const size_t c = (size_t)coff[m] + lp;
  st2(pos + 2 * c, make_double2(a.y, -a.x));  // -i (x + iy) = y - i x
  if (m >= 1) {
    const double s = (m & 1) ? -1.0 : 1.0;
    st2(neg + 2 * c, make_double2(s * b.y, -s * b.x));
  } else {
    st2(neg + 2 * c, make_double2(a.y, a.x));  // neg[0] = conj(pos[0]) (basis.py:330)
  }
}

// project (basis.py:276-316): the m-th sub-diagonal of W is
// i sum_l' V[k][l'] pos[m][l']; a warp per row k, lanes over l'.  With
// `neg == nullptr` the strict upper triangle is the skew completion
// -conj(lower^T) (laplacian.py:336-338); otherwise it is
// i (-1)^m sum_l' V[k][l'] neg[m][l'] (allow_complex).
__global__ void __launch_bounds__(256) k_basis_project(int n, int m0, const long long* __restrict__ off,
                                                       const long long* __restrict__ coff,
                                                       const double* __restrict__ vec,
                                                       const double* __restrict__ pos,
                                                       const double* __restrict__ neg, double* __restrict__ w,
                                                       int64_t ldw) {
  const int m = m0 + blockIdx.y;
  const int nl = n - max(m, 1);
  const int L = n - m;
  const int lane = threadIdx.x & 31;
  const int k = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (k >= L) return;
  const double* v = vec + off[m] + (size_t)k * nl;
  const double* cp = pos + 2 * (size_t)coff[m];
  const double* cn = neg ? neg + 2 * (size_t)coff[m] : nullptr;
  double2 a = make_double2(0.0, 0.0), b = make_double2(0.0, 0.0);
  for (int j = lane; j < nl; j += 32) {
    const double t = v[j];
    const double2 c = ld2(cp + 2 * j);
    a.x = fma(t, c.x, a.x);
    a.y = fma(t, c.y, a.y);
    if (cn && m >= 1) {
      const double2 d = ld2(cn + 2 * j);
      b.x = fma(t, d.x, b.x);
      b.y = fma(t, d.y, b.y);
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    a.x += __shfl_xor_sync(0xffffffff, a.x, o);
    a.y += __shfl_xor_sync(0xffffffff, a.y, o);
    b.x += __shfl_xor_sync(0xffffffff, b.x, o);
    b.y += __shfl_xor_sync(0xffffffff, b.y, o);
  }
  if (lane != 0) return;
  const double2 lo = make_double2(-a.y, a.x);  // i (x + iy)
  st2(w + ((size_t)(k + m) * ldw + k) * 2, lo);
  if (m == 0) return;
  if (!cn) {
    st2(w + ((size_t)k * ldw + k + m) * 2, make_double2(-lo.x, lo.y));  // -conj
  } else {
    const double s = (m & 1) ? -1.0 : 1.0;
    st2(w + ((size_t)k * ldw + k + m) * 2, make_double2(-s * b.y, s * b.x));
  }
}

static int check_range(int n, int m0, int m1) {
  if (n < 2) return fail(ZT_EINVAL, "matrix truncation must be at least 2, got " + std::to_string(n));
  if (m0 < 0 || m1 > n || m0 >= m1) return fail(ZT_EINVAL, "basis: bad order range");
  return ZT_OK;
}

int basis_vectors(int n, int m0, int m1, const long long* off, double* vec, cudaStream_t st) {
  int rc = check_range(n, m0, m1);
  if (rc) return rc;
  const int nlmax = n - max(m0, 1);
  dim3 grid((nlmax + 127) / 128, m1 - m0);
  k_basis_vectors<<<grid, 128, 0, st>>>(n, m0, off, vec);
  ZT_LAUNCHED();
  ZT_CUDA_CHECK(cudaGetLastError());
  return ZT_OK;
}

int basis_extract(int n, int m0, int m1, const long long* off, const long long* coff, const double* vec,
                  const double* w, int64_t ldw, double* pos, double* neg, cudaStream_t st) {
  int rc = check_range(n, m0, m1);
  if (rc) return rc;
  const int nlmax = n - max(m0, 1);
  dim3 grid((nlmax + 127) / 128, m1 - m0);
  k_basis_extract<<<grid, 128, 0, st>>>(n, m0, off, coff, vec, w, ldw, pos, neg);
  ZT_LAUNCHED();
  ZT_CUDA_CHECK(cudaGetLastError());
  return ZT_OK;
}

int basis_project(int n, int m0, int m1, const long long* off, const long long* coff, const double* vec,
                  const double* pos, const double* neg, double* w, int64_t ldw, cudaStream_t st) {
  int rc = check_range(n, m0, m1);
  if (rc) return rc;
  const int lmax = n - m0;
  dim3 grid((lmax + 7) / 8, m1 - m0);
  k_basis_project<<<grid, 256, 0, st>>>(n, m0, off, coff, vec, pos, neg, w, ldw);
  ZT_LAUNCHED();
  ZT_CUDA_CHECK(cudaGetLastError());
  return ZT_OK;
}

}  // namespace zt

namespace zt {

// ---------------------------------------------------------------------------
// Grid rendering (diagnostics.py:113-187): G[i][m] =
// sum_l w_lm Pbar_lm(cos theta_i), one thread per (theta_i, m), the fully
// normalised associated-Legendre recurrence evaluated in the reference's
// operation order (no FMA contraction); the azimuthal sum is a complex GEMM
// with the phase table e^{i m phi_j} (weight 2 for m >= 1).
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(128) k_grid_legendre(int n, int lmax, int nlat, const long long* __restrict__ coff,
                                                       const double* __restrict__ pos, double* __restrict__ g,
                                                       int64_t ldg) {
  const int m = blockIdx.y;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nlat || m > lmax) return;
  const double step = 3.141592653589793 / (double)(nlat - 1);
  const double th = (i == nlat - 1) ? 3.141592653589793 : __dmul_rn((double)i, step);  // np.linspace
  const double ct = cos(th), st = sin(th);
  double pmm = 1.0 / sqrt(4.0 * 3.141592653589793);
  for (int q = 1; q <= m; ++q) {
    const double s = -sqrt((2.0 * q + 1.0) / (2.0 * q));
    pmm = __dmul_rn(__dmul_rn(s, st), pmm);
  }
  const double* cm = pos + 2 * (size_t)coff[m];
  const int lo = max(m, 1);
  double gr = 0.0, gi = 0.0;
  auto add = [&](int l, double p) {
    if (lo <= l && l <= lmax) {
      gr = __dadd_rn(gr, __dmul_rn(cm[2 * (l - lo)], p));
      gi = __dadd_rn(gi, __dmul_rn(cm[2 * (l - lo) + 1], p));
    }
  };
  double pprev = pmm;
  add(m, pprev);
  if (m + 1 <= lmax) {
    double pcur = __dmul_rn(__dmul_rn(sqrt(2.0 * m + 3.0), ct), pmm);
    add(m + 1, pcur);
    const int top = min(lmax, n - 1);
    for (int l = m + 2; l <= top; ++l) {
      const double ll = (double)l * l - (double)m * m;
      const double a = sqrt((4.0 * l * l - 1.0) / ll);
      const double b = sqrt(((2.0 * l + 1.0) * (l - 1.0 + m) * (l - 1.0 - m)) / ((2.0 * l - 3.0) * ll));
      const double pn = __dsub_rn(__dmul_rn(__dmul_rn(a, ct), pcur), __dmul_rn(b, pprev));
      add(l, pn);
      pprev = pcur;
      pcur = pn;
    }
  }
  g[((size_t)i * ldg + m) * 2] = gr;
  g[((size_t)i * ldg + m) * 2 + 1] = gi;
}

__global__ void k_grid_phases(int lmax, int nlon, double* __restrict__ ph) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  const int m = blockIdx.y;
  if (j >= nlon || m > lmax) return;
  const double phi = (2.0 * 3.141592653589793 * (double)j) / (double)nlon;
  double s, c;
  sincos((double)m * phi, &s, &c);
  const double wgt = m == 0 ? 1.0 : 2.0;
  ph[((size_t)m * nlon + j) * 2] = c * wgt;
  ph[((size_t)m * nlon + j) * 2 + 1] = s * wgt;
}

int zgemm_rect(int m, int n, int k, const double* a, int64_t lda, const double* b, int64_t ldb, double* c,
               int64_t ldc, int algo, cudaStream_t st);

// field (complex, nlat x nlon; the caller keeps the real part) from the
// m >= 0 coefficients; work = nlat x (lmax+1) + (lmax+1) x nlon complex
int grid_eval(int n, int lmax, int nlat, int nlon, const long long* coff, const double* pos, double* work,
              double* field, cudaStream_t st) {
  if (n < 2 || lmax < 1 || lmax > n - 1 || nlat < 2 || nlon < 2) return fail(ZT_EINVAL, "grid_eval: bad sizes");
  double* g = work;
  double* ph = work + (size_t)nlat * (lmax + 1) * 2;
  k_grid_legendre<<<dim3((nlat + 127) / 128, lmax + 1), 128, 0, st>>>(n, lmax, nlat, coff, pos, g, lmax + 1);
  ZT_LAUNCHED();
  k_grid_phases<<<dim3((nlon + 127) / 128, lmax + 1), 128, 0, st>>>(lmax, nlon, ph);
  ZT_LAUNCHED();
  ZT_CUDA_CHECK(cudaGetLastError());
  return zgemm_rect(nlat, nlon, lmax + 1, g, lmax + 1, ph, nlon, field, nlon, 0, st);
}

}  // namespace zt
