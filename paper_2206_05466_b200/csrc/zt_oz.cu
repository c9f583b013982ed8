// FP64-accurate complex GEMM on the INT8 tensor cores (Ozaki scheme II with
// a Gaussian-integer split):
//
// * operands are scaled to integers (row / column power-of-two scales; the
//   line maximum is put at KB = 55 bits for K <= 4096, 54 up to K = 2^14, so
//   entries down to a quarter / half of their line's maximum keep all 53 of
//   their significant bits) and reduced modulo NMOD = 17 pairwise-coprime odd
//   moduli p <= 241 whose prime factors are all = 1 mod 4;
// * for such p, -1 has a square root iota mod p, so Z[i] / (p) splits into two
//   copies of Z / p: phi+(x + iy) = x + iota y and phi-(x + iy) = x - iota y
//   (mod p) are ring homomorphisms.  A complex product C = A B mod p is
//   therefore TWO real products, U = phi+(A) phi+(B) = Re C + iota Im C and
//   V = phi-(A) phi-(B) = Re C - iota Im C (mod p), instead of the four of the
//   4M form (or three of Karatsuba): 34 int8 GEMMs per complex product
//   (17 moduli x 2) instead of 64;
// * each real product runs on tcgen05 kind::i8 (int32 accumulation); the
//   epilogue forms (U + V) mod p = 2 Re C and (U - V) mod p = 2 iota Im C
//   and the CRT reconstruction folds 2^-1 and (2 iota)^-1 into its weights,
//   reassembling the exact integer product, which is scaled back.
//
// Moduli: 241 233 229 221(=13*17) 205(=5*41) 197 193 181 173 157 149 137 113
// 109 101 97 89, product M ~ 2^124.16: KB-bit operands up to K = 2^14 (the
// residue GEMM's exact-division range) with the complex sum bound
// 2 K 2^(2 KB) < M / 2 (oz_bits).
//
// Layouts (int8 centred residues, zero padded to 256 in every dimension):
//   A residues [NMOD][2][Mp][Kp]  planes phi+ (A), phi- (A)   (K-major rows)
//   B residues [NMOD][2][Np][Kp]  planes phi+ (B), phi- (B)   (K-major: B^T rows)
//   R residues [NMOD][2][Mp][Np]  ((U + V) + k_p) mod p, ((U - V) + k_p) mod p,
//                                 k_p = (p - 1) / 2, unsigned bytes in [0, p)
#include <cuda.h>

#include <algorithm>
#include <cmath>
#include <type_traits>
#include <type_traits>
#include <vector>

#include "zt_common.cuh"
#include "zt_tma.cuh"

namespace zt {

constexpr int OZ_NMOD = 17;
__constant__ int c_oz_p[OZ_NMOD];
__constant__ unsigned c_oz_m[OZ_NMOD];  // ceil(2^(31 + l) / p), l = ceil(log2 p)
__constant__ unsigned c_oz_s[OZ_NMOD];  // l - 1
static const int h_oz_p[OZ_NMOD] = {241, 233, 229, 221, 205, 197, 193, 181, 173,
                                    157, 149, 137, 113, 109, 101, 97,  89};
// row / column shift of a line holding a NaN or an infinity: the product's
// row / column is written as NaN (the residues of such a line are zero)
constexpr int OZ_BAD = -(1 << 29);
constexpr int OZ_MAXDEV = 64;

namespace oz {

// ---------------------------------------------------------------------------
// Residue GEMM (cta_group::2): a CTA pair computes one 256 x 256 tile of one
// modulus as two real products, U (phi+ planes) and V (phi- planes), into two
// 256-column TMEM accumulators per CTA.  The leader's single MMA thread
// issues M = 256, N = 256, K = 32 MMAs over both CTAs' shared memory (every
// SM runs 128 x 256 x 32 at 8 KB of operand per SM per MMA); U of the next
// tile starts as soon as the epilogue has drained U of this one, so the
// epilogue of every accumulator overlaps the MMAs of the other.  The
// epilogue keeps U's residues in registers (32 words per thread) and, when V
// lands, stores (U + V) and (U - V) mod p.
// ---------------------------------------------------------------------------
#ifndef OZ_SW128
#define OZ_SW128 1
#endif
#ifndef OZ_KPS
#define OZ_KPS 1
#endif
#ifndef OZ_STAGES
#define OZ_STAGES 6
#endif
#if OZ_SW128
// 128 B K blocks under the 128 B swizzle: one TMA box of 128 rows x 128 B per
// operand per stage (64 B blocks / 64 B swizzle: 213 -> 199.5 us per full
// product at N = 2048, 1545 -> 1441 us at N = 4096)
constexpr int TM = 256, TN = 256, TK = 128;  // pair tile; TK in bytes
constexpr int KPS = OZ_KPS;                  // K blocks per pipeline stage
#else
constexpr int TM = 256, TN = 256, TK = 64;  // pair tile; TK in bytes (64 B swizzle)
constexpr int KPS = 2;                     // K blocks per pipeline stage
#endif
constexpr int A_BYTES = 128 * TK;          // one CTA's 128 rows of an A plane
constexpr int B_BYTES = (TN / 2) * TK;     // one CTA's 128 columns of a B plane
constexpr int STAGE_BYTES = KPS * (A_BYTES + B_BYTES);
constexpr int STAGES = OZ_STAGES;
constexpr int EPI_WARPS = 16;             // 4 per TMEM lane quarter, 64 columns each
constexpr int THREADS = (2 + EPI_WARPS) * 32;
constexpr int SMEM = STAGES * STAGE_BYTES + 1024 + 256;
// D s32, A/B signed int8, K-major, M = 256 (pair), N = 256
constexpr uint32_t IDESC = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(TN >> 3) << 17) |
                           ((uint32_t)(TM >> 4) << 24);

// UMMA smem descriptor: K-major, TK-byte swizzle (64 B: layout 4; 128 B:
// layout 2), 8-row groups 8 TK bytes apart
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr) {
  return (uint64_t)((saddr & 0x3FFFF) >> 4) | ((uint64_t)1 << 16) | ((uint64_t)((8 * TK) >> 4) << 32) |
         ((uint64_t)1 << 46) | ((uint64_t)(TK == 128 ? 2 : 4) << 61);
}
__device__ __forceinline__ void mbar_arrive_tx(uint64_t* b, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
// shared::cluster address of the same variable in CTA `rank` of the cluster
__device__ __forceinline__ uint32_t mapa(uint32_t saddr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(saddr), "r"(rank));
  return r;
}
// Barrier waits with a suspend-time hint: a waiting warp is parked by the
// hardware until the phase completes instead of spinning (a spinning
// try_wait loop kept the XU pipe ~90% busy in ncu and starved the MMA
// thread's uniform-register moves)
constexpr uint32_t SUSPEND_NS = 0x989680;
__device__ __forceinline__ void wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity), "r"(SUSPEND_NS)
      : "memory");
}
__device__ __forceinline__ void mbar_wait_cluster(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1, %2;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity), "r"(SUSPEND_NS)
      : "memory");
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// TMA into this CTA's shared memory, completion counted on the leader's barrier
__device__ __forceinline__ void tma2d_pair(void* dst, const CUtensorMap* map, int c0, int c1, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, "
      "%3}], [%4];" ::"r"(smem_u32(dst)),
      "l"(map), "r"(c0), "r"(c1), "r"(bar)
      : "memory");
}
__device__ __forceinline__ void mma(uint32_t d, uint64_t a, uint64_t b, uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(d),
      "l"(a), "l"(b), "r"(IDESC), "r"(acc));
}
__device__ __forceinline__ bool elect_one() {
  uint32_t pred = 0;
  asm volatile(
      "{\n.reg .b32 rx;\n.reg .pred px;\nelect.sync rx|px, %1;\n@px mov.s32 %0, 1;\n}" : "+r"(pred) : "r"(0xffffffffu));
  return pred != 0;
}
// arrive on the barrier at this offset in both CTAs once the issued MMAs finish
__device__ __forceinline__ void commit_both(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_u32(bar)),
      "h"((unsigned short)3)
      : "memory");
}

#define OZ_LD32(v, addr)                                                                                         \
  asm volatile(                                                                                                  \
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"           \
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"                                 \
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),        \
        "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),  \
        "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), \
        "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])  \
      : "r"(addr))

struct GemmArgs {
  int nmod, mt, nt, kt;  // pair tiles per dimension (256 rows / columns) and K blocks (64 B)
  int lower;             // square: only the 256-tiles on or below the diagonal
  int bswap;             // B planes read swapped (phi- with U, phi+ with V): B = conj of the converted rows
  int mp, np;            // padded M, N (output leading dimension np)
  int8_t* r;             // [nmod][2][mp][np]
};

__host__ __device__ __forceinline__ int lower_count(int mt) { return mt * (mt + 1) / 2; }
// work item w -> modulus j, pair tile (tm, tn).  Within a modulus the tiles
// run in bands of GR row tiles, column tiles outer and rows inner inside a
// band (lower mode: the same bands over the tiles with tn <= tm).  For
// N <= 4096 a band is the whole modulus (column-major order); at N = 8192 the
// ~74 tiles in flight share 16 row tiles of A and ~5 column tiles of B, and
// the product runs ~3% faster than in column-major order (bands of 8: ~3%
// slower; the kernel runs power-capped at that size, so fewer L2 misses
// matter little).
constexpr int GR = 16;
__device__ __forceinline__ void work_of(const GemmArgs& g, int w, int per, int& j, int& tm, int& tn) {
  j = w / per;
  int t = w - j * per;
  if (g.lower) {
    int r0 = 0;
    for (;;) {
      const int gs = min(GR, g.mt - r0);
      const int cnt = gs * r0 + gs * (gs + 1) / 2;
      if (t < cnt) {
        if (t < gs * r0) {
          tn = t / gs;
          tm = r0 + t % gs;
        } else {
          t -= gs * r0;
          int c = 0;
          while (t >= gs - c) {
            t -= gs - c;
            ++c;
          }
          tn = r0 + c;
          tm = tn + t;
        }
        return;
      }
      t -= cnt;
      r0 += GR;
    }
  } else {
    const int r0 = (t / (GR * g.nt)) * GR;
    t -= r0 * g.nt;
    const int gs = min(GR, g.mt - r0);
    tn = t / gs;
    tm = r0 + t % gs;
  }
}

// (v + off) mod p in [0, p) for an int32 accumulator v (|v| <= K 120^2 <
// 89 2^22 for K <= 2^14) and off < p: u = v + p 2^22 + off lies in
// (0, 2^31), and floor(u / p) is EXACT as umulhi(u, m) >> s with the
// Granlund-Montgomery magic m = ceil(2^(31 + l) / p), l = ceil(log2 p),
// s = l - 1 (m p - 2^(31+l) < p <= 2^l): no correction step, FMA / ALU pipes
// only (a min-based correction lands on the slow XU pipe, which bound the
// epilogue at 106% XU in ncu).
// add = p 2^22 + off, np = -p (mod 2^32): u - q p as one IMAD with no negation
__device__ __forceinline__ uint32_t modx(int v, uint32_t add, uint32_t m, uint32_t s, uint32_t np) {
  const uint32_t u = (uint32_t)v + add;
  return u + (__umulhi(u, m) >> s) * np;
}
__device__ __forceinline__ void st256(int8_t* p, const uint32_t* w) {
  asm volatile("st.global.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "r"(w[0]), "r"(w[1]), "r"(w[2]),
               "r"(w[3]), "r"(w[4]), "r"(w[5]), "r"(w[6]), "r"(w[7])
               : "memory");
}
// two 16-bit lanes holding values in [0, 2p - 2]: subtract p from each lane
// that is >= p (no carries cross lanes: every lane stays in [0, 2^16))
__device__ __forceinline__ uint32_t lanes_mod(uint32_t x2, uint32_t np, uint32_t c1) {
  const uint32_t t = x2 + c1;                       // lane + 0x8000 - p: bit 15 set iff lane >= p
  const uint32_t msk = (t >> 15) & 0x00010001u;
  return x2 + msk * np;                             // msk * (2^32 - p) = -msk * p (mod 2^32)
}

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(THREADS, 1)
    k_oz_gemm(const __grid_constant__ CUtensorMap ma, const __grid_constant__ CUtensorMap mb, GemmArgs g) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;  // [2]: U, V accumulator ready
  uint64_t* tempty = tfull + 2;      // [2]: U, V accumulator drained (both CTAs' epilogues)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_rank();
  const int cl = blockIdx.x >> 1, ncl = gridDim.x >> 1;
  const int per = g.lower ? lower_count(g.mt) : g.mt * g.nt;
  const int total = g.nmod * per;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&tfull[s], 1);
      mbar_init(&tempty[s], 2 * EPI_WARPS);  // the leader's: both CTAs' epilogue warps
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  cluster_sync();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = *tmem_slot;
  pdl_trigger();
  pdl_wait();  // operands from the conversions; R still read by the previous reconstruction

  // producer and MMA issuer: the whole warp runs the loop (warp-uniform
  // values stay in uniform registers, no per-instruction uniformity loops)
  // and one elected lane issues — the issuer shares its SM sub-partition with
  // four epilogue warps, so its instruction count per stage matters
  if (warp == 0) {
    if (elect_one()) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(&ma) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(&mb) : "memory");
    }
    const uint32_t fb0 = mapa(smem_u32(&full[0]), 0);
    unsigned it = 0;
    for (int w = cl; w < total; w += ncl) {
      int j, tm, tn;
      work_of(g, w, per, j, tm, tn);
      for (int part = 0; part < 2; ++part) {
        const int ra = (j * 2 + part) * g.mp + tm * TM + rank * 128;
        const int rb = (j * 2 + (part ^ g.bswap)) * g.np + tn * TN + rank * (TN / 2);
        for (int kb = 0; kb < g.kt; kb += KPS, ++it) {
          const int s = it % STAGES;
          wait(&empty[s], ((it / STAGES) & 1) ^ 1);
          if (elect_one()) {
            unsigned char* st = smem + s * STAGE_BYTES;
            if (rank == 0) mbar_arrive_tx(&full[s], 2 * STAGE_BYTES);
#pragma unroll
            for (int u = 0; u < KPS; ++u) {
              unsigned char* su = st + u * (A_BYTES + B_BYTES);
              tma2d_pair(su, &ma, (kb + u) * TK, ra, fb0 + s * 8);
              tma2d_pair(su + A_BYTES, &mb, (kb + u) * TK, rb, fb0 + s * 8);
            }
          }
          __syncwarp();
        }
      }
    }
    // drain: every issued stage consumed before this CTA may exit
    for (int i = 0; i < STAGES; ++i, ++it) wait(&empty[it % STAGES], ((it / STAGES) & 1) ^ 1);
  } else if (warp == 1) {
    if (rank == 0) {
      const uint64_t dsm = sdesc(smem_u32(smem));
      unsigned it = 0, lt = 0;
      for (int w = cl; w < total; w += ncl, ++lt) {
        for (int part = 0; part < 2; ++part) {
          mbar_wait_cluster(&tempty[part], (lt & 1) ^ 1);
          asm volatile("tcgen05.fence::after_thread_sync;");
          const uint32_t d = tmem + part * TN;
          for (int kb = 0; kb < g.kt; kb += KPS, ++it) {
            const int s = it % STAGES;
            wait(&full[s], (it / STAGES) & 1);
            asm volatile("tcgen05.fence::after_thread_sync;");
            if (elect_one()) {
#pragma unroll
              for (int u = 0; u < KPS; ++u) {
                // descriptor address field = shared-memory byte address >> 4
                const uint64_t a = dsm + (uint64_t)((s * STAGE_BYTES + u * (A_BYTES + B_BYTES)) >> 4);
                const uint64_t b = a + (A_BYTES >> 4);
#pragma unroll
                for (int k = 0; k < TK / 32; ++k) mma(d, a + 2 * k, b + 2 * k, (kb | u | k) ? 1u : 0u);
              }
              commit_both(&empty[s]);
            }
            __syncwarp();
          }
          if (elect_one()) commit_both(&tfull[part]);
          __syncwarp();
        }
      }
    }
  } else {
    constexpr int CW = TN / (EPI_WARPS / 4);      // columns per epilogue warp
    const int q = warp & 3;                       // TMEM lane quarter = tile rows q*32 ..
    const int ch = ((warp - 2) >> 2) * CW;        // this warp's column group of the 256-column tile
    const uint32_t te_remote = mapa(smem_u32(&tempty[0]), 0);
    unsigned lt = 0;
    for (int w = cl; w < total; w += ncl, ++lt) {
      int j, tm, tn;
      work_of(g, w, per, j, tm, tn);
      const uint32_t p = (uint32_t)c_oz_p[j], pm = c_oz_m[j], ps = c_oz_s[j];
      const uint32_t k = p >> 1, c1 = (0x8000u - p) * 0x10001u, cim = (p - 1) * 0x10001u;
      const uint32_t np = 0u - p, a0 = p << 22, ak = (p << 22) + k;
      const int row = tm * TM + rank * 128 + q * 32 + lane;
      const uint32_t trow = tmem + ((uint32_t)(q * 32) << 16) + ch;
      // U mod p (offset 0) kept in registers, 4 bytes per word; V is taken
      // with offset k, so (U + V) + k = u + v and (U - V) + k = u - v + (p - 1)
      // (mod p), each in [0, 2p - 2] before one lane-wise correction.
      // TMEM is read 64 columns at a time (two loads in flight per wait).
      uint32_t ur[CW / 4];
      wait(&tfull[0], lt & 1);
      asm volatile("tcgen05.fence::after_thread_sync;");
#pragma unroll
      for (int c = 0; c < CW; c += 64) {
        uint32_t v[64];
        OZ_LD32(v, trow + c);
        OZ_LD32((v + 32), trow + c + 32);
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
        for (int e = 0; e < 16; ++e) {
          const uint32_t lo = modx((int)v[4 * e], a0, pm, ps, np) | (modx((int)v[4 * e + 1], a0, pm, ps, np) << 16);
          const uint32_t hi =
              modx((int)v[4 * e + 2], a0, pm, ps, np) | (modx((int)v[4 * e + 3], a0, pm, ps, np) << 16);
          ur[c / 4 + e] = __byte_perm(lo, hi, 0x6420);
        }
      }
      asm volatile("tcgen05.fence::before_thread_sync;");
      __syncwarp();
      if (lane == 0)
        asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(te_remote) : "memory");
      // V: combine and store (U + V) and (U - V)
      wait(&tfull[1], lt & 1);
      asm volatile("tcgen05.fence::after_thread_sync;");
      int8_t* out_s = g.r + ((size_t)(j * 2) * g.mp + row) * g.np + tn * TN + ch;
      int8_t* out_d = out_s + (size_t)g.mp * g.np;
#pragma unroll
      for (int c = 0; c < CW; c += 64) {
        uint32_t v[64];
        OZ_LD32(v, trow + TN + c);
        OZ_LD32((v + 32), trow + TN + c + 32);
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        uint32_t ws[16], wd[16];
#pragma unroll
        for (int e = 0; e < 16; ++e) {
          const uint32_t uw = ur[c / 4 + e];
          const uint32_t u01 = __byte_perm(uw, 0u, 0x4140), u23 = __byte_perm(uw, 0u, 0x4342);
          const uint32_t v01 = modx((int)v[4 * e], ak, pm, ps, np) | (modx((int)v[4 * e + 1], ak, pm, ps, np) << 16);
          const uint32_t v23 =
              modx((int)v[4 * e + 2], ak, pm, ps, np) | (modx((int)v[4 * e + 3], ak, pm, ps, np) << 16);
          const uint32_t s01 = lanes_mod(u01 + v01, np, c1), s23 = lanes_mod(u23 + v23, np, c1);
          const uint32_t d01 = lanes_mod(u01 - v01 + cim, np, c1), d23 = lanes_mod(u23 - v23 + cim, np, c1);
          ws[e] = __byte_perm(s01, s23, 0x6420);
          wd[e] = __byte_perm(d01, d23, 0x6420);
        }
        // 256-bit stores: every store fills whole 32-byte sectors of its row
        // (16-byte stores wrote each sector in two halves: 25 us of 240 at N = 2048)
        st256(out_s + c, ws);
        st256(out_s + c + 32, ws + 8);
        st256(out_d + c, wd);
        st256(out_d + c + 32, wd + 8);
      }
      asm volatile("tcgen05.fence::before_thread_sync;");
      __syncwarp();
      if (lane == 0)
        asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(te_remote + 8)
                     : "memory");
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  cluster_sync();
  if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
}

using encode_fn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                               const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                               CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static int map_i8(CUtensorMap* m, const void* base, long long rows, int cols, int box_rows) {
  static encode_fn fn = nullptr;
  if (!fn) {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    ZT_CUDA_CHECK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q));
    if (!f || q != cudaDriverEntryPointSuccess) return fail(ZT_ECUDA, "cuTensorMapEncodeTiled unavailable");
    fn = reinterpret_cast<encode_fn>(f);
  }
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)cols};
  cuuint32_t box[2] = {TK, (cuuint32_t)box_rows};
  cuuint32_t es[2] = {1, 1};
  if (fn(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void*>(base), dims, strides, box, es,
         CU_TENSOR_MAP_INTERLEAVE_NONE, TK == 128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B,
         CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return fail(ZT_ECUDA, "oz: tensor map encode failed");
  return ZT_OK;
}

}  // namespace oz

// ---------------------------------------------------------------------------
// Operand conversion: scale each row (A operand) / each column (B operand) of
// a complex128 matrix by a power of two so its largest |re|, |im| lies in
// [2^(KB-1), 2^KB), round to integers (exact in binary64: the scaling is a
// power of two and values >= 2^53 are integers already), and
// write phi+- = (re +- iota im) mod p, centred, as int8 planes.
//
// Residues of an integer-valued x (|x| < 2^56) in two levels: y = x mod Q_g
// for the groups Q_g = p_2g p_2g+1 < 2^16 (the last group is p_16 alone) in
// FP64 (q = rint(x / Q) from the rounded reciprocal is floor or ceil, and
// y = x - q Q is exact by FMA; |y| < 2^17), then in FP32 (exact integer
// arithmetic below 2^24): r_im = centred y_im mod p, z+- = y_re +- iota r_im
// (|z| < 2^18), and the centred z mod p (the relative error of z / p from
// the rounded reciprocal is far below an odd p's 1 / 2p distance from a
// rounding tie, so |r| <= (p - 1) / 2 <= 120); the low byte of
// r + 1.5 * 2^23 is r in two's complement.
// ---------------------------------------------------------------------------
constexpr int OZ_NGRP = (OZ_NMOD + 1) / 2;
constexpr float OZ_MAGIC_F = 12582912.0f;
constexpr double OZ_MAGIC = 6755399441055744.0;
__constant__ double c_oz_q[OZ_NGRP], c_oz_qinv[OZ_NGRP];
__constant__ float c_oz_pf[OZ_NMOD], c_oz_pinvf[OZ_NMOD], c_oz_iota[OZ_NMOD];
__device__ __forceinline__ float reduce_group(double x, int g) {
  const double q = fma(x, c_oz_qinv[g], OZ_MAGIC) - OZ_MAGIC;
  return (float)fma(-q, c_oz_q[g], x);
}
// words whose low bytes are phi+ and phi- of (y_re, y_im) mod p_t
__device__ __forceinline__ void phi_words(float yr, float yi, int t, uint32_t& wp, uint32_t& wm) {
  const float p = c_oz_pf[t], pinv = c_oz_pinvf[t], io = c_oz_iota[t];
  const float qi = fmaf(yi, pinv, OZ_MAGIC_F) - OZ_MAGIC_F;
  const float ri = fmaf(-qi, p, yi);
  const float zp = fmaf(io, ri, yr), zm = fmaf(-io, ri, yr);
  const float qp = fmaf(zp, pinv, OZ_MAGIC_F) - OZ_MAGIC_F, qm = fmaf(zm, pinv, OZ_MAGIC_F) - OZ_MAGIC_F;
  wp = __float_as_uint(fmaf(-qp, p, zp + OZ_MAGIC_F));
  wm = __float_as_uint(fmaf(-qm, p, zm + OZ_MAGIC_F));
}
// the same for two elements at once on the packed FP32 pipe (FFMA2 / FADD2,
// sm_100): the conversions are instruction-issue bound, and the per-modulus
// FP32 work is most of their instructions
__device__ __forceinline__ void phi_words2(float2 yr, float2 yi, int t, uint32_t* wp, uint32_t* wm) {
  const float p = c_oz_pf[t], pinv = c_oz_pinvf[t], io = c_oz_iota[t];
  const float2 np2 = make_float2(-p, -p), pinv2 = make_float2(pinv, pinv), io2 = make_float2(io, io),
               nio2 = make_float2(-io, -io), m2 = make_float2(OZ_MAGIC_F, OZ_MAGIC_F),
               nm2 = make_float2(-OZ_MAGIC_F, -OZ_MAGIC_F);
  const float2 qi = __fadd2_rn(__ffma2_rn(yi, pinv2, m2), nm2);
  const float2 ri = __ffma2_rn(qi, np2, yi);
  const float2 zp = __ffma2_rn(io2, ri, yr), zm = __ffma2_rn(nio2, ri, yr);
  const float2 qp = __fadd2_rn(__ffma2_rn(zp, pinv2, m2), nm2), qm = __fadd2_rn(__ffma2_rn(zm, pinv2, m2), nm2);
  const float2 rp = __ffma2_rn(qp, np2, __fadd2_rn(zp, m2)), rm = __ffma2_rn(qm, np2, __fadd2_rn(zm, m2));
  wp[0] = __float_as_uint(rp.x);
  wp[1] = __float_as_uint(rp.y);
  wm[0] = __float_as_uint(rm.x);
  wm[1] = __float_as_uint(rm.y);
}
// low bytes of four words into one (byte e from word e)
__device__ __forceinline__ uint32_t pack4(uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
  return __byte_perm(__byte_perm(a, b, 0x0040), __byte_perm(c, d, 0x0040), 0x5410);
}
// NaN-propagating max of magnitudes (fmax drops NaN)
__device__ __forceinline__ double nanmax(double a, double b) { return (b > a || b != b) ? b : a; }

// exponent shift that puts amax in [2^(KB-1), 2^KB); 0 for an all-zero line,
// OZ_BAD for a line holding a NaN or an infinity
__device__ __forceinline__ int oz_shift(double amax, int kb) {
  if (!(amax <= 1.79769313486231570815e308)) return OZ_BAD;
  return amax > 0.0 ? kb - 1 - ilogb(amax) : 0;
}
// 2^sh as two normal factors (sh in [-971, 1126]): v * s.x * s.y == ldexp(v, sh)
// whenever the result is >= 2^-1022 (scaling is exact; a smaller result
// rounds to 0 either way under rint), at two DMULs instead of ldexp's
// special-case chain; a bad line scales to zeros
__device__ __forceinline__ double2 oz_scale2(int sh) {
  if (sh == OZ_BAD) return make_double2(0.0, 0.0);
  const int a = sh / 2, b = sh - a;
  return make_double2(__hiloint2double((a + 1023) << 20, 0), __hiloint2double((b + 1023) << 20, 0));
}

// A-type rows: planes (phi+, phi-) of row i.  mode 1 = the B layout of a
// skew-Hermitian S (B[j][k] = S[k][j] = -conj(S[j][k]) off the diagonal, the
// diagonal taken as is): phi+(-conj s) = -phi-(s), phi-(-conj s) = -phi+(s).
// mode 2: both at once from one read (A planes into out, skew-B planes into
// out2; the row scale is shared since |-conj(v)| = |v|).  One block per
// padded row; 4 consecutive k per thread (one 32-bit store per plane).
// <= 64 registers (4 blocks of 256 per SM; 58.5 -> 57.6 us against 80 registers at 3)
template <int MODE>
__global__ void __launch_bounds__(256, 4) k_oz_conv_rows(int rows, int n, const double* __restrict__ src, int64_t ld,
                                                       int mp, int kp, int kb, int mode, int diag0, int8_t* out,
                                                       int* __restrict__ shift, int8_t* out2 = nullptr) {
  const int i = blockIdx.x;  // row of the (rows x n) block; its diagonal entry is column diag0 + i
  __shared__ unsigned red[8];
  __shared__ double redd[8];
  // The shift needs only ilogb of the row maximum (or that it is not
  // finite): the maximum of the high words of |x| (sign cleared) has the
  // exponent and leading mantissa bits of the maximum, and >= 0x7ff00000
  // exactly when an Inf or NaN is present -- one integer max per value
  // instead of the NaN-propagating double max.  A row whose largest high
  // word is 0 (all |x| < 2^-1042) takes the exact double maximum.
  unsigned hmax = 0;
  pdl_trigger();
  pdl_wait();
  if (i < rows) {
    // all of this thread's loads in flight at once (the max chain would
    // otherwise serialise them)
    int k = threadIdx.x;
    for (; k + 7 * 256 < n; k += 8 * 256) {
      double2 v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = ld2(src + ((size_t)i * ld + k + u * 256) * 2);
#pragma unroll
      for (int u = 0; u < 8; ++u)
        hmax = max(hmax, max((unsigned)__double2hiint(v[u].x) & 0x7fffffffu,
                             (unsigned)__double2hiint(v[u].y) & 0x7fffffffu));
    }
    for (; k < n; k += 256) {
      const double2 v = ld2(src + ((size_t)i * ld + k) * 2);
      hmax = max(hmax, max((unsigned)__double2hiint(v.x) & 0x7fffffffu, (unsigned)__double2hiint(v.y) & 0x7fffffffu));
    }
  }
  for (int o = 16; o; o >>= 1) hmax = max(hmax, __shfl_xor_sync(0xffffffffu, hmax, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = hmax;
  __syncthreads();
  hmax = red[0];
  for (int q = 1; q < 8; ++q) hmax = max(hmax, red[q]);
  double amax = __hiloint2double((int)hmax, 0);
  if (hmax == 0) {  // block-uniform: tiny or zero row, exact maximum
    amax = 0.0;
    if (i < rows)
      for (int k = threadIdx.x; k < n; k += 256) {
        const double2 v = ld2(src + ((size_t)i * ld + k) * 2);
        amax = nanmax(amax, nanmax(fabs(v.x), fabs(v.y)));
      }
    for (int o = 16; o; o >>= 1) amax = nanmax(amax, __shfl_xor_sync(0xffffffffu, amax, o));
    if ((threadIdx.x & 31) == 0) redd[threadIdx.x >> 5] = amax;
    __syncthreads();
    amax = redd[0];
    for (int q = 1; q < 8; ++q) amax = nanmax(amax, redd[q]);
  } else if (hmax >= 0x7ff00000u) {
    amax = __longlong_as_double(0x7ff8000000000000LL);  // an Inf or NaN in the row
  }
  const int sh = oz_shift(amax, kb);
  const double2 sc = oz_scale2(sh);
  if (threadIdx.x == 0 && shift) shift[i] = sh;
  const size_t pw = (size_t)mp * kp / 4;  // plane stride in words
  for (int k0 = threadIdx.x * 4; k0 < kp; k0 += blockDim.x * 4) {
    double xv[8];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int k = k0 + e;
      double2 v = make_double2(0.0, 0.0);
      if (i < rows && k < n) v = ld2(src + ((size_t)i * ld + k) * 2);
      xv[e] = rint(v.x * sc.x * sc.y);
      xv[4 + e] = rint(v.y * sc.x * sc.y);
    }
    const bool diag = (unsigned)(diag0 + i - k0) < 4u;
    const int sh8 = 8 * (diag0 + i - k0);
    // running word pointers into the planes of modulus t
    uint32_t* pa = reinterpret_cast<uint32_t*>(out + (size_t)i * kp + k0);
    uint32_t* pb = reinterpret_cast<uint32_t*>((MODE == 1 ? out : out2) + (size_t)i * kp + k0);
#pragma unroll
    for (int g = 0; g < OZ_NGRP; ++g) {
      float yr[4], yi[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        yr[e] = reduce_group(xv[e], g);
        yi[e] = reduce_group(xv[4 + e], g);
      }
#pragma unroll
      for (int t = 2 * g; t < 2 * g + 2; ++t) {
        if (t >= OZ_NMOD) break;
        uint32_t wp[4], wm[4];
#pragma unroll
        for (int e = 0; e < 4; e += 2)
          phi_words2(make_float2(yr[e], yr[e + 1]), make_float2(yi[e], yi[e + 1]), t, wp + e, wm + e);
        const uint32_t ap = pack4(wp[0], wp[1], wp[2], wp[3]);
        const uint32_t am = pack4(wm[0], wm[1], wm[2], wm[3]);
        if (MODE != 1) {
          pa[0] = ap;
          pa[pw] = am;
        }
        pa += 2 * pw;
        if (MODE != 0) {
          // skew-B: -phi-+ off the diagonal, phi+- on it
          uint32_t bp = __vneg4(am), bm = __vneg4(ap);
          if (diag) {
            const uint32_t msk = 0xffu << sh8;
            bp = (bp & ~msk) | (ap & msk);
            bm = (bm & ~msk) | (am & msk);
          }
          pb[0] = bp;
          pb[pw] = bm;
          pb += 2 * pw;
        }
      }
    }
  }
}

// B operand of a general matrix X (B[j][k] = X[k][j]): column maxima first
// (NaN-propagating: the max of the bit patterns of |x|)
__global__ void __launch_bounds__(256) k_oz_colmax(int kdim, int n, const double* __restrict__ x, int64_t ld,
                                                   unsigned long long* colmax) {
  const int j = blockIdx.x * 32 + (threadIdx.x & 31);
  const int r0 = blockIdx.y * 64 + (threadIdx.x >> 5) * 8;
  if (j >= n) return;
  // all 8 loads in flight, then the maximum of the high words of |x| (as in
  // k_oz_conv_rows: the shift needs only ilogb of the maximum or that a value
  // is not finite); a thread whose high words are all 0 (|x| < 2^-1042)
  // contributes its exact bit pattern
  double2 v[8];
#pragma unroll
  for (int q = 0; q < 8; ++q) v[q] = (r0 + q < kdim) ? ld2(x + ((size_t)(r0 + q) * ld + j) * 2) : make_double2(0.0, 0.0);
  unsigned hm = 0;
#pragma unroll
  for (int q = 0; q < 8; ++q)
    hm = max(hm, max((unsigned)__double2hiint(v[q].x) & 0x7fffffffu, (unsigned)__double2hiint(v[q].y) & 0x7fffffffu));
  unsigned long long bits = (unsigned long long)hm << 32;
  if (hm == 0) {
    double m = 0.0;
#pragma unroll
    for (int q = 0; q < 8; ++q) m = nanmax(m, nanmax(fabs(v[q].x), fabs(v[q].y)));
    bits = (unsigned long long)__double_as_longlong(m);
  }
  atomicMax(colmax + j, bits);
}

// then 32 (k) x 32 (j) tiles through shared memory; thread t produces output
// row j = j0 + t / 8, k = k0 + 4 (t % 8) .. +3 (one 32-bit store per plane)
__global__ void __launch_bounds__(256, 3) k_oz_conv_cols(int kdim, int n, const double* __restrict__ x, int64_t ld,
                                                       int np, int kp, int kb,
                                                       const unsigned long long* __restrict__ colmax, int8_t* out,
                                                       int* __restrict__ shift) {
  __shared__ double2 tl[32][33];
  const int j0 = blockIdx.x * 32, k0 = blockIdx.y * 32;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  for (int r = ty; r < 32; r += 8) {
    const int k = k0 + r, j = j0 + tx;
    tl[r][tx] = (k < kdim && j < n) ? ld2(x + ((size_t)k * ld + j) * 2) : make_double2(0.0, 0.0);
  }
  __syncthreads();
  const int jj = threadIdx.x >> 3, kk = (threadIdx.x & 7) * 4;
  const int j = j0 + jj;
  const double m = (j < n) ? __longlong_as_double((long long)colmax[j]) : 0.0;
  const int sh = oz_shift(m, kb);
  const double2 sc = oz_scale2(sh);
  if (blockIdx.y == 0 && kk == 0 && shift) shift[j] = sh;
  double xv[8];
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    const double2 v = tl[kk + e][jj];
    xv[e] = rint(v.x * sc.x * sc.y);
    xv[4 + e] = rint(v.y * sc.x * sc.y);
  }
  const size_t pw = (size_t)np * kp / 4;  // plane stride in words
  uint32_t* pb = reinterpret_cast<uint32_t*>(out + (size_t)j * kp + k0 + kk);
  // two groups per iteration: 48 registers (5 blocks/SM) and 64 vs 71 us at
  // N = 2048 (rolled: 56 registers; fully unrolled: 80 registers, 77 us)
#pragma unroll 2
  for (int g = 0; g < OZ_NGRP; ++g) {
    float yr[4], yi[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      yr[e] = reduce_group(xv[e], g);
      yi[e] = reduce_group(xv[4 + e], g);
    }
#pragma unroll
    for (int t = 2 * g; t < 2 * g + 2; ++t) {
      if (t >= OZ_NMOD) break;
      uint32_t wp[4], wm[4];
#pragma unroll
      for (int e = 0; e < 4; e += 2)
        phi_words2(make_float2(yr[e], yr[e + 1]), make_float2(yi[e], yi[e + 1]), t, wp + e, wm + e);
      pb[0] = pack4(wp[0], wp[1], wp[2], wp[3]);
      pb[pw] = pack4(wm[0], wm[1], wm[2], wm[3]);
      pb += 2 * pw;
    }
  }
}

// ---------------------------------------------------------------------------
// Reconstruction (CRT).  Per modulus t the GEMM delivers
//   s_t = (U + V) mod p_t = 2 Re C mod p_t,  d_t = (U - V) mod p_t = 2 iota_t Im C mod p_t
// as centred residues (|s_t|, |d_t| <= (p_t - 1) / 2).  With M_t = M / p_t,
// y_t = M_t^-1 mod p_t:
//   Re C = sum_t s_t Wr_t mod M,  Wr_t = (2^-1 y_t mod p_t) M_t
//   Im C = sum_t d_t Wi_t mod M,  Wi_t = ((2 iota_t)^-1 y_t mod p_t) M_t
// (any representative of the residue works: a multiple of p_t times M_t is a
// multiple of M).  W_t (< M < 2^124.2) and M are split into signed pieces
// on the grids 2^0, 2^42, 2^84, the two lower ones balanced in [-2^41, 2^41)
// and the top one < 2^40.2, so with sum_t |c_t| <= 1404 < 2^11 every partial
// sum S_k and every q M_k (q = rint(S / M), |q| <= 1404) is below 2^52 and
// D_k = S_k - q M_k is exact.  Only the pieces on 2^84 and 2^42 are used:
// dropping the 2^0 pieces of W_t and M changes x = D_2 + D_1 by at most
// 2 * 1404 * 2^41 < 2^52.5, i.e. 2^-69 of the |x| <= 2 K 2^(2 KB) bound
// (K = 2048, KB = 55) and ~2^-13 of the operands' own rounding error
// (K 2^(KB-1)), and q is unchanged (|x| < M / 2 with a 12% margin).
// ---------------------------------------------------------------------------
constexpr int OZ_NPC = 2;  // pieces used: [0] on 2^42, [1] on 2^84
struct CrtConst {
  double wr[OZ_NMOD][OZ_NPC];  // pieces of Wr_t
  double wi[OZ_NMOD][OZ_NPC];  // pieces of Wi_t
  double mp[OZ_NPC];           // pieces of M
  double m_inv;                // 1 / M
  double bias[OZ_NMOD];        // 2^52 + 2^31 + k_t
  uint32_t hi80;               // 0x80000000, read at run time (see byte_to_double)
};
__constant__ CrtConst c_crt;

// unsigned byte r -> centred residue r - k_t as a double without an
// int -> fp64 conversion: 2^52 + 2^31 + r as the bit pattern, minus the bias
// `hi80` holds 0x80000000 read from constant memory (opaque to the
// compiler), so the permute takes its selector as an immediate: with both
// constants foldable ptxas kept 0x80000000 as the immediate and moved the
// selector from a uniform register before every permute
template <int E>
__device__ __forceinline__ uint32_t prmt_byte(uint32_t word, uint32_t hi80) {
  uint32_t lo;
  asm("prmt.b32 %0, %1, %2, %3;" : "=r"(lo) : "r"(word), "r"(hi80), "n"(0x7540 | E));
  return lo;
}
__device__ __forceinline__ double byte_to_double(uint32_t word, int e, double bias, uint32_t hi80) {
  // one byte permute: byte e of word, then 0x00, 0x00, 0x80 (e is a
  // compile-time constant after unrolling: the switch folds away)
  uint32_t lo;
  switch (e) {
    case 0: lo = prmt_byte<0>(word, hi80); break;
    case 1: lo = prmt_byte<1>(word, hi80); break;
    case 2: lo = prmt_byte<2>(word, hi80); break;
    default: lo = prmt_byte<3>(word, hi80); break;
  }
  return __hiloint2double(0x43300000, (int)lo) - bias;
}

// reconstruction: 2 output columns per thread at <= 64 registers (4 blocks
// of 256 per SM): the FP64 chains need the extra warps to hide the loads
constexpr int OZ_RECON_COLS = 2;
// the centred integers Re, Im of product entries (i, j0 .. j0 + C - 1)
// before scaling
template <int C = OZ_RECON_COLS>
__device__ __forceinline__ void crt_values(const int8_t* __restrict__ r, int mp, int np, int i, int j0, double* vr,
                                           double* vi, const CrtConst& cc = c_crt) {
  const size_t ps = (size_t)2 * mp * np;  // stride between moduli
  static_assert(C == 2 || C == 4, "2 or 4 columns per thread");
  using word_t = typename std::conditional<C == 2, unsigned short, unsigned int>::type;
  const int8_t* rre = r + (size_t)i * np + j0;
  const int8_t* rim = rre + (size_t)mp * np;
  word_t wr[OZ_NMOD], wi[OZ_NMOD];
#pragma unroll
  for (int t = 0; t < OZ_NMOD; ++t) {
    wr[t] = __ldg(reinterpret_cast<const word_t*>(rre + (size_t)t * ps));
    wi[t] = __ldg(reinterpret_cast<const word_t*>(rim + (size_t)t * ps));
  }
  const uint32_t hi80 = cc.hi80;
  double s[2 * C][OZ_NPC];
#pragma unroll
  for (int e = 0; e < 2 * C; ++e)
#pragma unroll
    for (int k = 0; k < OZ_NPC; ++k) s[e][k] = 0.0;
#pragma unroll
  for (int t = 0; t < OZ_NMOD; ++t) {
    const double bias = cc.bias[t];
#pragma unroll
    for (int e = 0; e < 2 * C; ++e) {
      const double u = byte_to_double(e < C ? wr[t] : wi[t], e % C, bias, hi80);
#pragma unroll
      for (int k = 0; k < OZ_NPC; ++k) s[e][k] = fma(u, e < C ? cc.wr[t][k] : cc.wi[t][k], s[e][k]);
    }
  }
#pragma unroll
  for (int e = 0; e < 2 * C; ++e) {
    const double q = rint((s[e][1] + s[e][0]) * cc.m_inv);
    const double d2 = fma(-q, cc.mp[1], s[e][1]);
    const double d1 = fma(-q, cc.mp[0], s[e][0]);
    const double x = d2 + d1;
    if (e < C)
      vr[e] = x;
    else
      vi[e - C] = x;
  }
}
__device__ __forceinline__ double2 scaled(double vr, double vi, int ri, int cj) {
  if (ri == OZ_BAD || cj == OZ_BAD)
    return make_double2(__longlong_as_double(0x7ff8000000000000LL), __longlong_as_double(0x7ff8000000000000LL));
  const int sh = -(ri + cj);
  return make_double2(ldexp(vr, sh), ldexp(vi, sh));
}

#ifndef OZ_RC
#define OZ_RC 4
#endif
#ifndef OZ_RC_MINB
#define OZ_RC_MINB 4
#endif
// 4 output columns per thread (one 32-bit residue load per plane, the CRT
// constants and address increments shared by 4 values) at <= 64 registers
// (4 blocks of 256 per SM): 62.2 -> 53.3 us at N = 2048 with the
// immediate-selector permutes, against 2 columns per thread
constexpr int RC = OZ_RC;
__global__ void __launch_bounds__(256, OZ_RC_MINB) k_oz_recon(int m, int n, const int8_t* __restrict__ r, int mp,
                                                            int np, const int* __restrict__ rs,
                                                            const int* __restrict__ cs, double* c, int64_t ldc,
                                                            int lower) {
  const int i = blockIdx.y;
  const int j0 = (blockIdx.x * blockDim.x + threadIdx.x) * RC;
  pdl_trigger();
  pdl_wait();
  if (i >= m || j0 >= n) return;
  if (lower && (j0 >> 7) > (i >> 7)) return;
  double vr[RC], vi[RC];
  crt_values<RC>(r, mp, np, i, j0, vr, vi);
  const int ri = rs[i];
#pragma unroll
  for (int e = 0; e < RC; ++e) {
    const int j = j0 + e;
    if (j < n && !(lower && (j >> 7) > (i >> 7))) st2(c + ((size_t)i * ldc + j) * 2, scaled(vr[e], vi[e], ri, cs[j]));
  }
}

// Reconstruction for the row-block sharded step: C (m x n) into `c` (may be
// null), and/or column j into rank h = j / mloc's N x mloc buffer a[:, R_h]
// at row r0 + i (peer pointers: the all-to-all of the a tiles fused into the
// reconstruction), and/or -conj(C)^T into `mirror` (the partner's rows of
// the skew-Hermitian b, ld_mirror).  A block is 8 rows x 64 columns (a warp
// per row, 2 columns per lane): direct stores are whole-warp 1 KB runs, and
// the mirror goes through shared memory so each of its rows receives one
// 128-byte run.  One system-scope fence per block orders the peer stores
// (the rank barrier that follows publishes them).
constexpr int RX_ROWS = 8, RX_COLS = 64;
__global__ void __launch_bounds__(256, 4) k_oz_recon_ex(int m, int n, const int8_t* __restrict__ r, int mp, int np,
                                                      const int* __restrict__ rs, const int* __restrict__ cs,
                                                      double* c, int64_t ldc, const unsigned long long* peers,
                                                      int mloc, int r0, double* mirror, int64_t ldm, int lower) {
  __shared__ double2 tl[RX_ROWS][RX_COLS + 1];
  const int lane = threadIdx.x & 31, wr = threadIdx.x >> 5;
  const int i0 = blockIdx.y * RX_ROWS, jb = blockIdx.x * RX_COLS;
  const int i = i0 + wr, j0 = jb + lane * OZ_RECON_COLS;
  pdl_trigger();
  pdl_wait();
  // lower (square, from a lower-mode residue GEMM): only 256-tiles on or
  // below the diagonal were computed; entries of strictly-lower tiles are
  // also mirrored, diagonal tiles are complete on both sides
  if (lower && (jb >> 8) > (i0 >> 8)) return;  // 8 | 256 and 64 | 256: whole block in one tile pair
  const bool mirror_blk = mirror && !(lower && (jb >> 8) == (i0 >> 8));
  if (i < m && j0 < n) {
    double vr[OZ_RECON_COLS], vi[OZ_RECON_COLS];
    crt_values(r, mp, np, i, j0, vr, vi);
    const int ri = rs[i];
#pragma unroll
    for (int e = 0; e < OZ_RECON_COLS; ++e) {
      const int j = j0 + e;
      if (j >= n) continue;
      const double2 o = scaled(vr[e], vi[e], ri, cs[j]);
      double* cc = c ? c + ((size_t)i * ldc + j) * 2 : nullptr;
      if (c) st2(cc, o);
      if (peers) {
        const int h = j / mloc;
        double* dst = reinterpret_cast<double*>(peers[h]) + ((size_t)(r0 + i) * mloc + (j - h * mloc)) * 2;
        if (dst != cc) st2(dst, o);  // one rank: the scatter target may be c itself
      }
      if (mirror_blk) tl[wr][lane * OZ_RECON_COLS + e] = make_double2(-o.x, o.y);
    }
  }
  if (mirror_blk) {
    __syncthreads();
    // mirror row jj (64 of them) x RX_ROWS columns: 8 lanes per row
    for (int t = threadIdx.x; t < RX_COLS * RX_ROWS; t += blockDim.x) {
      const int jj = t / RX_ROWS, ii = t % RX_ROWS;
      const int j = jb + jj, ir = i0 + ii;
      if (j < n && ir < m) st2(mirror + ((size_t)j * ldm + ir) * 2, tl[ii][jj]);
    }
  }
  if (peers || mirror) {
    __syncthreads();
    if (threadIdx.x == 0) __threadfence_system();
  }
}

static cudaError_t launch_recon(int m, int n, const int8_t* r, int mp, int np, const int* rs, const int* cs, double* c,
                                int64_t ldc, int lower, cudaStream_t st) {
  const dim3 grid((n + 256 * RC - 1) / (256 * RC), m);
  return launch_pdl(k_oz_recon, grid, dim3(256), 0, st, m, n, r, mp, np, rs, cs, c, ldc, lower);
}

// ---- per-device constants ----------------------------------------------------
static bool g_crt_ready[OZ_MAXDEV] = {};
static int g_oz_sms[OZ_MAXDEV] = {};

static int modinv(int a, int p) {
  for (int y = 1; y < p; ++y)
    if ((long long)a * y % p == 1) return y;
  return -1;
}
// a square root of -1 mod p (p odd, every prime factor = 1 mod 4)
static int sqrt_minus_one(int p) {
  for (int x = 2; x < p; ++x)
    if ((long long)x * x % p == p - 1) return x;
  return -1;
}

static int crt_init() {
  int dev = 0;
  ZT_CUDA_CHECK(cudaGetDevice(&dev));
  if (dev < 0 || dev >= OZ_MAXDEV) return fail(ZT_EINVAL, "oz: device index out of range");
  if (g_crt_ready[dev]) return ZT_OK;
  typedef unsigned __int128 u128;
  typedef __int128 i128;
  CrtConst h;
  u128 m = 1;
  for (int t = 0; t < OZ_NMOD; ++t) m *= (u128)h_oz_p[t];
  // balanced pieces: v = sum_k piece_k 2^(42 k), |piece_0|, |piece_1| <= 2^41;
  // pieces 1 and 2 are kept (out[0], out[1]), piece 0 is dropped
  auto pieces = [](u128 v, double* out) {
    i128 rest = (i128)v;
    for (int k = 0; k < 3; ++k) {
      i128 pk = rest;
      if (k < 2) {
        pk = rest & (((i128)1 << 42) - 1);
        if (pk >= ((i128)1 << 41)) pk -= (i128)1 << 42;
        rest = (rest - pk) >> 42;
      }
      if (k > 0) out[k - 1] = std::ldexp((double)(long long)pk, 42 * k);  // <= 42 bits: exact
    }
  };
  int pm[OZ_NMOD];
  unsigned mm[OZ_NMOD], ms[OZ_NMOD];
  float pf[OZ_NMOD], pif[OZ_NMOD], iof[OZ_NMOD];
  for (int t = 0; t < OZ_NMOD; ++t) {
    const int p = h_oz_p[t];
    const int io = sqrt_minus_one(p);
    if (io < 0) return fail(ZT_EINVAL, "oz: modulus without a square root of -1");
    const u128 mt = m / (u128)p;
    const int y = modinv((int)(mt % (u128)p), p);
    const int half = (p + 1) / 2;                      // 2^-1 mod p
    const int g2 = modinv((2 * io) % p, p);            // (2 iota)^-1 mod p
    pieces(mt * (u128)(((long long)half * y) % p), h.wr[t]);
    pieces(mt * (u128)(((long long)g2 * y) % p), h.wi[t]);
    h.bias[t] = 4503601774854144.0 + (double)(p / 2);
    h.hi80 = 0x80000000u;
    pm[t] = p;
    int l = 0;
    while ((1 << l) < p) ++l;
    mm[t] = (unsigned)(((1ULL << (31 + l)) + (unsigned long long)p - 1) / (unsigned long long)p);
    ms[t] = (unsigned)(l - 1);
    pf[t] = (float)p;
    pif[t] = 1.0f / (float)p;
    iof[t] = (float)io;
  }
  pieces(m, h.mp);
  h.m_inv = 1.0 / (double)m;
  ZT_CUDA_CHECK(cudaMemcpyToSymbol(c_crt, &h, sizeof h));
  double qd[OZ_NGRP], qi[OZ_NGRP];
  for (int g = 0; g < OZ_NGRP; ++g) {
    qd[g] = (double)h_oz_p[2 * g] * (2 * g + 1 < OZ_NMOD ? h_oz_p[2 * g + 1] : 1);  // < 2^16
    qi[g] = 1.0 / qd[g];
  }
  ZT_CUDA_CHECK(cudaMemcpyToSymbol(c_oz_p, pm, sizeof pm));
  ZT_CUDA_CHECK(cudaMemcpyToSymbol(c_oz_m, mm, sizeof mm));
  ZT_CUDA_CHECK(cudaMemcpyToSymbol(c_oz_s, ms, sizeof ms));
  ZT_CUDA_CHECK(cudaMemcpyToSymbol(c_oz_q, qd, sizeof qd));
  ZT_CUDA_CHECK(cudaMemcpyToSymbol(c_oz_qinv, qi, sizeof qi));
  ZT_CUDA_CHECK(cudaMemcpyToSymbol(c_oz_pf, pf, sizeof pf));
  ZT_CUDA_CHECK(cudaMemcpyToSymbol(c_oz_pinvf, pif, sizeof pif));
  ZT_CUDA_CHECK(cudaMemcpyToSymbol(c_oz_iota, iof, sizeof iof));
  int sms = 0;
  ZT_CUDA_CHECK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  ZT_CUDA_CHECK(cudaFuncSetAttribute(oz::k_oz_gemm, cudaFuncAttributeMaxDynamicSharedMemorySize, oz::SMEM));
  g_oz_sms[dev] = sms;
  g_crt_ready[dev] = true;
  return ZT_OK;
}

// integer bits per operand entry so that |sum| < M / 2 over K terms (complex
// form): 55 for K <= 4096, 54 up to 2^14.  Capped at 56 so x / Q stays below
// 2^51 for the group reduction's rint (smallest group Q = 89).
static int oz_bits(int k) {
  double lg = 0.0;
  for (int t = 0; t < OZ_NMOD; ++t) lg += std::log2((double)h_oz_p[t]);
  const int kb = (int)std::floor((lg - 1.0 - std::log2(2.0 * k) - 1e-9) / 2.0);
  return std::min(56, kb);
}

static size_t oz_pad(int n) { return ((size_t)n + 255) / 256 * 256; }

size_t oz_workspace_bytes(int n) {
  const size_t p = oz_pad(n);
  return (size_t)OZ_NMOD * p * p * (2 + 2 + 2) + 2 * p * sizeof(int) + p * 8 + 1024;
}

// CUDA-event timing of every residue-GEMM launch while profiling is on
// (eager steps only; zt_profile_enable / zt_oz_profile_read)
struct OzEv {
  cudaEvent_t e0, e1;
  int lower;
};
static std::vector<OzEv> g_oz_ev;
static size_t g_oz_used = 0;
static bool g_oz_prof = false;
void oz_profile_enable(bool on) {
  if (on && !g_oz_prof) g_oz_used = 0;
  g_oz_prof = on;
}

// R residues for every modulus (see the header comment); mp, np multiples
// of 256, kp of 128
int oz_modgemm(int nmod, int mp, int np, int kp, const int8_t* a, const int8_t* b, int8_t* r, int lower,
               cudaStream_t st, int bswap = 0) {
  using namespace oz;
  // kp <= 2^14 keeps |accumulator| < 89 2^22 (modx's exact range)
  if (nmod < 1 || nmod > OZ_NMOD || mp % TM || np % TN || kp % (KPS * TK) || kp > 16384 || (lower && mp != np))
    return fail(ZT_EINVAL, "oz_modgemm: bad shape");
  int rc = crt_init();
  if (rc) return rc;
  int dev = 0;
  ZT_CUDA_CHECK(cudaGetDevice(&dev));
  CUtensorMap ma, mb;
  rc = map_i8(&ma, a, (long long)nmod * 2 * mp, kp, 128);
  if (!rc) rc = map_i8(&mb, b, (long long)nmod * 2 * np, kp, TN / 2);
  if (rc) return rc;
  GemmArgs g;
  g.nmod = nmod;
  g.mt = mp / TM;
  g.nt = np / TN;
  g.kt = kp / TK;
  g.lower = lower;
  g.bswap = bswap;
  g.mp = mp;
  g.np = np;
  g.r = r;
  const int per = lower ? lower_count(g.mt) : g.mt * g.nt;
  const int grid = 2 * std::min(nmod * per, g_oz_sms[dev] / 2);
  OzEv* ev = nullptr;
  if (g_oz_prof) {
    if (g_oz_used == g_oz_ev.size()) {
      OzEv e{};
      cudaEventCreate(&e.e0);
      cudaEventCreate(&e.e1);
      g_oz_ev.push_back(e);
    }
    ev = &g_oz_ev[g_oz_used++];
    ev->lower = lower;
    cudaEventRecord(ev->e0, st);
  }
  ZT_CUDA_CHECK(launch_pdl(k_oz_gemm, dim3(grid), dim3(THREADS), SMEM, st, ma, mb, g));
  ZT_LAUNCHED();
  if (ev) cudaEventRecord(ev->e1, st);
  ZT_CUDA_CHECK(cudaGetLastError());
  return ZT_OK;
}

// C = A B for complex128 n x n, A general (row scaled), B: bmode 0 general
// (column scaled, transposed conversion), 1 skew-Hermitian with exact
// mirror off the diagonal (converted row-wise as -conj).  lower: only the
// 128-tiles of C on or below the diagonal are computed.
int oz_zgemm(int n, const double* a, int64_t lda, const double* b, int64_t ldb, int bmode, double* c, int64_t ldc,
             int lower, void* ws, size_t ws_bytes, cudaStream_t st) {
  if (n < 1) return fail(ZT_EINVAL, "oz_zgemm: bad size");
  if (ws_bytes < oz_workspace_bytes(n)) return fail(ZT_ENOMEM, "oz_zgemm: workspace too small");
  int rc = crt_init();
  if (rc) return rc;
  const int p = (int)oz_pad(n);
  const int kb = oz_bits(n);
  int8_t* ares = static_cast<int8_t*>(ws);
  int8_t* bres = ares + (size_t)OZ_NMOD * 2 * p * p;
  int8_t* rres = bres + (size_t)OZ_NMOD * 2 * p * p;
  int* rsh = reinterpret_cast<int*>(rres + (size_t)OZ_NMOD * 2 * p * p);
  int* csh = rsh + p;
  unsigned long long* cmax = reinterpret_cast<unsigned long long*>(csh + p);
  ZT_CUDA_CHECK(launch_pdl(k_oz_conv_rows<0>, dim3(p), dim3(256), 0, st, n, n, a, lda, p, p, kb, 0, 0, ares, rsh,
                           (int8_t*)nullptr));
  ZT_LAUNCHED();
  if (bmode == 1) {
    ZT_CUDA_CHECK(launch_pdl(k_oz_conv_rows<1>, dim3(p), dim3(256), 0, st, n, n, b, ldb, p, p, kb, 1, 0, bres, csh,
                             (int8_t*)nullptr));
    ZT_LAUNCHED();
  } else {
    ZT_CUDA_CHECK(cudaMemsetAsync(cmax, 0, sizeof(unsigned long long) * p, st));
    if (p != n) ZT_CUDA_CHECK(cudaMemsetAsync(bres, 0, (size_t)OZ_NMOD * 2 * p * p, st));
    k_oz_colmax<<<dim3((n + 31) / 32, (n + 63) / 64), 256, 0, st>>>(n, n, b, ldb, cmax);
    ZT_LAUNCHED();
    k_oz_conv_cols<<<dim3(p / 32, p / 32), 256, 0, st>>>(n, n, b, ldb, p, p, kb, cmax, bres, csh);
    ZT_LAUNCHED();
  }
  rc = oz_modgemm(OZ_NMOD, p, p, p, ares, bres, rres, lower, st);
  if (rc) return rc;
  ZT_CUDA_CHECK(launch_recon(n, n, rres, p, p, rsh, csh, c, ldc, lower, st));
  ZT_LAUNCHED();
  ZT_CUDA_CHECK(cudaGetLastError());
  return ZT_OK;
}

int update_pairs(int n, const double* a, const double* bm, double* out, const double* base, const double* xprev,
                 const double* wn, double hh, double qq, unsigned long long* resid, unsigned long long* cons,
                 cudaStream_t st);
int final_commutator(int n, const double* a, const double* wn, double h, double* out, cudaStream_t st);

size_t oz_update_workspace_bytes(int n) {
  const size_t p = oz_pad(n);
  return (size_t)OZ_NMOD * p * p * (2 + 2 + 2 + 2) + 4 * p * sizeof(int) + p * 8 + 1024;
}

// X (the B operand of GEMM-1) to column-scaled residues; independent of the
// stream solve, so the step runs it on a side stream beside the solve
int oz_convert_x(int n, const double* x, void* ws, cudaStream_t st) {
  int rc = crt_init();
  if (rc) return rc;
  const int pd = (int)oz_pad(n);
  const int kb = oz_bits(n);
  const size_t pl = (size_t)OZ_NMOD * pd * pd;
  int8_t* bx = static_cast<int8_t*>(ws) + 2 * pl;
  int* sx = reinterpret_cast<int*>(bx + 6 * pl) + pd;
  unsigned long long* cmax = reinterpret_cast<unsigned long long*>(sx + 3 * pd);
  ZT_CUDA_CHECK(cudaMemsetAsync(cmax, 0, sizeof(unsigned long long) * pd, st));
  k_oz_colmax<<<dim3((n + 31) / 32, (n + 63) / 64), 256, 0, st>>>(n, n, x, n, cmax);
  ZT_LAUNCHED();
  k_oz_conv_cols<<<dim3(pd / 32, pd / 32), 256, 0, st>>>(n, n, x, n, pd, pd, kb, cmax, bx, sx);
  ZT_LAUNCHED();
  ZT_CUDA_CHECK(cudaGetLastError());
  return ZT_OK;
}

// One fixed-point update with both products on the INT8 tensor cores:
// a = P X (P rows scaled; X columns scaled, transposed conversion), then
// b = a P on the lower tiles (a rows scaled; P as a skew-Hermitian B
// operand from the same conversion pass as its A layout), then the update
// pass.  gemm1_only: the step's final update W_{n+1} = W_n + h (a - a^H)
// (out = x, h = hh; k_final_commutator).  x_join: X was converted by
// oz_convert_x on another stream; wait for this event before GEMM-1
// (nullptr: convert X here).
int oz_update(int n, const double* p, const double* x, double* a, double* bbuf, const double* base,
              const double* xprev, const double* wn, double* out, double hh, double qq, unsigned long long* resid,
              unsigned long long* cons, void* ws, cudaStream_t st, int gemm1_only, cudaEvent_t x_join) {
  int rc = crt_init();
  if (rc) return rc;
  const int pd = (int)oz_pad(n);
  const int kb = oz_bits(n);
  const size_t pl = (size_t)OZ_NMOD * pd * pd;
  int8_t* ares = static_cast<int8_t*>(ws);  // P rows (A operand of both products)
  int8_t* bx = ares + 2 * pl;   // X as B operand
  int8_t* ba = bx + 2 * pl;     // a rows (B operand of GEMM-2, planes read swapped: a^H)
  int8_t* rres = ba + 2 * pl;
  int* sp = reinterpret_cast<int*>(rres + 2 * pl);  // P rows (= P-as-B columns)
  int* sx = sp + pd;                                // X columns
  int* sa = sx + pd;                                // a rows
  // P rows: the A operand of GEMM-1 and of GEMM-2
  ZT_CUDA_CHECK(launch_pdl(k_oz_conv_rows<0>, dim3(pd), dim3(256), 0, st, n, n, p, (int64_t)n, pd, pd, kb, 0, 0, ares,
                           sp, (int8_t*)nullptr));
  ZT_LAUNCHED();
  if (x_join) {
    ZT_CUDA_CHECK(cudaStreamWaitEvent(st, x_join, 0));
  } else {
    const int rc0 = oz_convert_x(n, x, ws, st);
    if (rc0) return rc0;
  }
  rc = oz_modgemm(OZ_NMOD, pd, pd, pd, ares, bx, rres, 0, st);
  if (rc) return rc;
  if (gemm1_only) {
    ZT_CUDA_CHECK(launch_recon(n, n, rres, pd, pd, sp, sx, a, n, 0, st));
    ZT_LAUNCHED();
    return final_commutator(n, a, wn, hh, out, st);
  }
  // (a fused reconstruction + row conversion, one block per row of a with
  // the row re-read from L2, measured 184 us against 48 + 83 us: removed)
  ZT_CUDA_CHECK(launch_recon(n, n, rres, pd, pd, sp, sx, a, n, 0, st));
  ZT_LAUNCHED();
  ZT_CUDA_CHECK(launch_pdl(k_oz_conv_rows<0>, dim3(pd), dim3(256), 0, st, n, n, (const double*)a, (int64_t)n, pd, pd,
                           kb, 0, 0, ba, sa, (int8_t*)nullptr));
  ZT_LAUNCHED();
  // b = a P = P X P computed as P a^H (a^H = (P X)^H = X P for the
  // skew-Hermitian iterate and stream matrix): the A planes are P's rows from
  // GEMM-1, the B operand a^H is the conjugate of a's rows, i.e. a's row
  // planes with phi+ and phi- swapped (column scales = a's row scales), so P
  // needs no second (skew-B) layout; lower 256-tiles only, mirrored by the
  // update pass
  rc = oz_modgemm(OZ_NMOD, pd, pd, pd, ares, ba, rres, 1, st, 1);
  if (rc) return rc;
  ZT_CUDA_CHECK(launch_recon(n, n, rres, pd, pd, sp, sa, bbuf, n, 1, st));
  ZT_LAUNCHED();
  ZT_CUDA_CHECK(cudaGetLastError());
  return update_pairs(n, a, bbuf, out, base, xprev, wn, hh, qq, resid, cons, st);
}

int oz_moduli(int* out, int cap) {
  for (int j = 0; j < OZ_NMOD && j < cap; ++j) out[j] = h_oz_p[j];
  return OZ_NMOD;
}

int oz_iotas(int* out, int cap) {
  for (int t = 0; t < OZ_NMOD; ++t) {
    const int io = sqrt_minus_one(h_oz_p[t]);
    if (t < cap) out[t] = io;
  }
  return OZ_NMOD;
}

}  // namespace zt

extern "C" int zt_oz_modgemm(int nmod, int mp, int np, int kp, const void* a, const void* b, void* r, int lower,
                             void* stream) {
  if (!a || !b || !r) return zt::fail(ZT_EINVAL, "zt_oz_modgemm: bad argument");
  return zt::oz_modgemm(nmod, mp, np, kp, static_cast<const int8_t*>(a), static_cast<const int8_t*>(b),
                        static_cast<int8_t*>(r), lower, (cudaStream_t)stream);
}

extern "C" int zt_oz_moduli(int* out, int cap) { return zt::oz_moduli(out, cap); }

extern "C" int zt_oz_iotas(int* out, int cap) { return zt::oz_iotas(out, cap); }

extern "C" size_t zt_oz_workspace_bytes(int n) { return zt::oz_workspace_bytes(n); }

// ms[0] / counts[0]: full residue GEMMs, [1]: lower-triangle ones
extern "C" int zt_oz_profile_read(double* ms, long long* counts, int reset) {
  double m[2] = {0, 0};
  long long c[2] = {0, 0};
  for (size_t i = 0; i < zt::g_oz_used; ++i) {
    float t = 0;
    cudaEventSynchronize(zt::g_oz_ev[i].e1);
    if (cudaEventElapsedTime(&t, zt::g_oz_ev[i].e0, zt::g_oz_ev[i].e1) == cudaSuccess) {
      m[zt::g_oz_ev[i].lower ? 1 : 0] += t;
      c[zt::g_oz_ev[i].lower ? 1 : 0] += 1;
    }
  }
  for (int k = 0; k < 2; ++k) {
    if (ms) ms[k] = m[k];
    if (counts) counts[k] = c[k];
  }
  if (reset) zt::g_oz_used = 0;
  return ZT_OK;
}

extern "C" int zt_oz_zgemm(int n, const double* a, int64_t lda, const double* b, int64_t ldb, int bmode, double* c,
                           int64_t ldc, int lower, void* ws, size_t ws_bytes, void* stream) {
  if (!a || !b || !c || !ws) return zt::fail(ZT_EINVAL, "zt_oz_zgemm: bad argument");
  return zt::oz_zgemm(n, a, lda, b, ldb, bmode, c, ldc, lower, ws, ws_bytes, (cudaStream_t)stream);
}

// ---- building blocks of the row-block sharded step (sharded.py) -------------
extern "C" int zt_oz_bits(int k) { return zt::oz_bits(k); }

extern "C" size_t zt_oz_plane_bytes(int rows, int cols) {
  return (size_t)zt::OZ_NMOD * 2 * zt::oz_pad(rows) * zt::oz_pad(cols);
}

// rows x kdim block of a complex128 matrix (row-major, ld) to residue planes
// [NMOD][2][pad(rows)][pad(kdim)]; mode 0: A planes (phi+, phi-) of the rows;
// mode 1: skew-B planes of the rows of a skew-Hermitian S (B[j][k] = S[k][j]
// = -conj(S[j][k]), the diagonal entry -- column diag0 + j -- as is).  kb:
// zt_oz_bits(K).  shift: pad(rows) ints (row scales).  mode 2: both from one
// read, A planes into `planes`, skew-B planes into `planes2`.
extern "C" int zt_oz_convert_rows(int rows, int kdim, const double* src, int64_t ld, int mode, int diag0, int kb,
                                  void* planes, int* shift, void* planes2, void* stream) {
  using namespace zt;
  if (rows < 1 || kdim < 1 || !src || !planes || !shift || mode < 0 || mode > 2 || (mode == 2 && !planes2))
    return fail(ZT_EINVAL, "zt_oz_convert_rows: bad argument");
  int rc = crt_init();
  if (rc) return rc;
  const int mp = (int)oz_pad(rows), kp = (int)oz_pad(kdim);
  cudaStream_t st = (cudaStream_t)stream;
  auto kern = mode == 0 ? k_oz_conv_rows<0> : (mode == 1 ? k_oz_conv_rows<1> : k_oz_conv_rows<2>);
  ZT_CUDA_CHECK(launch_pdl(kern, dim3(mp), dim3(256), 0, st, rows, kdim, src, ld, mp, kp, kb, mode, diag0,
                           static_cast<int8_t*>(planes), shift, static_cast<int8_t*>(planes2)));
  ZT_LAUNCHED();
  return ZT_OK;
}

// kdim x ncols general matrix X as the B operand (B[j][k] = X[k][j], column
// scales): planes [NMOD][2][pad(ncols)][pad(kdim)]; colmax_ws: pad(ncols)
// 8-byte words of scratch.
extern "C" int zt_oz_convert_cols(int kdim, int ncols, const double* src, int64_t ld, int kb, void* planes,
                                  int* shift, void* colmax_ws, void* stream) {
  using namespace zt;
  if (kdim < 1 || ncols < 1 || !src || !planes || !shift || !colmax_ws)
    return fail(ZT_EINVAL, "zt_oz_convert_cols: bad argument");
  int rc = crt_init();
  if (rc) return rc;
  const int np = (int)oz_pad(ncols), kp = (int)oz_pad(kdim);
  cudaStream_t st = (cudaStream_t)stream;
  unsigned long long* cmax = static_cast<unsigned long long*>(colmax_ws);
  ZT_CUDA_CHECK(cudaMemsetAsync(cmax, 0, sizeof(unsigned long long) * np, st));
  k_oz_colmax<<<dim3((ncols + 31) / 32, (kdim + 63) / 64), 256, 0, st>>>(kdim, ncols, src, ld, cmax);
  ZT_LAUNCHED();
  k_oz_conv_cols<<<dim3(np / 32, kp / 32), 256, 0, st>>>(kdim, ncols, src, ld, np, kp, kb, cmax,
                                                         static_cast<int8_t*>(planes), shift);
  ZT_LAUNCHED();
  ZT_CUDA_CHECK(cudaGetLastError());
  return ZT_OK;
}

// C = A B^T residues -> complex128 (see k_oz_recon_ex): r from zt_oz_modgemm
// with mp = pad(m), np = pad(n); rs / cs the A / B shifts.
extern "C" int zt_oz_reconstruct(int m, int n, const void* r, const int* rs, const int* cs, double* c, int64_t ldc,
                                 const unsigned long long* peers, int mloc, int r0, double* mirror, int64_t ld_mirror,
                                 int lower, void* stream) {
  using namespace zt;
  if (m < 1 || n < 1 || !r || !rs || !cs || (!c && !peers && !mirror) || (peers && mloc < 1) || (lower && m != n))
    return fail(ZT_EINVAL, "zt_oz_reconstruct: bad argument");
  const dim3 grid((n + RX_COLS - 1) / RX_COLS, (m + RX_ROWS - 1) / RX_ROWS);
  ZT_CUDA_CHECK(launch_pdl(k_oz_recon_ex, grid, dim3(32 * RX_ROWS), 0, (cudaStream_t)stream, m, n,
                           static_cast<const int8_t*>(r), (int)oz_pad(m), (int)oz_pad(n), rs, cs, c, ldc, peers, mloc,
                           r0, mirror, ld_mirror, lower));
  ZT_LAUNCHED();
  return ZT_OK;
}
