// FP64-accurate complex GEMM on the INT8 tensor cores (Ozaki scheme II):
// operands are scaled to integers (row / column power-of-two scales, up to
// 53 significant bits), reduced modulo NMOD pairwise-coprime moduli <= 128,
// multiplied exactly per modulus by tcgen05 kind::i8 MMAs with int32
// accumulation (4M complex form: Re = Ar Br + (-Ai) Bi, Im = Ar Bi + Ai Br),
// reduced again modulo p in the epilogue, and reassembled by the Chinese
// remainder theorem into the exact integer product, then scaled back.
// 16 pairwise-coprime moduli <= 256 (M ~ 2^125.4): 53-bit operands up to
// K = 16384 with the 4M sum bound 2 K 2^106 < M / 2.
//
// Layouts (int8, zero padded to 128 in every dimension):
//   A residues [NMOD][3][Mp][Kp]  planes re, im, -im   (K-major rows)
//   B residues [NMOD][2][Np][Kp]  planes re, im        (K-major: B^T rows)
//   R residues [NMOD][2][Mp][Np]  (Re, Im of the product + floor(p_j / 2)) mod p_j,
//                                 unsigned bytes in [0, p_j)
#include <cuda.h>

#include <algorithm>
#include <cmath>
#include <type_traits>
#include <vector>

#include "zt_common.cuh"
#include "zt_tma.cuh"

namespace zt {

constexpr int OZ_NMOD = 16;
// pairwise coprime (256 = 2^8, 255 = 3 5 17, 253 = 11 23, 247 = 13 19,
// 217 = 7 31, the rest prime), product ~ 2^125.4; centred residues fit int8
__constant__ int c_oz_p[OZ_NMOD] = {256, 255, 253, 251, 247, 241, 239, 233, 229, 227, 223, 217, 211, 199, 197, 193};
// floor(2^32 / p)
__constant__ unsigned c_oz_m[OZ_NMOD] = {16777216, 16843009, 16976155, 17111423, 17388531, 17821441,
                                         17970574, 18433336, 18755315, 18920560, 19259943, 19792476,
                                         20355295, 21582750, 21801864, 22253716};
static const int h_oz_p[OZ_NMOD] = {256, 255, 253, 251, 247, 241, 239, 233, 229, 227, 223, 217, 211, 199, 197, 193};

namespace oz {

#ifndef OZ_TN
#define OZ_TN 256
#endif
// 128 x TN output tiles: TN = 256 halves the B-operand L2 traffic per MMA
// (the kernel is L2-bandwidth bound at TN = 128) at the price of a single
// TMEM accumulator buffer (Re + Im = 2 TN columns of 512)
// K stages of 64 bytes (64 B swizzle) so four stages fit: with two 128-byte
// stages the TMA latency of a stage exceeded the MMA time of the other
constexpr int TM = 128, TN = OZ_TN, TK = 64;  // TK in bytes
constexpr int NBUF = 512 / (2 * TN);         // TMEM accumulator buffers
constexpr int TILE_BYTES = 128 * TK;         // one 128-row int8 tile (A)
constexpr int B_TILE_BYTES = TN * TK;
constexpr int STAGE_BYTES = 3 * TILE_BYTES + 2 * B_TILE_BYTES;  // A re, im, -im; B re, im
constexpr int STAGES = 4;
#ifndef OZ_EPI_WARPS
#define OZ_EPI_WARPS 8
#endif
constexpr int EPI_WARPS = OZ_EPI_WARPS;  // EPI_WARPS / 4 per TMEM lane quarter, each a column group
constexpr int THREADS = (2 + EPI_WARPS) * 32;
constexpr int SMEM = STAGES * STAGE_BYTES + 1024 + 256;

__device__ __forceinline__ void mbar_arrive_tx(uint64_t* b, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive1(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void tma2d(void* dst, const CUtensorMap* map, int c0, int c1, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], "
      "[%4];" ::"r"(smem_u32(dst)),
      "l"(map), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}
// UMMA smem descriptor: K-major, 64 B swizzle, 8-row groups 512 B apart
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr) {
  return (uint64_t)((saddr & 0x3FFFF) >> 4) | ((uint64_t)1 << 16) | ((uint64_t)(512 >> 4) << 32) |
         ((uint64_t)1 << 46) | ((uint64_t)4 << 61);
}
// D s32, A/B signed int8, K-major, M = 128, N = 128
constexpr uint32_t IDESC = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(TN >> 3) << 17) |
                           ((uint32_t)(TM >> 4) << 24);

__device__ __forceinline__ void mma(uint32_t d, uint64_t a, uint64_t b, uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(d),
      "l"(a), "l"(b), "r"(IDESC), "r"(acc));
}
__device__ __forceinline__ void commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
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
  int nmod, mt, nt, kt;  // tiles per dimension (128 rows, TN columns) and K blocks (128 B)
  int lower;             // square: only tiles meeting the lower 128-block triangle
  int mp, np;            // padded M, N (output leading dimension np)
  int8_t* r;             // [nmod][2][mp][np]
};

// lower mode: tile (tm, tn) is needed iff its columns reach 128-block tm,
// i.e. tn * TN / 128 <= tm
__host__ __device__ __forceinline__ int lower_count(int mt) {
  int c = 0;
  for (int tm = 0; tm < mt; ++tm) c += tm * TM / TN + 1;
  return c;
}
__device__ __forceinline__ void work_of(const GemmArgs& g, int w, int per, int& j, int& tm, int& tn) {
  j = w / per;
  int t = w - j * per;
  if (g.lower) {
    tm = 0;
    while (t >= tm * TM / TN + 1) {
      t -= tm * TM / TN + 1;
      ++tm;
    }
    tn = t;
  } else {
    tm = t % g.mt;
    tn = t / g.mt;
  }
}

// (v + floor(p / 2)) mod p in [0, p) for an int32 accumulator v
// (|v| <= 2 K 128^2 <= 2^29 for K <= 16384): u = v + p 2^23 + floor(p / 2)
// lies in (0, 2^32); Barrett quotient from the high word of u floor(2^32 / p)
// (floor(u / p) or one less), one correction; integer pipe only.  The
// reconstruction subtracts floor(p / 2) again (centred residues, |c| <= 128).
__device__ __forceinline__ int modc(int v, int p, unsigned m) {
  const unsigned u = (unsigned)v + ((unsigned)p << 23) + ((unsigned)p >> 1);
  const unsigned r = u - __umulhi(u, m) * (unsigned)p;
  return (int)(r >= (unsigned)p ? r - p : r);
}

__global__ void __launch_bounds__(THREADS, 1)
    k_oz_gemm(const __grid_constant__ CUtensorMap ma, const __grid_constant__ CUtensorMap mb, GemmArgs g) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + NBUF;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + NBUF);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int per = g.lower ? lower_count(g.mt) : g.mt * g.nt;
  const int total = g.nmod * per;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int s = 0; s < NBUF; ++s) {
      mbar_init(&tfull[s], 1);
      mbar_init(&tempty[s], EPI_WARPS);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = *tmem_slot;
  if (warp == 0 && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(&ma) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&mb) : "memory");
  }
  pdl_trigger();
  pdl_wait();  // operands from the conversions; R still read by the previous reconstruction

  if (warp == 0) {
    if (lane == 0) {
      unsigned it = 0;
      for (int w = blockIdx.x; w < total; w += gridDim.x) {
        int j, tm, tn;
        work_of(g, w, per, j, tm, tn);
        const int ra = (j * 3) * g.mp + tm * TM, rb = (j * 2) * g.np + tn * TN;
        for (int kb = 0; kb < g.kt; ++kb, ++it) {
          const int s = it % STAGES;
          mbar_wait(&empty[s], ((it / STAGES) & 1) ^ 1);
          unsigned char* st = smem + s * STAGE_BYTES;
          mbar_arrive_tx(&full[s], STAGE_BYTES);
          tma2d(st, &ma, kb * TK, ra, &full[s]);
          tma2d(st + TILE_BYTES, &ma, kb * TK, ra + g.mp, &full[s]);
          tma2d(st + 2 * TILE_BYTES, &ma, kb * TK, ra + 2 * g.mp, &full[s]);
          tma2d(st + 3 * TILE_BYTES, &mb, kb * TK, rb, &full[s]);
          tma2d(st + 3 * TILE_BYTES + B_TILE_BYTES, &mb, kb * TK, rb + g.np, &full[s]);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      unsigned it = 0, lt = 0;
      for (int w = blockIdx.x; w < total; w += gridDim.x, ++lt) {
        const int ab = lt % NBUF;
        mbar_wait(&tempty[ab], ((lt / NBUF) & 1) ^ 1);
        asm volatile("tcgen05.fence::after_thread_sync;");
        const uint32_t dre = tmem + ab * 2 * TN, dim = dre + TN;
        for (int kb = 0; kb < g.kt; ++kb, ++it) {
          const int s = it % STAGES;
          mbar_wait(&full[s], (it / STAGES) & 1);
          asm volatile("tcgen05.fence::after_thread_sync;");
          const uint32_t base = smem_u32(smem + s * STAGE_BYTES);
          const uint32_t are = base, aim = base + TILE_BYTES, anim = base + 2 * TILE_BYTES;
          const uint32_t bre = base + 3 * TILE_BYTES, bim = bre + B_TILE_BYTES;
#pragma unroll
          for (int k = 0; k < TK / 32; ++k) {
            const uint32_t first = (kb | k) ? 1u : 0u;
            const uint32_t o = k * 32;
            mma(dre, sdesc(are + o), sdesc(bre + o), first);
            mma(dre, sdesc(anim + o), sdesc(bim + o), 1u);
            mma(dim, sdesc(are + o), sdesc(bim + o), first);
            mma(dim, sdesc(aim + o), sdesc(bre + o), 1u);
          }
          commit(&empty[s]);
        }
        commit(&tfull[ab]);
      }
    }
  } else {
    const int q = warp & 3;                  // TMEM lane quarter = tile rows q*32 ..
    constexpr int CW = TN / (EPI_WARPS / 4);      // columns per warp
    const int ch = ((warp - 2) >> 2) * CW;        // column group
    unsigned lt = 0;
    for (int w = blockIdx.x; w < total; w += gridDim.x, ++lt) {
      int j, tm, tn;
      work_of(g, w, per, j, tm, tn);
      const int ab = lt % NBUF;
      mbar_wait(&tfull[ab], (lt / NBUF) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;");
      const int p = c_oz_p[j];
      const unsigned pm = c_oz_m[j];
      const int row = tm * TM + q * 32 + lane;
      int8_t* rre = g.r + ((size_t)(j * 2) * g.mp + row) * g.np + tn * TN;
      int8_t* rim = rre + (size_t)g.mp * g.np;
#ifdef OZ_EXP_NOEPI
      if (p == 12345)
#endif
#pragma unroll 1
      for (int c0 = ch; c0 < ch + CW; c0 += 32) {
        uint32_t v[32], u[32];
        const uint32_t ta = tmem + ((uint32_t)(q * 32) << 16) + ab * 2 * TN + c0;
        OZ_LD32(v, ta);
        OZ_LD32(u, ta + TN);
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        uint32_t pk[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          uint32_t x = 0;
#pragma unroll
          for (int b = 0; b < 4; ++b) x |= ((uint32_t)(modc((int)v[4 * e + b], p, pm) & 0xff)) << (8 * b);
          pk[e] = x;
        }
        uint4* d = reinterpret_cast<uint4*>(rre + c0);
        d[0] = make_uint4(pk[0], pk[1], pk[2], pk[3]);
        d[1] = make_uint4(pk[4], pk[5], pk[6], pk[7]);
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          uint32_t x = 0;
#pragma unroll
          for (int b = 0; b < 4; ++b) x |= ((uint32_t)(modc((int)u[4 * e + b], p, pm) & 0xff)) << (8 * b);
          pk[e] = x;
        }
        d = reinterpret_cast<uint4*>(rim + c0);
        d[0] = make_uint4(pk[0], pk[1], pk[2], pk[3]);
        d[1] = make_uint4(pk[4], pk[5], pk[6], pk[7]);
      }
      asm volatile("tcgen05.fence::before_thread_sync;");
      __syncwarp();
      if (lane == 0) mbar_arrive1(&tempty[ab]);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
}

}  // namespace oz

// ---------------------------------------------------------------------------
// CTA-pair kernel (cta_group::2, the default): the complex product as two
// real products with K doubled, Re = [Ar | -Ai] [Br ; Bi] and
// Im = [Ai | Ar] [Br ; Bi], so a work item is ONE real 256 x 256 tile (Re or
// Im of a pair tile) with a single 256-column accumulator per CTA: the TMEM
// accumulators double-buffer and the mod-p epilogue of one item overlaps the
// MMAs of the next (the single-CTA kernel's Re + Im fill TMEM and its
// epilogue stalls the tensor pipe).  Each CTA of the pair loads 128 rows of
// the A plane and 128 of the 256 B columns per stage; the leader's single
// thread issues M = 256, N = 256 MMAs over both CTAs' shared memory, so every
// SM runs 128 x 256 x 32 MMAs (the full-rate shape) at 8 operand KB per
// million MACs.  No re-layout: the K halves read the existing re / im / -im
// planes.
// ---------------------------------------------------------------------------
namespace oz2 {
constexpr int TM = 256, TN = 256, TK = oz::TK;  // pair tile; TK in bytes
constexpr int A_BYTES = 128 * TK;               // one CTA's 128 rows of an A plane
constexpr int B_BYTES = (TN / 2) * TK;          // one CTA's 128 columns of a B plane
#ifndef OZ2_KPS
#define OZ2_KPS 2  // K blocks per pipeline stage (amortises the MMA thread's barrier work)
#endif
constexpr int KPS = OZ2_KPS;
constexpr int STAGE_BYTES = KPS * (A_BYTES + B_BYTES);  // [A kb0 | B kb0 | A kb1 | B kb1 ...]
#ifndef OZ2_STAGES
#define OZ2_STAGES (12 / OZ2_KPS)
#endif
constexpr int STAGES = OZ2_STAGES;
constexpr int NBUF = 2;  // TMEM accumulator buffers of TN columns
constexpr int EPI_WARPS = 8;
constexpr int THREADS = (2 + EPI_WARPS) * 32;
constexpr int SMEM = STAGES * STAGE_BYTES + 1024 + 256;
// D s32, A/B signed int8, K-major, M = 256 (pair), N = 256
constexpr uint32_t IDESC = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(TN >> 3) << 17) |
                           ((uint32_t)(TM >> 4) << 24);

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
__device__ __forceinline__ void mbar_wait_cluster(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
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
// arrive on the barrier at this offset in both CTAs once the issued MMAs finish
__device__ __forceinline__ void commit_both(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_u32(bar)),
      "h"((unsigned short)3)
      : "memory");
}

// work item w -> modulus j, part (0 Re, 1 Im), pair tile (tm, tn); lower
// mode: the 256 x 256 tiles meeting the lower 128-block triangle (tn <= tm)
__host__ __device__ __forceinline__ int lower_count(int mt) { return mt * (mt + 1) / 2; }
__device__ __forceinline__ void pair_work_of(const oz::GemmArgs& g, int w, int per, int& j, int& part, int& tm,
                                             int& tn) {
  j = w / (2 * per);
  int t = w - j * 2 * per;
  part = t & 1;
  t >>= 1;
  if (g.lower) {
    tm = 0;
    while (t > tm) {
      t -= tm + 1;
      ++tm;
    }
    tn = t;
  } else {
    tm = t % g.mt;
    tn = t / g.mt;
  }
}

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(THREADS, 1)
    k_oz_gemm2(const __grid_constant__ CUtensorMap ma, const __grid_constant__ CUtensorMap mb, oz::GemmArgs g) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + NBUF;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + NBUF);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_rank();
  const int cl = blockIdx.x >> 1, ncl = gridDim.x >> 1;
  const int per = g.lower ? lower_count(g.mt) : g.mt * g.nt;
  const int total = g.nmod * 2 * per;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int s = 0; s < NBUF; ++s) {
      mbar_init(&tfull[s], 1);
      mbar_init(&tempty[s], 2 * EPI_WARPS);  // leader's: both CTAs' epilogue warps
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

  if (warp == 0) {
    if (lane == 0) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(&ma) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(&mb) : "memory");
      const uint32_t fb0 = mapa(smem_u32(&full[0]), 0);
      unsigned it = 0;
      for (int w = cl; w < total; w += ncl) {
        int j, part, tm, tn;
        pair_work_of(g, w, per, j, part, tm, tn);
        // K half 0: A plane re (Re) / im (Im) with B re; half 1: -im (Re) / re (Im) with B im
        const int ra0 = (j * 3 + part) * g.mp + tm * TM + rank * 128;
        const int ra1 = (j * 3 + (part ? 0 : 2)) * g.mp + tm * TM + rank * 128;
        const int rb0 = (j * 2) * g.np + tn * TN + rank * (TN / 2), rb1 = rb0 + g.np;
        for (int kb = 0; kb < 2 * g.kt; kb += KPS, ++it) {
          const int s = it % STAGES;
          mbar_wait(&empty[s], ((it / STAGES) & 1) ^ 1);
          unsigned char* st = smem + s * STAGE_BYTES;
          if (rank == 0) oz::mbar_arrive_tx(&full[s], 2 * STAGE_BYTES);
#pragma unroll
          for (int u = 0; u < KPS; ++u) {
            const int kbu = kb + u;
            const bool h1 = kbu >= g.kt;
            const int kc = (h1 ? kbu - g.kt : kbu) * TK;
            unsigned char* su = st + u * (A_BYTES + B_BYTES);
            tma2d_pair(su, &ma, kc, h1 ? ra1 : ra0, fb0 + s * 8);
            tma2d_pair(su + A_BYTES, &mb, kc, h1 ? rb1 : rb0, fb0 + s * 8);
          }
        }
      }
      // drain: every issued stage consumed before this CTA may exit
      for (int i = 0; i < STAGES; ++i, ++it) mbar_wait(&empty[it % STAGES], ((it / STAGES) & 1) ^ 1);
    }
  } else if (warp == 1) {
    if (lane == 0 && rank == 0) {
      unsigned it = 0, lt = 0;
      for (int w = cl; w < total; w += ncl, ++lt) {
        const int ab = lt % NBUF;
        mbar_wait_cluster(&tempty[ab], ((lt / NBUF) & 1) ^ 1);
        asm volatile("tcgen05.fence::after_thread_sync;");
        const uint32_t d = tmem + ab * TN;
        for (int kb = 0; kb < 2 * g.kt; kb += KPS, ++it) {
          const int s = it % STAGES;
          mbar_wait(&full[s], (it / STAGES) & 1);
          asm volatile("tcgen05.fence::after_thread_sync;");
#pragma unroll
          for (int u = 0; u < KPS; ++u) {
            const uint32_t a = smem_u32(smem + s * STAGE_BYTES + u * (A_BYTES + B_BYTES)), b = a + A_BYTES;
#pragma unroll
            for (int k = 0; k < TK / 32; ++k)
              mma(d, oz::sdesc(a + k * 32), oz::sdesc(b + k * 32), (kb | u | k) ? 1u : 0u);
          }
          commit_both(&empty[s]);
        }
        commit_both(&tfull[ab]);
      }
    }
  } else {
    const int q = warp & 3;                       // TMEM lane quarter = tile rows q*32 ..
    const int ch = ((warp - 2) >> 2) * (TN / 2);  // column half
    const uint32_t te_remote = mapa(smem_u32(&tempty[0]), 0);
    unsigned lt = 0;
    for (int w = cl; w < total; w += ncl, ++lt) {
      int j, part, tm, tn;
      pair_work_of(g, w, per, j, part, tm, tn);
      const int ab = lt % NBUF;
      mbar_wait(&tfull[ab], (lt / NBUF) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;");
      const int p = c_oz_p[j];
      const unsigned pm = c_oz_m[j];
      const int row = tm * TM + rank * 128 + q * 32 + lane;
      int8_t* out = g.r + ((size_t)(j * 2 + part) * g.mp + row) * g.np + tn * TN;
#pragma unroll 1
      for (int c0 = ch; c0 < ch + TN / 2; c0 += 64) {
        uint32_t v[32], u[32];
        const uint32_t ta = tmem + ((uint32_t)(q * 32) << 16) + ab * TN + c0;
        OZ_LD32(v, ta);
        OZ_LD32(u, ta + 32);
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        uint32_t pk[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          uint32_t x = 0;
#pragma unroll
          for (int b = 0; b < 4; ++b) x |= ((uint32_t)(oz::modc((int)v[4 * e + b], p, pm) & 0xff)) << (8 * b);
          pk[e] = x;
        }
        uint4* dst = reinterpret_cast<uint4*>(out + c0);
        dst[0] = make_uint4(pk[0], pk[1], pk[2], pk[3]);
        dst[1] = make_uint4(pk[4], pk[5], pk[6], pk[7]);
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          uint32_t x = 0;
#pragma unroll
          for (int b = 0; b < 4; ++b) x |= ((uint32_t)(oz::modc((int)u[4 * e + b], p, pm) & 0xff)) << (8 * b);
          pk[e] = x;
        }
        dst[2] = make_uint4(pk[0], pk[1], pk[2], pk[3]);
        dst[3] = make_uint4(pk[4], pk[5], pk[6], pk[7]);
      }
      asm volatile("tcgen05.fence::before_thread_sync;");
      __syncwarp();
      if (lane == 0)
        asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(te_remote + ab * 8)
                     : "memory");
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  cluster_sync();
  if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
}
}  // namespace oz2

namespace oz {
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
         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return fail(ZT_ECUDA, "oz: tensor map encode failed");
  return ZT_OK;
}

}  // namespace oz

int oz_modgemm(int nmod, int mp, int np, int kp, const int8_t* a, const int8_t* b, int8_t* r, int lower,
               cudaStream_t st);

// ---------------------------------------------------------------------------
// Operand conversion: scale each row (A operand) / each column (B operand) of
// a complex128 matrix by a power of two so its largest |re|, |im| lies in
// [2^(KB-1), 2^KB), round to integers (exact in binary64 for KB <= 53), and
// write the centred residues mod every p_j as int8 planes.  Residues come
// from 18-bit limbs of |x| in 32-bit integer arithmetic (Barrett reduction),
// not from FP64 divisions.
// ---------------------------------------------------------------------------
// Residues of an integer-valued x (|x| < 2^53) for all 16 moduli in two
// levels: y = x mod Q_g for the eight pairs Q_g = p_2g p_2g+1 < 2^16 in FP64
// (q = rint(x / Q) from the rounded reciprocal is floor or ceil, and
// y = x - q Q is exact by FMA; |y| < 2^17), then the centred y mod p in FP32
// (exact integer arithmetic in a float; the relative error 2^-23 of y / p
// is far below the 1 / 2p distance of an odd p's quotient from a rounding
// tie, so |r| <= (p - 1) / 2, and p = 256 divides exactly: r in [-128, 128],
// whose byte is right mod 256); the low byte of r + 1.5 * 2^23 is r in two's
// complement.
constexpr int OZ_NGRP = OZ_NMOD / 2;
constexpr double OZ_MAGIC = 6755399441055744.0;
constexpr float OZ_MAGIC_F = 12582912.0f;
__constant__ double c_oz_q[OZ_NGRP], c_oz_qinv[OZ_NGRP];
__constant__ float c_oz_pf[OZ_NMOD], c_oz_pinvf[OZ_NMOD];
__device__ __forceinline__ float reduce_pair(double x, int g) {
  const double q = fma(x, c_oz_qinv[g], OZ_MAGIC) - OZ_MAGIC;
  return (float)fma(-q, c_oz_q[g], x);
}
// residue of y as the low byte of the returned word (yM = y + 1.5 * 2^23,
// exact for |y| < 2^22): r + 1.5 * 2^23 = fma(-q, p, yM)
__device__ __forceinline__ uint32_t res_word_f(float y, float yM, int t) {
  const float q = fmaf(y, c_oz_pinvf[t], OZ_MAGIC_F) - OZ_MAGIC_F;
  return __float_as_uint(fmaf(-q, c_oz_pf[t], yM));
}
// low bytes of four words into one (byte e from word e)
__device__ __forceinline__ uint32_t pack4(uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
  return __byte_perm(__byte_perm(a, b, 0x0040), __byte_perm(c, d, 0x0040), 0x5410);
}

// exponent shift that puts amax in [2^(KB-1), 2^KB); 0 for an all-zero line
__device__ __forceinline__ int oz_shift(double amax, int kb) { return amax > 0.0 ? kb - 1 - ilogb(amax) : 0; }
// 2^sh as two normal factors (sh in [-971, 1126]): v * s.x * s.y == ldexp(v, sh)
// whenever the result is >= 2^-1022 (scaling is exact; a smaller result
// rounds to 0 either way under rint), at two DMULs instead of ldexp's
// special-case chain
__device__ __forceinline__ double2 oz_scale2(int sh) {
  const int a = sh / 2, b = sh - a;
  return make_double2(__hiloint2double((a + 1023) << 20, 0), __hiloint2double((b + 1023) << 20, 0));
}

// A-type rows: planes (re, im, -im) of row i; mode 1 = the B layout of a
// skew-Hermitian S (B[j][k] = S[k][j] = -conj(S[j][k]) off the diagonal):
// planes (re, im) of that.  One block per padded row; 4 consecutive k per
// thread (one 32-bit store per plane).
// mode 2: both at once from one read (A planes into out, skew-B planes into
// out2; the row scale is shared since |-conj(v)| = |v|).
// conversions: <= 80 registers (3 blocks of 256 per SM) measured 5% faster
#ifndef OZ_CONV_MINB
#define OZ_CONV_MINB 3
#endif
// reconstruction: 2 output columns per thread at <= 64 registers (4 blocks
// of 256 per SM) measured 2% faster per step than 4 columns at 106
// registers (the FP64 chains need the extra warps to hide the loads)
#ifndef OZ_RECON_MINB
#define OZ_RECON_MINB 4
#endif
#ifndef OZ_RECON_COLS
#define OZ_RECON_COLS 2  // output columns per thread (4 or 2)
#endif
__global__ void __launch_bounds__(256, OZ_CONV_MINB) k_oz_conv_rows(int n, const double* __restrict__ src, int64_t ld, int mp,
                                                      int kp, int nmod, int kb, int mode, int8_t* out,
                                                      int* __restrict__ shift, int8_t* out2 = nullptr,
                                                      int* __restrict__ shift2 = nullptr) {
  const int i = blockIdx.x;
  __shared__ double red[8];
  double amax = 0.0;
  pdl_trigger();
  pdl_wait();
  if (i < n) {
    // all of this thread's loads in flight at once (the max chain would
    // otherwise serialise them: the dominant stall)
    int k = threadIdx.x;
    for (; k + 7 * 256 < n; k += 8 * 256) {
      double2 v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = ld2(src + ((size_t)i * ld + k + u * 256) * 2);
#pragma unroll
      for (int u = 0; u < 8; ++u) amax = fmax(amax, fmax(fabs(v[u].x), fabs(v[u].y)));
    }
    for (; k < n; k += 256) {
      const double2 v = ld2(src + ((size_t)i * ld + k) * 2);
      amax = fmax(amax, fmax(fabs(v.x), fabs(v.y)));
    }
  }
  for (int o = 16; o; o >>= 1) amax = fmax(amax, __shfl_xor_sync(0xffffffffu, amax, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = amax;
  __syncthreads();
  amax = red[0];
  for (int q = 1; q < 8; ++q) amax = fmax(amax, red[q]);
  const int sh = oz_shift(amax, kb);
  const double2 sc = oz_scale2(sh);
  if (threadIdx.x == 0 && shift) shift[i] = sh;
  if (threadIdx.x == 0 && shift2) shift2[i] = sh;
  for (int k0 = threadIdx.x * 4; k0 < kp; k0 += blockDim.x * 4) {
    double xv[8];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int k = k0 + e;
      double2 v = make_double2(0.0, 0.0);
      if (i < n && k < n) v = ld2(src + ((size_t)i * ld + k) * 2);
      xv[e] = rint(v.x * sc.x * sc.y);
      xv[4 + e] = rint(v.y * sc.x * sc.y);
    }
    // running word pointers into the planes of modulus t (advanced per
    // modulus: no 64-bit index arithmetic per store)
    const size_t pw = (size_t)mp * kp / 4;  // plane stride in words
    uint32_t* pa = reinterpret_cast<uint32_t*>(out + (size_t)i * kp + k0);
    uint32_t* pb = reinterpret_cast<uint32_t*>((mode == 1 ? out : out2) + (size_t)i * kp + k0);
#pragma unroll 1
    for (int g = 0; g < OZ_NGRP; ++g) {
    float yv[8], ym[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      yv[e] = reduce_pair(xv[e], g);
      ym[e] = yv[e] + OZ_MAGIC_F;
    }
#pragma unroll
    for (int t = 2 * g; t < 2 * g + 2; ++t) {
      uint32_t rw[8];
#pragma unroll
      for (int e = 0; e < 8; ++e) rw[e] = res_word_f(yv[e], ym[e], t);
      const uint32_t wr = pack4(rw[0], rw[1], rw[2], rw[3]);
      const uint32_t wi = pack4(rw[4], rw[5], rw[6], rw[7]);
      const uint32_t wn = __vneg4(wi);
      // skew-B layout (modes 1, 2): -re off the diagonal, re on it
      uint32_t wb = __vneg4(wr);
      if ((unsigned)(i - k0) < 4u) {
        const int sh8 = 8 * (i - k0);
        wb = (wb & ~(0xffu << sh8)) | (wr & (0xffu << sh8));
      }
#ifdef OZ_EXP_NOSTORE
      if (wr == 0x12345678u && wb == 1u && wn == 7u) {
#else
      if (mode != 1) {
#endif
        pa[0] = wr;
        pa[pw] = wi;
        pa[2 * pw] = wn;
      }
      pa += 3 * pw;
#ifdef OZ_EXP_NOSTORE
      if (wi == 0x12345678u && wb == 3u) {
#else
      if (mode != 0) {
#endif
        pb[0] = wb;
        pb[pw] = wi;
      }
      pb += 2 * pw;
    }
    }
  }
}

// B operand of a general matrix X (B[j][k] = X[k][j]): column maxima first
__global__ void __launch_bounds__(256) k_oz_colmax(int n, const double* __restrict__ x, int64_t ld,
                                                   unsigned long long* colmax) {
  const int j = blockIdx.x * 32 + (threadIdx.x & 31);
  const int r0 = blockIdx.y * 64 + (threadIdx.x >> 5) * 8;
  if (j >= n) return;
  double m = 0.0;
  for (int r = r0; r < min(r0 + 8, n); ++r) {
    const double2 v = ld2(x + ((size_t)r * ld + j) * 2);
    m = fmax(m, fmax(fabs(v.x), fabs(v.y)));
  }
  atomicMax(colmax + j, (unsigned long long)__double_as_longlong(m));
}

// then 32 (k) x 32 (j) tiles through shared memory; thread t produces output
// row j = j0 + t / 8, k = k0 + 4 (t % 8) .. +3 (one 32-bit store per plane)
__global__ void __launch_bounds__(256, OZ_CONV_MINB) k_oz_conv_cols(int n, const double* __restrict__ x, int64_t ld, int np,
                                                      int kp, int nmod, int kb,
                                                      const unsigned long long* __restrict__ colmax, int8_t* out,
                                                      int* __restrict__ shift) {
  __shared__ double2 tl[32][33];
  const int j0 = blockIdx.x * 32, k0 = blockIdx.y * 32;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  for (int r = ty; r < 32; r += 8) {
    const int k = k0 + r, j = j0 + tx;
    tl[r][tx] = (k < n && j < n) ? ld2(x + ((size_t)k * ld + j) * 2) : make_double2(0.0, 0.0);
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
#pragma unroll 1
  for (int g = 0; g < OZ_NGRP; ++g) {
    float yv[8], ym[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      yv[e] = reduce_pair(xv[e], g);
      ym[e] = yv[e] + OZ_MAGIC_F;
    }
#pragma unroll
    for (int t = 2 * g; t < 2 * g + 2; ++t) {
      uint32_t rw[8];
#pragma unroll
      for (int e = 0; e < 8; ++e) rw[e] = res_word_f(yv[e], ym[e], t);
      const uint32_t wr = pack4(rw[0], rw[1], rw[2], rw[3]);
      const uint32_t wi = pack4(rw[4], rw[5], rw[6], rw[7]);
      pb[0] = wr;
      pb[pw] = wi;
      pb += 2 * pw;
    }
  }
}

// ---------------------------------------------------------------------------
// Reconstruction (CRT): x = sum_t c_t W_t mod M with W_t = y_t M_t,
// M_t = M / p_t, y_t = M_t^-1 mod p_t, c_t = r_t - floor(p_t / 2) the
// centred residue (|c_t| <= 128; any representative works: a multiple of
// p_t times M_t is a multiple of M).  W_t (< M < 2^125.4) and M are split
// into three signed pieces on the grids 2^0, 2^42, 2^84, the two lower ones
// balanced in [-2^41, 2^41) and the top one < 2^41.4 in magnitude, so with
// sum |c_t| <= 2033 < 2^11 every partial sum S_k = sum_t c_t W_t,k and every
// q M_k (q = rint(S / M), |q| <= 2033) is below 2^52.4, D_k = S_k - q M_k is
// exact for the lower pieces (|D_k| < 2^53) and for the top one (it is
// (x - D_1 - D_0) / 2^84, |x| < 2^121: below 2^38), and x = D_2 + D_1 + D_0
// is the centred representative (|x| < M / 2 by the choice of KB).  (Four
// unsigned 32-bit pieces: 25% more FP64 work, measured 75 vs 62 us.)
// ---------------------------------------------------------------------------
constexpr int OZ_NPC = 3;
struct CrtConst {
  double w[OZ_NMOD][OZ_NPC];  // pieces of W_t
  double mp[OZ_NPC];          // pieces of M
  double m_inv;               // 1 / M
  double bias[OZ_NMOD];       // 2^52 + 2^31 + floor(p_t / 2)
};
__constant__ CrtConst c_crt;

// unsigned byte r -> centred residue r - floor(p / 2) as a double without an
// int -> fp64 conversion: 2^52 + 2^31 + r as the bit pattern, minus the bias
__device__ __forceinline__ double byte_to_double(uint32_t word, int e, double bias) {
  // one byte permute: byte e of word, then 0x00, 0x00, 0x80
  return __hiloint2double(0x43300000, (int)__byte_perm(word, 0x80000000u, 0x7540u | e)) - bias;
}

__global__ void __launch_bounds__(256, OZ_RECON_MINB) k_oz_recon(int m, int n, int nmod, const int8_t* __restrict__ r, int mp,
                                                  int np, const int* __restrict__ rs, const int* __restrict__ cs,
                                                  double* c, int64_t ldc, int lower) {
  const int i = blockIdx.y;
  const int j0 = (blockIdx.x * blockDim.x + threadIdx.x) * OZ_RECON_COLS;
  pdl_trigger();
  pdl_wait();
  if (i >= m || j0 >= n) return;
  if (lower && (j0 >> 7) > (i >> 7)) return;
  const size_t ps = (size_t)2 * mp * np;  // stride between moduli
  // C columns per thread (C = 4: one 32-bit word per modulus and plane; C = 2: 16-bit)
  constexpr int C = OZ_RECON_COLS;
  using word_t = typename std::conditional<C == 4, uint32_t, unsigned short>::type;
  const int8_t* rre = r + (size_t)i * np + j0;
  const int8_t* rim = rre + (size_t)mp * np;
  word_t wr[OZ_NMOD], wi[OZ_NMOD];
#pragma unroll
  for (int t = 0; t < OZ_NMOD; ++t) {
    wr[t] = __ldg(reinterpret_cast<const word_t*>(rre + (size_t)t * ps));
    wi[t] = __ldg(reinterpret_cast<const word_t*>(rim + (size_t)t * ps));
  }
  double s[2 * C][OZ_NPC];
#pragma unroll
  for (int e = 0; e < 2 * C; ++e)
#pragma unroll
    for (int k = 0; k < OZ_NPC; ++k) s[e][k] = 0.0;
#pragma unroll
  for (int t = 0; t < OZ_NMOD; ++t) {
    const double bias = c_crt.bias[t];
#pragma unroll
    for (int e = 0; e < 2 * C; ++e) {
      const double u = byte_to_double(e < C ? wr[t] : wi[t], e % C, bias);
#pragma unroll
      for (int k = 0; k < OZ_NPC; ++k) s[e][k] = fma(u, c_crt.w[t][k], s[e][k]);
    }
  }
  double vr[C], vi[C];
#pragma unroll
  for (int e = 0; e < 2 * C; ++e) {
    const double q = rint(((s[e][2] + s[e][1]) + s[e][0]) * c_crt.m_inv);
    const double d2 = fma(-q, c_crt.mp[2], s[e][2]);
    const double d1 = fma(-q, c_crt.mp[1], s[e][1]);
    const double d0 = fma(-q, c_crt.mp[0], s[e][0]);
    const double x = (d2 + d1) + d0;
    if (e < C)
      vr[e] = x;
    else
      vi[e - C] = x;
  }
#pragma unroll
  for (int e = 0; e < C; ++e) {
    const int j = j0 + e;
    if (j < n && !(lower && (j >> 7) > (i >> 7))) {
      const int sh = -(rs[i] + cs[j]);
      st2(c + ((size_t)i * ldc + j) * 2, make_double2(ldexp(vr[e], sh), ldexp(vi[e], sh)));
    }
  }
}

static cudaError_t launch_recon(int m, int n, int nmod, const int8_t* r, int mp, int np, const int* rs, const int* cs,
                                double* c, int64_t ldc, int lower, cudaStream_t st) {
  const dim3 grid((n + 256 * OZ_RECON_COLS - 1) / (256 * OZ_RECON_COLS), m);
  return launch_pdl(k_oz_recon, grid, dim3(256), 0, st, m, n, nmod, r, mp, np, rs, cs, c, ldc, lower);
}
static bool g_crt_ready = false;
static int crt_init() {
  typedef unsigned __int128 u128;
  typedef __int128 i128;
  CrtConst h;
  u128 m = 1;
  for (int t = 0; t < OZ_NMOD; ++t) m *= (u128)h_oz_p[t];
  // balanced pieces: v = sum_k piece_k 2^(42 k), |piece_0|, |piece_1| <= 2^41
  auto pieces = [](u128 v, double* out) {
    i128 rest = (i128)v;
    for (int k = 0; k < OZ_NPC; ++k) {
      i128 pk = rest;
      if (k < OZ_NPC - 1) {
        pk = rest & (((i128)1 << 42) - 1);
        if (pk >= ((i128)1 << 41)) pk -= (i128)1 << 42;
        rest = (rest - pk) >> 42;
      }
      out[k] = std::ldexp((double)(long long)pk, 42 * k);  // <= 42 bits: exact
    }
  };
  for (int t = 0; t < OZ_NMOD; ++t) {
    const int p = h_oz_p[t];
    const u128 mt = m / (u128)p;
    const int r = (int)(mt % (u128)p);
    int y = 1;
    while ((r * y) % p != 1) ++y;  // p <= 256: direct search
    const u128 w = mt * (u128)y;  // < M
    pieces(w, h.w[t]);
    h.bias[t] = 4503601774854144.0 + (double)(p / 2);
  }
  pieces(m, h.mp);
  h.m_inv = 1.0 / ((h.mp[2] + h.mp[1]) + h.mp[0]);
  ZT_CUDA_CHECK(cudaMemcpyToSymbol(c_crt, &h, sizeof h));
  double qd[OZ_NGRP], qi[OZ_NGRP];
  float pf[OZ_NMOD], pif[OZ_NMOD];
  for (int g = 0; g < OZ_NGRP; ++g) {
    qd[g] = (double)h_oz_p[2 * g] * h_oz_p[2 * g + 1];  // < 2^16
    qi[g] = 1.0 / qd[g];
  }
  for (int t = 0; t < OZ_NMOD; ++t) {
    pf[t] = (float)h_oz_p[t];
    pif[t] = 1.0f / (float)h_oz_p[t];
  }
  ZT_CUDA_CHECK(cudaMemcpyToSymbol(c_oz_q, qd, sizeof qd));
  ZT_CUDA_CHECK(cudaMemcpyToSymbol(c_oz_qinv, qi, sizeof qi));
  ZT_CUDA_CHECK(cudaMemcpyToSymbol(c_oz_pf, pf, sizeof pf));
  ZT_CUDA_CHECK(cudaMemcpyToSymbol(c_oz_pinvf, pif, sizeof pif));
  g_crt_ready = true;
  return ZT_OK;
}

// integer bits per operand entry so that |sum| < M / 2 over K terms (4M form)
static int oz_bits(int k) {
  double lg = 0.0;
  for (int t = 0; t < OZ_NMOD; ++t) lg += std::log2((double)h_oz_p[t]);
  const int kb = (int)std::floor((lg - 1.0 - std::log2(2.0 * k) - 1e-9) / 2.0);
  return std::min(53, kb);
}

size_t oz_workspace_bytes(int n) {
  const size_t p = ((size_t)n + 255) / 256 * 256;
  return (size_t)OZ_NMOD * p * p * (3 + 2 + 2) + 2 * p * sizeof(int) + p * 8 + 1024;
}

// C = A B for complex128 n x n, A general (row scaled), B: bmode 0 general
// (column scaled, transposed conversion), 1 skew-Hermitian with exact
// mirror off the diagonal (converted row-wise as -conj).  lower: only the
// 128-tiles of C on or below the diagonal are computed.
int oz_zgemm(int n, const double* a, int64_t lda, const double* b, int64_t ldb, int bmode, double* c, int64_t ldc,
             int lower, void* ws, size_t ws_bytes, cudaStream_t st) {
  if (n < 1) return fail(ZT_EINVAL, "oz_zgemm: bad size");
  if (ws_bytes < oz_workspace_bytes(n)) return fail(ZT_ENOMEM, "oz_zgemm: workspace too small");
  if (!g_crt_ready) {
    const int rc = crt_init();
    if (rc) return rc;
  }
  const int p = (n + 255) / 256 * 256;
  const int kb = oz_bits(n);
  int8_t* ares = static_cast<int8_t*>(ws);
  int8_t* bres = ares + (size_t)OZ_NMOD * 3 * p * p;
  int8_t* rres = bres + (size_t)OZ_NMOD * 2 * p * p;
  int* rsh = reinterpret_cast<int*>(rres + (size_t)OZ_NMOD * 2 * p * p);
  int* csh = rsh + p;
  unsigned long long* cmax = reinterpret_cast<unsigned long long*>(csh + p);
  ZT_CUDA_CHECK(launch_pdl(k_oz_conv_rows, dim3(p), dim3(256), 0, st, n, a, lda, p, p, OZ_NMOD, kb, 0, ares, rsh,
                           nullptr, nullptr));
  ZT_LAUNCHED();
  if (bmode == 1) {
    ZT_CUDA_CHECK(launch_pdl(k_oz_conv_rows, dim3(p), dim3(256), 0, st, n, b, ldb, p, p, OZ_NMOD, kb, 1, bres, csh,
                             nullptr, nullptr));
    ZT_LAUNCHED();
  } else {
    ZT_CUDA_CHECK(cudaMemsetAsync(cmax, 0, sizeof(unsigned long long) * p, st));
    if (p != n) ZT_CUDA_CHECK(cudaMemsetAsync(bres, 0, (size_t)OZ_NMOD * 2 * p * p, st));
    k_oz_colmax<<<dim3((n + 31) / 32, (n + 63) / 64), 256, 0, st>>>(n, b, ldb, cmax);
    ZT_LAUNCHED();
    k_oz_conv_cols<<<dim3(p / 32, p / 32), 256, 0, st>>>(n, b, ldb, p, p, OZ_NMOD, kb, cmax, bres, csh);
    ZT_LAUNCHED();
  }
  int rc = oz_modgemm(OZ_NMOD, p, p, p, ares, bres, rres, lower, st);
  if (rc) return rc;
  ZT_CUDA_CHECK(launch_recon(n, n, OZ_NMOD, rres, p, p, rsh, csh, c, ldc, lower, st));
  ZT_LAUNCHED();
  ZT_CUDA_CHECK(cudaGetLastError());
  return ZT_OK;
}

int update_pairs(int n, const double* a, const double* bm, double* out, const double* base, const double* xprev,
                 const double* wn, double hh, double qq, unsigned long long* resid, unsigned long long* cons,
                 cudaStream_t st);
int final_commutator(int n, const double* a, const double* wn, double h, double* out, cudaStream_t st);

size_t oz_update_workspace_bytes(int n) {
  const size_t p = ((size_t)n + 255) / 256 * 256;
  return (size_t)OZ_NMOD * p * p * (3 + 2 + 2 + 2) + 4 * p * sizeof(int) + p * 8 + 1024;
}

// One fixed-point update with both products on the INT8 tensor cores:
// a = P X (P rows scaled; X columns scaled, transposed conversion), then
// b = a P on the lower 128-tiles (a rows scaled; P as a skew-Hermitian B
// operand from the same conversion pass as its A layout), then the update
// pass.  gemm1_only: the step's final update W_{n+1} = W_n + h (a - a^H)
// (out = x, h = hh; k_final_commutator).
// X (the B operand of GEMM-1) to column-scaled residues; independent of the
// stream solve, so the step runs it on a side stream beside the solve
int oz_convert_x(int n, const double* x, void* ws, cudaStream_t st) {
  if (!g_crt_ready) {
    const int rc = crt_init();
    if (rc) return rc;
  }
  const int pd = (n + 255) / 256 * 256;
  const int kb = oz_bits(n);
  const size_t pl = (size_t)OZ_NMOD * pd * pd;
  int8_t* bx = static_cast<int8_t*>(ws) + 3 * pl;
  int* sx = reinterpret_cast<int*>(bx + 6 * pl) + pd;
  unsigned long long* cmax = reinterpret_cast<unsigned long long*>(sx + 3 * pd);
  ZT_CUDA_CHECK(cudaMemsetAsync(cmax, 0, sizeof(unsigned long long) * pd, st));
  k_oz_colmax<<<dim3((n + 31) / 32, (n + 63) / 64), 256, 0, st>>>(n, x, n, cmax);
  ZT_LAUNCHED();
  k_oz_conv_cols<<<dim3(pd / 32, pd / 32), 256, 0, st>>>(n, x, n, pd, pd, OZ_NMOD, kb, cmax, bx, sx);
  ZT_LAUNCHED();
  ZT_CUDA_CHECK(cudaGetLastError());
  return ZT_OK;
}

// x_join: X was converted by oz_convert_x on another stream; wait for this
// event before GEMM-1 (nullptr: convert X here)
int oz_update(int n, const double* p, const double* x, double* a, double* bbuf, const double* base,
              const double* xprev, const double* wn, double* out, double hh, double qq, unsigned long long* resid,
              unsigned long long* cons, void* ws, cudaStream_t st, int gemm1_only, cudaEvent_t x_join) {
  if (!g_crt_ready) {
    const int rc = crt_init();
    if (rc) return rc;
  }
  const int pd = (n + 255) / 256 * 256;
  const int kb = oz_bits(n);
  const size_t pl = (size_t)OZ_NMOD * pd * pd;
  int8_t* ares = static_cast<int8_t*>(ws);
  int8_t* bx = ares + 3 * pl;   // X as B operand
  int8_t* bp = bx + 2 * pl;     // P as B operand
  int8_t* rres = bp + 2 * pl;
  int* sp = reinterpret_cast<int*>(rres + 2 * pl);  // P rows (= P-as-B columns)
  int* sx = sp + pd;                                // X columns
  int* sa = sx + pd;                                // a rows
  unsigned long long* cmax = reinterpret_cast<unsigned long long*>(sa + 2 * pd);
  // P: A layout and skew-B layout in one pass
  ZT_CUDA_CHECK(launch_pdl(k_oz_conv_rows, dim3(pd), dim3(256), 0, st, n, p, (int64_t)n, pd, pd, OZ_NMOD, kb,
                           gemm1_only ? 0 : 2, ares, sp, gemm1_only ? nullptr : bp, nullptr));
  ZT_LAUNCHED();
  if (x_join) {
    ZT_CUDA_CHECK(cudaStreamWaitEvent(st, x_join, 0));
  } else {
    const int rc0 = oz_convert_x(n, x, ws, st);
    if (rc0) return rc0;
  }
  (void)cmax;
  int rc = oz_modgemm(OZ_NMOD, pd, pd, pd, ares, bx, rres, 0, st);
  if (rc) return rc;
  ZT_CUDA_CHECK(launch_recon(n, n, OZ_NMOD, rres, pd, pd, sp, sx, a, n, 0, st));
  ZT_LAUNCHED();
  if (gemm1_only) return final_commutator(n, a, wn, hh, out, st);
  ZT_CUDA_CHECK(launch_pdl(k_oz_conv_rows, dim3(pd), dim3(256), 0, st, n, (const double*)a, (int64_t)n, pd, pd,
                           OZ_NMOD, kb, 0, ares, sa, nullptr, nullptr));
  ZT_LAUNCHED();
  rc = oz_modgemm(OZ_NMOD, pd, pd, pd, ares, bp, rres, 1, st);
  if (rc) return rc;
  ZT_CUDA_CHECK(launch_recon(n, n, OZ_NMOD, rres, pd, pd, sa, sp, bbuf, n, 1, st));
  ZT_LAUNCHED();
  ZT_CUDA_CHECK(cudaGetLastError());
  return update_pairs(n, a, bbuf, out, base, xprev, wn, hh, qq, resid, cons, st);
}

static int g_oz_sms = 0;
// residue-GEMM kernel: 1 = single-CTA 128 x 256 tiles (default), 2 = the
// CTA-pair kernel (ZT_OZ_CTA=2 or zt_oz_set_cta(2); needs mp % 256 == 0;
// measured 5-20% slower)
static int g_oz_cta = 0;
int oz_set_cta(int c) {
  if (c != 0 && c != 1 && c != 2) return fail(ZT_EINVAL, "zt_oz_set_cta: 0 (default), 1 or 2");
  g_oz_cta = c;
  return ZT_OK;
}
static int oz_cta() {
  if (g_oz_cta) return g_oz_cta;
  static int env = -1;
  if (env < 0) {
    const char* e = getenv("ZT_OZ_CTA");
    env = (e && e[0] == '2') ? 2 : 1;
  }
  return env;
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

// R = A * B^T residues for every modulus (see header); mp, np, kp multiples of 128
int oz_modgemm(int nmod, int mp, int np, int kp, const int8_t* a, const int8_t* b, int8_t* r, int lower,
               cudaStream_t st) {
  using namespace oz;
  if (nmod < 1 || nmod > OZ_NMOD || mp % TM || np % TN || kp % TK || (lower && mp != np))
    return fail(ZT_EINVAL, "oz_modgemm: bad shape");
  const bool pair = oz_cta() == 2 && mp % oz2::TM == 0;
  CUtensorMap ma, mb;
  int rc = map_i8(&ma, a, (long long)nmod * 3 * mp, kp, 128);
  if (!rc) rc = map_i8(&mb, b, (long long)nmod * 2 * np, kp, pair ? oz2::TN / 2 : TN);
  if (rc) return rc;
  if (!g_oz_sms) {
    int dev;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_oz_sms, cudaDevAttrMultiProcessorCount, dev);
    ZT_CUDA_CHECK(cudaFuncSetAttribute(k_oz_gemm, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM));
    ZT_CUDA_CHECK(cudaFuncSetAttribute(oz2::k_oz_gemm2, cudaFuncAttributeMaxDynamicSharedMemorySize, oz2::SMEM));
  }
  GemmArgs g;
  g.nmod = nmod;
  g.mt = mp / TM;
  g.nt = np / TN;
  g.kt = kp / TK;
  g.lower = lower;
  g.mp = mp;
  g.np = np;
  g.r = r;
  if (pair) {
    g.mt = mp / oz2::TM;
    g.nt = np / oz2::TN;
  }
  const int per = pair ? 2 * (lower ? oz2::lower_count(g.mt) : g.mt * g.nt) : (lower ? lower_count(g.mt) : g.mt * g.nt);
  const int grid = pair ? 2 * std::min(nmod * per, g_oz_sms / 2) : std::min(nmod * per, g_oz_sms);
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
  if (pair)
    oz2::k_oz_gemm2<<<grid, oz2::THREADS, oz2::SMEM, st>>>(ma, mb, g);
  else
    ZT_CUDA_CHECK(launch_pdl(k_oz_gemm, dim3(grid), dim3(THREADS), SMEM, st, ma, mb, g));
  ZT_LAUNCHED();
  if (ev) cudaEventRecord(ev->e1, st);
  ZT_CUDA_CHECK(cudaGetLastError());
  return ZT_OK;
}

int oz_moduli(int* out, int cap) {
  for (int j = 0; j < OZ_NMOD && j < cap; ++j) out[j] = h_oz_p[j];
  return OZ_NMOD;
}

}  // namespace zt

extern "C" int zt_oz_modgemm(int nmod, int mp, int np, int kp, const void* a, const void* b, void* r, int lower,
                             void* stream) {
  if (!a || !b || !r) return zt::fail(ZT_EINVAL, "zt_oz_modgemm: bad argument");
  return zt::oz_modgemm(nmod, mp, np, kp, static_cast<const int8_t*>(a), static_cast<const int8_t*>(b),
                        static_cast<int8_t*>(r), lower, (cudaStream_t)stream);
}

extern "C" int zt_oz_set_cta(int c) { return zt::oz_set_cta(c); }

extern "C" int zt_oz_moduli(int* out, int cap) { return zt::oz_moduli(out, cap); }

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
