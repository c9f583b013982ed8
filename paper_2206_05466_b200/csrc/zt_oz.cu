// FP64-accurate complex GEMM on the INT8 tensor cores (Ozaki scheme II):
// operands are scaled to integers (row / column power-of-two scales, up to
// 53 significant bits), reduced modulo NMOD pairwise-coprime moduli <= 128,
// multiplied exactly per modulus by tcgen05 kind::i8 MMAs with int32
// accumulation (4M complex form: Re = Ar Br + (-Ai) Bi, Im = Ar Bi + Ai Br),
// reduced again modulo p in the epilogue, and reassembled by the Chinese
// remainder theorem into the exact integer product, then scaled back.
//
// Layouts (int8, zero padded to 128 in every dimension):
//   A residues [NMOD][3][Mp][Kp]  planes re, im, -im   (K-major rows)
//   B residues [NMOD][2][Np][Kp]  planes re, im        (K-major: B^T rows)
//   R residues [NMOD][2][Mp][Np]  Re, Im of the product mod p_j (centred)
#include <cuda.h>

#include <algorithm>

#include "zt_common.cuh"
#include "zt_tma.cuh"

namespace zt {

constexpr int OZ_NMOD = 18;
// pairwise coprime, product ~ 2^120.5
__constant__ int c_oz_p[OZ_NMOD] = {128, 127, 125, 121, 119, 117, 113, 109, 107,
                                    103, 101, 97,  89,  83,  79,  73,  71,  67};
static const int h_oz_p[OZ_NMOD] = {128, 127, 125, 121, 119, 117, 113, 109, 107,
                                    103, 101, 97,  89,  83,  79,  73,  71,  67};

namespace oz {

constexpr int TM = 128, TN = 128, TK = 128;  // TK in bytes
constexpr int TILE_BYTES = 128 * TK;         // one 128 x 128 int8 tile
constexpr int STAGE_BYTES = 5 * TILE_BYTES;  // A re, im, -im; B re, im
constexpr int STAGES = 2;
constexpr int THREADS = 6 * 32;
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
// UMMA smem descriptor: K-major, 128 B swizzle, 8-row groups 1024 B apart
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr) {
  return (uint64_t)((saddr & 0x3FFFF) >> 4) | ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32) |
         ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
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
  int nmod, mt, nt, kt;  // tiles per dimension (128) and K blocks (128 B)
  int lower;             // square: only tiles tm >= tn
  int mp, np;            // padded M, N (output leading dimension np)
  int8_t* r;             // [nmod][2][mp][np]
};

__device__ __forceinline__ void work_of(const GemmArgs& g, int w, int& j, int& tm, int& tn) {
  const int per = g.lower ? g.mt * (g.mt + 1) / 2 : g.mt * g.nt;
  j = w / per;
  int t = w - j * per;
  if (g.lower) {
    int c = (int)((sqrt(8.0 * t + 1.0) - 1.0) * 0.5);
    while ((c + 1) * (c + 2) / 2 <= t) ++c;
    while (c * (c + 1) / 2 > t) --c;
    tm = c;
    tn = t - c * (c + 1) / 2;
  } else {
    tm = t % g.mt;
    tn = t / g.mt;
  }
}

__device__ __forceinline__ int modc(int v, int p, double invp) {
  // centred residue of an int32 |v| < 2^31 (exact: the quotient is rounded
  // from a double and the product is formed in integers)
  const int q = __double2int_rn((double)v * invp);
  return v - q * p;
}

__global__ void __launch_bounds__(THREADS, 1)
    k_oz_gemm(const __grid_constant__ CUtensorMap ma, const __grid_constant__ CUtensorMap mb, GemmArgs g) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int per = g.lower ? g.mt * (g.mt + 1) / 2 : g.mt * g.nt;
  const int total = g.nmod * per;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&tfull[s], 1);
      mbar_init(&tempty[s], 4);
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

  if (warp == 0) {
    if (lane == 0) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(&ma) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(&mb) : "memory");
      unsigned it = 0;
      for (int w = blockIdx.x; w < total; w += gridDim.x) {
        int j, tm, tn;
        work_of(g, w, j, tm, tn);
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
          tma2d(st + 4 * TILE_BYTES, &mb, kb * TK, rb + g.np, &full[s]);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      unsigned it = 0, lt = 0;
      for (int w = blockIdx.x; w < total; w += gridDim.x, ++lt) {
        const int ab = lt & 1;
        mbar_wait(&tempty[ab], ((lt >> 1) & 1) ^ 1);
        asm volatile("tcgen05.fence::after_thread_sync;");
        const uint32_t dre = tmem + ab * 256, dim = dre + 128;
        for (int kb = 0; kb < g.kt; ++kb, ++it) {
          const int s = it % STAGES;
          mbar_wait(&full[s], (it / STAGES) & 1);
          asm volatile("tcgen05.fence::after_thread_sync;");
          const uint32_t base = smem_u32(smem + s * STAGE_BYTES);
          const uint32_t are = base, aim = base + TILE_BYTES, anim = base + 2 * TILE_BYTES;
          const uint32_t bre = base + 3 * TILE_BYTES, bim = base + 4 * TILE_BYTES;
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
    const int q = warp & 3;  // TMEM lane quarter = tile rows q*32 ..
    unsigned lt = 0;
    for (int w = blockIdx.x; w < total; w += gridDim.x, ++lt) {
      int j, tm, tn;
      work_of(g, w, j, tm, tn);
      const int ab = lt & 1;
      mbar_wait(&tfull[ab], (lt >> 1) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;");
      const int p = c_oz_p[j];
      const double invp = 1.0 / (double)p;
      const int row = tm * TM + q * 32 + lane;
      int8_t* rre = g.r + ((size_t)(j * 2) * g.mp + row) * g.np + tn * TN;
      int8_t* rim = rre + (size_t)g.mp * g.np;
#pragma unroll 1
      for (int c0 = 0; c0 < TN; c0 += 32) {
        uint32_t v[32];
        const uint32_t ta = tmem + ((uint32_t)(q * 32) << 16) + ab * 256 + c0;
        OZ_LD32(v, ta);
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        uint32_t pk[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          uint32_t x = 0;
#pragma unroll
          for (int b = 0; b < 4; ++b) x |= ((uint32_t)(modc((int)v[4 * e + b], p, invp) & 0xff)) << (8 * b);
          pk[e] = x;
        }
        uint4* d = reinterpret_cast<uint4*>(rre + c0);
        d[0] = make_uint4(pk[0], pk[1], pk[2], pk[3]);
        d[1] = make_uint4(pk[4], pk[5], pk[6], pk[7]);
        OZ_LD32(v, ta + 128);
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          uint32_t x = 0;
#pragma unroll
          for (int b = 0; b < 4; ++b) x |= ((uint32_t)(modc((int)v[4 * e + b], p, invp) & 0xff)) << (8 * b);
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

using encode_fn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                               const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                               CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static int map_i8(CUtensorMap* m, const void* base, long long rows, int cols) {
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
  cuuint32_t box[2] = {TK, 128};
  cuuint32_t es[2] = {1, 1};
  if (fn(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void*>(base), dims, strides, box, es,
         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return fail(ZT_ECUDA, "oz: tensor map encode failed");
  return ZT_OK;
}

}  // namespace oz

static int g_oz_sms = 0;

// R = A * B^T residues for every modulus (see header); mp, np, kp multiples of 128
int oz_modgemm(int nmod, int mp, int np, int kp, const int8_t* a, const int8_t* b, int8_t* r, int lower,
               cudaStream_t st) {
  using namespace oz;
  if (nmod < 1 || nmod > OZ_NMOD || mp % 128 || np % 128 || kp % 128 || (lower && mp != np))
    return fail(ZT_EINVAL, "oz_modgemm: bad shape");
  CUtensorMap ma, mb;
  int rc = map_i8(&ma, a, (long long)nmod * 3 * mp, kp);
  if (!rc) rc = map_i8(&mb, b, (long long)nmod * 2 * np, kp);
  if (rc) return rc;
  if (!g_oz_sms) {
    int dev;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_oz_sms, cudaDevAttrMultiProcessorCount, dev);
    ZT_CUDA_CHECK(cudaFuncSetAttribute(k_oz_gemm, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM));
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
  const int per = lower ? g.mt * (g.mt + 1) / 2 : g.mt * g.nt;
  const int grid = std::min(nmod * per, g_oz_sms);
  k_oz_gemm<<<grid, THREADS, SMEM, st>>>(ma, mb, g);
  ZT_LAUNCHED();
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

extern "C" int zt_oz_moduli(int* out, int cap) { return zt::oz_moduli(out, cap); }
