// kmx_tc.cu — K2 on the 5th-generation tensor cores: the batched
// multiprecision products of the KS path (bignat.py:327-330, the classical
// product the reference's mul() reduces to) as u8 x u8 -> s32 tcgen05.mma
// byte convolutions with TMEM accumulators.
//
// Formulation (one CTA per sub-product z; a = the longer operand, b = the
// shorter, both little-endian byte strings of La, Lb bytes):
//
//   c[k] = sum_i a[i] b[k-i]   (byte convolution; the product is sum_k c[k] 256^k)
//
// An output tile covers byte positions k0 + 16m + n, m < 128 (MMA M), n < 16
// (MMA N), so D[m][n] = sum_u A[m][u] B[n][u] with
//
//   A[m][u] = a[k0 + 16m + u]   and   B[n][u] = b[n - u].
//
// A needs no materialisation: in the K-major SWIZZLE_NONE canonical layout
// ((8,m),(16B,2)) : ((16B,SBO),(1,LBO)) row m of a core matrix sits 16 bytes
// after row m-1, so a plain zero-padded copy of a in shared memory IS the A
// operand with LBO = 16 and SBO = 128; stepping K by 32 bytes only moves the
// descriptor's start address.  B (16 shifted copies of the reversed b) is
// built once per product and reused by every output tile.  Each tile owns 16
// TMEM columns of s32 (sums of at most min(La,Lb) <= 33025 byte products, so
// no overflow) and its own mbarrier, so the epilogue of tile t overlaps the
// MMAs of tile t+1.
//
// Epilogue: thread m reads its 16 accumulators (tcgen05.ld 32x32b.x16), forms
// four 32-bit limb column sums (< 2^56), and one exact block carry scan turns
// the 512 limbs of the tile into normalised 32-bit digits; the carry out of
// the tile feeds the next tile.  The product is written in K2's band format
// (kmx_internal.h MulArgs) with zero band spills, so K3 is unchanged.
#include "kmx_internal.h"
#include "kmx_common.cuh"

namespace kmx {

namespace {

constexpr int TC_THREADS = 128;
constexpr int TC_M = 128;                  // MMA M (rows of a at 16-byte stride)
constexpr int TC_N = 16;                   // MMA N (byte shifts of b)
constexpr int TC_T = TC_M * TC_N;          // output byte positions per tile
constexpr int TC_LIMBS = TC_T / 4;         // product limbs per tile
constexpr int TC_MAXT = 16;                // tiles per CTA (TMEM: 16 x 16 columns)
constexpr int APRE = 2048 + 64;            // zero bytes before a (>= 2032 + 31 + 16)
constexpr int APOST = 2048 + 64;           // zero bytes after a
constexpr int BRPRE = 64;                  // zero bytes before reversed b
constexpr int BRPOST = 96;

// idesc: S32 accumulator (bits 4-5 = 2), A/B unsigned 8-bit (0), K-major,
// N >> 3 at bit 17, M >> 4 at bit 24.
constexpr uint32_t TC_IDESC = (2u << 4) | ((uint32_t)(TC_N >> 3) << 17) | ((uint32_t)(TC_M >> 4) << 24);

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

// SWIZZLE_NONE K-major smem matrix descriptor (sm_100: version 1 at bit 46).
__device__ __forceinline__ uint64_t sdesc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((addr >> 4) & 0x3FFFu) | ((uint64_t)((lbo >> 4) & 0x3FFFu) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFFu) << 32) | (1ull << 46);
}

__device__ __forceinline__ void mma_i8(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t accum) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}\n"
      :: "r"(tmem_d), "l"(adesc), "l"(bdesc), "r"(TC_IDESC), "r"(accum));
}

__device__ __forceinline__ void mma_commit(uint32_t mbar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" :: "r"(mbar)
               : "memory");
}

__device__ __forceinline__ void mbar_init(uint32_t mbar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(mbar), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint32_t mbar, uint32_t parity) {
  uint32_t done = 0;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}\n"
        : "=r"(done) : "r"(mbar), "r"(parity) : "memory");
  } while (!done);
}

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
      "{%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15}, [%16];\n"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
        "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// Carry maps {0,1} -> {0,1}: bit0 = f(0), bit1 = f(1).  compose(later, earlier).
__device__ __forceinline__ uint32_t cm2(uint32_t later, uint32_t earlier) {
  const uint32_t h0 = (later >> (earlier & 1u)) & 1u;
  const uint32_t h1 = (later >> ((earlier >> 1) & 1u)) & 1u;
  return h0 | (h1 << 1);
}
constexpr uint32_t CM2_ID = 2u;  // f(0)=0, f(1)=1

struct TcShared {
  unsigned long long mbar[TC_MAXT];
  uint32_t tmem_base;
  uint32_t warp_map[TC_THREADS / 32];
  unsigned long long carry;       // carry into the next tile
};

}  // namespace

// Shape gate: the longer operand slides (A), the shorter one is materialised
// 16 times (B); TMEM columns and shared memory bound the sizes.
static void tc_sizes(int ma, int mb, int* la, int* lb, int* steps, int* ntiles, size_t* smem) {
  const int lA = 4 * (ma > mb ? ma : mb), lB = 4 * (ma > mb ? mb : ma);
  const int ulo = -32 * ((lB - 1 + 31) / 32);
  const int S = (32 - ulo) / 32;
  *la = lA; *lb = lB; *steps = S;
  *ntiles = (lA + lB - 1 + TC_T - 1) / TC_T;
  const size_t apad = (size_t)APRE + lA + APOST;
  const size_t brpad = (size_t)BRPRE + lB + BRPOST;
  *smem = sizeof(TcShared) + apad + brpad + (size_t)512 * S + 512;
}

bool tc_supported(int ma, int mb) {
  int la, lb, S, nt;
  size_t smem;
  tc_sizes(ma, mb, &la, &lb, &S, &nt, &smem);
  return nt <= TC_MAXT && lb <= 33024 && smem <= 200 * 1024;
}

__global__ void __launch_bounds__(TC_THREADS) k_tcmul(MulArgs a) {
  extern __shared__ __align__(128) unsigned char tsm[];
  TcShared& sh = *reinterpret_cast<TcShared*>(tsm);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int z = blockIdx.x;

  // operand roles: A slides (longer), B is materialised (shorter)
  const bool sw = a.mb > a.ma;
  const uint32_t* Ag = (sw ? a.B + (long long)z * a.b_stride : a.A + (long long)z * a.a_stride);
  const uint32_t* Bg = (sw ? a.A + (long long)z * a.a_stride : a.B + (long long)z * a.b_stride);
  const int mA = sw ? a.mb : a.ma, mB = sw ? a.ma : a.mb;
  const int La = 4 * mA, Lb = 4 * mB;
  const int ulo = -32 * ((Lb - 1 + 31) / 32);
  const int S = (32 - ulo) / 32;
  const int ntiles = (La + Lb - 1 + TC_T - 1) / TC_T;
  const int mp = a.ma + a.mb;

  unsigned char* apad = tsm + ((sizeof(TcShared) + 127) & ~(size_t)127);
  unsigned char* brpad = apad + ((APRE + La + APOST + 127) & ~127);
  unsigned char* bmat = brpad + ((BRPRE + Lb + BRPOST + 127) & ~127);

  if (warp == 0) {
    // TMEM: 16 columns per tile, power of two >= 32
    uint32_t cols = 32;
    while (cols < (uint32_t)(ntiles * TC_N)) cols <<= 1;
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&sh.tmem_base)),
                 "r"(cols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    for (int t = 0; t < ntiles; t++) mbar_init(smem_u32(&sh.mbar[t]), 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    sh.carry = 0ull;
  }

  // A: zero-padded copy of the longer operand (word copies; APRE, La multiples of 4)
  {
    uint32_t* aw = reinterpret_cast<uint32_t*>(apad);
    const int nw = (APRE + La + APOST) / 4;
    for (int w = tid; w < nw; w += TC_THREADS) {
      const int j = w - APRE / 4;
      aw[w] = (j >= 0 && j < mA) ? __ldg(Ag + j) : 0u;
    }
    // reversed b: brpad[BRPRE + x] = b[Lb - 1 - x]
    uint32_t* bw = reinterpret_cast<uint32_t*>(brpad);
    const int nb = (BRPRE + Lb + BRPOST) / 4;
    for (int w = tid; w < nb; w += TC_THREADS) {
      const int j = w - BRPRE / 4;
      bw[w] = (j >= 0 && j < mB) ? __byte_perm(__ldg(Bg + (mB - 1 - j)), 0u, 0x0123) : 0u;
    }
  }
  __syncthreads();
  // B: for K-step s, a 512-byte block [g(2)][j(2)][r(8)][16 B] holding
  // B[n = 8g + r][u = ulo + 32s + 16j + kk] = brpad[BRPRE + Lb - 1 - n + u]
  {
    const uint32_t* bw = reinterpret_cast<const uint32_t*>(brpad);
    uint4* dst = reinterpret_cast<uint4*>(bmat);
    const int nchunks = 32 * S;
    for (int ci = tid; ci < nchunks; ci += TC_THREADS) {
      const int s = ci >> 5, g = (ci >> 4) & 1, j = (ci >> 3) & 1, r = ci & 7;
      const int n = 8 * g + r;
      const int o = BRPRE + Lb - 1 - n + ulo + 32 * s + 16 * j;
      const int w = o >> 2, sh8 = (o & 3) * 8;
      const uint32_t x0 = bw[w], x1 = bw[w + 1], x2 = bw[w + 2], x3 = bw[w + 3], x4 = bw[w + 4];
      dst[ci] = make_uint4(__funnelshift_r(x0, x1, sh8), __funnelshift_r(x1, x2, sh8),
                           __funnelshift_r(x2, x3, sh8), __funnelshift_r(x3, x4, sh8));
    }
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = sh.tmem_base;

  // ---- MMA issue: one thread, tile by tile, one commit per tile
  if (tid == 0) {
    const uint32_t abase = smem_u32(apad) + APRE;
    const uint32_t bbase = smem_u32(bmat);
    for (int t = 0; t < ntiles; t++) {
      const int k0 = t * TC_T;
      // valid u: a side  -k0 - 2032 <= u <= La - k0 - 1, b side ulo <= u < 32
      int slo = (-k0 - (TC_M - 1) * 16 - ulo);
      slo = slo <= 0 ? 0 : slo / 32;
      int shi = (La - k0 - 1 - ulo);
      shi = shi < 0 ? 0 : shi / 32 + 1;
      if (shi > S) shi = S;
      for (int s = slo; s < shi; s++) {
        const uint64_t ad = sdesc(abase + k0 + ulo + 32 * s, 16, 128);
        const uint64_t bd = sdesc(bbase + 512 * s, 128, 256);
        mma_i8(tmem + t * TC_N, ad, bd, s > slo ? 1u : 0u);
      }
      mma_commit(smem_u32(&sh.mbar[t]));  // empty tiles complete immediately
    }
  }

  // ---- epilogue: limb sums, exact carry scan, digits
  uint32_t* Pz = a.P + (long long)z * a.p_stride;
  for (int t = 0; t < ntiles; t++) {
    const int k0 = t * TC_T;
    int slo = (-k0 - (TC_M - 1) * 16 - ulo);
    slo = slo <= 0 ? 0 : slo / 32;
    int shi = (La - k0 - 1 - ulo);
    shi = shi < 0 ? 0 : shi / 32 + 1;
    if (shi > S) shi = S;
    uint32_t v[16];
    mbar_wait(smem_u32(&sh.mbar[t]), 0);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (shi > slo) {
      tmem_ld16(tmem + ((uint32_t)(32 * warp) << 16) + (uint32_t)(t * TC_N), v);
    } else {
#pragma unroll
      for (int i = 0; i < 16; i++) v[i] = 0u;
    }
    // four limb column sums (< 2^56) and local digits with carry-in 0
    uint32_t d[4];
    unsigned long long x = 0ull;
#pragma unroll
    for (int q = 0; q < 4; q++) {
      const unsigned long long sq = (unsigned long long)v[4 * q] + ((unsigned long long)v[4 * q + 1] << 8) +
                                    ((unsigned long long)v[4 * q + 2] << 16) +
                                    ((unsigned long long)v[4 * q + 3] << 24);
      x = (x >> 32) + sq;
      d[q] = (uint32_t)x;
    }
    const unsigned long long cout = x >> 32;
    // carry-in value from the previous thread (tile carry for thread 0)
    unsigned long long xin = __shfl_up_sync(0xffffffffu, cout, 1);
    __shared__ unsigned long long s_cout[TC_THREADS / 32];
    if (lane == 31) s_cout[warp] = cout;
    __syncthreads();
    if (lane == 0) xin = warp ? s_cout[warp - 1] : sh.carry;
    // overflow map of (D + xin + o) past 2^128, o in {0,1}
    const bool ones = (d[1] & d[2] & d[3]) == 0xFFFFFFFFu;
    const unsigned long long s0 = (unsigned long long)d[0] + xin;
    const uint32_t g = ones && (s0 >> 32) != 0ull;
    const uint32_t p = ones && ((s0 + 1ull) >> 32) != 0ull;
    uint32_t F = g | (p << 1);
#pragma unroll
    for (int dd = 1; dd < 32; dd <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, F, dd);
      if (lane >= dd) F = cm2(F, y);
    }
    if (lane == 31) sh.warp_map[warp] = F;
    __syncthreads();
    uint32_t E = __shfl_up_sync(0xffffffffu, F, 1);
    uint32_t W = CM2_ID;
    for (int w = 0; w < warp; w++) W = cm2(sh.warp_map[w], W);
    E = lane ? cm2(E, W) : W;
    const uint32_t oin = E & 1u;  // overflow of the previous thread (its o)
    const uint32_t Fin = cm2(F, W);  // block-inclusive: this thread's own o
    // final digits: D + xin + oin (mod 2^128)
    unsigned long long acc = s0 + oin;
    d[0] = (uint32_t)acc;
#pragma unroll
    for (int q = 1; q < 4; q++) {
      acc = (acc >> 32) + d[q];
      d[q] = (uint32_t)acc;
    }
    const int L = t * TC_LIMBS + 4 * tid;
    if (L + 4 <= mp) {
      *reinterpret_cast<uint4*>(Pz + L) = make_uint4(d[0], d[1], d[2], d[3]);
    } else {
#pragma unroll
      for (int q = 0; q < 4; q++)
        if (L + q < mp) Pz[L + q] = d[q];
    }
    __syncthreads();  // everyone has read sh.carry / s_cout / warp_map
    if (tid == TC_THREADS - 1) sh.carry = cout + (Fin & 1u);
  }
  for (int bi = tid; bi < a.nbands; bi += TC_THREADS) {
    unsigned long long* sp = a.spill + ((long long)z * a.nbands + bi) * 2;
    sp[0] = 0ull;
    sp[1] = 0ull;
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) {
    uint32_t cols = 32;
    while (cols < (uint32_t)(ntiles * TC_N)) cols <<= 1;
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(cols));
  }
}

cudaError_t launch_tcmul(const MulArgs& a, cudaStream_t st) {
  int la, lb, S, nt;
  size_t smem;
  tc_sizes(a.ma, a.mb, &la, &lb, &S, &nt, &smem);
  if (!tc_supported(a.ma, a.mb)) return cudaErrorNotSupported;
  if (a.nprod == 0) return cudaSuccess;
  static size_t s_max_set = 0;
  if (smem > 48 * 1024 && smem > s_max_set) {
    cudaError_t e = cudaFuncSetAttribute(k_tcmul, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    s_max_set = smem;
  }
  k_tcmul<<<a.nprod, TC_THREADS, smem, st>>>(a);
  g_launches++;
  return cudaGetLastError();
}

}  // namespace kmx
