// kmx_tc.cu — K2 on the 5th-generation tensor cores: the batched
// multiprecision products of the KS path (bignat.py:327-330, the classical
// product the reference's mul() reduces to) as u8 x u8 -> s32 tcgen05.mma
// byte convolutions with TMEM accumulators.
//
// Formulation (a = the longer operand, b = the shorter, both little-endian
// byte strings of La, Lb bytes):
//
//   c[k] = sum_i a[i] b[k-i]   (byte convolution; the product is sum_k c[k] 256^k)
//
// One MMA tile (M = 128, N = 16H) covers the byte positions
//
//   k0 + alpha_m + beta_n,   alpha_m = 16 (m % 8) + 128H (m / 8),
//                            beta_n  = (n % 16) + 128 (n / 16),
//
// a contiguous run of 2048H positions, as D[m][n] = sum_u A[m][u] B[n][u] with
//
//   A[m][u] = a[k0 + alpha_m + u]   and   B[n][u] = b[beta_n - u].
//
// A needs no materialisation: in the K-major SWIZZLE_NONE canonical layout
// ((8,m),(16B,2)) : ((16B,SBO),(1,LBO)) row r of a core matrix sits 16 bytes
// after row r-1, so a plain zero-padded copy of a in shared memory IS the A
// operand with LBO = 16 and SBO = 128H; stepping K by 32 bytes (or the tile by
// 2048H) only moves the descriptor's start address.  B (16H shifted, reversed
// copies of b) is built per K-chunk from a staged copy of b (half-warp byte
// permutes), multi-buffered against the MMAs with mbarriers, and shared by all tiles of
// the CTA (warp 0 issues the MMAs, warps 1-3 build B stages into an mbarrier
// ring).  In SS mode the MMA is paced by its shared-memory operand reads
// (~110 B/clk measured: tools/microbench/tc_peak.cu), so a wider N buys more
// MACs per A byte; the host picks H per shape from that cost model.
//
// TMEM: each tile owns 16H columns of 32-bit sums.  A sum has at most
// min(La,Lb) byte products < 2^16 each; read as u32 (the accumulator wraps, no
// saturation) it is exact for min(La,Lb) <= 65536.  Longer operands split
// the K-steps into segments of TC_SEG_STEPS (32 * 2048 = 65536 bytes of b):
// each segment accumulates into its own TMEM columns and the epilogue adds
// the segments' exact partial sums in 64-bit.
//
// Epilogue: thread m reads its 16H accumulators (tcgen05.ld 32x32b.x16),
// forms limb column sums (< 2^56), stages them in shared memory in limb
// order, and one exact block carry scan over {0,1} overflow maps normalises
// the tile's 512H limbs; the carry feeds the next tile of the CTA and the
// CTA's last carry becomes the band spill K3 folds in (K2's MulArgs contract).
#include <cstdio>
#include <cstdlib>
#include <map>
#include <mutex>
#include <vector>

#include "kmx_internal.h"
#include "kmx_common.cuh"
#include "kmx_pack.cuh"
#include "kmx_tcutil.cuh"

namespace kmx {

namespace {

constexpr int TC_EPI = 128;  // warps 0-3: epilogue (TMEM lane quarters)
constexpr int TC_MAX_COLS = 256;  // TMEM columns per CTA (two CTAs per SM fit)
constexpr int TC_SEG_LOG = 11;    // K-steps per exact accumulation segment: 2^11 * 32 B = 64 KB
__host__ __device__ inline int tc_nseg(int Lb, int S) {
  return Lb <= 65536 ? 1 : (S + (1 << TC_SEG_LOG) - 1) >> TC_SEG_LOG;
}

template <int H>
struct TcG {
  static constexpr int N = 16 * H;
  static constexpr int T = 2048 * H;                 // output byte positions per tile
  static constexpr int LIMBS = 512 * H;              // product limbs per tile
  static constexpr int SBO_A = 128 * H;              // A: stride of 8-row groups
  static constexpr int AMAX = 16 * 7 + SBO_A * 15;   // largest alpha_m
  static constexpr int APAD = (AMAX + 32 + 64 + 15) & ~15;
  static constexpr int BMAX = 15 + 128 * (H - 1);    // largest beta_n
  static constexpr int STEPB = 512 * H;              // B bytes per K-step
  // idesc: S32 accumulator (bits 4-5 = 2), A/B unsigned 8-bit, K-major,
  // N >> 3 at bit 17, M >> 4 = 8 at bit 24.
  static constexpr uint32_t IDESC = (2u << 4) | ((uint32_t)(N >> 3) << 17) | (8u << 24);
};


// K-steps u0 = ulo + 32 s, s in [0, S), and the steps tile t needs.
struct TcDims {
  int La, Lb, ulo, S, ntiles;
};
template <int H>
__host__ __device__ inline TcDims tc_dims(int mA, int mB) {
  TcDims d;
  d.La = 4 * mA;
  d.Lb = 4 * mB;
  d.ulo = -32 * ((d.Lb - 1 + 31) / 32);
  d.S = fdiv32(TcG<H>::BMAX - d.ulo) + 1;
  d.ntiles = (d.La + d.Lb - 1 + TcG<H>::T - 1) / TcG<H>::T;
  return d;
}
template <int H>
__host__ __device__ inline void tc_tile_steps(const TcDims& d, int t, int& slo, int& shi) {
  const int k0 = t * TcG<H>::T;
  slo = -fdiv32(k0 + TcG<H>::AMAX + 31 + d.ulo);  // ceil((-k0 - AMAX - 31 - ulo) / 32)
  if (slo < 0) slo = 0;
  shi = fdiv32(d.La - k0 - 1 - d.ulo) + 1;
  if (shi > d.S) shi = d.S;
}

constexpr int TC_MAXNB = 4;  // B ring stages

struct TcShared {
  unsigned long long bar_full[TC_MAXNB];   // B stage built (3 builder warps arrive)
  unsigned long long bar_empty[TC_MAXNB];  // MMAs that read the stage completed (commit)
  unsigned long long bar_done;             // all MMAs of the CTA completed
  unsigned long long bar_stage;            // bulk copies of the operands landed (TMA, complete_tx)
  unsigned long long s_cout[TC_EPI / 32];
  unsigned long long carry;                // carry into the next tile
  uint32_t tmem_base;
  uint32_t warp_map[TC_EPI / 32];
};

struct TcArgs {
  MulArgs m;
  int KC;       // K-steps per B stage
  int NB;       // B stages in the ring (2..TC_MAXNB)
  int TPC;      // tiles per CTA
  int nranges;  // CTAs per product = ceil(ntiles / TPC)
  int nseg;     // exact accumulation segments of the K-steps (tc_nseg)
  int fuse;     // pack the operands in the prologue (pk, P)
  int P;        // products per pair
  size_t ring;  // bytes of the B ring (>= the pack staging area when fused)
  int bulk;     // stage aligned operands with bulk async copies (KMX_TC_BULK, default 1)
  PackArgs pk;
};

__host__ __device__ inline size_t round128(size_t x) { return (x + 127) & ~(size_t)127; }

// zero padding around the staged b: the window words read by the B build
// lie in [(-BMAX - 32) / 4, (Lb + 128H + 96) / 4)
template <int H>
struct TcB {
  static constexpr int BPAD = (TcG<H>::BMAX + 128 + 15) & ~15;
};

template <int H>
__host__ __device__ inline size_t tc_ring(int KC, int NB, size_t stage) {
  const size_t r = (size_t)NB * KC * TcG<H>::STEPB;
  return r > stage ? r : round128(stage);
}
template <int H>
__host__ __device__ inline size_t tc_smem(int La, int Lb, int KC, int NB, size_t stage) {
  return round128(sizeof(TcShared)) + round128((size_t)La + 2 * TcG<H>::APAD) +
         round128((size_t)Lb + 2 * TcB<H>::BPAD) + tc_ring<H>(KC, NB, stage);
}


// ---------------------------------------------------------------- kernel
// Warp roles: warp 0 lane 0 issues the MMAs; warps 1..NW-1 build the B
// stages; all warps stage the operands; warps 0-3 run the epilogue (TMEM
// lanes 32w..32w+31 belong to warp w).  NW = 4 suits CTAs with one or two
// tiles (occupancy), NW = 8 CTAs whose B build is shared by more tiles.
template <int H, int NW>
__global__ void __launch_bounds__(32 * NW) k_tcmul(TcArgs ta) {
  constexpr int TC_THREADS = 32 * NW;  // warp 0: MMA issue, warps 1..NW-1: B build
  using G = TcG<H>;
  const MulArgs& a = ta.m;
  extern __shared__ __align__(128) unsigned char tsm[];
  TcShared& sh = *reinterpret_cast<TcShared*>(tsm);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int z = blockIdx.x / ta.nranges, rg = blockIdx.x % ta.nranges;

  // operand roles: A slides (longer), B is materialised (shorter)
  const bool sw = a.mb > a.ma;
  const uint32_t* Ag = sw ? a.B + (long long)z * a.b_stride : a.A + (long long)z * a.a_stride;
  const uint32_t* Bg = sw ? a.A + (long long)z * a.a_stride : a.B + (long long)z * a.b_stride;
  const int mA = sw ? a.mb : a.ma, mB = sw ? a.ma : a.mb;
  const TcDims d = tc_dims<H>(mA, mB);
  const int mp = a.ma + a.mb;
  const int t0 = rg * ta.TPC;
  const int t1 = min(d.ntiles, t0 + ta.TPC);
  const int nt = t1 - t0;
  const int KC = ta.KC, NB = ta.NB;

  unsigned char* apad = tsm + round128(sizeof(TcShared));
  unsigned char* bpad = apad + round128((size_t)d.La + 2 * G::APAD);
  unsigned char* bring = bpad + round128((size_t)d.Lb + 2 * TcB<H>::BPAD);

  // K-step span of the CTA's tiles
  int cs_lo = d.S, cs_hi = 0;
  for (int t = t0; t < t1; t++) {
    int slo, shi;
    tc_tile_steps<H>(d, t, slo, shi);
    if (slo < shi) {
      cs_lo = min(cs_lo, slo);
      cs_hi = max(cs_hi, shi);
    }
  }
  const int clo = cs_lo < cs_hi ? cs_lo / KC : 0;
  const int chi = cs_lo < cs_hi ? (cs_hi + KC - 1) / KC : 0;

  const int nseg = ta.nseg;
  uint32_t cols = 32;
  while (cols < (uint32_t)(nt * nseg * G::N)) cols <<= 1;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&sh.tmem_base)),
                 "r"(cols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    for (int i = 0; i < TC_MAXNB; i++) {
      mbar_init(smem_u32(&sh.bar_full[i]), TC_THREADS / 32 - 1);
      mbar_init(smem_u32(&sh.bar_empty[i]), 1);
    }
    mbar_init(smem_u32(&sh.bar_done), 1);
    mbar_init(smem_u32(&sh.bar_stage), 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    sh.carry = 0ull;
  }
  if (ta.fuse) {
    // fused K1: pack this product's two operands (pack ops s and P + s of the
    // pair) straight into the padded A and b buffers; the B ring stages the
    // coefficient vector meanwhile
    uint32_t* aw = reinterpret_cast<uint32_t*>(apad);
    uint32_t* bw = reinterpret_cast<uint32_t*>(bpad);
    constexpr int AP = G::APAD / 4, BP = TcB<H>::BPAD / 4;
    for (int w = tid; w < AP; w += TC_THREADS) {
      aw[w] = 0u;
      aw[AP + mA + w] = 0u;
    }
    for (int w = tid; w < BP; w += TC_THREADS) {
      bw[w] = 0u;
      bw[BP + mB + w] = 0u;
    }
    const int pair = z / ta.P, s = z - pair * ta.P;
    const int oa = sw ? ta.P + s : s, ob = sw ? s : ta.P + s;
    uint32_t* stage = reinterpret_cast<uint32_t*>(bring);
    pack_op<true>(ta.pk, pair, oa, stage, aw + AP, rg == 0);
    pack_op<true>(ta.pk, pair, ob, stage, bw + BP, rg == 0);
    __syncthreads();  // the ring is free again before the builders use it
  } else if (ta.bulk && (reinterpret_cast<uintptr_t>(Ag) & 15) == 0 && (reinterpret_cast<uintptr_t>(Bg) & 15) == 0 &&
             ((sw ? a.b_stride : a.a_stride) & 3) == 0 && ((sw ? a.a_stride : a.b_stride) & 3) == 0 &&
             (sw ? a.b_stride : a.a_stride) >= ((mA + 3) & ~3) && (sw ? a.a_stride : a.b_stride) >= ((mB + 3) & ~3)) {
    // Operands staged by two bulk async copies (TMA engine, cp.async.bulk
    // completing on an mbarrier): all bytes in flight at once with no register
    // round trip, while the threads zero the padding around them.  The copies
    // are rounded up to 16 bytes (the operand rows are padded to 4 limbs);
    // the rounding limbs are zeroed once they have landed.
    const int La16 = (d.La + 15) & ~15, Lb16 = (d.Lb + 15) & ~15;
    if (tid == 0) {
      const uint32_t bar = smem_u32(&sh.bar_stage);
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"((uint32_t)(La16 + Lb16))
                   : "memory");
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                       smem_u32(apad + G::APAD)),
                   "l"(Ag), "r"((uint32_t)La16), "r"(bar)
                   : "memory");
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                       smem_u32(bpad + TcB<H>::BPAD)),
                   "l"(Bg), "r"((uint32_t)Lb16), "r"(bar)
                   : "memory");
    }
    uint4* aw = reinterpret_cast<uint4*>(apad);
    uint4* bq = reinterpret_cast<uint4*>(bpad);
    const uint4 z4 = make_uint4(0u, 0u, 0u, 0u);
    constexpr int AQ = G::APAD / 16, BQ = TcB<H>::BPAD / 16;
    // padding outside the copies' byte ranges (no two writers on one byte)
    for (int w = tid; w < AQ; w += TC_THREADS) aw[w] = z4;
    for (int w = AQ + La16 / 16 + tid; w < 2 * AQ + d.La / 16; w += TC_THREADS) aw[w] = z4;
    for (int w = tid; w < BQ; w += TC_THREADS) bq[w] = z4;
    for (int w = BQ + Lb16 / 16 + tid; w < 2 * BQ + d.Lb / 16; w += TC_THREADS) bq[w] = z4;
    __syncthreads();  // the barrier's init (thread 0) precedes every wait
    mbar_wait(smem_u32(&sh.bar_stage), 0);
    // the rounding limbs past the operands (row padding, not operand data)
    uint32_t* a32 = reinterpret_cast<uint32_t*>(apad + G::APAD);
    uint32_t* b32 = reinterpret_cast<uint32_t*>(bpad + TcB<H>::BPAD);
    if (tid < (La16 - d.La) / 4) a32[mA + tid] = 0u;
    if (tid < (Lb16 - d.Lb) / 4) b32[mB + tid] = 0u;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  } else {
    // A: zero-padded copy of the longer operand; b: zero-padded copy of the shorter
    // (unaligned views, e.g. Karatsuba halves: 16-byte loads where possible)
    uint4* aw = reinterpret_cast<uint4*>(apad);
    const int nq = (d.La + 2 * G::APAD) / 16;
    const int qa = G::APAD / 16;
    const bool al = (mA & 3) == 0 && (reinterpret_cast<uintptr_t>(Ag) & 15) == 0;
    for (int w = tid; w < nq; w += TC_THREADS) {
      const int j = 4 * (w - qa);
      uint4 v = make_uint4(0u, 0u, 0u, 0u);
      if (j >= 0 && j < mA) {
        if (al) {
          v = __ldg(reinterpret_cast<const uint4*>(Ag + j));
        } else {
          v.x = __ldg(Ag + j);
          v.y = j + 1 < mA ? __ldg(Ag + j + 1) : 0u;
          v.z = j + 2 < mA ? __ldg(Ag + j + 2) : 0u;
          v.w = j + 3 < mA ? __ldg(Ag + j + 3) : 0u;
        }
      }
      aw[w] = v;
    }
    // b: 16-byte loads when aligned (BPAD is a multiple of 16 bytes)
    const int nbw = (d.Lb + 2 * TcB<H>::BPAD) / 4;
    const int ba = TcB<H>::BPAD / 4;
    if ((mB & 3) == 0 && (reinterpret_cast<uintptr_t>(Bg) & 15) == 0 && (nbw & 3) == 0) {
      uint4* bq = reinterpret_cast<uint4*>(bpad);
      for (int w = tid; w < nbw / 4; w += TC_THREADS) {
        const int j = 4 * w - ba;
        bq[w] = (j >= 0 && j < mB) ? __ldg(reinterpret_cast<const uint4*>(Bg + j)) : make_uint4(0u, 0u, 0u, 0u);
      }
    } else {
      uint32_t* bw = reinterpret_cast<uint32_t*>(bpad);
      for (int w = tid; w < nbw; w += TC_THREADS) {
        const int j = w - ba;
        bw[w] = (j >= 0 && j < mB) ? __ldg(Bg + j) : 0u;
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = sh.tmem_base;

  if (warp == 0) {
    // ---- MMA issuer
    if (lane == 0) {
      const uint32_t sA = smem_u32(apad) + G::APAD;
      uint32_t started = 0u;
      for (int c = clo; c < chi; c++) {
        const int k = c - clo, st = k % NB;
        mbar_wait(smem_u32(&sh.bar_full[st]), (uint32_t)((k / NB) & 1));
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const int sb = c * KC, se = min(d.S, sb + KC);
        const uint32_t sB = smem_u32(bring + (size_t)st * KC * G::STEPB);
        for (int t = t0; t < t1; t++) {
          int slo, shi;
          tc_tile_steps<H>(d, t, slo, shi);
          const int s0 = max(slo, sb), s1 = min(shi, se);
          const uint32_t abase = sA + (uint32_t)(t * G::T + d.ulo);
          // split [s0, s1) at the exact-accumulation segment boundaries
          for (int sa = s0; sa < s1;) {
            const int cell = (t - t0) + (sa >> TC_SEG_LOG) * nt;  // (tile, segment); nt = 0 stride if nseg == 1
            const int se2 = nseg > 1 ? min(s1, ((sa >> TC_SEG_LOG) + 1) << TC_SEG_LOG) : s1;
            const uint32_t dcol = tmem + (uint32_t)((nseg > 1 ? cell : t - t0) * G::N);
            const uint32_t bit = 1u << (nseg > 1 ? cell : t - t0);
            for (int s = sa; s < se2; s++) {
              const uint64_t ad = sdesc(abase + 32u * (uint32_t)s, 16, G::SBO_A);
              const uint64_t bd = sdesc(sB + (uint32_t)((s - sb) * G::STEPB), 128, 256);
              mma_i8(dcol, ad, bd, G::IDESC, (started & bit) ? 1u : 0u);
              started |= bit;
            }
            sa = se2;
          }
        }
        mma_commit(smem_u32(&sh.bar_empty[st]));
      }
      mma_commit(smem_u32(&sh.bar_done));
    }
    __syncwarp();
  } else {
    // ---- B builders: half-warp hb owns items hb, hb + 6, ...; an item is
    // (step, kc, j) and lane nl writes row n = nl + 16j of it:
    //   B[n][u0 + 16kc + kk] = b[nl + 128j - u0 - 16kc - kk]
    //     = byte (16 + nl - kk) of the 32-byte window at w0 = 128j - u0 - 16kc - 16
    const int hb = 2 * (warp - 1) + (lane >> 4), nl = lane & 15;
    const int A0 = (13 + nl) >> 2, r0 = (13 + nl) & 3;
    const uint32_t psel = (uint32_t)(r0 + 3) | ((uint32_t)(r0 + 2) << 4) | ((uint32_t)(r0 + 1) << 8) |
                          ((uint32_t)r0 << 12);
    const uint32_t* bw = reinterpret_cast<const uint32_t*>(bpad) + TcB<H>::BPAD / 4;
    constexpr int NHB = 2 * (TC_THREADS / 32 - 1);
    for (int c = clo; c < chi; c++) {
      const int k = c - clo, st = k % NB;
      if (k >= NB) mbar_wait(smem_u32(&sh.bar_empty[st]), (uint32_t)(((k / NB) - 1) & 1));
      unsigned char* bb = bring + (size_t)st * KC * G::STEPB;
      const int sb = c * KC, se = min(d.S, sb + KC);
      const int nitems = (se - sb) * 2 * H;
      for (int ib = 0; ib < nitems; ib += 2 * NHB) {
        uint32_t wv[2];
        int doff[2];
        bool valid[2];
#pragma unroll
        for (int x = 0; x < 2; x++) {
          const int it = ib + x * NHB + hb;
          valid[x] = it < nitems;
          const int sl = valid[x] ? it / (2 * H) : 0;
          const int rem = valid[x] ? it - sl * 2 * H : 0;
          const int kc = rem & 1, j = rem >> 1;
          const int u0 = d.ulo + 32 * (sb + sl);
          const int w0 = 128 * j - u0 - 16 * kc - 16;
          wv[x] = bw[(w0 >> 2) + nl];
          doff[x] = sl * G::STEPB + 256 * ((nl >> 3) + 2 * j) + 128 * kc + 16 * (nl & 7);
        }
#pragma unroll
        for (int x = 0; x < 2; x++) {
          uint32_t W[5];
#pragma unroll
          for (int q = 0; q < 5; q++) W[q] = __shfl_sync(0xffffffffu, wv[x], A0 - 3 + q, 16);
          if (valid[x]) {
            uint4 o;
            o.x = __byte_perm(W[3], W[4], psel);
            o.y = __byte_perm(W[2], W[3], psel);
            o.z = __byte_perm(W[1], W[2], psel);
            o.w = __byte_perm(W[0], W[1], psel);
            *reinterpret_cast<uint4*>(bb + doff[x]) = o;
          }
        }
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(smem_u32(&sh.bar_full[st]));
    }
  }
  mbar_wait(smem_u32(&sh.bar_done), 0);
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");

  // ---- epilogue: limb sums -> staged in limb order -> exact carry scan
  unsigned long long* stg = reinterpret_cast<unsigned long long*>(bring);  // 4096H bytes (NB*KC >= 8)
  uint32_t* Pz = a.P + (long long)z * a.p_stride;
  const int m = tid;
  const bool epi = warp < TC_EPI / 32;
  for (int t = t0; t < t1; t++) {
    int slo, shi;
    tc_tile_steps<H>(d, t, slo, shi);
    __syncthreads();  // previous tile's readers are done with stg / s_cout / warp_map
    if (epi) {
#pragma unroll
      for (int j = 0; j < H; j++) {
        unsigned long long ls[4] = {0ull, 0ull, 0ull, 0ull};
        if (nseg == 1) {
          if (slo < shi) {
            uint32_t v[16];
            tmem_ld16(tmem + ((uint32_t)(32 * warp) << 16) + (uint32_t)((t - t0) * G::N + 16 * j), v);
#pragma unroll
            for (int q = 0; q < 4; q++)
              ls[q] = (unsigned long long)v[4 * q] + ((unsigned long long)v[4 * q + 1] << 8) +
                      ((unsigned long long)v[4 * q + 2] << 16) + ((unsigned long long)v[4 * q + 3] << 24);
          }
        } else
        for (int g = 0; g < nseg; g++) {
          // segment g of this tile: K-steps [max(slo, g 2^SEG), min(shi, (g+1) 2^SEG))
          const int glo = nseg > 1 ? max(slo, g << TC_SEG_LOG) : slo;
          const int ghi = nseg > 1 ? min(shi, (g + 1) << TC_SEG_LOG) : shi;
          if (glo >= ghi) continue;
          uint32_t v[16];
          tmem_ld16(tmem + ((uint32_t)(32 * warp) << 16) + (uint32_t)(((t - t0) + g * nt) * G::N + 16 * j), v);
#pragma unroll
          for (int q = 0; q < 4; q++)
            ls[q] += (unsigned long long)v[4 * q] + ((unsigned long long)v[4 * q + 1] << 8) +
                     ((unsigned long long)v[4 * q + 2] << 16) + ((unsigned long long)v[4 * q + 3] << 24);
        }
        unsigned long long* dst = stg + 4 * (m & 7) + 32 * j + 32 * H * (m >> 3);
#pragma unroll
        for (int q = 0; q < 4; q++) dst[q] = ls[q];
      }
    }
    __syncthreads();
    // thread m: limbs [4H m, 4H m + 4H) of the tile, local digits with carry-in 0
    uint32_t dg[4 * H];
    unsigned long long cout = 0ull, xin = 0ull;
    uint32_t ones = 0xFFFFFFFFu;
    if (epi) {
      unsigned long long x = 0ull;
#pragma unroll
      for (int q = 0; q < 4 * H; q++) {
        x = (x >> 32) + stg[4 * H * m + q];
        dg[q] = (uint32_t)x;
      }
      cout = x >> 32;
      xin = __shfl_up_sync(0xffffffffu, cout, 1);
      if (lane == 31) sh.s_cout[warp] = cout;
#pragma unroll
      for (int q = 1; q < 4 * H; q++) ones &= dg[q];
    }
    __syncthreads();
    uint32_t F = 0u;
    unsigned long long s0 = 0ull;
    if (epi) {
      if (lane == 0) xin = warp ? sh.s_cout[warp - 1] : sh.carry;
      // overflow of (D + xin + o) past 2^(128H), o in {0,1} from the previous thread
      s0 = (unsigned long long)dg[0] + xin;
      const bool all1 = ones == 0xFFFFFFFFu;
      const uint32_t g = all1 && (s0 >> 32) != 0ull;
      const uint32_t p = all1 && ((s0 + 1ull) >> 32) != 0ull;
      F = g | (p << 1);
#pragma unroll
      for (int dd = 1; dd < 32; dd <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, F, dd);
        if (lane >= dd) F = cm2(F, y);
      }
      if (lane == 31) sh.warp_map[warp] = F;
    }
    __syncthreads();
    if (epi) {
      uint32_t E = __shfl_up_sync(0xffffffffu, F, 1);
      uint32_t Wm = CM2_ID;
      for (int w = 0; w < warp; w++) Wm = cm2(sh.warp_map[w], Wm);
      E = lane ? cm2(E, Wm) : Wm;
      const uint32_t Fin = cm2(F, Wm);
      unsigned long long acc = s0 + (E & 1u);
      dg[0] = (uint32_t)acc;
#pragma unroll
      for (int q = 1; q < 4 * H; q++) {
        acc = (acc >> 32) + dg[q];
        dg[q] = (uint32_t)acc;
      }
      const int L = t * G::LIMBS + 4 * H * m;
      if (L + 4 * H <= mp) {
#pragma unroll
        for (int q = 0; q < H; q++)
          *reinterpret_cast<uint4*>(Pz + L + 4 * q) =
              make_uint4(dg[4 * q], dg[4 * q + 1], dg[4 * q + 2], dg[4 * q + 3]);
      } else {
#pragma unroll
        for (int q = 0; q < 4 * H; q++)
          if (L + q < mp) Pz[L + q] = dg[q];
      }
      if (tid == TC_EPI - 1) sh.carry = cout + (Fin & 1u);
    }
  }
  __syncthreads();
  // band spills: zero inside the range, the range's carry on its top band
  {
    const int b0 = 2 * H * t0, b1 = min(a.nbands, 2 * H * t1);
    for (int bi = b0 + tid; bi < b1; bi += TC_THREADS) {
      unsigned long long* sp = a.spill + ((long long)z * a.nbands + bi) * 2;
      sp[0] = bi == 2 * H * t1 - 1 ? sh.carry : 0ull;
      sp[1] = 0ull;
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(cols));
}

// ------------------------------------------------- persistent, specialized
// Short products (one CTA range per product, one accumulation segment): a
// persistent CTA walks products z = blockIdx.x, + gridDim.x, ... with the
// warps specialized and every hand-off on an mbarrier, so one product's
// operand copy, B build, MMAs and epilogue overlap its neighbours':
//   warp 0 (lane 0)  MMA issue into TMEM accumulator buf = i & 1;
//   warps 1-3        B builders (as k_tcmul), ring phases continue across
//                    products; warp 1 lane 0 also clears the operands'
//                    rounding limbs once their bulk copies land;
//   warps 4-7        epilogue of product i from accumulator buf while the
//                    MMAs of product i+1 fill the other; warp 4 lane 0
//                    prefetches product i+2's operands into buffer buf (TMA
//                    bulk copies) as soon as product i's MMAs completed.
// Operand buffers, TMEM accumulators and the staging area are doubled; the
// epilogue has its own staging area (the B ring stays live).
struct TcSharedP {
  unsigned long long bar_full[TC_MAXNB];
  unsigned long long bar_empty[TC_MAXNB];
  unsigned long long bar_stage[2];      // bulk copies of product i landed (complete_tx)
  unsigned long long bar_ready[2];      // ... and its rounding limbs cleared
  unsigned long long bar_acc_full[2];   // MMAs of product i done (tcgen05.commit)
  unsigned long long bar_acc_empty[2];  // epilogue drained accumulator buf (4 warps)
  unsigned long long s_cout[TC_EPI / 32];
  unsigned long long carry;
  uint32_t tmem_base;
  uint32_t warp_map[TC_EPI / 32];
};

template <int H>
__host__ __device__ inline size_t tcp_abuf(int La) { return round128((size_t)La + 2 * TcG<H>::APAD + 16); }
template <int H>
__host__ __device__ inline size_t tcp_bbuf(int Lb) { return round128((size_t)Lb + 2 * TcB<H>::BPAD + 16); }
template <int H>
__host__ __device__ inline size_t tcp_smem(int La, int Lb, int KC, int NB) {
  return round128(sizeof(TcSharedP)) + 2 * tcp_abuf<H>(La) + 2 * tcp_bbuf<H>(Lb) + (size_t)NB * KC * TcG<H>::STEPB +
         (size_t)4096 * H;
}

template <int H>
__global__ void __launch_bounds__(256, 1) k_tcmul_p(TcArgs ta) {
  using G = TcG<H>;
  constexpr int THREADS = 256;
  const MulArgs& a = ta.m;
  extern __shared__ __align__(128) unsigned char tsm[];
  TcSharedP& sh = *reinterpret_cast<TcSharedP*>(tsm);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const bool sw = a.mb > a.ma;
  const int mA = sw ? a.mb : a.ma, mB = sw ? a.ma : a.mb;
  const long long astr = sw ? a.b_stride : a.a_stride, bstr = sw ? a.a_stride : a.b_stride;
  const uint32_t* Abase = sw ? a.B : a.A;
  const uint32_t* Bbase = sw ? a.A : a.B;
  const TcDims d = tc_dims<H>(mA, mB);
  const int mp = a.ma + a.mb;
  const int ntl = d.ntiles;  // all tiles of a product in this CTA
  const int KC = ta.KC, NB = ta.NB;
  const int La16 = (d.La + 15) & ~15, Lb16 = (d.Lb + 15) & ~15;
  unsigned char* abuf[2];
  unsigned char* bbuf[2];
  abuf[0] = tsm + round128(sizeof(TcSharedP));
  abuf[1] = abuf[0] + tcp_abuf<H>(d.La);
  bbuf[0] = abuf[1] + tcp_abuf<H>(d.La);
  bbuf[1] = bbuf[0] + tcp_bbuf<H>(d.Lb);
  unsigned char* bring = bbuf[1] + tcp_bbuf<H>(d.Lb);
  unsigned long long* stg = reinterpret_cast<unsigned long long*>(bring + (size_t)NB * KC * G::STEPB);
  // the CTA span of K-steps (the same for every product of the launch)
  int cs_lo = d.S, cs_hi = 0;
  for (int t = 0; t < ntl; t++) {
    int slo, shi;
    tc_tile_steps<H>(d, t, slo, shi);
    if (slo < shi) { cs_lo = min(cs_lo, slo); cs_hi = max(cs_hi, shi); }
  }
  const int clo = cs_lo < cs_hi ? cs_lo / KC : 0;
  const int chi = cs_lo < cs_hi ? (cs_hi + KC - 1) / KC : 0;
  const int nchunk = chi - clo;
  uint32_t acc_cols = 32;
  while (acc_cols < (uint32_t)(ntl * G::N)) acc_cols <<= 1;
  const uint32_t cols = 2 * acc_cols;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&sh.tmem_base)),
                 "r"(cols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  const int nmine = blockIdx.x < a.nprod ? (a.nprod - 1 - (int)blockIdx.x) / (int)gridDim.x + 1 : 0;
  auto prefetch = [&](int i) {  // thread-level: product i of this CTA into buffer i & 1
    const long long z = blockIdx.x + (long long)i * gridDim.x;
    const uint32_t bar = smem_u32(&sh.bar_stage[i & 1]);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"((uint32_t)(La16 + Lb16))
                 : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(abuf[i & 1] + G::APAD)),
                 "l"(Abase + z * astr), "r"((uint32_t)La16), "r"(bar)
                 : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(bbuf[i & 1] + TcB<H>::BPAD)),
                 "l"(Bbase + z * bstr), "r"((uint32_t)Lb16), "r"(bar)
                 : "memory");
  };
  // zero pads of both buffers (outside every copy's byte range)
  for (int bsel = 0; bsel < 2; bsel++) {
    uint4* aw = reinterpret_cast<uint4*>(abuf[bsel]);
    uint4* bq = reinterpret_cast<uint4*>(bbuf[bsel]);
    const uint4 z4 = make_uint4(0u, 0u, 0u, 0u);
    constexpr int AQ = G::APAD / 16, BQ = TcB<H>::BPAD / 16;
    for (int w = tid; w < AQ; w += THREADS) aw[w] = z4;
    for (int w = AQ + La16 / 16 + tid; w < 2 * AQ + d.La / 16 + 1; w += THREADS) aw[w] = z4;
    for (int w = tid; w < BQ; w += THREADS) bq[w] = z4;
    for (int w = BQ + Lb16 / 16 + tid; w < 2 * BQ + d.Lb / 16 + 1; w += THREADS) bq[w] = z4;
  }
  if (tid == 0) {
    for (int i = 0; i < TC_MAXNB; i++) {
      mbar_init(smem_u32(&sh.bar_full[i]), 3);
      mbar_init(smem_u32(&sh.bar_empty[i]), 1);
    }
    for (int i = 0; i < 2; i++) {
      mbar_init(smem_u32(&sh.bar_stage[i]), 1);
      mbar_init(smem_u32(&sh.bar_ready[i]), 1);
      mbar_init(smem_u32(&sh.bar_acc_full[i]), 1);
      mbar_init(smem_u32(&sh.bar_acc_empty[i]), 4);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = sh.tmem_base;
  if (tid == 0) {
    if (nmine > 0) prefetch(0);
    if (nmine > 1) prefetch(1);
  }

  if (warp == 0) {
    // ---------------- MMA issuer
    if (lane == 0) {
      long long kg = 0;  // ring chunk counter across products
      for (int i = 0; i < nmine; i++) {
        const int buf = i & 1;
        const uint32_t ph = (uint32_t)((i >> 1) & 1);
        mbar_wait(smem_u32(&sh.bar_ready[buf]), ph);
        mbar_wait(smem_u32(&sh.bar_acc_empty[buf]), ph ^ 1u);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t sA = smem_u32(abuf[buf]) + G::APAD;
        const uint32_t dacc = tmem + (uint32_t)buf * acc_cols;
        uint32_t started = 0u;
        for (int c = clo; c < chi; c++, kg++) {
          const int st = (int)(kg % NB);
          mbar_wait(smem_u32(&sh.bar_full[st]), (uint32_t)((kg / NB) & 1));
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          const int sb = c * KC, se = min(d.S, sb + KC);
          const uint32_t sB = smem_u32(bring + (size_t)st * KC * G::STEPB);
          for (int t = 0; t < ntl; t++) {
            int slo, shi;
            tc_tile_steps<H>(d, t, slo, shi);
            const int s0 = max(slo, sb), s1 = min(shi, se);
            const uint32_t abase = sA + (uint32_t)(t * G::T + d.ulo);
            const uint32_t dcol = dacc + (uint32_t)(t * G::N);
            for (int s = s0; s < s1; s++) {
              const uint64_t ad = sdesc(abase + 32u * (uint32_t)s, 16, G::SBO_A);
              const uint64_t bd = sdesc(sB + (uint32_t)((s - sb) * G::STEPB), 128, 256);
              mma_i8(dcol, ad, bd, G::IDESC, (started >> t) & 1u);
              started |= 1u << t;
            }
          }
          mma_commit(smem_u32(&sh.bar_empty[st]));
        }
        mma_commit(smem_u32(&sh.bar_acc_full[buf]));
      }
    }
    __syncwarp();
  } else if (warp < 4) {
    // ---------------- B builders (3 warps, 6 half-warps)
    const int hb = 2 * (warp - 1) + (lane >> 4), nl = lane & 15;
    const int A0 = (13 + nl) >> 2, r0 = (13 + nl) & 3;
    const uint32_t psel = (uint32_t)(r0 + 3) | ((uint32_t)(r0 + 2) << 4) | ((uint32_t)(r0 + 1) << 8) |
                          ((uint32_t)r0 << 12);
    constexpr int NHB = 6;
    long long kg = 0;
    for (int i = 0; i < nmine; i++) {
      const int buf = i & 1;
      const uint32_t ph = (uint32_t)((i >> 1) & 1);
      if (warp == 1) {
        mbar_wait(smem_u32(&sh.bar_stage[buf]), ph);
        if (lane == 0) {  // the rounding limbs past the operands (row padding, not operand data)
          uint32_t* a32 = reinterpret_cast<uint32_t*>(abuf[buf] + G::APAD);
          uint32_t* b32 = reinterpret_cast<uint32_t*>(bbuf[buf] + TcB<H>::BPAD);
          for (int w = mA; w < La16 / 4; w++) a32[w] = 0u;
          for (int w = mB; w < Lb16 / 4; w++) b32[w] = 0u;
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          mbar_arrive(smem_u32(&sh.bar_ready[buf]));
        }
        __syncwarp();
      }
      mbar_wait(smem_u32(&sh.bar_ready[buf]), ph);
      const uint32_t* bw = reinterpret_cast<const uint32_t*>(bbuf[buf]) + TcB<H>::BPAD / 4;
      for (int c = clo; c < chi; c++, kg++) {
        const int st = (int)(kg % NB);
        if (kg >= NB) mbar_wait(smem_u32(&sh.bar_empty[st]), (uint32_t)(((kg / NB) - 1) & 1));
        unsigned char* bb = bring + (size_t)st * KC * G::STEPB;
        const int sb = c * KC, se = min(d.S, sb + KC);
        const int nitems = (se - sb) * 2 * H;
        for (int ib = 0; ib < nitems; ib += 2 * NHB) {
          uint32_t wv[2];
          int doff[2];
          bool valid[2];
#pragma unroll
          for (int x = 0; x < 2; x++) {
            const int it = ib + x * NHB + hb;
            valid[x] = it < nitems;
            const int sl = valid[x] ? it / (2 * H) : 0;
            const int rem = valid[x] ? it - sl * 2 * H : 0;
            const int kc = rem & 1, j = rem >> 1;
            const int u0 = d.ulo + 32 * (sb + sl);
            const int w0 = 128 * j - u0 - 16 * kc - 16;
            wv[x] = bw[(w0 >> 2) + nl];
            doff[x] = sl * G::STEPB + 256 * ((nl >> 3) + 2 * j) + 128 * kc + 16 * (nl & 7);
          }
#pragma unroll
          for (int x = 0; x < 2; x++) {
            uint32_t W[5];
#pragma unroll
            for (int q = 0; q < 5; q++) W[q] = __shfl_sync(0xffffffffu, wv[x], A0 - 3 + q, 16);
            if (valid[x]) {
              uint4 o;
              o.x = __byte_perm(W[3], W[4], psel);
              o.y = __byte_perm(W[2], W[3], psel);
              o.z = __byte_perm(W[1], W[2], psel);
              o.w = __byte_perm(W[0], W[1], psel);
              *reinterpret_cast<uint4*>(bb + doff[x]) = o;
            }
          }
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (lane == 0) mbar_arrive(smem_u32(&sh.bar_full[st]));
      }
    }
  } else {
    // ---------------- epilogue (warps 4-7: TMEM lane quarter ew)
    const int ew = warp - 4, m = tid - 128;
    for (int i = 0; i < nmine; i++) {
      const int buf = i & 1;
      const uint32_t ph = (uint32_t)((i >> 1) & 1);
      const long long z = blockIdx.x + (long long)i * gridDim.x;
      mbar_wait(smem_u32(&sh.bar_acc_full[buf]), ph);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      // product i's operands are no longer read: prefetch product i + 2
      if (m == 0 && i + 2 < nmine) prefetch(i + 2);
      const uint32_t dacc = tmem + (uint32_t)buf * acc_cols;
      uint32_t* Pz = a.P + z * a.p_stride;
      if (m == 0) sh.carry = 0ull;
      for (int t = 0; t < ntl; t++) {
        int slo, shi;
        tc_tile_steps<H>(d, t, slo, shi);
        asm volatile("bar.sync 1, 128;" ::: "memory");  // previous tile's readers are done
#pragma unroll
        for (int j = 0; j < H; j++) {
          unsigned long long ls[4] = {0ull, 0ull, 0ull, 0ull};
          if (slo < shi) {
            uint32_t v[16];
            tmem_ld16(dacc + ((uint32_t)(32 * ew) << 16) + (uint32_t)(t * G::N + 16 * j), v);
#pragma unroll
            for (int q = 0; q < 4; q++)
              ls[q] = (unsigned long long)v[4 * q] + ((unsigned long long)v[4 * q + 1] << 8) +
                      ((unsigned long long)v[4 * q + 2] << 16) + ((unsigned long long)v[4 * q + 3] << 24);
          }
          unsigned long long* dst = stg + 4 * (m & 7) + 32 * j + 32 * H * (m >> 3);
#pragma unroll
          for (int q = 0; q < 4; q++) dst[q] = ls[q];
        }
        asm volatile("bar.sync 1, 128;" ::: "memory");
        uint32_t dg[4 * H];
        unsigned long long x = 0ull;
#pragma unroll
        for (int q = 0; q < 4 * H; q++) {
          x = (x >> 32) + stg[4 * H * m + q];
          dg[q] = (uint32_t)x;
        }
        const unsigned long long cout = x >> 32;
        unsigned long long xin = __shfl_up_sync(0xffffffffu, cout, 1);
        if (lane == 31) sh.s_cout[ew] = cout;
        uint32_t ones = 0xFFFFFFFFu;
#pragma unroll
        for (int q = 1; q < 4 * H; q++) ones &= dg[q];
        asm volatile("bar.sync 1, 128;" ::: "memory");
        if (lane == 0) xin = ew ? sh.s_cout[ew - 1] : sh.carry;
        const unsigned long long s0 = (unsigned long long)dg[0] + xin;
        const bool all1 = ones == 0xFFFFFFFFu;
        const uint32_t g = all1 && (s0 >> 32) != 0ull;
        const uint32_t p = all1 && ((s0 + 1ull) >> 32) != 0ull;
        uint32_t F = g | (p << 1);
#pragma unroll
        for (int dd = 1; dd < 32; dd <<= 1) {
          const uint32_t y = __shfl_up_sync(0xffffffffu, F, dd);
          if (lane >= dd) F = cm2(F, y);
        }
        if (lane == 31) sh.warp_map[ew] = F;
        asm volatile("bar.sync 1, 128;" ::: "memory");
        uint32_t E = __shfl_up_sync(0xffffffffu, F, 1);
        uint32_t Wm = CM2_ID;
        for (int w = 0; w < ew; w++) Wm = cm2(sh.warp_map[w], Wm);
        E = lane ? cm2(E, Wm) : Wm;
        const uint32_t Fin = cm2(F, Wm);
        unsigned long long acc = s0 + (E & 1u);
        dg[0] = (uint32_t)acc;
#pragma unroll
        for (int q = 1; q < 4 * H; q++) {
          acc = (acc >> 32) + dg[q];
          dg[q] = (uint32_t)acc;
        }
        const int L = t * G::LIMBS + 4 * H * m;
        if (L + 4 * H <= mp) {
#pragma unroll
          for (int q = 0; q < H; q++)
            *reinterpret_cast<uint4*>(Pz + L + 4 * q) =
                make_uint4(dg[4 * q], dg[4 * q + 1], dg[4 * q + 2], dg[4 * q + 3]);
        } else {
#pragma unroll
          for (int q = 0; q < 4 * H; q++)
            if (L + q < mp) Pz[L + q] = dg[q];
        }
        asm volatile("bar.sync 1, 128;" ::: "memory");  // every reader of sh.carry is done
        if (m == 127) sh.carry = cout + (Fin & 1u);
      }
      asm volatile("bar.sync 1, 128;" ::: "memory");
      // band spills: zero, the product's final carry on its top band
      for (int bi = m; bi < a.nbands; bi += 128) {
        unsigned long long* sp = a.spill + (z * a.nbands + bi) * 2;
        sp[0] = bi == 2 * H * ntl - 1 ? sh.carry : 0ull;
        sp[1] = 0ull;
      }
      asm volatile("bar.sync 1, 128;" ::: "memory");  // sh.carry read by all before the next product resets it
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(smem_u32(&sh.bar_acc_empty[buf]));
    }
  }
  (void)nchunk;
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(cols));
}

// ---------------------------------------------------------------- planning
struct TcPlan {
  int H, NW, KC, NB, TPC, nranges, ntiles, nseg;
  size_t smem;
  double cost;  // modelled cycles per product
  int persist = 0;  // k_tcmul_p (persistent, warp-specialized)
  int swz = 0;      // k_tcswz (kmx_tcs.cu): the pitch (32 / 64 / 128), 0 = this file's kernels
  TcsPlan sp;       // its plan
};

// KMX_TCS: -1 (default) the swizzled-window kernel joins the tuner's
// candidates and is the untuned default wherever it takes the shape; 0 off;
// 1 always (model-chosen pitch, no timing); 32 / 64 / 128 force that pitch.
int tcs_mode() {
  const char* v = getenv("KMX_TCS");
  return v && *v ? atoi(v) : -1;
}
// KMX_TCS_PERSIST: -1 (default) all forms are tuner candidates; 0 one-shot
// CTAs only; 1 the persistent form only (wherever its plan exists); 2 the
// M = 64 two-window form only (wherever the product fits it).
int tcs_persist_mode() {
  const char* v = getenv("KMX_TCS_PERSIST");
  return v && *v ? atoi(v) : -1;
}
// the swizzled-window plan of lowest modelled cost (or the forced pitch)
bool tcs_best(int ma, int mb, TcPlan& out) {
  const int mode = tcs_mode();
  if (mode == 0) return false;
  bool ok = false;
  for (int pitch : {32, 64, 128}) {
    if (mode >= 32 && mode != pitch) continue;
    TcsPlan sp;
    if (!(tcs_persist_mode() == 1 && tcs_plan(ma, mb, pitch, 1, sp)) && !tcs_plan(ma, mb, pitch, 0, sp)) continue;
    {  // the M = 64 two-window form where the product fits it (KMX_TCS_PERSIST=2 forces, 0 / 1 exclude)
      TcsPlan s64;
      if ((tcs_persist_mode() < 0 || tcs_persist_mode() == 2) && tcs_plan(ma, mb, pitch, 2, s64) &&
          (tcs_persist_mode() == 2 || s64.cost < sp.cost))
        sp = s64;
    }
    if (!ok || sp.cost < out.sp.cost) {
      out = TcPlan();
      out.swz = pitch;
      out.sp = sp;
      out.H = pitch / 16; out.NW = 4; out.KC = sp.KS; out.NB = 1; out.TPC = 1;
      out.nranges = sp.ntiles; out.ntiles = sp.ntiles; out.nseg = 1;
      out.smem = sp.smem; out.cost = sp.cost;
      ok = true;
    }
  }
  return ok;
}

int env_int_tc(const char* n, int dflt) {
  const char* v = getenv(n);
  return v && *v ? atoi(v) : dflt;
}

int tc_num_sms() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

// Cost model (cycles per product on one SM), calibrated by tools/tc_sweep.py:
// the SS-mode MMA is paced by its shared-memory operand reads, ~110 B/clk
// (tools/microbench/tc_peak.cu: M=128 N=16..128 -> 45/46/56/74 cycles), and
// never faster than the tensor floor 8H cycles per N=16H MMA; the B build
// costs ~38H cycles per K-step with 3 builder warps and ~17H with 7, shared
// by the CTA's tiles; a range takes the larger of the two.
template <int H>
double tc_cost(const TcDims& d, int TPC, int NW) {
  const double mma = (4096.0 + 512.0 * H) / 110.0 > 8.0 * H ? (4096.0 + 512.0 * H) / 110.0 : 8.0 * H;
  const double bld = (NW == 4 ? 38.0 : 17.0) * H;
  double cost = 0.0;
  for (int r0 = 0; r0 < d.ntiles; r0 += TPC) {
    int lo = d.S, hi = 0;
    long long steps = 0;
    for (int t = r0; t < min(d.ntiles, r0 + TPC); t++) {
      int slo, shi;
      tc_tile_steps<H>(d, t, slo, shi);
      if (shi > slo) {
        steps += shi - slo;
        lo = min(lo, slo);
        hi = max(hi, shi);
      }
    }
    const double m = (double)steps * mma, b = hi > lo ? (double)(hi - lo) * bld : 0.0;
    cost += m > b ? m : b;
  }
  return cost;
}

template <int H>
bool tc_plan_h(int ma, int mb, long long nprod, size_t stage, TcPlan& p, int kc_force = 0, int nw_force = 0) {
  const int mA = ma > mb ? ma : mb, mB = ma > mb ? mb : ma;
  const TcDims d = tc_dims<H>(mA, mB);
  const int nseg = tc_nseg(d.Lb, d.S);  // u32 accumulator exactness: <= 64 KB of b per segment
  if (nseg * TcG<H>::N > TC_MAX_COLS) return false;
  int KC = kc_force ? kc_force : env_int_tc("KMX_TC_KC", 16);
  if (KC < 4) KC = 4;
  int NB = env_int_tc("KMX_TC_NB", 2);
  if (NB < 2) NB = 2;
  if (NB > TC_MAXNB) NB = TC_MAXNB;
  if (NB * KC < 8) KC = (8 + NB - 1) / NB;  // epilogue staging needs 4096H bytes
  const size_t cap = 200 * 1024;
  while (tc_smem<H>(d.La, d.Lb, KC, NB, stage) > cap && (NB > 2 || KC > 8)) {
    if (NB > 2) NB--;
    else KC /= 2;
  }
  if (tc_smem<H>(d.La, d.Lb, KC, NB, stage) > cap) return false;
  int TPC = TC_MAX_COLS / (TcG<H>::N * nseg);
  if (TPC > d.ntiles) TPC = d.ntiles;
  const int tpc_env = env_int_tc("KMX_TC_TPC", 0);
  if (tpc_env > 0 && tpc_env < TPC) TPC = tpc_env;
  // enough CTAs to cover the SMs twice over
  while (TPC > 1 && nprod * ((d.ntiles + TPC - 1) / TPC) < 2LL * tc_num_sms()) TPC--;
  p.H = H;
  p.NW = nw_force ? nw_force : (env_int_tc("KMX_TC_NW", TPC <= 2 ? 4 : 8) == 4 ? 4 : 8);
  if (!kc_force && p.NW == 4 && env_int_tc("KMX_TC_KC", 0) == 0 && H <= 2) KC = 8;
  p.KC = KC;
  p.NB = NB;
  p.TPC = TPC;
  p.ntiles = d.ntiles;
  p.nranges = (d.ntiles + TPC - 1) / TPC;
  p.nseg = nseg;
  p.smem = tc_smem<H>(d.La, d.Lb, KC, NB, stage);
  p.cost = tc_cost<H>(d, TPC, p.NW);
  return true;
}

bool tc_plan(int ma, int mb, long long nprod, size_t stage, TcPlan& best) {
  const int force = env_int_tc("KMX_TC_H", 0);
  bool ok = false;
  TcPlan p;
#define KMX_TRY_H(HH)                                                   \
  if ((force == 0 || force == HH) && tc_plan_h<HH>(ma, mb, nprod, stage, p)) { \
    if (!ok || p.cost < best.cost) best = p;                            \
    ok = true;                                                          \
  }
  KMX_TRY_H(1) KMX_TRY_H(2) KMX_TRY_H(3) KMX_TRY_H(4) KMX_TRY_H(6) KMX_TRY_H(8)
#undef KMX_TRY_H
  return ok;
}

template <int H, int NW>
cudaError_t launch_hw(const TcArgs& ta, size_t smem, cudaStream_t st) {
  static size_t s_set = 0;
  if (smem > 32 * 1024 && smem > s_set) {  // + static shared memory (fused pack) past 48 KB
    cudaError_t e = cudaFuncSetAttribute(k_tcmul<H, NW>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    s_set = smem;
  }
  const long long grid = (long long)ta.m.nprod * ta.nranges;
  k_tcmul<H, NW><<<(unsigned)grid, 32 * NW, smem, st>>>(ta);
  return cudaGetLastError();
}
template <int H>
cudaError_t launch_h(const TcArgs& ta, int nw, size_t smem, cudaStream_t st) {
  return nw == 4 ? launch_hw<H, 4>(ta, smem, st) : launch_hw<H, 8>(ta, smem, st);
}

// ---------------------------------------------------------------- peak
// Dense tcgen05 u8 MMA throughput (M=128, N=256, K=32, SS): one elected
// thread per CTA issues back-to-back MMAs over 8 resident K-steps into one
// TMEM accumulator, committing every 32; the roofline denominator for K2.
template <int N>
__global__ void __launch_bounds__(128) k_tc_peak(int iters, unsigned long long* sink) {
  extern __shared__ __align__(128) unsigned char pk[];
  __shared__ uint32_t tbase;
  __shared__ __align__(8) unsigned long long bar;
  constexpr int KS = 8;
  constexpr uint32_t IDESC = (2u << 4) | ((uint32_t)(N >> 3) << 17) | (8u << 24);
  unsigned char* A = pk;
  unsigned char* B = pk + KS * 4096;
  for (int i = threadIdx.x; i < (KS * 4096 + KS * N * 32) / 4; i += 128)
    reinterpret_cast<uint32_t*>(pk)[i] = (uint32_t)i * 2654435761u;
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tbase)), "r"(256));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 0) {
    mbar_init(smem_u32(&bar), 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tm = tbase;
  if (threadIdx.x == 0) {
    for (int it = 0; it < iters; it++) {
      for (int k = 0; k < 32; k++) {
        const int s = k % KS;
        mma_i8(tm, sdesc(smem_u32(A) + 4096 * s, 128, 256), sdesc(smem_u32(B) + N * 32 * s, 128, 256), IDESC,
               (it | k) ? 1u : 0u);
      }
      mma_commit(smem_u32(&bar));
      mbar_wait(smem_u32(&bar), (uint32_t)(it & 1));
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (threadIdx.x < 32) {
    uint32_t v[16];
    tmem_ld16(tm, v);
    if (v[0] == 0x12345678u && v[1] == 0x9abcdef0u) sink[0] = v[2];
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tm), "r"(256));
  }
}

}  // namespace

// Dense SS-mode u8 MMA rate (multiply-accumulates per second, all SMs) for
// M = 128 and the given N (16..256): N = 256 is the device peak (the roofline
// denominator); the smaller N of K2's tiles give the same-shape ceiling,
// where each MMA re-reads its 4 KB A tile from shared memory.
template <int N>
double measure_tc_peak_n(int iters) {
  const size_t smem = 8 * 4096 + 8 * N * 32;
  if (cudaFuncSetAttribute(k_tc_peak<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
    return -1.0;
  unsigned long long* sink = nullptr;
  if (cudaMalloc(&sink, 8) != cudaSuccess) return -1.0;
  const int grid = tc_num_sms();
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  k_tc_peak<N><<<grid, 128, smem>>>(8, sink);
  float best = 1e30f;
  for (int rep = 0; rep < 3; rep++) {
    cudaEventRecord(e0);
    k_tc_peak<N><<<grid, 128, smem>>>(iters, sink);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(sink);
  if (cudaGetLastError() != cudaSuccess) return -1.0;
  return (double)grid * iters * 32 * 128.0 * N * 32 / (best * 1e-3);
}

double measure_tc_peak(int iters) { return measure_tc_peak_n<256>(iters); }

double measure_tc_peak_shape(int n, int iters) {
  switch (n) {
    case 16: return measure_tc_peak_n<16>(iters);
    case 32: return measure_tc_peak_n<32>(iters);
    case 48: return measure_tc_peak_n<48>(iters);
    case 64: return measure_tc_peak_n<64>(iters);
    case 96: return measure_tc_peak_n<96>(iters);
    case 128: return measure_tc_peak_n<128>(iters);
    case 256: return measure_tc_peak_n<256>(iters);
    default: return -1.0;
  }
}

namespace {
}  // namespace

bool tc_supported(int ma, int mb, size_t stage_bytes) {
  TcPlan p;
  if (tc_plan(ma, mb, 1 << 20, stage_bytes, p)) return true;
  // the swizzled-window kernel stages a window per K-chunk, not whole operands:
  // any length of the longer operand, up to 32768 limbs of the shorter
  return stage_bytes == 0 && tcs_best(ma, mb, p);
}

namespace {
cudaError_t launch_plan(const MulArgs& a, const TcPlan& p, cudaStream_t st, const PackArgs* pk, int P);

// The persistent kernel takes a tiling whose product fits one CTA range and
// one accumulation segment, with both accumulators in TMEM.
bool tcp_ok(int ma, int mb, const TcPlan& p) {
  if (p.nseg != 1) return false;
  const int mA = ma > mb ? ma : mb, mB = ma > mb ? mb : ma;
  size_t smem = 0;
  int ntl = 0, N = 16 * p.H;
  switch (p.H) {
#define KMX_TCP_CASE(HH) \
    case HH: { const TcDims d = tc_dims<HH>(mA, mB); ntl = d.ntiles; smem = tcp_smem<HH>(d.La, d.Lb, p.KC, p.NB); break; }
    KMX_TCP_CASE(1) KMX_TCP_CASE(2) KMX_TCP_CASE(3) KMX_TCP_CASE(4) KMX_TCP_CASE(6) KMX_TCP_CASE(8)
#undef KMX_TCP_CASE
    default: return false;
  }
  uint32_t acc = 32;
  while (acc < (uint32_t)(ntl * N)) acc <<= 1;
  return ntl <= 32 && 2 * acc <= 512 && smem <= 200 * 1024;
}

// Candidate tilings: every feasible H with KC in {8, 16} and NW in {4, 8},
// keeping those the model puts within 1.6x of its best.
std::vector<TcPlan> tc_candidates(int ma, int mb, long long nprod) {
  std::vector<TcPlan> v;
  double best = 1e300;
  for (int kc : {8, 16})
    for (int nw : {4, 8}) {
      TcPlan p;
#define KMX_CAND_H(HH)                                           \
  if (tc_plan_h<HH>(ma, mb, nprod, 0, p, kc, nw)) {              \
    v.push_back(p);                                              \
    best = p.cost < best ? p.cost : best;                        \
  }
      KMX_CAND_H(1) KMX_CAND_H(2) KMX_CAND_H(3) KMX_CAND_H(4) KMX_CAND_H(6) KMX_CAND_H(8)
#undef KMX_CAND_H
    }
  if (env_int_tc("KMX_TC_PERSIST", 0) == 2) {  // the persistent forms only (a forced test path)
    std::vector<TcPlan> only;
    for (const TcPlan& p : v)
      if (tcp_ok(ma, mb, p)) {
        TcPlan q = p;
        q.persist = 1; q.NW = 8; q.TPC = q.ntiles; q.nranges = 1;
        only.push_back(q);
      }
    if (!only.empty()) return only;
  }
  std::vector<TcPlan> out;
  if (tcs_mode() != 0)
    for (int form = 0; form < 3; form++)  // one-shot, persistent, M = 64 windows
    for (int pitch : {32, 64, 128}) {
      if (tcs_mode() >= 32 && tcs_mode() != pitch) continue;
      if (tcs_persist_mode() >= 0 && tcs_persist_mode() != form) continue;
      TcPlan q;
      q.sp = TcsPlan();
      if (!tcs_plan(ma, mb, pitch, form, q.sp)) continue;
      q.swz = pitch;
      q.H = pitch / 16; q.NW = 4; q.KC = q.sp.KS; q.NB = 1; q.TPC = 1;
      q.nranges = q.sp.ntiles; q.ntiles = q.sp.ntiles; q.nseg = 1;
      q.smem = q.sp.smem; q.cost = q.sp.cost;
      out.push_back(q);
    }
  // the persistent forms join the candidates only on request: measured at c2
  // they run 2.4x slower than the one-shot kernel (one MMA pipeline and one
  // 4-warp epilogue per CTA, 1-3 CTAs per SM, against ~8 one-shot CTAs whose
  // epilogues overlap each other's MMAs), and were never chosen
  const int pers = env_int_tc("KMX_TC_PERSIST", 0);
  // With swizzled-window candidates in the list (they won every measured shape)
  // only the tiled kernel's model-best tilings stay, as a cross-check; the wide
  // tiled field is timed only where the swizzled-window kernel has no plan.
  const bool have_swz = !out.empty();
  const double keep = have_swz ? 1.05 : 1.6;
  for (const TcPlan& p : v)
    if (p.cost <= keep * best) {
      out.push_back(p);
      if (have_swz) continue;
      if (pers && tcp_ok(ma, mb, p)) {  // the persistent form of the same tiling
        TcPlan q = p;
        q.persist = 1;
        q.NW = 8;
        q.TPC = q.ntiles;
        q.nranges = 1;
        out.push_back(q);
      }
      // fewer tiles per CTA (more, shorter CTAs): a better last wave on long
      // products whose CTAs fill an SM each
      for (int tpc : {p.TPC / 2, (p.TPC * 2) / 3}) {
        if (tpc < 1 || tpc >= p.TPC) continue;
        TcPlan q = p;
        q.TPC = tpc;
        q.nranges = (p.ntiles + tpc - 1) / tpc;
        bool dup = false;
        for (const TcPlan& r : out) dup |= r.H == q.H && r.KC == q.KC && r.NW == q.NW && r.TPC == q.TPC;
        if (!dup) out.push_back(q);
      }
    }
  return out;
}

struct TuneKey {
  int dev, ma, mb;
  long long nprod;
  bool operator<(const TuneKey& o) const {
    if (dev != o.dev) return dev < o.dev;
    return ma != o.ma ? ma < o.ma : (mb != o.mb ? mb < o.mb : nprod < o.nprod);
  }
};
int current_device() {
  int d = 0;
  cudaGetDevice(&d);
  return d;
}
std::mutex g_tune_mu;
std::map<TuneKey, TcPlan> g_tune;

// Measured plan choice, once per (shape, batch): the first call outside a CUDA
// graph capture times every candidate tiling on the caller's stream (second of
// two launches each, CUDA events; every candidate writes the same bit-exact
// product, so the output is valid whichever runs last) and caches the
// fastest.  The cost model alone misses by up to 30% on long products
// (tools/tc_sweep.py).  KMX_TC_AUTOTUNE=0, or any KMX_TC_H/KC/NW/NB/TPC
// override, keeps the model's choice.
bool tc_tuned_plan(const MulArgs& a, cudaStream_t st, TcPlan& p, bool* launched) {
  *launched = false;
  static const int on = env_int_tc("KMX_TC_AUTOTUNE", 1) && !getenv("KMX_TC_H") && !getenv("KMX_TC_KC") &&
                        !getenv("KMX_TC_NW") && !getenv("KMX_TC_NB") && !getenv("KMX_TC_TPC");
  if (!on) return false;
  if (a.flags_no_tune) return false;
  // small launches (e.g. single drop-in products) keep the model's plan: the
  // timing runs would cost more than any plan difference
  if ((double)a.nprod * a.ma * a.mb < (double)(1 << 24)) return false;
  const TuneKey key{current_device(), a.ma, a.mb, a.nprod};
  {
    std::lock_guard<std::mutex> lk(g_tune_mu);
    auto it = g_tune.find(key);
    if (it != g_tune.end()) { p = it->second; return true; }
  }
  // the lock is not held while timing: another thread tuning the same key
  // concurrently does redundant work but stores an equally valid plan
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(st, &cs) != cudaSuccess || cs != cudaStreamCaptureStatusNone) return false;
  std::vector<TcPlan> cands = tc_candidates(a.ma, a.mb, a.nprod);
  if (cands.size() < 2) return false;
  cudaEvent_t e0, e1;
  if (cudaEventCreate(&e0) != cudaSuccess || cudaEventCreate(&e1) != cudaSuccess) return false;
  float best_ms = 1e30f;
  int best = -1;
  for (size_t i = 0; i < cands.size(); i++) {
    if (launch_plan(a, cands[i], st, nullptr, 1) != cudaSuccess) continue;
    cudaEventRecord(e0, st);
    if (launch_plan(a, cands[i], st, nullptr, 1) != cudaSuccess) continue;
    cudaEventRecord(e1, st);
    if (cudaEventSynchronize(e1) != cudaSuccess) continue;
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best_ms) { best_ms = ms; best = (int)i; }
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  if (best < 0) return false;
  p = cands[best];
  {
    std::lock_guard<std::mutex> lk(g_tune_mu);
    g_tune[key] = p;
  }
  if (env_int_tc("KMX_TC_VERBOSE", 0))
    fprintf(stderr, "kmx_tc autotune: ma=%d mb=%d nprod=%d -> %s H=%d NW=%d KC=%d (%.4f ms of %zu candidates)\n", a.ma,
            a.mb, a.nprod, p.swz ? (p.sp.persist ? "swizzled-window persistent" : "swizzled-window") : "tiled", p.H, p.NW,
            p.KC, best_ms, cands.size());
  // re-run the winner last so the buffers hold its (identical) output in order
  if (launch_plan(a, p, st, nullptr, 1) != cudaSuccess) return false;
  *launched = true;
  return true;
}
}  // namespace

// K2 + K3 in one launch (kmx_tcs.cu, pair CTAs): when every product is one
// tile of a swizzled-window plan and K3 would be the warp-per-stream finish.
// Opt-in (KMX_FUSE_FIN=1): bit-exact, but measured slower than the two
// kernels at c2 (ks4: 118.7 us against 80.3 + 29.4; ks3: 212 against 99 + 62)
// -- a pair CTA holds its shared memory and TMEM through the finish, so fewer
// MMA phases overlap.  Returns true when the fused kernel ran.
bool launch_tcmul_finish(const MulArgs& a, const FinishArgs& fa, int batch, cudaStream_t st, cudaError_t* err) {
  *err = cudaSuccess;
  if (env_int_tc("KMX_FUSE_FIN", 0) == 0 || tcs_mode() == 0 || tcs_persist_mode() == 1) return false;
  if (fa.ns < 1 || fa.ns > 4 || fa.nprod_pair < 1 || a.nprod != (long long)batch * fa.nprod_pair) return false;
  if (!finish_use_warp(fa, batch) || finish_use_chunks(fa, batch)) return false;  // K3 = k_finish_w only
  bool ok = false;
  TcsPlan best;
  for (int pitch : {32, 64, 128}) {
    if (tcs_mode() >= 32 && tcs_mode() != pitch) continue;
    TcsPlan sp;
    if (!tcs_plan(a.ma, a.mb, pitch, 0, sp) || sp.ntiles != 1) continue;
    if (!ok || sp.cost < best.cost) best = sp;
    ok = true;
  }
  if (!ok) return false;
  *err = launch_tcs(a, best, st, &fa);
  return true;
}

cudaError_t launch_tcmul(const MulArgs& a, cudaStream_t st, const PackArgs* pk, int P) {
  TcPlan p;
  size_t stage = 0;
  if (pk) {
    int lmax = 0;
    for (int i = 0; i < pk->nops; i++) lmax = pk->op[i].len > lmax ? pk->op[i].len : lmax;
    stage = (size_t)(lmax + PK_PAD) * pk->in_words * 4;
  }
  const bool tiled_ok = tc_plan(a.ma, a.mb, a.nprod, stage, p);
  if (!tiled_ok && pk) return cudaErrorNotSupported;
  if (a.nprod == 0) return cudaSuccess;
  if (!pk && tiled_ok && env_int_tc("KMX_TC_PERSIST", 0) == 2 && tcp_ok(a.ma, a.mb, p)) {  // forced test path
    p.persist = 1; p.NW = 8; p.TPC = p.ntiles; p.nranges = 1;
    return launch_plan(a, p, st, nullptr, 1);
  }
  if (!pk) {
    TcPlan q;
    const bool swz_ok = tcs_best(a.ma, a.mb, q);
    if (!tiled_ok && !swz_ok) return cudaErrorNotSupported;
    if (swz_ok && tcs_mode() > 0) return launch_plan(a, q, st, nullptr, 1);  // forced, no timing runs
    // untuned default: the swizzled-window kernel wherever it takes the shape
    // (faster than the tiled kernel at every measured shape)
    if (swz_ok) p = q;
  }
  if (!pk) {
    bool launched = false;
    if (tc_tuned_plan(a, st, p, &launched) && launched) return cudaGetLastError();
  }
  return launch_plan(a, p, st, pk, P);
}

namespace {
template <int H>
cudaError_t launch_persist_h(const TcArgs& ta, int ma, int mb, cudaStream_t st) {
  const int mA = ma > mb ? ma : mb, mB = ma > mb ? mb : ma;
  const TcDims d = tc_dims<H>(mA, mB);
  const size_t smem = tcp_smem<H>(d.La, d.Lb, ta.KC, ta.NB);
  static size_t s_set = 0;
  if (smem > 48 * 1024 && smem > s_set) {
    cudaError_t e = cudaFuncSetAttribute(k_tcmul_p<H>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    s_set = smem;
  }
  int per_sm = 0;
  cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_tcmul_p<H>, 256, smem);
  if (e != cudaSuccess) return e;
  uint32_t acc = 32;
  while (acc < (uint32_t)(d.ntiles * 16 * H)) acc <<= 1;
  const int by_tmem = (int)(512 / (2 * acc));
  if (per_sm > by_tmem) per_sm = by_tmem;
  if (per_sm < 1) per_sm = 1;
  long long grid = (long long)tc_num_sms() * per_sm;
  if (grid > ta.m.nprod) grid = ta.m.nprod;
  if (grid < 1) return cudaSuccess;
  k_tcmul_p<H><<<(unsigned)grid, 256, smem, st>>>(ta);
  return cudaGetLastError();
}

cudaError_t launch_persist(const MulArgs& a, const TcPlan& p, cudaStream_t st) {
  TcArgs ta;
  memset(&ta, 0, sizeof ta);
  ta.m = a;
  ta.KC = p.KC;
  ta.NB = p.NB;
  ta.TPC = p.ntiles;
  ta.nranges = 1;
  ta.nseg = 1;
  ta.bulk = 1;
  if (a.nprod == 0) return cudaSuccess;
  switch (p.H) {
    case 1: return launch_persist_h<1>(ta, a.ma, a.mb, st);
    case 2: return launch_persist_h<2>(ta, a.ma, a.mb, st);
    case 3: return launch_persist_h<3>(ta, a.ma, a.mb, st);
    case 4: return launch_persist_h<4>(ta, a.ma, a.mb, st);
    case 6: return launch_persist_h<6>(ta, a.ma, a.mb, st);
    default: return launch_persist_h<8>(ta, a.ma, a.mb, st);
  }
}

cudaError_t launch_plan(const MulArgs& a, const TcPlan& p, cudaStream_t st, const PackArgs* pk, int P) {
  if (env_int_tc("KMX_TC_VERBOSE", 0))
    fprintf(stderr, "kmx_tc: ma=%d mb=%d nprod=%d -> H=%d NW=%d KC=%d NB=%d TPC=%d ranges=%d nseg=%d smem=%zu cost=%.0f%s\n",
            a.ma, a.mb, a.nprod, p.H, p.NW, p.KC, p.NB, p.TPC, p.nranges, p.nseg, p.smem, p.cost,
            p.persist ? " persistent" : "");
  if (p.swz && !pk) return launch_tcs(a, p.sp, st);
  if (p.persist && !pk) {
    // eligible only with bulk-copy-aligned operands (checked here, per launch)
    const bool swp = a.mb > a.ma;
    const long long as = swp ? a.b_stride : a.a_stride, bs = swp ? a.a_stride : a.b_stride;
    const int mA = swp ? a.mb : a.ma, mB = swp ? a.ma : a.mb;
    const bool al = ((reinterpret_cast<uintptr_t>(a.A) | reinterpret_cast<uintptr_t>(a.B)) & 15) == 0 &&
                    (as & 3) == 0 && (bs & 3) == 0 && as >= ((mA + 3) & ~3) && bs >= ((mB + 3) & ~3);
    if (al) return launch_persist(a, p, st);
  }
  TcArgs ta;
  ta.m = a;
  ta.bulk = env_int_tc("KMX_TC_BULK", 1);
  ta.KC = p.KC;
  ta.NB = p.NB;
  ta.fuse = pk != nullptr;
  ta.P = P;
  ta.ring = 0;
  if (pk) {
    ta.pk = *pk;
    ta.pk.stage = 1;
  }
  ta.TPC = p.TPC;
  ta.nranges = p.nranges;
  ta.nseg = p.nseg;
  cudaError_t e;
  switch (p.H) {
    case 1: e = launch_h<1>(ta, p.NW, p.smem, st); break;
    case 2: e = launch_h<2>(ta, p.NW, p.smem, st); break;
    case 3: e = launch_h<3>(ta, p.NW, p.smem, st); break;
    case 4: e = launch_h<4>(ta, p.NW, p.smem, st); break;
    case 6: e = launch_h<6>(ta, p.NW, p.smem, st); break;
    default: e = launch_h<8>(ta, p.NW, p.smem, st); break;
  }
  return e;
}
}  // namespace


namespace {
template <int H>
void tc_count(int ma, int mb, const TcPlan& p, long long out[8]) {
  const int mA = ma > mb ? ma : mb, mB = ma > mb ? mb : ma;
  const TcDims d = tc_dims<H>(mA, mB);
  long long mmas = 0, build_steps = 0;
  for (int r0 = 0; r0 < d.ntiles; r0 += p.TPC) {
    int lo = d.S, hi = 0;
    for (int t = r0; t < (r0 + p.TPC < d.ntiles ? r0 + p.TPC : d.ntiles); t++) {
      int slo, shi;
      tc_tile_steps<H>(d, t, slo, shi);
      if (shi > slo) {
        mmas += shi - slo;
        lo = slo < lo ? slo : lo;
        hi = shi > hi ? shi : hi;
      }
    }
    if (hi > lo) build_steps += hi - lo;
  }
  out[0] = 1; out[1] = H; out[2] = p.NW; out[3] = p.KC; out[4] = p.TPC;
  out[5] = mmas;
  // shared-memory bytes per product: each MMA reads its A tile (128 x 32 B)
  // and B tile (16H x 32 B); the builders write each staged B step once
  out[6] = mmas * (4096LL + 512LL * H) + build_steps * 512LL * H;
  out[7] = 128LL * 16 * H * 32 * mmas;  // issued byte MACs
}
}  // namespace

// The tiled tensor-core plan a launch of nprod products runs with (the
// autotuned one when cached, else the model's) and its work counts:
// out = {1, H, NW, KC, TPC, MMAs per product, smem operand bytes per product,
// issued byte MACs per product}.  false if the shape is not tensor-core.
bool tc_plan_info(int ma, int mb, long long nprod, long long out[8]) {
  TcPlan p, q;
  const bool tiled_ok = tc_plan(ma, mb, nprod, 0, p);
  if (tcs_best(ma, mb, q)) p = q;  // the untuned default
  else if (!tiled_ok) return false;
  {
    std::lock_guard<std::mutex> lk(g_tune_mu);
    auto it = g_tune.find(TuneKey{current_device(), ma, mb, nprod});
    if (it != g_tune.end()) p = it->second;
  }
  if (p.swz && p.sp.persist == 2) {  // M = 64 two-window form: A tile 64 x 32 B per MMA, rows up to 79 staged
    out[0] = 5; out[1] = p.H; out[2] = 4; out[3] = p.KC; out[4] = 1;
    out[5] = p.sp.mmas;
    out[6] = p.sp.mmas * (2048LL + 32LL * p.swz) + (16LL * 4 * (ma < mb ? ma : mb) + 79LL * p.swz + 4LL * (ma < mb ? ma : mb)) +
             2LL * 2 * (p.swz / 4) * 64 * 8;  // + the limb sums through shared memory (written, read)
    out[7] = 64LL * p.swz * 32 * p.sp.mmas;
    return true;
  }
  if (p.swz) {
    out[0] = 4; out[1] = p.H; out[2] = 4; out[3] = p.KC; out[4] = 1;
    out[5] = p.sp.mmas;
    // per MMA the A tile (128 x 32 B) and B tile (N x 32 B) are read; per CTA the
    // table (16 bytes per byte of b's chunk) and the a-window are written once
    out[6] = p.sp.mmas * (4096LL + 32LL * p.swz) +
             (long long)p.sp.ntiles * (16LL * 4 * (ma < mb ? ma : mb) + 127LL * p.swz + 4LL * (ma < mb ? ma : mb));
    out[7] = 128LL * p.swz * 32 * p.sp.mmas;
    return true;
  }
  switch (p.H) {
    case 1: tc_count<1>(ma, mb, p, out); break;
    case 2: tc_count<2>(ma, mb, p, out); break;
    case 3: tc_count<3>(ma, mb, p, out); break;
    case 4: tc_count<4>(ma, mb, p, out); break;
    case 6: tc_count<6>(ma, mb, p, out); break;
    default: tc_count<8>(ma, mb, p, out); break;
  }
  return true;
}

}  // namespace kmx
