// kmx_tcs.cu — K2 on the tensor cores without a per-K-step operand build:
// the byte convolution c[k] = sum_j a[k-j] b[j] of two packed operands
// (bignat.py:327-330, the classical product mul() reduces to) as
// tcgen05.mma kind::i8 with
//
//   A = sliding windows over the RAW bytes of a.  The bytes are stored once,
//       XOR-swizzled by their absolute shared-memory address, and read
//       through a SWIZZLE_32B / 64B / 128B K-major descriptor: rows are
//       PITCH = 32 / 64 / 128 bytes apart, so the M = 128 rows of one tile
//       span 128 * PITCH byte positions, and stepping K by 32 bytes only moves
//       the descriptor's start address (measured: the hardware swizzles on
//       absolute address bits, base_offset = 0, any 32-byte-aligned start;
//       tools/microbench/tc_swz.cu);
//   B = N = PITCH shifted, reversed copies of b.  They are never built per
//       K-step: ONE table of 8 byte phases
//           T[x][r][i] = b[r + c - 8x - i],   r < 8, i < 16   (128 B per x)
//       read with LBO = 256, SBO = 128 (SWIZZLE_NONE) makes row n = r + 8g,
//       K-half q of K-step s the entry x = 4s + g + 2q -- linear in g and q,
//       so a plain descriptor addresses it and consecutive K-steps advance
//       the start by 512 bytes.  Row n then holds b[beta_n - u],
//       beta_n = (n % 8) - 8 (n / 8) + N - 8: the N rows cover the N byte
//       offsets between two A rows (in a permuted order the epilogue undoes).
//
// D[m][n] = c[k0 + PITCH m + beta_n]: TMEM lane m owns PITCH contiguous
// byte positions = PITCH/4 product limbs, so the epilogue needs no
// shared-memory transpose: limb sums from the lane's own columns, a local
// carry chain, and one block scan of {0,1} carry maps.
//
// Compared with k_tcmul (kmx_tc.cu: 16H shifted copies rebuilt per K-step, N =
// 16H <= 128 at 38H builder cycles per step) the table costs 16 bytes of
// shared-memory writes per byte of b ONCE per CTA, N is 64 or 128 at no
// extra build cost, and a c2 ks4 product (2436 x 2436 bytes) is one tile of
// 79 MMAs instead of two tiles of 108.
//
// One CTA per (product, tile).  Long operands walk K in chunks of KS steps:
// per chunk the CTA stages the a-window the tile needs (127 PITCH + 32 KS
// bytes) and the table of that chunk of b; accumulation continues in TMEM.
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "kmx_internal.h"
#include "kmx_common.cuh"
#include "kmx_tcutil.cuh"
#include "kmx_finish.cuh"

namespace kmx {

namespace {

template <int PITCH>
struct SG {
  static constexpr int N = PITCH;
  static constexpr int T = 128 * PITCH;        // byte positions per tile
  static constexpr int LIMBS = 32 * PITCH;     // product limbs per tile
  static constexpr int LPT = PITCH / 4;        // limbs per TMEM lane
  static constexpr int BPT = PITCH / 8;        // 256-limb bands per tile
  static constexpr int AMAX = 127 * PITCH;     // offset of the last A row
  static constexpr uint32_t LT = PITCH == 128 ? 2u : PITCH == 64 ? 4u : 6u;  // descriptor layout type
  static constexpr uint32_t MASK = PITCH / 16 - 1;  // swizzle: address bits [4,4+B) ^= bits [7,7+B)
  static constexpr uint32_t IDESC = (2u << 4) | ((uint32_t)(N >> 3) << 17) | (8u << 24);
};

struct TcsDims {
  int La, Lb, ulo, S, ntiles;
};
template <int PITCH>
__host__ __device__ inline TcsDims tcs_dims(int mA, int mB) {
  TcsDims d;
  d.La = 4 * mA;
  d.Lb = 4 * mB;
  d.ulo = -32 * ((d.Lb - 1 + 31) / 32);
  d.S = fdiv32(SG<PITCH>::N - 1 - d.ulo) + 1;
  d.ntiles = (d.La + d.Lb - 1 + SG<PITCH>::T - 1) / SG<PITCH>::T;
  return d;
}
// K-steps [slo, shi) in which some row of tile t reads a byte of a
template <int PITCH>
__host__ __device__ inline void tcs_tile_steps(const TcsDims& d, int t, int& slo, int& shi) {
  const int k0 = t * SG<PITCH>::T;
  slo = -fdiv32(k0 + SG<PITCH>::AMAX + 31 + d.ulo);
  if (slo < 0) slo = 0;
  shi = fdiv32(d.La - k0 - 1 - d.ulo) + 1;
  if (shi > d.S) shi = d.S;
}

struct TcsShared {
  unsigned long long bar_mma;  // the chunk's MMAs completed (tcgen05.commit)
  unsigned long long s_cout[4];
  uint32_t tmem_base;
  uint32_t warp_map[4];
};

__host__ __device__ inline size_t r128(size_t x) { return (x + 127) & ~(size_t)127; }
__host__ __device__ inline size_t r1024(size_t x) { return (x + 1023) & ~(size_t)1023; }
template <int PITCH>
__host__ __device__ inline size_t tcs_abytes(int KS) { return r1024((size_t)SG<PITCH>::AMAX + 32 * KS + 64); }
// M = 64 form: rows up to R0 + 63 <= 79 are read
template <int PITCH>
__host__ __device__ inline size_t tcs_abytes64(int KS) { return r1024((size_t)79 * PITCH + 32 * KS + 64); }
template <int PITCH>
__host__ __device__ inline int tcs_rawbytes(int KS) { return (int)r128((size_t)32 * KS + PITCH + 96); }
template <int PITCH>
__host__ __device__ inline int tcs_entries(int KS) { return 4 * KS + PITCH / 8 + 2; }
template <int PITCH>
__host__ __device__ inline size_t tcs_smem(int KS) {
  return 1024 + r128(sizeof(TcsShared)) + tcs_abytes<PITCH>(KS) + tcs_rawbytes<PITCH>(KS) +
         (size_t)tcs_entries<PITCH>(KS) * 128;
}
template <int PITCH>
__host__ __device__ inline size_t tcs_smem64(int KS) {
  return 1024 + r128(sizeof(TcsShared)) + tcs_abytes64<PITCH>(KS) + tcs_rawbytes<PITCH>(KS) +
         (size_t)tcs_entries<PITCH>(KS) * 128;
}

constexpr int TCS_MAXT = 48;  // tiles per product the persistent kernel orders
struct TcsArgs {
  MulArgs m;
  int KS;      // K-steps per chunk
  int ntiles;  // CTAs per product
  int nch;     // accumulation chains per tile (K-step s -> chain (s - slo) % nch): 2 past 64 KB of b
  int NS;      // persistent kernel: operand stages in the ring
  unsigned char order[TCS_MAXT];  // persistent kernel: tiles by descending K-steps
  int smid, r0;  // M = 64 form: K-steps < smid read rows [r0, r0 + 64), the rest rows [0, 64)
};

__device__ __forceinline__ uint64_t sdesc_lt(uint32_t addr, uint32_t lbo, uint32_t sbo, uint32_t lt) {
  return sdesc(addr, lbo, sbo) | ((uint64_t)lt << 61);
}

// One lane polls the mbarrier, the warp joins at __syncwarp: every polling
// lane's try_wait is a shared-memory access, and this kernel is bound by
// shared-memory bandwidth (ncu: tensor-operand reads 73% + LSU 28% of the
// pipe with all 128 threads polling).
__device__ __forceinline__ void mbar_wait_warp(uint32_t mbar, uint32_t parity) {
  if ((threadIdx.x & 31) == 0) mbar_wait(mbar, parity);
  __syncwarp();
}

// The MMA is issued from WARP-UNIFORM code: every lane of the issuing warp
// runs the loop and computes the (uniform) descriptors, one elected lane
// executes the instruction.  With the loop inside an `if (lane == 0)` branch
// ptxas cannot prove the operands uniform and wraps every UTCIMMA in a
// vote / elect / 5x R2UR waterfall (~90 cycles per MMA, measured); issued
// this way the descriptors live in uniform registers.
__device__ __forceinline__ void mma_i8_elect(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                             uint32_t accum) {
  asm volatile(
      "{\n\t.reg .pred p, q;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "elect.sync _|q, 0xffffffff;\n\t"
      "@q tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accum));
}
__device__ __forceinline__ void mma_commit_elect(uint32_t mbar) {
  asm volatile(
      "{\n\t.reg .pred q;\n\t"
      "elect.sync _|q, 0xffffffff;\n\t"
      "@q tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}\n" ::"r"(mbar)
      : "memory");
}


// One K-chunk's operands for tile k0: the swizzled a-window, the raw bytes of
// b's chunk and its phase table, built by 128 threads (ptid) in three steps
// so a persistent producer can issue the NEXT chunk's global loads before it
// builds the current chunk's table:
//   tcs_load   global -> registers (the a-window's 16-byte pieces, b's words)
//   tcs_store  registers -> shared memory (a swizzled by address, b raw)
//   tcs_table  b raw -> phase table (after a barrier over the 128 threads)
constexpr int TCS_NA = 10;   // 16-byte a pieces per thread: (127*128 + 32*128) / 16 / 128
constexpr int TCS_NBW = 9;   // b words per thread: (32*128 + 128 + 96) / 4 / 128
constexpr int TCS_KSMAX = 128;
struct TcsRegs {
  uint4 va[TCS_NA];
  uint32_t vb[TCS_NBW];
};
template <int PITCH>
struct TcsChunk {  // geometry of one chunk (all warp-uniform)
  int aw0, nq, x0, nx, jb, nw;
  __device__ __forceinline__ TcsChunk(const TcsDims& d, int k0, int sb, int se, int amax = SG<PITCH>::AMAX) {
    using G = SG<PITCH>;
    const int cc = G::N - 8 - d.ulo;  // T[x][r][i] = b[r + cc - 8x - i]
    aw0 = k0 + d.ulo + 32 * sb;       // region byte o is a[aw0 + o]; a multiple of 32
    nq = (amax + 32 * (se - sb) + 15) / 16;  // amax: offset of the last A row that is read
    x0 = 4 * sb;
    nx = 4 * (se - sb) + G::N / 8 - 2;  // entries x0 .. x0 + nx - 1 are read
    const int jlo = cc - 8 * (x0 + nx - 1) - 15;  // lowest index r + cc - 8x - i
    jb = ((jlo >> 2) << 2) - 16;  // braw[k] = b[jb + k]: a multiple of 4, four spare words below (sliding loads)
    nw = (7 + cc - 8 * x0 - jb) / 4 + 1;
  }
};

template <int PITCH>
__device__ __forceinline__ void tcs_load(TcsRegs& R, const TcsChunk<PITCH>& c, const uint32_t* __restrict__ Ag,
                                         const uint32_t* __restrict__ Bg, int mA, int mB, bool a16, int ptid) {
#pragma unroll
  for (int k = 0; k < TCS_NA; k++) {
    const int q = 128 * k + ptid;
    const int j = (c.aw0 + 16 * q) >> 2;  // first limb of the piece (a multiple of 4, may be negative)
    uint4 v = make_uint4(0u, 0u, 0u, 0u);
    if (q < c.nq && j + 3 >= 0 && j < mA) {
      if (a16 && j >= 0 && j + 3 < mA) {
        v = __ldg(reinterpret_cast<const uint4*>(Ag + j));
      } else {
        v.x = (j >= 0 && j < mA) ? __ldg(Ag + j) : 0u;
        v.y = (j + 1 >= 0 && j + 1 < mA) ? __ldg(Ag + j + 1) : 0u;
        v.z = (j + 2 >= 0 && j + 2 < mA) ? __ldg(Ag + j + 2) : 0u;
        v.w = (j + 3 >= 0 && j + 3 < mA) ? __ldg(Ag + j + 3) : 0u;
      }
    }
    R.va[k] = v;
  }
#pragma unroll
  for (int k = 0; k < TCS_NBW; k++) {
    const int w = 128 * k + ptid;
    const int j = (c.jb >> 2) + w;
    R.vb[k] = (w < c.nw && j >= 0 && j < mB) ? __ldg(Bg + j) : 0u;
  }
}

template <int PITCH>
__device__ __forceinline__ void tcs_store(const TcsRegs& R, const TcsChunk<PITCH>& c, unsigned char* abuf,
                                          unsigned char* braw, int ptid) {
  using G = SG<PITCH>;
  const uint32_t abase = smem_u32(abuf);
#pragma unroll
  for (int k = 0; k < TCS_NA; k++) {
    const int q = 128 * k + ptid;
    if (q < c.nq) {
      const uint32_t L = abase + 16u * (uint32_t)q;
      const uint32_t P = L ^ (((L >> 7) & G::MASK) << 4);
      *reinterpret_cast<uint4*>(abuf + (P - abase)) = R.va[k];
    }
  }
  uint32_t* bw = reinterpret_cast<uint32_t*>(braw);
#pragma unroll
  for (int k = 0; k < TCS_NBW; k++) {
    const int w = 128 * k + ptid;
    if (w < c.nw) bw[w] = R.vb[k];
  }
}

// thread (r = ptid % 8, run = ptid / 8) builds a contiguous run of entries;
// consecutive entries move the 16-byte window down by 8 bytes, so five words
// slide through registers with two new loads per entry
template <int PITCH>
__device__ __forceinline__ void tcs_table(const TcsChunk<PITCH>& c, const TcsDims& d, const unsigned char* braw,
                                          unsigned char* tab, int ptid) {
  using G = SG<PITCH>;
  const int cc = G::N - 8 - d.ulo;
  const int r = ptid & 7, run = ptid >> 3;
  const int XB = (c.nx + 15) / 16;
  const int xa = run * XB, xe = min(c.nx, xa + XB);
  if (xa < xe) {
    const uint32_t* bw = reinterpret_cast<const uint32_t*>(braw);
    // entry bytes i = 0..15: braw[e - i], e = r + cc - 8 (x0 + x) - jb  (>= 15 + 16)
    const int e = r + cc - 8 * (c.x0 + xa) - c.jb;
    int wq = e >> 2;
    const int sh2 = e & 3;
    // output byte k of a word = byte (4 + sh2 - k) of {lo, hi}
    const uint32_t sel = (uint32_t)(4 + sh2) | ((uint32_t)(3 + sh2) << 4) | ((uint32_t)(2 + sh2) << 8) |
                         ((uint32_t)(1 + sh2) << 12);
    uint32_t w0 = bw[wq], w1 = bw[wq - 1], w2 = bw[wq - 2], w3 = bw[wq - 3], w4 = bw[wq - 4];
    unsigned char* dst = tab + (size_t)xa * 128 + r * 16;
    for (int x = xa; x < xe; x++) {
      uint4 o;
      o.x = __byte_perm(w1, w0, sel);
      o.y = __byte_perm(w2, w1, sel);
      o.z = __byte_perm(w3, w2, sel);
      o.w = __byte_perm(w4, w3, sel);
      *reinterpret_cast<uint4*>(dst) = o;
      dst += 128;
      wq -= 2;
      w0 = w2; w1 = w3; w2 = w4;
      w3 = bw[wq - 3];
      w4 = bw[wq - 4];
    }
  }
}


// Epilogue, first half: TMEM lane m's LPT limb sums -> digits with carry-in 0.
// Limbs 4c .. 4c+3 live in columns [N - 16 - 16c, N - 16c): the upper 8 columns
// (g odd) hold byte offsets 16c .. 16c+7, the lower 8 hold 16c+8 .. 16c+15.
// The chains' partial sums are added in 64 bits.  Returns the carry out.
template <int PITCH>
__device__ __forceinline__ unsigned long long tcs_limbs(uint32_t tacc, int nch, bool have,
                                                        uint32_t (&dg)[SG<PITCH>::LPT]) {
  using G = SG<PITCH>;
  unsigned long long x = 0ull;
#pragma unroll
  for (int c = 0; c < G::N / 16; c++) {
    unsigned long long ls[4] = {0ull, 0ull, 0ull, 0ull};
    if (have) {
      for (int ch = 0; ch < nch; ch++) {
        uint32_t v[16];
        tmem_ld16(tacc + (uint32_t)(ch * G::N + G::N - 16 - 16 * c), v);
#pragma unroll
        for (int q = 0; q < 4; q++) {
          const int o = q < 2 ? 8 + 4 * q : 4 * (q - 2);
          ls[q] += (unsigned long long)v[o] + ((unsigned long long)v[o + 1] << 8) +
                   ((unsigned long long)v[o + 2] << 16) + ((unsigned long long)v[o + 3] << 24);
        }
      }
    }
#pragma unroll
    for (int q = 0; q < 4; q++) {
      x = (x >> 32) + ls[q];
      dg[4 * c + q] = (uint32_t)x;
    }
  }
  return x >> 32;
}

// PAIR = false: one CTA per (product, tile).
// PAIR = true (single-tile products only): one CTA per polynomial PAIR.  It
// multiplies the pair's nprod_pair products one after the other and then runs
// K3 for the pair -- the warp-per-stream finish (kmx_finish.cuh: half sums /
// differences, exact halving and shifts, digit extraction), one warp per
// output stream, on the products it has just written (they sit in L2).  The
// finish instructions fill issue slots the other resident CTAs' MMA phases
// leave idle, and the separate K3 launch disappears.
template <int PITCH, bool PAIR>
__global__ void __launch_bounds__(128) k_tcswz(TcsArgs ta, FinishArgs fa) {
  using G = SG<PITCH>;
  const MulArgs& a = ta.m;
  extern __shared__ __align__(1024) unsigned char ssm_raw[];
  const int tid = threadIdx.x, lane = tid & 31;
  const int warp = __shfl_sync(0xffffffffu, tid >> 5, 0);  // warp-uniform for the compiler
  unsigned char* ssm = ssm_raw + ((1024u - (smem_u32(ssm_raw) & 1023u)) & 1023u);
  const int KS = ta.KS;
  unsigned char* abuf = ssm;                                     // swizzled a-window
  unsigned char* braw = abuf + tcs_abytes<PITCH>(KS);            // raw bytes of b's chunk
  unsigned char* tab = braw + tcs_rawbytes<PITCH>(KS);           // phase table
  TcsShared& sh = *reinterpret_cast<TcsShared*>(tab + (size_t)tcs_entries<PITCH>(KS) * 128);

  // operand roles: a slides (longer), b goes through the table (shorter)
  const bool sw = a.mb > a.ma;
  const int mA = sw ? a.mb : a.ma, mB = sw ? a.ma : a.mb;
  const TcsDims d = tcs_dims<PITCH>(mA, mB);
  const int mp = a.ma + a.mb;
  const int t = PAIR ? 0 : (int)(blockIdx.x % ta.ntiles);
  const int nz = PAIR ? fa.nprod_pair : 1;
  const long long z0 = PAIR ? (long long)blockIdx.x * fa.nprod_pair : (long long)(blockIdx.x / ta.ntiles);
  const int k0 = t * G::T;
  int slo, shi;
  tcs_tile_steps<PITCH>(d, t, slo, shi);

  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&sh.tmem_base)),
                 "r"((uint32_t)(ta.nch * G::N)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    mbar_init(smem_u32(&sh.bar_mma), 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  const uint32_t abase = smem_u32(abuf);
  uint32_t tmem = 0u;
  uint32_t phase = 0u;
  bool have_tmem = false;
  constexpr int LPT = G::LPT;

  for (int zi = 0; zi < nz; zi++) {
    const long long z = z0 + zi;
    const uint32_t* Ag = sw ? a.B + z * a.b_stride : a.A + z * a.a_stride;
    const uint32_t* Bg = sw ? a.A + z * a.a_stride : a.B + z * a.b_stride;
    const bool a16 = (reinterpret_cast<uintptr_t>(Ag) & 15) == 0;
    bool first = true;
    for (int sb = slo; sb < shi; sb += KS) {
      const int se = min(shi, sb + KS);
      if (!first) {
        // the previous chunk's MMAs still read the buffers (warp 0 polls, the
        // others join at the barrier)
        if (warp == 0) mbar_wait_warp(smem_u32(&sh.bar_mma), phase);
        __syncthreads();
        phase ^= 1u;
      }
      {
        const TcsChunk<PITCH> ck(d, k0, sb, se);
        TcsRegs R;
        tcs_load<PITCH>(R, ck, Ag, Bg, mA, mB, a16, tid);
        tcs_store<PITCH>(R, ck, abuf, braw, tid);
        __syncthreads();
        tcs_table<PITCH>(ck, d, braw, tab, tid);
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncthreads();
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      if (!have_tmem) {
        tmem = __shfl_sync(0xffffffffu, sh.tmem_base, 0);
        have_tmem = true;
      }
      if (warp == 0) {
        uint64_t ad = sdesc_lt(abase, 16, 8 * PITCH, G::LT);
        uint64_t bd = sdesc(smem_u32(tab), 256, 128);
        // K-step s accumulates into chain (s - slo) & (nch - 1): with more than
        // 64 KB of b the u32 sums are exact only per half of the K-steps (at
        // most 65536 byte products < 2^16 each); the epilogue adds the chains
        const int nch = ta.nch;
        for (int s = sb; s < se; s++) {
          const uint32_t ch = (uint32_t)(s - slo) & (uint32_t)(nch - 1);
          mma_i8_elect(tmem + ch * G::N, ad, bd, G::IDESC, (s - slo) >= nch ? 1u : 0u);
          ad += 2;   // + 32 bytes
          bd += 32;  // + 512 bytes
        }
        mma_commit_elect(smem_u32(&sh.bar_mma));
      }
      first = false;
    }
    if (!first) {
      if (warp == 0) mbar_wait_warp(smem_u32(&sh.bar_mma), phase);
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncthreads();
      phase ^= 1u;
    }
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (!have_tmem) {  // no K-step touches this tile (cannot happen for t < ntiles; kept for safety)
      __syncthreads();
      tmem = __shfl_sync(0xffffffffu, sh.tmem_base, 0);
      have_tmem = true;
    }

    // ---- epilogue: lane m = tid owns limbs [LPT m, LPT m + LPT) of the tile
    uint32_t dg[LPT];
    // (a tile with fewer K-steps than chains never wrote the later chains)
    const unsigned long long cout =
        tcs_limbs<PITCH>(tmem + ((uint32_t)(32 * warp) << 16), min(ta.nch, shi - slo), !first, dg);
    unsigned long long xin = __shfl_up_sync(0xffffffffu, cout, 1);
    if (lane == 31) sh.s_cout[warp] = cout;
    uint32_t ones = 0xFFFFFFFFu;
#pragma unroll
    for (int q = 1; q < LPT; q++) ones &= dg[q];
    // (also orders this product's TMEM reads before the next product's MMAs)
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (lane == 0) xin = warp ? sh.s_cout[warp - 1] : 0ull;
    // overflow of (digits + xin + o) past the lane's LPT limbs, o in {0,1} from the previous lane
    const unsigned long long s0 = (unsigned long long)dg[0] + xin;
    const bool all1 = ones == 0xFFFFFFFFu;
    const uint32_t gg = all1 && (s0 >> 32) != 0ull;
    const uint32_t pp = all1 && ((s0 + 1ull) >> 32) != 0ull;
    uint32_t F = gg | (pp << 1);
#pragma unroll
    for (int dd = 1; dd < 32; dd <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, F, dd);
      if (lane >= dd) F = cm2(F, y);
    }
    if (lane == 31) sh.warp_map[warp] = F;
    __syncthreads();
    uint32_t E = __shfl_up_sync(0xffffffffu, F, 1);
    uint32_t Wm = CM2_ID;
    for (int w = 0; w < warp; w++) Wm = cm2(sh.warp_map[w], Wm);
    // the tile's carry-in is 0: evaluate the composed maps at 0
    E = lane ? cm2(E, Wm) : Wm;
    const uint32_t Fin = cm2(F, Wm);
    unsigned long long acc = s0 + (E & 1u);
    dg[0] = (uint32_t)acc;
#pragma unroll
    for (int q = 1; q < LPT; q++) {
      acc = (acc >> 32) + dg[q];
      dg[q] = (uint32_t)acc;
    }
    uint32_t* Pz = a.P + z * a.p_stride;
    const int L = t * G::LIMBS + LPT * tid;
    if (L + LPT <= mp) {
#pragma unroll
      for (int q = 0; q < LPT / 4; q++)
        *reinterpret_cast<uint4*>(Pz + L + 4 * q) = make_uint4(dg[4 * q], dg[4 * q + 1], dg[4 * q + 2], dg[4 * q + 3]);
    } else {
#pragma unroll
      for (int q = 0; q < LPT; q++)
        if (L + q < mp) Pz[L + q] = dg[q];
    }
    // band spills: zero inside the tile, the tile's carry on its top band
    {
      const int b0 = G::BPT * t, b1 = min(a.nbands, G::BPT * (t + 1));
      if (tid < b1 - b0 && tid != G::BPT - 1) {
        unsigned long long* sp = a.spill + (z * a.nbands + b0 + tid) * 2;
        sp[0] = 0ull;
        sp[1] = 0ull;
      }
      if (tid == 127 && b0 + G::BPT - 1 < b1) {
        unsigned long long* sp = a.spill + (z * a.nbands + b0 + G::BPT - 1) * 2;
        sp[0] = cout + (Fin & 1u);
        sp[1] = 0ull;
      }
    }
  }
  if (PAIR) {
    // K3 for this pair: the products and spills above were written by this
    // CTA (visible after the barrier; read with plain loads, not ld.global.nc)
    __syncthreads();
    u32* fbuf = reinterpret_cast<u32*>(abuf) + warp * (FIN_HALO + FW_CH);
    if (warp < fa.ns)
      finish_warp_stream<GlobalDigitSink, false>(fa, (int)blockIdx.x, warp, fbuf, GlobalDigitSink{&fa});
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"((uint32_t)(ta.nch * G::N)));
}

// ------------------------------------------------------------------------
// M = 64 form for products of at most 64 + R0 rows of PITCH bytes (c2 ks4: 77
// rows of 64).  In a 128-row tile of such a product only ~39 rows are live at
// any K-step -- the rows whose A window holds bytes of a -- and the live band
// slides down by half a row per step.  An M = 128 instruction reads all 128
// rows of A from shared memory every step; here the K-steps are issued as
// M = 64 instructions over TWO row windows: the early steps (live rows high)
// read rows [R0, R0 + 64) into a second accumulator, the late steps rows
// [0, 64) into the first.  A step then reads 2 + 2 KB instead of 4 + 2 KB of
// shared memory (measured 36.6 against 62 SM cycles per step at N = 64, 3 CTAs
// per SM: tools/microbench/tc_m64.cu).  An M = 64 accumulator keeps tile row r
// in TMEM lane (r % 16) + 32 (r / 16) (same microbenchmark), so the epilogue
// passes the lanes' limb sums through shared memory into row order, adds the
// two windows where they overlap, and continues as k_tcswz does.
// ------------------------------------------------------------------------
template <int PITCH>
__global__ void __launch_bounds__(128) k_tcswz_m64(TcsArgs ta) {
  using G = SG<PITCH>;
  constexpr int LPT = G::LPT;
  constexpr uint32_t IDESC64 = (2u << 4) | ((uint32_t)(G::N >> 3) << 17) | (4u << 24);
  const MulArgs& a = ta.m;
  extern __shared__ __align__(1024) unsigned char ssm_raw[];
  const int tid = threadIdx.x, lane = tid & 31;
  const int warp = __shfl_sync(0xffffffffu, tid >> 5, 0);
  unsigned char* ssm = ssm_raw + ((1024u - (smem_u32(ssm_raw) & 1023u)) & 1023u);
  const int KS = ta.KS;
  unsigned char* abuf = ssm;
  unsigned char* braw = abuf + tcs_abytes64<PITCH>(KS);
  unsigned char* tab = braw + tcs_rawbytes<PITCH>(KS);
  TcsShared& sh = *reinterpret_cast<TcsShared*>(tab + (size_t)tcs_entries<PITCH>(KS) * 128);

  const bool sw = a.mb > a.ma;
  const int mA = sw ? a.mb : a.ma, mB = sw ? a.ma : a.mb;
  const TcsDims d = tcs_dims<PITCH>(mA, mB);
  const int mp = a.ma + a.mb;
  const long long z = blockIdx.x;
  int slo, shi;
  tcs_tile_steps<PITCH>(d, 0, slo, shi);
  const int R0 = ta.r0, smid = ta.smid;

  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&sh.tmem_base)),
                 "r"((uint32_t)(2 * G::N)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    mbar_init(smem_u32(&sh.bar_mma), 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  const uint32_t abase = smem_u32(abuf);
  const uint32_t* Ag = sw ? a.B + z * a.b_stride : a.A + z * a.a_stride;
  const uint32_t* Bg = sw ? a.A + z * a.a_stride : a.B + z * a.b_stride;
  const bool a16 = (reinterpret_cast<uintptr_t>(Ag) & 15) == 0;
  {
    // one chunk: the whole K span; rows up to R0 + 63 are read
    const TcsChunk<PITCH> ck(d, 0, slo, shi, (R0 + 63) * PITCH);
    TcsRegs R;
    tcs_load<PITCH>(R, ck, Ag, Bg, mA, mB, a16, tid);
    tcs_store<PITCH>(R, ck, abuf, braw, tid);
    __syncthreads();
    tcs_table<PITCH>(ck, d, braw, tab, tid);
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = __shfl_sync(0xffffffffu, sh.tmem_base, 0);
  if (warp == 0) {
    uint64_t ad0 = sdesc_lt(abase, 16, 8 * PITCH, G::LT);                              // rows [0, 64)
    uint64_t ad1 = sdesc_lt(abase + (uint32_t)(R0 * PITCH), 16, 8 * PITCH, G::LT);     // rows [R0, R0 + 64)
    uint64_t bd = sdesc(smem_u32(tab), 256, 128);
    for (int s = slo; s < shi; s++) {
      const bool hi = s < smid;
      mma_i8_elect(tmem + (hi ? (uint32_t)G::N : 0u), hi ? ad1 : ad0, bd, IDESC64,
                   (s == slo || s == smid) ? 0u : 1u);
      ad0 += 2; ad1 += 2;  // + 32 bytes
      bd += 32;            // + 512 bytes
    }
    mma_commit_elect(smem_u32(&sh.bar_mma));
    mbar_wait_warp(smem_u32(&sh.bar_mma), 0u);
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");

  // ---- limb sums of the two accumulators into row order (the table's shared memory is free now):
  // S[w][q][r] = sum of limb q of tile row r of window w, u64
  unsigned long long* S0 = reinterpret_cast<unsigned long long*>(tab);
  unsigned long long* S1 = S0 + LPT * 64;
  {
    // (tcgen05.ld is warp-wide: every lane loads, the lower half-warp holds the rows)
    const int tr = 16 * warp + (lane & 15);  // tile row held by TMEM lane 32 warp + lane, lane < 16
    const uint32_t tl = tmem + ((uint32_t)(32 * warp) << 16);
#pragma unroll
    for (int w = 0; w < 2; w++) {
      const bool have = w == 0 ? shi > smid && shi > slo : smid > slo;
      unsigned long long* Sw = w == 0 ? S0 : S1;
#pragma unroll
      for (int c = 0; c < G::N / 16; c++) {
        unsigned long long ls[4] = {0ull, 0ull, 0ull, 0ull};
        if (have) {  // warp-uniform
          uint32_t v[16];
          tmem_ld16(tl + (uint32_t)(w * G::N + G::N - 16 - 16 * c), v);
#pragma unroll
          for (int q = 0; q < 4; q++) {
            const int o = q < 2 ? 8 + 4 * q : 4 * (q - 2);
            ls[q] = (unsigned long long)v[o] + ((unsigned long long)v[o + 1] << 8) +
                    ((unsigned long long)v[o + 2] << 16) + ((unsigned long long)v[o + 3] << 24);
          }
        }
        if (lane < 16) {
#pragma unroll
          for (int q = 0; q < 4; q++) Sw[(4 * c + q) * 64 + tr] = ls[q];
        }
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();

  // ---- epilogue as k_tcswz: thread tid owns limbs [LPT tid, LPT tid + LPT) = row tid
  uint32_t dg[LPT];
  unsigned long long x = 0ull;
  {
    const int r = tid;
#pragma unroll
    for (int q = 0; q < LPT; q++) {
      unsigned long long lsq = 0ull;
      if (r < 64) lsq = S0[q * 64 + r];
      if (r >= R0 && r < R0 + 64) lsq += S1[q * 64 + r - R0];
      x = (x >> 32) + lsq;
      dg[q] = (uint32_t)x;
    }
  }
  const unsigned long long cout = x >> 32;
  unsigned long long xin = __shfl_up_sync(0xffffffffu, cout, 1);
  if (lane == 31) sh.s_cout[warp] = cout;
  uint32_t ones = 0xFFFFFFFFu;
#pragma unroll
  for (int q = 1; q < LPT; q++) ones &= dg[q];
  __syncthreads();
  if (lane == 0) xin = warp ? sh.s_cout[warp - 1] : 0ull;
  const unsigned long long s0 = (unsigned long long)dg[0] + xin;
  const bool all1 = ones == 0xFFFFFFFFu;
  const uint32_t gg = all1 && (s0 >> 32) != 0ull;
  const uint32_t pp = all1 && ((s0 + 1ull) >> 32) != 0ull;
  uint32_t F = gg | (pp << 1);
#pragma unroll
  for (int dd = 1; dd < 32; dd <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, F, dd);
    if (lane >= dd) F = cm2(F, y);
  }
  if (lane == 31) sh.warp_map[warp] = F;
  __syncthreads();
  uint32_t E = __shfl_up_sync(0xffffffffu, F, 1);
  uint32_t Wm = CM2_ID;
  for (int w = 0; w < warp; w++) Wm = cm2(sh.warp_map[w], Wm);
  E = lane ? cm2(E, Wm) : Wm;
  const uint32_t Fin = cm2(F, Wm);
  unsigned long long acc = s0 + (E & 1u);
  dg[0] = (uint32_t)acc;
#pragma unroll
  for (int q = 1; q < LPT; q++) {
    acc = (acc >> 32) + dg[q];
    dg[q] = (uint32_t)acc;
  }
  uint32_t* Pz = a.P + z * a.p_stride;
  const int L = LPT * tid;
  if (L + LPT <= mp) {
#pragma unroll
    for (int q = 0; q < LPT / 4; q++)
      *reinterpret_cast<uint4*>(Pz + L + 4 * q) = make_uint4(dg[4 * q], dg[4 * q + 1], dg[4 * q + 2], dg[4 * q + 3]);
  } else {
#pragma unroll
    for (int q = 0; q < LPT; q++)
      if (L + q < mp) Pz[L + q] = dg[q];
  }
  {
    const int b1 = min(a.nbands, G::BPT);
    if (tid < b1 && tid != G::BPT - 1) {
      unsigned long long* sp = a.spill + (z * a.nbands + tid) * 2;
      sp[0] = 0ull;
      sp[1] = 0ull;
    }
    if (tid == 127 && G::BPT - 1 < b1) {
      unsigned long long* sp = a.spill + (z * a.nbands + G::BPT - 1) * 2;
      sp[0] = cout + (Fin & 1u);
      sp[1] = 0ull;
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"((uint32_t)(2 * G::N)));
}

// ------------------------------------------------- persistent, specialized
// The same tiles through a persistent CTA (one per SM): work items (product,
// tile) in a static round-robin, heaviest tile class first, with the warps
// specialized and every hand-off on an mbarrier:
//   warps 0-3  epilogue of item i from TMEM accumulator i & 1 (lane quarter =
//              warp) while the MMAs of item i+1 fill the other accumulator;
//   warps 4-7  producers: the a-window, b's raw bytes and the phase table of
//              the next K-chunk into stage sc % NS of the operand ring;
//   warp 8     lane 0 issues the MMAs of each full stage and commits the
//              stage back to the producers.
// One product's operand build, MMAs and epilogue overlap its neighbours', and
// the K-chunks of long products are built while the previous chunk's MMAs run.
struct TcsSharedP {
  unsigned long long bar_full[4];       // stage built (128 producer threads arrive)
  unsigned long long bar_empty[4];      // the MMAs that read the stage completed (commit)
  unsigned long long bar_acc_full[2];   // the item's MMAs completed (commit)
  unsigned long long bar_acc_empty[2];  // the epilogue drained the accumulator (128 threads)
  unsigned long long s_cout[4];
  uint32_t tmem_base;
  uint32_t warp_map[4];
};
template <int PITCH>
__host__ __device__ inline size_t tcs_stage_bytes(int KS) {
  return tcs_abytes<PITCH>(KS) + tcs_rawbytes<PITCH>(KS) + r1024((size_t)tcs_entries<PITCH>(KS) * 128);
}
template <int PITCH>
__host__ __device__ inline size_t tcsp_smem(int KS, int NS) {
  return 1024 + (size_t)NS * tcs_stage_bytes<PITCH>(KS) + r128(sizeof(TcsSharedP));
}

template <int PITCH>
__global__ void __launch_bounds__(288, 1) k_tcswz_p(TcsArgs ta) {
  using G = SG<PITCH>;
  const MulArgs& a = ta.m;
  extern __shared__ __align__(1024) unsigned char ssm_raw[];
  const int tid = threadIdx.x, lane = tid & 31;
  const int warp = __shfl_sync(0xffffffffu, tid >> 5, 0);  // warp-uniform for the compiler
  unsigned char* ssm = ssm_raw + ((1024u - (smem_u32(ssm_raw) & 1023u)) & 1023u);
  const int KS = ta.KS, NS = ta.NS;
  const size_t stage_bytes = tcs_stage_bytes<PITCH>(KS);
  TcsSharedP& sh = *reinterpret_cast<TcsSharedP*>(ssm + (size_t)NS * stage_bytes);
  const bool sw = a.mb > a.ma;
  const int mA = sw ? a.mb : a.ma, mB = sw ? a.ma : a.mb;
  const long long astr = sw ? a.b_stride : a.a_stride, bstr = sw ? a.a_stride : a.b_stride;
  const uint32_t* Abase = sw ? a.B : a.A;
  const uint32_t* Bbase = sw ? a.A : a.B;
  const TcsDims d = tcs_dims<PITCH>(mA, mB);
  const int mp = a.ma + a.mb;
  const long long nitems = (long long)a.nprod * ta.ntiles;
  uint32_t COLS = 32;  // two accumulator buffers x nch chains
  while (COLS < (uint32_t)(2 * ta.nch * G::N)) COLS <<= 1;

  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&sh.tmem_base)),
                 "r"(COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    for (int i = 0; i < 4; i++) {
      mbar_init(smem_u32(&sh.bar_full[i]), 128);
      mbar_init(smem_u32(&sh.bar_empty[i]), 1);
    }
    for (int i = 0; i < 2; i++) {
      mbar_init(smem_u32(&sh.bar_acc_full[i]), 1);
      mbar_init(smem_u32(&sh.bar_acc_empty[i]), 128);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = __shfl_sync(0xffffffffu, sh.tmem_base, 0);

  if (warp >= 4 && warp < 8) {
    // ---------------- producers: the next chunk's global loads are in flight
    // while the current chunk's table is built
    const int ptid = tid - 128;
    long long sc = 0;
    long long it = blockIdx.x;
    int t = 0, slo = 0, shi = 0, sb = 0;
    const uint32_t *Ag = nullptr, *Bg = nullptr;
    bool a16 = false;
    bool valid = it < nitems;
    auto open_item = [&]() {
      t = ta.order[it / a.nprod];
      const long long z = it % a.nprod;
      Ag = Abase + z * astr;
      Bg = Bbase + z * bstr;
      a16 = (reinterpret_cast<uintptr_t>(Ag) & 15) == 0;
      tcs_tile_steps<PITCH>(d, t, slo, shi);
      sb = slo;
    };
    TcsRegs R;
    if (valid) {
      open_item();
      while (valid && slo >= shi) {  // (no empty tiles for t < ntiles; kept for safety)
        it += gridDim.x;
        valid = it < nitems;
        if (valid) open_item();
      }
    }
    if (valid) {
      const TcsChunk<PITCH> ck(d, t * G::T, sb, min(shi, sb + KS));
      tcs_load<PITCH>(R, ck, Ag, Bg, mA, mB, a16, ptid);
    }
    while (valid) {
      const int st = (int)(sc % NS);
      if (sc >= NS) mbar_wait_warp(smem_u32(&sh.bar_empty[st]), (uint32_t)(((sc / NS) - 1) & 1));
      unsigned char* abuf = ssm + (size_t)st * stage_bytes;
      unsigned char* braw = abuf + tcs_abytes<PITCH>(KS);
      unsigned char* tab = braw + tcs_rawbytes<PITCH>(KS);
      const TcsChunk<PITCH> ck(d, t * G::T, sb, min(shi, sb + KS));
      tcs_store<PITCH>(R, ck, abuf, braw, ptid);
      // advance to the next chunk (of this item or the next) and start its loads
      sb += KS;
      if (sb >= shi) {
        do {
          it += gridDim.x;
          valid = it < nitems;
          if (valid) open_item();
        } while (valid && slo >= shi);
      }
      if (valid) {
        const TcsChunk<PITCH> cn(d, t * G::T, sb, min(shi, sb + KS));
        tcs_load<PITCH>(R, cn, Ag, Bg, mA, mB, a16, ptid);
      }
      asm volatile("bar.sync 1, 128;" ::: "memory");
      tcs_table<PITCH>(ck, d, braw, tab, ptid);
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      mbar_arrive(smem_u32(&sh.bar_full[st]));
      sc++;
    }
  } else if (warp == 8) {
    // ---------------- MMA issuer (warp-uniform loop, one elected lane issues)
    {
      long long sc = 0, ac = 0;
      for (long long it = blockIdx.x; it < nitems; it += gridDim.x, ac++) {
        const int t = ta.order[it / a.nprod];
        int slo, shi;
        tcs_tile_steps<PITCH>(d, t, slo, shi);
        const int buf = (int)(ac & 1);
        if (ac >= 2) mbar_wait_warp(smem_u32(&sh.bar_acc_empty[buf]), (uint32_t)(((ac >> 1) - 1) & 1));
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t dcol = tmem + (uint32_t)(buf * ta.nch * G::N);
        const int nch = ta.nch;
        for (int sb = slo; sb < shi; sb += KS, sc++) {
          const int st = (int)(sc % NS);
          mbar_wait_warp(smem_u32(&sh.bar_full[st]), (uint32_t)((sc / NS) & 1));
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          const uint32_t sbase = smem_u32(ssm + (size_t)st * stage_bytes);
          uint64_t ad = sdesc_lt(sbase, 16, 8 * PITCH, G::LT);
          uint64_t bd = sdesc(sbase + (uint32_t)(tcs_abytes<PITCH>(KS) + tcs_rawbytes<PITCH>(KS)), 256, 128);
          const int se = min(shi, sb + KS);
          for (int s = sb; s < se; s++) {  // chain (s - slo) & (nch - 1), as in k_tcswz
            const uint32_t ch = (uint32_t)(s - slo) & (uint32_t)(nch - 1);
            mma_i8_elect(dcol + ch * G::N, ad, bd, G::IDESC, (s - slo) >= nch ? 1u : 0u);
            ad += 2;   // + 32 bytes
            bd += 32;  // + 512 bytes
          }
          mma_commit_elect(smem_u32(&sh.bar_empty[st]));
        }
        mma_commit_elect(smem_u32(&sh.bar_acc_full[buf]));
      }
    }
    __syncwarp();
  } else {
    // ---------------- epilogue (warps 0-3: TMEM lane quarter = warp)
    constexpr int LPT = G::LPT;
    long long ac = 0;
    for (long long it = blockIdx.x; it < nitems; it += gridDim.x, ac++) {
      const int t = ta.order[it / a.nprod];
      const long long z = it % a.nprod;
      int slo, shi;
      tcs_tile_steps<PITCH>(d, t, slo, shi);
      const int buf = (int)(ac & 1);
      mbar_wait_warp(smem_u32(&sh.bar_acc_full[buf]), (uint32_t)((ac >> 1) & 1));
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      uint32_t dg[LPT];
      const unsigned long long cout = tcs_limbs<PITCH>(
          tmem + ((uint32_t)(32 * warp) << 16) + (uint32_t)(buf * ta.nch * G::N), min(ta.nch, shi - slo), slo < shi, dg);
      // the accumulator is in registers: hand it back to the MMA warp
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      mbar_arrive(smem_u32(&sh.bar_acc_empty[buf]));
      unsigned long long xin = __shfl_up_sync(0xffffffffu, cout, 1);
      if (lane == 31) sh.s_cout[warp] = cout;
      uint32_t ones = 0xFFFFFFFFu;
#pragma unroll
      for (int q = 1; q < LPT; q++) ones &= dg[q];
      asm volatile("bar.sync 2, 128;" ::: "memory");
      if (lane == 0) xin = warp ? sh.s_cout[warp - 1] : 0ull;
      const unsigned long long s0 = (unsigned long long)dg[0] + xin;
      const bool all1 = ones == 0xFFFFFFFFu;
      const uint32_t gg = all1 && (s0 >> 32) != 0ull;
      const uint32_t pp = all1 && ((s0 + 1ull) >> 32) != 0ull;
      uint32_t F = gg | (pp << 1);
#pragma unroll
      for (int dd = 1; dd < 32; dd <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, F, dd);
        if (lane >= dd) F = cm2(F, y);
      }
      if (lane == 31) sh.warp_map[warp] = F;
      asm volatile("bar.sync 2, 128;" ::: "memory");
      uint32_t E = __shfl_up_sync(0xffffffffu, F, 1);
      uint32_t Wm = CM2_ID;
      for (int w = 0; w < warp; w++) Wm = cm2(sh.warp_map[w], Wm);
      E = lane ? cm2(E, Wm) : Wm;
      const uint32_t Fin = cm2(F, Wm);
      unsigned long long acc = s0 + (E & 1u);
      dg[0] = (uint32_t)acc;
#pragma unroll
      for (int q = 1; q < LPT; q++) {
        acc = (acc >> 32) + dg[q];
        dg[q] = (uint32_t)acc;
      }
      uint32_t* Pz = a.P + z * a.p_stride;
      const int L = t * G::LIMBS + LPT * tid;
      if (L + LPT <= mp) {
#pragma unroll
        for (int q = 0; q < LPT / 4; q++)
          *reinterpret_cast<uint4*>(Pz + L + 4 * q) = make_uint4(dg[4 * q], dg[4 * q + 1], dg[4 * q + 2], dg[4 * q + 3]);
      } else {
#pragma unroll
        for (int q = 0; q < LPT; q++)
          if (L + q < mp) Pz[L + q] = dg[q];
      }
      const int b0 = G::BPT * t, b1 = min(a.nbands, G::BPT * (t + 1));
      if (tid < b1 - b0 && tid != G::BPT - 1) {
        unsigned long long* sp = a.spill + (z * a.nbands + b0 + tid) * 2;
        sp[0] = 0ull;
        sp[1] = 0ull;
      }
      if (tid == 127 && b0 + G::BPT - 1 < b1) {
        unsigned long long* sp = a.spill + (z * a.nbands + b0 + G::BPT - 1) * 2;
        sp[0] = cout + (Fin & 1u);
        sp[1] = 0ull;
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(COLS));
}

int tcs_env(const char* n, int dflt) {
  const char* v = getenv(n);
  return v && *v ? atoi(v) : dflt;
}

int tcs_num_sms() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

// M = 64 form: the second window's first row R0 and the K-step smid from which every live row
// lies in [0, 64); false when the product does not fit the two windows
template <int PITCH>
bool tcs_m64_geom(const TcsDims& d, int* r0, int* smid) {
  using G = SG<PITCH>;
  if (d.ntiles != 1) return false;
  const int rows = (d.La + d.Lb - 1 + PITCH - 1) / PITCH;
  if (rows > 80) return false;
  const int R0 = rows > 64 ? 16 : 0;
  int slo, shi;
  tcs_tile_steps<PITCH>(d, 0, slo, shi);
  // live rows of K-step s: those whose 32-byte A window [PITCH m + o, +32), o = ulo + 32 s, meets [0, La)
  auto mlo = [&](int s) { const int o = d.ulo + 32 * s; const int t = -o - 31; return t <= 0 ? 0 : (t + PITCH - 1) / PITCH; };
  auto mhi = [&](int s) { const int o = d.ulo + 32 * s; const int t = d.La - 1 - o; return t < 0 ? -1 : t / PITCH; };
  int sm = slo;
  while (sm < shi && mhi(sm) > 63) sm++;
  for (int s = slo; s < sm; s++)
    if (mlo(s) < R0 || mhi(s) > R0 + 63) return false;
  for (int s = sm; s < shi; s++)
    if (mhi(s) > 63) return false;
  (void)G::N;
  *r0 = R0;
  *smid = sm;
  return true;
}

template <int PITCH>
bool tcs_plan_p(int ma, int mb, int persist, TcsPlan& p) {
  const int mA = ma > mb ? ma : mb, mB = ma > mb ? mb : ma;
  if (mB < 1) return false;
  const TcsDims d = tcs_dims<PITCH>(mA, mB);
  // u32 accumulators: at most 65536 byte products of < 2^16 per sum -> two chains up to 128 KB of b
  if (d.Lb > 131072) return false;
  p.nch = d.Lb > 65536 ? 2 : 1;
  if (persist && 2 * p.nch * PITCH > 512) return false;
  int ksmax = tcs_env("KMX_TCS_KS", 128);
  if (ksmax < 8) ksmax = 8;
  if (ksmax > TCS_KSMAX) ksmax = TCS_KSMAX;
  p.persist = persist;
  p.NS = 0;
  if (persist == 1) {
    if (d.ntiles > TCS_MAXT) return false;
    // three stages of the largest chunk that fits (two when one chunk is the whole K span)
    int NS = tcs_env("KMX_TCS_NS", 3);
    if (NS < 2) NS = 2;
    if (NS > 4) NS = 4;
    const size_t cap = 200 * 1024;
    while (ksmax > 8 && tcsp_smem<PITCH>(d.S < ksmax ? d.S : ksmax, NS) > cap) ksmax -= 8;
    if (tcsp_smem<PITCH>(d.S < ksmax ? d.S : ksmax, NS) > cap) return false;
    p.NS = NS;
  }
  const int nch = (d.S + ksmax - 1) / ksmax;
  const int KS = (d.S + nch - 1) / nch;
  p.pitch = PITCH;
  p.KS = KS;
  p.ntiles = d.ntiles;
  p.smem = persist == 1 ? tcsp_smem<PITCH>(KS, p.NS) : persist == 2 ? tcs_smem64<PITCH>(KS) : tcs_smem<PITCH>(KS);
  long long mmas = 0;
  for (int t = 0; t < d.ntiles; t++) {
    int slo, shi;
    tcs_tile_steps<PITCH>(d, t, slo, shi);
    if (shi > slo) mmas += shi - slo;
  }
  p.mmas = mmas;
  // modelled SM cycles per product: shared-memory operand reads at ~110 B/clk,
  // never below the tensor floor
  double per = (4096.0 + 32.0 * PITCH) / 110.0;
  const double fl = 128.0 * PITCH * 32 / 8192.0;
  if (persist == 2) {
    // M = 64 form: one chunk, no accumulation chains, the row-order buffers inside the table's memory
    int r0, smid;
    if (p.nch != 1 || KS < d.S || !tcs_m64_geom<PITCH>(d, &r0, &smid)) return false;
    if ((size_t)tcs_entries<PITCH>(KS) * 128 < (size_t)2 * SG<PITCH>::LPT * 64 * 8) return false;
    per = (2048.0 + 32.0 * PITCH) / 110.0;
  }
  p.cost = (double)mmas * (per > fl ? per : fl);
  return p.smem <= 200 * 1024;
}

template <int PITCH>
cudaError_t launch_p(const MulArgs& a, const TcsPlan& p, cudaStream_t st, const FinishArgs* fin) {
  TcsArgs ta;
  memset(&ta, 0, sizeof ta);
  ta.m = a;
  ta.KS = p.KS;
  ta.ntiles = p.ntiles;
  ta.NS = p.NS;
  ta.nch = p.nch;
  if (p.persist == 2) {  // M = 64 form (one CTA per product)
    {
      const int mA = a.ma > a.mb ? a.ma : a.mb, mB = a.ma > a.mb ? a.mb : a.ma;
      const TcsDims d = tcs_dims<PITCH>(mA, mB);
      if (fin || !tcs_m64_geom<PITCH>(d, &ta.r0, &ta.smid)) return cudaErrorInvalidValue;
      static size_t s_set3 = 0;
      if (p.smem > 48 * 1024 && p.smem > s_set3) {
        cudaError_t e = cudaFuncSetAttribute(k_tcswz_m64<PITCH>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)p.smem);
        if (e != cudaSuccess) return e;
        s_set3 = p.smem;
      }
      k_tcswz_m64<PITCH><<<(unsigned)a.nprod, 128, p.smem, st>>>(ta);
      return cudaGetLastError();
    }
  }
  if (p.persist) {
    static size_t s_set = 0;
    if (p.smem > 48 * 1024 && p.smem > s_set) {
      cudaError_t e = cudaFuncSetAttribute(k_tcswz_p<PITCH>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)p.smem);
      if (e != cudaSuccess) return e;
      s_set = p.smem;
    }
    // tiles by descending K-steps: the round-robin hands every CTA the same mix
    const int mA = a.ma > a.mb ? a.ma : a.mb, mB = a.ma > a.mb ? a.mb : a.ma;
    const TcsDims d = tcs_dims<PITCH>(mA, mB);
    int steps[TCS_MAXT];
    for (int t = 0; t < p.ntiles; t++) {
      int slo, shi;
      tcs_tile_steps<PITCH>(d, t, slo, shi);
      steps[t] = shi - slo;
      ta.order[t] = (unsigned char)t;
    }
    for (int i = 1; i < p.ntiles; i++)
      for (int j = i; j > 0 && steps[ta.order[j]] > steps[ta.order[j - 1]]; j--) {
        const unsigned char x = ta.order[j];
        ta.order[j] = ta.order[j - 1];
        ta.order[j - 1] = x;
      }
    int per_sm = (int)((220 * 1024) / (p.smem + 1024));
    const int by_tmem = 512 / (2 * p.nch * PITCH);
    if (per_sm > by_tmem) per_sm = by_tmem;
    if (per_sm < 1) per_sm = 1;
    const int cps = tcs_env("KMX_TCS_CPS", 0);
    if (cps > 0 && cps < per_sm) per_sm = cps;
    long long grid = (long long)tcs_num_sms() * per_sm;
    const long long nitems = (long long)a.nprod * p.ntiles;
    if (grid > nitems) grid = nitems;
    k_tcswz_p<PITCH><<<(unsigned)grid, 288, p.smem, st>>>(ta);
    return cudaGetLastError();
  }
  if (fin) {  // one CTA per pair, K3 fused (single-tile products)
    static size_t s_set2 = 0;
    if (p.smem > 48 * 1024 && p.smem > s_set2) {
      cudaError_t e =
          cudaFuncSetAttribute(k_tcswz<PITCH, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)p.smem);
      if (e != cudaSuccess) return e;
      s_set2 = p.smem;
    }
    k_tcswz<PITCH, true><<<(unsigned)(a.nprod / fin->nprod_pair), 128, p.smem, st>>>(ta, *fin);
    return cudaGetLastError();
  }
  static size_t s_set1 = 0;
  if (p.smem > 48 * 1024 && p.smem > s_set1) {
    cudaError_t e = cudaFuncSetAttribute(k_tcswz<PITCH, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)p.smem);
    if (e != cudaSuccess) return e;
    s_set1 = p.smem;
  }
  const long long grid = (long long)a.nprod * p.ntiles;
  FinishArgs nofin;
  memset(&nofin, 0, sizeof nofin);
  k_tcswz<PITCH, false><<<(unsigned)grid, 128, p.smem, st>>>(ta, nofin);
  return cudaGetLastError();
}

}  // namespace

bool tcs_plan(int ma, int mb, int pitch, int persist, TcsPlan& p) {
  switch (pitch) {
    case 32: return tcs_plan_p<32>(ma, mb, persist, p);
    case 64: return tcs_plan_p<64>(ma, mb, persist, p);
    case 128: return tcs_plan_p<128>(ma, mb, persist, p);
    default: return false;
  }
}

cudaError_t launch_tcs(const MulArgs& a, const TcsPlan& p, cudaStream_t st, const FinishArgs* fin) {
  if (a.nprod == 0) return cudaSuccess;
  if (fin && (p.persist != 0 || p.ntiles != 1 || fin->ns > 4 || fin->nprod_pair < 1 || a.nprod % fin->nprod_pair))
    return cudaErrorInvalidValue;
  if (tcs_env("KMX_TC_VERBOSE", 0))
    fprintf(stderr, "kmx_tcs: ma=%d mb=%d nprod=%d -> pitch=%d KS=%d tiles=%d smem=%zu mmas=%lld%s%s NS=%d\n", a.ma, a.mb,
            a.nprod, p.pitch, p.KS, p.ntiles, p.smem, p.mmas, p.persist == 2 ? " M=64 windows" : p.persist ? " persistent" : "",
            fin ? " pair CTAs + fused finish" : "", p.NS);
  switch (p.pitch) {
    case 32: return launch_p<32>(a, p, st, fin);
    case 64: return launch_p<64>(a, p, st, fin);
    default: return launch_p<128>(a, p, st, fin);
  }
}

}  // namespace kmx
