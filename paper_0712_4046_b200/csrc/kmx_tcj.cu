// kmx_tcj.cu -- K2 on the tensor cores for short products: the byte
// convolution of kmx_tc.cu with the shorter operand cut into J chunks that
// share every MMA.
//
// kmx_tc.cu's tile (M = 128 rows of the sliding operand a, N = 16H shifted
// copies of b) reads a 4 KB A operand from shared memory per MMA and covers
// 2048H output positions; on short operands (c2 ks4: 2436 bytes) N stays
// small and the kernel is paced by those A reads.  Here b = sum_j b_j 256^(j Lbj)
// is split into J chunks of Lbj bytes; column group j of the MMA holds the 16H0
// shifted copies of chunk j, so one MMA (N = 16 H0 J) computes
//
//   D[m][n in group j] = (a * b_j)[alpha_m + beta0_n]   (position + j Lbj in a*b)
//
// for all J chunks at once against the SAME A tile: the K span per product
// shrinks from Lb + BMAX to Lbj + BMAX0, and the A bytes per MAC drop by J.
// One tile covers the whole product (2048 H0 >= La + Lbj).  The chunks are
// staged in shared memory at a pitch P with zero gaps, so the builder's reads
// past a chunk's ends see zeros.  Exactness: a column sum has at most Lbj
// byte products < 2^16 (Lbj <= 65536 -> exact in the u32 accumulator).
//
// Epilogue: the J groups' limb sums (4 consecutive byte positions = 1 limb,
// Lbj is a multiple of 4) are accumulated into a u64 staging array at limb
// offsets j * Lbj / 4, one group per round (positions inside a group are a
// bijection, so a round has no conflicts), then one exact block carry scan
// normalises the product's ma + mb limbs.  No band spills (single tile).
#include <cstdio>
#include <cstdlib>

#include "kmx_common.cuh"
#include "kmx_internal.h"
#include "kmx_tcutil.cuh"

namespace kmx {
namespace {

constexpr int TJ_EPI = 128;
constexpr int TJ_MAXNB = 4;

struct TjShared {
  unsigned long long bar_full[TJ_MAXNB];
  unsigned long long bar_empty[TJ_MAXNB];
  unsigned long long bar_done;
  unsigned long long s_cout[TJ_EPI / 32];
  uint32_t tmem_base;
  uint32_t warp_map[TJ_EPI / 32];
};

struct TjArgs {
  MulArgs m;
  int H0, J, mBj;    // tile width (T = 2048 H0 positions), chunks, limbs per chunk
  int P;             // chunk pitch in the staged b (bytes, multiple of 16)
  int bpad, apad;    // zero padding in front of the staged b / a (bytes, multiple of 16)
  int KC, NB;        // K-steps per ring stage, ring stages
  int ulo, slo, shi; // K-steps u0 = ulo + 32 s, s in [slo, shi)
  int NL;            // staged limbs in the epilogue
  int sa_bytes, sb_bytes;  // staged a / b bytes (with padding)
};

__host__ __device__ inline size_t r128(size_t x) { return (x + 127) & ~(size_t)127; }

template <int NW>
__global__ void __launch_bounds__(32 * NW) k_tcmulj(TjArgs ta) {
  constexpr int THREADS = 32 * NW;
  const MulArgs& a = ta.m;
  extern __shared__ __align__(128) unsigned char tsm[];
  TjShared& sh = *reinterpret_cast<TjShared*>(tsm);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int z = blockIdx.x;
  const int H0 = ta.H0, J = ta.J;
  const int HJ = H0 * J, N = 16 * HJ, STEPB = 32 * N;
  const int KC = ta.KC, NB = ta.NB;

  const bool sw = a.mb > a.ma;  // A slides (longer), B is chunked (shorter)
  const uint32_t* Ag = sw ? a.B + (long long)z * a.b_stride : a.A + (long long)z * a.a_stride;
  const uint32_t* Bg = sw ? a.A + (long long)z * a.a_stride : a.B + (long long)z * a.b_stride;
  const int mA = sw ? a.mb : a.ma, mB = sw ? a.ma : a.mb;
  const int mp = a.ma + a.mb;

  unsigned char* apad = tsm + r128(sizeof(TjShared));
  unsigned char* bpad = apad + r128((size_t)ta.sa_bytes);
  unsigned char* bring = bpad + r128((size_t)ta.sb_bytes);

  uint32_t cols = 32;
  while (cols < (uint32_t)N) cols <<= 1;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&sh.tmem_base)),
                 "r"(cols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    for (int i = 0; i < TJ_MAXNB; i++) {
      mbar_init(smem_u32(&sh.bar_full[i]), THREADS / 32 - 1);
      mbar_init(smem_u32(&sh.bar_empty[i]), 1);
    }
    mbar_init(smem_u32(&sh.bar_done), 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  {
    // a: zero-padded copy; b: J chunks of mBj limbs at pitch P, zero gaps
    uint4* aw = reinterpret_cast<uint4*>(apad);
    const int naq = ta.sa_bytes / 16, a0 = ta.apad / 4;
    const bool al = (mA & 3) == 0 && (reinterpret_cast<uintptr_t>(Ag) & 15) == 0;
    for (int w = tid; w < naq; w += THREADS) {
      const int j = 4 * w - a0;
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
    uint32_t* bw = reinterpret_cast<uint32_t*>(bpad);
    const int nbw = ta.sb_bytes / 4, b0 = ta.bpad / 4, pw = ta.P / 4;
    for (int w = tid; w < nbw; w += THREADS) {
      const int r = w - b0;
      uint32_t v = 0u;
      if (r >= 0) {
        const int c = r / pw, o = r - c * pw;
        const int src = c * ta.mBj + o;
        if (c < J && o < ta.mBj && src < mB) v = __ldg(Bg + src);
      }
      bw[w] = v;
    }
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = sh.tmem_base;
  const int slo = ta.slo, shi = ta.shi;
  const int clo = slo / KC, chi = (shi + KC - 1) / KC;

  if (warp == 0) {
    // ---- MMA issuer (one tile, N = 16 H0 J columns)
    if (lane == 0) {
      const uint32_t idesc = (2u << 4) | ((uint32_t)(N >> 3) << 17) | (8u << 24);
      const uint32_t abase = smem_u32(apad) + (uint32_t)(ta.apad + ta.ulo);
      uint32_t started = 0u;
      for (int c = clo; c < chi; c++) {
        const int k = c - clo, st = k % NB;
        mbar_wait(smem_u32(&sh.bar_full[st]), (uint32_t)((k / NB) & 1));
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const int sb = c * KC;
        const int s0 = max(slo, sb), s1 = min(shi, sb + KC);
        const uint32_t sB = smem_u32(bring + (size_t)st * KC * STEPB);
        for (int s = s0; s < s1; s++) {
          const uint64_t ad = sdesc(abase + 32u * (uint32_t)s, 16, 128u * (uint32_t)H0);
          const uint64_t bd = sdesc(sB + (uint32_t)((s - sb) * STEPB), 128, 256);
          mma_i8(tmem, ad, bd, idesc, started);
          started = 1u;
        }
        mma_commit(smem_u32(&sh.bar_empty[st]));
      }
      mma_commit(smem_u32(&sh.bar_done));
    }
    __syncwarp();
  } else {
    // ---- B builders: item (step, kc, jq), jq = j H0 + jj; lane nl of a
    // half-warp writes row n = nl + 16 jq:
    //   B[n][u0 + 16kc + kk] = b''[j P + 128 jj + nl - u0 - 16kc - kk]
    const int hb = 2 * (warp - 1) + (lane >> 4), nl = lane & 15;
    const int A0 = (13 + nl) >> 2, r0 = (13 + nl) & 3;
    const uint32_t psel = (uint32_t)(r0 + 3) | ((uint32_t)(r0 + 2) << 4) | ((uint32_t)(r0 + 1) << 8) |
                          ((uint32_t)r0 << 12);
    const uint32_t* bw = reinterpret_cast<const uint32_t*>(bpad) + ta.bpad / 4;
    constexpr int NHB = 2 * (THREADS / 32 - 1);
    const int HJ2 = 2 * HJ;
    const uint32_t invH0 = (65536u + (uint32_t)H0 - 1u) / (uint32_t)H0;  // jq / H0 == (jq * invH0) >> 16 (jq < 256)
    for (int c = clo; c < chi; c++) {
      const int k = c - clo, st = k % NB;
      if (k >= NB) mbar_wait(smem_u32(&sh.bar_empty[st]), (uint32_t)(((k / NB) - 1) & 1));
      unsigned char* bb = bring + (size_t)st * KC * STEPB;
      const int sb = c * KC;
      const int s0 = max(slo, sb), s1 = min(shi, sb + KC);
      const int nitems = (s1 - s0) * HJ2;
      // item it = sl * 2HJ + rem, decoded incrementally (no integer division)
      int sl0 = 0, rem0 = hb, sl1 = 0, rem1 = hb + NHB;
      while (rem0 >= HJ2) { rem0 -= HJ2; sl0++; }
      while (rem1 >= HJ2) { rem1 -= HJ2; sl1++; }
      for (int ib = 0; ib < nitems; ib += 2 * NHB) {
        uint32_t wv[2];
        int doff[2];
        bool valid[2];
#pragma unroll
        for (int x = 0; x < 2; x++) {
          const int it = ib + x * NHB + hb;
          valid[x] = it < nitems;
          const int sl = x ? sl1 : sl0;
          const int rem = x ? rem1 : rem0;
          const int kc = rem & 1, jq = rem >> 1;
          const int jc = (int)(((uint32_t)jq * invH0) >> 16), jj = jq - jc * H0;
          const int u0 = ta.ulo + 32 * (s0 + sl);
          const int w0 = jc * ta.P + 128 * jj - u0 - 16 * kc - 16;
          wv[x] = bw[(w0 >> 2) + nl];
          doff[x] = (s0 + sl - sb) * STEPB + 256 * ((nl >> 3) + 2 * jq) + 128 * kc + 16 * (nl & 7);
        }
#pragma unroll
        for (int x = 0; x < 2; x++) {  // advance both items by 2 NHB
          if (x == 0) { rem0 += 2 * NHB; while (rem0 >= HJ2) { rem0 -= HJ2; sl0++; } }
          else { rem1 += 2 * NHB; while (rem1 >= HJ2) { rem1 -= HJ2; sl1++; } }
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

  // ---- epilogue: J rounds of limb sums into the staging array, then one
  // exact block carry scan over the product's mp limbs
  unsigned long long* stg = reinterpret_cast<unsigned long long*>(bring);
  const int NL = ta.NL;
  for (int i = tid; i < NL; i += THREADS) stg[i] = 0ull;
  __syncthreads();
  const bool epi = warp < TJ_EPI / 32;
  const int m = tid;
  const int lbase = epi ? 4 * (m & 7) + 32 * H0 * (m >> 3) : 0;
  for (int jc = 0; jc < J; jc++) {
    if (epi) {
      for (int jj = 0; jj < H0; jj++) {
        uint32_t v[16];
        tmem_ld16(tmem + ((uint32_t)(32 * warp) << 16) + (uint32_t)(16 * (jc * H0 + jj)), v);
        unsigned long long* dst = stg + lbase + 32 * jj + jc * ta.mBj;
#pragma unroll
        for (int q = 0; q < 4; q++)
          dst[q] += (unsigned long long)v[4 * q] + ((unsigned long long)v[4 * q + 1] << 8) +
                    ((unsigned long long)v[4 * q + 2] << 16) + ((unsigned long long)v[4 * q + 3] << 24);
      }
    }
    __syncthreads();
  }
  // thread m owns limbs [R m, R m + R): local digits with carry-in 0
  const int R = (mp + TJ_EPI - 1) / TJ_EPI;
  const int q0 = m * R, q1 = min(mp, q0 + R);
  unsigned long long cout = 0ull, xin = 0ull;
  uint32_t ones = 0xFFFFFFFFu;
  uint32_t d0 = 0u;
  if (epi) {
    unsigned long long x = 0ull;
    for (int q = q0; q < q1; q++) {
      x = (x >> 32) + stg[q];
      stg[q] = (uint32_t)x;
      if (q > q0) ones &= (uint32_t)x;
    }
    cout = x >> 32;
    d0 = q1 > q0 ? (uint32_t)stg[q0] : 0u;
    if (q1 <= q0) ones = 0xFFFFFFFFu;
    xin = __shfl_up_sync(0xffffffffu, cout, 1);
    if (lane == 31) sh.s_cout[warp] = cout;
  }
  __syncthreads();
  uint32_t F = 0u;
  unsigned long long s0 = 0ull;
  if (epi) {
    if (lane == 0) xin = warp ? sh.s_cout[warp - 1] : 0ull;
    // overflow of (D + xin + o) past 2^(32 R), o in {0,1} from the previous thread
    s0 = (unsigned long long)d0 + xin;
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
  uint32_t* Pz = a.P + (long long)z * a.p_stride;
  if (epi) {
    uint32_t E = __shfl_up_sync(0xffffffffu, F, 1);
    uint32_t Wm = CM2_ID;
    for (int w = 0; w < warp; w++) Wm = cm2(sh.warp_map[w], Wm);
    E = lane ? cm2(E, Wm) : Wm;
    unsigned long long acc = s0 + (E & 1u);
    if (q1 > q0) Pz[q0] = (uint32_t)acc;
    for (int q = q0 + 1; q < q1; q++) {
      acc = (acc >> 32) + (uint32_t)stg[q];
      Pz[q] = (uint32_t)acc;
    }
  }
  // single tile: no band spills
  for (int bi = tid; bi < a.nbands; bi += THREADS) {
    unsigned long long* sp = a.spill + ((long long)z * a.nbands + bi) * 2;
    sp[0] = 0ull;
    sp[1] = 0ull;
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(cols));
}

int env_tj(const char* n, int dflt) {
  const char* v = getenv(n);
  return v && *v ? atoi(v) : dflt;
}

struct TjPlan {
  TjArgs t;
  size_t smem;
  double cost;
  int NW;
};

// Geometry for chunk count J and tile width H0; false if infeasible.
bool tj_geometry(int ma, int mb, int H0, int J, TjPlan& p) {
  const int mA = ma > mb ? ma : mb, mB = ma > mb ? mb : ma;
  const int N = 16 * H0 * J;
  if (N > env_tj("KMX_TCJ_NMAX", 128) || J < 1) return false;
  const int mBj = (mB + J - 1) / J;
  if ((J - 1) * mBj >= mB) return false;  // every chunk non-empty
  const int La = 4 * mA, Lbj = 4 * mBj;
  if (Lbj > 65536) return false;           // u32 accumulator exactness
  const int T = 2048 * H0;
  if (La + Lbj > T + 1) return false;      // one tile covers every position
  const int BMAX0 = 15 + 128 * (H0 - 1);
  const int AMAX = 16 * 7 + 128 * H0 * 15;
  TjArgs& t = p.t;
  t.H0 = H0; t.J = J; t.mBj = mBj;
  t.P = (Lbj + BMAX0 + 128 + 15) & ~15;
  t.bpad = (BMAX0 + 160 + 15) & ~15;
  t.apad = (AMAX + 32 + 64 + 15) & ~15;
  t.sa_bytes = ((La + 15) & ~15) + 2 * t.apad;
  t.sb_bytes = t.bpad + J * t.P + t.bpad;
  t.ulo = -32 * ((Lbj - 1 + 31) / 32);
  const int S = fdiv32(BMAX0 - t.ulo) + 1;
  int slo = -fdiv32(AMAX + 31 + t.ulo);
  if (slo < 0) slo = 0;
  int shi = fdiv32(La - 1 - t.ulo) + 1;
  if (shi > S) shi = S;
  t.slo = slo; t.shi = shi;
  t.NL = 512 * H0 + (J - 1) * mBj;
  if (t.NL < ma + mb) t.NL = ma + mb;
  t.NB = env_tj("KMX_TCJ_NB", 2);
  if (t.NB < 2) t.NB = 2;
  if (t.NB > TJ_MAXNB) t.NB = TJ_MAXNB;
  t.KC = env_tj("KMX_TCJ_KC", N >= 256 ? 4 : 8);
  size_t ring = (size_t)t.NB * t.KC * 32 * N;
  if (ring < (size_t)t.NL * 8) ring = (size_t)t.NL * 8;
  p.smem = r128(sizeof(TjShared)) + r128(t.sa_bytes) + r128(t.sb_bytes) + ring;
  if (p.smem > 200 * 1024) return false;
  p.NW = env_tj("KMX_TCJ_NW", 8) == 4 ? 4 : 8;
  // modelled cycles per product: the K-steps, each paced by the larger of the
  // shared-memory operand bytes (A 4 KB + B 32N, ~110 B/clk) and the tensor
  // floor (N/2 cycles), plus the J epilogue rounds
  const int steps = shi - slo;
  const double per = (4096.0 + 32.0 * N) / 110.0 > N / 2.0 ? (4096.0 + 32.0 * N) / 110.0 : N / 2.0;
  p.cost = steps * per + 60.0 * J * H0 + 4.0 * (ma + mb);
  return true;
}

}  // namespace

// Best chunked plan for this shape (KMX_TCJ_H / KMX_TCJ_J force); false if
// none.  short_only: only plans whose chunking actually shortens the K span
// of a short product (H0 <= 2, J >= 3) -- the shapes where the config-5 sweep
// measured a gain over the tiled kernel.
bool tcj_plan(int ma, int mb, double* cost, bool short_only) {
  const int fh = env_tj("KMX_TCJ_H", 0), fj = env_tj("KMX_TCJ_J", 0);
  bool ok = false;
  double best = 0.0;
  for (int H0 : {1, 2, 3, 4, 6, 8}) {
    if (fh && fh != H0) continue;
    for (int J = 1; J <= 16; J++) {
      if (fj && fj != J) continue;
      TjPlan p;
      if (!tj_geometry(ma, mb, H0, J, p)) continue;
      if (!ok || p.cost < best) best = p.cost;
      ok = true;
    }
  }
  if (ok && short_only) {  // the model's best plan must be a short-product one
    ok = false;
    double b2 = 0.0;
    int bh = 0, bj = 0;
    for (int H0 : {1, 2, 3, 4, 6, 8})
      for (int J = 1; J <= 16; J++) {
        TjPlan p;
        if ((fh && fh != H0) || (fj && fj != J) || !tj_geometry(ma, mb, H0, J, p)) continue;
        if (!ok || p.cost < b2) { b2 = p.cost; bh = H0; bj = J; }
        ok = true;
      }
    ok = ok && bh <= 2 && bj >= 3;
  }
  if (cost) *cost = best;
  return ok;
}

cudaError_t launch_tcmulj(const MulArgs& a, cudaStream_t st) {
  const int fh = env_tj("KMX_TCJ_H", 0), fj = env_tj("KMX_TCJ_J", 0);
  TjPlan best;
  bool ok = false;
  for (int H0 : {1, 2, 3, 4, 6, 8}) {
    if (fh && fh != H0) continue;
    for (int J = 1; J <= 16; J++) {
      if (fj && fj != J) continue;
      TjPlan p;
      if (!tj_geometry(a.ma, a.mb, H0, J, p)) continue;
      if (!ok || p.cost < best.cost) best = p;
      ok = true;
    }
  }
  if (!ok) return cudaErrorNotSupported;
  if (a.nprod == 0) return cudaSuccess;
  best.t.m = a;
  if (env_tj("KMX_TC_VERBOSE", 0))
    fprintf(stderr, "kmx_tcj: ma=%d mb=%d nprod=%d -> H0=%d J=%d N=%d mBj=%d KC=%d steps=%d NL=%d smem=%zu NW=%d cost=%.0f\n",
            a.ma, a.mb, a.nprod, best.t.H0, best.t.J, 16 * best.t.H0 * best.t.J, best.t.mBj, best.t.KC,
            best.t.shi - best.t.slo, best.t.NL, best.smem, best.NW, best.cost);
  cudaError_t e;
  if (best.NW == 4) {
    e = cudaFuncSetAttribute(k_tcmulj<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)best.smem);
    if (e != cudaSuccess) return e;
    k_tcmulj<4><<<a.nprod, 128, best.smem, st>>>(best.t);
  } else {
    e = cudaFuncSetAttribute(k_tcmulj<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)best.smem);
    if (e != cudaSuccess) return e;
    k_tcmulj<8><<<a.nprod, 256, best.smem, st>>>(best.t);
  }
  return cudaGetLastError();
}

}  // namespace kmx
