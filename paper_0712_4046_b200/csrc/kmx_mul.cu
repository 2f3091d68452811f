// Batched schoolbook products on the integer pipe (sm_100a).
//
// One engine serves both multiply families of the path:
//   * k_mul  -- multiprecision integer products of the packed operands
//              (bignat.mul / _classical_int, bignat.py:323-380): 32x32->64
//              limb products accumulated in 96-bit column sums, one
//              IMAD.WIDE.U32 (carry-out) + half an IADD3.X per product;
//   * k_conv -- the univariate Z[x] products of the bivariate reductions
//              (UniMul, bipoly.py:23 / oracle.uni_schoolbook :58-69):
//              int32 x int32 -> int64 column sums, one IMAD.WIDE per term.
//
// Geometry.  A warp owns a band of CW consecutive product columns; its 32
// lanes form SPLIT row-groups of LPG = 32/SPLIT lanes, each lane holding 8
// consecutive columns (CW = 8*LPG), and the row-groups split the band's rows
// into SPLIT contiguous slices (partial sums are added across groups at the
// end).  Every warp walks only the rows its own columns need (exact to an
// 8-row block), so the zero-padding work is (CW + 8)/(m + CW) instead of the
// whole CTA's span.  A CTA of 8 warps stages the operand rows/columns its
// bands need in shared memory, TR rows at a time.  The inner loop is an 8x8
// register block: per 64 limb products two broadcast LDS.128 for a and two
// LDS.128 for the sliding b window, whose two 8-word halves swap roles every
// block (no register moves).
#include <cstdlib>

#include "kmx_common.cuh"
#include "kmx_internal.h"

namespace kmx {

// ----------------------------------------------------------- accumulators
struct AccBig {  // 96-bit unsigned column sums
  u32 c0[8], c1[8], c2[8];
  __device__ __forceinline__ void zero() {
#pragma unroll
    for (int r = 0; r < 8; r++) c0[r] = c1[r] = c2[r] = 0u;
  }
  __device__ __forceinline__ void mac(int r, u32 a, u32 b) { mac96(c0[r], c1[r], c2[r], a, b); }
  __device__ __forceinline__ void add_from_lane(int delta) {
#pragma unroll
    for (int r = 0; r < 8; r++) {
      const u32 o0 = __shfl_down_sync(0xffffffffu, c0[r], delta);
      const u32 o1 = __shfl_down_sync(0xffffffffu, c1[r], delta);
      const u32 o2 = __shfl_down_sync(0xffffffffu, c2[r], delta);
      asm("add.cc.u32 %0, %0, %3;\n\taddc.cc.u32 %1, %1, %4;\n\taddc.u32 %2, %2, %5;"
          : "+r"(c0[r]), "+r"(c1[r]), "+r"(c2[r])
          : "r"(o0), "r"(o1), "r"(o2));
    }
  }
};

struct AccI64 {  // signed 64-bit column sums
  long long s[8];
  __device__ __forceinline__ void zero() {
#pragma unroll
    for (int r = 0; r < 8; r++) s[r] = 0;
  }
  __device__ __forceinline__ void mac(int r, u32 a, u32 b) { s[r] += (long long)(int)a * (int)b; }
  __device__ __forceinline__ void add_from_lane(int delta) {
#pragma unroll
    for (int r = 0; r < 8; r++) s[r] += __shfl_down_sync(0xffffffffu, s[r], delta);
  }
};

template <class ACC>
__device__ __forceinline__ void mac_block(ACC& acc, const u32 av[8], const u32 lo[8], const u32 hi[8]) {
  // column r += a[v] * b[k_r - i_v]; window index 7 + r - v
#pragma unroll
  for (int v = 0; v < 8; v++) {
#pragma unroll
    for (int r = 0; r < 8; r++) {
      const int idx = 7 + r - v;
      acc.mac(r, av[v], idx < 8 ? lo[idx] : hi[idx - 8]);
    }
  }
}

__device__ __forceinline__ void lds8(u32 d[8], const u32* p) {
  const uint4 x = reinterpret_cast<const uint4*>(p)[0];
  const uint4 y = reinterpret_cast<const uint4*>(p)[1];
  d[0] = x.x; d[1] = x.y; d[2] = x.z; d[3] = x.w;
  d[4] = y.x; d[5] = y.y; d[6] = y.z; d[7] = y.w;
}

// nblk consecutive 8-row blocks: a rows at ap[0..8*nblk), window of block 0
// at bp[0..16), block t's window at bp[-8t .. -8t+16).
template <class ACC>
__device__ __forceinline__ void walk(ACC& acc, const u32* ap, const u32* bp, int nblk) {
  if (nblk <= 0) return;
  u32 wl[8], wh[8], av[8];
  lds8(wl, bp);
  lds8(wh, bp + 8);
  int t = 0;
  for (; t + 2 <= nblk; t += 2) {
    lds8(av, ap + 8 * t);
    mac_block(acc, av, wl, wh);
    lds8(wh, bp - 8 * (t + 1));      // next window = (wh_new, wl)
    lds8(av, ap + 8 * (t + 1));
    mac_block(acc, av, wh, wl);
    if (t + 2 < nblk) lds8(wl, bp - 8 * (t + 2));  // next window = (wl_new, wh)
  }
  if (t < nblk) {
    lds8(av, ap + 8 * t);
    mac_block(acc, av, wl, wh);
  }
}

// ------------------------------------------------------------------------
// Persistent warp workers.  A work unit is one band (CW columns) of one
// product; every warp repeatedly claims the next unit from a global counter
// (longest-first: bands from the middle of each product outwards, products
// interleaved), stages the operand rows / columns its band needs in its own
// shared-memory slice TR rows at a time (warp-synchronous, no CTA barriers),
// and walks exactly the rows its columns need.
// ------------------------------------------------------------------------
constexpr int MUL_WARPS = 8;

__device__ __forceinline__ int middle_out(int r, int nb) {
  const int mid = (nb - 1) >> 1;
  const int L = mid, R = nb - 1 - mid;
  if (r == 0) return mid;
  const int m0 = L < R ? L : R;
  if (r <= 2 * m0) {
    const int t = (r + 1) >> 1;
    return (r & 1) ? mid + t : mid - t;
  }
  const int k = r - 2 * m0;
  return L > R ? mid - m0 - k : mid + m0 + k;
}

__device__ __forceinline__ void cpa4_zfill(u32* sdst, const u32* gsrc, bool valid) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(sdst);
  const int n = valid ? 4 : 0;  // src-size 0: zero-fill
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(sa), "l"(gsrc), "r"(n));
}

// Skewed band schedule.  Lane p owns columns k = Kw + 8p + r (r < 8) and at
// step t multiplies rows i = t + 8p + v (v < 8): then every lane needs
// b[Kw + r - t - v] -- the same 16-word window for the whole warp (broadcast
// LDS.128), a sliding by 8 per step -- and its own a[t + 8p .. t + 8p + 7],
// and every lane's valid steps are the same interval
//   t in [max(Kw - mb + 1, -8*31), min(Kw + 7, ma - 1)],
// so the warp does no zero-padding work away from the product's ends.
// Steps are staged TR at a time: a[t0 .. t0+TR+256) and b[Kw-t0-TR+1 ..
// Kw-t0+8], double-buffered with cp.async (zero-filled out of range).
constexpr int SK_CW = 256;  // columns per warp band
template <int CW>
__device__ __forceinline__ void stage_skew(u32* buf, const u32* A, int ma, const u32* B, int mb, int Kw, int t0,
                                           int TR, int lane) {
  for (int x = lane; x < TR + CW; x += 32) {
    const int i = t0 + x;
    const bool ok = i >= 0 && i < ma;
    cpa4_zfill(buf + x, ok ? A + i : A, ok);
  }
  const int bbase = Kw - t0 - TR + 1;
  for (int x = lane; x < TR + 8; x += 32) {
    const int j = bbase + x;
    const bool ok = j >= 0 && j < mb;
    cpa4_zfill(buf + TR + CW + x, ok ? B + j : B, ok);
  }
  asm volatile("cp.async.commit_group;");
}

template <class ACC>
__device__ __forceinline__ void warp_band(ACC& acc, const u32* A, int ma, const u32* B, int mb, int Kw, int TR,
                                          u32* wsm) {
  constexpr int CW = SK_CW;
  const int p = threadIdx.x & 31;
  const int bufw = 2 * TR + CW + 8;
  acc.zero();
  int tlo = Kw - (mb - 1);
  if (tlo < -8 * 31) tlo = -8 * 31;
  const int thi = min(Kw + 7, ma - 1);
  if (thi < tlo) return;
  const int nblk = (thi - tlo + 8) >> 3;
  const int TRB = TR >> 3;
  const int nch = (nblk + TRB - 1) / TRB;
  stage_skew<CW>(wsm, A, ma, B, mb, Kw, tlo, TR, p);
  for (int c = 0; c < nch; c++) {
    u32* cur = wsm + (c & 1) * bufw;
    if (c + 1 < nch) {
      stage_skew<CW>(wsm + ((c + 1) & 1) * bufw, A, ma, B, mb, Kw, tlo + (c + 1) * TR, TR, p);
      asm volatile("cp.async.wait_group 1;");
    } else {
      asm volatile("cp.async.wait_group 0;");
    }
    __syncwarp();
    const int n = min(TRB, nblk - c * TRB);
    // a: per lane at cur[8s + 8p]; b window (broadcast) at cur[TR + CW + TR - 8 - 8s]
    walk(acc, cur + 8 * p, cur + TR + CW + TR - 8, n);
    __syncwarp();
  }
}

// ======================================================= bigint products
__global__ void __launch_bounds__(32 * MUL_WARPS) k_mul(MulArgs a) {
  extern __shared__ __align__(16) u32 smem[];
  constexpr int LPG = 32;
  constexpr int CW = SK_CW;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int grp = 0, p = lane;
  u32* wsm = smem + warp * 2 * (2 * a.TI + CW + 8);
  const int mp = a.ma + a.mb;
  const int nunits = a.nprod * a.nbands;
  // single-band products (mp <= CW): equal-cost units, assigned statically
  // (grid-stride over warps) -- no work counter to contend on
  const bool stat = a.nbands == 1;
  int u = stat ? blockIdx.x * MUL_WARPS + warp : 0;
  const int ustep = gridDim.x * MUL_WARPS;
  for (;; u += ustep) {
    if (!stat) {
      if (lane == 0) u = atomicAdd(a.counter, 1);
      u = __shfl_sync(0xffffffffu, u, 0);
    }
    if (u >= nunits) break;
    const int z = u % a.nprod;
    const int bi = middle_out(u / a.nprod, a.nbands);
    const int Kw = bi * CW;
    AccBig acc;
    warp_band(acc, a.A + (long long)z * a.a_stride, a.ma, a.B + (long long)z * a.b_stride, a.mb, Kw, a.TI, wsm);
    // ---- band normalization (group-0 lanes; others compute and discard)
    // digit y_r = c0_r + c1_{r-1} + c2_{r-2} (< 3 * 2^32)
    u32 p_c1 = __shfl_up_sync(0xffffffffu, acc.c1[7], 1, LPG);
    u32 p_c2 = __shfl_up_sync(0xffffffffu, acc.c2[7], 1, LPG);
    u32 p_c2b = __shfl_up_sync(0xffffffffu, acc.c2[6], 1, LPG);
    if (p == 0) p_c1 = p_c2 = p_c2b = 0u;
    u32 lo[8], hi[8];
#pragma unroll
    for (int r = 0; r < 8; r++) {
      const u64 y = (u64)acc.c0[r] + (r >= 1 ? acc.c1[r - 1] : p_c1) +
                    (r >= 2 ? acc.c2[r - 2] : (r == 1 ? p_c2 : p_c2b));
      lo[r] = (u32)y;
      hi[r] = (u32)(y >> 32);
    }
    u32 hprev = __shfl_up_sync(0xffffffffu, hi[7], 1, LPG);
    if (p == 0) hprev = 0u;
    i64 zz[8];
    u32 mr[8], M = CM_IDENT;
#pragma unroll
    for (int r = 0; r < 8; r++) {
      zz[r] = (i64)lo[r] + (r ? hi[r - 1] : hprev);
      mr[r] = cm_make(zz[r]);
      M = cm_compose(M, mr[r]);
    }
    u32 tot;
    const u32 exc = cm_seg_scan(M, LPG, nullptr, &tot);
    int c = cm_apply(exc, 0);
    u32 d[8];
#pragma unroll
    for (int r = 0; r < 8; r++) {
      d[r] = (u32)(zz[r] + c);
      c = cm_apply(mr[r], c);
    }
    if (grp == 0 && Kw < mp) {
      uint4* dst = reinterpret_cast<uint4*>(a.P + (long long)z * a.p_stride + Kw + 8 * p);
      dst[0] = make_uint4(d[0], d[1], d[2], d[3]);
      dst[1] = make_uint4(d[4], d[5], d[6], d[7]);
      if (p == LPG - 1) {
        const i64 s0 = (i64)c + hi[7] + acc.c1[7] + acc.c2[6];
        unsigned long long* sp = a.spill + ((long long)z * a.nbands + bi) * 2;
        sp[0] = (unsigned long long)s0;
        sp[1] = (unsigned long long)acc.c2[7];
      }
    }
  }
}

static int g_num_sms = 0;
static int num_sms() {
  if (!g_num_sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
    if (g_num_sms <= 0) g_num_sms = 148;
  }
  return g_num_sms;
}

template <class KERN>
static cudaError_t launch_persistent(KERN k, size_t smem, long long units, cudaStream_t st, void* args) {
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  int per_sm = 0;
  cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, 32 * MUL_WARPS, smem);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) per_sm = 1;
  long long grid = (long long)num_sms() * per_sm;
  const long long need = (units + MUL_WARPS - 1) / MUL_WARPS;
  if (grid > need) grid = need;
  if (grid < 1) grid = 1;
  void* kargs[] = {args};
  return cudaLaunchKernel((const void*)k, dim3((unsigned)grid), dim3(32 * MUL_WARPS), kargs, smem, st);
}

cudaError_t launch_mul(const MulArgs& a, cudaStream_t st) {
  const size_t smem = (size_t)MUL_WARPS * 2 * (2 * a.TI + SK_CW + 8) * sizeof(u32);
  MulArgs b = a;
  return launch_persistent(k_mul, smem, (long long)a.nprod * a.nbands, st, &b);
}

// tuning overrides (KMX_SPLIT=1|2|4, KMX_TR=rows) for sweeps; defaults below
static int env_int(const char* name, int dflt) {
  const char* v = getenv(name);
  return v && *v ? atoi(v) : dflt;
}

void mul_geometry(int ma, int mb, int* split, int* cw, int* nbands, int* tr) {
  const int m = ma < mb ? ma : mb;
  const int s = 1;
  const int CW = SK_CW;
  const int mp = ma + mb;
  *split = s;
  *cw = CW;
  *nbands = (mp + CW - 1) / CW;
  // rows per staged chunk (double-buffered per warp): the whole row span of a
  // band when it is short; a single-band product (mp <= CW) walks at most
  // max(ma, mb) + 8 steps, so it stages just that
  int T = ((m + CW + 7) & ~7);
  if (mp <= CW) T = ((ma > mb ? ma : mb) + 8 + 7 + 7) & ~7;
  int cap = 512;
  const int te = env_int("KMX_TR", 0);
  if (te >= 8) cap = te & ~7;
  if (T > cap) T = cap;
  *tr = T;
}

// ================================================= univariate Z[x] products
__global__ void __launch_bounds__(32 * MUL_WARPS) k_conv(ConvArgs a) {
  extern __shared__ __align__(16) u32 smem[];
  constexpr int CW = SK_CW;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int grp = 0, p = lane;
  u32* wsm = smem + warp * 2 * (2 * a.TI + CW + 8);
  const int nunits = a.nprod * a.nbands;
  const int kmax = 2 * a.L - 1;
  for (;;) {
    int u = 0;
    if (lane == 0) u = atomicAdd(a.counter, 1);
    u = __shfl_sync(0xffffffffu, u, 0);
    if (u >= nunits) break;
    const int z = u % a.nprod;
    const int bi = middle_out(u / a.nprod, a.nbands);
    const int Kw = bi * CW;
    AccI64 acc;
    warp_band(acc, reinterpret_cast<const u32*>(a.A + (long long)z * a.a_stride), a.L,
              reinterpret_cast<const u32*>(a.B + (long long)z * a.b_stride), a.L, Kw, a.TI, wsm);
    if (grp == 0) {
      int64_t* dst = a.P + (long long)z * a.p_stride + Kw + 8 * p;
#pragma unroll
      for (int r = 0; r < 8; r++)
        if (Kw + 8 * p + r < kmax) dst[r] = acc.s[r];
    }
  }
}

cudaError_t launch_conv(const ConvArgs& a, cudaStream_t st) {
  const size_t smem = (size_t)MUL_WARPS * 2 * (2 * a.TI + SK_CW + 8) * sizeof(u32);
  ConvArgs b = a;
  return launch_persistent(k_conv, smem, (long long)a.nprod * a.nbands, st, &b);
}

}  // namespace kmx
